// stream_inst_2.cu -- instantiations of stream_kernel for R = 17..24 (split for parallel builds).
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part2(StreamEntry *t) {
  t[stream_index(17, 1, 0)] = {launch_stream_t<17, 1, 0>, (const void *)stream_kernel<17, 1, 0>};
  t[stream_index(17, 1, 1)] = {launch_stream_t<17, 1, 1>, (const void *)stream_kernel<17, 1, 1>};
  t[stream_index(17, 2, 0)] = {launch_stream_t<17, 2, 0>, (const void *)stream_kernel<17, 2, 0>};
  t[stream_index(17, 2, 1)] = {launch_stream_t<17, 2, 1>, (const void *)stream_kernel<17, 2, 1>};
  t[stream_index(17, 4, 0)] = {launch_stream_t<17, 4, 0>, (const void *)stream_kernel<17, 4, 0>};
  t[stream_index(17, 4, 1)] = {launch_stream_t<17, 4, 1>, (const void *)stream_kernel<17, 4, 1>};
  t[stream_index(17, 8, 0)] = {launch_stream_t<17, 8, 0>, (const void *)stream_kernel<17, 8, 0>};
  t[stream_index(18, 1, 0)] = {launch_stream_t<18, 1, 0>, (const void *)stream_kernel<18, 1, 0>};
  t[stream_index(18, 1, 1)] = {launch_stream_t<18, 1, 1>, (const void *)stream_kernel<18, 1, 1>};
  t[stream_index(18, 2, 0)] = {launch_stream_t<18, 2, 0>, (const void *)stream_kernel<18, 2, 0>};
  t[stream_index(18, 2, 1)] = {launch_stream_t<18, 2, 1>, (const void *)stream_kernel<18, 2, 1>};
  t[stream_index(18, 4, 0)] = {launch_stream_t<18, 4, 0>, (const void *)stream_kernel<18, 4, 0>};
  t[stream_index(18, 4, 1)] = {launch_stream_t<18, 4, 1>, (const void *)stream_kernel<18, 4, 1>};
  t[stream_index(18, 8, 0)] = {launch_stream_t<18, 8, 0>, (const void *)stream_kernel<18, 8, 0>};
  t[stream_index(19, 1, 0)] = {launch_stream_t<19, 1, 0>, (const void *)stream_kernel<19, 1, 0>};
  t[stream_index(19, 1, 1)] = {launch_stream_t<19, 1, 1>, (const void *)stream_kernel<19, 1, 1>};
  t[stream_index(19, 2, 0)] = {launch_stream_t<19, 2, 0>, (const void *)stream_kernel<19, 2, 0>};
  t[stream_index(19, 2, 1)] = {launch_stream_t<19, 2, 1>, (const void *)stream_kernel<19, 2, 1>};
  t[stream_index(19, 4, 0)] = {launch_stream_t<19, 4, 0>, (const void *)stream_kernel<19, 4, 0>};
  t[stream_index(19, 4, 1)] = {launch_stream_t<19, 4, 1>, (const void *)stream_kernel<19, 4, 1>};
  t[stream_index(19, 8, 0)] = {launch_stream_t<19, 8, 0>, (const void *)stream_kernel<19, 8, 0>};
  t[stream_index(20, 1, 0)] = {launch_stream_t<20, 1, 0>, (const void *)stream_kernel<20, 1, 0>};
  t[stream_index(20, 1, 1)] = {launch_stream_t<20, 1, 1>, (const void *)stream_kernel<20, 1, 1>};
  t[stream_index(20, 2, 0)] = {launch_stream_t<20, 2, 0>, (const void *)stream_kernel<20, 2, 0>};
  t[stream_index(20, 2, 1)] = {launch_stream_t<20, 2, 1>, (const void *)stream_kernel<20, 2, 1>};
  t[stream_index(20, 4, 0)] = {launch_stream_t<20, 4, 0>, (const void *)stream_kernel<20, 4, 0>};
  t[stream_index(20, 4, 1)] = {launch_stream_t<20, 4, 1>, (const void *)stream_kernel<20, 4, 1>};
  t[stream_index(20, 8, 0)] = {launch_stream_t<20, 8, 0>, (const void *)stream_kernel<20, 8, 0>};
  t[stream_index(21, 1, 0)] = {launch_stream_t<21, 1, 0>, (const void *)stream_kernel<21, 1, 0>};
  t[stream_index(21, 1, 1)] = {launch_stream_t<21, 1, 1>, (const void *)stream_kernel<21, 1, 1>};
  t[stream_index(21, 2, 0)] = {launch_stream_t<21, 2, 0>, (const void *)stream_kernel<21, 2, 0>};
  t[stream_index(21, 2, 1)] = {launch_stream_t<21, 2, 1>, (const void *)stream_kernel<21, 2, 1>};
  t[stream_index(21, 4, 0)] = {launch_stream_t<21, 4, 0>, (const void *)stream_kernel<21, 4, 0>};
  t[stream_index(21, 4, 1)] = {launch_stream_t<21, 4, 1>, (const void *)stream_kernel<21, 4, 1>};
  t[stream_index(21, 8, 0)] = {launch_stream_t<21, 8, 0>, (const void *)stream_kernel<21, 8, 0>};
  t[stream_index(22, 1, 0)] = {launch_stream_t<22, 1, 0>, (const void *)stream_kernel<22, 1, 0>};
  t[stream_index(22, 1, 1)] = {launch_stream_t<22, 1, 1>, (const void *)stream_kernel<22, 1, 1>};
  t[stream_index(22, 2, 0)] = {launch_stream_t<22, 2, 0>, (const void *)stream_kernel<22, 2, 0>};
  t[stream_index(22, 2, 1)] = {launch_stream_t<22, 2, 1>, (const void *)stream_kernel<22, 2, 1>};
  t[stream_index(22, 4, 0)] = {launch_stream_t<22, 4, 0>, (const void *)stream_kernel<22, 4, 0>};
  t[stream_index(22, 4, 1)] = {launch_stream_t<22, 4, 1>, (const void *)stream_kernel<22, 4, 1>};
  t[stream_index(22, 8, 0)] = {launch_stream_t<22, 8, 0>, (const void *)stream_kernel<22, 8, 0>};
  t[stream_index(23, 1, 0)] = {launch_stream_t<23, 1, 0>, (const void *)stream_kernel<23, 1, 0>};
  t[stream_index(23, 1, 1)] = {launch_stream_t<23, 1, 1>, (const void *)stream_kernel<23, 1, 1>};
  t[stream_index(23, 2, 0)] = {launch_stream_t<23, 2, 0>, (const void *)stream_kernel<23, 2, 0>};
  t[stream_index(23, 2, 1)] = {launch_stream_t<23, 2, 1>, (const void *)stream_kernel<23, 2, 1>};
  t[stream_index(23, 4, 0)] = {launch_stream_t<23, 4, 0>, (const void *)stream_kernel<23, 4, 0>};
  t[stream_index(23, 4, 1)] = {launch_stream_t<23, 4, 1>, (const void *)stream_kernel<23, 4, 1>};
  t[stream_index(23, 8, 0)] = {launch_stream_t<23, 8, 0>, (const void *)stream_kernel<23, 8, 0>};
  t[stream_index(24, 1, 0)] = {launch_stream_t<24, 1, 0>, (const void *)stream_kernel<24, 1, 0>};
  t[stream_index(24, 1, 1)] = {launch_stream_t<24, 1, 1>, (const void *)stream_kernel<24, 1, 1>};
  t[stream_index(24, 2, 0)] = {launch_stream_t<24, 2, 0>, (const void *)stream_kernel<24, 2, 0>};
  t[stream_index(24, 2, 1)] = {launch_stream_t<24, 2, 1>, (const void *)stream_kernel<24, 2, 1>};
  t[stream_index(24, 4, 0)] = {launch_stream_t<24, 4, 0>, (const void *)stream_kernel<24, 4, 0>};
  t[stream_index(24, 4, 1)] = {launch_stream_t<24, 4, 1>, (const void *)stream_kernel<24, 4, 1>};
  t[stream_index(24, 8, 0)] = {launch_stream_t<24, 8, 0>, (const void *)stream_kernel<24, 8, 0>};
}
}  // namespace cpk
