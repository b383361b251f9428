// stream_inst_1.cu -- instantiations of stream_kernel for R = 9..16 (split for parallel builds).
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part1(StreamEntry *t) {
  t[stream_index(9, 1, 0)] = {launch_stream_t<9, 1, 0>, (const void *)stream_kernel<9, 1, 0>};
  t[stream_index(9, 1, 1)] = {launch_stream_t<9, 1, 1>, (const void *)stream_kernel<9, 1, 1>};
  t[stream_index(9, 2, 0)] = {launch_stream_t<9, 2, 0>, (const void *)stream_kernel<9, 2, 0>};
  t[stream_index(9, 2, 1)] = {launch_stream_t<9, 2, 1>, (const void *)stream_kernel<9, 2, 1>};
  t[stream_index(9, 4, 0)] = {launch_stream_t<9, 4, 0>, (const void *)stream_kernel<9, 4, 0>};
  t[stream_index(9, 4, 1)] = {launch_stream_t<9, 4, 1>, (const void *)stream_kernel<9, 4, 1>};
  t[stream_index(9, 8, 0)] = {launch_stream_t<9, 8, 0>, (const void *)stream_kernel<9, 8, 0>};
  t[stream_index(10, 1, 0)] = {launch_stream_t<10, 1, 0>, (const void *)stream_kernel<10, 1, 0>};
  t[stream_index(10, 1, 1)] = {launch_stream_t<10, 1, 1>, (const void *)stream_kernel<10, 1, 1>};
  t[stream_index(10, 2, 0)] = {launch_stream_t<10, 2, 0>, (const void *)stream_kernel<10, 2, 0>};
  t[stream_index(10, 2, 1)] = {launch_stream_t<10, 2, 1>, (const void *)stream_kernel<10, 2, 1>};
  t[stream_index(10, 4, 0)] = {launch_stream_t<10, 4, 0>, (const void *)stream_kernel<10, 4, 0>};
  t[stream_index(10, 4, 1)] = {launch_stream_t<10, 4, 1>, (const void *)stream_kernel<10, 4, 1>};
  t[stream_index(10, 8, 0)] = {launch_stream_t<10, 8, 0>, (const void *)stream_kernel<10, 8, 0>};
  t[stream_index(11, 1, 0)] = {launch_stream_t<11, 1, 0>, (const void *)stream_kernel<11, 1, 0>};
  t[stream_index(11, 1, 1)] = {launch_stream_t<11, 1, 1>, (const void *)stream_kernel<11, 1, 1>};
  t[stream_index(11, 2, 0)] = {launch_stream_t<11, 2, 0>, (const void *)stream_kernel<11, 2, 0>};
  t[stream_index(11, 2, 1)] = {launch_stream_t<11, 2, 1>, (const void *)stream_kernel<11, 2, 1>};
  t[stream_index(11, 4, 0)] = {launch_stream_t<11, 4, 0>, (const void *)stream_kernel<11, 4, 0>};
  t[stream_index(11, 4, 1)] = {launch_stream_t<11, 4, 1>, (const void *)stream_kernel<11, 4, 1>};
  t[stream_index(11, 8, 0)] = {launch_stream_t<11, 8, 0>, (const void *)stream_kernel<11, 8, 0>};
  t[stream_index(12, 1, 0)] = {launch_stream_t<12, 1, 0>, (const void *)stream_kernel<12, 1, 0>};
  t[stream_index(12, 1, 1)] = {launch_stream_t<12, 1, 1>, (const void *)stream_kernel<12, 1, 1>};
  t[stream_index(12, 2, 0)] = {launch_stream_t<12, 2, 0>, (const void *)stream_kernel<12, 2, 0>};
  t[stream_index(12, 2, 1)] = {launch_stream_t<12, 2, 1>, (const void *)stream_kernel<12, 2, 1>};
  t[stream_index(12, 4, 0)] = {launch_stream_t<12, 4, 0>, (const void *)stream_kernel<12, 4, 0>};
  t[stream_index(12, 4, 1)] = {launch_stream_t<12, 4, 1>, (const void *)stream_kernel<12, 4, 1>};
  t[stream_index(12, 8, 0)] = {launch_stream_t<12, 8, 0>, (const void *)stream_kernel<12, 8, 0>};
  t[stream_index(13, 1, 0)] = {launch_stream_t<13, 1, 0>, (const void *)stream_kernel<13, 1, 0>};
  t[stream_index(13, 1, 1)] = {launch_stream_t<13, 1, 1>, (const void *)stream_kernel<13, 1, 1>};
  t[stream_index(13, 2, 0)] = {launch_stream_t<13, 2, 0>, (const void *)stream_kernel<13, 2, 0>};
  t[stream_index(13, 2, 1)] = {launch_stream_t<13, 2, 1>, (const void *)stream_kernel<13, 2, 1>};
  t[stream_index(13, 4, 0)] = {launch_stream_t<13, 4, 0>, (const void *)stream_kernel<13, 4, 0>};
  t[stream_index(13, 4, 1)] = {launch_stream_t<13, 4, 1>, (const void *)stream_kernel<13, 4, 1>};
  t[stream_index(13, 8, 0)] = {launch_stream_t<13, 8, 0>, (const void *)stream_kernel<13, 8, 0>};
  t[stream_index(14, 1, 0)] = {launch_stream_t<14, 1, 0>, (const void *)stream_kernel<14, 1, 0>};
  t[stream_index(14, 1, 1)] = {launch_stream_t<14, 1, 1>, (const void *)stream_kernel<14, 1, 1>};
  t[stream_index(14, 2, 0)] = {launch_stream_t<14, 2, 0>, (const void *)stream_kernel<14, 2, 0>};
  t[stream_index(14, 2, 1)] = {launch_stream_t<14, 2, 1>, (const void *)stream_kernel<14, 2, 1>};
  t[stream_index(14, 4, 0)] = {launch_stream_t<14, 4, 0>, (const void *)stream_kernel<14, 4, 0>};
  t[stream_index(14, 4, 1)] = {launch_stream_t<14, 4, 1>, (const void *)stream_kernel<14, 4, 1>};
  t[stream_index(14, 8, 0)] = {launch_stream_t<14, 8, 0>, (const void *)stream_kernel<14, 8, 0>};
  t[stream_index(15, 1, 0)] = {launch_stream_t<15, 1, 0>, (const void *)stream_kernel<15, 1, 0>};
  t[stream_index(15, 1, 1)] = {launch_stream_t<15, 1, 1>, (const void *)stream_kernel<15, 1, 1>};
  t[stream_index(15, 2, 0)] = {launch_stream_t<15, 2, 0>, (const void *)stream_kernel<15, 2, 0>};
  t[stream_index(15, 2, 1)] = {launch_stream_t<15, 2, 1>, (const void *)stream_kernel<15, 2, 1>};
  t[stream_index(15, 4, 0)] = {launch_stream_t<15, 4, 0>, (const void *)stream_kernel<15, 4, 0>};
  t[stream_index(15, 4, 1)] = {launch_stream_t<15, 4, 1>, (const void *)stream_kernel<15, 4, 1>};
  t[stream_index(15, 8, 0)] = {launch_stream_t<15, 8, 0>, (const void *)stream_kernel<15, 8, 0>};
  t[stream_index(16, 1, 0)] = {launch_stream_t<16, 1, 0>, (const void *)stream_kernel<16, 1, 0>};
  t[stream_index(16, 1, 1)] = {launch_stream_t<16, 1, 1>, (const void *)stream_kernel<16, 1, 1>};
  t[stream_index(16, 2, 0)] = {launch_stream_t<16, 2, 0>, (const void *)stream_kernel<16, 2, 0>};
  t[stream_index(16, 2, 1)] = {launch_stream_t<16, 2, 1>, (const void *)stream_kernel<16, 2, 1>};
  t[stream_index(16, 4, 0)] = {launch_stream_t<16, 4, 0>, (const void *)stream_kernel<16, 4, 0>};
  t[stream_index(16, 4, 1)] = {launch_stream_t<16, 4, 1>, (const void *)stream_kernel<16, 4, 1>};
  t[stream_index(16, 8, 0)] = {launch_stream_t<16, 8, 0>, (const void *)stream_kernel<16, 8, 0>};
}
}  // namespace cpk
