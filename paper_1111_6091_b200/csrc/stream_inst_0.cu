// stream_inst_0.cu -- instantiations of stream_kernel for R = 1..8 (split for parallel builds).
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part0(StreamEntry *t) {
  t[stream_index(1, 1, 0)] = {launch_stream_t<1, 1, 0>, (const void *)stream_kernel<1, 1, 0>};
  t[stream_index(1, 1, 1)] = {launch_stream_t<1, 1, 1>, (const void *)stream_kernel<1, 1, 1>};
  t[stream_index(1, 2, 0)] = {launch_stream_t<1, 2, 0>, (const void *)stream_kernel<1, 2, 0>};
  t[stream_index(1, 2, 1)] = {launch_stream_t<1, 2, 1>, (const void *)stream_kernel<1, 2, 1>};
  t[stream_index(1, 4, 0)] = {launch_stream_t<1, 4, 0>, (const void *)stream_kernel<1, 4, 0>};
  t[stream_index(1, 4, 1)] = {launch_stream_t<1, 4, 1>, (const void *)stream_kernel<1, 4, 1>};
  t[stream_index(1, 8, 0)] = {launch_stream_t<1, 8, 0>, (const void *)stream_kernel<1, 8, 0>};
  t[stream_index(2, 1, 0)] = {launch_stream_t<2, 1, 0>, (const void *)stream_kernel<2, 1, 0>};
  t[stream_index(2, 1, 1)] = {launch_stream_t<2, 1, 1>, (const void *)stream_kernel<2, 1, 1>};
  t[stream_index(2, 2, 0)] = {launch_stream_t<2, 2, 0>, (const void *)stream_kernel<2, 2, 0>};
  t[stream_index(2, 2, 1)] = {launch_stream_t<2, 2, 1>, (const void *)stream_kernel<2, 2, 1>};
  t[stream_index(2, 4, 0)] = {launch_stream_t<2, 4, 0>, (const void *)stream_kernel<2, 4, 0>};
  t[stream_index(2, 4, 1)] = {launch_stream_t<2, 4, 1>, (const void *)stream_kernel<2, 4, 1>};
  t[stream_index(2, 8, 0)] = {launch_stream_t<2, 8, 0>, (const void *)stream_kernel<2, 8, 0>};
  t[stream_index(3, 1, 0)] = {launch_stream_t<3, 1, 0>, (const void *)stream_kernel<3, 1, 0>};
  t[stream_index(3, 1, 1)] = {launch_stream_t<3, 1, 1>, (const void *)stream_kernel<3, 1, 1>};
  t[stream_index(3, 2, 0)] = {launch_stream_t<3, 2, 0>, (const void *)stream_kernel<3, 2, 0>};
  t[stream_index(3, 2, 1)] = {launch_stream_t<3, 2, 1>, (const void *)stream_kernel<3, 2, 1>};
  t[stream_index(3, 4, 0)] = {launch_stream_t<3, 4, 0>, (const void *)stream_kernel<3, 4, 0>};
  t[stream_index(3, 4, 1)] = {launch_stream_t<3, 4, 1>, (const void *)stream_kernel<3, 4, 1>};
  t[stream_index(3, 8, 0)] = {launch_stream_t<3, 8, 0>, (const void *)stream_kernel<3, 8, 0>};
  t[stream_index(4, 1, 0)] = {launch_stream_t<4, 1, 0>, (const void *)stream_kernel<4, 1, 0>};
  t[stream_index(4, 1, 1)] = {launch_stream_t<4, 1, 1>, (const void *)stream_kernel<4, 1, 1>};
  t[stream_index(4, 2, 0)] = {launch_stream_t<4, 2, 0>, (const void *)stream_kernel<4, 2, 0>};
  t[stream_index(4, 2, 1)] = {launch_stream_t<4, 2, 1>, (const void *)stream_kernel<4, 2, 1>};
  t[stream_index(4, 4, 0)] = {launch_stream_t<4, 4, 0>, (const void *)stream_kernel<4, 4, 0>};
  t[stream_index(4, 4, 1)] = {launch_stream_t<4, 4, 1>, (const void *)stream_kernel<4, 4, 1>};
  t[stream_index(4, 8, 0)] = {launch_stream_t<4, 8, 0>, (const void *)stream_kernel<4, 8, 0>};
  t[stream_index(5, 1, 0)] = {launch_stream_t<5, 1, 0>, (const void *)stream_kernel<5, 1, 0>};
  t[stream_index(5, 1, 1)] = {launch_stream_t<5, 1, 1>, (const void *)stream_kernel<5, 1, 1>};
  t[stream_index(5, 2, 0)] = {launch_stream_t<5, 2, 0>, (const void *)stream_kernel<5, 2, 0>};
  t[stream_index(5, 2, 1)] = {launch_stream_t<5, 2, 1>, (const void *)stream_kernel<5, 2, 1>};
  t[stream_index(5, 4, 0)] = {launch_stream_t<5, 4, 0>, (const void *)stream_kernel<5, 4, 0>};
  t[stream_index(5, 4, 1)] = {launch_stream_t<5, 4, 1>, (const void *)stream_kernel<5, 4, 1>};
  t[stream_index(5, 8, 0)] = {launch_stream_t<5, 8, 0>, (const void *)stream_kernel<5, 8, 0>};
  t[stream_index(6, 1, 0)] = {launch_stream_t<6, 1, 0>, (const void *)stream_kernel<6, 1, 0>};
  t[stream_index(6, 1, 1)] = {launch_stream_t<6, 1, 1>, (const void *)stream_kernel<6, 1, 1>};
  t[stream_index(6, 2, 0)] = {launch_stream_t<6, 2, 0>, (const void *)stream_kernel<6, 2, 0>};
  t[stream_index(6, 2, 1)] = {launch_stream_t<6, 2, 1>, (const void *)stream_kernel<6, 2, 1>};
  t[stream_index(6, 4, 0)] = {launch_stream_t<6, 4, 0>, (const void *)stream_kernel<6, 4, 0>};
  t[stream_index(6, 4, 1)] = {launch_stream_t<6, 4, 1>, (const void *)stream_kernel<6, 4, 1>};
  t[stream_index(6, 8, 0)] = {launch_stream_t<6, 8, 0>, (const void *)stream_kernel<6, 8, 0>};
  t[stream_index(7, 1, 0)] = {launch_stream_t<7, 1, 0>, (const void *)stream_kernel<7, 1, 0>};
  t[stream_index(7, 1, 1)] = {launch_stream_t<7, 1, 1>, (const void *)stream_kernel<7, 1, 1>};
  t[stream_index(7, 2, 0)] = {launch_stream_t<7, 2, 0>, (const void *)stream_kernel<7, 2, 0>};
  t[stream_index(7, 2, 1)] = {launch_stream_t<7, 2, 1>, (const void *)stream_kernel<7, 2, 1>};
  t[stream_index(7, 4, 0)] = {launch_stream_t<7, 4, 0>, (const void *)stream_kernel<7, 4, 0>};
  t[stream_index(7, 4, 1)] = {launch_stream_t<7, 4, 1>, (const void *)stream_kernel<7, 4, 1>};
  t[stream_index(7, 8, 0)] = {launch_stream_t<7, 8, 0>, (const void *)stream_kernel<7, 8, 0>};
  t[stream_index(8, 1, 0)] = {launch_stream_t<8, 1, 0>, (const void *)stream_kernel<8, 1, 0>};
  t[stream_index(8, 1, 1)] = {launch_stream_t<8, 1, 1>, (const void *)stream_kernel<8, 1, 1>};
  t[stream_index(8, 2, 0)] = {launch_stream_t<8, 2, 0>, (const void *)stream_kernel<8, 2, 0>};
  t[stream_index(8, 2, 1)] = {launch_stream_t<8, 2, 1>, (const void *)stream_kernel<8, 2, 1>};
  t[stream_index(8, 4, 0)] = {launch_stream_t<8, 4, 0>, (const void *)stream_kernel<8, 4, 0>};
  t[stream_index(8, 4, 1)] = {launch_stream_t<8, 4, 1>, (const void *)stream_kernel<8, 4, 1>};
  t[stream_index(8, 8, 0)] = {launch_stream_t<8, 8, 0>, (const void *)stream_kernel<8, 8, 0>};
}
}  // namespace cpk
