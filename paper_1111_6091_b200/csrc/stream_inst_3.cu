// stream_inst_3.cu -- instantiations of stream_kernel for R = 25..32 (split for parallel builds).
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part3(StreamEntry *t) {
  t[stream_index(25, 1, 0)] = {launch_stream_t<25, 1, 0>, (const void *)stream_kernel<25, 1, 0>};
  t[stream_index(25, 1, 1)] = {launch_stream_t<25, 1, 1>, (const void *)stream_kernel<25, 1, 1>};
  t[stream_index(25, 2, 0)] = {launch_stream_t<25, 2, 0>, (const void *)stream_kernel<25, 2, 0>};
  t[stream_index(25, 2, 1)] = {launch_stream_t<25, 2, 1>, (const void *)stream_kernel<25, 2, 1>};
  t[stream_index(25, 4, 0)] = {launch_stream_t<25, 4, 0>, (const void *)stream_kernel<25, 4, 0>};
  t[stream_index(25, 4, 1)] = {launch_stream_t<25, 4, 1>, (const void *)stream_kernel<25, 4, 1>};
  t[stream_index(25, 8, 0)] = {launch_stream_t<25, 8, 0>, (const void *)stream_kernel<25, 8, 0>};
  t[stream_index(26, 1, 0)] = {launch_stream_t<26, 1, 0>, (const void *)stream_kernel<26, 1, 0>};
  t[stream_index(26, 1, 1)] = {launch_stream_t<26, 1, 1>, (const void *)stream_kernel<26, 1, 1>};
  t[stream_index(26, 2, 0)] = {launch_stream_t<26, 2, 0>, (const void *)stream_kernel<26, 2, 0>};
  t[stream_index(26, 2, 1)] = {launch_stream_t<26, 2, 1>, (const void *)stream_kernel<26, 2, 1>};
  t[stream_index(26, 4, 0)] = {launch_stream_t<26, 4, 0>, (const void *)stream_kernel<26, 4, 0>};
  t[stream_index(26, 4, 1)] = {launch_stream_t<26, 4, 1>, (const void *)stream_kernel<26, 4, 1>};
  t[stream_index(26, 8, 0)] = {launch_stream_t<26, 8, 0>, (const void *)stream_kernel<26, 8, 0>};
  t[stream_index(27, 1, 0)] = {launch_stream_t<27, 1, 0>, (const void *)stream_kernel<27, 1, 0>};
  t[stream_index(27, 1, 1)] = {launch_stream_t<27, 1, 1>, (const void *)stream_kernel<27, 1, 1>};
  t[stream_index(27, 2, 0)] = {launch_stream_t<27, 2, 0>, (const void *)stream_kernel<27, 2, 0>};
  t[stream_index(27, 2, 1)] = {launch_stream_t<27, 2, 1>, (const void *)stream_kernel<27, 2, 1>};
  t[stream_index(27, 4, 0)] = {launch_stream_t<27, 4, 0>, (const void *)stream_kernel<27, 4, 0>};
  t[stream_index(27, 4, 1)] = {launch_stream_t<27, 4, 1>, (const void *)stream_kernel<27, 4, 1>};
  t[stream_index(27, 8, 0)] = {launch_stream_t<27, 8, 0>, (const void *)stream_kernel<27, 8, 0>};
  t[stream_index(28, 1, 0)] = {launch_stream_t<28, 1, 0>, (const void *)stream_kernel<28, 1, 0>};
  t[stream_index(28, 1, 1)] = {launch_stream_t<28, 1, 1>, (const void *)stream_kernel<28, 1, 1>};
  t[stream_index(28, 2, 0)] = {launch_stream_t<28, 2, 0>, (const void *)stream_kernel<28, 2, 0>};
  t[stream_index(28, 2, 1)] = {launch_stream_t<28, 2, 1>, (const void *)stream_kernel<28, 2, 1>};
  t[stream_index(28, 4, 0)] = {launch_stream_t<28, 4, 0>, (const void *)stream_kernel<28, 4, 0>};
  t[stream_index(28, 4, 1)] = {launch_stream_t<28, 4, 1>, (const void *)stream_kernel<28, 4, 1>};
  t[stream_index(28, 8, 0)] = {launch_stream_t<28, 8, 0>, (const void *)stream_kernel<28, 8, 0>};
  t[stream_index(29, 1, 0)] = {launch_stream_t<29, 1, 0>, (const void *)stream_kernel<29, 1, 0>};
  t[stream_index(29, 1, 1)] = {launch_stream_t<29, 1, 1>, (const void *)stream_kernel<29, 1, 1>};
  t[stream_index(29, 2, 0)] = {launch_stream_t<29, 2, 0>, (const void *)stream_kernel<29, 2, 0>};
  t[stream_index(29, 2, 1)] = {launch_stream_t<29, 2, 1>, (const void *)stream_kernel<29, 2, 1>};
  t[stream_index(29, 4, 0)] = {launch_stream_t<29, 4, 0>, (const void *)stream_kernel<29, 4, 0>};
  t[stream_index(29, 4, 1)] = {launch_stream_t<29, 4, 1>, (const void *)stream_kernel<29, 4, 1>};
  t[stream_index(29, 8, 0)] = {launch_stream_t<29, 8, 0>, (const void *)stream_kernel<29, 8, 0>};
  t[stream_index(30, 1, 0)] = {launch_stream_t<30, 1, 0>, (const void *)stream_kernel<30, 1, 0>};
  t[stream_index(30, 1, 1)] = {launch_stream_t<30, 1, 1>, (const void *)stream_kernel<30, 1, 1>};
  t[stream_index(30, 2, 0)] = {launch_stream_t<30, 2, 0>, (const void *)stream_kernel<30, 2, 0>};
  t[stream_index(30, 2, 1)] = {launch_stream_t<30, 2, 1>, (const void *)stream_kernel<30, 2, 1>};
  t[stream_index(30, 4, 0)] = {launch_stream_t<30, 4, 0>, (const void *)stream_kernel<30, 4, 0>};
  t[stream_index(30, 4, 1)] = {launch_stream_t<30, 4, 1>, (const void *)stream_kernel<30, 4, 1>};
  t[stream_index(30, 8, 0)] = {launch_stream_t<30, 8, 0>, (const void *)stream_kernel<30, 8, 0>};
  t[stream_index(31, 1, 0)] = {launch_stream_t<31, 1, 0>, (const void *)stream_kernel<31, 1, 0>};
  t[stream_index(31, 1, 1)] = {launch_stream_t<31, 1, 1>, (const void *)stream_kernel<31, 1, 1>};
  t[stream_index(31, 2, 0)] = {launch_stream_t<31, 2, 0>, (const void *)stream_kernel<31, 2, 0>};
  t[stream_index(31, 2, 1)] = {launch_stream_t<31, 2, 1>, (const void *)stream_kernel<31, 2, 1>};
  t[stream_index(31, 4, 0)] = {launch_stream_t<31, 4, 0>, (const void *)stream_kernel<31, 4, 0>};
  t[stream_index(31, 4, 1)] = {launch_stream_t<31, 4, 1>, (const void *)stream_kernel<31, 4, 1>};
  t[stream_index(31, 8, 0)] = {launch_stream_t<31, 8, 0>, (const void *)stream_kernel<31, 8, 0>};
  t[stream_index(32, 1, 0)] = {launch_stream_t<32, 1, 0>, (const void *)stream_kernel<32, 1, 0>};
  t[stream_index(32, 1, 1)] = {launch_stream_t<32, 1, 1>, (const void *)stream_kernel<32, 1, 1>};
  t[stream_index(32, 2, 0)] = {launch_stream_t<32, 2, 0>, (const void *)stream_kernel<32, 2, 0>};
  t[stream_index(32, 2, 1)] = {launch_stream_t<32, 2, 1>, (const void *)stream_kernel<32, 2, 1>};
  t[stream_index(32, 4, 0)] = {launch_stream_t<32, 4, 0>, (const void *)stream_kernel<32, 4, 0>};
  t[stream_index(32, 4, 1)] = {launch_stream_t<32, 4, 1>, (const void *)stream_kernel<32, 4, 1>};
  t[stream_index(32, 8, 0)] = {launch_stream_t<32, 8, 0>, (const void *)stream_kernel<32, 8, 0>};
}
}  // namespace cpk
