// stream_inst_3.cu -- instantiations of stream_kernel for R = 25..32 (split for parallel builds).
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part3(StreamEntry *t) {
  t[stream_index(25, 1, 0)] = {launch_stream_t<25, 1, 0>, (const void *)stream_kernel<25, 1, 0>};
  t[stream_index(25, 1, 1)] = {launch_stream_t<25, 1, 1>, (const void *)stream_kernel<25, 1, 1>};
  t[stream_index(25, 2, 0)] = {launch_stream_t<25, 2, 0>, (const void *)stream_kernel<25, 2, 0>};
  t[stream_index(25, 2, 1)] = {launch_stream_t<25, 2, 1>, (const void *)stream_kernel<25, 2, 1>};
  t[stream_index(26, 1, 0)] = {launch_stream_t<26, 1, 0>, (const void *)stream_kernel<26, 1, 0>};
  t[stream_index(26, 1, 1)] = {launch_stream_t<26, 1, 1>, (const void *)stream_kernel<26, 1, 1>};
  t[stream_index(26, 2, 0)] = {launch_stream_t<26, 2, 0>, (const void *)stream_kernel<26, 2, 0>};
  t[stream_index(26, 2, 1)] = {launch_stream_t<26, 2, 1>, (const void *)stream_kernel<26, 2, 1>};
  t[stream_index(27, 1, 0)] = {launch_stream_t<27, 1, 0>, (const void *)stream_kernel<27, 1, 0>};
  t[stream_index(27, 1, 1)] = {launch_stream_t<27, 1, 1>, (const void *)stream_kernel<27, 1, 1>};
  t[stream_index(27, 2, 0)] = {launch_stream_t<27, 2, 0>, (const void *)stream_kernel<27, 2, 0>};
  t[stream_index(27, 2, 1)] = {launch_stream_t<27, 2, 1>, (const void *)stream_kernel<27, 2, 1>};
  t[stream_index(28, 1, 0)] = {launch_stream_t<28, 1, 0>, (const void *)stream_kernel<28, 1, 0>};
  t[stream_index(28, 1, 1)] = {launch_stream_t<28, 1, 1>, (const void *)stream_kernel<28, 1, 1>};
  t[stream_index(28, 2, 0)] = {launch_stream_t<28, 2, 0>, (const void *)stream_kernel<28, 2, 0>};
  t[stream_index(28, 2, 1)] = {launch_stream_t<28, 2, 1>, (const void *)stream_kernel<28, 2, 1>};
  t[stream_index(29, 1, 0)] = {launch_stream_t<29, 1, 0>, (const void *)stream_kernel<29, 1, 0>};
  t[stream_index(29, 1, 1)] = {launch_stream_t<29, 1, 1>, (const void *)stream_kernel<29, 1, 1>};
  t[stream_index(29, 2, 0)] = {launch_stream_t<29, 2, 0>, (const void *)stream_kernel<29, 2, 0>};
  t[stream_index(29, 2, 1)] = {launch_stream_t<29, 2, 1>, (const void *)stream_kernel<29, 2, 1>};
  t[stream_index(30, 1, 0)] = {launch_stream_t<30, 1, 0>, (const void *)stream_kernel<30, 1, 0>};
  t[stream_index(30, 1, 1)] = {launch_stream_t<30, 1, 1>, (const void *)stream_kernel<30, 1, 1>};
  t[stream_index(30, 2, 0)] = {launch_stream_t<30, 2, 0>, (const void *)stream_kernel<30, 2, 0>};
  t[stream_index(30, 2, 1)] = {launch_stream_t<30, 2, 1>, (const void *)stream_kernel<30, 2, 1>};
  t[stream_index(31, 1, 0)] = {launch_stream_t<31, 1, 0>, (const void *)stream_kernel<31, 1, 0>};
  t[stream_index(31, 1, 1)] = {launch_stream_t<31, 1, 1>, (const void *)stream_kernel<31, 1, 1>};
  t[stream_index(31, 2, 0)] = {launch_stream_t<31, 2, 0>, (const void *)stream_kernel<31, 2, 0>};
  t[stream_index(31, 2, 1)] = {launch_stream_t<31, 2, 1>, (const void *)stream_kernel<31, 2, 1>};
  t[stream_index(32, 1, 0)] = {launch_stream_t<32, 1, 0>, (const void *)stream_kernel<32, 1, 0>};
  t[stream_index(32, 1, 1)] = {launch_stream_t<32, 1, 1>, (const void *)stream_kernel<32, 1, 1>};
  t[stream_index(32, 2, 0)] = {launch_stream_t<32, 2, 0>, (const void *)stream_kernel<32, 2, 0>};
  t[stream_index(32, 2, 1)] = {launch_stream_t<32, 2, 1>, (const void *)stream_kernel<32, 2, 1>};
}
}  // namespace cpk
