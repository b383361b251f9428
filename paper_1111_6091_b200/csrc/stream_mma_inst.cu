// stream_mma_inst.cu -- instantiations of stream_mma_kernel<NT, MT, OP> (NT = 1..4 n-tiles of 8 ranks,
// MT = 1..8 m-tiles of 8 rows per warp, OP = MTTKRP / Y_L pass).
#include "stream_mma.cuh"

namespace cpk {
void register_stream_mma(StreamEntry *t) {
  t[mma_index(1, 1, 0)] = {launch_stream_mma_t<1, 1, 0>, (const void *)stream_mma_kernel<1, 1, 0>};
  t[mma_index(1, 1, 2)] = {launch_stream_mma_t<1, 1, 2>, (const void *)stream_mma_kernel<1, 1, 2>};
  t[mma_index(1, 2, 0)] = {launch_stream_mma_t<1, 2, 0>, (const void *)stream_mma_kernel<1, 2, 0>};
  t[mma_index(1, 2, 2)] = {launch_stream_mma_t<1, 2, 2>, (const void *)stream_mma_kernel<1, 2, 2>};
  t[mma_index(1, 3, 0)] = {launch_stream_mma_t<1, 3, 0>, (const void *)stream_mma_kernel<1, 3, 0>};
  t[mma_index(1, 3, 2)] = {launch_stream_mma_t<1, 3, 2>, (const void *)stream_mma_kernel<1, 3, 2>};
  t[mma_index(1, 4, 0)] = {launch_stream_mma_t<1, 4, 0>, (const void *)stream_mma_kernel<1, 4, 0>};
  t[mma_index(1, 4, 2)] = {launch_stream_mma_t<1, 4, 2>, (const void *)stream_mma_kernel<1, 4, 2>};
  t[mma_index(1, 5, 0)] = {launch_stream_mma_t<1, 5, 0>, (const void *)stream_mma_kernel<1, 5, 0>};
  t[mma_index(1, 5, 2)] = {launch_stream_mma_t<1, 5, 2>, (const void *)stream_mma_kernel<1, 5, 2>};
  t[mma_index(1, 6, 0)] = {launch_stream_mma_t<1, 6, 0>, (const void *)stream_mma_kernel<1, 6, 0>};
  t[mma_index(1, 6, 2)] = {launch_stream_mma_t<1, 6, 2>, (const void *)stream_mma_kernel<1, 6, 2>};
  t[mma_index(1, 7, 0)] = {launch_stream_mma_t<1, 7, 0>, (const void *)stream_mma_kernel<1, 7, 0>};
  t[mma_index(1, 7, 2)] = {launch_stream_mma_t<1, 7, 2>, (const void *)stream_mma_kernel<1, 7, 2>};
  t[mma_index(1, 8, 0)] = {launch_stream_mma_t<1, 8, 0>, (const void *)stream_mma_kernel<1, 8, 0>};
  t[mma_index(1, 8, 2)] = {launch_stream_mma_t<1, 8, 2>, (const void *)stream_mma_kernel<1, 8, 2>};
  t[mma_index(2, 1, 0)] = {launch_stream_mma_t<2, 1, 0>, (const void *)stream_mma_kernel<2, 1, 0>};
  t[mma_index(2, 1, 2)] = {launch_stream_mma_t<2, 1, 2>, (const void *)stream_mma_kernel<2, 1, 2>};
  t[mma_index(2, 2, 0)] = {launch_stream_mma_t<2, 2, 0>, (const void *)stream_mma_kernel<2, 2, 0>};
  t[mma_index(2, 2, 2)] = {launch_stream_mma_t<2, 2, 2>, (const void *)stream_mma_kernel<2, 2, 2>};
  t[mma_index(2, 3, 0)] = {launch_stream_mma_t<2, 3, 0>, (const void *)stream_mma_kernel<2, 3, 0>};
  t[mma_index(2, 3, 2)] = {launch_stream_mma_t<2, 3, 2>, (const void *)stream_mma_kernel<2, 3, 2>};
  t[mma_index(2, 4, 0)] = {launch_stream_mma_t<2, 4, 0>, (const void *)stream_mma_kernel<2, 4, 0>};
  t[mma_index(2, 4, 2)] = {launch_stream_mma_t<2, 4, 2>, (const void *)stream_mma_kernel<2, 4, 2>};
  t[mma_index(2, 5, 0)] = {launch_stream_mma_t<2, 5, 0>, (const void *)stream_mma_kernel<2, 5, 0>};
  t[mma_index(2, 5, 2)] = {launch_stream_mma_t<2, 5, 2>, (const void *)stream_mma_kernel<2, 5, 2>};
  t[mma_index(2, 6, 0)] = {launch_stream_mma_t<2, 6, 0>, (const void *)stream_mma_kernel<2, 6, 0>};
  t[mma_index(2, 6, 2)] = {launch_stream_mma_t<2, 6, 2>, (const void *)stream_mma_kernel<2, 6, 2>};
  t[mma_index(2, 7, 0)] = {launch_stream_mma_t<2, 7, 0>, (const void *)stream_mma_kernel<2, 7, 0>};
  t[mma_index(2, 7, 2)] = {launch_stream_mma_t<2, 7, 2>, (const void *)stream_mma_kernel<2, 7, 2>};
  t[mma_index(2, 8, 0)] = {launch_stream_mma_t<2, 8, 0>, (const void *)stream_mma_kernel<2, 8, 0>};
  t[mma_index(2, 8, 2)] = {launch_stream_mma_t<2, 8, 2>, (const void *)stream_mma_kernel<2, 8, 2>};
  t[mma_index(3, 1, 0)] = {launch_stream_mma_t<3, 1, 0>, (const void *)stream_mma_kernel<3, 1, 0>};
  t[mma_index(3, 1, 2)] = {launch_stream_mma_t<3, 1, 2>, (const void *)stream_mma_kernel<3, 1, 2>};
  t[mma_index(3, 2, 0)] = {launch_stream_mma_t<3, 2, 0>, (const void *)stream_mma_kernel<3, 2, 0>};
  t[mma_index(3, 2, 2)] = {launch_stream_mma_t<3, 2, 2>, (const void *)stream_mma_kernel<3, 2, 2>};
  t[mma_index(3, 3, 0)] = {launch_stream_mma_t<3, 3, 0>, (const void *)stream_mma_kernel<3, 3, 0>};
  t[mma_index(3, 3, 2)] = {launch_stream_mma_t<3, 3, 2>, (const void *)stream_mma_kernel<3, 3, 2>};
  t[mma_index(3, 4, 0)] = {launch_stream_mma_t<3, 4, 0>, (const void *)stream_mma_kernel<3, 4, 0>};
  t[mma_index(3, 4, 2)] = {launch_stream_mma_t<3, 4, 2>, (const void *)stream_mma_kernel<3, 4, 2>};
  t[mma_index(4, 1, 0)] = {launch_stream_mma_t<4, 1, 0>, (const void *)stream_mma_kernel<4, 1, 0>};
  t[mma_index(4, 1, 2)] = {launch_stream_mma_t<4, 1, 2>, (const void *)stream_mma_kernel<4, 1, 2>};
  t[mma_index(4, 2, 0)] = {launch_stream_mma_t<4, 2, 0>, (const void *)stream_mma_kernel<4, 2, 0>};
  t[mma_index(4, 2, 2)] = {launch_stream_mma_t<4, 2, 2>, (const void *)stream_mma_kernel<4, 2, 2>};
  t[mma_index(4, 3, 0)] = {launch_stream_mma_t<4, 3, 0>, (const void *)stream_mma_kernel<4, 3, 0>};
  t[mma_index(4, 3, 2)] = {launch_stream_mma_t<4, 3, 2>, (const void *)stream_mma_kernel<4, 3, 2>};
  t[mma_index(4, 4, 0)] = {launch_stream_mma_t<4, 4, 0>, (const void *)stream_mma_kernel<4, 4, 0>};
  t[mma_index(4, 4, 2)] = {launch_stream_mma_t<4, 4, 2>, (const void *)stream_mma_kernel<4, 4, 2>};
}
}  // namespace cpk
