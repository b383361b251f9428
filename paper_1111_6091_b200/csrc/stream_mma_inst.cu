// stream_mma_inst.cu -- lean instantiations of stream_mma_kernel<NT, MT, OP, false> (NT = 1..4 n-tiles
// of 8 ranks, MT = m-tiles of 8 rows per warp, OP = MTTKRP / Y_L pass / residual pass): plans
// without fcm staging, pre-wait prefetch or in-pass completion (stream_kernel.cuh, P_FCM).
#define CPK_MMA_FEAT false
#include "stream_inst.cuh"
#include "stream_mma.cuh"

namespace cpk {
void register_stream_mma(StreamEntry *t) { CPK_MMA_REG_MT8(1) CPK_MMA_REG_MT8(2) CPK_MMA_REG_MT4(3) CPK_MMA_REG_MT4(4) }
}  // namespace cpk
