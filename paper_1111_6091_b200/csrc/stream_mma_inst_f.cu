// stream_mma_inst_f.cu -- full-feature instantiations of stream_mma_kernel<NT, MT, OP, true> (fcm staging,
// pre-wait Z prefetch, sweep_tail / one-launch cp_mttkrp completion, deferred Gram job).
#define CPK_MMA_FEAT true
#include "stream_inst.cuh"
#include "stream_mma.cuh"

namespace cpk {
void register_stream_mma_f(StreamEntry *t) { CPK_MMA_REG_MT8(1) CPK_MMA_REG_MT8(2) CPK_MMA_REG_MT4(3) CPK_MMA_REG_MT4(4) }
}  // namespace cpk
