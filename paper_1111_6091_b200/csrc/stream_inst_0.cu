// stream_inst_0.cu -- stream_kernel instantiations for R = 1..8 (split for parallel builds).
#include "stream_inst.cuh"
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part0(StreamEntry *t) { CPK_STREAM_REG_8(1) }
}  // namespace cpk
