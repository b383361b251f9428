// stream_inst_3.cu -- stream_kernel instantiations for R = 25..32 (split for parallel builds).
#include "stream_inst.cuh"
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part3(StreamEntry *t) { CPK_STREAM_REG_8(25) }
}  // namespace cpk
