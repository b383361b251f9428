// stream_inst_1.cu -- stream_kernel instantiations for R = 9..16 (split for parallel builds).
#include "stream_inst.cuh"
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part1(StreamEntry *t) { CPK_STREAM_REG_8(9) }
}  // namespace cpk
