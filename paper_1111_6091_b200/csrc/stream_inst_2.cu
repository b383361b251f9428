// stream_inst_2.cu -- stream_kernel instantiations for R = 17..24 (split for parallel builds).
#include "stream_inst.cuh"
#include "stream_kernel.cuh"

namespace cpk {
void register_stream_part2(StreamEntry *t) { CPK_STREAM_REG_8(17) }
}  // namespace cpk
