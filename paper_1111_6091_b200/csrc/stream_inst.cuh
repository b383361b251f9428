// stream_inst.cuh -- X-macros of the streaming-kernel instantiation tables (stream_inst_*.cu,
// stream_mma_inst.cu): every (R, V, OP) of stream_kernel and every (NT, MT, OP) of
// stream_mma_kernel that make_stream_plan can select, registered by index in the kernel tables of
// capi.cu.  The tables are split over several translation units only to build in parallel.
#pragma once

// DFMA consumers: V in {1, 2, 4} for every op, V = 8 for MTTKRP and the Y_L pass
#define CPK_STREAM_REG(R, V, OP) t[stream_index(R, V, OP)] = {launch_stream_t<R, V, OP>, (const void *)stream_kernel<R, V, OP>};
#define CPK_STREAM_REG_R(R)                                                                               \
  CPK_STREAM_REG(R, 1, 0) CPK_STREAM_REG(R, 1, 1) CPK_STREAM_REG(R, 1, 2) CPK_STREAM_REG(R, 2, 0)       \
  CPK_STREAM_REG(R, 2, 1) CPK_STREAM_REG(R, 2, 2) CPK_STREAM_REG(R, 4, 0) CPK_STREAM_REG(R, 4, 1)       \
  CPK_STREAM_REG(R, 4, 2) CPK_STREAM_REG(R, 8, 0) CPK_STREAM_REG(R, 8, 2)
#define CPK_STREAM_REG_8(R0)                                                                              \
  CPK_STREAM_REG_R(R0 + 0) CPK_STREAM_REG_R(R0 + 1) CPK_STREAM_REG_R(R0 + 2) CPK_STREAM_REG_R(R0 + 3)   \
  CPK_STREAM_REG_R(R0 + 4) CPK_STREAM_REG_R(R0 + 5) CPK_STREAM_REG_R(R0 + 6) CPK_STREAM_REG_R(R0 + 7)

// FP64 tensor-core consumers: NT = 1, 2 with MT = 1..8; NT = 3, 4 with MT = 1..4; every op
// (CPK_MMA_FEAT: the translation unit's feature flag -- stream_mma_inst.cu lean, stream_mma_inst_f.cu full)
#define CPK_MMA_REG(NT, MT, OP) \
  t[mma_index(NT, MT, OP)] = {launch_stream_mma_t<NT, MT, OP, CPK_MMA_FEAT>, (const void *)stream_mma_kernel<NT, MT, OP, CPK_MMA_FEAT>};
#define CPK_MMA_REG_OPS(NT, MT) CPK_MMA_REG(NT, MT, 0) CPK_MMA_REG(NT, MT, 2) CPK_MMA_REG(NT, MT, 1)
#define CPK_MMA_REG_MT4(NT) CPK_MMA_REG_OPS(NT, 1) CPK_MMA_REG_OPS(NT, 2) CPK_MMA_REG_OPS(NT, 3) CPK_MMA_REG_OPS(NT, 4)
#define CPK_MMA_REG_MT8(NT) \
  CPK_MMA_REG_MT4(NT) CPK_MMA_REG_OPS(NT, 5) CPK_MMA_REG_OPS(NT, 6) CPK_MMA_REG_OPS(NT, 7) CPK_MMA_REG_OPS(NT, 8)
