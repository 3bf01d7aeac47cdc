// The decoder-step instantiation of the persistent engine (engine_kernel<true, false>, launched by
// pmpd_engine_run_decoder) in its own translation unit, with 10 consumer warps of 3 tiles per
// stage: 384 threads leave 166 registers per thread and the decoder paths (RMSNorm staging,
// attention, residual stream) run without spills.  Everything else is engine.cu.
#define PMPD_ENGINE_NCW 10
#define PMPD_ENGINE_TPW 3
#define PMPD_ENGINE_DEC_TU 1
#include "engine.cu"
