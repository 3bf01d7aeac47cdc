// The decoder-step instantiation of the persistent engine (engine_kernel<true, false>, launched by
// pmpd_engine_run_decoder) in its own translation unit, with 10 consumer warps of 3 tiles per
// stage: 384 threads leave 166 registers per thread and the decoder paths (RMSNorm staging,
// attention, residual stream) run without spills.  Everything else is engine.cu.
#ifndef PMPD_ENGINE_DEC_NCW
#define PMPD_ENGINE_DEC_NCW 10
#endif
#ifndef PMPD_ENGINE_DEC_TPW
#define PMPD_ENGINE_DEC_TPW 3
#endif
#define PMPD_ENGINE_NCW PMPD_ENGINE_DEC_NCW
#define PMPD_ENGINE_TPW PMPD_ENGINE_DEC_TPW
#define PMPD_ENGINE_DEC_TU 1
#include "engine.cu"
