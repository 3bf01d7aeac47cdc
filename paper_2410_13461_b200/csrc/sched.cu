// Device-side precision hook (north-star (d)): PrecisionSchedule.precision_at
// (pkg/src/pmpd/schedule.py:93-99) evaluated on the GPU from a device-resident
// switch-point table and step counter, as called once per decode step by
// generate (tinylm.py:512,518).
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

// One thread.  Launched WITHOUT programmatic-dependent-launch and never
// triggering early, so every kernel after it in the stream starts only after
// *p_out is written (the GEMVs read p before their own griddepcontrol.wait).
__global__ void sched_step_kernel(const int32_t* __restrict__ sched, int n_prec, int32_t* __restrict__ step,
                                  int32_t* __restrict__ p_out, int advance) {
  const int i = *step;
  int best = -1, highest = -1;
  for (int q = 0; q < n_prec; ++q) {
    const int p = sched[2 * q], st = sched[2 * q + 1];
    if (p <= 0) continue;  // unused entry of a fixed-capacity table
    if (p > highest) highest = p;
    if (st <= i && (best < 0 || p < best)) best = p;
  }
  *p_out = best < 0 ? highest : best;  // unreachable for a valid schedule (highest starts at 0)
  if (advance) *step = i + 1;
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" int pmpd_sched_step(const int32_t* sched, int32_t n_prec, int32_t* step, int32_t* p_out, int32_t advance,
                               void* stream) {
  if (n_prec < 1) return fail(PMPD_ERR_CONFIG, "schedule needs at least one precision");
  sched_step_kernel<<<1, 1, 0, as_stream(stream)>>>(sched, n_prec, step, p_out, advance);
  return check_launch("pmpd_sched_step");
}
