// Persistent decode engine: every quantized linear layer of one decode token
// in ONE cooperative kernel.
//
// Replaces the per-layer `h @ model.weights(name, p)` calls of one reference
// decode step (pkg/src/pmpd/tinylm.py:341-368, weights() 201-231) for the
// batch-1 decode path.  Why one kernel: at batch 1 every GEMV is a few
// microseconds of HBM traffic, so per-launch setup, pipeline ramp-up and the
// cross-CTA reduction dominate a per-op kernel.  Here
//   * a producer warp per SM streams the CTA's weight tiles of op 0, 1, 2, ...
//     through a shared-memory ring with 1-D TMA bulk copies, never waiting
//     for activations (weights do not depend on them) — only planes 0..p-1;
//   * consumer warps decode bit planes into u8 tensor-core fragments and run
//     mma.sync m16n8k32 (u8 x {s8,u8}) against an int16 two-digit activation
//     operand, int32 accumulation (see gemv.cu for the arithmetic);
//   * an epilogue warp reduces the consumer warps' per-n-group partials and
//     adds them (f32 atomics, performed at L2) into the op's output vector,
//     then publishes the op's completion on a grid-wide counter;
//   * the next op's consumers wait on that counter (acquire) and read one f32
//     per input element into an f16 activation vector in shared memory.  The
//     order of the split-K additions is not fixed, so the low bits of a result
//     may differ between runs (the per-op GEMV keeps a deterministic order);
//   * after the final output every CTA re-zeroes its slice of the vectors.
// Co-residency of all CTAs is guaranteed by a cooperative launch.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "decode_core.cuh"
#include "engine_tile.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

#ifndef PMPD_ENGINE_SB
#define PMPD_ENGINE_SB 4  // staging: float4 groups per thread per L2 round trip (4096 elements per pass)
#endif
constexpr int E_PROD = E_NCW;               // producer warp
constexpr int E_EPI = E_NCW + 1;            // epilogue warp
constexpr int E_THREADS = (E_NCW + 2) * 32;
constexpr int E_MAXSTAGE = 12;
constexpr int E_XMAX = 12288;               // max K of a staged activation vector

struct EngineOp {
  const uint8_t* planes;
  const uint8_t* scales;
  const float* aux;
  long long plane_bytes;
  int n_tiles, k_tiles, n_real, k_real;
  int src;        // -1: external input; else index of the op whose output feeds this one
  int src_col;    // first column of src's output used as input element 0
  int act;        // 0: identity; 1: silu(g) * u with u at column src_col + act_off
  int act_off;
  float in_alpha; // scale applied to the reduced source before the activation
  int max_slots;  // unused since the L2-atomic reduction (kept for the op-table ABI)
  float* part;    // this op's f32 output [n_tiles * 64]: zero at launch, split-K partials added at L2
  const unsigned char* nslots;  // unused (op-table ABI)
};

struct EngineArgs {
  const EngineOp* ops;
  int n_ops;
  const int32_t* p_dev;
  const __half* x_in;  // input of op 0 (f16)
  float* y_out;        // output of the last op (f32), y_alpha * reduced partials
  float y_alpha;
  unsigned* bar;       // [0]: op-completion tickets, [1]: CTAs done (self-resetting)
  int* status;
  long long* trace;    // optional timeline [G][n_ops][4] (globaltimer ns), null = off
};

PMPD_DEV long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// shared-memory plan (byte offsets)
constexpr int kSmBar = 0;                            // mbarriers
constexpr int kSmMisc = 256;                         // mx, flags
constexpr int kSmNs = 512;                           // per-source-n-group slot counts: [2][512] B
constexpr int kSmX = 1536;                           // f16 activations
constexpr int kSmXq = kSmX + E_XMAX * 2;             // per-warp int8 activation fragments
constexpr int kSmRed = kSmXq + E_NCW * E_TPW * 128;  // [2][E_NCW][64] f32
constexpr int kSmRedb = kSmRed + 2 * E_NCW * 64 * 4; // [2][E_NCW] f32
constexpr int kSmRing = (kSmRedb + 2 * E_NCW * 4 + 127) / 128 * 128;

struct Bars {
  uint64_t full[E_MAXSTAGE];
  uint64_t empty[E_MAXSTAGE];
  uint64_t red_full[2];
  uint64_t red_empty[2];
};

// 32-bit partition arithmetic (NT * (G + 1) < 2^32, checked in pmpd_engine_make_op): a 64-bit
// integer division is an emulated ~100-instruction routine, and these run on the op-to-op path.
PMPD_DEV int cta_of_tile(int t, int G, int NT) {
  return (int)(((unsigned)(t + 1) * (unsigned)G + (unsigned)NT - 1u) / (unsigned)NT) - 1;
}

PMPD_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PMPD_DEV unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p >= target: relaxed polls (an acquire load invalidates L1 on every
// iteration), then one acquire fence to order the subsequent reads.
#ifndef E_SPIN
#define E_SPIN 0
#endif
PMPD_DEV void wait_tickets(const unsigned* p, unsigned target) {
#if E_SPIN == 0
  while (ld_acquire(p) < target) __nanosleep(32);
#elif E_SPIN == 4
  while (ld_acquire(p) < target) {
  }
#elif E_SPIN == 1
  while (ld_relaxed(p) < target) __nanosleep(20);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#elif E_SPIN == 2
  while (ld_relaxed(p) < target) {
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
  // relaxed polls, then one acquire load of the same word (synchronizes-with the release adds)
  do {
    while (ld_relaxed(p) < target) __nanosleep(32);
  } while (ld_acquire(p) < target);
#endif
}

struct Range {
  int T0, T1, KT, NT;
};
PMPD_DEV Range range_of(const EngineOp& op, int c, int G) {
  Range r;
  r.NT = op.n_tiles * op.k_tiles;
  r.KT = op.k_tiles;
  r.T0 = (int)((unsigned)c * (unsigned)r.NT / (unsigned)G);
  r.T1 = (int)((unsigned)(c + 1) * (unsigned)r.NT / (unsigned)G);
  return r;
}

// ------------------------------------------------------------------ kernel
PMPD_DEV void consumer_loop(const int P, const EngineArgs& a, uint8_t* smem, Bars& bars, int G, int c,
                            int stage_bytes, int nstage) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tig = lane & 3;
  __half* xs = reinterpret_cast<__half*>(smem + kSmX);
  uint8_t* xq = smem + kSmXq + warp * E_TPW * 128;
  float* misc = reinterpret_cast<float*>(smem + kSmMisc);
  float* red = reinterpret_cast<float*>(smem + kSmRed);
  float* redb = reinterpret_cast<float*>(smem + kSmRedb);
  int slot = 0;     // ring slot (continues across ops)
  uint32_t phase = 0;
  int seg = 0;      // n-group segment counter (red double buffer)
  for (int oi = 0; oi < a.n_ops; ++oi) {
    const EngineOp& op = a.ops[oi];
    const Range r = range_of(op, c, G);
    // ---------------------------------------------------------- stage the input vector
    // k-tiles this CTA touches
    int lo0 = 0, hi0 = r.KT, lo1 = 0, hi1 = 0;
    if (r.T1 - r.T0 < r.KT && r.T1 > r.T0) {
      const int a0 = r.T0 % r.KT, b0 = (r.T1 - 1) % r.KT;
      if (a0 <= b0) {
        lo0 = a0;
        hi0 = b0 + 1;
      } else {
        lo0 = a0;
        hi0 = r.KT;
        lo1 = 0;
        hi1 = b0 + 1;
      }
    } else if (r.T1 <= r.T0) {
      hi0 = 0;
    }
    // per-n-group step normalisers of this op (static: prefetched before the grid wait)
    float idm_pre[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ngp = r.T0 / r.KT + i;
      idm_pre[i] = (r.T1 > r.T0 && ngp < op.n_tiles) ? __ldg(op.aux + ngp) : 0.f;
    }
    if (oi > 0) {
      // every op starts after ALL CTAs published ALL earlier ops (the ticket count is only a
      // safe completion test for a strict op-by-op order)
      if (threadIdx.x == 0) wait_tickets(a.bar, (unsigned)(oi * G));
      named_bar_sync(1, E_NCW * 32);
    }
    if (a.trace && threadIdx.x == 0) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 0] = gtimer();
    float mx = 0.f;
    const EngineOp* src = op.src >= 0 ? &a.ops[op.src] : nullptr;
    // Each thread stages groups of 4 consecutive elements, SB groups per batch: all
    // partial-slot loads of a batch are issued before any sum (one L2 round trip per batch).
    constexpr int SB = PMPD_ENGINE_SB;
    for (int seg2 = 0; seg2 < 2; ++seg2) {
      const int klo = (seg2 ? lo1 : lo0) * kTile, khi = (seg2 ? hi1 : hi0) * kTile;
      for (int kb = klo + 4 * threadIdx.x; kb < khi; kb += 4 * SB * E_NCW * 32) {
        float v[SB][4];
        if (!src) {
#pragma unroll
          for (int bi = 0; bi < SB; ++bi) {
            const int k = kb + bi * 4 * E_NCW * 32;
            if (k + 4 <= op.k_real) {
              const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.x_in + k));
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
              v[bi][0] = f0.x; v[bi][1] = f0.y; v[bi][2] = f1.x; v[bi][3] = f1.y;
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) v[bi][i] = (k + i < op.k_real) ? __half2float(a.x_in[k + i]) : 0.f;
            }
          }
        } else {
          // one f32 per element: the producing CTAs added their n-group partials into src->part
          const int nsrc = op.act == 1 ? 2 : 1;
          float4 acc[2][SB];
#pragma unroll
          for (int which = 0; which < 2; ++which) {
            if (which >= nsrc) break;
#pragma unroll
            for (int bi = 0; bi < SB; ++bi) {
              const int k = kb + bi * 4 * E_NCW * 32;
              const int n = op.src_col + which * op.act_off + k;
              acc[which][bi] = k < khi ? __ldcg(reinterpret_cast<const float4*>(src->part + n))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int bi = 0; bi < SB; ++bi) {
            const int k = kb + bi * 4 * E_NCW * 32;
            float r[2][4];
#pragma unroll
            for (int which = 0; which < 2; ++which) {
              if (which >= nsrc) break;
              const float4 s4 = acc[which][bi];
              r[which][0] = s4.x * op.in_alpha;
              r[which][1] = s4.y * op.in_alpha;
              r[which][2] = s4.z * op.in_alpha;
              r[which][3] = s4.w * op.in_alpha;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float g = r[0][i];
              if (op.act == 1) g = g / (1.f + __expf(-g)) * r[1][i];
              v[bi][i] = (k + i < op.k_real) ? g : 0.f;
            }
          }
        }
#pragma unroll
        for (int bi = 0; bi < SB; ++bi) {
          const int k = kb + bi * 4 * E_NCW * 32;
          if (k >= khi) break;
          const __half2 h01 = __floats2half2_rn(v[bi][0], v[bi][1]), h23 = __floats2half2_rn(v[bi][2], v[bi][3]);
          *reinterpret_cast<__half2*>(xs + k) = h01;
          *reinterpret_cast<__half2*>(xs + k + 2) = h23;
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(f01.x), fabsf(f01.y)), fmaxf(fabsf(f23.x), fabsf(f23.y))));
        }
      }
    }
    mx = warp_max(mx);
    if (lane == 0) misc[8 + warp] = mx;
    named_bar_sync(1, E_NCW * 32);
    mx = 0.f;
#pragma unroll
    for (int w = 0; w < E_NCW; ++w) mx = fmaxf(mx, misc[8 + w]);
    if (a.trace && threadIdx.x == 0) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 1] = gtimer();
    // ---------------------------------------------------------- tiles of this op
    int t = r.T0, ng = r.T0 / r.KT, kt = r.T0 % r.KT;
    int dacc[4][4];  // balanced-digit sums: [.][0|2] high, [.][1|3] low (lanes tig == 0)
    float bias = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) dacc[i][e] = 0;
    float qs = 0.f;
    long long tcyc = 0, tcalls = 0, scyc0 = a.trace ? clock64() : 0, fcyc = 0, fwait = 0;
    int ngi = 0;
    // activation scale per n-group: qs = E_QMAX * idm / mx (one reciprocal per op, none per group)
    const float qmx = mx > 0.f ? __fdividef(E_QMAX, mx) : 0.f;
    if (t < r.T1) qs = qmx * idm_pre[0];
    while (t < r.T1) {
      const int end = min(min(t + E_STILES, r.T1), t - kt + r.KT);
#ifndef PMPD_ENGINE_SKIP_MEMORY
      mbar_wait(&bars.full[slot], phase);
#endif
#ifdef PMPD_ENGINE_SKIP_COMPUTE
      if (false) {
#else
      if (warp < end - t) {
#endif
        if (a.trace) {
          const long long c0 = clock64();
          tile_dispatch(P, smem + kSmRing + slot * stage_bytes, end - t, warp, kt + warp, lane, xs, xq, qs, dacc,
                        bias);
          tcyc += clock64() - c0;
          ++tcalls;
        } else {
          tile_dispatch(P, smem + kSmRing + slot * stage_bytes, end - t, warp, kt + warp, lane, xs, xq, qs, dacc,
                        bias);
        }
      }
      __syncwarp();
#ifndef PMPD_ENGINE_SKIP_MEMORY
      if (lane == 0) mbar_arrive(&bars.empty[slot]);
#endif
      if (++slot == nstage) {
        slot = 0;
        phase ^= 1u;
      }
      kt += end - t;
      t = end;
      if (kt == r.KT || t == r.T1) {
        // hand the n-group partial to the epilogue warp (double-buffered)
        const long long f0 = a.trace ? clock64() : 0;
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&bars.red_empty[buf], ((seg >> 1) & 1) ^ 1);
        if (a.trace) fwait += clock64() - f0;
        float* rw = red + (buf * E_NCW + warp) * 64;
        const float ds = qs > 0.f ? __frcp_rn(qs) : 0.f;
        if (tig == 0) {
#pragma unroll
          for (int tt = 0; tt < 4; ++tt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              rw[16 * tt + gq + 8 * h] = fmaf(256.f, (float)dacc[tt][2 * h], (float)dacc[tt][2 * h + 1]) *
                                         (ds * (1.f / (float)(1 << tt)));
        }
        const float bs = warp_sum(bias);
        if (lane == 0) redb[buf * E_NCW + warp] = bs;
        __syncwarp();  // order every lane's partial stores before lane 0's release-arrive
        if (lane == 0) mbar_arrive(&bars.red_full[buf]);
        ++seg;
        if (a.trace) fcyc += clock64() - f0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) dacc[i][e] = 0;
        bias = 0.f;
        if (kt == r.KT) {
          kt = 0;
          ++ng;
          if (t < r.T1) {
            ++ngi;
            const float idm = ngi == 1 ? idm_pre[1] : ngi == 2 ? idm_pre[2] : ngi == 3 ? idm_pre[3] : __ldg(op.aux + ng);
            qs = qmx * idm;
          }
        }
      }
    }
    if (a.trace && threadIdx.x == 0) {
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 2] = gtimer();
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 4] = tcyc;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 5] = tcalls;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 6] = clock64() - scyc0;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 7] = (fwait << 32) | (fcyc & 0xffffffffll);
    }
  }
}

__global__ void __launch_bounds__(E_THREADS, 1) engine_kernel(const EngineArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + kSmBar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  int p = *a.p_dev;
  if (p < 1 || p > 4) {
    if (threadIdx.x == 0 && c == 0) atomicExch(a.status, PMPD_ERR_CONTRACT);
    p = p < 1 ? 1 : 4;
  }
  const int stage_bytes = E_STILES * (p + 1) * kTilePlaneBytes;
  uint32_t dyn_bytes;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_bytes));
  int nstage = (int)((dyn_bytes - kSmRing) / stage_bytes);
  nstage = nstage > E_MAXSTAGE ? E_MAXSTAGE : nstage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&bars.full[i], 1);
      mbar_init(&bars.empty[i], E_NCW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.red_full[i], E_NCW);
      mbar_init(&bars.red_empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == E_PROD) {
    // ------------------------------------------------------------ producer
#ifdef PMPD_ENGINE_SKIP_MEMORY
    if (false) {
#else
    if (lane == 0) {
#endif
      const uint64_t pol = policy_evict_first();
      int slot = 0, used = 0;
      uint32_t phase = 0;
      for (int oi = 0; oi < a.n_ops; ++oi) {
        const EngineOp& op = a.ops[oi];
        const Range r = range_of(op, c, G);
        int t = r.T0, kt = r.T0 % r.KT;
        while (t < r.T1) {
          const int end = min(min(t + E_STILES, r.T1), t - kt + r.KT);
          const int cnt = end - t;
          if (used) mbar_wait_backoff(&bars.empty[slot], phase ^ 1u);
          uint8_t* st = smem + kSmRing + slot * stage_bytes;
          mbar_arrive_expect_tx(&bars.full[slot], (uint32_t)(cnt * kTilePlaneBytes * (p + 1)));
          for (int j = 0; j < p; ++j)
            bulk_g2s_stream(st + j * E_STILES * kTilePlaneBytes,
                            op.planes + j * op.plane_bytes + (int64_t)t * kTilePlaneBytes, cnt * kTilePlaneBytes,
                            &bars.full[slot], pol);
          bulk_g2s_stream(st + p * E_STILES * kTilePlaneBytes, op.scales + (int64_t)t * kTileScaleBytes,
                          cnt * kTileScaleBytes, &bars.full[slot], pol);
          kt += cnt;
          if (kt == r.KT) kt = 0;
          t = end;
          if (++slot == nstage) {
            slot = 0;
            phase ^= 1u;
            used = 1;
          }
        }
      }
    }
  } else if (warp == E_EPI) {
    // ------------------------------------------------------------ epilogue
    float* red = reinterpret_cast<float*>(smem + kSmRed);
    float* redb = reinterpret_cast<float*>(smem + kSmRedb);
    int seg = 0;
    for (int oi = 0; oi < a.n_ops; ++oi) {
      const EngineOp& op = a.ops[oi];
      const Range r = range_of(op, c, G);
      int t = r.T0, ng = r.T0 / r.KT, kt = r.T0 % r.KT;
      while (t < r.T1) {
        const int seg_end = min(r.T1, t - kt + r.KT);
        const int buf = seg & 1;
#ifdef PMPD_ENGINE_EPI_SPIN
        mbar_wait(&bars.red_full[buf], (seg >> 1) & 1);
#else
        mbar_wait_backoff(&bars.red_full[buf], (seg >> 1) & 1);
#endif
        float bsum = 0.f;
#pragma unroll
        for (int w = 0; w < E_NCW; ++w) bsum += redb[buf * E_NCW + w];
        // split-K: every CTA holding tiles of n-group ng adds its partial at L2
        float* dst = op.part + (int64_t)ng * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nl = lane + 32 * h;
          float v = bsum;
#pragma unroll
          for (int w = 0; w < E_NCW; ++w) v += red[(buf * E_NCW + w) * 64 + nl];
          atomicAdd(dst + nl, v);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.red_empty[buf]);
        ++seg;
        kt += seg_end - t;
        t = seg_end;
        if (kt == r.KT) {
          kt = 0;
          ++ng;
        }
      }
      __syncwarp();  // lane 0's release covers the warp's partial stores (cumulativity)
      if (lane == 0) {
        // A CTA with no tiles in op oi must not publish it before every CTA has
        // published ops < oi: the ticket count is a completion test only if tickets
        // of op oi never precede the completion of op oi-1.
        if (oi > 0 && r.T1 <= r.T0) wait_tickets(a.bar, (unsigned)(oi * G));
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
        if (a.trace) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 3] = gtimer();
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    consumer_loop(p, a, smem, bars, G, c, stage_bytes, nstage);
  }
  // ---------------------------------------------------------------- final output
  __syncthreads();
  const EngineOp& last = a.ops[a.n_ops - 1];
  if (threadIdx.x == 0) wait_tickets(a.bar, (unsigned)(a.n_ops * G));
  __syncthreads();
  for (int ng = c; ng < last.n_tiles; ng += G) {
    for (int nl = threadIdx.x; nl < 64; nl += blockDim.x) {
      const int n = ng * 64 + nl;
      if (n < last.n_real) a.y_out[n] = a.y_alpha * __ldcg(last.part + n);
    }
  }
  __syncthreads();
  // Re-zero the accumulation vectors for the next launch.  Every read of ops 0..n-2 happened
  // before the final ticket; the last op's n-groups are zeroed by the CTA that just read them.
  for (int oi = 0; oi < a.n_ops; ++oi) {
    const EngineOp& op = a.ops[oi];
    for (int ng = c; ng < op.n_tiles; ng += G)
      for (int nl = threadIdx.x; nl < 64; nl += blockDim.x) op.part[(int64_t)ng * 64 + nl] = 0.f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.bar + 1, 1u) == (unsigned)(G - 1)) {
      a.bar[0] = 0;
      a.bar[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" {

int pmpd_engine_op_bytes(void) { return (int)sizeof(EngineOp); }

int pmpd_engine_grid(void) { return num_sms(); }

// partial slots per n-group of an op's output for the engine's grid
int pmpd_engine_max_slots(const pmpd_qtensor* t) {
  const int nt = t->n_tiles * t->k_tiles, g = num_sms();
  const int per = nt / g;
  return per >= 1 ? t->k_tiles / per + 2 : g;
}

int pmpd_engine_nslots(const pmpd_qtensor* t, uint8_t* out_host) {
  const int nt = t->n_tiles * t->k_tiles, g = num_sms(), kt = t->k_tiles;
  auto cta = [&](int tile) { return (int)(((int64_t)(tile + 1) * g + nt - 1) / nt) - 1; };
  for (int ng = 0; ng < t->n_tiles; ++ng) {
    const int n = cta(std::min((ng + 1) * kt, nt) - 1) - cta(ng * kt) + 1;
    if (n > 255) return fail(PMPD_ERR_CONFIG, "too many contributors per n-group");
    out_host[ng] = (uint8_t)n;
  }
  return PMPD_OK;
}

int pmpd_engine_make_op(const pmpd_qtensor* t, int32_t src, int32_t src_col, int32_t act, int32_t act_off,
                        float in_alpha, float* part_dev, int32_t max_slots, const uint8_t* nslots_dev,
                        void* op_host) {
  if (!t || !t->data || !op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  if (t->layout != PMPD_LAYOUT_KN || t->p_max != 4)
    return fail(PMPD_ERR_CONFIG, "the decode engine needs KN tiles with p_max 4");
  if (t->k_tiles * kTile > E_XMAX) return fail(PMPD_ERR_CONFIG, "engine input width above %d", E_XMAX);
  if ((int64_t)t->n_tiles * t->k_tiles * (num_sms() + 1) >= (int64_t)1 << 32)
    return fail(PMPD_ERR_CONFIG, "engine op too large for 32-bit tile partitioning");
  EngineOp op{};
  op.planes = static_cast<const uint8_t*>(t->data);
  op.scales = op.planes + (int64_t)t->p_max * t->plane_bytes;
  op.aux = reinterpret_cast<const float*>(op.scales + t->scale_bytes);
  op.plane_bytes = t->plane_bytes;
  op.n_tiles = t->n_tiles;
  op.k_tiles = t->k_tiles;
  op.n_real = t->n;
  op.k_real = t->k;
  op.src = src;
  op.src_col = src_col;
  op.act = act;
  op.act_off = act_off;
  op.in_alpha = in_alpha;
  op.max_slots = max_slots;
  op.part = part_dev;
  op.nslots = nslots_dev;
  if ((src_col & 3) || (act_off & 3)) return fail(PMPD_ERR_CONFIG, "engine input offsets must be multiples of 4");
  *static_cast<EngineOp*>(op_host) = op;
  return PMPD_OK;
}

int pmpd_engine_run_traced(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                           float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream);

int pmpd_engine_run(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                    float y_alpha, uint32_t* bar_dev, int32_t* status_dev, void* stream) {
  return pmpd_engine_run_traced(ops_dev, n_ops, p_dev, x_in, y_out, y_alpha, bar_dev, status_dev, nullptr, stream);
}

int pmpd_engine_run_traced(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                           float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream) {
  if (n_ops < 1) return fail(PMPD_ERR_CONFIG, "engine program is empty");
  EngineArgs a;
  a.ops = static_cast<const EngineOp*>(ops_dev);
  a.n_ops = n_ops;
  a.p_dev = p_dev;
  a.x_in = static_cast<const __half*>(x_in);
  a.y_out = y_out;
  a.y_alpha = y_alpha;
  a.bar = bar_dev;
  a.status = status_dev;
  a.trace = reinterpret_cast<long long*>(trace_dev);
  static int smem = 0;
  if (smem == 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    smem = optin;
    if (const char* e = getenv("PMPD_ENGINE_SMEM")) smem = atoi(e) < optin ? atoi(e) : optin;
    cudaFuncSetAttribute(engine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(E_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, engine_kernel, a);
  if (e != cudaSuccess) return fail(PMPD_ERR_CUDA, "engine launch: %s", cudaGetErrorString(e));
  return PMPD_OK;
}

}  // extern "C"
