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
//     adds them into the op's output vector at L2;
//   * the next op's consumers stage one value per input element into an f16
//     activation vector in shared memory.
// Every program uses COUNTED fixed-point accumulation: each output element is
// a u64 word whose top 10 bits count the contributing CTAs and whose low 54
// bits sum the contributions as 2^-24 fixed point (offset binary).  Integer
// addition is associative, so the result is bit-identical whatever order the
// split-K partials arrive in, and the word itself tells a consumer when all
// contributors have landed: no release fence, no grid-wide ticket on the
// op-to-op path.  Vectors rotate through three buffer sets by launch epoch;
// each CTA zeroes its slice of the previous launch's set as it goes.
// Instantiations: engine_kernel<DEC, TP> — DEC adds the decoder-step ops
// (attention, RMSNorm / attention-combine inputs, one counted residual stream),
// TP the tensor-parallel rank groups and peer copies (pmpd_engine_run_ranks).
// This translation unit builds <false, false> and <false, true> with 12 consumer
// warps; engine_dec.cu includes it with PMPD_ENGINE_DEC_TU to build <true, false>
// with 10 (fewer threads, more registers for the decoder paths).
// Sub-ops (set_slice / set_share) restrict an op to a block of its tensor on a
// subset of CTAs, all adding into the tensor's one output vector.
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
#ifndef PMPD_ENGINE_PROD_WARP
#define PMPD_ENGINE_PROD_WARP E_NCW
#endif
#ifndef PMPD_ENGINE_EPI_WARP
#define PMPD_ENGINE_EPI_WARP (E_NCW + 1)
#endif
#ifndef PMPD_ENGINE_PROD2
#define PMPD_ENGINE_PROD2 0  // 1: a second producer warp (on another scheduler) issues every other stage
#endif
constexpr int E_PROD = PMPD_ENGINE_PROD_WARP;  // producer warp
constexpr int E_EPI = PMPD_ENGINE_EPI_WARP;    // epilogue warp
constexpr int E_PROD_B = PMPD_ENGINE_PROD2 ? (E_PROD > E_EPI ? E_PROD : E_EPI) + 1 : E_PROD;  // second producer
constexpr int E_LASTW = E_PROD_B > (E_PROD > E_EPI ? E_PROD : E_EPI) ? E_PROD_B : (E_PROD > E_EPI ? E_PROD : E_EPI);
constexpr int E_THREADS = (E_LASTW + 1) * 32;  // warps above E_NCW without a role idle
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
  // ---- decoder-step extensions (pmpd_engine_op_set_io / pmpd_engine_make_attn_op)
  int kind;          // E_LINEAR or E_ATTN
  int in_mode;       // E_IN_SRC (src / x_in, as above), E_IN_RMSNORM (rmsnorm(resid) * gain), E_IN_ATTN
  const float* resid;
  const float* gain;
  float eps;
  float eps_inv_k;   // 1 / k_real (RMSNorm mean)
  int keep_out;      // part persists across launches (the residual stream): never re-zeroed
  float out_alpha;   // scale of the partials the epilogue adds into part
  // E_ATTN: q|k|v of the new token = src->part (f32 [3d]); part = per-(head, split) records
  __half* kc;
  __half* vc;
  const float* cos_t;
  const float* sin_t;
  const int32_t* T_dev;
  int n_heads, d_head, max_ctx;
  float scale;
  const int* bounds;  // optional [G + 1] tile-range boundaries per CTA (pmpd_engine_partition); null = even
  // ---- counted accumulation (linear-stack programs, pmpd_engine_op_set_counted)
  unsigned long long* acc;  // u64 [2][acc_len]: parity sets of counted words (the op's output; for a
                            // residual op the shared residual stream, for an attention op its records)
  long long acc_len;        // words per parity set
  int n_contrib;            // CTAs with a nonempty tile range (each adds 1 to the op's hint counter)
  const unsigned short* cum;  // E_IN_RMSNORM: contributions in each residual word at this point
  int rwait;                  // residual op: the RMSNorm op whose readers must be done before adding
  // tensor parallelism: a row-parallel op adds each partial into every rank's copy of its output
  // (n_peers > 0: peer[0..n_peers), this rank's own copy among them; sys = the copies live on
  // other GPUs: system-scope additions, and their consumers poll with system-scope loads)
  unsigned long long* peer[8];
  int n_peers;
  int sys;
  // sub-ops (pmpd_engine_op_set_slice / pmpd_engine_op_set_share): an op restricted to n-groups
  // [ng_off, ng_off + n_tiles) and k-tiles [k_off, k_off + k_tiles) of a tensor with n_tiles_full
  // x kt_mem tiles; sub-ops of one tensor add into one shared counted output (acc is its base)
  int ng_off, k_off, kt_mem, n_tiles_full;
  long long zero_len;  // words of the idle set this op zeroes (-1: acc_len; 0: another sub-op does)
  // the source op's counted output, copied into this op by pmpd_engine_link so that staging does
  // not first chase the source op's record through L2 (one dependent round trip per op)
  const unsigned long long* src_acc;
  long long src_acc_len;
  const unsigned char* src_nslots;
  int src_sys;
};
constexpr int E_LINEAR = 0, E_ATTN = 1;
constexpr int E_IN_SRC = 0, E_IN_RMSNORM = 2, E_IN_ATTN = 3;
constexpr int E_ASPLIT = 4;  // context splits per head in the attention op
PMPD_DEV int attn_rec(int dh) { return 4 + dh; }  // record: m, l, pad, pad, acc[dh] (16-byte aligned acc)

// ---- counted fixed-point words: [63:54] contributors, [53:0] sum of (rint(v * 2^24) + 2^43)
#ifndef PMPD_ENGINE_NOHINT
#define PMPD_ENGINE_NOHINT 1       // 0: consumers first wait for the relaxed per-op hint counter (measured slower)
#endif
#ifndef PMPD_ENGINE_ROTATE
#define PMPD_ENGINE_ROTATE 0  // 1: round-robin tile slots across stages (0: slot = warp)
#endif
#ifndef PMPD_ENGINE_SLOTMAP
#define PMPD_ENGINE_SLOTMAP 0  // 1: static slot order by scheduler load (needs E_NCW % 4 == 0)
#endif
#ifndef PMPD_ENGINE_RETRY_NS
#define PMPD_ENGINE_RETRY_NS 32    // back-off between re-reads of incomplete words
#endif
#ifndef PMPD_ENGINE_HINT_RELEASE
#define PMPD_ENGINE_HINT_RELEASE 0 // 1: the hint add is a release (orders the data adds before it)
#endif
// Three buffer sets per counted vector, used round-robin by launch epoch: launch L adds into set
// L % 3 and zeroes set (L - 1) % 3, the one launch L + 2 will use.  With peers on other GPUs
// (tensor parallelism) a peer may already be in launch L + 1 adding into set (L + 1) % 3 of this
// rank's copy while this rank finishes launch L, so the set being zeroed is never one a peer can
// still be writing (its last writes to set (L - 1) % 3 were all observed before launch L began).
constexpr int kSets = 3;
constexpr int kCntShift = 54;                  // up to 1023 contributions per word (the residual
                                               // stream accumulates every o / down partial of a step)
constexpr unsigned long long kValMask = (1ull << kCntShift) - 1;
constexpr long long kFixOff = 1ll << 43;       // per-contribution offset: keeps every addend >= 0
constexpr float kFixScale = 16777216.f;        // 2^24
constexpr float kFixUnscale = 5.9604644775390625e-8f;  // 2^-24
constexpr float kFixMax = 524288.f;            // |v| < 2^19 keeps rint(v * 2^24) inside +-2^43
// Contribution word of one partial; a non-finite or out-of-range partial still counts (so no
// consumer waits forever) but adds zero and flags the status word.
PMPD_DEV unsigned long long fix_encode(float v, int* status) {
  long long q = 0;
  if (fabsf(v) < kFixMax)
    q = __float2ll_rn(v * kFixScale);
  else if (status && *reinterpret_cast<volatile int*>(status) == 0)  // (no atomic storm on a NaN row)
    atomicExch(status, PMPD_ERR_INPUT);
  return (1ull << kCntShift) + (unsigned long long)(q + kFixOff);
}
PMPD_DEV int fix_count(unsigned long long w) { return (int)(w >> kCntShift); }
// value of a complete word with `cnt` contributions: one rounding of the exact sum to f32
PMPD_DEV float fix_decode(unsigned long long w, int cnt) {
  const long long t = (long long)(w & kValMask) - (long long)cnt * kFixOff;
  return __ll2float_rn(t) * kFixUnscale;
}
// single-writer words (attention records): count 1, raw f32 bits
PMPD_DEV unsigned long long raw_word(float v) { return (1ull << kCntShift) | (unsigned long long)__float_as_uint(v); }
PMPD_DEV float raw_value(unsigned long long w) { return __uint_as_float((unsigned)w); }
PMPD_DEV void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
PMPD_DEV void ld_relaxed_u64x2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
PMPD_DEV void ld_relaxed_sys_u64x2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
PMPD_DEV unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
PMPD_DEV void red_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
PMPD_DEV unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin watchdog (debug builds, -DPMPD_ENGINE_WATCHDOG): a word that never completes means a
// broken program (wrong counts); abort the launch (a CUDA error the host sees) instead of
// hanging.  Off by default: the trap path on the polling loops costs ~6 % on the 7B token.
PMPD_DEV void spin_watchdog(long long& t0) {
#ifdef PMPD_ENGINE_WATCHDOG
  if (++t0 > (1ll << 26)) __trap();
#endif
}

// Read NB groups of 4 consecutive counted words (16-byte aligned; on[i] = false skips the group
// and returns zeros; want[i] = expected count), re-reading until every word is complete: all
// loads of a round are issued before any check, so a round costs one L2 round trip.  `on` must
// not depend on `want` (the expected counts are loads themselves: the data loads would wait for
// them).  RAW: single-writer words holding f32 bits.
template <int NB, bool RAW = false>
PMPD_DEV void counted_read4(const unsigned long long* const (&p)[NB], const bool (&on)[NB], const int (&want)[NB],
                            float (&out)[NB][4]) {
  unsigned long long w[NB][4];
  long long t0 = 0;
  for (;;) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (on[i]) {
        ld_relaxed_u64x2(p[i], w[i][0], w[i][1]);
        ld_relaxed_u64x2(p[i] + 2, w[i][2], w[i][3]);
      } else {
        w[i][0] = w[i][1] = w[i][2] = w[i][3] = 0ull;
      }
    }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) ok = ok && (!on[i] || fix_count(w[i][e]) == want[i]);
    if (ok) break;
    spin_watchdog(t0);
    if (PMPD_ENGINE_RETRY_NS) __nanosleep(PMPD_ENGINE_RETRY_NS);
  }
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) out[i][e] = !on[i] ? 0.f : RAW ? raw_value(w[i][e]) : fix_decode(w[i][e], want[i]);
}
// Same for N single words (any alignment).
template <int N, bool RAW = false>
PMPD_DEV void counted_read_n(const unsigned long long* const (&p)[N], const int (&want)[N], float (&out)[N]) {
  unsigned long long w[N];
  long long t0 = 0;
  for (;;) {
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = ld_relaxed_u64(p[i]);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && fix_count(w[i]) == want[i];
    if (ok) break;
    spin_watchdog(t0);
    if (PMPD_ENGINE_RETRY_NS) __nanosleep(PMPD_ENGINE_RETRY_NS);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = RAW ? raw_value(w[i]) : fix_decode(w[i], want[i]);
}

// Poll the op's hint counter until every contributing CTA has issued its additions (a hint:
// the words themselves are validated by their counts).
PMPD_DEV void wait_hint(const unsigned* p, unsigned target) {
  long long t0 = 0;
  while ((int)(ld_relaxed_u32(p) - target) < 0) {
    spin_watchdog(t0);
    __nanosleep(32);
  }
}

struct EngineArgs {
  const EngineOp* ops;
  int n_ops;
  const int32_t* p_dev;
  const __half* x_in;  // input of op 0 (f16)
  float* y_out;        // output of the last op (f32), y_alpha * reduced partials
  float y_alpha;
  unsigned* bar;       // [0]: op-completion tickets, [1]: CTAs done (self-resetting), [2]: launch epoch,
                       // [3 + i]: op i's hint counter, [3 + n_ops + i]: readers of RMSNorm op i
  int* status;
  long long* trace;    // optional timeline [G][n_ops][4] (globaltimer ns), null = off
  int n_ranks;         // tensor-parallel emulation: op tables [n_ranks][n_ops], y_out [n_ranks][y_stride]
  int y_stride;
  // decoder programs: the counted residual stream [2][R_len] and its f32 starting value x0
  // (the embedding row), added in by CTA c for its slice at launch start
  unsigned long long* R;
  long long R_len;
  const float* x0;
  int d_real;
};

PMPD_DEV long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// shared-memory plan (byte offsets)
constexpr int kSmBar = 0;                            // mbarriers
constexpr int kSmMisc = 256;                         // mx, flags
constexpr int kSmX = 1536;                           // f16 activations
constexpr int kSmXq = kSmX + E_XMAX * 2;             // per-warp int8 activation fragments
constexpr int kSmRed = kSmXq + E_NCW * E_TPW * 128;  // [2][E_NCW][64] f32
#ifndef PMPD_ENGINE_LANEBIAS
#define PMPD_ENGINE_LANEBIAS 0  // 1: flush: every lane stores its bias partial, the epilogue reduces them
#endif
constexpr int kBiasPerWarp = PMPD_ENGINE_LANEBIAS ? 32 : 1;
constexpr int kSmRedb = kSmRed + 2 * E_NCW * 64 * 4; // [2][E_NCW][kBiasPerWarp] f32
constexpr int kSmRing = (kSmRedb + 2 * E_NCW * kBiasPerWarp * 4 + 127) / 128 * 128;

struct Bars {
  uint64_t full[E_MAXSTAGE];
  uint64_t empty[E_MAXSTAGE];
  uint64_t red_full[2];
  uint64_t red_empty[2];
};

// 32-bit partition arithmetic (NT * (G + 1) < 2^32, checked in pmpd_engine_make_op): a 64-bit
// integer division is an emulated ~100-instruction routine, and it runs on the op-to-op path.

struct Range {
  int T0, T1, KT, NT;
};
PMPD_DEV Range range_of(const EngineOp& op, int c, int G) {
  Range r;
  r.NT = op.n_tiles * op.k_tiles;
  r.KT = op.k_tiles;
  if (op.bounds) {  // cost-balanced partition computed on the host (pmpd_engine_partition)
    r.T0 = __ldg(op.bounds + c);
    r.T1 = __ldg(op.bounds + c + 1);
  } else {
    r.T0 = (int)((unsigned)c * (unsigned)r.NT / (unsigned)G);
    r.T1 = (int)((unsigned)(c + 1) * (unsigned)r.NT / (unsigned)G);
  }
  return r;
}

// L2 prefetch of this CTA's packed tiles of op `op` (active planes + scale blocks).  The smem
// ring holds less than an op's share of the weights, so while the consumers wait at an op
// boundary the ring is full and the TMA stream would stall; prefetching PMPD_ENGINE_PF ops ahead
// into the 126 MB L2 keeps HBM streaming through the op-to-op exchanges, and the ring then
// refills from L2.
#ifndef PMPD_ENGINE_PF
#define PMPD_ENGINE_PF 0  // measured slower at 1-4 ops ahead (round 2): the engine is sync-bound, not stream-bound
#endif
PMPD_DEV void prefetch_op(const EngineOp& op, int c, int G, int p) {
  if (op.kind != E_LINEAR || op.kt_mem != op.k_tiles) return;  // (k-sliced ops: not contiguous)
  const Range r = range_of(op, c, G);
  if (r.T1 <= r.T0) return;
  const uint32_t n = (uint32_t)(r.T1 - r.T0) * kTilePlaneBytes;
  for (int j = 0; j < p; ++j) bulk_prefetch_l2(op.planes + j * op.plane_bytes + (int64_t)r.T0 * kTilePlaneBytes, n);
  bulk_prefetch_l2(op.scales + (int64_t)r.T0 * kTileScaleBytes, (uint32_t)(r.T1 - r.T0) * kTileScaleBytes);
}

// Rolling L2 prefetch (PMPD_ENGINE_PFT tiles ahead of the TMA loads, issued in step with them):
// the cursor (pop, pt) walks this CTA's tiles op by op; pt < 0 = start of op pop's range.
#ifndef PMPD_ENGINE_PFT
#define PMPD_ENGINE_PFT 0
#endif
#ifndef PMPD_ENGINE_PFB
#define PMPD_ENGINE_PFB 0  // prefetch-when-blocked lead in tiles (0: off)
#endif
PMPD_DEV void pf_advance(const EngineOp* ops, int n_ops, int c, int G, int p, int& pop, int& pt, int n,
                         bool issue = true) {
  while (n > 0 && pop < n_ops) {
    const EngineOp& op = ops[pop];
    if (op.kind != E_LINEAR || op.kt_mem != op.k_tiles) {
      ++pop;
      pt = -1;
      continue;
    }
    const Range r = range_of(op, c, G);
    if (pt < r.T0) pt = r.T0;
    const int m = min(n, r.T1 - pt);
    if (m > 0) {
      const uint32_t nb = (uint32_t)m * kTilePlaneBytes;
      if (issue) {
        for (int j = 0; j < p; ++j)
          bulk_prefetch_l2(op.planes + j * op.plane_bytes + (int64_t)pt * kTilePlaneBytes, nb);
        bulk_prefetch_l2(op.scales + (int64_t)pt * kTileScaleBytes, (uint32_t)m * kTileScaleBytes);
      }
      pt += m;
      n -= m;
    }
    if (pt >= r.T1) {
      ++pop;
      pt = -1;
    }
  }
}

// ------------------------------------------------------------------ attention op
// One decode query over the KV cache of one layer (tinylm.py:344-358), as engine work units
// (head h, split s): RoPE of q (and of the new k, by the unit holding position T, which also
// appends k and v to the cache, tinylm.py:308-319), then the 12 consumer warps stream the
// unit's rows with an online softmax; the CTA folds the warps into one record (m, l, acc) that
// the next op's staging combines (E_IN_ATTN).  scratch: [E_NCW][4 + dh] f32 (shared).
template <int DPL>
PMPD_DEV void ld_halves(const __half* __restrict__ p, bool ok, float (&f)[DPL]) {
  if (!ok) {
#pragma unroll
    for (int j = 0; j < DPL; ++j) f[j] = 0.f;
    return;
  }
  if constexpr (DPL == 1) {
    f[0] = __half2float(*p);
  } else if constexpr (DPL == 2) {
    const float2 v = __half22float2(*reinterpret_cast<const __half2*>(p));
    f[0] = v.x;
    f[1] = v.y;
  } else {
    constexpr int W = DPL / 2;  // 32-bit words: 2 (uint2) or 4 (uint4)
    uint32_t w[W];
    if constexpr (DPL == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(p);
      w[0] = u.x;
      w[1] = u.y;
    } else {
      const uint4 u = *reinterpret_cast<const uint4*>(p);
      w[0] = u.x;
      w[1] = u.y;
      w[2] = u.z;
      w[3] = u.w;
    }
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      f[2 * i] = v.x;
      f[2 * i + 1] = v.y;
    }
  }
}

// Raw f16 storage of DPL halves (K/V rows kept packed in registers: two rows in flight per
// register budget of one converted row).
template <int DPL>
struct RawRow {
  static constexpr int W = DPL >= 2 ? DPL / 2 : 1;
  uint32_t w[W];
};
template <int DPL>
PMPD_DEV void ld_raw(const __half* __restrict__ p, bool ok, RawRow<DPL>& r) {
  if (!ok) {
#pragma unroll
    for (int i = 0; i < RawRow<DPL>::W; ++i) r.w[i] = 0u;
    return;
  }
  if constexpr (DPL == 1) {
    r.w[0] = (uint32_t)__half_as_ushort(*p);
  } else if constexpr (DPL == 2) {
    r.w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else if constexpr (DPL == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    r.w[0] = u.x;
    r.w[1] = u.y;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    r.w[0] = u.x;
    r.w[1] = u.y;
    r.w[2] = u.z;
    r.w[3] = u.w;
  }
}
template <int DPL>
PMPD_DEV void raw_to_f(const RawRow<DPL>& r, float (&f)[DPL]) {
  if constexpr (DPL == 1) {
    f[0] = __half2float(__ushort_as_half((unsigned short)r.w[0]));
  } else {
#pragma unroll
    for (int i = 0; i < DPL / 2; ++i) {
      const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&r.w[i]));
      f[2 * i] = v.x;
      f[2 * i + 1] = v.y;
    }
  }
}

// DPL consecutive counted words of the q|k|v op's output starting at element n
template <int DPL>
PMPD_DEV void read_qkv(const EngineOp& src, const unsigned long long* base, int n, float (&f)[DPL]) {
  const int want = __ldg(src.nslots + (n >> 6));
  if constexpr (DPL >= 4) {
    const unsigned long long* pp[DPL / 4];
    bool on[DPL / 4];
    int ww[DPL / 4];
    float o[DPL / 4][4];
#pragma unroll
    for (int i = 0; i < DPL / 4; ++i) {
      pp[i] = base + n + 4 * i;
      on[i] = true;
      ww[i] = want;
    }
    counted_read4<DPL / 4>(pp, on, ww, o);
#pragma unroll
    for (int i = 0; i < DPL; ++i) f[i] = o[i / 4][i % 4];
  } else {
    const unsigned long long* pp[DPL];
    int ww[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      pp[i] = base + n + i;
      ww[i] = want;
    }
    counted_read_n<DPL>(pp, ww, f);
  }
}

// q, k and v of one lane (3 x DPL counted words) in ONE round trip
template <int DPL>
PMPD_DEV void read_qkv3(const EngineOp& src, const unsigned long long* base, int nq, int d, float (&q)[DPL],
                        float (&k)[DPL], float (&v)[DPL]) {
  const int ns[3] = {nq, nq + d, nq + 2 * d};
  if constexpr (DPL >= 4) {
    constexpr int NB = 3 * (DPL / 4);
    const unsigned long long* pp[NB];
    bool on[NB];
    int ww[NB];
    float o[NB][4];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int n = ns[i / (DPL / 4)] + 4 * (i % (DPL / 4));
      pp[i] = base + n;
      on[i] = true;
      ww[i] = __ldg(src.nslots + (n >> 6));
    }
    counted_read4<NB>(pp, on, ww, o);
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      q[i] = o[i / 4][i % 4];
      k[i] = o[DPL / 4 + i / 4][i % 4];
      v[i] = o[2 * (DPL / 4) + i / 4][i % 4];
    }
  } else {
    const unsigned long long* pp[3 * DPL];
    int ww[3 * DPL];
    float o[3 * DPL];
#pragma unroll
    for (int i = 0; i < 3 * DPL; ++i) {
      const int n = ns[i / DPL] + i % DPL;
      pp[i] = base + n;
      ww[i] = __ldg(src.nslots + (n >> 6));
    }
    counted_read_n<3 * DPL>(pp, ww, o);
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      q[i] = o[i];
      k[i] = o[DPL + i];
      v[i] = o[2 * DPL + i];
    }
  }
}

#ifndef PMPD_ATTN_NOLOAD
#define PMPD_ATTN_NOLOAD 0
#endif
#ifndef PMPD_ATTN_DB
#define PMPD_ATTN_DB 0  // 1: two row batches in flight per warp
#endif
template <int DPL>
PMPD_DEV void attn_unit(const EngineOp& op, const EngineOp& src, int h, int s, int L, float* scratch, int warp,
                        int lane, int par, float* newrow, long long* tr) {
  constexpr int DH = 32 * DPL, HALF = DH / 2;
  constexpr int U = DPL <= 2 ? 8 : DPL == 4 ? 4 : 1;  // rows per batch per warp (two batches in flight, packed f16)
  const int d = op.n_heads * DH;
  const int chunk = (L + E_ASPLIT - 1) / E_ASPLIT;
  const int t0 = s * chunk, t1 = min(L, t0 + chunk);
  const int pos = L - 1;
  const bool append = *op.T_dev < op.max_ctx;  // row `pos` is this token's (written below)
  const bool first = lane < 16;
  const __half* kb = op.kc + h * DH + lane * DPL;
  const __half* vb = op.vc + h * DH + lane * DPL;
  // ---- independent of this token's q|k|v: issued before the ticket wait (bar != null)
  float c[DPL], sn[DPL];
#pragma unroll
  for (int j = 0; j < DPL; ++j) {
    const int jj = (lane * DPL + j) % HALF;
    c[j] = __ldg(op.cos_t + (int64_t)pos * HALF + jj);
    sn[j] = __ldg(op.sin_t + (int64_t)pos * HALF + jj);
  }
  // K/V rows of the next batch as packed f16 (issued before the q wait: independent of this token;
  // in the loop each batch is converted, then the following one is issued while it is used)
  RawRow<DPL> kc[U], vc[U];
#if PMPD_ATTN_DB
  RawRow<DPL> kn[U], vn[U];  // a second batch in flight
#endif
  const int tb0 = t0 + warp;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t = tb0 + u * E_NCW;
    const bool ok = !PMPD_ATTN_NOLOAD && t < t1 && !(append && t == pos);
    ld_raw<DPL>(kb + (int64_t)t * d, ok, kc[u]);
    ld_raw<DPL>(vb + (int64_t)t * d, ok, vc[u]);
#if PMPD_ATTN_DB
    const int t2 = t + U * E_NCW;
    const bool ok2 = !PMPD_ATTN_NOLOAD && t2 < t1 && !(append && t2 == pos);
    ld_raw<DPL>(kb + (int64_t)t2 * d, ok2, kn[u]);
    ld_raw<DPL>(vb + (int64_t)t2 * d, ok2, vn[u]);
#endif
  }
  // ---- q (and the new k, v) of this token: counted words of the q|k|v op (blocks until complete)
  const unsigned long long* qkv = src.acc + (long long)par * src.acc_len;
  float qr[DPL];
  const bool app = append && pos >= t0 && pos < t1;
  if (app && warp == 0) {
    // the unit holding position T: q, k and v in one round trip; k (post-RoPE) and v go to the
    // cache and, rounded to f16 as the cache holds them, to shared memory for the warp that owns
    // row T in this unit (no global re-read)
    float qa[DPL], ka[DPL], va[DPL];
    read_qkv3<DPL>(src, qkv, h * DH + lane * DPL, d, qa, ka, va);
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
      const float a = qa[j];
      const float b = __shfl_xor_sync(0xffffffffu, a, 16);  // RoPE partner dim j +- HALF
      qr[j] = first ? a * c[j] - b * sn[j] : a * c[j] + b * sn[j];
      const float ak = ka[j];
      const float bk = __shfl_xor_sync(0xffffffffu, ak, 16);
      const __half kh = __float2half(first ? ak * c[j] - bk * sn[j] : ak * c[j] + bk * sn[j]);
      const __half vh = __float2half(va[j]);
      op.kc[(int64_t)pos * d + h * DH + lane * DPL + j] = kh;
      op.vc[(int64_t)pos * d + h * DH + lane * DPL + j] = vh;
      newrow[lane * DPL + j] = __half2float(kh);
      newrow[DH + lane * DPL + j] = __half2float(vh);
    }
  } else {
    float qa[DPL];
    read_qkv<DPL>(src, qkv, h * DH + lane * DPL, qa);
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
      const float a = qa[j];
      const float b = __shfl_xor_sync(0xffffffffu, a, 16);  // RoPE partner dim j +- HALF
      qr[j] = first ? a * c[j] - b * sn[j] : a * c[j] + b * sn[j];
    }
  }
  named_bar_sync(1, E_NCW * 32);  // the new row (shared memory) is visible to every warp of the CTA
  if (tr && threadIdx.x == 0) tr[1] = gtimer();
  if (app) {  // the first batch skipped row `pos`: take it from shared memory
#pragma unroll
    for (int u = 0; u < U; ++u) {
#if PMPD_ATTN_DB
      if (tb0 + (U + u) * E_NCW == pos) {  // (second batch: the converted row goes there)
        float kf1[DPL], vf1[DPL];
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
          kf1[j] = newrow[lane * DPL + j];
          vf1[j] = newrow[DH + lane * DPL + j];
        }
        if constexpr (DPL == 1) {
          kn[u].w[0] = (uint32_t)__half_as_ushort(__float2half(kf1[0]));
          vn[u].w[0] = (uint32_t)__half_as_ushort(__float2half(vf1[0]));
        } else {
#pragma unroll
          for (int i = 0; i < DPL / 2; ++i) {
            const __half2 k2 = __floats2half2_rn(kf1[2 * i], kf1[2 * i + 1]);
            const __half2 v2 = __floats2half2_rn(vf1[2 * i], vf1[2 * i + 1]);
            kn[u].w[i] = *reinterpret_cast<const uint32_t*>(&k2);
            vn[u].w[i] = *reinterpret_cast<const uint32_t*>(&v2);
          }
        }
      }
#endif
      if (tb0 + u * E_NCW == pos) {
        float kf1[DPL], vf1[DPL];
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
          kf1[j] = newrow[lane * DPL + j];
          vf1[j] = newrow[DH + lane * DPL + j];
        }
        RawRow<DPL> kr1, vr1;
        if constexpr (DPL == 1) {
          kr1.w[0] = (uint32_t)__half_as_ushort(__float2half(kf1[0]));
          vr1.w[0] = (uint32_t)__half_as_ushort(__float2half(vf1[0]));
        } else {
#pragma unroll
          for (int i = 0; i < DPL / 2; ++i) {
            const __half2 k2 = __floats2half2_rn(kf1[2 * i], kf1[2 * i + 1]);
            const __half2 v2 = __floats2half2_rn(vf1[2 * i], vf1[2 * i + 1]);
            kr1.w[i] = *reinterpret_cast<const uint32_t*>(&k2);
            vr1.w[i] = *reinterpret_cast<const uint32_t*>(&v2);
          }
        }
        kc[u] = kr1;
        vc[u] = vr1;
      }
    }
  }
  float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
  for (int j = 0; j < DPL; ++j) acc[j] = 0.f;
  for (int tb = tb0; tb < t1; tb += E_NCW * U) {
    float kf[U][DPL], vf[U][DPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      raw_to_f<DPL>(kc[u], kf[u]);
      raw_to_f<DPL>(vc[u], vf[u]);
#if PMPD_ATTN_DB
      kc[u] = kn[u];
      vc[u] = vn[u];
#endif
    }
    constexpr int AHEAD = PMPD_ATTN_DB ? 2 : 1;  // batches in flight
    if (tb + AHEAD * E_NCW * U < t1) {  // the next batch(es) in flight while this one is used
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = tb + (AHEAD * U + u) * E_NCW;
#if PMPD_ATTN_DB
        ld_raw<DPL>(kb + (int64_t)t * d, !PMPD_ATTN_NOLOAD && t < t1, kn[u]);
        ld_raw<DPL>(vb + (int64_t)t * d, !PMPD_ATTN_NOLOAD && t < t1, vn[u]);
#else
        ld_raw<DPL>(kb + (int64_t)t * d, !PMPD_ATTN_NOLOAD && t < t1, kc[u]);
        ld_raw<DPL>(vb + (int64_t)t * d, !PMPD_ATTN_NOLOAD && t < t1, vc[u]);
#endif
      }
    }
    float sc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < DPL; ++j) a = fmaf(qr[j], kf[u][j], a);
      sc[u] = a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
    // online softmax, one rescale per batch: the U exponentials are independent (round 1 chained
    // a rescale through every row)
    float bm = m;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      sc[u] = tb + u * E_NCW < t1 ? sc[u] * op.scale : -INFINITY;
      bm = fmaxf(bm, sc[u]);
    }
    if (bm != -INFINITY) {
      const float corr = __expf(m - bm);  // m = -inf on the first rows: 0
      float ps = 0.f, pv[DPL];
#pragma unroll
      for (int j = 0; j < DPL; ++j) pv[j] = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float pe = __expf(sc[u] - bm);  // -inf rows: 0
        ps += pe;
#pragma unroll
        for (int j = 0; j < DPL; ++j) pv[j] = fmaf(pe, vf[u][j], pv[j]);
      }
      l = fmaf(l, corr, ps);
#pragma unroll
      for (int j = 0; j < DPL; ++j) acc[j] = fmaf(acc[j], corr, pv[j]);
      m = bm;
    }
  }
  float* wr = scratch + warp * (4 + DH);
  if (lane == 0) {
    wr[0] = m;
    wr[1] = l;
  }
#pragma unroll
  for (int j = 0; j < DPL; ++j) wr[4 + lane * DPL + j] = acc[j];
  named_bar_sync(1, E_NCW * 32);
  if (tr && threadIdx.x == 0) tr[3] = gtimer();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < E_NCW; ++w) M = fmaxf(M, scratch[w * (4 + DH)]);
  // single-writer record words (count 1, raw f32): the combine in the o op's staging polls them
  unsigned long long* rec = op.acc + (long long)par * op.acc_len + (int64_t)(h * E_ASPLIT + s) * (4 + DH);
  for (int e = threadIdx.x; e < DH + 2; e += E_NCW * 32) {
    float v = 0.f;
    for (int w = 0; w < E_NCW; ++w) {
      const float mw = scratch[w * (4 + DH)];
      const float wt = mw == -INFINITY ? 0.f : __expf(mw - M);
      v = fmaf(e < DH ? scratch[w * (4 + DH) + 4 + e] : scratch[w * (4 + DH) + 1], wt, v);
    }
    if (e < DH)
      st_relaxed_u64(rec + 4 + e, raw_word(v));
    else if (e == DH)
      st_relaxed_u64(rec + 1, raw_word(v));  // l
    else
      st_relaxed_u64(rec, raw_word(M));      // m
  }
  named_bar_sync(1, E_NCW * 32);  // scratch reused by the next unit
}

// The attention op of one CTA: its units (head, split) in turn.  Each unit issues the K/V cache
// loads that do not depend on this token before it waits for the token's q|k|v words.
__noinline__ __device__ void attn_op(const EngineOp& op, const EngineOp& src, int c, int G, float* scratch, int warp,
                                    int lane, int par, float* newrow, long long* tr) {
  const int L = min(*op.T_dev + 1, op.max_ctx);
  for (int u = c; u < op.n_heads * E_ASPLIT; u += G) {
    const int h = u / E_ASPLIT, s = u - h * E_ASPLIT;
    switch (op.d_head) {
      case 32: attn_unit<1>(op, src, h, s, L, scratch, warp, lane, par, newrow, tr); break;
      case 64: attn_unit<2>(op, src, h, s, L, scratch, warp, lane, par, newrow, tr); break;
      case 128: attn_unit<4>(op, src, h, s, L, scratch, warp, lane, par, newrow, tr); break;
      default: attn_unit<8>(op, src, h, s, L, scratch, warp, lane, par, newrow, tr); break;
    }
    tr = nullptr;
  }
}

// E_IN_ATTN staging (kept out of line: its live registers of split records would otherwise
// count against the consumer loop's tile body).  Returns max |x| of the staged f16 row.
__noinline__ __device__ float stage_attn_input(const EngineOp& op, const EngineOp& src, int lo0, int hi0, int lo1,
                                               int hi1, __half* xs, float* wscratch, int par, long long* tr) {
  float mx = 0.f;
  // only this CTA's k-tile ranges [lo0, hi0) and [lo1, hi1) are staged (the tiles read nothing
  // else): element u of the concatenated ranges maps to k = kof(u)
  const int len0 = (hi0 - lo0) * kTile, lr = len0 + (hi1 - lo1) * kTile;
  auto kof = [&](int u) { return u < len0 ? lo0 * kTile + u : lo1 * kTile + (u - len0); };
  // Each element combines the E_ASPLIT split records of its head (single-writer words of the
  // attention op, polled until written) with the per-(head, split) softmax weights
  // w = exp(m_s - M_h) / sum_s exp(m_s - M_h) l_s.  Every thread reads the values of up to SBA
  // batches of 4 elements, then the first n_heads threads the (m, l) words (written with the
  // values, so rarely re-polled) and the weights.  A range wider than one pass (rare: more than
  // 4 * SBA * threads elements in one CTA) is staged in passes after the weights.
  // (Measured: weights on dedicated warps in parallel with the values, 1.5 % slower on the 1.4B
  // decoder; weights first, then values, 1-3 % slower.)
  constexpr int SBA = 3;
  const int dh = src.d_head;
  const unsigned long long* recs = src.acc + (long long)par * src.acc_len;
  const int n_heads = src.n_heads;
  const int wthr = (n_heads + 31) & ~31;
  const int all = E_NCW * 32;
  (void)wthr;
  const bool one_pass = 4 * SBA * all >= lr;
  float* wts = wscratch;
  auto weights = [&](int hh) {
    const unsigned long long* pp[2 * E_ASPLIT];
    int ww[2 * E_ASPLIT];
    float ml[2 * E_ASPLIT];
#pragma unroll
    for (int q = 0; q < E_ASPLIT; ++q) {
      pp[2 * q] = recs + (int64_t)(hh * E_ASPLIT + q) * attn_rec(dh);
      pp[2 * q + 1] = pp[2 * q] + 1;
      ww[2 * q] = ww[2 * q + 1] = 1;
    }
    counted_read_n<2 * E_ASPLIT, true>(pp, ww, ml);
    float ms[E_ASPLIT], M = -INFINITY;
#pragma unroll
    for (int q = 0; q < E_ASPLIT; ++q) {
      ms[q] = ml[2 * q];
      M = fmaxf(M, ms[q]);
    }
    float den = 0.f;
#pragma unroll
    for (int q = 0; q < E_ASPLIT; ++q) {
      ms[q] = ms[q] == -INFINITY ? 0.f : __expf(ms[q] - M);
      den = fmaf(ms[q], ml[2 * q + 1], den);
    }
    const float id = den > 0.f ? __frcp_rn(den) : 0.f;
#pragma unroll
    for (int q = 0; q < E_ASPLIT; ++q) wts[hh * E_ASPLIT + q] = ms[q] * id;
  };
  // values of elements u = 4*vt + bi*4*vn + base (bi < SBA) into av, then (after the weights are
  // in shared memory) combined into xs
  auto values = [&](float (&av)[SBA * E_ASPLIT][4], int vt, int vn, int base) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      constexpr int NBH = 2 * E_ASPLIT;
      const unsigned long long* pp[NBH];
      bool on[NBH];
      int ww[NBH];
      float o[NBH][4];
      bool any = false;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int bi = 2 * half + b;
        const int u = base + 4 * vt + bi * 4 * vn;
        const int k = (bi < SBA && u < lr) ? kof(u) : op.k_real;
        const int hh = k < op.k_real ? k / dh : 0, e = k - hh * dh;
#pragma unroll
        for (int q = 0; q < E_ASPLIT; ++q) {
          pp[b * E_ASPLIT + q] = recs + (int64_t)(hh * E_ASPLIT + q) * attn_rec(dh) + 4 + e;
          on[b * E_ASPLIT + q] = k < op.k_real;
          ww[b * E_ASPLIT + q] = 1;
        }
        any = any || k < op.k_real;
      }
      if (!any) {
#pragma unroll
        for (int i = 0; i < NBH; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      } else {
        counted_read4<NBH, true>(pp, on, ww, o);
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int bi = 2 * half + b;
        if (bi >= SBA) break;
#pragma unroll
        for (int q = 0; q < E_ASPLIT; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i) av[bi * E_ASPLIT + q][i] = o[b * E_ASPLIT + q][i];
      }
    }
  };
  auto combine = [&](const float (&av)[SBA * E_ASPLIT][4], int vt, int vn, int base) {
#pragma unroll
    for (int bi = 0; bi < SBA; ++bi) {
      const int u = base + 4 * vt + bi * 4 * vn;
      if (u >= lr) break;
      const int k = kof(u);
      float o[4] = {0.f, 0.f, 0.f, 0.f};
      if (k < op.k_real) {
        const int hh = k / dh;
#pragma unroll
        for (int q = 0; q < E_ASPLIT; ++q) {
          const float w = wts[hh * E_ASPLIT + q];
#pragma unroll
          for (int e = 0; e < 4; ++e) o[e] = fmaf(w, av[bi * E_ASPLIT + q][e], o[e]);
        }
      }
      const __half2 h01 = __floats2half2_rn(o[0], o[1]), h23 = __floats2half2_rn(o[2], o[3]);
      *reinterpret_cast<__half2*>(xs + k) = h01;
      *reinterpret_cast<__half2*>(xs + k + 2) = h23;
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(f01.x), fabsf(f01.y)), fmaxf(fabsf(f23.x), fabsf(f23.y))));
    }
  };
  float av[SBA * E_ASPLIT][4];
  if (one_pass) {
    values(av, threadIdx.x, all, 0);
    if (tr && threadIdx.x == 0) tr[4] = gtimer();  // (PMPD_ENGINE_TRACE_ATTNSTAGE) values read
    for (int hh = threadIdx.x; hh < n_heads; hh += all) weights(hh);
    if (tr && threadIdx.x == 0) tr[5] = gtimer();
    named_bar_sync(1, E_NCW * 32);
    combine(av, threadIdx.x, all, 0);
  } else {
    for (int hh = threadIdx.x; hh < n_heads; hh += all) weights(hh);
    named_bar_sync(1, E_NCW * 32);
    for (int base = 0; base < lr; base += 4 * SBA * all) {
      values(av, threadIdx.x, all, base);
      combine(av, threadIdx.x, all, base);
    }
  }
  return mx;
}

// ------------------------------------------------------------------ kernel
template <bool DEC, bool TP>
PMPD_DEV void consumer_loop(const int P, const EngineArgs& a, uint8_t* smem, Bars& bars, int G, int c,
                            int stage_bytes, int nstage, unsigned epoch) {
  const int par = (int)(epoch % kSets);  // counted programs: the buffer set of this launch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tig = lane & 3;
  __half* xs = reinterpret_cast<__half*>(smem + kSmX);
  uint8_t* xq = smem + kSmXq + warp * E_TPW * 128;
  float* misc = reinterpret_cast<float*>(smem + kSmMisc);
  float* red = reinterpret_cast<float*>(smem + kSmRed);
  float* redb = reinterpret_cast<float*>(smem + kSmRedb);
  int slot = 0;     // ring slot (continues across ops)
  // Tile slots of a stage go to the warps round-robin, continuing where the previous stage
  // stopped: a partial stage (an n-group of 64 tiles is 24 + 24 + 16) gives its extra tiles to
  // different warps each time instead of always warps 0..3 (the last warp sets the op's end)
  int rot = 0;
  uint32_t phase = 0;
  int seg = 0;      // n-group segment counter (red double buffer)
  for (int oi = 0; oi < a.n_ops; ++oi) {
    const EngineOp& op = a.ops[oi];
    if (DEC && op.kind == E_ATTN) {
      // scratch: the warps' partial records (xs area); the appended row: the xq area (2 x d_head f32)
      const bool units = c < op.n_heads * E_ASPLIT;
      if (a.trace && threadIdx.x == 0 && units) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 0] = gtimer();
      attn_op(op, a.ops[op.src], c, G, reinterpret_cast<float*>(smem + kSmX), warp, lane, par,
              reinterpret_cast<float*>(smem + kSmXq), a.trace ? a.trace + ((int64_t)c * a.n_ops + oi) * 8 : nullptr);
      named_bar_sync(1, E_NCW * 32);  // scratch (xs) is reused by the next op's staging
      if (a.trace && threadIdx.x == 0 && units) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 2] = gtimer();
      continue;
    }
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
    // RMSNorm input of a row that fits one pass (K <= 4 * RN * 384): the gain is static, so its
    // loads are issued before the input wait and only the residual's round trip is on the op path
    constexpr int RN = 4, RN_K = 4 * RN * E_NCW * 32;
    const bool busy = r.T1 > r.T0;  // a CTA with no tiles in this op reads no input at all
    if (!busy) continue;             // (nor joins its staging barrier)
#if PMPD_ENGINE_PREDECODE
    // the op's first stage is usually in shared memory already: decode this warp's first tile of
    // it now, while the input is being staged (the ALU is otherwise idle until the exchange lands)
    uint32_t fa[2][4][4];
    bool pre = false;
    {
      const int end0 = min(min(r.T0 + E_STILES, r.T1), r.T0 - r.T0 % r.KT + r.KT);
      if (warp < end0 - r.T0 && mbar_try_wait(&bars.full[slot], phase)) {
        predecode_dispatch(P, smem + kSmRing + slot * stage_bytes, warp, lane, fa);
        pre = true;
      }
    }
#endif
    const bool rms1 = DEC && busy && op.in_mode == E_IN_RMSNORM && op.k_real <= RN_K;
    float4 gpre[RN];
    if (DEC) {
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        const int k = 4 * threadIdx.x + j * 4 * E_NCW * 32;
        gpre[j] = rms1 && k < op.k_real ? __ldg(reinterpret_cast<const float4*>(op.gain + k))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (!PMPD_ENGINE_NOHINT && op.src >= 0 && busy) {
      // wait (relaxed) until every contributor of the source op has issued its additions; the
      // staging below validates each word's count, so this only avoids polling the data lines
      // while they are still being produced
      if (threadIdx.x == 0) wait_hint(a.bar + 3 + op.src, (epoch + 1u) * (unsigned)a.ops[op.src].n_contrib);
      named_bar_sync(1, E_NCW * 32);
    }
    if (a.trace && threadIdx.x == 0) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 0] = gtimer();
#ifdef PMPD_ENGINE_TRACE_WARPS
    if (a.trace && threadIdx.x == 0) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 7] = 0x7fffffffffffffffll;
#endif
    float mx = 0.f;
    // a sub-op of the op whose whole input this CTA staged last: xs and max|x| are still valid
    const EngineOp* src = op.src >= 0 ? &a.ops[op.src] : nullptr;
    float inv = 1.f;  // E_IN_RMSNORM: 1 / sqrt(mean(resid^2) + eps) over the whole row
    // the counted residual stream R of this launch (decoder programs)
    const unsigned long long* Rp = DEC ? a.R + (long long)par * a.R_len : nullptr;
    if (DEC && rms1) {
      // one pass: resid * gain stays in registers while the sum of squares is reduced, then the
      // whole normalised row is written to xs as f16 (max |x| over the row, not just the k-range).
      // The residual words hold x0 plus every o / down partial so far: complete when their
      // count reaches cum[n-group] (static).
      float4 rg[RN];
      float ss = 0.f;
      {
        const unsigned long long* pp[RN];
        bool on[RN];
        int ww[RN];
        float q[RN][4];
#pragma unroll
        for (int j = 0; j < RN; ++j) {
          const int k = 4 * threadIdx.x + j * 4 * E_NCW * 32;
          on[j] = k < op.k_real;
          pp[j] = Rp + (on[j] ? k : 0);
          ww[j] = on[j] ? (int)__ldg(op.cum + (k >> 6)) : 0;
        }
        counted_read4<RN>(pp, on, ww, q);
#pragma unroll
        for (int j = 0; j < RN; ++j) {
          ss = fmaf(q[j][0], q[j][0], fmaf(q[j][1], q[j][1], fmaf(q[j][2], q[j][2], fmaf(q[j][3], q[j][3], ss))));
          rg[j] = make_float4(q[j][0] * gpre[j].x, q[j][1] * gpre[j].y, q[j][2] * gpre[j].z, q[j][3] * gpre[j].w);
        }
      }
      ss = warp_sum(ss);
      if (lane == 0) misc[32 + warp] = ss;
      named_bar_sync(1, E_NCW * 32);
      // this CTA has read its residual version: the next residual op may add into R (rwait)
      if (threadIdx.x == 0)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + 3 + a.n_ops + oi) : "memory");
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < E_NCW; ++w) tot += misc[32 + w];
      inv = rsqrtf(tot * op.eps_inv_k + op.eps);
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        const int k = 4 * threadIdx.x + j * 4 * E_NCW * 32;
        if (k < r.KT * kTile) {
          // (x * g) * inv: tinylm.py:293-295 up to one rounding order; zero past k_real
          const __half2 h01 = __floats2half2_rn(rg[j].x * inv, rg[j].y * inv);
          const __half2 h23 = __floats2half2_rn(rg[j].z * inv, rg[j].w * inv);
          *reinterpret_cast<__half2*>(xs + k) = h01;
          *reinterpret_cast<__half2*>(xs + k + 2) = h23;
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(f01.x), fabsf(f01.y)), fmaxf(fabsf(f23.x), fabsf(f23.y))));
        }
      }
      hi0 = hi1 = 0;  // staged already
      lo0 = lo1 = 0;
    } else if (DEC && busy && op.in_mode == E_IN_RMSNORM) {
      // one L2 pass: the whole f32 row lands in xs above the f16 staging area (bytes
      // [2*KT*64, 2*KT*64 + 4*K), checked at set_io) while its sum of squares accumulates; the
      // k-range is then staged from there without overlapping the f16 writes
      float* row = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(xs) + 2 * r.KT * kTile);
      float ss = 0.f;
      constexpr int RB = 4;
      for (int k0 = 4 * threadIdx.x; k0 < op.k_real; k0 += 4 * RB * E_NCW * 32) {
        const unsigned long long* pp[RB];
        bool on[RB];
        int ww[RB];
        float q[RB][4];
        float4 gq[RB];  // the gain rides in the same round trip; the row is stored as resid * gain
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          const int k = k0 + j * 4 * E_NCW * 32;
          on[j] = k < op.k_real;
          pp[j] = Rp + (on[j] ? k : 0);
          ww[j] = on[j] ? (int)__ldg(op.cum + (k >> 6)) : 0;
          gq[j] = k < op.k_real ? __ldg(reinterpret_cast<const float4*>(op.gain + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        counted_read4<RB>(pp, on, ww, q);
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          const int k = k0 + j * 4 * E_NCW * 32;
          ss = fmaf(q[j][0], q[j][0], fmaf(q[j][1], q[j][1], fmaf(q[j][2], q[j][2], fmaf(q[j][3], q[j][3], ss))));
          if (k < op.k_real)
            *reinterpret_cast<float4*>(row + k) =
                make_float4(q[j][0] * gq[j].x, q[j][1] * gq[j].y, q[j][2] * gq[j].z, q[j][3] * gq[j].w);
        }
      }
      ss = warp_sum(ss);
      if (lane == 0) misc[32 + warp] = ss;  // (misc[8..] holds max |x| below)
      named_bar_sync(1, E_NCW * 32);
      if (threadIdx.x == 0)
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + 3 + a.n_ops + oi) : "memory");
      float tot = 0.f;
#pragma unroll
      for (int w = 0; w < E_NCW; ++w) tot += misc[32 + w];
      inv = rsqrtf(tot * op.eps_inv_k + op.eps);
    } else if (DEC && op.in_mode == E_IN_RMSNORM) {
      hi0 = hi1 = lo0 = lo1 = 0;  // no tiles: nothing to stage
    } else if (DEC && op.in_mode == E_IN_ATTN) {
#ifdef PMPD_ENGINE_TRACE_ATTNSTAGE
      long long* atr = a.trace ? a.trace + ((int64_t)c * a.n_ops + oi) * 8 : nullptr;
#else
      long long* atr = nullptr;
#endif
      if (busy) mx = stage_attn_input(op, *src, lo0, hi0, lo1, hi1, xs, reinterpret_cast<float*>(smem + kSmXq), par, atr);
      hi0 = hi1 = 0;  // staged already (the generic loop below runs no iteration)
      lo0 = lo1 = 0;
    }
    // Each thread stages groups of 4 consecutive elements, SB groups per batch: all loads of a
    // batch are issued before any check (one L2 round trip per batch).
    // the op's staging fields in registers: the polling loads below clobber memory, so op.* would
    // be re-read (an L1 round trip on the exchange's critical path) on every batch and retry
    const int s_src_col = op.src_col, s_act_off = op.act_off, s_act = op.act, s_k_real = op.k_real;
    const float s_in_alpha = op.in_alpha;
    const unsigned long long* const s_src_acc = op.src_acc;
    const long long s_src_acc_len = op.src_acc_len;
    const unsigned char* const s_src_nslots = op.src_nslots;
    const int s_src_sys = op.src_sys;
    (void)s_src_sys;
    constexpr int SB = PMPD_ENGINE_SB;
    for (int seg2 = 0; seg2 < 2; ++seg2) {
      const int klo = (seg2 ? lo1 : lo0) * kTile, khi = (seg2 ? hi1 : hi0) * kTile;
      for (int kb = klo + 4 * threadIdx.x; kb < khi; kb += 4 * SB * E_NCW * 32) {
        float v[SB][4];
        if (DEC && op.in_mode == E_IN_RMSNORM) {
          const float* row = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(xs) + 2 * r.KT * kTile);
#pragma unroll
          for (int bi = 0; bi < SB; ++bi) {
            const int k = kb + bi * 4 * E_NCW * 32;
            const float4 rg =
                (k < khi && k < s_k_real) ? *reinterpret_cast<const float4*>(row + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            v[bi][0] = rg.x * inv;  // (x * g) * inv: tinylm.py:293-295 up to one rounding order
            v[bi][1] = rg.y * inv;
            v[bi][2] = rg.z * inv;
            v[bi][3] = rg.w * inv;
          }
        } else if (!src) {
#pragma unroll
          for (int bi = 0; bi < SB; ++bi) {
            const int k = kb + bi * 4 * E_NCW * 32;
            if (k + 4 <= s_k_real) {
              const uint2 raw = __ldg(reinterpret_cast<const uint2*>(a.x_in + k));
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
              v[bi][0] = f0.x; v[bi][1] = f0.y; v[bi][2] = f1.x; v[bi][3] = f1.y;
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) v[bi][i] = (k + i < s_k_real) ? __half2float(a.x_in[k + i]) : 0.f;
            }
          }
        } else {
          // counted source: one u64 word per element; every word's contributor count is checked
          // against the source n-group's (static) contributor number, re-reading the batch until
          // all have landed.  silu(g) * u reads the two halves in turn.
          const unsigned long long* sa = s_src_acc + (long long)par * s_src_acc_len;
          // (inline rather than counted_read4: measured 6 % faster on the 7B linear stack)
          for (int which = 0; which < (s_act == 1 ? 2 : 1); ++which) {
            unsigned long long w[SB][4];
            int want[SB];
#pragma unroll
            for (int bi = 0; bi < SB; ++bi) {
              const int k = kb + bi * 4 * E_NCW * 32;
              want[bi] = k < khi ? (int)__ldg(s_src_nslots + ((s_src_col + which * s_act_off + k) >> 6)) : 0;
            }
            long long t0 = 0;
            for (;;) {
#pragma unroll
              for (int bi = 0; bi < SB; ++bi) {
                const int k = kb + bi * 4 * E_NCW * 32;
                const int n = s_src_col + which * s_act_off + k;
                if (k < khi) {
                  if (TP && s_src_sys) {  // a row-parallel output other GPUs add into
                    ld_relaxed_sys_u64x2(sa + n, w[bi][0], w[bi][1]);
                    ld_relaxed_sys_u64x2(sa + n + 2, w[bi][2], w[bi][3]);
                  } else {
                    ld_relaxed_u64x2(sa + n, w[bi][0], w[bi][1]);
                    ld_relaxed_u64x2(sa + n + 2, w[bi][2], w[bi][3]);
                  }
                } else {
                  w[bi][0] = w[bi][1] = w[bi][2] = w[bi][3] = 0ull;
                }
              }
              bool ok = true;
#pragma unroll
              for (int bi = 0; bi < SB; ++bi)
#pragma unroll
                for (int i = 0; i < 4; ++i) ok = ok && fix_count(w[bi][i]) == want[bi];
              if (ok) break;
              spin_watchdog(t0);
              if (PMPD_ENGINE_RETRY_NS) __nanosleep(PMPD_ENGINE_RETRY_NS);
            }
#pragma unroll
            for (int bi = 0; bi < SB; ++bi) {
              const int k = kb + bi * 4 * E_NCW * 32;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float x = fix_decode(w[bi][i], want[bi]) * s_in_alpha;
                const float g = which == 0 ? x : __fdividef(v[bi][i], 1.f + __expf(-v[bi][i])) * x;
                v[bi][i] = (k + i < s_k_real) ? g : 0.f;
              }
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
#ifdef PMPD_ENGINE_TRACE_WARPS
    long long fwait_all = 0;
#endif
    int ngi = 0;
    // activation scale per n-group: qs = E_QMAX * idm / mx (one reciprocal per op, none per group)
    const float qmx = mx > 0.f ? __fdividef(E_QMAX, mx) : 0.f;
    if (t < r.T1) qs = qmx * idm_pre[0];
    while (t < r.T1) {
      const int end = min(min(t + E_STILES, r.T1), t - kt + r.KT);
#ifndef PMPD_ENGINE_SKIP_MEMORY
#ifdef PMPD_ENGINE_TRACE_WARPS  // probe: full-stage wait cycles of every consumer warp
      if (a.trace) {
        const long long w0 = clock64();
        mbar_wait(&bars.full[slot], phase);
        fwait_all += clock64() - w0;
      } else
#endif
      mbar_wait(&bars.full[slot], phase);
#endif
#if PMPD_ENGINE_SLOTMAP
      // second-tile slots of a partial stage go first to the warps of schedulers 2 and 3, then
      // 1 (shared with the epilogue warp), then 0 (shared with the producer warp)
      const int ws = ((0x4B >> (2 * (warp & 3))) & 3) * (E_NCW / 4) + (warp >> 2);
      (void)rot;
#elif PMPD_ENGINE_ROTATE
      const int ws = warp >= rot ? warp - rot : warp - rot + E_NCW;  // this warp's slot
      rot += end - t;
      rot %= E_NCW;
#else
      const int ws = warp;
      (void)rot;
#endif
#ifdef PMPD_ENGINE_SKIP_COMPUTE
      if (false) {
#else
      if (ws < end - t) {
#endif
#ifndef PMPD_ENGINE_TRACE_LOOPONLY
        if (a.trace) {
          const long long c0 = clock64();
          tile_dispatch(P, smem + kSmRing + slot * stage_bytes, end - t, ws, kt + ws, lane, xs, xq, qs, dacc, bias);
          tcyc += clock64() - c0;
          ++tcalls;
        } else
#else
        if (a.trace) ++tcalls;  // probe: only the loop's total cycles and call count (no clocks per call)
#endif
        {
#if PMPD_ENGINE_PREDECODE
          if (pre) {
            tile_dispatch_pre(P, smem + kSmRing + slot * stage_bytes, end - t, ws, kt + ws, lane, xs, xq, qs, dacc, bias,
                              fa);
            pre = false;
          } else
#endif
          tile_dispatch(P, smem + kSmRing + slot * stage_bytes, end - t, ws, kt + ws, lane, xs, xq, qs, dacc, bias);
        }
#ifdef PMPD_ENGINE_DOUBLE  // timing probe only: every stage's tiles decoded twice (wrong results)
        tile_dispatch(P, smem + kSmRing + slot * stage_bytes, end - t, ws, kt + ws, lane, xs, xq, qs, dacc, bias);
#endif
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
        // (the lane sum of the bias term is left to the epilogue: one 5-step shuffle chain per
        // segment there instead of on every consumer warp's path)
        if (PMPD_ENGINE_LANEBIAS) {
          redb[(buf * E_NCW + warp) * kBiasPerWarp + lane] = bias;
        } else {
          const float bs = warp_sum(bias);
          if (lane == 0) redb[buf * E_NCW + warp] = bs;
        }
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
#if defined(PMPD_ENGINE_TRACE_WSET)
    // probe: loop-end globaltimer of consumer warps 4*WSET .. 4*WSET+3 in slots 4..7
    if (a.trace && lane == 0 && (warp >> 2) == PMPD_ENGINE_TRACE_WSET)
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 4 + (warp & 3)] = gtimer();
    if (a.trace && threadIdx.x == 0) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 2] = gtimer();
#elif defined(PMPD_ENGINE_TRACE_WARPS)
    // probe layout: [4] sum over warps of call cycles, [5] sum of full-stage wait cycles,
    // [6] latest warp's loop end, [7] earliest warp's loop end (globaltimer)
    if (a.trace && lane == 0) {
      long long* tp = a.trace + ((int64_t)c * a.n_ops + oi) * 8;
      const unsigned long long g = gtimer();
      atomicAdd(reinterpret_cast<unsigned long long*>(tp + 4), (unsigned long long)tcyc);
      atomicAdd(reinterpret_cast<unsigned long long*>(tp + 5), (unsigned long long)fwait_all);
      atomicMax(reinterpret_cast<unsigned long long*>(tp + 6), g);
      atomicMin(reinterpret_cast<unsigned long long*>(tp + 7), g);
      if (warp == 0) tp[2] = (long long)g;
    }
#else
#ifdef PMPD_ENGINE_TRACE_ATTNSTAGE
    if (a.trace && threadIdx.x == 0 && op.in_mode == E_IN_ATTN) {
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 2] = gtimer();
    } else
#endif
    if (a.trace && threadIdx.x == 0) {
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 2] = gtimer();
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 4] = tcyc;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 5] = tcalls;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 6] = clock64() - scyc0;
      a.trace[((int64_t)c * a.n_ops + oi) * 8 + 7] = (fwait << 32) | (fcyc & 0xffffffffll);
    }
#endif
  }
}

// DEC: the decoder-step op kinds (attention, RMSNorm / attention-combine inputs, residual outputs);
// the linear-stack program runs the instantiation without them (no extra registers on its path).
// TP: the tensor-parallel instantiation (pmpd_engine_run_ranks): rank groups and peer copies;
// the single-GPU linear stack runs the instantiation without them (measured 5 % slower with).
template <bool DEC, bool TP>
__global__ void __launch_bounds__(E_THREADS, 1) engine_kernel(const EngineArgs a_in) {
  extern __shared__ __align__(128) uint8_t smem[];
  Bars& bars = *reinterpret_cast<Bars*>(smem + kSmBar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Tensor-parallel emulation (n_ranks > 1, linear-stack programs): the grid is split into
  // n_ranks groups of G CTAs; group r runs rank r's op table (its shards) and writes rank r's
  // slice of y_out.  Row-parallel outputs are counted vectors shared by all ranks, their counts
  // summing every rank's contributors: the cross-rank reduction is the same counted addition as
  // the split-K one (the multi-GPU form adds into every rank's copy over NVLink).
  const int nr = TP ? a_in.n_ranks : 1;
  const int G = gridDim.x / nr, rank = blockIdx.x / G, c = blockIdx.x - rank * G;
  const bool idle = rank >= nr;  // grid remainder when n_ranks does not divide it
  EngineArgs a = a_in;
  if constexpr (TP) {
    a.ops += (idle ? 0 : rank) * a.n_ops;
    a.y_out += (idle ? 0 : rank) * (long long)a.y_stride;
  }
  int p = *a.p_dev;
  if (p < 1 || p > 4) {
    if (threadIdx.x == 0 && c == 0) atomicExch(a.status, PMPD_ERR_CONTRACT);
    p = p < 1 ? 1 : 4;
  }
  // launch epoch (counted programs): advanced by the last CTA to finish, read by all at start
  const unsigned epoch = ld_relaxed_u32(a.bar + 2);
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

  if (idle) {
    // no work: only the launch's done counter below
  } else if (warp == E_PROD || warp == E_PROD_B) {
    // ------------------------------------------------------------ producer
    // (PROD2: both producer warps walk every stage; each issues its own half, so the TMA issue
    // load is split over two schedulers)
    const int pturn = (PMPD_ENGINE_PROD2 && warp == E_PROD_B) ? 1 : 0;
    int gstage = 0;
#ifndef PMPD_ENGINE_PROD_WARPWIDE
#define PMPD_ENGINE_PROD_WARPWIDE 0
#endif
    // PROD_WARPWIDE: the whole warp runs the producer loop (its addresses stay warp-uniform, so
    // each bulk copy is one instruction instead of an elect-one loop); lane 0 issues
    const bool issuer = PMPD_ENGINE_PROD_WARPWIDE ? lane == 0 : true;
#ifdef PMPD_ENGINE_SKIP_MEMORY
    if (false) {
#else
    if (PMPD_ENGINE_PROD_WARPWIDE || lane == 0) {
#endif
#ifdef PMPD_ENGINE_EVICT_NORMAL
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
      const uint64_t pol = policy_evict_first();
#endif
      int slot = 0, used = 0;
      uint32_t phase = 0;
      for (int oi = 1; oi < PMPD_ENGINE_PF && oi < a.n_ops; ++oi) prefetch_op(a.ops[oi], c, G, p);
      int pf_op = 0, pf_t = -1, pfb_ahead = 0;
      (void)pfb_ahead;
      if (PMPD_ENGINE_PFT > 0) pf_advance(a.ops, a.n_ops, c, G, p, pf_op, pf_t, PMPD_ENGINE_PFT);
      for (int oi = 0; oi < a.n_ops; ++oi) {
        const EngineOp& op = a.ops[oi];
        if (PMPD_ENGINE_PF > 0 && oi + PMPD_ENGINE_PF < a.n_ops) prefetch_op(a.ops[oi + PMPD_ENGINE_PF], c, G, p);
        if (DEC && op.kind == E_ATTN) continue;  // no weights
#ifdef PMPD_ENGINE_KV_PREFETCH  // measured slower: it delays the q|k|v weight loads
        if (DEC && oi + 1 < a.n_ops && a.ops[oi + 1].kind == E_ATTN) {
          // L2 prefetch of this CTA's attention K/V rows one op ahead: the rows do not depend on
          // this token, and loaded only when the attention op runs they queue behind the weight
          // stream (measured: the unit's row loop was 3.3 us of latency at 7B)
          const EngineOp& at = a.ops[oi + 1];
          const int L = min(*at.T_dev + 1, at.max_ctx), dh = at.d_head, d = at.n_heads * dh;
          const int chunk = (L + E_ASPLIT - 1) / E_ASPLIT;
          for (int u = c; u < at.n_heads * E_ASPLIT; u += G) {
            const int h = u / E_ASPLIT, s = u - h * E_ASPLIT;
            const int t0 = s * chunk, t1 = min(L - 1, t0 + chunk);  // row L-1 is written this step
            for (int t = t0; t < t1; ++t) {
              bulk_prefetch_l2(at.kc + (int64_t)t * d + h * dh, (uint32_t)dh * 2);
              bulk_prefetch_l2(at.vc + (int64_t)t * d + h * dh, (uint32_t)dh * 2);
            }
          }
        }
#endif
        const Range r = range_of(op, c, G);
        int t = r.T0, kt = r.T0 % r.KT;
        // the op's fields in registers (the copies below clobber memory, so reading op.* in the
        // loop would reload them every stage), the tile's index in the tensor tracked incrementally
        const uint8_t* const planes = op.planes;
        const uint8_t* const scales = op.scales;
        const long long plane_bytes = op.plane_bytes;
        const int kt_skip = op.kt_mem - r.KT;  // tensor k-tiles outside the slice, per n-group
        int64_t mt = (int64_t)(r.T0 / r.KT) * op.kt_mem + op.k_off + kt;
        while (t < r.T1) {
          const int end = min(min(t + E_STILES, r.T1), t - kt + r.KT);
          const int cnt = end - t;
#if PMPD_ENGINE_PFB > 0
          // prefetch-when-blocked: the ring is full (this SM's stream would stall), so pull the
          // tiles just beyond the ring into L2 while the consumers catch up (typically at an op
          // boundary, when HBM is otherwise idle); at most PMPD_ENGINE_PFB tiles ahead
          if (used && !mbar_try_wait(&bars.empty[slot], phase ^ 1u) && pfb_ahead < PMPD_ENGINE_PFB) {
            const int n = min(E_STILES, PMPD_ENGINE_PFB - pfb_ahead);
            pf_advance(a.ops, a.n_ops, c, G, p, pf_op, pf_t, n);
            pfb_ahead += n;
          }
#endif
          const bool mine = !PMPD_ENGINE_PROD2 || ((gstage++ & 1) == pturn);
#ifdef PMPD_ENGINE_PROD_SPIN
          if (used && mine) mbar_wait(&bars.empty[slot], phase ^ 1u);
#else
          if (used && mine) mbar_wait_backoff(&bars.empty[slot], phase ^ 1u);
#endif
          uint8_t* st = smem + kSmRing + slot * stage_bytes;
          // (a stage never crosses an n-group, so its tiles are contiguous in the tensor)
          if (issuer && mine) {
            mbar_arrive_expect_tx(&bars.full[slot], (uint32_t)(cnt * kTilePlaneBytes * (p + 1)));
            for (int j = 0; j < p; ++j)
              bulk_g2s_stream(st + j * E_STILES * kTilePlaneBytes, planes + j * plane_bytes + mt * kTilePlaneBytes,
                              cnt * kTilePlaneBytes, &bars.full[slot], pol);
            bulk_g2s_stream(st + p * E_STILES * kTilePlaneBytes, scales + mt * kTileScaleBytes, cnt * kTileScaleBytes,
                            &bars.full[slot], pol);
          }
          mt += cnt;
          if (PMPD_ENGINE_PFT > 0) pf_advance(a.ops, a.n_ops, c, G, p, pf_op, pf_t, cnt);
#if PMPD_ENGINE_PFB > 0
          // the load cursor passed cnt tiles: consume the prefetched lead, or move the prefetch
          // cursor along with the loads when there is none
          if (pfb_ahead >= cnt) {
            pfb_ahead -= cnt;
          } else {
            pf_advance(a.ops, a.n_ops, c, G, p, pf_op, pf_t, cnt - pfb_ahead, false);
            pfb_ahead = 0;
          }
#endif
          kt += cnt;
          if (kt == r.KT) {
            kt = 0;
            mt += kt_skip;
          }
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
    const int par = (int)(epoch % kSets);
    const int zset = (int)((epoch + kSets - 1) % kSets);  // the set the previous launch used
    if (DEC) {
      // residual stream: zero this CTA's slice of the idle parity set, then add x0 (the
      // embedding row, written before the launch) into slice c of this launch's set: one
      // contribution per word
      unsigned long long* Rc = a.R + (long long)par * a.R_len;
      unsigned long long* Ro = a.R + (long long)zset * a.R_len;
      for (long long i = a.R_len * c / G + lane, e = a.R_len * (c + 1) / G; i < e; i += 32) Ro[i] = 0ull;
      for (int i = (int)((long long)a.d_real * c / G) + lane, e = (int)((long long)a.d_real * (c + 1) / G); i < e;
           i += 32)
        red_relaxed_u64(Rc + i, fix_encode(__ldg(a.x0 + i), a.status));
    }
    int seg = 0;
    for (int oi = 0; oi < a.n_ops; ++oi) {
      const EngineOp& op = a.ops[oi];
      if (op.kind == E_LINEAR && op.keep_out && op.rwait >= 0 && lane == 0) {
        // residual op: its additions must not reach R before every reader of the previous
        // residual version has read it (always long since true: this op's inputs depend on
        // those readers' outputs; the wait makes it a guarantee)
        wait_hint(a.bar + 3 + a.n_ops + op.rwait, (epoch + 1u) * (unsigned)a.ops[op.rwait].n_contrib);
      }
      __syncwarp();
      if (op.kind == E_LINEAR) {
        const Range r = range_of(op, c, G);
        int t = r.T0, ng = r.T0 / r.KT, kt = r.T0 % r.KT;
        // (op fields in registers: the additions below clobber memory, op.* would be re-read per segment)
        const int e_ng_off = op.ng_off, e_n_peers = TP ? op.n_peers : 0, e_sys = TP ? op.sys : 0;
        const float e_out_alpha = op.out_alpha;
        const long long e_acc_len = op.acc_len;
        unsigned long long* acc = op.acc + (long long)par * e_acc_len;
        while (t < r.T1) {
          const int seg_end = min(r.T1, t - kt + r.KT);
          const int buf = seg & 1;
#ifdef PMPD_ENGINE_EPI_SPIN
          mbar_wait(&bars.red_full[buf], (seg >> 1) & 1);
#else
          mbar_wait_backoff(&bars.red_full[buf], (seg >> 1) & 1);
#endif
          float bsum = 0.f;
          if (PMPD_ENGINE_LANEBIAS) {
#pragma unroll
            for (int w = 0; w < E_NCW; ++w) bsum += redb[(buf * E_NCW + w) * kBiasPerWarp + lane];
            bsum = warp_sum(bsum);
          } else {
#pragma unroll
            for (int w = 0; w < E_NCW; ++w) bsum += redb[buf * E_NCW + w];
          }
          // split-K: every CTA holding tiles of n-group ng adds its partial at L2 as a counted
          // fixed-point contribution (residual ops add into the residual stream)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int nl = lane + 32 * h;
            float v = bsum;
#pragma unroll
            for (int w = 0; w < E_NCW; ++w) v += red[(buf * E_NCW + w) * 64 + nl];
            const unsigned long long w = fix_encode(DEC ? v * e_out_alpha : v, a.status);
            if (!TP || e_n_peers == 0) {
              red_relaxed_u64(acc + (int64_t)(e_ng_off + ng) * 64 + nl, w);
            } else {
              const long long off = (long long)par * e_acc_len + (int64_t)(e_ng_off + ng) * 64 + nl;
              for (int j = 0; j < e_n_peers; ++j) {
                if (e_sys)
                  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(op.peer[j] + off), "l"(w) : "memory");
                else
                  red_relaxed_u64(op.peer[j] + off, w);
              }
            }
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
        __syncwarp();
        if (lane == 0 && r.T1 > r.T0) {
          if (!PMPD_ENGINE_NOHINT) {
            if (PMPD_ENGINE_HINT_RELEASE)
              asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + 3 + oi) : "memory");
            else
              asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar + 3 + oi) : "memory");
          }
          if (a.trace) a.trace[((int64_t)c * a.n_ops + oi) * 8 + 3] = gtimer();
        }
      }
      if (!(op.kind == E_LINEAR && op.keep_out)) {
        // zero this CTA's slice of the op's idle parity set (outputs / attention records) for the
        // next launch (the residual stream's was zeroed at the start)
        unsigned long long* other = op.acc + (long long)zset * op.acc_len;
        const long long zl = op.zero_len >= 0 ? op.zero_len : op.acc_len;
        for (long long i = zl * c / G + lane, e = zl * (c + 1) / G; i < e; i += 32) other[i] = 0ull;
      }
    }
  } else if (warp < E_NCW) {
    // ------------------------------------------------------------ consumers
    consumer_loop<DEC, TP>(p, a, smem, bars, G, c, stage_bytes, nstage, epoch);
  }
  // ---------------------------------------------------------------- final output
  // CTA c finalizes n-groups c, c + G, ... of the last op from their complete counted words
  __syncthreads();
  const EngineOp& last = a.ops[a.n_ops - 1];
  {
    const int par = (int)(epoch % kSets);
    if (!PMPD_ENGINE_NOHINT && threadIdx.x == 0)
      wait_hint(a.bar + 3 + a.n_ops - 1, (epoch + 1u) * (unsigned)last.n_contrib);
    __syncthreads();
    const unsigned long long* la = last.acc + (long long)par * last.acc_len;
    for (int ng = c; !idle && ng < last.n_tiles; ng += G) {
      const int want = __ldg(last.nslots + ng);
      for (int nl = threadIdx.x; nl < 64; nl += blockDim.x) {
        const int n = ng * 64 + nl;
        unsigned long long w = ld_relaxed_u64(la + n);
        long long t0 = 0;
        while (fix_count(w) != want) {
          spin_watchdog(t0);
          __nanosleep(64);
          w = ld_relaxed_u64(la + n);
        }
        if (n < last.n_real) a.y_out[n] = a.y_alpha * fix_decode(w, want);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(a.bar + 1, 1u) == gridDim.x - 1) {
      a.bar[1] = 0;
      a.bar[2] = epoch + 1u;  // read by the next launch (kernel boundary orders it)
    }
  }
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

namespace {
// Cost-balanced tile partition (the stage geometry of this translation unit's kernel)
int partition_impl(const pmpd_qtensor* t, int32_t G, const int32_t* delta_host, int32_t* bounds_host) {
  if (!t || !bounds_host) return fail(PMPD_ERR_CONFIG, "null argument");
  if (G < 1) return fail(PMPD_ERR_CONFIG, "partition over %d CTAs", G);
  const int KT = t->k_tiles, NT = t->n_tiles * t->k_tiles;
  if (NT < 1) return fail(PMPD_ERR_CONFIG, "empty tensor");
  // cost in half tile-times
  static const int flush_cost = [] {  // half tile-times per n-group segment (PMPD_ENGINE_PART_FLUSH)
    const char* e = getenv("PMPD_ENGINE_PART_FLUSH");
    return e ? atoi(e) : 1;
  }();
  auto seg_cost = [&](int n) {  // n tiles of one n-group segment
    int cst = flush_cost;
    for (int s0 = 0; s0 < n; s0 += E_STILES) cst += 2 * ((std::min(n - s0, E_STILES) + E_NCW - 1) / E_NCW);
    return cst;
  };
  // greedy: from tile t, the largest end with cost <= budget
  auto cover = [&](int budget, int32_t* out) {
    int t0 = 0, c = 0;
    if (out) out[0] = 0;
    while (t0 < NT) {
      if (c == G) return G + 1;
      // a CTA measured slower than the rest (pmpd_engine_partition_w) gets a smaller budget
      int t1 = t0, cost = delta_host ? std::max(0, delta_host[c]) : 0;
      while (t1 < NT) {
        const int kt = t1 % KT, seg_end = std::min(NT, t1 - kt + KT);
        // largest prefix of this segment that still fits
        int lo = 0, hi = seg_end - t1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) / 2;
          if (cost + seg_cost(mid) <= budget) lo = mid; else hi = mid - 1;
        }
        if (lo == 0) break;
        cost += seg_cost(lo);
        t1 += lo;
        if (lo < seg_end - (t1 - lo)) break;  // segment not finished: the budget is spent
      }
      if (t1 == t0) return G + 1;  // budget below one tile
      ++c;
      if (out) out[c] = t1;
      t0 = t1;
    }
    if (out) for (int k = c + 1; k <= G; ++k) out[k] = NT;  // idle CTAs
    return c;
  };
  int lo = 1, hi = 1 << 30;
  {  // upper bound: the even split's cost
    int mx = 0;
    for (int c = 0; c < G; ++c) {
      const int a = (int)((int64_t)c * NT / G), b = (int)((int64_t)(c + 1) * NT / G);
      int cst = 0;
      for (int t1 = a; t1 < b;) {
        const int e = std::min(b, t1 - t1 % KT + KT);
        cst += seg_cost(e - t1);
        t1 = e;
      }
      mx = std::max(mx, cst + (delta_host ? std::max(0, delta_host[c]) : 0));
    }
    hi = mx;
  }
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (cover(mid, nullptr) <= G) hi = mid; else lo = mid + 1;
  }
  cover(lo, bounds_host);
  return PMPD_OK;
}
}  // namespace

#ifndef PMPD_ENGINE_DEC_TU
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
  op.kind = E_LINEAR;
  op.in_mode = E_IN_SRC;
  op.out_alpha = 1.f;
  op.rwait = -1;
  op.kt_mem = t->k_tiles;
  op.n_tiles_full = t->n_tiles;
  op.zero_len = -1;
  if ((src_col & 3) || (act_off & 3)) return fail(PMPD_ERR_CONFIG, "engine input offsets must be multiples of 4");
  *static_cast<EngineOp*>(op_host) = op;
  return PMPD_OK;
}

int pmpd_engine_run_traced(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                           float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream);

int pmpd_engine_op_set_io(void* op_host, int32_t in_mode, const float* resid_dev, const float* gain_dev, float eps,
                          int32_t keep_out, float out_alpha) {
  if (!op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "set_io applies to linear ops");
  if (in_mode != E_IN_SRC && in_mode != E_IN_RMSNORM && in_mode != E_IN_ATTN)
    return fail(PMPD_ERR_CONFIG, "unknown engine input mode %d", in_mode);
  if (in_mode == E_IN_RMSNORM && (!gain_dev || (op.k_real & 3) || (reinterpret_cast<uintptr_t>(gain_dev) & 15)))
    return fail(PMPD_ERR_CONFIG, "RMSNorm input needs a 16-byte aligned gain and K % 4 == 0");
  op.in_mode = in_mode;
  op.resid = resid_dev;
  op.gain = gain_dev;
  op.eps = eps;
  op.eps_inv_k = 1.f / (float)op.k_real;
  if (in_mode != E_IN_SRC && (op.k_off || op.k_tiles != op.kt_mem))
    return fail(PMPD_ERR_CONFIG, "RMSNorm / attention inputs need the op's whole k range (no k-slice)");
  if (in_mode == E_IN_ATTN && op.k_tiles * kTile > 3 * 4 * E_NCW * 32)
    return fail(PMPD_ERR_CONFIG, "attention-combine input wider than %d", 3 * 4 * E_NCW * 32);
  if (in_mode == E_IN_RMSNORM && 2 * op.k_tiles * kTile + 4 * op.k_real > 2 * E_XMAX)
    return fail(PMPD_ERR_CONFIG, "RMSNorm input row too wide for the staging area");
  op.keep_out = keep_out ? 1 : 0;
  op.out_alpha = out_alpha;
  return PMPD_OK;
}

int pmpd_engine_make_attn_op(int32_t src, int32_t n_heads, int32_t d_head, void* k_cache, void* v_cache,
                             const float* cos_dev, const float* sin_dev, const int32_t* T_dev, int32_t max_ctx,
                             float scale, void* records_dev, void* op_host) {
  if (!op_host || !k_cache || !v_cache || !cos_dev || !sin_dev || !T_dev || !records_dev)
    return fail(PMPD_ERR_CONFIG, "null argument");
  if (d_head != 32 && d_head != 64 && d_head != 128 && d_head != 256)
    return fail(PMPD_ERR_CONFIG, "engine attention needs d_head in {32, 64, 128, 256}");
  if ((int64_t)n_heads * E_ASPLIT * 4 > 3 * 1024) return fail(PMPD_ERR_CONFIG, "too many heads for the engine");
  if (src < 0) return fail(PMPD_ERR_CONFIG, "attention op needs a q|k|v source op");
  EngineOp op{};
  op.kind = E_ATTN;
  op.src = src;
  op.n_heads = n_heads;
  op.d_head = d_head;
  op.kc = static_cast<__half*>(k_cache);
  op.vc = static_cast<__half*>(v_cache);
  op.cos_t = cos_dev;
  op.sin_t = sin_dev;
  op.T_dev = T_dev;
  op.max_ctx = max_ctx;
  op.scale = scale;
  op.acc = static_cast<unsigned long long*>(records_dev);  // [2][pmpd_engine_attn_records()] words
  op.acc_len = (long long)n_heads * E_ASPLIT * (4 + d_head);
  op.rwait = -1;
  op.out_alpha = 1.f;
  op.zero_len = -1;
  *static_cast<EngineOp*>(op_host) = op;
  return PMPD_OK;
}

int pmpd_engine_attn_records(int32_t n_heads, int32_t d_head) { return n_heads * E_ASPLIT * (4 + d_head); }

// Cost-balanced tile partition for one op: the CTA tile ranges minimise the largest per-CTA cost,
// where a CTA's tiles run as stages of E_STILES cut at n-group boundaries, a stage of <= E_NCW tiles
// costs one tile-time (one tile per warp) and a fuller one two, and each n-group segment adds a
// flush (~0.5 tile-time).  An even split of the tiles gives some CTAs an extra stage or segment
// (e.g. 3 stage calls instead of 2 for o on 148 SMs).  Binary search on the budget, greedy cover.
int pmpd_engine_partition(const pmpd_qtensor* t, int32_t* bounds_host) {
  return pmpd_engine_partition_g(t, num_sms(), bounds_host);
}

int pmpd_engine_partition_g(const pmpd_qtensor* t, int32_t G, int32_t* bounds_host) {
  return pmpd_engine_partition_w(t, G, nullptr, bounds_host);
}

int pmpd_engine_partition_w(const pmpd_qtensor* t, int32_t G, const int32_t* delta_host, int32_t* bounds_host) {
  return partition_impl(t, G, delta_host, bounds_host);
}

int pmpd_engine_op_set_counted(void* op_host, void* acc_dev, const uint8_t* nslots_dev, int32_t n_contrib) {
  if (!op_host || !acc_dev || !nslots_dev) return fail(PMPD_ERR_CONFIG, "null argument");
  if (reinterpret_cast<uintptr_t>(acc_dev) & 15) return fail(PMPD_ERR_CONFIG, "counted accumulators must be 16-byte aligned");
  if (n_contrib < 1 || n_contrib > num_sms()) return fail(PMPD_ERR_CONFIG, "bad contributor count %d", n_contrib);
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "counted accumulation applies to linear ops");
  op.acc = static_cast<unsigned long long*>(acc_dev);
  op.acc_len = (long long)op.n_tiles_full * 64;  // sub-ops of one tensor share its whole output
  op.nslots = nslots_dev;
  op.n_contrib = n_contrib;
  return PMPD_OK;
}

int pmpd_engine_op_set_slice(void* op_host, int32_t ng0, int32_t ng1, int32_t kt0, int32_t kt1) {
  if (!op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "slices apply to linear ops");
  if (op.ng_off || op.k_off || op.n_tiles != op.n_tiles_full || op.k_tiles != op.kt_mem)
    return fail(PMPD_ERR_CONFIG, "op is already a slice");
  if (op.in_mode != E_IN_SRC || op.acc) return fail(PMPD_ERR_CONFIG, "slice an op before set_io / set_counted");
  if (ng0 < 0 || ng1 <= ng0 || ng1 > op.n_tiles || kt0 < 0 || kt1 <= kt0 || kt1 > op.k_tiles)
    return fail(PMPD_ERR_CONFIG, "slice [%d,%d) x [%d,%d) outside %d x %d tiles", ng0, ng1, kt0, kt1, op.n_tiles,
                op.k_tiles);
  const int64_t tiles_before = (int64_t)ng0 * op.k_tiles;
  op.planes += tiles_before * kTilePlaneBytes;  // plane j stays at planes + j * plane_bytes
  op.scales += tiles_before * kTileScaleBytes;
  op.aux += ng0;
  op.ng_off = ng0;
  op.n_real = std::min(op.n_real - ng0 * kTile, (ng1 - ng0) * kTile);
  op.n_tiles = ng1 - ng0;
  op.k_off = kt0;
  op.k_real = std::min(op.k_real - kt0 * kTile, (kt1 - kt0) * kTile);
  op.k_tiles = kt1 - kt0;
  op.src_col += kt0 * kTile;  // local input element 0 is tensor input element kt0 * 64
  return PMPD_OK;
}

int pmpd_engine_op_set_share(void* op_host, int32_t zero_output) {
  if (!op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "set_share applies to linear ops");
  op.zero_len = zero_output ? -1 : 0;
  return PMPD_OK;
}

int pmpd_engine_link(void* ops_host, int32_t n_ops) {
  if (!ops_host || n_ops < 1) return fail(PMPD_ERR_CONFIG, "null argument");
  EngineOp* ops = static_cast<EngineOp*>(ops_host);
  for (int i = 0; i < n_ops; ++i) {
    EngineOp& op = ops[i];
    if (op.kind != E_LINEAR || op.src < 0) continue;
    if (op.src >= i) return fail(PMPD_ERR_CONFIG, "op %d reads op %d, which does not precede it", i, op.src);
    const EngineOp& src = ops[op.src];
    op.src_acc = src.acc;
    op.src_acc_len = src.acc_len;
    op.src_nslots = src.nslots;
    op.src_sys = src.sys;
  }
  return PMPD_OK;
}

int pmpd_engine_op_set_peers(void* op_host, const void* const* peers_host, int32_t n_peers, int32_t sys_scope) {
  if (!op_host || (n_peers > 0 && !peers_host)) return fail(PMPD_ERR_CONFIG, "null argument");
  if (n_peers < 0 || n_peers > 8) return fail(PMPD_ERR_CONFIG, "1..8 peer copies, got %d", n_peers);
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "peer copies apply to linear ops");
  for (int j = 0; j < n_peers; ++j) {
    if (!peers_host[j] || (reinterpret_cast<uintptr_t>(peers_host[j]) & 15))
      return fail(PMPD_ERR_CONFIG, "peer copy %d must be a 16-byte aligned device pointer", j);
    op.peer[j] = static_cast<unsigned long long*>(const_cast<void*>(peers_host[j]));
  }
  op.n_peers = n_peers;
  op.sys = sys_scope ? 1 : 0;
  return PMPD_OK;
}

int pmpd_engine_op_set_residual(void* op_host, const uint16_t* cum_dev, int32_t rwait) {
  if (!op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  EngineOp& op = *static_cast<EngineOp*>(op_host);
  if (op.kind != E_LINEAR) return fail(PMPD_ERR_CONFIG, "residual wiring applies to linear ops");
  if (op.in_mode == E_IN_RMSNORM && !cum_dev) return fail(PMPD_ERR_CONFIG, "RMSNorm op needs its residual counts");
  op.cum = cum_dev;
  op.rwait = rwait;
  return PMPD_OK;
}

int pmpd_engine_op_set_bounds(void* op_host, const int32_t* bounds_dev) {
  if (!op_host) return fail(PMPD_ERR_CONFIG, "null argument");
  static_cast<EngineOp*>(op_host)->bounds = bounds_dev;
  return PMPD_OK;
}

int pmpd_engine_run(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                    float y_alpha, uint32_t* bar_dev, int32_t* status_dev, void* stream) {
  return pmpd_engine_run_traced(ops_dev, n_ops, p_dev, x_in, y_out, y_alpha, bar_dev, status_dev, nullptr, stream);
}

}  // extern "C"
#endif  // !PMPD_ENGINE_DEC_TU

namespace {
int engine_launch(bool dec, const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                  float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream,
                  void* R = nullptr, long long R_len = 0, int d_real = 0, int n_ranks = 1, int y_stride = 0,
                  bool tp = false) {
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
  a.R = static_cast<unsigned long long*>(R);
  a.R_len = R_len;
  a.x0 = dec ? static_cast<const float*>(x_in) : nullptr;
  a.d_real = d_real;
  a.n_ranks = n_ranks;
  a.y_stride = y_stride;
  if (dec && (!R || !x_in || R_len < d_real || (R_len & 63))) return fail(PMPD_ERR_CONFIG, "decoder residual stream");
  if (n_ranks < 1 || n_ranks > 8 || (n_ranks > 1 && (dec || trace_dev)))
    return fail(PMPD_ERR_CONFIG, "rank emulation: 1..8 ranks, linear-stack programs, no trace");
  static int smem = 0;
  if (smem == 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    smem = optin;
    if (const char* e = getenv("PMPD_ENGINE_SMEM")) smem = atoi(e) < optin ? atoi(e) : optin;
#ifdef PMPD_ENGINE_DEC_TU
    cudaFuncSetAttribute(engine_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
#else
    cudaFuncSetAttribute(engine_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(engine_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
#endif
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
#ifdef PMPD_ENGINE_DEC_TU
  (void)tp;
  const cudaError_t e = dec ? cudaLaunchKernelEx(&cfg, engine_kernel<true, false>, a) : cudaErrorInvalidValue;
#else
  const cudaError_t e = dec ? cudaErrorInvalidValue
                        : n_ranks > 1 || tp ? cudaLaunchKernelEx(&cfg, engine_kernel<false, true>, a)
                                            : cudaLaunchKernelEx(&cfg, engine_kernel<false, false>, a);
#endif
  if (e != cudaSuccess) return fail(PMPD_ERR_CUDA, "engine launch: %s", cudaGetErrorString(e));
  return PMPD_OK;
}
}  // namespace

extern "C" {

#ifdef PMPD_ENGINE_DEC_TU
// The decoder-step engine is compiled in its own translation unit (engine_dec.cu) with fewer
// consumer warps (PMPD_ENGINE_NCW 10, 3 tiles per warp per stage): at 384 threads the kernel gets
// 166 registers and no spills (at 448 threads it is capped at 128 and spilled 96 bytes; measured
// 15 % faster on the 1.4B decoder).  The linear-stack and tensor-parallel kernels keep 12 warps.
int pmpd_engine_run_decoder_tu(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const float* x0_dev,
                               void* resid_dev, int64_t resid_len, int32_t d_real, float* y_out, float y_alpha,
                               uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream) {
  return engine_launch(true, ops_dev, n_ops, p_dev, x0_dev, y_out, y_alpha, bar_dev, status_dev, trace_dev, stream,
                       resid_dev, resid_len, d_real);
}
#else
int pmpd_engine_run_decoder_tu(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const float* x0_dev,
                               void* resid_dev, int64_t resid_len, int32_t d_real, float* y_out, float y_alpha,
                               uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream);

int pmpd_engine_run_traced(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const void* x_in, float* y_out,
                           float y_alpha, uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream) {
  return engine_launch(false, ops_dev, n_ops, p_dev, x_in, y_out, y_alpha, bar_dev, status_dev, trace_dev, stream);
}

int pmpd_engine_run_ranks(const void* ops_dev, int32_t n_ops, int32_t n_ranks, const int32_t* p_dev, const void* x_in,
                          float* y_out, int32_t y_stride, float y_alpha, uint32_t* bar_dev, int32_t* status_dev,
                          void* stream) {
  return engine_launch(false, ops_dev, n_ops, p_dev, x_in, y_out, y_alpha, bar_dev, status_dev, nullptr, stream,
                       nullptr, 0, 0, n_ranks, y_stride, true);
}

int pmpd_engine_run_decoder(const void* ops_dev, int32_t n_ops, const int32_t* p_dev, const float* x0_dev,
                            void* resid_dev, int64_t resid_len, int32_t d_real, float* y_out, float y_alpha,
                            uint32_t* bar_dev, int32_t* status_dev, int64_t* trace_dev, void* stream) {
  return pmpd_engine_run_decoder_tu(ops_dev, n_ops, p_dev, x0_dev, resid_dev, resid_len, d_real, y_out, y_alpha,
                                    bar_dev, status_dev, trace_dev, stream);
}
#endif  // PMPD_ENGINE_DEC_TU

}  // extern "C"
