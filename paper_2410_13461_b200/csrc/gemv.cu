// Decode GEMV on the nested bit-plane format, batch 1..8, sm_100a.
//
// Replaces `h @ model.weights(name, p)` at the linear call sites of the
// reference decode loop (pkg/src/pmpd/tinylm.py:201-231 + 341-368) for the
// tiled layouts (PMPD_LAYOUT_KN: groups along N, every tinylm matrix;
// PMPD_LAYOUT_NK: groups along K, BASELINE config 1).
//
// Structure (one CTA per SM, stream-K over 64x64 tiles):
//   * warp NCW (producer): one elected lane streams the CTA's contiguous tile
//     range through a ring of shared-memory stages with 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx).  Only planes 0..p-1 are read;
//     p comes from device memory (the precision hook), so a precision switch is
//     a change of how many planes are fetched, never a weight reload.
//   * warps 0..NCW-1 (consumers): per tile, merge the p plane words into
//     nibble words, turn nibbles into fp16 A fragments with one LOP3 per half2
//     (exponent "magic" OR), and run mma.sync m16n8k16 swap-AB (A = weights
//     16 rows x 16 k, B = activations 16 k x 8 batch) with fp32 accumulation.
//   * KN: the per-(k, n-group) step is folded into B (B~ = x * step, fp16),
//     the group minimum enters as sum_k x*min (fp32), and the fp16 exponent
//     offsets are removed with a ones-MMA of B~.  NK: per-tile fp32 epilogue
//     acc += step * (D - off*Sx) + min * Sx.
//   * programmatic dependent launch: weights are prefetched before
//     griddepcontrol.wait; activations are read only after it.
//   * cross-CTA reduction of split n-groups through a workspace; the last CTA
//     (atomic ticket) sums the partials in CTA order -> deterministic.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "decode_core.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

#ifndef PMPD_GEMV_NCW
#define PMPD_GEMV_NCW 8
#endif
#ifndef PMPD_GEMV_NSTAGE
#define PMPD_GEMV_NSTAGE 4
#endif
constexpr int NCW = PMPD_GEMV_NCW;      // consumer warps
constexpr int NTHREADS = (NCW + 1) * 32;  // + producer warp
constexpr int NSTAGE = PMPD_GEMV_NSTAGE;  // smem ring depth
#ifndef PMPD_GEMV_TPW
#define PMPD_GEMV_TPW 2
#endif
constexpr int TPW = PMPD_GEMV_TPW;       // tiles per consumer warp per stage (ILP)
constexpr int STILES = NCW * TPW;        // tiles per stage
constexpr int MAXM = 8;
// Workspace: a FIXED-size counter region (so GEMVs of different widths sharing one
// workspace never see another shape's partials where they expect zeroed counters),
// one status word, then the split-K partials.
constexpr int kWsCounters = 16384;
constexpr int64_t kWsHead = (int64_t)kWsCounters * 4 + 256;
#ifndef PMPD_GEMV_ONEPASS
#define PMPD_GEMV_ONEPASS 1  // activations of every row staged / max-reduced in one pass (0: row by row)
#endif
constexpr int kXsMaxK = 12288;          // activations staged in smem when K <= this (batch 1)
constexpr int kXsMulti = 32768;         // batch 2..8: staged when m * K_pad <= this (64 KB)
constexpr int kXsBig = 49152;           // ... or <= this with a 2-stage ring (96 KB)
#ifndef PMPD_GEMV_XS2
#define PMPD_GEMV_XS2 1
#endif

struct GemvArgs {
  const uint8_t* planes;
  const uint8_t* scales;
  int64_t plane_bytes;
  int n_tiles, k_tiles, n_real, k_real, p_max;
  const int32_t* p_dev;
  const __half* x;
  int ldx, m;
  void* y;
  int y_dtype, ldy;
  float alpha;
  int accumulate;
  const float* aux;  // KN: per n-tile 1 / max(step)
  int* counters;   // [n_tiles]
  int* status;     // [1]
  float* partial;  // [n_tiles][max_slots][64][m]
  int max_slots;
  // fused input (staged-activation path only): 0 = x as given (f16); 1 = RMSNorm of the f32 row
  // xf (tinylm.py:293-295, gain, eps); 2 = silu(xf[k]) * xf[k + u_off] (tinylm.py:298,362-364)
  int in_mode;
  const float* xf;
  int ldxf;
  const float* gain;
  float eps;
  int u_off;
};

struct Smem {  // fits in the first 128 bytes of dynamic shared memory
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  int flag;
};

// ---------------------------------------------------------------- smem plan
// [Smem | ring: NSTAGE x (PMAX planes + scales) x STILES tiles | xs: staged
//  activations (XS) | xq: per-warp int8 activation fragments (KN) |
//  red/redb: cross-warp sums | qsc: per-n-group activation scales (KN)]
template <int PMAX, int MB, int XS>
struct Plan {
  static constexpr int kStage = STILES * (PMAX + 1) * kTilePlaneBytes;
  static constexpr int kRing = 128;
  // batch 2..8 with staged activations trades one ring stage for the 64 KB of x (XS = 1), or two
  // for 96 KB (XS = 2: e.g. 8 rows of K = 5632, 4 rows of K = 11008)
  // XS = 3: as 2, but only the CTA's own k-tiles are staged (a circular k range, see xmap)
  static constexpr int kNst = (MB > 1 && XS) ? (XS >= 2 ? 2 : 3) : NSTAGE;
  static constexpr int kXs = kRing + kNst * kStage;
  static constexpr int kXsBytes = XS ? (MB == 1 ? kXsMaxK * 2 : (XS >= 2 ? kXsBig : kXsMulti) * 2) : 0;
  static constexpr int kXq = kXs + kXsBytes;
  static constexpr int kXqRows = MB;
  static constexpr int kXqWarp = TPW * kXqRows * 2 * 64;  // lo + hi bytes per row and tile
  static constexpr int kRed = kXq + NCW * kXqWarp;
  static constexpr int kRedb = kRed + NCW * 64 * MB * 4;
  static constexpr int kMx = kRedb + NCW * MB * 4;  // per-row max |x| (KN)
  static constexpr int kBytes = kMx + MAXM * 4 + 32 * 4;
};

// 8 activations x[0..8) with x[i] = 0 for i >= n (the row's ragged end or an unaligned row),
// kept out of line so that the staging loop's many load sites stay small
__device__ __noinline__ uint4 load_x8_tail(const __half* src, int n) {
  __half tmp[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) tmp[i] = i < n ? src[i] : __float2half(0.f);
  return *reinterpret_cast<const uint4*>(tmp);
}

// Tile iteration without integer division: stages never straddle an n-group.
struct TileCursor {
  int t, ng, kt;
  PMPD_DEV int stage_end(int T1, int KT) const { return min(min(t + STILES, T1), t - kt + KT); }
};

// packed f32x2 arithmetic (sm_100 FMUL2 / FFMA2: each lane an IEEE mul.rn / fma.rn)
PMPD_DEV float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
PMPD_DEV float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// ---------------------------------------------------------------- consumer
// State of one consumer warp; run() is instantiated per (layout, p_max, p) so
// that the whole tile loop is specialised for the active precision.
template <int LAYOUT, int PMAX, int MB, int XS>
struct Consumer {
  using PL = Plan<PMAX, MB, XS>;
  static constexpr bool KN = LAYOUT == PMPD_LAYOUT_KN;
  const GemvArgs& a;
  Smem& sm;
  uint8_t* smem;
  const __half* xs;  // staged activations [MB][xld] (XS) or global x
  int xld;           // leading dimension of xs
  uint8_t* xq;       // KN: this warp's int8 activation fragments [rows][lo 64 | hi 64]
  float* red;
  float* redb;
  const float* mx;   // KN: per-row max |x| (smem)
  int warp, lane, gq, tig, T0, T1, KT, NT, G, c, M;
  // NK: f32 accumulators of the current n-group; KN: int32 hi/lo digit accumulators
  float acc[4][4];
  int dhi[4][4], dlo[4][4];
  float bias[MB];  // KN: this lane's part of sum_k x*min
  float qs[MB];    // KN: activation quantisation scale 32767 / (max|x_b| * max step_g)
  float ql[2];     // KN: qs of this lane's flush rows b = 2*tig + {0,1} (keeps qs[] in registers)
  // KN at batch 5..8: f16 HMMA (mma.sync m16n8k16, the batch rows are the 8 B columns).  The
  // decoded u8 bucket bytes become f16 SUBNORMALS (byte * 2^-24, exact: high byte zero) with one
  // PRMT per pair, and B = x * step * s (s a per-row power of two) is built in registers per tile
  // with no shared-memory round trip; f32 accumulation across the n-group's tiles.  The int8 path
  // re-quantised x * step per tile and row (~80 instructions per tile and row pair) and needed a
  // second IMMA per fragment at batch 8: batch 8 cost 2.8-4x batch 1.  (Batch 2..4 keep the
  // balanced-digit IMMA: one IMMA per fragment there, measured faster than this path.)
  static constexpr bool KH = KN && MB == MAXM;
  float2 hbias2; // KH: this lane's part of sum_k x[gq][k] * min (row gq), two partial sums
  const __half* xrow;  // KH, staged x: this lane's row gq
  float hs;      // KH: B scale of row gq (power of two: max |x * step * s| <= 2^14)
  float hl[2];   // KH: 1 / s of the lane's output rows 2 tig + {0, 1}
  // KN with unstaged activations: this lane's x pairs (raw half2) of the current stage's
  // tiles, loaded one stage ahead so the L2 latency overlaps the previous stage's MMAs
  static constexpr bool PF = KN && !XS && !KH;
  uint32_t xw[TPW][MB];
  // KH with unstaged activations: this lane's 16 x of row gq per tile, loaded one stage ahead
  static constexpr bool HPF = KH && !XS;
  uint2 xh[TPW][2][2];
  PMPD_DEV void prefetch_xh(uint2 (&dst)[TPW][2][2], int kt0, int cnt) const {
    const bool rowok = gq < M;
#pragma unroll
    for (int q = 0; q < TPW; ++q)
#pragma unroll
      for (int cch = 0; cch < 2; ++cch)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = (kt0 + warp + q * NCW) * kTile + 32 * cch + 16 * h + 4 * tig;
          dst[q][cch][h] = (rowok && warp + q * NCW < cnt) ? make_uint2(xword(gq, k), xword(gq, k + 2)) : make_uint2(0u, 0u);
        }
  }
  // KN, batch <= 4: balanced digits v = 256*hi + lo (both s8), hi of row b in B column 2b and lo in
  // column 2b+1 -> ONE u8 x s8 IMMA per fragment (lane tig = b holds both sums); batch 8 keeps two
  static constexpr bool BAL = KN && MB <= 4;
  static constexpr float kQMax = BAL ? 32639.f : 32767.f;

  PMPD_DEV void prefetch_x(uint32_t (&dst)[TPW][MB], int kt0, int cnt) const {
#pragma unroll
    for (int q = 0; q < TPW; ++q)
#pragma unroll
      for (int b = 0; b < MB; ++b)
        dst[q][b] = (warp + q * NCW < cnt && (MB == 1 || b < M))
                        ? xword(b, (kt0 + warp + q * NCW) * kTile + 2 * lane)
                        : 0u;
  }

  PMPD_DEV void reset() {
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[t][e] = 0.f;
        dhi[t][e] = 0;
        dlo[t][e] = 0;
      }
#pragma unroll
    for (int b = 0; b < MB; ++b) bias[b] = 0.f;
    hbias2 = make_float2(0.f, 0.f);
  }

  // floor to a power of two, clamped to [2^-100, 2^100]
  static PMPD_DEV float pow2_floor(float v) {
    v = fminf(fmaxf(v, 7.8886091e-31f), 1.2676506e30f);
    return __uint_as_float(__float_as_uint(v) & 0x7F800000u);
  }

  // set the KN activation scale for n-group ng
  PMPD_DEV void enter_group(int ng) {
    (void)kQMax;  // KN only
    if constexpr (KH) {
      const float idm = __ldg(a.aux + ng);
      const float mg = mx[min(gq, MB - 1)];
      hs = (mg > 0.f && idm > 0.f) ? pow2_floor(16384.f * idm / mg) : 1.f;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const float m = mx[min(2 * tig + cc, MB - 1)];
        hl[cc] = (m > 0.f && idm > 0.f) ? 1.f / pow2_floor(16384.f * idm / m) : 1.f;
      }
    } else if constexpr (KN) {
      const float idm = __ldg(a.aux + ng);
#pragma unroll
      for (int b = 0; b < MB; ++b) {
        const float m = mx[b];
        qs[b] = (m > 0.f && idm > 0.f) ? kQMax * idm / m : 0.f;
      }
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const float m = mx[MB == 1 ? 0 : min(BAL ? tig : 2 * tig + cc, MB - 1)];
        ql[cc] = (m > 0.f && idm > 0.f) ? kQMax * idm / m : 0.f;
      }
    }
  }

  // XS = 3: the staged row holds the CTA's k-tiles only, from k = xkb on, wrapping past the last
  // k-tile to 0 (a stream-K range that crosses an n-group boundary)
  int xkb = 0, xkp = 0;
  PMPD_DEV int xmap(int k) const {
    if constexpr (XS == 3) return k >= xkb ? k - xkb : k - xkb + xkp;
    return k;
  }

  // x[b][k..k+1] as float2 (zero outside [0, k_real))
  PMPD_DEV float2 xpair(int b, int k) const {
    if constexpr (XS) {
      return __half22float2(*reinterpret_cast<const __half2*>(xs + b * xld + xmap(k)));
    } else {
      const __half* xr = xs + (int64_t)b * xld;
      if (k + 1 < a.k_real) return __half22float2(*reinterpret_cast<const __half2*>(xr + k));
      return make_float2(k < a.k_real ? __half2float(xr[k]) : 0.f, 0.f);
    }
  }
  PMPD_DEV uint32_t xword(int b, int k) const {
    if constexpr (XS) {
      return *reinterpret_cast<const uint32_t*>(xs + b * xld + xmap(k));
    } else {
      const __half* xr = xs + (int64_t)b * xld;
      if (k + 1 < a.k_real) return __ldg(reinterpret_cast<const unsigned int*>(xr + k));
      return k < a.k_real ? (uint32_t)__half_as_ushort(xr[k]) : 0u;
    }
  }

  template <int P>
  PMPD_DEV void load_planes(const uint8_t* st, int wslot, uint32_t (&pw)[4][4]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < P) {
        const uint4 v = *reinterpret_cast<const uint4*>(st + j * STILES * kTilePlaneBytes +
                                                        wslot * kTilePlaneBytes + lane * 16);
        pw[j][0] = v.x;
        pw[j][1] = v.y;
        pw[j][2] = v.z;
        pw[j][3] = v.w;
      } else {
        pw[j][0] = pw[j][1] = pw[j][2] = pw[j][3] = 0u;
      }
    }
  }

  // ------------------------------------------------------------- KN tiles (IMMA)
  // Processes the TPW tiles {wslot + q*NCW} of one stage (all in the same n-group)
  // phase by phase so their dependency chains interleave.
  template <int P>
  PMPD_DEV void tile_kn(const uint8_t* st, int wslot, int kt, int cnt) {
    uint32_t pw[TPW][4][4];
    float2 dl[TPW], mn[TPW];
    bool live[TPW];
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      const int sl = wslot + q * NCW;
      live[q] = sl < cnt;
      if (live[q]) {
        load_planes<P>(st, sl, pw[q]);
        const float* sc = reinterpret_cast<const float*>(st + PMAX * STILES * kTilePlaneBytes + sl * kTileScaleBytes);
        dl[q] = *reinterpret_cast<const float2*>(sc + 2 * lane);
        mn[q] = *reinterpret_cast<const float2*>(sc + 64 + 2 * lane);
      }
    }
    // Activation operand: xq[b][k] = rint(x[b][k] * step[k] * qs[b]) as int16 (|.| <= 32767),
    // split into a u8 low digit and an s8 high digit.  Lane L owns k = 2L, 2L+1 (u16 stores);
    // storage is permuted so reader tig fetches {b0,b1} of both 32-k chunks with one LDS.128.
    const int wi = lane >> 1;
    const int pos = (((wi & 3) << 2) | (wi >> 2)) * 4 + 2 * (lane & 1);
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      if (!live[q]) continue;
      const int kk = (kt + q * NCW) * kTile + 2 * lane;
#pragma unroll
      for (int b = 0; b < MB; ++b) {
        if (MB == 1 || b < M) {
          float2 xf;
          if constexpr (PF)
            xf = __half22float2(*reinterpret_cast<const __half2*>(&xw[q][b]));
          else
            xf = xpair(b, kk);
          bias[b] = fmaf(xf.x, mn[q].x, fmaf(xf.y, mn[q].y, bias[b]));
          // 1.5 * 2^23 (+128 when balanced): the float's low 16 bits are rint(x*step*qs) (+128)
          constexpr float kMagic = BAL ? 12583040.f : 12582912.f;
          const float f0 = fmaf(xf.x * dl[q].x, qs[b], kMagic);
          const float f1 = fmaf(xf.y * dl[q].y, qs[b], kMagic);
          const uint32_t u0 = __float_as_uint(f0), u1 = __float_as_uint(f1);
          uint8_t* row = xq + (q * PL::kXqRows + b) * 128;
          *reinterpret_cast<uint16_t*>(row + pos) = (uint16_t)(__byte_perm(u0, u1, 0x0040) ^ (BAL ? 0x8080u : 0u));
          *reinterpret_cast<uint16_t*>(row + 64 + pos) = (uint16_t)__byte_perm(u0, u1, 0x0051);
        }
      }
    }
    __syncwarp();
    uint32_t bl[TPW][2][2], bh[TPW][2][2];
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      uint4 lo4 = make_uint4(0u, 0u, 0u, 0u), hi4 = lo4;
      if constexpr (BAL) {
        // column gq: row gq/2, high digits when gq is even, low digits when odd (loaded into hi4)
        if (live[q] && gq < 2 * (MB == 1 ? 1 : M)) {
          const uint8_t* row = xq + (q * PL::kXqRows + (gq >> 1)) * 128;
          hi4 = *reinterpret_cast<const uint4*>(row + ((gq & 1) ? 0 : 64) + tig * 16);
        }
      } else if (live[q] && gq < (MB == 1 ? 1 : M)) {
        const uint8_t* row = xq + (q * PL::kXqRows + (MB == 1 ? 0 : gq)) * 128;
        lo4 = *reinterpret_cast<const uint4*>(row + tig * 16);
        hi4 = *reinterpret_cast<const uint4*>(row + 64 + tig * 16);
      }
      bl[q][0][0] = lo4.x; bl[q][0][1] = lo4.y; bl[q][1][0] = lo4.z; bl[q][1][1] = lo4.w;
      bh[q][0][0] = hi4.x; bh[q][0][1] = hi4.y; bh[q][1][0] = hi4.z; bh[q][1][1] = hi4.w;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      if (!live[q]) continue;
#pragma unroll
      for (int cch = 0; cch < 2; ++cch) {
        const uint32_t pe[4] = {pw[q][0][2 * cch], pw[q][1][2 * cch], pw[q][2][2 * cch], pw[q][3][2 * cch]};
        const uint32_t po[4] = {pw[q][0][2 * cch + 1], pw[q][1][2 * cch + 1], pw[q][2][2 * cch + 1],
                                pw[q][3][2 * cch + 1]};
#define PMPD_KN_MTILE(T)                                                     \
  {                                                                          \
    uint32_t a0, a1, a2, a3;                                                 \
    nibble_to_u8<PMAX, P, T>(merge_planes<PMAX, P, T>(pe), a0, a1);          \
    nibble_to_u8<PMAX, P, T>(merge_planes<PMAX, P, T>(po), a2, a3);          \
    mma_u8s8_16832(dhi[T], a0, a1, a2, a3, bh[q][cch][0], bh[q][cch][1]);    \
    if constexpr (!BAL) mma_u8u8_16832(dlo[T], a0, a1, a2, a3, bl[q][cch][0], bl[q][cch][1]); \
  }
        PMPD_KN_MTILE(0)
        PMPD_KN_MTILE(1)
        PMPD_KN_MTILE(2)
        PMPD_KN_MTILE(3)
#undef PMPD_KN_MTILE
      }
    }
  }

  // ------------------------------------------------------------- KN tiles at batch 2..8 (HMMA)
  // The u8 fragments of tile_kn, read as f16 pairs: for k-chunk cch, A' = {a0 bytes 0-1, a1 bytes
  // 0-1, a0 bytes 2-3, a1 bytes 2-3} (and a2/a3 for the chunk's upper 16 k) is an m16n8k16 A
  // fragment whose logical k 2tig + e / 2tig + 8 + e are the physical k 4tig + e / 4tig + 2 + e;
  // B carries x * step of row gq at the same physical k, so each lane's B values are 4 runs of 4
  // consecutive k of its own row.
  template <int P>
  PMPD_DEV void tile_kh(const uint8_t* st, int wslot, int kt, int cnt) {
    uint32_t pw[TPW][4][4];
    bool live[TPW];
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      const int sl = wslot + q * NCW;
      live[q] = sl < cnt;
      if (live[q]) load_planes<P>(st, sl, pw[q]);
    }
    const bool rowok = gq < M;
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      if (!live[q]) continue;
      const int sl = wslot + q * NCW;
      const float* sc = reinterpret_cast<const float*>(st + PMAX * STILES * kTilePlaneBytes + sl * kTileScaleBytes);
      const int k0 = (kt + q * NCW) * kTile;
      // this lane's 16 x of row gq: staged rows are zero past M and past K (one 8-byte load per
      // 4 k); unstaged rows come from global memory with bounds
      uint2 xr[2][2];
#pragma unroll
      for (int cch = 0; cch < 2; ++cch)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = k0 + 32 * cch + 16 * h + 4 * tig;
          if constexpr (XS) {
            xr[cch][h] = *reinterpret_cast<const uint2*>(xrow + xmap(k));
          } else {
            xr[cch][h] = xh[q][cch][h];  // (prefetched a stage ahead by run())
            (void)rowok;
          }
        }
      uint32_t bfr[2][2][2];  // [cch][h][b0 | b1]
      const float2 hs2 = make_float2(hs, hs);
#pragma unroll
      for (int cch = 0; cch < 2; ++cch)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kl = 32 * cch + 16 * h + 4 * tig;
          const float2 x01 = __half22float2(*reinterpret_cast<const __half2*>(&xr[cch][h].x));
          const float2 x23 = __half22float2(*reinterpret_cast<const __half2*>(&xr[cch][h].y));
          const float4 d = *reinterpret_cast<const float4*>(sc + kl);
          const float4 mn = *reinterpret_cast<const float4*>(sc + 64 + kl);
          hbias2 = ffma2(x01, make_float2(mn.x, mn.y), hbias2);
          hbias2 = ffma2(x23, make_float2(mn.z, mn.w), hbias2);
          const float2 v01 = fmul2(fmul2(x01, make_float2(d.x, d.y)), hs2);
          const float2 v23 = fmul2(fmul2(x23, make_float2(d.z, d.w)), hs2);
          const __half2 b0 = __floats2half2_rn(v01.x, v01.y);
          const __half2 b1 = __floats2half2_rn(v23.x, v23.y);
          bfr[cch][h][0] = *reinterpret_cast<const uint32_t*>(&b0);
          bfr[cch][h][1] = *reinterpret_cast<const uint32_t*>(&b1);
        }
#pragma unroll
      for (int cch = 0; cch < 2; ++cch) {
        const uint32_t pe[4] = {pw[q][0][2 * cch], pw[q][1][2 * cch], pw[q][2][2 * cch], pw[q][3][2 * cch]};
        const uint32_t po[4] = {pw[q][0][2 * cch + 1], pw[q][1][2 * cch + 1], pw[q][2][2 * cch + 1],
                                pw[q][3][2 * cch + 1]};
#define PMPD_KH_MTILE(T)                                                                                  \
  {                                                                                                       \
    uint32_t a0, a1, a2, a3;                                                                              \
    nibble_to_u8<PMAX, P, T>(merge_planes<PMAX, P, T>(pe), a0, a1);                                       \
    nibble_to_u8<PMAX, P, T>(merge_planes<PMAX, P, T>(po), a2, a3);                                       \
    mma_f16_16816(acc[T], __byte_perm(a0, 0u, 0x4140), __byte_perm(a1, 0u, 0x4140), __byte_perm(a0, 0u, 0x4342), \
                  __byte_perm(a1, 0u, 0x4342), bfr[cch][0][0], bfr[cch][0][1]);                           \
    mma_f16_16816(acc[T], __byte_perm(a2, 0u, 0x4140), __byte_perm(a3, 0u, 0x4140), __byte_perm(a2, 0u, 0x4342), \
                  __byte_perm(a3, 0u, 0x4342), bfr[cch][1][0], bfr[cch][1][1]);                           \
  }
        PMPD_KH_MTILE(0)
        PMPD_KH_MTILE(1)
        PMPD_KH_MTILE(2)
        PMPD_KH_MTILE(3)
#undef PMPD_KH_MTILE
      }
    }
  }

  // ------------------------------------------------------------- NK tile (HMMA)
  template <int P>
  PMPD_DEV void tile_nk(const uint8_t* st, int wslot, int kt) {
    constexpr uint32_t ONES = 0x3C003C00u;
    const int k0 = kt * kTile;
    uint32_t pw[4][4];
    load_planes<P>(st, wslot, pw);
    const float* sc =
        reinterpret_cast<const float*>(st + PMAX * STILES * kTilePlaneBytes + wslot * kTileScaleBytes);
    uint32_t bfr[4][2];
    const bool live = gq < (MB == 1 ? 1 : M);
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int h = 0; h < 2; ++h) bfr[w][h] = live ? xword(gq, k0 + 16 * w + 2 * tig + 8 * h) : 0u;
    float cl[4][4];
    float sx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) cl[t][e] = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      mma_f16_16816(sx, ONES, ONES, ONES, ONES, bfr[w][0], bfr[w][1]);
      const uint32_t pj[4] = {pw[0][w], pw[1][w], pw[2][w], pw[3][w]};
#define PMPD_NK_MTILE(T)                                                   \
  {                                                                        \
    uint32_t a0, a1, a2, a3;                                               \
    nibble_to_frag<PMAX, P, T>(merge_planes<PMAX, P, T>(pj), a0, a1, a2, a3); \
    mma_f16_16816(cl[T], a0, a1, a2, a3, bfr[w][0], bfr[w][1]);            \
  }
      PMPD_NK_MTILE(0)
      PMPD_NK_MTILE(1)
      PMPD_NK_MTILE(2)
      PMPD_NK_MTILE(3)
#undef PMPD_NK_MTILE
    }
    // rows of this lane: n_l = 16t + gq + 8h -> scale slot gq*8 + 2t + h
    const float4 d0 = *reinterpret_cast<const float4*>(sc + gq * 8);
    const float4 d1 = *reinterpret_cast<const float4*>(sc + gq * 8 + 4);
    const float4 m0 = *reinterpret_cast<const float4*>(sc + 64 + gq * 8);
    const float4 m1 = *reinterpret_cast<const float4*>(sc + 64 + gq * 8 + 4);
    const float dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    const float mm[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const float d = fmaf(-row_offset(t, h), sx[cc], cl[t][2 * h + cc]);
          acc[t][2 * h + cc] = fmaf(dd[2 * t + h], d, fmaf(mm[2 * t + h], sx[cc], acc[t][2 * h + cc]));
        }
  }

  PMPD_DEV void store(int ng, int nl, int b, float v) {
    const int n = ng * kTile + nl;
    if (n >= a.n_real) return;
    v *= a.alpha;
    if (a.y_dtype == PMPD_DTYPE_F32) {
      float* yp = reinterpret_cast<float*>(a.y) + (int64_t)b * a.ldy + n;
      *yp = a.accumulate ? *yp + v : v;
    } else {
      __half* yp = reinterpret_cast<__half*>(a.y) + (int64_t)b * a.ldy + n;
      *yp = __float2half(a.accumulate ? __half2float(*yp) + v : v);
    }
  }

  // cross-warp, then (if the n-group is split across CTAs) cross-CTA reduction
  PMPD_DEV void flush(int ng) {
    const int Me = MB == 1 ? 1 : M;
    float* rw = red + warp * 64 * MB;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int b = BAL ? tig : 2 * tig + cc;
          if (b < Me && (!BAL || cc == 0)) {
            float v;
            if constexpr (KH) {
              // f16 subnormal weights carry 2^-24, m-tile T bytes 2^T, B the row's scale s
              v = acc[t][2 * h + cc] * (16777216.f / (float)(1 << t)) * hl[cc];
            } else if constexpr (BAL) {
              // columns 2b / 2b+1 of this lane = high / low digit sums of row b
              const float q = ql[0];
              const float ds = q > 0.f ? __fdividef(1.f, q) * (1.f / (float)(1 << t)) : 0.f;
              v = fmaf(256.f, (float)dhi[t][2 * h], (float)dhi[t][2 * h + 1]) * ds;
            } else if constexpr (KN) {
              // y = (256*hi + lo) * 2^-t / qs[b]
              const float q = ql[MB == 1 ? 0 : cc];
              const float ds = q > 0.f ? __fdividef(1.f, q) * (1.f / (float)(1 << t)) : 0.f;
              v = fmaf(256.f, (float)dhi[t][2 * h + cc], (float)dlo[t][2 * h + cc]) * ds;
            } else {
              v = acc[t][2 * h + cc];
            }
            rw[(16 * t + gq + 8 * h) * MB + b] = v;
          }
        }
    if constexpr (KH) {
      // this lane's bias is row gq's: sum over the 4 lanes of the row
      float hb = hbias2.x + hbias2.y;
      hb += __shfl_xor_sync(0xffffffffu, hb, 1);
      hb += __shfl_xor_sync(0xffffffffu, hb, 2);
      if (tig == 0 && gq < Me) redb[warp * MB + gq] = hb;
    } else if constexpr (KN) {
#pragma unroll
      for (int b = 0; b < MB; ++b)
        if (MB == 1 || b < M) {
          const float s = warp_sum(bias[b]);
          if (lane == 0) redb[warp * MB + b] = s;
        }
    }
    named_bar_sync(1, NCW * 32);
    const int tid = threadIdx.x;
    float vals[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + r * NCW * 32;
      if (e < 64 * Me) {
        const int nl = e / Me, b = e - nl * Me;
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < NCW; ++w) v += red[(w * 64 + nl) * MB + b];
        if constexpr (KN) {
#pragma unroll
          for (int w = 0; w < NCW; ++w) v += redb[w * MB + b];
        }
        vals[r] = v;
      }
    }
    const bool whole = (T0 <= ng * KT) && ((ng + 1) * KT <= T1);
    if (whole) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int e = tid + r * NCW * 32;
        if (e < 64 * Me) store(ng, e / Me, e % Me, vals[r]);
      }
    } else {
      const int tile_first = ng * KT, tile_last = min((ng + 1) * KT, NT) - 1;
      const int c_first = (int)(((int64_t)(tile_first + 1) * G + NT - 1) / NT) - 1;
      const int c_last = (int)(((int64_t)(tile_last + 1) * G + NT - 1) / NT) - 1;
      float* part = a.partial + (int64_t)ng * a.max_slots * 64 * Me;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int e = tid + r * NCW * 32;
        if (e < 64 * Me) part[(int64_t)(c - c_first) * 64 * Me + e] = vals[r];
      }
      named_bar_sync(1, NCW * 32);
      if (tid == 0) {
        __threadfence();  // cumulative: orders the CTA's partial stores (bar.sync) before the ticket
        sm.flag = (atomicAdd(&a.counters[ng], 1) == c_last - c_first);
      }
      named_bar_sync(1, NCW * 32);
      if (sm.flag) {
        __threadfence();
        for (int e = tid; e < 64 * Me; e += NCW * 32) {
          float v = 0.f;
          for (int s2 = 0; s2 <= c_last - c_first; ++s2) v += __ldcg(part + (int64_t)s2 * 64 * Me + e);
          store(ng, e / Me, e % Me, v);
        }
        if (tid == 0) a.counters[ng] = 0;
      }
    }
    named_bar_sync(1, NCW * 32);
    reset();
  }

  template <int P>
  PMPD_DEV void run() {
    reset();
    int si = 0;
    TileCursor cur{T0, T0 / KT, T0 % KT};
    enter_group(cur.ng);
    if constexpr (PF) prefetch_x(xw, cur.kt, cur.stage_end(T1, KT) - cur.t);
    if constexpr (HPF) prefetch_xh(xh, cur.kt, cur.stage_end(T1, KT) - cur.t);
    while (cur.t < T1) {
      const int end = cur.stage_end(T1, KT);
      const int slot = si % PL::kNst;
      uint32_t xn[TPW][MB];
      uint2 xhn[TPW][2][2];
      if constexpr (HPF) {
        int nkt = cur.kt + (end - cur.t);
        if (nkt == KT) nkt = 0;
        const TileCursor nx{end, 0, nkt};
        prefetch_xh(xhn, nkt, end < T1 ? nx.stage_end(T1, KT) - end : 0);
      }
      if constexpr (PF) {
        int nkt = cur.kt + (end - cur.t);
        if (nkt == KT) nkt = 0;
        const TileCursor nx{end, 0, nkt};
        prefetch_x(xn, nkt, end < T1 ? nx.stage_end(T1, KT) - end : 0);
      }
#ifndef PMPD_GEMV_SKIP_MEMORY
      mbar_wait(&sm.full[slot], (si / PL::kNst) & 1);
#endif
#ifdef PMPD_GEMV_SKIP_COMPUTE
      if (false) {
#else
      if (warp < end - cur.t) {
#endif
        if constexpr (KH) {
          tile_kh<P>(smem + PL::kRing + slot * PL::kStage, warp, cur.kt + warp, end - cur.t);
        } else if constexpr (KN) {
          tile_kn<P>(smem + PL::kRing + slot * PL::kStage, warp, cur.kt + warp, end - cur.t);
        } else {
#pragma unroll
          for (int q = 0; q < TPW; ++q)
            if (warp + q * NCW < end - cur.t)
              tile_nk<P>(smem + PL::kRing + slot * PL::kStage, warp + q * NCW, cur.kt + warp + q * NCW);
        }
      }
      __syncwarp();
#ifndef PMPD_GEMV_SKIP_MEMORY
      if (lane == 0) mbar_arrive(&sm.empty[slot]);
#endif
      if constexpr (PF) {
#pragma unroll
        for (int q = 0; q < TPW; ++q)
#pragma unroll
          for (int b = 0; b < MB; ++b) xw[q][b] = xn[q][b];
      }
      if constexpr (HPF) {
#pragma unroll
        for (int q = 0; q < TPW; ++q)
#pragma unroll
          for (int cch = 0; cch < 2; ++cch)
#pragma unroll
            for (int h = 0; h < 2; ++h) xh[q][cch][h] = xhn[q][cch][h];
      }
      const int ng = cur.ng;
      cur.kt += end - cur.t;
      cur.t = end;
      ++si;
      if (cur.kt == KT || cur.t == T1) flush(ng);
      if (cur.kt == KT) {
        cur.kt = 0;
        ++cur.ng;
        if (cur.t < T1) enter_group(cur.ng);
      }
    }
  }
};

// ---------------------------------------------------------------- kernel
template <int LAYOUT, int PMAX, int MB, int XS>
__global__ void __launch_bounds__(NTHREADS, 1) qgemv_kernel(const GemvArgs a) {
  using PL = Plan<PMAX, MB, XS>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NT = a.n_tiles * a.k_tiles, KT = a.k_tiles;
  const int G = gridDim.x, c = blockIdx.x;
  const int T0 = (int)((int64_t)c * NT / G), T1 = (int)((int64_t)(c + 1) * NT / G);

  // p is written by the precision hook, which completes before any kernel of
  // the step may start (it never triggers early), so it is safe to read here.
  int p = *a.p_dev;
  if (p < 1 || p > PMAX) {
    if (threadIdx.x == 0 && c == 0) atomicExch(a.status, PMPD_ERR_CONTRACT);
    p = p < 1 ? 1 : PMAX;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < PL::kNst; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
#ifdef PMPD_GEMV_SKIP_MEMORY
    if (false) {
#else
    if (lane == 0) {
#endif
      const uint64_t pol = policy_evict_first();
      int si = 0;
      TileCursor cur{T0, T0 / KT, T0 % KT};
      while (cur.t < T1) {
        const int end = cur.stage_end(T1, KT);
        const int cnt = end - cur.t, slot = si % PL::kNst;
        if (si >= PL::kNst) mbar_wait_backoff(&sm.empty[slot], ((si / PL::kNst) & 1) ^ 1);
        uint8_t* st = smem_raw + PL::kRing + slot * PL::kStage;
        mbar_arrive_expect_tx(&sm.full[slot], (uint32_t)(cnt * kTilePlaneBytes * (p + 1)));
        for (int j = 0; j < p; ++j)
          bulk_g2s_stream(st + j * STILES * kTilePlaneBytes,
                          a.planes + j * a.plane_bytes + (int64_t)cur.t * kTilePlaneBytes, cnt * kTilePlaneBytes,
                          &sm.full[slot], pol);
        bulk_g2s_stream(st + PMAX * STILES * kTilePlaneBytes, a.scales + (int64_t)cur.t * kTileScaleBytes,
                        cnt * kTileScaleBytes, &sm.full[slot], pol);
        cur.kt += cnt;
        cur.t = end;
        if (cur.kt == KT) cur.kt = 0;
        ++si;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  Consumer<LAYOUT, PMAX, MB, XS> cs{a, sm, smem_raw};
  cs.xq = smem_raw + PL::kXq + warp * PL::kXqWarp;
  cs.red = reinterpret_cast<float*>(smem_raw + PL::kRed);
  cs.redb = reinterpret_cast<float*>(smem_raw + PL::kRedb);
  float* mxs = reinterpret_cast<float*>(smem_raw + PL::kMx);
  cs.mx = mxs;
  cs.warp = warp;
  cs.lane = lane;
  cs.gq = lane >> 2;
  cs.tig = lane & 3;
  cs.T0 = T0;
  cs.T1 = T1;
  cs.KT = KT;
  cs.NT = NT;
  cs.G = G;
  cs.c = c;
  cs.M = a.m;
  if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
    // zero the int8 activation rows that stay unused (b >= M)
    for (int i = lane; i < PL::kXqWarp / 4; i += 32) reinterpret_cast<uint32_t*>(cs.xq)[i] = 0u;
  }
  pdl_wait();  // activations and the workspace belong to the predecessor until here
  const int Me = MB == 1 ? 1 : a.m;
  // XS = 3: this CTA's k-tiles [kt0, kt0 + nkt) mod KT (all of them once the range spans KT)
  const int nkt = XS == 3 ? min(T1 - T0, KT) : KT;
  const int xkb = XS == 3 && T1 - T0 < KT ? (T0 % KT) * kTile : 0;
  const int xsld = MB == 1 ? kXsMaxK : (XS == 3 ? ((NT + G - 1) / G < KT ? (NT + G - 1) / G : KT) : KT) * kTile;
  float* red32 = reinterpret_cast<float*>(smem_raw + PL::kMx) + MAXM;  // 32 floats of scratch
  if ((PMPD_GEMV_ONEPASS || XS == 3) && ((XS && a.in_mode == 0) || (!XS && LAYOUT == PMPD_LAYOUT_KN))) {
    // Every row in one pass: a thread issues its loads of all rows of a K chunk before it uses
    // any (one L2 round trip per chunk, not one per row), and the per-row max |x| of every row is
    // reduced across warps with ONE barrier (the per-row form below paid a round trip and two
    // barriers per row: batch 8 spent most of a small GEMV staging its activations).
    constexpr int STEP = NCW * 32 * 8;  // halves per pass of the CTA (8 per thread, one uint4)
    constexpr int R = MB <= 2 ? 4 : 2;  // passes per chunk (MB x R load sites: keeps the code small)
    const int kp = XS ? nkt * kTile : a.k_real;  // staged (local) columns per row
    const int kfull = KT * kTile;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) && ((a.ldx & 7) == 0);
    __half* xs = reinterpret_cast<__half*>(smem_raw + PL::kXs);
    float mr[MB];
#pragma unroll
    for (int b = 0; b < MB; ++b) mr[b] = 0.f;
    for (int k0 = 0; k0 < kp; k0 += R * STEP) {
      uint4 v[MB][R];
#pragma unroll
      for (int b = 0; b < MB; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = k0 + r * STEP + (int)threadIdx.x * 8;
          v[b][r] = make_uint4(0u, 0u, 0u, 0u);
          if ((MB == 1 || b < Me) && k < kp) {
            int kg = k;  // the column in x of local column k
            if constexpr (XS == 3) {
              kg = k + xkb;
              if (kg >= kfull) kg -= kfull;
            }
            const __half* src = a.x + (int64_t)b * a.ldx + kg;
            v[b][r] = (vec_ok && kg + 8 <= a.k_real) ? __ldg(reinterpret_cast<const uint4*>(src))
                                                     : load_x8_tail(src, a.k_real - kg);
          }
        }
#pragma unroll
      for (int b = 0; b < MB; ++b)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = k0 + r * STEP + (int)threadIdx.x * 8;
          if ((MB == 1 || b < Me) && k < kp) {
            const __half2* h2 = reinterpret_cast<const __half2*>(&v[b][r]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 fv = __half22float2(h2[i]);
              mr[b] = fmaxf(mr[b], fmaxf(fabsf(fv.x), fabsf(fv.y)));
            }
            if constexpr (XS) *reinterpret_cast<uint4*>(xs + b * xsld + k) = v[b][r];
          }
        }
    }
    if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
      float* rmx = reinterpret_cast<float*>(smem_raw + PL::kRed);  // [NCW][MB] (free until the first flush)
#pragma unroll
      for (int b = 0; b < MB; ++b) {
        const float m = warp_max(mr[b]);
        if (lane == 0) rmx[warp * MB + b] = m;
      }
      named_bar_sync(1, NCW * 32);
      if ((int)threadIdx.x < Me) {
        float r = 0.f;
        for (int w = 0; w < NCW; ++w) r = fmaxf(r, rmx[w * MB + threadIdx.x]);
        mxs[threadIdx.x] = r;
      }
    }
  } else
  for (int b = 0; b < Me; ++b) {
    float m = 0.f;
    if constexpr (XS) {
      // stage x (zero-padded to a multiple of 64) in shared memory once, tracking max |x|
      __half* xs = reinterpret_cast<__half*>(smem_raw + PL::kXs);
      const int kp = KT * kTile;
      if (a.in_mode != 0) {
        // fused producer op: the row is f32; RMSNorm needs its sum of squares first
        const float* xr = a.xf + (int64_t)b * a.ldxf;
        float inv = 1.f;
        if (a.in_mode == 1) {
          float ss = 0.f;
#pragma unroll 4
          for (int k = threadIdx.x; k < a.k_real; k += NCW * 32) {
            const float v = xr[k];
            ss = fmaf(v, v, ss);
          }
          ss = warp_sum(ss);
          if (lane == 0) red32[warp] = ss;
          named_bar_sync(1, NCW * 32);
          float tot = 0.f;
          for (int w = 0; w < NCW; ++w) tot += red32[w];
          inv = rsqrtf(tot / (float)a.k_real + a.eps);
          named_bar_sync(1, NCW * 32);  // red32 is reused for the max below
        }
#pragma unroll 2
        for (int k = threadIdx.x * 2; k < kp; k += NCW * 32 * 2) {
          float v[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int kk = k + i;
            float r = 0.f;
            if (kk < a.k_real) {
              if (a.in_mode == 1) {
                r = xr[kk] * inv * a.gain[kk];
              } else {
                const float g = xr[kk];
                r = g / (1.f + __expf(-g)) * xr[kk + a.u_off];
              }
            }
            v[i] = r;
          }
          const __half2 h = __floats2half2_rn(v[0], v[1]);
          const float2 f = __half22float2(h);
          m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
          *reinterpret_cast<__half2*>(xs + b * xsld + k) = h;
        }
      } else
      for (int k = threadIdx.x * 8; k < kp; k += NCW * 32 * 8) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        const __half* src = a.x + (int64_t)b * a.ldx + k;
        if (k + 8 <= a.k_real && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          v = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
          __half tmp[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) tmp[i] = (k + i < a.k_real) ? src[i] : __float2half(0.f);
          v = *reinterpret_cast<const uint4*>(tmp);
        }
        const __half2* h2 = reinterpret_cast<const __half2*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __half22float2(h2[i]);
          m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
        }
        *reinterpret_cast<uint4*>(xs + b * xsld + k) = v;
      }
    } else if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
      for (int k = threadIdx.x; k < a.k_real; k += NCW * 32)
        m = fmaxf(m, fabsf(__half2float(a.x[(int64_t)b * a.ldx + k])));
    }
    if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
      m = warp_max(m);
      if (lane == 0) red32[warp] = m;
      named_bar_sync(1, NCW * 32);
      if (threadIdx.x == 0) {
        float r = 0.f;
        for (int w = 0; w < NCW; ++w) r = fmaxf(r, red32[w]);
        mxs[b] = r;
      }
      named_bar_sync(1, NCW * 32);
    }
  }
  if constexpr (XS && LAYOUT == PMPD_LAYOUT_KN && MB == MAXM) {
    // the f16 HMMA path reads row gq of every lane: rows past m are zero
    __half* xs = reinterpret_cast<__half*>(smem_raw + PL::kXs);
    for (int i = Me * xsld + threadIdx.x * 8; i < MB * xsld; i += NCW * 32 * 8)
      *reinterpret_cast<uint4*>(xs + i) = make_uint4(0u, 0u, 0u, 0u);
  }
  named_bar_sync(1, NCW * 32);
  if constexpr (XS) {
    cs.xs = reinterpret_cast<__half*>(smem_raw + PL::kXs);
    cs.xld = xsld;
    cs.xrow = cs.xs + (int64_t)cs.gq * xsld;
    cs.xkb = xkb;
    cs.xkp = KT * kTile;
  } else {
    cs.xs = a.x;
    cs.xld = a.ldx;
  }
  switch (p) {
    case 4:
      if constexpr (PMAX >= 4) cs.template run<4>();
      break;
    case 3:
      if constexpr (PMAX >= 3) cs.template run<3>();
      break;
    case 2:
      if constexpr (PMAX >= 2) cs.template run<2>();
      break;
    default:
      cs.template run<1>();
      break;
  }
}

template <int LAYOUT, int PMAX, int MB, int XS>
int launch_m(const GemvArgs& a, int grid, cudaStream_t s) {
  using PL = Plan<PMAX, MB, XS>;
  static_assert(PL::kBytes <= 232448, "GEMV shared-memory plan exceeds 227 KB");
  const size_t smem = PL::kBytes;
  auto kern = qgemv_kernel<LAYOUT, PMAX, MB, XS>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) return fail(PMPD_ERR_CUDA, "qgemv launch: %s", cudaGetErrorString(e));
  return PMPD_OK;
}

// rows of x the batch-2..8 kernel stages: KN at batch 5..8 reads all 8 rows (the rows past m are
// zero-filled for the f16 HMMA path), NK and the smaller row bounds the m given
inline int rows_staged(int layout, int m) {
  return layout == PMPD_LAYOUT_KN && m > 4 ? MAXM : m;
}

template <int LAYOUT, int PMAX>
int launch(const GemvArgs& a, int grid, cudaStream_t s) {
  if (a.m == 1)
    return a.k_tiles * kTile <= kXsMaxK ? launch_m<LAYOUT, PMAX, 1, 1>(a, grid, s)
                                        : launch_m<LAYOUT, PMAX, 1, 0>(a, grid, s);
#ifdef PMPD_GEMV_ONLY_B1  // (experiment builds: batch-1 instantiations only)
  return fail(PMPD_ERR_CONFIG, "this build has batch-1 GEMVs only");
#else
  // batch 2..8: the row count is a template bound (2, 4 or 8) so every per-row loop unrolls
  // into registers; rows past m are masked
  const int staged = rows_staged(LAYOUT, a.m) * a.k_tiles * kTile;
  // ranged (XS = 3): the most k-tiles one CTA of this grid touches
  const int64_t ntl = (int64_t)a.n_tiles * a.k_tiles;
  const int per_cta = (int)std::min<int64_t>((ntl + grid - 1) / grid, a.k_tiles);
  const int ranged = rows_staged(LAYOUT, a.m) * per_cta * kTile;
  const int xs = staged <= kXsMulti ? 1
               : (PMPD_GEMV_XS2 && a.in_mode == 0 && staged <= kXsBig) ? 2
               : (PMPD_GEMV_XS2 && a.in_mode == 0 && ranged <= kXsBig) ? 3 : 0;
#define PMPD_GEMV_XS_LAUNCH(MB_)                                      \
  return xs == 1 ? launch_m<LAYOUT, PMAX, MB_, 1>(a, grid, s)         \
       : xs == 2 ? launch_m<LAYOUT, PMAX, MB_, 2>(a, grid, s)         \
       : xs == 3 ? launch_m<LAYOUT, PMAX, MB_, 3>(a, grid, s)         \
                 : launch_m<LAYOUT, PMAX, MB_, 0>(a, grid, s)
  if (a.m == 2) PMPD_GEMV_XS_LAUNCH(2);
  if (a.m <= 4) PMPD_GEMV_XS_LAUNCH(4);
  PMPD_GEMV_XS_LAUNCH(MAXM);
#undef PMPD_GEMV_XS_LAUNCH
#endif
}

int ctas_per_sm() {
  static int v = 0;
  if (v == 0) {
    const char* e = getenv("PMPD_GEMV_CTAS_PER_SM");
    v = e ? atoi(e) : 1;
    if (v < 1 || v > 4) v = 1;
  }
  return v;
}

// Split-K grid: one CTA per SM over the contiguous tile range (n-groups shared by 2-3 CTAs are
// reduced through the workspace).
int grid_for(const pmpd_qtensor* t) {
  const int nt = t->n_tiles * t->k_tiles;
  const int g = num_sms() * ctas_per_sm();
  return nt < g ? nt : g;
}

// Launch grid: one CTA per n-group (no cross-CTA reduction: saves the partial write, the ticket
// and a second L2 round trip, ~3 us) when the n-groups fit one wave, or two waves at batch <= 2
// (measured, decode sweep); the split-K grid otherwise.
int launch_grid(const pmpd_qtensor* t, int m) {
  const int sms = num_sms();
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("PMPD_GEMV_SPLITK");  // diagnostics: 1 forces the split-K grid
    mode = e ? atoi(e) : 0;
  }
  // batch >= 4 on long K (>= 128 k-tiles): the per-CTA tile count of the n-group grid makes it
  // compute-bound; the split-K grid is ~10 % faster there (tools/gemv_grid_sweep.py, 11008x4096)
  const bool long_k = m >= 4 && t->k_tiles >= 128;
  if (mode != 1 && !long_k && (t->n_tiles <= sms || (m <= 2 && t->n_tiles <= 2 * sms))) return t->n_tiles;
  return grid_for(t);
}

int slots_for(const pmpd_qtensor* t) {
  const int nt = t->n_tiles * t->k_tiles, g = grid_for(t);
  const int min_per_cta = nt / g;  // >= 1
  return t->k_tiles / min_per_cta + 2;
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" {

int pmpd_gemv_workspace_bytes(const pmpd_qtensor* t, int32_t m, int64_t* bytes) {
  if (!t || !bytes) return fail(PMPD_ERR_CONFIG, "null argument");
  if (m < 1 || m > MAXM) return fail(PMPD_ERR_INPUT, "decode GEMV batch must be in [1, %d], got %d", MAXM, m);
  if (!is_tiled(t->layout)) return fail(PMPD_ERR_CONFIG, "GEMV needs a tiled layout (KN or NK)");
  if (t->n_tiles > kWsCounters) return fail(PMPD_ERR_CONFIG, "GEMV output too wide (%d n-tiles)", t->n_tiles);
  const int64_t head = kWsHead;
  *bytes = head + (int64_t)t->n_tiles * slots_for(t) * 64 * m * 4;
  return PMPD_OK;
}

}  // extern "C"

namespace {
struct GemvIn {
  int mode;
  const void* x;  // f16 (mode 0) or f32 (modes 1, 2)
  int ldx;
  const float* gain;
  float eps;
  int u_off;
};

int gemv_impl(const pmpd_qtensor* t, const GemvIn& in, int32_t m, const int32_t* p_dev, void* y, int32_t y_dtype,
              int32_t ldy, float alpha, int32_t accumulate, void* ws, int64_t ws_bytes, void* stream) {
  const void* x = in.x;
  const int32_t ldx = in.ldx;

  if (!t || !t->data) return fail(PMPD_ERR_CONFIG, "null quantized tensor");
  if (!is_tiled(t->layout)) return fail(PMPD_ERR_CONFIG, "GEMV needs a tiled layout (KN or NK)");
  if (m < 1 || m > MAXM) return fail(PMPD_ERR_INPUT, "decode GEMV batch must be in [1, %d], got %d", MAXM, m);
  if (ldx < t->k || ldy < t->n) return fail(PMPD_ERR_INPUT, "leading dimensions too small");
  if (y_dtype != PMPD_DTYPE_F32 && y_dtype != PMPD_DTYPE_F16) return fail(PMPD_ERR_CONFIG, "bad output dtype");
  if ((reinterpret_cast<uintptr_t>(x) & 3) || (in.mode == 0 && (ldx & 1)))
    return fail(PMPD_ERR_INPUT, "x must be 4-byte aligned");
  int64_t need = 0;
  if (int e = pmpd_gemv_workspace_bytes(t, m, &need)) return e;
  if (!ws || ws_bytes < need) return fail(PMPD_ERR_INPUT, "workspace too small: need %lld bytes", (long long)need);
  GemvArgs a;
  a.planes = static_cast<const uint8_t*>(t->data);
  a.scales = a.planes + (int64_t)t->p_max * t->plane_bytes;
  a.aux = reinterpret_cast<const float*>(a.scales + t->scale_bytes);
  a.plane_bytes = t->plane_bytes;
  a.n_tiles = t->n_tiles;
  a.k_tiles = t->k_tiles;
  a.n_real = t->n;
  a.k_real = t->k;
  a.p_max = t->p_max;
  a.p_dev = p_dev;
  a.x = static_cast<const __half*>(x);
  a.ldx = ldx;
  a.m = m;
  a.y = y;
  a.y_dtype = y_dtype;
  a.ldy = ldy;
  a.alpha = alpha;
  a.accumulate = accumulate;
  a.in_mode = in.mode;
  a.xf = static_cast<const float*>(in.x);
  a.ldxf = in.ldx;
  a.gain = in.gain;
  a.eps = in.eps;
  a.u_off = in.u_off;
  if (in.mode != 0) {
    const int kp = t->k_tiles * kTile;
    const bool staged = m == 1 ? kp <= kXsMaxK : rows_staged(t->layout, m) * kp <= kXsMulti;
    if (!staged) return fail(PMPD_ERR_CONFIG, "fused GEMV input needs the staged-activation path (m*K too large)");
    if (in.mode == 1 && !in.gain) return fail(PMPD_ERR_CONFIG, "RMSNorm input needs a gain vector");
    if (in.mode == 2 && in.u_off < t->k) return fail(PMPD_ERR_CONFIG, "SwiGLU input needs u_off >= K");
  }
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  a.counters = reinterpret_cast<int*>(w8);
  a.status = reinterpret_cast<int*>(w8) + kWsCounters;
  a.partial = reinterpret_cast<float*>(w8 + kWsHead);
  a.max_slots = slots_for(t);
  const int grid = launch_grid(t, m);
  cudaStream_t s = as_stream(stream);
  const bool kn = t->layout == PMPD_LAYOUT_KN;
  switch (t->p_max) {
    case 4:
      return kn ? launch<PMPD_LAYOUT_KN, 4>(a, grid, s) : launch<PMPD_LAYOUT_NK, 4>(a, grid, s);
    case 3:
      return kn ? launch<PMPD_LAYOUT_KN, 3>(a, grid, s) : launch<PMPD_LAYOUT_NK, 3>(a, grid, s);
    case 2:
      return kn ? launch<PMPD_LAYOUT_KN, 2>(a, grid, s) : launch<PMPD_LAYOUT_NK, 2>(a, grid, s);
    default:
      return kn ? launch<PMPD_LAYOUT_KN, 1>(a, grid, s) : launch<PMPD_LAYOUT_NK, 1>(a, grid, s);
  }
}

}  // namespace

extern "C" {

int pmpd_gemv(const pmpd_qtensor* t, const void* x, int32_t ldx, int32_t m, const int32_t* p_dev, void* y,
              int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate, void* ws, int64_t ws_bytes,
              void* stream) {
  const GemvIn in{0, x, ldx, nullptr, 0.f, 0};
  return gemv_impl(t, in, m, p_dev, y, y_dtype, ldy, alpha, accumulate, ws, ws_bytes, stream);
}

int pmpd_gemv_fused(const pmpd_qtensor* t, int32_t in_mode, const float* xf, int32_t ldxf, int32_t m,
                    const float* gain, float eps, int32_t u_off, const int32_t* p_dev, void* y, int32_t y_dtype,
                    int32_t ldy, float alpha, int32_t accumulate, void* ws, int64_t ws_bytes, void* stream) {
  if (in_mode != PMPD_GEMV_IN_RMSNORM && in_mode != PMPD_GEMV_IN_SWIGLU)
    return fail(PMPD_ERR_CONFIG, "unknown fused GEMV input mode %d", in_mode);
  if (!xf || (reinterpret_cast<uintptr_t>(xf) & 3)) return fail(PMPD_ERR_INPUT, "f32 input must be 4-byte aligned");
  const GemvIn in{in_mode, xf, ldxf, gain, eps, u_off};
  return gemv_impl(t, in, m, p_dev, y, y_dtype, ldy, alpha, accumulate, ws, ws_bytes, stream);
}

}  // extern "C"
