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

#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

constexpr int NCW = 8;                  // consumer warps
constexpr int NTHREADS = (NCW + 1) * 32;  // + producer warp
constexpr int NSTAGE = 4;               // smem ring depth
constexpr int STILES = NCW;             // tiles per stage (one per consumer warp)
constexpr int MAXM = 8;

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
  int* counters;   // [n_tiles]
  int* status;     // [1]
  float* partial;  // [n_tiles][max_slots][64][m]
  int max_slots;
};

struct Smem {
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  int flag;
};

// ---------------------------------------------------------------- decode core
// Merge planes 0..P-1 of word (w, t) into a nibble word.  Plane j's bits for
// m-tile t sit at rotl(0x11111111 << b_j, t); select-merging keeps each
// plane's own bit positions (positions of unread planes hold garbage and are
// masked off by the fragment conversion).
template <int PMAX, int P>
PMPD_DEV uint32_t merge_planes(const uint32_t (&pw)[4], const int t) {
  uint32_t acc = pw[0];
  uint32_t have = 0x11111111u << (PMAX - 1);
#pragma unroll
  for (int j = 1; j < P; ++j) {
    const uint32_t sel = __funnelshift_l(have, have, t);  // positions already taken (rotated)
    acc = (acc & sel) | (pw[j] & ~sel);
    have |= 0x11111111u << (PMAX - 1 - j);
  }
  return acc;
}

// fp16 A fragment from one nibble word of m-tile t (see layout.cuh).  Every
// half2 takes one slot pair whose 4 code bits sit at mantissa bits o+t..o+t+3
// (o = 0 or 4) of each half; OR-ing the exponent of 2^(10-o-t) makes the half
// exactly 2^(10-o-t) + k (k = bucket index).  For t = 3 the o = 4 position
// would reach the exponent field, so all four pairs use o = 0 via rotations.
template <int PMAX, int P, int T>
PMPD_DEV void nibble_to_frag(uint32_t u, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  // nibble bits that come from loaded planes, and the constant bucket-centre bit
  constexpr uint32_t kLoaded = ((1u << PMAX) - 1) & ~((1u << (PMAX - P)) - 1);
  constexpr uint32_t kConst = (P < PMAX) ? (1u << (PMAX - P - 1)) : 0u;
  constexpr uint32_t m0 = (kLoaded * 0x00010001u) << T;
  constexpr uint32_t g0 = (((uint32_t)(25 - T) << 10) | (kConst << T)) * 0x00010001u;
  const uint32_t u8 = rotr32(u, 8);
  a0 = (u & m0) | g0;
  a2 = (u8 & m0) | g0;
  if constexpr (T < 3) {
    constexpr uint32_t m4 = ((kLoaded << 4) * 0x00010001u) << T;
    constexpr uint32_t g4 = (((uint32_t)(21 - T) << 10) | (kConst << (T + 4))) * 0x00010001u;
    a1 = (u & m4) | g4;
    a3 = (u8 & m4) | g4;
  } else {
    a1 = (rotr32(u, 4) & m0) | g0;
    a3 = (rotr32(u, 12) & m0) | g0;
  }
}

// fp16 value offset carried by each A row after the MMA: 2^(10-t) for rows
// gq (a0/a2), 2^(6-t) for rows gq+8 (a1/a3) except t = 3 (2^7 for both).
PMPD_DEV float row_offset(int t, int h) { return (h && t < 3) ? (float)(64 >> t) : (float)(1024 >> t); }

// ---------------------------------------------------------------- consumer
// State of one consumer warp; run() is instantiated per (layout, p_max, p) so
// that the whole tile loop is specialised for the active precision.
template <int LAYOUT, int PMAX>
struct Consumer {
  const GemvArgs& a;
  Smem& sm;
  uint8_t* ring;
  __half* bt;
  float* red;
  float* redb;
  int warp, lane, gq, tig, T0, T1, KT, NT, G, c, stage_bytes, M;
  float acc[4][4];
  float aux[4];      // KN: ones-MMA column sums of B~ (cols 2tig, 2tig+1)
  float bias[MAXM];  // KN: this lane's part of sum_k x*min

  PMPD_DEV void reset() {
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[t][e] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) aux[e] = 0.f;
#pragma unroll
    for (int b = 0; b < MAXM; ++b) bias[b] = 0.f;
  }

  template <int P>
  PMPD_DEV void tile(const uint8_t* st, int wslot, int tile_idx) {
    constexpr uint32_t ONES = 0x3C003C00u;
    const int k0 = (tile_idx % KT) * kTile;
    uint32_t pw[4][4];
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
    const float* sc =
        reinterpret_cast<const float*>(st + PMAX * STILES * kTilePlaneBytes + wslot * kTileScaleBytes);
    uint32_t bfr[4][2];
    if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
      // B~[b][k] = fp16(x[b][k] * step[k]); bias[b] += x[b][k] * min[k]; lane owns k = 2*lane, 2*lane+1
      const float2 dl = *reinterpret_cast<const float2*>(sc + 2 * lane);
      const float2 mn = *reinterpret_cast<const float2*>(sc + 64 + 2 * lane);
      const int kk = k0 + 2 * lane;
#pragma unroll
      for (int b = 0; b < MAXM; ++b) {
        if (b < M) {
          float2 xf = make_float2(0.f, 0.f);
          const __half* xr = a.x + (int64_t)b * a.ldx;
          if (kk + 1 < a.k_real) {
            xf = __half22float2(*reinterpret_cast<const __half2*>(xr + kk));
          } else if (kk < a.k_real) {
            xf.x = __half2float(xr[kk]);
          }
          reinterpret_cast<__half2*>(bt + b * 64)[lane] = __floats2half2_rn(xf.x * dl.x, xf.y * dl.y);
          bias[b] = fmaf(xf.x, mn.x, fmaf(xf.y, mn.y, bias[b]));
        }
      }
      __syncwarp();
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        bfr[w][0] = *reinterpret_cast<const uint32_t*>(bt + gq * 64 + 16 * w + 2 * tig);
        bfr[w][1] = *reinterpret_cast<const uint32_t*>(bt + gq * 64 + 16 * w + 2 * tig + 8);
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int w = 0; w < 4; ++w)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kk = k0 + 16 * w + 2 * tig + 8 * h;
          uint32_t v = 0;
          if (gq < M) {
            const __half* xr = a.x + (int64_t)gq * a.ldx;
            if (kk + 1 < a.k_real)
              v = __ldg(reinterpret_cast<const unsigned int*>(xr + kk));
            else if (kk < a.k_real)
              v = (uint32_t)__half_as_ushort(xr[kk]);
          }
          bfr[w][h] = v;
        }
    }

    float cl[4][4];
    float sx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) cl[t][e] = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if constexpr (LAYOUT == PMPD_LAYOUT_KN)
        mma_f16_16816(aux, ONES, ONES, ONES, ONES, bfr[w][0], bfr[w][1]);
      else
        mma_f16_16816(sx, ONES, ONES, ONES, ONES, bfr[w][0], bfr[w][1]);
      const uint32_t pj[4] = {pw[0][w], pw[1][w], pw[2][w], pw[3][w]};
      uint32_t a0, a1, a2, a3;
      // m-tile t = 0..3 (compile-time t: masks and exponents are immediates)
#define PMPD_MTILE(T)                                                            \
  {                                                                              \
    const uint32_t u = merge_planes<PMAX, P>(pj, T);                             \
    nibble_to_frag<PMAX, P, T>(u, a0, a1, a2, a3);                               \
    if constexpr (LAYOUT == PMPD_LAYOUT_KN)                                      \
      mma_f16_16816(acc[T], a0, a1, a2, a3, bfr[w][0], bfr[w][1]);               \
    else                                                                         \
      mma_f16_16816(cl[T], a0, a1, a2, a3, bfr[w][0], bfr[w][1]);                \
  }
      PMPD_MTILE(0)
      PMPD_MTILE(1)
      PMPD_MTILE(2)
      PMPD_MTILE(3)
#undef PMPD_MTILE
    }
    if constexpr (LAYOUT == PMPD_LAYOUT_NK) {
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
    float* rw = red + warp * 64 * MAXM;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int b = 2 * tig + cc;
          if (b < M) {
            float v = acc[t][2 * h + cc];
            if constexpr (LAYOUT == PMPD_LAYOUT_KN) v = fmaf(-row_offset(t, h), aux[cc], v);
            rw[(16 * t + gq + 8 * h) * MAXM + b] = v;
          }
        }
    if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
#pragma unroll
      for (int b = 0; b < MAXM; ++b)
        if (b < M) {
          const float s = warp_sum(bias[b]);
          if (lane == 0) redb[warp * MAXM + b] = s;
        }
    }
    named_bar_sync(1, NCW * 32);
    const int tid = threadIdx.x;
    float vals[2] = {0.f, 0.f};
    int nv = 0;
    for (int e = tid; e < 64 * M; e += NCW * 32, ++nv) {
      const int nl = e / M, b = e % M;
      float v = 0.f;
      for (int w = 0; w < NCW; ++w) v += red[(w * 64 + nl) * MAXM + b];
      if constexpr (LAYOUT == PMPD_LAYOUT_KN)
        for (int w = 0; w < NCW; ++w) v += redb[w * MAXM + b];
      vals[nv] = v;
    }
    const bool whole = (T0 <= ng * KT) && ((ng + 1) * KT <= T1);
    if (whole) {
      nv = 0;
      for (int e = tid; e < 64 * M; e += NCW * 32, ++nv) store(ng, e / M, e % M, vals[nv]);
    } else {
      const int tile_first = ng * KT, tile_last = min((ng + 1) * KT, NT) - 1;
      const int c_first = (int)(((int64_t)(tile_first + 1) * G + NT - 1) / NT) - 1;
      const int c_last = (int)(((int64_t)(tile_last + 1) * G + NT - 1) / NT) - 1;
      float* part = a.partial + (int64_t)ng * a.max_slots * 64 * M;
      nv = 0;
      for (int e = tid; e < 64 * M; e += NCW * 32, ++nv) part[(int64_t)(c - c_first) * 64 * M + e] = vals[nv];
      __threadfence();
      named_bar_sync(1, NCW * 32);
      if (tid == 0) sm.flag = (atomicAdd(&a.counters[ng], 1) == c_last - c_first);
      named_bar_sync(1, NCW * 32);
      if (sm.flag) {
        __threadfence();
        for (int e = tid; e < 64 * M; e += NCW * 32) {
          float v = 0.f;
          for (int s2 = 0; s2 <= c_last - c_first; ++s2) v += __ldcg(part + (int64_t)s2 * 64 * M + e);
          store(ng, e / M, e % M, v);
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
    for (int t = T0; t < T1; ++si) {
      const int end = min(min(t + STILES, T1), (t / KT + 1) * KT);
      const int slot = si % NSTAGE;
      const int ng = t / KT;
      mbar_wait(&sm.full[slot], (si / NSTAGE) & 1);
      if (warp < end - t) tile<P>(ring + slot * stage_bytes, warp, t + warp);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[slot]);
      t = end;
      if (t == T1 || t / KT != ng) flush(ng);
    }
  }
};

// ---------------------------------------------------------------- kernel
template <int LAYOUT, int PMAX>
__global__ void __launch_bounds__(NTHREADS, 2) qgemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int stage_bytes = STILES * (PMAX + 1) * kTilePlaneBytes;
  uint8_t* ring = smem_raw + 128;
  __half* bt_all = reinterpret_cast<__half*>(ring + NSTAGE * stage_bytes);  // KN: [NCW][MAXM][64]
  float* red = reinterpret_cast<float*>(bt_all + NCW * MAXM * 64);          // [NCW][64][MAXM]
  float* redb = red + NCW * 64 * MAXM;                                      // [NCW][MAXM]

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
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int si = 0;
      for (int t = T0; t < T1; ++si) {
        const int end = min(min(t + STILES, T1), (t / KT + 1) * KT);
        const int cnt = end - t, slot = si % NSTAGE;
        if (si >= NSTAGE) mbar_wait(&sm.empty[slot], ((si / NSTAGE) & 1) ^ 1);
        uint8_t* st = ring + slot * stage_bytes;
        mbar_arrive_expect_tx(&sm.full[slot], (uint32_t)(cnt * kTilePlaneBytes * (p + 1)));
        for (int j = 0; j < p; ++j)
          bulk_g2s_stream(st + j * STILES * kTilePlaneBytes,
                          a.planes + j * a.plane_bytes + (int64_t)t * kTilePlaneBytes, cnt * kTilePlaneBytes,
                          &sm.full[slot], pol);
        bulk_g2s_stream(st + PMAX * STILES * kTilePlaneBytes, a.scales + (int64_t)t * kTileScaleBytes,
                        cnt * kTileScaleBytes, &sm.full[slot], pol);
        t = end;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  Consumer<LAYOUT, PMAX> cs{a, sm, ring, bt_all + warp * MAXM * 64, red, redb};
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
  cs.stage_bytes = stage_bytes;
  cs.M = a.m;
  if constexpr (LAYOUT == PMPD_LAYOUT_KN) {
    for (int i = lane; i < MAXM * 64; i += 32) cs.bt[i] = __float2half(0.f);
    __syncwarp();
  }
  pdl_wait();  // activations and the workspace belong to the predecessor until here
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

template <int LAYOUT, int PMAX>
int launch(const GemvArgs& a, int grid, cudaStream_t s) {
  const int stage_bytes = STILES * (PMAX + 1) * kTilePlaneBytes;
  const size_t smem = 128 + (size_t)NSTAGE * stage_bytes + NCW * MAXM * 64 * sizeof(__half) +
                      (NCW * 64 * MAXM + NCW * MAXM) * sizeof(float);
  auto kern = qgemv_kernel<LAYOUT, PMAX>;
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

int grid_for(const pmpd_qtensor* t) {
  const int nt = t->n_tiles * t->k_tiles;
  return nt < num_sms() ? nt : num_sms();
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
  const int64_t head = ((int64_t)t->n_tiles * 4 + 4 + 255) / 256 * 256;
  *bytes = head + (int64_t)t->n_tiles * slots_for(t) * 64 * m * 4;
  return PMPD_OK;
}

int pmpd_gemv(const pmpd_qtensor* t, const void* x, int32_t ldx, int32_t m, const int32_t* p_dev, void* y,
              int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate, void* ws, int64_t ws_bytes,
              void* stream) {
  if (!t || !t->data) return fail(PMPD_ERR_CONFIG, "null quantized tensor");
  if (!is_tiled(t->layout)) return fail(PMPD_ERR_CONFIG, "GEMV needs a tiled layout (KN or NK)");
  if (m < 1 || m > MAXM) return fail(PMPD_ERR_INPUT, "decode GEMV batch must be in [1, %d], got %d", MAXM, m);
  if (ldx < t->k || ldy < t->n) return fail(PMPD_ERR_INPUT, "leading dimensions too small");
  if (y_dtype != PMPD_DTYPE_F32 && y_dtype != PMPD_DTYPE_F16) return fail(PMPD_ERR_CONFIG, "bad output dtype");
  if ((reinterpret_cast<uintptr_t>(x) & 3) || (ldx & 1)) return fail(PMPD_ERR_INPUT, "x must be 4-byte aligned");
  int64_t need = 0;
  if (int e = pmpd_gemv_workspace_bytes(t, m, &need)) return e;
  if (!ws || ws_bytes < need) return fail(PMPD_ERR_INPUT, "workspace too small: need %lld bytes", (long long)need);
  GemvArgs a;
  a.planes = static_cast<const uint8_t*>(t->data);
  a.scales = a.planes + (int64_t)t->p_max * t->plane_bytes;
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
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  a.counters = reinterpret_cast<int*>(w8);
  a.status = reinterpret_cast<int*>(w8) + t->n_tiles;
  a.partial = reinterpret_cast<float*>(w8 + ((int64_t)t->n_tiles * 4 + 4 + 255) / 256 * 256);
  a.max_slots = slots_for(t);
  const int grid = grid_for(t);
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

}  // extern "C"
