// Prefill GEMM on the nested bit-plane format, sm_100a tcgen05 tensor cores.
//
// Replaces `x @ model.weights(name, p)` at the linear call sites of the reference
// prefill (pkg/src/pmpd/tinylm.py:377-388 -> _forward 334-368, weights() 201-231)
// when x has many rows (a prompt): prefill is a real dense contraction, so the
// weights are dequantized once per CTA tile into f16 and fed to the 5th-gen
// tensor cores, instead of the batch<=8 decode GEMV (gemv.cu).
//
//   y[m][n] (+)= alpha * sum_k x[m][k] * W_p[n][k]       x: f16 [M][ldx], W: KN tiles
//
// CTA tile: 128 tokens (UMMA M) x 128 outputs (UMMA N = two 64-wide n-groups of the
// packed format), K in chunks of 64 (one packed tile row).  Per chunk, all 256 threads
//   * stage the x slice (128 x 64 f16) with cp.async into the UMMA K-major,
//     no-swizzle core-matrix layout (8 rows x 16 B per core matrix),
//   * dequantize the weight slice straight from planes 0..p-1 of the packed tiles:
//     bucket index -> fmaf(k, step, min) in f32 (bit-exact with the reference
//     dequantize, quant.py:199-215) -> f16, stored as W^T [n][k] in the same layout;
// then one thread issues 4 x tcgen05.mma.cta_group::1.kind::f16 (M128 N128 K16,
// f32 accumulator in TMEM) and tcgen05.commit arrives on the stage's mbarrier.  Two
// smem stages: the tensor core works on chunk c while the threads fill chunk c+1.
// Epilogue: tcgen05.ld (32x32b) of the accumulator rows -> alpha * acc (+ y) -> y.
#include <cuda_fp16.h>

#include "decode_core.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

constexpr int G_M = 128;        // tokens per CTA tile (UMMA M)
constexpr int G_N = 128;        // outputs per CTA tile (UMMA N): two packed n-groups
constexpr int G_KC = 64;        // K per chunk (one packed tile)
constexpr int G_THREADS = 256;
constexpr int G_STAGE_A = G_M * G_KC * 2;   // 16 KB
constexpr int G_STAGE_B = G_N * G_KC * 2;   // 16 KB
constexpr int G_STAGE = G_STAGE_A + G_STAGE_B;
constexpr int G_SMEM = 2 * G_STAGE + 1024;  // two stages + barriers / TMEM address
// UMMA no-swizzle K-major layout: core matrix (8 rows x 8 f16 = 128 B); K-adjacent core
// matrices LBO bytes apart, 8-row groups SBO bytes apart.
constexpr int G_LBO = 128;
constexpr int G_SBO = (G_KC / 8) * 128;     // 1024

PMPD_DEV uint32_t core_off(int row, int k) { return (row >> 3) * G_SBO + (k >> 3) * G_LBO + (row & 7) * 16 + (k & 7) * 2; }

// ------------------------------------------------------------------ tcgen05 wrappers
PMPD_DEV uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);             // start address
  d |= (uint64_t)((G_LBO >> 4) & 0x3FFF) << 16;       // leading byte offset (K direction)
  d |= (uint64_t)((G_SBO >> 4) & 0x3FFF) << 32;       // stride byte offset (M/N direction)
  d |= (uint64_t)1 << 46;                             // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE (bits 61-63)
  return d;
}
// kind::f16 instruction descriptor: f32 accumulator, f16 A and B, both K-major.
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(G_N >> 3) << 17) | ((uint32_t)(G_M >> 4) << 24);

PMPD_DEV void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
PMPD_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
PMPD_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
PMPD_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
PMPD_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

PMPD_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

PMPD_DEV void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
PMPD_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct GemmArgs {
  const uint8_t* planes;
  const uint8_t* scales;
  long long plane_bytes;
  int n_tiles, k_tiles, n_real, k_real;
  const __half* x;
  int M, ldx;
  void* y;
  int ldy, y_f16, accumulate;
  float alpha;
  const int32_t* p_dev;
  int* status;
};

// ------------------------------------------------------------------ weight dequant
// Thread (h, L, w) decodes word w of lane chunk L of packed tile h of this chunk: 32 codes
// (4 m-tiles t x 8 nibble slots s, layout.cuh kn_tile_coord), writes W^T[n][k] in f16.
template <int P>
PMPD_DEV void dequant_unit(const GemmArgs& g, int tile, int h, int L, int w, uint8_t* sb) {
  const int gq = L >> 2, tig = L & 3;
  uint32_t pw[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    pw[j] = j < P ? __ldg(reinterpret_cast<const uint32_t*>(g.planes + (int64_t)j * g.plane_bytes +
                                                             (int64_t)tile * kTilePlaneBytes + L * 16) + w)
                  : 0u;
  const int kb = 32 * (w >> 1) + 16 * (w & 1) + 4 * tig;  // 4 consecutive k of this word
  const float* sc = reinterpret_cast<const float*>(g.scales + (int64_t)tile * kTileScaleBytes);
  const float4 d4 = __ldg(reinterpret_cast<const float4*>(sc + kb));
  const float4 m4 = __ldg(reinterpret_cast<const float4*>(sc + 64 + kb));
  const float dl[4] = {d4.x, d4.y, d4.z, d4.w}, mn[4] = {m4.x, m4.y, m4.z, m4.w};
  constexpr uint32_t kLoaded = ((1u << 4) - 1) & ~((1u << (4 - P)) - 1);
  constexpr uint32_t kConst = (P < 4) ? (1u << (4 - P - 1)) : 0u;
#define PMPD_G_T(T)                                                                          \
  {                                                                                          \
    const uint32_t pe[4] = {pw[0], pw[1], pw[2], pw[3]};                                     \
    uint32_t u = merge_planes<4, P, T>(pe);                                                  \
    u = T ? rotr32(u, T) : u;                                                                \
    u = (u & (kLoaded * 0x11111111u)) | (kConst * 0x11111111u); /* 8 bucket indices */      \
    _Pragma("unroll") for (int hh = 0; hh < 2; ++hh) {                                       \
      __half v[4];                                                                           \
      _Pragma("unroll") for (int i = 0; i < 4; ++i) {                                        \
        const uint32_t kidx = (u >> (4 * (2 * i + hh))) & 15u;                               \
        const float kf = __uint_as_float(0x4B000000u | kidx) - 8388608.f;                    \
        v[i] = __float2half_rn(__fmaf_rn(kf, dl[i], mn[i]));                                 \
      }                                                                                      \
      const int n_l = h * 64 + 16 * T + gq + 8 * hh;                                         \
      *reinterpret_cast<uint2*>(sb + core_off(n_l, kb)) = *reinterpret_cast<const uint2*>(v); \
    }                                                                                        \
  }
  PMPD_G_T(0)
  PMPD_G_T(1)
  PMPD_G_T(2)
  PMPD_G_T(3)
#undef PMPD_G_T
}

PMPD_DEV void dequant_dispatch(int p, const GemmArgs& g, int tile, int h, int L, int w, uint8_t* sb) {
  switch (p) {
    case 4: dequant_unit<4>(g, tile, h, L, w, sb); break;
    case 3: dequant_unit<3>(g, tile, h, L, w, sb); break;
    case 2: dequant_unit<2>(g, tile, h, L, w, sb); break;
    default: dequant_unit<1>(g, tile, h, L, w, sb); break;
  }
}

__global__ void __launch_bounds__(G_THREADS, 1) gemm_kernel(const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mma_bar = reinterpret_cast<uint64_t*>(smem + 2 * G_STAGE);  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * G_STAGE + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = blockIdx.x, m0 = blockIdx.y * G_M;
  int p = *g.p_dev;
  if (p < 1 || p > 4) {
    if (tid == 0 && nb == 0 && blockIdx.y == 0 && g.status) atomicExch(g.status, PMPD_ERR_CONTRACT);
    p = p < 1 ? 1 : 4;
  }
  if (tid == 0) {
    mbar_init(&mma_bar[0], 1);
    mbar_init(&mma_bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(G_N)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int KC = g.k_tiles;
  // dequant unit of this thread: packed tile h (0/1) of the chunk, lane chunk L, word w
  const int uh = tid >> 7, uL = (tid >> 2) & 31, uw = tid & 3;
  const int ntile = 2 * nb + uh;
  for (int kc = 0; kc < KC; ++kc) {
    const int s = kc & 1;
    uint8_t* sa = smem + s * G_STAGE;
    uint8_t* sb = sa + G_STAGE_A;
    if (kc >= 2) mbar_wait(&mma_bar[s], ((kc - 2) >> 1) & 1);  // MMAs of chunk kc-2 have read stage s
    // x slice: 128 rows x 8 chunks of 16 B
#pragma unroll
    for (int i = 0; i < (G_M * G_KC / 8) / G_THREADS; ++i) {
      const int c = tid + i * G_THREADS, r = c >> 3, c8 = c & 7;
      const int m = m0 + r;
      const __half* src = g.x + (int64_t)(m < g.M ? m : 0) * g.ldx + kc * G_KC + 8 * c8;
      cp_async16(smem_u32(sa + core_off(r, 8 * c8)), src, m < g.M ? 16u : 0u);
    }
    // weight slice (an n-group past the matrix's last is zero)
    if (ntile < g.n_tiles) {
      dequant_dispatch(p, g, ntile * g.k_tiles + kc, uh, uL, uw, sb);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          *reinterpret_cast<uint2*>(sb + core_off(uh * 64 + 16 * t + (uL >> 2) + 8 * hh,
                                                  32 * (uw >> 1) + 16 * (uw & 1) + 4 * (uL & 3))) = make_uint2(0u, 0u);
    }
    cp_async_wait_all();
    fence_async_smem();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
      for (int k16 = 0; k16 < G_KC / 16; ++k16)
        umma_f16(tmem, smem_desc(a0 + k16 * 2 * G_LBO), smem_desc(b0 + k16 * 2 * G_LBO), kIdesc,
                 (kc > 0 || k16 > 0) ? 1u : 0u);
      umma_commit(&mma_bar[s]);
    }
  }
  // all MMAs done
  mbar_wait(&mma_bar[(KC - 1) & 1], ((KC - 1) >> 1) & 1);
  tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32*(w%4).., columns 64*(w/4)..+64
  {
    const int row = 32 * (warp & 3) + lane, m = m0 + row;
    const int c0 = 64 * (warp >> 2);
#pragma unroll
    for (int cc = 0; cc < 64; cc += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(c0 + cc), r);
      if (m < g.M) {
        const int n0 = nb * G_N + c0 + cc;
        if (g.y_f16) {
          __half* yr = static_cast<__half*>(g.y) + (int64_t)m * g.ldy + n0;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (n0 + i < g.n_real) {
              float v = g.alpha * __uint_as_float(r[i]);
              if (g.accumulate) v += __half2float(yr[i]);
              yr[i] = __float2half_rn(v);
            }
        } else {
          float* yr = static_cast<float*>(g.y) + (int64_t)m * g.ldy + n0;
          if (n0 + 16 <= g.n_real && (((uintptr_t)yr) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              float4 v = make_float4(g.alpha * __uint_as_float(r[i]), g.alpha * __uint_as_float(r[i + 1]),
                                     g.alpha * __uint_as_float(r[i + 2]), g.alpha * __uint_as_float(r[i + 3]));
              if (g.accumulate) {
                const float4 o = *reinterpret_cast<const float4*>(yr + i);
                v.x += o.x;
                v.y += o.y;
                v.z += o.z;
                v.w += o.w;
              }
              *reinterpret_cast<float4*>(yr + i) = v;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (n0 + i < g.n_real) yr[i] = g.alpha * __uint_as_float(r[i]) + (g.accumulate ? yr[i] : 0.f);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G_N) : "memory");
}

}  // namespace
}  // namespace pmpd

using namespace pmpd;

extern "C" int pmpd_gemm(const pmpd_qtensor* t, const void* x_dev, int32_t ldx, int32_t m, const int32_t* p_dev,
                         void* y_dev, int32_t y_dtype, int32_t ldy, float alpha, int32_t accumulate,
                         int32_t* status_dev, void* stream) {
  if (!t || !t->data || !x_dev || !y_dev || !p_dev) return fail(PMPD_ERR_CONFIG, "null argument");
  if (t->layout != PMPD_LAYOUT_KN || t->p_max != 4)
    return fail(PMPD_ERR_CONFIG, "the prefill GEMM needs KN tiles with p_max 4");
  if (m < 1) return fail(PMPD_ERR_INPUT, "prefill GEMM needs at least one row");
  if (t->k != t->k_tiles * kTile) return fail(PMPD_ERR_CONFIG, "prefill GEMM needs K a multiple of 64");
  if ((ldx & 7) || (reinterpret_cast<uintptr_t>(x_dev) & 15))
    return fail(PMPD_ERR_CONFIG, "prefill GEMM input must be 16-byte aligned rows");
  if (y_dtype != PMPD_DTYPE_F32 && y_dtype != PMPD_DTYPE_F16) return fail(PMPD_ERR_CONFIG, "bad output dtype");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, G_SMEM);
    attr = true;
  }
  GemmArgs g;
  g.planes = static_cast<const uint8_t*>(t->data);
  g.scales = g.planes + (int64_t)t->p_max * t->plane_bytes;
  g.plane_bytes = t->plane_bytes;
  g.n_tiles = t->n_tiles;
  g.k_tiles = t->k_tiles;
  g.n_real = t->n;
  g.k_real = t->k;
  g.x = static_cast<const __half*>(x_dev);
  g.M = m;
  g.ldx = ldx;
  g.y = y_dev;
  g.ldy = ldy;
  g.y_f16 = y_dtype == PMPD_DTYPE_F16;
  g.accumulate = accumulate;
  g.alpha = alpha;
  g.p_dev = p_dev;
  g.status = status_dev;
  dim3 grid((t->n_tiles + 1) / 2, (m + G_M - 1) / G_M);
  gemm_kernel<<<grid, G_THREADS, G_SMEM, as_stream(stream)>>>(g);
  return check_launch("prefill gemm launch");
}
