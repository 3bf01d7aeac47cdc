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
// CTA tile: NG packed n-groups (UMMA N = 64*NG outputs) x MB blocks of 128 tokens (UMMA M =
// 128 each; MB accumulators of 64*NG TMEM columns), K in chunks of 64 (one packed tile row),
// in a shared-memory ring of NS stages.  Both operands use the K-major 128-byte-swizzle
// layout (one 128 B row = the chunk's 64 k of one token / output; 16 B units XOR-swizzled by
// row & 7), the layout TMA writes for a full-width box:
//   * producer warp (one lane): TMA -- one 64 k x 128 row box of x per token block (2-D tensor
//     map, zero-filled past the last row) and the chunk's NG packed tiles as stored (planes
//     0..p-1 + scale blocks, 1-D bulk copies).
//   * 16 dequant warps: bucket indices -> the reference's dequantized weight in f32,
//     fmaf(k, step, min) (bit-exact with quant.py:199-215), rounded once to f16 (FADD2/FFMA2 on
//     two weights per instruction), W^T [n][k] (conflict-free swizzled 8 B stores);
//     fence.proxy.async (their own smem stores only: every load is async-proxy TMA);
//     then one thread issues MB x 4 tcgen05.mma.cta_group::1.kind::f16 (M128 N64*NG K16, f32
//     accumulators in TMEM) and tcgen05.commit frees the stage.  Each dequantized weight tile
//     feeds MB*128 tokens and each x box NG*64 outputs; (NG, MB) are chosen per launch to
//     balance that reuse against filling the 148 SMs.
// Epilogue: tcgen05.ld (32x32b) of the accumulator rows -> smem tile -> alpha * acc (+ y) -> y
// in coalesced row segments.
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "decode_core.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"
#include "pmpd_internal.h"

namespace pmpd {
namespace {

// split-K arrival counters, one per output tile of a launch (self-resetting; launches on one stream)
constexpr int kGemmSems = 1 << 16;
__device__ unsigned g_gemm_sem[kGemmSems];

#ifndef PMPD_GEMM_PDL
#define PMPD_GEMM_PDL 1  // programmatic dependent launch (weights streamed before the wait on x)
#endif
constexpr int G_BM = 128;       // tokens per UMMA M block
constexpr int G_NG1 = 64;       // outputs per packed n-group
constexpr int G_KC = 64;        // K per chunk (one packed tile)
#ifndef PMPD_GEMM_DQ_WARPS
#define PMPD_GEMM_DQ_WARPS 16
#endif
constexpr int G_DQ = PMPD_GEMM_DQ_WARPS * 32;  // dequant threads (a multiple of 256: 256 units per n-group)
constexpr int G_DQG = G_DQ / 256;              // n-groups dequantized in parallel
static_assert(G_DQ % 256 == 0, "dequant warps come in groups of 8");
constexpr int G_PROD = G_DQ / 32;      // TMA producer warp
constexpr int G_MMA = G_DQ / 32 + 1;   // tcgen05.mma issue warp
constexpr int G_THREADS = G_DQ + 64;
constexpr int G_STAGE_A1 = G_BM * G_KC * 2;  // 16 KB: one x block (f16, SW128 layout)
constexpr int G_STAGE_B1 = G_NG1 * G_KC * 2; // 8 KB: one dequantized W^T n-group (f16, SW128 layout)
constexpr int G_SMEM_MAX = 227 * 1024;

template <int NG, int MB>
struct Cfg {
  static constexpr int N = NG * G_NG1;
  static constexpr int STAGE_B = NG * G_STAGE_B1;
  // Two load rings, one K chunk per stage.  x (MB SW128 tiles, one TMA box per token block) is
  // read by the tensor core, so an x stage is free only when the chunk's MMAs complete; the packed
  // tiles (5 regions: planes 0..3, scales, [NG][512 B] each) are read by the dequant warps, so a
  // weight stage is free as soon as the chunk is dequantized.  Separate rings let the weight
  // stream run ahead of the MMAs: dequantization of chunk c no longer waits for the TMA that
  // could only start when MMA(c - NS) released a shared stage (measured: that chain, not the
  // dequant arithmetic, set the pace).
  static constexpr int STAGE_X = MB * G_STAGE_A1;
  static constexpr int WR = NG * kTilePlaneBytes;  // one plane (or scale) region
  static constexpr int STAGE_W = (5 * WR + 127) / 128 * 128;
#ifndef PMPD_GEMM_NB
#define PMPD_GEMM_NB 3
#endif
  static constexpr int NB = PMPD_GEMM_NB;  // dequantized weight buffers
  static constexpr int AVAIL = G_SMEM_MAX - 2048;
  static constexpr int NSW = 3;
  static constexpr int NSX_FIT = (AVAIL - NB * STAGE_B - NSW * STAGE_W) / STAGE_X;
  static constexpr int NSX = NSX_FIT > 6 ? 6 : NSX_FIT;
  static constexpr int BUFB = NB * STAGE_B;
  static constexpr int SMEM = BUFB + NSX * STAGE_X + NSW * STAGE_W + 2048;  // + barriers, TMEM address, alignment slack
  static constexpr int TMEM_COLS = MB * N <= 32 ? 32 : MB * N <= 64 ? 64 : MB * N <= 128 ? 128 : MB * N <= 256 ? 256 : 512;
  static_assert(MB * N <= 512, "accumulators exceed TMEM");
  static_assert(NSX >= 2, "x ring too shallow");
  static_assert(NB <= 4, "barrier slots");
  // kind::f16 instruction descriptor: f32 accumulator, f16 A and B, both K-major, M128 x N.
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(G_BM >> 4) << 24);
};

// 128-byte-swizzled K-major tile: row r at 128 r, 16 B unit c at (c ^ (r & 7)).
PMPD_DEV uint32_t sw128_off(int row, int k) { return row * 128 + ((((k >> 3) ^ row) & 7) << 4) + (k & 7) * 2; }

// ------------------------------------------------------------------ tcgen05 wrappers
// SW128 K-major descriptor: 8-row groups 1024 B apart (SBO); LBO unused (1); the K16 step
// within the 128 B row advances the start address by 32 B.
PMPD_DEV uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                          // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                          // layout type: SWIZZLE_128B
  return d;
}

// Warp-wide issue: every lane runs the loop (so its addresses and counters are warp-uniform and
// live in uniform registers), one elected lane issues.  Issuing from a `lane == 0` branch made
// the compiler rebuild every operand with ELECT / R2UR.BROADCAST loops (~17 instructions per MMA):
// with 4 dequant warps on the same scheduler the issue warp then fell behind the 128-cycle MMAs.
PMPD_DEV void umma_f16_elect(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo, uint32_t d_hi, uint32_t idesc,
                             uint32_t accum) {
  // (descriptor = {lo, hi}: only the 14-bit start address in lo moves, smem addresses never carry
  // out of it, so the 64-bit descriptors are two 32-bit moves, not a 64-bit add per MMA)
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t.reg .b32 e;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %3};\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "elect.sync e|p, 0xffffffff;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@p tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, q;\n\t}"
      ::"r"(d_tmem), "r"(a_lo), "r"(b_lo), "r"(d_hi), "r"(idesc), "r"(accum)
      : "memory");
}
// Commit arriving on the mbarrier at this offset in every CTA of ctaMask (the x stage is shared
// by the cluster's multicast, so it is free only when every CTA's MMAs have read it).
PMPD_DEV void umma_commit_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 e;\n\t"
      "elect.sync e|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
      ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
PMPD_DEV void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 e;\n\t"
      "elect.sync e|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
      ::"r"(smem_u32(bar))
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

PMPD_DEV void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
PMPD_DEV void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// x box into the same smem offset of every CTA in ctaMask (cluster multicast); each destination
// CTA's mbarrier at the same offset receives the bytes it got.
PMPD_DEV void tma_3d_mc(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// f32 load from the same shared-memory offset in cluster CTA `rank` (distributed shared memory)
PMPD_DEV uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
PMPD_DEV float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));  // (ordered by the volatile cluster barriers)
  return v;
}
PMPD_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
PMPD_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// TMA descriptors of one launch: x as [K/64 chunks][M rows][64 k] (f16, 128 B swizzle); the bit
// planes as [plane][n_tiles][k_tiles][128 words] with plane[j] boxing planes 0..j (one load for
// the p active planes); the scale blocks as [n_tiles][k_tiles][128 words].
struct alignas(64) GemmMaps {
  CUtensorMap x;
  CUtensorMap plane[4];
  CUtensorMap scale;
};

struct GemmArgs {
  const uint8_t* planes;
  const uint8_t* scales;
  long long plane_bytes;
  int n_tiles, k_tiles, n_real;
  int M;
  void* y;
  int ldy, y_f16, accumulate;
  float alpha;
  const int32_t* p_dev;
  int* status;
  int splitk;  // > 1: blockIdx.z takes K chunks [z*KC/S, (z+1)*KC/S); f32 y only
  unsigned* sem;  // per-output-tile arrival counters (zero between launches, self-resetting)
  float* ws;      // split-K partial slices [S][M][ldw]
  int ldw;
  int par_reduce; // 1: every CTA of the launch is resident at once, so the S splits of a tile wait for
                  // each other and each sums 1/S of the tile's rows (else the last arriver sums all)
  int dsm_reduce; // 1: the S splits of a tile are one thread-block cluster (along z) and sum their
                  // partial tiles through distributed shared memory (no workspace, no counters)
};

// ------------------------------------------------------------------ weight dequant
// Packed f32x2 arithmetic (sm_100 FADD2 / FFMA2: each lane is an IEEE fma.rn / add.rn).
PMPD_DEV float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
PMPD_DEV float2 fma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
// Bytes j0, j0+1 of w hold bucket indices k (< 256): f16x2 of fmaf(k, step, min), rounded once.
PMPD_DEV uint32_t bucket_pair_f16(uint32_t w, int j0, float2 step, float2 mn) {
#ifdef GEMM_DQ_NOFP  // timing probe only: integer stand-ins for the f32 arithmetic (wrong results)
  return __byte_perm(w, __float_as_uint(step.x) ^ __float_as_uint(mn.y), 0x7540 + j0) ^
         __byte_perm(w, __float_as_uint(step.y) + __float_as_uint(mn.x), 0x7541 + j0);
#endif
  const float2 kf = add2(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540 + j0)),
                                     __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7541 + j0))),
                         make_float2(-8388608.f, -8388608.f));  // 2^23 + k - 2^23 = k, exact
  const float2 v = fma2(kf, step, mn);
  const __half2 h = __floats2half2_rn(v.x, v.y);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Thread (L, w, half) decodes m-tiles 2*half, 2*half+1 of word w of lane chunk L of the chunk's
// packed tile (16 codes, layout.cuh kn_tile_coord) and writes W^T[n][k] in f16.  Every address
// is fixed per thread for the whole launch (only the stage / buffer bases move), so the caller
// hands in precomputed offsets: the loop body is the dequant arithmetic and nothing else.
struct DqOffsets {
  int ld;        // L*16 + w*4: this thread's word in a 512 B plane chunk
  int sc;        // 4*kb: this thread's 4 consecutive steps (mins at +256)
  int st[2][2];  // [m-tile t of the pair][row gq | gq+8]: swizzled 8 B store offsets
};

#ifdef GEMM_DQ_NOSTORE  // timing probe only: dequantize but keep the weights out of shared memory
__device__ uint32_t g_dq_sink;
#define PMPD_DQ_STORE(addr, a, b) { if ((a ^ b) == 0x12345678u) g_dq_sink = a; }
#else
#define PMPD_DQ_STORE(addr, a, b) *reinterpret_cast<uint2*>(addr) = make_uint2(a, b);
#endif
template <int P, int HALF>
PMPD_DEV void dequant_unit(const uint8_t* pl, int pstride, const uint8_t* scl, const DqOffsets& o, uint8_t* sb) {
  uint32_t pw[4];
#ifdef GEMM_DQ_NOLOAD  // timing probe only: operands from registers instead of shared memory
#pragma unroll
  for (int j = 0; j < 4; ++j) pw[j] = (uint32_t)(size_t)pl * (j + 1) + o.ld;
  const float4 d4 = make_float4(__int_as_float(o.sc), 1.f, 2.f, 3.f), m4 = make_float4(1.f, (float)(size_t)scl, 3.f, 4.f);
#else
#pragma unroll
  for (int j = 0; j < 4; ++j) pw[j] = j < P ? *reinterpret_cast<const uint32_t*>(pl + j * pstride + o.ld) : 0u;
  const float4 d4 = *reinterpret_cast<const float4*>(scl + o.sc);
  const float4 m4 = *reinterpret_cast<const float4*>(scl + 256 + o.sc);
#endif
  // Each weight is the reference's dequantized value in f32, fmaf(k, step, min) (bit-exact with
  // float32(dequantize(qt, p)), quant.py:199-215), rounded ONCE to f16 for the tensor core: the
  // same operand precision as the fp16 baseline.  (Rounding step and min to f16 first puts one
  // shared error on all 64 weights of a group; through a model that bias reached 2e-2 logits
  // error on an ill-conditioned step, tools/prefill_rounding_probe.py.)  Two weights per
  // instruction: k -> f32 by the 2^23 exponent magic, then FADD2 / FFMA2 / F2FP.PACK.
  const float2 d01 = make_float2(d4.x, d4.y), d23 = make_float2(d4.z, d4.w);
  const float2 m01 = make_float2(m4.x, m4.y), m23 = make_float2(m4.z, m4.w);
  constexpr uint32_t kLoaded = ((1u << 4) - 1) & ~((1u << (4 - P)) - 1);
  constexpr uint32_t kConst = (P < 4) ? (1u << (4 - P - 1)) : 0u;
  constexpr uint32_t kl = kLoaded * 0x01010101u, kc = kConst * 0x01010101u;
#define PMPD_G_T(T, I)                                                                               \
  {                                                                                                  \
    uint32_t u = merge_planes<4, P, T>(pw);                                                          \
    u = T ? rotr32(u, T) : u; /* nibble slot s = bucket index of row 16T+gq+8(s&1), k = kb+(s>>1) */ \
    const uint32_t ev = lop3_and_or(u, kl, kc);          /* byte j = bucket index (row gq, kb+j) */  \
    const uint32_t od = lop3_and_or(u >> 4, kl, kc);     /* byte j = bucket index (row gq+8, kb+j) */\
    const uint32_t ve0 = bucket_pair_f16(ev, 0, d01, m01), ve1 = bucket_pair_f16(ev, 2, d23, m23);   \
    const uint32_t vo0 = bucket_pair_f16(od, 0, d01, m01), vo1 = bucket_pair_f16(od, 2, d23, m23);   \
    PMPD_DQ_STORE(sb + o.st[I][0], ve0, ve1)                                                        \
    PMPD_DQ_STORE(sb + o.st[I][1], vo0, vo1)                                                        \
  }
  PMPD_G_T(2 * HALF, 0)
  PMPD_G_T(2 * HALF + 1, 1)
#undef PMPD_G_T
}

// The dequant warps, specialised per precision and per m-tile half (uniform per warp): for each
// K chunk wait for a free weight buffer (its MMAs of NB chunks ago completed) and the chunk's
// packed tiles, dequantize, then each warp arrives on the buffer's full barrier.  No CTA-wide
// barrier: warps run ahead independently and the MMA warp issues as soon as all have arrived.
template <int P, int NG, int MB, int HALF>
PMPD_DEV void dequant_loop_h(int KC, int ngn, const uint8_t* wring, uint8_t* bufs, uint64_t* wfull, uint64_t* wempty,
                             uint64_t* bfull, uint64_t* bempty, int g, const DqOffsets& o) {
  using C = Cfg<NG, MB>;
  constexpr int HN = (NG + G_DQG - 1) / G_DQG;  // n-groups per thread group
  int sw = 0, b = 0;                             // weight stage, weight buffer
  uint32_t wph = 0, bph = 0;                     // their mbarrier phases
#ifdef GEMM_TRACE
  long long tr_be = 0, tr_wf = 0, tr0 = clock64();
#endif
  for (int kc = 0; kc < KC; ++kc) {
    const uint8_t* w0 = wring + sw * C::STAGE_W;
    uint8_t* sb = bufs + b * C::STAGE_B;
#ifdef GEMM_TRACE
    long long t0 = clock64();
    if (kc >= C::NB) mbar_wait(&bempty[b], bph ^ 1u);
    long long t1 = clock64();
    mbar_wait(&wfull[sw], wph);
    tr_be += t1 - t0;
    tr_wf += clock64() - t1;
#else
    if (kc >= C::NB) mbar_wait(&bempty[b], bph ^ 1u);
    mbar_wait(&wfull[sw], wph);
#endif
#ifndef GEMM_SKIP_DEQUANT
#pragma unroll
    for (int i = 0; i < HN; ++i) {
      const int h = g + i * G_DQG;
      if (h < NG) {
        if (h < ngn) {
          dequant_unit<P, HALF>(w0 + h * kTilePlaneBytes, C::WR, w0 + 4 * C::WR + h * kTilePlaneBytes, o,
                                sb + h * G_STAGE_B1);
        } else {  // n-group past the matrix: zero weights
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              *reinterpret_cast<uint2*>(sb + h * G_STAGE_B1 + o.st[t][hh]) = make_uint2(0u, 0u);
        }
      }
    }
#endif
    fence_async_smem();  // this thread's dequant stores -> visible to the tensor core (async proxy)
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      mbar_arrive(&bfull[b]);
      mbar_arrive(&wempty[sw]);  // every load of the stage has returned (its values were stored)
    }
    if (++sw == C::NSW) {
      sw = 0;
      wph ^= 1u;
    }
    if (++b == C::NB) {
      b = 0;
      bph ^= 1u;
    }
  }
#ifdef GEMM_TRACE
  if (blockIdx.x % 16 == 0 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 352))
    printf("cta %d,%d dq thread %d: loop %lld cyc, wait bempty %lld, wait wfull %lld\n", blockIdx.x, blockIdx.y,
           threadIdx.x, clock64() - tr0, tr_be, tr_wf);
#endif
}

template <int P, int NG, int MB>
PMPD_DEV void dequant_loop(int KC, int ngn, const uint8_t* wring, uint8_t* bufs, uint64_t* wfull, uint64_t* wempty,
                           uint64_t* bfull, uint64_t* bempty, int tid) {
  // Thread (L, w, half) of an n-group's 256: warp wq = tt >> 5 of the 8 takes lane chunks
  // L = 8 (wq & 3) .. + 7 and m-tile half wq >> 2.  Lane l = [j>>2 : w>>1 : w&1 : j&3] (bit 4..0)
  // takes word w of chunk 8 (wq & 3) + j: the warp's 32 plane-word loads are 128 consecutive bytes
  // (one wavefront), and each 8-lane phase of the 128-bit scale loads reads 8 distinct 16 B slots
  // of one 128 B row (conflict-free; the former word-per-warp mapping cost a 4-way conflict on
  // every plane load and a 2-way one on every scale load).
  const int tt = tid & 255;  // unit within an n-group; thread group tid >> 8 takes n-groups h = g, g + G_DQG, ...
  const int wq = tt >> 5, l = tt & 31;
  const int uw = ((l >> 2) & 1) | (((l >> 3) & 1) << 1), uhalf = wq >> 2;
  const int uL = 8 * (wq & 3) + 4 * (l >> 4) + (l & 3);
  const int gq = uL >> 2, tig = uL & 3;
  const int kb = 32 * (uw >> 1) + 16 * (uw & 1) + 4 * tig;  // 4 consecutive k of this word
  DqOffsets o;
  o.ld = uL * 16 + uw * 4;
  o.sc = kb * 4;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) o.st[t][hh] = (int)sw128_off(16 * (2 * uhalf + t) + gq + 8 * hh, kb);
  if (uhalf == 0)
    dequant_loop_h<P, NG, MB, 0>(KC, ngn, wring, bufs, wfull, wempty, bfull, bempty, tid >> 8, o);
  else
    dequant_loop_h<P, NG, MB, 1>(KC, ngn, wring, bufs, wfull, wempty, bfull, bempty, tid >> 8, o);
}

// CL > 1: clusters of CL CTAs along N (same token rows, neighbouring n-blocks) share every x
// chunk: each CTA loads 128/CL rows of each block and multicasts them to the whole cluster, so
// the L2->SM traffic of x (the bulk of the load stream: 2 x 16 KB per chunk at MB = 2 against
// 10 KB of packed weights) drops CL-fold.
template <int NG, int MB, int CL>
__global__ void __launch_bounds__(G_THREADS, 1) gemm_kernel(const GemmArgs g, const __grid_constant__ GemmMaps maps) {
  using C = Cfg<NG, MB>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SW128 operand tiles need 1024-byte alignment
  // (offset the shared pointer itself: a round trip through uintptr_t loses the address space, and
  // every dequant load/store then compiled to a generic LD.E/ST.E on the long-scoreboard path)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* xring = smem + C::BUFB;                                                  // [NSX] x stages
  uint8_t* wring = xring + C::NSX * C::STAGE_X;                                     // [NSW] packed-tile stages
  uint64_t* xfull = reinterpret_cast<uint64_t*>(wring + C::NSW * C::STAGE_W);      // [NSX] x landed
  uint64_t* xempty = xfull + 8;                                                     // [NSX] x consumed (MMAs done)
  uint64_t* wfull = xfull + 16;                                                     // [NSW] packed tiles landed
  uint64_t* wempty = xfull + 24;                                                    // [NSW] packed tiles read
  uint64_t* bfull = xfull + 32;                                                     // [NB] weights dequantized
  uint64_t* bempty = xfull + 36;                                                    // [NB] weights consumed
  uint64_t* done_bar = xfull + 40;                                                  // every MMA of the CTA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + 41);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt0 = blockIdx.x * NG, m0 = blockIdx.y * (MB * G_BM);
  const int ngn = min(NG, g.n_tiles - nt0);  // n-groups of this CTA inside the matrix
  int p = *g.p_dev;
  if (p < 1 || p > 4) {
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && g.status) atomicExch(g.status, PMPD_ERR_CONTRACT);
    p = p < 1 ? 1 : 4;
  }
  if (tid == 0) {
    for (int i = 0; i < C::NSX; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], CL);  // one commit from every CTA of the cluster
    }
    for (int i = 0; i < C::NSW; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], G_DQ / 32);
    }
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(&bfull[i], G_DQ / 32);
      mbar_init(&bempty[i], 1);
    }
    mbar_init(done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // every CTA's barriers exist before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the next kernel of the stream may start its prologue (and, when
  // it is a GEMM, its weight stream and dequantization) once every CTA of this grid is running
  if (PMPD_GEMM_PDL) pdl_launch_dependents();
  const int crank = CL > 1 ? (int)cluster_rank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1);
  // this CTA's K chunks: all of them, or its split-K slice [kbase, kbase + KC)
  const int kbase = (int)(((long long)blockIdx.z * g.k_tiles) / g.splitk);
  const int KC = (int)(((long long)(blockIdx.z + 1) * g.k_tiles) / g.splitk) - kbase;
  // x blocks of this CTA that hold rows (blocks past M are neither loaded nor multiplied)
  const int mbn = min(MB, (g.M - m0 + G_BM - 1) / G_BM);

  if (warp == G_PROD) {
    // ---------------------------------------------------------------- TMA producer
    // One thread feeds both rings, never blocking on one while the other has a free stage: the
    // weight stream runs up to NSW chunks ahead of the dequant, x up to NSX ahead of the MMAs.
#ifdef GEMM_MMA_ONLY
    if (false) {
#else
    if (lane == 0) {
#endif
      int cx = 0, cw = 0, sx = 0, sw = 0;
      uint32_t xph = 0, wph = 0;
      // x is the previous kernel's output: it is loaded only after griddepcontrol.wait, which
      // this thread reaches once the weight ring's first fill is issued (the weights and the
      // precision word do not depend on the previous kernel)
      bool xok = !PMPD_GEMM_PDL;
      while (cx < KC || cw < KC) {
        bool idle = true;
        if (!xok && (cw == KC || cw == C::NSW)) {
          pdl_wait();
          xok = true;
        }
        if (cw < KC && (cw < C::NSW || mbar_try_wait(&wempty[sw], wph ^ 1u))) {
          uint8_t* dst = wring + sw * C::STAGE_W;
          mbar_arrive_expect_tx(&wfull[sw], (uint32_t)((p + 1) * C::WR));  // full boxes (zero-filled past the matrix)
          tma_4d(dst, &maps.plane[p - 1], 0, kbase + cw, nt0, 0, &wfull[sw]);  // planes 0..p-1
          tma_3d(dst + 4 * C::WR, &maps.scale, 0, kbase + cw, nt0, &wfull[sw]);
          ++cw;
          if (++sw == C::NSW) {
            sw = 0;
            wph ^= 1u;
          }
          idle = false;
        }
        if (xok && cx < KC && (cx < C::NSX || mbar_try_wait(&xempty[sx], xph ^ 1u))) {
          uint8_t* dst = xring + sx * C::STAGE_X;
#ifdef GEMM_SKIP_X  // timing probe only: x is not loaded (wrong results)
          mbar_arrive(&xfull[sx]);
#else
          mbar_arrive_expect_tx(&xfull[sx], (uint32_t)(mbn * G_STAGE_A1));
          if constexpr (CL > 1) {
            for (int mb = 0; mb < mbn; ++mb)
              tma_3d_mc(dst + mb * G_STAGE_A1 + crank * (G_STAGE_A1 / CL), &maps.x, 0, m0 + mb * G_BM + crank * (G_BM / CL),
                        kbase + cx, &xfull[sx], kMask);
          } else {
            for (int mb = 0; mb < mbn; ++mb) tma_3d(dst + mb * G_STAGE_A1, &maps.x, 0, m0 + mb * G_BM, kbase + cx, &xfull[sx]);
          }
#endif
          ++cx;
          if (++sx == C::NSX) {
            sx = 0;
            xph ^= 1u;
          }
          idle = false;
        }
        if (idle) __nanosleep(20);
      }
    }
  } else if (warp == G_MMA) {
    // ---------------------------------------------------------------- MMA issue (whole warp, one elected lane issues)
    {
      int sx = 0, b = 0;
      uint32_t xph = 0, bph = 0;
#ifdef GEMM_TRACE
      long long tw_b = 0, tw_x = 0, tstart = clock64();
#endif
      // descriptors: start address in bits [0,14) (16 B units); the K16 step adds 32 B = 2 units
      const uint64_t d0 = smem_desc_sw128(0);
      const uint32_t d_hi = (uint32_t)(d0 >> 32), d_lo = (uint32_t)d0;
      const uint32_t xa_lo = d_lo + (smem_u32(xring) >> 4), bb_lo = d_lo + (smem_u32(smem) >> 4);
      for (int kc = 0; kc < KC; ++kc) {
#ifndef GEMM_MMA_ONLY  // (timing probe: MMAs back to back on whatever the buffers hold)
#ifdef GEMM_TRACE
        long long t0 = clock64();
        mbar_wait(&bfull[b], bph);
        long long t1 = clock64();
        mbar_wait(&xfull[sx], xph);
        tw_b += t1 - t0;
        tw_x += clock64() - t1;
#else
        mbar_wait(&bfull[b], bph);  // the chunk's weights dequantized
        mbar_wait(&xfull[sx], xph); // and its x landed
#endif
#endif
        tc_fence_after();
        const uint32_t b_lo = bb_lo + (uint32_t)((b * C::STAGE_B) >> 4);
        const uint32_t a_lo = xa_lo + (uint32_t)((sx * C::STAGE_X) >> 4);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          if (mb < mbn) {
#ifndef GEMM_SKIP_MMA
#pragma unroll
            for (int k16 = 0; k16 < G_KC / 16; ++k16)
              umma_f16_elect(tmem + mb * C::N, a_lo + (uint32_t)((mb * G_STAGE_A1 + 32 * k16) >> 4), b_lo + 2u * k16, d_hi,
                             C::IDESC, (kc > 0 || k16 > 0) ? 1u : 0u);
#endif
          }
        }
        if constexpr (CL > 1)
          umma_commit_mc_elect(&xempty[sx], kMask);  // x stage reusable once every CTA of the cluster read it
        else
          umma_commit_elect(&xempty[sx]);  // x stage reusable
        umma_commit_elect(&bempty[b]);   // weight buffer reusable
        if (++sx == C::NSX) {
          sx = 0;
          xph ^= 1u;
        }
        if (++b == C::NB) {
          b = 0;
          bph ^= 1u;
        }
      }
      umma_commit_elect(done_bar);  // (tracks completion of every MMA issued before it)
#ifdef GEMM_TRACE
      if (lane == 0 && blockIdx.x % 16 == 0 && blockIdx.y == 0)
        printf("cta %d,%d KC %d: mma loop %lld cyc, wait bfull %lld, wait xfull %lld\n", blockIdx.x, blockIdx.y, KC,
               clock64() - tstart, tw_b, tw_x);
#endif
    }
  } else {
    // ---------------------------------------------------------------- dequant warps
#ifdef GEMM_MMA_ONLY
    if (false)
#endif
    switch (p) {
      case 4: dequant_loop<4, NG, MB>(KC, ngn, wring, smem, wfull, wempty, bfull, bempty, tid); break;
      case 3: dequant_loop<3, NG, MB>(KC, ngn, wring, smem, wfull, wempty, bfull, bempty, tid); break;
      case 2: dequant_loop<2, NG, MB>(KC, ngn, wring, smem, wfull, wempty, bfull, bempty, tid); break;
      default: dequant_loop<1, NG, MB>(KC, ngn, wring, smem, wfull, wempty, bfull, bempty, tid); break;
    }
  }
  // all MMAs done
  mbar_wait(done_bar, 0);
  tc_fence_after();
  // (the producer's griddepcontrol.wait returned before any MMA: the previous kernel has
  // completed; this makes its writes to y, the split-K workspace and the counters visible here)
  if (PMPD_GEMM_PDL) pdl_wait();
  // epilogue, per accumulator block: TMEM -> smem tile [128 rows][N (+1 pad)] f32 (warp w reads
  // TMEM lanes 32*(w%4).., columns half w/4), then all 256 threads write y in coalesced row
  // segments (the operand ring is free: every MMA has completed and every TMA landed).
  if (warp < G_DQ / 32) {
    constexpr int LDT = C::N + 1;  // padded row stride (floats): conflict-free column writes
    float* tile = reinterpret_cast<float*>(smem);
    // Split-K: every split writes alpha * its partial to its own slice of the workspace; the LAST
    // split to arrive at the tile (arrival counter) sums the slices in split order 0..S-1 (+ y
    // when accumulating) and writes y.  The sum order is fixed, so results are bit-reproducible
    // run to run, and no split waits for another (non-last splits simply exit).
    const int sk = g.splitk;
    const bool dsm = sk > 1 && g.dsm_reduce;
    const int n0 = nt0 * G_NG1;
    constexpr int Q = C::N / 4;  // 4-column quads per row
    for (int mb = 0; mb < mbn; ++mb) {
      const int row = 32 * (warp & 3) + lane;
      constexpr int NQ = G_DQ / 128;  // column groups: warps w and w+4 share TMEM lanes 32*(w&3)
      for (int cc = (warp >> 2) * (C::N / NQ); cc < ((warp >> 2) + 1) * (C::N / NQ); cc += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(mb * C::N + cc), r);
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[row * LDT + cc + i] = __uint_as_float(r[i]);
      }
      named_bar_sync(1, G_DQ);
      const int rows = min(G_BM, g.M - (m0 + mb * G_BM));
      if (dsm) {
        // split z of the cluster sums rows [z*rows/S, (z+1)*rows/S) of this block over the S
        // partial tiles in split order 0..S-1 (the arithmetic of the workspace path below, so the
        // result is the same bits) and writes y
        cluster_sync_all();  // every split's partial tile of this block is in its shared memory
        const int z = blockIdx.z;
        const int r_lo = (z * rows) / sk, r_hi = ((z + 1) * rows) / sk;
        for (int qi = tid + r_lo * Q; qi < r_hi * Q; qi += G_DQ) {
          const int rr = qi / Q, c4 = (qi % Q) * 4, n = n0 + c4;
          if (n >= g.n_real) continue;
          const uint32_t la = smem_u32(tile + rr * LDT + c4);
          float o[4] = {0.f, 0.f, 0.f, 0.f};
          // every split's 4 values are requested before any is used (one DSMEM round trip)
          float q[4][4];
#pragma unroll
          for (int zz = 0; zz < 4; ++zz) {
            if (zz < sk) {
              const uint32_t ra = dsmem_addr(la, (uint32_t)zz);
#pragma unroll
              for (int i = 0; i < 4; ++i) q[zz][i] = ld_dsmem_f32(ra + 4u * i);
            }
          }
#pragma unroll
          for (int zz = 0; zz < 4; ++zz)  // fixed order
            if (zz < sk) {
#pragma unroll
              for (int i = 0; i < 4; ++i) o[i] = __fadd_rn(o[i], __fmul_rn(g.alpha, q[zz][i]));  // (no FMA contraction)
            }
          const int64_t m = m0 + mb * G_BM + rr;
          float* yr = static_cast<float*>(g.y) + m * g.ldy + n;
          if (n + 4 <= g.n_real && (((uintptr_t)yr) & 15) == 0) {
            float4 ov = make_float4(o[0], o[1], o[2], o[3]);
            if (g.accumulate) {
              const float4 yq = *reinterpret_cast<const float4*>(yr);
              ov.x += yq.x;
              ov.y += yq.y;
              ov.z += yq.z;
              ov.w += yq.w;
            }
            *reinterpret_cast<float4*>(yr) = ov;
          } else {
            for (int i = 0; i < 4 && n + i < g.n_real; ++i) yr[i] = o[i] + (g.accumulate ? yr[i] : 0.f);
          }
        }
        cluster_sync_all();  // every split has read this block's tiles: they may be overwritten / freed
        continue;
      }
      for (int qi = tid; qi < rows * Q; qi += G_DQ) {
        const int rr = qi / Q, c4 = (qi % Q) * 4, n = n0 + c4;
        if (n >= g.n_real) continue;
        const float* tr = tile + rr * LDT + c4;
        float v[4] = {g.alpha * tr[0], g.alpha * tr[1], g.alpha * tr[2], g.alpha * tr[3]};
        const int64_t m = m0 + mb * G_BM + rr;
        if (sk > 1) {  // this split's slice of the workspace ([S][M][ldw] f32)
          float* wr = g.ws + ((int64_t)blockIdx.z * g.M + m) * g.ldw + n;
          *reinterpret_cast<float4*>(wr) = make_float4(v[0], v[1], v[2], v[3]);
        } else if (g.y_f16) {
          __half* yr = static_cast<__half*>(g.y) + m * g.ldy + n;
          if (n + 4 <= g.n_real && !g.accumulate && (((uintptr_t)yr) & 7) == 0) {
            const __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
            uint2 pk;
            pk.x = *reinterpret_cast<const uint32_t*>(&h0);
            pk.y = *reinterpret_cast<const uint32_t*>(&h1);
            *reinterpret_cast<uint2*>(yr) = pk;
          } else {
            for (int i = 0; i < 4 && n + i < g.n_real; ++i)
              yr[i] = __float2half_rn(v[i] + (g.accumulate ? __half2float(yr[i]) : 0.f));
          }
        } else {
          float* yr = static_cast<float*>(g.y) + m * g.ldy + n;
          if (n + 4 <= g.n_real && (((uintptr_t)yr) & 15) == 0) {
            float4 o = make_float4(v[0], v[1], v[2], v[3]);
            if (g.accumulate) {
              const float4 q = *reinterpret_cast<const float4*>(yr);
              o.x += q.x;
              o.y += q.y;
              o.z += q.z;
              o.w += q.w;
            }
            *reinterpret_cast<float4*>(yr) = o;
          } else {
            for (int i = 0; i < 4 && n + i < g.n_real; ++i) yr[i] = v[i] + (g.accumulate ? yr[i] : 0.f);
          }
        }
      }
      named_bar_sync(1, G_DQ);  // the tile is reused by the next block
    }
    if (sk > 1 && !dsm) {
      const int sem_id = blockIdx.y * gridDim.x + blockIdx.x;
      uint32_t* flag = reinterpret_cast<uint32_t*>(tile);  // the smem tile is free now
      int r_lo = 0, r_hi = min(mbn * G_BM, g.M - m0);        // rows of the tile this CTA sums
      if (g.par_reduce) {
        // all splits of the tile arrive, then each sums its share of the rows in split order
        if (tid == 0) {
          __threadfence();  // this split's slice before its arrival
          atomicAdd(g.sem + sem_id, 1u);
          while (*reinterpret_cast<volatile unsigned*>(g.sem + sem_id) < (unsigned)sk) __nanosleep(32);
          __threadfence();  // every split's slice is visible before the reads below
          *flag = 1u;
        }
        const int rows_all = r_hi;
        r_lo = (int)(((long long)blockIdx.z * rows_all) / sk);
        r_hi = (int)(((long long)(blockIdx.z + 1) * rows_all) / sk);
      } else if (tid == 0) {
        __threadfence();  // this split's slice before its arrival
        const unsigned old = atomicAdd(g.sem + sem_id, 1u);
        const bool last = old == (unsigned)(sk - 1);
        if (last) {
          g.sem[sem_id] = 0;  // self-reset for the next launch
          __threadfence();    // every other split's slice is visible before the reads below
        }
        *flag = last ? 1u : 0u;
      }
      named_bar_sync(1, G_DQ);
      if (*flag) {
        for (int qi = tid + r_lo * Q; qi < r_hi * Q; qi += G_DQ) {
          const int rr = qi / Q, c4 = (qi % Q) * 4, n = n0 + c4;
          if (n >= g.n_real) continue;
          const int64_t m = m0 + rr;
          float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int z = 0; z < sk; ++z) {  // fixed order
            const float4 q = __ldcg(reinterpret_cast<const float4*>(g.ws + ((int64_t)z * g.M + m) * g.ldw + n));
            o.x += q.x;
            o.y += q.y;
            o.z += q.z;
            o.w += q.w;
          }
          float* yr = static_cast<float*>(g.y) + m * g.ldy + n;
          if (n + 4 <= g.n_real && (((uintptr_t)yr) & 15) == 0) {
            if (g.accumulate) {
              const float4 q = *reinterpret_cast<const float4*>(yr);
              o.x += q.x;
              o.y += q.y;
              o.z += q.z;
              o.w += q.w;
            }
            *reinterpret_cast<float4*>(yr) = o;
          } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
            for (int i = 0; i < 4 && n + i < g.n_real; ++i) yr[i] = ov[i] + (g.accumulate ? yr[i] : 0.f);
          }
        }
      }
      if (g.par_reduce && tid == 0) {
        // second arrival: the split that completes it (every split has passed its wait) resets the
        // counter for the next launch
        if (atomicAdd(g.sem + sem_id, 1u) == 2u * (unsigned)sk - 1u) g.sem[sem_id] = 0;
      }
    }
  }
  else if (g.splitk > 1 && g.dsm_reduce) {
    // barrier.cluster counts every thread of the cluster: the producer and MMA warps take part in
    // the epilogue's two cluster barriers per accumulator block
    for (int mb = 0; mb < mbn; ++mb) {
      cluster_sync_all();
      cluster_sync_all();
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS) : "memory");
}

template <int NG, int MB, int CL>
int launch(const GemmArgs& g_in, const GemmMaps& maps, int m, int n_tiles, cudaStream_t st) {
  GemmArgs g = g_in;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_kernel<NG, MB, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NG, MB>::SMEM);
    if (CL > 1) cudaFuncSetAttribute(gemm_kernel<NG, MB, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  const int nb = (n_tiles + NG - 1) / NG;
  dim3 grid((nb + CL - 1) / CL * CL, (m + MB * G_BM - 1) / (MB * G_BM), g.splitk);  // (a padding n-block computes zeros)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(G_THREADS);
  cfg.dynamicSmemBytes = Cfg<NG, MB>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = g.dsm_reduce ? g.splitk : 1;  // (split-K through DSMEM: the splits of a tile)
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = PMPD_GEMM_PDL ? 2 : 1;
  if (g.par_reduce && !g.dsm_reduce) {
    // the splits of a tile wait for each other: only when every CTA of the launch is co-resident
    // (clusters of 2 need SM pairs, so fewer than the SM count may be resident at once)
    static int max_ctas = -1;
    if (max_ctas < 0) {
      int nc = 0;
      if (CL > 1) {
        cudaLaunchConfig_t q = cfg;
        q.gridDim = dim3(CL, 1, 1);
        if (cudaOccupancyMaxActiveClusters(&nc, gemm_kernel<NG, MB, CL>, &q) != cudaSuccess) nc = 0;
        cudaGetLastError();
        max_ctas = nc * CL;
      } else {
        max_ctas = num_sms();
      }
    }
    if ((int64_t)grid.x * grid.y * grid.z > max_ctas) g.par_reduce = 0;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_kernel<NG, MB, CL>, g, maps);
  if (e != cudaSuccess) return fail(PMPD_ERR_CUDA, "prefill gemm launch: %s", cudaGetErrorString(e));
  return check_launch("prefill gemm launch");
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
  GemmArgs g;
  g.planes = static_cast<const uint8_t*>(t->data);
  g.scales = g.planes + (int64_t)t->p_max * t->plane_bytes;
  g.plane_bytes = t->plane_bytes;
  g.n_tiles = t->n_tiles;
  g.k_tiles = t->k_tiles;
  g.n_real = t->n;
  g.M = m;
  g.y = y_dev;
  g.ldy = ldy;
  g.y_f16 = y_dtype == PMPD_DTYPE_F16;
  g.accumulate = accumulate;
  g.alpha = alpha;
  g.p_dev = p_dev;
  g.status = status_dev;
  // driver entry point resolved at run time: the library must load on hosts without libcuda
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(PMPD_ERR_CUDA, "prefill gemm: cuTensorMapEncodeTiled is unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  // (n-groups, token blocks) per CTA from a cost model fitted to the measured config-4 sweep
  // (tools/gemm_cfg_sweep.sh, 16 dequant warps, f32 y): a CTA spends ~0.214 + 0.111*NG + 0.192*MB us
  // per K chunk (dequant grows with NG, x loads and MMAs with MB); time ~ waves x chunks x that.  Fewer CTAs with more
  // operand reuse win when the extra wave of a finer split would cost more than the reuse saves.
  const int mblocks = (m + G_BM - 1) / G_BM, sms = num_sms();
  static const int cand[][2] = {{4, 2}, {2, 4}, {2, 2}, {4, 1}, {1, 4}, {2, 1}, {1, 2}, {1, 1}};
  // Split-K (f32 output only): S CTAs share one output tile, each over K/S chunks, and add their
  // partials at L2 (vector red); it pays when the tile grid alone cannot fill the SMs without
  // re-dequantizing the weights for every 128-row block.  The partial adds cost ~1.5 us per M outputs per
  // split (fitted).
  int ng = 1, mb = 1, splitk = 1;
  double best = 1e30;
  static const double sk_cost = [] {  // µs per 1M outputs per split (fitted; PMPD_GEMM_SKCOST overrides)
    const char* e = getenv("PMPD_GEMM_SKCOST");
    return e ? atof(e) : 1.49;
  }();
  const int kc_all = t->k_tiles;
  for (const auto& c : cand) {
    const int mbe = c[1] < mblocks ? c[1] : mblocks;
    if (c[1] > 1 && mblocks < c[1] && c[1] / 2 >= mblocks) continue;  // would leave a whole accumulator idle
    for (int sk = 1; sk <= 4; sk *= 2) {
      if (sk > 1 && (y_dtype != PMPD_DTYPE_F32 || kc_all < 8 * sk)) break;
      const int64_t ctas = (int64_t)((t->n_tiles + c[0] - 1) / c[0]) * ((mblocks + c[1] - 1) / c[1]) * sk;
      const double waves = (double)((ctas + sms - 1) / sms);
      const double cost = waves * ((kc_all + sk - 1) / sk) * (0.214 + 0.111 * c[0] + 0.192 * mbe) +
                          (sk > 1 ? sk_cost * 1e-6 * sk * m * t->n : 0.0);
      if (cost < best * 0.999) {
        best = cost;
        ng = c[0];
        mb = c[1];
        splitk = sk;
      }
    }
  }
  if (const char* e = getenv("PMPD_GEMM_SPLITK")) {  // diagnostics: force the split count
    const int v = atoi(e);
    if ((v == 1 || v == 2 || v == 4) && (v == 1 || y_dtype == PMPD_DTYPE_F32)) splitk = v;
  }
  if (splitk > t->k_tiles) splitk = 1;  // every split needs at least one K chunk
  if (const char* e = getenv("PMPD_GEMM_CFG")) {  // diagnostics: force "ng,mb"
    int a = 0, b = 0;
    if (sscanf(e, "%d,%d", &a, &b) == 2 && (a == 1 || a == 2 || a == 4) && (b == 1 || b == 2 || b == 4) && a * b <= 8) {
      ng = a;
      mb = b;
    }
  }
  const int kcs = 1;  // one K chunk per TMA box (both rings stage single chunks)
  // PMPD_GEMM_CL=2: x multicast across clusters of 2 CTAs along N (halves the x traffic from L2;
  // measured neutral to 2 % slower on the config-4 shapes and the 7B stack: the launch is bound
  // by the dequant warps and the MMA issue, not by the load stream), off by default
  static const int cl_env = [] {
    const char* e = getenv("PMPD_GEMM_CL");
    return e ? atoi(e) : 1;
  }();
  const int nblk = (t->n_tiles + ng - 1) / ng;
  const int cl = (cl_env == 2 && nblk >= 2) ? 2 : 1;
  const int nblk_pad = (nblk + cl - 1) / cl * cl;
  GemmMaps maps;
  // x: [K/64 chunks][m rows][64 k] f16, box 64 k x 128 rows x 1 chunk -> one SW128 tile (zero-filled past m)
  {
    const cuuint64_t gdim[3] = {(cuuint64_t)G_KC, (cuuint64_t)m, (cuuint64_t)t->k_tiles};
    const cuuint64_t gstride[2] = {(cuuint64_t)ldx * 2, (cuuint64_t)G_KC * 2};
    const cuuint32_t box[3] = {(cuuint32_t)G_KC, (cuuint32_t)(G_BM / cl), (cuuint32_t)kcs};  // (a cluster CTA's share)
    const cuuint32_t estride[3] = {1, 1, 1};
    const CUresult r = encode(&maps.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(x_dev), gdim, gstride, box,
                              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PMPD_ERR_CUDA, "prefill gemm: x tensor map (%d)", (int)r);
  }
  // planes: [4][n_tiles][k_tiles][128 words of one 512 B tile], box 128 x 1 x NG x (j+1);
  // scales: [n_tiles][k_tiles][128], box 128 x 1 x NG
  {
    const cuuint64_t gdim[4] = {128, (cuuint64_t)t->k_tiles, (cuuint64_t)t->n_tiles, 4};
    const cuuint64_t gstride[3] = {(cuuint64_t)kTilePlaneBytes, (cuuint64_t)t->k_tiles * kTilePlaneBytes,
                                   (cuuint64_t)g.plane_bytes};
    const cuuint32_t estride[4] = {1, 1, 1, 1};
    for (int j = 0; j < 5; ++j) {
      const cuuint32_t box[4] = {128, (cuuint32_t)kcs, (cuuint32_t)ng, (cuuint32_t)(j < 4 ? j + 1 : 1)};
      void* base = j < 4 ? const_cast<uint8_t*>(g.planes) : const_cast<uint8_t*>(g.scales);
      const CUresult r = encode(j < 4 ? &maps.plane[j] : &maps.scale, CU_TENSOR_MAP_DATA_TYPE_UINT32, j < 4 ? 4 : 3,
                                base, gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(PMPD_ERR_CUDA, "prefill gemm: weight tensor map (%d)", (int)r);
    }
  }
  cudaStream_t st = as_stream(stream);
  g.splitk = splitk;
  g.sem = nullptr;
  g.ws = nullptr;
  g.ldw = t->n_tiles * G_NG1;
  g.par_reduce = 0;
  g.dsm_reduce = 0;
  // PMPD_GEMM_DSM=1: the splits of a tile as one cluster reducing through DSMEM. Measured slower
  // (7B stack at 512 rows 10.3 vs 8.85 ms; 4096^2 at M=512 56 vs 37 us): clusters of 2-4 CTAs
  // with ~200 KB of shared memory each co-schedule worse than independent CTAs. Off by default.
  const char* dsm_e = getenv("PMPD_GEMM_DSM");
  const bool dsm_env = dsm_e ? atoi(dsm_e) != 0 : false;
  if (splitk > 1 && cl == 1 && dsm_env) {
    g.dsm_reduce = 1;  // no workspace, no counters: the clusters reduce on chip
  } else if (splitk > 1) {
    // split-K workspace (grown on demand; launches on one stream reuse it in order). A buffer
    // that is outgrown is retired, never freed: a CUDA graph captured earlier (the model's graphed
    // prefill) still holds its address.
    static float* ws_buf = nullptr;
    static size_t ws_cap = 0;
    const int tiles = nblk_pad * ((m + mb * G_BM - 1) / (mb * G_BM));
    const size_t need = (size_t)splitk * m * g.ldw * sizeof(float);
    if (tiles > kGemmSems || need > ((size_t)1 << 30)) {
      splitk = 1;
    } else {
      if (need > ws_cap) {
        const size_t want = std::max(need, std::min(2 * ws_cap, (size_t)1 << 30));
        float* nb = nullptr;
        if (cudaMalloc(&nb, want) != cudaSuccess) return fail(PMPD_ERR_CUDA, "prefill gemm: split-K workspace");
        ws_buf = nb;
        ws_cap = want;
      }
      void* sp = nullptr;
      if (cudaGetSymbolAddress(&sp, g_gemm_sem) != cudaSuccess) return fail(PMPD_ERR_CUDA, "prefill gemm counters");
      g.sem = static_cast<unsigned*>(sp);
      g.ws = ws_buf;
      // one wave (every CTA resident at once): the splits of a tile share its final reduction
      static const bool par_env = !getenv("PMPD_GEMM_SERIAL_REDUCE");
      g.par_reduce = par_env && (int64_t)tiles * splitk <= num_sms() ? 1 : 0;
    }
    g.splitk = splitk;
  }
#define PMPD_GEMM_LAUNCH(NG_, MB_) \
  return cl == 2 ? launch<NG_, MB_, 2>(g, maps, m, t->n_tiles, st) : launch<NG_, MB_, 1>(g, maps, m, t->n_tiles, st)
  if (ng == 1 && mb == 4) PMPD_GEMM_LAUNCH(1, 4);
  if (ng == 2 && mb == 4) PMPD_GEMM_LAUNCH(2, 4);
  if (ng == 4 && mb == 2) PMPD_GEMM_LAUNCH(4, 2);
  if (ng == 4) PMPD_GEMM_LAUNCH(4, 1);
  if (ng == 2 && mb == 2) PMPD_GEMM_LAUNCH(2, 2);
  if (ng == 2) PMPD_GEMM_LAUNCH(2, 1);
  if (mb == 2) PMPD_GEMM_LAUNCH(1, 2);
  PMPD_GEMM_LAUNCH(1, 1);
#undef PMPD_GEMM_LAUNCH
}
