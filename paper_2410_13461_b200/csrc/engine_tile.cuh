// Consumer tile body of the persistent decode engine (engine.cu), in a header so that
// tools/microbench/etile_bench.cu measures exactly this code in isolation.
//
// One warp, up to TPW tiles of one n-group per call: decode the P planes of each 64x64 KN tile
// into u8 tensor-core fragments (decode_core.cuh), quantize x*step into a two-digit int16 B
// operand, and accumulate mma.sync m16n8k32 (u8 x s8 / u8 x u8) into int32 dhi/dlo.
#pragma once
#include "decode_core.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"

#ifndef PMPD_ENGINE_NCW
#define PMPD_ENGINE_NCW 8
#endif
#ifndef PMPD_ENGINE_TPW
#define PMPD_ENGINE_TPW 2
#endif

namespace pmpd {
constexpr int E_NCW = PMPD_ENGINE_NCW;      // consumer warps
constexpr int E_TPW = PMPD_ENGINE_TPW;      // tiles per consumer warp per stage
constexpr int E_STILES = E_NCW * E_TPW;     // tiles per stage

// ------------------------------------------------------------------ consumer tile
template <int P>
PMPD_DEV void engine_tile(const uint8_t* st, int stiles_cnt, int wslot, int kt, int lane, const __half* xs,
                          uint8_t* xq, float qs, int (&dhi)[4][4], int (&dlo)[4][4], float& bias) {
  const int gq = lane >> 2, tig = lane & 3;
  uint32_t pw[E_TPW][4][4];
  float2 dl[E_TPW], mn[E_TPW];
  bool live[E_TPW];
#pragma unroll
  for (int q = 0; q < E_TPW; ++q) {
    const int sl = wslot + q * E_NCW;
    live[q] = sl < stiles_cnt;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < P && live[q]) {
        const uint4 v = *reinterpret_cast<const uint4*>(st + j * E_STILES * kTilePlaneBytes + sl * kTilePlaneBytes +
                                                        lane * 16);
        pw[q][j][0] = v.x;
        pw[q][j][1] = v.y;
        pw[q][j][2] = v.z;
        pw[q][j][3] = v.w;
      } else {
        pw[q][j][0] = pw[q][j][1] = pw[q][j][2] = pw[q][j][3] = 0u;
      }
    }
    if (live[q]) {
      const float* sc = reinterpret_cast<const float*>(st + P * E_STILES * kTilePlaneBytes + sl * kTileScaleBytes);
      dl[q] = *reinterpret_cast<const float2*>(sc + 2 * lane);
      mn[q] = *reinterpret_cast<const float2*>(sc + 64 + 2 * lane);
    } else {
      dl[q] = mn[q] = make_float2(0.f, 0.f);
    }
  }
  const int wi = lane >> 1;
  const int pos = (((wi & 3) << 2) | (wi >> 2)) * 4 + 2 * (lane & 1);
#pragma unroll
  for (int q = 0; q < E_TPW; ++q) {
    if (!live[q]) continue;
    const int kk = (kt + q * E_NCW) * kTile + 2 * lane;
    const float2 xf = __half22float2(*reinterpret_cast<const __half2*>(xs + kk));
    bias = fmaf(xf.x, mn[q].x, fmaf(xf.y, mn[q].y, bias));
    const float f0 = fmaf(xf.x * dl[q].x, qs, 12582912.f);
    const float f1 = fmaf(xf.y * dl[q].y, qs, 12582912.f);
    const uint32_t u0 = __float_as_uint(f0), u1 = __float_as_uint(f1);
    uint8_t* row = xq + q * 128;
    *reinterpret_cast<uint16_t*>(row + pos) = (uint16_t)__byte_perm(u0, u1, 0x0040);
    *reinterpret_cast<uint16_t*>(row + 64 + pos) = (uint16_t)__byte_perm(u0, u1, 0x0051);
  }
  __syncwarp();
  uint32_t bl[E_TPW][4], bh[E_TPW][4];
#pragma unroll
  for (int q = 0; q < E_TPW; ++q) {
    uint4 lo4 = make_uint4(0u, 0u, 0u, 0u), hi4 = lo4;
    if (live[q] && gq == 0) {
      lo4 = *reinterpret_cast<const uint4*>(xq + q * 128 + tig * 16);
      hi4 = *reinterpret_cast<const uint4*>(xq + q * 128 + 64 + tig * 16);
    }
    bl[q][0] = lo4.x; bl[q][1] = lo4.y; bl[q][2] = lo4.z; bl[q][3] = lo4.w;
    bh[q][0] = hi4.x; bh[q][1] = hi4.y; bh[q][2] = hi4.z; bh[q][3] = hi4.w;
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < E_TPW; ++q) {
    if (!live[q]) continue;
#pragma unroll
    for (int cch = 0; cch < 2; ++cch) {
      const uint32_t pe[4] = {pw[q][0][2 * cch], pw[q][1][2 * cch], pw[q][2][2 * cch], pw[q][3][2 * cch]};
      const uint32_t po[4] = {pw[q][0][2 * cch + 1], pw[q][1][2 * cch + 1], pw[q][2][2 * cch + 1],
                              pw[q][3][2 * cch + 1]};
#define PMPD_E_MTILE(T)                                                             \
  {                                                                                 \
    uint32_t a0, a1, a2, a3;                                                        \
    nibble_to_u8<4, P, T>(merge_planes<4, P, T>(pe), a0, a1);                       \
    nibble_to_u8<4, P, T>(merge_planes<4, P, T>(po), a2, a3);                       \
    mma_u8s8_16832(dhi[T], a0, a1, a2, a3, bh[q][2 * cch], bh[q][2 * cch + 1]);     \
    mma_u8u8_16832(dlo[T], a0, a1, a2, a3, bl[q][2 * cch], bl[q][2 * cch + 1]);     \
  }
      PMPD_E_MTILE(0)
      PMPD_E_MTILE(1)
      PMPD_E_MTILE(2)
      PMPD_E_MTILE(3)
#undef PMPD_E_MTILE
    }
  }
}

// Only the tile function is specialised per precision (keeps the kernel's code size,
// and so instruction-cache pressure, small).
PMPD_DEV void tile_dispatch(int p, const uint8_t* st, int cnt, int wslot, int kt, int lane, const __half* xs, uint8_t* xq,
                            float qs, int (&dhi)[4][4], int (&dlo)[4][4], float& bias) {
  switch (p) {
    case 4: engine_tile<4>(st, cnt, wslot, kt, lane, xs, xq, qs, dhi, dlo, bias); break;
    case 3: engine_tile<3>(st, cnt, wslot, kt, lane, xs, xq, qs, dhi, dlo, bias); break;
    case 2: engine_tile<2>(st, cnt, wslot, kt, lane, xs, xq, qs, dhi, dlo, bias); break;
    default: engine_tile<1>(st, cnt, wslot, kt, lane, xs, xq, qs, dhi, dlo, bias); break;
  }
}

}  // namespace pmpd
