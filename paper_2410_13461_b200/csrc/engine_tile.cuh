// Consumer tile body of the persistent decode engine (engine.cu), in a header so that
// tools/microbench/etile_bench.cu measures exactly this code in isolation.
//
// One warp, up to TPW tiles of one n-group per call: decode the P planes of each 64x64 KN tile
// into u8 tensor-core fragments (decode_core.cuh), quantize x*step into an int16 v split into two
// balanced s8 digits v = 256*hi + lo (lo in [-128, 127]), and accumulate ONE mma.sync m16n8k32
// (u8 x s8) per fragment with hi in B column 0 and lo in column 1: lane tig == 0 receives
// sum(a*hi) in d[.][0|2] and sum(a*lo) in d[.][1|3] (rows gq | gq+8).
#pragma once
#include "decode_core.cuh"
#include "layout.cuh"
#include "pmpd_common.cuh"

#ifndef PMPD_ENGINE_NCW
#define PMPD_ENGINE_NCW 12
#endif
#ifndef PMPD_ENGINE_TPW
#define PMPD_ENGINE_TPW 2
#endif
#ifndef PMPD_ENGINE_PREDECODE
#define PMPD_ENGINE_PREDECODE 0  // 1: decode the op's first tile per warp while its input is staged
#endif

namespace pmpd {
constexpr int E_NCW = PMPD_ENGINE_NCW;      // consumer warps
constexpr int E_TPW = PMPD_ENGINE_TPW;      // tiles per consumer warp per stage
constexpr int E_STILES = E_NCW * E_TPW;     // tiles per stage
// |v| bound of the int16 activation: hi = (v + 128) >> 8 must stay inside s8
constexpr float E_QMAX = 32639.f;

// ------------------------------------------------------------------ consumer tile
// A fragments (u8 codes) of tile slot wslot of a stage, decoded ahead (PMPD_ENGINE_PREDECODE):
// fa[cch][T] = {a0, a1, a2, a3} of m-tile T, k-chunk cch
template <int P>
PMPD_DEV void engine_predecode(const uint8_t* st, int wslot, int lane, uint32_t (&fa)[2][4][4]) {
  uint32_t pw[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j < P) {
      const uint4 v = *reinterpret_cast<const uint4*>(st + j * E_STILES * kTilePlaneBytes + wslot * kTilePlaneBytes +
                                                      lane * 16);
      pw[j][0] = v.x;
      pw[j][1] = v.y;
      pw[j][2] = v.z;
      pw[j][3] = v.w;
    } else {
      pw[j][0] = pw[j][1] = pw[j][2] = pw[j][3] = 0u;
    }
  }
#pragma unroll
  for (int cch = 0; cch < 2; ++cch) {
    const uint32_t pe[4] = {pw[0][2 * cch], pw[1][2 * cch], pw[2][2 * cch], pw[3][2 * cch]};
    const uint32_t po[4] = {pw[0][2 * cch + 1], pw[1][2 * cch + 1], pw[2][2 * cch + 1], pw[3][2 * cch + 1]};
#define PMPD_E_PRE(T)                                                                 \
    nibble_to_u8<4, P, T>(merge_planes<4, P, T>(pe), fa[cch][T][0], fa[cch][T][1]); \
    nibble_to_u8<4, P, T>(merge_planes<4, P, T>(po), fa[cch][T][2], fa[cch][T][3]);
    PMPD_E_PRE(0)
    PMPD_E_PRE(1)
    PMPD_E_PRE(2)
    PMPD_E_PRE(3)
#undef PMPD_E_PRE
  }
}

template <int P, bool PRE = false>
PMPD_DEV void engine_tile(const uint8_t* st, int stiles_cnt, int wslot, int kt, int lane, const __half* xs,
                          uint8_t* xq, float qs, int (&d)[4][4], float& bias,
                          const uint32_t (*fa)[4][4] = nullptr) {
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
      if (j < P && live[q] && !(PRE && q == 0)) {
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
    // 1.5 * 2^23 + 128: the low 16 bits of the float are (rint(x*step*qs) + 128) mod 2^16,
    // so byte 1 is the balanced high digit and byte 0 ^ 0x80 the balanced low digit
    const float f0 = fmaf(xf.x * dl[q].x, qs, 12583040.f);
    const float f1 = fmaf(xf.y * dl[q].y, qs, 12583040.f);
    const uint32_t u0 = __float_as_uint(f0), u1 = __float_as_uint(f1);
    uint8_t* row = xq + q * 128;
    *reinterpret_cast<uint16_t*>(row + pos) = (uint16_t)(__byte_perm(u0, u1, 0x0040) ^ 0x8080u);
    *reinterpret_cast<uint16_t*>(row + 64 + pos) = (uint16_t)__byte_perm(u0, u1, 0x0051);
  }
  __syncwarp();
  // B column 0 (lanes gq == 0) = high digits, column 1 (gq == 1) = low digits
  uint32_t bb[E_TPW][4];
#pragma unroll
  for (int q = 0; q < E_TPW; ++q) {
    uint4 b4 = make_uint4(0u, 0u, 0u, 0u);
    if (live[q] && gq < 2) b4 = *reinterpret_cast<const uint4*>(xq + q * 128 + (gq == 0 ? 64 : 0) + tig * 16);
    bb[q][0] = b4.x; bb[q][1] = b4.y; bb[q][2] = b4.z; bb[q][3] = b4.w;
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
    if (PRE && q == 0) {                                                            \
      a0 = fa[cch][T][0]; a1 = fa[cch][T][1]; a2 = fa[cch][T][2]; a3 = fa[cch][T][3]; \
    } else {                                                                        \
      nibble_to_u8<4, P, T>(merge_planes<4, P, T>(pe), a0, a1);                     \
      nibble_to_u8<4, P, T>(merge_planes<4, P, T>(po), a2, a3);                     \
    }                                                                               \
    mma_u8s8_16832(d[T], a0, a1, a2, a3, bb[q][2 * cch], bb[q][2 * cch + 1]);       \
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
                            float qs, int (&d)[4][4], float& bias) {
#ifdef PMPD_ENGINE_ONLY_P
  engine_tile<PMPD_ENGINE_ONLY_P>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias);
  return;
#endif
  switch (p) {
    case 4: engine_tile<4>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias); break;
    case 3: engine_tile<3>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias); break;
    case 2: engine_tile<2>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias); break;
    default: engine_tile<1>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias); break;
  }
}

#if PMPD_ENGINE_PREDECODE
PMPD_DEV void predecode_dispatch(int p, const uint8_t* st, int wslot, int lane, uint32_t (&fa)[2][4][4]) {
  switch (p) {
    case 4: engine_predecode<4>(st, wslot, lane, fa); break;
    case 3: engine_predecode<3>(st, wslot, lane, fa); break;
    case 2: engine_predecode<2>(st, wslot, lane, fa); break;
    default: engine_predecode<1>(st, wslot, lane, fa); break;
  }
}
PMPD_DEV void tile_dispatch_pre(int p, const uint8_t* st, int cnt, int wslot, int kt, int lane, const __half* xs,
                                uint8_t* xq, float qs, int (&d)[4][4], float& bias, const uint32_t (&fa)[2][4][4]) {
  switch (p) {
    case 4: engine_tile<4, true>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias, fa); break;
    case 3: engine_tile<3, true>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias, fa); break;
    case 2: engine_tile<2, true>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias, fa); break;
    default: engine_tile<1, true>(st, cnt, wslot, kt, lane, xs, xq, qs, d, bias, fa); break;
  }
}
#endif

}  // namespace pmpd
