// Consumer tile-loop microbenchmark (no TMA, no sync): where does the decode
// GEMV's per-tile time go?  Ablations via ABL: 0 full, 1 no MMA, 2 no B prep,
// 3 no plane decode, 4 loads only.  Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2410_13461_b200/csrc/decode_core.cuh"
using namespace pmpd;

template <int P, int ABL, int TPW>
__global__ void __launch_bounds__(512, 1) tile_bench(int iters, int nw, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tig = lane & 3;
  // layout: 16 tiles x (P planes + scales) + x (64*16 halves) + per-warp xq
  for (int i = threadIdx.x; i < 16 * 512 * (P + 1) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) ^ 0x9e3779b9u;
  __half* xs = reinterpret_cast<__half*>(sm + 16 * 512 * (P + 1));
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) xs[i] = __float2half(0.01f * (i % 97) - 0.4f);
  float* scl = reinterpret_cast<float*>(sm + P * 16 * 512);
  for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) scl[i] = 0.001f * (1 + i % 13);
  uint8_t* xq = sm + 16 * 512 * (P + 1) + 2048 + warp * TPW * 128;
  __syncthreads();
  int dhi[4][4] = {}, dlo[4][4] = {};
  float bias = 0.f, qs = 3.f;
  const uint8_t* st = sm;
  for (int it = 0; it < iters; ++it) {
    const int base = (warp * TPW + it) & 15;
    uint32_t pw[TPW][4][4];
    float2 dl[TPW], mn[TPW];
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      const int sl = (base + q * 8) & 15;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < P) {
          const uint4 v = *reinterpret_cast<const uint4*>(st + j * 16 * 512 + sl * 512 + lane * 16);
          pw[q][j][0] = v.x; pw[q][j][1] = v.y; pw[q][j][2] = v.z; pw[q][j][3] = v.w;
        } else {
          pw[q][j][0] = pw[q][j][1] = pw[q][j][2] = pw[q][j][3] = 0u;
        }
      }
      const float* sc = reinterpret_cast<const float*>(st + P * 16 * 512 + sl * 512);
      dl[q] = *reinterpret_cast<const float2*>(sc + 2 * lane);
      mn[q] = *reinterpret_cast<const float2*>(sc + 64 + 2 * lane);
    }
    uint32_t bl[TPW][4], bh[TPW][4];
    if (ABL != 2 && ABL != 4) {
      const int wi = lane >> 1;
      const int pos = (((wi & 3) << 2) | (wi >> 2)) * 4 + 2 * (lane & 1);
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int kk = ((base + q * 8) & 15) * 64 + 2 * lane;
        const float2 xf = __half22float2(*reinterpret_cast<const __half2*>(xs + (kk & 1023)));
        bias = fmaf(xf.x, mn[q].x, fmaf(xf.y, mn[q].y, bias));
        const float f0 = fmaf(xf.x * dl[q].x, qs, 12582912.f);
        const float f1 = fmaf(xf.y * dl[q].y, qs, 12582912.f);
        const uint32_t u0 = __float_as_uint(f0), u1 = __float_as_uint(f1);
        *reinterpret_cast<uint16_t*>(xq + q * 128 + pos) = (uint16_t)__byte_perm(u0, u1, 0x0040);
        *reinterpret_cast<uint16_t*>(xq + q * 128 + 64 + pos) = (uint16_t)__byte_perm(u0, u1, 0x0051);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        uint4 lo4 = make_uint4(0u, 0u, 0u, 0u), hi4 = lo4;
        if (gq == 0) {
          lo4 = *reinterpret_cast<const uint4*>(xq + q * 128 + tig * 16);
          hi4 = *reinterpret_cast<const uint4*>(xq + q * 128 + 64 + tig * 16);
        }
        bl[q][0] = lo4.x; bl[q][1] = lo4.y; bl[q][2] = lo4.z; bl[q][3] = lo4.w;
        bh[q][0] = hi4.x; bh[q][1] = hi4.y; bh[q][2] = hi4.z; bh[q][3] = hi4.w;
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int q = 0; q < TPW; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) { bl[q][i] = 0x01020304u * (i + 1) + it; bh[q][i] = 0x05060708u + i; }
    }
    if (ABL == 4) {
#pragma unroll
      for (int q = 0; q < TPW; ++q) dhi[0][0] ^= pw[q][0][0] ^ pw[q][1][3] ^ bl[q][0];
      continue;
    }
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
#pragma unroll
      for (int cch = 0; cch < 2; ++cch) {
        const uint32_t pe[4] = {pw[q][0][2 * cch], pw[q][1][2 * cch], pw[q][2][2 * cch], pw[q][3][2 * cch]};
        const uint32_t po[4] = {pw[q][0][2 * cch + 1], pw[q][1][2 * cch + 1], pw[q][2][2 * cch + 1], pw[q][3][2 * cch + 1]};
#define MT(T)                                                                       \
  {                                                                                 \
    uint32_t a0, a1, a2, a3;                                                        \
    if (ABL == 3) { a0 = pe[0] + T; a1 = pe[1]; a2 = po[0]; a3 = po[1]; }           \
    else {                                                                          \
      nibble_to_u8<4, P, T>(merge_planes<4, P, T>(pe), a0, a1);                     \
      nibble_to_u8<4, P, T>(merge_planes<4, P, T>(po), a2, a3);                     \
    }                                                                               \
    if (ABL == 1) { dhi[T][0] ^= a0 ^ bh[q][2*cch]; dhi[T][1] ^= a1; dlo[T][0] ^= a2 ^ bl[q][2*cch+1]; dlo[T][1] ^= a3; } \
    else {                                                                          \
      mma_u8s8_16832(dhi[T], a0, a1, a2, a3, bh[q][2 * cch], bh[q][2 * cch + 1]);   \
      mma_u8u8_16832(dlo[T], a0, a1, a2, a3, bl[q][2 * cch], bl[q][2 * cch + 1]);   \
    }                                                                               \
  }
        MT(0) MT(1) MT(2) MT(3)
#undef MT
      }
    }
  }
  unsigned acc = __float_as_uint(bias);
  for (int i = 0; i < 4; ++i) for (int e = 0; e < 4; ++e) acc ^= dhi[i][e] ^ dlo[i][e];
  if (acc == 0x12345) sink[0] = acc;
}

template <int ABL, int TPW>
void run(int nw, int sms) {
  const int P = 2;
  const size_t smem = 16 * 512 * (P + 1) + 2048 + 16 * TPW * 128 + 1024;
  auto k = tile_bench<P, ABL, TPW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned* sink; cudaMalloc(&sink, 64);
  const int iters = 2000;
  k<<<sms, nw * 32, smem>>>(10, nw, sink);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, nw * 32, smem>>>(iters, nw, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double tiles_per_sm = (double)nw * iters * TPW;
  printf("ABL %d TPW %d warps %2d: %6.1f tiles/us/SM   (%s)\n", ABL, TPW, nw, tiles_per_sm / (ms * 1e3),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nw : {8, 16}) {
    run<0, 2>(nw, sms); run<1, 2>(nw, sms); run<2, 2>(nw, sms); run<3, 2>(nw, sms); run<4, 2>(nw, sms);
    run<0, 1>(nw, sms);
  }
  return 0;
}
