// Throughput of the engine's exact tile body (engine_tile.cuh) in isolation: NW warps per SM,
// each calling tile_dispatch on a resident stage over and over.  Not product code.
#include <cstdio>
#include "../../paper_2410_13461_b200/csrc/engine_tile.cuh"
using namespace pmpd;

__global__ void __launch_bounds__(E_NCW * 32, 1) eb(int p, int iters, int nw, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stage_bytes = E_STILES * 5 * 512;
  for (int i = threadIdx.x; i < stage_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) ^ 0x9e3779b9u;
  float* scl = reinterpret_cast<float*>(sm + p * E_STILES * 512);
  for (int i = threadIdx.x; i < E_STILES * 128; i += blockDim.x) scl[i] = 0.001f * (1 + i % 13);
  __half* xs = reinterpret_cast<__half*>(sm + stage_bytes);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) xs[i] = __float2half(0.01f * (i % 97) - 0.4f);
  uint8_t* xq = sm + stage_bytes + 8192 + (warp % E_NCW) * E_TPW * 128 + (warp / E_NCW) * E_NCW * E_TPW * 128;
  __syncthreads();
  int dacc[4][4] = {};
  float bias = 0.f;
  const int w = warp % E_NCW;
#ifdef ETB_WAIT
  // the engine's per-stage bookkeeping: wait on an (already completed) full barrier, arrive on
  // an empty barrier (count E_NCW, never waited on here)
  __shared__ __align__(8) uint64_t bars[2];
  if (threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], (1 << 20) - 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bars[0]);
  __syncthreads();
#endif
  for (int it = 0; it < iters; ++it) {
#ifdef ETB_WAIT
    mbar_wait(&bars[0], 0);
#endif
    tile_dispatch(p, sm, E_STILES, w, (w + it) & 31, lane, xs, xq, 3.f, dacc, bias);
#ifdef ETB_WAIT
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[1]);
#endif
  }
  unsigned acc = __float_as_uint(bias);
  for (int i = 0; i < 4; ++i) for (int e = 0; e < 4; ++e) acc ^= dacc[i][e];
  if (acc == 0x12345) sink[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink; cudaMalloc(&sink, 64);
  const int smem = E_STILES * 5 * 512 + 8192 + 4 * E_NCW * E_TPW * 128 + 1024;
  cudaFuncSetAttribute(eb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int p : {4, 3, 2}) for (int nw : {E_NCW}) {
    const int iters = 2000;
    eb<<<sms, nw * 32, smem>>>(p, 10, nw, sink);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    eb<<<sms, nw * 32, smem>>>(p, iters, nw, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("p=%d warps %2d: %6.1f tiles/us/SM  (%.0f cycles per call per warp at 1.9GHz) %s\n", p, nw,
           (double)nw * iters * E_TPW / (ms * 1e3), ms * 1e-3 / iters * 1.9e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
