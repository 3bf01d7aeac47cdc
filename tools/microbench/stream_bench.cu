// TMA bulk-copy streaming microbenchmark: how many bytes in flight per SM does
// the producer/consumer ring need to saturate HBM on B200?  Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_13461_b200/csrc/pmpd_common.cuh"
using namespace pmpd;

__global__ void __launch_bounds__(288, 1) stream_kernel(const uint8_t* src, int64_t per_cta, int stage_bytes,
                                                        int nstage, int ncopies, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  uint8_t* ring = sm + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = src + (int64_t)blockIdx.x * per_cta;
  const int nst = (int)(per_cta / stage_bytes);
  if (warp == 8) {
    // ncopies > 0: one lane issues all copies; ncopies < 0: |ncopies| lanes issue one copy each
    const int nc = ncopies > 0 ? ncopies : -ncopies;
    const bool multi = ncopies < 0;
    if (lane < (multi ? nc : 1)) {
      const uint64_t pol = policy_evict_first();
      for (int si = 0; si < nst; ++si) {
        const int slot = si % nstage;
        if (si >= nstage) mbar_wait(&empty[slot], ((si / nstage) & 1) ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], stage_bytes);
        const int cb = stage_bytes / nc;
        for (int c = multi ? lane : 0; c < (multi ? lane + 1 : nc); ++c)
          bulk_g2s_stream(ring + slot * stage_bytes + c * cb, base + (int64_t)si * stage_bytes + c * cb, cb, &full[slot], pol);
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int si = 0; si < nst; ++si) {
    const int slot = si % nstage;
    mbar_wait(&full[slot], (si / nstage) & 1);
    acc += reinterpret_cast<const unsigned*>(ring + slot * stage_bytes)[threadIdx.x];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 0x12345678) sink[0] = acc;
}

__global__ void ldg_kernel(const int4* src, int64_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(src + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x1234567) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t bytes = 1LL << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  unsigned* sink; cudaMalloc(&sink, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  if (argc < 5) {
    for (int it = 0; it < 2; ++it) ldg_kernel<<<sms * 8, 512>>>((const int4*)buf, bytes / 16, (int4*)sink);
    cudaEventRecord(e0); ldg_kernel<<<sms * 8, 512>>>((const int4*)buf, bytes / 16, (int4*)sink); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("LDG.128 read: %.1f GB/s  %s\n", bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  const int g = atoi(argv[1]) * sms, sb = atoi(argv[2]), ns = atoi(argv[3]), nc = atoi(argv[4]);
  const int64_t per = bytes / g / sb * sb;
  const size_t smem = 1024 + (size_t)sb * ns;
  stream_kernel<<<g, 288, smem>>>(buf, per, sb, ns, nc, sink);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("warmup failed: %s\n", cudaGetErrorString(err)); return 1; }
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) stream_kernel<<<g, 288, smem>>>(buf, per, sb, ns, nc, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  err = cudaGetLastError();
  printf("grid %3d stage %6d B x %2d stages (%4d KB in flight/CTA) copies/stage %d: %7.1f GB/s  %s\n", g, sb, ns,
         sb * ns / 1024, nc, 3.0 * per * g / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
  return 0;
}
