// Cost of gpu-scope release/acquire operations inside a busy SM (TMA stream in the
// background, like the decode engine) vs an idle SM.  Not product code.
#include <cstdio>
#include <cstdint>
#include "../../paper_2410_13461_b200/csrc/pmpd_common.cuh"
using namespace pmpd;

__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

template <int MODE>
__global__ void __launch_bounds__(64, 1) fb(const uint8_t* src, size_t src_bytes, int stream, unsigned* ctr, float* part,
                                           long long* out, int iters) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NS = 6, SB = 24576;
  volatile int* stop = reinterpret_cast<volatile int*>(sm + 1024);
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1); *stop = 0; fence_barrier_init(); }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0 && stream) {
      uint32_t ph = 0; int s = 0; size_t off = (size_t)blockIdx.x * SB;
      for (int it = 0; !*stop; ++it) {
        if (it >= NS) { mbar_wait(&bars[s], ph); }
        mbar_arrive_expect_tx(&bars[s], SB);
        bulk_g2s(sm + 2048 + s * SB, src + off, SB, &bars[s]);
        off += 148 * SB; if (off + SB > src_bytes) off = (size_t)blockIdx.x * SB;
        if (++s == NS) { s = 0; if (it >= NS) ph ^= 1; }
      }
      // drain
    }
    return;
  }
  // warp 0: timed op
  long long tot = 0;
  float* mine = part + blockIdx.x * 64;
  for (int it = 0; it < iters; ++it) {
    mine[lane] = (float)it; mine[lane + 32] = (float)it;
    __syncwarp();
    long long t0 = clk();
    unsigned v = 0;
    if (lane == 0) {
      if (MODE == 0) asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr + blockIdx.x * 32) : "memory");
      if (MODE == 1) asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr + blockIdx.x * 32) : "memory");
      if (MODE == 2) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(ctr + blockIdx.x * 32) : "memory");
      if (MODE == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (MODE == 4) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + blockIdx.x * 32) : "memory");
      if (MODE == 5) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr + blockIdx.x * 32) : "memory");
      if (MODE == 6) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(ctr + blockIdx.x * 32), "r"(it) : "memory"); }
    }
    v = __shfl_sync(0xffffffffu, v, 0);
    long long t1 = clk();
    tot += t1 - t0 + (v == 0xdeadbeef);
    __nanosleep(500);
  }
  if (lane == 0) { out[blockIdx.x] = tot / iters; }
  if (threadIdx.x == 0) *stop = 1;
}

int main() {
  size_t bytes = (size_t)2 << 30;
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  unsigned* ctr; cudaMalloc(&ctr, 148 * 128); cudaMemset(ctr, 0, 148 * 128);
  float* part; cudaMalloc(&part, 148 * 64 * 4);
  long long* out; cudaMalloc(&out, 148 * 8);
  long long h[148];
  const char* names[] = {"atom.relaxed", "atom.release", "red.release", "fence.acq_rel", "ld.acquire", "ld.relaxed", "st.relaxed"};
  auto run = [&](auto kern, int mode, int stream) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 + 6 * 24576);
    kern<<<148, 64, 2048 + 6 * 24576>>>(src, bytes, stream, ctr, part, out, 2000);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    long long s = 0, mx = 0; for (int i = 0; i < 148; ++i) { s += h[i]; mx = h[i] > mx ? h[i] : mx; }
    printf("%-14s stream=%d: mean %6lld cyc  max %6lld  (%s)\n", names[mode], stream, s / 148, mx, cudaGetErrorString(e));
  };
  for (int st = 0; st < 2; ++st) {
    run(fb<0>, 0, st); run(fb<1>, 1, st); run(fb<2>, 2, st); run(fb<3>, 3, st); run(fb<4>, 4, st); run(fb<5>, 5, st); run(fb<6>, 6, st);
  }
  return 0;
}
