// SM-to-SM hop latency of an LL word (8-byte {payload, epoch}, relaxed st/ld at gpu scope)
// with and without a TMA weight stream on every SM.  Not product code.
#include <cstdio>
#include <cstdint>
#include "../../paper_2410_13461_b200/csrc/pmpd_common.cuh"
using namespace pmpd;

__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ uint64_t ld_rel(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint64_t ld_vol(const uint64_t* p) { uint64_t v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

template <int SLEEP, int VOL>
__global__ void __launch_bounds__(64, 1) pp(const uint8_t* src, size_t src_bytes, int stream, int inflight_stages,
                                           uint64_t* box, long long* out, int iters, int peer) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NS = 8, SB = 24576;
  volatile int* stop = reinterpret_cast<volatile int*>(box + 64);  // global: set by block 0 when done
  if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1); fence_barrier_init(); }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0 && stream) {
      int uses[8] = {0}; int s = 0; size_t off = (size_t)blockIdx.x * SB;
      long long issued = 0;
      while (!*stop) {
        if (uses[s] > 0) mbar_wait(&bars[s], (uses[s] - 1) & 1);
        (void)inflight_stages;
        mbar_arrive_expect_tx(&bars[s], SB);
        bulk_g2s(sm + 2048 + s * SB, src + off, SB, &bars[s]);
        ++uses[s]; ++issued;
        off += 148 * SB; if (off + SB > src_bytes) off = (size_t)blockIdx.x * SB;
        // consume immediately (like a fast consumer): wait for the stage inflight_stages back
        if (issued > inflight_stages) { int o = (int)((issued - 1 - inflight_stages) % NS); (void)o; }
        if (++s == NS) s = 0;
      }
      for (int i = 0; i < NS; ++i) if (uses[i] > 0) mbar_wait(&bars[i], (uses[i] - 1) & 1);
    }
  }
  if (warp == 0 && lane == 0 && (blockIdx.x == 0 || blockIdx.x == peer)) {
    const bool ping = blockIdx.x == 0;
    uint64_t* mine = box + (ping ? 0 : 16);
    uint64_t* theirs = box + (ping ? 16 : 0);
    long long t0 = clk();
    for (int it = 1; it <= iters; ++it) {
      if (ping) {
        st_rel(mine, (uint64_t)it << 32);
        while ((uint32_t)((VOL ? ld_vol(theirs) : ld_rel(theirs)) >> 32) != (uint32_t)it) { if (SLEEP) __nanosleep(SLEEP); }
      } else {
        while ((uint32_t)((VOL ? ld_vol(theirs) : ld_rel(theirs)) >> 32) != (uint32_t)it) { if (SLEEP) __nanosleep(SLEEP); }
        st_rel(mine, (uint64_t)it << 32);
      }
    }
    if (ping) { out[0] = (clk() - t0) / iters; *stop = 1; }
  }
}

int main() {
  size_t bytes = (size_t)2 << 30;
  uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  uint64_t* box; cudaMalloc(&box, 4096);
  long long* out; cudaMalloc(&out, 64);
  auto run = [&](auto kern, const char* name, int stream, int peer) {
    cudaMemset(box, 0, 4096);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 + 8 * 24576);
    kern<<<148, 64, 2048 + 8 * 24576>>>(src, bytes, stream, 8, box, out, 2000, peer);
    cudaError_t e = cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    fflush(stdout);
    printf("%-22s stream=%d peer=%3d: round trip %6lld cyc (one hop ~%lld)  %s\n", name, stream, peer, h, h / 2, cudaGetErrorString(e));
  };
  for (int st = 0; st < 2; ++st)
    for (int peer : {1, 74, 147}) {
      run(pp<0, 0>, "relaxed spin", st, peer);
      run(pp<32, 0>, "relaxed nanosleep32", st, peer);
      run(pp<0, 1>, "volatile spin", st, peer);
    }
  return 0;
}
