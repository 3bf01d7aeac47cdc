// Microbenchmark: legacy mma.sync throughput on sm_100a (HMMA f16, IMMA s8, IMMA s4),
// plus LOP3 throughput. Used to pick the decode-GEMV inner loop. Not product code.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define ITERS 4096

__global__ void k_hmma(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 ^ 0x3c00, a2 = a0 + 7, a3 = a0 * 3;
  uint32_t b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imma8(int* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 ^ 0x35, a2 = a0 + 7, a3 = a0 * 3;
  uint32_t b0 = 0x01010101u, b1 = 0x02020202u;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imma4(int* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 ^ 0x35, a2 = a0 + 7, a3 = a0 * 3;
  uint32_t b0 = 0x11111111u, b1 = 0x22222222u;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lop3(uint32_t* out, int iters) {
  uint32_t x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * (j + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(x[j]), "r"(x[(j + 1) & 7]), "r"(x[(j + 3) & 7]));
      x[j] = r;
    }
  }
  uint32_t s = 0; for (int j = 0; j < 8; ++j) s ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
double run(F f, int blocks, int threads, const char* name, double ops_per_thread_iter, void* buf) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(blocks, threads, buf, 16);  // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f(blocks, threads, buf, ITERS);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double total = (double)blocks * threads / 32.0 * ITERS * ops_per_thread_iter;  // warp-level instrs
  printf("%-8s blocks=%d threads=%d  %.3f ms  %.3e warp-instr/s  err=%s\n", name, blocks, threads, ms,
         total / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
  return total / (ms * 1e-3);
}

int main() {
  int dev = 0; cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d L2=%d clock=%d kHz smemOptin=%zu\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize, clk, pr.sharedMemPerBlockOptin);
  void* buf; cudaMalloc(&buf, 64 << 20);
  int sms = pr.multiProcessorCount;
  for (int tpb : {128, 256, 512}) {
    double h = run([](int b, int t, void* p, int it) { k_hmma<<<b, t>>>((float*)p, it); }, sms * 4, tpb, "hmma", 8, buf);
    printf("   hmma m16n8k16: %.1f TFLOPS dense-equiv\n", h * 4096 * 1e-12);
    double i8 = run([](int b, int t, void* p, int it) { k_imma8<<<b, t>>>((int*)p, it); }, sms * 4, tpb, "imma8", 8, buf);
    printf("   imma m16n8k32: %.1f TOPS\n", i8 * 8192 * 1e-12);
    double i4 = run([](int b, int t, void* p, int it) { k_imma4<<<b, t>>>((int*)p, it); }, sms * 4, tpb, "imma4", 8, buf);
    printf("   imma m16n8k64: %.1f TOPS\n", i4 * 16384 * 1e-12);
    double l = run([](int b, int t, void* p, int it) { k_lop3<<<b, t>>>((uint32_t*)p, it); }, sms * 4, tpb, "lop3", 8, buf);
    printf("   lop3: %.2f lane-op/clk/SM (at %d kHz)\n", l * 32 / (sms * (clk * 1e3)), clk);
  }
  return 0;
}
