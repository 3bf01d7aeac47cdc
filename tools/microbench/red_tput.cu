// L2 atomic throughput of red.relaxed.gpu.add.u64: G CTAs x T threads add into W distinct words,
// every word receiving (G*T*R)/W contributions.  Not product code.
#include <cstdio>
#include <cstdint>
__global__ void red_kernel(unsigned long long* w, int W, int R) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int r = 0; r < R; ++r) {
    const int i = (tid * 7 + r * 4099) % W;
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(w + i), "l"(1ull) : "memory");
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* w; cudaMalloc(&w, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int W : {4096, 12288, 65536}) for (int T : {64, 256}) for (int R : {8, 32}) {
    red_kernel<<<sms, T>>>(w, W, R);
    cudaEventRecord(e0);
    red_kernel<<<sms, T>>>(w, W, R);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double n = (double)sms * T * R;
    printf("W=%6d T=%3d R=%2d: %8.0f reds in %7.2f us = %6.1f G reds/s (%5.0f per word) %s\n", W, T, R, n, ms * 1e3,
           n / (ms * 1e-3) / 1e9, n / W, cudaGetErrorString(cudaGetLastError()));
  }
  // empty-kernel baseline
  cudaEventRecord(e0); red_kernel<<<sms, 64>>>(w, 4096, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("empty launch %.2f us\n", ms * 1e3);
  return 0;
}
