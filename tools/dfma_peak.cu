// Microbenchmark: fp64 FMA throughput of the B200 (no tensor cores), for the ALU roofline.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSm : {4, 8}) {
    int nb = sms * blocksPerSm, nt = 256, iters = 20000;
    k<<<nb, nt>>>(d, 100, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<<<nb, nt>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)nb * nt;
    printf("blocks/SM=%d  %.2f TFLOP/s fp64 FMA  (%.3f ms)\n", blocksPerSm, flops / ms / 1e9, ms);
  }
  return 0;
}
