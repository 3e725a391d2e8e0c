// Launch-latency microbenchmark: a CUDA graph of N dependent kernels (empty, and a 544-block
// 256-thread kernel touching 2 MB), time per node.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bench_launch tools/bench_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty() {}
__global__ void k_touch(double* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] += 1.0;
}
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* x; int n = 250000; cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
  for (int variant = 0; variant < 3; ++variant) {
    const int N = 200;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) {
      if (variant == 0) k_empty<<<1, 32, 0, s>>>();
      else if (variant == 1) k_empty<<<544, 256, 0, s>>>();
      else k_touch<<<544, 256, 0, s>>>(x, n);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("variant %d (%s): %.2f us per graph node\n", variant,
           variant == 0 ? "empty 1x32" : variant == 1 ? "empty 544x256" : "touch 2MB 544x256", ms * 1e3 / (10 * N));
  }
  return 0;
}
