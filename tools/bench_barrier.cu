// Grid-barrier microbenchmark (B200): ns per barrier for several implementations, 1 block/SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bench_barrier tools/bench_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Ctl { unsigned count; unsigned pad0[31]; unsigned release; unsigned pad1[31]; double tot[2][4]; };

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old; asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory"); return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0: cg grid sync; 1: counter + last-block release (threadfence version);
// 2: counter RED.release + all poll counter with ld.acquire (one thread per block)
// 3: same as 1 but with atom.release / ld.acquire instead of threadfence
__global__ void kbar(Ctl* ctl, double* part, int iters, int mode, double* out) {
  __shared__ double tot[3];
  unsigned gen = ld_relaxed(&ctl->release);
  unsigned base = ld_relaxed(&ctl->count);
  const unsigned nb = gridDim.x;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    ++gen;
    if (mode == 0) {
      cg::this_grid().sync();
    } else if (mode == 1 || mode == 3) {
      if (threadIdx.x < 32) {
        double* pp = part + (gen & 1) * 3 * nb;
        unsigned old = 0;
        if (threadIdx.x == 0) {
          __stcg(pp + blockIdx.x, 1.0); __stcg(pp + nb + blockIdx.x, 2.0); __stcg(pp + 2 * nb + blockIdx.x, 3.0);
          if (mode == 1) { __threadfence(); old = atomicAdd(&ctl->count, 1u); }
          else old = atom_add_release(&ctl->count, 1u);
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        double* tg = ctl->tot[gen & 1];
        if (old + 1u == base + gen * nb - (gen - 1) * 0 - 0 && false) {}
        if (old + 1u == (gen) * nb) {
          if (mode == 1) __threadfence(); else asm volatile("fence.acq_rel.gpu;" ::: "memory");
          double a0 = 0, a1 = 0, a2 = 0;
          for (int j = threadIdx.x; j < (int)nb; j += 32) { a0 += __ldcg(pp + j); a1 += __ldcg(pp + nb + j); a2 += __ldcg(pp + 2 * nb + j); }
          for (int o = 16; o > 0; o >>= 1) { a0 += __shfl_xor_sync(~0u, a0, o); a1 += __shfl_xor_sync(~0u, a1, o); a2 += __shfl_xor_sync(~0u, a2, o); }
          if (threadIdx.x == 0) {
            __stcg(tg, a0); __stcg(tg + 1, a1); __stcg(tg + 2, a2);
            tot[0] = a0;
            if (mode == 1) { __threadfence(); st_release(&ctl->release, gen); } else st_release(&ctl->release, gen);
          }
        } else if (threadIdx.x == 0) {
          if (mode == 1) { while ((int)(ld_relaxed(&ctl->release) - gen) < 0) {} __threadfence(); }
          else { while ((int)(ld_acquire(&ctl->release) - gen) < 0) {} }
          tot[0] = __ldcg(tg);
        }
      }
      __syncthreads();
      acc += tot[0];
    } else if (mode == 2) {
      if (threadIdx.x == 0) {
        red_add_release(&ctl->count, 1u);
        while ((int)(ld_acquire(&ctl->count) - gen * nb) < 0) {}
      }
      __syncthreads();
    }
  }
  if (mode == 2 && blockIdx.x == 0 && threadIdx.x == 0) ctl->release = gen;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  Ctl* ctl; double* part; double* out;
  cudaMalloc(&ctl, sizeof(Ctl)); cudaMalloc(&part, 6 * 2048 * 8); cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nb : {128, 148}) for (int threads : {128, 512}) for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(ctl, 0, sizeof(Ctl));
    int iters = 1000;
    void* args[] = {&ctl, &part, &iters, &mode, &out};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctl, 0, sizeof(Ctl));
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchCooperativeKernel((void*)kbar, nb, threads, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(err)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("blocks %d threads %d mode %d: %.1f ns/barrier\n", nb, threads, mode, ms * 1e6 / iters);
    }
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
  return 0;
}
