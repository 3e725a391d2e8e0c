// Microbenchmark of the regular-cell operator kernel (cellop.cuh) on the cfg2 fine level
// (32^3 cells, p = 2 tensor, all cells uncut): times kernel variants with CUDA events.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../paper_2010_00881_b200/csrc
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "cellop.cuh"
#include "layout.hpp"

using namespace fcm;

template <int M, int TS>
__global__ void __launch_bounds__(256, 4) k_reg(CellOp op) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* Ms = reinterpret_cast<double*>(smem + sizeof(Tab));
  load_tab(T, op);
  load_shared_matrix<M>(Ms, op);
  __syncthreads();
  const int wpb = blockDim.x >> 5;
  double* xs = Ms + M * padded<M>() + (threadIdx.x >> 5) * reg_scratch<M, TS>();
  reg_cells<M, TS, false>(op, T, Ms, xs, blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb);
}

__global__ void k_copy(double* y, const double* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i];
}
__global__ void k_empty() {}

template <int M, int TS>
void run(const char* name, CellOp op, int ncell, int reps) {
  const int cpb = 8 * (32 / TS);
  int nb = (ncell + cpb - 1) / cpb;
  size_t sm = sizeof(Tab) + ((size_t)M * padded<M>() + 8 * reg_scratch<M, TS>()) * 8;
  cudaFuncSetAttribute(k_reg<M, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) k_reg<M, TS><<<nb, 256, sm>>>(op);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k_reg<M, TS><<<nb, 256, sm>>>(op);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s TS=%d blocks=%5d  %8.2f us/launch  (%s)\n", name, TS, nb, ms * 1e3 / reps,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  Layout L;
  int n[3] = {32, 32, 32};
  L.build(3, n, 2, 0, 1, 0x3f);
  const int q = 2, m = L.m_level[q];
  const LevelTable& t = L.tables[q];
  int64_t nd = t.ndof;
  printf("ncell %lld  m %d  ndof %lld\n", (long long)L.ncell, m, (long long)nd);
  std::vector<double> K(m * m);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b <= a; ++b) K[a * m + b] = K[b * m + a] = 1.0 / (1 + a + b);
  double *dK, *dx, *dy;
  int64_t* dbase;
  int32_t* dstride;
  int16_t *dcmin, *dcmax;
  uint8_t* dkind;
  cudaMalloc(&dK, m * m * 8);
  cudaMalloc(&dx, nd * 8);
  cudaMalloc(&dy, nd * 8);
  cudaMalloc(&dbase, m * 8);
  cudaMalloc(&dstride, m * 12);
  cudaMalloc(&dcmin, m * 6);
  cudaMalloc(&dcmax, m * 6);
  cudaMalloc(&dkind, L.ncell);
  cudaMemcpy(dK, K.data(), m * m * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dbase, t.base.data(), m * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dstride, t.stride.data(), m * 12, cudaMemcpyHostToDevice);
  cudaMemcpy(dcmin, t.cmin.data(), m * 6, cudaMemcpyHostToDevice);
  cudaMemcpy(dcmax, t.cmax.data(), m * 6, cudaMemcpyHostToDevice);
  cudaMemset(dkind, 0, L.ncell);
  cudaMemset(dx, 0, nd * 8);
  cudaMemset(dy, 0, nd * 8);
  CellOp op{};
  op.nx = op.ny = op.nz = 32;
  op.m = m;
  op.ncell = (int)L.ncell;
  op.base = dbase; op.stride = dstride; op.cmin = dcmin; op.cmax = dcmax;
  for (int i = 0; i < 3; ++i) {
    op.ilo[i] = 0; op.ihi[i] = 31;
    for (int a = 0; a < m; ++a) {
      op.ilo[i] = std::max<int>(op.ilo[i], t.cmin[a * 3 + i]);
      op.ihi[i] = std::min<int>(op.ihi[i], t.cmax[a * 3 + i]);
    }
  }
  op.mode = OP_APPLY;
  op.kind = dkind;
  op.Kref = dK;
  op.ldK = m;
  op.alpha = 1e-8;
  op.in = dx;
  op.out = dy;
  op.coef = -1.0;
  const int reps = 200;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty kernel: %.2f us/launch\n", ms * 1e3 / reps);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k_copy<<<592, 256>>>(dy, dx, (int)nd);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy %lld doubles: %.2f us/launch\n", (long long)nd, ms * 1e3 / reps);
  run<27, 1>("reg apply m=27", op, op.ncell, reps);
  run<27, 2>("reg apply m=27", op, op.ncell, reps);
  run<27, 4>("reg apply m=27", op, op.ncell, reps);
  run<27, 8>("reg apply m=27", op, op.ncell, reps);
  return 0;
}
