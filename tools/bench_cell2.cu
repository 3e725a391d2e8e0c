// Microbenchmark of the regular-cell operator kernel (cellop.cuh) on the cfg2 fine level
// (32^3 cells, p = 2 tensor, all cells uncut): times kernel variants with CUDA events.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../paper_2010_00881_b200/csrc
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "cellop.cuh"
#include "layout.hpp"

using namespace fcm;
namespace fcm {
template <int M, int TS, bool FUSE, int KNOB>
__device__ __forceinline__ double reg_cells_k(const CellOp& op, const Tab& T, const double* __restrict__ Ms,
                                            double* xs_warp, int warp, int nwarps) {
  constexpr int RB = rows_of<M, TS>();
  constexpr int MP = padded<M>();
  constexpr int CPW = 32 / TS;
  const int lane = threadIdx.x & 31;
  const int slot = lane / TS;
  const int j = lane % TS;
  const int a_lo = j * RB;
  double* xs = xs_warp + slot * MP;
  const int nx = op.nx, ny = op.ny, ncell = op.ncell;
  const int ilx = op.ilo[0], ihx = op.ihi[0], ily = op.ilo[1], ihy = op.ihi[1];
  const int ilz = op.ilo[2], ihz = op.ihi[2];
  const bool apply = op.mode == OP_APPLY;
  const bool want_e = op.partials != nullptr;
  double* __restrict__ out = op.out;
  const double coef = op.coef;
  double energy = 0.0;
  const int per_round = nwarps * CPW;
  const int rounds = (ncell + per_round - 1) / per_round;
  for (int rnd = 0; rnd < rounds; ++rnd) {
    const int c = (rnd * nwarps + warp) * CPW + slot;
    bool act = c < ncell;
    double scale = 1.0;
    const double* Mg = nullptr;
    if (act) {
      if (apply) {
        const int k = op.kind[c];
        act = k != 2;
        scale = (k == 1) ? op.alpha : 1.0;
      } else {
        const int b = op.blk[c];
        act = b < 0;
        const int t = -b - 1;
        scale = (t >> 12) ? op.inv_alpha : 1.0;
        const int code = t & 0xff;
        if (code != 0) Mg = op.type_inv + code * M * M;
      }
    }
    int cx = 0, cy = 0, cz = 0;
    bool inner = false;
    if (act) {
      cx = c % nx;
      const int cyz = c / nx;
      cy = cyz % ny;
      cz = cyz / ny;
      inner = (cx >= ilx) & (cx <= ihx) & (cy >= ily) & (cy <= ihy) & (cz >= ilz) & (cz <= ihz);
      for (int a = j; a < M; a += TS)
        xs[a] = (KNOB & 1) ? 1.0 : ((inner || dof_free(T, a, cx, cy, cz)) ? load_in<FUSE>(op, dof_index(T, a, cx, cy, cz)) : 0.0);
    }
    __syncwarp();
    if (act) {
    // the gathered vector stays in shared memory (xs[b] is one broadcast word per cell), which
    // keeps the register footprint small enough for 4 resident blocks per SM
    double acc[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) acc[i] = 0.0;
    if ((KNOB & 2)) { acc[0] = xs[a_lo]; } else if (Mg == nullptr) {
#pragma unroll 9
      for (int b = 0; b < M; ++b) {
        const double xb = xs[b];
#pragma unroll
        for (int i = 0; i < RB; i += 2) {
          if (TS == 1 ? (i < M) : (a_lo + i < M)) {
            const double2 v = *reinterpret_cast<const double2*>(Ms + b * MP + a_lo + i);
            acc[i] = fma(v.x, xb, acc[i]);
            acc[i + 1] = fma(v.y, xb, acc[i + 1]);   // pad row (a = M) reads 0
          }
        }
      }
    } else {
#pragma unroll 9
      for (int b = 0; b < M; ++b) {
        const double xb = xs[b];
#pragma unroll
        for (int i = 0; i < RB; ++i)
          if (a_lo + i < M) acc[i] = fma(__ldg(Mg + (a_lo + i) * M + b), xb, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int a = a_lo + i;
      if (TS == 1 ? (i < M) : (a < M)) {
        if (inner || dof_free(T, a, cx, cy, cz)) {
          const int ia = dof_index(T, a, cx, cy, cz);
          const double y = scale * acc[i];
#if 1
          if (KNOB & 4) out[ia] = coef * y; else atomicAdd(out + ia, coef * y);
#elif defined(FCM_DEBUG_NORED)
          out[ia] = coef * y;   // timing experiment only (wrong result)
#else
          atomicAdd(out + ia, coef * y);
#endif
          if (want_e) energy = fma(xs[a], y, energy);
        }
      }
    }
    }  // act
    __syncwarp();
  }
  return energy;
}

}

template <int M, int TS, int KNOB>
__global__ void __launch_bounds__(256, 4) k_reg(CellOp op) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* Ms = reinterpret_cast<double*>(smem + sizeof(Tab));
  load_tab(T, op);
  load_shared_matrix<M>(Ms, op);
  __syncthreads();
  const int wpb = blockDim.x >> 5;
  double* xs = Ms + M * padded<M>() + (threadIdx.x >> 5) * reg_scratch<M, TS>();
  reg_cells_k<M, TS, false, KNOB>(op, T, Ms, xs, blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb);
}

__global__ void k_copy(double* y, const double* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i];
}
__global__ void k_empty() {}

template <int M, int TS, int KNOB = 0>
void run(const char* name, CellOp op, int ncell, int reps) {
  const int cpb = 8 * (32 / TS);
  int nb = (ncell + cpb - 1) / cpb;
  size_t sm = sizeof(Tab) + ((size_t)M * padded<M>() + 8 * reg_scratch<M, TS>()) * 8;
  cudaFuncSetAttribute(k_reg<M, TS, KNOB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) k_reg<M, TS, KNOB><<<nb, 256, sm>>>(op);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k_reg<M, TS, KNOB><<<nb, 256, sm>>>(op);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-22s knob=%d TS=%d blocks=%5d  %8.2f us/launch  (%s)\n", name, KNOB, TS, nb, ms * 1e3 / reps,
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
  for (int rep = 0; rep < 1; ++rep) {
  run<27, 2, 0>("reg apply m=27", op, op.ncell, reps);
  run<27, 2, 1>("reg no-gather", op, op.ncell, reps);
  run<27, 2, 2>("reg no-compute", op, op.ncell, reps);
  run<27, 2, 4>("reg store-not-red", op, op.ncell, reps);
  run<27, 2, 7>("reg nothing", op, op.ncell, reps);
  run<27, 8, 0>("reg apply m=27", op, op.ncell, reps);
  run<27, 8, 1>("reg no-gather", op, op.ncell, reps);
  run<27, 8, 2>("reg no-compute", op, op.ncell, reps);
  run<27, 8, 4>("reg store-not-red", op, op.ncell, reps);
  run<27, 8, 7>("reg nothing", op, op.ncell, reps);
  }
  return 0;
}
