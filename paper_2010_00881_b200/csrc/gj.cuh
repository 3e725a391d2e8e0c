// gj.cuh -- batched blocked Gauss-Jordan inversion of SPD blocks (setup), shared by the patch
// smoother (patch.cuh) and the multi-level hp solver (hpmg.cu).  Internal linkage: every
// translation unit that includes it gets its own copy.
#pragma once
#include <cstdint>

// ---- setup: symmetric equilibration around the Gauss-Jordan inversion ----------------------
// A = D^-1 S D^-1 with D = diag(1/sqrt(a_ii)) makes S's diagonal 1; then A^-1 = D S^-1 D.  GJ with
// diagonal pivots is backward stable only relative to the UNSCALED condition number; patches
// mixing physical and alpha = 1e-8 fictitious cells are graded by 1e8, so without the scaling
// their individual inverses lost ~1e-6 against LU/Cholesky (which are scaling-invariant).
// phase 0: d_i from the diagonal (identity slots: 1), stored; phase 1: reuse the stored d.
static __global__ void __launch_bounds__(256) k_equil(double* W, int MP, double* dvec, int phase) {
  extern __shared__ double dsh[];
  double* M = W + (int64_t)blockIdx.x * MP * MP;
  double* dv = dvec + (int64_t)blockIdx.x * MP;
  for (int i = threadIdx.x; i < MP; i += blockDim.x) {
    double d;
    if (phase == 0) {
      const double a = M[(int64_t)i * MP + i];
      d = (a > 0.0 && isfinite(a)) ? rsqrt(a) : 1.0;
      dv[i] = d;
    } else {
      d = dv[i];
    }
    dsh[i] = d;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x >> 5; i < MP; i += blockDim.x >> 5) {
    const double di = dsh[i];
    double* row = M + (int64_t)i * MP;
    for (int j = lane; j < MP; j += 32) row[j] *= di * dsh[j];
  }
}

// ---- setup: batched blocked Gauss-Jordan inversion (SPD, no pivoting) -----------------------
// step k: P = A_kk -> P^-1 (in place); A_kj := P^-1 A_kj (j != k); A_ij -= A_ik A_kj (i,j != k);
// A_ik := -A_ik P^-1 (i != k).  A^-1 overwrites A.
static __global__ void __launch_bounds__(256) k_gj_pivot(double* W, int MP, int k, int* status) {
  __shared__ double P[32][33];
  __shared__ double rowt[32], colt[32];
  double* A = W + (int64_t)blockIdx.x * MP * MP + (int64_t)(32 * k) * MP + 32 * k;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) P[e / 32][e % 32] = A[(int64_t)(e / 32) * MP + e % 32];
  __syncthreads();
  // in-place Gauss-Jordan on the 32x32 pivot block (SPD: diagonal pivots, no exchanges)
  for (int t = 0; t < 32; ++t) {
    if (threadIdx.x < 32) rowt[threadIdx.x] = P[t][threadIdx.x];
    else if (threadIdx.x < 64) colt[threadIdx.x - 32] = P[threadIdx.x - 32][t];
    __syncthreads();
    const double piv = rowt[t];
    if (threadIdx.x == 0 && !(piv > 0.0 && isfinite(piv))) status[blockIdx.x] = 1;
    const double ip = 1.0 / piv;
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int i = e / 32, j = e % 32;
      double v;
      if (i == t && j == t) v = ip;
      else if (i == t) v = rowt[j] * ip;
      else if (j == t) v = -colt[i] * ip;
      else v = P[i][j] - colt[i] * rowt[j] * ip;
      P[i][j] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) A[(int64_t)(e / 32) * MP + e % 32] = P[e / 32][e % 32];
}

// A_kj := P^-1 A_kj for column tile j (blockIdx.x), matrix blockIdx.y; skips j == k
static __global__ void __launch_bounds__(256) k_gj_row(double* W, int MP, int k) {
  const int j = blockIdx.x >= (unsigned)k ? blockIdx.x + 1 : blockIdx.x;
  __shared__ double P[32][33], B[32][33];
  double* M = W + (int64_t)blockIdx.y * MP * MP;
  const double* Pg = M + (int64_t)(32 * k) * MP + 32 * k;
  double* Bg = M + (int64_t)(32 * k) * MP + 32 * j;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    P[e / 32][e % 32] = Pg[(int64_t)(e / 32) * MP + e % 32];
    B[e / 32][e % 32] = Bg[(int64_t)(e / 32) * MP + e % 32];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    double s = 0.0;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) s = fma(P[r][t], B[t][c], s);
    Bg[(int64_t)r * MP + c] = s;
  }
}

// A_ik := -A_ik P^-1 for row tile i (blockIdx.x), skips i == k
static __global__ void __launch_bounds__(256) k_gj_col(double* W, int MP, int k) {
  const int i = blockIdx.x >= (unsigned)k ? blockIdx.x + 1 : blockIdx.x;
  __shared__ double P[32][33], B[32][33];
  double* M = W + (int64_t)blockIdx.y * MP * MP;
  const double* Pg = M + (int64_t)(32 * k) * MP + 32 * k;
  double* Bg = M + (int64_t)(32 * i) * MP + 32 * k;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    P[e / 32][e % 32] = Pg[(int64_t)(e / 32) * MP + e % 32];
    B[e / 32][e % 32] = Bg[(int64_t)(e / 32) * MP + e % 32];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    double s = 0.0;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) s = fma(B[r][t], P[t][c], s);
    Bg[(int64_t)r * MP + c] = -s;
  }
}

// trailing update A_ij -= A_ik A_kj over 64x64 output tiles (rows/cols of pivot block k
// skipped): grid (tiles, matrices); 256 threads, 4x4 outputs each, K = 32 staged in smem
static __global__ void __launch_bounds__(256) k_gj_update(double* W, int MP, int k) {
  const int nt64 = (MP + 63) / 64;
  const int ti = blockIdx.x / nt64, tj = blockIdx.x % nt64;
  __shared__ __align__(16) double U[32][64 + 2];   // U[t][r] = A[r0 + r][32k + t]
  __shared__ __align__(16) double V[32][64 + 2];   // V[t][c] = A[32k + t][c0 + c]
  double* M = W + (int64_t)blockIdx.y * MP * MP;
  const int r0 = 64 * ti, c0 = 64 * tj, kk = 32 * k;
  for (int e = threadIdx.x; e < 2048; e += blockDim.x) {
    const int r = e / 32, t = e % 32;   // coalesced along t (row-major source)
    U[t][r] = (r0 + r < MP) ? M[(int64_t)(r0 + r) * MP + kk + t] : 0.0;
    const int t2 = e / 64, c = e % 64;
    V[t2][c] = (c0 + c < MP) ? M[(int64_t)(kk + t2) * MP + c0 + c] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
#pragma unroll 4
  for (int t = 0; t < 32; ++t) {
    double u[4], v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u[i] = U[t][ty * 4 + i];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = V[t][tx * 4 + j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(u[i], v[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= MP || (r >= kk && r < kk + 32)) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c >= MP || (c >= kk && c < kk + 32)) continue;
      M[(int64_t)r * MP + c] -= acc[i][j];
    }
  }
}

