// coarse.cuh -- the coarsest level (p = 1, PAPER.md:226-228 Remark) solved by CG with the
// undamped elementwise additive-Schwarz preconditioner ("parallel CG solver and
// the additive Schwarz preconditioner"), reading R4: x0 = 0, stop at ||r|| < rtol ||r0||.
//
// The whole inner PCG runs in ONE cooperative launch.  It is the standard PCG recurrence
//   z_k = M r_k, beta_k = rz_k/rz_{k-1}, p_k = z_k + beta_k p_{k-1}, q_k = A p_k,
//   alpha_k = rz_k/(p_k.q_k), x += alpha_k p_k, r_{k+1} = r_k - alpha_k q_k,
// reorganised so that each iteration needs only TWO grid-wide barriers:
//   * q_k = A z_k + beta_k q_{k-1}      (w_k = A z_k is the only operator apply)
//   * p_k.q_k = z.Az + 2 beta z.q_{k-1} + beta^2 p_{k-1}.q_{k-1}   (A symmetric)
//   * z.Az and r.Mr are per-cell / per-block energies computed inside the scatter kernels
//   * r_{k+1} is formed on the fly inside the smoother's gather (r - alpha (w + beta q)),
//     so the vector update and the smoother share one phase.
// Phase S: q = w + beta q_old; x += alpha p; r' = r - alpha q; rr; z' += M r' (energy rz')
// Phase A: test rr; beta' = rz'/rz; w' += A z' (energy zAz); p = z' + beta' p; z'.q
// Vectors r, z, w, q are double-buffered (written in a phase while their previous value is
// gathered by other cells in the same phase).  The convergence test reads rr one phase late;
// the z computed speculatively in that phase is discarded (iteration count unchanged).
//
// Barriers: a sense-counting grid barrier in global memory that also REDUCES the two block
// partials of the phase: the last block to arrive sums them in block order (deterministic)
// and publishes the totals, so no block re-reads all partials.
#pragma once
#include <cooperative_groups.h>

#include "cellmma.cuh"
#include "cellop.cuh"

namespace fcm {

constexpr int kCtlFlags = 2048;   // >= co-resident blocks
struct GridCtl {          // zero-initialised device memory
  unsigned int release;   // generation released by the master block
  unsigned int pad[31];
  double tot[2];
  double pad2[14];
  unsigned int flags[kCtlFlags];  // per-block arrival generation (no same-address atomics)
};

struct CoarseArgs {
  CellOp A;                    // apply template (in/out set per phase)
  CellOp M;                    // AS smoother template (coef 1)
  int jacobi;                  // 1: z = D^{-1} r instead of the AS smoother
  const double* diag_inv;
  const double* b;
  double* x;
  double* r[2];
  double* z[2];
  double* w[2];
  double* q[2];
  double* p;
  int64_t n;
  double rtol2;
  int maxit;
  double* part;                // 2 * part_stride block partials
  int part_stride;
  GridCtl* ctl;
  int* iters;                  // [0] = this solve, [1] += this solve
  int nbl_A, nbl_M;            // blocks assigned to the individual lists of A / M
  // regular cells as fp64 MMA groups (cellmma.cuh); null: thread-per-cell path (reg_cells)
  const int32_t* gA_cells;
  const int32_t* gA_mat;
  int64_t nA;
  const int32_t* gS_cells;
  const int32_t* gS_mat;
  int64_t nS;
  // large levels: r_{k+1} is written by the vector loop and the smoother reads it after one
  // more grid barrier (one gather instead of the three of the fused form)
  int split_s;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid-wide barrier + deterministic all-reduce of two doubles (one partial per block).
// Every block publishes its partials and its arrival generation `gen` in its own flag word;
// block 0 polls all flags in parallel, sums the partials in block order, and releases.
// Must be called by every thread of every (co-resident) block with the same gen.
__device__ __forceinline__ double sum_blk_partials(const double* p, int n, double* bc) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) s += __ldcg(p + i);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *bc = s;
  }
  __syncthreads();
  return *bc;
}

// Default barrier: cooperative-groups grid sync (measured faster than the flag barrier below
// on B200 for 148-296 blocks); partial pairs alternate with the generation parity so a slow
// block can still read pair g while fast blocks write pair g+1.
__device__ __noinline__ void barrier_reduce2_cg(double va, double vb, double* part, int stride,
                                                unsigned gen, double* red, double& ta, double& tb) {
  __shared__ double s_tot[2];
  double* pa = part + (gen & 1) * 2 * stride;
  double* pb = pa + stride;
  va = block_sum(va, red);
  vb = block_sum(vb, red);
  if (threadIdx.x == 0) {
    pa[blockIdx.x] = va;
    pb[blockIdx.x] = vb;
  }
  cooperative_groups::this_grid().sync();
  ta = sum_blk_partials(pa, gridDim.x, &s_tot[0]);
  tb = sum_blk_partials(pb, gridDim.x, &s_tot[1]);
  __syncthreads();
}

// One cell phase: blocks [0, nbl) stream the individual list (group per cell), the other blocks
// run the regular population (thread(s) per cell) concurrently.  M == 0: all blocks generic;
// nbl == 0: every block does both populations.
template <int M, int G, bool FUSE>
__device__ __forceinline__ double coarse_cells(const CellOp& op, const Tab& T, const double* Ms,
                                               double* xsr, double* xs, int* ids, int nbl,
                                               const int32_t* gcells = nullptr, const int32_t* gmat = nullptr,
                                               int64_t ngroups = 0, const double* As = nullptr,
                                               int main_slot = 0) {
  const int wpb = blockDim.x >> 5;
  const int wib = threadIdx.x >> 5;
  if constexpr (M > 0 && M <= 32) {
    if (gcells) {   // MMA groups and the individual list, both grid-strided over every warp
      const int gw = blockIdx.x * wpb + wib, nw = gridDim.x * wpb;
      const double e = mma_cells<M, FUSE>(op, gcells, gmat, ngroups, T, As, main_slot, gw, nw);
      return e + list_cells<G, FUSE, (M > 0 && M <= 32 ? M : 0)>(op, T, gw, nw, xs, ids);
    }
  }
  if (M > 0 && nbl == 0) {
    double e = 0.0;
    if constexpr (M > 0)
      e = reg_cells<M, split_of<M>(), FUSE>(op, T, Ms, xsr, blockIdx.x * wpb + wib, gridDim.x * wpb);
    return e + list_cells<G, FUSE, (M > 0 && M <= 32 ? M : 0)>(op, T, blockIdx.x * wpb + wib, gridDim.x * wpb, xs, ids);
  }
  if (M == 0 || (int)blockIdx.x < nbl) {
    const int nb = M == 0 ? gridDim.x : nbl;
    return list_cells<G, FUSE, (M > 0 && M <= 32 ? M : 0)>(op, T, blockIdx.x * wpb + wib, nb * wpb, xs, ids);
  }
  if constexpr (M > 0)
    return reg_cells<M, split_of<M>(), FUSE>(op, T, Ms, xsr, (blockIdx.x - nbl) * wpb + wib,
                                             (gridDim.x - nbl) * wpb);
  return 0.0;
}

// smem: [Tab][MsA: M*MP][MsM: M*MP][reg scratch][list xs][list ids]
template <int M, int G>
__global__ void __launch_bounds__(256, (M > 0 && M <= 8) ? 4 : ((M > 0 && M <= 32) ? 3 : 2)) k_coarse_pcg(CoarseArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CPW = 32 / G;
  constexpr int MP = M > 0 ? padded<M>() : 0;
  const int wpb = blockDim.x >> 5;
  const int m = a.A.m;
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* MsA = reinterpret_cast<double*>(smem + sizeof(Tab));
  double* MsM = MsA + M * MP;
  constexpr int RS = M > 0 ? reg_scratch<(M > 0 ? M : 1), split_of<(M > 0 ? M : 1)>()>() : 0;
  double* xsr = MsM + M * MP + (threadIdx.x >> 5) * RS;
  double* xs0 = MsM + M * MP + wpb * RS;
  double* xs = xs0 + (threadIdx.x >> 5) * CPW * m;
  int* ids = reinterpret_cast<int*>(xs0 + wpb * CPW * m) + (threadIdx.x >> 5) * CPW * m;
  __shared__ double red[32];
  constexpr int FR = (M > 0 && M <= 32) ? ((M + 7) / 8) * ((M + 3) / 4) * 32 : 0;   // fragment doubles
  int* ids_end = reinterpret_cast<int*>(xs0 + wpb * CPW * m) + wpb * CPW * m;
  double* AsA = reinterpret_cast<double*>(ids_end + ((wpb * CPW * m) & 1));   // 8-byte aligned
  double* AsM = AsA + FR;
  load_tab(T, a.A);
  if constexpr (M > 0) {
    load_shared_matrix<M>(MsA, a.A);
    if (!a.jacobi) load_shared_matrix<M>(MsM, a.M);
  }
  if constexpr (M > 0 && M <= 32) {
    if (a.gA_cells) stage_fragments<M>(AsA, a.A.Kref, a.A.ldK);
    if (a.gS_cells && !a.jacobi) stage_fragments<M>(AsM, a.M.type_inv, M);
  }
  __syncthreads();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = a.n;
  // barrier generations continue from the previous launch's last release (no barrier of this
  // launch can complete before every block has read it)
  unsigned gen = ld_acquire_u32(&a.ctl->release);
  CellOp opA = a.A, opM = a.M;
  opA.partials = a.part;   // non-null: the cell paths accumulate energies
  opM.partials = a.part;

  // ---- start: x = 0, r = b, z = M r (rz), w = A z (zAz), p = z, q_old = 0 ---------------
  int cur = 0;  // index of the current r/z/w buffers; q_old = q[qc]
  int qc = 0;
  double s1 = 0.0, s2 = 0.0, t1, t2;
  for (int64_t i = tid; i < n; i += nth) {
    const double bi = a.b[i];
    a.x[i] = 0.0; a.r[0][i] = bi;
    a.z[0][i] = 0.0; a.z[1][i] = 0.0; a.w[0][i] = 0.0; a.w[1][i] = 0.0; a.q[0][i] = 0.0;
    s1 = fma(bi, bi, s1);
  }
  barrier_reduce2_cg(s1, 0.0, a.part, a.part_stride, ++gen, red, t1, t2);
  const double rr0 = t1;
  int it = 0;
  if (rr0 > 0.0) {
    // z0 = M r0
    if (a.jacobi) {
      s2 = 0.0;
      for (int64_t i = tid; i < n; i += nth) {
        const double zi = a.diag_inv[i] * a.r[0][i];
        a.z[0][i] = zi;
        s2 = fma(zi, a.r[0][i], s2);
      }
    } else {
      opM.in = a.r[0]; opM.in1 = nullptr; opM.out = a.z[0];
      s2 = coarse_cells<M, G, false>(opM, T, MsM, xsr, xs, ids, a.nbl_M, a.gS_cells, a.gS_mat, a.nS, AsM, 0);
    }
    barrier_reduce2_cg(s2, 0.0, a.part, a.part_stride, ++gen, red, t1, t2);
    double rz = t1;
    // w0 = A z0 ; p = z0
    opA.in = a.z[0]; opA.in1 = nullptr; opA.out = a.w[0];
    s1 = coarse_cells<M, G, false>(opA, T, MsA, xsr, xs, ids, a.nbl_A, a.gA_cells, a.gA_mat, a.nA, AsA, -1);
    for (int64_t i = tid; i < n; i += nth) a.p[i] = a.z[0][i];
    barrier_reduce2_cg(s1, 0.0, a.part, a.part_stride, ++gen, red, t1, t2);
    double pq = t1;
    double alpha = rz / pq;
    double beta = 0.0;
    while (true) {
      // ---- phase S ----------------------------------------------------------------------
      const int nx = cur ^ 1;
      double* rC = a.r[cur];
      double* rN = a.r[nx];
      double* wC = a.w[cur];
      const double* qO = a.q[qc];
      double* qN = a.q[qc ^ 1];
      double rr_loc = 0.0, rz_loc = 0.0;
      for (int64_t i = tid; i < n; i += nth) {
        const double qi = fma(beta, qO[i], wC[i]);
        qN[i] = qi;
        a.x[i] = fma(alpha, a.p[i], a.x[i]);
        const double ri = fma(-alpha, qi, rC[i]);
        rN[i] = ri;
        rr_loc = fma(ri, ri, rr_loc);
        a.w[nx][i] = 0.0;
        if (a.jacobi) {
          const double zi = a.diag_inv[i] * ri;
          a.z[nx][i] = zi;
          rz_loc = fma(zi, ri, rz_loc);
        }
      }
      if (!a.jacobi) {
        if (a.split_s) {   // r_{k+1} complete in memory first
          cooperative_groups::this_grid().sync();
          opM.in = rN; opM.in1 = nullptr;
          opM.out = a.z[nx];
          rz_loc = coarse_cells<M, G, false>(opM, T, MsM, xsr, xs, ids, a.nbl_M, a.gS_cells, a.gS_mat, a.nS, AsM, 0);
        } else {
          opM.in = rC; opM.in1 = wC; opM.in2 = qO; opM.c1 = -alpha; opM.c2 = beta;
          opM.out = a.z[nx];
          rz_loc = coarse_cells<M, G, true>(opM, T, MsM, xsr, xs, ids, a.nbl_M, a.gS_cells, a.gS_mat, a.nS, AsM, 0);
        }
      }
      double rr, rz_new;
      barrier_reduce2_cg(rr_loc, rz_loc, a.part, a.part_stride, ++gen, red, rr, rz_new);
      // ---- phase A ----------------------------------------------------------------------
      ++it;
      if (!(pq > 0.0) || rr < a.rtol2 * rr0 || it >= a.maxit) break;
      const double beta_n = rz_new / rz;
      rz = rz_new;
      double* zN = a.z[nx];
      opA.in = zN; opA.in1 = nullptr; opA.out = a.w[nx];
      const double zaz = coarse_cells<M, G, false>(opA, T, MsA, xsr, xs, ids, a.nbl_A, a.gA_cells, a.gA_mat, a.nA, AsA, -1);
      double zq = 0.0;
      for (int64_t i = tid; i < n; i += nth) {
        const double zi = zN[i];
        a.p[i] = fma(beta_n, a.p[i], zi);
        zq = fma(zi, qN[i], zq);
        a.z[cur][i] = 0.0;
      }
      double zAz, zqs;
      barrier_reduce2_cg(zaz, zq, a.part, a.part_stride, ++gen, red, zAz, zqs);
      pq = zAz + beta_n * (2.0 * zqs + beta_n * pq);
      alpha = rz / pq;
      beta = beta_n;
      cur = nx;
      qc ^= 1;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { a.iters[0] = it; a.iters[1] += it; }
}

}  // namespace fcm
