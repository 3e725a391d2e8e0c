// cellmma.cuh -- the regular-cell population of the operator apply (PAPER.md:163/169,
// r = b - A_q x) and of the additive-Schwarz smoother (Eq. AdditiveSchwarz) as
// what it is: a batched dense contraction Y = K [x_c1 ... x_c8] with ONE shared matrix K (the
// leading block of K_ref, or the shared Schwarz inverse of a boundary type) per group of 8
// cells.  fp64 tensor-core MMA (mma.sync m8n8k4 f64; tcgen05 has no fp64 kind): the K tiles
// live in registers for the whole kernel (one load per warp per matrix change), each group of
// 8 cells costs 8 gathers, ceil(M/8) x ceil(M/4) MMAs and 2 ceil(M/8) scatter-adds per lane.
// Fragment layouts (PTX ISA, m8n8k4 .f64): A 8x4 row: lane holds A[lane/4][lane%4];
// B 4x8 col: B[lane%4][lane/4]; C/D 8x8: D[lane/4][2*(lane%4) + {0,1}].
#pragma once
#include <cstdint>

#include "cellop.cuh"

namespace fcm {

struct MmaOp {
  CellOp op;                 // table / vectors / scales (op.mode selects kind vs blk scaling)
  const int32_t* grp_cells;  // [ngroups][8] cell indices (-1 padding)
  const int32_t* grp_mat;    // [ngroups] matrix slot: -1 = K_ref leading block, >= 0 type slot
  int64_t ngroups;
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// cell scale: apply -> 1 or alpha (kind), smooth -> 1 or 1/alpha (type flag)
__device__ __forceinline__ double cell_scale(const CellOp& op, int c) {
  if (c < 0) return 0.0;
  if (op.mode == OP_APPLY) return op.kind[c] == 1 ? op.alpha : 1.0;
  const int t = -op.blk[c] - 1;
  return (t >> 12) ? op.inv_alpha : 1.0;
}

template <int M>
__device__ __forceinline__ int mma_dof_index(const Tab& T, int a, int c, const CellOp& op) {
  if (c < 0 || a >= M) return -1;
  const int cx = c % op.nx, cyz = c / op.nx, cy = cyz % op.ny, cz = cyz / op.ny;
  if (!dof_free(T, a, cx, cy, cz)) return -1;
  return dof_index(T, a, cx, cy, cz);
}

// One warp per group of 8 cells (grid-stride over groups, groups sorted by matrix).
template <int M>
__device__ __forceinline__ double mma_cells(const MmaOp& g, const Tab& T, int warp, int nwarps) {
  constexpr int MT = (M + 7) / 8;   // row tiles
  constexpr int KT = (M + 3) / 4;   // k tiles
  const CellOp& op = g.op;
  const int lane = threadIdx.x & 31;
  const int ar = lane >> 2, ac = lane & 3;
  double A[MT][KT];
  int cur = -2;   // matrix slot held in A
  double energy = 0.0;
  const bool want_e = op.partials != nullptr;
  for (int64_t gi = warp; gi < g.ngroups; gi += nwarps) {
    const int slot = __ldg(g.grp_mat + gi);   // warp-uniform
    if (slot != cur) {
      const double* K = slot < 0 ? op.Kref : op.type_inv + (size_t)slot * M * M;
      const int ld = slot < 0 ? op.ldK : M;
#pragma unroll
      for (int rt = 0; rt < MT; ++rt)
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int r = rt * 8 + ar, k = kt * 4 + ac;
          A[rt][kt] = (r < M && k < M) ? __ldg(K + r * ld + k) : 0.0;
        }
      cur = slot;
    }
    const int* cells = g.grp_cells + gi * 8;
    const int cg = __ldg(cells + ar);            // B column / gather cell of this lane
    // gather: B[kt] = x[dof kt*4 + ac] of cell cg
    double B[KT];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int idx = mma_dof_index<M>(T, kt * 4 + ac, cg, op);
      B[kt] = idx >= 0 ? __ldg(op.in + idx) : 0.0;
    }
    const int c0 = __ldg(cells + 2 * ac), c1 = __ldg(cells + 2 * ac + 1);   // output cells
    const double s0 = op.coef * cell_scale(op, c0), s1 = op.coef * cell_scale(op, c1);
#pragma unroll
    for (int rt = 0; rt < MT; ++rt) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) dmma_8x8x4(d0, d1, A[rt][kt], B[kt], d0, d1);
      const int a = rt * 8 + ar;
      const int i0 = mma_dof_index<M>(T, a, c0, op), i1 = mma_dof_index<M>(T, a, c1, op);
      if (i0 >= 0) {
        atomicAdd(op.out + i0, s0 * d0);
        if (want_e) energy = fma(__ldg(op.in + i0), s0 / op.coef * d0, energy);
      }
      if (i1 >= 0) {
        atomicAdd(op.out + i1, s1 * d1);
        if (want_e) energy = fma(__ldg(op.in + i1), s1 / op.coef * d1, energy);
      }
    }
  }
  return energy;
}

}  // namespace fcm
