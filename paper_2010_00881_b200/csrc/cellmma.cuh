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

// group cell entry: cx | cy << 10 | cz << 20 | inner << 30 | scaled << 31 (inner: no
// Dirichlet DOF in the cell, so no validity test; scaled: the cell's scale is alpha (operator,
// fictitious cell) or 1/alpha (smoother, all-fictitious type) -- carried in the entry so no
// per-cell table lookup sits on the latency path), or -1 for padding; coordinates < 1023
constexpr int kMmaInner = 1 << 30;
constexpr unsigned kMmaScaled = 1u << 31;

struct MmaOp {
  CellOp op;                 // table / vectors / scales (op.mode selects kind vs blk scaling)
  const int32_t* grp_cells;  // [ngroups][8] packed cell coordinates (see kMmaInner), -1 padding
  const int32_t* grp_mat;    // [ngroups] matrix slot: -1 = K_ref leading block, >= 0 type slot
  int64_t ngroups;
  // fused copy cp_dst[0..cp_n) = cp_src (the next residual's "r = b"; cp_dst is not touched by
  // the cell work of this launch), done by every block in a grid-stride loop
  const double* cp_src;
  double* cp_dst;
  int64_t cp_n;
};

// volatile: mma.sync.aligned must stay in warp-converged code (a non-volatile asm may be
// duplicated into divergent branch arms); the callers order independent chains explicitly
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// cell scale: apply -> 1 or alpha (kind), smooth -> 1 or 1/alpha (type flag)
__device__ __forceinline__ double cell_scale(const CellOp& op, int pc) {
  if (pc == -1) return 0.0;
  if (!((unsigned)pc & kMmaScaled)) return 1.0;
  return op.mode == OP_APPLY ? op.alpha : op.inv_alpha;
}

// layout index of local DOF a of the packed cell pc, or -1 (padding / a >= M / Dirichlet)
template <int M>
__device__ __forceinline__ int mma_dof_index(const Tab& T, int a, int pc) {
  if (pc == -1 || a >= M) return -1;
  const int cx = pc & 1023, cy = (pc >> 10) & 1023, cz = (pc >> 20) & 1023;
  if (!(pc & kMmaInner) && !dof_free(T, a, cx, cy, cz)) return -1;
  return dof_index(T, a, cx, cy, cz);
}

// One warp per group of 8 cells (grid-stride over groups, groups sorted by matrix).  The
// block's main matrix (K_ref's leading block for the apply, type slot 0 for the smoother) is
// staged once per block in shared memory in FRAGMENT order (As[(rt*KT + kt)*32 + lane]), so
// every MMA reads its A fragment with one conflict-free LDS.64 and the registers stay few
// (4 blocks per SM); groups of other types read their fragments through L1.
template <int M>
__device__ __forceinline__ void stage_fragments(double* As, const double* K, int ld) {
  constexpr int MT = (M + 7) / 8, KT = (M + 3) / 4;
  for (int t = threadIdx.x; t < MT * KT * 32; t += blockDim.x) {
    const int lane = t & 31, f = t >> 5, rt = f / KT, kt = f % KT;
    const int r = rt * 8 + (lane >> 2), k = kt * 4 + (lane & 3);
    As[t] = (r < M && k < M) ? K[r * ld + k] : 0.0;
  }
}

template <int M, bool FUSE = false, bool PF = false>
__device__ __forceinline__ double mma_cells(const CellOp& op, const int32_t* __restrict__ grp_cells,
                                            const int32_t* __restrict__ grp_mat, int64_t ngroups,
                                            const Tab& T, const double* __restrict__ As,
                                            int main_slot, int warp, int nwarps) {
  constexpr int MT = (M + 7) / 8;   // row tiles
  constexpr int KT = (M + 3) / 4;   // k tiles
  const int lane = threadIdx.x & 31;
  const int ar = lane >> 2, ac = lane & 3;
  double energy = 0.0;
  const bool want_e = op.partials != nullptr;
  // software pipeline: the descriptor of the group two trips ahead and the gathered column of
  // the next group are loaded while this group's MMAs run (the gather latency is hidden)
  int n_slot = 0, n_cg = -1, n_c0 = -1, n_c1 = -1;   // next group
  int m_slot = 0, m_cg = -1, m_c0 = -1, m_c1 = -1;   // the one after
  auto load_desc = [&](int64_t g, int& sl, int& cg, int& c0, int& c1) {
    const int* cells = grp_cells + g * 8;
    sl = __ldg(grp_mat + g);
    cg = __ldg(cells + ar); c0 = __ldg(cells + 2 * ac); c1 = __ldg(cells + 2 * ac + 1);
  };
  double Bn[KT];
  auto gather = [&](int cg) {   // Bn[kt] = x[dof kt*4 + ac] of cell cg
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const int idx = mma_dof_index<M>(T, kt * 4 + ac, cg);
      Bn[kt] = idx >= 0 ? load_in<FUSE>(op, idx) : 0.0;
    }
  };
  // (PF = false, register-tight kernels: only the descriptor runs one trip ahead)
  if (warp < ngroups) load_desc(warp, n_slot, n_cg, n_c0, n_c1);
  if (warp + nwarps < ngroups) load_desc(warp + nwarps, m_slot, m_cg, m_c0, m_c1);
  if (PF) gather(n_cg);
  for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
    const int slot = n_slot;   // warp-uniform
    const int c0 = n_c0, c1 = n_c1;   // output cells
    if (!PF) gather(n_cg);
    double B[KT];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) B[kt] = Bn[kt];
    n_slot = m_slot; n_cg = m_cg; n_c0 = m_c0; n_c1 = m_c1;
    if (gi + 2 * nwarps < ngroups) load_desc(gi + 2 * nwarps, m_slot, m_cg, m_c0, m_c1);
    if (PF && gi + nwarps < ngroups) gather(n_cg);
    const double s0 = op.coef * cell_scale(op, c0), s1 = op.coef * cell_scale(op, c1);
    const bool main = slot == main_slot;
    const double* K = slot < 0 ? op.Kref : op.type_inv + (size_t)slot * M * M;
    const int ld = slot < 0 ? op.ldK : M;
    // row tiles in chunks of RC: k-steps outer, row tiles inner, so consecutive MMAs are
    // independent (RC accumulator pairs) instead of one dependent chain per row tile
    constexpr int RC = (PF && KT > 8) ? (MT < 4 ? MT : 4) : (MT < 8 ? MT : 8);
#pragma unroll
    for (int rb = 0; rb < MT; rb += RC) {
    double D[RC][2];
#pragma unroll
    for (int u = 0; u < RC; ++u) D[u][0] = D[u][1] = 0.0;
    if (main) {
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int u = 0; u < RC; ++u)
          if (rb + u < MT) dmma_8x8x4(D[u][0], D[u][1], As[((rb + u) * KT + kt) * 32 + lane], B[kt], D[u][0], D[u][1]);
    } else {
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int u = 0; u < RC; ++u)
          if (rb + u < MT) {
            const int r = (rb + u) * 8 + ar, k = kt * 4 + ac;
            const double af = (r < M && k < M) ? __ldg(K + r * ld + k) : 0.0;
            dmma_8x8x4(D[u][0], D[u][1], af, B[kt], D[u][0], D[u][1]);
          }
    }
#pragma unroll
    for (int u = 0; u < RC; ++u) {
      const int rt = rb + u;
      if (rt >= MT) break;
      const double d0 = D[u][0], d1 = D[u][1];
      const int a = rt * 8 + ar;
      int i0 = mma_dof_index<M>(T, a, c0), i1 = mma_dof_index<M>(T, a, c1);
      if (op.colour >= 0) {   // deterministic mode: scatter only the cells of this launch's colour
        if (c0 == -1 || cell_colour(c0 & 1023, (c0 >> 10) & 1023, (c0 >> 20) & 1023) != op.colour) i0 = -1;
        if (c1 == -1 || cell_colour(c1 & 1023, (c1 >> 10) & 1023, (c1 >> 20) & 1023) != op.colour) i1 = -1;
      }
      double x0 = 0.0, x1 = 0.0;
      if (want_e) {   // x(a, n) lives in lane n*4 + a%4, fragment B[a/4], a/4 in {2rt, 2rt+1}
        const int src0 = 2 * ac * 4 + (ar & 3), src1 = src0 + 4;
        const double p00 = __shfl_sync(0xffffffffu, B[2 * rt], src0);
        const double p10 = __shfl_sync(0xffffffffu, B[2 * rt], src1);
        double p01 = 0.0, p11 = 0.0;
        if (2 * rt + 1 < KT) {
          p01 = __shfl_sync(0xffffffffu, B[2 * rt + 1], src0);
          p11 = __shfl_sync(0xffffffffu, B[2 * rt + 1], src1);
        }
        x0 = (ar >> 2) ? p01 : p00;
        x1 = (ar >> 2) ? p11 : p10;
      }
      if (i0 >= 0) {
        atomicAdd(op.out + i0, s0 * d0);
        if (want_e) energy = fma(x0, s0 / op.coef * d0, energy);
      }
      if (i1 >= 0) {
        atomicAdd(op.out + i1, s1 * d1);
        if (want_e) energy = fma(x1, s1 / op.coef * d1, energy);
      }
    }
    }
  }
  return energy;
}

}  // namespace fcm
