// cellop.cuh -- the element-by-element "gather -> small dense GEMV -> scatter-add" primitive
// shared by the level operator apply (PAPER.md:163/169 r = b - A_l x; A_{l-1} = R A_l R^T,
// P:118, realised as leading element blocks) and the additive-Schwarz smoother
// (Eq. AdditiveSchwarz: x += omega sum_i P_i A_i^{-1} P_i^T r).
//
// Two populations of cells, two mappings:
//  * regular cells (uncut for the operator; shared-by-type blocks for the smoother) -- one
//    THREAD per cell: the m gathered values live in registers (compile-time M, full unroll),
//    the shared matrix (K_ref or the interior-type inverse) is broadcast from shared memory
//    (every lane reads the same word), other boundary types read through L1.  32 lanes =
//    32 consecutive cells along x, so every gather / scatter instruction is coalesced.
//  * individual cells (cut cells / irregular blocks) -- one GROUP of G lanes per cell over a
//    compact list; lane a owns rows a, a+G, ...; the individual matrix is streamed column-wise
//    (Mat[b*ld + a], symmetric) so the G lanes read consecutive addresses.
// The scatter is a fp64 red.global.add into the output vector.
#pragma once
#include <cstdint>

namespace fcm {

constexpr int kMaxM = 128;  // largest element block handled by the cell kernels

enum { OP_APPLY = 0, OP_SMOOTH = 1 };

struct Tab {  // level table in shared memory; stride along x is 1 for every DOF class
  int32_t base[kMaxM];
  int32_t sy[kMaxM];
  int32_t sz[kMaxM];
  int16_t cmin[kMaxM][3];
  int16_t cmax[kMaxM][3];
};

struct CellOp {
  int nx, ny, nz;
  int m;                      // level element DOFs m_q
  int32_t ncell;
  const int64_t* base;
  const int32_t* stride;
  const int16_t* cmin;
  const int16_t* cmax;
  int mode;                   // OP_APPLY / OP_SMOOTH
  // APPLY (regular): K_ref (kind 0) or alpha K_ref (kind 1); kind 2 cells are in the list
  const uint8_t* kind;
  const double* Kref;
  int ldK;
  double alpha;
  // SMOOTH (regular): blk < 0: t = -blk-1, type_inv[t & 0xff] * (t >> 12 ? 1/alpha : 1);
  //                   blk >= 0 cells are in the list
  const int32_t* blk;
  const double* type_inv;
  double inv_alpha;
  // individual cells: list[i] = cell, list_mats + i*list_ld^2 = its matrix (leading m block)
  const int32_t* list;
  int32_t nlist;
  const double* list_mats;
  int list_ld;
  // generic fallback (no compile-time M): per-cell selection over all cells
  const int32_t* cut_idx;
  const double* cutK;
  const double* irr_inv;
  // data: out[idx] += coef * scale * Mat * in_local
  const double* in;
  double* out;
  double coef;
  double* partials;           // optional per-block sum of in_local^T (scale Mat in_local)
};

__device__ __forceinline__ void load_tab(Tab& T, const CellOp& op) {
  for (int a = threadIdx.x; a < op.m; a += blockDim.x) {
    T.base[a] = (int32_t)op.base[a];
    T.sy[a] = op.stride[a * 3 + 1];
    T.sz[a] = op.stride[a * 3 + 2];
    for (int i = 0; i < 3; ++i) {
      T.cmin[a][i] = op.cmin[a * 3 + i];
      T.cmax[a][i] = op.cmax[a * 3 + i];
    }
  }
}

// shared matrix of the regular path (row-major M x M): K_ref leading block or interior inverse
template <int M>
__device__ __forceinline__ void load_shared_matrix(double* Ms, const CellOp& op) {
  if (op.mode == OP_APPLY) {
    for (int e = threadIdx.x; e < M * M; e += blockDim.x) Ms[e] = op.Kref[(e / M) * op.ldK + e % M];
  } else {
    for (int e = threadIdx.x; e < M * M; e += blockDim.x) Ms[e] = op.type_inv[e];  // type code 0
  }
}

template <int M>
__device__ __forceinline__ double reg_cells(const CellOp& op, const Tab& T, const double* __restrict__ Ms,
                                            int t0, int nth) {
  double energy = 0.0;
  for (int c = t0; c < op.ncell; c += nth) {
    double scale = 1.0;
    const double* Mg = nullptr;
    if (op.mode == OP_APPLY) {
      const int k = op.kind[c];
      if (k == 2) continue;
      scale = (k == 1) ? op.alpha : 1.0;
    } else {
      const int b = op.blk[c];
      if (b >= 0) continue;
      const int t = -b - 1;
      scale = (t >> 12) ? op.inv_alpha : 1.0;
      const int code = t & 0xff;
      if (code != 0) Mg = op.type_inv + code * M * M;
    }
    const int cx = c % op.nx;
    const int cyz = c / op.nx;
    const int cy = cyz % op.ny;
    const int cz = cyz / op.ny;
    double x[M];
    int idx[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      const bool ok = (cx >= T.cmin[a][0]) & (cx <= T.cmax[a][0]) & (cy >= T.cmin[a][1]) &
                      (cy <= T.cmax[a][1]) & (cz >= T.cmin[a][2]) & (cz <= T.cmax[a][2]);
      const int i = T.base[a] + cx + cy * T.sy[a] + cz * T.sz[a];
      idx[a] = ok ? i : -1;
      x[a] = ok ? __ldg(op.in + i) : 0.0;
    }
    if (Mg == nullptr) {
#pragma unroll
      for (int a = 0; a < M; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) acc = fma(Ms[a * M + b], x[b], acc);
        const double y = scale * acc;
        if (idx[a] >= 0) atomicAdd(op.out + idx[a], op.coef * y);
        energy = fma(x[a], y, energy);
      }
    } else {
#pragma unroll
      for (int a = 0; a < M; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) acc = fma(__ldg(Mg + a * M + b), x[b], acc);
        const double y = scale * acc;
        if (idx[a] >= 0) atomicAdd(op.out + idx[a], op.coef * y);
        energy = fma(x[a], y, energy);
      }
    }
  }
  return energy;
}

// Individual cells (op.list != nullptr) or, without a compile-time M, all cells with per-cell
// matrix selection.  Groups of G lanes per cell; xs/ids: per-warp shared scratch (CPW*m).
template <int G>
__device__ __forceinline__ double list_cells(const CellOp& op, const Tab& T, int warp, int nwarps,
                                             double* xs_warp, int* ids_warp) {
  constexpr int CPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const int m = op.m;
  double* xs = xs_warp + grp * m;
  int* ids = ids_warp + grp * m;
  const bool generic = op.list == nullptr;
  const int count = generic ? op.ncell : op.nlist;
  double energy = 0.0;
  const int per_round = nwarps * CPW;
  const int rounds = (count + per_round - 1) / per_round;
  for (int r = 0; r < rounds; ++r) {
    const int i = (r * nwarps + warp) * CPW + grp;
    const bool active = i < count;
    const int c = active ? (generic ? i : op.list[i]) : 0;
    if (active) {
      const int cx = c % op.nx;
      const int cyz = c / op.nx;
      const int cy = cyz % op.ny;
      const int cz = cyz / op.ny;
      for (int a = gl; a < m; a += G) {
        const bool ok = (cx >= T.cmin[a][0]) & (cx <= T.cmax[a][0]) & (cy >= T.cmin[a][1]) &
                        (cy <= T.cmax[a][1]) & (cz >= T.cmin[a][2]) & (cz <= T.cmax[a][2]);
        const int idx = T.base[a] + cx + cy * T.sy[a] + cz * T.sz[a];
        ids[a] = ok ? idx : -1;
        xs[a] = ok ? __ldg(op.in + idx) : 0.0;
      }
    }
    __syncwarp();
    if (active) {
      const double* Mat;
      int ld;
      double scale = 1.0;
      if (!generic) {
        ld = op.list_ld;
        Mat = op.list_mats + (size_t)i * ld * ld;
      } else if (op.mode == OP_APPLY) {
        const uint8_t k = op.kind[c];
        ld = op.ldK;
        if (k == 2) {
          Mat = op.cutK + (size_t)op.cut_idx[c] * ld * ld;
        } else {
          Mat = op.Kref;
          scale = (k == 1) ? op.alpha : 1.0;
        }
      } else {
        const int32_t b = op.blk[c];
        ld = m;
        if (b >= 0) {
          Mat = op.irr_inv + (size_t)b * m * m;
        } else {
          const int t = -b - 1;
          Mat = op.type_inv + (size_t)(t & 0xff) * m * m;
          scale = (t >> 12) ? op.inv_alpha : 1.0;
        }
      }
      for (int a = gl; a < m; a += G) {
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = Mat + a;
        int b = 0;
        for (; b + 2 <= m; b += 2) {
          acc0 = fma(__ldg(col + (size_t)b * ld), xs[b], acc0);
          acc1 = fma(__ldg(col + (size_t)(b + 1) * ld), xs[b + 1], acc1);
        }
        if (b < m) acc0 = fma(__ldg(col + (size_t)b * ld), xs[b], acc0);
        const double y = scale * (acc0 + acc1);
        const int id = ids[a];
        if (id >= 0) atomicAdd(op.out + id, op.coef * y);
        energy = fma(xs[a], y, energy);
      }
    }
    __syncwarp();
  }
  return energy;
}

__device__ __forceinline__ double block_sum(double v, double* red /* >= 32 doubles */) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    const int nw = (blockDim.x + 31) >> 5;
    s = (l < nw) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  }
  __syncthreads();
  return s;  // valid in thread 0
}

}  // namespace fcm
