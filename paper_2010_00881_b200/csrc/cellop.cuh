// cellop.cuh -- the element-by-element "gather -> small dense GEMV -> scatter-add" primitive
// shared by the level operator apply (PAPER.md:163/169 r = b - A_l x; A_{l-1} = R A_l R^T,
// P:118, realised as leading element blocks) and the additive-Schwarz smoother
// (Eq. AdditiveSchwarz: x += omega sum_i P_i A_i^{-1} P_i^T r).
//
// Two populations of cells, two mappings:
//  * regular cells (uncut for the operator; shared-by-type blocks for the smoother) -- TS
//    consecutive THREADS per cell (thread j owns a block of RB rows); the m gathered values
//    live in registers (compile-time M, full unroll); the shared matrix (K_ref or the
//    interior-type inverse) is read from shared memory as LDS.128 row pairs (all cells of a
//    warp read the same words); other boundary types read through L1.  Consecutive lanes are
//    consecutive cells along x, so every gather / scatter instruction is coalesced.  Cells away
//    from Dirichlet faces take a gather path without bounds tests.
//  * individual cells (cut cells / irregular blocks) -- one GROUP of G lanes per cell over a
//    compact list; lane a owns rows a, a+G, ...; the individual matrix is streamed column-wise
//    (Mat[b*ld + a], symmetric) so the G lanes read consecutive addresses.
// The scatter is a fp64 red.global.add into the output vector.
#pragma once
#include <cstdint>

namespace fcm {

constexpr int kMaxM = 128;  // largest element block handled by the cell kernels

enum { OP_APPLY = 0, OP_SMOOTH = 1 };

struct Tab {      // level table in shared memory; stride along x is 1 for every DOF class
  int4 g[kMaxM];  // {base, stride_y, stride_z, -}
  int4 lo[kMaxM]; // free cell range of local DOF a: c_i in [lo_i, hi_i]
  int4 hi[kMaxM];
};

struct CellOp {
  int nx, ny, nz;
  int m;                      // level element DOFs m_q
  int32_t ncell;
  const int64_t* base;
  const int32_t* stride;
  const int16_t* cmin;
  const int16_t* cmax;
  int ilo[3], ihi[3];         // cells whose every local DOF is free (no Dirichlet test needed)
  int mode;                   // OP_APPLY / OP_SMOOTH
  // APPLY (regular): K_ref (kind 0) or alpha K_ref (kind 1); kind 2 cells are in the list
  const uint8_t* kind;
  const double* Kref;
  int ldK;
  double alpha;
  // SMOOTH (regular): blk < 0: t = -blk-1, type_inv[t & 0xfff] * (t >> 12 ? 1/alpha : 1) (slot index);
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
  // fused input (FUSE template): value = in + c1 * (in1 + c2 * in2)
  const double* in1;
  const double* in2;
  double c1, c2;
  double* out;
  double coef;
  double* partials;           // per-block sum of in_local^T (scale Mat in_local), or nullptr
  int colour;                 // deterministic mode: only cells of this parity colour (-1: all)
};

// parity colour of a cell (2^d colours): cells of one colour share no DOF, so a launch restricted
// to one colour adds at most one contribution to every output entry (deterministic scatter)
__device__ __forceinline__ int cell_colour(int cx, int cy, int cz) { return (cx & 1) | ((cy & 1) << 1) | ((cz & 1) << 2); }

__device__ __forceinline__ void load_tab(Tab& T, const CellOp& op) {
  for (int a = threadIdx.x; a < op.m; a += blockDim.x) {
    T.g[a] = make_int4((int32_t)op.base[a], op.stride[a * 3 + 1], op.stride[a * 3 + 2], 0);
    T.lo[a] = make_int4(op.cmin[a * 3 + 0], op.cmin[a * 3 + 1], op.cmin[a * 3 + 2], 0);
    T.hi[a] = make_int4(op.cmax[a * 3 + 0], op.cmax[a * 3 + 1], op.cmax[a * 3 + 2], 0);
  }
}

template <bool FUSE>
__device__ __forceinline__ double load_in(const CellOp& op, int i) {
  double v = __ldg(op.in + i);
  if constexpr (FUSE) v = fma(op.c1, fma(op.c2, __ldg(op.in2 + i), __ldg(op.in1 + i)), v);
  return v;
}

__device__ __forceinline__ bool dof_free(const Tab& T, int a, int cx, int cy, int cz) {
  const int4 lo = T.lo[a], hi = T.hi[a];
  return (cx >= lo.x) & (cx <= hi.x) & (cy >= lo.y) & (cy <= hi.y) & (cz >= lo.z) & (cz <= hi.z);
}
__device__ __forceinline__ int dof_index(const Tab& T, int a, int cx, int cy, int cz) {
  const int4 g = T.g[a];
  return g.x + cx + cy * g.y + cz * g.z;
}

// shared matrix of the regular path, column-major with an even leading dimension MP so that
// rows (a, a+1) of one column are one 16-byte LDS.128: Ms[b*MP + a] = Mat[a][b].
template <int M> __host__ __device__ constexpr int padded() { return M + (M & 1); }
template <int M>
__device__ __forceinline__ void load_shared_matrix(double* Ms, const CellOp& op) {
  constexpr int MP = padded<M>();
  for (int e = threadIdx.x; e < M * MP; e += blockDim.x) {
    const int b = e / MP, a = e % MP;
    double v = 0.0;
    if (a < M) v = (op.mode == OP_APPLY) ? op.Kref[a * op.ldK + b] : op.type_inv[a * M + b];  // type code 0
    Ms[e] = v;
  }
}

// rows of a cell are split over TS consecutive threads (blocked: thread j owns rows
// [j*RB, j*RB+RB)), RB even so a thread's rows of one column are LDS.128 pairs.
template <int M> __host__ __device__ constexpr int split_of() {
  return M <= 4 ? 1 : (M <= 9 ? 2 : (M <= 16 ? 4 : 8));
}
template <int M, int TS> __host__ __device__ constexpr int rows_of() { return ((M + TS - 1) / TS + 1) / 2 * 2; }
// per-warp shared scratch of the regular path (doubles): one padded x vector per cell slot
template <int M, int TS> __host__ __device__ constexpr int reg_scratch() { return (32 / TS) * padded<M>(); }

// A warp holds CPW = 32/TS cells; lane = slot*TS + j.  The TS lanes of a cell gather its M
// values cooperatively (a = j, j+TS, ...) into shared memory, then every lane loads the whole
// vector into registers and computes its RB rows.  Warp-synchronous (uniform trip count).
template <int M, int TS, bool FUSE>
__device__ __forceinline__ double reg_cells(const CellOp& op, const Tab& T, const double* __restrict__ Ms,
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
        const int code = t & 0xfff;
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
      if (op.colour >= 0 && cell_colour(cx, cy, cz) != op.colour) act = false;
    }
    if (act) {
      for (int a = j; a < M; a += TS)
        xs[a] = (inner || dof_free(T, a, cx, cy, cz)) ? load_in<FUSE>(op, dof_index(T, a, cx, cy, cz)) : 0.0;
    }
    __syncwarp();
    if (act) {
    // the gathered vector stays in shared memory (xs[b] is one broadcast word per cell), which
    // keeps the register footprint small enough for 4 resident blocks per SM
    double acc[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) acc[i] = 0.0;
    if (Mg == nullptr) {
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
          atomicAdd(out + ia, coef * y);
          if (want_e) energy = fma(xs[a], y, energy);
        }
      }
    }
    }  // act
    __syncwarp();
  }
  return energy;
}

// Individual cells (op.list != nullptr) or, without a compile-time M, all cells with per-cell
// matrix selection.  Groups of G lanes per cell; xs/ids: per-warp shared scratch (CPW*m).
// MC: compile-time m (0 = runtime): the row loop is fully unrolled, so all m matrix loads of
// a row are in flight at once (one L2/HBM latency per cell instead of one per load pair)
template <int G, bool FUSE, int MC = 0>
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
  const int nx = op.nx, ny = op.ny;
  double* __restrict__ out = op.out;
  const double coef = op.coef;
  double energy = 0.0;
  const int per_round = nwarps * CPW;
  const int rounds = (count + per_round - 1) / per_round;
  for (int r = 0; r < rounds; ++r) {
    const int i = (r * nwarps + warp) * CPW + grp;
    bool active = i < count;
    const int c = active ? (generic ? i : op.list[i]) : 0;
    if (active && op.colour >= 0) active = cell_colour(c % nx, (c / nx) % ny, c / (nx * ny)) == op.colour;
    if (active) {
      const int cx = c % nx;
      const int cyz = c / nx;
      const int cy = cyz % ny;
      const int cz = cyz / ny;
      for (int a = gl; a < m; a += G) {
        const bool ok = dof_free(T, a, cx, cy, cz);
        const int idx = dof_index(T, a, cx, cy, cz);
        ids[a] = ok ? idx : -1;
        xs[a] = ok ? load_in<FUSE>(op, idx) : 0.0;
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
          Mat = op.type_inv + (size_t)(t & 0xfff) * m * m;
          scale = (t >> 12) ? op.inv_alpha : 1.0;
        }
      }
      for (int a = gl; a < m; a += G) {
        double acc0 = 0.0, acc1 = 0.0;
        const double* col = Mat + a;
        if constexpr (MC > 0) {
          double mv[MC];
#pragma unroll
          for (int b = 0; b < MC; ++b) mv[b] = __ldg(col + (size_t)b * ld);
          double acc2 = 0.0, acc3 = 0.0;
#pragma unroll
          for (int b = 0; b < MC; b += 4) {
            acc0 = fma(mv[b], xs[b], acc0);
            if (b + 1 < MC) acc1 = fma(mv[b + 1], xs[b + 1], acc1);
            if (b + 2 < MC) acc2 = fma(mv[b + 2], xs[b + 2], acc2);
            if (b + 3 < MC) acc3 = fma(mv[b + 3], xs[b + 3], acc3);
          }
          acc0 += acc2;
          acc1 += acc3;
        } else {
          int b = 0;
          for (; b + 16 <= m; b += 16) {   // 16 column loads in flight per trip
            double mv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) mv[j] = __ldg(col + (size_t)(b + j) * ld);
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
              acc0 = fma(mv[j], xs[b + j], acc0);
              acc1 = fma(mv[j + 1], xs[b + j + 1], acc1);
            }
          }
          for (; b + 2 <= m; b += 2) {
            acc0 = fma(__ldg(col + (size_t)b * ld), xs[b], acc0);
            acc1 = fma(__ldg(col + (size_t)(b + 1) * ld), xs[b + 1], acc1);
          }
          if (b < m) acc0 = fma(__ldg(col + (size_t)b * ld), xs[b], acc0);
        }
        const double y = scale * (acc0 + acc1);
        const int id = ids[a];
        if (id >= 0) atomicAdd(out + id, coef * y);
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
