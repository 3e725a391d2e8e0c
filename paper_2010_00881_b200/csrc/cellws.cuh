// cellws.cuh -- one elementwise cell operation (the level operator apply r = b - A_q x,
// PAPER.md:163/169 with A_{l-1} = R A_l R^T realised as leading element blocks, P:118/P:209-216;
// or one additive-Schwarz sweep x += omega sum_i P_i A_i^{-1} P_i^T r, Eq. AdditiveSchwarz
// P:254-257, elementwise blocks P:259) as ONE warp-specialised persistent launch, one CTA per SM:
//
//  * NS streaming warps apply the INDIVIDUAL matrices (cut-cell element matrices for the
//    operator, irregular Schwarz inverses for the smoother).  They are symmetric and stored
//    TILE-PACKED (patch.cuh layout: lower triangle of 32x32 tiles, off-diagonal tiles full,
//    diagonal tiles packed lower; m = 64: exactly m(m+1)/2).  Because the tile rows are laid out
//    in order, the leading m_q block of a level-m matrix is the first tile rows, each read only
//    up to row m_q: the operator of every level q streams its prefix of the ONE fine-level copy.
//    Tiles move by 1D bulk copies (cp.async.bulk, mbarrier complete_tx) into a two-stage ring
//    per warp that runs ahead across cells; a warp owns a whole cell (gather -> tiles ->
//    scatter), so its y accumulates in shared memory without atomics.
//  * NM MMA warps apply the REGULAR cells (shared K_ref block / shared Schwarz type inverse) as
//    fp64 tensor-core MMAs (cellmma.cuh), fragments of the main matrix staged once per CTA.
//
// The two populations used to be two block ranges of one launch (k_cell_mma), which the block
// scheduler ran one after the other; here they overlap on every SM: the MMA warps are bound by
// fp64 issue and the vector gathers, the streaming warps by HBM.
#pragma once
#include <cstdint>

#include "cellmma.cuh"
#include "patch.cuh"

namespace fcm {


struct TileListOp {
  const int32_t* list;   // [nlist] owned cell index of individual matrix i
  int32_t nlist;
  const double* mats;    // matrix i at mats + i * stride (tile-packed symmetric)
  int64_t stride;        // doubles per stored matrix
  int ntq;               // tiles per dimension at this level: ceil(m_q / 32)
};

// smem bytes of the streaming part (after Tab and the MMA fragments)
__host__ __device__ constexpr size_t ws_stream_smem(int ntq, int ns, int stg) {
  return (size_t)ns * stg * 1024 * 8 + (size_t)ns * stg * 8 + (size_t)ns * 32 * ntq * (8 + 8 + 4);
}

// Individual cells, streamed: warp w of nw per CTA.  xs / ys / ids: 32 ntq slots of this warp;
// ring: STG x 1024 doubles; bars: STG mbarriers.  The first STG tiles were
// already issued by the caller (before griddepcontrol.wait -- matrices are setup data).
// Returns sum over this warp's cells of x_c^T (M_c x_c) (operator energies).
template <int STG>
__device__ __forceinline__ void ws_issue(const TileListOp& tl, int ntl, int64_t gw, int64_t W, int64_t i,
                                         double* ring, uint64_t* bars, int m) {
  const int64_t k = i / ntl;
  const int t = (int)(i % ntl);
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  const int J = t - I * (I + 1) / 2;
  const int R = min(32, m - 32 * I);
  const int64_t cell = gw + k * W;
  const double* src = tl.mats + cell * tl.stride + tile_off(I, J);
  const uint32_t n = I == J ? (uint32_t)((R * (R + 1) / 2 + 1) & ~1) : (uint32_t)(R * 32);
  const int s = (int)(i % STG);
  mbar_expect_tx(&bars[s], n * 8);
  bulk_g2s(ring + s * 1024, src, n * 8, &bars[s]);
}

template <int NTQ, int STG>
__device__ __forceinline__ double ws_stream_cells(const CellOp& op, const TileListOp& tl, const Tab& T,
                                                  double* xs, double* ys, int* ids, double* ring, uint64_t* bars,
                                                  int64_t gw, int64_t W) {
  const int lane = threadIdx.x & 31;
  const int m = op.m, ntq = tl.ntq, ntl = ntq * (ntq + 1) / 2;
  const int64_t ncells = tl.nlist > gw ? (tl.nlist - gw + W - 1) / W : 0;
  const int64_t nitems = ncells * ntl;
  const int nx = op.nx, ny = op.ny;
  const double coef = op.coef;
  double energy = 0.0;
  int64_t item = 0;
  // software pipeline: the NEXT cell's slot indices and values are gathered into registers while
  // this cell's tiles stream (the list entry two cells ahead), so a cell starts with its x ready
  int idn[NTQ];
  double xn[NTQ];
  auto gather = [&](int64_t k) {
    int c = 0;
    if (k < ncells) c = __ldg(tl.list + gw + k * W);
    const int cx = c % nx, cyz = c / nx, cy = cyz % ny, cz = cyz / ny;
#pragma unroll
    for (int j = 0; j < NTQ; ++j) {
      const int l = lane + 32 * j;
      int idx = -1;
      if (k < ncells && l < m && dof_free(T, l, cx, cy, cz)) idx = dof_index(T, l, cx, cy, cz);
      idn[j] = idx;
    }
#pragma unroll
    for (int j = 0; j < NTQ; ++j) {   // branch-free: clamped address, select
      const double v = __ldg(op.in + max(idn[j], 0));
      xn[j] = idn[j] >= 0 ? v : 0.0;
    }
  };
  gather(0);
  for (int64_t k = 0; k < ncells; ++k) {
#pragma unroll
    for (int j = 0; j < NTQ; ++j) {
      const int l = lane + 32 * j;
      ids[l] = idn[j];
      xs[l] = xn[j];
      ys[l] = 0.0;
    }
    __syncwarp();
    gather(k + 1);
    for (int t = 0; t < ntl; ++t, ++item) {
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      const int J = t - I * (I + 1) / 2;
      const int R = min(32, m - 32 * I);
      const int s = (int)(item % STG);
      mbar_wait(&bars[s], (uint32_t)((item / STG) & 1));
      const double* tp = ring + s * 1024;
      const double xJ = xs[32 * J + lane];
      double yJ = 0.0;
      double p[32];
      if (I != J) {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const double a = r < R ? tp[r * 32 + lane] : 0.0;
          p[r] = a * xJ;
          yJ = fma(a, xs[32 * I + r], yJ);
        }
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const double a = (r < R && lane <= r) ? tp[r * (r + 1) / 2 + lane] : 0.0;
          p[r] = a * xJ;
          if (lane < r) yJ = fma(a, xs[32 * I + r], yJ);
        }
      }
      __syncwarp();
      if (lane == 0 && item + STG < nitems) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        ws_issue<STG>(tl, ntl, gw, W, item + STG, ring, bars, m);
      }
      const double yI = warp_reduce_scatter32(p);
      ys[32 * I + lane] += yI;
      ys[32 * J + lane] += yJ;
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < NTQ; ++j) {
      const int l = lane + 32 * j;
      if (l < m) {
        const int idx = ids[l];
        const double y = ys[l];
        if (idx >= 0) atomicAdd(op.out + idx, coef * y);
        energy = fma(xs[l], y, energy);
      }
    }
    __syncwarp();
  }
  return energy;
}

}  // namespace fcm
