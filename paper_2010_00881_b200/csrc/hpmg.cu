// hpmg.cu -- B200 (sm_100a) hp-multigrid on multi-level hp-refined finite cell grids (SURVEY
// §8(f4), Fig. hpmultigrid :219-224, blocks :259 / Fig. 7).
//
// The discretisation (gen_hp.cpp) numbers the DOFs by the coarsest hp level containing them, so
// every level (q, kc) of the sequence (p,k) ... (1,k), (1,k-1) ... (1,0) is a PREFIX of the fine
// vector: restriction is a pointer alias and prolongation an add on the prefix.  A
// leaf's DOF list is ascending, so its level-l DOFs are a prefix of the list and the level-l leaf
// matrix is the leading m_l x m_l block of the leaf matrix (P:209-216 hierarchical matrices).
//
// Hot path:
//   operator      k_hp_apply<NCH>: one warp per leaf, symmetric K_e read row by row (lanes own
//                 output columns: y_a = sum_b K_ba x_b, coalesced rows, no shuffles), x_e staged in
//                 shared memory, scatter by fp64 atomics.  HBM-bound on the leaf matrices.
//   smoother      k_hp_smooth<NT,NCH>: one CTA per Schwarz block (blocks sorted into size classes,
//                 one launch per class), A_i^{-1} streamed row by row the same way; x += w y by
//                 atomics (blocks overlap).  HBM-bound on the block inverses.
//   V-cycle       Algorithm 1 with the residual before every sweep (R1), captured into a CUDA
//                 graph when the coarse solve is direct (dense inverse GEMV).
//   FCG           flexible PCG, device-side scalars, one 8-byte D2H per iteration.
// Setup: blocks built on the host from the leaves' base elements (R26), assembled on the device
// from the leaf matrices (one CTA per block, leaves in sequence), inverted by the equilibrated
// batched blocked Gauss-Jordan of gj.cuh; the (1,0) matrix assembled densely (atomics) and
// inverted the same way for the direct coarse solve.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/fcm_mg.h"
#include "common.hpp"
#include "gj.cuh"

using namespace fcm;

namespace fcm {
void hp_disc_view(const fcm_hp_disc* d, int* dim, int* n, int* p, int* n_f, int64_t* ndof, std::vector<int64_t>* level_n,
                  const std::vector<int64_t>** leaf_ptr, const std::vector<int64_t>** leaf_kptr,
                  const std::vector<int32_t>** leaf_dofs, const std::vector<double>** leaf_K,
                  const std::vector<int32_t>** leaf_info);
}

#define HCU(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? FCM_ENOMEM : FCM_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
  } while (0)
#define HRC(call)            \
  do {                       \
    int rc_ = (call);        \
    if (rc_ < 0) return rc_; \
  } while (0)

namespace {

constexpr int kHpThreads = 256;
constexpr int kHpDotBlocks = 296;   // 2 x 148 SMs: fixed grid -> deterministic partial sums
constexpr int kHpMaxBlock = 4096;   // tile-streamed blocks: 64 KB of vectors + 128 KB of rings per CTA

// ---- kernels --------------------------------------------------------------------------------
template <int NCH>
__global__ void __launch_bounds__(kHpThreads) k_hp_apply(int64_t nleaf, const int64_t* __restrict__ lptr,
                                                         const int64_t* __restrict__ kptr,
                                                         const int32_t* __restrict__ dofs, const double* __restrict__ K,
                                                         const int32_t* __restrict__ mlev, const double* __restrict__ x,
                                                         double* __restrict__ y, double sign) {
  extern __shared__ double xs_all[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* xs = xs_all + wib * 32 * NCH;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t L = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; L < nleaf; L += nw) {
    const int ml = mlev[L];
    if (ml == 0) continue;
    const int64_t o = lptr[L];
    const int m = (int)(lptr[L + 1] - o);
    const double* __restrict__ Ke = K + kptr[L];
    for (int a = lane; a < ml; a += 32) xs[a] = x[dofs[o + a]];
    __syncwarp();
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
#pragma unroll 4
    for (int b = 0; b < ml; ++b) {
      const double xb = xs[b];
      const double* __restrict__ row = Ke + (int64_t)b * m;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int a = lane + 32 * c;
        if (a < ml) acc[c] = fma(__ldg(row + a), xb, acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int a = lane + 32 * c;
      if (a < ml) atomicAdd(&y[dofs[o + a]], sign * acc[c]);
    }
    __syncwarp();
  }
}

template <int NT, int NCH>
__global__ void __launch_bounds__(NT) k_hp_smooth(int64_t b0, int64_t b1, const int64_t* __restrict__ bptr,
                                                  const int32_t* __restrict__ bdofs, const int64_t* __restrict__ iptr,
                                                  const double* __restrict__ inv, const double* __restrict__ r,
                                                  double* __restrict__ x, double omega) {
  __shared__ double rs[NT * NCH];
  for (int64_t B = b0 + blockIdx.x; B < b1; B += gridDim.x) {
    const int64_t o = bptr[B];
    const int m = (int)(bptr[B + 1] - o);
    const double* __restrict__ A = inv + iptr[B];
    for (int a = threadIdx.x; a < m; a += NT) rs[a] = r[bdofs[o + a]];
    __syncthreads();
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    for (int b = 0; b < m; ++b) {
      const double rb = rs[b];
      const double* __restrict__ row = A + (int64_t)b * m;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int a = threadIdx.x + NT * c;
        if (a < m) acc[c] = fma(__ldg(row + a), rb, acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int a = threadIdx.x + NT * c;
      if (a < m) atomicAdd(&x[bdofs[o + a]], omega * acc[c]);
    }
    __syncthreads();
  }
}

// Packed symmetric Schwarz apply (the production smoother): A_i^{-1} stored lower-packed (row b
// holds A[b][0..b], offset b(b+1)/2 -- half the bytes of full storage).  One CTA per
// block, NW warps; warp w streams rows b = w, w + NW, ...: lanes own columns a = lane + 32c, so a
// row contributes y_a += A[b][a] r_b (a < b, column-owner registers, no reduction) and
// y_b += sum_{a<=b} A[b][a] r_a (the transposed half: one 5-shuffle warp reduction per row).  The
// per-warp column sums and the row sums meet in shared memory (fp64 shared atomics); the result
// is scattered x += omega y with global atomics (blocks overlap).
template <int NW, int NCH>
__device__ __forceinline__ void hp_sym_block(const double* __restrict__ A, int m, const double* rs, double* ys) {
  constexpr int PW = 32 * NCH;            // column panel width
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int P0 = 0; P0 < m; P0 += PW) {   // column panels (one unless m > 32 NCH)
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    // rows b >= P0 touch the panel (a <= b); warp w takes b = P0 + w, P0 + w + NW, ...
#pragma unroll 4
    for (int b = P0 + w; b < m; b += NW) {
      const double* __restrict__ row = A + (int64_t)b * (b + 1) / 2;
      const double rb = rs[b];
      double v[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int a = P0 + lane + 32 * c;
        v[c] = a <= b ? __ldg(row + a) : 0.0;
      }
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int a = P0 + lane + 32 * c;
        if (a < b) acc[c] = fma(v[c], rb, acc[c]);          // strictly lower: column-owner half
        if (a <= b) dot = fma(v[c], rs[a], dot);              // the row half (incl. the diagonal)
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      if (lane == 0) atomicAdd(&ys[b], dot);
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int a = P0 + lane + 32 * c;
      if (a < m) atomicAdd(&ys[a], acc[c]);
    }
  }
}

// Packed symmetric Schwarz apply (the production smoother): A_i^{-1} stored lower-packed (row b
// holds A[b][0..b], offset b(b+1)/2 -- half the bytes of full storage).  One CTA of
// NW warps per block (grid-stride over a range of blocks sorted by DESCENDING size, so the large
// blocks start first); warp w streams rows b = w, w + NW, ...: lanes own columns a = lane + 32c, so
// a row contributes y_a += A[b][a] r_b (a < b, column-owner registers, no reduction) and
// y_b += sum_{a<=b} A[b][a] r_a (the transposed half: one 5-shuffle warp reduction per row).  The
// per-warp column sums and the row sums meet in shared memory (fp64 shared atomics); the result is
// scattered x += omega y with global atomics (blocks overlap).  MAXCH caps the register chunks of
// the instance (blocks up to 32 MAXCH DOFs in one panel; larger ones loop over panels).
template <int NW, int MAXCH>
__global__ void __launch_bounds__(NW * 32) k_hp_smooth_sym(int64_t b0, int64_t b1, const int64_t* __restrict__ bptr,
                                                         const int32_t* __restrict__ bdofs,
                                                         const int64_t* __restrict__ iptr,
                                                         const double* __restrict__ inv, const double* __restrict__ r,
                                                         double* __restrict__ x, double omega, int mmax) {
  extern __shared__ double sm_sym[];
  double* rs = sm_sym;                    // [mmax]
  double* ys = sm_sym + mmax;             // [mmax]
  for (int64_t B = b0 + blockIdx.x; B < b1; B += gridDim.x) {
    const int64_t o = bptr[B];
    const int m = (int)(bptr[B + 1] - o);
    const double* __restrict__ A = inv + iptr[B];
    for (int a = threadIdx.x; a < m; a += NW * 32) {
      rs[a] = r[bdofs[o + a]];
      ys[a] = 0.0;
    }
    __syncthreads();
    const int nch = (m + 31) / 32;
    if (nch <= 1) hp_sym_block<NW, 1>(A, m, rs, ys);
    else if (nch <= 2 || MAXCH < 4) hp_sym_block<NW, (MAXCH < 2 ? MAXCH : 2)>(A, m, rs, ys);
    else if (nch <= 4 || MAXCH < 8) hp_sym_block<NW, (MAXCH < 4 ? MAXCH : 4)>(A, m, rs, ys);
    else if (nch <= 8 || MAXCH < 16) hp_sym_block<NW, (MAXCH < 8 ? MAXCH : 8)>(A, m, rs, ys);
    else hp_sym_block<NW, MAXCH>(A, m, rs, ys);
    __syncthreads();
    for (int a = threadIdx.x; a < m; a += NW * 32) atomicAdd(&x[bdofs[o + a]], omega * ys[a]);
    __syncthreads();
  }
}

// ---- large blocks: tile-packed inverses streamed by bulk copies ------------------------------
// Blocks with more than kHpTileMin DOFs store A_i^{-1} TILE-PACKED (the lower triangle of 32x32
// tiles, row-major over tile rows; off-diagonal tiles full 1024 doubles, diagonal tiles packed
// lower 528; padding rows/columns hold the identity of the padded inverse).  One CTA of 8 warps
// per block (grid-stride over the large blocks, descending size); each warp owns tiles
// t = w, w + 8, ... of the block and streams them through a 2-stage ring of 8 KB shared-memory
// stages filled by cp.async.bulk (mbarrier complete_tx), issuing across block boundaries.  A
// tile (I, J) is read row by row with lane = column: y_J += T^T r_I in a register, the row
// products y_I += T r_J by one 31-shuffle reduce-scatter (the layout and arithmetic of the
// patch-smoother streaming warps, patch.cuh).
constexpr int kHpTileMin = 128;
constexpr int kHpTileMax = 4096;
constexpr int kHpTileWarps = 8;
constexpr int kHpStages = 2;
constexpr int kHpDiag = 528;

__host__ __device__ inline int64_t hp_tile_pack_size(int nt) {
  return (int64_t)nt * (nt - 1) / 2 * 1024 + (int64_t)nt * kHpDiag;
}
__host__ __device__ inline int64_t hp_tile_off(int I, int J) {   // J <= I
  return (int64_t)I * (I - 1) / 2 * 1024 + (int64_t)I * kHpDiag + (int64_t)J * 1024;
}
__device__ __forceinline__ uint32_t hp_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void hp_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(hp_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void hp_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(hp_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void hp_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(hp_smem_u32(dst)), "l"(src), "r"(bytes), "r"(hp_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void hp_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(hp_smem_u32(bar)), "r"(parity) : "memory");
}
// 32 per-lane row partials -> lane r holds the warp sum of partial r (reduce-scatter butterfly)
__device__ __forceinline__ double hp_reduce_scatter32(double (&p)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int hh = 16; hh >= 1; hh >>= 1) {
    const bool up = lane & hh;
#pragma unroll
    for (int i = 0; i < hh; ++i) {
      const double send = up ? p[i] : p[i + hh];
      const double keep = up ? p[i + hh] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, hh);
    }
  }
  return p[0];
}

__global__ void __launch_bounds__(kHpTileWarps * 32, 1)
k_hp_smooth_tiles(int64_t b0, int64_t b1, const int64_t* __restrict__ bptr, const int32_t* __restrict__ bdofs,
                  const int64_t* __restrict__ iptr, const double* __restrict__ inv, const double* __restrict__ r,
                  double* __restrict__ x, double omega, int ntmax) {
  extern __shared__ __align__(128) double sm_t[];
  double* ring_all = sm_t;                                          // [8][2][1024]
  uint64_t* bars_all = (uint64_t*)(ring_all + kHpTileWarps * kHpStages * 1024);   // [8][2]
  double* xs = (double*)(bars_all + kHpTileWarps * kHpStages);      // [32 ntmax]
  double* ys = xs + 32 * ntmax;                                     // [32 ntmax]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* ring = ring_all + w * kHpStages * 1024;
  uint64_t* bars = bars_all + w * kHpStages;
  if (lane == 0)
    for (int s = 0; s < kHpStages; ++s) hp_mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // issue cursor of this warp over (block, tile) in processing order
  int64_t iB = b0 + blockIdx.x;
  int it = w;
  auto ntiles_of = [&](int64_t B) {
    const int m = (int)(bptr[B + 1] - bptr[B]);
    const int nt = (m + 31) / 32;
    return nt * (nt + 1) / 2;
  };
  auto advance = [&]() {   // next (block, tile) with a tile for this warp
    while (iB < b1) {
      if (it < ntiles_of(iB)) return true;
      iB += gridDim.x;
      it = w;
    }
    return false;
  };
  int64_t issued = 0;
  auto issue_next = [&]() {
    if (!advance()) return;
    int I = (int)((sqrtf(8.0f * it + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > it) --I;
    while ((I + 1) * (I + 2) / 2 <= it) ++I;
    const int J = it - I * (I + 1) / 2;
    const uint32_t bytes = (I == J ? kHpDiag : 1024) * 8;
    const int s = (int)(issued % kHpStages);
    hp_mbar_expect_tx(&bars[s], bytes);
    hp_bulk_g2s(ring + s * 1024, inv + iptr[iB] + hp_tile_off(I, J), bytes, &bars[s]);
    ++issued;
    it += kHpTileWarps;
  };
  if (lane == 0)
    for (int s = 0; s < kHpStages; ++s) issue_next();
  int64_t item = 0;
  for (int64_t B = b0 + blockIdx.x; B < b1; B += gridDim.x) {
    const int64_t o = bptr[B];
    const int m = (int)(bptr[B + 1] - o);
    const int nt = (m + 31) / 32;
    for (int a = threadIdx.x; a < 32 * nt; a += blockDim.x) {
      xs[a] = a < m ? r[bdofs[o + a]] : 0.0;
      ys[a] = 0.0;
    }
    __syncthreads();
    const int ntiles = nt * (nt + 1) / 2;
    for (int t = w; t < ntiles; t += kHpTileWarps) {
      int I = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > t) --I;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      const int J = t - I * (I + 1) / 2;
      const int s = (int)(item % kHpStages);
      hp_mbar_wait(&bars[s], (uint32_t)((item / kHpStages) & 1));
      const double* tl = ring + s * 1024;
      const double xJ = xs[32 * J + lane];
      double yJ = 0.0;
      double pr[32];
      if (I != J) {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const double a = tl[rr * 32 + lane];
          pr[rr] = a * xJ;
          yJ = fma(a, xs[32 * I + rr], yJ);
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const double a = lane <= rr ? tl[rr * (rr + 1) / 2 + lane] : 0.0;
          pr[rr] = a * xJ;
          if (lane < rr) yJ = fma(a, xs[32 * I + rr], yJ);
        }
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_next();
      }
      const double yI = hp_reduce_scatter32(pr);
      ++item;
      atomicAdd(&ys[32 * I + lane], yI);
      atomicAdd(&ys[32 * J + lane], yJ);
    }
    __syncthreads();
    for (int a = threadIdx.x; a < m; a += blockDim.x) atomicAdd(&x[bdofs[o + a]], omega * ys[a]);
    __syncthreads();
  }
}

// workspace (ld MP) -> tile-packed lower storage, symmetrised; grid (tiles of the largest block,
// blocks of the chunk)
__global__ void k_hp_pack_tiles(const double* W, int MP, const int64_t* __restrict__ dst_off,
                                const int32_t* __restrict__ bsize, double* inv) {
  const int m = bsize[blockIdx.y];
  const int nt = (m + 31) / 32;
  const int t = blockIdx.x;
  if (t >= nt * (nt + 1) / 2) return;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  const int J = t - I * (I + 1) / 2;
  const double* Wb = W + (int64_t)blockIdx.y * MP * MP;
  double* out = inv + dst_off[blockIdx.y] + hp_tile_off(I, J);
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int rr = e / 32, c = e % 32;
    const int gi = 32 * I + rr, gj = 32 * J + c;
    const double v = 0.5 * (Wb[(int64_t)gi * MP + gj] + Wb[(int64_t)gj * MP + gi]);
    if (I != J) out[e] = v;
    else if (c <= rr) out[rr * (rr + 1) / 2 + c] = v;
  }
}

// block assembly A_i = P_i^T A_l P_i: W (ld MP, one per block of the chunk) += the level blocks of
// every leaf holding a DOF of the block, mapped by amap (leaf-local level index -> block position,
// -1 for DOFs outside the block); the leaves of a block in sequence
__global__ void __launch_bounds__(256) k_hp_asm(double* W, int MP, const int64_t* __restrict__ cptr,
                                                const int64_t* __restrict__ cleaf, const int64_t* __restrict__ cmap,
                                                const int32_t* __restrict__ amap, const int64_t* __restrict__ kptr,
                                                const int64_t* __restrict__ lptr, const int32_t* __restrict__ mlev,
                                                const double* __restrict__ K, const int32_t* __restrict__ bsize) {
  double* Wb = W + (int64_t)blockIdx.x * MP * MP;
  for (int64_t t = cptr[blockIdx.x]; t < cptr[blockIdx.x + 1]; ++t) {
    const int64_t L = cleaf[t];
    const int ml = mlev[L];
    const int m = (int)(lptr[L + 1] - lptr[L]);
    const double* Ke = K + kptr[L];
    const int32_t* mp = amap + cmap[t];
    for (int e = threadIdx.x; e < ml * ml; e += blockDim.x) {
      const int a = e / ml, b = e % ml;
      const int pa = mp[a], pb = mp[b];
      if (pa >= 0 && pb >= 0) Wb[(int64_t)pa * MP + pb] += Ke[(int64_t)a * m + b];
    }
    __syncthreads();
  }
  const int mb = bsize[blockIdx.x];
  for (int l = mb + threadIdx.x; l < MP; l += blockDim.x) Wb[(int64_t)l * MP + l] = 1.0;
}

// dense assembly of a level matrix (direct coarse solve): warp per leaf, atomics
__global__ void k_hp_asm_dense(double* W, int64_t MP, int64_t nleaf, const int64_t* __restrict__ lptr,
                               const int64_t* __restrict__ kptr, const int32_t* __restrict__ dofs,
                               const double* __restrict__ K, const int32_t* __restrict__ mlev) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t L = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; L < nleaf; L += nw) {
    const int ml = mlev[L];
    const int64_t o = lptr[L];
    const int m = (int)(lptr[L + 1] - o);
    const double* Ke = K + kptr[L];
    for (int e = lane; e < ml * ml; e += 32) {
      const int a = e / ml, b = e % ml;
      atomicAdd(&W[(int64_t)dofs[o + a] * MP + dofs[o + b]], Ke[(int64_t)a * m + b]);
    }
  }
}

// symmetric equilibration of ONE large matrix (the dense coarse inverse; gj.cuh's k_equil keeps
// d in shared memory, which caps MP): phase 0 computes d_i = a_ii^-1/2, then W_ij *= d_i d_j
__global__ void k_hp_equil_d(const double* W, int64_t MP, double* d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < MP; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = W[i * MP + i];
    d[i] = (a > 0.0 && isfinite(a)) ? rsqrt(a) : 1.0;
  }
}
__global__ void k_hp_equil_scale(double* W, int64_t MP, const double* __restrict__ d) {
  for (int64_t i = blockIdx.x; i < MP; i += gridDim.x) {
    const double di = d[i];
    for (int64_t j = threadIdx.x; j < MP; j += blockDim.x) W[i * MP + j] *= di * d[j];
  }
}

__global__ void k_hp_identity_pad(double* W, int64_t MP, int64_t n) {
  for (int64_t l = n + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < MP; l += (int64_t)gridDim.x * blockDim.x)
    W[l * MP + l] = 1.0;
}

// the leading m x m block of each workspace matrix -> the block's lower-packed inverse
__global__ void k_hp_extract(const double* W, int MP, const int64_t* __restrict__ dst_off,
                             const int32_t* __restrict__ bsize, double* inv) {
  const double* Wb = W + (int64_t)blockIdx.x * MP * MP;
  const int m = bsize[blockIdx.x];
  double* out = inv + dst_off[blockIdx.x];
  // lower-packed, symmetrised: out[b(b+1)/2 + a] = (W_ba + W_ab) / 2, a <= b
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = warp; b < m; b += blockDim.x >> 5)
    for (int a = lane; a <= b; a += 32)
      out[(int64_t)b * (b + 1) / 2 + a] = 0.5 * (Wb[(int64_t)b * MP + a] + Wb[(int64_t)a * MP + b]);
}

// z = Ainv r (dense symmetric, row-major): warp per output row
__global__ void k_hp_gemv(const double* __restrict__ A, const double* __restrict__ r, double* __restrict__ z,
                          int64_t n, int64_t ld) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    double s = 0.0;
    const double* row = A + i * ld;
    for (int64_t j = lane; j < n; j += 32) s = fma(row[j], r[j], s);
    for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) z[i] = s;
  }
}

__device__ __forceinline__ double hp_block_sum(double v) {
  __shared__ double red[32];
  for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int off = 16; off; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  }
  return s;   // valid in thread 0
}

__global__ void k_hp_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = hp_block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// dst = sum of np partials (fixed order)
__global__ void k_hp_sum(const double* part, int np, double* dst) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = hp_block_sum(s);
  if (threadIdx.x == 0) *dst = s;
}

// device scalars of a CG / FCG iteration
struct HpScal {
  double rz, pq, rr, zr, zro, bb, rr0, pad;
};

// x += a p, r_old = r, r -= a q (a = rz / pq), partial r.r
__global__ void k_hp_cg_update(HpScal* s, double* __restrict__ x, double* __restrict__ r, double* __restrict__ r_old,
                               const double* __restrict__ p, const double* __restrict__ q, int64_t n, double* part) {
  const double a = s->rz / s->pq;
  double rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    const double ri = r[i];
    if (r_old) r_old[i] = ri;
    const double rn = fma(-a, q[i], ri);
    r[i] = rn;
    rr = fma(rn, rn, rr);
  }
  rr = hp_block_sum(rr);
  if (threadIdx.x == 0) part[blockIdx.x] = rr;
}

// p = z + beta p; beta = (zr - zro) / rz (flexible, Polak-Ribiere, R5) or zr / rz (standard CG,
// zro = 0)
__global__ void k_hp_cg_p(const HpScal* s, double* __restrict__ p, const double* __restrict__ z, int64_t n) {
  const double beta = (s->zr - s->zro) / s->rz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}
__global__ void k_hp_set(HpScal* s, int what) {
  if (threadIdx.x) return;
  if (what == 0) s->rz = s->zr;          // after the p update
  else if (what == 1) s->zro = 0.0;      // standard CG
  else if (what == 2) s->rr0 = s->rr;
}
__global__ void k_hp_copy(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}
__global__ void k_hp_add(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

// ---- handle -----------------------------------------------------------------------------------
struct HpClass {
  int64_t b0, b1;
  int nt, nch;      // warps per CTA, column chunks per lane
  int64_t mmax;     // largest block of the class (shared-memory size)
};

struct HpLevel {
  int64_t n = 0;
  double omega = 1.0;
  int32_t* mlev = nullptr;         // per leaf: number of level DOFs
  int max_ml = 0;
  bool has_blocks = false;
  int64_t nblk = 0, n_inv = 0, n_bdofs = 0;
  int64_t* bptr = nullptr;
  int32_t* bdofs = nullptr;
  int64_t* iptr = nullptr;
  double* inv = nullptr;
  std::vector<HpClass> cls;
  double* x = nullptr;             // V-cycle correction on this level
  double* r = nullptr;             // residual on this level (its prefix is the next level's b)
};

}  // namespace

struct fcm_hp {
  int dim = 2, n = 0, p = 1, n_f = 1, nlev = 0;
  int64_t ndof = 0, nleaf = 0;
  cudaStream_t stream = nullptr;    // the library's own stream (capturable)
  cudaStream_t ustream = nullptr;   // the caller's stream: joined by events at entry and exit
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaStream_t stream2 = nullptr;   // side branch: concurrent smoother size classes
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t* lptr = nullptr;
  int64_t* kptr = nullptr;
  int32_t* ldofs = nullptr;
  double* K = nullptr;
  std::vector<HpLevel> lev;
  int coarse = FCM_COARSE_DIRECT;
  double coarse_rtol = 1e-12;
  int coarse_maxit = 10000;
  int n_pre = 5, n_post = 5;
  double* cinv = nullptr;          // direct: dense inverse of the coarsest level, ld = n
  // work vectors (fine size) and scalars
  double *w_p = nullptr, *w_q = nullptr, *w_z = nullptr, *w_ro = nullptr, *w_r = nullptr;
  double *c_x = nullptr, *c_r = nullptr, *c_p = nullptr, *c_q = nullptr, *c_z = nullptr;   // coarse CG
  double* part = nullptr;
  HpScal* s = nullptr;             // outer
  HpScal* cs = nullptr;            // coarse
  double* h_pin = nullptr;         // pinned host scalar
  int64_t launches = 0, coarse_iters = 0, vcycles = 0;
  std::vector<void*> allocs;
  cudaGraphExec_t vgraph = nullptr;
  const double* vg_r = nullptr;
  double* vg_z = nullptr;
  int64_t vg_count = 0;

  template <class T>
  int alloc(T** p_, int64_t count) {
    void* q = nullptr;
    const size_t bytes = (size_t)std::max<int64_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FCM_ENOMEM, "fcm_hp: cudaMalloc of %zu bytes failed (%s)", bytes, cudaGetErrorString(e));
    }
    allocs.push_back(q);
    *p_ = (T*)q;
    return FCM_OK;
  }
  ~fcm_hp() {
    if (vgraph) cudaGraphExecDestroy(vgraph);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (stream) cudaStreamDestroy(stream);
    if (stream2) cudaStreamDestroy(stream2);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (void* q : allocs) cudaFree(q);
    if (h_pin) cudaFreeHost(h_pin);
  }
};

namespace {

bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && v[0] != '0';
}

int grid_for(int64_t n) { return (int)std::min<int64_t>(std::max<int64_t>((n + kHpThreads - 1) / kHpThreads, 1), 148 * 8); }

int nch_for(int m) {
  int c = 1;
  while (32 * c < m) c *= 2;
  return c;
}

int launch_apply(fcm_hp* h, int l, const double* x, double* y, double sign) {
  HpLevel& L = h->lev[l];
  const int nch = nch_for(L.max_ml);
  const int wpb = kHpThreads / 32;
  const size_t smem = (size_t)wpb * 32 * nch * 8;
  const int grid = (int)std::min<int64_t>((h->nleaf + wpb - 1) / wpb, 148 * 8);
#define HPA(C) case C: k_hp_apply<C><<<grid, kHpThreads, smem, h->stream>>>(h->nleaf, h->lptr, h->kptr, h->ldofs, h->K, L.mlev, x, y, sign); break;
  switch (nch) {
    HPA(1) HPA(2) HPA(4) HPA(8) HPA(16) HPA(32)
    default: return fail(FCM_EINVAL, "fcm_hp: leaf with %d level DOFs exceeds the kernel limit", L.max_ml);
  }
#undef HPA
  h->launches++;
  return FCM_OK;
}

// y = b - A_l x  (into y; b may alias nothing)
int residual(fcm_hp* h, int l, const double* b, const double* x, double* y) {
  const int64_t n = h->lev[l].n;
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(y, b, n);
  h->launches++;
  return launch_apply(h, l, x, y, -1.0);
}

// The size classes run CONCURRENTLY: the tile-streamed large blocks on the main stream (one CTA
// per SM, ~150 KB of rings) and the packed small blocks on a side stream, whose CTAs fill the
// remaining threads of the same SMs (fork / join by events; parallel branches in the graph).
int launch_smooth(fcm_hp* h, int l, const double* r, double* x, double omega) {
  HpLevel& L = h->lev[l];
  const bool fork = L.cls.size() > 1;
  if (fork) {
    HCU(cudaEventRecord(h->ev_fork, h->stream));
    HCU(cudaStreamWaitEvent(h->stream2, h->ev_fork, 0));
  }
  for (size_t ci = 0; ci < L.cls.size(); ++ci) {
    const HpClass& c = L.cls[ci];
    cudaStream_t st = (fork && ci > 0) ? h->stream2 : h->stream;
    const int64_t nb = c.b1 - c.b0;
    if (nb <= 0) continue;
    const int grid = (int)std::min<int64_t>(nb, 148 * 16);
    const int mmax = (int)c.mmax;
    if (c.nt == -1) {
      const int ntm = (mmax + 31) / 32;
      const size_t smt = (size_t)kHpTileWarps * kHpStages * 1024 * 8 + kHpTileWarps * kHpStages * 8 + 2 * 32 * ntm * 8;
      const int gt = (int)std::min<int64_t>(nb, 148);
      k_hp_smooth_tiles<<<gt, kHpTileWarps * 32, smt, st>>>(c.b0, c.b1, L.bptr, L.bdofs, L.iptr, L.inv, r, x,
                                                             omega, ntm);
      h->launches++;
      continue;
    }
    const size_t smem = (size_t)2 * mmax * 8;
#define HPS(NW, C)                                                                                    \
  if (c.nt == NW && c.nch == C) {                                                                     \
    k_hp_smooth_sym<NW, C><<<grid, NW * 32, smem, st>>>(c.b0, c.b1, L.bptr, L.bdofs, L.iptr, L.inv, r, x,        \
                                                        omega, mmax);                                 \
  } else
    HPS(8, 8) HPS(8, 16)
    return fail(FCM_EINVAL, "fcm_hp: no smoother kernel for class (%d warps, %d chunks)", c.nt, c.nch);
#undef HPS
    h->launches++;
  }
  if (fork) {
    HCU(cudaEventRecord(h->ev_join, h->stream2));
    HCU(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  }
  return FCM_OK;
}

// setup temporaries: freed on every return path (error returns included)
struct DevTmp {
  std::vector<void*> p;
  template <class T>
  cudaError_t alloc(T** ptr, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, bytes);
    if (e == cudaSuccess) p.push_back(q);
    *ptr = (T*)q;
    return e;
  }
  ~DevTmp() {
    for (void* q : p) cudaFree(q);
  }
};

int smooth_kernel_attrs() {
#define HPA2(NW, C) \
  HCU(cudaFuncSetAttribute((const void*)k_hp_smooth_sym<NW, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kHpMaxBlock * 8));
  HPA2(8, 8) HPA2(8, 16)
#undef HPA2
  HCU(cudaFuncSetAttribute((const void*)k_hp_smooth_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kHpTileWarps * kHpStages * 1024 * 8 + kHpTileWarps * kHpStages * 8 + 2 * kHpTileMax * 8));
  return FCM_OK;
}

int dot(fcm_hp* h, const double* a, const double* b, int64_t n, double* dst) {
  k_hp_dot<<<kHpDotBlocks, kHpThreads, 0, h->stream>>>(a, b, n, h->part);
  k_hp_sum<<<1, kHpThreads, 0, h->stream>>>(h->part, kHpDotBlocks, dst);
  h->launches += 2;
  return FCM_OK;
}

// coarse solve on the last level: z = A_0^{-1} b (direct) or CG + undamped elementwise AS
int coarse_solve(fcm_hp* h, const double* b, double* z) {
  const int l = h->nlev - 1;
  HpLevel& L = h->lev[l];
  const int64_t n = L.n;
  if (h->coarse == FCM_COARSE_DIRECT) {
    k_hp_gemv<<<grid_for(n * 32), kHpThreads, 0, h->stream>>>(h->cinv, b, z, n, n);
    h->launches++;
    return FCM_OK;
  }
  // CG (R4): x0 = 0, stop at ||r|| < rtol ||r0||
  HpScal* s = h->cs;
  HCU(cudaMemsetAsync(z, 0, n * 8, h->stream));
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(h->c_r, b, n);
  HRC(dot(h, b, b, n, &s->rr0));
  HCU(cudaMemcpyAsync(h->h_pin, &s->rr0, 8, cudaMemcpyDeviceToHost, h->stream));
  HCU(cudaStreamSynchronize(h->stream));
  const double rr0 = h->h_pin[0];
  if (rr0 == 0.0) return FCM_OK;
  k_hp_set<<<1, 32, 0, h->stream>>>(s, 1);
  HCU(cudaMemsetAsync(h->c_z, 0, n * 8, h->stream));
  HRC(launch_smooth(h, l, h->c_r, h->c_z, 1.0));
  HRC(dot(h, h->c_r, h->c_z, n, &s->rz));
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(h->c_p, h->c_z, n);
  h->launches += 3;
  int it = 0;
  const double tol2 = h->coarse_rtol * h->coarse_rtol * rr0;
  while (it < h->coarse_maxit) {
    HCU(cudaMemsetAsync(h->c_q, 0, n * 8, h->stream));
    HRC(launch_apply(h, l, h->c_p, h->c_q, 1.0));
    HRC(dot(h, h->c_p, h->c_q, n, &s->pq));
    k_hp_cg_update<<<kHpDotBlocks, kHpThreads, 0, h->stream>>>(s, z, h->c_r, nullptr, h->c_p, h->c_q, n, h->part);
    k_hp_sum<<<1, kHpThreads, 0, h->stream>>>(h->part, kHpDotBlocks, &s->rr);
    h->launches += 2;
    HCU(cudaMemcpyAsync(h->h_pin, &s->rr, 8, cudaMemcpyDeviceToHost, h->stream));
    HCU(cudaStreamSynchronize(h->stream));
    ++it;
    if (!(h->h_pin[0] == h->h_pin[0])) return fail(FCM_EINDEF, "fcm_hp: NaN in the coarse CG");
    if (h->h_pin[0] < tol2) break;
    HCU(cudaMemsetAsync(h->c_z, 0, n * 8, h->stream));
    HRC(launch_smooth(h, l, h->c_r, h->c_z, 1.0));
    HRC(dot(h, h->c_r, h->c_z, n, &s->zr));
    k_hp_cg_p<<<grid_for(n), kHpThreads, 0, h->stream>>>(s, h->c_p, h->c_z, n);
    k_hp_set<<<1, 32, 0, h->stream>>>(s, 0);
    h->launches += 2;
  }
  h->coarse_iters += it;
  return FCM_OK;
}

// Algorithm 1 on level l: x_l = V(b_l) with x = 0 on entry, residual before every sweep (R1)
int vcycle_level(fcm_hp* h, int l, const double* b, double* x) {
  if (l == h->nlev - 1) return coarse_solve(h, b, x);
  HpLevel& L = h->lev[l];
  const int64_t n = L.n;
  HCU(cudaMemsetAsync(x, 0, n * 8, h->stream));
  for (int s = 0; s < h->n_pre; ++s) {
    if (s == 0) HRC(launch_smooth(h, l, b, x, L.omega));   // x = 0: r = b
    else {
      HRC(residual(h, l, b, x, L.r));
      HRC(launch_smooth(h, l, L.r, x, L.omega));
    }
  }
  HRC(residual(h, l, b, x, L.r));
  HpLevel& C = h->lev[l + 1];
  HRC(vcycle_level(h, l + 1, L.r, C.x));                    // b_{l+1} = prefix of r_l
  k_hp_add<<<grid_for(C.n), kHpThreads, 0, h->stream>>>(x, C.x, C.n);   // x += R^T e
  h->launches++;
  for (int s = 0; s < h->n_post; ++s) {
    HRC(residual(h, l, b, x, L.r));
    HRC(launch_smooth(h, l, L.r, x, L.omega));
  }
  return FCM_OK;
}

int vcycle(fcm_hp* h, const double* r, double* z) {
  h->vcycles++;
  if (h->coarse != FCM_COARSE_DIRECT || h->nlev == 1 || getenv_flag("FCM_HOST_LOOP")) return vcycle_level(h, 0, r, z);
  // static launch sequence (direct coarse solve): replay a captured graph, rebuilt when the
  // vectors change
  if (!h->vgraph || h->vg_r != r || h->vg_z != z) {
    if (h->vgraph) { cudaGraphExecDestroy(h->vgraph); h->vgraph = nullptr; }
    cudaGraph_t g;
    HCU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t l0 = h->launches;
    const int rc = vcycle_level(h, 0, r, z);
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (rc < 0) {
      if (e == cudaSuccess) cudaGraphDestroy(g);
      return rc;
    }
    HCU(e);
    HCU(cudaGraphInstantiate(&h->vgraph, g, 0));
    cudaGraphDestroy(g);
    h->vg_r = r;
    h->vg_z = z;
    h->vg_count = h->launches - l0;
    h->launches = l0;
  }
  HCU(cudaGraphLaunch(h->vgraph, h->stream));
  h->launches += h->vg_count;
  return FCM_OK;
}

// ---- setup ------------------------------------------------------------------------------------
struct BlockSet {
  std::vector<std::vector<int32_t>> dofs;            // level indices, ascending
  std::vector<std::vector<int64_t>> leaves;          // contributing leaves
};

// Schwarz blocks of level l (reading R26): the level DOFs nonzero on one base element
// (elementwise) or on the 2^d base elements around a base vertex (patchwise); identical sets once
BlockSet build_blocks(int dim, int n, int block, int64_t nleaf, const std::vector<int64_t>& lptr,
                      const std::vector<int32_t>& ldofs, const std::vector<int32_t>& info,
                      const std::vector<int32_t>& mlev) {
  int64_t nbase = 1;
  for (int a = 0; a < dim; ++a) nbase *= n;
  std::vector<std::vector<int64_t>> base_leaves(nbase);
  for (int64_t L = 0; L < nleaf; ++L)
    if (mlev[L] > 0) base_leaves[info[L * 5 + 4]].push_back(L);
  std::vector<std::vector<int64_t>> groups;   // base elements per block
  if (block == FCM_BLOCK_ELEMENT) {
    for (int64_t be = 0; be < nbase; ++be) groups.push_back({be});
  } else {
    const int nv = n + 1;
    const int nz = dim == 3 ? nv : 1;
    for (int vz = 0; vz < nz; ++vz)
      for (int vy = 0; vy < nv; ++vy)
        for (int vx = 0; vx < nv; ++vx) {
          std::vector<int64_t> g;
          for (int c = 0; c < (1 << dim); ++c) {
            const int ex = vx - 1 + (c & 1), ey = vy - 1 + ((c >> 1) & 1), ez = dim == 3 ? vz - 1 + ((c >> 2) & 1) : 0;
            if (ex < 0 || ex >= n || ey < 0 || ey >= n || ez < 0 || (dim == 3 && ez >= n)) continue;
            g.push_back(((int64_t)ez * n + ey) * n + ex);
          }
          groups.push_back(g);
        }
  }
  // DOF -> leaves incidence of the level (a block's matrix needs every leaf holding its DOFs,
  // including leaves of neighbouring base elements: A_i is the ASSEMBLED submatrix, R11)
  int32_t nd = 0;
  for (int64_t L = 0; L < nleaf; ++L)
    for (int a = 0; a < mlev[L]; ++a) nd = std::max(nd, ldofs[lptr[L] + a] + 1);
  std::vector<int64_t> iptr(nd + 1, 0);
  for (int64_t L = 0; L < nleaf; ++L)
    for (int a = 0; a < mlev[L]; ++a) iptr[ldofs[lptr[L] + a] + 1]++;
  for (int32_t i = 0; i < nd; ++i) iptr[i + 1] += iptr[i];
  std::vector<int64_t> inc(iptr[nd]), fill(iptr.begin(), iptr.end() - 1);
  for (int64_t L = 0; L < nleaf; ++L)
    for (int a = 0; a < mlev[L]; ++a) inc[fill[ldofs[lptr[L] + a]]++] = L;
  BlockSet B;
  std::map<std::vector<int32_t>, int64_t> seen;
  for (const auto& g : groups) {
    std::vector<int32_t> d;
    for (int64_t be : g)
      for (int64_t L : base_leaves[be])
        for (int a = 0; a < mlev[L]; ++a) d.push_back(ldofs[lptr[L] + a]);
    if (d.empty()) continue;
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    if (seen.count(d)) continue;
    seen.emplace(d, (int64_t)B.dofs.size());
    std::vector<int64_t> lv;
    for (int32_t g2 : d) lv.insert(lv.end(), inc.begin() + iptr[g2], inc.begin() + iptr[g2 + 1]);
    std::sort(lv.begin(), lv.end());
    lv.erase(std::unique(lv.begin(), lv.end()), lv.end());
    B.dofs.push_back(std::move(d));
    B.leaves.push_back(std::move(lv));
  }
  return B;
}

// launch class of a block of m DOFs: 8 warps per CTA; register chunks MAXCH = 8 for m <= 256
// (one launch for all small and medium blocks, the instance dispatches per block), 16 for the
// large ones (panel width 512, panel loop above)
HpClass class_of(int m) {
  if (m > kHpTileMin) return {0, 0, -1, 0, m};   // tile-streamed (k_hp_smooth_tiles)
  return {0, 0, 8, 8, m};
}

int setup_level_blocks(fcm_hp* h, int l, int block, double omega, const std::vector<int64_t>& lptr,
                       const std::vector<int64_t>& kptr, const std::vector<int32_t>& ldofs,
                       const std::vector<int32_t>& info, const std::vector<int32_t>& mlev) {
  HpLevel& L = h->lev[l];
  L.omega = omega;
  BlockSet B = build_blocks(h->dim, h->n, block, h->nleaf, lptr, ldofs, info, mlev);
  const int64_t nb = (int64_t)B.dofs.size();
  // order by size (stable): one launch per size class
  std::vector<int64_t> ord(nb);
  for (int64_t i = 0; i < nb; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return B.dofs[a].size() > B.dofs[b].size(); });
  std::vector<int64_t> bptr(nb + 1, 0), iptr(nb + 1, 0);
  std::vector<int32_t> bd;
  for (int64_t k = 0; k < nb; ++k) {
    const auto& d = B.dofs[ord[k]];
    if ((int)d.size() > kHpMaxBlock)
      return fail(FCM_EINVAL, "fcm_hp: Schwarz block with %zu DOFs on level %d exceeds %d", d.size(), l, kHpMaxBlock);
    bptr[k + 1] = bptr[k] + (int64_t)d.size();
    const int64_t md = (int64_t)d.size();   // lower-packed, or tile-packed for the large blocks
    iptr[k + 1] = iptr[k] + (md > kHpTileMin ? hp_tile_pack_size((int)((md + 31) / 32)) : md * (md + 1) / 2);
    bd.insert(bd.end(), d.begin(), d.end());
  }
  L.nblk = nb;
  L.n_bdofs = bptr[nb];
  L.n_inv = iptr[nb];
  L.has_blocks = true;
  L.cls.clear();
  for (int64_t k = 0; k < nb;) {
    HpClass c = class_of((int)(bptr[k + 1] - bptr[k]));
    int64_t e = k;
    while (e < nb) {
      HpClass c2 = class_of((int)(bptr[e + 1] - bptr[e]));
      if (c2.nt != c.nt || c2.nch != c.nch) break;
      ++e;
    }
    c.b0 = k;
    c.b1 = e;
    c.mmax = bptr[k + 1] - bptr[k];   // blocks are sorted by descending size
    L.cls.push_back(c);
    k = e;
  }
  HRC(h->alloc(&L.bptr, nb + 1));
  HRC(h->alloc(&L.bdofs, L.n_bdofs));
  HRC(h->alloc(&L.iptr, nb + 1));
  HRC(h->alloc(&L.inv, L.n_inv));
  HCU(cudaMemcpyAsync(L.bptr, bptr.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(L.bdofs, bd.data(), bd.size() * 4, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(L.iptr, iptr.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaStreamSynchronize(h->stream));
  // contributions (block, leaf, map) in block order
  std::vector<int64_t> cptr(nb + 1, 0), cleaf, cmap;
  std::vector<int32_t> amap;
  for (int64_t k = 0; k < nb; ++k) {
    const auto& d = B.dofs[ord[k]];
    for (int64_t Lf : B.leaves[ord[k]]) {
      cleaf.push_back(Lf);
      cmap.push_back((int64_t)amap.size());
      for (int a = 0; a < mlev[Lf]; ++a) {
        const int32_t g = ldofs[lptr[Lf] + a];
        auto it = std::lower_bound(d.begin(), d.end(), g);
        amap.push_back(it != d.end() && *it == g ? (int32_t)(it - d.begin()) : -1);
      }
    }
    cptr[k + 1] = (int64_t)cleaf.size();
  }
  int64_t *d_cleaf = nullptr, *d_cmap = nullptr, *d_cptr = nullptr, *d_off = nullptr;
  int32_t *d_amap = nullptr, *d_bsize = nullptr, *d_status = nullptr;
  double *W = nullptr, *d_eq = nullptr;
  DevTmp tmp;
  HCU(tmp.alloc(&d_cleaf, std::max<size_t>(cleaf.size(), 1) * 8));
  HCU(tmp.alloc(&d_cmap, std::max<size_t>(cmap.size(), 1) * 8));
  HCU(tmp.alloc(&d_amap, std::max<size_t>(amap.size(), 1) * 4));
  HCU(cudaMemcpyAsync(d_cleaf, cleaf.data(), cleaf.size() * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(d_cmap, cmap.data(), cmap.size() * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(d_amap, amap.data(), amap.size() * 4, cudaMemcpyHostToDevice, h->stream));
  int rc = FCM_OK;
  // chunks of equal padded size MP, workspace <= 2 GiB
  const size_t wsz = (size_t)2 << 30;
  HCU(tmp.alloc(&W, wsz));
  int64_t maxchunk = 1;
  for (int64_t k = 0; k < nb;) {
    const int m0 = (int)(bptr[k + 1] - bptr[k]);
    const int MP = 32 * ((m0 + 31) / 32);
    int64_t e = k;
    const int64_t cap = std::max<int64_t>(1, (int64_t)(wsz / ((size_t)MP * MP * 8)));
    while (e < nb && e - k < cap && 32 * ((bptr[e + 1] - bptr[e] + 31) / 32) == MP) ++e;
    maxchunk = std::max(maxchunk, e - k);
    k = e;
  }
  HCU(tmp.alloc(&d_cptr, (maxchunk + 1) * 8));
  HCU(tmp.alloc(&d_off, maxchunk * 8));
  HCU(tmp.alloc(&d_bsize, maxchunk * 4));
  HCU(tmp.alloc(&d_status, maxchunk * 4));
  HCU(tmp.alloc(&d_eq, (size_t)maxchunk * 32 * ((kHpMaxBlock + 31) / 32) * 8));
  std::vector<int> status(maxchunk);
  for (int64_t k = 0; k < nb && rc == FCM_OK;) {
    const int m0 = (int)(bptr[k + 1] - bptr[k]);
    const int MP = 32 * ((m0 + 31) / 32);
    const int nt = MP / 32;
    int64_t e = k;
    const int64_t cap = std::max<int64_t>(1, (int64_t)(wsz / ((size_t)MP * MP * 8)));
    while (e < nb && e - k < cap && 32 * ((bptr[e + 1] - bptr[e] + 31) / 32) == MP) ++e;
    const int64_t nc = e - k;
    std::vector<int64_t> lcptr(nc + 1), off(nc);
    std::vector<int32_t> bs(nc);
    for (int64_t i = 0; i < nc; ++i) {
      lcptr[i] = cptr[k + i];
      off[i] = iptr[k + i];
      bs[i] = (int32_t)(bptr[k + i + 1] - bptr[k + i]);
    }
    lcptr[nc] = cptr[e];
    HCU(cudaMemcpyAsync(d_cptr, lcptr.data(), (nc + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    HCU(cudaMemcpyAsync(d_off, off.data(), nc * 8, cudaMemcpyHostToDevice, h->stream));
    HCU(cudaMemcpyAsync(d_bsize, bs.data(), nc * 4, cudaMemcpyHostToDevice, h->stream));
    HCU(cudaMemsetAsync(W, 0, (size_t)nc * MP * MP * 8, h->stream));
    HCU(cudaMemsetAsync(d_status, 0, nc * 4, h->stream));
    k_hp_asm<<<(unsigned)nc, 256, 0, h->stream>>>(W, MP, d_cptr, d_cleaf, d_cmap, d_amap, h->kptr, h->lptr, L.mlev, h->K, d_bsize);
    k_equil<<<(unsigned)nc, 256, MP * 8, h->stream>>>(W, MP, d_eq, 0);
    const int nt64 = (MP + 63) / 64;
    for (int t = 0; t < nt; ++t) {
      k_gj_pivot<<<(unsigned)nc, 256, 0, h->stream>>>(W, MP, t, d_status);
      if (nt > 1) {
        k_gj_row<<<dim3(nt - 1, (unsigned)nc), 256, 0, h->stream>>>(W, MP, t);
        k_gj_update<<<dim3(nt64 * nt64, (unsigned)nc), 256, 0, h->stream>>>(W, MP, t);
        k_gj_col<<<dim3(nt - 1, (unsigned)nc), 256, 0, h->stream>>>(W, MP, t);
      }
    }
    k_equil<<<(unsigned)nc, 256, MP * 8, h->stream>>>(W, MP, d_eq, 1);
    if (MP > kHpTileMin) {   // the chunk holds blocks of one padded size MP: all tiled or all packed
      const int ntm = MP / 32;
      k_hp_pack_tiles<<<dim3(ntm * (ntm + 1) / 2, (unsigned)nc), 256, 0, h->stream>>>(W, MP, d_off, d_bsize, L.inv);
    } else {
      k_hp_extract<<<(unsigned)nc, 256, 0, h->stream>>>(W, MP, d_off, d_bsize, L.inv);
    }
    HCU(cudaGetLastError());
    HCU(cudaMemcpyAsync(status.data(), d_status, nc * 4, cudaMemcpyDeviceToHost, h->stream));
    HCU(cudaStreamSynchronize(h->stream));
    for (int64_t i = 0; i < nc; ++i)
      if (status[i]) {
        rc = fail(FCM_ESINGULAR, "fcm_hp: singular Schwarz block %lld (%d DOFs) on level %d", (long long)(k + i), bs[i], l);
        break;
      }
    k = e;
  }
  HCU(cudaStreamSynchronize(h->stream));   // temporaries are freed by tmp
  return rc;
}

int setup_direct(fcm_hp* h, const std::vector<int32_t>& mlev) {
  const int l = h->nlev - 1;
  const int64_t n = h->lev[l].n;
  if (n > 40000) return fail(FCM_EINVAL, "fcm_hp: direct coarse solve of %lld DOFs (limit 40000: 12.8 GB dense inverse; use FCM_COARSE_AS_PCG)", (long long)n);
  const int64_t MP = 32 * ((n + 31) / 32);
  double *W = nullptr, *d_eq = nullptr;
  int* d_status = nullptr;
  DevTmp tmp;
  HCU(tmp.alloc(&W, (size_t)MP * MP * 8));
  HCU(tmp.alloc(&d_eq, (size_t)MP * 8));
  HCU(tmp.alloc(&d_status, 4));
  HCU(cudaMemsetAsync(W, 0, (size_t)MP * MP * 8, h->stream));
  HCU(cudaMemsetAsync(d_status, 0, 4, h->stream));
  k_hp_asm_dense<<<grid_for(h->nleaf * 32), kHpThreads, 0, h->stream>>>(W, MP, h->nleaf, h->lptr, h->kptr, h->ldofs, h->K,
                                                                        h->lev[l].mlev);
  k_hp_identity_pad<<<1, 256, 0, h->stream>>>(W, MP, n);
  k_hp_equil_d<<<grid_for(MP), kHpThreads, 0, h->stream>>>(W, MP, d_eq);
  k_hp_equil_scale<<<(unsigned)std::min<int64_t>(MP, 148 * 16), 256, 0, h->stream>>>(W, MP, d_eq);
  const int nt = (int)(MP / 32), nt64 = (int)((MP + 63) / 64);
  for (int t = 0; t < nt; ++t) {
    k_gj_pivot<<<1, 256, 0, h->stream>>>(W, (int)MP, t, d_status);
    if (nt > 1) {
      k_gj_row<<<dim3(nt - 1, 1), 256, 0, h->stream>>>(W, (int)MP, t);
      k_gj_update<<<dim3(nt64 * nt64, 1), 256, 0, h->stream>>>(W, (int)MP, t);
      k_gj_col<<<dim3(nt - 1, 1), 256, 0, h->stream>>>(W, (int)MP, t);
    }
  }
  k_hp_equil_scale<<<(unsigned)std::min<int64_t>(MP, 148 * 16), 256, 0, h->stream>>>(W, MP, d_eq);
  HRC(h->alloc(&h->cinv, n * n));
  HCU(cudaMemcpy2DAsync(h->cinv, n * 8, W, MP * 8, n * 8, n, cudaMemcpyDeviceToDevice, h->stream));
  int st = 0;
  HCU(cudaMemcpyAsync(&st, d_status, 4, cudaMemcpyDeviceToHost, h->stream));
  HCU(cudaStreamSynchronize(h->stream));
  (void)mlev;
  if (st) return fail(FCM_ESINGULAR, "fcm_hp: the coarse matrix (%lld DOFs) is not SPD", (long long)n);
  return FCM_OK;
}

bool check_vec(const void* p) { return p != nullptr; }

// stream-ordered against the caller's stream: work enqueued on the library stream after the
// caller's pending work, and the caller's stream waits for it on return
int enter(fcm_hp* h) {
  HCU(cudaEventRecord(h->ev_in, h->ustream));
  HCU(cudaStreamWaitEvent(h->stream, h->ev_in, 0));
  return FCM_OK;
}
int leave(fcm_hp* h, int rc) {
  if (cudaEventRecord(h->ev_out, h->stream) == cudaSuccess) cudaStreamWaitEvent(h->ustream, h->ev_out, 0);
  return rc;
}

}  // namespace

extern "C" int fcm_hp_setup(const fcm_hp_disc* d, const fcm_params* prm, fcm_hp** out) {
  clear_error();
  if (!d || !prm || !out) return fail(FCM_EINVAL, "fcm_hp_setup: NULL argument");
  if (!(prm->omega > 0) || prm->n_pre < 0 || prm->n_post < 0 ||
      (prm->block != FCM_BLOCK_ELEMENT && prm->block != FCM_BLOCK_PATCH) ||
      (prm->coarse != FCM_COARSE_DIRECT && prm->coarse != FCM_COARSE_AS_PCG) || prm->coarse_maxit < 0)
    return fail(FCM_EINVAL, "fcm_hp_setup: invalid parameters (coarse must be DIRECT or AS_PCG)");
  int dim, n, p, n_f;
  int64_t ndof;
  std::vector<int64_t> level_n;
  const std::vector<int64_t>*lptr, *kptr;
  const std::vector<int32_t>*ldofs, *info;
  const std::vector<double>* K;
  hp_disc_view(d, &dim, &n, &p, &n_f, &ndof, &level_n, &lptr, &kptr, &ldofs, &K, &info);
  if (ndof <= 0 || level_n.empty() || level_n.back() <= 0) return fail(FCM_EINVAL, "fcm_hp_setup: empty system");
  HRC(smooth_kernel_attrs());
  std::unique_ptr<fcm_hp> h(new fcm_hp());
  h->dim = dim; h->n = n; h->p = p; h->n_f = n_f; h->ndof = ndof;
  h->nleaf = (int64_t)lptr->size() - 1;
  h->nlev = (int)level_n.size();
  h->ustream = (cudaStream_t)prm->stream;
  HCU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  HCU(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  HCU(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
  HCU(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
  HCU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  HCU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  HRC(enter(h.get()));
  h->coarse = prm->coarse;
  h->coarse_rtol = prm->coarse_rtol;
  h->coarse_maxit = prm->coarse_maxit;
  h->n_pre = prm->n_pre;
  h->n_post = prm->n_post;
  HRC(h->alloc(&h->lptr, h->nleaf + 1));
  HRC(h->alloc(&h->kptr, h->nleaf + 1));
  HRC(h->alloc(&h->ldofs, (int64_t)ldofs->size()));
  HRC(h->alloc(&h->K, (int64_t)K->size()));
  HCU(cudaMemcpyAsync(h->lptr, lptr->data(), lptr->size() * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(h->kptr, kptr->data(), kptr->size() * 8, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(h->ldofs, ldofs->data(), ldofs->size() * 4, cudaMemcpyHostToDevice, h->stream));
  HCU(cudaMemcpyAsync(h->K, K->data(), K->size() * 8, cudaMemcpyHostToDevice, h->stream));
  h->lev.resize(h->nlev);
  std::vector<std::vector<int32_t>> mlev(h->nlev, std::vector<int32_t>(h->nleaf));
  for (int l = 0; l < h->nlev; ++l) {
    HpLevel& L = h->lev[l];
    L.n = level_n[l];
    for (int64_t Lf = 0; Lf < h->nleaf; ++Lf) {
      const int32_t* b = ldofs->data() + (*lptr)[Lf];
      const int32_t* e = ldofs->data() + (*lptr)[Lf + 1];
      mlev[l][Lf] = (int32_t)(std::lower_bound(b, e, (int32_t)L.n) - b);
      L.max_ml = std::max(L.max_ml, mlev[l][Lf]);
    }
    if (L.max_ml > 32 * 32) return fail(FCM_EINVAL, "fcm_hp_setup: a leaf carries %d DOFs (limit 1024)", L.max_ml);
    HRC(h->alloc(&L.mlev, h->nleaf));
    HCU(cudaMemcpyAsync(L.mlev, mlev[l].data(), h->nleaf * 4, cudaMemcpyHostToDevice, h->stream));
    HRC(h->alloc(&L.x, L.n));
    HRC(h->alloc(&L.r, L.n));
  }
  HCU(cudaStreamSynchronize(h->stream));
  for (int l = 0; l + 1 < h->nlev; ++l)
    HRC(setup_level_blocks(h.get(), l, prm->block, prm->omega, *lptr, *kptr, *ldofs, *info, mlev[l]));
  const int lc = h->nlev - 1;
  if (h->nlev == 1 || prm->coarse == FCM_COARSE_DIRECT) {
    HRC(setup_direct(h.get(), mlev[lc]));
  } else {
    HRC(setup_level_blocks(h.get(), lc, FCM_BLOCK_ELEMENT, 1.0, *lptr, *kptr, *ldofs, *info, mlev[lc]));
    const int64_t nc = h->lev[lc].n;
    HRC(h->alloc(&h->c_r, nc));
    HRC(h->alloc(&h->c_p, nc));
    HRC(h->alloc(&h->c_q, nc));
    HRC(h->alloc(&h->c_z, nc));
  }
  if (h->nlev == 1) h->coarse = FCM_COARSE_DIRECT;
  for (double** v : {&h->w_p, &h->w_q, &h->w_z, &h->w_ro, &h->w_r}) HRC(h->alloc(v, ndof));
  HRC(h->alloc(&h->part, kHpDotBlocks));
  HRC(h->alloc(&h->s, 1));
  HRC(h->alloc(&h->cs, 1));
  HCU(cudaMallocHost(&h->h_pin, 64));
  HCU(cudaStreamSynchronize(h->stream));
  leave(h.get(), FCM_OK);
  *out = h.release();
  return FCM_OK;
}

extern "C" int fcm_hp_destroy(fcm_hp* h) {
  if (h) cudaStreamSynchronize(h->stream);
  delete h;
  return FCM_OK;
}

extern "C" int fcm_hp_apply(fcm_hp* h, int32_t level, const double* x, double* y) {
  clear_error();
  if (!h || level < 0 || level >= h->nlev || !check_vec(x) || !check_vec(y))
    return fail(FCM_EINVAL, "fcm_hp_apply: invalid argument");
  HRC(enter(h));
  HCU(cudaMemsetAsync(y, 0, h->lev[level].n * 8, h->stream));
  HRC(launch_apply(h, level, x, y, 1.0));
  HCU(cudaGetLastError());
  return leave(h, FCM_OK);
}

extern "C" int fcm_hp_smooth(fcm_hp* h, int32_t level, const double* r, double* x) {
  clear_error();
  if (!h || level < 0 || level >= h->nlev || !h->lev[level].has_blocks || !check_vec(r) || !check_vec(x))
    return fail(FCM_EINVAL, "fcm_hp_smooth: invalid argument (level %d has no smoother)", level);
  HRC(enter(h));
  HRC(launch_smooth(h, level, r, x, h->lev[level].omega));
  HCU(cudaGetLastError());
  return leave(h, FCM_OK);
}

extern "C" int fcm_hp_time_smooth(fcm_hp* h, int32_t level, const double* r, double* x, int32_t reps, float* ms) {
  clear_error();
  if (!h || level < 0 || level >= h->nlev || !h->lev[level].has_blocks || !check_vec(r) || !check_vec(x) || reps < 1 ||
      !ms)
    return fail(FCM_EINVAL, "fcm_hp_time_smooth: invalid argument");
  HRC(enter(h));
  cudaEvent_t e0, e1;
  HCU(cudaEventCreate(&e0));
  HCU(cudaEventCreate(&e1));
  int rc = launch_smooth(h, level, r, x, h->lev[level].omega);   // warm-up
  HCU(cudaEventRecord(e0, h->stream));
  for (int i = 0; i < reps && rc >= 0; ++i) rc = launch_smooth(h, level, r, x, h->lev[level].omega);
  HCU(cudaEventRecord(e1, h->stream));
  HCU(cudaEventSynchronize(e1));
  float t = 0.f;
  HCU(cudaEventElapsedTime(&t, e0, e1));
  *ms = t / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return leave(h, rc);
}

extern "C" int fcm_hp_vcycle(fcm_hp* h, const double* r, double* z) {
  clear_error();
  if (!h || !check_vec(r) || !check_vec(z)) return fail(FCM_EINVAL, "fcm_hp_vcycle: invalid argument");
  HRC(enter(h));
  HRC(vcycle(h, r, z));
  HCU(cudaGetLastError());
  return leave(h, FCM_OK);
}

static int hp_pcg_body(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit, int32_t* iters,
                       double* hist) {
  const int64_t n = h->ndof;
  HpScal* s = h->s;
  h->coarse_iters = 0;
  h->vcycles = 0;
  HCU(cudaMemsetAsync(x, 0, n * 8, h->stream));
  if (iters) *iters = 0;
  HRC(dot(h, b, b, n, &s->bb));
  HCU(cudaMemcpyAsync(h->h_pin, &s->bb, 8, cudaMemcpyDeviceToHost, h->stream));
  HCU(cudaStreamSynchronize(h->stream));
  const double bb = h->h_pin[0];
  if (hist) hist[0] = bb == 0.0 ? 0.0 : 1.0;
  if (bb == 0.0 || maxit == 0) return FCM_OK;
  double* r = h->w_r;
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(r, b, n);
  h->launches++;
  HRC(vcycle(h, r, h->w_z));
  HRC(dot(h, r, h->w_z, n, &s->rz));
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(h->w_p, h->w_z, n);
  h->launches++;
  int it = 0, rc = FCM_NOT_CONVERGED;
  while (it < maxit) {
    HCU(cudaMemsetAsync(h->w_q, 0, n * 8, h->stream));
    HRC(launch_apply(h, 0, h->w_p, h->w_q, 1.0));
    HRC(dot(h, h->w_p, h->w_q, n, &s->pq));
    k_hp_cg_update<<<kHpDotBlocks, kHpThreads, 0, h->stream>>>(s, x, r, h->w_ro, h->w_p, h->w_q, n, h->part);
    k_hp_sum<<<1, kHpThreads, 0, h->stream>>>(h->part, kHpDotBlocks, &s->rr);
    h->launches += 2;
    HCU(cudaMemcpyAsync(h->h_pin, s, 3 * 8, cudaMemcpyDeviceToHost, h->stream));   // rz, pq, rr
    HCU(cudaStreamSynchronize(h->stream));
    ++it;
    const double pq = h->h_pin[1], rel2 = h->h_pin[2] / bb;
    if (hist) hist[it] = std::sqrt(rel2);
    if (!(pq > 0)) { rc = fail(FCM_EINDEF, "fcm_hp_pcg_solve: p^T A p = %g at iteration %d", pq, it); break; }
    if (rel2 < rtol * rtol) { rc = FCM_OK; break; }
    if (it >= maxit) break;
    HRC(vcycle(h, r, h->w_z));
    HRC(dot(h, h->w_z, r, n, &s->zr));
    HRC(dot(h, h->w_z, h->w_ro, n, &s->zro));
    k_hp_cg_p<<<grid_for(n), kHpThreads, 0, h->stream>>>(s, h->w_p, h->w_z, n);
    k_hp_set<<<1, 32, 0, h->stream>>>(s, 0);
    h->launches += 2;
  }
  if (iters) *iters = it;
  HCU(cudaGetLastError());
  return rc;
}

extern "C" int fcm_hp_pcg_solve(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit, int32_t* iters,
                                double* hist) {
  clear_error();
  if (!h || !check_vec(b) || !check_vec(x) || !(rtol > 0) || maxit < 0)
    return fail(FCM_EINVAL, "fcm_hp_pcg_solve: invalid argument");
  HRC(enter(h));
  return leave(h, hp_pcg_body(h, b, x, rtol, maxit, iters, hist));   // the caller's stream joins on every path
}

// stand-alone hp-multigrid: x_i = x_{i-1} + V(b - A x_{i-1}); one 8-byte D2H per cycle
static int hp_mg_body(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit, int32_t* iters,
                      double* hist) {
  const int64_t n = h->ndof;
  HpScal* s = h->s;
  h->coarse_iters = 0;
  h->vcycles = 0;
  HCU(cudaMemsetAsync(x, 0, n * 8, h->stream));
  if (iters) *iters = 0;
  HRC(dot(h, b, b, n, &s->bb));
  HCU(cudaMemcpyAsync(h->h_pin, &s->bb, 8, cudaMemcpyDeviceToHost, h->stream));
  HCU(cudaStreamSynchronize(h->stream));
  const double bb = h->h_pin[0];
  if (hist) hist[0] = bb == 0.0 ? 0.0 : 1.0;
  if (bb == 0.0 || maxit == 0) return FCM_OK;
  double* r = h->w_r;
  k_hp_copy<<<grid_for(n), kHpThreads, 0, h->stream>>>(r, b, n);
  h->launches++;
  int it = 0, rc = FCM_NOT_CONVERGED;
  while (it < maxit) {
    HRC(vcycle(h, r, h->w_z));
    k_hp_add<<<grid_for(n), kHpThreads, 0, h->stream>>>(x, h->w_z, n);   // x += V(r)
    h->launches++;
    HRC(residual(h, 0, b, x, r));                                          // r = b - A x
    HRC(dot(h, r, r, n, &s->rr));
    HCU(cudaMemcpyAsync(h->h_pin, &s->rr, 8, cudaMemcpyDeviceToHost, h->stream));
    HCU(cudaStreamSynchronize(h->stream));
    ++it;
    const double rel2 = h->h_pin[0] / bb;
    if (hist) hist[it] = std::sqrt(rel2);
    if (!(rel2 == rel2)) { rc = fail(FCM_EINDEF, "fcm_hp_mg_solve: NaN residual at cycle %d", it); break; }
    if (rel2 < rtol * rtol) { rc = FCM_OK; break; }
  }
  if (iters) *iters = it;
  HCU(cudaGetLastError());
  return rc;
}

extern "C" int fcm_hp_mg_solve(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit, int32_t* iters,
                               double* hist) {
  clear_error();
  if (!h || !check_vec(b) || !check_vec(x) || !(rtol > 0) || maxit < 0)
    return fail(FCM_EINVAL, "fcm_hp_mg_solve: invalid argument");
  HRC(enter(h));
  return leave(h, hp_mg_body(h, b, x, rtol, maxit, iters, hist));
}

extern "C" int fcm_hp_export_blocks(const fcm_hp* h, int32_t level, int64_t* n_blocks, int64_t* dof_entries,
                                    int64_t* inv_entries, int64_t* ptr, int32_t* dofs, double* inv) {
  clear_error();
  if (!h || level < 0 || level >= h->nlev) return fail(FCM_EINVAL, "fcm_hp_export_blocks: invalid argument");
  const HpLevel& L = h->lev[level];
  const bool direct = level == h->nlev - 1 && h->cinv;
  if (!L.has_blocks && !direct) return fail(FCM_EINVAL, "fcm_hp_export_blocks: level %d has no blocks", level);
  const int64_t nb = direct ? 1 : L.nblk;
  const int64_t nd = direct ? L.n : L.n_bdofs;
  int64_t ni = direct ? L.n * L.n : 0;
  std::vector<int64_t> hptr;
  HCU(cudaStreamSynchronize(h->stream));
  if (!direct) {   // full m x m per block in the export (the device keeps them lower-packed)
    hptr.resize(nb + 1);
    HCU(cudaMemcpy(hptr.data(), L.bptr, (nb + 1) * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < nb; ++i) ni += (hptr[i + 1] - hptr[i]) * (hptr[i + 1] - hptr[i]);
  }
  if (n_blocks) *n_blocks = nb;
  if (dof_entries) *dof_entries = nd;
  if (inv_entries) *inv_entries = ni;
  if (!ptr && !dofs && !inv) return FCM_OK;
  if (direct) {
    if (ptr) { ptr[0] = 0; ptr[1] = L.n; }
    if (dofs) for (int64_t i = 0; i < L.n; ++i) dofs[i] = (int32_t)i;
    HCU(cudaStreamSynchronize(h->stream));
    if (inv) HCU(cudaMemcpy(inv, h->cinv, ni * 8, cudaMemcpyDeviceToHost));
    return FCM_OK;
  }
  HCU(cudaStreamSynchronize(h->stream));
  if (ptr) HCU(cudaMemcpy(ptr, L.bptr, (nb + 1) * 8, cudaMemcpyDeviceToHost));
  if (dofs) HCU(cudaMemcpy(dofs, L.bdofs, nd * 4, cudaMemcpyDeviceToHost));
  if (inv) {
    std::vector<double> pk(L.n_inv);
    HCU(cudaMemcpy(pk.data(), L.inv, L.n_inv * 8, cudaMemcpyDeviceToHost));
    int64_t po = 0, fo = 0;
    for (int64_t i = 0; i < nb; ++i) {
      const int64_t m = hptr[i + 1] - hptr[i];
      const bool tiled = m > kHpTileMin;
      for (int64_t b = 0; b < m; ++b)
        for (int64_t a = 0; a <= b; ++a) {
          double v;
          if (!tiled) {
            v = pk[po + b * (b + 1) / 2 + a];
          } else {
            const int I = (int)(b / 32), J = (int)(a / 32), rr = (int)(b % 32), cc = (int)(a % 32);
            v = pk[po + hp_tile_off(I, J) + (I == J ? rr * (rr + 1) / 2 + cc : rr * 32 + cc)];
          }
          inv[fo + b * m + a] = v;
          inv[fo + a * m + b] = v;
        }
      po += tiled ? hp_tile_pack_size((int)((m + 31) / 32)) : m * (m + 1) / 2;
      fo += m * m;
    }
  }
  return FCM_OK;
}

extern "C" int fcm_hp_stats(const fcm_hp* h, int64_t* launches, int64_t* coarse_iters_total, int64_t* vcycles) {
  clear_error();
  if (!h) return fail(FCM_EINVAL, "fcm_hp_stats: NULL handle");
  if (launches) *launches = h->launches;
  if (coarse_iters_total) *coarse_iters_total = h->coarse_iters;
  if (vcycles) *vcycles = h->vcycles;
  return FCM_OK;
}
