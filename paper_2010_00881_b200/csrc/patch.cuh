// patch.cuh -- patchwise additive Schwarz at scale (config 3: PAPER.md:259 patchwise blocks,
// Table 1 P:316-320 m_max = (2p+1)^d, Eq. AdditiveSchwarz, block inversion P:326).
//
//  * INDIVIDUAL (irregular) patch inverses are stored TILE-PACKED SYMMETRIC: the lower triangle
//    of 32x32 tiles, row-major over tile rows; off-diagonal tiles full (1024 doubles, row-major),
//    diagonal tiles as packed lower triangles (528 doubles).  729-slot patches: 271,216 doubles
//    (+1.9 % over m(m+1)/2).  k_patch_irr streams them with 1D bulk copies (cp.async.bulk into a
//    per-warp ring of shared-memory stages, mbarrier completion): per tile a warp reads the 32
//    rows (lane = column), accumulates the transposed product in a register and the row
//    product with one butterfly reduce-scatter (31 shuffles per tile).
//  * REGULAR patches (every cell of the 4^d neighbourhood uncut and of one kind) of a tensor
//    Poisson level are applied by FAST DIAGONALISATION: A_i = s sum_g (x)_a (K|M)_a restricted
//    to the patch's per-axis slot sets, so A_i^{-1} = (S_z x S_y x S_x) D^{-1} (...)^T with the
//    1D generalised eigenvectors S_a^T M_a S_a = I, S_a^T K_a S_a = Lambda_a (setup, host) --
//    6 one-axis contractions of (2q+1)^3 values instead of a (2q+1)^3-square GEMV.
//  * SETUP: batched cell-loop assembly of A_i into a full workspace (ld = MP, multiple of 32),
//    batched blocked Gauss-Jordan inversion (32-wide pivot blocks; the trailing rank-32 update is
//    a batched register-blocked DFMA GEMM), then packing into tiles (symmetrised).
#pragma once
#include <cstdint>

#include "cellop.cuh"

namespace fcm {

constexpr int kTileDiag = 528;    // 32*33/2
constexpr int kIrrWarps = 8;      // k_patch_smooth: warps streaming the individual patches
constexpr int kIrrStages = 2;     // ring depth per streaming warp (8 KB stages)
constexpr int kFdWarps = 4;       // k_patch_smooth: warps applying the regular patches
constexpr int kFdMaxS = 9;        // 2q+1 <= 9 (q <= 4)

__host__ __device__ constexpr int64_t tile_pack_size(int nt) {
  return (int64_t)nt * (nt - 1) / 2 * 1024 + (int64_t)nt * kTileDiag;
}
__host__ __device__ inline int64_t tile_off(int I, int J) {   // J <= I
  return (int64_t)I * (I - 1) / 2 * 1024 + (int64_t)I * kTileDiag + (int64_t)J * 1024;
}

// ---- setup: cell-loop assembly --------------------------------------------------------------
struct PatchAsmArgs {
  int dim, mb, MP, ldK;
  int nx, ny, nz;
  int na[3];
  int nasm, aoff;
  const int64_t* anchors;     // [nblocks]
  const int16_t* alist;       // [nas][mq] compact (slot) per assembly cell: slot of local DOF a, -1
  int mq;
  const int8_t* dirich;       // [nblocks][mb]
  const uint8_t* kind;        // owned cells (single GPU); nullptr: every cell uncut physical (type blocks)
  const int32_t* cut_idx;
  const double* Kref;
  const double* cutK;
  double alpha;
  double* W;                  // [nblocks][MP][MP], zeroed
};

__global__ void __launch_bounds__(256) k_patch_asm(PatchAsmArgs a) {
  const int64_t blk = blockIdx.x;
  const int64_t A = a.anchors[blk];
  const int ax = (int)(A % a.na[0]), ay = (int)((A / a.na[0]) % a.na[1]), az = (int)(A / ((int64_t)a.na[0] * a.na[1]));
  double* W = a.W + blk * (int64_t)a.MP * a.MP;
  const int8_t* dir = a.dirich + blk * a.mb;
  const int ncz = a.dim == 3 ? a.nasm : 1, ncy = a.dim >= 2 ? a.nasm : 1;
  const int nas = a.nasm * ncy * ncz;
  const int mq = a.mq;
  for (int d = 0; d < nas; ++d) {
    const int cx = ax + a.aoff + d % a.nasm;
    const int cy = a.dim >= 2 ? ay + a.aoff + (d / a.nasm) % a.nasm : 0;
    const int cz = a.dim == 3 ? az + a.aoff + d / (a.nasm * a.nasm) : 0;
    if (cx < 0 || cy < 0 || cz < 0 || cx >= a.nx || cy >= a.ny || cz >= a.nz) continue;   // uniform
    const int64_t c = ((int64_t)cz * a.ny + cy) * a.nx + cx;
    const uint8_t k = a.kind ? a.kind[c] : 0;
    const double* K = k == 2 ? a.cutK + (int64_t)a.cut_idx[c] * a.ldK * a.ldK : a.Kref;
    const double s = k == 1 ? a.alpha : 1.0;
    const int16_t* sl = a.alist + (int64_t)d * mq;
    for (int e = threadIdx.x; e < mq * mq; e += blockDim.x) {
      const int ia = e / mq, ib = e % mq;
      const int li = sl[ia], lj = sl[ib];
      if (li < 0 || lj < 0 || dir[li] || dir[lj]) continue;
      W[(int64_t)li * a.MP + lj] += s * K[(int64_t)ia * a.ldK + ib];
    }
    __syncthreads();   // next cell may hit the same entries
  }
  // identity rows for absent / Dirichlet slots and the padding
  for (int l = threadIdx.x; l < a.MP; l += blockDim.x)
    if (l >= a.mb || dir[l]) W[(int64_t)l * a.MP + l] = 1.0;
}

#include "gj.cuh"

// off-diagonal tiles of the patch inverses are stored SWIZZLED (swz): element (r, c) at
// r * 32 + (c ^ r), so a lane can walk its row (lane = r) or its column (lane = c) of the tile
// without shared-memory bank conflicts (k_patch_smooth's shuffle-free tile product), and both
// walks address the element by one LOP3 (see SwzTile)
__host__ __device__ inline int tile_pos(int r, int c, bool swz) { return r * 32 + (swz ? (c ^ r) : c); }

// full workspace (ld MP) -> tile-packed lower storage (symmetrised); grid (tiles, matrices)
__global__ void k_pack_tiles(const double* W, int MP, int nt, double* out, int64_t stride, int swz) {
  int t = blockIdx.x;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  const int J = t - I * (I + 1) / 2;
  const double* M = W + (int64_t)blockIdx.y * MP * MP;
  double* o = out + (int64_t)blockIdx.y * stride + tile_off(I, J);
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    const int64_t gi = 32 * I + r, gj = 32 * J + c;
    const double v = 0.5 * (M[gi * MP + gj] + M[gj * MP + gi]);
    if (I != J) o[tile_pos(r, c, swz)] = v;
    else if (c <= r) o[r * (r + 1) / 2 + c] = v;
  }
}

// ---- hot path: individual patch inverses, streamed ------------------------------------------
struct PatchIrrOp {
  int nx, ny, nz;
  int na[3];
  int mb, nt;                 // block slots, tiles per dim (32 nt >= mb)
  int wpp;                    // streaming warps per patch (kIrrWarps / wpp patches in flight per CTA)
  int det;                    // deterministic mode: a patch's row sums added in a fixed warp order
  int swz;                    // off-diagonal tiles rotated (tile_pos): shuffle-free tile product
  int l2ef;                   // stream the inverses with an L2 evict_first policy
  int64_t stride;             // doubles per packed inverse
  int64_t n_irr;
  const int64_t* anchors;     // [n_irr] anchor of individual block i
  const int8_t* mem;          // [mb] member cell of slot l
  const int16_t* loc;         // [mb] local DOF of slot l
  int mo[8][3];
  const int64_t* base;        // level table
  const int32_t* stride3;
  const int16_t* cmin;
  const int16_t* cmax;
  int m;
  const double* inv;          // [n_irr][stride]
  const double* in;
  double* out;
  double coef;
  // dynamic scheduling (nullptr: static round-robin): [0] next individual patch, [1] next
  // fast-diagonalisation item, [2] CTAs done (the last one zeroes all three for the next launch)
  unsigned long long* sched;
  // diagnostic (FCM_PATCH_PROF=1, else nullptr): per CTA [0] start, [1] last streaming warp done,
  // [2] last fast-diagonalisation warp done (globaltimer ns)
  unsigned long long* prof;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// the same copy with an L2 eviction policy (evict_first for data read once per sweep, so the
// streamed inverses do not push the gathered / scattered vectors out of L2)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// 32 per-lane row partials -> lane r holds the warp sum of partial r (reduce-scatter butterfly)
__device__ __forceinline__ double warp_reduce_scatter32(double (&p)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      // keep half: lanes with bit h set keep the upper half [h, 2h), others the lower [0, h)
      const double send = up ? p[i] : p[i + h];
      const double keep = up ? p[i + h] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return p[0];
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One swizzled off-diagonal tile, lane l: y_J[l] += sum_r T[r][l] x_I[r] (column walk) and
// y_I[l] += sum_r T[l][r] x_J[r] (row walk).  T[r][l] sits at byte (tb | (8 l ^ 8 r)) + 256 r
// (the 256 r as the load's immediate) and T[l][r] at (rb | (8 l ^ 8 r)) with rb = tb + 256 l
// (tb 256-aligned, so OR = ADD below bit 8): each element costs one LOP3 and one LDS.64.  R steps in pairs
// (16-byte x broadcasts), four independent FMA chains.
template <int R>
struct SwzTile {
  static __device__ __forceinline__ void run(uint32_t tb, uint32_t rb, uint32_t lb, const double2* xI2,
                                             const double2* xJ2, double& a0, double& a1, double& b0, double& b1) {
    double c0, c1, r0, r1;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(c0) : "r"(tb | (lb ^ (8u * R))), "n"(256 * R));
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r0) : "r"(rb | (lb ^ (8u * R))));
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(c1) : "r"(tb | (lb ^ (8u * (R + 1)))), "n"(256 * (R + 1)));
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r1) : "r"(rb | (lb ^ (8u * (R + 1)))));
    const double2 xi = xI2[R >> 1], xj = xJ2[R >> 1];
    a0 = fma(c0, xi.x, a0);
    b0 = fma(r0, xj.x, b0);
    a1 = fma(c1, xi.y, a1);
    b1 = fma(r1, xj.y, b1);
    SwzTile<R + 2>::run(tb, rb, lb, xI2, xJ2, a0, a1, b0, b1);
  }
};
template <>
struct SwzTile<32> {
  static __device__ __forceinline__ void run(uint32_t, uint32_t, uint32_t, const double2*, const double2*, double&,
                                             double&, double&, double&) {}
};

// Individual patches, streamed: nw warps (index w) of the CTA, synchronised among themselves
// with named barrier bar_id.  xs/ys/ids: 32 nt slots each; ring: nw x kIrrStages x 1024
// doubles; bars: nw x kIrrStages mbarriers (initialised by the caller).
__device__ __forceinline__ void irr_loop(const PatchIrrOp& op, const Tab& T, double* xs, double* ys, int* ids,
                                         double* ring, uint64_t* bars_all, int w, int nw, int bar_id,
                                         int64_t p0, int64_t pstep, int wring, int64_t* pid) {
  const int lane = threadIdx.x & 31;
  const int MPd = 32 * op.nt;
  double* myring = ring + (size_t)wring * kIrrStages * 1024;
  uint64_t* bars = bars_all + wring * kIrrStages;
  const int nthr = nw * 32;
  const int tid = w * 32 + lane;
  const int nt = op.nt;
  const int ntiles = nt * (nt + 1) / 2;
  const int ntw = w < ntiles ? (ntiles - w + nw - 1) / nw : 0;   // tiles of this warp per patch
  // static: patch k of this group is p0 + k pstep; dynamic (op.sched): the group leader claims
  // patches from a global counter one patch ahead (pid[k & 1] = patch k, written at the top of
  // patch k - 1, visible to the group after the gather barrier, before any tile of patch k is
  // issued), so SMs that stream faster take more patches
  const bool dyn = op.sched != nullptr;
  const bool leader = w == 0 && lane == 0;
  auto patch_of = [&](int64_t k) -> int64_t { return dyn ? pid[k & 1] : p0 + k * pstep; };
  if (dyn) {
    if (leader) {
      pid[0] = (int64_t)atomicAdd(op.sched, 1ull);
      pid[1] = (int64_t)atomicAdd(op.sched, 1ull);
    }
    group_sync(bar_id, nthr);
  }
  const int64_t npatch = dyn ? INT64_MAX : (op.n_irr > p0 ? (op.n_irr - p0 + pstep - 1) / pstep : 0);
  // tile t = w + nw j of a patch (lower tiles row-major): (I0, J0) for j = 0, then J += nw with
  // the row carried (no division / square root per tile)
  int I0 = 0, J0 = w;
  while (J0 > I0) { J0 -= I0 + 1; ++I0; }
  auto next_tile = [&](int& I, int& J) {
    J += nw;
    while (J > I) { J -= I + 1; ++I; }
  };
  // the ring's producer (lane 0) walks the items (patch k, step j, tile (I, J)) of this warp in
  // order, kIrrStages ahead of the consumer; beyond the last patch it issues nothing
  const uint64_t pol = l2_evict_first_policy();
  int64_t is_k = 0;
  uint32_t is_i = 0;
  int is_j = 0, is_I = I0, is_J = J0;
  auto issue_next = [&]() {
    const int64_t b = patch_of(is_k);
    if (b < op.n_irr) {
      const double* src = op.inv + b * op.stride + tile_off(is_I, is_J);
      const uint32_t bytes = (is_I == is_J ? kTileDiag : 1024) * 8;
      const int s = (int)(is_i % kIrrStages);
      mbar_expect_tx(&bars[s], bytes);
      if (op.l2ef) bulk_g2s_hint(myring + s * 1024, src, bytes, &bars[s], pol);
      else bulk_g2s(myring + s * 1024, src, bytes, &bars[s]);
    }
    ++is_i;
    if (++is_j == ntw) {
      is_j = 0;
      ++is_k;
      is_I = I0;
      is_J = J0;
    } else {
      next_tile(is_I, is_J);
    }
  };
  if (lane == 0 && ntw > 0)
    for (int i = 0; i < kIrrStages; ++i) issue_next();
  uint32_t item = 0;
  for (int64_t k = 0; k < npatch; ++k) {
    const int64_t b = patch_of(k);
    if (b >= op.n_irr) break;   // dynamic: counter exhausted (same smem value for the whole group)
    if (dyn && k >= 1 && leader) pid[(k + 1) & 1] = (int64_t)atomicAdd(op.sched, 1ull);
    const int64_t A = op.anchors[b];
    const int ax = (int)(A % op.na[0]), ay = (int)((A / op.na[0]) % op.na[1]), az = (int)(A / ((int64_t)op.na[0] * op.na[1]));
    for (int l = tid; l < MPd; l += nthr) {
      int idx = -1;
      if (l < op.mb) {
        const int km = op.mem[l], a = op.loc[l];
        const int cx = ax + op.mo[km][0], cy = ay + op.mo[km][1], cz = az + op.mo[km][2];
        const bool ok = cx >= 0 && cy >= 0 && cz >= 0 && cx < op.nx && cy < op.ny && cz < op.nz && dof_free(T, a, cx, cy, cz);
        idx = ok ? dof_index(T, a, cx, cy, cz) : -1;
      }
      ids[l] = idx;
      xs[l] = idx >= 0 ? __ldg(op.in + idx) : 0.0;
      ys[l] = 0.0;
    }
    group_sync(bar_id, nthr);
    // deterministic mode: every warp runs the same number of tile steps; after each step the
    // warps add their row sums to ys one after the other (named barrier between)
    const int nsteps = op.det ? (ntiles + nw - 1) / nw : ntw;
    int I = I0, J = J0;
    for (int j = 0; j < nsteps; ++j) {
      if (j >= ntw) {   // det only: no tile left for this warp, keep the barrier count
        for (int k = 0; k < nw; ++k) group_sync(bar_id, nthr);
        continue;
      }
      if (j > 0) next_tile(I, J);
      const int s = (int)(item % kIrrStages);
      mbar_wait(&bars[s], (item / kIrrStages) & 1);
      const double* tl = myring + s * 1024;
      double yJ = 0.0, yI;
      if (I != J && op.swz) {
        // swizzled tile: lane l walks column l (y_J += T^T x_I) and row l (y_I += T x_J) together,
        // both conflict-free, no cross-lane reduction; x pairs as warp-uniform 16-byte broadcasts
        const uint32_t tb = smem_u32(tl), lb = 8u * lane;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        SwzTile<0>::run(tb, tb + 256u * lane, lb, reinterpret_cast<const double2*>(xs + 32 * I),
                        reinterpret_cast<const double2*>(xs + 32 * J), a0, a1, b0, b1);
        yJ = a0 + a1;
        yI = b0 + b1;
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_next();
        }
      } else {
        const double xJ = xs[32 * J + lane];
        double p[32];
        if (I != J) {
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const double a = tl[r * 32 + lane];
            p[r] = a * xJ;
            yJ = fma(a, xs[32 * I + r], yJ);
          }
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const double a = lane <= r ? tl[r * (r + 1) / 2 + lane] : 0.0;
            p[r] = a * xJ;
            if (lane < r) yJ = fma(a, xs[32 * I + r], yJ);
          }
        }
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_next();
        }
        yI = warp_reduce_scatter32(p);
      }
      ++item;
      if (!op.det) {
        atomicAdd(&ys[32 * I + lane], yI);
        atomicAdd(&ys[32 * J + lane], yJ);
      } else {
        for (int k = 0; k < nw; ++k) {
          if (k == w) {
            ys[32 * I + lane] += yI;
            ys[32 * J + lane] += yJ;
          }
          group_sync(bar_id, nthr);
        }
      }
    }
    group_sync(bar_id, nthr);
    for (int l = tid; l < op.mb; l += nthr) {
      const int idx = ids[l];
      if (idx >= 0) atomicAdd(op.out + idx, op.coef * ys[l]);
    }
    group_sync(bar_id, nthr);
  }
}

// ---- hot path: regular patches by fast diagonalisation --------------------------------------
struct PatchFdOp {
  int nx, ny, nz, dim;
  int na[3];
  int q, S;                   // level, slots per axis (2q+1)
  int64_t nreg;
  // low-rank individual patches (patch_wb.cuh) handled by the same warps after the regular ones:
  // z = A0^{-1} r, w = C z_S, x += coef (z - A0^{-1} P_S w)
  int64_t n_wb;
  const int64_t* wb_anchor;   // [n_wb]
  const int64_t* wb_soff;     // [n_wb + 1]
  const int16_t* wb_tS;       // S lists as TENSOR slots (x fastest)
  const int64_t* wb_coff;     // [n_wb + 1]
  const double* wb_C;         // k x k row-major per patch
  const int32_t* anchors;     // [nreg] regular anchors
  const int32_t* blk;         // per anchor: type code (alpha flag in bit 12 of -blk-1)
  const int* cls;             // [3][na] axis class of each anchor coordinate
  const double* tabs;         // [3][ncls][S*S + S]: S_a (row i = slot, col j = mode), lambda_a
  int ncls;
  double s_fac, inv_alpha;
  const int16_t* modeidx;     // [(q+1)^3] local DOF of element mode (kx,ky,kz), kx fastest
  const int64_t* base;
  const int32_t* stride3;
  const int16_t* cmin;
  const int16_t* cmax;
  int m;
  const double* in;
  double* out;
  double coef;
  unsigned long long* sched;  // dynamic scheduling: [1] next item (claimed kFdChunk at a time)
  int roll;                   // fd_pass ROLL form (FCM_FD_ROLL=0: fully unrolled passes)
};

constexpr int kFdChunk = 4;       // fast-diagonalisation items per dynamic claim

// slot s (0..2q) of an axis at vertex v: cell offset and 1D mode (vertex slots pick a cell in
// the grid: v-1 | internals of cell v-1 | v | internals of cell v | v+1)
__device__ __forceinline__ void fd_slot(int s, int q, int v, int n, int& cell, int& k) {
  if (s == 0) { cell = v - 1; k = 0; }
  else if (s < q) { cell = v - 1; k = s + 1; }
  else if (s == q) { if (v < n) { cell = v; k = 0; } else { cell = v - 1; k = 1; } }
  else if (s < 2 * q) { cell = v; k = s - q + 1; }
  else { cell = v; k = 1; }
}

// One one-axis contraction of the S^DIM slot tensor (x fastest) by a 1D factor Tm (S x S,
// row i = slot, column j = mode): forward out_j = sum_i Tm[i][j] in_i (S^T), backward
// out_i = sum_j Tm[i][j] in_j (S).  LINE-BASED: each lane owns whole lines along AXIS (S inputs
// and S outputs in registers, S independent accumulators), the factor is read as warp-uniform
// broadcast words.  SCALE (the last forward axis): multiply by sc / (lambda_x + lambda_y (+ lambda_z)).
// ROLL: the loop over the INPUT index stays rolled (one line value + S factor words + S FMAs per
// trip), so a pass is ~0.5 KB of code instead of ~3.2 KB and the six passes of a patch ~3 KB
// instead of ~20 KB: the fast-diagonalisation warps stop cycling the SM's instruction cache under
// the streaming warps' tile loop (ncu: stall_no_instructions was the largest stall of the fused
// kernel, two thirds of it in the streaming code).
template <int S, int DIM, int AXIS, bool FWD, bool SCALE, bool ROLL>
__device__ __forceinline__ void fd_pass(const double* __restrict__ in, double* __restrict__ out, const double* Tm,
                                        const double* lx, const double* ly, const double* lz, double sc) {
  constexpr int NLINE = DIM == 3 ? S * S : S;
  constexpr int ST = AXIS == 0 ? 1 : (AXIS == 1 ? S : S * S);
  const int lane = threadIdx.x & 31;
  if (ROLL) {
#pragma unroll 1
    for (int line = lane; line < NLINE; line += 32) {
      const int base = AXIS == 0 ? line * S : (AXIS == 1 ? (line / S) * S * S + line % S : line);
      double o[S];
#pragma unroll
      for (int b = 0; b < S; ++b) o[b] = 0.0;
      const double* pin = in + base;
      const double* pt = Tm;   // FWD: row a of the factor; backward: column a
#pragma unroll 1
      for (int a = 0; a < S; ++a) {
        const double va = *pin;
#pragma unroll
        for (int b = 0; b < S; ++b) o[b] = fma(FWD ? pt[b] : pt[b * S], va, o[b]);
        pin += ST;
        pt += FWD ? S : 1;
      }
      if (SCALE) {
        const int xx = line % S, yy = DIM == 3 ? line / S : 0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const double lam = DIM == 3 ? lx[xx] + ly[yy] + lz[j] : lx[xx] + ly[j];
          o[j] *= sc / lam;
        }
      }
#pragma unroll
      for (int j = 0; j < S; ++j) out[base + j * ST] = o[j];
    }
    return;
  }
#pragma unroll 1
  for (int line = lane; line < NLINE; line += 32) {
    const int base = AXIS == 0 ? line * S : (AXIS == 1 ? (line / S) * S * S + line % S : line);
    // an opaque zero, so the S^2 factor words are re-read per line (broadcast LDS) instead of
    // being hoisted into registers (S = 9: 162 registers -> spills)
    int z0;
    asm volatile("mov.b32 %0, 0;" : "=r"(z0));
    const double* Tl = Tm + z0;
    double v[S], o[S];
#pragma unroll
    for (int i = 0; i < S; ++i) {
      v[i] = in[base + i * ST];
      o[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int j = 0; j < S; ++j) {
        if (FWD) o[j] = fma(Tl[i * S + j], v[i], o[j]);
        else o[i] = fma(Tl[i * S + j], v[j], o[i]);
      }
    if (SCALE) {   // element (line, j) of the last axis: 3D line = y S + x, 2D line = x
      const int xx = line % S, yy = DIM == 3 ? line / S : 0;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const double lam = DIM == 3 ? lx[xx] + ly[yy] + lz[j] : lx[xx] + ly[j];
        o[j] *= sc / lam;
      }
    }
#pragma unroll
    for (int j = 0; j < S; ++j) out[base + j * ST] = o[j];
  }
}

// slot code of an INTERIOR anchor (every cell of the patch inside the grid, no Dirichlet DOF):
// local DOF a (bits 0-9) and, per axis, whether the slot's cell is v - 1 (bits 10, 11, 12)
__device__ __forceinline__ int fd_slot_code(int l, int S, int q, int DIM, const int16_t* midx) {
  const int sx = l % S, sy = (l / S) % S, sz = DIM == 3 ? l / (S * S) : 0;
  int cx, kx, cy, ky, cz = 2, kz = 0;
  fd_slot(sx, q, 2, 1 << 20, cx, kx);
  fd_slot(sy, q, 2, 1 << 20, cy, ky);
  if (DIM == 3) fd_slot(sz, q, 2, 1 << 20, cz, kz);
  const int a = midx[(kz * (q + 1) + ky) * (q + 1) + kx];
  return a | ((2 - cx) << 10) | ((2 - cy) << 11) | ((2 - cz) << 12);
}

// Regular patches by fast diagonalisation: nw warps (index w), independent (no CTA barrier).
// Compile-time S (slots per axis) and DIM: every lane owns slots l = lane + 32 j, whose DOF
// indices and gathered values live in registers (all NL loads in flight before the first use:
// the gather is one memory latency per patch, not one per slot), and the same slots are
// scattered at the end.  Interior anchors compute the indices from the slot-code table (one
// LDS + the level table entry); boundary anchors take the general path.  The six one-axis
// contractions are line-based (fd_pass).  wbase: nw x 2 S^d doubles.
template <int S, int DIM, bool ROLL>
__device__ __forceinline__ void fd_loop(const PatchFdOp& op, const Tab& T, const double* tab, const int16_t* midx,
                                        const int* scode, double* wbase, int w, int nw) {
  constexpr int S2 = S * S, N3 = DIM == 3 ? S2 * S : S2;
  constexpr int NL = (N3 + 31) / 32;
  constexpr int tsz = S * S + S;
  const int q = op.q;
  const int lane = threadIdx.x & 31;
  double* X = wbase + (size_t)w * 2 * N3;
  double* Y = X + N3;
  const double coef = op.coef;
  const int64_t ntot = op.nreg + op.n_wb;
  // static: item blockIdx.x nw + w + k gridDim.x nw; dynamic: chunks of kFdChunk consecutive
  // items (neighbouring anchors share gather lines) claimed from a global counter
  const bool dyn = op.sched != nullptr;
  auto claim = [&]() -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(op.sched + 1, (unsigned long long)kFdChunk);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  for (int64_t c0 = dyn ? claim() : (int64_t)blockIdx.x * nw + w; c0 < ntot;
       c0 = dyn ? claim() : c0 + (int64_t)gridDim.x * nw)
  for (int64_t i = c0, c1 = dyn ? min(c0 + kFdChunk, ntot) : c0 + 1; i < c1; ++i) {
    const bool lowrank = i >= op.nreg;
    const int64_t pw = i - op.nreg;
    const int A = lowrank ? (int)op.wb_anchor[pw] : op.anchors[i];
    const int vx = A % op.na[0], vy = (A / op.na[0]) % op.na[1], vz = A / (op.na[0] * op.na[1]);
    const int t = lowrank ? 0 : -op.blk[A] - 1;   // low-rank patches: physical regular A0
    const double sc = ((t >> 12) ? op.inv_alpha : 1.0) / op.s_fac;
    const double* Tx = tab + (0 * op.ncls + op.cls[vx]) * tsz;
    const double* Ty = tab + (1 * op.ncls + op.cls[op.na[0] + vy]) * tsz;
    const double* Tz = tab + (2 * op.ncls + (DIM == 3 ? op.cls[op.na[0] + op.na[1] + vz] : 0)) * tsz;
    const bool inner = vx >= 2 && vx <= op.nx - 2 && vy >= 2 && vy <= op.ny - 2 &&
                       (DIM == 2 || (vz >= 2 && vz <= op.nz - 2));
    int ids[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int l = lane + 32 * j;
      int idx = -1;
      if (l < N3) {
        if (inner) {
          const int code = scode[l];
          const int4 g = T.g[code & 1023];
          idx = g.x + (vx - ((code >> 10) & 1)) + (vy - ((code >> 11) & 1)) * g.y +
                (DIM == 3 ? (vz - ((code >> 12) & 1)) * g.z : 0);
        } else {
          const int sx = l % S, sy = (l / S) % S, sz = DIM == 3 ? l / S2 : 0;
          int cx, kx, cy, ky, cz = 0, kz = 0;
          fd_slot(sx, q, vx, op.nx, cx, kx);
          fd_slot(sy, q, vy, op.ny, cy, ky);
          if (DIM == 3) fd_slot(sz, q, vz, op.nz, cz, kz);
          if (cx >= 0 && cy >= 0 && cz >= 0 && cx < op.nx && cy < op.ny && cz < op.nz) {
            const int a = midx[(kz * (q + 1) + ky) * (q + 1) + kx];
            if (dof_free(T, a, cx, cy, cz)) idx = dof_index(T, a, cx, cy, cz);
          }
        }
      }
      ids[j] = idx;
    }
    {
      double xv[NL];
#pragma unroll
      for (int j = 0; j < NL; ++j) xv[j] = ids[j] >= 0 ? __ldg(op.in + ids[j]) : 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j)
        if (lane + 32 * j < N3) X[lane + 32 * j] = xv[j];
    }
    __syncwarp();
    // forward (S^T x S^T x S^T) X with the D^-1 scaling fused into the last axis, then backward
    auto fd_apply = [&]() {
      if (DIM == 3) {
        fd_pass<S, DIM, 0, true, false, ROLL>(X, Y, Tx, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 1, true, false, ROLL>(Y, X, Ty, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 2, true, true, ROLL>(X, Y, Tz, Tx + S2, Ty + S2, Tz + S2, sc);
        __syncwarp();
        fd_pass<S, DIM, 2, false, false, ROLL>(Y, X, Tz, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 1, false, false, ROLL>(X, Y, Ty, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 0, false, false, ROLL>(Y, X, Tx, nullptr, nullptr, nullptr, 0.0);
      } else {
        fd_pass<S, DIM, 0, true, false, ROLL>(X, Y, Tx, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 1, true, true, ROLL>(Y, X, Ty, Tx + S2, Ty + S2, nullptr, sc);
        __syncwarp();
        fd_pass<S, DIM, 1, false, false, ROLL>(X, Y, Ty, nullptr, nullptr, nullptr, 0.0);
        __syncwarp();
        fd_pass<S, DIM, 0, false, false, ROLL>(Y, X, Tx, nullptr, nullptr, nullptr, 0.0);
      }
      __syncwarp();
    };
    fd_apply();   // X = A0^{-1} r
    if (!lowrank) {
#pragma unroll
      for (int j = 0; j < NL; ++j)
        if (ids[j] >= 0) atomicAdd(op.out + ids[j], coef * X[lane + 32 * j]);
      __syncwarp();
      continue;
    }
    // low-rank patch: z = X kept in registers, z_S compacted into Y, X = P_S w with w = C z_S, then
    // X = A0^{-1} P_S w and x += coef (z - X).  C is symmetric (symmetrised at setup), so lane r
    // accumulates row r by walking COLUMN r of the row-major array: the loads of one step are
    // coalesced across the lanes and independent across steps (eight in flight), z_S[c] is a
    // warp-uniform shared-memory broadcast, no cross-lane reduction
    double zr[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) zr[j] = lane + 32 * j < N3 ? X[lane + 32 * j] : 0.0;
    const int64_t s0 = op.wb_soff[pw];
    const int k = (int)(op.wb_soff[pw + 1] - s0);
    const double* Cp = op.wb_C + op.wb_coff[pw];
    const int16_t* tS = op.wb_tS + s0;
    for (int c = lane; c < k; c += 32) Y[c] = X[tS[c]];
    __syncwarp();
    for (int l = lane; l < N3; l += 32) X[l] = 0.0;
    __syncwarp();
    for (int r0 = 0; r0 < k; r0 += 32) {
      const int r = min(r0 + lane, k - 1);
      const double* Cr = Cp + r;
      double sum = 0.0;
#pragma unroll 8
      for (int c = 0; c < k; ++c) sum = fma(__ldg(Cr + (int64_t)c * k), Y[c], sum);
      if (r0 + lane < k) X[tS[r]] = sum;
    }
    __syncwarp();
    fd_apply();
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (ids[j] >= 0) atomicAdd(op.out + ids[j], coef * (zr[j] - X[lane + 32 * j]));
    __syncwarp();
  }
}

__device__ __forceinline__ void load_tab_from(Tab& T, int m, const int64_t* base, const int32_t* stride3,
                                              const int16_t* cmin, const int16_t* cmax) {
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    T.g[a] = make_int4((int32_t)base[a], stride3[a * 3 + 1], stride3[a * 3 + 2], 0);
    T.lo[a] = make_int4(cmin[a * 3 + 0], cmin[a * 3 + 1], cmin[a * 3 + 2], 0);
    T.hi[a] = make_int4(cmax[a * 3 + 0], cmax[a * 3 + 1], cmax[a * 3 + 2], 0);
  }
}

// One patchwise smoother sweep in ONE launch, warp-specialised (one CTA per SM, persistent):
// warps [0, kIrrWarps) stream the individual patches' tile-packed inverses (HBM-bound), warps
// [kIrrWarps, kIrrWarps + kFdWarps) apply the regular patches by fast diagonalisation (latency
// / FMA-bound) -- the two populations overlap on every SM instead of queueing behind each
// other.  IRR / FD select the populations (fcm_mg_smooth_part).
// smem: [Tab][xs, ys: 32 nt doubles][ids: 32 nt ints][ring: kIrrWarps x kIrrStages x 8 KB]
//       [mbarriers][FD tables][modeidx][FD: kFdWarps x 2 S^d doubles]
template <int S, int DIM, bool IRR, bool FD>
__global__ void __launch_bounds__((kIrrWarps + kFdWarps) * 32, 1) k_patch_smooth(PatchIrrOp io, PatchFdOp fo) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  const int MPd = 32 * io.nt;
  const int ngrp = kIrrWarps / io.wpp;   // patches in flight per CTA
  double* xs0 = reinterpret_cast<double*>(smem + sizeof(Tab));
  // the ring starts 256-aligned in the shared window (SwzTile's OR addressing): the dynamic
  // segment is at least 16-aligned, so pad by up to 240 bytes (patch_smem reserves them)
  const uint32_t s0 = smem_u32(smem);
  const size_t o_ring = ((s0 + sizeof(Tab) + (size_t)ngrp * MPd * 20 + 255) / 256 * 256) - s0;
  double* ring = reinterpret_cast<double*>(smem + o_ring);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)kIrrWarps * kIrrStages * 1024);
  constexpr int tsz = S * S + S;
  int64_t* pids = reinterpret_cast<int64_t*>(bars + kIrrWarps * kIrrStages);   // 2 per group
  double* tab = reinterpret_cast<double*>(pids + 2 * kIrrWarps);
  int16_t* midx = reinterpret_cast<int16_t*>(tab + 3 * fo.ncls * tsz);
  const int nmi = (fo.q + 1) * (fo.q + 1) * (fo.q + 1);
  constexpr int N3 = DIM == 3 ? S * S * S : S * S;
  int* scode = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(midx) + ((nmi * 2 + 15) / 16) * 16);
  double* wbase = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(scode) + ((N3 * 4 + 15) / 16) * 16);
  const int w = threadIdx.x >> 5;
  load_tab_from(T, io.m, io.base, io.stride3, io.cmin, io.cmax);
  if (FD) {
    for (int e = threadIdx.x; e < 3 * fo.ncls * tsz; e += blockDim.x) tab[e] = fo.tabs[e];
    for (int e = threadIdx.x; e < nmi; e += blockDim.x) midx[e] = fo.modeidx[e];
  }
  __syncthreads();
  if (FD)
    for (int l = threadIdx.x; l < N3; l += blockDim.x) scode[l] = fd_slot_code(l, S, fo.q, DIM, midx);
  if (IRR && w < kIrrWarps && (threadIdx.x & 31) == 0)
    for (int s = 0; s < kIrrStages; ++s) mbar_init(&bars[w * kIrrStages + s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto now_ns = []() -> unsigned long long {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (io.prof && threadIdx.x == 0) io.prof[4 * blockIdx.x] = now_ns();
  if (w < kIrrWarps) {
    if (IRR) {
      const int g = w / io.wpp;
      double* xs = xs0 + (size_t)g * MPd * 2;
      double* ys = xs + MPd;
      int* ids = reinterpret_cast<int*>(xs0 + (size_t)ngrp * MPd * 2) + (size_t)g * MPd;
      irr_loop(io, T, xs, ys, ids, ring, bars, w % io.wpp, io.wpp, 1 + g, (int64_t)blockIdx.x * ngrp + g,
               (int64_t)gridDim.x * ngrp, w, pids + 2 * g);
    }
  } else {
    if (FD) {
      if (fo.roll) fd_loop<S, DIM, true>(fo, T, tab, midx, scode, wbase, w - kIrrWarps, kFdWarps);
      else fd_loop<S, DIM, false>(fo, T, tab, midx, scode, wbase, w - kIrrWarps, kFdWarps);
    }
  }
  if (io.prof && (threadIdx.x & 31) == 0) atomicMax(io.prof + 4 * blockIdx.x + (w < kIrrWarps ? 1 : 2), now_ns());
  if (io.sched) {   // the last CTA out re-arms the counters (every claim of this launch is done)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(io.sched + 2, 1ull) == gridDim.x - 1) {
        atomicExch(io.sched + 0, 0ull);
        atomicExch(io.sched + 1, 0ull);
        atomicExch(io.sched + 2, 0ull);
      }
    }
  }
}

}  // namespace fcm
