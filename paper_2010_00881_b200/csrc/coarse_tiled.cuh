// coarse_tiled.cuh -- the coarsest level (p = 1, PAPER.md:226-228 Remark) solved by CG with
// the undamped elementwise additive-Schwarz preconditioner (reading R4), for
// coarse levels small enough that every SM can hold its piece of the vertex grid, and every
// matrix that piece touches, in shared memory (config 2: 35,937 vertices; the inner solve is
// latency-bound there).
//
// Design (one cooperative launch for the whole inner solve, ONE grid barrier per iteration):
//  * Each CTA owns a brick T of the vertex grid (the p = 1 DOFs are the vertex modes, n_f per
//    vertex) and keeps r and s on T grown by two vertex rings (E2), u on T grown by one ring
//    (E1), and p, x on T in shared memory for the whole solve.  Every matrix its cells use is
//    staged in shared memory once per launch: the leading 2^d n_f block of K_ref, the shared
//    Schwarz inverses (one per boundary type), and the individual cut-cell matrices / Schwarz
//    inverses of the cells in its box (the host sizes the bricks so that they fit).
//  * The operator and the smoother are applied VERTEX-CENTRIC (gather only, no atomics):
//      (A v)_(v,i) = sum_{cells c ni v} s_c K_c[a_v(c)*nf+i, :] v_c
//      (M r)_(v,i) = sum_{cells c ni v} s_c A_c^{-1}[a_v(c)*nf+i, :] r_c
//    K_c = leading block of the cell matrix (K_ref scaled by 1 or alpha, or the cut cell's
//    own), A_c^{-1} = the cell's Schwarz inverse (scaled by 1/alpha for all-fictitious type
//    blocks).  Cells are visited in a fixed order, so every CTA that evaluates a vertex gets
//    bit-identical values.
//  * CG in the Chronopoulos-Gear form (same iterates as standard PCG in exact arithmetic):
//      u = M r, w = A u, gamma = (r,u), delta = (w,u), rho = (r,r)   [one all-reduce]
//      beta = gamma/gamma_old, alpha = gamma/(delta - beta*gamma/alpha_old)
//      p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s
//    After the all-reduce every CTA reads the w its neighbours published (E2 halo) and updates
//    s and r REDUNDANTLY on E2 with the same scalars; then u on E1 and w on T need no further
//    exchange.  Hence one grid-wide synchronisation per iteration, which also carries the
//    three dot products: accumulated with fp64 atomics (every CTA reads the same totals; the
//    summation order varies run to run), or, with FCM_TILED_ATOMIC=0, summed by every CTA in
//    block order (bit-reproducible).
//  * Stop when rho < rtol^2 rho_0 (recursive residual), iterations = x updates (as the
//    oracle's standard PCG, x0 = 0).
#pragma once
#include <climits>
#include <cstdint>

namespace fcm {

struct TiledArgs {
  int n[3];          // cells per axis (1 for absent axes)
  // bricks: [nblocks][6] = vertex origin (3), extents (3) of each CTA's brick T; they partition
  // the vertex box (the union of the free ranges of all components).  Per brick, E2 extents
  // are tile + 4 and the cell box tile + 3 (1 for absent axes).
  const int* brick;
  int tile[3];       // largest brick extents (reporting only)
  int blo[3];        // vertex box origin (host bookkeeping)
  int64_t voff[3];   // class-major offset of component j's vertex class
  int vlo[3][3];     // free vertex range of component j
  int vhi[3][3];
  int max_indiv;     // individual-matrix slots per CTA (host: max over bricks)
  int ntypes;        // shared Schwarz inverses (slots 0..ntypes-1 of type_inv), all staged
  // operator
  const uint8_t* kind;
  const int32_t* cut_idx;
  const double* cutK;
  int ldK;           // leading dimension of K_ref / cut matrices (fine element size)
  const double* Kref;
  double alpha;
  // smoother
  int jacobi;
  const double* diag_inv;
  const int32_t* blk;
  const double* type_inv;   // [ntypes][M1*M1]
  const double* irr_inv;    // [n_irr][M1*M1]
  double inv_alpha;
  // vectors (class-major, level 1)
  const double* b;
  double* x;
  double* wpub[2];          // published w (double-buffered by iteration parity)
  double* part;             // [2][3][nblocks]
  double* acc;              // [3][4] fp64-atomic dot accumulators, or null (see tiled_arrive_wait)
  struct TiledCtl* ctl;     // barrier state (zero-initialised once per handle)
  double rtol2;
  int maxit;
  int* iters;               // [0] = this solve, [1] += this solve
  unsigned long long* prof; // optional per-block phase times (ns): [nblocks][4]
  // constant-coefficient fast path (NF == 1): a vertex whose 2^d cells all use the K_ref block
  // (operator) or the type-0 Schwarz inverse (smoother) with one scale applies the 3^d-point
  // stencil sum_{kc,k2: o(k2)-o(kc)=d} Mat[kc][k2] instead of the per-cell gather (coefficients
  // read from the parameter bank, no shared-memory matrix traffic)
  int fast;
  double st_op[27];
  double st_sm[27];
};

__device__ __forceinline__ unsigned long long t_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned t_ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// cell code: -1 = no cell (outside the grid); otherwise the matrix offset in the staged
// matrix pool (doubles) | kScaleBit when the cell's scale is alpha (operator) or 1/alpha
// (smoother)
constexpr int kNoCell = -1;
constexpr int kScaleBit = 1 << 30;
// per-vertex flags: operator / smoother stencil applies, and its scale (alpha resp. 1/alpha)
constexpr int kVfOp = 1, kVfOpScaled = 2, kVfSm = 4, kVfSmScaled = 8;

// shared-memory layout (doubles first, then ints); see tiled_smem_bytes
template <int DIM, int NF>
struct TiledSmem {
  double* r;    // [NF][E2]
  double* s;    // [NF][E2]
  double* u;    // [NF][E2] (valid on E1)
  double* p;    // [NF][T]
  double* x;    // [NF][T]
  double* mat;  // pool: [K_ref block][types][individual]
  int* gidx;    // [NF][E2] class-major index or -1
  int* cop;     // [EC] operator code per cell
  int* csm;     // [EC] smoother code per cell
  unsigned char* vf;   // [E2] fast-path flags (kVf*)
  int* lsm;     // NF == 1: smoother rows (E1 vertices with a free DOF), stencil rows first;
  int* lop;     //          operator rows (T), stencil rows first; entry = l | cell base << 16
  int nsm, nop;
  int E2, EC, T;
  int e0, e01, ec0, ec01;   // strides of E2 and of the cell box
};

// matrices are symmetric: stored packed lower-triangular, entry (a, b), b <= a, at a(a+1)/2 + b
__host__ __device__ constexpr int packed_size(int m) { return m * (m + 1) / 2; }
__host__ __device__ constexpr int packed_at(int a, int b) {
  return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
}
// matrix slot stride in the pool: odd number of doubles, so that 32 lanes reading the same
// entry of 32 different slots hit distinct bank pairs (no conflicts beyond the 2 wavefronts)
__host__ __device__ constexpr int slot_stride(int m) { return packed_size(m) | 1; }
__host__ __device__ constexpr size_t tiled_smem_bytes(int dim, int nf, int E2, int E1, int EC, int T, int nmats) {
  return (size_t)(3 * nf * E2 + 2 * nf * T) * 8 + (size_t)nmats * slot_stride((1 << dim) * nf) * 8 +
         (size_t)nf * E2 * 4 + (size_t)EC * 8 + (size_t)((E2 + 15) & ~15) +
         (nf == 1 ? (size_t)(E1 + T) * 4 : 0) + 16;
}

// one row of the vertex-centric gather: sum over the 2^d cells around E2 entry l (local
// coordinates lx, ly, lz) of s_c Mat_c[a_v(c)*NF + i, :] . vec_c (all operands in smem)
template <int DIM, int NF, bool SMOOTH>
__device__ __forceinline__ double vertex_row(const TiledArgs& a, const TiledSmem<DIM, NF>& S,
                                             const double* __restrict__ vec, int l, int cb, int i) {
  constexpr int NC = 1 << DIM;
  const int e0 = S.e0, e01 = S.e01;
  const int ec0 = S.ec0, ec01 = S.ec01;
  const double scale = SMOOTH ? a.inv_alpha : a.alpha;
  double acc = 0.0;
  if constexpr (NF == 1) {
    // the 3^d neighbourhood of the vertex, loaded once into registers
    constexpr int N3 = DIM == 3 ? 27 : 9;
    double nb[N3];
#pragma unroll
    for (int q = 0; q < N3; ++q) {
      const int dx = q % 3 - 1, dy = (q / 3) % 3 - 1, dz = DIM == 3 ? q / 9 - 1 : 0;
      nb[q] = vec[l + dx + dy * e0 + dz * e01];
    }
    const int f = S.vf[l];
    if (f & (SMOOTH ? kVfSm : kVfOp)) {
      const double* st = SMOOTH ? a.st_sm : a.st_op;
#pragma unroll
      for (int q = 0; q < N3; ++q) acc = fma(st[q], nb[q], acc);
      return (f & (SMOOTH ? kVfSmScaled : kVfOpScaled)) ? scale * acc : acc;
    }
#pragma unroll
    for (int kc = 0; kc < NC; ++kc) {
      const int ox = kc & 1, oy = (kc >> 1) & 1, oz = (kc >> 2) & 1;
      const int code = SMOOTH ? S.csm[cb - (oz * ec01 + oy * ec0 + ox)] : S.cop[cb - (oz * ec01 + oy * ec0 + ox)];
      double t = 0.0;
      {
        const double* mat = S.mat + (code == kNoCell ? 0 : (code & (kScaleBit - 1)));
#pragma unroll
        for (int k2 = 0; k2 < NC; ++k2) {
          // corner k2 of the cell relative to the vertex (corner kc): offsets in {-1, 0, 1}
          const int q = ((k2 & 1) - ox + 1) + 3 * (((k2 >> 1) & 1) - oy + 1) +
                        (DIM == 3 ? 9 * (((k2 >> 2) & 1) - oz + 1) : 0);
          t = fma(mat[packed_at(kc, k2)], nb[q], t);
        }
      }
      if (code != kNoCell) acc = fma((code & kScaleBit) ? scale : 1.0, t, acc);
    }
  } else {
#pragma unroll
  for (int kc = 0; kc < NC; ++kc) {
    const int ox = kc & 1, oy = (kc >> 1) & 1, oz = (kc >> 2) & 1;
    // the cell box shares the E2 origin: cell local = vertex local - corner offset
    const int code = SMOOTH ? S.csm[cb - (oz * ec01 + oy * ec0 + ox)] : S.cop[cb - (oz * ec01 + oy * ec0 + ox)];
    if (code == kNoCell) continue;
    const double* mat = S.mat + (code & (kScaleBit - 1));
    const int base = l - (ox + oy * e0 + oz * e01);
    double t = 0.0;
#pragma unroll
    for (int k2 = 0; k2 < NC; ++k2) {
      const int d = (k2 & 1) + ((k2 >> 1) & 1) * e0 + ((k2 >> 2) & 1) * e01;
#pragma unroll
      for (int j = 0; j < NF; ++j)
        t = fma(mat[packed_at(kc * NF + i, k2 * NF + j)], vec[j * S.E2 + base + d], t);
    }
    acc = fma((code & kScaleBit) ? scale : 1.0, t, acc);
  }
  }
  return acc;
}

// deterministic block reduction of three values; result valid in warp 0
__device__ __forceinline__ void block_sum3(double& v0, double& v1, double& v2, double* red /*[3*32]*/) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) { red[w] = v0; red[32 + w] = v1; red[64 + w] = v2; }
  __syncthreads();
  if (w == 0) {
    double a0 = l < nw ? red[l] : 0.0, a1 = l < nw ? red[32 + l] : 0.0, a2 = l < nw ? red[64 + l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    v0 = a0; v1 = a1; v2 = a2;
  }
}

// Grid barrier fused with a deterministic all-reduce of three doubles.  Each block posts its
// partials in its own slot and adds 1 to one arrival counter (a single same-address RED per
// block, release semantics); one thread per block polls the counter (acquire) until every
// block of this generation has arrived (measured ~1.3 us on B200 for 128-148 blocks, vs ~4 us
// when the last arrival reduces and re-releases).  Then warp 0 of every block sums all
// partials in block order, so every block holds bit-identical totals.  Counter targets compare
// modulo 2^32; partials are double-buffered by generation parity.
struct TiledCtl {
  unsigned count;          // arrivals (monotone)
  unsigned pad0[31];
  unsigned base;           // count at the end of the previous launch (written by block 0 last)
  unsigned pad1[31];
  // global barrier generation at the end of the previous launch (written by block 0 last);
  // 64-bit and explicit, so the accumulator rotation (G % 3) never depends on the wrapping
  // 32-bit arrival counter (2^32 is not a multiple of the grid size)
  unsigned long long gbase;
};

__device__ __forceinline__ unsigned t_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void t_red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Arrival + wait: block partials posted, one RED per block, one polling thread; returns when
// every block of this generation has arrived (all threads synchronised).
// atomic_dots: the block sums are added with fp64 atomics into acc[G % 3][3] (G = global
// generation) instead of being posted per block; readers then load 3 doubles instead of
// 3 x gridDim partials (no same-line read storm on L2), at the price of a run-dependent
// summation order (every block still reads the same totals).  acc[(G+2) % 3] is zeroed by
// block 0 after barrier G: its last readers (generation G-1) have passed barrier G, and its
// next writers (generation G+2) start after barrier G+1, which block 0 reaches after the zeroing.
__device__ __noinline__ void tiled_arrive_wait(double v0, double v1, double v2, double* part,
                                               TiledCtl* ctl, unsigned target, unsigned gen,
                                               double* red, double* acc, unsigned long long G) {
  block_sum3(v0, v1, v2, red);
  const int nb = gridDim.x;
  double* pp = part + (size_t)(gen & 1) * 3 * nb;
  if (threadIdx.x == 0) {
    if (acc) {
      double* ac = acc + 4 * (G % 3);
      atomicAdd(ac, v0);
      atomicAdd(ac + 1, v1);
      atomicAdd(ac + 2, v2);
    } else {
      __stcg(pp + blockIdx.x, v0);
      __stcg(pp + nb + blockIdx.x, v1);
      __stcg(pp + 2 * nb + blockIdx.x, v2);
    }
    t_red_release(&ctl->count, 1u);   // orders this block's earlier global writes (w, partials)
    while ((int)(t_ld_acquire(&ctl->count) - target) < 0) {}
  }
  __syncthreads();
}
// Totals of generation gen, summed in block order by warp 0 (bit-identical on every block);
// call after tiled_arrive_wait; the caller synchronises before reading tot.
__device__ __forceinline__ void tiled_totals(const double* part, unsigned gen, double* tot, double* acc,
                                             unsigned long long G) {
  if (acc) {
    if (threadIdx.x < 3) tot[threadIdx.x] = __ldcg(acc + 4 * (G % 3) + threadIdx.x);
    if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 35) acc[4 * ((G + 2) % 3) + threadIdx.x - 32] = 0.0;
    return;
  }
  if (threadIdx.x < 32) {
    const int nb = gridDim.x, l = threadIdx.x;
    const double* pp = part + (size_t)(gen & 1) * 3 * nb;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int j = l; j < nb; j += 32) {
      a0 += __ldcg(pp + j);
      a1 += __ldcg(pp + nb + j);
      a2 += __ldcg(pp + 2 * nb + j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (l == 0) { tot[0] = a0; tot[1] = a1; tot[2] = a2; }
  }
}

constexpr int kTiledThreads = 512;

template <int DIM, int NF>
__global__ void __launch_bounds__(kTiledThreads, 1) k_coarse_tiled(TiledArgs a) {
  constexpr int NC = 1 << DIM;
  constexpr int M1 = NC * NF;
  constexpr int MM = slot_stride(M1);
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[96];
  __shared__ double tot[3];
  __shared__ int n_indiv;
  TiledSmem<DIM, NF> S;
  // brick of this block
  const int* br = a.brick + 6 * blockIdx.x;
  const int t0 = br[3], t1 = DIM > 1 ? br[4] : 1, t2 = DIM > 2 ? br[5] : 1;
  const int e0 = t0 + 4, e1 = DIM > 1 ? t1 + 4 : 1, e2d = DIM > 2 ? t2 + 4 : 1;
  const int ec0 = t0 + 3, ec1 = DIM > 1 ? t1 + 3 : 1, ec2 = DIM > 2 ? t2 + 3 : 1;
  const int ec01 = ec0 * ec1;
  S.E2 = e0 * e1 * e2d;
  S.EC = ec0 * ec1 * ec2;
  S.T = t0 * t1 * t2;
  S.e0 = e0; S.e01 = e0 * e1; S.ec0 = ec0; S.ec01 = ec01;
  const int o0 = br[0] - 2;
  const int o1 = DIM > 1 ? br[1] - 2 : 0;
  const int o2 = DIM > 2 ? br[2] - 2 : 0;
  const int nmat = 1 + a.ntypes + a.max_indiv;
  {
    double* d = reinterpret_cast<double*>(smem);
    S.r = d; d += NF * S.E2;
    S.s = d; d += NF * S.E2;
    S.u = d; d += NF * S.E2;
    S.p = d; d += NF * S.T;
    S.x = d; d += NF * S.T;
    S.mat = d; d += (size_t)nmat * MM;
    S.gidx = reinterpret_cast<int*>(d);
    S.cop = S.gidx + NF * S.E2;
    S.csm = S.cop + S.EC;
    S.vf = reinterpret_cast<unsigned char*>(S.csm + S.EC);
    S.lsm = reinterpret_cast<int*>(S.vf + ((S.E2 + 15) & ~15));
    const int ne1 = (t0 + 2) * (DIM > 1 ? t1 + 2 : 1) * (DIM > 2 ? t2 + 2 : 1);
    S.lop = S.lsm + ne1;
  }
  const int E2 = S.E2;
  // ---- one-time staging: K_ref block, shared Schwarz inverses, cell codes ----------------
  if (threadIdx.x == 0) n_indiv = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < M1 * M1; t += blockDim.x) {
    const int r = t / M1, c = t % M1;
    if (c <= r) S.mat[packed_at(r, c)] = a.Kref[r * a.ldK + c];
  }
  for (int t = threadIdx.x; t < a.ntypes * M1 * M1; t += blockDim.x) {
    const int k = t / (M1 * M1), r = (t / M1) % M1, c = t % M1;
    if (c <= r) S.mat[(1 + k) * MM + packed_at(r, c)] = a.type_inv[(size_t)k * M1 * M1 + r * M1 + c];
  }
  __syncthreads();
  const int indiv0 = (1 + a.ntypes) * MM;   // first individual slot (doubles)
  for (int t = threadIdx.x; t < S.EC; t += blockDim.x) {
    const int lx = t % ec0, ly = (t / ec0) % ec1, lz = t / ec01;
    const int cx = o0 + lx, cy = o1 + ly, cz = o2 + lz;
    int2 code = make_int2(kNoCell, kNoCell);
    if (cx >= 0 && cy >= 0 && cz >= 0 && cx < a.n[0] && cy < a.n[1] && cz < a.n[2]) {
      const int c = (cz * a.n[1] + cy) * a.n[0] + cx;
      const int k = a.kind[c];
      if (k == 2) {   // cut cell: its own (leading) matrix
        const int slot = atomicAdd(&n_indiv, 1);
        const double* src = a.cutK + (size_t)a.cut_idx[c] * a.ldK * a.ldK;
        double* dst = S.mat + indiv0 + slot * MM;
        for (int r = 0; r < M1; ++r)
          for (int c2 = 0; c2 <= r; ++c2) dst[packed_at(r, c2)] = __ldg(src + r * a.ldK + c2);
        code.x = indiv0 + slot * MM;
      } else {
        code.x = k == 1 ? kScaleBit : 0;
      }
      if (!a.jacobi) {
        const int bq = a.blk[c];
        if (bq >= 0) {   // irregular block: individual inverse
          const int slot = atomicAdd(&n_indiv, 1);
          const double* src = a.irr_inv + (size_t)bq * M1 * M1;
          double* dst = S.mat + indiv0 + slot * MM;
          for (int r = 0; r < M1; ++r)
            for (int c2 = 0; c2 <= r; ++c2) dst[packed_at(r, c2)] = __ldg(src + r * M1 + c2);
          code.y = indiv0 + slot * MM;
        } else {
          const int tt = -bq - 1;
          code.y = (1 + (tt & 0xfff)) * MM | ((tt >> 12) ? kScaleBit : 0);
        }
      }
    }
    S.cop[t] = code.x;
    S.csm[t] = code.y;
  }
  for (int t = threadIdx.x; t < NF * E2; t += blockDim.x) {
    const int j = t / E2, l = t % E2;
    const int v0 = o0 + l % e0, v1 = o1 + (l / e0) % e1, v2 = o2 + l / (e0 * e1);
    int g = -1;
    if (v0 >= a.vlo[j][0] && v0 <= a.vhi[j][0] && v1 >= a.vlo[j][1] && v1 <= a.vhi[j][1] &&
        v2 >= a.vlo[j][2] && v2 <= a.vhi[j][2]) {
      const int s0 = a.vhi[j][0] - a.vlo[j][0] + 1, s1 = a.vhi[j][1] - a.vlo[j][1] + 1;
      g = (int)a.voff[j] + (v0 - a.vlo[j][0]) + s0 * ((v1 - a.vlo[j][1]) + s1 * (v2 - a.vlo[j][2]));
    }
    S.gidx[t] = g;
    S.r[t] = g >= 0 ? a.b[g] : 0.0;
    S.s[t] = 0.0;
    S.u[t] = 0.0;
  }
  for (int t = threadIdx.x; t < NF * S.T; t += blockDim.x) { S.p[t] = 0.0; S.x[t] = 0.0; }
  __syncthreads();
  // fast-path flags of the E1 vertices (every block derives them from the same cell data, so
  // a vertex evaluated by several blocks still gets bit-identical values)
  for (int t = threadIdx.x; t < E2; t += blockDim.x) {
    const int lx = t % e0, ly = (t / e0) % e1, lz = t / (e0 * e1);
    int f = 0;
    const bool in1 = lx >= 1 && lx <= e0 - 2 && (DIM < 2 || (ly >= 1 && ly <= e1 - 2)) &&
                     (DIM < 3 || (lz >= 1 && lz <= e2d - 2));
    if (NF == 1 && a.fast && in1) {
      const int c0 = S.cop[lz * ec01 + ly * ec0 + lx], s0 = S.csm[lz * ec01 + ly * ec0 + lx];
      bool op = c0 != kNoCell && (c0 & ~kScaleBit) == 0, sm = !a.jacobi && s0 != kNoCell && (s0 & ~kScaleBit) == MM;
      for (int kc = 1; kc < NC; ++kc) {
        const int cl = (lz - ((kc >> 2) & 1)) * ec01 + (ly - ((kc >> 1) & 1)) * ec0 + (lx - (kc & 1));
        op = op && S.cop[cl] == c0;
        sm = sm && S.csm[cl] == s0;
      }
      if (op) f |= kVfOp | ((c0 & kScaleBit) ? kVfOpScaled : 0);
      if (sm) f |= kVfSm | ((s0 & kScaleBit) ? kVfSmScaled : 0);
    }
    S.vf[t] = (unsigned char)f;
  }
  // NF == 1: row lists, stencil rows first, so that warps do not diverge between the two
  // paths (the order inside a list does not change any value: rows are independent)
  __shared__ int lcnt[4];
  __shared__ int wcnt[32][4];
  if constexpr (NF == 1) {
    if (threadIdx.x < 4) lcnt[threadIdx.x] = 0;
    __syncthreads();
    const int gx = t0 + 2, gy = DIM > 1 ? t1 + 2 : 1, gz = DIM > 2 ? t2 + 2 : 1;
    const int ne1 = gx * gy * gz;
    const int lane = threadIdx.x & 31;
    for (int pass = 0; pass < 2; ++pass) {
      for (int t0 = 0; t0 < ne1; t0 += blockDim.x) {   // E1 entries, T entries flagged
        const int q = t0 + threadIdx.x;
        int l = 0, cb = 0;
        bool valid = false, inT = false;
        if (q < ne1) {
          const int lx = q % gx + 1, ly = DIM > 1 ? (q / gx) % gy + 1 : 0, lz = DIM > 2 ? q / (gx * gy) + 1 : 0;
          l = (lz * e1 + ly) * e0 + lx;
          cb = (lz * ec1 + ly) * ec0 + lx;
          valid = S.gidx[l] >= 0;
          inT = lx >= 2 && lx <= e0 - 3 && (DIM < 2 || (ly >= 2 && ly <= e1 - 3)) && (DIM < 3 || (lz >= 2 && lz <= e2d - 3));
        }
        const int f = valid ? S.vf[l] : 0;
        const unsigned lt = (1u << lane) - 1u;
        // smoother list (counter 0 = fast, 1 = general), operator list (2, 3).  Slots are
        // assigned in (chunk, warp, lane) order -- a deterministic row order, so each thread's
        // dot-product partials (and the block sums) are summed in the same order every launch
        const int wid = threadIdx.x >> 5;
        unsigned bfw[2], bgw[2];
        bool inw[2], fastw[2];
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          inw[w] = valid && (w == 0 || inT);
          fastw[w] = inw[w] && (f & (w == 0 ? kVfSm : kVfOp));
          bfw[w] = __ballot_sync(0xffffffffu, fastw[w]);
          bgw[w] = __ballot_sync(0xffffffffu, inw[w] && !fastw[w]);
          if (lane == 0) { wcnt[wid][2 * w] = __popc(bfw[w]); wcnt[wid][2 * w + 1] = __popc(bgw[w]); }
        }
        __syncthreads();
        if (pass == 1) {
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            int bfo = lcnt[2 * w], bgo = lcnt[2 * w + 1];
            for (int v = 0; v < wid; ++v) { bfo += wcnt[v][2 * w]; bgo += wcnt[v][2 * w + 1]; }
            int* lst = w == 0 ? S.lsm : S.lop;
            if (fastw[w]) lst[bfo + __popc(bfw[w] & lt)] = l | (cb << 16);
            else if (inw[w]) lst[bgo + __popc(bgw[w] & lt)] = l | (cb << 16);
          }
        }
        __syncthreads();
        if (threadIdx.x < 4)
          for (int v = 0; v < (int)(blockDim.x >> 5); ++v) lcnt[threadIdx.x] += wcnt[v][threadIdx.x];
        __syncthreads();
      }
      __syncthreads();
      if (pass == 0) {
        S.nsm = lcnt[0] + lcnt[1];
        S.nop = lcnt[2] + lcnt[3];
        __syncthreads();
        if (threadIdx.x == 0) { lcnt[1] = lcnt[0]; lcnt[0] = 0; lcnt[3] = lcnt[2]; lcnt[2] = 0; }
        __syncthreads();
      }
    }
  }
  // regions in local E2 coordinates: E1 = [1, tile+2], T = [2, tile+1] per present axis
  const int g1x = t0 + 2, g1y = DIM > 1 ? t1 + 2 : 1, g1z = DIM > 2 ? t2 + 2 : 1;
  const int nE1 = g1x * g1y * g1z;
  const int nT = S.T;
  const int shy1 = DIM > 1 ? 1 : 0, shz1 = DIM > 2 ? 1 : 0;
  const int shy2 = DIM > 1 ? 2 : 0, shz2 = DIM > 2 ? 2 : 0;
  auto t_local = [&](int q) {   // T entry q -> E2 linear index
    const int lx = q % t0 + 2, ly = (q / t0) % t1 + shy2, lz = q / (t0 * t1) + shz2;
    return (lz * e1 + ly) * e0 + lx;
  };

  auto smooth_E1 = [&]() {   // u = M r on E1
    if constexpr (NF == 1) {
      for (int k = threadIdx.x; k < S.nsm; k += blockDim.x) {
        const int e = S.lsm[k], l = e & 0xffff;
        S.u[l] = a.jacobi ? __ldg(a.diag_inv + S.gidx[l]) * S.r[l]
                          : vertex_row<DIM, NF, true>(a, S, S.r, l, e >> 16, 0);
      }
    } else {
    for (int t = threadIdx.x; t < NF * nE1; t += blockDim.x) {
      const int i = t / nE1, q = t % nE1;
      const int lx = q % g1x + 1, ly = (q / g1x) % g1y + shy1, lz = q / (g1x * g1y) + shz1;
      const int l = (lz * e1 + ly) * e0 + lx;
      const int gi = S.gidx[i * E2 + l];
      double u = 0.0;
      if (gi >= 0) {
        if (a.jacobi) u = __ldg(a.diag_inv + gi) * S.r[i * E2 + l];
        else u = vertex_row<DIM, NF, true>(a, S, S.r, l, (lz * ec1 + ly) * ec0 + lx, i);
      }
      S.u[i * E2 + l] = u;
    }
    }
  };
  // w = A u on T; publish w; partials (r,u), (w,u), (r,r)
  auto apply_T = [&](double* wout, double& g, double& dl, double& rh) {
    g = 0.0; dl = 0.0; rh = 0.0;
    if constexpr (NF == 1) {
      for (int k = threadIdx.x; k < S.nop; k += blockDim.x) {
        const int e = S.lop[k], l = e & 0xffff;
        const double w = vertex_row<DIM, NF, false>(a, S, S.u, l, e >> 16, 0);
        __stcg(wout + S.gidx[l], w);
        const double ri = S.r[l], ui = S.u[l];
        g = fma(ri, ui, g);
        dl = fma(w, ui, dl);
        rh = fma(ri, ri, rh);
      }
    } else {
    for (int t = threadIdx.x; t < NF * nT; t += blockDim.x) {
      const int i = t / nT, q = t % nT;
      const int lx = q % t0 + 2, ly = (q / t0) % t1 + shy2, lz = q / (t0 * t1) + shz2;
      const int l = (lz * e1 + ly) * e0 + lx;
      const int gi = S.gidx[i * E2 + l];
      if (gi < 0) continue;
      const double w = vertex_row<DIM, NF, false>(a, S, S.u, l, (lz * ec1 + ly) * ec0 + lx, i);
      __stcg(wout + gi, w);
      const double ri = S.r[i * E2 + l], ui = S.u[i * E2 + l];
      g = fma(ri, ui, g);
      dl = fma(w, ui, dl);
      rh = fma(ri, ri, rh);
    }
    }
  };

  // the arrival counter continues from the previous launch (every block passed the same
  // number of barriers, so it is a multiple of gridDim.x here)
  const unsigned cnt0 = t_ld_relaxed(&a.ctl->base);
  unsigned gen = 0;
  double g_loc, d_loc, r_loc;
  smooth_E1();
  __syncthreads();
  apply_T(a.wpub[0], g_loc, d_loc, r_loc);
  // w halo of the current generation, preloaded right after each barrier (overlaps the
  // partial-sum reduction); the first 4*blockDim entries of E2 live in registers
  double wl[4];
  auto preload_w = [&](const double* wv) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = k * blockDim.x + threadIdx.x;
      const int gi = t < NF * E2 ? S.gidx[t] : -1;
      wl[k] = gi >= 0 ? __ldcg(wv + gi) : 0.0;
    }
  };
  const unsigned long long G0 = *(volatile const unsigned long long*)&a.ctl->gbase;   // generation before this launch
  tiled_arrive_wait(g_loc, d_loc, r_loc, a.part, a.ctl, cnt0 + (gen + 1) * gridDim.x, gen + 1, red, a.acc, G0 + gen + 1);
  ++gen;
  preload_w(a.wpub[0]);
  tiled_totals(a.part, gen, tot, a.acc, G0 + gen);
  __syncthreads();
  double gamma = tot[0], delta = tot[1];
  const double rho0 = tot[2];
  double rho = rho0;
  double gamma_old = 1.0, alpha_old = 1.0;
  int it = 0;
  while (rho0 > 0.0 && !(rho < a.rtol2 * rho0) && it < a.maxit) {
    double beta, alpha;
    if (it == 0) {
      beta = 0.0;
      alpha = gamma / delta;
    } else {
      beta = gamma / gamma_old;
      alpha = gamma / (delta - beta * gamma / alpha_old);
    }
    if (!(alpha > 0.0) || !(gamma > 0.0)) break;   // breakdown (not SPD): keep x_it
    const unsigned long long tp0 = a.prof ? t_now() : 0ull;
    // s = w + beta s, r -= alpha s on E2 (w of the neighbours published before the barrier)
    const double* wv = a.wpub[it & 1];
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // preloaded part
      const int t = k * blockDim.x + threadIdx.x;
      if (t < NF * E2 && S.gidx[t] >= 0) {
        const double sv = fma(beta, S.s[t], wl[k]);
        S.s[t] = sv;
        S.r[t] = fma(-alpha, sv, S.r[t]);
      }
    }
    for (int t = 4 * blockDim.x + threadIdx.x; t < NF * E2; t += blockDim.x) {   // rest (large bricks)
      const int gi = S.gidx[t];
      if (gi < 0) continue;
      const double sv = fma(beta, S.s[t], __ldcg(wv + gi));
      S.s[t] = sv;
      S.r[t] = fma(-alpha, sv, S.r[t]);
    }
    // p = u + beta p, x += alpha p on T
    for (int t = threadIdx.x; t < NF * nT; t += blockDim.x) {
      const int i = t / nT, q = t % nT;
      const double pv = fma(beta, S.p[t], S.u[i * E2 + t_local(q)]);
      S.p[t] = pv;
      S.x[t] = fma(alpha, pv, S.x[t]);
    }
    ++it;
    gamma_old = gamma;
    alpha_old = alpha;
    __syncthreads();
    const unsigned long long tp1 = a.prof ? t_now() : 0ull;
    smooth_E1();
    __syncthreads();
    const unsigned long long tp2 = a.prof ? t_now() : 0ull;
    apply_T(a.wpub[it & 1], g_loc, d_loc, r_loc);
    __syncthreads();
    const unsigned long long tp3 = a.prof ? t_now() : 0ull;
    tiled_arrive_wait(g_loc, d_loc, r_loc, a.part, a.ctl, cnt0 + (gen + 1) * gridDim.x, gen + 1, red, a.acc, G0 + gen + 1);
    ++gen;
    preload_w(a.wpub[it & 1]);
    tiled_totals(a.part, gen, tot, a.acc, G0 + gen);
    __syncthreads();
    if (a.prof && threadIdx.x == 0) {
      const unsigned long long tp4 = t_now();
      unsigned long long* pr = a.prof + 4 * blockIdx.x;
      pr[0] += tp1 - tp0; pr[1] += tp2 - tp1; pr[2] += tp3 - tp2; pr[3] += tp4 - tp3;
    }
    gamma = tot[0];
    delta = tot[1];
    rho = tot[2];
  }
  // x on T -> global
  for (int t = threadIdx.x; t < NF * nT; t += blockDim.x) {
    const int i = t / nT, q = t % nT;
    const int gi = S.gidx[i * E2 + t_local(q)];
    if (gi >= 0) a.x[gi] = S.x[t];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.iters[0] = it;
    a.iters[1] += it;
    a.ctl->base = cnt0 + gen * gridDim.x;   // every block has read base (all passed barrier 1)
    a.ctl->gbase = G0 + gen;
  }
}

}  // namespace fcm
