// patch_wb.cuh -- individual Schwarz patches as low-rank corrections of the regular patch
// (additive Schwarz, Eq. AdditiveSchwarz, patchwise blocks P:259).
//
// An individual patch whose 2^d member cells are all uncut and physical differs from the regular
// patch of its boundary class only through its outer ring of assembly cells (cut or fictitious
// cells of the 4^d neighbourhood): A_i = A0 + P_S E P_S^T, where S are the k patch slots touched by
// those cells (k = 1 .. ~220 of 729 at q = 4) and E = sum over the ring's non-regular cells of
// (K_c - K_ref) on S.  A0 is a Kronecker sum of assembled 1D matrices, so A0^{-1} is the fast
// diagonalisation (S_z (x) S_y (x) S_x) D^{-1} (.)^T of patch.cuh.  With G = P_S^T A0^{-1} P_S,
// H = G^{-1} (the Schur complement of A0 onto S) and F = H + E (that of A_i, SPD), Woodbury gives
//     A_i^{-1} r = z - A0^{-1} P_S C P_S^T z,   z = A0^{-1} r,   C = H - H F^{-1} H   (k x k),
// exact in exact arithmetic.  Setup (fcm_mg.cu, setup_patch_wb) computes C per patch; the sweep
// streams k^2 doubles per patch instead of the 729 * 730 / 2 of an explicit inverse (config 3:
// 27.7k of the 60.8k level-4 individual patches, mean k = 41: 59 GB less per sweep) and spends two
// fast diagonalisations instead.
//
// k_patch_wb: NG groups of GW warps per CTA, a group per patch (grid-stride).  Gather r over the
// patch slots into a (2q+1)^d tensor, z = FD(r) (line-based: a thread per tensor line), w = C z_S
// (a warp per row), v = FD(P_S w), x += coef (z - v) on the present slots (fp64 atomics, patches
// overlap).
#pragma once
#include <cstdint>

#include "patch.cuh"

namespace fcm {

constexpr int kWbMaxK = 256;

struct PatchWbOp {
  int nx, ny, nz, dim;
  int na[3];
  int q, S, mb, ncls;
  int64_t n_wb;
  const int64_t* anchors;     // [n_wb]
  const int64_t* soff;        // [n_wb + 1] offsets into slots
  const int16_t* slots;       // S lists: block slot indices
  const int64_t* coff;        // [n_wb + 1] offsets into C
  const double* C;            // per patch k x k row-major
  const int16_t* tsl;         // [mb] tensor slot (linear, x fastest) of block slot l
  const int8_t* mem;          // [mb] member cell of slot l
  const int16_t* loc;         // [mb] local DOF of slot l
  int mo[8][3];
  const int* cls;             // [na0 + na1 + na2] FD axis class of each anchor coordinate
  const double* tabs;         // [3][ncls][S*S + S]
  double s_fac;
  const int64_t* base;
  const int32_t* stride3;
  const int16_t* cmin;
  const int16_t* cmax;
  int m;
  const double* in;
  double* out;
  double coef;
};

// Line-based fast diagonalisation of one patch by a group of GW warps: a thread owns one line of
// the S^DIM tensor along the contracted axis (S values in registers, S outputs; the factor is read
// as warp-uniform shared-memory broadcasts), D^-1 fused into the last forward axis.
template <int S, int DIM>
struct WbShape {
  static constexpr int N = DIM == 3 ? S * S * S : S * S;
  static constexpr int LINES = N / S;
  static constexpr int GW = (LINES + 31) / 32;          // warps per patch group
  static constexpr int NG = GW >= 8 ? 1 : 8 / GW;        // patch groups per CTA
  static constexpr int TSZ = S * S + S;
  // per-group shared memory (doubles): 3 tensors, zS / w, the three axis tables; then ids (int)
  static constexpr int GD = 3 * N + 2 * kWbMaxK + 3 * TSZ;
};

__device__ __forceinline__ void wb_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// out = contraction of in along axis ax (fwd: out[c] = sum_j T[j][c] in[j]; bwd: out[c] = sum_j
// T[c][j] in[j]); scale != nullptr: the last forward axis, out /= s_fac (lam_x + lam_y + lam_z)
template <int S, int DIM>
__device__ __forceinline__ void wb_line(const double* __restrict__ in, double* __restrict__ out,
                                        const double* __restrict__ T, int ax, bool fwd, int t,
                                        const double* tabs3, double s_fac, bool scale) {
  constexpr int LINES = WbShape<S, DIM>::LINES;
  constexpr int TSZ = WbShape<S, DIM>::TSZ;
  if (t >= LINES) return;
  int b, st;
  if (ax == 0) { b = t * S; st = 1; }
  else if (ax == 1) { b = (t / S) * S * S + t % S; st = S; }
  else { b = t; st = S * S; }
  double v[S];
#pragma unroll
  for (int j = 0; j < S; ++j) v[j] = in[b + j * st];
  double lam0 = 0.0;
  if (scale) {   // the line's fixed coordinates (the last forward axis is ax = DIM - 1)
    const int mx = b % S, my = (b / S) % S;
    lam0 = DIM == 3 ? tabs3[S * S + mx] + tabs3[TSZ + S * S + my] : tabs3[S * S + mx];
  }
#pragma unroll
  for (int c = 0; c < S; ++c) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) s = fma(fwd ? T[j * S + c] : T[c * S + j], v[j], s);
    if (scale) s /= s_fac * (lam0 + T[S * S + c]);
    out[b + c * st] = s;
  }
}

// t <- A0^{-1} t; w scratch; tb: the patch's three axis tables [3][TSZ]
template <int S, int DIM>
__device__ __forceinline__ void wb_fd_lines(double* t, double* w, const double* tb, double s_fac, int tid,
                                            int bar_id, int nthr) {
  constexpr int TSZ = WbShape<S, DIM>::TSZ;
  if (DIM == 3) {
    wb_line<S, DIM>(t, w, tb, 0, true, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(w, t, tb + TSZ, 1, true, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(t, w, tb + 2 * TSZ, 2, true, tid, tb, s_fac, true);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(w, t, tb + 2 * TSZ, 2, false, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(t, w, tb + TSZ, 1, false, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(w, t, tb, 0, false, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
  } else {
    wb_line<S, DIM>(t, w, tb, 0, true, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(w, t, tb + TSZ, 1, true, tid, tb, s_fac, true);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(t, w, tb + TSZ, 1, false, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
    wb_line<S, DIM>(w, t, tb, 0, false, tid, tb, s_fac, false);
    wb_bar(bar_id, nthr);
  }
}

// NG groups of GW warps per CTA, each group one patch at a time (patches p = blockIdx.x NG + g,
// stride gridDim.x NG), synchronised by named barrier 1 + g
template <int S, int DIM>
__global__ void __launch_bounds__(WbShape<S, DIM>::NG * WbShape<S, DIM>::GW * 32) k_patch_wb(PatchWbOp op) {
  using SH = WbShape<S, DIM>;
  constexpr int N = SH::N, TSZ = SH::TSZ, GW = SH::GW, NG = SH::NG;
  extern __shared__ __align__(16) unsigned char wb_sm[];
  Tab& T = *reinterpret_cast<Tab*>(wb_sm);
  const int g = threadIdx.x / (GW * 32), tid = threadIdx.x % (GW * 32), nthr = GW * 32;
  const int lane = tid & 31, warp = tid >> 5;
  double* gbase = reinterpret_cast<double*>(wb_sm + (sizeof(Tab) + 15) / 16 * 16);
  double* z = gbase + (size_t)g * SH::GD;   // [N]
  double* u = z + N;                        // [N]
  double* wk = u + N;                       // [N]
  double* zs = wk + N;                      // [kWbMaxK]
  double* tb = zs + 2 * kWbMaxK;            // [3][TSZ]
  int* ids = reinterpret_cast<int*>(gbase + (size_t)NG * SH::GD) + (size_t)g * op.mb;
  load_tab_from(T, op.m, op.base, op.stride3, op.cmin, op.cmax);
  __syncthreads();
  const int bar_id = 1 + g;
  for (int64_t p = (int64_t)blockIdx.x * NG + g; p < op.n_wb; p += (int64_t)gridDim.x * NG) {
    const int64_t A = op.anchors[p];
    const int ac[3] = {(int)(A % op.na[0]), (int)((A / op.na[0]) % op.na[1]),
                       (int)(A / ((int64_t)op.na[0] * op.na[1]))};
    int coff = 0;
    for (int ax = 0; ax < 3; ++ax) {
      const int c = op.cls[coff + ac[ax]];
      for (int e = tid; e < TSZ; e += nthr) tb[ax * TSZ + e] = op.tabs[((size_t)ax * op.ncls + c) * TSZ + e];
      coff += op.na[ax];
    }
    for (int e = tid; e < N; e += nthr) {
      z[e] = 0.0;
      u[e] = 0.0;
    }
    wb_bar(bar_id, nthr);
    for (int l = tid; l < op.mb; l += nthr) {   // gather r over the present slots
      const int km = op.mem[l], a = op.loc[l];
      const int cx = ac[0] + op.mo[km][0], cy = ac[1] + op.mo[km][1], cz = ac[2] + op.mo[km][2];
      const bool ok = cx >= 0 && cy >= 0 && cz >= 0 && cx < op.nx && cy < op.ny && cz < op.nz && dof_free(T, a, cx, cy, cz);
      const int idx = ok ? dof_index(T, a, cx, cy, cz) : -1;
      ids[l] = idx;
      if (idx >= 0) z[op.tsl[l]] = __ldg(op.in + idx);
    }
    wb_bar(bar_id, nthr);
    wb_fd_lines<S, DIM>(z, wk, tb, op.s_fac, tid, bar_id, nthr);   // z = A0^{-1} r
    const int64_t s0 = op.soff[p];
    const int k = (int)(op.soff[p + 1] - s0);
    const double* Cp = op.C + op.coff[p];
    for (int j = tid; j < k; j += nthr) zs[j] = z[op.tsl[op.slots[s0 + j]]];
    wb_bar(bar_id, nthr);
    for (int i = warp; i < k; i += GW) {          // w = C z_S, a warp per row
      double s = 0.0;
      for (int j = lane; j < k; j += 32) s = fma(__ldg(Cp + (int64_t)i * k + j), zs[j], s);
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) u[op.tsl[op.slots[s0 + i]]] = s;
    }
    wb_bar(bar_id, nthr);
    wb_fd_lines<S, DIM>(u, wk, tb, op.s_fac, tid, bar_id, nthr);   // u = A0^{-1} P_S w
    for (int l = tid; l < op.mb; l += nthr) {
      const int idx = ids[l];
      if (idx >= 0) {
        const int t = op.tsl[l];
        atomicAdd(op.out + idx, op.coef * (z[t] - u[t]));
      }
    }
    wb_bar(bar_id, nthr);
  }
}

template <int S, int DIM>
__host__ constexpr int wb_threads() { return WbShape<S, DIM>::NG * WbShape<S, DIM>::GW * 32; }

template <int S, int DIM>
__host__ size_t wb_smem(int mb) {
  using SH = WbShape<S, DIM>;
  return (sizeof(Tab) + 15) / 16 * 16 + (size_t)SH::NG * SH::GD * 8 + (size_t)SH::NG * mb * 4;
}

}  // namespace fcm
