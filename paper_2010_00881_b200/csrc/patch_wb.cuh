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
// k_patch_wb: one CTA per patch (grid-stride), 256 threads.  Gather r over the patch slots into a
// (2q+1)^d tensor, z = FD(r), w = C z_S (a warp per row), v = FD(P_S w), x += coef (z - v) on the
// present slots (fp64 atomics, patches overlap).
#pragma once
#include <cstdint>

#include "patch.cuh"

namespace fcm {

constexpr int kWbThreads = 256;
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

// one axis contraction of an S^DIM tensor in shared memory: out[.., m, ..] = sum_s T(s, m) in[.., s, ..]
// (fwd) or out[.., s, ..] = sum_m T(s, m) in[.., m, ..] (bwd) along axis ax; T row-major S x S
template <int S, int DIM>
__device__ __forceinline__ void wb_axis(const double* __restrict__ in, double* __restrict__ out,
                                        const double* __restrict__ T, int ax, bool fwd) {
  constexpr int N = DIM == 3 ? S * S * S : S * S;
  const int st = ax == 0 ? 1 : (ax == 1 ? S : S * S);
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int c = (e / st) % S;          // this output's coordinate along ax
    const int b = e - c * st;            // the tensor position with coordinate 0 along ax
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) s = fma(fwd ? T[j * S + c] : T[c * S + j], in[b + j * st], s);
    out[e] = s;
  }
  __syncthreads();
}

// t <- A0^{-1} t (fast diagonalisation), w: scratch of the same size; tx/ty/tz: the patch's tables
template <int S, int DIM>
__device__ __forceinline__ void wb_fd(double* t, double* w, const double* tx, const double* ty, const double* tz,
                                      double s_fac) {
  constexpr int N = DIM == 3 ? S * S * S : S * S;
  const double* tab[3] = {tx, ty, tz};
  // forward: modes along x, y (, z)
  wb_axis<S, DIM>(t, w, tab[0], 0, true);
  wb_axis<S, DIM>(w, t, tab[1], 1, true);
  double* cur = t;
  double* oth = w;
  if (DIM == 3) {
    wb_axis<S, DIM>(t, w, tab[2], 2, true);
    cur = w;
    oth = t;
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int mx = e % S, my = (e / S) % S, mz = DIM == 3 ? e / (S * S) : 0;
    double lam = tx[S * S + mx] + ty[S * S + my] + (DIM == 3 ? tz[S * S + mz] : 0.0);
    cur[e] = cur[e] / (s_fac * lam);
  }
  __syncthreads();
  // backward
  if (DIM == 3) {
    wb_axis<S, DIM>(cur, oth, tab[2], 2, false);
    wb_axis<S, DIM>(oth, cur, tab[1], 1, false);
    wb_axis<S, DIM>(cur, oth, tab[0], 0, false);
    // result in oth == t
  } else {
    wb_axis<S, DIM>(cur, oth, tab[1], 1, false);
    wb_axis<S, DIM>(oth, cur, tab[0], 0, false);
    // result in cur == t
  }
}

template <int S, int DIM>
__global__ void __launch_bounds__(kWbThreads) k_patch_wb(PatchWbOp op) {
  constexpr int N = DIM == 3 ? S * S * S : S * S;
  constexpr int TSZ = S * S + S;
  extern __shared__ __align__(16) unsigned char wb_sm[];
  Tab& T = *reinterpret_cast<Tab*>(wb_sm);
  double* z = reinterpret_cast<double*>(wb_sm + (sizeof(Tab) + 15) / 16 * 16);   // [N]
  double* u = z + N;                      // [N]
  double* wk = u + N;                     // [N] scratch
  double* zs = wk + N;                    // [kWbMaxK]
  double* ws = zs + kWbMaxK;              // [kWbMaxK]
  double* tb = ws + kWbMaxK;              // [3][TSZ] tables of this patch
  int* ids = reinterpret_cast<int*>(tb + 3 * TSZ);   // [mb]
  load_tab_from(T, op.m, op.base, op.stride3, op.cmin, op.cmax);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int64_t p = blockIdx.x; p < op.n_wb; p += gridDim.x) {
    const int64_t A = op.anchors[p];
    const int ac[3] = {(int)(A % op.na[0]), (int)((A / op.na[0]) % op.na[1]),
                       (int)(A / ((int64_t)op.na[0] * op.na[1]))};
    // tables of the patch's axis classes
    int coff = 0;
    for (int ax = 0; ax < 3; ++ax) {
      const int c = op.cls[coff + ac[ax]];
      for (int e = threadIdx.x; e < TSZ; e += blockDim.x) tb[ax * TSZ + e] = op.tabs[((size_t)ax * op.ncls + c) * TSZ + e];
      coff += op.na[ax];
    }
    for (int e = threadIdx.x; e < N; e += blockDim.x) z[e] = 0.0;
    __syncthreads();
    // gather r over the present slots
    for (int l = threadIdx.x; l < op.mb; l += blockDim.x) {
      const int km = op.mem[l], a = op.loc[l];
      const int cx = ac[0] + op.mo[km][0], cy = ac[1] + op.mo[km][1], cz = ac[2] + op.mo[km][2];
      const bool ok = cx >= 0 && cy >= 0 && cz >= 0 && cx < op.nx && cy < op.ny && cz < op.nz && dof_free(T, a, cx, cy, cz);
      const int idx = ok ? dof_index(T, a, cx, cy, cz) : -1;
      ids[l] = idx;
      if (idx >= 0) z[op.tsl[l]] = __ldg(op.in + idx);
    }
    __syncthreads();
    wb_fd<S, DIM>(z, wk, tb, tb + TSZ, tb + 2 * TSZ, op.s_fac);   // z = A0^{-1} r
    // w = C z_S
    const int64_t s0 = op.soff[p];
    const int k = (int)(op.soff[p + 1] - s0);
    const double* Cp = op.C + op.coff[p];
    for (int j = threadIdx.x; j < k; j += blockDim.x) zs[j] = z[op.tsl[op.slots[s0 + j]]];
    for (int e = threadIdx.x; e < N; e += blockDim.x) u[e] = 0.0;
    __syncthreads();
    for (int i = warp; i < k; i += nwarp) {
      double s = 0.0;
      for (int j = lane; j < k; j += 32) s = fma(__ldg(Cp + (int64_t)i * k + j), zs[j], s);
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) u[op.tsl[op.slots[s0 + i]]] = s;
    }
    __syncthreads();
    wb_fd<S, DIM>(u, wk, tb, tb + TSZ, tb + 2 * TSZ, op.s_fac);   // u = A0^{-1} P_S w
    for (int l = threadIdx.x; l < op.mb; l += blockDim.x) {
      const int idx = ids[l];
      if (idx >= 0) {
        const int t = op.tsl[l];
        atomicAdd(op.out + idx, op.coef * (z[t] - u[t]));
      }
    }
    __syncthreads();
  }
}

template <int S, int DIM>
__host__ size_t wb_smem(int mb) {
  constexpr int N = DIM == 3 ? S * S * S : S * S;
  return (sizeof(Tab) + 15) / 16 * 16 + (size_t)3 * N * 8 + (size_t)2 * kWbMaxK * 8 + (size_t)3 * (S * S + S) * 8 +
         (size_t)mb * 4;
}

}  // namespace fcm
