// quad.cu -- cut-cell space-tree quadrature on the device (SETUP).
//
// The same integral as the host generator (gen.cpp) and the oracle (oracle/quadrature.py):
// Poisson K_ab = int alpha grad N_a . grad N_b, f_a = int alpha N_a (Eq. weakform),
// cut cells integrated on a space tree of depth `depth` (reading R13): only cut
// boxes are bisected; uncut leaves are integrated exactly in Kronecker form from 1D
// sub-interval integrals; depth-limit cut leaves use a (p+1)^d Gauss rule with alpha per point.
//
// One CTA per cut cell:
//  1. every depth-D sub-box walks its ancestor chain (midpoints computed exactly like the host
//     recursion, round-to-nearest intrinsics, so box classification is bit-identical) and the
//     leaves are collected in shared memory (a full leaf at level l is recorded once, by the
//     descendant whose lower digits are zero);
//  2. the lower triangle of K is held in registers as 4x4 blocks (block pairs distributed over
//     the threads); a full leaf adds alpha*jac*g2*sum_g prod_a (K|M)_a from per-axis 1D tables;
//     a point leaf's Gauss points are processed in chunks of kQB points whose physical
//     gradients (and values, for f) are staged in shared memory, each thread then doing
//     register-blocked rank-1 updates of its blocks.
// Poisson only (elasticity keeps the host generator); m <= 128, depth <= 4.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/fcm_mg.h"
#include "common.hpp"
#include "layout.hpp"

namespace fcm {
namespace {

constexpr int kQThreads = 256;
constexpr int kQB = 16;          // Gauss points per staged chunk
constexpr int kQMaxNm = 128;
constexpr int kQMaxP = 8;
constexpr int kQMaxLeaves = 4096;   // 8^4 (depth <= 4)

struct QuadArgs {
  int dim, p, nm, depth;
  double h, alpha;
  int nx, ny;
  int64_t ncut;
  const int64_t* cells;   // [ncut] cell indices
  const int32_t* vptr;    // [ncut + 1] CSR: voids that touch cell i
  const int32_t* vidx;
  const double* vc;       // [nv * dim]
  const double* vr;       // [nv]
  double* K;              // [ncut][nm*nm]
  double* f;              // [ncut][nm]
};

__constant__ int c_modek[kQMaxNm * 3];
__constant__ double c_gx[kQMaxP + 1], c_gw[kQMaxP + 1];

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Voids::classify of gen.cpp over the cell's void list (same operation order, no contraction)
__device__ int q_classify(const double* lo, const double* hi, int dim, const QuadArgs& a, int v0, int v1) {
  bool misses_all = true;
  for (int t = v0; t < v1; ++t) {
    const int j = a.vidx[t];
    double far2 = 0, near2 = 0;
    for (int ax = 0; ax < dim; ++ax) {
      const double cc = a.vc[j * dim + ax];
      const double d0 = dsub(lo[ax], cc), d1 = dsub(hi[ax], cc);
      far2 = dadd(far2, fmax(dmul(d0, d0), dmul(d1, d1)));
      const double nr = fmax(0.0, fmax(dsub(lo[ax], cc), dsub(cc, hi[ax])));
      near2 = dadd(near2, dmul(nr, nr));
    }
    const double r2 = dmul(a.vr[j], a.vr[j]);
    if (far2 < r2) return 1;
    if (near2 < r2) misses_all = false;
  }
  return misses_all ? 0 : 2;
}
__device__ bool q_fict(const double* x, int dim, const QuadArgs& a, int v0, int v1) {
  for (int t = v0; t < v1; ++t) {
    const int j = a.vidx[t];
    double d2 = 0;
    for (int ax = 0; ax < dim; ++ax) {
      const double s = dsub(x[ax], a.vc[j * dim + ax]);
      d2 = dadd(d2, dmul(s, s));
    }
    if (d2 < dmul(a.vr[j], a.vr[j])) return true;
  }
  return false;
}

// 1D modes 0..p (integrated Legendre, reading R-B1) and derivatives at xi
__device__ __forceinline__ void q_modes1d(int p, double xi, double* v, double* d) {
  double P[kQMaxP + 2];
  P[0] = 1.0;
  P[1] = xi;
  for (int k = 1; k < p; ++k) P[k + 1] = ((2 * k + 1) * xi * P[k] - k * P[k - 1]) / (k + 1);
  v[0] = 0.5 * (1.0 - xi); d[0] = -0.5;
  v[1] = 0.5 * (1.0 + xi); d[1] = 0.5;
  for (int k = 2; k <= p; ++k) {
    v[k] = (P[k] - P[k - 2]) * rsqrt(2.0 * (2 * k - 1));
    d[k] = sqrt(0.5 * (2 * k - 1)) * P[k - 1];
  }
}

// physical box of the level-l ancestor of depth-D box b (host recursion: midpoints of the parent)
__device__ void q_box(int b, int l, int D, int dim, const double* clo, double h, double* lo, double* hi) {
  for (int ax = 0; ax < dim; ++ax) { lo[ax] = clo[ax]; hi[ax] = dadd(clo[ax], h); }
  for (int k = 1; k <= l; ++k) {
    const int child = (b >> (dim * (D - k))) & ((1 << dim) - 1);
    for (int ax = 0; ax < dim; ++ax) {
      const double mid = dmul(0.5, dadd(lo[ax], hi[ax]));
      if (child >> ax & 1) lo[ax] = mid; else hi[ax] = mid;
    }
  }
}

template <int BPT>
__global__ void __launch_bounds__(kQThreads) k_cut_quadrature(QuadArgs a) {
  __shared__ int leaves[kQMaxLeaves];      // (level << 24) | point flag << 23 | kind << 21 | box index
  __shared__ int scan[kQThreads];
  extern __shared__ __align__(16) double qsm[];
  double (*G)[3][kQMaxNm] = reinterpret_cast<double (*)[3][kQMaxNm]>(qsm);           // [kQB] gradients
  double (*V)[kQMaxNm] = reinterpret_cast<double (*)[kQMaxNm]>(qsm + kQB * 3 * kQMaxNm);  // [kQB] values
  __shared__ double W[kQB];                // w * alpha * jac
  __shared__ double T1[3][2][(kQMaxP + 1) * (kQMaxP + 1)];   // full leaf: per-axis M, K
  __shared__ double F1[3][kQMaxP + 1];
  __shared__ double leaf_al;
  const int dim = a.dim, p = a.p, nm = a.nm, D = a.depth, P1 = p + 1;
  const int nbox = 1 << (dim * D);
  const int NB = (nm + 3) / 4;
  const int nblk = NB * (NB + 1) / 2;
  const double h = a.h;
  const double jac = pow(0.5 * h, dim), g2 = (2.0 / h) * (2.0 / h);
  for (int64_t ci = blockIdx.x; ci < a.ncut; ci += gridDim.x) {
    const int64_t c = a.cells[ci];
    double clo[3] = {0, 0, 0};
    clo[0] = dmul((double)(c % a.nx), h);
    clo[1] = dmul((double)((c / a.nx) % a.ny), h);
    if (dim == 3) clo[2] = dmul((double)(c / ((int64_t)a.nx * a.ny)), h);
    const int v0 = a.vptr[ci], v1 = a.vptr[ci + 1];
    // ---- 1. leaves, in box order (deterministic): count, block scan, write ----------------
    const int per = (nbox + blockDim.x - 1) / blockDim.x;
    auto leaf_code = [&](int b) -> int {   // -1: not the representative of a leaf
      for (int l = 0; l <= D; ++l) {
        double lo[3], hi[3];
        q_box(b, l, D, dim, clo, h, lo, hi);
        const int kind = q_classify(lo, hi, dim, a, v0, v1);
        if (kind != 2) {
          const int low = dim * (D - l);
          return (b & ((1 << low) - 1)) == 0 ? ((l << 24) | (kind << 21) | b) : -1;
        }
      }
      return (D << 24) | (1 << 23) | b;   // cut down to the depth limit: point leaf
    };
    int cnt = 0;
    for (int b = threadIdx.x * per; b < min(nbox, (int)(threadIdx.x + 1) * per); ++b) cnt += leaf_code(b) >= 0;
    scan[threadIdx.x] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int t = 0; t < (int)blockDim.x; ++t) { const int v = scan[t]; scan[t] = run; run += v; }
      W[0] = (double)run;
    }
    __syncthreads();
    {
      int o = scan[threadIdx.x];
      for (int b = threadIdx.x * per; b < min(nbox, (int)(threadIdx.x + 1) * per); ++b) {
        const int code = leaf_code(b);
        if (code >= 0) leaves[o++] = code;
      }
    }
    const int nl = (int)W[0];
    __syncthreads();
    // ---- 2. accumulation --------------------------------------------------------------
    double acc[BPT][4][4];
#pragma unroll
    for (int k = 0; k < BPT; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[k][i][j] = 0.0;
    int bi[BPT], bj[BPT];
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      int t = threadIdx.x + k * blockDim.x;
      bi[k] = -1; bj[k] = -1;
      if (t < nblk) {   // lower block pair (bi >= bj) number t, row-major over the triangle
        int r = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
        while (r * (r + 1) / 2 > t) --r;
        while ((r + 1) * (r + 2) / 2 <= t) ++r;
        bi[k] = r;
        bj[k] = t - r * (r + 1) / 2;
      }
    }
    double facc = 0.0;   // f of mode threadIdx.x
    for (int li = 0; li < nl; ++li) {
      const int code = leaves[li];
      const int l = code >> 24, b = code & ((1 << 21) - 1);
      const bool point = (code >> 23) & 1;
      double lo[3], hi[3], rlo[3], rhi[3];
      q_box(b, l, D, dim, clo, h, lo, hi);
      for (int ax = 0; ax < dim; ++ax) {
        rlo[ax] = 2.0 * (lo[ax] - clo[ax]) / h - 1.0;
        rhi[ax] = 2.0 * (hi[ax] - clo[ax]) / h - 1.0;
      }
      if (!point) {
        const int kind = (code >> 21) & 3;
        if (threadIdx.x < dim * P1 * P1) {   // 1D integrals on the leaf interval
          const int ax = threadIdx.x / (P1 * P1), e = threadIdx.x % (P1 * P1), i = e / P1, j = e % P1;
          double m_ = 0, k_ = 0, f_ = 0;
          for (int g = 0; g < P1; ++g) {
            const double xi = 0.5 * (rlo[ax] + rhi[ax]) + 0.5 * (rhi[ax] - rlo[ax]) * c_gx[g];
            const double w = 0.5 * (rhi[ax] - rlo[ax]) * c_gw[g];
            double v[kQMaxP + 1], d[kQMaxP + 1];
            q_modes1d(p, xi, v, d);
            m_ += w * v[i] * v[j];
            k_ += w * d[i] * d[j];
            if (j == 0) f_ += w * v[i];
          }
          T1[ax][0][e] = m_;
          T1[ax][1][e] = k_;
          if (j == 0) F1[ax][i] = f_;
        }
        if (threadIdx.x == 0) leaf_al = kind == 1 ? a.alpha : 1.0;
        __syncthreads();
        const double s = leaf_al * jac * g2;
#pragma unroll
        for (int k = 0; k < BPT; ++k) {
          if (bi[k] < 0) continue;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int I = 4 * bi[k] + i;
            if (I >= nm) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int J = 4 * bj[k] + j;
              if (J >= nm || J > I) continue;
              double sum = 0.0;
              for (int g = 0; g < dim; ++g) {
                double t = 1.0;
                for (int ax = 0; ax < dim; ++ax)
                  t *= T1[ax][ax == g ? 1 : 0][c_modek[I * 3 + ax] * P1 + c_modek[J * 3 + ax]];
                sum += t;
              }
              acc[k][i][j] += s * sum;
            }
          }
        }
        if (threadIdx.x < nm) {
          double fv = leaf_al * jac;
          for (int ax = 0; ax < dim; ++ax) fv *= F1[ax][c_modek[threadIdx.x * 3 + ax]];
          facc += fv;
        }
        __syncthreads();
        continue;
      }
      // point leaf: (p+1)^d Gauss points, alpha per point, in chunks of kQB
      int npts = 1;
      for (int ax = 0; ax < dim; ++ax) npts *= P1;
      for (int q0 = 0; q0 < npts; q0 += kQB) {
        const int nq = min(kQB, npts - q0);
        for (int e = threadIdx.x; e < nq * nm; e += blockDim.x) {
          const int qq = e / nm, I = e % nm;
          int t = q0 + qq;
          double vv = 1.0, gg[3] = {1.0, 1.0, 1.0}, w = jac, x[3];
          for (int ax = 0; ax < dim; ++ax) {
            const int g = t % P1;
            t /= P1;
            const double xi = 0.5 * (rlo[ax] + rhi[ax]) + 0.5 * (rhi[ax] - rlo[ax]) * c_gx[g];
            w *= 0.5 * (rhi[ax] - rlo[ax]) * c_gw[g];
            double v[kQMaxP + 1], d[kQMaxP + 1];
            q_modes1d(p, xi, v, d);
            const int k = c_modek[I * 3 + ax];
            vv *= v[k];
            for (int gd = 0; gd < dim; ++gd) gg[gd] *= (gd == ax ? d[k] : v[k]);
            x[ax] = dadd(clo[ax], dmul(dmul(0.5, h), dadd(xi, 1.0)));
          }
          V[qq][I] = vv;
          for (int gd = 0; gd < 3; ++gd) G[qq][gd][I] = gd < dim ? gg[gd] * (2.0 / h) : 0.0;
          if (I == 0) W[qq] = w * (q_fict(x, dim, a, v0, v1) ? a.alpha : 1.0);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BPT; ++k) {
          if (bi[k] < 0) continue;
          const int I0 = 4 * bi[k], J0 = 4 * bj[k];
          for (int qq = 0; qq < nq; ++qq) {
            const double wq = W[qq];
            for (int gd = 0; gd < dim; ++gd) {
              double gi[4], gj[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                gi[i] = wq * G[qq][gd][I0 + i];   // I0 + i < 128 always (padded arrays)
                gj[i] = G[qq][gd][J0 + i];
              }
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[k][i][j] = fma(gi[i], gj[j], acc[k][i][j]);
            }
          }
        }
        if (threadIdx.x < nm)
          for (int qq = 0; qq < nq; ++qq) facc = fma(W[qq], V[qq][threadIdx.x], facc);
        __syncthreads();
      }
    }
    // ---- 3. output: lower triangle mirrored (exactly symmetric) ------------------------
    double* Ko = a.K + ci * (int64_t)nm * nm;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      if (bi[k] < 0) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int I = 4 * bi[k] + i, J = 4 * bj[k] + j;
          if (I >= nm || J >= nm || J > I) continue;
          Ko[(int64_t)I * nm + J] = acc[k][i][j];
          Ko[(int64_t)J * nm + I] = acc[k][i][j];
        }
    }
    if (threadIdx.x < nm) a.f[ci * (int64_t)nm + threadIdx.x] = facc;
    __syncthreads();
  }
}

}  // namespace
}  // namespace fcm

using namespace fcm;

#define QCU(call)                                                                            \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      rc = fail(e_ == cudaErrorMemoryAllocation ? FCM_ENOMEM : FCM_ECUDA, "%s: %s", #call,   \
                cudaGetErrorString(e_));                                                     \
      goto done;                                                                             \
    }                                                                                        \
  } while (0)

extern "C" int fcm_gen_cut_matrices_device(const fcm_grid* g, const fcm_physics* ph, int64_t n_voids,
                                           const double* centres, const double* radii, int64_t n_cut,
                                           const int64_t* cut_cells, double* cut_K, double* cut_f) {
  clear_error();
  if (!g || !ph) return fail(FCM_EINVAL, "NULL grid/physics");
  if (ph->kind != FCM_PHYS_POISSON || g->n_f != 1)
    return fail(FCM_EINVAL, "device quadrature: Poisson only (use fcm_gen_element_matrices)");
  if (ph->depth < 0 || ph->depth > 4) return fail(FCM_EINVAL, "device quadrature: depth must be <= 4");
  if (g->dim < 2 || g->dim > 3 || g->p < 1 || g->p > kQMaxP) return fail(FCM_EINVAL, "bad grid");
  if (n_cut < 0 || (n_cut > 0 && (!cut_cells || !cut_K))) return fail(FCM_EINVAL, "bad cut buffers");
  if (n_cut == 0) return FCM_OK;
  Layout L;
  L.build(g->dim, g->n, g->p, g->space, 1, g->dirichlet_faces);
  const int nm = (int)L.modes.size();
  if (nm > kQMaxNm) return fail(FCM_EINVAL, "device quadrature: m = %d > %d", nm, kQMaxNm);
  const int dim = g->dim;
  const int64_t nx = g->n[0], ny = g->n[1];
  const double h = g->h;
  // voids touching each cut cell (the host classify's "near" test on the cell box)
  std::vector<int32_t> vptr(n_cut + 1, 0);
  std::vector<std::vector<int32_t>> per(n_cut);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n_cut; ++i) {
    const int64_t c = cut_cells[i];
    double lo[3] = {(double)(c % nx) * h, (double)((c / nx) % ny) * h, dim == 3 ? (double)(c / (nx * ny)) * h : 0.0};
    for (int64_t j = 0; j < n_voids; ++j) {
      double near2 = 0;
      for (int a = 0; a < dim; ++a) {
        const double cc = centres[j * dim + a];
        const double nr = std::max(0.0, std::max(lo[a] - cc, cc - (lo[a] + h)));
        near2 += nr * nr;
      }
      if (near2 < radii[j] * radii[j]) per[i].push_back((int32_t)j);
    }
  }
  for (int64_t i = 0; i < n_cut; ++i) vptr[i + 1] = vptr[i] + (int32_t)per[i].size();
  std::vector<int32_t> vidx(vptr[n_cut]);
  for (int64_t i = 0; i < n_cut; ++i) std::copy(per[i].begin(), per[i].end(), vidx.begin() + vptr[i]);
  // Gauss rule and mode table
  std::vector<int> mk(kQMaxNm * 3, 0);
  for (int I = 0; I < nm; ++I)
    for (int a = 0; a < 3; ++a) mk[I * 3 + a] = L.modes[I].k[a];
  std::vector<double> gx(kQMaxP + 1, 0.0), gw(kQMaxP + 1, 0.0);
  {
    // Gauss-Legendre (p+1) points by Newton iteration on P_n (as gen.cpp)
    const int n = g->p + 1;
    for (int i = 0; i < (n + 1) / 2; ++i) {
      double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), z1, pp;
      do {
        double p1 = 1.0, p2 = 0.0;
        for (int j = 1; j <= n; ++j) { double p3 = p2; p2 = p1; p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j; }
        pp = n * (z * p1 - p2) / (z * z - 1.0);
        z1 = z;
        z = z1 - p1 / pp;
      } while (std::fabs(z - z1) > 1e-15);
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) { double p3 = p2; p2 = p1; p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j; }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      gx[i] = -z; gx[n - 1 - i] = z;
      gw[i] = gw[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
    }
  }
  int rc = FCM_OK;
  int64_t *d_cells = nullptr;
  int32_t *d_vptr = nullptr, *d_vidx = nullptr;
  double *d_vc = nullptr, *d_vr = nullptr, *d_K = nullptr, *d_f = nullptr;
  cudaStream_t st = nullptr;
  const int NB = (nm + 3) / 4, nblk = NB * (NB + 1) / 2;
  const int bpt = (nblk + kQThreads - 1) / kQThreads;
  int dev = 0, sms = 148;
  const int64_t chunk = std::min<int64_t>(n_cut, std::max<int64_t>(1, (int64_t)(1u << 30) / ((int64_t)nm * nm * 8)));
  QuadArgs qa{};
  const size_t dsm = (size_t)kQB * 4 * kQMaxNm * sizeof(double);
  QCU(cudaGetDevice(&dev));
  QCU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  QCU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  QCU(cudaFuncSetAttribute(k_cut_quadrature<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  QCU(cudaFuncSetAttribute(k_cut_quadrature<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  QCU(cudaFuncSetAttribute(k_cut_quadrature<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  QCU(cudaMemcpyToSymbolAsync(c_modek, mk.data(), mk.size() * sizeof(int), 0, cudaMemcpyHostToDevice, st));
  QCU(cudaMemcpyToSymbolAsync(c_gx, gx.data(), gx.size() * 8, 0, cudaMemcpyHostToDevice, st));
  QCU(cudaMemcpyToSymbolAsync(c_gw, gw.data(), gw.size() * 8, 0, cudaMemcpyHostToDevice, st));
  QCU(cudaMallocAsync((void**)&d_cells, n_cut * 8, st));
  QCU(cudaMallocAsync((void**)&d_vptr, (n_cut + 1) * 4, st));
  QCU(cudaMallocAsync((void**)&d_vidx, std::max<size_t>(1, vidx.size()) * 4, st));
  QCU(cudaMallocAsync((void**)&d_vc, std::max<int64_t>(1, n_voids * dim) * 8, st));
  QCU(cudaMallocAsync((void**)&d_vr, std::max<int64_t>(1, n_voids) * 8, st));
  QCU(cudaMallocAsync((void**)&d_K, chunk * nm * nm * 8, st));
  QCU(cudaMallocAsync((void**)&d_f, chunk * nm * 8, st));
  QCU(cudaMemcpyAsync(d_cells, cut_cells, n_cut * 8, cudaMemcpyHostToDevice, st));
  QCU(cudaMemcpyAsync(d_vptr, vptr.data(), (n_cut + 1) * 4, cudaMemcpyHostToDevice, st));
  if (!vidx.empty()) QCU(cudaMemcpyAsync(d_vidx, vidx.data(), vidx.size() * 4, cudaMemcpyHostToDevice, st));
  if (n_voids > 0) {
    QCU(cudaMemcpyAsync(d_vc, centres, n_voids * dim * 8, cudaMemcpyHostToDevice, st));
    QCU(cudaMemcpyAsync(d_vr, radii, n_voids * 8, cudaMemcpyHostToDevice, st));
  }
  qa.dim = dim; qa.p = g->p; qa.nm = nm; qa.depth = ph->depth; qa.h = h; qa.alpha = ph->alpha;
  qa.nx = (int)nx; qa.ny = (int)ny;
  qa.vidx = d_vidx; qa.vc = d_vc; qa.vr = d_vr; qa.K = d_K; qa.f = d_f;
  for (int64_t c0 = 0; c0 < n_cut; c0 += chunk) {
    const int64_t nc = std::min(chunk, n_cut - c0);
    qa.ncut = nc;
    qa.cells = d_cells + c0;
    qa.vptr = d_vptr + c0;
    const int grid = (int)std::min<int64_t>(nc, (int64_t)sms * 8);
    if (bpt <= 1) k_cut_quadrature<1><<<grid, kQThreads, dsm, st>>>(qa);
    else if (bpt == 2) k_cut_quadrature<2><<<grid, kQThreads, dsm, st>>>(qa);
    else k_cut_quadrature<3><<<grid, kQThreads, dsm, st>>>(qa);
    QCU(cudaGetLastError());
    QCU(cudaMemcpyAsync(cut_K + c0 * nm * nm, d_K, nc * nm * nm * 8, cudaMemcpyDeviceToHost, st));
    if (cut_f) QCU(cudaMemcpyAsync(cut_f + c0 * nm, d_f, nc * nm * 8, cudaMemcpyDeviceToHost, st));
    QCU(cudaStreamSynchronize(st));
  }
done:
  if (st) {
    for (void* p : {(void*)d_cells, (void*)d_vptr, (void*)d_vidx, (void*)d_vc, (void*)d_vr, (void*)d_K, (void*)d_f})
      if (p) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  return rc;
}
