// gen.cpp -- workload generator: exact cell classification and finite-cell element matrices.
// SETUP (not on the timed path).  Independent of the CPU oracle (no shared code).
//
// Weak form (Eq. weakform) with the indicator alpha:
//   Poisson     K_ab = int alpha grad N_a . grad N_b,   f_a = int alpha N_a (f = 1)
//   Elasticity  K_(a,i)(b,j) = int alpha [lam N_a,i N_b,j + mu N_a,j N_b,i + mu d_ij grad.grad]
// Cut cells: space tree of depth `depth` ("octree ... depth of 3", reading R13).
// Uncut leaves are integrated EXACTLY in Kronecker form from 1D sub-interval integrals
// (M = int N N, K = int N' N', D = int N' N on the leaf interval, (p+1)-point Gauss), which is
// the same integral as the leaf's tensor Gauss rule; depth-limit cut leaves use alpha per
// Gauss point (SPEC D-I1).
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/fcm_mg.h"
#include "common.hpp"
#include "layout.hpp"

namespace fcm {

// ---- Gauss-Legendre nodes by Newton iteration on P_n -----------------------------------
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), z1, pp;
    do {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      z1 = z;
      z = z1 - p1 / pp;
    } while (std::fabs(z - z1) > 1e-15);
    double p1 = 1.0, p2 = 0.0;
    for (int j = 1; j <= n; ++j) {
      double p3 = p2;
      p2 = p1;
      p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
    }
    pp = n * (z * p1 - p2) / (z * z - 1.0);
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// 1D modes 0..p and derivatives at xi (integrated Legendre, normalisation R-B1)
static void modes1d(int p, double xi, double* v, double* d) {
  double P[kMaxP + 2];
  P[0] = 1.0;
  P[1] = xi;
  for (int k = 1; k < p; ++k) P[k + 1] = ((2 * k + 1) * xi * P[k] - k * P[k - 1]) / (k + 1);
  v[0] = 0.5 * (1.0 - xi); d[0] = -0.5;
  v[1] = 0.5 * (1.0 + xi); d[1] = 0.5;
  for (int k = 2; k <= p; ++k) {
    v[k] = (P[k] - P[k - 2]) / std::sqrt(2.0 * (2 * k - 1));
    d[k] = std::sqrt(0.5 * (2 * k - 1)) * P[k - 1];
  }
}

// shared with the multi-level hp generator (gen_hp.cpp)
void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w) { gauss_legendre(n, x, w); }
void modes_1d(int p, double xi, double* v, double* d) { modes1d(p, xi, v, d); }

// 1D reference matrices on [-1, 1] of modes 0..p (row-major (p+1)^2): M_ij = int N_i N_j,
// K_ij = int N_i' N_j' (p+1-point Gauss: exact for degree 2p).  Used by the patch smoother's
// fast-diagonalisation setup (fcm_mg.cu), which checks K_ref against their Kronecker form.
void ref1d_matrices(int p, double* M, double* K) {
  std::vector<double> x, w;
  gauss_legendre(p + 1, x, w);
  const int P1 = p + 1;
  std::fill(M, M + P1 * P1, 0.0);
  std::fill(K, K + P1 * P1, 0.0);
  double v[kMaxP + 1], d[kMaxP + 1];
  for (int g = 0; g < P1; ++g) {
    modes1d(p, x[g], v, d);
    for (int i = 0; i < P1; ++i)
      for (int j = 0; j < P1; ++j) {
        M[i * P1 + j] += w[g] * v[i] * v[j];
        K[i * P1 + j] += w[g] * d[i] * d[j];
      }
  }
}

struct Voids {
  int dim;
  int64_t nv;
  const double* c;
  const double* r;
  // 0 phys, 1 fict (inside one open ball), 2 cut
  int classify(const double* lo, const double* hi) const {
    bool misses_all = true;
    for (int64_t j = 0; j < nv; ++j) {
      double far2 = 0, near2 = 0;
      for (int a = 0; a < dim; ++a) {
        double cc = c[j * dim + a];
        double d0 = lo[a] - cc, d1 = hi[a] - cc;
        far2 += std::max(d0 * d0, d1 * d1);
        double nr = std::max(0.0, std::max(lo[a] - cc, cc - hi[a]));
        near2 += nr * nr;
      }
      double r2 = r[j] * r[j];
      if (far2 < r2) return 1;
      if (near2 < r2) misses_all = false;
    }
    return misses_all ? 0 : 2;
  }
  bool fict(const double* x) const {
    for (int64_t j = 0; j < nv; ++j) {
      double d2 = 0;
      for (int a = 0; a < dim; ++a) { double t = x[a] - c[j * dim + a]; d2 += t * t; }
      if (d2 < r[j] * r[j]) return true;
    }
    return false;
  }
};

struct ElemGen {
  const Layout& L;
  int dim, p, n_f, m, nm;
  double h, alpha, lam = 0, mu = 0;
  bool elast;
  std::vector<double> gx, gw;  // (p+1)-point Gauss rule
  ElemGen(const Layout& L_, double h_, const fcm_physics& ph)
      : L(L_), dim(L_.dim), p(L_.p), n_f(L_.n_f), m(L_.m), nm((int)L_.modes.size()), h(h_),
        alpha(ph.alpha), elast(ph.kind == FCM_PHYS_ELASTICITY) {
    if (elast) {
      lam = ph.E * ph.nu / ((1 + ph.nu) * (1 - 2 * ph.nu));
      mu = ph.E / (2 * (1 + ph.nu));
    }
    gauss_legendre(p + 1, gx, gw);
  }

  // 1D integrals over [a,b] (reference coords): M, K (N'N'), D (N_i' N_j), F (int N_i)
  void sub1d(double a, double b, double* M, double* K, double* D, double* F) const {
    int P1 = p + 1;
    std::fill(M, M + P1 * P1, 0.0); std::fill(K, K + P1 * P1, 0.0);
    std::fill(D, D + P1 * P1, 0.0); std::fill(F, F + P1, 0.0);
    double v[kMaxP + 1], d[kMaxP + 1];
    for (int g = 0; g < P1; ++g) {
      double xi = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      double w = 0.5 * (b - a) * gw[g];
      modes1d(p, xi, v, d);
      for (int i = 0; i < P1; ++i) {
        F[i] += w * v[i];
        for (int j = 0; j < P1; ++j) {
          M[i * P1 + j] += w * v[i] * v[j];
          K[i * P1 + j] += w * d[i] * d[j];
          D[i * P1 + j] += w * d[i] * v[j];
        }
      }
    }
  }

  // add alpha * (exact integral over the reference box [lo,hi]) to Ke / fe
  void add_full_leaf(const double* lo, const double* hi, double al, double* Ke, double* fe) const {
    int P1 = p + 1;
    double M[3][(kMaxP + 1) * (kMaxP + 1)], K[3][(kMaxP + 1) * (kMaxP + 1)];
    double D[3][(kMaxP + 1) * (kMaxP + 1)], F[3][kMaxP + 1];
    for (int a = 0; a < dim; ++a) sub1d(lo[a], hi[a], M[a], K[a], D[a], F[a]);
    double jac = std::pow(0.5 * h, dim);      // dx = (h/2)^d dxi
    double g2 = (2.0 / h) * (2.0 / h);        // d/dx = (2/h) d/dxi
    for (int I = 0; I < nm; ++I) {
      const int* ki = L.modes[I].k;
      double fv = al * jac;
      for (int a = 0; a < dim; ++a) fv *= F[a][ki[a]];
      if (!elast) fe[I] += fv;
      for (int J = 0; J < nm; ++J) {
        const int* kj = L.modes[J].k;
        if (!elast) {
          double s = 0;
          for (int g = 0; g < dim; ++g) {
            double t = 1;
            for (int a = 0; a < dim; ++a) t *= (a == g ? K[a] : M[a])[ki[a] * P1 + kj[a]];
            s += t;
          }
          Ke[I * m + J] += al * jac * g2 * s;
        } else {
          // G_ce = int dN_I/dx_c dN_J/dx_e
          double G[3][3];
          for (int c = 0; c < dim; ++c)
            for (int e = 0; e < dim; ++e) {
              double t = 1;
              for (int a = 0; a < dim; ++a) {
                double f;
                if (a == c && a == e) f = K[a][ki[a] * P1 + kj[a]];
                else if (a == c) f = D[a][ki[a] * P1 + kj[a]];
                else if (a == e) f = D[a][kj[a] * P1 + ki[a]];
                else f = M[a][ki[a] * P1 + kj[a]];
                t *= f;
              }
              G[c][e] = t * g2 * jac * al;
            }
          double tr = 0;
          for (int c = 0; c < dim; ++c) tr += G[c][c];
          for (int c = 0; c < dim; ++c)
            for (int e = 0; e < dim; ++e) {
              double val = lam * G[c][e] + mu * G[e][c] + (c == e ? mu * tr : 0.0);
              Ke[(I * n_f + c) * m + (J * n_f + e)] += val;
            }
        }
      }
    }
  }

  // cut leaf at the depth limit: tensor Gauss rule, alpha per point
  void add_point_leaf(const double* lo, const double* hi, const double* cell_lo, const Voids& V,
                      double* Ke, double* fe, std::vector<double>& work) const {
    int P1 = p + 1;
    int npts = 1;
    for (int a = 0; a < dim; ++a) npts *= P1;
    double jac = std::pow(0.5 * h, dim);
    work.resize((size_t)nm * (dim + 1));
    double* val = work.data();
    double* grd = val + nm;
    double v[3][kMaxP + 1], d[3][kMaxP + 1];
    for (int q = 0; q < npts; ++q) {
      int t = q;
      double w = jac, x[3];
      for (int a = 0; a < dim; ++a) {
        int g = t % P1;
        t /= P1;
        double xi = 0.5 * (lo[a] + hi[a]) + 0.5 * (hi[a] - lo[a]) * gx[g];
        w *= 0.5 * (hi[a] - lo[a]) * gw[g];
        modes1d(p, xi, v[a], d[a]);
        x[a] = cell_lo[a] + 0.5 * h * (xi + 1.0);
      }
      double al = V.fict(x) ? alpha : 1.0;
      double wa = w * al;
      for (int I = 0; I < nm; ++I) {
        const int* k = L.modes[I].k;
        double vv = 1;
        for (int a = 0; a < dim; ++a) vv *= v[a][k[a]];
        val[I] = vv;
        for (int g = 0; g < dim; ++g) {
          double gg = 2.0 / h;
          for (int a = 0; a < dim; ++a) gg *= (a == g ? d[a][k[a]] : v[a][k[a]]);
          grd[I * dim + g] = gg;
        }
      }
      if (!elast) {
        for (int I = 0; I < nm; ++I) {
          fe[I] += wa * val[I];
          for (int J = 0; J < nm; ++J) {
            double s = 0;
            for (int g = 0; g < dim; ++g) s += grd[I * dim + g] * grd[J * dim + g];
            Ke[I * m + J] += wa * s;
          }
        }
      } else {
        for (int I = 0; I < nm; ++I)
          for (int J = 0; J < nm; ++J) {
            double dot = 0;
            for (int g = 0; g < dim; ++g) dot += grd[I * dim + g] * grd[J * dim + g];
            for (int c = 0; c < dim; ++c)
              for (int e = 0; e < dim; ++e) {
                double val2 = lam * grd[I * dim + c] * grd[J * dim + e] +
                              mu * grd[I * dim + e] * grd[J * dim + c] + (c == e ? mu * dot : 0.0);
                Ke[(I * n_f + c) * m + (J * n_f + e)] += wa * val2;
              }
          }
      }
    }
  }

  // recursive space tree over the physical sub-box [plo, phi] of the cell
  void tree(const double* plo, const double* phi, int level, int depth, const double* cell_lo,
            const Voids& V, double* Ke, double* fe, std::vector<double>& work) const {
    int kind = V.classify(plo, phi);
    double rlo[3], rhi[3];
    for (int a = 0; a < dim; ++a) {
      rlo[a] = 2.0 * (plo[a] - cell_lo[a]) / h - 1.0;
      rhi[a] = 2.0 * (phi[a] - cell_lo[a]) / h - 1.0;
    }
    if (kind != 2) { add_full_leaf(rlo, rhi, kind == 1 ? alpha : 1.0, Ke, fe); return; }
    if (level == depth) { add_point_leaf(rlo, rhi, cell_lo, V, Ke, fe, work); return; }
    double mid[3];
    for (int a = 0; a < dim; ++a) mid[a] = 0.5 * (plo[a] + phi[a]);
    for (int corner = 0; corner < (1 << dim); ++corner) {
      double clo[3], chi[3];
      for (int a = 0; a < dim; ++a) {
        bool up = corner >> a & 1;
        clo[a] = up ? mid[a] : plo[a];
        chi[a] = up ? phi[a] : mid[a];
      }
      tree(clo, chi, level + 1, depth, cell_lo, V, Ke, fe, work);
    }
  }
};

}  // namespace fcm

using namespace fcm;

static int check_grid(const fcm_grid* g) {
  if (!g) return fail(FCM_EINVAL, "grid is NULL");
  if (g->dim < 2 || g->dim > 3) return fail(FCM_EINVAL, "dim must be 2 or 3");
  if (g->p < 1 || g->p > kMaxP) return fail(FCM_EINVAL, "p must be in [1, 8]");
  if (g->space != 0 && g->space != 1) return fail(FCM_EINVAL, "space must be tensor(0) or trunk(1)");
  if (g->n_f != 1 && g->n_f != g->dim) return fail(FCM_EINVAL, "n_f must be 1 or dim");
  for (int a = 0; a < g->dim; ++a)
    if (g->n[a] < 1 || g->n[a] > 30000) return fail(FCM_EINVAL, "n[%d] out of range", a);
  if (!(g->h > 0)) return fail(FCM_EINVAL, "h must be > 0");
  return FCM_OK;
}

extern "C" int fcm_element_size(const fcm_grid* g) {
  int rc = check_grid(g);
  if (rc) return rc;
  Layout L;
  L.build(g->dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces);
  return L.m;
}

extern "C" int fcm_gen_classify(const fcm_grid* g, int64_t n_voids, const double* centres,
                                const double* radii, uint8_t* cell_kind, int64_t* n_cut) {
  clear_error();
  int rc = check_grid(g);
  if (rc) return rc;
  if (!cell_kind || (n_voids > 0 && (!centres || !radii))) return fail(FCM_EINVAL, "NULL buffer");
  Voids V{g->dim, n_voids, centres, radii};
  int64_t nx = g->n[0], ny = g->n[1], nz = g->dim == 3 ? g->n[2] : 1;
  int64_t ncell = nx * ny * nz, cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
  for (int64_t c = 0; c < ncell; ++c) {
    double lo[3] = {(double)(c % nx) * g->h, (double)((c / nx) % ny) * g->h, (double)(c / (nx * ny)) * g->h};
    double hi[3] = {lo[0] + g->h, lo[1] + g->h, lo[2] + g->h};
    int k = V.classify(lo, hi);
    cell_kind[c] = (uint8_t)k;
    cnt += k == 2;
  }
  if (n_cut) *n_cut = cnt;
  return FCM_OK;
}

extern "C" int fcm_gen_element_matrices(const fcm_grid* g, const fcm_physics* ph, int64_t n_voids,
                                        const double* centres, const double* radii, double* K_ref,
                                        double* f_ref, int64_t n_cut, const int64_t* cut_cells,
                                        double* cut_K, double* cut_f, double* f_traction,
                                        int32_t threads) {
  clear_error();
  int rc = check_grid(g);
  if (rc) return rc;
  if (!ph) return fail(FCM_EINVAL, "physics is NULL");
  if ((ph->kind == FCM_PHYS_ELASTICITY) != (g->n_f == g->dim && g->n_f > 1))
    return fail(FCM_EINVAL, "elasticity requires n_f == dim (and Poisson n_f == 1)");
  if (ph->depth < 0 || ph->depth > 8) return fail(FCM_EINVAL, "depth out of range");
  Layout L;
  L.build(g->dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces);
  ElemGen E(L, g->h, *ph);
  int m = L.m;
  Voids none{g->dim, 0, nullptr, nullptr};
  Voids V{g->dim, n_voids, centres, radii};
  std::vector<double> work;
  if (K_ref || f_ref) {
    std::vector<double> K((size_t)m * m, 0.0), f(m, 0.0);
    double lo[3] = {-1, -1, -1}, hi[3] = {1, 1, 1};
    E.add_full_leaf(lo, hi, 1.0, K.data(), f.data());
    if (K_ref) std::memcpy(K_ref, K.data(), sizeof(double) * m * m);
    if (f_ref) std::memcpy(f_ref, f.data(), sizeof(double) * m);
  }
  if (f_traction) {
    std::fill(f_traction, f_traction + m, 0.0);
    int face = ph->traction_face;
    if (face >= 0 && face < 2 * g->dim) {
      int axis = face / 2, side = face % 2;
      std::vector<double> M(81), K(81), D(81), F(9);
      E.sub1d(-1, 1, M.data(), K.data(), D.data(), F.data());
      for (int I = 0; I < (int)L.modes.size(); ++I) {
        const int* k = L.modes[I].k;
        if (k[axis] != side) continue;  // only the nodal mode at that end is nonzero on the face
        double v = std::pow(0.5 * g->h, g->dim - 1);
        for (int a = 0; a < g->dim; ++a) if (a != axis) v *= F[k[a]];
        f_traction[I * g->n_f + 0] = v;  // traction (1,0,0)
      }
    }
  }
  if (n_cut > 0) {
    if (!cut_cells || !cut_K) return fail(FCM_EINVAL, "cut buffers are NULL");
    int64_t nx = g->n[0], ny = g->n[1];
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel
    {
      std::vector<double> wk;
#pragma omp for schedule(dynamic, 4)
      for (int64_t i = 0; i < n_cut; ++i) {
        int64_t c = cut_cells[i];
        double lo[3] = {(double)(c % nx) * g->h, (double)((c / nx) % ny) * g->h,
                        (double)(c / (nx * ny)) * g->h};
        double hi[3] = {lo[0] + g->h, lo[1] + g->h, lo[2] + g->h};
        double* Ke = cut_K + (size_t)i * m * m;
        std::fill(Ke, Ke + (size_t)m * m, 0.0);
        std::vector<double> fe(m, 0.0);
        E.tree(lo, hi, 0, ph->depth, lo, V, Ke, fe.data(), wk);
        // exact symmetry (the integrals are symmetric; remove rounding asymmetry)
        for (int a = 0; a < m; ++a)
          for (int b = a + 1; b < m; ++b) {
            double s = 0.5 * (Ke[a * m + b] + Ke[b * m + a]);
            Ke[a * m + b] = Ke[b * m + a] = s;
          }
        if (cut_f) std::memcpy(cut_f + (size_t)i * m, fe.data(), sizeof(double) * m);
      }
    }
  }
  (void)none;
  return FCM_OK;
}
