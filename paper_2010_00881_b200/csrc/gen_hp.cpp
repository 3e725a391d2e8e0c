// gen_hp.cpp -- multi-level hp discretisation generator.  SETUP, host C++/OpenMP.
// Independent of the CPU oracle (no shared code).
//
// PAPER.md:99-102 (Sec. 2.2): refinement by superposition -- a refined element of depth j carries
// 2^d subelements of depth j+1 formed by uniform bisection, recursively up to kmax; elements cut
// by the immersed boundary are the refined ones.  Every element of every depth carries
// the tensor integrated-Legendre modes of order p on its topological entities; the activation
// rule (reading R25; the paper defers the rule set to [Zander2016]):
//   a depth-j entity is ACTIVE iff (j == 0 or every depth-j element adjacent to it inside the
//   domain exists)  [compatibility: overlay functions vanish on the overlay boundary]
//   and at least one existing adjacent depth-j element is a LEAF  [independence].
// DOF numbering: by the coarsest hp level containing the DOF (levels (p,k) ...
// (1,k), (1,k-1) ... (1,0)), descending, so every level is a prefix; components interleaved.
// Leaf systems: the superposed basis of the leaf and its ancestors (each a polynomial of degree
// <= p on the leaf), integrated by a space tree of depth `depth` below the leaf ((p+1)^d Gauss
// points per sub-box; alpha per point at depth-limit cut sub-boxes, R13).  Weak form as gen.cpp.
#include <algorithm>
#include <array>
#include <memory>
#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <unordered_map>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/fcm_mg.h"
#include "common.hpp"

namespace fcm {
void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w);   // gen.cpp
void modes_1d(int p, double xi, double* v, double* d);                    // gen.cpp
}

using namespace fcm;

struct fcm_hp_disc {
  int dim = 2, n = 0, p = 1, kmax = 0, n_f = 1, kdof = 0;
  int64_t ndof = 0;
  std::vector<int64_t> level_n;
  std::vector<int32_t> level_q, level_k;
  std::vector<int32_t> keys;        // ndof * 8
  std::vector<double> b;
  std::vector<int64_t> leaf_ptr, leaf_kptr;
  std::vector<int32_t> leaf_dofs, leaf_info;
  std::vector<double> leaf_K;
};

namespace {

constexpr int kMaxPhp = 8;

struct Geo {
  int dim;
  int64_t nv;
  const double* c;
  const double* r;
  // 0 phys, 1 fict (inside one open ball), 2 cut (reading R14)
  int classify(const double* lo, const double* hi) const {
    bool misses = true;
    for (int64_t j = 0; j < nv; ++j) {
      double far2 = 0, near2 = 0;
      for (int a = 0; a < dim; ++a) {
        const double cc = c[j * dim + a];
        const double d0 = lo[a] - cc, d1 = hi[a] - cc;
        far2 += std::max(d0 * d0, d1 * d1);
        const double nr = std::max(0.0, std::max(lo[a] - cc, cc - hi[a]));
        near2 += nr * nr;
      }
      const double r2 = r[j] * r[j];
      if (far2 < r2) return 1;
      if (near2 < r2) misses = false;
    }
    return misses ? 0 : 2;
  }
  bool fict(const double* x) const {
    for (int64_t j = 0; j < nv; ++j) {
      double d2 = 0;
      for (int a = 0; a < dim; ++a) {
        const double t = x[a] - c[j * dim + a];
        d2 += t * t;
      }
      if (d2 < r[j] * r[j]) return true;
    }
    return false;
  }
};

// element of depth j, integer coordinates idx on the depth-j grid (N_j = n 2^j per axis)
struct Elem {
  int j;
  int idx[3];
};

struct Tree {
  int dim, n, kmax;
  std::vector<std::unordered_map<int64_t, uint8_t>> lev;   // depth -> (linear index -> refined)
  int64_t N(int j) const { return (int64_t)n << j; }
  int64_t lin(int j, const int* idx) const {
    const int64_t Nj = N(j);
    int64_t l = 0;
    for (int a = dim - 1; a >= 0; --a) l = l * Nj + idx[a];
    return l;
  }
  // -1: absent, 0: leaf, 1: refined
  int state(int j, const int* idx) const {
    auto it = lev[j].find(lin(j, idx));
    return it == lev[j].end() ? -1 : it->second;
  }
  // R25
  bool active(int j, const int* X) const {
    const int64_t Nj = N(j);
    int lo[3] = {0, 0, 0}, cnt[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) {
      if (X[a] & 1) {
        lo[a] = (X[a] - 1) / 2;
        cnt[a] = 1;
      } else {
        const int v = X[a] / 2;
        lo[a] = v - 1;
        cnt[a] = 2;
        if (v == 0) { lo[a] = 0; cnt[a] = 1; }
        else if (v == Nj) { lo[a] = v - 1; cnt[a] = 1; }
      }
    }
    bool any_leaf = false;
    for (int k = 0; k < cnt[2]; ++k)
      for (int jj = 0; jj < cnt[1]; ++jj)
        for (int i = 0; i < cnt[0]; ++i) {
          int e[3] = {lo[0] + i, lo[1] + jj, lo[2] + k};
          const int s = state(j, e);
          if (s < 0) {
            if (j > 0) return false;
            continue;
          }
          if (s == 0) any_leaf = true;
        }
    return any_leaf;
  }
};

struct KeyRec {
  int64_t pk;      // packed (j, X, degs) for ordering within a level class
  int cl;          // coarsest level index containing it
};

inline int64_t pack_key(int j, const int* X, const int* dg) {
  int64_t k = j;
  for (int a = 2; a >= 0; --a) k = k * 65536 + X[a];
  for (int a = 2; a >= 0; --a) k = k * 16 + dg[a];
  return k;
}

}  // namespace

extern "C" int fcm_hp_generate(const fcm_hp_spec* s, fcm_hp_disc** out) {
  clear_error();
  if (!s || !out) return fail(FCM_EINVAL, "fcm_hp_generate: NULL argument");
  if (s->dim < 2 || s->dim > 3 || s->n < 1 || s->p < 1 || s->p > kMaxPhp || s->kmax < 0 || s->kmax > 7 ||
      (s->n_voids > 0 && (!s->centres || !s->radii)) || s->phys.depth < 0 || s->phys.depth > 8)
    return fail(FCM_EINVAL, "fcm_hp_generate: invalid spec (dim %d n %d p %d kmax %d)", s->dim, s->n, s->p, s->kmax);
  if (((int64_t)s->n << s->kmax) * 2 >= 65536) return fail(FCM_EINVAL, "fcm_hp_generate: n 2^kmax too large");
  const int dim = s->dim, n = s->n, p = s->p, kmax = s->kmax;
  const bool elast = s->phys.kind == FCM_PHYS_ELASTICITY;
  const int n_f = elast ? dim : 1;
  Geo geo{dim, s->n_voids, s->centres, s->radii};
  std::unique_ptr<fcm_hp_disc> D(new (std::nothrow) fcm_hp_disc());
  if (!D) return fail(FCM_ENOMEM, "fcm_hp_generate: host allocation");
  D->dim = dim; D->n = n; D->p = p; D->kmax = kmax; D->n_f = n_f;

  // ---- refinement trees ----
  Tree T{dim, n, kmax, std::vector<std::unordered_map<int64_t, uint8_t>>(kmax + 1)};
  std::vector<std::vector<Elem>> elems(kmax + 1);
  {
    const int nb = dim == 3 ? n : 1;
    for (int z = 0; z < nb; ++z)
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) elems[0].push_back(Elem{0, {x, y, dim == 3 ? z : 0}});
    for (int j = 0; j <= kmax; ++j) {
      const double h = 1.0 / (double)T.N(j);
      for (const Elem& e : elems[j]) {
        bool ref = false;
        if (j < kmax) {
          if (s->refine == FCM_HP_REFINE_ALL) ref = true;
          else {
            double lo[3], hi[3];
            for (int a = 0; a < dim; ++a) { lo[a] = e.idx[a] * h; hi[a] = lo[a] + h; }
            ref = geo.classify(lo, hi) == 2;
          }
        }
        T.lev[j][T.lin(j, e.idx)] = ref ? 1 : 0;
        if (ref)
          for (int c = 0; c < (1 << dim); ++c) {
            Elem ch{j + 1, {0, 0, 0}};
            for (int a = 0; a < dim; ++a) ch.idx[a] = 2 * e.idx[a] + ((c >> a) & 1);
            elems[j + 1].push_back(ch);
          }
      }
    }
  }

  // ---- element modes (tensor), active free entities -> scalar DOF keys ----
  std::vector<std::array<int, 3>> modes;
  {
    const int nz = dim == 3 ? p + 1 : 1;
    for (int kz = 0; kz < nz; ++kz)
      for (int ky = 0; ky <= p; ++ky)
        for (int kx = 0; kx <= p; ++kx) modes.push_back({kx, ky, kz});
  }
  const int nm = (int)modes.size();
  auto mode_X = [&](const Elem& e, int mi, int* X, int* dg) {
    for (int a = 0; a < 3; ++a) {
      if (a >= dim) { X[a] = 0; dg[a] = 0; continue; }
      const int k = modes[mi][a];
      X[a] = 2 * e.idx[a] + (k == 0 ? 0 : k == 1 ? 2 : 1);
      dg[a] = k >= 2 ? k : 0;
    }
  };
  auto free_entity = [&](int j, const int* X) {
    const int64_t Nj = T.N(j);
    for (int a = 0; a < dim; ++a) {
      if (X[a] & 1) continue;
      if (((s->dirichlet_faces >> (2 * a)) & 1) && X[a] == 0) return false;
      if (((s->dirichlet_faces >> (2 * a + 1)) & 1) && X[a] == 2 * Nj) return false;
    }
    return true;
  };
  std::map<int64_t, KeyRec> keymap;   // packed key -> record
  int kdof = 0;
  for (int j = 0; j <= kmax; ++j)
    for (const Elem& e : elems[j])
      for (int mi = 0; mi < nm; ++mi) {
        int X[3], dg[3];
        mode_X(e, mi, X, dg);
        if (!T.active(j, X) || !free_entity(j, X)) continue;
        keymap.emplace(pack_key(j, X, dg), KeyRec{0, 0});
        kdof = std::max(kdof, j);
      }
  D->kdof = kdof;
  // hp levels, finest first: (p,k) ... (1,k), (1,k-1) ... (1,0)
  const int nlev = p + kdof;
  for (int l = 0; l < nlev; ++l) {
    D->level_q.push_back(l < p ? p - l : 1);
    D->level_k.push_back(l < p ? kdof : kdof - (l - (p - 1)));
  }
  // coarsest level containing a DOF of order o, depth j
  std::vector<std::pair<int64_t, int64_t>> order;   // (-cl, packed key)
  for (auto& kv : keymap) {
    const int64_t pk = kv.first;
    int dg[3], o = 1;
    int64_t t = pk;
    for (int a = 0; a < 3; ++a) { dg[a] = (int)(t % 16); t /= 16; }
    for (int a = 0; a < 3; ++a) t /= 65536;
    const int j = (int)t;
    for (int a = 0; a < 3; ++a) o = std::max(o, dg[a] >= 2 ? dg[a] : 1);
    const int cl = o >= 2 ? p - o : (p - 1) + (kdof - j);
    kv.second.cl = cl;
    order.push_back({-(int64_t)cl, pk});
  }
  std::sort(order.begin(), order.end());
  std::unordered_map<int64_t, int64_t> sidx;   // packed key -> scalar index
  sidx.reserve(order.size() * 2);
  for (size_t i = 0; i < order.size(); ++i) sidx[order[i].second] = (int64_t)i;
  const int64_t nscal = (int64_t)order.size();
  D->ndof = nscal * n_f;
  D->level_n.assign(nlev, 0);
  for (auto& o : order)
    for (int l = 0; l <= (int)(-o.first); ++l) D->level_n[l] += n_f;
  // trailing levels without DOFs are dropped (every base element refined: (1,0) is empty)
  while (D->level_n.size() > 1 && D->level_n.back() == 0) {
    D->level_n.pop_back();
    D->level_q.pop_back();
    D->level_k.pop_back();
  }
  D->keys.assign((size_t)D->ndof * 8, 0);
  for (int64_t i = 0; i < nscal; ++i) {
    int64_t t = order[i].second;
    int dg[3], X[3];
    for (int a = 0; a < 3; ++a) { dg[a] = (int)(t % 16); t /= 16; }
    for (int a = 0; a < 3; ++a) { X[a] = (int)(t % 65536); t /= 65536; }
    for (int c = 0; c < n_f; ++c) {
      int32_t* k = &D->keys[(size_t)(i * n_f + c) * 8];
      k[0] = (int32_t)t;
      for (int a = 0; a < 3; ++a) { k[1 + a] = X[a]; k[4 + a] = dg[a]; }
      k[7] = c;
    }
  }

  // ---- leaves: superposed functions, quadrature ----
  std::vector<Elem> leaves;
  for (int j = 0; j <= kmax; ++j)
    for (const Elem& e : elems[j])
      if (T.state(j, e.idx) == 0) leaves.push_back(e);
  const int64_t nleaf = (int64_t)leaves.size();
  // per leaf: scalar functions (ancestor depth, mode, scalar index)
  struct Fn { int j, mi; int64_t si; };
  std::vector<std::vector<Fn>> lf(nleaf);
  D->leaf_ptr.assign(nleaf + 1, 0);
  D->leaf_kptr.assign(nleaf + 1, 0);
  D->leaf_info.assign((size_t)nleaf * 5, 0);
  for (int64_t L = 0; L < nleaf; ++L) {
    const Elem& e = leaves[L];
    for (int j = 0; j <= e.j; ++j) {
      Elem an{j, {0, 0, 0}};
      for (int a = 0; a < dim; ++a) an.idx[a] = e.idx[a] >> (e.j - j);
      for (int mi = 0; mi < nm; ++mi) {
        int X[3], dg[3];
        mode_X(an, mi, X, dg);
        auto it = sidx.find(pack_key(j, X, dg));
        if (it != sidx.end()) lf[L].push_back(Fn{j, mi, it->second});
      }
    }
    std::sort(lf[L].begin(), lf[L].end(), [](const Fn& a, const Fn& b) { return a.si < b.si; });
    const int64_t m = (int64_t)lf[L].size() * n_f;
    D->leaf_ptr[L + 1] = D->leaf_ptr[L] + m;
    D->leaf_kptr[L + 1] = D->leaf_kptr[L] + m * m;
    int32_t* inf = &D->leaf_info[(size_t)L * 5];
    inf[0] = e.j;
    for (int a = 0; a < 3; ++a) inf[1 + a] = e.idx[a];
    int base = 0;
    for (int a = dim - 1; a >= 0; --a) base = base * n + (e.idx[a] >> e.j);
    inf[4] = base;
  }
  try {
    D->leaf_dofs.assign(D->leaf_ptr[nleaf], 0);
    D->leaf_K.assign(D->leaf_kptr[nleaf], 0.0);
    D->b.assign(D->ndof, 0.0);
  } catch (...) {
    return fail(FCM_ENOMEM, "fcm_hp_generate: host allocation of the leaf systems");
  }
  std::vector<double> gx, gw;
  gauss_rule(p + 1, gx, gw);
  double lam = 0, mu = 0;
  if (elast) {
    lam = s->phys.E * s->phys.nu / ((1 + s->phys.nu) * (1 - 2 * s->phys.nu));
    mu = s->phys.E / (2 * (1 + s->phys.nu));
  }
  const int depth = s->phys.depth;
  const double alpha = s->phys.alpha;
  const int tface = s->phys.traction_face;
  std::vector<double> floads((size_t)D->leaf_ptr[nleaf], 0.0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t L = 0; L < nleaf; ++L) {
    const Elem& e = leaves[L];
    const std::vector<Fn>& F = lf[L];
    const int nfn = (int)F.size();
    const int m = nfn * n_f;
    double* K = &D->leaf_K[D->leaf_kptr[L]];
    double* f = &floads[D->leaf_ptr[L]];
    int32_t* dofs = &D->leaf_dofs[D->leaf_ptr[L]];
    for (int i = 0; i < nfn; ++i)
      for (int c = 0; c < n_f; ++c) dofs[i * n_f + c] = (int32_t)(F[i].si * n_f + c);
    const double hL = 1.0 / (double)T.N(e.j);
    double lo[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) lo[a] = e.idx[a] * hL;
    std::vector<double> val(nfn), grd((size_t)nfn * 3);
    // evaluate every function of the leaf at physical point x
    auto eval = [&](const double* x) {
      double v1[3][kMaxPhp + 1], d1[3][kMaxPhp + 1];
      int cur = -1;
      for (int i = 0; i < nfn; ++i) {
        const int j = F[i].j;
        const double h = 1.0 / (double)T.N(j);
        if (j != cur) {
          for (int a = 0; a < dim; ++a) {
            const double alo = (double)(e.idx[a] >> (e.j - j)) * h;
            modes_1d(p, 2.0 * (x[a] - alo) / h - 1.0, v1[a], d1[a]);
          }
          cur = j;
        }
        const auto& md = modes[F[i].mi];
        double v = 1.0;
        for (int a = 0; a < dim; ++a) v *= v1[a][md[a]];
        val[i] = v;
        for (int g = 0; g < dim; ++g) {
          double t = 2.0 / h;
          for (int a = 0; a < dim; ++a) t *= (a == g ? d1[a][md[a]] : v1[a][md[a]]);
          grd[(size_t)i * 3 + g] = t;
        }
      }
    };
    auto add_point = [&](const double* x, double wa) {
      eval(x);
      for (int i = 0; i < nfn; ++i) {
        const double* gi = &grd[(size_t)i * 3];
        if (!elast) f[i] += wa * val[i];
        for (int k = 0; k < nfn; ++k) {
          const double* gk = &grd[(size_t)k * 3];
          double dot = 0;
          for (int a = 0; a < dim; ++a) dot += gi[a] * gk[a];
          if (!elast) {
            K[(size_t)i * m + k] += wa * dot;
          } else {
            for (int c1 = 0; c1 < dim; ++c1)
              for (int c2 = 0; c2 < dim; ++c2) {
                double v = lam * gi[c1] * gk[c2] + mu * gi[c2] * gk[c1];
                if (c1 == c2) v += mu * dot;
                K[(size_t)(i * n_f + c1) * m + k * n_f + c2] += wa * v;
              }
          }
        }
      }
    };
    // space tree below the leaf (R13)
    struct Box { double lo[3], hi[3]; int lvl; };
    std::vector<Box> st;
    Box root;
    for (int a = 0; a < 3; ++a) { root.lo[a] = lo[a]; root.hi[a] = lo[a] + (a < dim ? hL : 0.0); }
    root.lvl = 0;
    st.push_back(root);
    while (!st.empty()) {
      Box bx = st.back();
      st.pop_back();
      const int kind = geo.classify(bx.lo, bx.hi);
      if (kind == 2 && bx.lvl < depth) {
        for (int c = 0; c < (1 << dim); ++c) {
          Box ch;
          ch.lvl = bx.lvl + 1;
          for (int a = 0; a < 3; ++a) {
            const double mid = 0.5 * (bx.lo[a] + bx.hi[a]);
            const bool up = a < dim && ((c >> a) & 1);
            ch.lo[a] = up ? mid : bx.lo[a];
            ch.hi[a] = a < dim ? (up ? bx.hi[a] : mid) : bx.hi[a];
          }
          st.push_back(ch);
        }
        continue;
      }
      const int P1 = p + 1;
      const int npt = dim == 3 ? P1 * P1 * P1 : P1 * P1;
      for (int g = 0; g < npt; ++g) {
        int gi[3] = {g % P1, (g / P1) % P1, dim == 3 ? g / (P1 * P1) : 0};
        double x[3] = {0, 0, 0}, w = 1.0;
        for (int a = 0; a < dim; ++a) {
          const double hh = bx.hi[a] - bx.lo[a];
          x[a] = bx.lo[a] + 0.5 * hh * (gx[gi[a]] + 1.0);
          w *= 0.5 * hh * gw[gi[a]];
        }
        double al = kind == 0 ? 1.0 : kind == 1 ? alpha : (geo.fict(x) ? alpha : 1.0);
        add_point(x, w * al);
      }
    }
    // traction (1,0,0) on face tface (R8, not alpha-weighted), leaves touching it
    if (tface >= 0 && elast) {
      const int ax = tface / 2, side = tface % 2;
      const bool on = side ? (e.idx[ax] == T.N(e.j) - 1) : (e.idx[ax] == 0);
      if (on) {
        const int P1 = p + 1;
        const int npt = dim == 3 ? P1 * P1 : P1;
        for (int g = 0; g < npt; ++g) {
          double x[3] = {lo[0], lo[1], lo[2]}, w = 1.0;
          x[ax] = lo[ax] + (side ? hL : 0.0);
          int t = g;
          for (int a = 0; a < dim; ++a) {
            if (a == ax) continue;
            const int k = t % P1;
            t /= P1;
            x[a] = lo[a] + 0.5 * hL * (gx[k] + 1.0);
            w *= 0.5 * hL * gw[k];
          }
          eval(x);
          for (int i = 0; i < nfn; ++i) f[i * n_f + 0] += w * val[i];
        }
      }
    }
    // Poisson f[] was accumulated per scalar function index i (n_f = 1): same layout
  }
  for (int64_t L = 0; L < nleaf; ++L)
    for (int64_t a = D->leaf_ptr[L]; a < D->leaf_ptr[L + 1]; ++a) D->b[D->leaf_dofs[a]] += floads[a];
  *out = D.release();
  return FCM_OK;
}

extern "C" int fcm_hp_disc_destroy(fcm_hp_disc* d) {
  delete d;
  return FCM_OK;
}

extern "C" int fcm_hp_disc_info(const fcm_hp_disc* d, int64_t* ndof, int32_t* nlevels, int64_t* nleaves,
                                int64_t* leaf_entries, int64_t* leaf_matrix_entries) {
  clear_error();
  if (!d) return fail(FCM_EINVAL, "fcm_hp_disc_info: NULL handle");
  const int64_t nl = (int64_t)d->leaf_ptr.size() - 1;
  if (ndof) *ndof = d->ndof;
  if (nlevels) *nlevels = (int32_t)d->level_n.size();
  if (nleaves) *nleaves = nl;
  if (leaf_entries) *leaf_entries = d->leaf_ptr[nl];
  if (leaf_matrix_entries) *leaf_matrix_entries = d->leaf_kptr[nl];
  return FCM_OK;
}

extern "C" int fcm_hp_disc_levels(const fcm_hp_disc* d, int64_t* ndofs, int32_t* q, int32_t* kc) {
  clear_error();
  if (!d) return fail(FCM_EINVAL, "fcm_hp_disc_levels: NULL handle");
  for (size_t l = 0; l < d->level_n.size(); ++l) {
    if (ndofs) ndofs[l] = d->level_n[l];
    if (q) q[l] = d->level_q[l];
    if (kc) kc[l] = d->level_k[l];
  }
  return FCM_OK;
}

extern "C" int fcm_hp_disc_keys(const fcm_hp_disc* d, int32_t* keys) {
  clear_error();
  if (!d || !keys) return fail(FCM_EINVAL, "fcm_hp_disc_keys: NULL argument");
  std::memcpy(keys, d->keys.data(), d->keys.size() * 4);
  return FCM_OK;
}

extern "C" int fcm_hp_disc_load(const fcm_hp_disc* d, double* b) {
  clear_error();
  if (!d || !b) return fail(FCM_EINVAL, "fcm_hp_disc_load: NULL argument");
  std::memcpy(b, d->b.data(), d->b.size() * 8);
  return FCM_OK;
}

extern "C" int fcm_hp_disc_leaves(const fcm_hp_disc* d, int64_t* leaf_ptr, int32_t* dofs, double* K, int32_t* info) {
  clear_error();
  if (!d) return fail(FCM_EINVAL, "fcm_hp_disc_leaves: NULL handle");
  if (leaf_ptr) std::memcpy(leaf_ptr, d->leaf_ptr.data(), d->leaf_ptr.size() * 8);
  if (dofs) std::memcpy(dofs, d->leaf_dofs.data(), d->leaf_dofs.size() * 4);
  if (K) std::memcpy(K, d->leaf_K.data(), d->leaf_K.size() * 8);
  if (info) std::memcpy(info, d->leaf_info.data(), d->leaf_info.size() * 4);
  return FCM_OK;
}

// accessors for hpmg.cu (same library)
namespace fcm {
const fcm_hp_disc* hp_disc_check(const fcm_hp_disc* d) { return d; }
void hp_disc_view(const fcm_hp_disc* d, int* dim, int* n, int* p, int* n_f, int64_t* ndof, std::vector<int64_t>* level_n,
                  const std::vector<int64_t>** leaf_ptr, const std::vector<int64_t>** leaf_kptr,
                  const std::vector<int32_t>** leaf_dofs, const std::vector<double>** leaf_K,
                  const std::vector<int32_t>** leaf_info) {
  *dim = d->dim; *n = d->n; *p = d->p; *n_f = d->n_f; *ndof = d->ndof;
  *level_n = d->level_n;
  *leaf_ptr = &d->leaf_ptr; *leaf_kptr = &d->leaf_kptr; *leaf_dofs = &d->leaf_dofs; *leaf_K = &d->leaf_K;
  *leaf_info = &d->leaf_info;
}
}  // namespace fcm
