// layout.hpp -- element modes, DOF classes and the class-major device layout.
// Implements the CONVENTIONS of include/fcm_mg.h (hierarchical local order, DOF keys,
// class-major prefix layout).  PAPER.md:34/62 (hierarchical integrated-Legendre basis),
// PAPER.md:188-216 (nested levels, hierarchical matrices), PAPER.md:199-206 (binary R).
#pragma once
#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace fcm {

constexpr int kMaxP = 8;

struct Mode {
  int k[3];   // 1D mode index per axis (0 for absent axes)
  int order;  // level tag
};

struct DofClass {
  int S;          // bitmask of internal axes
  int deg[3];     // internal degrees (0 for nodal / absent axes)
  int comp;       // field component
  int order;
  int lo[3], hi[3], size[3];   // free entity positions per axis, inclusive range
  int64_t off = 0, count = 0;  // offset in the layout, number of DOFs
};

// Per level q, per local element DOF a (< m_q): where the DOF of cell (cx,cy,cz) lives.
//   valid iff cmin[a][i] <= c_i <= cmax[a][i] for i < 3, idx = base[a] + sum_i c_i*stride[a][i]
struct LevelTable {
  int m = 0;
  int64_t ndof = 0;
  std::vector<int64_t> base;
  std::vector<int32_t> stride;  // m*3
  std::vector<int16_t> cmin, cmax;  // m*3
};

inline int order1d(int k) { return k < 2 ? 1 : k; }

struct Layout {
  int dim = 3, n[3] = {1, 1, 1}, p = 1, space = 0, n_f = 1;
  uint32_t dmask = 0;
  std::vector<Mode> modes;           // sorted hierarchical order
  int m = 0;                         // modes.size() * n_f
  std::vector<DofClass> classes;
  std::vector<int> dof_class;        // local DOF -> class
  std::vector<std::array<int, 3>> dof_off;  // local DOF -> entity offset per axis (0/1 nodal, 0 internal)
  std::vector<int> m_level;          // index q (1..p)
  std::vector<int64_t> ndof_level;   // index q
  std::vector<LevelTable> tables;    // index q
  int64_t ncell = 0;
  int zoff = 0;                      // slab offset of the last axis (global DOF keys)

  static int mode_order(const int k[3], int dim, int space) {
    int mx = 1, sum = 0;
    bool internal = false;
    for (int a = 0; a < dim; ++a) {
      mx = std::max(mx, order1d(k[a]));
      if (k[a] >= 2) { internal = true; sum += k[a]; }
    }
    if (space == 0) return mx;
    return internal ? sum : 1;
  }

  void build(int dim_, const int n_[3], int p_, int space_, int n_f_, uint32_t dmask_) {
    dim = dim_; p = p_; space = space_; n_f = n_f_; dmask = dmask_;
    for (int a = 0; a < 3; ++a) n[a] = (a < dim) ? n_[a] : 1;
    ncell = (int64_t)n[0] * n[1] * n[2];
    // ---- element modes, sorted by (order, S, deg_x, deg_y, deg_z, off) ----
    modes.clear();
    int kmax[3] = {p, dim > 1 ? p : 0, dim > 2 ? p : 0};
    for (int kz = 0; kz <= kmax[2]; ++kz)
      for (int ky = 0; ky <= kmax[1]; ++ky)
        for (int kx = 0; kx <= kmax[0]; ++kx) {
          Mode md;
          md.k[0] = kx; md.k[1] = ky; md.k[2] = kz;
          if (space == 1) {
            int sum = 0;
            for (int a = 0; a < dim; ++a) if (md.k[a] >= 2) sum += md.k[a];
            if (sum > p) continue;
          }
          md.order = mode_order(md.k, dim, space);
          modes.push_back(md);
        }
    auto key = [&](const Mode& md) {
      int S = 0, off = 0, deg[3] = {0, 0, 0};
      for (int a = 0; a < dim; ++a) {
        if (md.k[a] >= 2) { S |= 1 << a; deg[a] = md.k[a]; }
        else off |= md.k[a] << a;
      }
      return std::make_tuple(md.order, S, deg[0], deg[1], deg[2], off);
    };
    std::stable_sort(modes.begin(), modes.end(),
                     [&](const Mode& x, const Mode& y) { return key(x) < key(y); });
    m = (int)modes.size() * n_f;
    // ---- classes ----
    std::map<std::tuple<int, int, int, int, int, int>, int> cls_index;  // (order,S,dx,dy,dz,comp)
    std::vector<std::tuple<int, int, int, int, int, int>> cls_keys;
    for (auto& md : modes)
      for (int c = 0; c < n_f; ++c) {
        int S = 0, deg[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) if (md.k[a] >= 2) { S |= 1 << a; deg[a] = md.k[a]; }
        auto kk = std::make_tuple(md.order, S, deg[0], deg[1], deg[2], c);
        if (!cls_index.count(kk)) { cls_index[kk] = 0; cls_keys.push_back(kk); }
      }
    std::sort(cls_keys.begin(), cls_keys.end());
    classes.clear();
    for (size_t i = 0; i < cls_keys.size(); ++i) {
      auto& kk = cls_keys[i];
      cls_index[kk] = (int)i;
      DofClass dc;
      dc.order = std::get<0>(kk); dc.S = std::get<1>(kk);
      dc.deg[0] = std::get<2>(kk); dc.deg[1] = std::get<3>(kk); dc.deg[2] = std::get<4>(kk);
      dc.comp = std::get<5>(kk);
      dc.count = 1;
      for (int a = 0; a < 3; ++a) {
        if (a >= dim) { dc.lo[a] = 0; dc.hi[a] = 0; }
        else if (dc.S >> a & 1) { dc.lo[a] = 0; dc.hi[a] = n[a] - 1; }
        else {
          dc.lo[a] = (dmask >> (2 * a) & 1) ? 1 : 0;
          dc.hi[a] = (dmask >> (2 * a + 1) & 1) ? n[a] - 1 : n[a];
        }
        dc.size[a] = std::max(0, dc.hi[a] - dc.lo[a] + 1);
        dc.count *= dc.size[a];
      }
      classes.push_back(dc);
    }
    int64_t off = 0;
    for (auto& dc : classes) { dc.off = off; off += dc.count; }
    // ---- local DOF -> class ----
    dof_class.assign(m, 0);
    dof_off.assign(m, {0, 0, 0});
    for (size_t r = 0; r < modes.size(); ++r)
      for (int c = 0; c < n_f; ++c) {
        auto& md = modes[r];
        int S = 0, deg[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) if (md.k[a] >= 2) { S |= 1 << a; deg[a] = md.k[a]; }
        int a_loc = (int)r * n_f + c;
        dof_class[a_loc] = cls_index[std::make_tuple(md.order, S, deg[0], deg[1], deg[2], c)];
        for (int a = 0; a < dim; ++a) dof_off[a_loc][a] = md.k[a] < 2 ? md.k[a] : 0;
      }
    // ---- levels ----
    m_level.assign(p + 1, 0);
    ndof_level.assign(p + 1, 0);
    tables.assign(p + 1, LevelTable());
    for (int q = 1; q <= p; ++q) {
      int mq = 0;
      for (auto& md : modes) if (md.order <= q) mq += n_f;
      m_level[q] = mq;
      int64_t nd = 0;
      for (auto& dc : classes) if (dc.order <= q) nd += dc.count;
      ndof_level[q] = nd;
      LevelTable& t = tables[q];
      t.m = mq; t.ndof = nd;
      t.base.resize(mq); t.stride.resize(mq * 3); t.cmin.resize(mq * 3); t.cmax.resize(mq * 3);
      for (int a = 0; a < mq; ++a) {
        const DofClass& dc = classes[dof_class[a]];
        int64_t st[3] = {1, dc.size[0], (int64_t)dc.size[0] * dc.size[1]};
        int64_t b = dc.off;
        for (int i = 0; i < 3; ++i) {
          int o = dof_off[a][i];
          b += (int64_t)(o - dc.lo[i]) * st[i];
          t.stride[a * 3 + i] = (int32_t)st[i];
          t.cmin[a * 3 + i] = (int16_t)std::max(0, dc.lo[i] - o);
          t.cmax[a * 3 + i] = (int16_t)std::min(n[i] - 1, dc.hi[i] - o);
        }
        t.base[a] = b;
      }
    }
  }

  // DOF key of every layout slot of level q (CONVENTIONS of fcm_mg.h)
  void keys(int q, int64_t* out) const {
    int64_t W = 2 * (int64_t)n[0] + 1;
    for (auto& dc : classes) {
      if (dc.order > q) continue;
      for (int64_t i = 0; i < dc.count; ++i) {
        int64_t t = i;
        int64_t X[3] = {0, 0, 0};
        for (int a = 0; a < 3; ++a) {
          int64_t pos = dc.lo[a] + t % std::max(1, dc.size[a]);
          t /= std::max(1, dc.size[a]);
          if (a < dim) X[a] = (dc.S >> a & 1) ? 2 * pos + 1 : 2 * pos;
        }
        X[dim - 1] += 2 * (int64_t)zoff;
        int64_t k = (X[2] * W + X[1]) * W + X[0];
        k = ((k * (p + 1) + dc.deg[2]) * (p + 1) + dc.deg[1]) * (p + 1) + dc.deg[0];
        out[dc.off + i] = k * n_f + dc.comp;
      }
    }
  }

  // local index (in a cell) of the DOF with class `cls` and entity offsets `off`, or -1
  int local_of(int cls, const int off[3]) const {
    for (int a = 0; a < m; ++a) {
      if (dof_class[a] != cls) continue;
      bool ok = true;
      for (int i = 0; i < dim; ++i) if (dof_off[a][i] != off[i]) ok = false;
      if (ok) return a;
    }
    return -1;
  }

  void cell_coords(int64_t c, int cc[3]) const {
    cc[0] = (int)(c % n[0]);
    cc[1] = (int)((c / n[0]) % n[1]);
    cc[2] = (int)(c / ((int64_t)n[0] * n[1]));
  }

  // global layout index of local DOF a of cell cc on level table q, or -1 (Dirichlet)
  int64_t dof_index(int q, int a, const int cc[3]) const {
    const LevelTable& t = tables[q];
    int64_t idx = t.base[a];
    for (int i = 0; i < 3; ++i) {
      if (cc[i] < t.cmin[a * 3 + i] || cc[i] > t.cmax[a * 3 + i]) return -1;
      idx += (int64_t)cc[i] * t.stride[a * 3 + i];
    }
    return idx;
  }
};

}  // namespace fcm
