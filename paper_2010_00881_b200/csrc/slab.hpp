// slab.hpp -- host logic of the slab decomposition ("the same
// partition on every level"): the cell grid is cut into contiguous layers along the
// LAST axis (z in 3D, y in 2D); rank r owns cell layers [z0, z1).  Its local vector holds the
// DOFs of its own cells, both interface planes included (they are duplicated on the two
// neighbouring ranks); an interface DOF is OWNED (for dot products) by the lower rank.
// After every element-by-element scatter the two copies of an interface plane are summed
// (a + b == b + a, so both ranks hold bit-identical values).  Shared by the library and the
// host-only C-ABI functions the multi-process CPU tests call.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

#include "layout.hpp"

namespace fcm {

inline void slab_bounds(int n, int nranks, int rank, int* z0, int* z1) {
  const int base = n / nranks, rem = n % nranks;
  *z0 = rank * base + std::min(rank, rem);
  *z1 = *z0 + base + (rank < rem ? 1 : 0);
}

// Dirichlet mask of a slab: the slab-axis faces are box faces only at the ends of the grid
inline uint32_t slab_dmask(uint32_t dmask, int dim, int z0, int z1, int n) {
  const int ax = dim - 1;
  if (z0 > 0) dmask &= ~(1u << (2 * ax));
  if (z1 < n) dmask &= ~(1u << (2 * ax + 1));
  return dmask;
}

// Local layout of the slab (owned cells only), DOF keys offset to global positions.
inline void slab_layout(Layout& L, int dim, const int n_glob[3], int p, int space, int n_f,
                        uint32_t dmask_glob, int z0, int z1) {
  int nl[3] = {n_glob[0], n_glob[1], n_glob[2]};
  nl[dim - 1] = z1 - z0;
  L.build(dim, nl, p, space, n_f, slab_dmask(dmask_glob, dim, z0, z1, n_glob[dim - 1]));
  L.zoff = z0;
}

// Slots of level q lying on the local slab-axis vertex plane zl (0 = bottom, nz_local = top),
// in class order (identical on both ranks sharing the plane).
inline void plane_slots(const Layout& L, int q, int zl, std::vector<int32_t>& out) {
  out.clear();
  const int ax = L.dim - 1;
  for (const DofClass& dc : L.classes) {
    if (dc.order > q || (dc.S >> ax & 1)) continue;   // internal along the axis: no plane DOF
    if (zl < dc.lo[ax] || zl > dc.hi[ax] || dc.count == 0) continue;
    int64_t plane = 1;
    for (int i = 0; i < ax; ++i) plane *= dc.size[i];
    const int64_t first = dc.off + (int64_t)(zl - dc.lo[ax]) * plane;
    for (int64_t k = 0; k < plane; ++k) out.push_back((int32_t)(first + k));
  }
}

// Owner mask of level q: 0 on the bottom interface plane when a lower rank exists.
inline void owned_mask(const Layout& L, int q, bool has_lower, std::vector<uint8_t>& own) {
  own.assign(L.ndof_level[q], 1);
  if (!has_lower) return;
  std::vector<int32_t> b;
  plane_slots(L, q, 0, b);
  for (int32_t i : b) own[i] = 0;
}

// Global coarse (q = 1) slot of every local level-1 slot, the global layout being the one of
// the full grid (Lg).  The level-1 classes are the vertex classes (one per component).
inline void coarse_global_slots(const Layout& L, const Layout& Lg, std::vector<int64_t>& g) {
  g.assign(L.ndof_level[1], -1);
  const int ax = L.dim - 1;
  for (size_t ci = 0; ci < L.classes.size(); ++ci) {
    const DofClass& dc = L.classes[ci];
    if (dc.order > 1) continue;
    const DofClass* gc = nullptr;
    for (const DofClass& c2 : Lg.classes)
      if (c2.order == dc.order && c2.S == dc.S && c2.comp == dc.comp && c2.deg[0] == dc.deg[0] &&
          c2.deg[1] == dc.deg[1] && c2.deg[2] == dc.deg[2])
        gc = &c2;
    if (!gc) continue;
    for (int64_t i = 0; i < dc.count; ++i) {
      int64_t t = i, gi = gc->off, st = 1;
      for (int a = 0; a < 3; ++a) {
        const int sz = std::max(1, dc.size[a]);
        int pos = dc.lo[a] + (int)(t % sz);
        t /= sz;
        if (a == ax) pos += L.zoff;
        gi += (int64_t)(pos - gc->lo[a]) * st;
        st *= std::max(1, gc->size[a]);
      }
      g[dc.off + i] = gi;
    }
  }
}

}  // namespace fcm
