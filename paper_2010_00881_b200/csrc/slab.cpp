// slab.cpp -- host-only C-ABI functions of the slab decomposition (include/fcm_mg.h, "multi-
// GPU"): the partition, the local layout / interface planes / owner mask, and the global
// coarse mapping.  No CUDA: the multi-process CPU tests call these to check the host logic
// the library's NCCL path runs on.
#include <cstring>
#include <vector>

#include "../../include/fcm_mg.h"
#include "common.hpp"
#include "slab.hpp"

using namespace fcm;

static int check_grid(const fcm_grid* g) {
  if (!g || g->dim < 2 || g->dim > 3 || g->p < 1 || g->n_f < 1) return fail(FCM_EINVAL, "bad grid");
  for (int i = 0; i < g->dim; ++i)
    if (g->n[i] < 1) return fail(FCM_EINVAL, "bad grid extents");
  return FCM_OK;
}

extern "C" int fcm_slab_bounds(int32_t n, int32_t nranks, int32_t rank, int32_t* z_begin, int32_t* z_end) {
  clear_error();
  if (!z_begin || !z_end || nranks < 1 || rank < 0 || rank >= nranks || n < nranks)
    return fail(FCM_EINVAL, "bad slab partition (n=%d, nranks=%d, rank=%d)", n, nranks, rank);
  int a, b;
  slab_bounds(n, nranks, rank, &a, &b);
  *z_begin = a;
  *z_end = b;
  return FCM_OK;
}

extern "C" int fcm_slab_layout(const fcm_grid* g, int32_t z_begin, int32_t z_end, int32_t q, int64_t* ndofs,
                               int64_t* keys, uint8_t* owned, int64_t* n_lo, int32_t* lo_slots,
                               int64_t* n_hi, int32_t* hi_slots) {
  clear_error();
  int rc = check_grid(g);
  if (rc < 0) return rc;
  const int ax = g->dim - 1, n = g->n[ax];
  if (z_begin < 0 || z_end > n || z_begin >= z_end || q < 1 || q > g->p) return fail(FCM_EINVAL, "bad slab");
  Layout L;
  slab_layout(L, g->dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces, z_begin, z_end);
  if (ndofs) *ndofs = L.ndof_level[q];
  if (keys) {
    std::vector<int64_t> k(L.ndof_level[g->p]);
    L.keys(g->p, k.data());
    std::memcpy(keys, k.data(), L.ndof_level[q] * 8);   // the level-q vector is a prefix
  }
  if (owned) {
    std::vector<uint8_t> o;
    owned_mask(L, q, z_begin > 0, o);
    std::memcpy(owned, o.data(), o.size());
  }
  std::vector<int32_t> lo, hi;
  if (z_begin > 0) plane_slots(L, q, 0, lo);
  if (z_end < n) plane_slots(L, q, z_end - z_begin, hi);
  if (n_lo) *n_lo = (int64_t)lo.size();
  if (n_hi) *n_hi = (int64_t)hi.size();
  if (lo_slots && !lo.empty()) std::memcpy(lo_slots, lo.data(), lo.size() * 4);
  if (hi_slots && !hi.empty()) std::memcpy(hi_slots, hi.data(), hi.size() * 4);
  return FCM_OK;
}

extern "C" int fcm_slab_coarse_map(const fcm_grid* g, int32_t z_begin, int32_t z_end, int64_t* n_local,
                                   int64_t* global_slots) {
  clear_error();
  int rc = check_grid(g);
  if (rc < 0) return rc;
  const int ax = g->dim - 1, n = g->n[ax];
  if (z_begin < 0 || z_end > n || z_begin >= z_end) return fail(FCM_EINVAL, "bad slab");
  Layout L, Lg;
  slab_layout(L, g->dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces, z_begin, z_end);
  Lg.build(g->dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces);
  std::vector<int64_t> gs;
  coarse_global_slots(L, Lg, gs);
  if (n_local) *n_local = (int64_t)gs.size();
  if (global_slots) std::memcpy(global_slots, gs.data(), gs.size() * 8);
  return FCM_OK;
}
