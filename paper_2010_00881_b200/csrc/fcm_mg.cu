// fcm_mg.cu -- B200 (sm_100a) implementation of the C ABI in include/fcm_mg.h.
//
// Hot path:
//   (a3) level operator apply    k_cell_mma<M,G> OP_APPLY   r -= A_q x: regular
//                                cells as fp64 MMA groups + individual cut cells (list) in one launch
//   (a4) additive Schwarz        k_cell_mma<M,G> OP_SMOOTH  x += w M^-1 r;
//                                k_block_smooth for patch blocks (blocks.cuh)
//   (a5) restriction / prolong.  pointer alias (prefix) / k_axpy on the prefix
//   (a6) coarsest level p=1      k_coarse_tiled (shared-memory bricks) or k_coarse_pcg (grid-wide),
//                                cooperative, whole inner CG in one launch
//                                or k_dense_gemv with a setup-time inverse
//   (a2) V-cycle                 enqueue_vcycle (Algorithm 1), CUDA graph
//   (a1) flexible PCG            fcm_pcg_solve
//   (a7) BLAS-1                  deterministic block partials, device-resident scalars
// Setup (a0): Schwarz block classification (shared-by-type vs individual), block assembly
// A_i = P_i^T A_q P_i and in-place Gauss-Jordan inversion on the device.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/fcm_mg.h"
#include "cellop.cuh"
#include "coarse.cuh"
#include "coarse_tiled.cuh"
#include "blocks.cuh"
#include "patch.cuh"
#include "patch_wb.cuh"
#include "cellmma.cuh"
#include "cellws.cuh"
#include "common.hpp"
#include "layout.hpp"
#include "nccl_dl.hpp"
#include "slab.hpp"

namespace cg = cooperative_groups;
using namespace fcm;

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? FCM_ENOMEM : FCM_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                  \
  } while (0)

#define RC(call)           \
  do {                     \
    int rc_ = (call);      \
    if (rc_ < 0) return rc_; \
  } while (0)

namespace fcm {
void ref1d_matrices(int p, double* M, double* K);   // gen.cpp
}

namespace {

constexpr int kThreads = 256;
constexpr int kMaxPartials = 2048;

// coarse CG preconditioned by the geometric V-cycle (FCM_COARSE_GMG_PCG): device scalars
struct GcgScalars {
  double rz, rz_new, rr0, rr, pq;
  int it, maxit, flag, pad;
  double rtol2;
};

struct Scalars {
  double rz, pq, rr, zr, zr_old, bb;
  int flag;  // bit0: p^T A p <= 0
  int pad;
  double red[4];  // slab mode: all-reduced partial sums (pq | zr, zr_old | rz)
  // device-side FCG loop (k_fcg_check): iteration count, stop test, history
  int it, maxit;
  double rtol2;
};

struct LevelDev {
  int q = 0, m = 0, G = 32;
  int64_t ndof = 0;
  int64_t* base = nullptr;
  int32_t* stride = nullptr;
  int16_t* cmin = nullptr;
  int16_t* cmax = nullptr;
  // additive Schwarz
  bool has_as = false;
  double omega = 1.0;
  int32_t* blk = nullptr;
  double* irr_inv = nullptr;
  double* type_inv = nullptr;
  int64_t n_irr = 0;
  int32_t n_types = 0;
  int M = 0;                       // compile-time block size of the regular path (0: generic)
  const void* kreg = nullptr;      // k_cell_reg<M> (regular population)
  const void* klist = nullptr;     // k_cell_list<G> (individual list / generic)
  int32_t* irr_list = nullptr;     // cells with an individual Schwarz inverse (irr order)
  int ilo[3] = {0, 0, 0}, ihi[3] = {-1, -1, -1};  // cells with no Dirichlet DOF
  int ts = 1;                      // threads per cell of the regular path
  const void* kmma = nullptr;      // k_cell_mma<M>: regular cells as fp64 tensor-core MMAs
  int32_t* gA_cells = nullptr;     // apply groups (8 non-cut cells, K_ref)
  int32_t* gA_mat = nullptr;
  int64_t nA = 0;
  int32_t* gS_cells = nullptr;     // smoother groups (8 regular cells of one type slot)
  int32_t* gS_mat = nullptr;
  int64_t nS = 0;
  // warp-specialised launch (cellws.cuh): MMA warps for the regular cells + streaming warps for
  // the tile-packed individual matrices (operator: the fine cut-cell copy; smoother: irr_tp)
  const void* kws = nullptr;       // the level has warp-specialised launches (= kws_m[OP_APPLY])
  const void* kws_m[2] = {nullptr, nullptr};   // per mode (OP_APPLY / OP_SMOOTH): warp split variant
  int ws_threads[2] = {0, 0};      // threads per CTA
  size_t ws_smem_b[2] = {0, 0};    // dynamic smem
  int ntq = 0;                     // 32-tiles per dimension of the level block (ceil(m / 32))
  double* irr_tp = nullptr;        // tile-packed individual elementwise inverses (replaces irr_inv)
  int64_t irr_tps = 0;             // doubles per packed inverse
  std::vector<int32_t> blk_h;      // host copy of blk (tiled coarse setup)
  // patchwise blocks (blocks.cuh): anchors are grid vertices, blk is per anchor
  bool patch = false;
  int mb = 0;                      // block size (= m for elementwise)
  int nmem = 1;
  int mo[8][3] = {};
  int na[3] = {1, 1, 1};
  int64_t nanchor = 0;
  int8_t* d_mem = nullptr;
  int16_t* d_loc = nullptr;
  // patch levels at scale (patch.cuh): tile-packed individual inverses, regular-anchor list,
  // fast-diagonalisation tables
  int nt = 0;                      // 32x32 tiles per dimension of a packed inverse
  int64_t pstride = 0;             // doubles per packed inverse
  int64_t* irr_anchor = nullptr;   // [n_irr] anchor of individual block i
  unsigned long long* sched = nullptr;   // k_patch_smooth dynamic-scheduling counters (3, zeroed)
  bool swz = false;                      // patch inverses: off-diagonal tiles rotated (tile_pos)
  std::vector<int64_t> irr_col, reg_col;   // deterministic mode: colour ranges (27) of the sorted lists
  int32_t* reg_list = nullptr;     // regular anchors (fast diagonalisation / k_block_smooth)
  int64_t n_reg = 0;
  bool fd = false;
  double* fd_tabs = nullptr;       // [3][ncls][S*S + S]
  int* fd_cls = nullptr;           // [na0 + na1 + na2] axis class of each anchor coordinate
  int fd_ncls = 0;
  int16_t* fd_midx = nullptr;      // [(q+1)^3] local DOF of element mode (kx,ky,kz)
  double fd_s = 1.0;
  std::vector<double> fd_tabs_h;   // host copies (low-rank patch setup)
  std::vector<int> fd_cls_h;
  // individual patches as low-rank corrections of the regular patch (patch_wb.cuh)
  int64_t n_wb = 0;
  int64_t* wb_anchor = nullptr;    // [n_wb]
  int64_t* wb_soff = nullptr;      // [n_wb + 1]
  int16_t* wb_slots = nullptr;     // S lists (block slots)
  int64_t* wb_coff = nullptr;      // [n_wb + 1]
  double* wb_C = nullptr;          // k x k per patch
  int16_t* wb_tsl = nullptr;       // [mb] tensor slot of block slot l
  int16_t* wb_tS = nullptr;        // S lists as tensor slots (the fused path in k_patch_smooth)
  bool wb_fused = false;           // low-rank patches by k_patch_smooth's FD warps (else k_patch_wb)
  bool fd_roll = false;            // FD passes with the input loop rolled (small code; streaming-dominated levels)
  std::vector<int64_t> wb_anchor_h, wb_soff_h, wb_coff_h;
  std::vector<int16_t> wb_slots_h, wb_tsl_h;
  // slab mode: interface planes (exchange order) and the smoother increment vector
  int32_t* lo_idx = nullptr;
  int32_t* hi_idx = nullptr;
  int64_t n_lo = 0, n_hi = 0;
  double* d = nullptr;
  double* r2 = nullptr;            // second residual buffer (fused-copy V-cycle)
  // vectors
  double* x = nullptr;
  double* r = nullptr;
};

}  // namespace

struct fcm_mg {
  Layout L;
  fcm_grid g{};
  fcm_params prm{};
  cudaStream_t stream = nullptr;   // internal non-blocking stream (capturable)
  cudaStream_t ustream = nullptr;  // the caller's stream (params.stream)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaStream_t stream2 = nullptr;  // second branch: individual-cell kernels run concurrently
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int dev = 0, num_sms = 148;
  double alpha = 1e-8;
  int64_t ncell = 0, ncut = 0;
  int wb_mode = 0;                     // FCM_WB_KERNEL: 0 cost model, 1 always k_patch_wb, 2 always fused
  const double* Kref_host = nullptr;   // setup only (low-rank patch corrections)
  const double* cutK_host = nullptr;
  uint8_t* d_kind = nullptr;        // owned cells (= d_kind_ext + owned offset)
  int32_t* d_cut_idx = nullptr;
  uint8_t* d_kind_ext = nullptr;    // owned + ghost cell layers (Schwarz assembly)
  int32_t* d_cut_idx_ext = nullptr;
  int32_t* d_cut_list = nullptr;  // cut cells in cut order
  const void* kcoarse = nullptr;
  double* d_Kref = nullptr;
  double* d_cutK = nullptr;
  double* d_cutK_tp = nullptr;      // tile-packed copy of the cut-cell matrices (k_cell_ws levels)
  int64_t cut_tps = 0;              // doubles per packed cut-cell matrix
  std::vector<LevelDev> lev;  // index q = 1..p
  // coarse
  double* d_A0inv = nullptr;   // direct
  double* d_diag_inv = nullptr;  // Jacobi
  double* c_vec[9] = {};  // r[2], z[2], w[2], q[2], p
  double* c_part = nullptr;
  GridCtl* c_ctl = nullptr;
  int* d_coarse_iters = nullptr;
  int coarse_blocks = 0;
  // tiled coarse solver (coarse_tiled.cuh): used when every brick fits in shared memory
  const void* ktiled = nullptr;
  TiledArgs tiled{};
  int t_blocks = 0;
  size_t t_smem = 0;
  std::vector<double> t_feat;   // FCM_TILED_PROF: per-brick model features (calibration)
  // FCG
  double *f_b = nullptr, *f_x = nullptr, *f_r = nullptr, *f_ro = nullptr, *f_p = nullptr, *f_q = nullptr;
  Scalars* d_s = nullptr;
  Scalars* h_s = nullptr;  // pinned
  int* h_iters = nullptr;  // pinned
  double* d_partA = nullptr;
  double* d_partB = nullptr;
  double* d_partC = nullptr;
  // graphs
  cudaGraphExec_t g_vc = nullptr, g_it1 = nullptr, g_it2 = nullptr, g_init = nullptr, g_mgit = nullptr;
  cudaGraphExec_t g_solve = nullptr;   // whole FCG: init, it1, check, WHILE { it2, it1, check }
  int64_t n_loop = 0, n_head = 0;      // kernels per loop trip / in the head
  double* d_hist = nullptr;
  int hist_cap = 0;
  int64_t n_vc = 0, n_it1 = 0, n_it2 = 0, n_init = 0, n_mgit = 0;  // kernels per graph
  int64_t launches = 0;
  int64_t* count_target = nullptr;  // during capture: where launches are counted
  int64_t stat_coarse = 0, stat_vcycles = 0;
  std::vector<void*> allocs;
  // slab decomposition (slab.hpp; nranks == 1: single GPU, no collective)
  int rank = 0, nranks = 1, z0 = 0, z1 = 0;
  bool multi = false;               // slab mode (nranks > 1, or FCM_FORCE_SLAB on one rank: tests)
  int mma_bps = 4, list_bps = 8;    // blocks per SM of the MMA / list parts of k_cell_mma
  int ws_ctas = 148;                // CTAs of a k_cell_ws launch (num_sms; FCM_WS_CTAS: tests)
  // deterministic mode (FCM_DETERMINISTIC=1): every scatter in colour passes (2^d cell parities,
  // 27 vertex classes for patches) so each output entry receives at most one fp64 atomic per
  // launch, per-patch sums in a fixed warp order, energies by block-order dots, block-order
  // coarse sums: bit-identical results run to run (debugging; several times slower)
  bool det = false;
  unsigned long long* patch_prof = nullptr;   // FCM_PATCH_PROF=1: k_patch_smooth population end times
  int fd_roll_mode = -1;   // FCM_FD_ROLL: -1 per-level cost model, 0 never, 1 always (patch.cuh fd_pass ROLL)
  bool l2ef = true;    // stream read-once matrices with an L2 evict_first policy (FCM_L2_EVICT_FIRST=0: off)
  int pdl = 1;                      // programmatic dependent launch of k_cell_mma (FCM_PDL)
  int ext_lo = 0, ext_n = 0;        // ghost-extended cell layers along the slab axis (relative)
  int64_t cut_first = 0;            // first owned cut cell in the cut-matrix array
  ncclComm_t comm = nullptr;
  double* x_send = nullptr;         // [2][max plane] bottom / top
  double* x_recv = nullptr;
  uint8_t* d_own = nullptr;         // owner mask of the fine level (dots)
  fcm_mg* hg = nullptr;             // replicated global p = 1 problem (coarse solve)
  bool borrowed_stream = false;
  int32_t* c_pack = nullptr;        // owned local level-1 slots (allgather order)
  int64_t c_count = 0, c_max = 0;
  double* c_send = nullptr;
  double* c_recv = nullptr;         // [nranks][c_max]
  int64_t* c_unpack = nullptr;      // [nranks * c_max] global level-1 slot (-1 padding)
  // h-coarsening below p = 1 (FCM_COARSE_GMG_PCG, PAPER.md:227 Remark): child handles of the
  // p=1 problem on grids n/2, n/4, ... (their level 1 = the h-level; the last one solves
  // directly); per h-level right-hand side / solution buffers; the coarse CG scalars
  std::vector<fcm_mg*> gmg;         // h-levels 1..L
  std::vector<double*> gmg_b, gmg_x;   // [L + 1] (index 0 unused: the coarse CG's r / z)
  double gmg_omega = 1.0;
  GcgScalars* gcg = nullptr;
  cudaStream_t st_c[2] = {nullptr, nullptr};   // capture streams of the nested conditional bodies
  cudaGraphExec_t g_coarse = nullptr;          // stand-alone coarse solve (fcm_mg_coarse_solve)
  double *c_bst = nullptr, *c_xst = nullptr;   // its staged input / output
  int64_t n_gcg_body = 0;                      // kernels per coarse CG trip (launch accounting)
  int64_t n_coarse_g = 0;
  bool gmg_child = false;
  int64_t* c_extract = nullptr;     // [ndof_1 local] global level-1 slot
  // slab mode + h-coarsening (FCM_COARSE_GMG_PCG): DISTRIBUTED coarse solve -- the p=1 level
  // stays z-slab partitioned ("reuse the parallel data structures"), the coarse CG and the
  // h-level-0 smoothing run on the slabs with the interface exchange and all-reduced dots; the
  // restricted residual of h-level 1 is all-reduced and the geometric V-cycle below it runs
  // replicated (hg's h-levels).  The coarse CG is host-driven (one small D2H per iteration), so
  // the slab V-cycle/FCG run eagerly (no graphs: NCCL work stays out of conditional nodes).
  bool dist = false;
  bool eager = false;
  std::map<const void*, std::function<int()>> eager_fn;   // capture() bodies in eager mode
  double* d_dcg = nullptr;          // [8] reduced scalars of the distributed coarse CG
  double* h_dcg = nullptr;          // pinned copy
  int* h_ci = nullptr;              // pinned {iterations of the last coarse solve, total}
  int dist_cz0 = 0, dist_cz1 = 0;   // global coarse (h-level 1) vertex layers this slab restricts to
  double* c_bg = nullptr;
  double* c_xg = nullptr;

  template <typename T>
  int alloc(T** p, size_t n) {
    size_t bytes = std::max<size_t>(1, n * sizeof(T));
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess)
      return fail(FCM_ENOMEM, "cudaMalloc of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    allocs.push_back(*p);
    return FCM_OK;
  }
  void count(int64_t k = 1) {
    if (count_target) *count_target += k;
    else launches += k;
  }
  ~fcm_mg();
  void release() {
    if (!eager)   // eager mode stores sentinels, not graphs
      for (auto g : {g_vc, g_it1, g_it2, g_init, g_mgit, g_solve})
        if (g) cudaGraphExecDestroy(g);
    if (h_dcg) cudaFreeHost(h_dcg);
    if (h_ci) cudaFreeHost(h_ci);
    for (void* p : allocs) cudaFree(p);
    if (h_s) cudaFreeHost(h_s);
    if (h_iters) cudaFreeHost(h_iters);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (stream && !borrowed_stream) cudaStreamDestroy(stream);
    if (stream2) cudaStreamDestroy(stream2);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
};
fcm_mg::~fcm_mg() {
  if (hg) delete hg;
  for (fcm_mg* c : gmg) delete c;
  if (g_coarse) cudaGraphExecDestroy(g_coarse);
  for (auto st : st_c)
    if (st) cudaStreamDestroy(st);
  if (comm && nccl().ok) nccl().CommDestroy(comm);
  release();
}

// =========================================================================================
// kernels
// =========================================================================================
namespace {

// Regular population: one thread per cell (compile-time M); smem [Tab][Ms: M*MP doubles].
template <int M, int TS>
__global__ void __launch_bounds__(kThreads, 4) k_cell_reg(CellOp op) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* Ms = reinterpret_cast<double*>(smem + sizeof(Tab));
  __shared__ double red[32];
  load_tab(T, op);
  load_shared_matrix<M>(Ms, op);
  __syncthreads();
  const int wpb = blockDim.x >> 5;
  double* xs = Ms + M * padded<M>() + (threadIdx.x >> 5) * reg_scratch<M, TS>();
  const double e = reg_cells<M, TS, false>(op, T, Ms, xs, blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb);
  if (op.partials) {
    const double t = block_sum(e, red);
    if (threadIdx.x == 0) op.partials[blockIdx.x] = t;
  }
}

// One launch per cell operation: blocks [0, nb_mma) run the regular cells as fp64 MMAs
// (cellmma.cuh), the others the individual list (list_cells); every block also does its share
// of the fused copy.  smem [Tab][max(A fragments, list scratch)].
template <int M, int G>
__global__ void __launch_bounds__(kThreads, M > 32 ? 2 : 4) k_cell_mma(MmaOp g, int nb_mma) {
  extern __shared__ __align__(16) unsigned char smem[];
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* As = reinterpret_cast<double*>(smem + sizeof(Tab));
  __shared__ double red[32];
  load_tab(T, g.op);
  const bool apply = g.op.mode == OP_APPLY;
  const bool is_mma = (int)blockIdx.x < nb_mma;
  // programmatic dependent launch: let the next launch's blocks be scheduled as soon as every
  // block of this one is running; the prologue above and the staging below touch only static
  // data (tables, K_ref, Schwarz inverses), so they overlap the previous launch's tail, and
  // griddepcontrol.wait (a no-op without the launch attribute) orders the vector accesses
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (is_mma) stage_fragments<M>(As, apply ? g.op.Kref : g.op.type_inv, apply ? g.op.ldK : M);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int wpb = blockDim.x >> 5;
  double e;
  if (is_mma) {
    e = mma_cells<M>(g.op, g.grp_cells, g.grp_mat, g.ngroups, T, As, apply ? -1 : 0,
                     blockIdx.x * wpb + (threadIdx.x >> 5), nb_mma * wpb);
  } else {
    constexpr int CPW = 32 / G;
    double* xs = As + (threadIdx.x >> 5) * CPW * g.op.m;
    int* ids = reinterpret_cast<int*>(As + wpb * CPW * g.op.m) + (threadIdx.x >> 5) * CPW * g.op.m;
    e = list_cells<G, false, (M <= 32 ? M : 0)>(g.op, T, (blockIdx.x - nb_mma) * wpb + (threadIdx.x >> 5),
                                               (gridDim.x - nb_mma) * wpb, xs, ids);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.cp_n; i += (int64_t)gridDim.x * blockDim.x)
    g.cp_dst[i] = g.cp_src[i];
  if (g.op.partials) {
    const double t = block_sum(e, red);
    if (threadIdx.x == 0) g.op.partials[blockIdx.x] = t;
  }
}

// One cell operation as a warp-specialised persistent launch (cellws.cuh): warps [0, NS) stream
// the tile-packed individual matrices through STG-deep rings, warps [NS, NS + NM) run the regular
// cells as fp64 MMA groups.  smem [Tab][A fragments][ring: NS x STG x 8 KB][mbarriers][xs, ys, ids].
template <int M, int NS, int NM, int STG, bool PF = true>
__host__ __device__ constexpr size_t ws_smem() {
  return sizeof(Tab) + (size_t)((M + 7) / 8) * ((M + 3) / 4) * 32 * 8 + ws_stream_smem((M + 31) / 32, NS, STG);
}
template <int M, int NS, int NM, int STG, bool PF>
__global__ void __launch_bounds__((NS + NM) * 32, 1) k_cell_ws(MmaOp g, TileListOp tl) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int MT = (M + 7) / 8, KT = (M + 3) / 4;
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* As = reinterpret_cast<double*>(smem + sizeof(Tab));
  double* ring = As + MT * KT * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)NS * STG * 1024);
  double* xs0 = reinterpret_cast<double*>(bars + NS * STG);
  __shared__ double red[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MPd = 32 * tl.ntq;
  const int ntl = tl.ntq * (tl.ntq + 1) / 2;
  const int64_t gw = (int64_t)blockIdx.x * NS + w, W = (int64_t)gridDim.x * NS;
  load_tab(T, g.op);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const bool apply = g.op.mode == OP_APPLY;
  stage_fragments<M>(As, apply ? g.op.Kref : g.op.type_inv, apply ? g.op.ldK : M);
  if (w < NS && lane == 0)
    for (int s = 0; s < STG; ++s) mbar_init(&bars[w * STG + s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (w < NS && lane == 0) {   // the first tiles: setup data, so before griddepcontrol.wait
    const int64_t nitems = (tl.nlist > gw ? (tl.nlist - gw + W - 1) / W : 0) * ntl;
    for (int64_t i = 0; i < STG && i < nitems; ++i)
      ws_issue<STG>(tl, ntl, gw, W, i, ring + (size_t)w * STG * 1024, bars + w * STG, g.op.m);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double e;
  if (w < NS) {
    double* xs = xs0 + (size_t)w * MPd * 2;
    int* ids = reinterpret_cast<int*>(xs0 + (size_t)NS * MPd * 2) + (size_t)w * MPd;
    e = ws_stream_cells<(M + 31) / 32, STG>(g.op, tl, T, xs, xs + MPd, ids, ring + (size_t)w * STG * 1024,
                                            bars + w * STG, gw, W);
  } else {
    e = mma_cells<M, false, PF && (M + 3) / 4 <= 16>(g.op, g.grp_cells, g.grp_mat, g.ngroups, T, As, apply ? -1 : 0,
                                               blockIdx.x * NM + (w - NS), gridDim.x * NM);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.cp_n; i += (int64_t)gridDim.x * blockDim.x)
    g.cp_dst[i] = g.cp_src[i];
  if (g.op.partials) {
    const double t = block_sum(e, red);
    if (threadIdx.x == 0) g.op.partials[blockIdx.x] = t;
  }
}

// symmetric m x m matrices (row-major, consecutive at mstride doubles) -> tile-packed lower
// storage with nt tiles per dimension (patch.cuh layout; entries beyond m are 0); grid (tiles, matrices)
__global__ void k_pack_tiles_ld(const double* __restrict__ A, int m, int64_t mstride, int nt, double* __restrict__ out,
                                int64_t ostride) {
  const int t = blockIdx.x;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  const int J = t - I * (I + 1) / 2;
  const double* M = A + (int64_t)blockIdx.y * mstride;
  double* o = out + (int64_t)blockIdx.y * ostride + tile_off(I, J);
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    const int gi = 32 * I + r, gj = 32 * J + c;
    const double v = (gi < m && gj < m) ? 0.5 * (M[(int64_t)gi * m + gj] + M[(int64_t)gj * m + gi]) : 0.0;
    if (I != J) o[e] = v;
    else if (c <= r) o[r * (r + 1) / 2 + c] = v;
  }
}

// Individual population (or, without compile-time M, every cell): groups of G lanes per cell;
// smem [Tab][xs: wpb*CPW*m doubles][ids: wpb*CPW*m ints].  Partials at part_off + block.
template <int G>
__global__ void __launch_bounds__(kThreads) k_cell_list(CellOp op, int part_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CPW = 32 / G;
  const int wpb = blockDim.x >> 5;
  Tab& T = *reinterpret_cast<Tab*>(smem);
  double* xs0 = reinterpret_cast<double*>(smem + sizeof(Tab));
  double* xs = xs0 + (threadIdx.x >> 5) * CPW * op.m;
  int* ids = reinterpret_cast<int*>(xs0 + wpb * CPW * op.m) + (threadIdx.x >> 5) * CPW * op.m;
  __shared__ double red[32];
  load_tab(T, op);
  __syncthreads();
  const double e = list_cells<G, false>(op, T, blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb, xs, ids);
  if (op.partials) {
    const double t = block_sum(e, red);
    if (threadIdx.x == 0) op.partials[part_off + blockIdx.x] = t;
  }
}

// slab mode: interface planes (index lists in exchange order)
__global__ void k_zero_idx(double* __restrict__ v, const int32_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[idx[i]] = 0.0;
}
__global__ void k_pack2(double* __restrict__ buf, const double* __restrict__ v, const int32_t* __restrict__ lo,
                        int64_t nlo, const int32_t* __restrict__ hi, int64_t nhi, int64_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nlo + nhi; i += (int64_t)gridDim.x * blockDim.x)
    buf[i < nlo ? i : stride + i - nlo] = v[i < nlo ? lo[i] : hi[i - nlo]];
}
// v[plane] = v[plane] + received neighbour partial (a + b == b + a on both ranks)
__global__ void k_unpack_add2(double* __restrict__ v, const double* __restrict__ buf, const int32_t* __restrict__ lo,
                              int64_t nlo, const int32_t* __restrict__ hi, int64_t nhi, int64_t stride) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nlo + nhi; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i < nlo ? lo[i] : hi[i - nlo];
    v[j] = v[j] + buf[i < nlo ? i : stride + i - nlo];
  }
}
__global__ void k_gather32(double* __restrict__ out, const double* __restrict__ in, const int32_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}
__global__ void k_gather64(double* __restrict__ out, const double* __restrict__ in, const int64_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}
__global__ void k_scatter64(double* __restrict__ out, const double* __restrict__ in, const int64_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (idx[i] >= 0) out[idx[i]] = in[i];
}

// Programmatic dependent launch (launches through pdl_launch): wait until the preceding
// kernel has completed and its writes are visible, then let the next launch be scheduled.
// A no-op for ordinary launches.
#define FCM_PDL_ENTRY()                                      \
  do {                                                       \
    asm volatile("griddepcontrol.wait;" ::: "memory");       \
    asm volatile("griddepcontrol.launch_dependents;" :::);   \
  } while (0)

__global__ void k_fill(double* x, double v, int64_t n) {
  FCM_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}
__global__ void k_copy(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}
// y[0..n) += a x; dst[0..ncp) = src (fused copy of an unrelated buffer)
__global__ void k_axpy_copy(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n,
                            double* __restrict__ dst, const double* __restrict__ src, int64_t ncp) {
  FCM_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n || i < ncp; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) y[i] = fma(a, x[i], y[i]);
    if (i < ncp) dst[i] = src[i];
  }
}
__global__ void k_axpy(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
// partials[block] = sum a.b over the block's grid-stride range (fixed grid -> deterministic)
__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* partials,
                      const uint8_t* __restrict__ own = nullptr) {
  FCM_PDL_ENTRY();
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!own || own[i]) s = fma(a[i], b[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
// Deterministic sum of n block partials (fixed lane assignment and shuffle tree): warp 0
// reduces, the result is broadcast through shared memory.  Must be called by all threads.
__device__ __forceinline__ double sum_partials(const double* p, int n) {
  __shared__ double bc;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) s += p[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) bc = s;
  }
  __syncthreads();
  const double v = bc;
  __syncthreads();
  return v;
}
// x = 0, r = b (FCG start); z set later by the V-cycle
__global__ void k_fcg_start(double* x, double* r, const double* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = 0.0;
    r[i] = b[i];
  }
}
// rz = sum partials(z.r) (or the all-reduced value); p = z
__global__ void k_fcg_start2(Scalars* s, const double* part, int np, double* p, const double* z, int64_t n,
                             const double* pre = nullptr) {
  const double v = pre ? *pre : sum_partials(part, np);
  if (blockIdx.x == 0 && threadIdx.x == 0) s->rz = v;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i];
}
// pq = sum partials; alpha = rz/pq; x += alpha p; r_old = r; r -= alpha q; partial rr
__global__ void k_fcg_update1(Scalars* s, const double* part_pq, int npq, double* __restrict__ x,
                              double* __restrict__ r, double* __restrict__ r_old,
                              const double* __restrict__ p, const double* __restrict__ q, int64_t n,
                              double* part_rr, const uint8_t* __restrict__ own = nullptr,
                              const double* pre = nullptr) {
  FCM_PDL_ENTRY();
  __shared__ double red[32];
  const double pq = pre ? *pre : sum_partials(part_pq, npq);
  const double alpha = s->rz / pq;
  double rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = r[i];
    r_old[i] = ri;
    const double rn = fma(-alpha, q[i], ri);
    r[i] = rn;
    if (!own || own[i]) rr = fma(rn, rn, rr);
  }
  rr = block_sum(rr, red);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = rr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->pq = pq;
    if (!(pq > 0.0)) s->flag |= 1;
  }
}
__global__ void k_finalize(double* out, const double* part, int np) {
  FCM_PDL_ENTRY();
  const double v = sum_partials(part, np);
  if (threadIdx.x == 0) *out = v;
}
__global__ void k_finalize2(double* out, const double* partA, const double* partB, int np) {
  FCM_PDL_ENTRY();
  const double a = sum_partials(partA, np);
  const double b = sum_partials(partB, np);
  if (threadIdx.x == 0) { out[0] = a; out[1] = b; }
}
// partials of z.r and z.r_old (two sets)
__global__ void k_dot2(const double* __restrict__ z, const double* __restrict__ r,
                       const double* __restrict__ ro, int64_t n, double* partA, double* partB,
                       const uint8_t* __restrict__ own = nullptr) {
  FCM_PDL_ENTRY();
  __shared__ double red[32];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (own && !own[i]) continue;
    const double zi = z[i];
    s1 = fma(zi, r[i], s1);
    s2 = fma(zi, ro[i], s2);
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  if (threadIdx.x == 0) { partA[blockIdx.x] = s1; partB[blockIdx.x] = s2; }
}
// beta = (z.r - z.r_old) / rz_old ; rz = z.r ; p = z + beta p   (Polak-Ribiere, reading R5)
__global__ void k_fcg_update2(Scalars* s, const double* partA, const double* partB, int np,
                              double* __restrict__ p, const double* __restrict__ z, int64_t n,
                              const double* pre = nullptr) {
  FCM_PDL_ENTRY();
  const double zr = pre ? pre[0] : sum_partials(partA, np);
  const double zro = pre ? pre[1] : sum_partials(partB, np);
  const double beta = (zr - zro) / s->rz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) { s->zr = zr; s->zr_old = zro; }
  // rz updated by the last block to finish reading it: use a separate write after grid end
}
// device-side FCG loop: after each x-update, count the iteration, record ||r||/||b||, and keep
// the WHILE node running unless converged (strict <, reading R6), maxit reached, p^T A p <= 0
// or NaN (the host reports the reason after the single synchronisation)
__global__ void k_fcg_check(Scalars* s, cudaGraphConditionalHandle cond, double* hist) {
  if (threadIdx.x != 0) return;
  const int it = ++s->it;
  const double rel2 = s->rr / s->bb;
  if (hist && it <= s->maxit + 1) hist[it] = sqrt(rel2);
  const bool stop = (s->flag & 1) || !(rel2 == rel2) || rel2 < s->rtol2 || it >= s->maxit;
  cudaGraphSetConditional(cond, stop ? 0u : 1u);
}
__global__ void k_set_rz(Scalars* s) {
  FCM_PDL_ENTRY();
  if (threadIdx.x == 0) s->rz = s->zr;
}
// x = Ainv b (dense, row-major, symmetric)
__global__ void k_dense_gemv(const double* __restrict__ A, const double* __restrict__ b,
                             double* __restrict__ x, int64_t n) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < n;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s = fma(A[row * n + j], b[j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) x[row] = s;
  }
}

// ---- h-coarsening below p = 1 (FCM_COARSE_GMG_PCG; PAPER.md:227 Remark, reading R21) ----------
// free vertex boxes of a p = 1 level: one class per component, x fastest (layout.hpp)
struct GmgBox {
  int nf;
  int64_t off[3];
  int lo[3][3], size[3][3];
};
__device__ __forceinline__ int64_t gmg_index(const GmgBox& B, int c, const int x[3]) {
  return B.off[c] + (x[0] - B.lo[c][0]) + ((int64_t)(x[1] - B.lo[c][1]) + (int64_t)(x[2] - B.lo[c][2]) * B.size[c][1]) * B.size[c][0];
}
__device__ __forceinline__ bool gmg_in(const GmgBox& B, int c, const int x[3]) {
  return x[0] >= B.lo[c][0] && x[0] < B.lo[c][0] + B.size[c][0] && x[1] >= B.lo[c][1] &&
         x[1] < B.lo[c][1] + B.size[c][1] && x[2] >= B.lo[c][2] && x[2] < B.lo[c][2] + B.size[c][2];
}
__device__ __forceinline__ void gmg_decode(const GmgBox& B, int64_t i, int& c, int x[3]) {
  c = 0;
  while (c + 1 < B.nf && i >= B.off[c + 1]) ++c;
  int64_t t = i - B.off[c];
  x[0] = (int)(t % B.size[c][0]) + B.lo[c][0];
  t /= B.size[c][0];
  x[1] = (int)(t % B.size[c][1]) + B.lo[c][1];
  x[2] = (int)(t / B.size[c][1]) + B.lo[c][2];
}
// b_coarse = P^T r_fine: each coarse vertex gathers its 3^d fine neighbours with the (bi/tri)linear
// weights prod_a (1 - |d_a| / 2) (deterministic, no atomics)
__global__ void k_gmg_restrict(double* __restrict__ bc, const double* __restrict__ rf, GmgBox C, GmgBox F, int dim,
                               int64_t nc) {
  FCM_PDL_ENTRY();
  for (int64_t J = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; J < nc; J += (int64_t)gridDim.x * blockDim.x) {
    int c, X[3];
    gmg_decode(C, J, c, X);
    double s = 0.0;
    const int dz0 = dim == 3 ? -1 : 0, dz1 = dim == 3 ? 1 : 0;
    for (int dz = dz0; dz <= dz1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int x[3] = {2 * X[0] + dx, 2 * X[1] + dy, 2 * X[2] + dz};
          if (!gmg_in(F, c, x)) continue;
          const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
          s = fma(w, rf[gmg_index(F, c, x)], s);
        }
    bc[J] = s;
  }
}
// x_fine += P e_coarse: each fine vertex gathers its 1, 2, 4 or 8 coarse parents
__global__ void k_gmg_prolong(double* __restrict__ xf, const double* __restrict__ ec, GmgBox F, GmgBox C, int dim,
                              int64_t nfine) {
  FCM_PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfine; i += (int64_t)gridDim.x * blockDim.x) {
    int c, x[3];
    gmg_decode(F, i, c, x);
    double s = 0.0;
    const int nz = (dim == 3 && (x[2] & 1)) ? 2 : 1, ny = (x[1] & 1) ? 2 : 1, nx = (x[0] & 1) ? 2 : 1;
    for (int kz = 0; kz < nz; ++kz)
      for (int ky = 0; ky < ny; ++ky)
        for (int kx = 0; kx < nx; ++kx) {
          const int X[3] = {(x[0] - (nx - 1)) / 2 + kx, (x[1] - (ny - 1)) / 2 + ky, (x[2] - (nz - 1)) / 2 + kz};
          if (!gmg_in(C, c, X)) continue;
          s = fma((nx == 2 ? 0.5 : 1.0) * (ny == 2 ? 0.5 : 1.0) * (nz == 2 ? 0.5 : 1.0), ec[gmg_index(C, c, X)], s);
        }
    xf[i] += s;
  }
}
// distributed h-coarsening (slab mode): partial restriction of this slab's OWNED fine vertices
// (local slab-axis index >= own_lo) into the global coarse layers [cz0, cz1); the caller zeroes
// the global vector first and all-reduces it after (sum over slabs = P^T r of the whole grid)
__global__ void k_gmg_restrict_dist(double* __restrict__ bc, const double* __restrict__ rf, GmgBox C, GmgBox F,
                                    int dim, int zoff, int own_lo, int cz0, int cz1) {
  const int ax = dim - 1;
  for (int c = 0; c < C.nf; ++c) {
    int64_t plane = 1;
    for (int a = 0; a < ax; ++a) plane *= C.size[c][a];
    const int z0 = max(cz0, C.lo[c][ax]), z1 = min(cz1, C.lo[c][ax] + C.size[c][ax]);
    const int64_t n = z0 < z1 ? plane * (z1 - z0) : 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
      int X[3] = {0, 0, 0};
      int64_t u = t;
      for (int a = 0; a < ax; ++a) { X[a] = (int)(u % C.size[c][a]) + C.lo[c][a]; u /= C.size[c][a]; }
      X[ax] = z0 + (int)u;
      double s = 0.0;
      const int dz0 = dim == 3 ? -1 : 0, dz1 = dim == 3 ? 1 : 0;
      for (int dz = dz0; dz <= dz1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            int x[3] = {2 * X[0] + dx, 2 * X[1] + dy, dim == 3 ? 2 * X[2] + dz : 0};
            x[ax] -= zoff;   // global -> local slab index
            if (x[ax] < own_lo || !gmg_in(F, c, x)) continue;
            const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
            s = fma(w, rf[gmg_index(F, c, x)], s);
          }
      bc[gmg_index(C, c, X)] = s;
    }
  }
}
// x_local += P e_coarse (replicated e): every local fine vertex, interface planes included
__global__ void k_gmg_prolong_dist(double* __restrict__ xf, const double* __restrict__ ec, GmgBox F, GmgBox C,
                                   int dim, int zoff, int64_t nfine) {
  const int ax = dim - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nfine; i += (int64_t)gridDim.x * blockDim.x) {
    int c, x[3];
    gmg_decode(F, i, c, x);
    x[ax] += zoff;   // local -> global
    double s = 0.0;
    const int nz = (dim == 3 && (x[2] & 1)) ? 2 : 1, ny = (x[1] & 1) ? 2 : 1, nx = (x[0] & 1) ? 2 : 1;
    for (int kz = 0; kz < nz; ++kz)
      for (int ky = 0; ky < ny; ++ky)
        for (int kx = 0; kx < nx; ++kx) {
          const int X[3] = {(x[0] - (nx - 1)) / 2 + kx, (x[1] - (ny - 1)) / 2 + ky, (x[2] - (nz - 1)) / 2 + kz};
          if (!gmg_in(C, c, X)) continue;
          s = fma((nx == 2 ? 0.5 : 1.0) * (ny == 2 ? 0.5 : 1.0) * (nz == 2 ? 0.5 : 1.0), ec[gmg_index(C, c, X)], s);
        }
    xf[i] += s;
  }
}
// distributed coarse CG updates from all-reduced scalars d[]: {rz, pq, rr, rz_new, rr0}
__global__ void k_dcg_update(const double* __restrict__ d, double* __restrict__ x, double* __restrict__ r,
                             const double* __restrict__ p, const double* __restrict__ q, int64_t n) {
  const double a = d[0] / d[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    r[i] = fma(-a, q[i], r[i]);
  }
}
__global__ void k_dcg_update2(double* __restrict__ d, double* __restrict__ p, const double* __restrict__ z, int64_t n) {
  const double beta = d[3] / d[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}
__global__ void k_dcg_setrz(double* d) {
  if (threadIdx.x == 0) d[0] = d[3];
}

// coarse CG (standard PCG, P:343 form) around the geometric V-cycle; the loop is a device-side
// WHILE node, the V-cycle + beta part an IF node inside it (both set by k_gcg_check)
__global__ void k_gcg_init(GcgScalars* s, const double* pA, const double* pB, int np, double* p, const double* z,
                           int64_t n, cudaGraphConditionalHandle cw) {
  const double rz = sum_partials(pA, np), rr = sum_partials(pB, np);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->rz = rz; s->rr0 = rr; s->rr = rr; s->it = 0; s->flag = 0;
    cudaGraphSetConditional(cw, (rr > 0.0 && s->maxit > 0) ? 1u : 0u);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = z[i];
}
__global__ void k_gcg_update(GcgScalars* s, const double* ppq, int npq, double* __restrict__ x, double* __restrict__ r,
                             const double* __restrict__ p, const double* __restrict__ q, int64_t n, double* prr) {
  FCM_PDL_ENTRY();
  __shared__ double red[32];
  const double pq = sum_partials(ppq, npq);
  const double a = s->rz / pq;
  double rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    const double rn = fma(-a, q[i], r[i]);
    r[i] = rn;
    rr = fma(rn, rn, rr);
  }
  rr = block_sum(rr, red);
  if (threadIdx.x == 0) prr[blockIdx.x] = rr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s->pq = pq;
    if (!(pq > 0.0)) s->flag = 1;
  }
}
__global__ void k_gcg_check(GcgScalars* s, const double* prr, int np, cudaGraphConditionalHandle cw,
                            cudaGraphConditionalHandle ci, int* iters) {
  FCM_PDL_ENTRY();
  const double rr = sum_partials(prr, np);
  if (threadIdx.x == 0) {
    s->rr = rr;
    const int it = ++s->it;
    const bool stop = s->flag || !(rr == rr) || rr < s->rtol2 * s->rr0 || it >= s->maxit;
    cudaGraphSetConditional(cw, stop ? 0u : 1u);
    cudaGraphSetConditional(ci, stop ? 0u : 1u);
    if (stop) { iters[0] = it; iters[1] += it; }
  }
}
__global__ void k_gcg_update2(GcgScalars* s, const double* prz, int np, double* __restrict__ p,
                              const double* __restrict__ z, int64_t n) {
  FCM_PDL_ENTRY();
  const double rzn = sum_partials(prz, np);
  const double beta = rzn / s->rz;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) s->rz_new = rzn;
}
__global__ void k_gcg_setrz(GcgScalars* s) {
  FCM_PDL_ENTRY();
  if (threadIdx.x == 0) s->rz = s->rz_new;
}

// Inversion of SPD blocks: Cholesky A = L L^T (right-looking, L in shared memory), then
// X = A^{-1} column by column by forward/backward substitution (one thread per column,
// the column lives in the output block), symmetrised.  Backward stable.
// status[blk] = 1 if a pivot was not positive/finite (not SPD / singular).
__device__ void chol_inverse(double* L, double* X, int64_t m, int* bad) {
  // L: m*m working matrix (lower triangle used), X: output m*m (global)
  for (int64_t k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      const double d = L[k * m + k];
      if (!(d > 0.0 && isfinite(d))) *bad = 1;
      L[k * m + k] = sqrt(fmax(d, 1e-300));
    }
    __syncthreads();
    const double dk = L[k * m + k];
    for (int64_t i = k + 1 + threadIdx.x; i < m; i += blockDim.x) L[i * m + k] /= dk;
    __syncthreads();
    const int64_t r = m - k - 1;  // trailing lower triangle update
    for (int64_t e = threadIdx.x; e < r * r; e += blockDim.x) {
      const int64_t i = k + 1 + e / r, j = k + 1 + e % r;
      if (j <= i) L[i * m + j] -= L[i * m + k] * L[j * m + k];
    }
    __syncthreads();
  }
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    // forward: L y = e_j  (y_i = 0 for i < j)
    for (int64_t i = 0; i < j; ++i) X[i * m + j] = 0.0;
    for (int64_t i = j; i < m; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int64_t k = j; k < i; ++k) s -= L[i * m + k] * X[k * m + j];
      X[i * m + j] = s / L[i * m + i];
    }
    // backward: L^T x = y
    for (int64_t i = m - 1; i >= 0; --i) {
      double s = X[i * m + j];
      for (int64_t k = i + 1; k < m; ++k) s -= L[k * m + i] * X[k * m + j];
      X[i * m + j] = s / L[i * m + i];
    }
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int64_t i = e / m, j = e % m;
    if (i < j) {
      const double s = 0.5 * (X[i * m + j] + X[j * m + i]);
      X[i * m + j] = s;
      X[j * m + i] = s;
    }
  }
  __syncthreads();
}

__global__ void k_invert_blocks(double* mats, int m, int* status, int64_t nblocks) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* A = reinterpret_cast<double*>(smem);
  __shared__ int bad;
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    double* G = mats + blk * (int64_t)m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) A[e] = G[e];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    chol_inverse(A, G, m, &bad);
    if (threadIdx.x == 0) status[blk] = bad;
    __syncthreads();
  }
}

// same for blocks too large for shared memory (patch blocks, m_b up to 729): the Cholesky
// factor lives in a per-CTA global scratch (L2-resident)
__global__ void k_invert_blocks_global(double* mats, int m, int* status, int64_t nblocks, double* scratch) {
  __shared__ int bad;
  double* A = scratch + (size_t)blockIdx.x * m * m;
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    double* G = mats + blk * (int64_t)m * m;
    for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += blockDim.x) A[e] = G[e];
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    chol_inverse(A, G, m, &bad);
    if (threadIdx.x == 0) status[blk] = bad;
    __syncthreads();
  }
}

// dense inverse of the SPD coarse matrix (direct coarse solve): A is overwritten by its
// Cholesky factor, X receives A^{-1}.
__global__ void k_invert_dense(double* A, int64_t n, double* X, int* status) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  chol_inverse(A, X, n, &bad);
  if (threadIdx.x == 0) *status = bad;
}

// ---- compile-time M dispatch --------------------------------------------------------------
template <int M> constexpr int gsz() { return M <= 4 ? 4 : (M <= 8 ? 8 : (M <= 16 ? 16 : 32)); }
#define FCM_FOR_M(X) X(4) X(8) X(9) X(16) X(24) X(25) X(27)

const void* reg_kernel(int m, int* M_out) {
#define CASE(MM) case MM: *M_out = MM; return (const void*)k_cell_reg<MM, split_of<MM>()>;
  switch (m) { FCM_FOR_M(CASE) default: break; }
#undef CASE
  *M_out = 0;
  return nullptr;
}
const void* mma_kernel(int m) {
#define CASE(MM) case MM: return (const void*)k_cell_mma<MM, gsz<MM>()>;
  // 64 / 125: tensor p = 3 / 4 (configs 5 / 3); 60 / 96: trunk elasticity p = 2 / 3 (config 4)
  switch (m) { FCM_FOR_M(CASE) CASE(60) CASE(64) CASE(96) CASE(125) default: break; }
#undef CASE
  return nullptr;
}
// warp-specialised cell kernel (cellws.cuh) for the elementwise levels that carry most bytes:
// m = 27 / 64 / 125 (tensor p = 2 / 3 / 4); *ns = its streaming warps, *smem its dynamic smem
// variant (FCM_WS_VARIANT, measurement): 0 = 8 streaming warps x 2 stages + 8 MMA warps with
// the gather prefetch; 1 = the same without the prefetch; 2 = 4 streaming warps x 4 stages + 12
// MMA warps (prefetch); 3 = 2 without the prefetch
const void* ws_kernel(int m, int variant, int* nthreads, size_t* smem) {
#define WS(MM, NS, NM, STG, PF) \
  { *nthreads = (NS + NM) * 32; *smem = ws_smem<MM, NS, NM, STG>(); return (const void*)k_cell_ws<MM, NS, NM, STG, PF>; }
#define WSV(MM) \
  case MM: \
    switch (variant) { \
      case 1: WS(MM, 8, 8, 2, false) \
      case 2: WS(MM, 4, 12, 4, true) \
      case 3: WS(MM, 4, 12, 4, false) \
      default: WS(MM, 8, 8, 2, true) \
    }
  switch (m) {
    WSV(27)
    WSV(60)
    WSV(64)
    case 96: WS(96, 4, 8, 2, false)
    case 125: WS(125, 4, 8, 2, false)
    default: break;
  }
#undef WSV
#undef WS
  return nullptr;
}
const void* list_kernel(int G) {
  switch (G) {
    case 4: return (const void*)k_cell_list<4>;
    case 8: return (const void*)k_cell_list<8>;
    case 16: return (const void*)k_cell_list<16>;
    default: return (const void*)k_cell_list<32>;
  }
}
// coarse_group(): lanes per individual cell in the grid-wide coarse kernel.  Large coarse
// levels (config 4: 75k individual 24x24 blocks per phase) are latency-bound on the list, so
// m > 8 uses 8 lanes per cell (4 cells per warp in flight) instead of a whole warp.
constexpr int coarse_group(int m) { return m <= 4 ? 4 : 8; }
const void* coarse_kernel(int m, int G, int* M_out) {
#define CASE(MM) case MM: *M_out = MM; return (const void*)k_coarse_pcg<MM, coarse_group(MM)>;
  switch (m) { FCM_FOR_M(CASE) default: break; }
#undef CASE
  *M_out = 0;
  switch (G) {
    case 4: return (const void*)k_coarse_pcg<0, 4>;
    case 8: return (const void*)k_coarse_pcg<0, 8>;
    case 16: return (const void*)k_coarse_pcg<0, 16>;
    default: return (const void*)k_coarse_pcg<0, 32>;
  }
}
const void* tiled_kernel(int dim, int nf) {
  if (dim == 3 && nf == 1) return (const void*)k_coarse_tiled<3, 1>;
  if (dim == 3 && nf == 3) return (const void*)k_coarse_tiled<3, 3>;
  if (dim == 2 && nf == 1) return (const void*)k_coarse_tiled<2, 1>;
  return nullptr;
}

inline int grid_for(int64_t n, int sms) {
  int64_t b = (n + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)sms * 4));
}

}  // namespace

// =========================================================================================
// host helpers
// =========================================================================================
// Shared-memory opt-in of a kernel function: the attribute is per FUNCTION (shared by every
// handle and level in the process), so it is raised to the device maximum once instead of to
// the size one caller needs (a later, smaller setting would break an earlier handle).
static int allow_smem(const void* func, size_t need) {
  int dev = 0, mx = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  CU(cudaFuncGetAttributes(&fa, func));
  const int dyn_max = mx - (int)fa.sharedSizeBytes;   // static shared memory counts against the opt-in
  if (need > (size_t)dyn_max) return fail(FCM_EINVAL, "kernel needs %zu B of dynamic shared memory (max %d)", need, dyn_max);
  CU(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
  return FCM_OK;
}
static int gsz_rt(int M) { return M <= 4 ? 4 : (M <= 8 ? 8 : (M <= 16 ? 16 : 32)); }  // = gsz<M>()
static int group_size(int m) {
  if (m <= 4) return 4;
  if (m <= 8) return 8;
  if (m <= 16) return 16;
  return 32;
}

static int split_rt(int M) { return M <= 4 ? 1 : (M <= 9 ? 2 : (M <= 16 ? 4 : 8)); }  // = split_of<M>()
static size_t reg_scratch_rt(int M, int TS) { return (size_t)(32 / TS) * (M + (M & 1)); }
static size_t reg_smem(int M, int TS) {
  return sizeof(Tab) + ((size_t)M * (M + (M & 1)) + (kThreads / 32) * reg_scratch_rt(M, TS)) * sizeof(double);
}
static size_t mma_smem(int M) {
  return sizeof(Tab) + (size_t)((M + 7) / 8) * ((M + 3) / 4) * 32 * sizeof(double);
}
static size_t level_reg_smem(const LevelDev& Lv) { return reg_smem(Lv.M, Lv.ts); }
static size_t list_smem(int m, int G) {
  return sizeof(Tab) + (size_t)(kThreads / 32) * (32 / G) * m * (sizeof(double) + sizeof(int));
}
// coarse: [Tab][MsA][MsM][reg scratch][list scratch]
static size_t coarse_smem(int m, int M, int G) {
  const int TS = M > 0 ? split_rt(M) : 1;
  const size_t frag = (M > 0 && M <= 32) ? (size_t)2 * ((M + 7) / 8) * ((M + 3) / 4) * 32 * 8 + 8 : 0;
  return reg_smem(M, TS) + (size_t)M * (M + (M & 1)) * 8 + list_smem(m, G) - sizeof(Tab) + frag;
}

static CellOp make_op(fcm_mg* h, int q, int mode, const double* in, double* out, double coef,
                      double* partials) {
  LevelDev& Lv = h->lev[q];
  CellOp op{};
  op.colour = -1;
  op.nx = h->L.n[0]; op.ny = h->L.n[1]; op.nz = h->L.n[2];
  op.m = Lv.m;
  op.ncell = (int32_t)h->ncell;
  op.base = Lv.base; op.stride = Lv.stride; op.cmin = Lv.cmin; op.cmax = Lv.cmax;
  for (int i = 0; i < 3; ++i) { op.ilo[i] = Lv.ilo[i]; op.ihi[i] = Lv.ihi[i]; }
  op.mode = mode;
  op.kind = h->d_kind; op.cut_idx = h->d_cut_idx; op.Kref = h->d_Kref; op.cutK = h->d_cutK;
  op.ldK = h->L.m; op.alpha = h->alpha;
  op.blk = Lv.blk; op.irr_inv = Lv.irr_inv; op.type_inv = Lv.type_inv; op.inv_alpha = 1.0 / h->alpha;
  const bool mma = Lv.kmma && (mode == OP_APPLY ? Lv.gA_cells != nullptr : Lv.gS_cells != nullptr);
  if (Lv.M > 0 || mma) {   // the regular population has its own kernel: list = individual cells
    if (mode == OP_APPLY) {
      op.list = h->d_cut_list; op.nlist = (int32_t)h->ncut;
      op.list_mats = h->d_cutK + (size_t)h->cut_first * h->L.m * h->L.m; op.list_ld = h->L.m;
    } else {
      op.list = Lv.irr_list; op.nlist = (int32_t)Lv.n_irr; op.list_mats = Lv.irr_inv; op.list_ld = Lv.m;
    }
  }
  op.in = in; op.out = out; op.coef = coef; op.partials = partials;
  return op;
}

// the level's cell operation runs as one warp-specialised launch (cellws.cuh)
static bool ws_on(const LevelDev& Lv, int mode) {
  return Lv.kws && (mode == OP_APPLY || (!Lv.patch && Lv.has_as && (Lv.irr_tp || Lv.n_irr == 0)));
}
// grid of one cell-operator launch: regular thread-per-cell blocks + individual-list blocks
static void cellop_grid(const fcm_mg* h, int q, int mode, int* nb_reg, int* nb_list) {
  const LevelDev& Lv = h->lev[q];
  if (ws_on(Lv, mode)) {   // persistent: one CTA per SM
    *nb_reg = h->ws_ctas;
    *nb_list = 0;
    return;
  }
  const int64_t cap = (int64_t)h->num_sms * 8;
  const int64_t cpb = (kThreads / 32) * (32 / Lv.G);  // cells per block on the list path
  const bool mma = Lv.kmma && (mode == OP_APPLY ? Lv.gA_cells != nullptr : Lv.gS_cells != nullptr);
  if (mma) {
    // MMA blocks: h->mma_bps per SM (staging of the A fragments amortised over the groups a
    // warp loops over); list blocks: up to list_bps per SM
    const int64_t ng = mode == OP_APPLY ? Lv.nA : Lv.nS;
    *nb_reg = (int)std::max<int64_t>(1, std::min<int64_t>((ng + kThreads / 32 - 1) / (kThreads / 32),
                                                          (int64_t)h->num_sms * h->mma_bps));
    const int64_t nl = mode == OP_APPLY ? h->ncut : Lv.n_irr;
    *nb_list = (int)std::min<int64_t>((nl + cpb - 1) / cpb, (int64_t)h->num_sms * h->list_bps);
    return;
  }
  if (Lv.M > 0) {
    const int64_t ts = Lv.ts;
    const int64_t cells_per_blk = (kThreads / 32) * (32 / ts);
    *nb_reg = (int)std::min<int64_t>((h->ncell + cells_per_blk - 1) / cells_per_blk, cap);
    const int64_t nl = mode == OP_APPLY ? h->ncut : Lv.n_irr;
    *nb_list = (int)std::min<int64_t>((nl + cpb - 1) / cpb, cap);
  } else {
    *nb_reg = 0;
    *nb_list = (int)std::max<int64_t>(1, std::min<int64_t>((h->ncell + cpb - 1) / cpb, cap));
  }
}
static int dot_blocks(fcm_mg* h);
static int cellop_nblocks(const fcm_mg* h, int q, int mode) {
  if (h->det) return dot_blocks(const_cast<fcm_mg*>(h));   // energies by a block-order dot
  int a, b;
  cellop_grid(h, q, mode, &a, &b);
  return a + b;
}

// One cell-operator application = regular kernel + individual-list kernel; the list kernel
// runs on a forked branch (graph fork/join when captured) so both populations overlap.
static int copy(fcm_mg* h, double* y, const double* x, int64_t n);
static int launch_cellop_1(fcm_mg* h, int q, const CellOp& op, double* cp_dst, const double* cp_src, int64_t cp_n);
static int launch_cellop(fcm_mg* h, int q, const CellOp& op, double* cp_dst = nullptr,
                         const double* cp_src = nullptr, int64_t cp_n = 0) {
  if (!h->det) return launch_cellop_1(h, q, op, cp_dst, cp_src, cp_n);
  // deterministic mode: one launch per cell parity colour, then the energy as a block-order dot
  if (cp_dst) RC(copy(h, cp_dst, cp_src, cp_n));
  CellOp o = op;
  o.partials = nullptr;
  for (int k = 0; k < (1 << h->L.dim); ++k) {
    o.colour = k;
    RC(launch_cellop_1(h, q, o, nullptr, nullptr, 0));
  }
  if (op.partials) {
    k_dot<<<dot_blocks(h), kThreads, 0, h->stream>>>(op.in, op.out, h->lev[q].ndof, op.partials, nullptr);
    h->count();
    CU(cudaGetLastError());
  }
  return FCM_OK;
}
static int launch_cellop_1(fcm_mg* h, int q, const CellOp& op, double* cp_dst, const double* cp_src, int64_t cp_n) {
  const LevelDev& Lv = h->lev[q];
  int nb_reg, nb_list;
  cellop_grid(h, q, op.mode, &nb_reg, &nb_list);
  CellOp o = op;
  if (ws_on(Lv, op.mode)) {
    MmaOp g{};
    g.op = o;
    TileListOp tl{};
    tl.ntq = Lv.ntq;
    if (op.mode == OP_APPLY) {
      g.grp_cells = Lv.gA_cells; g.grp_mat = Lv.gA_mat; g.ngroups = Lv.nA;
      tl.list = h->d_cut_list; tl.nlist = (int32_t)h->ncut;
      tl.mats = h->d_cutK_tp + (size_t)h->cut_first * h->cut_tps; tl.stride = h->cut_tps;
    } else {
      g.grp_cells = Lv.gS_cells; g.grp_mat = Lv.gS_mat; g.ngroups = Lv.nS;
      tl.list = Lv.irr_list; tl.nlist = (int32_t)Lv.n_irr; tl.mats = Lv.irr_tp; tl.stride = Lv.irr_tps;
    }
    g.cp_src = cp_src; g.cp_dst = cp_dst; g.cp_n = cp_dst ? cp_n : 0;
    const char* wp = getenv("FCM_WS_PART");   // measurement hook, read per launch
    const int part = wp ? atoi(wp) : 0;
    if (part == 1) g.ngroups = 0;
    if (part == 2) tl.nlist = 0;
    void* args[] = {&g, &tl};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(h->ws_ctas);
    cfg.blockDim = dim3(Lv.ws_threads[op.mode]);
    cfg.dynamicSmemBytes = Lv.ws_smem_b[op.mode];
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = h->pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&cfg, Lv.kws_m[op.mode], args);
    h->count();
    if (e != cudaSuccess) return fail(FCM_ECUDA, "ws kernel launch: %s", cudaGetErrorString(e));
    return FCM_OK;
  }
  if (Lv.kmma && (op.mode == OP_APPLY ? Lv.gA_cells != nullptr : Lv.gS_cells != nullptr)) {
    // one launch: regular cells as fp64 MMA groups, the individual list in the other blocks
    MmaOp g{};
    g.op = o;
    if (op.mode == OP_APPLY) { g.grp_cells = Lv.gA_cells; g.grp_mat = Lv.gA_mat; g.ngroups = Lv.nA; }
    else { g.grp_cells = Lv.gS_cells; g.grp_mat = Lv.gS_mat; g.ngroups = Lv.nS; }
    g.cp_src = cp_src; g.cp_dst = cp_dst; g.cp_n = cp_dst ? cp_n : 0;
    int nbm = nb_reg;
    void* args[] = {&g, &nbm};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nb_reg + nb_list);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = std::max(mma_smem(Lv.m), list_smem(Lv.m, Lv.G));
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = h->pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&cfg, Lv.kmma, args);
    h->count();
    if (e != cudaSuccess) return fail(FCM_ECUDA, "mma kernel launch: %s", cudaGetErrorString(e));
    return FCM_OK;
  }
  if (cp_dst) RC(copy(h, cp_dst, cp_src, cp_n));   // other paths: the copy as its own launch
  int off = nb_reg;
  cudaError_t e = cudaSuccess;
  const bool fork = nb_reg > 0 && nb_list > 0;
  if (fork) {
    CU(cudaEventRecord(h->ev_fork, h->stream));
    CU(cudaStreamWaitEvent(h->stream2, h->ev_fork, 0));
  }
  if (nb_list > 0) {
    void* args[] = {&o, &off};
    e = cudaLaunchKernel(Lv.klist, dim3(nb_list), dim3(kThreads), args, list_smem(Lv.m, Lv.G),
                         fork ? h->stream2 : h->stream);
    h->count();
    if (e != cudaSuccess) return fail(FCM_ECUDA, "list kernel launch: %s", cudaGetErrorString(e));
  }
  if (nb_reg > 0) {
    void* args[] = {&o};
    e = cudaLaunchKernel(Lv.kreg, dim3(nb_reg), dim3(kThreads), args, level_reg_smem(Lv), h->stream);
    h->count();
    if (e != cudaSuccess) return fail(FCM_ECUDA, "regular kernel launch: %s", cudaGetErrorString(e));
  }
  if (fork) {
    CU(cudaEventRecord(h->ev_join, h->stream2));
    CU(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
  }
  return FCM_OK;
}

// launch with the programmatic-stream-serialization attribute (kernels that begin with
// FCM_PDL_ENTRY), so a launch's scheduling overlaps the tail of the previous one
template <typename... KArgs, typename... Args>
static cudaError_t pdl_launch(fcm_mg* h, void (*k)(KArgs...), dim3 grid, dim3 block, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = h->pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
static int fill(fcm_mg* h, double* x, double v, int64_t n) {
  if (n <= 0) return FCM_OK;
  CU(pdl_launch(h, k_fill, dim3(grid_for(n, h->num_sms)), dim3(kThreads), x, v, n));
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}
static int copy(fcm_mg* h, double* y, const double* x, int64_t n) {
  if (n <= 0) return FCM_OK;
  k_copy<<<grid_for(n, h->num_sms), kThreads, 0, h->stream>>>(y, x, n);
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}

#define NC(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) return fail(FCM_ENCCL, "%s: %s", #call, nccl().GetErrorString(r_)); \
  } while (0)

// slab mode: sum the two copies of every interface plane of level q: pack the
// bottom / top planes, grouped send/recv with the neighbours, add what came back.
static int exchange(fcm_mg* h, int q, double* v) {
  if (!h->multi) return FCM_OK;
  LevelDev& Lv = h->lev[q];
  const int64_t nlo = Lv.n_lo, nhi = Lv.n_hi, stride = h->lev[h->g.p].n_lo + h->lev[h->g.p].n_hi;
  if (nlo + nhi == 0) return FCM_OK;
  const int gb = grid_for(nlo + nhi, h->num_sms);
  k_pack2<<<gb, kThreads, 0, h->stream>>>(h->x_send, v, Lv.lo_idx, nlo, Lv.hi_idx, nhi, stride);
  h->count();
  CU(cudaGetLastError());
  NC(nccl().GroupStart());
  if (nlo > 0) {   // bottom plane <-> rank - 1 (its top plane)
    NC(nccl().Send(h->x_send, nlo, ncclFloat64, h->rank - 1, h->comm, h->stream));
    NC(nccl().Recv(h->x_recv, nlo, ncclFloat64, h->rank - 1, h->comm, h->stream));
  }
  if (nhi > 0) {   // top plane <-> rank + 1 (its bottom plane)
    NC(nccl().Send(h->x_send + stride, nhi, ncclFloat64, h->rank + 1, h->comm, h->stream));
    NC(nccl().Recv(h->x_recv + stride, nhi, ncclFloat64, h->rank + 1, h->comm, h->stream));
  }
  NC(nccl().GroupEnd());
  k_unpack_add2<<<gb, kThreads, 0, h->stream>>>(v, h->x_recv, Lv.lo_idx, nlo, Lv.hi_idx, nhi, stride);
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}

// all-reduce (sum) of n device doubles in place (slab mode)
static int allreduce(fcm_mg* h, double* v, int n) {
  if (!h->multi) return FCM_OK;
  NC(nccl().AllReduce(v, v, n, ncclFloat64, ncclSum, h->comm, h->stream));
  return FCM_OK;
}

// r = b - A_q x.  Slab mode: the lower rank owns an interface DOF, so only it starts from b
// there; the exchange then adds the two partial sums of A x (same result on both ranks).
static int residual(fcm_mg* h, int q, const double* b, const double* x, double* r, bool r_is_b = false) {
  LevelDev& Lv = h->lev[q];
  if (!r_is_b) RC(copy(h, r, b, Lv.ndof));
  if (Lv.n_lo > 0) {
    k_zero_idx<<<grid_for(Lv.n_lo, h->num_sms), kThreads, 0, h->stream>>>(r, Lv.lo_idx, Lv.n_lo);
    h->count();
  }
  RC(launch_cellop(h, q, make_op(h, q, OP_APPLY, x, r, -1.0, nullptr)));
  return exchange(h, q, r);
}
// y = A_q x (y overwritten)
static int apply_op(fcm_mg* h, int q, const double* x, double* y, double* partials) {
  RC(fill(h, y, 0.0, h->lev[q].ndof));
  RC(launch_cellop(h, q, make_op(h, q, OP_APPLY, x, y, 1.0, partials)));
  return exchange(h, q, y);
}
static size_t block_smem(int m, int mb) {
  (void)m;
  return sizeof(Tab) + (size_t)(kThreads / 32) * mb * (sizeof(double) + sizeof(int));
}
// patchwise smoother (patch.cuh): the individual (irregular) patches stream their tile-packed
// inverses (k_patch_irr, forked onto the second stream) while the regular patches run by fast
// diagonalisation (k_patch_fd) or, off the tensor-Poisson case, the dense shared-type kernel
static size_t patch_smem(const fcm_mg* h, int q);
// streaming warps per patch: about 8+ tiles per warp (level 4: 276 tiles -> 8 warps on one patch;
// level 3: 66 tiles -> 4; level 2: 10 tiles -> 1 warp per patch, 8 patches in flight per CTA)
static int patch_wpp(int nt) {
  const int ntiles = nt * (nt + 1) / 2;
  int w = 1;
  while (w < kIrrWarps && ntiles / (2 * w) > 8) w *= 2;
  return w;
}
template <int S, int DIM>
static const void* patch_kernel_s(int irr, int fd) {
  if (irr && fd) return (const void*)k_patch_smooth<S, DIM, true, true>;
  if (irr) return (const void*)k_patch_smooth<S, DIM, true, false>;
  return (const void*)k_patch_smooth<S, DIM, false, true>;
}
static const void* patch_kernel(int S, int dim, int irr, int fd) {
  if (dim == 3) return S == 3 ? patch_kernel_s<3, 3>(irr, fd) : S == 5 ? patch_kernel_s<5, 3>(irr, fd)
                     : S == 7 ? patch_kernel_s<7, 3>(irr, fd) : patch_kernel_s<9, 3>(irr, fd);
  return S == 3 ? patch_kernel_s<3, 2>(irr, fd) : S == 5 ? patch_kernel_s<5, 2>(irr, fd)
         : S == 7 ? patch_kernel_s<7, 2>(irr, fd) : patch_kernel_s<9, 2>(irr, fd);
}
static const void* wb_kernel(int S, int dim) {
  if (dim == 3) return S == 3 ? (const void*)k_patch_wb<3, 3> : S == 5 ? (const void*)k_patch_wb<5, 3>
                     : S == 7 ? (const void*)k_patch_wb<7, 3> : (const void*)k_patch_wb<9, 3>;
  return S == 3 ? (const void*)k_patch_wb<3, 2> : S == 5 ? (const void*)k_patch_wb<5, 2>
         : S == 7 ? (const void*)k_patch_wb<7, 2> : (const void*)k_patch_wb<9, 2>;
}
static int wb_threads_rt(int S, int dim) {
  if (dim == 3) return S == 3 ? wb_threads<3, 3>() : S == 5 ? wb_threads<5, 3>() : S == 7 ? wb_threads<7, 3>() : wb_threads<9, 3>();
  return S == 3 ? wb_threads<3, 2>() : S == 5 ? wb_threads<5, 2>() : S == 7 ? wb_threads<7, 2>() : wb_threads<9, 2>();
}
static size_t wb_smem_rt(int S, int dim, int mb) {
  if (dim == 3) return S == 3 ? wb_smem<3, 3>(mb) : S == 5 ? wb_smem<5, 3>(mb) : S == 7 ? wb_smem<7, 3>(mb) : wb_smem<9, 3>(mb);
  return S == 3 ? wb_smem<3, 2>(mb) : S == 5 ? wb_smem<5, 2>(mb) : S == 7 ? wb_smem<7, 2>(mb) : wb_smem<9, 2>(mb);
}

// patchwise smoother (patch.cuh): ONE warp-specialised launch (k_patch_smooth) streams the
// individual patches' tile-packed inverses and applies the regular patches by fast
// diagonalisation on the same SMs; off the tensor-Poisson case the regular patches use the
// dense shared-type kernel (k_block_smooth) after the streaming launch.
// the low-rank patches belong to the individual population (smoother part 1, and part 0)
static bool do_irr_wb(const fcm_mg* h, int q, int part) { return part != 2 && h->lev[q].n_wb > 0; }
static int launch_block_smooth(fcm_mg* h, int q, const double* r, double* x, double coef, int part = 0) {
  LevelDev& Lv = h->lev[q];
  const bool do_irr = part != 2 && Lv.n_irr > 0, do_reg = part != 1 && Lv.n_reg > 0;
  const bool fd = do_reg && Lv.fd;
  PatchIrrOp io{};
  io.nx = h->L.n[0]; io.ny = h->L.n[1]; io.nz = h->L.n[2];
  for (int i = 0; i < 3; ++i) io.na[i] = Lv.na[i];
  io.mb = Lv.mb; io.nt = Lv.nt; io.stride = Lv.pstride; io.n_irr = do_irr ? Lv.n_irr : 0;
  io.wpp = patch_wpp(Lv.nt);
  io.anchors = Lv.irr_anchor; io.mem = Lv.d_mem; io.loc = Lv.d_loc;
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 3; ++i) io.mo[k][i] = Lv.mo[k][i];
  io.base = Lv.base; io.stride3 = Lv.stride; io.cmin = Lv.cmin; io.cmax = Lv.cmax; io.m = Lv.m;
  io.inv = Lv.irr_inv; io.in = r; io.out = x; io.coef = coef;
  // dynamic patch claiming needs every streaming warp to own >= kIrrStages tiles per patch (its
  // ring runs at most one patch ahead of the claims)
  io.sched = Lv.sched && (Lv.nt * (Lv.nt + 1) / 2) / io.wpp >= kIrrStages ? Lv.sched : nullptr;
  PatchFdOp fo{};
  fo.nx = h->L.n[0]; fo.ny = h->L.n[1]; fo.nz = h->L.n[2]; fo.dim = h->L.dim;
  for (int i = 0; i < 3; ++i) fo.na[i] = Lv.na[i];
  fo.q = q; fo.S = 2 * q + 1; fo.nreg = fd ? Lv.n_reg : 0; fo.anchors = Lv.reg_list; fo.blk = Lv.blk;
  fo.cls = Lv.fd_cls; fo.tabs = Lv.fd_tabs; fo.ncls = Lv.fd ? Lv.fd_ncls : 0; fo.s_fac = Lv.fd_s;
  fo.inv_alpha = 1.0 / h->alpha; fo.modeidx = Lv.fd_midx;
  fo.base = Lv.base; fo.stride3 = Lv.stride; fo.cmin = Lv.cmin; fo.cmax = Lv.cmax; fo.m = Lv.m;
  fo.in = r; fo.out = x; fo.coef = coef;
  fo.sched = io.sched;
  fo.roll = Lv.fd_roll ? 1 : 0;
  // low-rank individual patches: by the fast-diagonalisation warps of the same launch (they finish
  // the regular patches long before the streaming warps; FCM_WB_KERNEL=1: separate k_patch_wb)
  const bool wb_fused = do_irr_wb(h, q, part) && Lv.wb_fused;
  fo.n_wb = wb_fused ? Lv.n_wb : 0;
  fo.wb_anchor = Lv.wb_anchor; fo.wb_soff = Lv.wb_soff; fo.wb_tS = Lv.wb_tS; fo.wb_coff = Lv.wb_coff; fo.wb_C = Lv.wb_C;
  io.det = h->det ? 1 : 0;
  io.swz = Lv.swz ? 1 : 0;
  io.l2ef = h->l2ef ? 1 : 0;
  const int ncol = h->det ? 27 : 1;
  for (int k = 0; k < ncol; ++k) {
    PatchIrrOp io2 = io;
    PatchFdOp fo2 = fo;
    if (h->det) {   // deterministic mode: the anchors of colour k (lists sorted by colour at setup)
      const int64_t i0 = Lv.irr_col[k], i1 = Lv.irr_col[k + 1];
      io2.anchors = Lv.irr_anchor + i0;
      io2.inv = Lv.irr_inv + i0 * Lv.pstride;
      io2.n_irr = do_irr ? i1 - i0 : 0;
      const int64_t r0 = Lv.reg_col[k], r1 = Lv.reg_col[k + 1];
      fo2.anchors = Lv.reg_list + r0;
      fo2.nreg = fd ? r1 - r0 : 0;
    }
    const bool di = io2.n_irr > 0, df = fo2.nreg + fo2.n_wb > 0;
    if (!di && !df) continue;
    const void* kf = patch_kernel(2 * q + 1, h->L.dim, di, df);
    void* args[] = {&io2, &fo2};
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(h->stream, &cap);
    const bool prof = h->patch_prof && cap == cudaStreamCaptureStatusNone;
    if (prof) {
      CU(cudaMemsetAsync(h->patch_prof, 0, (size_t)h->num_sms * 32, h->stream));
      io2.prof = h->patch_prof;
    }
    CU(cudaLaunchKernel(kf, dim3(h->num_sms), dim3((kIrrWarps + kFdWarps) * 32), args, patch_smem(h, q), h->stream));
    h->count();
    if (prof) {   // diagnostic: when did the two warp populations finish (ms after the first CTA started)
      std::vector<unsigned long long> t((size_t)h->num_sms * 4);
      CU(cudaMemcpyAsync(t.data(), h->patch_prof, t.size() * 8, cudaMemcpyDeviceToHost, h->stream));
      CU(cudaStreamSynchronize(h->stream));
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < h->num_sms; ++b) t0 = std::min(t0, t[4 * b]);
      double s[2][3] = {{1e30, 0, 0}, {1e30, 0, 0}};
      for (int b = 0; b < h->num_sms; ++b)
        for (int j = 0; j < 2; ++j) {
          const double ms = t[4 * b + 1 + j] ? (double)(t[4 * b + 1 + j] - t0) * 1e-6 : 0.0;
          s[j][0] = std::min(s[j][0], ms); s[j][1] += ms / h->num_sms; s[j][2] = std::max(s[j][2], ms);
        }
      fprintf(stderr, "[patch_prof] q=%d part=%d n_irr=%lld nreg=%lld n_wb=%lld: streaming done min/mean/max %.3f %.3f %.3f ms, FD done %.3f %.3f %.3f ms\n",
              q, part, (long long)io2.n_irr, (long long)fo2.nreg, (long long)fo2.n_wb, s[0][0], s[0][1], s[0][2], s[1][0], s[1][1], s[1][2]);
    }
  }
  if (do_irr_wb(h, q, part) && !Lv.wb_fused) {   // low-rank individual patches, separate launch
    PatchWbOp wo{};
    wo.nx = h->L.n[0]; wo.ny = h->L.n[1]; wo.nz = h->L.n[2]; wo.dim = h->L.dim;
    for (int i = 0; i < 3; ++i) wo.na[i] = Lv.na[i];
    wo.q = q; wo.S = 2 * q + 1; wo.mb = Lv.mb; wo.ncls = Lv.fd_ncls; wo.n_wb = Lv.n_wb;
    wo.anchors = Lv.wb_anchor; wo.soff = Lv.wb_soff; wo.slots = Lv.wb_slots; wo.coff = Lv.wb_coff; wo.C = Lv.wb_C;
    wo.tsl = Lv.wb_tsl; wo.mem = Lv.d_mem; wo.loc = Lv.d_loc;
    for (int k = 0; k < 8; ++k)
      for (int i = 0; i < 3; ++i) wo.mo[k][i] = Lv.mo[k][i];
    wo.cls = Lv.fd_cls; wo.tabs = Lv.fd_tabs; wo.s_fac = Lv.fd_s;
    wo.base = Lv.base; wo.stride3 = Lv.stride; wo.cmin = Lv.cmin; wo.cmax = Lv.cmax; wo.m = Lv.m;
    wo.in = r; wo.out = x; wo.coef = coef;
    void* args[] = {&wo};
    const int ng = wb_threads_rt(2 * q + 1, h->L.dim) / 32;   // upper bound of the patch groups per CTA
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((Lv.n_wb + ng - 1) / ng + Lv.n_wb / 8, (int64_t)h->num_sms * 3));
    CU(cudaLaunchKernel(wb_kernel(2 * q + 1, h->L.dim), dim3(grid), dim3(wb_threads_rt(2 * q + 1, h->L.dim)), args,
                        wb_smem_rt(2 * q + 1, h->L.dim, Lv.mb), h->stream));
    h->count();
  }
  if (do_reg && !Lv.fd) {
    BlockOp op{};
    op.colour = -1;
    op.nx = h->L.n[0]; op.ny = h->L.n[1]; op.nz = h->L.n[2];
    for (int i = 0; i < 3; ++i) op.na[i] = Lv.na[i];
    op.nanchor = Lv.nanchor;
    op.mb = Lv.mb;
    op.nmem = Lv.nmem;
    for (int k = 0; k < 8; ++k)
      for (int i = 0; i < 3; ++i) op.mo[k][i] = Lv.mo[k][i];
    op.mem = Lv.d_mem; op.loc = Lv.d_loc;
    op.m = Lv.m; op.base = Lv.base; op.stride = Lv.stride; op.cmin = Lv.cmin; op.cmax = Lv.cmax;
    op.blk = Lv.blk; op.type_inv = Lv.type_inv; op.irr_inv = nullptr; op.inv_alpha = 1.0 / h->alpha;
    op.in = r; op.out = x; op.coef = coef;
    const int64_t wpb = kThreads / 32;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((Lv.nanchor + wpb - 1) / wpb, (int64_t)h->num_sms * 8));
    for (int k = h->det ? 0 : -1; k < (h->det ? 27 : 0); ++k) {
      op.colour = k;
      k_block_smooth<<<nb, kThreads, block_smem(Lv.m, Lv.mb), h->stream>>>(op);
      h->count();
    }
  }
  CU(cudaGetLastError());
  return FCM_OK;
}

static int smooth_into(fcm_mg* h, int q, const double* r, double* x, double* cp_dst = nullptr,
                       const double* cp_src = nullptr) {
  if (h->lev[q].patch) {
    RC(launch_block_smooth(h, q, r, x, h->lev[q].omega));
    if (cp_dst) RC(copy(h, cp_dst, cp_src, h->lev[q].ndof));
    return FCM_OK;
  }
  return launch_cellop(h, q, make_op(h, q, OP_SMOOTH, r, x, h->lev[q].omega, nullptr), cp_dst, cp_src,
                       h->lev[q].ndof);
}
// x += omega M^-1 r.  Slab mode: the increment is exchanged (x itself is consistent), so it
// goes through d unless x is known to be zero.
static int smooth(fcm_mg* h, int q, const double* r, double* x, bool x_is_zero = false,
                  double* cp_dst = nullptr, const double* cp_src = nullptr) {
  if (!h->multi) return smooth_into(h, q, r, x, cp_dst, cp_src);
  LevelDev& Lv = h->lev[q];
  if (x_is_zero) {
    RC(smooth_into(h, q, r, x));
    return exchange(h, q, x);
  }
  RC(fill(h, Lv.d, 0.0, Lv.ndof));
  RC(smooth_into(h, q, r, Lv.d));
  RC(exchange(h, q, Lv.d));
  k_axpy<<<grid_for(Lv.ndof, h->num_sms), kThreads, 0, h->stream>>>(x, 1.0, Lv.d, Lv.ndof);
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}

static int enqueue_coarse(fcm_mg* h, const double* b, double* x);
// slab mode: replicated coarse solve -- all-gather the owned level-1 residual into the global
// p = 1 vector, solve on every rank with the global handle, keep the local slots
static int enqueue_coarse_slab(fcm_mg* h, const double* b, double* x) {
  const int64_t n1 = h->lev[1].ndof;
  k_gather32<<<grid_for(h->c_count, h->num_sms), kThreads, 0, h->stream>>>(h->c_send, b, h->c_pack, h->c_count);
  h->count();
  CU(cudaGetLastError());
  NC(nccl().AllGather(h->c_send, h->c_recv, h->c_max, ncclFloat64, h->comm, h->stream));
  const int64_t ntot = h->c_max * h->nranks;
  k_scatter64<<<grid_for(ntot, h->num_sms), kThreads, 0, h->stream>>>(h->c_bg, h->c_recv, h->c_unpack, ntot);
  h->count();
  CU(cudaGetLastError());
  fcm_mg* hg = h->hg;
  hg->count_target = h->count_target;
  const int rc = enqueue_coarse(hg, h->c_bg, h->c_xg);
  h->launches += hg->launches;
  hg->launches = 0;
  hg->count_target = nullptr;
  RC(rc);
  k_gather64<<<grid_for(n1, h->num_sms), kThreads, 0, h->stream>>>(x, h->c_xg, h->c_extract, n1);
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}

static int enqueue_coarse_gmg(fcm_mg* h, const double* b, double* x);
static int coarse_dist(fcm_mg* h, const double* b, double* x);
static int enqueue_coarse(fcm_mg* h, const double* b, double* x) {
  if (h->hg) return h->dist ? coarse_dist(h, b, x) : enqueue_coarse_slab(h, b, x);
  if (h->prm.coarse == FCM_COARSE_GMG_PCG) return enqueue_coarse_gmg(h, b, x);
  LevelDev& L1 = h->lev[1];
  const int64_t n = L1.ndof;
  if (h->prm.coarse == FCM_COARSE_DIRECT) {
    k_dense_gemv<<<grid_for(n * 32, h->num_sms), kThreads, 0, h->stream>>>(h->d_A0inv, b, x, n);
    h->count();
    CU(cudaGetLastError());
    return FCM_OK;
  }
  if (h->ktiled) {
    TiledArgs a = h->tiled;
    a.b = b;
    a.x = x;
    void* args[] = {&a};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(h->t_blocks);
    cfg.blockDim = dim3(kTiledThreads);
    cfg.dynamicSmemBytes = h->t_smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelExC(&cfg, h->ktiled, args));
    h->count();
    return FCM_OK;
  }
  CoarseArgs a{};
  a.A = make_op(h, 1, OP_APPLY, nullptr, nullptr, 1.0, nullptr);
  a.M = make_op(h, 1, OP_SMOOTH, nullptr, nullptr, 1.0, nullptr);
  a.jacobi = h->prm.coarse == FCM_COARSE_JACOBI_PCG;
  a.diag_inv = h->d_diag_inv;
  a.b = b; a.x = x;
  for (int i = 0; i < 2; ++i) {
    a.r[i] = h->c_vec[i]; a.z[i] = h->c_vec[2 + i]; a.w[i] = h->c_vec[4 + i]; a.q[i] = h->c_vec[6 + i];
  }
  a.p = h->c_vec[8];
  a.n = n;
  a.rtol2 = h->prm.coarse_rtol * h->prm.coarse_rtol;
  a.maxit = h->prm.coarse_maxit;
  a.part = h->c_part;
  a.part_stride = kMaxPartials;
  a.ctl = h->c_ctl;
  {  // split the grid between the individual lists and the regular population (coarse.cuh)
    const int nb = h->coarse_blocks;
    auto share = [&](int64_t nlist) {
      if (L1.M == 0) return nb;
      if (nlist <= 0 || nb < 2) return 0;
      int64_t v = (2 * nb * nlist + h->ncell - 1) / h->ncell;
      return (int)std::max<int64_t>(1, std::min<int64_t>(v, nb / 2));
    };
    a.nbl_A = share(h->ncut);
    a.nbl_M = share(L1.n_irr);
  }
  a.iters = h->d_coarse_iters;
  {   // fused r update in the smoother gather for L2-resident levels, split above ~2M DOFs
    const char* e = getenv("FCM_COARSE_SPLIT");
    a.split_s = e ? atoi(e) > 0 : (n >= (int64_t)2000000);
  }
  if (L1.kmma) {   // regular cells as fp64 MMA groups (cellmma.cuh)
    a.gA_cells = L1.gA_cells; a.gA_mat = L1.gA_mat; a.nA = L1.nA;
    if (!a.jacobi) { a.gS_cells = L1.gS_cells; a.gS_mat = L1.gS_mat; a.nS = L1.nS; }
  }
  void* args[] = {&a};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(h->coarse_blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = coarse_smem(L1.m, L1.M, L1.M > 0 ? coarse_group(L1.M) : L1.G);
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CU(cudaLaunchKernelExC(&cfg, h->kcoarse, args));
  h->count();
  return FCM_OK;
}


// ---- h-coarsening below p = 1 (FCM_COARSE_GMG_PCG): host side ------------------------------
static int dot_blocks(fcm_mg* h);
static GmgBox gmg_box(const Layout& L) {
  GmgBox B{};
  B.nf = L.n_f;
  for (int c = 0; c < L.n_f; ++c) {   // level-1 classes: the vertex class of each component first
    const DofClass& dc = L.classes[c];
    B.off[c] = dc.off;
    for (int a = 0; a < 3; ++a) { B.lo[c][a] = dc.lo[a]; B.size[c][a] = std::max(1, dc.size[a]); }
  }
  return B;
}
static void set_stream(fcm_mg* h, cudaStream_t st) {
  h->stream = st;
  for (fcm_mg* c : h->gmg) c->stream = st;
}
// Add a conditional node (WHILE / IF) on `cond` to the graph being captured on h->stream and
// capture its body -- body() enqueued with h and its h-level children switched to `sub`.
template <typename F>
static int captured_conditional(fcm_mg* h, cudaGraphConditionalHandle cond, cudaGraphConditionalNodeType type,
                                cudaStream_t sub, F&& body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CU(cudaStreamGetCaptureInfo_v3(h->stream, &st, nullptr, &g, &deps, nullptr, &nd));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CU(cudaGraphAddNode(&node, g, deps, nd, &cp));
  CU(cudaStreamUpdateCaptureDependencies(h->stream, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStream_t saved = h->stream;
  set_stream(h, sub);
  cudaError_t e = cudaStreamBeginCaptureToGraph(sub, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  int rc = e == cudaSuccess ? body() : FCM_ECUDA;
  cudaGraph_t outg;
  cudaError_t e2 = e == cudaSuccess ? cudaStreamEndCapture(sub, &outg) : e;
  set_stream(h, saved);
  if (rc < 0) return rc == FCM_ECUDA && e != cudaSuccess ? fail(FCM_ECUDA, "conditional body capture: %s", cudaGetErrorString(e)) : rc;
  if (e2 != cudaSuccess) return fail(FCM_ECUDA, "conditional body capture: %s", cudaGetErrorString(e2));
  return FCM_OK;
}
static cudaGraphConditionalHandle capture_cond_handle(fcm_mg* h, unsigned dflt, int* rc) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  cudaGraphConditionalHandle c = 0;
  cudaError_t e = cudaStreamGetCaptureInfo_v3(h->stream, &st, nullptr, &g, nullptr, nullptr, nullptr);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&c, g, dflt, cudaGraphCondAssignDefault);
  *rc = e == cudaSuccess ? FCM_OK : fail(FCM_ECUDA, "conditional handle: %s", cudaGetErrorString(e));
  return c;
}

// level-1 AS sweep with an explicit coefficient (the h-levels' damped smoother)
static int smooth_w(fcm_mg* h, const double* r, double* x, double w) {
  return launch_cellop(h, 1, make_op(h, 1, OP_SMOOTH, r, x, w, nullptr));
}
// geometric V-cycle on h-level i (0: this handle's level 1), x = 0 on entry, residual before
// every sweep (R1), trilinear transfers, dense solve on the coarsest grid (oracle:
// GeometricLevels.vcycle)
static int gmg_vcycle(fcm_mg* h, int i, const double* b, double* x) {
  const int L = (int)h->gmg.size();
  fcm_mg* hi = i == 0 ? h : h->gmg[i - 1];
  const int64_t n = hi->lev[1].ndof;
  if (i == L) {
    k_dense_gemv<<<grid_for(n * 32, h->num_sms), kThreads, 0, h->stream>>>(hi->d_A0inv, b, x, n);
    h->count();
    CU(cudaGetLastError());
    return FCM_OK;
  }
  double* r = hi->lev[1].r;
  const double w = h->gmg_omega;
  RC(fill(hi, x, 0.0, n));
  for (int s2 = 0; s2 < h->prm.n_pre; ++s2) {
    if (s2 == 0) { RC(smooth_w(hi, b, x, w)); continue; }
    RC(residual(hi, 1, b, x, r));
    RC(smooth_w(hi, r, x, w));
  }
  RC(residual(hi, 1, b, x, r));
  const GmgBox F = gmg_box(hi->L), C = gmg_box(h->gmg[i]->L);
  const int64_t nc = h->gmg[i]->lev[1].ndof;
  CU(pdl_launch(h, k_gmg_restrict, dim3(grid_for(nc, h->num_sms)), dim3(kThreads), h->gmg_b[i + 1],
                (const double*)r, C, F, h->L.dim, nc));
  h->count();
  RC(gmg_vcycle(h, i + 1, h->gmg_b[i + 1], h->gmg_x[i + 1]));
  CU(pdl_launch(h, k_gmg_prolong, dim3(grid_for(n, h->num_sms)), dim3(kThreads), x, (const double*)h->gmg_x[i + 1],
                F, C, h->L.dim, n));
  h->count();
  for (int s2 = 0; s2 < h->prm.n_post; ++s2) {
    RC(residual(hi, 1, b, x, r));
    RC(smooth_w(hi, r, x, w));
  }
  return FCM_OK;
}

// x = A_1^{-1} b by CG preconditioned with the geometric V-cycle, stop at ||r|| < rtol ||r0||
// (reading R4), as nested conditional graph nodes: must be enqueued inside a stream capture
static int enqueue_coarse_gmg(fcm_mg* h, const double* b, double* x) {
  cudaStreamCaptureStatus cs;
  CU(cudaStreamIsCapturing(h->stream, &cs));
  if (cs != cudaStreamCaptureStatusActive) return fail(FCM_EINVAL, "internal: GMG coarse solve outside a capture");
  const int64_t n = h->lev[1].ndof;
  double *r = h->c_vec[0], *z = h->c_vec[1], *p = h->c_vec[2], *q = h->c_vec[3];
  double *pA = h->c_part, *pB = h->c_part + kMaxPartials, *pC = h->c_part + 2 * kMaxPartials,
         *pD = h->c_part + 4 * kMaxPartials;
  const int nbd = dot_blocks(h);
  const int nbc = cellop_nblocks(h, 1, OP_APPLY);
  for (fcm_mg* c : h->gmg) c->count_target = h->count_target ? h->count_target : &h->launches;
  k_fcg_start<<<grid_for(n, h->num_sms), kThreads, 0, h->stream>>>(x, r, b, n);
  h->count();
  RC(gmg_vcycle(h, 0, r, z));
  CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), (const double*)r, (const double*)z, n, pA, (const uint8_t*)nullptr));
  CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), (const double*)r, (const double*)r, n, pB, (const uint8_t*)nullptr));
  h->count(2);
  int rc = FCM_OK;
  cudaGraphConditionalHandle cw = capture_cond_handle(h, 0, &rc);
  RC(rc);
  k_gcg_init<<<grid_for(n, h->num_sms), kThreads, 0, h->stream>>>(h->gcg, pA, pB, nbd, p, z, n, cw);
  h->count();
  CU(cudaGetLastError());
  int64_t* tgt = h->count_target ? h->count_target : &h->launches;
  const int64_t k0 = *tgt;
  rc = captured_conditional(h, cw, cudaGraphCondTypeWhile, h->st_c[0], [&]() -> int {
    RC(fill(h, q, 0.0, n));
    RC(launch_cellop(h, 1, make_op(h, 1, OP_APPLY, p, q, 1.0, pC)));
    CU(pdl_launch(h, k_gcg_update, dim3(nbd), dim3(kThreads), h->gcg, (const double*)pC, nbc, x, r, (const double*)p,
                  (const double*)q, n, pD));
    h->count();
    int rc2 = FCM_OK;
    cudaGraphConditionalHandle ci = capture_cond_handle(h, 0, &rc2);
    RC(rc2);
    CU(pdl_launch(h, k_gcg_check, dim3(1), dim3(32), h->gcg, (const double*)pD, nbd, cw, ci, h->d_coarse_iters));
    h->count();
    return captured_conditional(h, ci, cudaGraphCondTypeIf, h->st_c[1], [&]() -> int {
      RC(gmg_vcycle(h, 0, r, z));
      CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), (const double*)r, (const double*)z, n, pA,
                    (const uint8_t*)nullptr));
      CU(pdl_launch(h, k_gcg_update2, dim3(grid_for(n, h->num_sms)), dim3(kThreads), h->gcg, (const double*)pA, nbd,
                    p, (const double*)z, n));
      CU(pdl_launch(h, k_gcg_setrz, dim3(1), dim3(32), h->gcg));
      h->count(3);
      return FCM_OK;
    });
  });
  h->n_gcg_body = *tgt - k0;
  for (fcm_mg* c : h->gmg) c->count_target = nullptr;
  return rc;
}

// ---- distributed coarse solve (slab mode, FCM_COARSE_GMG_PCG) -------------------------------
// owner-masked dot of two local level-1 vectors, all-reduced into d[slot]
static int dot_dist(fcm_mg* h, const double* a, const double* b, int64_t n, int slot) {
  const int nbd = dot_blocks(h);
  k_dot<<<nbd, kThreads, 0, h->stream>>>(a, b, n, h->d_partA, h->d_own);
  k_finalize<<<1, 32, 0, h->stream>>>(h->d_dcg + slot, h->d_partA, nbd);
  h->count(2);
  CU(cudaGetLastError());
  return allreduce(h, h->d_dcg + slot, 1);
}
// damped level-1 AS sweep on the slab: x += w M^-1 r (increment summed over the interface)
static int smooth_dist(fcm_mg* h, const double* r, double* x, double w, bool x_is_zero) {
  LevelDev& L1 = h->lev[1];
  if (x_is_zero) {
    RC(launch_cellop(h, 1, make_op(h, 1, OP_SMOOTH, r, x, w, nullptr)));
    return exchange(h, 1, x);
  }
  RC(fill(h, L1.d, 0.0, L1.ndof));
  RC(launch_cellop(h, 1, make_op(h, 1, OP_SMOOTH, r, L1.d, w, nullptr)));
  RC(exchange(h, 1, L1.d));
  k_axpy<<<grid_for(L1.ndof, h->num_sms), kThreads, 0, h->stream>>>(x, 1.0, L1.d, L1.ndof);
  h->count();
  CU(cudaGetLastError());
  return FCM_OK;
}
// geometric V-cycle with h-level 0 on the slabs (same steps as gmg_vcycle at i = 0) and the
// levels below replicated (the global handle's gmg_vcycle from h-level 1)
static int gmg_vcycle_dist(fcm_mg* h, const double* b, double* x) {
  fcm_mg* hg = h->hg;
  LevelDev& L1 = h->lev[1];
  const int64_t n = L1.ndof;
  double* r = L1.r;
  const double w = hg->gmg_omega;
  RC(fill(h, x, 0.0, n));
  for (int s2 = 0; s2 < h->prm.n_pre; ++s2) {
    if (s2 == 0) { RC(smooth_dist(h, b, x, w, true)); continue; }
    RC(residual(h, 1, b, x, r));
    RC(smooth_dist(h, r, x, w, false));
  }
  RC(residual(h, 1, b, x, r));
  fcm_mg* c1 = hg->gmg[0];
  const int64_t nc = c1->lev[1].ndof;
  const GmgBox F = gmg_box(h->L), C = gmg_box(c1->L);
  CU(cudaMemsetAsync(hg->gmg_b[1], 0, nc * 8, h->stream));
  k_gmg_restrict_dist<<<grid_for(nc, h->num_sms), kThreads, 0, h->stream>>>(
      hg->gmg_b[1], r, C, F, h->L.dim, h->z0, h->rank > 0 ? 1 : 0, h->dist_cz0, h->dist_cz1);
  h->count();
  CU(cudaGetLastError());
  RC(allreduce(h, hg->gmg_b[1], (int)nc));
  hg->count_target = h->count_target;
  const int rc = gmg_vcycle(hg, 1, hg->gmg_b[1], hg->gmg_x[1]);
  h->launches += hg->launches;
  hg->launches = 0;
  hg->count_target = nullptr;
  RC(rc);
  k_gmg_prolong_dist<<<grid_for(n, h->num_sms), kThreads, 0, h->stream>>>(x, hg->gmg_x[1], F, C, h->L.dim, h->z0, n);
  h->count();
  CU(cudaGetLastError());
  for (int s2 = 0; s2 < h->prm.n_post; ++s2) {
    RC(residual(h, 1, b, x, r));
    RC(smooth_dist(h, r, x, w, false));
  }
  return FCM_OK;
}
// x = A_1^{-1} b by CG + the geometric V-cycle on the slabs, ||r|| < rtol ||r0|| (reading R4);
// host-driven: one D2H of the reduced scalars per iteration (eager mode)
static int coarse_dist(fcm_mg* h, const double* b, double* x) {
  const int64_t n = h->lev[1].ndof;
  double *r = h->c_vec[0], *z = h->c_vec[1], *pv = h->c_vec[2], *q = h->c_vec[3];
  const int g = grid_for(n, h->num_sms);
  k_fcg_start<<<g, kThreads, 0, h->stream>>>(x, r, b, n);
  h->count();
  RC(gmg_vcycle_dist(h, r, z));
  RC(dot_dist(h, r, z, n, 0));   // rz
  RC(dot_dist(h, r, r, n, 4));   // rr0
  RC(copy(h, pv, z, n));
  CU(cudaMemcpyAsync(h->h_dcg, h->d_dcg, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  const double rr0 = h->h_dcg[4];
  const double rtol2 = h->prm.coarse_rtol * h->prm.coarse_rtol;
  int it = 0;
  if (rr0 > 0.0 && h->prm.coarse_maxit > 0) {
    while (true) {
      RC(fill(h, q, 0.0, n));
      RC(launch_cellop(h, 1, make_op(h, 1, OP_APPLY, pv, q, 1.0, nullptr)));
      RC(exchange(h, 1, q));
      RC(dot_dist(h, pv, q, n, 1));   // pq
      k_dcg_update<<<g, kThreads, 0, h->stream>>>(h->d_dcg, x, r, pv, q, n);
      h->count();
      RC(dot_dist(h, r, r, n, 2));    // rr
      CU(cudaMemcpyAsync(h->h_dcg, h->d_dcg, 8 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
      CU(cudaStreamSynchronize(h->stream));
      ++it;
      const double pq = h->h_dcg[1], rr = h->h_dcg[2];
      if (!(pq > 0.0) || !(rr == rr) || rr < rtol2 * rr0 || it >= h->prm.coarse_maxit) break;
      RC(gmg_vcycle_dist(h, r, z));
      RC(dot_dist(h, r, z, n, 3));    // rz_new
      k_dcg_update2<<<g, kThreads, 0, h->stream>>>(h->d_dcg, pv, z, n);
      k_dcg_setrz<<<1, 32, 0, h->stream>>>(h->d_dcg);
      h->count(2);
      CU(cudaGetLastError());
    }
  }
  h->h_ci[0] = it;
  h->h_ci[1] += it;
  CU(cudaMemcpyAsync(h->hg->d_coarse_iters, h->h_ci, 2 * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));   // h_ci is reused by the next solve
  return FCM_OK;
}

// build the h-levels: Galerkin element matrices K_C = sum_f W_f^T K_f W_f of every coarse cell
// (W_f: trilinear weights of the coarse cell's 2^d vertices at child f's vertices, (x) I_nf), a
// child handle per level (p = 1 grid, its own elementwise AS); the coarsest solves directly
static thread_local bool tl_gmg_child = false;
static int setup_impl(const fcm_grid* g, const fcm_params* prm, const fcm_slab* slab, const double* K_ref,
                      const uint8_t* cell_kind, double alpha, int64_t n_cut, const int64_t* cut_cells,
                      const double* cut_K, int64_t n_cc, const int64_t* cc_cells, const double* cc_K1,
                      fcm_mg** out);
static int setup_gmg(fcm_mg* h, const double* K_ref, const std::vector<uint8_t>& kind_own,
                     const std::vector<int32_t>& cut_idx_own, const double* cut_K) {
  const Layout& L0 = h->L;
  const int dim = L0.dim, nf = L0.n_f, m = L0.m, m1 = L0.m_level[1];
  const int nv = 1 << dim;
  int n[3] = {L0.n[0], L0.n[1], L0.n[2]};
  auto even_all = [&]() {
    for (int a = 0; a < dim; ++a)
      if (n[a] % 2 || n[a] <= 4) return false;
    return true;
  };
  if (!even_all()) return fail(FCM_EINVAL, "GMG coarse solve needs even cell counts > 4 per axis (grid %d)", n[0]);
  // level-0 data: leading p=1 blocks
  std::vector<double> K1((size_t)m1 * m1);
  for (int r = 0; r < m1; ++r)
    for (int c = 0; c < m1; ++c) K1[(size_t)r * m1 + c] = K_ref[(size_t)r * m + c];
  std::vector<uint8_t> kinds = kind_own;
  std::vector<int64_t> ind_idx(kinds.size(), -1);   // cell -> index in ind_K
  std::vector<double> ind_K;
  for (size_t c = 0; c < kinds.size(); ++c)
    if (kinds[c] == 2) {
      ind_idx[c] = (int64_t)(ind_K.size() / ((size_t)m1 * m1));
      const double* src = cut_K + (size_t)cut_idx_own[c] * m * m;
      for (int r = 0; r < m1; ++r)
        for (int cc = 0; cc < m1; ++cc) ind_K.push_back(src[(size_t)r * m + cc]);
    }
  // trilinear child weights W_f[a_fine][A_coarse] (local DOF = vertex mode * nf + comp, mode = sum k_a 2^a)
  std::vector<std::vector<double>> W(nv, std::vector<double>((size_t)m1 * m1, 0.0));
  for (int f = 0; f < nv; ++f)
    for (int vf = 0; vf < nv; ++vf)
      for (int vc = 0; vc < nv; ++vc) {
        double w = 1.0;
        for (int a = 0; a < dim; ++a) {
          const double t = 0.5 * (((f >> a) & 1) + ((vf >> a) & 1));
          w *= ((vc >> a) & 1) ? t : 1.0 - t;
        }
        for (int c = 0; c < nf; ++c) W[f][(size_t)(vf * nf + c) * m1 + vc * nf + c] = w;
      }
  auto galerkin = [&](const std::vector<const double*>& Kf, const std::vector<double>& sc, double* out) {
    std::vector<double> T((size_t)m1 * m1);
    std::fill(out, out + (size_t)m1 * m1, 0.0);
    for (int f = 0; f < nv; ++f) {
      if (!Kf[f]) continue;
      // T = K_f W_f, out += W_f^T T
      for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m1; ++j) {
          double t = 0.0;
          for (int k = 0; k < m1; ++k) t += Kf[f][(size_t)i * m1 + k] * W[f][(size_t)k * m1 + j];
          T[(size_t)i * m1 + j] = t * sc[f];
        }
      for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m1; ++j) {
          double t = 0.0;
          for (int k = 0; k < m1; ++k) t += W[f][(size_t)k * m1 + i] * T[(size_t)k * m1 + j];
          out[(size_t)i * m1 + j] += t;
        }
    }
  };
  h->gmg_b.assign(1, nullptr);
  h->gmg_x.assign(1, nullptr);
  h->gmg_omega = dim == 3 ? 2.0 / 15.0 : 1.0 / 3.0;   // elementwise omega of P:300 (R21)
  while (even_all()) {
    int nc[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) nc[a] = n[a] / 2;
    const int64_t ncell_c = (int64_t)nc[0] * nc[1] * nc[2];
    std::vector<uint8_t> kc(ncell_c);
    std::vector<int64_t> icells;
    std::vector<double> iK;
    std::vector<double> K1c((size_t)m1 * m1);
    {
      std::vector<const double*> kf(nv, K1.data());
      std::vector<double> sc(nv, 1.0);
      galerkin(kf, sc, K1c.data());
    }
    std::vector<int64_t> ind_idx_c(ncell_c, -1);
    std::vector<double> tmp((size_t)m1 * m1);
    for (int64_t C = 0; C < ncell_c; ++C) {
      const int cx = (int)(C % nc[0]), cy = (int)((C / nc[0]) % nc[1]), cz = (int)(C / ((int64_t)nc[0] * nc[1]));
      std::vector<const double*> kf(nv, nullptr);
      std::vector<double> sc(nv, 1.0);
      int k0 = -1;
      bool uniform = true;
      for (int f = 0; f < nv; ++f) {
        const int fx = 2 * cx + (f & 1), fy = 2 * cy + ((f >> 1) & 1), fz = dim == 3 ? 2 * cz + ((f >> 2) & 1) : 0;
        const int64_t fc = ((int64_t)fz * n[1] + fy) * n[0] + fx;
        const int k = kinds[fc];
        if (k == 2) kf[f] = ind_K.data() + (size_t)ind_idx[fc] * m1 * m1;
        else { kf[f] = K1.data(); sc[f] = k == 1 ? h->alpha : 1.0; }
        if (k == 2 || (k0 >= 0 && k != k0)) uniform = false;
        k0 = k;
      }
      if (uniform) { kc[C] = (uint8_t)k0; continue; }
      kc[C] = 2;
      galerkin(kf, sc, tmp.data());
      ind_idx_c[C] = (int64_t)icells.size();
      icells.push_back(C);
      iK.insert(iK.end(), tmp.begin(), tmp.end());
    }
    // child handle: p = 1 on the coarse grid
    fcm_grid gc = h->g;
    gc.p = 1;
    for (int a = 0; a < dim; ++a) gc.n[a] = nc[a];
    gc.h = h->g.h * 2.0;
    for (int a = 0; a < dim; ++a) n[a] = nc[a];
    const bool bottom = !even_all();
    fcm_params pc = h->prm;
    pc.coarse = bottom ? FCM_COARSE_DIRECT : FCM_COARSE_AS_PCG;
    pc.stream = (void*)h->stream;
    fcm_mg* child = nullptr;
    tl_gmg_child = !bottom;
    const int rc = setup_impl(&gc, &pc, nullptr, K1c.data(), kc.data(), h->alpha, (int64_t)icells.size(),
                              icells.data(), iK.data(), 0, nullptr, nullptr, &child);
    tl_gmg_child = false;
    RC(rc);
    CU(cudaStreamSynchronize(child->stream));
    CU(cudaStreamDestroy(child->stream));
    child->stream = h->stream;
    child->borrowed_stream = true;
    h->gmg.push_back(child);
    double *bb, *xx;
    RC(h->alloc(&bb, child->lev[1].ndof));
    RC(h->alloc(&xx, child->lev[1].ndof));
    h->gmg_b.push_back(bb);
    h->gmg_x.push_back(xx);
    K1 = K1c;
    kinds = kc;
    ind_idx = ind_idx_c;
    ind_K.swap(iK);
  }
  const int64_t n1 = h->lev[1].ndof;
  for (int i = 0; i < 9; ++i) RC(h->alloc(&h->c_vec[i], n1));
  RC(h->alloc(&h->c_part, 6 * kMaxPartials));
  RC(h->alloc(&h->gcg, 1));
  RC(h->alloc(&h->c_bst, n1));
  RC(h->alloc(&h->c_xst, n1));
  GcgScalars gs{};
  gs.maxit = h->prm.coarse_maxit;
  gs.rtol2 = h->prm.coarse_rtol * h->prm.coarse_rtol;
  CU(cudaMemcpyAsync(h->gcg, &gs, sizeof(gs), cudaMemcpyHostToDevice, h->stream));
  for (auto& st : h->st_c) CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CU(cudaStreamSynchronize(h->stream));
  return FCM_OK;
}
// Algorithm 1 on level q: x = V_q(b), x~ = 0 on entry; reading R1.
static int enqueue_vcycle(fcm_mg* h, int q, const double* b, double* x) {
  if (q == 1) return enqueue_coarse(h, b, x);
  LevelDev& Lv = h->lev[q];
  const int64_t N = Lv.ndof;
  // single GPU, elementwise MMA path: the residual is double-buffered and each smoother launch
  // also writes "r = b" into the buffer the next residual scatters into (no copy launches)
  const bool fuse = Lv.kmma && !h->multi && !h->det && !Lv.patch && Lv.r2;
  double* rb[2] = {Lv.r, Lv.r2 ? Lv.r2 : Lv.r};
  int cur = 0;
  RC(fill(h, x, 0.0, N));
  for (int s = 0; s < h->prm.n_pre; ++s) {          // pre-smoothing
    if (s == 0) {
      RC(smooth(h, q, b, x, true, fuse ? rb[cur] : nullptr, b));   // x = 0: r = b
    } else {
      RC(residual(h, q, b, x, rb[cur], fuse));
      RC(smooth(h, q, rb[cur], x, false, fuse ? rb[cur ^ 1] : nullptr, b));
      if (fuse) cur ^= 1;
    }
  }
  if (h->prm.n_pre > 0) RC(residual(h, q, b, x, rb[cur], fuse));  // update residual
  else RC(copy(h, rb[cur], b, N));
  LevelDev& Lc = h->lev[q - 1];
  RC(enqueue_vcycle(h, q - 1, rb[cur], Lc.x));      // r_{l-1} = R r_l: prefix alias
  // x += R^T e (and, fused path, the next residual buffer = b)
  CU(pdl_launch(h, k_axpy_copy, dim3(grid_for(N, h->num_sms)), dim3(kThreads), x, 1.0, Lc.x, Lc.ndof, fuse ? rb[cur ^ 1] : nullptr, b,
                                                                    fuse ? N : 0));
  h->count();
  CU(cudaGetLastError());
  if (fuse) cur ^= 1;
  for (int s = 0; s < h->prm.n_post; ++s) {         // P:169 residual, post-smoothing
    RC(residual(h, q, b, x, rb[cur], fuse));
    const bool more = s + 1 < h->prm.n_post;
    RC(smooth(h, q, rb[cur], x, false, fuse && more ? rb[cur ^ 1] : nullptr, b));
    if (fuse) cur ^= 1;
  }
  return FCM_OK;
}

// capture a host enqueue sequence into an executable graph
template <typename F>
static int capture(fcm_mg* h, cudaGraphExec_t* exec, int64_t* nkernels, F&& body) {
  if (*exec) return FCM_OK;
  if (h->eager) {   // keep the body (it must capture by value); run_graph calls it
    h->eager_fn[(const void*)exec] = std::function<int()>(body);
    *exec = reinterpret_cast<cudaGraphExec_t>(exec);
    *nkernels = 0;
    return FCM_OK;
  }
  cudaGraph_t graph;
  *nkernels = 0;
  h->count_target = nkernels;
  CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int rc = body();
  cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
  h->count_target = nullptr;
  if (rc < 0) { if (e == cudaSuccess) cudaGraphDestroy(graph); return rc; }
  if (e != cudaSuccess) return fail(FCM_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(FCM_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  return FCM_OK;
}

static int run_graph(fcm_mg* h, cudaGraphExec_t g, int64_t nk) {
  if (h->eager) {
    auto it = h->eager_fn.find((const void*)g);
    if (it == h->eager_fn.end()) return fail(FCM_EINVAL, "internal: eager body missing");
    return it->second();
  }
  CU(cudaGraphLaunch(g, h->stream));
  h->launches += nk;
  return FCM_OK;
}

static int dot_blocks(fcm_mg* h) { return std::min(kMaxPartials, h->num_sms * 2); }

// Work is enqueued on the handle's own non-blocking stream (capturable into graphs); it is
// ordered after prior work on the caller's stream and the caller's stream after it.
struct StreamGuard {
  fcm_mg* h;
  explicit StreamGuard(fcm_mg* h_) : h(h_) {
    cudaEventRecord(h->ev_in, h->ustream);
    cudaStreamWaitEvent(h->stream, h->ev_in, 0);
  }
  ~StreamGuard() {
    cudaEventRecord(h->ev_out, h->stream);
    cudaStreamWaitEvent(h->ustream, h->ev_out, 0);
  }
};

// =========================================================================================
// setup
// =========================================================================================
// Block geometry of level q (blocks.cuh): elementwise (anchor = cell, one member cell,
// assembly cells = the 3^d neighbourhood) or patchwise (anchor = vertex, the 2^d member cells
// around it, assembly cells = the 4^d neighbourhood), reading R11.
struct BlockGeom {
  bool patch = false;
  int na[3] = {1, 1, 1};
  int nmem = 1;
  int mo[8][3] = {};
  int mb = 0;
  std::vector<int8_t> mem;
  std::vector<int16_t> loc;
  int nasm = 3, aoff = -1;
  std::vector<int16_t> amap;   // [nasm^d][mb]
};

static BlockGeom block_geom(const Layout& L, int q, bool patch) {
  BlockGeom g;
  const int dim = L.dim, mq = L.m_level[q];
  g.patch = patch;
  for (int i = 0; i < 3; ++i) g.na[i] = i < dim ? L.n[i] + (patch ? 1 : 0) : 1;
  g.nmem = patch ? 1 << dim : 1;
  for (int k = 0; k < g.nmem; ++k)
    for (int i = 0; i < 3; ++i) g.mo[k][i] = (patch && i < dim) ? ((k >> i) & 1) - 1 : 0;
  // identity of a DOF relative to the anchor: (class, X) with X = 2*entity position (nodal
  // axis) or 2*cell+1 (internal axis), as in the DOF keys
  auto ident = [&](int a, const int off[3]) {
    const DofClass& dc = L.classes[L.dof_class[a]];
    std::array<int, 4> k{L.dof_class[a], 0, 0, 0};
    for (int i = 0; i < dim; ++i)
      k[1 + i] = (dc.S >> i & 1) ? 2 * off[i] + 1 : 2 * (off[i] + L.dof_off[a][i]);
    return k;
  };
  std::map<std::array<int, 4>, int> id;
  std::vector<std::array<int, 4>> keys;
  for (int k = 0; k < g.nmem; ++k)
    for (int a = 0; a < mq; ++a) {
      auto key = ident(a, g.mo[k]);
      if (id.count(key)) continue;
      id[key] = g.mb++;
      keys.push_back(key);
      g.mem.push_back((int8_t)k);
      g.loc.push_back((int16_t)a);
    }
  g.nasm = patch ? 4 : 3;
  g.aoff = patch ? -2 : -1;
  const int nas = dim == 3 ? g.nasm * g.nasm * g.nasm : (dim == 2 ? g.nasm * g.nasm : g.nasm);
  g.amap.assign((size_t)nas * g.mb, -1);
  for (int d = 0; d < nas; ++d) {
    int ao[3] = {0, 0, 0};
    ao[0] = g.aoff + d % g.nasm;
    if (dim >= 2) ao[1] = g.aoff + (d / g.nasm) % g.nasm;
    if (dim == 3) ao[2] = g.aoff + d / (g.nasm * g.nasm);
    for (int a = 0; a < mq; ++a) {
      auto it = id.find(ident(a, ao));
      if (it != id.end()) g.amap[(size_t)d * g.mb + it->second] = (int16_t)a;
    }
  }
  return g;
}

// global layout index of block DOF l at anchor coordinates A (-1: absent or Dirichlet)
static int64_t block_dof_index(const Layout& L, int q, const BlockGeom& g, int l, const int A[3]) {
  int cc[3];
  for (int i = 0; i < 3; ++i) {
    cc[i] = A[i] + g.mo[g.mem[l]][i];
    if (cc[i] < 0 || cc[i] >= L.n[i]) return -1;
  }
  return L.dof_index(q, g.loc[l], cc);
}

// packed cell entry of an MMA group (cellmma.cuh): coordinates + "no Dirichlet DOF" flag
static int32_t mma_pack(const fcm_mg* h, int q, int64_t c, bool scaled) {
  int cc[3];
  h->L.cell_coords(c, cc);
  const LevelDev& Lv = h->lev[q];
  bool inner = true;
  for (int i = 0; i < 3; ++i) inner = inner && cc[i] >= Lv.ilo[i] && cc[i] <= Lv.ihi[i];
  return (int32_t)((unsigned)(cc[0] | (cc[1] << 10) | (cc[2] << 20) | (inner ? kMmaInner : 0)) |
                   (scaled ? kMmaScaled : 0u));
}


// ---- patch levels at scale (patch.cuh) -----------------------------------------------------
// Generalised symmetric eigenproblem K S = M S Lambda, S^T M S = I, for n <= 9 (host, fp64):
// M = L L^T, C = L^-1 K L^-T, cyclic Jacobi C = Q Lambda Q^T, S = L^-T Q.
static bool gen_eig(int n, const std::vector<double>& K, const std::vector<double>& M, std::vector<double>& S,
                    std::vector<double>& lam) {
  std::vector<double> Lc(n * n, 0.0), C(n * n), Q(n * n, 0.0), T(n * n);
  for (int j = 0; j < n; ++j) {
    double d = M[j * n + j];
    for (int k = 0; k < j; ++k) d -= Lc[j * n + k] * Lc[j * n + k];
    if (!(d > 0)) return false;
    Lc[j * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double v = M[i * n + j];
      for (int k = 0; k < j; ++k) v -= Lc[i * n + k] * Lc[j * n + k];
      Lc[i * n + j] = v / Lc[j * n + j];
    }
  }
  // T = L^-1 K (forward substitution per column), C = T L^-T (= L^-1 T^T)^T
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      double v = K[i * n + c];
      for (int k = 0; k < i; ++k) v -= Lc[i * n + k] * T[k * n + c];
      T[i * n + c] = v / Lc[i * n + i];
    }
  for (int r = 0; r < n; ++r)   // C[r][:] = L^-1 (T[r][:])^T
    for (int i = 0; i < n; ++i) {
      double v = T[r * n + i];
      for (int k = 0; k < i; ++k) v -= Lc[i * n + k] * C[r * n + k];
      C[r * n + i] = v / Lc[i * n + i];
    }
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < i; ++j) C[i * n + j] = C[j * n + i] = 0.5 * (C[i * n + j] + C[j * n + i]);
    Q[i * n + i] = 1.0;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? tot : off) += C[i * n + j] * C[i * n + j];
    if (off <= 1e-30 * (tot + off)) break;
    for (int p = 0; p < n; ++p)
      for (int r = p + 1; r < n; ++r) {
        const double apr = C[p * n + r];
        if (apr == 0.0) continue;
        const double th = (C[r * n + r] - C[p * n + p]) / (2.0 * apr);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < n; ++k) {   // columns p, r
          const double ckp = C[k * n + p], ckr = C[k * n + r];
          C[k * n + p] = c * ckp - sn * ckr;
          C[k * n + r] = sn * ckp + c * ckr;
        }
        for (int k = 0; k < n; ++k) {   // rows p, r
          const double cpk = C[p * n + k], crk = C[r * n + k];
          C[p * n + k] = c * cpk - sn * crk;
          C[r * n + k] = sn * cpk + c * crk;
        }
        for (int k = 0; k < n; ++k) {
          const double qkp = Q[k * n + p], qkr = Q[k * n + r];
          Q[k * n + p] = c * qkp - sn * qkr;
          Q[k * n + r] = sn * qkp + c * qkr;
        }
      }
  }
  lam.assign(n, 0.0);
  for (int i = 0; i < n; ++i) lam[i] = C[i * n + i];
  S.assign(n * n, 0.0);   // S = L^-T Q: back substitution per column
  for (int c = 0; c < n; ++c)
    for (int i = n - 1; i >= 0; --i) {
      double v = Q[i * n + c];
      for (int k = i + 1; k < n; ++k) v -= Lc[k * n + i] * S[k * n + c];
      S[i * n + c] = v / Lc[i * n + i];
    }
  return true;
}

// Fast-diagonalisation tables of a tensor Poisson patch level (patch.cuh k_patch_fd): valid
// when K_ref is the Kronecker form s (K (x) M (x) M + ...) of the 1D reference matrices
// (checked to 1e-12); per axis and per axis class (clipped distances of the vertex to the two
// faces, R = 2 as in the type key) the assembled 1D matrices over the present patch slots.
static int setup_patch_fd(fcm_mg* h, int q, const double* K_ref_host) {
  const Layout& L = h->L;
  LevelDev& Lv = h->lev[q];
  if (h->g.space != 0 || h->g.n_f != 1 || h->multi || q > 4) return FCM_OK;
  const int dim = L.dim, p = L.p, P1 = p + 1, S = 2 * q + 1;
  std::vector<double> M1(P1 * P1), K1(P1 * P1);
  ref1d_matrices(p, M1.data(), K1.data());
  const double sfac = std::pow(0.5 * h->g.h, dim - 2);
  // check K_ref against the Kronecker form
  double mx = 0.0, err = 0.0;
  const int m = L.m;
  for (int I = 0; I < m; ++I)
    for (int J = 0; J < m; ++J) {
      double sum = 0.0;
      for (int gd = 0; gd < dim; ++gd) {
        double t = 1.0;
        for (int a = 0; a < dim; ++a)
          t *= (a == gd ? K1 : M1)[L.modes[I].k[a] * P1 + L.modes[J].k[a]];
        sum += t;
      }
      const double kr = K_ref_host[(size_t)I * m + J];
      mx = std::max(mx, std::fabs(kr));
      err = std::max(err, std::fabs(kr - sfac * sum));
    }
  if (!(err <= 1e-12 * mx)) return FCM_OK;   // not Kronecker: dense k_block_smooth path
  const int R = 2, ncls = (R + 1) * (R + 1) + 1;
  const int tsz = S * S + S;
  std::vector<double> tabs((size_t)3 * ncls * tsz, 0.0);
  std::vector<int> cls;
  std::vector<int16_t> midx((q + 1) * (q + 1) * (q + 1), -1);
  for (int a = 0; a < L.m_level[q]; ++a) {
    const int* k = L.modes[a].k;
    midx[(k[2] * (q + 1) + k[1]) * (q + 1) + k[0]] = (int16_t)a;
  }
  for (int ax = 0; ax < 3; ++ax) {
    const int n = L.n[ax];
    const int na = ax < dim ? n + 1 : 1;
    std::vector<char> done(ncls, 0);
    for (int v = 0; v < na; ++v) {
      if (ax >= dim) { cls.push_back(0); continue; }
      const int lo = std::min(v, R), hi = std::min(n - v, R);
      const int ci = (lo == R && hi == R) ? 0 : 1 + lo * (R + 1) + hi;
      cls.push_back(ci);
      if (done[ci]) continue;
      done[ci] = 1;
      // slots present, assembled 1D matrices over the slots
      const bool dlo = (L.dmask >> (2 * ax)) & 1, dhi = (L.dmask >> (2 * ax + 1)) & 1;
      auto vslot_ok = [&](int P) { return P >= 0 && P <= n && !(P == 0 && dlo) && !(P == n && dhi); };
      std::vector<char> pres(S, 0);
      pres[0] = vslot_ok(v - 1);
      pres[q] = vslot_ok(v);
      pres[2 * q] = vslot_ok(v + 1);
      for (int s2 = 1; s2 < q; ++s2) pres[s2] = (v - 1 >= 0 && v - 1 < n);
      for (int s2 = q + 1; s2 < 2 * q; ++s2) pres[s2] = (v < n);
      auto slot_of = [&](int c, int k) -> int {   // cell c, 1D mode k -> patch slot or -1
        if (k >= 2) {
          if (k > q) return -1;
          if (c == v - 1) return k - 1;
          if (c == v) return q + k - 1;
          return -1;
        }
        const int P = c + k;
        if (P == v - 1) return 0;
        if (P == v) return q;
        if (P == v + 1) return 2 * q;
        return -1;
      };
      std::vector<double> Ka(S * S, 0.0), Ma(S * S, 0.0);
      for (int c = v - 2; c <= v + 1; ++c) {
        if (c < 0 || c >= n) continue;
        for (int i = 0; i <= q; ++i)
          for (int j = 0; j <= q; ++j) {
            const int si = slot_of(c, i), sj = slot_of(c, j);
            if (si < 0 || sj < 0 || !pres[si] || !pres[sj]) continue;
            Ka[si * S + sj] += K1[i * P1 + j];
            Ma[si * S + sj] += M1[i * P1 + j];
          }
      }
      std::vector<int> ps;
      for (int s2 = 0; s2 < S; ++s2) if (pres[s2]) ps.push_back(s2);
      const int nq = (int)ps.size();
      std::vector<double> Kc(nq * nq), Mc(nq * nq), Sv, lam;
      for (int i = 0; i < nq; ++i)
        for (int j = 0; j < nq; ++j) { Kc[i * nq + j] = Ka[ps[i] * S + ps[j]]; Mc[i * nq + j] = Ma[ps[i] * S + ps[j]]; }
      if (!gen_eig(nq, Kc, Mc, Sv, lam)) return FCM_OK;
      double* t = tabs.data() + ((size_t)ax * ncls + ci) * tsz;
      for (int i = 0; i < nq; ++i)
        for (int j = 0; j < nq; ++j) t[ps[i] * S + j] = Sv[i * nq + j];
      for (int j = 0; j < S; ++j) t[S * S + j] = j < nq ? lam[j] : 1.0;
    }
  }
  RC(h->alloc(&Lv.fd_tabs, tabs.size()));
  RC(h->alloc(&Lv.fd_cls, cls.size()));
  RC(h->alloc(&Lv.fd_midx, midx.size()));
  CU(cudaMemcpyAsync(Lv.fd_tabs, tabs.data(), tabs.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.fd_cls, cls.data(), cls.size() * 4, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.fd_midx, midx.data(), midx.size() * 2, cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  Lv.fd_ncls = ncls;
  Lv.fd_tabs_h = tabs;
  Lv.fd_cls_h = cls;
  Lv.fd_s = sfac;
  Lv.fd = !(getenv("FCM_PATCH_FD") && atoi(getenv("FCM_PATCH_FD")) == 0);
  return FCM_OK;
}

// k_patch_smooth's dynamic shared memory (layout in patch.cuh)
static size_t patch_smem(const fcm_mg* h, int q) {
  const LevelDev& Lv = h->lev[q];
  const int S = 2 * q + 1, S3 = h->L.dim == 3 ? S * S * S : S * S, nmi = (q + 1) * (q + 1) * (q + 1);
  const size_t MPd = 32 * (size_t)Lv.nt;
  size_t o = (sizeof(Tab) + (size_t)(kIrrWarps / patch_wpp(Lv.nt)) * MPd * 20 + 255) / 256 * 256 + 256;
  o += (size_t)kIrrWarps * kIrrStages * 1024 * 8 + (size_t)kIrrWarps * kIrrStages * 8 + (size_t)kIrrWarps * 2 * 8;
  o += (size_t)3 * (Lv.fd ? Lv.fd_ncls : 0) * (S * S + S) * 8 + ((nmi * 2 + 15) / 16) * 16;
  o += ((size_t)S3 * 4 + 15) / 16 * 16;   // FD slot codes
  o += (size_t)kFdWarps * 2 * S3 * 8;
  return o;
}

// Assemble and invert the patch blocks of level q: shared types (full storage, type_inv) and
// individual blocks (tile-packed, irr_inv), through a chunked workspace: k_patch_asm (cell
// loop) -> batched blocked Gauss-Jordan -> copy (types) / k_pack_tiles (individual).
static int setup_patch_blocks(fcm_mg* h, int q, const BlockGeom& g, const std::vector<int32_t>& blk,
                              const std::vector<int64_t>& blocks, int64_t ntypes, const std::vector<int8_t>& dir) {
  const Layout& L = h->L;
  LevelDev& Lv = h->lev[q];
  if (h->multi) return fail(FCM_EINVAL, "patchwise blocks are single-GPU (level %d)", q);
  const int dim = L.dim, mb = g.mb, mq = L.m_level[q];
  const int nt = (mb + 31) / 32, MP = 32 * nt;
  const int64_t nblk = (int64_t)blocks.size(), n_irr = nblk - ntypes;
  const int nas = (int)(g.amap.size() / mb);
  std::vector<int16_t> alist((size_t)nas * mq, -1);
  for (int d = 0; d < nas; ++d)
    for (int l = 0; l < mb; ++l) {
      const int a = g.amap[(size_t)d * mb + l];
      if (a >= 0) alist[(size_t)d * mq + a] = (int16_t)l;
    }
  Lv.nt = nt;
  Lv.pstride = tile_pack_size(nt);
  Lv.swz = !(getenv("FCM_TILE_SWZ") && atoi(getenv("FCM_TILE_SWZ")) == 0);
  RC(h->alloc(&Lv.type_inv, std::max<int64_t>(ntypes, 1) * mb * mb));
  RC(h->alloc(&Lv.irr_inv, std::max<int64_t>(n_irr, 1) * Lv.pstride));
  RC(h->alloc(&Lv.blk, blk.size()));
  RC(h->alloc(&Lv.irr_anchor, std::max<int64_t>(n_irr, 1)));
  if (!(getenv("FCM_PATCH_DYN") && atoi(getenv("FCM_PATCH_DYN")) == 0)) {
    RC(h->alloc(&Lv.sched, 3));
    CU(cudaMemsetAsync(Lv.sched, 0, 3 * sizeof(unsigned long long), h->stream));
  }
  CU(cudaMemcpyAsync(Lv.blk, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice, h->stream));
  if (n_irr > 0)
    CU(cudaMemcpyAsync(Lv.irr_anchor, blocks.data() + ntypes, n_irr * 8, cudaMemcpyHostToDevice, h->stream));
  // workspace chunk: up to 4 GiB and a quarter of the free memory
  size_t fr = 0, tot = 0;
  CU(cudaMemGetInfo(&fr, &tot));
  const size_t per = (size_t)MP * MP * 8 + (size_t)MP * 8 + (size_t)mb + 16;
  int64_t chunk = (int64_t)std::max<size_t>(1, std::min<size_t>((size_t)4 << 30, fr / 4) / per);
  chunk = std::min<int64_t>(chunk, std::max<int64_t>(nblk, 1));
  double* W = nullptr;
  int64_t* d_anc = nullptr;
  int8_t* d_dir = nullptr;
  int16_t* d_alist = nullptr;
  int* d_status = nullptr;
  double* d_equil = nullptr;
  CU(cudaMallocAsync((void**)&W, (size_t)chunk * MP * MP * 8, h->stream));
  CU(cudaMallocAsync((void**)&d_equil, (size_t)chunk * MP * 8, h->stream));
  CU(cudaMallocAsync((void**)&d_anc, (size_t)chunk * 8, h->stream));
  CU(cudaMallocAsync((void**)&d_dir, (size_t)chunk * mb, h->stream));
  CU(cudaMallocAsync((void**)&d_alist, alist.size() * 2, h->stream));
  CU(cudaMallocAsync((void**)&d_status, (size_t)chunk * 4, h->stream));
  CU(cudaMemcpyAsync(d_alist, alist.data(), alist.size() * 2, cudaMemcpyHostToDevice, h->stream));
  std::vector<int> status(chunk);
  int rc = FCM_OK;
  for (int64_t c0 = 0; c0 < nblk && rc == FCM_OK; ) {
    // types and individual blocks are never mixed in one chunk (different assembly)
    const bool types = c0 < ntypes;
    const int64_t nc = std::min<int64_t>(chunk, (types ? ntypes : nblk) - c0);
    CU(cudaMemcpyAsync(d_anc, blocks.data() + c0, nc * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(d_dir, dir.data() + (size_t)c0 * mb, (size_t)nc * mb, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemsetAsync(W, 0, (size_t)nc * MP * MP * 8, h->stream));
    CU(cudaMemsetAsync(d_status, 0, (size_t)nc * 4, h->stream));
    PatchAsmArgs aa{};
    aa.dim = dim; aa.mb = mb; aa.MP = MP; aa.ldK = L.m;
    aa.nx = L.n[0]; aa.ny = L.n[1]; aa.nz = L.n[2];
    for (int i = 0; i < 3; ++i) aa.na[i] = g.na[i];
    aa.nasm = g.nasm; aa.aoff = g.aoff;
    aa.anchors = d_anc; aa.alist = d_alist; aa.mq = mq; aa.dirich = d_dir;
    aa.kind = types ? nullptr : h->d_kind; aa.cut_idx = h->d_cut_idx;
    aa.Kref = h->d_Kref; aa.cutK = h->d_cutK; aa.alpha = h->alpha; aa.W = W;
    k_patch_asm<<<(unsigned)nc, 256, 0, h->stream>>>(aa);
    CU(cudaGetLastError());
    const int nt64 = (MP + 63) / 64;
    k_equil<<<(unsigned)nc, 256, MP * 8, h->stream>>>(W, MP, d_equil, 0);
    for (int k = 0; k < nt; ++k) {
      k_gj_pivot<<<(unsigned)nc, 256, 0, h->stream>>>(W, MP, k, d_status);
      if (nt > 1) {
        k_gj_row<<<dim3(nt - 1, (unsigned)nc), 256, 0, h->stream>>>(W, MP, k);
        k_gj_update<<<dim3(nt64 * nt64, (unsigned)nc), 256, 0, h->stream>>>(W, MP, k);
        k_gj_col<<<dim3(nt - 1, (unsigned)nc), 256, 0, h->stream>>>(W, MP, k);
      }
    }
    k_equil<<<(unsigned)nc, 256, MP * 8, h->stream>>>(W, MP, d_equil, 1);
    CU(cudaGetLastError());
    if (types) {
      if (MP == mb)
        CU(cudaMemcpyAsync(Lv.type_inv + (size_t)c0 * mb * mb, W, (size_t)nc * mb * mb * 8, cudaMemcpyDeviceToDevice,
                           h->stream));
      else   // one 2D copy per block (rows MP apart in the workspace)
        for (int64_t b = 0; b < nc; ++b)
          CU(cudaMemcpy2DAsync(Lv.type_inv + (size_t)(c0 + b) * mb * mb, (size_t)mb * 8, W + (size_t)b * MP * MP,
                               (size_t)MP * 8, (size_t)mb * 8, (size_t)mb, cudaMemcpyDeviceToDevice, h->stream));
    } else {
      k_pack_tiles<<<dim3(nt * (nt + 1) / 2, (unsigned)nc), 256, 0, h->stream>>>(
          W, MP, nt, Lv.irr_inv + (size_t)(c0 - ntypes) * Lv.pstride, Lv.pstride, Lv.swz ? 1 : 0);
      CU(cudaGetLastError());
    }
    CU(cudaMemcpyAsync(status.data(), d_status, nc * 4, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    for (int64_t b = 0; b < nc; ++b)
      if (status[b]) {
        rc = fail(FCM_ESINGULAR, "singular Schwarz block on level q=%d: %s patch block at anchor %lld", q,
                  types ? "shared-type" : "individual", (long long)blocks[c0 + b]);
        break;
      }
    c0 += nc;
  }
  for (void* ptr : {(void*)W, (void*)d_anc, (void*)d_dir, (void*)d_alist, (void*)d_status, (void*)d_equil})
    cudaFreeAsync(ptr, h->stream);
  CU(cudaStreamSynchronize(h->stream));
  if (rc != FCM_OK) return rc;
  Lv.n_irr = n_irr;
  std::vector<int32_t> reg;
  for (int64_t A = 0; A < (int64_t)blk.size(); ++A)
    if (blk[A] < 0 && blk[A] != kBlkNone && blk[A] != kBlkWb) reg.push_back((int32_t)A);
  if (h->det) {   // deterministic mode: regular patches grouped by vertex colour too
    auto colour = [&](int64_t A) {
      return (int)(A % g.na[0]) % 3 + 3 * ((int)((A / g.na[0]) % g.na[1]) % 3) +
             9 * ((int)(A / ((int64_t)g.na[0] * g.na[1])) % 3);
    };
    std::stable_sort(reg.begin(), reg.end(), [&](int32_t a, int32_t b) { return colour(a) < colour(b); });
    Lv.reg_col.assign(28, 0);
    for (int32_t A : reg) Lv.reg_col[colour(A) + 1]++;
    for (int k = 0; k < 27; ++k) Lv.reg_col[k + 1] += Lv.reg_col[k];
  }
  Lv.n_reg = (int64_t)reg.size();
  RC(h->alloc(&Lv.reg_list, std::max<size_t>(reg.size(), 1)));
  if (!reg.empty()) CU(cudaMemcpyAsync(Lv.reg_list, reg.data(), reg.size() * 4, cudaMemcpyHostToDevice, h->stream));
  RC(h->alloc(&Lv.d_mem, mb));
  RC(h->alloc(&Lv.d_loc, mb));
  CU(cudaMemcpyAsync(Lv.d_mem, g.mem.data(), mb, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.d_loc, g.loc.data(), mb * 2, cudaMemcpyHostToDevice, h->stream));
  Lv.patch = true;
  Lv.mb = mb;
  Lv.nmem = g.nmem;
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 3; ++i) Lv.mo[k][i] = g.mo[k][i];
  for (int i = 0; i < 3; ++i) Lv.na[i] = g.na[i];
  Lv.nanchor = (int64_t)blk.size();
  Lv.has_as = true;
  Lv.n_types = (int32_t)ntypes;
  Lv.blk_h = blk;
  CU(cudaStreamSynchronize(h->stream));
  return FCM_OK;
}

// n symmetric m x m matrices (consecutive at mstride) -> tile-packed (nt tiles per dimension)
static int pack_tiles(fcm_mg* h, const double* A, int m, int64_t mstride, int nt, double* out, int64_t ostride,
                      int64_t n) {
  const int ntiles = nt * (nt + 1) / 2;
  for (int64_t c0 = 0; c0 < n; c0 += 65535) {
    const int64_t cn = std::min<int64_t>(65535, n - c0);
    k_pack_tiles_ld<<<dim3(ntiles, (unsigned)cn), 256, 0, h->stream>>>(A + c0 * mstride, m, mstride, nt,
                                                                        out + c0 * ostride, ostride);
    CU(cudaGetLastError());
  }
  return FCM_OK;
}
static int free_alloc(fcm_mg* h, void* p) {
  auto it = std::find(h->allocs.begin(), h->allocs.end(), p);
  if (it != h->allocs.end()) h->allocs.erase(it);
  CU(cudaFree(p));
  return FCM_OK;
}

// Low-rank patch corrections (patch_wb.cuh): per patch, C = H - H F^{-1} H with G = P_S^T A0^{-1} P_S
// (from the fast-diagonalisation tables), H = G^{-1}, F = H + E, E = sum over the outer ring's
// non-regular cells of (K_c - K_ref) on S.  Host fp64 (OpenMP), k <= kWbMaxK.
static bool chol_inv(int k, std::vector<double>& A) {   // in place: A (SPD, k x k) -> A^{-1}
  std::vector<double> L((size_t)k * k, 0.0);
  for (int j = 0; j < k; ++j) {
    double d = A[(size_t)j * k + j];
    for (int t = 0; t < j; ++t) d -= L[(size_t)j * k + t] * L[(size_t)j * k + t];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double ljj = std::sqrt(d);
    L[(size_t)j * k + j] = ljj;
    for (int i = j + 1; i < k; ++i) {
      double v = A[(size_t)i * k + j];
      for (int t = 0; t < j; ++t) v -= L[(size_t)i * k + t] * L[(size_t)j * k + t];
      L[(size_t)i * k + j] = v / ljj;
    }
  }
  // inv(L) by forward substitution, then A^{-1} = inv(L)^T inv(L)
  std::vector<double> Li((size_t)k * k, 0.0);
  for (int c = 0; c < k; ++c)
    for (int i = c; i < k; ++i) {
      double v = i == c ? 1.0 : 0.0;
      for (int t = c; t < i; ++t) v -= L[(size_t)i * k + t] * Li[(size_t)t * k + c];
      Li[(size_t)i * k + c] = v / L[(size_t)i * k + i];
    }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = 0.0;
      for (int t = i; t < k; ++t) v += Li[(size_t)t * k + i] * Li[(size_t)t * k + j];
      A[(size_t)i * k + j] = A[(size_t)j * k + i] = v;
    }
  return true;
}

static int setup_patch_wb(fcm_mg* h, int q, const BlockGeom& g, const std::vector<int64_t>& wb,
                          const std::vector<std::vector<int16_t>>& wb_S, const std::vector<uint8_t>& kind,
                          const std::vector<int32_t>& cut_idx) {
  LevelDev& Lv = h->lev[q];
  Lv.n_wb = (int64_t)wb.size();
  if (wb.empty()) return FCM_OK;
  const Layout& L = h->L;
  const int dim = L.dim, mb = g.mb, S = 2 * q + 1, m = L.m, TSZ = S * S + S;
  const int N = dim == 3 ? S * S * S : S * S;
  const int nas = (int)(g.amap.size() / mb);
  // tensor slot of every block slot
  std::vector<int16_t> tsl(mb);
  for (int l = 0; l < mb; ++l) {
    int t = 0, mul = 1;
    for (int ax = 0; ax < dim; ++ax) {
      const int k1 = L.modes[g.loc[l]].k[ax], mo = g.mo[g.mem[l]][ax];
      const int sa = k1 >= 2 ? (mo == -1 ? k1 - 1 : q + k1 - 1) : (mo + k1 + 1) * q;
      t += sa * mul;
      mul *= S;
    }
    tsl[l] = (int16_t)t;
  }
  std::vector<int64_t> soff(wb.size() + 1, 0), coff(wb.size() + 1, 0);
  for (size_t p = 0; p < wb.size(); ++p) {
    const int64_t k = (int64_t)wb_S[p].size();
    soff[p + 1] = soff[p] + k;
    coff[p + 1] = coff[p] + k * k;
  }
  std::vector<int16_t> slots(soff.back());
  for (size_t p = 0; p < wb.size(); ++p) std::copy(wb_S[p].begin(), wb_S[p].end(), slots.begin() + soff[p]);
  std::vector<double> Call((size_t)coff.back());
  const int* cls = Lv.fd_cls_h.data();
  const double* tabs = Lv.fd_tabs_h.data();
  const int ncls = Lv.fd_ncls;
  const double sfac = Lv.fd_s, alpha = h->alpha;
  int bad = 0;
  int64_t bad_anchor = -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t p = 0; p < (int64_t)wb.size(); ++p) {
    const int64_t A = wb[p];
    const int ac[3] = {(int)(A % g.na[0]), (int)((A / g.na[0]) % g.na[1]), (int)(A / ((int64_t)g.na[0] * g.na[1]))};
    const std::vector<int16_t>& Sl = wb_S[p];
    const int k = (int)Sl.size();
    const double* tb[3];
    int co = 0;
    for (int ax = 0; ax < 3; ++ax) {
      tb[ax] = tabs + ((size_t)ax * ncls + cls[co + ac[ax]]) * TSZ;
      co += g.na[ax];
    }
    // U[i][mode] = prod_ax T_ax(slot_ax(i), mode_ax) / sqrt(sfac Lambda), G = U U^T
    std::vector<double> U((size_t)k * N);
    for (int i = 0; i < k; ++i) {
      const int t = tsl[Sl[i]];
      const int sx = t % S, sy = (t / S) % S, sz = dim == 3 ? t / (S * S) : 0;
      for (int e = 0; e < N; ++e) {
        const int mx = e % S, my = (e / S) % S, mz = dim == 3 ? e / (S * S) : 0;
        const double lam = tb[0][S * S + mx] + tb[1][S * S + my] + (dim == 3 ? tb[2][S * S + mz] : 0.0);
        double v = tb[0][sx * S + mx] * tb[1][sy * S + my] / std::sqrt(sfac * lam);
        if (dim == 3) v *= tb[2][sz * S + mz];
        U[(size_t)i * N + e] = v;
      }
    }
    std::vector<double> H((size_t)k * k), E((size_t)k * k, 0.0);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j <= i; ++j) {
        double v = 0.0;
        for (int e = 0; e < N; ++e) v += U[(size_t)i * N + e] * U[(size_t)j * N + e];
        H[(size_t)i * k + j] = H[(size_t)j * k + i] = v;   // G
      }
    bool ok = chol_inv(k, H);   // H = G^{-1}
    // E: the outer ring's non-regular cells, (K_c - K_ref) on S
    for (int d = 0; d < nas && ok; ++d) {
      int c3[3] = {ac[0] + g.aoff + d % g.nasm, dim >= 2 ? ac[1] + g.aoff + (d / g.nasm) % g.nasm : 0,
                   dim == 3 ? ac[2] + g.aoff + d / (g.nasm * g.nasm) : 0};
      bool inside = true;
      for (int i = 0; i < 3; ++i) inside = inside && c3[i] >= 0 && c3[i] < (i < dim ? L.n[i] : 1);
      if (!inside) continue;
      const int64_t c = ((int64_t)c3[2] * L.n[1] + c3[1]) * L.n[0] + c3[0];
      const int kd = kind[c];
      if (kd == 0) continue;
      const double* Kc = kd == 2 ? h->cutK_host + (size_t)cut_idx[c] * m * m : nullptr;
      for (int i = 0; i < k; ++i) {
        const int a = g.amap[(size_t)d * mb + Sl[i]];
        if (a < 0) continue;
        for (int j = 0; j < k; ++j) {
          const int b = g.amap[(size_t)d * mb + Sl[j]];
          if (b < 0) continue;
          const double kr = h->Kref_host[(size_t)a * m + b];
          E[(size_t)i * k + j] += (Kc ? Kc[(size_t)a * m + b] : alpha * kr) - kr;
        }
      }
    }
    // F = H + E -> F^{-1};  C = H - H F^{-1} H
    std::vector<double> F((size_t)k * k);
    for (size_t e = 0; e < F.size(); ++e) F[e] = H[e] + E[e];
    ok = ok && chol_inv(k, F);
    if (!ok) {
#pragma omp critical
      { bad = 1; bad_anchor = A; }
      continue;
    }
    std::vector<double> T1((size_t)k * k, 0.0);   // F^{-1} H
    for (int i = 0; i < k; ++i)
      for (int t = 0; t < k; ++t) {
        const double f = F[(size_t)i * k + t];
        for (int j = 0; j < k; ++j) T1[(size_t)i * k + j] += f * H[(size_t)t * k + j];
      }
    double* C = Call.data() + coff[p];
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        double v = 0.0;
        for (int t = 0; t < k; ++t) v += H[(size_t)i * k + t] * T1[(size_t)t * k + j];
        C[(size_t)i * k + j] = H[(size_t)i * k + j] - v;
      }
    for (int i = 0; i < k; ++i)   // symmetrise
      for (int j = 0; j < i; ++j) C[(size_t)i * k + j] = C[(size_t)j * k + i] = 0.5 * (C[(size_t)i * k + j] + C[(size_t)j * k + i]);
  }
  if (bad) return fail(FCM_ESINGULAR, "low-rank patch correction not SPD on level q=%d at anchor %lld", q, (long long)bad_anchor);
  RC(h->alloc(&Lv.wb_anchor, wb.size()));
  RC(h->alloc(&Lv.wb_soff, soff.size()));
  RC(h->alloc(&Lv.wb_slots, std::max<size_t>(slots.size(), 1)));
  RC(h->alloc(&Lv.wb_coff, coff.size()));
  RC(h->alloc(&Lv.wb_C, std::max<size_t>(Call.size(), 1)));
  RC(h->alloc(&Lv.wb_tsl, mb));
  std::vector<int16_t> tS(slots.size());
  for (size_t i = 0; i < slots.size(); ++i) tS[i] = tsl[slots[i]];
  RC(h->alloc(&Lv.wb_tS, std::max<size_t>(tS.size(), 1)));
  CU(cudaMemcpyAsync(Lv.wb_tS, tS.data(), tS.size() * 2, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_anchor, wb.data(), wb.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_soff, soff.data(), soff.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_slots, slots.data(), slots.size() * 2, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_coff, coff.data(), coff.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_C, Call.data(), Call.size() * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.wb_tsl, tsl.data(), mb * 2, cudaMemcpyHostToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  // fused into k_patch_smooth's fast-diagonalisation warps when they stay off the critical path:
  // the explicit patches' stream (at ~6 TB/s) must outlast the FD warps' work (measured ~21.5 ns per
  // 729-slot regular patch per GPU, a low-rank patch ~2.2 of them); level 4 of config 3: 11.8 ms
  // stream vs 8.9 ms FD (x 1.5) -> fused; level 3: 2.3 vs 4.6 ms -> separate (launch lists)
  {
    const double stream_s = (double)Lv.n_irr * Lv.pstride * 8 / 6.0e12;
    const double fd_s = ((double)Lv.n_reg + 2.2 * Lv.n_wb) * 21.5e-9 * N / 729.0;
    // rolled FD passes are slower per patch: with them the low-rank patches go to k_patch_wb (measured)
    Lv.wb_fused = h->wb_mode == 2 || (h->wb_mode == 0 && stream_s > 1.5 * fd_s && !Lv.fd_roll);
  }
  Lv.wb_anchor_h = wb;
  Lv.wb_soff_h = soff;
  Lv.wb_coff_h = coff;
  Lv.wb_slots_h = slots;
  Lv.wb_tsl_h = tsl;
  return FCM_OK;
}

static int setup_schwarz(fcm_mg* h, int q, const std::vector<uint8_t>& kind,
                         const std::vector<int32_t>& cut_idx) {
  const Layout& L = h->L;
  LevelDev& Lv = h->lev[q];
  const int dim = L.dim;
  const int nx = L.n[0], ny = L.n[1], nz = L.n[2];
  const bool patch = q >= 2 && h->prm.block == FCM_BLOCK_PATCH;   // coarse AS is elementwise (R11)
  const BlockGeom g = block_geom(L, q, patch);
  // cell arrays cover the owned cells plus the ghost layers of the slab (single GPU: the grid)
  const int sax = dim - 1;
  int elo[3] = {0, 0, 0}, ene[3] = {nx, ny, nz};
  elo[sax] = h->ext_lo;
  ene[sax] = h->ext_n;
  const int mb = g.mb;
  const int64_t nanchor = (int64_t)g.na[0] * g.na[1] * g.na[2];
  const int nas = (int)(g.amap.size() / std::max(1, mb));
  // classify blocks: regular (every existing assembly cell uncut, one kind) -> shared inverse
  // per boundary type (and 1/alpha scaling for all-fictitious); otherwise individual.
  const int R = patch ? 2 : 1;
  std::vector<int32_t> blk(nanchor);
  std::map<int, int64_t> type_rep;    // type key -> representative anchor
  std::vector<int> key_of(nanchor, -1);
  std::vector<uint8_t> alpha_of(nanchor, 0);
  std::vector<int64_t> irr;
  for (int64_t A = 0; A < nanchor; ++A) {
    int ac[3] = {(int)(A % g.na[0]), (int)((A / g.na[0]) % g.na[1]), (int)(A / ((int64_t)g.na[0] * g.na[1]))};
    bool any = false;
    for (int l = 0; l < mb && !any; ++l) any = block_dof_index(L, q, g, l, ac) >= 0;
    if (!any) { blk[A] = kBlkNone; continue; }
    int k0 = -1;
    bool regular = true;
    for (int d = 0; d < nas && regular; ++d) {
      int c3[3] = {ac[0] + g.aoff + d % g.nasm, dim >= 2 ? ac[1] + g.aoff + (d / g.nasm) % g.nasm : 0,
                   dim == 3 ? ac[2] + g.aoff + d / (g.nasm * g.nasm) : 0};
      bool inside = true;
      for (int i = 0; i < 3; ++i) inside = inside && c3[i] >= elo[i] && c3[i] < elo[i] + ene[i];
      if (!inside) continue;
      const int k = kind[((int64_t)(c3[2] - elo[2]) * ene[1] + (c3[1] - elo[1])) * ene[0] + (c3[0] - elo[0])];
      if (k == 2 || (k0 >= 0 && k != k0)) regular = false;
      k0 = k;
    }
    if (regular) {
      // boundary type: per axis the clipped distances of the anchor to both faces (0 = interior)
      int key = 0, mul = 1;
      for (int i = 0; i < dim; ++i) {
        const int gi = ac[i] + (i == sax ? h->z0 : 0);   // global position along the axis
        const int hiA = patch ? h->g.n[i] : h->g.n[i] - 1;
        const int lo = std::min(gi, R), hi = std::min(hiA - gi, R);
        const int ci = (lo == R && hi == R) ? 0 : 1 + lo * (R + 1) + hi;
        key += ci * mul;
        mul *= (R + 1) * (R + 1) + 1;
      }
      key_of[A] = key;
      alpha_of[A] = k0 == 1;
      if (!type_rep.count(key)) type_rep[key] = A;
    } else {
      blk[A] = (int32_t)irr.size();
      irr.push_back(A);
    }
  }
  // individual patches whose member cells are all uncut and physical: low-rank corrections of the
  // regular patch (patch_wb.cuh), when the level has fast-diagonalisation tables
  std::vector<int64_t> wb;
  std::vector<std::vector<int16_t>> wb_S;
  // levels with small patches keep the explicit inverses: a 125-slot inverse is 63 KB (~13 ns of
  // stream), less than the two fast diagonalisations that replace it (cfg3 level 2: 1.27 ms per sweep
  // explicit vs 1.52 ms low-rank); FCM_PATCH_WB=0 disables, =2 forces every patch level (tests)
  const int wb_env = getenv("FCM_PATCH_WB") ? atoi(getenv("FCM_PATCH_WB")) : 1;
  if (patch && Lv.fd && !h->det && !h->multi && h->cutK_host && h->Kref_host && wb_env != 0 &&
      (wb_env == 2 || mb >= 300)) {
    std::vector<int64_t> keep;
    for (int64_t A : irr) {
      int ac[3] = {(int)(A % g.na[0]), (int)((A / g.na[0]) % g.na[1]), (int)(A / ((int64_t)g.na[0] * g.na[1]))};
      bool inner_ok = true;
      for (int k = 0; k < g.nmem && inner_ok; ++k) {
        int c3[3] = {0, 0, 0};
        bool inside = true;
        for (int i = 0; i < dim; ++i) {
          c3[i] = ac[i] + g.mo[k][i];
          inside = inside && c3[i] >= 0 && c3[i] < L.n[i];
        }
        if (!inside) continue;
        inner_ok = kind[((int64_t)c3[2] * ene[1] + c3[1]) * ene[0] + c3[0]] == 0;
      }
      std::vector<char> touched(mb, 0);
      if (inner_ok)
        for (int d = 0; d < nas; ++d) {
          int c3[3] = {ac[0] + g.aoff + d % g.nasm, dim >= 2 ? ac[1] + g.aoff + (d / g.nasm) % g.nasm : 0,
                       dim == 3 ? ac[2] + g.aoff + d / (g.nasm * g.nasm) : 0};
          bool inside = true;
          for (int i = 0; i < 3; ++i) inside = inside && c3[i] >= 0 && c3[i] < (i < dim ? L.n[i] : 1);
          if (!inside || kind[((int64_t)c3[2] * ene[1] + c3[1]) * ene[0] + c3[0]] == 0) continue;
          for (int l = 0; l < mb; ++l)
            if (g.amap[(size_t)d * mb + l] >= 0 && block_dof_index(L, q, g, l, ac) >= 0) touched[l] = 1;
        }
      std::vector<int16_t> Sl;
      for (int l = 0; l < mb; ++l)
        if (touched[l]) Sl.push_back((int16_t)l);
      if (inner_ok && !Sl.empty() && (int)Sl.size() <= kWbMaxK) {
        blk[A] = kBlkWb;
        wb.push_back(A);
        wb_S.push_back(std::move(Sl));
      } else {
        blk[A] = (int32_t)keep.size();
        keep.push_back(A);
      }
    }
    irr.swap(keep);
  }
  if (patch && h->det) {   // deterministic mode: individual patches grouped by vertex colour (v mod 3)
    auto colour = [&](int64_t A) {
      return (int)(A % g.na[0]) % 3 + 3 * ((int)((A / g.na[0]) % g.na[1]) % 3) +
             9 * ((int)(A / ((int64_t)g.na[0] * g.na[1])) % 3);
    };
    std::stable_sort(irr.begin(), irr.end(), [&](int64_t a, int64_t b) { return colour(a) < colour(b); });
    Lv.irr_col.assign(28, 0);
    for (size_t i = 0; i < irr.size(); ++i) {
      blk[irr[i]] = (int32_t)i;
      Lv.irr_col[colour(irr[i]) + 1]++;
    }
    for (int k = 0; k < 27; ++k) Lv.irr_col[k + 1] += Lv.irr_col[k];
  }
  if (type_rep.size() > 4095) return fail(FCM_EINVAL, "too many Schwarz block types on level %d", q);
  std::map<int, int> slot_of;
  std::vector<int64_t> blocks;   // assembly list: types first (virtual all-physical), then irregular
  std::vector<uint8_t> virt;
  for (auto& kv : type_rep) {
    slot_of[kv.first] = (int)blocks.size();
    blocks.push_back(kv.second);
    virt.push_back(1);
  }
  for (int64_t A = 0; A < nanchor; ++A)
    if (key_of[A] >= 0) blk[A] = -(1 + (slot_of[key_of[A]] | (alpha_of[A] ? (1 << 12) : 0)));
  const int64_t ntypes = (int64_t)blocks.size();
  for (int64_t A : irr) { blocks.push_back(A); virt.push_back(0); }
  const int64_t nblk = (int64_t)blocks.size();
  // absent/Dirichlet flags per block row
  std::vector<int8_t> dir((size_t)nblk * mb);
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t A = blocks[b];
    int ac[3] = {(int)(A % g.na[0]), (int)((A / g.na[0]) % g.na[1]), (int)(A / ((int64_t)g.na[0] * g.na[1]))};
    for (int l = 0; l < mb; ++l) dir[(size_t)b * mb + l] = block_dof_index(L, q, g, l, ac) < 0;
  }
  if (patch) {
    RC(setup_patch_blocks(h, q, g, blk, blocks, ntypes, dir));
    {
      // Rolled FD passes (3 KB of code per patch instead of 20 KB) where the explicit stream dominates
      // the sweep: there the unrolled FD code cycling through the SM's instruction cache costs the
      // streaming warps more than the rolled loop costs the FD warps (cfg3, one box: level 4
      // 15.75 -> 14.83 ms with the low-rank patches in k_patch_wb; levels 3 / 2 are FD-bound and
      // lose 0.3 / 0.2 ms when rolled).  Regular-patch FD work as in the fusion model below.
      LevelDev& Lv = h->lev[q];
      const int64_t N = (int64_t)mb;
      const double stream_s = (double)Lv.n_irr * Lv.pstride * 8 / 6.0e12;
      const double fd_reg_s = (double)Lv.n_reg * 21.5e-9 * N / 729.0;
      Lv.fd_roll = h->fd_roll_mode == 1 || (h->fd_roll_mode < 0 && Lv.fd && stream_s > 2.0 * fd_reg_s);
    }
    return setup_patch_wb(h, q, g, wb, wb_S, kind, cut_idx);
  }
  // device buffers
  int64_t* d_anchors;
  uint8_t* d_virt;
  int16_t* d_amap;
  int8_t* d_dir;
  double* d_mats;
  int* d_status;
  RC(h->alloc(&d_anchors, nblk));
  RC(h->alloc(&d_virt, nblk));
  RC(h->alloc(&d_amap, g.amap.size()));
  RC(h->alloc(&d_dir, (size_t)nblk * mb));
  RC(h->alloc(&d_mats, (size_t)nblk * mb * mb));
  RC(h->alloc(&d_status, nblk));
  RC(h->alloc(&Lv.blk, nanchor));
  CU(cudaMemcpyAsync(d_anchors, blocks.data(), nblk * 8, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(d_virt, virt.data(), nblk, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(d_amap, g.amap.data(), g.amap.size() * 2, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(d_dir, dir.data(), dir.size(), cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(Lv.blk, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice, h->stream));
  BlockAsmArgs aa{};
  aa.nx = nx; aa.ny = ny; aa.nz = nz; aa.dim = dim; aa.mb = mb; aa.ldK = L.m;
  for (int i = 0; i < 3; ++i) { aa.lo[i] = elo[i]; aa.ne[i] = ene[i]; }
  for (int i = 0; i < 3; ++i) aa.na[i] = g.na[i];
  aa.nasm = g.nasm; aa.aoff = g.aoff;
  aa.anchors = d_anchors; aa.virt = d_virt; aa.amap = d_amap; aa.dirich = d_dir;
  aa.kind = h->d_kind_ext; aa.cut_idx = h->d_cut_idx_ext; aa.Kref = h->d_Kref; aa.cutK = h->d_cutK;
  aa.alpha = h->alpha; aa.out = d_mats;
  if (nblk > 0) {
    k_assemble_blocks<<<(unsigned)nblk, kThreads, 0, h->stream>>>(aa);
    CU(cudaGetLastError());
    int max_smem = 0;
    CU(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
    const size_t sm = (size_t)mb * mb * 8 + (size_t)mb * 8;
    if (sm + 64 <= (size_t)max_smem) {
      RC(allow_smem((const void*)k_invert_blocks, sm));
      int nbk = (int)std::min<int64_t>(nblk, (int64_t)h->num_sms * 8);
      k_invert_blocks<<<nbk, kThreads, sm, h->stream>>>(d_mats, mb, d_status, nblk);
    } else {   // large patch blocks: factor in a global scratch, one block per CTA at a time
      int nbk = (int)std::min<int64_t>(nblk, (int64_t)h->num_sms * 2);
      double* scratch = nullptr;
      CU(cudaMallocAsync((void**)&scratch, (size_t)nbk * mb * mb * 8, h->stream));
      k_invert_blocks_global<<<nbk, kThreads, 0, h->stream>>>(d_mats, mb, d_status, nblk, scratch);
      CU(cudaFreeAsync(scratch, h->stream));
    }
    CU(cudaGetLastError());
  }
  std::vector<int> status(nblk);
  CU(cudaMemcpyAsync(status.data(), d_status, nblk * 4, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  for (int64_t b = 0; b < nblk; ++b)
    if (status[b])
      return fail(FCM_ESINGULAR, "singular Schwarz block on level q=%d: %s %s block at anchor %lld", q,
                  b < ntypes ? "shared-type" : "individual", patch ? "patch" : "element",
                  (long long)blocks[b]);
  Lv.type_inv = d_mats;                       // slots 0..ntypes-1
  Lv.irr_inv = d_mats + (size_t)ntypes * mb * mb;
  Lv.n_irr = (int64_t)irr.size();
  if (!patch && Lv.kws && Lv.n_irr > 0) {
    // warp-specialised level: the individual inverses are streamed tile-packed (half the bytes
    // of full storage); the full copies are dropped, the shared types kept
    Lv.irr_tps = tile_pack_size(Lv.ntq);
    RC(h->alloc(&Lv.irr_tp, (size_t)Lv.n_irr * Lv.irr_tps));
    RC(pack_tiles(h, Lv.irr_inv, mb, (int64_t)mb * mb, Lv.ntq, Lv.irr_tp, Lv.irr_tps, Lv.n_irr));
    double* ti = nullptr;
    RC(h->alloc(&ti, (size_t)std::max<int64_t>(ntypes, 1) * mb * mb));
    if (ntypes > 0) CU(cudaMemcpyAsync(ti, d_mats, (size_t)ntypes * mb * mb * 8, cudaMemcpyDeviceToDevice, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    RC(free_alloc(h, d_mats));
    Lv.type_inv = ti;
    Lv.irr_inv = nullptr;
  }
  if (!patch) {
    std::vector<int32_t> il(irr.begin(), irr.end());
    RC(h->alloc(&Lv.irr_list, il.size()));
    CU(cudaMemcpyAsync(Lv.irr_list, il.data(), il.size() * 4, cudaMemcpyHostToDevice, h->stream));
  } else {
    RC(h->alloc(&Lv.d_mem, mb));
    RC(h->alloc(&Lv.d_loc, mb));
    CU(cudaMemcpyAsync(Lv.d_mem, g.mem.data(), mb, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(Lv.d_loc, g.loc.data(), mb * 2, cudaMemcpyHostToDevice, h->stream));
  }
  Lv.patch = patch;
  Lv.mb = mb;
  Lv.nmem = g.nmem;
  for (int k = 0; k < 8; ++k)
    for (int i = 0; i < 3; ++i) Lv.mo[k][i] = g.mo[k][i];
  for (int i = 0; i < 3; ++i) Lv.na[i] = g.na[i];
  Lv.nanchor = nanchor;
  Lv.has_as = true;
  Lv.n_types = (int32_t)ntypes;
  if (Lv.kmma && !patch && mb == Lv.m) {   // MMA groups: 8 regular cells of one type slot
    std::vector<std::vector<int32_t>> by_slot(ntypes);
    for (int64_t A = 0; A < nanchor; ++A)
      if (blk[A] < 0 && blk[A] != kBlkNone) by_slot[(-blk[A] - 1) & 0xfff].push_back((int32_t)A);
    std::vector<int32_t> gc, gm;
    for (int64_t t = 0; t < ntypes; ++t) {
      auto& v = by_slot[t];
      for (size_t i = 0; i < v.size(); i += 8) {
        for (size_t j = 0; j < 8; ++j) gc.push_back(i + j < v.size() ? mma_pack(h, q, v[i + j], ((-blk[v[i + j]] - 1) >> 12) & 1) : -1);
        gm.push_back((int32_t)t);
      }
    }
    Lv.nS = (int64_t)gm.size();
    RC(h->alloc(&Lv.gS_cells, std::max<size_t>(gc.size(), 1)));
    RC(h->alloc(&Lv.gS_mat, std::max<size_t>(gm.size(), 1)));
    if (!gc.empty()) {
      CU(cudaMemcpyAsync(Lv.gS_cells, gc.data(), gc.size() * 4, cudaMemcpyHostToDevice, h->stream));
      CU(cudaMemcpyAsync(Lv.gS_mat, gm.data(), gm.size() * 4, cudaMemcpyHostToDevice, h->stream));
    }
  }
  Lv.blk_h = blk;
  CU(cudaStreamSynchronize(h->stream));
  return FCM_OK;
}

// dense assembled level-1 matrix (host) for the direct coarse solver / Jacobi diagonal
static void coarse_dense(const fcm_mg* h, const std::vector<uint8_t>& kind,
                         const std::vector<int32_t>& cut_idx, const double* K_ref,
                         const double* cut_K, std::vector<double>* dense, std::vector<double>* diag) {
  const Layout& L = h->L;
  const int m1 = L.m_level[1], m = L.m;
  const int64_t n = L.ndof_level[1];
  if (dense) dense->assign((size_t)n * n, 0.0);
  if (diag) diag->assign(n, 0.0);
  std::vector<int64_t> idx(m1);
  for (int64_t c = 0; c < h->ncell; ++c) {
    int cc[3];
    L.cell_coords(c, cc);
    for (int a = 0; a < m1; ++a) idx[a] = L.dof_index(1, a, cc);
    const double* K = kind[c] == 2 ? cut_K + (size_t)cut_idx[c] * m * m : K_ref;
    double s = kind[c] == 1 ? h->alpha : 1.0;
    for (int a = 0; a < m1; ++a) {
      if (idx[a] < 0) continue;
      if (diag) (*diag)[idx[a]] += s * K[(size_t)a * m + a];
      if (dense)
        for (int b = 0; b < m1; ++b)
          if (idx[b] >= 0) (*dense)[(size_t)idx[a] * n + idx[b]] += s * K[(size_t)a * m + b];
    }
  }
}

// Tiled coarse solver (coarse_tiled.cuh): choose the vertex brick that minimises the
// per-SM work (redundant halo evaluation included) such that one brick per SM fits in shared
// memory; leaves h->ktiled null when the level is too large (the grid-wide kernel is used).
static int setup_tiled(fcm_mg* h) {
  const int env = getenv("FCM_COARSE_TILED") ? atoi(getenv("FCM_COARSE_TILED")) : 1;
  if (!env) return FCM_OK;
  const Layout& L = h->L;
  const int dim = L.dim, nf = L.n_f;
  const void* k = tiled_kernel(dim, nf);
  if (!k) return FCM_OK;
  const int NC = 1 << dim, M1 = NC * nf;
  if (L.m_level[1] != M1) return FCM_OK;
  // convention check: local DOF a < M1 is corner a / nf (bit i = offset along axis i), comp a % nf
  TiledArgs t{};
  for (int a = 0; a < M1; ++a) {
    const DofClass& dc = L.classes[L.dof_class[a]];
    if (dc.S != 0 || dc.order != 1 || dc.comp != a % nf) return FCM_OK;
    for (int i = 0; i < dim; ++i)
      if (L.dof_off[a][i] != ((a / nf) >> i & 1)) return FCM_OK;
    const int j = a % nf;
    t.voff[j] = dc.off;
    for (int i = 0; i < 3; ++i) { t.vlo[j][i] = dc.lo[i]; t.vhi[j][i] = dc.hi[i]; }
  }
  if (L.ndof_level[1] >= (1LL << 31)) return FCM_OK;
  int B[3];
  for (int i = 0; i < 3; ++i) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int j = 0; j < nf; ++j) { lo = std::min(lo, t.vlo[j][i]); hi = std::max(hi, t.vhi[j][i]); }
    t.blo[i] = lo;
    B[i] = hi - lo + 1;
    t.n[i] = L.n[i];
  }
  const LevelDev& L1 = h->lev[1];
  const bool jac = h->prm.coarse == FCM_COARSE_JACOBI_PCG;
  // individual matrices per cell (cut-cell operator block + irregular Schwarz inverse), and
  // their 3D prefix sums for box counts
  const int nx = L.n[0], ny = L.n[1], nz = L.n[2];
  std::vector<int> pre((size_t)(nx + 1) * (ny + 1) * (nz + 1), 0);
  auto P = [&](int x, int y, int z) -> int& { return pre[((size_t)z * (ny + 1) + y) * (nx + 1) + x]; };
  {
    std::vector<uint8_t> kind(h->ncell);
    CU(cudaMemcpy(kind.data(), h->d_kind, h->ncell, cudaMemcpyDeviceToHost));
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
          const int64_t c = ((int64_t)z * ny + y) * nx + x;
          const int w = (kind[c] == 2) + ((!jac && L1.blk_h[c] >= 0) ? 1 : 0);
          P(x + 1, y + 1, z + 1) = w + P(x, y + 1, z + 1) + P(x + 1, y, z + 1) + P(x + 1, y + 1, z) -
                                   P(x, y, z + 1) - P(x, y + 1, z) - P(x + 1, y, z) + P(x, y, z);
        }
  }
  auto box_count = [&](int x0, int x1, int y0, int y1, int z0, int z1) {  // inclusive cell box, clipped
    x0 = std::max(x0, 0); y0 = std::max(y0, 0); z0 = std::max(z0, 0);
    x1 = std::min(x1, nx - 1); y1 = std::min(y1, ny - 1); z1 = std::min(z1, nz - 1);
    if (x0 > x1 || y0 > y1 || z0 > z1) return 0;
    ++x1; ++y1; ++z1;
    return P(x1, y1, z1) - P(x0, y1, z1) - P(x1, y0, z1) - P(x1, y1, z0) + P(x0, y0, z1) + P(x0, y1, z0) +
           P(x1, y0, z0) - P(x0, y0, z0);
  };
  const int ntypes = jac ? 0 : L1.n_types;
  int max_smem = 0;
  CU(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  const size_t smem_cap = (size_t)max_smem - 2048;  // static shared memory of the kernel
  // Per-brick cost model (ns per iteration; least-squares fit of the per-brick phase times
  // measured on B200 with FCM_TILED_PROF/FCM_TILED_DUMP over 268 bricks of two partitions of
  // config 2, 5 % rms): smoother rows c_fs (stencil) / c_gs (gather), operator rows c_fo /
  // c_go, c_ind per individual matrix staged, c_upd per E2 entry.  The iteration time is the
  // slowest brick's, so a partition is scored by its maximum brick cost.
  const double c_fs = 1.95, c_gs = 3.2, c_fo = 3.17, c_go = 4.31, c_ind = 2.0, c_upd = 0.17;
  std::vector<uint8_t> kind_h(h->ncell);
  CU(cudaMemcpy(kind_h.data(), h->d_kind, h->ncell, cudaMemcpyDeviceToHost));
  const int B0 = B[0], B1 = B[1], B2 = B[2];
  std::vector<double> PS((size_t)(B0 + 1) * (B1 + 1) * (B2 + 1), 0.0), PO(PS.size(), 0.0);
  auto PI = [&](int x, int y, int z) { return ((size_t)z * (B1 + 1) + y) * (B0 + 1) + x; };
  for (int z = 0; z < B2; ++z)
    for (int y = 0; y < B1; ++y)
      for (int x = 0; x < B0; ++x) {
        const int gv[3] = {t.blo[0] + x, t.blo[1] + y, t.blo[2] + z};
        bool sm = nf == 1 && !jac && ntypes > 0, op = nf == 1;
        int s0 = 0, k0 = -1;
        for (int kc = 0; kc < NC; ++kc) {
          int c3[3] = {0, 0, 0};
          bool ex = true;
          for (int d = 0; d < dim; ++d) {
            c3[d] = gv[d] - ((kc >> d) & 1);
            ex = ex && c3[d] >= 0 && c3[d] < L.n[d];
          }
          if (!ex) { sm = op = false; break; }
          const int64_t c = ((int64_t)c3[2] * ny + c3[1]) * nx + c3[0];
          const int bq = sm ? L1.blk_h[c] : 0, kd = kind_h[c];   // (no Schwarz blocks with Jacobi)
          if (bq >= 0 || bq == kBlkNone || ((-bq - 1) & 0xfff) != 0 || (kc > 0 && bq != s0)) sm = false;
          if (kd == 2 || (kc > 0 && kd != k0)) op = false;
          s0 = bq; k0 = kd;
        }
        const double wsm = nf * (sm ? c_fs : c_gs), wop = nf * (op ? c_fo : c_go);
        PS[PI(x + 1, y + 1, z + 1)] = wsm + PS[PI(x, y + 1, z + 1)] + PS[PI(x + 1, y, z + 1)] + PS[PI(x + 1, y + 1, z)] -
                                      PS[PI(x, y, z + 1)] - PS[PI(x, y + 1, z)] - PS[PI(x + 1, y, z)] + PS[PI(x, y, z)];
        PO[PI(x + 1, y + 1, z + 1)] = wop + PO[PI(x, y + 1, z + 1)] + PO[PI(x + 1, y, z + 1)] + PO[PI(x + 1, y + 1, z)] -
                                      PO[PI(x, y, z + 1)] - PO[PI(x, y + 1, z)] - PO[PI(x + 1, y, z)] + PO[PI(x, y, z)];
      }
  // sum of per-vertex weights over an inclusive local vertex box, clipped to the vertex box
  auto vsum = [&](const std::vector<double>& Pw, const int lo[3], const int hi[3]) {
    int a[3], b[3];
    for (int d = 0; d < 3; ++d) {
      a[d] = std::max(lo[d], 0);
      b[d] = std::min(hi[d], B[d] - 1) + 1;
      if (a[d] >= b[d]) return 0.0;
    }
    return Pw[PI(b[0], b[1], b[2])] - Pw[PI(a[0], b[1], b[2])] - Pw[PI(b[0], a[1], b[2])] - Pw[PI(b[0], b[1], a[2])] +
           Pw[PI(a[0], a[1], b[2])] + Pw[PI(a[0], b[1], a[2])] + Pw[PI(b[0], a[1], a[2])] - Pw[PI(a[0], a[1], a[2])];
  };
  struct Brick { int lo[3], hi[3]; };   // local vertex coordinates, inclusive
  auto brick_cost = [&](const Brick& b) {
    int l1[3], h1[3];
    int64_t e2 = 1;
    for (int d = 0; d < 3; ++d) {
      const bool pr = d < dim;
      l1[d] = b.lo[d] - (pr ? 1 : 0); h1[d] = b.hi[d] + (pr ? 1 : 0);
      e2 *= pr ? b.hi[d] - b.lo[d] + 5 : 1;
    }
    int cl[3], ch[3];   // cell box of the brick
    for (int d = 0; d < 3; ++d) {
      cl[d] = d < dim ? t.blo[d] + b.lo[d] - 2 : 0;
      ch[d] = d < dim ? t.blo[d] + b.hi[d] + 1 : 0;
    }
    return vsum(PS, l1, h1) + vsum(PO, b.lo, b.hi) + c_upd * nf * e2 +
           c_ind * box_count(cl[0], ch[0], cl[1], ch[1], cl[2], ch[2]);
  };
  // shared-memory need of a brick (individual matrices of its cell box counted exactly)
  auto brick_smem = [&](const Brick& b, int* indiv) -> size_t {
    int lo[3], hi[3], ext[3];
    for (int d = 0; d < 3; ++d) {
      if (d < dim) { lo[d] = t.blo[d] + b.lo[d] - 2; hi[d] = t.blo[d] + b.hi[d] + 1; }
      else { lo[d] = 0; hi[d] = 0; }
      ext[d] = d < dim ? b.hi[d] - b.lo[d] + 1 : 1;
    }
    *indiv = box_count(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2]);
    const int E2 = (ext[0] + 4) * (dim > 1 ? ext[1] + 4 : 1) * (dim > 2 ? ext[2] + 4 : 1);
    const int EC = (ext[0] + 3) * (dim > 1 ? ext[1] + 3 : 1) * (dim > 2 ? ext[2] + 3 : 1);
    const int E1 = (ext[0] + 2) * (dim > 1 ? ext[1] + 2 : 1) * (dim > 2 ? ext[2] + 2 : 1);
    if (E2 >= 65536 || EC >= 32768) return SIZE_MAX;   // row-list entries pack (l, cell base) in 16 bits
    return tiled_smem_bytes(dim, nf, E2, E1, EC, ext[0] * ext[1] * ext[2], 1 + ntypes);
  };
  // a partition is feasible when, with the largest individual-matrix count of any brick, every
  // brick fits; returns the dynamic shared memory (0 = infeasible)
  auto part_smem = [&](const std::vector<Brick>& bs, int* max_indiv) -> size_t {
    size_t base = 0;
    int mi = 0;
    for (const Brick& b : bs) {
      int ind = 0;
      const size_t sm = brick_smem(b, &ind);
      if (sm == SIZE_MAX) return 0;
      base = std::max(base, sm);
      mi = std::max(mi, ind);
    }
    const size_t tot = base + (size_t)mi * slot_stride(M1) * 8;
    *max_indiv = mi;
    return tot <= smem_cap ? tot : 0;
  };
  auto part_cost = [&](const std::vector<Brick>& bs) {
    double c = 0.0;
    for (const Brick& b : bs) c = std::max(c, brick_cost(b));
    return c;
  };
  std::vector<Brick> best_bs;
  double best = 1e300;
  size_t best_sm = 0;
  int best_indiv = 0;
  auto consider = [&](std::vector<Brick>&& bs) {
    if (bs.empty() || (int)bs.size() > h->num_sms) return;
    const double c = part_cost(bs);
    if (c >= best) return;
    int mi = 0;
    const size_t sm = part_smem(bs, &mi);
    if (!sm) return;
    best = c; best_sm = sm; best_indiv = mi; best_bs = std::move(bs);
  };
  const char* ft = getenv("FCM_TILE");   // measurement override: "x,y,z" (uniform) or "bisect"
  const bool only_uniform = ft && strcmp(ft, "bisect") != 0, only_bisect = ft && !only_uniform;
  // (a) uniform bricks
  const int tzmax = dim > 2 ? B[2] : 1, tymax = dim > 1 ? B[1] : 1;
  for (int tz = 1; tz <= tzmax && !only_bisect; ++tz)
    for (int ty = 1; ty <= tymax; ++ty)
      for (int tx = 1; tx <= B[0]; ++tx) {
        if (only_uniform) {
          int fx = 0, fy = 1, fz = 1;
          sscanf(ft, "%d,%d,%d", &fx, &fy, &fz);
          if (tx != fx || ty != fy || tz != fz) continue;
        }
        const int tt[3] = {tx, ty, tz};
        const int ntl[3] = {(B[0] + tx - 1) / tx, (B[1] + ty - 1) / ty, (B[2] + tz - 1) / tz};
        if ((int64_t)ntl[0] * ntl[1] * ntl[2] > h->num_sms) continue;
        std::vector<Brick> bs;
        for (int kz = 0; kz < ntl[2]; ++kz)
          for (int ky = 0; ky < ntl[1]; ++ky)
            for (int kx = 0; kx < ntl[0]; ++kx) {
              Brick b;
              const int id[3] = {kx, ky, kz};
              for (int d = 0; d < 3; ++d) { b.lo[d] = id[d] * tt[d]; b.hi[d] = std::min(b.lo[d] + tt[d], B[d]) - 1; }
              bs.push_back(b);
            }
        consider(std::move(bs));
      }
  // (b) recursive bisection balancing the modelled cost (bricks of unequal size where cut
  //     cells make rows expensive); leaf counts up to one brick per SM
  std::function<void(const Brick&, int, std::vector<Brick>&)> bisect = [&](const Brick& b, int nl, std::vector<Brick>& out) {
    if (nl == 1) { out.push_back(b); return; }
    const int na = nl / 2, nb2 = nl - na;
    int ext[3], emax = 0;
    for (int d = 0; d < dim; ++d) { ext[d] = b.hi[d] - b.lo[d] + 1; emax = std::max(emax, ext[d]); }
    double bs = 1e300;
    Brick ba{}, bb{};
    for (int d = 0; d < dim; ++d) {
      if (ext[d] < 2 || 2 * ext[d] < emax) continue;   // split along the longer axes only
      for (int p = b.lo[d] + 1; p <= b.hi[d]; ++p) {
        Brick l = b, r = b;
        l.hi[d] = p - 1; r.lo[d] = p;
        int64_t vl = 1, vr = 1;
        for (int q = 0; q < dim; ++q) { vl *= l.hi[q] - l.lo[q] + 1; vr *= r.hi[q] - r.lo[q] + 1; }
        if (vl < na || vr < nb2) continue;
        const double sc = std::max(brick_cost(l) / na, brick_cost(r) / nb2);
        if (sc < bs) { bs = sc; ba = l; bb = r; }
      }
    }
    if (bs == 1e300) { out.clear(); return; }
    bisect(ba, na, out);
    if (out.empty()) return;
    bisect(bb, nb2, out);
  };
  if (!only_uniform) {
    Brick all{};
    for (int d = 0; d < 3; ++d) { all.lo[d] = 0; all.hi[d] = B[d] - 1; }
    for (int nl = h->num_sms; nl >= std::max(1, h->num_sms / 2); nl -= 4) {
      std::vector<Brick> bs;
      bisect(all, nl, bs);
      consider(std::move(bs));
    }
  }
  if (best_bs.empty()) return FCM_OK;
  if (getenv("FCM_TILED_PROF")) {   // features: fast/gather smoother rows, fast/gather operator rows, E2, indiv
    // (per-row unit weights: rerun the prefix sums with c_fast = 1, c_gen = 0 and vice versa)
    h->t_feat.clear();
    for (const Brick& b : best_bs) {
      int l1[3], h1[3];
      int64_t e2 = 1;
      for (int d = 0; d < 3; ++d) {
        const bool pr = d < dim;
        l1[d] = b.lo[d] - (pr ? 1 : 0); h1[d] = b.hi[d] + (pr ? 1 : 0);
        e2 *= pr ? b.hi[d] - b.lo[d] + 5 : 1;
      }
      const double ssum = vsum(PS, l1, h1), osum = vsum(PO, b.lo, b.hi);
      int64_t n1 = 1, nt = 1;
      for (int d = 0; d < 3; ++d) {
        n1 *= std::min(h1[d], B[d] - 1) - std::max(l1[d], 0) + 1;
        nt *= b.hi[d] - b.lo[d] + 1;
      }
      // rows: fast*c_fast + gen*c_gen = sum, fast + gen = n -> solve for the counts
      const double sg = (ssum - c_fs * n1 * nf) / (c_gs - c_fs), og = (osum - c_fo * nt * nf) / (c_go - c_fo);
      int ind = 0;
      brick_smem(b, &ind);
      for (double v : {n1 * nf - sg, sg, nt * nf - og, og, (double)e2, (double)ind}) h->t_feat.push_back(v);
    }
  }
  const int nb = (int)best_bs.size();
  std::vector<int> bh((size_t)6 * nb);
  for (int i = 0; i < 3; ++i) t.tile[i] = 0;
  for (int b = 0; b < nb; ++b)
    for (int d = 0; d < 3; ++d) {
      bh[6 * b + d] = t.blo[d] + best_bs[b].lo[d];
      bh[6 * b + 3 + d] = best_bs[b].hi[d] - best_bs[b].lo[d] + 1;
      t.tile[d] = std::max(t.tile[d], bh[6 * b + 3 + d]);
    }
  int* d_brick = nullptr;
  RC(h->alloc(&d_brick, bh.size()));
  CU(cudaMemcpy(d_brick, bh.data(), bh.size() * sizeof(int), cudaMemcpyHostToDevice));
  t.brick = d_brick;
  t.max_indiv = best_indiv;
  t.ntypes = ntypes;
  const size_t sm = best_sm;
  RC(allow_smem(k, sm));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTiledThreads, sm));
  if (per_sm < 1 || nb > per_sm * h->num_sms) return FCM_OK;
  t.kind = h->d_kind; t.cut_idx = h->d_cut_idx; t.cutK = h->d_cutK; t.ldK = L.m; t.Kref = h->d_Kref;
  t.alpha = h->alpha;
  t.jacobi = h->prm.coarse == FCM_COARSE_JACOBI_PCG;
  t.diag_inv = h->d_diag_inv;
  t.blk = L1.blk; t.type_inv = L1.type_inv; t.irr_inv = L1.irr_inv; t.inv_alpha = 1.0 / h->alpha;
  // constant-coefficient stencils of the fast path (scalar problems): offsets o(k) = corner
  // bits of local vertex mode k, coefficient of the neighbour at o(k2) - o(kc) (FCM_TILED_FAST=0
  // disables)
  t.fast = 0;
  if (nf == 1 && !(getenv("FCM_TILED_FAST") && atoi(getenv("FCM_TILED_FAST")) == 0)) {
    std::vector<double> K((size_t)L.m * L.m), Mi((size_t)M1 * M1, 0.0);
    CU(cudaStreamSynchronize(h->stream));   // the inverses were computed on the handle's stream
    CU(cudaMemcpy(K.data(), h->d_Kref, K.size() * 8, cudaMemcpyDeviceToHost));
    const bool sm = !t.jacobi && ntypes > 0;
    if (sm) CU(cudaMemcpy(Mi.data(), L1.type_inv, Mi.size() * 8, cudaMemcpyDeviceToHost));
    for (int q = 0; q < 27; ++q) { t.st_op[q] = 0.0; t.st_sm[q] = 0.0; }
    for (int kc = 0; kc < M1; ++kc)
      for (int k2 = 0; k2 < M1; ++k2) {
        int q = 0, mul = 1;
        for (int d = 0; d < dim; ++d, mul *= 3) q += (((k2 >> d) & 1) - ((kc >> d) & 1) + 1) * mul;
        t.st_op[q] += K[(size_t)kc * L.m + k2];
        if (sm) t.st_sm[q] += Mi[(size_t)kc * M1 + k2];
      }
    t.fast = 1;
  }
  const int64_t n1 = L.ndof_level[1];
  RC(h->alloc(&t.wpub[0], n1));
  RC(h->alloc(&t.wpub[1], n1));
  RC(h->alloc(&t.part, (size_t)6 * nb));
  t.acc = nullptr;
  // fp64-atomic dot accumulators (default; FCM_TILED_ATOMIC=0 = block-order partial sums,
  // bit-reproducible run to run, ~0.7 us slower per inner iteration at cfg2)
  if (!h->det && !(getenv("FCM_TILED_ATOMIC") && atoi(getenv("FCM_TILED_ATOMIC")) == 0)) {
    RC(h->alloc(&t.acc, 12));
    CU(cudaMemsetAsync(t.acc, 0, 12 * 8, h->stream));
  }
  RC(h->alloc(&t.ctl, 1));
  CU(cudaMemsetAsync(t.ctl, 0, sizeof(TiledCtl), h->stream));
  t.rtol2 = h->prm.coarse_rtol * h->prm.coarse_rtol;
  t.maxit = h->prm.coarse_maxit;
  t.iters = h->d_coarse_iters;
  if (getenv("FCM_TILED_PROF")) {
    RC(h->alloc(&t.prof, (size_t)4 * nb));
    CU(cudaMemsetAsync(t.prof, 0, (size_t)32 * nb, h->stream));
  }
  if (getenv("FCM_VERBOSE"))
    fprintf(stderr, "[fcm] tiled coarse: box %d x %d x %d, %d bricks (largest %d x %d x %d), modelled max "
            "brick cost %.0f ns/iteration, %d types, <= %d individual matrices per brick, smem %zu B\n",
            B[0], B[1], B[2], nb, t.tile[0], t.tile[1], t.tile[2], best, ntypes, best_indiv, sm);
  h->tiled = t;
  h->ktiled = k;
  h->t_blocks = nb;
  h->t_smem = sm;
  return FCM_OK;
}

static int setup_impl(const fcm_grid* g, const fcm_params* prm, const fcm_slab* slab, const double* K_ref,
                      const uint8_t* cell_kind, double alpha, int64_t n_cut, const int64_t* cut_cells,
                      const double* cut_K, int64_t n_cc, const int64_t* cc_cells, const double* cc_K1,
                      fcm_mg** out) {
  const bool gmg_child = tl_gmg_child;   // an h-level of a parent's GMG coarse solve
  tl_gmg_child = false;
  if (!g || !prm || !K_ref || !cell_kind || !out) return fail(FCM_EINVAL, "NULL argument");
  *out = nullptr;
  int me = fcm_element_size(g);
  if (me < 0) return me;
  if (me > kMaxM) return fail(FCM_EINVAL, "element size m=%d exceeds %d", me, kMaxM);
  if (n_cut < 0 || (n_cut > 0 && (!cut_cells || !cut_K))) return fail(FCM_EINVAL, "bad cut-cell buffers");
  if (!(alpha > 0)) return fail(FCM_EINVAL, "alpha must be > 0");
  if (prm->n_pre < 0 || prm->n_post < 0) return fail(FCM_EINVAL, "negative sweep count");
  if (prm->coarse < 0 || prm->coarse > 3) return fail(FCM_EINVAL, "unknown coarse solver");
  if (prm->block != FCM_BLOCK_ELEMENT && prm->block != FCM_BLOCK_PATCH) return fail(FCM_EINVAL, "unknown block kind %d", prm->block);
  const int dim = g->dim, sax = dim - 1;
  const int nsax = g->n[sax];
  std::unique_ptr<fcm_mg> h(new fcm_mg());
  h->g = *g;
  h->prm = *prm;
  h->alpha = alpha;
  h->gmg_child = gmg_child;
  // blocks per SM of the two k_cell_mma populations; clamped so that one launch never has more
  // blocks than the 2 * kMaxPartials energy partials d_partA/B/C hold (sum_partials reads them all)
  const int bps_cap = std::max(1, (2 * kMaxPartials) / (2 * std::max(1, h->num_sms)));
  if (const char* e = getenv("FCM_MMA_BPS")) h->mma_bps = std::min(bps_cap, std::max(1, atoi(e)));
  if (const char* e = getenv("FCM_LIST_BPS")) h->list_bps = std::min(bps_cap, std::max(1, atoi(e)));
  if (const char* e = getenv("FCM_PDL")) h->pdl = atoi(e) > 0;
  if (slab) {
    if (slab->nranks < 1 || slab->rank < 0 || slab->rank >= slab->nranks || slab->z_begin < 0 ||
        slab->z_end > nsax || slab->z_begin >= slab->z_end)
      return fail(FCM_EINVAL, "bad slab (rank %d of %d, layers [%d, %d))", slab->rank, slab->nranks,
                  slab->z_begin, slab->z_end);
    h->rank = slab->rank; h->nranks = slab->nranks; h->z0 = slab->z_begin; h->z1 = slab->z_end;
    h->multi = h->nranks > 1 || (getenv("FCM_FORCE_SLAB") && atoi(getenv("FCM_FORCE_SLAB")) > 0);
    if (h->nranks > 1 && prm->block == FCM_BLOCK_PATCH)
      return fail(FCM_EINVAL, "patchwise blocks are single-GPU (config 3); use elementwise blocks with slabs");
    if (h->multi && (n_cc < 0 || (n_cc > 0 && (!cc_cells || !cc_K1))))
      return fail(FCM_EINVAL, "slab setup needs every cut cell's leading p=1 block (replicated coarse level)");
  } else {
    h->z0 = 0; h->z1 = nsax;
  }
  h->ustream = (cudaStream_t)prm->stream;
  CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
  CU(cudaEventRecord(h->ev_in, h->ustream));
  CU(cudaStreamWaitEvent(h->stream, h->ev_in, 0));
  if (h->multi) {
    if (!nccl().ok) return fail(FCM_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    if (h->nranks == 1) NC(nccl().GetUniqueId(&id));   // forced slab mode on one rank
    else std::memcpy(&id, slab->nccl_id, sizeof(id));
    NC(nccl().CommInitRank(&h->comm, h->nranks, id, h->rank));
  }
  Layout& L = h->L;
  slab_layout(L, dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces, h->z0, h->z1);
  h->ncell = L.ncell;
  for (int q = 1; q <= g->p; ++q)
    if (L.ndof_level[q] <= 0) return fail(FCM_EINVAL, "level q=%d has no free DOFs (empty level)", q);
  if (h->ncell >= (1LL << 31) || L.ndof_level[g->p] >= (1LL << 31))
    return fail(FCM_EINVAL, "grid too large for 32-bit cell/DOF indexing on one device");
  CU(cudaGetDevice(&h->dev));
  CU(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->dev));
  h->det = getenv("FCM_DETERMINISTIC") && atoi(getenv("FCM_DETERMINISTIC")) > 0;
  if (getenv("FCM_PATCH_PROF") && atoi(getenv("FCM_PATCH_PROF"))) RC(h->alloc(&h->patch_prof, (int64_t)h->num_sms * 4));
  h->fd_roll_mode = getenv("FCM_FD_ROLL") ? atoi(getenv("FCM_FD_ROLL")) : -1;
  h->l2ef = !(getenv("FCM_L2_EVICT_FIRST") && atoi(getenv("FCM_L2_EVICT_FIRST")) == 0);
  if (h->det && h->multi) return fail(FCM_EINVAL, "deterministic mode is single-GPU");
  h->ws_ctas = h->num_sms;
  if (const char* e = getenv("FCM_WS_CTAS")) h->ws_ctas = std::min(h->num_sms, std::max(1, atoi(e)));
  // cells: owned layers [z0, z1) plus one ghost layer on each side that exists
  int64_t plane = 1;
  for (int i = 0; i < sax; ++i) plane *= g->n[i];
  const int zg0 = std::max(h->z0 - 1, 0), zg1 = std::min(h->z1 + 1, nsax);
  h->ext_lo = zg0 - h->z0;
  h->ext_n = zg1 - zg0;
  const int64_t ncell_ext = plane * (zg1 - zg0);
  const int64_t own_off = plane * (h->z0 - zg0);
  const int64_t c_ext0 = plane * zg0;   // global index of the first extended cell
  std::vector<uint8_t> kind(cell_kind + c_ext0, cell_kind + c_ext0 + ncell_ext);
  std::vector<int32_t> cut_idx(ncell_ext, -1);
  h->cut_first = -1;
  int64_t ncut_own = 0;
  for (int64_t i = 0; i < n_cut; ++i) {
    const int64_t c = cut_cells[i] - c_ext0;
    if (c < 0 || c >= ncell_ext || kind[c] != 2)
      return fail(FCM_EINVAL, "cut_cells[%lld] is not a cut cell of the (slab) grid", (long long)i);
    if (i > 0 && cut_cells[i] <= cut_cells[i - 1]) return fail(FCM_EINVAL, "cut_cells must be ascending");
    cut_idx[c] = (int32_t)i;
    if (c >= own_off && c < own_off + h->ncell) {
      if (h->cut_first < 0) h->cut_first = i;
      ++ncut_own;
    }
  }
  if (h->cut_first < 0) h->cut_first = 0;
  for (int64_t c = 0; c < ncell_ext; ++c) {
    if (kind[c] > 2) return fail(FCM_EINVAL, "cell_kind[%lld] = %d", (long long)(c + c_ext0), kind[c]);
    if (kind[c] == 2 && cut_idx[c] < 0) return fail(FCM_EINVAL, "cut cell %lld has no matrix", (long long)(c + c_ext0));
  }
  h->ncut = ncut_own;
  const int m = L.m;
  RC(h->alloc(&h->d_kind_ext, ncell_ext));
  RC(h->alloc(&h->d_cut_idx_ext, ncell_ext));
  h->d_kind = h->d_kind_ext + own_off;
  h->d_cut_idx = h->d_cut_idx_ext + own_off;
  RC(h->alloc(&h->d_Kref, (size_t)m * m));
  RC(h->alloc(&h->d_cutK, (size_t)std::max<int64_t>(n_cut, 1) * m * m));
  CU(cudaMemcpyAsync(h->d_kind_ext, kind.data(), ncell_ext, cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(h->d_cut_idx_ext, cut_idx.data(), ncell_ext * 4, cudaMemcpyHostToDevice, h->stream));
  {
    std::vector<int32_t> cl;
    for (int64_t i = h->cut_first; i < h->cut_first + ncut_own; ++i) cl.push_back((int32_t)(cut_cells[i] - c_ext0 - own_off));
    RC(h->alloc(&h->d_cut_list, cl.size()));
    CU(cudaMemcpyAsync(h->d_cut_list, cl.data(), cl.size() * 4, cudaMemcpyHostToDevice, h->stream));
  }
  CU(cudaMemcpyAsync(h->d_Kref, K_ref, (size_t)m * m * 8, cudaMemcpyHostToDevice, h->stream));
  if (n_cut > 0)
    CU(cudaMemcpyAsync(h->d_cutK, cut_K, (size_t)n_cut * m * m * 8, cudaMemcpyHostToDevice, h->stream));
  // owned-cell views for the host-side helpers (coarse_dense)
  std::vector<uint8_t> kind_own(kind.begin() + own_off, kind.begin() + own_off + h->ncell);
  std::vector<int32_t> cut_idx_own(cut_idx.begin() + own_off, cut_idx.begin() + own_off + h->ncell);
  // levels
  h->lev.assign(g->p + 1, LevelDev());
  int64_t max_plane = 0;
  for (int q = 1; q <= g->p; ++q) {
    LevelDev& Lv = h->lev[q];
    const LevelTable& T = L.tables[q];
    Lv.q = q; Lv.m = T.m; Lv.ndof = T.ndof; Lv.G = group_size(T.m);
    Lv.kreg = reg_kernel(T.m, &Lv.M);
    Lv.ts = Lv.M == 0 ? 1 : split_rt(Lv.M);
    for (int i = 0; i < 3; ++i) {
      Lv.ilo[i] = 0;
      Lv.ihi[i] = L.n[i] - 1;
      for (int a = 0; a < T.m; ++a) {
        Lv.ilo[i] = std::max<int>(Lv.ilo[i], T.cmin[a * 3 + i]);
        Lv.ihi[i] = std::min<int>(Lv.ihi[i], T.cmax[a * 3 + i]);
      }
    }
    Lv.klist = list_kernel(Lv.G);
    if (!(getenv("FCM_CELL_MMA") && atoi(getenv("FCM_CELL_MMA")) == 0)) {
      Lv.kmma = gsz_rt(Lv.m) == Lv.G ? mma_kernel(Lv.m) : nullptr;
      for (int i = 0; i < 3; ++i)
        if (L.n[i] >= 1023) Lv.kmma = nullptr;   // packed coordinates (padding = all ones)
      if (Lv.kmma) {
        RC(allow_smem(Lv.kmma, std::max(mma_smem(Lv.m), list_smem(Lv.m, Lv.G))));
        std::vector<int32_t> gc, gm;
        for (int64_t c = 0; c < h->ncell; ++c)
          if (kind_own[c] != 2) gc.push_back(mma_pack(h.get(), q, c, kind_own[c] == 1));
        while (gc.size() % 8) gc.push_back(-1);
        Lv.nA = (int64_t)gc.size() / 8;
        gm.assign(Lv.nA, -1);
        RC(h->alloc(&Lv.gA_cells, gc.size()));
        RC(h->alloc(&Lv.gA_mat, gm.size()));
        CU(cudaMemcpyAsync(Lv.gA_cells, gc.data(), gc.size() * 4, cudaMemcpyHostToDevice, h->stream));
        CU(cudaMemcpyAsync(Lv.gA_mat, gm.data(), gm.size() * 4, cudaMemcpyHostToDevice, h->stream));
        CU(cudaStreamSynchronize(h->stream));
      }
    }
    if (Lv.kmma && q >= 2 && !h->det && !(getenv("FCM_CELL_WS") && atoi(getenv("FCM_CELL_WS")) == 0)) {
      // measured on config 5 (profiles/r02_s2_ws_variants_cfg5.json): the operator is bound by its
      // MMA warps (12 MMA + 4 streaming warps), the smoother by its streaming warps (8 + 8)
      const char* ev = getenv("FCM_WS_VARIANT");
      for (int mode = 0; mode < 2; ++mode) {
        const int var = ev ? atoi(ev) : (mode == OP_APPLY ? (Lv.m > 32 ? 3 : 2) : (Lv.m > 32 ? 1 : 0));
        Lv.kws_m[mode] = ws_kernel(Lv.m, var, &Lv.ws_threads[mode], &Lv.ws_smem_b[mode]);
        if (Lv.kws_m[mode]) RC(allow_smem(Lv.kws_m[mode], Lv.ws_smem_b[mode]));
      }
      Lv.kws = Lv.kws_m[OP_APPLY];
      if (Lv.kws) Lv.ntq = (Lv.m + 31) / 32;
    }
    if (Lv.kreg) RC(allow_smem(Lv.kreg, level_reg_smem(Lv)));
    RC(allow_smem(Lv.klist, list_smem(Lv.m, Lv.G)));
    Lv.omega = q >= 2 ? prm->omega : 1.0;
    RC(h->alloc(&Lv.base, T.m));
    RC(h->alloc(&Lv.stride, T.m * 3));
    RC(h->alloc(&Lv.cmin, T.m * 3));
    RC(h->alloc(&Lv.cmax, T.m * 3));
    CU(cudaMemcpyAsync(Lv.base, T.base.data(), T.m * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(Lv.stride, T.stride.data(), T.m * 12, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(Lv.cmin, T.cmin.data(), T.m * 6, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(Lv.cmax, T.cmax.data(), T.m * 6, cudaMemcpyHostToDevice, h->stream));
    RC(h->alloc(&Lv.x, Lv.ndof));
    RC(h->alloc(&Lv.r, Lv.ndof));
    if (q >= 2) RC(h->alloc(&Lv.r2, Lv.ndof));
    if (h->multi) {   // interface planes of this level (slab.hpp), exchange order
      std::vector<int32_t> lo, hi;
      if (h->z0 > 0) plane_slots(L, q, 0, lo);
      if (h->z1 < nsax) plane_slots(L, q, h->z1 - h->z0, hi);
      Lv.n_lo = (int64_t)lo.size();
      Lv.n_hi = (int64_t)hi.size();
      RC(h->alloc(&Lv.lo_idx, lo.size()));
      RC(h->alloc(&Lv.hi_idx, hi.size()));
      if (!lo.empty()) CU(cudaMemcpyAsync(Lv.lo_idx, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice, h->stream));
      if (!hi.empty()) CU(cudaMemcpyAsync(Lv.hi_idx, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice, h->stream));
      RC(h->alloc(&Lv.d, Lv.ndof));
      max_plane = std::max<int64_t>(max_plane, Lv.n_lo + Lv.n_hi);
    }
  }
  if (h->multi) {
    RC(h->alloc(&h->x_send, 2 * std::max<int64_t>(max_plane, 1)));
    RC(h->alloc(&h->x_recv, 2 * std::max<int64_t>(max_plane, 1)));
  }
  {   // tile-packed copy of the cut-cell matrices for the warp-specialised levels (cellws.cuh)
    bool any_ws = false;
    for (int q = 2; q <= g->p; ++q) any_ws = any_ws || h->lev[q].kws != nullptr;
    if (any_ws) {
      const int ntf = (m + 31) / 32;
      h->cut_tps = tile_pack_size(ntf);
      RC(h->alloc(&h->d_cutK_tp, (size_t)std::max<int64_t>(n_cut, 1) * h->cut_tps));
      RC(pack_tiles(h.get(), h->d_cutK, m, (int64_t)m * m, ntf, h->d_cutK_tp, h->cut_tps, n_cut));
    }
  }
  h->dist = h->multi && prm->coarse == FCM_COARSE_GMG_PCG;
  h->eager = h->dist;
  // fast-diagonalisation tables first: the Schwarz setup of a patch level uses them for the
  // low-rank individual patches (patch_wb.cuh)
  if (prm->block == FCM_BLOCK_PATCH)
    for (int q = 2; q <= g->p; ++q) RC(setup_patch_fd(h.get(), q, K_ref));
  h->Kref_host = K_ref;
  h->cutK_host = cut_K;
  h->wb_mode = getenv("FCM_WB_KERNEL") ? atoi(getenv("FCM_WB_KERNEL")) : 0;
  for (int q = 1; q <= g->p; ++q)
    if (q >= 2 || ((prm->coarse == FCM_COARSE_AS_PCG || prm->coarse == FCM_COARSE_GMG_PCG) && !h->multi) || h->dist)
      RC(setup_schwarz(h.get(), q, kind, cut_idx));
  h->Kref_host = nullptr;
  h->cutK_host = nullptr;
  for (int q = 2; q <= g->p; ++q)
    if (h->lev[q].patch) {
      if (h->lev[q].n_wb > 0) RC(allow_smem(wb_kernel(2 * q + 1, g->dim), wb_smem_rt(2 * q + 1, g->dim, h->lev[q].mb)));
      if (!h->lev[q].fd) RC(allow_smem((const void*)k_block_smooth, block_smem(h->lev[q].m, h->lev[q].mb)));
      for (int f = 0; f < 3; ++f)
        RC(allow_smem(patch_kernel(2 * q + 1, g->dim, f != 2, f != 1), patch_smem(h.get(), q)));
    }
  RC(h->alloc(&h->d_coarse_iters, 2));
  CU(cudaMemsetAsync(h->d_coarse_iters, 0, 8, h->stream));
  // coarse level
  const int64_t n1 = L.ndof_level[1];
  if (h->multi) {
    // replicated global p = 1 problem: every rank solves it (fcm_slab; no inner-CG traffic)
    fcm_grid g1 = *g;
    g1.p = 1;
    const int m1 = L.m_level[1];
    std::vector<double> K1((size_t)m1 * m1);
    for (int r = 0; r < m1; ++r)
      for (int c = 0; c < m1; ++c) K1[(size_t)r * m1 + c] = K_ref[(size_t)r * m + c];
    fcm_params p1 = *prm;
    p1.stream = (void*)h->stream;
    fcm_mg* hg = nullptr;
    RC(setup_impl(&g1, &p1, nullptr, K1.data(), cell_kind, alpha, n_cc, cc_cells, cc_K1, 0, nullptr,
                  nullptr, &hg));
    h->hg = hg;
    CU(cudaStreamSynchronize(hg->stream));
    CU(cudaStreamDestroy(hg->stream));
    set_stream(hg, h->stream);   // its h-level children too (they borrowed hg's setup stream)
    hg->borrowed_stream = true;
    // all-gather maps: rank j's owned level-1 slots -> global level-1 slots
    Layout Lg;
    Lg.build(dim, g->n, 1, g->space, g->n_f, g->dirichlet_faces);
    std::vector<std::vector<int64_t>> own_glob(h->nranks);
    std::vector<int32_t> pack;
    std::vector<int64_t> extract;
    for (int j = 0; j < h->nranks; ++j) {
      int a0, a1;
      slab_bounds(nsax, h->nranks, j, &a0, &a1);
      Layout Lj;
      slab_layout(Lj, dim, g->n, g->p, g->space, g->n_f, g->dirichlet_faces, a0, a1);
      std::vector<int64_t> gs;
      coarse_global_slots(Lj, Lg, gs);
      std::vector<uint8_t> own;
      owned_mask(Lj, 1, a0 > 0, own);
      for (size_t i = 0; i < gs.size(); ++i)
        if (own[i]) {
          own_glob[j].push_back(gs[i]);
          if (j == h->rank) pack.push_back((int32_t)i);
        }
      if (j == h->rank) {
        if (a0 != h->z0 || a1 != h->z1) return fail(FCM_EINVAL, "slab [%d,%d) is not fcm_slab_bounds' partition", h->z0, h->z1);
        extract = gs;
      }
    }
    h->c_count = (int64_t)pack.size();
    h->c_max = 0;
    for (auto& v : own_glob) h->c_max = std::max<int64_t>(h->c_max, (int64_t)v.size());
    std::vector<int64_t> unpack((size_t)h->nranks * h->c_max, -1);
    for (int j = 0; j < h->nranks; ++j)
      for (size_t i = 0; i < own_glob[j].size(); ++i) unpack[(size_t)j * h->c_max + i] = own_glob[j][i];
    RC(h->alloc(&h->c_pack, pack.size()));
    RC(h->alloc(&h->c_unpack, unpack.size()));
    RC(h->alloc(&h->c_extract, extract.size()));
    RC(h->alloc(&h->c_send, h->c_max));
    RC(h->alloc(&h->c_recv, (size_t)h->nranks * h->c_max));
    RC(h->alloc(&h->c_bg, Lg.ndof_level[1]));
    RC(h->alloc(&h->c_xg, Lg.ndof_level[1]));
    CU(cudaMemcpyAsync(h->c_pack, pack.data(), pack.size() * 4, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(h->c_unpack, unpack.data(), unpack.size() * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(h->c_extract, extract.data(), extract.size() * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemsetAsync(h->c_send, 0, h->c_max * 8, h->stream));
    if (h->dist) {   // distributed coarse CG on the slab (coarse_dist)
      if (hg->gmg.empty()) return fail(FCM_EINVAL, "distributed h-coarsening needs at least one h-level");
      for (int i = 0; i < 4; ++i) RC(h->alloc(&h->c_vec[i], n1));
      RC(h->alloc(&h->d_dcg, 8));
      CU(cudaMemsetAsync(h->d_dcg, 0, 64, h->stream));
      CU(cudaMallocHost((void**)&h->h_dcg, 8 * sizeof(double)));
      CU(cudaMallocHost((void**)&h->h_ci, 2 * sizeof(int)));
      h->h_ci[0] = h->h_ci[1] = 0;
      // owned fine (p = 1) vertex layers [f0, f1] (global); the coarse layers they restrict to
      const int f0 = h->z0 + (h->rank > 0 ? 1 : 0), f1 = h->z1;
      h->dist_cz0 = f0 / 2;
      h->dist_cz1 = (f1 + 1) / 2 + 1;
    }
  } else if (gmg_child) {
    // an h-level of the parent's geometric V-cycle: operator + elementwise AS only
  } else if (prm->coarse == FCM_COARSE_GMG_PCG) {
    RC(setup_gmg(h.get(), K_ref, kind_own, cut_idx_own, cut_K));
  } else if (prm->coarse == FCM_COARSE_DIRECT) {
    if (n1 > 8192) return fail(FCM_EINVAL, "direct coarse solve limited to 8192 DOFs (level 1 has %lld)", (long long)n1);
    std::vector<double> A0;
    coarse_dense(h.get(), kind_own, cut_idx_own, K_ref, cut_K, &A0, nullptr);
    double* fac;
    int* st;
    RC(h->alloc(&h->d_A0inv, (size_t)n1 * n1));
    RC(h->alloc(&fac, (size_t)n1 * n1));
    RC(h->alloc(&st, 1));
    CU(cudaMemcpyAsync(fac, A0.data(), (size_t)n1 * n1 * 8, cudaMemcpyHostToDevice, h->stream));
    k_invert_dense<<<1, 1024, 0, h->stream>>>(fac, n1, h->d_A0inv, st);
    CU(cudaGetLastError());
    int sth = 0;
    CU(cudaMemcpyAsync(&sth, st, 4, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (sth) return fail(FCM_ESINGULAR, "coarse level matrix is singular / not SPD");
  } else {
    if (prm->coarse == FCM_COARSE_JACOBI_PCG) {
      std::vector<double> dg;
      coarse_dense(h.get(), kind_own, cut_idx_own, K_ref, cut_K, nullptr, &dg);
      for (auto& v : dg) v = 1.0 / v;
      RC(h->alloc(&h->d_diag_inv, n1));
      CU(cudaMemcpyAsync(h->d_diag_inv, dg.data(), n1 * 8, cudaMemcpyHostToDevice, h->stream));
    }
    for (int i = 0; i < 9; ++i) RC(h->alloc(&h->c_vec[i], n1));
    RC(h->alloc(&h->c_part, 4 * kMaxPartials));
    RC(h->alloc(&h->c_ctl, 1));
    CU(cudaMemsetAsync(h->c_ctl, 0, sizeof(GridCtl), h->stream));
    // cooperative grid: co-resident blocks
    const LevelDev& L1 = h->lev[1];
    int M1 = 0;
    h->kcoarse = coarse_kernel(L1.m, L1.G, &M1);
    size_t sm = coarse_smem(L1.m, M1, M1 > 0 ? coarse_group(M1) : L1.G);
    RC(allow_smem(h->kcoarse, sm));
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h->kcoarse, kThreads, sm);
    if (e != cudaSuccess || per_sm < 1) return fail(FCM_ECUDA, "coarse kernel occupancy query failed");
    // the cell phases run over ncell cells with up to 32 cells per warp: fill every SM
    int64_t want = std::max<int64_t>(1, std::max<int64_t>((n1 + kThreads - 1) / kThreads, h->ncell / 64));
    h->coarse_blocks = (int)std::min<int64_t>(want, (int64_t)h->num_sms * std::min(per_sm, 4));
    h->coarse_blocks = std::min(h->coarse_blocks, kMaxPartials);
    if (const char* env = getenv("FCM_COARSE_BLOCKS")) {  // tuning knob (co-residency capped)
      int v = atoi(env);
      if (v > 0) h->coarse_blocks = std::min<int64_t>(v, (int64_t)h->num_sms * per_sm);
    }
    RC(setup_tiled(h.get()));
    if (h->det && !h->ktiled)
      return fail(FCM_EINVAL, "deterministic mode: the grid-wide coarse kernel scatters with atomics; use the "
                  "tiled kernel (smaller p=1 level), coarse 'direct' or 'gmg_pcg'");
  }
  // FCG buffers
  const int64_t N = L.ndof_level[g->p];
  RC(h->alloc(&h->f_b, N)); RC(h->alloc(&h->f_x, N)); RC(h->alloc(&h->f_r, N));
  RC(h->alloc(&h->f_ro, N)); RC(h->alloc(&h->f_p, N)); RC(h->alloc(&h->f_q, N));
  RC(h->alloc(&h->d_s, 1));
  RC(h->alloc(&h->d_partA, 2 * kMaxPartials));
  RC(h->alloc(&h->d_partB, 2 * kMaxPartials));
  RC(h->alloc(&h->d_partC, 2 * kMaxPartials));
  if (h->multi) {
    std::vector<uint8_t> own;
    owned_mask(L, g->p, h->z0 > 0, own);
    RC(h->alloc(&h->d_own, own.size()));
    CU(cudaMemcpyAsync(h->d_own, own.data(), own.size(), cudaMemcpyHostToDevice, h->stream));
  }
  CU(cudaMallocHost((void**)&h->h_s, sizeof(Scalars)));
  CU(cudaMallocHost((void**)&h->h_iters, sizeof(int)));
  CU(cudaMemsetAsync(h->d_s, 0, sizeof(Scalars), h->stream));
  CU(cudaStreamSynchronize(h->stream));
  *out = h.release();
  return FCM_OK;
}

extern "C" int fcm_mg_setup(const fcm_grid* g, const fcm_params* prm, const double* K_ref,
                            const uint8_t* cell_kind, double alpha, int64_t n_cut,
                            const int64_t* cut_cells, const double* cut_K, fcm_mg** out) {
  clear_error();
  return setup_impl(g, prm, nullptr, K_ref, cell_kind, alpha, n_cut, cut_cells, cut_K, 0, nullptr, nullptr, out);
}

extern "C" int fcm_mg_setup_slab(const fcm_grid* g, const fcm_params* prm, const fcm_slab* slab,
                                 const double* K_ref, const uint8_t* cell_kind, double alpha,
                                 int64_t n_cut, const int64_t* cut_cells, const double* cut_K,
                                 int64_t n_coarse_cut, const int64_t* coarse_cut_cells,
                                 const double* coarse_cut_K1, fcm_mg** out) {
  clear_error();
  if (!slab) return fail(FCM_EINVAL, "NULL slab");
  return setup_impl(g, prm, slab, K_ref, cell_kind, alpha, n_cut, cut_cells, cut_K, n_coarse_cut,
                    coarse_cut_cells, coarse_cut_K1, out);
}

extern "C" int fcm_nccl_unique_id(void* id128) {
  clear_error();
  if (!id128) return fail(FCM_EINVAL, "NULL argument");
  if (!nccl().ok) return fail(FCM_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NC(nccl().GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return FCM_OK;
}

extern "C" int fcm_mg_destroy(fcm_mg* h) {
  clear_error();
  if (!h) return FCM_OK;
  cudaStreamSynchronize(h->stream);
  delete h;
  return FCM_OK;
}

extern "C" int fcm_mg_nlevels(const fcm_mg* h, int32_t* n) {
  if (!h || !n) return fail(FCM_EINVAL, "NULL argument");
  *n = h->g.p;
  return FCM_OK;
}
extern "C" int fcm_mg_ndofs(const fcm_mg* h, int32_t q, int64_t* n) {
  if (!h || !n || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad level");
  *n = h->L.ndof_level[q];
  return FCM_OK;
}
extern "C" int fcm_mg_level_m(const fcm_mg* h, int32_t q, int32_t* m) {
  if (!h || !m || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad level");
  *m = h->L.m_level[q];
  return FCM_OK;
}
extern "C" int fcm_mg_dof_keys(const fcm_mg* h, int64_t* keys) {
  if (!h || !keys) return fail(FCM_EINVAL, "NULL argument");
  for (int a = 0; a < h->L.dim; ++a)
    if (h->g.n[a] != h->g.n[0]) return fail(FCM_EINVAL, "DOF keys need nx == ny == nz");
  h->L.keys(h->g.p, keys);
  return FCM_OK;
}

extern "C" int fcm_mg_load(fcm_mg* h, const double* f_ref, const double* cut_f,
                           const double* f_traction, int32_t traction_face, double* b) {
  clear_error();
  if (!h || !f_ref || !b || (h->ncut > 0 && !cut_f)) return fail(FCM_EINVAL, "NULL argument");
  StreamGuard sg(h);
  const Layout& L = h->L;
  const int m = L.m, p = L.p;
  std::vector<uint8_t> kind(h->ncell);
  std::vector<int32_t> ci(h->ncell);
  CU(cudaMemcpyAsync(kind.data(), h->d_kind, h->ncell, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaMemcpyAsync(ci.data(), h->d_cut_idx, h->ncell * 4, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  std::vector<double> bh(L.ndof_level[p], 0.0);
  int tax = traction_face >= 0 ? traction_face / 2 : -1, tside = traction_face % 2;
  const int sax = L.dim - 1;
  for (int64_t c = 0; c < h->ncell; ++c) {
    int cc[3];
    L.cell_coords(c, cc);
    const double* f = kind[c] == 2 ? cut_f + (size_t)ci[c] * m : f_ref;
    double s = kind[c] == 1 ? h->alpha : 1.0;
    const int ct = tax >= 0 ? cc[tax] + (tax == sax ? h->z0 : 0) : 0;   // global coordinate
    bool tr = f_traction && tax >= 0 && ct == (tside ? h->g.n[tax] - 1 : 0);
    for (int a = 0; a < m; ++a) {
      int64_t i = L.dof_index(p, a, cc);
      if (i < 0) continue;
      bh[i] += s * f[a] + (tr ? f_traction[a] : 0.0);
    }
  }
  CU(cudaMemcpyAsync(b, bh.data(), bh.size() * 8, cudaMemcpyHostToDevice, h->stream));
  RC(exchange(h, p, b));   // slab mode: interface planes hold both ranks' contributions
  CU(cudaStreamSynchronize(h->stream));
  return FCM_OK;
}

extern "C" int fcm_apply(fcm_mg* h, int32_t q, const double* x, double* y) {
  clear_error();
  if (!h || !x || !y || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad argument");
  StreamGuard sg(h);
  return apply_op(h, q, x, y, nullptr);
}

extern "C" int fcm_mg_smooth(fcm_mg* h, int32_t q, const double* r, double* x) {
  clear_error();
  if (!h || !r || !x || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad argument");
  if (!h->lev[q].has_as) return fail(FCM_EINVAL, "level q=%d has no Schwarz smoother", q);
  StreamGuard sg(h);
  return smooth(h, q, r, x);
}

extern "C" int fcm_mg_smooth_part(fcm_mg* h, int32_t q, int32_t part, const double* r, double* x) {
  clear_error();
  if (!h || !r || !x || q < 1 || q > h->g.p || part < 0 || part > 2) return fail(FCM_EINVAL, "bad argument");
  if (!h->lev[q].has_as) return fail(FCM_EINVAL, "level q=%d has no Schwarz smoother", q);
  if (part == 0) return fcm_mg_smooth(h, q, r, x);
  if (!h->lev[q].patch || h->multi) return fail(FCM_EINVAL, "smoother parts exist on patchwise levels only");
  StreamGuard sg(h);
  return launch_block_smooth(h, q, r, x, h->lev[q].omega, part);
}

extern "C" int fcm_mg_coarse_solve(fcm_mg* h, const double* r, double* x, int32_t* iters) {
  clear_error();
  if (!h || !r || !x) return fail(FCM_EINVAL, "NULL argument");
  StreamGuard sg(h);
  if (h->prm.coarse == FCM_COARSE_GMG_PCG && !h->hg) {   // nested conditional nodes: graph only
    RC(capture(h, &h->g_coarse, &h->n_coarse_g, [&]() { return enqueue_coarse_gmg(h, h->c_bst, h->c_xst); }));
    CU(cudaMemcpyAsync(h->c_bst, r, h->lev[1].ndof * 8, cudaMemcpyDeviceToDevice, h->stream));
    RC(run_graph(h, h->g_coarse, h->n_coarse_g));
    CU(cudaMemcpyAsync(x, h->c_xst, h->lev[1].ndof * 8, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    RC(enqueue_coarse(h, r, x));
  }
  if (iters) {
    if (h->prm.coarse == FCM_COARSE_DIRECT) *iters = 0;
    else {
      const fcm_mg* hc = h->hg ? h->hg : h;   // slab mode: the replicated coarse handle counts
      CU(cudaMemcpyAsync(h->h_iters, hc->d_coarse_iters, 4, cudaMemcpyDeviceToHost, h->stream));
      CU(cudaStreamSynchronize(h->stream));
      *iters = *h->h_iters;
      if (hc->ktiled && hc->tiled.prof && !h->hg) {   // FCM_TILED_PROF: mean phase times per iteration
        std::vector<unsigned long long> pr((size_t)4 * h->t_blocks);
        CU(cudaMemcpy(pr.data(), h->tiled.prof, pr.size() * 8, cudaMemcpyDeviceToHost));
        double mx[4] = {0, 0, 0, 0}, mean[4] = {0, 0, 0, 0};
        for (int b = 0; b < h->t_blocks; ++b)
          for (int k = 0; k < 4; ++k) {
            mx[k] = std::max(mx[k], (double)pr[4 * b + k]);
            mean[k] += (double)pr[4 * b + k] / h->t_blocks;
          }
        fprintf(stderr, "[fcm] tiled phases (ns, summed over solves; mean/max over blocks): update %.0f/%.0f "
                "smooth %.0f/%.0f apply %.0f/%.0f allreduce %.0f/%.0f\n", mean[0], mx[0], mean[1], mx[1],
                mean[2], mx[2], mean[3], mx[3]);
        std::vector<std::pair<double, int>> w(h->t_blocks);
        for (int b = 0; b < h->t_blocks; ++b) w[b] = {(double)(pr[4 * b + 1] + pr[4 * b + 2]), b};
        std::sort(w.begin(), w.end());
        fprintf(stderr, "[fcm] smooth+apply per block: min %.0f median %.0f; top:", w[0].first, w[w.size() / 2].first);
        for (int k = 0; k < 8 && k < (int)w.size(); ++k)
          fprintf(stderr, " %d:%.0f", w[w.size() - 1 - k].second, w[w.size() - 1 - k].first);
        fprintf(stderr, "\n");
        if (getenv("FCM_TILED_DUMP"))
          for (int b = 0; b < h->t_blocks && (size_t)(6 * b + 5) < h->t_feat.size(); ++b)
            fprintf(stderr, "[fcm] brick %d feat %.0f %.0f %.0f %.0f %.0f %.0f time %llu %llu %llu %llu\n", b,
                    h->t_feat[6 * b], h->t_feat[6 * b + 1], h->t_feat[6 * b + 2], h->t_feat[6 * b + 3],
                    h->t_feat[6 * b + 4], h->t_feat[6 * b + 5], pr[4 * b], pr[4 * b + 1], pr[4 * b + 2], pr[4 * b + 3]);
        CU(cudaMemset(h->tiled.prof, 0, pr.size() * 8));
      }
    }
  }
  return FCM_OK;
}

static int capture_vcycle(fcm_mg* h) {
  const int p = h->g.p;
  return capture(h, &h->g_vc, &h->n_vc, [=]() { return enqueue_vcycle(h, p, h->f_r, h->lev[p].x); });
}

extern "C" int fcm_mg_vcycle(fcm_mg* h, const double* r, double* z) {
  clear_error();
  if (!h || !r || !z) return fail(FCM_EINVAL, "NULL argument");
  StreamGuard sg(h);
  const int p = h->g.p;
  const int64_t N = h->lev[p].ndof;
  RC(capture_vcycle(h));
  CU(cudaMemcpyAsync(h->f_r, r, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  RC(run_graph(h, h->g_vc, h->n_vc));
  CU(cudaMemcpyAsync(z, h->lev[p].x, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  h->stat_vcycles++;
  return FCM_OK;
}

static int capture_fcg(fcm_mg* h) {
  const int p = h->g.p;
  const int64_t N = h->lev[p].ndof;
  double* z = h->lev[p].x;
  const int nbd = dot_blocks(h);
  const int nbc = cellop_nblocks(h, p, OP_APPLY);
  // slab mode: partial sums are finalised on each rank, all-reduced, and the update kernels
  // read the reduced scalars (red[]); dots skip the interface DOFs this rank does not own
  const bool slab = h->multi;
  const uint8_t* own = slab ? h->d_own : nullptr;
  double* red = h->d_s->red;
  // init: x = 0, r = b, z = V(r), rz = z.r, p = z
  auto init_body = [=]() -> int {
    k_fcg_start<<<grid_for(N, h->num_sms), kThreads, 0, h->stream>>>(h->f_x, h->f_r, h->f_b, N);
    h->count();
    RC(enqueue_vcycle(h, p, h->f_r, z));
    CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), z, h->f_r, N, h->d_partA, own));
    h->count();
    if (slab) {
      CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), red + 3, h->d_partA, nbd));
      h->count();
      RC(allreduce(h, red + 3, 1));
    }
    k_fcg_start2<<<grid_for(N, h->num_sms), kThreads, 0, h->stream>>>(h->d_s, h->d_partA, nbd, h->f_p, z, N,
                                                                      slab ? red + 3 : nullptr);
    h->count();
    CU(cudaGetLastError());
    return FCM_OK;
  };
  // iteration part 1: q = A p (energy partials pq), update x, r, r_old, rr
  auto it1_body = [=](bool d2h) -> int {
    RC(fill(h, h->f_q, 0.0, N));
    RC(launch_cellop(h, p, make_op(h, p, OP_APPLY, h->f_p, h->f_q, 1.0, h->d_partB)));
    RC(exchange(h, p, h->f_q));
    if (slab) {
      CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), red, h->d_partB, nbc));
      h->count();
      RC(allreduce(h, red, 1));
    }
    CU(pdl_launch(h, k_fcg_update1, dim3(nbd), dim3(kThreads), h->d_s, h->d_partB, nbc, h->f_x, h->f_r, h->f_ro,
                                                    h->f_p, h->f_q, N, h->d_partC, own, slab ? red : nullptr));
    h->count();
    CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), &h->d_s->rr, h->d_partC, nbd));
    h->count();
    CU(cudaGetLastError());
    if (slab) RC(allreduce(h, &h->d_s->rr, 1));
    if (d2h) CU(cudaMemcpyAsync(h->h_s, h->d_s, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
    return FCM_OK;
  };
  // iteration part 2: z = V(r), beta, p = z + beta p
  auto it2_body = [=]() -> int {
    RC(enqueue_vcycle(h, p, h->f_r, z));
    CU(pdl_launch(h, k_dot2, dim3(nbd), dim3(kThreads), z, h->f_r, h->f_ro, N, h->d_partA, h->d_partB, own));
    h->count();
    if (slab) {
      CU(pdl_launch(h, k_finalize2, dim3(1), dim3(32), red + 1, h->d_partA, h->d_partB, nbd));
      h->count();
      RC(allreduce(h, red + 1, 2));
    }
    CU(pdl_launch(h, k_fcg_update2, dim3(grid_for(N, h->num_sms)), dim3(kThreads), h->d_s, h->d_partA, h->d_partB, nbd, h->f_p, z, N,
                                                                       slab ? red + 1 : nullptr));
    h->count();
    CU(pdl_launch(h, k_set_rz, dim3(1), dim3(32), h->d_s));
    h->count();
    CU(cudaGetLastError());
    return FCM_OK;
  };
  RC(capture(h, &h->g_init, &h->n_init, init_body));
  RC(capture(h, &h->g_it1, &h->n_it1, [=]() { return it1_body(true); }));
  RC(capture(h, &h->g_it2, &h->n_it2, it2_body));
  // the whole solve as ONE graph with a device-side WHILE loop (conditional node): no host
  // round trip per iteration (FCM_HOST_LOOP=1 keeps the per-iteration host loop)
  // (slab mode keeps the host loop: NCCL work is not placed inside conditional bodies)
  if (!h->g_solve && !h->multi && !(getenv("FCM_HOST_LOOP") && atoi(getenv("FCM_HOST_LOOP")) > 0)) {
    cudaGraph_t G, body;
    CU(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle cond;
    CU(cudaGraphConditionalHandleCreate(&cond, G, 1, cudaGraphCondAssignDefault));
    int64_t nk = 0;
    h->count_target = &nk;
    CU(cudaStreamBeginCaptureToGraph(h->stream, G, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    int rc = init_body();
    if (rc >= 0) rc = it1_body(false);
    if (rc >= 0) {
      k_fcg_check<<<1, 32, 0, h->stream>>>(h->d_s, cond, h->d_hist);
      h->count();
    }
    cudaGraphNode_t wnode = nullptr;
    if (rc >= 0) {
      cudaStreamCaptureStatus st;
      cudaGraph_t cg_;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      cudaError_t e = cudaStreamGetCaptureInfo_v3(h->stream, &st, nullptr, &cg_, &deps, nullptr, &ndeps);
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = cond;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      if (e == cudaSuccess) e = cudaGraphAddNode(&wnode, G, deps, ndeps, &cp);
      if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(h->stream, &wnode, 1, cudaStreamSetCaptureDependencies);
      if (e != cudaSuccess) rc = fail(FCM_ECUDA, "conditional node: %s", cudaGetErrorString(e));
      body = cp.conditional.phGraph_out[0];
    }
    cudaGraph_t Gout;
    cudaError_t e = cudaStreamEndCapture(h->stream, &Gout);
    h->n_head = nk;
    if (rc >= 0 && e == cudaSuccess) {
      nk = 0;
      CU(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      rc = it2_body();
      if (rc >= 0) rc = it1_body(false);
      if (rc >= 0) {
        k_fcg_check<<<1, 32, 0, h->stream>>>(h->d_s, cond, h->d_hist);
        h->count();
      }
      cudaGraph_t bout;
      e = cudaStreamEndCapture(h->stream, &bout);
      h->n_loop = nk;
    }
    h->count_target = nullptr;
    if (rc >= 0 && e == cudaSuccess) e = cudaGraphInstantiate(&h->g_solve, G, 0);
    cudaGraphDestroy(G);
    if (rc < 0) return rc;
    if (e != cudaSuccess) return fail(FCM_ECUDA, "device-loop graph: %s", cudaGetErrorString(e));
  }
  return FCM_OK;
}

static int pcg_core(fcm_mg* h, double rtol, int32_t maxit, int32_t* iters, double* hist) {
  const int p = h->g.p;
  const int64_t N = h->lev[p].ndof;
  if (maxit + 2 > h->hist_cap) {   // device history buffer (baked into the device-loop graph)
    if (h->g_solve) { cudaGraphExecDestroy(h->g_solve); h->g_solve = nullptr; }
    h->hist_cap = std::max(maxit + 2, 512);
    RC(h->alloc(&h->d_hist, h->hist_cap));
  }
  RC(capture_fcg(h));
  // ||b||^2
  const int nbd = dot_blocks(h);
  CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), h->f_b, h->f_b, N, h->d_partA, h->multi ? h->d_own : nullptr));
  CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), &h->d_s->bb, h->d_partA, nbd));
  h->count(2);
  RC(allreduce(h, &h->d_s->bb, 1));
  CU(cudaMemsetAsync(&h->d_s->flag, 0, sizeof(int), h->stream));
  CU(cudaMemcpyAsync(h->h_s, h->d_s, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  const double bb = h->h_s->bb;
  int it = 0;
  if (hist) hist[0] = bb > 0 ? 1.0 : 0.0;
  h->stat_coarse = 0;
  CU(cudaMemsetAsync((h->hg ? h->hg : h)->d_coarse_iters, 0, 8, h->stream));
  if (h->h_ci) h->h_ci[0] = h->h_ci[1] = 0;
  h->stat_vcycles = 0;
  if (!(bb > 0) || maxit == 0) {   // b = 0: x = 0 (R6); maxit = 0: no x-update, x = x0 = 0
    RC(fill(h, h->f_x, 0.0, N));
    if (iters) *iters = 0;
    return bb > 0 ? FCM_NOT_CONVERGED : FCM_OK;
  }
  if (h->g_solve) {   // one graph launch, one synchronisation
    h->h_s->it = 0;
    h->h_s->maxit = maxit;
    h->h_s->rtol2 = rtol * rtol;
    CU(cudaMemcpyAsync(&h->d_s->it, &h->h_s->it, sizeof(int) * 2 + sizeof(double), cudaMemcpyHostToDevice, h->stream));
    CU(cudaGraphLaunch(h->g_solve, h->stream));
    CU(cudaMemcpyAsync(h->h_s, h->d_s, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    const Scalars s = *h->h_s;
    it = s.it;
    h->launches += h->n_head + (int64_t)(it - 1) * h->n_loop;
    if (h->prm.coarse == FCM_COARSE_GMG_PCG && h->n_gcg_body > 0) {   // coarse CG trips beyond the first
      int ci[2] = {0, 0};
      CU(cudaMemcpy(ci, h->d_coarse_iters, 8, cudaMemcpyDeviceToHost));
      h->launches += std::max<int64_t>(0, ci[1] - it) * h->n_gcg_body;
    }
    h->stat_vcycles = it;
    if (hist && it > 0) {
      std::vector<double> hh(it + 1);
      CU(cudaMemcpy(hh.data(), h->d_hist, (it + 1) * sizeof(double), cudaMemcpyDeviceToHost));
      for (int i = 1; i <= it; ++i) hist[i] = hh[i];
    }
    if (iters) *iters = it;
    if (s.flag & 1) return fail(FCM_EINDEF, "p^T A p <= 0 at FCG iteration %d", it);
    const double rel = std::sqrt(s.rr / bb);
    if (!(rel == rel)) return fail(FCM_EINDEF, "NaN residual at FCG iteration %d", it);
    return rel < rtol ? FCM_OK : FCM_NOT_CONVERGED;
  }
  RC(run_graph(h, h->g_init, h->n_init));
  h->stat_vcycles++;
  int status = FCM_OK;
  while (true) {
    RC(run_graph(h, h->g_it1, h->n_it1));
    CU(cudaStreamSynchronize(h->stream));
    ++it;
    const Scalars s = *h->h_s;
    if (s.flag & 1) return fail(FCM_EINDEF, "p^T A p <= 0 at FCG iteration %d", it);
    const double rel = std::sqrt(s.rr / bb);
    if (hist) hist[it] = rel;
    if (!(rel == rel)) return fail(FCM_EINDEF, "NaN residual at FCG iteration %d", it);
    if (rel < rtol) break;
    if (it >= maxit) { status = FCM_NOT_CONVERGED; break; }
    RC(run_graph(h, h->g_it2, h->n_it2));
    h->stat_vcycles++;
  }
  if (iters) *iters = it;
  return status;
}

extern "C" int fcm_pcg_solve(fcm_mg* h, const double* b, double* x, double rtol, int32_t maxit,
                             int32_t* iters, double* relres_hist) {
  clear_error();
  if (!h || !b || !x || maxit < 0) return fail(FCM_EINVAL, "bad argument");
  StreamGuard sg(h);
  const int64_t N = h->lev[h->g.p].ndof;
  CU(cudaMemcpyAsync(h->f_b, b, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  int rc = pcg_core(h, rtol, maxit, iters, relres_hist);
  if (rc < 0) return rc;
  CU(cudaMemcpyAsync(x, h->f_x, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return rc;
}

extern "C" int fcm_pcg_solve_host(fcm_mg* h, const double* b_host, double* x_host, double rtol,
                                  int32_t maxit, int32_t* iters, double* relres_hist) {
  clear_error();
  if (!h || !b_host || !x_host || maxit < 0) return fail(FCM_EINVAL, "bad argument");
  StreamGuard sg(h);
  const int64_t N = h->lev[h->g.p].ndof;
  CU(cudaMemcpyAsync(h->f_b, b_host, N * 8, cudaMemcpyHostToDevice, h->stream));
  int rc = pcg_core(h, rtol, maxit, iters, relres_hist);
  if (rc < 0) return rc;
  CU(cudaMemcpyAsync(x_host, h->f_x, N * 8, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return rc;
}

// Multigrid as a stand-alone solver: x_i = x_{i-1} + V(b - A x_{i-1}).
// One graph per iteration: V-cycle on r, x += z, r = b - A x, rr = r.r (owned DOFs, summed
// over ranks), Scalars to the host; the host checks ||r_i||/||b|| (one sync per V-cycle).
static int mg_solve_core(fcm_mg* h, double rtol, int32_t maxit, int32_t* iters, double* hist) {
  const int p = h->g.p;
  const int64_t N = h->lev[p].ndof;
  double* z = h->lev[p].x;
  const int nbd = dot_blocks(h);
  const uint8_t* own = h->multi ? h->d_own : nullptr;
  if (!h->g_mgit) {
    RC(capture(h, &h->g_mgit, &h->n_mgit, [=]() -> int {
      RC(enqueue_vcycle(h, p, h->f_r, z));
      k_axpy<<<grid_for(N, h->num_sms), kThreads, 0, h->stream>>>(h->f_x, 1.0, z, N);
      h->count();
      RC(residual(h, p, h->f_b, h->f_x, h->f_r));
      CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), h->f_r, h->f_r, N, h->d_partA, own));
      CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), &h->d_s->rr, h->d_partA, nbd));
      h->count(2);
      CU(cudaGetLastError());
      RC(allreduce(h, &h->d_s->rr, 1));
      CU(cudaMemcpyAsync(h->h_s, h->d_s, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
      return FCM_OK;
    }));
  }
  CU(pdl_launch(h, k_dot, dim3(nbd), dim3(kThreads), h->f_b, h->f_b, N, h->d_partA, own));
  CU(pdl_launch(h, k_finalize, dim3(1), dim3(32), &h->d_s->bb, h->d_partA, nbd));
  h->count(2);
  RC(allreduce(h, &h->d_s->bb, 1));
  CU(cudaMemcpyAsync(h->h_s, h->d_s, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
  RC(fill(h, h->f_x, 0.0, N));
  RC(copy(h, h->f_r, h->f_b, N));   // r_0 = b (x_0 = 0)
  CU(cudaMemsetAsync((h->hg ? h->hg : h)->d_coarse_iters, 0, 8, h->stream));
  if (h->h_ci) h->h_ci[0] = h->h_ci[1] = 0;
  CU(cudaStreamSynchronize(h->stream));
  const double bb = h->h_s->bb;
  h->stat_coarse = 0;
  h->stat_vcycles = 0;
  int it = 0;
  if (hist) hist[0] = bb > 0 ? 1.0 : 0.0;
  int status = FCM_OK;
  if (bb > 0) {
    while (true) {
      if (it >= maxit) { status = FCM_NOT_CONVERGED; break; }
      RC(run_graph(h, h->g_mgit, h->n_mgit));
      CU(cudaStreamSynchronize(h->stream));
      ++it;
      h->stat_vcycles++;
      const double rel = std::sqrt(h->h_s->rr / bb);
      if (hist) hist[it] = rel;
      if (!(rel == rel)) return fail(FCM_EINDEF, "NaN residual at MG iteration %d", it);
      if (rel < rtol) break;
    }
  }
  if (iters) *iters = it;
  return status;
}

extern "C" int fcm_mg_solve(fcm_mg* h, const double* b, double* x, double rtol, int32_t maxit,
                            int32_t* iters, double* relres_hist) {
  clear_error();
  if (!h || !b || !x || maxit < 0) return fail(FCM_EINVAL, "bad argument");
  StreamGuard sg(h);
  const int64_t N = h->lev[h->g.p].ndof;
  CU(cudaMemcpyAsync(h->f_b, b, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  int rc = mg_solve_core(h, rtol, maxit, iters, relres_hist);
  if (rc < 0) return rc;
  CU(cudaMemcpyAsync(x, h->f_x, N * 8, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return rc;
}

extern "C" int fcm_mg_stats(const fcm_mg* h, int64_t* coarse_iters_total, int64_t* vcycles) {
  if (!h) return fail(FCM_EINVAL, "NULL handle");
  if (coarse_iters_total) {
    int v[2] = {0, 0};
    CU(cudaMemcpyAsync(v, (h->hg ? h->hg : h)->d_coarse_iters, 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    *coarse_iters_total = v[1];
  }
  if (vcycles) *vcycles = h->stat_vcycles;
  return FCM_OK;
}

extern "C" int fcm_mg_coarse_info(const fcm_mg* h, int32_t* kind, int32_t* blocks, int32_t* tile) {
  if (!h || !kind || !blocks) return fail(FCM_EINVAL, "NULL argument");
  if (h->hg) return fcm_mg_coarse_info(h->hg, kind, blocks, tile);
  if (h->prm.coarse == FCM_COARSE_DIRECT) { *kind = FCM_COARSE_KERNEL_DIRECT; *blocks = 0; }
  else if (h->prm.coarse == FCM_COARSE_GMG_PCG) { *kind = FCM_COARSE_KERNEL_GMG; *blocks = (int32_t)h->gmg.size(); }
  else if (h->ktiled) { *kind = FCM_COARSE_KERNEL_TILED; *blocks = h->t_blocks; }
  else { *kind = FCM_COARSE_KERNEL_GRID; *blocks = h->coarse_blocks; }
  if (tile)
    for (int i = 0; i < 3; ++i) tile[i] = h->ktiled ? h->tiled.tile[i] : 0;
  return FCM_OK;
}

extern "C" int fcm_mg_launch_count(const fcm_mg* h, int64_t* launches) {
  if (!h || !launches) return fail(FCM_EINVAL, "NULL argument");
  *launches = h->launches;
  return FCM_OK;
}

extern "C" const char* fcm_last_error(void) { return last_error().c_str(); }

extern "C" int fcm_mg_block_counts(const fcm_mg* h, int32_t q, int64_t* n_individual,
                                   int32_t* n_shared_types) {
  if (!h || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad level");
  if (n_individual) *n_individual = h->lev[q].n_irr + h->lev[q].n_wb;
  if (n_shared_types) *n_shared_types = h->lev[q].n_types;
  return FCM_OK;
}

extern "C" int fcm_mg_lowrank_info(const fcm_mg* h, int32_t q, int64_t* n_lowrank, int64_t* c_entries) {
  clear_error();
  if (!h || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad level");
  const LevelDev& Lv = h->lev[q];
  if (n_lowrank) *n_lowrank = Lv.n_wb;
  if (c_entries) *c_entries = Lv.n_wb > 0 ? Lv.wb_coff_h.back() : 0;
  return FCM_OK;
}

// Parity protocol: the block inverses exactly as the smoother applies them.
extern "C" int fcm_mg_export_block_inverses(const fcm_mg* h, int32_t q, int64_t* n_blocks, int32_t* block_size,
                                            int64_t* anchors, int32_t* dof_index, double* inv) {
  clear_error();
  if (!h || q < 1 || q > h->g.p) return fail(FCM_EINVAL, "bad handle or level");
  const LevelDev& Lv = h->lev[q];
  if (!n_blocks || !block_size) return fail(FCM_EINVAL, "NULL count arguments");
  if (q == 1 && h->prm.coarse == FCM_COARSE_DIRECT && h->d_A0inv) {   // the direct coarse inverse: one block
    const int64_t n1 = Lv.ndof;
    *n_blocks = 1;
    *block_size = (int32_t)n1;
    if (anchors) anchors[0] = 0;
    if (dof_index)
      for (int64_t l = 0; l < n1; ++l) dof_index[l] = (int32_t)l;
    if (inv) CU(cudaMemcpy(inv, h->d_A0inv, (size_t)n1 * n1 * 8, cudaMemcpyDeviceToHost));
    return FCM_OK;
  }
  if (!Lv.has_as) return fail(FCM_EINVAL, "level %d has no additive-Schwarz smoother", q);
  const BlockGeom g = block_geom(h->L, q, Lv.patch);
  const int mb = g.mb;
  std::vector<int64_t> list;
  for (int64_t A = 0; A < (int64_t)Lv.blk_h.size(); ++A)
    if (Lv.blk_h[A] != kBlkNone) list.push_back(A);
  *n_blocks = (int64_t)list.size();
  *block_size = mb;
  if (!anchors && !dof_index && !inv) return FCM_OK;
  const size_t mm = (size_t)mb * mb;
  std::vector<double> tmp(mm);
  for (size_t i = 0; i < list.size(); ++i) {
    const int64_t A = list[i];
    if (anchors) anchors[i] = A;
    int ac[3] = {(int)(A % g.na[0]), (int)((A / g.na[0]) % g.na[1]), (int)(A / ((int64_t)g.na[0] * g.na[1]))};
    if (dof_index)
      for (int l = 0; l < mb; ++l) dof_index[i * mb + l] = (int32_t)block_dof_index(h->L, q, g, l, ac);
    if (inv && Lv.blk_h[A] == kBlkWb) {   // low-rank patch: A0^{-1} - Z C Z^T, Z = A0^{-1}[:, S]
      const auto it = std::lower_bound(Lv.wb_anchor_h.begin(), Lv.wb_anchor_h.end(), A);
      const int64_t p = it - Lv.wb_anchor_h.begin();
      const int S = 2 * q + 1, TSZ = S * S + S, dim = h->L.dim;
      const int N = dim == 3 ? S * S * S : S * S;
      const int k = (int)(Lv.wb_soff_h[p + 1] - Lv.wb_soff_h[p]);
      std::vector<double> C((size_t)k * k);
      CU(cudaMemcpy(C.data(), Lv.wb_C + Lv.wb_coff_h[p], C.size() * 8, cudaMemcpyDeviceToHost));
      const double* tb[3];
      int co = 0;
      for (int ax = 0; ax < 3; ++ax) {
        tb[ax] = Lv.fd_tabs_h.data() + ((size_t)ax * Lv.fd_ncls + Lv.fd_cls_h[co + ac[ax]]) * TSZ;
        co += g.na[ax];
      }
      std::vector<double> U((size_t)mb * N, 0.0);   // U[l][mode], 0 for absent slots
      std::vector<char> pres(mb);
      for (int l = 0; l < mb; ++l) {
        pres[l] = block_dof_index(h->L, q, g, l, ac) >= 0;
        if (!pres[l]) continue;
        const int t = Lv.wb_tsl_h[l];
        const int sx = t % S, sy = (t / S) % S, sz = dim == 3 ? t / (S * S) : 0;
        for (int e = 0; e < N; ++e) {
          const int mx = e % S, my = (e / S) % S, mz = dim == 3 ? e / (S * S) : 0;
          const double lam = tb[0][S * S + mx] + tb[1][S * S + my] + (dim == 3 ? tb[2][S * S + mz] : 0.0);
          double v = tb[0][sx * S + mx] * tb[1][sy * S + my] / std::sqrt(Lv.fd_s * lam);
          if (dim == 3) v *= tb[2][sz * S + mz];
          U[(size_t)l * N + e] = v;
        }
      }
      std::vector<double> A0((size_t)mb * mb);
#pragma omp parallel for schedule(static)
      for (int a = 0; a < mb; ++a)
        for (int b = 0; b < mb; ++b) {
          double v = 0.0;
          for (int e = 0; e < N; ++e) v += U[(size_t)a * N + e] * U[(size_t)b * N + e];
          A0[(size_t)a * mb + b] = v;
        }
      const int16_t* Sl = Lv.wb_slots_h.data() + Lv.wb_soff_h[p];
      std::vector<double> ZC((size_t)mb * k, 0.0);   // Z C
      for (int a = 0; a < mb; ++a)
        for (int i = 0; i < k; ++i) {
          const double z = A0[(size_t)a * mb + Sl[i]];
          for (int j = 0; j < k; ++j) ZC[(size_t)a * k + j] += z * C[(size_t)i * k + j];
        }
#pragma omp parallel for schedule(static)
      for (int a = 0; a < mb; ++a)
        for (int b = 0; b < mb; ++b) {
          double v = A0[(size_t)a * mb + b];
          for (int j = 0; j < k; ++j) v -= ZC[(size_t)a * k + j] * A0[(size_t)b * mb + Sl[j]];
          inv[i * mm + (size_t)a * mb + b] = (pres[a] && pres[b]) ? v : (a == b ? 1.0 : 0.0);
        }
      continue;
    }
    if (inv) {
      const int32_t bq = Lv.blk_h[A];
      const double* src;
      double scale = 1.0;
      if (bq >= 0 && (Lv.patch || Lv.irr_tp)) {   // tile-packed lower triangle (patch.cuh / cellws.cuh)
        const int64_t ps = Lv.patch ? Lv.pstride : Lv.irr_tps;
        std::vector<double> pk(ps);
        CU(cudaMemcpy(pk.data(), (Lv.patch ? Lv.irr_inv : Lv.irr_tp) + (size_t)bq * ps, ps * 8, cudaMemcpyDeviceToHost));
        for (int r = 0; r < mb; ++r)
          for (int c = 0; c <= r; ++c) {
            const int I = r / 32, J = c / 32, rr = r % 32, cc = c % 32;
            const bool swz = Lv.patch && Lv.swz;
            const double v = I != J ? pk[tile_off(I, J) + tile_pos(rr, cc, swz)] : pk[tile_off(I, I) + rr * (rr + 1) / 2 + cc];
            inv[i * mm + (size_t)r * mb + c] = v;
            inv[i * mm + (size_t)c * mb + r] = v;
          }
        continue;
      }
      if (bq >= 0) {
        src = Lv.irr_inv + (size_t)bq * mm;
      } else {
        const int t = -bq - 1;
        src = Lv.type_inv + (size_t)(t & 0xfff) * mm;
        if (t >> 12) scale = 1.0 / h->alpha;
      }
      CU(cudaMemcpy(tmp.data(), src, mm * sizeof(double), cudaMemcpyDeviceToHost));
      for (size_t e = 0; e < mm; ++e) inv[i * mm + e] = tmp[e] * scale;
    }
  }
  return FCM_OK;
}
