/*
 * fcm_mg.h -- C ABI of the B200-native hierarchical p-multigrid for finite cell systems
 * (arXiv 2010.00881, "Hierarchical multigrid approaches for the finite cell method on
 * uniform and multi-level hp-refined grids").
 *
 * The library solves A_L x = b ("A_l x_l = b_l") for a finite-cell
 * discretisation (Eq. weakform) on a uniform Cartesian grid of cells with
 * an integrated-Legendre basis of order p, using flexible CG (PAPER.md:351
 * "the multigrid V-cycle ... primarily as a preconditioner within the CG method") around
 * one V-cycle of Algorithm 1 per iteration.  Level l <-> order q = l+1;
 * the levels are the arithmetic p-sequence p, p-1, ..., 1.
 *
 * All floating point is IEEE fp64.  Every function returns FCM_OK (0) or a negative error
 * code; fcm_last_error() returns a thread-local message describing the last failure.
 * Device pointers are CUDA device pointers on the handle's device; host pointers are
 * plain host memory.  No torch / C++ types cross this boundary.
 *
 * ---------------------------------------------------------------------------------------
 * CONVENTIONS (shared interface definitions; the CPU oracle implements them independently)
 * ---------------------------------------------------------------------------------------
 * Cells: c = (cz*ny + cy)*nx + cx (x fastest); cell (cx,cy,cz) = [cx h,(cx+1)h] x ...
 *
 * 1D modes (normalisation reading R-B1): k = 0: (1-xi)/2, k = 1: (1+xi)/2,
 *   k >= 2: (P_k - P_{k-2})/sqrt(2(2k-1)) (degree k).
 * Element modes: tuples (kx,ky[,kz]).  Tensor space: all (p+1)^d tuples.  Trunk space
 *   (PAPER.md:316-320): vertex modes and modes whose internal (k>=2) degrees sum to <= p.
 * Mode order (the level tag): tensor -> max of 1D orders (k<2 counts 1, k>=2 counts k);
 *   trunk -> 1 for vertex modes, else the sum of the internal degrees.
 * Local element order ("hierarchical"): modes sorted by the key
 *   (order, S, deg_x, deg_y, deg_z, off),  S = sum_{a: k_a>=2} 2^a,
 *   deg_a = k_a if k_a >= 2 else 0,  off = sum_{a: k_a<2} k_a 2^a;
 *   element DOF index = rank * n_f + component.  The level-q element DOFs are therefore the
 *   leading m_q entries, and every level matrix is the leading block.
 * Entities / DOFs: mode k_a < 2 is nodal on axis a (vertex index cell_a + k_a), k_a >= 2 is
 *   internal (the cell interval).  DOF key (identifies a global DOF independent of layout):
 *     X_a = 2*vertex_a (nodal) or 2*cell_a + 1 (internal); X = 0, deg = 0 for absent axes;
 *     key = ((((X_z*(2nx+1) + X_y)*(2nx+1) + X_x)*(p+1) + deg_z)*(p+1) + deg_y)*(p+1)
 *           + deg_x)*n_f + comp        (requires nx == ny == nz; int64)
 * Dirichlet (reading R7): every DOF of an entity on a face with bit (2*axis + side) set in
 *   dirichlet_faces (side 1 = upper face) is eliminated (u = 0 strongly).
 * Vector layout on the device ("class-major"): a DOF class is (S, degrees, component); each
 *   class is a dense array over its free entity positions (x fastest); classes are ordered
 *   by (order, S, deg_x, deg_y, deg_z, comp).  The level-q vector is the PREFIX of length
 *   ndofs(q) of the fine vector: restriction R = [I 0] is a pointer alias and R^T is
 *   zero extension (Eq. restrictionoperation).  fcm_mg_dof_keys() maps
 *   layout slots to DOF keys.
 * Element matrices: m x m row-major fp64, m = (number of element modes) * n_f, in the
 *   local order above, SYMMETRIC.  K_ref is the matrix of an uncut physical cell
 *   (alpha = 1); an uncut fictitious cell uses alpha * K_ref.
 */
#ifndef FCM_MG_H
#define FCM_MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---------------------------------------------------------------------- */
#define FCM_OK            0
#define FCM_NOT_CONVERGED 1   /* warning: solver hit maxit; outputs valid   */
#define FCM_EINVAL      (-1)  /* invalid argument (incl. an empty level)      */
#define FCM_ENOMEM      (-2)  /* device allocation failed; message states bytes           */
#define FCM_ESINGULAR   (-3)  /* singular / non-SPD Schwarz block; message names it       */
#define FCM_EINDEF      (-4)  /* p^T A p <= 0 in CG                          */
#define FCM_ECUDA       (-5)  /* CUDA runtime error                                      */
#define FCM_ENCCL       (-6)  /* NCCL error                                              */

/* ---- enums ------------------------------------------------------------------------------ */
#define FCM_SPACE_TENSOR 0
#define FCM_SPACE_TRUNK  1
#define FCM_BLOCK_ELEMENT 0   /* elementwise AS blocks (Fig. elementBlocks)   */
#define FCM_BLOCK_PATCH   1   /* patchwise: 2^d cells around a vertex (Fig. patchBlocks)    */
#define FCM_COARSE_DIRECT 0   /* dense direct solve of the p=1 level         */
#define FCM_COARSE_AS_PCG 1   /* CG + undamped elementwise AS at p=1         */
#define FCM_COARSE_JACOBI_PCG 2 /* CG + diagonal preconditioner (BASELINE.json variant)     */
#define FCM_COARSE_GMG_PCG 3  /* CG preconditioned by a geometric V-cycle over h-coarsened
                                 p=1 grids (PAPER.md:227 Remark; R21): trilinear P,
                                 Galerkin P^T A P element by element, elementwise AS on every
                                 h-level, dense solve on the coarsest grid; distributed over
                                 the slabs in slab mode (see multi-GPU below)               */
#define FCM_PHYS_POISSON 0
#define FCM_PHYS_ELASTICITY 1

/* Environment switches read at setup (defaults in brackets):
 *   FCM_DETERMINISTIC=1  [0] bit-reproducible mode (single GPU): every scatter runs in colour
 *                        passes (2^d cell parities; 27 vertex classes mod 3 for patches), so
 *                        each output entry receives at most one fp64 atomic per launch; per-
 *                        patch row sums in a fixed warp order; operator energies and coarse dot
 *                        sums in block order.  Two solves are bit-identical; several times
 *                        slower.  Needs coarse DIRECT, GMG_PCG or a p=1 level that fits the
 *                        tiled coarse kernel (FCM_EINVAL otherwise).
 *   FCM_CELL_WS=0        [1] elementwise levels q >= 2 with m in {27, 64, 125}: one warp-
 *                        specialised launch per cell operation (MMA warps for the regular cells,
 *                        bulk-copy streaming of tile-packed individual matrices); 0 = the
 *                        k_cell_mma block-range launch with full-storage matrices.
 *   FCM_CELL_MMA=0, FCM_PDL=0, FCM_HOST_LOOP=1, FCM_TILED_ATOMIC=0: generic cell kernels, no
 *                        programmatic dependent launch, per-iteration host loop, block-order
 *                        tiled coarse sums (fallback / reproducibility switches, tested).      */

/* Grid / discretisation. */
typedef struct fcm_grid {
  int32_t dim;              /* 2 or 3                                                    */
  int32_t n[3];             /* cells per axis; n[2] = 1 when dim == 2                    */
  double  h;                /* cell size (cells are cubes)                                */
  int32_t p;                /* polynomial order, 1 <= p <= 8                              */
  int32_t space;            /* FCM_SPACE_*                                                */
  int32_t n_f;              /* field components: 1 (Poisson) or dim (elasticity)          */
  uint32_t dirichlet_faces; /* bit 2*axis+side: u = 0 on that box face                    */
} fcm_grid;

/* Solver parameters (readings R2-R4). */
typedef struct fcm_params {
  int32_t block;            /* FCM_BLOCK_* for levels q >= 2 (coarse AS is elementwise)   */
  double  omega;            /* AS relaxation on levels q >= 2 (paper: 1/3, 2/15, 1/6, 1/18)*/
  int32_t n_pre, n_post;    /* smoothing sweeps (paper: 5, 5)                             */
  int32_t coarse;           /* FCM_COARSE_*                                               */
  double  coarse_rtol;      /* inner CG: stop when ||r|| < coarse_rtol ||r0|| (1e-12)    */
  int32_t coarse_maxit;     /* inner CG iteration cap                                     */
  void*   stream;           /* cudaStream_t for all work (NULL = legacy default stream)   */
} fcm_params;

/* Physics of the generator (Eq. weakform). */
typedef struct fcm_physics {
  int32_t kind;             /* FCM_PHYS_*                                                 */
  double  alpha;            /* fictitious-domain factor epsilon, 1e-8       */
  double  E, nu;            /* elasticity: Young's modulus, Poisson ratio                 */
  int32_t depth;            /* space-tree integration depth (3)             */
  int32_t traction_face;    /* face 2*axis+side with traction (1,0,0), or -1              */
} fcm_physics;

typedef struct fcm_mg fcm_mg;   /* opaque solver handle */

/* ==== workload generator (setup, not timed; independent of the oracle) =================
 * Voids are open balls ||x - c_j|| < r_j (Omega_fict); a point on a sphere is physical.   */

/* Number of element DOFs m for the grid (host only).  Returns m > 0 or a negative code.   */
int fcm_element_size(const fcm_grid* g);

/* Classify every cell: 0 = uncut physical, 1 = uncut fictitious, 2 = cut (exact box/ball
 * test).  cell_kind: host, ncell bytes.  *n_cut receives the number of cut cells.          */
int fcm_gen_classify(const fcm_grid* g, int64_t n_voids, const double* centres /*n_voids*dim*/,
                     const double* radii, uint8_t* cell_kind, int64_t* n_cut);

/* Element matrices and body loads (host buffers).  K_ref/f_ref: uncut physical cell (m*m, m).
 * For each of the n_cut cells listed in cut_cells (cell indices), the space-tree quadrature
 * (reading R13) gives cut_K[i] (m*m) and cut_f[i] (m).  Poisson f = 1;
 * elasticity body force 0.  f_traction (m, may be NULL): int_{face} N.(1,0,0) of one cell
 * face of type ph->traction_face.  Uses up to `threads` host threads (0 = all).            */
int fcm_gen_element_matrices(const fcm_grid* g, const fcm_physics* ph,
                             int64_t n_voids, const double* centres, const double* radii,
                             double* K_ref, double* f_ref, int64_t n_cut,
                             const int64_t* cut_cells, double* cut_K, double* cut_f,
                             double* f_traction, int32_t threads);

/* The cut-cell part of fcm_gen_element_matrices on the CURRENT CUDA DEVICE:
 * the same space-tree quadrature (reading R13) with one CTA per cut cell, box
 * classification bit-identical to the host generator, uncut leaves in Kronecker form, depth-
 * limit cut leaves with alpha per Gauss point.  Host in/out buffers as in
 * fcm_gen_element_matrices (cut_K n_cut*m*m, cut_f n_cut*m, cut_f may be NULL).
 * Poisson only, depth <= 4, m <= 128: otherwise FCM_EINVAL (use the host generator).       */
int fcm_gen_cut_matrices_device(const fcm_grid* g, const fcm_physics* ph, int64_t n_voids,
                                const double* centres, const double* radii, int64_t n_cut,
                                const int64_t* cut_cells, double* cut_K, double* cut_f);

/* ==== solver ============================================================================ */

/* Build the hierarchy on the current CUDA device ("cached during the solver
 * setup phase"): copies the host inputs (caller may free them on return), classifies the
 * Schwarz blocks of every level q >= 2 (and q = 1 for AS-PCG), assembles A_i = P_i^T A_q P_i
 * and inverts them on the device, factors the coarse level if direct.
 *   K_ref      host m*m;  cell_kind host ncell (0/1/2);  alpha the fictitious factor;
 *   cut_cells  host n_cut cell indices (ascending, kind 2);  cut_K host n_cut*m*m.
 * Errors: FCM_EINVAL (bad sizes, empty level), FCM_ENOMEM, FCM_ESINGULAR, FCM_ECUDA.      */
int fcm_mg_setup(const fcm_grid* g, const fcm_params* prm, const double* K_ref,
                 const uint8_t* cell_kind, double alpha, int64_t n_cut,
                 const int64_t* cut_cells, const double* cut_K, fcm_mg** out);

int fcm_mg_destroy(fcm_mg* h);

/* ==== multi-GPU: slab decomposition ================
 * The cell grid is cut into contiguous layers along the LAST axis (z in 3D, y in 2D); rank r
 * of N (one GPU each) owns cell layers [z_begin, z_end).  Its local vectors hold the DOFs of
 * its own cells in the class-major layout of the slab (both interface vertex planes
 * included, duplicated on the two neighbours); an interface DOF is owned by the LOWER rank
 * for dot products.  Every operator / smoother scatter is followed by a sum-exchange of the
 * interface planes over NCCL (grouped send/recv; a + b == b + a keeps both copies bit-
 * identical); dots are reduced with ncclAllReduce.  Schwarz blocks of cells next to an
 * interface are assembled with one ghost cell layer.  The coarse p = 1 problem is solved
 *  - REPLICATED for FCM_COARSE_AS_PCG / _JACOBI_PCG / _DIRECT: the owned coarse residuals are
 *    all-gathered and every rank runs the coarse solver on the full p = 1 grid (no per-
 *    iteration communication in the inner CG);
 *  - DISTRIBUTED for FCM_COARSE_GMG_PCG ("reuse the parallel data structures that
 *    have already been set up for the fine problem"): the inner CG and the h-level-0 smoothing
 *    run on the slabs (exchange + all-reduced owned dots), each slab restricts its OWNED p = 1
 *    residual rows to the global h-level-1 grid, the sum is all-reduced and the h-levels below
 *    run replicated; the slab prolongates into its own vertices.  The inner CG is host-driven
 *    (one 64-byte D2H per iteration), so the slab V-cycle and FCG run without CUDA graphs.
 * NCCL is loaded at run time (dlopen of libnccl.so.2, the one torch already loaded).
 * Patchwise blocks (FCM_BLOCK_PATCH) are single-GPU.                                        */

/* Balanced partition of n cell layers over nranks (host only).                              */
int fcm_slab_bounds(int32_t n, int32_t nranks, int32_t rank, int32_t* z_begin, int32_t* z_end);

/* Host-only description of the local layout of slab [z_begin, z_end) of the GLOBAL grid g at
 * level q: *ndofs local DOFs; keys (ndofs, may be NULL) their global DOF keys; owned (ndofs
 * bytes, may be NULL) 1 where this rank owns the DOF; the interface plane slots at the bottom
 * (*n_lo, lo_slots; empty when z_begin == 0) and top (*n_hi, hi_slots; empty when z_end == n)
 * in exchange order (the neighbour's matching plane lists the same DOFs in the same order).
 * Call with NULL arrays to get the sizes.                                                    */
int fcm_slab_layout(const fcm_grid* g, int32_t z_begin, int32_t z_end, int32_t q, int64_t* ndofs,
                    int64_t* keys, uint8_t* owned, int64_t* n_lo, int32_t* lo_slots,
                    int64_t* n_hi, int32_t* hi_slots);

/* Global level-1 slot of every local level-1 slot of the slab (host only).                  */
int fcm_slab_coarse_map(const fcm_grid* g, int32_t z_begin, int32_t z_end, int64_t* n_local,
                        int64_t* global_slots);

/* 128-byte NCCL unique id (call on rank 0 and broadcast the bytes to the other ranks).      */
int fcm_nccl_unique_id(void* id128);

typedef struct fcm_slab {
  int32_t rank, nranks;     /* this rank (uses the current CUDA device), number of ranks      */
  int32_t z_begin, z_end;   /* owned cell layers (fcm_slab_bounds)                            */
  const void* nccl_id;      /* 128 bytes from fcm_nccl_unique_id (ignored when nranks == 1)   */
} fcm_slab;

/* Slab version of fcm_mg_setup.  g is the GLOBAL grid; cell_kind the GLOBAL cell kinds;
 * cut_cells / cut_K the cut cells (global indices, ascending) of the owned layers AND of the
 * ghost layers z_begin-1 and z_end (when they exist); coarse_cut_cells / coarse_cut_K1 EVERY
 * cut cell of the grid with the leading m_1 x m_1 block of its matrix (replicated coarse
 * level).  Collective: every rank calls it with the same g, prm and nccl_id.               */
int fcm_mg_setup_slab(const fcm_grid* g, const fcm_params* prm, const fcm_slab* slab,
                      const double* K_ref, const uint8_t* cell_kind, double alpha,
                      int64_t n_cut, const int64_t* cut_cells, const double* cut_K,
                      int64_t n_coarse_cut, const int64_t* coarse_cut_cells,
                      const double* coarse_cut_K1, fcm_mg** out);

/* Number of levels (= p) and free DOFs of level q (1..p) (local DOFs of this rank).        */
int fcm_mg_nlevels(const fcm_mg* h, int32_t* nlevels);
int fcm_mg_ndofs(const fcm_mg* h, int32_t q, int64_t* n);
/* Element DOFs of level q (leading block size m_q).                                        */
int fcm_mg_level_m(const fcm_mg* h, int32_t q, int32_t* m);

/* Schwarz blocks of level q: *n_individual blocks with their own stored inverse (cut-
 * influenced neighbourhood) and *n_shared_types inverses shared by all regular blocks of a
 * boundary type (inverse scaled by 1/alpha for all-fictitious neighbourhoods).            */
int fcm_mg_block_counts(const fcm_mg* h, int32_t q, int64_t* n_individual, int32_t* n_shared_types);
/* Individual patches stored as low-rank corrections of the regular patch (patchwise levels with
 * fast diagonalisation, single GPU; FCM_PATCH_WB=0 disables): every member cell uncut and
 * physical, so A_i = A0 + P_S E P_S^T differs from the regular (Kronecker) patch matrix A0 only on
 * the k slots S touched by the outer ring's cut / fictitious cells, and (Woodbury)
 * A_i^{-1} r = z - A0^{-1} P_S C P_S^T z, z = A0^{-1} r, C = H - H (H + E)^{-1} H, H = (P_S^T A0^{-1}
 * P_S)^{-1} -- the same operator as the explicit inverse (Eq. AdditiveSchwarz), with k x k
 * instead of m(m+1)/2 stored numbers.  *n_lowrank of the *n_individual blocks of
 * fcm_mg_block_counts are of this kind; *c_entries = sum of k^2 (the C matrices, full storage).
 * fcm_mg_export_block_inverses expands them to explicit inverses.  Used on levels whose patches
 * have >= 300 slots (FCM_PATCH_WB=2: every patch level).                                     */
int fcm_mg_lowrank_info(const fcm_mg* h, int32_t q, int64_t* n_lowrank, int64_t* c_entries);

/* DOF keys of the fine layout (host buffer of ndofs(p) int64, see CONVENTIONS).            */
int fcm_mg_dof_keys(const fcm_mg* h, int64_t* keys);

/* Assemble a load vector in layout order (device b, ndofs(p)):
 * b = sum_c P_c^T f_c with f_c = f_ref (kind 0), alpha f_ref (kind 1), cut_f[i] (kind 2),
 * plus f_traction on every cell touching face `traction_face` (-1: none).  Host inputs.    */
int fcm_mg_load(fcm_mg* h, const double* f_ref, const double* cut_f,
                const double* f_traction, int32_t traction_face, double* b);

/* y = A_q x on level q (device vectors of ndofs(q)); PAPER.md:118 A_{l-1} = R A_l R^T.    */
int fcm_apply(fcm_mg* h, int32_t q, const double* x, double* y);

/* x += omega_q M_q^{-1} r (one additive-Schwarz smoothing update, Eq.
 * AdditiveSchwarz P:254-257) on level q; omega_q = params.omega (q >= 2) or 1 (q = 1).     */
int fcm_mg_smooth(fcm_mg* h, int32_t q, const double* r, double* x);

/* One population of a patchwise level's smoother (measurement, parity by parts): part 1 = the
 * individual (irregular) patches only (k_patch_irr, streaming the tile-packed inverses),
 * part 2 = the shared-type (regular) patches only, 0 = both (= fcm_mg_smooth).  Parts 1 and 2
 * sum to part 0 (up to the order of the fp64 scatter additions).  FCM_EINVAL on elementwise
 * levels.                                                                                   */
int fcm_mg_smooth_part(fcm_mg* h, int32_t q, int32_t part, const double* r, double* x);

/* x = A_1^{-1} r by the configured coarse solver; *iters (host, may be NULL)
 * receives the inner CG iterations (0 for direct).                                         */
int fcm_mg_coarse_solve(fcm_mg* h, const double* r, double* x, int32_t* iters);

/* z = V(r): one V-cycle of Algorithm 1 on the finest level, x~ = 0 on
 * entry, reading R1 (residual recomputed before each sweep).  Device vectors ndofs(p).     */
int fcm_mg_vcycle(fcm_mg* h, const double* r, double* z);

/* Flexible (Polak-Ribiere) PCG with one V-cycle per iteration (R5/R6):
 * x0 = 0, stop when the recursive ||r_k||/||b|| < rtol or after maxit iterations.
 * b, x: device, ndofs(p).  *iters (host) = number of x-updates.  relres_hist (host, may be
 * NULL, maxit+1 entries) receives ||r_k||/||b||.  Synchronises the stream.
 * Returns FCM_OK, FCM_NOT_CONVERGED (x valid), or an error.                               */
int fcm_pcg_solve(fcm_mg* h, const double* b, double* x, double rtol, int32_t maxit,
                  int32_t* iters, double* relres_hist);

/* Same as fcm_pcg_solve with HOST b and x (pinned or pageable): copies b in, solves,
 * copies x out, all inside the call (the end-to-end user path).                           */
int fcm_pcg_solve_host(fcm_mg* h, const double* b_host, double* x_host, double rtol,
                       int32_t maxit, int32_t* iters, double* relres_hist);

/* Multigrid as a stand-alone solver (the "MG" columns of the tables):
 * x_0 = 0, x_i = x_{i-1} + V(b - A x_{i-1}) with the true residual r_i = b - A x_i
 * recomputed after every V-cycle; stop when ||r_i||/||b|| < rtol or after maxit V-cycles.
 * b, x: device, ndofs(p).  *iters (host, may be NULL) = V-cycles done; relres_hist (host, may
 * be NULL, maxit+1 entries) receives ||r_i||/||b|| (the contraction numbers of P:357 are
 * hist[i]/hist[i-1]).  Synchronises the stream once per V-cycle.
 * Returns FCM_OK, FCM_NOT_CONVERGED (x valid), or an error (FCM_EINDEF on a NaN residual). */
int fcm_mg_solve(fcm_mg* h, const double* b, double* x, double rtol, int32_t maxit,
                 int32_t* iters, double* relres_hist);

/* Parity protocol (ladder L2/L4): export the additive-Schwarz block inverses
 * A_i^{-1} = (P_i^T A_q P_i)^{-1} (Eq. AdditiveSchwarz) exactly as level q's
 * smoother applies them, so that a reference implementation can run the same smoother and
 * V-cycle on identical setup data.  Two-call protocol: with all buffers NULL, *n_blocks and
 * *block_size receive the number of blocks with at least one free DOF and m_b (elementwise: the
 * level element size; patchwise: the (2q+1)^d-slot patch).  Otherwise (host buffers):
 *   anchors   [n_blocks]            anchor of block i (cell index, or vertex index x fastest over
 *                                   (n+1)^d for patches), ascending -- may be NULL;
 *   dof_index [n_blocks * m_b]      layout index (0 <= . < ndofs(q)) of block row l, -1 where the
 *                                   slot holds no free DOF (absent or Dirichlet: identity row);
 *   inv       [n_blocks * m_b^2]    the inverse, row-major, in the block's slot order; shared-type
 *                                   blocks are expanded (and scaled by 1/alpha for all-fictitious
 *                                   neighbourhoods), individual blocks unpacked.
 * Level 1 with the direct coarse solver exports the dense A_1^{-1} it applies as ONE block of
 * size ndofs(1) (dof_index = 0..ndofs(1)-1).
 * Errors: FCM_EINVAL (bad handle/level, level without a smoother), FCM_ECUDA.                */
int fcm_mg_export_block_inverses(const fcm_mg* h, int32_t q, int64_t* n_blocks, int32_t* block_size,
                                 int64_t* anchors, int32_t* dof_index, double* inv);

/* Statistics of the last fcm_pcg_solve / fcm_mg_solve: inner coarse CG iterations, V-cycles. */
int fcm_mg_stats(const fcm_mg* h, int64_t* coarse_iters_total, int64_t* vcycles);

/* Which coarse solver kernel the handle runs (for measurement and tests):
 * *kind = FCM_COARSE_KERNEL_DIRECT (dense inverse GEMV), _GRID (grid-wide cooperative PCG
 * over the cell population, any size) or _TILED (shared-memory bricks, one grid barrier per
 * iteration; chosen at setup when every brick and its matrices fit in shared memory);
 * *blocks = CTAs of the cooperative launch (0 for direct); tile[3] (may be NULL) = brick
 * size in vertices (tiled only, else 0).                                                   */
#define FCM_COARSE_KERNEL_DIRECT 0
#define FCM_COARSE_KERNEL_GRID 1
#define FCM_COARSE_KERNEL_TILED 2
#define FCM_COARSE_KERNEL_GMG 3   /* CG + geometric V-cycle (nested graph loop); blocks = h-levels */
int fcm_mg_coarse_info(const fcm_mg* h, int32_t* kind, int32_t* blocks, int32_t* tile);

/* Counters of kernels launched by the library since setup (for the bench's gpu_launches). */
int fcm_mg_launch_count(const fcm_mg* h, int64_t* launches);

/* ==== multi-level hp-refinement ========
 * A base grid of n^d cells on [0,1]^d whose elements are refined by SUPERPOSITION:
 * a refined element of depth j carries 2^d subelements of depth j+1, recursively up to kmax;
 * leaves are the elements without subelements.  Every element of every depth carries the tensor
 * integrated-Legendre modes of order p on its entities (vertices / edges / faces / interior of the
 * depth-j grid, doubled coordinates X as above).  Activation rule (reading R25, the rule set the
 * paper defers to [Zander2016]): a depth-j entity is active iff (compatibility) j = 0 or
 * every depth-j element adjacent to it inside the domain exists, and (independence) at least one
 * existing adjacent depth-j element is a leaf.  Dirichlet as R7.  A leaf's basis is the
 * superposition of the active free functions of the leaf and all its ancestors.
 * hp level sequence (Fig. hpmultigrid), finest first:
 *   (p,k), (p-1,k), ..., (1,k), (1,k-1), ..., (1,0)       (k = deepest depth carrying DOFs),
 * level (q, kc) = the DOFs of mode order <= q and depth <= kc; nested, so restriction is index
 * selection; trailing levels without DOFs are dropped.  DOF order of the library: by the COARSEST level containing the DOF
 * (descending), so every level is a PREFIX of the fine vector as on uniform grids.
 * Schwarz blocks (reading R26, Fig. 7 caption P:273 "granularity of the base elements"):
 * elementwise = the level DOFs nonzero on one BASE element; patchwise = those nonzero on the
 * 2^d base elements around a base vertex; identical blocks counted once.                   */
#define FCM_HP_REFINE_CUT 0   /* refine the elements cut by the immersed boundary        */
#define FCM_HP_REFINE_ALL 1   /* refine every element (uniform overlay; tests)                    */

typedef struct fcm_hp_spec {
  int32_t dim;              /* 2 or 3                                                         */
  int32_t n;                /* base cells per axis                                            */
  int32_t p;                /* order, 1 <= p <= 8                                             */
  int32_t kmax;             /* refinement depth, 0 <= kmax <= 8                               */
  int32_t refine;           /* FCM_HP_REFINE_*                                                */
  uint32_t dirichlet_faces; /* as fcm_grid                                                    */
  fcm_physics phys;         /* generator physics (alpha, E, nu, space-tree depth, traction)   */
  int64_t n_voids;          /* spherical voids (fictitious domain)               */
  const double* centres;    /* host [n_voids * dim]                                           */
  const double* radii;      /* host [n_voids]                                                 */
} fcm_hp_spec;

typedef struct fcm_hp_disc fcm_hp_disc;   /* opaque host discretisation (generator output) */
typedef struct fcm_hp fcm_hp;             /* opaque device solver handle                    */

/* Generator (setup, host C++/OpenMP, independent of the oracle): refinement trees, activation,
 * DOF numbering, leaf element matrices by the space tree of depth phys.depth BELOW EACH LEAF
 * ((p+1)^d Gauss points per sub-box, alpha per point at depth-limit cut sub-boxes, R13) and the
 * load vector (f = 1 Poisson, traction (1,0,0) on phys.traction_face, R8).  *out owns host
 * memory; free with fcm_hp_disc_destroy.  Errors: FCM_EINVAL (bad spec), FCM_ENOMEM.        */
int fcm_hp_generate(const fcm_hp_spec* spec, fcm_hp_disc** out);
int fcm_hp_disc_destroy(fcm_hp_disc* d);
/* Sizes: ndof, levels, leaves, total leaf DOF entries sum(m_e), total matrix entries sum(m_e^2). */
int fcm_hp_disc_info(const fcm_hp_disc* d, int64_t* ndof, int32_t* nlevels, int64_t* nleaves,
                     int64_t* leaf_entries, int64_t* leaf_matrix_entries);
/* Per level (finest first): ndofs (a prefix length), order q and depth cap kc.  Host [nlevels]. */
int fcm_hp_disc_levels(const fcm_hp_disc* d, int64_t* ndofs, int32_t* q, int32_t* kc);
/* DOF keys, host int32 [ndof * 8]: (depth j, X_x, X_y, X_z, deg_x, deg_y, deg_z, comp), X and
 * deg as the uniform convention on the depth-j grid (absent axes 0).  Load b, host [ndof].     */
int fcm_hp_disc_keys(const fcm_hp_disc* d, int32_t* keys);
int fcm_hp_disc_load(const fcm_hp_disc* d, double* b);
/* Leaves (any pointer may be NULL): leaf_ptr [nleaves+1] offsets into dofs; dofs [leaf_entries]
 * the leaf's global DOF indices, ascending (so each level's entries are a prefix); K
 * [leaf_matrix_entries] the leaf matrices m_e x m_e row-major in that order, concatenated;
 * info [nleaves * 5] = (depth, idx_x, idx_y, idx_z, base element index x fastest).           */
int fcm_hp_disc_leaves(const fcm_hp_disc* d, int64_t* leaf_ptr, int32_t* dofs, double* K, int32_t* info);

/* Device setup on the current CUDA device: copies the leaves, builds every level's Schwarz
 * blocks (prm->block, coarse level elementwise), assembles A_i = P_i^T A_l P_i from the leaf
 * matrices and inverts them (equilibrated blocked Gauss-Jordan), and the coarse solver
 * (FCM_COARSE_DIRECT: dense inverse of the (1,0) matrix; FCM_COARSE_AS_PCG: CG + undamped
 * elementwise AS, prm->coarse_rtol relative to ||r0||).  prm->omega is the fine-level relaxation.
 * The handle does not keep d.  Errors: FCM_EINVAL, FCM_ENOMEM, FCM_ESINGULAR, FCM_ECUDA.       */
int fcm_hp_setup(const fcm_hp_disc* d, const fcm_params* prm, fcm_hp** out);
int fcm_hp_destroy(fcm_hp* h);
/* y = A_l x on level l (0 = finest): element-by-element over the leaves;
 * x, y device [ndofs(l)].                                                                    */
int fcm_hp_apply(fcm_hp* h, int32_t level, const double* x, double* y);
/* x += omega_l sum_i P_i A_i^{-1} P_i^T r (Eq. AdditiveSchwarz); device [ndofs(l)]. */
int fcm_hp_smooth(fcm_hp* h, int32_t level, const double* r, double* x);
/* Measurement: reps back-to-back smoother sweeps of level l (x accumulates), timed with CUDA events
 * on the library's stream (no host gaps); *ms = mean per sweep.                                */
int fcm_hp_time_smooth(fcm_hp* h, int32_t level, const double* r, double* x, int32_t reps, float* ms);
/* z = one hp V-cycle of Algorithm 1 (R1) applied to r; device [ndof].              */
int fcm_hp_vcycle(fcm_hp* h, const double* r, double* z);
/* Flexible PCG with one hp V-cycle per iteration (as fcm_pcg_solve); relres_hist host
 * [maxit+1] or NULL.  FCM_NOT_CONVERGED when maxit is reached.                              */
int fcm_hp_pcg_solve(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit,
                     int32_t* iters, double* relres_hist);
/* hp-multigrid as a stand-alone solver: x_0 = 0, x_i = x_{i-1} + V(b - A x_{i-1})
 * until ||b - A x_i|| / ||b|| < rtol (strict) or maxit cycles; relres_hist host [maxit+1] or NULL
 * (the contraction numbers rho_i = hist[i] / hist[i-1], Eq. contraction).                */
int fcm_hp_mg_solve(fcm_hp* h, const double* b, double* x, double rtol, int32_t maxit,
                    int32_t* iters, double* relres_hist);
/* Identical-setup parity protocol for the hp smoother: level l's blocks and inverses.  Two-call:
 * with ptr/dofs/inv NULL, *n_blocks, *dof_entries (sum m_i) and *inv_entries (sum m_i^2) are set;
 * otherwise ptr [n_blocks+1], dofs [dof_entries] (level indices, ascending per block), inv
 * [inv_entries] (row-major per block, concatenated).  The coarse level with the direct solver
 * exports its dense inverse as one block.                                                    */
int fcm_hp_export_blocks(const fcm_hp* h, int32_t level, int64_t* n_blocks, int64_t* dof_entries,
                         int64_t* inv_entries, int64_t* ptr, int32_t* dofs, double* inv);
/* Launch counter and last-solve statistics (coarse CG iterations, V-cycles).                  */
int fcm_hp_stats(const fcm_hp* h, int64_t* launches, int64_t* coarse_iters_total, int64_t* vcycles);

/* Thread-local message of the last error ("" if none).                                     */
const char* fcm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FCM_MG_H */
