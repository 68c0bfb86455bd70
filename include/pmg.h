/*
 * pmg.h -- C ABI of the B200-native p-multigrid hot path of arXiv 1808.03595
 * ("Factorizing the factorization -- a spectral-element solver for elliptic equations with
 * linear operation count", Huismann, Stiller, Froehlich).  Citations: P:n = line n of the
 * paper's LaTeX source.
 *
 * Problem (Eq. helmholtz_equation):  lambda u - Laplace(u) = f on a box of
 * k1 x k2 x k3 cuboidal spectral elements of degree p (widths per direction), with
 * homogeneous Dirichlet conditions on the box boundary -- or homogeneous Neumann on
 * the faces selected by pmg_options.neumann.  All arithmetic is FP64.
 *
 * Conventions shared by every call
 *  - Every call returns pmg_status; PMG_OK = 0.  No C++ exception crosses the ABI.  On an
 *    error the thread-local message of pmg_last_error() says what was wrong.
 *  - Vector arguments are caller-owned DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *    unless the name ends in _host.  The library never frees or reallocates them.  All work
 *    is enqueued on the stream given in pmg_options.stream (NULL = legacy default stream)
 *    and is asynchronous unless stated otherwise.  The context owns its tables and
 *    workspaces, allocated in pmg_setup; no other call allocates device memory.
 *  - "grid" vectors hold one value per global GLL node: N_d = k_d p + 1 nodes per direction
 *    (boundary included), flat index i1 + N1 (i2 + N2 i3), x1 fastest.
 *  - "skeleton" (condensed, hat) vectors hold the element-boundary unknowns of one level in
 *    the library's record layout: one record per mesh vertex
 *    (v1, v2, v3), 0 <= v_d <= k_d, record index v1 + (k1+1)(v2 + (k2+1) v3); a record holds
 *    the interiors of the three faces and three edges leaving the vertex in +x_d direction,
 *    then the vertex itself: [f1: (p-1)^2][f2: (p-1)^2][f3: (p-1)^2][e1: p-1][e2][e3][vertex].
 *    Length = (k1+1)(k2+1)(k3+1) * (3(p-1)^2 + 3(p-1) + 1) doubles (pmg_level_info).
 *    Entries that are not free unknowns (on a Dirichlet face or outside the box) are zero on
 *    input and are written as zero on output.
 *  - Levels: l = 0 .. L with degrees p_l = p0 2^l (l < L), p_L = p, L = ceil(log2(p/p0))
 *    (reading R10).  Level L is the finest.
 *  - z-slabs (nranks > 1): every rank calls the same functions in the same
 *    order.  Grid vectors are the rank's slab: grid planes z0 p .. z1 p (both shared planes
 *    included; pmg_level_info's n_grid).  Skeleton vectors are local: the record planes zb .. z1
 *    of pmg_slab (n_skel), ghost planes included; every call refreshes the ghost planes of its
 *    skeleton inputs and outputs in place from the neighbour ranks, so on return every local
 *    plane holds the undivided vector's values.  pmg_condense, pmg_recover and the layout
 *    converters are one-GPU calls (pmg_solve condenses and recovers on slabs internally).
 */
#ifndef PMG_H
#define PMG_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmg_ctx pmg_ctx; /* opaque; owns all tables and workspaces */

typedef enum {
  PMG_OK = 0,
  PMG_EINVAL = -1,      /* invalid argument (message says which) */
  PMG_ECUDA = -2,       /* a CUDA runtime call or kernel launch failed */
  PMG_ENCCL = -3,       /* a NCCL call (or a loopback exchange) of the z-slab path failed */
  PMG_ENOCONV = -4,     /* pmg_solve: max_cycles reached before the tolerance (report filled) */
  PMG_EBREAKDOWN = -5,  /* coarse CG: p^T H p <= 0 */
  PMG_ENOMEM = -6       /* device allocation failed in pmg_setup */
} pmg_status;

typedef struct {
  int p0;             /* coarse degree, default 2 */
  int weight_degree;  /* degree of the weight polynomial, default 7; only 7 supported */
  int schedule;       /* 0: nu_pre = nu_post = 1 ("MG"); 1: 2^(L-l) */
  int neumann;        /* homogeneous Neumann faces (bitmask: bit 2d / 2d+1 = low / high face of
                         direction d); every other face is homogeneous
                         Dirichlet.  Default 0 (all Dirichlet).  All six Neumann needs lambda > 0. */
  int periodic;       /* periodic directions (bit d: direction d, "the ghost elements
                         stay part of the domain"): k_d even and >= 2, no Neumann bit on d, one GPU (nranks = 1),
                         vertex-star smoother, Jacobi-PCG coarse solver.  Grid vectors keep k_d p + 1 nodes along
                         d; the last plane duplicates plane 0: its input values are ignored and the outputs
                         (pmg_recover / pmg_solve / pmg_skel_to_grid) repeat plane 0 there.  Default 0. */
  int solver;         /* pmg_solve: 0 = multigrid fixpoint iteration (Alg. 4, "MG");
                         1 = Krylov-accelerated multigrid, inexact preconditioned CG with one V-cycle
                         from zero as preconditioner (Alg. 5; "kMG", with schedule 1 "kvMG") */
  int smoother;       /* 0 = vertex-star additive Schwarz (Alg. 2) (default); 1 = element-centred
                         3 x 3 x 3 block smoother (six face planes per block,
                         n_S = 3p - 1, weights of reading R17), 27 colours; one GPU only (nranks = 1) and
                         p <= 16 (else PMG_EINVAL) */
  double coarse_rtol; /* coarse CG relative tolerance, default 1e-4 (reading R11) */
  int coarse_maxit;   /* coarse CG iteration cap, default 10000 */
  int coarse_check;   /* coarse CG: host convergence poll every this many iterations, default 8 */
  int coarse_solver;  /* preconditioner of the coarse CG: 1 = Jacobi (reading R11), 2 = h-multigrid
                         V-cycle over element-merged p0 = 2 levels (NEXT-2, reading R16),
                         0 = automatic: h-multigrid iff more than 12288 elements, some k_d even with
                         k_d / 2 >= 2, and lambda L_min^2 < 100 (L_min the shortest box edge: a
                         mass-dominated coarse system converges fast under Jacobi) (default) */
  int rank, nranks;   /* z-slab decomposition over nranks processes / GPUs:
                         rank r owns element layers [z0_r, z1_r) (pmg_slab_plan); nranks = 1: one GPU */
  const void* nccl_id;/* nranks > 1 with NCCL: 128-byte ncclUniqueId from pmg_nccl_unique_id on rank 0,
                         broadcast by the caller (e.g. torch.distributed); the library creates and owns
                         the communicator.  The caller's current CUDA device is used. */
  void* loopback;     /* nranks > 1 in ONE process (correctness tests): a hub from pmg_loopback_create
                         shared by the nranks contexts, each driven by its own host thread and stream;
                         exchanges are host-synchronised device copies (no kernel waits on another
                         rank).  Exactly one of nccl_id / loopback must be set when nranks > 1. */
  void* stream;       /* cudaStream_t; NULL = default stream */
} pmg_options;

/* z-slab plan of rank `rank` (pure host arithmetic, no GPU needed).  Element layers are split
 * as z0 = floor(rank k3 / nranks), z1 = floor((rank+1) k3 / nranks) (k3 >= nranks required).
 * Local skeleton vectors of a rank hold the record planes zb .. z1 (zb = max(z0 - 1, 0)): one
 * ghost plane below (rank > 0) and the shared top plane z1, which is a ghost on every rank but
 * the last (there it is the Dirichlet plane k3, all zero).  Owned local planes are
 * [own_lo, own_hi): every global record plane is owned by exactly one rank.  A halo exchange
 * sends local plane own_lo to rank-1 (it lands in that rank's plane nplanes-1) and local plane
 * own_hi-1 to rank+1 (it lands in that rank's plane 0). */
typedef struct {
  int z0, z1;           /* owned element layers [z0, z1), global */
  int zb;               /* global index of local vertex plane 0 */
  int nplanes;          /* local vertex planes z1 - zb + 1 */
  int own_lo, own_hi;   /* owned local record planes */
  int lower, upper;     /* neighbour ranks, -1 if none */
} pmg_slab;
int pmg_slab_plan(int k3, int nranks, int rank, pmg_slab* out);   /* 0, or -1 on invalid input */

typedef struct {
  int cycles;         /* V-cycles performed (n_10 of P:636 when rtol = 1e-10); ipCG iterations for solver 1 */
  int converged;      /* 1 if ||r_n|| <= rtol ||r_0|| */
  double r0, r_final; /* ||r_hat||_2 over free skeleton unknowns, before / after */
  double rho;         /* (r_final / r0)^(1/cycles) */
  int coarse_iters;   /* total coarse CG iterations over the whole solve */
  double* history;    /* optional caller array (host) receiving ||r_n||, n = 0..cycles */
  int history_cap;    /* its capacity */
  /* phase times of the solve in milliseconds (CUDA events on the context stream):
   * condensation (Alg. 4 line 2, incl. the z-slab grid halo), the cycle loop (V-cycles + stopping
   * residuals + the per-cycle host read of ||r||), the coarse solves inside it (summed over cycles),
   * and the interior recovery */
  double t_condense, t_cycles, t_coarse, t_recover;
} pmg_report;

/* Multi-rank helpers.  pmg_nccl_unique_id writes a fresh 128-byte ncclUniqueId (call on rank 0
 * only).  pmg_loopback_create returns a hub for `nranks` contexts of one process (NULL on
 * failure); destroy it after every context that uses it. */
pmg_status pmg_nccl_unique_id(void* out128);
void* pmg_loopback_create(int nranks);
void pmg_loopback_destroy(void* hub);
/* the plan this context was set up with */
pmg_status pmg_slab_info(const pmg_ctx* ctx, pmg_slab* out);

/* Fill *opt with the defaults listed above. */
void pmg_default_options(pmg_options* opt);

/* Build the level hierarchy (host: GLL, 1-D mass/stiffness, element and star generalised
 * eigenpairs with identity padding at the boundary, weights, interpolation matrices, coarse
 * diagonal; device: tables and workspaces).  n_e[3] = (k1, k2, k3) >= 1; widths[d] is a HOST
 * array of k_d positive finite element widths; p in [2, 32] (p >= p0 for pmg_vcycle /
 * pmg_solve); lambda >= 0; opt may be NULL.  Errors: PMG_EINVAL, PMG_ENOMEM, PMG_ECUDA. */
pmg_status pmg_setup(pmg_ctx** out, const int n_e[3], const double* const widths[3], int p,
                     double lambda, const pmg_options* opt);
pmg_status pmg_destroy(pmg_ctx* ctx);

int pmg_num_levels(const pmg_ctx* ctx); /* L + 1, or -1 if ctx is NULL */
/* degree p_l, skeleton vector length (doubles, incl. padding records) and grid vector length */
pmg_status pmg_level_info(const pmg_ctx* ctx, int level, int* degree, long long* n_skel,
                          long long* n_grid);
/* 1-D GLL node coordinates of level `level` along direction d (HOST array of k_d p_l + 1). */
pmg_status pmg_grid_coords(const pmg_ctx* ctx, int level, int d, double* coords_host);

/* r_hat = f_hat - H_hat_l u_hat  (H_hat_l = sum_e Q_e (H_BB - H_BI H_II^-1 H_IB) Q_e^T,
 * P:117-123, evaluated matrix-free in O(p^3) per element: DESIGN.md "Residual kernel").
 * f_hat may be NULL, then r_hat = H_hat_l u_hat (operator apply).  u_hat and r_hat must not alias. */
pmg_status pmg_residual(pmg_ctx* ctx, int level, const double* u_hat, const double* f_hat,
                        double* r_hat);

/* u_hat += Smoother(r_hat): Alg. 2 with the star inverse of Alg. 1,
 * weights W_i, 8 race-free vertex colours.  r_hat and u_hat must not alias. */
pmg_status pmg_smooth(pmg_ctx* ctx, int level, const double* r_hat, double* u_hat);

/* f_coarse = J_hat_l^T r_fine (restriction, P:439, P:464 read as J_hat_l^T); level = fine level >= 1;
 * r_fine lives on level `level`, f_coarse on level-1 (overwritten). */
pmg_status pmg_restrict(pmg_ctx* ctx, int level, const double* r_fine, double* f_coarse);

/* u_fine += J_hat_l u_coarse (prolongation of the correction); level >= 1. */
pmg_status pmg_prolong(pmg_ctx* ctx, int level, const double* u_coarse, double* u_fine);

/* One V-cycle of Alg. 3 on the finest level: u_hat <- MultigridCycle(u_hat, f_hat).
 * With L = 0 it is u_hat <- u_hat + CG(f_hat - H_hat_0 u_hat) (reading R10b). */
pmg_status pmg_vcycle(pmg_ctx* ctx, double* u_hat, const double* f_hat);

/* f_hat = F_B - H_BI H_II^-1 F_I on the finest level (Alg. 4 line 2).  F_full is the grid
 * vector of the discrete weak right-hand side F = B f (pmg_weak_rhs); Dirichlet entries ignored. */
pmg_status pmg_condense(pmg_ctx* ctx, const double* F_full, double* f_hat);

/* u_full = (u_hat, H_II^-1 (F_I - H_IB u_hat)) on the finest level (Alg. 4 last line);
 * Dirichlet entries of u_full are written as 0. */
pmg_status pmg_recover(pmg_ctx* ctx, const double* u_hat, const double* F_full, double* u_full);

/* Alg. 4: condense, V-cycles from u_hat = 0 until ||r_hat|| <= rtol ||r_hat_0|| (reading R12) or
 * max_cycles, recover.  Synchronises the stream once per cycle to read the residual norm.
 * rep may be NULL.  Returns PMG_ENOCONV (with rep filled and u_full written) if not converged. */
pmg_status pmg_solve(pmg_ctx* ctx, const double* F_full, double* u_full, double rtol,
                     int max_cycles, pmg_report* rep);

/* Same as pmg_solve with HOST buffers: copies F_full_host (grid vector) to the device, solves,
 * copies u_full back to u_full_host, and synchronises.  Host buffers may be pageable or pinned. */
pmg_status pmg_solve_host(pmg_ctx* ctx, const double* F_full_host, double* u_full_host,
                          double rtol, int max_cycles, pmg_report* rep);

/* F = B f: GLL-lumped assembled mass times the nodal values f_nodal (grid vectors, finest level;
 * reading R8).  Dirichlet entries of F are written as 0. */
pmg_status pmg_weak_rhs(pmg_ctx* ctx, const double* f_nodal, double* F_full);

/* Layout converters between grid vectors and skeleton vectors of level `level`.
 * skel_from_grid copies free skeleton points (others 0); skel_to_grid writes the skeleton
 * values at skeleton points and 0 at element-interior and Dirichlet points. */
pmg_status pmg_skel_from_grid(pmg_ctx* ctx, int level, const double* grid, double* skel);
pmg_status pmg_skel_to_grid(pmg_ctx* ctx, int level, const double* skel, double* grid);

/* sqrt(sum of squares) of a skeleton vector of `level` (deterministic two-pass reduction);
 * synchronises the stream and returns the value in *out_host. */
pmg_status pmg_norm(pmg_ctx* ctx, int level, const double* x_hat, double* out_host);

/* Number of kernels this context launched since setup (all streams), for the bench's
 * gpu_launches count. */
long long pmg_launch_count(const pmg_ctx* ctx);

/* Kernel timing with CUDA events recorded on the context's stream (bench.py roofline).
 * pmg_timing_enable(ctx, 1) resets and starts bracketing every smoother sweep (the 8 colour
 * launches of the star kernel) and every residual evaluation (element kernel + gather) with
 * events; 0 stops.  pmg_timing_read synchronises the stream and returns the summed elapsed
 * milliseconds and the number of bracketed calls of `kind`:
 *   0 smoother sweep on the finest level, 1 residual on the finest level,
 *   2 smoother sweeps on all levels,      3 residuals on all levels (incl. coarse CG applies). */
pmg_status pmg_timing_enable(pmg_ctx* ctx, int enable);
pmg_status pmg_timing_read(pmg_ctx* ctx, int kind, double* total_ms, long long* count);

const char* pmg_last_error(void); /* thread-local message of the last failing call */

#ifdef __cplusplus
}
#endif
#endif /* PMG_H */
