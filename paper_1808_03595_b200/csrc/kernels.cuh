// Kernel declarations (kernels.cu) used by the orchestration layer (pmg_api.cu).
#pragma once
#include <cuda_runtime.h>

#include "pmg_internal.h"

namespace pmg {

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may be scheduled while
// its predecessor in the stream drains; it must execute pdl_wait() before touching anything the
// predecessor writes (griddepcontrol.wait returns once the predecessor has completed and its
// memory is visible; a no-op when the kernel was launched normally).  Prologues that only read
// setup tables run before the wait and overlap the predecessor's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// let the next kernel in the stream start launching once every block of this grid has executed this
// (its blocks then run their table prologue on free SM slots and wait in pdl_wait)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

bool pdl_enabled();   // PMG_NO_PDL=1 disables (A/B experiments)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

struct PcgState {
  double rz, bb, pq, alpha, beta, rr;
  int done, its, breakdown, its_sum;   // its_sum / breakdown accumulate over coarse solves (reset per pmg_solve)
};

// degree-specialised hot kernels (hot_kernels.cu)
// element operator Y_e = H_hat_e u_e of every element (etabP: padded table of 9 <= p <= 16, else unused)
cudaError_t launch_elem_apply(const LevelGeom& g, const double* u, const double* etab, const double* etabP, double lam,
                              double* Y, const int* done, cudaStream_t st);
// one colour of the star smoother (stabP: padded star table of 9 <= p <= 16, else unused)
cudaError_t launch_star(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                        double* u, const double* stab, const double* stabP, double lam, cudaStream_t st);
cudaError_t launch_gather_resid(const LevelGeom& g, const double* Y, const double* F, double* out, const int* done,
                                cudaStream_t st);
size_t hot_smem(int p, int which);   // which: 0 element, 1 star
// star smoother for 9 <= p <= 16 (star16.cu): padded star table stabP, rows of star16_stp(p) doubles
// per vertex line: S as NP x NP (zero padded), Lambda (padded with 1), s = S[c][:], w (padded 0)
cudaError_t launch_star16(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                          double* u, const double* stabP, double lam, cudaStream_t st);
int star16_np(int p);
cudaError_t star16_set_smem_attr();
// condensed element operator for 9 <= p <= 16 (elem16.cu): padded element table etabP, rows of
// elem16_etp(p) doubles per direction and 1-D element, built by elem16_table_row from an etab row
cudaError_t launch_elem16(const LevelGeom& g, const double* u, const double* etabP, double lam, double* Y, const int* done,
                          cudaStream_t st);
int elem16_etp(int p);
void elem16_table_row(int p, const double* et_row, double* out_row);
cudaError_t elem16_set_smem_attr();
// condensation (mode 0: Yc = H_BI H_II^-1 F_I on the face interiors) and interior recovery (mode 1:
// u_I = H_II^-1 (F_I - H_IB u_hat) into ug) for 9 <= p <= 16 (cr16.cu), DMMA cube transforms
cudaError_t launch_cr16(int mode, const LevelGeom& g, const double* Fg, const double* uh, const double* etabP, double lam,
                        double* Yc, double* ug, cudaStream_t st);
cudaError_t cr16_set_smem_attr();
cudaError_t hot_set_smem_attr(int bytes);

// p = 2 coarse operator tables (coarse_cg.cu): assembled 1-D lumped masses b_d[2k_d+1], assembled
// 1-D stiffness 5-point rows K_d[(2k_d+1) x 5] (offsets -2..2), per element c_e[6] and 1/D_e
struct CoarseTabs {
  const double *b1, *b2, *b3, *K1, *K2, *K3, *ce;
};

__global__ void k_pcg_coop_p2(LevelGeom g, CoarseTabs ct, const double* b, double* x, double* r, double* z,
                              double* pv, double* q, const double* dinv, double lam, double* part, PcgState* st,
                              double rtol, int maxit);
__global__ void k_pcg_coop_reg_p2(LevelGeom g, CoarseTabs ct, const double* b, double* xout, double* zpub,
                                  const double* dinv, double lam, double* part, PcgState* st, double rtol, int maxit);
__global__ void k_pcg_gv_p2(LevelGeom g, CoarseTabs ct, const double* b, double* xout, double* mbuf,
                            const double* dinv, double lam, double* part, PcgState* st, double rtol, int maxit);
// h-multigrid preconditioned coarse CG (reading R16): level 0 is the p0 = 2
// coarse system, level l + 1 the element-merged mesh; every level in p = 2 GRID layout
// (N_d = 2 k_d + 1 points per direction, x1 fastest; centres and non-free points held at 0).
constexpr int kMaxHLevels = 8;
struct HGridLev {
  int k1, k2, k3, N1, N2, N3, neu;
  long long n;                  // N1 N2 N3
  const double* b[3];           // assembled 1-D lumped mass per grid index
  const double* K[3];           // assembled 1-D stiffness, 5 entries (offsets -2..2) per grid index
  const double* E[3];           // per element index: {M[1], K[1][0], K[1][2], K[1][1]} (double4)
  const double* dinv;           // 1 / diag(H_hat) on free points, else 0 (grid)
  double *x, *f, *r;            // work vectors (grid)
  // transfer to level l + 1 (unused on the coarsest level)
  const int* pe[3];             // per fine grid index: coarse element
  const double* pw[3];          // per fine grid index: the 3 quadratic weights of that element's nodes
  const int* r0[3];             // per coarse grid index: first fine index with a nonzero weight
  const int* rn[3];             // ... and the count (<= 7)
  const double* rw[3];          // ... and the weights (7 per coarse index)
  double *t1, *t2;              // restriction scratch: N1c N2 N3 and N1c N2c N3 (this level's N2, N3)
};
struct HmgGridDev {
  int nlev;
  HGridLev L[kMaxHLevels];
  int ncf;                      // coarsest level solved exactly: its free unknowns (0: Jacobi sweeps instead)
  const int* cidx;              // their grid indices
  const double* cinv;           // dense inverse (ncf x ncf, row-major) of the coarsest condensed operator
  LevelGeom g0;                 // record geometry of level 0 (the CG's b / x layout)
};
__global__ void k_pcg_hmg_p2(HmgGridDev h, const double* b, double* xout, double* X, double* pv, double* q, double lam,
                             double* part, PcgState* st, double rtol, int maxit);
__global__ void k_resid_p2(LevelGeom g, CoarseTabs ct, const double* u, const double* f, double* r, double lam);
__global__ void k_build_coarse_ell(LevelGeom g, CoarseTabs ct, double lam, int* ellc, double* ella);
__global__ void k_pcg_gv_ell_p2(long long n, const double* b, double* xout, double* vec, double* mbuf, const double* dinv,
                                const int* ellc, const double* ella, double* part, PcgState* st, double rtol, int maxit);
size_t transfer_smem(int pf, int pc);
size_t condense_smem(int p, int ET, bool cube_in_smem);
size_t recover_smem(int p, int ET, bool cube_in_smem);

__global__ void k_skel_from_grid(LevelGeom g, const double* grid, double* skel);
__global__ void k_skel_to_grid(LevelGeom g, const double* skel, double* grid);
// skeleton values onto their grid points only (element interiors untouched; used by the recovery);
// hi_only: only the records of the three high box planes (v_d = k_d)
cudaError_t launch_skel_scatter(const LevelGeom& g, const double* skel, double* grid, cudaStream_t st, bool hi_only);
__global__ void k_weak_rhs(LevelGeom g, const double* b1, const double* b2, const double* b3, const double* f, double* F);
cudaError_t launch_restrict(const LevelGeom& gf, const LevelGeom& gc, const double* Jint, const double* rf, double* Z,
                            double* fc, double* uzero, int nt_local, size_t smem, int gather_blocks, cudaStream_t st);
__global__ void k_dot_fused(const double* a, const double* b, long long n, double* part, unsigned* ticket, double* out);
cudaError_t launch_prolong(const LevelGeom& gf, const LevelGeom& gc, const double* Jint, const double* uc, double* uf,
                           int nt, size_t smem, cudaStream_t st);
cudaError_t transfer_set_smem_attr(int bytes);

// element-centred block smoother (ec_smoother.cu)
size_t ec_smem(int p);
cudaError_t ec_set_smem_attr(int bytes);
void launch_ec(const LevelGeom& g, int c1, int c2, int c3, const double* r, double* u, const double* ectab,
               double lam, cudaStream_t st);
cudaError_t launch_condense_elem(int nb, int nt, size_t sm, cudaStream_t st, const LevelGeom& g, const double* Fg,
                                 const double* etab, double lam, double* Yc, double* cube_g);
cudaError_t launch_recover_elem(int nb, int nt, size_t sm, cudaStream_t st, const LevelGeom& g, const double* Fg,
                                const double* uh, const double* etab, double lam, double* ug, double* cube_g);
cudaError_t condense_recover_set_smem_attr(int bytes);
__global__ void k_condense_gather(LevelGeom g, const double* Fg, const double* Yc, double* fhat);
__global__ void k_dot_partial(const double* a, const double* b, long long n, double* part, const int* done);
__global__ void k_sum_final(const double* part, int nb, double* out);
__global__ void k_zero(double* x, long long n);
__global__ void k_axpy(double* y, const double* x, double a, long long n);
__global__ void k_ipcg_beta(double* ks);
__global__ void k_ipcg_dir(double* p, const double* z, const double* ks, long long n);
__global__ void k_ipcg_alpha(double* ks);
__global__ void k_ipcg_update(double* u, double* r, double* s, const double* p, const double* q, const double* ks,
                              long long n);
__global__ void k_pcg_init(const double* b, const double* dinv, double* x, double* r, double* z, double* pv,
                           long long n, double* part_rz, double* part_bb);
__global__ void k_pcg_init_final(const double* part_rz, const double* part_bb, int nb, PcgState* st);
__global__ void k_pcg_alpha(const double* part, int nb, PcgState* st);
__global__ void k_pcg_update(double* x, double* r, const double* pv, const double* q, long long n,
                             const PcgState* st, double* part);
__global__ void k_pcg_check(const double* part, int nb, PcgState* st, double rtol, int maxit);
__global__ void k_pcg_precond(const double* r, const double* dinv, double* z, long long n, const PcgState* st,
                              double* part);
__global__ void k_pcg_beta(const double* part, int nb, PcgState* st);
__global__ void k_pcg_pdir(double* pv, const double* z, long long n, const PcgState* st);

}  // namespace pmg
