// Kernel declarations (kernels.cu) used by the orchestration layer (pmg_api.cu).
#pragma once
#include <cuda_runtime.h>

#include "pmg_internal.h"

namespace pmg {

struct PcgState {
  double rz, bb, pq, alpha, beta, rr;
  int done, its, breakdown, its_sum;   // its_sum / breakdown accumulate over coarse solves (reset per pmg_solve)
};

// degree-specialised hot kernels (hot_kernels.cu)
cudaError_t launch_elem_apply(const LevelGeom& g, const double* u, const double* etab, double lam, double* Y,
                              const int* done, cudaStream_t st);
cudaError_t launch_star(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                        double* u, const double* stab, const double* stabT, double lam, cudaStream_t st);
cudaError_t launch_gather_resid(const LevelGeom& g, const double* Y, const double* F, double* out, const int* done,
                                cudaStream_t st);
size_t hot_smem(int p, int which);   // which: 0 element, 1 star
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
__global__ void k_pcg_cluster_p2(LevelGeom g, CoarseTabs ct, const double* b, double* xout, const double* dinv,
                                 double lam, int chunk, int halo, unsigned long long inv, PcgState* st, double rtol,
                                 int maxit);

size_t elem_apply_smem(int p, int ET);
size_t star_smem(int p, bool s_in_smem);
size_t transfer_smem(int pf, int pc);
size_t condense_smem(int p, int ET, bool cube_in_smem);
size_t recover_smem(int p, int ET, bool cube_in_smem);

__global__ void k_skel_from_grid(LevelGeom g, const double* grid, double* skel);
__global__ void k_skel_to_grid(LevelGeom g, const double* skel, double* grid);
__global__ void k_weak_rhs(LevelGeom g, const double* b1, const double* b2, const double* b3, const double* f, double* F);
__global__ void k_elem_apply(LevelGeom g, const double* u, const double* etab, double lam, double* Y, const int* done);
__global__ void k_gather_resid(LevelGeom g, const double* Y, const double* F, double* out, const int* done);
__global__ void k_star(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c, const double* r, double* u,
                       const double* stab, double lam, int s_in_smem);
__global__ void k_restrict_local(LevelGeom gf, int pc, const double* Jint, const double* rf, double* Z);
__global__ void k_restrict_gather(LevelGeom gc, const double* Z, double* fc);
__global__ void k_prolong(LevelGeom gf, LevelGeom gc, const double* Jint, const double* uc, double* uf);
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
