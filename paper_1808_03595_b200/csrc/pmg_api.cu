// C-ABI entry points (include/pmg.h) and the host orchestration of Alg. 2-4:
// smoother colour sweep, V-cycle, coarse CG driver, solve.  Citations: P:n = PAPER.md line n.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/pmg.h"
#include "comm.h"
#include "kernels.cuh"
#include "pmg_internal.h"

using namespace pmg;

namespace {
thread_local std::string g_err;

pmg_status fail(pmg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

constexpr int kThreads = 256;
constexpr int kRedBlocks = 592;  // 4 x 148 SMs; fixed so reductions are deterministic

int grid_for(long long n) {
  long long b = (n + kThreads - 1) / kThreads;
  return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

struct DevLevel {
  LevelGeom g;
  double* etab = nullptr;
  double* stab = nullptr;
  double* stabP = nullptr;   // padded star table of k_star16 (9 <= p <= 16)
  double* etabP = nullptr;   // padded element table of k_elem16 (9 <= p <= 16)
  double* ectab = nullptr;   // element-centred smoother tables (opt.smoother == 1)
  double* Jint = nullptr;
  double* u = nullptr;
  double* f = nullptr;
  double* r = nullptr;
};

}  // namespace

struct pmg_ctx {
  pmg_options opt;
  cudaStream_t st = nullptr;
  double lam = 0.0;
  int L = 0;
  std::vector<HostLevel> H;
  std::vector<DevLevel> D;
  double* Y = nullptr;       // element workspace  max_l nelem * YS
  double* Z = nullptr;       // restriction workspace
  double* cube = nullptr;    // condense/recover cube scratch (large p)
  int cube_blocks = 0;
  bool cube_in_smem = true;
  double* part = nullptr;    // reduction partials (2 x kRedBlocks)
  double* dres = nullptr;    // device scalar results
  unsigned* ticket = nullptr;  // k_dot_fused's arrival counter (0 between launches)
  PcgState* pcg = nullptr;
  double *cx = nullptr, *cr = nullptr, *cz = nullptr, *cp = nullptr, *cq = nullptr, *dinv = nullptr;
  double* bm[3] = {nullptr, nullptr, nullptr};
  double* Fdev = nullptr;    // grid buffers for pmg_solve_host (caller-sized: the rank's slab)
  double* Udev = nullptr;
  long long n_grid = 0;      // caller grid vector length (one GPU: whole grid; z-slab: planes z0 p .. z1 p)
  // z-slab decomposition (nranks > 1)
  Transport* tr = nullptr;   // nullptr on one GPU
  SlabPlan slab{};           // this rank's plan
  std::vector<SlabPlan> plans;
  LevelGeom g0g{};           // GLOBAL coarse geometry (the coarse CG runs replicated on every rank)
  double* f0g = nullptr;     // global coarse right-hand side / solution (nranks > 1)
  double* u0g = nullptr;
  double* agsend = nullptr;  // allgather staging: owned coarse planes, padded to ag_chunk
  double* agrecv = nullptr;  // nranks x ag_chunk
  long long ag_chunk = 0;
  double* cxl = nullptr;     // local coarse correction (L = 0, nranks > 1)
  double *kz = nullptr, *ks_ = nullptr, *kp = nullptr, *kq = nullptr, *kr = nullptr;   // ipCG vectors (Alg. 5)
  double* kscal = nullptr;   // ipCG device scalars [gamma, gamma0, delta, beta, q.p, alpha, breakdown]
  cudaGraphExec_t ipcg_exec = nullptr;
  double* Floc = nullptr;    // local grid buffers incl. the ghost element layer (nranks > 1)
  double* Uloc = nullptr;
  long long n_grid_loc = 0;
  long long launches = 0;
  int last_coarse_its = 0;
  long long coarse_its_total = 0;
  bool use_coop = false;     // coarse CG as one persistent cooperative kernel (p0 = 2)
  int coop_nb = 0;
  bool coop_reg = false;     // register-resident variant (one coarse unknown per thread)
  bool coop_gv = false;      // register-resident pipelined variant (one grid barrier per iteration)
  double* cgm = nullptr;     // its double-buffered m vector (2 n0)
  bool coop_ell = false;     // large coarse systems: pipelined grid-stride CG over ELL rows
  int ell_nb = 0;
  int* ellc = nullptr;       // 25 n0 column indices (column-major ELL), inside the ella block
  double* ella = nullptr;    // 25 n0 coefficients, then the indices (one block: one L2 window)
  cudaAccessPolicyWindow ell_win{};   // L2 persistence of the ELL rows (when the device allows it)
  bool ell_persist = false;
  bool l2_limit_set = false;          // this context raised cudaLimitPersistingL2CacheSize
  size_t l2_limit_prev = 0;           // ... from this value (restored on destroy)
  // h-multigrid preconditioned coarse CG (reading R16)
  bool use_hmg = false;
  int hmg_nb = 0;
  HmgGridDev hmg{};
  std::vector<HostLevel> hhost;      // h-levels 1.. (level 0 is H[0])
  std::vector<void*> hmg_allocs;     // device buffers owned by the h-hierarchy
  double *hpv = nullptr, *hq = nullptr, *hX = nullptr;   // h-multigrid CG grid vectors p, q, x
  double* ellv = nullptr;    // 8 n0 CG vectors
  double* ctab[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // CoarseTabs storage
  double* cV = nullptr;      // (unused)
  cudaGraphExec_t cycle_exec = nullptr;   // captured solve cycle (V-cycle + residual + norm^2)
  long long launches_per_cycle = 0;
  double* hres = nullptr;    // pinned host scalar
  bool no_graph = false;     // PMG_NO_GRAPH=1
  // pmg_report phase times: solve-phase events and the coarse-solve bracket (recorded as external
  // event nodes inside the captured cycle graph), created at setup
  cudaEvent_t ev_ph[4] = {nullptr, nullptr, nullptr, nullptr};   // start, condensed, cycles done, recovered
  cudaEvent_t ev_cg[2] = {nullptr, nullptr};                     // around the coarse solve of a V-cycle
  bool cg_mark = false;      // record ev_cg inside vcycle_dev (pmg_solve only)
  bool capturing = false;    // inside the cycle-graph capture: event records become external event nodes
  double t_coarse_acc = 0.0;
  // event timing (pmg_timing_enable)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Mark { int base; bool top; cudaEvent_t a, b; };   // base 0: smoother sweep, 1: residual
  std::vector<Mark> ev_marks;
};

namespace {
cudaEvent_t ev_get(pmg_ctx* c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void ev_reset(pmg_ctx* c) {
  for (auto& mk : c->ev_marks) { c->ev_pool.push_back(mk.a); c->ev_pool.push_back(mk.b); }
  c->ev_marks.clear();
}
struct TimedRegion {  // brackets one call with events on the context stream when timing is on
  pmg_ctx* c; int base; bool top; cudaEvent_t a = nullptr;
  TimedRegion(pmg_ctx* c_, int base_, bool top_) : c(c_), base(base_), top(top_) {
    if (c->timing) { a = ev_get(c); cudaEventRecord(a, c->st); }
  }
  ~TimedRegion() {
    if (!a) return;
    cudaEvent_t b = ev_get(c);
    cudaEventRecord(b, c->st);
    c->ev_marks.push_back({base, top, a, b});
  }
};
}  // namespace

#define LAUNCH_CHECK(ctx)                                                                   \
  do {                                                                                      \
    (ctx)->launches++;                                                                      \
    cudaError_t e_ = cudaGetLastError();                                                    \
    if (e_ != cudaSuccess) return fail(PMG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define CUDA_CHECK(call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return fail(PMG_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

namespace {

int* done_ptr(pmg_ctx* c) { return reinterpret_cast<int*>(reinterpret_cast<char*>(c->pcg) + offsetof(PcgState, done)); }

long long plane_len(const LevelGeom& g) { return (long long)g.V1 * g.V2 * g.RS; }

int nsm_dev(int dev) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// refresh the ghost record planes of a level-l skeleton vector from the neighbour ranks
pmg_status exchange(pmg_ctx* c, int l, double* x) {
  if (!c->tr) return PMG_OK;
  const LevelGeom& g = c->D[l].g;
  const long long n = plane_len(g);
  const bool lo = c->slab.lower >= 0, hi = c->slab.upper >= 0;
  std::string e = c->tr->halo(lo ? x + g.own_lo * n : nullptr, lo ? x : nullptr,
                              hi ? x + (long long)(g.own_hi - 1) * n : nullptr, hi ? x + (long long)(g.V3 - 1) * n : nullptr,
                              (size_t)n, c->st);
  if (!e.empty()) return fail(PMG_ENCCL, "halo exchange: " + e);
  return PMG_OK;
}

// ---------------------------------------------------------------- level operators (device)
pmg_status residual_dev(pmg_ctx* c, int l, const double* u, const double* f, double* r, const int* done = nullptr) {
  const DevLevel& D = c->D[l];
  TimedRegion tr(c, 1, l == c->L);
  if (D.g.p == 2 && l == 0 && c->ctab[0] && !c->tr && !D.g.per && !done) {   // p = 2: direct stencil form
    CoarseTabs ct{c->ctab[0], c->ctab[1], c->ctab[2], c->ctab[3], c->ctab[4], c->ctab[5], c->ctab[6]};
    k_resid_p2<<<grid_for(D.g.nskel), kThreads, 0, c->st>>>(D.g, ct, u, f, r, c->lam);
    LAUNCH_CHECK(c);
    return PMG_OK;
  }
  launch_elem_apply(D.g, u, D.etab, D.etabP, c->lam, c->Y, done, c->st);
  LAUNCH_CHECK(c);
  launch_gather_resid(D.g, c->Y, f, r, done, c->st);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status smooth_dev(pmg_ctx* c, int l, const double* r, double* u) {
  const DevLevel& D = c->D[l];
  const LevelGeom& g = D.g;
  TimedRegion tr(c, 0, l == c->L);
  if (c->opt.smoother == 1) {   // element-centred blocks (NEXT-4): 27 colours, element index mod 3
    for (int col = 0; col < 27; ++col) {
      launch_ec(g, col % 3, (col / 3) % 3, col / 9, r, u, D.ectab, c->lam, c->st);
      LAUNCH_CHECK(c);
    }
    return PMG_OK;
  }
  for (int col = 0; col < 8; ++col) {   // 8 vertex colours (parity), race-free
    // the z parity is that of the GLOBAL vertex plane, so a z-slab adds the colour corrections
    // of every point in the same order as one GPU (bitwise identical results)
    int c1 = col & 1, c2 = (col >> 1) & 1, c3 = ((col >> 2) & 1) ^ (g.zoff & 1);
    // vertices c_d, c_d + 2, ... <= k_d; a periodic direction stops below k_d (vertex k_d is vertex 0)
    int n1 = (g.per & 1) ? (g.k1 - c1 + 1) / 2 : (g.k1 - c1) / 2 + 1;
    int n2 = (g.per & 2) ? (g.k2 - c2 + 1) / 2 : (g.k2 - c2) / 2 + 1;
    int n3 = (g.per & 4) ? (g.k3 - c3 + 1) / 2 : (g.k3 - c3) / 2 + 1;
    long long nb = (long long)n1 * n2 * n3;
    launch_star(g, c1, c2, c3, n1, n2, nb, r, u, D.stab, D.stabP, c->lam, c->st);
    LAUNCH_CHECK(c);
  }
  return PMG_OK;
}

int zs_of(int pc) { int qc = pc + 1; return 3 * qc * qc + 3 * qc + 1; }

// per-record transfer kernels do O(p^3) work on O(p^2) data: size the block to the face
// (p <= 16: the register-tiled transforms have 3 (p - 1) row threads per record)
#ifndef PMG_TR_NT8
#define PMG_TR_NT8 32
#endif
int transfer_threads(int pf) { return pf <= 8 ? PMG_TR_NT8 : (pf <= 16 ? 64 : 256); }

pmg_status restrict_dev(pmg_ctx* c, int l, const double* rf, double* fc, double* uzero = nullptr) {
  const DevLevel& F = c->D[l];
  const DevLevel& C = c->D[l - 1];
  launch_restrict(F.g, C.g, F.Jint, rf, c->Z, fc, uzero, transfer_threads(F.g.p), transfer_smem(F.g.p, C.g.p),
                  grid_for(C.g.nskel), c->st);
  LAUNCH_CHECK(c);
  c->launches++;   // local + gather
  return PMG_OK;
}

pmg_status prolong_dev(pmg_ctx* c, int l, const double* uc, double* uf) {
  const DevLevel& F = c->D[l];
  const DevLevel& C = c->D[l - 1];
  launch_prolong(F.g, C.g, F.Jint, uc, uf, transfer_threads(F.g.p), transfer_smem(F.g.p, C.g.p), c->st);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status zero_dev(pmg_ctx* c, double* x, long long n) {
  launch_pdl(k_zero, dim3(grid_for(n)), dim3(kThreads), 0, c->st, x, n);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status dot_dev(pmg_ctx* c, const double* a, const double* b, long long n, double* out_dev) {
  launch_pdl(k_dot_fused, dim3(kRedBlocks), dim3(kThreads), 0, c->st, a, b, n, c->part, c->ticket, out_dev);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

// sum over the owned record planes of level l, summed over ranks (every rank gets the same value)
pmg_status dot_owned(pmg_ctx* c, int l, const double* a, const double* b, double* out_dev) {
  const LevelGeom& g = c->D[l].g;
  const long long n = plane_len(g), off = g.own_lo * n, cnt = (long long)(g.own_hi - g.own_lo) * n;
  pmg_status s = dot_dev(c, a + off, b + off, cnt, out_dev);
  if (s || !c->tr) return s;
  std::string e = c->tr->allreduce_sum(out_dev, 1, c->st);
  if (!e.empty()) return fail(PMG_ENCCL, "allreduce: " + e);
  return PMG_OK;
}

pmg_status norm_host(pmg_ctx* c, int l, const double* x, double* out) {
  pmg_status s = dot_owned(c, l, x, x, c->dres);
  if (s) return s;
  double h = 0;
  CUDA_CHECK(cudaMemcpyAsync(&h, c->dres, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_CHECK(cudaStreamSynchronize(c->st));
  *out = std::sqrt(h);
  return PMG_OK;
}

// Jacobi-PCG on H_hat_0 x = b from x = 0 (reading R11); device-resident scalars, the host
// polls the done flag every opt.coarse_check iterations.  Stops exactly at the first iteration
// with ||r|| <= rtol ||b|| (or at coarse_maxit), like the oracle.
pmg_status pcg_dev(pmg_ctx* c, const double* b, double* x) {
  TimedRegion tr(c, 2, true);
  const DevLevel& D = c->D[0];
  const long long n = c->g0g.nskel;
  if (c->use_coop) {   // one launch, no host synchronisation; statistics read at the end of solve
    LevelGeom g0 = c->g0g;
    double lam = c->lam, rtol = c->opt.coarse_rtol;
    int maxit = c->opt.coarse_maxit;
    double* part = c->part;
    PcgState* st = c->pcg;
    const double* dinv = c->dinv;
    CoarseTabs ct{c->ctab[0], c->ctab[1], c->ctab[2], c->ctab[3], c->ctab[4], c->ctab[5], c->ctab[6]};
    void* args[] = {&g0, &ct, (void*)&b, &x, &c->cr, &c->cz, &c->cp, &c->cq, (void*)&dinv, &lam, &part,
                    &st, &rtol, &maxit};
    void* args_reg[] = {&g0, &ct, (void*)&b, &x, &c->cz, (void*)&dinv, &lam, &part, &st, &rtol, &maxit};
    void* args_gv[] = {&g0, &ct, (void*)&b, &x, &c->cgm, (void*)&dinv, &lam, &part, &st, &rtol, &maxit};
    if (c->use_hmg) {   // CG preconditioned by the h-multigrid V-cycle (reading R16)
      void* args_h[] = {&c->hmg, (void*)&b, &x, &c->hX, &c->hpv, &c->hq, &lam, &part, &st, &rtol, &maxit};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c->hmg_nb);
      cfg.blockDim = dim3(kThreads);
      cfg.stream = c->st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void*)k_pcg_hmg_p2, args_h));
      c->launches++;
      return PMG_OK;
    }
    if (c->coop_ell && rtol >= 1e-11) {   // large coarse system: grid-stride pipelined CG on ELL rows
      long long n0 = g0.nskel;
      void* args_ell[] = {&n0, (void*)&b, &x, &c->ellv, &c->cgm, (void*)&dinv, &c->ellc, &c->ella, &part, &st, &rtol, &maxit};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c->ell_nb);
      cfg.blockDim = dim3(kThreads);
      cfg.stream = c->st;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[1].val.accessPolicyWindow = c->ell_win;
      cfg.attrs = attr;
      cfg.numAttrs = c->ell_persist ? 2 : 1;
      CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void*)k_pcg_gv_ell_p2, args_ell));
      c->launches++;
      return PMG_OK;
    }
    // the pipelined recurrence for the performance tolerance; the two-barrier kernel for the very
    // tight parity tolerances (attainable accuracy, see coarse_cg.cu)
    const bool gv = c->coop_gv && rtol >= 1e-11;
    const void* fn = gv ? (const void*)k_pcg_gv_p2 : (c->coop_reg ? (const void*)k_pcg_coop_reg_p2 : (const void*)k_pcg_coop_p2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->coop_nb);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // capturable cooperative launch
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelExC(&cfg, fn, gv ? args_gv : (c->coop_reg ? args_reg : args)));
    c->launches++;
    return PMG_OK;
  }
  (void)D;
  double* part2 = c->part + kRedBlocks;
  int* done = done_ptr(c);
  k_pcg_init<<<kRedBlocks, kThreads, 0, c->st>>>(b, c->dinv, x, c->cr, c->cz, c->cp, n, c->part, part2);
  LAUNCH_CHECK(c);
  k_pcg_init_final<<<1, 1024, 0, c->st>>>(c->part, part2, kRedBlocks, c->pcg);
  LAUNCH_CHECK(c);
  PcgState hs;
  const int chk = std::max(1, c->opt.coarse_check);
  for (;;) {
    for (int k = 0; k < chk; ++k) {
      pmg_status s = residual_dev(c, 0, c->cp, nullptr, c->cq, done);   // q = H p
      if (s) return s;
      k_dot_partial<<<kRedBlocks, kThreads, 0, c->st>>>(c->cp, c->cq, n, c->part, done);
      LAUNCH_CHECK(c);
      k_pcg_alpha<<<1, 1024, 0, c->st>>>(c->part, kRedBlocks, c->pcg);
      LAUNCH_CHECK(c);
      k_pcg_update<<<kRedBlocks, kThreads, 0, c->st>>>(x, c->cr, c->cp, c->cq, n, c->pcg, c->part);
      LAUNCH_CHECK(c);
      k_pcg_check<<<1, 1024, 0, c->st>>>(c->part, kRedBlocks, c->pcg, c->opt.coarse_rtol, c->opt.coarse_maxit);
      LAUNCH_CHECK(c);
      k_pcg_precond<<<kRedBlocks, kThreads, 0, c->st>>>(c->cr, c->dinv, c->cz, n, c->pcg, c->part);
      LAUNCH_CHECK(c);
      k_pcg_beta<<<1, 1024, 0, c->st>>>(c->part, kRedBlocks, c->pcg);
      LAUNCH_CHECK(c);
      k_pcg_pdir<<<kRedBlocks, kThreads, 0, c->st>>>(c->cp, c->cz, n, c->pcg);
      LAUNCH_CHECK(c);
    }
    CUDA_CHECK(cudaMemcpyAsync(&hs, c->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, c->st));
    CUDA_CHECK(cudaStreamSynchronize(c->st));
    if (hs.done) break;
  }
  c->last_coarse_its = hs.its;
  c->coarse_its_total += hs.its;
  if (hs.breakdown) return fail(PMG_EBREAKDOWN, "coarse CG breakdown: p^T H p <= 0");
  return PMG_OK;
}

int nu_of(const pmg_ctx* c, int l) { return c->opt.schedule == 0 ? 1 : (1 << (c->L - l)); }

// x_local = CG(H_hat_0, b_local).  One GPU: directly.  z-slabs: the owned coarse planes of every
// rank are gathered into the global coarse vector, every rank runs the same (bitwise identical)
// CG on the whole coarse system -- no collective inside the iteration -- and keeps its local
// planes, ghosts included (SURVEY 8(e) / NEXT-2 "allgather F_0 and solve redundantly").
pmg_status coarse_solve(pmg_ctx* c, const double* b, double* x) {
  if (!c->tr) return pcg_dev(c, b, x);
  const LevelGeom& g = c->D[0].g;
  const long long n = plane_len(g);
  const long long own = (long long)(g.own_hi - g.own_lo) * n;
  CUDA_CHECK(cudaMemsetAsync(c->agsend, 0, c->ag_chunk * sizeof(double), c->st));
  CUDA_CHECK(cudaMemcpyAsync(c->agsend, b + g.own_lo * n, own * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  std::string e = c->tr->allgather(c->agsend, c->agrecv, (size_t)c->ag_chunk, c->st);
  if (!e.empty()) return fail(PMG_ENCCL, "allgather: " + e);
  for (size_t q = 0; q < c->plans.size(); ++q) {
    const SlabPlan& P = c->plans[q];
    const long long cnt = (long long)(P.own_hi - P.own_lo) * n;
    CUDA_CHECK(cudaMemcpyAsync(c->f0g + (long long)P.z0 * n, c->agrecv + (long long)q * c->ag_chunk, cnt * sizeof(double),
                               cudaMemcpyDeviceToDevice, c->st));
  }
  c->tr->exclusive_begin();
  pmg_status s = pcg_dev(c, c->f0g, c->u0g);
  e = c->tr->exclusive_end(c->st);
  if (s) return s;
  if (!e.empty()) return fail(PMG_ECUDA, "coarse CG: " + e);
  CUDA_CHECK(cudaMemcpyAsync(x, c->u0g + (long long)c->slab.zb * n, g.nskel * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  return PMG_OK;
}

// residual with the halo refresh of u before and of r after (no-ops on one GPU)
pmg_status residual_x(pmg_ctx* c, int l, double* u, const double* f, double* r) {
  pmg_status s;
  if ((s = exchange(c, l, u))) return s;
  if ((s = residual_dev(c, l, u, f, r))) return s;
  return exchange(c, l, r);
}

// pmg_report t_coarse: event i (0 before, 1 after) around the coarse solve of a V-cycle inside pmg_solve
pmg_status mark_coarse(pmg_ctx* c, int i) {
  if (!c->cg_mark) return PMG_OK;
  if (c->capturing) CUDA_CHECK(cudaEventRecordWithFlags(c->ev_cg[i], c->st, cudaEventRecordExternal));
  else CUDA_CHECK(cudaEventRecord(c->ev_cg[i], c->st));
  return PMG_OK;
}

// Alg. 3.  r_top_valid: D[L].r already holds f - H u (saves one residual).
pmg_status vcycle_dev(pmg_ctx* c, double* u, const double* f, bool r_top_valid) {
  const int L = c->L;
  pmg_status s;
  // z-slabs: every operator reads ghost planes that the exchanges below refresh:
  // residual needs u's, smoother and restriction r's / f's, prolongation the coarse u's.
  if (L == 0) {  // reading R10b: u <- u + CG(f - H_0 u)
    DevLevel& D = c->D[0];
    if (!r_top_valid && (s = residual_x(c, 0, u, f, D.r))) return s;
    double* cx = c->tr ? c->cxl : c->cx;
    if ((s = mark_coarse(c, 0))) return s;
    if ((s = coarse_solve(c, D.r, cx))) return s;
    if ((s = mark_coarse(c, 1))) return s;
    k_axpy<<<grid_for(D.g.nskel), kThreads, 0, c->st>>>(u, cx, 1.0, D.g.nskel);
    LAUNCH_CHECK(c);
    return PMG_OK;
  }
  for (int l = L; l >= 1; --l) {
    DevLevel& D = c->D[l];
    double* ul = (l == L) ? u : D.u;
    const double* fl = (l == L) ? f : D.f;
    bool r_valid = (l == L) && r_top_valid;
    bool u_zero = false;
    if (l != L) u_zero = true;   // zeroed by the restriction kernel that produced f_l
    for (int i = 0; i < nu_of(c, l); ++i) {
      const double* rin = D.r;
      if (u_zero) rin = fl;                       // f - H 0 = f exactly
      else if (!r_valid && (s = residual_x(c, l, ul, fl, D.r))) return s;
      if ((s = smooth_dev(c, l, rin, ul))) return s;
      r_valid = false;
      u_zero = false;
    }
    if ((s = residual_x(c, l, ul, fl, D.r))) return s;
    // u_(l-1) <- 0 (Alg. 3) rides along with the restriction into level l-1 (not for the coarse CG's level)
    if ((s = restrict_dev(c, l, D.r, c->D[l - 1].f, l - 1 >= 1 ? c->D[l - 1].u : nullptr))) return s;
    if (l - 1 >= 1 && (s = exchange(c, l - 1, c->D[l - 1].f))) return s;
  }
  if ((s = mark_coarse(c, 0))) return s;
  if ((s = coarse_solve(c, c->D[0].f, c->D[0].u))) return s;
  if ((s = mark_coarse(c, 1))) return s;
  for (int l = 1; l <= L; ++l) {
    DevLevel& D = c->D[l];
    double* ul = (l == L) ? u : D.u;
    const double* fl = (l == L) ? f : D.f;
    if (l - 1 >= 1 && (s = exchange(c, l - 1, c->D[l - 1].u))) return s;
    if ((s = prolong_dev(c, l, c->D[l - 1].u, ul))) return s;
    for (int i = 0; i < nu_of(c, l); ++i) {
      if ((s = residual_x(c, l, ul, fl, D.r))) return s;
      if ((s = smooth_dev(c, l, D.r, ul))) return s;
    }
  }
  return PMG_OK;
}

pmg_status condense_dev(pmg_ctx* c, const double* F, double* fhat) {
  const DevLevel& D = c->D[c->L];
  if (D.etabP) {   // 9 <= p <= 16: DMMA cube transforms (cr16.cu)
    launch_cr16(0, D.g, F, nullptr, D.etabP, c->lam, c->Y, nullptr, c->st);
  } else {
    size_t sm = condense_smem(D.g.p, D.g.ET, c->cube_in_smem);
    int nb = c->cube_in_smem ? (int)std::min<long long>(D.g.nelem, 148LL * 8) : c->cube_blocks;
    launch_condense_elem(nb, kThreads, sm, c->st, D.g, F, D.etab, c->lam, c->Y, c->cube_in_smem ? nullptr : c->cube);
  }
  LAUNCH_CHECK(c);
  k_condense_gather<<<grid_for(D.g.nskel), kThreads, 0, c->st>>>(D.g, F, c->Y, fhat);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status recover_dev(pmg_ctx* c, const double* uhat, const double* F, double* ufull) {
  const DevLevel& D = c->D[c->L];
  if (D.etabP) {
    // 9 <= p <= 16: each element writes its grid block [0, p)^3 (interior and the skeleton points of its
    // vertex record), the high box planes come from their records
    launch_cr16(1, D.g, F, uhat, D.etabP, c->lam, nullptr, ufull, c->st);
    LAUNCH_CHECK(c);
    launch_skel_scatter(D.g, uhat, ufull, c->st, true);
  } else {
    // skeleton points from u_hat (non-free entries are zero), then every element interior
    launch_skel_scatter(D.g, uhat, ufull, c->st, false);
    LAUNCH_CHECK(c);
    size_t sm = recover_smem(D.g.p, D.g.ET, c->cube_in_smem);
    int nb = c->cube_in_smem ? (int)std::min<long long>(D.g.nelem, 148LL * 8) : c->cube_blocks;
    launch_recover_elem(nb, kThreads, sm, c->st, D.g, F, uhat, D.etab, c->lam, ufull, c->cube_in_smem ? nullptr : c->cube);
  }
  LAUNCH_CHECK(c);
  return PMG_OK;
}

// One iteration of Alg. 5 (ipCG with a V-cycle preconditioner) on the device; ends with
// ||r||^2 in dres.  Vectors: r = kr, s = ks_, p = kp, q = kq, z = kz; scalars in kscal.
pmg_status ipcg_iter(pmg_ctx* c) {
  DevLevel& D = c->D[c->L];
  const long long n = D.g.nskel;
  pmg_status s;
  // z = MultigridCycle(0, r): the top-level residual of u = 0 is r itself (no operator call)
  CUDA_CHECK(cudaMemcpyAsync(D.r, c->kr, n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  if ((s = zero_dev(c, c->kz, n))) return s;
  if ((s = vcycle_dev(c, c->kz, c->kr, true))) return s;
  if ((s = dot_owned(c, c->L, c->kz, c->kr, c->kscal + 0))) return s;   // gamma  = z^T r
  if ((s = dot_owned(c, c->L, c->kz, c->ks_, c->kscal + 1))) return s;  // gamma0 = z^T s
  k_ipcg_beta<<<1, 1, 0, c->st>>>(c->kscal);                              // beta = (gamma - gamma0) / delta
  LAUNCH_CHECK(c);
  k_ipcg_dir<<<grid_for(n), kThreads, 0, c->st>>>(c->kp, c->kz, c->kscal, n);   // p = beta p + z
  LAUNCH_CHECK(c);
  if ((s = residual_x(c, c->L, c->kp, nullptr, c->kq))) return s;         // q = H p
  if ((s = dot_owned(c, c->L, c->kq, c->kp, c->kscal + 4))) return s;   // q^T p
  k_ipcg_alpha<<<1, 1, 0, c->st>>>(c->kscal);                             // alpha = gamma / q^T p
  LAUNCH_CHECK(c);
  k_ipcg_update<<<grid_for(n), kThreads, 0, c->st>>>(D.u, c->kr, c->ks_, c->kp, c->kq, c->kscal, n);
  LAUNCH_CHECK(c);
  return dot_owned(c, c->L, c->kr, c->kr, c->dres);
}

pmg_status solve_dev(pmg_ctx* c, const double* F, double* ufull, double rtol, int max_cycles, pmg_report* rep) {
  DevLevel& D = c->D[c->L];
  pmg_status s;
  c->coarse_its_total = 0;
  c->t_coarse_acc = 0.0;
  CUDA_CHECK(cudaEventRecord(c->ev_ph[0], c->st));
  CUDA_CHECK(cudaMemsetAsync(c->pcg, 0, sizeof(PcgState), c->st));
  const double* Floc = F;
  if (c->tr) {
    // the caller's slab holds grid planes z0 p .. z1 p; the local buffer adds the ghost element
    // layer below (planes zb p .. z0 p - 1), received from the lower rank, for the condensation
    const LevelGeom& g = D.g;
    const long long pl = (long long)(g.k1 * g.p + 1) * (g.k2 * g.p + 1);
    const long long ghost = (long long)(c->slab.z0 - c->slab.zb) * g.p * pl;
    CUDA_CHECK(cudaMemcpyAsync(c->Floc + ghost, F, c->n_grid * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    const long long n = (long long)g.p * pl;   // the p planes below the rank's top plane go up
    std::string e = c->tr->shift_up(c->Floc + c->n_grid_loc - pl - n, c->Floc, (size_t)n, c->st);
    if (!e.empty()) return fail(PMG_ENCCL, "grid halo: " + e);
    Floc = c->Floc;
  }
  if ((s = condense_dev(c, Floc, D.f))) return s;
  if ((s = exchange(c, c->L, D.f))) return s;
  CUDA_CHECK(cudaEventRecord(c->ev_ph[1], c->st));
  if ((s = zero_dev(c, D.u, D.g.nskel))) return s;
  if ((s = residual_x(c, c->L, D.u, D.f, D.r))) return s;
  double r0, rn;
  if ((s = norm_host(c, c->L, D.r, &r0))) return s;
  rn = r0;
  int cycles = 0;
  if (rep && rep->history && rep->history_cap > 0) rep->history[0] = r0;
  const bool krylov = c->opt.solver == 1;
  if (krylov) {   // Alg. 5 initialisation: r = F - H u (above), s = r, p = 0, delta = 1
    const long long n = D.g.nskel;
    CUDA_CHECK(cudaMemcpyAsync(c->kr, D.r, n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CUDA_CHECK(cudaMemcpyAsync(c->ks_, D.r, n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CUDA_CHECK(cudaMemsetAsync(c->kp, 0, n * sizeof(double), c->st));
    const double init[8] = {0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    CUDA_CHECK(cudaMemcpyAsync(c->kscal, init, sizeof(init), cudaMemcpyHostToDevice, c->st));
    CUDA_CHECK(cudaStreamSynchronize(c->st));   // `init` is a host stack array
  }
  // One cycle = V-cycle + residual + ||r||^2 into dres.  When the whole cycle is free of host
  // synchronisation (cooperative coarse CG) it is captured once into a CUDA graph and replayed:
  // ~60 kernel launches per cycle become one graph launch.
  const bool graph_ok = c->use_coop && c->st != nullptr && !c->timing && !c->no_graph && (!c->tr || c->tr->graph_safe());
  c->cg_mark = true;   // bracket the coarse solve of every V-cycle (pmg_report t_coarse)
  if (graph_ok && !c->cycle_exec) {
    long long l0 = c->launches;
    cudaGraph_t gr = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    pmg_status cs;
    c->capturing = true;
    if (krylov) {
      cs = ipcg_iter(c);
    } else {
      cs = vcycle_dev(c, D.u, D.f, true);
      if (!cs) cs = residual_x(c, c->L, D.u, D.f, D.r);
      if (!cs) cs = dot_owned(c, c->L, D.r, D.r, c->dres);
    }
    c->capturing = false;
    cudaError_t ce = cudaStreamEndCapture(c->st, &gr);
    if (cs) { if (gr) cudaGraphDestroy(gr); return cs; }
    if (ce != cudaSuccess) return fail(PMG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&c->cycle_exec, gr, 0);
    cudaGraphDestroy(gr);
    if (ce != cudaSuccess) { c->cycle_exec = nullptr; return fail(PMG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce)); }
    c->launches_per_cycle = c->launches - l0;
    c->launches = l0;
  }
  while (rn > rtol * r0 && cycles < max_cycles) {
    if (graph_ok) {
      CUDA_CHECK(cudaGraphLaunch(c->cycle_exec, c->st));
      c->launches += c->launches_per_cycle;
      CUDA_CHECK(cudaMemcpyAsync(c->hres, c->dres, sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CUDA_CHECK(cudaStreamSynchronize(c->st));
      rn = std::sqrt(*c->hres);
    } else if (krylov) {
      if ((s = ipcg_iter(c))) return s;
      double h = 0;
      CUDA_CHECK(cudaMemcpyAsync(&h, c->dres, sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CUDA_CHECK(cudaStreamSynchronize(c->st));
      rn = std::sqrt(h);
    } else {
      if ((s = vcycle_dev(c, D.u, D.f, true))) return s;
      if ((s = residual_x(c, c->L, D.u, D.f, D.r))) return s;
      if ((s = norm_host(c, c->L, D.r, &rn))) return s;
    }
    ++cycles;
    if (rep && rep->history && cycles < rep->history_cap) rep->history[cycles] = rn;
    float cms = 0.f;   // the cycle's stream work has completed (its residual norm was read)
    if (cudaEventElapsedTime(&cms, c->ev_cg[0], c->ev_cg[1]) == cudaSuccess) c->t_coarse_acc += cms;
    else cudaGetLastError();   // not recorded (no coarse solve): not an error of the solve
  }
  c->cg_mark = false;
  CUDA_CHECK(cudaEventRecord(c->ev_ph[2], c->st));
  if (c->tr) {
    if ((s = exchange(c, c->L, D.u))) return s;
    if ((s = recover_dev(c, D.u, c->Floc, c->Uloc))) return s;
    const LevelGeom& g = D.g;
    const long long pl = (long long)(g.k1 * g.p + 1) * (g.k2 * g.p + 1);
    const long long ghost = (long long)(c->slab.z0 - c->slab.zb) * g.p * pl;
    CUDA_CHECK(cudaMemcpyAsync(ufull, c->Uloc + ghost, c->n_grid * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  } else if ((s = recover_dev(c, D.u, F, ufull))) {
    return s;
  }
  if (c->use_coop) {
    PcgState hs;
    CUDA_CHECK(cudaMemcpyAsync(&hs, c->pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, c->st));
    CUDA_CHECK(cudaStreamSynchronize(c->st));
    c->coarse_its_total = hs.its_sum;
    if (hs.breakdown) return fail(PMG_EBREAKDOWN, "coarse CG breakdown: p^T H p <= 0");
  }
  if (krylov) {
    double ks[8];
    CUDA_CHECK(cudaMemcpyAsync(ks, c->kscal, sizeof(ks), cudaMemcpyDeviceToHost, c->st));
    CUDA_CHECK(cudaStreamSynchronize(c->st));
    if (ks[6] != 0.0) return fail(PMG_EBREAKDOWN, "ipCG breakdown: p^T H p <= 0");
  }
  CUDA_CHECK(cudaEventRecord(c->ev_ph[3], c->st));
  bool conv = rn <= rtol * r0;
  if (rep) {
    float t[3] = {0.f, 0.f, 0.f};
    CUDA_CHECK(cudaEventSynchronize(c->ev_ph[3]));
    for (int i = 0; i < 3; ++i) CUDA_CHECK(cudaEventElapsedTime(&t[i], c->ev_ph[i], c->ev_ph[i + 1]));
    rep->t_condense = t[0];
    rep->t_cycles = t[1];
    rep->t_recover = t[2];
    rep->t_coarse = c->t_coarse_acc;
    rep->cycles = cycles;
    rep->converged = conv ? 1 : 0;
    rep->r0 = r0;
    rep->r_final = rn;
    rep->rho = (cycles > 0 && r0 > 0) ? std::pow(rn / r0, 1.0 / cycles) : 0.0;
    rep->coarse_iters = (int)c->coarse_its_total;
  }
  if (!conv) return fail(PMG_ENOCONV, "pmg_solve: max_cycles reached before rtol");
  return PMG_OK;
}

void free_ctx(pmg_ctx* c) {
  if (!c) return;
  for (auto& D : c->D) {
    cudaFree(D.etab); cudaFree(D.stab); cudaFree(D.stabP); cudaFree(D.etabP); cudaFree(D.ectab); cudaFree(D.Jint);
    cudaFree(D.u); cudaFree(D.f); cudaFree(D.r);
  }
  cudaFree(c->ticket);
  cudaFree(c->Y); cudaFree(c->Z); cudaFree(c->cube); cudaFree(c->part); cudaFree(c->dres); cudaFree(c->pcg);
  cudaFree(c->cgm); cudaFree(c->ella); cudaFree(c->ellv);
  for (void* a : c->hmg_allocs) cudaFree(a);
  cudaFree(c->hpv); cudaFree(c->hq); cudaFree(c->hX);
  cudaFree(c->cx); cudaFree(c->cr); cudaFree(c->cz); cudaFree(c->cp); cudaFree(c->cq); cudaFree(c->dinv);
  for (int d = 0; d < 3; ++d) cudaFree(c->bm[d]);
  cudaFree(c->Fdev); cudaFree(c->Udev);
  cudaFree(c->f0g); cudaFree(c->u0g); cudaFree(c->agsend); cudaFree(c->agrecv); cudaFree(c->cxl);
  cudaFree(c->Floc); cudaFree(c->Uloc);
  cudaFree(c->kz); cudaFree(c->ks_); cudaFree(c->kp); cudaFree(c->kq); cudaFree(c->kr); cudaFree(c->kscal);
  if (c->ipcg_exec) cudaGraphExecDestroy(c->ipcg_exec);
  delete c->tr;
  for (int i = 0; i < 7; ++i) cudaFree(c->ctab[i]);
  cudaFree(c->cV);
  if (c->cycle_exec) cudaGraphExecDestroy(c->cycle_exec);
  if (c->hres) cudaFreeHost(c->hres);
  ev_reset(c);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_ph) if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_cg) if (e) cudaEventDestroy(e);
  delete c;
}

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, count) * sizeof(T));
}

pmg_status upload(double** dst, const std::vector<double>& v) {
  if (dalloc(dst, v.size()) != cudaSuccess) return fail(PMG_ENOMEM, "cudaMalloc failed (tables)");
  if (!v.empty()) CUDA_CHECK(cudaMemcpy(*dst, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
  return PMG_OK;
}

pmg_status check_level(const pmg_ctx* c, int level) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (level < 0 || level > c->L) return fail(PMG_EINVAL, "level out of range");
  return PMG_OK;
}

}  // namespace

extern "C" {

void pmg_default_options(pmg_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->p0 = 2;
  o->weight_degree = 7;
  o->schedule = 0;
  o->solver = 0;
  o->neumann = 0;
  o->periodic = 0;
  o->coarse_rtol = 1e-4;
  o->coarse_maxit = 10000;
  o->coarse_check = 8;
  o->coarse_solver = 0;
  o->smoother = 0;
  o->rank = 0;
  o->nranks = 1;
  o->nccl_id = nullptr;
  o->stream = nullptr;
}

const char* pmg_last_error(void) { return g_err.c_str(); }

pmg_status pmg_setup(pmg_ctx** out, const int n_e[3], const double* const widths[3], int p, double lambda,
                     const pmg_options* opt) {
  if (!out) return fail(PMG_EINVAL, "out is NULL");
  *out = nullptr;
  if (!n_e || !widths) return fail(PMG_EINVAL, "n_e / widths is NULL");
  for (int d = 0; d < 3; ++d) {
    if (n_e[d] < 1) return fail(PMG_EINVAL, "n_e[d] must be >= 1");
    if (!widths[d]) return fail(PMG_EINVAL, "widths[d] is NULL");
    for (int e = 0; e < n_e[d]; ++e)
      if (!(widths[d][e] > 0.0) || !std::isfinite(widths[d][e])) return fail(PMG_EINVAL, "element widths must be positive and finite");
  }
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(PMG_EINVAL, "lambda must be >= 0 and finite");
  pmg_options o;
  pmg_default_options(&o);
  if (opt) o = *opt;
  if (o.p0 < 2) return fail(PMG_EINVAL, "p0 must be >= 2");
  if (p < 2 || p > 32) return fail(PMG_EINVAL, "degree p must be in [2, 32]");
  if (p < o.p0) return fail(PMG_EINVAL, "p must be >= p0");
  if (o.weight_degree != 7) return fail(PMG_EINVAL, "only weight_degree = 7 is implemented (P:316)");
  if (o.schedule != 0 && o.schedule != 1) return fail(PMG_EINVAL, "schedule must be 0 or 1");
  if (o.solver != 0 && o.solver != 1) return fail(PMG_EINVAL, "solver must be 0 (MG) or 1 (ipCG)");
  if (o.coarse_solver < 0 || o.coarse_solver > 2) return fail(PMG_EINVAL, "coarse_solver must be 0 (auto), 1 (Jacobi) or 2 (h-multigrid)");
  if (o.neumann < 0 || o.neumann > 63) return fail(PMG_EINVAL, "neumann is a 6-bit face mask");
  if (o.neumann == 63 && lambda == 0.0) return fail(PMG_EINVAL, "all-Neumann Poisson (lambda = 0) is singular");
  if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks) return fail(PMG_EINVAL, "need 0 <= rank < nranks");
  if (o.nranks > 1 && n_e[2] < o.nranks) return fail(PMG_EINVAL, "z-slabs: k3 >= nranks required");
  if (o.nranks > 1 && o.p0 != 2) return fail(PMG_EINVAL, "z-slabs: the replicated coarse CG needs p0 = 2");
  if (!(o.coarse_rtol > 0.0) || o.coarse_maxit < 1) return fail(PMG_EINVAL, "coarse_rtol > 0 and coarse_maxit >= 1 required");
  if (o.smoother != 0 && o.smoother != 1) return fail(PMG_EINVAL, "smoother must be 0 (vertex stars) or 1 (element-centred blocks)");
  if (o.smoother == 1 && o.nranks > 1) return fail(PMG_EINVAL, "the element-centred smoother runs on one GPU (nranks = 1)");
  if (o.smoother == 1 && p > 16) return fail(PMG_EINVAL, "the element-centred smoother supports p <= 16");
  if (o.periodic < 0 || o.periodic > 7) return fail(PMG_EINVAL, "periodic is a 3-bit direction mask");
  if (o.periodic) {
    for (int d = 0; d < 3; ++d) {
      if (!((o.periodic >> d) & 1)) continue;
      if (n_e[d] < 2 || n_e[d] % 2) return fail(PMG_EINVAL, "a periodic direction needs an even k_d >= 2 (8 star colours)");
      if ((o.neumann >> (2 * d)) & 3) return fail(PMG_EINVAL, "a periodic direction has no Neumann faces");
    }
    if (o.nranks > 1) return fail(PMG_EINVAL, "periodic directions run on one GPU (nranks = 1)");
    if (o.smoother == 1) return fail(PMG_EINVAL, "periodic directions: vertex-star smoother only");
    if (o.coarse_solver == 2) return fail(PMG_EINVAL, "periodic directions: Jacobi-PCG coarse solver only");
    if (o.periodic == 7 && o.neumann == 0 && lambda == 0.0) return fail(PMG_EINVAL, "fully periodic Poisson (lambda = 0) is singular");
  }

  pmg_ctx* c = new (std::nothrow) pmg_ctx();
  if (!c) return fail(PMG_ENOMEM, "host allocation failed");
  c->opt = o;
  slab_plan(n_e[2], o.nranks, o.rank, &c->slab);
  for (int q = 0; q < o.nranks; ++q) { SlabPlan P; slab_plan(n_e[2], o.nranks, q, &P); c->plans.push_back(P); }
  {
    std::string e = make_transport(o.rank, o.nranks, o.nccl_id, o.loopback, &c->tr);
    if (!e.empty()) { delete c; return fail(o.loopback ? PMG_EINVAL : PMG_ENCCL, e); }
  }
  c->st = static_cast<cudaStream_t>(o.stream);
  c->lam = lambda;
  int L = 0;
  while ((o.p0 << L) < p) ++L;
  c->L = L;
  std::vector<int> deg;
  for (int l = 0; l < L; ++l) deg.push_back(o.p0 << l);
  deg.push_back(p);
  c->H.resize(L + 1);
  c->D.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    std::string err = build_level(c->H[l], deg[l], n_e, widths, lambda, o.weight_degree, o.neumann, o.periodic);
    if (!err.empty()) { free_ctx(c); return fail(PMG_EINVAL, err); }
    if (l >= 1) build_interp(c->H[l], deg[l - 1]);
    if (o.smoother == 1) {   // every level (pmg_smooth may be called on any level)
      err = build_ec_tables(c->H[l], n_e, widths, o.neumann);
      if (!err.empty()) { free_ctx(c); return fail(PMG_EINVAL, err); }
    }
  }
  std::vector<double> diag;
  coarse_diag(c->H[0], lambda, diag);
  std::vector<double> dinv(diag.size());
  for (size_t i = 0; i < diag.size(); ++i) dinv[i] = diag[i] != 0.0 ? 1.0 / diag[i] : 0.0;

  int dev = 0;
  cudaGetDevice(&dev);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  size_t max_elem = 0, max_star = 0, max_tr = 0;
  size_t Ylen = 0, Zlen = 0;
  pmg_status s;
  c->g0g = c->H[0].g;
  const SlabPlan& sp = c->slab;
  for (int l = 0; l <= L; ++l) {
    DevLevel& D = c->D[l];
    const HostLevel& Hl = c->H[l];
    D.g = Hl.g;
    std::vector<double> et = Hl.etab, st = Hl.stab;
    if (c->tr) {
      // the rank's slab: vertex planes zb .. z1, element layers zb .. z1-1 (one ghost layer
      // below); direction-3 rows of the element / star tables sliced to match
      LevelGeom& g = D.g;
      const int k1 = g.k1, k2 = g.k2, V1 = g.V1, V2 = g.V2;
      g.k3 = sp.z1 - sp.zb;
      g.V3 = g.k3 + 1;
      g.nrec = (long long)g.V1 * g.V2 * g.V3;
      g.nskel = g.nrec * g.RS;
      g.nelem = (long long)g.k1 * g.k2 * g.k3;
      g.zoff = sp.zb;
      g.K3 = Hl.g.k3;
      g.own_lo = sp.own_lo;
      g.own_hi = sp.own_hi;
      et.assign(Hl.etab.begin(), Hl.etab.begin() + (size_t)(k1 + k2) * g.ET);
      et.insert(et.end(), Hl.etab.begin() + (size_t)(k1 + k2 + sp.zb) * g.ET, Hl.etab.begin() + (size_t)(k1 + k2 + sp.z1) * g.ET);
      st.assign(Hl.stab.begin(), Hl.stab.begin() + (size_t)(V1 + V2) * g.ST);
      st.insert(st.end(), Hl.stab.begin() + (size_t)(V1 + V2 + sp.zb) * g.ST, Hl.stab.begin() + (size_t)(V1 + V2 + sp.z1 + 1) * g.ST);
    }
    if ((s = upload(&D.etab, et)) || (s = upload(&D.stab, st))) { free_ctx(c); return s; }
    if (D.g.p >= 5 && D.g.p <= 16) {   // k_star16's padded table: NP x NP S, then Lambda (pad 1), s, w (pad 0)
      const int n = D.g.n, NP = star16_np(D.g.p), STP = NP * NP + 3 * NP;
      const size_t rows = st.size() / D.g.ST;
      std::vector<double> sp(rows * STP, 0.0);
      for (size_t q = 0; q < rows; ++q) {
        const double* src = st.data() + q * D.g.ST;
        double* dst = sp.data() + q * STP;
        for (int j = 0; j < n; ++j)
          for (int a = 0; a < n; ++a) dst[j * NP + a] = src[j * n + a];
        for (int a = 0; a < NP; ++a) {
          dst[NP * NP + a] = a < n ? src[n * n + a] : 1.0;
          dst[NP * NP + NP + a] = a < n ? src[n * n + n + a] : 0.0;
          dst[NP * NP + 2 * NP + a] = a < n ? src[n * n + 2 * n + a] : 0.0;
        }
      }
      if ((s = upload(&D.stabP, sp))) { free_ctx(c); return s; }
    }
    if (D.g.p >= 9 && D.g.p <= 16) {
      const int ETP = elem16_etp(D.g.p);   // k_elem16's padded element table
      const size_t erows = et.size() / D.g.ET;
      std::vector<double> ep(erows * ETP, 0.0);
      for (size_t q = 0; q < erows; ++q) elem16_table_row(D.g.p, et.data() + q * D.g.ET, ep.data() + q * ETP);
      if ((s = upload(&D.etabP, ep))) { free_ctx(c); return s; }
    }
    max_elem = std::max(max_elem, hot_smem(D.g.p, 0));
    max_star = std::max(max_star, hot_smem(D.g.p, 1));
    if (l >= 1 && (s = upload(&D.Jint, c->H[l].Jint))) { free_ctx(c); return s; }
    if (o.smoother == 1 && (s = upload(&D.ectab, c->H[l].ectab))) { free_ctx(c); return s; }
    if (dalloc(&D.u, D.g.nskel) || dalloc(&D.f, D.g.nskel) || dalloc(&D.r, D.g.nskel)) { free_ctx(c); return fail(PMG_ENOMEM, "cudaMalloc failed (level vectors)"); }
    cudaMemset(D.u, 0, D.g.nskel * sizeof(double));
    cudaMemset(D.f, 0, D.g.nskel * sizeof(double));
    cudaMemset(D.r, 0, D.g.nskel * sizeof(double));
    Ylen = std::max<size_t>(Ylen, (size_t)D.g.nelem * D.g.YS);
    if (l >= 1) {
      Zlen = std::max<size_t>(Zlen, (size_t)D.g.nrec * zs_of(deg[l - 1]));
      max_tr = std::max(max_tr, transfer_smem(D.g.p, deg[l - 1]));
    }
  }
  const LevelGeom& gt = c->D[L].g;
  c->cube_in_smem = std::max(condense_smem(p, gt.ET, true), recover_smem(p, gt.ET, true)) <= (size_t)smem_optin;
  size_t max_cond = condense_smem(p, gt.ET, c->cube_in_smem), max_rec = recover_smem(p, gt.ET, c->cube_in_smem);
  Ylen = std::max<size_t>(Ylen, (size_t)gt.nelem * 6 * gt.m * gt.m);
  if (max_elem > (size_t)smem_optin || max_star > (size_t)smem_optin || max_tr > (size_t)smem_optin ||
      max_cond > (size_t)smem_optin || max_rec > (size_t)smem_optin) {
    free_ctx(c);
    return fail(PMG_EINVAL, "shared-memory plan exceeds the device limit for this p");
  }
  if (cudaMalloc(reinterpret_cast<void**>(&c->ticket), sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(c->ticket, 0, sizeof(unsigned)) != cudaSuccess) {
    free_ctx(c);
    return fail(PMG_ENOMEM, "cudaMalloc failed (ticket)");
  }
  if (dalloc(&c->Y, Ylen) || dalloc(&c->Z, Zlen) || dalloc(&c->part, 16384) || dalloc(&c->dres, 8) ||
      dalloc(&c->pcg, 1)) {
    free_ctx(c);
    return fail(PMG_ENOMEM, "cudaMalloc failed (workspaces)");
  }
  if (o.solver == 1) {
    const long long nt = c->D[L].g.nskel;
    if (dalloc(&c->kz, nt) || dalloc(&c->ks_, nt) || dalloc(&c->kp, nt) || dalloc(&c->kq, nt) || dalloc(&c->kr, nt) ||
        dalloc(&c->kscal, 8)) {
      free_ctx(c);
      return fail(PMG_ENOMEM, "cudaMalloc failed (ipCG vectors)");
    }
  }
  if (!c->cube_in_smem) {
    c->cube_blocks = 296;
    if (dalloc(&c->cube, (size_t)c->cube_blocks * gt.m * gt.m * gt.m)) { free_ctx(c); return fail(PMG_ENOMEM, "cudaMalloc failed (cube)"); }
  }
  long long n0 = c->g0g.nskel;
  if (c->tr) {
    const long long pl = plane_len(c->D[0].g);
    int maxown = 0;
    for (const SlabPlan& P : c->plans) maxown = std::max(maxown, P.own_hi - P.own_lo);
    c->ag_chunk = (long long)maxown * pl;
    const LevelGeom& gt_ = c->D[L].g;
    c->n_grid_loc = (long long)(gt_.k1 * p + 1) * (gt_.k2 * p + 1) * (gt_.k3 * p + 1);
    if (dalloc(&c->f0g, n0) || dalloc(&c->u0g, n0) || dalloc(&c->agsend, c->ag_chunk) ||
        dalloc(&c->agrecv, c->ag_chunk * o.nranks) || dalloc(&c->cxl, c->D[0].g.nskel) ||
        dalloc(&c->Floc, c->n_grid_loc) || dalloc(&c->Uloc, c->n_grid_loc)) {
      free_ctx(c);
      return fail(PMG_ENOMEM, "cudaMalloc failed (z-slab buffers)");
    }
    cudaMemset(c->f0g, 0, n0 * sizeof(double));
    cudaMemset(c->Floc, 0, c->n_grid_loc * sizeof(double));
  }
  if (dalloc(&c->cx, n0) || dalloc(&c->cr, n0) || dalloc(&c->cz, n0) || dalloc(&c->cp, n0) || dalloc(&c->cq, n0)) {
    free_ctx(c);
    return fail(PMG_ENOMEM, "cudaMalloc failed (coarse CG vectors)");
  }
  if ((s = upload(&c->dinv, dinv))) { free_ctx(c); return s; }
  for (int d = 0; d < 3; ++d) {
    std::vector<double> xw, ww;
    gll(p, xw, ww);
    int kd = n_e[d];
    std::vector<double> b(kd * p + 1, 0.0);
    for (int e = 0; e < kd; ++e)
      for (int t = 0; t <= p; ++t) b[e * p + t] += 0.5 * widths[d][e] * ww[t];
    if ((o.periodic >> d) & 1) {   // node k_d p is node 0
      b[0] += b[kd * p];
      b[kd * p] = b[0];
    }
    if ((s = upload(&c->bm[d], b))) { free_ctx(c); return s; }
  }
  c->n_grid = (long long)(n_e[0] * p + 1) * (n_e[1] * p + 1) * ((sp.z1 - sp.z0) * p + 1);
  if (dalloc(&c->Fdev, c->n_grid) || dalloc(&c->Udev, c->n_grid)) { free_ctx(c); return fail(PMG_ENOMEM, "cudaMalloc failed (grid buffers)"); }
  // the attribute is per function, not per context: always allow the device maximum so that
  // several contexts with different degrees can coexist
  cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
  cudaError_t e3 = transfer_set_smem_attr(smem_optin);
  cudaError_t e4 = cudaSuccess;
  if (o.smoother == 1) {
    if (ec_smem(p) > (size_t)smem_optin) { free_ctx(c); return fail(PMG_EINVAL, "element-centred smoother: shared memory exceeds the device limit"); }
    e4 = ec_set_smem_attr(smem_optin);
  }
  cudaError_t e5 = condense_recover_set_smem_attr(smem_optin);
  cudaError_t e6 = cudaSuccess;
  if (e6 == cudaSuccess) e6 = hot_set_smem_attr(smem_optin);
  if (e6 == cudaSuccess) e6 = star16_set_smem_attr();
  if (e6 == cudaSuccess) e6 = elem16_set_smem_attr();
  if (e6 == cudaSuccess) e6 = cr16_set_smem_attr();
  if (e1 || e2 || e3 || e4 || e5 || e6) { free_ctx(c); return fail(PMG_ECUDA, "cudaFuncSetAttribute failed"); }
  // the h-multigrid coarse solver (below) is chosen from the mesh alone: when it will run, the
  // ELL rows of the Jacobi-PCG (and their L2 set-aside, which slows every other streaming kernel)
  // are not built
  auto hmg_choice = [&](bool& want, bool& coarsenable0) {
    const LevelGeom& g0 = c->g0g;
    const int k0[3] = {g0.k1, g0.k2, g0.k3};
    auto halvable = [](int kd) { return kd % 2 == 0 && kd / 2 >= 2; };
    coarsenable0 = halvable(k0[0]) || halvable(k0[1]) || halvable(k0[2]);
    const long long ne0 = (long long)k0[0] * k0[1] * k0[2];
    // automatic choice: a large coarse system whose Jacobi-PCG iteration count grows with the mesh,
    // i.e. not mass dominated: lambda L_min^2 < 100 (L_min the shortest box edge; config 4's
    // lambda = 100 on (0, 2 pi) converges in ~45 Jacobi-PCG iterations and stays on Jacobi)
    double Lmin = 1e300;
    for (int d = 0; d < 3; ++d) {
      double Ld = 0.0;
      for (int e = 0; e < n_e[d]; ++e) Ld += widths[d][e];
      Lmin = std::min(Lmin, Ld);
    }
    const bool grid_fits = (long long)(2 * k0[0] + 1) * (2 * k0[1] + 1) * (2 * k0[2] + 1) < (1LL << 31);   // int grid indices
    want = c->D[0].g.p == 2 && !o.periodic && grid_fits &&
           (o.coarse_solver == 2 ||
            (o.coarse_solver == 0 && ne0 > 12288 && coarsenable0 && lambda * Lmin * Lmin < 100.0));
  };
  bool hmg_want = false, hmg_coarsenable = false;
  hmg_choice(hmg_want, hmg_coarsenable);
  // persistent cooperative coarse CG when the coarse degree is 2 and the device supports it
  {
    int coop = 0, nsm = 0, per_sm = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_coop_p2, kThreads, 0);
    const char* env = std::getenv("PMG_COARSE_MULTIKERNEL");
    // periodic meshes take the multi-kernel Jacobi-PCG (its operator is the wrapped element operator)
    if (coop && per_sm > 0 && c->D[0].g.p == 2 && !(env && env[0] == '1') && !o.periodic) {
      long long want = (c->g0g.nskel + kThreads - 1) / kThreads;
      long long cap = std::min<long long>((long long)per_sm * nsm, 1344);
      c->coop_nb = (int)std::max<long long>(1, std::min(want, cap));
      c->use_coop = true;
      std::vector<double> tabs[7];
      coarse_tables(c->H[0], lambda, tabs);
      for (int i = 0; i < 7; ++i)
        if ((s = upload(&c->ctab[i], tabs[i]))) { free_ctx(c); return s; }
      const char* ng = std::getenv("PMG_NO_GRAPH");
      c->no_graph = ng && ng[0] == '1';
      if (cudaMallocHost(reinterpret_cast<void**>(&c->hres), sizeof(double)) != cudaSuccess) {
        free_ctx(c);
        return fail(PMG_ENOMEM, "cudaMallocHost failed");
      }
      {
        int per_sm_reg = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_reg, k_pcg_coop_reg_p2, kThreads, 0);
        const long long need = (c->g0g.nskel + kThreads - 1) / kThreads;
        const char* re = std::getenv("PMG_COARSE_REG");
        if (!(re && re[0] == '0') && per_sm_reg > 0 && need <= std::min<long long>((long long)per_sm_reg * nsm, 1344)) {
          c->coop_reg = true;
          c->coop_nb = (int)need;
          int per_sm_gv = 0;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_gv, k_pcg_gv_p2, kThreads, 0);
          const char* ge = std::getenv("PMG_COARSE_GV");
          if (!(ge && ge[0] == '0') && per_sm_gv > 0 && need <= (long long)per_sm_gv * nsm &&
              dalloc(&c->cgm, 2 * c->g0g.nskel) == cudaSuccess)
            c->coop_gv = true;
        }
        // more coarse unknowns than the register-resident kernels can hold: ELL rows + grid-stride
        int per_sm_ell = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_ell, k_pcg_gv_ell_p2, kThreads, 0);
        const char* le = std::getenv("PMG_COARSE_ELL");
        if (!c->coop_gv && !hmg_want && !(le && le[0] == '0') && per_sm_ell > 0) {
          const long long n0e = c->g0g.nskel;
          if (dalloc(&c->ella, 25 * n0e + (25 * n0e + 1) / 2) == cudaSuccess &&
              dalloc(&c->ellv, 8 * n0e) == cudaSuccess && (c->cgm || dalloc(&c->cgm, 2 * n0e) == cudaSuccess)) {
            c->ellc = reinterpret_cast<int*>(c->ella + 25 * n0e);
            // the rows are re-read every iteration: ask L2 to keep them (set-aside persisting lines)
            int maxp = 0, maxwin = 0;
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
            cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
            // opt-in (PMG_L2PERSIST=1): the set-aside speeds the coarse CG up but slows every other
            // streaming kernel of the solve more (config 4: 61.8 vs 60.4 ms per solve)
            const char* np_ = std::getenv("PMG_L2PERSIST");
            const size_t rows = sizeof(double) * (size_t)(25 * n0e + (25 * n0e + 1) / 2);
            if (maxp > 0 && maxwin > 0 && np_ && np_[0] == '1') {
              size_t cur = 0;
              cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
              const size_t want = std::min<size_t>((size_t)maxp, rows);
              c->l2_limit_prev = cur;   // restored by pmg_destroy
              c->l2_limit_set = true;
              if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
              cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
              c->ell_win.base_ptr = c->ella;
              c->ell_win.num_bytes = std::min<size_t>(rows, (size_t)maxwin);
              c->ell_win.hitRatio = (float)std::min(1.0, (double)cur / (double)c->ell_win.num_bytes);
              c->ell_win.hitProp = cudaAccessPropertyPersisting;
              c->ell_win.missProp = cudaAccessPropertyStreaming;
              c->ell_persist = cur > 0;
            }
            cudaGetLastError();
            CoarseTabs ct{c->ctab[0], c->ctab[1], c->ctab[2], c->ctab[3], c->ctab[4], c->ctab[5], c->ctab[6]};
            k_build_coarse_ell<<<grid_for(n0e), kThreads>>>(c->g0g, ct, lambda, c->ellc, c->ella);
            if (cudaGetLastError() == cudaSuccess) {
              c->coop_ell = true;
              c->ell_nb = (int)std::min<long long>((long long)per_sm_ell * nsm, std::max<long long>(1, (n0e + kThreads - 1) / kThreads));
              c->ell_nb = std::min(c->ell_nb, 2048);
            }
          } else {
            cudaGetLastError();
          }
        }
      }
      const char* nbenv = std::getenv("PMG_COOP_BLOCKS");   // tuning experiments only
      if (nbenv && std::atoi(nbenv) > 0) c->coop_nb = (int)std::min<long long>(std::atoi(nbenv), cap);
    }
  }
  // h-multigrid coarse preconditioner (reading R16): element-merged p0 = 2 levels
  {
    const LevelGeom& g0 = c->g0g;
    const int k0[3] = {g0.k1, g0.k2, g0.k3};
    auto halvable = [](int kd) { return kd % 2 == 0 && kd / 2 >= 2; };
    auto coarsenable = [&](const int* k) { return halvable(k[0]) || halvable(k[1]) || halvable(k[2]); };
    const bool want = c->use_coop && hmg_want;
    if (o.coarse_solver == 2 && !(c->use_coop && hmg_coarsenable)) {
      free_ctx(c);
      return fail(PMG_EINVAL, "coarse_solver = 2 needs p0 = 2 and some k_d even with k_d / 2 >= 2");
    }
    if (want) {
      // widths of every h-level (pairwise sums), host tables, ELL rows, 1/diag, transfers
      std::vector<std::vector<double>> wl[3];
      for (int d = 0; d < 3; ++d) wl[d].push_back(std::vector<double>(widths[d], widths[d] + n_e[d]));
      int kl[3] = {k0[0], k0[1], k0[2]};
      std::vector<const HostLevel*> hl{&c->H[0]};
      c->hhost.reserve(kMaxHLevels);
      // coarsen until a level has at most 1500 free unknowns (the dense coarsest solve; as the oracle)
      auto nfree_p2 = [&](const int* k) {
        long long f = 1;
        for (int d = 0; d < 3; ++d) {
          const bool lo = (o.neumann >> (2 * d)) & 1, hi_ = (o.neumann >> (2 * d + 1)) & 1;
          f *= (long long)(2 * k[d] + 1) - (lo ? 0 : 1) - (hi_ ? 0 : 1);
        }
        return f - (long long)k[0] * k[1] * k[2];   // free grid points minus element centres
      };
      while (coarsenable(kl) && nfree_p2(kl) > 1500 && (int)hl.size() < kMaxHLevels) {
        int kn[3];
        const double* wp[3];
        for (int d = 0; d < 3; ++d) {   // semi-coarsening: only halvable directions merge
          const bool hv = halvable(kl[d]);
          kn[d] = hv ? kl[d] / 2 : kl[d];
          std::vector<double> w2(kn[d]);
          for (int e = 0; e < kn[d]; ++e) w2[e] = hv ? wl[d].back()[2 * e] + wl[d].back()[2 * e + 1] : wl[d].back()[e];
          wl[d].push_back(w2);
        }
        for (int d = 0; d < 3; ++d) wp[d] = wl[d].back().data();
        c->hhost.emplace_back();
        std::string err = build_level(c->hhost.back(), 2, kn, wp, lambda, o.weight_degree, o.neumann);
        if (!err.empty()) { free_ctx(c); return fail(PMG_EINVAL, "h-level: " + err); }
        hl.push_back(&c->hhost.back());
        for (int d = 0; d < 3; ++d) kl[d] = kn[d];
      }
      HmgGridDev& h = c->hmg;
      h.nlev = (int)hl.size();
      h.g0 = c->g0g;
      bool ok = true;
      auto dal = [&](double** ptr, size_t cnt) {
        if (!ok || dalloc(ptr, cnt) != cudaSuccess) { ok = false; return; }
        c->hmg_allocs.push_back(*ptr);
        cudaMemset(*ptr, 0, cnt * sizeof(double));
      };
      auto up_d = [&](const std::vector<double>& v) -> const double* {
        double* p_ = nullptr;
        dal(&p_, std::max<size_t>(1, v.size()));
        if (ok) cudaMemcpy(p_, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice);
        return p_;
      };
      auto up_i = [&](const std::vector<int>& v) -> const int* {
        double* p_ = nullptr;
        dal(&p_, std::max<size_t>(1, (v.size() + 1) / 2));
        if (ok) cudaMemcpy(p_, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice);
        return reinterpret_cast<const int*>(p_);
      };
      // p = 2 record entry -> (g1, g2, g3) (parities of the record offset, as decode2 on the device)
      auto rec_point = [](const LevelGeom& g, long long idx, int* G) {
        const long long rec = idx / 7;
        const int o = (int)(idx - rec * 7);
        const long long r2 = rec / g.V1;
        G[0] = 2 * (int)(rec - r2 * g.V1) + ((0x0E >> o) & 1);
        G[1] = 2 * (int)(r2 % g.V2) + ((0x15 >> o) & 1);
        G[2] = 2 * (int)(r2 / g.V2) + ((0x23 >> o) & 1);
      };
      for (int l = 0; l < h.nlev && ok; ++l) {
        const HostLevel& HL = *hl[l];
        const LevelGeom& g = HL.g;
        HGridLev& L = h.L[l];
        L.k1 = g.k1; L.k2 = g.k2; L.k3 = g.k3;
        L.N1 = 2 * g.k1 + 1; L.N2 = 2 * g.k2 + 1; L.N3 = 2 * g.k3 + 1;
        L.neu = o.neumann;
        L.n = (long long)L.N1 * L.N2 * L.N3;
        std::vector<double> tabs[7], E[3];
        coarse_tables(HL, lambda, tabs);
        hgrid_elem_rows(HL, E);
        for (int d = 0; d < 3; ++d) {
          L.b[d] = up_d(tabs[d]);
          L.K[d] = up_d(tabs[3 + d]);
          L.E[d] = up_d(E[d]);
        }
        // 1 / diag(H_hat) from the record-layout diagonal, scattered to the grid
        std::vector<double> dg, di((size_t)L.n, 0.0);
        coarse_diag(HL, lambda, dg);
        for (long long i = 0; i < g.nskel; ++i) {
          if (dg[i] == 0.0) continue;
          int G[3];
          rec_point(g, i, G);
          if (G[0] < L.N1 && G[1] < L.N2 && G[2] < L.N3) di[G[0] + L.N1 * ((long long)G[1] + (long long)L.N2 * G[2])] = 1.0 / dg[i];
        }
        L.dinv = up_d(di);
        dal(&L.x, L.n);
        dal(&L.f, L.n);
        dal(&L.r, L.n);
        if (l + 1 < h.nlev) {
          const LevelGeom& gc = hl[l + 1]->g;
          const int kf[3] = {g.k1, g.k2, g.k3}, kc[3] = {gc.k1, gc.k2, gc.k3};
          for (int d = 0; d < 3; ++d) {
            std::vector<int> pe, r0, rn;
            std::vector<double> pw, rw;
            std::string err = build_h_transfer_1d(kf[d], wl[d][l].data(), kc[d], wl[d][l + 1].data(), pe, pw, r0, rn, rw);
            if (!err.empty()) { free_ctx(c); return fail(PMG_EINVAL, err); }
            L.pe[d] = up_i(pe); L.pw[d] = up_d(pw);
            L.r0[d] = up_i(r0); L.rn[d] = up_i(rn); L.rw[d] = up_d(rw);
          }
          dal(&L.t1, (size_t)(2 * gc.k1 + 1) * L.N2 * L.N3);
          dal(&L.t2, (size_t)(2 * gc.k1 + 1) * (2 * gc.k2 + 1) * L.N3);
        }
      }
      if (ok) {
        const long long n0h = h.L[0].n;
        if (dalloc(&c->hpv, n0h) != cudaSuccess || dalloc(&c->hq, n0h) != cudaSuccess ||
            dalloc(&c->hX, n0h) != cudaSuccess)
          ok = false;
      }
      // coarsest level: dense inverse over its free unknowns (<= 1500, as the oracle), assembled
      // from its ELL rows (built on the device in record layout); Cholesky-based inversion on the host
      h.ncf = 0;
      if (ok) {
        const int Lc = h.nlev - 1;
        const HostLevel& HL = *hl[Lc];
        const long long n = HL.g.nskel;
        std::vector<double> tabs[7];
        coarse_tables(HL, lambda, tabs);
        double* ctd[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        double *val_d = nullptr, *col_d = nullptr;
        for (int i = 0; i < 7; ++i) ctd[i] = const_cast<double*>(up_d(tabs[i]));
        dal(&val_d, 25 * n);
        dal(&col_d, (25 * n + 1) / 2);
        std::vector<double> val(25 * n), dg;
        std::vector<int> col(25 * n);
        if (ok) {
          CoarseTabs ct{ctd[0], ctd[1], ctd[2], ctd[3], ctd[4], ctd[5], ctd[6]};
          k_build_coarse_ell<<<grid_for(n), kThreads>>>(HL.g, ct, lambda, reinterpret_cast<int*>(col_d), val_d);
          cudaDeviceSynchronize();
          cudaMemcpy(val.data(), val_d, val.size() * sizeof(double), cudaMemcpyDeviceToHost);
          cudaMemcpy(col.data(), col_d, col.size() * sizeof(int), cudaMemcpyDeviceToHost);
        }
        coarse_diag(HL, lambda, dg);
        std::vector<int> fidx, pos(n, -1);
        for (long long i = 0; i < n; ++i) if (dg[i] != 0.0) { pos[i] = (int)fidx.size(); fidx.push_back((int)i); }
        const int nf = (int)fidx.size();
        if (ok && nf > 0 && nf <= 1500) {
          std::vector<double> A((size_t)nf * nf, 0.0);
          for (int a = 0; a < nf; ++a)
            for (int kx = 0; kx < 25; ++kx) {
              const long long e = (long long)kx * n + fidx[a];
              if (val[e] != 0.0 && pos[col[e]] >= 0) A[(size_t)a * nf + pos[col[e]]] += val[e];
            }
          // Cholesky A = L L^T, then A^-1 column by column
          bool spd = true;
          for (int j = 0; j < nf && spd; ++j) {
            double d = A[(size_t)j * nf + j];
            for (int k = 0; k < j; ++k) d -= A[(size_t)j * nf + k] * A[(size_t)j * nf + k];
            if (!(d > 0.0)) { spd = false; break; }
            d = std::sqrt(d);
            A[(size_t)j * nf + j] = d;
            for (int i = j + 1; i < nf; ++i) {
              double v = A[(size_t)i * nf + j];
              for (int k = 0; k < j; ++k) v -= A[(size_t)i * nf + k] * A[(size_t)j * nf + k];
              A[(size_t)i * nf + j] = v / d;
            }
          }
          if (spd) {
            std::vector<double> inv((size_t)nf * nf), y(nf);
            for (int cidx_ = 0; cidx_ < nf; ++cidx_) {
              for (int i = 0; i < nf; ++i) {             // L y = e_c
                double v = (i == cidx_) ? 1.0 : 0.0;
                for (int k = 0; k < i; ++k) v -= A[(size_t)i * nf + k] * y[k];
                y[i] = v / A[(size_t)i * nf + i];
              }
              for (int i = nf - 1; i >= 0; --i) {        // L^T x = y
                double v = y[i];
                for (int k = i + 1; k < nf; ++k) v -= A[(size_t)k * nf + i] * y[k];
                y[i] = v / A[(size_t)i * nf + i];
              }
              for (int i = 0; i < nf; ++i) inv[(size_t)i * nf + cidx_] = y[i];
            }
            // record indices -> grid indices of the coarsest level
            const HGridLev& LC = h.L[Lc];
            std::vector<int> gidx(nf);
            for (int a = 0; a < nf; ++a) {
              int G[3];
              rec_point(HL.g, fidx[a], G);
              gidx[a] = (int)(G[0] + LC.N1 * ((long long)G[1] + (long long)LC.N2 * G[2]));
            }
            h.cinv = up_d(inv);
            h.cidx = up_i(gidx);
            if (ok) h.ncf = nf;
          }
        }
      }
      int per_sm_h = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_h, k_pcg_hmg_p2, kThreads, 0);
      if (!ok || per_sm_h <= 0 || cudaGetLastError() != cudaSuccess) {
        free_ctx(c);
        return fail(PMG_ENOMEM, "h-multigrid coarse solver: allocation / setup failed");
      }
      c->hmg_nb = (int)std::min<long long>((long long)per_sm_h * nsm_dev(dev),
                                           std::max<long long>(1, (h.L[0].n + kThreads - 1) / kThreads));
      c->hmg_nb = std::min(c->hmg_nb, 2048);
      c->use_hmg = true;
    }
  }
  if (c->tr && !c->use_coop) {
    free_ctx(c);
    return fail(PMG_EINVAL, "z-slabs need the cooperative coarse CG (p0 = 2, cooperative launch support)");
  }
  for (auto& e : c->ev_ph)
    if (cudaEventCreate(&e) != cudaSuccess) { free_ctx(c); return fail(PMG_ECUDA, "setup: cudaEventCreate"); }
  for (auto& e : c->ev_cg)
    if (cudaEventCreate(&e) != cudaSuccess) { free_ctx(c); return fail(PMG_ECUDA, "setup: cudaEventCreate"); }
  cudaError_t es = cudaDeviceSynchronize();
  if (es != cudaSuccess) { free_ctx(c); return fail(PMG_ECUDA, std::string("setup: ") + cudaGetErrorString(es)); }
  *out = c;
  return PMG_OK;
}

pmg_status pmg_destroy(pmg_ctx* c) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  cudaStreamSynchronize(c->st);
  if (c->l2_limit_set) {   // release the set-aside persisting L2 lines of the coarse ELL rows
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c->l2_limit_prev);
    cudaGetLastError();
  }
  free_ctx(c);
  return PMG_OK;
}

int pmg_num_levels(const pmg_ctx* c) { return c ? c->L + 1 : -1; }

pmg_status pmg_level_info(const pmg_ctx* c, int level, int* degree, long long* n_skel, long long* n_grid) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  const LevelGeom& g = c->D[level].g;
  if (degree) *degree = g.p;
  if (n_skel) *n_skel = g.nskel;   // local (ghost planes included) on z-slabs
  if (n_grid) *n_grid = (long long)(g.k1 * g.p + 1) * (g.k2 * g.p + 1) * ((c->slab.z1 - c->slab.z0) * g.p + 1);
  return PMG_OK;
}

pmg_status pmg_grid_coords(const pmg_ctx* c, int level, int d, double* coords_host) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (d < 0 || d > 2 || !coords_host) return fail(PMG_EINVAL, "bad direction or NULL output");
  const auto& x = c->H[level].coords[d];
  if (d == 2) {   // the rank's slab: nodes z0 p .. z1 p (the whole line on one GPU)
    const int p = c->H[level].p;
    std::memcpy(coords_host, x.data() + (size_t)c->slab.z0 * p, (size_t)((c->slab.z1 - c->slab.z0) * p + 1) * sizeof(double));
  } else {
    std::memcpy(coords_host, x.data(), x.size() * sizeof(double));
  }
  return PMG_OK;
}

pmg_status pmg_residual(pmg_ctx* c, int level, const double* u_hat, const double* f_hat, double* r_hat) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (!u_hat || !r_hat) return fail(PMG_EINVAL, "NULL vector");
  if (u_hat == r_hat) return fail(PMG_EINVAL, "u_hat and r_hat must not alias");
  return residual_x(c, level, const_cast<double*>(u_hat), f_hat, r_hat);   // z-slabs: ghosts refreshed
}

pmg_status pmg_smooth(pmg_ctx* c, int level, const double* r_hat, double* u_hat) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (!u_hat || !r_hat) return fail(PMG_EINVAL, "NULL vector");
  if (u_hat == r_hat) return fail(PMG_EINVAL, "u_hat and r_hat must not alias");
  if ((s = exchange(c, level, const_cast<double*>(r_hat)))) return s;
  if ((s = smooth_dev(c, level, r_hat, u_hat))) return s;
  return exchange(c, level, u_hat);
}

pmg_status pmg_restrict(pmg_ctx* c, int level, const double* r_fine, double* f_coarse) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (level < 1) return fail(PMG_EINVAL, "restrict needs a fine level >= 1");
  if (!r_fine || !f_coarse) return fail(PMG_EINVAL, "NULL vector");
  if ((s = exchange(c, level, const_cast<double*>(r_fine)))) return s;
  if ((s = restrict_dev(c, level, r_fine, f_coarse))) return s;
  return exchange(c, level - 1, f_coarse);
}

pmg_status pmg_prolong(pmg_ctx* c, int level, const double* u_coarse, double* u_fine) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (level < 1) return fail(PMG_EINVAL, "prolong needs a fine level >= 1");
  if (!u_coarse || !u_fine) return fail(PMG_EINVAL, "NULL vector");
  if ((s = exchange(c, level - 1, const_cast<double*>(u_coarse)))) return s;
  if ((s = prolong_dev(c, level, u_coarse, u_fine))) return s;
  return exchange(c, level, u_fine);
}

pmg_status pmg_vcycle(pmg_ctx* c, double* u_hat, const double* f_hat) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (!u_hat || !f_hat) return fail(PMG_EINVAL, "NULL vector");
  pmg_status s;
  if ((s = exchange(c, c->L, const_cast<double*>(f_hat)))) return s;
  if ((s = vcycle_dev(c, u_hat, f_hat, false))) return s;
  return exchange(c, c->L, u_hat);
}

pmg_status pmg_condense(pmg_ctx* c, const double* F_full, double* f_hat) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (c->tr) return fail(PMG_EINVAL, "pmg_condense: one GPU only (pmg_solve condenses on z-slabs)");
  if (!F_full || !f_hat) return fail(PMG_EINVAL, "NULL vector");
  return condense_dev(c, F_full, f_hat);
}

pmg_status pmg_recover(pmg_ctx* c, const double* u_hat, const double* F_full, double* u_full) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (c->tr) return fail(PMG_EINVAL, "pmg_recover: one GPU only (pmg_solve recovers on z-slabs)");
  if (!u_hat || !F_full || !u_full) return fail(PMG_EINVAL, "NULL vector");
  return recover_dev(c, u_hat, F_full, u_full);
}

pmg_status pmg_solve(pmg_ctx* c, const double* F_full, double* u_full, double rtol, int max_cycles, pmg_report* rep) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (!F_full || !u_full) return fail(PMG_EINVAL, "NULL vector");
  if (!(rtol > 0.0) || max_cycles < 0) return fail(PMG_EINVAL, "rtol > 0 and max_cycles >= 0 required");
  return solve_dev(c, F_full, u_full, rtol, max_cycles, rep);
}

pmg_status pmg_solve_host(pmg_ctx* c, const double* F_host, double* u_host, double rtol, int max_cycles, pmg_report* rep) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (!F_host || !u_host) return fail(PMG_EINVAL, "NULL vector");
  CUDA_CHECK(cudaMemcpyAsync(c->Fdev, F_host, c->n_grid * sizeof(double), cudaMemcpyHostToDevice, c->st));
  pmg_status s = pmg_solve(c, c->Fdev, c->Udev, rtol, max_cycles, rep);
  if (s != PMG_OK && s != PMG_ENOCONV) return s;
  CUDA_CHECK(cudaMemcpyAsync(u_host, c->Udev, c->n_grid * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CUDA_CHECK(cudaStreamSynchronize(c->st));
  return s;
}

pmg_status pmg_weak_rhs(pmg_ctx* c, const double* f_nodal, double* F_full) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (!f_nodal || !F_full) return fail(PMG_EINVAL, "NULL vector");
  LevelGeom g = c->D[c->L].g;   // the caller's slab: element layers z0 .. z1-1
  g.k3 = c->slab.z1 - c->slab.z0;
  g.zoff = c->slab.z0;
  k_weak_rhs<<<grid_for(c->n_grid), kThreads, 0, c->st>>>(g, c->bm[0], c->bm[1], c->bm[2], f_nodal, F_full);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status pmg_skel_from_grid(pmg_ctx* c, int level, const double* grid, double* skel) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (!grid || !skel) return fail(PMG_EINVAL, "NULL vector");
  if (c->tr) return fail(PMG_EINVAL, "layout converters: one GPU only");
  k_skel_from_grid<<<grid_for(c->D[level].g.nskel), kThreads, 0, c->st>>>(c->D[level].g, grid, skel);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status pmg_skel_to_grid(pmg_ctx* c, int level, const double* skel, double* grid) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (!grid || !skel) return fail(PMG_EINVAL, "NULL vector");
  if (c->tr) return fail(PMG_EINVAL, "layout converters: one GPU only");
  const LevelGeom& g = c->D[level].g;
  long long ng = (long long)(g.k1 * g.p + 1) * (g.k2 * g.p + 1) * (g.k3 * g.p + 1);
  k_skel_to_grid<<<grid_for(ng), kThreads, 0, c->st>>>(g, skel, grid);
  LAUNCH_CHECK(c);
  return PMG_OK;
}

pmg_status pmg_norm(pmg_ctx* c, int level, const double* x_hat, double* out_host) {
  pmg_status s = check_level(c, level);
  if (s) return s;
  if (!x_hat || !out_host) return fail(PMG_EINVAL, "NULL pointer");
  return norm_host(c, level, x_hat, out_host);
}

long long pmg_launch_count(const pmg_ctx* c) { return c ? c->launches : -1; }

int pmg_slab_plan(int k3, int nranks, int rank, pmg_slab* out) {
  SlabPlan P;
  if (!out || slab_plan(k3, nranks, rank, &P) != 0) return -1;
  out->z0 = P.z0; out->z1 = P.z1; out->zb = P.zb; out->nplanes = P.nplanes;
  out->own_lo = P.own_lo; out->own_hi = P.own_hi; out->lower = P.lower; out->upper = P.upper;
  return 0;
}

pmg_status pmg_slab_info(const pmg_ctx* c, pmg_slab* out) {
  if (!c || !out) return fail(PMG_EINVAL, "NULL argument");
  const SlabPlan& P = c->slab;
  out->z0 = P.z0; out->z1 = P.z1; out->zb = P.zb; out->nplanes = P.nplanes;
  out->own_lo = P.own_lo; out->own_hi = P.own_hi; out->lower = P.lower; out->upper = P.upper;
  return PMG_OK;
}

pmg_status pmg_nccl_unique_id(void* out128) {
  if (!out128) return fail(PMG_EINVAL, "NULL output");
  std::string e = nccl_unique_id(out128);
  return e.empty() ? PMG_OK : fail(PMG_ENCCL, e);
}

void* pmg_loopback_create(int nranks) { return loopback_create(nranks); }
void pmg_loopback_destroy(void* hub) { loopback_destroy(hub); }

pmg_status pmg_timing_enable(pmg_ctx* c, int enable) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  CUDA_CHECK(cudaStreamSynchronize(c->st));
  ev_reset(c);
  c->timing = enable != 0;
  return PMG_OK;
}

pmg_status pmg_timing_read(pmg_ctx* c, int kind, double* total_ms, long long* count) {
  if (!c) return fail(PMG_EINVAL, "ctx is NULL");
  if (kind < 0 || kind > 4 || !total_ms || !count) return fail(PMG_EINVAL, "bad kind or NULL output");
  CUDA_CHECK(cudaStreamSynchronize(c->st));
  double tot = 0.0;
  long long n = 0;
  for (auto& mk : c->ev_marks) {
    if (kind == 4) {
      if (mk.base != 2) continue;
    } else {
      if (mk.base != (kind & 1)) continue;
      if (kind < 2 && !mk.top) continue;
    }
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, mk.a, mk.b));
    tot += ms;
    ++n;
  }
  *total_ms = tot;
  *count = n;
  return PMG_OK;
}

}  // extern "C"
