// Coarse-grid solver (reading R11): Jacobi-preconditioned CG on the condensed p0 = 2
// system, as ONE persistent cooperative kernel (grid-wide barriers between the phases of an
// iteration).  The coarse solve is latency bound: a multi-kernel CG spends
// ~10 launches per iteration; here the whole solve is one launch with 2 grid barriers per
// iteration.
//
// Operator: at p = 2 every element has one interior point, so the element Schur complement is
//   H_hat_e = H_BB,e - (1/D_e) c_e c_e^T,  c_e[f] = a_f P_b P_a on the 6 face centres,
// (reading R1 with m = 1) and sum_e H_BB,e is the assembled tensor-product operator
//   H = lam B3(x)B2(x)B1 + B3(x)B2(x)K1 + B3(x)K2(x)B1 + K3(x)B2(x)B1
// restricted to the skeleton with zero element interiors (B_d / K_d the assembled 1-D lumped
// mass / stiffness, 5-point along each grid line).  So q = H_hat p is a 13-point line stencil
// minus rank-one element corrections, V_e = (c_e . p_e) / D_e, evaluated on the fly.
//
// Every block reduces the per-block partial sums itself in a fixed order, so all blocks take the
// same (bitwise identical) decisions on alpha, beta and convergence without another barrier,
// and the result is deterministic.  Iteration and stopping rule as the oracle's pcg(): x = 0,
// r = b, z = D^-1 r, p = z; q = H p, alpha = r.z / p.q, x += alpha p, r -= alpha q, stop when
// ||r|| <= rtol ||b||, z = D^-1 r, beta = r.z_new / r.z, p = z + beta p.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace cg = cooperative_groups;

namespace pmg {

// sum of the block's values -> thread 0
__device__ __forceinline__ double block_reduce(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// totals of two per-block partial arrays, identical in every block: the whole block loads the
// partials (one L2 round trip: every thread at most ceil(nb / blockDim) loads), warp xor-trees, then
// the warp sums in fixed order -- the same partition and order in every block, so every block
// gets bitwise the same totals (deterministic, no extra grid barrier).  `red` holds 2 x 32 doubles.
__device__ __forceinline__ void grid_totals(const double* pa, const double* pb, int nb, double* red,
                                            double& ta, double& tb) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += __ldcg(&pa[i]);
    if (pb) b += __ldcg(&pb[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  __syncthreads();
  if (lane == 0) { red[w] = a; red[32 + w] = b; }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
  for (int i = 0; i < nw; ++i) { sa += red[i]; sb += red[32 + i]; }
  ta = sa;
  tb = sb;
}

// Skeleton-vector index of a point, or -1 outside the box (no memory access here)
// p = 2 specialisation of skel_index: shifts instead of divisions by p, 32-bit record math (the
// coarse level has < 2^31 entries).  Record offset of the point from the parities (t1,t2,t3):
// (0,1,1) f1 = 0, (1,0,1) f2 = 1, (1,1,0) f3 = 2, (1,0,0) e1 = 3, (0,1,0) e2 = 4, (0,0,1) e3 = 5,
// (0,0,0) vertex = 6, packed as nibbles of 0xF0152436 indexed by t1 + 2 t2 + 4 t3.
__device__ __forceinline__ long long sidx2(const LevelGeom& g, int g1, int g2, int g3) {
  const int key = (g1 & 1) | ((g2 & 1) << 1) | ((g3 & 1) << 2);
  const int off = (int)((0xF0152436u >> (4 * key)) & 0xFu);
  const int rec = (g1 >> 1) + g.V1 * ((g2 >> 1) + g.V2 * (g3 >> 1));
  return (long long)rec * 7 + off;
}

__device__ __forceinline__ long long sidx_or_neg(const LevelGeom& g, int g1, int g2, int g3) {
  return inside(g, g1, g2, g3) ? sidx2(g, g1, g2, g3) : -1LL;
}

// p = 2 entry decode: record = idx / 7 (constant divisor), parities from the record offset
__device__ __forceinline__ Entry decode2(const LevelGeom& g, long long idx) {
  Entry E;
  const int i = (int)idx;
  const int rec = i / 7, o = i - rec * 7;
  const int r2 = rec / g.V1;
  E.v1 = rec - r2 * g.V1;
  E.v3 = r2 / g.V2;
  E.v2 = r2 - E.v3 * g.V2;
  E.g1 = 2 * E.v1 + ((0x0E >> o) & 1);
  E.g2 = 2 * E.v2 + ((0x15 >> o) & 1);
  E.g3 = 2 * E.v3 + ((0x23 >> o) & 1);
  E.type = o;            // 0-2 faces, 3-5 edges, 6 vertex (m = 1)
  E.a = 0; E.b = 0;
  return E;
}

// Branch-free gather: all loads are issued back to back (a predicated index, then a select), so an
// entry costs one L2 round trip instead of a chain of dependent ones.  p is written inside the
// kernel -> L2 path (__ldcg).
__device__ __forceinline__ double ld_sel(const double* p, long long i) {
  const double v = __ldcg(&p[i < 0 ? 0 : i]);
  return i < 0 ? 0.0 : v;
}

// accessor of the grid kernel: global vector, L2 path
struct GlobalAcc {
  const double* p;
  __device__ __forceinline__ double operator()(long long i) const { return ld_sel(p, i); }
};

// q = H_hat p at one skeleton entry (p = 2); the element corrections V_e(p) of the (at most two)
// elements adjacent to a face centre are evaluated on the fly.  `p(i)` returns the vector at global
// skeleton index i (0 for i < 0).
template <class Acc>
__device__ __forceinline__ double apply_entry(const LevelGeom& g, const CoarseTabs& ct, const Acc& p,
                                              long long idx, double lam) {
  Entry E = decode2(g, idx);
  if (!is_free(g, E.g1, E.g2, E.g3)) return 0.0;
  const int G[3] = {E.g1, E.g2, E.g3};
  const int N[3] = {2 * g.k1, 2 * g.k2, 2 * g.k3};
  // indices: centre, then per direction the offsets -2, -1, +1, +2 along the line
  long long ix[13];
  ix[0] = idx;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
    const bool full = ((G[da] & 1) == 0) || ((G[db] & 1) == 0);   // the line lies on the skeleton
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = (j < 2) ? j - 2 : j - 1;
      const int s = G[d] + o;
      int h[3] = {G[0], G[1], G[2]};
      h[d] = s;
      const bool ok = s >= 0 && s <= N[d] && (full || (s & 1) == 0);   // element interiors are zero
      ix[1 + 4 * d + j] = ok ? sidx2(g, h[0], h[1], h[2]) : -1LL;
    }
  }
  // face centre: the two adjacent elements' face-centre indices
  long long fx[12];
  double cw[2][7];
  const bool face = E.type < 3;
  if (face) {
    const int d = E.type;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      int e[3] = {E.v1, E.v2, E.v3};
      if (side == 1) e[d] -= 1;
      const bool ein = e[d] >= 0 && e[d] < (d == 0 ? g.k1 : (d == 1 ? g.k2 : g.k3));   // Neumann face: one element
      if (!ein) e[d] = 0;
      const long long el = e[0] + (long long)g.k1 * (e[1] + (long long)g.k2 * e[2]);
#pragma unroll
      for (int i = 0; i < 7; ++i) cw[side][i] = ein ? __ldg(&ct.ce[el * 7 + i]) : 0.0;
      const int b1 = 2 * e[0], b2 = 2 * e[1], b3 = 2 * e[2];
      fx[6 * side + 0] = sidx_or_neg(g, b1, b2 + 1, b3 + 1);
      fx[6 * side + 1] = sidx_or_neg(g, b1 + 2, b2 + 1, b3 + 1);
      fx[6 * side + 2] = sidx_or_neg(g, b1 + 1, b2, b3 + 1);
      fx[6 * side + 3] = sidx_or_neg(g, b1 + 1, b2 + 2, b3 + 1);
      fx[6 * side + 4] = sidx_or_neg(g, b1 + 1, b2 + 1, b3);
      fx[6 * side + 5] = sidx_or_neg(g, b1 + 1, b2 + 1, b3 + 2);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 12; ++i) fx[i] = -1;
  }
  double v[13], fv[12];
#pragma unroll
  for (int i = 0; i < 13; ++i) v[i] = p(ix[i]);
#pragma unroll
  for (int i = 0; i < 12; ++i) fv[i] = p(fx[i]);
  const double* B[3] = {ct.b1, ct.b2, ct.b3};
  const double* K[3] = {ct.K1, ct.K2, ct.K3};
  double q = lam * __ldg(&B[0][G[0]]) * __ldg(&B[1][G[1]]) * __ldg(&B[2][G[2]]) * v[0];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
    const double* Kr = K[d] + (size_t)G[d] * 5;
    double acc = __ldg(&Kr[2]) * v[0];
    acc = fma(__ldg(&Kr[0]), v[1 + 4 * d], acc);
    acc = fma(__ldg(&Kr[1]), v[2 + 4 * d], acc);
    acc = fma(__ldg(&Kr[3]), v[3 + 4 * d], acc);
    acc = fma(__ldg(&Kr[4]), v[4 + 4 * d], acc);
    q = fma(__ldg(&B[da][G[da]]) * __ldg(&B[db][G[db]]), acc, q);
  }
  if (face) {
    const int d = E.type;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 6; ++i) s = fma(cw[side][i], fv[6 * side + i], s);
      // c_e[2d + side] without a runtime array index (keeps cw in registers)
      const double cd = (d == 0) ? cw[side][side] : ((d == 1) ? cw[side][2 + side] : cw[side][4 + side]);
      q = fma(-cd, s * cw[side][6], q);
    }
  }
  return q;
}

// Read-only accessor for the standalone residual (the vector is not written in the kernel: L1 path)
struct RoAcc {
  const double* p;
  __device__ __forceinline__ double operator()(long long i) const {
    const double v = __ldg(&p[i < 0 ? 0 : i]);
    return i < 0 ? 0.0 : v;
  }
};

// Condensed residual at p = 2 (one GPU, not periodic): r = f - H_hat u (f = NULL: H_hat u) on free entries, 0 elsewhere,
// one thread per skeleton entry with the line stencil + element corrections above (no element
// workspace; the p = 2 element kernel ran 27 points per CTA).
__global__ void __launch_bounds__(256) k_resid_p2(LevelGeom g, CoarseTabs ct, const double* __restrict__ u,
                                                 const double* __restrict__ f, double* __restrict__ r, double lam) {
  const long long n = g.nskel;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Entry E = decode2(g, i);
    if (!is_free(g, E.g1, E.g2, E.g3)) { r[i] = 0.0; continue; }
    const double hu = apply_entry(g, ct, RoAcc{u}, i, lam);
    r[i] = f ? f[i] - hu : hu;   // f = NULL: the operator application H_hat u
  }
}

// The same row of H_hat written out once: q[idx] = sum_k a[k] p[jx[k]] with the 13 line-stencil
// entries first and the 12 face-centre entries of the (up to two) adjacent elements after them.
// Unused slots point at idx itself with a zero coefficient (a harmless load).  The row never changes
// during a solve, so a thread that owns idx for the whole solve builds it once and keeps it in
// registers; each iteration is then 25 independent loads and 25 FMA.
constexpr int kRowLen = 25;

__device__ __forceinline__ void build_row(const LevelGeom& g, const CoarseTabs& ct, long long idx, double lam,
                                          int* jx, double* a) {
#pragma unroll
  for (int k = 0; k < kRowLen; ++k) { jx[k] = (int)idx; a[k] = 0.0; }
  Entry E = decode2(g, idx);
  if (!is_free(g, E.g1, E.g2, E.g3)) return;
  const int G[3] = {E.g1, E.g2, E.g3};
  const int N[3] = {2 * g.k1, 2 * g.k2, 2 * g.k3};
  const double* B[3] = {ct.b1, ct.b2, ct.b3};
  const double* K[3] = {ct.K1, ct.K2, ct.K3};
  double c0 = lam * __ldg(&B[0][G[0]]) * __ldg(&B[1][G[1]]) * __ldg(&B[2][G[2]]);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
    const bool full = ((G[da] & 1) == 0) || ((G[db] & 1) == 0);
    const double w = __ldg(&B[da][G[da]]) * __ldg(&B[db][G[db]]);
    const double* Kr = K[d] + (size_t)G[d] * 5;
    c0 = fma(w, __ldg(&Kr[2]), c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = (j < 2) ? j - 2 : j - 1;
      const int s = G[d] + o;
      int h[3] = {G[0], G[1], G[2]};
      h[d] = s;
      if (s >= 0 && s <= N[d] && (full || (s & 1) == 0)) {
        jx[1 + 4 * d + j] = (int)sidx2(g, h[0], h[1], h[2]);
        a[1 + 4 * d + j] = w * __ldg(&Kr[(j < 2) ? j : j + 1]);
      }
    }
  }
  a[0] = c0;
  if (E.type < 3) {
    const int d = E.type;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      int e[3] = {E.v1, E.v2, E.v3};
      if (side == 1) e[d] -= 1;
      if (e[d] < 0 || e[d] >= (d == 0 ? g.k1 : (d == 1 ? g.k2 : g.k3))) continue;   // Neumann face: one element
      const long long el = e[0] + (long long)g.k1 * (e[1] + (long long)g.k2 * e[2]);
      double cw[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) cw[i] = __ldg(&ct.ce[el * 7 + i]);
      const double cd = (d == 0) ? cw[side] : ((d == 1) ? cw[2 + side] : cw[4 + side]);
      const int b1 = 2 * e[0], b2 = 2 * e[1], b3 = 2 * e[2];
      const int fb[6][3] = {{b1, b2 + 1, b3 + 1}, {b1 + 2, b2 + 1, b3 + 1}, {b1 + 1, b2, b3 + 1},
                            {b1 + 1, b2 + 2, b3 + 1}, {b1 + 1, b2 + 1, b3}, {b1 + 1, b2 + 1, b3 + 2}};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        if (inside(g, fb[i][0], fb[i][1], fb[i][2])) {
          jx[13 + 6 * side + i] = (int)sidx2(g, fb[i][0], fb[i][1], fb[i][2]);
          a[13 + 6 * side + i] = -cd * cw[6] * cw[i];
        }
      }
    }
  }
}

// Register-resident variant: when the grid has at least one thread per coarse unknown, each thread
// keeps x, r, z, p, q, D^-1 of its entry in registers for the whole solve.  Only z is published to
// global memory (the neighbours' stencil reads it after the barrier), so an iteration costs one
// L2 round trip for the stencil and one per partial-sum exchange, plus the two grid barriers.
__global__ void __launch_bounds__(256) k_pcg_coop_reg_p2(LevelGeom g, CoarseTabs ct, const double* __restrict__ b,
                                                        double* __restrict__ xout, double* __restrict__ zpub,
                                                        const double* __restrict__ dinv, double lam,
                                                        double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[64];
  const int nb = gridDim.x;
  double* part_a = part;           // p.q
  double* part_b = part + nb;      // r.r (b.b at init)
  double* part_c = part + 2 * nb;  // r.z
  const long long n = g.nskel;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool own = i < n;
  const double bi = own ? b[i] : 0.0, di = own ? dinv[i] : 0.0;
  double x = 0.0, r = bi, z = di * bi, pv = 0.0, q = 0.0;
  int jx[kRowLen];
  double arow[kRowLen];
  build_row(g, ct, own ? i : 0, lam, jx, arow);
  if (own) zpub[i] = z;
  double s1 = block_reduce(r * z, red);
  if (threadIdx.x == 0) part_c[blockIdx.x] = s1;
  double s2 = block_reduce(bi * bi, red);
  if (threadIdx.x == 0) part_b[blockIdx.x] = s2;
  grid.sync();
  double rz, bb;
  grid_totals(part_c, part_b, nb, red, rz, bb);
  double beta = 0.0;
  int its = 0, breakdown = 0;
  bool done = (bb == 0.0);
  while (!done) {
    // p = z + beta p ; q = H_hat z + beta q ; partial p.q
    if (own) {
      pv = fma(beta, pv, z);
      double zl[kRowLen];
#pragma unroll
      for (int k = 0; k < kRowLen; ++k) zl[k] = __ldcg(&zpub[jx[k]]);
      double hz = 0.0;
#pragma unroll
      for (int k = 0; k < kRowLen; ++k) hz = fma(arow[k], zl[k], hz);
      q = fma(beta, q, hz);
    }
    const double spq = block_reduce(pv * q, red);
    if (threadIdx.x == 0) part_a[blockIdx.x] = spq;
    grid.sync();
    double pq, unused;
    grid_totals(part_a, nullptr, nb, red, pq, unused);
    if (!(pq > 0.0)) { breakdown = 1; break; }
    const double alpha = rz / pq;
    x = fma(alpha, pv, x);
    r = fma(-alpha, q, r);
    z = di * r;
    if (own) zpub[i] = z;
    const double srr = block_reduce(r * r, red);
    if (threadIdx.x == 0) part_b[blockIdx.x] = srr;
    const double srz = block_reduce(r * z, red);
    if (threadIdx.x == 0) part_c[blockIdx.x] = srz;
    grid.sync();
    double rr, rzn;
    grid_totals(part_b, part_c, nb, red, rr, rzn);
    ++its;
    if (sqrt(rr) <= rtol * sqrt(bb) || its >= maxit) break;
    beta = rzn / rz;
    rz = rzn;
  }
  if (own) xout[i] = x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its = its;
    st->its_sum += its;
    if (breakdown) st->breakdown = 1;
    st->done = 1;
    st->bb = bb;
  }
}

// ------------------------------------------------------------------------------------------
// Pipelined (single-reduction) Jacobi-PCG, Ghysels & Vanroose's recurrence: the same Krylov
// iterates as k_pcg_coop_reg_p2 in exact arithmetic (reading R11: "CG" on the coarse level,
// P:440), but every iteration needs ONE grid barrier instead of two: the dot products
// (r,u), (w,u), (r,r) of iteration i and the publication of m_i = D^-1 w_i share it, and the
// operator application n_i = H m_i runs after it, overlapping nothing but needing nothing else.
//   r0 = b, u0 = D^-1 r0, w0 = H u0;  per iteration:
//     gamma = (r,u), delta = (w,u), rho = (r,r)          [barrier]   stop if sqrt(rho) <= rtol |b|
//     m = D^-1 w (published before the barrier), n = H m
//     beta = gamma / gamma_old, alpha = gamma / (delta - beta gamma / alpha_old)   (first: 0, gamma/delta)
//     z = n + beta z, q = m + beta q, s = w + beta s, p = u + beta p
//     x += alpha p, r -= alpha s, u -= alpha q, w -= alpha z
// Stops at the first iterate with ||r|| <= rtol ||b||, as the oracle's pcg().  m is double-
// buffered (iteration parity) because neighbours may still read m_i while m_(i+1) is written;
// so are the per-block partial sums.  Used when the requested coarse tolerance is >= 1e-11 (the
// recurrence's attainable accuracy is a few orders above the standard one's); tighter requests
// (the 1e-13 parity runs) take the two-barrier kernel.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void block_reduce3(double a, double b, double c, double* red, int nb_part_slot,
                                              double* pa, double* pb, double* pc) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  __syncthreads();
  if (lane == 0) { red[w] = a; red[32 + w] = b; red[64 + w] = c; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0, sc = 0.0;
    for (int i = 0; i < nw; ++i) { sa += red[i]; sb += red[32 + i]; sc += red[64 + i]; }
    pa[nb_part_slot] = sa;
    pb[nb_part_slot] = sb;
    pc[nb_part_slot] = sc;
  }
}

__device__ __forceinline__ void grid_totals3(const double* pa, const double* pb, const double* pc, int nb, double* red,
                                             double& ta, double& tb, double& tc) {
  double a = 0.0, b = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += __ldcg(&pa[i]);
    b += __ldcg(&pb[i]);
    c += __ldcg(&pc[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  __syncthreads();
  if (lane == 0) { red[w] = a; red[32 + w] = b; red[64 + w] = c; }
  __syncthreads();
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (int i = 0; i < nw; ++i) { sa += red[i]; sb += red[32 + i]; sc += red[64 + i]; }
  ta = sa; tb = sb; tc = sc;
}

__global__ void __launch_bounds__(256) k_pcg_gv_p2(LevelGeom g, CoarseTabs ct, const double* __restrict__ b,
                                                  double* __restrict__ xout, double* __restrict__ mbuf,
                                                  const double* __restrict__ dinv, double lam,
                                                  double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  const int nb = gridDim.x;
  const long long n = g.nskel;
  double* mb[2] = {mbuf, mbuf + n};                 // m_i in mb[i & 1]; u0 is published in mb[1]
  double* pt[2][3] = {{part, part + nb, part + 2 * nb}, {part + 3 * nb, part + 4 * nb, part + 5 * nb}};
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool own = i < n;
  const double bi = own ? b[i] : 0.0, di = own ? dinv[i] : 0.0;
  int jx[kRowLen];
  double arow[kRowLen];
  build_row(g, ct, own ? i : 0, lam, jx, arow);
  auto apply = [&](const double* v) {
    double zl[kRowLen];
#pragma unroll
    for (int k = 0; k < kRowLen; ++k) zl[k] = __ldcg(&v[jx[k]]);
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < kRowLen; ++k) h = fma(arow[k], zl[k], h);
    return h;
  };
  double x = 0.0, r = bi, u = di * bi;
  if (own) mb[1][i] = u;
  grid.sync();
  double w = own ? apply(mb[1]) : 0.0;
  double m = di * w;
  if (own) mb[0][i] = m;
  block_reduce3(r * u, w * u, r * r, red, blockIdx.x, pt[0][0], pt[0][1], pt[0][2]);
  grid.sync();
  double z = 0.0, q = 0.0, s = 0.0, pv = 0.0;
  double gamma_old = 1.0, alpha_old = 1.0, bb = -1.0;
  int its = 0, breakdown = 0;
  for (int it = 0;; ++it) {
    // n_i = H m_i is issued first: its L2 loads overlap the partial-sum loads of grid_totals3
    const double nv = own ? apply(mb[it & 1]) : 0.0;
    double gamma, delta, rho;
    grid_totals3(pt[it & 1][0], pt[it & 1][1], pt[it & 1][2], nb, red, gamma, delta, rho);
    if (it == 0) bb = rho;                            // ||b||^2 (r0 = b)
    if (bb == 0.0 || sqrt(rho) <= rtol * sqrt(bb) || its >= maxit) break;
    double alpha, beta;
    if (it == 0) {
      beta = 0.0;
      alpha = gamma / delta;
      if (!(delta > 0.0)) { breakdown = 1; break; }
    } else {
      beta = gamma / gamma_old;
      const double den = delta - beta * gamma / alpha_old;
      if (!(den > 0.0)) { breakdown = 1; break; }
      alpha = gamma / den;
    }
    z = fma(beta, z, nv);
    q = fma(beta, q, m);
    s = fma(beta, s, w);
    pv = fma(beta, pv, u);
    x = fma(alpha, pv, x);
    r = fma(-alpha, s, r);
    u = fma(-alpha, q, u);
    w = fma(-alpha, z, w);
    m = di * w;
    if (own) mb[(it + 1) & 1][i] = m;
    ++its;
    gamma_old = gamma;
    alpha_old = alpha;
    block_reduce3(r * u, w * u, r * r, red, blockIdx.x, pt[(it + 1) & 1][0], pt[(it + 1) & 1][1], pt[(it + 1) & 1][2]);
    grid.sync();
  }
  if (own) xout[i] = x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its = its;
    st->its_sum += its;
    if (breakdown) st->breakdown = 1;
    st->done = 1;
    st->bb = bb;
  }
}

// ------------------------------------------------------------------------------------------
// Pipelined Jacobi-PCG for coarse systems too large for one thread per unknown (more unknowns
// than resident threads: 16^3+ elements at p0 = 2): the same recurrence as k_pcg_gv_p2, grid-
// stride over the unknowns, the CG vectors in global memory (L2-resident at these sizes), and
// the rows of H_hat written out once at setup in column-major ELL form (k_build_coarse_ell: 25
// index / coefficient pairs per unknown, build_row above), so an operator application is 25
// coalesced loads of the row plus 25 gathers -- no index arithmetic in the iteration.
// ------------------------------------------------------------------------------------------
__global__ void k_build_coarse_ell(LevelGeom g, CoarseTabs ct, double lam, int* __restrict__ ellc,
                                   double* __restrict__ ella) {
  const long long n = g.nskel;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int jx[kRowLen];
    double a[kRowLen];
    build_row(g, ct, i, lam, jx, a);
#pragma unroll
    for (int k = 0; k < kRowLen; ++k) {
      ellc[k * n + i] = jx[k];
      ella[k * n + i] = a[k];
    }
  }
}

// vec: 8 n doubles [x | r | u | w | z | q | s | p]; mbuf: 2 n (m_i in slot i & 1)
__global__ void __launch_bounds__(256) k_pcg_gv_ell_p2(long long n, const double* __restrict__ b,
                                                      double* __restrict__ xout, double* __restrict__ vec,
                                                      double* __restrict__ mbuf, const double* __restrict__ dinv,
                                                      const int* __restrict__ ellc, const double* __restrict__ ella,
                                                      double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  const int nb = gridDim.x;
  const long long T = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double *X = vec, *R = vec + n, *U = vec + 2 * n, *W = vec + 3 * n, *Z = vec + 4 * n, *Q = vec + 5 * n,
         *S = vec + 6 * n, *Pv = vec + 7 * n;
  double* mb[2] = {mbuf, mbuf + n};
  double* pt[2][3] = {{part, part + nb, part + 2 * nb}, {part + 3 * nb, part + 4 * nb, part + 5 * nb}};
  auto apply = [&](const double* v, long long j) {
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < kRowLen; ++k) h = fma(__ldg(&ella[k * n + j]), __ldcg(&v[__ldg(&ellc[k * n + j])]), h);
    return h;
  };
  // r0 = b, u0 = D^-1 b (published in mb[1] for w0 = H u0)
  for (long long j = t0; j < n; j += T) {
    const double bj = b[j], uj = dinv[j] * bj;
    X[j] = 0.0; R[j] = bj; U[j] = uj; Z[j] = 0.0; Q[j] = 0.0; S[j] = 0.0; Pv[j] = 0.0;
    mb[1][j] = uj;
  }
  grid.sync();
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (long long j = t0; j < n; j += T) {
    const double w = apply(mb[1], j), m = dinv[j] * w, rj = R[j], uj = U[j];
    W[j] = w;
    mb[0][j] = m;
    sa = fma(rj, uj, sa); sb = fma(w, uj, sb); sc = fma(rj, rj, sc);
  }
  block_reduce3(sa, sb, sc, red, blockIdx.x, pt[0][0], pt[0][1], pt[0][2]);
  grid.sync();
  double gamma_old = 1.0, alpha_old = 1.0, bb = -1.0;
  int its = 0, breakdown = 0;
  for (int it = 0;; ++it) {
    double gamma, delta, rho;
    grid_totals3(pt[it & 1][0], pt[it & 1][1], pt[it & 1][2], nb, red, gamma, delta, rho);
    if (it == 0) bb = rho;
    if (bb == 0.0 || sqrt(rho) <= rtol * sqrt(bb) || its >= maxit) break;
    double alpha, beta;
    if (it == 0) {
      beta = 0.0;
      if (!(delta > 0.0)) { breakdown = 1; break; }
      alpha = gamma / delta;
    } else {
      beta = gamma / gamma_old;
      const double den = delta - beta * gamma / alpha_old;
      if (!(den > 0.0)) { breakdown = 1; break; }
      alpha = gamma / den;
    }
    const double* mcur = mb[it & 1];
    double* mnext = mb[(it + 1) & 1];
    sa = 0.0; sb = 0.0; sc = 0.0;
    for (long long j = t0; j < n; j += T) {
      const double nv = apply(mcur, j), m = __ldcg(&mcur[j]);
      const double z = fma(beta, Z[j], nv), q = fma(beta, Q[j], m);
      const double w0 = W[j], s = fma(beta, S[j], w0), pv = fma(beta, Pv[j], U[j]);
      const double x = fma(alpha, pv, X[j]), r = fma(-alpha, s, R[j]);
      const double u = fma(-alpha, q, U[j]), w = fma(-alpha, z, w0);
      Z[j] = z; Q[j] = q; S[j] = s; Pv[j] = pv; X[j] = x; R[j] = r; U[j] = u; W[j] = w;
      mnext[j] = dinv[j] * w;
      sa = fma(r, u, sa); sb = fma(w, u, sb); sc = fma(r, r, sc);
    }
    ++its;
    gamma_old = gamma;
    alpha_old = alpha;
    block_reduce3(sa, sb, sc, red, blockIdx.x, pt[(it + 1) & 1][0], pt[(it + 1) & 1][1], pt[(it + 1) & 1][2]);
    grid.sync();
  }
  for (long long j = t0; j < n; j += T) xout[j] = X[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its = its;
    st->its_sum += its;
    if (breakdown) st->breakdown = 1;
    st->done = 1;
    st->bb = bb;
  }
}

// ------------------------------------------------------------------------------------------
// CG on the coarse system with the h-multigrid V-cycle as preconditioner (reading R16,
// oracle/hmg.py), matrix-free on the p = 2 GRID layout of every h-level.
//
// Every h-level is a p = 2 mesh; its vectors are (2k_1+1)(2k_2+1)(2k_3+1) grid arrays, x1 fastest,
// with the element centres (all three indices odd) and the non-free points held at zero.  The
// condensed operator at p = 2 (see the header of this file) is evaluated on the fly:
//   q_i = lam B1 B2 B3 v_i + sum_d (B_a B_b) sum_{o=-2..2} K_d[G_d][o] v_{i + o s_d}
//         - sum_{elements e with i a face centre of e} H_{c,i} (H_cB v_B) / H_cc,
// the 1-D assembled lumped masses B_d and stiffness rows K_d per grid index, and per direction and
// element index the centre row of the element's 1-D matrices (m = M[1], K[1][0], K[1][2], K[1][1]):
//   H_{c, face d low}  = K_d[1][0] m_a m_b,   H_{c, face d high} = K_d[1][2] m_a m_b,
//   H_cc = lam m1 m2 m3 + K_1[1][1] m2 m3 + m1 K_2[1][1] m3 + m1 m2 K_3[1][1].
// An operator application reads one vector (stencil neighbours from L1 / L2) and writes one: about
// 16 B per point instead of the 300 B of an assembled 25-entry ELL row.  The transfers are
// tensor-product 1-D tables: prolongation = the coarse element's quadratic at the fine node with the
// centre value replaced by its harmonic extension -H_cB u_B / H_cc; restriction = its exact
// transpose (a gather of <= 7 fine nodes per direction, plus the centre gathers redistributed to the
// face centres).
// ------------------------------------------------------------------------------------------
// experiment builds (-DPMG_HMG_TRACE): block 0 stamps %globaltimer at every grid barrier of the
// h-multigrid CG (first 8192 barriers of a launch) -> pmg_debug_hmg_trace
#ifndef PMG_HMG_MINB
#define PMG_HMG_MINB 2   // blocks per SM of k_pcg_hmg_p2 (register cap 128)
#endif
#ifdef PMG_HMG_TRACE
__device__ unsigned long long g_hmg_trace[2 * 8192];
__device__ int g_hmg_ntrace;
#define HSYNC(tag)                                                                            \
  do {                                                                                        \
    grid.sync();                                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_hmg_ntrace < 8192) {                         \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
      g_hmg_trace[2 * g_hmg_ntrace] = t_;                                                     \
      g_hmg_trace[2 * g_hmg_ntrace + 1] = (tag);                                              \
      g_hmg_ntrace++;                                                                         \
    }                                                                                         \
  } while (0)
#else
#define HSYNC(tag) grid.sync()
#endif

namespace {
constexpr double kHmgOmega = 0.6;
constexpr int kHmgNu = 2, kHmgCoarsest = 40;

// the 4-entry element row e of a per-direction table (two 16-byte read-only loads)
__device__ __forceinline__ double4 ld_row4(const double* t, int e) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(t) + 2 * e);
  const double2 b = __ldg(reinterpret_cast<const double2*>(t) + 2 * e + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// 1 / x from the hardware approximation and one cubic Newton step (error e^3 of the ~2^-23
// approximation: below double rounding); replaces the FP64 division sequence in the stencils
__device__ __forceinline__ double hg_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

__device__ __forceinline__ void hg_decode(const HGridLev& L, long long i, int& g1, int& g2, int& g3) {
  const unsigned u = (unsigned)i, t = u / (unsigned)L.N1;
  g1 = (int)(u - t * (unsigned)L.N1);
  g3 = (int)(t / (unsigned)L.N2);
  g2 = (int)(t - (unsigned)g3 * (unsigned)L.N2);
}

__device__ __forceinline__ bool hg_free(const HGridLev& L, int g1, int g2, int g3) {
  if (g1 & g2 & g3 & 1) return false;   // element centre: condensed out
  return free_1d(g1, L.N1 - 1, L.neu & 1, (L.neu >> 1) & 1) && free_1d(g2, L.N2 - 1, (L.neu >> 2) & 1, (L.neu >> 3) & 1) &&
         free_1d(g3, L.N3 - 1, (L.neu >> 4) & 1, (L.neu >> 5) & 1);
}

// Point pairs: the grid sweeps below give each thread the two x1-neighbours P0 = (2j, g2, g3) and
// P1 = (2j + 1, g2, g3) (P1 absent at j = k1).  Both share the x1-line loads, the x2 / x3 tables and
// the coarse element of the transfers, and the point types of a pair depend on (g2, g3) only, so
// the lanes of a warp (consecutive j) take the same branch.
struct HPair {
  int i0;            // grid index of P0 (h-level grids have < 2^31 points)
  int j, g2, g3;
  bool h1, f0, f1;   // P1 exists; P0 / P1 are free unknowns
};

__device__ __forceinline__ HPair hg_pair(const HGridLev& L, long long ip) {
  HPair P;
  const unsigned np1 = (unsigned)L.k1 + 1u;
  const unsigned u = (unsigned)ip, row = u / np1;
  P.j = (int)(u - row * np1);
  P.g3 = (int)(row / (unsigned)L.N2);
  P.g2 = (int)(row - (unsigned)P.g3 * (unsigned)L.N2);
  P.i0 = 2 * P.j + L.N1 * (int)row;
  const int G1 = 2 * P.j;
  P.h1 = G1 + 1 < L.N1;
  const bool f23 = free_1d(P.g2, L.N2 - 1, (L.neu >> 2) & 1, (L.neu >> 3) & 1) &&
                   free_1d(P.g3, L.N3 - 1, (L.neu >> 4) & 1, (L.neu >> 5) & 1);
  P.f0 = f23 && free_1d(G1, L.N1 - 1, L.neu & 1, (L.neu >> 1) & 1);
  P.f1 = f23 && P.h1 && !((P.g2 & 1) && (P.g3 & 1));   // odd x1 index: interior along x1; (o, o, o) is a centre
  return P;
}

__device__ __forceinline__ long long hg_npairs(const HGridLev& L) { return (long long)(L.k1 + 1) * L.N2 * L.N3; }

// plain vector (written inside the kernel: plain loads, ordered by the grid barriers)
struct HV {
  const double* p;
  __device__ __forceinline__ double operator()(int j) const { return p[j]; }
};
// omega D^-1 f: the first damped-Jacobi sweep from zero, evaluated where the second sweep reads it
struct HW {
  const double *d, *f;
  __device__ __forceinline__ double operator()(int j) const { return kHmgOmega * __ldg(&d[j]) * f[j]; }
};

// (H_cB v_B) / H_cc of the element with centre grid index ic
template <class Acc>
__device__ __forceinline__ double hg_centre(const HGridLev& L, const Acc& v, int ic, double lam, double4 E1,
                                            double4 E2, double4 E3) {
  const int s2 = L.N1, s3 = L.N1 * L.N2;
  const double m23 = E2.x * E3.x, m13 = E1.x * E3.x, m12 = E1.x * E2.x;
  double s = m23 * fma(E1.y, v(ic - 1), E1.z * v(ic + 1));
  s = fma(m13, fma(E2.y, v(ic - s2), E2.z * v(ic + s2)), s);
  s = fma(m12, fma(E3.y, v(ic - s3), E3.z * v(ic + s3)), s);
  const double hcc = fma(lam * E1.x, m23, fma(E1.w, m23, fma(E2.w, m13, E3.w * m12)));
  return s * hg_rcp(hcc);
}

// (H_hat v) at the pair's points (values at non-free points are meaningless; callers mask);
// v is zero at centres and non-free points.  Every load of the pair -- the x1 line, the x2 / x3 lines
// of both points, the tables and the six neighbours of the (up to two) element centres next to
// the pair's face centre -- is issued up front with out-of-range indices clamped to i0 (a harmless
// load whose coefficient is zero), so an application costs one memory round trip, not three.
template <class Acc>
__device__ __forceinline__ void hg_apply2(const HGridLev& L, const Acc& v, const HPair& P, double lam, double& q0,
                                          double& q1) {
  const int i0 = P.i0, s2 = L.N1, s3 = L.N1 * L.N2;
  const int G1 = 2 * P.j, g2 = P.g2, g3 = P.g3;
  const bool lo = P.j >= 1, h1 = P.h1, h2 = G1 + 2 < L.N1;
  auto cl = [&](bool ok, int k) { return ok ? k : i0; };
  auto cz = [](bool ok, double x) { return ok ? x : 0.0; };
  // ---- loads ----
  const double va = v(cl(lo, i0 - 2)), vb = v(cl(lo, i0 - 1)), vc = v(i0), vd = v(cl(h1, i0 + 1)), ve = v(cl(h2, i0 + 2));
  const bool y0 = g2 >= 2, y1 = g2 >= 1, y3 = g2 + 1 < L.N2, y4 = g2 + 2 < L.N2;
  const bool z0 = g3 >= 2, z1 = g3 >= 1, z3 = g3 + 1 < L.N3, z4 = g3 + 2 < L.N3;
  const double a20 = v(cl(y0, i0 - 2 * s2)), a21 = v(cl(y1, i0 - s2)), a23 = v(cl(y3, i0 + s2)), a24 = v(cl(y4, i0 + 2 * s2));
  const double a30 = v(cl(z0, i0 - 2 * s3)), a31 = v(cl(z1, i0 - s3)), a33 = v(cl(z3, i0 + s3)), a34 = v(cl(z4, i0 + 2 * s3));
  const int i1 = cl(h1, i0 + 1);
  const double b20 = v(cl(h1 && y0, i1 - 2 * s2)), b21 = v(cl(h1 && y1, i1 - s2)), b23 = v(cl(h1 && y3, i1 + s2)),
               b24 = v(cl(h1 && y4, i1 + 2 * s2));
  const double b30 = v(cl(h1 && z0, i1 - 2 * s3)), b31 = v(cl(h1 && z1, i1 - s3)), b33 = v(cl(h1 && z3, i1 + s3)),
               b34 = v(cl(h1 && z4, i1 + 2 * s3));
  // face centre of the pair: kind 1 = P0 (even, odd, odd) normal to x1; 2 = P1 (odd, odd, even) normal to
  // x3; 3 = P1 (odd, even, odd) normal to x2; 0 = none.  Side 0: the element above, 1: below.
  const bool o2 = g2 & 1, o3 = g3 & 1;
  const int kind = (o2 && o3) ? 1 : ((o2 && h1) ? 2 : ((o3 && h1) ? 3 : 0));
  const int ea = kind == 1 ? (g2 - 1) >> 1 : P.j < L.k1 ? P.j : 0;           // x1 element (kinds 2, 3)
  const int Gd = kind == 1 ? G1 : (kind == 2 ? g3 : g2);
  const int kd = kind == 1 ? L.k1 : (kind == 2 ? L.k3 : L.k2);
  const int sd = kind == 1 ? 1 : (kind == 2 ? s3 : s2);
  const int fc = kind == 1 ? i0 : i1;                                   // the face centre
  const bool ok0 = kind != 0 && (Gd >> 1) < kd, ok1 = kind != 0 && (Gd >> 1) >= 1;
  const int ed0 = ok0 ? (Gd >> 1) : 0, ed1 = ok1 ? (Gd >> 1) - 1 : 0;
  // tangential element rows: kind 1: x2 and x3; kind 2: x1 and x2; kind 3: x1 and x3
  const double4 Ta = kind == 1 ? ld_row4(L.E[1], (g2 - 1) >> 1) : ld_row4(L.E[0], ea);
  const double4 Tb = kind == 2 ? ld_row4(L.E[1], o2 ? (g2 - 1) >> 1 : 0)
                               : ld_row4(L.E[2], o3 ? (g3 - 1) >> 1 : 0);
  const double* Ed = L.E[kind == 1 ? 0 : (kind == 2 ? 2 : 1)];
  const double4 N0 = ld_row4(Ed, ed0), N1 = ld_row4(Ed, ed1);
  const int c0 = cl(ok0, fc + sd), c1 = cl(ok1, fc - sd);
  const double u0m1 = v(cl(ok0, c0 - 1)), u0p1 = v(cl(ok0, c0 + 1)), u0m2 = v(cl(ok0, c0 - s2)), u0p2 = v(cl(ok0, c0 + s2)),
               u0m3 = v(cl(ok0, c0 - s3)), u0p3 = v(cl(ok0, c0 + s3));
  const double u1m1 = v(cl(ok1, c1 - 1)), u1p1 = v(cl(ok1, c1 + 1)), u1m2 = v(cl(ok1, c1 - s2)), u1p2 = v(cl(ok1, c1 + s2)),
               u1m3 = v(cl(ok1, c1 - s3)), u1p3 = v(cl(ok1, c1 + s3));
  const double B2 = __ldg(&L.b[1][g2]), B3 = __ldg(&L.b[2][g3]), B1a = __ldg(&L.b[0][G1]);
  const double B1b = h1 ? __ldg(&L.b[0][G1 + 1]) : 0.0;
  const double* K1a = L.K[0] + 5 * G1;
  const double* K1b = L.K[0] + 5 * (h1 ? G1 + 1 : G1);
  const double* K2r = L.K[1] + 5 * g2;
  const double* K3r = L.K[2] + 5 * g3;
  // ---- arithmetic ----
  const double B23 = B2 * B3;
  double x1 = __ldg(&K1a[2]) * vc;
  x1 = fma(__ldg(&K1a[0]), cz(lo, va), x1);
  x1 = fma(__ldg(&K1a[1]), cz(lo, vb), x1);
  x1 = fma(__ldg(&K1a[3]), cz(h1, vd), x1);
  x1 = fma(__ldg(&K1a[4]), cz(h2, ve), x1);
  const double k20 = __ldg(&K2r[0]), k21 = __ldg(&K2r[1]), k22 = __ldg(&K2r[2]), k23 = __ldg(&K2r[3]), k24 = __ldg(&K2r[4]);
  const double k30 = __ldg(&K3r[0]), k31 = __ldg(&K3r[1]), k32 = __ldg(&K3r[2]), k33 = __ldg(&K3r[3]), k34 = __ldg(&K3r[4]);
  auto line = [&](double c, double m2, double m1, double p1, double p2, double k0, double k1, double k2, double k3,
                  double k4, bool e0, bool e1, bool e3, bool e4) {
    double acc = k2 * c;
    acc = fma(k0, cz(e0, m2), acc);
    acc = fma(k1, cz(e1, m1), acc);
    acc = fma(k3, cz(e3, p1), acc);
    acc = fma(k4, cz(e4, p2), acc);
    return acc;
  };
  q0 = lam * B1a * B23 * vc;
  q0 = fma(B23, x1, q0);
  q0 = fma(B1a * B3, line(vc, a20, a21, a23, a24, k20, k21, k22, k23, k24, y0, y1, y3, y4), q0);
  q0 = fma(B1a * B2, line(vc, a30, a31, a33, a34, k30, k31, k32, k33, k34, z0, z1, z3, z4), q0);
  const double vdd = cz(h1, vd);
  double y1s = __ldg(&K1b[2]) * vdd;
  y1s = fma(__ldg(&K1b[1]), vc, y1s);
  y1s = fma(__ldg(&K1b[3]), cz(h2, ve), y1s);
  q1 = lam * B1b * B23 * vdd;
  q1 = fma(B23, y1s, q1);
  q1 = fma(B1b * B3, line(vdd, b20, b21, b23, b24, k20, k21, k22, k23, k24, h1 && y0, h1 && y1, h1 && y3, h1 && y4), q1);
  q1 = fma(B1b * B2, line(vdd, b30, b31, b33, b34, k30, k31, k32, k33, k34, h1 && z0, h1 && z1, h1 && z3, h1 && z4), q1);
  if (kind != 0) {
    // element rows in direction order (E1, E2, E3) for the two sides
    auto corr = [&](const double4& Nn, double um1, double up1, double um2, double up2, double um3, double up3, int side) {
      const double4 E1 = kind == 1 ? Nn : Ta;
      const double4 E2 = kind == 1 ? Ta : (kind == 2 ? Tb : Nn);
      const double4 E3 = kind == 1 ? Tb : (kind == 2 ? Nn : Tb);
      const double m23 = E2.x * E3.x, m13 = E1.x * E3.x, m12 = E1.x * E2.x;
      double s = m23 * fma(E1.y, um1, E1.z * up1);
      s = fma(m13, fma(E2.y, um2, E2.z * up2), s);
      s = fma(m12, fma(E3.y, um3, E3.z * up3), s);
      const double hcc = fma(lam * E1.x, m23, fma(E1.w, m23, fma(E2.w, m13, E3.w * m12)));
      const double mab = kind == 1 ? m23 : (kind == 2 ? m12 : m13);
      return (side ? Nn.z : Nn.y) * mab * (s * hg_rcp(hcc));
    };
    double c = 0.0;
    if (ok0) c += corr(N0, u0m1, u0p1, u0m2, u0p2, u0m3, u0p3, 0);
    if (ok1) c += corr(N1, u1m1, u1p1, u1m2, u1p2, u1m3, u1p3, 1);
    if (kind == 1) q0 -= c; else q1 -= c;
  }
}

// prolongation into the pair's points of level F from the coarse level C vector xc: the coarse
// element's quadratic with the centre value replaced by its harmonic extension -H_cB u_B / H_cc
// (both points lie in the same coarse element)
__device__ __forceinline__ void hg_prolong2(const HGridLev& F, const HGridLev& C, const double* xc, const HPair& P,
                                            double lam, double& s0, double& s1) {
  const int G1 = 2 * P.j;
  const int ec1 = __ldg(&F.pe[0][G1]), ec2 = __ldg(&F.pe[1][P.g2]), ec3 = __ldg(&F.pe[2][P.g3]);
  const int cs2 = C.N1, cs3 = C.N1 * C.N2;
  const int cb = 2 * ec1 + cs2 * (2 * ec2) + cs3 * (2 * ec3);
  double wa[3], wb[3], w2[3], w3[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    wa[t] = __ldg(&F.pw[0][3 * G1 + t]);
    wb[t] = P.h1 ? __ldg(&F.pw[0][3 * G1 + 3 + t]) : 0.0;
    w2[t] = __ldg(&F.pw[1][3 * P.g2 + t]);
    w3[t] = __ldg(&F.pw[2][3 * P.g3 + t]);
  }
  const double4 E1 = ld_row4(C.E[0], ec1), E2 = ld_row4(C.E[1], ec2), E3 = ld_row4(C.E[2], ec3);
  const double uc = -hg_centre(C, HV{xc}, cb + 1 + cs2 + cs3, lam, E1, E2, E3);
  s0 = 0.0;
  s1 = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double u = (a == 1 && b == 1 && c == 1) ? uc : xc[cb + a + cs2 * b + cs3 * c];
        sa = fma(wa[a], u, sa);
        sb = fma(wb[a], u, sb);
      }
      t0 = fma(w2[b], sa, t0);
      t1 = fma(w2[b], sb, t1);
    }
    s0 = fma(w3[c], t0, s0);
    s1 = fma(w3[c], t1, s1);
  }
}

// Restriction R = P^T from level F to level C, tensor-product form in three passes (barriers between):
//   T1 = (R_1 x I x I) r_f,  T2 = (I x R_2 x I) T1,  T3 = (I x I x R_3) T2  (the transposed 1-D
// interpolations, <= 7 fine nodes per coarse node), then f_c = E^T T3: a free coarse face centre adds
// -H_cf / H_cc times T3 at the centres of its (up to two) elements (the transposed harmonic extension).
__device__ __forceinline__ double hg_dot7(const double* __restrict__ w, int n, const double* v, long long stride) {
  double s = 0.0;
#pragma unroll
  for (int a = 0; a < 7; ++a)
    if (a < n) s = fma(__ldg(&w[a]), v[a * stride], s);
  return s;
}

__device__ __forceinline__ double hg_t3(const HGridLev& F, const HGridLev& C, int J1, int J2, int J3) {
  const long long plane = (long long)C.N1 * C.N2;
  const int c0 = __ldg(&F.r0[2][J3]), nc = __ldg(&F.rn[2][J3]);
  return hg_dot7(F.rw[2] + 7 * J3, nc, F.t2 + J1 + (long long)C.N1 * J2 + plane * c0, plane);
}

__device__ __forceinline__ double hg_restrict(const HGridLev& F, const HGridLev& C, int J1, int J2, int J3, double lam) {
  double s = hg_t3(F, C, J1, J2, J3);
  if ((J1 & 1) + (J2 & 1) + (J3 & 1) == 2) {   // coarse face centre: the centres' harmonic-extension share
    const int d = (J1 & 1) == 0 ? 0 : ((J2 & 1) == 0 ? 1 : 2);
    const int Jd = d == 0 ? J1 : (d == 1 ? J2 : J3);
    const int kd = d == 0 ? C.k1 : (d == 1 ? C.k2 : C.k3);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int ed = (Jd >> 1) - side;
      if (ed < 0 || ed >= kd) continue;
      const int e1 = d == 0 ? ed : (J1 - 1) >> 1, e2 = d == 1 ? ed : (J2 - 1) >> 1, e3 = d == 2 ? ed : (J3 - 1) >> 1;
      const double4 E1 = ld_row4(C.E[0], e1);
      const double4 E2 = ld_row4(C.E[1], e2);
      const double4 E3 = ld_row4(C.E[2], e3);
      const double m23 = E2.x * E3.x, m13 = E1.x * E3.x, m12 = E1.x * E2.x;
      const double hcc = fma(lam * E1.x, m23, fma(E1.w, m23, fma(E2.w, m13, E3.w * m12)));
      const double kf = d == 0 ? (side ? E1.z : E1.y) : (d == 1 ? (side ? E2.z : E2.y) : (side ? E3.z : E3.y));
      const double mab = d == 0 ? m23 : (d == 1 ? m13 : m12);
      s = fma(-(kf * mab) * hg_rcp(hcc), hg_t3(F, C, 2 * e1 + 1, 2 * e2 + 1, 2 * e3 + 1), s);
    }
  }
  return s;
}

// z = V-cycle(f_0) into h.L[0].x; h.L[0].f holds the right-hand side.  With rz_part set, the block's
// partial of f_0 . z (the CG's r.z) is formed in the last level-0 sweep and published before the
// V-cycle's final barrier, which then doubles as the CG's reduction barrier.
__device__ void hg_vcycle(const HmgGridDev& h, cg::grid_group& grid, long long t0, long long T, double lam,
                          double* red, double* rz_part) {
  const int Lc = h.nlev - 1;
  for (int l = 0; l < Lc; ++l) {
    const HGridLev& L = h.L[l];
    const long long np = hg_npairs(L);
    // the two pre-sweeps from zero in one pass: x1 = omega D^-1 f is local, so
    // x2_i = x1_i + omega d_i (f_i - sum_j A_ij x1_j) gathers omega d_j f_j directly
    static_assert(kHmgNu == 2, "the fused sweeps below are written for nu = 2");
    for (long long ip = t0; ip < np; ip += T) {
      const HPair P = hg_pair(L, ip);
      double a0, a1;
      hg_apply2(L, HW{L.dinv, L.f}, P, lam, a0, a1);
      {
        const double wd = kHmgOmega * __ldg(&L.dinv[P.i0]), fi = L.f[P.i0];
        L.x[P.i0] = P.f0 ? fma(wd, fi - a0, wd * fi) : 0.0;
      }
      if (P.h1) {
        const double wd = kHmgOmega * __ldg(&L.dinv[P.i0 + 1]), fi = L.f[P.i0 + 1];
        L.x[P.i0 + 1] = P.f1 ? fma(wd, fi - a1, wd * fi) : 0.0;
      }
    }
    HSYNC(1 + 100 * l);
    for (long long ip = t0; ip < np; ip += T) {
      const HPair P = hg_pair(L, ip);
      double a0, a1;
      hg_apply2(L, HV{L.x}, P, lam, a0, a1);
      L.r[P.i0] = P.f0 ? L.f[P.i0] - a0 : 0.0;
      if (P.h1) L.r[P.i0 + 1] = P.f1 ? L.f[P.i0 + 1] - a1 : 0.0;
    }
    HSYNC(2 + 100 * l);
    const HGridLev& C = h.L[l + 1];
    {   // T1[J1, G2, G3] = sum_a R_1(J1, a) r[a, G2, G3]
      const long long n1 = (long long)C.N1 * L.N2 * L.N3;
      for (long long j = t0; j < n1; j += T) {
        const unsigned row = (unsigned)j / (unsigned)C.N1, J1 = (unsigned)j - row * (unsigned)C.N1;
        L.t1[j] = hg_dot7(L.rw[0] + 7 * J1, __ldg(&L.rn[0][J1]), L.r + (long long)L.N1 * row + __ldg(&L.r0[0][J1]), 1);
      }
    }
    HSYNC(12 + 100 * l);
    {   // T2[J1, J2, G3] = sum_b R_2(J2, b) T1[J1, b, G3]
      const long long n2 = (long long)C.N1 * C.N2 * L.N3;
      for (long long j = t0; j < n2; j += T) {
        const unsigned t = (unsigned)j / (unsigned)C.N1, J1 = (unsigned)j - t * (unsigned)C.N1;
        const unsigned G3 = t / (unsigned)C.N2, J2 = t - G3 * (unsigned)C.N2;
        L.t2[j] = hg_dot7(L.rw[1] + 7 * J2, __ldg(&L.rn[1][J2]),
                          L.t1 + J1 + (long long)C.N1 * (__ldg(&L.r0[1][J2]) + (long long)L.N2 * G3), C.N1);
      }
    }
    HSYNC(13 + 100 * l);
    for (long long j = t0; j < C.n; j += T) {
      int J1, J2, J3;
      hg_decode(C, j, J1, J2, J3);
      C.f[j] = hg_free(C, J1, J2, J3) ? hg_restrict(L, C, J1, J2, J3, lam) : 0.0;
    }
    HSYNC(3 + 100 * l);
  }
  const HGridLev& LC = h.L[Lc];
  if (h.ncf > 0) {                       // coarsest level: x = A^-1 f (dense inverse, warp per row)
    const int lane = (int)(t0 & 31);
    for (long long i = t0 >> 5; i < h.ncf; i += T >> 5) {
      const double* row = h.cinv + i * (long long)h.ncf;
      double s = 0.0;
      for (int j = lane; j < h.ncf; j += 32) s = fma(__ldg(&row[j]), LC.f[__ldg(&h.cidx[j])], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) LC.x[__ldg(&h.cidx[i])] = s;
    }
  } else if (blockIdx.x == 0) {          // large coarsest level: block 0, Jacobi sweeps, block barriers
    const long long np = hg_npairs(LC);
    for (long long i = threadIdx.x; i < LC.n; i += blockDim.x) LC.x[i] = kHmgOmega * __ldg(&LC.dinv[i]) * LC.f[i];
    __syncthreads();
    for (int sw = 1; sw < kHmgCoarsest; ++sw) {
      for (long long ip = threadIdx.x; ip < np; ip += blockDim.x) {
        const HPair P = hg_pair(LC, ip);
        double a0, a1;
        hg_apply2(LC, HV{LC.x}, P, lam, a0, a1);
        LC.r[P.i0] = P.f0 ? LC.f[P.i0] - a0 : 0.0;
        if (P.h1) LC.r[P.i0 + 1] = P.f1 ? LC.f[P.i0 + 1] - a1 : 0.0;
      }
      __syncthreads();
      for (long long i = threadIdx.x; i < LC.n; i += blockDim.x) LC.x[i] = fma(kHmgOmega * __ldg(&LC.dinv[i]), LC.r[i], LC.x[i]);
      __syncthreads();
    }
  }
  HSYNC(4);
  for (int l = Lc - 1; l >= 0; --l) {
    const HGridLev& L = h.L[l];
    const HGridLev& C = h.L[l + 1];
    const long long np = hg_npairs(L);
    for (long long ip = t0; ip < np; ip += T) {
      const HPair P = hg_pair(L, ip);
      if (!(P.f0 || P.f1)) continue;
      double s0, s1;
      hg_prolong2(L, C, C.x, P, lam, s0, s1);
      if (P.f0) L.x[P.i0] += s0;
      if (P.f1) L.x[P.i0 + 1] += s1;
    }
    HSYNC(5 + 100 * l);
    // two post-sweeps, each one pass, ping-pong x -> r -> x (r is free here)
    for (long long ip = t0; ip < np; ip += T) {
      const HPair P = hg_pair(L, ip);
      double a0, a1;
      hg_apply2(L, HV{L.x}, P, lam, a0, a1);
      L.r[P.i0] = P.f0 ? fma(kHmgOmega * __ldg(&L.dinv[P.i0]), L.f[P.i0] - a0, L.x[P.i0]) : 0.0;
      if (P.h1) L.r[P.i0 + 1] = P.f1 ? fma(kHmgOmega * __ldg(&L.dinv[P.i0 + 1]), L.f[P.i0 + 1] - a1, L.x[P.i0 + 1]) : 0.0;
    }
    HSYNC(6 + 100 * l);
    double srz = 0.0;
    for (long long ip = t0; ip < np; ip += T) {
      const HPair P = hg_pair(L, ip);
      double a0, a1;
      hg_apply2(L, HV{L.r}, P, lam, a0, a1);
      double x0 = 0.0, x1 = 0.0;
      if (P.f0) {
        const double fi = L.f[P.i0];
        x0 = fma(kHmgOmega * __ldg(&L.dinv[P.i0]), fi - a0, L.r[P.i0]);
        srz = fma(fi, x0, srz);
      }
      if (P.f1) {
        const double fi = L.f[P.i0 + 1];
        x1 = fma(kHmgOmega * __ldg(&L.dinv[P.i0 + 1]), fi - a1, L.r[P.i0 + 1]);
        srz = fma(fi, x1, srz);
      }
      L.x[P.i0] = x0;
      if (P.h1) L.x[P.i0 + 1] = x1;
    }
    if (l == 0 && rz_part) block_reduce3(srz, srz, srz, red, blockIdx.x, rz_part, rz_part, rz_part);
    HSYNC(7 + 100 * l);
  }
  if (Lc == 0 && rz_part) {   // a single h-level (the dense solve alone): r.z after it
    const HGridLev& L = h.L[0];
    double srz = 0.0;
    for (long long i = t0; i < L.n; i += T) srz = fma(L.f[i], L.x[i], srz);
    block_reduce3(srz, srz, srz, red, blockIdx.x, rz_part, rz_part, rz_part);
    HSYNC(8);
  }
}
}  // namespace

// Standard PCG (as mg.pcg / hmg.pcg_hmg): x = 0, r = b, z = M^-1 r, p = z; q = A p, alpha = r.z / p.q,
// x += alpha p, r -= alpha q, stop at ||r|| <= rtol ||b||, z = M^-1 r, beta = r.z_new / r.z, p = z + beta p.
// b and xout are skeleton-record vectors of the p0 = 2 level (geometry h.g0); inside, r lives in
// h.L[0].f (the V-cycle's right-hand side), z in h.L[0].x, x / p / q in the grid arrays X / pv / q.
__global__ void __launch_bounds__(256, PMG_HMG_MINB) k_pcg_hmg_p2(HmgGridDev h, const double* __restrict__ b, double* __restrict__ xout,
                                                   double* __restrict__ X, double* __restrict__ pv,
                                                   double* __restrict__ q, double lam, double* __restrict__ part,
                                                   PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  const int nb = gridDim.x;
  const HGridLev& L0 = h.L[0];
  const long long n = L0.n, np = hg_npairs(L0);
  const long long T = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double* R = L0.f;
  double* Z = L0.x;
  double *pa = part, *pb = part + nb, *pc = part + 2 * nb;
  double sb = 0.0;
  for (long long i = t0; i < n; i += T) {   // record layout -> grid layout (free points only)
    int g1, g2, g3;
    hg_decode(L0, i, g1, g2, g3);
    const double bi = hg_free(L0, g1, g2, g3) ? b[sidx2(h.g0, g1, g2, g3)] : 0.0;
    X[i] = 0.0;
    R[i] = bi;
    sb = fma(bi, bi, sb);
  }
  block_reduce3(sb, 0.0, 0.0, red, blockIdx.x, pa, pb, pc);
  HSYNC(9);
  double bb, d1, d2;
  grid_totals3(pa, pb, pc, nb, red, bb, d1, d2);
  int its = 0, breakdown = 0;
  if (bb > 0.0) {
    // partial sums: p.q in pa, r.r in pb, r.z in pc -- consecutive reductions use different
    // buffers, so a block that runs ahead never overwrites a partial another block still reads.
    // Two grid barriers per iteration besides the V-cycle's: with p_new = z + beta p,
    // q_new = H z + beta q_old, so the direction, the operator application (z is complete after
    // the V-cycle) and p.q share one phase; r.z is reduced inside the V-cycle's last sweep
    hg_vcycle(h, grid, t0, T, lam, red, pc);
    double rz, pq;
    grid_totals3(pc, pc, pc, nb, red, rz, d1, d2);
    double beta = 0.0;
    for (;;) {
      double spq = 0.0;
      for (long long ip = t0; ip < np; ip += T) {
        const HPair P = hg_pair(L0, ip);
        double a0, a1;
        hg_apply2(L0, HV{Z}, P, lam, a0, a1);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (k == 1 && !P.h1) break;
          const long long i = P.i0 + k;
          const double hz = (k ? P.f1 : P.f0) ? (k ? a1 : a0) : 0.0;
          const double pvi = its == 0 ? Z[i] : fma(beta, pv[i], Z[i]);
          const double qi = its == 0 ? hz : fma(beta, q[i], hz);
          pv[i] = pvi;
          q[i] = qi;
          spq = fma(pvi, qi, spq);
        }
      }
      block_reduce3(spq, spq, spq, red, blockIdx.x, pa, pa, pa);
      HSYNC(10);
      grid_totals3(pa, pa, pa, nb, red, pq, d1, d2);
      if (!(pq > 0.0)) { breakdown = 1; break; }
      const double alpha = rz / pq;
      double srr = 0.0;
      for (long long i = t0; i < n; i += 4 * T) {   // four points per thread in flight
        double xv[4], pvv[4], qv[4], rv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const long long ik = i + k * T < n ? i + k * T : i;
          xv[k] = X[ik]; pvv[k] = pv[ik]; qv[k] = q[ik]; rv[k] = R[ik];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (i + k * T >= n) break;
          X[i + k * T] = fma(alpha, pvv[k], xv[k]);
          const double ri = fma(-alpha, qv[k], rv[k]);
          R[i + k * T] = ri;
          srr = fma(ri, ri, srr);
        }
      }
      block_reduce3(srr, srr, srr, red, blockIdx.x, pb, pb, pb);
      HSYNC(11);
      double rr;
      grid_totals3(pb, pb, pb, nb, red, rr, d1, d2);
      ++its;
      if (sqrt(rr) <= rtol * sqrt(bb) || its >= maxit) break;
      hg_vcycle(h, grid, t0, T, lam, red, pc);
      double rzn;
      grid_totals3(pc, pc, pc, nb, red, rzn, d1, d2);
      beta = rzn / rz;
      rz = rzn;
    }
  }
  // grid layout -> record layout (every record entry written; outside the box / non-free: 0)
  const long long nrec = h.g0.nskel;
  for (long long j = t0; j < nrec; j += T) {
    const Entry E = decode2(h.g0, j);
    const bool in = E.g1 <= 2 * h.g0.k1 && E.g2 <= 2 * h.g0.k2 && E.g3 <= 2 * h.g0.k3;
    xout[j] = in ? X[E.g1 + L0.N1 * ((long long)E.g2 + (long long)L0.N2 * E.g3)] : 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its = its;
    st->its_sum += its;
    if (breakdown) st->breakdown = 1;
    st->done = 1;
    st->bb = bb;
  }
}

// Two grid barriers per iteration: with p_new = z + beta p and q = H_hat p,
//   q_new = H_hat z + beta q_old,
// so the direction update, the operator application (on z, complete after the previous barrier)
// and the partial p.q share one phase; the x / r / z update and the partials r.r, r.z the other.
__global__ void __launch_bounds__(256) k_pcg_coop_p2(LevelGeom g, CoarseTabs ct, const double* __restrict__ b,
                                                    double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                                    double* __restrict__ pv, double* __restrict__ q,
                                                    const double* __restrict__ dinv, double lam,
                                                    double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[64];
  const int nb = gridDim.x;
  double* part_a = part;           // p.q
  double* part_b = part + nb;      // r.r (b.b at init)
  double* part_c = part + 2 * nb;  // r.z
  const long long n = g.nskel;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  double s1 = 0.0, s2 = 0.0;
  for (long long i = tid; i < n; i += nth) {
    const double bi = b[i], zi = dinv[i] * bi;
    x[i] = 0.0; r[i] = bi; z[i] = zi; pv[i] = 0.0; q[i] = 0.0;
    s1 = fma(bi, zi, s1); s2 = fma(bi, bi, s2);
  }
  s1 = block_reduce(s1, red);
  if (threadIdx.x == 0) part_c[blockIdx.x] = s1;
  s2 = block_reduce(s2, red);
  if (threadIdx.x == 0) part_b[blockIdx.x] = s2;
  grid.sync();
  double rz, bb, dummy;
  grid_totals(part_c, part_b, nb, red, rz, bb);
  (void)dummy;
  double beta = 0.0;
  int its = 0, breakdown = 0;
  bool done = (bb == 0.0);
  while (!done) {
    // phase 1: p = z + beta p ; q = H_hat z + beta q ; partial p.q
    double spq = 0.0;
    for (long long i = tid; i < n; i += nth) {
      const double pi_ = fma(beta, pv[i], z[i]);
      const double qi = fma(beta, q[i], apply_entry(g, ct, GlobalAcc{z}, i, lam));
      pv[i] = pi_;
      q[i] = qi;
      spq = fma(pi_, qi, spq);
    }
    spq = block_reduce(spq, red);
    if (threadIdx.x == 0) part_a[blockIdx.x] = spq;
    grid.sync();
    double pq, unused;
    grid_totals(part_a, nullptr, nb, red, pq, unused);
    if (!(pq > 0.0)) { breakdown = 1; break; }
    const double alpha = rz / pq;
    // phase 2: x += alpha p ; r -= alpha q ; z = D^-1 r ; partials r.r, r.z
    double srr = 0.0, srz = 0.0;
    for (long long i = tid; i < n; i += nth) {
      x[i] = fma(alpha, pv[i], x[i]);
      const double ri = fma(-alpha, q[i], r[i]);
      r[i] = ri;
      const double zi = dinv[i] * ri;
      z[i] = zi;
      srr = fma(ri, ri, srr);
      srz = fma(ri, zi, srz);
    }
    srr = block_reduce(srr, red);
    if (threadIdx.x == 0) part_b[blockIdx.x] = srr;
    srz = block_reduce(srz, red);
    if (threadIdx.x == 0) part_c[blockIdx.x] = srz;
    grid.sync();
    double rr, rzn;
    grid_totals(part_b, part_c, nb, red, rr, rzn);
    ++its;
    if (sqrt(rr) <= rtol * sqrt(bb) || its >= maxit) break;
    beta = rzn / rz;
    rz = rzn;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->its = its;
    st->its_sum += its;
    if (breakdown) st->breakdown = 1;
    st->done = 1;
    st->bb = bb;
  }
}


#ifdef PMG_HMG_TRACE
// copy the barrier trace (pairs: globaltimer ns, tag) to host memory and reset it; returns the count
extern "C" int pmg_debug_hmg_trace(unsigned long long* out, int cap) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, g_hmg_ntrace, sizeof(int));
  n = n < cap ? n : cap;
  cudaMemcpyFromSymbol(out, g_hmg_trace, sizeof(unsigned long long) * 2 * n);
  const int z = 0;
  cudaMemcpyToSymbol(g_hmg_ntrace, &z, sizeof(int));
  return n;
}
#endif
}  // namespace pmg
