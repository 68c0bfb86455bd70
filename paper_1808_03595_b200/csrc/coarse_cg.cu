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
// oracle/hmg.py): one cooperative launch; every step of the V-cycle is a grid-stride loop over the
// level's unknowns followed by a grid barrier; the coarsest level (a few hundred unknowns) is
// smoothed by block 0 alone with block barriers.  Damped Jacobi (omega = 0.6), two sweeps before and
// after the coarse correction, 40 sweeps on the coarsest level -- the oracle's constants.
// ------------------------------------------------------------------------------------------
namespace {
constexpr double kHmgOmega = 0.6;
constexpr int kHmgNu = 2, kHmgCoarsest = 40;

__device__ __forceinline__ double ell_row(const double* __restrict__ val, const int* __restrict__ col, long long n,
                                          long long i, const double* __restrict__ v) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kRowLen; ++k) s = fma(__ldg(&val[k * n + i]), __ldcg(&v[__ldg(&col[k * n + i])]), s);
  return s;
}

// one CSR row reduced by a whole warp: lane j takes entries j, j + 32, ... in order, then a fixed
// xor tree (deterministic); every lane returns the row value.  The transfer rows are up to ~125
// long (restriction), too long for one thread's dependent load chain.
__device__ __forceinline__ double csr_row_warp(const int* __restrict__ ptr, const int* __restrict__ col,
                                               const double* __restrict__ val, long long i,
                                               const double* __restrict__ v, int lane) {
  double s = 0.0;
  const int k1 = __ldg(&ptr[i + 1]);
  for (int k = __ldg(&ptr[i]) + lane; k < k1; k += 32) s = fma(__ldg(&val[k]), __ldcg(&v[__ldg(&col[k])]), s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// one CSR row by one thread (the prolongation rows: at most 26 entries, one coarse element's
// skeleton; a warp per row would leave most lanes idle and serialise the rows)
__device__ __forceinline__ double csr_row_thread(const int* __restrict__ ptr, const int* __restrict__ col,
                                                 const double* __restrict__ val, long long i,
                                                 const double* __restrict__ v) {
  double s = 0.0;
  const int k1 = __ldg(&ptr[i + 1]);
  for (int k = __ldg(&ptr[i]); k < k1; ++k) s = fma(__ldg(&val[k]), __ldcg(&v[__ldg(&col[k])]), s);
  return s;
}

// z = V-cycle(f_0) into h.x[0]; h.f[0] holds the right-hand side.  With rz_part set, the block's
// partial of f_0 . z (the CG's r.z) is formed in the last level-0 sweep and published before the
// V-cycle's final barrier, which then doubles as the CG's reduction barrier.
__device__ void hmg_vcycle(const HmgDev& h, cg::grid_group& grid, long long t0, long long T,
                           double* red = nullptr, double* rz_part = nullptr) {
  const int L = h.nlev - 1;
  for (int l = 0; l < L; ++l) {
    const long long n = h.n[l];
    double *x = h.x[l], *r = h.r[l];
    const double *f = h.f[l], *di = h.dinv[l];
    // the two pre-sweeps from zero in one pass: x1 = omega D^-1 f is local, so
    // x2_i = x1_i + omega d_i (f_i - sum_j A_ij x1_j) gathers omega d_j f_j directly
    static_assert(kHmgNu == 2, "the fused sweeps below are written for nu = 2");
    for (long long i = t0; i < n; i += T) {
      const double* val = h.Aval[l];
      const int* col = h.Acol[l];
      double ax = 0.0;
#pragma unroll
      for (int k = 0; k < kRowLen; ++k) {
        const int j = __ldg(&col[k * n + i]);
        ax = fma(__ldg(&val[k * n + i]), kHmgOmega * __ldg(&di[j]) * __ldcg(&f[j]), ax);
      }
      const double x1 = kHmgOmega * di[i] * f[i];
      x[i] = fma(kHmgOmega * di[i], f[i] - ax, x1);
    }
    grid.sync();
    for (long long i = t0; i < n; i += T) r[i] = f[i] - ell_row(h.Aval[l], h.Acol[l], n, i, x);
    grid.sync();
    const long long nc = h.n[l + 1];
    for (long long i = t0 >> 5; i < nc; i += T >> 5) {
      const double v = csr_row_warp(h.Rptr[l], h.Rcol[l], h.Rval[l], i, r, (int)(t0 & 31));
      if ((t0 & 31) == 0) h.f[l + 1][i] = v;
    }
    grid.sync();
  }
  if (h.ncf > 0) {                       // coarsest level: x = A^-1 f (dense inverse, warp per row)
    const int lane = (int)(t0 & 31);
    for (long long i = t0 >> 5; i < h.ncf; i += T >> 5) {
      const double* row = h.cinv + i * (long long)h.ncf;
      double s = 0.0;
      for (int j = lane; j < h.ncf; j += 32) s = fma(__ldg(&row[j]), __ldcg(&h.f[L][__ldg(&h.cidx[j])]), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) h.x[L][__ldg(&h.cidx[i])] = s;
    }
  } else if (blockIdx.x == 0) {          // large coarsest level: block 0, Jacobi sweeps, block barriers
    const long long n = h.n[L];
    double *x = h.x[L], *r = h.r[L];
    const double *f = h.f[L], *di = h.dinv[L];
    for (long long i = threadIdx.x; i < n; i += blockDim.x) x[i] = kHmgOmega * di[i] * f[i];
    __syncthreads();
    for (int s = 1; s < kHmgCoarsest; ++s) {
      for (long long i = threadIdx.x; i < n; i += blockDim.x) r[i] = f[i] - ell_row(h.Aval[L], h.Acol[L], n, i, x);
      __syncthreads();
      for (long long i = threadIdx.x; i < n; i += blockDim.x) x[i] = fma(kHmgOmega * di[i], r[i], x[i]);
      __syncthreads();
    }
  }
  grid.sync();
  for (int l = L - 1; l >= 0; --l) {
    const long long n = h.n[l];
    double *x = h.x[l], *r = h.r[l];
    const double *f = h.f[l], *di = h.dinv[l];
    for (long long i = t0; i < n; i += T) x[i] += csr_row_thread(h.Pptr[l], h.Pcol[l], h.Pval[l], i, h.x[l + 1]);
    grid.sync();
    // two post-sweeps, each one pass, ping-pong x -> r -> x (r is free here)
    for (long long i = t0; i < n; i += T) r[i] = fma(kHmgOmega * di[i], f[i] - ell_row(h.Aval[l], h.Acol[l], n, i, x), x[i]);
    grid.sync();
    double srz = 0.0;
    for (long long i = t0; i < n; i += T) {
      const double xi = fma(kHmgOmega * di[i], f[i] - ell_row(h.Aval[l], h.Acol[l], n, i, r), r[i]);
      x[i] = xi;
      srz = fma(f[i], xi, srz);
    }
    if (l == 0 && rz_part) block_reduce3(srz, srz, srz, red, blockIdx.x, rz_part, rz_part, rz_part);
    grid.sync();
  }
  if (L == 0 && rz_part) {   // a single h-level (the dense solve alone): r.z after it
    const long long n = h.n[0];
    double srz = 0.0;
    for (long long i = t0; i < n; i += T) srz = fma(h.f[0][i], __ldcg(&h.x[0][i]), srz);
    block_reduce3(srz, srz, srz, red, blockIdx.x, rz_part, rz_part, rz_part);
    grid.sync();
  }
}
}  // namespace

// Standard PCG (as mg.pcg / hmg.pcg_hmg): x = 0, r = b, z = M^-1 r, p = z; q = A p, alpha = r.z / p.q,
// x += alpha p, r -= alpha q, stop at ||r|| <= rtol ||b||, z = M^-1 r, beta = r.z_new / r.z, p = z + beta p.
// r lives in h.f[0] (the V-cycle's right-hand side), z in h.x[0].
__global__ void __launch_bounds__(256) k_pcg_hmg_p2(HmgDev h, const double* __restrict__ b, double* __restrict__ xout,
                                                   double* __restrict__ pv, double* __restrict__ q,
                                                   double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  const int nb = gridDim.x;
  const long long n = h.n[0];
  const long long T = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double* R = h.f[0];
  double* Z = h.x[0];
  double *pa = part, *pb = part + nb, *pc = part + 2 * nb;
  double sb = 0.0;
  for (long long i = t0; i < n; i += T) {
    const double bi = b[i];
    xout[i] = 0.0;
    R[i] = bi;
    sb = fma(bi, bi, sb);
  }
  block_reduce3(sb, 0.0, 0.0, red, blockIdx.x, pa, pb, pc);
  grid.sync();
  double bb, d1, d2;
  grid_totals3(pa, pb, pc, nb, red, bb, d1, d2);
  int its = 0, breakdown = 0;
  if (bb > 0.0) {
    // partial sums: p.q in pa, r.r in pb, r.z in pc -- consecutive reductions use different
    // buffers, so a block that runs ahead never overwrites a partial another block still reads.
    // Two grid barriers per iteration besides the V-cycle's: with p_new = z + beta p,
    // q_new = H z + beta q_old, so the direction, the operator application (z is complete after
    // the V-cycle) and p.q share one phase; r.z is reduced inside the V-cycle's last sweep
    hmg_vcycle(h, grid, t0, T, red, pc);
    double rz, pq;
    grid_totals3(pc, pc, pc, nb, red, rz, d1, d2);
    {
      double spq = 0.0;
      for (long long i = t0; i < n; i += T) {
        const double zi = Z[i];
        const double qi = ell_row(h.Aval[0], h.Acol[0], n, i, Z);
        pv[i] = zi;
        q[i] = qi;
        spq = fma(zi, qi, spq);
      }
      block_reduce3(spq, spq, spq, red, blockIdx.x, pa, pa, pa);
      grid.sync();
      grid_totals3(pa, pa, pa, nb, red, pq, d1, d2);
    }
    for (;;) {
      if (!(pq > 0.0)) { breakdown = 1; break; }
      const double alpha = rz / pq;
      double srr = 0.0;
      for (long long i = t0; i < n; i += T) {
        xout[i] = fma(alpha, pv[i], xout[i]);
        const double ri = fma(-alpha, q[i], R[i]);
        R[i] = ri;
        srr = fma(ri, ri, srr);
      }
      block_reduce3(srr, srr, srr, red, blockIdx.x, pb, pb, pb);
      grid.sync();
      double rr;
      grid_totals3(pb, pb, pb, nb, red, rr, d1, d2);
      ++its;
      if (sqrt(rr) <= rtol * sqrt(bb) || its >= maxit) break;
      hmg_vcycle(h, grid, t0, T, red, pc);
      double rzn;
      grid_totals3(pc, pc, pc, nb, red, rzn, d1, d2);
      const double beta = rzn / rz;
      rz = rzn;
      double spq = 0.0;
      for (long long i = t0; i < n; i += T) {
        const double pvi = fma(beta, pv[i], Z[i]);
        const double qi = fma(beta, q[i], ell_row(h.Aval[0], h.Acol[0], n, i, Z));
        pv[i] = pvi;
        q[i] = qi;
        spq = fma(pvi, qi, spq);
      }
      block_reduce3(spq, spq, spq, red, blockIdx.x, pa, pa, pa);
      grid.sync();
      grid_totals3(pa, pa, pa, nb, red, pq, d1, d2);
    }
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

}  // namespace pmg
