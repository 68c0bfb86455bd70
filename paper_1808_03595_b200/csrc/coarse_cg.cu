// Coarse-grid solver (reading R11): Jacobi-preconditioned CG on the condensed p0 = 2
// system, as ONE persistent cooperative kernel (grid-wide barriers between the phases of an
// iteration).  The coarse solve is latency bound: a multi-kernel CG spends
// ~10 launches per iteration; here the whole solve is one launch.
//
// Every block reduces the per-block partial sums itself in a fixed order, so all blocks take the
// same (bitwise identical) decisions on alpha, beta and convergence without another barrier,
// and the result is deterministic.  The iteration and stopping rule are those of the oracle's
// pcg(): x = 0, r = b, z = D^-1 r, p = z; per iteration q = H p, alpha = r.z / p.q,
// x += alpha p, r -= alpha q, stop when ||r|| <= rtol ||b||, z = D^-1 r, beta = r.z_new / r.z,
// p = z + beta p.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace cg = cooperative_groups;

namespace pmg {

// y_e = H_hat_e u_B for one p = 2 element (26 boundary values, compact element-output order of
// k_elem_apply): H_BB u_B = (H_e u~)_B with u~ = u_B extended by a zero interior, minus the face
// corrections C_f = P_b P_a a_f V, V = (sum_f a_f P_b P_a u_f) / (lam + L1 + L2 + L3).
__device__ void elem_apply_p2(const LevelGeom& g, long long e, const double* __restrict__ u,
                              const double* __restrict__ etab, double lam, double* __restrict__ Ye) {
  const int p = 2, ET = g.ET;
  const int e1 = (int)(e % g.k1), e2 = (int)((e / g.k1) % g.k2), e3 = (int)(e / ((long long)g.k1 * g.k2));
  const double* T[3] = {etab + (size_t)e1 * ET, etab + (size_t)(g.k1 + e2) * ET, etab + (size_t)(g.k1 + g.k2 + e3) * ET};
  double c[27];
#pragma unroll
  for (int t3 = 0; t3 < 3; ++t3)
#pragma unroll
    for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
      for (int t1 = 0; t1 < 3; ++t1) {
        const int i = (t3 * 3 + t2) * 3 + t1;
        if (t1 == 1 && t2 == 1 && t3 == 1) { c[i] = 0.0; continue; }
        c[i] = __ldcg(&u[skel_index(g, e1 * p + t1, e2 * p + t2, e3 * p + t3)]);   // u changes in-kernel: L2 path
      }
  double M[3][3], K[3][9];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int i = 0; i < 3; ++i) M[d][i] = __ldg(&T[d][et_M(p) + i]);
#pragma unroll
    for (int i = 0; i < 9; ++i) K[d][i] = __ldg(&T[d][et_K(p) + i]);
  }
  // face corrections (m = 1): T_f = P_b P_a u_f ; E = sum a_f T_f ; V = E / D
  double Pd[3], a0[3], a1[3], Ld[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    Pd[d] = __ldg(&T[d][et_P(p)]);
    a0[d] = __ldg(&T[d][et_a0(p)]);
    a1[d] = __ldg(&T[d][et_a1(p)]);
    Ld[d] = __ldg(&T[d][et_lam(p)]);
  }
  // face centre values: x1 faces (t1 = 0, 2; t2 = t3 = 1), x2 faces, x3 faces
  const double uf[6] = {c[(1 * 3 + 1) * 3 + 0], c[(1 * 3 + 1) * 3 + 2], c[(1 * 3 + 0) * 3 + 1],
                        c[(1 * 3 + 2) * 3 + 1], c[(0 * 3 + 1) * 3 + 1], c[(2 * 3 + 1) * 3 + 1]};
  const double PbPa[3] = {Pd[2] * Pd[1], Pd[2] * Pd[0], Pd[1] * Pd[0]};
  double E = 0.0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int d = f >> 1;
    E += ((f & 1) ? a1[d] : a0[d]) * PbPa[d] * uf[f];
  }
  const double V = E / (lam + Ld[0] + Ld[1] + Ld[2]);
  // outputs in the compact order: faces (6), edges (12), vertices (8)
  auto Hu = [&](int t1, int t2, int t3) -> double {
    double y = lam * M[0][t1] * M[1][t2] * M[2][t3] * c[(t3 * 3 + t2) * 3 + t1];
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      s1 += K[0][t1 * 3 + s] * c[(t3 * 3 + t2) * 3 + s];
      s2 += K[1][t2 * 3 + s] * c[(t3 * 3 + s) * 3 + t1];
      s3 += K[2][t3 * 3 + s] * c[(s * 3 + t2) * 3 + t1];
    }
    return y + M[1][t2] * M[2][t3] * s1 + M[0][t1] * M[2][t3] * s2 + M[0][t1] * M[1][t2] * s3;
  };
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int d = f >> 1, s = (f & 1) * 2;
    int t1 = 1, t2 = 1, t3 = 1;
    if (d == 0) t1 = s; else if (d == 1) t2 = s; else t3 = s;
    Ye[f] = Hu(t1, t2, t3) - ((f & 1) ? a1[d] : a0[d]) * PbPa[d] * V;
  }
#pragma unroll
  for (int qe = 0; qe < 12; ++qe) {
    const int d = qe >> 2, sA = (qe & 1) * 2, sB = ((qe >> 1) & 1) * 2;
    int t1, t2, t3;
    if (d == 0) { t1 = 1; t2 = sA; t3 = sB; } else if (d == 1) { t2 = 1; t1 = sA; t3 = sB; } else { t3 = 1; t1 = sA; t2 = sB; }
    Ye[6 + qe] = Hu(t1, t2, t3);
  }
#pragma unroll
  for (int qv = 0; qv < 8; ++qv) Ye[18 + qv] = Hu((qv & 1) * 2, ((qv >> 1) & 1) * 2, ((qv >> 2) & 1) * 2);
}

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

// total of the per-block partials, identical in every block (fixed order: lane-strided sums, then a
// shuffle tree), broadcast to all threads of the block
__device__ __forceinline__ double grid_total(const double* part, int nb, double* bcast) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) s += __ldcg(&part[i]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *bcast = s;
  }
  __syncthreads();
  double t = *bcast;
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) k_pcg_coop_p2(LevelGeom g, const double* __restrict__ b, double* __restrict__ x,
                                                    double* __restrict__ r, double* __restrict__ z, double* __restrict__ pv,
                                                    double* __restrict__ q, const double* __restrict__ dinv,
                                                    const double* __restrict__ etab, double lam, double* __restrict__ Y,
                                                    double* __restrict__ part, PcgState* st, double rtol, int maxit) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  __shared__ double bc;
  const int nb = gridDim.x;
  double* part_a = part;           // p.q, then r.z at init
  double* part_b = part + nb;      // r.r, then b.b at init
  double* part_c = part + 2 * nb;  // r.z
  const long long n = g.nskel;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  // init
  double s1 = 0.0, s2 = 0.0;
  for (long long i = tid; i < n; i += nth) {
    const double bi = b[i], zi = dinv[i] * bi;
    x[i] = 0.0; r[i] = bi; z[i] = zi; pv[i] = zi;
    s1 += bi * zi; s2 += bi * bi;
  }
  s1 = block_reduce(s1, red);
  if (threadIdx.x == 0) part_a[blockIdx.x] = s1;
  s2 = block_reduce(s2, red);
  if (threadIdx.x == 0) part_b[blockIdx.x] = s2;
  grid.sync();
  double rz = grid_total(part_a, nb, &bc);
  const double bb = grid_total(part_b, nb, &bc);
  int its = 0, breakdown = 0;
  bool done = (bb == 0.0);
  grid.sync();   // everyone has read the partials before they are overwritten
  while (!done) {
    // q = H p : element phase
    for (long long e = tid; e < g.nelem; e += nth) elem_apply_p2(g, e, pv, etab, lam, Y + e * g.YS);
    grid.sync();
    // gather phase + partial p.q
    double spq = 0.0;
    {
      const int m = 1, mm = 1, YS = g.YS;
      for (long long idx = tid; idx < n; idx += nth) {
        Entry E = decode_entry(g, idx);
        double s = 0.0;
        if (is_free(g, E.g1, E.g2, E.g3)) {
          auto el = [&](int a1, int a2, int a3) -> size_t {
            return ((size_t)a1 + (size_t)g.k1 * ((size_t)a2 + (size_t)g.k2 * a3)) * YS;
          };
          if (E.type < 3) {
            const int d = E.type;
            int w1 = E.v1, w2 = E.v2, w3 = E.v3;
            if (d == 0) w1 -= 1; else if (d == 1) w2 -= 1; else w3 -= 1;
            s = __ldcg(&Y[el(w1, w2, w3) + (2 * d + 1) * mm]) + __ldcg(&Y[el(E.v1, E.v2, E.v3) + (2 * d) * mm]);
          } else if (E.type < 6) {
            const int d = E.type - 3;
            for (int bB = 0; bB < 2; ++bB)
              for (int bA = 0; bA < 2; ++bA) {
                int a1 = E.v1, a2 = E.v2, a3 = E.v3;
                if (d == 0) { a2 += bA - 1; a3 += bB - 1; } else if (d == 1) { a1 += bA - 1; a3 += bB - 1; }
                else { a1 += bA - 1; a2 += bB - 1; }
                s += __ldcg(&Y[el(a1, a2, a3) + 6 * mm + (4 * d + (1 - bA) + 2 * (1 - bB)) * m]);
              }
          } else {
            for (int c3 = 0; c3 < 2; ++c3)
              for (int c2 = 0; c2 < 2; ++c2)
                for (int c1 = 0; c1 < 2; ++c1)
                  s += __ldcg(&Y[el(E.v1 - 1 + c1, E.v2 - 1 + c2, E.v3 - 1 + c3) + 6 * mm + 12 * m +
                                 (1 - c1) + 2 * (1 - c2) + 4 * (1 - c3)]);
          }
        }
        q[idx] = s;
        spq += pv[idx] * s;
      }
    }
    spq = block_reduce(spq, red);
    if (threadIdx.x == 0) part_a[blockIdx.x] = spq;
    grid.sync();
    const double pq = grid_total(part_a, nb, &bc);
    if (!(pq > 0.0)) { breakdown = 1; break; }
    const double alpha = rz / pq;
    // x += alpha p ; r -= alpha q ; z = D^-1 r ; partials r.r and r.z
    double srr = 0.0, srz = 0.0;
    for (long long i = tid; i < n; i += nth) {
      x[i] += alpha * pv[i];
      const double ri = r[i] - alpha * q[i];
      r[i] = ri;
      const double zi = dinv[i] * ri;
      z[i] = zi;
      srr += ri * ri;
      srz += ri * zi;
    }
    srr = block_reduce(srr, red);
    if (threadIdx.x == 0) part_b[blockIdx.x] = srr;
    srz = block_reduce(srz, red);
    if (threadIdx.x == 0) part_c[blockIdx.x] = srz;
    grid.sync();
    const double rr = grid_total(part_b, nb, &bc);
    const double rzn = grid_total(part_c, nb, &bc);
    ++its;
    if (sqrt(rr) <= rtol * sqrt(bb) || its >= maxit) break;
    const double beta = rzn / rz;
    rz = rzn;
    for (long long i = tid; i < n; i += nth) pv[i] = z[i] + beta * pv[i];
    grid.sync();
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
