// Element-centred block smoother (oracle/ecsmoother.py).
//
// For element e the block is the 3 x 3 x 3 element cube centred on it (full overlap);
// after condensation its unknowns lie on the six planes through the faces of the centre element
// (local positions c_lo = p - 1, c_hi = 2p - 1 of the n3 = 3p - 1 block points per direction).
// The block inverse is the fast-diagonalisation inverse of the full block restricted to the
// planes, with six faces instead of the star's three (73 n3^3 operations):
//   1. gather the six planes of r_hat, each point divided by the number of planes through it;
//   2. forward 2-D transforms of every plane (S_slow^T F S_fast);
//   3. core: E(a) = sum over the six planes of S_d[c][a_d] T_{d,c}(other two indices),
//      V = E / (lambda + Lambda_1 + Lambda_2 + Lambda_3), and per plane the contraction
//      G_{d,c} = sum_{a_d} S_d[c][a_d] V (three passes, one per normal direction: each thread
//      owns one (a_slow, a_fast) pair and loops over a_d; fixed order, no atomics);
//   4. back transforms U_{d,c} = S_slow G S_fast^T;
//   5. weighted scatter-add into u_hat (weights of reading R17), each point written once.
// Blocks whose windows overlap may share points, so the sweep runs in 27 colours (element
// indices mod 3 per direction): the points of one colour are disjoint and the read-modify-write
// of u_hat is race-free (the star's 8-colouring argument, A.3, with stride 3).
//
// One CTA of 512 threads per block; planes and workspace in shared memory (12 n3^2 doubles,
// 212 KB at p = 16, the supported maximum); the three 1-D eigenvector matrices are staged in
// shared memory too when they fit (p <= 14), else read from the L2-resident table.  Degree-templated
// (2 <= p <= 16): every loop fully unrolled with compile-time strides.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {
namespace {

constexpr int kEcThreads = 512;

// plane d: slow / fast in-plane directions (same orientation as the star planes)
__device__ __forceinline__ int ec_slow(int d) { return d == 2 ? 1 : 2; }
__device__ __forceinline__ int ec_fast(int d) { return d == 0 ? 1 : 0; }

// 1 / x: MUFU approximation + two Newton steps (the star kernels' reciprocal)
__device__ __forceinline__ double ec_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// sum_k x[k * SX] y[k * SY], k < N, four independent partial sums (k ascending within each)
template <int N, int SX, int SY>
__device__ __forceinline__ double ec_dot(const double* x, const double* y) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < N; ++k) s[k & 3] = fma(x[k * SX], y[k * SY], s[k & 3]);
  return (s[0] + s[1]) + (s[2] + s[3]);
}

template <int P>
__global__ void __launch_bounds__(kEcThreads) k_ec_block(LevelGeom g, int c1, int c2, int c3, int n1, int n2,
                                                       const double* __restrict__ r, double* __restrict__ u,
                                                       const double* __restrict__ ectab, double lam) {
  extern __shared__ double sm[];
  constexpr int p = P, n = 3 * P - 1, nn = n * n, ES = n * n + 4 * n;
  constexpr int clo = p - 1, chi = 2 * p - 1;
  const int b = blockIdx.x, i1 = b % n1, rest = b / n1, i2 = rest % n2, i3 = rest / n2;
  const int e[3] = {c1 + 3 * i1, c2 + 3 * i2, c3 + 3 * i3};
  const int tid = threadIdx.x;
  double* F = sm;                  // 6 planes (d, s): index (2d + s) * nn + A * n + B
  double* G = sm + 6 * nn;         // 6 planes workspace
  double* vec = sm + 12 * nn;      // per direction: Lambda, s_lo, s_hi, omega (4n each)
  double* Ssm = vec + 12 * n;      // S_d staged (STAGE), 3 nn
  const double* S[3];
  for (int d = 0; d < 3; ++d) {
    const int row = (d == 0 ? 0 : (d == 1 ? g.k1 : g.k1 + g.k2)) + e[d];
    S[d] = ectab + (size_t)row * ES;
  }
  for (int i = tid; i < 12 * n; i += kEcThreads) {
    const int d = i / (4 * n), o = i - d * 4 * n;
    vec[i] = __ldg(&S[d][nn + o]);
  }
  // S_d staged in shared memory when the three fit next to the planes (p <= 14): the transforms
  // then address it as Ssm + d nn (shared loads); otherwise straight from the L2-resident table
  constexpr bool STAGE = (15 * nn + 12 * n) * 8 <= 227 * 1024;
  if (STAGE) {
    for (int i = tid; i < 3 * nn; i += kEcThreads) {
      const int d = i / nn;
      Ssm[i] = __ldg(&S[d][i - d * nn]);
    }
  }
  auto Smat = [&](int d) -> const double* { return STAGE ? Ssm + d * nn : S[d]; };
  pdl_wait();
  pdl_trigger();
  // 1. gather
  const int o[3] = {(e[0] - 1) * p + 1, (e[1] - 1) * p + 1, (e[2] - 1) * p + 1};
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, B = rr - A * n, d = pl >> 1;
    int j[3];
    j[d] = (pl & 1) ? chi : clo;
    j[ec_slow(d)] = A;
    j[ec_fast(d)] = B;
    const int g1 = o[0] + j[0], g2 = o[1] + j[1], g3 = o[2] + j[2];
    double v = 0.0;
    if (is_free(g, g1, g2, g3)) {
      const int np = 1 + (A == clo || A == chi) + (B == clo || B == chi);
      v = __ldg(&r[skel_index_t<P>(g, g1, g2, g3)]) / (double)np;
    }
    F[i] = v;
  }
  __syncthreads();
  // 2. forward transforms: X = F S_fast (into G), T = S_slow^T X (into F)
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, bb = rr - A * n;
    G[i] = ec_dot<n, 1, n>(F + pl * nn + A * n, Smat(ec_fast(pl >> 1)) + bb);
  }
  __syncthreads();
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, a = rr / n, bb = rr - a * n;
    F[i] = ec_dot<n, n, n>(Smat(ec_slow(pl >> 1)) + a, G + pl * nn + bb);
  }
  __syncthreads();
  // 3. core, one pass per normal direction d: the thread owns the (a_slow, a_fast) pair of plane d
  //    and loops over a_d.  T_{q,s} is indexed [a_slow(q)][a_fast(q)]:
  //    q = 0: [a3][a2], q = 1: [a3][a1], q = 2: [a2][a1].
  const double *L1 = vec, *L2 = vec + 4 * n, *L3 = vec + 8 * n;   // Lambda, then s_lo at +n, s_hi at +2n
  const double *T0 = F, *T1 = F + nn, *T2 = F + 2 * nn, *T3 = F + 3 * nn, *T4 = F + 4 * nn, *T5 = F + 5 * nn;
  for (int i = tid; i < 3 * nn; i += kEcThreads) {
    const int d = i / nn, rr = i - d * nn, as = rr / n, af = rr - as * n;
    double glo = 0.0, ghi = 0.0;
    if (d == 0) {                  // (a3, a2) fixed, a1 runs
      const int a3 = as, a2 = af;
      const double t0 = T0[a3 * n + a2], t1 = T1[a3 * n + a2];
      const double base = lam + L2[a2] + L3[a3];
      const double c2l = L2[n + a2], c2h = L2[2 * n + a2], c3l = L3[n + a3], c3h = L3[2 * n + a3];
#pragma unroll
      for (int a1 = 0; a1 < n; ++a1) {
        double E = L1[n + a1] * t0;
        E = fma(L1[2 * n + a1], t1, E);
        E = fma(c2l, T2[a3 * n + a1], E);
        E = fma(c2h, T3[a3 * n + a1], E);
        E = fma(c3l, T4[a2 * n + a1], E);
        E = fma(c3h, T5[a2 * n + a1], E);
        const double V = E * ec_rcp(base + L1[a1]);
        glo = fma(L1[n + a1], V, glo);
        ghi = fma(L1[2 * n + a1], V, ghi);
      }
    } else if (d == 1) {           // (a3, a1) fixed, a2 runs
      const int a3 = as, a1 = af;
      const double t2 = T2[a3 * n + a1], t3 = T3[a3 * n + a1];
      const double base = lam + L1[a1] + L3[a3];
      const double c1l = L1[n + a1], c1h = L1[2 * n + a1], c3l = L3[n + a3], c3h = L3[2 * n + a3];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double E = c1l * T0[a3 * n + a2];
        E = fma(c1h, T1[a3 * n + a2], E);
        E = fma(L2[n + a2], t2, E);
        E = fma(L2[2 * n + a2], t3, E);
        E = fma(c3l, T4[a2 * n + a1], E);
        E = fma(c3h, T5[a2 * n + a1], E);
        const double V = E * ec_rcp(base + L2[a2]);
        glo = fma(L2[n + a2], V, glo);
        ghi = fma(L2[2 * n + a2], V, ghi);
      }
    } else {                       // (a2, a1) fixed, a3 runs
      const int a2 = as, a1 = af;
      const double t4 = T4[a2 * n + a1], t5 = T5[a2 * n + a1];
      const double base = lam + L1[a1] + L2[a2];
      const double c1l = L1[n + a1], c1h = L1[2 * n + a1], c2l = L2[n + a2], c2h = L2[2 * n + a2];
#pragma unroll
      for (int a3 = 0; a3 < n; ++a3) {
        double E = c1l * T0[a3 * n + a2];
        E = fma(c1h, T1[a3 * n + a2], E);
        E = fma(c2l, T2[a3 * n + a1], E);
        E = fma(c2h, T3[a3 * n + a1], E);
        E = fma(L3[n + a3], t4, E);
        E = fma(L3[2 * n + a3], t5, E);
        const double V = E * ec_rcp(base + L3[a3]);
        glo = fma(L3[n + a3], V, glo);
        ghi = fma(L3[2 * n + a3], V, ghi);
      }
    }
    G[(2 * d) * nn + rr] = glo;
    G[(2 * d + 1) * nn + rr] = ghi;
  }
  __syncthreads();
  // 4. back transforms: X = G S_fast^T (into F), U = S_slow X (into G)
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, a = rr / n, B = rr - a * n;
    F[i] = ec_dot<n, 1, 1>(G + pl * nn + a * n, Smat(ec_fast(pl >> 1)) + B * n);
  }
  __syncthreads();
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, B = rr - A * n;
    G[i] = ec_dot<n, 1, n>(Smat(ec_slow(pl >> 1)) + A * n, F + pl * nn + B);
  }
  __syncthreads();
  // 5. weighted scatter-add: a point on several planes is written by the lowest (d, s) plane
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, B = rr - A * n, d = pl >> 1;
    int j[3];
    j[d] = (pl & 1) ? chi : clo;
    j[ec_slow(d)] = A;
    j[ec_fast(d)] = B;
    bool dup = false;
    for (int q = 0; q < d; ++q) dup |= (j[q] == clo || j[q] == chi);
    if (dup) continue;
    const int g1 = o[0] + j[0], g2 = o[1] + j[1], g3 = o[2] + j[2];
    if (!is_free(g, g1, g2, g3)) continue;
    const double w = vec[3 * n + j[0]] * vec[7 * n + j[1]] * vec[11 * n + j[2]];
    const long long idx = skel_index_t<P>(g, g1, g2, g3);
    u[idx] = fma(w, G[i], u[idx]);
  }
}

// ------------------------------------------------------------------------------------------
// DMMA variant (p <= 13): the same five steps, the 24 plane transforms per block on the FP64
// tensor cores (mma.sync.m8n8k4.f64: one warp instruction = 256 FMA from two fragment loads, where
// the DFMA transforms need two shared loads per FMA -- the DFMA kernel is shared-memory-bandwidth
// bound).  Planes, workspace and S_d are stored NP x LD (NP = n_S rounded up to 8, LD = NP + 4),
// zero outside n_S x n_S, so the padded products are exact.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void ec_dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// C(8x8 tile mi, ni) = op(A) op(B), NP x NP operands with leading dimension LD; one warp.
// TA: A is read transposed (A[k][i]); TB: B is read transposed (B[j][k]).
template <int NP, int LD, bool TA, bool TB>
__device__ __forceinline__ void ec_tile(const double* A, const double* B, double* C, int mi, int ni, int lane) {
  const int r = lane >> 2, q = lane & 3;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int kk = 0; kk < NP / 4; ++kk) {
    const int i = 8 * mi + r, k = 4 * kk + q, j = 8 * ni + r;
    ec_dmma884(c0, c1, TA ? A[k * LD + i] : A[i * LD + k], TB ? B[j * LD + k] : B[k * LD + j]);
  }
  C[(8 * mi + r) * LD + 8 * ni + 2 * q] = c0;
  C[(8 * mi + r) * LD + 8 * ni + 2 * q + 1] = c1;
}

template <int P> struct EcMmaCfg {
  static constexpr int n = 3 * P - 1, NP = (n + 7) / 8 * 8, LD = NP + 4, PS = NP * LD, TPP = (NP / 8) * (NP / 8);
  static constexpr int total = 15 * PS + 12 * n;   // F (6 planes), G (6), S (3), vectors
};

template <int P>
__global__ void __launch_bounds__(kEcThreads) k_ec_block_mma(LevelGeom g, int c1, int c2, int c3, int n1, int n2,
                                                           const double* __restrict__ r, double* __restrict__ u,
                                                           const double* __restrict__ ectab, double lam) {
  using C = EcMmaCfg<P>;
  extern __shared__ double sm[];
  constexpr int p = P, n = C::n, nn = n * n, NP = C::NP, LD = C::LD, PS = C::PS, ES = n * n + 4 * n;
  constexpr int clo = p - 1, chi = 2 * p - 1, NW = kEcThreads / 32;
  const int b = blockIdx.x, i1 = b % n1, rest = b / n1, i2 = rest % n2, i3 = rest / n2;
  const int e[3] = {c1 + 3 * i1, c2 + 3 * i2, c3 + 3 * i3};
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* F = sm;                  // plane (2d + s) at F + (2d + s) PS, [A][B] at A LD + B
  double* G = sm + 6 * PS;
  double* Ssm = sm + 12 * PS;      // S_d at Ssm + d PS, [j][a]
  double* vec = sm + 15 * PS;      // per direction: Lambda, s_lo, s_hi, omega (4n each)
  const double* Sg[3];
  for (int d = 0; d < 3; ++d) {
    const int row = (d == 0 ? 0 : (d == 1 ? g.k1 : g.k1 + g.k2)) + e[d];
    Sg[d] = ectab + (size_t)row * ES;
  }
  for (int i = tid; i < 12 * n; i += kEcThreads) {
    const int d = i / (4 * n), o = i - d * 4 * n;
    vec[i] = __ldg(&Sg[d][nn + o]);
  }
  for (int i = tid; i < 3 * NP * NP; i += kEcThreads) {
    const int d = i / (NP * NP), rr = i - d * NP * NP, A = rr / NP, B = rr - A * NP;
    Ssm[d * PS + A * LD + B] = (A < n && B < n) ? __ldg(&Sg[d][A * n + B]) : 0.0;
  }
  pdl_wait();
  pdl_trigger();
  // 1. gather (zero padding)
  const int o[3] = {(e[0] - 1) * p + 1, (e[1] - 1) * p + 1, (e[2] - 1) * p + 1};
  for (int i = tid; i < 6 * NP * NP; i += kEcThreads) {
    const int pl = i / (NP * NP), rr = i - pl * NP * NP, A = rr / NP, B = rr - A * NP, d = pl >> 1;
    double v = 0.0;
    if (A < n && B < n) {
      int j[3];
      j[d] = (pl & 1) ? chi : clo;
      j[ec_slow(d)] = A;
      j[ec_fast(d)] = B;
      const int g1 = o[0] + j[0], g2 = o[1] + j[1], g3 = o[2] + j[2];
      if (is_free(g, g1, g2, g3)) {
        const int np = 1 + (A == clo || A == chi) + (B == clo || B == chi);
        v = __ldg(&r[skel_index_t<P>(g, g1, g2, g3)]) / (double)np;
      }
    }
    F[pl * PS + A * LD + B] = v;
  }
  __syncthreads();
  // 2. forward: X = F S_fast (into G), T = S_slow^T X (into F)
  for (int job = warp; job < 6 * C::TPP; job += NW) {
    const int pl = job / C::TPP, t = job - pl * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    ec_tile<NP, LD, false, false>(F + pl * PS, Ssm + ec_fast(pl >> 1) * PS, G + pl * PS, mi, ni, lane);
  }
  __syncthreads();
  for (int job = warp; job < 6 * C::TPP; job += NW) {
    const int pl = job / C::TPP, t = job - pl * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    ec_tile<NP, LD, true, false>(Ssm + ec_slow(pl >> 1) * PS, G + pl * PS, F + pl * PS, mi, ni, lane);
  }
  __syncthreads();
  // 3. core (as k_ec_block; T and G at stride LD; the padding of G stays zero from step 2)
  const double *L1 = vec, *L2 = vec + 4 * n, *L3 = vec + 8 * n;
  const double *T0 = F, *T1 = F + PS, *T2 = F + 2 * PS, *T3 = F + 3 * PS, *T4 = F + 4 * PS, *T5 = F + 5 * PS;
  for (int i = tid; i < 3 * nn; i += kEcThreads) {
    const int d = i / nn, rr = i - d * nn, as = rr / n, af = rr - as * n;
    double glo = 0.0, ghi = 0.0;
    if (d == 0) {
      const int a3 = as, a2 = af;
      const double t0 = T0[a3 * LD + a2], t1 = T1[a3 * LD + a2];
      const double base = lam + L2[a2] + L3[a3];
      const double c2l = L2[n + a2], c2h = L2[2 * n + a2], c3l = L3[n + a3], c3h = L3[2 * n + a3];
#pragma unroll
      for (int a1 = 0; a1 < n; ++a1) {
        double E = L1[n + a1] * t0;
        E = fma(L1[2 * n + a1], t1, E);
        E = fma(c2l, T2[a3 * LD + a1], E);
        E = fma(c2h, T3[a3 * LD + a1], E);
        E = fma(c3l, T4[a2 * LD + a1], E);
        E = fma(c3h, T5[a2 * LD + a1], E);
        const double V = E * ec_rcp(base + L1[a1]);
        glo = fma(L1[n + a1], V, glo);
        ghi = fma(L1[2 * n + a1], V, ghi);
      }
    } else if (d == 1) {
      const int a3 = as, a1 = af;
      const double t2 = T2[a3 * LD + a1], t3 = T3[a3 * LD + a1];
      const double base = lam + L1[a1] + L3[a3];
      const double c1l = L1[n + a1], c1h = L1[2 * n + a1], c3l = L3[n + a3], c3h = L3[2 * n + a3];
#pragma unroll
      for (int a2 = 0; a2 < n; ++a2) {
        double E = c1l * T0[a3 * LD + a2];
        E = fma(c1h, T1[a3 * LD + a2], E);
        E = fma(L2[n + a2], t2, E);
        E = fma(L2[2 * n + a2], t3, E);
        E = fma(c3l, T4[a2 * LD + a1], E);
        E = fma(c3h, T5[a2 * LD + a1], E);
        const double V = E * ec_rcp(base + L2[a2]);
        glo = fma(L2[n + a2], V, glo);
        ghi = fma(L2[2 * n + a2], V, ghi);
      }
    } else {
      const int a2 = as, a1 = af;
      const double t4 = T4[a2 * LD + a1], t5 = T5[a2 * LD + a1];
      const double base = lam + L1[a1] + L2[a2];
      const double c1l = L1[n + a1], c1h = L1[2 * n + a1], c2l = L2[n + a2], c2h = L2[2 * n + a2];
#pragma unroll
      for (int a3 = 0; a3 < n; ++a3) {
        double E = c1l * T0[a3 * LD + a2];
        E = fma(c1h, T1[a3 * LD + a2], E);
        E = fma(c2l, T2[a3 * LD + a1], E);
        E = fma(c2h, T3[a3 * LD + a1], E);
        E = fma(L3[n + a3], t4, E);
        E = fma(L3[2 * n + a3], t5, E);
        const double V = E * ec_rcp(base + L3[a3]);
        glo = fma(L3[n + a3], V, glo);
        ghi = fma(L3[2 * n + a3], V, ghi);
      }
    }
    G[(2 * d) * PS + as * LD + af] = glo;
    G[(2 * d + 1) * PS + as * LD + af] = ghi;
  }
  __syncthreads();
  // 4. back: X = G S_fast^T (into F), U = S_slow X (into G)
  for (int job = warp; job < 6 * C::TPP; job += NW) {
    const int pl = job / C::TPP, t = job - pl * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    ec_tile<NP, LD, false, true>(G + pl * PS, Ssm + ec_fast(pl >> 1) * PS, F + pl * PS, mi, ni, lane);
  }
  __syncthreads();
  for (int job = warp; job < 6 * C::TPP; job += NW) {
    const int pl = job / C::TPP, t = job - pl * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    ec_tile<NP, LD, false, false>(Ssm + ec_slow(pl >> 1) * PS, F + pl * PS, G + pl * PS, mi, ni, lane);
  }
  __syncthreads();
  // 5. weighted scatter-add (each point once, from its lowest plane)
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, B = rr - A * n, d = pl >> 1;
    int j[3];
    j[d] = (pl & 1) ? chi : clo;
    j[ec_slow(d)] = A;
    j[ec_fast(d)] = B;
    bool dup = false;
    for (int q = 0; q < d; ++q) dup |= (j[q] == clo || j[q] == chi);
    if (dup) continue;
    const int g1 = o[0] + j[0], g2 = o[1] + j[1], g3 = o[2] + j[2];
    if (!is_free(g, g1, g2, g3)) continue;
    const double w = vec[3 * n + j[0]] * vec[7 * n + j[1]] * vec[11 * n + j[2]];
    const long long idx = skel_index_t<P>(g, g1, g2, g3);
    u[idx] = fma(w, G[pl * PS + A * LD + B], u[idx]);
  }
}

}  // namespace

size_t ec_smem(int p) {   // planes + workspace + vectors (the minimum; S staged when it fits)
  const int n = ec_n(p);
  return sizeof(double) * (size_t)(12 * n * n + 12 * n);
}


#define PMG_EC_DEGREES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
#define PMG_EC_MMA_DEGREES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13)

// PMG_EC_VARIANT=dfma forces the DFMA kernel at every degree (A/B and parity of the two variants)
static bool ec_use_mma(int p) {
  const char* v = std::getenv("PMG_EC_VARIANT");
  return p <= 13 && !(v && v[0] == 'd');
}

cudaError_t ec_set_smem_attr(int bytes) {
  cudaError_t e = cudaSuccess, a;
#define PMG_EC_ATTR(P) \
  a = cudaFuncSetAttribute(k_ec_block<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
  if (a != cudaSuccess) e = a;
  PMG_EC_DEGREES(PMG_EC_ATTR)
#undef PMG_EC_ATTR
#define PMG_EC_MMA_ATTR(P) \
  a = cudaFuncSetAttribute(k_ec_block_mma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
  if (a != cudaSuccess) e = a;
  PMG_EC_MMA_DEGREES(PMG_EC_MMA_ATTR)
#undef PMG_EC_MMA_ATTR
  return e;
}

// one colour (c1, c2, c3) in {0,1,2}^3 of the element-centred sweep
void launch_ec(const LevelGeom& g, int c1, int c2, int c3, const double* r, double* u, const double* ectab,
               double lam, cudaStream_t st) {
  const int n1 = (g.k1 - c1 + 2) / 3, n2 = (g.k2 - c2 + 2) / 3, n3 = (g.k3 - c3 + 2) / 3;
  const long long nb = (long long)n1 * n2 * n3;
  if (nb <= 0) return;
  if (ec_use_mma(g.p)) {
    switch (g.p) {
#define PMG_EC_MMA_CASE(P) \
  case P: \
    launch_pdl(k_ec_block_mma<P>, dim3((unsigned)nb), dim3(kEcThreads), sizeof(double) * (size_t)EcMmaCfg<P>::total, st, g, \
               c1, c2, c3, n1, n2, r, u, ectab, lam); \
    return;
      PMG_EC_MMA_DEGREES(PMG_EC_MMA_CASE)
#undef PMG_EC_MMA_CASE
      default: break;
    }
  }
  const int n = ec_n(g.p);
  const bool stage = (15 * n * n + 12 * n) * 8 <= 227 * 1024;   // as the kernel's STAGE (p <= 14)
  const size_t smem = ec_smem(g.p) + (stage ? sizeof(double) * (size_t)(3 * n * n) : 0);
  switch (g.p) {
#define PMG_EC_CASE(P) \
  case P: \
    launch_pdl(k_ec_block<P>, dim3((unsigned)nb), dim3(kEcThreads), smem, st, g, c1, c2, c3, n1, n2, r, u, ectab, lam); \
    break;
    PMG_EC_DEGREES(PMG_EC_CASE)
#undef PMG_EC_CASE
    default: break;
  }
}

}  // namespace pmg
