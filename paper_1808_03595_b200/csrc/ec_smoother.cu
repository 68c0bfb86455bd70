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
// One CTA of 256 threads per block; planes and workspace in shared memory (12 n3^2 doubles,
// 212 KB at p = 16, the supported maximum); the 1-D eigenvector matrices are read from the
// L2-resident table.  Runtime degree: this is the NEXT-4 smoother, correctness first.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {
namespace {

constexpr int kEcThreads = 256;

// plane d: slow / fast in-plane directions (same orientation as the star planes)
__device__ __forceinline__ int ec_slow(int d) { return d == 2 ? 1 : 2; }
__device__ __forceinline__ int ec_fast(int d) { return d == 0 ? 1 : 0; }

__global__ void __launch_bounds__(kEcThreads) k_ec_block(LevelGeom g, int c1, int c2, int c3, int n1, int n2,
                                                       const double* __restrict__ r, double* __restrict__ u,
                                                       const double* __restrict__ ectab, double lam) {
  extern __shared__ double sm[];
  const int p = g.p, n = ec_n(p), nn = n * n, ES = ec_table_stride(p);
  const int clo = p - 1, chi = 2 * p - 1;
  const int b = blockIdx.x, i1 = b % n1, rest = b / n1, i2 = rest % n2, i3 = rest / n2;
  const int e[3] = {c1 + 3 * i1, c2 + 3 * i2, c3 + 3 * i3};
  const int tid = threadIdx.x;
  double* F = sm;                  // 6 planes (d, s): index (2d + s) * nn + A * n + B
  double* G = sm + 6 * nn;         // 6 planes workspace
  double* vec = sm + 12 * nn;      // per direction: Lambda, s_lo, s_hi, omega (4n each)
  const double* S[3];
  for (int d = 0; d < 3; ++d) {
    const int row = (d == 0 ? 0 : (d == 1 ? g.k1 : g.k1 + g.k2)) + e[d];
    S[d] = ectab + (size_t)row * ES;
  }
  for (int i = tid; i < 12 * n; i += kEcThreads) {
    const int d = i / (4 * n), o = i - d * 4 * n;
    vec[i] = __ldg(&S[d][nn + o]);
  }
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
      v = __ldg(&r[skel_index(g, g1, g2, g3)]) / (double)np;
    }
    F[i] = v;
  }
  __syncthreads();
  // 2. forward transforms: X = F S_fast (into G), T = S_slow^T X (into F)
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, bb = rr - A * n;
    const double* Sf = S[ec_fast(pl >> 1)];
    const double* Fr = F + pl * nn + A * n;
    double s = 0.0;
    for (int B = 0; B < n; ++B) s = fma(Fr[B], __ldg(&Sf[B * n + bb]), s);
    G[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, a = rr / n, bb = rr - a * n;
    const double* Ss = S[ec_slow(pl >> 1)];
    const double* X = G + pl * nn + bb;
    double s = 0.0;
    for (int A = 0; A < n; ++A) s = fma(__ldg(&Ss[A * n + a]), X[A * n], s);
    F[i] = s;
  }
  __syncthreads();
  // 3. core, one pass per normal direction d: thread owns (a_slow, a_fast), loops over a_d
  const double* Lv[3] = {vec, vec + 4 * n, vec + 8 * n};
  for (int i = tid; i < 3 * nn; i += kEcThreads) {
    const int d = i / nn, rr = i - d * nn, as = rr / n, af = rr - as * n;
    int a[3];
    a[ec_slow(d)] = as;
    a[ec_fast(d)] = af;
    double glo = 0.0, ghi = 0.0;
    for (int ad = 0; ad < n; ++ad) {
      a[d] = ad;
      double E = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int idx = a[ec_slow(q)] * n + a[ec_fast(q)];
        E = fma(Lv[q][n + a[q]], F[(2 * q) * nn + idx], E);
        E = fma(Lv[q][2 * n + a[q]], F[(2 * q + 1) * nn + idx], E);
      }
      const double V = E / (lam + Lv[0][a[0]] + Lv[1][a[1]] + Lv[2][a[2]]);
      glo = fma(Lv[d][n + ad], V, glo);
      ghi = fma(Lv[d][2 * n + ad], V, ghi);
    }
    G[(2 * d) * nn + rr] = glo;
    G[(2 * d + 1) * nn + rr] = ghi;
  }
  __syncthreads();
  // 4. back transforms: X = G S_fast^T (into F), U = S_slow X (into G)
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, a = rr / n, B = rr - a * n;
    const double* Sf = S[ec_fast(pl >> 1)];
    const double* Gr = G + pl * nn + a * n;
    double s = 0.0;
    for (int bb = 0; bb < n; ++bb) s = fma(Gr[bb], __ldg(&Sf[B * n + bb]), s);
    F[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < 6 * nn; i += kEcThreads) {
    const int pl = i / nn, rr = i - pl * nn, A = rr / n, B = rr - A * n;
    const double* Ss = S[ec_slow(pl >> 1)];
    const double* X = F + pl * nn + B;
    double s = 0.0;
    for (int a = 0; a < n; ++a) s = fma(__ldg(&Ss[A * n + a]), X[a * n], s);
    G[i] = s;
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
    const double w = Lv[0][3 * n + j[0]] * Lv[1][3 * n + j[1]] * Lv[2][3 * n + j[2]];
    const long long idx = skel_index(g, g1, g2, g3);
    u[idx] = fma(w, G[i], u[idx]);
  }
}

}  // namespace

size_t ec_smem(int p) {
  const int n = ec_n(p);
  return sizeof(double) * (size_t)(12 * n * n + 12 * n);
}

cudaError_t ec_set_smem_attr(int bytes) {
  return cudaFuncSetAttribute(k_ec_block, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// one colour (c1, c2, c3) in {0,1,2}^3 of the element-centred sweep
void launch_ec(const LevelGeom& g, int c1, int c2, int c3, const double* r, double* u, const double* ectab,
               double lam, cudaStream_t st) {
  const int n1 = (g.k1 - c1 + 2) / 3, n2 = (g.k2 - c2 + 2) / 3, n3 = (g.k3 - c3 + 2) / 3;
  const long long nb = (long long)n1 * n2 * n3;
  if (nb <= 0) return;
  launch_pdl(k_ec_block, dim3((unsigned)nb), dim3(kEcThreads), ec_smem(g.p), st, g, c1, c2, c3, n1, n2, r, u, ectab, lam);
}

}  // namespace pmg
