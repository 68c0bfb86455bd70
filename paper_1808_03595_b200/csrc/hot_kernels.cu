// Degree-specialised hot kernels (template on p): the condensed element operator and the star
// smoother.  Same arithmetic as the runtime-p reference kernels in kernels.cu (and the same
// citations: P:117-123 / reading R1 for the element operator; Alg. 1 + Alg. 2, for the
// star), re-organised for throughput:
//   - all six faces (three star planes) advance through each transform step together, so a
//     CTA synchronises 6 times per element / star instead of ~20;
//   - transform operands are laid out so that one operand is a warp broadcast and the other is
//     read by consecutive lanes (conflict-free shared memory);
//   - 1/D = 1/(lambda + L1 + L2 + L3) via rcp.approx + two Newton steps (no IEEE division slow path);
//   - block size chosen per degree so small-p elements do not leave most threads idle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {

// 1/x by rcp.approx and one cubic Newton step r (1 + e + e^2), e = 1 - x r (error e^3)
__device__ __forceinline__ double rcp_c3(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// FP64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row) B(4x8, col); lane l holds A[l/4][l%4],
// B[l%4][l/4] and D[l/4][2(l%4) + {0,1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// C = A * B for NP x NP row-major shared-memory matrices (leading dimension LD); one warp, tile (mi, ni)
template <int NP, int LD>
__device__ __forceinline__ void dmma_tile(const double* A, const double* B, double* Cm, int mi, int ni, int lane) {
  const int r = lane >> 2, q = lane & 3;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int kk = 0; kk < NP / 4; ++kk) dmma884(c0, c1, A[(8 * mi + r) * LD + 4 * kk + q], B[(4 * kk + q) * LD + 8 * ni + r]);
  Cm[(8 * mi + r) * LD + 8 * ni + 2 * q] = c0;
  Cm[(8 * mi + r) * LD + 8 * ni + 2 * q + 1] = c1;
}

template <int P> struct ElemCfg {
  static constexpr int M = P - 1, Q = P + 1, MM = M * M, QQ = Q * Q;
  static constexpr int NT = (P <= 4) ? 64 : (P <= 10 ? 128 : 256);
  // shared layout (doubles)
  // X aliases G in the forward transform and T in the back transform (G/T are dead there)
  static constexpr int oUc = 0, oT = oUc + 6 * QQ, oG = oT + 6 * MM;
  static constexpr int oTab = oG + 6 * MM;
  // per-direction table block: Lam[M], P[M][M], Pt[M][M], a0[M], a1[M], Mq[Q], K[Q][Q]
  static constexpr int tLam = 0, tP = M, tPt = M + MM, ta0 = M + 2 * MM, ta1 = 2 * M + 2 * MM,
                       tM = 3 * M + 2 * MM, tK = 3 * M + 2 * MM + Q, TB = 3 * M + 2 * MM + Q + QQ;
  static constexpr int total = oTab + 3 * TB;
};

template <int P>
size_t elem_t_smem() { return sizeof(double) * ElemCfg<P>::total; }

template <int P>
__device__ __forceinline__ double getUc(const double* Uc, int t1, int t2, int t3) {
  constexpr int Q = P + 1, QQ = Q * Q;
  if (t1 == 0 || t1 == P) return Uc[((t1 == P) ? 1 : 0) * QQ + t3 * Q + t2];
  if (t2 == 0 || t2 == P) return Uc[(2 + ((t2 == P) ? 1 : 0)) * QQ + t3 * Q + t1];
  return Uc[(4 + ((t3 == P) ? 1 : 0)) * QQ + t2 * Q + t1];
}

template <int P>
__global__ void __launch_bounds__(ElemCfg<P>::NT) k_elem_apply_t(LevelGeom g, const double* __restrict__ u,
                                                                 const double* __restrict__ etab, double lam,
                                                                 double* __restrict__ Y, const int* __restrict__ done) {
  pdl_wait();
  pdl_trigger();
  using C = ElemCfg<P>;
  constexpr int M = C::M, Q = C::Q, MM = C::MM, QQ = C::QQ, NT = C::NT, TB = C::TB;
  if (done && *done) return;
  extern __shared__ double sm[];
  double* Uc = sm + C::oUc;
  double* T = sm + C::oT;
  double* G = sm + C::oG;
  double* tb = sm + C::oTab;
  const long long e = blockIdx.x;
  const int e1 = (int)(e % g.k1), e2 = (int)((e / g.k1) % g.k2), e3 = (int)(e / ((long long)g.k1 * g.k2));
  const int tid = threadIdx.x;
  const int ET = g.ET;
  // tables: rebuild the per-direction block [Lam, P, Pt, a0, a1, M, K] from the global layout
  {
    const double* src[3] = {etab + (size_t)e1 * ET, etab + (size_t)(g.k1 + e2) * ET, etab + (size_t)(g.k1 + g.k2 + e3) * ET};
    for (int i = tid; i < 3 * TB; i += NT) {
      const int d = i / TB, o = i - d * TB;
      const double* s = src[d];
      double v;
      if (o < C::tP) v = s[et_lam(P) + o];
      else if (o < C::tPt) v = s[et_P(P) + (o - C::tP)];
      else if (o < C::ta0) { int r = o - C::tPt, ia = r / M, b = r - ia * M; v = s[et_P(P) + b * M + ia]; }
      else if (o < C::ta1) v = s[et_a0(P) + (o - C::ta0)];
      else if (o < C::tM) v = s[et_a1(P) + (o - C::ta1)];
      else if (o < C::tK) v = s[et_M(P) + (o - C::tM)];
      else v = s[et_K(P) + (o - C::tK)];
      tb[i] = v;
    }
  }
  for (int i = tid; i < 6 * QQ; i += NT) {
    const int f = i / QQ, r = i - f * QQ, A = r / Q, B = r - A * Q, d = f >> 1, s = f & 1;
    int t1, t2, t3;
    if (d == 0) { t1 = s * P; t3 = A; t2 = B; }
    else if (d == 1) { t2 = s * P; t3 = A; t1 = B; }
    else { t3 = s * P; t2 = A; t1 = B; }
    int G1 = e1 * P + t1, G2 = e2 * P + t2, G3 = e3 * P + t3;
    wrap_pt(g, G1, G2, G3);   // periodic: the last element's high faces are plane 0
    Uc[i] = __ldg(&u[skel_index_t<P>(g, G1, G2, G3)]);
  }
  __syncthreads();
  // tangential directions of face f: a (fast) = x2 for d = 0 else x1; b (slow) = x3 for d < 2 else x2
  // forward A: X_f[ib][ba] = sum_ia U_f[ib][ia] Pt_a[ia][ba]   (X in G's space)
  double* X = G;
  for (int i = tid; i < 6 * MM; i += NT) {
    const int f = i / MM, r = i - f * MM, ib = r / M, ba = r - ib * M, d = f >> 1, da = (d == 0) ? 1 : 0;
    const double* U = Uc + f * QQ + (ib + 1) * Q + 1;
    const double* Pt = tb + da * TB + C::tPt;
    double s = 0.0;
#pragma unroll
    for (int ia = 0; ia < M; ++ia) s = fma(U[ia], Pt[ia * M + ba], s);
    X[i] = s;
  }
  __syncthreads();
  // forward B: T_f[bb][ba] = sum_ib Pt_b[ib][bb] X_f[ib][ba]
  for (int i = tid; i < 6 * MM; i += NT) {
    const int f = i / MM, r = i - f * MM, bb = r / M, ba = r - bb * M, d = f >> 1, db = (d == 2) ? 1 : 2;
    const double* Pt = tb + db * TB + C::tPt;
    const double* Xf = X + f * MM;
    double s = 0.0;
#pragma unroll
    for (int ib = 0; ib < M; ++ib) s = fma(Pt[ib * M + bb], Xf[ib * M + ba], s);
    T[i] = s;
  }
  __syncthreads();
  {
    const double *L1 = tb + C::tLam, *L2 = tb + TB + C::tLam, *L3 = tb + 2 * TB + C::tLam;
    const double *a10 = tb + C::ta0, *a11 = tb + C::ta1;
    const double *a20 = tb + TB + C::ta0, *a21 = tb + TB + C::ta1;
    const double *a30 = tb + 2 * TB + C::ta0, *a31 = tb + 2 * TB + C::ta1;
    const double *T0 = T, *T1 = T + MM, *T2 = T + 2 * MM, *T3 = T + 3 * MM, *T4 = T + 4 * MM, *T5 = T + 5 * MM;
    for (int i = tid; i < 3 * MM; i += NT) {
      const int pass = i / MM, r = i - pass * MM, hi = r / M, lo = r - hi * M;
      double g0 = 0.0, g1 = 0.0;
      if (pass == 0) {          // (b3, b2), reduce over b1 -> faces 0, 1
        const int b3 = hi, b2 = lo;
        const double tA = T0[r], tB = T1[r], c2 = a20[b2], c2b = a21[b2], c3 = a30[b3], c3b = a31[b3];
        const double base = lam + L2[b2] + L3[b3];
#pragma unroll
        for (int b1 = 0; b1 < M; ++b1) {
          double E = a10[b1] * tA;
          E = fma(a11[b1], tB, E);
          E = fma(c2, T2[b3 * M + b1], E);
          E = fma(c2b, T3[b3 * M + b1], E);
          E = fma(c3, T4[b2 * M + b1], E);
          E = fma(c3b, T5[b2 * M + b1], E);
          const double V = E * rcp_nr(base + L1[b1]);
          g0 = fma(a10[b1], V, g0);
          g1 = fma(a11[b1], V, g1);
        }
      } else if (pass == 1) {   // (b3, b1), reduce over b2 -> faces 2, 3
        const int b3 = hi, b1 = lo;
        const double tA = T2[r], tB = T3[r], c1 = a10[b1], c1b = a11[b1], c3 = a30[b3], c3b = a31[b3];
        const double base = lam + L1[b1] + L3[b3];
#pragma unroll
        for (int b2 = 0; b2 < M; ++b2) {
          double E = c1 * T0[b3 * M + b2];
          E = fma(c1b, T1[b3 * M + b2], E);
          E = fma(a20[b2], tA, E);
          E = fma(a21[b2], tB, E);
          E = fma(c3, T4[b2 * M + b1], E);
          E = fma(c3b, T5[b2 * M + b1], E);
          const double V = E * rcp_nr(base + L2[b2]);
          g0 = fma(a20[b2], V, g0);
          g1 = fma(a21[b2], V, g1);
        }
      } else {                  // (b2, b1), reduce over b3 -> faces 4, 5
        const int b2 = hi, b1 = lo;
        const double tA = T4[r], tB = T5[r], c1 = a10[b1], c1b = a11[b1], c2 = a20[b2], c2b = a21[b2];
        const double base = lam + L1[b1] + L2[b2];
#pragma unroll
        for (int b3 = 0; b3 < M; ++b3) {
          double E = c1 * T0[b3 * M + b2];
          E = fma(c1b, T1[b3 * M + b2], E);
          E = fma(c2, T2[b3 * M + b1], E);
          E = fma(c2b, T3[b3 * M + b1], E);
          E = fma(a30[b3], tA, E);
          E = fma(a31[b3], tB, E);
          const double V = E * rcp_nr(base + L3[b3]);
          g0 = fma(a30[b3], V, g0);
          g1 = fma(a31[b3], V, g1);
        }
      }
      G[(2 * pass) * MM + r] = g0;
      G[(2 * pass + 1) * MM + r] = g1;
    }
  }
  __syncthreads();
  // back A: X_f[bb][ia] = sum_ba G_f[bb][ba] P_a[ba][ia]   (X in T's space)
  X = T;
  for (int i = tid; i < 6 * MM; i += NT) {
    const int f = i / MM, r = i - f * MM, bb = r / M, ia = r - bb * M, d = f >> 1, da = (d == 0) ? 1 : 0;
    const double* Pa = tb + da * TB + C::tP;
    const double* Gf = G + f * MM + bb * M;
    double s = 0.0;
#pragma unroll
    for (int ba = 0; ba < M; ++ba) s = fma(Gf[ba], Pa[ba * M + ia], s);
    X[i] = s;
  }
  __syncthreads();
  // back B: C_f[ib][ia] = sum_bb P_b[bb][ib] X_f[bb][ia]   (into G's space)
  for (int i = tid; i < 6 * MM; i += NT) {
    const int f = i / MM, r = i - f * MM, ib = r / M, ia = r - ib * M, d = f >> 1, db = (d == 2) ? 1 : 2;
    const double* Pb = tb + db * TB + C::tP;
    const double* Xf = X + f * MM;
    double s = 0.0;
#pragma unroll
    for (int bb = 0; bb < M; ++bb) s = fma(Pb[bb * M + ib], Xf[bb * M + ia], s);
    G[i] = s;
  }
  __syncthreads();
  // outputs: H_BB u (line sums over the closed faces) minus the face corrections
  const double *M1 = tb + C::tM, *M2 = tb + TB + C::tM, *M3 = tb + 2 * TB + C::tM;
  const double *K1 = tb + C::tK, *K2 = tb + TB + C::tK, *K3 = tb + 2 * TB + C::tK;
  double* Ye = Y + (size_t)e * g.YS;
  constexpr int YS = 6 * MM + 12 * M + 8;
  for (int o = tid; o < YS; o += NT) {
    int t1, t2, t3;
    double corr = 0.0;
    if (o < 6 * MM) {
      const int f = o / MM, r = o - f * MM, A = r / M, B = r - A * M, d = f >> 1, s = f & 1;
      if (d == 0) { t1 = s * P; t3 = A + 1; t2 = B + 1; }
      else if (d == 1) { t2 = s * P; t3 = A + 1; t1 = B + 1; }
      else { t3 = s * P; t2 = A + 1; t1 = B + 1; }
      corr = G[o];
    } else if (o < 6 * MM + 12 * M) {
      const int r = o - 6 * MM, qe = r / M, i = r - qe * M, d = qe >> 2, sA = qe & 1, sB = (qe >> 1) & 1;
      if (d == 0) { t1 = i + 1; t2 = sA * P; t3 = sB * P; }
      else if (d == 1) { t2 = i + 1; t1 = sA * P; t3 = sB * P; }
      else { t3 = i + 1; t1 = sA * P; t2 = sB * P; }
    } else {
      const int qv = o - 6 * MM - 12 * M;
      t1 = (qv & 1) * P; t2 = ((qv >> 1) & 1) * P; t3 = ((qv >> 2) & 1) * P;
    }
    const bool bd1 = (t1 == 0 || t1 == P), bd2 = (t2 == 0 || t2 == P), bd3 = (t3 == 0 || t3 == P);
    double y = lam * M1[t1] * M2[t2] * M3[t3] * getUc<P>(Uc, t1, t2, t3);
    double s = 0.0;
    if (bd2 || bd3) {
#pragma unroll
      for (int t = 0; t <= P; ++t) s = fma(K1[t1 * Q + t], getUc<P>(Uc, t, t2, t3), s);
    } else {
      s = K1[t1 * Q] * getUc<P>(Uc, 0, t2, t3) + K1[t1 * Q + P] * getUc<P>(Uc, P, t2, t3);
    }
    y = fma(M2[t2] * M3[t3], s, y);
    s = 0.0;
    if (bd1 || bd3) {
#pragma unroll
      for (int t = 0; t <= P; ++t) s = fma(K2[t2 * Q + t], getUc<P>(Uc, t1, t, t3), s);
    } else {
      s = K2[t2 * Q] * getUc<P>(Uc, t1, 0, t3) + K2[t2 * Q + P] * getUc<P>(Uc, t1, P, t3);
    }
    y = fma(M1[t1] * M3[t3], s, y);
    s = 0.0;
    if (bd1 || bd2) {
#pragma unroll
      for (int t = 0; t <= P; ++t) s = fma(K3[t3 * Q + t], getUc<P>(Uc, t1, t2, t), s);
    } else {
      s = K3[t3 * Q] * getUc<P>(Uc, t1, t2, 0) + K3[t3 * Q + P] * getUc<P>(Uc, t1, t2, P);
    }
    y = fma(M1[t1] * M2[t2], s, y);
    Ye[o] = y - corr;
  }
}

// ------------------------------------------------------------------------------------------
// star smoother, P <= 8 (Alg. 1 + Alg. 2; the p = 9..16 kernel is star16.cu):
//   - every global load of the star (S rows, eigen/weight vectors, the three r planes, and the
//     u values the star will update) is issued up front as cp.async (LDGSTS) into shared memory,
//     so the whole gather costs one L2 round trip; the u prefetch turns the final read-modify-
//     write into plain stores (the point sets of one colour are disjoint, so nobody
//     else writes those u entries during the launch);
//   - S^T is not loaded: the transposed operands read S with swapped indices;
//   - the cross-group G3 partials are first reduced inside each warp with shuffles and then
//     through the (idle) X buffer, so shared memory per CTA drops to ~37 KB at p = 8 and the
//     launch bound admits 5 CTAs per SM: one colour of a 16^3 mesh (<= 729 stars) runs as a
//     single wave on 148 SMs.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 8 : 0;   // src-size 0: zero fill, no global access
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Compile-time point maps.  A skeleton point is addressed relative to a base record as
//   bits 0-11: offset inside the record (face / edge / vertex slot, as skel_index_t),
//   bits 12-14: record coordinate d is (base - 1) [star maps] or (base + 1) [element maps],
//   bits 15-17: the point's local coordinate t_d inside that record is 0,
// so the per-point index arithmetic of a gather / scatter is two multiply-adds instead of the
// divisions and branches of skel_index_t.
constexpr unsigned rec_slot(int m, int t1, int t2, int t3) {
  if (t1 == 0) {
    if (t2 == 0) return (t3 == 0) ? (unsigned)(3 * m * m + 3 * m) : (unsigned)(3 * m * m + 2 * m + t3 - 1);
    if (t3 == 0) return (unsigned)(3 * m * m + m + t2 - 1);
    return (unsigned)((t3 - 1) * m + (t2 - 1));
  }
  if (t2 == 0) return (t3 == 0) ? (unsigned)(3 * m * m + t1 - 1) : (unsigned)(m * m + (t3 - 1) * m + (t1 - 1));
  return (unsigned)(2 * m * m + (t2 - 1) * m + (t1 - 1));
}

template <int P> struct StarMap { unsigned v[3 * (2 * P - 1) * (2 * P - 1)]; };
// star plane d, position (A, B) of the (2p-1)^2 plane (A slow), relative to the star's vertex record
template <int P> __host__ __device__ constexpr StarMap<P> make_star_map() {
  StarMap<P> s{};
  constexpr int N = 2 * P - 1, NN = N * N, c = P - 1, m = P - 1;
  for (int i = 0; i < 3 * NN; ++i) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    int j[3] = {0, 0, 0};
    if (d == 0) { j[0] = c; j[1] = B; j[2] = A; } else if (d == 1) { j[1] = c; j[0] = B; j[2] = A; } else { j[2] = c; j[0] = B; j[1] = A; }
    int t[3] = {0, 0, 0};
    unsigned code = 0;
    for (int k = 0; k < 3; ++k) {
      const int rel = j[k] - c;
      if (rel < 0) { t[k] = P + rel; code |= 1u << (12 + k); } else { t[k] = rel; }
      if (t[k] == 0) code |= 1u << (15 + k);
    }
    s.v[i] = code | rec_slot(m, t[0], t[1], t[2]);
  }
  return s;
}
template <int P> __device__ const StarMap<P> kStarMap = make_star_map<P>();

template <int P> struct ElemMap { unsigned v[6 * (P - 1) * (P - 1) + 12 * (P - 1) + 8]; };
// element boundary point o of the Y enumeration, relative to the element's low-corner record
template <int P> constexpr ElemMap<P> make_elem_map() {
  ElemMap<P> s{};
  constexpr int M = P - 1, MM = M * M, YS = 6 * MM + 12 * M + 8;
  for (int o = 0; o < YS; ++o) {
    int t[3] = {0, 0, 0};
    if (o < 6 * MM) {
      const int f = o / MM, r = o - f * MM, A = r / M, B = r - A * M, d = f >> 1, sd = f & 1;
      if (d == 0) { t[0] = sd * P; t[2] = A + 1; t[1] = B + 1; }
      else if (d == 1) { t[1] = sd * P; t[2] = A + 1; t[0] = B + 1; }
      else { t[2] = sd * P; t[1] = A + 1; t[0] = B + 1; }
    } else if (o < 6 * MM + 12 * M) {
      const int r = o - 6 * MM, qe = r / M, i = r - qe * M, d = qe >> 2, sA = qe & 1, sB = (qe >> 1) & 1;
      if (d == 0) { t[0] = i + 1; t[1] = sA * P; t[2] = sB * P; }
      else if (d == 1) { t[1] = i + 1; t[0] = sA * P; t[2] = sB * P; }
      else { t[2] = i + 1; t[0] = sA * P; t[1] = sB * P; }
    } else {
      const int qv = o - 6 * MM - 12 * M;
      t[0] = (qv & 1) * P; t[1] = ((qv >> 1) & 1) * P; t[2] = ((qv >> 2) & 1) * P;
    }
    unsigned code = 0;
    for (int k = 0; k < 3; ++k)
      if (t[k] == P) { t[k] = 0; code |= 1u << (12 + k); }
    s.v[o] = code | rec_slot(M, t[0], t[1], t[2]);
  }
  return s;
}
template <int P> __device__ const ElemMap<P> kElemMap = make_elem_map<P>();

template <int P> struct FaceMap { unsigned v[6 * (P + 1) * (P + 1)]; };
// closed face f = 2d + s, position (A slow, B fast) as in the element kernels' face arrays,
// relative to the element's low-corner record (same encoding as ElemMap)
template <int P> constexpr FaceMap<P> make_face_map() {
  FaceMap<P> s{};
  constexpr int Q = P + 1, QQ = Q * Q;
  for (int i = 0; i < 6 * QQ; ++i) {
    const int f = i / QQ, r = i - f * QQ, A = r / Q, B = r - A * Q, d = f >> 1, sd = f & 1;
    int t[3] = {0, 0, 0};
    if (d == 0) { t[0] = sd * P; t[2] = A; t[1] = B; }
    else if (d == 1) { t[1] = sd * P; t[2] = A; t[0] = B; }
    else { t[2] = sd * P; t[1] = A; t[0] = B; }
    unsigned code = 0;
    for (int k = 0; k < 3; ++k)
      if (t[k] == P) { t[k] = 0; code |= 1u << (12 + k); }
    s.v[i] = code | rec_slot(P - 1, t[0], t[1], t[2]);
  }
  return s;
}
template <int P> __device__ const FaceMap<P> kFaceMap = make_face_map<P>();

// record-index delta of map code bits 12-14 (sign applied by the caller)
__device__ __forceinline__ long long rec_delta(unsigned e, int V1, long long V12) {
  return (long long)((e >> 12) & 1u) + (long long)V1 * ((e >> 13) & 1u) + V12 * ((e >> 14) & 1u);
}

// C = op(A) op(B) for NP x NP shared-memory matrices (leading dimension LD), one warp, tile (mi, ni);
// TA / TB: read A / B transposed (A[i][k] = As[k][i], B[k][j] = Bs[j][k])
template <int NP, int LD, bool TA, bool TB>
__device__ __forceinline__ void dmma_tile_t(const double* A, const double* B, double* Cm, int mi, int ni, int lane) {
  const int r = lane >> 2, q = lane & 3;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll
  for (int kk = 0; kk < NP / 4; ++kk) {
    const int i = 8 * mi + r, k = 4 * kk + q, j = 8 * ni + r;
    const double a = TA ? A[k * LD + i] : A[i * LD + k];
    const double b = TB ? B[j * LD + k] : B[k * LD + j];
    dmma884(c0, c1, a, b);
  }
  Cm[(8 * mi + r) * LD + 8 * ni + 2 * q] = c0;
  Cm[(8 * mi + r) * LD + 8 * ni + 2 * q + 1] = c1;
}

// p <= 8: n_S padded to 8 / 16, 4 warps, 5 CTAs per SM; 9 <= p <= 16: n_S padded to 32, 8 warps
// (lanes own a1, each warp one a3 group), one CTA per SM, G3 warp partials in their own buffer
template <int P> struct StarPfCfg {
  static constexpr int N = 2 * P - 1, NN = N * N, C = P - 1;
  static constexpr int NP = (N <= 8) ? 8 : (N <= 16 ? 16 : 32), LD = NP + 4, MS = NP * LD, TPP = (NP / 8) * (NP / 8);
#ifndef PMG_STAR_MINB
#define PMG_STAR_MINB 5
#endif
  static constexpr int NW = (P <= 8) ? 4 : 8, NT = 32 * NW, MINB = (P <= 8) ? PMG_STAR_MINB : 1;
  static constexpr int GS = NP, GPW = 32 / GS, NG = NW * GPW, A3IT = (N + NG - 1) / NG;
  static constexpr bool P3SEP = NW * NN > 3 * MS;
  static constexpr int oFT = 0, oX = 3 * MS, oG = 6 * MS, oS = 9 * MS, oU = 12 * MS, oVec = oU + 3 * NN,
                       oBase = oVec + 9 * N, oP3 = P3SEP ? oBase + 8 : oX, endP3 = P3SEP ? oP3 + NW * NN : oBase + 8;
  // the compile-time point map, copied to shared memory in the prologue (before the dependency
  // wait): every later map read is a shared load instead of a dependent global round trip
  static constexpr int oMap = endP3, total = oMap + (3 * NN + 1) / 2;
};

template <int P>
size_t star_pf_smem() { return sizeof(double) * StarPfCfg<P>::total; }

template <int P>
__global__ void __launch_bounds__(StarPfCfg<P>::NT, StarPfCfg<P>::MINB)
    k_star_pf(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c, const double* __restrict__ r,
              double* __restrict__ u, const double* __restrict__ stab, double lam) {
  using C = StarPfCfg<P>;
  constexpr int N = C::N, NN = C::NN, c = C::C, NT = C::NT, NP = C::NP, LD = C::LD, MS = C::MS;
  constexpr int GS = C::GS, GPW = C::GPW, NG = C::NG;
  extern __shared__ double sm[];
  const int b = blockIdx.x, i1 = b % n1c, rest = b / n1c, i2 = rest % n2c, i3 = rest / n2c;
  const int v1 = c1 + 2 * i1, v2 = c2 + 2 * i2, v3 = c3 + 2 * i3;
  if (star_empty(g, v1, v2, v3)) return;
  if (v3 < g.own_lo) return;   // ghost star below the slab: computed by the lower rank
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, ST = g.ST;
  const size_t row[3] = {(size_t)v1, (size_t)(g.V1 + v2), (size_t)(g.V1 + g.V2 + v3)};
  double* FT = sm + C::oFT;
  double* X = sm + C::oX;
  double* Gs = sm + C::oG;
  double* Ssm = sm + C::oS;
  double* Up = sm + C::oU;
  double* vec = sm + C::oVec;
  constexpr int RS = 3 * (P - 1) * (P - 1) + 3 * (P - 1) + 1;
  const long long V12 = (long long)g.V1 * g.V2;
  const long long rec0 = v1 + g.V1 * (long long)v2 + V12 * v3;
  // interior stars (the common case) touch only inside, free points: no per-point tests
  const bool interior = ((v1 > 0 && v1 < g.k1) || (g.per & 1)) && ((v2 > 0 && v2 < g.k2) || (g.per & 2)) &&
                        ((v3 > 0 && v3 + g.zoff < g.K3) || (g.per & 4));
  unsigned* map_s = reinterpret_cast<unsigned*>(sm + C::oMap);
  for (int i = tid; i < 3 * NN; i += NT) map_s[i] = __ldg(&kStarMap<P>.v[i]);
  // point of map entry e: record coordinate w_d = v_d - bit; free iff (w_d > 0 or t_d > 0) and
  // w_d < k_d (global in z); stored (readable) iff w_d >= 0
  auto pt_free = [&](unsigned e) {   // global test (w3 + zoff is the global record plane), Neumann faces free
    const int w1 = v1 - (int)((e >> 12) & 1u), w2 = v2 - (int)((e >> 13) & 1u), w3 = v3 - (int)((e >> 14) & 1u);
    const int W3 = w3 + g.zoff;
    // the point is G_d = w_d p + t_d (0 <= t_d < p), t_d == 0 iff bit 15 + d
    const bool z1 = e & (1u << 15), z2 = e & (1u << 16), z3 = e & (1u << 17);
    return ((g.per & 1) || (w1 >= 0 && (w1 > 0 || !z1 || (g.neu & 1)) && (w1 < g.k1 || (z1 && w1 == g.k1 && (g.neu & 2))))) &&
           ((g.per & 2) || (w2 >= 0 && (w2 > 0 || !z2 || (g.neu & 4)) && (w2 < g.k2 || (z2 && w2 == g.k2 && (g.neu & 8))))) &&
           ((g.per & 4) || (w3 >= 0 && (W3 > 0 || !z3 || (g.neu & 16)) && (W3 < g.K3 || (z3 && W3 == g.K3 && (g.neu & 32)))));
  };
  // record base index of each of the 8 record-offset codes (-1: record outside the stored box)
  long long* s_base = reinterpret_cast<long long*>(sm + C::oBase);
  if (tid < 8) {
    const int b1 = tid & 1, b2 = (tid >> 1) & 1, b3 = (tid >> 2) & 1;
    const bool ok = !((v1 == 0 && b1 && !(g.per & 1)) || (v2 == 0 && b2 && !(g.per & 2)) || (v3 == 0 && b3 && !(g.per & 4)));
    const int w1 = wrap_rec(v1 - b1, g.k1, g.per & 1), w2 = wrap_rec(v2 - b2, g.k2, g.per & 2),
              w3 = wrap_rec(v3 - b3, g.k3, g.per & 4);   // periodic: record k-1 for v = 0
    s_base[tid] = ok ? (w1 + g.V1 * (long long)w2 + V12 * w3) * RS : -1LL;
  }
  const size_t srow[3] = {row[0] * ST, row[1] * ST, row[2] * ST};
  __syncthreads();
  // group 0: S rows, eigen/weight vectors (setup tables: before the dependency wait), the r planes
  for (int i = tid; i < 3 * NN; i += NT) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    cp_async8(&Ssm[d * MS + A * LD + B], &stab[srow[d] + rr], true);
  }
  for (int i = tid; i < 9 * N; i += NT) { const int d = i / (3 * N); cp_async8(&vec[i], &stab[srow[d] + NN + i - d * 3 * N], true); }
  pdl_wait();
  pdl_trigger();
  for (int i = tid; i < 3 * NN; i += NT) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    const unsigned e = map_s[i];
    const long long base = s_base[(e >> 12) & 7u];
    const bool ok = base >= 0;
    cp_async8(&FT[d * MS + A * LD + B], &r[ok ? base + (e & 0xFFFu) : 0], ok);
  }
  cp_async_commit();
  // group 1: the u entries this star updates (0 where the point is not free)
  for (int i = tid; i < 3 * NN; i += NT) {
    const unsigned e = map_s[i];
    const long long base = s_base[(e >> 12) & 7u];
    const bool ok = base >= 0 && (interior || pt_free(e));
    cp_async8(&Up[i], &u[ok ? base + (e & 0xFFFu) : 0], ok);
  }
  cp_async_commit();
  // zero the padding rows / columns of F, S and G (the transforms read them; must be finite)
  constexpr int PADN = NP * NP - NN, PC = NP - N;   // columns N.. of rows < N, then rows N..
  for (int i = tid; i < 3 * PADN; i += NT) {
    const int d = i / PADN, k = i - d * PADN;
    int A, B;
    if (k < N * PC) { A = k / PC; B = N + (k - A * PC); }
    else { const int k2 = k - N * PC; A = N + k2 / NP; B = k2 - (A - N) * NP; }
    const int o = d * MS + A * LD + B;
    FT[o] = 0.0;
    Ssm[o] = 0.0;
    Gs[o] = 0.0;
  }
  cp_async_wait<1>();
  __syncthreads();
  // inverse multiplicity on the two lines through the vertex of each plane
  for (int i = tid; i < 3 * 2 * N; i += NT) {
    const int d = i / (2 * N), rr = i - d * 2 * N, line = rr / N, t = rr - line * N;
    const int A = line ? t : c, B = line ? c : t;
    if (line && t == c) continue;     // the vertex itself: scaled once, by the row pass
    FT[d * MS + A * LD + B] *= 1.0 / (double)(1 + (A == c) + (B == c));
  }
  __syncthreads();
  // forward: X_d = F_d S_a ; T_d = S_b^T X_d
  for (int job = warp; job < 3 * C::TPP; job += C::NW) {
    const int d = job / C::TPP, t = job - d * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    dmma_tile_t<NP, LD, false, false>(FT + d * MS, Ssm + (d == 0 ? 1 : 0) * MS, X + d * MS, mi, ni, lane);
  }
  __syncthreads();
  for (int job = warp; job < 3 * C::TPP; job += C::NW) {
    const int d = job / C::TPP, t = job - d * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    dmma_tile_t<NP, LD, true, false>(Ssm + (d == 2 ? 1 : 2) * MS, X + d * MS, FT + d * MS, mi, ni, lane);
  }
  __syncthreads();
  // single-pass core (as k_star_dm); G3 partials reduced in-warp, then across warps through X
  {
    const double *L1 = vec, *s1 = vec + N, *L2 = vec + 3 * N, *s2 = vec + 4 * N, *L3 = vec + 6 * N, *s3 = vec + 7 * N;
    const double *T1 = FT, *T2 = FT + MS, *T3 = FT + 2 * MS;
    const int grp = warp * GPW + lane / GS, a1 = lane % GS;
    const bool va = a1 < N;
    const int a1c = va ? a1 : 0;
    const double s1a = va ? s1[a1c] : 0.0, L1a = L1[a1c];
    double g3[N];
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2) g3[a2] = 0.0;
    for (int k = 0; k < C::A3IT; ++k) {
      const int a3 = grp + k * NG;
      const bool act = a3 < N;
      const int a3c = act ? a3 : 0;
      const double on = (act && va) ? 1.0 : 0.0;
      const double t2 = on * T2[a3c * LD + a1c], s3v = on * s3[a3c], base = lam + L1a + L3[a3c];
      const double s1v = on * s1a;
      double g2 = 0.0;
      double v[GS];
#pragma unroll
      for (int a2 = 0; a2 < GS; ++a2) v[a2] = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        double E = s1v * T1[a3c * LD + a2];
        E = fma(s2[a2], t2, E);
        E = fma(s3v, T3[a2 * LD + a1c], E);
        const double V = E * rcp_nr(base + L2[a2]);
        g2 = fma(s2[a2], V, g2);
        g3[a2] = fma(s3v, V, g3[a2]);
        v[a2] = s1v * V;
      }
#pragma unroll
      for (int off = GS / 2; off >= 1; off >>= 1) {
        const bool upper = (a1 & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
          const double send = upper ? v[j] : v[j + off];
          const double keep = upper ? v[j + off] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (act && va) {
        Gs[a3 * LD + a1] = v[0];               // G1[a3][a2 = a1]
        Gs[MS + a3 * LD + a1] = g2;            // G2[a3][a1]
      }
    }
#pragma unroll
    for (int off = GS; off < 32; off <<= 1) {
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) g3[a2] += __shfl_xor_sync(0xffffffffu, g3[a2], off);
    }
    double* P3 = sm + C::oP3;
    if (va && lane < GS) {
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) P3[warp * NN + a2 * N + a1] = g3[a2];
    }
    __syncthreads();
    for (int i = tid; i < NN; i += NT) {
      const int a2 = i / N, a1_ = i - a2 * N;
      double s_ = 0.0;
#pragma unroll
      for (int w = 0; w < C::NW; ++w) s_ += P3[w * NN + i];
      Gs[2 * MS + a2 * LD + a1_] = s_;
    }
  }
  __syncthreads();
  // back: X_d = G_d S_a^T ; U_d = S_b X_d (into G)
  for (int job = warp; job < 3 * C::TPP; job += C::NW) {
    const int d = job / C::TPP, t = job - d * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    dmma_tile_t<NP, LD, false, true>(Gs + d * MS, Ssm + (d == 0 ? 1 : 0) * MS, X + d * MS, mi, ni, lane);
  }
  __syncthreads();
  for (int job = warp; job < 3 * C::TPP; job += C::NW) {
    const int d = job / C::TPP, t = job - d * C::TPP, mi = t / (NP / 8), ni = t - mi * (NP / 8);
    dmma_tile_t<NP, LD, false, false>(Ssm + (d == 2 ? 1 : 2) * MS, X + d * MS, Gs + d * MS, mi, ni, lane);
  }
  cp_async_wait<0>();
  __syncthreads();
  const double *w1 = vec + 2 * N, *w2 = vec + 5 * N, *w3 = vec + 8 * N;
  for (int i = tid; i < 3 * NN; i += NT) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    int j1, j2, j3;
    if (d == 0) { j1 = c; j2 = B; j3 = A; }
    else if (d == 1) { j2 = c; j1 = B; j3 = A; if (j1 == c) continue; }
    else { j3 = c; j1 = B; j2 = A; if (j1 == c || j2 == c) continue; }
    const unsigned e = map_s[i];
    if (!interior && !pt_free(e)) continue;
    u[s_base[(e >> 12) & 7u] + (e & 0xFFFu)] = fma(w1[j1] * w2[j2] * w3[j3], Gs[d * MS + A * LD + B], Up[i]);
  }
}

// ------------------------------------------------------------------------------------------
// element operator for P <= 8, latency-oriented version of k_elem_dm (same arithmetic and
// citations: P:117-123, reading R1):
//   - one cp.async pass stages the element's three table rows (contiguous in etab) and its
//     (p+1)^3 - (p-1)^3 boundary values -- scattered straight into a zero-interior (p+1)^3 cube --
//     so the gather is one L2 round trip with no index decoding of the table layout;
//   - H_BB u is then three plain line sums through the cube for every output (the zero interior
//     makes the edge / vertex / face cases identical, no branches);
//   - only the padded P_d is built; the transposed operands of the DMMA transforms read it with
//     swapped indices.
// ------------------------------------------------------------------------------------------
template <int P> struct ElemPfCfg {
  // p <= 4: direct m x m face transforms, tight m x m arrays; p > 4: 8 x 8 DMMA tiles (leading dim 12)
  static constexpr int M = P - 1, Q = P + 1, MM = M * M, QQ = Q * Q, QQQ = Q * QQ, MP = 8, LD = (P <= 4) ? M : 12,
                       MS = (P <= 4) ? MM : MP * LD, NPP = (P <= 4) ? 0 : 3 * MS;
  // p <= 4: two warps per element (with the direct transforms: p = 4 residual 1.12 -> 1.00 ms)
  static constexpr int NT = (P <= 4) ? 64 : 128, NW = NT / 32, MINB = (NT == 64) ? 16 : 8;
  static constexpr int ET = (P - 1) + 2 * (P - 1) * (P - 1) + 2 * (P - 1) + (P + 1) + (P + 1) * (P + 1);
  static constexpr int YS = 6 * MM + 12 * M + 8;
  static constexpr int oCube = 0, oTab = QQQ, oPp = oTab + 3 * ET, oA = oPp + NPP, oT = oA + 6 * MS,
                       oG = oT + 6 * MS, oInv = oG + 6 * MS, oMap = oInv + MM * M, total = oMap + (YS + 1) / 2;
};

template <int P>
size_t elem_pf_smem() { return sizeof(double) * ElemPfCfg<P>::total; }

// boundary point o (0 <= o < YS) of the element in the Y enumeration -> local (t1, t2, t3)
template <int P>
__device__ __forceinline__ void ys_point(int o, int& t1, int& t2, int& t3) {
  constexpr int M = P - 1, MM = M * M;
  if (o < 6 * MM) {
    const int f = o / MM, r = o - f * MM, A = r / M, B = r - A * M, d = f >> 1, s = f & 1;
    if (d == 0) { t1 = s * P; t3 = A + 1; t2 = B + 1; }
    else if (d == 1) { t2 = s * P; t3 = A + 1; t1 = B + 1; }
    else { t3 = s * P; t2 = A + 1; t1 = B + 1; }
  } else if (o < 6 * MM + 12 * M) {
    const int r = o - 6 * MM, qe = r / M, i = r - qe * M, d = qe >> 2, sA = qe & 1, sB = (qe >> 1) & 1;
    if (d == 0) { t1 = i + 1; t2 = sA * P; t3 = sB * P; }
    else if (d == 1) { t2 = i + 1; t1 = sA * P; t3 = sB * P; }
    else { t3 = i + 1; t1 = sA * P; t2 = sB * P; }
  } else {
    const int qv = o - 6 * MM - 12 * M;
    t1 = (qv & 1) * P; t2 = ((qv >> 1) & 1) * P; t3 = ((qv >> 2) & 1) * P;
  }
}

template <int P>
__global__ void __launch_bounds__(ElemPfCfg<P>::NT, ElemPfCfg<P>::MINB)
    k_elem_pf(LevelGeom g, const double* __restrict__ u, const double* __restrict__ etab, double lam,
              double* __restrict__ Y, const int* __restrict__ done) {
  using C = ElemPfCfg<P>;
  constexpr int M = C::M, Q = C::Q, MM = C::MM, QQ = C::QQ, NT = C::NT, ET = C::ET, LD = C::LD,
                MS = C::MS, MP = C::MP, YS = C::YS;
  extern __shared__ double sm[];
  double* cube = sm + C::oCube;
  double* tb = sm + C::oTab;
  double* Pp = sm + C::oPp;
  double* Ab = sm + C::oA;
  double* T = sm + C::oT;
  double* G = sm + C::oG;
  double* invD = sm + C::oInv;
  const long long e = blockIdx.x;
  const int e1 = (int)(e % g.k1), e2 = (int)((e / g.k1) % g.k2), e3 = (int)(e / ((long long)g.k1 * g.k2));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const double* src[3] = {etab + (size_t)e1 * ET, etab + (size_t)(g.k1 + e2) * ET, etab + (size_t)(g.k1 + g.k2 + e3) * ET};
    for (int i = tid; i < 3 * ET; i += NT) {
      const int d = i / ET;
      cp_async8(&tb[i], src[d] + (i - d * ET), true);
    }
    unsigned* map_s = reinterpret_cast<unsigned*>(sm + C::oMap);   // the point map, before the wait
    for (int o = tid; o < YS; o += NT) map_s[o] = __ldg(&kElemMap<P>.v[o]);
    __syncthreads();
    pdl_wait();
  pdl_trigger();
    if (done && *done) return;   // (uniform per block; the issued cp.async only target this block's smem)
    constexpr int RS = 3 * MM + 3 * M + 1;
    const long long V12 = (long long)g.V1 * g.V2;
    auto rb = [&](unsigned code) {   // record of the map code's +1 offsets (periodic: wrapped)
      const int w1 = wrap_rec(e1 + (int)(code & 1u), g.k1, g.per & 1), w2 = wrap_rec(e2 + (int)((code >> 1) & 1u), g.k2, g.per & 2),
                w3 = wrap_rec(e3 + (int)((code >> 2) & 1u), g.k3, g.per & 4);
      return (w1 + g.V1 * (long long)w2 + V12 * w3) * RS;
    };
    for (int o = tid; o < YS; o += NT) {
      int t1, t2, t3;
      ys_point<P>(o, t1, t2, t3);
      const unsigned m_ = map_s[o];
      cp_async8(&cube[(t3 * Q + t2) * Q + t1], &u[rb((m_ >> 12) & 7u) + (m_ & 0xFFFu)], true);
    }
    cp_async_commit();
    for (int i = tid; i < M * MM; i += NT) {        // zero interior of the cube
      const int a3 = i / MM, rr = i - a3 * MM, a2 = rr / M, a1 = rr - a2 * M;
      cube[((a3 + 1) * Q + a2 + 1) * Q + a1 + 1] = 0.0;
    }
    if constexpr (P > 4)
      for (int i = tid; i < 6 * MS; i += NT) G[i] = 0.0;
    cp_async_wait<0>();
    __syncthreads();
  }
  const double* Lv[3] = {tb + et_lam(P), tb + ET + et_lam(P), tb + 2 * ET + et_lam(P)};
  // the face interior value (A, B) of face f in the zero-interior cube
  auto face_pt = [&](int f, int A, int B) {
    const int d = f >> 1, sd = (f & 1) * P;
    return (d == 0) ? ((A + 1) * Q + B + 1) * Q + sd : ((d == 1) ? ((A + 1) * Q + sd) * Q + B + 1 : (sd * Q + A + 1) * Q + B + 1);
  };
  if constexpr (P <= 4) {
    // m <= 3: the face transforms as direct m x m products from the table rows (the padded 8 x 8
    // DMMA tiles of p > 4 would be > 85 % zeros, and their staging made the kernel shared-memory bound)
    for (int i = tid; i < 6 * MM; i += NT) {        // X_f[A][ba] = sum_B U_f[A][B] P_a[ba][B]  (into T)
      const int f = i / MM, r = i - f * MM, A = r / M, ba = r - A * M, d = f >> 1, da = (d == 0) ? 1 : 0;
      const double* Pa = tb + da * ET + et_P(P) + ba * M;
      double x = 0.0;
#pragma unroll
      for (int B = 0; B < M; ++B) x = fma(cube[face_pt(f, A, B)], Pa[B], x);
      T[f * MS + A * LD + ba] = x;
    }
    for (int i = tid; i < MM * M; i += NT) {        // 1/D over the interior eigen-triples
      const int b3 = i / MM, rr = i - b3 * MM, b2 = rr / M, b1 = rr - b2 * M;
      invD[i] = rcp_nr(lam + Lv[0][b1] + Lv[1][b2] + Lv[2][b3]);
    }
    __syncthreads();
    for (int i = tid; i < 6 * MM; i += NT) {        // T_f[bb][ba] = sum_A P_b[bb][A] X_f[A][ba]  (into Ab)
      const int f = i / MM, r = i - f * MM, bb = r / M, ba = r - bb * M, d = f >> 1, db = (d == 2) ? 1 : 2;
      const double* Pb = tb + db * ET + et_P(P) + bb * M;
      double t = 0.0;
#pragma unroll
      for (int A = 0; A < M; ++A) t = fma(Pb[A], T[f * MS + A * LD + ba], t);
      Ab[f * MS + bb * LD + ba] = t;
    }
  } else {
  for (int i = tid; i < 3 * MP * MP; i += NT) {     // padded P_d[b][i]
    const int d = i / (MP * MP), rr = i - d * MP * MP, A = rr / MP, B = rr - A * MP;
    Pp[d * MS + A * LD + B] = (A < M && B < M) ? tb[d * ET + et_P(P) + A * M + B] : 0.0;
  }
  for (int i = tid; i < 6 * MP * MP; i += NT) {     // padded face interiors from the cube
    const int f = i / (MP * MP), rr = i - f * MP * MP, A = rr / MP, B = rr - A * MP;
    Ab[f * MS + A * LD + B] = (A < M && B < M) ? cube[face_pt(f, A, B)] : 0.0;
  }
  for (int i = tid; i < MM * M; i += NT) {          // 1/D over the interior eigen-triples
    const int b3 = i / MM, rr = i - b3 * MM, b2 = rr / M, b1 = rr - b2 * M;
    invD[i] = rcp_nr(lam + Lv[0][b1] + Lv[1][b2] + Lv[2][b3]);
  }
  __syncthreads();
  for (int f = warp; f < 6; f += C::NW) {            // forward A: X_f = U_f P_a^T  (into T)
    const int d = f >> 1, da = (d == 0) ? 1 : 0;
    dmma_tile_t<MP, LD, false, true>(Ab + f * MS, Pp + da * MS, T + f * MS, 0, 0, lane);
  }
  __syncthreads();
  for (int f = warp; f < 6; f += C::NW) {            // forward B: T_f = P_b X_f  (into Ab)
    const int d = f >> 1, db = (d == 2) ? 1 : 2;
    dmma_tile_t<MP, LD, false, false>(Pp + db * MS, T + f * MS, Ab + f * MS, 0, 0, lane);
  }
  }
  __syncthreads();
  {
    const double *a10 = tb + et_a0(P), *a11 = tb + et_a1(P);
    const double *a20 = tb + ET + et_a0(P), *a21 = tb + ET + et_a1(P);
    const double *a30 = tb + 2 * ET + et_a0(P), *a31 = tb + 2 * ET + et_a1(P);
    const double *T0 = Ab, *T1 = Ab + MS, *T2 = Ab + 2 * MS, *T3 = Ab + 3 * MS, *T4 = Ab + 4 * MS, *T5 = Ab + 5 * MS;
    for (int i = tid; i < 3 * MM; i += NT) {
      const int pass = i / MM, r = i - pass * MM, hi = r / M, lo = r - hi * M;
      double g0 = 0.0, g1 = 0.0;
      if (pass == 0) {          // (b3, b2), reduce over b1 -> faces 0, 1
        const int b3 = hi, b2 = lo;
        const double tA = T0[b3 * LD + b2], tB = T1[b3 * LD + b2], c2 = a20[b2], c2b = a21[b2], c3 = a30[b3], c3b = a31[b3];
#pragma unroll
        for (int b1 = 0; b1 < M; ++b1) {
          double Ev = a10[b1] * tA;
          Ev = fma(a11[b1], tB, Ev);
          Ev = fma(c2, T2[b3 * LD + b1], Ev);
          Ev = fma(c2b, T3[b3 * LD + b1], Ev);
          Ev = fma(c3, T4[b2 * LD + b1], Ev);
          Ev = fma(c3b, T5[b2 * LD + b1], Ev);
          const double V = Ev * invD[(b3 * M + b2) * M + b1];
          g0 = fma(a10[b1], V, g0);
          g1 = fma(a11[b1], V, g1);
        }
        G[0 * MS + b3 * LD + b2] = g0;
        G[1 * MS + b3 * LD + b2] = g1;
      } else if (pass == 1) {   // (b3, b1), reduce over b2 -> faces 2, 3
        const int b3 = hi, b1 = lo;
        const double tA = T2[b3 * LD + b1], tB = T3[b3 * LD + b1], c1 = a10[b1], c1b = a11[b1], c3 = a30[b3], c3b = a31[b3];
#pragma unroll
        for (int b2 = 0; b2 < M; ++b2) {
          double Ev = c1 * T0[b3 * LD + b2];
          Ev = fma(c1b, T1[b3 * LD + b2], Ev);
          Ev = fma(a20[b2], tA, Ev);
          Ev = fma(a21[b2], tB, Ev);
          Ev = fma(c3, T4[b2 * LD + b1], Ev);
          Ev = fma(c3b, T5[b2 * LD + b1], Ev);
          const double V = Ev * invD[(b3 * M + b2) * M + b1];
          g0 = fma(a20[b2], V, g0);
          g1 = fma(a21[b2], V, g1);
        }
        G[2 * MS + b3 * LD + b1] = g0;
        G[3 * MS + b3 * LD + b1] = g1;
      } else {                  // (b2, b1), reduce over b3 -> faces 4, 5
        const int b2 = hi, b1 = lo;
        const double tA = T4[b2 * LD + b1], tB = T5[b2 * LD + b1], c1 = a10[b1], c1b = a11[b1], c2 = a20[b2], c2b = a21[b2];
#pragma unroll
        for (int b3 = 0; b3 < M; ++b3) {
          double Ev = c1 * T0[b3 * LD + b2];
          Ev = fma(c1b, T1[b3 * LD + b2], Ev);
          Ev = fma(c2, T2[b3 * LD + b1], Ev);
          Ev = fma(c2b, T3[b3 * LD + b1], Ev);
          Ev = fma(a30[b3], tA, Ev);
          Ev = fma(a31[b3], tB, Ev);
          const double V = Ev * invD[(b3 * M + b2) * M + b1];
          g0 = fma(a30[b3], V, g0);
          g1 = fma(a31[b3], V, g1);
        }
        G[4 * MS + b2 * LD + b1] = g0;
        G[5 * MS + b2 * LD + b1] = g1;
      }
    }
  }
  __syncthreads();
  if constexpr (P <= 4) {
    for (int i = tid; i < 6 * MM; i += NT) {        // X_f[bb][B] = sum_ba G_f[bb][ba] P_a[ba][B]  (into T)
      const int f = i / MM, r = i - f * MM, bb = r / M, B = r - bb * M, d = f >> 1, da = (d == 0) ? 1 : 0;
      const double* Pa = tb + da * ET + et_P(P) + B;
      double x = 0.0;
#pragma unroll
      for (int ba = 0; ba < M; ++ba) x = fma(G[f * MS + bb * LD + ba], Pa[ba * M], x);
      T[f * MS + bb * LD + B] = x;
    }
    __syncthreads();
    for (int i = tid; i < 6 * MM; i += NT) {        // C_f[A][B] = sum_bb P_b[bb][A] X_f[bb][B]  (into G)
      const int f = i / MM, r = i - f * MM, A = r / M, B = r - A * M, d = f >> 1, db = (d == 2) ? 1 : 2;
      const double* Pb = tb + db * ET + et_P(P) + A;
      double c = 0.0;
#pragma unroll
      for (int bb = 0; bb < M; ++bb) c = fma(Pb[bb * M], T[f * MS + bb * LD + B], c);
      G[f * MS + A * LD + B] = c;
    }
  } else {
  for (int f = warp; f < 6; f += C::NW) {            // back A: X_f = G_f P_a   (into T)
    const int d = f >> 1, da = (d == 0) ? 1 : 0;
    dmma_tile_t<MP, LD, false, false>(G + f * MS, Pp + da * MS, T + f * MS, 0, 0, lane);
  }
  __syncthreads();
  for (int f = warp; f < 6; f += C::NW) {            // back B: C_f = P_b^T X_f  (into G)
    const int d = f >> 1, db = (d == 2) ? 1 : 2;
    dmma_tile_t<MP, LD, true, false>(Pp + db * MS, T + f * MS, G + f * MS, 0, 0, lane);
  }
  }
  __syncthreads();
  const double *M1 = tb + et_M(P), *M2 = tb + ET + et_M(P), *M3 = tb + 2 * ET + et_M(P);
  const double *K1 = tb + et_K(P), *K2 = tb + ET + et_K(P), *K3 = tb + 2 * ET + et_K(P);
  double* Ye = Y + (size_t)e * g.YS;
  for (int o = tid; o < YS; o += NT) {
    int t1, t2, t3;
    ys_point<P>(o, t1, t2, t3);
    const double* c1 = cube + (t3 * Q + t2) * Q;     // line along x1
    const double* c2 = cube + t3 * QQ + t1;          // line along x2 (stride Q)
    const double* c3 = cube + t2 * Q + t1;           // line along x3 (stride QQ)
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    // a line through a face point along the face normal crosses the zero interior: only its two
    // end values are nonzero (the skipped terms are exact zeros, the sums are unchanged)
    const int nd = o < 6 * MM ? (o / MM) >> 1 : 3;
    if (nd == 0) {
      s1 = fma(K1[t1 * Q + P], c1[P], K1[t1 * Q] * c1[0]);
    } else {
#pragma unroll
      for (int t = 0; t <= P; ++t) s1 = fma(K1[t1 * Q + t], c1[t], s1);
    }
    if (nd == 1) {
      s2 = fma(K2[t2 * Q + P], c2[P * Q], K2[t2 * Q] * c2[0]);
    } else {
#pragma unroll
      for (int t = 0; t <= P; ++t) s2 = fma(K2[t2 * Q + t], c2[t * Q], s2);
    }
    if (nd == 2) {
      s3 = fma(K3[t3 * Q + P], c3[P * QQ], K3[t3 * Q] * c3[0]);
    } else {
#pragma unroll
      for (int t = 0; t <= P; ++t) s3 = fma(K3[t3 * Q + t], c3[t * QQ], s3);
    }
    const double m1 = M1[t1], m2 = M2[t2], m3 = M3[t3];
    double y = lam * m1 * m2 * m3 * c1[t1];
    y = fma(m2 * m3, s1, y);
    y = fma(m1 * m3, s2, y);
    y = fma(m1 * m2, s3, y);
    if (o < 6 * MM) {
      const int f = o / MM, r = o - f * MM, A = r / M, B = r - A * M;
      y -= G[f * MS + A * LD + B];
    }
    Ye[o] = y;
  }
}

// ------------------------------------------------------------------------------------------
// star smoother, 17 <= P <= 32 (same arithmetic and citations as k_star_t: Alg. 1 + Alg. 2,
// P:294-331): the twelve n_S x n_S transforms on DMMA with n_S padded to 64 (LD 68), S read from
// the L2-resident star tables (guarded: zero outside n_S) instead of being staged, the 3-pass core
// of k_star_t (a single-pass core's cross-warp partials do not fit next to two padded plane
// triples in 227 KB).  A DFMA transform needs two shared-memory loads per FMA; a DMMA does 256 FMA
// per two fragment loads.
// ------------------------------------------------------------------------------------------
template <int P> struct StarTmCfg {
  // n_S padded to a multiple of 8 (40 ... 64), leading dimension = 4 mod 8 (conflict-free fragments)
  static constexpr int N = 2 * P - 1, NN = N * N, C = P - 1, NP = (N + 7) / 8 * 8, LD = NP + 4, MS = NP * LD;
  static constexpr int NT = 256, NW = 8, TB = NP / 8, TPP = TB * TB;
  static constexpr int oFT = 0, oG = 3 * MS, oVec = 6 * MS, total = oVec + 9 * N;
};

template <int P>
size_t star_tm_smem() { return sizeof(double) * StarTmCfg<P>::total; }

// C(8x8 tile mi, ni) = A B with element accessors a(i, k), b(k, j); one warp
template <int KT, class FA, class FB>
__device__ __forceinline__ void dmma_tile_fn(const FA& a, const FB& b, double* Cm, int ldc, int mi, int ni, int lane) {
  const int r = lane >> 2, q = lane & 3;
  double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < KT / 4; ++kk) dmma884(c0, c1, a(8 * mi + r, 4 * kk + q), b(4 * kk + q, 8 * ni + r));
  Cm[(8 * mi + r) * ldc + 8 * ni + 2 * q] = c0;
  Cm[(8 * mi + r) * ldc + 8 * ni + 2 * q + 1] = c1;
}

template <int P>
__global__ void __launch_bounds__(256, 1) k_star_tm(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c,
                                                   const double* __restrict__ r, double* __restrict__ u,
                                                   const double* __restrict__ stab, double lam) {
  using C = StarTmCfg<P>;
  constexpr int N = C::N, NN = C::NN, c = C::C, NT = C::NT, NP = C::NP, LD = C::LD, MS = C::MS, TPP = C::TPP;
  extern __shared__ double sm[];
  const int b = blockIdx.x, i1 = b % n1c, rest = b / n1c, i2 = rest % n2c, i3 = rest / n2c;
  const int v1 = c1 + 2 * i1, v2 = c2 + 2 * i2, v3 = c3 + 2 * i3;
  if (star_empty(g, v1, v2, v3)) return;
  if (v3 < g.own_lo) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, ST = g.ST;
  const double* S[3] = {stab + (size_t)v1 * ST, stab + (size_t)(g.V1 + v2) * ST, stab + (size_t)(g.V1 + g.V2 + v3) * ST};
  double* FT = sm + C::oFT;
  double* Gs = sm + C::oG;
  double* vec = sm + C::oVec;
  for (int i = tid; i < 9 * N; i += NT) { const int d = i / (3 * N); vec[i] = __ldg(&S[d][NN + i - d * 3 * N]); }
  for (int i = tid; i < 3 * MS; i += NT) FT[i] = 0.0;           // padding must be finite (zero)
  pdl_wait();
  pdl_trigger();
  __syncthreads();
  const int o1 = (v1 - 1) * P + 1, o2 = (v2 - 1) * P + 1, o3 = (v3 - 1) * P + 1;
  for (int i = tid; i < 3 * NN; i += NT) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    int j1, j2, j3;
    if (d == 0) { j1 = c; j2 = B; j3 = A; } else if (d == 1) { j2 = c; j1 = B; j3 = A; } else { j3 = c; j1 = B; j2 = A; }
    int g1 = o1 + j1, g2 = o2 + j2, g3 = o3 + j3;
    wrap_pt(g, g1, g2, g3);
    const double val = inside(g, g1, g2, g3) ? __ldg(&r[skel_index_t<P>(g, g1, g2, g3)]) : 0.0;
    FT[d * MS + A * LD + B] = val * (1.0 / (double)(1 + (A == c) + (B == c)));   // inverse multiplicity
  }
  __syncthreads();
  auto sget = [](const double* Sd, int row, int col) { return (row < N && col < N) ? __ldg(&Sd[row * N + col]) : 0.0; };
  // forward A: X_d = F_d S_a  (X into G's space)
  for (int job = warp; job < 3 * TPP; job += C::NW) {
    const int d = job / TPP, t = job - d * TPP, mi = t / C::TB, ni = t - mi * C::TB;
    const double* Fd = FT + d * MS;
    const double* Sa = S[d == 0 ? 1 : 0];
    dmma_tile_fn<NP>([&](int i, int k) { return Fd[i * LD + k]; }, [&](int k, int j) { return sget(Sa, k, j); },
                     Gs + d * MS, LD, mi, ni, lane);
  }
  __syncthreads();
  // forward B: T_d = S_b^T X_d  (into FT)
  for (int job = warp; job < 3 * TPP; job += C::NW) {
    const int d = job / TPP, t = job - d * TPP, mi = t / C::TB, ni = t - mi * C::TB;
    const double* Xd = Gs + d * MS;
    const double* Sb = S[d == 2 ? 1 : 2];
    dmma_tile_fn<NP>([&](int i, int k) { return sget(Sb, k, i); }, [&](int k, int j) { return Xd[k * LD + j]; },
                     FT + d * MS, LD, mi, ni, lane);
  }
  __syncthreads();
  // fused core (expand / D^-1 / contract), three passes each reducing along one axis (k_star_t)
  {
    const double *L1 = vec, *s1 = vec + N, *L2 = vec + 3 * N, *s2 = vec + 4 * N, *L3 = vec + 6 * N, *s3 = vec + 7 * N;
    const double *T1 = FT, *T2 = FT + MS, *T3 = FT + 2 * MS;
    for (int i = tid; i < 3 * NN; i += NT) {
      const int pass = i / NN, rr = i - pass * NN, hi = rr / N, lo = rr - hi * N;
      double acc = 0.0;
      if (pass == 0) {          // G1[a3][a2] = sum_a1 s1[a1] E
        const int a3 = hi, a2 = lo;
        const double t1 = T1[a3 * LD + a2], x2 = s2[a2], x3 = s3[a3], base = lam + L2[a2] + L3[a3];
#pragma unroll 8
        for (int a1 = 0; a1 < N; ++a1) {
          double E = s1[a1] * t1;
          E = fma(x2, T2[a3 * LD + a1], E);
          E = fma(x3, T3[a2 * LD + a1], E);
          acc = fma(s1[a1], E * rcp_c3(base + L1[a1]), acc);
        }
      } else if (pass == 1) {   // G2[a3][a1] = sum_a2 s2[a2] E
        const int a3 = hi, a1 = lo;
        const double t2 = T2[a3 * LD + a1], x1 = s1[a1], x3 = s3[a3], base = lam + L1[a1] + L3[a3];
#pragma unroll 8
        for (int a2 = 0; a2 < N; ++a2) {
          double E = x1 * T1[a3 * LD + a2];
          E = fma(s2[a2], t2, E);
          E = fma(x3, T3[a2 * LD + a1], E);
          acc = fma(s2[a2], E * rcp_c3(base + L2[a2]), acc);
        }
      } else {                  // G3[a2][a1] = sum_a3 s3[a3] E
        const int a2 = hi, a1 = lo;
        const double t3 = T3[a2 * LD + a1], x1 = s1[a1], x2 = s2[a2], base = lam + L1[a1] + L2[a2];
#pragma unroll 8
        for (int a3 = 0; a3 < N; ++a3) {
          double E = x1 * T1[a3 * LD + a2];
          E = fma(x2, T2[a3 * LD + a1], E);
          E = fma(s3[a3], t3, E);
          acc = fma(s3[a3], E * rcp_c3(base + L3[a3]), acc);
        }
      }
      Gs[pass * MS + hi * LD + lo] = acc;
    }
  }
  __syncthreads();
  // back A: X_d = G_d S_a^T  (into FT) ; back B: U_d = S_b X_d  (into G)
  for (int job = warp; job < 3 * TPP; job += C::NW) {
    const int d = job / TPP, t = job - d * TPP, mi = t / C::TB, ni = t - mi * C::TB;
    const double* Gd = Gs + d * MS;
    const double* Sa = S[d == 0 ? 1 : 0];
    dmma_tile_fn<NP>([&](int i, int k) { return Gd[i * LD + k]; }, [&](int k, int j) { return sget(Sa, j, k); },
                     FT + d * MS, LD, mi, ni, lane);
  }
  __syncthreads();
  for (int job = warp; job < 3 * TPP; job += C::NW) {
    const int d = job / TPP, t = job - d * TPP, mi = t / C::TB, ni = t - mi * C::TB;
    const double* Xd = FT + d * MS;
    const double* Sb = S[d == 2 ? 1 : 2];
    dmma_tile_fn<NP>([&](int i, int k) { return sget(Sb, i, k); }, [&](int k, int j) { return Xd[k * LD + j]; },
                     Gs + d * MS, LD, mi, ni, lane);
  }
  __syncthreads();
  const double *w1 = vec + 2 * N, *w2 = vec + 5 * N, *w3 = vec + 8 * N;
  for (int i = tid; i < 3 * NN; i += NT) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    int j1, j2, j3;
    if (d == 0) { j1 = c; j2 = B; j3 = A; }
    else if (d == 1) { j2 = c; j1 = B; j3 = A; if (j1 == c) continue; }
    else { j3 = c; j1 = B; j2 = A; if (j1 == c || j2 == c) continue; }
    int g1 = o1 + j1, g2 = o2 + j2, g3 = o3 + j3;
    wrap_pt(g, g1, g2, g3);
    if (!is_free(g, g1, g2, g3)) continue;
    u[skel_index_t<P>(g, g1, g2, g3)] += w1[j1] * w2[j2] * w3[j3] * Gs[d * MS + A * LD + B];
  }
}

// ------------------------------------------------------------------------------------------
// star smoother, P <= 4: one WARP per star, four stars per CTA (same arithmetic and citations as
// k_star_pf: Alg. 1 + Alg. 2).  At n_S <= 7 a 128-thread star leaves most lanes idle
// in every phase; here each warp runs its star alone with __syncwarp only (no CTA barrier), the
// G3 partials of the warp's four a3 groups are reduced with two xor shuffles, and 20 stars share
// an SM.
// ------------------------------------------------------------------------------------------
template <int P> struct StarWCfg {
  static constexpr int N = 2 * P - 1, NN = N * N, C = P - 1, NP = 8, LD = 12, MS = NP * LD;
  static constexpr int SPB = 4, NT = 32 * SPB;                // stars (warps) per block
  static constexpr int GS = 8, GPW = 4, A3IT = (N + GPW - 1) / GPW;
  static constexpr int oFT = 0, oX = 3 * MS, oG = 6 * MS, oS = 9 * MS, oU = 12 * MS, oVec = oU + 3 * NN,
                       oBase = oVec + 9 * N, per_star = oBase + 8, oMap = SPB * per_star, total = oMap + (3 * NN + 1) / 2;
};

template <int P>
size_t star_w_smem() { return sizeof(double) * StarWCfg<P>::total; }

template <int P>
__global__ void __launch_bounds__(128) k_star_w(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c, long long nstars,
                                               const double* __restrict__ r, double* __restrict__ u,
                                               const double* __restrict__ stab, double lam) {
  using C = StarWCfg<P>;
  constexpr int N = C::N, NN = C::NN, c = C::C, NP = C::NP, LD = C::LD, MS = C::MS, GS = C::GS;
  extern __shared__ double smem_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sm = smem_all + warp * C::per_star;
  // the point map in shared memory, shared by the block's four stars (before any early exit)
  unsigned* map_s = reinterpret_cast<unsigned*>(smem_all + C::oMap);
  for (int i = threadIdx.x; i < 3 * NN; i += C::NT) map_s[i] = __ldg(&kStarMap<P>.v[i]);
  __syncthreads();
  const long long b = (long long)blockIdx.x * C::SPB + warp;
  if (b >= nstars) return;
  const int i1 = (int)(b % n1c), rest = (int)(b / n1c), i2 = rest % n2c, i3 = rest / n2c;
  const int v1 = c1 + 2 * i1, v2 = c2 + 2 * i2, v3 = c3 + 2 * i3;
  if (star_empty(g, v1, v2, v3)) return;
  if (v3 < g.own_lo) return;
  const int ST = g.ST;
  double* FT = sm + C::oFT;
  double* X = sm + C::oX;
  double* Gs = sm + C::oG;
  double* Ssm = sm + C::oS;
  double* Up = sm + C::oU;
  double* vec = sm + C::oVec;
  constexpr int RS = 3 * (P - 1) * (P - 1) + 3 * (P - 1) + 1;
  const long long V12 = (long long)g.V1 * g.V2;
  const long long rec0 = v1 + g.V1 * (long long)v2 + V12 * v3;
  const bool interior = ((v1 > 0 && v1 < g.k1) || (g.per & 1)) && ((v2 > 0 && v2 < g.k2) || (g.per & 2)) &&
                        ((v3 > 0 && v3 + g.zoff < g.K3) || (g.per & 4));
  auto pt_free = [&](unsigned e) {   // global test (w3 + zoff is the global record plane), Neumann faces free
    const int w1 = v1 - (int)((e >> 12) & 1u), w2 = v2 - (int)((e >> 13) & 1u), w3 = v3 - (int)((e >> 14) & 1u);
    const int W3 = w3 + g.zoff;
    // the point is G_d = w_d p + t_d (0 <= t_d < p), t_d == 0 iff bit 15 + d
    const bool z1 = e & (1u << 15), z2 = e & (1u << 16), z3 = e & (1u << 17);
    return ((g.per & 1) || (w1 >= 0 && (w1 > 0 || !z1 || (g.neu & 1)) && (w1 < g.k1 || (z1 && w1 == g.k1 && (g.neu & 2))))) &&
           ((g.per & 2) || (w2 >= 0 && (w2 > 0 || !z2 || (g.neu & 4)) && (w2 < g.k2 || (z2 && w2 == g.k2 && (g.neu & 8))))) &&
           ((g.per & 4) || (w3 >= 0 && (W3 > 0 || !z3 || (g.neu & 16)) && (W3 < g.K3 || (z3 && W3 == g.K3 && (g.neu & 32)))));
  };
  long long* s_base = reinterpret_cast<long long*>(sm + C::oBase);
  if (lane < 8) {
    const int b1 = lane & 1, b2 = (lane >> 1) & 1, b3 = (lane >> 2) & 1;
    const bool ok = !((v1 == 0 && b1 && !(g.per & 1)) || (v2 == 0 && b2 && !(g.per & 2)) || (v3 == 0 && b3 && !(g.per & 4)));
    const int w1 = wrap_rec(v1 - b1, g.k1, g.per & 1), w2 = wrap_rec(v2 - b2, g.k2, g.per & 2),
              w3 = wrap_rec(v3 - b3, g.k3, g.per & 4);   // periodic: record k-1 for v = 0
    s_base[lane] = ok ? (w1 + g.V1 * (long long)w2 + V12 * w3) * RS : -1LL;
  }
  const size_t srow[3] = {(size_t)v1 * ST, (size_t)(g.V1 + v2) * ST, (size_t)(g.V1 + g.V2 + v3) * ST};
  for (int i = lane; i < 3 * NN; i += 32) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    cp_async8(&Ssm[d * MS + A * LD + B], &stab[srow[d] + rr], true);
  }
  for (int i = lane; i < 9 * N; i += 32) { const int d = i / (3 * N); cp_async8(&vec[i], &stab[srow[d] + NN + i - d * 3 * N], true); }
  pdl_wait();
  pdl_trigger();
  __syncwarp();
  for (int i = lane; i < 3 * NN; i += 32) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    const unsigned e = map_s[i];
    const long long base = s_base[(e >> 12) & 7u];
    const bool ok = base >= 0;
    cp_async8(&FT[d * MS + A * LD + B], &r[ok ? base + (e & 0xFFFu) : 0], ok);
  }
  cp_async_commit();
  for (int i = lane; i < 3 * NN; i += 32) {
    const unsigned e = map_s[i];
    const long long base = s_base[(e >> 12) & 7u];
    const bool ok = base >= 0 && (interior || pt_free(e));
    cp_async8(&Up[i], &u[ok ? base + (e & 0xFFFu) : 0], ok);
  }
  cp_async_commit();
  constexpr int PADN = NP * NP - NN, PC = NP - N;
  for (int i = lane; i < 3 * PADN; i += 32) {
    const int d = i / PADN, k = i - d * PADN;
    int A, B;
    if (k < N * PC) { A = k / PC; B = N + (k - A * PC); }
    else { const int k2 = k - N * PC; A = N + k2 / NP; B = k2 - (A - N) * NP; }
    const int o = d * MS + A * LD + B;
    FT[o] = 0.0;
    Ssm[o] = 0.0;
    Gs[o] = 0.0;
  }
  cp_async_wait<1>();
  __syncwarp();
  for (int i = lane; i < 3 * 2 * N; i += 32) {   // inverse multiplicity
    const int d = i / (2 * N), rr = i - d * 2 * N, line = rr / N, t = rr - line * N;
    const int A = line ? t : c, B = line ? c : t;
    if (line && t == c) continue;
    FT[d * MS + A * LD + B] *= 1.0 / (double)(1 + (A == c) + (B == c));
  }
  __syncwarp();
#pragma unroll
  for (int d = 0; d < 3; ++d) dmma_tile_t<NP, LD, false, false>(FT + d * MS, Ssm + (d == 0 ? 1 : 0) * MS, X + d * MS, 0, 0, lane);
  __syncwarp();
#pragma unroll
  for (int d = 0; d < 3; ++d) dmma_tile_t<NP, LD, true, false>(Ssm + (d == 2 ? 1 : 2) * MS, X + d * MS, FT + d * MS, 0, 0, lane);
  __syncwarp();
  {
    const double *L1 = vec, *s1 = vec + N, *L2 = vec + 3 * N, *s2 = vec + 4 * N, *L3 = vec + 6 * N, *s3 = vec + 7 * N;
    const double *T1 = FT, *T2 = FT + MS, *T3 = FT + 2 * MS;
    const int grp = lane / GS, a1 = lane % GS;
    const bool va = a1 < N;
    const int a1c = va ? a1 : 0;
    const double s1a = va ? s1[a1c] : 0.0, L1a = L1[a1c];
    double g3[N];
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2) g3[a2] = 0.0;
#pragma unroll
    for (int k = 0; k < C::A3IT; ++k) {
      const int a3 = grp + k * C::GPW;
      const bool act = a3 < N;
      const int a3c = act ? a3 : 0;
      const double on = (act && va) ? 1.0 : 0.0;
      const double t2 = on * T2[a3c * LD + a1c], s3v = on * s3[a3c], base = lam + L1a + L3[a3c];
      const double s1v = on * s1a;
      double g2 = 0.0;
      double v[GS];
#pragma unroll
      for (int a2 = 0; a2 < GS; ++a2) v[a2] = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        double E = s1v * T1[a3c * LD + a2];
        E = fma(s2[a2], t2, E);
        E = fma(s3v, T3[a2 * LD + a1c], E);
        const double V = E * rcp_nr(base + L2[a2]);
        g2 = fma(s2[a2], V, g2);
        g3[a2] = fma(s3v, V, g3[a2]);
        v[a2] = s1v * V;
      }
#pragma unroll
      for (int off = GS / 2; off >= 1; off >>= 1) {
        const bool upper = (a1 & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
          const double send = upper ? v[j] : v[j + off];
          const double keep = upper ? v[j + off] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (act && va) {
        Gs[a3 * LD + a1] = v[0];
        Gs[MS + a3 * LD + a1] = g2;
      }
    }
#pragma unroll
    for (int off = GS; off < 32; off <<= 1) {
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) g3[a2] += __shfl_xor_sync(0xffffffffu, g3[a2], off);
    }
    if (va && lane < GS) {
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) Gs[2 * MS + a2 * LD + a1] = g3[a2];
    }
  }
  __syncwarp();
#pragma unroll
  for (int d = 0; d < 3; ++d) dmma_tile_t<NP, LD, false, true>(Gs + d * MS, Ssm + (d == 0 ? 1 : 0) * MS, X + d * MS, 0, 0, lane);
  __syncwarp();
#pragma unroll
  for (int d = 0; d < 3; ++d) dmma_tile_t<NP, LD, false, false>(Ssm + (d == 2 ? 1 : 2) * MS, X + d * MS, Gs + d * MS, 0, 0, lane);
  cp_async_wait<0>();
  __syncwarp();
  const double *w1 = vec + 2 * N, *w2 = vec + 5 * N, *w3 = vec + 8 * N;
  for (int i = lane; i < 3 * NN; i += 32) {
    const int d = i / NN, rr = i - d * NN, A = rr / N, B = rr - A * N;
    int j1, j2, j3;
    if (d == 0) { j1 = c; j2 = B; j3 = A; }
    else if (d == 1) { j2 = c; j1 = B; j3 = A; if (j1 == c) continue; }
    else { j3 = c; j1 = B; j2 = A; if (j1 == c || j2 == c) continue; }
    const unsigned e = map_s[i];
    if (!interior && !pt_free(e)) continue;
    u[s_base[(e >> 12) & 7u] + (e & 0xFFFu)] = fma(w1[j1] * w2[j2] * w3[j3], Gs[d * MS + A * LD + B], Up[i]);
  }
}

// ------------------------------------------------------------------------------------------
// star smoother at p = 2 (n_S = 3: 27-point stars, 19 skeleton points): one THREAD per star.  The
// same arithmetic as k_star_w (Alg. 1 + Alg. 2, reading R19): the three 3 x 3 planes
// through the vertex with the inverse multiplicity on the two lines through it, the
// forward transforms T_d = S_slow^T F_d S_fast, the fused core over the 27 eigen-triples
// V = E / (lambda + L1 + L2 + L3), the back transforms and the weighted scatter-add -- all in
// registers, with the compile-time point map folded into immediates.  A warp per 27-point star
// (k_star_w) left most lanes idle: the p = 2 sweep ran at 1.6 % of the HBM bound.
// ------------------------------------------------------------------------------------------
#ifndef PMG_STARP2_MINB
#define PMG_STARP2_MINB 3   // 168 registers, small spills: 0.83 -> 0.75 ms per sweep at 128^3 elements
#endif
__global__ void __launch_bounds__(128, PMG_STARP2_MINB) k_star_p2(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c, long long nstars,
                                                const double* __restrict__ r, double* __restrict__ u,
                                                const double* __restrict__ stab, double lam) {
  constexpr int P = 2, N = 3, NN = 9, c = 1, RS = 7;
  constexpr StarMap<P> map = make_star_map<P>();
  pdl_wait();
  pdl_trigger();
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= nstars) return;
  const int i1 = (int)(b % n1c), rest = (int)(b / n1c), i2 = rest % n2c, i3 = rest / n2c;
  const int v1 = c1 + 2 * i1, v2 = c2 + 2 * i2, v3 = c3 + 2 * i3;
  if (star_empty(g, v1, v2, v3)) return;
  if (v3 < g.own_lo) return;
  const long long V12 = (long long)g.V1 * g.V2;
  const bool interior = ((v1 > 0 && v1 < g.k1) || (g.per & 1)) && ((v2 > 0 && v2 < g.k2) || (g.per & 2)) &&
                        ((v3 > 0 && v3 + g.zoff < g.K3) || (g.per & 4));
  auto pt_free = [&](unsigned e) {   // as k_star_w
    const int w1 = v1 - (int)((e >> 12) & 1u), w2 = v2 - (int)((e >> 13) & 1u), w3 = v3 - (int)((e >> 14) & 1u);
    const int W3 = w3 + g.zoff;
    const bool z1 = e & (1u << 15), z2 = e & (1u << 16), z3 = e & (1u << 17);
    return ((g.per & 1) || (w1 >= 0 && (w1 > 0 || !z1 || (g.neu & 1)) && (w1 < g.k1 || (z1 && w1 == g.k1 && (g.neu & 2))))) &&
           ((g.per & 2) || (w2 >= 0 && (w2 > 0 || !z2 || (g.neu & 4)) && (w2 < g.k2 || (z2 && w2 == g.k2 && (g.neu & 8))))) &&
           ((g.per & 4) || (w3 >= 0 && (W3 > 0 || !z3 || (g.neu & 16)) && (W3 < g.K3 || (z3 && W3 == g.K3 && (g.neu & 32)))));
  };
  long long base[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int b1 = q & 1, b2 = (q >> 1) & 1, b3 = (q >> 2) & 1;
    const bool ok = !((v1 == 0 && b1 && !(g.per & 1)) || (v2 == 0 && b2 && !(g.per & 2)) || (v3 == 0 && b3 && !(g.per & 4)));
    const int w1 = wrap_rec(v1 - b1, g.k1, g.per & 1), w2 = wrap_rec(v2 - b2, g.k2, g.per & 2),
              w3 = wrap_rec(v3 - b3, g.k3, g.per & 4);
    base[q] = ok ? (w1 + g.V1 * (long long)w2 + V12 * w3) * RS : -1LL;
  }
  const double* St[3] = {stab + (size_t)v1 * g.ST, stab + (size_t)(g.V1 + v2) * g.ST, stab + (size_t)(g.V1 + g.V2 + v3) * g.ST};
  // gather the three planes (inverse multiplicity on the lines through the vertex)
  double F[3][NN];
#pragma unroll
  for (int i = 0; i < 3 * NN; ++i) {
    const int d = i / NN, A = (i % NN) / N, B = i % N;
    const unsigned e = map.v[i];
    const long long bb = base[(e >> 12) & 7u];
    const double x = bb >= 0 ? __ldg(&r[bb + (e & 0xFFFu)]) : 0.0;
    F[d][A * N + B] = x * (1.0 / (double)(1 + (A == c) + (B == c)));
  }
  // forward transforms: T_d[a][b] = sum_{A,B} S_slow[A][a] F_d[A][B] S_fast[B][b]
  // (plane 0: A = j3, B = j2; plane 1: A = j3, B = j1; plane 2: A = j2, B = j1)
  double T[3][NN];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double* Sf = St[d == 0 ? 1 : 0];
    const double* Ss = St[d == 2 ? 1 : 2];
    double X[NN];
#pragma unroll
    for (int A = 0; A < N; ++A)
#pragma unroll
      for (int bq = 0; bq < N; ++bq) {
        double x = 0.0;
#pragma unroll
        for (int B = 0; B < N; ++B) x = fma(F[d][A * N + B], __ldg(&Sf[B * N + bq]), x);
        X[A * N + bq] = x;
      }
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int bq = 0; bq < N; ++bq) {
        double t = 0.0;
#pragma unroll
        for (int A = 0; A < N; ++A) t = fma(__ldg(&Ss[A * N + a]), X[A * N + bq], t);
        T[d][a * N + bq] = t;
      }
  }
  // core over the eigen-triples: T1 = T[0][a3][a2], T2 = T[1][a3][a1], T3 = T[2][a2][a1]
  double Lm[3][N], sv[3][N];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int a = 0; a < N; ++a) {
      Lm[d][a] = __ldg(&St[d][NN + a]);
      sv[d][a] = __ldg(&St[d][NN + N + a]);
    }
  double G[3][NN];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int k = 0; k < NN; ++k) G[d][k] = 0.0;
#pragma unroll
  for (int a3 = 0; a3 < N; ++a3)
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2)
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        double E = sv[0][a1] * T[0][a3 * N + a2];
        E = fma(sv[1][a2], T[1][a3 * N + a1], E);
        E = fma(sv[2][a3], T[2][a2 * N + a1], E);
        const double V = E * rcp_nr(lam + Lm[0][a1] + Lm[1][a2] + Lm[2][a3]);
        G[0][a3 * N + a2] = fma(sv[0][a1], V, G[0][a3 * N + a2]);
        G[1][a3 * N + a1] = fma(sv[1][a2], V, G[1][a3 * N + a1]);
        G[2][a2 * N + a1] = fma(sv[2][a3], V, G[2][a2 * N + a1]);
      }
  // back transforms U_d[A][B] = sum_{a,b} S_slow[A][a] G_d[a][b] S_fast[B][b], weighted scatter-add
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double* Sf = St[d == 0 ? 1 : 0];
    const double* Ss = St[d == 2 ? 1 : 2];
    double X[NN];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int B = 0; B < N; ++B) {
        double x = 0.0;
#pragma unroll
        for (int bq = 0; bq < N; ++bq) x = fma(G[d][a * N + bq], __ldg(&Sf[B * N + bq]), x);
        X[a * N + B] = x;
      }
#pragma unroll
    for (int A = 0; A < N; ++A)
#pragma unroll
      for (int B = 0; B < N; ++B) {
        int j1, j2, j3;
        if (d == 0) { j1 = c; j2 = B; j3 = A; }
        else if (d == 1) { j2 = c; j1 = B; j3 = A; if (j1 == c) continue; }
        else { j3 = c; j1 = B; j2 = A; if (j1 == c || j2 == c) continue; }
        const unsigned e = map.v[d * NN + A * N + B];
        const long long bb = base[(e >> 12) & 7u];
        if (bb < 0 || !(interior || pt_free(e))) continue;
        double uu = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) uu = fma(__ldg(&Ss[A * N + a]), X[a * N + B], uu);
        const double w = __ldg(&St[0][NN + 2 * N + j1]) * __ldg(&St[1][NN + 2 * N + j2]) * __ldg(&St[2][NN + 2 * N + j3]);
        double* dst = &u[bb + (e & 0xFFFu)];
        *dst = fma(w, uu, *dst);
      }
  }
}

// ------------------------------------------------------------------------------------------
// residual gather, degree-templated: one block per vertex record (3-D grid, no index division),
// one thread per record slot.  Same sums in the same order as k_gather_resid (kernels.cu):
// r = F - sum over the elements sharing the point of their outputs Y.
// ------------------------------------------------------------------------------------------
template <int P> struct GatherCfg {
  static constexpr int RS = 3 * (P - 1) * (P - 1) + 3 * (P - 1) + 1;
  static constexpr int R = RS >= 128 ? 1 : 256 / RS;                        // records per block
  static constexpr int NT = R > 1 ? 256 : (RS < 64 ? 64 : (RS < 128 ? 128 : 256));
};

template <int P>
__global__ void __launch_bounds__(256) k_gather_resid_t(LevelGeom g, const double* __restrict__ Y,
                                                        const double* __restrict__ F, double* __restrict__ out,
                                                        const int* __restrict__ done) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  constexpr int m = P - 1, mm = m * m, RS = 3 * mm + 3 * m + 1, YS = 6 * mm + 12 * m + 8;
  // R consecutive records along x1 per block (low degrees: a record has only 7 ... 127 slots); their
  // R x RS slots are one contiguous range of the skeleton vector
  constexpr int R = GatherCfg<P>::R;
  const int v2 = blockIdx.y, v3 = blockIdx.z, v1b = blockIdx.x * R;
  const bool own = owned_plane(g, v3);
  // Y offsets of the (up to) 8 elements around vertex v: bit d of c set = element v_d along d, clear =
  // element v_d - 1 (periodic: wrapped); -1 outside the box (Neumann faces have one side)
  __shared__ long long ebs[R][8];
  for (int i = threadIdx.x; i < 8 * R; i += blockDim.x) {
    const int c = i & 7, v1 = v1b + (i >> 3);
    int a1 = v1 - 1 + (c & 1), a2 = v2 - 1 + ((c >> 1) & 1), a3 = v3 - 1 + ((c >> 2) & 1);
    a1 = wrap_rec(a1, g.k1, g.per & 1);
    a2 = wrap_rec(a2, g.k2, g.per & 2);
    a3 = wrap_rec(a3, g.k3, g.per & 4);
    const bool in = a1 >= 0 && a2 >= 0 && a3 >= 0 && a1 < g.k1 && a2 < g.k2 && a3 < g.k3;
    ebs[i >> 3][c] = in ? ((long long)a1 + (long long)g.k1 * ((long long)a2 + (long long)g.k2 * a3)) * YS : -1LL;
  }
  __syncthreads();
  const long long rec0 = v1b + (long long)g.V1 * (v2 + (long long)g.V2 * v3);
  const int nrec = min(R, g.V1 - v1b);
  for (int j = threadIdx.x; j < nrec * RS; j += blockDim.x) {
  const int ri = j / RS, o = j - ri * RS, v1 = v1b + ri;
  const long long rec = rec0 + ri;
  const long long* eb = ebs[ri];
  auto yat = [&](int c, int off) -> double { const long long b_ = eb[c]; return b_ >= 0 ? Y[b_ + off] : 0.0; };
  {
    int t1 = 0, t2 = 0, t3 = 0, type, a = 0, b = 0;
    if (o < 3 * mm) {
      type = o / mm;
      const int rr = o - type * mm;
      a = rr / m; b = rr - a * m;
      if (type == 0) { t3 = a + 1; t2 = b + 1; } else if (type == 1) { t3 = a + 1; t1 = b + 1; } else { t2 = a + 1; t1 = b + 1; }
    } else if (o < 3 * mm + 3 * m) {
      const int rr = o - 3 * mm, d = rr / m;
      type = 3 + d;
      a = rr - d * m;
      if (d == 0) t1 = a + 1; else if (d == 1) t2 = a + 1; else t3 = a + 1;
    } else {
      type = 6;
    }
    double r = 0.0;
    if (own && is_free(g, v1 * P + t1, v2 * P + t2, v3 * P + t3)) {
      double s_ = 0.0;
      if (type < 3) {            // face normal to d: the element below along d (its high face) and v's
        const int d = type, oo = a * m + b;
        s_ = yat(7 & ~(1 << d), (2 * d + 1) * mm + oo) + yat(7, (2 * d) * mm + oo);
      } else if (type < 6) {     // edge along d: the four elements around it
        const int d = type - 3, da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
        for (int bB = 0; bB < 2; ++bB)
          for (int bA = 0; bA < 2; ++bA) {
            const int qe = 4 * d + (1 - bA) + 2 * (1 - bB);
            s_ += yat((1 << d) | (bA << da) | (bB << db), 6 * mm + qe * m + a);
          }
      } else {                   // vertex: the eight elements
        for (int c3 = 0; c3 < 2; ++c3)
          for (int c2 = 0; c2 < 2; ++c2)
            for (int c1 = 0; c1 < 2; ++c1) {
              const int qv = (1 - c1) + 2 * (1 - c2) + 4 * (1 - c3);
              s_ += yat(c1 | (c2 << 1) | (c3 << 2), 6 * mm + 12 * m + qv);
            }
      }
      r = F ? F[rec * RS + o] - s_ : s_;
    }
    out[rec * RS + o] = r;
  }
  }
}

// ------------------------------------------------------------------------------------------
// dispatch: one production kernel per degree range
//   element operator: k_elem_pf (p <= 8), k_elem16 (9..16, elem16.cu), k_elem_apply_t (17..32)
//   star smoother:    k_star_w (p <= 4 and >= star_w_min stars per colour), k_star_pf (p <= 4),
//                     k_star16 (5..16, star16.cu), k_star_tm (17..32)
// ------------------------------------------------------------------------------------------
// stars per colour from which k_star_w (warp per star, p <= 4) replaces k_star_pf; PMG_STAR_W_MIN
// overrides the default (tests force the kernel onto small parity meshes with 0)
static long long star_w_min(long long dflt) {
  const char* e = std::getenv("PMG_STAR_W_MIN");
  return (e && e[0]) ? std::atoll(e) : dflt;
}

template <int P>
cudaError_t launch_elem_p(const LevelGeom& g, const double* u, const double* etab, const double* etabP, double lam,
                          double* Y, const int* done, cudaStream_t st) {
  if constexpr (P <= 8)
    return launch_pdl(k_elem_pf<P>, dim3((unsigned)g.nelem), dim3(ElemPfCfg<P>::NT), elem_pf_smem<P>(), st, g, u, etab, lam,
                      Y, done);
  else if constexpr (P <= 16)
    return launch_elem16(g, u, etabP, lam, Y, done, st);
  else
    return launch_pdl(k_elem_apply_t<P>, dim3((unsigned)g.nelem), dim3(ElemCfg<P>::NT), elem_t_smem<P>(), st, g, u, etab,
                      lam, Y, done);
}

template <int P>
cudaError_t launch_star_p(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                          double* u, const double* stab, const double* stabP, double lam, cudaStream_t st) {
  if constexpr (P >= 5 && P <= 16) {
    return launch_star16(g, c1, c2, c3, n1c, n2c, nb, r, u, stabP, lam, st);
  } else if constexpr (P == 2) {
    return launch_pdl(k_star_p2, dim3((unsigned)((nb + 127) / 128)), dim3(128), 0, st, g, c1, c2, c3, n1c, n2c, nb, r, u,
                      stab, lam);
  } else if constexpr (P <= 4) {
    {
      // warp per star pays off once a colour has many waves of 128-thread stars (large meshes);
      // for a few hundred stars the shorter per-star chain of k_star_pf wins (measured, config 2)
      if (nb >= star_w_min(4LL * 148 * StarPfCfg<P>::MINB))
        return launch_pdl(k_star_w<P>, dim3((unsigned)((nb + StarWCfg<P>::SPB - 1) / StarWCfg<P>::SPB)),
                          dim3(StarWCfg<P>::NT), star_w_smem<P>(), st, g, c1, c2, c3, n1c, n2c, nb, r, u, stab, lam);
    }
    return launch_pdl(k_star_pf<P>, dim3((unsigned)nb), dim3(StarPfCfg<P>::NT), star_pf_smem<P>(), st, g, c1, c2, c3, n1c,
                      n2c, r, u, stab, lam);
  } else {
    return launch_pdl(k_star_tm<P>, dim3((unsigned)nb), dim3(StarTmCfg<P>::NT), star_tm_smem<P>(), st, g, c1, c2, c3, n1c,
                      n2c, r, u, stab, lam);
  }
}

#define PMG_DEGREES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)

cudaError_t launch_elem_apply(const LevelGeom& g, const double* u, const double* etab, const double* etabP, double lam,
                              double* Y, const int* done, cudaStream_t st) {
  switch (g.p) {
#define CASE(P) \
  case P: return launch_elem_p<P>(g, u, etab, etabP, lam, Y, done, st);
    PMG_DEGREES(CASE)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gather_resid(const LevelGeom& g, const double* Y, const double* F, double* out, const int* done,
                                cudaStream_t st) {
  switch (g.p) {
#define CASE(P)                                                                                     \
  case P: {                                                                                         \
    constexpr int R = GatherCfg<P>::R;                                                              \
    const dim3 grid((unsigned)((g.V1 + R - 1) / R), (unsigned)g.V2, (unsigned)g.V3);                \
    return launch_pdl(k_gather_resid_t<P>, grid, dim3(GatherCfg<P>::NT), 0, st, g, Y, F, out, done); \
  }
    PMG_DEGREES(CASE)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_star(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                        double* u, const double* stab, const double* stabP, double lam, cudaStream_t st) {
  switch (g.p) {
#define CASE(P) \
  case P: return launch_star_p<P>(g, c1, c2, c3, n1c, n2c, nb, r, u, stab, stabP, lam, st);
    PMG_DEGREES(CASE)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

// dynamic shared memory of the production kernels (which 0: element operator, 1: star smoother;
// the p = 9..16 kernels have fixed footprints set in star16.cu / elem16.cu)
size_t hot_smem(int p, int which) {
  switch (p) {
#define CASE(P)                                                                                              \
  case P:                                                                                                    \
    if (which == 0) return P <= 8 ? elem_pf_smem<(P <= 8 ? P : 2)>() : (P > 16 ? elem_t_smem<P>() : 0);      \
    return P <= 4 ? std::max(star_pf_smem<(P <= 4 ? P : 2)>(), star_w_smem<(P <= 4 ? P : 2)>())            \
                  : (P > 16 ? star_tm_smem<(P > 16 ? P : 17)>() : 0);
    PMG_DEGREES(CASE)
#undef CASE
    default: return 0;
  }
}

cudaError_t hot_set_smem_attr(int bytes) {
  cudaError_t e = cudaSuccess;
#define SET(K)                                                                        \
  {                                                                                   \
    cudaError_t a = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
    if (a != cudaSuccess) e = a;                                                      \
  }
#define CASE8(P) SET(k_elem_pf<P>)
#define CASE4(P) SET(k_star_w<P>) SET(k_star_pf<P>)
#define CASE32(P) SET(k_elem_apply_t<P>) SET(k_star_tm<P>)
  CASE8(2) CASE8(3) CASE8(4) CASE8(5) CASE8(6) CASE8(7) CASE8(8)
  CASE4(2) CASE4(3) CASE4(4)
  CASE32(17) CASE32(18) CASE32(19) CASE32(20) CASE32(21) CASE32(22) CASE32(23) CASE32(24) CASE32(25) CASE32(26)
  CASE32(27) CASE32(28) CASE32(29) CASE32(30) CASE32(31) CASE32(32)
#undef CASE8
#undef CASE4
#undef CASE32
#undef SET
  return e;
}

}  // namespace pmg
