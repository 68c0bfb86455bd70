// Star smoother for 9 <= p <= 16: Alg. 2 with the Alg. 1 star inverse (P:294-305,
// reading R2-R4, R7), one CTA of 4 warps per star, three CTAs resident per SM.
//
// Same arithmetic as k_star_pf (hot_kernels.cu), re-planned for occupancy (ncu, round 2 start:
// k_star_pf<16> held one 256-thread CTA per SM, 12 % achieved occupancy, 16.6 % FP64 pipe, and
// spent half its instructions in the gather / scatter index arithmetic):
//   - shared memory per CTA is 7 padded n_S x n_S matrices (66.8 KB at p = 16): the three star
//     planes F_d, which become T_d after the forward transforms, then G_d (the core writes
//     G1[a3][:] over T1[a3][:] and G2[a3][:] over T2[a3][:], rows only the writing warp reads),
//     then U_d; the three S_d; one transform scratch X (the faces are transformed one at a time);
//   - the transforms are DMMA GEMMs with 2 x 2 (n_S padded to 32) or 1 x 2 tile blocks per warp
//     (one shared-memory fragment load per DMMA at 2 x 2), operands padded to a multiple of 8;
//   - the star table is read in a padded layout (S as NP x NP, zero padding; Lambda padded with 1)
//     with 16-byte cp.async, so no padding loop runs per star;
//   - gather and scatter walk the star's 12 face-interior blocks (contiguous (p-1)^2 runs of the
//     vertex records) and its 3 vertex lines with per-block base tables: a few
//     integer operations per point;
//   - core: lanes own a1, each warp two a3 values per pass (shared loads of s2, Lambda2 and the T3
//     row serve both), a2 in registers; G2 accumulates in a register, G3 over the warp's passes in
//     registers and then over the 4 warps in a fixed-order tree, G1 by a butterfly reduce-scatter
//     of the 16 values of an a2 chunk of both a3 (one 64-bit shuffle per value);
//   - 1/D by rcp.approx and one cubic Newton step, r (1 + e + e^2), e = 1 - D r (error e^3).
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {
namespace {

__device__ __forceinline__ double rcp3(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cpa16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K)); }

}  // namespace

template <int P> struct Star16 {
  static constexpr int N = 2 * P - 1, NN = N * N, C = P - 1, M = P - 1, MM = M * M;
  static constexpr int NP = (N + 7) / 8 * 8;          // 16 (p <= 8), 24 (p <= 12) or 32
  static constexpr int LD = NP + 4;                    // = 4 or 12 mod 16: conflict-free fragment loads
  static constexpr int MS = NP * LD;
  static constexpr int NT = 128, NW = 4;
  // core lane groups: GS lanes own a1 (16 for n_S <= 16, else the whole warp); NG groups per CTA
  static constexpr int GS = NP <= 16 ? 16 : 32, NG = NW * (32 / GS);
  static constexpr int MINB = NP <= 16 ? 5 : 3;       // CTAs per SM (registers / shared memory)
  static constexpr int STP = NP * NP + 3 * NP;         // padded star-table row
  static constexpr int RS = 3 * MM + 3 * M + 1;
  // shared memory (doubles): planes, S, X, vectors (Lambda, s, w per direction, NP each), 8 record
  // bases, 12 face-block sources, 6 line sources (lower / upper segment of each vertex line)
  static constexpr int oR = 0, oS = 3 * MS, oX = 6 * MS, oVec = 7 * MS, oBase = oVec + 9 * NP,
                       oFb = oBase + 8, oLb = oFb + 12, total = oLb + 6;
};

template <int P>
size_t star16_smem() { return sizeof(double) * Star16<P>::total; }

// C = op(A) op(B) for NP x NP shared-memory matrices (leading dimension LD), 4 warps
template <int NP, int LD, bool TA, bool TB>
__device__ __forceinline__ void gemm4(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ Cm,
                                      int warp, int lane) {
  // tile blocks per job: 2 x 2 at n_S padded to 32 (4 jobs), 1 x 2 at 24 (6 jobs), 1 x 1 at 16 (4 jobs)
  constexpr int T = NP / 8, BR = (T >= 4 && T % 2 == 0) ? 2 : 1, BC = T >= 3 ? 2 : 1, JC = (T + BC - 1) / BC,
                NJ = (T / BR) * JC;
  const int r = lane >> 2, q = lane & 3;
  for (int job = warp; job < NJ; job += 4) {
    const int mi0 = (job / JC) * BR, ni0 = (job % JC) * BC;
    double c[BR][BC][2];
#pragma unroll
    for (int i = 0; i < BR; ++i)
#pragma unroll
      for (int j = 0; j < BC; ++j) c[i][j][0] = c[i][j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NP / 4; ++kk) {
      const int k = 4 * kk + q;
      double a[BR], b[BC];
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        const int ii = 8 * (mi0 + i) + r;
        a[i] = TA ? A[k * LD + ii] : A[ii * LD + k];
      }
#pragma unroll
      for (int j = 0; j < BC; ++j) {
        const int jj = 8 * (ni0 + j) + r;
        b[j] = (ni0 + j < T) ? (TB ? B[jj * LD + k] : B[k * LD + jj]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < BR; ++i)
#pragma unroll
        for (int j = 0; j < BC; ++j)
          if (ni0 + j < T) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < BR; ++i)
#pragma unroll
      for (int j = 0; j < BC; ++j)
        if (ni0 + j < T) {
          double2* dst = reinterpret_cast<double2*>(Cm + (8 * (mi0 + i) + r) * LD + 8 * (ni0 + j) + 2 * q);
          *dst = make_double2(c[i][j][0], c[i][j][1]);
        }
  }
}

template <int P>
__global__ void __launch_bounds__(128, Star16<P>::MINB)
    k_star16(LevelGeom g, int c1, int c2, int c3, int n1c, int n2c, const double* __restrict__ r,
             double* __restrict__ u, const double* __restrict__ stabP, double lam) {
  using K = Star16<P>;
  constexpr int N = K::N, NN = K::NN, C = K::C, M = K::M, MM = K::MM, NP = K::NP, LD = K::LD, MS = K::MS, NT = K::NT,
                STP = K::STP, RS = K::RS;
  extern __shared__ double sm[];
  const int v1 = c1 + 2 * (int)blockIdx.x, v2 = c2 + 2 * (int)blockIdx.y, v3 = c3 + 2 * (int)blockIdx.z;   // 3-D grid
  if (star_empty(g, v1, v2, v3)) return;
  if (v3 < g.own_lo) return;   // ghost star below the slab: computed by the lower rank
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* R = sm + K::oR;
  double* Ssm = sm + K::oS;
  double* X = sm + K::oX;
  double* vec = sm + K::oVec;
  long long* base = reinterpret_cast<long long*>(sm + K::oBase);
  long long* fb = reinterpret_cast<long long*>(sm + K::oFb);
  long long* lb = reinterpret_cast<long long*>(sm + K::oLb);
  const long long V12 = (long long)g.V1 * g.V2;
  // ---- setup tables (before the dependency wait): S_d padded NP x NP, then Lambda, s, w
  {
    auto row = [&](int d) -> size_t {   // star-table row of the vertex line along direction d
      return d == 0 ? (size_t)v1 : (d == 1 ? (size_t)(g.V1 + v2) : (size_t)(g.V1 + g.V2 + v3));
    };
    constexpr int CH = NP / 2;   // 16-byte chunks per row
    for (int i = tid; i < 3 * NP * CH; i += NT) {
      const int d = i / (NP * CH), rr = i - d * NP * CH, A = rr / CH, ch = rr - A * CH;
      cpa16(&Ssm[d * MS + A * LD + 2 * ch], stabP + row(d) * STP + A * NP + 2 * ch);
    }
    for (int i = tid; i < 3 * (3 * NP / 2); i += NT) {
      const int d = i / (3 * NP / 2), ch = i - d * (3 * NP / 2);
      cpa16(&vec[d * 3 * NP + 2 * ch], stabP + row(d) * STP + NP * NP + 2 * ch);
    }
    cpa_commit();
  }
  if (tid < 8) {   // record (v - b) for offset bits b = (b1, b2, b3); -1 if outside the stored box
    const int b1 = tid & 1, b2 = (tid >> 1) & 1, b3 = (tid >> 2) & 1;
    const bool ok = !((v1 == 0 && b1 && !(g.per & 1)) || (v2 == 0 && b2 && !(g.per & 2)) || (v3 == 0 && b3 && !(g.per & 4)));
    const int w1 = wrap_rec(v1 - b1, g.k1, g.per & 1), w2 = wrap_rec(v2 - b2, g.k2, g.per & 2),
              w3 = wrap_rec(v3 - b3, g.k3, g.per & 4);   // periodic: record k - 1 for v = 0
    base[tid] = ok ? (w1 + g.V1 * (long long)w2 + V12 * w3) * RS : -1LL;
  }
  __syncthreads();
  if (tid < 12) {   // face block f = 4 d + 2 qa + qb: interior of face d of the record on side (qa, qb)
    const int d = tid >> 2, qa = (tid >> 1) & 1, qb = tid & 1;
    // plane 0 (normal x1): A ~ x3, B ~ x2; plane 1: A ~ x3, B ~ x1; plane 2: A ~ x2, B ~ x1
    const int bA = qa ? 0 : 1, bB = qb ? 0 : 1;
    int bits;
    if (d == 0) bits = (bB << 1) | (bA << 2);
    else if (d == 1) bits = bB | (bA << 2);
    else bits = bB | (bA << 1);
    const long long b = base[bits];
    fb[tid] = b < 0 ? -1LL : b + d * MM;
  } else if (tid >= 32 && tid < 38) {   // vertex line e (0: x1, 1: x2, 2: x3), side lo / hi
    const int e = (tid - 32) >> 1, hi = (tid - 32) & 1;
    const long long b = base[hi ? 0 : (1 << e)];
    lb[tid - 32] = b < 0 ? -1LL : b + 3 * MM + e * M;
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  // ---- gather the three star planes of r (zero outside the stored box)
  // face blocks: thread t owns block positions l = t, t + NT (decoded once), for all 12 blocks
#pragma unroll
  for (int k = 0; k < (MM + NT - 1) / NT; ++k) {
    const int l = tid + k * NT;
    if (l < MM) {
      const int Al = l / M, Bl = l - Al * M, lo = Al * LD + Bl;
#pragma unroll
      for (int f = 0; f < 12; ++f) {
        const int d = f >> 2, qa = (f >> 1) & 1, qb = f & 1;
        const long long b = fb[f];
        cpa8(&R[d * MS + qa * P * LD + qb * P + lo], r + (b < 0 ? 0 : b + l), b >= 0);
      }
    }
  }
  // the two vertex lines of each plane: plane 0 rows A = c (x2 line) / cols B = c (x3 line), plane 1
  // A = c (x1 line) / B = c (x3 line), plane 2 A = c (x1 line) / B = c (x2 line)
  for (int idx = tid; idx < 6 * N; idx += NT) {
    const int pl = idx / N, j = idx - pl * N, d = pl >> 1, col = pl & 1;   // col: line along the A index
    const int e = (d == 0) ? (col ? 2 : 1) : (d == 1 ? (col ? 2 : 0) : (col ? 1 : 0));
    long long src;
    if (j < C) src = lb[2 * e] < 0 ? -1LL : lb[2 * e] + j;
    else if (j == C) src = base[0] < 0 ? -1LL : base[0] + 3 * MM + 3 * M;
    else src = lb[2 * e + 1] < 0 ? -1LL : lb[2 * e + 1] + (j - P);
    const int o = col ? (j * LD + C) : (C * LD + j);
    cpa8(&R[d * MS + o], r + (src < 0 ? 0 : src), src >= 0);
  }
  cpa_commit();
  // zero the padding rows / columns of the planes (read by the transforms)
  if constexpr (NP > N) {
    constexpr int PC = NP - N, PADN = NP * NP - NN;
    for (int i = tid; i < 3 * PADN; i += NT) {
      const int d = i / PADN, k = i - d * PADN;
      int A, B;
      if (k < N * PC) { A = k / PC; B = N + (k - A * PC); }
      else { const int k2 = k - N * PC; A = N + k2 / NP; B = k2 - (A - N) * NP; }
      R[d * MS + A * LD + B] = 0.0;
    }
  }
  cpa_wait<0>();
  __syncthreads();
  // inverse multiplicity on the two lines through the vertex of each plane
  for (int i = tid; i < 3 * 2 * N; i += NT) {
    const int d = i / (2 * N), rr = i - d * 2 * N, line = rr / N, t = rr - line * N;
    const int A = line ? t : C, B = line ? C : t;
    if (line && t == C) continue;   // the vertex: scaled once, by the row pass
    R[d * MS + A * LD + B] *= (A == C && B == C) ? (1.0 / 3.0) : 0.5;
  }
  __syncthreads();
  // ---- forward transforms, one plane at a time: X = F_d S_B ; T_d = S_A^T X (over F_d)
#pragma unroll 1
  for (int d = 0; d < 3; ++d) {
    const int sB = (d == 0) ? 1 : 0, sA = (d == 2) ? 1 : 2;
    gemm4<NP, LD, false, false>(R + d * MS, Ssm + sB * MS, X, warp, lane);
    __syncthreads();
    gemm4<NP, LD, true, false>(Ssm + sA * MS, X, R + d * MS, warp, lane);
    __syncthreads();
  }
  // ---- core: the GS lanes of a group own a1, each pass two a3 values (a, a + NG) of the group
  {
    constexpr int GS = K::GS, NG = K::NG;
    const double *L1 = vec, *s1 = vec + NP, *L2 = vec + 3 * NP, *s2 = vec + 4 * NP, *L3 = vec + 6 * NP, *s3 = vec + 7 * NP;
    double* T1 = R;            // T1[a3][a2] -> G1[a3][a2]
    double* T2 = R + MS;       // T2[a3][a1] -> G2[a3][a1]
    const double* T3 = R + 2 * MS;   // T3[a2][a1]
    const int a1 = lane & (GS - 1), grp = warp * (32 / GS) + lane / GS;
    const bool va = a1 < N;
    const int a1c = va ? a1 : 0;
    const double s1a = va ? s1[a1c] : 0.0, L1a = L1[a1c];
    double g3[N];
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2) g3[a2] = 0.0;
    constexpr int PASSES = ((N + NG - 1) / NG + 1) / 2;
#pragma unroll 1
    for (int it = 0; it < PASSES; ++it) {
      const int a = grp + 2 * NG * it, b = a + NG;
      const bool ta = a < N, tb = b < N;
      const int ac = ta ? a : grp, bc = tb ? b : grp;   // invalid: a row this group owns (no cross-group race)
      const double ona = (ta && va) ? 1.0 : 0.0, onb = (tb && va) ? 1.0 : 0.0;
      const double t2a = ona * T2[ac * LD + a1c], t2b = onb * T2[bc * LD + a1c];
      const double s3a = ona * s3[ac], s3b = onb * s3[bc];
      const double s1va = ona * s1a, s1vb = onb * s1a;
      const double baseA = lam + L1a + L3[ac], baseB = lam + L1a + L3[bc];
      double g2a = 0.0, g2b = 0.0;
#pragma unroll
      for (int ch = 0; ch < NP / 8; ++ch) {
        double w[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int a2 = 8 * ch + j;
          if (a2 < N) {
            const double t3 = T3[a2 * LD + a1c], s2v = s2[a2], L2v = L2[a2];
            double Ea = s1va * T1[ac * LD + a2];
            double Eb = s1vb * T1[bc * LD + a2];
            Ea = fma(s2v, t2a, Ea);
            Eb = fma(s2v, t2b, Eb);
            Ea = fma(s3a, t3, Ea);
            Eb = fma(s3b, t3, Eb);
            const double Va = Ea * rcp3(baseA + L2v), Vb = Eb * rcp3(baseB + L2v);
            g2a = fma(s2v, Va, g2a);
            g2b = fma(s2v, Vb, g2b);
            g3[a2] = fma(s3a, Va, g3[a2]);
            g3[a2] = fma(s3b, Vb, g3[a2]);
            w[j] = s1a * Va;
            w[8 + j] = s1a * Vb;
          } else {
            w[j] = 0.0;
            w[8 + j] = 0.0;
          }
        }
        // reduce-scatter of the 16 values over the GS lanes of the group (sum over a1): lane l of the
        // group ends with the total of value l / (GS / 16) (GS = 32: the lane pair l, l ^ 1 holds it twice)
#pragma unroll
        for (int off = GS / 2, half = 8; half >= 1; off >>= 1, half >>= 1) {
          const bool upper = (lane & off) != 0;
#pragma unroll
          for (int j = 0; j < half; ++j) {
            const double send = upper ? w[j] : w[j + half];
            const double keep = upper ? w[j + half] : w[j];
            w[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        double tot = w[0];
        if constexpr (GS == 32) tot += __shfl_xor_sync(0xffffffffu, w[0], 1);
        const int k = (GS == 32) ? (a1 >> 1) : a1, a2 = 8 * ch + (k & 7);
        if ((GS == 16 || (lane & 1) == 0) && a2 < N) {
          if (k < 8) { if (ta) T1[a * LD + a2] = tot; }
          else if (tb) T1[b * LD + a2] = tot;
        }
      }
      if (va) {
        if (ta) T2[a * LD + a1] = g2a;
        if (tb) T2[b * LD + a1] = g2b;
      }
    }
    if constexpr (GS == 16) {   // the two groups of a warp share a1: add them first
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) g3[a2] += __shfl_xor_sync(0xffffffffu, g3[a2], 16);
    }
    // G3 = sum over the four warps' partials, fixed order (w0 + w2) + (w1 + w3): T3's region and X
    __syncthreads();   // every group is done reading T3
    double* G3 = R + 2 * MS;
    const bool wr = va && lane < GS;
    if (wr) {
      if (warp == 0) {
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) G3[a2 * LD + a1] = g3[a2];
      } else if (warp == 1) {
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) X[a2 * LD + a1] = g3[a2];
      }
    }
    __syncthreads();
    if (wr) {
      if (warp == 2) {
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) G3[a2 * LD + a1] += g3[a2];
      } else if (warp == 3) {
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) X[a2 * LD + a1] += g3[a2];
      }
    }
    __syncthreads();
    for (int i = tid; i < N * 32; i += NT) {
      const int a2 = i >> 5, a1_ = i & 31;
      if (a1_ < N) G3[a2 * LD + a1_] += X[a2 * LD + a1_];
    }
    __syncthreads();
  }
  // ---- back transforms, one plane at a time: X = G_d S_B^T ; U_d = S_A X (over G_d)
#pragma unroll 1
  for (int d = 0; d < 3; ++d) {
    const int sB = (d == 0) ? 1 : 0, sA = (d == 2) ? 1 : 2;
    gemm4<NP, LD, false, true>(R + d * MS, Ssm + sB * MS, X, warp, lane);
    __syncthreads();
    gemm4<NP, LD, false, false>(Ssm + sA * MS, X, R + d * MS, warp, lane);
    __syncthreads();
  }
  // ---- weighted scatter-add of the unique star points (u += W U; one colour's stars are disjoint)
  const double *w1 = vec + 2 * NP, *w2 = vec + 5 * NP, *w3 = vec + 8 * NP;
  // Points that are not unknowns (Dirichlet faces, stored entries outside the box) get U = 0
  // exactly: their rows of S_d are identity rows, their r entries are zero, and the vertex row s_d
  // vanishes on them, so u there is rewritten unchanged and no free-point test is needed.  Faces:
  // loads of the thread's u entries first (two block positions x 12 blocks), then the stores.
  constexpr int KR = (MM + NT - 1) / NT;
  double uo[KR][12];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int l = tid + k * NT;
#pragma unroll
    for (int f = 0; f < 12; ++f) {
      const long long b = fb[f];
      uo[k][f] = (l < MM && b >= 0) ? u[b + l] : 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int l = tid + k * NT;
    if (l < MM) {
      const int Al = l / M, Bl = l - Al * M;
#pragma unroll
      for (int f = 0; f < 12; ++f) {
        const int d = f >> 2, qa = (f >> 1) & 1, qb = f & 1;
        const int A = Al + qa * P, B = Bl + qb * P;
        const long long b = fb[f];
        if (b < 0) continue;
        const double W = d == 0 ? w2[B] * w3[A] : (d == 1 ? w1[B] * w3[A] : w1[B] * w2[A]);
        u[b + l] = fma(W, R[d * MS + A * LD + B], uo[k][f]);
      }
    }
  }
  // the three vertex lines (x2 line and x3 line from plane 0 -- the vertex with the x2 line --, x1 line
  // from plane 1)
  if (tid < 3 * N) {
    const int e3 = tid / N, j = tid - e3 * N;   // e3: 0 = x2 line, 1 = x3 line, 2 = x1 line
    if (!(e3 > 0 && j == C)) {
      const int e = e3 == 0 ? 1 : (e3 == 1 ? 2 : 0);
      long long src;
      if (j < C) src = lb[2 * e] < 0 ? -1LL : lb[2 * e] + j;
      else if (j == C) src = base[0] < 0 ? -1LL : base[0] + 3 * MM + 3 * M;
      else src = lb[2 * e + 1] < 0 ? -1LL : lb[2 * e + 1] + (j - P);
      int o;
      double W;
      if (e3 == 0) { o = C * LD + j; W = w2[j]; }                 // plane 0, A = c, B = j
      else if (e3 == 1) { o = j * LD + C; W = w3[j]; }            // plane 0, A = j, B = c
      else { o = MS + C * LD + j; W = w1[j]; }                    // plane 1, A = c, B = j
      if (src >= 0) {
        const double uold = u[src];
        u[src] = fma(W, R[o], uold);
      }
    }
  }
}

cudaError_t launch_star16(const LevelGeom& g, int c1, int c2, int c3, int n1c, int n2c, long long nb, const double* r,
                          double* u, const double* stabP, double lam, cudaStream_t st) {
  switch (g.p) {
#define CASE(PP)                                                                                                     \
  case PP:                                                                                                           \
    return launch_pdl(k_star16<PP>, dim3((unsigned)n1c, (unsigned)n2c, (unsigned)(nb / ((long long)n1c * n2c))),     \
                      dim3(Star16<PP>::NT), star16_smem<PP>(), st, g, c1, c2, c3, n1c, n2c, r, u, stabP, lam);
    CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

int star16_np(int p) { return (2 * p - 1 + 7) / 8 * 8; }

cudaError_t star16_set_smem_attr() {
  cudaError_t e = cudaSuccess;
#define CASE(PP)                                                                                   \
  {                                                                                                \
    cudaError_t a = cudaFuncSetAttribute(k_star16<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)star16_smem<PP>());                                  \
    if (a != cudaSuccess) e = a;                                                                   \
  }
  CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
  return e;
}

}  // namespace pmg
