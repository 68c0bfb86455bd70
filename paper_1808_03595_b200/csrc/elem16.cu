// Condensed element operator for 9 <= p <= 16 (P:117-123 with the O(p^3) evaluation of reading R1,
// SURVEY App. A.1): Y_e = H_hat_e u_e = H_BB u_e - C u_e on the element's boundary points, one CTA of
// 4 warps per element, three CTAs per SM.  Same arithmetic as k_elem_pf16 (hot_kernels.cu),
// re-planned from its ncu profile (round 2 start: shared-memory bound, L1/TEX 90 %, 44 % of the
// samples in the gather / table set-up):
//   - the element's tables come from a padded per-(direction, 1-D element) table that is the shared
//     memory image itself (P_d as MP x 20, Lambda, a0, a1, M, K~ = M^-1 K row-scaled): one 16-byte
//     cp.async stream, no set-up loops;
//   - the six closed faces are gathered once into (MP+1) x 20 arrays; the DMMA transforms read the
//     face interiors from them with a (1, 1) offset (the padded index is the t = p boundary line,
//     multiplied by a zero table entry or -- for H_BB -- the wanted boundary term);
//   - H_BB's tangential line sums of the face interiors are one DMMA GEMM pair per face accumulated
//     into one tile set, Z = U K~_a^T + K~_b U (the M factors of the two terms folded into K~), so
//     only the t = 0 terms and the normal terms remain scalar;
//   - the Schur correction runs in one pass over the interior eigen-triples (lanes b1, 2 groups per
//     warp, b3 per group, b2 in registers): E, V = E / D (rcp + one cubic Newton step), the x2-face
//     contractions in registers, the x3-face contractions in register arrays reduced over the 8
//     groups in a fixed-order tree, the x1-face contractions by a 16-lane butterfly reduce-scatter.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {
namespace {

__device__ __forceinline__ double rcp3e(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ void dmma_e(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa8e(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cpa16e(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

}  // namespace

// padded element table row (host: pmg_api.cu), per direction d and 1-D element e_d:
//   [oP]  P[b][i] = S[i][b] M_II[i]  (MP x LDT, zero padded)
//   [oL]  Lambda[b] (MP, padded with 1)      [oA0] a0[b], [oA1] a1[b] (MP, zero padded)
//   [oM]  M[t], t = 0..p (LDT, zero padded)  [oK]  K~[t][t'] = K[t][t'] / M[t] ((P+1) x LDT, zero padded)
//   [oS]  S[i][b] (MP x LDT, zero padded): interior eigenvectors, S^T K_II S = Lambda, S^T M_II S = I
template <int P> struct Elem16 {
  static constexpr int M = P - 1, Q = P + 1, MM = M * M;
  static constexpr int MP = (P + 7) / 8 * 8;               // transform size; index MP-1 >= m reaches t = p
  static constexpr int LDT = (MP + 1 + 3) / 8 * 8 + 4;      // >= MP + 1 and = 4 (mod 8): conflict-free DMMA fragments
  static constexpr int UR = MP + 1;                          // closed-face rows (>= Q)
  static constexpr int FS = UR * LDT;                        // closed-face stride
  static constexpr int MS = MP * LDT;                        // transform matrix stride
  static constexpr int oP = 0, oL = MS, oA0 = oL + MP, oA1 = oA0 + MP, oM = oA1 + MP, oK = oM + LDT,
                       ETP = oK + Q * LDT + ((Q * LDT) & 1);
  // the table row continues with S[i][b] (MP x LDT) for condensation / recovery (cr16.cu); the
  // element operator copies only the first ETP doubles of a row
  static constexpr int oS = ETP, ETS = ETP + MS;
  static constexpr int NT = 128;
  static constexpr int YS = 6 * MM + 12 * M + 8;
  // shared memory (doubles): three table rows, six closed faces, X (6 MS), T / G / C (6 MS)
  static constexpr int oTab = 0, oU = 3 * ETP, oX = oU + 6 * FS, oT = oX + 6 * MS, total = oT + 6 * MS;
};

template <int P>
size_t elem16_smem2() { return sizeof(double) * Elem16<P>::total; }

int elem16_etp(int p) {   // row stride of the padded element table
  switch (p) {
#define CASE(PP) case PP: return Elem16<PP>::ETS;
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return 0;
  }
}

// host: padded element-table row from the element-table row (layout of pmg_internal.h)
void elem16_table_row(int p, const double* et, double* out) {
  const int m = p - 1, q = p + 1;
  int MP = (p + 7) / 8 * 8, LDT = (MP + 1 + 3) / 8 * 8 + 4;
  const int oL = MP * LDT, oA0 = oL + MP, oA1 = oA0 + MP, oM = oA1 + MP, oK = oM + LDT;
  for (int b = 0; b < m; ++b)
    for (int i = 0; i < m; ++i) out[b * LDT + i] = et[et_P(p) + b * m + i];
  for (int b = 0; b < MP; ++b) {
    out[oL + b] = b < m ? et[et_lam(p) + b] : 1.0;
    out[oA0 + b] = b < m ? et[et_a0(p) + b] : 0.0;
    out[oA1 + b] = b < m ? et[et_a1(p) + b] : 0.0;
  }
  for (int t = 0; t < q; ++t) out[oM + t] = et[et_M(p) + t];
  for (int t = 0; t < q; ++t)
    for (int s = 0; s < q; ++s) out[oK + t * LDT + s] = et[et_K(p) + t * q + s] / et[et_M(p) + t];
  const int oS = oK + q * LDT + ((q * LDT) & 1);
  for (int i = 0; i < m; ++i)
    for (int b = 0; b < m; ++b) out[oS + i * LDT + b] = et[et_S(p) + i * m + b];
}

template <int P>
__global__ void __launch_bounds__(128, 3)
    k_elem16(LevelGeom g, const double* __restrict__ u, const double* __restrict__ etabP, double lam,
             double* __restrict__ Y, const int* __restrict__ done) {
  using K = Elem16<P>;
  constexpr int M = K::M, Q = K::Q, MM = K::MM, MP = K::MP, LDT = K::LDT, UR = K::UR, FS = K::FS, MS = K::MS,
                ETP = K::ETP, NT = K::NT, YS = K::YS;
  constexpr int RS = 3 * MM + 3 * M + 1;
  extern __shared__ double sm[];
  double* tb = sm + K::oTab;
  double* Uc = sm + K::oU;
  double* X = sm + K::oX;
  double* T = sm + K::oT;
  const int e1 = blockIdx.x, e2 = blockIdx.y, e3 = blockIdx.z;   // 3-D grid over the elements
  const long long e = e1 + (long long)g.k1 * (e2 + (long long)g.k2 * e3);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- tables (before the dependency wait)
  {
    for (int i = tid; i < 3 * (ETP / 2); i += NT) {
      const int d = i / (ETP / 2), ch = i - d * (ETP / 2);
      const size_t row = d == 0 ? (size_t)e1 : (d == 1 ? (size_t)(g.k1 + e2) : (size_t)(g.k1 + g.k2 + e3));
      cpa16e(tb + d * ETP + 2 * ch, etabP + row * K::ETS + 2 * ch);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  // closed-face rows / columns beyond t = p (p < MP) are read by the padded transforms: zero them
  if constexpr (UR > Q) {   // p < MP: rows and columns Q .. MP of the closed faces are read
    for (int i = tid; i < 6 * UR * (UR - Q); i += NT) {
      const int f = i / (UR * (UR - Q)), rr = i - f * UR * (UR - Q), a = rr / (UR - Q), b = Q + rr - a * (UR - Q);
      Uc[f * FS + a * LDT + b] = 0.0;   // columns Q .. MP of every row
      Uc[f * FS + b * LDT + a] = 0.0;   // rows Q .. MP
    }
  }
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  // ---- gather the six closed faces: face f = 2 d + s (normal d at t_d = s p), rows tb (slow
  // tangential direction db), columns ta (fast tangential direction da); the face interior is a
  // contiguous (p-1)^2 run of one record, the rim comes from edge and vertex slots
  {
    const long long V12 = (long long)g.V1 * g.V2;
    const long long rec0 = e1 + g.V1 * (long long)e2 + V12 * e3;
    auto recb = [&](int o1, int o2, int o3) {   // record e + o (periodic: the last element wraps to 0)
      if (!g.per) return (rec0 + o1 + g.V1 * (long long)o2 + V12 * o3) * RS;
      const int w1 = wrap_rec(e1 + o1, g.k1, g.per & 1), w2 = wrap_rec(e2 + o2, g.k2, g.per & 2),
                w3 = wrap_rec(e3 + o3, g.k3, g.per & 4);
      return (w1 + g.V1 * (long long)w2 + V12 * w3) * RS;
    };
#pragma unroll
    for (int k = 0; k < (MM + NT - 1) / NT; ++k) {   // face interiors: thread = block position l
      const int l = tid + k * NT;
      if (l < MM) {
        const int A = l / M, B = l - A * M, lo = (A + 1) * LDT + B + 1;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          const int d = f >> 1, s = f & 1;
          cpa8e(&Uc[f * FS + lo], u + recb(d == 0 ? s : 0, d == 1 ? s : 0, d == 2 ? s : 0) + d * MM + l);
        }
      }
    }
    // rim: 4 p points per face, (tb, ta) walked around the boundary
    for (int idx = tid; idx < 6 * 4 * P; idx += NT) {
      const int f = idx / (4 * P), rr = idx - f * 4 * P, side = rr / P, i = rr - side * P, d = f >> 1, s = f & 1;
      int ta, tbb;
      if (side == 0) { tbb = 0; ta = i; } else if (side == 1) { ta = P; tbb = i; }
      else if (side == 2) { tbb = P; ta = P - i; } else { ta = 0; tbb = P - i; }
      // element-local (t1, t2, t3): d normal, a = fast, b = slow tangential direction
      int x1, x2, x3;
      if (d == 0) { x1 = s * P; x2 = ta; x3 = tbb; }
      else if (d == 1) { x2 = s * P; x1 = ta; x3 = tbb; }
      else { x3 = s * P; x1 = ta; x2 = tbb; }
      const int o1 = x1 == P, o2 = x2 == P, o3 = x3 == P;   // t = p: next record, local 0
      if (o1) x1 = 0;
      if (o2) x2 = 0;
      if (o3) x3 = 0;
      int slot;
      if (x1 == 0) {
        if (x2 == 0) slot = (x3 == 0) ? 3 * MM + 3 * M : 3 * MM + 2 * M + x3 - 1;
        else if (x3 == 0) slot = 3 * MM + M + x2 - 1;
        else slot = (x3 - 1) * M + (x2 - 1);
      } else if (x2 == 0) {
        slot = (x3 == 0) ? 3 * MM + x1 - 1 : MM + (x3 - 1) * M + (x1 - 1);
      } else {
        slot = 2 * MM + (x2 - 1) * M + (x1 - 1);
      }
      cpa8e(&Uc[f * FS + tbb * LDT + ta], u + recb(o1, o2, o3) + slot);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const int r8 = lane >> 2, q4 = lane & 3;
  // ---- forward transforms: X_f = U_f P_a^T, then T_f = P_b X_f.  Jobs = (face, 8-row tile panel):
  // 6 T8 jobs per stage over the 4 warps, each panel 1 x T8 tiles (one A fragment per k step serves
  // every tile of the panel)
  constexpr int T8 = MP / 8, NJ = 6 * T8;
  auto panel = [&](auto TA, auto TB, const double* A, int lda, const double* B, int ldb, double* Cm, int ldc, int mi) {
    double c[T8][2];
#pragma unroll
    for (int j = 0; j < T8; ++j) c[j][0] = c[j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < MP / 4; ++kk) {
      const int k = 4 * kk + q4, ii = 8 * mi + r8;
      const double a = decltype(TA)::value ? A[k * lda + ii] : A[ii * lda + k];
#pragma unroll
      for (int j = 0; j < T8; ++j) {
        const int jj = 8 * j + r8;
        dmma_e(c[j][0], c[j][1], a, decltype(TB)::value ? B[jj * ldb + k] : B[k * ldb + jj]);
      }
    }
#pragma unroll
    for (int j = 0; j < T8; ++j)
      *reinterpret_cast<double2*>(Cm + (8 * mi + r8) * ldc + 8 * j + 2 * q4) = make_double2(c[j][0], c[j][1]);
  };
  using TT = std::true_type;
  using FF = std::false_type;
  for (int job = warp; job < NJ; job += 4) {   // X_f = U_f,int P_a^T
    const int f = job / T8, mi = job - f * T8, d = f >> 1, da = (d == 0) ? 1 : 0;
    panel(FF{}, TT{}, Uc + f * FS + LDT + 1, LDT, tb + da * ETP + K::oP, LDT, X + f * MS, LDT, mi);
  }
  __syncthreads();
  for (int job = warp; job < NJ; job += 4) {   // T_f = P_b X_f
    const int f = job / T8, mi = job - f * T8, d = f >> 1, db = (d == 2) ? 1 : 2;
    panel(FF{}, FF{}, tb + db * ETP + K::oP, LDT, X + f * MS, LDT, T + f * MS, LDT, mi);
  }
  __syncthreads();
  // ---- core over the interior eigen-triples (b1 lanes, b3 per 16-lane group, b2 in registers)
  {
    const double *a10 = tb + K::oA0, *a11 = tb + K::oA1;
    const double *a20 = tb + ETP + K::oA0, *a21 = tb + ETP + K::oA1;
    const double *a30 = tb + 2 * ETP + K::oA0, *a31 = tb + 2 * ETP + K::oA1;
    const double *L1 = tb + K::oL, *L2 = tb + ETP + K::oL, *L3 = tb + 2 * ETP + K::oL;
    const int b1 = lane & 15, grp = warp * 2 + (lane >> 4);
    const bool vb1 = b1 < M;
    const int b1c = vb1 ? b1 : 0;
    const double c10 = vb1 ? a10[b1c] : 0.0, c11 = vb1 ? a11[b1c] : 0.0, L1v = L1[b1c];
    double g4[M], g5[M];
#pragma unroll
    for (int b2 = 0; b2 < M; ++b2) g4[b2] = g5[b2] = 0.0;
#pragma unroll 1
    for (int it = 0; it < 2; ++it) {
      const int b3 = grp + 8 * it;
      const bool vb3 = b3 < M;
      const int b3c = vb3 ? b3 : grp;   // invalid: a row this group owns (no cross-group race)
      const double on = (vb1 && vb3) ? 1.0 : 0.0;
      const double t2 = on * T[2 * MS + b3c * LDT + b1c], t3 = on * T[3 * MS + b3c * LDT + b1c];
      const double c30 = on * a30[b3c], c31 = on * a31[b3c], c10v = on * c10, c11v = on * c11;
      const double base = lam + L1v + L3[b3c];
      double g2 = 0.0, g3 = 0.0;
#pragma unroll
      for (int ch = 0; ch < MP / 8; ++ch) {
        double w[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int b2 = 8 * ch + j;
          if (b2 < M) {
            double E = c10v * T[0 * MS + b3c * LDT + b2];
            E = fma(c11v, T[1 * MS + b3c * LDT + b2], E);
            E = fma(a20[b2], t2, E);
            E = fma(a21[b2], t3, E);
            E = fma(c30, T[4 * MS + b2 * LDT + b1c], E);
            E = fma(c31, T[5 * MS + b2 * LDT + b1c], E);
            const double V = E * rcp3e(base + L2[b2]);
            g2 = fma(a20[b2], V, g2);
            g3 = fma(a21[b2], V, g3);
            g4[b2] = fma(c30, V, g4[b2]);
            g5[b2] = fma(c31, V, g5[b2]);
            w[j] = c10 * V;
            w[8 + j] = c11 * V;
          } else {
            w[j] = 0.0;
            w[8 + j] = 0.0;
          }
        }
        // reduce-scatter over the 16 lanes of the group: lane b1 ends with value b1 (j = b1 & 7 of
        // face 0 for b1 < 8, of face 1 for b1 >= 8)
#pragma unroll
        for (int off = 8, half = 8; off >= 1; off >>= 1, half >>= 1) {
          const bool upper = (lane & off) != 0;
#pragma unroll
          for (int j = 0; j < half; ++j) {
            const double send = upper ? w[j] : w[j + half];
            const double keep = upper ? w[j + half] : w[j];
            w[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        const int b2 = 8 * ch + (b1 & 7);
        if (vb3 && b2 < M) T[(b1 >> 3) * MS + b3 * LDT + b2] = w[0];   // G0 / G1 over T0 / T1 row b3
      }
      if (vb3 && vb1) {
        T[2 * MS + b3 * LDT + b1] = g2;
        T[3 * MS + b3 * LDT + b1] = g3;
      }
    }
    // G4 / G5: the two groups of a warp, then the four warps (w0 + w2) + (w1 + w3) through X
#pragma unroll
    for (int b2 = 0; b2 < M; ++b2) {
      g4[b2] += __shfl_xor_sync(0xffffffffu, g4[b2], 16);
      g5[b2] += __shfl_xor_sync(0xffffffffu, g5[b2], 16);
    }
    __syncthreads();   // every group is done reading T4 / T5
    const bool wr = vb1 && lane < 16;
    double* P0 = X;             // partial of warps 1 (+3)
    if (wr && (warp == 0 || warp == 2)) {
      double* dst = T + 4 * MS;
      if (warp == 0) {
#pragma unroll
        for (int b2 = 0; b2 < M; ++b2) { dst[b2 * LDT + b1] = g4[b2]; dst[MS + b2 * LDT + b1] = g5[b2]; }
      }
    } else if (wr && warp == 1) {
#pragma unroll
      for (int b2 = 0; b2 < M; ++b2) { P0[b2 * LDT + b1] = g4[b2]; P0[MS + b2 * LDT + b1] = g5[b2]; }
    }
    __syncthreads();
    if (wr && warp == 2) {
      double* dst = T + 4 * MS;
#pragma unroll
      for (int b2 = 0; b2 < M; ++b2) { dst[b2 * LDT + b1] += g4[b2]; dst[MS + b2 * LDT + b1] += g5[b2]; }
    } else if (wr && warp == 3) {
#pragma unroll
      for (int b2 = 0; b2 < M; ++b2) { P0[b2 * LDT + b1] += g4[b2]; P0[MS + b2 * LDT + b1] += g5[b2]; }
    }
    __syncthreads();
    for (int i = tid; i < 2 * M * 16; i += NT) {
      const int h = i / (M * 16), rr = i - h * M * 16, b2 = rr >> 4, b1_ = rr & 15;
      if (b1_ < M) T[(4 + h) * MS + b2 * LDT + b1_] += P0[h * MS + b2 * LDT + b1_];
    }
    __syncthreads();
  }
  // ---- back transforms: X_f = G_f P_a, then C_f = P_b^T X_f (into T)
  for (int job = warp; job < NJ; job += 4) {
    const int f = job / T8, mi = job - f * T8, d = f >> 1, da = (d == 0) ? 1 : 0;
    panel(FF{}, FF{}, T + f * MS, LDT, tb + da * ETP + K::oP, LDT, X + f * MS, LDT, mi);
  }
  __syncthreads();
  for (int job = warp; job < NJ; job += 4) {
    const int f = job / T8, mi = job - f * T8, d = f >> 1, db = (d == 2) ? 1 : 2;
    panel(TT{}, FF{}, tb + db * ETP + K::oP, LDT, X + f * MS, LDT, T + f * MS, LDT, mi);
  }
  __syncthreads();
  // ---- H_BB tangential line sums of the face interiors: Z_f = U_f K~_a^T + K~_b U_f (t = 1 .. MP;
  // beyond t = p the table is zero), both products accumulated in one tile panel (into X)
  for (int job = warp; job < NJ; job += 4) {
    const int f = job / T8, mi = job - f * T8, d = f >> 1, da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
    const double* U = Uc + f * FS + LDT + 1;                 // U[tb-1][t-1]
    const double* Ka = tb + da * ETP + K::oK + LDT + 1;      // Ka[ta-1][t-1] = K~_a[ta][t]
    const double* Kb = tb + db * ETP + K::oK + LDT + 1;
    double c[T8][2];
#pragma unroll
    for (int j = 0; j < T8; ++j) c[j][0] = c[j][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < MP / 4; ++kk) {
      const int k = 4 * kk + q4, ii = 8 * mi + r8;
      const double ua = U[ii * LDT + k], kb = Kb[ii * LDT + k];
#pragma unroll
      for (int j = 0; j < T8; ++j) {
        const int jj = 8 * j + r8;
        dmma_e(c[j][0], c[j][1], ua, Ka[jj * LDT + k]);     // sum_t U[tb][t] K~a[ta][t]
        dmma_e(c[j][0], c[j][1], kb, U[k * LDT + jj]);      // sum_t K~b[tb][t] U[t][ta]
      }
    }
#pragma unroll
    for (int j = 0; j < T8; ++j)
      *reinterpret_cast<double2*>(X + f * MS + (8 * mi + r8) * LDT + 8 * j + 2 * q4) = make_double2(c[j][0], c[j][1]);
  }
  __syncthreads();
  // ---- outputs: face interiors (thread = block position (A, B), all six faces), then edges and
  // vertices (all three lines lie on the element boundary)
  auto Mv = [&](int d) { return tb + d * ETP + K::oM; };
  auto Kt = [&](int d) { return tb + d * ETP + K::oK; };
  double* Ye = Y + (size_t)e * g.YS;
#pragma unroll
  for (int k = 0; k < (MM + NT - 1) / NT; ++k) {
    const int l = tid + k * NT;
    if (l < MM) {
      const int A = l / M, B = l - A * M, ta = B + 1, tbb = A + 1;
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        const int d = f >> 1, s_ = f & 1, da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2, td = s_ * P;
        const double* Uf = Uc + f * FS;
        const double* Kd = Kt(d);
        double z = X[f * MS + A * LDT + B];
        z = fma(Kt(db)[tbb * LDT], Uf[ta], z);                           // t = 0 term along b
        z = fma(Kd[td * LDT], Uc[(2 * d) * FS + tbb * LDT + ta], z);     // normal line: the two faces
        z = fma(Kd[td * LDT + P], Uc[(2 * d + 1) * FS + tbb * LDT + ta], z);
        z = fma(lam, Uf[tbb * LDT + ta], z);
        // t = 0 term along a after the M_a[ta] scaling: M_a[ta] K~_a[ta][0] = K_a[ta][0] = K_a[0][ta]
        // = M_a[0] K~_a[0][ta] (K symmetric), read along the row: lanes of consecutive ta hit
        // consecutive banks instead of a column at stride LDT
        const double za = fma(Mv(da)[0] * Kt(da)[ta], Uf[tbb * LDT], Mv(da)[ta] * z);
        Ye[f * MM + l] = Mv(d)[td] * Mv(db)[tbb] * za - T[f * MS + A * LDT + B];
      }
    }
  }
  // a boundary line along d through (t1, t2, t3) lies in a face whose normal n != d has t_n in {0, p}:
  // in that face's closed array it is a row (d the fast direction) or a column
  // TR: the line of the point's own edge direction d, whose K~ row t_d varies over the lanes: summed
  // as sum_t K~_d[t][t_d] M_d[t] u(t) = M_d[t_d] sum_t K~_d[t_d][t] u(t) (K symmetric), the row read
  // along consecutive t_d (no stride-LDT bank conflicts)
  auto line = [&](int d, int t1, int t2, int t3, auto TR) -> double {
    int n;
    if (d != 0 && (t1 == 0 || t1 == P)) n = 0;
    else if (d != 1 && (t2 == 0 || t2 == P)) n = 1;
    else n = 2;
    const int tn = n == 0 ? t1 : (n == 1 ? t2 : t3);
    const int fa = (n == 0) ? 1 : 0;                        // fast direction of the face
    const int ta = fa == 0 ? t1 : t2, tbb = n == 2 ? t2 : t3;
    const double* Uf = Uc + (2 * n + (tn == P ? 1 : 0)) * FS;
    const double* ptr = (d == fa) ? Uf + tbb * LDT : Uf + ta;
    const int st = (d == fa) ? 1 : LDT;
    const int td = d == 0 ? t1 : (d == 1 ? t2 : t3);
    double z = 0.0;
    if constexpr (decltype(TR)::value) {
      const double* Kc = Kt(d) + td;
      const double* Md = Mv(d);
#pragma unroll
      for (int t = 0; t <= P; ++t) z = fma(Kc[t * LDT], Md[t] * ptr[t * st], z);
    } else {
      const double* Kr = Kt(d) + td * LDT;
#pragma unroll
      for (int t = 0; t <= P; ++t) z = fma(Kr[t], ptr[t * st], z);
    }
    return z;
  };
  for (int o = 6 * MM + tid; o < YS; o += NT) {
    int t1, t2, t3, de = -1;
    if (o < 6 * MM + 12 * M) {
      const int r = o - 6 * MM, qe = r / M, i = r - qe * M, d = qe >> 2, sA = qe & 1, sB = (qe >> 1) & 1;
      if (d == 0) { t1 = i + 1; t2 = sA * P; t3 = sB * P; }
      else if (d == 1) { t2 = i + 1; t1 = sA * P; t3 = sB * P; }
      else { t3 = i + 1; t1 = sA * P; t2 = sB * P; }
      de = d;
    } else {
      const int qv = o - 6 * MM - 12 * M;
      t1 = (qv & 1) * P; t2 = ((qv >> 1) & 1) * P; t3 = ((qv >> 2) & 1) * P;
    }
    // the point's own value: in the face normal x1 if t1 is on the boundary, else x2, else x3
    const int n = (t1 == 0 || t1 == P) ? 0 : ((t2 == 0 || t2 == P) ? 1 : 2);
    const int tn = n == 0 ? t1 : (n == 1 ? t2 : t3);
    const int ta = n == 0 ? t2 : t1, tbb = n == 2 ? t2 : t3;
    double z = lam * Uc[(2 * n + (tn == P ? 1 : 0)) * FS + tbb * LDT + ta];
    if (de < 0) {   // vertex: every K~ row index is 0 or p
      z += line(0, t1, t2, t3, FF{});
      z += line(1, t1, t2, t3, FF{});
      z += line(2, t1, t2, t3, FF{});
      Ye[o] = Mv(0)[t1] * Mv(1)[t2] * Mv(2)[t3] * z;
    } else {        // edge along de: Y = M_a M_b (M_de[t_de] (lam u + two cross lines) + own line)
      const int da = de == 0 ? 1 : 0, db = de == 2 ? 1 : 2;
      const int tde = de == 0 ? t1 : (de == 1 ? t2 : t3);
      z += line(da, t1, t2, t3, FF{});
      z += line(db, t1, t2, t3, FF{});
      const double ze = fma(Mv(de)[tde], z, line(de, t1, t2, t3, TT{}));
      Ye[o] = Mv(da)[da == 0 ? t1 : t2] * Mv(db)[db == 1 ? t2 : t3] * ze;
    }
  }
}

cudaError_t launch_elem16(const LevelGeom& g, const double* u, const double* etabP, double lam, double* Y, const int* done,
                          cudaStream_t st) {
  switch (g.p) {
#define CASE(PP)                                                                                                      \
  case PP:                                                                                                            \
    return launch_pdl(k_elem16<PP>, dim3((unsigned)g.k1, (unsigned)g.k2, (unsigned)g.k3), dim3(Elem16<PP>::NT),            \
                      elem16_smem2<PP>(), st, g, u, etabP, lam, Y, done);
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t elem16_set_smem_attr() {
  cudaError_t e = cudaSuccess;
#define CASE(PP)                                                                                   \
  {                                                                                                \
    cudaError_t a = cudaFuncSetAttribute(k_elem16<PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)elem16_smem2<PP>());                                 \
    if (a != cudaSuccess) e = a;                                                                   \
  }
  CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
  return e;
}

}  // namespace pmg
