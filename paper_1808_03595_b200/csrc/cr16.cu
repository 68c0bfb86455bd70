// Static condensation and interior recovery for 9 <= p <= 16 (Alg. 4 lines 2 and 6, P:494 / P:501;
// P:117-122): the O(p^4) part of the solve, with the interior fast diagonalisation
// H_II^-1 = (S (x) S (x) S) D^-1 (S^T (x) S^T (x) S^T) (P:253-261 applied to the element interior).
// Same arithmetic as k_condense_elem / k_recover_elem (kernels.cu), re-planned for the tensor cores:
//   - the (p-1)^3 interior cube is a (p-1)^2 x (p-1) matrix (rows = the two slow indices) and each of
//     the three directional transforms is one DMMA GEMM against S_d (padded to 16), stored rotated
//     so that the next direction becomes the fast index (three passes restore the layout);
//   - 8 warps per CTA, two CTAs per SM (103 KB of shared memory: two cube buffers, the six face
//     arrays, the interior tables);
//   - the face transforms T_f = P_b U_f P_a^T (recovery) and Y_f = P_b^T G_f P_a (condensation) are
//     16 x 16 DMMA GEMMs; the divide by D uses rcp + one cubic Newton step.
//   condense:  V = (S^T (x) S^T (x) S^T) F_I / D;  G_f = sum_{b_d} a_f V;  Yc_f = (P_b^T (x) P_a^T) G_f
//   recover:   u_I = (S (x) S (x) S) [ ((S^T (x) S^T (x) S^T) F_I - sum_f a_f (x) T_f) / D ],
//              T_f = (P_b (x) P_a) u_f
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {
namespace {

__device__ __forceinline__ double rcp3c(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ void dmma_c(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cpa8c(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cpa16c(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}

}  // namespace

template <int P> struct CR16 {
  static constexpr int M = P - 1, MM = M * M, MP = 16, LD = 20, MS = MP * LD;
  // padded element-table row (elem16.cu): P at 0, Lambda at MS, a0, a1 (MP each), ..., S at oS
  static constexpr int oP = 0, oL = MS, oA0 = MS + MP, oA1 = MS + 2 * MP;
  static constexpr int Q = P + 1, LDT = 20, oM = oA1 + MP, oK = oM + LDT, ETP = oK + Q * LDT + ((Q * LDT) & 1),
                       oS = ETP, ETS = ETP + MS;
  // shared per direction: P (MS), Lambda, a0, a1 (3 MP), S (MS)
  static constexpr int TB = 2 * MS + 3 * MP;
  static constexpr int CR = MM;                 // cube rows; the last 8-row tile reads past them (unused rows)
  static constexpr int CB = CR * LD + 8 * LD;   // cube buffer incl. the overrun of the last tile
  static constexpr int NT = 256, NW = 8;
  static constexpr int oTab = 0, oC0 = 3 * TB, oC1 = oC0 + CB, oF = oC1 + CB, total = oF + 6 * MS;
};

template <int P>
size_t cr16_smem() { return sizeof(double) * CR16<P>::total; }

// one directional transform of the cube: out[(b m + r_hi)][r_lo] = sum_i in[(r_hi m + r_lo)][i] S(i, b),
// S(i, b) = S[i][b] (transpose = true: S^T applied) or S[b][i]; rows r = r_hi m + r_lo of `in`
template <int P, bool TR>
__device__ __forceinline__ void cube_pass(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ S,
                                          int warp, int lane) {
  using K = CR16<P>;
  constexpr int M = K::M, LD = K::LD, RT = (K::CR + 7) / 8;
  const int r8 = lane >> 2, q4 = lane & 3;
  double sb[4][2];   // the B fragments of S: the same for every row panel of the pass
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = 4 * kk + q4, jj = 8 * j + r8;
      sb[kk][j] = TR ? S[k * LD + jj] : S[jj * LD + k];
    }
  for (int mi = warp; mi < RT; mi += K::NW) {
    double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const double a = in[(8 * mi + r8) * LD + 4 * kk + q4];
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_c(c[j][0], c[j][1], a, sb[kk][j]);
    }
    const int row = 8 * mi + r8;
    if (row < K::CR) {
      const int rh = row / M, rl = row - rh * M;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b = 8 * j + 2 * q4 + h;
          if (b < M) out[(b * M + rh) * LD + rl] = c[j][h];
        }
    }
  }
}

// C (16 x 16, ld LD) = op(A) op(B), one 8-row panel per job: 12 jobs over 8 warps
template <bool TA, bool TB>
__device__ __forceinline__ void face_panel(const double* A, const double* B, double* Cm, int mi, int lane) {
  constexpr int LD = 20;
  const int r8 = lane >> 2, q4 = lane & 3;
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = 4 * kk + q4, ii = 8 * mi + r8;
    const double a = TA ? A[k * LD + ii] : A[ii * LD + k];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int jj = 8 * j + r8;
      dmma_c(c[j][0], c[j][1], a, TB ? B[jj * LD + k] : B[k * LD + jj]);
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
    *reinterpret_cast<double2*>(Cm + (8 * mi + r8) * LD + 8 * j + 2 * q4) = make_double2(c[j][0], c[j][1]);
}

// MODE 0: condensation (writes Yc), MODE 1: recovery (writes the interior of ug)
template <int P, int MODE>
__global__ void __launch_bounds__(256, 2)
    k_cr16(LevelGeom g, const double* __restrict__ Fg, const double* __restrict__ uh, const double* __restrict__ etabP,
           double lam, double* __restrict__ Yc, double* __restrict__ ug) {
  using K = CR16<P>;
  constexpr int M = K::M, MM = K::MM, MS = K::MS, LD = K::LD, TB = K::TB, NT = K::NT, ETS = K::ETS;
  constexpr int RS = 3 * MM + 3 * M + 1;
  extern __shared__ double sm[];
  double* tb = sm + K::oTab;
  double* C0 = sm + K::oC0;
  double* C1 = sm + K::oC1;
  double* Fa = sm + K::oF;   // six 16 x LD face arrays
  const int e1 = blockIdx.x, e2 = blockIdx.y, e3 = blockIdx.z;
  const long long e = e1 + (long long)g.k1 * (e2 + (long long)g.k2 * e3);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tables: per direction P, (Lambda, a0, a1), S
  for (int i = tid; i < 3 * (TB / 2); i += NT) {
    const int d = i / (TB / 2), ch = i - d * (TB / 2);
    const size_t row = d == 0 ? (size_t)e1 : (d == 1 ? (size_t)(g.k1 + e2) : (size_t)(g.k1 + g.k2 + e3));
    const double* src = etabP + row * ETS;
    const int o = 2 * ch;   // [0, MS + 3 MP) from the row start, then [MS + 3 MP, TB) from oS
    cpa16c(tb + d * TB + o, o < MS + 3 * 16 ? src + o : src + K::oS + (o - (MS + 3 * 16)));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  // padding column (index m) of both cube buffers: read by the transforms against zero S rows
  for (int r = tid; r < 2 * (K::CR + 8); r += NT) {
    double* B = r < K::CR + 8 ? C0 : C1;
    const int rr = r < K::CR + 8 ? r : r - (K::CR + 8);
    for (int c = M; c < 16; ++c) B[rr * LD + c] = 0.0;
  }
  pdl_wait();
  pdl_trigger();
  const long long N1 = (long long)g.k1 * P + 1, N2 = (long long)g.k2 * P + 1;
  // F_I -> C0[(i3 m + i2)][i1]
  for (int r = tid; r < MM; r += NT) {   // one interior grid row (i3, i2) per thread
    const int i3 = r / M, i2 = r - i3 * M;
    const double* src = Fg + (e1 * P + 1) + N1 * ((e2 * P + i2 + 1) + N2 * (long long)(e3 * P + i3 + 1));
#pragma unroll
    for (int i1 = 0; i1 < M; ++i1) cpa8c(&C0[r * LD + i1], src + i1);
  }
  if (MODE == 1) {   // face interiors of u_hat -> Fa[f][A][B] (A slow, B fast tangential index)
    const long long V12 = (long long)g.V1 * g.V2;
    for (int i = tid; i < 6 * MM; i += NT) {
      const int f = i / MM, l = i - f * MM, A = l / M, B = l - A * M, d = f >> 1, s = f & 1;
      // the face's record e + s e_d (periodic: the last element's high face is on record plane 0)
      const int w1 = wrap_rec(e1 + (d == 0 ? s : 0), g.k1, g.per & 1), w2 = wrap_rec(e2 + (d == 1 ? s : 0), g.k2, g.per & 2),
                w3 = wrap_rec(e3 + (d == 2 ? s : 0), g.k3, g.per & 4);
      const long long rb = (w1 + g.V1 * (long long)w2 + V12 * w3) * RS;
      cpa8c(&Fa[f * MS + A * LD + B], uh + rb + d * MM + l);
    }
    // padding rows / columns of the face arrays (read by the face transforms against zero P entries)
    for (int i = tid; i < 6 * 16; i += NT) {
      const int f = i >> 4, t = i & 15;
      for (int c = M; c < 16; ++c) { Fa[f * MS + t * LD + c] = 0.0; Fa[f * MS + c * LD + t] = 0.0; }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  const double *S1 = tb + 0 * TB + MS + 3 * 16, *S2 = tb + 1 * TB + MS + 3 * 16, *S3 = tb + 2 * TB + MS + 3 * 16;
  auto Pd = [&](int d) { return tb + d * TB; };
  const double *L1 = tb + MS, *L2 = tb + TB + MS, *L3 = tb + 2 * TB + MS;
  // forward transforms S^T along x1, x2, x3: C0 -> C1 -> C0 -> C1 ([b3][b2][b1] in C1)
  cube_pass<P, true>(C0, C1, S1, warp, lane);
  __syncthreads();
  cube_pass<P, true>(C1, C0, S2, warp, lane);
  __syncthreads();
  cube_pass<P, true>(C0, C1, S3, warp, lane);
  if (MODE == 1) {   // T_f = P_b U_f P_a^T into Fa (X scratch: C0, free now)
    double* X = C0;
    for (int job = warp; job < 12; job += K::NW) {   // X_f = U_f P_a^T
      const int f = job >> 1, mi = job & 1, d = f >> 1, da = (d == 0) ? 1 : 0;
      face_panel<false, true>(Fa + f * MS, Pd(da), X + f * MS, mi, lane);
    }
    __syncthreads();
    for (int job = warp; job < 12; job += K::NW) {   // T_f = P_b X_f
      const int f = job >> 1, mi = job & 1, d = f >> 1, db = (d == 2) ? 1 : 2;
      face_panel<false, false>(Pd(db), X + f * MS, Fa + f * MS, mi, lane);
    }
    __syncthreads();
    for (int r = tid; r < 6 * 16; r += NT)   // the scratch covered C0's padding column: zero it again
      for (int c = M; c < 16; ++c) C0[r * LD + c] = 0.0;
  }
  __syncthreads();
  // divide by D (recovery: after subtracting E = sum_f a_f (x) T_f), in C1
  {
    const double *a10 = tb + MS + 16, *a11 = tb + MS + 32, *a20 = tb + TB + MS + 16, *a21 = tb + TB + MS + 32,
                 *a30 = tb + 2 * TB + MS + 16, *a31 = tb + 2 * TB + MS + 32;
    for (int r = tid; r < MM; r += NT) {   // one row (b3, b2) per thread
      const int b3 = r / M, b2 = r - b3 * M;
      const double base = lam + L2[b2] + L3[b3];
      double t0 = 0.0, t1 = 0.0, c2 = 0.0, c3 = 0.0, c4 = 0.0, c5 = 0.0;
      if (MODE == 1) {
        t0 = Fa[0 * MS + b3 * LD + b2];
        t1 = Fa[1 * MS + b3 * LD + b2];
        c2 = a20[b2]; c3 = a21[b2]; c4 = a30[b3]; c5 = a31[b3];
      }
#pragma unroll
      for (int b1 = 0; b1 < M; ++b1) {
        double v = C1[r * LD + b1];
        if (MODE == 1) {
          double E = a10[b1] * t0;
          E = fma(a11[b1], t1, E);
          E = fma(c2, Fa[2 * MS + b3 * LD + b1], E);
          E = fma(c3, Fa[3 * MS + b3 * LD + b1], E);
          E = fma(c4, Fa[4 * MS + b2 * LD + b1], E);
          E = fma(c5, Fa[5 * MS + b2 * LD + b1], E);
          v -= E;
        }
        C1[r * LD + b1] = v * rcp3c(base + L1[b1]);
      }
    }
  }
  __syncthreads();
  if (MODE == 0) {
    // G_f[A][B] = sum_{b_d} a_f[b_d] V (into Fa, zero padded), then Yc_f = P_b^T G_f P_a; one (A, B)
    // per thread for all six faces (six independent accumulation chains)
    {
      const int A = tid >> 4, B = tid & 15;
      double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (A < M && B < M) {
        const double *a10 = tb + MS + 16, *a11 = tb + MS + 32, *a20 = tb + TB + MS + 16, *a21 = tb + TB + MS + 32,
                     *a30 = tb + 2 * TB + MS + 16, *a31 = tb + 2 * TB + MS + 32;
#pragma unroll
        for (int t = 0; t < M; ++t) {
          const double v0 = C1[(A * M + B) * LD + t];   // faces normal to x1: (b3, b2) = (A, B), b1 = t
          const double v1 = C1[(A * M + t) * LD + B];   // normal to x2: (b3, b1) = (A, B), b2 = t
          const double v2 = C1[(t * M + A) * LD + B];   // normal to x3: (b2, b1) = (A, B), b3 = t
          acc[0] = fma(a10[t], v0, acc[0]);
          acc[1] = fma(a11[t], v0, acc[1]);
          acc[2] = fma(a20[t], v1, acc[2]);
          acc[3] = fma(a21[t], v1, acc[3]);
          acc[4] = fma(a30[t], v2, acc[4]);
          acc[5] = fma(a31[t], v2, acc[5]);
        }
      }
#pragma unroll
      for (int f = 0; f < 6; ++f) Fa[f * MS + A * LD + B] = acc[f];
    }
    __syncthreads();
    double* X = C0;
    for (int job = warp; job < 12; job += K::NW) {   // X_f = G_f P_a
      const int f = job >> 1, mi = job & 1, d = f >> 1, da = (d == 0) ? 1 : 0;
      face_panel<false, false>(Fa + f * MS, Pd(da), X + f * MS, mi, lane);
    }
    __syncthreads();
    for (int job = warp; job < 12; job += K::NW) {   // Y_f = P_b^T X_f (into Fa)
      const int f = job >> 1, mi = job & 1, d = f >> 1, db = (d == 2) ? 1 : 2;
      face_panel<true, false>(Pd(db), X + f * MS, Fa + f * MS, mi, lane);
    }
    __syncthreads();
    double* Ye = Yc + (size_t)e * 6 * MM;
    for (int l = tid; l < MM; l += NT) {   // block position l for all six faces
      const int A = l / M, B = l - A * M;
#pragma unroll
      for (int f = 0; f < 6; ++f) Ye[f * MM + l] = Fa[f * MS + A * LD + B];
    }
  } else {
    // back transforms S along x1, x2, x3: C1 -> C0 -> C1 -> C0 ([i3][i2][i1] in C0), then store;
    // meanwhile vertex record e of u_hat is staged in Fa (the T faces are dead)
    {
      const long long rb = (e1 + g.V1 * (long long)e2 + (long long)g.V1 * g.V2 * e3) * RS;
      for (int i = tid; i < RS; i += NT) cpa8c(&Fa[i], uh + rb + i);
      asm volatile("cp.async.commit_group;\n" ::);
    }
    cube_pass<P, false>(C1, C0, S1, warp, lane);
    __syncthreads();
    cube_pass<P, false>(C0, C1, S2, warp, lane);
    __syncthreads();
    cube_pass<P, false>(C1, C0, S3, warp, lane);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // the element's grid block t in [0, p)^3: interior points from C0, the points with some t_d = 0
    // from vertex record e (its faces, edges and vertex are exactly those points; staged in Fa).  The
    // planes t_d = p of the last element of a row belong to the next record: launch_skel_scatter_hi.
    for (int r = tid; r < P * P; r += NT) {   // one grid row (t3, t2) of p points per thread
      const int t3 = r / P, t2 = r - t3 * P;
      double* dst = ug + (long long)e1 * P + N1 * ((e2 * P + t2) + N2 * (long long)(e3 * P + t3));
      const double* Rec = Fa;   // record e, RS entries
      if (t2 > 0 && t3 > 0) {
        dst[0] = Rec[(t3 - 1) * M + (t2 - 1)];                           // face f1 interior
        const double* row = C0 + ((t3 - 1) * M + (t2 - 1)) * LD;
#pragma unroll
        for (int t1 = 1; t1 < P; ++t1) dst[t1] = row[t1 - 1];
      } else if (t2 == 0 && t3 == 0) {
        dst[0] = Rec[3 * MM + 3 * M];                                    // vertex
#pragma unroll
        for (int t1 = 1; t1 < P; ++t1) dst[t1] = Rec[3 * MM + t1 - 1];   // edge e1
      } else if (t2 == 0) {                                              // t3 > 0: edge e3, face f2
        dst[0] = Rec[3 * MM + 2 * M + t3 - 1];
#pragma unroll
        for (int t1 = 1; t1 < P; ++t1) dst[t1] = Rec[MM + (t3 - 1) * M + t1 - 1];
      } else {                                                           // t3 == 0, t2 > 0: edge e2, face f3
        dst[0] = Rec[3 * MM + M + t2 - 1];
#pragma unroll
        for (int t1 = 1; t1 < P; ++t1) dst[t1] = Rec[2 * MM + (t2 - 1) * M + t1 - 1];
      }
    }
  }
}

cudaError_t launch_cr16(int mode, const LevelGeom& g, const double* Fg, const double* uh, const double* etabP, double lam,
                        double* Yc, double* ug, cudaStream_t st) {
  const dim3 grid((unsigned)g.k1, (unsigned)g.k2, (unsigned)g.k3);
  switch (g.p) {
#define CASE(PP)                                                                                                    \
  case PP:                                                                                                          \
    return mode == 0 ? launch_pdl(k_cr16<PP, 0>, grid, dim3(256), cr16_smem<PP>(), st, g, Fg, uh, etabP, lam, Yc, ug) \
                     : launch_pdl(k_cr16<PP, 1>, grid, dim3(256), cr16_smem<PP>(), st, g, Fg, uh, etabP, lam, Yc, ug);
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t cr16_set_smem_attr() {
  cudaError_t e = cudaSuccess;
#define CASE(PP)                                                                                            \
  {                                                                                                         \
    cudaError_t a = cudaFuncSetAttribute(k_cr16<PP, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cr16_smem<PP>()); \
    cudaError_t b = cudaFuncSetAttribute(k_cr16<PP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cr16_smem<PP>()); \
    if (a != cudaSuccess) e = a;                                                                            \
    if (b != cudaSuccess) e = b;                                                                            \
  }
  CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
  return e;
}

}  // namespace pmg
