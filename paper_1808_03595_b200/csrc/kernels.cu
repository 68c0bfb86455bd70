// FP64 CUDA kernels of the p-multigrid path for sm_100a (B200) besides the degree-specialised
// element operator and star smoother (hot_kernels.cu, star16.cu, elem16.cu).  Citations: P:n =
// PAPER.md line n.
//
//   k_restrict_local  per fine record: J^T of its faces/edges (closed, coarse)
//   k_restrict_gather coarse record entries gather the closed contributions
//   k_prolong         u_f += J_hat u_c per fine record
//   k_condense_elem / k_condense_gather   F_hat = F_B - H_BI H_II^-1 F_I
//   k_recover_elem    u_I = H_II^-1 (F_I - H_IB u_hat)
//   converters, weak RHS, BLAS-1, coarse-CG pieces.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "layout.cuh"

namespace pmg {

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("PMG_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// ------------------------------------------------------------------------------------------
// layout converters and weak right-hand side
// ------------------------------------------------------------------------------------------
__global__ void k_skel_from_grid(LevelGeom g, const double* __restrict__ grid, double* __restrict__ skel) {
  const long long N1 = (long long)g.k1 * g.p + 1, N2 = (long long)g.k2 * g.p + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.nskel;
       idx += (long long)gridDim.x * blockDim.x) {
    Entry E = decode_entry(g, idx);
    double v = 0.0;
    if (is_free(g, E.g1, E.g2, E.g3)) v = grid[E.g1 + N1 * (E.g2 + N2 * E.g3)];
    skel[idx] = v;
  }
}

__global__ void k_skel_to_grid(LevelGeom g, const double* __restrict__ skel, double* __restrict__ grid) {
  const int N1 = g.k1 * g.p + 1, N2 = g.k2 * g.p + 1, N3 = g.k3 * g.p + 1;
  const long long tot = (long long)N1 * N2 * N3;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int i1 = (int)(idx % N1);
    long long r = idx / N1;
    int i2 = (int)(r % N2), i3 = (int)(r / N2);
    bool sk = (i1 % g.p == 0) || (i2 % g.p == 0) || (i3 % g.p == 0);
    double v = 0.0;
    int w1 = i1, w2 = i2, w3 = i3;
    wrap_pt(g, w1, w2, w3);   // periodic: the duplicate last plane shows plane 0
    if (sk && is_free(g, w1, w2, w3)) v = skel[skel_index(g, w1, w2, w3)];
    grid[idx] = v;
  }
}

// skeleton values -> their grid points only (the recovery writes every element interior): one block
// per vertex record (3-D grid), the record's face interiors, edge interiors and vertex; entries of the
// record that lie outside the box (faces / edges of records on the high box faces) are skipped
template <int P>
__global__ void __launch_bounds__(128) k_skel_scatter_t(LevelGeom g, const double* __restrict__ skel,
                                                        double* __restrict__ grid, int o1, int o2, int o3) {
  pdl_wait();
  pdl_trigger();
  constexpr int m = P - 1, mm = m * m, RS = 3 * mm + 3 * m + 1;
  const int v1 = blockIdx.x + o1, v2 = blockIdx.y + o2, v3 = blockIdx.z + o3;   // record (offset grid)
  const long long N1 = (long long)g.k1 * P + 1, N2 = (long long)g.k2 * P + 1;
  const int r1 = ((g.per & 1) && v1 == g.k1) ? 0 : v1, r2 = ((g.per & 2) && v2 == g.k2) ? 0 : v2,
            r3 = ((g.per & 4) && v3 == g.k3) ? 0 : v3;   // periodic: the duplicate plane shows plane 0
  const double* R = skel + (r1 + (long long)g.V1 * (r2 + (long long)g.V2 * r3)) * RS;
  const long long g0 = (long long)v1 * P + N1 * ((long long)v2 * P + N2 * (long long)v3 * P);
  const bool in1 = v1 < g.k1, in2 = v2 < g.k2, in3 = v3 < g.k3;
  for (int l = threadIdx.x; l < mm; l += blockDim.x) {
    const int a = l / m, b = l - a * m;   // a: slow, b: fast in-face index (record layout)
    if (in2 && in3) grid[g0 + N1 * ((b + 1) + N2 * (long long)(a + 1))] = R[l];                 // f1: (t3, t2)
    if (in1 && in3) grid[g0 + (b + 1) + N1 * N2 * (long long)(a + 1)] = R[mm + l];              // f2: (t3, t1)
    if (in1 && in2) grid[g0 + (b + 1) + N1 * (long long)(a + 1)] = R[2 * mm + l];               // f3: (t2, t1)
  }
  for (int t = threadIdx.x; t < m; t += blockDim.x) {
    if (in1) grid[g0 + t + 1] = R[3 * mm + t];
    if (in2) grid[g0 + N1 * (t + 1)] = R[3 * mm + m + t];
    if (in3) grid[g0 + N1 * N2 * (long long)(t + 1)] = R[3 * mm + 2 * m + t];
  }
  if (threadIdx.x == 0) grid[g0] = R[3 * mm + 3 * m];
}

cudaError_t launch_skel_scatter(const LevelGeom& g, const double* skel, double* grid, cudaStream_t st, bool hi_only) {
  if (hi_only) {   // the records of the three high box planes (v_d = k_d)
    cudaError_t e;
    const LevelGeom* gp = &g;
    auto one = [&](dim3 grd, int o1, int o2, int o3) -> cudaError_t {
      switch (gp->p) {
#define CASE(P) case P: return launch_pdl(k_skel_scatter_t<P>, grd, dim3(128), 0, st, g, skel, grid, o1, o2, o3);
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14)
        CASE(15) CASE(16) CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24) CASE(25) CASE(26)
        CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
        default: return cudaErrorInvalidValue;
      }
    };
    if ((e = one(dim3(1, (unsigned)g.V2, (unsigned)g.V3), g.k1, 0, 0)) != cudaSuccess) return e;
    if ((e = one(dim3((unsigned)g.V1, 1, (unsigned)g.V3), 0, g.k2, 0)) != cudaSuccess) return e;
    return one(dim3((unsigned)g.V1, (unsigned)g.V2, 1), 0, 0, g.k3);
  }
  const dim3 grd((unsigned)g.V1, (unsigned)g.V2, (unsigned)g.V3);
  switch (g.p) {
#define CASE(P) case P: return launch_pdl(k_skel_scatter_t<P>, grd, dim3(128), 0, st, g, skel, grid, 0, 0, 0);
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14)
    CASE(15) CASE(16) CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24) CASE(25) CASE(26)
    CASE(27) CASE(28) CASE(29) CASE(30) CASE(31) CASE(32)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

// F = b1[i1] b2[i2] b3[i3] f (assembled GLL-lumped mass is a tensor product of 1-D assembled masses)
__global__ void k_weak_rhs(LevelGeom g, const double* __restrict__ b1, const double* __restrict__ b2,
                           const double* __restrict__ b3, const double* __restrict__ f, double* __restrict__ F) {
  const int N1 = g.k1 * g.p + 1, N2 = g.k2 * g.p + 1, N3 = g.k3 * g.p + 1;
  const long long tot = (long long)N1 * N2 * N3;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    int i1 = (int)(idx % N1);
    long long r = idx / N1;
    int i2 = (int)(r % N2), i3 = (int)(r / N2);
    F[idx] = is_free(g, i1, i2, i3) ? b3[i3 + g.zoff * g.p] * b2[i2] * b1[i1] * f[idx] : 0.0;   // b3: global line
  }
}

// ------------------------------------------------------------------------------------------
// restriction J_hat^T (two phases) and prolongation J_hat
// ------------------------------------------------------------------------------------------
size_t transfer_smem(int pf, int pc) {
  int mf = pf - 1, qc = pc + 1;
  size_t rt = (size_t)(3 * qc * qc + 3 * qc + 1 + mf * qc + mf * qc + mf * mf + qc * mf);
  // register-tiled kernels (pf <= 16): closed coarse record (even length), J padded to even rows, X of 3 faces
  size_t tl = (size_t)(3 * qc * qc + 3 * qc + 2 + mf * (qc + 1) + 3 * qc * mf + 3 * mf * mf + 3 * mf + 2);
  return sizeof(double) * (rt > tl ? rt : tl);
}

// register-tiled face transforms of the transfer kernels (compile-time degrees, p_f <= 16): a thread
// owns one row (or column) of a face in registers and reads J as broadcast 16-byte shared loads, one
// load per two FMAs instead of two loads per FMA; every output is summed in the same order as in
// the plain loops, so the results are bitwise the same
template <int PF_, int PC_> struct TransferTile {
  static constexpr bool on = PF_ > 0 && PF_ <= 16;
  static constexpr int MF = PF_ > 0 ? PF_ - 1 : 1, QC = PC_ + 1, QP = (QC + 1) & ~1;
};

// Z[v] = [3 closed coarse faces qc x qc][3 closed coarse edges qc][vertex]
// PF_ / PC_ > 0: degrees known at compile time (unrolled loops, constant divisions); 0: runtime
template <int PF_, int PC_>
__global__ void k_restrict_local_t(LevelGeom gf, int pc_rt, const double* __restrict__ Jint,
                                   const double* __restrict__ rf, double* __restrict__ Z) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double smt[];
  double* sm = smt;
  using TT = TransferTile<PF_, PC_>;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (TT::on) {
    constexpr int MF = TT::MF, QC = TT::QC, QP = TT::QP, ZSc = 3 * QC * QC + 3 * QC + 1;
    double* Jp = sm;                // MF x QP (rows padded to an even length)
    double* X3 = Jp + MF * QP;      // 3 x MF x QC
    double* F3 = X3 + 3 * MF * QC;  // the record's 3 face interiors (contiguous in the record)
    for (int i = tid; i < MF * QP; i += nt) {
      const int ia = i / QP, al = i - ia * QP;
      Jp[i] = al < QC ? Jint[ia * QC + al] : 0.0;
    }
    const long long rec = blockIdx.x;
    const double* R = rf + rec * gf.RS;
    double* Zr = Z + rec * ZSc;
    for (int i = tid; i < 3 * MF * MF; i += nt) F3[i] = R[i];
    __syncthreads();
    for (int row = tid; row < 3 * MF; row += nt) {   // X[d][ib][:] = sum_ia F_d[ib][ia] J[ia][:]
      const double* F = F3 + row * MF;               // row = d * MF + ib
      double x[QP];
#pragma unroll
      for (int al = 0; al < QP; ++al) x[al] = 0.0;
#pragma unroll 3
      for (int ia = 0; ia < MF; ++ia) {
        const double fv = F[ia];
#pragma unroll
        for (int a2 = 0; a2 < QP / 2; ++a2) {
          const double2 j = *reinterpret_cast<const double2*>(Jp + ia * QP + 2 * a2);
          x[2 * a2] = fma(fv, j.x, x[2 * a2]);
          x[2 * a2 + 1] = fma(fv, j.y, x[2 * a2 + 1]);
        }
      }
#pragma unroll
      for (int al = 0; al < QC; ++al) X3[row * QC + al] = x[al];
    }
    __syncthreads();
    for (int c = tid; c < 3 * QC; c += nt) {         // Z[d][:][al] = sum_ib J[ib][:] X[d][ib][al]
      const int d = c / QC, al = c - d * QC;
      double z[QP];
#pragma unroll
      for (int be = 0; be < QP; ++be) z[be] = 0.0;
#pragma unroll 3
      for (int ib = 0; ib < MF; ++ib) {
        const double xv = X3[(d * MF + ib) * QC + al];
#pragma unroll
        for (int b2 = 0; b2 < QP / 2; ++b2) {
          const double2 j = *reinterpret_cast<const double2*>(Jp + ib * QP + 2 * b2);
          z[2 * b2] = fma(j.x, xv, z[2 * b2]);
          z[2 * b2 + 1] = fma(j.y, xv, z[2 * b2 + 1]);
        }
      }
#pragma unroll
      for (int be = 0; be < QC; ++be) Zr[d * QC * QC + be * QC + al] = z[be];
    }
    for (int i = tid; i < 3 * QC; i += nt) {
      const int d = i / QC, al = i - d * QC;
      const double* E = R + off_edge(MF, d);
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < MF; ++t) s += Jp[t * QP + al] * E[t];
      Zr[3 * QC * QC + i] = s;
    }
    if (tid == 0) Zr[ZSc - 1] = R[off_vert(MF)];
    return;
  }
  const int pc = PC_ > 0 ? PC_ : pc_rt;
  const int mf = PF_ > 0 ? PF_ - 1 : gf.m, qc = pc + 1, ZS = 3 * qc * qc + 3 * qc + 1;
  double* J = sm;             // mf x qc
  double* X = J + mf * qc;    // mf x qc
  for (int i = tid; i < mf * qc; i += nt) J[i] = Jint[i];
  __syncthreads();
  const long long rec = blockIdx.x;
  const double* R = rf + rec * gf.RS;
  double* Zr = Z + rec * ZS;
  for (int d = 0; d < 3; ++d) {
    const double* F = R + off_face(mf, d);
    for (int i = tid; i < mf * qc; i += nt) {  // X[ib][al] = sum_ia F[ib][ia] J[ia][al]
      int ib = i / qc, al = i - ib * qc;
      double s = 0.0;
      for (int ia = 0; ia < mf; ++ia) s += F[ib * mf + ia] * J[ia * qc + al];
      X[i] = s;
    }
    __syncthreads();
    for (int i = tid; i < qc * qc; i += nt) {  // Z[be][al] = sum_ib J[ib][be] X[ib][al]
      int be = i / qc, al = i - be * qc;
      double s = 0.0;
      for (int ib = 0; ib < mf; ++ib) s += J[ib * qc + be] * X[ib * qc + al];
      Zr[d * qc * qc + i] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < 3 * qc; i += nt) {
    int d = i / qc, al = i - d * qc;
    const double* E = R + off_edge(mf, d);
    double s = 0.0;
    for (int t = 0; t < mf; ++t) s += J[t * qc + al] * E[t];
    Zr[3 * qc * qc + i] = s;
  }
  if (tid == 0) Zr[ZS - 1] = R[off_vert(mf)];
}

template <int PC_>
__global__ void k_restrict_gather_t(LevelGeom gc, const double* __restrict__ Z, double* __restrict__ fc,
                                    double* __restrict__ uzero) {
  pdl_wait();
  pdl_trigger();
  const int pc = PC_ > 0 ? PC_ : gc.p, qc = pc + 1, ZS = 3 * qc * qc + 3 * qc + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < gc.nskel;
       idx += (long long)gridDim.x * blockDim.x) {
    Entry E;
    if (PC_ > 1 && gc.nskel < (1ll << 31)) E = decode_entry_t<(PC_ > 1 ? PC_ : 2)>(gc, (unsigned)idx);
    else E = decode_entry(gc, idx);
    double s = 0.0;
    if (is_free(gc, E.g1, E.g2, E.g3) && owned_plane(gc, E.v3)) {
      const int G[3] = {E.g1, E.g2, E.g3};
      const int K[3] = {gc.k1, gc.k2, gc.k3};
      int cand[3][2], loc[3][2], nc[3];   // candidate records along d and the point's local coordinate there
      bool mult[3];
      for (int d = 0; d < 3; ++d) {
        mult[d] = (G[d] % pc) == 0;
        cand[d][0] = G[d] / pc;
        loc[d][0] = G[d] - cand[d][0] * pc;
        nc[d] = 1;
        const bool per = (gc.per >> d) & 1;
        if (mult[d] && (cand[d][0] - 1 >= 0 || per)) {   // periodic: plane 0 closes the last record
          cand[d][1] = cand[d][0] - 1 >= 0 ? cand[d][0] - 1 : K[d] - 1;
          loc[d][1] = pc;
          nc[d] = 2;
        }
        if (cand[d][0] > K[d]) nc[d] = 0;  // cannot happen for points inside the box
      }
      auto rec = [&](int w1, int w2, int w3) -> long long {
        return ((long long)w1 + (long long)gc.V1 * ((long long)w2 + (long long)gc.V2 * w3)) * ZS;
      };
      // faces normal to d containing the point: w_d = G_d / pc, tangential candidates
      for (int d = 0; d < 3; ++d) {
        if (!mult[d]) continue;
        const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
        for (int ib = 0; ib < nc[db]; ++ib)
          for (int ia = 0; ia < nc[da]; ++ia) {
            int w[3];
            w[d] = G[d] / pc; w[da] = cand[da][ia]; w[db] = cand[db][ib];
            const int be = loc[db][ib], al = loc[da][ia];
            s += Z[rec(w[0], w[1], w[2]) + d * qc * qc + be * qc + al];
          }
      }
      // edges along d containing the point
      for (int d = 0; d < 3; ++d) {
        const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
        if (!(mult[da] && mult[db])) continue;
        for (int i = 0; i < nc[d]; ++i) {
          int w[3];
          w[d] = cand[d][i]; w[da] = G[da] / pc; w[db] = G[db] / pc;
          s += Z[rec(w[0], w[1], w[2]) + 3 * qc * qc + d * qc + loc[d][i]];
        }
      }
      if (mult[0] && mult[1] && mult[2]) s += Z[rec(G[0] / pc, G[1] / pc, G[2] / pc) + ZS - 1];
    }
    fc[idx] = s;
    if (uzero) uzero[idx] = 0.0;   // Alg. 3: u_(l-1) <- 0 before its smoothing, fused here
  }
}

template <int PF_, int PC_>
__global__ void k_prolong_t(LevelGeom gf, LevelGeom gc, const double* __restrict__ Jint,
                            const double* __restrict__ uc, double* __restrict__ uf) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double smt[];
  double* sm = smt;
  using TT = TransferTile<PF_, PC_>;
  const int pf = PF_ > 0 ? PF_ : gf.p, mf = pf - 1, pc = PC_ > 0 ? PC_ : gc.p, qc = pc + 1;
  double* C = sm;                      // 3 qc^2 closed faces, 3 qc closed edges, 1 vertex
  // tiled: J rows padded to an even length on a 16-byte boundary (Jld = QP), else mf x qc
  const int Jld = TT::on ? TT::QP : qc;
  double* J = C + (TT::on ? ((3 * qc * qc + 3 * qc + 2) & ~1) : 3 * qc * qc + 3 * qc + 1);
  double* X = J + mf * Jld;            // qc x mf (tiled: 3 faces)
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long rec = blockIdx.x;
  const int v1 = (int)(rec % gf.V1), v2 = (int)((rec / gf.V1) % gf.V2), v3 = (int)(rec / ((long long)gf.V1 * gf.V2));
  for (int i = tid; i < mf * Jld; i += nt) {
    const int ia = i / Jld, al = i - ia * Jld;
    J[i] = al < qc ? Jint[ia * qc + al] : 0.0;
  }
  for (int i = tid; i < 3 * qc * qc; i += nt) {
    int d = i / (qc * qc), rr = i - d * qc * qc, be = rr / qc, al = rr - be * qc;
    int G1 = v1 * pc, G2 = v2 * pc, G3 = v3 * pc;
    if (d == 0) { G3 += be; G2 += al; } else if (d == 1) { G3 += be; G1 += al; } else { G2 += be; G1 += al; }
    wrap_pt(gc, G1, G2, G3);   // periodic: the closed face of the last record ends on plane 0
    long long ci;
    if constexpr (PC_ > 0) ci = skel_index_t<(PC_ > 0 ? PC_ : 1)>(gc, G1, G2, G3);
    else ci = skel_index(gc, G1, G2, G3);
    C[i] = inside(gc, G1, G2, G3) ? uc[ci] : 0.0;
  }
  for (int i = tid; i < 3 * qc + 1; i += nt) {
    int G1 = v1 * pc, G2 = v2 * pc, G3 = v3 * pc;
    if (i < 3 * qc) {
      int d = i / qc, al = i - d * qc;
      if (d == 0) G1 += al; else if (d == 1) G2 += al; else G3 += al;
    }
    wrap_pt(gc, G1, G2, G3);
    long long ci;
    if constexpr (PC_ > 0) ci = skel_index_t<(PC_ > 0 ? PC_ : 1)>(gc, G1, G2, G3);
    else ci = skel_index(gc, G1, G2, G3);
    C[3 * qc * qc + i] = inside(gc, G1, G2, G3) ? uc[ci] : 0.0;
  }
  double* Ur = uf + rec * gf.RS;
  if constexpr (TT::on) {   // the fine record is staged, updated in shared memory and written back whole (coalesced)
    constexpr int MF = TT::MF, QC = TT::QC, RSc = 3 * MF * MF + 3 * MF + 1;
    double* Us = X + 3 * QC * MF;
    for (int i = tid; i < RSc; i += nt) Us[i] = Ur[i];
  }
  __syncthreads();
  if constexpr (TT::on) {
    constexpr int MF = TT::MF, QC = TT::QC, QP = TT::QP, RSc = 3 * MF * MF + 3 * MF + 1;
    double* Us = X + 3 * QC * MF;
    for (int row = tid; row < 3 * QC; row += nt) {   // X[d][be][:] = sum_al C_d[be][al] J[:][al]
      const double* Cr = C + row * QC;               // row = d * QC + be
      double cr[QC];
#pragma unroll
      for (int al = 0; al < QC; ++al) cr[al] = Cr[al];
#pragma unroll 3
      for (int ia = 0; ia < MF; ++ia) {
        double sx = 0.0;
#pragma unroll
        for (int a2 = 0; a2 < QP / 2; ++a2) {
          const double2 j = *reinterpret_cast<const double2*>(J + ia * QP + 2 * a2);
          sx = fma(cr[2 * a2], j.x, sx);
          if (2 * a2 + 1 < QC) sx = fma(cr[2 * a2 + 1 < QC ? 2 * a2 + 1 : 0], j.y, sx);
        }
        X[row * MF + ia] = sx;
      }
    }
    __syncthreads();
    for (int c = tid; c < 3 * MF; c += nt) {         // F_d[:][ia] = sum_be J[:][be] X[d][be][ia]
      const int d = c / MF, ia = c - d * MF;
      double xc[QC];
#pragma unroll
      for (int be = 0; be < QC; ++be) xc[be] = X[(d * QC + be) * MF + ia];
      int g1 = v1 * PF_, g2 = v2 * PF_, g3 = v3 * PF_;
      if (d == 0) g2 += ia + 1; else g1 += ia + 1;
#pragma unroll 3
      for (int ib = 0; ib < MF; ++ib) {
        double sf = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < QP / 2; ++b2) {
          const double2 j = *reinterpret_cast<const double2*>(J + ib * QP + 2 * b2);
          sf = fma(j.x, xc[2 * b2], sf);
          if (2 * b2 + 1 < QC) sf = fma(j.y, xc[2 * b2 + 1 < QC ? 2 * b2 + 1 : 0], sf);
        }
        const int h1 = g1, h2 = d == 2 ? g2 + ib + 1 : g2, h3 = d == 2 ? g3 : g3 + ib + 1;
        if (is_free(gf, h1, h2, h3)) Us[off_face(MF, d) + ib * MF + ia] += sf;
      }
    }
    for (int i = tid; i < 3 * MF + 1; i += nt) {
      int g1 = v1 * PF_, g2 = v2 * PF_, g3 = v3 * PF_;
      double s;
      if (i < 3 * MF) {
        const int d = i / MF, t = i - d * MF;
        const double* Ce = C + 3 * QC * QC + d * QC;
        s = 0.0;
#pragma unroll
        for (int al = 0; al < QC; ++al) s += J[t * QP + al] * Ce[al];
        if (d == 0) g1 += t + 1; else if (d == 1) g2 += t + 1; else g3 += t + 1;
      } else {
        s = C[3 * QC * QC + 3 * QC];
      }
      if (is_free(gf, g1, g2, g3)) Us[off_edge(MF, 0) + i] += s;   // edges then vertex are contiguous
    }
    __syncthreads();
    for (int i = tid; i < RSc; i += nt) Ur[i] = Us[i];
    return;
  }
  for (int d = 0; d < 3; ++d) {
    const double* Cd = C + d * qc * qc;
    for (int i = tid; i < qc * mf; i += nt) {  // X[be][ia] = sum_al C[be][al] J[ia][al]
      int be = i / mf, ia = i - be * mf;
      double s = 0.0;
      for (int al = 0; al < qc; ++al) s += Cd[be * qc + al] * J[ia * qc + al];
      X[i] = s;
    }
    __syncthreads();
    for (int i = tid; i < mf * mf; i += nt) {  // F[ib][ia] = sum_be J[ib][be] X[be][ia]
      int ib = i / mf, ia = i - ib * mf;
      double s = 0.0;
      for (int be = 0; be < qc; ++be) s += J[ib * qc + be] * X[be * mf + ia];
      int g1 = v1 * pf, g2 = v2 * pf, g3 = v3 * pf;
      if (d == 0) { g3 += ib + 1; g2 += ia + 1; } else if (d == 1) { g3 += ib + 1; g1 += ia + 1; } else { g2 += ib + 1; g1 += ia + 1; }
      if (is_free(gf, g1, g2, g3)) Ur[off_face(mf, d) + i] += s;
    }
    __syncthreads();
  }
  for (int i = tid; i < 3 * mf + 1; i += nt) {
    int g1 = v1 * pf, g2 = v2 * pf, g3 = v3 * pf;
    double s;
    if (i < 3 * mf) {
      int d = i / mf, t = i - d * mf;
      const double* Ce = C + 3 * qc * qc + d * qc;
      s = 0.0;
      for (int al = 0; al < qc; ++al) s += J[t * qc + al] * Ce[al];
      if (d == 0) g1 += t + 1; else if (d == 1) g2 += t + 1; else g3 += t + 1;
    } else {
      s = C[3 * qc * qc + 3 * qc];
    }
    if (is_free(gf, g1, g2, g3)) Ur[off_edge(mf, 0) + i] += s;   // edges then vertex are contiguous
  }
}

// ------------------------------------------------------------------------------------------
// condensation and interior recovery (O(p^4) per element via the interior fast diagonalisation)
// cube[i3][i2][i1] in shared memory when it fits, else in a global scratch slot per block
// ------------------------------------------------------------------------------------------
// MT > 0: compile-time m (line held in registers, loops unrolled); MT = 0: runtime m
template <int MT>
__device__ void cube_transform(double* cube, int m_rt, const double* S1, const double* S2, const double* S3,
                               bool transpose) {
  // transpose = true: out[b] = sum_i S[i][b] in[i]  (S^T);  false: out[i] = sum_b S[i][b] in[b]
  const int m = MT ? MT : m_rt;
  const int tid = threadIdx.x, nt = blockDim.x, mm = m * m;
  double tmp[MT ? MT : 32];
  double lin[MT ? MT : 1];
  for (int dir = 0; dir < 3; ++dir) {
    const double* S = dir == 0 ? S1 : (dir == 1 ? S2 : S3);
    for (int line = tid; line < mm; line += nt) {
      int A = line / m, B = line - A * m;
      int base, stride;
      if (dir == 0) { base = (A * m + B) * m; stride = 1; }          // (i3, i2), along i1
      else if (dir == 1) { base = A * mm + B; stride = m; }         // (i3, i1), along i2
      else { base = A * m + B; stride = mm; }                       // (i2, i1), along i3
      if (MT) {
#pragma unroll
        for (int i = 0; i < (MT ? MT : 1); ++i) lin[i] = cube[base + i * stride];
#pragma unroll
        for (int o = 0; o < (MT ? MT : 1); ++o) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < (MT ? MT : 1); ++i) s = fma(transpose ? S[i * m + o] : S[o * m + i], lin[i], s);
          tmp[o] = s;
        }
      } else {
        for (int o = 0; o < m; ++o) {
          double s = 0.0;
          for (int i = 0; i < m; ++i) s += (transpose ? S[i * m + o] : S[o * m + i]) * cube[base + i * stride];
          tmp[o] = s;
        }
      }
      for (int o = 0; o < m; ++o) cube[base + o * stride] = tmp[o];
    }
    __syncthreads();
  }
}

size_t condense_smem(int p, int ET, bool cube_in_smem) {
  int m = p - 1;
  return sizeof(double) * (size_t)((cube_in_smem ? m * m * m : 0) + 6 * m * m + m * m + 3 * ET + 6 * (p + 1) * (p + 1));
}

// Yc[e] (6 m^2) = (H_BI H_II^-1 F_I) on the six face interiors of element e
// PT > 0: compile-time degree; PT = 0: runtime degree
template <int PT>
__global__ void __launch_bounds__(256) k_condense_elem(LevelGeom g, const double* __restrict__ Fg,
                                                       const double* __restrict__ etab, double lam,
                                                       double* __restrict__ Yc, double* __restrict__ cube_g) {
  extern __shared__ double sm[];
  const int p = PT ? PT : g.p, m = p - 1, mm = m * m, ET = g.ET;
  const bool cube_in_smem = (cube_g == nullptr);
  double* G = sm;
  double* X = G + 6 * mm;
  double* tb = X + mm;
  double* cube = cube_in_smem ? (tb + 3 * ET + 6 * (p + 1) * (p + 1)) : cube_g + (size_t)blockIdx.x * mm * m;
  const long long N1 = (long long)g.k1 * p + 1, N2 = (long long)g.k2 * p + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (long long e = blockIdx.x; e < g.nelem; e += gridDim.x) {
    const int e1 = (int)(e % g.k1), e2 = (int)((e / g.k1) % g.k2), e3 = (int)(e / ((long long)g.k1 * g.k2));
    const double* src[3] = {etab + (size_t)e1 * ET, etab + (size_t)(g.k1 + e2) * ET, etab + (size_t)(g.k1 + g.k2 + e3) * ET};
    __syncthreads();
    for (int i = tid; i < 3 * ET; i += nt) { int d = i / ET; tb[i] = src[d][i - d * ET]; }
    for (int i = tid; i < mm * m; i += nt) {
      int i3 = i / mm, r = i - i3 * mm, i2 = r / m, i1 = r - i2 * m;
      cube[i] = Fg[(e1 * p + i1 + 1) + N1 * ((e2 * p + i2 + 1) + N2 * (long long)(e3 * p + i3 + 1))];
    }
    __syncthreads();
    cube_transform<PT ? PT - 1 : 0>(cube, m, tb + et_S(p), tb + ET + et_S(p), tb + 2 * ET + et_S(p), true);
    const double *L1 = tb + et_lam(p), *L2 = tb + ET + et_lam(p), *L3 = tb + 2 * ET + et_lam(p);
    for (int i = tid; i < mm * m; i += nt) {
      int b3 = i / mm, r = i - b3 * mm, b2 = r / m, b1 = r - b2 * m;
      cube[i] /= (lam + L1[b1] + L2[b2] + L3[b3]);
    }
    __syncthreads();
    // contract to faces: G_f[bb][ba] = sum_{bd} a_f[bd] V
    for (int i = tid; i < 6 * mm; i += nt) {
      int f = i / mm, r = i - f * mm, A = r / m, B = r - A * m, d = f >> 1, s = f & 1;
      const double* af = tb + d * ET + (s ? et_a1(p) : et_a0(p));
      double acc = 0.0;
      for (int t = 0; t < m; ++t) {
        int b1, b2, b3;
        if (d == 0) { b1 = t; b3 = A; b2 = B; } else if (d == 1) { b2 = t; b3 = A; b1 = B; } else { b3 = t; b2 = A; b1 = B; }
        acc += af[t] * cube[(b3 * m + b2) * m + b1];
      }
      G[i] = acc;
    }
    __syncthreads();
    for (int f = 0; f < 6; ++f) {
      const int d = f >> 1, da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
      const double* Pa = tb + da * ET + et_P(p);
      const double* Pb = tb + db * ET + et_P(p);
      const double* Gf = G + f * mm;
      for (int i = tid; i < mm; i += nt) {
        int bb = i / m, ia = i - bb * m;
        double s = 0.0;
        for (int ba = 0; ba < m; ++ba) s += Gf[bb * m + ba] * Pa[ba * m + ia];
        X[i] = s;
      }
      __syncthreads();
      for (int i = tid; i < mm; i += nt) {
        int ib = i / m, ia = i - ib * m;
        double s = 0.0;
        for (int bb = 0; bb < m; ++bb) s += Pb[bb * m + ib] * X[bb * m + ia];
        Yc[(size_t)e * 6 * mm + f * mm + i] = s;
      }
      __syncthreads();
    }
  }
}

__global__ void k_condense_gather(LevelGeom g, const double* __restrict__ Fg, const double* __restrict__ Yc,
                                  double* __restrict__ fhat) {
  const int m = g.m, mm = m * m;
  const long long N1 = (long long)g.k1 * g.p + 1, N2 = (long long)g.k2 * g.p + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.nskel;
       idx += (long long)gridDim.x * blockDim.x) {
    Entry E = decode_entry(g, idx);
    double r = 0.0;
    if (is_free(g, E.g1, E.g2, E.g3) && owned_plane(g, E.v3)) {
      r = Fg[E.g1 + N1 * (E.g2 + N2 * (long long)E.g3)];
      if (E.type < 3) {
        const int d = E.type, o = E.a * m + E.b;
        int w1 = E.v1, w2 = E.v2, w3 = E.v3;
        if (d == 0) w1 -= 1; else if (d == 1) w2 -= 1; else w3 -= 1;
        w1 = wrap_rec(w1, g.k1, g.per & 1);   // periodic: element k - 1 precedes element 0
        w2 = wrap_rec(w2, g.k2, g.per & 2);
        w3 = wrap_rec(w3, g.k3, g.per & 4);
        const bool lo_in = w1 >= 0 && w2 >= 0 && w3 >= 0;                               // Neumann face: one side
        const bool hi_in = E.v1 < g.k1 && E.v2 < g.k2 && E.v3 < g.k3;
        size_t elo = lo_in ? (size_t)w1 + (size_t)g.k1 * ((size_t)w2 + (size_t)g.k2 * w3) : 0;
        size_t ehi = hi_in ? (size_t)E.v1 + (size_t)g.k1 * ((size_t)E.v2 + (size_t)g.k2 * E.v3) : 0;
        r -= (lo_in ? Yc[elo * 6 * mm + (2 * d + 1) * mm + o] : 0.0) + (hi_in ? Yc[ehi * 6 * mm + (2 * d) * mm + o] : 0.0);
      }
    }
    fhat[idx] = r;
  }
}

// u_I = S (x) S (x) S [ (S^T (x) S^T (x) S^T F_I - sum_f a_f (x) T_f) / D ],  T_f = (P_b (x) P_a) u_f
template <int PT>
__global__ void __launch_bounds__(256) k_recover_elem(LevelGeom g, const double* __restrict__ Fg,
                                                      const double* __restrict__ uh, const double* __restrict__ etab,
                                                      double lam, double* __restrict__ ug, double* __restrict__ cube_g) {
  extern __shared__ double sm[];
  const int p = PT ? PT : g.p, m = p - 1, mm = m * m, ET = g.ET, q = p + 1;
  const bool cube_in_smem = (cube_g == nullptr);
  double* T = sm;              // 6 mm
  double* X = T + 6 * mm;      // mm
  double* tb = X + mm;         // 3 ET
  double* Uf = tb + 3 * ET;    // 6 q^2 (face interiors use m^2 of each)
  double* cube = cube_in_smem ? (Uf + 6 * q * q) : cube_g + (size_t)blockIdx.x * mm * m;
  const long long N1 = (long long)g.k1 * p + 1, N2 = (long long)g.k2 * p + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (long long e = blockIdx.x; e < g.nelem; e += gridDim.x) {
    const int e1 = (int)(e % g.k1), e2 = (int)((e / g.k1) % g.k2), e3 = (int)(e / ((long long)g.k1 * g.k2));
    const double* src[3] = {etab + (size_t)e1 * ET, etab + (size_t)(g.k1 + e2) * ET, etab + (size_t)(g.k1 + g.k2 + e3) * ET};
    __syncthreads();
    for (int i = tid; i < 3 * ET; i += nt) { int d = i / ET; tb[i] = src[d][i - d * ET]; }
    for (int i = tid; i < mm * m; i += nt) {
      int i3 = i / mm, r = i - i3 * mm, i2 = r / m, i1 = r - i2 * m;
      cube[i] = Fg[(e1 * p + i1 + 1) + N1 * ((e2 * p + i2 + 1) + N2 * (long long)(e3 * p + i3 + 1))];
    }
    for (int i = tid; i < 6 * mm; i += nt) {  // face interiors of u_hat
      int f = i / mm, r = i - f * mm, A = r / m, B = r - A * m, d = f >> 1, s = f & 1, t1, t2, t3;
      if (d == 0) { t1 = s * p; t3 = A + 1; t2 = B + 1; } else if (d == 1) { t2 = s * p; t3 = A + 1; t1 = B + 1; }
      else { t3 = s * p; t2 = A + 1; t1 = B + 1; }
      int G1 = e1 * p + t1, G2 = e2 * p + t2, G3 = e3 * p + t3;
      wrap_pt(g, G1, G2, G3);
      Uf[i] = uh[skel_index(g, G1, G2, G3)];
    }
    __syncthreads();
    for (int f = 0; f < 6; ++f) {
      const int d = f >> 1, da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
      const double* Pa = tb + da * ET + et_P(p);
      const double* Pb = tb + db * ET + et_P(p);
      const double* U = Uf + f * mm;
      for (int i = tid; i < mm; i += nt) {
        int ib = i / m, ba = i - ib * m;
        double s = 0.0;
        for (int ia = 0; ia < m; ++ia) s += U[ib * m + ia] * Pa[ba * m + ia];
        X[i] = s;
      }
      __syncthreads();
      for (int i = tid; i < mm; i += nt) {
        int bb = i / m, ba = i - bb * m;
        double s = 0.0;
        for (int ib = 0; ib < m; ++ib) s += Pb[bb * m + ib] * X[ib * m + ba];
        T[f * mm + i] = s;
      }
      __syncthreads();
    }
    cube_transform<PT ? PT - 1 : 0>(cube, m, tb + et_S(p), tb + ET + et_S(p), tb + 2 * ET + et_S(p), true);
    const double *L1 = tb + et_lam(p), *L2 = tb + ET + et_lam(p), *L3 = tb + 2 * ET + et_lam(p);
    const double *a10 = tb + et_a0(p), *a11 = tb + et_a1(p);
    const double *a20 = tb + ET + et_a0(p), *a21 = tb + ET + et_a1(p);
    const double *a30 = tb + 2 * ET + et_a0(p), *a31 = tb + 2 * ET + et_a1(p);
    for (int i = tid; i < mm * m; i += nt) {
      int b3 = i / mm, r = i - b3 * mm, b2 = r / m, b1 = r - b2 * m;
      double E = a10[b1] * T[0 * mm + b3 * m + b2] + a11[b1] * T[1 * mm + b3 * m + b2] +
                 a20[b2] * T[2 * mm + b3 * m + b1] + a21[b2] * T[3 * mm + b3 * m + b1] +
                 a30[b3] * T[4 * mm + b2 * m + b1] + a31[b3] * T[5 * mm + b2 * m + b1];
      cube[i] = (cube[i] - E) / (lam + L1[b1] + L2[b2] + L3[b3]);
    }
    __syncthreads();
    cube_transform<PT ? PT - 1 : 0>(cube, m, tb + et_S(p), tb + ET + et_S(p), tb + 2 * ET + et_S(p), false);
    for (int i = tid; i < mm * m; i += nt) {
      int i3 = i / mm, r = i - i3 * mm, i2 = r / m, i1 = r - i2 * m;
      ug[(e1 * p + i1 + 1) + N1 * ((e2 * p + i2 + 1) + N2 * (long long)(e3 * p + i3 + 1))] = cube[i];
    }
  }
}

size_t recover_smem(int p, int ET, bool cube_in_smem) {
  int m = p - 1, q = p + 1;
  return sizeof(double) * (size_t)(7 * m * m + 3 * ET + 6 * q * q + (cube_in_smem ? m * m * m : 0));
}

// ------------------------------------------------------------------------------------------
// BLAS-1 (deterministic fixed-grid two-pass reductions) and coarse CG pieces
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
  }
  return s;
}

__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, long long n,
                              double* __restrict__ part, const int* __restrict__ done) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// a.b in one launch: per-block partials, and the block that arrives last (atomic ticket) sums them
// in block order -- the same deterministic result as k_dot_partial + k_sum_final, one launch fewer.
// `ticket` must be 0 on entry; the last block resets it.
__global__ void k_dot_fused(const double* __restrict__ a, const double* __restrict__ b, long long n,
                            double* __restrict__ part, unsigned* __restrict__ ticket, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ bool last;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) t += __ldcg(&part[i]);
  t = block_sum(t);
  if (threadIdx.x == 0) {
    *out = t;
    *ticket = 0u;
  }
}

__global__ void k_sum_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_zero(double* __restrict__ x, long long n) {
  pdl_wait();
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) x[i] = 0.0;
}

// ---- Alg. 5 (ipCG) vector steps; scalars live on the device: ks = [gamma, gamma0,
// delta, beta, q.p, alpha, breakdown]
__global__ void k_ipcg_beta(double* ks) {
  pdl_wait();
  pdl_trigger();        // beta = (gamma - gamma0) / delta ; delta = gamma
  ks[3] = (ks[0] - ks[1]) / ks[2];
  ks[2] = ks[0];
}
__global__ void k_ipcg_dir(double* __restrict__ p, const double* __restrict__ z, const double* __restrict__ ks,
                           long long n) {
  pdl_wait();
  pdl_trigger();        // p = beta p + z
  const double beta = ks[3];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}
__global__ void k_ipcg_alpha(double* ks) {
  pdl_wait();
  pdl_trigger();       // alpha = gamma / (q.p)
  if (!(ks[4] > 0.0)) ks[6] = 1.0;
  ks[5] = ks[0] / ks[4];
}
__global__ void k_ipcg_update(double* __restrict__ u, double* __restrict__ r, double* __restrict__ s,
                              const double* __restrict__ p, const double* __restrict__ q, const double* __restrict__ ks,
                              long long n) {
  pdl_wait();
  pdl_trigger();     // s = r ; u += alpha p ; r -= alpha q
  const double alpha = ks[5];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double ri = r[i];
    s[i] = ri;
    u[i] = fma(alpha, p[i], u[i]);
    r[i] = fma(-alpha, q[i], ri);
  }
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) y[i] += a * x[i];
}

// x = 0, r = b, z = Dinv r, p = z;  partials of r.z and b.b
__global__ void k_pcg_init(const double* __restrict__ b, const double* __restrict__ dinv, double* __restrict__ x,
                           double* __restrict__ r, double* __restrict__ z, double* __restrict__ pv, long long n,
                           double* __restrict__ part_rz, double* __restrict__ part_bb) {
  double s1 = 0.0, s2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double bi = b[i], zi = dinv[i] * bi;
    x[i] = 0.0; r[i] = bi; z[i] = zi; pv[i] = zi;
    s1 += bi * zi; s2 += bi * bi;
  }
  s1 = block_sum(s1);
  if (threadIdx.x == 0) part_rz[blockIdx.x] = s1;
  s2 = block_sum(s2);
  if (threadIdx.x == 0) part_bb[blockIdx.x] = s2;
}

__global__ void k_pcg_init_final(const double* __restrict__ part_rz, const double* __restrict__ part_bb, int nb,
                                 PcgState* st) {
  double s1 = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) { s1 += part_rz[i]; s2 += part_bb[i]; }
  s1 = block_sum(s1);
  s2 = block_sum(s2);
  if (threadIdx.x == 0) {
    st->rz = s1; st->bb = s2; st->its = 0; st->breakdown = 0;
    st->done = (s2 == 0.0) ? 1 : 0;
  }
}

__global__ void k_pcg_alpha(const double* __restrict__ part, int nb, PcgState* st) {
  if (st->done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    st->pq = s;
    if (!(s > 0.0)) { st->breakdown = 1; st->done = 1; }
    else st->alpha = st->rz / s;
  }
}

// x += alpha p; r -= alpha q; partial r.r
__global__ void k_pcg_update(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ pv,
                             const double* __restrict__ q, long long n, const PcgState* __restrict__ st,
                             double* __restrict__ part) {
  if (st->done) return;
  const double a = st->alpha;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * pv[i];
    double ri = r[i] - a * q[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_pcg_check(const double* __restrict__ part, int nb, PcgState* st, double rtol, int maxit) {
  if (st->done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    st->its += 1;
    st->rr = s;
    if (sqrt(s) <= rtol * sqrt(st->bb) || st->its >= maxit) st->done = 1;
  }
}

// z = Dinv r; partial r.z
__global__ void k_pcg_precond(const double* __restrict__ r, const double* __restrict__ dinv, double* __restrict__ z,
                              long long n, const PcgState* __restrict__ st, double* __restrict__ part) {
  if (st->done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double zi = dinv[i] * r[i];
    z[i] = zi;
    s += r[i] * zi;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_pcg_beta(const double* __restrict__ part, int nb, PcgState* st) {
  if (st->done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) { st->beta = s / st->rz; st->rz = s; }
}

__global__ void k_pcg_pdir(double* __restrict__ pv, const double* __restrict__ z, long long n,
                           const PcgState* __restrict__ st) {
  if (st->done) return;
  const double bt = st->beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    pv[i] = z[i] + bt * pv[i];
}

// ------------------------------------------------------------------------------------------
// degree dispatch of the condense / recover kernels (compile-time p for the supported degrees)
// ------------------------------------------------------------------------------------------
#define PMG_CR_DEGREES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)

cudaError_t launch_condense_elem(int nb, int nt, size_t sm, cudaStream_t st, const LevelGeom& g, const double* Fg,
                                 const double* etab, double lam, double* Yc, double* cube_g) {
  switch (g.p) {
#define CASE(P) \
  case P: k_condense_elem<P><<<nb, nt, sm, st>>>(g, Fg, etab, lam, Yc, cube_g); break;
    PMG_CR_DEGREES(CASE)
#undef CASE
    default: k_condense_elem<0><<<nb, nt, sm, st>>>(g, Fg, etab, lam, Yc, cube_g);
  }
  return cudaGetLastError();
}

cudaError_t launch_recover_elem(int nb, int nt, size_t sm, cudaStream_t st, const LevelGeom& g, const double* Fg,
                                const double* uh, const double* etab, double lam, double* ug, double* cube_g) {
  switch (g.p) {
#define CASE(P) \
  case P: k_recover_elem<P><<<nb, nt, sm, st>>>(g, Fg, uh, etab, lam, ug, cube_g); break;
    PMG_CR_DEGREES(CASE)
#undef CASE
    default: k_recover_elem<0><<<nb, nt, sm, st>>>(g, Fg, uh, etab, lam, ug, cube_g);
  }
  return cudaGetLastError();
}

cudaError_t condense_recover_set_smem_attr(int bytes) {
  cudaError_t e = cudaSuccess;
#define CASE(P)                                                                                              \
  {                                                                                                          \
    cudaError_t a = cudaFuncSetAttribute(k_condense_elem<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
    cudaError_t b = cudaFuncSetAttribute(k_recover_elem<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);  \
    if (a != cudaSuccess) e = a;                                                                             \
    if (b != cudaSuccess) e = b;                                                                             \
  }
  PMG_CR_DEGREES(CASE)
  CASE(0)
#undef CASE
  return e;
}

}  // namespace pmg

namespace pmg {

// restriction / prolongation launchers: compile-time degree pairs of the hierarchies the solver
// builds (p_l = 2 p_(l-1), and the top levels of p = 12, 24), the runtime kernels otherwise
#define PMG_TRANSFER_PAIRS(X) X(4, 2) X(8, 4) X(16, 8) X(32, 16) X(12, 8) X(24, 16) X(3, 2) X(6, 4)

cudaError_t launch_restrict(const LevelGeom& gf, const LevelGeom& gc, const double* Jint, const double* rf, double* Z,
                            double* fc, double* uzero, int nt_local, size_t smem, int gather_blocks, cudaStream_t st) {
  const int pf = gf.p, pc = gc.p;
  cudaError_t e = cudaSuccess;
  bool done = false;
#define CASE(A, B)                                                                                           \
  if (!done && pf == A && pc == B) {                                                                         \
    e = launch_pdl(k_restrict_local_t<A, B>, dim3((unsigned)gf.nrec), dim3(nt_local), smem, st, gf, pc, Jint, rf, Z); \
    done = true;                                                                                             \
  }
  PMG_TRANSFER_PAIRS(CASE)
#undef CASE
  if (!done)
    e = launch_pdl(k_restrict_local_t<0, 0>, dim3((unsigned)gf.nrec), dim3(nt_local), smem, st, gf, pc, Jint, rf, Z);
  if (e != cudaSuccess) return e;
  switch (pc) {
    case 2: return launch_pdl(k_restrict_gather_t<2>, dim3(gather_blocks), dim3(256), 0, st, gc, (const double*)Z, fc, uzero);
    case 4: return launch_pdl(k_restrict_gather_t<4>, dim3(gather_blocks), dim3(256), 0, st, gc, (const double*)Z, fc, uzero);
    case 8: return launch_pdl(k_restrict_gather_t<8>, dim3(gather_blocks), dim3(256), 0, st, gc, (const double*)Z, fc, uzero);
    case 16: return launch_pdl(k_restrict_gather_t<16>, dim3(gather_blocks), dim3(256), 0, st, gc, (const double*)Z, fc, uzero);
    default: return launch_pdl(k_restrict_gather_t<0>, dim3(gather_blocks), dim3(256), 0, st, gc, (const double*)Z, fc, uzero);
  }
}

cudaError_t launch_prolong(const LevelGeom& gf, const LevelGeom& gc, const double* Jint, const double* uc, double* uf,
                           int nt, size_t smem, cudaStream_t st) {
  const int pf = gf.p, pc = gc.p;
#define CASE(A, B)                                                                                           \
  if (pf == A && pc == B)                                                                                    \
    return launch_pdl(k_prolong_t<A, B>, dim3((unsigned)gf.nrec), dim3(nt), smem, st, gf, gc, Jint, uc, uf);
  PMG_TRANSFER_PAIRS(CASE)
#undef CASE
  return launch_pdl(k_prolong_t<0, 0>, dim3((unsigned)gf.nrec), dim3(nt), smem, st, gf, gc, Jint, uc, uf);
}

cudaError_t transfer_set_smem_attr(int bytes) {
  cudaError_t e = cudaSuccess;
#define CASE(A, B)                                                                                           \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_restrict_local_t<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); \
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_prolong_t<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  PMG_TRANSFER_PAIRS(CASE)
#undef CASE
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_restrict_local_t<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_prolong_t<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  return e;
}

}  // namespace pmg
