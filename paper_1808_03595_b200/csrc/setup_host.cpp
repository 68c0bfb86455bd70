// Host-side setup of the p-multigrid hierarchy (not timed).
//
//  - GLL nodes/weights and the reference stiffness K_hat = D^T W D.
//  - Element interior generalised eigenpairs S^T K_II S = Lambda, S^T M_II S = I per direction
//    and element width (used by the O(p^3) condensed operator, P:123 / DESIGN.md R1).
//  - Star 1-D matrices assembled from the two elements adjoining each vertex line, outer ends
//    dropped (n_S = 2p - 1), identity-padded at decoupled points, and their
//    generalised eigenpairs.
//  - Weight polynomial of degree 7 at the star points.
//  - 1-D interpolation between level degrees.
//  - diag(H_hat) of the coarse level for the Jacobi-preconditioned coarse CG (reading R11).
//
// Eigenpairs come from a cyclic Jacobi rotation method on the symmetric matrix
// M^-1/2 K M^-1/2 (M is diagonal), accurate to a few ulps for n <= 63.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pmg_internal.h"

namespace pmg {

static void legendre(int p, double x, double& Pp, double& Pm1) {
  double p0 = 1.0, p1 = x;
  if (p == 0) { Pp = 1.0; Pm1 = 0.0; return; }
  for (int n = 1; n < p; ++n) {
    double p2 = ((2.0 * n + 1.0) * x * p1 - n * p0) / (n + 1.0);
    p0 = p1; p1 = p2;
  }
  Pp = p1; Pm1 = p0;
}

void gll(int p, std::vector<double>& x, std::vector<double>& w) {
  x.assign(p + 1, 0.0);
  w.assign(p + 1, 0.0);
  for (int i = 0; i <= p; ++i) x[i] = -std::cos(M_PI * i / p);
  for (int i = 1; i < p; ++i) {
    double xi = x[i];
    for (int it = 0; it < 100; ++it) {
      double P, Pm1;
      legendre(p, xi, P, Pm1);
      double dx = (xi * P - Pm1) / ((p + 1) * P);   // Newton on (1-x^2) P'_p / p
      xi -= dx;
      if (std::fabs(dx) < 1e-16) break;
    }
    x[i] = xi;
  }
  x[0] = -1.0; x[p] = 1.0;
  std::vector<double> y(x);
  for (int i = 0; i <= p; ++i) x[i] = 0.5 * (y[i] - y[p - i]);
  for (int i = 0; i <= p; ++i) {
    double P, Pm1;
    legendre(p, x[i], P, Pm1);
    w[i] = 2.0 / (p * (p + 1.0) * P * P);
  }
}

// GLL differentiation matrix D[i][j] = l_j'(x_i) (closed form for Lobatto nodes)
static std::vector<double> gll_diff(int p, const std::vector<double>& x) {
  int q = p + 1;
  std::vector<double> D(q * q, 0.0), Lp(q);
  for (int i = 0; i < q; ++i) { double Pm1; legendre(p, x[i], Lp[i], Pm1); }
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      if (i != j) D[i * q + j] = Lp[i] / (Lp[j] * (x[i] - x[j]));
    }
  D[0] = -0.25 * p * (p + 1);
  D[q * q - 1] = 0.25 * p * (p + 1);
  return D;
}

// K_hat[i][j] = sum_q w_q D[q][i] D[q][j]
static std::vector<double> ref_stiffness(int p, const std::vector<double>& x, const std::vector<double>& w) {
  int q = p + 1;
  std::vector<double> D = gll_diff(p, x), K(q * q, 0.0);
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      double s = 0;
      for (int r = 0; r < q; ++r) s += w[r] * D[r * q + i] * D[r * q + j];
      K[i * q + j] = s;
    }
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < i; ++j) { double a = 0.5 * (K[i * q + j] + K[j * q + i]); K[i * q + j] = K[j * q + i] = a; }
  return K;
}

// Cyclic Jacobi: A (n x n, symmetric, destroyed) = V diag(lam) V^T
static void sym_eig(int n, std::vector<double> A, std::vector<double>& V, std::vector<double>& lam) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, tot = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) { double a = A[i * n + j] * A[i * n + j]; tot += a; if (i != j) off += a; }
    if (off <= 1e-32 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = A[p * n + q];
        if (apq == 0.0) continue;
        double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {   // columns p, q
          double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {   // rows p, q
          double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  lam.resize(n);
  for (int i = 0; i < n; ++i) lam[i] = A[i * n + i];
}

// generalised eigenproblem K S = M S Lambda with diagonal M > 0: S^T M S = I
static void gen_eig_diagM(int n, const std::vector<double>& K, const std::vector<double>& Mdiag,
                          std::vector<double>& S, std::vector<double>& lam) {
  std::vector<double> A(n * n), Q;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[i * n + j] = K[i * n + j] / std::sqrt(Mdiag[i] * Mdiag[j]);
  sym_eig(n, A, Q, lam);
  S.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) S[i * n + j] = Q[i * n + j] / std::sqrt(Mdiag[i]);
}

// w(t) = 1 - 35 t^4 + 84 t^5 - 70 t^6 + 20 t^7: the degree-7 polynomial with w(0) = 1, w(1) = 0
// and vanishing first three derivatives at t = 0 and t = 1 (R5).
static double weight7(double t) {
  double t2 = t * t, t4 = t2 * t2;
  return 1.0 + t4 * (-35.0 + t * (84.0 + t * (-70.0 + 20.0 * t)));
}

std::string build_level(HostLevel& L, int p, const int k[3], const double* const widths[3],
                        double lambda, int weight_degree, int neumann, int periodic) {
  (void)lambda;
  if (weight_degree != 7) return "only weight_degree = 7 is implemented (P:316)";
  if (p < 2 || p > 32) return "degree p must be in [2, 32]";
  L.p = p;
  LevelGeom& g = L.g;
  g.p = p; g.m = p - 1; g.n = 2 * p - 1;
  g.k1 = k[0]; g.k2 = k[1]; g.k3 = k[2];
  g.V1 = k[0] + 1; g.V2 = k[1] + 1; g.V3 = k[2] + 1;
  int m = g.m, n = g.n, q = p + 1, c = p - 1;
  g.RS = 3 * m * m + 3 * m + 1;
  g.YS = 6 * m * m + 12 * m + 8;
  g.ET = elem_table_stride(p);
  g.ST = star_table_stride(p);
  g.nrec = (long long)g.V1 * g.V2 * g.V3;
  g.nskel = g.nrec * g.RS;
  g.nelem = (long long)k[0] * k[1] * k[2];
  g.zoff = 0; g.K3 = k[2]; g.own_lo = 0; g.own_hi = g.V3;
  g.neu = neumann;
  g.per = periodic;

  std::vector<double> xi, wq;
  gll(p, xi, wq);
  std::vector<double> Kh = ref_stiffness(p, xi, wq);

  // coordinates
  for (int d = 0; d < 3; ++d) {
    L.coords[d].assign(k[d] * p + 1, 0.0);
    double x0 = 0.0;
    for (int e = 0; e < k[d]; ++e) {
      double h = widths[d][e];
      for (int t = 0; t <= p; ++t) L.coords[d][e * p + t] = x0 + 0.5 * (xi[t] + 1.0) * h;
      x0 += h;
    }
  }

  // element tables
  L.etab.assign((size_t)(k[0] + k[1] + k[2]) * g.ET, 0.0);
  size_t base = 0;
  for (int d = 0; d < 3; ++d)
    for (int e = 0; e < k[d]; ++e, ++base) {
      double h = widths[d][e];
      double* T = &L.etab[base * g.ET];
      std::vector<double> M(q), K(q * q);
      for (int i = 0; i < q; ++i) M[i] = 0.5 * h * wq[i];
      for (int i = 0; i < q * q; ++i) K[i] = (2.0 / h) * Kh[i];
      std::vector<double> KII(m * m), MI(m), S, lam;
      for (int i = 0; i < m; ++i) {
        MI[i] = M[i + 1];
        for (int j = 0; j < m; ++j) KII[i * m + j] = K[(i + 1) * q + (j + 1)];
      }
      gen_eig_diagM(m, KII, MI, S, lam);
      for (int b = 0; b < m; ++b) T[et_lam(p) + b] = lam[b];
      for (int b = 0; b < m; ++b)
        for (int i = 0; i < m; ++i) T[et_P(p) + b * m + i] = S[i * m + b] * MI[i];
      for (int i = 0; i < m * m; ++i) T[et_S(p) + i] = S[i];
      for (int b = 0; b < m; ++b) {
        double a0 = 0, a1 = 0;
        for (int i = 0; i < m; ++i) { a0 += S[i * m + b] * K[(i + 1) * q + 0]; a1 += S[i * m + b] * K[(i + 1) * q + p]; }
        T[et_a0(p) + b] = a0;
        T[et_a1(p) + b] = a1;
      }
      for (int i = 0; i < q; ++i) T[et_M(p) + i] = M[i];
      for (int i = 0; i < q * q; ++i) T[et_K(p) + i] = K[i];
    }

  // star tables
  L.stab.assign((size_t)(g.V1 + g.V2 + g.V3) * g.ST, 0.0);
  base = 0;
  for (int d = 0; d < 3; ++d)
    for (int v = 0; v <= k[d]; ++v, ++base) {
      double* T = &L.stab[base * g.ST];
      std::vector<double> M(n, 0.0), K(n * n, 0.0);
      const bool per = (periodic >> d) & 1;
      for (int side = 0; side < 2; ++side) {
        int e = v - 1 + side;
        if (per) e = ((e % k[d]) + k[d]) % k[d];   // periodic: the line wraps (vertex k_d is vertex 0)
        if (e < 0 || e >= k[d]) continue;
        double h = widths[d][e];
        for (int t = 0; t <= p; ++t) {
          int j = side * p - 1 + t;
          if (j < 0 || j >= n) continue;
          M[j] += 0.5 * h * wq[t];
          for (int s = 0; s <= p; ++s) {
            int i = side * p - 1 + s;
            if (i >= 0 && i < n) K[j * n + i] += (2.0 / h) * Kh[t * q + s];
          }
        }
      }
      std::vector<int> cpl;
      for (int j = 0; j < n; ++j) {
        long long gg = (long long)(v - 1) * p + 1 + j;   // unknowns of the star line (Dirichlet ends padded)
        if (per || free_1d((int)gg, k[d] * p, (neumann >> (2 * d)) & 1, (neumann >> (2 * d + 1)) & 1)) cpl.push_back(j);
      }
      int nc = (int)cpl.size();
      std::vector<double> S(n * n, 0.0), lamv(n, 1.0);
      for (int j = 0; j < n; ++j) S[j * n + j] = 1.0;
      if (nc > 0) {
        std::vector<double> Kc(nc * nc), Mc(nc), Sc, lc;
        for (int a = 0; a < nc; ++a) {
          Mc[a] = M[cpl[a]];
          for (int b = 0; b < nc; ++b) Kc[a * nc + b] = K[cpl[a] * n + cpl[b]];
        }
        gen_eig_diagM(nc, Kc, Mc, Sc, lc);
        for (int a = 0; a < nc; ++a) {
          S[cpl[a] * n + cpl[a]] = 0.0;
        }
        for (int a = 0; a < nc; ++a)
          for (int b = 0; b < nc; ++b) S[cpl[a] * n + cpl[b]] = Sc[a * nc + b];
        for (int b = 0; b < nc; ++b) lamv[cpl[b]] = lc[b];
      }
      for (int i = 0; i < n * n; ++i) T[i] = S[i];
      for (int a = 0; a < n; ++a) T[n * n + a] = lamv[a];
      for (int a = 0; a < n; ++a) T[n * n + n + a] = S[c * n + a];
      for (int j = 0; j < n; ++j) {
        double t;
        if (j < c) t = 0.5 * (1.0 - xi[j + 1]);
        else if (j == c) t = 0.0;
        else t = 0.5 * (1.0 + xi[j - c]);
        T[n * n + 2 * n + j] = weight7(t);
      }
    }
  return "";
}

// Element-centred block tables (oracle/ecsmoother.py): per direction
// and element line e the 1-D mass / stiffness of the elements e-1, e, e+1 (those in the mesh)
// assembled on the n3 = 3p - 1 block points (outer ends dropped), identity-padded at the
// points outside the domain or on a Dirichlet end, and their generalised eigenpairs; the rows of
// S at the centre element's faces; the 1-D weight of reading R17:
//   omega_e = 1/2 [(1 + [e = 0]) w_{X_e} + (1 + [e = k-1]) w_{X_{e+1}}],
// w_V(x) = w(reference distance from V) on the two elements adjoining V.
std::string build_ec_tables(HostLevel& L, const int k[3], const double* const widths[3], int neumann) {
  const int p = L.p, n = ec_n(p), q = p + 1, ES = ec_table_stride(p);
  const int clo = p - 1, chi = 2 * p - 1;
  if (p > 16) return "element-centred smoother: level degree p must be <= 16";
  std::vector<double> xi, wq;
  gll(p, xi, wq);
  std::vector<double> Kh = ref_stiffness(p, xi, wq);
  L.ectab.assign((size_t)(k[0] + k[1] + k[2]) * ES, 0.0);
  size_t base = 0;
  for (int d = 0; d < 3; ++d)
    for (int e = 0; e < k[d]; ++e, ++base) {
      double* T = &L.ectab[base * ES];
      std::vector<double> M(n, 0.0), K(n * n, 0.0);
      for (int side = 0; side < 3; ++side) {
        const int el = e - 1 + side;
        if (el < 0 || el >= k[d]) continue;
        const double h = widths[d][el];
        for (int t = 0; t <= p; ++t) {
          const int j = side * p - 1 + t;
          if (j < 0 || j >= n) continue;
          M[j] += 0.5 * h * wq[t];
          for (int s = 0; s <= p; ++s) {
            const int i = side * p - 1 + s;
            if (i >= 0 && i < n) K[j * n + i] += (2.0 / h) * Kh[t * q + s];
          }
        }
      }
      std::vector<int> cpl;
      for (int j = 0; j < n; ++j) {
        const long long gg = (long long)(e - 1) * p + 1 + j;
        if (free_1d((int)gg, k[d] * p, (neumann >> (2 * d)) & 1, (neumann >> (2 * d + 1)) & 1)) cpl.push_back(j);
      }
      const int nc = (int)cpl.size();
      std::vector<double> S(n * n, 0.0), lamv(n, 1.0);
      for (int j = 0; j < n; ++j) S[j * n + j] = 1.0;
      if (nc > 0) {
        std::vector<double> Kc(nc * nc), Mc(nc), Sc, lc;
        for (int a = 0; a < nc; ++a) {
          Mc[a] = M[cpl[a]];
          for (int b = 0; b < nc; ++b) Kc[a * nc + b] = K[cpl[a] * n + cpl[b]];
        }
        gen_eig_diagM(nc, Kc, Mc, Sc, lc);
        for (int a = 0; a < nc; ++a) S[cpl[a] * n + cpl[a]] = 0.0;
        for (int a = 0; a < nc; ++a)
          for (int b = 0; b < nc; ++b) S[cpl[a] * n + cpl[b]] = Sc[a * nc + b];
        for (int b = 0; b < nc; ++b) lamv[cpl[b]] = lc[b];
      }
      for (int i = 0; i < n * n; ++i) T[i] = S[i];
      for (int a = 0; a < n; ++a) {
        T[n * n + a] = lamv[a];
        T[n * n + n + a] = S[clo * n + a];
        T[n * n + 2 * n + a] = S[chi * n + a];
      }
      const double mlo = (e == 0) ? 2.0 : 1.0, mhi = (e == k[d] - 1) ? 2.0 : 1.0;
      for (int j = 0; j < n; ++j) {
        const int side = (j + 1) / p, t = (j + 1) - side * p;   // element e - 1 + side, local node t
        const double u = 0.5 * (xi[t] + 1.0);                    // reference position in that element
        double wlo = 0.0, whi = 0.0;                             // w_{X_e}, w_{X_{e+1}}
        if (side == 0) wlo = weight7(1.0 - u);
        else if (side == 1) { wlo = weight7(u); whi = weight7(1.0 - u); }
        else whi = weight7(u);
        T[n * n + 3 * n + j] = 0.5 * (mlo * wlo + mhi * whi);
      }
    }
  return "";
}

std::string build_interp(HostLevel& fine, int pc) {
  int pf = fine.p;
  std::vector<double> xc, wc, xf, wf;
  gll(pc, xc, wc);
  gll(pf, xf, wf);
  // barycentric weights of the coarse nodes
  std::vector<double> bw(pc + 1, 1.0);
  for (int a = 0; a <= pc; ++a)
    for (int b = 0; b <= pc; ++b)
      if (a != b) bw[a] /= (xc[a] - xc[b]);
  fine.Jint.assign((size_t)(pf - 1) * (pc + 1), 0.0);
  for (int i = 1; i < pf; ++i) {
    double x = xf[i];
    int hit = -1;
    for (int a = 0; a <= pc; ++a) if (x == xc[a]) hit = a;
    double den = 0;
    std::vector<double> num(pc + 1);
    for (int a = 0; a <= pc; ++a) {
      if (hit >= 0) { num[a] = (a == hit) ? 1.0 : 0.0; continue; }
      num[a] = bw[a] / (x - xc[a]);
      den += num[a];
    }
    for (int a = 0; a <= pc; ++a) fine.Jint[(i - 1) * (pc + 1) + a] = hit >= 0 ? num[a] : num[a] / den;
  }
  return "";
}

static long long host_skel_index(const LevelGeom& g, int g1, int g2, int g3) {
  int p = g.p, m = g.m;
  int r1 = g1 / p, t1 = g1 - r1 * p;
  int r2 = g2 / p, t2 = g2 - r2 * p;
  int r3 = g3 / p, t3 = g3 - r3 * p;
  long long rec = r1 + (long long)g.V1 * (r2 + (long long)g.V2 * r3);
  int off;
  if (t1 == 0) {
    if (t2 == 0) off = (t3 == 0) ? 3 * m * m + 3 * m : 3 * m * m + 2 * m + t3 - 1;
    else if (t3 == 0) off = 3 * m * m + m + t2 - 1;
    else off = (t3 - 1) * m + (t2 - 1);
  } else if (t2 == 0) {
    off = (t3 == 0) ? 3 * m * m + t1 - 1 : m * m + (t3 - 1) * m + (t1 - 1);
  } else {
    off = 2 * m * m + (t2 - 1) * m + (t1 - 1);
  }
  return rec * g.RS + off;
}

// p = 2 coarse operator tables (see coarse_cg.cu): tabs[0..2] = assembled 1-D lumped masses b_d,
// tabs[3..5] = assembled 1-D stiffness rows K_d[i][o + 2], o = -2..2, tabs[6] = per element
// [c_e[0..5], 1 / D_e] with c_e[2d + s] = a_{d,s} P_b P_a and D_e = lambda + L1 + L2 + L3.
std::string coarse_tables(const HostLevel& L, double lambda, std::vector<double> tabs[7]) {
  const LevelGeom& g = L.g;
  if (g.p != 2) return "coarse tables need p = 2";
  const int p = 2, q = 3;
  const int k[3] = {g.k1, g.k2, g.k3};
  size_t base = 0;
  for (int d = 0; d < 3; ++d) {
    const int n = 2 * k[d] + 1;
    tabs[d].assign(n, 0.0);
    tabs[3 + d].assign((size_t)n * 5, 0.0);
    for (int e = 0; e < k[d]; ++e) {
      const double* T = &L.etab[(base + e) * g.ET];
      for (int t = 0; t <= p; ++t) {
        tabs[d][2 * e + t] += T[et_M(p) + t];
        for (int s = 0; s <= p; ++s) tabs[3 + d][(size_t)(2 * e + t) * 5 + (s - t + 2)] += T[et_K(p) + t * q + s];
      }
    }
    base += k[d];
  }
  tabs[6].assign((size_t)g.nelem * 7, 0.0);
  for (int e3 = 0; e3 < g.k3; ++e3)
    for (int e2 = 0; e2 < g.k2; ++e2)
      for (int e1 = 0; e1 < g.k1; ++e1) {
        const double* T[3] = {&L.etab[(size_t)e1 * g.ET], &L.etab[(size_t)(g.k1 + e2) * g.ET],
                              &L.etab[(size_t)(g.k1 + g.k2 + e3) * g.ET]};
        const long long el = e1 + (long long)g.k1 * (e2 + (long long)g.k2 * e3);
        double* c = &tabs[6][(size_t)el * 7];
        for (int d = 0; d < 3; ++d) {
          const int da = (d == 0) ? 1 : 0, db = (d == 2) ? 1 : 2;
          const double PbPa = T[db][et_P(p)] * T[da][et_P(p)];
          c[2 * d] = T[d][et_a0(p)] * PbPa;
          c[2 * d + 1] = T[d][et_a1(p)] * PbPa;
        }
        c[6] = 1.0 / (lambda + T[0][et_lam(p)] + T[1][et_lam(p)] + T[2][et_lam(p)]);
      }
  return "";
}

std::string coarse_diag(const HostLevel& L, double lambda, std::vector<double>& diag) {
  const LevelGeom& g = L.g;
  int p = g.p, m = g.m, q = p + 1;
  diag.assign((size_t)g.nskel, 0.0);
  std::vector<double> dl(q * q * q);
  for (int e3 = 0; e3 < g.k3; ++e3)
    for (int e2 = 0; e2 < g.k2; ++e2)
      for (int e1 = 0; e1 < g.k1; ++e1) {
        const double* T[3] = {&L.etab[(size_t)e1 * g.ET], &L.etab[(size_t)(g.k1 + e2) * g.ET],
                              &L.etab[(size_t)(g.k1 + g.k2 + e3) * g.ET]};
        const double *M1 = T[0] + et_M(p), *M2 = T[1] + et_M(p), *M3 = T[2] + et_M(p);
        const double *K1 = T[0] + et_K(p), *K2 = T[1] + et_K(p), *K3 = T[2] + et_K(p);
        for (int t3 = 0; t3 <= p; ++t3)
          for (int t2 = 0; t2 <= p; ++t2)
            for (int t1 = 0; t1 <= p; ++t1) {
              bool b1 = (t1 == 0 || t1 == p), b2 = (t2 == 0 || t2 == p), b3 = (t3 == 0 || t3 == p);
              if (!(b1 || b2 || b3)) continue;
              double v = lambda * M1[t1] * M2[t2] * M3[t3] + K1[t1 * q + t1] * M2[t2] * M3[t3] +
                         M1[t1] * K2[t2 * q + t2] * M3[t3] + M1[t1] * M2[t2] * K3[t3 * q + t3];
              int nb = (int)b1 + (int)b2 + (int)b3;
              if (nb == 1) {  // face interior: subtract (H_BI H_II^-1 H_IB)_bb
                int d = b1 ? 0 : (b2 ? 1 : 2);
                int s = (d == 0 ? t1 : (d == 1 ? t2 : t3)) == p;
                const double* af = T[d] + (s ? et_a1(p) : et_a0(p));
                int ia = 0, ib = 0, da = 0, db = 0;   // tangential directions a (fast), b (slow)
                if (d == 0) { da = 1; db = 2; ia = t2 - 1; ib = t3 - 1; }
                if (d == 1) { da = 0; db = 2; ia = t1 - 1; ib = t3 - 1; }
                if (d == 2) { da = 0; db = 1; ia = t1 - 1; ib = t2 - 1; }
                const double *Sa = T[da] + et_S(p), *Sb = T[db] + et_S(p);
                const double *La = T[da] + et_lam(p), *Lb = T[db] + et_lam(p), *Ld = T[d] + et_lam(p);
                double Ma = T[da][et_M(p) + ia + 1], Mb = T[db][et_M(p) + ib + 1];
                double sum = 0;
                for (int bd = 0; bd < m; ++bd)
                  for (int bb = 0; bb < m; ++bb)
                    for (int ba = 0; ba < m; ++ba) {
                      double sa = Sa[ia * m + ba], sb = Sb[ib * m + bb];
                      sum += af[bd] * af[bd] * sa * sa * sb * sb / (lambda + Ld[bd] + La[ba] + Lb[bb]);
                    }
                v -= Ma * Ma * Mb * Mb * sum;
              }
              int g1 = e1 * p + t1, g2 = e2 * p + t2, g3 = e3 * p + t3;
              if (g.per & 1) g1 %= g.k1 * p;   // periodic: the last element's high faces are plane 0
              if (g.per & 2) g2 %= g.k2 * p;
              if (g.per & 4) g3 %= g.k3 * p;
              bool fr = ((g.per & 1) || free_1d(g1, g.k1 * p, g.neu & 1, (g.neu >> 1) & 1)) &&
                        ((g.per & 2) || free_1d(g2, g.k2 * p, (g.neu >> 2) & 1, (g.neu >> 3) & 1)) &&
                        ((g.per & 4) || free_1d(g3, g.k3 * p, (g.neu >> 4) & 1, (g.neu >> 5) & 1));
              if (fr) diag[host_skel_index(g, g1, g2, g3)] += v;
            }
      }
  return "";
}

}  // namespace pmg

namespace pmg {

// h-multigrid level tables (reading R16), p = 2 GRID layout.
// Per direction d and element index e: the centre row of the element's 1-D matrices,
// {M[1], K[1][0], K[1][2], K[1][1]} (physical: M = h/2 w, K = 2/h K_hat).
std::string hgrid_elem_rows(const HostLevel& L, std::vector<double> E[3]) {
  const LevelGeom& g = L.g;
  if (g.p != 2) return "h-level tables need p = 2";
  const int k[3] = {g.k1, g.k2, g.k3};
  size_t base = 0;
  for (int d = 0; d < 3; ++d) {
    E[d].assign((size_t)4 * k[d], 0.0);
    for (int e = 0; e < k[d]; ++e) {
      const double* T = &L.etab[(base + e) * g.ET];
      E[d][4 * e + 0] = T[et_M(2) + 1];
      E[d][4 * e + 1] = T[et_K(2) + 3 + 0];
      E[d][4 * e + 2] = T[et_K(2) + 3 + 2];
      E[d][4 * e + 3] = T[et_K(2) + 3 + 1];
    }
    base += k[d];
  }
  return "";
}

// 1-D h-transfer tables of one direction between a fine p = 2 line of kf elements (widths wf) and
// the coarse line of kc elements (kf = 2 kc: merged pairs, widths wc[e] = wf[2e] + wf[2e+1];
// kf = kc: kept).  Fine node G lies in coarse element ec = min(G / (2 kf / kc), kc - 1) at local
// position x (sums of fine widths from the element's left end); its weights are the quadratic
// Lagrange basis on the coarse element's GLL nodes {-1, 0, 1} at xi = 2 x / wc[ec] - 1
// (oracle/hmg.py::h_prolongation).  Restriction rows: for coarse node J the contiguous fine range
// with a nonzero weight W(G, J) (<= 7 nodes), weights in order (exact transpose).
std::string build_h_transfer_1d(int kf, const double* wf, int kc, const double* wc, std::vector<int>& pe,
                                std::vector<double>& pw, std::vector<int>& r0, std::vector<int>& rn,
                                std::vector<double>& rw) {
  if (!(kf == kc || kf == 2 * kc)) return "h-transfer: k_fine must be k_coarse or 2 k_coarse";
  const int ratio = kf / kc, nf = 2 * kf + 1, nc = 2 * kc + 1;
  pe.assign(nf, 0);
  pw.assign((size_t)3 * nf, 0.0);
  for (int G = 0; G < nf; ++G) {
    const int ec = std::min(G / (2 * ratio), kc - 1);
    const int t = G - 2 * ratio * ec;
    double x;
    if (ratio == 2) {
      const double h1 = wf[2 * ec], h2 = wf[2 * ec + 1];
      const double pos[5] = {0.0, 0.5 * h1, h1, h1 + 0.5 * h2, h1 + h2};
      x = pos[t];
    } else {
      const double h = wf[ec];
      const double pos[3] = {0.0, 0.5 * h, h};
      x = pos[t];
    }
    const double xi = 2.0 * x / wc[ec] - 1.0;
    pe[G] = ec;
    pw[3 * G + 0] = 0.5 * xi * (xi - 1.0);
    pw[3 * G + 1] = 1.0 - xi * xi;
    pw[3 * G + 2] = 0.5 * xi * (xi + 1.0);
  }
  r0.assign(nc, 0);
  rn.assign(nc, 0);
  rw.assign((size_t)7 * nc, 0.0);
  auto W = [&](int G, int J) {
    const int t = J - 2 * pe[G];
    return (t >= 0 && t <= 2) ? pw[3 * G + t] : 0.0;
  };
  for (int J = 0; J < nc; ++J) {
    int lo = -1, hi = -1;
    for (int G = 0; G < nf; ++G)
      if (W(G, J) != 0.0) { if (lo < 0) lo = G; hi = G; }
    if (lo < 0) continue;
    if (hi - lo + 1 > 7) return "h-transfer: restriction row longer than 7";
    r0[J] = lo;
    rn[J] = hi - lo + 1;
    for (int G = lo; G <= hi; ++G) rw[(size_t)7 * J + (G - lo)] = W(G, J);
  }
  return "";
}

}  // namespace pmg
