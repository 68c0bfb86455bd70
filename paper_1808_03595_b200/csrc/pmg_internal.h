// Internal declarations shared by the host setup (setup_host.cpp) and the CUDA side.
// Not part of the C ABI (see include/pmg.h).
#pragma once
#include <string>
#include <vector>

#if defined(__CUDACC__)
#define PMG_HD __host__ __device__
#else
#define PMG_HD
#endif

namespace pmg {

// Geometry of one level on the device (record layout).
struct LevelGeom {
  int p, m, n;          // degree, m = p - 1 (element interior), n = 2p - 1 (star extent n_S)
  int k1, k2, k3;       // elements per direction
  int V1, V2, V3;       // vertices per direction (k_d + 1)
  int RS;               // record stride: 3m^2 + 3m + 1
  int YS;               // element output stride: 6m^2 + 12m + 8
  int ET;               // element table stride (per direction, per 1-D element)
  int ST;               // star table stride (per direction, per vertex line)
  long long nrec;       // V1 V2 V3
  long long nskel;      // nrec * RS
  long long nelem;      // k1 k2 k3
  // z-slab decomposition: this geometry holds vertex planes
  // zoff .. zoff + k3 of a global mesh with K3 element layers.  Dirichlet tests (is_free) use the
  // global plane zoff + v3; array bounds (inside) stay local.  Element-gathered skeleton values
  // (residual, condensed RHS, restriction) are computed on the owned record planes
  // [own_lo, own_hi); the other (ghost) planes are filled by the halo exchange.
  // One GPU: zoff = 0, K3 = k3, own_lo = 0, own_hi = V3.
  int zoff, K3, own_lo, own_hi;
  // homogeneous Neumann faces (NEXT-3): bit 2d / 2d+1 = low / high face of direction d;
  // every other face is homogeneous Dirichlet
  int neu;
  // periodic directions (NEXT-3): bit d.  Global indices along d are taken modulo k_d p:
  // record plane k_d duplicates plane 0 and holds no unknown; neighbour accesses wrap (wrap_pt).
  int per;
};

// the record coordinate w (possibly -1 or k) of a periodic direction, wrapped into [0, k)
PMG_HD inline int wrap_rec(int w, int k, bool periodic) {
  return periodic ? (w < 0 ? w + k : (w >= k ? w - k : w)) : w;
}

// is global 1-D index G (0 <= G <= n_el p) an unknown along a direction with the given end flags?
PMG_HD inline bool free_1d(int G, int n_el_p, bool neu_lo, bool neu_hi) {
  return G >= 0 && G <= n_el_p && (G > 0 || neu_lo) && (G < n_el_p || neu_hi);
}

// Element table, per direction d and 1-D element e_d (width h), m = p - 1, q = p + 1:
//   [0, m)            Lambda_d  (interior generalised eigenvalues, S^T K_II S = Lambda)
//   [m, m+m^2)        P_d[b][i] = S[i][b] M[i]   (S^T M_II, forward face transform)
//   [.., +m^2)        S_d[i][b]                  (interior eigenvectors, S^T M_II S = I)
//   [.., +m)          a0[b] = sum_i S[i][b] K[i][0]   (expansion vector of the low face)
//   [.., +m)          a1[b] = sum_i S[i][b] K[i][p]   (expansion vector of the high face)
//   [.., +q)          M diag (h/2 w)
//   [.., +q^2)        K[i][j] (2/h K_hat)
PMG_HD inline int elem_table_stride(int p) { int m = p - 1, q = p + 1; return m + 2 * m * m + 2 * m + q + q * q; }
PMG_HD inline int et_lam(int) { return 0; }
PMG_HD inline int et_P(int p) { return p - 1; }
PMG_HD inline int et_S(int p) { int m = p - 1; return m + m * m; }
PMG_HD inline int et_a0(int p) { int m = p - 1; return m + 2 * m * m; }
PMG_HD inline int et_a1(int p) { int m = p - 1; return 2 * m + 2 * m * m; }
PMG_HD inline int et_M(int p) { int m = p - 1; return 3 * m + 2 * m * m; }
PMG_HD inline int et_K(int p) { int m = p - 1; return 3 * m + 2 * m * m + p + 1; }

// Star table, per direction d and vertex line v_d, n = 2p - 1, c = p - 1:
//   [0, n^2)   S[j][a]  (padded generalised eigenvectors of the assembled 1-D star, S^T M S = I)
//   [.., +n)   Lambda[a] (padded with 1 at decoupled points)
//   [.., +n)   s[a] = S[c][a]  (the vertex row, "S_I0^T" of Alg. 1)
//   [.., +n)   w[j]  weight polynomial at star point j (1 at the vertex)
PMG_HD inline int star_table_stride(int p) { int n = 2 * p - 1; return n * n + 3 * n; }

// Element-centred block table, per direction d and element line
// e_d, n3 = 3p - 1 (three elements, outer block ends dropped), planes at c_lo = p - 1, c_hi = 2p - 1:
//   [0, n3^2)   S[j][a]   (padded generalised eigenvectors of the assembled 1-D block, S^T M S = I)
//   [.., +n3)   Lambda[a] (padded with 1 at decoupled points)
//   [.., +n3)   S[c_lo][a]
//   [.., +n3)   S[c_hi][a]
//   [.., +n3)   omega[j]  (1-D weight, reading R17)
PMG_HD inline int ec_n(int p) { return 3 * p - 1; }
PMG_HD inline int ec_table_stride(int p) { int n = 3 * p - 1; return n * n + 4 * n; }

struct HostLevel {
  int p;
  LevelGeom g;
  std::vector<double> etab;      // (k1 + k2 + k3) * ET
  std::vector<double> stab;      // (V1 + V2 + V3) * ST
  std::vector<double> ectab;     // (k1 + k2 + k3) * ec_table_stride(p) (element-centred smoother only)
  std::vector<double> Jint;      // (p - 1) x (p_c + 1): rows 1..p-1 of J (coarse -> this level)
  std::vector<double> coords[3];
};

// Host setup; returns an empty string on success, else an error message.
std::string build_level(HostLevel& L, int p, const int k[3], const double* const widths[3],
                        double lambda, int weight_degree, int neumann = 0, int periodic = 0);
std::string build_interp(HostLevel& fine, int p_coarse);
// element-centred block tables (fills L.ectab; L built by build_level with the same k, widths)
std::string build_ec_tables(HostLevel& L, const int k[3], const double* const widths[3], int neumann);
// diag(H_hat) for the given level in skeleton record layout (free entries only, others 0).
std::string coarse_diag(const HostLevel& L, double lambda, std::vector<double>& diag);
// p = 2 coarse CG operator tables (coarse_cg.cu)
std::string coarse_tables(const HostLevel& L, double lambda, std::vector<double> tabs[7]);
// 1-D GLL nodes and weights (p >= 1)
void gll(int p, std::vector<double>& x, std::vector<double>& w);
// h-multigrid (reading R16) p = 2 grid-layout tables: per direction the element centre rows
// {M[1], K[1][0], K[1][2], K[1][1]}, and the 1-D transfer tables between a fine and a coarse line
std::string hgrid_elem_rows(const HostLevel& L, std::vector<double> E[3]);
std::string build_h_transfer_1d(int kf, const double* wf, int kc, const double* wc, std::vector<int>& pe,
                                std::vector<double>& pw, std::vector<int>& r0, std::vector<int>& rn,
                                std::vector<double>& rw);

}  // namespace pmg
