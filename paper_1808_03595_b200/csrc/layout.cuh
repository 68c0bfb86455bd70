// Device helpers for the skeleton record layout.
#pragma once
#include "pmg_internal.h"

namespace pmg {

__host__ __device__ inline int off_face(int m, int d) { return d * m * m; }
__host__ __device__ inline int off_edge(int m, int d) { return 3 * m * m + d * m; }
__host__ __device__ inline int off_vert(int m) { return 3 * m * m + 3 * m; }

// Skeleton point (global GLL indices, 0 <= g_d <= k_d p, at least one g_d a multiple of p)
// -> index into a skeleton vector.
__device__ __forceinline__ long long skel_index(const LevelGeom& g, int g1, int g2, int g3) {
  const int p = g.p, m = g.m;
  const int r1 = g1 / p, t1 = g1 - r1 * p;
  const int r2 = g2 / p, t2 = g2 - r2 * p;
  const int r3 = g3 / p, t3 = g3 - r3 * p;
  const long long rec = r1 + (long long)g.V1 * (r2 + (long long)g.V2 * r3);
  int off;
  if (t1 == 0) {
    if (t2 == 0) off = (t3 == 0) ? off_vert(m) : off_edge(m, 2) + t3 - 1;
    else if (t3 == 0) off = off_edge(m, 1) + t2 - 1;
    else off = off_face(m, 0) + (t3 - 1) * m + (t2 - 1);
  } else if (t2 == 0) {
    off = (t3 == 0) ? off_edge(m, 0) + t1 - 1 : off_face(m, 1) + (t3 - 1) * m + (t1 - 1);
  } else {
    off = off_face(m, 2) + (t2 - 1) * m + (t1 - 1);
  }
  return rec * g.RS + off;
}

// skel_index with the degree known at compile time (divisions by p become multiply-shifts)
template <int P>
__device__ __forceinline__ long long skel_index_t(const LevelGeom& g, int g1, int g2, int g3) {
  constexpr int m = P - 1;
  const int r1 = g1 / P, t1 = g1 - r1 * P;
  const int r2 = g2 / P, t2 = g2 - r2 * P;
  const int r3 = g3 / P, t3 = g3 - r3 * P;
  const long long rec = r1 + (long long)g.V1 * (r2 + (long long)g.V2 * r3);
  int off;
  if (t1 == 0) {
    if (t2 == 0) off = (t3 == 0) ? off_vert(m) : off_edge(m, 2) + t3 - 1;
    else if (t3 == 0) off = off_edge(m, 1) + t2 - 1;
    else off = off_face(m, 0) + (t3 - 1) * m + (t2 - 1);
  } else if (t2 == 0) {
    off = (t3 == 0) ? off_edge(m, 0) + t1 - 1 : off_face(m, 1) + (t3 - 1) * m + (t1 - 1);
  } else {
    off = off_face(m, 2) + (t2 - 1) * m + (t1 - 1);
  }
  return rec * (3 * m * m + 3 * m + 1) + off;
}

// periodic directions: a global point index beyond either end (star / element neighbour accesses)
// wrapped into [0, k_d p) (one GPU: z-periodic meshes are not split into slabs)
__device__ __forceinline__ void wrap_pt(const LevelGeom& g, int& g1, int& g2, int& g3) {
  if (g.per & 1) { const int n = g.k1 * g.p; g1 = g1 < 0 ? g1 + n : (g1 >= n ? g1 - n : g1); }
  if (g.per & 2) { const int n = g.k2 * g.p; g2 = g2 < 0 ? g2 + n : (g2 >= n ? g2 - n : g2); }
  if (g.per & 4) { const int n = g.k3 * g.p; g3 = g3 < 0 ? g3 + n : (g3 >= n ? g3 - n : g3); }
}

__device__ __forceinline__ bool inside(const LevelGeom& g, int g1, int g2, int g3) {
  return g1 >= 0 && g2 >= 0 && g3 >= 0 && g1 <= g.k1 * g.p && g2 <= g.k2 * g.p && g3 <= g.k3 * g.p;
}
// free unknown: strictly inside the GLOBAL box (g3 is local; the slab starts at vertex plane zoff)
// Neumann faces (g.neu) keep their points as unknowns; in a periodic direction the last plane
// (index k_d p) duplicates plane 0 and is not an unknown (callers wrap neighbour points first)
__device__ __forceinline__ bool is_free(const LevelGeom& g, int g1, int g2, int g3) {
  const int G3 = g3 + g.zoff * g.p;
  if (g.per) {
    if ((g.per & 1) ? !(g1 >= 0 && g1 < g.k1 * g.p) : !free_1d(g1, g.k1 * g.p, g.neu & 1, (g.neu >> 1) & 1)) return false;
    if ((g.per & 2) ? !(g2 >= 0 && g2 < g.k2 * g.p) : !free_1d(g2, g.k2 * g.p, (g.neu >> 2) & 1, (g.neu >> 3) & 1)) return false;
    return (g.per & 4) ? (G3 >= 0 && G3 < g.K3 * g.p) : free_1d(G3, g.K3 * g.p, (g.neu >> 4) & 1, (g.neu >> 5) & 1);
  }
  return free_1d(g1, g.k1 * g.p, g.neu & 1, (g.neu >> 1) & 1) && free_1d(g2, g.k2 * g.p, (g.neu >> 2) & 1, (g.neu >> 3) & 1) &&
         free_1d(G3, g.K3 * g.p, (g.neu >> 4) & 1, (g.neu >> 5) & 1);
}
// a box-corner star has no unknown iff the three faces meeting at the corner are Dirichlet (a
// periodic direction has no corner); in a periodic direction the star at vertex k_d is the one at 0
__device__ __forceinline__ bool star_empty(const LevelGeom& g, int v1, int v2, int v3) {
  if (g.per) {
    if (((g.per & 1) && v1 >= g.k1) || ((g.per & 2) && v2 >= g.k2) || ((g.per & 4) && v3 >= g.k3)) return true;
    if (g.per & 7) {
      const bool c1 = !(g.per & 1) && (v1 == 0 || v1 == g.k1), c2 = !(g.per & 2) && (v2 == 0 || v2 == g.k2),
                 c3 = !(g.per & 4) && (v3 + g.zoff == 0 || v3 + g.zoff == g.K3);
      if (!(c1 && c2 && c3)) return false;
    }
  }
  const int V3 = v3 + g.zoff;
  const bool c1 = v1 == 0 || v1 == g.k1, c2 = v2 == 0 || v2 == g.k2, c3 = V3 == 0 || V3 == g.K3;
  if (!(c1 && c2 && c3)) return false;
  const int f1 = v1 == 0 ? 0 : 1, f2 = v2 == 0 ? 2 : 3, f3 = V3 == 0 ? 4 : 5;
  return !((g.neu >> f1) & 1) && !((g.neu >> f2) & 1) && !((g.neu >> f3) & 1);
}
// record plane v3 (local) carries element-gathered values on this rank
__device__ __forceinline__ bool owned_plane(const LevelGeom& g, int v3) { return v3 >= g.own_lo && v3 < g.own_hi; }

// Skeleton-vector entry -> record vertex, entity type (0-2 faces, 3-5 edges, 6 vertex),
// local indices (a = slow, b = fast for faces; a for edges) and global point.
struct Entry {
  int v1, v2, v3, type, a, b, g1, g2, g3;
};

__device__ __forceinline__ Entry decode_entry(const LevelGeom& g, long long idx) {
  Entry E;
  const int m = g.m, p = g.p;
  long long rec = idx / g.RS;
  int o = (int)(idx - rec * g.RS);
  E.v1 = (int)(rec % g.V1);
  long long r2 = rec / g.V1;
  E.v2 = (int)(r2 % g.V2);
  E.v3 = (int)(r2 / g.V2);
  E.g1 = E.v1 * p; E.g2 = E.v2 * p; E.g3 = E.v3 * p;
  E.a = 0; E.b = 0;
  if (o < 3 * m * m) {
    E.type = o / (m * m);
    int r = o - E.type * m * m;
    E.a = r / m; E.b = r - E.a * m;
    if (E.type == 0) { E.g3 += E.a + 1; E.g2 += E.b + 1; }
    else if (E.type == 1) { E.g3 += E.a + 1; E.g1 += E.b + 1; }
    else { E.g2 += E.a + 1; E.g1 += E.b + 1; }
  } else if (o < 3 * m * m + 3 * m) {
    int r = o - 3 * m * m;
    int d = r / m;
    E.type = 3 + d;
    E.a = r - d * m;
    if (d == 0) E.g1 += E.a + 1; else if (d == 1) E.g2 += E.a + 1; else E.g3 += E.a + 1;
  } else {
    E.type = 6;
  }
  return E;
}

// decode_entry with the degree known at compile time and a vector shorter than 2^31 entries:
// 32-bit arithmetic, divisions by RS, m^2 and m become multiply-shifts
template <int P>
__device__ __forceinline__ Entry decode_entry_t(const LevelGeom& g, unsigned idx) {
  constexpr int m = P - 1, mm = m * m;
  constexpr unsigned RS = 3 * mm + 3 * m + 1;
  Entry E;
  const unsigned rec = idx / RS;
  const int o = (int)(idx - rec * RS);
  const unsigned r2 = rec / (unsigned)g.V1;
  E.v1 = (int)(rec - r2 * (unsigned)g.V1);
  E.v3 = (int)(r2 / (unsigned)g.V2);
  E.v2 = (int)(r2 - (unsigned)E.v3 * (unsigned)g.V2);
  E.g1 = E.v1 * P; E.g2 = E.v2 * P; E.g3 = E.v3 * P;
  E.a = 0; E.b = 0;
  if (o < 3 * mm) {
    E.type = o / (mm > 0 ? mm : 1);
    const int r = o - E.type * mm;
    E.a = r / m; E.b = r - E.a * m;
    if (E.type == 0) { E.g3 += E.a + 1; E.g2 += E.b + 1; }
    else if (E.type == 1) { E.g3 += E.a + 1; E.g1 += E.b + 1; }
    else { E.g2 += E.a + 1; E.g1 += E.b + 1; }
  } else if (o < 3 * mm + 3 * m) {
    const int r = o - 3 * mm;
    const int d = r / m;
    E.type = 3 + d;
    E.a = r - d * m;
    if (d == 0) E.g1 += E.a + 1; else if (d == 1) E.g2 += E.a + 1; else E.g3 += E.a + 1;
  } else {
    E.type = 6;
  }
  return E;
}

}  // namespace pmg
