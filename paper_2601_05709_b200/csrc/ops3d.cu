// 3D kernels of liblsgpu: Kuhn-tetrahedron P1 operators on a structured box.
//
// Mesh (oracle/grid.py, mesh.cu): node (i,j,k) = (k(ny+1)+j)(nx+1)+i; cell
// (i,j,k) holds six tetrahedra m = 0..5 following the axis permutation
// (a,b,c) = KUHN[m] along the path P0 = v000, P1 = P0+e_a, P2 = P1+e_b,
// P3 = v111.  With D_a = u(P1)-u(P0), D_b = u(P2)-u(P1), D_c = u(P3)-u(P2):
//   grad N = (-e_a/h_a, e_a/h_a - e_b/h_b, e_b/h_b - e_c/h_c, e_c/h_c),
//   du/dx_a = D_a/h_a, du/dx_b = D_b/h_b, du/dx_c = D_c/h_c,
// so every operator reduces to three "fluxes" F_a, F_b, F_c per tet and the
// contributions -F_a, F_a-F_b, F_b-F_c, F_c to the four path vertices.
//
// Execution (march3s, march3s.cuh): a CTA of 8 warps covers 30 node columns
// (x, lanes 1..30 of each warp) and 8 node rows (y, one warp each; warp 0 is a
// halo row whose outputs belong to the tile below) and marches along z.  Planes
// are staged in shared memory by cp.async two planes ahead; x-neighbours come
// through shuffles; each lane evaluates the six tets of cell (i, j, k) and the
// contributions to the eight corners are combined with shuffles (x) and one
// shared-memory exchange (y).  Every node is summed by one thread in a fixed
// order: deterministic, no atomics.
//
// Material word (uint32, lsg_material): bits 3m..3m+2 = n_in of tet m
// (number of its 4 quadrature points with phi < 0), bit 18 = cell valid,
// bits 19..21 = Dirichlet on ux, uy, uz of the node.
// H1 word (lsg_h1_words): bits 4m..4m+3 = frozen flags of tet m's quadrature
// points, bit 24 = cell valid, bit 25 = Dirichlet (all components).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "ops.h"

namespace lsg {
namespace d3 {

constexpr int kStrip = 30;
#ifndef LSG_M3_WARPS
#define LSG_M3_WARPS 8
#endif
constexpr int kWarps = LSG_M3_WARPS;  // node rows per CTA (one of them halo)
constexpr int kThreads = kWarps * 32;
constexpr int kMaxPartials = 4096;
constexpr int kEwThreads = 256;
constexpr double kA = 0.5854101966249685, kB = 0.1381966011250105;  // 4-point rule

struct Geo {
  int nx, ny, nz;
  double h[3], ih[3];
};

// Kuhn permutation m -> axes (a, b, c); corner bit per axis: x=1, y=2, z=4.
__host__ __device__ constexpr int perm(int m, int s) {
  return (m == 0) ? (s == 0 ? 0 : s == 1 ? 1 : 2)
       : (m == 1) ? (s == 0 ? 0 : s == 1 ? 2 : 1)
       : (m == 2) ? (s == 0 ? 1 : s == 1 ? 0 : 2)
       : (m == 3) ? (s == 0 ? 1 : s == 1 ? 2 : 0)
       : (m == 4) ? (s == 0 ? 2 : s == 1 ? 0 : 1)
                  : (s == 0 ? 2 : s == 1 ? 1 : 0);
}
__host__ __device__ constexpr int corner(int m, int v) {  // path vertex v of tet m
  return v == 0 ? 0 : v == 1 ? (1 << perm(m, 0)) : v == 2 ? ((1 << perm(m, 0)) | (1 << perm(m, 1))) : 7;
}

// ---------------------------------------------------------------------------
// Physics
// ---------------------------------------------------------------------------
struct Elast {
  static constexpr int NIN = 3, NOUT = 3;
  static constexpr bool kTable = false;
  double lam, mu, w0, w1;  // w(n) = w0 + w1 n = |T| (inside n + outside (4-n)) / 4
  double ih[3];
  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 18) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return (w >> 19) & 7u; }

  // Folded constants: F_d[q] = w sigma[q][d] / h_d with sigma from raw edge
  // differences D_d = u(next path vertex) - u(this one) along axis d:
  //   q != d: F_d[q] = w (A[d] D_d[q] + B[d][q] D_q[d]),  A[d] = mu/h_d^2, B = mu/(h_d h_q)
  //   q == d: F_d[d] = w (2 A[d] D_d[d] + L[d] tr),        L[d] = lam/h_d, tr = sum_d D_d[d]/h_d
  double A[3], B[3][3], L[3];

  template <int M>
  __device__ __forceinline__ void tet(const double (*u)[NIN], uint32_t word, double (*c)[NOUT]) const {
    constexpr int a = perm(M, 0), b = perm(M, 1), cc = perm(M, 2);
    constexpr int P0 = 0, P1 = corner(M, 1), P2 = corner(M, 2), P3 = 7;
    const double w = valid(word) ? fma((double)((word >> (3 * M)) & 7u), w1, w0) : 0.0;
    double D[3][3];  // D[axis][comp]
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      D[a][q] = u[P1][q] - u[P0][q];
      D[b][q] = u[P2][q] - u[P1][q];
      D[cc][q] = u[P3][q] - u[P2][q];
    }
    const double tr = fma(D[0][0], ih[0], fma(D[1][1], ih[1], D[2][2] * ih[2]));
    double T[3][3];  // unweighted fluxes T[axis][comp] = sigma[comp][axis] / h_axis
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        T[d][q] = (q == d) ? fma(2.0 * A[d], D[d][d], L[d] * tr)
                           : fma(A[d], D[d][q], B[d][q] * D[q][d]);
    // weighted contributions -wT_a, w(T_a - T_b), w(T_b - T_c), wT_c via FMA
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      c[P0][q] = fma(-w, T[a][q], c[P0][q]);
      c[P1][q] = fma(w, T[a][q] - T[b][q], c[P1][q]);
      c[P2][q] = fma(w, T[b][q] - T[cc][q], c[P2][q]);
      c[P3][q] = fma(w, T[cc][q], c[P3][q]);
    }
  }

  __device__ __forceinline__ void cell(const double (*u)[NIN], uint32_t word, int, int, int,
                                       double (*c)[NOUT]) const {
#pragma unroll
    for (int v = 0; v < 8; ++v)
#pragma unroll
      for (int q = 0; q < NOUT; ++q) c[v][q] = 0.0;
    tet<0>(u, word, c); tet<1>(u, word, c); tet<2>(u, word, c);
    tet<3>(u, word, c); tet<4>(u, word, c); tet<5>(u, word, c);
  }
};

// Cubic cells (h_x = h_y = h_z, cfg3 and cfg5): with s = w mu/h^2, l = w lam/h^2
// (w = |T| times the tet's ersatz weight) and the raw edge differences D^x,
// D^y, D^z along the tet's x-, y- and z-directed path edges, the stress is
//   sigma_aa = l (D^x_x + D^y_y + D^z_z) + 2 s D^a_a,  sigma_ab = s (D^a_b + D^b_a),
// and the tet adds the column sigma e_a to the flux of its a-directed edge (the
// edge's start corner receives -flux, its end corner +flux).  Every path edge
// is one of the cube's 12 edges, so the cell evaluates each edge difference
// once (36 subtractions instead of 54), sums the fluxes of the tets sharing an
// edge, and forms each corner's contribution as the divergence of its three
// edges: ~170 fp64 instructions per cell and field against ~240 tet by tet.
struct ElastC {
  static constexpr int NIN = 3, NOUT = 3;
  static constexpr bool kTable = true;  // per-CTA shared table of the tet weights
  double w0, w1;  // |T| (inside n + outside (4-n)) / 4 = w0 + w1 n
  double cs, cl;  // mu / h^2, lam / h^2

  // tab[n] = w(n) mu/h^2, tab[8 + n] = w(n) lam/h^2, tab[16 + n] = 2 w(n) mu/h^2
  // for n = 0..4; index 7 (what invalid cells look up) gives 0
  __device__ __forceinline__ void fill_table(double *tab, int t) const {
    if (t < 24) {
      const int n = t & 7;
      const double w = n <= 4 ? fma((double)n, w1, w0) : 0.0;
      tab[t] = t < 8 ? w * cs : t < 16 ? w * cl : 2.0 * (w * cs);
    }
  }
  __device__ __forceinline__ static bool valid(uint32_t w) { return Elast::valid(w); }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return Elast::mask(w); }

  // the six stress components (xx, yy, zz, xy, xz, yz) of tet M
  template <int M>
  __device__ __forceinline__ static void sigma(const double *Dx, const double *Dy, const double *Dz,
                                               uint32_t nbits, const double *tab, double (&sg)[6]) {
    const uint32_t n = (nbits >> (3 * M)) & 7u;
    const double s = tab[n], l = tab[8 + n], s2 = tab[16 + n];
    const double lt = l * (Dx[0] + Dy[1] + Dz[2]);
    sg[0] = fma(s2, Dx[0], lt);
    sg[1] = fma(s2, Dy[1], lt);
    sg[2] = fma(s2, Dz[2], lt);
    sg[3] = s * (Dx[1] + Dy[0]);
    sg[4] = s * (Dx[2] + Dz[0]);
    sg[5] = s * (Dy[2] + Dz[1]);
  }

  __device__ __forceinline__ void cell(const double (*u)[NIN], uint32_t word, int, int, int,
                                       double (*c)[NOUT], const double *tab) const {
    const uint32_t nb = valid(word) ? word : 0x3ffffu;  // invalid: every tet reads index 7
    // cell edges (corner bits x = 1, y = 2, z = 4): X_yz from corner 2y+4z,
    // Y_xz from x+4z, Z_xy from x+2y
    double X00[3], X10[3], X01[3], X11[3], Y00[3], Y10[3], Y01[3], Y11[3], Z00[3], Z10[3], Z01[3], Z11[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      X00[q] = u[1][q] - u[0][q]; X10[q] = u[3][q] - u[2][q]; X01[q] = u[5][q] - u[4][q]; X11[q] = u[7][q] - u[6][q];
      Y00[q] = u[2][q] - u[0][q]; Y10[q] = u[3][q] - u[1][q]; Y01[q] = u[6][q] - u[4][q]; Y11[q] = u[7][q] - u[5][q];
      Z00[q] = u[4][q] - u[0][q]; Z10[q] = u[5][q] - u[1][q]; Z01[q] = u[6][q] - u[2][q]; Z11[q] = u[7][q] - u[3][q];
    }
    // tets (perm): 0 (x,y,z) X00 Y10 Z11, 1 (x,z,y) X00 Y11 Z10, 2 (y,x,z) X10 Y00 Z11,
    //              3 (y,z,x) X11 Y00 Z01, 4 (z,x,y) X01 Y11 Z00, 5 (z,y,x) X11 Y01 Z00
    double s0[6], s1[6], s2[6], s3[6], s4[6], s5[6];
    sigma<0>(X00, Y10, Z11, nb, tab, s0);
    sigma<1>(X00, Y11, Z10, nb, tab, s1);
    sigma<2>(X10, Y00, Z11, nb, tab, s2);
    sigma<3>(X11, Y00, Z01, nb, tab, s3);
    sigma<4>(X01, Y11, Z00, nb, tab, s4);
    sigma<5>(X11, Y01, Z00, nb, tab, s5);
    // flux columns: x-edge (xx, xy, xz), y-edge (xy, yy, yz), z-edge (xz, yz, zz)
    constexpr int CX[3] = {0, 3, 4}, CY[3] = {3, 1, 5}, CZ[3] = {4, 5, 2};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double fx00 = s0[CX[q]] + s1[CX[q]], fx10 = s2[CX[q]], fx01 = s4[CX[q]], fx11 = s3[CX[q]] + s5[CX[q]];
      const double fy00 = s2[CY[q]] + s3[CY[q]], fy10 = s0[CY[q]], fy01 = s5[CY[q]], fy11 = s1[CY[q]] + s4[CY[q]];
      const double fz00 = s4[CZ[q]] + s5[CZ[q]], fz10 = s1[CZ[q]], fz01 = s3[CZ[q]], fz11 = s0[CZ[q]] + s2[CZ[q]];
      c[0][q] = -(fx00 + fy00) - fz00;
      c[1][q] = (fx00 - fy10) - fz10;
      c[2][q] = (fy00 - fx10) - fz01;
      c[3][q] = (fx10 + fy10) - fz11;
      c[4][q] = (fz00 - fx01) - fy01;
      c[5][q] = (fx01 + fz10) - fy11;
      c[6][q] = (fy01 + fz01) - fx11;
      c[7][q] = (fx11 + fy11) + fz11;
    }
  }
};

struct H1;
struct H1 {
  static constexpr int NIN = 3, NOUT = 3;
  static constexpr bool kTable = false;
  int nx, ny, nz;
  double m;          // mw |T| / 20
  double sw_t;       // sw |T|
  double fz;         // fp |T| / 4
  double pen[3];     // npen * facet area / 12 for faces normal to x, y, z
  double ih[3];
  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 24) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return ((w >> 25) & 1u) ? 7u : 0u; }

  template <int M>
  __device__ __forceinline__ void tet(const double (*u)[NIN], uint32_t word, double (*c)[NOUT]) const {
    constexpr int a = perm(M, 0), b = perm(M, 1), cc = perm(M, 2);
    constexpr int P[4] = {0, corner(M, 1), corner(M, 2), 7};
    const uint32_t fq = (word >> (4 * M)) & 15u;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double Fa = sw_t * (u[P[1]][q] - u[P[0]][q]) * ih[a] * ih[a];
      const double Fb = sw_t * (u[P[2]][q] - u[P[1]][q]) * ih[b] * ih[b];
      const double Fc = sw_t * (u[P[3]][q] - u[P[2]][q]) * ih[cc] * ih[cc];
      const double s = u[P[0]][q] + u[P[1]][q] + u[P[2]][q] + u[P[3]][q];
      c[P[0]][q] += -Fa + m * (u[P[0]][q] + s);
      c[P[1]][q] += Fa - Fb + m * (u[P[1]][q] + s);
      c[P[2]][q] += Fb - Fc + m * (u[P[2]][q] + s);
      c[P[3]][q] += Fc + m * (u[P[3]][q] + s);
      if (fq) {
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          if (fq & (1u << qq)) {
            double uq = 0.0;
#pragma unroll
            for (int v = 0; v < 4; ++v) uq += (v == qq ? kA : kB) * u[P[v]][q];
#pragma unroll
            for (int v = 0; v < 4; ++v) c[P[v]][q] += fz * (v == qq ? kA : kB) * uq;
          }
        }
      }
    }
  }

  // boundary normal penalty: faces of the box split along the in-face
  // diagonal through corners (0,0) and (1,1); facet mass |f|/12 (1 + delta).
  __device__ __forceinline__ void face(int axis, int side, const double (*u)[NIN], double (*c)[NOUT]) const {
    const int u1 = axis == 0 ? 1 : 0, v1 = axis == 2 ? 1 : 2;  // in-face axes (ascending)
    const int base = side ? (1 << axis) : 0;
    const int c00 = base, c10 = base | (1 << u1), c11 = base | (1 << u1) | (1 << v1),
              c01 = base | (1 << v1);
    const int tris[2][3] = {{c00, c10, c11}, {c00, c11, c01}};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double s = u[tris[t][0]][axis] + u[tris[t][1]][axis] + u[tris[t][2]][axis];
#pragma unroll
      for (int v = 0; v < 3; ++v) c[tris[t][v]][axis] += pen[axis] * (u[tris[t][v]][axis] + s);
    }
  }

  __device__ __forceinline__ void cell(const double (*u)[NIN], uint32_t word, int i, int j, int k,
                                       double (*c)[NOUT]) const {
#pragma unroll
    for (int v = 0; v < 8; ++v)
#pragma unroll
      for (int q = 0; q < NOUT; ++q) c[v][q] = 0.0;
    if (!valid(word)) return;
    tet<0>(u, word, c); tet<1>(u, word, c); tet<2>(u, word, c);
    tet<3>(u, word, c); tet<4>(u, word, c); tet<5>(u, word, c);
    if (pen[0] != 0.0 || pen[1] != 0.0 || pen[2] != 0.0) {
      if (i == 0) face(0, 0, u, c);
      if (i == nx - 1) face(0, 1, u, c);
      if (j == 0) face(1, 0, u, c);
      if (j == ny - 1) face(1, 1, u, c);
      if (k == 0) face(2, 0, u, c);
      if (k == nz - 1) face(2, 1, u, c);
    }
  }
};

// Fused compliance + shape-derivative RHS for KB states at once.
// The velocity form without the optional boundary-normal / frozen terms
// (the BASELINE configs: mass + alpha vector Laplacian): per component the
// six tets' stiffness fluxes k_a D_a with compile-time first-touch corners,
// and the cell mass assembled per corner as m (n_v u_v + sum_{t ∋ v} s_t)
// from the six tet sums s_t (n_v = 6 tets at corners 0 and 7, 2 elsewhere),
// instead of the per-tet mass products of H1.
struct H1P {
  static constexpr int NIN = 3, NOUT = 3;
  static constexpr bool kTable = false;
  double m;      // mw |T| / 20
  double ka[3];  // sw |T| / h_a^2
  __device__ __forceinline__ static bool valid(uint32_t w) { return H1::valid(w); }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return H1::mask(w); }

  static __host__ __device__ constexpr bool in_tet(int M, int v) {
    return v == 0 || v == 7 || corner(M, 1) == v || corner(M, 2) == v;
  }
  static __host__ __device__ constexpr bool touched(int M, int v) {  // by a tet < M
    return M > 0 && (in_tet(M - 1, v) || touched(M - 1, v));
  }
  template <int M, int V>
  __device__ __forceinline__ static void put(double (*c)[NOUT], int q, double x) {
    if constexpr (touched(M, V)) c[V][q] += x; else c[V][q] = x;
  }
  template <int M>
  __device__ __forceinline__ void tet(const double (*u)[NIN], int q, double (*c)[NOUT],
                                      double &st) const {
    constexpr int a = perm(M, 0), b = perm(M, 1), cc = perm(M, 2);
    constexpr int P1 = corner(M, 1), P2 = corner(M, 2);
    const double Fa = ka[a] * (u[P1][q] - u[0][q]);
    const double Fb = ka[b] * (u[P2][q] - u[P1][q]);
    const double Fc = ka[cc] * (u[7][q] - u[P2][q]);
    put<M, 0>(c, q, -Fa);
    put<M, P1>(c, q, Fa - Fb);
    put<M, P2>(c, q, Fb - Fc);
    put<M, 7>(c, q, Fc);
    st = (u[0][q] + u[7][q]) + (u[P1][q] + u[P2][q]);
  }
  template <int V>
  __device__ __forceinline__ void mass(const double (*u)[NIN], int q, const double (&S)[6],
                                       double (*c)[NOUT]) const {
    double sv = 0.0;
    int nv = 0;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const bool in = (V == 0 || V == 7 || corner(t, 1) == V || corner(t, 2) == V);
      if (in) { sv += S[t]; ++nv; }
    }
    c[V][q] = fma(m, fma((double)nv, u[V][q], sv), c[V][q]);
  }

  __device__ __forceinline__ void cell(const double (*u)[NIN], uint32_t word, int, int, int,
                                       double (*c)[NOUT]) const {
    if (!valid(word)) {
#pragma unroll
      for (int v = 0; v < 8; ++v)
#pragma unroll
        for (int q = 0; q < NOUT; ++q) c[v][q] = 0.0;
      return;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double S[6];
      tet<0>(u, q, c, S[0]); tet<1>(u, q, c, S[1]); tet<2>(u, q, c, S[2]);
      tet<3>(u, q, c, S[3]); tet<4>(u, q, c, S[4]); tet<5>(u, q, c, S[5]);
      mass<0>(u, q, S, c); mass<1>(u, q, S, c); mass<2>(u, q, S, c); mass<3>(u, q, S, c);
      mass<4>(u, q, S, c); mass<5>(u, q, S, c); mass<6>(u, q, S, c); mass<7>(u, q, S, c);
    }
  }
};

template <int KB>
struct Shape {
  static constexpr int NIN = 3 * KB, NOUT = 6;
  static constexpr bool kTable = false;
  double lam, mu, vol_t, inv_volume, w0, w1;
  double ih[3];
  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 18) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t) { return 0u; }

  template <int M>
  __device__ __forceinline__ void tet(const double (*u)[NIN], uint32_t word, double (*c)[NOUT],
                                      bool count, double *part) const {
    constexpr int a = perm(M, 0), b = perm(M, 1), cc = perm(M, 2);
    constexpr int P0 = 0, P1 = corner(M, 1), P2 = corner(M, 2), P3 = 7;
    const bool ok = valid(word);
    const uint32_t n = ok ? ((word >> (3 * M)) & 7u) : 0u;
    const double w = ok ? fma((double)n, w1, w0) : 0.0;
    double bulk[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double dens = 0.0;
#pragma unroll
    for (int f = 0; f < KB; ++f) {
      double G[3][3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        G[q][a] = (u[P1][3 * f + q] - u[P0][3 * f + q]) * ih[a];
        G[q][b] = (u[P2][3 * f + q] - u[P1][3 * f + q]) * ih[b];
        G[q][cc] = (u[P3][3 * f + q] - u[P2][3 * f + q]) * ih[cc];
      }
      const double tr = G[0][0] + G[1][1] + G[2][2];
      double S[3][3], E[3][3];
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          E[p][q] = 0.5 * (G[p][q] + G[q][p]);
          S[p][q] = 2.0 * mu * E[p][q] + (p == q ? lam * tr : 0.0);
        }
      double d = 0.0;
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) d += S[p][q] * E[p][q];
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double gts = 0.0;
#pragma unroll
          for (int r = 0; r < 3; ++r) gts += G[r][p] * S[r][q];
          bulk[p][q] += 2.0 * gts - (p == q ? d : 0.0);
        }
      dens += d;
    }
    // vec_cost: X_d = w bulk[:, d] / h_d ; vec_vol: v e_d / h_d
    const double v = vol_t * (double)n * 0.25 * inv_volume;
    double Xa[3], Xb[3], Xc[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      Xa[q] = w * bulk[q][a] * ih[a];
      Xb[q] = w * bulk[q][b] * ih[b];
      Xc[q] = w * bulk[q][cc] * ih[cc];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      c[P0][q] -= Xa[q];
      c[P1][q] += Xa[q] - Xb[q];
      c[P2][q] += Xb[q] - Xc[q];
      c[P3][q] += Xc[q];
    }
    c[P0][3 + a] -= v * ih[a];
    c[P1][3 + a] += v * ih[a];
    c[P1][3 + b] -= v * ih[b];
    c[P2][3 + b] += v * ih[b];
    c[P2][3 + cc] -= v * ih[cc];
    c[P3][3 + cc] += v * ih[cc];
    if (count) {
      part[0] += w * dens;
      part[1] += vol_t * (double)n * 0.25;
    }
  }

  __device__ __forceinline__ void cell(const double (*u)[NIN], uint32_t word, bool count,
                                       double (*c)[NOUT], double *part) const {
#pragma unroll
    for (int v = 0; v < 8; ++v)
#pragma unroll
      for (int q = 0; q < NOUT; ++q) c[v][q] = 0.0;
    tet<0>(u, word, c, count, part); tet<1>(u, word, c, count, part);
    tet<2>(u, word, c, count, part); tet<3>(u, word, c, count, part);
    tet<4>(u, word, c, count, part); tet<5>(u, word, c, count, part);
  }
};

// PCGQ: the stencil half of the split pass A (q = A p, p.q; p formed by pcg_prep)
enum Act { APPLY = 0, RESID = 1, STATS = 3, SHAPE = 4, PCGQ = 5 };

struct MArgs {
  const uint32_t *words;
  const double *x, *x2, *b;
  double *y, *y2;
  const double *dinv;
  lsg_pcg_scalars *scal;
  double *partials;
  uint32_t *counters;
  double *out;
  int seg, nzseg, nstrips, accumulate;
};

template <int ACT>
struct Traits {
  static constexpr int NP = (ACT == RESID) ? 3 : (ACT == PCGQ) ? 1
                         : (ACT == STATS) ? 3 : (ACT == SHAPE) ? 2 : 0;
  static constexpr unsigned MAXMASK = (ACT == STATS) ? 4u : 0u;
};

template <int ACT>
__device__ __forceinline__ void finalize(const MArgs &a, int rhs, const double *tot) {
  if constexpr (ACT == RESID) {
    lsg_pcg_scalars &s = a.scal[rhs];
    s.bb = tot[0];
    s.rr = tot[1];
    s.rho = tot[2];
    s.atol = fmax(s.atol, s.reserved[0] * sqrt(tot[0]));
    s.beta = 0.0;
    s.first = 1.0;
    if (tot[0] == 0.0) {
      s.zero_rhs = 1.0;
      s.done = 1.0;
    } else if (sqrt(tot[1]) < s.atol) {
      s.done = 1.0;
    }
  } else if constexpr (ACT == PCGQ) {
    lsg_pcg_scalars &s = a.scal[rhs];
    s.pq = tot[0];
    s.reserved[2] = s.alpha;  // alpha_{i-1}, still pending on odd iterations
    s.alpha = s.rho / tot[0];
  } else if constexpr (ACT == STATS) {
    a.out[0] = tot[0];
    a.out[1] = tot[1];
    a.out[2] = tot[2];
  } else if constexpr (ACT == SHAPE) {
    if (a.accumulate) {
      a.out[0] += tot[0];
    } else {
      a.out[0] = tot[0];
      a.out[1] = tot[1];
    }
  }
}

}  // namespace d3
}  // namespace lsg

#include "march3s.cuh"

namespace lsg {
namespace d3 {

// ---------------------------------------------------------------------------
// Elementwise kernels
// ---------------------------------------------------------------------------
// M^-1 is read by both elementwise passes of every right-hand side (8 times per
// cfg5 iteration).  When the batch is far larger than L2 the passes ask L2 to
// evict it last (cfg5 PCG iteration 439.6 -> 434.0 us); batches near the L2
// size measured ~0.7% slower with the hint, so they keep the normal priority.
template <bool KEEP>
__device__ __forceinline__ uint64_t l2_policy() {
  uint64_t pol = 0;
  if constexpr (KEEP) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
template <bool KEEP>
__device__ __forceinline__ double ld_policy(const double *p, uint64_t pol) {
  if constexpr (KEEP) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
    return v;
  } else {
    return __ldg(p);
  }
}

template <bool KEEP>
__global__ void __launch_bounds__(kEwThreads)
    pcg_update(int64_t n, const double *dinv, double *r, const double *q, lsg_pcg_scalars *scal,
               double *partials, uint32_t *counters) {
  __shared__ double scratch[2 * (kEwThreads / 32)];
  pdl_wait();
  const int rhs = blockIdx.y;
  lsg_pcg_scalars &s = scal[rhs];
  if (s.done != 0.0) return;
  const double alpha = s.alpha;
  const size_t off = (size_t)rhs * (size_t)n;
  double part[2] = {0.0, 0.0};
  const uint64_t pol = l2_policy<KEEP>();
  const int64_t stride = (int64_t)gridDim.x * kEwThreads;
  for (int64_t base = (int64_t)blockIdx.x * kEwThreads + threadIdx.x; base < n; base += 4 * stride) {
    double Q[4], R[4], D[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + u * stride;
      if (t < n) {
        Q[u] = __ldcs(q + off + t);  // q is dead after this pass: evict-first keeps p and r in L2
        D[u] = ld_policy<KEEP>(dinv + t, pol);
        R[u] = r[off + t];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + u * stride;
      if (t < n) {
        const double ro = fma(-alpha, Q[u], R[u]);
        r[off + t] = ro;
        part[0] += ro * (ro * D[u]);
        part[1] += ro * ro;
      }
    }
  }
  double tot[2];
  const int nblk = gridDim.x;
  if (block_partial_and_total<2, 0u>(part, partials + (size_t)rhs * nblk * 2, counters + rhs,
                                     blockIdx.x, nblk, scratch, tot)) {
    if (threadIdx.x == 0) {
      s.iters += 1.0;
      s.rz_new = tot[0];
      s.rr = tot[1];
      s.reserved[1] = (((int)s.iters - 1) & 1) ? 2.0 : 1.0;  // pending x updates (as 2D)
      if (sqrt(tot[1]) < s.atol) s.done = 1.0;
      else if (s.iters >= s.maxiter || !isfinite(tot[1]) || !isfinite(tot[0])) s.done = 2.0;
      else {
        s.beta = tot[0] / s.rho;
        s.rho = tot[0];
        s.first = 0.0;
      }
    }
  }
}

// Split pass A, first half (elementwise, HBM-bound): p = D^-1 r + beta p_old
// and, on even iterations i >= 2, the two pending x updates of iterations i-2
// and i-1 (three direction buffers rotate, so p_{i-2} is still there: x is
// read and written every second iteration only).  The stencil half
// (march3s<PH, PCGQ>) then reads only p.  Used in 3D, where a fused pass A is
// fp64-issue-bound.
template <bool KEEP>
__global__ void __launch_bounds__(kEwThreads, 4)  // 4 CTAs/SM: the grid is one full wave
    pcg_prep(int64_t n, const double *dinv, const double *r, const double *p_old,
             const double *p_old2, double *p_new, double *x, const lsg_pcg_scalars *scal) {
  pdl_wait();
  const int rhs = blockIdx.y;
  const lsg_pcg_scalars &s = scal[rhs];
  if (s.done != 0.0) return;
  const double beta = s.beta, al = s.alpha, al2 = s.reserved[2];
  const int it = (int)s.iters;
  const bool upd = it >= 2 && (it & 1) == 0;
  const size_t off = (size_t)rhs * (size_t)n;
  const uint64_t pol = l2_policy<KEEP>();
  const int64_t stride = (int64_t)gridDim.x * kEwThreads;
  for (int64_t base = (int64_t)blockIdx.x * kEwThreads + threadIdx.x; base < n; base += 4 * stride) {
    double R[4], P[4], D[4], X[4], P2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + u * stride;
      if (t < n) {
        R[u] = __ldg(r + off + t);
        P[u] = __ldg(p_old + off + t);
        D[u] = ld_policy<KEEP>(dinv + t, pol);
        if (upd) {
          X[u] = x[off + t];
          P2[u] = __ldg(p_old2 + off + t);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + u * stride;
      if (t < n) {
        p_new[off + t] = fma(beta, P[u], R[u] * D[u]);
        if (upd) x[off + t] = fma(al, P[u], fma(al2, P2[u], X[u]));
      }
    }
  }
}

__device__ __forceinline__ void cell_phi(const double *phi, int64_t n0, int64_t nxp, int64_t plane,
                                         double *pc) {
#pragma unroll
  for (int cidx = 0; cidx < 8; ++cidx)
    pc[cidx] = phi[n0 + (cidx & 1) + ((cidx >> 1) & 1) * nxp + ((cidx >> 2) & 1) * plane];
}

// chi at quadrature point q of tet m, bit-exact with oracle/fem.py phi_at_quad_sign
__device__ __forceinline__ int tet_chi(const double *pc, int m, int q) {
  int P[4] = {0, 0, 0, 7};
  const int a = perm(m, 0), b = perm(m, 1);
  P[1] = 1 << a;
  P[2] = (1 << a) | (1 << b);
  double v = __dmul_rn(kA, pc[P[q]]);
  for (int o = 0; o < 4; ++o)
    if (o != q) v = __dadd_rn(v, __dmul_rn(kB, pc[P[o]]));
  return v < 0.0;
}

__global__ void material_kernel(Geo g, const double *phi, const uint8_t *bcmask, uint32_t *words) {
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  const int64_t nn = plane * (g.nz + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int k = (int)(node / plane);
  const int j = (int)((node - k * plane) / nxp);
  const int i = (int)(node - k * plane - (int64_t)j * nxp);
  uint32_t w = ((uint32_t)(bcmask ? bcmask[node] : 0) & 7u) << 19;
  if (i < g.nx && j < g.ny && k < g.nz) {
    double pc[8];
    cell_phi(phi, node, nxp, plane, pc);
    for (int m = 0; m < 6; ++m) {
      int n = 0;
      for (int q = 0; q < 4; ++q) n += tet_chi(pc, m, q);
      w |= (uint32_t)n << (3 * m);
    }
    w |= 1u << 18;
  }
  words[node] = w;
}

__global__ void indicator_kernel(Geo g, const double *phi, double *chi) {
  const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 6 * ncell) return;
  const int64_t c = t / 6;
  const int m = (int)(t - c * 6);
  const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny), k = (int)(c / ((int64_t)g.nx * g.ny));
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  double pc[8];
  cell_phi(phi, ((int64_t)k * (g.ny + 1) + j) * nxp + i, nxp, plane, pc);
  for (int q = 0; q < 4; ++q) chi[t * 4 + q] = tet_chi(pc, m, q);
}

__global__ void h1_words_kernel(Geo g, const uint8_t *frozen_q, int zero_dirichlet, uint32_t *words) {
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  const int64_t nn = plane * (g.nz + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int k = (int)(node / plane);
  const int j = (int)((node - k * plane) / nxp);
  const int i = (int)(node - k * plane - (int64_t)j * nxp);
  uint32_t w = 0;
  if (i < g.nx && j < g.ny && k < g.nz) {
    w |= 1u << 24;
    if (frozen_q) {
      const int64_t c = ((int64_t)k * g.ny + j) * g.nx + i;
      for (int m = 0; m < 6; ++m)
        for (int q = 0; q < 4; ++q) w |= (frozen_q[(c * 6 + m) * 4 + q] ? 1u : 0u) << (4 * m + q);
    }
  }
  if (zero_dirichlet && (i == 0 || j == 0 || k == 0 || i == g.nx || j == g.ny || k == g.nz))
    w |= 1u << 25;
  words[node] = w;
}

// Jacobi diagonal: loop over the 8 cells x 6 tets around the node.
template <class PH>
__global__ void diag_kernel(PH ph, Geo g, const uint32_t *words, int kind, double p0, double p1,
                            double *d) {
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  const int64_t nn = plane * (g.nz + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int k = (int)(node / plane);
  const int j = (int)((node - k * plane) / nxp);
  const int i = (int)(node - k * plane - (int64_t)j * nxp);
  double acc[3] = {0.0, 0.0, 0.0};
  for (int cidx = 0; cidx < 8; ++cidx) {
    const int di = cidx & 1, dj = (cidx >> 1) & 1, dk = (cidx >> 2) & 1;
    const int ci = i - di, cj = j - dj, ck = k - dk;  // cell whose corner cidx is this node
    if (ci < 0 || cj < 0 || ck < 0 || ci >= g.nx || cj >= g.ny || ck >= g.nz) continue;
    const uint32_t w = words[((int64_t)ck * (g.ny + 1) + cj) * nxp + ci];
    if (!PH::valid(w)) continue;
    // unit cell: the node is corner cidx; apply the cell operator to e_node
    double U[8][3];
    for (int q = 0; q < 3; ++q) {
      for (int v = 0; v < 8; ++v)
        for (int t = 0; t < 3; ++t) U[v][t] = 0.0;
      U[cidx][q] = 1.0;
      double C[8][3];
      ph.cell(U, w, ci, cj, ck, C);
      acc[q] += C[cidx][q];
    }
  }
  const uint32_t m = PH::mask(words[node]);
  for (int q = 0; q < 3; ++q) d[node * 3 + q] = ((m >> q) & 1u) ? 1.0 : acc[q];
}

__global__ void reciprocal_kernel(int64_t n, double *d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) d[t] = fabs(d[t]) > 0.0 ? 1.0 / d[t] : 1.0;
}

__global__ void zero_if_flag(int64_t n, lsg_pcg_scalars *scal, double *x) {
  const int rhs = blockIdx.y;
  if (scal[rhs].zero_rhs == 0.0) return;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    x[(size_t)rhs * n + t] = 0.0;
}

__global__ void init_scalars(int k, lsg_pcg_scalars *scal, double rtol, double atol, double maxiter) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= k) return;
  lsg_pcg_scalars s = {};
  s.atol = atol;
  s.maxiter = maxiter;
  s.first = 1.0;
  s.reserved[0] = rtol;
  scal[r] = s;
}

__global__ void velocity_rhs_kernel(int64_t nn, const uint32_t *words, const double *vc,
                                    const double *vv, double lam, double *b) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const bool pin = (words[node] >> 25) & 1u;
  for (int c = 0; c < 3; ++c) {
    const double v = vc[node * 3 + c] + lam * vv[node * 3 + c];
    b[node * 3 + c] = pin ? 0.0 : -v;
  }
}

// generic S0/S1 quadrature tensors -> vector, gathered over the 8 x 6 incident tets
__global__ void tensor_rhs_kernel(Geo g, const double *s0, const double *s1, double *vec) {
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  const int64_t nn = plane * (g.nz + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int k = (int)(node / plane);
  const int j = (int)((node - k * plane) / nxp);
  const int i = (int)(node - k * plane - (int64_t)j * nxp);
  const double wq = g.h[0] * g.h[1] * g.h[2] / 6.0 / 4.0;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int cidx = 0; cidx < 8; ++cidx) {
    const int ci = i - (cidx & 1), cj = j - ((cidx >> 1) & 1), ck = k - ((cidx >> 2) & 1);
    if (ci < 0 || cj < 0 || ck < 0 || ci >= g.nx || cj >= g.ny || ck >= g.nz) continue;
    const int64_t c = ((int64_t)ck * g.ny + cj) * g.nx + ci;
    for (int m = 0; m < 6; ++m) {
      int v = -1;
      for (int vv = 0; vv < 4; ++vv)
        if (corner(m, vv) == cidx) v = vv;
      if (v < 0) continue;
      double gr[3] = {0.0, 0.0, 0.0};
      const int a = perm(m, 0), b = perm(m, 1), cc = perm(m, 2);
      if (v == 0) gr[a] = -g.ih[a];
      if (v == 1) { gr[a] = g.ih[a]; gr[b] = -g.ih[b]; }
      if (v == 2) { gr[b] = g.ih[b]; gr[cc] = -g.ih[cc]; }
      if (v == 3) gr[cc] = g.ih[cc];
      const int64_t t = c * 6 + m;
      for (int q = 0; q < 4; ++q) {
        const double Nv = (q == v) ? kA : kB;
        for (int comp = 0; comp < 3; ++comp) {
          double val = 0.0;
          if (s1) {
            const double *S = s1 + ((t * 4 + q) * 3 + comp) * 3;
            val += S[0] * gr[0] + S[1] * gr[1] + S[2] * gr[2];
          }
          if (s0) val += s0[(t * 4 + q) * 3 + comp] * Nv;
          acc[comp] += wq * val;
        }
      }
    }
  }
  for (int comp = 0; comp < 3; ++comp) vec[node * 3 + comp] = acc[comp];
}

// S1 of the cost per tet and quadrature point (parity path)
__global__ void s1_kernel(Geo g, double lam, double mu, double ersatz, double inside, int k,
                          const double *u, const double *phi, double *s1) {
  const int64_t ncell = (int64_t)g.nx * g.ny * g.nz;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 6 * ncell) return;
  const int64_t c = t / 6;
  const int m = (int)(t - c * 6);
  const int i = (int)(c % g.nx), j = (int)((c / g.nx) % g.ny), kk = (int)(c / ((int64_t)g.nx * g.ny));
  const int64_t nxp = g.nx + 1, plane = nxp * (g.ny + 1);
  const int64_t n0 = ((int64_t)kk * (g.ny + 1) + j) * nxp + i;
  const int64_t nn = plane * (g.nz + 1);
  const int a = perm(m, 0), b = perm(m, 1), cc = perm(m, 2);
  const int P[4] = {0, 1 << a, (1 << a) | (1 << b), 7};
  auto nid = [&](int cidx) { return n0 + (cidx & 1) + ((cidx >> 1) & 1) * nxp + ((cidx >> 2) & 1) * plane; };
  double bulk[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int f = 0; f < k; ++f) {
    const double *U = u + (size_t)f * nn * 3;
    double G[3][3];
    for (int q = 0; q < 3; ++q) {
      G[q][a] = (U[nid(P[1]) * 3 + q] - U[nid(P[0]) * 3 + q]) / g.h[a];
      G[q][b] = (U[nid(P[2]) * 3 + q] - U[nid(P[1]) * 3 + q]) / g.h[b];
      G[q][cc] = (U[nid(P[3]) * 3 + q] - U[nid(P[2]) * 3 + q]) / g.h[cc];
    }
    const double tr = G[0][0] + G[1][1] + G[2][2];
    double S[3][3], E[3][3], d = 0.0;
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) {
        E[p][q] = 0.5 * (G[p][q] + G[q][p]);
        S[p][q] = 2.0 * mu * E[p][q] + (p == q ? lam * tr : 0.0);
      }
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) d += S[p][q] * E[p][q];
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) {
        double gts = 0.0;
        for (int r = 0; r < 3; ++r) gts += G[r][p] * S[r][q];
        bulk[p][q] += 2.0 * gts - (p == q ? d : 0.0);
      }
  }
  double pc[8];
  cell_phi(phi, n0, nxp, plane, pc);
  for (int q = 0; q < 4; ++q) {
    const double A = tet_chi(pc, m, q) ? inside : ersatz;
    for (int p = 0; p < 3; ++p)
      for (int r = 0; r < 3; ++r) s1[((t * 4 + q) * 3 + p) * 3 + r] = A * bulk[p][r];
  }
}

__global__ void cfl_kernel(int64_t nn, Geo g, const double *v, double *partials, uint32_t *counter,
                           double *out) {
  __shared__ double scratch[kEwThreads / 32];
  double m[1] = {0.0};
  for (int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; node < nn;
       node += (int64_t)gridDim.x * blockDim.x)
    m[0] = fmax(m[0], fabs(v[node * 3]) * g.ih[0] + fabs(v[node * 3 + 1]) * g.ih[1] +
                          fabs(v[node * 3 + 2]) * g.ih[2]);
  double tot[1];
  if (block_partial_and_total<1, 1u>(m, partials, counter, blockIdx.x, gridDim.x, scratch, tot))
    if (threadIdx.x == 0) out[0] = tot[0];
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static Geo geo_of(const lsg_grid &gr) {
  Geo g;
  g.nx = gr.n[0];
  g.ny = gr.n[1];
  g.nz = gr.n[2];
  for (int a = 0; a < 3; ++a) {
    g.h[a] = (gr.hi[a] - gr.lo[a]) / gr.n[a];
    g.ih[a] = 1.0 / g.h[a];
  }
  return g;
}

static int64_t nodes_of(const Geo &g) { return (int64_t)(g.nx + 1) * (g.ny + 1) * (g.nz + 1); }

static Elast make_elast(const Geo &g, const lsg_op &op) {
  Elast e;
  const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
  const double inside = op.p[3] > 0.0 ? op.p[3] : 1.0;
  e.lam = op.p[0];
  e.mu = op.p[1];
  e.w0 = vol * op.p[2];
  e.w1 = vol * (inside - op.p[2]) / 4.0;
  for (int a = 0; a < 3; ++a) {
    e.ih[a] = g.ih[a];
    e.A[a] = e.mu * g.ih[a] * g.ih[a];
    e.L[a] = e.lam * g.ih[a];
    for (int q = 0; q < 3; ++q) e.B[a][q] = e.mu * g.ih[a] * g.ih[q];
  }
  return e;
}

static bool is_cubic(const Geo &g) {
  return fabs(g.h[1] - g.h[0]) <= 1e-14 * g.h[0] && fabs(g.h[2] - g.h[0]) <= 1e-14 * g.h[0];
}

static ElastC make_elast_cubic(const Geo &g, const lsg_op &op) {
  const Elast e = make_elast(g, op);
  ElastC c;
  c.w0 = e.w0;
  c.w1 = e.w1;
  c.cs = e.A[0];
  c.cl = e.lam * g.ih[0] * g.ih[0];
  return c;
}

static H1 make_h1(const Geo &g, const lsg_op &op) {
  H1 h;
  const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
  h.nx = g.nx;
  h.ny = g.ny;
  h.nz = g.nz;
  h.m = op.p[0] * vol / 20.0;
  h.sw_t = op.p[1] * vol;
  h.fz = op.p[3] * vol / 4.0;
  const double fa[3] = {0.5 * g.h[1] * g.h[2], 0.5 * g.h[0] * g.h[2], 0.5 * g.h[0] * g.h[1]};
  for (int a = 0; a < 3; ++a) {
    h.pen[a] = op.p[2] * fa[a] / 12.0;
    h.ih[a] = g.ih[a];
  }
  return h;
}

static H1P make_h1_plain(const Geo &g, const lsg_op &op) {
  H1P h;
  const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
  h.m = op.p[0] * vol / 20.0;
  for (int a = 0; a < 3; ++a) h.ka[a] = op.p[1] * vol * g.ih[a] * g.ih[a];
  return h;
}

int64_t partials_per_rhs(const lsg_grid &) { return kMaxPartials; }

static void launch_geometry(const Geo &g, int k, int ctas_per_sm, int &seg, int &nzseg, dim3 &grid) {
  const int64_t nstrips = ceil_div(g.nx + 1, kStrip);
  const int64_t tiles = ceil_div(g.ny + 1, kWarps - 1);
  // z-segments (one halo plane each): the grid runs in rounds of `slots` resident
  // CTAs, each CTA marching seg + 1 planes, so the launch costs about
  // rounds x (seg + 1) plane steps; take the segment count that minimises it
  // (cfg5: 3 segments of 33 planes = 2 rounds for a half batch of the PCG and 4
  // for the k = 4 apply; measured against 4 segments: PCG iteration 451 -> 442 us,
  // apply 232 -> 230 us).  Segments of 5..48 planes: shorter ones pay more in halo
  // planes and pipeline fill than the model says (cfg3: 5 planes fill one round,
  // PCG iteration 28.2 -> 26.6 us), longer ones leave a tail.
  const int64_t per_seg = nstrips * tiles * k;
  const int64_t slots = (int64_t)num_sms() * (ctas_per_sm > 0 ? ctas_per_sm : 2);
  const int64_t nzp = g.nz + 1;
  constexpr int64_t smax = 48, smin = 5;
  int64_t best_s = nzp, best_cost = -1;
  for (int64_t ns = 1; ns <= nzp; ++ns) {
    const int64_t s = ceil_div(nzp, ns);
    if ((s > smax && ns < nzp) || (s < smin && ns > 1)) continue;
    const int64_t nseg = ceil_div(nzp, s);
    const int64_t cost = ceil_div(nseg * per_seg, slots) * (s + 1);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_s = s;
    }
  }
  int64_t s = best_s;
  while (nstrips * tiles * ceil_div(nzp, s) > kMaxPartials) s *= 2;
  seg = (int)s;
  nzseg = (int)ceil_div(nzp, s);
  grid = dim3((unsigned)nstrips, (unsigned)tiles, (unsigned)(nzseg * k));
}

template <class PH, int ACT>
static int launch(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  static int ctas = -1;
  constexpr size_t smem = Stage<PH, ACT>::bytes;
  if (ctas < 0) {
    cudaFuncSetAttribute(march3s<PH, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, march3s<PH, ACT>, kThreads, smem) !=
        cudaSuccess)
      ctas = 2;
  }
  dim3 grid;
  launch_geometry(g, k, ctas, a.seg, a.nzseg, grid);
  a.nstrips = (int)ceil_div(g.nx + 1, kStrip);
  if (ACT == PCGQ) {
    if (launch_pdl(march3s<PH, ACT>, grid, dim3(kThreads), smem, st, ph, g, a) != cudaSuccess)
      return check_launch("march3d launch");
  } else {
    march3s<PH, ACT><<<grid, kThreads, smem, st>>>(ph, g, a);
  }
  return check_launch("march3d");
}

template <int ACT>
static int dispatch(const lsg_op &op, MArgs a, int k, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  a.words = static_cast<const uint32_t *>(op.words);
  if (op.kind == LSG_OP_ELASTICITY) {
    if (is_cubic(g)) return launch<ElastC, ACT>(make_elast_cubic(g, op), g, a, k, st);
    return launch<Elast, ACT>(make_elast(g, op), g, a, k, st);
  }
  if (op.kind == LSG_OP_H1) {
    if (op.p[2] == 0.0 && op.p[3] == 0.0) return launch<H1P, ACT>(make_h1_plain(g, op), g, a, k, st);
    return launch<H1, ACT>(make_h1(g, op), g, a, k, st);
  }
  set_error("unknown operator kind %d", op.kind);
  return LSG_ERR_ARG;
}

int apply(const lsg_op &op, int k, const double *x, double *y, cudaStream_t st) {
  MArgs a = {};
  a.x = x;
  a.y = y;
  return dispatch<APPLY>(op, a, k, st);
}

int diag(const lsg_op &op, double *d, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = nodes_of(g);
  const unsigned nb = (unsigned)ceil_div(nn, 128);
  const uint32_t *w = static_cast<const uint32_t *>(op.words);
  if (op.kind == LSG_OP_ELASTICITY)
    diag_kernel<Elast><<<nb, 128, 0, st>>>(make_elast(g, op), g, w, op.kind, op.p[0], op.p[1], d);
  else
    diag_kernel<H1><<<nb, 128, 0, st>>>(make_h1(g, op), g, w, op.kind, op.p[0], op.p[1], d);
  return check_launch("diag3d");
}

int inv_diag(const lsg_op &op, double *d, cudaStream_t st) {
  int rc = diag(op, d, st);
  if (rc) return rc;
  const int64_t n = 3 * nodes_of(geo_of(op.grid));
  reciprocal_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d);
  return check_launch("inv_diag3d");
}

int pcg_start(const lsg_op &op, lsg_pcg_ws &ws, double rtol, double atol, double maxiter,
              cudaStream_t st) {
  const int64_t n = 3 * nodes_of(geo_of(op.grid));
  ws.parity = 0;
  init_scalars<<<(unsigned)ceil_div(ws.k, 64), 64, 0, st>>>(ws.k, ws.scal, rtol, atol, maxiter);
  int rc = check_launch("init_scalars3d");
  if (rc) return rc;
  MArgs a = {};
  a.x = ws.x;
  a.b = ws.b;
  a.y = ws.r;
  a.dinv = ws.dinv;
  a.scal = ws.scal;
  a.partials = ws.partials;
  a.counters = ws.counters;
  rc = dispatch<RESID>(op, a, ws.k, st);
  if (rc) return rc;
  // the first pass A reads p_old = ring[2] = ws.p_ring with beta = 0: it must be finite
  if (cudaMemsetAsync(ws.p_ring, 0, sizeof(double) * (size_t)n * ws.k, st) != cudaSuccess)
    return check_launch("pcg_start3d memset");
  zero_if_flag<<<dim3(64, ws.k), 256, 0, st>>>(n, ws.scal, ws.x);
  return check_launch("zero_if_flag3d");
}

// One 3D PCG iteration (elementwise p-pass, stencil q = A p, update) of a
// batch of right-hand sides; `after_prep` is recorded once the p-pass is queued.
static int iterate_once(const lsg_op &op, const lsg_pcg_ws &ws, int parity, int64_t n, dim3 eg,
                        cudaStream_t st, cudaEvent_t after_prep, int keep_dinv) {
  MArgs a = {};
  a.y = ws.q;
  a.dinv = ws.dinv;
  a.scal = ws.scal;
  a.partials = ws.partials;
  a.counters = ws.counters;
  double *const ring[3] = {ws.p, ws.p_alt, ws.p_ring};
  const int ph = parity;  // iteration index mod 3 = slot of the new direction
  double *p_new = ring[ph], *p_old = ring[ph == 0 ? 2 : ph - 1];
  double *p_old2 = ring[ph == 2 ? 0 : ph + 1];
  if (launch_pdl(keep_dinv ? pcg_prep<true> : pcg_prep<false>, eg, dim3(kEwThreads), 0, st, n, ws.dinv,
                 (const double *)ws.r, (const double *)p_old, (const double *)p_old2, p_new, ws.x,
                 (const lsg_pcg_scalars *)ws.scal) != cudaSuccess)
    return check_launch("pcg_prep3d launch");
  int rc = check_launch("pcg_prep3d");
  if (rc) return rc;
  if (after_prep && cudaEventRecord(after_prep, st) != cudaSuccess) return check_launch("event");
  a.x = p_new;
  rc = dispatch<PCGQ>(op, a, ws.k, st);
  if (rc) return rc;
  if (launch_pdl(keep_dinv ? pcg_update<true> : pcg_update<false>, eg, dim3(kEwThreads), 0, st, n, ws.dinv,
                 ws.r, (const double *)ws.q, ws.scal, ws.partials, ws.counters) != cudaSuccess)
    return check_launch("pcg_update3d launch");
  return check_launch("pcg_update3d");
}

// The right-hand sides of one batch starting at r0 (pointer offsets only).
static lsg_pcg_ws sub_ws(const lsg_pcg_ws &ws, int r0, int k, int64_t n) {
  lsg_pcg_ws g = ws;
  const size_t off = (size_t)r0 * (size_t)n;
  g.k = k;
  g.x = ws.x + off;
  g.b = ws.b + off;
  g.r = ws.r + off;
  g.p = ws.p + off;
  g.q = ws.q + off;
  g.p_alt = ws.p_alt + off;
  g.p_ring = ws.p_ring + off;
  g.scal = ws.scal + r0;
  g.partials = ws.partials + (size_t)r0 * kMaxPartials * 8;
  g.counters = ws.counters + r0;
  return g;
}

// A batch of k >= 2 right-hand sides runs as two halves on two streams, the
// second half's iteration starting once the first half's p-pass is done, so
// that one half's HBM-bound elementwise passes can run beside the other
// half's fp64-bound stencil (cfg5: 471 -> 461 us per iteration; the stencil
// still takes every free SM, so the overlap is partial).  LSG_PCG3D_STREAMS=1
// keeps one stream.
static int streams3d() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_PCG3D_STREAMS");
    v = e ? atoi(e) : 2;
    if (v != 2) v = 1;
  }
  return v;
}

int pcg_iterate(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st) {
  const int64_t n = 3 * nodes_of(geo_of(op.grid));
  constexpr int ew = 4;  // elementwise CTAs per SM: the grid is one wave at 4 CTAs/SM
  auto grid_for = [&](int k) {
    int64_t need = ceil_div(n, (int64_t)kEwThreads * 4);
    int64_t slots = (int64_t)num_sms() * ew / k;
    if (slots < 1) slots = 1;
    return dim3((unsigned)(need < slots ? need : slots), (unsigned)k);
  };
  // seven vectors per right-hand side move per iteration; the M^-1 hint pays when
  // they exceed L2 several times over
  const int keep_dinv = (int64_t)ws.k * n * 8 * 7 > 4 * l2_bytes() ? 1 : 0;
  if (streams3d() == 2 && ws.k >= 2) {
    // library-owned second stream and events, one set per device
    constexpr int kMaxDev = 64;
    static cudaStream_t st2s[kMaxDev] = {};
    static cudaEvent_t evs[kMaxDev][3] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return check_launch("pcg3d device");
    if (!st2s[dev]) {
      if (cudaStreamCreateWithFlags(&st2s[dev], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&evs[dev][0], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&evs[dev][1], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&evs[dev][2], cudaEventDisableTiming) != cudaSuccess)
        return check_launch("pcg3d streams");
    }
    cudaStream_t st2 = st2s[dev];
    cudaEvent_t ev_fork = evs[dev][0], ev_prep = evs[dev][1], ev_join = evs[dev][2];
    const int k1 = ws.k / 2, k2 = ws.k - k1;
    const lsg_pcg_ws w1 = sub_ws(ws, 0, k1, n), w2 = sub_ws(ws, k1, k2, n);
    const dim3 g1 = grid_for(k1), g2 = grid_for(k2);
    if (cudaEventRecord(ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(st2, ev_fork, 0) != cudaSuccess)
      return check_launch("pcg3d fork");
    for (int it = 0; it < niter; ++it) {
      int rc = iterate_once(op, w1, ws.parity, n, g1, st, ev_prep, keep_dinv);
      if (rc) return rc;
      if (cudaStreamWaitEvent(st2, ev_prep, 0) != cudaSuccess) return check_launch("pcg3d wait");
      rc = iterate_once(op, w2, ws.parity, n, g2, st2, nullptr, keep_dinv);
      if (rc) return rc;
      ws.parity = ws.parity == 2 ? 0 : ws.parity + 1;
    }
    if (cudaEventRecord(ev_join, st2) != cudaSuccess || cudaStreamWaitEvent(st, ev_join, 0) != cudaSuccess)
      return check_launch("pcg3d join");
    return LSG_OK;
  }
  const dim3 eg = grid_for(ws.k);
  for (int it = 0; it < niter; ++it) {
    int rc = iterate_once(op, ws, ws.parity, n, eg, st, nullptr, keep_dinv);
    if (rc) return rc;
    ws.parity = ws.parity == 2 ? 0 : ws.parity + 1;
  }
  return LSG_OK;
}

// lsg_pcg_finish: apply the pending x updates of converged right-hand sides
// (after iteration L = iters - 1: alpha_L p_L and, for odd L, first
// alpha_{L-1} p_{L-1}), then clear the pending flags.
__global__ void __launch_bounds__(kEwThreads)
    pcg_finish_kernel(int64_t n, const double *r0, const double *r1, const double *r2, double *x,
                      const lsg_pcg_scalars *scal) {
  const int rhs = blockIdx.y;
  const lsg_pcg_scalars &s = scal[rhs];
  if (s.done == 0.0 || s.reserved[1] == 0.0) return;
  const int L = (int)s.iters - 1;
  const double *const ring[3] = {r0, r1, r2};
  const size_t off = (size_t)rhs * (size_t)n;
  const double *pL = ring[L % 3] + off, *pL1 = ring[(L + 2) % 3] + off;
  const double al = s.alpha, al2 = s.reserved[2];
  const bool two = s.reserved[1] > 1.5;
  for (int64_t t = (int64_t)blockIdx.x * kEwThreads + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * kEwThreads) {
    double xv = x[off + t];
    if (two) xv = fma(al2, pL1[t], xv);
    x[off + t] = fma(al, pL[t], xv);
  }
}

__global__ void clear_pending(int k, lsg_pcg_scalars *scal) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < k && scal[r].done != 0.0) scal[r].reserved[1] = 0.0;
}

int pcg_finish(const lsg_op &op, lsg_pcg_ws &ws, cudaStream_t st) {
  const int64_t n = 3 * nodes_of(geo_of(op.grid));
  int64_t nb = ceil_div(n, kEwThreads);
  if (nb > 4 * num_sms()) nb = 4 * num_sms();
  pcg_finish_kernel<<<dim3((unsigned)nb, (unsigned)ws.k), kEwThreads, 0, st>>>(
      n, ws.p, ws.p_alt, ws.p_ring, ws.x, ws.scal);
  int rc = check_launch("pcg_finish3d");
  if (rc) return rc;
  clear_pending<<<(unsigned)ceil_div(ws.k, 64), 64, 0, st>>>(ws.k, ws.scal);
  return check_launch("clear_pending3d");
}

template <int KB>
static int shape_chunk(const Geo &g, const lsg_op &op, const double *u, double volume, double *vc,
                       double *vv, double *out, double *partials, uint32_t *counter, int chunk,
                       cudaStream_t st) {
  Shape<KB> ph;
  const double vol = g.h[0] * g.h[1] * g.h[2] / 6.0;
  const double inside = op.p[3] > 0.0 ? op.p[3] : 1.0;
  ph.lam = op.p[0];
  ph.mu = op.p[1];
  ph.vol_t = vol;
  ph.inv_volume = 1.0 / volume;
  ph.w0 = vol * op.p[2];
  ph.w1 = vol * (inside - op.p[2]) / 4.0;
  for (int a = 0; a < 3; ++a) ph.ih[a] = g.ih[a];
  MArgs a = {};
  a.words = static_cast<const uint32_t *>(op.words);
  a.x = u;
  a.y = vc;
  a.y2 = vv;
  a.out = out;
  a.partials = partials;
  a.counters = counter;
  a.accumulate = chunk > 0;
  return launch<Shape<KB>, SHAPE>(ph, g, a, 1, st);
}

int shape_rhs(const lsg_op &op, int k, const double *u, double volume, double *vc, double *vv,
              double *out, double *partials, uint32_t *counter, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = nodes_of(g);
  int done = 0, chunk = 0;
  while (done < k) {
    const int left = k - done;
    const double *uc = u + (size_t)done * nn * 3;
    int rc, kb;
    (void)left;  // one state per launch in 3D (static shared memory of the 2-state variant > 48 KB)
    kb = 1;
    rc = shape_chunk<1>(g, op, uc, volume, vc, vv, out, partials, counter, chunk, st);
    if (rc) return rc;
    done += kb;
    ++chunk;
  }
  return LSG_OK;
}

int velocity_stats(const lsg_op &h1, const double *theta, const double *vec, double *out,
                   double *partials, uint32_t *counter, cudaStream_t st) {
  MArgs a = {};
  a.x = theta;
  a.x2 = vec;
  a.out = out;
  a.partials = partials;
  a.counters = counter;
  return dispatch<STATS>(h1, a, 1, st);
}

int material(const lsg_grid &grid, const double *phi, const uint8_t *bcmask, void *words,
             cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = nodes_of(g);
  material_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, phi, bcmask,
                                                               static_cast<uint32_t *>(words));
  return check_launch("material3d");
}

int indicator(const lsg_grid &grid, const double *phi, double *chi, cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nt = 6LL * g.nx * g.ny * g.nz;
  indicator_kernel<<<(unsigned)ceil_div(nt, 128), 128, 0, st>>>(g, phi, chi);
  return check_launch("indicator3d");
}

int h1_words(const lsg_grid &grid, const uint8_t *frozen_q, int zero_dirichlet, void *words,
             cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = nodes_of(g);
  h1_words_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, frozen_q, zero_dirichlet,
                                                               static_cast<uint32_t *>(words));
  return check_launch("h1_words3d");
}

int velocity_rhs(const lsg_op &h1, const double *vc, const double *vv, double lam, double *b,
                 cudaStream_t st) {
  const int64_t nn = nodes_of(geo_of(h1.grid));
  velocity_rhs_kernel<<<(unsigned)ceil_div(nn, 256), 256, 0, st>>>(
      nn, static_cast<const uint32_t *>(h1.words), vc, vv, lam, b);
  return check_launch("velocity_rhs3d");
}

int tensor_rhs(const lsg_grid &grid, const double *s0, const double *s1, double *vec,
               cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = nodes_of(g);
  tensor_rhs_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, s0, s1, vec);
  return check_launch("tensor_rhs3d");
}

int s1_tensor(const lsg_op &op, int k, const double *u, const double *phi, double *s1,
              cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nt = 6LL * g.nx * g.ny * g.nz;
  s1_kernel<<<(unsigned)ceil_div(nt, 128), 128, 0, st>>>(g, op.p[0], op.p[1], op.p[2],
                                                         op.p[3] > 0.0 ? op.p[3] : 1.0, k, u, phi, s1);
  return check_launch("s1_3d");
}

int cfl_speed(const lsg_grid &grid, const double *v, double *out, double *partials,
              uint32_t *counter, cudaStream_t st) {
  const Geo g = geo_of(grid);
  cfl_kernel<<<296, kEwThreads, 0, st>>>(nodes_of(g), g, v, partials, counter, out);
  return check_launch("cfl3d");
}

}  // namespace d3
}  // namespace lsg
