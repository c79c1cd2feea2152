// 2D structured P1 operators as warp-marching stencils (sm_100a, fp64).
//
// Layout (reference conventions, mesh.py:132-150, fem.py:88-96): node
// (i, j) has index j*(nx+1)+i; vector fields interleave (ux, uy) per node,
// so one node is one 16-byte double2 load.  Cell (i, j) holds the lower
// triangle (v(i,j), v(i+1,j), v(i+1,j+1)) and the upper triangle
// (v(i,j), v(i+1,j+1), v(i,j+1)).
//
// Execution: one warp owns a strip of 30 node columns (lanes 1..30; lanes 0
// and 31 are halo columns whose outputs are discarded) and a segment of node
// rows, and marches upward one node row at a time.  At every step each lane
// loads its node of the new row (coalesced 16 B/lane), fetches the right
// neighbour with one shuffle, evaluates the two triangles of its cell
// (i, row-1) from the four corner values held in registers, keeps the
// contributions to its own two corners and shuffles the two right-hand
// corner contributions to lane+1.  A node row is final after the cell rows
// below and above it have been visited, and is written exactly once.  No
// shared memory, no atomics: every node's sum is formed in a fixed order by
// one thread, so results are deterministic.
//
// HBM traffic per apply: 16 B read + 16 B written per node and RHS plus one
// material byte per node; halo columns (2/32) and one halo row per segment
// are re-read from L2.
#pragma once

#include "common.cuh"

namespace lsg {
namespace d2 {

constexpr int kStrip = 30;  // owned node columns per warp
constexpr int kWarps = 4;   // warps per CTA
constexpr int kThreads = kWarps * 32;

struct Geo {
  int nx, ny;
  double hx, hy;
};

// Node vectors of NC interleaved components (2: displacement / velocity,
// 1: temperature): one 16-byte or 8-byte access per node.
template <int NC>
__device__ __forceinline__ void ldg_node(const double *base, int64_t node, double *v) {
  if constexpr (NC == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2 *>(base) + node);
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = __ldg(base + node);
  }
}
template <int NC>
__device__ __forceinline__ void ld_node(const double *base, int64_t node, double *v) {
  if constexpr (NC == 2) {
    const double2 t = reinterpret_cast<const double2 *>(base)[node];
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = base[node];
  }
}
template <int NC>
__device__ __forceinline__ void st_node(double *base, int64_t node, const double *v) {
  if constexpr (NC == 2) reinterpret_cast<double2 *>(base)[node] = make_double2(v[0], v[1]);
  else base[node] = v[0];
}

// ---------------------------------------------------------------------------
// Elasticity (fem.py:397-411).  Word (uint8, written by lsg_material):
//   bits 0-1 n_in of the lower triangle, bits 2-3 n_in of the upper triangle
//   (number of its three edge-midpoint quadrature points with phi < 0),
//   bit 4 cell valid, bit 5 / 6 Dirichlet on ux / uy of the node.
// Element weight w = |T| * abar, abar = (n_in + (3 - n_in) * ersatz) / 3
// (evaluated as w0 + w1 n_in: no table, so no local-memory indexing),
// which equals sum_q (|T|/3) A_q of the reference's coefficient.
// With raw differences dP = u(right) - u(left), dQ = u(top) - u(bottom):
//   A = w/hx * sigma e_x = w (k1 dPx + k2 dQy, k3 dPy + k4 dQx)
//   B = w/hy * sigma e_y = w (k4 dPy + k5 dQx, k2 dPx + k6 dQy)
// lower: r_a = -A, r_b = A - B, r_c = B ; upper: r_a = -B, r_c = A, r_d = B - A.
// ---------------------------------------------------------------------------
struct Elast {
  static constexpr int NC = 2, NIN = 2, NOUT = 2;
  double k1, k2, k3, k4, k5, k6;
  double w0, w1;  // w(n_in) = w0 + w1 * n_in = |T| (n_in + (3 - n_in) ersatz) / 3

  __device__ __forceinline__ double wof(uint32_t n) const { return fma((double)n, w1, w0); }

  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 4) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return (w >> 5) & 3u; }

  __device__ __forceinline__ void tri(double dPx, double dPy, double dQx, double dQy, double w,
                                      double &Ax, double &Ay, double &Bx, double &By) const {
    Ax = w * fma(k1, dPx, k2 * dQy);
    Ay = w * fma(k3, dPy, k4 * dQx);
    Bx = w * fma(k4, dPy, k5 * dQx);
    By = w * fma(k2, dPx, k6 * dQy);
  }

  __device__ __forceinline__ void cell(const double *u00, const double *u10, const double *u01,
                                       const double *u11, uint32_t word, int, int, double *c00,
                                       double *c10, double *c01, double *c11) const {
    double wl, wu;
    weights(word, wl, wu);
    cell_w(u00, u10, u01, u11, wl, wu, c00, c10, c01, c11);
  }
  // element weights of the cell's lower / upper triangle (0 for invalid cells)
  __device__ __forceinline__ void weights(uint32_t word, double &wl, double &wu) const {
    const double v = valid(word) ? 1.0 : 0.0;
    wl = wof(word & 3u) * v;
    wu = wof((word >> 2) & 3u) * v;
  }
  // the cell with its weights given (shared by several right-hand sides)
  __device__ __forceinline__ void cell_w(const double *u00, const double *u10, const double *u01,
                                         const double *u11, double wl, double wu, double *c00,
                                         double *c10, double *c01, double *c11) const {
    double ALx, ALy, BLx, BLy, AUx, AUy, BUx, BUy;
    // lower (a=00, b=10, c=11): dP = u10 - u00, dQ = u11 - u10
    tri(u10[0] - u00[0], u10[1] - u00[1], u11[0] - u10[0], u11[1] - u10[1], wl, ALx, ALy, BLx, BLy);
    // upper (a=00, c=11, d=01): dP = u11 - u01, dQ = u01 - u00
    tri(u11[0] - u01[0], u11[1] - u01[1], u01[0] - u00[0], u01[1] - u00[1], wu, AUx, AUy, BUx, BUy);
    c00[0] = -ALx - BUx;  c00[1] = -ALy - BUy;
    c10[0] = ALx - BLx;   c10[1] = ALy - BLy;
    c11[0] = BLx + AUx;   c11[1] = BLy + AUy;
    c01[0] = BUx - AUx;   c01[1] = BUy - AUy;
  }

  // Jacobi diagonal of node (i, j) from the words of cells (i,j), (i-1,j),
  // (i,j-1), (i-1,j-1): sum_e w_e ((lam+mu)(d_c N)^2 + mu |grad N|^2).
  __device__ __forceinline__ void diag(uint32_t w00, uint32_t wm0, uint32_t w0m, uint32_t wmm,
                                       double *d) const {
    auto wl = [&](uint32_t w) { return valid(w) ? wof(w & 3u) : 0.0; };
    auto wu = [&](uint32_t w) { return valid(w) ? wof((w >> 2) & 3u) : 0.0; };
    const double wx = wl(w00) + wu(wmm);   // gradient (+-1/hx, 0)
    const double wy = wu(w00) + wl(wmm);   // gradient (0, +-1/hy)
    const double wxy = wl(wm0) + wu(w0m);  // gradient (+-1/hx, -+1/hy)
    d[0] = (wx + wxy) * k1 + (wy + wxy) * k5;
    d[1] = (wx + wxy) * k3 + (wy + wxy) * k6;
  }
};

// ---------------------------------------------------------------------------
// Scalar diffusion (a grad u, grad v) with the ersatz conductivity of the heat
// models (models/heat.py:113-119, fem.py:388-394).  Same material word as
// Elast (bit 5 = Dirichlet on the node).  With dP = u(right) - u(left),
// dQ = u(top) - u(bottom) the fluxes are X = w dP / hx^2, Y = w dQ / hy^2:
// lower r_a = -X, r_b = X - Y, r_c = Y ; upper r_a = -Y, r_c = X, r_d = Y - X.
// ---------------------------------------------------------------------------
struct Lap {
  static constexpr int NC = 1, NIN = 1, NOUT = 1;
  double w0, w1;      // |T| abar(n_in) = w0 + w1 n_in
  double ihx2, ihy2;  // 1 / hx^2, 1 / hy^2

  __device__ __forceinline__ double wof(uint32_t n) const { return fma((double)n, w1, w0); }
  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 4) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return (w >> 5) & 1u; }

  __device__ __forceinline__ void cell(const double *u00, const double *u10, const double *u01,
                                       const double *u11, uint32_t word, int, int, double *c00,
                                       double *c10, double *c01, double *c11) const {
    double wl, wu;
    weights(word, wl, wu);
    cell_w(u00, u10, u01, u11, wl, wu, c00, c10, c01, c11);
  }
  // element weights of the cell's lower / upper triangle (0 for invalid cells)
  __device__ __forceinline__ void weights(uint32_t word, double &wl, double &wu) const {
    const double v = valid(word) ? 1.0 : 0.0;
    wl = wof(word & 3u) * v;
    wu = wof((word >> 2) & 3u) * v;
  }
  // the cell with its weights given (shared by several right-hand sides)
  __device__ __forceinline__ void cell_w(const double *u00, const double *u10, const double *u01,
                                         const double *u11, double wl, double wu, double *c00,
                                         double *c10, double *c01, double *c11) const {
    const double XL = wl * ihx2 * (u10[0] - u00[0]), YL = wl * ihy2 * (u11[0] - u10[0]);
    const double XU = wu * ihx2 * (u11[0] - u01[0]), YU = wu * ihy2 * (u01[0] - u00[0]);
    c00[0] = -XL - YU;
    c10[0] = XL - YL;
    c11[0] = YL + XU;
    c01[0] = YU - XU;
  }

  // sum_e w_e |grad N|^2 over the six triangles around the node
  __device__ __forceinline__ void diag(uint32_t w00, uint32_t wm0, uint32_t w0m, uint32_t wmm,
                                       double *d) const {
    auto wl = [&](uint32_t w) { return valid(w) ? wof(w & 3u) : 0.0; };
    auto wu = [&](uint32_t w) { return valid(w) ? wof((w >> 2) & 3u) : 0.0; };
    d[0] = (wl(w00) + wu(wmm)) * ihx2 + (wu(w00) + wl(wmm)) * ihy2 +
           (wl(wm0) + wu(w0m)) * (ihx2 + ihy2);
  }
};

// ---------------------------------------------------------------------------
// H1 velocity form (velocity.py:98-127), componentwise:
//   B = mw M + sw K_lap + fp M_frozen + np * boundary normal mass.
// Word (uint8, lsg_h1_words): bits 0-2 frozen flags of the lower triangle's
// quadrature points (edges (0,1), (1,2), (0,2)), bits 3-5 the upper's,
// bit 6 Dirichlet (both components), bit 7 cell valid.
// ---------------------------------------------------------------------------
struct H1 {
  static constexpr int NC = 2, NIN = 2, NOUT = 2;
  int nx, ny;
  double m;       // mw * |T| / 12
  double ax, ay;  // sw * |T| / hx^2, sw * |T| / hy^2
  double fz;      // fp * |T| / 3 * 0.5 * 0.5 (per frozen quadrature point and vertex)
  double nbx, nby;  // npen * hx / 6, npen * hy / 6 (facet mass along bottom/top, left/right)

  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 7) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t w) { return ((w >> 6) & 1u) ? 3u : 0u; }

  __device__ __forceinline__ void cell(const double *u00, const double *u10, const double *u01,
                                       const double *u11, uint32_t word, int i, int j, double *c00,
                                       double *c10, double *c01, double *c11) const {
    if (!valid(word)) {
#pragma unroll
      for (int c = 0; c < 2; ++c) c00[c] = c10[c] = c01[c] = c11[c] = 0.0;
      return;
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      // lower (00, 10, 11)
      const double dxl = u10[c] - u00[c], dyl = u11[c] - u10[c];
      const double sl = u00[c] + u10[c] + u11[c];
      // upper (00, 11, 01)
      const double dxu = u11[c] - u01[c], dyu = u01[c] - u00[c];
      const double su = u00[c] + u11[c] + u01[c];
      double r00 = -ax * dxl - ay * dyu + m * (2.0 * u00[c] + sl + su);
      double r10 = ax * dxl - ay * dyl + m * (u10[c] + sl);
      double r11 = ay * dyl + ax * dxu + m * (2.0 * u11[c] + sl + su);
      double r01 = -ax * dxu + ay * dyu + m * (u01[c] + su);
      if (word & 0x3fu) {  // frozen mass at edge midpoints
        const double e0 = 0.5 * (u00[c] + u10[c]), e1 = 0.5 * (u10[c] + u11[c]);
        const double e2 = 0.5 * (u00[c] + u11[c]);
        const double f0 = 0.5 * (u00[c] + u11[c]), f1 = 0.5 * (u11[c] + u01[c]);
        const double f2 = 0.5 * (u00[c] + u01[c]);
        const double b0 = (word & 1u) ? 2.0 * fz : 0.0, b1 = (word & 2u) ? 2.0 * fz : 0.0;
        const double b2 = (word & 4u) ? 2.0 * fz : 0.0, b3 = (word & 8u) ? 2.0 * fz : 0.0;
        const double b4 = (word & 16u) ? 2.0 * fz : 0.0, b5 = (word & 32u) ? 2.0 * fz : 0.0;
        r00 += b0 * e0 + b2 * e2 + b3 * f0 + b5 * f2;
        r10 += b0 * e0 + b1 * e1;
        r11 += b1 * e1 + b2 * e2 + b3 * f0 + b4 * f1;
        r01 += b4 * f1 + b5 * f2;
      }
      // boundary normal penalty: normal y on bottom/top, x on left/right
      if (c == 1) {
        if (j == 0) { r00 += nbx * (2.0 * u00[1] + u10[1]); r10 += nbx * (u00[1] + 2.0 * u10[1]); }
        if (j == ny - 1) { r01 += nbx * (2.0 * u01[1] + u11[1]); r11 += nbx * (u01[1] + 2.0 * u11[1]); }
      } else {
        if (i == 0) { r00 += nby * (2.0 * u00[0] + u01[0]); r01 += nby * (u00[0] + 2.0 * u01[0]); }
        if (i == nx - 1) { r10 += nby * (2.0 * u10[0] + u11[0]); r11 += nby * (u10[0] + 2.0 * u11[0]); }
      }
      c00[c] = r00; c10[c] = r10; c11[c] = r11; c01[c] = r01;
    }
  }

  // Diagonal contributions of one cell to the corner `corner`
  // (0: 00, 1: 10, 2: 01, 3: 11) for cell (i, j).
  __device__ __forceinline__ void corner_diag(uint32_t w, int corner, int i, int j, double *d) const {
    if (!valid(w)) return;
    double lap = 0.0, mass = 0.0, fr = 0.0;
    switch (corner) {
      case 0:  // lower a (x-type), upper a (y-type)
        lap = ax + ay; mass = 4.0 * m;
        fr = ((w & 1u) ? 1 : 0) + ((w & 4u) ? 1 : 0) + ((w & 8u) ? 1 : 0) + ((w & 32u) ? 1 : 0);
        break;
      case 1:  // lower b (xy-type)
        lap = ax + ay; mass = 2.0 * m;
        fr = ((w & 1u) ? 1 : 0) + ((w & 2u) ? 1 : 0);
        break;
      case 3:  // lower c (y-type), upper c (x-type)
        lap = ax + ay; mass = 4.0 * m;
        fr = ((w & 2u) ? 1 : 0) + ((w & 4u) ? 1 : 0) + ((w & 8u) ? 1 : 0) + ((w & 16u) ? 1 : 0);
        break;
      default:  // 2: upper d (xy-type)
        lap = ax + ay; mass = 2.0 * m;
        fr = ((w & 16u) ? 1 : 0) + ((w & 32u) ? 1 : 0);
        break;
    }
    const double base = lap + mass + fr * fz;
    double nx_ = 0.0, ny_ = 0.0;
    const int ci = (corner & 1), cj = (corner >> 1);  // corner offsets
    if (j == 0 && cj == 0) ny_ += 2.0 * nbx;
    if (j == ny - 1 && cj == 1) ny_ += 2.0 * nbx;
    if (i == 0 && ci == 0) nx_ += 2.0 * nby;
    if (i == nx - 1 && ci == 1) nx_ += 2.0 * nby;
    d[0] += base + nx_;
    d[1] += base + ny_;
  }

  __device__ __forceinline__ void diag(uint32_t w00, uint32_t wm0, uint32_t w0m, uint32_t wmm,
                                       int i, int j, double *d) const {
    d[0] = d[1] = 0.0;
    corner_diag(w00, 0, i, j, d);
    corner_diag(wm0, 1, i - 1, j, d);
    corner_diag(w0m, 2, i, j - 1, d);
    corner_diag(wmm, 3, i - 1, j - 1, d);
  }
};

}  // namespace d2
}  // namespace lsg
