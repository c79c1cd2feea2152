// Inverse-elasticity model kernels (reference models/inverse.py), 2D.
//
// The model's states and adjoints are ordinary batched elasticity solves
// (ops2d.cu); what is specific to it is
//   * the misfit pass (inverse.py:180-233): e = u - v - g, f = u - g,
//     M e (P1 mass, edge-midpoint rule, exact: |T|/12 (1 + delta_ab)),
//     M_G f (facet mass on the measured facets, 2-point Gauss, exact:
//     |f|/6 (1 + delta_ab)), the adjoint right-hand sides
//       head = -alpha M e - beta M_G f (zeroed on the partial clamp),
//       tail = alpha M e (zeroed on the whole boundary),
//     and the cost J = sum_k alpha/2 e.Me + beta/2 f.M_G f -- one node-gather
//     pass, deterministic (fixed-order block reduction, no atomics);
//   * the S0 / S1 tensors of the Kohn-Vogelius derivative (inverse.py:235-279)
//     per triangle and quadrature point, contracted afterwards by the
//     node-gather tensor_rhs kernel;
//   * the right-hand sides of the strain projections (inverse.py:142-155).
#include <math.h>

#include "common.cuh"
#include "ops.h"

namespace lsg {
namespace inv {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 1024;

struct G2 {
  int nx, ny;
  double hx, hy;
};

static G2 geo(const lsg_grid &g) {
  G2 o;
  o.nx = g.n[0];
  o.ny = g.n[1];
  o.hx = (g.hi[0] - g.lo[0]) / g.n[0];
  o.hy = (g.hi[1] - g.lo[1]) / g.n[1];
  return o;
}

// Mass stencil of node (i, j): (M x)_a = |T|/12 sum_{T ∋ a} (2 x_a + sum_{b in T, b != a} x_b).
// `val(ii, jj, c)` returns component c of the field at node (ii, jj).
template <class F>
__device__ __forceinline__ void mass_at(const G2 &g, int i, int j, F val, double *out) {
  const double w = 0.5 * g.hx * g.hy / 12.0;
  const bool cL = i > 0, cR = i < g.nx, cB = j > 0, cT = j < g.ny;
  for (int c = 0; c < 2; ++c) {
    const double xa = val(i, j, c);
    double s = 0.0;
    int nt = 0;
    if (cR && cT) {  // cell (i, j): lower (00,10,11), upper (00,11,01)
      s += val(i + 1, j, c) + val(i + 1, j + 1, c);
      s += val(i + 1, j + 1, c) + val(i, j + 1, c);
      nt += 2;
    }
    if (cL && cT) {  // cell (i-1, j): node is 10 of the lower triangle (00, 10, 11)
      s += val(i - 1, j, c) + val(i, j + 1, c);
      nt += 1;
    }
    if (cR && cB) {  // cell (i, j-1): node is 01 of the upper triangle (00, 11, 01)
      s += val(i, j - 1, c) + val(i + 1, j, c);
      nt += 1;
    }
    if (cL && cB) {  // cell (i-1, j-1): node is 11 of both triangles
      s += val(i - 1, j - 1, c) + val(i, j - 1, c);
      s += val(i - 1, j - 1, c) + val(i - 1, j, c);
      nt += 2;
    }
    out[c] = w * (2.0 * nt * xa + s);
  }
}

// flags bit 0: facet (node, node+1) is measured; bit 1: facet (node, node+nx+1)
__global__ void misfit_kernel(G2 g, int k, const double *u, const double *v, const double *gm,
                              const uint8_t *flags, const uint8_t *pmask, double alpha, double beta,
                              double *head, double *tail, double *partials, uint32_t *counter,
                              double *out) {
  __shared__ double scratch[kThreads / 32];
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  double part[1] = {0.0};
  for (int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; node < nn;
       node += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
    const bool bnd = i == 0 || j == 0 || i == g.nx || j == g.ny;
    const uint32_t pm = pmask ? pmask[node] : 0u;
    const uint32_t fr = flags[node], fl = i > 0 ? flags[node - 1] : 0u;
    const uint32_t fu = flags[node], fd = j > 0 ? flags[node - nxp] : 0u;
    for (int r = 0; r < k; ++r) {
      const size_t off = (size_t)r * nn * 2;
      auto e = [&](int ii, int jj, int c) {
        const int64_t n = (int64_t)jj * nxp + ii;
        return u[off + n * 2 + c] - v[off + n * 2 + c] - gm[off + n * 2 + c];
      };
      auto f = [&](int64_t n, int c) { return u[off + n * 2 + c] - gm[off + n * 2 + c]; };
      double me[2];
      mass_at(g, i, j, e, me);
      double mf[2] = {0.0, 0.0};
      for (int c = 0; c < 2; ++c) {
        const double fa = f(node, c);
        if (fr & 1u) mf[c] += g.hx / 6.0 * (2.0 * fa + f(node + 1, c));
        if (fl & 1u) mf[c] += g.hx / 6.0 * (2.0 * fa + f(node - 1, c));
        if (fu & 2u) mf[c] += g.hy / 6.0 * (2.0 * fa + f(node + nxp, c));
        if (fd & 2u) mf[c] += g.hy / 6.0 * (2.0 * fa + f(node - nxp, c));
        const double ea = e(i, j, c);
        part[0] += 0.5 * alpha * ea * me[c] + 0.5 * beta * fa * mf[c];
        const double h = -alpha * me[c] - beta * mf[c];
        head[off + node * 2 + c] = ((pm >> c) & 1u) ? 0.0 : h;
        tail[off + node * 2 + c] = bnd ? 0.0 : alpha * me[c];
      }
    }
  }
  double tot[1];
  if (block_partial_and_total<1, 0u>(part, partials, counter, blockIdx.x, gridDim.x, scratch, tot))
    if (threadIdx.x == 0) out[0] = tot[0];
}

// Triangle t of cell (i, j): vertex nodes (reference order) and the
// constant gradients of their basis functions.
struct Tri {
  int64_t n[3];
  double gx[3], gy[3];
};

__device__ __forceinline__ Tri tri_of(const G2 &g, int i, int j, bool upper) {
  const int64_t nxp = g.nx + 1;
  const int64_t n00 = (int64_t)j * nxp + i, n10 = n00 + 1, n01 = n00 + nxp, n11 = n01 + 1;
  const double ax = 1.0 / g.hx, ay = 1.0 / g.hy;
  Tri t;
  if (!upper) {  // (00, 10, 11)
    t.n[0] = n00; t.n[1] = n10; t.n[2] = n11;
    t.gx[0] = -ax; t.gy[0] = 0.0;
    t.gx[1] = ax;  t.gy[1] = -ay;
    t.gx[2] = 0.0; t.gy[2] = ay;
  } else {  // (00, 11, 01)
    t.n[0] = n00; t.n[1] = n11; t.n[2] = n01;
    t.gx[0] = 0.0; t.gy[0] = -ay;
    t.gx[1] = ax;  t.gy[1] = 0.0;
    t.gx[2] = -ax; t.gy[2] = ay;
  }
  return t;
}

// jac[a][b] = d u_a / d x_b
__device__ __forceinline__ void jac_of(const Tri &t, const double *f, double (&J)[2][2]) {
  J[0][0] = J[0][1] = J[1][0] = J[1][1] = 0.0;
  for (int v = 0; v < 3; ++v) {
    const double fx = f[t.n[v] * 2], fy = f[t.n[v] * 2 + 1];
    J[0][0] += fx * t.gx[v];
    J[0][1] += fx * t.gy[v];
    J[1][0] += fy * t.gx[v];
    J[1][1] += fy * t.gy[v];
  }
}

__device__ __forceinline__ void stress_of(const double (&J)[2][2], double lam, double mu,
                                          double (&S)[2][2]) {
  const double exy = 0.5 * (J[0][1] + J[1][0]);
  const double tr = J[0][0] + J[1][1];
  S[0][0] = 2.0 * mu * J[0][0] + lam * tr;
  S[1][1] = 2.0 * mu * J[1][1] + lam * tr;
  S[0][1] = S[1][0] = 2.0 * mu * exy;
}

// sigma : eps(J)
__device__ __forceinline__ double pair_of(const double (&S)[2][2], const double (&J)[2][2]) {
  return S[0][0] * J[0][0] + S[1][1] * J[1][1] + S[0][1] * (J[0][1] + J[1][0]);
}

__device__ __forceinline__ int neg_mid(double a, double b) { return (0.5 * a + 0.5 * b) < 0.0; }

// S0 (E, 3, 2) and S1 (E, 3, 2, 2) of the Kohn-Vogelius misfit, summed over
// the k measurement pairs (inverse.py:235-279).  proj = (k, 3, 2N): nodal
// projections of eps_xx, eps_xy, eps_yy of g, each stored as (value, 0).
__global__ void tensors_kernel(G2 g, int k, const double *u, const double *v, const double *p,
                               const double *q, const double *gm, const double *proj,
                               const double *phi, double a_in, double a_out, double lam, double mu,
                               double alpha, double *s0, double *s1) {
  const int64_t ncell = (int64_t)g.nx * g.ny;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * ncell) return;
  const int64_t c = t >> 1;
  const bool upper = t & 1;
  const int j = (int)(c / g.nx), i = (int)(c - (int64_t)j * g.nx);
  const Tri T = tri_of(g, i, j, upper);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  // quadrature points on edges (0,1), (1,2), (0,2) (fem.py:43-45)
  const int qa[3] = {0, 1, 0}, qb[3] = {1, 2, 2};
  double aq[3];
  for (int qq = 0; qq < 3; ++qq)
    aq[qq] = neg_mid(phi[T.n[qa[qq]]], phi[T.n[qb[qq]]]) ? a_in : a_out;
  double S0[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  double S1[3][2][2] = {};
  for (int r = 0; r < k; ++r) {
    const size_t off = (size_t)r * nn * 2;
    double Ju[2][2], Jv[2][2], Jp[2][2], Jq[2][2], Jg[2][2], Jy[2][2];
    jac_of(T, u + off, Ju);
    jac_of(T, v + off, Jv);
    jac_of(T, p + off, Jp);
    jac_of(T, q + off, Jq);
    jac_of(T, gm + off, Jg);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) Jy[a][b] = Jv[a][b] + Jg[a][b];
    double Su[2][2], Sp[2][2], Sq[2][2], Sy[2][2];
    stress_of(Ju, lam, mu, Su);
    stress_of(Jp, lam, mu, Sp);
    stress_of(Jq, lam, mu, Sq);
    stress_of(Jy, lam, mu, Sy);
    // gradients of the projected strain components: ge[comp][d], comp = xx, xy, yy
    double ge[3][2];
    for (int cc = 0; cc < 3; ++cc) {
      const double *P = proj + ((size_t)r * 3 + cc) * nn * 2;
      ge[cc][0] = ge[cc][1] = 0.0;
      for (int vv = 0; vv < 3; ++vv) {
        ge[cc][0] += P[T.n[vv] * 2] * T.gx[vv];
        ge[cc][1] += P[T.n[vv] * 2] * T.gy[vv];
      }
    }
    // drift_d = sum_ij sig_q[i][j] d/dx_d eps_g[i][j]
    double drift[2];
    for (int d = 0; d < 2; ++d)
      drift[d] = Sq[0][0] * ge[0][d] + 2.0 * Sq[0][1] * ge[1][d] + Sq[1][1] * ge[2][d];
    const double pairing = pair_of(Su, Jp) + pair_of(Sy, Jq);
    double M[2][2];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b)
        M[a][b] = Ju[0][a] * Sp[0][b] + Ju[1][a] * Sp[1][b] + Jp[0][a] * Su[0][b] +
                  Jp[1][a] * Su[1][b] + Jv[0][a] * Sq[0][b] + Jv[1][a] * Sq[1][b] +
                  Jq[0][a] * Sy[0][b] + Jq[1][a] * Sy[1][b];
    for (int qq = 0; qq < 3; ++qq) {
      double bulk[2];
      for (int cc = 0; cc < 2; ++cc) {
        const int64_t na = T.n[qa[qq]], nb = T.n[qb[qq]];
        const double ea = u[off + na * 2 + cc] - v[off + na * 2 + cc] - gm[off + na * 2 + cc];
        const double eb = u[off + nb * 2 + cc] - v[off + nb * 2 + cc] - gm[off + nb * 2 + cc];
        bulk[cc] = 0.5 * ea + 0.5 * eb;
      }
      for (int d = 0; d < 2; ++d)
        S0[qq][d] += -alpha * (Jg[0][d] * bulk[0] + Jg[1][d] * bulk[1]) + aq[qq] * drift[d];
      const double scal = 0.5 * alpha * (bulk[0] * bulk[0] + bulk[1] * bulk[1]) + aq[qq] * pairing;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) S1[qq][a][b] += (a == b ? scal : 0.0) - aq[qq] * M[a][b];
    }
  }
  for (int qq = 0; qq < 3; ++qq) {
    for (int d = 0; d < 2; ++d) s0[(t * 3 + qq) * 2 + d] = S0[qq][d];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) s1[((t * 3 + qq) * 2 + a) * 2 + b] = S1[qq][a][b];
  }
}

// Right-hand sides of the strain projections: out (k, 3, 2N), component cc
// of pair r = sum_{T ∋ a} |T|/3 eps_cc(g_r)|_T, stored as (value, 0).
__global__ void strain_rhs_kernel(G2 g, int k, const double *gm, double *out) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  const double w = 0.5 * g.hx * g.hy / 3.0;
  for (int r = 0; r < k; ++r) {
    const double *G = gm + (size_t)r * nn * 2;
    double acc[3] = {0.0, 0.0, 0.0};
    // the (up to) six triangles around the node
    const int ci[4] = {i, i - 1, i, i - 1}, cj[4] = {j, j, j - 1, j - 1};
    for (int cc = 0; cc < 4; ++cc) {
      if (ci[cc] < 0 || cj[cc] < 0 || ci[cc] >= g.nx || cj[cc] >= g.ny) continue;
      for (int up = 0; up < 2; ++up) {
        // which triangles of the cell contain the node
        const bool has = (cc == 0) || (cc == 3) || (cc == 1 && !up) || (cc == 2 && up);
        if (!has) continue;
        const Tri T = tri_of(g, ci[cc], cj[cc], up);
        double J[2][2];
        jac_of(T, G, J);
        acc[0] += w * J[0][0];
        acc[1] += w * 0.5 * (J[0][1] + J[1][0]);
        acc[2] += w * J[1][1];
      }
    }
    for (int cc = 0; cc < 3; ++cc) {
      double *O = out + ((size_t)r * 3 + cc) * nn * 2;
      O[node * 2] = acc[cc];
      O[node * 2 + 1] = 0.0;
    }
  }
}

}  // namespace inv

int inverse_misfit(const lsg_grid &grid, int k, const double *u, const double *v, const double *g,
                   const uint8_t *flags, const uint8_t *pmask, double alpha, double beta,
                   double *head, double *tail, double *out, double *partials, uint32_t *counter,
                   cudaStream_t st) {
  const inv::G2 g2 = inv::geo(grid);
  const int64_t nn = (int64_t)(g2.nx + 1) * (g2.ny + 1);
  int64_t nb = ceil_div(nn, inv::kThreads);
  if (nb > inv::kMaxBlocks) nb = inv::kMaxBlocks;
  inv::misfit_kernel<<<(unsigned)nb, inv::kThreads, 0, st>>>(g2, k, u, v, g, flags, pmask, alpha,
                                                             beta, head, tail, partials, counter,
                                                             out);
  return check_launch("inverse_misfit");
}

int inverse_tensors(const lsg_grid &grid, int k, const double *u, const double *v, const double *p,
                    const double *q, const double *g, const double *proj, const double *phi,
                    double a_in, double a_out, double lam, double mu, double alpha, double *s0,
                    double *s1, cudaStream_t st) {
  const inv::G2 g2 = inv::geo(grid);
  const int64_t ne = 2 * (int64_t)g2.nx * g2.ny;
  inv::tensors_kernel<<<(unsigned)ceil_div(ne, 128), 128, 0, st>>>(
      g2, k, u, v, p, q, g, proj, phi, a_in, a_out, lam, mu, alpha, s0, s1);
  return check_launch("inverse_tensors");
}

int strain_projection_rhs(const lsg_grid &grid, int k, const double *g, double *out,
                          cudaStream_t st) {
  const inv::G2 g2 = inv::geo(grid);
  const int64_t nn = (int64_t)(g2.nx + 1) * (g2.ny + 1);
  inv::strain_rhs_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g2, k, g, out);
  return check_launch("strain_projection_rhs");
}

}  // namespace lsg
