// The 2D warp-marching kernel and its per-action epilogues (see march2d.cuh
// for the data layout and the operator physics).
#pragma once

#include "march2d.cuh"

namespace lsg {
namespace d2 {

enum Act { APPLY = 0, RESID = 1, PCG = 2, STATS = 3, SHAPE = 4 };

#ifndef LSG_M2_PCG_MINB
#define LSG_M2_PCG_MINB 1  // resident CTAs per SM the PCG pass is register-capped for
#endif

// Arguments shared by every marching launch (unused fields stay null).
struct MArgs {
  const void *words;
  const double *x;     // APPLY/RESID/STATS: input field ; PCG: r_{i-1} ; SHAPE: u (KB fields)
  const double *x2;    // PCG: p_{i-1} ; STATS: vec
  const double *x3;    // PCG: q_{i-1}
  const double *b;     // RESID: b
  double *y;           // APPLY: y ; RESID: r ; PCG: q_i ; SHAPE: vec_cost
  double *y2;          // PCG: p_i ; SHAPE: vec_vol
  double *y3;          // PCG: r_i
  const double *dinv;  // RESID / PCG: inverse Jacobi diagonal (1 on Dirichlet dofs)
  double *xs;          // PCG: the iterate x (x += alpha_{i-1} p_{i-1} is done here)
  lsg_pcg_scalars *scal;
  double *partials;
  uint32_t *counters;
  double *out;         // STATS / SHAPE scalar outputs
  int seg;             // node rows per segment
  int nstrips;
  int accumulate;      // SHAPE: add into vec_cost / out[0] (later RHS chunks)
};

// Compliance + shape-derivative physics for KB load cases at once
// (compliance.py:111-139, base.py:150-158, velocity.py:129-142).
// in = KB displacement fields, out = (vec_cost[2], vec_vol[2]).
template <int KB>
struct Shape {
  static constexpr int NC = 2, NIN = 2 * KB, NOUT = 4;
  double lam, mu, area, inv_hx, inv_hy, inv_volume;
  double w0, w1;  // |T| * abar(n_in) = w0 + w1 n_in

  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 4) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t) { return 0u; }

  // bulk = sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I), row-major; dens = sum_k sigma:eps.
  __device__ __forceinline__ void tri(const double *dP, const double *dQ, double *bulk,
                                      double &dens) const {
    bulk[0] = bulk[1] = bulk[2] = bulk[3] = 0.0;
    dens = 0.0;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const double Px = dP[2 * k] * inv_hx, Py = dP[2 * k + 1] * inv_hx;
      const double Qx = dQ[2 * k] * inv_hy, Qy = dQ[2 * k + 1] * inv_hy;
      const double exx = Px, eyy = Qy, exy = 0.5 * (Py + Qx);
      const double tr = exx + eyy;
      const double sxx = 2.0 * mu * exx + lam * tr, syy = 2.0 * mu * eyy + lam * tr;
      const double sxy = 2.0 * mu * exy;
      const double d = sxx * exx + syy * eyy + 2.0 * sxy * exy;
      bulk[0] += 2.0 * (Px * sxx + Py * sxy) - d;  // G = [[Px, Qx], [Py, Qy]]
      bulk[1] += 2.0 * (Px * sxy + Py * syy);
      bulk[2] += 2.0 * (Qx * sxx + Qy * sxy);
      bulk[3] += 2.0 * (Qx * sxy + Qy * syy) - d;
      dens += d;
    }
  }

  __device__ __forceinline__ void cell(const double *u00, const double *u10, const double *u01,
                                       const double *u11, uint32_t word, bool count, int, int,
                                       double *c00, double *c10, double *c01, double *c11,
                                       double *part) const {
    const bool ok = valid(word);
    const uint32_t nl = ok ? (word & 3u) : 0u, nu = ok ? ((word >> 2) & 3u) : 0u;
    const double wl = ok ? fma((double)nl, w1, w0) : 0.0, wu = ok ? fma((double)nu, w1, w0) : 0.0;
    double dP[NIN], dQ[NIN], bl[4], bu[4], dl, du;
#pragma unroll
    for (int t = 0; t < NIN; ++t) { dP[t] = u10[t] - u00[t]; dQ[t] = u11[t] - u10[t]; }
    tri(dP, dQ, bl, dl);  // lower (00, 10, 11)
#pragma unroll
    for (int t = 0; t < NIN; ++t) { dP[t] = u11[t] - u01[t]; dQ[t] = u01[t] - u00[t]; }
    tri(dP, dQ, bu, du);  // upper (00, 11, 01)
    // cost part: X = w bulk (1/hx, 0), Y = w bulk (0, 1/hy)
    const double XLx = wl * bl[0] * inv_hx, XLy = wl * bl[2] * inv_hx;
    const double YLx = wl * bl[1] * inv_hy, YLy = wl * bl[3] * inv_hy;
    const double XUx = wu * bu[0] * inv_hx, XUy = wu * bu[2] * inv_hx;
    const double YUx = wu * bu[1] * inv_hy, YUy = wu * bu[3] * inv_hy;
    c00[0] = -XLx - YUx;  c00[1] = -XLy - YUy;
    c10[0] = XLx - YLx;   c10[1] = XLy - YLy;
    c11[0] = YLx + XUx;   c11[1] = YLy + XUy;
    c01[0] = YUx - XUx;   c01[1] = YUy - XUy;
    // volume part: |T| n_in / (3 V) * grad N
    const double vl = area * (double)nl * (1.0 / 3.0) * inv_volume;
    const double vu = area * (double)nu * (1.0 / 3.0) * inv_volume;
    c00[2] = -vl * inv_hx;  c00[3] = -vu * inv_hy;
    c10[2] = vl * inv_hx;   c10[3] = -vl * inv_hy;
    c11[2] = vu * inv_hx;   c11[3] = vl * inv_hy;
    c01[2] = -vu * inv_hx;  c01[3] = vu * inv_hy;
    if (count) {
      part[0] += wl * dl + wu * du;
      part[1] += area * (double)(nl + nu) * (1.0 / 3.0);
    }
  }
};

// Thermal compliance + shape derivative for KB heat terms at once
// (models/heat.py:124-166): per term t with weight c_t, state u_t, source
// samples f_q (and optionally grad f_q) at the three edge-midpoint points,
//   J   += c_t int A |grad u|^2,
//   S1_q = c_t ((2 u_q f_q - A_q |grad u|^2) I + 2 A_q grad u (x) grad u),
//   S0_q = c_t 2 u_q grad f_q,
// contracted with the test functions: vec_a += sum_q (|T|/3) (S0_q N_a(x_q)
// + S1_q grad N_a).  grad u is constant per triangle, so only sum_q A_q =
// 3 abar enters the S1 term.  in = KB temperature fields; out =
// (vec_cost[2], vec_vol[2]) as for Shape.
template <int KB>
struct HeatShape {
  static constexpr int NC = 1, NIN = KB, NOUT = 4;
  int nx;
  double area, inv_hx, inv_hy, inv_volume;
  double w0, w1;        // |T| abar(n_in) = w0 + w1 n_in
  double cw[KB];        // term weights
  const double *fq;     // (KB, E, 3) source samples
  const double *gq;     // (KB, E, 3, 2) source gradients, or null
  int64_t ecount;       // number of triangles E (stride of one term in fq / gq)
  __device__ __forceinline__ int64_t estride() const { return ecount; }

  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 4) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t) { return 0u; }

  __device__ __forceinline__ void cell(const double *u00, const double *u10, const double *u01,
                                       const double *u11, uint32_t word, bool count, int i, int j,
                                       double *c00, double *c10, double *c01, double *c11,
                                       double *part) const {
    const bool ok = valid(word);
    const uint32_t nl = ok ? (word & 3u) : 0u, nu = ok ? ((word >> 2) & 3u) : 0u;
    const double wl = ok ? fma((double)nl, w1, w0) : 0.0, wu = ok ? fma((double)nu, w1, w0) : 0.0;
    const double qw = ok ? area * (1.0 / 3.0) : 0.0;  // quadrature weight (0 off the grid)
    // element indices (fem order: lower 2c, upper 2c+1); clamp halo cells to a valid index
    const int64_t cidx = ok ? ((int64_t)j * nx + i) : 0;
    const int64_t el = 2 * cidx, eu = el + 1;
    double Mxx = 0.0, Mxy = 0.0, Myy = 0.0, Nxx = 0.0, Nxy = 0.0, Nyy = 0.0, dens = 0.0;
    // S0 vertex sums: lower (00, 10, 11), upper (00, 11, 01)
    double sL[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    double sU[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const double c = cw[k];
      const double *f = fq + (size_t)k * (size_t)estride() * 3;
      // lower: grad u = ((u10 - u00)/hx, (u11 - u10)/hy)
      {
        const double gx = (u10[k] - u00[k]) * inv_hx, gy = (u11[k] - u10[k]) * inv_hy;
        const double q0 = 0.5 * (u00[k] + u10[k]), q1 = 0.5 * (u10[k] + u11[k]),
                     q2 = 0.5 * (u00[k] + u11[k]);
        const double uf = q0 * f[el * 3] + q1 * f[el * 3 + 1] + q2 * f[el * 3 + 2];
        const double g2 = gx * gx + gy * gy;
        const double diag = 2.0 * qw * uf - wl * g2;
        Mxx += c * (diag + 2.0 * wl * gx * gx);
        Myy += c * (diag + 2.0 * wl * gy * gy);
        Mxy += c * (2.0 * wl * gx * gy);
        dens += c * wl * g2;
        if (gq) {
          const double *G = gq + (size_t)k * (size_t)estride() * 6 + el * 6;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const double t0 = c * qw * q0 * G[d], t1 = c * qw * q1 * G[2 + d], t2 = c * qw * q2 * G[4 + d];
            sL[0][d] += t0 + t2;  // vertex A in edges (A,B), (A,C)
            sL[1][d] += t0 + t1;  // vertex B in (A,B), (B,C)
            sL[2][d] += t1 + t2;  // vertex C in (B,C), (A,C)
          }
        }
      }
      // upper (A, B, C) = (00, 11, 01): grad u = ((u11 - u01)/hx, (u01 - u00)/hy)
      {
        const double gx = (u11[k] - u01[k]) * inv_hx, gy = (u01[k] - u00[k]) * inv_hy;
        const double q0 = 0.5 * (u00[k] + u11[k]), q1 = 0.5 * (u11[k] + u01[k]),
                     q2 = 0.5 * (u00[k] + u01[k]);
        const double uf = q0 * f[eu * 3] + q1 * f[eu * 3 + 1] + q2 * f[eu * 3 + 2];
        const double g2 = gx * gx + gy * gy;
        const double diag = 2.0 * qw * uf - wu * g2;
        Nxx += c * (diag + 2.0 * wu * gx * gx);
        Nyy += c * (diag + 2.0 * wu * gy * gy);
        Nxy += c * (2.0 * wu * gx * gy);
        dens += c * wu * g2;
        if (gq) {
          const double *G = gq + (size_t)k * (size_t)estride() * 6 + eu * 6;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const double t0 = c * qw * q0 * G[d], t1 = c * qw * q1 * G[2 + d], t2 = c * qw * q2 * G[4 + d];
            sU[0][d] += t0 + t2;
            sU[1][d] += t0 + t1;
            sU[2][d] += t1 + t2;
          }
        }
      }
    }
    // S1 sums against grad N: lower (-1/hx, 0), (1/hx, -1/hy), (0, 1/hy);
    // upper (0, -1/hy), (1/hx, 0), (-1/hx, 1/hy)
    const double ax = inv_hx, ay = inv_hy;
    c00[0] = -Mxx * ax + (-Nxy * ay) + sL[0][0] + sU[0][0];
    c00[1] = -Mxy * ax + (-Nyy * ay) + sL[0][1] + sU[0][1];
    c10[0] = Mxx * ax - Mxy * ay + sL[1][0];
    c10[1] = Mxy * ax - Myy * ay + sL[1][1];
    c11[0] = Mxy * ay + Nxx * ax + sL[2][0] + sU[1][0];
    c11[1] = Myy * ay + Nxy * ax + sL[2][1] + sU[1][1];
    c01[0] = -Nxx * ax + Nxy * ay + sU[2][0];
    c01[1] = -Nxy * ax + Nyy * ay + sU[2][1];
    // volume part: |T| n_in / (3 V) * grad N (as Shape)
    const double vl = area * (double)nl * (1.0 / 3.0) * inv_volume;
    const double vu = area * (double)nu * (1.0 / 3.0) * inv_volume;
    c00[2] = -vl * inv_hx;  c00[3] = -vu * inv_hy;
    c10[2] = vl * inv_hx;   c10[3] = -vl * inv_hy;
    c11[2] = vu * inv_hx;   c11[3] = vl * inv_hy;
    c01[2] = -vu * inv_hx;  c01[3] = vu * inv_hy;
    if (count) {
      part[0] += dens;
      part[1] += area * (double)(nl + nu) * (1.0 / 3.0);
    }
  }
};

template <class PH, int ACT>
struct Traits {
  static constexpr int NP = (ACT == RESID) ? 3 : (ACT == PCG) ? 5 : (ACT == STATS) ? 3
                                                                     : (ACT == SHAPE) ? 2 : 0;
  static constexpr unsigned MAXMASK = (ACT == STATS) ? 4u : 0u;
};

template <class PH>
__device__ __forceinline__ void node_diag(const PH &ph, uint32_t w00, uint32_t wm0, uint32_t w0m,
                                          uint32_t wmm, int i, int j, double *d);
template <>
__device__ __forceinline__ void node_diag<Elast>(const Elast &ph, uint32_t w00, uint32_t wm0,
                                                 uint32_t w0m, uint32_t wmm, int, int, double *d) {
  ph.diag(w00, wm0, w0m, wmm, d);
}
template <>
__device__ __forceinline__ void node_diag<Lap>(const Lap &ph, uint32_t w00, uint32_t wm0,
                                               uint32_t w0m, uint32_t wmm, int, int, double *d) {
  ph.diag(w00, wm0, w0m, wmm, d);
}
template <>
__device__ __forceinline__ void node_diag<H1>(const H1 &ph, uint32_t w00, uint32_t wm0,
                                              uint32_t w0m, uint32_t wmm, int i, int j, double *d) {
  ph.diag(w00, wm0, w0m, wmm, i, j, d);
}

// End of single-pass PCG iteration i for one right-hand side, from the five
// sums of the pass: tot = {p.q, z.q, q.M^-1 q, r.z, r.r} of p_i, q_i = A p_i,
// z_i = M^-1 r_i and the explicit residual r_i = r_{i-1} - alpha_{i-1} q_{i-1}.
// scipy cg's stopping rule on ||r_i|| (x already holds x_i: the pass folded
// x += alpha_{i-1} p_{i-1} in), else alpha_i = r_i.z_i / p_i.q_i and
//   rz_{i+1} = rz_i - 2 alpha_i z_i.q_i + alpha_i^2 q_i.M^-1 q_i,
// the exact expansion of (r_i - alpha q_i).M^-1(r_i - alpha q_i), so that
// beta_{i+1} = rz_{i+1} / rz_i is known before the pass that forms r_{i+1}
// (one reduction per iteration: D'Azevedo, Eijkhout & Romine's reduced-
// synchronisation CG).  rz itself is recomputed exactly every pass.
__device__ __forceinline__ void pcg_decide(lsg_pcg_scalars &s, const double *tot) {
  const double pq = tot[0], zq = tot[1], qdq = tot[2], rz = tot[3], rr = tot[4];
  s.rr = rr;
  s.pq = pq;
  if (s.first == 0.0) {
    s.iters += 1.0;
    if (sqrt(rr) < s.atol) {
      s.done = 1.0;
      return;
    }
    if (s.iters >= s.maxiter || !isfinite(rr) || !isfinite(rz)) {
      s.done = 2.0;
      return;
    }
  }
  const double alpha = rz / pq;
  const double rz_next = fma(alpha * alpha, qdq, fma(-2.0 * alpha, zq, rz));
  if (!isfinite(alpha) || !isfinite(rz_next)) {  // breakdown: report, do not spin
    s.done = 2.0;
    return;
  }
  s.rho = rz;
  s.alpha = alpha;
  s.beta = rz_next / rz;
  s.rz_new = rz_next;
  s.first = 0.0;
}

template <int ACT>
__device__ __forceinline__ void finalize(const MArgs &a, int rhs, const double *tot) {
  if constexpr (ACT == RESID) {
    lsg_pcg_scalars &s = a.scal[rhs];
    s.bb = tot[0];
    s.rr = tot[1];
    s.rho = tot[2];
    const double bn = sqrt(tot[0]);
    s.atol = fmax(s.atol, s.reserved[0] * bn);
    s.beta = 0.0;
    s.first = 1.0;
    if (tot[0] == 0.0) {
      s.zero_rhs = 1.0;
      s.done = 1.0;
    } else if (sqrt(tot[1]) < s.atol) {
      s.done = 1.0;
    }
  } else if constexpr (ACT == PCG) {
    pcg_decide(a.scal[rhs], tot);
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

// ----------------------------------------------------------------------------
// The marching skeleton.  PH = Elast | H1 (operators) or Shape<KB>.
//
// Loop structure: two node-row register sets (SA, SB) and two accumulator
// sets alternate roles, the loop is unrolled by two so no state is copied
// between rows, and the global loads of row r+2 are issued while row r+1 is
// processed.  Loads are branch-free: columns outside the grid load a clamped
// (valid) address and get material word 0, so their cells contribute nothing.
// ----------------------------------------------------------------------------
// One marching task (strip group bx, row segment by, right-hand side rhs):
// the body shared by the per-launch kernel below and the persistent PCG.
// Adds this thread's reduction terms to part[].
template <class PH, int ACT, class W>
__device__ __forceinline__ void march_core(const PH &ph, const Geo &g, const MArgs &a, int bx,
                                           int by, int rhs,
                                           double (&part)[Traits<PH, ACT>::NP > 0 ? Traits<PH, ACT>::NP : 1]) {
  constexpr int NC = PH::NC;  // components per node of each input field
  constexpr int NIN = PH::NIN, NOUT = PH::NOUT;
  constexpr int NF = (ACT == SHAPE) ? NIN / NC : 1;  // fields read per node (SHAPE: states)
  constexpr bool HAS_DINV = (ACT == RESID);
  static_assert(ACT != PCG, "the PCG pass is march_pcg");

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = bx * kWarps + warp;
  const W *words = static_cast<const W *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);

  const int i = strip * kStrip - 1 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool own = node_ok && lane >= 1 && lane <= kStrip;
  const int ic = min(max(i, 0), nx);  // clamped column: always a valid address
  const int J0 = by * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const size_t voff = (ACT == SHAPE) ? 0 : (size_t)rhs * (size_t)nn * NC;
  const double *xin = a.x + voff + (size_t)ic * NC;
  const double *dvin = (HAS_DINV ? a.dinv : a.x) + (size_t)ic * NC;
  const W *win = words + ic;

  struct Raw {
    double v[NF][NC];
    double dv[NC];
    uint32_t wc;
  };
  struct Row {
    double in[NIN], rt[NIN], raw[NC], dg[NC];
    uint32_t wc;
  };

  auto fetch = [&](int r, Raw &f) {
    const int64_t off = (int64_t)r * nxp;
    f.wc = node_ok ? (uint32_t)__ldg(win + off) : 0u;
    if constexpr (ACT == SHAPE) {
#pragma unroll
      for (int k = 0; k < NF; ++k) ldg_node<NC>(xin + (size_t)k * nn * NC, off, f.v[k]);
    } else {
      ldg_node<NC>(xin, off, f.v[0]);
      if constexpr (HAS_DINV) ldg_node<NC>(dvin, off, f.dv);
    }
  };

  // Operator input of node row r (masked) + raw value + inverse diagonal.
  auto prepare = [&](int r, const Raw &f, Row &S) {
    S.wc = f.wc;
    if constexpr (ACT == SHAPE) {
#pragma unroll
      for (int k = 0; k < NF; ++k)
#pragma unroll
        for (int c = 0; c < NC; ++c) S.in[k * NC + c] = f.v[k][c];
    } else {
      const uint32_t m = PH::mask(f.wc);
      double v[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) v[c] = f.v[0][c];
      if constexpr (HAS_DINV) {
#pragma unroll
        for (int c = 0; c < NC; ++c) S.dg[c] = f.dv[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        S.raw[c] = v[c];
        S.in[c] = ((m >> c) & 1u) ? 0.0 : v[c];
      }
    }
#pragma unroll
    for (int t = 0; t < NIN; ++t) S.rt[t] = __shfl_down_sync(0xffffffffu, S.in[t], 1);
  };

  auto emit = [&](int r, const Row &S, const double *accv) {
    const int64_t node = (int64_t)r * nxp + i;
    if constexpr (ACT == SHAPE) {  // outputs are velocity-space (2-component) vectors
      double2 *vc = reinterpret_cast<double2 *>(a.y);
      double2 o = make_double2(accv[0], accv[1]);
      if (a.accumulate) {
        const double2 old = vc[node];
        o.x += old.x;
        o.y += old.y;
      } else {
        reinterpret_cast<double2 *>(a.y2)[node] = make_double2(accv[2], accv[3]);
      }
      vc[node] = o;
    } else {
      const uint32_t m = PH::mask(S.wc);
      double yv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) yv[c] = ((m >> c) & 1u) ? S.raw[c] : accv[c];
      if constexpr (ACT == APPLY) {
        st_node<NC>(a.y + voff, node, yv);
      } else if constexpr (ACT == RESID) {
        double bv[NC], rv[NC];
        ldg_node<NC>(a.b + voff, node, bv);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          rv[c] = bv[c] - yv[c];
          part[0] += bv[c] * bv[c];
          part[1] += rv[c] * rv[c];
          part[2] += rv[c] * (rv[c] * S.dg[c]);
        }
        st_node<NC>(a.y + voff, node, rv);
      } else if constexpr (ACT == STATS) {
        double vv[NC];
        ldg_node<NC>(a.x2, node, vv);
        double sp = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          part[0] += S.raw[c] * yv[c];
          part[1] += vv[c] * S.raw[c];
          sp += fabs(S.raw[c]) / (c == 0 ? g.hx : g.hy);
        }
        part[2] = fmax(part[2], sp);
      }
    }
  };

  // One row step: new row r (register set Sn, from raw f) closes cell row
  // r-1 against the previous row Sp; emits row r-1 (accumulator ap) and
  // starts the accumulation of row r (an).
  auto step = [&](int r, const Raw &f, const Row &Sp, Row &Sn, double *ap, double *an) {
    prepare(r, f, Sn);
    double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
    if constexpr (ACT == SHAPE) {
      ph.cell(Sp.in, Sp.rt, Sn.in, Sn.rt, Sp.wc, own && (r - 1) >= J0, i, r - 1, c00, c10, c01,
              c11, part);
    } else {
      ph.cell(Sp.in, Sp.rt, Sn.in, Sn.rt, Sp.wc, i, r - 1, c00, c10, c01, c11);
    }
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);
      double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
      if (lane == 0) up10 = up11 = 0.0;
      ap[t] += c00[t] + up10;
      an[t] = c01[t] + up11;
    }
    if (own && (r - 1) >= J0) emit(r - 1, Sp, ap);
  };

  const int jstart = max(J0 - 1, 0);
  const int rend = min(J1, ny);
  Row SA, SB;
  double accA[NOUT], accB[NOUT];
  // two rows in flight (deeper prefetch rings measured slower for the apply:
  // cfg2 / cfg4 with L2 flushed, 2 rows 24.6 / 69.5 us, 4 rows 22.7 / 73.7,
  // 6 rows 24.6 / 80.9, 8 rows 26.7 / 96.3 -- registers 66 -> 80+, fewer CTAs)
  Raw fA, fB;
  {
    Raw f0;
    fetch(jstart, f0);
    fetch(min(jstart + 1, rend), fA);
    fetch(min(jstart + 2, rend), fB);
    prepare(jstart, f0, SA);
  }
#pragma unroll
  for (int t = 0; t < NOUT; ++t) accA[t] = 0.0;

  bool last_in_b = false;  // which register set holds row rend after the loop
  int r = jstart + 1;
  while (r <= rend) {
    step(r, fA, SA, SB, accA, accB);
    fetch(min(r + 2, rend), fA);
    if (++r > rend) { last_in_b = true; break; }
    step(r, fB, SB, SA, accB, accA);
    fetch(min(r + 2, rend), fB);
    ++r;
  }
  if (J1 == ny + 1 && own && ny >= J0) {
    if (last_in_b) emit(ny, SB, accB);
    else emit(ny, SA, accA);
  }
}

// ----------------------------------------------------------------------------
// Single-pass PCG iteration task (strip group bx, row segment by, rhs): the
// marching skeleton above specialised for the PCG pass,
//   r_i = r_{i-1} - alpha_{i-1} q_{i-1}, z = M^-1 r_i, p_i = z + beta_i p_{i-1}
// on every node the task touches (halo nodes recompute their neighbours'
// values bit for bit); owned nodes store r_i, p_i, q_i = A p_i and
// x += alpha_{i-1} p_{i-1}, and sum p.q, z.q, q.M^-1 q, r.z, r.r.
// The five inputs per node (r_{i-1}, p_{i-1}, q_{i-1}, M^-1 and, on owned
// nodes, x) are prefetched into a register ring kPcgDepth rows deep: the
// loads of rows r+1 and r+2 are in flight while row r is computed.  (A
// shared-memory ring fed by per-thread cp.async, which frees those registers,
// measured slower: 55.4 vs 55.9 us at cfg2 but 234 vs 210 us at cfg4.)
// COH: the inputs were written earlier in the same launch (the persistent
// kernel, across grid barriers): coherent loads instead of the read-only path.
// ----------------------------------------------------------------------------
constexpr int kPcgDepth = 3;   // node rows in the register ring
constexpr int kPcgFields = 5;  // r, p, q, M^-1, x

template <class PH, bool COH = false>
__device__ __forceinline__ void march_pcg(const PH &ph, const Geo &g, const MArgs &a, int bx,
                                          int by, int rhs, bool first, double beta,
                                          double alpha_prev, double (&part)[5],
                                          int warp_in_task = -1) {
  constexpr int NC = PH::NC, NOUT = PH::NOUT, D = kPcgDepth;
  static_assert(PH::NIN == NC, "PCG operators read one field");
  const int lane = threadIdx.x & 31;
  const int warp = warp_in_task >= 0 ? warp_in_task : (int)(threadIdx.x >> 5);
  const int strip = bx * kWarps + warp;
  const uint8_t *words = static_cast<const uint8_t *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);
  const int i = strip * kStrip - 1 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool own = node_ok && lane >= 1 && lane <= kStrip;
  const int ic = min(max(i, 0), nx);  // clamped column: always a valid address
  const int J0 = by * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const size_t voff = (size_t)rhs * (size_t)nn * NC;
  const double *r_in = a.x + voff, *p_in = a.x2 + voff, *q_in = a.x3 + voff;

  struct Row {
    double in[NC], rt[NC], raw[NC], dg[NC], z[NC];
    uint32_t wc;
  };
  uint32_t wring[D];
  double ring[D][kPcgFields][NC];
  auto ldn = [&](const double *src, int64_t node, double *v) {
    if constexpr (COH) ld_node<NC>(src, node, v);  // written earlier in this launch
    else ldg_node<NC>(src, node, v);
  };

  auto fetch = [&](int r, int s) {
    const int64_t node = (int64_t)r * nxp + ic;
    wring[s] = node_ok ? (uint32_t)__ldg(words + node) : 0u;
    ldn(r_in, node, ring[s][0]);
    if (!first) {
      ldn(p_in, node, ring[s][1]);
      ldn(q_in, node, ring[s][2]);
    }
    ldg_node<NC>(a.dinv, node, ring[s][3]);
    if (!first && own && r >= J0 && r < J1) ld_node<NC>(a.xs + voff, node, ring[s][4]);
  };

  auto prepare = [&](int r, int s, Row &S) {
    S.wc = wring[s];
    const uint32_t m = PH::mask(S.wc);
    double R[NC], P[NC], Q[NC], v[NC], rv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      R[c] = ring[s][0][c];
      S.dg[c] = ring[s][3][c];
      P[c] = ring[s][1][c];
      Q[c] = ring[s][2][c];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      rv[c] = first ? R[c] : fma(-alpha_prev, Q[c], R[c]);
      S.z[c] = rv[c] * S.dg[c];  // M^-1 = diag(1/D) (fem.py:303-305)
      v[c] = first ? S.z[c] : fma(beta, P[c], S.z[c]);
    }
    if (own && r >= J0 && r < J1) {
      const int64_t node = (int64_t)r * nxp + i;
      st_node<NC>(a.y3 + voff, node, rv);
      st_node<NC>(a.y2 + voff, node, v);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        part[3] += rv[c] * S.z[c];
        part[4] += rv[c] * rv[c];
      }
      if (!first) {  // x_i = x_{i-1} + alpha_{i-1} p_{i-1}
        double X[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) X[c] = fma(alpha_prev, P[c], ring[s][4][c]);
        st_node<NC>(a.xs + voff, node, X);
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      S.raw[c] = v[c];
      S.in[c] = ((m >> c) & 1u) ? 0.0 : v[c];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) S.rt[c] = __shfl_down_sync(0xffffffffu, S.in[c], 1);
  };

  auto emit = [&](int r, const Row &S, const double *accv) {
    const int64_t node = (int64_t)r * nxp + i;
    const uint32_t m = PH::mask(S.wc);
    double yv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) yv[c] = ((m >> c) & 1u) ? S.raw[c] : accv[c];
    st_node<NC>(a.y + voff, node, yv);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      part[0] += S.raw[c] * yv[c];
      part[1] += S.z[c] * yv[c];
      part[2] += yv[c] * (yv[c] * S.dg[c]);
    }
  };

  auto step = [&](int r, int s, const Row &Sp, Row &Sn, double *ap, double *an) {
    prepare(r, s, Sn);
    double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
    ph.cell(Sp.in, Sp.rt, Sn.in, Sn.rt, Sp.wc, i, r - 1, c00, c10, c01, c11);
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);
      double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
      if (lane == 0) up10 = up11 = 0.0;
      ap[t] += c00[t] + up10;
      an[t] = c01[t] + up11;
    }
    if (own && (r - 1) >= J0) emit(r - 1, Sp, ap);
  };

  const int jstart = max(J0 - 1, 0);
  const int rend = min(J1, ny);
  Row SA, SB;
  double accA[NOUT], accB[NOUT];
#pragma unroll
  for (int s = 0; s < D; ++s) fetch(min(jstart + s, rend), s);
  prepare(jstart, 0, SA);
  fetch(min(jstart + D, rend), 0);
#pragma unroll
  for (int t = 0; t < NOUT; ++t) accA[t] = 0.0;
  bool last_in_b = false;  // which register set holds row rend after the loop
  int r = jstart + 1;      // row r lives in ring slot (r - jstart) % D
  constexpr int U = (D % 2 == 0) ? D : 2 * D;  // ring slot and register-set parity both repeat
  while (r <= rend) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (r <= rend) {
        const int s = (u + 1) % D;
        if (u % 2 == 0) step(r, s, SA, SB, accA, accB);
        else step(r, s, SB, SA, accB, accA);
        last_in_b = (u % 2 == 0);
        fetch(min(r + D, rend), s);
        ++r;
      }
    }
  }
  if (J1 == ny + 1 && own && ny >= J0) {
    if (last_in_b) emit(ny, SB, accB);
    else emit(ny, SA, accA);
  }
}

// ----------------------------------------------------------------------------
// Single-pass PCG iteration without a stored q ("recompute" pass, 2D).
//
// Same iteration as march_pcg (same five sums, same decisions), but q_{i-1}
// is not read back from memory: the pass re-applies the operator to p_{i-1},
// which it reads anyway to form p_i, so per right-hand side and iteration it
// moves 6 vectors (reads r, p, x; writes r, p, x) instead of 8.  The extra
// stencil costs ~45 fp64 instructions per cell.  q_{i-1} at a node is summed
// by the same code in the same order wherever it is recomputed (owner or halo
// warp), so every warp forms the same r_i, z_i, p_i of a node.
//
// Two stencils run one row apart: at step r the old stencil closes
// q_{i-1} of row r-1, that row's r_i / z_i / p_i are formed (and r_i, p_i,
// x_i stored on owned nodes), and the new stencil closes q_i of row r-2,
// whose sums p.q, z.q, q.M^-1 q are taken.  Halo: two columns each side (a
// warp owns lanes 2..29: kStripRq columns) and two rows below each segment.
//
// Iteration 0 needs no special case: pcg_start zeroes the p_{-1} buffer and
// alpha_{-1} = beta_0 = 0, so r_0 - 0 q, 0 p + z and x + 0 p are exact.
//
// Prefetch ring in shared memory: every lane copies its own node of each
// source row (p_{i-1}, r_{i-1}, M^-1, x; 16-byte cp.async; word: the aligned
// 4-byte chunk that holds it) A rows ahead and reads back only what it copied
// itself, so per-thread cp.async.wait_group orders the ring (no barriers).
// Against register rings this frees ~48 registers (4 instead of 3 CTAs/SM).
// A = 3 measured best on small batched grids (cfg2: 51.6 vs 52.5 us), A = 2
// on large ones (cfg4: 183 vs 198 us).  (Also measured and removed: the register ring,
// 52.9 / 185 us; a software-pipelined variant whose two stencils overlap as
// independent chains with all row state in the ring, 57.3 / 204 us; keeping
// the masked inputs in registers, 79 / 254 us; two right-hand sides per warp
// sharing words, weights, masks and M^-1 (168 registers, 3 CTAs/SM), 54.7 vs
// 49.5 us on the same box; strength-reduced ring/row addressing, no change; a
// per-CTA shared table of w(n) k_j instead of the weight arithmetic, 66.0 vs
// 51.6 us -- lane-divergent table reads on the critical path; branch-free
// masked sums with predicated stores and two steps per basic block, 53.7 vs
// 51.6 us; steps skewed by one row so that the two stencils are independent
// chains (three rows of p_i in registers, 126 registers), 53.2 vs 51.2 us.)
// ----------------------------------------------------------------------------
constexpr int kStripRq = 28;

template <int NC, int A>
struct RqRing {
  static constexpr int FS = 32 * NC;            // doubles per field per slot
  static constexpr int SLOT = 4 * FS + 16;      // p, r, M^-1, x + 32 words
  static constexpr int D = A + 1;               // slots
  static constexpr int WARP = D * SLOT;         // doubles per warp
};

template <int N>
__device__ __forceinline__ void cp_async_wait_all_but() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <class PH, int A, bool FIRST>
__device__ __forceinline__ void march_pcg_rqs(const PH &ph, const Geo &g, const MArgs &a, int bx,
                                              int by, int rhs, double beta, double alpha_prev,
                                              double (&part)[5], double *ring) {
  constexpr int NC = PH::NC, NOUT = PH::NOUT;
  using RG = RqRing<NC, A>;
  constexpr int D = RG::D, FS = RG::FS;
  static_assert(PH::NIN == NC, "PCG operators read one field");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = bx * kWarps + warp;
  const uint8_t *words = static_cast<const uint8_t *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);
  const int i = strip * kStripRq - 2 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool own = node_ok && lane >= 2 && lane <= kStripRq + 1;
  const int ic = min(max(i, 0), nx);
  const int J0 = by * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const size_t voff = (size_t)rhs * (size_t)nn * NC;
  const double *r_in = a.x + voff, *p_in = a.x2 + voff;
  double *xs = a.xs + voff;
  double *myring = ring + (size_t)warp * RG::WARP;

  struct Old {
    double raw[NC];
    uint32_t wc;
  };
  struct New {
    double raw[NC], z[NC], dg[NC];
    uint32_t wc;
  };

  auto cpy = [&](double *dst, const double *src) {
    if constexpr (NC == 2) cp_async16(dst, src);
    else cp_async8(dst, src);
  };
  // FIRST: r_{i-1} and p_{i-1} are dead once this pass has read them; when the new
  // r_i, p_i of the whole batch fit in L2 beside them (and the six vectors do not),
  // copying them with an evict-first policy leaves L2 to the vectors the next pass
  // reads (cfg2: 49.9 -> 46.9 us).  It loses on larger systems (cfg4: 176 -> 196 us), so
  // the launcher decides (launch_pcg_rq).
  uint64_t pol_first = 0;
  if constexpr (FIRST) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
  auto cpy_dead = [&](double *dst, const double *src) {
    if constexpr (FIRST) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      if constexpr (NC == 2)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src),
                     "l"(pol_first));
      else
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src),
                     "l"(pol_first));
    } else {
      cpy(dst, src);
    }
  };
  // issue the copies of row r into slot sl (one commit group per row)
  auto fetch = [&](int r, int sl) {
    double *S = myring + sl * RG::SLOT;
    const int64_t node = (int64_t)r * nxp + ic;
    cpy_dead(S + 0 * FS + lane * NC, p_in + node * NC);
    cpy_dead(S + 1 * FS + lane * NC, r_in + node * NC);
    cpy(S + 2 * FS + lane * NC, a.dinv + node * NC);
    if (own && r >= J0 && r < J1) cpy(S + 3 * FS + lane * NC, xs + node * NC);
    uint32_t *W = reinterpret_cast<uint32_t *>(S + 4 * FS);
    const int64_t wq = node & ~(int64_t)3;
    if (wq + 4 <= nn) cp_async4(W + lane, words + wq);
    else W[lane] = (uint32_t)words[node] << (8 * (node & 3));  // the grid's last 1-3 nodes
    cp_async_commit();
  };
  auto ld = [&](int sl, int f, double *v) {
    const double *S = myring + sl * RG::SLOT + f * FS + lane * NC;
    if constexpr (NC == 2) {
      const double2 t = *reinterpret_cast<const double2 *>(S);
      v[0] = t.x;
      v[1] = t.y;
    } else {
      v[0] = S[0];
    }
  };
  auto word = [&](int r, int sl) -> uint32_t {
    const uint32_t w4 = reinterpret_cast<const uint32_t *>(myring + sl * RG::SLOT + 4 * FS)[lane];
    const int64_t node = (int64_t)r * nxp + ic;
    return node_ok ? (w4 >> (8 * (uint32_t)(node & 3))) & 0xffu : 0u;
  };
  auto prep_old = [&](int r, int sl, Old &O) {
    O.wc = word(r, sl);
    ld(sl, 0, O.raw);
  };
  auto derive = [&](const double *raw, uint32_t wc, double *in, double *rt) {
    const uint32_t m = PH::mask(wc);
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = ((m >> c) & 1u) ? 0.0 : raw[c];
#pragma unroll
    for (int c = 0; c < NC; ++c) rt[c] = __shfl_down_sync(0xffffffffu, in[c], 1);
  };
  auto cells = [&](int rlow, const auto &P, const auto &Nr, double *ap, double *an) {
    double inP[NC], rtP[NC], inN[NC], rtN[NC];
    derive(P.raw, P.wc, inP, rtP);
    derive(Nr.raw, Nr.wc, inN, rtN);
    double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
    ph.cell(inP, rtP, inN, rtN, P.wc, i, rlow, c00, c10, c01, c11);
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      const double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);  // lane 0: halo, unused
      const double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
      ap[t] += c00[t] + up10;
      an[t] = c01[t] + up11;
    }
  };
  auto form = [&](int r, int sl, const Old &O, const double *accq, New &Nw) {
    const uint32_t m = PH::mask(O.wc);
    double R[NC], rv[NC], v[NC];
    ld(sl, 1, R);
    ld(sl, 2, Nw.dg);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double q = ((m >> c) & 1u) ? O.raw[c] : accq[c];
      rv[c] = fma(-alpha_prev, q, R[c]);
      Nw.z[c] = rv[c] * Nw.dg[c];
      v[c] = fma(beta, O.raw[c], Nw.z[c]);
    }
    if (own && r >= J0 && r < J1) {
      const int64_t node = (int64_t)r * nxp + i;
      st_node<NC>(a.y3 + voff, node, rv);
      st_node<NC>(a.y2 + voff, node, v);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        part[3] += rv[c] * Nw.z[c];
        part[4] += rv[c] * rv[c];
      }
      double X[NC];
      ld(sl, 3, X);
#pragma unroll
      for (int c = 0; c < NC; ++c) X[c] = fma(alpha_prev, O.raw[c], X[c]);
      st_node<NC>(xs, node, X);
    }
    Nw.wc = O.wc;
#pragma unroll
    for (int c = 0; c < NC; ++c) Nw.raw[c] = v[c];
  };
  auto emit = [&](int r, const New &Nw, const double *accv) {
    if (!(own && r >= J0 && r < J1)) return;
    const uint32_t m = PH::mask(Nw.wc);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double yv = ((m >> c) & 1u) ? Nw.raw[c] : accv[c];
      part[0] += Nw.raw[c] * yv;
      part[1] += Nw.z[c] * yv;
      part[2] += yv * (yv * Nw.dg[c]);
    }
  };

  const int jstart = max(J0 - 2, 0);
  const int rend = min(J1 + 1, ny);
  auto nxt = [](int s) { return s + 1 == D ? 0 : s + 1; };
  // rows jstart .. jstart + A in slots 0 .. A (= D - 1)
#pragma unroll
  for (int s = 0; s < D; ++s) fetch(min(jstart + s, rend), s);
  Old OA, OB;
  New NA, NB;
  double aoA[NOUT], aoB[NOUT], anA[NOUT], anB[NOUT];
  cp_async_wait_all_but<D - 1>();  // row jstart
  prep_old(jstart, 0, OA);
#pragma unroll
  for (int t = 0; t < NOUT; ++t) aoA[t] = 0.0;

  // step r: slot sp holds row r, sf = the slot before it holds row r-1
  auto step = [&](int r, int sp, int sf, bool newcells, Old &Op, Old &On, double *aop, double *aon,
                  New &Np, New &Nn, double *anp, double *ann) {
    cp_async_wait_all_but<A - 1>();  // row r has landed (rows up to r + A - 1 issued)
    prep_old(r, sp, On);
    cells(r - 1, Op, On, aop, aon);
    form(r - 1, sf, Op, aop, Nn);
    if (newcells) {
      cells(r - 2, Np, Nn, anp, ann);
      emit(r - 2, Np, anp);
    } else {
#pragma unroll
      for (int t = 0; t < NOUT; ++t) ann[t] = 0.0;
    }
    fetch(min(r + A, rend), sf);  // row r-1's slot is free again
  };

  bool last_in_b = false;
  int r = jstart + 1;
  int sf = 0, sp = 1;
  if (r <= rend) {
    step(r, sp, sf, false, OA, OB, aoA, aoB, NB, NA, anB, anA);
    last_in_b = true;
    sf = sp;
    sp = nxt(sp);
    ++r;
  }
  while (r <= rend) {
    step(r, sp, sf, true, OB, OA, aoB, aoA, NA, NB, anA, anB);
    last_in_b = false;
    sf = sp;
    sp = nxt(sp);
    if (++r > rend) break;
    step(r, sp, sf, true, OA, OB, aoA, aoB, NB, NA, anB, anA);
    last_in_b = true;
    sf = sp;
    sp = nxt(sp);
    ++r;
  }
  cp_async_wait_all_but<0>();
  if (rend == ny && jstart < ny) {  // sf now holds row ny
    if (last_in_b) {
      form(ny, sf, OB, aoB, NB);
      cells(ny - 1, NA, NB, anA, anB);
      emit(ny - 1, NA, anA);
      emit(ny, NB, anB);
    } else {
      form(ny, sf, OA, aoA, NA);
      cells(ny - 1, NB, NA, anB, anA);
      emit(ny - 1, NB, anB);
      emit(ny, NA, anA);
    }
  }
}

// No minimum-blocks bound: ptxas settles at 122 registers (4 CTAs/SM).  Measured
// against it: a minBlocks of 1 (176 registers, 2 CTAs/SM) 9-13% slower, 5
// (96 registers, small spills) 3-8% slower, 6 (80 registers) 30% slower.
template <class PH, int A, bool FIRST>
__global__ void __launch_bounds__(kThreads) march_pcg_rqs_kernel(PH ph, Geo g, MArgs a) {
  constexpr int NP = 5;
  __shared__ double scratch[NP * kWarps];
  __shared__ __align__(16) double ring[kWarps * RqRing<PH::NC, A>::WARP];
  pdl_wait();  // launched with launch_pdl: the previous iteration's pass must be done
  const int rhs = blockIdx.z;
  const lsg_pcg_scalars &s = a.scal[rhs];
  if (s.done != 0.0) return;
  double part[NP];
#pragma unroll
  for (int t = 0; t < NP; ++t) part[t] = 0.0;
  march_pcg_rqs<PH, A, FIRST>(ph, g, a, blockIdx.x, blockIdx.y, rhs, s.beta, s.alpha, part, ring);
  const int nblk = gridDim.x * gridDim.y;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  double tot[NP];
  const size_t pbase = (size_t)rhs * (size_t)nblk * NP;
  if (block_partial_and_total<NP, 0u>(part, a.partials + pbase, a.counters + rhs, blk, nblk,
                                      scratch, tot)) {
    if (threadIdx.x == 0) pcg_decide(a.scal[rhs], tot);
  }
}

// ----------------------------------------------------------------------------
// The elasticity apply for two right-hand sides per warp (k >= 2): the same
// march as march_core<Elast, APPLY>, with the word, the element weights and
// the Dirichlet mask of a cell row formed once for both fields, and two
// independent dependency chains per warp (the one-field apply is latency-
// bound on short row segments).  Odd k: the last pair's second field is the
// first one again, computed but not stored.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) apply2_kernel(Elast ph, Geo g, MArgs a, int k) {
  constexpr int NC = 2, NOUT = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = blockIdx.x * kWarps + warp;
  const uint8_t *words = static_cast<const uint8_t *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);
  const int r0 = 2 * (int)blockIdx.z;
  const bool two = r0 + 1 < k;
  const int rr[2] = {r0, two ? r0 + 1 : r0};
  const int i = strip * kStrip - 1 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool own = node_ok && lane >= 1 && lane <= kStrip;
  const int ic = min(max(i, 0), nx);
  const int J0 = blockIdx.y * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const double *xin[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) xin[j] = a.x + (size_t)rr[j] * (size_t)nn * NC + (size_t)ic * NC;
  const uint8_t *win = words + ic;

  struct Raw {
    double v[2][NC];
    uint32_t wc;
  };
  struct Row {
    double in[2][NC], rt[2][NC], raw[2][NC];
    uint32_t wc;
  };
  auto fetch = [&](int r, Raw &f) {
    const int64_t off = (int64_t)r * nxp;
    f.wc = node_ok ? (uint32_t)__ldg(win + off) : 0u;
#pragma unroll
    for (int j = 0; j < 2; ++j) ldg_node<NC>(xin[j], off, f.v[j]);
  };
  auto prepare = [&](const Raw &f, Row &S) {
    S.wc = f.wc;
    const uint32_t m = Elast::mask(f.wc);
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        S.raw[j][c] = f.v[j][c];
        S.in[j][c] = ((m >> c) & 1u) ? 0.0 : f.v[j][c];
      }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < NC; ++c) S.rt[j][c] = __shfl_down_sync(0xffffffffu, S.in[j][c], 1);
  };
  auto emit = [&](int r, const Row &S, const double (*accv)[NOUT]) {
    const int64_t node = (int64_t)r * nxp + i;
    const uint32_t m = Elast::mask(S.wc);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (j == 1 && !two) break;
      double yv[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) yv[c] = ((m >> c) & 1u) ? S.raw[j][c] : accv[j][c];
      st_node<NC>(a.y + (size_t)rr[j] * (size_t)nn * NC, node, yv);
    }
  };
  auto step = [&](int r, const Raw &f, const Row &Sp, Row &Sn, double (*ap)[NOUT], double (*an)[NOUT]) {
    prepare(f, Sn);
    double wl, wu;
    ph.weights(Sp.wc, wl, wu);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
      ph.cell_w(Sp.in[j], Sp.rt[j], Sn.in[j], Sn.rt[j], wl, wu, c00, c10, c01, c11);
#pragma unroll
      for (int t = 0; t < NOUT; ++t) {
        double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);
        double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
        if (lane == 0) up10 = up11 = 0.0;
        ap[j][t] += c00[t] + up10;
        an[j][t] = c01[t] + up11;
      }
    }
    if (own && (r - 1) >= J0) emit(r - 1, Sp, ap);
  };

  const int jstart = max(J0 - 1, 0);
  const int rend = min(J1, ny);
  Row SA, SB;
  double accA[2][NOUT], accB[2][NOUT];
  Raw fA, fB;
  {
    Raw f0;
    fetch(jstart, f0);
    fetch(min(jstart + 1, rend), fA);
    fetch(min(jstart + 2, rend), fB);
    prepare(f0, SA);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int t = 0; t < NOUT; ++t) accA[j][t] = 0.0;
  bool last_in_b = false;
  int r = jstart + 1;
  while (r <= rend) {
    step(r, fA, SA, SB, accA, accB);
    fetch(min(r + 2, rend), fA);
    if (++r > rend) { last_in_b = true; break; }
    step(r, fB, SB, SA, accB, accA);
    fetch(min(r + 2, rend), fB);
    ++r;
  }
  if (J1 == ny + 1 && own && ny >= J0) {
    if (last_in_b) emit(ny, SB, accB);
    else emit(ny, SA, accA);
  }
}

// ----------------------------------------------------------------------------
// The apply with its prefetch ring in shared memory (per-lane cp.async of the
// node's field and the aligned word chunk, kApplyAhead rows ahead, no
// barriers: each lane reads back only its own copies).  Same march, same
// arithmetic and summation order as march_core<PH, APPLY>; the register ring
// of march_core holds only two rows because deeper register rings cost
// resident CTAs.
// ----------------------------------------------------------------------------
#ifndef LSG_APPLY_AHEAD
#define LSG_APPLY_AHEAD 6
#endif
constexpr int kApplyAhead = LSG_APPLY_AHEAD;

template <class PH>
__global__ void __launch_bounds__(kThreads) apply_s_kernel(PH ph, Geo g, MArgs a) {
  constexpr int NC = PH::NC, NOUT = PH::NOUT, A = kApplyAhead, D = A + 1;
  constexpr int FS = 32 * NC;        // doubles per slot: the field
  constexpr int SLOT = FS + 16;      // + 32 words
  __shared__ __align__(16) double ring_all[kWarps * D * SLOT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = blockIdx.x * kWarps + warp;
  const uint8_t *words = static_cast<const uint8_t *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);
  const int i = strip * kStrip - 1 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool own = node_ok && lane >= 1 && lane <= kStrip;
  const int ic = min(max(i, 0), nx);
  const int J0 = blockIdx.y * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const size_t voff = (size_t)blockIdx.z * (size_t)nn * NC;
  const double *xin = a.x + voff;
  double *myring = ring_all + (size_t)warp * D * SLOT;

  struct Row {
    double in[NC], rt[NC], raw[NC];
    uint32_t wc;
  };
  auto fetch = [&](int r, int sl) {
    double *S = myring + sl * SLOT;
    const int64_t node = (int64_t)r * nxp + ic;
    if constexpr (NC == 2) cp_async16(S + lane * NC, xin + node * NC);
    else cp_async8(S + lane * NC, xin + node * NC);
    uint32_t *W = reinterpret_cast<uint32_t *>(S + FS);
    const int64_t wq = node & ~(int64_t)3;
    if (wq + 4 <= nn) cp_async4(W + lane, words + wq);
    else W[lane] = (uint32_t)words[node] << (8 * (node & 3));
    cp_async_commit();
  };
  auto prepare = [&](int r, int sl, Row &S) {
    const double *P = myring + sl * SLOT;
    const uint32_t w4 = reinterpret_cast<const uint32_t *>(P + FS)[lane];
    const int64_t node = (int64_t)r * nxp + ic;
    S.wc = node_ok ? (w4 >> (8 * (uint32_t)(node & 3))) & 0xffu : 0u;
    const uint32_t m = PH::mask(S.wc);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      S.raw[c] = P[lane * NC + c];
      S.in[c] = ((m >> c) & 1u) ? 0.0 : S.raw[c];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) S.rt[c] = __shfl_down_sync(0xffffffffu, S.in[c], 1);
  };
  auto emit = [&](int r, const Row &S, const double *accv) {
    const int64_t node = (int64_t)r * nxp + i;
    const uint32_t m = PH::mask(S.wc);
    double yv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) yv[c] = ((m >> c) & 1u) ? S.raw[c] : accv[c];
    st_node<NC>(a.y + voff, node, yv);
  };
  auto step = [&](int r, int sl, const Row &Sp, Row &Sn, double *ap, double *an) {
    cp_async_wait_all_but<A - 1>();  // row r has landed
    prepare(r, sl, Sn);
    double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
    ph.cell(Sp.in, Sp.rt, Sn.in, Sn.rt, Sp.wc, i, r - 1, c00, c10, c01, c11);
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);
      double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
      if (lane == 0) up10 = up11 = 0.0;
      ap[t] += c00[t] + up10;
      an[t] = c01[t] + up11;
    }
    if (own && (r - 1) >= J0) emit(r - 1, Sp, ap);
  };

  const int jstart = max(J0 - 1, 0);
  const int rend = min(J1, ny);
  auto nxt = [](int s) { return s + 1 == D ? 0 : s + 1; };
  // rows jstart .. jstart + A in slots 0 .. A
#pragma unroll
  for (int s = 0; s < D; ++s) fetch(min(jstart + s, rend), s);
  Row SA, SB;
  double accA[NOUT], accB[NOUT];
  cp_async_wait_all_but<D - 1>();
  prepare(jstart, 0, SA);
#pragma unroll
  for (int t = 0; t < NOUT; ++t) accA[t] = 0.0;
  bool last_in_b = false;
  int r = jstart + 1, sl = 1;
  // step r consumes slot sl (row r); the slot of row r - 1 is refilled with row r + A
  int sfree = 0;
  while (r <= rend) {
    step(r, sl, SA, SB, accA, accB);
    fetch(min(r + A, rend), sfree);
    sfree = sl;
    sl = nxt(sl);
    if (++r > rend) { last_in_b = true; break; }
    step(r, sl, SB, SA, accB, accA);
    fetch(min(r + A, rend), sfree);
    sfree = sl;
    sl = nxt(sl);
    ++r;
  }
  cp_async_wait_all_but<0>();
  if (J1 == ny + 1 && own && ny >= J0) {
    if (last_in_b) emit(ny, SB, accB);
    else emit(ny, SA, accA);
  }
}

template <class PH, int ACT, class W>
__global__ void __launch_bounds__(kThreads) march(PH ph, Geo g, MArgs a) {
  constexpr int NP = Traits<PH, ACT>::NP;
  constexpr int NPA = NP > 0 ? NP : 1;
  __shared__ double scratch[NPA * kWarps];
  const int rhs = blockIdx.z;
  double part[NPA];
#pragma unroll
  for (int t = 0; t < NPA; ++t) part[t] = 0.0;
  if constexpr (ACT == PCG) {
    const lsg_pcg_scalars &s = a.scal[rhs];
    if (s.done != 0.0) return;  // uniform across the CTA (x is final: nothing pending)
    march_pcg<PH>(ph, g, a, blockIdx.x, blockIdx.y, rhs, s.first != 0.0, s.beta, s.alpha, part);
  } else {
    if constexpr (ACT == RESID) {
      if (a.scal[rhs].done != 0.0) return;
    }
    march_core<PH, ACT, W>(ph, g, a, blockIdx.x, blockIdx.y, rhs, part);
  }

  if constexpr (NP > 0) {
    const int nblk = gridDim.x * gridDim.y;
    const int blk = blockIdx.y * gridDim.x + blockIdx.x;
    double tot[NPA];
    const size_t pbase = (size_t)rhs * (size_t)nblk * NP;
    if (block_partial_and_total<NP, Traits<PH, ACT>::MAXMASK>(part, a.partials + pbase,
                                                              a.counters + rhs, blk, nblk,
                                                              scratch, tot)) {
      if (threadIdx.x == 0) finalize<ACT>(a, rhs, tot);
    }
  }
}

}  // namespace d2
}  // namespace lsg
