// 2D kernels of liblsgpu: operator apply and fused PCG passes (warp
// marching, see march2d.cuh), fused compliance + shape-derivative RHS,
// velocity statistics, material words and the PCG update pass.
#include <math.h>

#include "march2d.cuh"
#include "ops.h"

namespace lsg {
namespace d2 {

enum Act { APPLY = 0, RESID = 1, PCGA = 2, STATS = 3, SHAPE = 4 };

// Arguments shared by every marching launch (unused fields stay null).
struct MArgs {
  const void *words;
  const double *x;   // APPLY/RESID/STATS: input field ; PCGA: r ; SHAPE: u (KB fields)
  const double *x2;  // PCGA: p_old ; STATS: vec
  const double *b;   // RESID: b
  double *y;         // APPLY: y ; RESID: r ; PCGA: q ; SHAPE: vec_cost
  double *y2;        // PCGA: p (written) ; SHAPE: vec_vol
  lsg_pcg_scalars *scal;
  double *partials;
  uint32_t *counters;
  double *out;       // STATS / SHAPE scalar outputs
  int seg;           // node rows per segment
  int nstrips;
  int accumulate;    // SHAPE: add into vec_cost / out[0] (later RHS chunks)
};

// Compliance + shape-derivative physics for KB load cases at once
// (compliance.py:111-139, base.py:150-158, velocity.py:129-142).
// in = KB displacement fields, out = (vec_cost[2], vec_vol[2]).
template <int KB>
struct Shape {
  static constexpr int NIN = 2 * KB, NOUT = 4;
  double lam, mu, area, inv_hx, inv_hy, inv_volume;
  double w0, w1;  // |T| * abar(n_in) = w0 + w1 n_in

  __device__ __forceinline__ static bool valid(uint32_t w) { return (w >> 4) & 1u; }
  __device__ __forceinline__ static uint32_t mask(uint32_t) { return 0u; }

  // bulk = sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I), row-major; dens = sum_k sigma:eps.
  // Triangle given by the raw x- and y-differences of each field.
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
                                       const double *u11, uint32_t word, bool count, double *c00,
                                       double *c10, double *c01, double *c11, double *part) const {
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
    c00[2] = -vl * inv_hx;              c00[3] = -vu * inv_hy;
    c10[2] = vl * inv_hx;               c10[3] = -vl * inv_hy;
    c11[2] = vu * inv_hx;               c11[3] = vl * inv_hy;
    c01[2] = -vu * inv_hx;              c01[3] = vu * inv_hy;
    if (count) {
      part[0] += wl * dl + wu * du;
      part[1] += area * (double)(nl + nu) * (1.0 / 3.0);
    }
  }
};

template <class PH>
struct NP_of { static constexpr int v = 0; };

template <class PH, int ACT>
struct Traits {
  static constexpr int NP = (ACT == RESID) ? 3 : (ACT == PCGA) ? 1 : (ACT == STATS) ? 3
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
__device__ __forceinline__ void node_diag<H1>(const H1 &ph, uint32_t w00, uint32_t wm0,
                                              uint32_t w0m, uint32_t wmm, int i, int j, double *d) {
  ph.diag(w00, wm0, w0m, wmm, i, j, d);
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
  } else if constexpr (ACT == PCGA) {
    lsg_pcg_scalars &s = a.scal[rhs];
    s.pq = tot[0];
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

// ----------------------------------------------------------------------------
// The marching skeleton.  PH = Elast | H1 (operators) or Shape<KB>.
// ----------------------------------------------------------------------------
template <class PH, int ACT, class W>
__global__ void __launch_bounds__(kThreads) march(PH ph, Geo g, MArgs a) {
  constexpr int NIN = PH::NIN, NOUT = PH::NOUT;
  constexpr int NP = Traits<PH, ACT>::NP;
  constexpr int NPA = NP > 0 ? NP : 1;
  __shared__ double scratch[NPA * kWarps];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int strip = blockIdx.x * kWarps + warp;
  const int rhs = blockIdx.z;
  const W *words = static_cast<const W *>(a.words);
  const int nx = g.nx, ny = g.ny;
  const int64_t nxp = nx + 1;
  const int64_t nn = nxp * (ny + 1);

  double beta = 0.0;
  bool first = false;
  if constexpr (ACT == PCGA || ACT == RESID) {
    const lsg_pcg_scalars &s = a.scal[rhs];
    if (s.done != 0.0) return;  // uniform across the CTA
    if constexpr (ACT == PCGA) {
      first = s.first != 0.0;
      beta = s.beta;
    }
  }

  const int i = strip * kStrip - 1 + lane;
  const bool node_ok = (strip < a.nstrips) && i >= 0 && i <= nx;
  const bool left_ok = node_ok && i >= 1;
  const bool own = node_ok && lane >= 1 && lane <= kStrip;
  const int J0 = blockIdx.y * a.seg;
  const int J1 = min(J0 + a.seg, ny + 1);
  const size_t voff = (ACT == SHAPE) ? 0 : (size_t)rhs * (size_t)nn * 2;

  double part[NPA];
#pragma unroll
  for (int t = 0; t < NPA; ++t) part[t] = 0.0;

  double in_prev[NIN], rt_prev[NIN], raw_prev[2], dg_prev[2];
  double in_new[NIN], rt_new[NIN], raw_new[2], dg_new[2];
  double acc[NOUT], nxt[NOUT];
  uint32_t wc_cur = 0, wl_cur = 0;

  auto load_words = [&](int r, uint32_t &wc, uint32_t &wl) {
    wc = wl = 0u;
    if (r < 0) return;
    const int64_t node = (int64_t)r * nxp + i;
    if (node_ok) wc = (uint32_t)__ldg(words + node);
    if (left_ok) wl = (uint32_t)__ldg(words + node - 1);
  };

  // Input of node row r (masked for the operator) + raw value + diagonal.
  auto load_row = [&](int r, uint32_t wc, uint32_t wl, uint32_t wcp, uint32_t wlp, double *in,
                      double *raw, double *dg) {
    const int64_t node = (int64_t)r * nxp + i;
    if constexpr (ACT == SHAPE) {
#pragma unroll
      for (int k = 0; k < NIN / 2; ++k) {
        double2 v = node_ok
                        ? __ldg(reinterpret_cast<const double2 *>(a.x + ((size_t)k * nn + node) * 2))
                        : make_double2(0.0, 0.0);
        in[2 * k] = v.x;
        in[2 * k + 1] = v.y;
      }
      raw[0] = raw[1] = 0.0;
      dg[0] = dg[1] = 1.0;
    } else {
      const uint32_t m = node_ok ? PH::mask(wc) : 0u;
      dg[0] = dg[1] = 1.0;
      if constexpr (ACT == RESID || ACT == PCGA) {
        if (node_ok) node_diag<PH>(ph, wc, wl, wcp, wlp, i, r, dg);
        if (m & 1u) dg[0] = 1.0;
        if (m & 2u) dg[1] = 1.0;
      }
      double2 v;
      if constexpr (ACT == PCGA) {
        // z = M^-1 r with M^-1 = diag(1/D) (fem.py:303-305); p = z + beta p_old
        const double2 rv = node_ok
                               ? __ldg(reinterpret_cast<const double2 *>(a.x + voff) + node)
                               : make_double2(0.0, 0.0);
        const double zx = rv.x * (1.0 / dg[0]), zy = rv.y * (1.0 / dg[1]);
        if (first) {
          v = make_double2(zx, zy);
        } else {
          const double2 po = node_ok
                                 ? __ldg(reinterpret_cast<const double2 *>(a.x2 + voff) + node)
                                 : make_double2(0.0, 0.0);
          v = make_double2(fma(beta, po.x, zx), fma(beta, po.y, zy));
        }
        if (own && r >= J0 && r < J1) reinterpret_cast<double2 *>(a.y2 + voff)[node] = v;
      } else {
        v = node_ok ? __ldg(reinterpret_cast<const double2 *>(a.x + voff) + node)
                    : make_double2(0.0, 0.0);
      }
      raw[0] = v.x;
      raw[1] = v.y;
      in[0] = (m & 1u) ? 0.0 : v.x;
      in[1] = (m & 2u) ? 0.0 : v.y;
    }
  };

  auto emit = [&](int r, uint32_t wc, const double *accv, const double *raw, const double *dg) {
    const int64_t node = (int64_t)r * nxp + i;
    if constexpr (ACT == SHAPE) {
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
      const uint32_t m = PH::mask(wc);
      const double yx = (m & 1u) ? raw[0] : accv[0];
      const double yy = (m & 2u) ? raw[1] : accv[1];
      if constexpr (ACT == APPLY) {
        reinterpret_cast<double2 *>(a.y + voff)[node] = make_double2(yx, yy);
      } else if constexpr (ACT == RESID) {
        const double2 bv = __ldg(reinterpret_cast<const double2 *>(a.b + voff) + node);
        const double rx = bv.x - yx, ry = bv.y - yy;
        reinterpret_cast<double2 *>(a.y + voff)[node] = make_double2(rx, ry);
        part[0] += bv.x * bv.x + bv.y * bv.y;
        part[1] += rx * rx + ry * ry;
        part[2] += rx * (rx * (1.0 / dg[0])) + ry * (ry * (1.0 / dg[1]));
      } else if constexpr (ACT == PCGA) {
        reinterpret_cast<double2 *>(a.y + voff)[node] = make_double2(yx, yy);
        part[0] += raw[0] * yx + raw[1] * yy;
      } else if constexpr (ACT == STATS) {
        const double2 vv = __ldg(reinterpret_cast<const double2 *>(a.x2) + node);
        part[0] += raw[0] * yx + raw[1] * yy;
        part[1] += vv.x * raw[0] + vv.y * raw[1];
        part[2] = fmax(part[2], fabs(raw[0]) / g.hx + fabs(raw[1]) / g.hy);
      }
    }
  };

  // ---- prologue: words of rows jstart-1, jstart; input of row jstart -------
  const int jstart = max(J0 - 1, 0);
  {
    uint32_t wcm, wlm;
    load_words(jstart - 1, wcm, wlm);
    load_words(jstart, wc_cur, wl_cur);
    load_row(jstart, wc_cur, wl_cur, wcm, wlm, in_prev, raw_prev, dg_prev);
  }
#pragma unroll
  for (int t = 0; t < NIN; ++t) rt_prev[t] = __shfl_down_sync(0xffffffffu, in_prev[t], 1);
#pragma unroll
  for (int t = 0; t < NOUT; ++t) acc[t] = 0.0;

  const int rend = min(J1, ny);
  for (int r = jstart + 1; r <= rend; ++r) {
    uint32_t wc_new, wl_new;
    load_words(r, wc_new, wl_new);
    load_row(r, wc_new, wl_new, wc_cur, wl_cur, in_new, raw_new, dg_new);
#pragma unroll
    for (int t = 0; t < NIN; ++t) rt_new[t] = __shfl_down_sync(0xffffffffu, in_new[t], 1);

    double c00[NOUT], c10[NOUT], c01[NOUT], c11[NOUT];
    if constexpr (ACT == SHAPE) {
      ph.cell(in_prev, rt_prev, in_new, rt_new, wc_cur, own && (r - 1) >= J0, c00, c10, c01, c11,
              part);
    } else {
      ph.cell(in_prev, rt_prev, in_new, rt_new, wc_cur, i, r - 1, c00, c10, c01, c11);
    }
#pragma unroll
    for (int t = 0; t < NOUT; ++t) {
      double up10 = __shfl_up_sync(0xffffffffu, c10[t], 1);
      double up11 = __shfl_up_sync(0xffffffffu, c11[t], 1);
      if (lane == 0) up10 = up11 = 0.0;
      acc[t] += c00[t] + up10;
      nxt[t] = c01[t] + up11;
    }
    if (own && (r - 1) >= J0) emit(r - 1, wc_cur, acc, raw_prev, dg_prev);
#pragma unroll
    for (int t = 0; t < NIN; ++t) {
      in_prev[t] = in_new[t];
      rt_prev[t] = rt_new[t];
    }
    raw_prev[0] = raw_new[0]; raw_prev[1] = raw_new[1];
    dg_prev[0] = dg_new[0];   dg_prev[1] = dg_new[1];
#pragma unroll
    for (int t = 0; t < NOUT; ++t) acc[t] = nxt[t];
    wc_cur = wc_new;
    wl_cur = wl_new;
  }
  if (J1 == ny + 1 && own && ny >= J0) emit(ny, wc_cur, acc, raw_prev, dg_prev);

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

// ----------------------------------------------------------------------------
// PCG pass B (elementwise): x += alpha p ; r -= alpha q ; rz = r.M^-1 r ; rr.
// ----------------------------------------------------------------------------
constexpr int kEwThreads = 256;

template <class PH>
__global__ void __launch_bounds__(kEwThreads)
    pcg_update(PH ph, Geo g, const uint8_t *words, double *x, double *r, const double *p,
               const double *q, lsg_pcg_scalars *scal, double *partials, uint32_t *counters) {
  __shared__ double scratch[2 * (kEwThreads / 32)];
  const int rhs = blockIdx.y;
  lsg_pcg_scalars &s = scal[rhs];
  if (s.done != 0.0) return;
  const double alpha = s.alpha;
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * kEwThreads + threadIdx.x;
  const size_t voff = (size_t)rhs * (size_t)nn * 2;
  double part[2] = {0.0, 0.0};
  if (node < nn) {
    const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
    const uint32_t w00 = words[node];
    const uint32_t wm0 = i > 0 ? words[node - 1] : 0u;
    const uint32_t w0m = j > 0 ? words[node - nxp] : 0u;
    const uint32_t wmm = (i > 0 && j > 0) ? words[node - nxp - 1] : 0u;
    double dg[2];
    node_diag<PH>(ph, w00, wm0, w0m, wmm, i, j, dg);
    const uint32_t m = PH::mask(w00);
    if (m & 1u) dg[0] = 1.0;
    if (m & 2u) dg[1] = 1.0;
    double2 *xv = reinterpret_cast<double2 *>(x + voff);
    double2 *rv = reinterpret_cast<double2 *>(r + voff);
    const double2 pv = __ldg(reinterpret_cast<const double2 *>(p + voff) + node);
    const double2 qv = __ldg(reinterpret_cast<const double2 *>(q + voff) + node);
    double2 xo = xv[node], ro = rv[node];
    xo.x = fma(alpha, pv.x, xo.x);
    xo.y = fma(alpha, pv.y, xo.y);
    ro.x = fma(-alpha, qv.x, ro.x);
    ro.y = fma(-alpha, qv.y, ro.y);
    xv[node] = xo;
    rv[node] = ro;
    part[0] = ro.x * (ro.x * (1.0 / dg[0])) + ro.y * (ro.y * (1.0 / dg[1]));
    part[1] = ro.x * ro.x + ro.y * ro.y;
  }
  double tot[2];
  const int nblk = gridDim.x;
  if (block_partial_and_total<2, 0u>(part, partials + (size_t)rhs * nblk * 2, counters + rhs,
                                     blockIdx.x, nblk, scratch, tot)) {
    if (threadIdx.x == 0) {
      s.iters += 1.0;
      s.rz_new = tot[0];
      s.rr = tot[1];
      if (sqrt(tot[1]) < s.atol) {
        s.done = 1.0;
      } else if (s.iters >= s.maxiter) {
        s.done = 2.0;  // iteration cap exhausted: SolverError on the host
      } else {
        s.beta = tot[0] / s.rho;
        s.rho = tot[0];
        s.first = 0.0;
      }
    }
  }
}

// ----------------------------------------------------------------------------
// Material words (levelset.py:65-67, models/base.py:117-119).
// ----------------------------------------------------------------------------
__device__ __forceinline__ int neg_mid(double a, double b) { return (0.5 * a + 0.5 * b) < 0.0; }

__global__ void material_kernel(Geo g, const double *phi, const uint8_t *bcmask, uint8_t *words) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  uint32_t w = ((uint32_t)(bcmask ? bcmask[node] : 0) & 3u) << 5;
  if (i < g.nx && j < g.ny) {
    const double p00 = phi[node], p10 = phi[node + 1];
    const double p01 = phi[node + nxp], p11 = phi[node + nxp + 1];
    // lower (a,b,c) = (00,10,11): edges (0,1), (1,2), (0,2) (fem.py:43-45)
    const int nl = neg_mid(p00, p10) + neg_mid(p10, p11) + neg_mid(p00, p11);
    // upper (a,c,d) = (00,11,01)
    const int nu = neg_mid(p00, p11) + neg_mid(p11, p01) + neg_mid(p00, p01);
    w |= (uint32_t)nl | ((uint32_t)nu << 2) | (1u << 4);
  }
  words[node] = (uint8_t)w;
}

__global__ void indicator_kernel(Geo g, const double *phi, double *chi) {
  const int64_t ncell = (int64_t)g.nx * g.ny;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  const int j = (int)(c / g.nx), i = (int)(c - (int64_t)j * g.nx);
  const int64_t nxp = g.nx + 1;
  const int64_t n0 = (int64_t)j * nxp + i;
  const double p00 = phi[n0], p10 = phi[n0 + 1], p01 = phi[n0 + nxp], p11 = phi[n0 + nxp + 1];
  double *lo = chi + c * 6, *up = lo + 3;
  lo[0] = neg_mid(p00, p10); lo[1] = neg_mid(p10, p11); lo[2] = neg_mid(p00, p11);
  up[0] = neg_mid(p00, p11); up[1] = neg_mid(p11, p01); up[2] = neg_mid(p00, p01);
}

// H1 words: frozen quadrature bits + zero-Dirichlet on boundary nodes.
__global__ void h1_words_kernel(Geo g, const uint8_t *frozen_q, int zero_dirichlet, uint8_t *words) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  uint32_t w = 0;
  if (i < g.nx && j < g.ny) {
    w |= 1u << 7;
    if (frozen_q) {
      const int64_t c = (int64_t)j * g.nx + i;
      const uint8_t *f = frozen_q + c * 6;
      for (int q = 0; q < 6; ++q) w |= (f[q] ? 1u : 0u) << q;
    }
  }
  if (zero_dirichlet && (i == 0 || j == 0 || i == g.nx || j == g.ny)) w |= 1u << 6;
  words[node] = (uint8_t)w;
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
  lsg_pcg_scalars s;
  s.atol = atol;
  s.rho = s.alpha = s.beta = s.rr = s.pq = s.bb = 0.0;
  s.iters = 0.0;
  s.done = 0.0;
  s.zero_rhs = 0.0;
  s.maxiter = maxiter;
  s.first = 1.0;
  s.rz_new = 0.0;
  s.reserved[0] = rtol;
  s.reserved[1] = s.reserved[2] = 0.0;
  scal[r] = s;
}

// b = -(vc + lam vv), Dirichlet dofs of the velocity form zeroed.
__global__ void velocity_rhs_kernel(int64_t nn, const uint8_t *words, const double *vc,
                                    const double *vv, double lam, double *b) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const bool pin = (words[node] >> 6) & 1u;
  for (int c = 0; c < 2; ++c) {
    const double v = vc[node * 2 + c] + lam * vv[node * 2 + c];
    b[node * 2 + c] = pin ? 0.0 : -v;
  }
}

// Generic tensor pair -> vector, gather over the six incident triangles of a node.
__global__ void tensor_rhs_kernel(Geo g, const double *s0, const double *s1, double *vec) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  const double ihx = 1.0 / g.hx, ihy = 1.0 / g.hy;
  const double w = 0.5 * g.hx * g.hy / 3.0;  // quadrature weight |T|/3
  // (cell di, cell dj, triangle 0 lower / 1 upper, local vertex, gx, gy)
  struct Inc { int di, dj, t, v; double gx, gy; };
  const Inc inc[6] = {{0, 0, 0, 0, -ihx, 0.0},  {0, 0, 1, 0, 0.0, -ihy},
                      {-1, 0, 0, 1, ihx, -ihy}, {-1, -1, 0, 2, 0.0, ihy},
                      {-1, -1, 1, 1, ihx, 0.0}, {0, -1, 1, 2, -ihx, ihy}};
  // barycentric value of local vertex v at quadrature point q (edges (0,1),(1,2),(0,2))
  const double bary[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
  double acc[2] = {0.0, 0.0};
  for (int e = 0; e < 6; ++e) {
    const int ci = i + inc[e].di, cj = j + inc[e].dj;
    if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) continue;
    const int64_t t = 2 * ((int64_t)cj * g.nx + ci) + inc[e].t;
    for (int q = 0; q < 3; ++q) {
      for (int c = 0; c < 2; ++c) {
        double v = 0.0;
        if (s1) {
          const double *S = s1 + ((t * 3 + q) * 2 + c) * 2;
          v += S[0] * inc[e].gx + S[1] * inc[e].gy;
        }
        if (s0) v += s0[(t * 3 + q) * 2 + c] * bary[q][inc[e].v];
        acc[c] += w * v;
      }
    }
  }
  vec[node * 2] = acc[0];
  vec[node * 2 + 1] = acc[1];
}

// S1 of the cost per element and quadrature point (parity/debug path):
// S1_q = A_q sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I)   (compliance.py:128-139)
__global__ void s1_kernel(Geo g, double lam, double mu, double ersatz, double inside, int k,
                          const double *u,
                          const double *phi, double *s1) {
  const int64_t ncell = (int64_t)g.nx * g.ny;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * ncell) return;
  const int64_t c = t >> 1;
  const bool upper = t & 1;
  const int j = (int)(c / g.nx), i = (int)(c - (int64_t)j * g.nx);
  const int64_t nxp = g.nx + 1;
  const int64_t n00 = (int64_t)j * nxp + i, n10 = n00 + 1, n01 = n00 + nxp, n11 = n01 + 1;
  const int64_t nn = nxp * (g.ny + 1);
  double bulk[4] = {0, 0, 0, 0};
  for (int f = 0; f < k; ++f) {
    const double *U = u + (size_t)f * nn * 2;
    double Px, Py, Qx, Qy;
    if (!upper) {
      Px = (U[n10 * 2] - U[n00 * 2]) / g.hx;  Py = (U[n10 * 2 + 1] - U[n00 * 2 + 1]) / g.hx;
      Qx = (U[n11 * 2] - U[n10 * 2]) / g.hy;  Qy = (U[n11 * 2 + 1] - U[n10 * 2 + 1]) / g.hy;
    } else {
      Px = (U[n11 * 2] - U[n01 * 2]) / g.hx;  Py = (U[n11 * 2 + 1] - U[n01 * 2 + 1]) / g.hx;
      Qx = (U[n01 * 2] - U[n00 * 2]) / g.hy;  Qy = (U[n01 * 2 + 1] - U[n00 * 2 + 1]) / g.hy;
    }
    const double exx = Px, eyy = Qy, exy = 0.5 * (Py + Qx), tr = exx + eyy;
    const double sxx = 2.0 * mu * exx + lam * tr, syy = 2.0 * mu * eyy + lam * tr, sxy = 2.0 * mu * exy;
    const double d = sxx * exx + syy * eyy + 2.0 * sxy * exy;
    bulk[0] += 2.0 * (Px * sxx + Py * sxy) - d;
    bulk[1] += 2.0 * (Px * sxy + Py * syy);
    bulk[2] += 2.0 * (Qx * sxx + Qy * sxy);
    bulk[3] += 2.0 * (Qx * sxy + Qy * syy) - d;
  }
  const double p00 = phi[n00], p10 = phi[n10], p01 = phi[n01], p11 = phi[n11];
  int chi[3];
  if (!upper) { chi[0] = neg_mid(p00, p10); chi[1] = neg_mid(p10, p11); chi[2] = neg_mid(p00, p11); }
  else        { chi[0] = neg_mid(p00, p11); chi[1] = neg_mid(p11, p01); chi[2] = neg_mid(p00, p01); }
  for (int q = 0; q < 3; ++q) {
    const double A = chi[q] ? inside : ersatz;
    for (int e = 0; e < 4; ++e) s1[(t * 3 + q) * 4 + e] = A * bulk[e];
  }
}

// max_i sum_d |v_d| / h_d
__global__ void cfl_kernel(int64_t nn, double ihx, double ihy, const double *v, double *partials,
                           uint32_t *counter, double *out) {
  __shared__ double scratch[kEwThreads / 32];
  double m[1] = {0.0};
  for (int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; node < nn;
       node += (int64_t)gridDim.x * blockDim.x)
    m[0] = fmax(m[0], fabs(v[node * 2]) * ihx + fabs(v[node * 2 + 1]) * ihy);
  double tot[1];
  if (block_partial_and_total<1, 1u>(m, partials, counter, blockIdx.x, gridDim.x, scratch, tot))
    if (threadIdx.x == 0) out[0] = tot[0];
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------
static Geo geo_of(const lsg_grid &g) {
  Geo o;
  o.nx = g.n[0];
  o.ny = g.n[1];
  o.hx = (g.hi[0] - g.lo[0]) / g.n[0];
  o.hy = (g.hi[1] - g.lo[1]) / g.n[1];
  return o;
}

static int nstrips_of(const Geo &g) { return (int)ceil_div(g.nx + 1, kStrip); }

// Rows per segment: enough warps in flight (>= ~16 per SM) without making
// the one-row halo per segment expensive.
static int seg_of(const Geo &g, int k) {
  const int64_t strips = nstrips_of(g);
  const int64_t rows = g.ny + 1;
  const int64_t target_warps = 148 * 24;
  int seg = 64;
  while (seg > 8 && strips * ceil_div(rows, seg) * k < target_warps) seg >>= 1;
  return seg;
}

static dim3 march_grid(const Geo &g, int seg, int k) {
  return dim3((unsigned)ceil_div(nstrips_of(g), kWarps), (unsigned)ceil_div(g.ny + 1, seg),
              (unsigned)k);
}

int64_t partials_per_rhs(const lsg_grid &grid) {
  const Geo g = geo_of(grid);
  int64_t best = 0;
  for (int k : {1, 2, 4, 8, 16, 64}) {
    const dim3 mg = march_grid(g, seg_of(g, k), k);
    best = best > (int64_t)mg.x * mg.y ? best : (int64_t)mg.x * mg.y;
  }
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const int64_t ew = ceil_div(nn, kEwThreads);
  best = best > ew ? best : ew;
  return best > 1024 ? best : 1024;
}

static Elast make_elast(const Geo &g, const lsg_op &op) {
  const double lam = op.p[0], mu = op.p[1], eps = op.p[2];
  const double hx = g.hx, hy = g.hy, area = 0.5 * hx * hy;
  Elast e;
  e.k1 = (lam + 2.0 * mu) / (hx * hx);
  e.k2 = lam / (hx * hy);
  e.k3 = mu / (hx * hx);
  e.k4 = mu / (hx * hy);
  e.k5 = mu / (hy * hy);
  e.k6 = (lam + 2.0 * mu) / (hy * hy);
  const double inside = op.p[3] > 0.0 ? op.p[3] : 1.0;
  e.w0 = area * eps;
  e.w1 = area * (inside - eps) / 3.0;
  return e;
}

static H1 make_h1(const Geo &g, const lsg_op &op) {
  const double mw = op.p[0], sw = op.p[1], npen = op.p[2], fp = op.p[3];
  const double area = 0.5 * g.hx * g.hy;
  H1 h;
  h.nx = g.nx;
  h.ny = g.ny;
  h.m = mw * area / 12.0;
  h.ax = sw * area / (g.hx * g.hx);
  h.ay = sw * area / (g.hy * g.hy);
  h.fz = fp * area / 3.0 * 0.25;
  h.nbx = npen * g.hx / 6.0;
  h.nby = npen * g.hy / 6.0;
  return h;
}

template <class PH, int ACT>
static int launch_march(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  a.seg = seg_of(g, k);
  a.nstrips = nstrips_of(g);
  const dim3 grid = march_grid(g, a.seg, k);
  march<PH, ACT, uint8_t><<<grid, kThreads, 0, st>>>(ph, g, a);
  return check_launch("march2d");
}

template <int ACT>
static int dispatch_op(const lsg_op &op, MArgs a, int k, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  if (op.kind == LSG_OP_ELASTICITY) return launch_march<Elast, ACT>(make_elast(g, op), g, a, k, st);
  if (op.kind == LSG_OP_H1) return launch_march<H1, ACT>(make_h1(g, op), g, a, k, st);
  set_error("unknown operator kind %d", op.kind);
  return LSG_ERR_ARG;
}

int apply(const lsg_op &op, int k, const double *x, double *y, cudaStream_t st) {
  MArgs a = {};
  a.words = op.words;
  a.x = x;
  a.y = y;
  return dispatch_op<APPLY>(op, a, k, st);
}

template <class PH>
__global__ void diag_kernel(PH ph, Geo g, const uint8_t *words, double *d) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  const uint32_t w00 = words[node];
  const uint32_t wm0 = i > 0 ? words[node - 1] : 0u;
  const uint32_t w0m = j > 0 ? words[node - nxp] : 0u;
  const uint32_t wmm = (i > 0 && j > 0) ? words[node - nxp - 1] : 0u;
  double dg[2];
  node_diag<PH>(ph, w00, wm0, w0m, wmm, i, j, dg);
  const uint32_t m = PH::mask(w00);
  d[node * 2] = (m & 1u) ? 1.0 : dg[0];
  d[node * 2 + 1] = (m & 2u) ? 1.0 : dg[1];
}

int diag(const lsg_op &op, double *d, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const unsigned nb = (unsigned)ceil_div(nn, kEwThreads);
  const uint8_t *w = static_cast<const uint8_t *>(op.words);
  if (op.kind == LSG_OP_ELASTICITY) diag_kernel<Elast><<<nb, kEwThreads, 0, st>>>(make_elast(g, op), g, w, d);
  else if (op.kind == LSG_OP_H1) diag_kernel<H1><<<nb, kEwThreads, 0, st>>>(make_h1(g, op), g, w, d);
  else { set_error("unknown operator kind %d", op.kind); return LSG_ERR_ARG; }
  return check_launch("diag2d");
}

int pcg_start(const lsg_op &op, lsg_pcg_ws &ws, double rtol, double atol, double maxiter,
              cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t n = 2 * (int64_t)(g.nx + 1) * (g.ny + 1);
  ws.parity = 0;
  init_scalars<<<(unsigned)ceil_div(ws.k, 64), 64, 0, st>>>(ws.k, ws.scal, rtol, atol, maxiter);
  int rc = check_launch("init_scalars");
  if (rc) return rc;
  MArgs a = {};
  a.words = op.words;
  a.x = ws.x;
  a.b = ws.b;
  a.y = ws.r;
  a.scal = ws.scal;
  a.partials = ws.partials;
  a.counters = ws.counters;
  rc = dispatch_op<RESID>(op, a, ws.k, st);
  if (rc) return rc;
  zero_if_flag<<<dim3(64, ws.k), 256, 0, st>>>(n, ws.scal, ws.x);
  return check_launch("zero_if_flag");
}

int pcg_iterate(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const uint8_t *w = static_cast<const uint8_t *>(op.words);
  MArgs a = {};
  a.words = op.words;
  a.x = ws.r;
  a.y = ws.q;
  a.scal = ws.scal;
  a.partials = ws.partials;
  a.counters = ws.counters;
  const dim3 eg((unsigned)ceil_div(nn, kEwThreads), (unsigned)ws.k);
  for (int it = 0; it < niter; ++it) {
    double *p_old = ws.parity ? ws.p_alt : ws.p;
    double *p_new = ws.parity ? ws.p : ws.p_alt;
    a.x2 = p_old;
    a.y2 = p_new;
    int rc = dispatch_op<PCGA>(op, a, ws.k, st);
    if (rc) return rc;
    if (op.kind == LSG_OP_ELASTICITY)
      pcg_update<Elast><<<eg, kEwThreads, 0, st>>>(make_elast(g, op), g, w, ws.x, ws.r, p_new, ws.q,
                                                    ws.scal, ws.partials, ws.counters);
    else
      pcg_update<H1><<<eg, kEwThreads, 0, st>>>(make_h1(g, op), g, w, ws.x, ws.r, p_new, ws.q,
                                                 ws.scal, ws.partials, ws.counters);
    rc = check_launch("pcg_update2d");
    if (rc) return rc;
    ws.parity ^= 1;
  }
  return LSG_OK;
}

template <int KB>
static int shape_chunk(const Geo &g, const lsg_op &op, const double *u, double volume, double *vc,
                       double *vv, double *out, double *partials, uint32_t *counter, int chunk,
                       cudaStream_t st) {
  Shape<KB> ph;
  const double area = 0.5 * g.hx * g.hy;
  ph.lam = op.p[0];
  ph.mu = op.p[1];
  ph.area = area;
  ph.inv_hx = 1.0 / g.hx;
  ph.inv_hy = 1.0 / g.hy;
  ph.inv_volume = 1.0 / volume;
  const double inside = op.p[3] > 0.0 ? op.p[3] : 1.0;
  ph.w0 = area * op.p[2];
  ph.w1 = area * (inside - op.p[2]) / 3.0;
  MArgs a = {};
  a.words = op.words;
  a.x = u;
  a.y = vc;
  a.y2 = vv;
  a.out = out;
  a.partials = partials;
  a.counters = counter;
  a.accumulate = chunk > 0;
  return launch_march<Shape<KB>, SHAPE>(ph, g, a, 1, st);
}

int shape_rhs(const lsg_op &op, int k, const double *u, double volume, double *vc, double *vv,
              double *out, double *partials, uint32_t *counter, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  int done = 0, chunk = 0;
  while (done < k) {
    const int left = k - done;
    const double *uc = u + (size_t)done * nn * 2;
    int rc, kb;
    if (left >= 4) { kb = 4; rc = shape_chunk<4>(g, op, uc, volume, vc, vv, out, partials, counter, chunk, st); }
    else if (left >= 2) { kb = 2; rc = shape_chunk<2>(g, op, uc, volume, vc, vv, out, partials, counter, chunk, st); }
    else { kb = 1; rc = shape_chunk<1>(g, op, uc, volume, vc, vv, out, partials, counter, chunk, st); }
    if (rc) return rc;
    done += kb;
    ++chunk;
  }
  return LSG_OK;
}

int velocity_stats(const lsg_op &h1, const double *theta, const double *vec, double *out,
                   double *partials, uint32_t *counter, cudaStream_t st) {
  MArgs a = {};
  a.words = h1.words;
  a.x = theta;
  a.x2 = vec;
  a.out = out;
  a.partials = partials;
  a.counters = counter;
  return dispatch_op<STATS>(h1, a, 1, st);
}

int material(const lsg_grid &grid, const double *phi, const uint8_t *bcmask, void *words,
             cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  material_kernel<<<(unsigned)ceil_div(nn, 256), 256, 0, st>>>(g, phi, bcmask,
                                                               static_cast<uint8_t *>(words));
  return check_launch("material2d");
}

int indicator(const lsg_grid &grid, const double *phi, double *chi, cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nc = (int64_t)g.nx * g.ny;
  indicator_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(g, phi, chi);
  return check_launch("indicator2d");
}

int h1_words(const lsg_grid &grid, const uint8_t *frozen_q, int zero_dirichlet, void *words,
             cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  h1_words_kernel<<<(unsigned)ceil_div(nn, 256), 256, 0, st>>>(g, frozen_q, zero_dirichlet,
                                                               static_cast<uint8_t *>(words));
  return check_launch("h1_words2d");
}

int velocity_rhs(const lsg_op &h1, const double *vc, const double *vv, double lam, double *b,
                 cudaStream_t st) {
  const Geo g = geo_of(h1.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  velocity_rhs_kernel<<<(unsigned)ceil_div(nn, 256), 256, 0, st>>>(
      nn, static_cast<const uint8_t *>(h1.words), vc, vv, lam, b);
  return check_launch("velocity_rhs2d");
}

int tensor_rhs(const lsg_grid &grid, const double *s0, const double *s1, double *vec,
               cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  tensor_rhs_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, s0, s1, vec);
  return check_launch("tensor_rhs2d");
}

int s1_tensor(const lsg_op &op, int k, const double *u, const double *phi, double *s1,
              cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t ne = 2 * (int64_t)g.nx * g.ny;
  s1_kernel<<<(unsigned)ceil_div(ne, 128), 128, 0, st>>>(g, op.p[0], op.p[1], op.p[2],
                                                          op.p[3] > 0.0 ? op.p[3] : 1.0, k, u, phi, s1);
  return check_launch("s1_2d");
}

int cfl_speed(const lsg_grid &grid, const double *v, double *out, double *partials,
              uint32_t *counter, cudaStream_t st) {
  const Geo g = geo_of(grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  cfl_kernel<<<296, kEwThreads, 0, st>>>(nn, 1.0 / g.hx, 1.0 / g.hy, v, partials, counter, out);
  return check_launch("cfl2d");
}

}  // namespace d2
}  // namespace lsg
