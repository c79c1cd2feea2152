// 2D kernels of liblsgpu: operator apply and the single-pass PCG iteration
// (warp marching, see march2d.cuh), fused compliance + shape-derivative RHS,
// velocity statistics and material words.
#include <math.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include "march2d_ops.cuh"
#include "ops.h"

namespace lsg {
namespace d2 {

constexpr int kEwThreads = 256;

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

// Launch geometry.  The marching kernels run as (about) one wave: the number
// of row segments is chosen so that cta_columns * segments * k fills the
// resident CTA slots of the 148 SMs (occupancy queried per kernel), which
// keeps the one-halo-row-per-segment overhead small on large grids and avoids
// a tail wave on small ones.
constexpr int kMaxPartials = 4096;  // >= CTAs per rhs of any launch below

static int seg_for(const Geo &g, int k, int ctas_per_sm, int nstrips = -1) {
  const int64_t cols = ceil_div(nstrips < 0 ? nstrips_of(g) : nstrips, kWarps);
  const int64_t rows = g.ny + 1;
  int64_t slots = (int64_t)num_sms() * (ctas_per_sm > 0 ? ctas_per_sm : 4);
  int64_t nseg = slots / (cols * k);
  if (nseg < 1) nseg = 1;
  int64_t seg = ceil_div(rows, nseg);
  if (seg < 4) seg = 4;
  while (cols * ceil_div(rows, seg) > kMaxPartials) seg *= 2;
  return (int)seg;
}

static dim3 march_grid(const Geo &g, int seg, int k) {
  return dim3((unsigned)ceil_div(nstrips_of(g), kWarps), (unsigned)ceil_div(g.ny + 1, seg),
              (unsigned)k);
}

int64_t partials_per_rhs(const lsg_grid &) { return kMaxPartials; }

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

static Lap make_lap(const Geo &g, const lsg_op &op) {
  const double eps = op.p[0], inside = op.p[1] > 0.0 ? op.p[1] : 1.0;
  const double area = 0.5 * g.hx * g.hy;
  Lap l;
  l.w0 = area * eps;
  l.w1 = area * (inside - eps) / 3.0;
  l.ihx2 = 1.0 / (g.hx * g.hx);
  l.ihy2 = 1.0 / (g.hy * g.hy);
  return l;
}

// components per node of the operator's fields
static int nc_of(const lsg_op &op) { return op.kind == LSG_OP_LAPLACE ? 1 : 2; }

template <class PH, int ACT>
static int launch_march(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  static int ctas_per_sm = -1;
  if (ctas_per_sm < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, march<PH, ACT, uint8_t>,
                                                      kThreads, 0) != cudaSuccess)
      ctas_per_sm = 4;
  }
  a.seg = seg_for(g, k, ctas_per_sm);
  a.nstrips = nstrips_of(g);
  const dim3 grid = march_grid(g, a.seg, k);
  march<PH, ACT, uint8_t><<<grid, kThreads, 0, st>>>(ph, g, a);
  return check_launch("march2d");
}

// The recompute-q PCG pass (march_pcg_rqs): 28-column strips, its own
// occupancy-sized grid.  LSG_PCG2D_RQ=0 keeps the stored-q pass (march_pcg);
// LSG_RQ_AHEAD=2|3 overrides the prefetch depth.
static bool pcg_rq_on() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_PCG2D_RQ");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <class PH, int A, bool FIRST>
static int launch_pcg_rq_hint(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  static int ctas_per_sm = -1;
  if (ctas_per_sm < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, march_pcg_rqs_kernel<PH, A, FIRST>,
                                                      kThreads, 0) != cudaSuccess)
      ctas_per_sm = 4;
  }
  a.nstrips = (int)ceil_div(g.nx + 1, kStripRq);
  a.seg = seg_for(g, k, ctas_per_sm, a.nstrips);
  const dim3 grid((unsigned)ceil_div(a.nstrips, kWarps), (unsigned)ceil_div(g.ny + 1, a.seg),
                  (unsigned)k);
  if (launch_pdl(march_pcg_rqs_kernel<PH, A, FIRST>, grid, dim3(kThreads), 0, st, ph, g, a) != cudaSuccess)
    return check_launch("march2d_pcg_rq launch");
  return check_launch("march2d_pcg_rq");
}

template <class PH, int A>
static int launch_pcg_rq(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  // evict-first copies of the dead r_{i-1}, p_{i-1} (march_pcg_rqs): for batches whose six
  // vectors overflow L2 while the two new ones fit in it with room to spare.  Measured
  // (off -> on): cfg2 1024x256 k=8 49.9 -> 46.9 us, 1024x512 k=4 50.5 -> 48.2, k=6 38.8 ->
  // 38.2; outside the band it loses (k=10 62.9 -> 66.1, k=12 73.3 -> 78.4, cfg4 176 -> 196),
  // and so does a single field of the same size (2048x1024 k=1 49.9 -> 52.4).
  const int64_t vec = (int64_t)k * (g.nx + 1) * (g.ny + 1) * PH::NC * 8;
  const bool first = k >= 4 && 6 * vec > l2_bytes() && 10 * vec <= 3 * l2_bytes();
  return first ? launch_pcg_rq_hint<PH, A, true>(ph, g, a, k, st)
               : launch_pcg_rq_hint<PH, A, false>(ph, g, a, k, st);
}

template <class PH>
static int launch_pcg_rq_depth(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  static int forced = -1;
  if (forced < 0) {
    const char *e = getenv("LSG_RQ_AHEAD");
    forced = e ? atoi(e) : 0;
  }
  // measured: 3 rows ahead pays only on small batched grids (cfg2 1024x256 k=8:
  // 51.6 vs 52.5 us); 2 elsewhere (4096x2048 k=1: 183 vs 198; 2048x1024 k=2: 94 vs 98)
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const int depth = (forced == 2 || forced == 3) ? forced : (k > 1 && nn < (1 << 20) ? 3 : 2);
  return depth == 3 ? launch_pcg_rq<PH, 3>(ph, g, a, k, st) : launch_pcg_rq<PH, 2>(ph, g, a, k, st);
}

static int dispatch_pcg_rq(const lsg_op &op, MArgs a, int k, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  if (op.kind == LSG_OP_ELASTICITY) return launch_pcg_rq_depth<Elast>(make_elast(g, op), g, a, k, st);
  if (op.kind == LSG_OP_H1) return launch_pcg_rq_depth<H1>(make_h1(g, op), g, a, k, st);
  if (op.kind == LSG_OP_LAPLACE) return launch_pcg_rq_depth<Lap>(make_lap(g, op), g, a, k, st);
  set_error("unknown operator kind %d", op.kind);
  return LSG_ERR_ARG;
}

template <int ACT>
static int dispatch_op(const lsg_op &op, MArgs a, int k, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  if (op.kind == LSG_OP_ELASTICITY) return launch_march<Elast, ACT>(make_elast(g, op), g, a, k, st);
  if (op.kind == LSG_OP_H1) return launch_march<H1, ACT>(make_h1(g, op), g, a, k, st);
  if (op.kind == LSG_OP_LAPLACE) return launch_march<Lap, ACT>(make_lap(g, op), g, a, k, st);
  set_error("unknown operator kind %d", op.kind);
  return LSG_ERR_ARG;
}

// The apply with a shared-memory prefetch ring (apply_s_kernel); LSG_APPLY_SMEM=0
// keeps the register-ring march.
static bool apply_s_on() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_APPLY_SMEM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <class PH>
static int launch_apply_s(const PH &ph, const Geo &g, MArgs a, int k, cudaStream_t st) {
  static int ctas_per_sm = -1;
  if (ctas_per_sm < 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                             &ctas_per_sm, apply_s_kernel<PH>, kThreads, 0) != cudaSuccess)
    ctas_per_sm = 4;
  a.seg = seg_for(g, k, ctas_per_sm);
  a.nstrips = nstrips_of(g);
  const dim3 grid = march_grid(g, a.seg, k);
  apply_s_kernel<PH><<<grid, kThreads, 0, st>>>(ph, g, a);
  return check_launch("apply_s2d");
}

// Two fields per warp for batched elasticity applies (L2 flushed: cfg2 k = 8
// 23.5 -> 22.5 us, 2048x1024 k = 2 39.0 -> 35.8 us); LSG_APPLY2=0 keeps one.
static bool apply2_on() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_APPLY2");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int apply(const lsg_op &op, int k, const double *x, double *y, cudaStream_t st) {
  MArgs a = {};
  a.words = op.words;
  a.x = x;
  a.y = y;
  // even k only: an odd batch would carry a duplicate field (measured slower at k = 3)
  if (op.kind == LSG_OP_ELASTICITY && k >= 2 && k % 2 == 0 && apply2_on()) {
    const Geo g = geo_of(op.grid);
    static int ctas_per_sm = -1;
    if (ctas_per_sm < 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                               &ctas_per_sm, apply2_kernel, kThreads, 0) != cudaSuccess)
      ctas_per_sm = 4;
    const int kp = (k + 1) / 2;
    a.seg = seg_for(g, kp, ctas_per_sm);
    a.nstrips = nstrips_of(g);
    const dim3 grid = march_grid(g, a.seg, kp);
    apply2_kernel<<<grid, kThreads, 0, st>>>(make_elast(g, op), g, a, k);
    return check_launch("apply2_2d");
  }
  if (k == 1 && apply_s_on()) {  // measured: cfg4 67.5 -> 65.5 us; batched fields do better
                                 // with apply2 (even k) or the register ring (odd k)
    const Geo g = geo_of(op.grid);
    if (op.kind == LSG_OP_ELASTICITY) return launch_apply_s<Elast>(make_elast(g, op), g, a, k, st);
    if (op.kind == LSG_OP_H1) return launch_apply_s<H1>(make_h1(g, op), g, a, k, st);
    if (op.kind == LSG_OP_LAPLACE) return launch_apply_s<Lap>(make_lap(g, op), g, a, k, st);
  }
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
  constexpr int NC = PH::NC;
  double dg[NC];
  node_diag<PH>(ph, w00, wm0, w0m, wmm, i, j, dg);
  const uint32_t m = PH::mask(w00);
#pragma unroll
  for (int c = 0; c < NC; ++c) d[node * NC + c] = ((m >> c) & 1u) ? 1.0 : dg[c];
}

__global__ void reciprocal_kernel(int64_t n, double *d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) d[t] = fabs(d[t]) > 0.0 ? 1.0 / d[t] : 1.0;  // fem.py:303-305 'safe'
}

int inv_diag(const lsg_op &op, double *d, cudaStream_t st) {
  int rc = diag(op, d, st);
  if (rc) return rc;
  const Geo g = geo_of(op.grid);
  const int64_t n = nc_of(op) * (int64_t)(g.nx + 1) * (g.ny + 1);
  reciprocal_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(n, d);
  return check_launch("inv_diag2d");
}

int diag(const lsg_op &op, double *d, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const unsigned nb = (unsigned)ceil_div(nn, kEwThreads);
  const uint8_t *w = static_cast<const uint8_t *>(op.words);
  if (op.kind == LSG_OP_ELASTICITY) diag_kernel<Elast><<<nb, kEwThreads, 0, st>>>(make_elast(g, op), g, w, d);
  else if (op.kind == LSG_OP_H1) diag_kernel<H1><<<nb, kEwThreads, 0, st>>>(make_h1(g, op), g, w, d);
  else if (op.kind == LSG_OP_LAPLACE) diag_kernel<Lap><<<nb, kEwThreads, 0, st>>>(make_lap(g, op), g, w, d);
  else { set_error("unknown operator kind %d", op.kind); return LSG_ERR_ARG; }
  return check_launch("diag2d");
}

int pcg_start(const lsg_op &op, lsg_pcg_ws &ws, double rtol, double atol, double maxiter,
              cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t n = nc_of(op) * (int64_t)(g.nx + 1) * (g.ny + 1);
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
  a.dinv = ws.dinv;
  rc = dispatch_op<RESID>(op, a, ws.k, st);
  if (rc) return rc;
  // p_{-1} = 0 (the buffer the first pass reads as p_{i-1}): with alpha_{-1} =
  // beta_0 = 0 the recompute pass needs no first-iteration branch
  if (cudaMemsetAsync(ws.p, 0, sizeof(double) * (size_t)n * ws.k, st) != cudaSuccess)
    return check_launch("memset p");
  zero_if_flag<<<dim3(64, ws.k), 256, 0, st>>>(n, ws.scal, ws.x);
  return check_launch("zero_if_flag");
}


// ----------------------------------------------------------------------------
// Persistent PCG (2D): all `niter` single-pass iterations in one cooperative
// launch, one grid-wide barrier per iteration instead of one kernel boundary.
// Every CTA keeps the per-RHS scalars in shared memory and reduces the per-CTA
// partials itself in one fixed order, so all CTAs take identical decisions
// (deterministic results); CTA 0 mirrors the scalars to global memory.  Same
// algorithm and stopping rule as march<.., PCG> (pcg_decide).  The partials
// alternate between two buffers by iteration: a CTA still reading iteration
// i's sums cannot be overtaken by a writer of iteration i+2 (barrier i+1).
// ----------------------------------------------------------------------------
namespace cgrp = cooperative_groups;

constexpr int kPcgSums = Traits<Elast, PCG>::NP;  // p.q, z.q, q.M^-1 q, r.z, r.r

template <class PH, int KMAX>
__global__ void __launch_bounds__(kThreads)
    pcg_persistent(PH ph, Geo g, MArgs a, int k, int tx, int ty, int niter, int parity0,
                   double *r_even, double *r_odd, double *p_even, double *p_odd, double *q_even,
                   double *q_odd, double *pbuf) {
  constexpr int NS = kPcgSums;
  constexpr int G = KMAX >= 2 ? 2 : 1;  // right-hand sides per block reduction
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double scratch[NS * G * kWarps];
  __shared__ lsg_pcg_scalars s_sc[KMAX];
  __shared__ double s_part[KMAX * NS];
  __shared__ int s_all;
  const int ncta = gridDim.x, cta = blockIdx.x;
  for (int t = threadIdx.x; t < KMAX; t += kThreads) {
    if (t < k) s_sc[t] = a.scal[t];
    else s_sc[t].done = 1.0;
  }
  __syncthreads();
  int parity = parity0;
  const int ntask = tx * ty * k;
  for (int it = 0; it < niter; ++it, parity ^= 1) {
    if (threadIdx.x == 0) {
      int all = 1;
      for (int r = 0; r < KMAX; ++r) all &= s_sc[r].done != 0.0;
      s_all = all;
    }
    for (int t = threadIdx.x; t < KMAX * NS; t += kThreads) s_part[t] = 0.0;
    __syncthreads();
    if (s_all) break;  // identical in every CTA: no barrier is skipped by only some
    MArgs aa = a;
    aa.x = parity ? r_odd : r_even;  // r_{i-1}
    aa.y3 = parity ? r_even : r_odd;  // r_i
    aa.x2 = parity ? p_odd : p_even;
    aa.y2 = parity ? p_even : p_odd;
    aa.x3 = parity ? q_odd : q_even;
    aa.y = parity ? q_even : q_odd;
    for (int t = cta; t < ntask; t += ncta) {
      const int rhs = t / (tx * ty), rem = t - rhs * (tx * ty);
      const lsg_pcg_scalars &sc = s_sc[rhs];
      if (sc.done != 0.0) continue;
      double part[NS];
#pragma unroll
      for (int v = 0; v < NS; ++v) part[v] = 0.0;
      march_pcg<PH, true>(ph, g, aa, rem % tx, rem / tx, rhs, sc.first != 0.0, sc.beta, sc.alpha,
                          part);
      block_reduce<NS, 0u>(part, scratch);
      if (threadIdx.x == 0)
#pragma unroll
        for (int v = 0; v < NS; ++v) s_part[rhs * NS + v] += part[v];
      __syncthreads();
    }
    double *pw = pbuf + (size_t)(it & 1) * ncta * KMAX * NS;
    for (int t = threadIdx.x; t < KMAX * NS; t += kThreads) pw[(size_t)cta * KMAX * NS + t] = s_part[t];
    grid.sync();
    // every CTA: the same fixed-order sums over all CTAs, then the same decisions
    for (int r0 = 0; r0 < k; r0 += G) {
      double acc[G * NS];
#pragma unroll
      for (int v = 0; v < G * NS; ++v) acc[v] = 0.0;
      for (int c = threadIdx.x; c < ncta; c += kThreads)
#pragma unroll
        for (int v = 0; v < G * NS; ++v)
          if (r0 * NS + v < KMAX * NS) acc[v] += __ldcg(pw + (size_t)c * KMAX * NS + r0 * NS + v);
      block_reduce<G * NS, 0u>(acc, scratch);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const int r = r0 + gg;
          if (r >= k || s_sc[r].done != 0.0) continue;
          pcg_decide(s_sc[r], acc + gg * NS);
          if (cta == 0) a.scal[r] = s_sc[r];
        }
      }
      __syncthreads();
    }
  }
}

// ----------------------------------------------------------------------------
// Cluster PCG for the smallest systems (<= kClusterCtas * kTasksPerCta marching
// tasks, e.g. cfg1): one thread-block cluster of 16 CTAs runs every iteration
// of a chunk.  Each CTA holds 3 tasks (12 warps); per iteration the warps' sums
// are combined in fixed order in shared memory, the 16 CTA sums are read by
// every CTA through distributed shared memory in rank order (same totals, same
// decisions everywhere) and one cluster barrier per iteration replaces the
// grid-wide barrier and the global partials of the cooperative kernel.  The
// CTA sums alternate between two buffers by iteration (a CTA that runs ahead
// cannot overwrite sums another CTA is still reading).  Data written in one
// iteration and read (halo) by other CTAs in the next is ordered by the
// barrier's release/acquire at cluster scope.
// ----------------------------------------------------------------------------
constexpr int kClusterCtas = 16;
constexpr int kTasksPerCta = 3;

template <class PH, int KMAX>
__global__ void __launch_bounds__(kThreads * kTasksPerCta, 1)
    pcg_cluster(PH ph, Geo g, MArgs a, int k, int tx, int ty, int niter, int parity0,
                double *r_even, double *r_odd, double *p_even, double *p_odd, double *q_even,
                double *q_odd) {
  constexpr int NS = kPcgSums;
  constexpr int NW = kWarps * kTasksPerCta;
  constexpr int NV = KMAX * NS;
  cgrp::cluster_group cl = cgrp::this_cluster();
  __shared__ double s_warp[NW][NV];
  __shared__ double s_cta[2][NV];
  __shared__ lsg_pcg_scalars s_sc[KMAX];
  __shared__ int s_all;
  const int rank = (int)cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = warp / kWarps, wt = warp % kWarps;
  for (int t = threadIdx.x; t < KMAX; t += blockDim.x) {
    if (t < k) s_sc[t] = a.scal[t];
    else s_sc[t].done = 1.0;
  }
  __syncthreads();
  int parity = parity0;
  const int ntask = tx * ty * k;
  const int nslot = kClusterCtas * kTasksPerCta;
  for (int it = 0; it < niter; ++it, parity ^= 1) {
    if (threadIdx.x == 0) {
      int all = 1;
      for (int r = 0; r < KMAX; ++r) all &= s_sc[r].done != 0.0;
      s_all = all;
    }
    for (int t = threadIdx.x; t < NW * NV; t += blockDim.x) (&s_warp[0][0])[t] = 0.0;
    __syncthreads();
    if (s_all) break;  // identical in every CTA of the cluster
    MArgs aa = a;
    aa.x = parity ? r_odd : r_even;
    aa.y3 = parity ? r_even : r_odd;
    aa.x2 = parity ? p_odd : p_even;
    aa.y2 = parity ? p_even : p_odd;
    aa.x3 = parity ? q_odd : q_even;
    aa.y = parity ? q_even : q_odd;
    for (int t = rank * kTasksPerCta + slot; t < ntask; t += nslot) {
      const int rhs = t / (tx * ty), rem = t - rhs * (tx * ty);
      const lsg_pcg_scalars &sc = s_sc[rhs];
      if (sc.done != 0.0) continue;  // uniform across the task's warps
      double part[NS];
#pragma unroll
      for (int v = 0; v < NS; ++v) part[v] = 0.0;
      march_pcg<PH, true>(ph, g, aa, rem % tx, rem / tx, rhs, sc.first != 0.0, sc.beta, sc.alpha,
                          part, wt);
#pragma unroll
      for (int v = 0; v < NS; ++v) {
        const double w = warp_sum(part[v]);
        if (lane == 0) s_warp[warp][rhs * NS + v] += w;
      }
    }
    __syncthreads();
    double *mine = s_cta[it & 1];
    for (int v = threadIdx.x; v < NV; v += blockDim.x) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w) acc += s_warp[w][v];
      mine[v] = acc;
    }
    cl.sync();  // every CTA's sums (and this iteration's vectors) are published
    if (threadIdx.x < NV) {
      double tot = 0.0;
      for (int c = 0; c < kClusterCtas; ++c) tot += cl.map_shared_rank(mine, c)[threadIdx.x];
      s_warp[0][threadIdx.x] = tot;  // reuse: totals per (rhs, sum)
    }
    __syncthreads();
    if (threadIdx.x < KMAX) {
      const int r = threadIdx.x;
      if (r < k && s_sc[r].done == 0.0) {
        pcg_decide(s_sc[r], &s_warp[0][r * NS]);
        if (rank == 0) a.scal[r] = s_sc[r];
      }
    }
    __syncthreads();
  }
  cl.sync();  // no CTA exits while another may still read its shared memory
}

template <class PH, int KMAX>
static int launch_cluster_k(const PH &ph, const Geo &g, MArgs a, lsg_pcg_ws &ws, int niter,
                            cudaStream_t st) {
  static int ok = -1;
  if (ok < 0) {
    ok = 0;
    if (cudaFuncSetAttribute(pcg_cluster<PH, KMAX>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kClusterCtas);
      cfg.blockDim = dim3(kThreads * kTasksPerCta);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kClusterCtas;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, pcg_cluster<PH, KMAX>, &cfg) == cudaSuccess &&
          nclusters >= 1)
        ok = 1;
    }
    cudaGetLastError();  // a failed probe (no 16-CTA cluster fits) only selects the fallback
  }
  if (!ok) return 1;
  a.nstrips = nstrips_of(g);
  a.seg = seg_for(g, ws.k, 3);
  const dim3 mg = march_grid(g, a.seg, ws.k);
  const int k = ws.k, tx = (int)mg.x, ty = (int)mg.y, parity = ws.parity;
  double *re = ws.r, *ro = ws.r_alt, *pe = ws.p, *po = ws.p_alt, *qe = ws.q, *qo = ws.q_alt;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCtas);
  cfg.blockDim = dim3(kThreads * kTasksPerCta);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kClusterCtas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, pcg_cluster<PH, KMAX>, ph, g, a, k, tx, ty, niter, parity, re, ro, pe, po,
                         qe, qo) != cudaSuccess)
    return check_launch("pcg_cluster");
  ws.parity ^= (niter & 1);
  return check_launch("pcg_cluster");
}

// LSG_PCG2D_CLUSTER=0 keeps the cooperative persistent kernel for small systems.
static bool cluster_on() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_PCG2D_CLUSTER");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// 1 = not applicable (too many tasks, or no cluster of 16 fits): use another path
template <class PH>
static int launch_cluster(const PH &ph, const Geo &g, MArgs a, lsg_pcg_ws &ws, int niter,
                          cudaStream_t st) {
  if (!cluster_on()) return 1;
  const int seg = seg_for(g, ws.k, 3);
  const dim3 mg = march_grid(g, seg, ws.k);
  if ((int64_t)mg.x * mg.y * ws.k > (int64_t)kClusterCtas * kTasksPerCta) return 1;
  if (ws.k == 1) return launch_cluster_k<PH, 1>(ph, g, a, ws, niter, st);
  if (ws.k <= 4) return launch_cluster_k<PH, 4>(ph, g, a, ws, niter, st);
  if (ws.k <= 8) return launch_cluster_k<PH, 8>(ph, g, a, ws, niter, st);
  return 1;
}

// LSG_PCG2D_PERSISTENT=0 keeps the two-kernel (graph-replayed) iteration.
static bool persistent_on() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_PCG2D_PERSISTENT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <class PH, int KMAX>
static int launch_persistent_k(const PH &ph, const Geo &g, MArgs a, lsg_pcg_ws &ws, int niter,
                               cudaStream_t st) {
  static int per_sm = -1;
  if (per_sm < 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_persistent<PH, KMAX>, kThreads,
                                                    0) != cudaSuccess)
    per_sm = 0;
  if (per_sm <= 0) return 1;  // not launchable cooperatively: caller falls back
  static int ctas_march = -1;
  if (ctas_march < 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_march, march<PH, PCG, uint8_t>,
                                                    kThreads, 0) != cudaSuccess)
    ctas_march = 4;
  a.seg = seg_for(g, ws.k, ctas_march);
  {
    // (short tasks win on small grids -- cfg1: 4 rows 7.0 us, 8 rows 8.6, 16 rows
    // 11.7: the per-iteration barrier and reductions are cheaper than a longer march)
    // mid-size systems: 8-row tasks while that still gives every SM one (velocity
    // solve of cfg2, 1024x256: 14.5 -> 13.2 us; 512x256: 12.3 -> 10.8 us); with fewer
    // tasks the longer march costs more than the barriers it saves (320x160: 7.9 vs 9.1)
    if (a.seg < 8) {
      const dim3 m8 = march_grid(g, 8, ws.k);
      if ((int64_t)m8.x * m8.y * ws.k >= num_sms()) a.seg = 8;
    }
  }
  a.nstrips = nstrips_of(g);
  const dim3 mg = march_grid(g, a.seg, ws.k);
  const int ntask = (int)(mg.x * mg.y * ws.k);
  // one task per CTA (cfg1 PCG iteration 7.9 -> 7.0 us against filling every SM:
  // fewer partials to reduce and CTAs to barrier)
  int ncta = ntask;
  if (ncta > per_sm * num_sms()) ncta = per_sm * num_sms();
  int k = ws.k, tx = (int)mg.x, ty = (int)mg.y, parity = ws.parity;
  double *re = ws.r, *ro = ws.r_alt, *pe = ws.p, *po = ws.p_alt, *qe = ws.q, *qo = ws.q_alt;
  double *pbuf = ws.partials;
  PH phc = ph;
  Geo gc = g;
  void *args[] = {&phc, &gc, &a, &k, &tx, &ty, &niter, &parity, &re, &ro, &pe, &po, &qe, &qo, &pbuf};
  const cudaError_t le = cudaLaunchCooperativeKernel((void *)pcg_persistent<PH, KMAX>, dim3((unsigned)ncta),
                                                     dim3(kThreads), args, 0, st);
  if (le == cudaErrorCooperativeLaunchTooLarge) {  // e.g. a partitioned device: caller falls back
    cudaGetLastError();
    return 1;
  }
  if (le != cudaSuccess) return check_launch("pcg_persistent");
  ws.parity ^= (niter & 1);
  return check_launch("pcg_persistent");
}

template <class PH>
static int launch_persistent(const PH &ph, const Geo &g, MArgs a, lsg_pcg_ws &ws, int niter,
                             cudaStream_t st) {
  if (ws.k == 1) return launch_persistent_k<PH, 1>(ph, g, a, ws, niter, st);
  if (ws.k <= 4) return launch_persistent_k<PH, 4>(ph, g, a, ws, niter, st);
  return launch_persistent_k<PH, 8>(ph, g, a, ws, niter, st);
}

// Small systems only: there the two kernel boundaries per iteration dominate;
// on large ones the work does and the grid barriers + cross-CTA reductions
// would cost more than the launches they replace (cfg2: 112 vs 59 us).
bool pcg_persistent_ok(const lsg_op &op, const lsg_pcg_ws &ws) {
  constexpr int64_t limit = 600000;  // dofs x rhs (cfg1 and the velocity solves: yes; cfg2 state: no)
  if (!persistent_on() || ws.k > 8 || op.grid.dim != 2) return false;
  if (op.kind != LSG_OP_ELASTICITY && op.kind != LSG_OP_H1 && op.kind != LSG_OP_LAPLACE) return false;
  const int64_t nn = (int64_t)(op.grid.n[0] + 1) * (op.grid.n[1] + 1);
  return nn * nc_of(op) * ws.k <= limit;
}

int pcg_iterate(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  MArgs a = {};
  a.words = op.words;
  a.x = ws.r;
  a.y = ws.q;
  a.scal = ws.scal;
  a.partials = ws.partials;
  a.counters = ws.counters;
  a.dinv = ws.dinv;
  a.xs = ws.x;
  if (pcg_persistent_ok(op, ws)) {
    int rc = 1;
    if (op.kind == LSG_OP_ELASTICITY) rc = launch_cluster<Elast>(make_elast(g, op), g, a, ws, niter, st);
    else if (op.kind == LSG_OP_H1) rc = launch_cluster<H1>(make_h1(g, op), g, a, ws, niter, st);
    else rc = launch_cluster<Lap>(make_lap(g, op), g, a, ws, niter, st);
    if (rc <= 0) return rc;
    if (op.kind == LSG_OP_ELASTICITY) rc = launch_persistent<Elast>(make_elast(g, op), g, a, ws, niter, st);
    else if (op.kind == LSG_OP_H1) rc = launch_persistent<H1>(make_h1(g, op), g, a, ws, niter, st);
    else rc = launch_persistent<Lap>(make_lap(g, op), g, a, ws, niter, st);
    if (rc <= 0) return rc;  // launched (0) or failed (< 0); 1 = not cooperative, fall through
  }
  for (int it = 0; it < niter; ++it) {
    const bool odd = ws.parity != 0;
    a.x = odd ? ws.r_alt : ws.r;  // r, p, q of the previous iteration ...
    a.x2 = odd ? ws.p_alt : ws.p;
    a.x3 = odd ? ws.q_alt : ws.q;
    a.y3 = odd ? ws.r : ws.r_alt;  // ... and of this one
    a.y2 = odd ? ws.p : ws.p_alt;
    a.y = odd ? ws.q : ws.q_alt;
    int rc = pcg_rq_on() ? dispatch_pcg_rq(op, a, ws.k, st) : dispatch_op<PCG>(op, a, ws.k, st);
    if (rc) return rc;
    ws.parity ^= 1;
  }
  return LSG_OK;
}

// The single-pass iteration leaves nothing pending in 2D: x_i is formed in the
// pass that tests r_i, so a right-hand side stops with its final x.
int pcg_finish(const lsg_op &, lsg_pcg_ws &, cudaStream_t) { return LSG_OK; }

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

template <int KB>
static int heat_chunk(const Geo &g, const lsg_op &op, const double *u, const double *cw,
                      const double *fq, const double *gq, double volume, double *vc, double *vv,
                      double *out, double *partials, uint32_t *counter, int chunk, cudaStream_t st) {
  HeatShape<KB> ph;
  const double area = 0.5 * g.hx * g.hy;
  const double eps = op.p[0], inside = op.p[1] > 0.0 ? op.p[1] : 1.0;
  ph.nx = g.nx;
  ph.area = area;
  ph.inv_hx = 1.0 / g.hx;
  ph.inv_hy = 1.0 / g.hy;
  ph.inv_volume = 1.0 / volume;
  ph.w0 = area * eps;
  ph.w1 = area * (inside - eps) / 3.0;
  for (int t = 0; t < KB; ++t) ph.cw[t] = cw[t];
  ph.fq = fq;
  ph.gq = gq;
  ph.ecount = 2 * (int64_t)g.nx * g.ny;
  MArgs a = {};
  a.words = op.words;
  a.x = u;
  a.y = vc;
  a.y2 = vv;
  a.out = out;
  a.partials = partials;
  a.counters = counter;
  a.accumulate = chunk > 0;
  return launch_march<HeatShape<KB>, SHAPE>(ph, g, a, 1, st);
}

int heat_shape(const lsg_op &op, int k, const double *u, const double *weights, const double *fq,
               const double *gq, double volume, double *vc, double *vv, double *out,
               double *partials, uint32_t *counter, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  const int64_t ne = 2 * (int64_t)g.nx * g.ny;
  int done = 0, chunk = 0;
  while (done < k) {
    const int kb = (k - done) >= 2 ? 2 : 1;
    const double *uc = u + (size_t)done * nn;
    const double *fc = fq + (size_t)done * ne * 3;
    const double *gc = gq ? gq + (size_t)done * ne * 6 : nullptr;
    const int rc = kb == 2 ? heat_chunk<2>(g, op, uc, weights + done, fc, gc, volume, vc, vv, out,
                                           partials, counter, chunk, st)
                           : heat_chunk<1>(g, op, uc, weights + done, fc, gc, volume, vc, vv, out,
                                           partials, counter, chunk, st);
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
