// The reference's own level-set scheme on the device, 2D:
// Crank-Nicolson Petrov-Galerkin transport (levelset.py:137-169) and the
// Petrov-Galerkin Euler/AB2 reinitialisation (levelset.py:172-216), matrix-
// free.  The step matrices are non-symmetric, so they are solved with a
// right-Jacobi-preconditioned BiCGStab to a tight tolerance (they stand in
// for the reference's SuperLU).
//
// Operators (lsg_op kinds):
//   LSG_OP_PG_TRANSPORT  A = m_hat + sign dt half  (p0 dt, p1 h, p2 sign, p3 smooth),
//                        aux[0] = theta (2 N)
//   LSG_OP_PG_REINIT     A = m_hat(direction of grad aux[1]), s from aux[0] = phi0
//                        (p0 dt, p1 h); lsg_pg_reinit_rhs also reads aux[2] = previous iterate
// Element quantities (per triangle, edge-midpoint rule, weights |T|/3):
//   hat_qa = bary_qa + tau_q (v_q . grad N_a),  m_hat_ab = sum_q w hat_qa bary_qb,
//   half_ab = 1/2 sum_q w hat_qa (v_q . grad N_b) [+ 1/2 h^2 |T| grad N_a . grad N_b].
// Kernels gather, per node, the row of every incident triangle (6 of them):
// one thread per node, fixed summation order, no atomics.
#include <math.h>

#include <vector>

#include "common.cuh"
#include "ops.h"

namespace lsg {
namespace pg {

struct Geo {
  int nx, ny;
  double hx, hy, area;
};

static Geo geo_of(const lsg_grid &g) {
  Geo o;
  o.nx = g.n[0];
  o.ny = g.n[1];
  o.hx = (g.hi[0] - g.lo[0]) / g.n[0];
  o.hy = (g.hi[1] - g.lo[1]) / g.n[1];
  o.area = 0.5 * o.hx * o.hy;
  return o;
}

__device__ __constant__ double kBary[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};

// The 6 triangles around node (i, j): cell offset, lower(0)/upper(1), local index.
struct Inc {
  int di, dj, t, a;
};
__device__ __constant__ Inc kInc[6] = {{0, 0, 0, 0}, {0, 0, 1, 0}, {-1, 0, 0, 1},
                                       {-1, -1, 0, 2}, {-1, -1, 1, 1}, {0, -1, 1, 2}};

// Node ids and gradients of triangle (cell ci, cj, type t).
__device__ __forceinline__ void tri_nodes(const Geo &g, int ci, int cj, int t, int64_t *nd,
                                          double (*gr)[2]) {
  const int64_t nxp = g.nx + 1;
  const int64_t n00 = (int64_t)cj * nxp + ci, n10 = n00 + 1, n01 = n00 + nxp, n11 = n01 + 1;
  const double ix = 1.0 / g.hx, iy = 1.0 / g.hy;
  if (t == 0) {  // lower (00, 10, 11)
    nd[0] = n00; nd[1] = n10; nd[2] = n11;
    gr[0][0] = -ix; gr[0][1] = 0.0;
    gr[1][0] = ix;  gr[1][1] = -iy;
    gr[2][0] = 0.0; gr[2][1] = iy;
  } else {       // upper (00, 11, 01)
    nd[0] = n00; nd[1] = n11; nd[2] = n01;
    gr[0][0] = 0.0; gr[0][1] = -iy;
    gr[1][0] = ix;  gr[1][1] = 0.0;
    gr[2][0] = -ix; gr[2][1] = iy;
  }
}

__device__ __forceinline__ double tau_of(double speed_sq, double dt, double h) {
  return 0.5 / sqrt(1.0 / (dt * dt) + speed_sq / (h * h));
}

// gradient_norm_guard (levelset.py:109-118)
__device__ __forceinline__ void guard(const double *p, double *d) {
  const double mag = sqrt(p[0] * p[0] + p[1] * p[1]);
  const double eps = 1e-12 * (1.0 + mag);
  const double s = sqrt(mag * mag + eps * eps);
  d[0] = p[0] / s;
  d[1] = p[1] / s;
}

struct OpArgs {
  int kind;
  double dt, h, sign;
  int smooth;
  const double *theta, *phi0, *cur, *prev;
};

// velocity at the quadrature points of one triangle and the row-a entries of
// m_hat (M[b]) and half (H[b]); also hat_qa (for the reinit load)
__device__ void element_row(const Geo &g, const OpArgs &o, const int64_t *nd, double (*gr)[2],
                            int a, double *M, double *H, double *hat_a, double *sq) {
  double vq[3][2], tq[3];
  if (o.kind == LSG_OP_PG_TRANSPORT) {
    double th[3][2];
    for (int v = 0; v < 3; ++v) {
      th[v][0] = o.theta[nd[v] * 2];
      th[v][1] = o.theta[nd[v] * 2 + 1];
    }
    for (int q = 0; q < 3; ++q) {
      for (int c = 0; c < 2; ++c)
        vq[q][c] = kBary[q][0] * th[0][c] + kBary[q][1] * th[1][c] + kBary[q][2] * th[2][c];
      tq[q] = tau_of(vq[q][0] * vq[q][0] + vq[q][1] * vq[q][1], o.dt, o.h);
    }
  } else {
    // frozen smoothed sign at the quadrature points, direction of grad(cur)
    double p0[3], pc[3];
    for (int v = 0; v < 3; ++v) {
      p0[v] = o.phi0[nd[v]];
      pc[v] = o.cur[nd[v]];
    }
    double gc[2] = {0.0, 0.0};
    for (int v = 0; v < 3; ++v) {
      gc[0] += gr[v][0] * pc[v];
      gc[1] += gr[v][1] * pc[v];
    }
    double dir[2];
    guard(gc, dir);
    for (int q = 0; q < 3; ++q) {
      double s = kBary[q][0] * p0[0] + kBary[q][1] * p0[1] + kBary[q][2] * p0[2];
      s = s / sqrt(s * s + o.h * o.h);
      sq[q] = s;
      tq[q] = tau_of(s * s, o.dt, o.h);
      vq[q][0] = s * dir[0];
      vq[q][1] = s * dir[1];
    }
  }
  const double w = g.area / 3.0;
  for (int b = 0; b < 3; ++b) M[b] = H[b] = 0.0;
  for (int q = 0; q < 3; ++q) {
    double conv[3];
    for (int v = 0; v < 3; ++v) conv[v] = vq[q][0] * gr[v][0] + vq[q][1] * gr[v][1];
    const double hat = kBary[q][a] + tq[q] * conv[a];
    hat_a[q] = hat;
    for (int b = 0; b < 3; ++b) {
      M[b] += w * hat * kBary[q][b];
      H[b] += 0.5 * w * hat * conv[b];
    }
  }
  if (o.kind == LSG_OP_PG_TRANSPORT && o.smooth) {
    for (int b = 0; b < 3; ++b)
      H[b] += 0.5 * o.h * o.h * g.area * (gr[a][0] * gr[b][0] + gr[a][1] * gr[b][1]);
  }
}

// mode 0: y = A x ; mode 1: y = diag(A) ; mode 2: reinit right-hand side
__global__ void gather_kernel(Geo g, OpArgs o, int mode, const double *x, double *y) {
  const int64_t nxp = g.nx + 1;
  const int64_t nn = nxp * (g.ny + 1);
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const int j = (int)(node / nxp), i = (int)(node - (int64_t)j * nxp);
  double acc = 0.0;
  for (int e = 0; e < 6; ++e) {
    const int ci = i + kInc[e].di, cj = j + kInc[e].dj;
    if (ci < 0 || cj < 0 || ci >= g.nx || cj >= g.ny) continue;
    int64_t nd[3];
    double gr[3][2], M[3], H[3], hat[3], sq[3];
    tri_nodes(g, ci, cj, kInc[e].t, nd, gr);
    const int a = kInc[e].a;
    element_row(g, o, nd, gr, a, M, H, hat, sq);
    if (mode == 1) {
      acc += (o.kind == LSG_OP_PG_TRANSPORT) ? M[a] + o.sign * o.dt * H[a] : M[a];
    } else if (mode == 0) {
      for (int b = 0; b < 3; ++b) {
        const double Ab = (o.kind == LSG_OP_PG_TRANSPORT) ? M[b] + o.sign * o.dt * H[b] : M[b];
        acc += Ab * x[nd[b]];
      }
    } else {
      // reinit rhs row: (m_hat cur)_a + dt (load_a + diffusion_a)   (levelset.py:205-212)
      double gc[2] = {0.0, 0.0}, gp[2] = {0.0, 0.0};
      for (int v = 0; v < 3; ++v) {
        const double c = o.cur[nd[v]], pv = o.prev[nd[v]];
        gc[0] += gr[v][0] * c;  gc[1] += gr[v][1] * c;
        gp[0] += gr[v][0] * pv; gp[1] += gr[v][1] * pv;
      }
      const double mc = sqrt(gc[0] * gc[0] + gc[1] * gc[1]);
      const double mp = sqrt(gp[0] * gp[0] + gp[1] * gp[1]);
      double row = 0.0;
      for (int b = 0; b < 3; ++b) row += M[b] * o.cur[nd[b]];
      const double w = g.area / 3.0;
      double load = 0.0;
      for (int q = 0; q < 3; ++q) load += w * (0.5 * sq[q] * (mp - 3.0 * mc) + sq[q]) * hat[q];
      const double diff = 0.5 * o.h * o.h * g.area *
                          ((gp[0] - 3.0 * gc[0]) * gr[a][0] + (gp[1] - 3.0 * gc[1]) * gr[a][1]);
      acc += row + o.dt * (load + diff);
    }
  }
  y[node] = acc;
}

static OpArgs args_of(const lsg_op &op) {
  OpArgs o;
  o.kind = op.kind;
  o.dt = op.p[0];
  o.h = op.p[1];
  o.sign = op.p[2];
  o.smooth = op.p[3] != 0.0;
  o.theta = op.aux[0];
  o.phi0 = op.aux[0];
  o.cur = op.aux[1];
  o.prev = op.aux[2];
  return o;
}

int apply(const lsg_op &op, const double *x, double *y, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  gather_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, args_of(op), 0, x, y);
  return check_launch("pg_apply");
}

int diag(const lsg_op &op, double *d, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  gather_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, args_of(op), 1, nullptr, d);
  return check_launch("pg_diag");
}

int reinit_rhs(const lsg_op &op, double *rhs, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t nn = (int64_t)(g.nx + 1) * (g.ny + 1);
  gather_kernel<<<(unsigned)ceil_div(nn, 128), 128, 0, st>>>(g, args_of(op), 2, nullptr, rhs);
  return check_launch("pg_reinit_rhs");
}

// ---------------------------------------------------------------------------
// Right-Jacobi-preconditioned BiCGStab with device-resident scalars.
// Scalars (device, 16 doubles): 0 rho, 1 alpha, 2 omega, 3 rho1, 4 (r0,v),
// 5 (t,s), 6 (t,t), 7 (r,r), 8 (b,b), 9 (s,s)
// ---------------------------------------------------------------------------
constexpr int kT = 256;
constexpr int kDotBlocks = 296;

// deterministic dot products of up to 3 pairs, written to sc[out0..]
__global__ void dots_kernel(int64_t n, const double *a0, const double *b0, const double *a1,
                            const double *b1, double *sc, int o0, int o1, double *partials,
                            uint32_t *counter) {
  __shared__ double scratch[2 * (kT / 32)];
  double v[2] = {0.0, 0.0};
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < n; t += (int64_t)gridDim.x * kT) {
    v[0] += a0[t] * b0[t];
    if (a1) v[1] += a1[t] * b1[t];
  }
  double tot[2];
  if (block_partial_and_total<2, 0u>(v, partials, counter, blockIdx.x, gridDim.x, scratch, tot)) {
    if (threadIdx.x == 0) {
      sc[o0] = tot[0];
      if (a1) sc[o1] = tot[1];
    }
  }
}

// p = r + beta (p - omega v), beta = (rho1/rho)(alpha/omega); phat = dinv p
__global__ void bicg_p(int64_t n, const double *r, double *p, const double *v, const double *dinv,
                       double *phat, const double *sc, int first) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  double pv;
  if (first) {
    pv = r[t];
  } else {
    const double beta = (sc[3] / sc[0]) * (sc[1] / sc[2]);
    pv = r[t] + beta * (p[t] - sc[2] * v[t]);
  }
  p[t] = pv;
  phat[t] = dinv[t] * pv;
}

// alpha = rho1 / (r0, v); s = r - alpha v; shat = dinv s
__global__ void bicg_s(int64_t n, const double *r, const double *v, const double *dinv, double *s,
                       double *shat, double *sc) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  const double alpha = sc[3] / sc[4];
  if (t == 0) sc[1] = alpha;  // every thread computes the same alpha; one stores it
  const double sv = r[t] - alpha * v[t];
  s[t] = sv;
  shat[t] = dinv[t] * sv;
}

// omega = (t,s)/(t,t); x += alpha phat + omega shat; r = s - omega t; rho = rho1
__global__ void bicg_x(int64_t n, double *x, double *r, const double *s, const double *tt,
                       const double *phat, const double *shat, double *sc) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  const double omega = sc[6] > 0.0 ? sc[5] / sc[6] : 0.0;
  const double alpha = sc[3] / sc[4];
  x[t] += alpha * phat[t] + omega * shat[t];
  r[t] = s[t] - omega * tt[t];
}

__global__ void bicg_finish_scalars(double *sc) {
  // after bicg_x: record omega and rho for the next iteration
  const double omega = sc[6] > 0.0 ? sc[5] / sc[6] : 0.0;
  sc[2] = omega;
  sc[0] = sc[3];
}

__global__ void resid_kernel(int64_t n, const double *b, const double *ax, double *r, double *r0) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  const double v = b[t] - ax[t];
  r[t] = v;
  r0[t] = v;
}

__global__ void reciprocal(int64_t n, double *d) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t < n) d[t] = fabs(d[t]) > 0.0 ? 1.0 / d[t] : 1.0;
}


// ---------------------------------------------------------------------------
// Restarted GMRES(m), right-Jacobi-preconditioned, classical Gram-Schmidt with
// one re-orthogonalisation (CGS2): the robust solver behind lsg_bicgstab when
// BiCGStab stagnates or breaks down (the PG step matrices turn strongly
// non-normal when |theta| dt / h grows; the reference factorises them with
// splu, levelset.py:165,204).  Vector work on the device with fixed-order
// reductions; the (m+1) x m Hessenberg least-squares problem on the host.
// ---------------------------------------------------------------------------
constexpr int kGmM = 48;  // Krylov dimension per cycle

// out[i] partials: sum_t V_i[t] w[t], grid (kDotBlocks, nv)
__global__ void gm_dots(int64_t n, const double *V, int nv, const double *w, double *partials) {
  __shared__ double scratch[kT / 32];
  const int i = blockIdx.y;
  const double *vi = V + (size_t)i * n;
  double v[1] = {0.0};
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < n; t += (int64_t)gridDim.x * kT)
    v[0] += vi[t] * w[t];
  block_reduce<1, 0u>(v, scratch);
  if (threadIdx.x == 0) partials[(size_t)i * gridDim.x + blockIdx.x] = v[0];
}

// fixed-order totals of gm_dots' partials, one block per vector
__global__ void gm_dots_finish(const double *partials, int nblk, double *out) {
  __shared__ double scratch[kT / 32];
  const int i = blockIdx.x;
  double v[1] = {0.0};
  for (int c = threadIdx.x; c < nblk; c += kT) v[0] += partials[(size_t)i * nblk + c];
  block_reduce<1, 0u>(v, scratch);
  if (threadIdx.x == 0) out[i] = v[0];
}

// w -= sum_{i < nv} h_i V_i
__global__ void gm_update(int64_t n, const double *V, int nv, const double *h, double *w) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  double acc = w[t];
  for (int i = 0; i < nv; ++i) acc -= h[i] * V[(size_t)i * n + t];
  w[t] = acc;
}

__global__ void gm_scale(int64_t n, const double *w, double s, double *out) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t < n) out[t] = s * w[t];
}

__global__ void gm_precond(int64_t n, const double *dinv, const double *v, double *z) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t < n) z[t] = dinv[t] * v[t];
}

// x += dinv (sum_{i < nv} y_i V_i)
__global__ void gm_combine(int64_t n, const double *V, int nv, const double *y, const double *dinv,
                           double *x) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t >= n) return;
  double acc = 0.0;
  for (int i = 0; i < nv; ++i) acc += y[i] * V[(size_t)i * n + t];
  x[t] += dinv[t] * acc;
}

__global__ void gm_resid(int64_t n, const double *b, const double *ax, double *r) {
  const int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (t < n) r[t] = b[t] - ax[t];
}

int64_t gmres_work_doubles(int64_t n) {
  return (int64_t)(kGmM + 4) * n + (int64_t)(kGmM + 1) * (kDotBlocks + 2) + 32;
}

static int gmres(const lsg_op &op, const double *b, double *x, double *work, double target,
                 int maxit, int *iters, double *resid, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t n = (int64_t)(g.nx + 1) * (g.ny + 1);
  const int m = kGmM;
  double *dinv = work, *w = dinv + n, *z = w + n, *V = z + n;      // V: (m+1) n
  double *hdev = V + (size_t)(m + 1) * n;                          // m+1
  double *part = hdev + (m + 1);                                   // (m+1) kDotBlocks
  double *hout = part + (size_t)(m + 1) * kDotBlocks;              // m+1
  const unsigned nb = (unsigned)ceil_div(n, kT);
  int rc;
  if ((rc = diag(op, dinv, st))) return rc;
  reciprocal<<<nb, kT, 0, st>>>(n, dinv);
  auto norm = [&](const double *v, double &out) -> int {
    gm_dots<<<dim3(kDotBlocks, 1), kT, 0, st>>>(n, v, 1, v, part);
    gm_dots_finish<<<1, kT, 0, st>>>(part, kDotBlocks, hout);
    double h;
    cudaMemcpyAsync(&h, hout, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("gmres sync");
    out = sqrt(h);
    return check_launch("gmres norm");
  };
  // projections h = V[0..nv)^T w on the host
  auto project = [&](int nv, double *h) -> int {
    gm_dots<<<dim3(kDotBlocks, nv), kT, 0, st>>>(n, V, nv, w, part);
    gm_dots_finish<<<nv, kT, 0, st>>>(part, kDotBlocks, hout);
    cudaMemcpyAsync(h, hout, nv * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("gmres sync");
    return check_launch("gmres project");
  };
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gv(m + 1), h(m + 1), h2(m + 1), y(m);
  int total = 0;
  double beta = 0.0;
  while (true) {
    if ((rc = apply(op, x, w, st))) return rc;
    gm_resid<<<nb, kT, 0, st>>>(n, b, w, V);
    if ((rc = norm(V, beta))) return rc;
    *resid = beta;
    *iters = total;
    if (!(beta > target) || total >= maxit) break;
    gm_scale<<<nb, kT, 0, st>>>(n, V, 1.0 / beta, V);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int jend = -1;
    for (int j = 0; j < m && total < maxit; ++j) {
      gm_precond<<<nb, kT, 0, st>>>(n, dinv, V + (size_t)j * n, z);
      if ((rc = apply(op, z, w, st))) return rc;
      if ((rc = project(j + 1, h.data()))) return rc;  // CGS, then one re-orthogonalisation
      cudaMemcpyAsync(hdev, h.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, st);
      gm_update<<<nb, kT, 0, st>>>(n, V, j + 1, hdev, w);
      if ((rc = project(j + 1, h2.data()))) return rc;
      cudaMemcpyAsync(hdev, h2.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, st);
      gm_update<<<nb, kT, 0, st>>>(n, V, j + 1, hdev, w);
      double hn;
      if ((rc = norm(w, hn))) return rc;
      ++total;
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = h[i] + h2[i];
      H[(size_t)(j + 1) * m + j] = hn;
      if (hn > 0.0) gm_scale<<<nb, kT, 0, st>>>(n, w, 1.0 / hn, V + (size_t)(j + 1) * n);
      for (int i = 0; i < j; ++i) {  // previous Givens rotations
        const double a = H[(size_t)i * m + j], c = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * c;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
      }
      const double a = H[(size_t)j * m + j], c = H[(size_t)(j + 1) * m + j];
      const double r = hypot(a, c);
      cs[j] = r > 0.0 ? a / r : 1.0;
      sn[j] = r > 0.0 ? c / r : 0.0;
      H[(size_t)j * m + j] = r;
      H[(size_t)(j + 1) * m + j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      jend = j;
      if (!(fabs(gv[j + 1]) > target) || hn == 0.0) break;
    }
    if (jend < 0) break;
    for (int i = jend; i >= 0; --i) {  // back substitution
      double acc = gv[i];
      for (int k = i + 1; k <= jend; ++k) acc -= H[(size_t)i * m + k] * y[k];
      y[i] = H[(size_t)i * m + i] != 0.0 ? acc / H[(size_t)i * m + i] : 0.0;
    }
    cudaMemcpyAsync(hdev, y.data(), (jend + 1) * sizeof(double), cudaMemcpyHostToDevice, st);
    gm_combine<<<nb, kT, 0, st>>>(n, V, jend + 1, hdev, dinv, x);
    if ((rc = check_launch("gmres cycle"))) return rc;
  }
  return LSG_OK;
}

static int bicgstab_only(const lsg_op &op, const double *b, double *x, double *work, double rtol, int maxit,
             int *iters, double *resid, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t n = (int64_t)(g.nx + 1) * (g.ny + 1);
  // work layout: r, r0, p, v, s, t, phat, shat, dinv (9 n) | sc (16) | partials (2 kDotBlocks) | counter
  double *r = work, *r0 = r + n, *p = r0 + n, *v = p + n, *s = v + n, *tt = s + n;
  double *phat = tt + n, *shat = phat + n, *dinv = shat + n;
  double *sc = dinv + n, *part = sc + 16;
  uint32_t *cnt = reinterpret_cast<uint32_t *>(part + 2 * kDotBlocks);
  const unsigned nb = (unsigned)ceil_div(n, kT);
  int rc;
  cudaMemsetAsync(cnt, 0, sizeof(uint32_t), st);
  cudaMemsetAsync(sc, 0, 16 * sizeof(double), st);
  if ((rc = diag(op, dinv, st))) return rc;
  reciprocal<<<nb, kT, 0, st>>>(n, dinv);
  if ((rc = apply(op, x, v, st))) return rc;
  resid_kernel<<<nb, kT, 0, st>>>(n, b, v, r, r0);
  dots_kernel<<<kDotBlocks, kT, 0, st>>>(n, r, r, b, b, sc, 7, 8, part, cnt);
  if ((rc = check_launch("bicgstab init"))) return rc;
  double host[16];
  cudaMemcpyAsync(host, sc, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("bicgstab sync");
  const double target = rtol * sqrt(host[8]);
  *iters = 0;
  *resid = sqrt(host[7]);
  if (host[8] == 0.0) {
    cudaMemsetAsync(x, 0, n * sizeof(double), st);
    *resid = 0.0;
    return check_launch("bicgstab zero");
  }
  for (int it = 0; it < maxit && *resid > target; ++it) {
    // rho1 = (r0, r)
    dots_kernel<<<kDotBlocks, kT, 0, st>>>(n, r0, r, nullptr, nullptr, sc, 3, 0, part, cnt);
    bicg_p<<<nb, kT, 0, st>>>(n, r, p, v, dinv, phat, sc, it == 0);
    if ((rc = apply(op, phat, v, st))) return rc;
    dots_kernel<<<kDotBlocks, kT, 0, st>>>(n, r0, v, nullptr, nullptr, sc, 4, 0, part, cnt);
    bicg_s<<<nb, kT, 0, st>>>(n, r, v, dinv, s, shat, sc);
    if ((rc = apply(op, shat, tt, st))) return rc;
    dots_kernel<<<kDotBlocks, kT, 0, st>>>(n, tt, s, tt, tt, sc, 5, 6, part, cnt);
    bicg_x<<<nb, kT, 0, st>>>(n, x, r, s, tt, phat, shat, sc);
    bicg_finish_scalars<<<1, 1, 0, st>>>(sc);
    dots_kernel<<<kDotBlocks, kT, 0, st>>>(n, r, r, nullptr, nullptr, sc, 7, 0, part, cnt);
    if ((rc = check_launch("bicgstab iteration"))) return rc;
    cudaMemcpyAsync(host, sc, sizeof(host), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("bicgstab sync");
    *iters = it + 1;
    *resid = sqrt(host[7]);
  }
  return LSG_OK;
}

// BiCGStab first (cheap per iteration); if it stagnates or breaks down, the
// solve restarts from the caller's initial guess with GMRES(m).  Returns
// LSG_ERR_NOCONV when neither reaches ||r|| <= rtol ||b||.
int bicgstab(const lsg_op &op, const double *b, double *x, double *work, double rtol, int maxit,
             int *iters, double *resid, cudaStream_t st) {
  const Geo g = geo_of(op.grid);
  const int64_t n = (int64_t)(g.nx + 1) * (g.ny + 1);
  double *x0 = work;  // the initial guess, kept for a restart
  double *rest = work + n;
  cudaMemcpyAsync(x0, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  int rc = bicgstab_only(op, b, x, rest, rtol, maxit, iters, resid, st);
  if (rc) return rc;
  // ||b|| for the target (BiCGStab's own scalar slot 8 holds (b,b))
  double bb = 0.0;
  cudaMemcpyAsync(&bb, rest + 9 * n + 8, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("bicgstab sync");
  const double target = rtol * sqrt(bb);
  if (*resid <= target) return LSG_OK;  // converged (NaN fails this test)
  cudaMemcpyAsync(x, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  int it2 = 0;
  rc = gmres(op, b, x, rest, target, maxit, &it2, resid, st);
  *iters += it2;
  if (rc) return rc;
  // rtol stands in for a direct solve (1e-14); late in a run the reference's own
  // PG/AB2 reinitialisation inflates |phi| to ~1e15 and Krylov methods floor
  // near 1e-13 relative -- still far below anything that moves the signs of phi
  // at the quadrature points, which is all the loop consumes.  Accept up to
  // 1e3 x the target, fail loudly beyond.
  if (!(*resid <= 1e3 * target)) {
    set_error("PG solve did not converge: residual %.3e > %.3e after %d iterations", *resid, target,
              *iters);
    return LSG_ERR_NOCONV;
  }
  return LSG_OK;
}

}  // namespace pg
}  // namespace lsg
