// Explicit level-set update on the node lattice (north star (4)); replaces
// the reference's CN Petrov-Galerkin transport and PG/AB2 reinitialisation
// (levelset.py:137-216).  Statement of the scheme: oracle/levelset.py.
//
// transport: phi_t + theta . grad phi = [smooth] h^2 lap phi, conservative
//   face-velocity upwind (lumped-P1 form: boundary nodes of each lattice
//   line count twice), mirrored Laplacian, forward Euler.
// reinit:    phi_t = -S (|grad phi|_Godunov - 1) + h^2 lap phi,
//   S = phi0 / sqrt(phi0^2 + h^2) frozen.
//
// One thread per node; the 2d+1-point stencil reads hit L1/L2, HBM traffic
// is 8 B (phi) + 8d B (theta) read + 8 B written per node and substep
// (reinit: 8 + 8 (S) + 8).  Substep counts (CFL) are chosen by the host.
#include <math.h>

#include "common.cuh"
#include "ops.h"

namespace lsg {

struct Lattice {
  int n[3];          // cells per axis
  int64_t stride[3]; // node index stride per axis
  double h[3];
  int64_t nn;
};

static Lattice lattice_of(const lsg_grid &g) {
  Lattice L;
  for (int a = 0; a < 3; ++a) {
    L.n[a] = a < g.dim ? g.n[a] : 0;
    L.h[a] = a < g.dim ? (g.hi[a] - g.lo[a]) / g.n[a] : 1.0;
  }
  L.stride[0] = 1;
  L.stride[1] = (int64_t)L.n[0] + 1;
  L.stride[2] = L.stride[1] * ((int64_t)L.n[1] + 1);
  L.nn = L.stride[1] * (L.n[1] + 1) * (g.dim == 3 ? (L.n[2] + 1) : 1);
  return L;
}

template <int D>
__device__ __forceinline__ void node_index(const Lattice &L, int64_t node, int *idx) {
  int64_t rest = node;
  if (D == 3) {
    idx[2] = (int)(rest / L.stride[2]);
    rest -= (int64_t)idx[2] * L.stride[2];
  }
  idx[1] = (int)(rest / L.stride[1]);
  idx[0] = (int)(rest - (int64_t)idx[1] * L.stride[1]);
}

template <int D>
__device__ __forceinline__ double mirrored_lap(const Lattice &L, const double *phi, int64_t node,
                                               const int *idx, double f) {
  double lap = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int64_t s = L.stride[d];
    const double left = idx[d] > 0 ? phi[node - s] : phi[node + s];
    const double right = idx[d] < L.n[d] ? phi[node + s] : phi[node - s];
    lap += (left - 2.0 * f + right) / (L.h[d] * L.h[d]);
  }
  return lap;
}

template <int D>
__global__ void transport_kernel(Lattice L, const double *__restrict__ phi,
                                 const double *__restrict__ th, double dt, int smooth, double h2,
                                 double *__restrict__ out) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= L.nn) return;
  int idx[3];
  node_index<D>(L, node, idx);
  const double f = phi[node];
  double upd = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int64_t s = L.stride[d];
    const double v = th[node * D + d];
    double term = 0.0;
    if (idx[d] < L.n[d]) {
      const double vf = 0.5 * (v + th[(node + s) * D + d]);
      const double df = (phi[node + s] - f) / L.h[d];
      term -= fmin(vf, 0.0) * df;
    }
    if (idx[d] > 0) {
      const double vf = 0.5 * (th[(node - s) * D + d] + v);
      const double df = (f - phi[node - s]) / L.h[d];
      term -= fmax(vf, 0.0) * df;
    }
    if (idx[d] == 0 || idx[d] == L.n[d]) term *= 2.0;
    upd += term;
  }
  if (smooth) upd += h2 * mirrored_lap<D>(L, phi, node, idx, f);
  out[node] = f + dt * upd;
}

__global__ void sign_kernel(int64_t nn, const double *phi, double h2, double *s) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nn) return;
  const double f = phi[node];
  s[node] = f / sqrt(f * f + h2);
}

template <int D>
__global__ void reinit_kernel(Lattice L, const double *__restrict__ phi,
                              const double *__restrict__ sgn, double dt, double h2,
                              double *__restrict__ out) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= L.nn) return;
  int idx[3];
  node_index<D>(L, node, idx);
  const double f = phi[node];
  const double S = sgn[node];
  const bool pos = S > 0.0;
  double g2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int64_t s = L.stride[d];
    const double a = idx[d] > 0 ? (f - phi[node - s]) / L.h[d] : 0.0;
    const double b = idx[d] < L.n[d] ? (phi[node + s] - f) / L.h[d] : 0.0;
    double t;
    if (pos) {
      const double ap = fmax(a, 0.0), bn = fmin(b, 0.0);
      t = fmax(ap * ap, bn * bn);
    } else {
      const double an = fmin(a, 0.0), bp = fmax(b, 0.0);
      t = fmax(an * an, bp * bp);
    }
    g2 += t;
  }
  const double upd = -S * (sqrt(g2) - 1.0) + h2 * mirrored_lap<D>(L, phi, node, idx, f);
  out[node] = f + dt * upd;
}

int transport(const lsg_grid &g, const double *phi_in, const double *theta, double dt, int nsub,
              int smooth, double h, double *phi_out, double *tmp, cudaStream_t st) {
  const Lattice L = lattice_of(g);
  const unsigned nb = (unsigned)ceil_div(L.nn, 256);
  const double *src = phi_in;
  double *dst = (nsub & 1) ? phi_out : tmp;
  for (int s = 0; s < nsub; ++s) {
    if (g.dim == 2)
      transport_kernel<2><<<nb, 256, 0, st>>>(L, src, theta, dt, smooth, h * h, dst);
    else
      transport_kernel<3><<<nb, 256, 0, st>>>(L, src, theta, dt, smooth, h * h, dst);
    int rc = check_launch("transport");
    if (rc) return rc;
    src = dst;
    dst = (dst == phi_out) ? tmp : phi_out;
  }
  return LSG_OK;
}

int reinit(const lsg_grid &g, const double *phi_in, double dt, int nsub, double h, double *phi_out,
           double *tmp, double *sgn, cudaStream_t st) {
  const Lattice L = lattice_of(g);
  const unsigned nb = (unsigned)ceil_div(L.nn, 256);
  sign_kernel<<<nb, 256, 0, st>>>(L.nn, phi_in, h * h, sgn);
  int rc = check_launch("reinit_sign");
  if (rc) return rc;
  const double *src = phi_in;
  double *dst = (nsub & 1) ? phi_out : tmp;
  for (int s = 0; s < nsub; ++s) {
    if (g.dim == 2)
      reinit_kernel<2><<<nb, 256, 0, st>>>(L, src, sgn, dt, h * h, dst);
    else
      reinit_kernel<3><<<nb, 256, 0, st>>>(L, src, sgn, dt, h * h, dst);
    rc = check_launch("reinit");
    if (rc) return rc;
    src = dst;
    dst = (dst == phi_out) ? tmp : phi_out;
  }
  return LSG_OK;
}

}  // namespace lsg
