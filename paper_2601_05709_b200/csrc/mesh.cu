// Device-side mesh arrays, bit-identical to the reference's build_rect_mesh
// (mesh.py:132-150) and to its 3D Kuhn extension (oracle/grid.py).
//
// Coordinates follow numpy.linspace exactly: step = (hi - lo) / n,
// x_i = fl(fl(i * step) + lo) with separately rounded multiply and add (no
// FMA), and x_n = hi.
#include "common.cuh"
#include "ops.h"

namespace lsg {

struct Axes {
  int dim;
  int n[3];
  double lo[3], hi[3], step[3];
};

__device__ __forceinline__ double lin(const Axes &A, int a, int i) {
  if (i == A.n[a]) return A.hi[a];
  return __dadd_rn(__dmul_rn((double)i, A.step[a]), A.lo[a]);
}

__global__ void vertices_kernel(Axes A, int64_t nn, double *xyz) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nn) return;
  const int64_t nxp = A.n[0] + 1, nyp = A.n[1] + 1;
  const int i = (int)(v % nxp);
  const int j = (int)((v / nxp) % nyp);
  xyz[v * A.dim] = lin(A, 0, i);
  xyz[v * A.dim + 1] = lin(A, 1, j);
  if (A.dim == 3) xyz[v * 3 + 2] = lin(A, 2, (int)(v / (nxp * nyp)));
}

__global__ void elements2d_kernel(int nx, int ny, int32_t *conn) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)nx * ny) return;
  const int j = (int)(c / nx), i = (int)(c - (int64_t)j * nx);
  const int32_t a = j * (nx + 1) + i, b = a + 1, d = a + (nx + 1), cc = d + 1;
  int32_t *lo = conn + c * 6;
  lo[0] = a; lo[1] = b; lo[2] = cc;  // lower (a, b, c)
  lo[3] = a; lo[4] = cc; lo[5] = d;  // upper (a, c, d)
}

// Kuhn tetrahedra: tet m of cell c follows the axis permutation KUHN[m]
// along the path v0 -> v0+e_a -> v0+e_a+e_b -> v0+(1,1,1).
__constant__ int kKuhn[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

__global__ void elements3d_kernel(int nx, int ny, int nz, int32_t *conn) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ncell = (int64_t)nx * ny * nz;
  if (t >= 6 * ncell) return;
  const int64_t c = t / 6;
  const int m = (int)(t - c * 6);
  const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((int64_t)nx * ny));
  int off[3] = {0, 0, 0};
  auto vid = [&](int a, int b, int cc) { return (int32_t)(((int64_t)cc * (ny + 1) + b) * (nx + 1) + a); };
  int32_t *o = conn + t * 4;
  o[0] = vid(i, j, k);
  for (int s = 0; s < 3; ++s) {
    off[kKuhn[m][s]] += 1;
    o[s + 1] = vid(i + off[0], j + off[1], k + off[2]);
  }
}

int mesh_vertices(const lsg_grid &g, double *xyz, cudaStream_t st) {
  Axes A;
  A.dim = g.dim;
  int64_t nn = 1;
  for (int a = 0; a < 3; ++a) {
    A.n[a] = a < g.dim ? g.n[a] : 0;
    A.lo[a] = g.lo[a];
    A.hi[a] = g.hi[a];
    A.step[a] = a < g.dim ? (g.hi[a] - g.lo[a]) / (double)g.n[a] : 0.0;
    if (a < g.dim) nn *= (int64_t)g.n[a] + 1;
  }
  vertices_kernel<<<(unsigned)ceil_div(nn, 256), 256, 0, st>>>(A, nn, xyz);
  return check_launch("mesh_vertices");
}

int mesh_elements(const lsg_grid &g, int32_t *conn, cudaStream_t st) {
  if (g.dim == 2) {
    const int64_t nc = (int64_t)g.n[0] * g.n[1];
    elements2d_kernel<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(g.n[0], g.n[1], conn);
  } else {
    const int64_t nt = 6LL * g.n[0] * g.n[1] * g.n[2];
    elements3d_kernel<<<(unsigned)ceil_div(nt, 256), 256, 0, st>>>(g.n[0], g.n[1], g.n[2], conn);
  }
  return check_launch("mesh_elements");
}

}  // namespace lsg
