// Internal host-side interface between the C ABI (abi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include "../../include/lsgpu.h"

namespace lsg {

namespace d2 {
int64_t partials_per_rhs(const lsg_grid &g);
int apply(const lsg_op &op, int k, const double *x, double *y, cudaStream_t st);
int diag(const lsg_op &op, double *d, cudaStream_t st);
int inv_diag(const lsg_op &op, double *d, cudaStream_t st);
int pcg_start(const lsg_op &op, lsg_pcg_ws &ws, double rtol, double atol, double maxiter,
              cudaStream_t st);
int pcg_iterate(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st);
int pcg_finish(const lsg_op &op, lsg_pcg_ws &ws, cudaStream_t st);
bool pcg_persistent_ok(const lsg_op &op, const lsg_pcg_ws &ws);
int shape_rhs(const lsg_op &op, int k, const double *u, double volume, double *vc, double *vv,
              double *out, double *partials, uint32_t *counter, cudaStream_t st);
int heat_shape(const lsg_op &op, int k, const double *u, const double *weights, const double *fq,
               const double *gq, double volume, double *vc, double *vv, double *out,
               double *partials, uint32_t *counter, cudaStream_t st);
int velocity_stats(const lsg_op &h1, const double *theta, const double *vec, double *out,
                   double *partials, uint32_t *counter, cudaStream_t st);
int material(const lsg_grid &g, const double *phi, const uint8_t *bcmask, void *words,
             cudaStream_t st);
int indicator(const lsg_grid &g, const double *phi, double *chi, cudaStream_t st);
int h1_words(const lsg_grid &g, const uint8_t *frozen_q, int zero_dirichlet, void *words,
             cudaStream_t st);
int velocity_rhs(const lsg_op &h1, const double *vc, const double *vv, double lam, double *b,
                 cudaStream_t st);
int tensor_rhs(const lsg_grid &g, const double *s0, const double *s1, double *vec, cudaStream_t st);
int s1_tensor(const lsg_op &op, int k, const double *u, const double *phi, double *s1,
              cudaStream_t st);
int cfl_speed(const lsg_grid &g, const double *v, double *out, double *partials, uint32_t *counter,
              cudaStream_t st);
}  // namespace d2

namespace d3 {
int64_t partials_per_rhs(const lsg_grid &g);
int apply(const lsg_op &op, int k, const double *x, double *y, cudaStream_t st);
int diag(const lsg_op &op, double *d, cudaStream_t st);
int inv_diag(const lsg_op &op, double *d, cudaStream_t st);
int pcg_start(const lsg_op &op, lsg_pcg_ws &ws, double rtol, double atol, double maxiter,
              cudaStream_t st);
int pcg_iterate(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st);
int pcg_finish(const lsg_op &op, lsg_pcg_ws &ws, cudaStream_t st);
int shape_rhs(const lsg_op &op, int k, const double *u, double volume, double *vc, double *vv,
              double *out, double *partials, uint32_t *counter, cudaStream_t st);
int velocity_stats(const lsg_op &h1, const double *theta, const double *vec, double *out,
                   double *partials, uint32_t *counter, cudaStream_t st);
int material(const lsg_grid &g, const double *phi, const uint8_t *bcmask, void *words,
             cudaStream_t st);
int indicator(const lsg_grid &g, const double *phi, double *chi, cudaStream_t st);
int h1_words(const lsg_grid &g, const uint8_t *frozen_q, int zero_dirichlet, void *words,
             cudaStream_t st);
int velocity_rhs(const lsg_op &h1, const double *vc, const double *vv, double lam, double *b,
                 cudaStream_t st);
int tensor_rhs(const lsg_grid &g, const double *s0, const double *s1, double *vec, cudaStream_t st);
int s1_tensor(const lsg_op &op, int k, const double *u, const double *phi, double *s1,
              cudaStream_t st);
int cfl_speed(const lsg_grid &g, const double *v, double *out, double *partials, uint32_t *counter,
              cudaStream_t st);
}  // namespace d3

// dimension-generic
int mesh_vertices(const lsg_grid &g, double *xyz, cudaStream_t st);
int mesh_elements(const lsg_grid &g, int32_t *conn, cudaStream_t st);
int transport(const lsg_grid &g, const double *phi_in, const double *theta, double dt, int nsub,
              int smooth, double h, double *phi_out, double *tmp, cudaStream_t st);
int pcg_iterate_graph(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st);
void graph_stats(double *out);

namespace pg {  // the reference's own level-set scheme, 2D (pg2d.cu)
int apply(const lsg_op &op, const double *x, double *y, cudaStream_t st);
int diag(const lsg_op &op, double *d, cudaStream_t st);
int reinit_rhs(const lsg_op &op, double *rhs, cudaStream_t st);
int64_t gmres_work_doubles(int64_t n);
int bicgstab(const lsg_op &op, const double *b, double *x, double *work, double rtol, int maxit,
             int *iters, double *resid, cudaStream_t st);
}  // namespace pg
// inverse-elasticity model (inverse2d.cu), 2D
int inverse_misfit(const lsg_grid &grid, int k, const double *u, const double *v, const double *g,
                   const uint8_t *flags, const uint8_t *pmask, double alpha, double beta,
                   double *head, double *tail, double *out, double *partials, uint32_t *counter,
                   cudaStream_t st);
int inverse_tensors(const lsg_grid &grid, int k, const double *u, const double *v, const double *p,
                    const double *q, const double *g, const double *proj, const double *phi,
                    double a_in, double a_out, double lam, double mu, double alpha, double *s0,
                    double *s1, cudaStream_t st);
int strain_projection_rhs(const lsg_grid &grid, int k, const double *g, double *out,
                          cudaStream_t st);
int reinit(const lsg_grid &g, const double *phi_in, double dt, int nsub, double h, double *phi_out,
           double *tmp, double *sgn, cudaStream_t st);

}  // namespace lsg
