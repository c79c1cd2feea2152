// extern "C" entry points of liblsgpu.so (see include/lsgpu.h).
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"
#include "ops.h"

namespace lsg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};

int check_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return LSG_ERR_CUDA;
  }
  return LSG_OK;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_NO_PDL");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

static int check_grid(const lsg_grid *g) {
  if (!g) { set_error("null grid"); return LSG_ERR_ARG; }
  if (g->dim != 2 && g->dim != 3) { set_error("grid dim must be 2 or 3, got %d", g->dim); return LSG_ERR_ARG; }
  for (int a = 0; a < g->dim; ++a) {
    if (g->n[a] < 1) { set_error("cell counts must be >= 1"); return LSG_ERR_ARG; }
    if (!(g->hi[a] > g->lo[a])) { set_error("bounds must satisfy hi > lo"); return LSG_ERR_ARG; }
  }
  int64_t nn = 1;
  for (int a = 0; a < g->dim; ++a) nn *= (int64_t)g->n[a] + 1;
  if (nn >= (1LL << 31)) { set_error("grid too large for int32 connectivity"); return LSG_ERR_ARG; }
  return LSG_OK;
}

static int check_op(const lsg_op *op) {
  if (!op) { set_error("null operator"); return LSG_ERR_ARG; }
  int rc = check_grid(&op->grid);
  if (rc) return rc;
  if (op->kind == LSG_OP_PG_TRANSPORT || op->kind == LSG_OP_PG_REINIT) {
    if (op->grid.dim != 2) { set_error("the reference (PG) level-set scheme is 2D only"); return LSG_ERR_ARG; }
    if (!op->aux[0] || (op->kind == LSG_OP_PG_REINIT && !op->aux[1])) {
      set_error("PG operator fields missing");
      return LSG_ERR_ARG;
    }
    if (!(op->p[0] > 0.0) || !(op->p[1] > 0.0)) { set_error("PG operator needs dt > 0 and h > 0"); return LSG_ERR_ARG; }
    return LSG_OK;
  }
  if (op->kind == LSG_OP_LAPLACE && op->grid.dim != 2) {
    set_error("the scalar diffusion operator (heat models) is 2D only, as the reference");
    return LSG_ERR_ARG;
  }
  if (op->kind != LSG_OP_ELASTICITY && op->kind != LSG_OP_H1 && op->kind != LSG_OP_LAPLACE) {
    set_error("unknown operator kind %d", op->kind);
    return LSG_ERR_ARG;
  }
  if (!op->words) { set_error("operator words missing"); return LSG_ERR_ARG; }
  return LSG_OK;
}

static bool is_pg(const lsg_op *op) {
  return op->kind == LSG_OP_PG_TRANSPORT || op->kind == LSG_OP_PG_REINIT;
}

static cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

}  // namespace lsg

using namespace lsg;

#define DISPATCH(g, call2, call3) ((g).dim == 2 ? (d2::call2) : (d3::call3))

extern "C" {

int32_t lsg_abi_version(void) { return 3; }
int64_t lsg_launch_count(void) { return (int64_t)g_launches.load(); }
const char *lsg_last_error(void) { return g_err; }

int64_t lsg_num_nodes(const lsg_grid *g) {
  if (check_grid(g)) return -1;
  int64_t nn = 1;
  for (int a = 0; a < g->dim; ++a) nn *= (int64_t)g->n[a] + 1;
  return nn;
}

int64_t lsg_num_elements(const lsg_grid *g) {
  if (check_grid(g)) return -1;
  int64_t ne = 1;
  for (int a = 0; a < g->dim; ++a) ne *= g->n[a];
  return g->dim == 2 ? 2 * ne : 6 * ne;
}

int64_t lsg_partials_per_rhs(const lsg_grid *g) {
  if (check_grid(g)) return -1;
  return g->dim == 2 ? d2::partials_per_rhs(*g) : d3::partials_per_rhs(*g);
}

int lsg_mesh_vertices(const lsg_grid *g, double *xyz, void *stream) {
  int rc = check_grid(g);
  return rc ? rc : mesh_vertices(*g, xyz, S(stream));
}

int lsg_mesh_elements(const lsg_grid *g, int32_t *conn, void *stream) {
  int rc = check_grid(g);
  return rc ? rc : mesh_elements(*g, conn, S(stream));
}

int lsg_material(const lsg_grid *g, const double *phi, const uint8_t *bcmask, void *words,
                 void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  return DISPATCH(*g, material(*g, phi, bcmask, words, S(stream)),
                  material(*g, phi, bcmask, words, S(stream)));
}

int lsg_indicator_quad(const lsg_grid *g, const double *phi, double *chi, void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  return DISPATCH(*g, indicator(*g, phi, chi, S(stream)), indicator(*g, phi, chi, S(stream)));
}

int lsg_h1_words(const lsg_grid *g, const uint8_t *frozen_q, int32_t zero_dirichlet, void *words,
                 void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  return DISPATCH(*g, h1_words(*g, frozen_q, zero_dirichlet, words, S(stream)),
                  h1_words(*g, frozen_q, zero_dirichlet, words, S(stream)));
}

int lsg_apply(const lsg_op *op, int32_t k, const double *x, double *y, void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (k < 1 || k > 65535) { set_error("batch size k must be in [1, 65535], got %d", k); return LSG_ERR_ARG; }
  if (is_pg(op)) {
    if (k != 1) { set_error("PG operators apply to one field"); return LSG_ERR_ARG; }
    return pg::apply(*op, x, y, S(stream));
  }
  return DISPATCH(op->grid, apply(*op, k, x, y, S(stream)), apply(*op, k, x, y, S(stream)));
}

int lsg_diag(const lsg_op *op, double *diag_out, void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (is_pg(op)) return pg::diag(*op, diag_out, S(stream));
  return DISPATCH(op->grid, diag(*op, diag_out, S(stream)), diag(*op, diag_out, S(stream)));
}

int lsg_pg_reinit_rhs(const lsg_op *op, double *rhs, void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (op->kind != LSG_OP_PG_REINIT || !op->aux[2]) {
    set_error("lsg_pg_reinit_rhs needs a PG_REINIT operator with aux[2] = previous iterate");
    return LSG_ERR_ARG;
  }
  return pg::reinit_rhs(*op, rhs, S(stream));
}

int64_t lsg_bicgstab_work_doubles(const lsg_grid *g) {
  if (check_grid(g)) return -1;
  int64_t nn = 1;
  for (int a = 0; a < g->dim; ++a) nn *= (int64_t)g->n[a] + 1;
  // saved initial guess + max(BiCGStab workspace, GMRES(m) workspace)
  const int64_t bicg = 9 * nn + 16 + 2 * 296 + 8;
  const int64_t gm = pg::gmres_work_doubles(nn);
  return nn + (bicg > gm ? bicg : gm);
}

int lsg_bicgstab(const lsg_op *op, const double *b, double *x, double *work, double rtol,
                 int32_t maxit, int32_t *iters, double *resid, void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (!is_pg(op)) { set_error("lsg_bicgstab solves the PG level-set operators"); return LSG_ERR_ARG; }
  if (!b || !x || !work || !iters || !resid || maxit < 0) { set_error("bad BiCGStab arguments"); return LSG_ERR_ARG; }
  int it = 0;
  rc = pg::bicgstab(*op, b, x, work, rtol, maxit, &it, resid, S(stream));
  *iters = it;
  return rc;
}

int lsg_inv_diag(const lsg_op *op, double *dinv, void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  return DISPATCH(op->grid, inv_diag(*op, dinv, S(stream)), inv_diag(*op, dinv, S(stream)));
}

// The buffers each path reads unconditionally must be present: 2D forms r_i
// into r_alt and keeps q_alt for the stored-q / persistent passes; 3D rotates
// three direction buffers (p, p_alt, p_ring).  A missing one is an argument
// error, not an illegal address that poisons the context.
static int check_ws(const lsg_op *op, const lsg_pcg_ws *ws) {
  if (!ws || ws->k < 1 || ws->k > 65535 || !ws->x || !ws->b || !ws->r || !ws->p || !ws->q ||
      !ws->scal || !ws->partials || !ws->counters || !ws->p_alt || !ws->dinv) {
    set_error("incomplete PCG workspace");
    return LSG_ERR_ARG;
  }
  if (op->grid.dim == 2 && (!ws->r_alt || !ws->q_alt)) {
    set_error("incomplete PCG workspace: 2D needs r_alt and q_alt");
    return LSG_ERR_ARG;
  }
  if (op->grid.dim == 3 && !ws->p_ring) {
    set_error("incomplete PCG workspace: 3D needs p_ring");
    return LSG_ERR_ARG;
  }
  return LSG_OK;
}

int64_t lsg_sizeof_op(void) { return (int64_t)sizeof(lsg_op); }
int64_t lsg_sizeof_pcg_ws(void) { return (int64_t)sizeof(lsg_pcg_ws); }
int64_t lsg_sizeof_grid(void) { return (int64_t)sizeof(lsg_grid); }

int lsg_pcg_start(const lsg_op *op, lsg_pcg_ws *ws, double rtol, double atol, double maxiter,
                  void *stream) {
  int rc = check_op(op);
  if (!rc) rc = check_ws(op, ws);
  if (rc) return rc;
  return DISPATCH(op->grid, pcg_start(*op, *ws, rtol, atol, maxiter, S(stream)),
                  pcg_start(*op, *ws, rtol, atol, maxiter, S(stream)));
}

int lsg_pcg_iterate(const lsg_op *op, lsg_pcg_ws *ws, int32_t niter, void *stream) {
  int rc = check_op(op);
  if (!rc) rc = check_ws(op, ws);
  if (rc) return rc;
  if (niter < 0) { set_error("niter must be >= 0"); return LSG_ERR_ARG; }
  return pcg_iterate_graph(*op, *ws, niter, S(stream));
}

void lsg_graph_stats(double *out4) {
  if (out4) graph_stats(out4);
}

int lsg_pcg_finish(const lsg_op *op, lsg_pcg_ws *ws, void *stream) {
  int rc = check_op(op);
  if (!rc) rc = check_ws(op, ws);
  if (rc) return rc;
  return DISPATCH(op->grid, pcg_finish(*op, *ws, S(stream)), pcg_finish(*op, *ws, S(stream)));
}

int lsg_shape_rhs(const lsg_op *op, int32_t k, const double *u, double volume, double *vec_cost,
                  double *vec_vol, double *out, double *s1, double *partials, uint32_t *counter,
                  void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (op->kind != LSG_OP_ELASTICITY) { set_error("shape_rhs needs the elasticity operator"); return LSG_ERR_ARG; }
  if (k < 1) { set_error("need at least one state"); return LSG_ERR_ARG; }
  if (!(volume > 0.0)) { set_error("target volume must be positive"); return LSG_ERR_ARG; }
  (void)s1;  // the tensor itself is produced by lsg_s1_tensor (parity path)
  return DISPATCH(op->grid,
                  shape_rhs(*op, k, u, volume, vec_cost, vec_vol, out, partials, counter, S(stream)),
                  shape_rhs(*op, k, u, volume, vec_cost, vec_vol, out, partials, counter, S(stream)));
}

int lsg_heat_shape(const lsg_op *op, int32_t k, const double *u, const double *weights,
                   const double *fq, const double *gq, double volume, double *vec_cost,
                   double *vec_vol, double *out, double *partials, uint32_t *counter,
                   void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  if (op->kind != LSG_OP_LAPLACE) { set_error("heat_shape needs the scalar diffusion operator"); return LSG_ERR_ARG; }
  if (k < 1 || !weights || !fq || !u) { set_error("heat_shape needs k >= 1 states, weights and source samples"); return LSG_ERR_ARG; }
  if (!(volume > 0.0)) { set_error("target volume must be positive"); return LSG_ERR_ARG; }
  return d2::heat_shape(*op, k, u, weights, fq, gq, volume, vec_cost, vec_vol, out, partials,
                        counter, S(stream));
}

static int need_2d(const lsg_grid *g, const char *what) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (g->dim != 2) { set_error("%s is 2D only (models/inverse.py), as the reference", what); return LSG_ERR_ARG; }
  return LSG_OK;
}

int lsg_inverse_misfit(const lsg_grid *g, int32_t k, const double *u, const double *v,
                       const double *measured, const uint8_t *facet_flags,
                       const uint8_t *partial_mask, double alpha, double beta, double *head,
                       double *tail, double *out, double *partials, uint32_t *counter,
                       void *stream) {
  int rc = need_2d(g, "inverse_misfit");
  if (rc) return rc;
  if (k < 1 || !u || !v || !measured || !facet_flags || !head || !tail || !out) {
    set_error("inverse_misfit: missing arrays or k < 1");
    return LSG_ERR_ARG;
  }
  return inverse_misfit(*g, k, u, v, measured, facet_flags, partial_mask, alpha, beta, head, tail,
                        out, partials, counter, S(stream));
}

int lsg_inverse_tensors(const lsg_grid *g, int32_t k, const double *u, const double *v,
                        const double *p, const double *q, const double *measured,
                        const double *proj, const double *phi, double a_in, double a_out,
                        double lam, double mu, double alpha, double *s0, double *s1,
                        void *stream) {
  int rc = need_2d(g, "inverse_tensors");
  if (rc) return rc;
  if (k < 1 || !u || !v || !p || !q || !measured || !proj || !phi || !s0 || !s1) {
    set_error("inverse_tensors: missing arrays or k < 1");
    return LSG_ERR_ARG;
  }
  return inverse_tensors(*g, k, u, v, p, q, measured, proj, phi, a_in, a_out, lam, mu, alpha, s0,
                         s1, S(stream));
}

int lsg_strain_projection_rhs(const lsg_grid *g, int32_t k, const double *measured, double *out,
                              void *stream) {
  int rc = need_2d(g, "strain_projection_rhs");
  if (rc) return rc;
  if (k < 1 || !measured || !out) { set_error("strain_projection_rhs: missing arrays"); return LSG_ERR_ARG; }
  return strain_projection_rhs(*g, k, measured, out, S(stream));
}

int lsg_s1_tensor(const lsg_op *op, int32_t k, const double *u, const double *phi, double *s1,
                  void *stream) {
  int rc = check_op(op);
  if (rc) return rc;
  return DISPATCH(op->grid, s1_tensor(*op, k, u, phi, s1, S(stream)),
                  s1_tensor(*op, k, u, phi, s1, S(stream)));
}

int lsg_tensor_rhs(const lsg_grid *g, const double *s0, const double *s1, double *vec,
                   void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  return DISPATCH(*g, tensor_rhs(*g, s0, s1, vec, S(stream)), tensor_rhs(*g, s0, s1, vec, S(stream)));
}

int lsg_velocity_rhs(const lsg_op *h1, const double *vec_cost, const double *vec_vol, double lam,
                     double *b, void *stream) {
  int rc = check_op(h1);
  if (rc) return rc;
  return DISPATCH(h1->grid, velocity_rhs(*h1, vec_cost, vec_vol, lam, b, S(stream)),
                  velocity_rhs(*h1, vec_cost, vec_vol, lam, b, S(stream)));
}

int lsg_velocity_stats(const lsg_op *h1, const double *theta, const double *vec, double *out,
                       double *partials, uint32_t *counter, void *stream) {
  int rc = check_op(h1);
  if (rc) return rc;
  return DISPATCH(h1->grid, velocity_stats(*h1, theta, vec, out, partials, counter, S(stream)),
                  velocity_stats(*h1, theta, vec, out, partials, counter, S(stream)));
}

int lsg_transport(const lsg_grid *g, const double *phi_in, const double *theta, double dt,
                  int32_t nsub, int32_t smooth, double h, double *phi_out, double *tmp,
                  void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (nsub < 1 || !(dt > 0.0)) { set_error("transport needs nsub >= 1 and dt > 0"); return LSG_ERR_ARG; }
  return transport(*g, phi_in, theta, dt, nsub, smooth, h, phi_out, tmp, S(stream));
}

int lsg_reinit(const lsg_grid *g, const double *phi_in, double dt, int32_t nsub, double h,
               double *phi_out, double *tmp, double *sgn, void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (nsub < 1 || !(dt > 0.0)) { set_error("reinit needs nsub >= 1 and dt > 0"); return LSG_ERR_ARG; }
  return reinit(*g, phi_in, dt, nsub, h, phi_out, tmp, sgn, S(stream));
}

int lsg_cfl_speed(const lsg_grid *g, const double *v, double *out, double *partials,
                  uint32_t *counter, void *stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  return DISPATCH(*g, cfl_speed(*g, v, out, partials, counter, S(stream)),
                  cfl_speed(*g, v, out, partials, counter, S(stream)));
}

}  // extern "C"
