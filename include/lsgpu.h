/*
 * lsgpu.h -- C ABI of liblsgpu.so, the B200 (sm_100a) hot path of the
 * level-set compliance loop.
 *
 * The reference (lsopt 0.1.0, /root/reference/pkg/src/lsopt) is pure
 * Python/numpy/scipy and has no C ABI; its drop-in seams are the Python
 * functions listed beside each entry point below.
 * The package paper_2601_05709_b200 binds these symbols through ctypes and
 * re-exposes the reference's Python entry points on top of them.
 *
 * Conventions
 *   - Every array is a caller-owned DEVICE pointer (fp64 unless stated).
 *     Nothing in the library allocates device memory.
 *   - Vector fields interleave components, dof = dim*node + c, exactly like
 *     the reference (fem.py:88-96); a batch of k fields is k contiguous
 *     vectors of dim*N doubles.
 *   - Node numbering is the reference's: 2D vid = j*(nx+1)+i (mesh.py:137),
 *     3D vid = (k*(ny+1)+j)*(nx+1)+i.
 *   - `stream` is a cudaStream_t passed as void*; NULL = legacy default
 *     stream.  Calls only enqueue work; none synchronises the device.
 *   - Return value 0 = success, <0 = error; lsg_last_error() returns a
 *     thread-local message.  LSG_ERR_ARG maps to ConfigError, LSG_ERR_CUDA
 *     to RuntimeError on the Python side.
 *   - Reductions are deterministic (fixed-order two-level sums, no float
 *     atomics): identical inputs give bitwise-identical outputs.
 */
#ifndef LSGPU_H
#define LSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSG_OK 0
#define LSG_ERR_ARG -1
#define LSG_ERR_CUDA -2
#define LSG_ERR_NOCONV -3 /* an iterative solve missed its tolerance (SolverError) */

/* Structured box mesh [lo, hi] with n[a] cells per axis; dim = 2 (right
 * triangles split along the lower-left/upper-right diagonal, mesh.py:140-150)
 * or 3 (six Kuhn tetrahedra per hexahedron). n[2], lo[2], hi[2] are ignored
 * when dim == 2. */
typedef struct {
  int32_t dim;
  int32_t n[3];
  double lo[3];
  double hi[3];
} lsg_grid;

/* Operator kinds for lsg_op. */
#define LSG_OP_ELASTICITY 1 /* ersatz-material linear elasticity (fem.py:397-411) */
#define LSG_OP_H1 2         /* velocity form, velocity.py:98-127 */
/* The reference's own level-set scheme (2D), non-symmetric step operators:
 *   PG_TRANSPORT: m_hat + sign*dt*half of levelset.py:150-164; p0 = dt,
 *                 p1 = h, p2 = sign (+1 left / -1 right), p3 = smooth;
 *                 aux[0] = theta (2N).
 *   PG_REINIT:    m_hat of levelset.py:196-204; p0 = dt, p1 = h;
 *                 aux[0] = phi0 (frozen sign), aux[1] = current iterate,
 *                 aux[2] = previous iterate (lsg_pg_reinit_rhs only). */
#define LSG_OP_PG_TRANSPORT 3
#define LSG_OP_PG_REINIT 4
/* Scalar diffusion (a grad u, grad v) with the two-phase conductivity of the
 * heat models (models/heat.py:113-119, fem.py:388-394), 2D only as the
 * reference: words = lsg_material words (bit 5 = Dirichlet node),
 * p0 = outside (contrast, heat.py:34), p1 = inside conductivity. */
#define LSG_OP_LAPLACE 5

/* Matrix-free operator description.
 *   ELASTICITY: words = per-node material word written by lsg_material
 *               (uint8 in 2D, uint32 in 3D); p0 = lambda, p1 = mu,
 *               p2 = outside (ersatz) coefficient, p3 = inside coefficient
 *               (MaterialIndicator(inside, outside), base.py:100-121;
 *               0 is read as 1), p4..p5 unused.
 *   H1:         words = per-node form word written by lsg_h1_words;
 *               p0 = mass_weight, p1 = stiffness_weight,
 *               p2 = boundary_normal_penalty, p3 = frozen_penalty.
 * Dirichlet dofs (bits in the words) are eliminated symmetrically:
 *   y = m.*A(m.*x) + (1-m).*x (fem.py:274-291). */
typedef struct {
  int32_t kind;
  int32_t pad_;
  lsg_grid grid;
  const void *words;
  double p[6];
  const double *aux[4]; /* auxiliary device fields (PG operators), else NULL */
} lsg_op;

/* Per right-hand-side PCG scalars (device memory, 16 doubles each). */
typedef struct {
  double atol;     /* max(atol, rtol*||b||) -- scipy cg stopping threshold */
  double rho;      /* r.z of the current iterate */
  double alpha;
  double beta;
  double rr;       /* ||r||^2 (recursive residual) */
  double pq;
  double bb;       /* ||b||^2 */
  double iters;    /* completed iterations */
  double done;     /* 1 once ||r|| < atol (or b == 0) */
  double zero_rhs; /* 1 if b == 0: x is returned as b (scipy cg semantics) */
  double maxiter;
  double first;    /* 1 until the first p = z has been formed */
  double rz_new;
  double reserved[3];
} lsg_pcg_scalars;

/* PCG workspace; every pointer is device memory owned by the caller.
 *   x, b, r, p, q, p_alt : k * n doubles each (n = dim * num_nodes);
 *   r_alt, q_alt  : k * n doubles each (2D), p_ring: k * n doubles (3D)
 *   scal          : k lsg_pcg_scalars
 *   partials      : k * lsg_partials_per_rhs() * 8 doubles
 *   counters      : k uint32, zero-initialised once by the caller
 *   dinv          : n doubles, lsg_inv_diag of the operator (shared by all k)
 * 2D runs one fused pass per iteration: it forms r_i = r_{i-1} - alpha q_{i-1},
 * z = M^-1 r_i, p_i = z + beta p_{i-1}, x += alpha p_{i-1} and q_i = A p_i with
 * neighbouring CTAs recomputing r_i and p_i in their halo, so r and p are
 * double-buffered (r/r_alt, p/p_alt).  The default pass recomputes
 * q_{i-1} = A p_{i-1} instead of reading it; q/q_alt are used by the small-
 * system persistent kernel and the stored-q variant.  3D runs an elementwise
 * pass that forms p, the stencil pass, and an update pass, with three
 * direction buffers (p, p_alt, p_ring); a batch of k >= 2 runs as two halves
 * on two streams (the caller's and a library-owned one per device, joined back
 * into the caller's stream).  lsg_pcg_iterate serialises its graph captures
 * and launches behind one lock; with LSG_NO_GRAPHS=1, calls from several host
 * threads on one device must not overlap.  `parity` (which buffers are current) is owned
 * by the library: lsg_pcg_start resets it, lsg_pcg_iterate advances it once
 * per iteration. */
typedef struct {
  int32_t k;
  int32_t parity;
  double *x;
  const double *b;
  double *r;
  double *p;
  double *q;
  lsg_pcg_scalars *scal;
  double *partials;
  uint32_t *counters;
  double *p_alt;
  const double *dinv; /* n doubles: inverse Jacobi diagonal from lsg_inv_diag */
  double *p_ring;     /* 3D: third direction buffer (k x n); x is updated every
                         second iteration with two directions at once */
  double *r_alt;      /* 2D: second residual buffer (k x n) */
  double *q_alt;      /* 2D: second A p buffer (k x n) */
} lsg_pcg_ws;

int32_t lsg_abi_version(void);
/* sizeof of the ABI structs as compiled into the library: bindings assert
 * their mirrors against these (lsg_op is 160 bytes: it ends in aux[4]). */
int64_t lsg_sizeof_op(void);
int64_t lsg_sizeof_pcg_ws(void);
int64_t lsg_sizeof_grid(void);
const char *lsg_last_error(void);
/* Number of kernels this library has launched in the process so far. */
int64_t lsg_launch_count(void);

/* Number of nodes / elements / blocks-per-rhs used by the reductions. */
int64_t lsg_num_nodes(const lsg_grid *g);
int64_t lsg_num_elements(const lsg_grid *g);
int64_t lsg_partials_per_rhs(const lsg_grid *g);

/* Mesh generation on the device -- replaces build_rect_mesh's arrays
 * (mesh.py:132-150): xyz (N, dim) coordinates bit-identical to np.linspace,
 * conn (E, dim+1) int32 element connectivity in the reference order. */
int lsg_mesh_vertices(const lsg_grid *g, double *xyz, void *stream);
int lsg_mesh_elements(const lsg_grid *g, int32_t *conn, void *stream);

/* Material words from the level set -- replaces MaterialIndicator.at_quad
 * + LevelSetField.indicator_quad (models/base.py:117-119, levelset.py:65-67).
 * phi: N doubles; bcmask: N bytes (bit c = Dirichlet on component c);
 * words: N uint8 (2D) / uint32 (3D). */
int lsg_material(const lsg_grid *g, const double *phi, const uint8_t *bcmask,
                 void *words, void *stream);

/* Per-quadrature-point indicator chi (E, nq) as doubles, for parity checks
 * against LevelSetField.indicator_quad (levelset.py:65-67). */
int lsg_indicator_quad(const lsg_grid *g, const double *phi, double *chi, void *stream);

/* Velocity-form words (H1 operator): frozen quadrature bits and the
 * zero-Dirichlet flag.  frozen_q: (E, nq) bytes (nonzero = inside the frozen
 * subdomain) or NULL; zero_dirichlet pins every boundary node. */
int lsg_h1_words(const lsg_grid *g, const uint8_t *frozen_q, int32_t zero_dirichlet,
                 void *words, void *stream);

/* y = A x for k stacked vectors -- replaces the CSR product K @ u of the
 * assembled, Dirichlet-eliminated operator (fem.py:141-150, 274-291). */
int lsg_apply(const lsg_op *op, int32_t k, const double *x, double *y, void *stream);

/* Jacobi diagonal of the eliminated operator (fem.py:303-305), n doubles. */
int lsg_diag(const lsg_op *op, double *diag, void *stream);
/* Its inverse as the PCG uses it: 1/d, with 1 where d == 0 (fem.py:303-305).
 * Shared by every right-hand side of a batch; computed once per operator. */
int lsg_inv_diag(const lsg_op *op, double *dinv, void *stream);

/* Batched Jacobi-PCG with scipy cg semantics (fem.py:294-316 via
 * scipy.sparse.linalg.cg): stop when ||r|| < max(atol, rtol*||b||), checked
 * before each iteration; b == 0 returns x = b.  x holds the warm start on
 * entry.  lsg_pcg_start computes r = b - A x and the stopping thresholds;
 * lsg_pcg_iterate enqueues `niter` more iterations (2D: one kernel each,
 * 3D: three); converged right-hand sides freeze.  Poll ws->scal (done, iters).
 * 2D: lsg_pcg_start zeroes ws->p (the first pass reads it as p_{-1}). */
int lsg_pcg_start(const lsg_op *op, lsg_pcg_ws *ws, double rtol, double atol,
                  double maxiter, void *stream);
int lsg_pcg_iterate(const lsg_op *op, lsg_pcg_ws *ws, int32_t niter, void *stream);
/* Diagnostics of the PCG chunk graphs (lsg_pcg_iterate replays CUDA graphs):
 * out4 = {cache hits, in-place updates, instantiations, host seconds spent
 * capturing + updating/instantiating}.  LSG_NO_GRAPHS=1 in the environment
 * launches the chunk kernels directly instead. */
void lsg_graph_stats(double *out4);

/* 2D: the single pass of iteration i forms x_i together with r_i, so nothing
 * is pending.  3D: the updates x += alpha p of iterations i-2 and i-1 are
 * folded into the elementwise pass of every even iteration i (directions
 * rotate through p, p_alt, p_ring), which halves the x traffic; a right-hand
 * side that has just converged has one or two updates pending.  Call
 * lsg_pcg_finish once after the last lsg_pcg_iterate, before reading x. */
int lsg_pcg_finish(const lsg_op *op, lsg_pcg_ws *ws, void *stream);

/* Fused compliance evaluation + shape-derivative right-hand side --
 * replaces ComplianceModel.cost/constraint/derivative (compliance.py:111-139,
 * base.py:150-158) + VelocitySolver._derivative_vector (velocity.py:129-142):
 *   vec_cost_a = sum_e |e| abar_e bulk_e grad N_a,
 *                bulk_e = sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I)
 *   vec_vol_a  = sum_e |e| (n_in/nq) / V grad N_a
 *   out[0] = J = sum_k sum_e |e| abar_e sigma_k:eps_k ; out[1] = int chi.
 * u: k fields; words from lsg_material; out: 2 doubles (device).
 * s1: reserved, pass NULL (the tensor itself never touches memory on the hot
 * path; lsg_s1_tensor materialises it for parity checks).
 * partials: lsg_partials_per_rhs() x 4 doubles; counter: one zero-initialised
 * uint32. */
int lsg_shape_rhs(const lsg_op *op, int32_t k, const double *u, double volume,
                  double *vec_cost, double *vec_vol, double *out, double *s1,
                  double *partials, uint32_t *counter, void *stream);

/* Thermal compliance and its shape derivative for k heat terms in one pass
 * (replaces HeatModel.cost / constraint / derivative, models/heat.py:124-166,
 * and the S0/S1 contraction of velocity.py:129-142).  op = LSG_OP_LAPLACE;
 * u = k temperature fields (k, N); weights = k host doubles (term weights);
 * fq = source samples at the quadrature points (k, E, 3) (device);
 * gq = source gradients (k, E, 3, 2) or NULL (S0 = 0).  Writes vec_cost and
 * vec_vol (2N each, velocity space) and out[0] = J, out[1] = subzero volume;
 * partials/counter as for lsg_shape_rhs. */
int lsg_heat_shape(const lsg_op *op, int32_t k, const double *u, const double *weights,
                   const double *fq, const double *gq, double volume, double *vec_cost,
                   double *vec_vol, double *out, double *partials, uint32_t *counter,
                   void *stream);

/* Inverse-elasticity model (models/inverse.py, 2D), k measurement pairs,
 * fields (k, 2N) interleaved.
 *
 * lsg_inverse_misfit replaces InverseElasticityModel._misfits / adjoint /
 * cost (inverse.py:180-233): with e = u - v - g and f = u - g it writes the
 * adjoint right-hand sides head = -alpha M e - beta M_G f (zeroed on the dofs
 * flagged in partial_mask, bit c = component c) and tail = alpha M e (zeroed
 * on the whole boundary), and out[0] = J = sum_k alpha/2 e.Me + beta/2 f.M_G f.
 * M = P1 mass (edge-midpoint rule), M_G = facet mass of the measured facets:
 * facet_flags[node] bit 0 = facet (node, node+1) measured, bit 1 = facet
 * (node, node+nx+1).  partials/counter: >= 1024 doubles / one uint32 (zero).
 *
 * lsg_inverse_tensors replaces InverseElasticityModel.derivative
 * (inverse.py:235-279): S0 (E,3,2) and S1 (E,3,2,2) at the quadrature points,
 * summed over the pairs; p, q = the two adjoint families; proj (k,3,2N) =
 * nodal projections of eps_xx, eps_xy, eps_yy of g stored as (value, 0);
 * A_q = a_in where phi < 0 at the point, a_out elsewhere.
 *
 * lsg_strain_projection_rhs writes the right-hand sides of those projections
 * (inverse.py:142-155): out (k,3,2N), sum over the triangles at a node of
 * |T|/3 eps_cc(g), as (value, 0). */
int lsg_inverse_misfit(const lsg_grid *g, int32_t k, const double *u, const double *v,
                       const double *measured, const uint8_t *facet_flags,
                       const uint8_t *partial_mask, double alpha, double beta, double *head,
                       double *tail, double *out, double *partials, uint32_t *counter,
                       void *stream);
int lsg_inverse_tensors(const lsg_grid *g, int32_t k, const double *u, const double *v,
                        const double *p, const double *q, const double *measured,
                        const double *proj, const double *phi, double a_in, double a_out,
                        double lam, double mu, double alpha, double *s0, double *s1,
                        void *stream);
int lsg_strain_projection_rhs(const lsg_grid *g, int32_t k, const double *measured, double *out,
                              void *stream);

/* S1 of the cost per element and quadrature point, (E, nq, dim, dim), for
 * parity with ComplianceModel.derivative's tensor (compliance.py:128-139):
 * S1_q = A_q sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I), A_q from phi. */
int lsg_s1_tensor(const lsg_op *op, int32_t k, const double *u, const double *phi, double *s1,
                  void *stream);

/* Generic tensor pair -> derivative vector (velocity.py:129-142):
 * vec_(a,c) = sum_q w_q (S0_q[c] N_a(x_q) + S1_q[c,:] . grad N_a);
 * s0: (E,nq,dim) or NULL, s1: (E,nq,dim,dim) or NULL. */
int lsg_tensor_rhs(const lsg_grid *g, const double *s0, const double *s1, double *vec,
                   void *stream);

/* b = -(vec_cost + lam * vec_vol), with Dirichlet dofs of the H1 operator
 * zeroed (velocity.py:144-148). */
int lsg_velocity_rhs(const lsg_op *h1, const double *vec_cost, const double *vec_vol,
                     double lam, double *b, void *stream);

/* Velocity statistics after the H1 solve (velocity.py:149-154):
 * out[0] = theta^T B theta, out[1] = vec . theta (vec = -b on free dofs,
 * passed explicitly), out[2] = max_i sum_d |theta_d,i| / h_d (CFL speed).
 * partials/counter as for lsg_shape_rhs. */
int lsg_velocity_stats(const lsg_op *h1, const double *theta, const double *vec,
                       double *out, double *partials, uint32_t *counter, void *stream);

/* Explicit level-set update (north star (4); replaces levelset.transport /
 * reinitialize, levelset.py:137-216).  Both run `nsub` forward-Euler
 * substeps of size dt, ping-ponging between phi_out and tmp; the result is in
 * phi_out.  transport: conservative face-velocity upwind + [smooth] h^2 lap.
 * reinit: Godunov, frozen S = phi0/sqrt(phi0^2+h^2) (sgn: N doubles scratch). */
int lsg_transport(const lsg_grid *g, const double *phi_in, const double *theta, double dt,
                  int32_t nsub, int32_t smooth, double h, double *phi_out, double *tmp,
                  void *stream);
int lsg_reinit(const lsg_grid *g, const double *phi_in, double dt, int32_t nsub, double h,
               double *phi_out, double *tmp, double *sgn, void *stream);

/* Reference-scheme reinitialisation right-hand side (levelset.py:205-212):
 * rhs = m_hat cur + dt (load + diffusion), PG_REINIT operator (aux[0..2]). */
int lsg_pg_reinit_rhs(const lsg_op *op, double *rhs, void *stream);

/* Solve A x = b for a PG operator to ||r|| <= rtol ||b|| (x holds the initial
 * guess) -- the reference factorises these matrices with splu
 * (levelset.py:165,204).  Right-Jacobi BiCGStab first; if it stagnates or
 * breaks down, restarted GMRES(48) with CGS2 from the same initial guess;
 * LSG_ERR_NOCONV if neither converges within maxit iterations.  Unlike the
 * other entry points it synchronises `stream` per iteration to test
 * convergence.  work: lsg_bicgstab_work_doubles(g) doubles of device memory. */
int64_t lsg_bicgstab_work_doubles(const lsg_grid *g);
int lsg_bicgstab(const lsg_op *op, const double *b, double *x, double *work, double rtol,
                 int32_t maxit, int32_t *iters, double *resid, void *stream);

/* max_i sum_d |v_d,i| / h_d over a vector field (CFL speed), out: 1 double. */
int lsg_cfl_speed(const lsg_grid *g, const double *v, double *out, double *partials,
                  uint32_t *counter, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LSGPU_H */
