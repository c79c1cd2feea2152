// 3D (Kuhn tetrahedra) kernels -- placeholder until the 3D marching kernels land.
#include "common.cuh"
#include "ops.h"

namespace lsg {
namespace d3 {

static int todo() {
  set_error("3D operators are not built in this revision");
  return LSG_ERR_ARG;
}

int64_t partials_per_rhs(const lsg_grid &) { return 1024; }
int apply(const lsg_op &, int, const double *, double *, cudaStream_t) { return todo(); }
int diag(const lsg_op &, double *, cudaStream_t) { return todo(); }
int inv_diag(const lsg_op &, double *, cudaStream_t) { return todo(); }
int pcg_start(const lsg_op &, lsg_pcg_ws &, double, double, double, cudaStream_t) { return todo(); }
int pcg_iterate(const lsg_op &, lsg_pcg_ws &, int, cudaStream_t) { return todo(); }
int shape_rhs(const lsg_op &, int, const double *, double, double *, double *, double *, double *,
              uint32_t *, cudaStream_t) { return todo(); }
int velocity_stats(const lsg_op &, const double *, const double *, double *, double *, uint32_t *,
                   cudaStream_t) { return todo(); }
int material(const lsg_grid &, const double *, const uint8_t *, void *, cudaStream_t) { return todo(); }
int indicator(const lsg_grid &, const double *, double *, cudaStream_t) { return todo(); }
int h1_words(const lsg_grid &, const uint8_t *, int, void *, cudaStream_t) { return todo(); }
int velocity_rhs(const lsg_op &, const double *, const double *, double, double *, cudaStream_t) { return todo(); }
int tensor_rhs(const lsg_grid &, const double *, const double *, double *, cudaStream_t) { return todo(); }
int s1_tensor(const lsg_op &, int, const double *, const double *, double *, cudaStream_t) { return todo(); }
int cfl_speed(const lsg_grid &, const double *, double *, double *, uint32_t *, cudaStream_t) { return todo(); }

}  // namespace d3
}  // namespace lsg
