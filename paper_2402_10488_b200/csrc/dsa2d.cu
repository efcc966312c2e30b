// dsa2d.cu -- K5: consistent DSA for XY geometry (placeholder until the
// matrix-free Krylov solver lands).
#include "rte_internal.cuh"

namespace rte {
void dsa2d_setup(rte_ctx*, cudaStream_t) {
  throw Error(RTE_ERR_UNSUPPORTED, "dsa: xy geometry not implemented in this build");
}
void dsa2d_solve(rte_ctx*, const double*, double*, const int*, int, cudaStream_t) {
  throw Error(RTE_ERR_UNSUPPORTED, "dsa: xy geometry not implemented in this build");
}
void dsa2d_destroy(void*) {}
}  // namespace rte
