// fo_owner.cu -- placeholder, replaced by the patch kernel
#include "fo_kernels.cuh"
namespace fo {
fo_status build_patch_plan(fo_mesh m) { m->plan.n_patches = 0; m->scatter = FO_SCATTER_ATOMIC; return FO_OK; }
fo_status launch_owner(fo_mesh, const double*, double*, double*, cudaStream_t) {
  set_error("owner kernel not built"); return FO_ESTATE; }
}
