// Specialised pseudo-step paths (see wd_fused.cuh).
#include "wd_fused.cuh"

namespace wd {

void fused_plan(FusedPlan& fp, const FusedInputs& in) {
  fp.active = 0;
  fp.in = in;
}

void fused_step(const FusedPlan&, const double*, double*, Status*, double*, cudaStream_t) {}

void fused_release(FusedPlan& fp) { fp.active = 0; }

}  // namespace wd
