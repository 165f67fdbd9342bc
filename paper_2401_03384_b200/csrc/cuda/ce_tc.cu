// tcgen05 TF32 implicit-GEMM path (filled in by the tensor-core milestone).
#include "ce_tc.h"

bool ce_tc_plan(const CeProblem&, TcPlan* out) {
  out->valid = 0;
  return false;
}

cudaError_t ce_launch_tc(const TcPlan&, const float*, const float*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
