// Tensor-core (tcgen05, kind::tf32) implicit-GEMM path: plan + launcher.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_device.h"

struct TcPlan {
  int valid = 0;
};

// Decides whether a lowered problem maps onto the tcgen05 kernel and fills the plan.
bool ce_tc_plan(const CeProblem& p, TcPlan* out);
cudaError_t ce_launch_tc(const TcPlan& plan, const float* A, const float* B, float* C, cudaStream_t s);
