// Host-side launchers for every kernel family (all stream-ordered, no syncs).
#pragma once

#include <cuda_runtime.h>

#include "ce_device.h"

cudaError_t ce_launch_direct(const CeSimtDesc& d, const float* A, const float* B, float* C, cudaStream_t s);
// out_span: elements of C zeroed before a split-K (atomic) reduction
cudaError_t ce_launch_reduce(const CeSimtDesc& d, const float* A, const float* B, float* C, int64_t out_span,
                             cudaStream_t s);
cudaError_t ce_launch_tiled(const CeSimtDesc& d, const float* A, const float* B, float* C, int a_kfast,
                            int b_kfast, cudaStream_t s);
// Family (c): pure axis permutation of a unary problem whose input and output unit-stride
// axes differ (smem-tiled transpose, coalesced on both sides).
bool ce_permute_supported(const CeProblem& p);
int ce_permute_describe(const CeProblem& p, char* buf, int n);  // diagnostics
int ce_stream_describe(const CeSimtDesc& d, char* buf, int n);  // diagnostics
cudaError_t ce_launch_permute(const CeProblem& p, const float* A, float* C, cudaStream_t s);
cudaError_t ce_launch_fill(float* dst, int64_t n, uint64_t seed, cudaStream_t s);
