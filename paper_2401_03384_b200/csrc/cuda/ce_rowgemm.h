// Row GEMMs with few contracted and few output columns (see ce_rowgemm.cu): out[m, n] =
// sum_k A[m, k] B[k, n] over millions of rows m with K, N <= 32 (K x N <= 256) and a small B -- the rank
// contractions of the reshaped-ring layers' pixel tensors (RTR conv1: 3.2M pixels x 4, K = 9,
// N = 16).  On the tensor cores each 128-row tile pads K to 32 and pays an epilogue for a
// handful of columns.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_device.h"

#define CE_ROW_MAXV 8
#define CE_ROW_MAXKN 32

struct CeRowDesc {
  int32_t nm;                    // M vars, fastest first (the first is C's unit-stride one)
  int64_t m_ext[CE_ROW_MAXV], m_sa[CE_ROW_MAXV], m_sc[CE_ROW_MAXV];
  int64_t M;
  int32_t K, N;
  int64_t ka[CE_ROW_MAXKN], kb[CE_ROW_MAXKN];  // A / B offsets of the K values
  int64_t nb[CE_ROW_MAXKN], nc[CE_ROW_MAXKN];  // B / C offsets of the N values
  int32_t accumulate;
};

bool ce_rowgemm_plan(const CeProblem& p, CeRowDesc* out);
cudaError_t ce_launch_rowgemm(const CeRowDesc& d, const float* A, const float* B, float* C, cudaStream_t s);
