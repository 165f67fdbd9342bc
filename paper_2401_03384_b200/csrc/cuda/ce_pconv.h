// Plane convolutions with few channels (see ce_pconv.cu): the steps of a convolution whose
// feature operand has its two gathered (spatial) axes innermost and whose filter is small --
// RTR conv1's X (3 planes of 112x112 per sample) against a 9-channel 7x7 filter, and that
// step's two adjoints.  On the tensor cores these need an explicit tap expansion (49x the
// input) or a col2im split; here a CTA stages one plane tile with its halo in shared memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_device.h"

#define CE_PCONV_MAXPL 4
#define CE_PCONV_MAXC 16

struct CePconvDesc {
  int32_t kind;  // 0: out[pl, y, x, co] = sum_{ci,i,j} F[pl, gather, ci] G[ci, co, i, j]
                 // 1: out[ci, co, i, j] = sum_{pl,y,x} F[pl, gather, ci] D[pl, y, x, co] (filter gradient)
  int32_t npl;   // plane vars (outermost first is not required: decoded by division)
  int64_t pl_ext[CE_PCONV_MAXPL], pl_sf[CE_PCONV_MAXPL], pl_so[CE_PCONV_MAXPL];  // so: C (kind 0) / D (kind 1)
  int64_t P;
  // positions y (axis 0) and x (axis 1): extent, stride in C (kind 0) / D (kind 1)
  int32_t OY, OX;
  int64_t sy, sx;
  // taps: extent, sign (feature index = position + sign * tap + c), stride in G (kind 0) / C (kind 1)
  int32_t KH, KW, sgn_h, sgn_w;
  int64_t ti, tj;
  // feature operand F: gathered axes' offsets, extents and strides
  int64_t c_h, c_w, H, W, fh, fw;
  int32_t Ci, Co;
  int64_t fci[CE_PCONV_MAXC];  // F strides of the ci values
  int64_t gci[CE_PCONV_MAXC];  // G (kind 0) / C (kind 1) strides of the ci values
  int64_t gco[CE_PCONV_MAXC];  // G (kind 0) / D (kind 1) strides of the co values
  int64_t cco[CE_PCONV_MAXC];  // C strides of the co values
  int32_t accumulate;          // kind 0: C += result
  int32_t tiles_y, tiles_x;    // CTA tiles per plane
  int64_t items;               // kind 1: work items (plane x tile), CTAs
  int32_t ctas;
};

// Structure check + descriptor for one lowered problem (F = operand A, G / D = operand B).
bool ce_pconv_plan(const CeProblem& p, CePconvDesc* out);
// kind 1 accumulates into C with atomics: the caller zeroes C first (unless accumulating).
cudaError_t ce_launch_pconv(const CePconvDesc& d, const float* F, const float* G, float* C, cudaStream_t s);
