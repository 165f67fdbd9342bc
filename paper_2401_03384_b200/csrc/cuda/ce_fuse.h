// Fused kernels along plan chains, see ce_fuse.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_device.h"
#include "ce_tc.h"  // TcDiv

#define CE_DW2_OUTER 4

// Two chained depthwise stencils Y0 -(axis u, filter Fa)-> Y1 -(axis v, filter Fb)-> Y2 over a
// unit-stride lane axis r (see ce_fuse.cu).  Strides in elements.
struct CeDw2Desc {
  int32_t KT, J, SA, SB;        // taps (both steps), outputs per thread, tap signs
  int32_t lq, njb;              // CTA tile: lane quads, blocks of J outputs along w
  int32_t R;                    // lane extent
  TcDiv dr4, dwb, du;           // lane chunks, w tiles, u tiles (CTA grid)
  int32_t U;                    // extent along u
  int32_t nouter;
  TcDiv odiv[CE_DW2_OUTER];
  int64_t os0[CE_DW2_OUTER], os1[CE_DW2_OUTER], os2[CE_DW2_OUTER];  // outer strides in Y0 / Y1 / Y2
  uint32_t threads;             // CTAs
  int32_t ca, Xa;               // first gather: x = ca + u + SA*p in [0, Xa), Y0 stride a0
  int64_t a0, v0;               // Y0 strides of the gathered axis u and of the axis v
  int64_t u1, u2;               // Y1 / Y2 strides of u
  int32_t cb, Xb;               // second gather: x = cb + w + SB*q in [0, Xb), Y1 stride v1
  int64_t v1;
  int32_t W;                    // output extent along w, Y2 stride w2
  int64_t w2;
  int32_t fa_r, fa_q, fb_r, fb_q;  // filter strides (lane, tap)
  int32_t write_mid;            // 1: Y1 is stored too (a later step reads it)
};

// Structure check + descriptor for two lowered problems (p2 reads p1's output as its A).
bool ce_dw2_plan(const CeProblem& p1, const CeProblem& p2, bool write_mid, CeDw2Desc* out);
cudaError_t ce_launch_dw2(const CeDw2Desc& d, const float* Y0, const float* Fa, const float* Fb, float* Y1, float* Y2,
                          cudaStream_t s);

// 3xTF32 operand split: hi = TF32(x) (round to nearest), lo = x - hi, n elements.
cudaError_t ce_launch_split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s);
