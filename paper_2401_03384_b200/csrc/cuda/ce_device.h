// Device problem descriptor shared by the host lowering (csrc/host/ce_lower.cpp)
// and every kernel family.
//
// Every pairwise step the executor runs — the forward node of
// pairwise_eval (reference kernels.cpp:425-470) and the two adjoint nodes
// (input / factor gradient) — is lowered to ONE generalized form:
//
//   out[z, m, n] (+)= sum_k  A[z, m, k] * B[z, n, k]
//
// over integer index variables ("vars"), each of class Z (batch: A, B, out),
// M (A and out), N (B and out) or K (A and B, summed).  A var is a single
// atom, a merged group of atoms is never needed because operands keep their
// own strides.  An operand axis is either PLAIN (index = one var, memory
// offset = value * stride) or GATHERED (a convolution feature axis):
//
//   idx = sp * value(pv) + sq * value(qv) + c      (pv in M/N, qv in K)
//   wrap == 0 : term contributes 0 unless 0 <= idx < extent  (Full/Same/Valid)
//   wrap == 1 : idx taken modulo extent                       (Circular)
//
// which restates feature_index() (kernels.cpp:298-315) for the forward node
// and its exact adjoints for the gradient nodes.
#pragma once

#include <stdint.h>

#define CE_MAX_VARS 16
#define CE_MAX_GATHER 4

enum CeVarClass { CE_Z = 0, CE_M = 1, CE_N = 2, CE_K = 3 };

struct CeGather {
  int32_t pv, qv;   // var indices
  int32_t sp, sq;   // +1 / -1
  int64_t c;        // constant offset
  int64_t extent;   // feature length (bounds or modulus)
  int64_t stride;   // element stride of the gathered axis
  int32_t wrap;
  int32_t pad_;
};

struct CeProblem {
  int32_t nv;
  int32_t unary;        // 1: no B operand (pure reduce / broadcast / permute)
  int32_t accumulate;   // 1: out += result (split-K partial sums / grad accumulation)
  int32_t ng_a, ng_b;
  int64_t ext[CE_MAX_VARS];
  int32_t cls[CE_MAX_VARS];
  int64_t sa[CE_MAX_VARS];   // plain stride of var v in A (0 = absent)
  int64_t sb[CE_MAX_VARS];   // plain stride of var v in B
  int64_t sc[CE_MAX_VARS];   // stride of var v in out (Z/M/N vars only)
  CeGather ga[CE_MAX_GATHER];
  CeGather gb[CE_MAX_GATHER];
  // 1: that operand is a caller-owned buffer with no slack past its logical span (set per
  // launch), so no float4 access may run past a row whose extent is not a multiple of 4
  // (workspace buffers are allocated in 256-B units and padded per row)
  int32_t exact_a, exact_b, exact_c;
};

// Compact per-class var lists the SIMT kernels iterate over (built on host).
struct CeSimtDesc {
  CeProblem p;
  int32_t nz, nm, nn, nk;
  int32_t zv[CE_MAX_VARS], mv[CE_MAX_VARS], nvv[CE_MAX_VARS], kv[CE_MAX_VARS];
  int64_t Z, M, N, K;  // products of extents per class
  // direct kernel: output vars ordered fastest-first (host sorts by out stride)
  int32_t nout;
  int32_t ov[CE_MAX_VARS];
};
