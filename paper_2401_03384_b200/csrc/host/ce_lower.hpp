// Lowering of one pairwise node (forward, or one of its two adjoints) onto the
// generalized device problem of csrc/cuda/ce_device.h.
#pragma once

#include <vector>

#include "../cuda/ce_device.h"
#include "ce_ir.hpp"

namespace ce {

// A strided view of a tensor whose axes carry the atoms of `subs`.
struct View {
  Subscripts subs;
  std::vector<int64_t> dims;
  std::vector<int64_t> strides;  // elements
};

View dense_view(const Subscripts& subs, const std::vector<int64_t>& dims);
// Row-major with the innermost pitch rounded up to a multiple of `align`
// elements (16-byte rows for TMA legality, SURVEY §7 "TMA legality").
View padded_view(const Subscripts& subs, const std::vector<int64_t>& dims, int64_t align);
int64_t view_span(const View& v);  // elements to allocate

enum class Adjoint { Forward, GradLeft, GradRight };

// Forward:   out = op(A, B)            (A: left post-self-sum, B: right)
// GradLeft:  out = dA from (dC, B)     (a = left view only for shape/subs, c = dC)
// GradRight: out = dB from (A, dC)
// The returned problem's A/B operand pointers are, respectively:
//   Forward (A, B), GradLeft (dC, B), GradRight (A, dC).
CeProblem lower_pairwise(const PairwiseOp& op, const View& left, const View& right, const View& result,
                         const View& out, Adjoint which);

// out[atoms of out] = sum over atoms of `in` missing from out; atoms of out
// missing from `in` broadcast.  Restates sum_unique_modes (kernels.cpp:144-187)
// plus permute (tensor.cpp:50-94) and their adjoint (broadcast).
CeProblem lower_unary(const View& in, const View& out);

// Builds the per-class var lists and iteration orders the SIMT kernels need.
CeSimtDesc simt_desc(const CeProblem& p);

}  // namespace ce
