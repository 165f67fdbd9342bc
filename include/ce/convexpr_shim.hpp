// convexpr_shim.hpp — the reference-side binding of libce (header-only C++).
//
// A `convexpr` user keeps calling the reference's by-value API and gets the B200 executor:
//
//   convexpr::ExecutionResult execute(const convexpr::EvaluationPlan&,
//                                     const std::vector<convexpr::DenseTensor>&)
//                                                     (sequencer.hpp:88, sequencer.cpp:403-447)
//   convexpr::DenseTensor pairwise_eval(const convexpr::DenseTensor&, const convexpr::DenseTensor&,
//                                       const convexpr::PairwiseOp&)      (kernels.hpp:105)
//
// are mirrored as convexpr_b200::execute / convexpr_b200::pairwise_eval with the same
// arguments (plus an optional ce_ctx).  The caller's plan is replayed EXACTLY: its node list
// (operand ids and each node's result order) and its per-atom ConvModeMap are handed to
// ce_plan_from_nodes, so left-to-right, from-joins, hand-edited and mixed-mode plans run the
// tree they describe.  Inputs are FP64 host tensors (rounded to FP32 on upload, as the device
// computes in FP32/TF32); outputs come back as FP64.  ExecutionResult.multiplications and
// peak_intermediate_elements are the reference's quantities (sum of flops_actual over the
// nodes, largest node result), computed by libce's bit-exact host IR.
// Errors: the reference's exception types (ParseError, ShapeError, PlanError, OverflowError)
// for the matching ce_status codes, std::runtime_error otherwise.
//
// Build: include this after the convexpr headers; link libce.so (cudart is inside it).
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ce/ce.h"
#include "convexpr/checked_int.hpp"
#include "convexpr/kernels.hpp"
#include "convexpr/sequencer.hpp"
#include "convexpr/tensor.hpp"

namespace convexpr_b200 {

inline void ce_throw(ce_status st) {
  if (st == CE_OK) return;
  const std::string msg = ce_last_error();
  switch (st) {
    case CE_ERR_PARSE: throw convexpr::ParseError(msg, 0);
    case CE_ERR_SHAPE: throw convexpr::ShapeError(msg);
    case CE_ERR_PLAN: throw convexpr::PlanError(msg);
    case CE_ERR_OVERFLOW: throw convexpr::OverflowError(msg);
    default: throw std::runtime_error("libce: " + msg);
  }
}

// One context (stream + workspace) per process on device 0 unless the caller passes its own.
inline ce_ctx* default_ctx() {
  static ce_ctx* ctx = [] {
    ce_ctx* c = nullptr;
    ce_options o{CE_MATH_AUTO, 1, nullptr};
    ce_throw(ce_ctx_create(0, &o, &c));
    return c;
  }();
  return ctx;
}

// ConvModeMap -> "h=same,w=circular" (ce.h's per-atom mode argument)
inline std::string mode_map(const convexpr::ConvModeMap& modes) {
  std::string s;
  for (const auto& [atom, mode] : modes) s += (s.empty() ? "" : ",") + ("(" + atom.name + ")=") + convexpr::to_string(mode);
  return s.empty() ? "same" : s;
}

struct PlanHandle {
  ce_plan* p = nullptr;
  ~PlanHandle() { ce_plan_destroy(p); }
};
struct ExecHandle {
  ce_executor* e = nullptr;
  ~ExecHandle() { ce_executor_destroy(e); }
};

inline convexpr::ExecutionResult execute(const convexpr::EvaluationPlan& plan,
                                         const std::vector<convexpr::DenseTensor>& inputs,
                                         ce_ctx* ctx = nullptr) {
  if (!ctx) ctx = default_ctx();
  const int n = static_cast<int>(plan.spec.inputs.size());
  if (static_cast<int>(inputs.size()) != n) throw convexpr::ShapeError("execute: wrong number of input tensors");
  for (int i = 0; i < n; ++i)
    if (inputs[static_cast<std::size_t>(i)].shape != plan.env.dims[static_cast<std::size_t>(i)])
      throw convexpr::ShapeError("execute: input " + std::to_string(i) + " shape mismatch");
  const std::string expr = convexpr::render(plan.spec);
  std::vector<int64_t> dims;
  std::vector<int> ranks;
  for (const auto& d : plan.env.dims) {
    dims.insert(dims.end(), d.begin(), d.end());
    ranks.push_back(static_cast<int>(d.size()));
  }
  std::vector<int> joins;
  std::vector<std::string> results;
  for (const auto& node : plan.nodes) {
    joins.push_back(node.left);
    joins.push_back(node.right);
    results.push_back(convexpr::render(node.op.result));
  }
  std::vector<const char*> res_ptrs;
  for (const auto& r : results) res_ptrs.push_back(r.c_str());
  PlanHandle p;
  ce_throw(ce_plan_from_nodes(expr.c_str(), dims.data(), ranks.data(), n, mode_map(plan.modes).c_str(),
                              convexpr::to_string(plan.cost_mode), joins.data(), res_ptrs.data(),
                              static_cast<int>(plan.nodes.size()), &p.p));
  ExecHandle ex;
  ce_throw(ce_executor_create(ctx, p.p, 0, &ex.e));
  std::vector<std::vector<float>> f32(inputs.size());
  std::vector<const float*> ptrs;
  for (std::size_t i = 0; i < inputs.size(); ++i) {
    f32[i].assign(inputs[i].data.begin(), inputs[i].data.end());
    ptrs.push_back(f32[i].data());
  }
  ce_plan_info info;
  ce_throw(ce_plan_get_info(p.p, &info));
  std::vector<int64_t> od(info.out_dims, info.out_dims + info.out_rank);
  convexpr::ExecutionResult r;
  r.output = convexpr::DenseTensor(od);
  std::vector<float> out(r.output.data.size());
  ce_throw(ce_execute_host(ex.e, ptrs.data(), out.data()));
  r.output.data.assign(out.begin(), out.end());
  r.multiplications = (static_cast<convexpr::u128>(info.flops_actual_hi) << 64) | info.flops_actual_lo;
  r.peak_intermediate_elements = info.peak_intermediate_elements;
  return r;
}

// pairwise_eval for an arbitrary PairwiseOp: the one-node plan "L,R->RESULT|convs" with the
// op's own result order and per-axis modes.
inline convexpr::DenseTensor pairwise_eval(const convexpr::DenseTensor& a, const convexpr::DenseTensor& b,
                                           const convexpr::PairwiseOp& op, ce_ctx* ctx = nullptr) {
  convexpr::ExpressionSpec spec;
  spec.inputs = {op.left, op.right};
  spec.output = op.result;
  for (const auto& ax : op.conv_axes) spec.conv_atoms.push_back(ax.atom);
  convexpr::EvaluationPlan plan;
  plan.spec = spec;
  plan.env.dims = {op.left_dims, op.right_dims};
  for (const auto& ax : op.conv_axes) plan.modes[ax.atom] = ax.mode;
  convexpr::PlanNode node;
  node.left = 0;
  node.right = 1;
  node.op = op;
  plan.nodes.push_back(node);
  return execute(plan, {a, b}, ctx).output;
}

}  // namespace convexpr_b200
