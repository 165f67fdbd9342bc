// Planner: FLOP-minimal pairwise evaluation trees (the conv-extended netcon
// sequencer).  Same API and bit-identical output as the reference
// proj/include/convexpr/sequencer.hpp:14-95 (optimal / left_to_right /
// enumerate_all / plan_from_joins / plan_cost / tree_encoding / plan_to_json).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "ce_ir.hpp"

namespace ce {

struct PlanError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct PlanNode {
  int left = -1, right = -1;  // operand ids: inputs 0..N-1, node j is N+j
  PairwiseOp op;
  u128 cost = 0;
};

struct EvaluationPlan {
  ExpressionSpec spec;
  ShapeEnv env;
  ConvModeMap modes;
  CostMode cost_mode = CostMode::Inference;
  std::vector<PlanNode> nodes;
  Subscripts root_subs;
  std::vector<int64_t> root_dims;
  u128 total_cost = 0;
  uint64_t peak_intermediate_elements = 0;
};

struct OptimalOptions {
  int max_inputs = 16;
  bool cost_capped = false;
};

EvaluationPlan left_to_right(const ExpressionSpec& spec, const ShapeEnv& env,
                             const ConvModeMap& modes, CostMode cost_mode = CostMode::Inference);
EvaluationPlan optimal(const ExpressionSpec& spec, const ShapeEnv& env, const ConvModeMap& modes,
                       CostMode cost_mode = CostMode::Inference, OptimalOptions options = {});
std::vector<EvaluationPlan> enumerate_all(const ExpressionSpec& spec, const ShapeEnv& env,
                                          const ConvModeMap& modes,
                                          CostMode cost_mode = CostMode::Inference);
EvaluationPlan plan_from_joins(const ExpressionSpec& spec, const ShapeEnv& env,
                               const ConvModeMap& modes, CostMode cost_mode,
                               const std::vector<std::pair<int, int>>& joins);
// A caller's plan replayed node by node (the reference's EvaluationPlan is a plain struct its
// callers may build or edit, sequencer.hpp:30-41): node j joins operand ids (left, right)
// (inputs 0..N-1, node k is N+k) and keeps exactly `results[j]`'s atoms in that order, i.e.
// make_pairwise_op(..., keep = set(results[j]), modes, results[j]) as the planner's node_op
// (sequencer.cpp:117-123).  Costs, total and peak are recomputed as build_plan does.
EvaluationPlan plan_from_nodes(const ExpressionSpec& spec, const ShapeEnv& env, const ConvModeMap& modes,
                               CostMode cost_mode, const std::vector<std::pair<int, int>>& joins,
                               const std::vector<Subscripts>& results);
u128 plan_cost(const EvaluationPlan& plan, CostMode mode);
std::string tree_encoding(const EvaluationPlan& plan);
std::string plan_to_json(const EvaluationPlan& plan);

}  // namespace ce
