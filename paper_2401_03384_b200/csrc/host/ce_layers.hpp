// Tensorized-layer zoo (paper Appendix A): conv_einsum strings, factor shapes,
// parameter counts and rank-for-compression.  Same API/outputs as the reference
// proj/include/convexpr/layers.hpp:12-99; these produce every BASELINE config.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "ce_plan.hpp"

namespace ce {

enum class LayerKind {
  Standard, CP, RCP, TK, RTK, TT, RTT, TR, RTR, BT, HT, InterleavedGroup, SeparableDepthwise,
};
const char* to_string(LayerKind k);
LayerKind layer_kind_from_string(std::string_view s);
std::vector<LayerKind> all_layer_kinds();

struct LayerSpec {
  LayerKind kind = LayerKind::Standard;
  std::vector<int64_t> t_factors = {1};
  std::vector<int64_t> s_factors = {1};
  int64_t filter_h = 3, filter_w = 3;
  int64_t feature_h = 32, feature_w = 32;
  int64_t batch = 1;
  std::vector<int64_t> ranks;

  int64_t t_total() const;
  int64_t s_total() const;
  int order() const { return static_cast<int>(t_factors.size()); }
};

std::size_t rank_slot_count(LayerKind kind, int m);
void validate(const LayerSpec& layer);

struct LayerExpression {
  ExpressionSpec spec;
  ShapeEnv env;
  std::vector<std::string> tensor_names;
};

LayerExpression expression(const LayerSpec& layer);
u128 param_count(const LayerSpec& layer);
int64_t rank_for_compression(const LayerSpec& layer, double cr);
LayerSpec with_compression_rank(LayerSpec layer, double cr);
EvaluationPlan theorem_reduced_plan(const LayerSpec& layer, CostMode cost_mode = CostMode::Inference);
std::vector<std::pair<std::string, LayerSpec>> resnet34_cp_blocks(int64_t batch, double cr);
std::string layer_to_json(const LayerSpec& layer);

}  // namespace ce
