// TEST INFRASTRUCTURE ONLY — never part of the product.
//
// Compiles include/ce/convexpr_shim.hpp (the reference-side binding a convexpr maintainer
// would add) against the UNMODIFIED reference headers and library objects
// (oracle/Makefile builds them in place from /root/reference/proj) and libce.so, then, for a
// set of plans the reference itself builds -- optimal, left_to_right, plan_from_joins, a
// hand-edited node result order, explicit per-atom Full/Valid/Circular mode maps, a
// multi-way (forced circular) atom, a self-contraction -- runs
//   convexpr::execute(plan, inputs)        (the reference, FP64 CPU)
//   convexpr_b200::execute(plan, inputs)   (libce through the shim, FP32/TF32 on the GPU)
// and a single convexpr::pairwise_eval vs convexpr_b200::pairwise_eval, printing one JSON
// line per case: normwise max error, and whether multiplications / peak / output shape are
// identical.  tests/test_integration_shim.py builds it (CPU) and runs it (GPU).
//   shim_check [--math fp32|auto]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "convexpr/expression.hpp"
#include "convexpr/kernels.hpp"
#include "convexpr/sequencer.hpp"
#include "convexpr/tensor.hpp"
#include "ce/convexpr_shim.hpp"

using namespace convexpr;

namespace {

double nerr(const DenseTensor& y, const DenseTensor& ref) {
  double num = 0, den = 1e-300;
  for (std::size_t i = 0; i < ref.data.size(); ++i) {
    num = std::max(num, std::fabs(y.data[i] - ref.data[i]));
    den = std::max(den, std::fabs(ref.data[i]));
  }
  return num / den;
}

std::vector<DenseTensor> inputs_for(const ShapeEnv& env, uint64_t seed) {
  std::vector<DenseTensor> ts;
  for (std::size_t i = 0; i < env.dims.size(); ++i) {
    DenseTensor t = fill_random(env.dims[i], seed + i);
    for (double& v : t.data) v = static_cast<double>(static_cast<float>(v));  // what the device sees
    ts.push_back(std::move(t));
  }
  return ts;
}

void report(const char* name, const EvaluationPlan& plan, ce_ctx* ctx) {
  auto ins = inputs_for(plan.env, 1000);
  ExecutionResult ref = execute(plan, ins);
  ExecutionResult got = convexpr_b200::execute(plan, ins, ctx);
  const bool shape_ok = got.output.shape == ref.output.shape;
  std::printf(
      "{\"case\": \"%s\", \"tree\": \"%s\", \"err\": %.3e, \"shape_equal\": %s, \"mults_equal\": %s, "
      "\"peak_equal\": %s, \"mults\": \"%s\"}\n",
      name, plan.nodes.empty() ? "0" : tree_encoding(plan).c_str(), shape_ok ? nerr(got.output, ref.output) : 1e30,
      shape_ok ? "true" : "false", got.multiplications == ref.multiplications ? "true" : "false",
      got.peak_intermediate_elements == ref.peak_intermediate_elements ? "true" : "false",
      to_decimal_string(ref.multiplications).c_str());
}

EvaluationPlan make(const std::string& expr, std::vector<std::vector<int64_t>> dims, ConvMode mode, CostMode cm,
                    int which, const std::vector<std::pair<int, int>>& joins = {}) {
  ExpressionSpec spec = parse(expr);
  ShapeEnv env = make_shape_env(spec, std::move(dims));
  ConvModeMap modes = resolve_conv_modes(spec, mode);
  if (which == 1) return left_to_right(spec, env, modes, cm);
  if (which == 2) return plan_from_joins(spec, env, modes, cm, joins);
  return optimal(spec, env, modes, cm);
}

}  // namespace

int main(int argc, char** argv) {
  int math = CE_MATH_AUTO;
  for (int i = 1; i + 1 < argc; ++i)
    if (!std::strcmp(argv[i], "--math")) math = std::strcmp(argv[i + 1], "fp32") == 0 ? CE_MATH_FP32_SIMT : CE_MATH_AUTO;
  ce_ctx* ctx = nullptr;
  ce_options o{math, 1, nullptr};
  if (ce_ctx_create(0, &o, &ctx) != CE_OK) {
    std::fprintf(stderr, "ce_ctx_create: %s\n", ce_last_error());
    return 2;
  }
  const std::string cp = "bshw,rt,rs,rh,rw->bthw|hw";
  const std::vector<std::vector<int64_t>> cpd = {{4, 12, 10, 9}, {6, 10}, {6, 12}, {6, 3}, {6, 3}};
  try {
    report("cp optimal same inference", make(cp, cpd, ConvMode::Same, CostMode::Inference, 0), ctx);
    report("cp optimal same training", make(cp, cpd, ConvMode::Same, CostMode::Training, 0), ctx);
    report("cp left_to_right same", make(cp, cpd, ConvMode::Same, CostMode::Inference, 1), ctx);
    report("cp from_joins full", make(cp, cpd, ConvMode::Full, CostMode::Inference, 2, {{0, 3}, {5, 4}, {6, 2}, {7, 1}}),
           ctx);
    report("cp optimal valid", make(cp, cpd, ConvMode::Valid, CostMode::Inference, 0), ctx);
    report("cp optimal circular", make(cp, cpd, ConvMode::Circular, CostMode::Inference, 0), ctx);
    {
      // mixed per-atom modes (h full, w circular) on the optimal tree
      ExpressionSpec spec = parse(cp);
      ShapeEnv env = make_shape_env(spec, cpd);
      ConvModeMap modes{{Atom("h"), ConvMode::Full}, {Atom("w"), ConvMode::Circular}};
      report("cp optimal mixed h=full w=circular", optimal(spec, env, modes, CostMode::Inference), ctx);
      // a hand-edited plan: node 0's result order reversed (still keeps every needed atom)
      EvaluationPlan p = optimal(spec, env, resolve_conv_modes(spec, ConvMode::Same), CostMode::Inference);
      Subscripts rev(p.nodes[0].op.result.rbegin(), p.nodes[0].op.result.rend());
      std::set<Atom> keep(rev.begin(), rev.end());
      const PairwiseOp op0 = p.nodes[0].op;
      p.nodes[0].op = make_pairwise_op(op0.left, op0.left_dims, op0.right, op0.right_dims, keep, p.modes, rev);
      // downstream nodes consume the reordered operand: rebuild them with their own result orders
      std::vector<Subscripts> subs(spec.inputs.begin(), spec.inputs.end());
      std::vector<std::vector<int64_t>> dims(env.dims.begin(), env.dims.end());
      subs.push_back(p.nodes[0].op.result);
      dims.push_back(p.nodes[0].op.result_dims);
      for (std::size_t j = 1; j < p.nodes.size(); ++j) {
        PlanNode& nd = p.nodes[j];
        std::set<Atom> k(nd.op.result.begin(), nd.op.result.end());
        nd.op = make_pairwise_op(subs[static_cast<std::size_t>(nd.left)], dims[static_cast<std::size_t>(nd.left)],
                                 subs[static_cast<std::size_t>(nd.right)], dims[static_cast<std::size_t>(nd.right)], k,
                                 p.modes, nd.op.result);
        subs.push_back(nd.op.result);
        dims.push_back(nd.op.result_dims);
      }
      report("cp hand-edited result order", p, ctx);
    }
    // multi-way conv atom (x in three inputs -> forced circular) and a self-contraction
    report("three-way circular", make("ax,bx,cx->abx|x", {{3, 8}, {4, 8}, {5, 8}}, ConvMode::Same, CostMode::Inference, 0),
           ctx);
    report("self-contraction", make("abc,cd->ad", {{3, 4, 5}, {5, 6}}, ConvMode::Same, CostMode::Inference, 0), ctx);
    report("tk layer training", make("bshw,(r1)t,(r2)s,(r1)(r2)hw->bthw|hw", {{2, 16, 7, 7}, {5, 12}, {6, 16}, {5, 6, 3, 3}},
                                     ConvMode::Same, CostMode::Training, 0),
           ctx);
    {
      // pairwise_eval with an op the planner would not build (result order permuted)
      ExpressionSpec spec = parse("bhwr,rh->bhwr|h");
      ShapeEnv env = make_shape_env(spec, {{2, 9, 5, 4}, {4, 3}});
      Subscripts res = {Atom("r"), Atom("w"), Atom("b"), Atom("h")};
      std::set<Atom> keep(res.begin(), res.end());
      PairwiseOp op = make_pairwise_op(spec.inputs[0], env.dims[0], spec.inputs[1], env.dims[1], keep,
                                       resolve_conv_modes(spec, ConvMode::Valid), res);
      auto ins = inputs_for(env, 7);
      DenseTensor ref = pairwise_eval(ins[0], ins[1], op);
      DenseTensor got = convexpr_b200::pairwise_eval(ins[0], ins[1], op, ctx);
      std::printf("{\"case\": \"pairwise_eval custom result order valid\", \"tree\": \"(0 1)\", \"err\": %.3e, "
                  "\"shape_equal\": %s, \"mults_equal\": true, \"peak_equal\": true, \"mults\": \"%s\"}\n",
                  got.shape == ref.shape ? nerr(got, ref) : 1e30, got.shape == ref.shape ? "true" : "false",
                  to_decimal_string(flops_actual(op)).c_str());
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "shim_check: %s\n", e.what());
    return 1;
  }
  ce_ctx_destroy(ctx);
  return 0;
}
