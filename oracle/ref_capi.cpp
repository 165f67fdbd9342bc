// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libconvexpr_ref.so).  tests/ and bench.py's reference arm load it
// with ctypes to (a) pin the planner/cost/layer outputs bit-exactly, (b) pin the
// numpy restatement in oracle/np_oracle.py, and (c) time the reference CPU
// executor (`execute`, sequencer.cpp:403-447) as the CPU baseline.
//
// Every entry point returns 0 on success and a SPEC-style status otherwise
// (2 parse, 3 shape, 4 numeric, 5 plan, 6 overflow, 1 other); the message is
// available from ref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <exception>
#include <string>
#include <vector>

#include "convexpr/cost.hpp"
#include "convexpr/expression.hpp"
#include "convexpr/kernels.hpp"
#include "convexpr/layers.hpp"
#include "convexpr/reference.hpp"
#include "convexpr/sequencer.hpp"
#include "convexpr/tensor.hpp"

using namespace convexpr;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    return fail(2, e.what());
  } catch (const ShapeError& e) {
    return fail(3, e.what());
  } catch (const PlanError& e) {
    return fail(5, e.what());
  } catch (const OverflowError& e) {
    return fail(6, e.what());
  } catch (const std::exception& e) {
    return fail(1, e.what());
  }
}

void put(const std::string& s, char* out, int cap) {
  if (static_cast<int>(s.size()) + 1 > cap) throw std::runtime_error("output buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
}

std::vector<std::vector<int64_t>> unflatten(const int64_t* dims, const int* ranks, int n) {
  std::vector<std::vector<int64_t>> out;
  int64_t pos = 0;
  for (int i = 0; i < n; ++i) {
    out.emplace_back(dims + pos, dims + pos + ranks[i]);
    pos += ranks[i];
  }
  return out;
}

std::string u128s(u128 v) { return to_decimal_string(v); }

struct Problem {
  ExpressionSpec spec;
  ShapeEnv env;
  ConvModeMap modes;
};

Problem make_problem(const char* expr, const int64_t* dims, const int* ranks, int n,
                     const char* mode) {
  Problem p;
  p.spec = parse(expr);
  p.env = make_shape_env(p.spec, unflatten(dims, ranks, n));
  p.modes = resolve_conv_modes(p.spec, conv_mode_from_string(mode));
  return p;
}

std::vector<DenseTensor> wrap_inputs(const Problem& p, const double* const* inputs) {
  std::vector<DenseTensor> ts;
  for (std::size_t i = 0; i < p.env.dims.size(); ++i) {
    DenseTensor t(p.env.dims[i]);
    std::memcpy(t.data.data(), inputs[i], sizeof(double) * t.data.size());
    ts.push_back(std::move(t));
  }
  return ts;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Plan JSON (sequencer.cpp:466-480) + "\n" + tree encoding + "\n" + training/inference
// plan_cost of the chosen tree.  which: 0 optimal, 1 left_to_right.
int ref_plan(const char* expr, const int64_t* dims, const int* ranks, int n, const char* mode,
             const char* cost_mode, int which, int capped, char* out, int cap) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    CostMode cm = cost_mode_from_string(cost_mode);
    EvaluationPlan plan;
    if (which == 0) {
      OptimalOptions o;
      o.cost_capped = capped != 0;
      plan = optimal(p.spec, p.env, p.modes, cm, o);
    } else {
      plan = left_to_right(p.spec, p.env, p.modes, cm);
    }
    std::string s = plan_to_json(plan);
    s += "\n";
    s += plan.nodes.empty() ? std::string("0") : tree_encoding(plan);
    s += "\n" + u128s(plan_cost(plan, CostMode::Inference)) + " " +
         u128s(plan_cost(plan, CostMode::Training));
    put(s, out, cap);
  });
}

// Number of trees and the minimum cost over enumerate_all (sequencer.cpp:343-362).
int ref_enumerate(const char* expr, const int64_t* dims, const int* ranks, int n, const char* mode,
                  const char* cost_mode, char* out, int cap) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    auto plans = enumerate_all(p.spec, p.env, p.modes, cost_mode_from_string(cost_mode));
    u128 best = 0;
    bool first = true;
    for (const auto& pl : plans) {
      if (first || pl.total_cost < best) best = pl.total_cost;
      first = false;
    }
    put(std::to_string(plans.size()) + " " + u128s(best), out, cap);
  });
}

// Reference execute() (sequencer.cpp:403-447) on caller FP64 buffers.  info gets
// "multiplications peak_elems seconds".
int ref_execute(const char* expr, const int64_t* dims, const int* ranks, int n, const char* mode,
                int which, const double* const* inputs, double* out, int64_t out_cap, char* info,
                int cap) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    EvaluationPlan plan = which == 0 ? optimal(p.spec, p.env, p.modes, CostMode::Inference)
                                     : left_to_right(p.spec, p.env, p.modes, CostMode::Inference);
    auto ts = wrap_inputs(p, inputs);
    auto t0 = std::chrono::steady_clock::now();
    ExecutionResult r = execute(plan, ts);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (r.output.size() > out_cap) throw std::runtime_error("output buffer too small");
    std::memcpy(out, r.output.data.data(), sizeof(double) * r.output.data.size());
    put(u128s(r.multiplications) + " " + std::to_string(r.peak_intermediate_elements) + " " +
            std::to_string(secs),
        info, cap);
  });
}

// Timing helper for the CPU baseline: plans once (cost_mode), then runs execute()
// `reps` times and reports the best wall time in seconds (steady_clock).
int ref_time_execute(const char* expr, const int64_t* dims, const int* ranks, int n,
                     const char* mode, const char* cost_mode, const double* const* inputs,
                     int reps, double* best_seconds) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    EvaluationPlan plan = optimal(p.spec, p.env, p.modes, cost_mode_from_string(cost_mode));
    auto ts = wrap_inputs(p, inputs);
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      ExecutionResult r = execute(plan, ts);
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (s < best) best = s;
      if (r.output.size() < 1) throw std::runtime_error("empty output");
    }
    *best_seconds = best;
  });
}

// As ref_time_execute, and also returns ExecutionResult.multiplications (the sum of
// flops_actual over the executed nodes, sequencer.cpp:429) as a decimal string in `mults`.
int ref_time_execute2(const char* expr, const int64_t* dims, const int* ranks, int n, const char* mode,
                      const char* cost_mode, const double* const* inputs, int reps, double* best_seconds,
                      char* mults, int cap) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    EvaluationPlan plan = optimal(p.spec, p.env, p.modes, cost_mode_from_string(cost_mode));
    auto ts = wrap_inputs(p, inputs);
    double best = 1e30;
    u128 m = 0;
    for (int i = 0; i < reps; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      ExecutionResult r = execute(plan, ts);
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (s < best) best = s;
      m = r.multiplications;
    }
    *best_seconds = best;
    put(u128s(m), mults, cap);
  });
}

// reference::eval (reference.cpp:76-222): brute-force nested sum.
int ref_eval_brute(const char* expr, const int64_t* dims, const int* ranks, int n,
                   const char* mode, const double* const* inputs, double* out, int64_t out_cap) {
  return guard([&] {
    Problem p = make_problem(expr, dims, ranks, n, mode);
    auto ts = wrap_inputs(p, inputs);
    DenseTensor r = reference::eval(p.spec, p.env, p.modes, ts);
    if (r.size() > out_cap) throw std::runtime_error("output buffer too small");
    std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
  });
}

// One pairwise op built exactly as the planner builds nodes (sequencer.cpp:118-124):
// expr "L,R->RES|convs"; keep = RES atoms; result order = RES.  Runs pairwise_eval
// (kernels.cpp:425-470).  info: "flops_actual fwd g1 g2 result_dims..." (training costs).
int ref_pairwise(const char* expr, const int64_t* dims, const int* ranks, const char* mode,
                 const double* a, const double* b, double* out, int64_t out_cap, char* info,
                 int cap) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    if (spec.inputs.size() != 2) throw std::runtime_error("ref_pairwise needs two inputs");
    auto d = unflatten(dims, ranks, 2);
    ConvModeMap modes = resolve_conv_modes(spec, conv_mode_from_string(mode));
    std::set<Atom> keep(spec.output.begin(), spec.output.end());
    PairwiseOp op = make_pairwise_op(spec.inputs[0], d[0], spec.inputs[1], d[1], keep, modes,
                                     spec.output);
    std::string s = u128s(flops_actual(op));
    CostBreakdown cb = pairwise_cost(op, CostMode::Training);
    s += " " + u128s(cb.forward) + " " + u128s(cb.g1) + " " + u128s(cb.g2);
    for (auto x : op.result_dims) s += " " + std::to_string(x);
    if (a && b && out) {
      DenseTensor ta(d[0]), tb(d[1]);
      std::memcpy(ta.data.data(), a, sizeof(double) * ta.data.size());
      std::memcpy(tb.data.data(), b, sizeof(double) * tb.data.size());
      DenseTensor r = pairwise_eval(ta, tb, op);
      if (r.size() > out_cap) throw std::runtime_error("output buffer too small");
      std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    }
    put(s, info, cap);
  });
}

// Layer zoo (layers.cpp): descriptor JSON in, "expr\n[[dims]..]\nparam_count\nranks" out.
// cr > 0 applies with_compression_rank first.
int ref_layer(const char* layer_json, double cr, char* out, int cap) {
  return guard([&] {
    LayerSpec l = layer_from_json(layer_json);
    if (cr > 0) l = with_compression_rank(l, cr);
    LayerExpression ex = expression(l);
    std::string s = render(ex.spec) + "\n[";
    for (std::size_t i = 0; i < ex.env.dims.size(); ++i) {
      s += i ? ",[" : "[";
      for (std::size_t j = 0; j < ex.env.dims[i].size(); ++j)
        s += (j ? "," : "") + std::to_string(ex.env.dims[i][j]);
      s += "]";
    }
    s += "]\n" + u128s(param_count(l)) + "\n";
    for (std::size_t i = 0; i < l.ranks.size(); ++i) s += (i ? " " : "") + std::to_string(l.ranks[i]);
    put(s, out, cap);
  });
}

// theorem_reduced_plan (layers.cpp:374-398) JSON + tree encoding.
int ref_theorem_plan(const char* layer_json, const char* cost_mode, char* out, int cap) {
  return guard([&] {
    LayerSpec l = layer_from_json(layer_json);
    EvaluationPlan plan = theorem_reduced_plan(l, cost_mode_from_string(cost_mode));
    put(plan_to_json(plan) + "\n" + tree_encoding(plan), out, cap);
  });
}

// resnet34_cp_blocks (layers.cpp:400-423): one layer_to_json per line.
int ref_resnet34(int64_t batch, double cr, char* out, int cap) {
  return guard([&] {
    std::string s;
    for (auto& [name, l] : resnet34_cp_blocks(batch, cr)) s += name + " " + layer_to_json(l) + "\n";
    put(s, out, cap);
  });
}

// fill_random (tensor.cpp:125-130).
int ref_fill_random(const int64_t* shape, int rank, uint64_t seed, double* out) {
  return guard([&] {
    DenseTensor t = fill_random(std::vector<int64_t>(shape, shape + rank), seed);
    std::memcpy(out, t.data.data(), sizeof(double) * t.data.size());
  });
}

// parse/render/classify (expression.cpp): "render\natom:class ..." in map order.
int ref_parse(const char* expr, char* out, int cap) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    std::string s = render(spec) + "\n";
    bool first = true;
    for (auto& [a, c] : classify(spec)) {
      s += (first ? "" : " ") + a.name + ":" + to_string(c);
      first = false;
    }
    put(s, out, cap);
  });
}

// Wire formats (tensor.cpp:132-186, layers.cpp:425-467), for the F3 parity tests.
int ref_tensor_to_json(const int64_t* shape, int rank, const double* data, char* out, int cap) {
  return guard([&] {
    DenseTensor t(std::vector<int64_t>(shape, shape + rank));
    std::memcpy(t.data.data(), data, sizeof(double) * t.data.size());
    put(tensor_to_json(t), out, cap);
  });
}

int ref_tensor_from_json(const char* text, int64_t* shape, int* rank, double* data, int64_t cap, int64_t* count) {
  return guard([&] {
    DenseTensor t = tensor_from_json(text);
    *rank = static_cast<int>(t.shape.size());
    for (std::size_t i = 0; i < t.shape.size(); ++i) shape[i] = t.shape[i];
    *count = static_cast<int64_t>(t.data.size());
    if (*count > cap) throw std::runtime_error("data buffer too small");
    std::memcpy(data, t.data.data(), sizeof(double) * t.data.size());
  });
}

int ref_tensor_to_binary(const int64_t* shape, int rank, const double* data, unsigned char* out, int64_t cap,
                         int64_t* len) {
  return guard([&] {
    DenseTensor t(std::vector<int64_t>(shape, shape + rank));
    std::memcpy(t.data.data(), data, sizeof(double) * t.data.size());
    std::ostringstream os;
    tensor_write_binary(t, os);
    const std::string s = os.str();
    *len = static_cast<int64_t>(s.size());
    if (*len > cap) throw std::runtime_error("buffer too small");
    std::memcpy(out, s.data(), s.size());
  });
}

int ref_layer_json_roundtrip(const char* layer_json, char* out, int cap) {
  return guard([&] { put(layer_to_json(layer_from_json(layer_json)), out, cap); });
}

// merge_like_modes / unmerge_modes (kernels.cpp:246-286): "merged_subs\nrecord" out (record as
// "compound=member:dim,...;..."), permuted data in `out`; unmerged subscripts + dims back.
int ref_merge_like_modes(const char* expr1, const int64_t* dims, const double* data, double* out, char* info,
                         int cap) {
  return guard([&] {
    // expr1: a one-input expression "subs->output|convs" whose classify() gives the classes
    ExpressionSpec spec = parse(expr1);
    const Subscripts& subs = spec.inputs.at(0);
    DenseTensor t(std::vector<int64_t>(dims, dims + subs.size()));
    std::memcpy(t.data.data(), data, sizeof(double) * t.data.size());
    auto [m, msubs, rec] = merge_like_modes(t, subs, classify(spec));
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
    std::string r;
    for (const auto& g : rec.groups) {
      r += (r.empty() ? "" : ";") + g.compound.name + "=";
      for (std::size_t k = 0; k < g.members.size(); ++k)
        r += (k ? "," : "") + g.members[k].name + ":" + std::to_string(g.member_dims[k]);
    }
    auto [u, usubs] = unmerge_modes(m, msubs, rec);
    std::string ud;
    for (std::size_t i = 0; i < u.shape.size(); ++i) ud += (i ? "," : "") + std::to_string(u.shape[i]);
    std::string md;
    for (std::size_t i = 0; i < m.shape.size(); ++i) md += (i ? "," : "") + std::to_string(m.shape[i]);
    put(render(msubs) + "\n" + md + "\n" + r + "\n" + render(usubs) + "\n" + ud, info, cap);
  });
}

}  // extern "C"
