// Planner implementation.  Parity anchors in /root/reference/proj/src/sequencer.cpp:
//   atom table + keep rule + subset subscripts   31-136
//   tree assembly                                140-177
//   exact subset DP with (cost, peak, encoding)   216-272
//   cost-capped variant                           276-310
//   enumeration / explicit joins / cost          316-401
//   encoding + JSON                              449-480
#include "ce_plan.hpp"

#include <algorithm>
#include <bit>
#include <limits>

namespace ce {

namespace {

// Per-atom facts the planner needs, in canonical first-appearance order.
struct AtomRow {
  Atom atom;
  uint32_t carriers = 0;                        // bit i: input i carries the atom
  bool kept_by_output = false;
  int64_t closed_dim = 1;                       // dim once all carriers are joined
  std::vector<std::pair<int, int64_t>> occ;     // (input, dim) per carrier
};

struct SubsetInfo {
  bool ready = false;
  Subscripts subs;
  std::vector<int64_t> dims;
};

class SubsetTable {
 public:
  SubsetTable(const ExpressionSpec& s, const ShapeEnv& e, const ConvModeMap& m, CostMode cm)
      : spec_(s), env_(e), modes_(m), cost_mode_(cm), n_(static_cast<int>(s.inputs.size())) {
    if (n_ < 1) throw PlanError("expression has no inputs");
    if (n_ > 30) throw PlanError("too many inputs");
    for (const Atom& a : spec_.all_atoms()) {
      AtomRow row;
      row.atom = a;
      row.kept_by_output = spec_.in_output(a);
      for (int i = 0; i < n_; ++i) {
        const int ax = find_atom(spec_.inputs[static_cast<std::size_t>(i)], a);
        if (ax < 0) continue;
        row.carriers |= 1u << i;
        row.occ.emplace_back(i, env_.dims[static_cast<std::size_t>(i)][static_cast<std::size_t>(ax)]);
      }
      if (spec_.is_conv(a)) {
        auto it = modes_.find(a);
        if (it == modes_.end()) throw PlanError("no conv mode assigned to atom '" + a.name + "'");
        const bool multiway = row.occ.size() >= 3;
        if (multiway && it->second != ConvMode::Circular)
          throw PlanError("multi-way conv atom '" + a.name + "' requires circular mode");
        int64_t hi = 0, lo = std::numeric_limits<int64_t>::max();
        for (const auto& o : row.occ) {
          hi = std::max(hi, o.second);
          lo = std::min(lo, o.second);
        }
        if (multiway && it->second.stride != 1) throw PlanError("multi-way conv atom '" + a.name + "' cannot be strided");
        row.closed_dim = multiway ? hi : conv_output_dim(it->second.mode, hi, lo, it->second.stride);
      } else {
        row.closed_dim = row.occ.front().second;
      }
      rows_.push_back(std::move(row));
    }
    table_.resize(std::size_t{1} << n_);
  }

  int n() const { return n_; }
  uint32_t all() const { return n_ == 32 ? ~0u : (1u << n_) - 1u; }
  const ExpressionSpec& spec() const { return spec_; }
  const ShapeEnv& env() const { return env_; }
  const ConvModeMap& modes() const { return modes_; }
  CostMode cost_mode() const { return cost_mode_; }

  // Subscripts of the intermediate covering `mask` (sequencer.cpp:92-109):
  // singletons are the raw input; otherwise an atom survives iff it is in the
  // output or some carrier lies outside the subset.
  const SubsetInfo& info(uint32_t mask) {
    SubsetInfo& e = table_[mask];
    if (e.ready) return e;
    e.ready = true;
    if (std::popcount(mask) == 1) {
      const auto i = static_cast<std::size_t>(std::countr_zero(mask));
      e.subs = spec_.inputs[i];
      e.dims = env_.dims[i];
      return e;
    }
    for (const auto& r : rows_) {
      if (!(r.carriers & mask)) continue;
      const bool closed = (r.carriers & ~mask) == 0;
      if (closed && !r.kept_by_output) continue;
      e.subs.push_back(r.atom);
      e.dims.push_back(closed ? r.closed_dim : first_dim_inside(r, mask));
    }
    return e;
  }

  std::set<Atom> keep(uint32_t mask) const {
    std::set<Atom> k;
    for (const auto& r : rows_)
      if (r.kept_by_output || (r.carriers & ~mask)) k.insert(r.atom);
    return k;
  }

  PairwiseOp join(uint32_t l, uint32_t r) {
    const SubsetInfo& a = info(l);
    const SubsetInfo& b = info(r);
    const SubsetInfo& res = info(l | r);
    return make_pairwise_op(a.subs, a.dims, b.subs, b.dims, keep(l | r), modes_, res.subs);
  }

  u128 cost(const PairwiseOp& op) const { return pairwise_cost(op, cost_mode_).total; }

 private:
  static int64_t first_dim_inside(const AtomRow& r, uint32_t mask) {
    for (const auto& o : r.occ)
      if (mask & (1u << o.first)) return o.second;
    return -1;
  }

  const ExpressionSpec& spec_;
  const ShapeEnv& env_;
  const ConvModeMap& modes_;
  CostMode cost_mode_;
  int n_;
  std::vector<AtomRow> rows_;
  std::vector<SubsetInfo> table_;
};

using Split = std::pair<uint32_t, uint32_t>;

EvaluationPlan build_plan(SubsetTable& t, const std::vector<Split>& order) {
  EvaluationPlan plan;
  plan.spec = t.spec();
  plan.env = t.env();
  plan.modes = t.modes();
  plan.cost_mode = t.cost_mode();
  std::vector<int> id(std::size_t{1} << t.n(), -1);
  for (int i = 0; i < t.n(); ++i) id[std::size_t{1} << i] = i;
  uint64_t peak = 0;
  for (const auto& [l, r] : order) {
    PlanNode node;
    node.left = id[l];
    node.right = id[r];
    node.op = t.join(l, r);
    node.cost = t.cost(node.op);
    plan.total_cost = add_checked(plan.total_cost, node.cost);
    peak = std::max(peak, static_cast<uint64_t>(node.op.result_elements()));
    id[l | r] = t.n() + static_cast<int>(plan.nodes.size());
    plan.nodes.push_back(std::move(node));
  }
  plan.peak_intermediate_elements = peak;
  if (t.n() == 1) {
    const auto& in0 = t.spec().inputs[0];
    for (std::size_t j = 0; j < in0.size(); ++j)
      if (t.spec().in_output(in0[j])) {
        plan.root_subs.push_back(in0[j]);
        plan.root_dims.push_back(t.env().dims[0][j]);
      }
  } else {
    const auto& root = t.info(t.all());
    plan.root_subs = root.subs;
    plan.root_dims = root.dims;
  }
  return plan;
}

void postorder(uint32_t mask, const std::vector<Split>& split, std::vector<Split>& out) {
  if (std::popcount(mask) == 1) return;
  const Split s = split[mask];
  postorder(s.first, split, out);
  postorder(s.second, split, out);
  out.push_back(s);
}

struct Best {
  bool valid = false;
  u128 cost = 0;
  uint64_t peak = 0;
  std::string enc;
  Split split{0, 0};
};

// Exact DP over subsets; a finite cap drops partial plans above it and reports
// the cheapest dropped total through *over.
std::vector<Best> subset_dp(SubsetTable& t, bool capped, u128 cap, u128* over) {
  std::vector<Best> best(std::size_t{1} << t.n());
  for (int i = 0; i < t.n(); ++i) {
    best[std::size_t{1} << i].valid = true;
    best[std::size_t{1} << i].enc = std::to_string(i);
  }
  bool dropped = false;
  u128 cheapest_dropped = 0;
  std::vector<uint32_t> masks;
  for (uint32_t m = 1; m <= t.all(); ++m)
    if (std::popcount(m) >= 2) masks.push_back(m);
  std::stable_sort(masks.begin(), masks.end(),
                   [](uint32_t a, uint32_t b) { return std::popcount(a) < std::popcount(b); });

  for (uint32_t mask : masks) {
    Best& cell = best[mask];
    const uint32_t lowest = mask & (~mask + 1u);
    for (uint32_t sub = (mask - 1) & mask; sub; sub = (sub - 1) & mask) {
      if (!(sub & lowest)) continue;  // left child always holds the lowest input
      const uint32_t rest = mask & ~sub;
      const Best& a = best[sub];
      const Best& b = best[rest];
      if (!a.valid || !b.valid) continue;
      const PairwiseOp op = t.join(sub, rest);
      const u128 total = add_checked(add_checked(a.cost, b.cost), t.cost(op));
      if (capped && total > cap) {
        if (!dropped || total < cheapest_dropped) cheapest_dropped = total;
        dropped = true;
        continue;
      }
      const uint64_t peak =
          std::max({a.peak, b.peak, static_cast<uint64_t>(op.result_elements())});
      if (cell.valid && (total > cell.cost || (total == cell.cost && peak > cell.peak))) continue;
      std::string enc = "(" + a.enc + " " + b.enc + ")";
      if (cell.valid && total == cell.cost && peak == cell.peak && enc >= cell.enc) continue;
      cell = Best{true, total, peak, std::move(enc), {sub, rest}};
    }
  }
  *over = dropped ? cheapest_dropped : 0;
  return best;
}

void enumerate_rec(std::vector<Split>& split, SubsetTable& t, std::vector<EvaluationPlan>& out) {
  // first unsplit internal subset, depth first from the root
  uint32_t pending = 0;
  std::vector<uint32_t> stack{t.all()};
  while (!stack.empty() && !pending) {
    const uint32_t m = stack.back();
    stack.pop_back();
    if (std::popcount(m) == 1) continue;
    if (split[m].first == 0) {
      pending = m;
    } else {
      stack.push_back(split[m].first);
      stack.push_back(split[m].second);
    }
  }
  if (!pending) {
    std::vector<Split> order;
    postorder(t.all(), split, order);
    out.push_back(build_plan(t, order));
    return;
  }
  const uint32_t lowest = pending & (~pending + 1u);
  for (uint32_t sub = (pending - 1) & pending; sub; sub = (sub - 1) & pending) {
    if (!(sub & lowest)) continue;
    split[pending] = {sub, pending & ~sub};
    enumerate_rec(split, t, out);
    split[pending] = {0, 0};
  }
}

}  // namespace

EvaluationPlan left_to_right(const ExpressionSpec& spec, const ShapeEnv& env,
                             const ConvModeMap& modes, CostMode cost_mode) {
  SubsetTable t(spec, env, modes, cost_mode);
  std::vector<Split> order;
  uint32_t acc = 1;
  for (int i = 1; i < t.n(); ++i) {
    order.push_back({acc, 1u << i});
    acc |= 1u << i;
  }
  return build_plan(t, order);
}

EvaluationPlan optimal(const ExpressionSpec& spec, const ShapeEnv& env, const ConvModeMap& modes,
                       CostMode cost_mode, OptimalOptions options) {
  SubsetTable t(spec, env, modes, cost_mode);
  if (t.n() > options.max_inputs)
    throw PlanError("expression has " + std::to_string(t.n()) + " inputs, over the cap of " +
                    std::to_string(options.max_inputs));
  if (t.n() == 1) return build_plan(t, {});
  std::vector<Best> best;
  u128 over = 0;
  if (!options.cost_capped) {
    best = subset_dp(t, false, 0, &over);
  } else {
    for (u128 cap = 1;;) {
      best = subset_dp(t, true, cap, &over);
      if (best[t.all()].valid) break;
      cap = std::max(mul_checked(cap, 2), over);
    }
  }
  std::vector<Split> split(std::size_t{1} << t.n());
  for (uint32_t m = 1; m <= t.all(); ++m)
    if (best[m].valid && std::popcount(m) >= 2) split[m] = best[m].split;
  std::vector<Split> order;
  postorder(t.all(), split, order);
  return build_plan(t, order);
}

std::vector<EvaluationPlan> enumerate_all(const ExpressionSpec& spec, const ShapeEnv& env,
                                          const ConvModeMap& modes, CostMode cost_mode) {
  SubsetTable t(spec, env, modes, cost_mode);
  if (t.n() > 6) throw PlanError("enumerate_all supports at most 6 inputs");
  std::vector<EvaluationPlan> out;
  if (t.n() == 1) {
    out.push_back(build_plan(t, {}));
    return out;
  }
  std::vector<Split> split(std::size_t{1} << t.n(), {0, 0});
  enumerate_rec(split, t, out);
  return out;
}

EvaluationPlan plan_from_joins(const ExpressionSpec& spec, const ShapeEnv& env,
                               const ConvModeMap& modes, CostMode cost_mode,
                               const std::vector<std::pair<int, int>>& joins) {
  SubsetTable t(spec, env, modes, cost_mode);
  if (static_cast<int>(joins.size()) != t.n() - 1)
    throw PlanError("plan_from_joins: expected " + std::to_string(t.n() - 1) + " joins");
  std::vector<uint32_t> mask;
  std::vector<char> used;
  for (int i = 0; i < t.n(); ++i) {
    mask.push_back(1u << i);
    used.push_back(0);
  }
  std::vector<Split> order;
  for (const auto& [l, r] : joins) {
    const int count = static_cast<int>(mask.size());
    if (l < 0 || r < 0 || l >= count || r >= count || l == r)
      throw PlanError("plan_from_joins: operand id out of range");
    if (used[static_cast<std::size_t>(l)] || used[static_cast<std::size_t>(r)])
      throw PlanError("plan_from_joins: operand used twice");
    used[static_cast<std::size_t>(l)] = used[static_cast<std::size_t>(r)] = 1;
    const uint32_t lm = mask[static_cast<std::size_t>(l)], rm = mask[static_cast<std::size_t>(r)];
    order.push_back({lm, rm});
    mask.push_back(lm | rm);
    used.push_back(0);
  }
  if (mask.back() != t.all()) throw PlanError("plan_from_joins: joins do not cover all inputs");
  return build_plan(t, order);
}

EvaluationPlan plan_from_nodes(const ExpressionSpec& spec, const ShapeEnv& env, const ConvModeMap& modes,
                               CostMode cost_mode, const std::vector<std::pair<int, int>>& joins,
                               const std::vector<Subscripts>& results) {
  const int n = static_cast<int>(spec.inputs.size());
  if (joins.size() != results.size()) throw PlanError("plan_from_nodes: one result per join expected");
  if (n > 1 && static_cast<int>(joins.size()) != n - 1)
    throw PlanError("plan_from_nodes: expected " + std::to_string(n - 1) + " nodes");
  for (const auto& a : spec.conv_atoms)
    if (!modes.count(a)) throw ShapeError("plan_from_nodes: no convolution mode for atom '" + a.name + "'");
  EvaluationPlan plan;
  plan.spec = spec;
  plan.env = env;
  plan.modes = modes;
  plan.cost_mode = cost_mode;
  std::vector<Subscripts> subs(spec.inputs.begin(), spec.inputs.end());
  std::vector<std::vector<int64_t>> dims(env.dims.begin(), env.dims.end());
  std::vector<char> used(static_cast<std::size_t>(n), 0);
  uint64_t peak = 0;
  for (std::size_t j = 0; j < joins.size(); ++j) {
    const auto [l, r] = joins[j];
    const int count = static_cast<int>(subs.size());
    if (l < 0 || r < 0 || l >= count || r >= count || l == r)
      throw PlanError("plan_from_nodes: operand id out of range");
    if (used[static_cast<std::size_t>(l)] || used[static_cast<std::size_t>(r)])
      throw PlanError("plan_from_nodes: operand used twice");
    used[static_cast<std::size_t>(l)] = used[static_cast<std::size_t>(r)] = 1;
    // an atom the rest of the plan still needs (output, or an operand not joined yet) must survive
    for (const Subscripts* side : {&subs[static_cast<std::size_t>(l)], &subs[static_cast<std::size_t>(r)]})
      for (const Atom& a : *side) {
        bool needed = spec.in_output(a);
        for (int k = 0; k < count && !needed; ++k)
          if (k != l && k != r && !used[static_cast<std::size_t>(k)] && find_atom(subs[static_cast<std::size_t>(k)], a) >= 0)
            needed = true;
        if (needed && find_atom(results[j], a) < 0)
          throw PlanError("plan_from_nodes: node " + std::to_string(j) + " drops atom '" + a.name +
                          "' that a later node or the output needs");
      }
    const std::set<Atom> keep(results[j].begin(), results[j].end());
    PlanNode node;
    node.left = l;
    node.right = r;
    node.op = make_pairwise_op(subs[static_cast<std::size_t>(l)], dims[static_cast<std::size_t>(l)],
                               subs[static_cast<std::size_t>(r)], dims[static_cast<std::size_t>(r)], keep, modes,
                               results[j]);
    node.cost = pairwise_cost(node.op, cost_mode).total;
    plan.total_cost = add_checked(plan.total_cost, node.cost);
    peak = std::max(peak, static_cast<uint64_t>(node.op.result_elements()));
    subs.push_back(node.op.result);
    dims.push_back(node.op.result_dims);
    used.push_back(0);
    plan.nodes.push_back(std::move(node));
  }
  plan.peak_intermediate_elements = peak;
  if (plan.nodes.empty()) {
    const auto& in0 = spec.inputs[0];
    for (std::size_t j = 0; j < in0.size(); ++j)
      if (spec.in_output(in0[j])) {
        plan.root_subs.push_back(in0[j]);
        plan.root_dims.push_back(env.dims[0][j]);
      }
  } else {
    plan.root_subs = plan.nodes.back().op.result;
    plan.root_dims = plan.nodes.back().op.result_dims;
    for (const Atom& a : spec.output)
      if (find_atom(plan.root_subs, a) < 0)
        throw ShapeError("execute: root is missing output atom '" + a.name + "'");
  }
  return plan;
}

u128 plan_cost(const EvaluationPlan& plan, CostMode mode) {
  u128 total = 0;
  for (const auto& n : plan.nodes) total = add_checked(total, pairwise_cost(n.op, mode).total);
  return total;
}

std::string tree_encoding(const EvaluationPlan& plan) {
  std::vector<std::string> enc;
  for (std::size_t i = 0; i < plan.spec.inputs.size(); ++i) enc.push_back(std::to_string(i));
  for (const auto& n : plan.nodes)
    enc.push_back("(" + enc[static_cast<std::size_t>(n.left)] + " " +
                  enc[static_cast<std::size_t>(n.right)] + ")");
  return enc.back();
}

namespace {
// nlohmann::json prints integers that fit u64 as numbers and we mirror the
// reference's decimal-string fallback for larger costs (sequencer.cpp:460-463).
std::string json_cost(u128 v) {
  if (v <= std::numeric_limits<uint64_t>::max()) return u128_to_string(v);
  return "\"" + u128_to_string(v) + "\"";
}
}  // namespace

std::string plan_to_json(const EvaluationPlan& plan) {
  // Keys in lexicographic order, as nlohmann's std::map-backed objects dump them.
  std::string s = "{\"nodes\":[";
  for (std::size_t i = 0; i < plan.nodes.size(); ++i) {
    const auto& n = plan.nodes[i];
    s += (i ? ",{" : "{");
    s += "\"cost\":" + json_cost(n.cost) + ",\"left\":" + std::to_string(n.left) +
         ",\"result\":\"" + render(n.op.result) + "\",\"right\":" + std::to_string(n.right) + "}";
  }
  s += "],\"peak_elems\":" + std::to_string(plan.peak_intermediate_elements) +
       ",\"total_cost\":" + json_cost(plan.total_cost) + "}";
  return s;
}

}  // namespace ce
