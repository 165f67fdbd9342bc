// Host IR for conv_einsum.  Behavioural parity targets (all in /root/reference/proj):
//   checked arithmetic   include/convexpr/checked_int.hpp:17-41
//   parse/render/classify src/expression.cpp:56-246
//   ShapeEnv / SplitMix64 src/tensor.cpp:107-231
//   conv modes / roles    src/kernels.cpp:18-142
//   flops_actual          src/kernels.cpp:472-505
//   pairwise_cost         src/cost.cpp:15-43
#include "ce_ir.hpp"

#include <algorithm>
#include <cstdlib>
#include <cctype>

namespace ce {

// ----------------------------------------------------------------------------- u128
u128 mul_checked(u128 a, u128 b) {
  if (a == 0 || b == 0) return 0;
  const u128 r = a * b;
  if (r / a != b) throw OverflowError("cost multiplication overflow");
  return r;
}

u128 add_checked(u128 a, u128 b) {
  const u128 r = a + b;
  if (r < a) throw OverflowError("cost addition overflow");
  return r;
}

std::string u128_to_string(u128 v) {
  if (v == 0) return "0";
  char buf[48];
  int n = 0;
  for (; v; v /= 10) buf[n++] = static_cast<char>('0' + static_cast<int>(v % 10));
  std::string s;
  while (n) s.push_back(buf[--n]);
  return s;
}

ParseError::ParseError(const std::string& msg, std::size_t pos)
    : std::runtime_error(msg + " (at position " + std::to_string(pos) + ")"), position(pos) {}

// ----------------------------------------------------------------------------- spec
const char* to_string(AtomClass c) {
  static const char* names[] = {"convolution", "batch", "contraction", "free", "self-contraction"};
  return names[static_cast<int>(c)];
}

int find_atom(const Subscripts& subs, const Atom& a) {
  for (std::size_t i = 0; i < subs.size(); ++i)
    if (subs[i] == a) return static_cast<int>(i);
  return -1;
}

bool ExpressionSpec::is_conv(const Atom& a) const { return find_atom(conv_atoms, a) >= 0; }
bool ExpressionSpec::in_output(const Atom& a) const { return find_atom(output, a) >= 0; }

int ExpressionSpec::occurrence_count(const Atom& a) const {
  int n = 0;
  for (const auto& s : inputs) n += find_atom(s, a) >= 0 ? 1 : 0;
  return n;
}

Subscripts ExpressionSpec::all_atoms() const {
  Subscripts seen;
  for (const auto& s : inputs)
    for (const auto& a : s)
      if (find_atom(seen, a) < 0) seen.push_back(a);
  return seen;
}

namespace {

// Token stream over the source with original byte offsets for diagnostics.
struct Lexer {
  enum Kind { kAtom, kComma, kArrow, kPipe, kEnd };
  struct Tok {
    Kind kind;
    std::string name;
    std::size_t pos;
  };
  std::vector<Tok> toks;

  explicit Lexer(std::string_view s) {
    std::size_t i = 0;
    auto space = [&](char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; };
    while (i < s.size()) {
      const char c = s[i];
      if (space(c)) {
        ++i;
      } else if (c == ',') {
        toks.push_back({kComma, {}, i++});
      } else if (c == '|') {
        toks.push_back({kPipe, {}, i++});
      } else if (c == '-') {
        if (i + 1 >= s.size() || s[i + 1] != '>') throw ParseError("expected '->' after '-'", i);
        toks.push_back({kArrow, {}, i});
        i += 2;
      } else if (c == '(') {
        const std::size_t open = i++;
        std::string name;
        for (; i < s.size() && s[i] != ')'; ++i) {
          if (space(s[i])) continue;
          if (!std::isalnum(static_cast<unsigned char>(s[i])))
            throw ParseError("invalid character in parenthesized atom name", i);
          name.push_back(s[i]);
        }
        if (i >= s.size()) throw ParseError("unbalanced '('", open);
        ++i;
        if (name.empty()) throw ParseError("empty parenthesized atom name", open);
        toks.push_back({kAtom, std::move(name), open});
      } else if (c == ')') {
        throw ParseError("unbalanced ')'", i);
      } else if (std::isalpha(static_cast<unsigned char>(c))) {
        toks.push_back({kAtom, std::string(1, c), i++});
      } else {
        throw ParseError(std::string("unexpected character '") + c + "'", i);
      }
    }
    toks.push_back({kEnd, {}, s.size()});
  }
};

void reject_repeats(const Subscripts& subs, const char* where, std::size_t pos) {
  std::set<std::string> seen;
  for (const auto& a : subs)
    if (!seen.insert(a.name).second)
      throw ParseError("atom '" + a.name + "' repeated within " + where, pos);
}

}  // namespace

ExpressionSpec parse(std::string_view source) {
  Lexer lx(source);
  const auto& t = lx.toks;
  std::size_t i = 0;
  ExpressionSpec spec;

  // inputs: subs ("," subs)* "->"
  spec.inputs.emplace_back();
  std::size_t arrow_pos = 0;
  for (;; ++i) {
    if (t[i].kind == Lexer::kAtom) {
      spec.inputs.back().push_back(Atom{t[i].name});
    } else if (t[i].kind == Lexer::kComma) {
      if (spec.inputs.back().empty()) throw ParseError("empty input subscript list", t[i].pos);
      spec.inputs.emplace_back();
    } else if (t[i].kind == Lexer::kArrow) {
      arrow_pos = t[i].pos;
      ++i;
      break;
    } else {
      throw ParseError("expected atom, ',' or '->' in inputs", t[i].pos);
    }
  }
  if (spec.inputs.back().empty()) throw ParseError("empty input subscript list", arrow_pos);

  for (; t[i].kind == Lexer::kAtom; ++i) spec.output.push_back(Atom{t[i].name});

  Subscripts listed;
  if (t[i].kind == Lexer::kPipe) {
    ++i;
    bool need_atom = true;
    for (; t[i].kind != Lexer::kEnd; ++i) {
      if (t[i].kind == Lexer::kAtom) {
        listed.push_back(Atom{t[i].name});
        need_atom = false;
      } else if (t[i].kind == Lexer::kComma) {
        if (need_atom) throw ParseError("expected conv atom before ','", t[i].pos);
        need_atom = true;
      } else {
        throw ParseError("unexpected token in conv list", t[i].pos);
      }
    }
    if (listed.empty()) throw ParseError("'|' with no conv atoms", t[i].pos);
  }
  if (t[i].kind != Lexer::kEnd)
    throw ParseError(t[i].kind == Lexer::kArrow ? "duplicate '->'" : "unexpected trailing token",
                     t[i].pos);

  const std::size_t end = source.size();
  for (const auto& s : spec.inputs) reject_repeats(s, "one input subscript list", end);
  reject_repeats(spec.output, "the output subscript list", end);
  reject_repeats(listed, "the conv list", end);
  for (const auto& a : spec.output)
    if (spec.occurrence_count(a) == 0)
      throw ParseError("output atom '" + a.name + "' absent from all inputs", end);
  for (const auto& a : listed) {
    if (!spec.in_output(a)) throw ParseError("conv atom '" + a.name + "' absent from output", end);
    if (spec.occurrence_count(a) < 2)
      throw ParseError("conv atom '" + a.name + "' present in fewer than two inputs", end);
  }
  for (const auto& a : spec.output)
    if (find_atom(listed, a) >= 0) spec.conv_atoms.push_back(a);
  return spec;
}

std::string render(const Subscripts& subs) {
  std::string s;
  for (const auto& a : subs) s += a.name.size() == 1 ? a.name : "(" + a.name + ")";
  return s;
}

std::string render(const ExpressionSpec& spec) {
  std::string s;
  for (std::size_t i = 0; i < spec.inputs.size(); ++i) s += (i ? "," : "") + render(spec.inputs[i]);
  s += "->" + render(spec.output);
  if (!spec.conv_atoms.empty()) s += "|" + render(spec.conv_atoms);
  return s;
}

std::map<Atom, AtomClass> classify(const ExpressionSpec& spec) {
  std::map<Atom, AtomClass> out;
  for (const auto& a : spec.all_atoms()) {
    AtomClass c;
    if (spec.is_conv(a)) {
      c = AtomClass::Convolution;
    } else {
      const bool shared = spec.occurrence_count(a) >= 2, kept = spec.in_output(a);
      c = shared ? (kept ? AtomClass::BatchProduct : AtomClass::Contraction)
                 : (kept ? AtomClass::Free : AtomClass::SelfContraction);
    }
    out.emplace(a, c);
  }
  return out;
}

// ----------------------------------------------------------------------------- shapes
int64_t element_count(const std::vector<int64_t>& shape) {
  int64_t n = 1;
  for (int64_t d : shape) n *= d;
  return n;
}

std::vector<int64_t> row_major_strides(const std::vector<int64_t>& shape) {
  std::vector<int64_t> st(shape.size());
  int64_t acc = 1;
  for (std::size_t i = shape.size(); i-- > 0;) {
    st[i] = acc;
    acc *= shape[i];
  }
  return st;
}

int64_t ShapeEnv::dim_of(const ExpressionSpec& spec, const Atom& a) const {
  for (std::size_t i = 0; i < spec.inputs.size(); ++i) {
    const int ax = find_atom(spec.inputs[i], a);
    if (ax >= 0) return dims[i][static_cast<std::size_t>(ax)];
  }
  throw ShapeError("atom '" + a.name + "' not present in any input");
}

ShapeEnv make_shape_env(const ExpressionSpec& spec, std::vector<std::vector<int64_t>> dims) {
  if (dims.size() != spec.inputs.size())
    throw ShapeError("shape env: expected " + std::to_string(spec.inputs.size()) +
                     " dim lists, got " + std::to_string(dims.size()));
  for (std::size_t i = 0; i < dims.size(); ++i) {
    if (dims[i].size() != spec.inputs[i].size())
      throw ShapeError("shape env: input " + std::to_string(i) + " expects " +
                       std::to_string(spec.inputs[i].size()) + " dims, got " +
                       std::to_string(dims[i].size()));
    for (int64_t d : dims[i])
      if (d < 1) throw ShapeError("shape env: dimensions must be positive");
  }
  for (const auto& a : spec.all_atoms()) {
    std::vector<int64_t> occ;
    for (std::size_t i = 0; i < spec.inputs.size(); ++i) {
      const int ax = find_atom(spec.inputs[i], a);
      if (ax >= 0) occ.push_back(dims[i][static_cast<std::size_t>(ax)]);
    }
    const bool uniform = std::all_of(occ.begin(), occ.end(), [&](int64_t d) { return d == occ[0]; });
    if (uniform) continue;
    if (!spec.is_conv(a))
      throw ShapeError("atom '" + a.name + "' carries unequal dimensions across inputs");
    if (occ.size() >= 3)
      throw ShapeError("multi-way conv atom '" + a.name + "' requires equal dimensions");
  }
  return ShapeEnv{std::move(dims)};
}

uint64_t SplitMix64::next() {
  state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double SplitMix64::next_unit() { return 2.0 * (static_cast<double>(next() >> 11) * 0x1.0p-53) - 1.0; }

int64_t SplitMix64::next_in(int64_t lo, int64_t hi) {
  return lo + static_cast<int64_t>(next() % static_cast<uint64_t>(hi - lo + 1));
}

// ----------------------------------------------------------------------------- modes
const char* to_string(ConvMode m) {
  static const char* names[] = {"full", "same", "valid", "circular"};
  return names[static_cast<int>(m)];
}

ConvMode conv_mode_from_string(std::string_view s) {
  for (ConvMode m : {ConvMode::Full, ConvMode::Same, ConvMode::Valid, ConvMode::Circular})
    if (s == to_string(m)) return m;
  throw std::invalid_argument("unknown conv mode: " + std::string(s));
}

ConvModeSpec conv_mode_spec_from_string(std::string_view s) {
  const std::size_t slash = s.find('/');
  if (slash == std::string_view::npos) return ConvModeSpec(conv_mode_from_string(s));
  const std::string st(s.substr(slash + 1));
  char* end = nullptr;
  const long long v = std::strtoll(st.c_str(), &end, 10);
  if (st.empty() || *end != '\0' || v < 1) throw std::invalid_argument("bad conv stride in '" + std::string(s) + "'");
  return ConvModeSpec(conv_mode_from_string(s.substr(0, slash)), v);
}

int64_t conv_output_dim(ConvMode mode, int64_t feature, int64_t filter, int64_t stride) {
  const int64_t s = stride;
  switch (mode) {
    case ConvMode::Full: return (feature + filter - 2) / s + 1;
    case ConvMode::Valid:
      if (feature < filter) throw ShapeError("valid convolution requires feature >= filter");
      return (feature - filter) / s + 1;
    case ConvMode::Same:
    case ConvMode::Circular: return (feature + s - 1) / s;
  }
  return 0;
}

ConvModeMap resolve_conv_modes(const ExpressionSpec& spec, ConvModeSpec requested) {
  ConvModeMap m;
  for (const auto& a : spec.conv_atoms)
    m[a] = spec.occurrence_count(a) >= 3 ? ConvModeSpec(ConvMode::Circular) : requested;
  return m;
}

// ----------------------------------------------------------------------------- roles
PairwiseOp make_pairwise_op(const Subscripts& left, const std::vector<int64_t>& left_dims,
                            const Subscripts& right, const std::vector<int64_t>& right_dims,
                            const std::set<Atom>& keep, const ConvModeMap& conv_modes,
                            const std::optional<Subscripts>& result_order) {
  if (left.size() != left_dims.size() || right.size() != right_dims.size())
    throw ShapeError("pairwise op: subscript/dimension length mismatch");
  PairwiseOp op;
  op.left = left;
  op.right = right;
  op.left_dims = left_dims;
  op.right_dims = right_dims;
  std::map<Atom, int64_t> kept_dim;

  // Shared atoms in left order, then right-only atoms in right order
  // (kernels.cpp:124-128 fixes this canonical order).
  auto shared = [&](const Atom& a, int64_t dl, int64_t dr) {
    auto mode = conv_modes.find(a);
    if (mode != conv_modes.end()) {
      ConvAxis ax;
      ax.atom = a;
      ax.mode = mode->second.mode;
      ax.stride = mode->second.stride;
      ax.feature_on_left = dl >= dr;
      ax.feature_dim = std::max(dl, dr);
      ax.filter_dim = std::min(dl, dr);
      ax.output_dim = conv_output_dim(ax.mode, ax.feature_dim, ax.filter_dim, ax.stride);
      kept_dim[a] = ax.output_dim;
      op.conv_axes.push_back(ax);
      return;
    }
    if (dl != dr)
      throw ShapeError("atom '" + a.name + "' has mismatched dimensions " + std::to_string(dl) +
                       " vs " + std::to_string(dr));
    if (keep.count(a)) {
      op.batch_atoms.push_back(a);
      op.batch_dims.push_back(dl);
      kept_dim[a] = dl;
    } else {
      op.contraction_atoms.push_back(a);
      op.contraction_dims.push_back(dl);
    }
  };
  auto single = [&](const Atom& a, int64_t d, Subscripts& free, std::vector<int64_t>& free_dims,
                    Subscripts& self) {
    if (keep.count(a)) {
      free.push_back(a);
      free_dims.push_back(d);
      kept_dim[a] = d;
    } else {
      self.push_back(a);
    }
  };
  for (std::size_t i = 0; i < left.size(); ++i) {
    const int j = find_atom(right, left[i]);
    if (j >= 0)
      shared(left[i], left_dims[i], right_dims[static_cast<std::size_t>(j)]);
    else
      single(left[i], left_dims[i], op.left_free, op.left_free_dims, op.left_self);
  }
  for (std::size_t j = 0; j < right.size(); ++j)
    if (find_atom(left, right[j]) < 0)
      single(right[j], right_dims[j], op.right_free, op.right_free_dims, op.right_self);

  if (result_order) {
    op.result = *result_order;
    if (op.result.size() != kept_dim.size())
      throw ShapeError("pairwise op: result order does not match kept atoms");
  } else {
    for (const auto& a : left)
      if (kept_dim.count(a)) op.result.push_back(a);
    for (const auto& a : right)
      if (kept_dim.count(a) && find_atom(left, a) < 0) op.result.push_back(a);
  }
  for (const auto& a : op.result) {
    auto it = kept_dim.find(a);
    if (it == kept_dim.end())
      throw ShapeError("pairwise op: result atom '" + a.name + "' is not kept by this node");
    op.result_dims.push_back(it->second);
  }
  return op;
}

namespace {
u128 non_conv_product(const PairwiseOp& op) {
  u128 f = 1;
  for (const auto* v : {&op.batch_dims, &op.contraction_dims, &op.left_free_dims, &op.right_free_dims})
    for (int64_t d : *v) f = mul_checked(f, static_cast<u128>(d));
  return f;
}

// Number of (n, k) pairs the direct loop visits on one conv axis.
int64_t conv_pairs(const ConvAxis& ax) {
  if (ax.stride > 1) {  // (extension) count the in-range feature indices directly
    if (ax.mode == ConvMode::Circular) return ax.output_dim * ax.filter_dim;
    const int64_t s = ax.stride, c = ax.mode == ConvMode::Same ? same_offset(ax.filter_dim) : 0;
    const int64_t sq = ax.mode == ConvMode::Valid ? 1 : -1;
    int64_t count = 0;
    for (int64_t n = 0; n < ax.output_dim; ++n)
      for (int64_t k = 0; k < ax.filter_dim; ++k) {
        const int64_t x = s * n + c + sq * k;
        count += x >= 0 && x < ax.feature_dim;
      }
    return count;
  }
  switch (ax.mode) {
    case ConvMode::Full:
    case ConvMode::Circular: return ax.feature_dim * ax.filter_dim;
    case ConvMode::Valid: return (ax.feature_dim - ax.filter_dim + 1) * ax.filter_dim;
    case ConvMode::Same: {
      const int64_t off = same_offset(ax.filter_dim);
      int64_t count = 0;
      for (int64_t n = 0; n < ax.output_dim; ++n) {
        // taps k with 0 <= n + off - k < feature
        const int64_t lo = std::max<int64_t>(0, n + off - ax.feature_dim + 1);
        const int64_t hi = std::min<int64_t>(ax.filter_dim - 1, n + off);
        count += hi >= lo ? hi - lo + 1 : 0;
      }
      return count;
    }
  }
  return 0;
}
}  // namespace

u128 flops_actual(const PairwiseOp& op) {
  u128 f = non_conv_product(op);
  for (const auto& ax : op.conv_axes) {
    u128 pairs = (ax.mode == ConvMode::Same || ax.stride > 1) ? static_cast<u128>(conv_pairs(ax))
                 : ax.mode == ConvMode::Valid
                     ? mul_checked(static_cast<u128>(ax.feature_dim - ax.filter_dim + 1),
                                   static_cast<u128>(ax.filter_dim))
                     : mul_checked(static_cast<u128>(ax.feature_dim), static_cast<u128>(ax.filter_dim));
    f = mul_checked(f, pairs);
  }
  return f;
}

// ----------------------------------------------------------------------------- cost
const char* to_string(CostMode m) { return m == CostMode::Inference ? "inference" : "training"; }

CostMode cost_mode_from_string(std::string_view s) {
  if (s == "inference") return CostMode::Inference;
  if (s == "training") return CostMode::Training;
  throw std::invalid_argument("unknown cost mode: " + std::string(s));
}

CostBreakdown pairwise_cost(const PairwiseOp& op, CostMode mode) {
  const u128 f = non_conv_product(op);
  CostBreakdown c;
  c.forward = c.g1 = c.g2 = f;
  for (const auto& ax : op.conv_axes) {
    const u128 x = static_cast<u128>(ax.feature_dim), l = static_cast<u128>(ax.filter_dim),
               xo = static_cast<u128>(ax.output_dim);
    // (a strided axis -- extension -- visits output x filter pairs, not feature x filter)
    c.forward = mul_checked(c.forward, mul_checked(ax.stride > 1 ? xo : x, l));
    c.g1 = mul_checked(c.g1, mul_checked(xo, l));
    c.g2 = mul_checked(c.g2, mul_checked(x, xo));
  }
  if (mode == CostMode::Inference) {
    c.g1 = c.g2 = 0;
    c.total = c.forward;
  } else {
    c.total = add_checked(add_checked(c.forward, c.g1), c.g2);
  }
  return c;
}

}  // namespace ce
