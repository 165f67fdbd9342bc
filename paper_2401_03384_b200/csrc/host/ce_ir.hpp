// conv_einsum host IR: atoms, expressions, shapes, pairwise roles and the
// tnn-cost model.  API-compatible re-statement of the reference `convexpr`
// headers (proj/include/convexpr/{checked_int,expression,tensor,kernels,cost}.hpp)
// in namespace `ce`, so both can be linked into one test binary.  Every
// function here must agree with the reference bit for bit (tests/test_planner.py).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace ce {

// ---- 128-bit checked arithmetic (checked_int.hpp:11-42) ---------------------
using u128 = unsigned __int128;

struct OverflowError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
u128 mul_checked(u128 a, u128 b);
u128 add_checked(u128 a, u128 b);
std::string u128_to_string(u128 v);

// ---- errors ------------------------------------------------------------------
struct ParseError : std::runtime_error {
  ParseError(const std::string& msg, std::size_t pos);
  std::size_t position;
};
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- expression IR (expression.hpp:15-83) ------------------------------------
struct Atom {
  std::string name;
  Atom() = default;
  Atom(std::string n) : name(std::move(n)) {}
  Atom(const char* n) : name(n) {}
  friend bool operator==(const Atom& a, const Atom& b) { return a.name == b.name; }
  friend bool operator<(const Atom& a, const Atom& b) { return a.name < b.name; }
};
using Subscripts = std::vector<Atom>;

enum class AtomClass { Convolution, BatchProduct, Contraction, Free, SelfContraction };
const char* to_string(AtomClass c);

struct ExpressionSpec {
  std::vector<Subscripts> inputs;
  Subscripts output;
  Subscripts conv_atoms;  // canonical order = output order

  bool is_conv(const Atom& a) const;
  int occurrence_count(const Atom& a) const;
  bool in_output(const Atom& a) const;
  Subscripts all_atoms() const;  // first appearance over inputs, left to right
  std::size_t input_count() const { return inputs.size(); }
};

ExpressionSpec parse(std::string_view source);
std::string render(const Subscripts& subs);
std::string render(const ExpressionSpec& spec);
std::map<Atom, AtomClass> classify(const ExpressionSpec& spec);

int find_atom(const Subscripts& subs, const Atom& a);  // -1 when absent

// ---- shapes (tensor.hpp:20-87) -------------------------------------------------
int64_t element_count(const std::vector<int64_t>& shape);
std::vector<int64_t> row_major_strides(const std::vector<int64_t>& shape);

struct ShapeEnv {
  std::vector<std::vector<int64_t>> dims;
  int64_t dim_of(const ExpressionSpec& spec, const Atom& a) const;
};
ShapeEnv make_shape_env(const ExpressionSpec& spec, std::vector<std::vector<int64_t>> dims);

// SplitMix64 (tensor.cpp:107-130): the deterministic input generator.  The
// device generator in csrc/cuda/ce_fill.cu evaluates the same stream in closed
// form (element i uses state seed + (i+1)*golden).
struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t seed) : state(seed) {}
  uint64_t next();
  double next_unit();
  int64_t next_in(int64_t lo, int64_t hi);
};

// ---- convolution modes (kernels.hpp:15-33) ---------------------------------------
enum class ConvMode { Full, Same, Valid, Circular };
const char* to_string(ConvMode m);
ConvMode conv_mode_from_string(std::string_view s);
// Extension (outside the reference semantics): a conv atom may
// carry an output stride s ("same/2"): output position n reads feature index s*n + (the
// stride-1 map's offset), e.g. Same x = s*n + floor((L-1)/2) - k, and the output length
// becomes Full floor((X+L-2)/s)+1, Same / Circular ceil(X/s), Valid floor((X-L)/s)+1.  Stride 1
// is exactly the reference's ConvMode (kernels.hpp:15-33), bit-exact everywhere.
struct ConvModeSpec {
  ConvMode mode = ConvMode::Same;
  int64_t stride = 1;
  ConvModeSpec() = default;
  ConvModeSpec(ConvMode m, int64_t s = 1) : mode(m), stride(s) {}  // NOLINT: implicit from ConvMode
  operator ConvMode() const { return mode; }                       // NOLINT
};
ConvModeSpec conv_mode_spec_from_string(std::string_view s);  // "same" | "same/2"
int64_t conv_output_dim(ConvMode mode, int64_t feature, int64_t filter, int64_t stride = 1);
using ConvModeMap = std::map<Atom, ConvModeSpec>;
ConvModeMap resolve_conv_modes(const ExpressionSpec& spec, ConvModeSpec requested);
inline int64_t same_offset(int64_t filter) { return (filter - 1) / 2; }

// ---- pairwise op (kernels.hpp:35-72) --------------------------------------------
struct ConvAxis {
  Atom atom;
  ConvMode mode = ConvMode::Same;
  bool feature_on_left = true;
  int64_t feature_dim = 1;
  int64_t filter_dim = 1;
  int64_t output_dim = 1;
  int64_t stride = 1;  // extension, see ConvModeSpec
};

struct PairwiseOp {
  Subscripts left, right, result;
  std::vector<int64_t> left_dims, right_dims, result_dims;
  std::vector<ConvAxis> conv_axes;
  Subscripts batch_atoms, contraction_atoms, left_free, right_free, left_self, right_self;
  std::vector<int64_t> batch_dims, contraction_dims, left_free_dims, right_free_dims;
  int64_t result_elements() const { return element_count(result_dims); }
};

PairwiseOp make_pairwise_op(const Subscripts& left, const std::vector<int64_t>& left_dims,
                            const Subscripts& right, const std::vector<int64_t>& right_dims,
                            const std::set<Atom>& keep, const ConvModeMap& conv_modes,
                            const std::optional<Subscripts>& result_order = std::nullopt);

u128 flops_actual(const PairwiseOp& op);

// ---- cost model (cost.hpp:8-32) ---------------------------------------------------
enum class CostMode { Inference, Training };
const char* to_string(CostMode m);
CostMode cost_mode_from_string(std::string_view s);

struct CostBreakdown {
  u128 forward = 0, g1 = 0, g2 = 0, total = 0;
};
CostBreakdown pairwise_cost(const PairwiseOp& op, CostMode mode);

}  // namespace ce
