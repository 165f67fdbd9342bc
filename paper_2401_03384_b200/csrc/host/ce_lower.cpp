// Lowering.  The forward index maps restate feature_index()
// (/root/reference/proj/src/kernels.cpp:298-315); the adjoint maps are the
// exact Jacobian transposes listed in SURVEY §8 row A11.
#include <cstdlib>
#include "ce_lower.hpp"

#include <stdexcept>

#include <algorithm>
#include <numeric>

namespace ce {

View dense_view(const Subscripts& subs, const std::vector<int64_t>& dims) {
  return View{subs, dims, row_major_strides(dims)};
}

View padded_view(const Subscripts& subs, const std::vector<int64_t>& dims, int64_t align) {
  View v{subs, dims, std::vector<int64_t>(dims.size())};
  // The innermost axis is padded to `align` elements (16-B row pitch for TMA), except a
  // short one whose product with its short neighbour is already aligned (RTR's 10x10 rank
  // pairs): left dense, the pair stays one contiguous run that merges into one unit.
  static const int pair = [] {  // CE_PAD_PAIR: 0 off, 2 any neighbour (experiment)
    const char* e = std::getenv("CE_PAD_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  const std::size_t n = dims.size();
  // (both axes short: a CP `bhwr` with r = 27 keeps its padded pitch, which the stencil
  // and filter-gradient kernels need for float4 rows)
  const bool dense_pair = pair && n >= 2 && dims[n - 1] % align != 0 && dims[n - 1] < 32 &&
                          (dims[n - 2] < 32 || pair == 2) && (dims[n - 1] * dims[n - 2]) % align == 0;
  int64_t acc = 1;
  for (std::size_t i = n; i-- > 0;) {
    v.strides[i] = acc;
    acc *= (i + 1 == n && !dense_pair) ? (dims[i] + align - 1) / align * align : dims[i];
  }
  return v;
}

int64_t view_span(const View& v) {
  int64_t hi = 0;
  for (std::size_t i = 0; i < v.dims.size(); ++i) hi += (v.dims[i] - 1) * v.strides[i];
  return hi + 1;
}

namespace {

class ProblemBuilder {
 public:
  ProblemBuilder() { p_ = CeProblem{}; }

  int var(int64_t extent, int cls) {
    if (p_.nv >= CE_MAX_VARS) throw ShapeError("pairwise step has too many index variables for the device path");
    const int v = p_.nv++;
    p_.ext[v] = extent;
    p_.cls[v] = cls;
    return v;
  }
  // plain axis `atom` of a view (if present) gets var v
  void plain(int v, const View* a, const View* b, const View* c, const Atom& atom) {
    auto stride = [&](const View* w) -> int64_t {
      if (!w) return 0;
      const int ax = find_atom(w->subs, atom);
      return ax < 0 ? 0 : w->strides[static_cast<std::size_t>(ax)];
    };
    p_.sa[v] = stride(a);
    p_.sb[v] = stride(b);
    p_.sc[v] = stride(c);
  }
  void gather(bool on_a, const View& w, const Atom& atom, int pv, int qv, int sp, int sq, int64_t c,
              bool wrap) {
    const int ax = find_atom(w.subs, atom);
    if (ax < 0) throw ShapeError("lowering: gathered atom '" + atom.name + "' missing");
    CeGather g{};
    g.pv = pv;
    g.qv = qv;
    g.sp = sp;
    g.sq = sq;
    g.c = c;
    g.extent = w.dims[static_cast<std::size_t>(ax)];
    g.stride = w.strides[static_cast<std::size_t>(ax)];
    g.wrap = wrap ? 1 : 0;
    int32_t& n = on_a ? p_.ng_a : p_.ng_b;
    if (n >= CE_MAX_GATHER) throw ShapeError("pairwise step has too many convolution axes for the device path");
    (on_a ? p_.ga : p_.gb)[n++] = g;
  }
  // stride of `atom` in view w (0 when absent), used to set a single operand stride
  static int64_t stride_in(const View& w, const Atom& atom) {
    const int ax = find_atom(w.subs, atom);
    return ax < 0 ? 0 : w.strides[static_cast<std::size_t>(ax)];
  }
  CeProblem& p() { return p_; }

 private:
  CeProblem p_;
};

struct Affine {
  int sp, sq;
  int64_t c;
  bool wrap;
};
// x = f(n, k): the forward feature index (kernels.cpp:298-315); a strided axis (extension,
// ConvModeSpec) scales the output position: x = s*n + ...
Affine forward_map(const ConvAxis& ax) {
  const int s = static_cast<int>(ax.stride);
  switch (ax.mode) {
    case ConvMode::Full: return {s, -1, 0, false};
    case ConvMode::Same: return {s, -1, same_offset(ax.filter_dim), false};
    case ConvMode::Valid: return {s, 1, 0, false};
    case ConvMode::Circular: return {s, -1, 0, true};
  }
  return {s, -1, 0, false};
}
// n = g(x, k): which output position a feature element x meets tap k at.
Affine inverse_map(const ConvAxis& ax) {
  switch (ax.mode) {
    case ConvMode::Full: return {1, 1, 0, false};
    case ConvMode::Same: return {1, 1, -same_offset(ax.filter_dim), false};
    case ConvMode::Valid: return {1, -1, 0, false};
    case ConvMode::Circular: return {1, 1, 0, true};
  }
  return {1, 1, 0, false};
}

}  // namespace

CeProblem lower_pairwise(const PairwiseOp& op, const View& left, const View& right, const View& result,
                         const View& out, Adjoint which) {
  ProblemBuilder b;
  const View* A = which == Adjoint::GradLeft ? &result : &left;
  const View* B = which == Adjoint::GradRight ? &result : &right;
  // var class of each non-conv role under the three lowerings
  enum Role { kBatch, kContract, kLFree, kRFree };
  static const int kClass[3][4] = {
      /*Forward  */ {CE_Z, CE_K, CE_M, CE_N},
      /*GradLeft */ {CE_Z, CE_N, CE_M, CE_K},
      /*GradRight*/ {CE_Z, CE_M, CE_K, CE_N},
  };
  const int w = static_cast<int>(which);
  auto plain_role = [&](const Subscripts& atoms, const std::vector<int64_t>& dims, Role r) {
    for (std::size_t i = 0; i < atoms.size(); ++i) b.plain(b.var(dims[i], kClass[w][r]), A, B, &out, atoms[i]);
  };
  plain_role(op.batch_atoms, op.batch_dims, kBatch);
  plain_role(op.contraction_atoms, op.contraction_dims, kContract);
  plain_role(op.left_free, op.left_free_dims, kLFree);
  plain_role(op.right_free, op.right_free_dims, kRFree);

  for (const ConvAxis& ax : op.conv_axes) {
    const Atom& a = ax.atom;
    if (which == Adjoint::Forward) {
      // p = output position (with the feature side), q = tap (summed)
      const int pv = b.var(ax.output_dim, ax.feature_on_left ? CE_M : CE_N);
      const int qv = b.var(ax.filter_dim, CE_K);
      const Affine f = forward_map(ax);
      b.p().sc[pv] = ProblemBuilder::stride_in(out, a);
      if (ax.feature_on_left) {
        b.gather(true, *A, a, pv, qv, f.sp, f.sq, f.c, f.wrap);
        b.p().sb[qv] = ProblemBuilder::stride_in(*B, a);
      } else {
        b.gather(false, *B, a, pv, qv, f.sp, f.sq, f.c, f.wrap);
        b.p().sa[qv] = ProblemBuilder::stride_in(*A, a);
      }
      continue;
    }
    // Which operand of the original node is being differentiated, and is it the feature?
    const bool grad_of_left = which == Adjoint::GradLeft;
    const bool grad_is_feature = grad_of_left == ax.feature_on_left;
    // The dC operand sits on the A side for GradLeft and on the B side for GradRight;
    // the other original operand sits on the opposite side.
    const bool dc_on_a = grad_of_left;
    const View& dc = dc_on_a ? *A : *B;
    const View& other = dc_on_a ? *B : *A;
    if (grad_is_feature) {
      // (a strided axis has no affine inverse: the executor upsamples dC and lowers a
      // stride-1 op over it, see Executor::build_backward)
      if (ax.stride != 1) throw std::logic_error("lower_pairwise: strided feature gradient needs an upsampled dC");
      // d feature[x] = sum_k filter[k] * dC[g(x, k)] : p' = x (side of dC), q' = k
      const int pv = b.var(ax.feature_dim, dc_on_a ? CE_M : CE_N);
      const int qv = b.var(ax.filter_dim, CE_K);
      const Affine g = inverse_map(ax);
      b.p().sc[pv] = ProblemBuilder::stride_in(out, a);
      b.gather(dc_on_a, dc, a, pv, qv, g.sp, g.sq, g.c, g.wrap);
      (dc_on_a ? b.p().sb : b.p().sa)[qv] = ProblemBuilder::stride_in(other, a);
    } else {
      // d filter[k] = sum_n feature[f(n, k)] * dC[n] : p' = k (side of the feature), q' = n
      const int pv = b.var(ax.filter_dim, dc_on_a ? CE_N : CE_M);
      const int qv = b.var(ax.output_dim, CE_K);
      const Affine f = forward_map(ax);
      b.p().sc[pv] = ProblemBuilder::stride_in(out, a);
      // feature index = sp*n + sq*k + c with n = q', k = p'
      b.gather(!dc_on_a, other, a, pv, qv, f.sq, f.sp, f.c, f.wrap);
      (dc_on_a ? b.p().sa : b.p().sb)[qv] = ProblemBuilder::stride_in(dc, a);
    }
  }
  return b.p();
}

CeProblem lower_unary(const View& in, const View& out) {
  ProblemBuilder b;
  b.p().unary = 1;
  for (std::size_t i = 0; i < in.subs.size(); ++i) {
    const bool kept = find_atom(out.subs, in.subs[i]) >= 0;
    const int v = b.var(in.dims[i], kept ? CE_M : CE_K);
    b.plain(v, &in, nullptr, &out, in.subs[i]);
  }
  for (std::size_t i = 0; i < out.subs.size(); ++i)
    if (find_atom(in.subs, out.subs[i]) < 0) b.plain(b.var(out.dims[i], CE_M), &in, nullptr, &out, out.subs[i]);
  return b.p();
}

CeSimtDesc simt_desc(const CeProblem& p) {
  CeSimtDesc d{};
  d.p = p;
  d.Z = d.M = d.N = d.K = 1;
  // Per class, order vars fastest-first by the stride of the operand that
  // streams them (A for M/K, B for N, out for Z) so consecutive threads touch
  // consecutive addresses.
  auto key = [&](int v) -> int64_t {
    const int64_t g = [&] {
      for (int i = 0; i < p.ng_a; ++i)
        if (p.ga[i].pv == v || p.ga[i].qv == v) return p.ga[i].stride;
      for (int i = 0; i < p.ng_b; ++i)
        if (p.gb[i].pv == v || p.gb[i].qv == v) return p.gb[i].stride;
      return int64_t{0};
    }();
    switch (p.cls[v]) {
      case CE_M: return p.sa[v] ? p.sa[v] : (g ? g : p.sc[v]);
      case CE_N: return p.sb[v] ? p.sb[v] : (g ? g : p.sc[v]);
      case CE_K: return p.sa[v] ? p.sa[v] : (p.sb[v] ? p.sb[v] : g);
      default: return p.sc[v];
    }
  };
  std::vector<int> order(static_cast<std::size_t>(p.nv));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return key(a) < key(c); });
  for (int v : order) {
    switch (p.cls[v]) {
      case CE_Z: d.zv[d.nz++] = v; d.Z *= p.ext[v]; break;
      case CE_M: d.mv[d.nm++] = v; d.M *= p.ext[v]; break;
      case CE_N: d.nvv[d.nn++] = v; d.N *= p.ext[v]; break;
      default: d.kv[d.nk++] = v; d.K *= p.ext[v]; break;
    }
  }
  // direct kernel: output vars by out stride, fastest first
  std::vector<int> outv;
  for (int v = 0; v < p.nv; ++v)
    if (p.cls[v] != CE_K) outv.push_back(v);
  std::stable_sort(outv.begin(), outv.end(), [&](int a, int c) { return p.sc[a] < p.sc[c]; });
  for (int v : outv) d.ov[d.nout++] = v;
  return d;
}

}  // namespace ce
