// Executor implementation.  Structure follows the reference's execute()
// (sequencer.cpp:403-447) and pairwise_eval (kernels.cpp:425-470):
//   self-contraction pre-sum (sum_unique_modes, kernels.cpp:144-187)
//   -> core (grouped_conv_core, kernels.cpp:320-399)
//   -> result in op.result order; the root permute to spec.output
//      (sequencer.cpp:439-445) is fused into the last node's store.
// Backward (absent from the reference) walks the nodes in reverse, producing
// dA / dB with the adjoint lowerings of ce_lower.cpp.
#include "ce_exec.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <stdexcept>

#include "../cuda/ce_kernels.h"

namespace ce {

namespace {
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

Subscripts minus(const Subscripts& s, const Subscripts& drop) {
  Subscripts out;
  for (const auto& a : s)
    if (find_atom(drop, a) < 0) out.push_back(a);
  return out;
}

std::vector<int64_t> dims_of(const View& v, const Subscripts& subs) {
  std::vector<int64_t> d;
  for (const auto& a : subs) d.push_back(v.dims[static_cast<std::size_t>(find_atom(v.subs, a))]);
  return d;
}
}  // namespace

Executor::Executor(const EvaluationPlan& plan, bool want_backward, ExecConfig cfg)
    : plan_(plan), want_backward_(want_backward), cfg_(cfg) {
  n_ = static_cast<int>(plan_.spec.inputs.size());
  for (int i = 0; i < n_; ++i) {
    id_view_.push_back(dense_view(plan_.spec.inputs[static_cast<std::size_t>(i)], plan_.env.dims[static_cast<std::size_t>(i)]));
    id_ref_.push_back({BufRef::kInput, i});
  }
  build_forward();
  if (want_backward_) build_backward();
  if (hoist_packs()) {
    reset_build();
    build_forward();
    if (want_backward_) build_backward();
  }
  early_packs(fwd_);
  early_packs(bwd_);
  static const bool fuse_on = [] {  // CE_FUSE=0: no node fusion
    const char* e = std::getenv("CE_FUSE");
    return !(e && *e == '0');
  }();
  // (recompute first: the forward pass's intermediates are then read by no backward step,
  // so a fused forward pair need not store its intermediate)
  if (want_backward_ && cfg_.recompute) add_recompute();
  if (fuse_on && tc_math()) {
    fuse_chains(fwd_);
    fuse_chains(bwd_);
  }
  // hazards by buffer identity first (the happens-before order assign_offsets may alias
  // under), then again once buffers share memory (those extra edges are already implied)
  compute_deps(fwd_);
  compute_deps(bwd_);
  share_sms(bwd_);
  assign_offsets();
  if (ws_reuse_mode_ >= 2) {  // (mode 1 shares only along edges the identity hazards already imply)
    compute_deps(fwd_);
    compute_deps(bwd_);
  }
  if (const char* e = std::getenv("CE_CONCURRENT"); e && *e == '0') concurrent_ = false;
  if (const char* e = std::getenv("CE_STREAMS")) n_streams_ = std::max(2, std::min(kMaxStreams, std::atoi(e)));
  if (const char* dbg = std::getenv("CE_DEBUG"); dbg && *dbg == '1') std::fputs(describe().c_str(), stderr);
}

void Executor::reset_build() {
  fwd_.clear();
  bwd_.clear();
  packs_.clear();
  pack_log_.clear();
  buf_bytes_.clear();
  buf_owner_.clear();
  id_view_.resize(static_cast<std::size_t>(n_));
  id_ref_.resize(static_cast<std::size_t>(n_));
  for (int s = 0; s < 2; ++s) {
    red_view_[s].clear();
    red_ref_[s].clear();
  }
  pending_flops_ = 0;
}

// Layout hoisting (CE_HOIST: 0 off, 1 (default) node results, 2 also gradient buffers:
// measured worse on RTR 64->128, 44 -> 52 ms, the gradient producers' stores fragment).
// A repack of a buffer our own step produced costs a full HBM round trip of it (RTR's 5-GB
// intermediates: 2.5-3.2 ms each); writing the buffer in the packed layout in the first
// place costs only the producer's epilogue pattern.  The first pack of each such buffer
// names its layout: each atom's output stride is read off the pack's axis that holds it
// (atoms merged into one pack axis keep their relative strides).  Returns whether any
// layout changed (the caller rebuilds the steps).
bool Executor::hoist_packs() {
  static const int mode = [] {
    const char* e = std::getenv("CE_HOIST");
    return e ? std::atoi(e) : 1;
  }();
  if (mode <= 0 || !tc_math()) return false;
  bool changed = false;
  std::set<std::pair<int, bool>> seen;
  for (const PackLog& r : pack_log_) {
    if (r.src.kind != BufRef::kWork || r.pk.ng_a != 0) continue;
    const auto it = buf_owner_.find(r.src.index);
    if (it == buf_owner_.end()) continue;
    const int id = it->second.first;
    const bool grad = it->second.second;
    if (grad ? mode < 2 : mode < 1) continue;
    std::map<int, View>& lay = grad ? grad_layout_ : res_layout_;
    // only the buffer's first pack (its first consumer's layout) is a candidate
    if (!seen.insert({id, grad}).second) continue;
    const View& v = id_view_[static_cast<std::size_t>(id)];
    double elems = 1, pk_elems = 1;
    for (int64_t d : v.dims) elems *= static_cast<double>(d);
    for (int k = 0; k < r.pk.nv; ++k) pk_elems *= static_cast<double>(r.pk.ext[k]);
    if (elems != pk_elems) continue;  // not a pure permute of the whole buffer
    // only buffers whose round trip matters (>= 64 MB): small packs are cheap, and their
    // consumers' tile plans are tuned to the padded result order
    static const double min_elems = [] {  // CE_HOIST_MIN_MB (default 64)
      const char* e = std::getenv("CE_HOIST_MIN_MB");
      return (e ? std::atof(e) : 64.0) * 1024.0 * 1024.0 / 4.0;
    }();
    if (elems < min_elems) continue;
    View nv = v;
    bool ok = true;
    for (std::size_t i = 0; i < v.dims.size() && ok; ++i) {
      if (v.dims[i] == 1) continue;
      const int64_t st = v.strides[i];
      ok = false;
      for (int k = 0; k < r.pk.nv; ++k) {
        const int64_t s0 = r.pk.sa[k];
        if (s0 <= 0 || st < s0 || st % s0 != 0 || (st / s0) * v.dims[i] > r.pk.ext[k]) continue;
        nv.strides[i] = r.pk.sc[k] * (st / s0);
        ok = true;
        break;
      }
    }
    if (!ok) continue;
    // the producer's epilogue writes runs along the new unit-stride atom: under 8 floats
    // (32-B sectors) its stores fragment (RTR's N0 with s1 = 4 innermost: node0 2.5 ->
    // 5.7 ms and dW4 0.9 -> 7.1 ms, measured), so such layouts are not hoisted
    int64_t inner = 0;
    for (std::size_t i = 0; i < nv.dims.size(); ++i)
      if (nv.dims[i] > 1 && nv.strides[i] == 1) inner = nv.dims[i];
    if (inner < 8) continue;
    lay[id] = nv;
    changed = true;
  }
  return changed;
}

Executor::~Executor() {
  if (ws_) cudaFree(ws_);
  if (tail_flags_) cudaFree(tail_flags_);
  for (auto* list : {&fwd_, &bwd_})
    for (Step& st : *list) {
      if (st.ev0) cudaEventDestroy(st.ev0);
      if (st.ev1) cudaEventDestroy(st.ev1);
    }
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto* list : {&fwd_, &bwd_})
    for (Step& st : *list)
      if (st.done) cudaEventDestroy(st.done);
  for (int k = 0; k < kMaxStreams - 1; ++k) {
    if (aux_[k]) cudaStreamDestroy(aux_[k]);
    if (join_ev_[k]) cudaEventDestroy(join_ev_[k]);
  }
  if (fork_ev_) cudaEventDestroy(fork_ev_);
}

// Two references that may touch the same bytes: the same caller buffer, or workspace
// buffers whose assigned ranges intersect (distinct buffers share memory when their
// lifetimes are disjoint, see assign_offsets).
bool Executor::overlap(const BufRef& x, const BufRef& y) const {
  if (x.kind == BufRef::kNone || x.kind != y.kind) return false;
  if (x.index == y.index) return true;
  if (x.kind != BufRef::kWork || buf_off_.empty()) return false;
  const auto i = static_cast<std::size_t>(x.index), j = static_cast<std::size_t>(y.index);
  return buf_off_[i] < buf_off_[j] + buf_bytes_[j] && buf_off_[j] < buf_off_[i] + buf_bytes_[i];
}

// Liveness-based workspace placement (the reference keeps every intermediate
// alive, sequencer.cpp:421-433).  Two buffers may share memory only when every step touching
// one HAPPENS BEFORE every step touching the other in the passes' existing dependency order
// (the forward pass entirely precedes the backward pass; within a pass, the transitive
// closure of the identity hazards of compute_deps), so sharing never adds a synchronisation
// the side streams did not already have.  Buffers are placed largest first at the lowest
// offset free of every placed buffer they may not share with.  CE_WS_REUSE=0: bump layout.
void Executor::assign_offsets() {
  const std::size_t nb = buf_bytes_.size();
  ws_unshared_ = 0;
  for (int64_t b : buf_bytes_) ws_unshared_ += b;
  buf_off_.assign(nb, 0);
  // CE_WS_REUSE: 0 bump layout; 1 share only along the existing happens-before order (no
  // new synchronisation: cfg2 step within noise of the bump layout); 2 share whenever the
  // lifetimes are disjoint on the step timeline (the hazard edges this adds between side
  // streams cost the cfg2 step ~7%, same-box A/B).  Default: 1, or 2 when the bump layout
  // would exceed CE_WS_TIGHT_GB (16) -- e.g. cfg3's 64->128 layer at B=256: 54 -> 22 GB.
  static const int reuse_env = [] {
    const char* e = std::getenv("CE_WS_REUSE");
    return e ? std::atoi(e) : -1;
  }();
  static const double tight_gb = [] {
    const char* e = std::getenv("CE_WS_TIGHT_GB");
    return e ? std::atof(e) : 16.0;
  }();
  const int reuse = reuse_env >= 0 ? reuse_env : (static_cast<double>(ws_unshared_) > tight_gb * 1073741824.0 ? 2 : 1);
  ws_reuse_mode_ = reuse;
  if (!reuse) {
    int64_t off = 0;
    for (std::size_t i = 0; i < nb; ++i) {
      buf_off_[i] = off;
      off += buf_bytes_[i];
    }
    ws_bytes_ = off;
    return;
  }
  // global step index t: forward steps 0..F-1, backward steps F..F+B-1
  const std::size_t F = fwd_.size(), T = F + bwd_.size();
  std::vector<std::vector<uint64_t>> before(T, std::vector<uint64_t>((T + 63) / 64, 0));  // before[t]: steps ordered before t
  auto set = [&](std::size_t t, std::size_t u) { before[t][u / 64] |= 1ull << (u % 64); };
  auto get = [&](std::size_t t, std::size_t u) { return (before[t][u / 64] >> (u % 64)) & 1ull; };
  for (std::size_t t = 0; t < T; ++t) {
    const bool bwd = t >= F;
    const Step& st = bwd ? bwd_[t - F] : fwd_[t];
    if (bwd)
      for (std::size_t u = 0; u < F; ++u) set(t, u);
    for (int d : st.deps) {
      const std::size_t u = (bwd ? F : 0) + static_cast<std::size_t>(d);
      set(t, u);
      for (std::size_t w = 0; w < before[t].size(); ++w) before[t][w] |= before[u][w];
    }
  }
  std::vector<std::vector<std::size_t>> uses(nb);
  std::vector<int> last(nb, -1);
  {
    std::size_t t = 0;
    for (const auto* list : {&fwd_, &bwd_})
      for (const Step& st : *list) {
        for (const BufRef* r : {&st.a, &st.b, &st.c, &st.b2, &st.c2})
          if (r->kind == BufRef::kWork) {
            const auto i = static_cast<std::size_t>(r->index);
            if (uses[i].empty() || uses[i].back() != t) uses[i].push_back(t);
            last[i] = static_cast<int>(t);
          }
        ++t;
      }
  }
  auto ordered = [&](std::size_t x, std::size_t y) {  // every use of x happens before every use of y
    if (reuse >= 2) return !uses[x].empty() && !uses[y].empty() && uses[x].back() < uses[y].front();
    for (std::size_t u : uses[y])
      for (std::size_t v : uses[x])
        if (!get(u, v)) return false;
    return true;
  };
  std::vector<int> first(nb, INT32_MAX);
  for (std::size_t i = 0; i < nb; ++i)
    if (!uses[i].empty()) first[i] = static_cast<int>(uses[i].front());
  std::vector<std::size_t> order(nb);
  for (std::size_t i = 0; i < nb; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
    if (buf_bytes_[x] != buf_bytes_[y]) return buf_bytes_[x] > buf_bytes_[y];
    return first[x] < first[y];
  });
  std::vector<std::size_t> placed;
  ws_bytes_ = 0;
  for (std::size_t i : order) {
    if (last[i] < 0) continue;  // never referenced by a step (e.g. an intermediate a fusion keeps on chip)
    std::vector<std::pair<int64_t, int64_t>> busy;  // ranges of placed buffers alive with i
    for (std::size_t j : placed)
      if (!(ordered(i, j) || ordered(j, i))) busy.push_back({buf_off_[j], buf_off_[j] + buf_bytes_[j]});
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (const auto& r : busy) {
      if (off + buf_bytes_[i] <= r.first) break;
      off = std::max(off, r.second);
    }
    buf_off_[i] = off;
    ws_bytes_ = std::max(ws_bytes_, off + buf_bytes_[i]);
    placed.push_back(i);
  }
}

// Read-after-write, write-after-write and write-after-read hazards between the steps of
// one pass (buffers that may share bytes, overlap()).
void Executor::compute_deps(std::vector<Step>& steps) const {
  auto same = [this](const BufRef& x, const BufRef& y) { return overlap(x, y); };
  for (std::size_t i = 0; i < steps.size(); ++i) {
    Step& si = steps[i];
    si.deps.clear();
    for (std::size_t j = 0; j < i; ++j) {
      const Step& sj = steps[j];
      bool hazard = false;
      for (const BufRef* w : {&sj.c, &sj.c2})
        for (const BufRef* r : {&si.a, &si.b, &si.b2, &si.c, &si.c2}) hazard = hazard || same(*w, *r);  // RAW, WAW
      for (const BufRef* r : {&sj.a, &sj.b, &sj.b2})
        for (const BufRef* w : {&si.c, &si.c2}) hazard = hazard || same(*r, *w);  // WAR
      if (hazard) si.deps.push_back(static_cast<int>(j));
    }
  }
}

void Executor::launch_pass(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s, int which) {
  if (profiling_) {
    // capture with per-step event records so the timings are back-to-back device time,
    // free of host enqueue gaps; the graph is not cached
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
      run(steps, need, s);
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    cuda_check(cudaStreamEndCapture(s, &graph), "cudaStreamEndCapture");
    cuda_check(cudaGraphInstantiate(&exec, graph, 0), "cudaGraphInstantiate");
    cuda_check(cudaGraphLaunch(exec, s), "cudaGraphLaunch");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    return;
  }
  // inside a caller's stream capture (a whole training step captured as one CUDA graph) the
  // steps are launched directly, so they become nodes of the caller's graph
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(s, &cap), "cudaStreamIsCapturing");
  if (!use_graphs_ || cap != cudaStreamCaptureStatusNone) {
    run(steps, need, s);
    return;
  }
  // replay key: every bound pointer plus the requested-gradient mask
  std::vector<const void*> key;
  key.reserve(steps.size() * 3 + 16);
  for (const Step& st : steps) {
    key.push_back(resolve(st.a));
    key.push_back(resolve(st.b));
    key.push_back(resolve(st.c));
    if (st.kind == Step::kDw2) {
      key.push_back(resolve(st.b2));
      key.push_back(resolve(st.c2));
    }
  }
  if (need)
    for (char c : *need) key.push_back(reinterpret_cast<const void*>(static_cast<uintptr_t>(c)));
  GraphCache& g = graphs_[which];
  if (g.exec && g.key == key) {
    cuda_check(cudaGraphLaunch(g.exec, s), "cudaGraphLaunch");
    last_launches_ = g.launches;
    return;
  }
  cudaGraph_t graph = nullptr;
  cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  try {
    run(steps, need, s);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  cuda_check(cudaStreamEndCapture(s, &graph), "cudaStreamEndCapture");
  if (g.exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(g.exec, graph, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
  }
  if (!g.exec) cuda_check(cudaGraphInstantiate(&g.exec, graph, 0), "cudaGraphInstantiate");
  cudaGraphDestroy(graph);
  g.key = std::move(key);
  g.launches = last_launches_;
  cuda_check(cudaGraphLaunch(g.exec, s), "cudaGraphLaunch");
}

namespace {
// Logical (compulsory) element counts of A, B and C of a lowered problem.
double operand_elems(const CeProblem& p, int which) {
  double n = 1;
  if (which == 2) {
    for (int v = 0; v < p.nv; ++v)
      if (p.cls[v] != CE_K) n *= static_cast<double>(p.ext[v]);
    return n;
  }
  const int64_t* s = which == 0 ? p.sa : p.sb;
  const CeGather* g = which == 0 ? p.ga : p.gb;
  const int ng = which == 0 ? p.ng_a : p.ng_b;
  if (which == 1 && p.unary) return 0;
  for (int v = 0; v < p.nv; ++v)
    if (s[v]) n *= static_cast<double>(p.ext[v]);
  for (int i = 0; i < ng; ++i) n *= static_cast<double>(g[i].extent);
  return n;
}
double problem_bytes(const CeProblem& p) {
  return 4.0 * (operand_elems(p, 0) + operand_elems(p, 1) + operand_elems(p, 2));
}
}  // namespace

int64_t Executor::alloc(int64_t elems) {
  buf_bytes_.push_back((elems * 4 + 255) / 256 * 256);
  return static_cast<int64_t>(buf_bytes_.size()) - 1;
}

std::vector<int64_t> Executor::output_dims() const {
  std::vector<int64_t> d;
  if (plan_.nodes.empty()) {
    for (const auto& a : plan_.spec.output) d.push_back(plan_.env.dim_of(plan_.spec, a));
  } else {
    const auto& op = plan_.nodes.back().op;
    for (const auto& a : plan_.spec.output)
      d.push_back(op.result_dims[static_cast<std::size_t>(find_atom(op.result, a))]);
  }
  return d;
}

namespace {
// A unary permute that rewrites one operand of `p` so that the vars in
// `inner_order` become its innermost axes (inner_order[0] unit-stride, innermost
// pitch padded to 16 B) and every other axis keeps its relative order.  Returns
// the pack problem and patches p's strides for that operand in place.
CeProblem repack(CeProblem& p, bool side_b, const std::vector<int>& inner_order, int64_t* span,
                 const int64_t* partner = nullptr, bool out_c_order = false) {
  int64_t* s = side_b ? p.sb : p.sa;
  CeGather* g = side_b ? p.gb : p.ga;
  const int ng = side_b ? p.ng_b : p.ng_a;
  struct Ax { int64_t stride, ext; int var, gi, rank; };
  std::vector<Ax> ax;
  auto rank_of = [&](int v) {
    for (std::size_t i = 0; i < inner_order.size(); ++i)
      if (inner_order[i] == v) return static_cast<int>(i);
    return 1 << 20;
  };
  for (int v = 0; v < p.nv; ++v)
    if (s[v]) ax.push_back({s[v], p.ext[v], v, -1, rank_of(v)});
  for (int i = 0; i < ng; ++i) ax.push_back({g[i].stride, g[i].extent, -1, i, 1 << 20});
  // innermost first: listed vars in order, then the rest by ascending original stride
  std::stable_sort(ax.begin(), ax.end(), [](const Ax& x, const Ax& y) {
    if (x.rank != y.rank) return x.rank < y.rank;
    return x.stride < y.stride;
  });
  // the output vars among the rest take their slots in C's stride order: the tile units they
  // form then enumerate columns / rows in C order, so the epilogue's 4-column groups are
  // contiguous in C (float4 stores) -- K vars keep their slots (same K units)
  // Default since the end of round 2 (CE_PACK_CORDER=0 off): cfg3 stack 62.15 -> 61.49 ms (RTR
  // 64->128 26.08 -> 25.41 ms), cfg2 step and cfg4 unchanged within noise (same-box A/B x2-3).
  // (Round 1, before the row GEMMs / plane convolutions: conv1 17.0 -> 17.4 ms, cfg2 +0.3%.)
  static const bool c_order = [] {
    const char* e = std::getenv("CE_PACK_CORDER");
    return !(e && *e == '0');
  }();
  if (c_order || out_c_order) {
    std::vector<std::size_t> slots;
    std::vector<Ax> outs;
    for (std::size_t i = 0; i < ax.size(); ++i)
      if (ax[i].rank >= (1 << 20) && ax[i].var >= 0 && p.cls[ax[i].var] != CE_K && p.sc[ax[i].var]) {
        slots.push_back(i);
        outs.push_back(ax[i]);
      }
    std::stable_sort(outs.begin(), outs.end(), [&](const Ax& x, const Ax& y) { return p.sc[x.var] < p.sc[y.var]; });
    for (std::size_t k = 0; k < slots.size(); ++k) ax[slots[k]] = outs[k];
  }
  CeProblem pk{};
  pk.unary = 1;
  int64_t acc = 1;
  for (std::size_t i = 0; i < ax.size(); ++i) {
    // the listed vars stay contiguous (so they can merge into one K unit); the first
    // axis after them starts on a 16-byte boundary (TMA stride legality)
    if (i > 0 && ax[i].rank >= (1 << 20) && ax[i - 1].rank < (1 << 20)) acc = (acc + 3) / 4 * 4;
    // listed vars that do not chain in the partner operand cannot merge: keep 16-byte strides
    if (partner && i > 0 && ax[i].rank < (1 << 20) && ax[i].var >= 0 && ax[i - 1].var >= 0 &&
        partner[ax[i].var] != partner[ax[i - 1].var] * p.ext[ax[i - 1].var])
      acc = (acc + 3) / 4 * 4;
    const int v = pk.nv++;
    pk.ext[v] = ax[i].ext;
    pk.cls[v] = CE_M;
    pk.sa[v] = ax[i].stride;
    pk.sc[v] = acc;
    if (ax[i].var >= 0) s[ax[i].var] = acc; else g[ax[i].gi].stride = acc;
    acc *= ax[i].ext;
  }
  *span = acc;
  return pk;
}

// Explicit tap expansion ("im2col") of one operand: every gathered axis (p, q) of that
// side becomes two plain axes p and q of a new buffer E (out-of-range taps written as
// zeros, circular ones wrapped), so the step itself has no gather on that side and the
// tensor cores can take it.  Used when the gather sits on the operand's unit-stride axis
// (RTR's X[b,s,h+i,w+j] contracted over the taps only), which neither TMA boxes nor a
// repack can express.  `inner_order` vars become E's innermost axes as in repack().
// Returns the unary gather problem that writes E and patches p in place.
CeProblem expand(CeProblem& p, bool side_b, const std::vector<int>& inner_order, int64_t* span) {
  int64_t* s = side_b ? p.sb : p.sa;
  CeGather* g = side_b ? p.gb : p.ga;
  int& ng = side_b ? p.ng_b : p.ng_a;
  struct Ax { int64_t key; int var, rank; };
  std::vector<Ax> ax;
  auto rank_of = [&](int v) {
    for (std::size_t i = 0; i < inner_order.size(); ++i)
      if (inner_order[i] == v) return static_cast<int>(i);
    return 1 << 20;
  };
  std::vector<int> seen(static_cast<std::size_t>(p.nv), 0);
  for (int v = 0; v < p.nv; ++v)
    if (s[v]) {
      ax.push_back({s[v], v, rank_of(v)});
      seen[static_cast<std::size_t>(v)] = 1;
    }
  for (int i = 0; i < ng; ++i)
    for (int v : {g[i].qv, g[i].pv})
      if (!seen[static_cast<std::size_t>(v)]) {
        ax.push_back({g[i].stride, v, rank_of(v)});
        seen[static_cast<std::size_t>(v)] = 1;
      }
  std::stable_sort(ax.begin(), ax.end(), [](const Ax& x, const Ax& y) {
    if (x.rank != y.rank) return x.rank < y.rank;
    return x.key < y.key;
  });
  CeProblem pk{};
  pk.unary = 1;
  std::vector<int> pvar(static_cast<std::size_t>(p.nv), -1);
  int64_t acc = 1;
  std::vector<int64_t> ns(static_cast<std::size_t>(p.nv), 0);
  for (std::size_t i = 0; i < ax.size(); ++i) {
    if (i > 0 && ax[i].rank >= (1 << 20) && ax[i - 1].rank < (1 << 20)) acc = (acc + 3) / 4 * 4;
    const int v = pk.nv++;
    pvar[static_cast<std::size_t>(ax[i].var)] = v;
    pk.ext[v] = p.ext[ax[i].var];
    pk.cls[v] = CE_M;
    pk.sa[v] = s[ax[i].var];  // 0 for the gathered vars
    pk.sc[v] = acc;
    ns[static_cast<std::size_t>(ax[i].var)] = acc;
    acc *= p.ext[ax[i].var];
  }
  for (int i = 0; i < ng; ++i) {
    CeGather G = g[i];
    G.pv = pvar[static_cast<std::size_t>(g[i].pv)];
    G.qv = pvar[static_cast<std::size_t>(g[i].qv)];
    pk.ga[pk.ng_a++] = G;
  }
  for (std::size_t i = 0; i < ax.size(); ++i) s[ax[i].var] = ns[static_cast<std::size_t>(ax[i].var)];
  ng = 0;
  *span = acc;
  return pk;
}

// Layout signature of a pack (a unary permute):(extent, input stride, output stride) of
// every axis with extent > 1, in input-stride order.  Two packs with equal signatures
// of the same buffer produce identical bytes.
std::vector<int64_t> pack_signature(const CeProblem& pk) {
  std::vector<std::array<int64_t, 3>> ax;
  for (int v = 0; v < pk.nv; ++v)
    if (pk.ext[v] > 1) ax.push_back({pk.sa[v], pk.ext[v], pk.sc[v]});
  std::sort(ax.begin(), ax.end());
  std::vector<int64_t> sig;
  for (const auto& a : ax) sig.insert(sig.end(), a.begin(), a.end());
  return sig;
}

// Family (c) tile / block permute kernels for large tensors; below CE_PERM_SMALL elements
// (default 2^20) the one-thread-per-output stream kernel (coalesced writes, gathered reads
// served by L2) finishes sooner than the tiled kernels' fixed cost.
bool use_permute(const CeProblem& pk) {
  static const double small = [] {
    const char* e = std::getenv("CE_PERM_SMALL");
    return e ? std::atof(e) : 1048576.0;
  }();
  double n = 1;
  for (int v = 0; v < pk.nv; ++v)
    if (pk.cls[v] != CE_K) n *= static_cast<double>(pk.ext[v]);
  return n >= small && ce_permute_supported(pk);
}

int inner_var(const CeProblem& p, bool side_b) {
  const int64_t* s = side_b ? p.sb : p.sa;
  for (int v = 0; v < p.nv; ++v)
    if (s[v] == 1 && p.ext[v] > 1) return v;
  return -1;
}

// An operand of `q` read from an existing repack of its buffer instead: every var (and
// gathered axis) stride is mapped through the pack's axes (atoms merged into one pack axis
// keep their relative strides).  False if a stride has no image.
bool remap_operand(CeProblem& q, bool side_b, const CeProblem& pk) {
  auto map = [&](int64_t st, int64_t ext, int64_t* out) {
    for (int k = 0; k < pk.nv; ++k) {
      const int64_t s0 = pk.sa[k];
      if (s0 <= 0 || st < s0 || st % s0 != 0 || (st / s0) * ext > pk.ext[k]) continue;
      *out = pk.sc[k] * (st / s0);
      return true;
    }
    return false;
  };
  int64_t* s = side_b ? q.sb : q.sa;
  CeGather* g = side_b ? q.gb : q.ga;
  const int ng = side_b ? q.ng_b : q.ng_a;
  for (int v = 0; v < q.nv; ++v)
    if (s[v] && q.ext[v] > 1 && !map(s[v], q.ext[v], &s[v])) return false;
  for (int i = 0; i < ng; ++i)
    if (!map(g[i].stride, g[i].extent, &g[i].stride)) return false;
  return true;
}

// Plain K vars shared by A and B, ordered by their stride in `side` (ascending).
std::vector<int> shared_k_order(const CeProblem& p, bool by_b) {
  std::vector<int> v;
  for (int i = 0; i < p.nv; ++i)
    if (p.cls[i] == CE_K && p.sa[i] && p.sb[i]) v.push_back(i);
  const int64_t* s = by_b ? p.sb : p.sa;
  std::stable_sort(v.begin(), v.end(), [&](int x, int y) { return s[x] < s[y]; });
  return v;
}
}  // namespace

void Executor::add_problem(std::vector<Step>& list, const CeProblem& p0, BufRef a, BufRef b, BufRef c, int node,
                           const std::string& label) {
  CeProblem p = p0;
  Step st;
  st.node = node;
  st.label = label;
  if (std::getenv("CE_DESCRIBE_PROBLEMS")) {  // diagnostics: the lowered problem of every step
    static const char* cn = "ZMNK";
    std::fprintf(stderr, "[%s] nv=%d unary=%d acc=%d\n", label.c_str(), p.nv, p.unary, p.accumulate);
    for (int v = 0; v < p.nv; ++v)
      std::fprintf(stderr, "  v%d %c ext=%lld sa=%lld sb=%lld sc=%lld\n", v, cn[p.cls[v]], (long long)p.ext[v],
                   (long long)p.sa[v], (long long)p.sb[v], (long long)p.sc[v]);
    for (int side = 0; side < 2; ++side)
      for (int g = 0; g < (side ? p.ng_b : p.ng_a); ++g) {
        const CeGather& G = side ? p.gb[g] : p.ga[g];
        std::fprintf(stderr, "  g%c%d pv=%d qv=%d sp=%d sq=%d c=%lld extent=%lld stride=%lld wrap=%d\n", side ? 'B' : 'A',
                     g, G.pv, G.qv, G.sp, G.sq, (long long)G.c, (long long)G.extent, (long long)G.stride, G.wrap);
      }
  }
  // Tiny contractions (K <= 8, e.g. ResNet conv1's 3 input channels) with a large output
  // are output-bandwidth problems: the streaming SIMT kernel writes them with float4
  // stores and no per-tile epilogue, where the TC path would pad K to 32 and pay a
  // ~5 us epilogue for every 128-row tile.
  // plane convolutions with few channels (RTR conv1's X * W4 and its adjoints, ce_pconv.cu):
  // staged-window SIMT kernels instead of a 49x tap expansion / col2im split.  CE_PCONV=0 off.
  static const bool pconv_on = [] {
    const char* e = std::getenv("CE_PCONV");
    return !(e && *e == '0');
  }();
  if (pconv_on && ce_pconv_plan(p, &st.pconv)) {
    st.kind = Step::kPconv;
    st.a = a;
    st.b = b;
    st.c = c;
    st.flops = pending_flops_;
    st.bytes = problem_bytes(p);
    if (st.pconv.kind == 1) {
      int64_t span = 0;
      for (int v = 0; v < p.nv; ++v)
        if (p.cls[v] != CE_K) span += (p.ext[v] - 1) * p.sc[v];
      st.zero_elems = span + 1;
    }
    list.push_back(st);
    return;
  }
  // row GEMMs with few columns over millions of rows (ce_rowgemm.cu): one thread per row.
  // CE_ROWGEMM=0 off.
  static const bool row_on = [] {
    const char* e = std::getenv("CE_ROWGEMM");
    return !(e && *e == '0');
  }();
  if (row_on && ce_rowgemm_plan(p, &st.row)) {
    st.kind = Step::kRow;
    st.a = a;
    st.b = b;
    st.c = c;
    st.flops = pending_flops_;
    st.bytes = problem_bytes(p);
    list.push_back(st);
    return;
  }
  const bool tiny_k = [&] {
    int64_t k = 1, outs = 1;
    for (int v = 0; v < p.nv; ++v) (p.cls[v] == CE_K ? k : outs) *= p.ext[v];
    for (int g = 0; g < p.ng_a; ++g) k *= 1;  // gathered taps are K vars already counted
    static const int64_t kmax = [] {  // CE_TINYK: K bound of this rule (experiment knob)
      const char* e = std::getenv("CE_TINYK");
      return e ? std::atoll(e) : 8;
    }();
    return k <= kmax && outs >= (1ll << 20);
  }();
  auto try_col2im = [&]() -> bool {
    static const bool col2im_on = [] {  // CE_COL2IM=0: no col2im split
      const char* e = std::getenv("CE_COL2IM");
      return !(e && *e == '0');
    }();
    for (int side = 0; side < 2 && col2im_on && !p.unary; ++side) {
      // col2im split of a convolution whose taps are contracted together with plain K vars
      // (RTR conv1's dX = sum_{r,i,j} dZ[b,c,h-i,w-j,r] F[r,i,j]: the SIMT K-lane kernel
      // re-walks all 441 terms per output):  T[b,c,u_h,u_w,i,j] = sum_r dZ[b,c,u_h,u_w,r] F[r,i,j]
      // on the tensor cores (u = the gathered feature index as a plain axis, taps outermost
      // in T), then C = sum_{i,j} T[b,c,h-i,w-j,i,j], a 49-term gather-sum.
      const int ng = side ? p.ng_b : p.ng_a;
      if (ng == 0 || ng > 2 || (side ? p.ng_a : p.ng_b)) continue;
      const CeGather* gs = side ? p.gb : p.ga;
      const int64_t* ss = side ? p.sb : p.sa;
      const int64_t* os = side ? p.sa : p.sb;
      bool fits = true;
      double taps = 1, plain_k = 1, t_elems = 1, g_elems = 1;
      for (int g = 0; g < ng; ++g) {
        const int pv = gs[g].pv, qv = gs[g].qv;
        // (p: an output position, q: a filter tap -- a gather whose "taps" outnumber its
        // positions is a filter gradient, which the stream kernel's dwgrad path handles)
        if (gs[g].wrap || p.cls[pv] == CE_K || ss[pv] || os[pv] || p.cls[qv] != CE_K || ss[qv] || !os[qv] ||
            p.ext[pv] < p.ext[qv])
          fits = false;
        for (int h = 0; h < ng; ++h)
          if (h != g && (gs[h].pv == pv || gs[h].qv == qv || gs[h].pv == qv || gs[h].qv == pv)) fits = false;
        taps *= static_cast<double>(p.ext[qv]);
        t_elems *= static_cast<double>(gs[g].extent) * static_cast<double>(p.ext[qv]);
        g_elems *= static_cast<double>(gs[g].extent);
      }
      if (!fits) continue;
      std::vector<char> is_p(static_cast<std::size_t>(p.nv), 0);
      for (int g = 0; g < ng; ++g) is_p[static_cast<std::size_t>(gs[g].pv)] = 1;
      for (int v = 0; v < p.nv; ++v) {
        if (p.cls[v] == CE_K && ss[v] && os[v]) plain_k *= static_cast<double>(p.ext[v]);
        if (p.cls[v] != CE_K && !is_p[static_cast<std::size_t>(v)]) t_elems *= static_cast<double>(p.ext[v]);
        if (ss[v]) g_elems *= static_cast<double>(p.ext[v]);
      }
      if (taps < 9 || plain_k < 2 || t_elems >= 2147483647.0 || t_elems > std::max(536870912.0, 8.0 * g_elems))
        continue;
      // step 1: gathers replaced by plain feature axes u; p vars vanish; taps become outputs
      CeProblem q1 = p;
      int64_t* s1 = side ? q1.sb : q1.sa;
      int uvar[2] = {-1, -1};
      for (int g = 0; g < ng; ++g) {
        if (q1.nv >= CE_MAX_VARS) fits = false;
        if (!fits) break;
        const int u = q1.nv++;
        uvar[g] = u;
        q1.ext[u] = gs[g].extent;
        q1.cls[u] = side ? CE_N : CE_M;
        q1.sa[u] = q1.sb[u] = q1.sc[u] = 0;
        s1[u] = gs[g].stride;
        const int pv = gs[g].pv, qv = gs[g].qv;
        q1.ext[pv] = 1;
        q1.sa[pv] = q1.sb[pv] = q1.sc[pv] = 0;
        q1.cls[qv] = side ? CE_M : CE_N;
      }
      if (!fits) continue;
      (side ? q1.ng_b : q1.ng_a) = 0;
      q1.accumulate = 0;
      // T layout: the gathered operand's non-K axes in its stride order (innermost first,
      // pitch padded to 16 B), then the partner's, then the taps outermost (so the gather-sum
      // reads T along the gathered operand's unit-stride axis)
      std::vector<int> lay;
      for (int pass = 0; pass < 3; ++pass) {
        std::vector<int> vs;
        for (int v = 0; v < q1.nv; ++v) {
          if (q1.ext[v] <= 1 || q1.cls[v] == CE_K) continue;
          bool tap = false;
          for (int g = 0; g < ng; ++g) tap |= v == gs[g].qv;
          const int64_t* s1o = side ? q1.sa : q1.sb;
          const bool mine = s1[v] != 0 && !tap, theirs = s1o[v] != 0 && !tap;
          if ((pass == 0 && mine) || (pass == 1 && theirs && !mine) || (pass == 2 && tap)) vs.push_back(v);
        }
        const int64_t* key = pass == 1 ? (side ? q1.sa : q1.sb) : s1;
        std::stable_sort(vs.begin(), vs.end(), [&](int x, int y) { return pass == 2 ? x < y : key[x] < key[y]; });
        lay.insert(lay.end(), vs.begin(), vs.end());
      }
      int64_t acc = 1;
      std::vector<int64_t> tstr(static_cast<std::size_t>(q1.nv), 0);
      for (std::size_t i = 0; i < lay.size(); ++i) {
        tstr[static_cast<std::size_t>(lay[i])] = acc;
        acc *= i == 0 ? (q1.ext[lay[i]] + 3) / 4 * 4 : q1.ext[lay[i]];
      }
      for (int v = 0; v < q1.nv; ++v) q1.sc[v] = q1.cls[v] == CE_K ? 0 : tstr[static_cast<std::size_t>(v)];
      // step 2: C[...] (+)= sum_taps T[..., u = sp*p + sq*q + c, ..., q]
      CeProblem q2 = p;
      q2.unary = 1;
      q2.ng_a = ng;
      q2.ng_b = 0;
      for (int v = 0; v < q2.nv; ++v) {
        q2.sb[v] = 0;
        bool tap = false;
        for (int g = 0; g < ng; ++g) tap |= v == gs[g].qv;
        if (p.cls[v] == CE_K && !tap) {
          q2.ext[v] = 1;  // contracted in step 1
          q2.sa[v] = q2.sc[v] = 0;
          continue;
        }
        q2.sa[v] = is_p[static_cast<std::size_t>(v)] ? 0 : tstr[static_cast<std::size_t>(v)];
      }
      for (int g = 0; g < ng; ++g) {
        q2.ga[g] = gs[g];
        q2.ga[g].stride = tstr[static_cast<std::size_t>(uvar[g])];
      }
      const BufRef tref{BufRef::kWork, alloc(acc)};
      add_problem(list, q1, a, b, tref, node, label + ":col2im-gemm");
      add_problem(list, q2, tref, BufRef{}, c, node, label + ":col2im-sum");
      return true;
    }
    return false;
  };
  if (tc_math() && !p.unary && !tiny_k) {
    {
      // an N = 1 convolution (input gradient over every factor index) is memory-bound on the
      // tensor cores with the taps as shifted boxes (each dZ element read once per tap):
      // the col2im split reads it once
      double n_ext = 1;
      for (int v = 0; v < p.nv; ++v)
        if (p.cls[v] == CE_N) n_ext *= static_cast<double>(p.ext[v]);
      if (n_ext == 1 && p.ng_a + p.ng_b > 0 && try_col2im()) return;
    }
    // Circular (wrap-around) gathers -- the reference's multi-way conv atoms, kernels.cpp:38-43,
    // 298-315 -- cannot be TMA boxes: the operand is first copied with its wrapped axes
    // unrolled (E[i] = A[(i + lo) mod X] over the whole index range the step reads), after
    // which the step is an ordinary shifted-box convolution.  CE_TC_UNWRAP=0: SIMT instead.
    static const bool unwrap_on = [] {
      const char* e = std::getenv("CE_TC_UNWRAP");
      return !(e && *e == '0');
    }();
    for (int side = 0; side < 2 && unwrap_on; ++side) {
      const int ng = side ? p.ng_b : p.ng_a;
      CeGather* gs = side ? p.gb : p.ga;
      bool wraps = false;
      for (int g = 0; g < ng; ++g) wraps |= gs[g].wrap != 0;
      if (!wraps || p.nv + ng + 1 > CE_MAX_VARS) continue;
      int64_t* ss = side ? p.sb : p.sa;
      struct Ax { int64_t stride, ext; int var, g; };
      std::vector<Ax> ax;
      for (int v = 0; v < p.nv; ++v)
        if (ss[v]) ax.push_back({ss[v], p.ext[v], v, -1});
      std::vector<int64_t> lo(static_cast<std::size_t>(ng), 0), ext_g(static_cast<std::size_t>(ng), 0);
      for (int g = 0; g < ng; ++g) {
        const CeGather& G = gs[g];
        const int64_t P = p.ext[G.pv] - 1, Q = p.ext[G.qv] - 1;
        const int64_t l = G.c + std::min<int64_t>(0, G.sp * P) + std::min<int64_t>(0, G.sq * Q);
        const int64_t h = G.c + std::max<int64_t>(0, G.sp * P) + std::max<int64_t>(0, G.sq * Q);
        lo[static_cast<std::size_t>(g)] = G.wrap ? l : 0;
        ext_g[static_cast<std::size_t>(g)] = G.wrap ? h - l + 1 : G.extent;
        ax.push_back({G.stride, ext_g[static_cast<std::size_t>(g)], -1, g});
      }
      std::stable_sort(ax.begin(), ax.end(), [](const Ax& x, const Ax& y) { return x.stride < y.stride; });
      CeProblem pk{};
      pk.unary = 1;
      const int dummy = pk.nv++;  // the copy's (extent-1) K var every gather pairs with
      pk.ext[dummy] = 1;
      pk.cls[dummy] = CE_K;
      int64_t acc = 1;
      for (std::size_t i = 0; i < ax.size(); ++i) {
        if (i == 1) acc = (acc + 3) / 4 * 4;  // 16-B rows (TMA stride legality)
        const int v = pk.nv++;
        pk.ext[v] = ax[i].ext;
        pk.cls[v] = CE_M;
        pk.sc[v] = acc;
        if (ax[i].var >= 0) {
          pk.sa[v] = ax[i].stride;
          ss[ax[i].var] = acc;
        } else {
          CeGather& G = gs[ax[i].g];
          CeGather E{};
          E.pv = v;
          E.qv = dummy;
          E.sp = 1;
          E.sq = 0;
          E.c = lo[static_cast<std::size_t>(ax[i].g)];
          E.extent = G.extent;
          E.stride = G.stride;
          E.wrap = G.wrap;
          pk.ga[pk.ng_a++] = E;
          if (G.wrap) {
            G.c -= E.c;
            G.extent = ax[i].ext;
            G.wrap = 0;
          }
          G.stride = acc;
        }
        acc *= ax[i].ext;
      }
      Step es;
      es.kind = Step::kDirect;
      es.desc = simt_desc(pk);
      es.a = side ? b : a;
      es.c = {BufRef::kWork, alloc(acc)};
      es.node = node;
      es.label = label + (side ? ":unwrapB" : ":unwrapA");
      es.bytes = 4.0 * static_cast<double>(acc) + 4.0 * operand_elems(pk, 0);
      (side ? b : a) = es.c;
      list.push_back(es);
    }
    bool ok = ce_tc_plan(p, &st.tc);
    // A legal plan whose K units are fragmented (both operands K-major but their K vars
    // chain differently, e.g. a hoisted [.. r0 s1] intermediate against a factor stored
    // [r0 r1 t1 s1]: 10 K units of 4 padded to 32) is scored against the repacks below.
    double k_elems = 1;
    for (int v = 0; v < p.nv; ++v)
      if (p.cls[v] == CE_K) k_elems *= static_cast<double>(p.ext[v]);
    const bool k_waste = ok && static_cast<double>(st.tc.params.k_iters) * 32.0 > 2.0 * k_elems + 64.0;
    if (!ok || k_waste) {
      // tf32 tensor cores need both operands K-major over the same K unit: repack
      // the operand(s) whose unit-stride axis is not a shared K var, mirroring the
      // partner's K order so contiguous K vars still merge into one unit.
      const int ia = inner_var(p, false), ib = inner_var(p, true);
      const bool a_ok = ia >= 0 && p.cls[ia] == CE_K && p.sb[ia];
      const bool b_ok = ib >= 0 && p.cls[ib] == CE_K && p.sa[ib];
      struct Attempt {
        bool pack_a, pack_b;
        std::vector<int> order;
      };
      std::vector<Attempt> attempts;
      if (a_ok && (k_waste || !(b_ok && ib == ia))) attempts.push_back({false, true, shared_k_order(p, false)});
      if (b_ok && (k_waste || !a_ok)) attempts.push_back({true, false, shared_k_order(p, true)});
      {
        // both operands repacked with one K order (contiguous, so the K vars merge)
        std::vector<int> order = shared_k_order(p, a_ok ? false : true);
        const std::vector<int> all = order;
        if (!a_ok && !b_ok) {
          std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p.ext[x] > p.ext[y]; });
          if (!order.empty()) order.resize(1);
        }
        attempts.push_back({true, true, order});
        // or every shared K var innermost in both (one merged K unit: RTR 64->64's X * W over
        // s1 s2 s3 = 64 instead of a 4-wide unit padded to 32; scored after, so ties keep the
        // single-var layout)
        if (!a_ok && !b_ok && all.size() > 1) attempts.push_back({true, true, all});
      }
      // every layout that the tensor cores accept is scored (stages at ~0.25 us per SM plus
      // pack traffic at ~3 TB/s; a pack the forward pass already made is free): the first
      // legal layout can leave a 4-wide K unit padded to 32 where packing both operands
      // merges the K vars into one 40-wide unit (RTR)
      static const bool first_legal = [] {
        const char* e = std::getenv("CE_PACK_FIRST");
        return e && *e == '1';
      }();
      auto reusable = [&](BufRef src, const CeProblem& pk) -> const PackRecord* {
        for (const PackRecord& r : packs_)
          if (r.src.kind == src.kind && r.src.index == src.index && pack_signature(r.pk) == pack_signature(pk))
            return &r;
        return nullptr;
      };
      double best_us = 1e300;
      int best = -1;
      if (k_waste) {  // the legal plan as it is
        const TcParams& P = st.tc.params;
        best_us = static_cast<double>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_iters * 0.25 / 148.0;
      }
      CeProblem best_q{}, best_pks[2];
      int64_t best_spans[2] = {0, 0};
      TcPlan best_t;
      for (std::size_t ai = 0; ai < attempts.size(); ++ai) {
        const Attempt& at = attempts[ai];
        if (at.order.empty() || (first_legal && best >= 0)) continue;
        CeProblem q = p;
        CeProblem pks[2];
        int64_t spans[2] = {0, 0};
        if (at.pack_a) pks[0] = repack(q, false, at.order, &spans[0], at.pack_b ? nullptr : p.sb);
        if (at.pack_b) pks[1] = repack(q, true, at.order, &spans[1], at.pack_a ? nullptr : p.sa);
        TcPlan t;
        if (!ce_tc_plan(q, &t)) continue;
        const TcParams& P = t.params;
        double us = static_cast<double>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_iters * 0.25 / 148.0;
        for (int side = 0; side < 2; ++side)
          if ((side ? at.pack_b : at.pack_a) && !reusable(side ? b : a, pks[side]))
            us += 8.0 * operand_elems(pks[side], 0) / 3.0e6;
        if (us < best_us) {
          best_us = us;
          best = static_cast<int>(ai);
          best_q = q;
          best_pks[0] = pks[0];
          best_pks[1] = pks[1];
          best_spans[0] = spans[0];
          best_spans[1] = spans[1];
          best_t = t;
        }
      }
      // or read one operand from a repack of its buffer an earlier step already made (free;
      // e.g. RTR 64->128's dW1 reads N0 and dN1 in the layouts node1 and dN0's step packed
      // them into), the other as it is or repacked to match.  CE_PACK_REUSE=0 off.
      static const bool reuse_on = [] {
        const char* e = std::getenv("CE_PACK_REUSE");
        return !(e && *e == '0');
      }();
      int reuse_side = -1;
      const PackRecord* reuse_rec = nullptr;
      const PackRecord* reuse_rec2 = nullptr;  // the other operand's reused repack (both reused)
      bool reuse_pack_other = false;
      CeProblem reuse_pk{};
      int64_t reuse_span = 0;
      for (int side = 0; side < 2 && reuse_on && !first_legal; ++side) {
        const BufRef src = side ? b : a;
        for (const PackRecord& r : packs_) {
          if (r.src.kind != src.kind || r.src.index != src.index) continue;
          // (repacks of >= 16 MB: smaller ones are cheap to redo)
          static const double min_elems = [] {  // CE_PACK_REUSE_MIN_MB (default 16)
            const char* e = std::getenv("CE_PACK_REUSE_MIN_MB");
            return (e ? std::atof(e) : 16.0) * 1024.0 * 1024.0 / 4.0;
          }();
          if (operand_elems(r.pk, 0) < min_elems) continue;
          CeProblem q = p;
          if (!remap_operand(q, side == 1, r.pk)) continue;
          for (int other = 0; other < 3; ++other) {
            CeProblem q2 = q;
            CeProblem pk2{};
            int64_t span2 = 0;
            const PackRecord* r2 = nullptr;
            if (other == 2) {  // the other operand from an existing repack too
              const BufRef osrc = side ? a : b;
              for (const PackRecord& x : packs_)
                if (x.src.kind == osrc.kind && x.src.index == osrc.index && operand_elems(x.pk, 0) >= min_elems) {
                  CeProblem q3 = q;
                  if (remap_operand(q3, side == 0, x.pk)) {
                    q2 = q3;
                    r2 = &x;
                    break;
                  }
                }
              if (!r2) continue;
            } else if (other) {
              std::vector<int> order = shared_k_order(q, side == 1);
              if (order.empty()) continue;
              pk2 = repack(q2, side == 0, order, &span2, side ? q.sb : q.sa);
            }
            TcPlan t;
            if (!ce_tc_plan(q2, &t)) continue;
            const TcParams& P = t.params;
            double us = static_cast<double>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_iters * 0.25 / 148.0;
            if (other == 1 && !reusable(side ? a : b, pk2)) us += 8.0 * operand_elems(pk2, 0) / 3.0e6;
            // MN-major operands read natively cost more per stage than the model's K-major rate
            // (x4: without it RTR 64->64's input gradient took a reused b-innermost dY and
            // went 1.9 -> 2.9 ms; with it cfg2 0.960 -> 0.949 ms, cfg3 69.0 -> 67.9 ms)
            static const double mn_pen = [] {  // CE_PACK_REUSE_MNPEN (default 4)
              const char* e = std::getenv("CE_PACK_REUSE_MNPEN");
              return e ? std::atof(e) : 4.0;
            }();
            // (split-K reductions -- filter gradients: few outputs, huge K -- stream the MN-major
            // rows at full rate; tile-parallel steps such as a conv's input gradient do not)
            if (P.k_split == 1 && P.oa.mn_major) us *= mn_pen;
            if (P.k_split == 1 && P.ob.mn_major) us *= mn_pen;
            if (us < best_us) {
              best_us = us;
              best = -1;
              reuse_side = side;
              reuse_rec = &r;
              reuse_rec2 = r2;
              reuse_pack_other = other == 1;
              reuse_pk = pk2;
              reuse_span = span2;
              best_q = q2;
              best_t = t;
            }
          }
        }
      }
      if (reuse_side >= 0) {
        (reuse_side ? b : a) = reuse_rec->dst;
        if (reuse_rec2) (reuse_side ? a : b) = reuse_rec2->dst;
        if (reuse_pack_other) {
          const int side = 1 - reuse_side;
          const BufRef src = side ? b : a;
          if (const PackRecord* r = reusable(src, reuse_pk)) {
            (side ? b : a) = r->dst;
          } else {
            Step ps;
            ps.kind = use_permute(reuse_pk) ? Step::kPermute : Step::kDirect;
            ps.desc = simt_desc(reuse_pk);
            ps.a = src;
            ps.c = {BufRef::kWork, alloc(reuse_span)};
            ps.node = node;
            ps.label = label + (side ? ":packB" : ":packA");
            ps.bytes = 8.0 * operand_elems(reuse_pk, 0);
            (side ? b : a) = ps.c;
            packs_.push_back({src, reuse_pk, ps.c});
            pack_log_.push_back({src, reuse_pk, &list == &fwd_});
            list.push_back(ps);
          }
        }
        p = best_q;
        st.tc = best_t;
        ok = true;
      }
      if (best >= 0) {
        const Attempt& at = attempts[static_cast<std::size_t>(best)];
        for (int side = 0; side < 2; ++side) {
          if (!(side ? at.pack_b : at.pack_a)) continue;
          // an identical repack of the same buffer done by the forward pass is reused
          // (forward always runs before backward on the same inputs)
          const BufRef src = side ? b : a;
          if (const PackRecord* r = reusable(src, best_pks[side])) {
            (side ? b : a) = r->dst;
            continue;
          }
          Step ps;
          ps.kind = use_permute(best_pks[side]) ? Step::kPermute : Step::kDirect;
          ps.desc = simt_desc(best_pks[side]);
          ps.a = src;
          ps.c = {BufRef::kWork, alloc(best_spans[side])};
          ps.node = node;
          ps.label = label + (side ? ":packB" : ":packA");
          ps.bytes = 8.0 * operand_elems(best_pks[side], 0);
          (side ? b : a) = ps.c;
          packs_.push_back({src, best_pks[side], ps.c});
          pack_log_.push_back({src, best_pks[side], &list == &fwd_});
          list.push_back(ps);
        }
        p = best_q;
        st.tc = best_t;
        ok = true;
      }
    }
    static const bool expand_on = [] {  // CE_EXPAND=0: no tap expansion
      const char* e = std::getenv("CE_EXPAND");
      return !(e && *e == '0');
    }();
    for (int side = 0; side < 2 && !ok && expand_on; ++side) {
      // the operand's unit-stride axis is a convolution gather: expand its taps
      const int ngs = side ? p.ng_b : p.ng_a;
      const CeGather* gs = side ? p.gb : p.ga;
      const int64_t* ss = side ? p.sb : p.sa;
      const int64_t* ps = side ? p.sa : p.sb;
      bool inner_gather = false;
      for (int i = 0; i < ngs; ++i) inner_gather |= gs[i].stride == 1;
      if (!inner_gather || inner_var(p, side == 1) >= 0) continue;
      std::vector<int> in_op(static_cast<std::size_t>(p.nv), 0);
      double e_elems = 1, outs = 1, partner = 1;
      for (int v = 0; v < p.nv; ++v) {
        bool g = false;
        for (int i = 0; i < ngs; ++i) g |= gs[i].pv == v || gs[i].qv == v;
        in_op[static_cast<std::size_t>(v)] = ss[v] != 0 || g;
        if (in_op[static_cast<std::size_t>(v)]) e_elems *= static_cast<double>(p.ext[v]);
        if (p.cls[v] != CE_K) outs *= static_cast<double>(p.ext[v]);
        if (ps[v]) partner *= static_cast<double>(p.ext[v]);
      }
      if (e_elems >= 2147483647.0 || (e_elems > 2.0 * std::max(outs, partner) && e_elems > 536870912.0)) continue;
      // E's innermost axes: the K vars it shares with the partner, in the partner's order
      std::vector<int> korder;
      for (int v = 0; v < p.nv; ++v)
        if (p.cls[v] == CE_K && ps[v] && in_op[static_cast<std::size_t>(v)]) korder.push_back(v);
      std::stable_sort(korder.begin(), korder.end(), [&](int x, int y) { return ps[x] < ps[y]; });
      for (const auto& order : {korder, std::vector<int>{}}) {
        if (ok) break;
        for (int pack_partner = 0; pack_partner < 2 && !ok; ++pack_partner) {
          if (pack_partner && order.empty()) continue;
          CeProblem q = p;
          int64_t span = 0, pspan = 0;
          const CeProblem pk = expand(q, side == 1, order, &span);
          CeProblem ppk{};
          // (output vars in C order: the expanded step's tile columns then match C, e.g. RTR
          // X*F writing 10x10 rank pairs as contiguous 100-float rows)
          if (pack_partner) ppk = repack(q, side == 0, order, &pspan, nullptr, true);
          TcPlan t;
          if (!ce_tc_plan(q, &t)) continue;
          Step es;
          es.kind = Step::kDirect;
          es.desc = simt_desc(pk);
          es.a = side ? b : a;
          es.c = {BufRef::kWork, alloc(span)};
          es.node = node;
          es.label = label + (side ? ":expandB" : ":expandA");
          es.bytes = 4.0 * static_cast<double>(span) + 4.0 * operand_elems(pk, 0);
          (side ? b : a) = es.c;
          list.push_back(es);
          if (pack_partner) {
            Step ps2;
            ps2.kind = use_permute(ppk) ? Step::kPermute : Step::kDirect;
            ps2.desc = simt_desc(ppk);
            ps2.a = side ? a : b;
            ps2.c = {BufRef::kWork, alloc(pspan)};
            ps2.node = node;
            ps2.label = label + (side ? ":packA" : ":packB");
            ps2.bytes = 8.0 * operand_elems(ppk, 0);
            (side ? a : b) = ps2.c;
            pack_log_.push_back({ps2.a, ppk, &list == &fwd_});
            list.push_back(ps2);
          }
          p = q;
          st.tc = t;
          ok = true;
        }
      }
    }
    if (!ok && try_col2im()) return;
    // CE_MN_REPACK: 2 (default) only the double-MN-major rule, 1 both long-K repack rules below,
    // 0 none.  Native MN-major operands are read by the MMA directly, so the single-MN-major
    // repack no longer pays: cfg2 step 1.186 -> 1.133 ms with 2 (same-box A/B x3, round 2)
    static const int mn_repack = [] {
      const char* e = std::getenv("CE_MN_REPACK");
      return e ? std::atoi(e) : 2;
    }();
    if (ok && mn_repack >= 1 && st.tc.params.oa.mn_major && st.tc.params.ob.mn_major && st.tc.params.k_iters > 64) {
      // Both operands would be transposed in shared memory every stage: over a long K
      // loop that is smem-bandwidth bound (measured 2.2x slower than the MMA).  Repack B
      // once with its largest shared K var innermost so only A is transposed in-kernel.
      std::vector<int> order = shared_k_order(p, false);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p.ext[x] > p.ext[y]; });
      if (!order.empty() && p.ext[order[0]] >= 32) {
        order.resize(1);
        CeProblem q = p;
        int64_t span = 0;
        CeProblem pk = repack(q, true, order, &span, nullptr);
        TcPlan t;
        if (ce_tc_plan(q, &t) && !t.params.ob.mn_major) {
          Step ps;
          ps.kind = use_permute(pk) ? Step::kPermute : Step::kDirect;
          ps.desc = simt_desc(pk);
          ps.a = b;
          ps.c = {BufRef::kWork, alloc(span)};
          ps.node = node;
          ps.label = label + ":packB";
          ps.bytes = 8.0 * operand_elems(pk, 0);
          b = ps.c;
          pack_log_.push_back({ps.a, pk, &list == &fwd_});
          list.push_back(ps);
          p = q;
          st.tc = t;
        }
      }
    }
    static const int repack_mn = [] {  // experiment knob: 1 = repack every MN-major operand
      const char* e = std::getenv("CE_REPACK_MN");
      return e ? std::atoi(e) : 0;
    }();
    if (ok && (st.tc.params.oa.mn_major || st.tc.params.ob.mn_major) &&
        ((st.tc.params.k_iters > 64 && mn_repack == 1) || repack_mn == 1)) {
      // One MN-major operand over a long K loop (factor gradients: K = every b,h,w): its
      // 4 KB [32 K][32 MN] boxes plus the in-smem transpose make the TMA producer, not the
      // MMA, the bottleneck (measured 1.4 us per stage against 0.39 us K-major).  A single
      // repack to the partner's K unit costs one HBM round trip of that operand.
      const bool side_b = !st.tc.params.oa.mn_major;
      const int partner_inner = inner_var(p, !side_b);
      std::vector<int> order;
      int64_t kin = 0;  // K extent that becomes contiguous (one K unit) after the repack
      if (partner_inner >= 0 && p.cls[partner_inner] == CE_K) {
        // the partner's shared K vars in its stride order: the chained prefix merges into
        // one K unit in both operands
        order = shared_k_order(p, !side_b);
        const int64_t* ps = side_b ? p.sa : p.sb;
        kin = 1;
        for (std::size_t i = 0; i < order.size(); ++i) {
          if (i > 0 && ps[order[i]] != ps[order[i - 1]] * p.ext[order[i - 1]]) break;
          kin *= p.ext[order[i]];
        }
      } else {
        order = shared_k_order(p, side_b);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return p.ext[x] > p.ext[y]; });
        if (!order.empty()) order.resize(1);
        kin = order.empty() ? 0 : p.ext[order[0]];
      }
      if (!order.empty() && kin >= 32) {
        CeProblem q = p;
        int64_t span = 0;
        CeProblem pk = repack(q, side_b, order, &span, side_b ? p.sa : p.sb);
        TcPlan t;
        if (ce_tc_plan(q, &t) && !t.params.oa.mn_major && !t.params.ob.mn_major) {
          const BufRef src = side_b ? b : a;
          bool reused = false;
          for (const PackRecord& r : packs_) {  // the forward pass may have packed it already
            if (r.src.kind != src.kind || r.src.index != src.index) continue;
            if (pack_signature(r.pk) == pack_signature(pk)) {
              (side_b ? b : a) = r.dst;
              reused = true;
              break;
            }
          }
          if (!reused) {
            Step ps;
            ps.kind = use_permute(pk) ? Step::kPermute : Step::kDirect;
            ps.desc = simt_desc(pk);
            ps.a = src;
            ps.c = {BufRef::kWork, alloc(span)};
            ps.node = node;
            ps.label = label + (side_b ? ":packB" : ":packA");
            ps.bytes = 8.0 * operand_elems(pk, 0);
            (side_b ? b : a) = ps.c;
            packs_.push_back({src, pk, ps.c});
            pack_log_.push_back({src, pk, &list == &fwd_});
            list.push_back(ps);
          }
          p = q;
          st.tc = t;
        }
      }
    }
    // Split-K steps whose output layout admits neither vectorised nor TMA reductions (a filter
    // gradient whose unit-stride axis is a tap, e.g. dW[r1][r2][h][w] with the taps as grid
    // units) would add every partial tile with scalar atomics.  When the output is small they
    // reduce instead into a staging buffer laid out [M vars][N vars][rest] (M innermost, in
    // A's order, so the tile rows chain and bulk reduce-adds take them) that one permute then
    // writes in the caller's layout.  CE_TC_STAGE_SPLITK=0 off.
    static const bool stage_on = [] {
      const char* e = std::getenv("CE_TC_STAGE_SPLITK");
      return !(e && *e == '0');
    }();
    if (ok && stage_on && cfg_.math == 0 && st.tc.params.k_split > 1 && st.tc.params.c_tma == 0) {
      double out_elems = 1;
      for (int v = 0; v < p.nv; ++v)
        if (p.cls[v] != CE_K) out_elems *= static_cast<double>(p.ext[v]);
      if (out_elems <= 16.0 * 1048576.0) {
        CeProblem q = p;
        std::vector<int> vs;
        for (int cls : {CE_M, CE_N, CE_Z}) {
          std::vector<int> part;
          for (int v = 0; v < p.nv; ++v)
            if (p.cls[v] == cls && p.ext[v] > 1) part.push_back(v);
          // (vars plain in the operand first, by its strides: they form the tile units; vars
          // only reached through a gather -- the filter taps -- outermost)
          const int64_t* op = cls == CE_N ? p.sb : p.sa;
          auto key = [&](int v) { return op[v] ? op[v] : INT64_MAX; };
          std::stable_sort(part.begin(), part.end(), [&](int x, int y) { return key(x) < key(y); });
          vs.insert(vs.end(), part.begin(), part.end());
        }
        int64_t acc = 1;
        for (std::size_t i = 0; i < vs.size(); ++i) {
          if (i == 1) acc = (acc + 3) / 4 * 4;
          q.sc[vs[i]] = acc;
          acc *= p.ext[vs[i]];
        }
        for (int v = 0; v < q.nv; ++v)
          if (q.cls[v] != CE_K && q.ext[v] == 1) q.sc[v] = 0;
        TcPlan t;
        if (ce_tc_plan(q, &t) && t.params.c_tma != 0 && t.params.k_split > 1) {
          const BufRef tmp{BufRef::kWork, alloc(acc)};
          Step ts = st;
          ts.kind = Step::kTc;
          ts.tc = t;
          ts.a = a;
          ts.b = b;
          ts.c = tmp;
          ts.desc = simt_desc(q);
          ts.flops = pending_flops_;
          ts.bytes = problem_bytes(q);
          push_tc(list, ts);
          // staging -> the caller's layout (a unary permute over the output vars)
          CeProblem pk{};
          pk.unary = 1;
          for (int v = 0; v < p.nv; ++v) {
            if (p.cls[v] == CE_K || p.ext[v] == 1) continue;
            const int u = pk.nv++;
            pk.ext[u] = p.ext[v];
            pk.cls[u] = CE_M;
            pk.sa[u] = q.sc[v];
            pk.sc[u] = p.sc[v];
          }
          Step ps;
          ps.kind = use_permute(pk) ? Step::kPermute : Step::kDirect;
          ps.desc = simt_desc(pk);
          ps.a = tmp;
          ps.c = c;
          ps.node = node;
          ps.label = label + ":unstage";
          ps.bytes = 8.0 * out_elems;
          list.push_back(ps);
          return;
        }
      }
    }
    if (ok) {
      st.kind = Step::kTc;
      st.a = a;
      st.b = b;
      st.c = c;
      st.desc = simt_desc(p);
      st.flops = pending_flops_;
      st.bytes = problem_bytes(p);
      if (cfg_.math == 2) {
        // 3xTF32: both operands split into TF32-exact hi and FP32 remainder lo (same layouts), then
        // C = hi*hi + hi*lo + lo*hi -- the dropped lo*lo term is ~2^-22 relative (FP32-level)
        auto span = [&](bool side_b) {
          const int64_t* ss = side_b ? p.sb : p.sa;
          const CeGather* g = side_b ? p.gb : p.ga;
          const int ng = side_b ? p.ng_b : p.ng_a;
          int64_t n = 1;
          for (int v = 0; v < p.nv; ++v)
            if (ss[v]) n += (p.ext[v] - 1) * ss[v];
          for (int i = 0; i < ng; ++i) n += (g[i].extent - 1) * g[i].stride;
          return n;
        };
        BufRef hi[2], lo[2];
        for (int side = 0; side < 2; ++side) {
          const int64_t n = span(side == 1);
          Step sp;
          sp.kind = Step::kSplit;
          sp.a = side ? b : a;
          sp.c = hi[side] = {BufRef::kWork, alloc(n)};
          sp.c2 = lo[side] = {BufRef::kWork, alloc(n)};
          sp.zero_elems = n;
          sp.node = node;
          sp.label = label + (side ? ":splitB" : ":splitA");
          sp.bytes = 12.0 * static_cast<double>(n);
          list.push_back(sp);
        }
        const BufRef pa[3] = {hi[0], hi[0], lo[0]}, pb[3] = {hi[1], lo[1], hi[1]};
        for (int t = 0; t < 3; ++t) {
          Step s3 = st;
          s3.a = pa[t];
          s3.b = pb[t];
          s3.tc.accum = t > 0 ? 1 : 0;
          if (t > 0) {
            s3.flops = 0;  // (the algorithmic FLOPs are credited once)
            s3.label = label + (t == 1 ? ":3xtf32-hl" : ":3xtf32-lh");
          }
          list.push_back(s3);
        }
        return;
      }
      push_tc(list, st);
      return;
    }
  }
  st.a = a;
  st.b = b;
  st.c = c;
  st.desc = simt_desc(p);
  st.flops = pending_flops_;
  st.bytes = problem_bytes(p);
  const CeSimtDesc& d = st.desc;
  const int64_t outs = d.Z * d.M * d.N;
  if (p.unary && use_permute(p)) {
    st.kind = Step::kPermute;
  } else if (d.K >= 1024 && outs < 148 * 256 && (p.unary || d.K <= 32 || d.M < 16 || d.N < 16 || outs < 4096)) {
    st.kind = Step::kReduce;
    int64_t span = 0;
    for (int v = 0; v < p.nv; ++v)
      if (p.cls[v] != CE_K) span += (p.ext[v] - 1) * p.sc[v];
    st.zero_elems = span + 1;
  } else if (p.unary || d.K <= 32 || d.M < 16 || d.N < 16) {
    st.kind = Step::kDirect;
  } else {
    st.kind = Step::kTiled;
    auto min_stride = [&](const int32_t* vars, int n, const int64_t* s) {
      int64_t m = INT64_MAX;
      for (int i = 0; i < n; ++i)
        if (s[vars[i]]) m = std::min(m, s[vars[i]]);
      return m;
    };
    st.a_kfast = min_stride(d.kv, d.nk, p.sa) < min_stride(d.mv, d.nm, p.sa);
    st.b_kfast = min_stride(d.kv, d.nk, p.sb) < min_stride(d.nvv, d.nn, p.sb);
  }
  list.push_back(st);
}

// Node fusion along plan chains: a depthwise stencil step whose output is
// the A operand of a later depthwise stencil step (CP's `bhwr,rh->bhwr` -> `bhwr,rw->bhwr`,
// layers.cpp:184-190, and the two input-gradient adjoints of that pair in the backward pass)
// becomes one fused step (ce_fuse.cu).  The intermediate is still stored when any other step
// of either pass reads it (the forward's Y1 feeds the backward's filter gradient).
void Executor::fuse_chains(std::vector<Step>& list) {
  auto refs_elsewhere = [&](const BufRef& r, const Step* x, const Step* y) {
    for (const auto* l : {&fwd_, &bwd_})
      for (const Step& st : *l) {
        if (&st == x || &st == y) continue;
        for (const BufRef* q : {&st.a, &st.b, &st.c, &st.b2, &st.c2})
          if (q->kind == r.kind && q->index == r.index) return true;
      }
    return false;
  };
  auto same = [](const BufRef& x, const BufRef& y) { return x.kind != BufRef::kNone && x.kind == y.kind && x.index == y.index; };
  for (std::size_t i = 0; i < list.size(); ++i) {
    Step& si = list[i];
    if (si.kind != Step::kDirect || si.a.kind != BufRef::kWork || si.c.kind != BufRef::kWork) continue;
    for (std::size_t j = i + 1; j < list.size(); ++j) {
      Step& sj = list[j];
      if (sj.kind != Step::kDirect || !same(sj.a, si.c) || sj.c.kind != BufRef::kWork) continue;
      // moving sj up to i's slot: nothing in between may touch its output, write its filter,
      // or write what si reads / produces
      bool ok = true;
      for (std::size_t k = i + 1; k < j && ok; ++k) {
        const Step& sk = list[k];
        for (const BufRef* w : {&sk.c, &sk.c2})
          ok = ok && !same(*w, sj.c) && !same(*w, sj.b) && !same(*w, si.c) && !same(*w, si.a) && !same(*w, si.b);
        for (const BufRef* r : {&sk.a, &sk.b, &sk.b2}) ok = ok && !same(*r, sj.c);
      }
      if (!ok) break;
      const bool write_mid = refs_elsewhere(si.c, &si, &sj);
      // When the intermediate must be stored anyway (training: the backward's filter gradient
      // reads it) fusion saves only its re-read, and the two stencil launches stream at
      // ~4.8 TB/s against ~3 TB/s for the fused tile kernel: fuse those pairs only while the
      // intermediate is small enough for the saved launch to dominate (CP cr 0.1 layers:
      // conv1 1.23 -> 1.15 ms; R = 275 @56: 376 -> 432 us, not fused).  CE_FUSE_MAX_MB: 96 ->
      // 256 at the end of round 2 (cfg4 cr 1.0 stack 36.20 -> 35.62 ms: the 128 @28 and 256 @14
      // layers fuse; cfg2 / cfg3 / cfg4 cr 0.1 unchanged, same-box A/B x2).
      static const double max_mb = [] {
        const char* e = std::getenv("CE_FUSE_MAX_MB");
        return e ? std::atof(e) : 256.0;
      }();
      if (write_mid && 4.0 * operand_elems(si.desc.p, 2) > max_mb * 1048576.0) break;
      CeDw2Desc d{};
      if (!ce_dw2_plan(si.desc.p, sj.desc.p, write_mid, &d)) break;
      Step f = si;
      f.kind = Step::kDw2;
      f.dw2 = d;
      f.b2 = sj.b;
      f.c2 = sj.c;
      if (!write_mid) f.c = BufRef{};
      f.flops = si.flops + sj.flops;
      f.bytes = problem_bytes(sj.desc.p) - 4.0 * operand_elems(sj.desc.p, 0) + 4.0 * operand_elems(si.desc.p, 0) +
                (write_mid ? 4.0 * operand_elems(si.desc.p, 2) : 0.0);
      f.label = si.label + "+" + sj.label;
      list[i] = f;
      list.erase(list.begin() + static_cast<std::ptrdiff_t>(j));
      break;
    }
  }
}

// Gradient checkpointing: the backward pass starts by re-running every
// forward step that writes workspace (the node results and repacks its steps read; the root
// node writes the caller's output and is skipped) into fresh buffers, and every backward
// reference to a forward-written buffer is redirected to its recomputed twin.  The forward
// pass's buffers then die with the forward pass (assign_offsets shares their memory with the
// backward's), and backward() no longer depends on a preceding forward().
void Executor::add_recompute() {
  std::map<int64_t, int64_t> twin;  // forward-written workspace buffer id -> backward copy
  for (const Step& st : fwd_)
    for (const BufRef* w : {&st.c, &st.c2})
      if (w->kind == BufRef::kWork && !twin.count(w->index)) {
        twin[w->index] = static_cast<int64_t>(buf_bytes_.size());
        buf_bytes_.push_back(buf_bytes_[static_cast<std::size_t>(w->index)]);
      }
  auto remap = [&](Step& st) {
    for (BufRef* r : {&st.a, &st.b, &st.c, &st.b2, &st.c2})
      if (r->kind == BufRef::kWork && twin.count(r->index)) r->index = twin[r->index];
  };
  std::vector<Step> pre;
  for (const Step& st : fwd_) {
    if (st.c.kind != BufRef::kWork && st.c2.kind != BufRef::kWork) continue;
    Step r = st;
    r.node = -1;  // always runs (node ids of backward steps index operand gradients)
    r.label = "recompute:" + st.label;
    r.ev0 = r.ev1 = r.done = nullptr;
    remap(r);
    pre.push_back(r);
  }
  for (Step& st : bwd_) remap(st);
  bwd_.insert(bwd_.begin(), pre.begin(), pre.end());
}

// Repacks of caller buffers (factors, X, dY: ready when the pass starts) are issued at the
// start of the pass instead of right before their consumer, so they run on side streams
// while earlier steps compute (the list order is the issue order, see run_concurrent).
// Opt-in (CE_EARLY_PACKS=1): neutral on the graph-replayed cfg2 step (0.989 vs 0.991 ms,
// same-box A/B x3) -- the packs already overlap the kernel before their consumer.
void Executor::early_packs(std::vector<Step>& list) {
  static const bool on = [] {
    const char* e = std::getenv("CE_EARLY_PACKS");
    return e && *e == '1';
  }();
  if (!on) return;
  auto caller = [](const BufRef& r) { return r.kind == BufRef::kInput || r.kind == BufRef::kDOut; };
  auto early = [&](const Step& st) {
    return (st.kind == Step::kPermute || st.kind == Step::kDirect) && caller(st.a) && st.b.kind == BufRef::kNone &&
           st.c.kind == BufRef::kWork && st.label.find(":pack") != std::string::npos;
  };
  std::vector<Step> head, rest;
  for (Step& st : list) {
    if (!early(st)) {
      rest.push_back(std::move(st));
      continue;
    }
    // (its output is a fresh workspace buffer: only a later step may touch it)
    bool used_before = false;
    for (const Step& x : rest)
      for (const BufRef* r : {&x.a, &x.b, &x.c, &x.b2, &x.c2})
        used_before |= r->kind == BufRef::kWork && r->index == st.c.index;
    (used_before ? rest : head).push_back(std::move(st));
  }
  list.clear();
  for (Step& st : head) list.push_back(std::move(st));
  for (Step& st : rest) list.push_back(std::move(st));
}

// Sibling TC steps (consecutive in the list, neither depending on the other -- a node's two
// adjoints) run concurrently on two streams; each persistent grid would otherwise take every
// SM and the second would wait for the first's CTAs to drain.  They get SM budgets
// proportional to their MMA work (tiles x K stages x MMA width) so both finish together.
// CE_SM_SHARE=0 off.
void Executor::share_sms(std::vector<Step>& steps) {
  // Opt-in: cfg2 step 0.969 -> 0.956 ms, but cfg3 72.6 -> 96.6 ms and cfg4 8.4 -> 10.6 ms
  // (one-round split-K siblings then need several rounds), and every budgeted kernel runs on a
  // fraction of the GPU.  0 off (default), 1 proportional to the MMA work, 2 min-max rounds.
  static const int mode = [] {
    const char* e = std::getenv("CE_SM_SHARE");
    return e ? std::atoi(e) : 0;
  }();
  if (mode <= 0) return;
  const std::size_t n = steps.size();
  std::vector<std::vector<char>> reach(n, std::vector<char>(n, 0));  // reach[i][j]: i after j
  for (std::size_t i = 0; i < n; ++i)
    for (int j : steps[i].deps) {
      reach[i][static_cast<std::size_t>(j)] = 1;
      for (std::size_t k = 0; k < n; ++k)
        if (reach[static_cast<std::size_t>(j)][k]) reach[i][k] = 1;
    }
  // the plan node whose adjoint a backward step computes: the consumer of its operand id
  std::vector<int> consumer(static_cast<std::size_t>(n_) + plan_.nodes.size(), -1);
  for (std::size_t jj = 0; jj < plan_.nodes.size(); ++jj) {
    consumer[static_cast<std::size_t>(plan_.nodes[jj].left)] = static_cast<int>(jj);
    consumer[static_cast<std::size_t>(plan_.nodes[jj].right)] = static_cast<int>(jj);
  }
  auto pnode = [&](const Step& st) {
    return st.node >= 0 && static_cast<std::size_t>(st.node) < consumer.size() ? consumer[static_cast<std::size_t>(st.node)]
                                                                               : -1;
  };
  auto work = [](const Step& st) {
    const TcParams& P = st.tc.params;
    return static_cast<double>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_iters * P.n_mma;
  };
  for (std::size_t i = 0; i < n; ++i) {
    if (steps[i].kind != Step::kTc || steps[i].tc.sm_budget) continue;
    std::size_t k = i + 1;
    while (k < n && steps[k].kind != Step::kTc) ++k;
    if (k >= n || steps[k].tc.sm_budget || reach[k][i] || pnode(steps[i]) < 0 || pnode(steps[k]) != pnode(steps[i]))
      continue;
    // budgets minimising the later finish: rounds of items x per-item time (K stages x MMA
    // width); kept only if that beats running each on all SMs one after the other
    auto items = [](const Step& st) {
      const TcParams& P = st.tc.params;
      return static_cast<int64_t>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_split;
    };
    auto per_item = [](const Step& st) {
      const TcParams& P = st.tc.params;
      return static_cast<double>((P.k_iters + P.k_split - 1) / P.k_split) * P.n_mma;
    };
    const int64_t ia = items(steps[i]), ib = items(steps[k]);
    const double ta = per_item(steps[i]), tb = per_item(steps[k]);
    auto rounds = [](int64_t it, int64_t sms) { return static_cast<double>((it + sms - 1) / sms); };
    const double serial = rounds(ia, 148) * ta + rounds(ib, 148) * tb;
    double best = 1e300;
    int ba = 0;
    for (int x = 8; x <= 140; ++x) {
      const double c = std::max(rounds(ia, x) * ta, rounds(ib, 148 - x) * tb);
      if (c < best) {
        best = c;
        ba = x;
      }
    }
    if (mode == 1) {
      static const double bias = [] {  // CE_SM_BIAS: weight of the first (chain) sibling's work
        const char* e = std::getenv("CE_SM_BIAS");
        return e ? std::atof(e) : 1.0;
      }();
      const double wa = bias * work(steps[i]), wb = work(steps[k]);
      ba = std::max(16, std::min(132, static_cast<int>(148.0 * wa / (wa + wb) + 0.5)));
      best = 0;
    }
    if (ba > 0 && best < 0.9 * serial) {
      steps[i].tc.sm_budget = ba;
      steps[k].tc.sm_budget = 148 - ba;
    }
    i = k;
  }
}

void Executor::push_tc(std::vector<Step>& list, Step& st) {
  // CE_SPLITK_ZERO_STEP=0: the launch zeroes C itself (a memset node right before the kernel,
  // which also ends the PDL chain)
  static const bool zero_step = [] {
    const char* e = std::getenv("CE_SPLITK_ZERO_STEP");
    return !(e && *e == '0');
  }();
  // Opt-in (CE_TC_TAIL_ZERO=1): a TC launch that will split its partial last round into K
  // chunks gets C zeroed by the same kind of early zero step, so every chunk adds without the
  // chunk-0-first flag handshake (and the split then also applies from 16 K stages,
  // CE_TC_TAIL_ZKMIN).  Measured: 0.964 -> 0.989 ms with the 16-stage threshold (tt1.0's
  // 24/27-stage convs), 0.966 -> 0.968 ms at 48 stages -- not kept.
  static const bool tail_zero = [] {
    const char* e = std::getenv("CE_TC_TAIL_ZERO");
    return e && *e == '1';
  }();
  const bool tail = tail_zero && st.kind == Step::kTc && st.tc.params.k_split == 1 && !st.tc.accum &&
                    st.tc.out_span > 0 && ce_tc_tail_split(st.tc);
  if (tail) st.tc.tail_zeroed = 1;
  if (zero_step && st.kind == Step::kTc && (st.tc.params.k_split > 1 || tail) && !st.tc.accum && st.tc.out_span > 0) {
    Step z;
    z.kind = Step::kZero;
    z.c = st.c;
    z.zero_elems = st.tc.out_span;
    z.node = st.node;
    z.label = st.label + ":zero";
    auto touches = [&](const Step& x) {
      for (const BufRef* r : {&x.a, &x.b, &x.c, &x.b2, &x.c2})
        if (r->kind == st.c.kind && r->index == st.c.index && r->kind != BufRef::kNone) return true;
      return false;
    };
    std::size_t at = 0;
    for (std::size_t i = list.size(); i-- > 0;)
      if (touches(list[i])) {
        at = i + 1;
        break;
      }
    list.insert(list.begin() + static_cast<std::ptrdiff_t>(at), z);
    st.tc.zeroed = 1;
  }
  list.push_back(st);
}

void Executor::build_forward() {
  const auto& spec = plan_.spec;
  const View out_view = dense_view(spec.output, output_dims());
  if (plan_.nodes.empty()) {
    // single input: self-contraction sum + reorder (sequencer.cpp:415-420, 439-445)
    add_problem(fwd_, lower_unary(id_view_[0], out_view), id_ref_[0], {}, {BufRef::kOutput, 0}, -1, "unary");
    return;
  }
  for (int s = 0; s < 2; ++s) {
    red_view_[s].resize(plan_.nodes.size());
    red_ref_[s].resize(plan_.nodes.size());
  }
  for (std::size_t j = 0; j < plan_.nodes.size(); ++j) {
    const PlanNode& node = plan_.nodes[j];
    const PairwiseOp& op = node.op;
    const int ids[2] = {node.left, node.right};
    const Subscripts* selfs[2] = {&op.left_self, &op.right_self};
    for (int s = 0; s < 2; ++s) {
      const View& full = id_view_[static_cast<std::size_t>(ids[s])];
      if (selfs[s]->empty()) {
        red_view_[s][j] = full;
        red_ref_[s][j] = id_ref_[static_cast<std::size_t>(ids[s])];
        continue;
      }
      const Subscripts kept = minus(full.subs, *selfs[s]);
      View tmp = padded_view(kept, dims_of(full, kept), 4);
      BufRef ref{BufRef::kWork, alloc(view_span(tmp))};
      add_problem(fwd_, lower_unary(full, tmp), id_ref_[static_cast<std::size_t>(ids[s])], {}, ref,
                  static_cast<int>(j), "self-sum");
      red_view_[s][j] = tmp;
      red_ref_[s][j] = ref;
    }
    const bool last = j + 1 == plan_.nodes.size();
    const int rid = n_ + static_cast<int>(j);
    View res = last ? out_view
                    : res_layout_.count(rid) ? res_layout_.at(rid) : padded_view(op.result, op.result_dims, 4);
    BufRef res_ref = last ? BufRef{BufRef::kOutput, 0} : BufRef{BufRef::kWork, alloc(view_span(res))};
    if (!last) buf_owner_[res_ref.index] = {rid, false};
    pending_flops_ = 2.0 * static_cast<double>(flops_actual(op));
    add_problem(fwd_, lower_pairwise(op, red_view_[0][j], red_view_[1][j], res, res, Adjoint::Forward),
                red_ref_[0][j], red_ref_[1][j], res_ref, static_cast<int>(j), "node" + std::to_string(j));
    id_view_.push_back(res);
    id_ref_.push_back(res_ref);
  }
}

void Executor::build_backward() {
  const auto& spec = plan_.spec;
  const View dout_view = dense_view(spec.output, output_dims());
  if (plan_.nodes.empty()) {
    add_problem(bwd_, lower_unary(dout_view, id_view_[0]), {BufRef::kDOut, 0}, {}, {BufRef::kDInput, 0}, -1,
                "grad:0");
    return;
  }
  // gradient buffer per operand id: inputs -> user dinputs, nodes -> workspace (node layout)
  std::vector<View> gview(id_view_.size());
  std::vector<BufRef> gref(id_view_.size());
  for (std::size_t id = 0; id < id_view_.size(); ++id) {
    if (static_cast<int>(id) < n_) {
      gview[id] = id_view_[id];
      gref[id] = {BufRef::kDInput, static_cast<int64_t>(id)};
    } else if (id + 1 == id_view_.size()) {
      gview[id] = dout_view;
      gref[id] = {BufRef::kDOut, 0};
    } else {
      // the forward result's layout unless a hoisted gradient layout was chosen
      const int gid = static_cast<int>(id);
      gview[id] = grad_layout_.count(gid) ? grad_layout_.at(gid) : id_view_[id];
      gref[id] = {BufRef::kWork, alloc(view_span(gview[id]))};
      buf_owner_[gref[id].index] = {gid, true};
    }
  }
  for (std::size_t jj = plan_.nodes.size(); jj-- > 0;) {
    const PlanNode& node = plan_.nodes[jj];
    const PairwiseOp& op = node.op;
    const std::size_t cid = static_cast<std::size_t>(n_) + jj;
    const int ids[2] = {node.left, node.right};
    const Subscripts* selfs[2] = {&op.left_self, &op.right_self};
    // the gradient that continues the chain (w.r.t. an intermediate) is issued before the
    // leaf gradient (w.r.t. an input) when only the right operand is an intermediate.
    // CE_CHAIN_FIRST=0: always left first.
    static const bool chain_first = [] {
      const char* e = std::getenv("CE_CHAIN_FIRST");
      return !(e && *e == '0');
    }();
    const bool swap = chain_first && ids[0] < n_ && ids[1] >= n_;
    for (int si = 0; si < 2; ++si) {
      const int s = swap ? 1 - si : si;
      std::vector<Step>& gl = bwd_;
      pending_flops_ = 2.0 * static_cast<double>(flops_actual(op));
      const auto id = static_cast<std::size_t>(ids[s]);
      const Adjoint which = s == 0 ? Adjoint::GradLeft : Adjoint::GradRight;
      const std::string label = "grad:" + std::to_string(id);
      // Strided conv axes (extension) whose feature is this operand: x = s*n + ... has no
      // affine inverse, so dC is upsampled (zeros between the s-spaced outputs) and the
      // gradient lowered as the stride-1 op over the upsampled positions j = s*n.
      PairwiseOp gop = op;
      View dcv = gview[cid];
      BufRef dcr = gref[cid];
      {
        std::vector<int64_t> up_dims = dcv.dims;
        bool any = false;
        for (ConvAxis& ax : gop.conv_axes) {
          if (ax.stride == 1 || ax.feature_on_left != (s == 0)) continue;
          const int r = find_atom(gop.result, ax.atom);
          // j = s*n < s*out; a circular axis keeps the feature length (its wrap is mod X, and
          // s*(out-1) < X), so the stride-1 op is exactly the reference's circular map
          ax.output_dim = ax.mode == ConvMode::Circular ? ax.feature_dim : ax.output_dim * ax.stride;
          ax.stride = 1;
          gop.result_dims[static_cast<std::size_t>(r)] = ax.output_dim;
          const int d = find_atom(dcv.subs, ax.atom);
          up_dims[static_cast<std::size_t>(d)] = ax.output_dim;
          any = true;
        }
        if (any) {
          const View up = padded_view(dcv.subs, up_dims, 4);
          const BufRef upr{BufRef::kWork, alloc(view_span(up))};
          Step z;
          z.kind = Step::kZero;
          z.c = upr;
          z.zero_elems = view_span(up);
          z.node = static_cast<int>(id);
          z.label = label + ":upsample-zero";
          bwd_.push_back(z);
          // dC[.., n, ..] -> up[.., s*n, ..]: the up view with the strided atoms' strides scaled
          View dst = up;
          dst.dims = dcv.dims;
          for (const ConvAxis& ax : op.conv_axes)
            if (ax.stride != 1 && ax.feature_on_left == (s == 0))
              dst.strides[static_cast<std::size_t>(find_atom(dst.subs, ax.atom))] *= ax.stride;
          pending_flops_ = 0;
          add_problem(bwd_, lower_unary(dcv, dst), dcr, {}, upr, static_cast<int>(id), label + ":upsample");
          pending_flops_ = 2.0 * static_cast<double>(flops_actual(op));
          dcv = up;
          dcr = upr;
        }
      }
      const BufRef a = s == 0 ? dcr : red_ref_[0][jj];
      const BufRef b = s == 0 ? red_ref_[1][jj] : dcr;
      if (selfs[s]->empty()) {
        add_problem(gl, lower_pairwise(gop, red_view_[0][jj], red_view_[1][jj], dcv, gview[id], which), a, b,
                    gref[id], static_cast<int>(id), label);
      } else {
        // d(reduced) then broadcast back over the self-contracted atoms
        View tmp = padded_view(red_view_[s][jj].subs, red_view_[s][jj].dims, 4);
        BufRef tref{BufRef::kWork, alloc(view_span(tmp))};
        add_problem(gl, lower_pairwise(gop, red_view_[0][jj], red_view_[1][jj], dcv, tmp, which), a, b, tref,
                    static_cast<int>(id), label);
        pending_flops_ = 0;
        add_problem(gl, lower_unary(tmp, gview[id]), tref, {}, gref[id], static_cast<int>(id), label + ":bcast");
      }
    }
  }
}

float* Executor::resolve(const BufRef& r) const {
  switch (r.kind) {
    case BufRef::kInput: return const_cast<float*>(inputs_[r.index]);
    case BufRef::kOutput: return out_;
    case BufRef::kWork:
      return reinterpret_cast<float*>((ext_ws_ ? ext_ws_ : ws_) + buf_off_[static_cast<std::size_t>(r.index)]);
    case BufRef::kDOut: return const_cast<float*>(dout_);
    case BufRef::kDInput: return r.index < static_cast<int64_t>(dinputs_.size()) ? dinputs_[r.index] : nullptr;
    default: return nullptr;
  }
}

std::string Executor::describe() const {
  static const char* kinds[] = {"direct", "tiled", "tc", "zero", "reduce", "permute", "dw2", "split", "pconv", "row"};
  std::string out;
  char line[512];
  for (const auto* list : {&fwd_, &bwd_})
    for (const Step& st : *list) {
      int n = std::snprintf(line, sizeof line, "%s %s %s", list == &fwd_ ? "fwd" : "bwd", st.label.c_str(), kinds[st.kind]);
      if (st.kind == Step::kTc) {
        const TcParams& P = st.tc.params;
        std::snprintf(line + n, sizeof line - n,
                      " bn=%d rows=%d cols=%d mma_n=%d tiles=%dx%dx%d split=%d kit=%d amn=%d bmn=%d tr=%d mc=%d ctma=%d%s\n", st.tc.bn,
                      P.m_rows, P.n_cols, P.n_mma, P.tiles_m, P.tiles_n, P.grid_z, P.k_split, P.k_iters, P.oa.mn_major,
                      P.ob.mn_major, P.transpose_store, P.mcast, P.c_tma,
                      st.tc.sm_budget ? (" sms=" + std::to_string(st.tc.sm_budget)).c_str() : "");
        if (std::getenv("CE_DESCRIBE_UNITS")) {
          std::string u = " ";
          n = static_cast<int>(std::strlen(line)) - 1;  // before the newline
          for (int pass = 0; pass < 3; ++pass) {
            u += pass == 2 ? " gu=[" : pass ? " nt=[" : "mt=[";
            const int32_t* list = pass == 2 ? P.gu : pass ? P.nt : P.mt;
            for (int i = 0; i < (pass == 2 ? P.ng : pass ? P.nn : P.nm); ++i) {
              const TcUnit& U = P.u[list[i]];
              u += std::to_string(U.box) + "/" + std::to_string(U.ext) + ":";
              for (int k = 0; k < U.nv; ++k) u += std::to_string(U.vext[k]) + "@" + std::to_string(U.sc[k]) + (k + 1 < U.nv ? "," : "");
              u += " ";
            }
            u += "]";
          }
          std::snprintf(line + n, sizeof line - n, "%s\n", u.c_str());
        }
      } else if (st.kind == Step::kRow) {
        std::snprintf(line + n, sizeof line - n, " rows=%lld K=%d N=%d\n", static_cast<long long>(st.row.M), st.row.K,
                      st.row.N);
      } else if (st.kind == Step::kPconv) {
        const CePconvDesc& q = st.pconv;
        std::snprintf(line + n, sizeof line - n, " kind=%d planes=%lld pos=%dx%d taps=%dx%d signs=%d,%d ci=%d co=%d\n",
                      q.kind, static_cast<long long>(q.P), q.OY, q.OX, q.KH, q.KW, q.sgn_h, q.sgn_w, q.Ci, q.Co);
      } else if (st.kind == Step::kDw2) {
        std::snprintf(line + n, sizeof line - n, " fused taps=%d J=%d signs=%d,%d store_mid=%d\n", st.dw2.KT, st.dw2.J,
                      st.dw2.SA, st.dw2.SB, st.dw2.write_mid);
      } else if (st.kind == Step::kPermute) {
        char pd[256];
        ce_permute_describe(st.desc.p, pd, sizeof pd);
        static const char* bk[] = {"none", "in", "out", "ws", "dout", "din"};
        std::snprintf(line + n, sizeof line - n, " %s src=%s:%lld\n", pd, bk[st.a.kind], (long long)st.a.index);
      } else {
        char sd[256] = "";
        if (st.kind == Step::kDirect || st.kind == Step::kReduce) ce_stream_describe(st.desc, sd, sizeof sd);
        std::snprintf(line + n, sizeof line - n, " Z=%lld M=%lld N=%lld K=%lld (tc: %s) %s\n", (long long)st.desc.Z,
                      (long long)st.desc.M, (long long)st.desc.N, (long long)st.desc.K,
                      st.desc.p.unary ? "unary" : st.tc.why, sd);
      }
      out += line;
    }
  return out;
}

void Executor::ensure_workspace() {
  if (!ext_ws_ && !ws_ && ws_bytes_ > 0) cuda_check(cudaMalloc(&ws_, static_cast<size_t>(ws_bytes_)), "cudaMalloc(workspace)");
  if (!tail_flags_) {
    // the TC kernel's tail-split flags: a zeroed region per TC step (each launch leaves it zero)
    std::size_t n = 0;
    for (const auto* list : {&fwd_, &bwd_})
      for (const Step& st : *list) n += st.kind == Step::kTc;
    if (n > 0) {
      const std::size_t bytes = n * kTailFlags * sizeof(uint32_t);
      cuda_check(cudaMalloc(&tail_flags_, bytes), "cudaMalloc(tail flags)");
      cuda_check(cudaMemset(tail_flags_, 0, bytes), "cudaMemset(tail flags)");
      std::size_t i = 0;
      for (auto* list : {&fwd_, &bwd_})
        for (Step& st : *list)
          if (st.kind == Step::kTc) st.tc.tail_flags = tail_flags_ + kTailFlags * i++;
    }
  }
}

int Executor::tc_steps(bool bwd) const {
  int n = 0;
  for (const auto& s : bwd ? bwd_ : fwd_) n += s.kind == Step::kTc;
  return n;
}

void Executor::run(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s) {
  if (concurrent_ && !profiling_) {
    run_concurrent(steps, need, s);
    return;
  }
  for (Step& st : steps) {
    st.ran = false;
    if (need && st.node >= 0 && !(*need)[static_cast<std::size_t>(st.node)]) continue;
    if (!resolve(st.kind == Step::kDw2 ? st.c2 : st.c)) continue;  // gradient not requested
    st.ran = true;
    launch_step(st, s);
  }
}

void Executor::run_concurrent(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s) {
  for (int k = 0; k < n_streams_ - 1; ++k)
    if (!aux_[k]) {
      cuda_check(cudaStreamCreateWithFlags(&aux_[k], cudaStreamNonBlocking), "cudaStreamCreate");
      cuda_check(cudaEventCreateWithFlags(&join_ev_[k], cudaEventDisableTiming), "cudaEventCreate");
    }
  if (!fork_ev_) cuda_check(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "cudaEventCreate");
  const int kStreams = n_streams_;
  cudaStream_t streams[kMaxStreams] = {s};
  for (int k = 1; k < kStreams; ++k) streams[k] = aux_[k - 1];
  int last[kMaxStreams];
  bool joined[kMaxStreams] = {true};
  for (int k = 0; k < kStreams; ++k) last[k] = -1;
  for (int k = 1; k < kStreams; ++k) joined[k] = false;
  bool forked = false;
  std::vector<int> sid(steps.size(), -1);
  for (std::size_t i = 0; i < steps.size(); ++i) {
    Step& st = steps[i];
    st.ran = false;
    if (need && st.node >= 0 && !(*need)[static_cast<std::size_t>(st.node)]) continue;
    if (!resolve(st.kind == Step::kDw2 ? st.c2 : st.c)) continue;
    st.ran = true;
    if (!st.done) cuda_check(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming), "cudaEventCreate");
    // continue the chain of a dependency when it is the last step of its stream,
    // otherwise take an idle stream, otherwise the stream whose tail is oldest
    int pick = -1;
    for (int j : st.deps)
      if (steps[static_cast<std::size_t>(j)].ran && last[sid[static_cast<std::size_t>(j)]] == j) {
        pick = sid[static_cast<std::size_t>(j)];
        break;
      }
    if (pick < 0)
      for (int k = 0; k < kStreams && pick < 0; ++k)
        if (last[k] < 0) pick = k;
    if (pick < 0) {
      pick = 0;
      for (int k = 1; k < kStreams; ++k)
        if (last[k] < last[pick]) pick = k;
    }
    if (!joined[pick]) {
      if (!forked) {
        cuda_check(cudaEventRecord(fork_ev_, s), "cudaEventRecord");
        forked = true;
      }
      cuda_check(cudaStreamWaitEvent(streams[pick], fork_ev_, 0), "cudaStreamWaitEvent");
      joined[pick] = true;
    }
    for (int j : st.deps) {
      const Step& dep = steps[static_cast<std::size_t>(j)];
      if (dep.ran && sid[static_cast<std::size_t>(j)] != pick)
        cuda_check(cudaStreamWaitEvent(streams[pick], dep.done, 0), "cudaStreamWaitEvent");
    }
    launch_step(st, streams[pick]);
    cuda_check(cudaEventRecord(st.done, streams[pick]), "cudaEventRecord");
    sid[i] = pick;
    last[pick] = static_cast<int>(i);
  }
  for (int k = 1; k < kStreams; ++k)
    if (joined[k]) {
      cuda_check(cudaEventRecord(join_ev_[k - 1], streams[k]), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(s, join_ev_[k - 1], 0), "cudaStreamWaitEvent");
    }
}

namespace {
// the step's SIMT descriptor with the caller-owned-buffer flags of its operands
CeSimtDesc exact(const Step& st) {
  auto user = [](const BufRef& r) { return r.kind != BufRef::kWork && r.kind != BufRef::kNone ? 1 : 0; };
  CeSimtDesc d = st.desc;
  d.p.exact_a = user(st.a);
  d.p.exact_b = user(st.b);
  d.p.exact_c = user(st.c);
  return d;
}
}  // namespace

void Executor::launch_step(Step& st, cudaStream_t s) {
  const float* A = resolve(st.a);
  const float* B = resolve(st.b);
  float* C = resolve(st.c);
  {
    if (profiling_) {
      if (!st.ev0) {
        cuda_check(cudaEventCreate(&st.ev0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&st.ev1), "cudaEventCreate");
      }
      // External: inside stream capture this becomes an event-record node we can time
      cuda_check(cudaEventRecordWithFlags(st.ev0, s, cudaEventRecordExternal), "cudaEventRecord");
    }
    cudaError_t e = cudaSuccess;
    switch (st.kind) {
      case Step::kDirect: e = ce_launch_direct(exact(st), A, B, C, s); break;
      case Step::kTiled: e = ce_launch_tiled(st.desc, A, B, C, st.a_kfast, st.b_kfast, s); break;
      case Step::kTc: e = ce_launch_tc(st.tc, A, B, C, s); break;
      case Step::kZero: e = cudaMemsetAsync(C, 0, static_cast<size_t>(st.zero_elems) * 4, s); break;
      case Step::kReduce: e = ce_launch_reduce(exact(st), A, B, C, st.zero_elems, s); break;
      case Step::kPermute: e = ce_launch_permute(st.desc.p, A, C, s); break;
      case Step::kDw2: e = ce_launch_dw2(st.dw2, A, B, resolve(st.b2), C, resolve(st.c2), s); break;
      case Step::kSplit: e = ce_launch_split_tf32(A, C, resolve(st.c2), st.zero_elems, s); break;
      case Step::kRow: e = ce_launch_rowgemm(st.row, A, B, C, s); break;
      case Step::kPconv:
        if (st.pconv.kind == 1) e = cudaMemsetAsync(C, 0, static_cast<size_t>(st.zero_elems) * 4, s);
        if (e == cudaSuccess) e = ce_launch_pconv(st.pconv, A, B, C, s);
        break;
    }
    cuda_check(e, st.label.c_str());
    if (profiling_) cuda_check(cudaEventRecordWithFlags(st.ev1, s, cudaEventRecordExternal), "cudaEventRecord");
    if (st.kind != Step::kZero) ++last_launches_;  // (kernels only: a zero step is a memset)
  }
}

std::vector<Executor::StepTime> Executor::step_times(bool bwd) {
  std::vector<StepTime> out;
  // debug: CE_TIMELINE=1 prints each step's start / end relative to the pass's first step
  static const bool timeline = [] {
    const char* e = std::getenv("CE_TIMELINE");
    return e && *e == '1';
  }();
  cudaEvent_t first = nullptr;
  for (Step& st : bwd ? bwd_ : fwd_) {
    if (!st.ran || !st.ev0) continue;
    cuda_check(cudaEventSynchronize(st.ev1), "cudaEventSynchronize");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, st.ev0, st.ev1), "cudaEventElapsedTime");
    out.push_back({st.label, static_cast<int>(st.kind), ms, st.flops, st.bytes});
    if (timeline) {
      if (!first) first = st.ev0;
      float t0 = 0;
      cudaEventElapsedTime(&t0, first, st.ev0);
      std::fprintf(stderr, "timeline %s %-22s start %9.1f us  end %9.1f us\n", bwd ? "bwd" : "fwd", st.label.c_str(),
                   t0 * 1e3, (t0 + ms) * 1e3);
    }
  }
  return out;
}

void Executor::forward(const float* const* inputs, float* out, cudaStream_t s) {
  ensure_workspace();
  inputs_.assign(inputs, inputs + n_);
  out_ = out;
  last_launches_ = 0;
  launch_pass(fwd_, nullptr, s, 0);
  fwd_inputs_ = inputs_;
  fwd_ran_ = true;
}

void Executor::backward(const float* const* inputs, const float* dout, float* const* dinputs, cudaStream_t s) {
  if (!want_backward_) throw std::runtime_error("executor was created without backward support");
  // the backward reads the intermediates (and repacked inputs) the preceding forward left in
  // the workspace: it must have run on these very input buffers (unless it recomputes them)
  if (!cfg_.recompute) {
    if (!fwd_ran_) throw std::runtime_error("backward: no forward has run on this executor");
    for (int i = 0; i < n_; ++i)
      if (fwd_inputs_[static_cast<std::size_t>(i)] != inputs[i])
        throw std::runtime_error("backward: input " + std::to_string(i) +
                                 " is not the buffer the last forward ran on (run forward on these inputs first)");
  }
  ensure_workspace();
  dout_ = dout;
  // intermediate gradients are only needed above requested inputs
  std::vector<char> need(id_view_.size(), 0);
  for (int i = 0; i < n_; ++i) need[static_cast<std::size_t>(i)] = dinputs && dinputs[i] != nullptr;
  for (std::size_t j = 0; j < plan_.nodes.size(); ++j)
    need[static_cast<std::size_t>(n_) + j] =
        need[static_cast<std::size_t>(plan_.nodes[j].left)] || need[static_cast<std::size_t>(plan_.nodes[j].right)];
  inputs_.assign(inputs, inputs + n_);
  dinputs_.assign(n_, nullptr);
  for (int i = 0; i < n_ && dinputs; ++i) dinputs_[static_cast<std::size_t>(i)] = dinputs[i];
  last_launches_ = 0;
  launch_pass(bwd_, plan_.nodes.empty() ? nullptr : &need, s, 1);
}

}  // namespace ce
