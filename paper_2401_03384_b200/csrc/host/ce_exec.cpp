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
  if (ws_bytes_ > 0) cuda_check(cudaMalloc(&ws_, static_cast<size_t>(ws_bytes_)), "cudaMalloc(workspace)");
}

Executor::~Executor() {
  if (ws_) cudaFree(ws_);
}

int64_t Executor::alloc(int64_t elems) {
  const int64_t off = ws_bytes_;
  ws_bytes_ += (elems * 4 + 255) / 256 * 256;
  return off;
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

void Executor::add_problem(std::vector<Step>& list, const CeProblem& p, BufRef a, BufRef b, BufRef c, int node,
                           const std::string& label) {
  Step st;
  st.a = a;
  st.b = b;
  st.c = c;
  st.node = node;
  st.label = label;
  st.desc = simt_desc(p);
  const CeSimtDesc& d = st.desc;
  if (cfg_.math == 0 && !p.unary && ce_tc_plan(p, &st.tc)) {
    st.kind = Step::kTc;
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
    View res = last ? out_view : padded_view(op.result, op.result_dims, 4);
    BufRef res_ref = last ? BufRef{BufRef::kOutput, 0} : BufRef{BufRef::kWork, alloc(view_span(res))};
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
      gview[id] = id_view_[id];  // same padded layout as the forward result
      gref[id] = {BufRef::kWork, alloc(view_span(gview[id]))};
    }
  }
  for (std::size_t jj = plan_.nodes.size(); jj-- > 0;) {
    const PlanNode& node = plan_.nodes[jj];
    const PairwiseOp& op = node.op;
    const std::size_t cid = static_cast<std::size_t>(n_) + jj;
    const int ids[2] = {node.left, node.right};
    const Subscripts* selfs[2] = {&op.left_self, &op.right_self};
    for (int s = 0; s < 2; ++s) {
      const auto id = static_cast<std::size_t>(ids[s]);
      const Adjoint which = s == 0 ? Adjoint::GradLeft : Adjoint::GradRight;
      const std::string label = "grad:" + std::to_string(id);
      const BufRef a = s == 0 ? gref[cid] : red_ref_[0][jj];
      const BufRef b = s == 0 ? red_ref_[1][jj] : gref[cid];
      if (selfs[s]->empty()) {
        add_problem(bwd_, lower_pairwise(op, red_view_[0][jj], red_view_[1][jj], gview[cid], gview[id], which), a, b,
                    gref[id], static_cast<int>(id), label);
      } else {
        // d(reduced) then broadcast back over the self-contracted atoms
        View tmp = padded_view(red_view_[s][jj].subs, red_view_[s][jj].dims, 4);
        BufRef tref{BufRef::kWork, alloc(view_span(tmp))};
        add_problem(bwd_, lower_pairwise(op, red_view_[0][jj], red_view_[1][jj], gview[cid], tmp, which), a, b, tref,
                    static_cast<int>(id), label);
        add_problem(bwd_, lower_unary(tmp, gview[id]), tref, {}, gref[id], static_cast<int>(id), label + ":bcast");
      }
    }
  }
}

float* Executor::resolve(const BufRef& r) const {
  switch (r.kind) {
    case BufRef::kInput: return const_cast<float*>(inputs_[r.index]);
    case BufRef::kOutput: return out_;
    case BufRef::kWork: return reinterpret_cast<float*>(ws_ + r.index);
    case BufRef::kDOut: return const_cast<float*>(dout_);
    case BufRef::kDInput: return r.index < static_cast<int64_t>(dinputs_.size()) ? dinputs_[r.index] : nullptr;
    default: return nullptr;
  }
}

int Executor::tc_steps(bool bwd) const {
  int n = 0;
  for (const auto& s : bwd ? bwd_ : fwd_) n += s.kind == Step::kTc;
  return n;
}

void Executor::run(const std::vector<Step>& steps, cudaStream_t s) {
  for (const Step& st : steps) {
    const float* A = resolve(st.a);
    const float* B = resolve(st.b);
    float* C = resolve(st.c);
    if (!C) continue;  // gradient not requested
    cudaError_t e = cudaSuccess;
    switch (st.kind) {
      case Step::kDirect: e = ce_launch_direct(st.desc, A, B, C, s); break;
      case Step::kTiled: e = ce_launch_tiled(st.desc, A, B, C, st.a_kfast, st.b_kfast, s); break;
      case Step::kTc: e = ce_launch_tc(st.tc, A, B, C, s); break;
      case Step::kZero: e = cudaMemsetAsync(C, 0, static_cast<size_t>(st.zero_elems) * 4, s); break;
    }
    cuda_check(e, st.label.c_str());
    ++last_launches_;
  }
}

void Executor::forward(const float* const* inputs, float* out, cudaStream_t s) {
  inputs_.assign(inputs, inputs + n_);
  out_ = out;
  last_launches_ = 0;
  run(fwd_, s);
}

void Executor::backward(const float* const* inputs, const float* dout, float* const* dinputs, cudaStream_t s) {
  if (!want_backward_) throw std::runtime_error("executor was created without backward support");
  dout_ = dout;
  // intermediate gradients are only needed above requested inputs
  std::vector<char> need(id_view_.size(), 0);
  for (int i = 0; i < n_; ++i) need[static_cast<std::size_t>(i)] = dinputs && dinputs[i] != nullptr;
  for (std::size_t j = 0; j < plan_.nodes.size(); ++j)
    need[static_cast<std::size_t>(n_) + j] =
        need[static_cast<std::size_t>(plan_.nodes[j].left)] || need[static_cast<std::size_t>(plan_.nodes[j].right)];
  std::vector<Step> todo;
  for (const Step& st : bwd_)
    if (plan_.nodes.empty() || need[static_cast<std::size_t>(st.node)]) todo.push_back(st);
  inputs_.assign(inputs, inputs + n_);
  dinputs_.assign(n_, nullptr);
  for (int i = 0; i < n_ && dinputs; ++i) dinputs_[static_cast<std::size_t>(i)] = dinputs[i];
  last_launches_ = 0;
  run(todo, s);
}

}  // namespace ce
