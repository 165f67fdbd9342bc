// Device plan executor: the B200 replacement for execute()
// (/root/reference/proj/src/sequencer.cpp:403-447) and, per node, for
// pairwise_eval (kernels.cpp:425-470), plus the backward pass the reference
// does not have.  A plan is compiled ONCE into a flat list of kernel steps over
// symbolic buffers (inputs / output / workspace offsets); each call only binds
// pointers and launches, stream-ordered, optionally replayed as a CUDA graph.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../cuda/ce_device.h"
#include "../cuda/ce_fuse.h"
#include "../cuda/ce_pconv.h"
#include "../cuda/ce_rowgemm.h"
#include "../cuda/ce_tc.h"
#include "ce_lower.hpp"
#include "ce_plan.hpp"

namespace ce {

struct BufRef {
  enum Kind { kNone, kInput, kOutput, kWork, kDOut, kDInput } kind = kNone;
  int64_t index = 0;  // input index, or workspace buffer id (its offset is assigned by liveness)
};

struct Step {
  enum Kind { kDirect, kTiled, kTc, kZero, kReduce, kPermute, kDw2, kSplit, kPconv, kRow } kind = kDirect;
  CeSimtDesc desc{};
  int a_kfast = 0, b_kfast = 0;
  TcPlan tc{};
  BufRef a, b, c;
  // kDw2 (two chained depthwise stencils, ce_fuse.h): a -(b)-> c (stored only when read
  // later; else kNone) -(b2)-> c2
  CeDw2Desc dw2{};
  BufRef b2, c2;
  CePconvDesc pconv{};  // kPconv (ce_pconv.h); kind 1 zeroes zero_elems of C first
  CeRowDesc row{};      // kRow (ce_rowgemm.h)
  int64_t zero_elems = 0;
  double flops = 0;   // algorithmic FLOPs (2 x flops_actual of the node / adjoint)
  double bytes = 0;   // compulsory bytes (|A| + |B| + |C|) x 4
  bool ran = false;   // launched by the last call
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int node = -1;
  std::string label;
  std::vector<int> deps;        // earlier steps of the same pass with a buffer hazard
  cudaEvent_t done = nullptr;   // recorded after the step (cross-stream edges)
};

struct ExecConfig {
  int math = 0;  // 0 auto (TF32 tensor cores where mappable), 1 FP32 SIMT only, 2 3xTF32 tensor cores
  // gradient checkpointing: the forward pass keeps no
  // intermediates; the backward pass recomputes them first (one extra forward's work)
  bool recompute = false;
};

class Executor {
 public:
  Executor(const EvaluationPlan& plan, bool want_backward, ExecConfig cfg);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  void forward(const float* const* inputs, float* out, cudaStream_t s);
  void backward(const float* const* inputs, const float* dout, float* const* dinputs, cudaStream_t s);

  const EvaluationPlan& plan() const { return plan_; }
  int64_t workspace_bytes() const { return ws_bytes_; }
  // bytes a bump allocator (every buffer alive for the whole executor) would need
  int64_t workspace_bytes_unshared() const { return ws_unshared_; }
  int last_launches() const { return last_launches_; }
  int tc_steps(bool bwd) const;
  const std::vector<Step>& forward_steps() const { return fwd_; }
  const std::vector<Step>& backward_steps() const { return bwd_; }
  std::vector<int64_t> output_dims() const;
  std::string describe() const;  // one line per kernel step (no CUDA calls)
  void set_profiling(bool on) { profiling_ = on; }
  // per launched step of the last forward (bwd=false) or backward call:
  // label, kind, device ms (CUDA events on the launch stream), flops, bytes
  struct StepTime {
    std::string label;
    int kind;
    float ms;
    double flops, bytes;
  };
  std::vector<StepTime> step_times(bool bwd);

 private:
  int64_t alloc(int64_t elems);
  void ensure_workspace();
  void add_problem(std::vector<Step>& list, const CeProblem& p, BufRef a, BufRef b, BufRef c, int node,
                   const std::string& label);
  // split-K TC step: its C memset becomes a kZero step placed right after the last earlier
  // step touching C, so it runs off the critical path (on a side stream)
  void push_tc(std::vector<Step>& list, Step& st);
  void early_packs(std::vector<Step>& list);
  void share_sms(std::vector<Step>& steps);
  void build_forward();
  void build_backward();
  void run(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s);
  void run_concurrent(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s);
  void launch_step(Step& st, cudaStream_t s);
  void compute_deps(std::vector<Step>& steps) const;
  void assign_offsets();
  void fuse_chains(std::vector<Step>& list);
  void add_recompute();
  bool tc_math() const { return cfg_.math == 0 || cfg_.math == 2; }
  bool overlap(const BufRef& x, const BufRef& y) const;
  float* resolve(const BufRef& r) const;

  EvaluationPlan plan_;
  bool want_backward_;
  ExecConfig cfg_;
  int n_ = 0;
  // per operand id (inputs then nodes): view as consumed by its node (after self-sum)
  std::vector<View> id_view_;      // full view of operand id (inputs dense, nodes padded)
  std::vector<BufRef> id_ref_;
  std::vector<View> red_view_[2];  // per node, post-self-sum view of left/right
  std::vector<BufRef> red_ref_[2];
  std::vector<Step> fwd_, bwd_;
  int64_t ws_bytes_ = 0, ws_unshared_ = 0;
  std::vector<int64_t> buf_bytes_, buf_off_;  // per workspace buffer id
  int ws_reuse_mode_ = 0;
  char* ws_ = nullptr;
  char* ext_ws_ = nullptr;
  uint32_t* tail_flags_ = nullptr;  // kTailFlags zeroed words per TC step (tail split)
  // bound per call
  std::vector<const float*> inputs_;
  std::vector<const float*> fwd_inputs_;  // inputs of the last forward (its intermediates are in ws_)
  bool fwd_ran_ = false;
  float* out_ = nullptr;
  const float* dout_ = nullptr;
  std::vector<float*> dinputs_;
  int last_launches_ = 0;
  bool profiling_ = false;
  double pending_flops_ = 0;  // FLOPs credited to the next add_problem (build time)
  struct PackRecord {
    BufRef src;
    CeProblem pk;
    BufRef dst;
  };
  std::vector<PackRecord> packs_;  // forward repacks, reusable by later steps
  // Layout hoisting: a workspace buffer one of our own steps writes (a node result or its
  // gradient) that a consumer repacks is instead written in the packed layout by its
  // producer (operand id -> view; the other readers take the new strides), see hoist_packs
  struct PackLog {
    BufRef src;
    CeProblem pk;
    bool fwd;
  };
  std::vector<PackLog> pack_log_;
  std::map<int, View> res_layout_, grad_layout_;
  std::map<int64_t, std::pair<int, bool>> buf_owner_;  // workspace buffer -> (operand id, gradient?)
  void reset_build();
  bool hoist_packs();
  // CUDA-graph replay of a pass: valid while the bound pointers are unchanged
  struct GraphCache {
    std::vector<const void*> key;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
  };
  GraphCache graphs_[2];
  bool use_graphs_ = false;
  // independent steps (e.g. the input- and factor-gradient of one node, a repack and the
  // step before it) run on side streams, forked from and joined back into the caller's
  static constexpr int kMaxStreams = 8;
  int n_streams_ = 4;  // CE_STREAMS (2..8): the caller's stream + side streams
  bool concurrent_ = true;
  cudaStream_t aux_[kMaxStreams - 1] = {};
  cudaEvent_t fork_ev_ = nullptr, join_ev_[kMaxStreams - 1] = {};
  void launch_pass(std::vector<Step>& steps, const std::vector<char>* need, cudaStream_t s, int which);

 public:
  void set_use_graphs(bool on) { use_graphs_ = on; }
  // Run on a caller-owned arena of >= workspace_bytes() (e.g. one arena a context shares
  // among its recompute executors: they keep nothing between calls); nullptr: own arena.
  void bind_workspace(char* base) { ext_ws_ = base; }
  bool recompute() const { return cfg_.recompute; }
};

}  // namespace ce
