// extern "C" boundary (include/ce/ce.h) over the host planner and the device
// executor.  Exceptions never cross the ABI: they become ce_status codes with
// a thread-local message (SPEC.md:542 exit-code mapping).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is bound with dlopen

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "../../include/ce/ce.h"
#include "cuda/ce_kernels.h"
#include "host/ce_exec.hpp"
#include "host/ce_io.hpp"
#include "host/ce_layers.hpp"

using namespace ce;

struct ce_plan {
  EvaluationPlan plan;
};

struct ce_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ce_options opts{};
  // ce_conv_einsum cache: key = expression | shapes | mode | cost_mode
  std::map<std::string, std::unique_ptr<Executor>> cached;
  // data-parallel communicator (ce_ctx_init_comm)
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t comm_in = nullptr, comm_out = nullptr;
  // arena shared by the context's recompute executors (they keep nothing between calls, and
  // every call is ordered on the ctx stream): sized to the largest of them
  char* arena = nullptr;
  size_t arena_bytes = 0;
};

struct ce_executor {
  ce_ctx* ctx = nullptr;
  std::unique_ptr<Executor> ex;
};

// (wire formats) copy a vector to a caller buffer of `cap` entries; *count gets the size
template <class T>
static void fill_out(const std::vector<T>& v, T* out, int64_t cap, int64_t* count) {
  if (count) *count = static_cast<int64_t>(v.size());
  if (static_cast<int64_t>(v.size()) > cap || (!out && !v.empty()))
    throw std::runtime_error("output buffer too small (need " + std::to_string(v.size()) + ")");
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
}

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
ce_status guard(F&& f) {
  try {
    f();
    return CE_OK;
  } catch (const ParseError& e) {
    g_err = e.what();
    return CE_ERR_PARSE;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return CE_ERR_SHAPE;
  } catch (const PlanError& e) {
    g_err = e.what();
    return CE_ERR_PLAN;
  } catch (const OverflowError& e) {
    g_err = e.what();
    return CE_ERR_OVERFLOW;
  } catch (const CudaError& e) {
    g_err = e.what();
    return CE_ERR_CUDA;
  } catch (const NcclError& e) {
    g_err = e.what();
    return CE_ERR_NCCL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::string(e.what()).rfind("CUDA error", 0) == 0 ? CE_ERR_CUDA : CE_ERR_OTHER;
  }
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void copy_out(const std::string& s, char* buf, size_t cap) {
  if (!buf || s.size() + 1 > cap) throw std::runtime_error("output buffer too small (need " + std::to_string(s.size() + 1) + ")");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

std::vector<std::vector<int64_t>> split_dims(const int64_t* dims, const int* ranks, int n) {
  std::vector<std::vector<int64_t>> out;
  int64_t pos = 0;
  for (int i = 0; i < n; ++i) {
    out.emplace_back(dims + pos, dims + pos + ranks[i]);
    pos += ranks[i];
  }
  return out;
}

void split_u128(u128 v, uint64_t* lo, uint64_t* hi) {
  *lo = static_cast<uint64_t>(v);
  if (hi) *hi = static_cast<uint64_t>(v >> 64);
}

// The conv-mode argument of every plan-building entry point: either one mode name, applied
// through resolve_conv_modes (kernels.cpp:38-43: atoms shared by >= 3 inputs become Circular),
// or an explicit per-atom ConvModeMap (kernels.hpp:27-32) as "h=same,w=circular,(r1)=full"
// that must name every convolution atom of the expression (and nothing else).
ConvModeMap modes_arg(const ExpressionSpec& spec, const char* mode) {
  const std::string m(mode ? mode : "");
  if (m.find('=') == std::string::npos) return resolve_conv_modes(spec, conv_mode_spec_from_string(m));
  ConvModeMap out;
  std::size_t pos = 0;
  while (pos <= m.size()) {
    const std::size_t end = std::min(m.find(',', pos), m.size());
    const std::string item = m.substr(pos, end - pos);
    const std::size_t eq = item.find('=');
    if (eq == std::string::npos) throw ShapeError("mode map entry without '=': '" + item + "'");
    std::string name = item.substr(0, eq);
    if (name.size() >= 2 && name.front() == '(' && name.back() == ')') name = name.substr(1, name.size() - 2);
    const Atom a(name);
    if (!spec.is_conv(a)) throw ShapeError("mode map names '" + name + "', which is not a convolution atom");
    if (out.count(a)) throw ShapeError("mode map names '" + name + "' twice");
    out[a] = conv_mode_spec_from_string(item.substr(eq + 1));
    pos = end + 1;
  }
  for (const auto& a : spec.conv_atoms)
    if (!out.count(a)) throw ShapeError("mode map has no mode for convolution atom '" + a.name + "'");
  return out;
}

// Subscripts of a result string such as "bhw(r2)" (the tokens of the reference's parser).
Subscripts parse_subscripts(const std::string& s) {
  ExpressionSpec one = parse(s + "->" + s);
  return one.output;
}

// A one-node plan for pairwise_eval with the planner's node construction.
EvaluationPlan pairwise_plan(const char* expr, const int64_t* dims, const int* ranks, const char* mode) {
  EvaluationPlan plan;
  plan.spec = parse(expr);
  if (plan.spec.inputs.size() != 2) throw ShapeError("pairwise expression must have exactly two inputs");
  plan.env = make_shape_env(plan.spec, split_dims(dims, ranks, 2));
  plan.modes = modes_arg(plan.spec, mode);
  std::set<Atom> keep(plan.spec.output.begin(), plan.spec.output.end());
  PlanNode node;
  node.left = 0;
  node.right = 1;
  node.op = make_pairwise_op(plan.spec.inputs[0], plan.env.dims[0], plan.spec.inputs[1], plan.env.dims[1], keep,
                             plan.modes, plan.spec.output);
  node.cost = pairwise_cost(node.op, CostMode::Inference).total;
  plan.total_cost = node.cost;
  plan.root_subs = node.op.result;
  plan.root_dims = node.op.result_dims;
  plan.peak_intermediate_elements = static_cast<uint64_t>(node.op.result_elements());
  plan.nodes.push_back(std::move(node));
  return plan;
}

// NCCL entry points resolved at run time from the libnccl.so.2 already loaded in the
// process (torch's) or, failing that, the system one.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
  ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(dlsym(h, "ncclCommAbort"));
    api.get_async_error = reinterpret_cast<decltype(api.get_async_error)>(dlsym(h, "ncclCommGetAsyncError"));
  });
  if (!api.all_reduce || !api.comm_init_rank || !api.get_unique_id || !api.group_start || !api.group_end)
    throw NcclError("NCCL unavailable: " + (why.empty() ? std::string("missing symbols") : why));
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw NcclError(std::string("NCCL error in ") + what + ": " +
                    (nccl().error_string ? nccl().error_string(r) : std::to_string(static_cast<int>(r))));
}

// Non-blocking health check of a communicator (ncclCommGetAsyncError): a peer that died or a
// network failure surfaces here instead of as a hang in a later collective.  On an error the
// communicator is aborted (its pending work is cancelled) and CE_ERR_NCCL is raised.
void comm_health(ce_ctx* ctx) {
  if (!ctx->comm || !nccl().get_async_error) return;
  ncclResult_t async = ncclSuccess;
  nccl_ok(nccl().get_async_error(ctx->comm, &async), "ncclCommGetAsyncError");
  if (async != ncclSuccess && async != ncclInProgress) {
    const std::string why = nccl().error_string ? nccl().error_string(async) : std::to_string(static_cast<int>(async));
    if (nccl().comm_abort) nccl().comm_abort(ctx->comm);
    ctx->comm = nullptr;
    throw NcclError("NCCL communicator failed asynchronously: " + why);
  }
}

void fill_stats(const Executor& ex, ce_exec_stats* st, bool bwd) {
  if (!st) return;
  u128 m = 0;
  for (const auto& n : ex.plan().nodes) m = add_checked(m, flops_actual(n.op));
  split_u128(m, &st->multiplications_lo, &st->multiplications_hi);
  st->peak_intermediate_elements = ex.plan().peak_intermediate_elements;
  st->kernels_launched = ex.last_launches();
  st->tc_steps = ex.tc_steps(bwd);
}

}  // namespace

extern "C" {

const char* ce_last_error(void) { return g_err.c_str(); }
const char* ce_version(void) { return "ce 0.1 (sm_100a, tcgen05 tf32 + fp32 simt)"; }

ce_status ce_parse(const char* expr, char* rendered, size_t rendered_cap, char* classes, size_t classes_cap) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    copy_out(render(spec), rendered, rendered_cap);
    std::string s;
    for (const auto& [a, c] : classify(spec)) s += (s.empty() ? "" : " ") + a.name + ":" + to_string(c);
    copy_out(s, classes, classes_cap);
  });
}

ce_status ce_plan_create(const char* expr, const int64_t* dims, const int* ranks, int n_inputs, const char* mode,
                         const char* cost_mode, int strategy, ce_plan** out) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    ShapeEnv env = make_shape_env(spec, split_dims(dims, ranks, n_inputs));
    ConvModeMap modes = modes_arg(spec, mode);
    CostMode cm = cost_mode_from_string(cost_mode);
    auto p = std::make_unique<ce_plan>();
    if (strategy == CE_PLAN_LEFT_TO_RIGHT) {
      p->plan = left_to_right(spec, env, modes, cm);
    } else {
      OptimalOptions o;
      o.cost_capped = strategy == CE_PLAN_OPTIMAL_CAPPED;
      p->plan = optimal(spec, env, modes, cm, o);
    }
    *out = p.release();
  });
}

ce_status ce_plan_from_joins(const char* expr, const int64_t* dims, const int* ranks, int n_inputs, const char* mode,
                             const char* cost_mode, const int* joins, int n_joins, ce_plan** out) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    ShapeEnv env = make_shape_env(spec, split_dims(dims, ranks, n_inputs));
    std::vector<std::pair<int, int>> j;
    for (int i = 0; i < n_joins; ++i) j.push_back({joins[2 * i], joins[2 * i + 1]});
    auto p = std::make_unique<ce_plan>();
    p->plan = plan_from_joins(spec, env, modes_arg(spec, mode), cost_mode_from_string(cost_mode), j);
    *out = p.release();
  });
}

ce_status ce_plan_from_nodes(const char* expr, const int64_t* dims, const int* ranks, int n_inputs, const char* mode,
                             const char* cost_mode, const int* joins, const char* const* results, int n_nodes,
                             ce_plan** out) {
  return guard([&] {
    ExpressionSpec spec = parse(expr);
    ShapeEnv env = make_shape_env(spec, split_dims(dims, ranks, n_inputs));
    std::vector<std::pair<int, int>> j;
    std::vector<Subscripts> res;
    for (int i = 0; i < n_nodes; ++i) {
      j.push_back({joins[2 * i], joins[2 * i + 1]});
      res.push_back(parse_subscripts(results[i]));
    }
    auto p = std::make_unique<ce_plan>();
    p->plan = plan_from_nodes(spec, env, modes_arg(spec, mode), cost_mode_from_string(cost_mode), j, res);
    *out = p.release();
  });
}

void ce_plan_destroy(ce_plan* plan) { delete plan; }

ce_status ce_plan_json(const ce_plan* plan, char* buf, size_t cap) {
  return guard([&] { copy_out(plan_to_json(plan->plan), buf, cap); });
}

ce_status ce_plan_tree_encoding(const ce_plan* plan, char* buf, size_t cap) {
  return guard([&] { copy_out(plan->plan.nodes.empty() ? std::string("0") : tree_encoding(plan->plan), buf, cap); });
}

ce_status ce_plan_get_info(const ce_plan* plan, ce_plan_info* info) {
  return guard([&] {
    const EvaluationPlan& p = plan->plan;
    *info = ce_plan_info{};
    info->n_inputs = static_cast<int>(p.spec.inputs.size());
    info->n_nodes = static_cast<int>(p.nodes.size());
    std::vector<int64_t> od;
    if (p.nodes.empty()) {
      for (const auto& a : p.spec.output) od.push_back(p.env.dim_of(p.spec, a));
    } else {
      const auto& op = p.nodes.back().op;
      for (const auto& a : p.spec.output) od.push_back(op.result_dims[static_cast<std::size_t>(find_atom(op.result, a))]);
    }
    if (od.size() > 16) throw ShapeError("output rank above 16");
    info->out_rank = static_cast<int>(od.size());
    for (std::size_t i = 0; i < od.size(); ++i) info->out_dims[i] = od[i];
    split_u128(p.total_cost, &info->total_cost_lo, &info->total_cost_hi);
    split_u128(plan_cost(p, CostMode::Inference), &info->inference_cost_lo, &info->inference_cost_hi);
    split_u128(plan_cost(p, CostMode::Training), &info->training_cost_lo, &info->training_cost_hi);
    u128 f = 0;
    for (const auto& n : p.nodes) f = add_checked(f, flops_actual(n.op));
    split_u128(f, &info->flops_actual_lo, &info->flops_actual_hi);
    info->peak_intermediate_elements = p.peak_intermediate_elements;
  });
}

ce_status ce_plan_node(const ce_plan* plan, int node, int* left, int* right, char* result_subs, size_t cap,
                       uint64_t* flops_actual_lo, uint64_t* cost_lo) {
  return guard([&] {
    const auto& n = plan->plan.nodes.at(static_cast<std::size_t>(node));
    *left = n.left;
    *right = n.right;
    copy_out(render(n.op.result), result_subs, cap);
    split_u128(flops_actual(n.op), flops_actual_lo, nullptr);
    split_u128(n.cost, cost_lo, nullptr);
  });
}

ce_status ce_layer_expression(const char* kind, const int64_t* t_factors, int n_t, const int64_t* s_factors, int n_s,
                              int64_t filter_h, int64_t filter_w, int64_t feature_h, int64_t feature_w, int64_t batch,
                              const int64_t* ranks, int n_ranks, double cr, char* expr_out, size_t expr_cap,
                              int64_t* dims_out, int dims_cap, int* ranks_of_input, int* n_inputs, int64_t* ranks_out,
                              int* n_ranks_out, uint64_t* param_count_out) {
  return guard([&] {
    LayerSpec l;
    l.kind = layer_kind_from_string(kind);
    l.t_factors.assign(t_factors, t_factors + n_t);
    l.s_factors.assign(s_factors, s_factors + n_s);
    l.filter_h = filter_h;
    l.filter_w = filter_w;
    l.feature_h = feature_h;
    l.feature_w = feature_w;
    l.batch = batch;
    if (cr > 0) {
      l.ranks.assign(rank_slot_count(l.kind, l.order()), 1);
      l = with_compression_rank(l, cr);
    } else {
      l.ranks.assign(ranks, ranks + n_ranks);
    }
    LayerExpression ex = expression(l);
    // ranks_of_input / ranks_out are caller arrays of CE_MAX_LAYER_INPUTS / CE_MAX_LAYER_RANKS
    if (ex.env.dims.size() > CE_MAX_LAYER_INPUTS)
      throw ShapeError("layer has " + std::to_string(ex.env.dims.size()) + " inputs (CE_MAX_LAYER_INPUTS " +
                       std::to_string(CE_MAX_LAYER_INPUTS) + ")");
    if (l.ranks.size() > CE_MAX_LAYER_RANKS)
      throw ShapeError("layer has " + std::to_string(l.ranks.size()) + " rank slots (CE_MAX_LAYER_RANKS " +
                       std::to_string(CE_MAX_LAYER_RANKS) + ")");
    copy_out(render(ex.spec), expr_out, expr_cap);
    int pos = 0;
    for (std::size_t i = 0; i < ex.env.dims.size(); ++i) {
      ranks_of_input[i] = static_cast<int>(ex.env.dims[i].size());
      for (int64_t d : ex.env.dims[i]) {
        if (pos >= dims_cap) throw std::runtime_error("dims_out too small");
        dims_out[pos++] = d;
      }
    }
    *n_inputs = static_cast<int>(ex.env.dims.size());
    for (std::size_t i = 0; i < l.ranks.size(); ++i) ranks_out[i] = l.ranks[i];
    *n_ranks_out = static_cast<int>(l.ranks.size());
    split_u128(param_count(l), param_count_out, nullptr);
  });
}


ce_status ce_tensor_to_json(const int64_t* shape, int rank, const double* data, char* buf, size_t cap,
                            size_t* len_out) {
  return guard([&] {
    const std::string s = tensor_to_json(std::vector<int64_t>(shape, shape + rank), data);
    if (len_out) *len_out = s.size() + 1;
    copy_out(s, buf, cap);
  });
}

ce_status ce_tensor_from_json(const char* text, int64_t* shape, int shape_cap, int* rank, double* data,
                              int64_t data_cap, int64_t* count) {
  return guard([&] {
    std::vector<int64_t> sh;
    std::vector<double> d;
    tensor_from_json(text, &sh, &d);
    int64_t r = 0;
    fill_out(sh, shape, shape_cap, &r);
    *rank = static_cast<int>(r);
    fill_out(d, data, data_cap, count);
  });
}

ce_status ce_tensor_to_binary(const int64_t* shape, int rank, const double* data, unsigned char* buf, size_t cap,
                              size_t* len_out) {
  return guard([&] {
    const std::string s = tensor_to_binary(std::vector<int64_t>(shape, shape + rank), data);
    if (len_out) *len_out = s.size();
    if (!buf || s.size() > cap) throw std::runtime_error("output buffer too small (need " + std::to_string(s.size()) + ")");
    std::memcpy(buf, s.data(), s.size());
  });
}

ce_status ce_tensor_from_binary(const unsigned char* bytes, size_t len, int64_t* shape, int shape_cap, int* rank,
                                double* data, int64_t data_cap, int64_t* count) {
  return guard([&] {
    std::vector<int64_t> sh;
    std::vector<double> d;
    tensor_from_binary(std::string(reinterpret_cast<const char*>(bytes), len), &sh, &d);
    int64_t r = 0;
    fill_out(sh, shape, shape_cap, &r);
    *rank = static_cast<int>(r);
    fill_out(d, data, data_cap, count);
  });
}

ce_status ce_layer_to_json(const char* kind, const int64_t* t_factors, int n_t, const int64_t* s_factors, int n_s,
                           int64_t filter_h, int64_t filter_w, int64_t feature_h, int64_t feature_w, int64_t batch,
                           const int64_t* ranks, int n_ranks, char* buf, size_t cap) {
  return guard([&] {
    LayerSpec l;
    l.kind = layer_kind_from_string(kind);
    l.t_factors.assign(t_factors, t_factors + n_t);
    l.s_factors.assign(s_factors, s_factors + n_s);
    l.filter_h = filter_h;
    l.filter_w = filter_w;
    l.feature_h = feature_h;
    l.feature_w = feature_w;
    l.batch = batch;
    l.ranks.assign(ranks, ranks + n_ranks);
    copy_out(layer_to_json(l), buf, cap);
  });
}

ce_status ce_layer_from_json(const char* text, char* kind, size_t kind_cap, int64_t* t_factors, int* n_t,
                             int64_t* s_factors, int* n_s, int64_t* hw5, int64_t* ranks, int* n_ranks) {
  return guard([&] {
    const LayerSpec l = layer_from_json(text);
    copy_out(to_string(l.kind), kind, kind_cap);
    int64_t n = 0;
    fill_out(l.t_factors, t_factors, CE_MAX_LAYER_RANKS, &n);
    *n_t = static_cast<int>(n);
    fill_out(l.s_factors, s_factors, CE_MAX_LAYER_RANKS, &n);
    *n_s = static_cast<int>(n);
    fill_out(l.ranks, ranks, CE_MAX_LAYER_RANKS, &n);
    *n_ranks = static_cast<int>(n);
    hw5[0] = l.filter_h;
    hw5[1] = l.filter_w;
    hw5[2] = l.feature_h;
    hw5[3] = l.feature_w;
    hw5[4] = l.batch;
  });
}

ce_status ce_plan_describe_steps(const ce_plan* plan, int want_backward, int math, char* buf, size_t cap) {
  return guard([&] {
    ExecConfig cfg;
    cfg.math = math;
    cfg.recompute = (want_backward & CE_EXEC_RECOMPUTE) != 0;
    Executor ex(plan->plan, (want_backward & ~CE_EXEC_RECOMPUTE) != 0, cfg);
    copy_out(ex.describe() + "workspace_bytes " + std::to_string(ex.workspace_bytes()) + "\n" +
                 "workspace_bytes_unshared " + std::to_string(ex.workspace_bytes_unshared()) + "\n",
             buf, cap);
  });
}

ce_status ce_ctx_create(int device, const ce_options* opts, ce_ctx** out) {
  return guard([&] {
    auto c = std::make_unique<ce_ctx>();
    c->device = device;
    if (opts) c->opts = *opts;
    cuda_ok(cudaSetDevice(device), "cudaSetDevice");
    if (c->opts.stream) {
      c->stream = static_cast<cudaStream_t>(c->opts.stream);
    } else {
      cuda_ok(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      c->own_stream = true;
    }
    *out = c.release();
  });
}

void ce_ctx_destroy(ce_ctx* ctx) {
  if (!ctx) return;
  ctx->cached.clear();
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->comm_stream);
    if (nccl().comm_destroy) nccl().comm_destroy(ctx->comm);
    cudaStreamDestroy(ctx->comm_stream);
    cudaEventDestroy(ctx->comm_in);
    cudaEventDestroy(ctx->comm_out);
  }
  if (ctx->arena) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->arena);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void* ce_ctx_stream(ce_ctx* ctx) { return ctx->stream; }

ce_status ce_ctx_synchronize(ce_ctx* ctx) {
  return guard([&] { cuda_ok(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); });
}

ce_status ce_ctx_alloc(ce_ctx* ctx, size_t bytes, void** out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    *out = nullptr;
    cuda_ok(cudaMalloc(out, bytes ? bytes : 1), "cudaMalloc");
  });
}

ce_status ce_ctx_free(ce_ctx* ctx, void* p) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (p) cuda_ok(cudaFree(p), "cudaFree");
  });
}

ce_status ce_ctx_memcpy(ce_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream), "cudaMemcpyAsync");
    cuda_ok(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  });
}

ce_status ce_fill_random(ce_ctx* ctx, float* dst, int64_t n, uint64_t seed) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_ok(ce_launch_fill(dst, n, seed, ctx->stream), "fill_random");
  });
}

ce_status ce_executor_create(ce_ctx* ctx, const ce_plan* plan, int want_backward, ce_executor** out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    auto e = std::make_unique<ce_executor>();
    e->ctx = ctx;
    ExecConfig cfg;
    cfg.math = ctx->opts.math;
    cfg.recompute = (want_backward & CE_EXEC_RECOMPUTE) != 0;
    e->ex = std::make_unique<Executor>(plan->plan, (want_backward & ~CE_EXEC_RECOMPUTE) != 0, cfg);
    e->ex->set_use_graphs(ctx->opts.use_graphs != 0);
    *out = e.release();
  });
}

void ce_executor_destroy(ce_executor* ex) { delete ex; }

namespace {
// recompute executors run on the context's shared arena (grown, after a stream sync, when a
// larger one is bound)
void bind_shared_arena(ce_executor* ex) {
  if (!ex->ex->recompute()) return;
  ce_ctx* c = ex->ctx;
  const size_t need = static_cast<size_t>(ex->ex->workspace_bytes());
  if (need > c->arena_bytes) {
    if (c->arena) {
      cuda_ok(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
      cuda_ok(cudaFree(c->arena), "cudaFree");
      c->arena = nullptr;
      c->arena_bytes = 0;
    }
    cuda_ok(cudaMalloc(reinterpret_cast<void**>(&c->arena), need), "cudaMalloc(shared arena)");
    c->arena_bytes = need;
  }
  ex->ex->bind_workspace(c->arena);
}
}  // namespace

ce_status ce_ctx_workspace_bytes(ce_ctx* ctx, size_t* bytes) {
  return guard([&] { *bytes = ctx->arena_bytes; });
}

ce_status ce_execute(ce_executor* ex, const float* const* inputs, float* out, ce_exec_stats* stats) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ex->ctx->device), "cudaSetDevice");
    bind_shared_arena(ex);
    ex->ex->forward(inputs, out, ex->ctx->stream);
    fill_stats(*ex->ex, stats, false);
  });
}

ce_status ce_backward(ce_executor* ex, const float* const* inputs, const float* dout, float* const* dinputs,
                      ce_exec_stats* stats) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ex->ctx->device), "cudaSetDevice");
    bind_shared_arena(ex);
    ex->ex->backward(inputs, dout, dinputs, ex->ctx->stream);
    fill_stats(*ex->ex, stats, true);
  });
}

ce_status ce_executor_set_profiling(ce_executor* ex, int enable) {
  return guard([&] { ex->ex->set_profiling(enable != 0); });
}

ce_status ce_executor_profile(ce_executor* ex, int backward, int max_steps, int* n_steps, char* labels,
                              size_t labels_cap, int* kinds, float* ms, double* flops, double* bytes) {
  return guard([&] {
    auto t = ex->ex->step_times(backward != 0);
    std::string names;
    const int n = std::min<int>(max_steps, static_cast<int>(t.size()));
    for (int i = 0; i < n; ++i) {
      names += t[static_cast<std::size_t>(i)].label + "\n";
      kinds[i] = t[static_cast<std::size_t>(i)].kind;
      ms[i] = t[static_cast<std::size_t>(i)].ms;
      flops[i] = t[static_cast<std::size_t>(i)].flops;
      bytes[i] = t[static_cast<std::size_t>(i)].bytes;
    }
    *n_steps = n;
    copy_out(names, labels, labels_cap);
  });
}

ce_status ce_execute_host(ce_executor* ex, const float* const* host_inputs, float* host_out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ex->ctx->device), "cudaSetDevice");
    const EvaluationPlan& p = ex->ex->plan();
    cudaStream_t s = ex->ctx->stream;
    std::vector<float*> dev(p.spec.inputs.size());
    for (std::size_t i = 0; i < dev.size(); ++i) {
      const size_t bytes = static_cast<size_t>(element_count(p.env.dims[i])) * 4;
      cuda_ok(cudaMallocAsync(&dev[i], bytes, s), "cudaMallocAsync");
      cuda_ok(cudaMemcpyAsync(dev[i], host_inputs[i], bytes, cudaMemcpyHostToDevice, s), "H2D");
    }
    const size_t obytes = static_cast<size_t>(element_count(ex->ex->output_dims())) * 4;
    float* dout = nullptr;
    cuda_ok(cudaMallocAsync(&dout, obytes, s), "cudaMallocAsync");
    bind_shared_arena(ex);
    ex->ex->forward(dev.data(), dout, s);
    cuda_ok(cudaMemcpyAsync(host_out, dout, obytes, cudaMemcpyDeviceToHost, s), "D2H");
    for (float* d : dev) cudaFreeAsync(d, s);
    cudaFreeAsync(dout, s);
    cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}

ce_status ce_pairwise_eval(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, const char* mode,
                           const float* a, const float* b, float* out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    ExecConfig cfg;
    cfg.math = ctx->opts.math;
    Executor ex(pairwise_plan(expr, dims, ranks, mode), false, cfg);
    const float* ins[2] = {a, b};
    ex.forward(ins, out, ctx->stream);
    cuda_ok(cudaStreamSynchronize(ctx->stream), "pairwise_eval");
  });
}

ce_status ce_pairwise_grad(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, const char* mode,
                           const float* a, const float* b, const float* dout, float* da, float* db) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    ExecConfig cfg;
    cfg.math = ctx->opts.math;
    Executor ex(pairwise_plan(expr, dims, ranks, mode), true, cfg);
    const float* ins[2] = {a, b};
    float* dins[2] = {da, db};
    // backward reuses the forward's workspace (self-contraction sums), so run it first
    float* scratch = nullptr;
    cuda_ok(cudaMallocAsync(&scratch, static_cast<size_t>(element_count(ex.output_dims())) * 4, ctx->stream),
            "cudaMallocAsync");
    ex.forward(ins, scratch, ctx->stream);
    ex.backward(ins, dout, dins, ctx->stream);
    cuda_ok(cudaFreeAsync(scratch, ctx->stream), "cudaFreeAsync");
    cuda_ok(cudaStreamSynchronize(ctx->stream), "pairwise_grad");
  });
}

ce_status ce_flops_actual(const char* expr, const int64_t* dims, const int* ranks, const char* mode, uint64_t* lo,
                          uint64_t* hi) {
  return guard([&] { split_u128(flops_actual(pairwise_plan(expr, dims, ranks, mode).nodes[0].op), lo, hi); });
}

// ------------------------------------------------------------------ like-mode merging
namespace {
Subscripts parse_subs(const char* subs) {
  ExpressionSpec spec = parse(std::string(subs) + "->");
  return spec.inputs.at(0);
}
AtomClass class_from_string(const std::string& c) {
  for (AtomClass k : {AtomClass::Convolution, AtomClass::BatchProduct, AtomClass::Contraction, AtomClass::Free,
                      AtomClass::SelfContraction})
    if (c == to_string(k)) return k;
  throw ShapeError("merge: unknown atom class '" + c + "'");
}
}  // namespace

ce_status ce_merge_like_modes(ce_ctx* ctx, const char* subs, const int64_t* dims, const char* classes,
                              const float* in, float* out, char* merged_subs, size_t subs_cap, int64_t* merged_dims,
                              int* merged_rank, char* record, size_t record_cap) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    const Subscripts sub = parse_subs(subs);
    const std::vector<int64_t> d(dims, dims + sub.size());
    std::map<Atom, AtomClass> cls;
    {
      std::string s = classes;
      std::size_t pos = 0;
      while (pos < s.size()) {
        const std::size_t end = std::min(s.find(' ', pos), s.size());
        const std::string tok = s.substr(pos, end - pos);
        pos = end + 1;
        if (tok.empty()) continue;
        const std::size_t colon = tok.rfind(':');
        if (colon == std::string::npos) throw ShapeError("merge: class entry '" + tok + "' is not atom:class");
        cls[Atom{tok.substr(0, colon)}] = class_from_string(tok.substr(colon + 1));
      }
    }
    // canonical class order; members keep their order of appearance (kernels.cpp:249-264)
    std::vector<std::pair<AtomClass, Subscripts>> groups = {
        {AtomClass::BatchProduct, {}}, {AtomClass::Contraction, {}}, {AtomClass::Free, {}}, {AtomClass::Convolution, {}}};
    for (const Atom& a : sub) {
      auto it = cls.find(a);
      if (it == cls.end()) throw ShapeError("merge: atom '" + a.name + "' has no class");
      const int g = it->second == AtomClass::BatchProduct ? 0
                    : (it->second == AtomClass::Contraction || it->second == AtomClass::SelfContraction) ? 1
                    : it->second == AtomClass::Free ? 2 : 3;
      groups[static_cast<std::size_t>(g)].second.push_back(a);
    }
    Subscripts order;
    std::vector<int64_t> odims;
    for (const auto& g : groups)
      for (const Atom& a : g.second) {
        order.push_back(a);
        odims.push_back(d[static_cast<std::size_t>(find_atom(sub, a))]);
      }
    // the data movement: one permute (family c) into the canonical order
    const CeProblem p = lower_unary(dense_view(sub, d), dense_view(order, odims));
    if (element_count(d) > 0) {
      cudaError_t e = ce_permute_supported(p) ? ce_launch_permute(p, in, out, ctx->stream)
                                              : ce_launch_direct(simt_desc(p), in, nullptr, out, ctx->stream);
      cuda_ok(e, "merge_like_modes permute");
    }
    // the reshape: compound axes per class (singletons and conv atoms keep their own axes)
    Subscripts msubs;
    std::vector<int64_t> mdims;
    std::string rec;
    std::size_t pos = 0;
    for (const auto& [c, members] : groups) {
      if (members.empty()) continue;
      if (members.size() == 1 || c == AtomClass::Convolution) {
        for (const Atom& a : members) {
          msubs.push_back(a);
          mdims.push_back(odims[pos++]);
        }
        continue;
      }
      std::string name;
      int64_t dim = 1;
      rec += rec.empty() ? "" : ";";
      std::string mem;
      for (const Atom& a : members) {
        name += a.name;
        mem += (mem.empty() ? "" : ",") + a.name + ":" + std::to_string(odims[pos]);
        dim *= odims[pos++];
      }
      msubs.push_back(Atom{name});
      mdims.push_back(dim);
      rec += name + "=" + mem;
    }
    copy_out(render(msubs), merged_subs, subs_cap);
    for (std::size_t i = 0; i < mdims.size(); ++i) merged_dims[i] = mdims[i];
    *merged_rank = static_cast<int>(mdims.size());
    copy_out(rec, record, record_cap);
  });
}

ce_status ce_unmerge_modes(const char* subs, const int64_t* dims, const char* record, char* out_subs,
                           size_t subs_cap, int64_t* out_dims, int* out_rank) {
  return guard([&] {
    const Subscripts sub = parse_subs(subs);
    // record: "compound=member:dim,member:dim;..."
    std::map<std::string, std::vector<std::pair<std::string, int64_t>>> groups;
    std::string r = record ? record : "";
    std::size_t pos = 0;
    while (pos < r.size()) {
      const std::size_t end = std::min(r.find(';', pos), r.size());
      const std::string g = r.substr(pos, end - pos);
      pos = end + 1;
      const std::size_t eq = g.find('=');
      if (eq == std::string::npos) throw ShapeError("unmerge: malformed record group '" + g + "'");
      auto& mem = groups[g.substr(0, eq)];
      std::size_t q = eq + 1;
      while (q < g.size()) {
        const std::size_t e2 = std::min(g.find(',', q), g.size());
        const std::string m = g.substr(q, e2 - q);
        q = e2 + 1;
        const std::size_t colon = m.rfind(':');
        if (colon == std::string::npos) throw ShapeError("unmerge: malformed member '" + m + "'");
        mem.push_back({m.substr(0, colon), std::stoll(m.substr(colon + 1))});
      }
    }
    Subscripts os;
    std::vector<int64_t> od;
    for (std::size_t i = 0; i < sub.size(); ++i) {
      auto it = groups.find(sub[i].name);
      if (it == groups.end()) {
        os.push_back(sub[i]);
        od.push_back(dims[i]);
        continue;
      }
      int64_t prod = 1;
      for (const auto& [n, dd] : it->second) {
        os.push_back(Atom{n});
        od.push_back(dd);
        prod *= dd;
      }
      if (prod != dims[i]) throw ShapeError("unmerge: compound '" + sub[i].name + "' dim does not match its members");
    }
    copy_out(render(os), out_subs, subs_cap);
    for (std::size_t i = 0; i < od.size(); ++i) out_dims[i] = od[i];
    *out_rank = static_cast<int>(od.size());
  });
}

ce_status ce_conv_einsum(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, int n_inputs,
                         const char* mode, const char* cost_mode, const float* const* inputs, float* out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    std::string key = std::string(expr) + "|" + mode + "|" + cost_mode;
    int64_t pos = 0;
    for (int i = 0; i < n_inputs; ++i) {
      key += "|";
      for (int r = 0; r < ranks[i]; ++r) key += std::to_string(dims[pos++]) + ",";
    }
    auto it = ctx->cached.find(key);
    if (it == ctx->cached.end()) {
      ExpressionSpec spec = parse(expr);
      ShapeEnv env = make_shape_env(spec, split_dims(dims, ranks, n_inputs));
      EvaluationPlan plan = optimal(spec, env, modes_arg(spec, mode), cost_mode_from_string(cost_mode));
      ExecConfig cfg;
      cfg.math = ctx->opts.math;
      auto ex = std::make_unique<Executor>(plan, false, cfg);
      ex->set_use_graphs(ctx->opts.use_graphs != 0);
      it = ctx->cached.emplace(key, std::move(ex)).first;
    }
    it->second->forward(inputs, out, ctx->stream);
  });
}

ce_status ce_nccl_unique_id(void* id128) {
  return guard([&] {
    ncclUniqueId id;
    nccl_ok(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof id);
  });
}

ce_status ce_ctx_init_comm(ce_ctx* ctx, int nranks, int rank, const void* id128) {
  return guard([&] {
    if (ctx->comm) throw std::runtime_error("context already has a communicator");
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    nccl_ok(nccl().comm_init_rank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
    cuda_ok(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_ok(cudaEventCreateWithFlags(&ctx->comm_in, cudaEventDisableTiming), "cudaEventCreate");
    cuda_ok(cudaEventCreateWithFlags(&ctx->comm_out, cudaEventDisableTiming), "cudaEventCreate");
  });
}

ce_status ce_allreduce_grads(ce_ctx* ctx, float* const* bufs, const int64_t* counts, int n) {
  return guard([&] {
    if (!ctx->comm) throw std::runtime_error("ce_allreduce_grads: no communicator (ce_ctx_init_comm)");
    comm_health(ctx);
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    cuda_ok(cudaEventRecord(ctx->comm_in, ctx->stream), "cudaEventRecord");
    cuda_ok(cudaStreamWaitEvent(ctx->comm_stream, ctx->comm_in, 0), "cudaStreamWaitEvent");
    const NcclApi& api = nccl();
    nccl_ok(api.group_start(), "ncclGroupStart");
    for (int i = 0; i < n; ++i)
      if (bufs[i] && counts[i] > 0)
        nccl_ok(api.all_reduce(bufs[i], bufs[i], static_cast<size_t>(counts[i]), ncclFloat32, ncclSum, ctx->comm,
                               ctx->comm_stream),
                "ncclAllReduce");
    nccl_ok(api.group_end(), "ncclGroupEnd");
    cuda_ok(cudaEventRecord(ctx->comm_out, ctx->comm_stream), "cudaEventRecord");
  });
}

ce_status ce_comm_wait(ce_ctx* ctx) {
  return guard([&] {
    if (!ctx->comm) return;
    comm_health(ctx);
    cuda_ok(cudaStreamWaitEvent(ctx->stream, ctx->comm_out, 0), "cudaStreamWaitEvent");
  });
}

ce_status ce_comm_check(ce_ctx* ctx) {
  return guard([&] {
    if (!ctx->comm) throw std::runtime_error("ce_comm_check: no communicator (ce_ctx_init_comm)");
    comm_health(ctx);
  });
}

}  // extern "C"
