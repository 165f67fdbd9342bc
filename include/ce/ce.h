/*
 * ce.h — C ABI of the B200-native conv_einsum executor (libce.so).
 *
 * The reference (`convexpr`, /root/reference/proj) is a C++20 library with no
 * FFI: its hot path is the by-value C++ pair
 *     ExecutionResult execute(const EvaluationPlan&, const std::vector<DenseTensor>&)
 *                                                        (sequencer.hpp:88, sequencer.cpp:403-447)
 *     DenseTensor pairwise_eval(const DenseTensor&, const DenseTensor&, const PairwiseOp&)
 *                                                        (kernels.hpp:105, kernels.cpp:425-470)
 * fed by parse (expression.hpp:78) -> make_shape_env (tensor.hpp:83) ->
 * resolve_conv_modes (kernels.hpp:30) -> optimal/left_to_right (sequencer.hpp:44-63).
 * These entry points are what a maintainer's FFI for that path would bind
 * (see INTEGRATION.md for the ctypes / C++ shims).  Plain pointers and sizes,
 * no torch types.  Tensors are FP32, dense row-major in the subscript order of
 * the expression (input i: spec.inputs[i], output: spec.output), resident in
 * device memory unless the function name says "host".
 *
 * Errors: every call returns ce_status (aligned with SPEC.md:542 exit codes:
 * 2 parse, 3 shape, 4 numeric, 1 other; plus planner/overflow/CUDA codes);
 * ce_last_error() gives the thread-local message of the last failure.
 * Threading: calls on one ce_ctx are stream-ordered and not re-entrant;
 * different contexts (GPUs) may be driven from different host threads.
 */
#ifndef CE_CE_H
#define CE_CE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CE_OK = 0,
  CE_ERR_OTHER = 1,
  CE_ERR_PARSE = 2,    /* ParseError        expression.hpp:15-20  */
  CE_ERR_SHAPE = 3,    /* ShapeError        tensor.hpp:16-18      */
  CE_ERR_NUMERIC = 4,
  CE_ERR_PLAN = 5,     /* PlanError         sequencer.hpp:14-16   */
  CE_ERR_OVERFLOW = 6, /* OverflowError     checked_int.hpp:13-15 */
  CE_ERR_CUDA = 7,
  CE_ERR_NCCL = 8,
  CE_ERR_UNSUPPORTED = 9
} ce_status;

const char* ce_last_error(void);
const char* ce_version(void);

/* ---------------------------------------------------------------- host IR -- */
/* parse + render + classify (expression.hpp:76-83).  `rendered` gets render(spec);
 * `classes` gets "atom:class" pairs separated by spaces in atom-name order. */
ce_status ce_parse(const char* expr, char* rendered, size_t rendered_cap, char* classes, size_t classes_cap);

/* ---------------------------------------------------------------- planner -- */
typedef struct ce_plan ce_plan;

typedef enum { CE_PLAN_OPTIMAL = 0, CE_PLAN_LEFT_TO_RIGHT = 1, CE_PLAN_OPTIMAL_CAPPED = 2 } ce_plan_strategy;

/* dims: all input dims concatenated; ranks[i]: number of axes of input i.
 * mode: "full" | "same" | "valid" | "circular" applied through resolve_conv_modes
 * (kernels.cpp:38-43: atoms shared by >= 3 inputs become circular), or an explicit per-atom
 * ConvModeMap (kernels.hpp:27-32) "h=same,w=circular,(r1)=full" naming every conv atom
 * (accepted by every entry point below that takes a mode).
 * cost_mode: "inference" | "training" (cost.hpp:8).
 * Replaces: optimal()/left_to_right() (sequencer.hpp:44-63). */
ce_status ce_plan_create(const char* expr, const int64_t* dims, const int* ranks, int n_inputs, const char* mode,
                         const char* cost_mode, int strategy, ce_plan** out);
/* plan_from_joins (sequencer.hpp:70-73): joins[2*j], joins[2*j+1] = (left id, right id). */
ce_status ce_plan_from_joins(const char* expr, const int64_t* dims, const int* ranks, int n_inputs,
                             const char* mode, const char* cost_mode, const int* joins, int n_joins,
                             ce_plan** out);
/* Replays a caller's EvaluationPlan (sequencer.hpp:30-41) exactly: node j joins operand ids
 * joins[2j], joins[2j+1] (inputs 0..N-1, node k is N+k) and keeps exactly the atoms of
 * results[j] in that order ("bhw(r2)", the plan_to_json "result" field), with the per-atom
 * modes of `mode`.  This is what the reference's execute(plan, inputs) runs; the optimal /
 * left_to_right / from_joins entry points re-derive the result orders instead. */
ce_status ce_plan_from_nodes(const char* expr, const int64_t* dims, const int* ranks, int n_inputs,
                             const char* mode, const char* cost_mode, const int* joins,
                             const char* const* results, int n_nodes, ce_plan** out);
void ce_plan_destroy(ce_plan* plan);
/* plan_to_json (sequencer.cpp:466-480), byte-identical to the reference. */
ce_status ce_plan_json(const ce_plan* plan, char* buf, size_t cap);
/* tree_encoding (sequencer.cpp:449-457); "0" for single-input plans. */
ce_status ce_plan_tree_encoding(const ce_plan* plan, char* buf, size_t cap);

typedef struct {
  int n_inputs, n_nodes, out_rank;
  int64_t out_dims[16];
  uint64_t total_cost_lo, total_cost_hi;         /* plan.total_cost (u128) under the plan's mode */
  uint64_t inference_cost_lo, inference_cost_hi; /* plan_cost(plan, Inference) */
  uint64_t training_cost_lo, training_cost_hi;   /* plan_cost(plan, Training) */
  uint64_t flops_actual_lo, flops_actual_hi;     /* sum of flops_actual over nodes (executed MACs) */
  uint64_t peak_intermediate_elements;
} ce_plan_info;
ce_status ce_plan_get_info(const ce_plan* plan, ce_plan_info* info);

/* Per-node description: "left right result_subs flops_actual_lo cost" for diagnostics. */
ce_status ce_plan_node(const ce_plan* plan, int node, int* left, int* right, char* result_subs, size_t cap,
                       uint64_t* flops_actual_lo, uint64_t* cost_lo);

/* The kernel steps an executor would launch for this plan (no device needed):
 * one line per step "fwd|bwd label kind details", then "workspace_bytes N" (liveness-
 * shared arena) and "workspace_bytes_unshared N" (every buffer alive throughout). */
ce_status ce_plan_describe_steps(const ce_plan* plan, int want_backward, int math, char* buf, size_t cap);
/* (want_backward takes the same CE_EXEC_RECOMPUTE flag as ce_executor_create) */

/* ----------------------------------------------------------------- layers -- */
#define CE_MAX_LAYER_INPUTS 32 /* capacity of ranks_of_input[] (entries) */
#define CE_MAX_LAYER_RANKS 32  /* capacity of ranks_out[] (entries) */
/* expression() (layers.hpp:71): kind name as in layer_kind_from_string (layers.cpp:29-45).
 * With cr > 0 the ranks are solved by rank_for_compression (layers.cpp:341-366) and
 * written to ranks_out.  dims_out/ranks_of_input receive the per-input shapes.
 * ranks_of_input must hold CE_MAX_LAYER_INPUTS entries and ranks_out CE_MAX_LAYER_RANKS;
 * a layer needing more fails with CE_ERR_SHAPE before anything is written to them. */
ce_status ce_layer_expression(const char* kind, const int64_t* t_factors, int n_t, const int64_t* s_factors,
                              int n_s, int64_t filter_h, int64_t filter_w, int64_t feature_h, int64_t feature_w,
                              int64_t batch, const int64_t* ranks, int n_ranks, double cr, char* expr_out,
                              size_t expr_cap, int64_t* dims_out, int dims_cap, int* ranks_of_input,
                              int* n_inputs, int64_t* ranks_out, int* n_ranks_out, uint64_t* param_count);

/* ----------------------------------------------------------------- device -- */
typedef struct ce_ctx ce_ctx;

typedef enum {
  CE_MATH_AUTO = 0,      /* tcgen05 TF32 tensor cores where the step maps onto them, FP32 SIMT elsewhere */
  CE_MATH_FP32_SIMT = 1, /* FP32 CUDA-core kernels only (accuracy anchor) */
  CE_MATH_3XTF32 = 2     /* tensor cores with split operands: hi*hi + hi*lo + lo*hi, ~FP32 accuracy */
} ce_math;

typedef struct {
  int math;           /* ce_math */
  int use_graphs;     /* capture execute/backward into CUDA graphs on first call */
  void* stream;       /* optional cudaStream_t to run on (NULL: ctx creates its own) */
} ce_options;

ce_status ce_ctx_create(int device, const ce_options* opts, ce_ctx** out);
void ce_ctx_destroy(ce_ctx* ctx);
void* ce_ctx_stream(ce_ctx* ctx); /* the cudaStream_t all work of this ctx is ordered on */
ce_status ce_ctx_synchronize(ce_ctx* ctx);

/* Device memory for callers without their own CUDA runtime (the CLI, FFI bindings):
 * cudaMalloc / cudaFree on the ctx's device, and stream-ordered copies on the ctx stream
 * (ce_ctx_memcpy returns once the copy completed). */
ce_status ce_ctx_alloc(ce_ctx* ctx, size_t bytes, void** out);
ce_status ce_ctx_free(ce_ctx* ctx, void* p);
ce_status ce_ctx_memcpy(ce_ctx* ctx, void* dst, const void* src, size_t bytes); /* any direction (UVA) */

/* Device SplitMix64 fill (tensor.cpp:107-130): dst[i] = (float) fill_random(seed)[i]. */
ce_status ce_fill_random(ce_ctx* ctx, float* dst, int64_t n, uint64_t seed);

/* ------------------------------------------------------------ executor ----- */
typedef struct ce_executor ce_executor;

typedef struct {
  uint64_t multiplications_lo, multiplications_hi; /* ExecutionResult.multiplications (sequencer.hpp:82) */
  uint64_t peak_intermediate_elements;             /* ExecutionResult.peak_intermediate_elements */
  int kernels_launched;                            /* kernels launched by the last call */
  int tc_steps;                                    /* steps that ran on tcgen05 tensor cores */
} ce_exec_stats;

/* Binds a plan to a context and sizes its workspace (intermediates, packed
 * operands and, with want_backward, gradient buffers).  want_backward: 0, 1, or
 * 1 | CE_EXEC_RECOMPUTE: gradient checkpointing -- execute keeps no
 * intermediates for the backward pass, ce_backward recomputes them first (one more forward's
 * work, a smaller workspace, and no need for a preceding ce_execute). */
#define CE_EXEC_RECOMPUTE 0x100
/* Bytes of the arena a context shares among its CE_EXEC_RECOMPUTE executors (the largest
 * workspace of any of them bound so far; executors that keep intermediates own theirs). */
ce_status ce_ctx_workspace_bytes(ce_ctx* ctx, size_t* bytes);
ce_status ce_executor_create(ce_ctx* ctx, const ce_plan* plan, int want_backward, ce_executor** out);
void ce_executor_destroy(ce_executor* ex);
/* execute (sequencer.cpp:403-447): inputs[i] device FP32 dense in spec.inputs[i]
 * order; out device FP32 dense in spec.output order.  Stream-ordered. */
ce_status ce_execute(ce_executor* ex, const float* const* inputs, float* out, ce_exec_stats* stats);
/* Gradients of <dout, execute(inputs)> w.r.t. each input (NULL entries skipped).
 * Requires a preceding ce_execute on this executor with the same inputs: the
 * intermediates it left in the workspace are reused (no recompute). */
ce_status ce_backward(ce_executor* ex, const float* const* inputs, const float* dout, float* const* dinputs,
                      ce_exec_stats* stats);
/* Per-kernel device timing: when enabled, every launched step is bracketed by
 * CUDA events on the ctx stream.  ce_executor_profile reports the last forward
 * (backward = 0) or backward call: newline-separated labels, kind (0 direct,
 * 1 tiled, 2 tensor-core, 3 memset, 4 reduce, 5 permute, 6 fused chain), ms, algorithmic
 * FLOPs and bytes. */
ce_status ce_executor_set_profiling(ce_executor* ex, int enable);
ce_status ce_executor_profile(ce_executor* ex, int backward, int max_steps, int* n_steps, char* labels,
                              size_t labels_cap, int* kinds, float* ms, double* flops, double* bytes);
/* Host-buffer convenience (e2e path): H2D copy, execute, D2H copy, synchronize. */
ce_status ce_execute_host(ce_executor* ex, const float* const* host_inputs, float* host_out);

/* ------------------------------------------------------------ wire formats - */
/* The reference's serialisations, FP64 on the wire like DenseTensor
 * (tensor.hpp:24-36).  *_len / *count receive the required size even when the buffer is
 * too small (then CE_ERR_OTHER), so a NULL/0 call queries it.
 * tensor_to_json (tensor.cpp:132-137): {"data":[...],"shape":[...]}, numbers as nlohmann's
 * dump() prints them (shortest round trip). */
ce_status ce_tensor_to_json(const int64_t* shape, int rank, const double* data, char* buf, size_t cap,
                            size_t* len_out);
/* tensor_from_json (tensor.cpp:139-147): CE_ERR_PARSE on malformed text, CE_ERR_SHAPE when
 * the data length does not match the shape. */
ce_status ce_tensor_from_json(const char* text, int64_t* shape, int shape_cap, int* rank, double* data,
                              int64_t data_cap, int64_t* count);
/* tensor_write_binary / tensor_read_binary (tensor.cpp:149-186): little-endian u64 rank,
 * u64 dims, f64 payload; CE_ERR_SHAPE on a truncated stream. */
ce_status ce_tensor_to_binary(const int64_t* shape, int rank, const double* data, unsigned char* buf, size_t cap,
                              size_t* len_out);
ce_status ce_tensor_from_binary(const unsigned char* bytes, size_t len, int64_t* shape, int shape_cap, int* rank,
                                double* data, int64_t data_cap, int64_t* count);
/* layer_to_json / layer_from_json (layers.cpp:425-467).  ce_layer_from_json fills kind,
 * T / S factors (CE_MAX_LAYER_RANKS entries each), hw = {H, W, Hp, Wp, B} and the ranks
 * (a scalar "rank" is broadcast to every slot, as the reference does); validate() errors
 * (layers.cpp) come back as CE_ERR_SHAPE. */
ce_status ce_layer_to_json(const char* kind, const int64_t* t_factors, int n_t, const int64_t* s_factors, int n_s,
                           int64_t filter_h, int64_t filter_w, int64_t feature_h, int64_t feature_w, int64_t batch,
                           const int64_t* ranks, int n_ranks, char* buf, size_t cap);
ce_status ce_layer_from_json(const char* text, char* kind, size_t kind_cap, int64_t* t_factors, int* n_t,
                             int64_t* s_factors, int* n_s, int64_t* hw5, int64_t* ranks, int* n_ranks);

/* ------------------------------------------------------------ pairwise ----- */
/* pairwise_eval (kernels.cpp:425-470) for the op make_pairwise_op builds from
 * expr "L,R->RES|convs" with keep = RES and result order RES (the planner's node
 * construction, sequencer.cpp:118-124).  a, b, out: device FP32 dense. */
ce_status ce_pairwise_eval(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, const char* mode,
                           const float* a, const float* b, float* out);
/* Adjoints of the same op: da = d<dout, op(a,b)>/da, db likewise (NULL to skip). */
ce_status ce_pairwise_grad(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, const char* mode,
                           const float* a, const float* b, const float* dout, float* da, float* db);

/* flops_actual (kernels.cpp:472-505) of the pairwise op built from expr "L,R->RES|convs"
 * as in ce_pairwise_eval: exact executed multiply-adds, u128 as two u64. */
ce_status ce_flops_actual(const char* expr, const int64_t* dims, const int* ranks, const char* mode, uint64_t* lo,
                          uint64_t* hi);

/* ------------------------------------------------------ like-mode merging -- */
/* merge_like_modes (kernels.hpp:88-94, kernels.cpp:246-265) on the device: permutes `in`
 * (FP32, dense in `subs` order, shape `dims`) into `out` in the canonical class order
 * batch | contraction (+ self) | free | convolution (members in their order of appearance),
 * and reports the merged subscripts / dims: each class's atoms become one compound atom
 * named by concatenating the member names, except singletons and convolution atoms
 * (kernels.cpp:191-235).  `classes` lists "atom:class" pairs as ce_parse emits them.
 * `record` receives the MergeRecord as text "compound=member:dim,member:dim;..." for
 * ce_unmerge_modes.  Stream-ordered on the ctx stream. */
ce_status ce_merge_like_modes(ce_ctx* ctx, const char* subs, const int64_t* dims, const char* classes,
                              const float* in, float* out, char* merged_subs, size_t subs_cap, int64_t* merged_dims,
                              int* merged_rank, char* record, size_t record_cap);
/* unmerge_modes (kernels.cpp:267-286): a reshape (no data movement): every compound atom of
 * `subs` named in `record` is expanded back into its members. */
ce_status ce_unmerge_modes(const char* subs, const int64_t* dims, const char* record, char* out_subs,
                           size_t subs_cap, int64_t* out_dims, int* out_rank);

/* ------------------------------------------------------------ conv_einsum -- */
/* The paper's call form conv_einsum("...", T1, T2, ...): parse ->
 * make_shape_env -> resolve_conv_modes -> optimal(cost_mode) -> execute, with the
 * plan and its executor cached in the context by (expression, shapes, mode,
 * cost_mode).  inputs/out: device FP32 dense; stream-ordered on the ctx stream. */
ce_status ce_conv_einsum(ce_ctx* ctx, const char* expr, const int64_t* dims, const int* ranks, int n_inputs,
                         const char* mode, const char* cost_mode, const float* const* inputs, float* out);

/* ------------------------------------------------------------ data parallel  */
/* Batch-sharded training: factors are replicated, each rank runs its
 * batch slice, and the factor gradients are summed across ranks.  NCCL is bound at
 * run time (the libnccl.so.2 already in the process, e.g. torch's, else the system one).
 * ce_nccl_unique_id: 128 bytes to hand from rank 0 to every rank (any transport). */
ce_status ce_nccl_unique_id(void* id128);
/* Joins the context to an nranks-wide communicator (one context per GPU). */
ce_status ce_ctx_init_comm(ce_ctx* ctx, int nranks, int rank, const void* id128);
/* In-place sum all-reduce of n FP32 device buffers, one NCCL group.  Runs on the
 * context's communication stream after the work already queued on the ctx stream,
 * so it overlaps later ctx work (e.g. the next layer's backward); ce_comm_wait
 * orders the ctx stream after every collective issued so far. */
ce_status ce_allreduce_grads(ce_ctx* ctx, float* const* bufs, const int64_t* counts, int n);
ce_status ce_comm_wait(ce_ctx* ctx);
/* Non-blocking communicator health poll (ncclCommGetAsyncError; also done by
 * ce_allreduce_grads and ce_comm_wait): CE_ERR_NCCL after an asynchronous failure, in which
 * case the communicator has been aborted and the context no longer has one. */
ce_status ce_comm_check(ce_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* CE_CE_H */
