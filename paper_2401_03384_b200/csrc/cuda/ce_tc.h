// Tensor-core path (families a + b1): tcgen05 kind::tf32 implicit GEMM fed by
// TMA, accumulating in TMEM.
//
// A lowered problem (ce_device.h) is mapped onto "units": index variables
// merged where they are memory-contiguous in every TMA operand.  Each operand
// becomes a <=5-D TMA tensor map; per tile and per K-iteration the producer
// computes every TMA coordinate as an affine function of unit values
// (coordinate = cst + c0*val[u0] + c1*val[u1]), which is how the convolution's
// shifted taps (x = sp*p + sq*q + c) and Same/Full zero padding (TMA OOB fill)
// are expressed without any im2col buffer.
//
//   A (M side) tile: 128 rows x 32 K  (K-major: one box; MN-major: 4 boxes of 32)
//   B (N side) tile: BN rows x 32 K
//   D: 128 x BN fp32 in TMEM -> registers -> (smem transpose) -> global scatter
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_device.h"

#define TC_MAX_UNITS 14
#define TC_BM 128
#define TC_BK 32
#define kTailFlags 512  // tail-split flag words per TC step (>= groups of one launch)

enum TcSrc { TC_SRC_MTILE = 0, TC_SRC_NTILE = 1, TC_SRC_GRID = 2, TC_SRC_K = 3 };

// Unsigned division by a launch constant d >= 1 as a multiply-high and shift (exact for
// dividends below 2^31): the per-tile index decoding would otherwise be ~20 dependent
// integer divisions on the start-up path of every role.
struct TcDiv {
  uint32_t d, mul, shr;
};

inline TcDiv tc_div(uint32_t d) {
  TcDiv r{d, 0, 0};
  if (d <= 1) return r;
  int l = 0;
  while ((1ull << l) < d) ++l;  // ceil(log2 d)
  const int p = 31 + l;
  r.mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
  r.shr = static_cast<uint32_t>(p - 32);
  return r;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t tc_quo(uint32_t x, const TcDiv& v) {
  return v.d == 1 ? x : (__umulhi(x, v.mul) >> v.shr);
}
#endif

struct TcUnit {
  int32_t ext;    // extent (product of member var extents)
  int32_t box;    // tile/block extent along this unit (1 for grid / loop units)
  int32_t src;    // TcSrc
  int32_t nv;     // member vars, innermost first
  int32_t vext[4];
  int64_t sc[4];  // out stride of each member var (0 for K units)
  TcDiv dbox, dtiles, dext, dvext[4];  // fast division by box, ceil(ext/box), ext, vext[k]
};

struct TcDim {    // one TMA coordinate
  int32_t u0, u1; // unit ids (-1 = none)
  int32_t c0, c1; // coefficients
  int32_t cst;
};

struct TcOperand {
  TcDim dim[5];
  int32_t mn_major;   // 0: K-major (box = 32 K x rows), 1: MN-major (nsub boxes of 32 MN x 32 K)
  int32_t nsub;       // TMA issues per stage
  int32_t stage_bytes;
  int32_t wide;       // MN-major loaded as ONE unswizzled [32 K rows][wbox MN] box (wbox <= 128)
  int32_t wbox;
};

struct TcParams {
  CUtensorMap ta;     // 64-byte aligned, first members
  CUtensorMap tb;
  CUtensorMap tc;     // C, for the TMA-store epilogue (c_tma != 0)
  TcOperand oa, ob;
  // TMA-store epilogue: each epilogue warp stages its 32-row x 32-column block of a chunk in
  // shared memory and one lane issues a bulk tensor store (or, for split-K / tail chunks, a
  // bulk tensor reduce-add) -- asynchronous full-line writes instead of per-thread stores.
  // c_tma: 0 off, 1 rows innermost in C (block staged column-major), 2 columns innermost
  // (row-major, 128B swizzle).  TMA dim d of C carries unit cdim_u[d] (-1 none) plus the
  // warp's row offset (cdim_q[d] == 1) or the chunk's column offset (cdim_q[d] == 2).
  int32_t c_tma;
  int32_t cdim_u[5], cdim_q[5];
  int32_t c_slab;     // rows of the outermost M unit per warp (its coordinate advances by q * c_slab)
  // c_wrap > 0: the single M unit is [inner vars chaining in C, flat extent c_wrap][outer vars]
  // (e.g. [w h][b] of an NCHW output, b not contiguous with h w): C dim cdim_q == 3 takes the
  // inner index and cdim_q == 4 the outer one; a warp's 32 rows that cross into the next outer
  // index are stored twice, the second box at inner coordinate - c_wrap (TMA clips both)
  int32_t c_wrap;
  int32_t acc_out;    // 1: every item adds into C (a 3xTF32 correction launch); no memset, no tail split
  TcUnit u[TC_MAX_UNITS];
  int32_t nunits;
  int32_t nm, mt[3];      // M-tile units, row order fastest first
  int32_t nn, nt[3];      // N-tile units, column order fastest first
  int32_t ng, gu[8];      // grid units
  int32_t nk, ku[6];      // K-loop units, fastest first
  int32_t m_rows;         // rows filled by A per tile (<= 128)
  int32_t n_cols;         // columns filled by B per tile (<= BN)
  int32_t n_mma;          // MMA N (multiple of 16)
  int32_t k_iters;        // K iterations in total
  int32_t k_split;        // CTAs along K (atomic epilogue when > 1)
  int32_t transpose_store;// stage through smem so lanes write consecutive columns
  uint32_t idesc;         // tcgen05 instruction descriptor
  int32_t tiles_m, tiles_n, grid_z;
  // K-loop odometer, precomputed on the host so the producer does no division:
  // coordinate[d] = base[d] + sum_i digit_i * kstep_{a,b}[i][d], digit_i < kcount[i]
  int32_t kcount[6];
  int32_t kstep_a[6][5], kstep_b[6][5];
  // carry deltas: coordinate change when digit i increments and every lower digit wraps to 0
  // (the producer advances its coordinates incrementally instead of re-deriving them)
  int32_t kdelta_a[6][5], kdelta_b[6][5];
  // MMAs (of K=8) issued for the last chunk of K digit 0 when it is the 32-wide K block of a
  // single unit whose extent is not a multiple of 32 (its tail rows are TMA zero fill); else 4
  int32_t ktail_kk;
  TcDiv dpm;       // ceil(tiles_m / cluster size): M tiles are dealt per work group
  TcDiv dtn;       // tiles_n
  TcDiv dsplit;    // pm * tiles_n * grid_z: work items per K split
  int32_t k_per;   // K iterations per split
  // Tail split (set per launch): the n_items work items are dealt in full rounds of ngroups;
  // the sk_r items of a partial last round are each cut into tl_s K chunks run by otherwise
  // idle groups -- chunk 0 stores, the others wait for its flag and add.  sk_r == 0: off.
  uint32_t n_items;  // work items of the full decomposition (tiles x K splits)
  uint32_t sk_full;  // items handled whole (a multiple of ngroups)
  uint32_t sk_r;     // tail items, each split into tl_s K chunks
  int32_t tl_s;      // K chunks per tail item
  uint32_t* tl_flags;// per tail item: chunks finished (chunk 0 first); zero between launches
  int32_t tl_zeroed; // 1: C was zeroed beforehand -- every tail chunk adds, no flag handshake
  int32_t tl_first;  // 1: a group runs its tail chunk before its whole items (the chunks' store /
                     // flag / add handshake then overlaps the whole items' mainloops)
  TcDiv dkit;        // k_iters
  // contiguous assignment (set per launch for many small tiles, no K split, no pairs):
  // group g takes items [g*ipg + min(g, rem), ...) in order, so the tile origins advance
  // incrementally instead of being re-decoded per tile
  int32_t contig;
  uint32_t ipg, irem;
  // 2-CTA cluster along M: each CTA TMA-loads mc_half rows of the B tile and multicasts
  // them to both CTAs (B is read from L2 once per CTA pair instead of once per CTA)
  int32_t mcast;           // 1: launched with cluster dims (2,1,1)
  int32_t mc_half;         // B rows loaded per CTA (multiple of 8)
  int32_t mc_ndim;         // TMA dim of B that carries the N tile
  int32_t native_mn;       // MN-major operands read by the MMA directly (no smem transpose)
  uint32_t mn_lbo16;       // MN-major smem descriptor: LBO >> 4 (next 32-MN box)
  uint32_t mn_desc_hi;     //   bits 32..63: SBO >> 4, version 1, layout type
  uint32_t mn_kstep16;     //   start-address advance per K=8 MMA, >> 4
  int32_t dbg;             // debug: bit0 skip MMAs, bit1 skip TMA loads (timing experiments only)
};

// Host-side plan: everything except the pointer-dependent tensor maps.
struct TcPlan {
  int valid = 0;
  int bn = 0;                 // template tile N (64 / 128 / 256)
  TcParams params{};          // maps filled at launch
  // tensor-map geometry per operand (innermost first)
  int rank_a = 0, rank_b = 0;
  uint64_t gdim_a[5]{}, gdim_b[5]{};
  uint64_t gstride_a[5]{}, gstride_b[5]{};  // bytes, [0] unused
  uint32_t box_a[5]{}, box_b[5]{};
  int swz_a = 3, swz_b = 3;   // CUtensorMapSwizzle: 3 128B (K-major), 4 128B_ATOM_32B (native MN-major), 0 none (wide)
  // C tensor map geometry for the TMA-store epilogue (params.c_tma != 0)
  uint64_t gdim_c[5]{}, gstride_c[5]{};
  uint32_t box_c[5]{};
  int swz_c = 0;
  const void* cached_c = nullptr;
  int64_t out_span = 0;       // elements of C to zero before a split-K launch
  uint32_t* tail_flags = nullptr;  // kTailFlags zeroed words owned by the executor (tail split)
  int accum = 0;                   // add into C instead of storing (3xTF32 correction terms)
  int zeroed = 0;                  // split-K: C is zeroed by a separate (earlier) executor step
  int sm_budget = 0;               // > 0: SMs this launch may occupy (it co-runs with a sibling step)
  int tail_zeroed = 0;             // the executor zeroes C before the launch (tail chunks all add)
  const void* cached_a = nullptr;
  const void* cached_b = nullptr;
  const char* why = "";       // reason when not valid (diagnostics)
};

// Decides whether a lowered problem maps onto the tcgen05 kernel and fills the plan.
bool ce_tc_plan(const CeProblem& p, TcPlan* out);
// Whether the launch of this plan will split a partial last round into K chunks (tail split,
// see ce_tc.cu) on the current device -- the executor then zeroes C beforehand.
bool ce_tc_tail_split(const TcPlan& plan);
cudaError_t ce_launch_tc(TcPlan& plan, const float* A, const float* B, float* C, cudaStream_t s);
