// SIMT kernel families for the generalized pairwise step (see ce_device.h).
//
//  * ce_direct_kernel — one thread per output element, odometer over the K
//    vars.  Used where K is tiny (depthwise / batch-only convolutions such as
//    CP's `bhwr,rh->bhwr`, Hadamard and outer products),
//    for unary steps (sum_unique_modes kernels.cpp:144-187, broadcast of its
//    adjoint, permutes) and as the universal fallback for any index map
//    (Circular wrap, >2 conv axes).  HBM-bound by construction.
//  * ce_tiled_kernel — 64x64x16 shared-memory tiled FP32 gather-GEMM for large-K
//    steps the tensor-core path does not take (anchor + fallback of family a/b1).
//  * ce_fill_kernel — SplitMix64 (reference tensor.cpp:107-130) in closed form.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <numeric>
#include <cstdlib>
#include <vector>
#include <cstdio>
#include <cstring>

#include "ce_device.h"
#include "ce_kernels.h"
#include "ce_launch.h"
#include "ce_tc.h"  // TcDiv fast division

namespace {

bool simt_stream_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CE_SIMT_STREAM");
    return !(e && *e == '0');
  }();
  return on;
}

__device__ __forceinline__ bool gather_index(const CeGather& g, int64_t p, int64_t q, int64_t* off) {
  int64_t x = g.sp * p + g.sq * q + g.c;
  if (g.wrap) {
    x %= g.extent;
    if (x < 0) x += g.extent;
  } else if (x < 0 || x >= g.extent) {
    return false;
  }
  *off = x * g.stride;
  return true;
}

// ----------------------------------------------------------------------------- direct
__global__ void __launch_bounds__(256) ce_direct_kernel(const CeSimtDesc d, const float* __restrict__ A,
                                                        const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  const CeProblem& p = d.p;
  const int64_t total = d.Z * d.M * d.N;
  for (int64_t flat = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; flat < total;
       flat += (int64_t)gridDim.x * blockDim.x) {
    int64_t val[CE_MAX_VARS];
    int64_t rest = flat, offA = 0, offB = 0, offC = 0;
    for (int i = 0; i < d.nout; ++i) {
      const int v = d.ov[i];
      const int64_t e = p.ext[v];
      val[v] = rest % e;
      rest /= e;
      offA += val[v] * p.sa[v];
      offB += val[v] * p.sb[v];
      offC += val[v] * p.sc[v];
    }
    for (int i = 0; i < d.nk; ++i) val[d.kv[i]] = 0;
    float acc = 0.f;
    int64_t kA = 0, kB = 0;
    for (int64_t k = 0; k < d.K; ++k) {
      int64_t a_off = offA + kA, b_off = offB + kB;
      bool ok = true;
      for (int g = 0; g < p.ng_a && ok; ++g) {
        int64_t o;
        ok = gather_index(p.ga[g], val[p.ga[g].pv], val[p.ga[g].qv], &o);
        a_off += o;
      }
      for (int g = 0; g < p.ng_b && ok; ++g) {
        int64_t o;
        ok = gather_index(p.gb[g], val[p.gb[g].pv], val[p.gb[g].qv], &o);
        b_off += o;
      }
      if (ok) acc += p.unary ? __ldg(A + a_off) : __ldg(A + a_off) * __ldg(B + b_off);
      // odometer over K vars (first var fastest)
      for (int i = 0; i < d.nk; ++i) {
        const int v = d.kv[i];
        if (++val[v] < p.ext[v]) {
          kA += p.sa[v];
          kB += p.sb[v];
          break;
        }
        kA -= (p.ext[v] - 1) * p.sa[v];
        kB -= (p.ext[v] - 1) * p.sb[v];
        val[v] = 0;
      }
    }
    if (p.accumulate)
      C[offC] += acc;
    else
      C[offC] = acc;
  }
}

// ----------------------------------------------------------------------------- reduce
// Few outputs, long K (e.g. the depthwise filter gradient of CP's `bhwr,rh->bhwr`:
// 48 outputs x 8192 terms): one CTA per (output, K split), 256 threads stride
// the K range, warp-shuffle + smem tree reduction, one atomicAdd per CTA when split.
__global__ void __launch_bounds__(256) ce_reduce_kernel(const CeSimtDesc d, const float* __restrict__ A,
                                                        const float* __restrict__ B, float* __restrict__ C,
                                                        int64_t k_per_split) {
  ce_pdl_enter();
  const CeProblem& p = d.p;
  __shared__ float warp_sum[8];
  int64_t val[CE_MAX_VARS];
  int64_t rest = blockIdx.x, offA = 0, offB = 0, offC = 0;
  for (int i = 0; i < d.nout; ++i) {
    const int v = d.ov[i];
    const int64_t e = p.ext[v];
    val[v] = rest % e;
    rest /= e;
    offA += val[v] * p.sa[v];
    offB += val[v] * p.sb[v];
    offC += val[v] * p.sc[v];
  }
  const int64_t k_begin = blockIdx.y * k_per_split;
  const int64_t k_end = min(d.K, k_begin + k_per_split);
  float acc = 0.f;
  for (int64_t k = k_begin + threadIdx.x; k < k_end; k += blockDim.x) {
    int64_t r = k, a_off = offA, b_off = offB;
    for (int i = 0; i < d.nk; ++i) {
      const int v = d.kv[i];
      val[v] = r % p.ext[v];
      r /= p.ext[v];
      a_off += val[v] * p.sa[v];
      b_off += val[v] * p.sb[v];
    }
    bool ok = true;
    for (int g = 0; g < p.ng_a && ok; ++g) {
      int64_t o;
      ok = gather_index(p.ga[g], val[p.ga[g].pv], val[p.ga[g].qv], &o);
      a_off += o;
    }
    for (int g = 0; g < p.ng_b && ok; ++g) {
      int64_t o;
      ok = gather_index(p.gb[g], val[p.gb[g].pv], val[p.gb[g].qv], &o);
      b_off += o;
    }
    if (ok) acc += p.unary ? __ldg(A + a_off) : __ldg(A + a_off) * __ldg(B + b_off);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? warp_sum[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) {
      if (gridDim.y > 1 || p.accumulate)
        atomicAdd(C + offC, acc);
      else
        C[offC] = acc;
    }
  }
}


// ----------------------------------------------------------------------------- stream
// Streaming SIMT kernel for small-K steps (depthwise / batch-only convolutions, Hadamard
// and outer products, unary sums and broadcasts) and few-output long-K reductions (the
// depthwise filter gradients): one thread per output element and K slice, with all index
// state in 32-bit registers.  The host orders the output vars so that the lane var is
// unit-stride in the streamed operand (coalesced 128-B warp accesses), replaces every
// division by a multiply-shift (TcDiv) and rewrites each gathered (convolution) index
// idx = sp*p + sq*q + c as an affine function of the output and K var values that the
// K odometer updates incrementally.  A K slice > 1 accumulates with atomics into C.
constexpr int SV_O = 8, SV_K = 6, SV_G = 2;
struct SvDesc {
  int32_t nout, nk, nga, ngb, unary, mode;  // mode 0 store, 1 accumulate, 2 atomic
  int32_t vec, vec_b, vec_c;                // VEC=4 path (see ce_stream_kernel)
  int32_t lext;                             // lane var extent (VEC=4: the last group may be partial)
  int32_t klane;                            // 1: warp per output, lanes along K
  int32_t a_bcast;                          // VEC=4 with A independent of the lane var
  int32_t jrep, l1ext;                      // output slot 1 values per thread, slot 1 extent
  int32_t g_inv1, b_inv1, bfix1;            // gathers / B / B and its gathers independent of slot 1
  int32_t stencil;                          // depthwise stencil path: taps (0 = off)
  int32_t dwgrad;                           // depthwise filter-gradient path: taps (0 = off)
  int32_t oext[SV_O];
  TcDiv odiv[SV_O];
  int32_t osa[SV_O], osb[SV_O], osc[SV_O];
  int32_t kext[SV_K];
  TcDiv kdiv[SV_K];
  int32_t ksa[SV_K], ksb[SV_K];
  // gathers, compacted: g < ng, on operand gop[g] (0 = A, 1 = B)
  int32_t ng, gop[2 * SV_G];
  int32_t gc[2 * SV_G], gext[2 * SV_G], gstride[2 * SV_G], gwrap[2 * SV_G];
  int32_t go[2 * SV_G][SV_O];  // coefficient of output slot i in the gathered index
  int32_t gk[2 * SV_G][SV_K];  // coefficient of K slot j
  uint32_t outs, K, kper;
};

__device__ __forceinline__ int32_t sv_mod(int32_t x, int32_t e) {
  const int32_t r = x % e;
  return r < 0 ? r + e : r;
}

// VEC = 4: each thread owns 4 consecutive values of the lane var (slot 0, unit stride and
// 16-B aligned in A, never gathered), loading A as float4; B and C use float4 when they
// are unit-stride along the lane var too (flags set by the host), else 4 scalars.
template <int VEC, int NG>
__global__ void __launch_bounds__(256) ce_stream_kernel(const SvDesc d, const float* __restrict__ A,
                                                        const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  const uint32_t o = blockIdx.x * 256u + threadIdx.x;
  if (o >= d.outs) return;  // outs counts threads (lane var / VEC, slot 1 / jrep)
  // ---- output index decoding, once per thread
  int32_t offA = 0, offB = 0, offC = 0, lane0 = 0, lane1 = 0;
  int32_t gidx0[NG > 0 ? NG : 1];
#pragma unroll
  for (int g = 0; g < NG; ++g) gidx0[g] = d.gc[g];
  uint32_t rest = o;
#pragma unroll
  for (int i = 0; i < SV_O; ++i) {
    if (i < d.nout) {
      const uint32_t q = tc_quo(rest, d.odiv[i]);
      int32_t v = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.oext[i]));
      rest = q;
      if (i == 0) {
        v *= VEC;
        lane0 = v;
      } else if (i == 1) {
        v *= d.jrep;
        lane1 = v;
      }
      offA += v * d.osa[i];
      offB += v * d.osb[i];
      offC += v * d.osc[i];
#pragma unroll
      for (int g = 0; g < NG; ++g) gidx0[g] += v * d.go[g][i];
    }
  }
  // ---- K slice start, once per thread
  const uint32_t k0 = blockIdx.y * d.kper;
  const uint32_t k1 = min(d.K, k0 + d.kper);
  int32_t kv0[SV_K];
  rest = k0;
#pragma unroll
  for (int j = 0; j < SV_K; ++j) {
    kv0[j] = 0;
    if (j < d.nk) {
      const uint32_t q = tc_quo(rest, d.kdiv[j]);
      kv0[j] = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.kext[j]));
      rest = q;
      offA += kv0[j] * d.ksa[j];
      offB += kv0[j] * d.ksb[j];
#pragma unroll
      for (int g = 0; g < NG; ++g) gidx0[g] += kv0[j] * d.gk[g][j];
    }
  }
  const int32_t sb0 = d.osb[0];
  const int32_t sa1 = d.nout > 1 ? d.osa[1] : 0, sb1 = d.nout > 1 ? d.osb[1] : 0, sc1 = d.nout > 1 ? d.osc[1] : 0;
  // ---- jrep consecutive values of output slot 1 per thread (amortises the decoding)
  for (int jj = 0; jj < d.jrep; ++jj) {
    if (jj > 0 && lane1 + jj >= d.l1ext) break;
    int32_t pa = offA + jj * sa1, pb = offB + jj * sb1;
    int32_t gidx[NG > 0 ? NG : 1];
#pragma unroll
    for (int g = 0; g < NG; ++g) gidx[g] = gidx0[g] + jj * (d.nout > 1 ? d.go[g][1] : 0);
    int32_t kv[SV_K];
#pragma unroll
    for (int j = 0; j < SV_K; ++j) kv[j] = kv0[j];
    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
    for (uint32_t k = k0; k < k1; ++k) {
      int32_t a = pa, b = pb;
      bool ok = true;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        int32_t x = gidx[g];
        if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
        ok = ok && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
        if (d.gop[g])
          b += x * d.gstride[g];
        else
          a += x * d.gstride[g];
      }
      if (ok) {
        if (VEC == 1) {
          acc[0] += d.unary ? __ldg(A + a) : __ldg(A + a) * __ldg(B + b);
        } else {
          float xa[4];
          if (d.a_bcast) {
            xa[0] = xa[1] = xa[2] = xa[3] = __ldg(A + a);
          } else {
            const float4 va = __ldg(reinterpret_cast<const float4*>(A + a));
            xa[0] = va.x;
            xa[1] = va.y;
            xa[2] = va.z;
            xa[3] = va.w;
          }
          if (d.unary) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] += xa[e];
          } else if (d.vec_b) {
            const float4 vb = __ldg(reinterpret_cast<const float4*>(B + b));
            acc[0] += xa[0] * vb.x;
            acc[1] += xa[1] * vb.y;
            acc[2] += xa[2] * vb.z;
            acc[3] += xa[3] * vb.w;
          } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (lane0 + e < d.lext) acc[e] += xa[e] * __ldg(B + b + e * sb0);
          }
        }
      }
      // K odometer (slot 0 fastest); the gathered indices move with it
#pragma unroll
      for (int j = 0; j < SV_K; ++j) {
        if (j < d.nk) {
          if (++kv[j] < d.kext[j]) {
            pa += d.ksa[j];
            pb += d.ksb[j];
#pragma unroll
            for (int g = 0; g < NG; ++g) gidx[g] += d.gk[g][j];
            break;
          }
          const int32_t back = d.kext[j] - 1;
          pa -= back * d.ksa[j];
          pb -= back * d.ksb[j];
#pragma unroll
          for (int g = 0; g < NG; ++g) gidx[g] -= back * d.gk[g][j];
          kv[j] = 0;
        }
      }
    }
    const int32_t pc = offC + jj * sc1;
    if (VEC == 4 && d.vec_c) {
      float4* cp = reinterpret_cast<float4*>(C + pc);
      const float4 v = make_float4(acc[0], acc[1], acc[2], acc[VEC - 1]);
      if (d.mode == 2) {
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(cp), "f"(v.x), "f"(v.y),
                     "f"(v.z), "f"(v.w)
                     : "memory");
      } else if (d.mode == 1) {
        float4 c = *cp;
        c.x += v.x;
        c.y += v.y;
        c.z += v.z;
        c.w += v.w;
        *cp = c;
      } else {
        *cp = v;
      }
    } else {
      const int32_t sc0 = d.osc[0];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        if (VEC > 1 && lane0 + e >= d.lext) break;
        float* cp = C + pc + e * sc0;
        if (d.mode == 2)
          atomicAdd(cp, acc[e]);
        else if (d.mode == 1)
          *cp += acc[e];
        else
          *cp = acc[e];
      }
    }
  }
}


__device__ __forceinline__ void xa4(const SvDesc& d, const float* p, float (&xa)[4]) {
  if (d.a_bcast) {
    xa[0] = xa[1] = xa[2] = xa[3] = __ldg(p);
  } else {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    xa[0] = v.x;
    xa[1] = v.y;
    xa[2] = v.z;
    xa[3] = v.w;
  }
}
__device__ __forceinline__ void xb4(const SvDesc& d, const float* p, bool full0, int32_t lane0, float (&xb)[4]) {
  if (d.vec_b) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    xb[0] = v.x;
    xb[1] = v.y;
    xb[2] = v.z;
    xb[3] = v.w;
  } else if (full0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) xb[e] = __ldg(p + e * d.osb[0]);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) xb[e] = lane0 + e < d.lext ? __ldg(p + e * d.osb[0]) : 0.f;
  }
}

// Register-blocked VEC=4 variant: a thread owns 4 lane values x 4 consecutive values of
// output slot 1; per K term the B vector is loaded once (when it does not depend on slot 1,
// e.g. the depthwise factor F[r, k]) and reused for the 4 slot-1 outputs, so a 3-tap
// stencil costs ~1 float4 load + 4 FMAs per 4 outputs instead of a full index walk.
template <int NG>
__global__ void __launch_bounds__(256) ce_stream_blk_kernel(const SvDesc d, const float* __restrict__ A,
                                                            const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  constexpr int J = 4;
  const uint32_t o = blockIdx.x * 256u + threadIdx.x;
  if (o >= d.outs) return;
  int32_t offA = 0, offB = 0, offC = 0, lane0 = 0, lane1 = 0;
  int32_t gidx[NG > 0 ? NG : 1];
#pragma unroll
  for (int g = 0; g < NG; ++g) gidx[g] = d.gc[g];
  uint32_t rest = o;
#pragma unroll
  for (int i = 0; i < SV_O; ++i) {
    if (i < d.nout) {
      const uint32_t q = tc_quo(rest, d.odiv[i]);
      int32_t v = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.oext[i]));
      rest = q;
      if (i == 0) {
        v *= 4;
        lane0 = v;
      } else if (i == 1) {
        v *= J;
        lane1 = v;
      }
      offA += v * d.osa[i];
      offB += v * d.osb[i];
      offC += v * d.osc[i];
#pragma unroll
      for (int g = 0; g < NG; ++g) gidx[g] += v * d.go[g][i];
    }
  }
  const uint32_t k0 = blockIdx.y * d.kper;
  const uint32_t k1 = min(d.K, k0 + d.kper);
  int32_t kv[SV_K];
  rest = k0;
#pragma unroll
  for (int j = 0; j < SV_K; ++j) {
    kv[j] = 0;
    if (j < d.nk) {
      const uint32_t q = tc_quo(rest, d.kdiv[j]);
      kv[j] = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.kext[j]));
      rest = q;
      offA += kv[j] * d.ksa[j];
      offB += kv[j] * d.ksb[j];
#pragma unroll
      for (int g = 0; g < NG; ++g) gidx[g] += kv[j] * d.gk[g][j];
    }
  }
  const int32_t sa1 = d.osa[1], sb1 = d.osb[1];
  const bool full0 = lane0 + 4 <= d.lext;
  int nj = d.l1ext - lane1;
  nj = nj < J ? nj : J;
  float acc[J][4];
#pragma unroll
  for (int jj = 0; jj < J; ++jj)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[jj][e] = 0.f;
  for (uint32_t k = k0; k < k1; ++k) {
    if (d.g_inv1) {
      // gathers and B independent of slot 1: one validity test and one B vector per term
      int32_t a = offA, b = offB;
      bool ok = true;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        int32_t x = gidx[g];
        if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
        ok = ok && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
        if (d.gop[g])
          b += x * d.gstride[g];
        else
          a += x * d.gstride[g];
      }
      if (ok) {
        float xb[4] = {1.f, 1.f, 1.f, 1.f};
        if (!d.unary && d.b_inv1) xb4(d, B + b, full0, lane0, xb);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          if (jj >= nj) break;
          float xa[4];
          xa4(d, A + a + jj * sa1, xa);
          if (!d.unary && !d.b_inv1) xb4(d, B + b + jj * sb1, full0, lane0, xb);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[jj][e] += xa[e] * xb[e];
        }
      }
    } else if (d.bfix1) {
      // B (and its gathers) independent of slot 1, only A's gathers move with it (the
      // depthwise filter gradient: dY[b,h,w,r] shared by the taps of X[b,h+kh-1,w,r])
      int32_t b = offB;
      bool okb = true;
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        if (!d.gop[g]) continue;
        int32_t x = gidx[g];
        if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
        okb = okb && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
        b += x * d.gstride[g];
      }
      if (okb) {
        float xb[4] = {1.f, 1.f, 1.f, 1.f};
        if (!d.unary) xb4(d, B + b, full0, lane0, xb);
#pragma unroll
        for (int jj = 0; jj < J; ++jj) {
          if (jj >= nj) break;
          int32_t a = offA + jj * sa1;
          bool ok = true;
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            if (d.gop[g]) continue;
            int32_t x = gidx[g] + jj * d.go[g][1];
            if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
            ok = ok && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
            a += x * d.gstride[g];
          }
          if (!ok) continue;
          float xa[4];
          xa4(d, A + a, xa);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[jj][e] += xa[e] * xb[e];
        }
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        if (jj >= nj) break;
        int32_t a = offA + jj * sa1, b = offB + jj * sb1;
        bool ok = true;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          int32_t x = gidx[g] + jj * d.go[g][1];
          if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
          ok = ok && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
          if (d.gop[g])
            b += x * d.gstride[g];
          else
            a += x * d.gstride[g];
        }
        if (!ok) continue;
        float xa[4], xb[4] = {1.f, 1.f, 1.f, 1.f};
        xa4(d, A + a, xa);
        if (!d.unary) xb4(d, B + b, full0, lane0, xb);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[jj][e] += xa[e] * xb[e];
      }
    }
    // K odometer
#pragma unroll
    for (int j = 0; j < SV_K; ++j) {
      if (j < d.nk) {
        if (++kv[j] < d.kext[j]) {
          offA += d.ksa[j];
          offB += d.ksb[j];
#pragma unroll
          for (int g = 0; g < NG; ++g) gidx[g] += d.gk[g][j];
          break;
        }
        const int32_t back = d.kext[j] - 1;
        offA -= back * d.ksa[j];
        offB -= back * d.ksb[j];
#pragma unroll
        for (int g = 0; g < NG; ++g) gidx[g] -= back * d.gk[g][j];
        kv[j] = 0;
      }
    }
  }
  const int32_t sc1 = d.osc[1], sc0 = d.osc[0];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    if (jj >= nj) break;
    const int32_t pc = offC + jj * sc1;
    if (d.vec_c) {
      float4* cp = reinterpret_cast<float4*>(C + pc);
      const float4 v = make_float4(acc[jj][0], acc[jj][1], acc[jj][2], acc[jj][3]);
      if (d.mode == 2) {
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(cp), "f"(v.x), "f"(v.y),
                     "f"(v.z), "f"(v.w)
                     : "memory");
      } else if (d.mode == 1) {
        float4 c = *cp;
        c.x += v.x;
        c.y += v.y;
        c.z += v.z;
        c.w += v.w;
        *cp = c;
      } else {
        *cp = v;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (lane0 + e >= d.lext) break;
        float* cp = C + pc + e * sc0;
        if (d.mode == 2)
          atomicAdd(cp, acc[jj][e]);
        else if (d.mode == 1)
          *cp += acc[jj][e];
        else
          *cp = acc[jj][e];
      }
    }
  }
}


// Depthwise 1-D stencil (CP's `bhwr,rh->bhwr` family and its input-gradient adjoint):
// one gathered A axis x = gc + SA*p + SB*q over the conv output var p (slot 1) and the tap
// q (the only K var), B = F[lane, q].  A thread owns 4 lanes x J consecutive p: the
// J+KT-1 input rows of its window are loaded once into registers (float4) and reused by
// every tap -- a register sliding window instead of KT loads per output.
template <int KT, int J, int SA, int SB>
__global__ void __launch_bounds__(256) ce_dw_kernel(const SvDesc d, const float* __restrict__ A,
                                                    const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  const uint32_t o = blockIdx.x * 256u + threadIdx.x;
  if (o >= d.outs) return;
  int32_t offA = 0, offB = 0, offC = 0, lane0 = 0, p0 = 0;
  int32_t x00 = d.gc[0];
  uint32_t rest = o;
#pragma unroll
  for (int i = 0; i < SV_O; ++i) {
    if (i < d.nout) {
      const uint32_t q = tc_quo(rest, d.odiv[i]);
      int32_t v = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.oext[i]));
      rest = q;
      if (i == 0) {
        v *= 4;
        lane0 = v;
      } else if (i == 1) {
        v *= J;
        p0 = v;
      }
      offA += v * d.osa[i];
      offB += v * d.osb[i];
      offC += v * d.osc[i];
      x00 += v * d.go[0][i];
    }
  }
  // taps of this thread's 4 lanes
  float bq[KT][4];
  const float* pb = B + offB;
  const int32_t sb0 = d.osb[0], ksb = d.ksb[0];
#pragma unroll
  for (int q = 0; q < KT; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) bq[q][e] = lane0 + e < d.lext ? __ldg(pb + q * ksb + e * sb0) : 0.f;
  // window rows t = SA*jj + SB*q in [TMIN, TMAX]
  constexpr int TMIN = (SA > 0 ? 0 : -(J - 1)) + (SB > 0 ? 0 : -(KT - 1));
  constexpr int NW = J + KT - 1;
  float4 rw[NW];
  const int32_t gext = d.gext[0], gstr = d.gstride[0];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int32_t x = x00 + TMIN + w;
    if (static_cast<uint32_t>(x) < static_cast<uint32_t>(gext)) {
      const float* pa = A + offA + x * gstr;
      if (d.a_bcast) {
        const float v = __ldg(pa);
        rw[w] = make_float4(v, v, v, v);
      } else {
        rw[w] = __ldg(reinterpret_cast<const float4*>(pa));
      }
    } else {
      rw[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const int32_t sc1 = d.osc[1], sc0 = d.osc[0];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) {
    if (p0 + jj >= d.l1ext) break;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      const float4 r = rw[SA * jj + SB * q - TMIN];
      a0 += r.x * bq[q][0];
      a1 += r.y * bq[q][1];
      a2 += r.z * bq[q][2];
      a3 += r.w * bq[q][3];
    }
    const int32_t pc = offC + jj * sc1;
    if (d.vec_c) {
      float4* cp = reinterpret_cast<float4*>(C + pc);
      if (d.mode == 1) {
        float4 c = *cp;
        *cp = make_float4(c.x + a0, c.y + a1, c.z + a2, c.w + a3);
      } else {
        *cp = make_float4(a0, a1, a2, a3);
      }
    } else {
      const float av[4] = {a0, a1, a2, a3};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (lane0 + e >= d.lext) break;
        float* cp = C + pc + e * sc0;
        if (d.mode == 1)
          *cp += av[e];
        else
          *cp = av[e];
      }
    }
  }
}


// Depthwise filter gradient (the reduce adjoint of the stencil): dF[lane, q] =
// sum_k A[.., x = gc + SA*p + SB*q, .., lane] * B[.., p, .., lane] with p (the gathered
// K var) fastest.  A thread owns 4 lanes x all KT taps over a K slice; the KT rows of A
// live in a register window that shifts by one row per p step (4 steps' loads issued
// together), so a K step costs one float4 of A, one of B and 4*KT FMAs.  Threads map
// lane groups fastest (coalesced) then K slices; slices add atomically.
template <int KT, int SA, int SB>
__global__ void __launch_bounds__(256) ce_dwgrad_kernel(const SvDesc d, const float* __restrict__ A,
                                                        const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  // few lane quads (outs <= 256): the K slices of one CTA are first summed in shared memory
  // (block-scope atomics), then one global atomic per (CTA, output) -- so the K range can be
  // cut into enough slices to fill the GPU without every slice contending on the same words
  __shared__ float sred[256 * KT * 4];
  const bool cta_red = d.mode == 2 && d.outs <= 256;
  if (cta_red) {
    for (int i = threadIdx.x; i < static_cast<int>(d.outs) * KT * 4; i += 256) sred[i] = 0.f;
    __syncthreads();
  }
  const uint32_t t = blockIdx.x * 256u + threadIdx.x;
  const uint32_t nslices = (d.K + d.kper - 1) / d.kper;
  const bool live = t < d.outs * nslices;
  const uint32_t slice = tc_quo(live ? t : 0u, d.odiv[0]);
  const uint32_t o = (live ? t : 0u) - slice * d.outs;
  const int32_t lane0 = static_cast<int32_t>(o) * 4;
  const uint32_t k0 = slice * d.kper;
  const uint32_t k1 = live ? min(d.K, k0 + d.kper) : k0;
  int32_t kv[SV_K];
  int32_t offAk = 0, offBk = 0;
  uint32_t rest = k0;
#pragma unroll
  for (int j = 0; j < SV_K; ++j) {
    kv[j] = 0;
    if (j < d.nk) {
      const uint32_t q = tc_quo(rest, d.kdiv[j]);
      kv[j] = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.kext[j]));
      rest = q;
      if (j > 0) {
        offAk += kv[j] * d.ksa[j];
        offBk += kv[j] * d.ksb[j];
      }
    }
  }
  const int32_t gext = d.gext[0], gstr = d.gstride[0], gc = d.gc[0], ext0 = d.kext[0], ksb0 = d.ksb[0];
  const float* Al = A + lane0 * d.osa[0];
  const float* Bl = B + lane0 * d.osb[0];
  const bool full4 = lane0 + 4 <= d.lext;
  const int32_t sb0 = d.osb[0];
  auto row = [&](int32_t x) -> float4 {
    if (static_cast<uint32_t>(x) >= static_cast<uint32_t>(gext)) return make_float4(0.f, 0.f, 0.f, 0.f);
    return __ldg(reinterpret_cast<const float4*>(Al + offAk + x * gstr));
  };
  auto brow = [&](int32_t pp) -> float4 {
    const float* pb = Bl + offBk + pp * ksb0;
    if (d.vec_b) return __ldg(reinterpret_cast<const float4*>(pb));
    float4 b;
    b.x = __ldg(pb);
    b.y = full4 || lane0 + 1 < d.lext ? __ldg(pb + sb0) : 0.f;
    b.z = full4 || lane0 + 2 < d.lext ? __ldg(pb + 2 * sb0) : 0.f;
    b.w = full4 || lane0 + 3 < d.lext ? __ldg(pb + 3 * sb0) : 0.f;
    return b;
  };
  // the row entering the window at step p (SA == SB: the last tap's row, else the first)
  auto enter_x = [&](int32_t pp) { return SA == SB ? gc + SA * pp + SB * (KT - 1) : gc + SA * pp; };
  float4 w[KT];
  float acc[KT][4];
#pragma unroll
  for (int q = 0; q < KT; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[q][e] = 0.f;
  auto fma_step = [&](const float4& b) {
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      acc[q][0] += w[q].x * b.x;
      acc[q][1] += w[q].y * b.y;
      acc[q][2] += w[q].z * b.z;
      acc[q][3] += w[q].w * b.w;
    }
  };
  auto shift_in = [&](const float4& nr) {
    if (SA == SB) {
#pragma unroll
      for (int q = 0; q + 1 < KT; ++q) w[q] = w[q + 1];
      w[KT - 1] = nr;
    } else {
#pragma unroll
      for (int q = KT - 1; q > 0; --q) w[q] = w[q - 1];
      w[0] = nr;
    }
  };
  uint32_t k = k0;
  while (k < k1) {
    // a run of consecutive p without a carry into the other K vars
    const int32_t p = kv[0];
    const int32_t run = min(static_cast<int32_t>(k1 - k), ext0 - p);
#pragma unroll
    for (int q = 0; q < KT; ++q) w[q] = row(gc + SA * p + SB * q);
    int32_t j = 0;
    for (; j + 4 <= run; j += 4) {
      float4 bb[4], nr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bb[u] = brow(p + j + u);
        nr[u] = row(enter_x(p + j + u + 1));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        fma_step(bb[u]);
        shift_in(nr[u]);
      }
    }
    for (; j < run; ++j) {
      const float4 b = brow(p + j);
      const float4 nr = row(enter_x(p + j + 1));
      fma_step(b);
      shift_in(nr);
    }
    k += static_cast<uint32_t>(run);
    kv[0] = p + run;
    if (kv[0] >= ext0) {
      kv[0] = 0;
#pragma unroll
      for (int jj = 1; jj < SV_K; ++jj) {
        if (jj < d.nk) {
          if (++kv[jj] < d.kext[jj]) {
            offAk += d.ksa[jj];
            offBk += d.ksb[jj];
            break;
          }
          const int32_t back = d.kext[jj] - 1;
          offAk -= back * d.ksa[jj];
          offBk -= back * d.ksb[jj];
          kv[jj] = 0;
        }
      }
    }
  }
  const int32_t sc0 = d.osc[0], sc1 = d.osc[1];
  if (cta_red) {
    if (live)
#pragma unroll
      for (int q = 0; q < KT; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) atomicAdd_block(&sred[(o * KT + q) * 4 + e], acc[q][e]);
    __syncthreads();
    // the CTA's outputs: quads present in it (all of them once it spans >= outs threads)
    for (int i = threadIdx.x; i < static_cast<int>(d.outs) * KT * 4; i += 256) {
      const int e = i & 3, q = (i >> 2) % KT, oq = (i >> 2) / KT;
      if (oq * 4 + e < d.lext && sred[i] != 0.f) atomicAdd(C + (oq * 4 + e) * sc0 + q * sc1, sred[i]);
    }
    return;
  }
  if (!live) return;
  const int32_t offC = lane0 * d.osc[0];
#pragma unroll
  for (int q = 0; q < KT; ++q)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (lane0 + e >= d.lext) break;
      float* cp = C + offC + q * sc1 + e * sc0;
      if (d.mode == 2)
        atomicAdd(cp, acc[q][e]);
      else if (d.mode == 1)
        *cp += acc[q][e];
      else
        *cp = acc[q][e];
    }
}

// K-lane mode: a warp per output, lanes striding the K range (for steps whose streamed
// operand is contiguous along a K var, e.g. the input gradient of RTR's first node:
// 900 contiguous terms per output), combined with a warp-shuffle tree.
template <int NG>
__global__ void __launch_bounds__(256) ce_stream_klane_kernel(const SvDesc d, const float* __restrict__ A,
                                                              const float* __restrict__ B, float* __restrict__ C) {
  ce_pdl_enter();
  const uint32_t o = blockIdx.x * 8u + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o >= d.outs) return;  // warp-uniform
  int32_t offA = 0, offB = 0, offC = 0;
  int32_t gbase[NG > 0 ? NG : 1];
#pragma unroll
  for (int g = 0; g < NG; ++g) gbase[g] = d.gc[g];
  uint32_t rest = o;
#pragma unroll
  for (int i = 0; i < SV_O; ++i) {
    if (i < d.nout) {
      const uint32_t q = tc_quo(rest, d.odiv[i]);
      const int32_t v = static_cast<int32_t>(rest - q * static_cast<uint32_t>(d.oext[i]));
      rest = q;
      offA += v * d.osa[i];
      offB += v * d.osb[i];
      offC += v * d.osc[i];
#pragma unroll
      for (int g = 0; g < NG; ++g) gbase[g] += v * d.go[g][i];
    }
  }
  const uint32_t k0 = blockIdx.y * d.kper;
  const uint32_t k1 = min(d.K, k0 + d.kper);
  float acc = 0.f;
  for (uint32_t k = k0 + lane; k < k1; k += 32) {
    int32_t a = offA, b = offB;
    int32_t gidx[NG > 0 ? NG : 1];
#pragma unroll
    for (int g = 0; g < NG; ++g) gidx[g] = gbase[g];
    uint32_t r = k;
#pragma unroll
    for (int j = 0; j < SV_K; ++j) {
      if (j < d.nk) {
        const uint32_t q = tc_quo(r, d.kdiv[j]);
        const int32_t v = static_cast<int32_t>(r - q * static_cast<uint32_t>(d.kext[j]));
        r = q;
        a += v * d.ksa[j];
        b += v * d.ksb[j];
#pragma unroll
        for (int g = 0; g < NG; ++g) gidx[g] += v * d.gk[g][j];
      }
    }
    bool ok = true;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      int32_t x = gidx[g];
      if (d.gwrap[g]) x = sv_mod(x, d.gext[g]);
      ok = ok && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.gext[g]);
      if (d.gop[g])
        b += x * d.gstride[g];
      else
        a += x * d.gstride[g];
    }
    if (ok) acc += d.unary ? __ldg(A + a) : __ldg(A + a) * __ldg(B + b);
  }
#pragma unroll
  for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (lane == 0) {
    if (d.mode == 2)
      atomicAdd(C + offC, acc);
    else if (d.mode == 1)
      C[offC] += acc;
    else
      C[offC] = acc;
  }
}

// Builds the stream descriptor; false when the problem exceeds its limits (then the
// int64 reference kernels run).  *span = elements of C an atomic reduction must zero.
bool sv_build(const CeSimtDesc& sd, const float* A, const float* B, const float* C, SvDesc* out, int64_t* span,
              const char** why = nullptr) {
  auto fail = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  // merge vars that are contiguous in every operand (same role, not gathered): fewer
  // index digits per thread and longer lane runs (e.g. RTR's (r3)(r0) output pair)
  CeProblem p = sd.p;
  auto gathered = [&](int v) {
    for (int g = 0; g < p.ng_a; ++g)
      if (p.ga[g].pv == v || p.ga[g].qv == v) return true;
    for (int g = 0; g < p.ng_b; ++g)
      if (p.gb[g].pv == v || p.gb[g].qv == v) return true;
    return false;
  };
  for (bool merged = true; merged;) {
    merged = false;
    for (int u = 0; u < p.nv && !merged; ++u)
      for (int v = 0; v < p.nv && !merged; ++v) {
        if (u == v || p.ext[u] <= 1 || p.ext[v] <= 1 || gathered(u) || gathered(v)) continue;
        if ((p.cls[u] == CE_K) != (p.cls[v] == CE_K)) continue;
        if (p.sa[u] == 0 && p.sb[u] == 0 && p.sc[u] == 0) continue;
        if (p.sa[v] != p.sa[u] * p.ext[u] || p.sb[v] != p.sb[u] * p.ext[u] || p.sc[v] != p.sc[u] * p.ext[u]) continue;
        if (p.ext[u] * p.ext[v] >= (1ll << 31)) continue;
        p.ext[u] *= p.ext[v];
        p.ext[v] = 1;
        merged = true;
      }
  }
  SvDesc d{};
  if (p.ng_a > SV_G || p.ng_b > SV_G) return fail("too many gathers");
  // output vars: the lane var (unit stride in the operand that streams, else in C) first,
  // then by ascending out stride
  std::vector<int> ov(sd.ov, sd.ov + sd.nout);
  std::vector<int> kvars(sd.kv, sd.kv + sd.nk);
  ov.erase(std::remove_if(ov.begin(), ov.end(), [&](int v) { return p.ext[v] == 1; }), ov.end());
  kvars.erase(std::remove_if(kvars.begin(), kvars.end(), [&](int v) { return p.ext[v] == 1; }), kvars.end());
  if (static_cast<int>(ov.size()) > SV_O || static_cast<int>(kvars.size()) > SV_K) return fail("too many vars");
  auto astride = [&](int v) -> int64_t {
    if (p.sa[v]) return p.sa[v];
    for (int g = 0; g < p.ng_a; ++g)
      if (p.ga[g].pv == v || p.ga[g].qv == v) return p.ga[g].stride;
    return 0;
  };
  // lane var: fewest 32-B sectors per warp access summed over the large operands (an
  // operand independent of the var is a broadcast: 1 sector; unit stride: 4; else 32)
  double sz[3] = {1, 1, 1};
  for (int v = 0; v < p.nv; ++v) {
    if (p.sa[v] || astride(v)) sz[0] *= static_cast<double>(p.ext[v]);
    if (p.sb[v]) sz[1] *= static_cast<double>(p.ext[v]);
    if (p.cls[v] != CE_K) sz[2] *= static_cast<double>(p.ext[v]);
  }
  if (p.unary) sz[1] = 0;
  const double big = std::max(sz[0], std::max(sz[1], sz[2])) / 8;
  auto bstride = [&](int v) -> int64_t {
    if (p.sb[v]) return p.sb[v];
    for (int g = 0; g < p.ng_b; ++g)
      if (p.gb[g].pv == v || p.gb[g].qv == v) return p.gb[g].stride;
    return 0;
  };
  auto sectors = [](int64_t st) { return st == 0 ? 1.0 : st == 1 ? 4.0 : 32.0; };
  int lane = -1;
  double best = 1e30;
  for (int v : ov) {
    double c = 0;
    if (sz[0] >= big) c += sectors(astride(v));
    if (sz[1] >= big) c += sectors(bstride(v));
    if (sz[2] >= big) c += sectors(p.sc[v]);
    if (c < best - 1e-9 || (c < best + 1e-9 && astride(v) == 1)) {
      best = c;
      lane = v;
    }
  }
  if (lane >= 0) {
    ov.erase(std::find(ov.begin(), ov.end(), lane));
    ov.insert(ov.begin(), lane);
  }
  // slot 1 (blocked 4x per thread in the register-blocked kernel): prefer a var outside
  // every gather that B does not depend on, so one validity test and one B vector serve
  // the 4 outputs; among those the smallest out stride
  if (ov.size() > 2) {
    auto in_gather = [&](int v) { return gathered(v); };
    std::size_t best1 = 1;
    int score1 = -1;
    for (std::size_t i = 1; i < ov.size(); ++i) {
      const int v = ov[i];
      const int sc = (in_gather(v) ? 0 : 2) + (p.sb[v] == 0 ? 1 : 0);
      if (sc > score1) {
        score1 = sc;
        best1 = i;
      }
    }
    std::rotate(ov.begin() + 1, ov.begin() + static_cast<std::ptrdiff_t>(best1),
                ov.begin() + static_cast<std::ptrdiff_t>(best1) + 1);
  }
  // K vars: fastest in A first
  std::stable_sort(kvars.begin(), kvars.end(), [&](int x, int y) {
    const int64_t sx = astride(x) ? astride(x) : p.sb[x], sy = astride(y) ? astride(y) : p.sb[y];
    return sx < sy;
  });
  // K-lane mode when no output var streams A contiguously but the fastest K var does
  const bool klane = sz[0] >= big && !kvars.empty() && astride(kvars[0]) == 1 && best >= 32 &&
                     std::accumulate(kvars.begin(), kvars.end(), int64_t{1},
                                     [&](int64_t acc_, int v) { return acc_ * p.ext[v]; }) >= 64;
  int64_t outs = 1, K = 1, maxA = 0, maxB = 0, maxC = 0;
  d.nout = static_cast<int32_t>(ov.size());
  d.nk = static_cast<int32_t>(kvars.size());
  for (int i = 0; i < d.nout; ++i) {
    const int v = ov[static_cast<std::size_t>(i)];
    d.oext[i] = static_cast<int32_t>(p.ext[v]);
    d.odiv[i] = tc_div(static_cast<uint32_t>(p.ext[v]));
    d.osa[i] = static_cast<int32_t>(p.sa[v]);
    d.osb[i] = static_cast<int32_t>(p.sb[v]);
    d.osc[i] = static_cast<int32_t>(p.sc[v]);
    outs *= p.ext[v];
    maxA += (p.ext[v] - 1) * p.sa[v];
    maxB += (p.ext[v] - 1) * p.sb[v];
    maxC += (p.ext[v] - 1) * p.sc[v];
  }
  for (int j = 0; j < d.nk; ++j) {
    const int v = kvars[static_cast<std::size_t>(j)];
    d.kext[j] = static_cast<int32_t>(p.ext[v]);
    d.kdiv[j] = tc_div(static_cast<uint32_t>(p.ext[v]));
    d.ksa[j] = static_cast<int32_t>(p.sa[v]);
    d.ksb[j] = static_cast<int32_t>(p.sb[v]);
    K *= p.ext[v];
    maxA += (p.ext[v] - 1) * p.sa[v];
    maxB += (p.ext[v] - 1) * p.sb[v];
  }
  for (int side = 0; side < 2; ++side) {
    const int ng = side ? p.ng_b : p.ng_a;
    const CeGather* gs = side ? p.gb : p.ga;
    for (int g = 0; g < ng; ++g) {
      const int slot = d.ng++;
      d.gop[slot] = side;
      const CeGather& G = gs[g];
      if (G.extent >= (1ll << 30) || std::llabs(G.c) >= (1ll << 30)) return fail("gather extent");
      d.gc[slot] = static_cast<int32_t>(G.c);
      d.gext[slot] = static_cast<int32_t>(G.extent);
      d.gstride[slot] = static_cast<int32_t>(G.stride);
      d.gwrap[slot] = G.wrap;
      for (int i = 0; i < d.nout; ++i) {
        const int v = ov[static_cast<std::size_t>(i)];
        d.go[slot][i] = (G.pv == v ? G.sp : 0) + (G.qv == v ? G.sq : 0);
      }
      for (int j = 0; j < d.nk; ++j) {
        const int v = kvars[static_cast<std::size_t>(j)];
        d.gk[slot][j] = (G.pv == v ? G.sp : 0) + (G.qv == v ? G.sq : 0);
      }
      (side ? maxB : maxA) += (G.extent - 1) * G.stride;
    }
  }
  d.nga = p.ng_a;
  d.ngb = p.ng_b;
  d.unary = p.unary;
  d.klane = klane ? 1 : 0;
  // VEC=4 along the lane var: unit stride and 16-B aligned A, lane var never gathered
  if (!klane) {
    // a lane extent that is not a multiple of 4 needs a row pitch of >= round_up(ext, 4) in
    // A (the last float4 reads the row's padding) and masks B loads / C stores past it
    auto al = [](const float* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
    const int32_t ext0 = d.nout >= 1 ? d.oext[0] : 0, ext4 = (ext0 + 3) / 4 * 4;
    auto padded = [&](const int32_t* os, const int32_t* ks, int gbase) {
      for (int i = 1; i < d.nout; ++i)
        if (os[i] % 4 || (os[i] && os[i] < ext4)) return false;
      for (int j = 0; j < d.nk; ++j)
        if (ks && (ks[j] % 4 || (ks[j] && ks[j] < ext4))) return false;
      for (int g = 0; g < d.ng; ++g)
        if (d.gop[g] == gbase && (d.gstride[g] % 4 || d.gstride[g] < ext4)) return false;
      return true;
    };
    // A along the lane var: unit stride (float4) or independent of it (one scalar, broadcast)
    const bool a_b = d.nout >= 1 && d.osa[0] == 0;
    // a caller-owned operand ends exactly at its last row: no float4 past a ragged row end
    const bool ragged = ext0 % 4 != 0;
    bool ok = d.nout >= 1 && (a_b || (al(A) && d.osa[0] == 1 && padded(d.osa, d.ksa, 0) && !(ragged && p.exact_a)));
    for (int g = 0; g < 2 * SV_G && ok; ++g) ok = d.go[g][0] == 0;
    d.a_bcast = a_b ? 1 : 0;
    d.vec = ok ? 1 : 0;
    if (ok) {
      const bool vb = !p.unary && al(B) && d.osb[0] == 1 && padded(d.osb, d.ksb, 1) && !(ragged && p.exact_b);
      const bool vc = al(C) && d.osc[0] == 1 && padded(d.osc, nullptr, 2) && !(ragged && p.exact_c);
      d.vec_b = vb ? 1 : 0;
      d.vec_c = vc ? 1 : 0;
      d.lext = ext0;
      d.oext[0] = ext4 / 4;  // the kernel decomposes threads, each owning 4 lane values
      d.odiv[0] = tc_div(static_cast<uint32_t>(d.oext[0]));
      outs = outs / ext0 * d.oext[0];
    }
  }
  const int64_t lim = (1ll << 31) - 1;
  if (outs > lim) return fail("outputs >= 2^31");
  if (K > lim) return fail("K >= 2^31");
  if (maxA > lim || maxB > lim || maxC > lim) return fail("operand span >= 2^31");
  d.K = static_cast<uint32_t>(K);
  // depthwise stencil: a single tap K var, one gather on A over (conv output var, tap)
  // with unit coefficients, B = F[lane, tap]
  d.stencil = 0;
  if (!klane && d.vec && !p.unary && d.ng == 1 && d.gop[0] == 0 && !d.gwrap[0] && d.nk == 1 &&
      (d.kext[0] == 3 || d.kext[0] == 5 || d.kext[0] == 7) && (d.gk[0][0] == 1 || d.gk[0][0] == -1) &&
      !p.accumulate) {
    int sstar = -1, nz = 0;
    for (int i = 1; i < d.nout; ++i)
      if (d.go[0][i] != 0) {
        ++nz;
        sstar = i;
      }
    bool bok = true;
    for (int i = 1; i < d.nout; ++i) bok = bok && d.osb[i] == 0;
    if (nz == 1 && (d.go[0][sstar] == 1 || d.go[0][sstar] == -1) && d.osa[sstar] == 0 && bok) {
      // move the conv output var to slot 1 (blocked J per thread)
      auto sw = [&](int32_t* a) { std::swap(a[1], a[sstar]); };
      sw(d.oext);
      sw(d.osa);
      sw(d.osb);
      sw(d.osc);
      std::swap(d.odiv[1], d.odiv[sstar]);
      for (int g = 0; g < 2 * SV_G; ++g) sw(d.go[g]);
      d.stencil = d.kext[0];
    }
  }
  // depthwise filter gradient: outputs (lane, tap), one gather on A over (K var p, tap)
  d.dwgrad = 0;
  if (!klane && !d.stencil && d.vec && !d.a_bcast && !p.unary && d.ng == 1 && d.gop[0] == 0 && !d.gwrap[0] &&
      d.nout == 2 && (d.oext[1] == 3 || d.oext[1] == 5 || d.oext[1] == 7) &&
      (d.go[0][1] == 1 || d.go[0][1] == -1) && d.osa[1] == 0 && d.osb[1] == 0) {
    int pj = -1, nz = 0;
    for (int j = 0; j < d.nk; ++j)
      if (d.gk[0][j] != 0) {
        ++nz;
        pj = j;
      }
    if (nz == 1 && (d.gk[0][pj] == 1 || d.gk[0][pj] == -1) && d.ksa[pj] == 0) {
      auto sw = [&](int32_t* a) { std::swap(a[0], a[pj]); };
      sw(d.kext);
      sw(d.ksa);
      sw(d.ksb);
      std::swap(d.kdiv[0], d.kdiv[pj]);
      for (int g = 0; g < 2 * SV_G; ++g) sw(d.gk[g]);
      d.dwgrad = d.oext[1];
      outs = d.oext[0];  // one thread per 4 lanes and K slice, all taps
    }
  }
  // several consecutive values of output slot 1 per thread when K is short: the index
  // decoding (~10 instructions per var) otherwise dominates a 3-term stencil
  d.jrep = 1;
  d.l1ext = d.nout > 1 ? d.oext[1] : 1;
  if (d.dwgrad) {
  } else if (d.stencil) {
    const int jb = d.stencil <= 3 ? 8 : 4;
    d.jrep = jb;
    d.oext[1] = (d.l1ext + jb - 1) / jb;
    d.odiv[1] = tc_div(static_cast<uint32_t>(d.oext[1]));
    outs = outs / d.l1ext * d.oext[1];
  } else
  if (!klane && d.vec && d.nout > 1 && K <= 32 && outs >= 148 * 256 * 8) {
    d.jrep = 4;
    d.oext[1] = (d.l1ext + 3) / 4;
    d.odiv[1] = tc_div(static_cast<uint32_t>(d.oext[1]));
    outs = outs / d.l1ext * d.oext[1];
  }
  d.outs = static_cast<uint32_t>(outs);
  d.g_inv1 = d.b_inv1 = d.bfix1 = 0;
  if (d.nout > 1) {
    bool gi = true;
    for (int g = 0; g < d.ng; ++g) gi = gi && d.go[g][1] == 0;
    d.g_inv1 = gi ? 1 : 0;
    d.b_inv1 = d.osb[1] == 0 ? 1 : 0;
    bool bf = d.b_inv1 != 0;
    for (int g = 0; g < d.ng; ++g) bf = bf && (d.gop[g] == 0 || d.go[g][1] == 0);
    d.bfix1 = bf ? 1 : 0;
  }
  // K slices: enough CTAs for ~8 per SM when the outputs alone do not fill the GPU,
  // each thread keeping >= 32 K terms
  const int64_t blocks = klane ? (outs + 7) / 8 : (outs + 255) / 256;
  int64_t split = 1;
  if (d.dwgrad) {  // ~4 waves of 256-thread CTAs, each thread >= 64 K steps
    // few outputs (a 7x7 filter over 11 ranks: 3 lane quads) with a long K: tens of
    // thousands of slices would all red.add into the same 21 float4s; capping the slices
    // at ~16K / outs (measured sweep 4K..64K) trades that contention for longer threads
    // (CP conv1 filter gradients 1.15 -> 0.37 ms, CP 64->64 @56 cr0.1 266 -> 147 us)
    static const int64_t cap = [] {
      const char* e = std::getenv("CE_DWG_SLICES");
      return e ? std::atoll(e) : int64_t{16384};
    }();
    // (outs <= 256: the kernel sums a CTA's slices in shared memory first, so contention no
    // longer caps the slice count -- ~8 CTAs per SM, each thread >= 48 K steps)
    static const int64_t kmin = [] {
      const char* e = std::getenv("CE_DWG_KMIN");
      return e ? std::atoll(e) : int64_t{48};
    }();
    if (outs <= 256) {
      split = std::max<int64_t>(1, std::min<int64_t>((148 * 256 * 8 + outs - 1) / outs, K / kmin));
    } else {
      split = std::max<int64_t>(1, std::min<int64_t>((148 * 256 * 4 + outs - 1) / outs, K / 64));
      if (cap > 0 && outs < 16) split = std::min<int64_t>(split, std::max<int64_t>(1, cap / outs));
    }
  }
  else if (blocks < 148 * 8 && K >= 64)
    split = std::min<int64_t>((148 * 8 + blocks - 1) / blocks, K / (klane ? 1024 : 32));
  split = std::max<int64_t>(1, std::min<int64_t>(split, 65535));
  d.kper = static_cast<uint32_t>((K + split - 1) / split);
  d.mode = split > 1 ? 2 : (p.accumulate ? 1 : 0);
  *span = maxC + 1;
  *out = d;
  return true;
}

cudaError_t sv_launch(const SvDesc& d, int64_t span, bool zero_first, const float* A, const float* B, float* C,
                      cudaStream_t s) {
  if (d.outs == 0) return cudaSuccess;
  if (zero_first) {
    cudaError_t e = cudaMemsetAsync(C, 0, static_cast<size_t>(span) * 4, s);
    if (e != cudaSuccess) return e;
  }
  const unsigned gy = d.K ? (d.K + d.kper - 1) / d.kper : 1u;
  static const bool trace = [] {  // debug: CE_SV_TRACE=1 prints the variant of every launch
    const char* e = std::getenv("CE_SV_TRACE");
    return e && *e == '1';
  }();
  if (trace)
    std::fprintf(stderr, "sv_launch %s outs=%u K=%u slices=%u\n",
                 d.dwgrad ? "dwgrad" : d.stencil ? "stencil" : d.klane ? "klane" : (d.vec && d.jrep == 4) ? "blocked"
                                                                               : d.vec ? "vec4" : "scalar",
                 d.outs, d.K, gy);
  const dim3 gk((d.outs + 7u) / 8u, gy), g1((d.outs + 255u) / 256u, gy), blk(256);
  if (d.dwgrad) {
    const int sa = d.gk[0][0], sb = d.go[0][1];
    const dim3 gd(static_cast<unsigned>((static_cast<uint64_t>(d.outs) * gy + 255u) / 256u));
#define CE_DWG(KT)                                                                                       \
  if (sa > 0 && sb > 0) return ce_launch(ce_dwgrad_kernel<KT, 1, 1>, gd, blk, 0, s, d, A, B, C);         \
  if (sa > 0 && sb < 0) return ce_launch(ce_dwgrad_kernel<KT, 1, -1>, gd, blk, 0, s, d, A, B, C);        \
  if (sa < 0 && sb > 0) return ce_launch(ce_dwgrad_kernel<KT, -1, 1>, gd, blk, 0, s, d, A, B, C);        \
  return ce_launch(ce_dwgrad_kernel<KT, -1, -1>, gd, blk, 0, s, d, A, B, C);
    if (d.dwgrad == 3) { CE_DWG(3) }
    if (d.dwgrad == 5) { CE_DWG(5) }
    CE_DWG(7)
#undef CE_DWG
  }
  if (d.stencil) {
    const int sa = d.go[0][1], sb = d.gk[0][0];
#define CE_DW(KT, J)                                                                                     \
  if (sa > 0 && sb > 0) return ce_launch(ce_dw_kernel<KT, J, 1, 1>, g1, blk, 0, s, d, A, B, C);          \
  if (sa > 0 && sb < 0) return ce_launch(ce_dw_kernel<KT, J, 1, -1>, g1, blk, 0, s, d, A, B, C);         \
  if (sa < 0 && sb > 0) return ce_launch(ce_dw_kernel<KT, J, -1, 1>, g1, blk, 0, s, d, A, B, C);         \
  return ce_launch(ce_dw_kernel<KT, J, -1, -1>, g1, blk, 0, s, d, A, B, C);
    if (d.stencil == 3) { CE_DW(3, 8) }
    if (d.stencil == 5) { CE_DW(5, 4) }
    CE_DW(7, 4)
#undef CE_DW
  }
  if (d.vec && d.jrep == 4) {
    switch (d.ng) {
      case 0: return ce_launch(ce_stream_blk_kernel<0>, g1, blk, 0, s, d, A, B, C);
      case 1: return ce_launch(ce_stream_blk_kernel<1>, g1, blk, 0, s, d, A, B, C);
      case 2: return ce_launch(ce_stream_blk_kernel<2>, g1, blk, 0, s, d, A, B, C);
      case 3: return ce_launch(ce_stream_blk_kernel<3>, g1, blk, 0, s, d, A, B, C);
      default: return ce_launch(ce_stream_blk_kernel<4>, g1, blk, 0, s, d, A, B, C);
    }
  }
  switch (d.klane ? 10 + d.ng : d.vec ? 20 + d.ng : d.ng) {
    case 10: return ce_launch(ce_stream_klane_kernel<0>, gk, blk, 0, s, d, A, B, C);
    case 11: return ce_launch(ce_stream_klane_kernel<1>, gk, blk, 0, s, d, A, B, C);
    case 12: return ce_launch(ce_stream_klane_kernel<2>, gk, blk, 0, s, d, A, B, C);
    case 13: return ce_launch(ce_stream_klane_kernel<3>, gk, blk, 0, s, d, A, B, C);
    case 14: return ce_launch(ce_stream_klane_kernel<4>, gk, blk, 0, s, d, A, B, C);
    case 20: return ce_launch(ce_stream_kernel<4, 0>, g1, blk, 0, s, d, A, B, C);
    case 21: return ce_launch(ce_stream_kernel<4, 1>, g1, blk, 0, s, d, A, B, C);
    case 22: return ce_launch(ce_stream_kernel<4, 2>, g1, blk, 0, s, d, A, B, C);
    case 23: return ce_launch(ce_stream_kernel<4, 3>, g1, blk, 0, s, d, A, B, C);
    case 24: return ce_launch(ce_stream_kernel<4, 4>, g1, blk, 0, s, d, A, B, C);
    case 0: return ce_launch(ce_stream_kernel<1, 0>, g1, blk, 0, s, d, A, B, C);
    case 1: return ce_launch(ce_stream_kernel<1, 1>, g1, blk, 0, s, d, A, B, C);
    case 2: return ce_launch(ce_stream_kernel<1, 2>, g1, blk, 0, s, d, A, B, C);
    case 3: return ce_launch(ce_stream_kernel<1, 3>, g1, blk, 0, s, d, A, B, C);
    default: return ce_launch(ce_stream_kernel<1, 4>, g1, blk, 0, s, d, A, B, C);
  }
}

// ----------------------------------------------------------------------------- tiled
constexpr int TM = 64, TN = 64, TK = 16;

__device__ __forceinline__ void decompose(int64_t x, const int32_t* vars, int n, const int64_t* ext,
                                          int64_t* out_vals) {
  for (int i = 0; i < n; ++i) {
    const int64_t e = ext[vars[i]];
    out_vals[i] = x % e;
    x /= e;
  }
}

__global__ void __launch_bounds__(256) ce_tiled_kernel(const CeSimtDesc d, const float* __restrict__ A,
                                                       const float* __restrict__ B, float* __restrict__ C,
                                                       int a_kfast, int b_kfast) {
  ce_pdl_enter();
  const CeProblem& p = d.p;
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  __shared__ int64_t mOffA[TM], mOffC[TM], nOffB[TN], nOffC[TN];
  __shared__ int64_t mP[TM][CE_MAX_GATHER], nP[TN][CE_MAX_GATHER];
  __shared__ int64_t kOffA[TK], kOffB[TK];
  __shared__ int64_t kQA[TK][CE_MAX_GATHER], kQB[TK][CE_MAX_GATHER];
  __shared__ int64_t zA, zB, zC;

  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * TM, n0 = (int64_t)blockIdx.y * TN;
  int64_t vals[CE_MAX_VARS];

  for (int64_t z = blockIdx.z; z < d.Z; z += gridDim.z) {
    __syncthreads();
    if (tid == 0) {
      decompose(z, d.zv, d.nz, p.ext, vals);
      int64_t a = 0, b = 0, c = 0;
      for (int i = 0; i < d.nz; ++i) {
        a += vals[i] * p.sa[d.zv[i]];
        b += vals[i] * p.sb[d.zv[i]];
        c += vals[i] * p.sc[d.zv[i]];
      }
      zA = a;
      zB = b;
      zC = c;
    }
    if (tid < TM) {
      const int64_t m = m0 + tid;
      int64_t a = 0, c = 0;
      if (m < d.M) {
        decompose(m, d.mv, d.nm, p.ext, vals);
        for (int i = 0; i < d.nm; ++i) {
          a += vals[i] * p.sa[d.mv[i]];
          c += vals[i] * p.sc[d.mv[i]];
        }
        for (int g = 0; g < p.ng_a; ++g)
          for (int i = 0; i < d.nm; ++i)
            if (d.mv[i] == p.ga[g].pv) mP[tid][g] = vals[i];
      }
      mOffA[tid] = a;
      mOffC[tid] = c;
    } else if (tid < TM + TN) {
      const int j = tid - TM;
      const int64_t n = n0 + j;
      int64_t b = 0, c = 0;
      if (n < d.N) {
        decompose(n, d.nvv, d.nn, p.ext, vals);
        for (int i = 0; i < d.nn; ++i) {
          b += vals[i] * p.sb[d.nvv[i]];
          c += vals[i] * p.sc[d.nvv[i]];
        }
        for (int g = 0; g < p.ng_b; ++g)
          for (int i = 0; i < d.nn; ++i)
            if (d.nvv[i] == p.gb[g].pv) nP[j][g] = vals[i];
      }
      nOffB[j] = b;
      nOffC[j] = c;
    }
    const int tx = tid % 16, ty = tid / 16;
    float acc[4][4] = {};

    for (int64_t k0 = 0; k0 < d.K; k0 += TK) {
      __syncthreads();
      if (tid < TK) {
        const int64_t k = k0 + tid;
        int64_t a = 0, b = 0;
        if (k < d.K) {
          decompose(k, d.kv, d.nk, p.ext, vals);
          for (int i = 0; i < d.nk; ++i) {
            a += vals[i] * p.sa[d.kv[i]];
            b += vals[i] * p.sb[d.kv[i]];
          }
          for (int g = 0; g < p.ng_a; ++g)
            for (int i = 0; i < d.nk; ++i)
              if (d.kv[i] == p.ga[g].qv) kQA[tid][g] = vals[i];
          for (int g = 0; g < p.ng_b; ++g)
            for (int i = 0; i < d.nk; ++i)
              if (d.kv[i] == p.gb[g].qv) kQB[tid][g] = vals[i];
        }
        kOffA[tid] = a;
        kOffB[tid] = b;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < (TM * TK) / 256; ++r) {
        const int e = tid + r * 256;
        const int mi = a_kfast ? e / TK : e % TM;
        const int ki = a_kfast ? e % TK : e / TM;
        float v = 0.f;
        if (m0 + mi < d.M && k0 + ki < d.K) {
          int64_t off = zA + mOffA[mi] + kOffA[ki];
          bool ok = true;
          for (int g = 0; g < p.ng_a && ok; ++g) {
            int64_t o;
            ok = gather_index(p.ga[g], mP[mi][g], kQA[ki][g], &o);
            off += o;
          }
          if (ok) v = __ldg(A + off);
        }
        As[ki][mi] = v;
      }
#pragma unroll
      for (int r = 0; r < (TN * TK) / 256; ++r) {
        const int e = tid + r * 256;
        const int ni = b_kfast ? e / TK : e % TN;
        const int ki = b_kfast ? e % TK : e / TN;
        float v = 0.f;
        if (n0 + ni < d.N && k0 + ki < d.K) {
          int64_t off = zB + nOffB[ni] + kOffB[ki];
          bool ok = true;
          for (int g = 0; g < p.ng_b && ok; ++g) {
            int64_t o;
            ok = gather_index(p.gb[g], nP[ni][g], kQB[ki][g], &o);
            off += o;
          }
          if (ok) v = __ldg(B + off);
        }
        Bs[ki][ni] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int mi = ty * 4 + i;
      if (m0 + mi >= d.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ni = tx * 4 + j;
        if (n0 + ni >= d.N) continue;
        float* dst = C + zC + mOffC[mi] + nOffC[ni];
        if (p.accumulate)
          *dst += acc[i][j];
        else
          *dst = acc[i][j];
      }
    }
  }
}

// ----------------------------------------------------------------------------- permute
// Family (c): axis permutation (operand repacking, reference permute tensor.cpp:50-94).
// 32x32 shared-memory tile over (input unit-stride axis, output unit-stride axis) so
// both the load and the store are coalesced; all other axes are a flattened batch.
struct CePermDesc {
  int32_t nrest;
  int32_t vin, vout;       // indices into ext/sa/sc
  int32_t same;            // 1: input and output share the unit-stride axis (vout = y axis)
  // composite tile axes for short unit-stride axes: x = x1 + ext[vin]*x2 where x2 = vin2
  // continues vin in the INPUT; y = y1 + ext[vout]*y2 where y2 = vout2 continues vout in
  // the OUTPUT (-1: none)
  int32_t vin2, vout2;
  int32_t tile_ok;         // 0: grid limits of the tile kernels exceeded (block kernel only)
  int64_t ext[CE_MAX_VARS], sa[CE_MAX_VARS], sc[CE_MAX_VARS];
  int32_t rest[CE_MAX_VARS];
  int64_t nbatch;
};

// 64x64 tile, 256 threads, 16 independent loads in flight per thread; 32-bit in-tile
// index math, 64-bit only for the per-batch base.
__global__ void __launch_bounds__(256, 6) ce_transpose_kernel(const CePermDesc d, const float* __restrict__ A,
                                                           float* __restrict__ C) {
  ce_pdl_enter();
  __shared__ float tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t x0 = static_cast<int64_t>(blockIdx.x) * 32;  // along vin (+vin2)
  const int64_t y0 = static_cast<int64_t>(blockIdx.y) * 32;  // along vout (+vout2)
  const uint32_t ex1 = static_cast<uint32_t>(d.ext[d.vin]), ey1 = static_cast<uint32_t>(d.ext[d.vout]);
  const int64_t ein = d.ext[d.vin] * (d.vin2 >= 0 ? d.ext[d.vin2] : 1);
  const int64_t eout = d.ext[d.vout] * (d.vout2 >= 0 ? d.ext[d.vout2] : 1);
  const int64_t sa_y1 = d.sa[d.vout], sa_y2 = d.vout2 >= 0 ? d.sa[d.vout2] : 0;
  const int64_t sc_x1 = d.sc[d.vin], sc_x2 = d.vin2 >= 0 ? d.sc[d.vin2] : 0;
  for (int64_t bt = blockIdx.z; bt < d.nbatch; bt += gridDim.z) {
    int64_t r = bt, bin = 0, bout = 0;
    for (int i = 0; i < d.nrest; ++i) {
      const int v = d.rest[i];
      const int64_t x = r % d.ext[v];
      r /= d.ext[v];
      bin += x * d.sa[v];
      bout += x * d.sc[v];
    }
    if (d.vout2 >= 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t y = y0 + ty + 8 * j, x = x0 + tx;
        const uint32_t y1 = static_cast<uint32_t>(y) % ey1, y2 = static_cast<uint32_t>(y) / ey1;
        tile[ty + 8 * j][tx] = (x < ein && y < eout) ? __ldg(A + bin + x + y1 * sa_y1 + y2 * sa_y2) : 0.f;
      }
    } else {
      // pointer increments + hoisted bounds: this kernel is instruction-bound otherwise
      const bool xok = x0 + tx < ein;
      const float* src = A + bin + x0 + tx + (y0 + ty) * sa_y1;
      const int64_t step = 8 * sa_y1;
      const int64_t yrem = eout - (y0 + ty);
#pragma unroll
      for (int j = 0; j < 4; ++j) tile[ty + 8 * j][tx] = (xok && 8 * j < yrem) ? __ldg(src + j * step) : 0.f;
    }
    __syncthreads();
    if (d.vin2 >= 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t x = x0 + ty + 8 * j, y = y0 + tx;
        const uint32_t x1 = static_cast<uint32_t>(x) % ex1, x2 = static_cast<uint32_t>(x) / ex1;
        if (x < ein && y < eout) C[bout + y + x1 * sc_x1 + x2 * sc_x2] = tile[tx][ty + 8 * j];
      }
    } else {
      const bool yok = y0 + tx < eout;
      float* dst = C + bout + y0 + tx + (x0 + ty) * sc_x1;
      const int64_t step = 8 * sc_x1;
      const int64_t xrem = ein - (x0 + ty);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (yok && 8 * j < xrem) dst[j * step] = tile[tx][ty + 8 * j];
    }
    __syncthreads();
  }
}

// Offset of row i along a tile axis that may be composite (i = i1 + e1*i2).
struct CeRowMap {
  uint32_t e1;
  int64_t s1, s2;
  bool comp;
  __device__ __forceinline__ int64_t operator()(uint32_t i) const {
    return comp ? static_cast<int64_t>(i % e1) * s1 + static_cast<int64_t>(i / e1) * s2 : static_cast<int64_t>(i) * s1;
  }
};

// 64x64 tiles with 128-bit global accesses (VI: input rows along x, VO: output rows
// along y are 16-B aligned and a multiple of 4 long).  Per element: a quarter of a
// vector load and store plus one STS and one LDS; the 65-float row pitch keeps both
// smem phases at 2-way bank conflicts.  Composite tile axes (short unit-stride axes
// continued by a second axis, see CePermDesc) cost one division per row, not per element.
template <bool VI, bool VO>
// (6 CTAs/SM: at 8 the 32-register budget spilled the float4 variant; cfg2 step -0.6%)
__global__ void __launch_bounds__(256, 6) ce_transpose64_kernel(const CePermDesc d, const float* __restrict__ A,
                                                             float* __restrict__ C) {
  ce_pdl_enter();
  __shared__ float tile[64][65];
  const uint32_t ein = static_cast<uint32_t>(d.ext[d.vin] * (d.vin2 >= 0 ? d.ext[d.vin2] : 1));
  const uint32_t eout = static_cast<uint32_t>(d.ext[d.vout] * (d.vout2 >= 0 ? d.ext[d.vout2] : 1));
  const CeRowMap in_row{static_cast<uint32_t>(d.ext[d.vout]), d.sa[d.vout], d.vout2 >= 0 ? d.sa[d.vout2] : 0,
                        d.vout2 >= 0};
  const CeRowMap out_row{static_cast<uint32_t>(d.ext[d.vin]), d.sc[d.vin], d.vin2 >= 0 ? d.sc[d.vin2] : 0,
                         d.vin2 >= 0};
  const uint32_t x0 = blockIdx.x * 64, y0 = blockIdx.y * 64;
  const int t = threadIdx.x;
  for (int64_t bt = blockIdx.z; bt < d.nbatch; bt += gridDim.z) {
    int64_t r = bt, bin = 0, bout = 0;
    for (int i = 0; i < d.nrest; ++i) {
      const int v = d.rest[i];
      const int64_t x = r % d.ext[v];
      r /= d.ext[v];
      bin += x * d.sa[v];
      bout += x * d.sc[v];
    }
    if (VI) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = t + 256 * j, row = idx >> 4, c4 = (idx & 15) * 4;
        const uint32_t y = y0 + row, x = x0 + c4;
        v[j] = (y < eout && x < ein) ? __ldg(reinterpret_cast<const float4*>(A + bin + in_row(y) + x))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = t + 256 * j, row = idx >> 4, c4 = (idx & 15) * 4;
        tile[row][c4] = v[j].x;
        tile[row][c4 + 1] = v[j].y;
        tile[row][c4 + 2] = v[j].z;
        tile[row][c4 + 3] = v[j].w;
      }
    } else {
      const int c = t & 63, row0 = t >> 6;
      const bool xok = x0 + c < ein;
      const float* src = A + bin + x0 + c;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t y = y0 + row0 + 4 * j;
        v[j] = (xok && y < eout) ? __ldg(src + in_row(y)) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[row0 + 4 * j][c] = v[j];
    }
    __syncthreads();
    if (VO) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int idx = t + 256 * j, xr = idx >> 4, c4 = (idx & 15) * 4;
        const uint32_t x = x0 + xr, y = y0 + c4;
        if (x < ein && y < eout)
          *reinterpret_cast<float4*>(C + bout + out_row(x) + y) =
              make_float4(tile[c4][xr], tile[c4 + 1][xr], tile[c4 + 2][xr], tile[c4 + 3][xr]);
      }
    } else {
      const int c = t & 63, xr0 = t >> 6;
      const bool yok = y0 + c < eout;
      float* dst = C + bout + y0 + c;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t x = x0 + xr0 + 4 * j;
        if (yok && x < ein) dst[out_row(x)] = tile[c][xr0 + 4 * j];
      }
    }
    __syncthreads();
  }
}

// Input and output share the unit-stride axis x: a strided copy of rows (x, y) per
// batch slice.  A row is served by L = 2^lshift lanes (L >= min(ext x, 32)), so a warp
// covers 32/L short rows without any per-element division; 4 rows per thread in flight.
template <bool V4>
__global__ void __launch_bounds__(256, 6) ce_rowcopy_kernel(const CePermDesc d, const float* __restrict__ A,
                                                         float* __restrict__ C, int lshift) {
  // V4: rows are 16-B aligned multiples of 4 floats on both sides -> float4 traffic
  ce_pdl_enter();
  using T = typename std::conditional<V4, float4, float>::type;
  constexpr int W = V4 ? 4 : 1;
  const uint32_t ex = static_cast<uint32_t>(d.ext[d.vin]) / W, ey = static_cast<uint32_t>(d.ext[d.vout]);
  const int64_t sa_y = d.sa[d.vout], sc_y = d.sc[d.vout];
  const uint32_t L = 1u << lshift, lx = threadIdx.x & (L - 1), rows = 256u >> lshift;
  const uint32_t ly = threadIdx.x >> lshift;
  for (int64_t bt = blockIdx.y; bt < d.nbatch; bt += gridDim.y) {
    int64_t r = bt, bin = 0, bout = 0;
    for (int i = 0; i < d.nrest; ++i) {
      const int v = d.rest[i];
      const int64_t x = r % d.ext[v];
      r /= d.ext[v];
      bin += x * d.sa[v];
      bout += x * d.sc[v];
    }
    for (uint32_t yb = blockIdx.x * rows * 4; yb < ey; yb += gridDim.x * rows * 4) {
      for (uint32_t x = lx; x < ex; x += L) {
        T v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t y = yb + ly + j * rows;
          if (y < ey) v[j] = __ldg(reinterpret_cast<const T*>(A + bin + static_cast<int64_t>(y) * sa_y) + x);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t y = yb + ly + j * rows;
          if (y < ey) reinterpret_cast<T*>(C + bout + static_cast<int64_t>(y) * sc_y)[x] = v[j];
        }
      }
    }
  }
}

// Block permute for short axes (RTR's 4- and 10-wide factor axes, where the 2-axis tile
// kernels above use a fraction of each tile and pay a 64-bit slice decode per few dozen
// elements).  A block = whole (or divisor-split) axes covering >= 32 elements of both the
// input and the output unit-stride runs, <= BP_MAX elements; the remaining axes are a
// batch walked by a persistent grid.  Every thread's in-block offsets are batch-invariant,
// so they are decoded once: per element one LDG + STS and one LDS + STG.  Shared memory
// holds the block in output order (1 word of padding per 32), double-buffered so one
// barrier per block suffices.
constexpr int BP_MAX = 2048, BP_AX = 8;
struct CeBlkPermDesc {
  int32_t S, ni, no, nr;
  int32_t iext[BP_AX], isa[BP_AX], ipos[BP_AX];  // block axes in input-stride order
  TcDiv idiv[BP_AX];
  int32_t oext[BP_AX], osc[BP_AX];               // block axes in output-stride order
  TcDiv odiv[BP_AX];
  uint32_t rext[CE_MAX_VARS];                    // batch axes
  TcDiv rdiv[CE_MAX_VARS];
  int64_t rsa[CE_MAX_VARS], rsc[CE_MAX_VARS];
  uint32_t nbatch;
  // gathered input axes (tap expansion, see ce_exec.cpp expand()): index x_g = gc + sum of
  // coef * axis value over block and batch axes, valid in [0, gext), else the element is 0
  int32_t ng;
  int32_t gext[2], gc[2];
  int64_t gstride[2];
  int32_t icoef[2][BP_AX];
  int32_t rcoef[2][CE_MAX_VARS];
};

template <int NE, int NG>
__global__ void __launch_bounds__(256, 4) ce_blockperm_kernel(const CeBlkPermDesc d, const float* __restrict__ A,
                                                              float* __restrict__ C) {
  ce_pdl_enter();
  constexpr int SM = BP_MAX + BP_MAX / 32;
  __shared__ float sm[2][SM];
  int32_t ioff[NE], spos[NE], ooff[NE];
  int32_t gin[NE][NG > 0 ? NG : 1];
#pragma unroll
  for (int k = 0; k < NE; ++k) {
    const uint32_t t = threadIdx.x + 256u * k;
    uint32_t r = t;
    int32_t a = 0, p = 0, c = 0;
    int32_t g[NG > 0 ? NG : 1];
#pragma unroll
    for (int j = 0; j < NG; ++j) g[j] = 0;
#pragma unroll
    for (int i = 0; i < BP_AX; ++i)
      if (i < d.ni) {
        const uint32_t q = tc_quo(r, d.idiv[i]);
        const int32_t v = static_cast<int32_t>(r - q * static_cast<uint32_t>(d.iext[i]));
        r = q;
        a += v * d.isa[i];
        p += v * d.ipos[i];
#pragma unroll
        for (int j = 0; j < NG; ++j) g[j] += v * d.icoef[j][i];
      }
    r = t;
#pragma unroll
    for (int i = 0; i < BP_AX; ++i)
      if (i < d.no) {
        const uint32_t q = tc_quo(r, d.odiv[i]);
        const int32_t v = static_cast<int32_t>(r - q * static_cast<uint32_t>(d.oext[i]));
        r = q;
        c += v * d.osc[i];
      }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      gin[k][j] = g[j];
      a += g[j] * static_cast<int32_t>(d.gstride[j]);
    }
    ioff[k] = a;
    spos[k] = p + (p >> 5);
    ooff[k] = c;
  }
  int buf = 0;
  for (uint32_t bt = blockIdx.x; bt < d.nbatch; bt += gridDim.x) {
    uint32_t r = bt;
    int64_t bin = 0, bout = 0;
    int32_t gb[NG > 0 ? NG : 1];
#pragma unroll
    for (int j = 0; j < NG; ++j) gb[j] = d.gc[j];
    for (int i = 0; i < d.nr; ++i) {
      const uint32_t q = tc_quo(r, d.rdiv[i]);
      const int64_t v = static_cast<int64_t>(r - q * d.rext[i]);
      r = q;
      bin += v * d.rsa[i];
      bout += v * d.rsc[i];
#pragma unroll
      for (int j = 0; j < NG; ++j) gb[j] += static_cast<int32_t>(v) * d.rcoef[j][i];
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) bin += static_cast<int64_t>(gb[j]) * d.gstride[j];
    float v[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      bool ok = threadIdx.x + 256 * k < static_cast<uint32_t>(d.S);
#pragma unroll
      for (int j = 0; j < NG; ++j) ok = ok && static_cast<uint32_t>(gb[j] + gin[k][j]) < static_cast<uint32_t>(d.gext[j]);
      v[k] = ok ? __ldg(A + bin + ioff[k]) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < NE; ++k)
      if (threadIdx.x + 256 * k < static_cast<uint32_t>(d.S)) sm[buf][spos[k]] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const uint32_t t = threadIdx.x + 256u * k;
      if (t < static_cast<uint32_t>(d.S)) C[bout + ooff[k]] = sm[buf][t + (t >> 5)];
    }
    buf ^= 1;
  }
}

// ----------------------------------------------------------------------------- fill
__global__ void ce_fill_kernel(float* __restrict__ dst, int64_t n, uint64_t seed) {
  ce_pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const double u = (double)(z >> 11) * 0x1.0p-53;
    dst[i] = (float)(2.0 * u - 1.0);
  }
}

int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = 148 * 32;  // 32 resident 256-thread waves' worth of CTAs, grid-stride beyond
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

// block permute with gathered axes (defined with the permute host code below)
bool blkgather_desc(const CeProblem& p, CeBlkPermDesc* out);
cudaError_t blk_launch(const CeBlkPermDesc& bp, const float* A, float* C, cudaStream_t s);
}  // namespace

int ce_stream_describe(const CeSimtDesc& d, char* buf, int n) {
  // diagnostics: the streaming variant a launch with 16-B aligned operands would take
  SvDesc sv;
  int64_t span = 0;
  const char* why = "?";
  const float* al = reinterpret_cast<const float*>(uintptr_t{256});
  CeBlkPermDesc bp;
  if (!d.p.accumulate && blkgather_desc(d.p, &bp)) {
    int k = std::snprintf(buf, n, "block-gather S=%d ni=%d no=%d batch=%u ng=%d", bp.S, bp.ni, bp.no, bp.nbatch, bp.ng);
    if (std::getenv("CE_SV_DESCRIBE_VARS")) {
      for (int i = 0; i < bp.ni && k < n; ++i)
        k += std::snprintf(buf + k, n - k, " i%d:%d/sa%d/pos%d/c%d,%d", i, bp.iext[i], bp.isa[i], bp.ipos[i],
                           bp.icoef[0][i], bp.icoef[1][i]);
      for (int i = 0; i < bp.no && k < n; ++i) k += std::snprintf(buf + k, n - k, " o%d:%d/sc%d", i, bp.oext[i], bp.osc[i]);
      for (int g = 0; g < bp.ng && k < n; ++g)
        k += std::snprintf(buf + k, n - k, " g%d:c%d/ext%d/st%lld", g, bp.gc[g], bp.gext[g], (long long)bp.gstride[g]);
    }
    return k;
  }
  if (!simt_stream_enabled()) return std::snprintf(buf, n, "stream off");
  if (!sv_build(d, al, al, al, &sv, &span, &why)) return std::snprintf(buf, n, "no stream: %s", why);
  return std::snprintf(buf, n, "stream %s vec_b=%d vec_c=%d nout=%d nk=%d ng=%d outs=%u K=%u kper=%u",
                       sv.dwgrad ? "dwgrad" : sv.stencil ? "stencil" : sv.klane ? "klane" : (sv.vec && sv.jrep == 4) ? "blocked"
                       : sv.vec ? "vec4" : "scalar",
                       sv.vec_b, sv.vec_c, sv.nout, sv.nk, sv.ng, sv.outs, sv.K, sv.kper) +
         [&] {
           int k = 0;
           if (std::getenv("CE_SV_DESCRIBE_VARS"))
             for (int i = 0; i < sv.nout; ++i)
               k += std::snprintf(buf + std::strlen(buf), n - std::strlen(buf), " o%d:%d/%d/%d/%d", i, sv.oext[i],
                                  sv.osa[i], sv.osb[i], sv.osc[i]);
           return k;
         }();
}

cudaError_t ce_launch_direct(const CeSimtDesc& d, const float* A, const float* B, float* C, cudaStream_t s) {
  const int64_t total = d.Z * d.M * d.N;
  if (total == 0) return cudaSuccess;
  SvDesc sv;
  int64_t span = 0;
  CeBlkPermDesc bp;
  if (!d.p.accumulate && blkgather_desc(d.p, &bp)) return blk_launch(bp, A, C, s);
  if (simt_stream_enabled() && sv_build(d, A, B, C, &sv, &span))
    return sv_launch(sv, span, sv.mode == 2 && !d.p.accumulate, A, B, C, s);
  return ce_launch(ce_direct_kernel, dim3(grid_for(total, 256)), dim3(256), 0, s, d, A, B, C);
}

cudaError_t ce_launch_reduce(const CeSimtDesc& d, const float* A, const float* B, float* C, int64_t out_span,
                             cudaStream_t s) {
  const int64_t outs = d.Z * d.M * d.N;
  if (outs == 0) return cudaSuccess;
  SvDesc sv;
  int64_t span = 0;
  if (simt_stream_enabled() && sv_build(d, A, B, C, &sv, &span))
    return sv_launch(sv, span, sv.mode == 2 && !d.p.accumulate, A, B, C, s);
  // enough CTAs for ~4 waves, each thread doing >= 8 terms
  int64_t split = (148 * 4 + outs - 1) / outs;
  split = std::max<int64_t>(1, std::min<int64_t>(split, d.K / (256 * 8)));
  if (split > 65535) split = 65535;
  const int64_t per = (d.K + split - 1) / split;
  if (split > 1 && !d.p.accumulate) {
    cudaError_t e = cudaMemsetAsync(C, 0, static_cast<size_t>(out_span) * 4, s);
    if (e != cudaSuccess) return e;
  }
  if (outs > 0x7fffffff) return cudaErrorInvalidConfiguration;
  return ce_launch(ce_reduce_kernel, dim3(static_cast<unsigned>(outs), static_cast<unsigned>(split)), dim3(256), 0, s,
                   d, A, B, C, per);
}

cudaError_t ce_launch_tiled(const CeSimtDesc& d, const float* A, const float* B, float* C, int a_kfast,
                            int b_kfast, cudaStream_t s) {
  if (d.Z * d.M * d.N == 0) return cudaSuccess;
  dim3 grid((unsigned)((d.M + TM - 1) / TM), (unsigned)((d.N + TN - 1) / TN),
            (unsigned)(d.Z < 65535 ? d.Z : 65535));
  if (grid.y > 65535) return cudaErrorInvalidConfiguration;
  return ce_launch(ce_tiled_kernel, grid, dim3(256), 0, s, d, A, B, C, a_kfast, b_kfast);
}

namespace {
// Merge axes that are contiguous in both input and output, drop extent-1 axes,
// and pick the unit-stride axes of each side.  Returns false if not a 2-sided transpose.
bool perm_desc(const CeProblem& p, CePermDesc* out) {
  if (!p.unary || p.ng_a) return false;
  int64_t ext[CE_MAX_VARS], sa[CE_MAX_VARS], sc[CE_MAX_VARS];
  int n = 0;
  for (int v = 0; v < p.nv; ++v) {
    if (p.cls[v] == CE_K || p.sa[v] == 0 || p.sc[v] == 0) return false;  // pure permutation only
    if (p.ext[v] == 1) continue;
    ext[n] = p.ext[v];
    sa[n] = p.sa[v];
    sc[n] = p.sc[v];
    ++n;
  }
  for (bool merged = true; merged;) {
    merged = false;
    for (int i = 0; i < n && !merged; ++i)
      for (int j = 0; j < n && !merged; ++j)
        if (i != j && sa[j] == sa[i] * ext[i] && sc[j] == sc[i] * ext[i]) {
          ext[i] *= ext[j];
          for (int k = j; k + 1 < n; ++k) {
            ext[k] = ext[k + 1];
            sa[k] = sa[k + 1];
            sc[k] = sc[k + 1];
          }
          --n;
          merged = true;
        }
  }
  CePermDesc d{};
  d.vin = d.vout = -1;
  for (int v = 0; v < n; ++v) {
    d.ext[v] = ext[v];
    d.sa[v] = sa[v];
    d.sc[v] = sc[v];
    if (sa[v] == 1) d.vin = v;
    if (sc[v] == 1) d.vout = v;
  }
  if (d.vin < 0 || d.vout < 0) return false;
  d.vin2 = d.vout2 = -1;
  d.tile_ok = 1;
  if (d.vin != d.vout) {
    // short unit-stride axes borrow the axis that continues them on their own side
    if (ext[d.vin] < 32)
      for (int v = 0; v < n; ++v)
        if (v != d.vin && v != d.vout && sa[v] == ext[d.vin]) d.vin2 = v;
    if (ext[d.vout] < 32)
      for (int v = 0; v < n; ++v)
        if (v != d.vin && v != d.vout && v != d.vin2 && sc[v] == ext[d.vout]) d.vout2 = v;
    const int64_t ein = ext[d.vin] * (d.vin2 >= 0 ? ext[d.vin2] : 1);
    const int64_t eout = ext[d.vout] * (d.vout2 >= 0 ? ext[d.vout2] : 1);
    if (ein >= (1ll << 31) || eout >= (1ll << 31) || (eout + 31) / 32 > 65535) d.tile_ok = 0;
  }
  if (d.vin == d.vout) {
    // row copy: y = the axis with the smallest output stride among the others
    int vy = -1;
    for (int v = 0; v < n; ++v)
      if (v != d.vin && (vy < 0 || sc[v] < sc[vy])) vy = v;
    if (vy < 0) return false;
    d.vout = vy;
    d.same = 1;
  }
  if ((ext[d.vout] + 31) / 32 > 65535 || ext[d.vin] >= (1ll << 31) || ext[d.vout] >= (1ll << 31)) d.tile_ok = 0;
  d.nbatch = 1;
  for (int v = 0; v < n; ++v)
    if (v != d.vin && v != d.vout && v != d.vin2 && v != d.vout2) {
      d.rest[d.nrest++] = v;
      d.nbatch *= ext[v];
    }
  *out = d;
  return true;
}

// Block decomposition for ce_blockperm_kernel (see there); false when no block of
// <= BP_MAX elements covers 32-element runs on both sides.
struct BpAx {
  int64_t ext, sa, sc;
  int64_t coef[2];  // gather coefficients
  bool in;
};

bool blk_build(std::vector<BpAx> ax, int ng, const int64_t* gstride, CeBlkPermDesc* out) {
  int64_t S = 1;
  auto key_in = [&](const BpAx& a) {  // input-side stride (gathered axes: through the gather)
    int64_t k = a.sa;
    for (int g = 0; g < ng; ++g) k += std::llabs(a.coef[g]) * gstride[g];
    return k;
  };
  auto add = [&](std::size_t i, int64_t q) {  // take q (| ext) of axis i into the block
    if (q < ax[i].ext)
      ax.push_back({ax[i].ext / q, ax[i].sa * q, ax[i].sc * q, {ax[i].coef[0] * q, ax[i].coef[1] * q}, false});
    ax[i].ext = q;
    ax[i].in = true;
    S *= q;
  };
  auto sorted = [&](bool by_out) {
    std::vector<std::size_t> o(ax.size());
    for (std::size_t i = 0; i < o.size(); ++i) o[i] = i;
    std::stable_sort(o.begin(), o.end(), [&](std::size_t x, std::size_t y) {
      return by_out ? ax[x].sc < ax[y].sc : key_in(ax[x]) < key_in(ax[y]);
    });
    return o;
  };
  // each side's stride-order prefix must cover >= 32 elements; an axis that overshoots is
  // split at its smallest sufficient divisor (its outer part stays a separate axis)
  for (bool by_out : {true, false}) {
    bool done = false;
    for (int guard = 0; guard < 2 * CE_MAX_VARS && !done; ++guard) {
      int64_t prod = 1;
      bool added = false;
      for (std::size_t i : sorted(by_out)) {
        if (prod >= 32) break;
        if (ax[i].in) {
          prod *= ax[i].ext;
          continue;
        }
        int64_t q = 2;
        while (q < ax[i].ext && (ax[i].ext % q || prod * q < 32)) ++q;
        q = std::min(q, ax[i].ext);
        if (S * q > BP_MAX) return false;
        add(i, q);
        added = true;
        break;
      }
      if (!added) {
        if (prod < 32) return false;
        done = true;
      }
    }
    if (!done) return false;
  }
  // grow along the output order to ~1024 elements (fewer batch iterations, longer store runs)
  for (std::size_t i : sorted(true)) {
    if (S >= 1024) break;
    if (ax[i].in) continue;
    if (S * ax[i].ext <= BP_MAX) {
      add(i, ax[i].ext);
      continue;
    }
    int64_t q = BP_MAX / S;
    while (q >= 2 && ax[i].ext % q) --q;
    if (q >= 2) add(i, q);
    break;
  }
  CeBlkPermDesc d{};
  d.S = static_cast<int32_t>(S);
  int64_t span_a = 0, span_c = 0, nb = 1, pos = 1;
  std::vector<int64_t> opos(ax.size(), 0);
  for (std::size_t i : sorted(true)) {
    if (!ax[i].in) continue;
    if (d.no >= BP_AX) return false;
    d.oext[d.no] = static_cast<int32_t>(ax[i].ext);
    d.odiv[d.no] = tc_div(static_cast<uint32_t>(ax[i].ext));
    d.osc[d.no] = static_cast<int32_t>(ax[i].sc);
    ++d.no;
    opos[i] = pos;
    pos *= ax[i].ext;
    span_c += (ax[i].ext - 1) * ax[i].sc;
  }
  for (std::size_t i : sorted(false)) {
    if (!ax[i].in) {
      if (d.nr >= CE_MAX_VARS) return false;
      d.rext[d.nr] = static_cast<uint32_t>(ax[i].ext);
      d.rdiv[d.nr] = tc_div(static_cast<uint32_t>(ax[i].ext));
      d.rsa[d.nr] = ax[i].sa;
      d.rsc[d.nr] = ax[i].sc;
      for (int g = 0; g < ng; ++g) {
        if (std::llabs(ax[i].coef[g]) * ax[i].ext >= (1ll << 30)) return false;
        d.rcoef[g][d.nr] = static_cast<int32_t>(ax[i].coef[g]);
      }
      ++d.nr;
      nb *= ax[i].ext;
      continue;
    }
    if (d.ni >= BP_AX) return false;
    d.iext[d.ni] = static_cast<int32_t>(ax[i].ext);
    d.idiv[d.ni] = tc_div(static_cast<uint32_t>(ax[i].ext));
    d.isa[d.ni] = static_cast<int32_t>(ax[i].sa);
    d.ipos[d.ni] = static_cast<int32_t>(opos[i]);
    for (int g = 0; g < ng; ++g) d.icoef[g][d.ni] = static_cast<int32_t>(ax[i].coef[g]);
    ++d.ni;
    span_a += (ax[i].ext - 1) * key_in(ax[i]);
  }
  d.ng = ng;
  if (span_a >= (1ll << 31) || span_c >= (1ll << 31) || nb >= (1ll << 31)) return false;
  d.nbatch = static_cast<uint32_t>(nb);
  *out = d;
  return true;
}


bool blkperm_desc(const CePermDesc& pd, CeBlkPermDesc* out) {
  std::vector<BpAx> ax;
  for (int v = 0; v < CE_MAX_VARS; ++v)
    if (pd.ext[v] > 1) ax.push_back({pd.ext[v], pd.sa[v], pd.sc[v], {0, 0}, false});
  return blk_build(ax, 0, nullptr, out);
}

// auto: the block kernel where the 2-axis tile kernels leave most of a tile idle
bool use_blkperm(const CePermDesc& d, CeBlkPermDesc* bp) {
  static const int mode = [] {  // CE_PERM_BLOCK: 0 never, 1 whenever viable, unset = auto
    const char* e = std::getenv("CE_PERM_BLOCK");
    return e ? std::atoi(e) : -1;
  }();
  if (!d.tile_ok) return blkperm_desc(d, bp);
  if (mode == 0 || !blkperm_desc(d, bp)) return false;
  if (mode == 1) return true;
  // small packs (factor matrices, a few MB) run as fast on the tile kernels' wider grids
  if (static_cast<int64_t>(bp->S) * bp->nbatch < (int64_t{1} << 22)) return false;
  if (d.same) return d.ext[d.vin] < 12 || d.ext[d.vin] * d.ext[d.vout] < 1024;
  const int64_t ein = d.ext[d.vin] * (d.vin2 >= 0 ? d.ext[d.vin2] : 1);
  const int64_t eout = d.ext[d.vout] * (d.vout2 >= 0 ? d.ext[d.vout2] : 1);
  return ein < 32 || eout < 32;
}
}  // namespace

namespace {
template <int NG>
cudaError_t blk_launch_ng(const CeBlkPermDesc& bp, const float* A, float* C, cudaStream_t s) {
  const dim3 grid(std::min<uint32_t>(bp.nbatch, 148 * 4));
  if (bp.S <= 256) return ce_launch(ce_blockperm_kernel<1, NG>, grid, dim3(256), 0, s, bp, A, C);
  if (bp.S <= 512) return ce_launch(ce_blockperm_kernel<2, NG>, grid, dim3(256), 0, s, bp, A, C);
  if (bp.S <= 1024) return ce_launch(ce_blockperm_kernel<4, NG>, grid, dim3(256), 0, s, bp, A, C);
  return ce_launch(ce_blockperm_kernel<8, NG>, grid, dim3(256), 0, s, bp, A, C);
}
cudaError_t blk_launch(const CeBlkPermDesc& bp, const float* A, float* C, cudaStream_t s) {
  if (bp.nbatch == 0) return cudaSuccess;
  switch (bp.ng) {
    case 0: return blk_launch_ng<0>(bp, A, C, s);
    case 1: return blk_launch_ng<1>(bp, A, C, s);
    default: return blk_launch_ng<2>(bp, A, C, s);
  }
}

// Tap expansion (a unary step whose input is gathered, ce_exec.cpp expand()) as a block
// permute with gathered input axes; false if the problem is not of that form.
bool blkgather_desc(const CeProblem& p, CeBlkPermDesc* out) {
  static const bool on = [] {
    const char* e = std::getenv("CE_BLK_GATHER");
    return !(e && *e == '0');
  }();
  if (!on || !p.unary || p.ng_a < 1 || p.ng_a > 2 || p.ng_b) return false;
  int64_t gstride[2] = {0, 0};
  for (int g = 0; g < p.ng_a; ++g) {
    if (p.ga[g].wrap || p.ga[g].extent >= (1ll << 30) || std::llabs(p.ga[g].c) >= (1ll << 30)) return false;
    gstride[g] = p.ga[g].stride;
  }
  std::vector<BpAx> ax;
  for (int v = 0; v < p.nv; ++v) {
    if (p.ext[v] <= 1) continue;
    if (p.cls[v] == CE_K || p.sc[v] == 0) return false;
    BpAx a{p.ext[v], p.sa[v], p.sc[v], {0, 0}, false};
    for (int g = 0; g < p.ng_a; ++g)
      a.coef[g] = (p.ga[g].pv == v ? p.ga[g].sp : 0) + (p.ga[g].qv == v ? p.ga[g].sq : 0);
    ax.push_back(a);
  }
  CeBlkPermDesc d;
  if (!blk_build(ax, p.ng_a, gstride, &d)) return false;
  for (int g = 0; g < p.ng_a; ++g) {
    d.gc[g] = static_cast<int32_t>(p.ga[g].c);
    d.gext[g] = static_cast<int32_t>(p.ga[g].extent);
    d.gstride[g] = gstride[g];
  }
  *out = d;
  return true;
}
}  // namespace

int ce_permute_describe(const CeProblem& p, char* buf, int n) {
  CePermDesc d;
  if (!perm_desc(p, &d)) return std::snprintf(buf, n, "unsupported");
  CeBlkPermDesc bp;
  if (use_blkperm(d, &bp)) {
    int k = std::snprintf(buf, n, "block S=%d ni=%d no=%d batch=%u |", bp.S, bp.ni, bp.no, bp.nbatch);
    for (int v = 0; v < CE_MAX_VARS && k < n; ++v)
      if (d.ext[v] > 0) k += std::snprintf(buf + k, n - k, " %lld:%lld/%lld", (long long)d.ext[v], (long long)d.sa[v],
                                           (long long)d.sc[v]);
    return k;
  }
  int k = std::snprintf(buf, n, "%s vin=%d vout=%d vin2=%d vout2=%d |", d.same ? "rowcopy" : "transpose", d.vin, d.vout,
                        d.vin2, d.vout2);
  for (int v = 0; v < CE_MAX_VARS && k < n; ++v)
    if (d.ext[v] > 0) k += std::snprintf(buf + k, n - k, " %lld:%lld/%lld", (long long)d.ext[v], (long long)d.sa[v],
                                         (long long)d.sc[v]);
  return k;
}

bool ce_permute_supported(const CeProblem& p) {
  CePermDesc d;
  CeBlkPermDesc bp;
  return perm_desc(p, &d) && (d.tile_ok || blkperm_desc(d, &bp));
}

cudaError_t ce_launch_permute(const CeProblem& p, const float* A, float* C, cudaStream_t s) {
  CePermDesc d;
  if (!perm_desc(p, &d)) return cudaErrorInvalidValue;
  CeBlkPermDesc bp;
  if (use_blkperm(d, &bp)) {
    if (bp.nbatch == 0) return cudaSuccess;
    const dim3 grid(std::min<uint32_t>(bp.nbatch, 148 * 4));
    return blk_launch(bp, A, C, s);
  }
  if (d.same) {
    bool v4 = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
              d.ext[d.vin] % 4 == 0 && d.sa[d.vout] % 4 == 0 && d.sc[d.vout] % 4 == 0;
    for (int i = 0; i < d.nrest; ++i) v4 = v4 && d.sa[d.rest[i]] % 4 == 0 && d.sc[d.rest[i]] % 4 == 0;
    const int64_t ex = d.ext[d.vin] / (v4 ? 4 : 1);
    int lshift = 0;
    while (lshift < 5 && (1ll << lshift) < ex) ++lshift;
    const int64_t rows_per_cta = (256 >> lshift) * 4;
    const int64_t per_slice = (d.ext[d.vout] + rows_per_cta - 1) / rows_per_cta;
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(per_slice, (148 * 16 + d.nbatch - 1) / d.nbatch));
    const int64_t gy = std::min<int64_t>(d.nbatch, 65535);
    const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
    if (v4) return ce_launch(ce_rowcopy_kernel<true>, grid, dim3(256), 0, s, d, A, C, lshift);
    return ce_launch(ce_rowcopy_kernel<false>, grid, dim3(256), 0, s, d, A, C, lshift);
  }
  const int64_t ein = d.ext[d.vin] * (d.vin2 >= 0 ? d.ext[d.vin2] : 1);
  const int64_t eout = d.ext[d.vout] * (d.vout2 >= 0 ? d.ext[d.vout2] : 1);
  if (ein >= 16 && eout >= 16) {
    // vector paths need every row start 16-B aligned on that side
    bool vi = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && ein % 4 == 0 && d.sa[d.vout] % 4 == 0 &&
              (d.vout2 < 0 || d.sa[d.vout2] % 4 == 0);
    bool vo = (reinterpret_cast<uintptr_t>(C) & 15) == 0 && eout % 4 == 0 && d.sc[d.vin] % 4 == 0 &&
              (d.vin2 < 0 || d.sc[d.vin2] % 4 == 0);
    for (int i = 0; i < d.nrest; ++i) {
      vi = vi && d.sa[d.rest[i]] % 4 == 0;
      vo = vo && d.sc[d.rest[i]] % 4 == 0;
    }
    const int64_t gx = (ein + 63) / 64, gy = (eout + 63) / 64;
    if (gx <= 0x7fffffff && gy <= 65535) {
      // enough CTAs to fill the machine, batch slices looped beyond that
      const int64_t gz = std::max<int64_t>(1, std::min<int64_t>({d.nbatch, 65535, (148 * 24 + gx * gy - 1) / (gx * gy)}));
      const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(gz));
      if (vi && vo) return ce_launch(ce_transpose64_kernel<true, true>, grid, dim3(256), 0, s, d, A, C);
      if (vi) return ce_launch(ce_transpose64_kernel<true, false>, grid, dim3(256), 0, s, d, A, C);
      if (vo) return ce_launch(ce_transpose64_kernel<false, true>, grid, dim3(256), 0, s, d, A, C);
      return ce_launch(ce_transpose64_kernel<false, false>, grid, dim3(256), 0, s, d, A, C);
    }
  }
  const int64_t gx = (ein + 31) / 32, gy = (eout + 31) / 32;
  if (gx > 0x7fffffff || gy > 65535) return cudaErrorInvalidConfiguration;
  const int64_t gz = std::min<int64_t>(d.nbatch, 65535);
  return ce_launch(ce_transpose_kernel,
                   dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(gz)), dim3(256), 0,
                   s, d, A, C);
}

cudaError_t ce_launch_fill(float* dst, int64_t n, uint64_t seed, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  return ce_launch(ce_fill_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, dst, n, seed);
}
