// Node fusion along plan chains: two consecutive depthwise stencils, e.g. the
// CP layer's `bhwr,rh->bhwr` then `bhwr,rw->bhwr` (layers.cpp:184-190; the reference
// materialises every node, sequencer.cpp:421-433), or their input-gradient adjoints in the
// backward pass, run as ONE separable 2-D stencil pass:
//
//   Y1[.., u, v, r] = sum_p Fa[r, p] Y0[.., xa(u, p), v, r]          (first node, axis u)
//   Y2[.., u, w, r] = sum_q Fb[r, q] Y1[.., u, xb(w, q), r]          (second node, axis v)
//
// with xa / xb the gathered feature indices of kernels.cpp:298-315 (or their adjoints,
// SURVEY A11).  A thread owns 4 lanes of r (float4) x J consecutive outputs along w: the
// J+KT-1 values of Y1 its window needs are computed in registers from Y0 (KT loads each) and
// never round-trip through HBM; Y1 is stored only when a later step reads it (the backward
// pass's filter gradient), and then only the thread's own J positions.  HBM traffic: |Y0| +
// |Y2| (+ |Y1|) instead of 2|Y0| + 2|Y1|-ish for the two stencil launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ce_fuse.h"
#include "ce_launch.h"

namespace {

// CTA tile: lq lane quads (4 lanes each) x kUT rows along u x njb*J outputs along w (+ one
// outer index), lq * kUT * njb = 256 threads (the host picks lq / njb from the lane and w
// extents).  Stage 1: each (quad, Y1 column) item slides down u with a register window of
// kUT+KT-1 rows of Y0 and writes kUT values of Y1 to shared memory (and, when a later step
// reads Y1, the tile's own columns to global).  Stage 2: each thread computes J consecutive
// Y2 outputs of one row from a J+KT-1 window of the shared Y1 tile.  Global loads per Y2
// output: (kUT+KT-1)/kUT * (WT+KT-1)/WT, instead of ~2 (J+KT-1)/J for two stencil launches
// plus the Y1 round trip.
constexpr int kDw2Threads = 256, kUT = 8, kJ = 8;  // stage-2 threads; stage 1 uses all lq * NC

template <int KT, int SA, int SB>
__global__ void __launch_bounds__(512) ce_dw2_kernel(const CeDw2Desc d, const float* __restrict__ Y0,
                                                              const float* __restrict__ Fa,
                                                              const float* __restrict__ Fb, float* __restrict__ Y1,
                                                              float* __restrict__ Y2) {
  constexpr int TMIN = SB > 0 ? 0 : -(KT - 1);
  const int lq = d.lq, njb = d.njb, WT = njb * kJ, NC = WT + KT - 1;
  extern __shared__ float4 sy1[];  // [kUT][NC][lq]
  ce_pdl_enter();
  // tile decode: blockIdx.x = lane chunk (fastest), w tile, u tile, outer index
  uint32_t rest = blockIdx.x;
  uint32_t q = tc_quo(rest, d.dr4);  // dr4: lane chunks of lq quads
  const int32_t lc = static_cast<int32_t>(rest - q * d.dr4.d);
  rest = q;
  q = tc_quo(rest, d.dwb);
  const int32_t w0 = static_cast<int32_t>(rest - q * d.dwb.d) * WT;
  rest = q;
  q = tc_quo(rest, d.du);
  const int32_t u0 = static_cast<int32_t>(rest - q * d.du.d) * kUT;
  rest = q;
  int64_t o0 = 0, o1 = 0, o2 = 0;
#pragma unroll
  for (int i = 0; i < CE_DW2_OUTER; ++i) {
    if (i < d.nouter) {
      const uint32_t qq = tc_quo(rest, d.odiv[i]);
      const int64_t v = static_cast<int64_t>(rest - qq * d.odiv[i].d);
      rest = qq;
      o0 += v * d.os0[i];
      o1 += v * d.os1[i];
      o2 += v * d.os2[i];
    }
  }
  const int tid = threadIdx.x;
  const int quad = tid % lq;
  const int32_t lane0 = (lc * lq + quad) * 4;
  const bool lanes_in = lane0 < d.R;
  // ---- stage 1: Y1 columns x = xlo + c, c in [0, NC)
  const int32_t xlo = d.cb + w0 + TMIN;
  {
    float fa[KT][4];
#pragma unroll
    for (int p = 0; p < KT; ++p)
#pragma unroll
      for (int e = 0; e < 4; ++e) fa[p][e] = lane0 + e < d.R ? __ldg(Fa + (lane0 + e) * d.fa_r + p * d.fa_q) : 0.f;
    // rows t of Y0 the window needs: xa(u, p) = ca + u + SA*p over u in [u0, u0+kUT)
    constexpr int RMIN = SA > 0 ? 0 : -(KT - 1);
    constexpr int NR = kUT + KT - 1;
    {
      const int c = tid / lq;  // blockDim = lq * NC: one Y1 column per thread
      const int32_t x = xlo + c;
      float4 y[kUT];
#pragma unroll
      for (int i = 0; i < kUT; ++i) y[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lanes_in && static_cast<uint32_t>(x) < static_cast<uint32_t>(d.Xb)) {
        const float* base = Y0 + o0 + lane0 + static_cast<int64_t>(x) * d.v0;
        float4 rw[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int32_t t = d.ca + u0 + RMIN + r;
          rw[r] = static_cast<uint32_t>(t) < static_cast<uint32_t>(d.Xa)
                      ? __ldg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(t) * d.a0))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < kUT; ++i)
#pragma unroll
          for (int p = 0; p < KT; ++p) {
            const float4 r = rw[i + SA * p - RMIN];
            y[i].x += r.x * fa[p][0];
            y[i].y += r.y * fa[p][1];
            y[i].z += r.z * fa[p][2];
            y[i].w += r.w * fa[p][3];
          }
        // the tile's own Y1 columns (x in [w0, w0+WT)) go to global when a later step reads Y1
        if (Y1 != nullptr && x >= w0 && x < w0 + WT) {
          float* dst = Y1 + o1 + lane0 + static_cast<int64_t>(x) * d.v1;
#pragma unroll
          for (int i = 0; i < kUT; ++i)
            if (u0 + i < d.U) *reinterpret_cast<float4*>(dst + static_cast<int64_t>(u0 + i) * d.u1) = y[i];
        }
      }
#pragma unroll
      for (int i = 0; i < kUT; ++i) sy1[(i * NC + c) * lq + quad] = y[i];
    }
  }
  __syncthreads();
  // ---- stage 2: thread -> (quad, row i, w block jb)
  {
    const int i = (tid / lq) % kUT, jb = tid / (lq * kUT);
    const int32_t u = u0 + i, wj = w0 + jb * kJ;
    if (!lanes_in || u >= d.U || jb >= njb || tid >= kDw2Threads) return;
    float fb[KT][4];
#pragma unroll
    for (int p = 0; p < KT; ++p)
#pragma unroll
      for (int e = 0; e < 4; ++e) fb[p][e] = lane0 + e < d.R ? __ldg(Fb + (lane0 + e) * d.fb_r + p * d.fb_q) : 0.f;
    float4 win[kJ + KT - 1];
#pragma unroll
    for (int k = 0; k < kJ + KT - 1; ++k) win[k] = sy1[(i * NC + jb * kJ + k) * lq + quad];
    float* dst = Y2 + o2 + lane0 + static_cast<int64_t>(u) * d.u2;
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj) {
      if (wj + jj >= d.W) break;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int qq = 0; qq < KT; ++qq) {
        const float4 r = win[jj + SB * qq - TMIN];
        acc.x += r.x * fb[qq][0];
        acc.y += r.y * fb[qq][1];
        acc.z += r.z * fb[qq][2];
        acc.w += r.w * fb[qq][3];
      }
      *reinterpret_cast<float4*>(dst + static_cast<int64_t>(wj + jj) * d.w2) = acc;
    }
  }
}

// One depthwise stencil step in the canonical form the fused kernel needs.
struct Stencil {
  int lane = -1, conv = -1, tap = -1;  // vars: lane (batch, unit stride), conv output, tap
  int64_t ca = 0;                       // gather constant
  int sq = 0;                           // tap coefficient (+1 / -1)
  int64_t X = 0, gstride = 0;           // feature extent and A stride of the gathered axis
  std::vector<int> plain;               // other vars: plain in A and C, absent from B
};

bool as_stencil(const CeProblem& p, Stencil* s) {
  if (p.unary || p.accumulate || p.ng_a != 1 || p.ng_b != 0) return false;
  const CeGather& g = p.ga[0];
  if (g.wrap || g.sp != 1 || (g.sq != 1 && g.sq != -1)) return false;
  s->conv = g.pv;
  s->tap = g.qv;
  s->ca = g.c;
  s->sq = g.sq;
  s->X = g.extent;
  s->gstride = g.stride;
  if (p.cls[s->tap] != CE_K || p.sa[s->tap] || !p.sb[s->tap] || p.sc[s->tap]) return false;
  if (p.ext[s->tap] != 3 && p.ext[s->tap] != 5 && p.ext[s->tap] != 7) return false;
  if (p.sa[s->conv] || p.sb[s->conv] || !p.sc[s->conv]) return false;
  for (int v = 0; v < p.nv; ++v) {
    if (v == s->conv || v == s->tap || p.ext[v] == 1) continue;
    if (p.cls[v] == CE_K) return false;  // the tap is the only contracted var
    if (p.sa[v] == 1 && p.sc[v] == 1 && p.sb[v]) {
      if (s->lane >= 0) return false;
      s->lane = v;
    } else if (p.sa[v] && p.sc[v] && !p.sb[v]) {
      s->plain.push_back(v);
    } else {
      return false;
    }
  }
  return s->lane >= 0;
}

int64_t pad4(int64_t x) { return (x + 3) / 4 * 4; }

}  // namespace

bool ce_dw2_plan(const CeProblem& p1, const CeProblem& p2, bool write_mid, CeDw2Desc* out) {
  Stencil s1, s2;
  if (!as_stencil(p1, &s1) || !as_stencil(p2, &s2)) return false;
  const int KT = static_cast<int>(p1.ext[s1.tap]);
  if (p2.ext[s2.tap] != KT) return false;
  CeDw2Desc d{};
  const int64_t R = p1.ext[s1.lane];
  if (p2.ext[s2.lane] != R || p2.sa[s2.lane] != 1) return false;
  // rows of Y0 / Y1 / Y2 hold a 16-B padded lane run (float4 loads and stores of the pad)
  auto lane_ok = [&](const CeProblem& p, const Stencil& s, bool a_side) {
    const int64_t* st = a_side ? p.sa : p.sc;
    for (int v : s.plain)
      if (st[v] % 4 || st[v] < pad4(R)) return false;
    if (a_side && (s.gstride % 4 || s.gstride < pad4(R))) return false;
    if (!a_side && (p.sc[s.conv] % 4 || p.sc[s.conv] < pad4(R))) return false;
    return true;
  };
  if (!lane_ok(p1, s1, true) || !lane_ok(p1, s1, false) || !lane_ok(p2, s2, true) || !lane_ok(p2, s2, false))
    return false;
  // the second step's gathered axis v must be a plain axis of Y1 (the first step's output)
  int v1 = -1;
  for (int v : s1.plain)
    if (p1.sc[v] == s2.gstride && p1.ext[v] == s2.X) v1 = v;
  if (v1 < 0) return false;
  // every other Y1 axis of the second step matches a Y1 axis of the first by stride and extent;
  // the first step's conv axis u becomes a plain axis of the second
  int u2 = -1;
  std::vector<std::pair<int, int>> outer;  // (var in p1, var in p2)
  for (int v : s2.plain) {
    if (p2.sa[v] == p1.sc[s1.conv] && p2.ext[v] == p1.ext[s1.conv]) {
      u2 = v;
      continue;
    }
    int m = -1;
    for (int w : s1.plain)
      if (w != v1 && p1.sc[w] == p2.sa[v] && p1.ext[w] == p2.ext[v]) m = w;
    if (m < 0) return false;
    outer.push_back({m, v});
  }
  if (u2 < 0 || outer.size() + 2 != s1.plain.size() + 1 || static_cast<int>(outer.size()) > CE_DW2_OUTER) return false;
  // tile shape: njb blocks of kJ outputs along w (power of two covering W, <= 8) and lq lane
  // quads, lq * kUT * njb = 256 threads; narrow lane extents trade quads for w blocks
  const int TMIN = s2.sq > 0 ? 0 : -(KT - 1);
  const int64_t W = p2.ext[s2.conv];
  const int64_t r4 = (R + 3) / 4;
  int njb = 1;
  while (njb < 8 && njb * kJ < W) njb *= 2;
  int lq = kDw2Threads / (kUT * njb);
  while (lq > 2 * r4 && lq > 1 && njb < 8 && njb * kJ < 2 * W) {
    lq /= 2;
    njb *= 2;
  }
  const int WT = njb * kJ;
  if (write_mid) {
    // every Y1 position x in [0, Xb) is stored by exactly one tile, from its halo'd columns
    const int64_t wb = (W + WT - 1) / WT;
    if (wb * WT < s2.X || -s2.ca - TMIN < 0 || -s2.ca - TMIN > KT - 1) return false;
  }
  d.KT = KT;
  d.J = kJ;
  d.lq = lq;
  d.njb = njb;
  d.SA = s1.sq;
  d.SB = s2.sq;
  d.R = static_cast<int32_t>(R);
  const int64_t lchunks = (r4 + lq - 1) / lq, wbk = (W + WT - 1) / WT, U = p1.ext[s1.conv];
  const int64_t ut = (U + kUT - 1) / kUT;
  d.dr4 = tc_div(static_cast<uint32_t>(lchunks));
  d.dwb = tc_div(static_cast<uint32_t>(wbk));
  d.du = tc_div(static_cast<uint32_t>(ut));
  d.U = static_cast<int32_t>(U);
  double threads = static_cast<double>(lchunks * wbk * ut);  // CTAs
  d.nouter = static_cast<int32_t>(outer.size());
  for (std::size_t i = 0; i < outer.size(); ++i) {
    const int a = outer[i].first, b = outer[i].second;
    d.odiv[i] = tc_div(static_cast<uint32_t>(p1.ext[a]));
    d.os0[i] = p1.sa[a];
    d.os1[i] = p1.sc[a];
    d.os2[i] = p2.sc[b];
    threads *= static_cast<double>(p1.ext[a]);
  }
  if (threads >= 2147483647.0 || U >= (1 << 30) || W >= (1 << 30) || s1.X >= (1 << 30) || s2.X >= (1 << 30))
    return false;
  d.threads = static_cast<uint32_t>(threads);
  d.ca = static_cast<int32_t>(s1.ca);
  d.Xa = static_cast<int32_t>(s1.X);
  d.a0 = s1.gstride;
  d.v0 = p1.sa[v1];
  d.u1 = p1.sc[s1.conv];
  d.u2 = p2.sc[u2];
  d.cb = static_cast<int32_t>(s2.ca);
  d.Xb = static_cast<int32_t>(s2.X);
  d.v1 = s2.gstride;
  d.W = static_cast<int32_t>(W);
  d.w2 = p2.sc[s2.conv];
  d.fa_r = static_cast<int32_t>(p1.sb[s1.lane]);
  d.fa_q = static_cast<int32_t>(p1.sb[s1.tap]);
  d.fb_r = static_cast<int32_t>(p2.sb[s2.lane]);
  d.fb_q = static_cast<int32_t>(p2.sb[s2.tap]);
  d.write_mid = write_mid ? 1 : 0;
  *out = d;
  return true;
}

cudaError_t ce_launch_dw2(const CeDw2Desc& d, const float* Y0, const float* Fa, const float* Fb, float* Y1, float* Y2,
                          cudaStream_t s) {
  if (d.threads == 0) return cudaSuccess;
  if (!d.write_mid) Y1 = nullptr;
  const dim3 grid(d.threads), blk(d.lq * (d.njb * kJ + d.KT - 1));  // d.threads counts CTAs
  const size_t smem = static_cast<size_t>(kUT) * (d.njb * kJ + d.KT - 1) * d.lq * sizeof(float4);
  auto go = [&](void (*k)(CeDw2Desc, const float*, const float*, const float*, float*, float*)) -> cudaError_t {
    if (smem > 48 * 1024) {  // opt-in above 48 KB (lq = 32 tiles with 7 taps: 57 KB); per device
      int dev = 0;
      cudaGetDevice(&dev);
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      if (e != cudaSuccess) return e;
    }
    return ce_launch(k, grid, blk, smem, s, d, Y0, Fa, Fb, Y1, Y2);
  };
#define CE_DW2(KT)                                                                                           \
  if (d.SA > 0 && d.SB > 0) return go(ce_dw2_kernel<KT, 1, 1>);                                              \
  if (d.SA > 0 && d.SB < 0) return go(ce_dw2_kernel<KT, 1, -1>);                                             \
  if (d.SA < 0 && d.SB > 0) return go(ce_dw2_kernel<KT, -1, 1>);                                             \
  return go(ce_dw2_kernel<KT, -1, -1>);
  if (d.KT == 3) { CE_DW2(3) }
  if (d.KT == 5) { CE_DW2(5) }
  CE_DW2(7)
#undef CE_DW2
}

// 3xTF32 operand split (CE_MATH_3XTF32): hi = x rounded to TF32 (cvt.rna), lo = x - hi (exact in
// FP32); the step then runs as hi*hi + hi*lo + lo*hi on the tensor cores, ~FP32 accuracy.
namespace {
__global__ void __launch_bounds__(256) ce_split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi,
                                                            float* __restrict__ lo, int64_t n) {
  ce_pdl_enter();
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * 256) {
    const float v = x[i];
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
    const float h = __uint_as_float(t);
    hi[i] = h;
    lo[i] = v - h;
  }
}
}  // namespace

cudaError_t ce_launch_split_tf32(const float* x, float* hi, float* lo, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  return ce_launch(ce_split_tf32_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, x, hi, lo, n);
}
