// Plane convolutions with few channels (ce_pconv.h).
//
// A step qualifies when its feature operand F (operand A) is gathered along exactly two axes
// (position p, tap q: feature index = p + sign * q + c, or the adjoint form with the roles of
// p and q swapped) and every other var is a "plane" var (F and the output), a contracted
// channel ci (F and the filter), or an output channel co (filter and output), with at most 16
// channels each side.  This is the shape of the reference's grouped_conv_core
// (kernels.cpp:320-399) for a conv atom shared by the input and one small factor, e.g. RTR
// conv1 (layers.cpp:263-275): X[b, s3, h, w] against W4[r3, r0, i, j], 3 planes of 112x112 per
// sample, 7x7 taps, 9 output channels.
//
// kind 0 (forward, and the input gradient, which has the same form with the tap sign
// flipped): a CTA owns one plane and a 16 x 32 position tile; it stages the tile's input
// window (16 + KH - 1) x (32 + KW - 1) x Ci and the whole filter in shared memory, then each
// thread accumulates 4 positions x Co outputs over Ci x KH x KW terms (the filter values are
// warp-uniform broadcasts).  Compulsory traffic |F| + |C| (+ the halo re-reads, served by L2).
//
// kind 1 (filter gradient): persistent CTAs walk (plane, tile) items; per item the input
// window and the output-gradient tile are staged, and thread (i, ci, co, row group)
// accumulates the KW taps of one filter row over its rows of the tile in registers.  At the
// end the row groups are summed in shared memory and each CTA adds its partial filter
// gradient with one atomic per element.
#include "ce_pconv.h"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace {

constexpr int kMaxTap = 8;

// kind 0 tile: 32 x 32 positions, 128 threads; thread (ty, xg) owns row ty, positions
// 8 xg .. 8 xg + 7, so for each (filter row, ci) it loads its 8 + KW - 1 window once (float4)
// and reuses it for all KW taps: (8 + KW - 1) / 4 + KW * CO shared loads per 8 KW CO FMAs.
constexpr int kTY0 = 32, kTX0 = 32;
// kind 1 tile: 16 x 32 positions, 256 threads
constexpr int kTY1 = 16, kTX1 = 32;

__host__ __device__ constexpr int pad4(int x) { return (x + 3) / 4 * 4; }

template <int CO, int KW>
__global__ void __launch_bounds__(128) ce_pconv_kernel(const CePconvDesc d, const float* __restrict__ F,
                                                       const float* __restrict__ G, float* __restrict__ C) {
  extern __shared__ __align__(16) float sm[];
  constexpr int TXP = pad4(kTX0 + KW - 1 + 4);  // window row pitch (the last float4 may run past)
  constexpr int WIN = pad4(8 + KW - 1);
  const int KH = d.KH, Ci = d.Ci;
  const int TYH = kTY0 + KH - 1;
  float* sw = sm;                                // [KH][KW][Ci][CO]
  float* sin = sm + pad4(KH * KW * Ci * CO);     // [Ci][TYH][TXP]
  int64_t bid = blockIdx.x;
  const int tx_t = static_cast<int>(bid % d.tiles_x);
  bid /= d.tiles_x;
  const int ty_t = static_cast<int>(bid % d.tiles_y);
  int64_t rem = bid / d.tiles_y;
  int64_t of = 0, oc = 0;
  for (int k = 0; k < d.npl; ++k) {
    const int64_t v = rem % d.pl_ext[k];
    rem /= d.pl_ext[k];
    of += v * d.pl_sf[k];
    oc += v * d.pl_so[k];
  }
  for (int e = threadIdx.x; e < KH * KW * Ci * CO; e += blockDim.x) {
    const int co = e % CO;
    const int r = e / CO;
    const int ci = r % Ci;
    const int t = r / Ci;
    // staged by window offset m: tap j = m (sign +1) or KW - 1 - m (sign -1)
    const int m = t % KW;
    const int j = d.sgn_w > 0 ? m : KW - 1 - m;
    sw[e] = co < d.Co ? G[(t / KW) * d.ti + j * d.tj + d.gci[ci] + d.gco[co]] : 0.f;
  }
  const int y0 = ty_t * kTY0, x0 = tx_t * kTX0;
  const int64_t hb = y0 + d.c_h - (d.sgn_h > 0 ? 0 : KH - 1);
  const int64_t wb = x0 + d.c_w - (d.sgn_w > 0 ? 0 : KW - 1);
  // one position per thread and iteration, its Ci channels in turn (adjacent in F for
  // channels-last inputs); no runtime divisions
  for (int r = threadIdx.x; r < TYH * TXP; r += blockDim.x) {
    const int hh = r / TXP, ww = r % TXP;
    const int64_t h = hb + hh, w = wb + ww;
    const bool in = ww < kTX0 + KW - 1 && h >= 0 && h < d.H && w >= 0 && w < d.W;
    const float* src = F + of + h * d.fh + w * d.fw;
    for (int ci = 0; ci < Ci; ++ci) sin[(ci * TYH + hh) * TXP + ww] = in ? src[d.fci[ci]] : 0.f;
  }
  __syncthreads();
  const int ty = threadIdx.x >> 2, xg = threadIdx.x & 3;
  float acc[8][CO];
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int c = 0; c < CO; ++c) acc[k][c] = 0.f;
  for (int i = 0; i < KH; ++i) {
    const int hh = ty + (d.sgn_h > 0 ? i : KH - 1 - i);
    for (int ci = 0; ci < Ci; ++ci) {
      const float4* row = reinterpret_cast<const float4*>(sin + (ci * TYH + hh) * TXP + 8 * xg);
      float win[WIN];
#pragma unroll
      for (int q = 0; q < WIN / 4; ++q) {
        const float4 v = row[q];
        win[4 * q] = v.x;
        win[4 * q + 1] = v.y;
        win[4 * q + 2] = v.z;
        win[4 * q + 3] = v.w;
      }
      const float* wp = sw + (i * KW * Ci + ci) * CO;
#pragma unroll
      for (int m = 0; m < KW; ++m) {
        float wv[CO];
#pragma unroll
        for (int c = 0; c < CO; ++c) wv[c] = wp[m * Ci * CO + c];
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int c = 0; c < CO; ++c) acc[k][c] = fmaf(win[k + m], wv[c], acc[k][c]);
      }
    }
  }
  // stage the tile's outputs [TY][TX][CO] and write them with consecutive threads on
  // consecutive (x, co): C's channels-last rows come out as contiguous runs
  __syncthreads();
  float* so = sm;
  constexpr int OP = kTX0 * CO + 1;  // row pitch = 1 mod 32: a warp's 8 rows in distinct banks
#pragma unroll
  for (int k = 0; k < 8; ++k)
#pragma unroll
    for (int c = 0; c < CO; ++c) so[ty * OP + (8 * xg + k) * CO + c] = acc[k][c];
  __syncthreads();
  const int Co = d.Co;
  // per-lane channel offsets from shared memory (indexing the kernel parameters with a
  // lane-dependent index would serialise the constant-bank reads)
  // (32-bit offsets inside the tile: the planner bounds the tile's span)
  __shared__ int s_cco[CO];
  if (threadIdx.x < CO) s_cco[threadIdx.x] = threadIdx.x < Co ? static_cast<int>(d.cco[threadIdx.x]) : 0;
  __syncthreads();
  float* cb = C + oc + static_cast<int64_t>(y0) * d.sy + static_cast<int64_t>(x0) * d.sx;
  const int syi = static_cast<int>(d.sy), sxi = static_cast<int>(d.sx);
  const int ylim = d.OY - y0, xlim = d.OX - x0;
  for (int e = threadIdx.x; e < kTY0 * kTX0 * CO; e += blockDim.x) {
    const int c = e % CO;
    const int r = e / CO;
    const int yy = r / kTX0, xx = r % kTX0;
    if (c >= Co || yy >= ylim || xx >= xlim) continue;
    float* p = cb + (yy * syi + xx * sxi + s_cco[c]);
    const float v = so[yy * OP + xx * CO + c];
    *p = d.accumulate ? *p + v : v;
  }
}

template <int KW>
__global__ void __launch_bounds__(256) ce_pconv_wgrad_kernel(const CePconvDesc d, const float* __restrict__ F,
                                                             const float* __restrict__ D, float* __restrict__ C) {
  extern __shared__ __align__(16) float sm[];
  constexpr int TXH = kTX1 + KW - 1;
  constexpr int TXP = TXH | 1;  // odd pitch: the filter rows of a warp's lanes fall in different banks
  const int KH = d.KH, Ci = d.Ci, Co = d.Co;
  const int TYH = kTY1 + KH - 1;
  float* sf = sm;                          // [Ci][TYH][TXP]
  float* sd = sm + Ci * TYH * TXP;         // [kTY1][kTX1][Co]
  const int owners = KH * Ci * Co;
  const int groups = max(1, static_cast<int>(blockDim.x) / owners);
  const int o = threadIdx.x % owners, rg = threadIdx.x / owners;
  const bool active = rg < groups;
  const int co = o % Co, ci = (o / Co) % Ci, i = o / (Co * Ci);
  const int ioff = d.sgn_h > 0 ? i : KH - 1 - i;
  float acc[KW];
#pragma unroll
  for (int j = 0; j < KW; ++j) acc[j] = 0.f;
  for (int64_t item = blockIdx.x; item < d.items; item += gridDim.x) {
    int64_t bid = item;
    const int tx_t = static_cast<int>(bid % d.tiles_x);
    bid /= d.tiles_x;
    const int ty_t = static_cast<int>(bid % d.tiles_y);
    int64_t rem = bid / d.tiles_y;
    int64_t of = 0, od = 0;
    for (int k = 0; k < d.npl; ++k) {
      const int64_t v = rem % d.pl_ext[k];
      rem /= d.pl_ext[k];
      of += v * d.pl_sf[k];
      od += v * d.pl_so[k];
    }
    const int y0 = ty_t * kTY1, x0 = tx_t * kTX1;
    const int64_t hb = y0 + d.c_h - (d.sgn_h > 0 ? 0 : KH - 1);
    const int64_t wb = x0 + d.c_w - (d.sgn_w > 0 ? 0 : KW - 1);
    __syncthreads();  // the previous item's tiles are consumed
    for (int r = threadIdx.x; r < TYH * TXH; r += blockDim.x) {
      const int hh = r / TXH, ww = r % TXH;
      const int64_t h = hb + hh, w = wb + ww;
      const bool in = h >= 0 && h < d.H && w >= 0 && w < d.W;
      const float* src = F + of + h * d.fh + w * d.fw;
      for (int c = 0; c < Ci; ++c) sf[(c * TYH + hh) * TXP + ww] = in ? src[d.fci[c]] : 0.f;
    }
    for (int r = threadIdx.x; r < kTY1 * kTX1; r += blockDim.x) {
      const int y = y0 + r / kTX1, x = x0 + r % kTX1;
      const bool in = y < d.OY && x < d.OX;
      const float* src = D + od + y * d.sy + x * d.sx;
      for (int c = 0; c < Co; ++c) sd[r * Co + c] = in ? src[d.gco[c]] : 0.f;
    }
    __syncthreads();
    if (!active) continue;
    for (int y = rg; y < kTY1; y += groups) {
      const float* fr = sf + (ci * TYH + y + ioff) * TXP;
      const float* dr = sd + y * kTX1 * Co + co;
      // register window over the row: position x reads F[x .. x + KW - 1]
      float win[KW];
#pragma unroll
      for (int m = 0; m < KW - 1; ++m) win[m] = fr[m];
#pragma unroll
      for (int x = 0; x < kTX1; ++x) {
        win[KW - 1] = fr[x + KW - 1];
        const float dv = dr[x * Co];
#pragma unroll
        for (int m = 0; m < KW; ++m) acc[m] = fmaf(win[m], dv, acc[m]);  // window offset m
#pragma unroll
        for (int m = 0; m < KW - 1; ++m) win[m] = win[m + 1];
      }
    }
  }
  // sum the row groups, one atomic per filter element per CTA
  __syncthreads();
  float* red = sm;  // [groups][owners][KW]
  if (active)
#pragma unroll
    for (int j = 0; j < KW; ++j) red[(rg * owners + o) * KW + j] = acc[j];
  __syncthreads();
  for (int e = threadIdx.x; e < owners * KW; e += blockDim.x) {
    float s = 0.f;
    for (int g = 0; g < groups; ++g) s += red[g * owners * KW + e];
    const int m = e % KW, oo = e / KW;
    const int j = d.sgn_w > 0 ? m : KW - 1 - m;  // window offset -> tap
    const int c_o = oo % Co, c_i = (oo / Co) % Ci, ii = oo / (Co * Ci);
    atomicAdd(C + ii * d.ti + j * d.tj + d.gci[c_i] + d.cco[c_o], s);
  }
}

int co_instance(int co) {
  for (int c : {1, 2, 3, 4, 6, 8, 9, 12, 16})
    if (co <= c) return c;
  return -1;
}

bool kw_supported(int kw) { return kw == 3 || kw == 5 || kw == 7; }

size_t fwd_smem(const CePconvDesc& d) {
  const int co = co_instance(d.Co);
  const int txp = pad4(kTX0 + d.KW - 1 + 4);
  const size_t in = static_cast<size_t>(pad4(d.KH * d.KW * d.Ci * co) + (kTY0 + d.KH - 1) * txp * d.Ci);
  const size_t out = static_cast<size_t>(kTY0 * (kTX0 * co + 1));
  return 4 * std::max(in, out);
}

size_t wgrad_smem(const CePconvDesc& d) {
  const int txp = (kTX1 + d.KW - 1) | 1;
  const size_t tiles = static_cast<size_t>((kTY1 + d.KH - 1) * txp * d.Ci + kTY1 * kTX1 * d.Co);
  const int owners = d.KH * d.Ci * d.Co;
  const size_t red = static_cast<size_t>(std::max(1, 256 / owners) * owners * d.KW);
  return 4 * std::max(tiles, red);
}

template <int CO, int KW>
cudaError_t launch_fwd(const CePconvDesc& d, const float* F, const float* G, float* C, cudaStream_t s) {
  const size_t smem = fwd_smem(d);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ce_pconv_kernel<CO, KW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = d.P * d.tiles_y * d.tiles_x;
  ce_pconv_kernel<CO, KW><<<static_cast<unsigned>(blocks), 128, smem, s>>>(d, F, G, C);
  return cudaGetLastError();
}

template <int KW>
cudaError_t launch_wgrad(const CePconvDesc& d, const float* F, const float* D, float* C, cudaStream_t s) {
  const size_t smem = wgrad_smem(d);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ce_pconv_wgrad_kernel<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  ce_pconv_wgrad_kernel<KW><<<static_cast<unsigned>(d.ctas), 256, smem, s>>>(d, F, D, C);
  return cudaGetLastError();
}

template <int KW>
cudaError_t launch_fwd_co(const CePconvDesc& d, const float* F, const float* G, float* C, cudaStream_t s) {
  switch (co_instance(d.Co)) {
    case 1: return launch_fwd<1, KW>(d, F, G, C, s);
    case 2: return launch_fwd<2, KW>(d, F, G, C, s);
    case 3: return launch_fwd<3, KW>(d, F, G, C, s);
    case 4: return launch_fwd<4, KW>(d, F, G, C, s);
    case 6: return launch_fwd<6, KW>(d, F, G, C, s);
    case 8: return launch_fwd<8, KW>(d, F, G, C, s);
    case 9: return launch_fwd<9, KW>(d, F, G, C, s);
    case 12: return launch_fwd<12, KW>(d, F, G, C, s);
    case 16: return launch_fwd<16, KW>(d, F, G, C, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool ce_pconv_plan(const CeProblem& p, CePconvDesc* out) {
  if (p.unary || p.ng_a != 2 || p.ng_b != 0) return false;
  CePconvDesc d{};
  const CeGather& g0 = p.ga[0].stride >= p.ga[1].stride ? p.ga[0] : p.ga[1];  // axis 0 = outer (h)
  const CeGather& g1 = p.ga[0].stride >= p.ga[1].stride ? p.ga[1] : p.ga[0];
  const CeGather* gs[2] = {&g0, &g1};
  // kind 0: pv = position (output), qv = tap (filter); kind 1: pv = tap (output), qv = position
  double b_elems = 1, c_elems = 1;
  for (int v = 0; v < p.nv; ++v) {
    if (p.sb[v]) b_elems *= static_cast<double>(p.ext[v]);
    if (p.sc[v]) c_elems *= static_cast<double>(p.ext[v]);
  }
  const int kind = b_elems <= 16384 ? 0 : (c_elems <= 16384 ? 1 : -1);
  if (kind < 0) return false;
  d.kind = kind;
  std::vector<char> used(static_cast<std::size_t>(p.nv), 0);
  int64_t posx[2], tapx[2], pos_s[2], tap_s[2];
  for (int a = 0; a < 2; ++a) {
    const CeGather& g = *gs[a];
    if (g.wrap || g.pv < 0 || g.qv < 0) return false;
    const int pos = kind == 0 ? g.pv : g.qv, tap = kind == 0 ? g.qv : g.pv;
    const int psign = kind == 0 ? g.sp : g.sq, tsign = kind == 0 ? g.sq : g.sp;
    if (psign != 1 || (tsign != 1 && tsign != -1)) return false;
    if (p.sa[pos] || p.sa[tap]) return false;
    if (kind == 0 && (p.cls[pos] == CE_K || !p.sc[pos] || p.sb[pos] || p.cls[tap] != CE_K || !p.sb[tap] || p.sc[tap]))
      return false;
    if (kind == 1 && (p.cls[pos] != CE_K || !p.sb[pos] || p.sc[pos] || p.cls[tap] == CE_K || !p.sc[tap] || p.sb[tap]))
      return false;
    used[static_cast<std::size_t>(pos)] = used[static_cast<std::size_t>(tap)] = 1;
    posx[a] = p.ext[pos];
    tapx[a] = p.ext[tap];
    pos_s[a] = kind == 0 ? p.sc[pos] : p.sb[pos];
    tap_s[a] = kind == 0 ? p.sb[tap] : p.sc[tap];
    (a == 0 ? d.sgn_h : d.sgn_w) = tsign;
    (a == 0 ? d.c_h : d.c_w) = g.c;
    (a == 0 ? d.H : d.W) = g.extent;
    (a == 0 ? d.fh : d.fw) = g.stride;
  }
  if (tapx[0] > kMaxTap || !kw_supported(static_cast<int>(tapx[1]))) return false;
  d.OY = static_cast<int32_t>(posx[0]);
  d.OX = static_cast<int32_t>(posx[1]);
  d.sy = pos_s[0];
  d.sx = pos_s[1];
  d.KH = static_cast<int32_t>(tapx[0]);
  d.KW = static_cast<int32_t>(tapx[1]);
  d.ti = tap_s[0];
  d.tj = tap_s[1];
  // remaining vars: planes, contracted channels ci, output channels co
  std::vector<int> ci_v, co_v;
  d.P = 1;
  for (int v = 0; v < p.nv; ++v) {
    if (used[static_cast<std::size_t>(v)] || p.ext[v] == 1) continue;
    const bool a = p.sa[v] != 0, b = p.sb[v] != 0, c = p.sc[v] != 0;
    if (kind == 0 && a && c && !b) {
      if (d.npl == CE_PCONV_MAXPL) return false;
      d.pl_ext[d.npl] = p.ext[v];
      d.pl_sf[d.npl] = p.sa[v];
      d.pl_so[d.npl++] = p.sc[v];
      d.P *= p.ext[v];
    } else if (kind == 1 && a && b && !c) {
      if (d.npl == CE_PCONV_MAXPL) return false;
      d.pl_ext[d.npl] = p.ext[v];
      d.pl_sf[d.npl] = p.sa[v];
      d.pl_so[d.npl++] = p.sb[v];
      d.P *= p.ext[v];
    } else if (a && (kind == 0 ? (b && !c) : (c && !b))) {
      ci_v.push_back(v);
    } else if (!a && b && c) {
      co_v.push_back(v);
    } else {
      return false;
    }
  }
  // channel tables (at most 2 vars each, <= 16 combined values)
  auto table = [&](const std::vector<int>& vs, int64_t* s1, const int64_t* src1, int64_t* s2, const int64_t* src2,
                   int32_t* n) {
    int64_t cnt = 1;
    for (int v : vs) cnt *= p.ext[v];
    if (vs.size() > 2 || cnt > CE_PCONV_MAXC) return false;
    *n = static_cast<int32_t>(cnt);
    for (int64_t e = 0; e < cnt; ++e) {
      int64_t r = e, o1 = 0, o2 = 0;
      for (int k = static_cast<int>(vs.size()) - 1; k >= 0; --k) {  // last var fastest
        const int v = vs[static_cast<std::size_t>(k)];
        const int64_t x = r % p.ext[v];
        r /= p.ext[v];
        o1 += x * src1[v];
        o2 += x * src2[v];
      }
      s1[e] = o1;
      s2[e] = o2;
    }
    return true;
  };
  if (kind == 0) {
    if (!table(ci_v, d.fci, p.sa, d.gci, p.sb, &d.Ci)) return false;
    if (!table(co_v, d.gco, p.sb, d.cco, p.sc, &d.Co)) return false;
  } else {
    if (!table(ci_v, d.fci, p.sa, d.gci, p.sc, &d.Ci)) return false;
    if (!table(co_v, d.gco, p.sb, d.cco, p.sc, &d.Co)) return false;
  }
  d.accumulate = p.accumulate;
  d.tiles_y = kind == 0 ? (d.OY + kTY0 - 1) / kTY0 : (d.OY + kTY1 - 1) / kTY1;
  d.tiles_x = kind == 0 ? (d.OX + kTX0 - 1) / kTX0 : (d.OX + kTX1 - 1) / kTX1;
  // worth it only for large planes (the TC path's expansion / col2im costs scale with them)
  // (CE_PCONV_MIN: the position threshold, read per plan so tests can lower it)
  const char* mn = std::getenv("CE_PCONV_MIN");
  const double min_pos = mn ? std::atof(mn) : static_cast<double>(1 << 20);
  const double positions = static_cast<double>(d.P) * d.OY * d.OX;
  if (positions < min_pos || d.OX < 16) return false;
  if (kind == 0) {
    if (co_instance(d.Co) < 0 || fwd_smem(d) > 200 * 1024) return false;
    int64_t cmax = 0;
    for (int c = 0; c < d.Co; ++c) cmax = std::max<int64_t>(cmax, d.cco[c] < 0 ? -d.cco[c] : d.cco[c]);
    const int64_t ay = d.sy < 0 ? -d.sy : d.sy, ax = d.sx < 0 ? -d.sx : d.sx;
    if (ay * kTY0 + ax * kTX0 + cmax >= (1ll << 31)) return false;  // 32-bit in-tile offsets
  } else {
    if (d.KH * d.Ci * d.Co > 256 || d.accumulate || wgrad_smem(d) > 200 * 1024) return false;
    d.items = d.P * d.tiles_y * d.tiles_x;
    d.ctas = static_cast<int32_t>(std::min<int64_t>(d.items, 148 * 4));
  }
  *out = d;
  return true;
}

cudaError_t ce_launch_pconv(const CePconvDesc& d, const float* F, const float* G, float* C, cudaStream_t s) {
  if (d.kind == 1) {
    switch (d.KW) {
      case 3: return launch_wgrad<3>(d, F, G, C, s);
      case 5: return launch_wgrad<5>(d, F, G, C, s);
      case 7: return launch_wgrad<7>(d, F, G, C, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (d.KW) {
    case 3: return launch_fwd_co<3>(d, F, G, C, s);
    case 5: return launch_fwd_co<5>(d, F, G, C, s);
    case 7: return launch_fwd_co<7>(d, F, G, C, s);
    default: return cudaErrorInvalidValue;
  }
}
