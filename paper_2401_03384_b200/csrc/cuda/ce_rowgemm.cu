// Row GEMMs with few contracted and few output columns (ce_rowgemm.h).
//
// One thread per row m: it reads the row's K values of A once into registers and produces all
// N outputs from a B held in shared memory (warp-uniform reads), where the generic stream
// kernel would re-read the row for every output and decode every term.  The rows are ordered
// with C's unit-stride var fastest, so each output column is written by a warp as consecutive
// elements.  Compulsory traffic |A| + |C|; the FLOPs (K x N per row, <= 1024) are noise.
#include "ce_rowgemm.h"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace {

template <int KT, int NT>
__global__ void __launch_bounds__(256) ce_rowgemm_kernel(const CeRowDesc d, const float* __restrict__ A,
                                                         const float* __restrict__ B, float* __restrict__ C) {
  __shared__ float bs[KT * NT];
  __shared__ int ka[KT], nc[NT];
  const int K = d.K, N = d.N;
  for (int e = threadIdx.x; e < KT * NT; e += blockDim.x) {
    const int k = e / NT, n = e % NT;
    bs[e] = (k < K && n < N) ? B[d.kb[k] + d.nb[n]] : 0.f;
  }
  if (threadIdx.x < KT) ka[threadIdx.x] = threadIdx.x < K ? static_cast<int>(d.ka[threadIdx.x]) : 0;
  if (threadIdx.x < NT) nc[threadIdx.x] = threadIdx.x < N ? static_cast<int>(d.nc[threadIdx.x]) : 0;
  __syncthreads();
  const uint32_t M = static_cast<uint32_t>(d.M);  // (< 2^31, see the planner)
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    uint32_t r = m;
    int64_t oa = 0, oc = 0;
    for (int i = 0; i < d.nm; ++i) {
      const uint32_t e = static_cast<uint32_t>(d.m_ext[i]);
      const uint32_t q = r / e;
      const uint32_t v = r - q * e;
      r = q;
      oa += static_cast<int64_t>(v) * d.m_sa[i];
      oc += static_cast<int64_t>(v) * d.m_sc[i];
    }
    float a[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) a[k] = k < K ? __ldg(A + oa + ka[k]) : 0.f;
    float* cp = C + oc;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      if (n >= N) break;
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < KT; ++k) acc = fmaf(a[k], bs[k * NT + n], acc);
      float* p = cp + nc[n];
      *p = d.accumulate ? *p + acc : acc;
    }
  }
}

int round_up(int x) { return x <= 8 ? 8 : x <= 16 ? 16 : 32; }

template <int KT, int NT>
cudaError_t launch(const CeRowDesc& d, const float* A, const float* B, float* C, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((d.M + 255) / 256, 148 * 16);
  ce_rowgemm_kernel<KT, NT><<<static_cast<unsigned>(blocks), 256, 0, s>>>(d, A, B, C);
  return cudaGetLastError();
}

}  // namespace

bool ce_rowgemm_plan(const CeProblem& p, CeRowDesc* out) {
  if (p.unary || p.ng_a != 0 || p.ng_b != 0) return false;
  CeRowDesc d{};
  std::vector<int> ms, ks, ns;
  double b_elems = 1;
  for (int v = 0; v < p.nv; ++v) {
    if (p.ext[v] == 1) continue;
    const bool a = p.sa[v] != 0, b = p.sb[v] != 0, c = p.sc[v] != 0;
    if (b) b_elems *= static_cast<double>(p.ext[v]);
    if (a && c && !b) ms.push_back(v);
    else if (a && b && !c) ks.push_back(v);
    else if (!a && b && c) ns.push_back(v);
    else return false;
  }
  if (ms.empty() || ms.size() > CE_ROW_MAXV || b_elems > 4096) return false;
  // M vars: C's unit-stride one first (coalesced stores), then by C stride
  std::stable_sort(ms.begin(), ms.end(), [&](int x, int y) { return p.sc[x] < p.sc[y]; });
  d.M = 1;
  for (int v : ms) {
    d.m_ext[d.nm] = p.ext[v];
    d.m_sa[d.nm] = p.sa[v];
    d.m_sc[d.nm++] = p.sc[v];
    d.M *= p.ext[v];
  }
  auto table = [&](const std::vector<int>& vs, int64_t* o1, const int64_t* s1, int64_t* o2, const int64_t* s2,
                   int32_t* n) {
    int64_t cnt = 1;
    for (int v : vs) cnt *= p.ext[v];
    if (cnt > CE_ROW_MAXKN) return false;
    *n = static_cast<int32_t>(cnt);
    for (int64_t e = 0; e < cnt; ++e) {
      int64_t r = e, a = 0, b = 0;
      for (int v : vs) {
        const int64_t x = r % p.ext[v];
        r /= p.ext[v];
        a += x * s1[v];
        b += x * s2[v];
      }
      if (a >= (1ll << 31) || b >= (1ll << 31)) return false;
      o1[e] = a;
      o2[e] = b;
    }
    return true;
  };
  if (!table(ks, d.ka, p.sa, d.kb, p.sb, &d.K)) return false;
  if (!table(ns, d.nb, p.sb, d.nc, p.sc, &d.N)) return false;
  // every row costs (padded K) x (padded N) FMAs and shared-memory reads: beyond 256 the
  // kernel is instruction-bound (RTR 64->128's K = N = 40 rows: 4.2 -> 272 ms)
  if (round_up(d.K) * round_up(d.N) > 256) return false;
  // (only where the tensor cores do badly: millions of rows, a few columns)
  const char* mn = std::getenv("CE_ROWGEMM_MIN");
  const double min_rows = mn ? std::atof(mn) : static_cast<double>(1 << 20);
  if (static_cast<double>(d.M) < min_rows || d.M >= (1ll << 31)) return false;
  d.accumulate = p.accumulate;
  *out = d;
  return true;
}

cudaError_t ce_launch_rowgemm(const CeRowDesc& d, const float* A, const float* B, float* C, cudaStream_t s) {
  const int kt = round_up(d.K), nt = round_up(d.N);
  if (kt == 8 && nt == 8) return launch<8, 8>(d, A, B, C, s);
  if (kt == 8 && nt == 16) return launch<8, 16>(d, A, B, C, s);
  if (kt == 8 && nt == 32) return launch<8, 32>(d, A, B, C, s);
  if (kt == 16 && nt == 8) return launch<16, 8>(d, A, B, C, s);
  if (kt == 16 && nt == 16) return launch<16, 16>(d, A, B, C, s);
  return launch<32, 8>(d, A, B, C, s);  // (kt * nt <= 256: 32 x 8 is the last shape)
}
