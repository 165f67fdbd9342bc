// Host planner for the tcgen05 implicit-GEMM path (see cuda/ce_tc.h).
//
// Given a lowered pairwise step, decide:
//   * units: vars merged where contiguous in every TMA operand;
//   * per operand: K-major (K unit innermost) or MN-major (tile unit innermost);
//   * the K block (32 K indices per stage) both operands enumerate identically;
//   * M tile (<=128 rows) and N tile (<=256 columns) boxes, grid and K-loop units;
//   * split-K for steps with few output tiles and long K (factor gradients).
// Anything that does not fit (wrap-around Circular taps, >5 TMA dims, strides
// not multiple of 16 B, no unit-stride axis) returns false and the executor uses
// the SIMT kernels (ce_simt.cu).
#include <algorithm>
#include <cstdio>
#include <functional>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../cuda/ce_tc.h"

namespace {

struct Axis {          // one TMA dim of an operand, before unit assignment
  bool gather = false;
  int v0 = -1, v1 = -1;  // plain: v0; gather: p = v0, q = v1
  int c0 = 1, c1 = 0;
  int64_t cst = 0;
  int64_t ext = 0;
  int64_t stride = 0;    // elements
};

std::vector<Axis> axes_of(const CeProblem& p, bool is_a) {
  std::vector<Axis> ax;
  const int64_t* s = is_a ? p.sa : p.sb;
  for (int v = 0; v < p.nv; ++v)
    if (s[v]) {
      Axis a;
      a.v0 = v;
      a.ext = p.ext[v];
      a.stride = s[v];
      ax.push_back(a);
    }
  const int ng = is_a ? p.ng_a : p.ng_b;
  const CeGather* g = is_a ? p.ga : p.gb;
  for (int i = 0; i < ng; ++i) {
    Axis a;
    a.gather = true;
    a.v0 = g[i].pv;
    a.v1 = g[i].qv;
    a.c0 = g[i].sp;
    a.c1 = g[i].sq;
    a.cst = g[i].c;
    a.ext = g[i].extent;
    a.stride = g[i].stride;
    ax.push_back(a);
  }
  // extent-1 plain axes carry nothing
  ax.erase(std::remove_if(ax.begin(), ax.end(), [](const Axis& a) { return !a.gather && a.ext == 1; }), ax.end());
  std::sort(ax.begin(), ax.end(), [](const Axis& x, const Axis& y) { return x.stride < y.stride; });
  return ax;
}

bool in_gather(const CeProblem& p, int v) {
  for (int i = 0; i < p.ng_a; ++i)
    if (p.ga[i].pv == v || p.ga[i].qv == v) return true;
  for (int i = 0; i < p.ng_b; ++i)
    if (p.gb[i].pv == v || p.gb[i].qv == v) return true;
  return false;
}

// Group of vars forming one unit (innermost first).
struct Group {
  std::vector<int> vars;
  int64_t ext = 1;
  int cls = 0;
};

// Merge var `outer` onto group g if it continues g's innermost-first stride chain
// in every TMA operand (A, B).  Out strides are not required to chain: the
// epilogue decomposes units back into vars.
bool chains(const CeProblem& p, const Group& g, int outer, bool in_c) {
  const int inner = g.vars.back();
  for (const int64_t* s : {p.sa, p.sb}) {
    const bool hi = s[inner] != 0, ho = s[outer] != 0;
    if (hi != ho) return false;
    if (hi && s[outer] != s[inner] * p.ext[inner]) return false;
  }
  // (in_c: the unit must also be one strided axis of C, so a TMA map can store its tiles)
  if (in_c && p.sc[inner] && p.sc[outer] != p.sc[inner] * p.ext[inner]) return false;
  return true;
}

int64_t pow2ceil(int64_t x) {
  int64_t r = 1;
  while (r < x) r <<= 1;
  return r;
}

}  // namespace

namespace {
bool tc_plan_impl(const CeProblem& p, TcPlan* plan, bool units_chain_in_c);
}

// The plan proper; short-K launches (stores dominate) whose units do not chain in C are
// re-planned with units that do, so the TMA-store epilogue can take them (e.g. a [b,t,h,w]
// output of a rank -> channel GEMM: one [h w] x t tile per sample instead of tiles across b).
bool ce_tc_plan(const CeProblem& p, TcPlan* plan) {
  if (!tc_plan_impl(p, plan, false)) return false;
  // opt-in (CE_TC_CTMA_RECHAIN=1): the re-chained tiles (2 per 14x14 sample, one ragged) cost
  // what the faster stores save -- cfg2 step 1.118-1.125 vs 1.103-1.141 ms (same-box A/B x3)
  static const bool rechain = [] {
    const char* e = std::getenv("CE_TC_CTMA_RECHAIN");
    return e && *e == '1';
  }();
  if (rechain && plan->params.c_tma == 0 && plan->params.k_iters <= 8 && plan->params.k_split == 1) {
    TcPlan alt;
    const bool ok2 = tc_plan_impl(p, &alt, true);
    if (ok2 && alt.params.c_tma != 0) *plan = alt;
  }
  return true;
}

namespace {
bool tc_plan_impl(const CeProblem& p, TcPlan* plan, bool units_chain_in_c) {
  *plan = TcPlan{};
  auto fail = [&](const char* why) {
    plan->valid = 0;
    plan->why = why;
    return false;
  };
  if (p.unary) return fail("unary");
  for (int i = 0; i < p.ng_a; ++i)
    if (p.ga[i].wrap) return fail("circular wrap");
  for (int i = 0; i < p.ng_b; ++i)
    if (p.gb[i].wrap) return fail("circular wrap");

  // ---------------------------------------------------------------- units
  // Seed groups from single vars, then greedily chain contiguous same-class plain vars.
  std::vector<Group> groups;
  std::vector<int> order(static_cast<std::size_t>(p.nv));
  for (int v = 0; v < p.nv; ++v) order[static_cast<std::size_t>(v)] = v;
  // chain candidates by the stride they have in A (else B)
  auto key = [&](int v) { return p.sa[v] ? p.sa[v] : p.sb[v]; };
  std::sort(order.begin(), order.end(), [&](int x, int y) { return key(x) < key(y); });
  std::vector<int> unit_of(static_cast<std::size_t>(p.nv), -1);
  for (int v : order) {
    if (p.ext[v] == 1 && !in_gather(p, v)) {
      // size-1 vars vanish: attach to nothing (value always 0)
      continue;
    }
    bool merged = false;
    if (!in_gather(p, v)) {
      for (std::size_t gi = 0; gi < groups.size() && !merged; ++gi) {
        Group& g = groups[gi];
        if (g.cls != p.cls[v] || in_gather(p, g.vars.back()) || g.vars.size() >= 4) continue;
        if (chains(p, g, v, units_chain_in_c)) {
          g.vars.push_back(v);
          g.ext *= p.ext[v];
          unit_of[static_cast<std::size_t>(v)] = static_cast<int>(gi);
          merged = true;
        }
      }
    }
    if (!merged) {
      Group g;
      g.vars = {v};
      g.ext = p.ext[v];
      g.cls = p.cls[v];
      unit_of[static_cast<std::size_t>(v)] = static_cast<int>(groups.size());
      groups.push_back(g);
    }
  }
  if (static_cast<int>(groups.size()) > TC_MAX_UNITS) return fail("too many units");

  // operand dims in units
  auto build = [&](bool is_a, std::vector<Axis>& out) -> bool {
    std::vector<Axis> ax = axes_of(p, is_a);
    for (Axis& a : ax) {
      if (a.gather) continue;
      const int u = unit_of[static_cast<std::size_t>(a.v0)];
      if (groups[static_cast<std::size_t>(u)].vars.front() != a.v0) { a.ext = -1; continue; }  // merged into inner
      a.ext = groups[static_cast<std::size_t>(u)].ext;
    }
    ax.erase(std::remove_if(ax.begin(), ax.end(), [](const Axis& a) { return a.ext < 0; }), ax.end());
    out = ax;
    return true;
  };
  std::vector<Axis> A, B;
  build(true, A);
  build(false, B);
  if (A.empty() || B.empty()) return fail("empty operand");
  if (A.size() > 5 || B.size() > 5) return fail("more than 5 TMA dims");
  if (A.front().stride != 1 || A.front().gather) return fail("A has no unit-stride plain axis");
  if (B.front().stride != 1 || B.front().gather) return fail("B has no unit-stride plain axis");
  for (const auto* ops : {&A, &B})
    for (std::size_t i = 1; i < ops->size(); ++i)
      if (((*ops)[i].stride * 4) % 16 != 0) return fail("stride not a multiple of 16 bytes");

  auto ucls = [&](int v) { return p.cls[v]; };
  auto uid = [&](int v) { return unit_of[static_cast<std::size_t>(v)]; };
  const int innerA = A.front().v0, innerB = B.front().v0;
  const int ia_cls = ucls(innerA), ib_cls = ucls(innerB);
  // MN-major operands (the tile unit innermost in memory) are TMA-loaded as [32 K rows][32 MN]
  // SWIZZLE_128B boxes -- exactly the UMMA MN-major SW128 canonical layout -- and read by the
  // MMA with the transpose bits of the instruction descriptor (native_mn, the default), or
  // (CE_TC_NATIVE_MN=0) transposed to K-major in shared memory by the transposer warps.
  int a_mn = -1, b_mn = -1;
  std::vector<std::pair<int, int>> kblock;  // (unit, box)
  auto has_plain = [&](const std::vector<Axis>& ops, int u) {
    for (const Axis& a : ops)
      if (!a.gather && uid(a.v0) == u) return true;
    return false;
  };
  if (ia_cls == CE_K) {
    a_mn = 0;
    kblock = {{uid(innerA), TC_BK}};
    if (ib_cls == CE_K && uid(innerB) == uid(innerA)) {
      b_mn = 0;
    } else if (ib_cls == CE_N && has_plain(B, uid(innerA))) {
      b_mn = 1;
    } else {
      return fail("K blocks of A and B disagree");
    }
  } else if (ia_cls == CE_M) {
    a_mn = 1;
    if (ib_cls == CE_K) {
      b_mn = 0;
      if (!has_plain(A, uid(innerB))) return fail("K block of B not addressable in A");
      kblock = {{uid(innerB), TC_BK}};
    } else if (ib_cls == CE_N) {
      b_mn = 1;
      // K rows from K units addressable in both operands (plain, or gathered with q-coef +1),
      // ordered by A's stride
      int64_t remaining = TC_BK;
      for (const Axis& a : A) {
        if (remaining == 1) break;
        int u = -1;
        if (!a.gather && ucls(a.v0) == CE_K) u = uid(a.v0);
        if (a.gather && ucls(a.v1) == CE_K && a.c1 == 1) u = uid(a.v1);
        if (u < 0) continue;
        bool in_b = false;
        for (const Axis& b : B) {
          if (!b.gather && uid(b.v0) == u) in_b = true;
          if (b.gather && uid(b.v1) == u && b.c1 == 1) in_b = true;
        }
        if (!in_b) continue;
        const int64_t e = groups[static_cast<std::size_t>(u)].ext;
        int64_t box = std::min(remaining, pow2ceil(e));
        kblock.push_back({u, static_cast<int>(box)});
        remaining /= box;
      }
      if (kblock.empty()) return fail("no shared K unit for MN-major operands");
      if (remaining > 1) kblock.back().second *= static_cast<int>(remaining);
    } else {
      return fail("B inner axis class");
    }
  } else {
    return fail("A inner axis class");
  }

  // ---------------------------------------------------------------- tiles
  std::vector<TcUnit> U(groups.size());
  for (std::size_t i = 0; i < groups.size(); ++i) {
    TcUnit& t = U[i];
    t = TcUnit{};
    t.ext = static_cast<int32_t>(groups[i].ext);
    t.box = 1;
    t.nv = static_cast<int32_t>(groups[i].vars.size());
    for (int k = 0; k < t.nv; ++k) {
      const int v = groups[i].vars[static_cast<std::size_t>(k)];
      t.vext[k] = static_cast<int32_t>(p.ext[v]);
      t.sc[k] = p.sc[v];
    }
    const int c = groups[i].cls;
    t.src = c == CE_K ? TC_SRC_K : TC_SRC_GRID;
    if (groups[i].ext >= (1ll << 31)) return fail("extent above 2^31");
  }
  for (auto& kb : kblock) U[static_cast<std::size_t>(kb.first)].box = kb.second;

  TcParams& P = plan->params;
  std::memset(&P, 0, sizeof(P));
  // M tile from A, N tile from B
  static const bool cinner = [] {  // CE_TC_CINNER=0: tile search ignores C's unit-stride axis
    const char* e = std::getenv("CE_TC_CINNER");
    return !(e && *e == '0');
  }();
  static const bool nalign = [] {  // CE_TC_NALIGN=0: balanced N boxes not kept 16-B aligned
    const char* e = std::getenv("CE_TC_NALIGN");
    return !(e && *e == '0');
  }();
  static const bool balance_n = [] {  // CE_TC_BALANCE_N=0: widest N boxes (previous tiling)
    const char* e = std::getenv("CE_TC_BALANCE_N");
    return !(e && *e == '0');
  }();
  auto tile = [&](const std::vector<Axis>& ops, bool mn_major, int cls, int cap, int32_t* list, int32_t* n,
                  int src) -> int {
    int rows = 1;
    if (mn_major) {
      const int u = uid(ops.front().v0);
      const int box = std::min<int>(cap, static_cast<int>((U[static_cast<std::size_t>(u)].ext + 31) / 32 * 32));
      U[static_cast<std::size_t>(u)].box = box;
      U[static_cast<std::size_t>(u)].src = src;
      list[(*n)++] = u;
      return box;
    }
    // candidate tile units in the operand's stride order (up to 3)
    std::vector<int> cand;
    for (const Axis& a : ops) {
      if (cand.size() >= 3) break;
      int u = -1;
      if (!a.gather && ucls(a.v0) == cls) u = uid(a.v0);
      if (a.gather && ucls(a.v0) == cls && a.c0 == 1) u = uid(a.v0);
      if (u < 0 || U[static_cast<std::size_t>(u)].src != TC_SRC_GRID) continue;
      if (std::find(cand.begin(), cand.end(), u) != cand.end()) continue;
      cand.push_back(u);
    }
    if (cand.empty()) return rows;
    // (re-planned for the TMA-store epilogue: one M unit, C's unit-stride one when it leads,
    // so each warp's 32 rows are 128 contiguous bytes of C per column)
    if (units_chain_in_c && cls == CE_M && cand.size() > 1) cand.erase(cand.begin() + 1, cand.end());
    // Boxes minimising the number of tiles (every tile costs a full M=128 / N MMA), then
    // maximising the rows used: e.g. a 14x14 image stack tiles as [14 w][1 h][9 b] (98%
    // of the rows useful) instead of [14 w][9 h] (77%).
    std::vector<int64_t> ext;
    for (int u : cand) ext.push_back(U[static_cast<std::size_t>(u)].ext);
    const bool minbox = cls == CE_N && balance_n;
    std::vector<int> best(cand.size(), 1);
    int64_t best_tiles = INT64_MAX, best_rows = minbox ? INT64_MAX : 0;
    std::vector<int> b(cand.size(), 1);
    std::function<void(std::size_t, int)> search = [&](std::size_t i, int room) {
      if (i == cand.size()) {
        int64_t tiles = 1, r = 1;
        bool split_cinner = false;
        for (std::size_t j = 0; j < cand.size(); ++j) {
          tiles *= (ext[j] + b[j] - 1) / b[j];
          r *= b[j];
          // an M unit that is C's unit-stride axis, cut into boxes of < 4: every tile row
          // then writes runs shorter than 16 B (RTR dZ rows: 2 of a 10-float run; tt1.0's
          // NCHW output 2 of 14 w).  Measured: cfg2 step -1.2%, tt1.0 711 -> 688 us, RTR
          // 64->128 61.6 -> 58.6 ms; a box of 4 (RTR @56) is better left alone (5.10 vs 5.27 ms)
          const TcUnit& uu = U[static_cast<std::size_t>(cand[j])];
          split_cinner |= cinner && cls == CE_M && uu.nv >= 1 && uu.sc[0] == 1 && b[j] < ext[j] && b[j] < 4;
        }
        if (split_cinner) tiles = tiles * 3 / 2;
        // M: the MMA is always 128 rows, so use as many as fit; N: the MMA width follows the
        // tile, so among equal tile counts the narrowest box pads least (273 -> 2 x 137)
        if (tiles < best_tiles || (tiles == best_tiles && (minbox ? r < best_rows : r > best_rows))) {
          best_tiles = tiles;
          best_rows = r;
          best = b;
        }
        return;
      }
      const int hi = static_cast<int>(std::min<int64_t>(ext[i], room));
      for (int x = hi; x >= 1; --x) {
        // only boxes that are the full extent or change the tile count are worth trying
        if (!minbox && x < hi && (ext[i] + x - 1) / x == (ext[i] + x) / (x + 1)) continue;
        // (balanced N boxes stay multiples of 4 so every N tile starts 16-B aligned in C and
        // the epilogue keeps its float4 column groups: 275 = 140 + 135, not 138 + 137)
        if (minbox && nalign && x < hi && ext[i] >= 8) {
          if (x % 4 || (x > 4 && (ext[i] + x - 1) / x == (ext[i] + x - 5) / (x - 4))) continue;
        } else if (minbox && x < hi && x > 1 && (ext[i] + x - 1) / x == (ext[i] + x - 2) / (x - 1)) {
          continue;
        }
        b[i] = x;
        search(i + 1, room / x);
      }
      b[i] = 1;
    };
    search(0, cap);
    for (std::size_t j = 0; j < cand.size(); ++j) {
      if (best[j] <= 1 && j > 0) continue;  // box 1: leave it a grid unit
      const int u = cand[j];
      U[static_cast<std::size_t>(u)].box = best[j];
      U[static_cast<std::size_t>(u)].src = src;
      list[(*n)++] = u;
      rows *= best[j];
    }
    return rows;
  };
  P.m_rows = tile(A, a_mn == 1, CE_M, TC_BM, P.mt, &P.nm, TC_SRC_MTILE);
  // N tile: up to 256 columns
  static const int ncap_env = [] {
    const char* e = std::getenv("CE_TC_NCAP");  // experiment knob: cap the N tile
    return e ? std::atoi(e) : 256;
  }();
  int ncap = ncap_env;
  if (balance_n && ncap == 256 && b_mn == 0) {
    // a launch with fewer work items than half the SMs: narrower N tiles double them
    const std::vector<TcUnit> U0 = U;
    int32_t nt0[TC_MAX_UNITS];
    int32_t nn0 = 0;
    const int cols = tile(B, false, CE_N, 256, nt0, &nn0, TC_SRC_NTILE);
    U = U0;
    double out_elems = 1, k_elems = 1;
    for (int v = 0; v < p.nv; ++v) (p.cls[v] != CE_K ? out_elems : k_elems) *= static_cast<double>(p.ext[v]);
    // (a long K loop is split across CTAs instead: split-K fills the machine)
    if (cols >= 128 && k_elems <= 64.0 * TC_BK && out_elems / (static_cast<double>(P.m_rows) * cols) < 74)
      ncap = 128;
  }
  {
    // factor-only GEMMs (e.g. TT's core x factor products, 273 x 256 x 3 outputs): a dozen or
    // two work items whose epilogues drain one 128 x 256 tile per CTA at per-CTA store speed.
    // Halve the N tile (down to 64 columns, either B orientation) while the launch has fewer
    // items than a quarter of the SMs: tt1.0's six factor GEMMs 18 -> 45-65 items, cfg2 step
    // 0.948 -> 0.939 ms (same-box A/B x3), cfg3 / cfg4 plans unchanged.  CE_TC_FEW_ITEMS=0 off, >1: the item threshold.
    static const int few = [] {
      const char* e = std::getenv("CE_TC_FEW_ITEMS");
      return e ? std::atoi(e) : 1;
    }();
    if (few > 0 && ncap_env == 256) {
      double out_elems = 1, k_elems = 1;
      for (int v = 0; v < p.nv; ++v) (p.cls[v] != CE_K ? out_elems : k_elems) *= static_cast<double>(p.ext[v]);
      if (k_elems <= 64.0 * TC_BK) {
        const std::vector<TcUnit> U0 = U;
        while (ncap > 64) {
          int32_t nt0[TC_MAX_UNITS];
          int32_t nn0 = 0;
          const int cols = tile(B, b_mn == 1, CE_N, ncap, nt0, &nn0, TC_SRC_NTILE);
          U = U0;
          if (out_elems / (static_cast<double>(P.m_rows) * cols) >= (few > 1 ? few : 37)) break;
          ncap /= 2;
        }
      }
    }
    // store-bound launches (a K loop of a few stages, e.g. the rank -> channel 1x1 GEMMs writing
    // a [b,t,h,w] activation): half-width N tiles run on the LEAN instances, two CTAs per SM,
    // so two epilogues drain per SM.  CE_TC_SHORTK_NCAP=0 off.
  }
  {
    // store-bound launches (a K loop of a few stages, e.g. the rank -> channel 1x1 GEMMs writing
    // a [b,t,h,w] activation): N tiles of at most 128 columns run on the LEAN instances, two
    // CTAs per SM, so two epilogues drain per SM.  CE_TC_SHORTK_NCAP=<K stages> (0 off).
    static const int shortk_kmax = [] {
      const char* e = std::getenv("CE_TC_SHORTK_NCAP");
      return e ? std::atoi(e) : 4;
    }();
    double k_elems = 1, n_elems = 1;
    for (int v = 0; v < p.nv; ++v) {
      if (p.cls[v] == CE_K) k_elems *= static_cast<double>(p.ext[v]);
      if (p.cls[v] == CE_N) n_elems *= static_cast<double>(p.ext[v]);
    }
    if (n_elems > 128 && k_elems <= static_cast<double>(shortk_kmax) * TC_BK) ncap = std::min(ncap, 128);
    // experiment (CE_TC_N3=<K stages>): 257..384 columns in three <=128-wide tiles when the K
    // loop is short enough for the LEAN instances (tt1.0's N = 273 convs: 392 tiles over 148
    // SMs = 2.65 rounds, or 588 over 296 LEAN slots = 1.99)
    static const int n3_kmax = [] {
      const char* e = std::getenv("CE_TC_N3");
      return e ? std::atoi(e) : 0;
    }();
    if (n3_kmax > 0 && n_elems > 256 && n_elems <= 384 && k_elems <= static_cast<double>(n3_kmax) * TC_BK)
      ncap = std::min(ncap, 128);
  }
  P.n_cols = tile(B, b_mn == 1, CE_N, ncap, P.nt, &P.nn, TC_SRC_NTILE);
  if (P.nm == 0) return fail("no M tile unit");
  if (P.nn == 0) {
    // N = 1 (e.g. an input gradient contracting every factor index: dX = sum dZ * F): one
    // B row per stage; the MMA's other 15 columns read stale shared memory and are never
    // stored.  An N var that merely failed to tile still fails.
    for (int v = 0; v < p.nv; ++v)
      if (p.cls[v] == CE_N && p.ext[v] > 1) return fail("no N tile unit");
    // memory-bound: worth it only when the 32-wide K boxes are mostly useful data
    if (kblock.empty() || U[static_cast<std::size_t>(kblock.front().first)].ext < 16)
      return fail("N = 1 with a short K unit");
  }
  P.n_mma = static_cast<int32_t>((P.n_cols + 15) / 16 * 16);
  plan->bn = P.n_mma <= 64 ? 64 : P.n_mma <= 128 ? 128 : 256;
  if (b_mn == 1 && P.n_cols % 32) return fail("MN-major B tile must be a multiple of 32");

  // Store-completing traversal: when a grid unit continues C's unit-stride run past the tile
  // (RTR's dZ: the N tile holds r3, C's 10-float inner run, and t1 -- stride 10 -- is a grid
  // unit), consecutive work items should cover that unit's values so the pieces of each
  // 32-B sector are written close together in time (one CTA, back to back, in contiguous
  // mode) instead of by tiles far apart, which left partial sectors for L2 to write back.  The
  // unit becomes the fastest M digit with a box of 1 (no change to the tile's rows).
  // CE_TC_GFIRST=0 off.
  {
    static const bool gfirst_on = [] {
      const char* e = std::getenv("CE_TC_GFIRST");
      return !(e && *e == '0');
    }();
    int64_t run = 0;  // C-contiguous elements covered by the tile unit holding C's unit-stride var
    for (int pass = 0; pass < 2 && gfirst_on && run == 0; ++pass)
      for (int i = 0; i < (pass ? P.nn : P.nm); ++i) {
        const TcUnit& u = U[static_cast<std::size_t>(pass ? P.nt[i] : P.mt[i])];
        if (u.nv < 1 || u.sc[0] != 1) continue;
        run = u.vext[0];
        for (int k = 1; k < u.nv && u.sc[k] == run; ++k) run *= u.vext[k];
        if (u.box < u.ext) run = 0;  // the tile cuts the run itself
      }
    if (run > 0 && run < 8 * 4 && P.nm < 3) {  // (runs of >= 32 floats already fill whole sectors)
      for (std::size_t i = 0; i < U.size(); ++i) {
        TcUnit& g = U[i];
        if (g.src != TC_SRC_GRID || g.nv < 1 || g.sc[0] != run || g.ext < 2) continue;
        for (int j = P.nm; j > 0; --j) P.mt[j] = P.mt[j - 1];
        P.mt[0] = static_cast<int32_t>(i);
        ++P.nm;
        g.src = TC_SRC_MTILE;
        g.box = 1;
        break;
      }
    }
  }

  // grid / K-loop units
  for (std::size_t i = 0; i < U.size(); ++i) {
    if (U[i].src == TC_SRC_GRID) P.gu[P.ng++] = static_cast<int32_t>(i);
    if (P.ng > 8) return fail("too many grid units");
  }
  for (auto& kb : kblock) P.ku[P.nk++] = kb.first;
  for (std::size_t i = 0; i < U.size(); ++i) {
    if (U[i].src != TC_SRC_K) continue;
    bool in_block = false;
    for (auto& kb : kblock) in_block |= kb.first == static_cast<int>(i);
    if (!in_block) {
      if (P.nk >= 6) return fail("too many K units");
      P.ku[P.nk++] = static_cast<int32_t>(i);
    }
  }

  // ---------------------------------------------------------------- TMA dims
  auto dims_for = [&](const std::vector<Axis>& ops, bool mn_major, TcOperand& o, uint64_t* gdim, uint64_t* gstride,
                      uint32_t* box, int* rank) -> bool {
    // order: inner, then box>1 dims in K-block order (MN-major) or tile order (K-major), then the rest
    std::vector<const Axis*> ord{&ops.front()};
    auto boxed_unit = [&](const Axis& a) -> int {
      if (!a.gather) return uid(a.v0);
      const int up = uid(a.v0), uq = uid(a.v1);
      if (U[static_cast<std::size_t>(up)].box > 1) return up;
      if (U[static_cast<std::size_t>(uq)].box > 1) return uq;
      return up;
    };
    std::vector<int> pref;
    if (mn_major)
      for (auto& kb : kblock) pref.push_back(kb.first);
    else
      for (int i = 0; i < (&o == &P.oa ? P.nm : P.nn); ++i) pref.push_back((&o == &P.oa ? P.mt : P.nt)[i]);
    for (int u : pref)
      for (const Axis& a : ops)
        if (&a != &ops.front() && boxed_unit(a) == u && U[static_cast<std::size_t>(u)].box > 1) ord.push_back(&a);
    for (const Axis& a : ops)
      if (std::find(ord.begin(), ord.end(), &a) == ord.end()) ord.push_back(&a);
    *rank = static_cast<int>(ord.size());
    int64_t rows = 1;
    for (int d = 0; d < 5; ++d) {
      TcDim& td = o.dim[d];
      td = TcDim{-1, -1, 0, 0, 0};
      if (d >= *rank) {
        gdim[d] = 1;
        box[d] = 1;
        gstride[d] = gstride[d - 1] * gdim[d - 1];
        continue;
      }
      const Axis& a = *ord[static_cast<std::size_t>(d)];
      gdim[d] = static_cast<uint64_t>(a.ext);
      gstride[d] = static_cast<uint64_t>(a.stride) * 4;
      if (!a.gather) {
        td.u0 = uid(a.v0);
        td.c0 = 1;
        box[d] = static_cast<uint32_t>(U[static_cast<std::size_t>(td.u0)].box);
      } else {
        td.u0 = uid(a.v0);
        td.c0 = a.c0;
        td.u1 = uid(a.v1);
        td.c1 = a.c1;
        td.cst = static_cast<int32_t>(a.cst);
        const int b0 = U[static_cast<std::size_t>(td.u0)].box, b1 = U[static_cast<std::size_t>(td.u1)].box;
        if (b0 > 1 && b1 > 1) return false;
        if ((b0 > 1 && a.c0 != 1) || (b1 > 1 && a.c1 != 1)) return false;
        box[d] = static_cast<uint32_t>(std::max(b0, b1));
      }
      if (d == 0) {
        box[0] = 32;  // 128-byte rows (SWIZZLE_128B)
      } else {
        rows *= box[d];
      }
      if (box[d] > 256) return false;
    }
    if (gstride[0] != 4) return false;
    o.mn_major = mn_major ? 1 : 0;
    if (mn_major) {
      if (rows != TC_BK) return false;
      o.nsub = U[static_cast<std::size_t>(uid(ops.front().v0))].box / 32;
      o.stage_bytes = o.nsub * 32 * 128;
    } else {
      o.nsub = 1;
      o.stage_bytes = static_cast<int32_t>(rows * 128);
    }
    return true;
  };
  if (!dims_for(A, a_mn == 1, P.oa, plan->gdim_a, plan->gstride_a, plan->box_a, &plan->rank_a))
    return fail("A TMA dims");
  if (!dims_for(B, b_mn == 1, P.ob, plan->gdim_b, plan->gstride_b, plan->box_b, &plan->rank_b))
    return fail("B TMA dims");
  // An MN-major A is fetched as one unswizzled [32 K][<=128 MN] box (512-B rows: one TMA
  // per stage instead of nsub 4-KB boxes, 4x longer DRAM runs); the transposer warps then
  // write the swizzled K-major blocks the MMA reads.
  static const bool wide_on = [] {
    const char* e = std::getenv("CE_TC_WIDE");
    return !(e && *e == '0');
  }();
  static const bool native_on = [] {
    const char* e = std::getenv("CE_TC_NATIVE_MN");
    return !(e && *e == '0');
  }();
  P.native_mn = native_on ? 1 : 0;
  {
    // MN-major tf32 smem layout (probe knobs while the layout is being pinned on hardware):
    // CE_TC_MN_LAYOUT (UMMA layout type, default 1 = SWIZZLE_128B_BASE32B), CE_TC_MN_TMASWZ
    // (CUtensorMapSwizzle of the MN-major boxes, default 4 = 128B_ATOM_32B), CE_TC_MN_SBO /
    // CE_TC_MN_LBO (bytes), CE_TC_MN_KSTEP (bytes per K=8 step)
    auto env = [](const char* k, int d) {
      const char* e = std::getenv(k);
      return e ? std::atoi(e) : d;
    };
    static const int layout = env("CE_TC_MN_LAYOUT", 1), tmaswz = env("CE_TC_MN_TMASWZ", 4),
                     sbo = env("CE_TC_MN_SBO", 512), lbo = env("CE_TC_MN_LBO", 4096), kstep = env("CE_TC_MN_KSTEP", 1024);
    P.mn_lbo16 = static_cast<uint32_t>(lbo >> 4);
    P.mn_desc_hi = static_cast<uint32_t>(sbo >> 4) | (1u << 14) | (static_cast<uint32_t>(layout) << 29);
    P.mn_kstep16 = static_cast<uint32_t>(kstep >> 4);
    if (P.native_mn) {
      if (a_mn == 1) plan->swz_a = tmaswz;
      if (b_mn == 1) plan->swz_b = tmaswz;
    }
  }
  P.oa.wide = 0;
  P.ob.wide = 0;
  if (wide_on && !P.native_mn && a_mn == 1 && P.oa.nsub >= 2 && P.oa.nsub <= 4) {
    P.oa.wide = 1;
    P.oa.wbox = P.oa.nsub * 32;
    plan->box_a[0] = static_cast<uint32_t>(P.oa.wbox);
    plan->swz_a = 0;
  }
  if (a_mn == 0 && P.oa.stage_bytes != P.m_rows * 128) return fail("A rows");
  if (b_mn == 0 && P.ob.stage_bytes != P.n_cols * 128) return fail("B rows");
  if (P.ob.stage_bytes > plan->bn * 128) return fail("B tile too large");

  // ---------------------------------------------------------------- grid
  P.nunits = static_cast<int32_t>(U.size());
  for (std::size_t i = 0; i < U.size(); ++i) P.u[i] = U[i];
  int64_t tm = 1, tn = 1, gz = 1, ki = 1;
  for (int i = 0; i < P.nm; ++i) tm *= (U[P.mt[i]].ext + U[P.mt[i]].box - 1) / U[P.mt[i]].box;
  for (int i = 0; i < P.nn; ++i) tn *= (U[P.nt[i]].ext + U[P.nt[i]].box - 1) / U[P.nt[i]].box;
  for (int i = 0; i < P.ng; ++i) gz *= U[P.gu[i]].ext;
  for (int i = 0; i < P.nk; ++i) ki *= (U[P.ku[i]].ext + U[P.ku[i]].box - 1) / U[P.ku[i]].box;
  if (tm > 0x7fffffff || tn > 65535 || ki > 0x7fffffff) return fail("grid too large");
  P.tiles_m = static_cast<int32_t>(tm);
  P.tiles_n = static_cast<int32_t>(tn);
  P.grid_z = static_cast<int32_t>(gz);
  P.k_iters = static_cast<int32_t>(ki);
  P.k_split = 1;
  // K odometer steps: digit i of the K loop moves unit ku[i] by its box
  for (int i = 0; i < 6; ++i) {
    P.kcount[i] = 1;
    for (int d = 0; d < 5; ++d) P.kstep_a[i][d] = P.kstep_b[i][d] = 0;
  }
  for (int i = 0; i < P.nk; ++i) {
    const TcUnit& u = U[static_cast<std::size_t>(P.ku[i])];
    P.kcount[i] = (u.ext + u.box - 1) / u.box;
    for (int d = 0; d < 5; ++d) {
      for (const auto* o : {&P.oa, &P.ob}) {
        const TcDim& t = o->dim[d];
        int step = 0;
        if (t.u0 == P.ku[i]) step += t.c0 * u.box;
        if (t.u1 == P.ku[i]) step += t.c1 * u.box;
        (o == &P.oa ? P.kstep_a : P.kstep_b)[i][d] = step;
      }
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int d = 0; d < 5; ++d) {
      int da = P.kstep_a[i][d], db = P.kstep_b[i][d];
      for (int v = 0; v < i; ++v) {
        da -= (P.kcount[v] - 1) * P.kstep_a[v][d];
        db -= (P.kcount[v] - 1) * P.kstep_b[v][d];
      }
      P.kdelta_a[i][d] = da;
      P.kdelta_b[i][d] = db;
    }
  P.ktail_kk = 4;
  if (P.nk >= 1 && kblock.size() == 1 && kblock[0].second == TC_BK && P.ku[0] == kblock[0].first) {
    const int64_t ext = U[static_cast<std::size_t>(P.ku[0])].ext;
    const int64_t rem = ext - static_cast<int64_t>(TC_BK) * (P.kcount[0] - 1);
    P.ktail_kk = static_cast<int32_t>((rem + 7) / 8);
  }
  // output span (for zeroing before split-K accumulation)
  int64_t span = 0;
  for (int v = 0; v < p.nv; ++v)
    if (p.cls[v] != CE_K) span += (p.ext[v] - 1) * p.sc[v];
  plan->out_span = span + 1;
  // Epilogue store orientation: lanes along rows (plain) or along columns (transposed
  // through smem).  Pick the one whose warp-wide store touches fewer 32-byte sectors,
  // judged on the first 32 rows / columns of a tile (same offset math as the kernel).
  {
    auto offsets = [&](const int32_t* list, int n, int count) {
      std::vector<int64_t> offs;
      for (int local = 0; local < count; ++local) {
        int64_t off = 0;
        int64_t rest = local;
        bool ok = true;
        for (int i = 0; i < n; ++i) {
          const TcUnit& u = U[static_cast<std::size_t>(list[i])];
          int64_t v = rest % u.box;
          rest /= u.box;
          if (v >= u.ext) ok = false;
          for (int k = 0; k < u.nv; ++k) {
            off += (v % u.vext[k]) * u.sc[k];
            v /= u.vext[k];
          }
        }
        if (ok && rest == 0) offs.push_back(off);
      }
      return offs;
    };
    auto sectors = [](const std::vector<int64_t>& offs) {
      std::vector<int64_t> sec;
      for (int64_t o : offs) sec.push_back(o / 8);  // 8 floats per 32-B sector
      std::sort(sec.begin(), sec.end());
      return static_cast<int>(std::unique(sec.begin(), sec.end()) - sec.begin());
    };
    const int rows_sec = sectors(offsets(P.mt, P.nm, std::min(32, P.m_rows)));
    const int cols_sec = sectors(offsets(P.nt, P.nn, std::min(32, P.n_cols)));
    P.transpose_store = cols_sec < rows_sec ? 1 : 0;
  }
  // instruction descriptor: D f32, A/B tf32, A/B major (bits 15/16: 1 = MN-major, read
  // natively), N >> 3, M >> 4
  const uint32_t major_bits = P.native_mn ? (static_cast<uint32_t>(a_mn == 1) << 15) |
                                                (static_cast<uint32_t>(b_mn == 1) << 16)
                                          : 0u;
  P.idesc = (1u << 4) | (2u << 7) | (2u << 10) | major_bits | (static_cast<uint32_t>(P.n_mma >> 3) << 17) |
            (static_cast<uint32_t>(TC_BM >> 4) << 24);
  // 2-CTA cluster with B multicast: K-major B whose N tile is one unit (TMA dim 1)
  static const bool mcast_enabled = [] {
    const char* e = std::getenv("CE_TC_MCAST");
    return !(e && *e == '0');
  }();
  P.mcast = 0;
  // CTA pairs (cta_group::2 + B multicast) for every launch (CE_TC_PAIR=1): once the kernel ran
  // below its register cap, single-CTA launches measured faster on the cfg2 step (1.195 vs
  // 1.216 ms, same-box A/B x3) and equal or better on most layers profiled
  // Default (CE_TC_PAIR=3): pairs only for wide (> 128 column) tile-parallel launches with 25..47
  // K stages -- above the LEAN instances, below the tail split (which the pair path lacks) --
  // where halving each CTA's B bytes per stage relieves the L2-fed N=256 mainloop: tt1.0's
  // node3 / dN1 convs 53.7 -> 45.6 us, cfg2 step 0.938 -> 0.929 ms (same-box A/B x4), cfg3
  // unchanged.  CE_TC_PAIR=2: every wide launch of >= 16 stages (tk1.0's convs lose their tail
  // split and TMA store: 59.9 -> 72.2 us); 1: every eligible launch; 0: none.
  static const int pair_mode = [] {
    const char* e = std::getenv("CE_TC_PAIR");
    return e ? std::atoi(e) : 3;
  }();
  const bool pair_enabled = pair_mode == 1 ||
                            (pair_mode == 2 && P.n_cols > 128 && ki >= 16 && tm * tn * gz >= 148) ||
                            (pair_mode == 3 && P.n_cols > 128 && ki > 24 && ki < 48 && tm * tn * gz >= 148);
  // (CE_TC_PAIR=0 now means no cluster at all: the older single-CTA multicast variant
  // (mcast 1) hung on a CP 64->64 @56 layer's split-K launch and is no longer planned)
  if (mcast_enabled && pair_enabled && b_mn == 0 && P.nn == 1 && P.tiles_m >= 2 && P.n_cols >= 64 &&
      P.ob.dim[1].u0 == P.nt[0]) {
    const int half = ((P.n_cols + 1) / 2 + 7) / 8 * 8;
    if (2 * half <= plan->bn) {
      P.mc_half = half;
      P.mc_ndim = 1;
      plan->box_b[1] = static_cast<uint32_t>(half);
      if (pair_enabled) {
        // CTA pair, M=256 cta_group::2 MMAs: each CTA stages its own half of the B columns
        P.mcast = 2;
        P.ob.stage_bytes = half * 128;
        P.n_mma = 2 * half;
        P.idesc = (1u << 4) | (2u << 7) | (2u << 10) | major_bits | (static_cast<uint32_t>(P.n_mma >> 3) << 17) |
                  (static_cast<uint32_t>((2 * TC_BM) >> 4) << 24);
      } else {
        P.mcast = 1;  // B halves multicast to both CTAs, M=128 MMAs per CTA
        P.ob.stage_bytes = 2 * half * 128;
      }
    }
  }
  // split-K when the output grid cannot fill the 148 SMs and K is long: as many K slices
  // as fit in ONE wave of CTAs (a second, partial wave would cost a whole extra slice time)
  {
    const int64_t csize = P.mcast ? 2 : 1;
    const int64_t ctas = (tm + csize - 1) / csize * csize * tn * gz;
    // CE_SPLITK_SMS: SMs a split-K launch may fill (default all 148; the leaf gradients it
    // serves run beside the backward chain)
    static const int64_t sk_sms = [] {
      const char* e = std::getenv("CE_SPLITK_SMS");
      return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t{148};
    }();
    int split = 1;
    if (ctas < 148 && ki >= 16)
      split = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sk_sms / ctas, ki / 8)));
    if (gz * split > 65535) return fail("grid z too large");
    P.k_split = split;
  }
  // fast-division constants for the per-tile index decoding (ce_tc.h TcDiv)
  for (int i = 0; i < P.nunits; ++i) {
    TcUnit& u = P.u[i];
    u.dbox = tc_div(static_cast<uint32_t>(u.box));
    u.dtiles = tc_div(static_cast<uint32_t>((u.ext + u.box - 1) / u.box));
    u.dext = tc_div(static_cast<uint32_t>(u.ext));
    for (int k = 0; k < 4; ++k) u.dvext[k] = tc_div(k < u.nv ? static_cast<uint32_t>(u.vext[k]) : 1u);
  }
  {
    const int64_t csize = P.mcast ? 2 : 1;
    const int64_t pm = (P.tiles_m + csize - 1) / csize;
    P.dpm = tc_div(static_cast<uint32_t>(pm));
    P.dtn = tc_div(static_cast<uint32_t>(P.tiles_n));
    P.dsplit = tc_div(static_cast<uint32_t>(pm * P.tiles_n * P.grid_z));
    P.k_per = (P.k_iters + P.k_split - 1) / P.k_split;
    if (pm * P.tiles_n * P.grid_z * P.k_split >= (1ll << 31)) return fail("too many work items");
  }
  // TMA-store epilogue (TcParams::c_tma): C must be a <= 5-D tensor map over the tile units --
  // the M units (a warp's 32 rows = full boxes of the inner M units times an even share of
  // the outermost one), one N unit (32-column chunks), the grid units, each unit's vars
  // chaining in C, and the M or N inner var C's unit-stride axis.  No box may reach into a
  // neighbouring tile (N tiles multiples of 32 or a single N tile; past the tensor's extent
  // TMA clips).  CE_TC_CTMA=0 off.
  {
    static const bool ctma_on = [] {
      const char* e = std::getenv("CE_TC_CTMA");
      return !(e && *e == '0');
    }();
    P.c_tma = 0;
    P.c_wrap = 0;
    auto chain = [&](const TcUnit& u) {
      for (int k = 1; k < u.nv; ++k)
        if (u.sc[k] != u.sc[k - 1] * u.vext[k - 1]) return false;
      return true;
    };
    bool ok = ctma_on && P.nm >= 1 && P.nn == 1 && P.mcast == 0 && P.nm + 1 + P.ng <= 5;
    int64_t inner_rows = 1;  // rows of a warp's slab covered by the M units below the last
    for (int i = 0; ok && i + 1 < P.nm; ++i) inner_rows *= P.u[P.mt[i]].box;
    const int64_t slab_last = ok ? 32 / std::max<int64_t>(inner_rows, 1) : 0;  // last M unit's share per warp
    if (ok) {
      const TcUnit& ul = P.u[P.mt[P.nm - 1]];
      ok = inner_rows <= 32 && 32 % inner_rows == 0 && slab_last > 0 && ul.box % slab_last == 0 &&
           inner_rows * ul.box == P.m_rows;
    }
    // a single M unit whose vars chain in C only in two groups (inner vars, then outer vars:
    // [w h][b] of an NCHW output, the tile's 128 flat rows crossing b) is stored as two C dims,
    // a warp slab crossing into the next outer index with a second, shifted box (c_wrap)
    int wrap_split = 0;  // number of inner vars
    int64_t wrap_ext = 0;
    // opt-in (CE_TC_CWRAP=1): on cfg2's [w h][b] NCHW outputs the bulk stores of 32-row x
    // 32-column boxes (32 separate 128-B rows each) were slower than the warps' coalesced
    // per-column stores: step 1.008 -> 1.09 ms (same-box A/B x3)
    static const bool wrap_on = [] {
      const char* e = std::getenv("CE_TC_CWRAP");
      return e && *e == '1';
    }();
    if (ok && wrap_on && P.nm == 1 && !chain(P.u[P.mt[0]]) && P.nm + 2 + P.ng <= 5) {
      const TcUnit& u = P.u[P.mt[0]];
      int j = 1;
      int64_t e = u.vext[0];
      while (j < u.nv && u.sc[j] == u.sc[j - 1] * u.vext[j - 1]) e *= u.vext[j++];
      bool outer_chain = true;
      for (int k = j + 1; k < u.nv; ++k) outer_chain = outer_chain && u.sc[k] == u.sc[k - 1] * u.vext[k - 1];
      if (j < u.nv && outer_chain && e >= 32 && u.sc[j] % 4 == 0 && e * (u.ext / e) == u.ext) {
        wrap_split = j;
        wrap_ext = e;
      }
    }
    for (int i = 0; ok && i < P.nm; ++i) ok = wrap_split > 0 || chain(P.u[P.mt[i]]);
    const TcUnit& un = P.u[P.nt[0]];
    ok = ok && chain(un) && (P.n_cols % 32 == 0 || P.tiles_n == 1);
    for (int i = 0; i < P.ng && ok; ++i) ok = chain(P.u[P.gu[i]]);
    if (ok && wrap_split > 0 && P.nm + 2 + P.ng > 5) ok = false;
    if (ok) {
      const TcUnit& um0 = P.u[P.mt[0]];
      const bool rows_inner = um0.sc[0] == 1;
      const bool cols_inner = un.sc[0] == 1;
      ok = rows_inner != cols_inner;
      static const bool rows_mode = [] {  // CE_TC_CTMA=2: only the columns-innermost mode
        const char* e = std::getenv("CE_TC_CTMA");
        return !(e && *e == '2');
      }();
      ok = ok && (rows_mode || cols_inner);
      // every stride but the inner one 16-B aligned
      for (int i = 0; ok && i < P.nm; ++i) ok = (rows_inner && i == 0) || P.u[P.mt[i]].sc[0] % 4 == 0;
      ok = ok && (cols_inner || un.sc[0] % 4 == 0);
      for (int i = 0; ok && i < P.ng; ++i) ok = P.u[P.gu[i]].sc[0] % 4 == 0;
      if (ok) {
        P.c_tma = rows_inner ? 1 : 2;
        int d = 0;
        auto put = [&](int unit, int q, uint32_t box) {
          const TcUnit& u = P.u[unit];
          P.cdim_u[d] = unit;
          P.cdim_q[d] = q;
          plan->gdim_c[d] = static_cast<uint64_t>(u.ext);
          plan->gstride_c[d] = static_cast<uint64_t>(u.sc[0]) * 4;
          plan->box_c[d] = box;
          ++d;
        };
        auto put_rows = [&] {  // M units fastest first; the last one carries the warp offset
          if (wrap_split > 0) {  // inner vars (flat extent wrap_ext) and outer vars as two dims
            const TcUnit& u = P.u[P.mt[0]];
            P.cdim_u[d] = P.mt[0];
            P.cdim_q[d] = 3;
            plan->gdim_c[d] = static_cast<uint64_t>(wrap_ext);
            plan->gstride_c[d] = static_cast<uint64_t>(u.sc[0]) * 4;
            plan->box_c[d] = 32;
            ++d;
            P.cdim_u[d] = P.mt[0];
            P.cdim_q[d] = 4;
            plan->gdim_c[d] = static_cast<uint64_t>(u.ext / wrap_ext);
            plan->gstride_c[d] = static_cast<uint64_t>(u.sc[wrap_split]) * 4;
            plan->box_c[d] = 1;
            ++d;
            return;
          }
          for (int i = 0; i + 1 < P.nm; ++i) put(P.mt[i], 0, static_cast<uint32_t>(P.u[P.mt[i]].box));
          put(P.mt[P.nm - 1], 1, static_cast<uint32_t>(slab_last));
        };
        if (rows_inner) {
          put_rows();
          put(P.nt[0], 2, 32);
        } else {
          put(P.nt[0], 2, 32);
          put_rows();
        }
        for (int i = 0; i < P.ng; ++i) put(P.gu[i], 0, 1);
        for (; d < 5; ++d) {
          P.cdim_u[d] = -1;
          P.cdim_q[d] = 0;
          plan->gdim_c[d] = 1;
          plan->gstride_c[d] = plan->gstride_c[d - 1] * plan->gdim_c[d - 1];
          plan->box_c[d] = 1;
        }
        P.c_slab = static_cast<int32_t>(slab_last);
        P.c_wrap = static_cast<int32_t>(wrap_split > 0 ? wrap_ext : 0);
        plan->swz_c = rows_inner ? 0 : 3;  // CU_TENSOR_MAP_SWIZZLE_128B for row-major 128-B rows
      }
    }
  }
  plan->valid = 1;
  plan->why = "ok";
  return true;
}
}  // namespace
