// tcgen05 kind::tf32 implicit-GEMM kernel for sm_100a (families a + b1).
//
// Persistent and warp-specialised: grid = min(#work groups, #SMs); a work group is one
// CTA, or a CTA pair (cluster of 2 along M) that shares the B tile through TMA
// multicast.  320 threads:
//   warp 0 lane 0 : TMA producer   (cp.async.bulk.tensor.5d -> STAGES-deep smem ring;
//                                    B halves multicast to both CTAs of a pair)
//   warp 1 lane 0 : MMA issuer     (tcgen05.mma.cta_group::1.kind::tf32 into one of two
//                                    TMEM accumulators, tcgen05.commit -> mbarriers)
//   warps 2..5    : epilogue       (tcgen05.ld 32x32b -> registers -> [smem transpose] ->
//                                    global scatter / atomic add for split-K)
//   warps 6..9    : transposers    (MN-major TMA boxes -> K-major layout, in place)
// Two TMEM accumulators let the epilogue of tile t overlap the mainloop of tile t+1.
// Operand tiles are 128-byte K-major rows with the 128B swizzle shared by TMA and the
// UMMA descriptors.  Convolution taps are K-loop iterations whose TMA coordinates are
// shifted (ce_tc.h); Same/Full padding is TMA's OOB zero fill.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ce_launch.h"
#include "ce_tc.h"

namespace {

constexpr int kEpiWarps = 4;
constexpr int kXposeWarps = 4;
constexpr int kThreads = 64 + 32 * kEpiWarps + 32 * kXposeWarps;
constexpr int kStagePitch = 36;  // floats per staged row: 16-B aligned, conflict-free float4 phases

// Debug flags (timing experiments, phase stamps) are compiled in only with -DCE_TC_DEBUG=1
// (`make TC_DEBUG=1`): their branches cost registers, and the kernel already runs at the
// register cap (spills raise the cfg2 step time measurably).
#ifndef CE_TC_DEBUG
#define CE_TC_DEBUG 0
#endif
#define TC_DBG(p) (CE_TC_DEBUG ? (p).dbg : 0)

// Debug-only phase timestamps (P.dbg & 32): [cta][slot] = %globaltimer (ns).
__device__ unsigned long long g_tc_ts[160 * 16];
// Debug-only per-iteration timestamps of CTA 0 (P.dbg & 512): [role][iteration], role 0
// producer (after its empty wait), 1 MMA issuer (after its full wait).
__device__ unsigned long long g_tc_it[3 * 256];

__device__ __forceinline__ void stamp_it(const TcParams& P, int role, uint32_t gi) {
  if ((TC_DBG(P) & 512) && blockIdx.x == 0 && gi < 256) {  // role 2: epilogue, slot tile*4 + phase
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles (cheap; same SM for all roles)
    g_tc_it[role * 256 + gi] = static_cast<unsigned long long>(t);
  }
}
__device__ __forceinline__ void stamp(const TcParams& P, int slot) {
  if (TC_DBG(P) & 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 160) g_tc_ts[blockIdx.x * 16 + slot] = t;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Shared::cluster address of the same smem location in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// Arrive on an mbarrier of another CTA of the cluster (release at cluster scope).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Wait that also acquires what other CTAs of the cluster released into this barrier.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, const int c[5]) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
      : "memory");
}

// CTA-pair load: the box lands in this CTA's smem, completion is signalled on an
// mbarrier that may live in the peer CTA (`bar_cluster` is a shared::cluster address).
__device__ __forceinline__ void tma_load_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, const int c[5]) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar_cluster)
      : "memory");
}

// Same box delivered to the same smem offset (and mbarrier) of every CTA in `mask`.
__device__ __forceinline__ void tma_load_mc(void* dst, const CUtensorMap* map, uint64_t* bar, const int c[5],
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
      "{%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// SM100 UMMA shared-memory descriptor, K-major SWIZZLE_128B: start>>4 [0,14),
// LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4 [32,46) = 1024 B between
// 8-row groups, version 1 [46,48), layout SWIZZLE_128B (2) [61,64).
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// SM100 UMMA shared-memory descriptor for an MN-major tf32 operand.  32-bit MN-major
// operands use the SWIZZLE_128B_BASE32B layout (type 1; CUTLASS Layout_MN_SW128_32B_Atom:
// 32-B chunks of a 128-B row XOR-swizzled, 4-row atoms), which TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: 32 MN floats per 128-B row, one row per K index,
// LBO = 4096 B to the next 32-MN box, SBO = 512 B to the next 4-row K atom.  A K=8 step
// advances the start address by 8 rows (1024 B).  The upper word (SBO, version, layout)
// and LBO come from the host (TcParams::mn_desc_hi / mn_lbo16).
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t addr, uint32_t lbo16, uint32_t hi) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>(lbo16 & 0x3FFF) << 16) |
         (static_cast<uint64_t>(hi) << 32);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// M=256 MMA over a CTA pair (issued by the even CTA): A rows 0-127 from this CTA's smem,
// 128-255 from the peer's; B columns split in halves the same way; D rows per CTA's TMEM.
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Arrive (when the MMAs retire) on the same mbarrier offset of every CTA in `mask`.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Split TMEM load: issue without waiting, and a wait that ties the destination registers
// (so no use can be scheduled before the data has landed).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// Vector reduction into global memory (split-K epilogue): 4 consecutive floats, one request.
__device__ __forceinline__ void red_add_v4(float* p, float4 v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Bulk tensor store / reduce-add of a staged shared-memory box (TMA-store epilogue).
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const void* src, const int c[5], bool add) {
  if (add)
    asm volatile(
        "cp.reduce.async.bulk.tensor.5d.global.shared::cta.add.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
        "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
        : "memory");
  else
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Named barrier of one epilogue warp group (ids 1 and 2).
__device__ __forceinline__ void epi_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(32 * kEpiWarps) : "memory"); }

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// In-place transpose of one 4 KB SWIZZLE_128B block from the TMA MN-major layout
// ([32 K rows][32 MN], row k at k*128, 16-B chunk c/4 stored at chunk (c/4)^(k%8))
// to the UMMA K-major layout ([32 MN rows][32 K], chunk kk/4 of row r at (kk/4)^(r%8)).
// Lane l reads MN column l (conflict-free: one 128-B row per step), then writes its
// K-major row with 16-B stores (conflict-free per 8-lane phase).
__device__ __forceinline__ void xpose_block(uint8_t* blk, int lane) {
  float v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k)
    v[k] = *reinterpret_cast<const float*>(blk + k * 128 + (((lane >> 2) ^ (k & 7)) << 4) + ((lane & 3) << 2));
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(blk + lane * 128 + ((j ^ (lane & 7)) << 4)) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

struct Tile {
  int32_t val[TC_MAX_UNITS];  // tile origins / grid digits per unit (K units 0)
  int split;
  int ntile;                  // linear N-tile index (the column tables depend only on it)
};

// Work item w of a group of `csize` CTAs (rank within the group): m tiles are dealt
// in groups of csize (m fastest), then n, z and the K split.  The highest M digit may
// run past its extent for the last odd group: those rows are simply invalid (TMA OOB
// zero fill, no store).
__device__ __forceinline__ void decode_work(const TcParams& P, uint32_t w, uint32_t rank, uint32_t csize, Tile& T) {
  for (int i = 0; i < TC_MAX_UNITS; ++i) T.val[i] = 0;
  uint32_t t = tc_quo(w, P.dpm);
  uint32_t m = (w - t * P.dpm.d) * csize + rank;
  const uint32_t tn = tc_quo(t, P.dtn);
  T.ntile = static_cast<int>(t - tn * P.dtn.d);
  for (int i = 0; i < P.nm; ++i) {
    const TcUnit& u = P.u[P.mt[i]];
    if (i + 1 == P.nm) {
      T.val[P.mt[i]] = static_cast<int32_t>(m) * u.box;
    } else {
      const uint32_t q = tc_quo(m, u.dtiles);
      T.val[P.mt[i]] = static_cast<int32_t>(m - q * u.dtiles.d) * u.box;
      m = q;
    }
  }
  for (int i = 0; i < P.nn; ++i) {
    const TcUnit& u = P.u[P.nt[i]];
    const uint32_t q = tc_quo(t, u.dtiles);
    T.val[P.nt[i]] = static_cast<int32_t>(t - q * u.dtiles.d) * u.box;
    t = q;
  }
  for (int i = 0; i < P.ng; ++i) {
    const TcUnit& u = P.u[P.gu[i]];
    const uint32_t q = tc_quo(t, u.dext);
    T.val[P.gu[i]] = static_cast<int32_t>(t - q * u.dext.d);
    t = q;
  }
  T.split = static_cast<int>(t);
}

// Work sequence of one group: whole items group, group + ngroups, ... below sk_full, then
// (tail split) one K chunk of a tail item: the sk_r items of a partial last round are each cut
// into tl_s K chunks, one per group (group u -> item sk_full + u / tl_s, chunk u % tl_s).
// Chunk 0 stores its partial tile; chunks > 0 wait for it (tl_flags) and add theirs.
struct WorkIter {
  uint32_t w;         // next whole item
  uint32_t wend;      // contiguous mode: end of this group's items
  uint32_t tail;      // this group's tail unit, or ~0u (none / consumed)
  bool seq;           // the item returned last was the previous item + 1 (contiguous mode)
};

__device__ __forceinline__ void work_begin(const TcParams& P, uint32_t group, uint32_t ngroups, WorkIter& it) {
  (void)ngroups;
  it.w = group;
  it.wend = 0;
  it.seq = false;
  if (P.contig) {
    it.w = group * P.ipg + min(group, P.irem);
    it.wend = it.w + P.ipg + (group < P.irem ? 1u : 0u);
  }
  it.tail = (P.sk_r > 0 && group < P.sk_r * P.tl_s) ? group : ~0u;
}

// T <- the tile of the next item in decode_work's order (M units fastest, then N units,
// then grid units; single CTA groups, no K split).
__device__ __forceinline__ void advance_tile(const TcParams& P, Tile& T) {
  for (int i = 0; i < P.nm; ++i) {
    const TcUnit& u = P.u[P.mt[i]];
    const int32_t v = T.val[P.mt[i]] + u.box;
    if (v < u.ext) {
      T.val[P.mt[i]] = v;
      return;
    }
    T.val[P.mt[i]] = 0;
  }
  for (int i = 0; i < P.nn; ++i) {
    const TcUnit& u = P.u[P.nt[i]];
    const int32_t v = T.val[P.nt[i]] + u.box;
    if (v < u.ext) {
      T.val[P.nt[i]] = v;
      T.ntile += 1;
      return;
    }
    T.val[P.nt[i]] = 0;
  }
  T.ntile = 0;
  for (int i = 0; i < P.ng; ++i) {
    const TcUnit& u = P.u[P.gu[i]];
    const int32_t v = T.val[P.gu[i]] + 1;
    if (v < u.ext) {
      T.val[P.gu[i]] = v;
      return;
    }
    T.val[P.gu[i]] = 0;
  }
}

// Next segment: item (full-decomposition index), K range [k0, k1), atomic epilogue flag, and
// the tail chunk (-1 for whole items).
__device__ __forceinline__ bool work_next(const TcParams& P, uint32_t ngroups, WorkIter& it, uint32_t& item, int& k0,
                                          int& k1, bool& atomic, int& chunk) {
  chunk = -1;
  if (P.tl_first && it.tail != ~0u) {  // the tail chunk first (see TcParams::tl_first)
    const uint32_t t = it.tail / static_cast<uint32_t>(P.tl_s);
    chunk = static_cast<int>(it.tail - t * static_cast<uint32_t>(P.tl_s));
    it.tail = ~0u;
    item = P.sk_full + t;
    it.seq = false;
    k0 = chunk * P.k_iters / P.tl_s;
    k1 = (chunk + 1) * P.k_iters / P.tl_s;
    atomic = chunk > 0 || P.tl_zeroed;
    return true;
  }
  if (P.contig) {
    if (it.w >= it.wend) return false;
    it.seq = item == it.w - 1 && it.w != 0;
    item = it.w++;
    k0 = 0;
    k1 = P.k_iters;
    atomic = P.acc_out != 0;
    return true;
  }
  const uint32_t whole = P.sk_r > 0 ? P.sk_full : P.n_items;
  if (it.w < whole) {
    item = it.w;
    it.w += ngroups;
    const int split = static_cast<int>(tc_quo(item, P.dsplit));
    k0 = split * P.k_per;
    k1 = min(P.k_iters, k0 + P.k_per);
    atomic = P.k_split > 1 || P.acc_out != 0;
    return true;
  }
  if (it.tail == ~0u) return false;
  const uint32_t t = it.tail / static_cast<uint32_t>(P.tl_s);
  chunk = static_cast<int>(it.tail - t * static_cast<uint32_t>(P.tl_s));
  it.tail = ~0u;
  item = P.sk_full + t;
  k0 = chunk * P.k_iters / P.tl_s;
  k1 = (chunk + 1) * P.k_iters / P.tl_s;
  atomic = chunk > 0 || P.tl_zeroed;
  return true;
}

__device__ __forceinline__ void coords(const TcOperand& o, const int32_t* val, int c[5]) {
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const TcDim& t = o.dim[d];
    int x = t.cst;
    if (t.u0 >= 0) x += t.c0 * val[t.u0];
    if (t.u1 >= 0) x += t.c1 * val[t.u1];
    c[d] = x;
  }
}

// Offset in C of tile-local index `local` along the unit list (first fastest); -1 if outside.
__device__ __forceinline__ int64_t tile_offset(const TcParams& P, const int32_t* list, int n, const int32_t* val,
                                               int local) {
  int64_t off = 0;
  uint32_t rest = static_cast<uint32_t>(local);
  for (int i = 0; i < n; ++i) {
    const TcUnit& u = P.u[list[i]];
    const uint32_t q = tc_quo(rest, u.dbox);
    const uint32_t d = rest - q * u.dbox.d;
    rest = q;
    uint32_t v = static_cast<uint32_t>(val[list[i]]) + d;
    if (v >= static_cast<uint32_t>(u.ext)) return -1;
    for (int k = 0; k < u.nv; ++k) {
      const uint32_t vq = tc_quo(v, u.dvext[k]);
      off += static_cast<int64_t>(v - vq * u.dvext[k].d) * u.sc[k];
      v = vq;
    }
  }
  return rest == 0 ? off : -1;
}

// PAIR: CTA pair (cluster of 2) running M=256 tcgen05.mma.cta_group::2 issued by the even
// CTA; each CTA stages its own 128 A rows and half of the B columns, so per-SM smem traffic
// per MMA drops by a quarter and the ring gets deeper.
// LEAN: no transposer warps (native MN-major or K-major operands only), 192 threads and a
// shared-memory footprint under half an SM, so two CTAs are resident per SM -- two of this
// launch, or one of it and the PDL-launched next kernel, whose set-up (barriers, TMEM
// allocation, first tile decode) then overlaps this kernel's last epilogue.  Short-K steps.
template <int BN, int STAGES, bool PAIR, bool LEAN>
__global__ void __launch_bounds__(LEAN ? 64 + 32 * kEpiWarps : kThreads, LEAN ? 2 : 1)
    ce_tc_kernel(const __grid_constant__ TcParams Pg, float* __restrict__ C) {
  constexpr int NT = LEAN ? 64 + 32 * kEpiWarps : kThreads;
  constexpr int A_BYTES = TC_BM * 128;
  constexpr int B_BYTES = PAIR ? BN * 64 : BN * 128;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on smem_raw (not an integer round trip) so the
  // compiler keeps the shared address space and emits LDS/STS rather than generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  constexpr int EPI_GROUPS = (BN == 64 && !LEAN) ? 2 : 1;  // small tiles: a second epilogue warp group
  float* stage_out = reinterpret_cast<float*>(sB + STAGES * B_BYTES);  // [EPI_GROUPS*kEpiWarps][32][kStagePitch]
  int64_t* col_off = reinterpret_cast<int64_t*>(stage_out + EPI_GROUPS * kEpiWarps * 32 * kStagePitch);  // [2][BN]
  int64_t* grp_off = col_off + 2 * BN;                                  // [2][BN/4]: 16-B column groups
  int64_t* row_tab = grp_off + 2 * (BN / 4);                            // [2][128]: row offsets in C
  Tile* tiles = reinterpret_cast<Tile*>(row_tab + 2 * TC_BM);           // [0] producer, [1+g] epilogue group g
  uint64_t* full = reinterpret_cast<uint64_t*>(tiles + 4);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* ready = tempty + 2;       // [STAGES] stage transposed to K-major (MN-major operands only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready + STAGES);
  // Kernel parameters are read through dependent, dynamically indexed loads (unit lists ->
  // units -> extents); from the constant bank each of those is a cold miss on the start-up
  // path of every role.  One coalesced copy into shared memory up front instead.
  TcParams* sP = reinterpret_cast<TcParams*>(smem_raw + ((smem_u32(tmem_slot + 4) - smem_u32(smem_raw) + 63u) & ~63u));
  {
    const uint4* src = reinterpret_cast<const uint4*>(&Pg);
    uint4* dst = reinterpret_cast<uint4*>(sP);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(TcParams) / 16); i += NT) dst[i] = src[i];
  }
  const TcParams& P = *sP;
  if (TC_DBG(Pg) & 128) return;  // timing experiment: launch cost only
  // MN-major operands are either read by the MMA directly (native: transpose bits in the
  // instruction descriptor, MN-major smem descriptors) or transposed in smem by warps 6..9
  const bool xpose = !LEAN && !Pg.native_mn && (Pg.oa.mn_major || Pg.ob.mn_major);
  // (the single-CTA B multicast, mcast 1, is no longer planned -- see ce_tc_plan.cpp;
  // compiled out so the non-pair instances carry no multicast code)
  constexpr bool mc = false;
  const uint32_t csize = (mc || PAIR) ? 2u : 1u;
  uint32_t rank = 0;
  if (csize == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const bool leader = rank == 0;
  const uint32_t group = blockIdx.x / csize, ngroups = gridDim.x / csize;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) stamp(Pg, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mc ? csize : 1u);  // released by the MMA of every CTA that reads the stage
      mbar_init(&ready[s], (PAIR ? 2 : 1) * 32 * kXposeWarps);  // PAIR: both CTAs' transposers
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (PAIR ? 2 : 1) * 32 * kEpiWarps);  // PAIR: both CTAs' epilogues
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&Pg.ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&Pg.tb) : "memory");
    if (Pg.c_tma) asm volatile("prefetch.tensormap [%0];" ::"l"(&Pg.tc) : "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (csize == 2)
    cluster_sync();  // partner's barriers initialised before any multicast lands
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) stamp(P, 1);
  // Let the next kernel of the stream be scheduled (PDL).  The wait for the previous kernel
  // (griddepcontrol.wait) is deferred to each role's first global-memory access: the set-up
  // above and the first tile's decoding / address tables overlap the predecessor's tail.
  ce_pdl_trigger();

  if (TC_DBG(P) & 64) {
    // timing experiment: set-up and tear-down only
  } else if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------- TMA producer
      // Single issuing thread: everything in the per-stage loop is register arithmetic
      // (the loop period is this thread's instruction latency when the ring is not full).
      const uint32_t bytes = static_cast<uint32_t>(P.oa.stage_bytes + P.ob.stage_bytes);
      const uint32_t full_lead = PAIR ? mapa(&full[0], 0) : 0u;
      const int dbg = TC_DBG(Pg);
      const int nsub_a = P.oa.nsub, nsub_b = P.ob.nsub;
      const int mc_ndim = P.mc_ndim, mc_half = P.mc_half;
      // digit-0 deltas live in registers; carries (rare) and per-tile set-up read shared memory
      int kd0_a[5], kd0_b[5];
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        kd0_a[d] = P.kdelta_a[0][d];
        kd0_b[d] = P.kdelta_b[0][d];
      }
      const int kc0 = P.kcount[0];
      uint32_t gi = 0;  // global stage counter across tiles
      Tile& T = tiles[0];
      if (dbg & 32) stamp(P, 9);  // producer entered (after griddepcontrol.wait)
      WorkIter wi;
      work_begin(P, group, ngroups, wi);
      uint32_t item;
      int k0, k1, chunk;
      bool seg_atomic;
      item = 0xffffffffu;
      while (work_next(P, ngroups, wi, item, k0, k1, seg_atomic, chunk)) {
        if (wi.seq)
          advance_tile(P, T);
        else
          decode_work(P, item, rank, csize, T);
        int ca[5], cb[5], dig[6];
        coords(P.oa, T.val, ca);
        coords(P.ob, T.val, cb);
        if (csize == 2) cb[mc_ndim] += static_cast<int>(rank) * mc_half;  // this CTA's half of the B rows
#pragma unroll
        for (int u = 0; u < 6; ++u) dig[u] = 0;
        if (k0 != 0) {  // split-K slice: start the odometer mid-way
          int x = k0;
#pragma unroll
          for (int u = 0; u < 6; ++u) {
            dig[u] = x % P.kcount[u];
            x /= P.kcount[u];
#pragma unroll
            for (int d = 0; d < 5; ++d) {
              ca[d] += dig[u] * P.kstep_a[u][d];
              cb[d] += dig[u] * P.kstep_b[u][d];
            }
          }
        }
        if (gi == 0) {
          if (dbg & 32) stamp(P, 8);  // producer ready to issue its first load
          ce_pdl_wait();              // operands written by the previous kernel are visible
        }
        for (int it = k0; it < k1; ++it, ++gi) {
          const int s = static_cast<int>(gi % STAGES);
          mbar_wait(&empty[s], ((gi / STAGES) & 1) ^ 1);
          if (dbg & 512) stamp_it(P, 0, gi);
          if (dbg & 2) {
            if (!PAIR || xpose || leader) mbar_arrive(&full[s]);
          } else if (PAIR && !xpose) {
            // both halves complete on the even CTA's barrier, which expects the pair's bytes
            if (leader) mbar_expect_tx(&full[s], 2 * bytes);
            tma_load_pair(sA + s * A_BYTES, &Pg.ta, full_lead + 8u * s, ca);
            for (int j = 1; j < nsub_a; ++j) {  // native MN-major A: [32 K][32 MN] boxes at 4 KB steps
              const int cj[5] = {ca[0] + 32 * j, ca[1], ca[2], ca[3], ca[4]};
              tma_load_pair(sA + s * A_BYTES + j * 4096, &Pg.ta, full_lead + 8u * s, cj);
            }
            tma_load_pair(sB + s * B_BYTES, &Pg.tb, full_lead + 8u * s, cb);
          } else {
            // timing experiments: 2048 skips the A loads, 4096 the B loads
            const uint32_t exp_bytes =
                bytes - ((dbg & 2048) ? P.oa.stage_bytes : 0) - ((dbg & 4096) ? P.ob.stage_bytes : 0);
            mbar_expect_tx(&full[s], exp_bytes);
            // K-major: one box; MN-major: nsub boxes of [32 K rows][32 MN] at 4 KB steps
            if (!(dbg & 2048)) {
              tma_load(sA + s * A_BYTES, &Pg.ta, &full[s], ca);
              for (int j = 1; j < nsub_a && !P.oa.wide; ++j) {
                const int cj[5] = {ca[0] + 32 * j, ca[1], ca[2], ca[3], ca[4]};
                tma_load(sA + s * A_BYTES + j * 4096, &Pg.ta, &full[s], cj);
              }
            }
            if (dbg & 4096) {
            } else if (mc) {
              tma_load_mc(sB + s * B_BYTES + rank * mc_half * 128, &Pg.tb, &full[s], cb, 0x3);
            } else {
              tma_load(sB + s * B_BYTES, &Pg.tb, &full[s], cb);
              for (int j = 1; j < nsub_b; ++j) {
                const int cj[5] = {cb[0] + 32 * j, cb[1], cb[2], cb[3], cb[4]};
                tma_load(sB + s * B_BYTES + j * 4096, &Pg.tb, &full[s], cj);
              }
            }
          }
          // advance the K odometer: digit 0 almost always, carries rarely
          if (++dig[0] < kc0) {
#pragma unroll
            for (int d = 0; d < 5; ++d) {
              ca[d] += kd0_a[d];
              cb[d] += kd0_b[d];
            }
          } else {
            dig[0] = 0;
            bool carry = true;
#pragma unroll
            for (int u = 1; u < 6; ++u) {
              if (carry) {
                if (++dig[u] < P.kcount[u]) {
                  carry = false;
#pragma unroll
                  for (int d = 0; d < 5; ++d) {
                    ca[d] += P.kdelta_a[u][d];
                    cb[d] += P.kdelta_b[u][d];
                  }
                } else {
                  dig[u] = 0;
                }
              }
            }
          }
        }
      }
      stamp(P, 2);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------------------------------------------------- MMA issuer
      const int dbg = TC_DBG(Pg);
      const uint32_t idesc = P.idesc;
      const int kc0 = P.kcount[0], ktail = P.ktail_kk;
      // descriptors of stage 0; stage s and K step kk add (s * bytes + kk * 32) >> 4 to the
      // 14-bit start-address field (smem < 256 KB, so the add never carries out of it)
      const bool a_nat = P.native_mn && P.oa.mn_major, b_nat = P.native_mn && P.ob.mn_major;
      const uint64_t adesc0 = a_nat ? mnmajor_desc(smem_u32(sA), P.mn_lbo16, P.mn_desc_hi) : kmajor_desc(smem_u32(sA));
      const uint64_t bdesc0 = b_nat ? mnmajor_desc(smem_u32(sB), P.mn_lbo16, P.mn_desc_hi) : kmajor_desc(smem_u32(sB));
      // per K=8 step: +32 B inside a K-major 128-B row, +1024 B (one 8-row atom) MN-major
      const uint64_t astep = a_nat ? P.mn_kstep16 : 2, bstep = b_nat ? P.mn_kstep16 : 2;
      uint32_t gi = 0, local = 0;
      WorkIter wi;
      work_begin(P, group, ngroups, wi);
      uint32_t item = 0xffffffffu;
      int k0, k1, chunk;
      bool seg_atomic;
      for (; work_next(P, ngroups, wi, item, k0, k1, seg_atomic, chunk); ++local) {
        const int acc = static_cast<int>(local & 1);
        int d0 = k0 % kc0;  // K digit 0 of the first iteration (for the K tail)
        if (PAIR)
          mbar_wait_cluster(&tempty[acc], ((local >> 1) & 1) ^ 1);  // both epilogues drained it
        else
          mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * BN);
        for (int it = k0; it < k1; ++it, ++gi) {
          const int s = static_cast<int>(gi % STAGES);
          if (PAIR && xpose)
            mbar_wait_cluster(&ready[s], (gi / STAGES) & 1);
          else
            mbar_wait(xpose ? &ready[s] : &full[s], (gi / STAGES) & 1);
          if (dbg & 32) {
            if (gi == 0) stamp(P, 7);
            stamp_it(P, 1, gi);
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = adesc0 + static_cast<uint64_t>((s * A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + static_cast<uint64_t>((s * B_BYTES) >> 4);
          const int nkk = (d0 == kc0 - 1) ? ktail : TC_BK / 8;
          if (++d0 == kc0) d0 = 0;
          if (!(dbg & 1)) {
#pragma unroll
            for (int kk = 0; kk < TC_BK / 8; ++kk) {  // K=8 per tf32 MMA
              if (kk < nkk) {
                if (PAIR)
                  mma_tf32_pair(d_tmem, ad + astep * kk, bd + bstep * kk, idesc, (it > k0 || kk > 0) ? 1u : 0u);
                else
                  mma_tf32(d_tmem, ad + astep * kk, bd + bstep * kk, idesc, (it > k0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          if (dbg & 16)
            mbar_arrive(&empty[s]);  // timing experiment (with bit 0, no multicast): plain arrive
          else if (PAIR)
            mma_commit_pair(&empty[s]);  // the slot of this stage in both CTAs
          else if (mc)
            mma_commit_mc(&empty[s], 0x3);  // both CTAs wrote this stage's B halves
          else
            mma_commit(&empty[s]);  // frees the smem slot once these MMAs retire
        }
        if (PAIR)
          mma_commit_pair(&tfull[acc]);  // both CTAs' accumulators of this tile complete
        else
          mma_commit(&tfull[acc]);  // accumulator of this tile complete
      }
      stamp(P, 3);
    }
  } else if (warp >= 2 + kEpiWarps && (xpose || EPI_GROUPS == 1)) {
    // ------------------------------------------------------------ transposer warps
    // MN-major operand boxes -> K-major layout in place, then hand the stage to the MMA.
    if (xpose) {
      const int xw = warp - (2 + kEpiWarps);
      uint32_t gi = 0;
      WorkIter wi;
      work_begin(P, group, ngroups, wi);
      uint32_t item = 0xffffffffu;
      int k0, k1, chunk;
      bool seg_atomic;
      while (work_next(P, ngroups, wi, item, k0, k1, seg_atomic, chunk)) {
        for (int it = k0; it < k1; ++it, ++gi) {
          const int s = static_cast<int>(gi % STAGES);
          mbar_wait(&full[s], (gi / STAGES) & 1);
          if (P.oa.mn_major && P.oa.wide) {
            // [32 K][wbox MN] unswizzled: every warp reads its 32-MN slab first (the
            // K-major blocks overwrite the whole stage), then writes block xw
            const int wbox = P.oa.wbox;
            const float* st = reinterpret_cast<const float*>(sA + s * A_BYTES);
            float v[32];
            if (32 * xw < wbox) {
#pragma unroll
              for (int k = 0; k < 32; ++k) v[k] = st[k * wbox + 32 * xw + lane];
            }
            asm volatile("bar.sync 3, %0;" ::"n"(32 * kXposeWarps) : "memory");
            if (32 * xw < wbox) {
              uint8_t* blk = sA + s * A_BYTES + xw * 4096;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(blk + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                    make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
          } else if (P.oa.mn_major && !(TC_DBG(P) & 8192)) {
            for (int j = xw; j < P.oa.nsub; j += kXposeWarps) xpose_block(sA + s * A_BYTES + j * 4096, lane);
          }
          if (P.ob.mn_major && !(TC_DBG(P) & 8192))
            for (int j = xw; j < P.ob.nsub; j += kXposeWarps) xpose_block(sB + s * B_BYTES + j * 4096, lane);
          // generic-proxy smem writes must be visible to the tensor core (async proxy)
          if (!(TC_DBG(P) & 16384)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (PAIR && !leader)
            mbar_arrive_cluster(mapa(&ready[s], 0));  // the even CTA issues the pair's MMAs
          else
            mbar_arrive(&ready[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    // Per tile: one thread decodes the work item, the warps fill the row / column offset
    // tables (overlapping the MMAs), then each warp drains its TMEM lane quarter 32 columns
    // at a time.  Columns that are contiguous and 16-B aligned in C (the padded channel-
    // last intermediates) go out as 128-bit stores; anything else element by element.
    // BN=64 without MN-major operands: the transposer warps form a second group; group g
    // drains accumulator g (alternate tiles), so two tiles' epilogues are in flight
    const int ngrp = (EPI_GROUPS == 2 && !xpose) ? 2 : 1;
    const int grp = warp >= 2 + kEpiWarps ? 1 : 0;
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;     // accumulator row owned by this thread
    const int ew = warp - 2;           // 0..7
    const int et = threadIdx.x - 64 - grp * 32 * kEpiWarps;  // 0..127 within the group
    float* stage = stage_out + ew * 32 * kStagePitch;

    const int dbg = TC_DBG(Pg);
    const int n_cols = P.n_cols, m_rows = P.m_rows;
    const bool tstore = P.transpose_store != 0;
    const bool c_al = (reinterpret_cast<uintptr_t>(C) & 15u) == 0;
    uint32_t local = 0;
    Tile& T = tiles[1 + grp];
    int cols_for[2] = {-1, -1};  // N tile whose column tables each accumulator buffer holds
    WorkIter wi;
    work_begin(P, group, ngroups, wi);
    uint32_t item = 0xffffffffu;
    int k0, k1, chunk;
    bool atomic;
    for (; work_next(P, ngroups, wi, item, k0, k1, atomic, chunk); ++local) {
      const int acc = static_cast<int>(local & 1);
      // the CTA's last item: once its accumulator is full every MMA (and every smem read of
      // the operand ring) is done and no load follows, so its TMA-store chunks may each take
      // their own staging buffer in the ring instead of waiting for the previous chunk's
      // store to release the warp's single buffer
      bool last_item = false;
      if (!PAIR && P.c_tma) {
        WorkIter nx = wi;
        uint32_t it2;
        int a2, b2, c2;
        bool at2;
        last_item = !work_next(P, ngroups, nx, it2, a2, b2, at2, c2);
      }
      if (et == 0) {  // (also for the other group's tiles: the incremental advance needs every item)
        if (wi.seq)
          advance_tile(P, T);
        else
          decode_work(P, item, rank, csize, T);
      }
      if (ngrp == 2 && acc != grp) continue;  // the other group's tile
      const bool est = (dbg & 512) && et == 0 && grp == 0 && local < 128;
      if (est) stamp_it(P, 2, static_cast<uint32_t>(local / ngrp) * 4 + 0);
      epi_bar(1 + grp);  // decoded tile visible (and the previous tile's tables are no longer read)
      // address tables for this tile (overlaps the MMAs)
      int64_t* cols = col_off + acc * BN;
      int64_t* gcol = grp_off + acc * (BN / 4);
      int64_t* rtab = row_tab + acc * TC_BM;
      int64_t base = 0;
      for (int i = 0; i < P.ng; ++i) {
        const TcUnit& u = P.u[P.gu[i]];
        uint32_t v = static_cast<uint32_t>(T.val[P.gu[i]]);
        for (int k = 0; k < u.nv; ++k) {
          const uint32_t vq = tc_quo(v, u.dvext[k]);
          base += static_cast<int64_t>(v - vq * u.dvext[k].d) * u.sc[k];
          v = vq;
        }
      }
      // column tables depend only on the N tile: most launches have a single N tile, so they
      // are built once per accumulator buffer
      if (T.ntile != cols_for[acc]) {
        for (int c = et; c < BN; c += 32 * kEpiWarps) cols[c] = c < n_cols ? tile_offset(P, P.nt, P.nn, T.val, c) : -1;
        epi_bar(1 + grp);
        for (int g = et; g < BN / 4; g += 32 * kEpiWarps) {
          const int64_t c0 = cols[4 * g];
          const bool ok = c_al && c0 >= 0 && (c0 & 3) == 0 && cols[4 * g + 1] == c0 + 1 && cols[4 * g + 2] == c0 + 2 &&
                          cols[4 * g + 3] == c0 + 3;
          gcol[g] = ok ? c0 : -1;
        }
        cols_for[acc] = T.ntile;
      }
      const int64_t ro = row < m_rows ? tile_offset(P, P.mt, P.nm, T.val, row) : -1;
      const int64_t roff = ro < 0 ? -1 : base + ro;  // row offset in C, -1 outside the tile
      rtab[row] = roff;
      // TMA-store coordinates of this tile, taken while T is stable (thread 0 of the group
      // rewrites T for the next item as soon as its own chunks are out)
      int cbase[5];
#pragma unroll
      for (int d = 0; d < 5; ++d) cbase[d] = P.c_tma && P.cdim_u[d] >= 0 ? T.val[P.cdim_u[d]] : 0;
      epi_bar(1 + grp);  // tables visible to all epilogue warps
      if ((dbg & 32) && et == 0 && local == 0) stamp(P, 10);
      if (est) stamp_it(P, 2, static_cast<uint32_t>(local / ngrp) * 4 + 1);
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      if (est) stamp_it(P, 2, static_cast<uint32_t>(local / ngrp) * 4 + 2);
      if ((dbg & 32) && et == 0 && local == 0) stamp(P, 4);
      if (dbg & 8) {  // timing experiment: skip the epilogue body
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        if (PAIR && !leader)
          mbar_arrive_cluster(mapa(&tempty[acc], 0));
        else
          mbar_arrive(&tempty[acc]);
        continue;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (local == 0) ce_pdl_wait();  // (long complete: the producer waited before its loads)
      if (chunk > 0 && !P.tl_zeroed) {  // tail chunk: chunk 0 of this item must have stored its partial tile
        if (et == 0) {
          const uint32_t* f = P.tl_flags + (item - P.sk_full);
          uint32_t v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          } while (v == 0);
        }
        epi_bar(1 + grp);
      }
      const bool empty_k = k1 <= k0;
      const uint32_t t_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
      // TMEM loads double-buffered against the stores: chunk c+1 is read while chunk c drains
      const int nch = min(BN / 32, (n_cols + 31) / 32);
      auto process = [&](uint32_t (&r)[32], int ch) {
          if (empty_k)
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0;
          if (dbg & 4) {
            // timing experiment: TMEM loads only, no stores
            if (r[0] == 0x7fffffffu) C[0] = 0.f;
          } else if (tstore) {
            // stage this warp's 32x32 block row-major; then each lane writes 4 consecutive columns
            // of one row (8 lanes cover a row: 128 B per row, 4 rows per instruction)
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(stage + lane * kStagePitch + 4 * j) =
                  make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                              __uint_as_float(r[4 * j + 3]));
            __syncwarp();
            const int g = lane & 7, sub = lane >> 3;
            const int64_t gc = gcol[ch * 8 + g];
#pragma unroll 4
            for (int k = 0; k < 8; ++k) {
              const int rr = 4 * k + sub;
              const int64_t rt = rtab[q * 32 + rr];
              if (rt < 0) continue;
              const float4 v = *reinterpret_cast<const float4*>(stage + rr * kStagePitch + 4 * g);
              if (gc >= 0 && (rt & 3) == 0) {
                float* dst = C + rt + gc;
                if (atomic)
                  red_add_v4(dst, v);
                else
                  *reinterpret_cast<float4*>(dst) = v;
              } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int64_t co = cols[ch * 32 + 4 * g + i];
                  if (co < 0) continue;
                  if (atomic)
                    atomicAdd(C + rt + co, vv[i]);
                  else
                    C[rt + co] = vv[i];
                }
              }
            }
            __syncwarp();
          } else if (roff >= 0) {
            float* crow = C + roff;
            bool vec = (roff & 3) == 0;
            int64_t gc[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              gc[g] = gcol[ch * 8 + g];
              vec = vec && gc[g] >= 0;
            }
            if (vec) {
#pragma unroll
              for (int g = 0; g < 8; ++g) {
                const float4 v = make_float4(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1]),
                                             __uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3]));
                if (atomic)
                  red_add_v4(crow + gc[g], v);
                else
                  *reinterpret_cast<float4*>(crow + gc[g]) = v;
              }
            } else {
              int64_t co[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) co[i] = cols[ch * 32 + i];
              if (atomic) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (co[i] >= 0) atomicAdd(crow + co[i], __uint_as_float(r[i]));
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (co[i] >= 0) crow[co[i]] = __uint_as_float(r[i]);
              }
            }
          }
      };
      // one 32-column chunk in flight: a second buffer (measured neutral) would hold 32 more
      // registers in a kernel that sits at its 168-register cap
      uint32_t ra[32];
      if (P.c_tma) {
        // TMA-store epilogue: this warp's 32 x 32 block of each chunk -> its 4 KB staging
        // buffer (1024-B aligned) -> one bulk tensor store (reduce-add when accumulating)
        uint8_t* buf1 = reinterpret_cast<uint8_t*>(stage_out) + ew * 4096;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          uint8_t* buf = last_item ? smem + (ew * (BN / 32) + ch) * 4096 : buf1;
          tmem_ld32_issue(t_base + ch * 32, ra);
          tmem_ld_wait(ra);
          if (empty_k)
#pragma unroll
            for (int i = 0; i < 32; ++i) ra[i] = 0;
          if (lane == 0 && !last_item) bulk_wait_read();  // the previous store has read the buffer
          __syncwarp();
          if (P.c_tma == 1) {  // rows innermost: column-major block, lanes write consecutive words
            float* b = reinterpret_cast<float*>(buf);
#pragma unroll
            for (int i = 0; i < 32; ++i) b[i * 32 + lane] = __uint_as_float(ra[i]);
          } else {  // columns innermost: row-major 128-B rows, 16-B chunks swizzled (SWIZZLE_128B)
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4(__uint_as_float(ra[4 * j]), __uint_as_float(ra[4 * j + 1]),
                              __uint_as_float(ra[4 * j + 2]), __uint_as_float(ra[4 * j + 3]));
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          int wrap_tail = 32;  // first row of this warp's slab past the wrapped unit's inner extent
          if (lane == 0) {
            int c[5];
            int wrap_d = -1;
#pragma unroll
            for (int d = 0; d < 5; ++d) {
              const int qd = P.cdim_q[d];
              c[d] = cbase[d] + (qd == 1 ? q * P.c_slab : qd == 2 ? ch * 32 : 0);
              if (qd == 3) wrap_d = d;
            }
            if (wrap_d >= 0) {  // flat row index -> (inner, outer) of the wrapped M unit
              const int f = cbase[wrap_d] + q * 32;
              const int io = f / P.c_wrap;
              const int ii = f - io * P.c_wrap;
#pragma unroll
              for (int d = 0; d < 5; ++d) {
                if (P.cdim_q[d] == 3) c[d] = ii;
                if (P.cdim_q[d] == 4) c[d] = io;
              }
              wrap_tail = min(32, P.c_wrap - ii);  // TMA clips the rows past the inner extent
            }
            tma_store(&Pg.tc, buf, c, atomic);
          }
          if (P.c_wrap) {
            // rows that cross into the next outer index: per-thread stores of this lane's row
            // (a second box would need a negative start coordinate, which bulk stores reject)
            wrap_tail = __shfl_sync(0xffffffffu, wrap_tail, 0);
            const int64_t rt = rtab[q * 32 + lane];
            if (lane >= wrap_tail && rt >= 0) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int64_t co = cols[ch * 32 + i];
                if (co < 0) continue;
                if (atomic)
                  atomicAdd(C + rt + co, __uint_as_float(ra[i]));
                else
                  C[rt + co] = __uint_as_float(ra[i]);
              }
            }
          }
        }
        if (chunk >= 0 && !P.tl_zeroed && lane == 0) bulk_wait_all();  // tail chunk: writes done before its flag
      } else {
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          tmem_ld32_issue(t_base + ch * 32, ra);
          tmem_ld_wait(ra);
          process(ra, ch);
        }
      }
      if (est) stamp_it(P, 2, static_cast<uint32_t>(local / ngrp) * 4 + 3);
      if (chunk >= 0 && !P.tl_zeroed) {  // tail chunk stored / added: count it; the last one resets the flag
        epi_bar(1 + grp);
        if (et == 0) {
          uint32_t* f = P.tl_flags + (item - P.sk_full);
          __threadfence();
          if (atomicAdd(f, 1u) + 1u == static_cast<uint32_t>(P.tl_s)) atomicExch(f, 0u);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (PAIR && !leader)
        mbar_arrive_cluster(mapa(&tempty[acc], 0));  // the even CTA's MMA owns the pair's TMEM writes
      else
        mbar_arrive(&tempty[acc]);  // accumulator may be overwritten by tile t+2
    }
    if (P.c_tma && lane == 0) bulk_wait_all();  // bulk stores complete before the CTA exits
    if (threadIdx.x == 64) stamp(P, 5);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) {
    cluster_sync();  // the peer's MMAs and epilogue are done with this CTA's TMEM and barriers
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  } else {
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    if (mc) cluster_sync();  // no CTA exits while its partner may still signal its barriers
  }
  if (threadIdx.x == 0) stamp(P, 6);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// swizzle: a CUtensorMapSwizzle value (0 none, 3 128B, 4 128B with 32-B atoms)
bool encode(CUtensorMap* map, const void* ptr, const uint64_t* gdim, const uint64_t* gstride, const uint32_t* box,
            int swizzle) {
  EncodeTiledFn fn = encoder();
  if (!fn) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t boxes[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    dims[i] = gdim[i];
    boxes[i] = box[i];
  }
  uint64_t last = 16;
  for (int i = 1; i < 5; ++i) {
    uint64_t s = gstride[i];
    if (s == 0 || s % 16) s = (last + 15) / 16 * 16;
    strides[i - 1] = s;
    last = s * dims[i];
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(ptr), dims, strides, boxes, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, static_cast<CUtensorMapSwizzle>(swizzle),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

// SM count of the current device (cached per device: one process may drive several GPUs)
int sm_count() {
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

template <int BN, int STAGES, bool PAIR, bool LEAN = false>
cudaError_t launch(const TcParams& P, float* C, cudaStream_t s, int per_sm, int sms) {
  constexpr int smem =
      STAGES * (TC_BM * 128 + (PAIR ? BN * 64 : BN * 128)) + ((BN == 64 && !LEAN) ? 2 : 1) * kEpiWarps * 32 * kStagePitch * 4 +
      (2 * BN + 2 * (BN / 4) + 2 * TC_BM) * 8 + 4 * static_cast<int>(sizeof(Tile)) + 8 * (3 * STAGES + 4) + 16 + 64 +
      static_cast<int>(sizeof(TcParams)) + 1024;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  static_assert(!LEAN || smem <= 113 * 1024, "LEAN: two CTAs per SM");
  // the last item's TMA-store chunks are staged in the operand ring (one 4 KB buffer per warp
  // and 32-column chunk, see the epilogue)
  static_assert(STAGES * (TC_BM * 128 + (PAIR ? BN * 64 : BN * 128)) >=
                    ((BN == 64 && !LEAN) ? 2 : 1) * kEpiWarps * (BN / 32) * 4096,
                "operand ring too small for the last item's staging");
  // the dynamic-smem opt-in is a per-device function attribute
  static bool configured[kMaxDevices] = {};
  const int dev = current_device();
  if (!configured[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(ce_tc_kernel<BN, STAGES, PAIR, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (cudaFuncSetAttribute(ce_tc_kernel<BN, STAGES, PAIR, LEAN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
        cudaSuccess)
      cudaGetLastError();
    configured[dev] = true;
  }
  const int csize = P.mcast ? 2 : 1;
  const int64_t groups = (static_cast<int64_t>(P.tiles_m) + csize - 1) / csize * P.tiles_n * P.grid_z * P.k_split;
  const int64_t max_groups = std::max<int64_t>(1, static_cast<int64_t>(sms) * per_sm / csize);
  const int grid = static_cast<int>((groups < max_groups ? groups : max_groups) * csize);
  (void)grid;
  return ce_launch_cluster(ce_tc_kernel<BN, STAGES, PAIR, LEAN>, dim3(grid), dim3(LEAN ? 64 + 32 * kEpiWarps : kThreads),
                           smem, s,
                           static_cast<unsigned>(csize),
                           P, C);
}

int debug_flags() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CE_TC_DBG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

}  // namespace

namespace {
// Launch shape of a plan on the current device: LEAN instance and CTAs per SM, SMs used, work
// items, groups (persistent CTAs, or CTA pairs), and the tail split of a partial last round
// (r items cut into S K chunks; S = 1: none).
struct TcShape {
  bool lean;
  int per_sm, sms;
  int64_t items, ngroups;
  bool contig;
  int64_t r;
  int S;
};
TcShape tc_shape(const TcPlan& plan) {
  const TcParams& P = plan.params;
  static const int lean_mode = [] {
    const char* e = getenv("CE_TC_LEAN");
    return e ? atoi(e) : 2;
  }();
  // (32 since the end of round 2: cfg3's 256->512 @7 layer 1.38 -> 0.90 ms, stack 62.55 ->
  // 62.13 ms, cfg2 / cfg4 unchanged (same-box A/B x2-3); 40 loses on cfg3)
  static const int lean_kmax = [] {
    const char* e = getenv("CE_TC_LEAN_KMAX");
    return e ? atoi(e) : 32;
  }();
  static const bool contig_on = [] {
    const char* e = getenv("CE_TC_CONTIG");
    return !(e && *e == '0');
  }();
  static const int tail_on = [] {
    const char* e = getenv("CE_TC_TAIL");
    return e ? atoi(e) : 1;
  }();
  // (long K loops only when chunk 0 stores and the others wait for it: with ~24 K stages that
  // fixup costs what the shorter round saves -- tt1.0's 24/27-stage convs were slower,
  // tk1.0's 72-stage convs 74 -> 68 us; with C zeroed beforehand every chunk just adds)
  static const int tail_kmin = [] {
    const char* e = getenv("CE_TC_TAIL_KMIN");
    return e ? atoi(e) : 48;
  }();
  static const int tail_zkmin = [] {
    const char* e = getenv("CE_TC_TAIL_ZKMIN");
    return e ? atoi(e) : 16;
  }();
  TcShape t{};
  t.lean = lean_mode > 0 && !P.mcast && plan.bn <= 128 && P.k_per <= lean_kmax &&
           (P.native_mn || (!P.oa.mn_major && !P.ob.mn_major)) && !(P.oa.mn_major && P.oa.wide);
  t.per_sm = t.lean ? (lean_mode >= 2 ? 2 : 1) : 1;
  t.sms = plan.sm_budget > 0 ? std::min(plan.sm_budget, sm_count()) : sm_count();
  const int64_t csize = P.mcast ? 2 : 1;
  t.items = (static_cast<int64_t>(P.tiles_m) + csize - 1) / csize * P.tiles_n * P.grid_z * P.k_split;
  t.ngroups = std::min<int64_t>(t.items, std::max<int64_t>(1, static_cast<int64_t>(t.sms) * t.per_sm / csize));
  t.contig = contig_on && csize == 1 && P.k_split == 1 && t.items >= 4 * t.ngroups;
  t.r = 0;
  t.S = 1;
  const int kmin = plan.tail_zeroed ? tail_zkmin : tail_kmin;
  if (tail_on && !plan.accum && (plan.tail_flags || plan.tail_zeroed) && !t.contig && P.k_split == 1 && csize == 1 &&
      t.items > t.ngroups && t.items % t.ngroups != 0 && P.k_iters >= kmin) {
    const int64_t r = t.items % t.ngroups;
    const int64_t S = std::min<int64_t>({4, t.ngroups / r, P.k_iters / 4});
    if (S >= 2 && r <= kTailFlags) {
      t.r = r;
      t.S = static_cast<int>(S);
    }
  }
  return t;
}
}  // namespace

bool ce_tc_tail_split(const TcPlan& plan) {
  TcPlan q = plan;
  q.tail_zeroed = 1;  // (the flags buffer is bound at run time; the zeroed mode needs none)
  return tc_shape(q).S > 1;
}

cudaError_t ce_launch_tc(TcPlan& plan, const float* A, const float* B, float* C, cudaStream_t s) {
  if (!plan.valid) return cudaErrorInvalidValue;
  TcParams& P = plan.params;
  P.dbg = debug_flags();
  {
    // debug: CE_TC_DBG_AT=n applies the debug flags to the n-th TC launch of the process only
    static const int at = [] {
      const char* e = getenv("CE_TC_DBG_AT");
      return e ? atoi(e) : -1;
    }();
    static int counter = 0;
    if (at >= 0 && counter++ != at) P.dbg = 0;
  }
  if (plan.cached_a != A) {
    if (!encode(&P.ta, A, plan.gdim_a, plan.gstride_a, plan.box_a, plan.swz_a)) return cudaErrorInvalidValue;
    plan.cached_a = A;
  }
  if (plan.cached_b != B) {
    if (!encode(&P.tb, B, plan.gdim_b, plan.gstride_b, plan.box_b, plan.swz_b)) return cudaErrorInvalidValue;
    plan.cached_b = B;
  }
  if (P.c_tma) {
    // (a caller's output that is not 16-B aligned falls back to the per-thread stores)
    const bool al = (reinterpret_cast<uintptr_t>(C) & 15u) == 0;
    if (!al) {
      P.c_tma = 0;
    } else if (plan.cached_c != C) {
      if (!encode(&P.tc, C, plan.gdim_c, plan.gstride_c, plan.box_c, plan.swz_c)) return cudaErrorInvalidValue;
      plan.cached_c = C;
    }
  }
  if (static_cast<int64_t>(P.tiles_m) * P.tiles_n * P.grid_z * P.k_split >= (1ll << 32))
    return cudaErrorInvalidConfiguration;
  // LEAN instances (two CTAs per SM, see ce_tc_kernel) for short K loops with N tiles <= 128
  // and no in-smem transposes.  CE_TC_LEAN: 0 off, 1 one CTA of this launch per SM (the
  // second slot takes the next kernel's set-up), 2 (default) two CTAs of this launch per SM.
  // cfg2 step (same-box A/B x3): off 1.127-1.131, 1 1.131-1.138, 2 1.119-1.121 ms.
  const TcShape sh = tc_shape(plan);
  const bool lean = sh.lean;
  const int per_sm = sh.per_sm;
  const int sms = sh.sms;
  {
    P.n_items = static_cast<uint32_t>(sh.items);
    P.sk_full = 0;
    P.sk_r = 0;
    P.contig = 0;
    if (sh.contig) {
      P.contig = 1;
      P.ipg = static_cast<uint32_t>(sh.items / sh.ngroups);
      P.irem = static_cast<uint32_t>(sh.items % sh.ngroups);
    }
    P.dkit = tc_div(static_cast<uint32_t>(std::max(1, P.k_iters)));
    // tail split of a partial last round (see work_next): the r items left after the full
    // rounds are each cut into S = min(4, ngroups / r) K chunks run by the otherwise idle
    // groups; chunk 0 stores, the others wait for it (P.tl_flags, zeroed by the executor and
    // left zero by the last chunk) and add -- or, when the executor zeroed C beforehand
    // (plan.tail_zeroed), every chunk adds without a handshake.  CE_TC_TAIL=0 off.
    P.tl_s = 1;
    P.tl_flags = plan.tail_flags;
    P.tl_zeroed = 0;
    static const bool tail_first = [] {  // CE_TC_TAIL_FIRST=0: tail chunks after the whole items
      const char* e = getenv("CE_TC_TAIL_FIRST");
      return !(e && *e == '0');
    }();
    P.tl_first = tail_first ? 1 : 0;
    P.acc_out = plan.accum ? 1 : 0;
    if (sh.S > 1) {
      P.sk_full = static_cast<uint32_t>(sh.items - sh.r);
      P.sk_r = static_cast<uint32_t>(sh.r);
      P.tl_s = sh.S;
      P.tl_zeroed = plan.tail_zeroed ? 1 : 0;
    }
  }
  if (P.k_split > 1 && !plan.accum && !plan.zeroed) {
    cudaError_t e = cudaMemsetAsync(C, 0, static_cast<size_t>(plan.out_span) * 4, s);
    if (e != cudaSuccess) return e;
  }
  if (P.mcast == 2) {
    switch (plan.bn) {
      case 64: return launch<64, 9, true>(P, C, s, 1, sms);
      case 128: return launch<128, 8, true>(P, C, s, 1, sms);
      default: return launch<256, 6, true>(P, C, s, 1, sms);
    }
  }
  if (lean) {
    if (plan.bn == 64) return launch<64, 3, false, true>(P, C, s, per_sm, sms);
    return launch<128, 2, false, true>(P, C, s, per_sm, sms);
  }
  switch (plan.bn) {
    case 64: return launch<64, 7, false>(P, C, s, 1, sms);
    case 128: return launch<128, 6, false>(P, C, s, 1, sms);
    default: return launch<256, 4, false>(P, C, s, 1, sms);
  }
}

// Debug only (not part of include/ce/ce.h): copy the phase timestamps of the last
// launch with CE_TC_DBG & 32.  n <= 160*8.
extern "C" int ce_debug_tc_timestamps(unsigned long long* out, int n) {  // n <= 160*16
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_tc_ts, sizeof(unsigned long long) * n));
}
extern "C" int ce_debug_tc_iter_timestamps(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_tc_it, sizeof(unsigned long long) * 768));
}
