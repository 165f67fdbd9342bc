// tcgen05 kind::tf32 implicit-GEMM kernel for sm_100a (families a + b1).
//
// One CTA = one 128 x BN output tile (x one K split).  128 threads:
//   warp 0 lane 0 : TMA producer   (cp.async.bulk.tensor.5d -> smem ring, mbarrier tx)
//   warp 1 lane 0 : MMA issuer     (tcgen05.mma.cta_group::1.kind::tf32, D in TMEM)
//   warp 2        : TMEM allocator (tcgen05.alloc / dealloc)
//   all 4 warps   : epilogue       (tcgen05.ld 32x32b -> registers -> scatter store)
// Operand tiles are 128-byte rows with the hardware 128B swizzle shared by TMA and
// the UMMA smem descriptors.  Convolution taps are K-loop iterations whose TMA
// coordinates are shifted (ce_tc.h); Same/Full padding is TMA's OOB zero fill.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include "ce_tc.h"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // SM100 UMMA shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
  // version 1 [46,48), base offset 0, layout SWIZZLE_128B (2) [61,64).
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
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

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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

// Value of every unit for this CTA (tile origins / grid digits); K units filled per iteration.
__device__ __forceinline__ void tile_values(const TcParams& P, int32_t* val, int split_out[1]) {
  for (int i = 0; i < P.nunits; ++i) val[i] = 0;
  int64_t x = blockIdx.x;
  for (int i = 0; i < P.nm; ++i) {
    const TcUnit& u = P.u[P.mt[i]];
    const int32_t n = (u.ext + u.box - 1) / u.box;
    val[P.mt[i]] = static_cast<int32_t>(x % n) * u.box;
    x /= n;
  }
  x = blockIdx.y;
  for (int i = 0; i < P.nn; ++i) {
    const TcUnit& u = P.u[P.nt[i]];
    const int32_t n = (u.ext + u.box - 1) / u.box;
    val[P.nt[i]] = static_cast<int32_t>(x % n) * u.box;
    x /= n;
  }
  x = blockIdx.z;
  split_out[0] = static_cast<int>(x % P.k_split);
  x /= P.k_split;
  for (int i = 0; i < P.ng; ++i) {
    const TcUnit& u = P.u[P.gu[i]];
    val[P.gu[i]] = static_cast<int32_t>(x % u.ext);
    x /= u.ext;
  }
}

__device__ __forceinline__ void k_values(const TcParams& P, int it, int32_t* val) {
  for (int i = 0; i < P.nk; ++i) {
    const TcUnit& u = P.u[P.ku[i]];
    const int32_t n = (u.ext + u.box - 1) / u.box;
    val[P.ku[i]] = (it % n) * u.box;
    it /= n;
  }
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

// Offset in C of a tile-local index `local` along the given unit list (first fastest); -1 if outside.
__device__ __forceinline__ int64_t tile_offset(const TcParams& P, const int32_t* list, int n, const int32_t* val,
                                               int local) {
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    const TcUnit& u = P.u[list[i]];
    const int d = local % u.box;
    local /= u.box;
    int64_t v = static_cast<int64_t>(val[list[i]]) + d;
    if (v >= u.ext) return -1;
    for (int k = 0; k < u.nv; ++k) {
      off += (v % u.vext[k]) * u.sc[k];
      v /= u.vext[k];
    }
  }
  return local == 0 ? off : -1;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1) ce_tc_kernel(const __grid_constant__ TcParams P, float* __restrict__ C) {
  constexpr int A_BYTES = TC_BM * 128;
  constexpr int B_BYTES = BN * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  int64_t* row_off = reinterpret_cast<int64_t*>(tmem_slot + 4);  // [128]
  int64_t* col_off = row_off + TC_BM;                               // [BN]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int32_t val[TC_MAX_UNITS];
  int split;
  tile_values(P, val, &split);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&P.ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&P.tb) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // epilogue address tables (independent of the mainloop)
  for (int r = threadIdx.x; r < TC_BM; r += 128)
    row_off[r] = r < P.m_rows ? tile_offset(P, P.mt, P.nm, val, r) : -1;
  for (int c = threadIdx.x; c < BN; c += 128) col_off[c] = c < P.n_cols ? tile_offset(P, P.nt, P.nn, val, c) : -1;
  int64_t base = 0;
  for (int i = 0; i < P.ng; ++i) {
    const TcUnit& u = P.u[P.gu[i]];
    int64_t v = val[P.gu[i]];
    for (int k = 0; k < u.nv; ++k) {
      base += (v % u.vext[k]) * u.sc[k];
      v /= u.vext[k];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int per = (P.k_iters + P.k_split - 1) / P.k_split;
  const int k0 = split * per;
  const int k1 = min(P.k_iters, k0 + per);

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    const uint32_t bytes = static_cast<uint32_t>(P.oa.stage_bytes + P.ob.stage_bytes);
    for (int it = k0, i = 0; it < k1; ++it, ++i) {
      const int s = i % STAGES;
      const uint32_t round = static_cast<uint32_t>(i / STAGES);
      mbar_wait(&empty[s], (round & 1) ^ 1);
      k_values(P, it, val);
      mbar_expect_tx(&full[s], bytes);
      int c[5];
      coords(P.oa, val, c);
      for (int j = 0; j < P.oa.nsub; ++j) {
        int cj[5] = {c[0] + 32 * j, c[1], c[2], c[3], c[4]};
        tma_load(sA + s * A_BYTES + j * 4096, &P.ta, &full[s], cj);
      }
      coords(P.ob, val, c);
      for (int j = 0; j < P.ob.nsub; ++j) {
        int cj[5] = {c[0] + 32 * j, c[1], c[2], c[3], c[4]};
        tma_load(sB + s * B_BYTES + j * 4096, &P.tb, &full[s], cj);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    for (int it = k0, i = 0; it < k1; ++it, ++i) {
      const int s = i % STAGES;
      const uint32_t round = static_cast<uint32_t>(i / STAGES);
      mbar_wait(&full[s], round & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
      for (int kk = 0; kk < TC_BK / 8; ++kk) {
        // K-major: advance 32 B inside the swizzled 128-B row; MN-major: next 8-row K group (1 KB)
        const uint64_t ad = P.oa.mn_major ? smem_desc(a0 + kk * 1024, P.mn_lbo, P.mn_sbo) : smem_desc(a0 + kk * 32, 16, 1024);
        const uint64_t bd = P.ob.mn_major ? smem_desc(b0 + kk * 1024, P.mn_lbo, P.mn_sbo) : smem_desc(b0 + kk * 32, 16, 1024);
        mma_tf32(tmem, ad, bd, P.idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&empty[s]);  // frees the smem slot once these MMAs retire
    }
    mma_commit(accf);  // accumulator complete
  }
  __syncwarp();

  // ------------------------------------------------------------ epilogue
  mbar_wait(accf, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  const bool atomic = P.k_split > 1;
  const bool empty_k = k1 <= k0;
  float* stage = reinterpret_cast<float*>(sA) + warp * 32 * 33;  // mainloop smem is free now
#pragma unroll 1
  for (int ch = 0; ch < BN / 32; ++ch) {
    if (ch * 32 >= P.n_cols) break;
    uint32_t r[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + ch * 32, r);
    if (empty_k)
      for (int i = 0; i < 32; ++i) r[i] = 0;
    if (P.transpose_store) {
      for (int i = 0; i < 32; ++i) stage[lane * 33 + i] = __uint_as_float(r[i]);
      __syncwarp();
      const int64_t co = col_off[ch * 32 + lane];
      for (int rr = 0; rr < 32; ++rr) {
        const int64_t ro = row_off[warp * 32 + rr];
        if (ro < 0 || co < 0) continue;
        const float v = stage[rr * 33 + lane];
        if (atomic)
          atomicAdd(C + base + ro + co, v);
        else
          C[base + ro + co] = v;
      }
      __syncwarp();
    } else {
      const int64_t ro = row_off[row];
      if (ro >= 0) {
        for (int i = 0; i < 32; ++i) {
          const int64_t co = col_off[ch * 32 + i];
          if (co < 0) continue;
          const float v = __uint_as_float(r[i]);
          if (atomic)
            atomicAdd(C + base + ro + co, v);
          else
            C[base + ro + co] = v;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
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

bool encode(CUtensorMap* map, const void* ptr, const uint64_t* gdim, const uint64_t* gstride, const uint32_t* box) {
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
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int STAGES>
cudaError_t launch(const TcParams& P, float* C, cudaStream_t s) {
  constexpr int smem = STAGES * (TC_BM * 128 + BN * 128) + 1024 + 256 + (TC_BM + BN) * 8 + 64;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(ce_tc_kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(static_cast<unsigned>(P.tiles_m), static_cast<unsigned>(P.tiles_n),
            static_cast<unsigned>(P.grid_z * P.k_split));
  ce_tc_kernel<BN, STAGES><<<grid, 128, smem, s>>>(P, C);
  return cudaGetLastError();
}

}  // namespace

cudaError_t ce_launch_tc(TcPlan& plan, const float* A, const float* B, float* C, cudaStream_t s) {
  if (!plan.valid) return cudaErrorInvalidValue;
  TcParams& P = plan.params;
  P.mn_lbo = 4096;
  P.mn_sbo = 1024;
  if (const char* e = getenv("CE_MN_LBO")) P.mn_lbo = atoi(e);
  if (const char* e = getenv("CE_MN_SBO")) P.mn_sbo = atoi(e);
  if (const char* e = getenv("CE_IDESC_XOR")) P.idesc ^= static_cast<uint32_t>(strtoul(e, nullptr, 0));
  if (plan.cached_a != A) {
    if (!encode(&P.ta, A, plan.gdim_a, plan.gstride_a, plan.box_a)) return cudaErrorInvalidValue;
    plan.cached_a = A;
  }
  if (plan.cached_b != B) {
    if (!encode(&P.tb, B, plan.gdim_b, plan.gstride_b, plan.box_b)) return cudaErrorInvalidValue;
    plan.cached_b = B;
  }
  if (P.k_split > 1) {
    cudaError_t e = cudaMemsetAsync(C, 0, static_cast<size_t>(plan.out_span) * 4, s);
    if (e != cudaSuccess) return e;
  }
  switch (plan.bn) {
    case 64: return launch<64, 8>(P, C, s);
    case 128: return launch<128, 6>(P, C, s);
    default: return launch<256, 4>(P, C, s);
  }
}
