// TMA load throughput microbenchmark (tool, not product): one producer thread per CTA
// streams boxes of [32 floats (128 B, SWIZZLE_128B)][rows] into an S-stage smem ring, a
// consumer thread releases stages.  Reports GB/s per SM and per chip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu -lcuda
//   tools/tma_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int S>
__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int rows, int nbox,
                                                    int iters, long rows_total, long* sink, int depth3, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* ring = smem;
  const int stage_bytes = nbox * rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // each CTA walks its own slice of rows
  const long per_cta = rows_total / gridDim.x;
  const long base = per_cta * blockIdx.x;
  if (threadIdx.x == 0) {
    long rcur = 0;
    const long rspan = (per_cta - rows) / rows * rows;
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      const uint32_t ph = ((it / S) & 1) ^ 1;
      if (mode & 2)
        asm volatile(
            "{\n.reg .pred p;\nT1:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra T1;\n}\n" ::"r"(
                su(&empty[s])),
            "r"(ph)
            : "memory");
      else
        asm volatile(
            "{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(
                su(&empty[s])),
            "r"(ph)
            : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(stage_bytes)
                   : "memory");
      for (int j = 0; j < nbox; ++j) {
        const long r = base + rcur;
        rcur += rows;
        if (rcur >= rspan) rcur = 0;
        const int c0 = 0, c1 = static_cast<int>(r), c2 = 0;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(su(ring + s * stage_bytes + j * rows * 128)),
            "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(su(&full[s]))
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    long acc = 0;
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      if (mode & 1)
        asm volatile(
            "{\n.reg .pred p;\nT2:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra T2;\n}\n" ::"r"(
                su(&full[s])),
            "r"(ph)
            : "memory");
      else
        asm volatile(
            "{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(
                su(&full[s])),
            "r"(ph)
            : "memory");
      acc += ring[s * stage_bytes + 5];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    if (acc == 123456789) sink[0] = acc;
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S>
void run(Enc enc, float* buf, long* sink, int nsm, size_t pitch, size_t foot, int rows, int nbox, int depth3, int mode = 0) {
  // 3-D map: [32 floats][rows_total/depth3 rows, stride pitch][depth3, stride pitch*rows_total/depth3]
  const long rows_total = static_cast<long>(foot / pitch);
  const long r1 = rows_total / depth3;
  CUtensorMap map;
  cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(r1), static_cast<cuuint64_t>(depth3)};
  cuuint64_t strides[2] = {pitch, pitch * r1};
  cuuint32_t box[3] = {32, static_cast<cuuint32_t>(rows / depth3), static_cast<cuuint32_t>(depth3)};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed rows %d depth3 %d\n", rows, depth3);
    return;
  }
  const int stage_bytes = nbox * rows * 128;
  const int smem = S * stage_bytes + 2 * S * 8 + 1024;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(tma_stream<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, nsm}) {
    const int iters = 400;
    tma_stream<S><<<grid, 64, smem>>>(map, rows, nbox, 20, r1, sink, 1, mode);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_stream<S><<<grid, 64, smem>>>(map, rows, nbox, iters, r1, sink, 1, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = static_cast<double>(grid) * iters * stage_bytes;
    printf("mode %d S %2d pitch %4zu foot %5zuMB box %3dx%d boxes/stage %d grid %3d : %7.1f GB/s/SM %7.0f GB/s chip %6.3f us/stage %6.1f ns/box\n",
           mode, S, pitch, foot >> 20, rows / depth3, depth3, nbox, grid, bytes / grid / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / 1e9, ms * 1e3 / iters, ms * 1e6 / iters / nbox);
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fp);
  const size_t big = 1ull << 30;
  float* buf;
  cudaMalloc(&buf, big * 2);
  cudaMemset(buf, 0, big * 2);
  long* sink;
  cudaMalloc(&sink, 8);
  const size_t l2 = size_t(24) << 20;
  for (int rows : {32, 128, 256}) {
    run<2>(enc, buf, sink, nsm, 128, l2, rows, 1, 1);
    run<4>(enc, buf, sink, nsm, 128, l2, rows, 1, 1);
    run<6>(enc, buf, sink, nsm, 128, l2, rows, 1, 1);
    run<12>(enc, buf, sink, nsm, 128, l2, rows, 1, 1);
    run<6>(enc, buf, sink, nsm, 128, l2, rows, 2, 1);
    run<6>(enc, buf, sink, nsm, 128, l2, rows, 4, 1);
    run<6>(enc, buf, sink, nsm, 928, l2, rows, 1, 1);
    run<6>(enc, buf, sink, nsm, 128, big, rows, 1, 1);
    run<6>(enc, buf, sink, nsm, 928, big, rows, 1, 1);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(e));
  return 0;
}
