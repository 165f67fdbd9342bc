// Bulk / TMA store throughput (tool): smem -> global with cp.async.bulk (1-D rows) and
// cp.async.bulk.tensor (2-D boxes); per SM and chip GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void bulk_rows(float* out, long pitch_f, int row_bytes, int rows, int reps) {
  extern __shared__ __align__(128) uint8_t sm[];
  if (threadIdx.x < 32) {
    for (int r = 0; r < reps; ++r) {
      for (int i = threadIdx.x; i < rows; i += 32) {
        float* dst = out + (static_cast<long>(blockIdx.x) * rows + i) * pitch_f;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su(sm + (i % 64) * row_bytes)),
                     "r"(row_bytes)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void tma_store(const __grid_constant__ CUtensorMap map, int rows_box, int nbox, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  if (threadIdx.x == 0) {
    for (int r = 0; r < reps; ++r) {
      for (int j = 0; j < nbox; ++j) {
        const int c1 = (blockIdx.x * nbox + j) * rows_box;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map), "r"(0),
                     "r"(c1), "r"(su(sm + (j % 4) * rows_box * 128))
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  float* buf;
  cudaMalloc(&buf, 1l << 31);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int row_bytes : {512, 928, 1024}) {
    for (int grid : {1, 148}) {
      const int rows = 128, reps = 20;
      bulk_rows<<<grid, 32, 64 * row_bytes>>>(buf, 256, row_bytes, rows, 2);
      cudaEventRecord(e0);
      bulk_rows<<<grid, 32, 64 * row_bytes>>>(buf, 256, row_bytes, rows, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double b = 1.0 * grid * rows * row_bytes * reps;
      printf("bulk rows %4dB grid %3d: %7.1f GB/s/SM %8.0f GB/s chip\n", row_bytes, grid, b / grid / ms / 1e6, b / ms / 1e6);
    }
  }
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fp);
  for (int rows_box : {32, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {32, 1u << 22};
    cuuint64_t strides[1] = {928};
    cuuint32_t box[2] = {32, static_cast<cuuint32_t>(rows_box)};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 148}) {
      const int nbox = 8, reps = 20;
      tma_store<<<grid, 32, 4 * rows_box * 128 + 1024>>>(map, rows_box, nbox, 2);
      cudaEventRecord(e0);
      tma_store<<<grid, 32, 4 * rows_box * 128 + 1024>>>(map, rows_box, nbox, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double b = 1.0 * grid * nbox * rows_box * 128 * reps;
      printf("tma store box 32x%3d (pitch 928) grid %3d: %7.1f GB/s/SM %8.0f GB/s chip\n", rows_box, grid, b / grid / ms / 1e6,
             b / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
