// Store-throughput probe for the TC epilogue's row-mode pattern: each warp writes a 32-row x
// NCOL tile where a lane owns a row (rows contiguous in memory) and columns sit `cstride` floats
// apart (C = [b, t, h, w], rows = hw, columns = t).  Reports GB/s for several CTA counts / warps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void st_rows(float* C, int ncol, long cstride, long tile_stride, int tiles_per_cta) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int t = 0; t < tiles_per_cta; ++t) {
    long tile = (long)(blockIdx.x * tiles_per_cta + t);
    const long r = tile * tile_stride + warp * 32 + lane;  // C = [b][256][196], rows = (b, hw)
    float* base = C + (r / 196) * 256 * 196 + r % 196;
#pragma unroll 4
    for (int c = 0; c < ncol; ++c) base[c * cstride] = (float)c;
  }
}
// same tile, but each lane writes float4 of 4 consecutive rows (8 lanes per 32 rows)
__global__ void st_rows_v4(float* C, int ncol, long cstride, long tile_stride, int tiles_per_cta) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int t = 0; t < tiles_per_cta; ++t) {
    long tile = (long)(blockIdx.x * tiles_per_cta + t);
    const long r = tile * tile_stride + warp * 32 + (lane & 7) * 4;
    float* base = C + (r / 196) * 256 * 196 + r % 196;
#pragma unroll 4
    for (int c = lane >> 3; c < ncol; c += 4)
      *reinterpret_cast<float4*>(base + c * cstride) = make_float4(c, c, c, c);
  }
}
// TC epilogue transposed-store pattern: a warp owns 32 rows x NCOL columns of a row-major C
// (pitch floats); per 32-column chunk, 8 instructions each storing 4 rows x 128 B (lane ->
// row 4k + lane/8, columns 4*(lane%8)).
__global__ void st_tr(float* C, int ncol, long pitch, int tiles_per_cta) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int t = 0; t < tiles_per_cta; ++t) {
    const long row0 = ((long)(blockIdx.x * tiles_per_cta + t) * (blockDim.x / 32) + warp) * 32;
    for (int ch = 0; ch < ncol / 32; ++ch) {
#pragma unroll 4
      for (int k = 0; k < 8; ++k) {
        const long r = row0 + 4 * k + (lane >> 3);
        *reinterpret_cast<float4*>(C + r * pitch + ch * 32 + 4 * (lane & 7)) = make_float4(k, k, k, k);
      }
    }
  }
}
int main() {
  const long cstride = 196;
  float* C;
  size_t bytes = 1ull << 30;
  cudaMalloc(&C, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v4 = 0; v4 < 2; ++v4)
  for (int warps : {4, 8, 16})
    for (int ctas : {148, 296, 592}) {
      const int ncol = 128, tiles = 2;
      const long tile_stride = 32 * warps;  // rows of consecutive tiles contiguous
      
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        if (v4) st_rows_v4<<<ctas, 32 * warps>>>(C, ncol, cstride, tile_stride, tiles);
        else st_rows<<<ctas, 32 * warps>>>(C, ncol, cstride, tile_stride, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gb = (double)ctas * tiles * warps * 32 * ncol * 4 / 1e9;
        if (it == 2) printf("v4=%d warps=%2d ctas=%3d  %.2f us  %.0f GB/s  per-CTA %.1f GB/s\n", v4, warps, ctas, ms * 1e3, gb / (ms * 1e-3), gb / (ms * 1e-3) / ctas);
      }
    }
  for (int warps : {4, 8})
    for (int ctas : {148, 296}) {
      const int ncol = 224, tiles = 1;
      const long pitch = 232;
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        st_tr<<<ctas, 32 * warps>>>(C, ncol, pitch, tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double gb = (double)ctas * tiles * warps * 32 * ncol * 4 / 1e9;
        if (it == 2) printf("tr warps=%d ctas=%3d  %.2f us  %.0f GB/s  per-CTA %.1f GB/s\n", warps, ctas, ms * 1e3, gb / (ms * 1e-3), gb / (ms * 1e-3) / ctas);
      }
    }
  return 0;
}
