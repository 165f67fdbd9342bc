// Store-throughput microbenchmark (tool): each CTA of 128 threads writes `per_cta` bytes
// with float4 or float stores, rows coalesced; reports GB/s per SM and chip.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void st4(float4* out, long per_cta_f4, int reps) {
  float4* base = out + blockIdx.x * per_cta_f4;
  float4 v = make_float4(threadIdx.x, 1, 2, 3);
  for (int r = 0; r < reps; ++r)
    for (long i = threadIdx.x; i < per_cta_f4; i += blockDim.x) base[i] = v;
}
__global__ void st1(float* out, long per_cta, int reps) {
  float* base = out + blockIdx.x * per_cta;
  for (int r = 0; r < reps; ++r)
    for (long i = threadIdx.x; i < per_cta; i += blockDim.x) base[i] = i;
}
// strided rows like the epilogue: 32 rows per warp-instruction? each thread writes its own row (stride pitch)
__global__ void strow(float* out, long pitch, int cols, int reps) {
  float* base = out + static_cast<long>(blockIdx.x) * 128 * pitch;
  for (int r = 0; r < reps; ++r)
    for (int c = 0; c < cols; c += 4)
      *reinterpret_cast<float4*>(base + threadIdx.x * pitch + c) = make_float4(c, 1, 2, 3);
}
int main() {
  float* buf;
  cudaMalloc(&buf, 1l << 31);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) {
    for (int grid : {1, 16, 148}) {
      const long per = 128 * 1024 / 16;  // 128 KB per CTA per rep
      const int reps = 20;
      st4<<<grid, threads>>>(reinterpret_cast<float4*>(buf), per, 2);
      cudaEventRecord(e0);
      st4<<<grid, threads>>>(reinterpret_cast<float4*>(buf), per, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double b = 1.0 * grid * per * 16 * reps;
      printf("st4 thr %3d grid %3d: %7.1f GB/s/SM %8.0f GB/s chip\n", threads, grid, b / grid / ms / 1e6, b / ms / 1e6);
      st1<<<grid, threads>>>(buf, per * 4, 2);
      cudaEventRecord(e0);
      st1<<<grid, threads>>>(buf, per * 4, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("st1 thr %3d grid %3d: %7.1f GB/s/SM %8.0f GB/s chip\n", threads, grid, b / grid / ms / 1e6, b / ms / 1e6);
    }
  }
  for (int grid : {1, 148}) {
    const int reps = 20;
    strow<<<grid, 128>>>(buf, 232, 232, 2);
    cudaEventRecord(e0);
    strow<<<grid, 128>>>(buf, 232, 232, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double b = 1.0 * grid * 128 * 232 * 4 * reps;
    printf("strow(thread=row, float4) grid %3d: %7.1f GB/s/SM %8.0f GB/s chip\n", grid, b / grid / ms / 1e6, b / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
