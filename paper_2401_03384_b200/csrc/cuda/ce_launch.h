// Kernel launch helper with Programmatic Dependent Launch (PDL).
//
// Every kernel of the executor starts with ce_pdl_enter(): it lets the next
// kernel in the stream be scheduled immediately (griddepcontrol.launch_dependents)
// and then waits for the previous kernel's completion and memory flush
// (griddepcontrol.wait) before touching global memory.  Launch latency and the
// successor's prologue (barrier init, TMEM allocation, descriptor prefetch) thus
// overlap the predecessor's tail.  CE_PDL=0 disables the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

__device__ __forceinline__ void ce_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void ce_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void ce_pdl_enter() {
  ce_pdl_trigger();
  ce_pdl_wait();
}

inline bool ce_pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("CE_PDL");
    v = (e && *e == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename... Exp, typename... Act>
cudaError_t ce_launch(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ce_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}
