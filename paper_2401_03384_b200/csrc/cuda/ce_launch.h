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
#include <mutex>
#include <set>
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

// Every kernel asks for the maximum shared-memory carveout: the tcgen05 kernels need
// ~216 KB, and an SM whose carveout differs from the next kernel's must drain and
// reconfigure before that kernel's CTAs can land (which also defeats PDL overlap).
// CE_CARVEOUT=0 leaves the driver default.
inline void ce_prefer_max_smem(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> seen;
  static const bool on = [] {
    const char* e = std::getenv("CE_CARVEOUT");
    return !(e && *e == '0');
  }();
  if (!on) return;
  // (a function attribute is set per device: key on (kernel, device))
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (seen.insert({fn, dev}).second) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

template <typename... Exp, typename... Act>
cudaError_t ce_launch_cluster(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              unsigned cluster_x, Act&&... args) {
  ce_prefer_max_smem(reinterpret_cast<const void*>(kernel));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (ce_pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

template <typename... Exp, typename... Act>
cudaError_t ce_launch(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Act&&... args) {
  return ce_launch_cluster(kernel, grid, block, smem, s, 1u, std::forward<Act>(args)...);
}
