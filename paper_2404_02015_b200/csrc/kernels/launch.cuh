// Host launcher: every kernel of a prefill/decode job goes through launch(),
// which sets programmatic stream serialization (PDL) unless disabled, so a
// kernel's prologue -- and the GEMM's weight streaming, which does not depend
// on the previous kernel -- overlaps the tail of its predecessor.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <utility>

namespace mux {

// Process-wide switch (default on); "pdl" option of mux_unit_set_option.
bool& pdl_enabled();

// Force-load kernels now (CUDA lazy loading would otherwise load a kernel at
// its first launch, which can wait for the device to idle -- a deadlock when
// an earlier kernel of the same process spins on a tensor-parallel peer).
//
// Debug (MUX_CARVEOUT=1): every job kernel prefers the maximum shared-memory
// carveout, so no L1/shared reconfiguration can sit between a GEMM and its
// neighbours. Measured: no change in decode rounds (profiles/r02_gemm_st.txt),
// so it is off by default.
inline bool max_carveout_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MUX_CARVEOUT");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

template <typename... K>
inline cudaError_t preload(K... kernels) {
  cudaError_t err = cudaSuccess;
  cudaFuncAttributes attr;
  ((err = err == cudaSuccess ? cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(kernels)) : err), ...);
  if (err == cudaSuccess && max_carveout_enabled())
    ((err = err == cudaSuccess ? cudaFuncSetAttribute(reinterpret_cast<const void*>(kernels),
                                                      cudaFuncAttributePreferredSharedMemoryCarveout,
                                                      cudaSharedmemCarveoutMaxShared)
                               : err),
     ...);
  return err;
}

// Kernel attributes (cudaFuncSetAttribute) are per device: a process that
// drives units on several GPUs must set them once on EACH device it launches
// on. Returns the first error of f() on the current device.
class PerDeviceOnce {
 public:
  template <typename F>
  cudaError_t run(F&& f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu_);
    if (done_ & (1ull << dev)) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) done_ |= 1ull << dev;
    return e;
  }

 private:
  std::mutex mu_;
  unsigned long long done_ = 0;
};

template <typename... P, typename... A>
inline cudaError_t launch(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          A&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

}  // namespace mux
