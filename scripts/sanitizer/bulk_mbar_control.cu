// Racecheck control (TEST INFRASTRUCTURE): the minimal correct pattern K1
// uses -- one thread issues cp.async.bulk global->shared with mbarrier
// complete_tx, every thread waits on the mbarrier phase, then reads the
// bytes; the slot is refilled only after all readers arrive on an "empty"
// mbarrier. If compute-sanitizer --tool racecheck reports hazards here, its
// model of non-tensor bulk copies does not follow mbarrier completion.
// nvcc -gencode arch=compute_100a,code=sm_100a -o bulk_mbar_control bulk_mbar_control.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void ring(const uint4* src, float* out, int rounds) {
  __shared__ __align__(128) uint4 buf[2][256];  // 2 x 4 KiB
  __shared__ __align__(8) uint64_t full[2], empty[2];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(blockDim.x / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* b, uint32_t par) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su32(b)), "r"(par) : "memory");
  };
  float acc = 0.f;
  for (int i = 0; i < rounds; ++i) {
    const int s = i & 1;
    if (threadIdx.x == 0) {
      if (i >= 2) wait(&empty[s], ((i >> 1) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(4096) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(su32(buf[s])),
                   "l"(src + (i % 8) * 256), "r"(su32(&full[s])) : "memory");
    }
    wait(&full[s], (i >> 1) & 1);
    const uint4 v = buf[s][threadIdx.x];
    acc += __uint_as_float(v.x) + __uint_as_float(v.w);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint4* src;
  float* out;
  cudaMalloc(&src, 8 * 4096);
  cudaMemset(src, 0, 8 * 4096);
  cudaMalloc(&out, 4 * 256 * 4);
  ring<<<4, 256>>>(src, out, 16);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("bulk_mbar_control: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
