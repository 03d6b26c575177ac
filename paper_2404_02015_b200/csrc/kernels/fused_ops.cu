// K5: the small LLaMA ops around the GEMMs, fused where a pass over the
// activations is needed anyway: embedding + RMSNorm, residual RMSNorm, row
// argmax (greedy sampling), row gather, and deterministic weight
// initialisation. All HBM-bound; one CTA per token row.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"
#include "launch.cuh"

namespace mux {
namespace {

constexpr int kRowThreads = 256;

__device__ __forceinline__ float block_sum(float v, float* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) t += scratch[w];
  __syncthreads();
  return t;
}

// y = x * rsqrt(mean(x^2) + eps) * w, rounded to bf16. x lives in resid (fp32).
__device__ void rmsnorm_row(const float* x, const float* w, __nv_bfloat16* y, int hidden, float eps,
                            float* scratch) {
  float ss = 0.f;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) ss = fmaf(x[i], x[i], ss);
  const float tot = block_sum(ss, scratch);
  const float inv = rsqrtf(tot / static_cast<float>(hidden) + eps);
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) y[i] = __float2bfloat16_rn(x[i] * inv * w[i]);
}

__global__ void __launch_bounds__(kRowThreads) embed_rmsnorm_kernel(
    const __nv_bfloat16* emb, const int32_t* tokens, const float* norm_w, float* resid,
    __nv_bfloat16* xn, int hidden, float eps) {
  __shared__ float scratch[32];
  grid_dep_wait();
  grid_dep_launch();
  const int t = blockIdx.x;
  const int64_t tok = tokens[t];
  const __nv_bfloat16* e = emb + tok * hidden;
  float* x = resid + static_cast<int64_t>(t) * hidden;
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) x[i] = __bfloat162float(e[i]);
  __syncthreads();
  rmsnorm_row(x, norm_w, xn + static_cast<int64_t>(t) * hidden, hidden, eps, scratch);
}

// Rows strided over at most one CTA per SM of the partition, float4 loads
// kept in registers between the two passes, norm weights read after the
// reduction (L2-resident). Few registers (kVec = exact float4s per thread)
// and no shared memory beyond the reduction scratch: the kernel's CTAs fit
// beside a GEMM CTA (224 KB smem, 46 K registers), so they are resident
// before the residual GEMM ends and the next GEMM's CTAs can start their
// prologue and weight stream while the norm runs (PDL).
template <int kVec>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_rows_kernel(const float* resid, const float* norm_w,
                                                                   __nv_bfloat16* xn, int T, int hidden, float eps) {
  __shared__ float scratch[32];
  const int n4 = hidden / 4;
  // norm weights do not depend on the predecessor: in registers before the wait
  const float4* w = reinterpret_cast<const float4*>(norm_w);
  float4 g[kVec];
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    g[k] = i < n4 ? w[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  grid_dep_wait();
  grid_dep_launch();
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const float4* x = reinterpret_cast<const float4*>(resid + static_cast<int64_t>(t) * hidden);
    float4 v[kVec];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = threadIdx.x + k * kRowThreads;
      v[k] = i < n4 ? x[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      ss = fmaf(v[k].x, v[k].x, fmaf(v[k].y, v[k].y, fmaf(v[k].z, v[k].z, fmaf(v[k].w, v[k].w, ss))));
    }
    const float inv = rsqrtf(block_sum(ss, scratch) / static_cast<float>(hidden) + eps);
    uint2* y = reinterpret_cast<uint2*>(xn + static_cast<int64_t>(t) * hidden);
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = threadIdx.x + k * kRowThreads;
      if (i < n4)
        y[i] = make_uint2(pack_bf16(v[k].x * inv * g[k].x, v[k].y * inv * g[k].y),
                          pack_bf16(v[k].z * inv * g[k].z, v[k].w * inv * g[k].w));
    }
  }
}

constexpr unsigned long long kTpSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s

template <int kVec>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_tp_kernel(float* resid, const float* parts, int64_t part_stride,
                                                                 int tp, const int* counter, uint32_t expected,
                                                                 const float* norm_w, __nv_bfloat16* xn, int hidden,
                                                                 float eps) {
  __shared__ float scratch[32];
  grid_dep_wait();
  if (threadIdx.x == 0) {
    // every rank's GEMM CTAs have stored their partials and signalled; a
    // peer that never signals (dead rank, mismatched launch) aborts the
    // kernel after kTpSpinTimeoutNs instead of hanging the GPU: __trap()
    // turns it into a launch failure the host reports.
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
      if (static_cast<int32_t>(v - expected) >= 0) break;
      __nanosleep(64);
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > kTpSpinTimeoutNs) __trap();
    }
  }
  __syncthreads();
  // Only now let the next kernel (the next GEMM, 1 CTA/SM) be scheduled: an
  // early launch would park it on the SMs the peer ranks' GEMMs need when
  // ranks share a GPU, and gains nothing while this grid waits on peers.
  grid_dep_launch();
  const int t = blockIdx.x;
  float4* x = reinterpret_cast<float4*>(resid + static_cast<int64_t>(t) * hidden);
  const float4* w = reinterpret_cast<const float4*>(norm_w);
  const int n4 = hidden / 4;
  float4 v[kVec];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < n4) {
      float4 a = x[i];
      for (int src = 0; src < tp; ++src) {  // fixed rank order: identical on every rank
        const float4 p = reinterpret_cast<const float4*>(parts + src * part_stride + static_cast<int64_t>(t) * hidden)[i];
        a.x += p.x;
        a.y += p.y;
        a.z += p.z;
        a.w += p.w;
      }
      x[i] = a;
      v[k] = a;
    } else {
      v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    ss = fmaf(v[k].x, v[k].x, fmaf(v[k].y, v[k].y, fmaf(v[k].z, v[k].z, fmaf(v[k].w, v[k].w, ss))));
  }
  const float inv = rsqrtf(block_sum(ss, scratch) / static_cast<float>(hidden) + eps);
  uint2* y = reinterpret_cast<uint2*>(xn + static_cast<int64_t>(t) * hidden);
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < n4) {
      const float4 g = w[i];
      y[i] = make_uint2(pack_bf16(v[k].x * inv * g.x, v[k].y * inv * g.y),
                        pack_bf16(v[k].z * inv * g.z, v[k].w * inv * g.w));
    }
  }
}

__global__ void __launch_bounds__(kRowThreads) argmax_kernel(const float* logits, int V, int32_t* out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  grid_dep_wait();
  grid_dep_launch();
  const float* row = logits + static_cast<int64_t>(blockIdx.x) * V;
  float best = -INFINITY;
  int bi = V;  // sentinel above any index; NaN logits never win
  auto take = [&](float v, int i) {
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  };
  if ((V & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    // 128-bit loads, kUnroll of them in flight per thread (a scalar loop
    // keeps one load in flight and is latency-bound: 63 us for 32000 logits)
    constexpr int kUnroll = 8;
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int n4 = V >> 2;
    for (int base = threadIdx.x; base < n4; base += kUnroll * kRowThreads) {
      float4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int j = base + u * kRowThreads;
        v[u] = j < n4 ? r4[j] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = 4 * (base + u * kRowThreads);
        take(v[u].x, i);
        take(v[u].y, i + 1);
        take(v[u].z, i + 2);
        take(v[u].w, i + 3);
      }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) take(row[i], i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[warp] = best;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float b0 = sv[0];
    int i0 = si[0];
    for (int w = 1; w < (blockDim.x >> 5); ++w)
      if (sv[w] > b0 || (sv[w] == b0 && si[w] < i0)) {
        b0 = sv[w];
        i0 = si[w];
      }
    out[blockIdx.x] = i0 < V ? i0 : 0;
  }
}

__global__ void gather_rows_kernel(const uint4* src, const int32_t* idx, uint4* dst, int vec_per_row) {
  grid_dep_wait();
  grid_dep_launch();
  const int r = blockIdx.x;
  const int64_t s = static_cast<int64_t>(idx[r]) * vec_per_row;
  const int64_t d = static_cast<int64_t>(r) * vec_per_row;
  for (int i = threadIdx.x; i < vec_per_row; i += blockDim.x) dst[d + i] = src[s + i];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void init_normal_kernel(__nv_bfloat16* dst, int64_t n, uint64_t seed, float std) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const uint64_t r = splitmix64(seed ^ splitmix64(static_cast<uint64_t>(i)));
    const float u1 = (static_cast<float>(r >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>((r >> 16) & 0xFFFFFF) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.f * __logf(u1)) * __cosf(6.28318530718f * u2);
    dst[i] = __float2bfloat16_rn(z * std);
  }
}

__global__ void fill_kernel(float* dst, int64_t n, float v) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) dst[i] = v;
}

}  // namespace

cudaError_t preload_fused_ops() {
  return preload(embed_rmsnorm_kernel, rmsnorm_rows_kernel<2>, rmsnorm_rows_kernel<4>, rmsnorm_rows_kernel<5>,
                 rmsnorm_rows_kernel<8>,
                 rmsnorm_rows_kernel<16>, rmsnorm_tp_kernel<2>, rmsnorm_tp_kernel<4>, rmsnorm_tp_kernel<8>,
                 rmsnorm_tp_kernel<16>, argmax_kernel, gather_rows_kernel, init_normal_kernel, fill_kernel);
}

cudaError_t embed_rmsnorm(const void* emb, const int32_t* tokens, const float* norm_w, float* resid,
                          void* xn, int T, int hidden, float eps, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  return launch(embed_rmsnorm_kernel, dim3(T), dim3(kRowThreads), 0, stream,
                reinterpret_cast<const __nv_bfloat16*>(emb), tokens, norm_w, resid,
                reinterpret_cast<__nv_bfloat16*>(xn), hidden, eps);
}

cudaError_t rmsnorm_rows(const float* resid, const float* norm_w, void* xn, int T, int hidden, float eps,
                         cudaStream_t stream, int max_ctas) {
  if (T <= 0) return cudaSuccess;
  if (hidden % 4 != 0 || hidden > 4 * kRowThreads * 16) return cudaErrorInvalidValue;
  __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(xn);
  const int per = (hidden / 4 + kRowThreads - 1) / kRowThreads;
  auto k = per <= 2 ? rmsnorm_rows_kernel<2> : per <= 4 ? rmsnorm_rows_kernel<4>
         : per <= 5 ? rmsnorm_rows_kernel<5> : per <= 8 ? rmsnorm_rows_kernel<8> : rmsnorm_rows_kernel<16>;
  static const int env_ctas = getenv("MUX_NORM_CTAS") ? atoi(getenv("MUX_NORM_CTAS")) : -1;  // debug override
  if (env_ctas >= 0) max_ctas = env_ctas;
  const int grid = max_ctas > 0 ? std::min(T, max_ctas) : T;
  return launch(k, dim3(grid), dim3(kRowThreads), 0, stream, resid, norm_w, y, T, hidden, eps);
}

cudaError_t rmsnorm_tp(float* resid, const float* parts, int64_t part_stride, int tp, const int* counter,
                       uint32_t expected, const float* norm_w, void* xn, int T, int hidden, float eps,
                       cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (hidden % 4 != 0 || hidden > 4 * kRowThreads * 16) return cudaErrorInvalidValue;
  __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(xn);
  const int per = (hidden / 4 + kRowThreads - 1) / kRowThreads;
  auto k = per <= 2 ? rmsnorm_tp_kernel<2> : per <= 4 ? rmsnorm_tp_kernel<4>
         : per <= 8 ? rmsnorm_tp_kernel<8> : rmsnorm_tp_kernel<16>;
  return launch(k, dim3(T), dim3(kRowThreads), 0, stream, resid, parts, part_stride, tp, counter, expected, norm_w, y,
                hidden, eps);
}

cudaError_t argmax_rows(const float* logits, int T, int V, int32_t* out, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  return launch(argmax_kernel, dim3(T), dim3(kRowThreads), 0, stream, logits, V, out);
}

cudaError_t gather_rows_bf16(const void* src, const int32_t* idx, void* dst, int n, int cols,
                             cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  return launch(gather_rows_kernel, dim3(n), dim3(128), 0, stream, reinterpret_cast<const uint4*>(src), idx,
                reinterpret_cast<uint4*>(dst), cols / 8);
}

cudaError_t init_normal_bf16(void* dst, int64_t n, uint64_t seed, float std, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  init_normal_kernel<<<148 * 8, 256, 0, stream>>>(reinterpret_cast<__nv_bfloat16*>(dst), n, seed, std);
  return cudaGetLastError();
}

cudaError_t fill_f32(float* dst, int64_t n, float v, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  fill_kernel<<<148 * 4, 256, 0, stream>>>(dst, n, v);
  return cudaGetLastError();
}

}  // namespace mux
