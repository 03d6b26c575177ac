// RoPE + bf16 packing helpers shared by K2 (kv_append.cu) and the fused
// decode layer chain (layer_chain.cu). One lane holds 4 consecutive dims of
// a 128-dim head; rotate_half partners live in lane ^ 16.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace mux {

static __device__ __forceinline__ void unpack4(uint2 v, float (&x)[4]) {
  x[0] = bf16_lo(v.x);
  x[1] = bf16_hi(v.x);
  x[2] = bf16_lo(v.y);
  x[3] = bf16_hi(v.y);
}

static __device__ __forceinline__ uint2 pack4(const float (&x)[4]) {
  return make_uint2(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]));
}

// rotate_half RoPE on 4 dims held by this lane; partner dims live in lane^16.
// Explicit _rn intrinsics: no FMA contraction, so the CPU oracle's float32
// arithmetic reproduces it bit for bit.
static __device__ __forceinline__ void rope4(float (&x)[4], const float* cs, int lane) {
  float other[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) other[k] = __shfl_xor_sync(0xffffffffu, x[k], 16);
  const int f0 = (lane & 15) * 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float c = cs[2 * (f0 + k)];
    const float s = cs[2 * (f0 + k) + 1];
    if (lane < 16) {
      x[k] = __fsub_rn(__fmul_rn(x[k], c), __fmul_rn(other[k], s));
    } else {
      x[k] = __fadd_rn(__fmul_rn(x[k], c), __fmul_rn(other[k], s));
    }
  }
}

// Same rotation with this lane's (cos, sin) pairs already in registers:
// cs8 = cs[2*f0 .. 2*f0+7], f0 = (lane & 15) * 4 (two 16-byte loads).
static __device__ __forceinline__ void rope4_pre(float (&x)[4], const float4 (&cs8)[2], int lane) {
  float other[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) other[k] = __shfl_xor_sync(0xffffffffu, x[k], 16);
  const float c[4] = {cs8[0].x, cs8[0].z, cs8[1].x, cs8[1].z};
  const float s[4] = {cs8[0].y, cs8[0].w, cs8[1].y, cs8[1].w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (lane < 16) {
      x[k] = __fsub_rn(__fmul_rn(x[k], c[k]), __fmul_rn(other[k], s[k]));
    } else {
      x[k] = __fadd_rn(__fmul_rn(x[k], c[k]), __fmul_rn(other[k], s[k]));
    }
  }
}

}  // namespace mux
