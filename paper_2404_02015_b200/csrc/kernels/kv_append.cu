// K2: KV append with block allocation.
//
// Replaces the device side of BlockPool::alloc(llm, rid, +1) / admit's prompt
// rows (/root/reference/proj/src/scheduler.cpp:105, kv_manager.cpp:87-120):
// the host pool decides which 4 KiB head-blocks a new 16-token row gets
// (csrc/host/kv.cpp), table_update scatters those ids into the device block
// tables, and kv_append writes each token's K (after RoPE) and V into slot
// pos % 16 of its (layer, head) blocks. One warp per (token, head); lane =
// 4 dims (8-byte loads/stores, 256 B per warp per block row).
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"
#include "launch.cuh"
#include "rope.cuh"

namespace mux {
namespace {

constexpr int kDim = 128;

__global__ void __launch_bounds__(256) kv_append_kernel(const AppendArgs a) {
  const int warp_global = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const bool active = warp_global < a.T * a.H;
  // Everything but the QKV output is fixed before this job's kernels run
  // (token positions / slots staged by the host, block tables by
  // table_update, the RoPE table): resolve the destination blocks and this
  // lane's (cos, sin) before the PDL dependency wait, so only the qkv read
  // sits between the QKV GEMM and the K/V stores.
  int t = 0, h = 0, pos = 0, kid = 0, vid = 0;
  float4 cs8[2] = {};
  if (active) {
    t = warp_global / a.H;
    h = warp_global - t * a.H;
    pos = a.tok_pos[t];
    const int slot = a.tok_slot[t];
    const int rr = a.rowlist[static_cast<int64_t>(slot) * a.max_rows + (pos >> 4)];
    const int32_t* rec = a.rowrec + static_cast<int64_t>(rr) * a.row_width + (a.layer * a.H + h) * 2;
    kid = rec[0];
    vid = rec[1];
    const float4* cs = reinterpret_cast<const float4*>(a.rope + static_cast<int64_t>(min(pos, a.rope_positions - 1)) * 128);
    const int f0 = (lane & 15) * 4;  // dims f0..f0+3 -> floats 2*f0 .. 2*f0+7
    cs8[0] = cs[f0 / 2];
    cs8[1] = cs[f0 / 2 + 1];
  }
  grid_dep_wait();
  grid_dep_launch();
  if (!active) return;

  const int64_t tok_base = static_cast<int64_t>(t) * 3 * a.H * kDim;
  const __nv_bfloat16* qkv = reinterpret_cast<const __nv_bfloat16*>(a.qkv);
  const uint2 qv = *reinterpret_cast<const uint2*>(qkv + tok_base + (0 * a.H + h) * kDim + lane * 4);
  const uint2 kv = *reinterpret_cast<const uint2*>(qkv + tok_base + (1 * a.H + h) * kDim + lane * 4);
  const uint2 vv = *reinterpret_cast<const uint2*>(qkv + tok_base + (2 * a.H + h) * kDim + lane * 4);
  float q[4], k[4];
  unpack4(qv, q);
  unpack4(kv, k);
  rope4_pre(q, cs8, lane);
  rope4_pre(k, cs8, lane);
  const uint2 kr = pack4(k);
  if (a.q_out != nullptr) {
    __nv_bfloat16* qo = reinterpret_cast<__nv_bfloat16*>(a.q_out);
    *reinterpret_cast<uint2*>(qo + (static_cast<int64_t>(t) * a.H + h) * kDim + lane * 4) = pack4(q);
    // Rotated k back in place too, for the prefill attention that reads it.
    __nv_bfloat16* qkv_w = const_cast<__nv_bfloat16*>(qkv);
    *reinterpret_cast<uint2*>(qkv_w + tok_base + (1 * a.H + h) * kDim + lane * 4) = kr;
  }
  uint8_t* pool = reinterpret_cast<uint8_t*>(a.pool);
  const int64_t off = static_cast<int64_t>(pos & 15) * 256 + lane * 8;
  *reinterpret_cast<uint2*>(pool + static_cast<int64_t>(kid) * 4096 + off) = kr;
  *reinterpret_cast<uint2*>(pool + static_cast<int64_t>(vid) * 4096 + off) = vv;
}

__global__ void __launch_bounds__(256) table_update_kernel(const TableUpdateArgs a) {
  grid_dep_wait();
  grid_dep_launch();
  const int i = blockIdx.x;
  const int slot = a.meta[3 * i + 0];
  const int row = a.meta[3 * i + 1];
  const int rec = a.meta[3 * i + 2];
  const int4* src = reinterpret_cast<const int4*>(a.ids + static_cast<int64_t>(i) * a.row_width);
  int32_t* dst32 = a.rowrec + static_cast<int64_t>(rec) * a.row_width;
  if ((a.row_width & 3) == 0) {
    int4* dst = reinterpret_cast<int4*>(dst32);
    for (int j = threadIdx.x; j < a.row_width / 4; j += blockDim.x) dst[j] = src[j];
  } else {
    const int32_t* s32 = a.ids + static_cast<int64_t>(i) * a.row_width;
    for (int j = threadIdx.x; j < a.row_width; j += blockDim.x) dst32[j] = s32[j];
  }
  if (threadIdx.x == 0) a.rowlist[static_cast<int64_t>(slot) * a.max_rows + row] = rec;
}

}  // namespace

cudaError_t preload_kv_append() { return preload(kv_append_kernel, table_update_kernel); }

cudaError_t kv_append(const AppendArgs& a, cudaStream_t stream) {
  if (a.T <= 0) return cudaSuccess;
  const int warps = a.T * a.H;
  const int blocks = (warps + 7) / 8;
  return launch(kv_append_kernel, dim3(blocks), dim3(256), 0, stream, a);
}

cudaError_t table_update(const TableUpdateArgs& a, cudaStream_t stream) {
  if (a.n <= 0) return cudaSuccess;
  return launch(table_update_kernel, dim3(a.n), dim3(256), 0, stream, a);
}

}  // namespace mux
