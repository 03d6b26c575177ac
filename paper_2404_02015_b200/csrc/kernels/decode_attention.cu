// K1: head-wise paged decode attention over the unified KV block pool.
//
// Work it replaces: the c_ctx * avg_context term of decode_step_latency
// (/root/reference/proj/src/cost_model.cpp:85-94), with context semantics
// ctx_i = prompt + 1 + steps_done (/root/reference/proj/src/scheduler.cpp:107)
// over head-blocks of block_tokens=16 x head_dim=128 bf16
// (/root/reference/proj/src/kv_manager.cpp:25-40).
//
// Data layout in HBM
//   pool    [n_blocks][16][128] bf16   one 4 KiB head-block = K or V of one
//                                      (layer, head) for 16 tokens
//   rowrec  [n_rowrec][L][H][2] int32  physical ids of one 16-token row
//   rowlist [slots][max_rows]   int32  row records of a request, in order
//
// One CTA = one (request, head, KV split). A producer warp resolves the row
// ids and streams K and V head-blocks with cp.async.bulk (4 KiB, one
// instruction each) into an S-stage shared-memory ring guarded by mbarriers;
// four consumer warps each take every fourth row and keep an online softmax
// (lane = 8 contiguous dims, half-warp = token parity, transposing butterfly
// reduction for q.k). Warps are merged through shared memory at the end.
// Algorithmic bytes per (request, head): ctx * 2 * 128 * 2 (K+V) + q + o.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace mux {
namespace {

constexpr int kDim = 128;
constexpr int kBlockTok = 16;
constexpr int kBlockBytes = kBlockTok * kDim * 2;  // 4096
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kMaxIdsPerSplit = 1024;  // rows handled by one CTA (16K tokens)

template <int S>
struct __align__(128) AttnSmem {
  uint8_t kv[S][2][kBlockBytes];
  uint64_t full[S];
  uint64_t empty[S];
  int2 ids[kMaxIdsPerSplit];
  float red_m[kConsumerWarps];
  float red_l[kConsumerWarps];
  float red_o[kConsumerWarps][kDim];
  int last;  // this CTA is the last split of its (member, head) to finish
};

template <int S, typename OutT>
__global__ void __launch_bounds__(kThreads)
decode_attention_kernel(const DecodeAttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  AttnSmem<S>& sm = *reinterpret_cast<AttnSmem<S>*>(smem_raw);

  const int split = blockIdx.x;
  const int h = blockIdx.y;
  // Longest-first order (host sorted by ctx) so the ragged tail is short.
  const int b = a.order != nullptr ? a.order[blockIdx.z] : blockIdx.z;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  const int ctx = a.ctx[b];
  const int nrows_total = (ctx + kBlockTok - 1) / kBlockTok;
  const int rps = a.rows_per_split_dev != nullptr ? *a.rows_per_split_dev : a.rows_per_split;
  const int r0 = split * rps;
  const int r1 = min(nrows_total, r0 + rps);
  const int n = max(0, r1 - r0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer warp: resolve ids, then stream K/V blocks.
    // The tables, contexts and every row but the one holding this step's
    // new token (written by the K2 launch just before) are fixed before the
    // job: the ids and the first S stages of older rows are issued before
    // the PDL dependency wait, overlapping the predecessor's tail.
    const int slot = a.slots[b];
    const int32_t* rl = a.rowlist + static_cast<int64_t>(slot) * a.max_rows;
    const int col = (a.layer * a.H + h) * 2;
    for (int i = lane; i < n; i += 32) {
      int rr = __ldg(rl + r0 + i);
      const int32_t* rec = a.rowrec + static_cast<int64_t>(rr) * a.row_width + col;
      sm.ids[i] = make_int2(__ldg(rec), __ldg(rec + 1));
    }
    __syncwarp();
    const int n_early = min(min(n, S), max(0, nrows_total - 1 - r0));
    const uint64_t pol = policy_evict_first();
    const uint8_t* pool = reinterpret_cast<const uint8_t*>(a.pool);
    // The request's last row holds only ctx - 16*(rows-1) valid tokens: copy
    // just those (256 B each); the consumers mask the rest by `valid` and
    // skip their V rows, so the stale smem tail is never used.
    const uint32_t last_bytes = static_cast<uint32_t>(ctx - (nrows_total - 1) * kBlockTok) * (kBlockBytes / kBlockTok);
    auto issue = [&](int i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&sm.empty[s], ((i / S) - 1) & 1);
      const int2 id = sm.ids[i];
      const uint32_t bytes = r0 + i == nrows_total - 1 ? last_bytes : kBlockBytes;
      mbar_arrive_expect_tx(&sm.full[s], 2 * bytes);
      bulk_g2s_stream(sm.kv[s][0], pool + static_cast<int64_t>(id.x) * kBlockBytes, bytes, &sm.full[s], pol);
      bulk_g2s_stream(sm.kv[s][1], pool + static_cast<int64_t>(id.y) * kBlockBytes, bytes, &sm.full[s], pol);
    };
    if (lane == 0)
      for (int i = 0; i < n_early; ++i) issue(i);
    grid_dep_wait();  // the new token's K/V (K2) and q
    grid_dep_launch();
    if (lane == 0)
      for (int i = n_early; i < n; ++i) issue(i);
    return;
  }
  grid_dep_wait();  // q comes from K2
  grid_dep_launch();

  // ---------------- consumer warps
  const int half = lane >> 4;  // token parity handled by this half-warp
  const int c = lane & 15;     // dims [8c, 8c+8)
  float q[8];
  {
    const uint4 v4 = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(a.q) +
                                                     (static_cast<int64_t>(b) * a.H + h) * kDim + c * 8);
    const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      q[2 * k] = bf16_lo(w[k]) * a.scale_log2;
      q[2 * k + 1] = bf16_hi(w[k]) * a.scale_log2;
    }
  }
  // Which token (within its parity) this lane's reduced score belongs to.
  const int jsel = (((c >> 3) & 1) << 2) | (((c >> 2) & 1) << 1) | ((c >> 1) & 1);

  float m_run = -INFINITY, l_run = 0.f;
  float acc[8];
#pragma unroll
  for (int d = 0; d < 8; ++d) acc[d] = 0.f;

  for (int i = warp; i < n; i += kConsumerWarps) {
    const int s = i % S;
    mbar_wait(&sm.full[s], (i / S) & 1);
    const uint8_t* kblk = sm.kv[s][0];
    const uint8_t* vblk = sm.kv[s][1];
    const int valid = min(kBlockTok, ctx - (r0 + i) * kBlockTok);

    // q . k for the 8 tokens of this lane's parity, 8 dims each.
    float part[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = 2 * j + half;
      const uint4 kv4 = *reinterpret_cast<const uint4*>(kblk + t * 256 + c * 16);
      const uint32_t w[4] = {kv4.x, kv4.y, kv4.z, kv4.w};
      float acc_s = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc_s = fmaf(q[2 * k], bf16_lo(w[k]), acc_s);
        acc_s = fmaf(q[2 * k + 1], bf16_hi(w[k]), acc_s);
      }
      part[j] = acc_s;
    }
    // Transposing butterfly over the 16 lanes of the half-warp: 8 values ->
    // one full dot product per lane (lanes c, c^1 hold the same token).
    {
      const bool lo8 = (c & 8) == 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float send = lo8 ? part[4 + k] : part[k];
        float keep = lo8 ? part[k] : part[4 + k];
        part[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
      const bool lo4 = (c & 4) == 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float send = lo4 ? part[2 + k] : part[k];
        float keep = lo4 ? part[k] : part[2 + k];
        part[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      const bool lo2 = (c & 2) == 0;
      {
        float send = lo2 ? part[1] : part[0];
        float keep = lo2 ? part[0] : part[1];
        part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
    }
    const int tok = 2 * jsel + half;
    const float score = tok < valid ? part[0] : -INFINITY;

    float m_blk = score;
    m_blk = fmaxf(m_blk, __shfl_xor_sync(0xffffffffu, m_blk, 16));
    m_blk = fmaxf(m_blk, __shfl_xor_sync(0xffffffffu, m_blk, 8));
    m_blk = fmaxf(m_blk, __shfl_xor_sync(0xffffffffu, m_blk, 4));
    m_blk = fmaxf(m_blk, __shfl_xor_sync(0xffffffffu, m_blk, 2));
    const float m_new = fmaxf(m_run, m_blk);
    const float alpha = exp2f(m_run - m_new);  // m_run=-inf -> 0
    const float p = tok < valid ? exp2f(score - m_new) : 0.f;
    float p_sum = p;
    p_sum += __shfl_xor_sync(0xffffffffu, p_sum, 16);
    p_sum += __shfl_xor_sync(0xffffffffu, p_sum, 8);
    p_sum += __shfl_xor_sync(0xffffffffu, p_sum, 4);
    p_sum += __shfl_xor_sync(0xffffffffu, p_sum, 2);
    l_run = l_run * alpha + p_sum;
    m_run = m_new;
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[d] *= alpha;

    // p . V for this lane's parity: fetch p of token 2j+half from its owner.
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int src = (half << 4) | (((j >> 2) & 1) << 3) | (((j >> 1) & 1) << 2) | ((j & 1) << 1);
      const float pj = __shfl_sync(0xffffffffu, p, src);
      if (pj != 0.f) {  // also skips never-written slots past `valid`
        const int t = 2 * j + half;
        const uint4 v4 = *reinterpret_cast<const uint4*>(vblk + t * 256 + c * 16);
        const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[2 * k] = fmaf(pj, bf16_lo(w[k]), acc[2 * k]);
          acc[2 * k + 1] = fmaf(pj, bf16_hi(w[k]), acc[2 * k + 1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
  }

  // Merge the two parities, then the four warps.
#pragma unroll
  for (int d = 0; d < 8; ++d) acc[d] += __shfl_xor_sync(0xffffffffu, acc[d], 16);
  if (lane < 16) {
#pragma unroll
    for (int d = 0; d < 8; ++d) sm.red_o[warp][c * 8 + d] = acc[d];
  }
  if (lane == 0) {
    sm.red_m[warp] = m_run;
    sm.red_l[warp] = l_run;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");

  const int d = threadIdx.x;  // 0..127
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, sm.red_m[w]);
  float L = 0.f, O = 0.f;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    const float f = sm.red_m[w] == -INFINITY ? 0.f : exp2f(sm.red_m[w] - M);
    L = fmaf(sm.red_l[w], f, L);
    O = fmaf(sm.red_o[w][d], f, O);
  }
  const int64_t bh = static_cast<int64_t>(b) * a.H + h;
  if (a.splits == 1) {
    const float val = L > 0.f ? O / L : 0.f;
    OutT* out = reinterpret_cast<OutT*>(a.out);
    if constexpr (sizeof(OutT) == 4) {
      out[bh * kDim + d] = val;
    } else {
      out[bh * kDim + d] = __float2bfloat16_rn(val);
    }
  } else {
    float* po = a.part_o + (bh * a.splits + split) * kDim;
    po[d] = L > 0.f ? O / L : 0.f;
    if (d == 0) {
      float* pml = a.part_ml + (bh * a.splits + split) * 2;
      pml[0] = M;
      pml[1] = L;
    }
    if (a.split_count != nullptr) {
      // The last split of this (member, head) to finish merges all of them
      // (threadfence-reduction pattern): no second launch on the critical path.
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
      if (d == 0) sm.last = atomicAdd(a.split_count + bh, 1) == a.splits - 1;
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
      if (sm.last) {
        __threadfence();
        const float* pml = a.part_ml + bh * a.splits * 2;
        float Mx = -INFINITY;
        for (int s2 = 0; s2 < a.splits; ++s2)
          if (__ldcg(pml + 2 * s2 + 1) > 0.f) Mx = fmaxf(Mx, __ldcg(pml + 2 * s2));
        float Lt = 0.f, Ot = 0.f;
        for (int s2 = 0; s2 < a.splits; ++s2) {
          const float l = __ldcg(pml + 2 * s2 + 1);
          if (l <= 0.f) continue;
          const float f = exp2f(__ldcg(pml + 2 * s2) - Mx) * l;
          Lt += f;
          Ot = fmaf(__ldcg(a.part_o + (bh * a.splits + s2) * kDim + d), f, Ot);
        }
        const float val = Lt > 0.f ? Ot / Lt : 0.f;
        OutT* out = reinterpret_cast<OutT*>(a.out);
        if constexpr (sizeof(OutT) == 4) {
          out[bh * kDim + d] = val;
        } else {
          out[bh * kDim + d] = __float2bfloat16_rn(val);
        }
        if (d == 0) a.split_count[bh] = 0;  // ready for the next launch
      }
    }
  }
}

// Merge KV splits: O = sum_s O_s L_s 2^(M_s - M) / sum_s L_s 2^(M_s - M).
template <typename OutT>
__global__ void __launch_bounds__(128) decode_attention_combine(const DecodeAttnArgs a) {
  grid_dep_wait();
  grid_dep_launch();
  const int64_t bh = blockIdx.x;
  const int d = threadIdx.x;
  const float* pml = a.part_ml + bh * a.splits * 2;
  float M = -INFINITY;
  for (int s = 0; s < a.splits; ++s)
    if (pml[2 * s + 1] > 0.f) M = fmaxf(M, pml[2 * s]);
  float L = 0.f, O = 0.f;
  for (int s = 0; s < a.splits; ++s) {
    const float l = pml[2 * s + 1];
    if (l <= 0.f) continue;
    const float f = exp2f(pml[2 * s] - M) * l;
    L += f;
    O = fmaf(a.part_o[(bh * a.splits + s) * kDim + d], f, O);
  }
  const float val = L > 0.f ? O / L : 0.f;
  OutT* out = reinterpret_cast<OutT*>(a.out);
  if constexpr (sizeof(OutT) == 4) {
    out[bh * kDim + d] = val;
  } else {
    out[bh * kDim + d] = __float2bfloat16_rn(val);
  }
}

template <int S, typename OutT>
cudaError_t launch_decode(const DecodeAttnArgs& a, cudaStream_t stream) {
  const size_t smem = sizeof(AttnSmem<S>);
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([&] {
    return cudaFuncSetAttribute(decode_attention_kernel<S, OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem));
  });
  if (ce != cudaSuccess) return ce;
  dim3 grid(a.splits, a.H, a.B);
  cudaError_t e = launch(decode_attention_kernel<S, OutT>, grid, dim3(kThreads), smem, stream, a);
  if (e == cudaSuccess && a.splits > 1 && a.split_count == nullptr)
    e = launch(decode_attention_combine<OutT>, dim3(a.B * a.H), dim3(128), 0, stream, a);
  return e;
}

}  // namespace

int decode_attention_max_rows_per_split() { return kMaxIdsPerSplit; }

cudaError_t preload_decode_attention() {
  cudaError_t e = preload(decode_attention_kernel<4, float>, decode_attention_kernel<4, __nv_bfloat16>,
                          decode_attention_combine<float>, decode_attention_combine<__nv_bfloat16>);
  // attributes set at unit creation: no first launch inside a graph capture
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(decode_attention_kernel<4, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(AttnSmem<4>)));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(decode_attention_kernel<4, __nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(sizeof(AttnSmem<4>)));
}

cudaError_t decode_attention(const DecodeAttnArgs& a, bool fp32_out, cudaStream_t stream) {
  if (a.B <= 0) return cudaSuccess;
  if (a.rows_per_split > kMaxIdsPerSplit || a.rows_per_split <= 0) return cudaErrorInvalidValue;
  if (fp32_out) return launch_decode<4, float>(a, stream);
  return launch_decode<4, __nv_bfloat16>(a, stream);
}

}  // namespace mux
