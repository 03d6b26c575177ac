// Fused decode layer chain: every projection of a decode layer between two
// attention launches, in ONE persistent tcgen05 kernel.
//
// Work it replaces: the decode_base term of decode_step_latency
// (/root/reference/proj/src/cost_model.cpp:85-94) -- the weight-streaming
// projections of a decode job -- plus the RMSNorm / SiLU / RoPE + KV-append
// element-wise steps between them (K2 and K5).
//
// A decode GEMM (M = batch <= 256 tokens) is a pure weight stream: the
// weights (HBM) never depend on the previous step, only the activations
// (L2-resident) do. As separate launches every projection pays a launch /
// pipeline-fill head and an epilogue tail with the SMs' HBM streams idle.
// Here one CTA per SM streams the weights of all jobs back to back through
// its ring -- the producer warp runs ahead into the next projection while
// the current one finishes -- and only the activation (B) loads and MMAs
// wait for the data dependency, a grid barrier per step.
//
// Jobs (the standard decode layer, one launch per layer):
//   o      : resid  += attn  Wo^T      then norm:  xn = rmsnorm(resid) * ffn_norm
//   gu     : gu32   += xn    Wgu^T     then silu:  act = SiLU(gate) * up, gu32 = 0
//   down   : resid  += act   Wdown^T   then norm:  xn = rmsnorm(resid) * next attn_norm
//   qkv    : qkv32  += xn    Wqkv^T    then rope:  q = RoPE(q), K/V -> head-blocks, qkv32 = 0
// Every job's epilogue is a TMA fp32 reduce-add of the persistent stream-K
// pieces (no fixups, no partner waits); the non-linear step runs after the
// grid barrier that follows the job, spread over all CTAs' epilogue warps.
// Numerics match the separate kernels: the fp32 sums are rounded to bf16
// exactly where the unfused path rounds them (qkv before RoPE, act, xn).
//
// Co-residency of all CTAs (grid = the partition's SMs, 1 CTA/SM) is
// required by the grid barriers and guaranteed by a cooperative launch.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"
#include "rope.cuh"

namespace mux {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kAStageBytes = kBM * kBK * 2;
constexpr int kThreads = 256;
constexpr int kEpiThreads = 128;
constexpr int kChunkBytes = 32 * kBM * 4;
constexpr int kSmemBudget = 224 * 1024;

unsigned long long* g_chain_timing = nullptr;

struct ChainRunDev {
  int n_jobs;
  ChainJob job[kChainMaxJobs];
  int M, n_tile, stages_a, stages_b;
  uint32_t tmem_cols;
  unsigned* bar;
  unsigned bar_base;
  ChainPost post;
  unsigned long long* timing;  // debug: [grid][64] globaltimer stamps, or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define STAMP(cond, slot) \
  do { if (r.timing != nullptr && (cond)) r.timing[blockIdx.x * 64 + (slot)] = gtimer(); } while (0)

struct ChainMaps {
  CUtensorMap x[kChainMaxJobs];
  CUtensorMap out[kChainMaxJobs];
};

__device__ __forceinline__ int64_t range_begin(int64_t iters, int c, int grid) { return iters * c / grid; }

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

__device__ __forceinline__ void bar_arrive(unsigned* bar) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

__device__ __forceinline__ void bar_wait(const unsigned* bar, unsigned target) {
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    if (static_cast<int>(v - target) >= 0) break;
    __nanosleep(20);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// ---- element-wise steps between jobs (128 epilogue threads of every CTA) --

// The element-wise steps run on one warp per SM sub-partition, so they are
// written for memory-level parallelism: every thread issues all of its loads
// for an iteration before using any of them.

// xn[r] = bf16(resid[r] * rsqrt(mean(resid[r]^2) + eps) * w), rows c, c+G, ...
// (hidden <= 8192: at most 16 float4 per thread, all in flight at once)
__device__ void post_norm(const ChainPost& p, const float* w, int c, int G, int M, float* red) {
  const int t = threadIdx.x - 128;
  const int n4 = p.hidden / 4;
  const float4* wv = reinterpret_cast<const float4*>(w);
  for (int r = c; r < M; r += G) {
    const float4* x = reinterpret_cast<const float4*>(p.resid + static_cast<int64_t>(r) * p.hidden);
    float4 v[16], g[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = t + k * kEpiThreads;
      v[k] = i < n4 ? x[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      g[k] = i < n4 ? wv[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      ss = fmaf(v[k].x, v[k].x, fmaf(v[k].y, v[k].y, fmaf(v[k].z, v[k].z, fmaf(v[k].w, v[k].w, ss))));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((t & 31) == 0) red[t >> 5] = ss;
    epi_bar();
    const float tot = red[0] + red[1] + red[2] + red[3];
    epi_bar();
    const float inv = rsqrtf(tot / static_cast<float>(p.hidden) + p.eps);
    uint2* y = reinterpret_cast<uint2*>(p.xn + static_cast<int64_t>(r) * p.hidden);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int i = t + k * kEpiThreads;
      if (i < n4)
        y[i] = make_uint2(pack_bf16(v[k].x * inv * g[k].x, v[k].y * inv * g[k].y),
                          pack_bf16(v[k].z * inv * g[k].z, v[k].w * inv * g[k].w));
    }
  }
}

// act = bf16(SiLU(bf16(gate)) * bf16(up)) from the interleaved fp32 sums
// (gate_i, up_i) -- the unfused path rounds the GEMM output to bf16 first --
// then zero gu32 for the next layer's reduce-add. 8 float4 per thread in flight.
__device__ void post_silu(const ChainPost& p, int c, int G, int M) {
  constexpr int kU = 16;
  const int t = threadIdx.x - 128;
  const int64_t n = static_cast<int64_t>(M) * p.ffn / 2;  // float4 = 2 (gate, up) pairs
  const int64_t stride = static_cast<int64_t>(G) * kEpiThreads;
  float4* gu = reinterpret_cast<float4*>(p.gu32);
  uint32_t* act = reinterpret_cast<uint32_t*>(p.act);
  for (int64_t e0 = static_cast<int64_t>(c) * kEpiThreads + t; e0 < n; e0 += stride * kU) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = e0 + u * stride;
      v[u] = e < n ? gu[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < n) {
        gu[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float g0 = bf16_round(v[u].x), u0 = bf16_round(v[u].y), g1 = bf16_round(v[u].z), u1 = bf16_round(v[u].w);
        const float s0 = g0 / (1.f + expf(-g0));
        const float s1 = g1 / (1.f + expf(-g1));
        act[e] = pack_bf16(s0 * u0, s1 * u1);
      }
    }
  }
}

// K2 fused: per (member, head) warp task -- round the fp32 q/k/v sums to bf16
// (as the unfused QKV GEMM stores them), RoPE q and k, write rotated q and the
// new token's K/V into slot pos % 16 of the (layer, head) head-blocks.
// 4 tasks per warp in flight (their q/k/v loads and block-table lookups).
__device__ void post_qkv_append(const ChainPost& p, int c, int G, int M) {
  constexpr int kU = 4;
  const int lane = threadIdx.x & 31;
  const int w = (threadIdx.x >> 5) - 4;
  const int H = p.heads;
  const int64_t tasks = static_cast<int64_t>(M) * H;
  const int64_t stride = static_cast<int64_t>(G) * 4;
  for (int64_t t0 = static_cast<int64_t>(c) * 4 + w; t0 < tasks; t0 += stride * kU) {
    float4 qa[kU], ka[kU], va[kU];
    int kid[kU], vid[kU], pos[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t task = t0 + u * stride;
      if (task < tasks) {
        const int t = static_cast<int>(task / H), h = static_cast<int>(task % H);
        const float* base = p.qkv32 + static_cast<int64_t>(t) * 3 * H * 128;
        qa[u] = reinterpret_cast<const float4*>(base + (0 * H + h) * 128)[lane];
        ka[u] = reinterpret_cast<const float4*>(base + (1 * H + h) * 128)[lane];
        va[u] = reinterpret_cast<const float4*>(base + (2 * H + h) * 128)[lane];
        pos[u] = p.ctx[t] - 1;
        const int rr = p.rowlist[static_cast<int64_t>(p.slots[t]) * p.max_rows + (pos[u] >> 4)];
        const int32_t* rec = p.rowrec + static_cast<int64_t>(rr) * p.row_width + (p.layer * H + h) * 2;
        kid[u] = rec[0];
        vid[u] = rec[1];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t task = t0 + u * stride;
      if (task >= tasks) continue;
      const int t = static_cast<int>(task / H), h = static_cast<int>(task % H);
      float* base = p.qkv32 + static_cast<int64_t>(t) * 3 * H * 128;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(base + (0 * H + h) * 128)[lane] = z;
      reinterpret_cast<float4*>(base + (1 * H + h) * 128)[lane] = z;
      reinterpret_cast<float4*>(base + (2 * H + h) * 128)[lane] = z;
      float q[4] = {bf16_round(qa[u].x), bf16_round(qa[u].y), bf16_round(qa[u].z), bf16_round(qa[u].w)};
      float k[4] = {bf16_round(ka[u].x), bf16_round(ka[u].y), bf16_round(ka[u].z), bf16_round(ka[u].w)};
      const float v[4] = {va[u].x, va[u].y, va[u].z, va[u].w};
      const float* cs = p.rope + static_cast<int64_t>(min(pos[u], p.rope_positions - 1)) * 128;
      rope4(q, cs, lane);
      rope4(k, cs, lane);
      *reinterpret_cast<uint2*>(p.q + (static_cast<int64_t>(t) * H + h) * 128 + lane * 4) = pack4(q);
      uint8_t* pool = reinterpret_cast<uint8_t*>(p.pool);
      const int64_t off = static_cast<int64_t>(pos[u] & 15) * 256 + lane * 8;
      *reinterpret_cast<uint2*>(pool + static_cast<int64_t>(kid[u]) * 4096 + off) = pack4(k);
      *reinterpret_cast<uint2*>(pool + static_cast<int64_t>(vid[u]) * 4096 + off) = pack4(v);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
layer_chain_kernel(const __grid_constant__ ChainMaps maps, const ChainRunDev r) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int SA = r.stages_a, SB = r.stages_b;
  const int b_stage_bytes = r.n_tile * kBK * 2;
  uint8_t* a_st = base;
  uint8_t* b_st = base + SA * kAStageBytes;
  uint8_t* stage_out = b_st + SB * b_stage_bytes;
  uint64_t* full_a = reinterpret_cast<uint64_t*>(stage_out + 2 * kChunkBytes);
  uint64_t* empty_a = full_a + SA;
  uint64_t* full_b = empty_a + SA;
  uint64_t* empty_b = full_b + SB;
  uint64_t* tm_full = empty_b + SB;  // [2]
  uint64_t* tm_empty = tm_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int G = gridDim.x;
  // barrier k of this launch completes when all G CTAs arrived k+1 times
  auto target = [&](int k) { return r.bar_base + static_cast<unsigned>(k + 1) * static_cast<unsigned>(G); };

  if (warp == 0 && lane == 0) {
    for (int j = 0; j < r.n_jobs; ++j) {
      prefetch_tmap(&maps.x[j]);
      prefetch_tmap(&maps.out[j]);
    }
    for (int s = 0; s < SA; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&empty_a[s], 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tm_full[b], 1);
      mbar_init(&tm_empty[b], kEpiThreads / 32);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_dyn(tmem_slot, r.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- weight producer: every job's tiles, back to back.
    // Besides the smem ring it keeps an L2 prefetch window kPrefetch tiles
    // ahead (crossing into the next jobs): while the consumers sit in a grid
    // barrier or an element-wise step, HBM keeps streaming weights into L2.
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      constexpr int kPrefetch = 24;  // tiles (384 KiB per SM, ~57 MB over 148 SMs)
      // prefetch cursor: (job, tile index within this CTA's range)
      int pj = 0;
      int64_t pit = range_begin(r.job[0].iters, c, G);
      int64_t pend = range_begin(r.job[0].iters, c + 1, G);  // divisions only on job switches
      auto prefetch_next = [&]() {
        while (pj < r.n_jobs && pit >= pend) {
          if (++pj < r.n_jobs) {
            pit = range_begin(r.job[pj].iters, c, G);
            pend = range_begin(r.job[pj].iters, c + 1, G);
          }
        }
        if (pj >= r.n_jobs) return;
        const ChainJob& pb = r.job[pj];
        // contiguous tiles (m, kbi) -> offset it * 16 KiB (tiles are [m][kb] contiguous)
        prefetch_l2(pb.w + pit * kAStageBytes, kAStageBytes);
        ++pit;
      };
      for (int k = 0; k < kPrefetch; ++k) prefetch_next();
      int s = 0, round = 0;
      for (int j = 0; j < r.n_jobs; ++j) {
        STAMP(true, j * 8 + 6);
        const ChainJob& jb = r.job[j];
        const int64_t it0 = range_begin(jb.iters, c, G), it1 = range_begin(jb.iters, c + 1, G);
        for (int64_t it = it0; it < it1; ++it) {
          if (round > 0) mbar_wait(&empty_a[s], (round - 1) & 1);
          mbar_arrive_expect_tx(&full_a[s], kAStageBytes);
          // tile `it` of the flattened [m][kb] space is stored contiguously
          bulk_g2s_stream(a_st + s * kAStageBytes, jb.w + it * kAStageBytes, kAStageBytes, &full_a[s], pol);
          prefetch_next();
          if (++s == SA) {
            s = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == 3) {
    // ---------------- activation producer: job j waits for its input
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();
      const uint32_t bytes = static_cast<uint32_t>(b_stage_bytes);
      grid_dep_wait();  // job 0's input (attention output) comes from the previous kernel
      int s = 0, round = 0;
      for (int j = 0; j < r.n_jobs; ++j) {
        if (j > 0) bar_wait(r.bar, target(2 * j - 1));  // job j-1 and its element-wise step done
        STAMP(true, j * 8 + 0);
        const ChainJob& jb = r.job[j];
        const int64_t it0 = range_begin(jb.iters, c, G), it1 = range_begin(jb.iters, c + 1, G);
        int kbi = static_cast<int>(it0 % jb.kb);
        for (int64_t it = it0; it < it1; ++it) {
          if (round > 0) mbar_wait(&empty_b[s], (round - 1) & 1);
          mbar_arrive_expect_tx(&full_b[s], bytes);
          tma_load_2d(b_st + s * b_stage_bytes, &maps.x[j], &full_b[s], kbi * kBK, 0, pol);
          if (++s == SB) {
            s = 0;
            ++round;
          }
          if (++kbi == jb.kb) kbi = 0;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = umma_idesc_bf16(kBM, r.n_tile);
    int seg = 0, sa = 0, ra = 0, sb = 0, rb = 0;
    for (int j = 0; j < r.n_jobs; ++j) {
      const ChainJob& jb = r.job[j];
      int64_t it = range_begin(jb.iters, c, G);
      const int64_t it1 = range_begin(jb.iters, c + 1, G);
      while (it < it1) {
        const int64_t t = it / jb.kb;
        const int64_t seg_begin = it;
        const int64_t seg_end = min(it1, (t + 1) * jb.kb);
        const int b = seg & 1;
        if (seg >= 2) mbar_wait(&tm_empty[b], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(b * r.n_tile);
        for (; it < seg_end; ++it) {
          mbar_wait(&full_a[sa], ra & 1);
          mbar_wait(&full_b[sb], rb & 1);
          STAMP(lane == 0 && it == range_begin(jb.iters, c, G), j * 8 + 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(a_st + sa * kAStageBytes);
            const uint32_t b_addr = smem_u32(b_st + sb * b_stage_bytes);
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(acc, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                        (it != seg_begin || kk != 0) ? 1u : 0u);
            umma_commit(&empty_a[sa]);
            umma_commit(&empty_b[sb]);
            if (it == seg_end - 1) umma_commit(&tm_full[b]);
          }
          __syncwarp();
          if (++sa == SA) {
            sa = 0;
            ++ra;
          }
          if (++sb == SB) {
            sb = 0;
            ++rb;
          }
        }
        ++seg;
      }
      STAMP(lane == 0, j * 8 + 2);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: reduce-add pieces, barrier, element-wise step, barrier
    const int q = warp - 4;
    const int etid = threadIdx.x - 128;
    const int fl = q * 32 + lane;
    const bool leader = etid == 0;
    int seg = 0, sbuf = 0;
    grid_dep_wait();  // outputs (resid, gu32, qkv32) are read by the previous kernels
    for (int j = 0; j < r.n_jobs; ++j) {
      const ChainJob& jb = r.job[j];
      int64_t it = range_begin(jb.iters, c, G);
      const int64_t it1 = range_begin(jb.iters, c + 1, G);
      const int nchunk = (r.M + 31) / 32;
      while (it < it1) {
        const int64_t t = it / jb.kb;
        const int64_t seg_end = min(it1, (t + 1) * jb.kb);
        const int b = seg & 1;
        const int m = static_cast<int>(t);
        mbar_wait(&tm_full[b], (seg >> 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * r.n_tile);
        for (int k = 0; k < nchunk; ++k) {
          float v[32];
          tmem_ld_32x32b_x32(acc + k * 32, v);
          if (k == nchunk - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tm_empty[b]);
          }
          if (leader) bulk_wait_read<1>();
          epi_bar();
          float* sf = reinterpret_cast<float*>(stage_out + sbuf * kChunkBytes);
#pragma unroll
          for (int i = 0; i < 32; ++i) sf[i * kBM + fl] = v[i];
          fence_async_smem();
          epi_bar();
          if (leader) {
            tma_reduce_add_2d(&maps.out[j], sf, m * kBM, k * 32);  // rows >= M are clipped
            bulk_commit();
          }
          sbuf ^= 1;
        }
        it = seg_end;
        ++seg;
      }
      // barrier 2j: every CTA's pieces of job j have landed
      if (leader) {
        STAMP(true, j * 8 + 3);
        bulk_wait<0>();
        bar_arrive(r.bar);
        bar_wait(r.bar, target(2 * j));
        STAMP(true, j * 8 + 4);
      }
      epi_bar();
      const int post = jb.post;
      if (post == kPostNorm) {
        post_norm(r.post, jb.norm_w, c, G, r.M, red);
      } else if (post == kPostSilu) {
        post_silu(r.post, c, G, r.M);
      } else if (post == kPostQkvAppend) {
        post_qkv_append(r.post, c, G, r.M);
      }
      // barrier 2j+1: the element-wise step is complete everywhere
      epi_bar();
      STAMP(leader, j * 8 + 5);
      if (leader) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        bar_arrive(r.bar);
      }
    }
    if (leader) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) grid_dep_launch();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, r.tmem_cols);
  }
}

bool g_coop_pdl_ok = true;  // cooperative + PDL attributes accepted together?

}  // namespace

void chain_debug_timing(void* buf) { g_chain_timing = static_cast<unsigned long long*>(buf); }
bool chain_coop_pdl() { return g_coop_pdl_ok; }

cudaError_t preload_layer_chain() { return preload(layer_chain_kernel); }

cudaError_t layer_chain(const ChainArgs& a, cudaStream_t stream) {
  if (a.n_jobs <= 0 || a.n_jobs > kChainMaxJobs || a.M <= 0 || a.M > 256) return cudaErrorInvalidValue;
  ChainRunDev r{};
  r.n_jobs = a.n_jobs;
  r.M = a.M;
  r.n_tile = gemm_pick_n_tile(a.M);
  const int b_stage = r.n_tile * kBK * 2;
  r.stages_b = r.n_tile > 128 ? 2 : 3;
  r.stages_a = std::min(10, (kSmemBudget - r.stages_b * b_stage - 2 * kChunkBytes) / kAStageBytes);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * r.n_tile)) cols <<= 1;
  r.tmem_cols = cols;
  r.bar = a.bar;
  r.bar_base = a.bar_base;
  r.post = a.post;
  r.timing = g_chain_timing;
  ChainMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  for (int j = 0; j < a.n_jobs; ++j) {
    ChainJob jb = a.job[j];
    jb.kb = (jb.K + kBK - 1) / kBK;
    jb.m_tiles = (jb.N + kBM - 1) / kBM;
    jb.iters = static_cast<int64_t>(jb.m_tiles) * jb.kb;
    r.job[j] = jb;
    std::memcpy(&maps.x[j], a.tmap_x[j], sizeof(CUtensorMap));
    std::memcpy(&maps.out[j], a.tmap_out[j], sizeof(CUtensorMap));
  }
  const size_t smem = 1024 + static_cast<size_t>(r.stages_a) * kAStageBytes + static_cast<size_t>(r.stages_b) * b_stage +
                      2 * kChunkBytes + (2 * (r.stages_a + r.stages_b) + 4) * 8 + 16 + 64;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(layer_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && g_coop_pdl_ok) ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, layer_chain_kernel, maps, r);
  if (e != cudaSuccess && cfg.numAttrs == 2) {
    (void)cudaGetLastError();
    g_coop_pdl_ok = false;  // this driver refuses cooperative + PDL: cooperative alone
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, layer_chain_kernel, maps, r);
  }
  return e;
}

}  // namespace mux
