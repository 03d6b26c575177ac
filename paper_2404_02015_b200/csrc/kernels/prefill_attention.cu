// K3: causal varlen prefill attention on the 5th-generation tensor cores.
//
// Work it replaces: the attention part of prefill_latency
// (/root/reference/proj/src/cost_model.cpp:75-83) -- causal softmax(q k^T /
// sqrt(128)) v over every prompt of a prefill job, head_dim 128, after
// kv_append has rotated q and k (RoPE) and written k/v into the head-blocks
// (the K/V read here are the same bytes, straight from the QKV GEMM output).
//
// One CTA = (128-query tile of one sequence, head). Flash-attention over
// 128-key tiles with both contractions on tcgen05:
//   S_j = Q K_j^T      UMMA 128x128x128, A = Q (smem, K-major), B = K_j (smem,
//                      K-major), fp32 accumulator in TMEM (double-buffered so
//                      S_{j+1} is computed while the softmax reads S_j)
//   O_j = P_j V_j      UMMA 128x128x128, A = P_j (bf16, written to smem by the
//                      softmax in the canonical SW128 K-major image), B = V_j
//                      (smem, MN-major: the same TMA box as K, other descriptor)
// Warp 8 = TMA producer + MMA issuer (one elected lane); warps 0-7 = softmax,
// two warps per TMEM lane quarter, a thread owns half (64 keys / 64 output
// dims) of one query row: online max/sum in fp32, causal + sequence-end
// masking. The output accumulates in TMEM across key tiles; when
// a row's max moves, its O row is rescaled in place (tcgen05.ld/st) before
// the next P V is issued.
// K/V tiles stream through a 2-stage TMA ring (SWIZZLE_128B boxes of 64 dims
// x 128 tokens over the [T][3][H][128] QKV buffer).
// FLOPs per (sequence of length n, head): 4 * 128 * n * (n + 1) / 2 (causal).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace mux {
namespace {

constexpr int kTile = 128;                   // queries per CTA, keys per KV tile
constexpr int kHalfBytes = kTile * 64 * 2;   // one 64-dim SW128 half of a tile: 16 KiB
constexpr int kTileBytes = 2 * kHalfBytes;   // 128 x 128 bf16
constexpr int kStages = 2;
constexpr int kSoftmaxWarps = 8;             // 2 per TMEM lane quarter: each owns 64 of a row's 128 keys
constexpr int kThreads = (kSoftmaxWarps + 1) * 32;  // + 1 TMA/MMA warp
constexpr uint32_t kTmemCols = 512;          // S0 [0,128) S1 [128,256) O [256,384)
constexpr size_t kSmemBytes = 1024 + kTileBytes /*Q*/ + kStages * 2 * kTileBytes /*K,V*/ +
                              kTileBytes /*P*/ + 256 /*barriers*/ + 4 * 2 * 128 * 4 /*row exchange*/;

struct Bars {
  uint64_t q_full;
  uint64_t k_full[kStages];
  uint64_t k_empty[kStages];
  uint64_t v_full[kStages];
  uint64_t v_empty[kStages];
  uint64_t s_full[2];
  uint64_t s_empty[2];
  uint64_t p_full;
  uint64_t o_full;
  uint64_t q_empty;  // persistent: the item's last Q K^T done, Q buffer reusable
  uint64_t o_empty;  // persistent: the softmax warps have read the item's O
  uint32_t tmem;
  uint32_t pad[3];
  float mx[2][2][128];  // [tile parity][key half][row]: partial row maxima
  float ls[2][128];     // [key half][row]: partial row sums (end)
};

// MN-major SW128 descriptor (B = V: N = head dims contiguous, K = keys):
// 8-key groups 1024 B apart (SBO), the second 64-dim half 16 KiB away (LBO).
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(kHalfBytes >> 4) << 16;  // LBO: next 64-wide MN atom column
  d |= static_cast<uint64_t>(1024 >> 4) << 32;        // SBO: next 8-row group along K
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Item of round r for CTA c: rounds alternate direction (snake) over the
// heaviest-first item list, so every CTA gets a mix of long and short causal
// rows instead of the c-th heaviest of every round.
__device__ __forceinline__ int snake_item(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }

__global__ void __launch_bounds__(kThreads, 1)
prefill_attention_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                         const PrefillAttnArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];  // aligned below (a 1 KiB-aligned declaration costs 1 KiB of static smem)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* q_s = base;
  uint8_t* kv_s = q_s + kTileBytes;                 // [stage][K|V][2 halves]
  uint8_t* p_s = kv_s + kStages * 2 * kTileBytes;   // [2 halves][128 rows][128 B]
  Bars& bar = *reinterpret_cast<Bars*>(p_s + kTileBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent: CTA c takes one work item per round in snake order over the
  // heaviest-first list (item = tile index * H + head). TMEM, barriers and the pipeline
  // counters live across items; the next item's Q / K_0 / V_0 loads and its
  // first Q K^T overlap the current item's last P V and epilogue.
  const int n_items = a.n_tiles * a.H;

  if (threadIdx.x == 0) {
    mbar_init(&bar.q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar.s_full[s], 1);
      mbar_init(&bar.s_empty[s], kSoftmaxWarps);
    }
    mbar_init(&bar.p_full, kSoftmaxWarps);
    mbar_init(&bar.o_full, 1);
    mbar_init(&bar.q_empty, 1);
    mbar_init(&bar.o_empty, kSoftmaxWarps);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kTmemCols>(&bar.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  grid_dep_wait();  // q / k / v come from kv_append and the QKV GEMM
  if (threadIdx.x == 0) grid_dep_launch();
  const uint32_t tmem = bar.tmem;

  if (warp == kSoftmaxWarps) {
    if (elect_one()) {
      // ---------------- TMA producer + MMA issuer
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();  // re-read by the other q tiles of this head
      const uint32_t idesc_qk = umma_idesc_bf16(kTile, kTile);
      const uint32_t idesc_pv = umma_idesc_bf16(kTile, 128) | (1u << 16);  // B (V) MN-major
      const uint32_t q_addr = smem_u32(q_s), p_addr = smem_u32(p_s);
      int jg = 0;  // key tiles issued by this CTA before the current item (global ring / buffer counter)
      int it = 0;
      for (int round = 0;; ++round, ++it) {
        const int item = snake_item(round, blockIdx.x, gridDim.x);
        if (item >= n_items) break;
        const int h = item % a.H;
        const int tile = a.tiles[item / a.H];
        const int seq = tile >> 16, qt = tile & 0xFFFF;
        const int s0 = a.seq_start[seq];
        const int q0 = qt * kTile;
        const int n_kv = qt + 1;  // causal: key tiles 0..qt
        if (it > 0) mbar_wait(&bar.q_empty, (it - 1) & 1);  // the previous item's Q K^T are done
        mbar_arrive_expect_tx(&bar.q_full, kTileBytes);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(q_s + hh * kHalfBytes, &tq, &bar.q_full, h * 128 + hh * 64, s0 + q0, pol_q);
        // K and V of a tile have separate ring slots and barriers: K_j's slot
        // frees when S_j = Q K_j^T completes (early), V_j's when P_j V_j does,
        // so the next K load never waits behind a P V. g = global tile index.
        auto load_k = [&](int j) {
          const int g = jg + j, st = g % kStages;
          if (g >= kStages) mbar_wait(&bar.k_empty[st], ((g / kStages) - 1) & 1);
          uint8_t* dst = kv_s + st * 2 * kTileBytes;
          mbar_arrive_expect_tx(&bar.k_full[st], kTileBytes);
          for (int hh = 0; hh < 2; ++hh)
            tma_load_2d(dst + hh * kHalfBytes, &tkv, &bar.k_full[st], (a.H + h) * 128 + hh * 64, s0 + j * kTile, pol_kv);
        };
        auto load_v = [&](int j) {
          const int g = jg + j, st = g % kStages;
          if (g >= kStages) mbar_wait(&bar.v_empty[st], ((g / kStages) - 1) & 1);
          uint8_t* dst = kv_s + st * 2 * kTileBytes + kTileBytes;
          mbar_arrive_expect_tx(&bar.v_full[st], kTileBytes);
          for (int hh = 0; hh < 2; ++hh)
            tma_load_2d(dst + hh * kHalfBytes, &tkv, &bar.v_full[st], (2 * a.H + h) * 128 + hh * 64, s0 + j * kTile,
                        pol_kv);
        };
        auto issue_qk = [&](int j) {
          const int g = jg + j, st = g % kStages, sb = g & 1;
          mbar_wait(&bar.k_full[st], (g / kStages) & 1);
          if (g >= 2) mbar_wait(&bar.s_empty[sb], ((g >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(kv_s + st * 2 * kTileBytes);
  #pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
            umma_bf16(tmem + sb * kTile, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_qk,
                      kk > 0 ? 1u : 0u);
          }
          umma_commit(&bar.s_full[sb]);
          umma_commit(&bar.k_empty[st]);
        };
        load_k(0);
        load_v(0);
        if (n_kv > 1) {
          load_k(1);
          load_v(1);
        }
        mbar_wait(&bar.q_full, it & 1);
        issue_qk(0);
        for (int j = 0; j < n_kv; ++j) {
          const int g = jg + j;
          if (j + 1 < n_kv) issue_qk(j + 1);
          if (j + 1 == n_kv) umma_commit(&bar.q_empty);  // fires once this item's last Q K^T is done
          // K_{j+2} goes into S_j's K slot as soon as S_j is done (issued one
          // iteration ago): a full iteration ahead of Q K_{j+2}^T.
          if (j + kStages < n_kv) load_k(j + kStages);
          if (j + 1 < n_kv && j + 1 >= kStages) load_v(j + 1);  // waits for P_{j-1} V_{j-1}
          // the previous item's O must have been read before P_0 V_0 overwrites it
          if (j == 0 && it > 0) mbar_wait(&bar.o_empty, (it - 1) & 1);
          // O_j = P_j V_j once the softmax has written P_j
          mbar_wait(&bar.p_full, g & 1);
          const int st = g % kStages;
          mbar_wait(&bar.v_full[st], (g / kStages) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(kv_s + st * 2 * kTileBytes + kTileBytes);
  #pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            umma_bf16(tmem + 2 * kTile, umma_desc_sw128(p_addr + (kk >> 2) * kHalfBytes + (kk & 3) * 32),
                      umma_desc_sw128_mn(v_addr + kk * 2048), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&bar.o_full);
          umma_commit(&bar.v_empty[st]);
        }
        jg += n_kv;
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps: thread = (query row, key half)
    // Warps w and w+4 share TMEM lane quarter w%4 (rows 32*(w%4)..+31) and
    // split the 128 keys of a tile (and the 128 output dims) in halves; the
    // row max is exchanged through smem once per tile (double-buffered by
    // tile parity, so one barrier per tile), the row sums once at the end.
    const int quarter = warp & 3, hf = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    uint8_t* p_row = p_s + hf * kHalfBytes + row * 128;
    const uint32_t o_addr = tmem + lane_base + 2 * kTile + hf * 64;
    int jg = 0;
    for (int round = 0;; ++round) {
      const int item = snake_item(round, blockIdx.x, gridDim.x);
      if (item >= n_items) break;
      const int h = item % a.H;
      const int tile = a.tiles[item / a.H];
      const int seq = tile >> 16, qt = tile & 0xFFFF;
      const int s0 = a.seq_start[seq];
      const int len = a.seq_start[seq + 1] - s0;
      const int q0 = qt * kTile;
      const int n_kv = qt + 1;
      const int qi = q0 + row;               // sequence-local query index
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n_kv; ++j) {
        const int g = jg + j;
        const int sb = g & 1;
        mbar_wait(&bar.s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_base + sb * kTile + hf * 64;
        const int kmax = min(qi, len - 1) - j * kTile - hf * 64;  // keys [0, kmax] of this half are visible
        // S read once (64 keys of this half into registers); the S buffer is
        // handed back right away so Q K_{j+2}^T can start.
        float v[64];
        tmem_ld_32x32b_x32(s_addr, *reinterpret_cast<float(*)[32]>(v));
        tmem_ld_32x32b_x32(s_addr + 32, *reinterpret_cast<float(*)[32]>(v + 32));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.s_empty[sb]);
        // partial row max over this half, exchanged with the partner warp
        // Tiles below the diagonal and inside the sequence need no masking:
        // the fast path is 3-input max, paired FMA, bare MUFU.EX2, paired add.
        const bool full = kmax >= 63;
        float mx = -INFINITY;
        if (full) {
  #pragma unroll
          for (int i = 0; i < 64; i += 2) mx = fmax3(mx, v[i], v[i + 1]);
        } else {
  #pragma unroll
          for (int i = 0; i < 64; ++i)
            if (i <= kmax) mx = fmaxf(mx, v[i]);
        }
        bar.mx[g & 1][hf][row] = mx;
        asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
        mx = fmaxf(mx, bar.mx[g & 1][hf ^ 1][row]);
        // Lazy rescaling: the running max only moves (and O is rescaled) when
        // the tile's max exceeds it by more than 2^8; otherwise P = exp2(s - m)
        // stays <= 256 under the stale max, and l / O share that max, so the
        // final O / l is unchanged.
        const float m_tile = mx * a.scale_log2;
        const bool move = m_tile > m_run + 8.f;
        const float m_new = move ? m_tile : m_run;
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = move ? exp2f(m_run - m_use) : 1.f;
        // P = exp2(s - m) -> packed bf16 in registers while P_{j-1} V_{j-1} runs
        float psum = 0.f;
        uint32_t pk[32];
        if (full) {
          float s0 = 0.f, s1 = 0.f;
  #pragma unroll
          for (int i = 0; i < 64; i += 2) {
            float x0, x1;
            ffma2(x0, x1, v[i], v[i + 1], a.scale_log2, a.scale_log2, -m_use, -m_use);
            const float p0 = ex2_ftz(x0), p1 = ex2_ftz(x1);
            fadd2(s0, s1, p0, p1);
            pk[i >> 1] = pack_bf16(p0, p1);
          }
          psum = s0 + s1;
        } else {
  #pragma unroll
          for (int i = 0; i < 64; i += 2) {
            const float p0 = i <= kmax ? exp2f(fmaf(v[i], a.scale_log2, -m_use)) : 0.f;
            const float p1 = i + 1 <= kmax ? exp2f(fmaf(v[i + 1], a.scale_log2, -m_use)) : 0.f;
            psum += p0 + p1;
            pk[i >> 1] = pack_bf16(p0, p1);
          }
        }
        if (g > 0) {
          // the previous P V (this item's or the previous item's last) is
          // complete: the P buffer is free and O may be rescaled
          mbar_wait(&bar.o_full, (g - 1) & 1);
          tc_fence_after();
        }
        // keys [64hf + 8chunk, +8) in the SW128 K-major image of this half's row
  #pragma unroll
        for (int chunk = 0; chunk < 8; ++chunk)
          *reinterpret_cast<uint4*>(p_row + ((chunk ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * chunk], pk[4 * chunk + 1], pk[4 * chunk + 2], pk[4 * chunk + 3]);
        if (j > 0 && __any_sync(0xffffffffu, move)) {
  #pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            float o[32];
            tmem_ld_32x32b_x32(o_addr + c * 32, o);
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st_32x32b_x32(o_addr + c * 32, o);
          }
        }
        l_run = l_run * alpha + psum;
        m_run = m_new;
        tc_fence_before();
        fence_async_smem();  // P (generic writes) -> the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.p_full);
      }
      bar.ls[hf][row] = l_run;
      asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
      const float l_tot = l_run + bar.ls[hf ^ 1][row];
      mbar_wait(&bar.o_full, (jg + n_kv - 1) & 1);
      tc_fence_after();
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                            (static_cast<int64_t>(s0 + qi) * a.H + h) * 128 + hf * 64);
  #pragma unroll
      for (int c = 0; c < 2; ++c) {
        float v[32];
        tmem_ld_32x32b_x32(o_addr + c * 32, v);  // all lanes: .sync.aligned
        if (qi < len) {
  #pragma unroll
          for (int u = 0; u < 4; ++u)
            dst[c * 4 + u] = make_uint4(pack_bf16(v[8 * u] * inv, v[8 * u + 1] * inv),
                                        pack_bf16(v[8 * u + 2] * inv, v[8 * u + 3] * inv),
                                        pack_bf16(v[8 * u + 4] * inv, v[8 * u + 5] * inv),
                                        pack_bf16(v[8 * u + 6] * inv, v[8 * u + 7] * inv));
        }
      }
      tc_fence_before();  // O read: the next item's P_0 V_0 may overwrite it
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.o_empty);
      jg += n_kv;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}


// ---------------------------------------------------------------------------
// K3, split-group form (MUX_K3=2). Two softmax groups of four warps each take
// alternate key tiles of the same 128-query tile (group g: tiles j with
// j % 2 == g), one thread per query row over all 128 keys of a tile. Each
// group is a complete flash attention with its own running max / sum, its own
// S and O in TMEM (S_g = cols [128g, +128), O_g = [256 + 128g, +128)) and its
// own P buffer, so no per-tile row-max exchange is needed and the groups run
// out of phase: one group's exps overlap the other group's MMAs. The epilogue
// merges (m0, l0, O0) with (m1, l1, O1); group g writes output dims
// [64g, 64g + 64).
constexpr int kGroupWarps = 4;
constexpr int kThreads2 = (2 * kGroupWarps + 1) * 32;  // + 1 TMA/MMA warp
struct Bars2 {
  uint64_t q_full, q_empty, o_empty;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], s_empty[2], p_full[2], o_full[2];
  uint32_t tmem;
  uint32_t pad;
};
// Q + 2 stages of K and V + P0, P1 + barriers: 224.2 KiB of the 227 KiB a
// CTA may hold (the dynamic window starts 1 KiB-aligned after the 1 KiB the
// driver reserves; checked in the kernel). The epilogue's (m, l) exchange
// lives in the P buffers, idle once the item's P V are done.
constexpr size_t kSmem2 = kTileBytes + kStages * 2 * kTileBytes + 2 * kTileBytes + sizeof(Bars2);

__global__ void __launch_bounds__(kThreads2, 1)
prefill_attention_split_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                               const PrefillAttnArgs a) {
  // no __align__(1024) on the declaration: it costs 1 KiB of static shared
  // memory, and Q + K/V + P + barriers need all but ~850 B of the 227 KiB
  extern __shared__ __align__(16) uint8_t smem_split[];
  if ((smem_u32(smem_split) & 1023u) != 0) __trap();  // SW128 images need 1 KiB alignment
  uint8_t* q_s = smem_split;
  uint8_t* kv_s = q_s + kTileBytes;                 // [stage][K|V][2 halves]
  uint8_t* p_s = kv_s + kStages * 2 * kTileBytes;   // [group][2 halves][128 rows][128 B]
  Bars2& bar = *reinterpret_cast<Bars2*>(p_s + 2 * kTileBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = a.n_tiles * a.H;

  if (threadIdx.x == 0) {
    mbar_init(&bar.q_full, 1);
    mbar_init(&bar.q_empty, 1);
    mbar_init(&bar.o_empty, 2 * kGroupWarps);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar.k_full[s], 1);
      mbar_init(&bar.k_empty[s], 1);
      mbar_init(&bar.v_full[s], 1);
      mbar_init(&bar.v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bar.s_full[g], 1);
      mbar_init(&bar.s_empty[g], kGroupWarps);
      mbar_init(&bar.p_full[g], kGroupWarps);
      mbar_init(&bar.o_full[g], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kTmemCols>(&bar.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  grid_dep_wait();  // q / k / v come from kv_append and the QKV GEMM
  if (threadIdx.x == 0) grid_dep_launch();
  const uint32_t tmem = bar.tmem;

  if (warp == 2 * kGroupWarps) {
    if (elect_one()) {
      // ---------------- TMA producer + MMA issuer
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_last();
      const uint32_t idesc_qk = umma_idesc_bf16(kTile, kTile);
      const uint32_t idesc_pv = umma_idesc_bf16(kTile, 128) | (1u << 16);  // B (V) MN-major
      const uint32_t q_addr = smem_u32(q_s);
      int jg = 0;                 // key tiles of earlier items (K/V ring position)
      int nq0 = 0, nq1 = 0;       // Q K^T issued per group (S_g uses)
      int np0 = 0, np1 = 0;       // P V issued per group
      for (int round = 0, it = 0;; ++round, ++it) {
        const int item = snake_item(round, blockIdx.x, gridDim.x);
        if (item >= n_items) break;
        const int h = item % a.H;
        const int tile = a.tiles[item / a.H];
        const int seq = tile >> 16, qt = tile & 0xFFFF;
        const int s0 = a.seq_start[seq];
        const int n_kv = qt + 1;
        if (it > 0) mbar_wait(&bar.q_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(&bar.q_full, kTileBytes);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(q_s + hh * kHalfBytes, &tq, &bar.q_full, h * 128 + hh * 64, s0 + qt * kTile, pol_q);
        auto load = [&](int j, bool v) {
          const int g = jg + j, st = g % kStages;
          uint64_t* empty = v ? &bar.v_empty[st] : &bar.k_empty[st];
          uint64_t* full = v ? &bar.v_full[st] : &bar.k_full[st];
          if (g >= kStages) mbar_wait(empty, ((g / kStages) - 1) & 1);
          uint8_t* dst = kv_s + st * 2 * kTileBytes + (v ? kTileBytes : 0);
          mbar_arrive_expect_tx(full, kTileBytes);
          for (int hh = 0; hh < 2; ++hh)
            tma_load_2d(dst + hh * kHalfBytes, &tkv, full, ((v ? 2 : 1) * a.H + h) * 128 + hh * 64, s0 + j * kTile,
                        pol_kv);
        };
        auto issue_qk = [&](int j) {
          const int gt = jg + j, st = gt % kStages, grp = j & 1;
          const int u = grp ? nq1++ : nq0++;
          if (u >= 1) mbar_wait(&bar.s_empty[grp], (u - 1) & 1);  // the group has read its previous S
          mbar_wait(&bar.k_full[st], (gt / kStages) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(kv_s + st * 2 * kTileBytes);
  #pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
            umma_bf16(tmem + grp * kTile, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_qk,
                      kk > 0 ? 1u : 0u);
          }
          umma_commit(&bar.s_full[grp]);
          umma_commit(&bar.k_empty[st]);
          if (j + 1 == n_kv) umma_commit(&bar.q_empty);  // the item's last Q K^T: Q reusable
        };
        auto issue_pv = [&](int j) {
          const int gt = jg + j, st = gt % kStages, grp = j & 1;
          const int u = grp ? np1++ : np0++;
          // the previous item's epilogue read both O before this item's first P V
          if (j == 0 && it > 0) mbar_wait(&bar.o_empty, (it - 1) & 1);
          mbar_wait(&bar.p_full[grp], u & 1);
          mbar_wait(&bar.v_full[st], (gt / kStages) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(kv_s + st * 2 * kTileBytes + kTileBytes);
          const uint32_t p_addr = smem_u32(p_s + grp * kTileBytes);
  #pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tmem + 2 * kTile + grp * kTile, umma_desc_sw128(p_addr + (kk >> 2) * kHalfBytes + (kk & 3) * 32),
                      umma_desc_sw128_mn(v_addr + kk * 2048), idesc_pv, (j >= 2 || kk > 0) ? 1u : 0u);
          umma_commit(&bar.o_full[grp]);
          umma_commit(&bar.v_empty[st]);
        };
        load(0, false);
        load(0, true);
        if (n_kv > 1) load(1, false);
        mbar_wait(&bar.q_full, it & 1);
        issue_qk(0);
        if (n_kv > 1) issue_qk(1);
        for (int j = 0; j < n_kv; ++j) {
          if (j + 2 < n_kv) {
            load(j + 2, false);  // K_{j+2} into Q K_j^T's slot (done or nearly)
            issue_qk(j + 2);
          }
          if (j + 1 < n_kv) load(j + 1, true);  // V_{j+1} into P_{j-1} V_{j-1}'s slot
          issue_pv(j);
        }
        jg += n_kv;
      }
    }
    __syncwarp();
  } else if (warp < 2 * kGroupWarps) {
    // ---------------- softmax groups: thread = query row, all 128 keys of a tile
    const int grp = warp / kGroupWarps, quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + grp * kTile;
    const uint32_t o_addr = tmem + lane_base + 2 * kTile + grp * kTile;
    uint8_t* p_row = p_s + grp * kTileBytes + row * 128;
    int cnt0 = 0, cnt1 = 0;  // tiles each group processed in earlier items
    for (int round = 0, it = 0;; ++round, ++it) {
      const int item = snake_item(round, blockIdx.x, gridDim.x);
      if (item >= n_items) break;
      const int h = item % a.H;
      const int tile = a.tiles[item / a.H];
      const int seq = tile >> 16, qt = tile & 0xFFFF;
      const int s0 = a.seq_start[seq];
      const int len = a.seq_start[seq + 1] - s0;
      const int n_kv = qt + 1;
      const int qi = qt * kTile + row;
      const int mine = (n_kv - grp + 1) / 2;  // tiles of this group in the item
      float m_run = -INFINITY, l_run = 0.f;
      for (int t = 0; t < mine; ++t) {
        const int j = 2 * t + grp;
        const int u = (grp ? cnt1 : cnt0) + t;  // this group's global tile count
        mbar_wait(&bar.s_full[grp], u & 1);
        tc_fence_after();
        float v[128];
  #pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(s_addr + c * 32, *reinterpret_cast<float(*)[32]>(v + 32 * c));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.s_empty[grp]);  // S_g may take Q K_{j+2}^T
        const int kmax = min(qi, len - 1) - j * kTile;  // keys [0, kmax] of this tile are visible
        const bool full = kmax >= 127;
        float mx = -INFINITY;
        if (full) {
  #pragma unroll
          for (int i = 0; i < 128; i += 2) mx = fmax3(mx, v[i], v[i + 1]);
        } else {
  #pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i <= kmax) mx = fmaxf(mx, v[i]);
        }
        const float m_tile = mx * a.scale_log2;
        const bool move = m_tile > m_run + 8.f;  // lazy rescaling (see the one-group kernel)
        const float m_new = move ? m_tile : m_run;
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = move ? exp2f(m_run - m_use) : 1.f;
        // the group's previous P V (this item's or an earlier item's) is done:
        // its P buffer is free and O_g may be rescaled. Waiting here (not
        // after the exps) lets each 8-key chunk of P go to smem as soon as it
        // is computed, so no packed copy of the row is held in registers.
        if (u >= 1) {
          mbar_wait(&bar.o_full[grp], (u - 1) & 1);
          tc_fence_after();
        }
        float psum = 0.f;
        if (full) {
          float sa = 0.f, sb = 0.f;
  #pragma unroll
          for (int c8 = 0; c8 < 16; ++c8) {
            uint32_t pk[4];
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 8 * c8 + 2 * e;
              float x0, x1;
              ffma2(x0, x1, v[i], v[i + 1], a.scale_log2, a.scale_log2, -m_use, -m_use);
              const float p0 = ex2_ftz(x0), p1 = ex2_ftz(x1);
              fadd2(sa, sb, p0, p1);
              pk[e] = pack_bf16(p0, p1);
            }
            *reinterpret_cast<uint4*>(p_row + (c8 >> 3) * kHalfBytes + (((c8 & 7) ^ (row & 7)) << 4)) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          psum = sa + sb;
        } else {
  #pragma unroll
          for (int c8 = 0; c8 < 16; ++c8) {
            uint32_t pk[4];
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 8 * c8 + 2 * e;
              const float p0 = i <= kmax ? exp2f(fmaf(v[i], a.scale_log2, -m_use)) : 0.f;
              const float p1 = i + 1 <= kmax ? exp2f(fmaf(v[i + 1], a.scale_log2, -m_use)) : 0.f;
              psum += p0 + p1;
              pk[e] = pack_bf16(p0, p1);
            }
            *reinterpret_cast<uint4*>(p_row + (c8 >> 3) * kHalfBytes + (((c8 & 7) ^ (row & 7)) << 4)) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        if (t > 0 && __any_sync(0xffffffffu, move)) {
  #pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tmem_ld_32x32b_x32(o_addr + c * 32, o);
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st_32x32b_x32(o_addr + c * 32, o);
          }
        }
        l_run = l_run * alpha + psum;
        m_run = m_new;
        tc_fence_before();
        fence_async_smem();  // P (generic writes) -> the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.p_full[grp]);
      }
      // ---- epilogue: merge the two groups; group g writes dims [64g, 64g + 64)
      const int n0 = (n_kv + 1) / 2, n1 = n_kv / 2;  // tiles of group 0 / 1 in this item
      // every P V of the item is done: O final, both P buffers idle
      mbar_wait(&bar.o_full[0], (cnt0 + n0 - 1) & 1);
      if (n1 > 0) mbar_wait(&bar.o_full[1], (cnt1 + n1 - 1) & 1);
      tc_fence_after();
      float* ml_mine = reinterpret_cast<float*>(p_s + grp * kTileBytes);
      const float* ml_other = reinterpret_cast<const float*>(p_s + (grp ^ 1) * kTileBytes);
      ml_mine[row] = m_run;
      ml_mine[128 + row] = l_run;
      asm volatile("bar.sync 1, %0;" ::"n"(2 * kGroupWarps * 32) : "memory");
      const float mo = ml_other[row], lo = ml_other[128 + row];
      asm volatile("bar.sync 1, %0;" ::"n"(2 * kGroupWarps * 32) : "memory");  // read: P buffers reusable
      const float m0 = grp ? mo : m_run, l0 = grp ? lo : l_run;
      const float m1 = grp ? m_run : mo, l1 = grp ? l_run : lo;
      const float m = fmaxf(m0, m1);
      const float a0 = l0 > 0.f ? exp2f(m0 - m) : 0.f;
      const float a1 = l1 > 0.f ? exp2f(m1 - m) : 0.f;
      const float lt = l0 * a0 + l1 * a1;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                            (static_cast<int64_t>(s0 + qi) * a.H + h) * 128 + grp * 64);
      const uint32_t o0 = tmem + lane_base + 2 * kTile + grp * 64;
  #pragma unroll
      for (int c = 0; c < 2; ++c) {
        float x[32], y[32];
        tmem_ld_32x32b_x32(o0 + c * 32, x);  // all lanes: .sync.aligned
        if (n1 > 0) {
          tmem_ld_32x32b_x32(o0 + kTile + c * 32, y);
        } else {
  #pragma unroll
          for (int i = 0; i < 32; ++i) y[i] = 0.f;
        }
        if (qi < len) {
  #pragma unroll
          for (int u = 0; u < 4; ++u) {
            float z[8];
  #pragma unroll
            for (int e = 0; e < 8; ++e) z[e] = (x[8 * u + e] * a0 + y[8 * u + e] * a1) * inv;
            dst[c * 4 + u] = make_uint4(pack_bf16(z[0], z[1]), pack_bf16(z[2], z[3]), pack_bf16(z[4], z[5]),
                                        pack_bf16(z[6], z[7]));
          }
        }
      }
      tc_fence_before();  // both O read: the next item's first P V may overwrite them
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar.o_empty);
      cnt0 += n0;
      cnt1 += n1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace

size_t prefill_attention_smem() { return kSmemBytes; }

cudaError_t preload_prefill_attention() { return preload(prefill_attention_kernel, prefill_attention_split_kernel); }

cudaError_t prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.T <= 0 || a.n_tiles <= 0) return cudaSuccess;
  static const int env_k3 = getenv("MUX_K3") ? atoi(getenv("MUX_K3")) : 2;  // 1: the one-group form
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([] {
    cudaError_t e = cudaFuncSetAttribute(prefill_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(prefill_attention_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem2));
  });
  if (ce != cudaSuccess) return ce;
  CUtensorMap tq, tkv;
  std::memcpy(&tq, a.tmap_q, sizeof(CUtensorMap));
  std::memcpy(&tkv, a.tmap_qkv, sizeof(CUtensorMap));
  const int n_items = a.n_tiles * a.H;
  const int grid = std::max(1, std::min(n_items, a.max_ctas > 0 ? a.max_ctas : 148));
  if (env_k3 == 2) {
    cudaError_t e = launch(prefill_attention_split_kernel, dim3(grid), dim3(kThreads2), kSmem2, stream, tq, tkv, a);
    if (e == cudaErrorLaunchOutOfResources) {  // diagnostics for the resource budget of this form
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(prefill_attention_split_kernel));
      int optin = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      std::fprintf(stderr, "K3 split: regs %d maxThreads %d static smem %zu maxDyn %d requested dyn %zu optin %d threads %d\n",
                   fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, kSmem2, optin,
                   kThreads2);
    }
    return e;
  }
  return launch(prefill_attention_kernel, dim3(grid), dim3(kThreads), kSmemBytes, stream, tq, tkv, a);
}

}  // namespace mux
