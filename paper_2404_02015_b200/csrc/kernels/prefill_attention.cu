// K3: causal varlen prefill attention on the 5th-generation tensor cores.
//
// Work it replaces: the attention part of prefill_latency
// (/root/reference/proj/src/cost_model.cpp:75-83) -- causal softmax(q k^T /
// sqrt(128)) v over every prompt of a prefill job, head_dim 128, after
// kv_append has rotated q and k (RoPE) and written k/v into the head-blocks
// (the K/V read here are the same bytes, straight from the QKV GEMM output).
//
// Persistent: each CTA walks a list of items (128-query tile of one sequence,
// head); its MMA warp streams the items' key tiles back to back, Q
// double-buffered by item. Flash-attention over 128-key tiles with both
// contractions on tcgen05:
//   S_j = Q K_j^T      UMMA 128x128x128, A = Q (smem, K-major), B = K_j (smem,
//                      K-major), fp32 accumulator in TMEM (double-buffered so
//                      S_{j+1} is computed while the softmax reads S_j)
//   O_j = P_j V_j      UMMA 128x128x128, A = P_j from TENSOR MEMORY (the
//                      softmax stores bf16 pairs with tcgen05.st, row = lane,
//                      64 columns; no shared-memory traffic for P), B = V_j
//                      (smem, MN-major: the same TMA box as K, other descriptor)
// Warp 8 = TMA producer + MMA issuer (one elected lane); warps 0-7 = softmax,
// two warps per TMEM lane quarter, a thread owns half (64 keys / 64 output
// dims) of one query row: online max/sum in fp32, causal + sequence-end
// masking (masked scores set to -inf); in full tiles exp2 runs on MUFU for 5 of 8 pairs and as an
// FMA-pipe polynomial for 3. The output accumulates in TMEM across key tiles; when
// a row's max moves, its O row is rescaled in place (tcgen05.ld/st) before
// the next P V is issued.
// K/V tiles stream through a kStages-deep TMA ring (SWIZZLE_128B boxes of 64
// dims x 128 tokens over the [T][3][H][128] QKV buffer).
// FLOPs per (sequence of length n, head): 4 * 128 * n * (n + 1) / 2 (causal).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
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
// kParts softmax warps per TMEM lane quarter, each owning kKeys of a row's
// 128 keys (and 128 / kParts of its output dims). 2 (8 softmax warps) is
// the measured best: 4 parts (16 warps) ran 4096 tokens x 40 heads in 263
// instead of 245 us (profiles/r02_k3_parts.txt).
#ifndef MUX_K3_PARTS
#define MUX_K3_PARTS 2
#endif
constexpr int kParts = MUX_K3_PARTS;
constexpr int kKeys = kTile / kParts;
static_assert(kKeys == 64, "P is written as one 32-column tcgen05.st of bf16 pairs per part: kParts must be 2");
constexpr int kSoftmaxWarps = 4 * kParts;
constexpr int kThreads = (kSoftmaxWarps + 1) * 32;  // + 1 TMA/MMA warp
constexpr uint32_t kTmemCols = 512;          // S0 [0,128) S1 [128,256) O [256,384) P [384,448)
constexpr uint32_t kPCol = 384;              // P: bf16 pairs, row = lane (the PV MMA's A operand)
constexpr size_t kSmemBytes = 1024 + 2 * kTileBytes /*Q, double-buffered*/ + kStages * 2 * kTileBytes /*K,V*/ +
                              256 /*barriers*/ + 3 * kParts * 128 * 4 /*row exchange*/;

struct Bars {
  uint64_t q_full[2];  // per Q buffer (item parity)
  uint64_t k_full[kStages];
  uint64_t k_empty[kStages];
  uint64_t v_full[kStages];
  uint64_t v_empty[kStages];
  uint64_t s_full[2];
  uint64_t s_empty[2];
  uint64_t p_full;
  uint64_t o_full;
  uint64_t q_empty[2];  // per Q buffer: the item's last Q K^T done, buffer reusable
  uint64_t o_empty;  // persistent: the softmax warps have read the item's O
  uint32_t tmem;
  uint32_t pad[3];
  int4 items[4];  // MMA thread: descriptor ring {h, row0, q0, n_kv} by round & 3
  float mx[2][kParts][128];  // [tile parity][key part][row]: partial row maxima
  float ls[kParts][128];     // [key part][row]: partial row sums (end)
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

// exp2(v * scale - m) of a thread's kKeys scores, packed to bf16 pairs;
// returns the fp32 sum. kP of every 8 pairs use the FMA-pipe polynomial.
template <int kP>
__device__ __forceinline__ float exp_pack(const float (&v)[kKeys], float scale, float m, uint32_t (&pk)[kKeys / 2]) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int i = 0; i < kKeys; i += 2) {
    float x0, x1, p0, p1;
    ffma2(x0, x1, v[i], v[i + 1], scale, scale, -m, -m);
    if (((i >> 1) & 7) < kP) {
      ex2_poly2(p0, p1, x0, x1);
    } else {
      p0 = ex2_ftz(x0);
      p1 = ex2_ftz(x1);
    }
    fadd2(s0, s1, p0, p1);
    pk[i >> 1] = pack_bf16(p0, p1);
  }
  return s0 + s1;
}

// kPoly of every 8 exp2 pairs of a full tile run as the FMA-pipe polynomial
// (ex2_poly2) instead of MUFU.EX2. The back-to-back MUFU block held a third of
// the softmax warps' stall samples (FMA pipe 9% busy); 3 of 8 pairs on the
// FMA pipe: 4096 tokens x 40 heads 200.8 -> 195.9 us (4 of 8: no better).
template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
prefill_attention_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                         const PrefillAttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* q_s = base;
  uint8_t* kv_s = q_s + 2 * kTileBytes;             // [stage][K|V][2 halves]
  Bars& bar = *reinterpret_cast<Bars*>(kv_s + kStages * 2 * kTileBytes);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent: CTA c takes one work item per round in snake order over the
  // heaviest-first list (item = tile index * H + head). TMEM, barriers and the pipeline
  // counters live across items; the next item's Q / K_0 / V_0 loads and its
  // first Q K^T overlap the current item's last P V and epilogue.
  const int n_items = a.n_tiles * a.H;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar.q_full[b], 1);
      mbar_init(&bar.q_empty[b], 1);
    }
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
      // One flat stream of key tiles g over this CTA's items (rounds r), walked
      // by four cursors: the K loads run two tiles ahead, V one, Q K^T one, and
      // P V last. Q is double-buffered by item parity, so the next item's Q
      // load and its first Q K^T are issued while the current item's last
      // softmax and P V run (short prompts are one or two key tiles per item).
      struct Cur {
        int r, j, g, h, row0, q0, n_kv;
        bool valid;
      };
      // Descriptors are loaded once per item by the leading (K-load) cursor
      // into a 4-deep ring the trailing cursors read (they lag by at most
      // three key tiles); the next item's tile word is prefetched a round
      // ahead, so entering an item costs one global-load latency, not two.
      int pf_tile = 0;
      auto fill = [&](int r) {
        const int item = snake_item(r, blockIdx.x, gridDim.x);
        int4 d = make_int4(0, 0, 0, 0);  // n_kv = 0: past the last item
        if (item < n_items) {
          const int tile = r == 0 ? a.tiles[item / a.H] : pf_tile;
          const int qt = tile & 0xFFFF;
          d = make_int4(item % a.H, a.seq_start[tile >> 16], qt * kTile, qt + 1);  // causal: key tiles 0..qt
          const int item_n = snake_item(r + 1, blockIdx.x, gridDim.x);
          pf_tile = item_n < n_items ? a.tiles[item_n / a.H] : 0;
        }
        bar.items[r & 3] = d;
      };
      auto fetch = [&](Cur& c, bool lead) {
        if (lead) fill(c.r);
        const int4 d = bar.items[c.r & 3];
        c.valid = d.w > 0;
        c.h = d.x;
        c.row0 = d.y;
        c.q0 = d.z;
        c.n_kv = d.w;
      };
      auto advance = [&](Cur& c, bool lead = false) {
        ++c.g;
        if (++c.j == c.n_kv) {
          ++c.r;
          c.j = 0;
          fetch(c, lead);
        }
      };
      Cur start{0, 0, 0, 0, 0, 0, 0, false};
      fetch(start, true);
      auto load_q = [&](const Cur& c) {
        const int b = c.r & 1;
        if (c.r >= 2) mbar_wait(&bar.q_empty[b], ((c.r >> 1) - 1) & 1);  // item r-2's Q K^T are done
        mbar_arrive_expect_tx(&bar.q_full[b], kTileBytes);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(q_s + b * kTileBytes + hh * kHalfBytes, &tq, &bar.q_full[b], c.h * 128 + hh * 64, c.row0 + c.q0,
                      pol_q);
      };
      // K and V of a tile have separate ring slots and barriers: K_g's slot
      // frees when S_g = Q K_g^T completes (early), V_g's when P_g V_g does,
      // so the next K load never waits behind a P V.
      auto load_k = [&](const Cur& c) {
        if (c.j == 0) load_q(c);
        const int st = c.g % kStages;
        if (c.g >= kStages) mbar_wait(&bar.k_empty[st], ((c.g / kStages) - 1) & 1);
        uint8_t* dst = kv_s + st * 2 * kTileBytes;
        mbar_arrive_expect_tx(&bar.k_full[st], kTileBytes);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(dst + hh * kHalfBytes, &tkv, &bar.k_full[st], (a.H + c.h) * 128 + hh * 64, c.row0 + c.j * kTile,
                      pol_kv);
      };
      auto load_v = [&](const Cur& c) {
        const int st = c.g % kStages;
        if (c.g >= kStages) mbar_wait(&bar.v_empty[st], ((c.g / kStages) - 1) & 1);
        uint8_t* dst = kv_s + st * 2 * kTileBytes + kTileBytes;
        mbar_arrive_expect_tx(&bar.v_full[st], kTileBytes);
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(dst + hh * kHalfBytes, &tkv, &bar.v_full[st], (2 * a.H + c.h) * 128 + hh * 64,
                      c.row0 + c.j * kTile, pol_kv);
      };
      auto issue_qk = [&](const Cur& c) {
        const int st = c.g % kStages, sb = c.g & 1, b = c.r & 1;
        mbar_wait(&bar.k_full[st], (c.g / kStages) & 1);
        if (c.g >= 2) mbar_wait(&bar.s_empty[sb], ((c.g >> 1) - 1) & 1);
        if (c.j == 0) mbar_wait(&bar.q_full[b], (c.r >> 1) & 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(q_s + b * kTileBytes);
        const uint32_t k_addr = smem_u32(kv_s + st * 2 * kTileBytes);
  #pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kHalfBytes + (kk & 3) * 32;
          umma_bf16(tmem + sb * kTile, umma_desc_sw128(q_addr + off), umma_desc_sw128(k_addr + off), idesc_qk,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(&bar.s_full[sb]);
        umma_commit(&bar.k_empty[st]);
        if (c.j + 1 == c.n_kv) umma_commit(&bar.q_empty[b]);  // fires once the item's last Q K^T is done
      };
      if (start.valid) {
        Cur kl = start, vl = start, qk = start, pv = start;
        for (int n = 0; n < kStages && kl.valid; ++n, advance(kl, true)) load_k(kl);
        for (int n = 0; n < kStages && vl.valid; ++n, advance(vl)) load_v(vl);
        issue_qk(qk);
        advance(qk);
        while (pv.valid) {
          // S_{g+1} while the softmax reads S_g; the next item's first S goes
          // after this item's last P V, which the epilogue waits for
          const bool qk_after = qk.valid && qk.r != pv.r;
          if (qk.valid && !qk_after) {
            issue_qk(qk);
            advance(qk);
          }
          if (kl.valid) {  // K_{g+2} into S_g's K slot as soon as S_g is done
            load_k(kl);
            advance(kl, true);
          }
          if (vl.valid && vl.g == pv.g + 1) {  // V_{g+1}: waits for P_{g-1} V_{g-1}
            load_v(vl);
            advance(vl);
          }
          // the previous item's O must have been read before P_0 V_0 overwrites it
          if (pv.j == 0 && pv.r > 0) mbar_wait(&bar.o_empty, (pv.r - 1) & 1);
          // O_g = P_g V_g once the softmax has written P_g
          mbar_wait(&bar.p_full, pv.g & 1);
          const int st = pv.g % kStages;
          mbar_wait(&bar.v_full[st], (pv.g / kStages) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(kv_s + st * 2 * kTileBytes + kTileBytes);
  #pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            umma_ts_bf16(tmem + 2 * kTile, tmem + kPCol + kk * 8, umma_desc_sw128_mn(v_addr + kk * 2048), idesc_pv,
                         (pv.j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&bar.o_full);
          umma_commit(&bar.v_empty[st]);
          if (qk_after) {
            issue_qk(qk);
            advance(qk);
          }
          advance(pv);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps: thread = (query row, key part)
    // Warps w, w+4, w+8, ... share TMEM lane quarter w%4 (rows 32*(w%4)..+31)
    // and split the 128 keys of a tile (and the 128 output dims) into kParts
    // parts of kKeys; the row max is exchanged through smem once per tile
    // (double-buffered by tile parity, so one barrier per tile), the row sums
    // once at the end.
    const int quarter = warp & 3, part = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    // this part's keys in P's SW128 K-major image: half (part*kKeys)/64, 16-B chunks from (part*kKeys%64)/8
    const uint32_t o_addr = tmem + lane_base + 2 * kTile + part * kKeys;
    int jg = 0;
    // Item descriptors are prefetched: the next item's tile word is loaded
    // when an item starts, its sequence bounds before the epilogue, so no
    // item begins on two dependent global loads (short prompts: 1-2 key tiles
    // per item).
    int item = snake_item(0, blockIdx.x, gridDim.x);
    int tile_c = 0, s0_c = 0, s1_c = 0;
    if (item < n_items) {
      tile_c = a.tiles[item / a.H];
      s0_c = a.seq_start[tile_c >> 16];
      s1_c = a.seq_start[(tile_c >> 16) + 1];
    }
    for (int round = 0; item < n_items; ++round) {
      const int h = item % a.H;
      const int qt = tile_c & 0xFFFF;
      const int s0 = s0_c;
      const int len = s1_c - s0_c;
      const int item_n = snake_item(round + 1, blockIdx.x, gridDim.x);
      const int tile_n = item_n < n_items ? a.tiles[item_n / a.H] : 0;
      const int q0 = qt * kTile;
      const int n_kv = qt + 1;
      const int qi = q0 + row;               // sequence-local query index
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n_kv; ++j) {
        const int g = jg + j;
        const int sb = g & 1;
        mbar_wait(&bar.s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        const uint32_t s_addr = tmem + lane_base + sb * kTile + part * kKeys;
        const int kmax = min(qi, len - 1) - j * kTile - part * kKeys;  // keys [0, kmax] of this part are visible
        // S read once (this part's keys into registers); the S buffer is
        // handed back right away so Q K_{j+2}^T can start.
        float v[kKeys];
  #pragma unroll
        for (int c = 0; c < kKeys / 32; ++c) tmem_ld_32x32b_x32(s_addr + c * 32, *reinterpret_cast<float(*)[32]>(v + 32 * c));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.s_empty[sb]);
        // partial row max over this part, exchanged with the quarter's other
        // warps. Tiles below the diagonal and inside the sequence need no
        // masking: the fast path is 3-input max, paired FMA, bare MUFU.EX2,
        // paired add.
        const bool full = kmax >= kKeys - 1;
        if (!full) {
          // masked keys -> -inf: MUFU.EX2 maps them to exactly +0 below
  #pragma unroll
          for (int i = 0; i < kKeys; ++i)
            if (i > kmax) v[i] = -INFINITY;
        }
        float mx = -INFINITY;
  #pragma unroll
        for (int i = 0; i < kKeys; i += 2) mx = fmax3(mx, v[i], v[i + 1]);
        bar.mx[g & 1][part][row] = mx;
        asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
  #pragma unroll
        for (int o = 0; o < kParts; ++o)
          if (o != part) mx = fmaxf(mx, bar.mx[g & 1][o][row]);
        // Lazy rescaling: the running max only moves (and O is rescaled) when
        // the tile's max exceeds it by more than 2^8; otherwise P = exp2(s - m)
        // stays <= 256 under the stale max, and l / O share that max, so the
        // final O / l is unchanged.
        const float m_tile = mx * a.scale_log2;
        const bool move = m_tile > m_run + 8.f;
        const float m_new = move ? m_tile : m_run;
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = move ? exp2f(m_run - m_use) : 1.f;
        // P = exp2(s - m) -> packed bf16 in registers while P_{j-1} V_{j-1} runs;
        // masked tiles keep every exponential on MUFU (exact zeros for -inf)
        uint32_t pk[kKeys / 2];
        const float psum = full ? exp_pack<kPoly>(v, a.scale_log2, m_use, pk) : exp_pack<0>(v, a.scale_log2, m_use, pk);
        if (g > 0) {
          // the previous P V (this item's or the previous item's last) is
          // complete: the P buffer is free and O may be rescaled
          mbar_wait(&bar.o_full, (g - 1) & 1);
          tc_fence_after();
        }
        // this part's keys as bf16 pairs in its row's lane, columns [kPCol + part*kKeys/2, +kKeys/2)
  #pragma unroll
        for (int c = 0; c < kKeys / 64; ++c)
          tmem_st_32x32b_x32(tmem + lane_base + kPCol + part * (kKeys / 2) + c * 32,
                             *reinterpret_cast<const float(*)[32]>(pk + 32 * c));
        if (j > 0 && __any_sync(0xffffffffu, move)) {
  #pragma unroll 1
          for (int c = 0; c < kKeys / 32; ++c) {
            float o[32];
            tmem_ld_32x32b_x32(o_addr + c * 32, o);
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st_32x32b_x32(o_addr + c * 32, o);
          }
        }
        l_run = l_run * alpha + psum;
        m_run = m_new;
        tc_fence_before();  // P stored to TMEM (tcgen05.wait::st) -> the P V MMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar.p_full);
      }
      if (item_n < n_items) {  // in flight during the epilogue
        s0_c = a.seq_start[tile_n >> 16];
        s1_c = a.seq_start[(tile_n >> 16) + 1];
      }
      bar.ls[part][row] = l_run;
      asm volatile("bar.sync 1, %0;" ::"n"(kSoftmaxWarps * 32) : "memory");
      float l_tot = 0.f;
  #pragma unroll
      for (int o = 0; o < kParts; ++o) l_tot += bar.ls[o][row];
      mbar_wait(&bar.o_full, (jg + n_kv - 1) & 1);
      tc_fence_after();
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) +
                                            (static_cast<int64_t>(s0 + qi) * a.H + h) * 128 + part * kKeys);
  #pragma unroll
      for (int c = 0; c < kKeys / 32; ++c) {
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
      item = item_n;
      tile_c = tile_n;
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

// MUX_K3_POLY (0, 3 or 4; read once) picks how many of every 8 exp2 pairs run
// on the FMA pipe. 3 is the measured best (profiles/r02_k3_exp_poly.txt).
using PrefillKernel = void (*)(const CUtensorMap, const CUtensorMap, const PrefillAttnArgs);
static PrefillKernel prefill_kernel_pick() {
  static const int poly = getenv("MUX_K3_POLY") ? atoi(getenv("MUX_K3_POLY")) : 3;
  switch (poly) {
    case 0: return prefill_attention_kernel<0>;
    case 4: return prefill_attention_kernel<4>;
    default: return prefill_attention_kernel<3>;
  }
}

cudaError_t preload_prefill_attention() { return preload(prefill_kernel_pick()); }

cudaError_t prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.T <= 0 || a.n_tiles <= 0) return cudaSuccess;
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run([] {
    return cudaFuncSetAttribute(prefill_kernel_pick(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemBytes));
  });
  if (ce != cudaSuccess) return ce;
  CUtensorMap tq, tkv;
  std::memcpy(&tq, a.tmap_q, sizeof(CUtensorMap));
  std::memcpy(&tkv, a.tmap_qkv, sizeof(CUtensorMap));
  const int n_items = a.n_tiles * a.H;
  const int grid = std::max(1, std::min(n_items, a.max_ctas > 0 ? a.max_ctas : 148));
  return launch(prefill_kernel_pick(), dim3(grid), dim3(kThreads), kSmemBytes, stream, tq, tkv, a);
}

}  // namespace mux
