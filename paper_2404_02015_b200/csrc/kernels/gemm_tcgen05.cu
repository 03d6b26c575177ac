// K4: bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Work it replaces: the prefill_coef * tokens and decode_base terms of the
// reference's pricing model (/root/reference/proj/src/cost_model.cpp:75-94):
// the QKV / O / gate-up / down / LM-head projections of every prefill and
// decode job.
//
//   D[M x N] = X[M x K] * W[N x K]^T      (X activations, W nn.Linear weight)
//
// Weight-stationary swap-AB tiling: the UMMA "A" operand is a 128-row slice
// of W and "B" up to 256 activation rows, so D^T tiles of 128 x n_tile
// accumulate in TMEM (fp32). A decode batch (M <= 256) reads each weight byte
// exactly once -- the HBM-bound regime -- and prefill tiles over tokens.
//
// Persistent stream-K: grid = #SMs; the flattened (tile, k-block) iteration
// space is cut into equal contiguous ranges, one per CTA, so every SM streams
// the same number of weight bytes regardless of how many 128-row tiles the
// projection has (no wave quantisation, no split-K planes). A tile cut
// between CTAs is finished in-kernel: the CTA holding the tile's first
// k-segment (it reaches that segment last) adds its partners' fp32 partials
// in a fixed order -- deterministic -- and applies the real epilogue;
// partners publish partials with release/acquire flags tagged by a launch
// epoch. Every CTA publishes at most one partial and only waits on CTAs of
// higher index that never wait on it, so the scheme cannot deadlock even
// when the grid is not fully co-resident.
//
// Warp roles: warp 0 = TMA producer, warp 1 = MMA issuer (one elected lane),
// warp 2 = TMEM allocator, warps 4..7 = epilogue. Accumulators are double
// buffered in TMEM so the epilogue of one segment overlaps the MMAs of the
// next; operands flow through an S-stage shared-memory ring (SWIZZLE_128B
// boxes, 64 K-elements per stage, full/empty mbarriers, tcgen05.commit frees
// a stage).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "launch.cuh"

namespace mux {
namespace {

constexpr int kBM = 128;  // W rows per tile (UMMA M)
constexpr int kBK = 64;   // K per stage (one 128-byte swizzle atom)
constexpr int kAStageBytes = kBM * kBK * 2;
constexpr int kThreads = 384;               // warps 0-3 roles, warps 4-11 two epilogue groups
constexpr int kEpiThreads = 128;            // one epilogue group: a warp per TMEM lane quarter
constexpr int kEpiGroups = 2;
constexpr int kChunkBytes = 32 * kBM * 4;  // one epilogue chunk: 32 tokens x 128 fp32
constexpr int kSmemBudget = 224 * 1024;     // A ring + B ring + 2 staging chunks

struct PeerMaps {
  CUtensorMap m[kMaxTp - 1];
};

struct GemmRun {
  const uint8_t* w_tiled;  // pre-tiled weights (weight_tile), or null -> TMA map
  void* out;
  float* partials;  // [grid][n_tile][128] fp32
  int* flags;       // [grid]
  int epoch;
  int M, N, K, ldo;
  int n_tile, stages_a, stages_b;
  int kb;           // k-blocks per tile
  int m_tiles;      // ceil(N / 128)
  int64_t iters;    // tiles * kb
  // Prefill schedule (several token tiles): n_dp data-parallel rounds of
  // whole tiles (tile j*G + c), raster-grouped group_m weight tiles wide so
  // the tiles in flight share their weight and activation k-slices in L2,
  // then stream-K over the remaining sk_iters. Decode: n_dp = 0, group_m =
  // 0, sk_iters = iters (pure stream-K).
  int n_dp, group_m, n_tok_tiles;
  int64_t sk_iters;
  int epi;
  uint32_t tmem_cols;
  unsigned long long* timing;  // debug: [grid][4] globaltimer stamps, or null
  // Tensor-parallel fan-out (kStoreF32 only): every finished tile is also
  // stored through peers.m[0..n_peers) (the same slot on the other ranks of
  // the mesh, NVLink peer memory), and once all of a CTA's stores have landed
  // it adds 1 to signal[0..n_signal) (this rank's and every peer's counter).
  QkvRopeArgs qr;   // kQkvRope
  int a_split;      // bulk copies per weight stage (1, 2, 4)
  int n_stg;        // epilogue staging buffers (1 or 2)
  int dbg_nomma;    // debug (MUX_GEMM_NOMMA): stream operands without MMAs
  int dbg_bres;     // debug (MUX_GEMM_BRES): load only the first SB activation stages, reuse them
  int n_peers;
  int n_signal;
  int* signal[kMaxTp];
  // Cross-launch L2 prefetch: once this CTA has issued its last weight load,
  // it prefetches the first pf_stages tiles of its range in the NEXT decode
  // GEMM of the chain (same flattened [m][kb] tile layout, contiguous), so
  // HBM keeps streaming through this launch's tail and the next one's head.
  const uint8_t* next_w;
  int next_grid;
  int pf_stages;
  int64_t next_iters;
  // fused RMSNorm of the residual rows (see GemmArgs::norm_w)
  const float* norm_w;
  __nv_bfloat16* norm_out;
  unsigned* norm_bar;
  unsigned norm_target;
  float norm_eps;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 32-bit index math: the host guarantees iters * grid < 2^32 (plan()), and a
// 64-bit division is a ~100-instruction call that sat on the producer's path
// to its first weight load.
__device__ __forceinline__ int64_t range_begin(int64_t iters, int c, int grid) {
  return static_cast<int64_t>(static_cast<uint32_t>(iters) * static_cast<uint32_t>(c) / static_cast<uint32_t>(grid));
}

// The work of one CTA as a sequence of segments: (tile, k-block range); the
// same sequence is walked by the producers, the MMA issuer and the epilogue.
struct SegGen {
  int64_t sk, sk_end;
  int j;
  __device__ SegGen(const GemmRun& r, int c, int G)
      : sk(range_begin(r.sk_iters, c, G)), sk_end(range_begin(r.sk_iters, c + 1, G)), j(0) {}
  // tile (m, nt), k-blocks [kb0, kb1); sk: stream-K piece of the tile whose
  // stream-K iterations are [lo, lo + kb)
  __device__ bool next(const GemmRun& r, int c, int G, int& m, int& nt, int& kb0, int& kb1, bool& skp, int64_t& lo) {
    int64_t tile;
    if (j < r.n_dp) {
      tile = static_cast<int64_t>(j) * G + c;
      ++j;
      kb0 = 0;
      kb1 = r.kb;
      skp = false;
      lo = 0;
    } else {
      if (sk >= sk_end) return false;
      const int64_t st = static_cast<uint32_t>(sk) / static_cast<uint32_t>(r.kb);
      lo = st * r.kb;
      kb0 = static_cast<int>(sk - lo);
      const int64_t e = min(sk_end, lo + r.kb);
      kb1 = static_cast<int>(e - lo);
      sk = e;
      skp = true;
      tile = static_cast<int64_t>(r.n_dp) * G + st;
    }
    if (r.group_m <= 0) {
      const uint32_t t32 = static_cast<uint32_t>(tile), mt = static_cast<uint32_t>(r.m_tiles);
      nt = static_cast<int>(t32 / mt);
      m = static_cast<int>(t32 - static_cast<uint32_t>(nt) * mt);
    } else {
      const int64_t per = static_cast<int64_t>(r.group_m) * r.n_tok_tiles;
      const uint32_t g = static_cast<uint32_t>(tile) / static_cast<uint32_t>(per);
      const uint32_t in = static_cast<uint32_t>(tile) - g * static_cast<uint32_t>(per);
      const int gm = min(r.group_m, r.m_tiles - static_cast<int>(g) * r.group_m);  // last group may be narrower
      nt = static_cast<int>(in / static_cast<uint32_t>(gm));
      m = static_cast<int>(g) * r.group_m + static_cast<int>(in - static_cast<uint32_t>(nt) * static_cast<uint32_t>(gm));
    }
    return true;
  }
};

__device__ __forceinline__ bool sg_has_more(const SegGen& sg, const GemmRun& r) {
  return sg.j < r.n_dp || sg.sk < sg.sk_end;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Named barriers: 1 + g for epilogue group g, 3 for both groups. Immediate
// ids: a register id makes ptxas reserve all 16 barriers, and then no other
// kernel's CTA (RMSNorm, K2 under PDL) can be co-resident with a GEMM CTA.
__device__ __forceinline__ void epi_bar(int g) {
  if (g == 0) asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
  else asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");
}
__device__ __forceinline__ void epi_bar_all() {
  asm volatile("bar.sync 3, %0;" ::"n"(kEpiGroups * kEpiThreads) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
gemm_tn_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
               const __grid_constant__ CUtensorMap tout, const GemmRun r, const __grid_constant__ PeerMaps peers) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB-aligned carve-up; pointer arithmetic on smem_raw itself keeps the
  // shared address space visible to the compiler (STS/LDS, not generic ST/LD).
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // Separate rings: weights (A, HBM-streamed) run SA stages deep, the small
  // L2-resident activation tiles (B) only SB, so more weight bytes are in
  // flight per SM than a shared ring of the same smem would allow.
  const int SA = r.stages_a, SB = r.stages_b;
  const int b_stage_bytes = r.n_tile * kBK * 2;
  uint8_t* a_st = base;
  uint8_t* b_st = base + SA * kAStageBytes;
  uint8_t* stage_out = b_st + SB * b_stage_bytes;  // 2 x 16 KiB epilogue staging
  uint64_t* full_a = reinterpret_cast<uint64_t*>(stage_out + r.n_stg * kChunkBytes);
  uint64_t* empty_a = full_a + SA;
  uint64_t* full_b = empty_a + SA;
  uint64_t* empty_b = full_b + SB;
  uint64_t* tm_full = empty_b + SB;  // [2]
  uint64_t* tm_empty = tm_full + 2;  // [2]
  uint64_t* pbar = tm_empty + 2;     // fixer's partial prefetch
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + 1);
  int* meta_pos = reinterpret_cast<int*>(tmem_slot + 4);  // kQkvRope: [256] token positions
  int* meta_id = meta_pos + 256;                          //            [256] K or V block ids
  float* norm_red = reinterpret_cast<float*>(meta_pos);   // fused RMSNorm (never with kQkvRope): [8]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int G = gridDim.x;
  if (r.timing != nullptr && threadIdx.x == 0) r.timing[c * 64 + 0] = gtimer();

  if (warp == 0 && lane == 0) {
    if (r.w_tiled == nullptr) prefetch_tmap(&tw);
    prefetch_tmap(&tx);
    prefetch_tmap(&tout);
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
      mbar_init(&tm_empty[b], kEpiGroups * kEpiThreads / 32);
    }
    mbar_init(pbar, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_dyn(tmem_slot, r.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (r.timing != nullptr && threadIdx.x == 0) r.timing[c * 64 + 15] = gtimer();
  if (threadIdx.x == 0) grid_dep_launch();

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------ TMA producers
    // warp 0 streams the weight tiles, warp 3 the activation tiles.
    if (elect_one()) {
      const bool is_a = warp == 0;
      if (is_a && r.timing != nullptr) r.timing[c * 64 + 32] = gtimer();
      // Weights do not depend on earlier kernels: warp 0 starts streaming
      // them while the predecessor drains (PDL); activations must wait.
      if (!is_a) grid_dep_wait();
      if (!is_a && r.dbg_nomma == 2) return;  // debug: weights only
      const uint64_t pol = is_a ? policy_evict_first()   // weights: streamed once per step
                                : policy_evict_last();   // activations: re-read by every CTA
      const int SS = is_a ? SA : SB;
      uint64_t* fb = is_a ? full_a : full_b;
      uint64_t* eb = is_a ? empty_a : empty_b;
      const uint32_t bytes = is_a ? kAStageBytes : b_stage_bytes;
      // Segments (tile, k-block range) with incremental stage counters: no
      // 64-bit division in the issue loop.
      if (is_a && r.timing != nullptr) r.timing[c * 64 + 33] = gtimer();
      SegGen sg(r, c, G);
      int m, nt, kb0, kb1;
      bool skp;
      int64_t lo;
      int s = 0, round = 0;
      if (is_a && r.timing != nullptr) r.timing[c * 64 + 34] = gtimer();
      int64_t issued = 0, pf_at = -1;
      if (is_a && r.next_w != nullptr && c < r.next_grid) {
        // start the prefetch when ~SA stages of this range remain
        const int64_t mine = range_begin(r.sk_iters, c + 1, G) - range_begin(r.sk_iters, c, G) +
                             static_cast<int64_t>(r.n_dp) * r.kb;
        pf_at = mine > SA ? mine - SA : 0;
      }
      while (sg.next(r, c, G, m, nt, kb0, kb1, skp, lo)) {
        for (int kbi = kb0; kbi < kb1; ++kbi) {
          if (!is_a && r.dbg_bres && round > 0) break;  // debug: resident activations
          if (round > 0) mbar_wait(&eb[s], (round - 1) & 1);
          if (is_a && round == 0 && s == 0 && r.timing != nullptr) r.timing[c * 64 + 35] = gtimer();
          mbar_arrive_expect_tx(&fb[s], bytes);
          if (is_a && round == 0 && s == 0 && r.timing != nullptr) r.timing[c * 64 + 36] = gtimer();
          if (is_a) {
            if (r.w_tiled != nullptr) {
              // one contiguous, pre-swizzled 16 KiB UMMA tile: a_split bulk copies
              const uint8_t* src = r.w_tiled + (static_cast<int64_t>(m) * r.kb + kbi) * kAStageBytes;
              const uint32_t piece = kAStageBytes / r.a_split;
              for (int pc = 0; pc < r.a_split; ++pc)
                bulk_g2s_stream(a_st + s * kAStageBytes + pc * piece, src + pc * piece, piece, &fb[s], pol);
            } else {
              tma_load_2d(a_st + s * kAStageBytes, &tw, &fb[s], kbi * kBK, m * kBM, pol);
            }
          } else {
            tma_load_2d(b_st + s * b_stage_bytes, &tx, &fb[s], kbi * kBK, nt * r.n_tile, pol);
          }
          if (is_a && round == 0 && s == 0 && r.timing != nullptr) r.timing[c * 64 + 19] = gtimer();
          if (issued++ == pf_at) {
            const int64_t b0 = range_begin(r.next_iters, c, r.next_grid);
            const int64_t b1 = min(range_begin(r.next_iters, c + 1, r.next_grid), b0 + r.pf_stages);
            for (int64_t t = b0; t < b1; ++t) prefetch_l2(r.next_w + t * kAStageBytes, kAStageBytes);
          }
          if (++s == SS) {
            s = 0;
            ++round;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_bf16(kBM, r.n_tile);
    int i = 0, seg = 0;
    int sa = 0, ra = 0, sb = 0, rb = 0;  // ring slots and their round parities
    SegGen sg(r, c, G);
    int m, nt, kb0, kb1;
    bool skp;
    int64_t lo;
    while (sg.next(r, c, G, m, nt, kb0, kb1, skp, lo)) {
      const int b = seg & 1;
      if (seg >= 2) mbar_wait(&tm_empty[b], ((seg >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + static_cast<uint32_t>(b * r.n_tile);
      for (int kbi = kb0; kbi < kb1; ++kbi, ++i) {
        mbar_wait(&full_a[sa], ra & 1);
        if (i == 0 && r.timing != nullptr && lane == 0) r.timing[c * 64 + 4] = gtimer();
        if (r.dbg_nomma != 2 && !(r.dbg_bres && rb > 0)) mbar_wait(&full_b[sb], rb & 1);
        if (i == 0 && r.timing != nullptr && lane == 0) r.timing[c * 64 + 5] = gtimer();
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(a_st + sa * kAStageBytes);
          const uint32_t b_addr = smem_u32(b_st + sb * b_stage_bytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            if (r.dbg_nomma == 1 || r.dbg_nomma == 2) break;
            if (r.dbg_nomma == 3 && (kbi & 1)) break;  // debug: MMAs on every other stage only
            // Advance along K inside the swizzle atom: 16 bf16 = 32 bytes.
            umma_bf16(acc, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                      (kbi != kb0 || kk != 0) ? 1u : 0u);
          }
          if (r.dbg_nomma == 1 || r.dbg_nomma == 2) {  // debug: pure streaming rate (results are garbage)
            mbar_arrive(&empty_a[sa]);
            if (r.dbg_nomma < 2) mbar_arrive(&empty_b[sb]);
            if (kbi == kb1 - 1) mbar_arrive(&tm_full[b]);
          } else {
            umma_commit(&empty_a[sa]);
            if (!r.dbg_bres) umma_commit(&empty_b[sb]);
            if (kbi == kb1 - 1) umma_commit(&tm_full[b]);
          }
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
    if (r.timing != nullptr && lane == 0) r.timing[c * 64 + 1] = gtimer();
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue
    // Each chunk (32 tokens of the tile) goes TMEM -> registers -> a 16 KiB
    // shared staging buffer -> global by asynchronous bulk copies issued by
    // one leader thread, so no thread ever waits on a global store. Two
    // groups of four warps (one warp per TMEM lane quarter each) take the
    // even and odd chunks, each with its own staging buffer and leader: the
    // epilogue of the last segment -- on the launch's critical path -- runs
    // two chunks at a time.
    grid_dep_wait();  // partials / flags / out may still be in use by the predecessor
    const int eg = (warp - 4) >> 2;  // epilogue group
    const int q = warp & 3;          // TMEM lane quarter this warp may access (warp id % 4)
    const int etid = (threadIdx.x - 128) & (kEpiThreads - 1);
    const int fl = q * 32 + lane;  // feature row of this thread inside the tile
    const bool leader = etid == 0;
    const bool lead0 = leader && eg == 0;
    const bool residual = r.epi == static_cast<int>(Epilogue::kResidualAddF32);
    int seg = 0;
    uint32_t pphase = 0;
    SegGen sg(r, c, G);
    int m, nt, kb0, kb1;
    bool skp;
    int64_t tile_lo;
    uint8_t* st = stage_out + eg * kChunkBytes;  // this group's staging buffer
    while (sg.next(r, c, G, m, nt, kb0, kb1, skp, tile_lo)) {
      const int64_t tile_hi = tile_lo + r.kb;  // stream-K iterations of this tile (skp)
      const bool seg_last = !sg_has_more(sg, r);
      // Whole (data-parallel) tiles need no fixup; residual adds neither:
      // every piece reduce-adds into the fp32 residual stream (order of the
      // <= few pieces is not fixed). Other epilogues are nonlinear or
      // rounding, so stream-K pieces are summed first.
      const bool first = residual || !skp || kb0 == 0;
      const bool last = residual || !skp || kb1 == r.kb;
      const int b = seg & 1;
      const int tok0 = nt * r.n_tile;
      const int nchunk = (r.n_tile + 31) / 32;
      int n_part = 0;
      const float* pstage = reinterpret_cast<const float*>(a_st);  // idle A ring at the last segment
      if (first && !last) {
        // Fixer (always this CTA's last segment): wait for the partners of
        // this tile, then bulk-prefetch all their chunks into the A ring.
        int p_hi = c + 1;
        while (p_hi < G && range_begin(r.sk_iters, p_hi, G) < tile_hi) ++p_hi;
        n_part = p_hi - (c + 1);
        if (lead0)
          for (int p = c + 1; p < p_hi; ++p)
            while (ld_acquire(r.flags + p) != r.epoch) __nanosleep(32);
        if (lead0 && r.timing != nullptr) r.timing[c * 64 + 6] = gtimer();
      }
      const bool rope = first && r.epi == static_cast<int>(Epilogue::kQkvRope);
      const int part = m / max(1, r.qr.H), head = m % max(1, r.qr.H);  // kQkvRope: q/k/v and head of the tile
      if (rope) {
        // token positions and K/V block ids of this tile's tokens, fetched
        // while the MMAs still run (read after the staging barrier below);
        // both groups must have left the previous segment's tables first
        epi_bar_all();
        for (int i = etid; i < r.n_tile; i += kEpiThreads) {
          const int tt = tok0 + i;
          if (tt < r.M) {
            const int pos = r.qr.tok_pos[tt];
            meta_pos[i] = pos;
            if (part > 0) {
              const int rr = r.qr.rowlist[static_cast<int64_t>(r.qr.tok_slot[tt]) * r.qr.max_rows + (pos >> 4)];
              meta_id[i] = r.qr.rowrec[static_cast<int64_t>(rr) * r.qr.row_width + (r.qr.layer * r.qr.H + head) * 2 +
                                       (part - 1)];
            }
          }
        }
      }
      mbar_wait(&tm_full[b], (seg >> 1) & 1);
      tc_fence_after();
      if (lead0 && r.timing != nullptr && seg < 4) r.timing[c * 64 + 9 + seg] = gtimer();
      if (eg >= nchunk) {  // no chunk for this group (n_tile <= 32): hand TMEM back now
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tm_empty[b]);
      }
      if (n_part > 0) {
        // All MMAs of this CTA are complete, so the A ring is idle now.
        if (lead0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          mbar_arrive_expect_tx(pbar, static_cast<uint32_t>(n_part * nchunk * kChunkBytes));
          for (int pi = 0; pi < n_part; ++pi)
            for (int k = 0; k < nchunk; ++k)
              bulk_g2s(a_st + (pi * nchunk + k) * kChunkBytes,
                       r.partials + (static_cast<int64_t>(c + 1 + pi) * 8 + k) * (kChunkBytes / 4), kChunkBytes, pbar);
        }
        mbar_wait(pbar, pphase);
        pphase ^= 1;
        if (lead0 && r.timing != nullptr) r.timing[c * 64 + 7] = gtimer();
      }
      const uint32_t acc = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * r.n_tile);
      for (int k = eg; k < nchunk; k += kEpiGroups) {
        const int cc = k * 32;
        float v[32];
        tmem_ld_32x32b_x32(acc + cc, v);
        const bool stamp = lead0 && r.timing != nullptr && seg_last && k < 4;
        if (stamp) r.timing[c * 64 + 20 + k] = gtimer();
        if (k + kEpiGroups >= nchunk) {  // this group's accumulators consumed: hand TMEM back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tm_empty[b]);
        }
        for (int pi = 0; pi < n_part; ++pi) {  // partner order = CTA order: deterministic
          const float* src = pstage + (pi * nchunk + k) * (kChunkBytes / 4) + fl;
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += src[j * kBM];
        }
        // Staging buffer: wait until the bulk group that last read it is done.
        if (leader) bulk_wait_read<0>();
        epi_bar(eg);
        if (stamp) r.timing[c * 64 + 24 + k] = gtimer();
        const bool silu = first && r.epi == static_cast<int>(Epilogue::kSiluMulBf16);
        const bool fp32_rows = !first || residual || silu || r.epi == static_cast<int>(Epilogue::kStoreF32);
        if (fp32_rows) {
          float* sf = reinterpret_cast<float*>(st);
#pragma unroll
          for (int j = 0; j < 32; ++j) sf[j * kBM + fl] = v[j];
        } else {  // kStoreBf16
          __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(st);
#pragma unroll
          for (int j = 0; j < 32; ++j) sh[j * kBM + fl] = __float2bfloat16_rn(v[j]);
        }
        if (silu) {
          // kSiluMulBf16: feature rows come in (gate_i, up_i) pairs. The fp32
          // chunk is staged first; each thread then turns 16 adjacent pairs of
          // one token into 16 bf16 act[token][i] (no shuffles, all ILP).
          epi_bar(eg);
          const float4* sf4 = reinterpret_cast<const float4*>(st) + (etid >> 2) * (kBM / 4) + (etid & 3) * 8;
          uint32_t packed[8];
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) {
            const float4 gu = sf4[q2];  // gate, up, gate, up
            const float s0 = gu.x / (1.f + expf(-gu.x));
            const float s1 = gu.z / (1.f + expf(-gu.z));
            packed[q2] = pack_bf16(s0 * gu.y, s1 * gu.w);
          }
          epi_bar(eg);
          uint4* dst = reinterpret_cast<uint4*>(st + (etid >> 2) * kBM + (etid & 3) * 32);
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
        if (rope) {
          // K2 fused: thread = (token jj of the chunk, dims [d0, d0+16) and
          // their rotate_half partners d0+64..); the same _rn arithmetic as
          // kv_append, on the same bf16-rounded values.
          epi_bar(eg);
          const int jj = etid >> 2, d0 = (etid & 3) * 16;
          const int tt = tok0 + cc + jj;
          if (tt < r.M) {
            __nv_bfloat16* rowp = reinterpret_cast<__nv_bfloat16*>(st) + jj * kBM;
            uint4 lo4[2] = {reinterpret_cast<uint4*>(rowp + d0)[0], reinterpret_cast<uint4*>(rowp + d0)[1]};
            uint4 hi4[2] = {reinterpret_cast<uint4*>(rowp + 64 + d0)[0], reinterpret_cast<uint4*>(rowp + 64 + d0)[1]};
            const int pos = meta_pos[cc + jj];
            if (part < 2) {
              const float* cs = r.qr.rope + static_cast<int64_t>(min(pos, r.qr.rope_positions - 1)) * 128;
              uint32_t* lw = reinterpret_cast<uint32_t*>(lo4);
              uint32_t* hw = reinterpret_cast<uint32_t*>(hi4);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float l0 = bf16_lo(lw[i]), l1 = bf16_hi(lw[i]), h0 = bf16_lo(hw[i]), h1 = bf16_hi(hw[i]);
                const float c0 = cs[2 * (d0 + 2 * i)], s0 = cs[2 * (d0 + 2 * i) + 1];
                const float c1 = cs[2 * (d0 + 2 * i + 1)], s1 = cs[2 * (d0 + 2 * i + 1) + 1];
                lw[i] = pack_bf16(__fsub_rn(__fmul_rn(l0, c0), __fmul_rn(h0, s0)),
                                  __fsub_rn(__fmul_rn(l1, c1), __fmul_rn(h1, s1)));
                hw[i] = pack_bf16(__fadd_rn(__fmul_rn(h0, c0), __fmul_rn(l0, s0)),
                                  __fadd_rn(__fmul_rn(h1, c1), __fmul_rn(l1, s1)));
              }
              reinterpret_cast<uint4*>(rowp + d0)[0] = lo4[0];
              reinterpret_cast<uint4*>(rowp + d0)[1] = lo4[1];
              reinterpret_cast<uint4*>(rowp + 64 + d0)[0] = hi4[0];
              reinterpret_cast<uint4*>(rowp + 64 + d0)[1] = hi4[1];
            }
            __nv_bfloat16* dst;
            if (part == 0) {
              dst = reinterpret_cast<__nv_bfloat16*>(r.qr.q_out) + (static_cast<int64_t>(tt) * r.qr.H + head) * 128;
            } else {
              dst = reinterpret_cast<__nv_bfloat16*>(static_cast<uint8_t*>(r.qr.pool) +
                                                     static_cast<int64_t>(meta_id[cc + jj]) * 4096 + (pos & 15) * 256);
            }
            reinterpret_cast<uint4*>(dst + d0)[0] = lo4[0];
            reinterpret_cast<uint4*>(dst + d0)[1] = lo4[1];
            reinterpret_cast<uint4*>(dst + 64 + d0)[0] = hi4[0];
            reinterpret_cast<uint4*>(dst + 64 + d0)[1] = hi4[1];
          }
        }
        fence_async_smem();
        epi_bar(eg);
        if (leader) {
          if (!first) {
            // partner: publish the whole chunk (fixed slot of this CTA)
            bulk_s2g(r.partials + (static_cast<int64_t>(c) * 8 + k) * (kChunkBytes / 4), st, kChunkBytes);
          } else if (residual) {
            tma_reduce_add_2d(&tout, st, m * kBM, tok0 + cc);  // rows >= M are clipped by TMA
          } else if (silu) {
            tma_store_2d(&tout, st, m * (kBM / 2), tok0 + cc);
          } else {
            tma_store_2d(&tout, st, m * kBM, tok0 + cc);
            for (int pr = 0; pr < r.n_peers; ++pr) tma_store_2d(&peers.m[pr], st, m * kBM, tok0 + cc);
          }
          bulk_commit();
          if (stamp) r.timing[c * 64 + 28 + k] = gtimer();
        }
      }
      if (!first) {  // publish: both groups' partial bulk writes complete, then the flag
        if (leader) bulk_wait<0>();
        epi_bar_all();
        if (lead0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_release(r.flags + c, r.epoch);
          if (r.timing != nullptr) r.timing[c * 64 + 8] = gtimer();
        }
      }
      if (lead0 && r.timing != nullptr && seg < 4) r.timing[c * 64 + 16 + seg] = gtimer();
      ++seg;
    }
    // Staging smem must outlive the bulk stores' reads of it; completion of
    // the writes themselves is only needed before a signal to the TP peers
    // (dependent kernels see them through grid completion).
    if (leader) {
      if (r.n_signal > 0) bulk_wait<0>();
      else bulk_wait_read<0>();
    }
    if (r.n_signal > 0) epi_bar_all();  // both groups' stores have landed
    if (r.norm_w != nullptr) {
      // Fused RMSNorm: wait until every CTA's reduce-adds into the residual
      // have landed (grid barrier: all CTAs are co-resident on an exclusive
      // partition), then normalise this CTA's share of the token rows.
      if (leader) bulk_wait<0>();
      epi_bar_all();
      if (lead0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(r.norm_bar, 1u);
        while (static_cast<int>(static_cast<unsigned>(ld_acquire(reinterpret_cast<const int*>(r.norm_bar))) -
                                r.norm_target) < 0)
          __nanosleep(64);
      }
      epi_bar_all();
      const int nt4 = r.N / 4;  // float4s per row (N = hidden)
      const int t0 = static_cast<int>(static_cast<int64_t>(r.M) * c / G);
      const int t1 = static_cast<int>(static_cast<int64_t>(r.M) * (c + 1) / G);
      const int et = threadIdx.x - 128;  // 0..255 over both groups
      for (int t = t0; t < t1; ++t) {
        const float4* x = reinterpret_cast<const float4*>(static_cast<const float*>(r.out) +
                                                          static_cast<int64_t>(t) * r.ldo);
        float ss = 0.f;
        for (int i = et; i < nt4; i += kEpiGroups * kEpiThreads) {
          const float4 v = __ldcg(x + i);
          ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) norm_red[warp - 4] = ss;
        epi_bar_all();
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < kEpiGroups * kEpiThreads / 32; ++w) tot += norm_red[w];
        const float inv = rsqrtf(tot / static_cast<float>(r.N) + r.norm_eps);
        uint2* y = reinterpret_cast<uint2*>(r.norm_out + static_cast<int64_t>(t) * r.N);
        const float4* g = reinterpret_cast<const float4*>(r.norm_w);
        for (int i = et; i < nt4; i += kEpiGroups * kEpiThreads) {
          const float4 v = __ldcg(x + i);
          const float4 gw = g[i];
          y[i] = make_uint2(pack_bf16(v.x * inv * gw.x, v.y * inv * gw.y), pack_bf16(v.z * inv * gw.z, v.w * inv * gw.w));
        }
        epi_bar_all();  // norm_red is reused by the next row
      }
    }
    if (lead0 && r.n_signal > 0) {
      // every store of this CTA (local + peers) has completed: publish
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int d = 0; d < r.n_signal; ++d)
        asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(r.signal[d]) : "memory");
    }
    if (r.timing != nullptr && threadIdx.x == 128) r.timing[c * 64 + 2] = gtimer();
  }
  // Reconverge the role warps (elected producer / MMA lanes) before the
  // block barrier: a diverged warp would arrive early and let warp 2 free
  // TMEM while the epilogue still reads it.
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (r.timing != nullptr && threadIdx.x == 0) r.timing[c * 64 + 3] = gtimer();
  if (r.timing != nullptr && threadIdx.x == 128) r.timing[c * 64 + 13] = gtimer();
  if (r.timing != nullptr && threadIdx.x == 32) r.timing[c * 64 + 14] = gtimer();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, r.tmem_cols);
  }
}

// Row-major [N][K] bf16 -> [m_tile][k_block][128 rows][128 B] with the
// 128-byte swizzle applied (16-B chunk c of row r stored at chunk c ^ (r & 7)),
// i.e. exactly the shared-memory image a SWIZZLE_128B TMA box would produce.
// Rows / columns past N / K are zero. One thread per 16-byte chunk.
__global__ void weight_tile_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int N, int K,
                                   int kb, int64_t chunks, bool inverse) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < chunks; i += stride) {
    const int c = static_cast<int>(i & 7);
    const int64_t rest = i >> 3;
    const int r = static_cast<int>(rest & 127);
    const int64_t tile = rest >> 7;
    const int kbi = static_cast<int>(tile % kb);
    const int64_t m = tile / kb;
    const int64_t row = m * kBM + r;
    const int64_t col = static_cast<int64_t>(kbi) * kBK + c * 8;
    const int64_t d = (tile * 128 + r) * 8 + (c ^ (r & 7));
    const bool in = row < N && col < K;
    if (!inverse) {
      dst[d] = in ? src[(row * K + col) / 8] : make_uint4(0, 0, 0, 0);
    } else if (in) {
      dst[(row * K + col) / 8] = src[d];
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

uint32_t pow2_cols(int n) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(n)) c <<= 1;
  return c;
}

}  // namespace

bool make_tmap_bf16(void* tmap_out, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_stride_bytes, uint32_t box_rows) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = fn(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

bool make_tmap_2d(void* tmap_out, const void* base, bool fp32, uint64_t rows, uint64_t cols,
                  uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = fn(reinterpret_cast<CUtensorMap*>(tmap_out),
                    fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

bool make_tmap_gemm_out(void* tmap_out, const void* out, int epi, int M, int N, int ldo) {
  const bool fp32 = epi == static_cast<int>(Epilogue::kResidualAddF32) || epi == static_cast<int>(Epilogue::kStoreF32);
  const bool silu = epi == static_cast<int>(Epilogue::kSiluMulBf16);
  const uint64_t cols = silu ? static_cast<uint64_t>(N / 2) : static_cast<uint64_t>(N);
  const uint64_t stride = static_cast<uint64_t>(ldo) * (fp32 ? 4 : 2);
  return make_tmap_2d(tmap_out, out, fp32, static_cast<uint64_t>(M), cols, stride, 32, silu ? kBM / 2 : kBM);
}

int gemm_pick_n_tile(int M) {
  int n = ((M + 15) / 16) * 16;
  if (n > 256) n = 256;
  if (n < 16) n = 16;
  return n;
}

size_t gemm_partials_floats(int max_grid) { return static_cast<size_t>(max_grid) * 8 * (kChunkBytes / 4); }

size_t weight_tiled_bytes(int N, int K) {
  return static_cast<size_t>((N + kBM - 1) / kBM) * ((K + kBK - 1) / kBK) * kAStageBytes;
}

cudaError_t weight_tile(const void* src, int N, int K, void* dst, bool inverse, cudaStream_t stream) {
  if (K % 8 != 0) return cudaErrorInvalidValue;
  const int kb = (K + kBK - 1) / kBK;
  const int64_t chunks = static_cast<int64_t>(weight_tiled_bytes(N, K)) / 16;
  const int blocks = static_cast<int>(std::min<int64_t>((chunks + 255) / 256, 148 * 16));
  if (!inverse)
    weight_tile_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint4*>(src),
                                                   reinterpret_cast<uint4*>(dst), N, K, kb, chunks, false);
  else
    weight_tile_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const uint4*>(src),
                                                   reinterpret_cast<uint4*>(dst), N, K, kb, chunks, true);
  return cudaGetLastError();
}

cudaError_t preload_gemm() { return preload(gemm_tn_kernel, weight_tile_kernel); }

static unsigned long long* g_debug_timing = nullptr;
void gemm_debug_timing(void* buf) { g_debug_timing = static_cast<unsigned long long*>(buf); }

// Tiling, pipeline depths, grid and schedule of one launch (no side effects).
static void plan(const GemmArgs& a, GemmRun& r, int& grid_out, size_t& smem_out) {
  r.w_tiled = static_cast<const uint8_t*>(a.w_tiled);
  r.timing = g_debug_timing;
  r.out = a.out;
  r.partials = a.partials;
  r.flags = a.flags;
  r.epoch = a.epoch;
  r.M = a.M;
  r.N = a.N;
  r.K = a.K;
  r.ldo = a.ldo;
  r.n_tile = gemm_pick_n_tile(a.M);
  const int b_stage = r.n_tile * kBK * 2;
  r.stages_b = r.n_tile > 128 ? 2 : 3;
  // Debug overrides for pipeline-depth sweeps (scripts/gemm_micro.py).
  static const int env_sb = getenv("MUX_GEMM_SB") ? atoi(getenv("MUX_GEMM_SB")) : 0;
  static const int env_sa = getenv("MUX_GEMM_SA") ? atoi(getenv("MUX_GEMM_SA")) : 0;
  if (env_sb > 0) r.stages_b = env_sb;
  static const int env_split = getenv("MUX_GEMM_ASPLIT") ? atoi(getenv("MUX_GEMM_ASPLIT")) : 1;
  r.a_split = (env_split == 2 || env_split == 4 || env_split == 8) ? env_split : 1;
  static const int env_nomma = getenv("MUX_GEMM_NOMMA") ? atoi(getenv("MUX_GEMM_NOMMA")) : 0;
  r.dbg_nomma = env_nomma;
  static const int env_bres = getenv("MUX_GEMM_BRES") ? atoi(getenv("MUX_GEMM_BRES")) : 0;
  r.dbg_bres = env_bres;
  const int meta_bytes = a.epi == Epilogue::kQkvRope ? 2 * 256 * 4 : 0;  // token positions + block ids
  static const int env_stg = getenv("MUX_GEMM_STG") ? atoi(getenv("MUX_GEMM_STG")) : 2;
  static const int env_budget = getenv("MUX_GEMM_SMEM_KB") ? atoi(getenv("MUX_GEMM_SMEM_KB")) * 1024 : kSmemBudget;
  r.n_stg = 2;  // one staging buffer per epilogue group
  (void)env_stg;
  r.stages_a = (env_budget - meta_bytes - r.stages_b * b_stage - r.n_stg * kChunkBytes) / kAStageBytes;
  if (env_sa > 0) r.stages_a = std::min(env_sa, r.stages_a);
  else if (r.stages_a > 10) r.stages_a = 10;
  // The fixer prefetches up to 2 partners x ceil(n_tile/32) chunks into the A ring.
  r.kb = (a.K + kBK - 1) / kBK;
  r.m_tiles = (a.N + kBM - 1) / kBM;
  const int n_tiles_tok = (a.M + r.n_tile - 1) / r.n_tile;
  r.iters = static_cast<int64_t>(r.m_tiles) * n_tiles_tok * r.kb;
  r.epi = static_cast<int>(a.epi);
  r.qr = a.qkv;
  r.n_tok_tiles = n_tiles_tok;
  r.tmem_cols = pow2_cols(r.n_tile + (r.n_tile > 32 ? r.n_tile : 32));
  int grid = a.grid > 0 ? a.grid : 148;
  // Enough k-blocks per CTA that the fixed per-CTA cost and the fixup
  // partials stay small next to the weight bytes it streams.
  int64_t min_iters = a.min_iters > 0 ? a.min_iters : 1;
  // Residual epilogues reduce-add their pieces (no fixup): keep the whole
  // machine streaming even for small projections (O of 7B: 2048 k-blocks).
  static const int env_rmin = getenv("MUX_GEMM_RES_MIN_ITERS") ? atoi(getenv("MUX_GEMM_RES_MIN_ITERS")) : 8;
  if (a.epi == Epilogue::kResidualAddF32) min_iters = std::min<int64_t>(min_iters, env_rmin);
  if (static_cast<int64_t>(grid) * min_iters > r.iters) grid = static_cast<int>(std::max<int64_t>(1, r.iters / min_iters));
  // Non-residual epilogues sum pieces in a fixer: keep every tile in <= 3
  // pieces (<= 2 partners) so their chunks fit the idle A ring.
  if (r.epi != static_cast<int>(Epilogue::kResidualAddF32)) {
    const int nchunk = (r.n_tile + 31) / 32;
    const int max_partners = (r.stages_a * kAStageBytes) / (nchunk * kChunkBytes);
    // a range of R iterations lets a tile meet at most ceil(kb / R) + 1 ranges
    const int64_t need_r = (r.kb + max_partners - 1) / std::max(1, max_partners);
    if (static_cast<int64_t>(grid) * need_r > r.iters) grid = static_cast<int>(std::max<int64_t>(1, r.iters / need_r));
  }
  // Schedule: decode (one token tile) = pure stream-K; prefill = grouped
  // data-parallel rounds + stream-K over the last 1-2 waves of tiles (so
  // every stream-K range spans >= one tile's k-blocks: <= 2 partners).
  static const int env_group = getenv("MUX_GEMM_GROUP_M") ? atoi(getenv("MUX_GEMM_GROUP_M")) : 8;
  const int64_t tiles = static_cast<int64_t>(r.m_tiles) * n_tiles_tok;
  if (n_tiles_tok > 1 && env_group > 0) {
    r.n_dp = static_cast<int>(std::max<int64_t>(0, tiles / grid - 1));
    r.group_m = env_group;
  } else {
    r.n_dp = 0;
    r.group_m = 0;
  }
  r.sk_iters = (tiles - static_cast<int64_t>(r.n_dp) * grid) * r.kb;
  smem_out = 1024 + static_cast<size_t>(r.stages_a) * kAStageBytes + static_cast<size_t>(r.stages_b) * b_stage +
             r.n_stg * kChunkBytes + (2 * (r.stages_a + r.stages_b) + 6) * 8 + 16 + std::max(meta_bytes, 64);
  grid_out = grid;
}

cudaError_t gemm_bf16_tn(const GemmArgs& a, cudaStream_t stream) {
  if (a.M <= 0 || a.N <= 0) return cudaSuccess;
  if (gemm_2sm_eligible(a)) return gemm_2sm(a, stream);
  // tmap_x must have been encoded with box rows == gemm_pick_n_tile(M).
  GemmRun r{};
  int grid = 0;
  size_t smem = 0;
  plan(a, r, grid, smem);
  // device index math is 32-bit (range_begin): iters * (grid + 1) must fit
  if (static_cast<uint64_t>(r.iters) * static_cast<uint64_t>(grid + 1) >= (1ull << 32)) return cudaErrorInvalidValue;
  if (a.next_w != nullptr && a.pf_stages > 0 && r.n_tok_tiles == 1) {
    // the next decode GEMM of the chain: same tokens, same partition
    GemmArgs na = a;
    na.N = a.next_N;
    na.K = a.next_K;
    na.epi = a.next_epi;
    GemmRun nr{};
    int ngrid = 0;
    size_t nsmem = 0;
    plan(na, nr, ngrid, nsmem);
    if (static_cast<uint64_t>(nr.iters) * static_cast<uint64_t>(ngrid + 1) >= (1ull << 32)) return cudaErrorInvalidValue;
    r.next_w = static_cast<const uint8_t*>(a.next_w);
    r.next_grid = ngrid;
    r.next_iters = nr.sk_iters;
    r.pf_stages = a.pf_stages;
  }
  if (a.norm_w != nullptr) {
    // decode residual GEMMs only: one token tile, the whole grid co-resident
    if (a.epi != Epilogue::kResidualAddF32 || r.n_tok_tiles != 1 || a.norm_bar == nullptr || a.N % 4 != 0)
      return cudaErrorInvalidValue;
    r.norm_w = a.norm_w;
    r.norm_out = static_cast<__nv_bfloat16*>(a.norm_out);
    r.norm_bar = a.norm_bar;
    r.norm_target = a.norm_base + static_cast<unsigned>(grid);
    r.norm_eps = a.norm_eps;
  }
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run(
      [] { return cudaFuncSetAttribute(gemm_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448); });
  if (ce != cudaSuccess) return ce;
  r.n_peers = a.n_peers;
  r.n_signal = a.n_signal;
  for (int d = 0; d < kMaxTp; ++d) r.signal[d] = a.signal[d];
  PeerMaps pm;
  std::memset(&pm, 0, sizeof(pm));
  for (int d = 0; d < a.n_peers; ++d) std::memcpy(&pm.m[d], a.tmap_peers[d], sizeof(CUtensorMap));
  CUtensorMap tw, tx, to;
  if (a.tmap_w != nullptr) std::memcpy(&tw, a.tmap_w, sizeof(CUtensorMap));
  else std::memset(&tw, 0, sizeof(CUtensorMap));
  std::memcpy(&tx, a.tmap_x, sizeof(CUtensorMap));
  std::memcpy(&to, a.tmap_out, sizeof(CUtensorMap));
  if (a.grid_out != nullptr) *a.grid_out = grid;
  return launch(gemm_tn_kernel, dim3(grid), dim3(kThreads), smem, stream, tw, tx, to, r, pm);
}

}  // namespace mux
