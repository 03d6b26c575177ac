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
// Decode forms (plan()): token tiles of 16..256 run on CTA PAIRS (template
// PAIR: clusters of two, one tcgen05.mma.cta_group::2 of M = 256 per
// k-block, each CTA staging its 128 weight rows and half the token tile);
// single-CTA launches with many units per CTA stage two 128-row weight tiles
// per activation stage (st = 2); token tiles of <= 64 that pairs cannot take
// run two CTAs per SM (EG = 1) so the next projection's CTAs stream under PDL.
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
// Warps 0-3: roles; then EG epilogue groups of four warps. EG = 2 (one CTA
// per SM, the big ring) for decode batches above 64 tokens; EG = 1 with a
// <= 113 KB ring for smaller batches, so TWO GEMM CTAs fit one SM: under PDL
// the next projection's CTAs start streaming their weights while this one
// drains, and colocated models' GEMMs on different streams co-reside.
template <int EG>
constexpr int threads_of() { return 128 + EG * 128; }
constexpr int kEpiThreads = 128;            // one epilogue group: a warp per TMEM lane quarter
constexpr int kChunkBytes = 32 * kBM * 4;  // one epilogue chunk: 32 tokens x 128 fp32
constexpr int kSmemBudget = 224 * 1024;     // A ring + B ring + 2 staging chunks
constexpr int kDualSmemBudget = 110 * 1024;  // EG = 1: rings + staging of one of two CTAs per SM
constexpr int kPreIssue = 2;                // weight stages issued before the block barrier

struct PeerMaps {
  CUtensorMap m[kMaxTp - 1];
};

struct GemmRun {
  const uint8_t* w_tiled;  // pre-tiled weights (weight_tile), or null -> TMA map
  void* out;
  float* partials;  // [grid][2 slots][8 chunks][32 x 128] fp32
  int* flags;       // [grid][2 slots]
  int epoch;
  int M, N, K, ldo;
  int n_tile, stages_a, stages_b;
  int kb;           // k-blocks per tile
  int m_tiles;      // ceil(N / 128) / st: weight units along N
  int st;           // 128-row weight tiles per unit (2: one activation stage feeds two MMAs)
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
  unsigned long long* timing;  // debug: [grid][64] globaltimer stamps, or null
  int dbg_nomma;    // debug (MUX_GEMM_NOMMA=1): stream operands without MMAs
  int eg;           // epilogue groups of the instantiation (template EG)
  int pair;         // CTA-pair mode (template PAIR): 256-row units, cta_group::2 MMAs
  // Tensor-parallel fan-out (kStoreF32 only): every finished tile is also
  // stored through peers.m[0..n_peers) (the same slot on the other ranks of
  // the mesh, NVLink peer memory), and once all of a CTA's stores have landed
  // it adds 1 to signal[0..n_signal) (this rank's and every peer's counter).
  int n_peers;
  int n_signal;
  int* signal[kMaxTp];
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

// The CTA whose stream-K range holds iteration `it` (ranges are contiguous
// and ascending; start the search at a CTA known to be close).
__device__ __forceinline__ int cta_of(int64_t iters, int64_t it, int hint, int G) {
  int a = hint;
  while (a > 0 && range_begin(iters, a, G) > it) --a;
  while (a + 1 < G && range_begin(iters, a + 1, G) <= it) ++a;
  return a;
}

// The work of one CTA as a sequence of segments: (tile, k-block range); the
// same sequence is walked by the producers, the MMA issuer and the epilogue.
//
// Stream-K pieces and who finishes a cut tile. A tile cut into P pieces
// (CTAs a..b, P = b - a + 1) is finished by one "fixer": a for P = 2 (the
// tile's first piece is a's LAST segment, so a reaches it last and its
// partner b published the tile's end as b's FIRST segment), a + 1 for P >= 3
// (a middle CTA whose whole range lies inside the tile: it has nothing else
// to do, so it should not be the one others wait for). For P >= 3 the first
// piece is again a's last segment; a walks it FIRST (rot_lo / rot_hi) so
// that partial is published early too. Partners publish into slot 1 (a's
// rotated first piece) or slot 0 (the piece at the start of their range):
// every publish precedes every wait inside a CTA, and a CTA waits only as
// the fixer of its last segment, so no cycle can form.
struct SegGen {
  int64_t sk, sk_end;      // stream-K iterations walked in order
  int64_t rot_lo, rot_hi;  // walked first when rot_lo < rot_hi
  int j;
  __device__ SegGen(const GemmRun& r, int c, int G)
      : sk(range_begin(r.sk_iters, c, G)), sk_end(range_begin(r.sk_iters, c + 1, G)), rot_lo(0), rot_hi(0), j(0) {
    if (r.epi != static_cast<int>(Epilogue::kResidualAddF32) && sk_end > sk && c + 2 <= G) {
      const int64_t last_lo = static_cast<int64_t>(static_cast<uint32_t>(sk_end - 1) / static_cast<uint32_t>(r.kb)) * r.kb;
      if (last_lo > sk && sk_end < last_lo + r.kb && range_begin(r.sk_iters, c + 2, G) < last_lo + r.kb) {
        rot_lo = last_lo;
        rot_hi = sk_end;
        sk_end = last_lo;
      }
    }
  }
  // tile (m, nt), k-blocks [kb0, kb1); skp: stream-K piece of the tile whose
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
      int64_t s0, e;
      if (rot_lo < rot_hi) {
        s0 = rot_lo;
        e = rot_hi;
        rot_hi = rot_lo;  // consumed
      } else {
        if (sk >= sk_end) return false;
        s0 = sk;
        const int64_t t0 = static_cast<int64_t>(static_cast<uint32_t>(s0) / static_cast<uint32_t>(r.kb)) * r.kb;
        e = min(sk_end, t0 + r.kb);
        sk = e;
      }
      const int64_t st = static_cast<uint32_t>(s0) / static_cast<uint32_t>(r.kb);
      lo = st * r.kb;
      kb0 = static_cast<int>(s0 - lo);
      kb1 = static_cast<int>(e - lo);
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
  __device__ bool has_more(const GemmRun& r) const { return j < r.n_dp || rot_lo < rot_hi || sk < sk_end; }
};

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
template <int EG>
__device__ __forceinline__ void epi_bar_all() {
  if constexpr (EG == 1) asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
  else asm volatile("bar.sync 3, %0;" ::"n"(2 * kEpiThreads) : "memory");
}

#define STAMP(cond, slot) \
  do { if (r.timing != nullptr && (cond)) r.timing[c * 64 + (slot)] = gtimer(); } while (0)

// PAIR: the CTAs of a cluster pair (one TPC) share each 256-row weight unit:
// each stages its own 128 weight rows and HALF of the token tile, and the
// leader's single tcgen05.mma.cta_group::2 (M = 256) reads the token operand
// from both CTAs' shared memory. Per SM that stages and reads half the
// activation bytes of the single-CTA form: 48 instead of 64 KiB of shared-
// memory traffic per 16 KiB of weights (the MMAs' operand reads stall the
// weight stream near the 128 B/clk port limit at 128 tokens). Stream-K runs
// over pairs; each rank fixes up / publishes its own 128-row half.
template <int EG, bool PAIR>
__global__ void __launch_bounds__(threads_of<EG>(), 3 - EG)
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
  const int b_stage_bytes = (PAIR ? r.n_tile / 2 : r.n_tile) * kBK * 2;  // pair: this CTA's token half
  uint8_t* a_st = base;
  const int a_stage_bytes = r.st * kAStageBytes;  // st weight tiles of one k-block
  uint8_t* b_st = base + SA * a_stage_bytes;
  uint8_t* stage_out = b_st + SB * b_stage_bytes;  // 2 x 16 KiB epilogue staging
  constexpr int kEpiGroups = EG;
  uint64_t* full_a = reinterpret_cast<uint64_t*>(stage_out + kEpiGroups * kChunkBytes);
  uint64_t* empty_a = full_a + SA;
  uint64_t* full_b = empty_a + SA;
  uint64_t* empty_b = full_b + SB;
  uint64_t* tm_full = empty_b + SB;  // [2]
  uint64_t* tm_empty = tm_full + 2;  // [2]
  uint64_t* pbar = tm_empty + 2;     // fixer's partial prefetch
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // stream-K participant: the CTA, or the CTA pair in PAIR mode
  const int rank = PAIR ? static_cast<int>(cluster_rank()) : 0;
  const int c = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int G = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // flags / partials slot of participant p's CTA of this rank
  auto pid = [&](int p) { return PAIR ? 2 * p + rank : p; };
  const int me = pid(c);
  STAMP(threadIdx.x == 0, 0);

  // Weight producer state (warp 0, lane 0). Weights do not depend on earlier
  // kernels, so the first stages are issued right after the barriers are
  // initialised -- beside TMEM allocation, before the block barrier -- and
  // under PDL while the predecessor drains (only kPreIssue: every issue
  // costs ~0.2 us, which the rest of the CTA would wait for at the barrier).
  SegGen pg(r, c, G);
  int pm = 0, pkb = 0, pkb1 = 0, ps = 0, pround = 0;
  bool pvalid = false;
  uint64_t wpol = 0;
  auto a_next = [&]() -> bool {
    if (pvalid && ++pkb < pkb1) return true;
    int nt, kb0;
    bool skp;
    int64_t lo;
    pvalid = pg.next(r, c, G, pm, nt, kb0, pkb1, skp, lo);
    pkb = kb0;
    return pvalid;
  };
  auto a_issue = [&]() {
    if (pround > 0) mbar_wait(&empty_a[ps], (pround - 1) & 1);
    if constexpr (PAIR) {
      // both CTAs' 16 KiB count on the leader's barrier; the tiled weights
      // are a [tiles * 128][64] tensor (rows already in the SW128 image)
      if (rank == 0) mbar_arrive_expect_tx(&full_a[ps], 2u * kAStageBytes);
      const int mt = 2 * pm + rank;
      tma_load_2d_pair(a_st + ps * kAStageBytes, &tw, map_to_rank(smem_u32(&full_a[ps]), 0), 0,
                       (mt * r.kb + pkb) * kBM, wpol);
      if (++ps == SA) {
        ps = 0;
        ++pround;
      }
      return;
    }
    mbar_arrive_expect_tx(&full_a[ps], static_cast<uint32_t>(a_stage_bytes));
    for (int j = 0; j < r.st; ++j) {
      const int mt = pm * r.st + j;  // 128-row weight tile
      uint8_t* dst = a_st + ps * a_stage_bytes + j * kAStageBytes;
      if (r.w_tiled != nullptr)  // one contiguous, pre-swizzled 16 KiB UMMA tile
        bulk_g2s_stream(dst, r.w_tiled + (static_cast<int64_t>(mt) * r.kb + pkb) * kAStageBytes, kAStageBytes,
                        &full_a[ps], wpol);
      else
        tma_load_2d(dst, &tw, &full_a[ps], pkb * kBK, mt * kBM, wpol);
    }
    if (++ps == SA) {
      ps = 0;
      ++pround;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
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
        // the leader's counts both CTAs' epilogue warps in PAIR mode
        mbar_init(&tm_empty[b], (PAIR ? 2 : 1) * kEpiGroups * kEpiThreads / 32);
      }
      mbar_init(pbar, 1);
      fence_barrier_init();
      wpol = policy_evict_first();  // weights: streamed once per step
      STAMP(true, 32);
      // (PAIR: the peer's copies complete on the leader's barriers, so none
      // is issued before the cluster barrier below)
      if constexpr (!PAIR)
        for (int k = 0; k < kPreIssue && a_next(); ++k) a_issue();
      STAMP(true, 19);
      if (r.w_tiled == nullptr) prefetch_tmap(&tw);
      prefetch_tmap(&tx);
      prefetch_tmap(&tout);
    }
    __syncwarp();
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(r.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc_dyn(tmem_slot, r.tmem_cols);
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  STAMP(threadIdx.x == 0, 15);
  if (threadIdx.x == 0) grid_dep_launch();

  if (warp == 0) {
    // ------------------------------------------------ weight producer
    if (lane == 0)
      while (a_next()) a_issue();
    __syncwarp();
  } else if (warp == 3) {
    // -------------------------------------------- activation producer
    if (elect_one()) {
      grid_dep_wait();  // activations come from the predecessor
      const uint64_t pol = policy_evict_last();  // re-read by every CTA
      const uint32_t bytes = static_cast<uint32_t>(b_stage_bytes);
      const uint32_t full_b_leader = PAIR ? map_to_rank(smem_u32(full_b), 0) : 0u;
      SegGen sg(r, c, G);
      int m, nt, kb0, kb1;
      bool skp;
      int64_t lo;
      int s = 0, round = 0;
      while (sg.next(r, c, G, m, nt, kb0, kb1, skp, lo)) {
        for (int kbi = kb0; kbi < kb1; ++kbi) {
          if (round > 0) mbar_wait(&empty_b[s], (round - 1) & 1);
          if constexpr (PAIR) {
            if (rank == 0) mbar_arrive_expect_tx(&full_b[s], 2 * bytes);
            tma_load_2d_pair(b_st + s * b_stage_bytes, &tx, full_b_leader + s * 8, kbi * kBK,
                             nt * r.n_tile + rank * (r.n_tile / 2), pol);
          } else {
            mbar_arrive_expect_tx(&full_b[s], bytes);
            tma_load_2d(b_st + s * b_stage_bytes, &tx, &full_b[s], kbi * kBK, nt * r.n_tile, pol);
          }
          if (++s == SB) {
            s = 0;
            ++round;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 && (!PAIR || rank == 0)) {
    // ------------------------------------------------------ MMA issuer
    // (PAIR: the leader issues one M = 256 MMA for both CTAs)
    const uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * kBM : kBM, r.n_tile);
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
      const uint32_t acc = tmem + static_cast<uint32_t>(b * r.st * r.n_tile);
      for (int kbi = kb0; kbi < kb1; ++kbi, ++i) {
        mbar_wait(&full_a[sa], ra & 1);
        STAMP(i == 0 && lane == 0, 4);
        mbar_wait(&full_b[sb], rb & 1);
        STAMP(i == 0 && lane == 0, 5);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(a_st + sa * a_stage_bytes);
          const uint32_t b_addr = smem_u32(b_st + sb * b_stage_bytes);
          if constexpr (PAIR) {
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma2_bf16(acc, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                         (kbi != kb0 || kk != 0) ? 1u : 0u);
            umma2_commit_both(&empty_a[sa]);
            umma2_commit_both(&empty_b[sb]);
            if (kbi == kb1 - 1) umma2_commit_both(&tm_full[b]);
          } else if (r.dbg_nomma) {  // debug: pure streaming rate (results are garbage)
            mbar_arrive(&empty_a[sa]);
            mbar_arrive(&empty_b[sb]);
            if (kbi == kb1 - 1) mbar_arrive(&tm_full[b]);
          } else {
            for (int j = 0; j < r.st; ++j)  // st weight tiles share this activation stage
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk)  // along K inside the swizzle atom: 16 bf16 = 32 bytes
                umma_bf16(acc + static_cast<uint32_t>(j * r.n_tile), umma_desc_sw128(a_addr + j * kAStageBytes + kk * 32),
                          umma_desc_sw128(b_addr + kk * 32), idesc, (kbi != kb0 || kk != 0) ? 1u : 0u);
            umma_commit(&empty_a[sa]);
            umma_commit(&empty_b[sb]);
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
    STAMP(lane == 0, 1);
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
    const bool silu = r.epi == static_cast<int>(Epilogue::kSiluMulBf16);
    int seg = 0;
    uint32_t pphase = 0;
    SegGen sg(r, c, G);
    int m, nt, kb0, kb1;
    bool skp;
    int64_t tile_lo;
    uint8_t* st = stage_out + eg * kChunkBytes;  // this group's staging buffer
    const float* pstage = reinterpret_cast<const float*>(a_st);  // fixer: the idle A ring at its last segment
    while (sg.next(r, c, G, m, nt, kb0, kb1, skp, tile_lo)) {
      const bool seg_last = !sg.has_more(r);
      // Role of this piece. Residual epilogues reduce-add every piece into
      // the fp32 residual stream (order of the <= few pieces is not fixed);
      // the others are nonlinear or rounding, so the pieces are summed in a
      // fixed order by the tile's fixer (see SegGen).
      int pa = c, pb = c, fix = c;
      if (skp && !residual) {
        pa = kb0 == 0 ? c : cta_of(r.sk_iters, tile_lo, c, G);
        pb = kb1 == r.kb ? c : cta_of(r.sk_iters, tile_lo + r.kb - 1, c, G);
        fix = pb - pa <= 1 ? pa : pa + 1;  // pa == pb: the whole tile in one piece
      }
      const bool partner = c != fix;
      const int n_part = partner ? 0 : pb - pa;
      const int b = seg & 1;
      const int tok0 = nt * r.n_tile;
      const int nct = (r.n_tile + 31) / 32;  // 32-token chunks of one 128-row tile
      const int nchunk = r.st * nct;          // chunks of the unit (tile j = k / nct)
      if (n_part > 0 && lead0) {
        for (int p = pa; p <= pb; ++p) {
          if (p == fix) continue;
          int* f = r.flags + 2 * pid(p) + (p == pa ? 1 : 0);
          while (ld_acquire(f) != r.epoch) __nanosleep(32);
          // every published flag has exactly one reader: clear it, so a
          // replay of the same launch (CUDA graph, same epoch) waits again
          *f = 0;
        }
        STAMP(true, 6);
      }
      mbar_wait(&tm_full[b], (seg >> 1) & 1);
      tc_fence_after();
      STAMP(lead0 && seg < 4, 9 + seg);
      if (eg >= nchunk) {  // no chunk for this group (n_tile <= 32): hand TMEM back now
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(map_to_rank(smem_u32(&tm_empty[b]), 0));
          else mbar_arrive(&tm_empty[b]);
        }
      }
      if (n_part > 0) {
        // All MMAs of this CTA are complete (this is its last segment), so
        // the A ring is idle: bulk-prefetch every partner chunk into it.
        if (lead0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          mbar_arrive_expect_tx(pbar, static_cast<uint32_t>(n_part * nchunk * kChunkBytes));
          int pi = 0;
          for (int p = pa; p <= pb; ++p) {
            if (p == fix) continue;
            const float* src =
                r.partials + (static_cast<int64_t>(2 * pid(p) + (p == pa ? 1 : 0)) * 8) * (kChunkBytes / 4);
            for (int k = 0; k < nchunk; ++k)
              bulk_g2s(a_st + (pi * nchunk + k) * kChunkBytes, src + k * (kChunkBytes / 4), kChunkBytes, pbar);
            ++pi;
          }
        }
        mbar_wait(pbar, pphase);
        pphase ^= 1;
        STAMP(lead0, 7);
      }
      const int slot = c == pa ? 1 : 0;  // partner: where this piece is published
      const uint32_t acc = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * r.st * r.n_tile);
      for (int k = eg; k < nchunk; k += kEpiGroups) {
        const int tj = k / nct;                  // weight tile of the unit
        const int cc = (k - tj * nct) * 32;      // token offset inside the tile
        const int mrow = PAIR ? 2 * m + rank : m * r.st + tj;  // 128-row output tile
        const bool stamp = r.timing != nullptr && lead0 && seg_last && k < 4;
        float v[32];
        tmem_ld_32x32b_x32(acc + tj * r.n_tile + cc, v);
        if (stamp) r.timing[c * 64 + 20 + k] = gtimer();
        if (k + kEpiGroups >= nchunk) {  // this group's accumulators consumed: hand TMEM back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(map_to_rank(smem_u32(&tm_empty[b]), 0));
          else mbar_arrive(&tm_empty[b]);
        }
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
        if (partner || residual || r.epi == static_cast<int>(Epilogue::kStoreF32)) {
          float* sf = reinterpret_cast<float*>(st);  // [32 tokens][128 features] fp32
#pragma unroll
          for (int j = 0; j < 32; ++j) sf[j * kBM + fl] = v[j];
        } else if (silu) {
          // Feature rows come in (gate_i, up_i) pairs on adjacent lanes: the
          // even lane finishes tokens 0..15 of the chunk, the odd lane tokens
          // 16..31, one shuffle per token. Output act [32 tokens][64] bf16.
          const bool odd = lane & 1;
          __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(st) + (odd ? 16 * (kBM / 2) : 0) + (fl >> 1);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[16 + j], 1);
            const float g = odd ? recv : v[j];
            const float u = odd ? v[16 + j] : recv;
            // ex2.approx + rcp.approx: within 2 fp32 ulp of the IEEE
            // g / (1 + expf(-g)), far below the bf16 rounding of the output
            sh[j * (kBM / 2)] = __float2bfloat16_rn(g * rcp_approx(1.f + __expf(-g)) * u);
          }
        } else {  // kStoreBf16: [32 tokens][128 features] bf16
          __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(st);
#pragma unroll
          for (int j = 0; j < 32; ++j) sh[j * kBM + fl] = __float2bfloat16_rn(v[j]);
        }
        fence_async_smem();
        epi_bar(eg);
        if (leader) {
          if (partner) {
            bulk_s2g(r.partials + (static_cast<int64_t>(2 * me + slot) * 8 + k) * (kChunkBytes / 4), st, kChunkBytes);
          } else if (residual) {
            tma_reduce_add_2d(&tout, st, mrow * kBM, tok0 + cc);  // rows >= M are clipped by TMA
          } else if (silu) {
            tma_store_2d(&tout, st, mrow * (kBM / 2), tok0 + cc);
          } else {
            tma_store_2d(&tout, st, mrow * kBM, tok0 + cc);
            for (int pr = 0; pr < r.n_peers; ++pr) tma_store_2d(&peers.m[pr], st, mrow * kBM, tok0 + cc);
          }
          bulk_commit();
          if (stamp) r.timing[c * 64 + 28 + k] = gtimer();
        }
      }
      if (partner) {  // publish: both groups' partial bulk writes complete, then the flag
        if (leader) bulk_wait<0>();
        epi_bar_all<EG>();
        if (lead0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          st_release(r.flags + 2 * me + slot, r.epoch);
          STAMP(true, 8);
        }
      }
      STAMP(lead0 && seg < 4, 16 + seg);
      ++seg;
    }
    // Staging smem must outlive the bulk stores' reads of it; completion of
    // the writes themselves is only needed before a signal to the TP peers
    // (dependent kernels see them through grid completion).
    if (leader) {
      if (r.n_signal > 0) bulk_wait<0>();
      else bulk_wait_read<0>();
    }
    if (r.n_signal > 0) {
      epi_bar_all<EG>();  // both groups' stores have landed
      if (lead0) {
        // every store of this CTA (local + peers) has completed: publish
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (int d = 0; d < r.n_signal; ++d)
          asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(r.signal[d]) : "memory");
      }
    }
    STAMP(threadIdx.x == 128, 2);
  }
  // Reconverge the role warps (elected producer / MMA lanes) before the
  // block barrier: a diverged warp would arrive early and let warp 2 free
  // TMEM while the epilogue still reads it.
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  // PAIR: the peer's epilogue arrivals on this CTA's barriers and the
  // leader's MMAs into this CTA's TMEM are done before either deallocates
  if constexpr (PAIR) cluster_sync_all();
  STAMP(threadIdx.x == 0, 3);
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(r.tmem_cols) : "memory");
    else
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

bool make_tmap_w_rows(void* tmap_out, const void* w_tiled, int N, int K) {
  const uint64_t rows = static_cast<uint64_t>((N + kBM - 1) / kBM) * ((K + kBK - 1) / kBK) * kBM;
  return make_tmap_2d(tmap_out, w_tiled, false, rows, kBK, kBK * 2, kBM, kBK);
}

bool make_tmap_gemm_out(void* tmap_out, const void* out, int epi, int M, int N, int ldo) {
  const bool fp32 = epi == static_cast<int>(Epilogue::kResidualAddF32) || epi == static_cast<int>(Epilogue::kStoreF32);
  const bool silu = epi == static_cast<int>(Epilogue::kSiluMulBf16);
  const uint64_t cols = silu ? static_cast<uint64_t>(N / 2) : static_cast<uint64_t>(N);
  const uint64_t stride = static_cast<uint64_t>(ldo) * (fp32 ? 4 : 2);
  return make_tmap_2d(tmap_out, out, fp32, static_cast<uint64_t>(M), cols, stride, 32, silu ? kBM / 2 : kBM);
}

// Token-tile rows: one tile up to 256 tokens (a multiple of 16); beyond, the
// fewest tiles of <= 256 with the tokens split evenly, in multiples of 32 --
// the epilogue's chunk -- so no chunk crosses into the next token tile
// (322 -> 2 x 192 instead of 256 + 66).
int gemm_pick_n_tile(int M) {
  const int tiles = std::max(1, (M + 255) / 256);
  const int per = (M + tiles - 1) / tiles;
  int n = tiles == 1 ? ((per + 15) / 16) * 16 : ((per + 31) / 32) * 32;
  if (n > 256) n = 256;
  if (n < 16) n = 16;
  return n;
}

size_t gemm_partials_floats(int max_grid) { return static_cast<size_t>(max_grid) * 2 * 8 * (kChunkBytes / 4); }

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

// Attributes are set here too (per device, at unit creation), so no launch
// inside a CUDA-graph capture is the first one on its device.
static cudaError_t configure_gemm() {
  cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_tn_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(gemm_tn_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 116 * 1024);
}

cudaError_t preload_gemm() {
  cudaError_t e = preload(gemm_tn_kernel<1, false>, gemm_tn_kernel<2, false>, gemm_tn_kernel<2, true>, weight_tile_kernel);
  return e != cudaSuccess ? e : configure_gemm();
}

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
  // CTA pairs (PAIR instantiation; default, MUX_GEMM_PAIR=0 off): token
  // tiles of 65..256 rows (one CTA per SM; several token tiles for prefill
  // shapes the 256 x 256 pair tiles of gemm_2sm would leave unbalanced), an
  // even number of 128-row weight tiles, the half-box activation map and the
  // row view of the tiled weights given.
  static const int env_pair = getenv("MUX_GEMM_PAIR") ? atoi(getenv("MUX_GEMM_PAIR")) : 1;
  const int w_tiles0 = (a.N + kBM - 1) / kBM;
  // (MUX_GEMM_PAIR_MIN_TILE: smallest token tile run on pairs, default 16 =
  // every decode tile: decode rounds at batch 8-64 run 11-14% faster on pairs
  // than in the two-CTAs-per-SM form, profiles/r02_gemm_pair_small.txt; that
  // form remains for launches pairs cannot take: odd weight-tile counts,
  // tensor-parallel units, weights without the tiled layout)
  static const int env_pair_min = getenv("MUX_GEMM_PAIR_MIN_TILE") ? atoi(getenv("MUX_GEMM_PAIR_MIN_TILE")) : 16;
  r.pair = env_pair != 0 && r.n_tile >= std::max(16, env_pair_min) && w_tiles0 % 2 == 0 && a.tmap_x_half != nullptr &&
                   a.tmap_w_rows != nullptr && a.n_peers == 0 && a.n_signal == 0 && (a.grid <= 0 || a.grid >= 2)
               ? 1
               : 0;
  const int b_stage = (r.pair ? r.n_tile / 2 : r.n_tile) * kBK * 2;
  static const int env_dual = getenv("MUX_GEMM_DUAL") ? atoi(getenv("MUX_GEMM_DUAL")) : 1;
  r.eg = (env_dual && r.n_tile <= 64 && !r.pair) ? 1 : 2;
  r.stages_b = r.pair ? 4 : (r.n_tile > 128 ? 2 : 3);
  // Debug overrides for pipeline-depth sweeps (scripts/gemm_micro.py).
  static const int env_sb = getenv("MUX_GEMM_SB") ? atoi(getenv("MUX_GEMM_SB")) : 0;
  static const int env_sa = getenv("MUX_GEMM_SA") ? atoi(getenv("MUX_GEMM_SA")) : 0;
  if (env_sb > 0) r.stages_b = env_sb;
  static const int env_nomma = getenv("MUX_GEMM_NOMMA") ? atoi(getenv("MUX_GEMM_NOMMA")) : 0;
  r.dbg_nomma = env_nomma != 0;
  static const int env_budget = getenv("MUX_GEMM_SMEM_KB") ? atoi(getenv("MUX_GEMM_SMEM_KB")) * 1024 : kSmemBudget;
  // two co-resident CTAs: (228 KB - 2 x 1 KB reserved) / 2 minus alignment slack
  const int budget = r.eg == 1 ? kDualSmemBudget : env_budget;
  // Two 128-row weight tiles per unit (st = 2): each activation stage feeds
  // two MMAs, halving the activation bytes re-read from L2 and staged per
  // weight byte. Decode only (one token tile of <= 128), an even number of
  // weight tiles, one CTA per SM (the dual ring is too small for 32 KiB stages).
  // Pays when every CTA streams many units; with few units per CTA the
  // doubled unit size lengthens the stream-K fixup (the fixer sums partners'
  // 8-chunk partials) and the last epilogue. Measured on the 9 decode shapes
  // of 7B/13B at M = 128 (profiles/r02_gemm_st.txt): LM head +12%, gate-up 13B
  // +6%, down +3-7%; QKV -36-45%, O -5-15%, gate-up 7B -11%. Auto (default):
  // on when a CTA's range holds >= 16 two-tile units (residual epilogue: no
  // fixup) or >= 48 (fixup epilogues). MUX_GEMM_ST=1 off, =2 forced.
  static const int env_st = getenv("MUX_GEMM_ST") ? atoi(getenv("MUX_GEMM_ST")) : 0;
  const int w_tiles = (a.N + kBM - 1) / kBM;
  const bool st_ok = !r.pair && r.eg == 2 && a.M <= 128 && w_tiles % 2 == 0;
  bool st2 = env_st == 2;
  if (env_st == 0 && st_ok) {
    const int64_t per_cta = static_cast<int64_t>(w_tiles / 2) * ((a.K + kBK - 1) / kBK) / std::max(1, a.grid > 0 ? a.grid : 148);
    st2 = per_cta >= (a.epi == Epilogue::kResidualAddF32 ? 16 : 48);
  }
  r.st = (st2 && st_ok) ? 2 : 1;
  // one activation stage now covers twice the weight bytes: two stages keep
  // the same activation lead, and the freed 16 KiB buys a fifth weight stage
  if (r.st == 2 && env_sb <= 0) r.stages_b = 2;
  r.stages_a = (budget - r.stages_b * b_stage - r.eg * kChunkBytes) / (r.st * kAStageBytes);
  if (env_sa > 0) r.stages_a = std::min(env_sa, r.stages_a);
  else if (r.stages_a > 10 / r.st) r.stages_a = 10 / r.st;
  r.kb = (a.K + kBK - 1) / kBK;
  r.m_tiles = w_tiles / (r.pair ? 2 : r.st);  // units along N
  const int n_tiles_tok = (a.M + r.n_tile - 1) / r.n_tile;
  r.iters = static_cast<int64_t>(r.m_tiles) * n_tiles_tok * r.kb;
  r.epi = static_cast<int>(a.epi);
  r.n_tok_tiles = n_tiles_tok;
  r.tmem_cols = pow2_cols(r.st * r.n_tile + (r.st * r.n_tile > 32 ? r.st * r.n_tile : 32));
  // grid = stream-K participants: CTAs, or CTA pairs (launched as 2 x grid)
  int grid = a.grid > 0 ? a.grid : 148;
  if (r.pair) grid /= 2;
  // Enough k-blocks per CTA that the fixed per-CTA cost and the fixup
  // partials stay small next to the weight bytes it streams.
  int64_t min_iters = a.min_iters > 0 ? a.min_iters : 1;
  // Residual epilogues reduce-add their pieces (no fixup): keep the whole
  // machine streaming even for small projections (O of 7B: 2048 k-blocks).
  static const int env_rmin = getenv("MUX_GEMM_RES_MIN_ITERS") ? atoi(getenv("MUX_GEMM_RES_MIN_ITERS")) : 8;
  if (a.epi == Epilogue::kResidualAddF32) min_iters = std::min<int64_t>(min_iters, env_rmin);
  if (static_cast<int64_t>(grid) * min_iters > r.iters) grid = static_cast<int>(std::max<int64_t>(1, r.iters / min_iters));
  // Non-residual epilogues sum pieces in a fixer: keep every tile in few
  // enough pieces that the partners' chunks fit the fixer's idle A ring.
  if (r.epi != static_cast<int>(Epilogue::kResidualAddF32)) {
    const int nchunk = r.st * ((r.n_tile + 31) / 32);
    const int max_partners = (r.stages_a * r.st * kAStageBytes) / (nchunk * kChunkBytes);
    // a range of R iterations lets a tile meet at most ceil(kb / R) + 1 ranges
    const int64_t need_r = (r.kb + max_partners - 1) / std::max(1, max_partners);
    if (static_cast<int64_t>(grid) * need_r > r.iters) grid = static_cast<int>(std::max<int64_t>(1, r.iters / need_r));
  }
  // Schedule: decode (one token tile) = pure stream-K; prefill = grouped
  // data-parallel rounds + stream-K over the last 1-2 waves of tiles (so
  // every stream-K range spans >= one tile's k-blocks: <= 2 pieces).
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
  smem_out = 1024 + static_cast<size_t>(r.stages_a) * r.st * kAStageBytes + static_cast<size_t>(r.stages_b) * b_stage +
             r.eg * kChunkBytes + (2 * (r.stages_a + r.stages_b) + 6) * 8 + 16;
  grid_out = r.pair ? 2 * grid : grid;
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
  static PerDeviceOnce configured;
  cudaError_t ce = configured.run(configure_gemm);
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
  if (r.pair) {
    // clusters of two CTAs (one TPC) + programmatic dependent launch
    std::memcpy(&tw, a.tmap_w_rows, sizeof(CUtensorMap));
    std::memcpy(&tx, a.tmap_x_half, sizeof(CUtensorMap));
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads_of<2>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, gemm_tn_kernel<2, true>, tw, tx, to, r, pm);
  }
  if (r.eg == 1) return launch(gemm_tn_kernel<1, false>, dim3(grid), dim3(threads_of<1>()), smem, stream, tw, tx, to, r, pm);
  return launch(gemm_tn_kernel<2, false>, dim3(grid), dim3(threads_of<2>()), smem, stream, tw, tx, to, r, pm);
}

}  // namespace mux
