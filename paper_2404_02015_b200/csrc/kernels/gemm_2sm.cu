// K4 prefill path on CTA pairs: tcgen05.mma.cta_group::2.
//
// Same product as gemm_tcgen05.cu (D[M x N] = X[M x K] W[N x K]^T with the
// weights pre-tiled into 16 KiB SWIZZLE_128B tiles), for prefill token counts
// (M > 256). A single-SM 128 x 256 tile needs ~188 B/clk of shared memory
// (TMA writes of A and B plus the UMMA reads of both) against 128 B/clk, so
// it cannot pass ~68% of the tensor peak. Here two CTAs on one TPC compute a
// 256 (weights) x 256 (tokens) tile together: each CTA stages its own 128
// weight rows and HALF of the token tile, and one 2-SM UMMA reads the token
// operand from both CTAs' shared memory -- 64 KB of shared-memory traffic
// per SM per k-block against 512 tensor cycles.
//
// Roles (per CTA, 256 threads): warp 0 TMA producer (its A tile + its B
// half), warp 1 MMA issuer on the leader CTA (rank 0) / stage relay on rank
// 1 (forwards "my stage landed" to the leader's barrier), warp 2 TMEM
// allocator (cta_group::2, both CTAs), warps 4-7 epilogue (TMEM -> smem ->
// TMA store of this CTA's 128 weight rows). Data-parallel over tile pairs
// with grouped rasterisation (8 weight tiles per group share their k-slices
// in L2); accumulators double-buffered in TMEM (2 x 256 columns).
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

constexpr int kBM = 128;                     // weight rows per CTA (UMMA M = 256 per pair)
constexpr int kBN = 256;                     // tokens per pair tile (UMMA N), 128 staged per CTA
constexpr int kBK = 64;
constexpr int kStageA = kBM * kBK * 2;       // 16 KiB
constexpr int kStageB = (kBN / 2) * kBK * 2; // 16 KiB
constexpr int kThreads = 256;
constexpr int kEpiThreads = 128;
constexpr int kChunkBytes = 32 * kBM * 4;    // 32 tokens x 128 fp32
constexpr int kGroupPairs = 4;               // raster group: 4 pairs = 8 weight tiles

struct Run2 {
  const uint8_t* w_tiled;
  int M, N, K, kb, m_pairs, n_tiles, tiles, epi;
};

__device__ __forceinline__ void tile_coords(const Run2& r, int t, int& pm, int& pn) {
  const int per = kGroupPairs * r.n_tiles;
  const int g = t / per, in = t - g * per;
  const int gm = min(kGroupPairs, r.m_pairs - g * kGroupPairs);
  pn = in / gm;
  pm = g * kGroupPairs + (in - pn * gm);
}

template <int kStages>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm_2sm_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
                const __grid_constant__ CUtensorMap tout, const Run2 r) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* a_st = base;
  uint8_t* b_st = a_st + kStages * kStageA;
  uint8_t* stage_out = b_st + kStages * kStageB;  // 2 x 16 KiB
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + 2 * kChunkBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tm_full = empty + kStages;
  uint64_t* tm_empty = tm_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, P = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tm_full[b], 1);
      mbar_init(&tm_empty[b], 2 * kEpiThreads / 32);  // epilogue warps of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  grid_dep_wait();  // activations / residual come from the previous kernels
  if (threadIdx.x == 0) grid_dep_launch();

  if (warp == 0) {
    // ---------------- producer: this CTA's weight tile and token half, both
    // counted on the LEADER's full barrier (2-CTA TMA), which the leader arms
    // for the pair's 64 KiB per stage
    if (elect_one()) {
      const uint64_t pol = policy_evict_last();  // weight / token tiles are re-read within the raster group
      const uint32_t full_leader = map_to_rank(smem_u32(full), 0);
      int s = 0, round = 0;
      for (int t = pair; t < r.tiles; t += P) {
        int pm, pn;
        tile_coords(r, t, pm, pn);
        const int m = 2 * pm + static_cast<int>(rank);
        for (int kbi = 0; kbi < r.kb; ++kbi) {
          if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (kStageA + kStageB));
          // tiled weights viewed as [tiles * 128 rows][64]: tile (m, kbi) starts at row (m * kb + kbi) * 128
          tma_load_2d_pair(a_st + s * kStageA, &tw, full_leader + s * 8, 0, (m * r.kb + kbi) * kBM, pol);
          tma_load_2d_pair(b_st + s * kStageB, &tx, full_leader + s * 8, kbi * kBK,
                           pn * kBN + static_cast<int>(rank) * (kBN / 2), pol);
          if (++s == kStages) {
            s = 0;
            ++round;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one() && rank == 0) {
      // ---------------- MMA issuer (leader CTA): D[256 x 256] per tile
      int s = 0, round = 0, seg = 0;
      const uint32_t idesc = umma_idesc_bf16(2 * kBM, kBN);
      for (int t = pair; t < r.tiles; t += P, ++seg) {
        const int b = seg & 1;
        if (seg >= 2) mbar_wait(&tm_empty[b], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(b * kBN);
        for (int kbi = 0; kbi < r.kb; ++kbi) {
          mbar_wait(&full[s], round & 1);  // both CTAs' stages landed
          tc_fence_after();
          const uint32_t a_addr = smem_u32(a_st + s * kStageA), b_addr = smem_u32(b_st + s * kStageB);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            umma2_bf16(acc, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), idesc,
                       (kbi > 0 || kk > 0) ? 1u : 0u);
          umma2_commit_both(&empty[s]);
          if (kbi == r.kb - 1) umma2_commit_both(&tm_full[b]);
          if (++s == kStages) {
            s = 0;
            ++round;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue: this CTA's 128 weight rows x 256 tokens
    const int q = warp & 3;
    const int etid = threadIdx.x - 128;
    const int fl = q * 32 + lane;
    const bool leader = etid == 0;
    const uint32_t tm_empty_leader = map_to_rank(smem_u32(tm_empty), 0);
    int seg = 0, sbuf = 0;
    for (int t = pair; t < r.tiles; t += P, ++seg) {
      int pm, pn;
      tile_coords(r, t, pm, pn);
      const int m = 2 * pm + static_cast<int>(rank);
      const int b = seg & 1;
      mbar_wait(&tm_full[b], (seg >> 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * kBN);
      constexpr int nchunk = kBN / 32;
      for (int k = 0; k < nchunk; ++k) {
        const int tok0 = pn * kBN + k * 32;
        float v[32];
        tmem_ld_32x32b_x32(acc + k * 32, v);
        if (k == nchunk - 1) {  // accumulators consumed: hand the buffer back to the leader
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tm_empty_leader + b * 8);
        }
        if (leader) bulk_wait_read<1>();
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        uint8_t* st = stage_out + sbuf * kChunkBytes;
        const bool silu = r.epi == static_cast<int>(Epilogue::kSiluMulBf16);
        if (r.epi == static_cast<int>(Epilogue::kStoreBf16)) {
          __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(st);
#pragma unroll
          for (int j = 0; j < 32; ++j) sh[j * kBM + fl] = __float2bfloat16_rn(v[j]);
        } else {
          float* sf = reinterpret_cast<float*>(st);
#pragma unroll
          for (int j = 0; j < 32; ++j) sf[j * kBM + fl] = v[j];
        }
        if (silu) {
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          const float4* sf4 = reinterpret_cast<const float4*>(st) + (etid >> 2) * (kBM / 4) + (etid & 3) * 8;
          uint32_t packed[8];
#pragma unroll
          for (int q2 = 0; q2 < 8; ++q2) {
            const float4 gu = sf4[q2];  // gate, up, gate, up
            const float s0 = gu.x / (1.f + expf(-gu.x));
            const float s1 = gu.z / (1.f + expf(-gu.z));
            packed[q2] = pack_bf16(s0 * gu.y, s1 * gu.w);
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          uint4* dst = reinterpret_cast<uint4*>(st + (etid >> 2) * kBM + (etid & 3) * 32);
          dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        }
        fence_async_smem();
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (leader) {
          if (r.epi == static_cast<int>(Epilogue::kResidualAddF32)) tma_reduce_add_2d(&tout, st, m * kBM, tok0);
          else if (silu) tma_store_2d(&tout, st, m * (kBM / 2), tok0);
          else tma_store_2d(&tout, st, m * kBM, tok0);
          bulk_commit();
        }
        sbuf ^= 1;
      }
    }
    if (leader) bulk_wait_read<0>();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs and TMEM reads are done before deallocation
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace

bool gemm_2sm_eligible(const GemmArgs& a) {
  static const int env = getenv("MUX_GEMM_2SM") ? atoi(getenv("MUX_GEMM_2SM")) : 1;
  // Below min_m tokens the stream-K CTA-pair path of gemm_tcgen05.cu (token
  // tiles split evenly, every SM busy) wins over data-parallel 256 x 256 pair
  // tiles, whose count is too small to balance (MUX_GEMM_2SM_MIN_M; measured
  // crossover ~1000 tokens on the 7B/13B shapes, profiles/r02_gemm_2sm_min_m.txt).
  static const int min_m = getenv("MUX_GEMM_2SM_MIN_M") ? atoi(getenv("MUX_GEMM_2SM_MIN_M")) : 1000;
  if (a.N % 256 != 0 || a.M <= std::max(256, min_m)) return false;
  // Data-parallel pair tiles: when the last round would leave most pairs idle
  // (e.g. 80 tiles on 74 pairs), the single-SM stream-K path balances better.
  const int tiles = (a.N / 256) * ((a.M + kBN - 1) / kBN);
  const int pairs = std::max(1, std::min(tiles, (a.grid > 0 ? a.grid : 148) / 2));
  const int rounds = (tiles + pairs - 1) / pairs;
  if (10 * tiles < 7 * rounds * pairs) return false;
  return env != 0 && a.tmap_x128 != nullptr && a.w_tiled != nullptr &&
         a.K % 64 == 0 && a.n_peers == 0 && a.n_signal == 0 &&
         (a.epi == Epilogue::kStoreBf16 || a.epi == Epilogue::kSiluMulBf16 || a.epi == Epilogue::kResidualAddF32 ||
          a.epi == Epilogue::kStoreF32) &&
         (a.grid <= 0 || a.grid >= 2);
}

cudaError_t gemm_2sm(const GemmArgs& a, cudaStream_t stream) {
  Run2 r{};
  r.w_tiled = static_cast<const uint8_t*>(a.w_tiled);
  r.M = a.M;
  r.N = a.N;
  r.K = a.K;
  r.kb = a.K / kBK;
  r.m_pairs = a.N / (2 * kBM);
  r.n_tiles = (a.M + kBN - 1) / kBN;
  r.tiles = r.m_pairs * r.n_tiles;
  r.epi = static_cast<int>(a.epi);
  const int sms = a.grid > 0 ? a.grid : 148;
  const int pairs = std::max(1, std::min(r.tiles, sms / 2));
  static const int env_st = getenv("MUX_GEMM_2SM_STAGES") ? atoi(getenv("MUX_GEMM_2SM_STAGES")) : 6;
  CUtensorMap tw, tx, to;
  // the tiled weights as a [tiles * 128][64] bf16 tensor (rows are already in
  // the SWIZZLE_128B image: copied unswizzled)
  const uint64_t w_rows = static_cast<uint64_t>((a.N + kBM - 1) / kBM) * r.kb * kBM;
  if (!make_tmap_2d(&tw, a.w_tiled, false, w_rows, kBK, kBK * 2, kBM, kBK)) return cudaErrorInvalidValue;
  std::memcpy(&tx, a.tmap_x128, sizeof(CUtensorMap));
  std::memcpy(&to, a.tmap_out, sizeof(CUtensorMap));
  if (a.grid_out != nullptr) *a.grid_out = 2 * pairs;
  // cluster dims come from __cluster_dims__; no PDL attribute on this launch
  // (compute-bound prefill: the launch gap is negligible)
  auto go = [&](auto kernel, int stages) -> cudaError_t {
    const size_t smem = 1024 + static_cast<size_t>(stages) * (kStageA + kStageB) + 2 * kChunkBytes +
                        (2 * stages + 4) * 8 + 16;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kernel<<<dim3(2 * pairs), dim3(kThreads), smem, stream>>>(tw, tx, to, r);
    return cudaGetLastError();
  };
  if (env_st == 4) return go(gemm_2sm_kernel<4>, 4);
  if (env_st == 5) return go(gemm_2sm_kernel<5>, 5);
  return go(gemm_2sm_kernel<6>, 6);
}

cudaError_t preload_gemm_2sm() { return preload(gemm_2sm_kernel<4>, gemm_2sm_kernel<5>, gemm_2sm_kernel<6>); }

}  // namespace mux
