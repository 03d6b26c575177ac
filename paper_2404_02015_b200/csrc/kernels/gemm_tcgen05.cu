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
// of W and "B" is up to 256 activation rows, so D^T tiles of 128 x n_tile
// accumulate in TMEM (fp32). A decode batch (M <= 256) therefore reads each
// weight byte exactly once -- the HBM-bound regime -- and prefill tiles over
// tokens. Warp roles: warp 0 = TMA producer (elected lane), warp 1 = MMA
// issuer (elected lane), warp 2 = TMEM allocator, warps 4..7 = epilogue
// (tcgen05.ld 32 lanes x 32 columns each). K is pipelined through an
// S-stage shared-memory ring (SWIZZLE_128B boxes, 64 K-elements per stage)
// with full/empty mbarriers; tcgen05.commit releases stages.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"

namespace mux {
namespace {

constexpr int kBM = 128;          // W rows per CTA (UMMA M)
constexpr int kBK = 64;           // K per stage (one 128-byte swizzle atom)
constexpr int kAStageBytes = kBM * kBK * 2;
constexpr int kThreads = 256;
constexpr int kSmemBudget = 200 * 1024;

struct GemmRun {
  void* out;
  int M, N, K, ldo;
  int n_tile, stages;
  int kb_total, kb_per_split;
  int epi;
  uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kThreads, 1)
gemm_tn_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
               const GemmRun r) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled stages.
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = r.stages;
  const int b_stage_bytes = r.n_tile * kBK * 2;
  uint8_t* a_st = base;
  uint8_t* b_st = base + S * kAStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(b_st + S * b_stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_blk = blockIdx.x;
  const int n_blk = blockIdx.y;
  const int split = blockIdx.z;
  const int kb0 = split * r.kb_per_split;
  const int nk = min(r.kb_total, kb0 + r.kb_per_split) - kb0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tw);
    prefetch_tmap(&tx);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_dyn(tmem_slot, r.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by every CTA
      const uint32_t bytes = kAStageBytes + b_stage_bytes;
      for (int i = 0; i < nk; ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], bytes);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(a_st + s * kAStageBytes, &tw, &full[s], kc, m_blk * kBM, pol_w);
        tma_load_2d(b_st + s * b_stage_bytes, &tx, &full[s], kc, n_blk * r.n_tile, pol_x);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc_bf16(kBM, r.n_tile);
    for (int i = 0; i < nk; ++i) {
      const int s = i % S;
      mbar_wait(&full[s], (i / S) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t a_addr = smem_u32(a_st + s * kAStageBytes);
        const uint32_t b_addr = smem_u32(b_st + s * b_stage_bytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          // Advance along K inside the swizzle atom: 16 bf16 = 32 bytes.
          umma_bf16(tmem, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                    idesc, (i | kk) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        if (i == nk - 1) umma_commit(done);
      }
      __syncwarp();
    }
    if (nk <= 0 && elect_one()) mbar_arrive(done);
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter this warp may access
    mbar_wait(done, 0);
    tc_fence_after();
    const int feat = m_blk * kBM + q * 32 + lane;  // W row = output column
    const int tok0 = n_blk * r.n_tile;
    for (int c = 0; c < r.n_tile; c += 32) {
      float v[32];
      if (nk > 0) {
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      const int jmax = min(32, min(r.n_tile - c, r.M - (tok0 + c)));
      if (r.epi == static_cast<int>(Epilogue::kStoreBf16)) {
        if (feat < r.N) {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(r.out);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < jmax) o[static_cast<int64_t>(tok0 + c + j) * r.ldo + feat] = __float2bfloat16_rn(v[j]);
        }
      } else if (r.epi == static_cast<int>(Epilogue::kPartialF32) ||
                 r.epi == static_cast<int>(Epilogue::kStoreF32)) {
        if (feat < r.N) {
          float* o = reinterpret_cast<float*>(r.out) + static_cast<int64_t>(split) * r.M * r.ldo;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < jmax) o[static_cast<int64_t>(tok0 + c + j) * r.ldo + feat] = v[j];
        }
      } else {  // kSiluMulBf16: even row = gate_i, odd row = up_i
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(r.out);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float up = __shfl_xor_sync(0xffffffffu, v[j], 1);
          if ((lane & 1) == 0 && j < jmax && feat < r.N) {
            const float g = v[j];
            const float act = g / (1.f + __expf(-g)) * up;
            o[static_cast<int64_t>(tok0 + c + j) * r.ldo + (feat >> 1)] = __float2bfloat16_rn(act);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, r.tmem_cols);
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

int gemm_pick_n_tile(int M) {
  int n = ((M + 15) / 16) * 16;
  if (n > 256) n = 256;
  if (n < 16) n = 16;
  return n;
}

cudaError_t gemm_bf16_tn(const GemmArgs& a, cudaStream_t stream) {
  if (a.M <= 0 || a.N <= 0) return cudaSuccess;
  // tmap_x must have been encoded with box rows == gemm_pick_n_tile(M).
  GemmRun r{};
  r.out = a.out;
  r.M = a.M;
  r.N = a.N;
  r.K = a.K;
  r.ldo = a.ldo;
  r.n_tile = gemm_pick_n_tile(a.M);
  const int stage_bytes = kAStageBytes + r.n_tile * kBK * 2;
  r.stages = kSmemBudget / stage_bytes;
  if (r.stages > 8) r.stages = 8;
  r.kb_total = (a.K + kBK - 1) / kBK;
  const int splits = a.epi == Epilogue::kPartialF32 ? (a.splits < 1 ? 1 : a.splits) : 1;
  r.kb_per_split = (r.kb_total + splits - 1) / splits;
  r.epi = static_cast<int>(a.epi);
  r.tmem_cols = pow2_cols(r.n_tile);
  const size_t smem = 1024 + static_cast<size_t>(r.stages) * stage_bytes + (2 * r.stages + 1) * 8 + 16;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap tw, tx;
  std::memcpy(&tw, a.tmap_w, sizeof(CUtensorMap));
  std::memcpy(&tx, a.tmap_x, sizeof(CUtensorMap));
  dim3 grid((a.N + kBM - 1) / kBM, (a.M + r.n_tile - 1) / r.n_tile, splits);
  gemm_tn_kernel<<<grid, kThreads, smem, stream>>>(tw, tx, r);
  return cudaGetLastError();
}

}  // namespace mux
