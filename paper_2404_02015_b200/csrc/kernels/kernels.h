// Launch interfaces of the sm_100a kernels (host-callable, stream-ordered).
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace mux {

// ---- K1 decode attention -------------------------------------------------
struct DecodeAttnArgs {
  const void* q;            // [B][H][128] bf16 (already RoPE-rotated)
  const void* pool;         // [n_blocks][16][128] bf16
  const int32_t* rowrec;    // [n_rowrec][L*H*2]
  const int32_t* rowlist;   // [slots][max_rows]
  const int32_t* slots;     // [B] device-table slot of each member
  const int32_t* ctx;       // [B] cached tokens incl. the one appended this step
  const int32_t* order;     // [B] CTA z -> member (longest ctx first), or null
  void* out;                // [B][H][128] bf16 or fp32
  float* part_o;            // [B][H][splits][128] (splits > 1)
  float* part_ml;           // [B][H][splits][2]   (splits > 1)
  int* split_count;         // [B][H] zeroed: the last split CTA merges in-kernel (null: combine launch)
  int B, H, layer, max_rows, row_width;
  int splits, rows_per_split;
  // Rows per split from device memory (staged with the job's metadata), so
  // one CUDA-graph capture serves every context length; null: rows_per_split.
  const int32_t* rows_per_split_dev;
  float scale_log2;         // log2(e) / sqrt(128)
};
cudaError_t decode_attention(const DecodeAttnArgs& a, bool fp32_out, cudaStream_t stream);
int decode_attention_max_rows_per_split();

// ---- K2 KV append (+ RoPE) and block-table maintenance --------------------
struct AppendArgs {
  const void* qkv;          // [T][3][H][128] bf16 (q | k | v per token)
  void* q_out;              // [T][H][128] bf16 rotated q (may be null)
  void* pool;               // [n_blocks][16][128] bf16
  const int32_t* rowrec;
  const int32_t* rowlist;
  const int32_t* tok_slot;  // [T] slot of the request owning the token
  const int32_t* tok_pos;   // [T] position of the token in its request
  const float* rope;        // [max_pos][64][2] (cos, sin)
  int T, H, layer, max_rows, row_width;
  int rope_positions;
};
cudaError_t kv_append(const AppendArgs& a, cudaStream_t stream);

// Scatter freshly allocated rows into the device block tables:
//   rowrec[rec[i]][:] = ids[i][:], rowlist[slot[i]][row[i]] = rec[i]
struct TableUpdateArgs {
  const int32_t* meta;      // [n][3] (slot, row, rowrec)
  const int32_t* ids;       // [n][row_width]
  int32_t* rowrec;
  int32_t* rowlist;
  int n, row_width, max_rows;
};
cudaError_t table_update(const TableUpdateArgs& a, cudaStream_t stream);

// ---- K4 tcgen05 GEMM: D[M x N] = X[M x K] * W[N x K]^T -------------------
// Weight-stationary tiling: every CTA owns 128 rows of W (one UMMA M=128
// tile) and up to 256 activation rows (UMMA N), so decode batches (M <= 256)
// stream each weight byte exactly once.
constexpr int kMaxKvSplits = 16;  // K1 context splits per (member, head): the workspace's split scratch
constexpr int kMaxTp = 8;  // tensor-parallel ranks of one mesh (node-local)

enum class Epilogue : int {
  kStoreBf16 = 0,      // out bf16 [M][ldo]
  kResidualAddF32 = 1, // out fp32 [M][ldo] += D (the residual stream; single owner per element)
  kSiluMulBf16 = 2,    // W rows interleaved (gate, up) pairs: out bf16 [M][N/2]
  kStoreF32 = 3,       // out fp32 [M][ldo]
};
struct GemmArgs {
  const void* w_tiled;      // weights in weight_tile() layout (preferred), or null
  const void* tmap_w;       // else: CUtensorMap* over row-major W (host memory)
  const void* tmap_x;       // box rows must equal gemm_pick_n_tile(M)
  const void* tmap_x128 = nullptr;  // same tensor, box 128 rows: enables the 2-SM prefill path (M > 256)
  // Decode CTA-pair mode (MUX_GEMM_PAIR): the activations with box rows =
  // gemm_pick_n_tile(M) / 2, and the tiled weights as a [tiles * 128][64]
  // bf16 tensor (make_tmap_w_rows).
  const void* tmap_x_half = nullptr;
  const void* tmap_w_rows = nullptr;
  const void* tmap_out;     // make_tmap_gemm_out(): box 32 tokens x 128 (SiLU: 64) features
  void* out;
  float* partials;          // stream-K fixup scratch: gemm_partials_floats(grid) floats
  int* flags;               // [grid] ints, zero-initialised once
  int epoch;                // distinct (> 0) for every launch sharing `flags`
  int grid;                 // persistent CTAs (#SMs)
  int min_iters;            // cap the grid so every CTA gets >= min_iters k-blocks (0 = no cap)
  int M, N, K;
  int ldo;
  Epilogue epi;
  // Tensor parallelism (kStoreF32): also store every tile through these
  // maps (host CUtensorMap*, peer ranks' slots) and signal the counters
  // once per CTA when its stores have landed. grid_out receives the grid.
  int n_peers = 0;
  const void* tmap_peers[kMaxTp - 1] = {};
  int n_signal = 0;
  int* signal[kMaxTp] = {};
  int* grid_out = nullptr;
};
cudaError_t gemm_bf16_tn(const GemmArgs& a, cudaStream_t stream);
// Prefill GEMMs on CTA pairs (tcgen05 cta_group::2, gemm_2sm.cu); gemm_bf16_tn
// dispatches there when gemm_2sm_eligible (M > 256, N % 256 == 0, plain
// store / SiLU / residual / fp32 epilogue, tmap_x128 set; MUX_GEMM_2SM=0 off).
bool gemm_2sm_eligible(const GemmArgs& a);
cudaError_t gemm_2sm(const GemmArgs& a, cudaStream_t stream);
cudaError_t preload_gemm_2sm();
int gemm_pick_n_tile(int M);
// The tiled weights (weight_tile layout) as a [ceil(N/128) * ceil(K/64) * 128][64]
// bf16 tensor, box 128 x 64, no swizzle (the bytes already hold the SW128 image).
bool make_tmap_w_rows(void* tmap_out, const void* w_tiled, int N, int K);
bool make_tmap_gemm_out(void* tmap_out, const void* out, int epi, int M, int N, int ldo);
// B200 weight layout: [ceil(N/128)][ceil(K/64)] contiguous 16 KiB UMMA tiles,
// pre-swizzled (SWIZZLE_128B), zero-padded. inverse=true converts back.
size_t weight_tiled_bytes(int N, int K);
cudaError_t weight_tile(const void* src, int N, int K, void* dst, bool inverse, cudaStream_t stream);
size_t gemm_partials_floats(int max_grid);
void gemm_debug_timing(void* buf);  // [grid][64] u64 globaltimer stamps per CTA, null = off
// Encode a 2-D bf16 tensor map (rows x cols, cols contiguous) with a
// box of box_rows x 64 and 128-byte swizzle. Returns false on failure.
// Plain 2-D map (no swizzle), box box_rows x box_cols, bf16 or fp32.
bool make_tmap_2d(void* tmap_out, const void* base, bool fp32, uint64_t rows, uint64_t cols,
                  uint64_t row_stride_bytes, uint32_t box_rows, uint32_t box_cols);
bool make_tmap_bf16(void* tmap_out, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_stride_bytes, uint32_t box_rows);

// ---- K5 small fused ops ---------------------------------------------------
cudaError_t embed_rmsnorm(const void* emb, const int32_t* tokens, const float* norm_w,
                          float* resid, void* xn, int T, int hidden, float eps,
                          cudaStream_t stream);
// xn[t] = bf16(resid[t] * rsqrt(mean(resid[t]^2) + eps) * w)
cudaError_t rmsnorm_rows(const float* resid, const float* norm_w, void* xn, int T, int hidden, float eps,
                         cudaStream_t stream, int max_ctas = 0);
// Tensor-parallel residual update + RMSNorm: waits until *counter has reached
// `expected` (every rank's row-parallel GEMM stored its partial here), then
// resid[t] += parts[0][t] + ... + parts[tp-1][t] (rank order), xn = rmsnorm.
// parts[src] = parts + src * part_stride floats, rows of `hidden`.
cudaError_t rmsnorm_tp(float* resid, const float* parts, int64_t part_stride, int tp, const int* counter,
                       uint32_t expected, const float* norm_w, void* xn, int T, int hidden, float eps,
                       cudaStream_t stream);
// Row argmax of fp32 logits; writes token ids (lowest index on ties).
cudaError_t argmax_rows(const float* logits, int T, int V, int32_t* out, cudaStream_t stream);
// Gather rows: dst[i] = src[idx[i]] (bf16 rows of `cols`).
cudaError_t gather_rows_bf16(const void* src, const int32_t* idx, void* dst, int n, int cols,
                             cudaStream_t stream);
// ---- K3 causal varlen prefill attention (tcgen05 flash attention) ---------
struct PrefillAttnArgs {
  const void* q;            // [T][H][128] bf16 rotated
  const void* qkv;          // [T][3][H][128] bf16 (k rotated in-place by kv_append)
  void* out;                // [T][H][128] bf16
  const int32_t* seq_start; // [nseq + 1]
  const int32_t* tiles;     // [n_tiles] (seq << 16) | q_tile, heaviest (largest q_tile) first
  const void* tmap_q;       // make_tmap_bf16(q, T, H*128, .., box_rows 128)   (host memory)
  const void* tmap_qkv;     // make_tmap_bf16(qkv, T, 3*H*128, .., box_rows 128)
  int n_tiles, nseq, H, T;
  float scale_log2;
  int max_ctas = 0;         // persistent grid (the partition's SMs); 0 = 148
};
cudaError_t prefill_attention(const PrefillAttnArgs& a, cudaStream_t stream);
size_t prefill_attention_smem();
// Deterministic N(0, std) init of a bf16 buffer from (seed, index).
cudaError_t init_normal_bf16(void* dst, int64_t n, uint64_t seed, float std, cudaStream_t stream);
cudaError_t fill_f32(float* dst, int64_t n, float v, cudaStream_t stream);

// Load every libmux kernel (see launch.cuh: preload); one per translation unit.
cudaError_t preload_decode_attention();
cudaError_t preload_kv_append();
cudaError_t preload_gemm();
cudaError_t preload_prefill_attention();
cudaError_t preload_fused_ops();

}  // namespace mux
