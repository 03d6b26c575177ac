// B200 device runtime: the unified KV block pool in HBM, per-model LLaMA
// weights and device block tables, per-partition workspaces, and the
// prefill / decode job forwards that UnitSim::launch
// (/root/reference/proj/src/sim_engine.cpp:308-330) only priced.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "mux/kv.hpp"
#include "../kernels/kernels.h"

namespace mux {

struct ModelDims {
  std::string name;
  int layers = 0;
  int heads = 0;
  int head_dim = 128;
  int hidden = 0;
  int ffn = 0;
  int vocab = 32000;
  float norm_eps = 1e-5f;
  float rope_theta = 10000.f;
  // Tensor parallelism (Megatron): this shard holds heads [r*heads, (r+1)*heads)
  // and FFN columns [r*ffn, (r+1)*ffn) of the full model; `heads` and `ffn`
  // above are the LOCAL counts. tp_size == 1: the whole model.
  int tp_rank = 0;
  int tp_size = 1;
};

// Device buffer (cudaMalloc), owned.
struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  DevMem() = default;
  explicit DevMem(size_t n);
  ~DevMem();
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevMem& operator=(DevMem&& o) noexcept;
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

struct PinnedMem {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedMem() = default;
  explicit PinnedMem(size_t n);
  ~PinnedMem();
  PinnedMem(const PinnedMem&) = delete;
  PinnedMem& operator=(const PinnedMem&) = delete;
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// One colocated LLaMA model: weights + its block tables in HBM.
class Llama {
 public:
  Llama(const ModelDims& d, int max_slots, int max_rows, int64_t max_rowrecs);
  const ModelDims& dims() const { return d_; }
  int row_width() const { return 2 * d_.layers * d_.heads; }
  int qkv_cols() const { return 3 * d_.heads * d_.head_dim; }
  int max_slots() const { return max_slots_; }
  int max_rows() const { return max_rows_; }
  int64_t max_rowrecs() const { return max_rowrecs_; }
  int64_t weight_bytes() const;
  void init_random(uint64_t seed, float std, cudaStream_t s);
  // Upload one tensor from host in device layout (see capi docs). Returns false on bad name/size.
  bool set_tensor(const std::string& name, int layer, const void* host, size_t bytes, cudaStream_t s);
  bool get_tensor(const std::string& name, int layer, void* host, size_t bytes, cudaStream_t s) const;

  // weights (bf16 unless noted)
  DevMem embed, lm_head, final_norm;                 // final_norm fp32
  std::vector<DevMem> wqkv, wo, wgu, wdown;          // per layer
  std::vector<DevMem> attn_norm, ffn_norm;           // fp32
  // GEMM weights (lm_head, wqkv, wo, wgu, wdown) live in the B200 tiled
  // layout of weight_tile(): contiguous pre-swizzled 16 KiB UMMA tiles.
  // device block tables
  DevMem rowrec;    // [max_rowrecs][row_width] int32
  DevMem rowlist;   // [max_slots][max_rows] int32
  DevMem last_tok;  // [max_slots] int32: most recent token of each slot

 private:
  // (rows, cols) of a named tensor; tiled = stored in the GEMM tile layout.
  DevMem* tensor(const std::string& name, int layer, int* rows, int* cols, bool* tiled);
  ModelDims d_;
  int max_slots_, max_rows_;
  int64_t max_rowrecs_;
};

// Tensor-parallel mailbox of one partition (the fused GEMM -> allreduce of
// the row-parallel O / down projections). Layout of every rank's box:
//   slots [2][tp][rows][hidden] fp32   slot s, written by rank src
//   counters [2] int32                 bumped by every CTA of every rank's GEMM
// Rank src's GEMM stores its fp32 partial tile straight into slot (s, src) of
// every rank (NVLink peer stores by TMA) and then signals their counter s;
// each rank's rmsnorm_tp waits for its counter and sums the tp slots in rank
// order, so the residual stream stays bit-identical on every rank. Slot 0
// serves the O projection, slot 1 the down projection: a rank can only reach
// a slot again after every peer has consumed it (see runtime.cu).
struct TpLink {
  int rank = 0, size = 1;
  int rows = 0, hidden = 0;
  DevMem box;
  void* peer[8] = {};        // every rank's box as mapped in this process (peer[rank] = own)
  bool ipc_opened[8] = {};
  uint32_t expected[2] = {0, 0};
  size_t slot_floats() const { return static_cast<size_t>(rows) * hidden; }
  float* slot(int r, int s, int src) const {
    return static_cast<float*>(peer[r]) + (static_cast<size_t>(s) * size + src) * slot_floats();
  }
  int* counter(int r, int s) const {
    return reinterpret_cast<int*>(static_cast<float*>(peer[r]) + 2 * size * slot_floats()) + s;
  }
  bool connected() const {
    for (int r = 0; r < size; ++r)
      if (peer[r] == nullptr) return false;
    return true;
  }
  ~TpLink();
};

// Per-partition scratch for one running job.
struct Workspace {
  int max_tokens = 0;    // prefill token budget or max decode batch
  int max_decode = 0;    // decode members the K1 split scratch is sized for
  int max_hidden = 0, max_qkv = 0, max_ffn = 0, max_vocab = 0, max_heads = 0;
  DevMem resid, xn, qkv, q, attn, act, logits, ints, attn_part_o, attn_part_ml, attn_split_count, xlast;
  DevMem gemm_partials, gemm_flags;  // stream-K fixup scratch of this partition's GEMMs
  int gemm_epoch = 0;
  int sms = 148;           // SMs of the partition this workspace's jobs run on
  bool exclusive = false;  // a green partition: no other stream's kernels share its SMs
  std::unique_ptr<TpLink> tp;  // tensor-parallel mailbox (tp_size > 1)
  PinnedMem host_ints[2];  // double-buffered staging for per-job metadata
  cudaEvent_t staged[2] = {nullptr, nullptr};
  int cur = 0;
  // Next staging buffer: waits until the copy that last used it completed.
  int32_t* stage_begin();
  // Enqueue the copy of the first n_ints of the staging buffer and flip.
  void stage_commit(size_t n_ints, cudaStream_t stream);
  ~Workspace();
  // int32 views into `ints`
  int32_t *tokens, *slots, *ctx, *tok_slot, *tok_pos, *seq_start, *out_tok, *last_rows;
  Workspace(int max_tokens, int max_batch_rows, int hidden, int qkv, int ffn, int vocab, int heads,
            int max_decode_batch, int grid);
};

// Per-launch K1 timing: an event pair around every decode-attention launch.
struct AttnTimer {
  std::vector<cudaEvent_t> spare;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  double total_ms = 0.0;
  double bytes = 0.0;
  int64_t launches = 0;
  double pending_bytes = 0.0;
  cudaEvent_t get();
  void harvest();  // synchronises pending pairs and accumulates
  ~AttnTimer();
};

class Runtime {
 public:
  Runtime(int device, int64_t pool_blocks, int max_pos);
  ~Runtime();
  int device() const { return device_; }
  int64_t pool_blocks() const { return pool_blocks_; }
  void* pool() const { return pool_.p; }
  const float* rope() const { return rope_.as<float>(); }
  int rope_positions() const { return max_pos_; }
  int num_sms() const { return num_sms_; }
  int64_t launches() const { return launches_; }
  void set_gemm_min_iters(int v) { gemm_min_iters_ = v; }
  void count_launch(int64_t n = 1) { launches_ += n; }
  // Per-launch CUDA events around every decode GEMM (M <= 256) on its
  // stream, accumulating the weight bytes it streams (null = off).
  void set_gemm_timer(AttnTimer* t) { gemm_timer_ = t; }
  // CUDA graphs for decode jobs: one capture per (model, workspace, batch,
  // K1 splits, tokens staged or gathered), replayed on later calls.
  void set_graphs(bool on) { use_graphs_ = on; }
  // Debug / measurement (MUX_DEBUG_SKIP, option "debug_skip"): decode jobs
  // skip kernel classes (1 K2, 2 RMSNorm, 4 K1, 8 RMSNorm over one row);
  // outputs are garbage, the remaining kernels' timings are not. Never
  // captured into graphs.
  void set_debug_skip(int mask) { dbg_skip_ = mask; }
  int64_t graph_captures() const { return graph_captures_; }

  // Cached tensor map for an activation buffer viewed as rows x cols bf16.
  const void* act_tmap(const void* base, int rows, int cols, int box_rows);
  const void* w_rows_tmap(const void* w_tiled, int N, int K);  // make_tmap_w_rows, cached
  // Cached store map of a GEMM output (exact M rows: TMA clips the tail).
  const void* out_tmap(const void* out, int epi, int M, int N, int ldo);

  // Block-table maintenance: copy pending rows of `llm` (host pool) to the
  // model's device tables on `stream` (through pinned staging).
  void upload_rows(muxsim::BlockPool& pool, int llm, Llama& m, cudaStream_t stream);

  // Jobs. Members are (slot, ctx) pairs; ctx = cached tokens incl. the new one.
  void decode(Llama& m, Workspace& ws, int n, const int32_t* slots_host, const int32_t* ctx_host,
              const int32_t* tokens_host /*nullable: use last_tok*/, int32_t* out_host /*nullable*/,
              cudaStream_t stream, AttnTimer* timer = nullptr);
  void prefill(Llama& m, Workspace& ws, int n, const int32_t* slots_host, const int32_t* lens_host,
               const int32_t* tokens_host, int32_t* out_host /*nullable*/, cudaStream_t stream);

  // Decode-forward building blocks, exposed for tests/bench.
  void gemm(const void* w_tiled, const void* x, int M, int N, int K, void* out, int ldo, int epi,
            Workspace& ws, cudaStream_t stream);
  // Row-parallel projection + the fused allreduce (tp > 1): out partial of
  // X[M x K] W[N x K]^T to every rank's slot `s`, then resid += sum of ranks'
  // slots and xn = rmsnorm(resid) * norm_w on this rank.
  void row_parallel_norm(const void* w_tiled, const void* x, int M, int N, int K, int s, const float* norm_w,
                         float eps, Workspace& ws, cudaStream_t stream);

 private:
  int device_;
  int num_sms_;
  int64_t pool_blocks_;
  int max_pos_;
  int64_t launches_ = 0;
  AttnTimer* gemm_timer_ = nullptr;
  struct GraphKey {
    const void* model;
    const void* ws;
    int n, splits;
    bool tokens;
    bool operator<(const GraphKey& o) const {
      return std::tie(model, ws, n, splits, tokens) < std::tie(o.model, o.ws, o.n, o.splits, o.tokens);
    }
  };
  struct GraphEntry {
    cudaGraphExec_t exec;
    int64_t kernels;  // kernels per replay (launch accounting)
    uint64_t used;    // LRU clock
  };
  static constexpr size_t kMaxGraphs = 384;
  bool use_graphs_ = true;
  int dbg_skip_ = 0;
  std::map<GraphKey, GraphEntry> graphs_;
  std::map<GraphKey, int> graph_seen_;
  uint64_t graph_clock_ = 0;
  int64_t graph_captures_ = 0;
  int gemm_min_iters_ = 8;  // scripts/min_iters_sweep.py: 8 is never slower on the whole GPU, -6..-11% at batch 128
  DevMem pool_;
  DevMem rope_;
  struct StageSlot {
    DevMem dev;
    std::unique_ptr<PinnedMem> host;
    cudaEvent_t done = nullptr;
    size_t cap = 0;
  };
  StageSlot ring_[4];
  std::vector<DevMem> retired_dev_;
  std::vector<std::unique_ptr<PinnedMem>> retired_host_;
  int ring_next_ = 0;
  std::map<std::tuple<const void*, int, int, int>, std::vector<unsigned char>> tmaps_;
  std::map<std::tuple<const void*, int, int, int>, std::vector<unsigned char>> out_tmaps_;
};

void check_cuda(cudaError_t e, const char* what);

}  // namespace mux
