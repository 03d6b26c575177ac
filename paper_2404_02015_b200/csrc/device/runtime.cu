// B200 device runtime: KV pool, LLaMA weights/tables, job forwards.
#include "runtime.h"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../kernels/kernels.h"
#include "../kernels/launch.cuh"
#include "../kernels/ptx.cuh"

namespace mux {

bool& pdl_enabled() {
  static bool on = true;
  return on;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("cuda error in ") + what + ": " + cudaGetErrorString(e));
}

DevMem::DevMem(size_t n) : bytes(n) {
  if (n > 0) check_cuda(cudaMalloc(&p, n), "cudaMalloc");
}
DevMem::~DevMem() {
  if (p) cudaFree(p);
}
DevMem& DevMem::operator=(DevMem&& o) noexcept {
  if (this != &o) {
    if (p) cudaFree(p);
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}
PinnedMem::PinnedMem(size_t n) : bytes(n) {
  if (n > 0) check_cuda(cudaMallocHost(&p, n), "cudaMallocHost");
}
PinnedMem::~PinnedMem() {
  if (p) cudaFreeHost(p);
}

namespace {

constexpr int kEpiStoreBf16 = 0, kEpiResidual = 1, kEpiSilu = 2, kEpiStoreF32 = 3;

__global__ void gather_last_tok(const int32_t* last_tok, const int32_t* slots, int32_t* tokens, int n) {
  grid_dep_wait();
  grid_dep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tokens[i] = last_tok[slots[i]];
}

__global__ void scatter_last_tok(int32_t* last_tok, const int32_t* slots, const int32_t* tokens, int n) {
  grid_dep_wait();
  grid_dep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) last_tok[slots[i]] = tokens[i];
}

int gemm_n_tile(int M) { return gemm_pick_n_tile(M); }

}  // namespace

// ------------------------------------------------------------------ Llama

Llama::Llama(const ModelDims& d, int max_slots, int max_rows, int64_t max_rowrecs)
    : d_(d), max_slots_(max_slots), max_rows_(max_rows), max_rowrecs_(max_rowrecs) {
  if (d.head_dim != 128) throw std::invalid_argument("llama: head_dim must be 128");
  if (d.hidden % 64 != 0 || d.ffn % 64 != 0) throw std::invalid_argument("llama: hidden/ffn must be multiples of 64");
  const int hid = d.hidden, ffn = d.ffn, V = d.vocab, qkv = 3 * d.heads * 128, att = d.heads * 128;
  embed = DevMem(static_cast<size_t>(V) * hid * 2);  // row-major: gathered by token id
  lm_head = DevMem(weight_tiled_bytes(V, hid));
  final_norm = DevMem(static_cast<size_t>(hid) * 4);
  for (int l = 0; l < d.layers; ++l) {
    wqkv.emplace_back(weight_tiled_bytes(qkv, hid));
    wo.emplace_back(weight_tiled_bytes(hid, att));
    wgu.emplace_back(weight_tiled_bytes(2 * ffn, hid));
    wdown.emplace_back(weight_tiled_bytes(hid, ffn));
    attn_norm.emplace_back(static_cast<size_t>(hid) * 4);
    ffn_norm.emplace_back(static_cast<size_t>(hid) * 4);
  }
  rowrec = DevMem(static_cast<size_t>(max_rowrecs) * row_width() * 4);
  rowlist = DevMem(static_cast<size_t>(max_slots) * max_rows * 4);
  last_tok = DevMem(static_cast<size_t>(max_slots) * 4);
  check_cuda(cudaMemset(rowlist.p, 0, rowlist.bytes), "memset rowlist");
  check_cuda(cudaMemset(last_tok.p, 0, last_tok.bytes), "memset last_tok");
}

int64_t Llama::weight_bytes() const {
  int64_t t = embed.bytes + lm_head.bytes;
  for (int l = 0; l < d_.layers; ++l) t += wqkv[l].bytes + wo[l].bytes + wgu[l].bytes + wdown[l].bytes;
  return t;
}

void Llama::init_random(uint64_t seed, float std, cudaStream_t s) {
  uint64_t k = seed * 0x100000001B3ull;
  auto init = [&](DevMem& m) { check_cuda(init_normal_bf16(m.p, m.bytes / 2, ++k, std, s), "init"); };
  auto ones = [&](DevMem& m) { check_cuda(fill_f32(m.as<float>(), m.bytes / 4, 1.f, s), "fill"); };
  init(embed);
  init(lm_head);
  ones(final_norm);
  for (int l = 0; l < d_.layers; ++l) {
    init(wqkv[l]);
    init(wo[l]);
    init(wgu[l]);
    init(wdown[l]);
    ones(attn_norm[l]);
    ones(ffn_norm[l]);
  }
}

DevMem* Llama::tensor(const std::string& name, int layer, int* rows, int* cols, bool* tiled) {
  const int hid = d_.hidden, ffn = d_.ffn, att = d_.heads * 128;
  auto per_layer = [&](std::vector<DevMem>& v) -> DevMem* {
    return layer >= 0 && layer < d_.layers ? &v[layer] : nullptr;
  };
  struct Shape { DevMem* m; int r, c; bool t; };
  Shape sh{nullptr, 0, 0, false};
  if (name == "embed") sh = {&embed, d_.vocab, hid, false};
  else if (name == "lm_head") sh = {&lm_head, d_.vocab, hid, true};
  else if (name == "final_norm") sh = {&final_norm, 1, hid * 2, false};
  else if (name == "wqkv") sh = {per_layer(wqkv), qkv_cols(), hid, true};
  else if (name == "wo") sh = {per_layer(wo), hid, att, true};
  else if (name == "wgu") sh = {per_layer(wgu), 2 * ffn, hid, true};
  else if (name == "wdown") sh = {per_layer(wdown), hid, ffn, true};
  else if (name == "attn_norm") sh = {per_layer(attn_norm), 1, hid * 2, false};
  else if (name == "ffn_norm") sh = {per_layer(ffn_norm), 1, hid * 2, false};
  *rows = sh.r;
  *cols = sh.c;  // in bf16 units (fp32 norms count as 2)
  *tiled = sh.t;
  return sh.m;
}

// Megatron shard of a full host tensor: column-parallel QKV (rows of this
// rank's heads in each of q/k/v) and gate/up (rows of this rank's FFN
// columns; the (gate_i, up_i) interleave keeps them contiguous), row-parallel
// O / down (this rank's input columns). Returns false if `name` is replicated.
static bool shard_rows(const ModelDims& d, const std::string& name, const uint16_t* full, std::vector<uint16_t>& out) {
  const int r = d.tp_rank, tp = d.tp_size, hid = d.hidden;
  const int64_t hl = static_cast<int64_t>(d.heads) * 128, hf = hl * tp;  // local / full attention width
  const int64_t fl = d.ffn, ff = fl * tp;
  if (name == "wqkv") {
    out.resize(3 * hl * hid);
    for (int part = 0; part < 3; ++part)
      std::memcpy(out.data() + part * hl * hid, full + (part * hf + r * hl) * hid, hl * hid * 2);
  } else if (name == "wgu") {
    out.resize(2 * fl * hid);
    std::memcpy(out.data(), full + 2 * r * fl * hid, 2 * fl * hid * 2);
  } else if (name == "wo" || name == "wdown") {
    const int64_t loc = name == "wo" ? hl : fl, tot = name == "wo" ? hf : ff;
    out.resize(static_cast<size_t>(hid) * loc);
    for (int64_t row = 0; row < hid; ++row) std::memcpy(out.data() + row * loc, full + row * tot + r * loc, loc * 2);
  } else {
    return false;
  }
  return true;
}

bool Llama::set_tensor(const std::string& name, int layer, const void* host, size_t bytes, cudaStream_t s) {
  int rows = 0, cols = 0;
  bool tiled = false;
  DevMem* m = tensor(name, layer, &rows, &cols, &tiled);
  std::vector<uint16_t> shard;
  if (m != nullptr && d_.tp_size > 1 && static_cast<size_t>(rows) * cols * 2 * d_.tp_size == bytes &&
      shard_rows(d_, name, static_cast<const uint16_t*>(host), shard)) {
    host = shard.data();  // a full tensor was given: keep this rank's shard
    bytes = shard.size() * 2;
  }
  if (!m || static_cast<size_t>(rows) * cols * 2 != bytes) return false;
  if (!tiled) {
    check_cuda(cudaMemcpyAsync(m->p, host, bytes, cudaMemcpyHostToDevice, s), "set_tensor");
  } else {
    DevMem tmp(bytes);
    check_cuda(cudaMemcpyAsync(tmp.p, host, bytes, cudaMemcpyHostToDevice, s), "set_tensor");
    check_cuda(weight_tile(tmp.p, rows, cols, m->p, false, s), "weight_tile");
    check_cuda(cudaStreamSynchronize(s), "set_tensor sync");
  }
  check_cuda(cudaStreamSynchronize(s), "set_tensor sync");
  return true;
}

bool Llama::get_tensor(const std::string& name, int layer, void* host, size_t bytes, cudaStream_t s) const {
  int rows = 0, cols = 0;
  bool tiled = false;
  DevMem* m = const_cast<Llama*>(this)->tensor(name, layer, &rows, &cols, &tiled);
  if (!m || static_cast<size_t>(rows) * cols * 2 != bytes) return false;
  if (!tiled) {
    check_cuda(cudaMemcpyAsync(host, m->p, bytes, cudaMemcpyDeviceToHost, s), "get_tensor");
  } else {
    DevMem tmp(bytes);
    check_cuda(weight_tile(m->p, rows, cols, tmp.p, true, s), "weight_untile");
    check_cuda(cudaMemcpyAsync(host, tmp.p, bytes, cudaMemcpyDeviceToHost, s), "get_tensor");
    check_cuda(cudaStreamSynchronize(s), "get_tensor sync");
  }
  check_cuda(cudaStreamSynchronize(s), "get_tensor sync");
  return true;
}

// -------------------------------------------------------------- Workspace

Workspace::Workspace(int max_tok, int max_batch_rows, int hidden, int qkv_cols, int ffn, int vocab,
                     int heads, int max_decode_batch, int grid)
    : max_tokens(max_tok), max_decode(max_decode_batch), max_hidden(hidden), max_qkv(qkv_cols), max_ffn(ffn), max_vocab(vocab),
      max_heads(heads) {
  const size_t T = std::max(max_tok, 16);
  // Activation buffers get >= 256 rows so any n_tile box stays in bounds.
  const size_t Tp = std::max<size_t>(T, 256);
  resid = DevMem(Tp * hidden * 4);
  xn = DevMem(Tp * hidden * 2);
  qkv = DevMem(Tp * qkv_cols * 2);
  q = DevMem(Tp * heads * 128 * 2);
  attn = DevMem(Tp * heads * 128 * 2);
  act = DevMem(Tp * ffn * 2);
  gemm_partials = DevMem(gemm_partials_floats(grid) * 4);
  gemm_flags = DevMem(static_cast<size_t>(std::max(grid, 1024)) * 4);
  check_cuda(cudaMemset(gemm_flags.p, 0, gemm_flags.bytes), "memset flags");
  const size_t rows_out = std::max<size_t>(max_batch_rows, 256);
  logits = DevMem(rows_out * vocab * 4);
  xlast = DevMem(rows_out * hidden * 2);
  const size_t kv_splits = kMaxKvSplits;
  attn_part_o = DevMem(static_cast<size_t>(max_decode_batch) * heads * kv_splits * 128 * 4);
  attn_part_ml = DevMem(static_cast<size_t>(max_decode_batch) * heads * kv_splits * 2 * 4);
  attn_split_count = DevMem(static_cast<size_t>(max_decode_batch) * heads * 4);
  check_cuda(cudaMemset(attn_split_count.p, 0, attn_split_count.bytes), "memset split counters");
  // ints: tokens[T] slots[T] ctx[T] tok_slot[T] tok_pos[T] seq_start[T+1] out_tok[T] last_rows[T]
  const size_t n_ints = 8 * T + 8;
  ints = DevMem(n_ints * 4);
  for (int i = 0; i < 2; ++i) {
    new (&host_ints[i]) PinnedMem(n_ints * 4);
    check_cuda(cudaEventCreateWithFlags(&staged[i], cudaEventDisableTiming), "event");
  }
  int32_t* b = ints.as<int32_t>();
  tokens = b;
  slots = b + T;
  ctx = b + 2 * T;
  tok_slot = b + 3 * T;
  tok_pos = b + 4 * T;
  seq_start = b + 5 * T;
  out_tok = b + 6 * T + 1;
  last_rows = b + 7 * T + 1;
}

cudaEvent_t AttnTimer::get() {
  if (!spare.empty()) {
    cudaEvent_t e = spare.back();
    spare.pop_back();
    return e;
  }
  cudaEvent_t e;
  check_cuda(cudaEventCreate(&e), "event");
  return e;
}

void AttnTimer::harvest() {
  for (auto& pr : pending) {
    check_cuda(cudaEventSynchronize(pr.second), "timer sync");
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, pr.first, pr.second), "timer elapsed");
    total_ms += ms;
    launches += 1;
    spare.push_back(pr.first);
    spare.push_back(pr.second);
  }
  pending.clear();
  bytes += pending_bytes;
  pending_bytes = 0.0;
}

AttnTimer::~AttnTimer() {
  for (cudaEvent_t e : spare) cudaEventDestroy(e);
  for (auto& pr : pending) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
}

Workspace::~Workspace() {
  for (int i = 0; i < 2; ++i)
    if (staged[i]) cudaEventDestroy(staged[i]);
}

int32_t* Workspace::stage_begin() {
  check_cuda(cudaEventSynchronize(staged[cur]), "stage wait");
  return host_ints[cur].as<int32_t>();
}

void Workspace::stage_commit(size_t n_ints, cudaStream_t stream) {
  check_cuda(cudaMemcpyAsync(ints.p, host_ints[cur].p, n_ints * 4, cudaMemcpyHostToDevice, stream),
             "meta copy");
  check_cuda(cudaEventRecord(staged[cur], stream), "stage record");
  cur ^= 1;
}

TpLink::~TpLink() {
  for (int r = 0; r < size; ++r)
    if (ipc_opened[r] && peer[r] != nullptr) cudaIpcCloseMemHandle(peer[r]);
}

// ---------------------------------------------------------------- Runtime

Runtime::Runtime(int device, int64_t pool_blocks, int max_pos)
    : device_(device), pool_blocks_(pool_blocks), max_pos_(max_pos) {
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  check_cuda(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device), "sm count");
  check_cuda(preload_decode_attention(), "preload");
  check_cuda(preload_kv_append(), "preload");
  check_cuda(preload_gemm(), "preload");
  check_cuda(preload_gemm_2sm(), "preload");
  check_cuda(preload_prefill_attention(), "preload");
  check_cuda(preload_fused_ops(), "preload");
  check_cuda(preload(gather_last_tok, scatter_last_tok), "preload");
  if (const char* g = getenv("MUX_GRAPHS")) use_graphs_ = atoi(g) != 0;  // A/B switch (option "graphs")
  if (const char* k = getenv("MUX_DEBUG_SKIP")) dbg_skip_ = atoi(k);   // option "debug_skip"
  pool_ = DevMem(static_cast<size_t>(pool_blocks) * 4096);
  // RoPE table [max_pos][64][(cos, sin)], computed in double, stored fp32.
  std::vector<float> tab(static_cast<size_t>(max_pos) * 128);
  for (int p = 0; p < max_pos; ++p) {
    for (int i = 0; i < 64; ++i) {
      const double inv_freq = 1.0 / std::pow(10000.0, 2.0 * i / 128.0);
      const double ang = static_cast<double>(p) * inv_freq;
      tab[static_cast<size_t>(p) * 128 + 2 * i] = static_cast<float>(std::cos(ang));
      tab[static_cast<size_t>(p) * 128 + 2 * i + 1] = static_cast<float>(std::sin(ang));
    }
  }
  rope_ = DevMem(tab.size() * 4);
  check_cuda(cudaMemcpy(rope_.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice), "rope upload");
}

Runtime::~Runtime() {
  for (StageSlot& s : ring_)
    if (s.done) cudaEventDestroy(s.done);
  for (auto& g : graphs_) cudaGraphExecDestroy(g.second.exec);
}

const void* Runtime::act_tmap(const void* base, int rows, int cols, int box_rows) {
  auto key = std::make_tuple(base, rows, cols, box_rows);
  auto it = tmaps_.find(key);
  if (it != tmaps_.end()) return it->second.data();
  std::vector<unsigned char> raw(128 + 64);
  // CUtensorMap must be 64-byte aligned; std::vector data is 16-aligned, so
  // keep an aligned copy inside the buffer.
  unsigned char* aligned = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw.data()) + 63) & ~uintptr_t(63));
  if (!make_tmap_bf16(aligned, base, rows, cols, static_cast<uint64_t>(cols) * 2, box_rows))
    throw std::runtime_error("act tensor map encode failed");
  std::vector<unsigned char> stored(aligned, aligned + 128);
  auto ins = tmaps_.emplace(key, std::move(stored));
  return ins.first->second.data();
}

void Runtime::gemm(const void* w_tiled, const void* x, int M, int N, int K, void* out, int ldo, int epi,
                   Workspace& ws, cudaStream_t stream) {
  // The X map is viewed over max(M, 256) rows: buffers are sized for it and
  // rows past M are never stored.
  const int rows = std::max(M, 256);
  GemmArgs g{};
  g.w_tiled = w_tiled;
  g.tmap_x = act_tmap(x, rows, K, gemm_n_tile(M));
  if (M > 256) g.tmap_x128 = act_tmap(x, rows, K, 128);  // 2-SM prefill path (gemm_2sm.cu)
  // CTA-pair mode (MUX_GEMM_PAIR). Not for tensor-parallel units: when the
  // ranks of a mesh share one GPU (the tests), a rank's rmsnorm_tp spinners
  // can leave no TPC with two free SMs for the peer's cluster launches.
  if (gemm_n_tile(M) >= 16 && w_tiled != nullptr && !ws.tp) {
    g.tmap_x_half = act_tmap(x, rows, K, gemm_n_tile(M) / 2);
    g.tmap_w_rows = w_rows_tmap(w_tiled, N, K);
  }
  g.tmap_out = out_tmap(out, epi, M, N, ldo);
  g.out = out;
  g.partials = ws.gemm_partials.as<float>();
  g.flags = ws.gemm_flags.as<int>();
  g.epoch = ++ws.gemm_epoch;
  g.grid = ws.sms;  // persistent grid = the partition's SMs
  g.min_iters = gemm_min_iters_;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldo = ldo;
  g.epi = static_cast<Epilogue>(epi);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool timed = gemm_timer_ != nullptr && M <= 256;
  if (timed) {
    e0 = gemm_timer_->get();
    e1 = gemm_timer_->get();
    check_cuda(cudaEventRecord(e0, stream), "timer");
  }
  check_cuda(gemm_bf16_tn(g, stream), "gemm");
  if (timed) {
    check_cuda(cudaEventRecord(e1, stream), "timer");
    gemm_timer_->pending.emplace_back(e0, e1);
    gemm_timer_->pending_bytes += static_cast<double>(N) * K * 2;  // decode: the weights, streamed once
  }
  launches_ += 1;
}

const void* Runtime::w_rows_tmap(const void* w_tiled, int N, int K) {
  auto key = std::make_tuple(w_tiled, N, K, -1);
  auto it = tmaps_.find(key);
  if (it != tmaps_.end()) return it->second.data();
  std::vector<unsigned char> raw(128 + 64);
  unsigned char* aligned = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw.data()) + 63) & ~uintptr_t(63));
  if (!make_tmap_w_rows(aligned, w_tiled, N, K)) throw std::runtime_error("weight-row tensor map encode failed");
  auto ins = tmaps_.emplace(key, std::vector<unsigned char>(aligned, aligned + 128));
  return ins.first->second.data();
}

const void* Runtime::out_tmap(const void* out, int epi, int M, int N, int ldo) {
  auto key = std::make_tuple(out, M, N * 8 + epi, ldo);
  auto it = out_tmaps_.find(key);
  if (it != out_tmaps_.end()) return it->second.data();
  std::vector<unsigned char> raw(128 + 64);
  unsigned char* aligned = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw.data()) + 63) & ~uintptr_t(63));
  if (!make_tmap_gemm_out(aligned, out, epi, M, N, ldo)) throw std::runtime_error("out tensor map encode failed");
  auto ins = out_tmaps_.emplace(key, std::vector<unsigned char>(aligned, aligned + 128));
  return ins.first->second.data();
}

void Runtime::row_parallel_norm(const void* w_tiled, const void* x, int M, int N, int K, int s, const float* norm_w,
                                float eps, Workspace& ws, cudaStream_t stream) {
  TpLink& tp = *ws.tp;
  if (!tp.connected()) throw std::logic_error("tensor parallel: mailbox peers not connected");
  // slot rows are packed at this model's hidden size (<= the unit's largest)
  if (M > tp.rows || N > tp.hidden) throw std::invalid_argument("tensor parallel: mailbox too small");
  const int rows = std::max(M, 256);
  GemmArgs g{};
  g.w_tiled = w_tiled;
  g.tmap_x = act_tmap(x, rows, K, gemm_n_tile(M));
  float* own = tp.slot(tp.rank, s, tp.rank);
  g.tmap_out = out_tmap(own, kEpiStoreF32, M, N, N);
  g.out = own;
  for (int r = 0, k = 0; r < tp.size; ++r) {
    g.signal[r] = tp.counter(r, s);
    if (r != tp.rank) g.tmap_peers[k++] = out_tmap(tp.slot(r, s, tp.rank), kEpiStoreF32, M, N, N);
  }
  g.n_peers = tp.size - 1;
  g.n_signal = tp.size;
  int grid = 0;
  g.grid_out = &grid;
  g.partials = ws.gemm_partials.as<float>();
  g.flags = ws.gemm_flags.as<int>();
  g.epoch = ++ws.gemm_epoch;
  g.grid = ws.sms;
  g.min_iters = gemm_min_iters_;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ldo = N;
  g.epi = Epilogue::kStoreF32;
  check_cuda(gemm_bf16_tn(g, stream), "gemm (row-parallel)");
  // Every rank launches the same grid for the same shapes (equal partitions),
  // so each counter receives grid signals from each of the tp ranks.
  tp.expected[s] += static_cast<uint32_t>(grid) * tp.size;
  check_cuda(rmsnorm_tp(ws.resid.as<float>(), tp.slot(tp.rank, s, 0), static_cast<int64_t>(tp.slot_floats()), tp.size,
                        tp.counter(tp.rank, s), tp.expected[s], norm_w, ws.xn.p, M, N, eps, stream),
             "rmsnorm_tp");
  launches_ += 2;
}

void Runtime::upload_rows(muxsim::BlockPool& bp, int llm, Llama& m, cudaStream_t stream) {
  check_cuda(cudaSetDevice(device_), "cudaSetDevice");  // units of one process may sit on different GPUs
  std::vector<muxsim::RowDelta>& pend = bp.pending_rows(llm);
  if (pend.empty()) return;
  // A tensor-parallel rank holds heads [r*H/tp, (r+1)*H/tp) of every row:
  // its columns (layer, local head, kv) of the mesh-wide row record, whose
  // ids are already rank-local (BlockPool::enable_physical(tp)).
  // Two pool forms: the unit's own pool registers the rank's head slice
  // (row width W, rank-local ids, shards 1); a mesh-wide pool (the lockstep
  // engine's shared decisions) registers full rows sharded over the ranks.
  const int W = m.row_width();
  const int rank = m.dims().tp_rank, hl = m.dims().heads;
  const int tp = bp.row_width(llm) == W ? 1 : m.dims().tp_size;
  if (W * tp != bp.row_width(llm)) throw std::logic_error("upload_rows: row width mismatch");
  if (tp > 1 && bp.shards() != tp) throw std::logic_error("upload_rows: pool ids are not sharded over the TP ranks");
  const size_t n = pend.size();
  const size_t meta_ints = (3 * n + 3) & ~size_t(3);  // keep the id block 16-byte aligned
  const size_t need = (meta_ints + n * static_cast<size_t>(W)) * 4;
  StageSlot& slot = ring_[ring_next_];
  ring_next_ = (ring_next_ + 1) % 4;
  if (slot.done == nullptr) check_cuda(cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming), "event");
  // The slot's previous copy + scatter must be complete before it is reused.
  check_cuda(cudaEventSynchronize(slot.done), "stage wait");
  if (need > slot.cap) {
    // Grow without freeing on the job path (cudaFree / cudaFreeHost
    // synchronise the device): the old buffers retire until destruction.
    size_t cap = std::max<size_t>({need, slot.cap * 2, 1 << 20});
    retired_dev_.push_back(std::move(slot.dev));
    if (slot.host) retired_host_.push_back(std::move(slot.host));
    slot.dev = DevMem(cap);
    slot.host = std::make_unique<PinnedMem>(cap);
    slot.cap = cap;
  }
  int32_t* meta = slot.host->as<int32_t>();
  int32_t* ids = meta + meta_ints;
  for (size_t i = 0; i < n; ++i) {
    const muxsim::RowDelta& d = pend[i];
    if (d.slot >= m.max_slots() || d.row >= m.max_rows() || d.rowrec >= m.max_rowrecs())
      throw std::runtime_error("upload_rows: device table capacity exceeded (slot " +
                               std::to_string(d.slot) + ", row " + std::to_string(d.row) + ")");
    meta[3 * i] = d.slot;
    meta[3 * i + 1] = d.row;
    meta[3 * i + 2] = d.rowrec;
    const int32_t* src = bp.row_ids(llm, d.rowrec);
    for (int j = 0; j < W; ++j) {
      // local column (l*hl + h)*2 + kv  <-  mesh column (l*hl*tp + rank*hl + h)*2 + kv
      const int lh = j >> 1, l = lh / hl, h = lh - l * hl;
      const int32_t id = tp == 1 ? src[j] : src[((l * hl * tp + rank * hl + h) << 1) | (j & 1)];
      if (id >= pool_blocks_) throw std::runtime_error("upload_rows: block id beyond the device pool");
      ids[i * W + j] = id;
    }
  }
  check_cuda(cudaMemcpyAsync(slot.dev.p, slot.host->p, need, cudaMemcpyHostToDevice, stream), "stage copy");
  TableUpdateArgs t{};
  t.meta = slot.dev.as<int32_t>();
  t.ids = slot.dev.as<int32_t>() + meta_ints;
  t.rowrec = m.rowrec.as<int32_t>();
  t.rowlist = m.rowlist.as<int32_t>();
  t.n = static_cast<int>(n);
  t.row_width = W;
  t.max_rows = m.max_rows();
  check_cuda(table_update(t, stream), "table_update");
  launches_ += 1;
  check_cuda(cudaEventRecord(slot.done, stream), "stage record");
  pend.clear();
}

void Runtime::decode(Llama& m, Workspace& ws, int n, const int32_t* slots_host, const int32_t* ctx_host,
                     const int32_t* tokens_host, int32_t* out_host, cudaStream_t stream,
                     AttnTimer* timer) {
  if (n <= 0) return;
  check_cuda(cudaSetDevice(device_), "cudaSetDevice");  // units of one process may sit on different GPUs
  if (n > ws.max_tokens || n > ws.max_decode)
    throw std::invalid_argument("decode: batch of " + std::to_string(n) + " exceeds the unit's max_batch " +
                                std::to_string(ws.max_decode));
  const ModelDims& d = m.dims();
  const int T = std::max(ws.max_tokens, 16);
  int32_t* h = ws.stage_begin();
  for (int i = 0; i < n; ++i) {
    h[T + i] = slots_host[i];
    h[2 * T + i] = ctx_host[i];
    h[4 * T + i] = ctx_host[i] - 1;
    if (tokens_host) h[i] = tokens_host[i];
  }
  // K1 visits members longest-context first (LPT): the ragged tail of the
  // launch is then made of the shortest requests.
  int32_t* order = h + 3 * T;
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order, order + n, [&](int32_t x, int32_t y) { return ctx_host[x] > ctx_host[y]; });
  const int hid = d.hidden, H = d.heads, L = d.layers;
  int max_ctx = 0;
  for (int i = 0; i < n; ++i) max_ctx = std::max(max_ctx, ctx_host[i]);
  const int max_rows_req = (max_ctx + 15) / 16;
  // KV splits: enough CTAs to fill the GPU a few times over.
  int splits = 1;
  // (the last split merges in-kernel, so small batches can afford ~2 rows per split)
  while (splits < kMaxKvSplits && n * H * splits < 4 * ws.sms && (max_rows_req + splits * 2 - 1) / (splits * 2) >= 2)
    splits *= 2;
  while ((max_rows_req + splits - 1) / splits > decode_attention_max_rows_per_split()) splits *= 2;
  if (splits > kMaxKvSplits)  // the split scratch holds kMaxKvSplits per (member, head)
    throw std::invalid_argument("decode: context of " + std::to_string(max_ctx) + " tokens exceeds K1's " +
                                std::to_string(kMaxKvSplits * decode_attention_max_rows_per_split() * 16));
  h[5 * T] = std::max(1, (max_rows_req + splits - 1) / splits);  // K1 rows per split (seq_start[0])
  ws.stage_commit(5 * static_cast<size_t>(T) + 1, stream);

  // Everything below is a pure function of (model, workspace, n, splits,
  // whether tokens are staged): it is enqueued directly, or captured once
  // into a CUDA graph and replayed (per-step data all comes through the
  // staged metadata and device tables).
  auto enqueue = [&]() {
  if (!tokens_host) {
    check_cuda(launch(gather_last_tok, dim3((n + 127) / 128), dim3(128), 0, stream, m.last_tok.as<int32_t>(),
                      ws.slots, ws.tokens, n), "gather_last_tok");
    launches_ += 1;
  }
  check_cuda(embed_rmsnorm(m.embed.p, ws.tokens, m.attn_norm[0].as<float>(), ws.resid.as<float>(), ws.xn.p,
                           n, hid, d.norm_eps, stream), "embed");
  launches_ += 1;
  DecodeAttnArgs at{};
  at.q = ws.q.p;
  at.pool = pool_.p;
  at.rowrec = m.rowrec.as<int32_t>();
  at.rowlist = m.rowlist.as<int32_t>();
  at.slots = ws.slots;
  at.ctx = ws.ctx;
  at.order = ws.tok_slot;  // staged above
  at.out = ws.attn.p;
  at.part_o = ws.attn_part_o.as<float>();
  at.part_ml = ws.attn_part_ml.as<float>();
  at.split_count = ws.attn_split_count.as<int>();  // the last split of each (member, head) merges
  at.B = n;
  at.H = H;
  at.max_rows = m.max_rows();
  at.row_width = m.row_width();
  at.splits = splits;
  at.rows_per_split = decode_attention_max_rows_per_split();  // bound; the value is staged
  at.rows_per_split_dev = ws.seq_start;
  at.scale_log2 = 1.4426950408889634f / std::sqrt(128.f);
  // Algorithmic bytes of one K1 launch: K+V of every cached token, q in, o out.
  double attn_bytes = 0.0;
  for (int i = 0; i < n; ++i) attn_bytes += static_cast<double>(ctx_host[i]) * H * 128 * 2 * 2;
  attn_bytes += static_cast<double>(n) * H * 128 * 2 * 2;

  AppendArgs ap{};
  ap.qkv = ws.qkv.p;
  ap.q_out = ws.q.p;
  ap.pool = pool_.p;
  ap.rowrec = m.rowrec.as<int32_t>();
  ap.rowlist = m.rowlist.as<int32_t>();
  ap.tok_slot = ws.slots;
  ap.tok_pos = ws.tok_pos;
  ap.rope = rope_.as<float>();
  ap.T = n;
  ap.H = H;
  ap.max_rows = m.max_rows();
  ap.row_width = m.row_width();
  ap.rope_positions = max_pos_;

  // Debug (MUX_DEBUG_SKIP bitmask; outputs are garbage, timings are not): the
  // marginal in-step cost of a kernel class. 1 = K2, 2 = RMSNorm, 4 = K1,
  // 8 = RMSNorm over one row only (the launch boundary without the work).
  const int dbg_skip = dbg_skip_;
  for (int l = 0; l < L; ++l) {
    ap.layer = l;
    gemm(m.wqkv[l].p, ws.xn.p, n, m.qkv_cols(), hid, ws.qkv.p, m.qkv_cols(), kEpiStoreBf16, ws, stream);
    if (!(dbg_skip & 1)) {
      check_cuda(kv_append(ap, stream), "kv_append");
      launches_ += 1;
    }
    at.layer = l;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timer) {
      e0 = timer->get();
      e1 = timer->get();
      check_cuda(cudaEventRecord(e0, stream), "timer");
    }
    if (!(dbg_skip & 4)) {
      check_cuda(decode_attention(at, false, stream), "decode_attention");
      launches_ += 1;
    }
    if (timer) {
      check_cuda(cudaEventRecord(e1, stream), "timer");
      timer->pending.emplace_back(e0, e1);
      timer->pending_bytes += attn_bytes;
    }
    const float* next_norm = l + 1 < L ? m.attn_norm[l + 1].as<float>() : m.final_norm.as<float>();
    if (d.tp_size > 1) {
      row_parallel_norm(m.wo[l].p, ws.attn.p, n, hid, H * 128, 0, m.ffn_norm[l].as<float>(), d.norm_eps, ws, stream);
      gemm(m.wgu[l].p, ws.xn.p, n, 2 * d.ffn, hid, ws.act.p, d.ffn, kEpiSilu, ws, stream);
      row_parallel_norm(m.wdown[l].p, ws.act.p, n, hid, d.ffn, 1, next_norm, d.norm_eps, ws, stream);
      continue;
    }
    gemm(m.wo[l].p, ws.attn.p, n, hid, H * 128, ws.resid.p, hid, kEpiResidual, ws, stream);
    if (!(dbg_skip & 2)) {
      check_cuda(rmsnorm_rows(ws.resid.as<float>(), m.ffn_norm[l].as<float>(), ws.xn.p, (dbg_skip & 8) ? 1 : n, hid,
                              d.norm_eps, stream, ws.sms),
                 "rmsnorm");
      launches_ += 1;
    }
    gemm(m.wgu[l].p, ws.xn.p, n, 2 * d.ffn, hid, ws.act.p, d.ffn, kEpiSilu, ws, stream);
    gemm(m.wdown[l].p, ws.act.p, n, hid, d.ffn, ws.resid.p, hid, kEpiResidual, ws, stream);
    if (!(dbg_skip & 2)) {
      check_cuda(rmsnorm_rows(ws.resid.as<float>(), next_norm, ws.xn.p, (dbg_skip & 8) ? 1 : n, hid, d.norm_eps,
                              stream, ws.sms),
                 "rmsnorm");
      launches_ += 1;
    }
  }
  gemm(m.lm_head.p, ws.xn.p, n, d.vocab, hid, ws.logits.p, d.vocab, kEpiStoreF32, ws, stream);
  check_cuda(argmax_rows(ws.logits.as<float>(), n, d.vocab, ws.out_tok, stream), "argmax");
  check_cuda(launch(scatter_last_tok, dim3((n + 127) / 128), dim3(128), 0, stream, m.last_tok.as<int32_t>(),
                    ws.slots, ws.out_tok, n), "scatter_last_tok");
  launches_ += 2;
  };
  // Graphs: single-rank decode without per-launch timing (the TP path's
  // mailbox counters advance per call; timers record events per launch).
  if (use_graphs_ && timer == nullptr && gemm_timer_ == nullptr && d.tp_size == 1 && dbg_skip_ == 0) {
    const GraphKey key{&m, &ws, n, splits, tokens_host != nullptr};
    auto it = graphs_.find(key);
    // capture on a key's second use: a batch size seen once (serving under
    // churn) is cheaper to enqueue than to capture and instantiate
    const bool capture = it == graphs_.end() && ++graph_seen_[key] >= 2;
    if (it == graphs_.end() && !capture) {
      enqueue();
    } else {
    if (it == graphs_.end()) {
      if (graphs_.size() >= kMaxGraphs) {  // bounded cache: drop the least recently used
        auto lru = graphs_.begin();
        for (auto g = graphs_.begin(); g != graphs_.end(); ++g)
          if (g->second.used < lru->second.used) lru = g;
        cudaGraphExecDestroy(lru->second.exec);
        graph_seen_.erase(lru->first);
        graphs_.erase(lru);
      }
      const int64_t l0 = launches_;
      check_cuda(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "graph capture");
      cudaGraph_t graph = nullptr;
      try {
        enqueue();
      } catch (...) {
        cudaStreamEndCapture(stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      check_cuda(cudaStreamEndCapture(stream, &graph), "graph capture end");
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      check_cuda(ie, "graph instantiate");
      it = graphs_.emplace(key, GraphEntry{exec, launches_ - l0, 0}).first;
      launches_ = l0;
      graph_captures_ += 1;
    }
    it->second.used = ++graph_clock_;
    check_cuda(cudaGraphLaunch(it->second.exec, stream), "graph launch");
    launches_ += it->second.kernels;
    }
  } else {
    enqueue();
  }
  if (out_host)
    check_cuda(cudaMemcpyAsync(out_host, ws.out_tok, n * 4, cudaMemcpyDeviceToHost, stream), "out copy");
}

void Runtime::prefill(Llama& m, Workspace& ws, int n, const int32_t* slots_host, const int32_t* lens_host,
                      const int32_t* tokens_host, int32_t* out_host, cudaStream_t stream) {
  if (n <= 0) return;
  check_cuda(cudaSetDevice(device_), "cudaSetDevice");  // units of one process may sit on different GPUs
  const ModelDims& d = m.dims();
  int T = 0;
  for (int i = 0; i < n; ++i) T += lens_host[i];
  if (T > ws.max_tokens) throw std::invalid_argument("prefill: tokens exceed workspace");
  const int cap = std::max(ws.max_tokens, 16);
  int32_t* h = ws.stage_begin();
  int t = 0;
  for (int i = 0; i < n; ++i) {
    h[cap + i] = slots_host[i];
    h[5 * cap + i] = t;
    for (int p = 0; p < lens_host[i]; ++p, ++t) {
      h[t] = tokens_host[t];
      h[3 * cap + t] = slots_host[i];
      h[4 * cap + t] = p;
    }
    h[7 * cap + 1 + i] = t - 1;
  }
  h[5 * cap + n] = T;
  // K3 work list: (sequence, 128-query tile), longest causal row first.
  int n_tiles = 0;
  int32_t* tiles = h + 2 * cap;
  int max_qt = 0;
  for (int i = 0; i < n; ++i) max_qt = std::max(max_qt, (lens_host[i] - 1) / 128);
  for (int qt = max_qt; qt >= 0; --qt)
    for (int i = 0; i < n; ++i)
      if (qt * 128 < lens_host[i]) tiles[n_tiles++] = (i << 16) | qt;
  ws.stage_commit(8 * static_cast<size_t>(cap) + 8, stream);

  const int hid = d.hidden, H = d.heads, L = d.layers;
  check_cuda(embed_rmsnorm(m.embed.p, ws.tokens, m.attn_norm[0].as<float>(), ws.resid.as<float>(), ws.xn.p,
                           T, hid, d.norm_eps, stream), "embed");
  launches_ += 1;
  AppendArgs ap{};
  ap.qkv = ws.qkv.p;
  ap.q_out = ws.q.p;
  ap.pool = pool_.p;
  ap.rowrec = m.rowrec.as<int32_t>();
  ap.rowlist = m.rowlist.as<int32_t>();
  ap.tok_slot = ws.tok_slot;
  ap.tok_pos = ws.tok_pos;
  ap.rope = rope_.as<float>();
  ap.T = T;
  ap.H = H;
  ap.max_rows = m.max_rows();
  ap.row_width = m.row_width();
  ap.rope_positions = max_pos_;
  PrefillAttnArgs pa{};
  pa.q = ws.q.p;
  pa.qkv = ws.qkv.p;
  pa.out = ws.attn.p;
  pa.seq_start = ws.seq_start;
  pa.tiles = ws.ctx;  // staged above
  const int view_rows = std::max(cap, 256);
  pa.tmap_q = act_tmap(ws.q.p, view_rows, H * 128, 128);
  pa.tmap_qkv = act_tmap(ws.qkv.p, view_rows, 3 * H * 128, 128);
  pa.n_tiles = n_tiles;
  pa.nseq = n;
  pa.H = H;
  pa.T = T;
  pa.scale_log2 = 1.4426950408889634f / std::sqrt(128.f);
  pa.max_ctas = ws.sms;
  for (int l = 0; l < L; ++l) {
    ap.layer = l;
    gemm(m.wqkv[l].p, ws.xn.p, T, m.qkv_cols(), hid, ws.qkv.p, m.qkv_cols(), kEpiStoreBf16, ws, stream);
    check_cuda(kv_append(ap, stream), "kv_append");
    launches_ += 1;
    check_cuda(prefill_attention(pa, stream), "prefill_attention");
    launches_ += 1;
    const float* next_norm = l + 1 < L ? m.attn_norm[l + 1].as<float>() : m.final_norm.as<float>();
    if (d.tp_size > 1) {
      row_parallel_norm(m.wo[l].p, ws.attn.p, T, hid, H * 128, 0, m.ffn_norm[l].as<float>(), d.norm_eps, ws, stream);
      gemm(m.wgu[l].p, ws.xn.p, T, 2 * d.ffn, hid, ws.act.p, d.ffn, kEpiSilu, ws, stream);
      row_parallel_norm(m.wdown[l].p, ws.act.p, T, hid, d.ffn, 1, next_norm, d.norm_eps, ws, stream);
      continue;
    }
    gemm(m.wo[l].p, ws.attn.p, T, hid, H * 128, ws.resid.p, hid, kEpiResidual, ws, stream);
    check_cuda(rmsnorm_rows(ws.resid.as<float>(), m.ffn_norm[l].as<float>(), ws.xn.p, T, hid, d.norm_eps, stream),
               "rmsnorm");
    launches_ += 1;
    gemm(m.wgu[l].p, ws.xn.p, T, 2 * d.ffn, hid, ws.act.p, d.ffn, kEpiSilu, ws, stream);
    gemm(m.wdown[l].p, ws.act.p, T, hid, d.ffn, ws.resid.p, hid, kEpiResidual, ws, stream);
    check_cuda(rmsnorm_rows(ws.resid.as<float>(), next_norm, ws.xn.p, T, hid, d.norm_eps, stream), "rmsnorm");
    launches_ += 1;
  }
  check_cuda(gather_rows_bf16(ws.xn.p, ws.last_rows, ws.xlast.p, n, hid, stream), "gather");
  launches_ += 1;
  gemm(m.lm_head.p, ws.xlast.p, n, d.vocab, hid, ws.logits.p, d.vocab, kEpiStoreF32, ws, stream);
  check_cuda(argmax_rows(ws.logits.as<float>(), n, d.vocab, ws.out_tok, stream), "argmax");
  check_cuda(launch(scatter_last_tok, dim3((n + 127) / 128), dim3(128), 0, stream, m.last_tok.as<int32_t>(),
                    ws.slots, ws.out_tok, n), "scatter_last_tok");
  launches_ += 2;
  if (out_host)
    check_cuda(cudaMemcpyAsync(out_host, ws.out_tok, n * 4, cudaMemcpyDeviceToHost, stream), "out copy");
}

}  // namespace mux
