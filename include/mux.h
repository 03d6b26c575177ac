/*
 * mux.h -- C ABI of the B200-native MuxServe hot path (libmux.so).
 *
 * Plain C: pointers, sizes and status codes only; no C++ or torch types cross
 * it. Every entry point names the reference interface it replaces
 * (/root/reference/proj/...). The reference has no FFI of its own (its API is
 * C++), so this is the surface a foreign host (ctypes, cgo,
 * JNI) binds; INTEGRATION.md shows the bindings.
 *
 * Status codes mirror the reference's exception classes:
 *   MUX_OK             success
 *   MUX_EINVAL   (1)   std::invalid_argument / std::domain_error / ConfigError
 *   MUX_EINFEAS  (2)   InfeasibleError          (/root/reference/proj/tools/muxsim.cpp:51-53)
 *   MUX_EINTERNAL(3)   std::logic_error and everything else (incl. CUDA errors)
 * mux_last_error() returns the message of the last failure on this thread
 * (the reference's what() text where one exists).
 *
 * Device pointers are raw CUDA pointers on the unit's device; host pointers
 * are borrowed for the duration of the call. Calls are stream-ordered on the
 * partition they name; mux_unit_sync() waits for all of them.
 */
#ifndef MUX_H_
#define MUX_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MUX_API __attribute__((visibility("default")))
#else
#define MUX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MUX_OK 0
#define MUX_EINVAL 1
#define MUX_EINFEAS 2
#define MUX_EINTERNAL 3

/* AllocResult.error (kv_manager.hpp:32-39): 0 = None (ok), 1 = Pool, 2 = Quota. */
#define MUX_ALLOC_OK 0
#define MUX_ALLOC_POOL 1
#define MUX_ALLOC_QUOTA 2

MUX_API const char* mux_last_error(void);
MUX_API const char* mux_version(void);

/* ---- geometry and quotas --------------------------------------------- */

/* blocks_for_tokens (kv_manager.hpp:28-29, kv_manager.cpp:30-35). */
MUX_API int mux_blocks_for_tokens(int num_layers, int num_heads, int block_tokens, int64_t tokens,
                          int64_t* out);

/* init_token_block_quota (kv_manager.hpp:117-119, kv_manager.cpp:222-280). */
MUX_API int mux_init_token_block_quota(int n, const double* rate, const double* blocks_per_token,
                               const double* mean_request_tokens, int64_t kv_blocks,
                               double floor_frac, int64_t* out_quotas);

/* adapt_quota (kv_manager.hpp:132-135, kv_manager.cpp:282-323). */
MUX_API int mux_adapt_quota(int n, const double* utilizations, const int64_t* quotas,
                    int64_t floor_blocks, double low_mark, double high_mark, double step_frac,
                    int64_t* out_quotas);

/* ---- unified head-wise block pool (BlockPool, kv_manager.hpp:48-105) ---- */

typedef struct mux_pool mux_pool;

/* BlockPool(total_blocks) (kv_manager.hpp:50). physical != 0 also assigns
 * physical 4 KiB head-block ids (the B200 extension); physical = k > 1 shards
 * them head-wise over k tensor-parallel ranks, each rank's ids in
 * [0, total_blocks / k) (a TP mesh's per-GPU pool slices). */
MUX_API int mux_pool_create(int64_t total_blocks, int physical, mux_pool** out);
MUX_API void mux_pool_destroy(mux_pool* pool);
/* register_llm (kv_manager.hpp:53). */
MUX_API int mux_pool_register_llm(mux_pool* pool, int llm, int num_layers, int num_heads, int head_dim,
                          int bytes_per_element, int block_tokens);
/* admit (kv_manager.hpp:59-60); *result = MUX_ALLOC_*. */
MUX_API int mux_pool_admit(mux_pool* pool, int llm, int64_t request_id, int64_t prompt_tokens,
                   int64_t total_tokens, int* result);
/* alloc (kv_manager.hpp:65). */
MUX_API int mux_pool_alloc(mux_pool* pool, int llm, int64_t request_id, int64_t add_tokens,
                   int enforce_quota, int* result);
/* The same alloc for n members of one decode round (one call instead of n):
 * results[i] is the AllocResult code of rids[i]; identical to n calls. */
MUX_API int mux_pool_alloc_n(mux_pool* pool, int llm, int n, const int64_t* request_ids, int64_t add_tokens,
                             int enforce_quota, int* results);
/* free_request (kv_manager.hpp:69). */
MUX_API int mux_pool_free_request(mux_pool* pool, int llm, int64_t request_id);
/* set_quota / quota / used / committed / request_tokens (kv_manager.hpp:71-79). */
MUX_API int mux_pool_set_quota(mux_pool* pool, int llm, int64_t blocks);
MUX_API int mux_pool_llm_stats(const mux_pool* pool, int llm, int64_t* quota, int64_t* used,
                       int64_t* committed);
MUX_API int mux_pool_request_tokens(const mux_pool* pool, int llm, int64_t request_id, int64_t* tokens);
/* free_blocks / total_blocks / committed_total (kv_manager.hpp:80-83). */
MUX_API int mux_pool_totals(const mux_pool* pool, int64_t* free_blocks, int64_t* total_blocks,
                    int64_t* committed_total);
/* check_conservation (kv_manager.hpp:87). */
MUX_API int mux_pool_check(const mux_pool* pool);
/* Physical block table of one request: [rows][layer][head][K/V] int32. */
MUX_API int mux_pool_block_table(const mux_pool* pool, int llm, int64_t request_id, int32_t* out,
                         int64_t capacity, int64_t* n_out);
MUX_API int mux_pool_slot(const mux_pool* pool, int llm, int64_t request_id, int* slot);

/* ---- engine: run_simulation (sim_engine.hpp:81-83) -------------------- */

typedef struct {
  const char* name;
  int num_layers, num_heads, head_dim, hidden_size;
  int64_t weight_bytes;
  int bytes_per_element;
  double rate, mean_prompt_tokens, mean_output_tokens;  /* LlmEntry (placement.hpp:38-43) */
  /* B200 execution (ignored when priced): FFN width and vocabulary. */
  int ffn, vocab;
} mux_llm_entry;

typedef struct {
  int unit;           /* index into the placement's unit list */
  int llm;            /* index into the entries array */
  int tp_degree;
  double num_sm;
} mux_placed_llm;

typedef struct {
  int num_nodes, gpus_per_node;
  int64_t gpu_memory_bytes;
  int n_units;
  const int* unit_mesh_size;   /* [n_units] gpus per mesh (tp) */
  int n_placed;
  const mux_placed_llm* placed;
  /* LatencyProfile (cost_model.hpp:33-50); NULL fields use the defaults. */
  const double* profile;       /* 7 doubles in declaration order, or NULL */
  /* EngineParams (sim_engine.hpp:15-28) */
  int scheduler;               /* 0 ADBS, 1 FCFS, 2 round-robin */
  double kappa, quota_period_s;
  int64_t token_budget;
  int block_tokens;
  double warmup_s, decode_sm, prefill_min_sm, activation_reserve_frac, quota_floor_frac;
  /* NULL: the reference's decode cost form. Else 4 doubles {decode_fixed_ms,
   * decode_row_ms, decode_bctx_ms, decode_sm_exponent}: the HBM-bound form
   * (B200 extension,
   * LatencyProfile::decode_form 1; DESIGN §4 "measured latency profile"). */
  const double* decode_hbm;
  /* NULL: QuotaAdaptParams defaults. Else 3 doubles {low_mark, high_mark,
   * step_frac} (kv_manager.hpp QuotaAdaptParams; config keys
   * sim.quota_low_mark / quota_high_mark / quota_step_frac, config.cpp:242-244). */
  const double* quota_adapt;
  /* NULL: the reference's tp_speedup = eta * tp (cost_model.cpp:43-47). Else
   * 2 doubles {allreduce_alpha_ms, allreduce_ms_per_mib}: a tp > 1 job costs
   * t(1)/tp + 2 * num_layers * (alpha + per_mib * tokens * hidden * 4 B / MiB)
   * (B200 extension, LatencyProfile::tp_scaled; DESIGN §4 "f1"). */
  const double* tp_allreduce;
} mux_sim_config;

typedef struct {
  int64_t id;
  int llm;                     /* entry index */
  double arrival_s;
  int prompt_len, output_len;
} mux_request;

typedef struct {
  int64_t id;
  int llm;
  double arrival_s, first_token_s, done_s;
  int prompt_len, output_len;
} mux_record;

/* Priced run (the reference simulator's semantics, bit-identical). */
MUX_API int mux_simulate(const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries,
                 int n_requests, const mux_request* trace, mux_record* records_out);

/* Priced run plus the per-unit pool statistics behind the reference's
 * poolstats.json / metrics.json "units" (sim_engine.hpp:48-71,
 * commands.cpp:89-121). Release with mux_sim_stats_destroy. */
typedef struct mux_sim_stats mux_sim_stats;
typedef struct {
  int unit;
  int64_t total_blocks;
  int n_llms;
  int64_t n_samples;
} mux_unit_stats;
typedef struct {
  int llm;                     /* entry index */
  double rate, avg_used_blocks;
  int64_t final_quota_blocks;
  double resource_usage;
} mux_unit_llm_stats;
typedef struct {
  double t_s;
  int llm;                     /* entry index */
  int64_t used_blocks, quota_blocks;
} mux_pool_sample;
MUX_API int mux_simulate_stats(const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries,
                               int n_requests, const mux_request* trace, mux_record* records_out,
                               mux_sim_stats** stats_out);
MUX_API int mux_sim_stats_units(const mux_sim_stats* stats, int* n_units);
MUX_API int mux_sim_stats_unit(const mux_sim_stats* stats, int unit, mux_unit_stats* out);
MUX_API int mux_sim_stats_llms(const mux_sim_stats* stats, int unit, mux_unit_llm_stats* out /* [n_llms] */);
MUX_API int mux_sim_stats_samples(const mux_sim_stats* stats, int unit, mux_pool_sample* out /* [n_samples] */);
MUX_API void mux_sim_stats_destroy(mux_sim_stats* stats);

/* Realizable parallel candidates (llm_parallel_candidates,
 * placement.cpp:57-103, plus the engine's shardability filter: tp must divide
 * num_heads and, when entry.ffn > 0, the FFN width). One
 * candidate per (model, realizable tp in tp_list) in entry order; llm = entry
 * index. Profile blocks as in mux_sim_config (NULL = defaults). sm_list NULL
 * or n_sm 0 = {0.1, ..., 1.0}. MUX_EINFEAS (reference InfeasibleError) when a
 * model has no width that both fits and shards. */
typedef struct {
  int llm;
  int tp_degree;
  double num_sm;
  int batch;
  double est_tpt;
  int saturated;
} mux_candidate;
MUX_API int mux_parallel_candidates(int n_entries, const mux_llm_entry* entries, int num_nodes, int gpus_per_node,
                                    int64_t gpu_memory_bytes, const double* profile, const double* decode_hbm,
                                    const double* tp_allreduce, int n_tp, const int* tp_list, int n_sm,
                                    const double* sm_list, double activation_reserve_frac, int max_batch,
                                    mux_candidate* out, int capacity, int* n_out);

/* slo_reference_latency_ms (metrics.cpp:21-27): the unloaded latency a
 * request's SLO is a multiple of. profile: 7 doubles or NULL (defaults). */
MUX_API int mux_slo_reference_latency_ms(const mux_llm_entry* entry, const double* profile, int tp_degree,
                                         int prompt_len, int output_len, double* out_ms);

/* ---- kernels (device pointers; stream = cudaStream_t or NULL) --------- */

/* K1: head-wise paged decode attention for one layer (the work priced by
 * the c_ctx term of decode_step_latency, cost_model.cpp:85-94).
 * q [B][H][128] bf16, pool [blocks][16][128] bf16, rowrec [*][L*H*2] int32,
 * rowlist [slots][max_rows] int32, slots/ctx [B] int32, out [B][H][128]
 * (fp32 if out_fp32 else bf16). kv_splits = 0 picks automatically. */
MUX_API int mux_decode_attention_headwise(const void* q, const void* pool, const int32_t* rowrec,
                                  const int32_t* rowlist, const int32_t* slots,
                                  const int32_t* ctx, int B, int H, int num_layers, int layer,
                                  int max_rows, int max_ctx, void* out, int out_fp32,
                                  int kv_splits, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* K2: RoPE + KV append (the device side of BlockPool::alloc's new token,
 * scheduler.cpp:105). qkv [T][3][H][128] bf16; q_out [T][H][128] (nullable). */
MUX_API int mux_kv_append(const void* qkv, void* q_out, void* pool, const int32_t* rowrec,
                  const int32_t* rowlist, const int32_t* tok_slot, const int32_t* tok_pos,
                  const float* rope_table, int rope_positions, int T, int H, int num_layers,
                  int layer, int max_rows, void* stream);
/* K3: causal varlen prefill attention (the attention term of prefill_latency,
 * cost_model.cpp:75-83) on tcgen05. q [T][H][128] bf16 (rotated), qkv
 * [T][3][H][128] bf16 (k rotated), out [T][H][128] bf16; seq_lens (host)
 * split the T tokens into nseq prompts. Synchronises the stream. Environment
 * (read per call, tests only): MUX_K3_CTAS caps the persistent grid. */
MUX_API int mux_prefill_attention(const void* q, const void* qkv, void* out, const int32_t* seq_lens, int nseq,
                                  int H, void* stream);
/* RoPE table [positions][64][(cos,sin)] fp32, theta 10000, head_dim 128. */
MUX_API int mux_rope_table(int positions, float* out);

/* K4: D[M x N] = X[M x K] * W[N x K]^T on tcgen05 (bf16 in, fp32 acc),
 * persistent stream-K over `grid` CTAs (0 = one per SM).
 * epilogue: 0 bf16 store, 1 fp32 residual add (out += D),
 * 2 SiLU(gate)*up over interleaved rows -> bf16 [M][N/2], 3 fp32 store. */
MUX_API int mux_gemm_bf16(const void* x, const void* w, int w_tiled, int M, int N, int K, void* out,
                  int epilogue, int grid, void* stream);
/* B200 weight layout for K4: [ceil(N/128)][ceil(K/64)] contiguous, pre-swizzled
 * 16 KiB UMMA tiles (one bulk copy each). w [N][K] row-major bf16 -> out
 * (mux_weight_tiled_bytes(N, K) bytes); inverse != 0 converts back. */
MUX_API int mux_weight_tile(const void* w, int N, int K, void* out, int inverse, void* stream);
MUX_API int64_t mux_weight_tiled_bytes(int N, int K);
/* Debug: per-CTA globaltimer stamps of every K4 launch ([grid][4] u64:
 * start, MMA issue done, epilogue done, exit) into buf; NULL turns it off. */
MUX_API void mux_debug_gemm_timing(void* buf);

/* ---- device unit: one GPU, its KV pool and colocated models ---------- */

typedef struct mux_unit mux_unit;

typedef struct {
  int device;
  int n_llms;
  const mux_llm_entry* llms;
  int64_t pool_blocks;          /* logical pool (count semantics) */
  int64_t device_pool_blocks;   /* physically allocated head-blocks (0 = pool_blocks) */
  int max_batch;                /* decode members per job */
  int max_prefill_tokens;       /* prompt tokens per prefill job */
  int max_ctx;                  /* longest request (tokens) */
  int max_slots;                /* live requests per model */
  uint64_t init_seed;           /* random N(0, init_std) weights; 0 = leave for set_tensor */
  float init_std;
  int partitions;               /* concurrent job streams */
  /* SM partitions (P1, the spatial multiplexing of scheduler.cpp:50-54 /
   * sim_engine.cpp:16-18): partition_sms[p] > 0 gives partition p its own
   * green context with that many SMs (rounded up to the hardware granule),
   * carved disjointly in order; <= 0 or a NULL array = a plain stream over
   * all SMs. Kernels size their persistent grids to their partition. */
  const int* partition_sms;
  /* Tensor parallelism over the unit's mesh: this process is
   * rank tp_rank of tp_size; it holds heads [r*H/tp, (r+1)*H/tp) and FFN
   * columns [r*ffn/tp, ...) of every model (H % tp == 0, ffn % tp == 0) and a
   * pool_blocks slice of floor(total/tp) head-blocks. 0/1 = no TP. */
  int tp_rank, tp_size;
} mux_unit_config;

MUX_API int mux_unit_create(const mux_unit_config* cfg, mux_unit** out);
MUX_API void mux_unit_destroy(mux_unit* unit);
/* The unit's block pool (owned by the unit; do not destroy). */
MUX_API mux_pool* mux_unit_pool(mux_unit* unit);
/* Upload / read one weight tensor in device layout:
 *  embed, lm_head [vocab][hidden] bf16; final_norm [hidden] fp32;
 *  per layer: wqkv [3*H*128][hidden], wo [hidden][H*128],
 *  wgu [2*ffn][hidden] rows interleaved (gate_0, up_0, gate_1, ...),
 *  wdown [hidden][ffn] bf16; attn_norm, ffn_norm [hidden] fp32. */
MUX_API int mux_unit_set_tensor(mux_unit* unit, int llm, const char* name, int layer, const void* host,
                        size_t bytes);
MUX_API int mux_unit_get_tensor(mux_unit* unit, int llm, const char* name, int layer, void* host,
                        size_t bytes);
/* Fill the whole KV pool with N(0, std) bf16 (benchmarks). */
MUX_API int mux_unit_init_kv(mux_unit* unit, uint64_t seed, float std);
/* Device pointers for tests: pool, rowrec/rowlist/last_tok of a model. */
MUX_API int mux_unit_device_ptrs(mux_unit* unit, int llm, void** pool, void** rowrec, void** rowlist,
                         int* max_rows, int* row_width);
/* Prefill job (sim_engine.cpp:308 launch of a Prefill JobPlan): requests must
 * be admitted in the unit pool; tokens = concatenated prompts (host);
 * out_tokens (host, nullable) receives each request's first token. */
MUX_API int mux_unit_prefill(mux_unit* unit, int llm, int n, const int64_t* request_ids,
                     const int32_t* tokens, int32_t* out_tokens, int partition);
/* Decode job: every member already grew by one token in the pool (the ADBS
 * decode round, scheduler.cpp:105). tokens (host, nullable) = input tokens;
 * NULL uses each request's last generated token (device resident). */
MUX_API int mux_unit_decode(mux_unit* unit, int llm, int n, const int64_t* request_ids,
                    const int32_t* tokens, int32_t* out_tokens, int partition);
MUX_API int mux_unit_sync(mux_unit* unit);
/* Device-side timing: record event `slot` (0..63) on a partition stream;
 * elapsed milliseconds between two recorded slots (synchronises). */
MUX_API int mux_unit_record(mux_unit* unit, int partition, int slot);
MUX_API int mux_unit_elapsed(mux_unit* unit, int slot_a, int slot_b, float* ms);
/* Per-launch decode-attention timing (CUDA events around every K1 launch):
 * enable, then read the summed kernel milliseconds and launch count. */
MUX_API int mux_unit_attn_timing(mux_unit* unit, int enable);
MUX_API int mux_unit_attn_time(mux_unit* unit, double* total_ms, int64_t* launches, double* bytes);
/* The decode GEMMs (M <= 256) timed while mux_unit_attn_timing is on: event
 * pairs around every launch, bytes = the weights each streams (N*K*2). */
MUX_API int mux_unit_gemm_time(mux_unit* unit, double* total_ms, int64_t* launches, double* bytes);
/* Tensor-parallel mailbox of a partition (the fused row-parallel GEMM ->
 * allreduce): its device pointer and a CUDA IPC handle (64 bytes) that the
 * other ranks of the mesh open with mux_unit_tp_connect. Replaces the
 * reference's tp_speedup = eta * tp pricing (cost_model.cpp:43-47). */
MUX_API int mux_unit_tp_mailbox(mux_unit* unit, int partition, void** dev_ptr, void* ipc_handle);
/* Map rank peer_rank's mailbox: from its IPC handle (other process), or its
 * device pointer when the peer lives in this process (handle = NULL). */
MUX_API int mux_unit_tp_connect(mux_unit* unit, int partition, int peer_rank, const void* ipc_handle,
                                void* dev_ptr);
/* Debug: the partition's two mailbox counters and their expected values
 * (out[4] = counter0, counter1, expected0, expected1), read on a side stream. */
MUX_API int mux_unit_tp_debug(mux_unit* unit, int partition, uint32_t* out);
/* SMs of a partition (its green context's, or the device's). */
/* SM routing (option "sm_route"): every ADBS job runs on a green context
 * whose SMs are sized by its JobPlan.sm_demand (scheduler.cpp:50-54, :95;
 * priced by sim_engine.cpp:16-18, 308-330). One record per routed job of the
 * last engine run: the scheduling pass, the SM run [first_unit, +units) of
 * the device's green-context units, its SM count and the workspace used
 * (first_unit -1: no free SMs were left, the job shared the whole device). */
typedef struct {
  int64_t pass, job;
  int llm, kind;               /* kind: 0 prefill, 1 decode */
  double sm_demand;
  int first_unit, units, sms, workspace;
  uint64_t busy_units;         /* bit k: unit k held by another in-flight job */
} mux_route_record;
MUX_API int mux_unit_route_log(mux_unit* unit, mux_route_record* out, int64_t cap, int64_t* n_out);
/* The device's green-context units (8-SM granules, remainder last). */
MUX_API int mux_unit_route_units(mux_unit* unit, int* n_units, int* unit_sms, int cap);
/* %smid of `blocks` CTAs launched on the green context of one SM run. */
MUX_API int mux_unit_probe_route(mux_unit* unit, int first_unit, int units, int blocks, int* out);
MUX_API int mux_unit_partition_sms(mux_unit* unit, int partition, int* sms);
/* Debug: launch `blocks` CTAs on a partition and record each CTA's %smid
 * into out (host, [blocks]); synchronises. Proves partition disjointness. */
MUX_API int mux_unit_probe_smids(mux_unit* unit, int partition, int blocks, int* out);
/* Kernel launches issued by this unit so far (all libmux kernels). */
MUX_API int64_t mux_unit_launches(mux_unit* unit);
/* Tuning knobs: "gemm_min_iters" (k-blocks per GEMM CTA floor, default 8);
 * "pdl" (programmatic dependent launch between job kernels, default 1);
 * "graphs" (decode jobs replayed from cached CUDA graphs, default 1);
 * "debug_skip" (measurement: decode jobs skip kernel classes, bitmask 1 K2,
 * 2 RMSNorm, 4 K1; outputs are garbage; bench.py times the GEMM stream so);
 * "prefill_on_partition" (prefill jobs on their model's partition);
 * "pass_green" (partitions = [whole GPU | a whole-GPU stream per model |
 * a green partition per model]; decode jobs use the green partitions only in
 * passes holding decode jobs of two or more models);
 * "align_decode" (real-time runs: a decode job is held off the device until
 * the other models' decode jobs already running have been retired, so the
 * colocated models' steps start together and run in rounds). */
MUX_API int mux_unit_set_option(mux_unit* unit, const char* key, int64_t value);
/* Scheduling passes of the last lockstep / measured run, and how many of
 * them put their decode jobs on green partitions (option "pass_green":
 * decode jobs of two or more models in one pass). Replaces nothing in the
 * reference: its launch (sim_engine.cpp:308-330) prices sm_demand shares. */
MUX_API int mux_unit_pass_stats(mux_unit* unit, int64_t* passes, int64_t* green_passes);

/* Lockstep run: the engine's decisions are those of mux_simulate (oracle
 * timing), and every launched job executes on the unit's GPU. Synthetic
 * prompt tokens come from (seed, request id). tokens_out (nullable) receives
 * all generated tokens, request-major in trace order; each request writes
 * output_len tokens. Single-unit placements only; entries[i] must describe
 * the unit's model i (rates and mean lengths seed the ADBS quotas). */
MUX_API int mux_unit_run_lockstep(mux_unit* unit, const mux_sim_config* cfg, int n_entries,
                          const mux_llm_entry* entries, int n_requests, const mux_request* trace,
                          uint64_t prompt_seed, mux_record* records_out, int32_t* tokens_out);

/* Measured run: the same engine and ADBS decisions process,
 * but every job's completion time is its measured device time (CUDA events
 * from the start of its scheduling pass, the pass's jobs running concurrently
 * on their partitions) instead of the pricing model's. Records then carry
 * real TTFT / latency; throughput = tokens / last done time. */
/* Pool statistics (poolstats.json) of the unit's last lockstep / measured
 * run; release with mux_sim_stats_destroy. */
MUX_API int mux_unit_last_stats(mux_unit* unit, mux_sim_stats** out);
MUX_API int mux_unit_run_measured(mux_unit* unit, const mux_sim_config* cfg, int n_entries,
                                  const mux_llm_entry* entries, int n_requests, const mux_request* trace,
                                  uint64_t prompt_seed, mux_record* records_out, int32_t* tokens_out);
/* Real-time run ("CUDA-event-driven completions, measured
 * interference instead of kappa"): jobs are launched asynchronously and
 * overlap on the device across scheduling passes, as in the deployed system;
 * the engine's clock is the device's (CUDA events from one origin), each
 * completion is processed when its event fires, and idle gaps before the
 * next arrival are skipped rather than waited out. Replaces the priced
 * completion of UnitSim::launch (sim_engine.cpp:308-330). Same arguments and
 * outputs as mux_unit_run_measured. */
MUX_API int mux_unit_run_realtime(mux_unit* unit, const mux_sim_config* cfg, int n_entries,
                                  const mux_llm_entry* entries, int n_requests, const mux_request* trace,
                                  uint64_t prompt_seed, mux_record* records_out, int32_t* tokens_out);

#ifdef __cplusplus
}
#endif

#endif /* MUX_H_ */
