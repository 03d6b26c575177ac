// Unified head-wise KV block pool: count semantics + physical head-block ids.
//
// Drop-in for /root/reference/proj/include/muxsim/kv_manager.hpp:13-135. The
// count-level behaviour (admission-time worst-case reservation, quota gate
// before pool gate, atomic row-delta growth, free-all-at-finish) is identical
// to the reference BlockPool, which only counts blocks
// (kv_manager.hpp:88-104). On top of it this pool can hand out *physical*
// 4 KiB head-block ids (the B200 KV cache): every new 16-token row of a
// request pops 2*L*H ids from one LIFO free stack, in (layer, head, K/V)
// order, so any allocation the count oracle accepts also succeeds physically
// (no contiguity requirement). Per-request state lives in dense arrays keyed
// by the unit-local request index rather than std::map (the reference spends
// 77% of its hot loop in map lookups inside alloc).
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

#include "mux/spec.hpp"

namespace muxsim {

struct MemoryLayout {
  std::int64_t weights_bytes = 0;
  std::int64_t activation_reserve_bytes = 0;
  std::int64_t kv_bytes = 0;

  static MemoryLayout for_mesh(std::int64_t mesh_bytes, std::int64_t weights_bytes,
                               double activation_reserve_frac);
};

double blocks_per_token(const LLMSpec& spec, int block_tokens);
std::int64_t blocks_for_tokens(const LLMSpec& spec, int block_tokens, std::int64_t tokens);
std::int64_t block_bytes(const LLMSpec& spec, int block_tokens);

enum class AllocError { None, Pool, Quota };

struct AllocResult {
  bool ok = false;
  AllocError error = AllocError::None;
};

// One physical row handed out by the pool: request `slot` got row-record
// `rowrec` as its row number `row`; the record's 2*L*H block ids are in
// BlockPool::row_ids(llm, rowrec). Consumed by the device-table uploader.
struct RowDelta {
  int slot = -1;
  int row = -1;
  int rowrec = -1;
};

class BlockPool {
 public:
  explicit BlockPool(std::int64_t total_blocks);

  void register_llm(int llm, const LLMSpec* spec, int block_tokens);
  int num_llms() const { return static_cast<int>(llms_.size()); }

  AllocResult admit(int llm, std::int64_t request_id, std::int64_t prompt_tokens,
                    std::int64_t total_tokens);
  AllocResult alloc(int llm, std::int64_t request_id, std::int64_t add_tokens, bool enforce_quota);
  void free_request(int llm, std::int64_t request_id);

  void set_quota(int llm, std::int64_t blocks);
  std::int64_t quota(int llm) const;
  std::int64_t used(int llm) const;
  std::int64_t committed(int llm) const;
  std::int64_t request_tokens(int llm, std::int64_t request_id) const;
  std::int64_t total_used() const;
  std::int64_t committed_total() const { return committed_total_; }
  std::int64_t free_blocks() const { return free_blocks_; }
  std::int64_t total_blocks() const { return total_blocks_; }

  void check_conservation() const;

  // ---- physical layer (B200 extension) ---------------------------------
  // Turn on physical id assignment. Must be called before any allocation.
  // Ids are int32 in [0, total_blocks). Every registered model gets a slot
  // space (one device block-table row list per live request).
  // shards > 1 (a tensor-parallel mesh): the pool is head-sharded
  // over `shards` ranks, each holding floor(total / shards) blocks of its own
  // device memory. A row's column (layer, head, kv) takes a rank-local id
  // from the free stack of rank head / (H / shards); every row costs
  // 2*L*H / shards blocks per rank, so the mesh-wide count check (the
  // reference's decisions, unchanged) implies every rank's stack has room.
  void enable_physical(int shards = 1);
  int shards() const { return shards_; }
  bool physical() const { return physical_; }
  int rows_of(int llm, std::int64_t request_id) const;
  int slot_of(int llm, std::int64_t request_id) const;
  // Row-record indices of a request, in row order.
  const std::vector<std::int32_t>& row_records(int llm, std::int64_t request_id) const;
  // The 2*L*H physical ids of one row record: index (layer*H + head)*2 + kv.
  const std::int32_t* row_ids(int llm, int rowrec) const;
  int row_width(int llm) const;           // 2*L*H
  int rowrec_capacity(int llm) const;     // row records ever materialised
  int slot_capacity(int llm) const;       // slots ever materialised
  int max_rows_seen(int llm) const;
  // Row deltas since the last drain, in allocation order.
  std::vector<RowDelta>& pending_rows(int llm);
  // Physical block table of one request, [rows][layer][head][kv] flattened.
  std::vector<std::int32_t> block_table(int llm, std::int64_t request_id) const;
  std::int64_t physical_free() const;
  // Shard (tensor-parallel rank) of column j of a row of `llm`.
  int shard_of_column(int llm, int j) const;

 private:
  struct Req {
    std::int64_t tokens = 0;
    std::int64_t reserve = -1;  // -1: admitted without a reservation
    int slot = -1;
    std::vector<std::int32_t> rows;  // row records, physical mode only
  };

  struct Model {
    const LLMSpec* spec = nullptr;
    int block_tokens = 16;
    std::int64_t row_blocks = 0;  // 2 * L * H
    std::int64_t quota = 0;
    std::int64_t used = 0;
    std::int64_t committed = 0;
    // Request table: dense for small non-negative ids, hashed otherwise.
    std::vector<std::int32_t> dense;  // id -> index into reqs, -1 = absent
    std::unordered_map<std::int64_t, std::int32_t> sparse;
    std::vector<Req> reqs;
    std::vector<std::int32_t> free_req;
    std::int64_t live = 0;
    // physical
    std::vector<std::int32_t> rowrec_ids;  // [rowrec][row_blocks]
    std::vector<std::int32_t> free_rowrec;
    std::vector<std::int32_t> free_slot;
    int next_slot = 0;
    int max_rows = 0;
    std::vector<RowDelta> pending;
  };

  static constexpr std::int64_t kDenseLimit = std::int64_t(1) << 22;

  Model& model(int llm);
  const Model& model(int llm) const;
  std::int32_t find(const Model& m, std::int64_t id) const;
  std::int32_t find_or_add(Model& m, std::int64_t id);
  void erase(Model& m, std::int64_t id, std::int32_t idx);
  std::int64_t rows_for(const Model& m, std::int64_t tokens) const {
    return (tokens + m.block_tokens - 1) / m.block_tokens;
  }
  void grow_physical(Model& m, Req& r, std::int64_t new_rows);
  void release_physical(Model& m, Req& r);

  std::int64_t total_blocks_ = 0;
  std::int64_t free_blocks_ = 0;
  std::int64_t committed_total_ = 0;
  std::vector<Model> llms_;
  bool physical_ = false;
  int shards_ = 1;
  std::vector<std::vector<std::int32_t>> free_ids_;  // per shard, LIFO; back() is the next id handed out
};

struct QuotaInput {
  double rate = 0.0;
  double blocks_per_token = 0.0;
  double mean_request_tokens = 0.0;
};

std::vector<std::int64_t> init_token_block_quota(const std::vector<QuotaInput>& llms,
                                                 std::int64_t kv_blocks,
                                                 double floor_frac = 0.02);

struct QuotaAdaptParams {
  double low_mark = 0.5;
  double high_mark = 0.9;
  double step_frac = 0.1;
};

std::vector<std::int64_t> adapt_quota(const std::vector<double>& utilizations,
                                      const std::vector<std::int64_t>& quotas,
                                      std::int64_t floor_blocks,
                                      const QuotaAdaptParams& params = {});

}  // namespace muxsim
