// Per-unit serving engine: event loop, ADBS passes, quota ticks, job launch.
//
// Drop-in for /root/reference/proj/include/muxsim/sim_engine.hpp:15-83 (same
// types and run_simulation signature). The reference engine only *prices* a
// job (sim_engine.cpp:308-330); here launch() also hands every JobPlan to a
// JobExecutor, which runs it on the GPU (csrc/device/executor.cu):
//
//  * lockstep mode  -- completion times come from the pricing model, so every
//    scheduling/allocation decision is bit-identical to the reference oracle,
//    while the executor runs the real kernels for each job (tokens are real);
//  * priced mode    -- no executor: exactly the reference simulator.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mux/adbs.hpp"
#include "mux/kv.hpp"
#include "mux/spec.hpp"
#include "mux/topology.hpp"

namespace muxsim {

struct EngineParams {
  SchedKind scheduler = SchedKind::Adbs;
  double kappa = 0.1;
  double quota_period_s = 10.0;
  std::int64_t token_budget = 4096;
  int block_tokens = 16;
  double warmup_s = 0.0;
  double decode_sm = 0.5;
  double prefill_min_sm = 0.3;
  double activation_reserve_frac = 0.1;
  double quota_floor_frac = 0.02;
  QuotaAdaptParams adapt;
  double eps = 1e-9;
};

struct RequestRecord {
  std::int64_t id = -1;
  std::string llm;
  double arrival_s = 0.0;
  double first_token_s = 0.0;
  double done_s = 0.0;
  int prompt_len = 1;
  int output_len = 1;
};

struct PoolSample {
  double t_s = 0.0;
  std::string llm;
  std::int64_t used_blocks = 0;
  std::int64_t quota_blocks = 0;
};

struct UnitLlmStats {
  std::string llm;
  double rate = 0.0;
  double avg_used_blocks = 0.0;
  std::int64_t final_quota_blocks = 0;
  double resource_usage = 0.0;
};

struct UnitStats {
  int unit = 0;
  std::int64_t total_blocks = 0;
  std::vector<UnitLlmStats> llms;
  std::vector<PoolSample> samples;
};

struct SimResult {
  std::vector<RequestRecord> records;
  std::vector<UnitStats> units;
};

double interference_adjust(double total_running_sm, double own_sm, double kappa);

// ---- B200 extension: where a launched job actually runs ------------------

struct JobLaunch {
  int unit = 0;
  std::int64_t job_id = 0;
  int llm = -1;  // unit-local model index
  JobKind kind = JobKind::Prefill;
  const std::vector<int>* members = nullptr;  // unit-local request indices
  double sm_demand = 0.0;
  double now_ms = 0.0;
  const UnitState* state = nullptr;  // requests: prompt_len / steps_done / global_id
  BlockPool* pool = nullptr;         // physical block tables of the members
};

class JobExecutor {
 public:
  virtual ~JobExecutor() = default;
  // Physical head-block ids are needed by any executor that touches KV.
  virtual bool wants_physical() const { return true; }
  // Tensor-parallel ranks the physical ids are sharded over (head-wise,
  // BlockPool::enable_physical); 1 = one device pool for the whole unit.
  virtual int physical_shards() const { return 1; }
  virtual void attach_unit(int unit, const std::vector<const LLMSpec*>& specs, BlockPool& pool) = 0;
  // After one scheduling pass, before its launches: upload new block-table rows.
  virtual void begin_pass(int unit, BlockPool& pool) = 0;
  // The pass's plans, before begin_pass: lets an executor place the jobs as a
  // set (e.g. SM partitions only when several models' decode jobs share it).
  virtual void plan_pass(int unit, const std::vector<JobPlan>& plans) { (void)unit; (void)plans; }
  virtual void launch(const JobLaunch& job) = 0;
  // The engine is about to retire job_id (free its requests' blocks): the
  // executor must make sure the job's device work has finished.
  virtual void retire(int unit, std::int64_t job_id) = 0;
  virtual void detach_unit(int unit) = 0;
  // Measured mode: job durations come from the device instead
  // of the pricing model. After all launches of a scheduling pass the engine
  // asks for each job's measured milliseconds (the executor waits for it).
  virtual bool measured() const { return false; }
  virtual double measure(int unit, std::int64_t job_id) { (void)unit; (void)job_id; return 0.0; }
  // Real-time mode ("CUDA-event-driven completions"): jobs of
  // different passes overlap on the device as they do in the deployed
  // system, and the engine's clock is the device's. After launching, the
  // engine polls: poll_done returns the in-flight job that completed first
  // if it did so by `until_ms` (its device completion time in *t_ms), else
  // false once the clock reaches until_ms. With nothing in flight the engine
  // fast-forwards the clock to its next event (advance_to): idle time is not
  // waited out. Contention between concurrent jobs is measured, not priced.
  virtual bool realtime() const { return false; }
  virtual bool poll_done(int unit, double until_ms, std::int64_t* job_id, double* t_ms) {
    (void)unit; (void)until_ms; (void)job_id; (void)t_ms;
    return false;
  }
  virtual void advance_to(int unit, double t_ms) { (void)unit; (void)t_ms; }
};

SimResult run_simulation(const Cluster& cluster, const PlacementResult& placement,
                         const std::vector<LlmEntry>& entries, const std::vector<Request>& trace,
                         const LatencyProfile& prof, const EngineParams& params);

// Same run, with every job executed by `exec` (lockstep mode). exec may be null.
SimResult run_simulation(const Cluster& cluster, const PlacementResult& placement,
                         const std::vector<LlmEntry>& entries, const std::vector<Request>& trace,
                         const LatencyProfile& prof, const EngineParams& params,
                         JobExecutor* exec);

}  // namespace muxsim
