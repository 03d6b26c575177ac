// C ABI (include/mux.h): exception -> status mapping, handles, and the
// lockstep JobExecutor that runs the engine's JobPlans on the GPU.
#include "../../include/mux.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "device/runtime.h"
#include "kernels/kernels.h"
#include "kernels/launch.cuh"
#include "mux/planner.hpp"
#include "mux/engine.hpp"
#include "mux/kv.hpp"

using muxsim::BlockPool;

namespace {
void check_cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS)
    throw std::runtime_error(std::string("cuda driver error in ") + what + ": CUresult " + std::to_string(r));
}

// Driver entry points, resolved through the runtime so libmux.so loads on a
// host without libcuda (the CPU test suite only needs the control plane).
template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    throw std::runtime_error(std::string("driver entry point unavailable: ") + name);
  return reinterpret_cast<F>(p);
}
struct GreenApi {
  decltype(&cuDeviceGet) device_get = driver_fn<decltype(&cuDeviceGet)>("cuDeviceGet");
  decltype(&cuDeviceGetDevResource) get_resource = driver_fn<decltype(&cuDeviceGetDevResource)>("cuDeviceGetDevResource");
  decltype(&cuDevSmResourceSplitByCount) split =
      driver_fn<decltype(&cuDevSmResourceSplitByCount)>("cuDevSmResourceSplitByCount");
  decltype(&cuDevResourceGenerateDesc) gen_desc = driver_fn<decltype(&cuDevResourceGenerateDesc)>("cuDevResourceGenerateDesc");
  decltype(&cuGreenCtxCreate) create = driver_fn<decltype(&cuGreenCtxCreate)>("cuGreenCtxCreate");
  decltype(&cuGreenCtxStreamCreate) stream_create = driver_fn<decltype(&cuGreenCtxStreamCreate)>("cuGreenCtxStreamCreate");
  decltype(&cuGreenCtxDestroy) destroy = driver_fn<decltype(&cuGreenCtxDestroy)>("cuGreenCtxDestroy");
};
GreenApi& green_api() {
  static GreenApi* api = new GreenApi();
  return *api;
}

// Each CTA records the SM it ran on (and lingers so the grid spreads out).
__global__ void probe_smid_kernel(int* out) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const long long t0 = clock64();
  while (clock64() - t0 < 200000) {
  }
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(smid);
}
}  // namespace

struct mux_pool {
  BlockPool* bp = nullptr;
  std::unique_ptr<BlockPool> owned;
  std::deque<muxsim::LLMSpec> specs;  // stable addresses for register_llm
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MUX_OK;
  } catch (const muxsim::InfeasibleError& e) {
    g_err = e.what();
    return MUX_EINFEAS;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MUX_EINVAL;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return MUX_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MUX_EINTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return MUX_EINTERNAL;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

int alloc_code(const muxsim::AllocResult& r) {
  if (r.ok) return MUX_ALLOC_OK;
  return r.error == muxsim::AllocError::Quota ? MUX_ALLOC_QUOTA : MUX_ALLOC_POOL;
}

muxsim::LLMSpec spec_of(const mux_llm_entry& e) {
  muxsim::LLMSpec s;
  s.name = e.name ? e.name : "";
  s.num_layers = e.num_layers;
  s.num_heads = e.num_heads;
  s.head_dim = e.head_dim;
  s.hidden_size = e.hidden_size;
  s.weight_bytes = e.weight_bytes;
  s.bytes_per_element = e.bytes_per_element;
  return s;
}

struct SimInputs {
  muxsim::Cluster cluster;
  muxsim::PlacementResult placement;
  std::vector<muxsim::LlmEntry> entries;
  std::vector<muxsim::Request> trace;
  muxsim::LatencyProfile prof;
  muxsim::EngineParams params;
};

// LatencyProfile from the ABI's optional blocks: the reference's 7 fields
// (cost_model.hpp:33-40), the HBM decode form and the measured TP allreduce
// terms (B200 extensions; NULL = the reference's defaults / forms).
muxsim::LatencyProfile profile_of(const double* p, const double* decode_hbm, const double* tp_allreduce) {
  muxsim::LatencyProfile prof;
  if (p) {
    prof.prefill_ms_per_token = p[0];
    prof.decode_base_ms = p[1];
    prof.decode_ctx_ms_per_token = p[2];
    prof.tp_efficiency = p[3];
    prof.sm_saturation_point = p[4];
    prof.batch_knee = p[5];
    prof.reference_scale = p[6];
  }
  if (decode_hbm) {
    prof.decode_form = 1;
    prof.decode_fixed_ms = decode_hbm[0];
    prof.decode_row_ms = decode_hbm[1];
    prof.decode_bctx_ms = decode_hbm[2];
    prof.decode_sm_exponent = decode_hbm[3];
  }
  if (tp_allreduce) {
    prof.allreduce_alpha_ms = tp_allreduce[0];
    prof.allreduce_ms_per_mib = tp_allreduce[1];
  }
  return prof;
}

SimInputs build_inputs(const mux_sim_config* c, int n_entries, const mux_llm_entry* entries, int n_req,
                       const mux_request* trace) {
  require(c != nullptr && entries != nullptr && (n_req == 0 || trace != nullptr), "null argument");
  SimInputs in;
  in.cluster.num_nodes = c->num_nodes;
  in.cluster.gpus_per_node = c->gpus_per_node;
  in.cluster.gpu_memory_bytes = c->gpu_memory_bytes;
  for (int i = 0; i < n_entries; ++i) {
    muxsim::LlmEntry e;
    e.spec = spec_of(entries[i]);
    e.rate = entries[i].rate;
    e.mean_prompt_tokens = entries[i].mean_prompt_tokens;
    e.mean_output_tokens = entries[i].mean_output_tokens;
    in.entries.push_back(e);
  }
  in.placement.backend = "greedy";
  int gpu = 0;
  for (int u = 0; u < c->n_units; ++u) {
    muxsim::LLMUnit lu;
    lu.mesh.node = 0;
    for (int g = 0; g < c->unit_mesh_size[u]; ++g) lu.mesh.gpu_ids.push_back(gpu++);
    in.placement.units.push_back(lu);
  }
  for (int i = 0; i < c->n_placed; ++i) {
    const mux_placed_llm& p = c->placed[i];
    require(p.unit >= 0 && p.unit < c->n_units && p.llm >= 0 && p.llm < n_entries, "bad placement");
    muxsim::PlacedLlm pl;
    pl.llm = p.llm;
    pl.candidate.tp_degree = p.tp_degree;
    pl.candidate.num_sm = p.num_sm;
    in.placement.units[p.unit].llms.push_back(pl);
  }
  for (int i = 0; i < n_req; ++i) {
    require(trace[i].llm >= 0 && trace[i].llm < n_entries, "trace llm out of range");
    muxsim::Request r;
    r.id = trace[i].id;
    r.llm = in.entries[trace[i].llm].spec.name;
    r.arrival_s = trace[i].arrival_s;
    r.prompt_len = trace[i].prompt_len;
    r.output_len = trace[i].output_len;
    in.trace.push_back(r);
  }
  in.prof = profile_of(c->profile, c->decode_hbm, c->tp_allreduce);
  in.params.scheduler = static_cast<muxsim::SchedKind>(c->scheduler);
  in.params.kappa = c->kappa;
  in.params.quota_period_s = c->quota_period_s;
  in.params.token_budget = c->token_budget;
  in.params.block_tokens = c->block_tokens;
  in.params.warmup_s = c->warmup_s;
  in.params.decode_sm = c->decode_sm;
  in.params.prefill_min_sm = c->prefill_min_sm;
  in.params.activation_reserve_frac = c->activation_reserve_frac;
  in.params.quota_floor_frac = c->quota_floor_frac;
  if (c->quota_adapt) {
    in.params.adapt.low_mark = c->quota_adapt[0];
    in.params.adapt.high_mark = c->quota_adapt[1];
    in.params.adapt.step_frac = c->quota_adapt[2];
  }
  return in;
}

void export_records(const muxsim::SimResult& res, const SimInputs& in, mux_record* out) {
  if (out == nullptr) return;
  std::unordered_map<std::string, int> idx;
  for (size_t i = 0; i < in.entries.size(); ++i) idx[in.entries[i].spec.name] = static_cast<int>(i);
  for (size_t i = 0; i < res.records.size(); ++i) {
    const muxsim::RequestRecord& r = res.records[i];
    out[i] = {r.id, idx[r.llm], r.arrival_s, r.first_token_s, r.done_s, r.prompt_len, r.output_len};
  }
}

uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace

// SM routing of ADBS jobs (option sm_route): every job runs on a green
// context whose SM set is sized by its JobPlan.sm_demand (scheduler.cpp:50-54
// prefill, :95 decode) -- the spatial share the reference prices with
// sm_scaling_* and interference_adjust (sim_engine.cpp:16-18, 308-330). The
// device's SMs are split once into green-context granules (8-SM groups; the
// remainder outside them is the last unit); a job takes the first free
// contiguous run of units whose SM count reaches round(sm_demand x SMs), or
// the largest free run when rounding leaves less. ADBS keeps the demands of
// concurrent jobs <= 1, so concurrent jobs land on disjoint SM sets. The green
// context of each (first unit, units) run is created on first use and cached.
struct SmRouter {
  struct Part {
    CUgreenCtx g = nullptr;
    cudaStream_t s = nullptr;
    int sms = 0;
  };
  bool ready = false;
  int device = 0;
  int total_sms = 0;
  std::vector<CUdevResource> units;
  std::vector<int> unit_sms;
  std::vector<int64_t> owner;  // job holding each unit, -1 = free
  std::map<std::pair<int, int>, Part> parts;

  void init(int dev) {
    if (ready) return;
    GreenApi& ga = green_api();
    device = dev;
    CUdevice d = 0;
    check_cu(ga.device_get(&d, dev), "cuDeviceGet");
    CUdevResource all{};
    check_cu(ga.get_resource(d, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
    unsigned int nb = 0;
    check_cu(ga.split(nullptr, &nb, &all, nullptr, 0, 8), "cuDevSmResourceSplitByCount(query)");
    units.resize(nb);
    CUdevResource rem{};
    check_cu(ga.split(units.data(), &nb, &all, &rem, 0, 8), "cuDevSmResourceSplitByCount");
    units.resize(nb);
    if (rem.sm.smCount > 0) units.push_back(rem);
    total_sms = 0;
    for (const CUdevResource& r : units) {
      unit_sms.push_back(static_cast<int>(r.sm.smCount));
      total_sms += static_cast<int>(r.sm.smCount);
    }
    owner.assign(units.size(), -1);
    ready = true;
  }
  // (first unit, units) for a demand; (-1, 0) when every unit is taken.
  std::pair<int, int> pick(double demand) const {
    const int want = std::max(1, static_cast<int>(std::lround(demand * total_sms)));
    const int n = static_cast<int>(units.size());
    int best_start = -1, best_len = 0, best_sms = 0;
    for (int i = 0; i < n; ++i) {
      if (owner[i] >= 0) continue;
      int sms = 0, j = i;
      while (j < n && owner[j] < 0 && sms < want) sms += unit_sms[j++];
      if (sms >= want) return {i, j - i};
      if (sms > best_sms) best_start = i, best_len = j - i, best_sms = sms;
      i = j - 1;
    }
    return {best_start, best_len};
  }
  Part& part(int start, int len) {
    auto key = std::make_pair(start, len);
    auto it = parts.find(key);
    if (it != parts.end()) return it->second;
    GreenApi& ga = green_api();
    Part p;
    CUdevResourceDesc desc;
    std::vector<CUdevResource> rs(units.begin() + start, units.begin() + start + len);
    check_cu(ga.gen_desc(&desc, rs.data(), static_cast<unsigned>(rs.size())), "cuDevResourceGenerateDesc");
    CUdevice d = 0;
    check_cu(ga.device_get(&d, device), "cuDeviceGet");
    check_cu(ga.create(&p.g, desc, d, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
    CUstream cs;
    check_cu(ga.stream_create(&cs, p.g, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
    p.s = reinterpret_cast<cudaStream_t>(cs);
    for (int k = start; k < start + len; ++k) p.sms += unit_sms[k];
    return parts.emplace(key, p).first->second;
  }
  void take(int start, int len, int64_t job) {
    for (int k = start; k < start + len; ++k) owner[k] = job;
  }
  void release(int64_t job) {
    for (int64_t& o : owner)
      if (o == job) o = -1;
  }
  ~SmRouter() {
    for (auto& kv : parts) {
      if (kv.second.s) cudaStreamDestroy(kv.second.s);
      if (kv.second.g) green_api().destroy(kv.second.g);
    }
  }
};

// One routed job, for mux_unit_route_log (tests, serving analysis).
struct RouteRecord {
  int64_t pass, job;
  int llm, kind;  // kind: 0 prefill, 1 decode
  double sm_demand;
  int first_unit, units, sms, workspace;
  uint64_t busy_units;  // units held by other in-flight jobs at this launch
};

// Pool statistics of a run (SimResult.units) behind poolstats.json.
struct mux_sim_stats {
  std::vector<muxsim::UnitStats> units;
  std::unordered_map<std::string, int> idx;  // model name -> entry index
};

// -------------------------------------------------------------------- unit

struct mux_unit {
  std::unique_ptr<mux_sim_stats> last_stats;  // of the last lockstep / measured run
  bool prefill_on_partition = false;          // option: prefill jobs on their model's partition
  // option pass_green: partitions are [whole GPU | one whole-GPU stream per
  // model | one green partition per model]; a pass's decode jobs take the
  // green partitions only when decode jobs of two or more models share it.
  bool pass_green = false;
  bool align_decode = false;  // option align_decode (real-time mode): colocated decode steps in rounds
  bool sm_route = false;      // option sm_route: every job on an SM run sized by its sm_demand
  SmRouter router;
  std::vector<int64_t> ws_owner;   // sm_route: job holding each workspace (-1 free)
  std::vector<RouteRecord> route_log;
  int64_t passes = 0, green_passes = 0;  // of the last lockstep / measured run
  std::unique_ptr<mux::Runtime> rt;
  std::deque<muxsim::LLMSpec> specs;
  std::vector<std::unique_ptr<mux::Llama>> models;
  mux_pool pool;
  std::vector<cudaStream_t> streams;
  std::vector<CUgreenCtx> green;  // one per SM-partitioned stream (nullptr = whole device)
  std::vector<int> sms;           // SMs each partition may use
  std::vector<std::unique_ptr<mux::Workspace>> ws;
  cudaEvent_t ev[64] = {};
  bool timing = false;
  mux::AttnTimer timer;
  mux::AttnTimer gemm_timer;  // decode GEMM launches while timing is on
  int max_batch = 0;
  int max_prefill = 0;
  ~mux_unit() {
    if (rt) cudaDeviceSynchronize();
    ws.clear();
    for (cudaStream_t s : streams) cudaStreamDestroy(s);
    for (CUgreenCtx g : green)
      if (g) green_api().destroy(g);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
  cudaStream_t stream(int p) {
    if (p < 0 || p >= static_cast<int>(streams.size())) throw std::invalid_argument("bad partition");
    return streams[p];
  }
  mux::Llama& model(int llm) {
    if (llm < 0 || llm >= static_cast<int>(models.size())) throw std::invalid_argument("bad llm index");
    return *models[llm];
  }
};

namespace {

// Lockstep executor: JobPlans decided by the engine (oracle timing) run on
// the unit's GPU; completion is consumed only after the device finished.
class GpuExecutor : public muxsim::JobExecutor {
 public:
  GpuExecutor(mux_unit* u, uint64_t prompt_seed, const std::vector<muxsim::Request>& trace, bool measured = false,
              bool realtime = false)
      : u_(u), seed_(prompt_seed), measured_(measured || realtime), realtime_(realtime) {
    for (size_t i = 0; i < trace.size(); ++i) row_of_id_[trace[i].id] = static_cast<int>(i);
    tokens_.resize(trace.size());
    check(cudaEventCreateWithFlags(&tables_ready_, cudaEventDisableTiming));
    check(cudaEventCreate(&pass_start_));
    check(cudaEventCreate(&t0_ev_));
  }
  ~GpuExecutor() override {
    for (auto& kv : jobs_) cudaEventDestroy(kv.second.done);
    cudaEventDestroy(tables_ready_);
    cudaEventDestroy(pass_start_);
    cudaEventDestroy(t0_ev_);
    if (upload_) {
      cudaStreamSynchronize(upload_);
      cudaStreamDestroy(upload_);
    }
  }

  bool measured() const override { return measured_ && !realtime_; }
  int physical_shards() const override { return u_->models.empty() ? 1 : u_->models[0]->dims().tp_size; }
  bool realtime() const override { return realtime_; }

  // Real-time clock: host steady clock since the run started plus the idle
  // time skipped by advance_to; job completions are device-event times on
  // the same origin (t0 recorded with the device idle).
  double clock_ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_host_).count() +
           skipped_ms_;
  }

  void advance_to(int, double t_ms) override {
    const double c = clock_ms();
    if (t_ms > c) skipped_ms_ += t_ms - c;
  }

  bool poll_done(int, double until_ms, std::int64_t* job_id, double* t_ms) override {
    release_held();
    for (;;) {
      // the earliest completed in-flight job (device time)
      std::int64_t best = -1;
      double best_t = 0.0;
      for (std::int64_t id : inflight_) {
        if (jobs_.at(id).held) continue;
        cudaError_t q = cudaEventQuery(jobs_.at(id).done);
        if (q == cudaErrorNotReady) continue;
        check(q);
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, t0_ev_, jobs_.at(id).done));
        const double t = static_cast<double>(ms) + jobs_.at(id).skipped_ms;
        if (best < 0 || t < best_t) best = id, best_t = t;
      }
      if (best >= 0 && best_t <= until_ms) {
        inflight_.erase(std::find(inflight_.begin(), inflight_.end(), best));
        *job_id = best;
        *t_ms = best_t;
        return true;
      }
      if (clock_ms() >= until_ms) return false;
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }

  // Device time from the start of the pass (its block-table upload included)
  // to the end of this job, waiting for it.
  double measure(int, std::int64_t job_id) override {
    auto it = jobs_.find(job_id);
    if (it == jobs_.end()) throw std::logic_error("measured: unknown job");
    check(cudaEventSynchronize(it->second.done));
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, pass_start_, it->second.done));
    return static_cast<double>(ms);
  }

  void attach_unit(int, const std::vector<const muxsim::LLMSpec*>& specs, BlockPool& pool) override {
    if (specs.size() != u_->models.size()) throw std::invalid_argument("lockstep: model count mismatch");
    for (size_t i = 0; i < specs.size(); ++i) {
      const mux::ModelDims& d = u_->models[i]->dims();
      if (specs[i]->num_layers != d.layers || specs[i]->num_heads != d.heads * d.tp_size)
        throw std::invalid_argument("lockstep: model " + specs[i]->name + " does not match the unit");
    }
    if (pool.total_blocks() > INT32_MAX) throw std::invalid_argument("lockstep: pool too large");
    if (realtime_) {
      // table uploads on their own stream: stream 0 may be running a prefill
      check(cudaStreamCreateWithFlags(&upload_, cudaStreamNonBlocking));
      check(cudaDeviceSynchronize());
      check(cudaEventRecord(t0_ev_, upload_));
      check(cudaEventSynchronize(t0_ev_));
      t0_host_ = std::chrono::steady_clock::now();
    }
  }

  void begin_pass(int, BlockPool& pool) override {
    if (realtime_) {
      for (int i = 0; i < static_cast<int>(u_->models.size()); ++i)
        u_->rt->upload_rows(pool, i, *u_->models[i], upload_);
      check(cudaEventRecord(tables_ready_, upload_));
      for (cudaStream_t s : u_->streams) check(cudaStreamWaitEvent(s, tables_ready_, 0));
      return;
    }
    cudaStream_t s0 = u_->streams[0];
    if (measured_) check(cudaEventRecord(pass_start_, s0));
    for (int i = 0; i < static_cast<int>(u_->models.size()); ++i)
      u_->rt->upload_rows(pool, i, *u_->models[i], s0);
    check(cudaEventRecord(tables_ready_, s0));
    for (size_t p = 1; p < u_->streams.size(); ++p) check(cudaStreamWaitEvent(u_->streams[p], tables_ready_, 0));
  }

  void plan_pass(int, const std::vector<muxsim::JobPlan>& plans) override {
    std::vector<char> decodes(u_->models.size(), 0);
    int n = 0;
    for (const muxsim::JobPlan& p : plans)
      if (p.kind == muxsim::JobKind::Decode && !decodes[p.llm]) decodes[p.llm] = 1, ++n;
    green_pass_ = n >= 2;
    u_->green_passes += green_pass_ ? 1 : 0;
    ++u_->passes;
  }

  void launch(const muxsim::JobLaunch& j) override {
    const muxsim::UnitState& st = *j.state;
    const int P = static_cast<int>(u_->streams.size());
    // Decode jobs run on their model's partition. Prefill jobs run on the
    // ungreened stream 0 (all SMs) unless prefill_on_partition is set: then
    // every job of a model stays inside its green partition (stream 0's
    // kernels may otherwise occupy the SMs of the other model's partition).
    const bool own = j.kind != muxsim::JobKind::Prefill || u_->prefill_on_partition;
    int part = !own || P == 1 ? 0 : 1 + (j.llm % (P - 1));
    if (u_->pass_green) {
      // Per-pass choice: a decode job alone in its pass gets the whole GPU
      // (a green share would leave the other SMs idle); decode jobs of
      // several models split the SMs by their green partitions. Prefill
      // follows its model's decode placement when prefill_on_partition.
      const int n = static_cast<int>(u_->models.size());
      if (P != 1 + 2 * n) throw std::invalid_argument("pass_green: the unit needs 1 + 2 x models partitions");
      part = !own ? 0 : (green_pass_ ? 1 + n + j.llm : 1 + j.llm);
    }
    cudaStream_t s = u_->streams[part];
    mux::Workspace* wsp = u_->ws[part].get();
    if (u_->sm_route) {
      // the job's own SM run, sized by its sm_demand, and a free workspace
      SmRouter& R = u_->router;
      R.init(u_->rt->device());
      int w = 0;
      while (w < static_cast<int>(u_->ws_owner.size()) && u_->ws_owner[w] >= 0) ++w;
      if (w == static_cast<int>(u_->ws_owner.size()))
        throw std::logic_error("sm_route: more concurrent jobs than workspaces (create the unit with models + 1 partitions)");
      uint64_t busy = 0;
      for (size_t k = 0; k < R.owner.size() && k < 64; ++k)
        if (R.owner[k] >= 0) busy |= 1ull << k;
      const std::pair<int, int> run = R.pick(j.sm_demand);
      int sms = u_->rt->num_sms();
      if (run.first >= 0) {
        SmRouter::Part& pt = R.part(run.first, run.second);
        R.take(run.first, run.second, j.job_id);
        s = pt.s;
        sms = pt.sms;
      } else {
        s = u_->streams[0];  // every unit taken by rounding: share the whole device
      }
      u_->ws_owner[w] = j.job_id;
      wsp = u_->ws[w].get();
      wsp->sms = sms;
      wsp->exclusive = run.first >= 0;
      check(cudaStreamWaitEvent(s, tables_ready_, 0));
      u_->route_log.push_back({u_->passes, j.job_id, j.llm, j.kind == muxsim::JobKind::Prefill ? 0 : 1, j.sm_demand,
                               run.first, run.second, sms, w, busy});
    }
    mux::Llama& m = *u_->models[j.llm];
    mux::Workspace& ws = *wsp;
    const int n = static_cast<int>(j.members->size());
    Job job;
    job.members = *j.members;
    if (realtime_ && trace_) {
      check(cudaEventCreate(&job.start));
      check(cudaEventRecord(job.start, s));  // held jobs re-record at release
    }
    // pinned result buffers are recycled: cudaFreeHost synchronises the
    // device, which would serialise the real-time mode's overlapping jobs
    for (auto it = spare_out_.begin(); it != spare_out_.end(); ++it)
      if ((*it)->bytes >= static_cast<size_t>(n) * 4) {
        job.out = std::move(*it);
        spare_out_.erase(it);
        break;
      }
    if (!job.out) job.out = std::make_unique<mux::PinnedMem>(std::max<size_t>(static_cast<size_t>(n) * 4, 1024));
    std::vector<int32_t> slots(n), aux(n);
    for (int i = 0; i < n; ++i) {
      const int rid = (*j.members)[i];
      slots[i] = j.pool->slot_of(j.llm, rid);
      if (j.kind == muxsim::JobKind::Prefill) {
        aux[i] = st.requests[rid].prompt_len;
      } else {
        aux[i] = static_cast<int32_t>(j.pool->request_tokens(j.llm, rid));
      }
    }
    if (j.kind == muxsim::JobKind::Prefill) {
      std::vector<int32_t> toks;
      for (int i = 0; i < n; ++i) {
        const muxsim::UnitRequest& r = st.requests[(*j.members)[i]];
        for (int p = 0; p < r.prompt_len; ++p)
          toks.push_back(static_cast<int32_t>(mix64(seed_ ^ mix64(static_cast<uint64_t>(r.global_id) * 131071u + p)) %
                                              static_cast<uint64_t>(m.dims().vocab)));
      }
      u_->rt->prefill(m, ws, n, slots.data(), aux.data(), toks.data(), job.out->as<int32_t>(), s);
    } else if (realtime_ && u_->align_decode) {
      // Aligned decode rounds (option align_decode): a decode job waits,
      // unlaunched, for the other models' decode jobs already on the device;
      // it is enqueued once the engine has retired them, i.e. right after
      // their models' next steps were launched, so colocated decode steps
      // start together and share the GPU in rounds, as in bench.py.
      for (int64_t id : inflight_) {
        const Job& o = jobs_.at(id);
        if (!o.held && o.decode && o.llm != j.llm) job.wait_for.push_back(id);
      }
      job.part = part;
      job.slots = slots;
      job.aux = aux;
      job.held = !job.wait_for.empty();
      if (!job.held)
        u_->rt->decode(m, ws, n, slots.data(), aux.data(), nullptr, job.out->as<int32_t>(), s, nullptr);
    } else {
      u_->rt->decode(m, ws, n, slots.data(), aux.data(), nullptr, job.out->as<int32_t>(), s,
                     u_->timing ? &u_->timer : nullptr);
    }
    job.decode = j.kind != muxsim::JobKind::Prefill;
    check(cudaEventCreateWithFlags(&job.done, measured_ ? cudaEventDefault : cudaEventDisableTiming));
    if (!job.held) check(cudaEventRecord(job.done, s));
    job.llm = j.llm;
    if (realtime_) {
      job.skipped_ms = skipped_ms_;  // nothing in flight skips time, so this is fixed for the job
      inflight_.push_back(j.job_id);
    }
    job.global_ids.resize(n);
    for (int i = 0; i < n; ++i) job.global_ids[i] = st.requests[(*j.members)[i]].global_id;
    jobs_.emplace(j.job_id, std::move(job));
  }

  void retire(int, std::int64_t job_id) override {
    auto it = jobs_.find(job_id);
    if (it == jobs_.end()) throw std::logic_error("lockstep: retire of unknown job");
    Job& job = it->second;
    check(cudaEventSynchronize(job.done));
    if (u_->sm_route) {
      u_->router.release(job_id);
      for (int64_t& o : u_->ws_owner)
        if (o == job_id) o = -1;
    }
    const int32_t* out = job.out->as<int32_t>();
    for (size_t i = 0; i < job.global_ids.size(); ++i) {
      auto r = row_of_id_.find(job.global_ids[i]);
      if (r != row_of_id_.end()) tokens_[r->second].push_back(out[i]);
    }
    if (job.start) {
      float a = 0.f, b = 0.f;
      check(cudaEventElapsedTime(&a, t0_ev_, job.start));
      check(cudaEventElapsedTime(&b, t0_ev_, job.done));
      timeline_ << job.llm << ',' << (job.decode ? "decode" : "prefill") << ',' << job.global_ids.size() << ','
                << a + job.skipped_ms << ',' << b + job.skipped_ms << '\n';
      cudaEventDestroy(job.start);
    }
    cudaEventDestroy(job.done);
    spare_out_.push_back(std::move(job.out));
    jobs_.erase(it);
  }

  void detach_unit(int) override {
    check(cudaDeviceSynchronize());
    if (trace_) {
      std::FILE* f = std::fopen(std::getenv("MUX_RT_TIMELINE"), "w");
      if (f) {
        std::fputs("llm,kind,batch,start_ms,end_ms\n", f);
        std::fputs(timeline_.str().c_str(), f);
        std::fclose(f);
      }
    }
  }

  const std::vector<std::vector<int32_t>>& tokens() const { return tokens_; }

 private:
  struct Job {
    int llm = -1;
    std::vector<int> members;
    std::vector<int64_t> global_ids;
    std::unique_ptr<mux::PinnedMem> out;
    cudaEvent_t done = nullptr;
    double skipped_ms = 0.0;  // real-time mode: idle time skipped before the launch
    cudaEvent_t start = nullptr;  // MUX_RT_TIMELINE: when the job's stream reached it
    // align_decode: a held decode job (not yet on the device), the jobs it
    // waits for, and what its enqueue needs
    bool decode = false, held = false;
    int part = 0;
    std::vector<int64_t> wait_for;
    std::vector<int32_t> slots, aux;
  };

  // Enqueue the held decode jobs whose awaited jobs the engine has retired.
  void release_held() {
    for (int64_t id : inflight_) {
      Job& jb = jobs_.at(id);
      if (!jb.held) continue;
      bool ready = true;
      for (int64_t w : jb.wait_for) ready = ready && jobs_.find(w) == jobs_.end();
      if (!ready) continue;
      cudaStream_t s = u_->streams[jb.part];
      if (jb.start) check(cudaEventRecord(jb.start, s));
      u_->rt->decode(*u_->models[jb.llm], *u_->ws[jb.part], static_cast<int>(jb.slots.size()), jb.slots.data(),
                     jb.aux.data(), nullptr, jb.out->as<int32_t>(), s, nullptr);
      check(cudaEventRecord(jb.done, s));
      jb.held = false;
    }
  }
  static void check(cudaError_t e) { mux::check_cuda(e, "lockstep executor"); }
  mux_unit* u_;
  uint64_t seed_;
  bool measured_ = false;
  cudaEvent_t pass_start_ = nullptr;
  std::unordered_map<int64_t, int> row_of_id_;
  std::vector<std::vector<int32_t>> tokens_;
  std::unordered_map<int64_t, Job> jobs_;
  cudaEvent_t tables_ready_ = nullptr;
  bool green_pass_ = false;  // this pass's decode jobs run on green partitions
  // real-time mode
  bool realtime_ = false;
  cudaStream_t upload_ = nullptr;
  cudaEvent_t t0_ev_ = nullptr;
  std::chrono::steady_clock::time_point t0_host_{};
  double skipped_ms_ = 0.0;
  std::vector<int64_t> inflight_;
  std::vector<std::unique_ptr<mux::PinnedMem>> spare_out_;
  // debug: MUX_RT_TIMELINE=<csv> writes every real-time job's device
  // start / end (ms from the run's origin) at detach
  bool trace_ = std::getenv("MUX_RT_TIMELINE") != nullptr;
  std::ostringstream timeline_;
};

}  // namespace

extern "C" {

const char* mux_last_error(void) { return g_err.c_str(); }
const char* mux_version(void) { return "mux-b200 0.1 (sm_100a)"; }

int mux_blocks_for_tokens(int num_layers, int num_heads, int block_tokens, int64_t tokens, int64_t* out) {
  return guarded([&] {
    muxsim::LLMSpec s;
    s.num_layers = num_layers;
    s.num_heads = num_heads;
    *out = muxsim::blocks_for_tokens(s, block_tokens, tokens);
  });
}

int mux_init_token_block_quota(int n, const double* rate, const double* bpt, const double* mean_tokens,
                               int64_t kv_blocks, double floor_frac, int64_t* out) {
  return guarded([&] {
    std::vector<muxsim::QuotaInput> in(n);
    for (int i = 0; i < n; ++i) in[i] = {rate[i], bpt[i], mean_tokens[i]};
    std::vector<int64_t> q = muxsim::init_token_block_quota(in, kv_blocks, floor_frac);
    std::copy(q.begin(), q.end(), out);
  });
}

int mux_adapt_quota(int n, const double* util, const int64_t* quotas, int64_t floor_blocks, double low,
                    double high, double step, int64_t* out) {
  return guarded([&] {
    muxsim::QuotaAdaptParams p{low, high, step};
    std::vector<int64_t> q = muxsim::adapt_quota(std::vector<double>(util, util + n),
                                                 std::vector<int64_t>(quotas, quotas + n), floor_blocks, p);
    std::copy(q.begin(), q.end(), out);
  });
}

int mux_pool_create(int64_t total_blocks, int physical, mux_pool** out) {
  return guarded([&] {
    auto p = std::make_unique<mux_pool>();
    p->owned = std::make_unique<BlockPool>(total_blocks);
    p->bp = p->owned.get();
    if (physical) p->bp->enable_physical(physical);  // physical > 1: ids sharded over that many TP ranks
    *out = p.release();
  });
}

void mux_pool_destroy(mux_pool* pool) { delete pool; }

int mux_pool_register_llm(mux_pool* pool, int llm, int layers, int heads, int head_dim, int bpe, int block_tokens) {
  return guarded([&] {
    muxsim::LLMSpec s;
    s.name = "llm" + std::to_string(llm);
    s.num_layers = layers;
    s.num_heads = heads;
    s.head_dim = head_dim;
    s.hidden_size = heads * head_dim;
    s.weight_bytes = 1;
    s.bytes_per_element = bpe;
    pool->specs.push_back(s);
    pool->bp->register_llm(llm, &pool->specs.back(), block_tokens);
  });
}

int mux_pool_admit(mux_pool* pool, int llm, int64_t rid, int64_t prompt, int64_t total, int* result) {
  return guarded([&] { *result = alloc_code(pool->bp->admit(llm, rid, prompt, total)); });
}

int mux_pool_alloc(mux_pool* pool, int llm, int64_t rid, int64_t add, int enforce, int* result) {
  return guarded([&] { *result = alloc_code(pool->bp->alloc(llm, rid, add, enforce != 0)); });
}

int mux_pool_alloc_n(mux_pool* pool, int llm, int n, const int64_t* rids, int64_t add, int enforce, int* results) {
  return guarded([&] {
    require(n >= 0 && (n == 0 || (rids != nullptr && results != nullptr)), "null argument");
    for (int i = 0; i < n; ++i) results[i] = alloc_code(pool->bp->alloc(llm, rids[i], add, enforce != 0));
  });
}

int mux_pool_free_request(mux_pool* pool, int llm, int64_t rid) {
  return guarded([&] { pool->bp->free_request(llm, rid); });
}

int mux_pool_set_quota(mux_pool* pool, int llm, int64_t blocks) {
  return guarded([&] { pool->bp->set_quota(llm, blocks); });
}

int mux_pool_llm_stats(const mux_pool* pool, int llm, int64_t* quota, int64_t* used, int64_t* committed) {
  return guarded([&] {
    if (quota) *quota = pool->bp->quota(llm);
    if (used) *used = pool->bp->used(llm);
    if (committed) *committed = pool->bp->committed(llm);
  });
}

int mux_pool_request_tokens(const mux_pool* pool, int llm, int64_t rid, int64_t* tokens) {
  return guarded([&] { *tokens = pool->bp->request_tokens(llm, rid); });
}

int mux_pool_totals(const mux_pool* pool, int64_t* free_blocks, int64_t* total, int64_t* committed) {
  return guarded([&] {
    if (free_blocks) *free_blocks = pool->bp->free_blocks();
    if (total) *total = pool->bp->total_blocks();
    if (committed) *committed = pool->bp->committed_total();
  });
}

int mux_pool_check(const mux_pool* pool) {
  return guarded([&] { pool->bp->check_conservation(); });
}

int mux_pool_block_table(const mux_pool* pool, int llm, int64_t rid, int32_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&] {
    if (!pool->bp->physical()) throw std::logic_error("block pool: physical ids are disabled");
    std::vector<int32_t> t = pool->bp->block_table(llm, rid);
    *n_out = static_cast<int64_t>(t.size());
    if (out) std::copy_n(t.begin(), std::min<int64_t>(cap, *n_out), out);
  });
}

int mux_pool_slot(const mux_pool* pool, int llm, int64_t rid, int* slot) {
  return guarded([&] { *slot = pool->bp->slot_of(llm, rid); });
}

int mux_simulate(const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries, int n_requests,
                 const mux_request* trace, mux_record* records_out) {
  return guarded([&] {
    SimInputs in = build_inputs(cfg, n_entries, entries, n_requests, trace);
    muxsim::SimResult res = muxsim::run_simulation(in.cluster, in.placement, in.entries, in.trace, in.prof, in.params);
    export_records(res, in, records_out);
  });
}

int mux_simulate_stats(const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries, int n_requests,
                       const mux_request* trace, mux_record* records_out, mux_sim_stats** stats_out) {
  return guarded([&] {
    require(stats_out != nullptr, "null argument");
    *stats_out = nullptr;
    SimInputs in = build_inputs(cfg, n_entries, entries, n_requests, trace);
    muxsim::SimResult res = muxsim::run_simulation(in.cluster, in.placement, in.entries, in.trace, in.prof, in.params);
    export_records(res, in, records_out);
    auto st = std::make_unique<mux_sim_stats>();
    for (size_t i = 0; i < in.entries.size(); ++i) st->idx[in.entries[i].spec.name] = static_cast<int>(i);
    st->units = std::move(res.units);
    *stats_out = st.release();
  });
}

void mux_sim_stats_destroy(mux_sim_stats* st) { delete st; }

int mux_sim_stats_units(const mux_sim_stats* st, int* n_units) {
  return guarded([&] {
    require(st != nullptr && n_units != nullptr, "null argument");
    *n_units = static_cast<int>(st->units.size());
  });
}

int mux_sim_stats_unit(const mux_sim_stats* st, int u, mux_unit_stats* out) {
  return guarded([&] {
    require(st != nullptr && out != nullptr, "null argument");
    require(u >= 0 && u < static_cast<int>(st->units.size()), "unit out of range");
    const muxsim::UnitStats& us = st->units[u];
    out->unit = us.unit;
    out->total_blocks = us.total_blocks;
    out->n_llms = static_cast<int>(us.llms.size());
    out->n_samples = static_cast<int64_t>(us.samples.size());
  });
}

int mux_sim_stats_llms(const mux_sim_stats* st, int u, mux_unit_llm_stats* out) {
  return guarded([&] {
    require(st != nullptr && out != nullptr, "null argument");
    require(u >= 0 && u < static_cast<int>(st->units.size()), "unit out of range");
    const muxsim::UnitStats& us = st->units[u];
    for (size_t i = 0; i < us.llms.size(); ++i) {
      const muxsim::UnitLlmStats& m = us.llms[i];
      out[i] = {st->idx.at(m.llm), m.rate, m.avg_used_blocks, m.final_quota_blocks, m.resource_usage};
    }
  });
}

int mux_sim_stats_samples(const mux_sim_stats* st, int u, mux_pool_sample* out) {
  return guarded([&] {
    require(st != nullptr && out != nullptr, "null argument");
    require(u >= 0 && u < static_cast<int>(st->units.size()), "unit out of range");
    const muxsim::UnitStats& us = st->units[u];
    for (size_t i = 0; i < us.samples.size(); ++i) {
      const muxsim::PoolSample& p = us.samples[i];
      out[i] = {p.t_s, st->idx.at(p.llm), p.used_blocks, p.quota_blocks};
    }
  });
}

int mux_parallel_candidates(int n_entries, const mux_llm_entry* entries, int num_nodes, int gpus_per_node,
                            int64_t gpu_memory_bytes, const double* profile, const double* decode_hbm,
                            const double* tp_allreduce, int n_tp, const int* tp_list, int n_sm,
                            const double* sm_list, double activation_reserve_frac, int max_batch,
                            mux_candidate* out, int capacity, int* n_out) {
  return guarded([&] {
    require(n_entries >= 0 && (n_entries == 0 || entries != nullptr) && n_out != nullptr, "null argument");
    require(n_tp >= 0 && (n_tp == 0 || tp_list != nullptr) && n_sm >= 0 && (n_sm == 0 || sm_list != nullptr),
            "null argument");
    std::vector<muxsim::LlmEntry> llms;
    std::vector<int> ffn;
    for (int i = 0; i < n_entries; ++i) {
      muxsim::LlmEntry e;
      e.spec = spec_of(entries[i]);
      e.rate = entries[i].rate;
      e.mean_prompt_tokens = entries[i].mean_prompt_tokens;
      e.mean_output_tokens = entries[i].mean_output_tokens;
      llms.push_back(e);
      ffn.push_back(entries[i].ffn);
    }
    muxsim::Cluster cl;
    cl.num_nodes = num_nodes;
    cl.gpus_per_node = gpus_per_node;
    cl.gpu_memory_bytes = gpu_memory_bytes;
    muxsim::CandidateParams cp;
    if (n_tp) cp.tp_list.assign(tp_list, tp_list + n_tp);
    if (n_sm) cp.sm_list.assign(sm_list, sm_list + n_sm);
    cp.activation_reserve_frac = activation_reserve_frac;
    cp.max_batch = max_batch;
    auto cands = muxsim::realizable_parallel_candidates(llms, cl, profile_of(profile, decode_hbm, tp_allreduce), cp, ffn);
    int n = 0;
    for (size_t i = 0; i < cands.size(); ++i)
      for (const auto& c : cands[i]) {
        if (out != nullptr && n < capacity)
          out[n] = {static_cast<int>(i), c.tp_degree, c.num_sm, c.batch, c.est_tpt, c.saturated ? 1 : 0};
        ++n;
      }
    *n_out = n;
  });
}

int mux_slo_reference_latency_ms(const mux_llm_entry* entry, const double* profile, int tp_degree, int prompt_len,
                                 int output_len, double* out_ms) {
  return guarded([&] {
    require(entry != nullptr && out_ms != nullptr, "null argument");
    const muxsim::LLMSpec spec = spec_of(*entry);
    muxsim::LatencyProfile prof;
    if (profile) {
      prof.prefill_ms_per_token = profile[0];
      prof.decode_base_ms = profile[1];
      prof.decode_ctx_ms_per_token = profile[2];
      prof.tp_efficiency = profile[3];
      prof.sm_saturation_point = profile[4];
      prof.batch_knee = profile[5];
      prof.reference_scale = profile[6];
    }
    // metrics.cpp:21-27: one prefill over the prompt + output_len-1 decode
    // steps, context growing by one token per step, whole SM budget
    muxsim::ExecConfig cfg{tp_degree, 1.0};
    double t = muxsim::prefill_latency(spec, prof, cfg, 1, prompt_len);
    for (int k = 1; k < output_len; ++k) t += muxsim::decode_step_latency(spec, prof, cfg, 1, prompt_len + k);
    *out_ms = t;
  });
}

int mux_decode_attention_headwise(const void* q, const void* pool, const int32_t* rowrec, const int32_t* rowlist,
                                  const int32_t* slots, const int32_t* ctx, int B, int H, int num_layers,
                                  int layer, int max_rows, int max_ctx, void* out, int out_fp32, int kv_splits,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    require(H > 0 && B >= 0 && layer >= 0 && layer < num_layers, "decode attention: bad shape");
    mux::DecodeAttnArgs a{};
    a.q = q;
    a.pool = pool;
    a.rowrec = rowrec;
    a.rowlist = rowlist;
    a.slots = slots;
    a.ctx = ctx;
    a.out = out;
    a.B = B;
    a.H = H;
    a.layer = layer;
    a.max_rows = max_rows;
    a.row_width = 2 * num_layers * H;
    const int rows = std::max(1, (max_ctx + 15) / 16);
    int splits = kv_splits > 0 ? kv_splits : 1;
    while ((rows + splits - 1) / splits > mux::decode_attention_max_rows_per_split()) splits *= 2;
    a.splits = splits;
    a.rows_per_split = (rows + splits - 1) / splits;
    if (splits > 1) {
      const size_t need = static_cast<size_t>(B) * H * splits * (128 + 2) * 4;
      require(workspace != nullptr && workspace_bytes >= need, "decode attention: workspace too small");
      a.part_o = static_cast<float*>(workspace);
      a.part_ml = a.part_o + static_cast<size_t>(B) * H * splits * 128;
    }
    a.scale_log2 = 1.4426950408889634f / std::sqrt(128.f);
    mux::check_cuda(mux::decode_attention(a, out_fp32 != 0, static_cast<cudaStream_t>(stream)), "decode_attention");
  });
}

int mux_prefill_attention(const void* q, const void* qkv, void* out, const int32_t* seq_lens, int nseq, int H,
                          void* stream) {
  return guarded([&] {
    require(nseq > 0 && H > 0 && seq_lens != nullptr, "prefill attention: bad shape");
    std::vector<int32_t> meta(nseq + 1, 0);
    int T = 0, max_qt = 0;
    for (int i = 0; i < nseq; ++i) {
      require(seq_lens[i] > 0, "prefill attention: empty sequence");
      meta[i] = T;
      T += seq_lens[i];
      max_qt = std::max(max_qt, (seq_lens[i] - 1) / 128);
    }
    meta[nseq] = T;
    require(nseq < 65536 && max_qt < 65536, "prefill attention: too many sequences");
    for (int qt = max_qt; qt >= 0; --qt)
      for (int i = 0; i < nseq; ++i)
        if (qt * 128 < seq_lens[i]) meta.push_back((i << 16) | qt);
    const int n_tiles = static_cast<int>(meta.size()) - (nseq + 1);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static mux::DevMem& d = *new mux::DevMem();  // grows; the call synchronises before returning
    if (d.bytes < meta.size() * 4) d = mux::DevMem(std::max<size_t>(meta.size() * 4, 1 << 16));
    mux::check_cuda(cudaMemcpyAsync(d.p, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, s), "meta");
    alignas(64) unsigned char tq[128], tkv[128];
    if (!mux::make_tmap_bf16(tq, q, T, static_cast<uint64_t>(H) * 128, static_cast<uint64_t>(H) * 256, 128) ||
        !mux::make_tmap_bf16(tkv, qkv, T, static_cast<uint64_t>(3 * H) * 128, static_cast<uint64_t>(3 * H) * 256, 128))
      throw std::runtime_error("prefill attention: tensor map encode failed");
    mux::PrefillAttnArgs a{};
    a.q = q;
    a.qkv = qkv;
    a.out = out;
    a.seq_start = d.as<int32_t>();
    a.tiles = d.as<int32_t>() + nseq + 1;
    a.tmap_q = tq;
    a.tmap_qkv = tkv;
    a.n_tiles = n_tiles;
    a.nseq = nseq;
    a.H = H;
    a.T = T;
    a.scale_log2 = 1.4426950408889634f / std::sqrt(128.f);
    // test hook: a small persistent grid puts many items on each CTA
    if (const char* e = std::getenv("MUX_K3_CTAS")) a.max_ctas = std::atoi(e);
    mux::check_cuda(mux::prefill_attention(a, s), "prefill_attention");
    mux::check_cuda(cudaStreamSynchronize(s), "prefill_attention sync");
  });
}

int mux_kv_append(const void* qkv, void* q_out, void* pool, const int32_t* rowrec, const int32_t* rowlist,
                  const int32_t* tok_slot, const int32_t* tok_pos, const float* rope, int rope_positions, int T,
                  int H, int num_layers, int layer, int max_rows, void* stream) {
  return guarded([&] {
    mux::AppendArgs a{};
    a.qkv = qkv;
    a.q_out = q_out;
    a.pool = pool;
    a.rowrec = rowrec;
    a.rowlist = rowlist;
    a.tok_slot = tok_slot;
    a.tok_pos = tok_pos;
    a.rope = rope;
    a.T = T;
    a.H = H;
    a.layer = layer;
    a.max_rows = max_rows;
    a.row_width = 2 * num_layers * H;
    a.rope_positions = rope_positions;
    mux::check_cuda(mux::kv_append(a, static_cast<cudaStream_t>(stream)), "kv_append");
  });
}

int mux_rope_table(int positions, float* out) {
  return guarded([&] {
    for (int p = 0; p < positions; ++p)
      for (int i = 0; i < 64; ++i) {
        const double inv_freq = 1.0 / std::pow(10000.0, 2.0 * i / 128.0);
        const double ang = static_cast<double>(p) * inv_freq;
        out[static_cast<size_t>(p) * 128 + 2 * i] = static_cast<float>(std::cos(ang));
        out[static_cast<size_t>(p) * 128 + 2 * i + 1] = static_cast<float>(std::sin(ang));
      }
  });
}

void mux_debug_gemm_timing(void* buf) { mux::gemm_debug_timing(buf); }

int64_t mux_weight_tiled_bytes(int N, int K) { return static_cast<int64_t>(mux::weight_tiled_bytes(N, K)); }

int mux_weight_tile(const void* w, int N, int K, void* out, int inverse, void* stream) {
  return guarded([&] {
    require(N > 0 && K > 0 && K % 8 == 0, "weight_tile: bad shape");
    mux::check_cuda(mux::weight_tile(w, N, K, out, inverse != 0, static_cast<cudaStream_t>(stream)), "weight_tile");
  });
}

int mux_gemm_bf16(const void* x, const void* w, int w_tiled, int M, int N, int K, void* out, int epilogue, int grid,
                  void* stream) {
  return guarded([&] {
    require(M > 0 && N > 0 && K > 0 && K % 8 == 0 && N % 8 == 0, "gemm: bad shape");
    require(epilogue >= 0 && epilogue <= 3, "gemm: bad epilogue");
    require(epilogue != 2 || N % 16 == 0, "gemm: SiLU epilogue needs N % 16 == 0");
    // Stream-K scratch for direct calls (tests), one set per device (the
    // runtime gives every partition its own). Calls on one device are
    // serialised by the caller's stream order, as with any shared scratch.
    struct Scratch {
      float* partials = nullptr;
      int* flags = nullptr;
      int epoch = 0;
    };
    static std::mutex mu;
    static std::map<int, Scratch> per_dev;
    constexpr int kMaxGrid = 1024;
    int dev = 0;
    mux::check_cuda(cudaGetDevice(&dev), "gemm device");
    std::lock_guard<std::mutex> lk(mu);
    Scratch& sc = per_dev[dev];
    if (sc.partials == nullptr) {
      mux::check_cuda(cudaMalloc(&sc.partials, mux::gemm_partials_floats(kMaxGrid) * 4), "gemm scratch");
      mux::check_cuda(cudaMalloc(&sc.flags, 2 * kMaxGrid * 4), "gemm flags");
      mux::check_cuda(cudaMemset(sc.flags, 0, 2 * kMaxGrid * 4), "gemm flags");
    }
    float* partials = sc.partials;
    int* flags = sc.flags;
    int& epoch = sc.epoch;
    int sms = 148;
    mux::check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "gemm SM count");
    alignas(64) unsigned char tw[128], tx[128], to[128], tx128[128], txh[128], twr[128];
    const int n_tile = mux::gemm_pick_n_tile(M);
    if ((!w_tiled && !mux::make_tmap_bf16(tw, w, N, K, static_cast<uint64_t>(K) * 2, 128)) ||
        !mux::make_tmap_bf16(tx, x, M, K, static_cast<uint64_t>(K) * 2, n_tile))
      throw std::runtime_error("gemm: tensor map encode failed");
    const int ldo = epilogue == 2 ? N / 2 : N;
    if (!mux::make_tmap_gemm_out(to, out, epilogue, M, N, ldo)) throw std::runtime_error("gemm: out map encode failed");
    mux::GemmArgs g{};
    g.tmap_out = to;
    g.w_tiled = w_tiled ? w : nullptr;
    g.tmap_w = w_tiled ? nullptr : tw;
    g.tmap_x = tx;
    // prefill shapes with tiled weights may run on CTA pairs (gemm_2sm.cu)
    if (w_tiled && M > 256 && mux::make_tmap_bf16(tx128, x, M, K, static_cast<uint64_t>(K) * 2, 128)) g.tmap_x128 = tx128;
    // decode shapes with tiled weights may run on CTA pairs (MUX_GEMM_PAIR)
    if (w_tiled && n_tile >= 16 &&
        mux::make_tmap_bf16(txh, x, M, K, static_cast<uint64_t>(K) * 2, n_tile / 2) &&
        mux::make_tmap_w_rows(twr, w, N, K)) {
      g.tmap_x_half = txh;
      g.tmap_w_rows = twr;
    }
    g.out = out;
    g.partials = partials;
    g.flags = flags;
    g.epoch = ++epoch;
    g.grid = std::min(kMaxGrid, grid > 0 ? grid : sms);
    g.M = M;
    g.N = N;
    g.K = K;
    g.ldo = ldo;
    g.epi = static_cast<mux::Epilogue>(epilogue);
    mux::check_cuda(mux::gemm_bf16_tn(g, static_cast<cudaStream_t>(stream)), "gemm");
  });
}

int mux_unit_create(const mux_unit_config* cfg, mux_unit** out) {
  return guarded([&] {
    require(cfg != nullptr && cfg->n_llms > 0 && cfg->llms != nullptr, "unit: bad config");
    auto u = std::make_unique<mux_unit>();
    const int64_t dev_blocks = cfg->device_pool_blocks > 0 ? std::min(cfg->device_pool_blocks, cfg->pool_blocks)
                                                           : cfg->pool_blocks;
    const int max_ctx = std::max(cfg->max_ctx, 16);
    u->rt = std::make_unique<mux::Runtime>(cfg->device, dev_blocks, max_ctx + 16);
    u->pool.owned = std::make_unique<BlockPool>(cfg->pool_blocks);
    u->pool.bp = u->pool.owned.get();
    u->pool.bp->enable_physical();
    u->max_batch = std::max(1, cfg->max_batch);
    u->max_prefill = std::max(16, cfg->max_prefill_tokens);
    const int max_rows = (max_ctx + 15) / 16;
    int hid = 0, qkv = 0, ffn = 0, vocab = 0, heads = 0;
    const int tp = std::max(1, cfg->tp_size), tp_rank = tp > 1 ? cfg->tp_rank : 0;
    require(tp <= mux::kMaxTp && tp_rank >= 0 && tp_rank < tp, "unit: bad tensor-parallel rank/size");
    for (int i = 0; i < cfg->n_llms; ++i) {
      const mux_llm_entry& e = cfg->llms[i];
      // the reference planner never checks head divisibility.
      require(e.head_dim == 128 && e.bytes_per_element == 2,
              "unit: the kernels serve head_dim 128, bf16 (4 KiB head-blocks of 16 tokens)");
      require(e.num_heads % tp == 0 && e.ffn % tp == 0,
              "unit: heads and ffn must be divisible by tp_size (reference planner emits e.g. 30b at tp 8)");
      u->specs.push_back(spec_of(e));
      u->specs.back().num_heads = e.num_heads / tp;  // this rank's head slice of the pool rows
      u->pool.bp->register_llm(i, &u->specs.back(), 16);
      u->pool.bp->set_quota(i, cfg->pool_blocks);  // no quota until a scheduler sets one
      mux::ModelDims d;
      d.name = u->specs.back().name;
      d.layers = e.num_layers;
      d.heads = e.num_heads / tp;
      d.head_dim = e.head_dim;
      d.hidden = e.hidden_size;
      d.ffn = e.ffn / tp;
      d.vocab = e.vocab;
      d.tp_rank = tp_rank;
      d.tp_size = tp;
      const int64_t row_blocks = 2ll * e.num_layers * d.heads;
      const int64_t max_rowrecs = std::max<int64_t>(1, cfg->pool_blocks / row_blocks);
      const int slots = cfg->max_slots > 0 ? cfg->max_slots : static_cast<int>(std::min<int64_t>(max_rowrecs, 1 << 20));
      u->models.push_back(std::make_unique<mux::Llama>(d, slots, max_rows, max_rowrecs));
      if (cfg->init_seed != 0) u->models.back()->init_random(cfg->init_seed + 7919ull * i, cfg->init_std, nullptr);
      hid = std::max(hid, d.hidden);
      qkv = std::max(qkv, 3 * d.heads * 128);
      ffn = std::max(ffn, d.ffn);
      vocab = std::max(vocab, d.vocab);
      heads = std::max(heads, d.heads);
    }
    const int P = std::max(1, cfg->partitions);
    // Green-context SM partitions: the device's SMs are split once into
    // 8-SM granules (the sm_100 partition granularity; on B200 that yields
    // 15 symmetric granules = 120 SMs plus a 28-SM remainder outside the
    // symmetric set); partition p takes the next ceil(want/8) granules, the
    // remainder joins the first partition that runs out of granules (else the
    // last green partition), so partitions are disjoint by construction.
    std::vector<CUdevResource> granules;
    CUdevResource remainder{};
    bool remainder_free = false;
    size_t next_granule = 0;
    int last_green = -1;
    if (cfg->partition_sms != nullptr) {
      bool any = false;
      for (int p = 0; p < P; ++p) any = any || cfg->partition_sms[p] > 0;
      if (any) {
        GreenApi& ga = green_api();
        CUdevice dev = 0;
        CUdevResource all{};
        check_cu(ga.device_get(&dev, cfg->device), "cuDeviceGet");
        check_cu(ga.get_resource(dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
        unsigned int nb = 0;
        check_cu(ga.split(nullptr, &nb, &all, nullptr, 0, 8), "cuDevSmResourceSplitByCount(query)");
        granules.resize(nb);
        check_cu(ga.split(granules.data(), &nb, &all, &remainder, 0, 8), "cuDevSmResourceSplitByCount");
        granules.resize(nb);
        remainder_free = remainder.sm.smCount > 0;
        for (int p = 0; p < P; ++p)
          if (cfg->partition_sms[p] > 0) last_green = p;
      }
    }
    for (int p = 0; p < P; ++p) {
      const int want = cfg->partition_sms ? cfg->partition_sms[p] : 0;
      cudaStream_t s;
      CUgreenCtx g = nullptr;
      int sms = u->rt->num_sms();
      if (want > 0) {
        GreenApi& ga = green_api();
        int take = 0, got = 0;
        while (got < want && next_granule + take < granules.size()) got += granules[next_granule + take++].sm.smCount;
        std::vector<CUdevResource> parts(granules.begin() + next_granule, granules.begin() + next_granule + take);
        if (remainder_free && (got < want || p == last_green)) {
          parts.push_back(remainder);
          got += remainder.sm.smCount;
          remainder_free = false;
        }
        if (got < want) {
          std::string sizes;
          for (const CUdevResource& r : granules) sizes += " " + std::to_string(r.sm.smCount);
          throw std::invalid_argument("partition_sms: not enough SMs left for partition " + std::to_string(p) +
                                      " (granules:" + sizes + ")");
        }
        CUdevResourceDesc desc;
        check_cu(ga.gen_desc(&desc, parts.data(), static_cast<unsigned>(parts.size())), "cuDevResourceGenerateDesc");
        next_granule += take;
        CUdevice dev = 0;
        check_cu(ga.device_get(&dev, cfg->device), "cuDeviceGet");
        check_cu(ga.create(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
        CUstream cs;
        check_cu(ga.stream_create(&cs, g, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
        s = reinterpret_cast<cudaStream_t>(cs);
        sms = got;
      } else {
        mux::check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
      }
      u->streams.push_back(s);
      u->green.push_back(g);
      u->sms.push_back(sms);
      const int max_tok = std::max(u->max_prefill, u->max_batch);
      u->ws.push_back(std::make_unique<mux::Workspace>(max_tok, std::max(u->max_batch, 256), hid, qkv, ffn, vocab,
                                                       heads, u->max_batch, u->rt->num_sms()));
      u->ws.back()->sms = sms;
      u->ws.back()->exclusive = g != nullptr;
      if (tp > 1) {
        auto link = std::make_unique<mux::TpLink>();
        link->rank = tp_rank;
        link->size = tp;
        link->rows = std::max(max_tok, 256);
        link->hidden = hid;
        link->box = mux::DevMem(2 * tp * link->slot_floats() * 4 + 256);
        mux::check_cuda(cudaMemset(link->box.p, 0, link->box.bytes), "tp mailbox");
        link->peer[tp_rank] = link->box.p;
        u->ws.back()->tp = std::move(link);
      }
    }
    for (auto& e : u->ev) mux::check_cuda(cudaEventCreate(&e), "event");
    mux::check_cuda(cudaDeviceSynchronize(), "unit create");
    *out = u.release();
  });
}

void mux_unit_destroy(mux_unit* unit) { delete unit; }

mux_pool* mux_unit_pool(mux_unit* unit) { return unit ? &unit->pool : nullptr; }

int mux_unit_set_tensor(mux_unit* u, int llm, const char* name, int layer, const void* host, size_t bytes) {
  return guarded([&] {
    if (!u->model(llm).set_tensor(name, layer, host, bytes, u->streams[0]))
      throw std::invalid_argument(std::string("set_tensor: unknown tensor or size mismatch: ") + name);
  });
}

int mux_unit_get_tensor(mux_unit* u, int llm, const char* name, int layer, void* host, size_t bytes) {
  return guarded([&] {
    if (!u->model(llm).get_tensor(name, layer, host, bytes, u->streams[0]))
      throw std::invalid_argument(std::string("get_tensor: unknown tensor or size mismatch: ") + name);
  });
}

int mux_unit_init_kv(mux_unit* u, uint64_t seed, float std) {
  return guarded([&] {
    mux::check_cuda(mux::init_normal_bf16(u->rt->pool(), u->rt->pool_blocks() * 2048, seed, std, u->streams[0]),
                    "init kv");
    u->rt->count_launch();
    mux::check_cuda(cudaStreamSynchronize(u->streams[0]), "init kv sync");
  });
}

int mux_unit_device_ptrs(mux_unit* u, int llm, void** pool, void** rowrec, void** rowlist, int* max_rows,
                         int* row_width) {
  return guarded([&] {
    mux::Llama& m = u->model(llm);
    if (pool) *pool = u->rt->pool();
    if (rowrec) *rowrec = m.rowrec.p;
    if (rowlist) *rowlist = m.rowlist.p;
    if (max_rows) *max_rows = m.max_rows();
    if (row_width) *row_width = m.row_width();
  });
}

int mux_unit_prefill(mux_unit* u, int llm, int n, const int64_t* rids, const int32_t* tokens, int32_t* out_tokens,
                     int partition) {
  return guarded([&] {
    mux::Llama& m = u->model(llm);
    cudaStream_t s = u->stream(partition);
    u->rt->upload_rows(*u->pool.bp, llm, m, s);
    std::vector<int32_t> slots(n), lens(n);
    for (int i = 0; i < n; ++i) {
      slots[i] = u->pool.bp->slot_of(llm, rids[i]);
      lens[i] = static_cast<int32_t>(u->pool.bp->request_tokens(llm, rids[i]));
      require(slots[i] >= 0 && lens[i] > 0, "prefill: request not admitted");
    }
    u->rt->prefill(m, *u->ws[partition], n, slots.data(), lens.data(), tokens, out_tokens, s);
  });
}

int mux_unit_decode(mux_unit* u, int llm, int n, const int64_t* rids, const int32_t* tokens, int32_t* out_tokens,
                    int partition) {
  return guarded([&] {
    mux::Llama& m = u->model(llm);
    cudaStream_t s = u->stream(partition);
    u->rt->upload_rows(*u->pool.bp, llm, m, s);
    std::vector<int32_t> slots(n), ctx(n);
    for (int i = 0; i < n; ++i) {
      slots[i] = u->pool.bp->slot_of(llm, rids[i]);
      ctx[i] = static_cast<int32_t>(u->pool.bp->request_tokens(llm, rids[i]));
      require(slots[i] >= 0 && ctx[i] > 0, "decode: request has no cached tokens");
    }
    u->rt->decode(m, *u->ws[partition], n, slots.data(), ctx.data(), tokens, out_tokens, s,
                  u->timing ? &u->timer : nullptr);
  });
}

int mux_unit_sync(mux_unit* u) {
  return guarded([&] { mux::check_cuda(cudaDeviceSynchronize(), "sync"); });
}

int mux_unit_record(mux_unit* u, int partition, int slot) {
  return guarded([&] {
    require(slot >= 0 && slot < 64, "event slot out of range");
    mux::check_cuda(cudaEventRecord(u->ev[slot], u->stream(partition)), "record");
  });
}

int mux_unit_elapsed(mux_unit* u, int a, int b, float* ms) {
  return guarded([&] {
    require(a >= 0 && a < 64 && b >= 0 && b < 64, "event slot out of range");
    mux::check_cuda(cudaEventSynchronize(u->ev[b]), "elapsed sync");
    mux::check_cuda(cudaEventElapsedTime(ms, u->ev[a], u->ev[b]), "elapsed");
  });
}

int mux_unit_attn_timing(mux_unit* u, int enable) {
  return guarded([&] {
    u->timer.harvest();
    u->gemm_timer.harvest();
    u->timing = enable != 0;
    u->rt->set_gemm_timer(u->timing ? &u->gemm_timer : nullptr);
    for (mux::AttnTimer* t : {&u->timer, &u->gemm_timer}) {
      t->total_ms = 0.0;
      t->bytes = 0.0;
      t->launches = 0;
    }
  });
}

int mux_unit_gemm_time(mux_unit* u, double* total_ms, int64_t* launches, double* bytes) {
  return guarded([&] {
    u->gemm_timer.harvest();
    if (total_ms) *total_ms = u->gemm_timer.total_ms;
    if (launches) *launches = u->gemm_timer.launches;
    if (bytes) *bytes = u->gemm_timer.bytes;
  });
}

int mux_unit_attn_time(mux_unit* u, double* total_ms, int64_t* launches, double* bytes) {
  return guarded([&] {
    u->timer.harvest();
    if (total_ms) *total_ms = u->timer.total_ms;
    if (launches) *launches = u->timer.launches;
    if (bytes) *bytes = u->timer.bytes;
  });
}

int64_t mux_unit_launches(mux_unit* u) { return u ? u->rt->launches() : -1; }

int mux_unit_pass_stats(mux_unit* u, int64_t* passes, int64_t* green_passes) {
  return guarded([&] {
    if (u == nullptr) throw std::invalid_argument("null unit");
    if (passes) *passes = u->passes;
    if (green_passes) *green_passes = u->green_passes;
  });
}

int mux_unit_tp_mailbox(mux_unit* u, int partition, void** dev_ptr, void* ipc_handle) {
  return guarded([&] {
    u->stream(partition);
    mux::TpLink* t = u->ws[partition]->tp.get();
    require(t != nullptr, "tp mailbox: unit was created without tensor parallelism");
    if (dev_ptr) *dev_ptr = t->box.p;
    if (ipc_handle) {
      cudaIpcMemHandle_t h;
      mux::check_cuda(cudaIpcGetMemHandle(&h, t->box.p), "cudaIpcGetMemHandle");
      std::memcpy(ipc_handle, &h, sizeof(h));
    }
  });
}

int mux_unit_tp_connect(mux_unit* u, int partition, int peer_rank, const void* ipc_handle, void* dev_ptr) {
  return guarded([&] {
    u->stream(partition);
    mux::TpLink* t = u->ws[partition]->tp.get();
    require(t != nullptr, "tp connect: unit was created without tensor parallelism");
    require(peer_rank >= 0 && peer_rank < t->size && peer_rank != t->rank, "tp connect: bad peer rank");
    require(t->peer[peer_rank] == nullptr, "tp connect: peer already connected");
    if (ipc_handle != nullptr) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, ipc_handle, sizeof(h));
      void* p = nullptr;
      mux::check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      t->peer[peer_rank] = p;
      t->ipc_opened[peer_rank] = true;
    } else {
      require(dev_ptr != nullptr, "tp connect: need an IPC handle or a device pointer");
      t->peer[peer_rank] = dev_ptr;
    }
  });
}

int mux_unit_tp_debug(mux_unit* u, int partition, uint32_t* out) {
  return guarded([&] {
    u->stream(partition);
    mux::TpLink* t = u->ws[partition]->tp.get();
    require(t != nullptr, "tp debug: no tensor parallelism");
    cudaStream_t side;
    mux::check_cuda(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "side stream");
    mux::PinnedMem h(8);
    mux::check_cuda(cudaMemcpyAsync(h.p, t->counter(t->rank, 0), 8, cudaMemcpyDeviceToHost, side), "counter read");
    mux::check_cuda(cudaStreamSynchronize(side), "counter sync");
    cudaStreamDestroy(side);
    out[0] = h.as<uint32_t>()[0];
    out[1] = h.as<uint32_t>()[1];
    out[2] = t->expected[0];
    out[3] = t->expected[1];
  });
}

int mux_unit_route_log(mux_unit* u, mux_route_record* out, int64_t cap, int64_t* n_out) {
  return guarded([&] {
    require(n_out != nullptr, "route log: null count");
    *n_out = static_cast<int64_t>(u->route_log.size());
    for (int64_t i = 0; out && i < std::min<int64_t>(cap, *n_out); ++i) {
      const RouteRecord& r = u->route_log[i];
      out[i] = mux_route_record{r.pass, r.job, r.llm, r.kind, r.sm_demand, r.first_unit, r.units, r.sms, r.workspace,
                                r.busy_units};
    }
  });
}

int mux_unit_route_units(mux_unit* u, int* n_units, int* unit_sms, int cap) {
  return guarded([&] {
    u->router.init(u->rt->device());
    *n_units = static_cast<int>(u->router.units.size());
    for (int i = 0; unit_sms && i < std::min(cap, *n_units); ++i) unit_sms[i] = u->router.unit_sms[i];
  });
}

int mux_unit_probe_route(mux_unit* u, int first_unit, int units, int blocks, int* out) {
  return guarded([&] {
    require(blocks > 0, "probe: blocks must be positive");
    u->router.init(u->rt->device());
    require(first_unit >= 0 && units > 0 && first_unit + units <= static_cast<int>(u->router.units.size()),
            "probe: bad SM run");
    cudaStream_t s = u->router.part(first_unit, units).s;
    mux::DevMem d(static_cast<size_t>(blocks) * 4);
    probe_smid_kernel<<<blocks, 32, 0, s>>>(d.as<int>());
    mux::check_cuda(cudaGetLastError(), "probe");
    mux::check_cuda(cudaMemcpyAsync(out, d.p, static_cast<size_t>(blocks) * 4, cudaMemcpyDeviceToHost, s), "probe copy");
    mux::check_cuda(cudaStreamSynchronize(s), "probe sync");
  });
}

int mux_unit_partition_sms(mux_unit* u, int partition, int* sms) {
  return guarded([&] {
    u->stream(partition);
    *sms = u->sms[partition];
  });
}

int mux_unit_probe_smids(mux_unit* u, int partition, int blocks, int* out) {
  return guarded([&] {
    require(blocks > 0, "probe: blocks must be positive");
    cudaStream_t s = u->stream(partition);
    mux::DevMem d(static_cast<size_t>(blocks) * 4);
    probe_smid_kernel<<<blocks, 32, 0, s>>>(d.as<int>());
    mux::check_cuda(cudaGetLastError(), "probe");
    mux::check_cuda(cudaMemcpyAsync(out, d.p, static_cast<size_t>(blocks) * 4, cudaMemcpyDeviceToHost, s), "probe copy");
    mux::check_cuda(cudaStreamSynchronize(s), "probe sync");
  });
}

int mux_unit_set_option(mux_unit* u, const char* key, int64_t value) {
  return guarded([&] {
    const std::string k = key ? key : "";
    if (k == "gemm_min_iters") u->rt->set_gemm_min_iters(static_cast<int>(value));
    else if (k == "pdl") mux::pdl_enabled() = value != 0;
    else if (k == "graphs") u->rt->set_graphs(value != 0);
    else if (k == "debug_skip") u->rt->set_debug_skip(static_cast<int>(value));
    else if (k == "prefill_on_partition") u->prefill_on_partition = value != 0;
    else if (k == "pass_green") u->pass_green = value != 0;
    else if (k == "align_decode") u->align_decode = value != 0;
    else if (k == "sm_route") {
      require(!u->pass_green && !u->align_decode, "sm_route excludes pass_green and align_decode");
      u->sm_route = value != 0;
      u->ws_owner.assign(u->ws.size(), -1);
    }
    else throw std::invalid_argument("unknown option: " + k);
  });
}

namespace {
int run_unit(mux_unit* u, const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries, int n_requests,
             const mux_request* trace, uint64_t prompt_seed, mux_record* records_out, int32_t* tokens_out,
             bool measured, bool realtime = false) {
  return guarded([&] {
    require(cfg->n_units == 1, "lockstep: single-unit placements only");
    const int tp = u->models.empty() ? 1 : u->models[0]->dims().tp_size;
    require(cfg->unit_mesh_size != nullptr && cfg->unit_mesh_size[0] == tp,
            "GPU engines: the unit's mesh size must equal the unit's tensor-parallel size");
    // every rank of a mesh must take the same decisions: priced durations
    // (lockstep) are rank-independent, measured device times are not
    require(tp == 1 || (!measured && !realtime), "tensor-parallel units run the lockstep engine only");
    // The kernels address 16-token head-blocks of 128 bf16 dims (4 KiB,
    // kv_manager.cpp:37-40 at the catalog's geometry); the host pool must
    // build rows of the same size.
    require(cfg->block_tokens == 16, "GPU engines: block_tokens must be 16 (the kernels' head-block geometry)");
    require(n_entries == static_cast<int>(u->models.size()), "lockstep: entries must describe the unit's models");
    SimInputs in = build_inputs(cfg, n_entries, entries, n_requests, trace);
    u->passes = u->green_passes = 0;
    u->route_log.clear();
    if (u->sm_route) {
      require(u->ws.size() >= u->models.size() + 1, "sm_route: the unit needs models + 1 partitions (workspaces)");
      u->ws_owner.assign(u->ws.size(), -1);
      if (u->router.ready) u->router.owner.assign(u->router.owner.size(), -1);
    }
    GpuExecutor exec(u, prompt_seed, in.trace, measured, realtime);
    muxsim::SimResult res =
        muxsim::run_simulation(in.cluster, in.placement, in.entries, in.trace, in.prof, in.params, &exec);
    export_records(res, in, records_out);
    u->last_stats = std::make_unique<mux_sim_stats>();
    for (size_t i = 0; i < in.entries.size(); ++i) u->last_stats->idx[in.entries[i].spec.name] = static_cast<int>(i);
    u->last_stats->units = res.units;
    if (tokens_out) {
      size_t off = 0;
      for (int i = 0; i < n_requests; ++i) {
        const auto& t = exec.tokens()[i];
        if (static_cast<int>(t.size()) != trace[i].output_len)
          throw std::logic_error("lockstep: request " + std::to_string(trace[i].id) + " produced " +
                                 std::to_string(t.size()) + " tokens, expected " + std::to_string(trace[i].output_len));
        std::copy(t.begin(), t.end(), tokens_out + off);
        off += t.size();
      }
    }
  });
}
}  // namespace

int mux_unit_run_lockstep(mux_unit* u, const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries,
                          int n_requests, const mux_request* trace, uint64_t prompt_seed, mux_record* records_out,
                          int32_t* tokens_out) {
  return run_unit(u, cfg, n_entries, entries, n_requests, trace, prompt_seed, records_out, tokens_out, false);
}

int mux_unit_run_measured(mux_unit* u, const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries,
                          int n_requests, const mux_request* trace, uint64_t prompt_seed, mux_record* records_out,
                          int32_t* tokens_out) {
  return run_unit(u, cfg, n_entries, entries, n_requests, trace, prompt_seed, records_out, tokens_out, true);
}

int mux_unit_run_realtime(mux_unit* u, const mux_sim_config* cfg, int n_entries, const mux_llm_entry* entries,
                          int n_requests, const mux_request* trace, uint64_t prompt_seed, mux_record* records_out,
                          int32_t* tokens_out) {
  return run_unit(u, cfg, n_entries, entries, n_requests, trace, prompt_seed, records_out, tokens_out, false, true);
}

int mux_unit_last_stats(mux_unit* u, mux_sim_stats** out) {
  return guarded([&] {
    require(u != nullptr && out != nullptr, "null argument");
    require(u->last_stats != nullptr, "no lockstep / measured run yet");
    *out = new mux_sim_stats(*u->last_stats);
  });
}

}  // extern "C"
