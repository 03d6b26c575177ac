// Differential fuzz (TEST INFRASTRUCTURE): the product's BlockPool and engine
// against the reference oracle, compiled in place with -Dmuxsim=muxref
// (oracle/Makefile) so both live in one binary. Every counter, every
// allocation result and every request record must be bit-identical.
//
//   diff_fuzz pool  <seed> <ops>        random admit/alloc/free/quota streams
//   diff_fuzz sim   <seed> <scenarios>  random units + traces, all 3 policies
//   diff_fuzz phys  <seed> <ops>        physical ids: disjoint, in range, LIFO
#define muxsim muxref
#include "muxsim/kv_manager.hpp"
#include "muxsim/placement.hpp"
#include "muxsim/rng.hpp"
#include "muxsim/sim_engine.hpp"
#include "muxsim/workload.hpp"
#undef muxsim

#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "mux/engine.hpp"
#include "mux/kv.hpp"

namespace {

int g_fail = 0;
long g_runs = 0, g_records = 0, g_errors = 0;

#define EXPECT(cond, ...)                                      \
  do {                                                         \
    if (!(cond)) {                                             \
      std::fprintf(stderr, "MISMATCH %s:%d: ", __FILE__, __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);                       \
      std::fprintf(stderr, "\n");                              \
      if (++g_fail > 20) std::exit(1);                         \
    }                                                          \
  } while (0)

muxsim::LLMSpec mine_spec(const muxref::LLMSpec& s) {
  return {s.name, s.num_layers, s.num_heads, s.head_dim, s.hidden_size, s.weight_bytes,
          s.bytes_per_element};
}

int err_code(muxref::AllocError e) { return static_cast<int>(e); }
int err_code(muxsim::AllocError e) { return static_cast<int>(e); }

// ------------------------------------------------------------------ pool fuzz
int fuzz_pool(std::uint64_t seed, int ops, bool physical) {
  std::mt19937_64 rng(seed);
  auto pick = [&](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  const int n = pick(1, 4);
  std::vector<muxref::LLMSpec> rs;
  for (int i = 0; i < n; ++i)
    rs.push_back({"m" + std::to_string(i), pick(1, 3), pick(1, 4), 128, 4096, 1000, 2});
  std::vector<muxsim::LLMSpec> ms;
  for (auto& s : rs) ms.push_back(mine_spec(s));
  const std::int64_t total = pick(50, 2000);
  muxref::BlockPool ref(total);
  muxsim::BlockPool mine(total);
  for (int i = 0; i < n; ++i) {
    ref.register_llm(i, &rs[i], 16);
    mine.register_llm(i, &ms[i], 16);
  }
  if (physical) mine.enable_physical();
  for (int i = 0; i < n; ++i) {
    std::int64_t q = pick(0, static_cast<int>(total));
    ref.set_quota(i, q);
    mine.set_quota(i, q);
  }
  std::vector<std::set<std::int64_t>> live(n);
  for (int op = 0; op < ops; ++op) {
    int llm = pick(0, n - 1);
    int kind = pick(0, 9);
    if (kind <= 3) {  // admit a fresh id
      std::int64_t id = pick(0, 1) ? pick(0, 500) : (std::int64_t(1) << 40) + pick(0, 50);
      if (live[llm].count(id)) continue;
      int prompt = pick(1, 64);
      int total_toks = prompt + pick(0, 64);
      auto a = ref.admit(llm, id, prompt, total_toks);
      auto b = mine.admit(llm, id, prompt, total_toks);
      EXPECT(a.ok == b.ok && err_code(a.error) == err_code(b.error), "admit op %d", op);
      if (a.ok) live[llm].insert(id);
    } else if (kind <= 6) {  // grow
      std::int64_t id;
      if (!live[llm].empty() && pick(0, 4)) {
        auto it = live[llm].begin();
        std::advance(it, pick(0, static_cast<int>(live[llm].size()) - 1));
        id = *it;
      } else {
        id = pick(600, 700);
      }
      int add = pick(0, 3) ? 1 : pick(0, 40);
      bool enforce = pick(0, 1);
      auto a = ref.alloc(llm, id, add, enforce);
      auto b = mine.alloc(llm, id, add, enforce);
      EXPECT(a.ok == b.ok && err_code(a.error) == err_code(b.error), "alloc op %d", op);
      if (a.ok) live[llm].insert(id);
    } else if (kind <= 8) {  // free
      if (live[llm].empty()) continue;
      auto it = live[llm].begin();
      std::advance(it, pick(0, static_cast<int>(live[llm].size()) - 1));
      ref.free_request(llm, *it);
      mine.free_request(llm, *it);
      live[llm].erase(it);
    } else {
      std::int64_t q = pick(0, static_cast<int>(total));
      ref.set_quota(llm, q);
      mine.set_quota(llm, q);
    }
    EXPECT(ref.free_blocks() == mine.free_blocks(), "free op %d", op);
    EXPECT(ref.committed_total() == mine.committed_total(), "committed_total op %d", op);
    for (int i = 0; i < n; ++i) {
      EXPECT(ref.used(i) == mine.used(i), "used llm %d op %d", i, op);
      EXPECT(ref.committed(i) == mine.committed(i), "committed llm %d op %d", i, op);
      EXPECT(ref.quota(i) == mine.quota(i), "quota llm %d op %d", i, op);
      for (std::int64_t id : live[i])
        EXPECT(ref.request_tokens(i, id) == mine.request_tokens(i, id), "tokens op %d", op);
    }
    mine.check_conservation();
    if (physical && (op % 97 == 0 || op == ops - 1)) {
      // Every live physical id is distinct and inside the pool.
      std::vector<char> seen(static_cast<size_t>(total), 0);
      std::int64_t count = 0;
      for (int i = 0; i < n; ++i)
        for (std::int64_t id : live[i])
          for (std::int32_t b : mine.block_table(i, id)) {
            EXPECT(b >= 0 && b < total, "id range");
            EXPECT(!seen[b], "duplicate physical id %d", b);
            seen[b] = 1;
            count += 1;
          }
      EXPECT(count == mine.total_used(), "physical count %lld vs used %lld", (long long)count,
             (long long)mine.total_used());
    }
  }
  // Unknown frees are logic errors on both sides.
  bool r_threw = false, m_threw = false;
  try { ref.free_request(0, 987654321); } catch (const std::logic_error&) { r_threw = true; }
  try { mine.free_request(0, 987654321); } catch (const std::logic_error&) { m_threw = true; }
  EXPECT(r_threw && m_threw, "unknown free");
  return 0;
}

// ------------------------------------------------------------------- sim fuzz
void compare_results(const muxref::SimResult& a, const muxsim::SimResult& b, const char* tag) {
  EXPECT(a.records.size() == b.records.size(), "%s record count", tag);
  for (size_t i = 0; i < std::min(a.records.size(), b.records.size()); ++i) {
    const auto& x = a.records[i];
    const auto& y = b.records[i];
    EXPECT(x.id == y.id && x.llm == y.llm && x.arrival_s == y.arrival_s &&
               x.first_token_s == y.first_token_s && x.done_s == y.done_s &&
               x.prompt_len == y.prompt_len && x.output_len == y.output_len,
           "%s record %zu (id %lld): first %.17g/%.17g done %.17g/%.17g", tag, i,
           (long long)x.id, x.first_token_s, y.first_token_s, x.done_s, y.done_s);
  }
  EXPECT(a.units.size() == b.units.size(), "%s unit count", tag);
  for (size_t u = 0; u < std::min(a.units.size(), b.units.size()); ++u) {
    const auto& x = a.units[u];
    const auto& y = b.units[u];
    EXPECT(x.unit == y.unit && x.total_blocks == y.total_blocks, "%s unit hdr", tag);
    EXPECT(x.samples.size() == y.samples.size(), "%s samples", tag);
    for (size_t k = 0; k < std::min(x.samples.size(), y.samples.size()); ++k)
      EXPECT(x.samples[k].t_s == y.samples[k].t_s && x.samples[k].llm == y.samples[k].llm &&
                 x.samples[k].used_blocks == y.samples[k].used_blocks &&
                 x.samples[k].quota_blocks == y.samples[k].quota_blocks,
             "%s sample %zu", tag, k);
    for (size_t k = 0; k < std::min(x.llms.size(), y.llms.size()); ++k)
      EXPECT(x.llms[k].avg_used_blocks == y.llms[k].avg_used_blocks &&
                 x.llms[k].final_quota_blocks == y.llms[k].final_quota_blocks &&
                 x.llms[k].resource_usage == y.llms[k].resource_usage,
             "%s llm stats %zu", tag, k);
  }
}

int fuzz_sim(std::uint64_t seed, int scenarios) {
  std::mt19937_64 rng(seed);
  auto pick = [&](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
  auto real = [&](double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(rng); };
  const std::int64_t kGiB = 1LL << 30;
  for (int sc = 0; sc < scenarios; ++sc) {
    int n = pick(1, 4);
    muxref::Cluster rc;
    rc.num_nodes = 1;
    rc.gpus_per_node = 2;
    rc.gpu_memory_bytes = static_cast<std::int64_t>(real(0.02, 2.0) * kGiB);
    std::vector<muxref::LlmEntry> re;
    muxref::WorkloadSpec ws;
    ws.horizon_s = real(2.0, 25.0);
    ws.seed = rng();
    for (int i = 0; i < n; ++i) {
      muxref::LLMSpec s{"m" + std::to_string(i), pick(1, 4), pick(1, 8), 128, 4096,
                        static_cast<std::int64_t>(pick(1, 20)) * 1000000, 2};
      double rate = real(0.5, 12.0);
      double mp = real(8.0, 300.0), mo = real(2.0, 200.0);
      re.push_back({s, rate, mp, mo});
      ws.llms.push_back({s.name, rate, muxref::LengthDist::lognormal(mp), muxref::LengthDist::lognormal(mo)});
    }
    std::vector<muxref::Request> rtrace = muxref::gen_workload(ws);
    muxref::PlacementResult rp;
    rp.backend = "greedy";
    muxref::LLMUnit unit;
    unit.mesh.node = 0;
    unit.mesh.gpu_ids = {0};
    int split = pick(0, 1) && n > 1 ? pick(1, n - 1) : n;  // optionally a second unit
    for (int i = 0; i < split; ++i) unit.llms.push_back({i, {1, 0.5, 8, 0.0, false}});
    rp.units.push_back(unit);
    muxref::LLMUnit unit2;
    unit2.mesh.node = 0;
    unit2.mesh.gpu_ids = {1};
    for (int i = split; i < n; ++i) unit2.llms.push_back({i, {1, 0.5, 8, 0.0, false}});
    rp.units.push_back(unit2);
    muxref::LatencyProfile rprof;
    rprof.decode_base_ms = real(2.0, 20.0);
    muxref::EngineParams rpar;
    rpar.kappa = real(0.0, 0.3);
    rpar.quota_period_s = real(0.5, 5.0);
    rpar.token_budget = pick(64, 4096);
    rpar.decode_sm = pick(0, 1) ? 0.5 : real(0.2, 0.7);
    rpar.prefill_min_sm = real(0.1, 0.4);
    rpar.warmup_s = real(0.0, 1.0);

    // mirror everything into the product's types
    muxsim::Cluster mc{rc.num_nodes, rc.gpus_per_node, rc.gpu_memory_bytes, rc.sms_per_gpu};
    std::vector<muxsim::LlmEntry> me;
    for (auto& e : re) me.push_back({mine_spec(e.spec), e.rate, e.mean_prompt_tokens, e.mean_output_tokens});
    muxsim::PlacementResult mp;
    mp.backend = rp.backend;
    for (auto& u : rp.units) {
      muxsim::LLMUnit mu;
      mu.mesh.node = u.mesh.node;
      mu.mesh.gpu_ids = u.mesh.gpu_ids;
      for (auto& pl : u.llms)
        mu.llms.push_back({pl.llm, {pl.candidate.tp_degree, pl.candidate.num_sm, pl.candidate.batch,
                                     pl.candidate.est_tpt, pl.candidate.saturated}});
      mp.units.push_back(mu);
    }
    std::vector<muxsim::Request> mtrace;
    for (auto& r : rtrace) mtrace.push_back({r.id, r.llm, r.arrival_s, r.prompt_len, r.output_len});
    muxsim::LatencyProfile mprof;
    mprof.decode_base_ms = rprof.decode_base_ms;

    for (int pol = 0; pol < 3; ++pol) {
      rpar.scheduler = static_cast<muxref::SchedKind>(pol);
      muxsim::EngineParams mpar;
      mpar.scheduler = static_cast<muxsim::SchedKind>(pol);
      mpar.kappa = rpar.kappa;
      mpar.quota_period_s = rpar.quota_period_s;
      mpar.token_budget = rpar.token_budget;
      mpar.decode_sm = rpar.decode_sm;
      mpar.prefill_min_sm = rpar.prefill_min_sm;
      mpar.warmup_s = rpar.warmup_s;
      std::string rerr, merr;
      muxref::SimResult a;
      muxsim::SimResult b;
      try { a = muxref::run_simulation(rc, rp, re, rtrace, rprof, rpar); } catch (const std::exception& e) { rerr = e.what(); }
      try { b = muxsim::run_simulation(mc, mp, me, mtrace, mprof, mpar); } catch (const std::exception& e) { merr = e.what(); }
      EXPECT(rerr == merr, "scenario %d policy %d: errors differ: '%s' vs '%s'", sc, pol, rerr.c_str(), merr.c_str());
      if (!rerr.empty()) g_errors += 1;
      if (rerr.empty()) {
        g_runs += 1;
        g_records += static_cast<long>(a.records.size());
        char tag[64];
        std::snprintf(tag, sizeof tag, "sc%d/pol%d", sc, pol);
        compare_results(a, b, tag);
      }
    }
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::string mode = argc > 1 ? argv[1] : "pool";
  std::uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
  int count = argc > 3 ? std::atoi(argv[3]) : 1000;
  if (mode == "pool") {
    for (int s = 0; s < 20; ++s) fuzz_pool(seed * 1000 + s, count, false);
  } else if (mode == "phys") {
    for (int s = 0; s < 20; ++s) fuzz_pool(seed * 1000 + s, count, true);
  } else if (mode == "sim") {
    fuzz_sim(seed, count);
  } else {
    std::fprintf(stderr, "usage: diff_fuzz pool|phys|sim seed count\n");
    return 2;
  }
  std::printf("diff_fuzz %s seed=%llu count=%d runs=%ld records=%ld both_threw=%ld mismatches=%d\n",
              mode.c_str(), (unsigned long long)seed, count, g_runs, g_records, g_errors, g_fail);
  return g_fail == 0 ? 0 : 1;
}
