// Golden-vector generator (TEST INFRASTRUCTURE): runs the UNMODIFIED reference
// (oracle/_ref/libmuxsim_core.a, /root/reference/proj/src) on the BASELINE
// config analogues of SURVEY.md Appendix B and writes trace + records + pool
// samples as JSON. Regenerate with tests/golden/make_golden.sh.
#include <cstdio>
#include <string>
#include <vector>

#include "muxsim/kv_manager.hpp"
#include "muxsim/placement.hpp"
#include "muxsim/sim_engine.hpp"
#include "muxsim/workload.hpp"

using namespace muxsim;

namespace {

constexpr std::int64_t kGiB = 1LL << 30;

struct Scenario {
  std::string name;
  int gpus;  // one mesh of this many gpus
  double mem_gib;
  std::vector<LlmEntry> entries;
  double horizon_s;
  std::uint64_t seed;
  bool constant_lengths = false;
  double quota_period_s = 10.0;
  double warmup_s = 0.0;
  std::int64_t token_budget = 4096;
};

LLMSpec named(std::string name, int L, int H, int hidden, double wbytes) {
  return {std::move(name), L, H, 128, hidden, static_cast<std::int64_t>(wbytes), 2};
}

void dump(FILE* f, const Scenario& sc, const std::vector<Request>& trace, const char* pol,
          const SimResult& res, bool first) {
  std::fprintf(f, "%s\"%s\": {\"records\": [", first ? "" : ", ", pol);
  for (size_t i = 0; i < res.records.size(); ++i) {
    const RequestRecord& r = res.records[i];
    std::fprintf(f, "%s[%lld, \"%s\", %.17g, %.17g, %.17g, %d, %d]", i ? ", " : "", (long long)r.id,
                 r.llm.c_str(), r.arrival_s, r.first_token_s, r.done_s, r.prompt_len, r.output_len);
  }
  std::fprintf(f, "], \"units\": [");
  for (size_t u = 0; u < res.units.size(); ++u) {
    const UnitStats& s = res.units[u];
    std::fprintf(f, "%s{\"unit\": %d, \"total_blocks\": %lld, \"llms\": [", u ? ", " : "", s.unit,
                 (long long)s.total_blocks);
    for (size_t k = 0; k < s.llms.size(); ++k)
      std::fprintf(f, "%s[\"%s\", %.17g, %lld, %.17g]", k ? ", " : "", s.llms[k].llm.c_str(),
                   s.llms[k].avg_used_blocks, (long long)s.llms[k].final_quota_blocks,
                   s.llms[k].resource_usage);
    std::fprintf(f, "], \"samples\": [");
    for (size_t k = 0; k < s.samples.size(); ++k)
      std::fprintf(f, "%s[%.17g, \"%s\", %lld, %lld]", k ? ", " : "", s.samples[k].t_s,
                   s.samples[k].llm.c_str(), (long long)s.samples[k].used_blocks,
                   (long long)s.samples[k].quota_blocks);
    std::fprintf(f, "]}");
  }
  std::fprintf(f, "]}");
  (void)sc;
  (void)trace;
}

void run(const Scenario& sc, const std::string& dir) {
  WorkloadSpec ws;
  ws.horizon_s = sc.horizon_s;
  ws.seed = sc.seed;
  for (const LlmEntry& e : sc.entries)
    ws.llms.push_back(
        {e.spec.name, e.rate,
         sc.constant_lengths ? LengthDist::constant(e.mean_prompt_tokens) : LengthDist::lognormal(e.mean_prompt_tokens),
         sc.constant_lengths ? LengthDist::constant(e.mean_output_tokens) : LengthDist::lognormal(e.mean_output_tokens)});
  std::vector<Request> trace = gen_workload(ws);
  Cluster c;
  c.num_nodes = 1;
  c.gpus_per_node = sc.gpus;
  c.gpu_memory_bytes = static_cast<std::int64_t>(sc.mem_gib * kGiB);
  PlacementResult p;
  p.backend = "greedy";
  LLMUnit u;
  u.mesh.node = 0;
  for (int g = 0; g < sc.gpus; ++g) u.mesh.gpu_ids.push_back(g);
  for (size_t i = 0; i < sc.entries.size(); ++i)
    u.llms.push_back({static_cast<int>(i), {sc.gpus, 0.5, 8, 0.0, false}});
  p.units.push_back(u);

  std::string path = dir + "/sim_" + sc.name + ".json";
  FILE* f = std::fopen(path.c_str(), "w");
  std::fprintf(f, "{\"name\": \"%s\", \"gpus\": %d, \"gpu_memory_bytes\": %lld, \"params\": "
               "{\"quota_period_s\": %.17g, \"warmup_s\": %.17g, \"token_budget\": %lld}, \"entries\": [",
               sc.name.c_str(), sc.gpus, (long long)c.gpu_memory_bytes, sc.quota_period_s, sc.warmup_s,
               (long long)sc.token_budget);
  for (size_t i = 0; i < sc.entries.size(); ++i) {
    const LlmEntry& e = sc.entries[i];
    std::fprintf(f, "%s[\"%s\", %d, %d, %d, %lld, %.17g, %.17g, %.17g]", i ? ", " : "",
                 e.spec.name.c_str(), e.spec.num_layers, e.spec.num_heads, e.spec.hidden_size,
                 (long long)e.spec.weight_bytes, e.rate, e.mean_prompt_tokens, e.mean_output_tokens);
  }
  std::fprintf(f, "], \"trace\": [");
  for (size_t i = 0; i < trace.size(); ++i)
    std::fprintf(f, "%s[%lld, \"%s\", %.17g, %d, %d]", i ? ", " : "", (long long)trace[i].id,
                 trace[i].llm.c_str(), trace[i].arrival_s, trace[i].prompt_len, trace[i].output_len);
  std::fprintf(f, "], \"results\": {");
  const char* names[3] = {"adbs", "fcfs", "rr"};
  for (int pol = 0; pol < 3; ++pol) {
    EngineParams ep;
    ep.scheduler = static_cast<SchedKind>(pol);
    ep.quota_period_s = sc.quota_period_s;
    ep.warmup_s = sc.warmup_s;
    ep.token_budget = sc.token_budget;
    SimResult res;
    try {
      res = run_simulation(c, p, sc.entries, trace, LatencyProfile{}, ep);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s/%s: %s\n", sc.name.c_str(), names[pol], e.what());
      throw;
    }
    dump(f, sc, trace, names[pol], res, pol == 0);
  }
  std::fprintf(f, "}}\n");
  std::fclose(f);
  std::printf("%s: %zu requests\n", path.c_str(), trace.size());
}

}  // namespace

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";
  LLMSpec tiny_a = named("tiny-a", 2, 4, 512, 8e6), tiny_b = named("tiny-b", 4, 2, 256, 4e6);
  LLMSpec m7 = named("7b", 32, 32, 4096, 13.5e9), m13 = named("13b", 40, 40, 5120, 26e9);
  // cfg1: 2 tiny models on one 1 GiB GPU, rates 8/2, ShareGPT-shaped lengths.
  run({"cfg1_tiny", 1, 1.0, {{tiny_a, 8.0, 161.0, 338.0}, {tiny_b, 2.0, 161.0, 338.0}}, 60.0, 11}, dir);
  // cfg2: 7B@4 + 13B@2 on one 180 GiB B200.
  run({"cfg2_7b13b", 1, 180.0, {{m7, 4.0, 161.0, 338.0}, {m13, 2.0, 161.0, 338.0}}, 120.0, 1}, dir);
  // cfg3: 7B/7B/13B/13B on a tp=2 mesh, rates 4/2/2/1.
  LLMSpec a7 = m7, b7 = m7, c13 = m13, d13 = m13;
  a7.name = "a7"; b7.name = "b7"; c13.name = "c13"; d13.name = "d13";
  run({"cfg3_tp2", 2, 180.0, {{a7, 4.0, 161.0, 338.0}, {b7, 2.0, 161.0, 338.0}, {c13, 2.0, 161.0, 338.0},
                              {d13, 1.0, 161.0, 338.0}}, 60.0, 2}, dir);
  // Acceptance C1's contention scenario (acceptance.cpp:100-133), 15 s horizon.
  LLMSpec x7 = m7, y7 = m7;
  x7.name = "llm-long"; y7.name = "llm-short";
  Scenario c1{"contention_c1", 4, 7.5, {{x7, 10.0, 128.0, 384.0}, {y7, 80.0, 64.0, 64.0}}, 15.0, 42};
  c1.constant_lengths = true;
  c1.quota_period_s = 1.0;
  c1.warmup_s = 8.0;
  c1.token_budget = 768;
  run(c1, dir);
  return 0;
}
