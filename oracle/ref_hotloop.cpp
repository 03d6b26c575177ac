// Reference CPU hot-loop timing (TEST/BENCH INFRASTRUCTURE): the unmodified
// reference engine (oracle/_ref/libmuxsim_core.a) on the config-2 analogue at
// saturating rates (SURVEY.md Appendix B "Hot-loop timing": 7B@20 + 13B@10 rps,
// 600 s). Prints simulated decode-token decisions per wall-second on 1 core.
#include <chrono>
#include <cstdio>

#include "muxsim/placement.hpp"
#include "muxsim/sim_engine.hpp"
#include "muxsim/workload.hpp"

using namespace muxsim;

int main(int argc, char** argv) {
  double horizon = argc > 1 ? std::atof(argv[1]) : 600.0;
  LLMSpec m7{"7b", 32, 32, 128, 4096, static_cast<std::int64_t>(13.5e9), 2};
  LLMSpec m13{"13b", 40, 40, 128, 5120, static_cast<std::int64_t>(26e9), 2};
  std::vector<LlmEntry> entries = {{m7, 20.0, 161.0, 338.0}, {m13, 10.0, 161.0, 338.0}};
  WorkloadSpec ws;
  ws.horizon_s = horizon;
  ws.seed = 1;
  for (auto& e : entries)
    ws.llms.push_back({e.spec.name, e.rate, LengthDist::lognormal(161.0), LengthDist::lognormal(338.0)});
  std::vector<Request> trace = gen_workload(ws);
  Cluster c;
  c.gpus_per_node = 1;
  c.gpu_memory_bytes = 180LL << 30;
  PlacementResult p;
  LLMUnit u;
  u.mesh.gpu_ids = {0};
  u.llms = {{0, {1, 0.5, 8, 0.0, false}}, {1, {1, 0.5, 8, 0.0, false}}};
  p.units.push_back(u);
  auto t0 = std::chrono::steady_clock::now();
  SimResult r = run_simulation(c, p, entries, trace, LatencyProfile{}, EngineParams{});
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  long long decode_tokens = 0;
  for (const RequestRecord& rec : r.records) decode_tokens += rec.output_len - 1;
  std::printf("{\"requests\": %zu, \"decode_tokens\": %lld, \"wall_s\": %.6f, \"decisions_per_s\": %.1f}\n",
              r.records.size(), decode_tokens, s, decode_tokens / s);
  return 0;
}
