// Golden-vector generator (TEST INFRASTRUCTURE): the UNMODIFIED reference's
// llm_parallel_candidates (oracle/_ref/libmuxsim_core.a, placement.cpp:57-103)
// over catalog models x rates x clusters x profiles; the product's
// realizable_parallel_candidates must equal it minus the tp widths that do not
// divide num_heads (tests/test_control_plane.py). Regenerate with
// tests/golden/make_golden.sh.
#include <cstdio>
#include <string>
#include <vector>

#include "muxsim/placement.hpp"

using namespace muxsim;

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";
  FILE* f = std::fopen((dir + "/candidates.json").c_str(), "w");
  const LLMSpec models[] = {{"7b", 32, 32, 128, 4096, static_cast<std::int64_t>(13.5e9), 2},
                            {"13b", 40, 40, 128, 5120, static_cast<std::int64_t>(26e9), 2},
                            {"30b", 60, 52, 128, 6656, static_cast<std::int64_t>(65e9), 2},
                            {"65b", 80, 64, 128, 8192, static_cast<std::int64_t>(130e9), 2}};
  const double rates[] = {0.0, 0.5, 4.0, 40.0};
  const double mem_gib[] = {80.0, 180.0};
  const int gpus[] = {2, 8};
  // default profile, and the B200-measured one (profiles/r01_b200_profile_7b.json, rounded)
  LatencyProfile p0;
  LatencyProfile p1{0.01292, 3.6653, 0.00056571, 0.9, 0.405405, 90.51, 131072.0};
  const LatencyProfile* profs[] = {&p0, &p1};
  std::fprintf(f, "{\"cases\": [");
  bool first = true;
  for (int pi = 0; pi < 2; ++pi)
    for (double mem : mem_gib)
      for (int g : gpus)
        for (double rate : rates) {
          std::vector<LlmEntry> llms;
          for (const LLMSpec& m : models) llms.push_back({m, rate, 161.0, 338.0});
          Cluster cl{1, g, static_cast<std::int64_t>(mem * (1LL << 30)), 1.0};
          PlacementParams pp;
          std::fprintf(f, "%s{\"profile\": %d, \"mem_gib\": %.17g, \"gpus\": %d, \"rate\": %.17g, ", first ? "" : ", ",
                       pi, mem, g, rate);
          first = false;
          try {
            auto c = llm_parallel_candidates(llms, cl, *profs[pi], pp);
            std::fprintf(f, "\"candidates\": [");
            for (size_t i = 0; i < c.size(); ++i) {
              std::fprintf(f, "%s[", i ? ", " : "");
              for (size_t k = 0; k < c[i].size(); ++k)
                std::fprintf(f, "%s[%d, %.17g, %d, %.17g, %d]", k ? ", " : "", c[i][k].tp_degree, c[i][k].num_sm,
                             c[i][k].batch, c[i][k].est_tpt, c[i][k].saturated ? 1 : 0);
              std::fprintf(f, "]");
            }
            std::fprintf(f, "]}");
          } catch (const std::exception& e) {
            std::fprintf(f, "\"error\": \"%s\"}", e.what());
          }
        }
  std::fprintf(f, "]}\n");
  std::fclose(f);
  return 0;
}
