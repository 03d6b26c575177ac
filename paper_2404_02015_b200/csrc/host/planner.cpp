// Realizable parallel candidates: the reference's per-model
// candidate search (placement.cpp:57-103) with the head-divisibility filter
// the B200 engine's tensor parallelism needs and the profile's tp cost.
#include "mux/planner.hpp"

#include <algorithm>
#include <cmath>

namespace muxsim {

namespace {

std::vector<double> sm_shares(const CandidateParams& p) {
  if (!p.sm_list.empty()) return p.sm_list;
  std::vector<double> out;
  for (int i = 1; i <= 10; ++i) out.push_back(i / 10.0);
  return out;
}

}  // namespace

bool tp_realizable(const LLMSpec& spec, int tp_degree, int ffn) {
  if (tp_degree != 1 && tp_degree != 2 && tp_degree != 4 && tp_degree != 8) return false;
  if (spec.num_heads % tp_degree != 0) return false;
  return ffn <= 0 || ffn % tp_degree == 0;
}

std::vector<std::vector<ParallelCandidate>> realizable_parallel_candidates(
    const std::vector<LlmEntry>& llms, const Cluster& cluster, const LatencyProfile& prof,
    const CandidateParams& params, const std::vector<int>& ffn) {
  cluster.validate();
  prof.validate();
  if (!ffn.empty() && ffn.size() != llms.size())
    throw std::invalid_argument("parallel candidates: ffn needs one width per model");
  const std::vector<double> shares = sm_shares(params);
  const double usable = 1.0 - params.activation_reserve_frac;
  std::vector<std::vector<ParallelCandidate>> out(llms.size());
  for (size_t i = 0; i < llms.size(); ++i) {
    const LlmEntry& e = llms[i];
    e.spec.validate();
    const double req_kv = e.spec.kv_bytes_per_token() * (e.mean_prompt_tokens + e.mean_output_tokens);
    for (int tp : params.tp_list) {
      if (tp > cluster.gpus_per_node) continue;  // node-local meshes
      if (!tp_realizable(e.spec, tp, ffn.empty() ? 0 : ffn[i])) continue;
      double kv = usable * tp * static_cast<double>(cluster.gpu_memory_bytes) -
                  static_cast<double>(e.spec.weight_bytes);
      if (kv <= 0.0) continue;
      int max_batch = static_cast<int>(std::clamp<double>(std::floor(kv / req_kv), 1.0, params.max_batch));
      if (e.rate <= 0.0) {
        out[i].push_back({tp, shares.front(), 1, 0.0, false});
        continue;
      }
      // smallest SM share whose stable batch keeps up with the rate
      ThroughputEstimate est{};
      bool met = false;
      for (double sm : shares) {
        est = estimate_throughput(e.spec, prof, sm, tp, e.rate, {}, e.mean_prompt_tokens,
                                  e.mean_output_tokens, max_batch);
        if (!est.saturated) {
          out[i].push_back({tp, sm, est.batch, est.throughput, false});
          met = true;
          break;
        }
      }
      if (!met) out[i].push_back({tp, shares.back(), est.batch, est.throughput, true});
    }
    if (out[i].empty())
      throw InfeasibleError("llm '" + e.spec.name + "' does not fit any mesh at any realizable tensor-parallel width");
  }
  return out;
}

}  // namespace muxsim
