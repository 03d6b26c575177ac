// Planner-side candidate generation for realizable plans.
//
// The reference's llm_parallel_candidates (/root/reference/proj/src/
// placement.cpp:57-103) offers every tp width in tp_list whose mesh holds the
// weights. The B200 engine shards each model Megatron-style by head
// (DESIGN §7), so a width that does not divide num_heads (30B's 52 heads at
// tp 8) cannot run; the reference planner would still propose it (SURVEY §0
// fact 2). This restates the candidate search with that filter and with the
// profile's measured tensor-parallel cost (LatencyProfile::tp_scaled). Named
// apart from the reference's symbol so the drop-in build (the reference
// planner linked against this library) keeps its own.
#pragma once

#include <vector>

#include "mux/topology.hpp"

namespace muxsim {

struct CandidateParams {
  std::vector<double> sm_list;  // empty -> {0.1, ..., 1.0} (placement.cpp:23-28)
  std::vector<int> tp_list = {1, 2, 4, 8};
  double activation_reserve_frac = 0.1;
  int max_batch = 256;
};

// A tp width the engine can shard the model over: a valid mesh width that
// divides the head count (and the FFN width when known, ffn <= 0 = unknown).
bool tp_realizable(const LLMSpec& spec, int tp_degree, int ffn = 0);

// Per-model candidates, one per realizable tp width (placement.cpp:57-103
// plus the tp_realizable filter). Throws InfeasibleError naming the model
// when no width both fits and shards.
std::vector<std::vector<ParallelCandidate>> realizable_parallel_candidates(
    const std::vector<LlmEntry>& llms, const Cluster& cluster, const LatencyProfile& prof,
    const CandidateParams& params, const std::vector<int>& ffn = {});

}  // namespace muxsim
