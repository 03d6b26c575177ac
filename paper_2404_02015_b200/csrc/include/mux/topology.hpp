// Placement and trace types the engine consumes.
//
// These are the boundary inputs of the hot path: the
// planner's output (/root/reference/proj/include/muxsim/placement.hpp:21-75)
// and one trace row (/root/reference/proj/include/muxsim/workload.hpp:68-74).
// When this library is linked *into* the reference's own planner/CLI (the
// drop-in build, tests/native/Makefile), MUX_USE_REFERENCE_TOPOLOGY pulls the
// reference's definitions instead so both sides share one set of types.
#pragma once

#ifdef MUX_USE_REFERENCE_TOPOLOGY
#include "muxsim/placement.hpp"
#include "muxsim/workload.hpp"
#else

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mux/spec.hpp"

namespace muxsim {

class InfeasibleError : public std::runtime_error {
 public:
  explicit InfeasibleError(const std::string& what) : std::runtime_error(what) {}
};

struct Cluster {
  int num_nodes = 1;
  int gpus_per_node = 1;
  std::int64_t gpu_memory_bytes = 0;
  double sms_per_gpu = 1.0;
  void validate() const;
};

struct Mesh {
  int node = 0;
  std::vector<int> gpu_ids;
  int size() const { return static_cast<int>(gpu_ids.size()); }
};

struct MeshGroup {
  std::vector<Mesh> meshes;
};

struct LlmEntry {
  LLMSpec spec;
  double rate = 0.0;
  double mean_prompt_tokens = 1.0;
  double mean_output_tokens = 1.0;
};

struct ParallelCandidate {
  int tp_degree = 1;
  double num_sm = 1.0;
  int batch = 1;
  double est_tpt = 0.0;
  bool saturated = false;
};

struct PlacedLlm {
  int llm = -1;
  ParallelCandidate candidate;
};

struct LLMUnit {
  Mesh mesh;
  std::vector<PlacedLlm> llms;
};

struct PlacementResult {
  std::string backend;
  std::vector<LLMUnit> units;
  double est_total_tpt = 0.0;
  double objective = 0.0;
};

struct Request {
  std::int64_t id = 0;
  std::string llm;
  double arrival_s = 0.0;
  int prompt_len = 1;
  int output_len = 1;
};

}  // namespace muxsim

#endif  // MUX_USE_REFERENCE_TOPOLOGY
