// ADBS scheduling pass and the FCFS / round-robin baselines.
//
// Decision semantics follow /root/reference/proj/src/scheduler.cpp:40-259
// exactly (they are the parity target: JobPlans must be bit-identical), the
// code is this repo's own. One pass = prefill phase (prefill priority, SM
// share gate, FIFO admission under the token budget with head-of-line
// blocking on memory) then one decode round per model while SM shares last.
#include "mux/adbs.hpp"

#include <algorithm>
#include <limits>
#include <stdexcept>

namespace muxsim {

namespace {

constexpr std::int64_t kUnbounded = std::numeric_limits<std::int64_t>::max();

// What a policy lets the shared pass do this time.
struct PassPolicy {
  std::vector<int> prefill_order;  // models allowed to prefill, in priority order
  std::vector<int> decode_order;   // models allowed a decode round, in order
  std::int64_t admit_below = kUnbounded;
};

bool decode_work_ready(const UnitState& s, const std::vector<int>& order) {
  return std::any_of(order.begin(), order.end(), [&](int li) {
    return !s.llms[li].decoding.empty() && !s.llms[li].decode_running;
  });
}

// Admit as many waiting requests of model `li` as the token budget, the
// admission bound and the pool allow. Stops at the first memory refusal.
void fill_prefill(UnitState& s, const SchedulerParams& p, const PassPolicy& pol, int li,
                  JobPlan& plan) {
  LlmQueues& q = s.llms[li];
  while (!q.waiting.empty()) {
    const int rid = q.waiting.front();
    const UnitRequest& r = s.requests[rid];
    if (r.global_id >= pol.admit_below) return;
    if (!plan.members.empty() && plan.prompt_tokens + r.prompt_len > p.token_budget) return;
    // Reserve the final footprint (prompt + every generated token but the last).
    if (!s.pool->admit(li, rid, r.prompt_len, r.prompt_len + r.output_len - 1).ok) return;
    plan.members.push_back(rid);
    plan.prompt_tokens += r.prompt_len;
    q.waiting.pop_front();
  }
}

bool try_prefill_phase(UnitState& s, const SchedulerParams& p, const PassPolicy& pol,
                       std::vector<JobPlan>& out) {
  const int n = static_cast<int>(s.llms.size());
  double share = decode_work_ready(s, pol.decode_order) ? std::min(s.free_sm, 1.0 - p.decode_sm)
                                                        : s.free_sm;
  share = std::max(p.prefill_min_sm, share);
  const bool fits = share <= s.free_sm + p.eps;
  bool candidate = false;
  for (int li : pol.prefill_order) {
    LlmQueues& q = s.llms[li];
    if (q.waiting.empty() || s.requests[q.waiting.front()].global_id >= pol.admit_below) continue;
    candidate = true;
    if (!fits) break;  // an SM shortage blocks every model alike
    JobPlan plan;
    plan.llm = li;
    plan.kind = JobKind::Prefill;
    plan.sm_demand = share;
    fill_prefill(s, p, pol, li, plan);
    if (plan.members.empty()) continue;  // memory-blocked: next model's turn
    q.prefill_running = true;
    s.running_prefills += 1;
    s.running_jobs += 1;
    s.free_sm -= share;
    s.prefill_cursor = (li + 1) % n;
    out.push_back(std::move(plan));
    s.prefill_waiting = false;
    return true;
  }
  s.prefill_waiting = candidate;
  return false;
}

void decode_phase(UnitState& s, const SchedulerParams& p, const PassPolicy& pol,
                  std::vector<JobPlan>& out) {
  const int n = static_cast<int>(s.llms.size());
  for (int li : pol.decode_order) {
    LlmQueues& q = s.llms[li];
    if (q.decoding.empty() || q.decode_running) continue;
    if (p.decode_sm > s.free_sm + p.eps) continue;
    JobPlan plan;
    plan.llm = li;
    plan.kind = JobKind::Decode;
    plan.sm_demand = p.decode_sm;
    double ctx = 0.0;
    for (int rid : q.decoding) {
      // One more token of cache per step; a full pool skips the member.
      if (!s.pool->alloc(li, rid, 1, false).ok) continue;
      const UnitRequest& r = s.requests[rid];
      plan.members.push_back(rid);
      ctx += r.prompt_len + 1 + r.steps_done;
    }
    if (plan.members.empty()) continue;
    plan.avg_context = ctx / static_cast<double>(plan.members.size());
    q.decode_running = true;
    s.running_jobs += 1;
    s.free_sm -= p.decode_sm;
    s.decode_cursor = (li + 1) % n;
    out.push_back(std::move(plan));
  }
}

std::vector<JobPlan> run_pass(UnitState& s, const SchedulerParams& p, const PassPolicy& pol) {
  std::vector<JobPlan> out;
  bool launched = false;
  if (s.running_prefills == 0) launched = try_prefill_phase(s, p, pol, out);
  // A blocked prefill holds decodes back, except on a fully idle unit where
  // only decode completions can free what it waits for.
  const bool idle_escape = s.prefill_waiting && s.running_jobs == 0 && !launched;
  if (!s.prefill_waiting || idle_escape) decode_phase(s, p, pol, out);
  return out;
}

std::vector<int> rotation(int n, int start) {
  std::vector<int> v(n);
  for (int k = 0; k < n; ++k) v[k] = (start + k) % n;
  return v;
}

std::vector<JobPlan> adbs(UnitState& s, const SchedulerParams& p) {
  const int n = static_cast<int>(s.llms.size());
  PassPolicy pol;
  pol.prefill_order = rotation(n, s.prefill_cursor);
  pol.decode_order = rotation(n, s.decode_cursor);
  return run_pass(s, p, pol);
}

int busy_model(const UnitState& s) {
  for (size_t i = 0; i < s.llms.size(); ++i)
    if (s.llms[i].prefill_running || s.llms[i].decode_running) return static_cast<int>(i);
  return -1;
}

int earliest_waiting_model(const UnitState& s) {
  int who = -1;
  std::int64_t best = kUnbounded;
  for (size_t i = 0; i < s.llms.size(); ++i) {
    if (s.llms[i].waiting.empty()) continue;
    std::int64_t gid = s.requests[s.llms[i].waiting.front()].global_id;
    if (gid < best) {
      best = gid;
      who = static_cast<int>(i);
    }
  }
  return who;
}

int earliest_outstanding_model(UnitState& s) {
  int who = -1;
  std::int64_t best = kUnbounded;
  for (size_t i = 0; i < s.llms.size(); ++i) {
    std::deque<int>& act = s.llms[i].active;
    while (!act.empty() && s.requests[act.front()].finished) act.pop_front();
    if (act.empty()) continue;
    std::int64_t gid = s.requests[act.front()].global_id;
    if (gid < best) {
      best = gid;
      who = static_cast<int>(i);
    }
  }
  return who;
}

// FCFS: temporal sharing, the owner of the oldest outstanding request holds
// the mesh; it may prefill only when it also owns the oldest waiting request.
std::vector<JobPlan> fcfs(UnitState& s, const SchedulerParams& p) {
  int owner = busy_model(s);
  if (owner < 0) owner = earliest_outstanding_model(s);
  if (owner < 0) return {};
  PassPolicy pol;
  if (earliest_waiting_model(s) == owner) pol.prefill_order.push_back(owner);
  pol.decode_order.push_back(owner);
  return run_pass(s, p, pol);
}

// Round-robin: whole-mesh turns; a turn is a prefill batch (with the owner's
// own decodes under it) or, with nothing to prefill, one decode round.
std::vector<JobPlan> round_robin(UnitState& s, const SchedulerParams& p) {
  const int n = static_cast<int>(s.llms.size());
  auto has_work = [&](int li) { return !s.llms[li].waiting.empty() || !s.llms[li].decoding.empty(); };
  auto next_owner = [&](int from) {
    for (int k = 1; k <= n; ++k)
      if (has_work((from + k) % n)) return (from + k) % n;
    return from;
  };

  if (s.rr_turn_open) {
    bool over = s.rr_turn_had_prefill ? s.running_prefills == 0 : s.running_jobs == 0;
    if (over) {
      s.rr_owner = next_owner(s.rr_owner);
      s.rr_turn_open = false;
      s.rr_turn_had_prefill = false;
    }
  }
  if (!s.rr_turn_open && !has_work(s.rr_owner)) s.rr_owner = next_owner(s.rr_owner);

  for (int i = 0; i < n; ++i) {
    if (i == s.rr_owner) continue;
    if (s.llms[i].prefill_running || s.llms[i].decode_running) return {};
  }

  for (int attempt = 0; attempt < n; ++attempt) {
    PassPolicy pol;
    pol.prefill_order = {s.rr_owner};
    pol.decode_order = {s.rr_owner};
    std::vector<JobPlan> out = run_pass(s, p, pol);
    for (const JobPlan& plan : out) {
      s.rr_turn_open = true;
      if (plan.kind == JobKind::Prefill) s.rr_turn_had_prefill = true;
    }
    if (!out.empty()) return out;
    if (s.running_jobs != 0) break;
    int next = next_owner(s.rr_owner);
    if (next == s.rr_owner) break;
    s.rr_owner = next;  // an owner stuck on an idle mesh yields its turn
  }
  return {};
}

}  // namespace

std::vector<JobPlan> schedule(SchedKind kind, UnitState& state, const SchedulerParams& params) {
  if (state.pool == nullptr) throw std::logic_error("scheduler: unit state has no block pool");
  switch (kind) {
    case SchedKind::Adbs: return adbs(state, params);
    case SchedKind::Fcfs: return fcfs(state, params);
    case SchedKind::RoundRobin: return round_robin(state, params);
  }
  throw std::logic_error("scheduler: unknown policy");
}

}  // namespace muxsim
