"""Host-side mirror of the reference hot-path API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/muxsim/kv_manager.hpp, scheduler.hpp,
sim_engine.hpp); everything executes in libmux.so. The device unit
(:class:`Unit`) is the B200 extension: the KV pool in HBM, colocated LLaMA
models and the prefill/decode jobs that ``UnitSim::launch``
(/root/reference/proj/src/sim_engine.cpp:308-330) only priced.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from ._lib import (ALLOC_OK, ALLOC_POOL, ALLOC_QUOTA, LlmEntry as _CEntry, PlacedLlm, Record,
                   Request as _CRequest, SimConfig, UnitConfig, check, lib)
from ._lib import Candidate as _Candidate, RouteRecord as _RouteRecord
from ._lib import PoolSample as _PoolSample, UnitLlmStats as _UnitLlmStats, UnitStats as _UnitStats

# ----------------------------------------------------------------- model specs


@dataclass(frozen=True)
class LLMSpec:
    """cost_model.hpp:11-21 plus the FFN width / vocabulary a real forward needs
    (the reference catalog has neither)."""
    name: str
    num_layers: int
    num_heads: int
    head_dim: int = 128
    hidden_size: int = 0
    weight_bytes: int = 1
    bytes_per_element: int = 2
    ffn: int = 0
    vocab: int = 32000

    def kv_bytes_per_token(self) -> float:
        return 2.0 * self.num_layers * self.num_heads * self.head_dim * self.bytes_per_element


# Reference catalog (config.cpp:12-22) extended with LLaMA-1 FFN sizes and vocab.
CATALOG = {
    "7b": LLMSpec("7b", 32, 32, 128, 4096, int(13.5e9), 2, 11008, 32000),
    "13b": LLMSpec("13b", 40, 40, 128, 5120, int(26e9), 2, 13824, 32000),
    "30b": LLMSpec("30b", 60, 52, 128, 6656, int(65e9), 2, 17920, 32000),
    "65b": LLMSpec("65b", 80, 64, 128, 8192, int(130e9), 2, 22016, 32000),
    # BASELINE config 1 (SURVEY.md Appendix B "Tiny"), head_dim 128 so that
    # block bytes agree with the big models (sim_engine.cpp:180-184).
    "tiny-a": LLMSpec("tiny-a", 2, 4, 128, 512, 8_000_000, 2, 1024, 512),
    "tiny-b": LLMSpec("tiny-b", 4, 2, 128, 256, 4_000_000, 2, 512, 512),
}


def spec(name: str, alias: str | None = None) -> LLMSpec:
    s = CATALOG[name]
    if alias:
        s = LLMSpec(alias, *[getattr(s, f) for f in
                             ("num_layers", "num_heads", "head_dim", "hidden_size", "weight_bytes",
                              "bytes_per_element", "ffn", "vocab")])
    return s


def _c_entry(s: LLMSpec, rate=0.0, mean_prompt=1.0, mean_output=1.0, keep=None) -> _CEntry:
    name = s.name.encode()
    if keep is not None:
        keep.append(name)
    return _CEntry(name, s.num_layers, s.num_heads, s.head_dim, s.hidden_size, s.weight_bytes,
                   s.bytes_per_element, rate, mean_prompt, mean_output, s.ffn, s.vocab)


# -------------------------------------------------------------- geometry/quota

def blocks_for_tokens(s: LLMSpec, block_tokens: int, tokens: int) -> int:
    out = C.c_int64()
    check(lib.mux_blocks_for_tokens(s.num_layers, s.num_heads, block_tokens, tokens, C.byref(out)))
    return out.value


def blocks_per_token(s: LLMSpec, block_tokens: int) -> float:
    return 2.0 * s.num_layers * s.num_heads / block_tokens


@dataclass
class QuotaInput:
    rate: float = 0.0
    blocks_per_token: float = 0.0
    mean_request_tokens: float = 0.0


def init_token_block_quota(llms: Sequence[QuotaInput], kv_blocks: int, floor_frac: float = 0.02):
    n = len(llms)
    arr = C.c_double * max(n, 1)
    out = (C.c_int64 * max(n, 1))()
    check(lib.mux_init_token_block_quota(n, arr(*[q.rate for q in llms]),
                                         arr(*[q.blocks_per_token for q in llms]),
                                         arr(*[q.mean_request_tokens for q in llms]),
                                         kv_blocks, floor_frac, out))
    return list(out[:n])


def adapt_quota(utilizations: Sequence[float], quotas: Sequence[int], floor_blocks: int,
                low_mark=0.5, high_mark=0.9, step_frac=0.1):
    n = len(quotas)
    out = (C.c_int64 * max(n, 1))()
    check(lib.mux_adapt_quota(n, (C.c_double * max(n, 1))(*utilizations),
                              (C.c_int64 * max(n, 1))(*quotas), floor_blocks, low_mark, high_mark,
                              step_frac, out))
    return list(out[:n])


# ------------------------------------------------------------------- BlockPool

@dataclass
class AllocResult:
    ok: bool
    error: str  # "none" | "pool" | "quota"


_ERR = {ALLOC_OK: "none", ALLOC_POOL: "pool", ALLOC_QUOTA: "quota"}


class BlockPool:
    """kv_manager.hpp:48-105 over the C ABI, with physical head-block ids."""

    def __init__(self, total_blocks: int, physical: bool = True, _handle=None, shards: int = 1):
        """shards > 1: physical ids sharded head-wise over that many TP ranks."""
        self._owned = _handle is None
        if _handle is None:
            h = C.c_void_p()
            check(lib.mux_pool_create(total_blocks, (shards if shards > 1 else 1) if physical else 0, C.byref(h)))
            _handle = h.value
        self._h = _handle

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            lib.mux_pool_destroy(self._h)
            self._h = None

    def register_llm(self, llm: int, s: LLMSpec, block_tokens: int = 16):
        check(lib.mux_pool_register_llm(self._h, llm, s.num_layers, s.num_heads, s.head_dim,
                                        s.bytes_per_element, block_tokens))

    def admit(self, llm, request_id, prompt_tokens, total_tokens) -> AllocResult:
        r = C.c_int()
        check(lib.mux_pool_admit(self._h, llm, request_id, prompt_tokens, total_tokens, C.byref(r)))
        return AllocResult(r.value == ALLOC_OK, _ERR[r.value])

    def alloc(self, llm, request_id, add_tokens, enforce_quota) -> AllocResult:
        r = C.c_int()
        check(lib.mux_pool_alloc(self._h, llm, request_id, add_tokens, 1 if enforce_quota else 0,
                                 C.byref(r)))
        return AllocResult(r.value == ALLOC_OK, _ERR[r.value])

    def alloc_n(self, llm, request_ids, add_tokens, enforce_quota) -> list[AllocResult]:
        """alloc() for every member of a decode round in one C call;
        request_ids: a sequence of ints or a ctypes int64 array."""
        ids = request_ids if isinstance(request_ids, C.Array) else (C.c_int64 * len(request_ids))(*request_ids)
        n = len(ids)
        res = (C.c_int * max(n, 1))()
        check(lib.mux_pool_alloc_n(self._h, llm, n, ids, add_tokens, 1 if enforce_quota else 0, res))
        return [AllocResult(r == ALLOC_OK, _ERR[r]) for r in res[:n]]

    def alloc_n_ok(self, llm, request_ids, add_tokens, enforce_quota) -> bool:
        """alloc_n() reporting only whether every member's allocation
        succeeded (the decode round's hot path: no per-member result objects)."""
        ids = request_ids if isinstance(request_ids, C.Array) else (C.c_int64 * len(request_ids))(*request_ids)
        n = len(ids)
        res = (C.c_int * max(n, 1))()
        check(lib.mux_pool_alloc_n(self._h, llm, n, ids, add_tokens, 1 if enforce_quota else 0, res))
        return not any(res[:n])

    def free_request(self, llm, request_id):
        check(lib.mux_pool_free_request(self._h, llm, request_id))

    def set_quota(self, llm, blocks):
        check(lib.mux_pool_set_quota(self._h, llm, blocks))

    def _stats(self, llm):
        q, u, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.mux_pool_llm_stats(self._h, llm, C.byref(q), C.byref(u), C.byref(c)))
        return q.value, u.value, c.value

    def quota(self, llm):
        return self._stats(llm)[0]

    def used(self, llm):
        return self._stats(llm)[1]

    def committed(self, llm):
        return self._stats(llm)[2]

    def request_tokens(self, llm, request_id):
        t = C.c_int64()
        check(lib.mux_pool_request_tokens(self._h, llm, request_id, C.byref(t)))
        return t.value

    def _totals(self):
        f, t, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.mux_pool_totals(self._h, C.byref(f), C.byref(t), C.byref(c)))
        return f.value, t.value, c.value

    def free_blocks(self):
        return self._totals()[0]

    def total_blocks(self):
        return self._totals()[1]

    def committed_total(self):
        return self._totals()[2]

    def total_used(self):
        f, t, _ = self._totals()
        return t - f

    def check_conservation(self):
        check(lib.mux_pool_check(self._h))

    def block_table(self, llm, request_id) -> list[int]:
        n = C.c_int64()
        check(lib.mux_pool_block_table(self._h, llm, request_id, None, 0, C.byref(n)))
        buf = (C.c_int32 * max(n.value, 1))()
        check(lib.mux_pool_block_table(self._h, llm, request_id, buf, n.value, C.byref(n)))
        return list(buf[:n.value])

    def slot(self, llm, request_id) -> int:
        s = C.c_int()
        check(lib.mux_pool_slot(self._h, llm, request_id, C.byref(s)))
        return s.value


# ------------------------------------------------------------------ simulate

@dataclass
class TraceRequest:
    id: int
    llm: int            # index into the entries
    arrival_s: float
    prompt_len: int
    output_len: int


@dataclass
class EngineParams:
    """sim_engine.hpp:15-28 defaults."""
    scheduler: int = 0  # 0 ADBS, 1 FCFS, 2 round-robin
    kappa: float = 0.1
    quota_period_s: float = 10.0
    token_budget: int = 4096
    block_tokens: int = 16
    warmup_s: float = 0.0
    decode_sm: float = 0.5
    prefill_min_sm: float = 0.3
    activation_reserve_frac: float = 0.1
    quota_floor_frac: float = 0.02
    # QuotaAdaptParams (kv_manager.hpp; config sim.quota_low_mark /
    # quota_high_mark / quota_step_frac, config.cpp:242-244)
    quota_low_mark: float = 0.5
    quota_high_mark: float = 0.9
    quota_step_frac: float = 0.1


@dataclass
class Entry:
    spec: LLMSpec
    rate: float = 0.0
    mean_prompt_tokens: float = 1.0
    mean_output_tokens: float = 1.0


@dataclass
class Placement:
    """Units (mesh sizes) and which entries each serves."""
    mesh_sizes: list[int]
    members: list[list[int]]                 # per unit: entry indices
    num_sm: float = 0.5
    tp_degree: dict = field(default_factory=dict)  # entry index -> plan tp_degree (metrics' placed_tp)
    gpu_ids: list = field(default_factory=list)    # per unit: the plan's gpu_ids (empty: consecutive)


@dataclass
class _Built:
    cfg: SimConfig
    keep: list = field(default_factory=list)


def _profile_blocks(profile: Sequence[float] | None):
    """The ABI's profile blocks from a flat list: the reference's 7
    LatencyProfile doubles (cost_model.hpp:33-40), optionally followed by the
    HBM decode form's 4 (decode_fixed_ms, decode_row_ms, decode_bctx_ms,
    decode_sm_exponent; LatencyProfile::decode_form 1) and/or the measured TP
    allreduce's 2 (allreduce_alpha_ms, allreduce_ms_per_mib): lengths 7, 9
    (+TP), 11 (+HBM) or 13 (+HBM +TP)."""
    if profile is None:
        return None, None, None
    n = len(profile)
    if n not in (7, 9, 11, 13):
        raise ValueError("profile: 7 reference values, + 4 HBM decode-form values and/or + 2 TP allreduce values")
    prof = (C.c_double * 7)(*profile[:7])
    hbm = (C.c_double * 4)(*profile[7:11]) if n >= 11 else None
    tpar = (C.c_double * 2)(*profile[-2:]) if n in (9, 13) else None
    return prof, hbm, tpar


def _build_config(gpu_memory_bytes: int, num_gpus: int, placement: Placement, params: EngineParams,
                  profile: Sequence[float] | None) -> _Built:
    keep = []
    sizes = (C.c_int * len(placement.mesh_sizes))(*placement.mesh_sizes)
    placed_list = [PlacedLlm(u, e, placement.mesh_sizes[u], placement.num_sm)
                   for u, mem in enumerate(placement.members) for e in mem]
    placed = (PlacedLlm * max(len(placed_list), 1))(*placed_list)
    prof, hbm, tpar = _profile_blocks(profile)
    adapt = (C.c_double * 3)(params.quota_low_mark, params.quota_high_mark, params.quota_step_frac)
    keep += [sizes, placed, prof, hbm, tpar, adapt]
    cfg = SimConfig(1, num_gpus, gpu_memory_bytes, len(placement.mesh_sizes), sizes, len(placed_list),
                    placed, prof, params.scheduler, params.kappa, params.quota_period_s,
                    params.token_budget, params.block_tokens, params.warmup_s, params.decode_sm,
                    params.prefill_min_sm, params.activation_reserve_frac, params.quota_floor_frac, hbm,
                    adapt, tpar)
    return _Built(cfg, keep)


def _c_entries(entries: Sequence[Entry], keep):
    arr = (_CEntry * len(entries))(*[_c_entry(e.spec, e.rate, e.mean_prompt_tokens,
                                             e.mean_output_tokens, keep) for e in entries])
    keep.append(arr)
    return arr


def _c_trace(trace: Sequence[TraceRequest]):
    return (_CRequest * max(len(trace), 1))(*[_CRequest(r.id, r.llm, r.arrival_s, r.prompt_len,
                                                        r.output_len) for r in trace])


@dataclass
class UnitLlmStat:
    """UnitLlmStats (sim_engine.hpp:57-63); llm = entry index."""
    llm: int
    rate: float
    avg_used_blocks: float
    final_quota_blocks: int
    resource_usage: float


@dataclass
class UnitStat:
    """UnitStats (sim_engine.hpp:65-70): pool statistics of one unit;
    samples are (t_s, llm entry index, used_blocks, quota_blocks)."""
    unit: int
    total_blocks: int
    llms: list
    samples: list


def simulate(entries: Sequence[Entry], trace: Sequence[TraceRequest], placement: Placement,
             gpu_memory_bytes: int, params: EngineParams | None = None,
             profile: Sequence[float] | None = None, stats: bool = False):
    """run_simulation (sim_engine.cpp:370-413), priced. Records sorted by id;
    with stats=True returns (records, [UnitStat]) -- SimResult.units."""
    params = params or EngineParams()
    b = _build_config(gpu_memory_bytes, sum(placement.mesh_sizes), placement, params, profile)
    ents = _c_entries(entries, b.keep)
    recs = (Record * max(len(trace), 1))()
    if not stats:
        check(lib.mux_simulate(C.byref(b.cfg), len(entries), ents, len(trace), _c_trace(trace), recs))
        return list(recs[:len(trace)])
    h = C.c_void_p()
    check(lib.mux_simulate_stats(C.byref(b.cfg), len(entries), ents, len(trace), _c_trace(trace), recs,
                                 C.byref(h)))
    units = _read_stats(h)
    return list(recs[:len(trace)]), units


def _read_stats(h) -> list:
    """Copy a mux_sim_stats handle into UnitStat objects and release it."""
    try:
        n = C.c_int()
        check(lib.mux_sim_stats_units(h, C.byref(n)))
        units = []
        for u in range(n.value):
            us = _UnitStats()
            check(lib.mux_sim_stats_unit(h, u, C.byref(us)))
            ll = (_UnitLlmStats * max(us.n_llms, 1))()
            check(lib.mux_sim_stats_llms(h, u, ll))
            ps = (_PoolSample * max(us.n_samples, 1))()
            check(lib.mux_sim_stats_samples(h, u, ps))
            units.append(UnitStat(us.unit, us.total_blocks,
                                  [UnitLlmStat(m.llm, m.rate, m.avg_used_blocks, m.final_quota_blocks,
                                               m.resource_usage) for m in ll[:us.n_llms]],
                                  [(p.t_s, p.llm, p.used_blocks, p.quota_blocks) for p in ps[:us.n_samples]]))
        return units
    finally:
        lib.mux_sim_stats_destroy(h)


def slo_reference_latency_ms(s: LLMSpec, profile: Sequence[float] | None, tp_degree: int, prompt_len: int,
                             output_len: int) -> float:
    """metrics.cpp:21-27 (cost model in libmux.so)."""
    keep = []
    e = _c_entry(s, keep=keep)
    prof = None if profile is None else (C.c_double * 7)(*profile[:7])  # SLO reference: reference form
    out = C.c_double()
    check(lib.mux_slo_reference_latency_ms(C.byref(e), prof, tp_degree, prompt_len, output_len, C.byref(out)))
    return out.value


@dataclass
class ParallelCandidate:
    """ParallelCandidate (placement.hpp:45-52)."""
    tp_degree: int
    num_sm: float
    batch: int
    est_tpt: float
    saturated: bool


def parallel_candidates(entries: Sequence[Entry], gpus_per_node: int, gpu_memory_bytes: int, num_nodes: int = 1,
                        profile: Sequence[float] | None = None, tp_list: Sequence[int] = (1, 2, 4, 8),
                        sm_list: Sequence[float] | None = None, activation_reserve_frac: float = 0.1,
                        max_batch: int = 256) -> list[list[ParallelCandidate]]:
    """llm_parallel_candidates (placement.cpp:57-103) restricted to tp widths
    the engine can shard (tp | num_heads, tp | ffn): one list per entry,
    ascending in tp_list order. Raises Infeasible when a model has none."""
    keep = []
    ents = _c_entries(entries, keep)
    prof, hbm, tpar = _profile_blocks(profile)
    tps = (C.c_int * max(1, len(tp_list)))(*tp_list)
    sms = (C.c_double * max(1, len(sm_list or ())))(*(sm_list or ()))
    cap = max(1, len(entries) * len(tp_list))
    out = (_Candidate * cap)()
    n = C.c_int()
    check(lib.mux_parallel_candidates(len(entries), ents, num_nodes, gpus_per_node, gpu_memory_bytes, prof, hbm, tpar,
                                      len(tp_list), tps, len(sm_list or ()), sms, activation_reserve_frac, max_batch,
                                      out, cap, C.byref(n)))
    res = [[] for _ in entries]
    for c in out[:n.value]:
        res[c.llm].append(ParallelCandidate(c.tp_degree, c.num_sm, c.batch, c.est_tpt, bool(c.saturated)))
    return res


# ---------------------------------------------------------------------- Unit

def _ptr(x) -> int | None:
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return int(x)


def byte_share_partitions(specs: Sequence[LLMSpec], ctx_tokens: Sequence[int], total_sms: int = 148,
                          granule: int = 8) -> list[int]:
    """SMs of each colocated decode job's green partition, proportional to the
    HBM bytes the job streams per round (its weights + the K/V of its members'
    contexts): decode is HBM-bound, so equal per-SM bandwidth demand lets the
    jobs finish their rounds together. The reference expresses the same split
    as a JobPlan's sm_demand share (scheduler.cpp:50-54, sim_engine.cpp:16-18).
    Shares are whole 8-SM granules (the sm_100 green-context granularity),
    largest-remainder rounded; the unit's leftover SMs join the last
    partition (Unit creation does that)."""
    bytes_ = [s.weight_bytes + c * s.kv_bytes_per_token() for s, c in zip(specs, ctx_tokens)]
    n = len(specs)
    units = total_sms // granule
    if n == 0 or units < n:
        raise ValueError("not enough SM granules for one partition per job")
    tot = sum(bytes_)
    exact = [b / tot * units for b in bytes_]
    share = [max(1, int(e)) for e in exact]
    while sum(share) > units:
        share[max(range(n), key=lambda i: share[i] - exact[i])] -= 1
    for i in sorted(range(n), key=lambda i: share[i] - exact[i])[: units - sum(share)]:
        share[i] += 1
    return [g * granule for g in share]


class Unit:
    """One GPU: the unified KV pool in HBM plus colocated LLaMA models."""

    def __init__(self, specs: Sequence[LLMSpec], pool_blocks: int, device: int = 0,
                 device_pool_blocks: int = 0, max_batch: int = 256, max_prefill_tokens: int = 4096,
                 max_ctx: int = 4096, max_slots: int = 0, init_seed: int = 0,
                 init_std: float = 0.02, partitions: int = 2, partition_sms: Sequence[int] | None = None,
                 tp_rank: int = 0, tp_size: int = 1):
        """partition_sms[p] > 0 puts partition p on its own green context of
        that many SMs (the SM share a JobPlan's sm_demand asks for)."""
        self.specs = list(specs)
        self._keep = []
        ents = (_CEntry * len(specs))(*[_c_entry(s, keep=self._keep) for s in specs])
        self._keep.append(ents)
        psms = None
        if partition_sms is not None:
            if len(partition_sms) != partitions:
                raise ValueError("partition_sms needs one entry per partition")
            psms = (C.c_int * partitions)(*partition_sms)
            self._keep.append(psms)
        cfg = UnitConfig(device, len(specs), ents, pool_blocks, device_pool_blocks, max_batch,
                         max_prefill_tokens, max_ctx, max_slots, init_seed, init_std, partitions, psms,
                         tp_rank, tp_size)
        h = C.c_void_p()
        check(lib.mux_unit_create(C.byref(cfg), C.byref(h)))
        self._h = h.value
        self.pool = BlockPool(0, _handle=lib.mux_unit_pool(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib.mux_unit_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def set_tensor(self, llm: int, name: str, layer: int, host_array) -> None:
        """host_array: a contiguous numpy array in device layout (see mux.h)."""
        check(lib.mux_unit_set_tensor(self._h, llm, name.encode(), layer,
                                      host_array.ctypes.data, host_array.nbytes))

    def get_tensor(self, llm: int, name: str, layer: int, host_array) -> None:
        check(lib.mux_unit_get_tensor(self._h, llm, name.encode(), layer,
                                      host_array.ctypes.data, host_array.nbytes))

    def init_kv(self, seed: int = 1, std: float = 1.0):
        check(lib.mux_unit_init_kv(self._h, seed, std))

    def device_ptrs(self, llm: int):
        pool, rr, rl = C.c_void_p(), C.c_void_p(), C.c_void_p()
        mr, rw = C.c_int(), C.c_int()
        check(lib.mux_unit_device_ptrs(self._h, llm, C.byref(pool), C.byref(rr), C.byref(rl),
                                       C.byref(mr), C.byref(rw)))
        return pool.value, rr.value, rl.value, mr.value, rw.value

    @staticmethod
    def _ids(request_ids):
        return (C.c_int64 * len(request_ids))(*request_ids)

    def prefill(self, llm: int, request_ids: Sequence[int], tokens, out=None, partition: int = 0):
        """tokens: int32 numpy array (concatenated prompts); out: int32 numpy or None."""
        check(lib.mux_unit_prefill(self._h, llm, len(request_ids), self._ids(request_ids),
                                   tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                                   None if out is None else out.ctypes.data_as(C.POINTER(C.c_int32)),
                                   partition))

    def decode(self, llm: int, request_ids: Sequence[int], tokens=None, out=None, partition: int = 0,
               ids_c=None):
        ids = ids_c if ids_c is not None else self._ids(request_ids)
        check(lib.mux_unit_decode(
            self._h, llm, len(request_ids), ids,
            None if tokens is None else tokens.ctypes.data_as(C.POINTER(C.c_int32)),
            None if out is None else out.ctypes.data_as(C.POINTER(C.c_int32)), partition))

    def sync(self):
        check(lib.mux_unit_sync(self._h))

    def record(self, partition: int, slot: int):
        check(lib.mux_unit_record(self._h, partition, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(lib.mux_unit_elapsed(self._h, a, b, C.byref(ms)))
        return ms.value

    def attn_timing(self, enable: bool):
        check(lib.mux_unit_attn_timing(self._h, 1 if enable else 0))

    def attn_time(self):
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        check(lib.mux_unit_attn_time(self._h, C.byref(ms), C.byref(n), C.byref(by)))
        return ms.value, n.value, by.value

    def gemm_time(self):
        """(total ms, launches, weight bytes) of the decode GEMMs timed while
        attn_timing is on."""
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        check(lib.mux_unit_gemm_time(self._h, C.byref(ms), C.byref(n), C.byref(by)))
        return ms.value, n.value, by.value

    def tp_mailbox(self, partition: int):
        """(device pointer, 64-byte CUDA IPC handle) of a partition's TP mailbox."""
        ptr = C.c_void_p()
        handle = (C.c_ubyte * 64)()
        check(lib.mux_unit_tp_mailbox(self._h, partition, C.byref(ptr), handle))
        return ptr.value, bytes(handle)

    def tp_connect(self, partition: int, peer_rank: int, handle: bytes | None = None, ptr: int | None = None):
        """Map a peer rank's mailbox: IPC handle (other process) or pointer (same process)."""
        h = None if handle is None else (C.c_ubyte * 64).from_buffer_copy(handle)
        check(lib.mux_unit_tp_connect(self._h, partition, peer_rank, h, ptr))

    def last_stats(self) -> list:
        """Pool statistics (SimResult.units) of the last run_lockstep / measured run."""
        h = C.c_void_p()
        check(lib.mux_unit_last_stats(self._h, C.byref(h)))
        return _read_stats(h)

    def partition_sms(self, partition: int) -> int:
        v = C.c_int()
        check(lib.mux_unit_partition_sms(self._h, partition, C.byref(v)))
        return v.value

    def probe_smids(self, partition: int, blocks: int):
        out = (C.c_int * blocks)()
        check(lib.mux_unit_probe_smids(self._h, partition, blocks, out))
        return list(out)

    def route_log(self) -> list[dict]:
        """Jobs of the last engine run with option sm_route: pass, job, llm,
        kind (0 prefill / 1 decode), sm_demand, SM run and its SM count."""
        n = C.c_int64()
        check(lib.mux_unit_route_log(self._h, None, 0, C.byref(n)))
        buf = (_RouteRecord * max(n.value, 1))()
        check(lib.mux_unit_route_log(self._h, buf, n.value, C.byref(n)))
        return [{"pass": r.pass_, "job": r.job, "llm": r.llm, "kind": r.kind, "sm_demand": r.sm_demand,
                 "first_unit": r.first_unit, "units": r.units, "sms": r.sms, "workspace": r.workspace,
                 "busy_units": r.busy_units}
                for r in buf[:n.value]]

    def route_units(self) -> list[int]:
        """SMs of each green-context unit of the device (sm_route's granules)."""
        n = C.c_int()
        buf = (C.c_int * 64)()
        check(lib.mux_unit_route_units(self._h, C.byref(n), buf, 64))
        return list(buf[:n.value])

    def probe_route(self, first_unit: int, units: int, blocks: int) -> list[int]:
        out = (C.c_int * blocks)()
        check(lib.mux_unit_probe_route(self._h, first_unit, units, blocks, out))
        return list(out)

    def launches(self) -> int:
        return int(lib.mux_unit_launches(self._h))

    def set_option(self, key: str, value: int):
        check(lib.mux_unit_set_option(self._h, key.encode(), value))

    def pass_stats(self) -> tuple[int, int]:
        """(passes, green passes) of the last lockstep / measured run."""
        a, b = C.c_int64(), C.c_int64()
        check(lib.mux_unit_pass_stats(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def run_lockstep(self, entries: Sequence[Entry], trace: Sequence[TraceRequest],
                     gpu_memory_bytes: int, params: EngineParams | None = None,
                     prompt_seed: int = 11, num_sm: float = 0.5, profile=None, measured: bool = False,
                     realtime: bool = False, mesh_size: int = 1):
        """Engine decisions priced by the oracle model, every job run on this GPU
        (mesh_size > 1: this unit is one rank of a tensor-parallel mesh of that
        many GPUs, created with tp_size = mesh_size; lockstep only)
        (measured=True: job durations are the measured device times instead;
        realtime=True: jobs overlap across passes and complete when their
        device events fire, mux_unit_run_realtime).
        Returns (records, tokens) with tokens[i] the output of trace[i]."""
        params = params or EngineParams()
        placement = Placement([mesh_size], [list(range(len(entries)))], num_sm)
        b = _build_config(gpu_memory_bytes, mesh_size, placement, params, profile)
        ents = _c_entries(entries, b.keep)
        recs = (Record * max(len(trace), 1))()
        total = sum(r.output_len for r in trace)
        toks = (C.c_int32 * max(total, 1))()
        fn = (lib.mux_unit_run_realtime if realtime else
              lib.mux_unit_run_measured if measured else lib.mux_unit_run_lockstep)
        check(fn(self._h, C.byref(b.cfg), len(entries), ents, len(trace), _c_trace(trace), prompt_seed, recs, toks))
        out, off = [], 0
        for r in trace:
            out.append(list(toks[off:off + r.output_len]))
            off += r.output_len
        return list(recs[:len(trace)]), out


# ------------------------------------------------------------ kernel wrappers

def decode_attention_headwise(q, pool_ptr, rowrec_ptr, rowlist_ptr, slots, ctx, num_layers: int,
                              layer: int, max_rows: int, max_ctx: int, out, kv_splits: int = 0,
                              workspace=None, stream=None):
    """K1 for one layer; q/out/slots/ctx are torch CUDA tensors."""
    B, H = q.shape[0], q.shape[1]
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    check(lib.mux_decode_attention_headwise(
        _ptr(q), _ptr(pool_ptr), _ptr(rowrec_ptr), _ptr(rowlist_ptr), _ptr(slots), _ptr(ctx), B, H,
        num_layers, layer, max_rows, max_ctx, _ptr(out), 1 if out.dtype.itemsize == 4 else 0,
        kv_splits, _ptr(workspace), ws_bytes, _ptr(stream)))


def prefill_attention(q, qkv, out, seq_lens, stream=None):
    """K3 (tcgen05): causal attention of each prompt; q/qkv/out torch CUDA bf16
    tensors [T,H,128] / [T,3,H,128] / [T,H,128]; seq_lens host ints."""
    lens = (C.c_int32 * len(seq_lens))(*seq_lens)
    check(lib.mux_prefill_attention(_ptr(q), _ptr(qkv), _ptr(out), lens, len(seq_lens), q.shape[1],
                                    _ptr(stream)))


def kv_append(qkv, q_out, pool_ptr, rowrec_ptr, rowlist_ptr, tok_slot, tok_pos, rope, T: int, H: int,
              num_layers: int, layer: int, max_rows: int, stream=None):
    check(lib.mux_kv_append(_ptr(qkv), _ptr(q_out), _ptr(pool_ptr), _ptr(rowrec_ptr),
                            _ptr(rowlist_ptr), _ptr(tok_slot), _ptr(tok_pos), _ptr(rope),
                            rope.shape[0], T, H, num_layers, layer, max_rows, _ptr(stream)))


def rope_table(positions: int):
    import numpy as np
    out = np.empty((positions, 64, 2), dtype=np.float32)
    check(lib.mux_rope_table(positions, out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def gemm_bf16(x, w, out, epilogue: int = 0, grid: int = 0, stream=None, w_tiled=None):
    """x @ w.T on tcgen05 (x [M,K], w [N,K] bf16 CUDA tensors). epilogue: 0 store
    bf16, 1 out += (fp32), 2 SiLU(gate)*up of interleaved rows, 3 store fp32.
    w_tiled: the same weights in weight_tile() layout (streamed by bulk copy)."""
    M, K = x.shape
    N = w.shape[0]
    src = w if w_tiled is None else w_tiled
    check(lib.mux_gemm_bf16(_ptr(x), _ptr(src), 0 if w_tiled is None else 1, M, N, K, _ptr(out), epilogue,
                            grid, _ptr(stream)))


def weight_tile(w, stream=None):
    """Row-major [N,K] bf16 CUDA tensor -> uint8 tensor in the B200 tile layout."""
    import torch
    N, K = w.shape
    out = torch.empty(int(lib.mux_weight_tiled_bytes(N, K)), dtype=torch.uint8, device=w.device)
    check(lib.mux_weight_tile(_ptr(w), N, K, _ptr(out), 0, _ptr(stream)))
    return out
