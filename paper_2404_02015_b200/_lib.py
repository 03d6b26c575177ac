"""ctypes binding of libmux.so (include/mux.h).

The product path is the C ABI; this module only declares it. Importing it
loads the in-tree ``libmux.so`` and fails loudly when it is missing -- there
is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmux.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "mux.h")

MUX_OK, MUX_EINVAL, MUX_EINFEAS, MUX_EINTERNAL = 0, 1, 2, 3
ALLOC_OK, ALLOC_POOL, ALLOC_QUOTA = 0, 1, 2

i32, i64, f32, f64, u64 = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_uint64
vp, sz = C.c_void_p, C.c_size_t
P = C.POINTER


class MuxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[mux status {code}] {msg}")
        self.code = code


class InvalidArgument(MuxError, ValueError):
    pass


class Infeasible(MuxError):
    pass


class LogicError(MuxError):
    pass


class LlmEntry(C.Structure):
    _fields_ = [("name", C.c_char_p), ("num_layers", C.c_int), ("num_heads", C.c_int),
                ("head_dim", C.c_int), ("hidden_size", C.c_int), ("weight_bytes", i64),
                ("bytes_per_element", C.c_int), ("rate", f64), ("mean_prompt_tokens", f64),
                ("mean_output_tokens", f64), ("ffn", C.c_int), ("vocab", C.c_int)]


class PlacedLlm(C.Structure):
    _fields_ = [("unit", C.c_int), ("llm", C.c_int), ("tp_degree", C.c_int), ("num_sm", f64)]


class SimConfig(C.Structure):
    _fields_ = [("num_nodes", C.c_int), ("gpus_per_node", C.c_int), ("gpu_memory_bytes", i64),
                ("n_units", C.c_int), ("unit_mesh_size", P(C.c_int)), ("n_placed", C.c_int),
                ("placed", P(PlacedLlm)), ("profile", P(f64)), ("scheduler", C.c_int),
                ("kappa", f64), ("quota_period_s", f64), ("token_budget", i64),
                ("block_tokens", C.c_int), ("warmup_s", f64), ("decode_sm", f64),
                ("prefill_min_sm", f64), ("activation_reserve_frac", f64),
                ("quota_floor_frac", f64), ("decode_hbm", P(f64)),
                ("quota_adapt", P(f64)), ("tp_allreduce", P(f64))]


class Candidate(C.Structure):
    _fields_ = [("llm", C.c_int), ("tp_degree", C.c_int), ("num_sm", f64), ("batch", C.c_int),
                ("est_tpt", f64), ("saturated", C.c_int)]


class RouteRecord(C.Structure):
    _fields_ = [("pass_", i64), ("job", i64), ("llm", C.c_int), ("kind", C.c_int), ("sm_demand", f64),
                ("first_unit", C.c_int), ("units", C.c_int), ("sms", C.c_int), ("workspace", C.c_int),
                ("busy_units", u64)]


class Request(C.Structure):
    _fields_ = [("id", i64), ("llm", C.c_int), ("arrival_s", f64), ("prompt_len", C.c_int),
                ("output_len", C.c_int)]


class Record(C.Structure):
    _fields_ = [("id", i64), ("llm", C.c_int), ("arrival_s", f64), ("first_token_s", f64),
                ("done_s", f64), ("prompt_len", C.c_int), ("output_len", C.c_int)]


class UnitStats(C.Structure):
    _fields_ = [("unit", C.c_int), ("total_blocks", i64), ("n_llms", C.c_int), ("n_samples", i64)]


class UnitLlmStats(C.Structure):
    _fields_ = [("llm", C.c_int), ("rate", f64), ("avg_used_blocks", f64), ("final_quota_blocks", i64),
                ("resource_usage", f64)]


class PoolSample(C.Structure):
    _fields_ = [("t_s", f64), ("llm", C.c_int), ("used_blocks", i64), ("quota_blocks", i64)]


class UnitConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("n_llms", C.c_int), ("llms", P(LlmEntry)),
                ("pool_blocks", i64), ("device_pool_blocks", i64), ("max_batch", C.c_int),
                ("max_prefill_tokens", C.c_int), ("max_ctx", C.c_int), ("max_slots", C.c_int),
                ("init_seed", u64), ("init_std", f32), ("partitions", C.c_int),
                ("partition_sms", P(C.c_int)), ("tp_rank", C.c_int), ("tp_size", C.c_int)]


_SIGS = {
    "mux_last_error": (C.c_char_p, []),
    "mux_version": (C.c_char_p, []),
    "mux_blocks_for_tokens": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, P(i64)]),
    "mux_init_token_block_quota": (C.c_int, [C.c_int, P(f64), P(f64), P(f64), i64, f64, P(i64)]),
    "mux_adapt_quota": (C.c_int, [C.c_int, P(f64), P(i64), i64, f64, f64, f64, P(i64)]),
    "mux_pool_create": (C.c_int, [i64, C.c_int, P(vp)]),
    "mux_pool_destroy": (None, [vp]),
    "mux_pool_register_llm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "mux_pool_admit": (C.c_int, [vp, C.c_int, i64, i64, i64, P(C.c_int)]),
    "mux_pool_alloc": (C.c_int, [vp, C.c_int, i64, i64, C.c_int, P(C.c_int)]),
    "mux_pool_alloc_n": (C.c_int, [vp, C.c_int, C.c_int, P(i64), i64, C.c_int, P(C.c_int)]),
    "mux_pool_free_request": (C.c_int, [vp, C.c_int, i64]),
    "mux_pool_set_quota": (C.c_int, [vp, C.c_int, i64]),
    "mux_pool_llm_stats": (C.c_int, [vp, C.c_int, P(i64), P(i64), P(i64)]),
    "mux_pool_request_tokens": (C.c_int, [vp, C.c_int, i64, P(i64)]),
    "mux_pool_totals": (C.c_int, [vp, P(i64), P(i64), P(i64)]),
    "mux_pool_check": (C.c_int, [vp]),
    "mux_pool_block_table": (C.c_int, [vp, C.c_int, i64, P(i32), i64, P(i64)]),
    "mux_pool_slot": (C.c_int, [vp, C.c_int, i64, P(C.c_int)]),
    "mux_simulate": (C.c_int, [P(SimConfig), C.c_int, P(LlmEntry), C.c_int, P(Request), P(Record)]),
    "mux_simulate_stats": (C.c_int, [P(SimConfig), C.c_int, P(LlmEntry), C.c_int, P(Request), P(Record),
                                     P(vp)]),
    "mux_sim_stats_units": (C.c_int, [vp, P(C.c_int)]),
    "mux_sim_stats_unit": (C.c_int, [vp, C.c_int, P(UnitStats)]),
    "mux_sim_stats_llms": (C.c_int, [vp, C.c_int, P(UnitLlmStats)]),
    "mux_sim_stats_samples": (C.c_int, [vp, C.c_int, P(PoolSample)]),
    "mux_sim_stats_destroy": (None, [vp]),
    "mux_parallel_candidates": (C.c_int, [C.c_int, P(LlmEntry), C.c_int, C.c_int, i64, P(f64), P(f64), P(f64),
                                          C.c_int, P(C.c_int), C.c_int, P(f64), f64, C.c_int, P(Candidate),
                                          C.c_int, P(C.c_int)]),
    "mux_slo_reference_latency_ms": (C.c_int, [P(LlmEntry), P(f64), C.c_int, C.c_int, C.c_int, P(f64)]),
    "mux_decode_attention_headwise": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                                C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int,
                                                vp, sz, vp]),
    "mux_prefill_attention": (C.c_int, [vp, vp, vp, P(i32), C.c_int, C.c_int, vp]),
    "mux_kv_append": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_int, vp]),
    "mux_rope_table": (C.c_int, [C.c_int, P(f32)]),
    "mux_gemm_bf16": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp]),
    "mux_weight_tile": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp]),
    "mux_weight_tiled_bytes": (i64, [C.c_int, C.c_int]),
    "mux_unit_tp_mailbox": (C.c_int, [vp, C.c_int, P(vp), vp]),
    "mux_unit_tp_connect": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "mux_unit_tp_debug": (C.c_int, [vp, C.c_int, P(C.c_uint32)]),
    "mux_unit_partition_sms": (C.c_int, [vp, C.c_int, P(C.c_int)]),
    "mux_unit_probe_smids": (C.c_int, [vp, C.c_int, C.c_int, P(C.c_int)]),
    "mux_unit_route_log": (C.c_int, [vp, vp, i64, P(i64)]),
    "mux_unit_route_units": (C.c_int, [vp, P(C.c_int), P(C.c_int), C.c_int]),
    "mux_unit_probe_route": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, P(C.c_int)]),
    "mux_unit_set_option": (C.c_int, [vp, C.c_char_p, i64]),
    "mux_debug_gemm_timing": (None, [vp]),
    "mux_unit_create": (C.c_int, [P(UnitConfig), P(vp)]),
    "mux_unit_destroy": (None, [vp]),
    "mux_unit_pool": (vp, [vp]),
    "mux_unit_set_tensor": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_int, vp, sz]),
    "mux_unit_get_tensor": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_int, vp, sz]),
    "mux_unit_init_kv": (C.c_int, [vp, u64, f32]),
    "mux_unit_device_ptrs": (C.c_int, [vp, C.c_int, P(vp), P(vp), P(vp), P(C.c_int), P(C.c_int)]),
    "mux_unit_prefill": (C.c_int, [vp, C.c_int, C.c_int, P(i64), P(i32), P(i32), C.c_int]),
    "mux_unit_decode": (C.c_int, [vp, C.c_int, C.c_int, P(i64), P(i32), P(i32), C.c_int]),
    "mux_unit_sync": (C.c_int, [vp]),
    "mux_unit_record": (C.c_int, [vp, C.c_int, C.c_int]),
    "mux_unit_elapsed": (C.c_int, [vp, C.c_int, C.c_int, P(f32)]),
    "mux_unit_attn_timing": (C.c_int, [vp, C.c_int]),
    "mux_unit_attn_time": (C.c_int, [vp, P(f64), P(i64), P(f64)]),
    "mux_unit_gemm_time": (C.c_int, [vp, P(f64), P(i64), P(f64)]),
    "mux_unit_launches": (i64, [vp]),
    "mux_unit_pass_stats": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)]),
    "mux_unit_last_stats": (C.c_int, [vp, P(vp)]),
    "mux_unit_run_lockstep": (C.c_int, [vp, P(SimConfig), C.c_int, P(LlmEntry), C.c_int,
                                        P(Request), u64, P(Record), P(i32)]),
    "mux_unit_run_measured": (C.c_int, [vp, P(SimConfig), C.c_int, P(LlmEntry), C.c_int,
                                        P(Request), u64, P(Record), P(i32)]),
    "mux_unit_run_realtime": (C.c_int, [vp, P(SimConfig), C.c_int, P(LlmEntry), C.c_int,
                                        P(Request), u64, P(Record), P(i32)]),
}


def header_symbols() -> list[str]:
    """Every function declared in include/mux.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^MUX_API\s+[\w\s\*]*?\b(mux_\w+)\s*\(", text, re.M)))


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libmux.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status == MUX_OK:
        return
    msg = (lib.mux_last_error() or b"").decode()
    cls = {MUX_EINVAL: InvalidArgument, MUX_EINFEAS: Infeasible}.get(status, LogicError)
    raise cls(status, msg)
