"""Wire formats of the reference's `muxsim simulate`, so the
B200 engine is a drop-in for that command: the experiment config JSON
(subset the engine consumes), plan.json, trace.csv in, records.csv out.

Format sources (reference, read-only):
  config        /root/reference/proj/src/config.cpp:216-321 (cluster / llms /
                workload.power_law / sim / profile; decode_sm defaults to
                the profile's f_sat, :277)
  plan.json     /root/reference/proj/src/commands.cpp:165-217 placement_from_json
  trace.csv     /root/reference/proj/src/workload.cpp:138-215 save/load_trace
  records.csv   /root/reference/proj/src/commands.cpp:74-87 write_records_csv
  metrics.json  /root/reference/proj/src/metrics.cpp:40-167 compute_metrics /
                report_to_json (nlohmann ordered_json dump(2))
  poolstats.json /root/reference/proj/src/commands.cpp:89-121 poolstats_json
  rates         /root/reference/proj/src/workload.cpp:78-86 gen_rates
The engine itself is libmux.so (priced: mux_simulate, bit-identical to the
reference; lockstep / measured: a GPU unit).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

from .host import CATALOG, EngineParams, Entry, LLMSpec, Placement, TraceRequest, slo_reference_latency_ms

GIB = 1 << 30

# LatencyProfile fields in declaration order (cost_model.hpp:33-40)
PROFILE_KEYS = ["prefill_ms_per_token", "decode_base_ms", "decode_ctx_ms_per_token", "tp_efficiency",
                "sm_saturation_point", "batch_knee", "reference_scale"]
PROFILE_DEFAULTS = [0.25, 12.0, 0.005, 0.9, 0.5, 16.0, 32.0 * 4096.0]
# B200 extension: the HBM-bound decode form (LatencyProfile::decode_form 1,
# DESIGN §4). A profile block holding all three keys selects it; the
# reference's configs never carry them, so their parsing is unchanged.
HBM_KEYS = ["decode_fixed_ms", "decode_row_ms", "decode_bctx_ms", "decode_sm_exponent"]
SCHEDULERS = {"adbs": 0, "fcfs": 1, "round_robin": 2, "rr": 2}


class ConfigError(ValueError):
    """The reference's ConfigError (CLI exit code 1)."""


@dataclass
class Experiment:
    num_nodes: int
    gpus_per_node: int
    gpu_memory_bytes: int
    names: list[str]
    entries: list[Entry]
    params: EngineParams
    profile: list[float]
    horizon_s: float = 60.0
    seed: int = 0
    extra: dict = field(default_factory=dict)
    slo_scales: list = field(default_factory=lambda: [1.0, 2.0, 4.0, 8.0, 16.0])  # config.hpp:61
    slo_reference_tp_one: bool = False                                           # config.hpp:60


def _mean_len(d, what):
    kind = d.get("kind")
    if kind == "constant":
        return float(d["value"])
    if kind in ("lognormal", "empirical"):
        if "mean" in d:
            return float(d["mean"])
        vals = d.get("values") or []
        if vals:
            return sum(vals) / len(vals)
    raise ConfigError(f"{what}: unsupported length distribution {d!r}")


def gen_rates(n, alpha, max_rate):
    """workload.cpp:78-86."""
    if n < 1 or not alpha >= 0.0 or not max_rate > 0.0:
        raise ConfigError("power_law: need n >= 1, alpha >= 0, max_rate_rps > 0")
    return [max_rate * (i + 1) ** (-alpha) for i in range(n)]


def load_config(path: str, catalog: dict[str, LLMSpec] | None = None) -> Experiment:
    catalog = catalog or CATALOG
    with open(path) as f:
        try:
            root = json.load(f)
        except json.JSONDecodeError as e:
            raise ConfigError(f"config: invalid JSON: {e}") from None
    cl = root.get("cluster") or {}
    try:
        num_nodes, gpn = int(cl["num_nodes"]), int(cl["gpus_per_node"])
        mem = int(round(float(cl["gpu_memory_gb"]) * GIB))  # GiB (config.cpp:141)
    except KeyError as e:
        raise ConfigError(f"cluster: missing {e}") from None
    llms = root.get("llms") or []
    if not llms:
        raise ConfigError("config: 'llms' must be a non-empty array")
    wl = root.get("workload") or {}
    rates = [float(m.get("rate_rps", 0.0)) for m in llms]
    if "power_law" in wl:
        pl = wl["power_law"]
        rates = gen_rates(len(llms), float(pl["alpha"]), float(pl["max_rate_rps"]))
    names, entries = [], []
    for m, rate in zip(llms, rates):
        model = m.get("model")
        if model not in catalog:
            raise ConfigError(f"llm '{m.get('name')}': unknown model '{model}'")
        spec = catalog[model]
        name = m.get("name", model)
        names.append(name)
        entries.append(Entry(LLMSpec(name, spec.num_layers, spec.num_heads, spec.head_dim, spec.hidden_size,
                                     spec.weight_bytes, spec.bytes_per_element, spec.ffn, spec.vocab),
                             rate, _mean_len(m.get("prompt_len", {"kind": "constant", "value": 1}), "prompt_len"),
                             _mean_len(m.get("output_len", {"kind": "constant", "value": 1}), "output_len")))
    prof = list(PROFILE_DEFAULTS)
    hbm = {}
    for k, v in (root.get("profile") or {}).items():
        if k in HBM_KEYS:
            hbm[k] = float(v)
            continue
        if k not in PROFILE_KEYS:
            raise ConfigError(f"profile: unknown key '{k}'")
        prof[PROFILE_KEYS.index(k)] = float(v)
    if hbm:
        if len(hbm) != len(HBM_KEYS):
            raise ConfigError("profile: the HBM decode form needs " + ", ".join(HBM_KEYS))
        prof += [hbm[k] for k in HBM_KEYS]
    p = EngineParams()
    sim = root.get("sim") or {}
    if "scheduler" in sim:
        if sim["scheduler"] not in SCHEDULERS:
            raise ConfigError(f"sim.scheduler: unknown '{sim['scheduler']}'")
        p.scheduler = SCHEDULERS[sim["scheduler"]]
    for k in ("kappa", "quota_period_s", "warmup_s", "decode_sm", "prefill_min_sm", "activation_reserve_frac",
              "quota_floor_frac"):
        if k in sim:
            setattr(p, k, float(sim[k]))
    for k in ("token_budget", "block_tokens"):
        if k in sim:
            setattr(p, k, int(sim[k]))
    if "decode_sm" not in sim:
        p.decode_sm = prof[PROFILE_KEYS.index("sm_saturation_point")]
    exp = Experiment(num_nodes, gpn, mem, names, entries, p, prof, float(wl.get("horizon_s", 60.0)),
                     int(wl.get("seed", 0)), {"root": root})
    if exp.horizon_s <= 0.0:
        raise ConfigError("workload.horizon_s must be positive")
    scales = (root.get("metrics") or {}).get("slo_scales")
    if scales is not None:
        if not isinstance(scales, list) or not scales or any(float(x) <= 0.0 for x in scales):
            raise ConfigError("metrics.slo_scales must be a non-empty list of positive numbers")
        exp.slo_scales = [float(x) for x in scales]
    exp.slo_reference_tp_one = bool(sim.get("slo_reference_tp_one", False))
    return exp


def load_plan(path: str, names: list[str]) -> Placement:
    """plan.json -> units (mesh size = len(gpu_ids)) and their members."""
    with open(path) as f:
        try:
            root = json.load(f)
        except json.JSONDecodeError as e:
            raise ConfigError(f"plan: invalid JSON: {e}") from None
    if not isinstance(root, dict) or not isinstance(root.get("units"), list):
        raise ConfigError("plan: expected an object with a 'units' array")
    sizes, members, tp = [], [], {}
    for u in root["units"]:
        if not isinstance(u, dict) or not isinstance(u.get("gpu_ids"), list):
            raise ConfigError("plan: each unit needs a gpu_ids array")
        sizes.append(len(u["gpu_ids"]))
        mem = []
        for m in u.get("models", []):
            if m.get("name") not in names:
                raise ConfigError(f"plan: model '{m.get('name')}' is not in the config")
            mem.append(names.index(m["name"]))
            tp[names.index(m["name"])] = int(m.get("tp_degree", len(u["gpu_ids"])))  # commands.cpp:205
        members.append(mem)
    return Placement(sizes, members, tp_degree=tp)


def load_trace(path: str, names: list[str]) -> list[TraceRequest]:
    """trace.csv (workload.cpp:174-215): header, then id,llm,arrival_s,prompt_len,output_len."""
    out = []
    with open(path) as f:
        saw_header = False
        for no, line in enumerate(f, 1):
            line = line.rstrip("\n").rstrip("\r")
            if not line:
                continue
            if not saw_header:
                if line != "id,llm,arrival_s,prompt_len,output_len":
                    raise ConfigError(f"{path}:{no}: expected header 'id,llm,arrival_s,prompt_len,output_len'")
                saw_header = True
                continue
            fs = line.split(",")
            if len(fs) != 5:
                raise ConfigError(f"{path}:{no}: expected 5 fields, got {len(fs)}")
            if fs[1] not in names:
                raise ConfigError(f"{path}:{no}: model '{fs[1]}' is not in the config")
            try:
                r = TraceRequest(int(fs[0]), names.index(fs[1]), float(fs[2]), int(fs[3]), int(fs[4]))
            except ValueError:
                raise ConfigError(f"{path}:{no}: malformed row '{line}'") from None
            if r.arrival_s < 0 or r.prompt_len < 1 or r.output_len < 1:
                raise ConfigError(f"{path}:{no}: bad values '{line}'")
            out.append(r)
    return out


def save_trace(path: str, trace: list[TraceRequest], names: list[str]) -> None:
    with open(path, "w") as f:
        f.write("id,llm,arrival_s,prompt_len,output_len\n")
        for r in trace:
            f.write("%d,%s,%.17g,%d,%d\n" % (r.id, names[r.llm], r.arrival_s, r.prompt_len, r.output_len))


def write_records_csv(path: str, records, names: list[str]) -> None:
    """commands.cpp:74-87, byte for byte (printf %.9f == Python %.9f)."""
    with open(path, "wb") as f:
        f.write(b"id,llm,arrival_s,ttft_s,tpot_s,done_s\n")
        for r in records:
            ttft = r.first_token_s - r.arrival_s
            tpot = (r.done_s - r.first_token_s) / (r.output_len - 1) if r.output_len > 1 else 0.0
            f.write(b"%d,%s,%.9f,%.9f,%.9f,%.9f\n" % (r.id, names[r.llm].encode(), r.arrival_s, ttft, tpot,
                                                   r.done_s))


# ------------------------------------------------------------ metrics.json

def _dump(obj) -> str:
    """nlohmann::ordered_json::dump(2) + newline: insertion-ordered keys,
    2-space indent, shortest round-trip doubles (integral ones as "2.0"),
    fixed notation below 1e15 and exponent form (1e-05, 1e+15) outside
    [1e-4, 1e15) -- Python's repr differs only in [1e15, 1e16)."""
    def num(x: float) -> str:
        if math.isnan(x) or math.isinf(x):
            return "null"
        if x == 0.0:
            return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
        # shortest round-trip digits (as nlohmann's grisu2 to_chars), value = digits * 10^k
        sign = "-" if x < 0 else ""
        mant, _, exp = ("%r" % abs(x)).partition("e")
        ip, _, fp = mant.partition(".")
        digits = (ip + fp).lstrip("0")
        k = (int(exp) if exp else 0) - len(fp)
        stripped = digits.rstrip("0")
        k += len(digits) - len(stripped)
        digits = stripped
        n = k + len(digits)
        if k >= 0 and n <= 15:
            return sign + digits + "0" * k + ".0"
        if 0 < n <= 15:
            return sign + digits[:n] + "." + digits[n:]
        if -4 < n <= 0:
            return sign + "0." + "0" * (-n) + digits
        e = n - 1
        m = digits[0] + ("." + digits[1:] if len(digits) > 1 else "")
        return sign + m + "e" + ("-" if e < 0 else "+") + "%02d" % abs(e)

    def enc(o, ind):
        pad, pad2 = "  " * ind, "  " * (ind + 1)
        if isinstance(o, dict):
            if not o:
                return "{}"
            return "{\n" + ",\n".join(f"{pad2}{json.dumps(k)}: {enc(v, ind + 1)}" for k, v in o.items()) + "\n" + pad + "}"
        if isinstance(o, list):
            if not o:
                return "[]"
            return "[\n" + ",\n".join(pad2 + enc(v, ind + 1) for v in o) + "\n" + pad + "]"
        if isinstance(o, bool):
            return "true" if o else "false"
        if isinstance(o, int):
            return str(o)
        if isinstance(o, float):
            return num(o)
        if isinstance(o, str):
            return json.dumps(o)
        raise TypeError(type(o))
    return enc(obj, 0) + "\n"


def _percentile(values, p):
    """metrics.cpp:12-19, nearest rank: sorted[ceil(p*n)-1]."""
    v = sorted(values)
    return v[math.ceil(p * len(v)) - 1]


def compute_metrics(records, exp: Experiment, placement: Placement) -> dict:
    """metrics.cpp:40-113 over the engine's records (any engine: priced,
    lockstep or measured). Returns the report as plain values."""
    if exp.horizon_s <= 0.0:
        raise ConfigError("horizon must be positive")
    scales = exp.slo_scales
    total_rate = sum(e.rate for e in exp.entries)
    overall_met, overall_total = [0] * len(scales), 0
    report = {"aggregated_throughput_rps": 0.0, "llms": []}
    for li, (name, e) in enumerate(zip(exp.names, exp.entries)):
        if li not in placement.tp_degree:
            raise ConfigError(f"plan does not place model '{name}'")  # commands.cpp:66-68
        tp_ref = 1 if exp.slo_reference_tp_one else placement.tp_degree[li]
        ttft, tpot, lat = [], [], []
        met, total, completed = [0] * len(scales), 0, 0
        for r in records:
            if r.llm != li:
                continue
            total += 1
            if r.done_s <= exp.horizon_s:
                completed += 1
            ttft.append(r.first_token_s - r.arrival_s)
            if r.output_len > 1:
                tpot.append((r.done_s - r.first_token_s) / float(r.output_len - 1))
            e2e = r.done_s - r.arrival_s
            lat.append(e2e / float(r.output_len))
            ref_s = slo_reference_latency_ms(e.spec, exp.profile, tp_ref, r.prompt_len, r.output_len) / 1000.0
            for si, sc in enumerate(scales):
                if e2e <= sc * ref_s * (1.0 + 1e-9):
                    met[si] += 1

        def mean(v):
            s = 0.0
            for x in v:
                s += x
            return s / len(v) if v else 0.0

        def p99(v):
            return _percentile(v, 0.99) if v else 0.0
        m = {"name": name, "rate": e.rate, "completed": completed, "throughput_rps": completed / exp.horizon_s,
             "mean_ttft_s": mean(ttft), "p99_ttft_s": p99(ttft), "mean_tpot_s": mean(tpot), "p99_tpot_s": p99(tpot),
             "mean_latency_s": mean(lat), "p99_latency_s": p99(lat),
             "slo_attainment": [met[si] / total if total else 0.0 for si in range(len(scales))]}
        for si in range(len(scales)):
            overall_met[si] += met[si]
        overall_total += total
        weight = e.rate / total_rate if total_rate > 0.0 else 0.0
        report["aggregated_throughput_rps"] += weight * m["throughput_rps"]
        report["llms"].append(m)
    report["overall_slo"] = [overall_met[si] / overall_total if overall_total else 0.0 for si in range(len(scales))]
    return report


def _max_resource_gap(units) -> float:
    """metrics.cpp:115-124."""
    rs = [m.resource_usage for u in units for m in u.llms if m.rate > 0.0]
    gap = 0.0
    for i in range(len(rs)):
        for j in range(i + 1, len(rs)):
            gap = max(gap, abs(rs[i] - rs[j]))
    return gap


def _unit_models(u, names):
    return [{"name": names[m.llm], "rate_rps": m.rate, "avg_used_blocks": m.avg_used_blocks,
             "final_quota_blocks": m.final_quota_blocks, "resource_usage": m.resource_usage} for m in u.llms]


def metrics_json(report: dict, exp: Experiment, units) -> str:
    """report_to_json (metrics.cpp:126-167)."""
    j = {"horizon_s": exp.horizon_s, "aggregated_throughput_rps": report["aggregated_throughput_rps"],
         "slo_scales": list(exp.slo_scales), "overall_slo_attainment": report["overall_slo"],
         "max_resource_gap": _max_resource_gap(units),
         "models": [{"name": m["name"], "rate_rps": m["rate"], "completed": m["completed"],
                     "throughput_rps": m["throughput_rps"], "mean_ttft_s": m["mean_ttft_s"],
                     "p99_ttft_s": m["p99_ttft_s"], "mean_tpot_s": m["mean_tpot_s"], "p99_tpot_s": m["p99_tpot_s"],
                     "mean_latency_s": m["mean_latency_s"], "p99_latency_s": m["p99_latency_s"],
                     "slo_attainment": m["slo_attainment"]} for m in report["llms"]],
         "units": [{"unit": u.unit, "total_blocks": u.total_blocks, "models": _unit_models(u, exp.names)}
                   for u in units]}
    return _dump(j)


def poolstats_json(units, names: list[str]) -> str:
    """poolstats_json (commands.cpp:89-121)."""
    j = {"units": [{"unit": u.unit, "total_blocks": u.total_blocks, "models": _unit_models(u, names),
                    "samples": [{"t_s": t, "llm": names[li], "used_blocks": used, "quota_blocks": quota}
                                for t, li, used, quota in u.samples]} for u in units]}
    return _dump(j)
