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
  rates         /root/reference/proj/src/workload.cpp:78-86 gen_rates
The engine itself is libmux.so (priced: mux_simulate, bit-identical to the
reference; lockstep / measured: a GPU unit).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

from .host import CATALOG, EngineParams, Entry, LLMSpec, Placement, TraceRequest

GIB = 1 << 30

# LatencyProfile fields in declaration order (cost_model.hpp:33-40)
PROFILE_KEYS = ["prefill_ms_per_token", "decode_base_ms", "decode_ctx_ms_per_token", "tp_efficiency",
                "sm_saturation_point", "batch_knee", "reference_scale"]
PROFILE_DEFAULTS = [0.25, 12.0, 0.005, 0.9, 0.5, 16.0, 32.0 * 4096.0]
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
    horizon_s: float = 0.0
    seed: int = 0
    extra: dict = field(default_factory=dict)


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
    for k, v in (root.get("profile") or {}).items():
        if k not in PROFILE_KEYS:
            raise ConfigError(f"profile: unknown key '{k}'")
        prof[PROFILE_KEYS.index(k)] = float(v)
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
    return Experiment(num_nodes, gpn, mem, names, entries, p, prof, float(wl.get("horizon_s", 0.0)),
                      int(wl.get("seed", 0)), {"root": root})


def load_plan(path: str, names: list[str]) -> Placement:
    """plan.json -> units (mesh size = len(gpu_ids)) and their members."""
    with open(path) as f:
        try:
            root = json.load(f)
        except json.JSONDecodeError as e:
            raise ConfigError(f"plan: invalid JSON: {e}") from None
    if not isinstance(root, dict) or not isinstance(root.get("units"), list):
        raise ConfigError("plan: expected an object with a 'units' array")
    sizes, members = [], []
    for u in root["units"]:
        if not isinstance(u, dict) or not isinstance(u.get("gpu_ids"), list):
            raise ConfigError("plan: each unit needs a gpu_ids array")
        sizes.append(len(u["gpu_ids"]))
        mem = []
        for m in u.get("models", []):
            if m.get("name") not in names:
                raise ConfigError(f"plan: model '{m.get('name')}' is not in the config")
            mem.append(names.index(m["name"]))
        members.append(mem)
    return Placement(sizes, members)


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
