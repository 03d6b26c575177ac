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
# B200 extension: the measured tensor-parallel allreduce in place of
# tp_speedup = eta * tp (LatencyProfile::tp_scaled, f1). Both keys or none.
TP_KEYS = ["allreduce_alpha_ms", "allreduce_ms_per_mib"]
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


def _fail(msg):
    raise ConfigError("config: " + msg)


def _check_keys(obj, ctx, allowed):
    """config.cpp:28-39: unknown keys are errors."""
    for k in obj:
        if k not in allowed:
            _fail(f"unknown key '{k}' in {ctx}")


def _is_num(v):
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _num(obj, ctx, key, default=None, required=False):
    if key not in obj:
        if required:
            _fail(f"{ctx} is missing required key '{key}'")
        return default
    v = obj[key]
    if not _is_num(v):
        _fail(f"{ctx}.{key} must be a number")
    return float(v)


def _int(obj, ctx, key, default=None, required=False):
    if key not in obj:
        if required:
            _fail(f"{ctx} is missing required key '{key}'")
        return default
    v = obj[key]
    if not isinstance(v, int) or isinstance(v, bool):
        _fail(f"{ctx}.{key} must be an integer")
    return int(v)


def _num_list(v, where):
    if not isinstance(v, list):
        _fail(f"{where} must be an array of numbers")
    for e in v:
        if not _is_num(e):
            _fail(f"{where} element must be a number")
    return [float(e) for e in v]


def _mean_len(d, ctx):
    """parse_dist (config.cpp:106-125) + LengthDist::mean (workload.cpp:66-76):
    the empirical mean is weighted."""
    if not isinstance(d, dict):
        _fail(f"{ctx} must be an object with a 'kind'")
    if "kind" not in d:
        _fail(f"{ctx} is missing required key 'kind'")
    kind = d["kind"]
    if not isinstance(kind, str):
        _fail(f"{ctx}.kind must be a string")
    if kind == "constant":
        _check_keys(d, ctx, ("kind", "value"))
        v = _num(d, ctx, "value", required=True)
        if not v >= 1.0:
            raise ConfigError("length dist: constant value must be >= 1")
        return v
    if kind == "lognormal":
        _check_keys(d, ctx, ("kind", "mean", "sigma"))
        mean = _num(d, ctx, "mean", required=True)
        sigma = _num(d, ctx, "sigma", 0.8)
        if not mean >= 1.0:
            raise ConfigError("length dist: lognormal mean must be >= 1")
        if not sigma >= 0.0:
            raise ConfigError("length dist: sigma must be >= 0")
        return mean
    if kind == "empirical":
        _check_keys(d, ctx, ("kind", "values", "weights"))
        if "values" not in d:
            _fail(f"{ctx} is missing required key 'values'")
        if "weights" not in d:
            _fail(f"{ctx} is missing required key 'weights'")
        vals = _num_list(d["values"], ctx + ".values")
        ws = _num_list(d["weights"], ctx + ".weights")
        if not vals or len(vals) != len(ws):
            raise ConfigError("length dist: empirical values/weights must be non-empty and equal length")
        total = acc = 0.0
        for v, w in zip(vals, ws):
            if not v >= 1.0:
                raise ConfigError("length dist: empirical values must be >= 1")
            if not w >= 0.0:
                raise ConfigError("length dist: empirical weights must be >= 0")
        for v, w in zip(vals, ws):  # workload.cpp:70-75, same summation order
            total += w
            acc += v * w
        if not total > 0.0:
            raise ConfigError("length dist: empirical weights must not all be zero")
        return acc / total
    _fail(f"{ctx}.kind must be constant, lognormal, or empirical")


def gen_rates(n, alpha, max_rate):
    """workload.cpp:78-86."""
    if n < 1 or not alpha >= 0.0 or not max_rate > 0.0:
        raise ConfigError("power_law: need n >= 1, alpha >= 0, max_rate_rps > 0")
    return [max_rate * (i + 1) ** (-alpha) for i in range(n)]


def load_config(path: str, catalog: dict[str, LLMSpec] | None = None) -> Experiment:
    """parse_config (config.cpp:260-321) over the keys the engine consumes,
    with the reference's key, type and range checks (ConfigError = CLI exit 1)."""
    catalog = catalog or CATALOG
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        _fail(f"cannot open '{path}'")
    try:
        root = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(f"invalid JSON: {e}")
    if not isinstance(root, dict):
        _fail("top level must be an object")
    _check_keys(root, "config", ("cluster", "llms", "workload", "placement", "profile", "sim", "metrics",
                                 "ablate", "outputs"))
    if "cluster" not in root:
        _fail("config is missing required key 'cluster'")
    cl = root["cluster"]
    if not isinstance(cl, dict):
        _fail("cluster must be an object")
    _check_keys(cl, "cluster", ("num_nodes", "gpus_per_node", "gpu_memory_gb"))
    num_nodes = _int(cl, "cluster", "num_nodes", required=True)
    gpn = _int(cl, "cluster", "gpus_per_node", required=True)
    gb = _num(cl, "cluster", "gpu_memory_gb", required=True)
    if gb <= 0.0:
        _fail("cluster.gpu_memory_gb must be positive")
    if num_nodes < 1 or gpn < 1:
        _fail("cluster: num_nodes and gpus_per_node must be >= 1")
    mem = int(round(gb * GIB))  # llround(gb * 2^30) (config.cpp:141)
    if "llms" not in root:
        _fail("config is missing required key 'llms'")
    llms = root["llms"]
    if not isinstance(llms, list) or not llms:
        _fail("llms must be a non-empty array")
    names, entries, seen = [], [], set()
    for i, m in enumerate(llms):
        ctx = f"llms[{i}]"
        if not isinstance(m, dict):
            _fail(ctx + " must be an object")
        _check_keys(m, ctx, ("name", "model", "rate_rps", "prompt_len", "output_len"))
        for k in ("name", "model"):
            if k not in m:
                _fail(f"{ctx} is missing required key '{k}'")
            if not isinstance(m[k], str):
                _fail(f"{ctx}.{k} must be a string")
        name, model = m["name"], m["model"]
        if not name or "," in name:
            _fail(ctx + ".name must be non-empty and comma-free")
        if name in seen:
            _fail(f"duplicate model name '{name}'")
        seen.add(name)
        if model not in catalog:
            _fail(f"{ctx}.model '{model}' is not in the catalog ({', '.join(catalog)})")
        rate = _num(m, ctx, "rate_rps", 0.0)
        if rate < 0.0:
            _fail(ctx + ".rate_rps must be >= 0")
        spec = catalog[model]
        names.append(name)
        # LlmConfig defaults: constant 128 prompt / 64 output (config.hpp:26-27)
        mp = _mean_len(m["prompt_len"], ctx + ".prompt_len") if "prompt_len" in m else 128.0
        mo = _mean_len(m["output_len"], ctx + ".output_len") if "output_len" in m else 64.0
        entries.append(Entry(LLMSpec(name, spec.num_layers, spec.num_heads, spec.head_dim, spec.hidden_size,
                                     spec.weight_bytes, spec.bytes_per_element, spec.ffn, spec.vocab),
                             rate, mp, mo))
    horizon, seed = 60.0, 0
    wl = root.get("workload")
    if wl is not None:
        if not isinstance(wl, dict):
            _fail("workload must be an object")
        _check_keys(wl, "workload", ("horizon_s", "seed", "power_law"))
        horizon = _num(wl, "workload", "horizon_s", horizon)
        if horizon <= 0.0:
            _fail("workload.horizon_s must be positive")
        seed = _int(wl, "workload", "seed", 0)
        if seed < 0:
            _fail("workload.seed must be >= 0")
        if "power_law" in wl:
            pl = wl["power_law"]
            if not isinstance(pl, dict):
                _fail("workload.power_law must be an object")
            _check_keys(pl, "workload.power_law", ("alpha", "max_rate_rps"))
            alpha = _num(pl, "workload.power_law", "alpha", required=True)
            mx = _num(pl, "workload.power_law", "max_rate_rps", required=True)
            if alpha < 0.0:
                _fail("workload.power_law.alpha must be >= 0")
            if mx <= 0.0:
                _fail("workload.power_law.max_rate_rps must be positive")
            for e, r in zip(entries, gen_rates(len(entries), alpha, mx)):
                e.rate = r
    pc = root.get("placement")
    if pc is not None:
        if not isinstance(pc, dict):
            _fail("placement must be an object")
        _check_keys(pc, "placement", ("backend", "sm_list", "tp_list", "max_batch", "max_ilp_dims"))
        if pc.get("backend", "greedy") not in ("greedy", "ilp"):
            _fail("placement.backend must be greedy or ilp")
    prof = list(PROFILE_DEFAULTS)
    hbm, tpk = {}, {}
    pr = root.get("profile")
    if pr is not None:
        if not isinstance(pr, dict):
            _fail("profile must be an object")
        _check_keys(pr, "profile", PROFILE_KEYS + HBM_KEYS + TP_KEYS)
        for k in pr:
            v = _num(pr, "profile", k)
            if k in HBM_KEYS:
                hbm[k] = v
            elif k in TP_KEYS:
                tpk[k] = v
            else:
                prof[PROFILE_KEYS.index(k)] = v
    if hbm:
        if len(hbm) != len(HBM_KEYS):
            raise ConfigError("profile: the HBM decode form needs " + ", ".join(HBM_KEYS))
        prof += [hbm[k] for k in HBM_KEYS]
    if tpk:
        if len(tpk) != len(TP_KEYS):
            raise ConfigError("profile: the measured TP allreduce needs " + ", ".join(TP_KEYS))
        if min(tpk.values()) < 0.0:
            _fail("latency profile: allreduce terms must be >= 0")
        prof += [tpk[k] for k in TP_KEYS]
    # LatencyProfile::validate (cost_model.cpp:49-59), reported as ConfigError
    pp, db, dc, tpe, sat, knee, rs = prof[:7]
    if not (pp > 0.0 and db > 0.0 and dc >= 0.0):
        _fail("latency profile: coefficients must be positive")
    if not (tpe > 0.5 and tpe <= 1.0):
        _fail("latency profile: tp_efficiency must be in (0.5, 1]")
    if not (sat > 0.0 and sat <= 1.0):
        _fail("latency profile: sm_saturation_point must be in (0, 1]")
    if not knee >= 1.0:
        _fail("latency profile: batch_knee must be >= 1")
    if not rs > 0.0:
        _fail("latency profile: reference_scale must be positive")
    p = EngineParams()
    sim = root.get("sim")
    decode_sm_set = False
    tp_one = False
    if sim is not None:
        if not isinstance(sim, dict):
            _fail("sim must be an object")
        _check_keys(sim, "sim", ("scheduler", "kappa", "quota_period_s", "token_budget", "block_tokens",
                                 "warmup_s", "decode_sm", "prefill_min_sm", "activation_reserve_frac",
                                 "quota_floor_frac", "quota_low_mark", "quota_high_mark", "quota_step_frac",
                                 "slo_reference_tp_one"))
        if "scheduler" in sim:
            sched = sim["scheduler"]
            if sched not in ("adbs", "fcfs", "round_robin"):
                _fail("sim.scheduler must be adbs, fcfs, or round_robin")
            p.scheduler = SCHEDULERS[sched]
        for k in ("kappa", "quota_period_s", "warmup_s", "decode_sm", "prefill_min_sm", "activation_reserve_frac",
                  "quota_floor_frac"):
            setattr(p, k, _num(sim, "sim", k, getattr(p, k)))
        p.quota_low_mark = _num(sim, "sim", "quota_low_mark", p.quota_low_mark)
        p.quota_high_mark = _num(sim, "sim", "quota_high_mark", p.quota_high_mark)
        p.quota_step_frac = _num(sim, "sim", "quota_step_frac", p.quota_step_frac)
        for k in ("token_budget", "block_tokens"):
            setattr(p, k, _int(sim, "sim", k, getattr(p, k)))
        decode_sm_set = "decode_sm" in sim
        if "slo_reference_tp_one" in sim:
            if not isinstance(sim["slo_reference_tp_one"], bool):
                _fail("sim.slo_reference_tp_one must be a boolean")
            tp_one = sim["slo_reference_tp_one"]
        if p.kappa < 0.0:
            _fail("sim.kappa must be >= 0")
        if p.quota_period_s <= 0.0:
            _fail("sim.quota_period_s must be positive")
        if p.token_budget < 1:
            _fail("sim.token_budget must be >= 1")
        if p.block_tokens < 1:
            _fail("sim.block_tokens must be >= 1")
        if p.warmup_s < 0.0:
            _fail("sim.warmup_s must be >= 0")
        if p.decode_sm <= 0.0 or p.decode_sm > 1.0:
            _fail("sim.decode_sm must be in (0, 1]")
        if p.prefill_min_sm <= 0.0 or p.prefill_min_sm > 1.0:
            _fail("sim.prefill_min_sm must be in (0, 1]")
        if p.activation_reserve_frac < 0.0 or p.activation_reserve_frac >= 1.0:
            _fail("sim.activation_reserve_frac must be in [0, 1)")
    if not decode_sm_set:
        p.decode_sm = prof[PROFILE_KEYS.index("sm_saturation_point")]
    exp = Experiment(num_nodes, gpn, mem, names, entries, p, prof, horizon, seed, {"root": root})
    met = root.get("metrics")
    if met is not None:
        if not isinstance(met, dict):
            _fail("metrics must be an object")
        _check_keys(met, "metrics", ("slo_scales",))
        if "slo_scales" in met:
            scales = _num_list(met["slo_scales"], "metrics.slo_scales")
            if not scales:
                _fail("metrics.slo_scales must be non-empty")
            if any(x <= 0.0 for x in scales):
                _fail("metrics.slo_scales entries must be positive")
            exp.slo_scales = scales
    ab = root.get("ablate")
    if ab is not None:
        if not isinstance(ab, dict):
            _fail("ablate must be an object")
        _check_keys(ab, "ablate", ("rate_scales",))
        if "rate_scales" in ab:
            rsc = _num_list(ab["rate_scales"], "ablate.rate_scales")
            if not rsc or any(x <= 0.0 for x in rsc):
                _fail("ablate.rate_scales must be non-empty with positive entries")
    out = root.get("outputs")
    if out is not None:
        if not isinstance(out, dict):
            _fail("outputs must be an object")
        _check_keys(out, "outputs", ("trace", "plan", "dir", "sweep"))
    exp.slo_reference_tp_one = bool(tp_one)
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
    sizes, members, tp, gpus = [], [], {}, []
    for u in root["units"]:
        if not isinstance(u, dict) or not isinstance(u.get("gpu_ids"), list):
            raise ConfigError("plan: each unit needs a gpu_ids array")
        sizes.append(len(u["gpu_ids"]))
        gpus.append([int(g) for g in u["gpu_ids"]])
        mem = []
        for m in u.get("models", []):
            if m.get("name") not in names:
                raise ConfigError(f"plan: model '{m.get('name')}' is not in the config")
            mem.append(names.index(m["name"]))
            tp[names.index(m["name"])] = int(m.get("tp_degree", len(u["gpu_ids"])))  # commands.cpp:205
        members.append(mem)
    return Placement(sizes, members, tp_degree=tp, gpu_ids=gpus)


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
