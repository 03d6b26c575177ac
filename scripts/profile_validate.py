"""Does the measured latency profile (calibrate.py) make the
priced engine track real serving? One trace (serve.py's 7B + 13B workload),
runs: measured on the B200 (completions at device time), priced with the
reference's default LatencyProfile, priced with the calibrated profile in the
reference's decode form, and (when the profile holds wire.HBM_KEYS) priced
with the HBM-bound decode form.

    python scripts/profile_validate.py gpurun_out/b200_profile_7b.json [--rates 20,10 --horizon 8]
    # CPU only, against a stored measured run of the same trace:
    python scripts/profile_validate.py P.json --measured-from profiles/r01_profile_validation.json:low_load
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_02015_b200 as mux  # noqa: E402
from paper_2404_02015_b200 import wire  # noqa: E402
from serve import GIB, make_trace  # noqa: E402


def summary(recs, trace):
    out_tokens = sum(r.output_len for r in trace)
    first = min(r.arrival_s for r in recs)
    makespan = max(r.done_s for r in recs) - first
    tpot = [(r.done_s - r.first_token_s) / max(1, r.output_len - 1) for r in recs]
    ttft = [r.first_token_s - r.arrival_s for r in recs]
    return {"tok_per_s": round(out_tokens / makespan, 1), "makespan_s": round(makespan, 3),
            "tpot_ms_mean": round(1e3 * sum(tpot) / len(tpot), 3), "ttft_ms_mean": round(1e3 * sum(ttft) / len(ttft), 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("profile")
    ap.add_argument("--models", default="7b,13b")
    ap.add_argument("--rates", default="20,10")
    ap.add_argument("--horizon", type=float, default=8.0)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--kappa", type=float, default=None,
                    help="interference coefficient of the priced runs with the calibrated profile (sim_engine.cpp:16-18)")
    ap.add_argument("--hbm-sm-exponent", type=float, default=None,
                    help="override decode_sm_exponent of the HBM-form run (0: jobs on whole-GPU streams, "
                         "where the SM share is not enforced)")
    ap.add_argument("--measured-from", default=None,
                    help="FILE:KEY of an earlier output whose measured_b200 summary (same trace) is reused")
    a = ap.parse_args()
    pj = json.load(open(a.profile))
    prof = dict(pj["profile"], **pj.get("profile_hbm", {}))
    prof_list = [prof[k] for k in wire.PROFILE_KEYS]
    models = a.models.split(",")
    rates = [float(x) for x in a.rates.split(",")]
    specs = [mux.spec(m, f"{m}.{i}") for i, m in enumerate(models)]
    raw = make_trace(specs, rates, a.horizon, a.seed)
    trace = [mux.TraceRequest(i, llm, t, p, o) for i, (t, llm, p, o) in enumerate(raw)]
    entries = [mux.Entry(s, r, 161.0, 338.0) for s, r in zip(specs, rates)]
    gpu_mem = int(180 * GIB)
    placement = mux.Placement([1], [list(range(len(specs)))])
    out = {"workload": {"models": models, "rates_rps": rates, "horizon_s": a.horizon, "requests": len(trace)},
           "profile": prof}
    variants = [("priced_default", None), ("priced_b200", prof_list)]
    if all(k in prof for k in wire.HBM_KEYS):
        hbm = [prof[k] for k in wire.HBM_KEYS]
        if a.hbm_sm_exponent is not None:
            hbm[wire.HBM_KEYS.index("decode_sm_exponent")] = a.hbm_sm_exponent
        variants.append(("priced_b200_hbm", prof_list + hbm))
    for name, pl in variants:
        params = mux.EngineParams()
        if pl is not None:
            params.decode_sm = prof["sm_saturation_point"]  # config.cpp:277: decode_sm defaults to f_sat
            if a.kappa is not None:
                params.kappa = a.kappa
        recs = mux.simulate(entries, trace, placement, gpu_mem, params, pl)
        out[name] = summary(recs, trace)
    if a.measured_from:
        path, key = a.measured_from.rsplit(":", 1)
        old = json.load(open(path))[key]
        if old["workload"]["requests"] != len(trace):
            raise SystemExit("--measured-from: a different trace")
        out["measured_b200"] = old["measured_b200"]
        out["measured_b200"]["from"] = a.measured_from
    else:
        weights = sum(s.weight_bytes for s in specs)
        logical = (gpu_mem - weights - round(0.1 * gpu_mem)) // 4096
        unit = mux.Unit(specs, pool_blocks=logical, device_pool_blocks=logical, max_batch=512,
                        max_prefill_tokens=4096, max_ctx=2048 + 64, max_slots=len(trace) + 8, init_seed=1,
                        init_std=0.02, partitions=len(specs) + 1)
        try:
            unit.init_kv(seed=5, std=1.0)
            recs, _ = unit.run_lockstep(entries, trace, gpu_mem, mux.EngineParams(), measured=True)
        finally:
            unit.close()
        out["measured_b200"] = summary(recs, trace)
    m = out["measured_b200"]
    for name, _ in variants:
        out[name]["tok_per_s_vs_measured"] = round(out[name]["tok_per_s"] / m["tok_per_s"], 3)
        out[name]["tpot_vs_measured"] = round(out[name]["tpot_ms_mean"] / m["tpot_ms_mean"], 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
