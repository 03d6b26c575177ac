"""Priced engine with a calibrated B200 profile against REAL-TIME serving
runs of the same trace (serve.py --realtime output JSON): tok/s and mean
TPOT ratios for the reference decode form and the HBM decode form at the
given interference coefficients (sim_engine.cpp:16-18).

    python scripts/profile_validate_rt.py profiles/r02_b200_profile_7b.json RUN.json [RUN2.json ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import paper_2404_02015_b200 as mux  # noqa: E402
from paper_2404_02015_b200 import wire  # noqa: E402
from profile_validate import summary  # noqa: E402
from serve import GIB, make_trace  # noqa: E402


def main():
    pj = json.load(open(sys.argv[1]))
    prof = dict(pj["profile"], **pj.get("profile_hbm", {}))
    base = [prof[k] for k in wire.PROFILE_KEYS]
    hbm = [prof[k] for k in wire.HBM_KEYS]
    hbm[wire.HBM_KEYS.index("decode_sm_exponent")] = 0.0  # the real-time runs use whole-GPU streams
    out = []
    for path in sys.argv[2:]:
        rt = json.load(open(path))
        w = rt["workload"]
        specs = [mux.spec(m, f"{m}.{i}") for i, m in enumerate(w["models"])]
        raw = make_trace(specs, w["rates_rps"], w["horizon_s"], w["seed"])
        trace = [mux.TraceRequest(i, llm, t, p, o) for i, (t, llm, p, o) in enumerate(raw)]
        entries = [mux.Entry(s, r, 161.0, 338.0) for s, r in zip(specs, w["rates_rps"])]
        placement = mux.Placement([1], [list(range(len(specs)))])
        row = {"run": os.path.basename(path), "rates_rps": w["rates_rps"], "horizon_s": w["horizon_s"],
               "realtime": {"tok_per_s": rt["value"], "tpot_ms_mean": rt["tpot_ms"]["mean"]}}
        for form, pl in (("reference_form", base), ("hbm_form", base + hbm)):
            for kappa in (0.1, 2.0):
                params = mux.EngineParams()
                params.decode_sm = prof["sm_saturation_point"]
                params.kappa = kappa
                recs = mux.simulate(entries, trace, placement, int(180 * GIB), params, pl)
                s = summary(recs, trace)
                row[f"{form}_kappa{kappa}"] = {"tok_per_s": s["tok_per_s"], "tpot_ms_mean": s["tpot_ms_mean"],
                                               "tok_s_vs_realtime": round(s["tok_per_s"] / rt["value"], 3),
                                               "tpot_vs_realtime": round(s["tpot_ms_mean"] / rt["tpot_ms"]["mean"], 3)}
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
