"""The acceptance-C1 contention shape (scripts/sched_ablation_realtime.sh)
priced by the engine with the B200 profile (reference decode form, and the
HBM-bound form with the timeline's kappa = 2), beside the real-time
measurements: does the priced engine reproduce the real-time ordering?

    python scripts/sched_ablation_priced.py profiles/r01_scheduler_ablation_realtime.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_02015_b200 as mux  # noqa: E402
from paper_2404_02015_b200 import wire  # noqa: E402
from serve import GIB, make_trace  # noqa: E402


def main(meas_path):
    pj = json.load(open(os.path.join(ROOT, "profiles", "r01_b200_profile_7b.json")))
    prof = pj["profile"]
    ref = [prof[k] for k in wire.PROFILE_KEYS]
    hbm = ref + [pj["profile_hbm"][k] for k in wire.HBM_KEYS]
    hbm[-1] = 0.0  # whole-GPU streams: the SM share is not enforced
    meas = {}
    for line in open(meas_path):
        d = json.loads(line)
        meas[(d["workload"]["gpu_memory_gib"], d["workload"]["scheduler"])] = d["value"]
    specs = [mux.spec("7b", "7b.0"), mux.spec("7b", "7b.1")]
    rates, lengths = (10.0, 80.0), ((128, 384), (64, 64))
    raw = [(t, llm, lengths[llm][0], lengths[llm][1]) for t, llm, _, _ in make_trace(specs, rates, 8.0, 3)]
    trace = [mux.TraceRequest(i, llm, t, p, o) for i, (t, llm, p, o) in enumerate(raw)]
    entries = [mux.Entry(s, r, float(p), float(o)) for s, r, (p, o) in zip(specs, rates, lengths)]
    out = {}
    for mem in (34.0, 40.0):
        for sched, code in (("adbs", 0), ("fcfs", 1), ("rr", 2)):
            row = {"realtime_b200": meas.get((mem, sched))}
            for name, pl, kappa in (("priced_ref_form", ref, 0.1), ("priced_hbm_form_kappa2", hbm, 2.0)):
                params = mux.EngineParams(scheduler=code, kappa=kappa, decode_sm=prof["sm_saturation_point"])
                recs = mux.simulate(entries, trace, mux.Placement([1], [[0, 1]]), int(mem * GIB), params, pl)
                makespan = max(r.done_s for r in recs) - min(r.arrival_s for r in recs)
                row[name] = round(sum(r.output_len for r in trace) / makespan, 1)
            out[f"mem{int(mem)}_{sched}"] = row
            print(mem, sched, row, flush=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r01_scheduler_ablation_priced.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
