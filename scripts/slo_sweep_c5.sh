#!/bin/bash
# f3: SLO-attainment sweep of config 5 (19 LLMs, 7B-65B, power-law alpha 0.9)
# over four arrival-rate levels (scripts/c5, made by scripts/c5/make_c5.py
# with the unmodified reference planner). Per level: the priced engine (the
# reference's pricing with the B200-measured profile) and the real-time GPU
# engine through the muxsim_cli drop-in; every unit of the 8-GPU plan runs on
# its own GPU (one after another on a smaller box). metrics.json carries the
# reference's SLO attainment per scale (metrics.cpp:42-109).
set -u
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/slo_c5}
engines=${2:-"priced realtime"}
mkdir -p $out
for r in 5 10 20 40; do
  for eng in $engines; do
    timeout 1800 python -m paper_2404_02015_b200.muxsim_cli -c scripts/c5/cfg_r$r.json -p scripts/c5/plan_r$r.json \
      -t scripts/c5/trace_r$r.csv -o $out/${eng}_r$r --engine $eng > $out/${eng}_r$r.log 2>&1
    python - "$out/${eng}_r$r" "$eng" "$r" >> $out/summary.jsonl <<'PY'
import json, sys
d, eng, r = sys.argv[1:]
try:
    m = json.load(open(d + "/metrics.json"))
    print(json.dumps({"engine": eng, "max_rate_rps": float(r), "requests": sum(x["completed"] for x in m["models"]),
                      "aggregated_throughput_rps": m["aggregated_throughput_rps"],
                      "slo_attainment": m["overall_slo_attainment"],
                      "per_model_p99_latency_s": {x["name"]: x.get("p99_latency_s") for x in m["models"]}}))
except Exception as e:
    print(json.dumps({"engine": eng, "max_rate_rps": float(r), "error": str(e)}))
PY
  done
done
cat $out/summary.jsonl
