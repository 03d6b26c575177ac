#!/bin/bash
# Scheduler ablation with acceptance C1's own parameters (
# /root/reference/proj/tests/acceptance.cpp:100-160, configs/contention.json):
# llm-long 7B 10 rps x 128/384 and llm-short 7B 80 rps x 64/64 (constant
# lengths), seed 42, horizon 40 s, quota period 1.0 s, token budget 768,
# warm-up 8 s. C1's 4 x 7.5 GiB mesh becomes one B200 with the same global
# pool (30 GiB: pool = mem - weights - 10% reserve, sim_engine.cpp:172-186).
# Trace: scripts/c1/trace.csv (reference `muxsim gen-workload`, seed 42).
# Per scheduler: the priced engine (reference cost model) and the real-time
# GPU engine, both through the muxsim_cli drop-in; metrics.json carries the
# reference's aggregated_throughput_rps (rate-weighted) and max_resource_gap.
set -u
cd "$(dirname "$0")/.."
out=${1:-gpurun_out/sched_c1}
mkdir -p $out
for eng in priced realtime; do
  for s in adbs fcfs round_robin; do
    timeout 900 python -m paper_2404_02015_b200.muxsim_cli -c scripts/c1/cfg_$s.json -p scripts/c1/plan.json \
      -t scripts/c1/trace.csv -o $out/${eng}_$s --engine $eng > $out/${eng}_$s.log 2>&1
    python - "$out/${eng}_$s" "$eng" "$s" >> $out/summary.jsonl <<'PY'
import json, sys
d, eng, s = sys.argv[1:]
try:
    m = json.load(open(d + "/metrics.json"))
    rec = [l.split(",") for l in open(d + "/records.csv").read().split("\n")[1:] if l]
    print(json.dumps({"engine": eng, "scheduler": s, "aggregated_throughput_rps": m["aggregated_throughput_rps"],
                      "max_resource_gap": m["max_resource_gap"],
                      "completed": {x["name"]: x["completed"] for x in m["models"]},
                      "mean_ttft_s": {x["name"]: x["mean_ttft_s"] for x in m["models"]},
                      "slo_attainment_x8": m["overall_slo_attainment"]}))
except Exception as e:
    print(json.dumps({"engine": eng, "scheduler": s, "error": str(e)}))
PY
  done
done
cat $out/summary.jsonl
