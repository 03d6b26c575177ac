#!/bin/bash
# C1 scheduler ablation through the priced engine with the B200-measured
# profile (reference form + HBM decode form, profiles/r01_b200_profile_7b.json)
# at kappa 0.1 (reference default) and 2.0 (timeline-measured in round 1).
set -u
cd "$(dirname "$0")/.."
out=${1:-/tmp/c1_priced_b200}
mkdir -p $out
for kappa in 0.1 2.0; do
  for s in adbs fcfs round_robin; do
    python - "$s" "$kappa" "$out" <<'PY'
import json, sys
s, kappa, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
cfg = json.load(open(f"scripts/c1/cfg_{s}.json"))
prof = json.load(open("profiles/r01_b200_profile_7b.json"))
cfg["profile"] = dict(prof["profile"], **prof["profile_hbm"])
cfg["sim"]["kappa"] = kappa
json.dump(cfg, open(f"{out}/cfg_{s}_{kappa}.json", "w"), indent=1)
PY
    python -m paper_2404_02015_b200.muxsim_cli -c $out/cfg_${s}_$kappa.json -p scripts/c1/plan.json -t scripts/c1/trace.csv \
      -o $out/out_${s}_$kappa --engine priced > /dev/null
    python -c "
import json; m=json.load(open('$out/out_${s}_$kappa/metrics.json'))
print(json.dumps({'engine': 'priced (B200 profile)', 'kappa': $kappa, 'scheduler': '$s', 'aggregated_throughput_rps': m['aggregated_throughput_rps'], 'max_resource_gap': m['max_resource_gap'], 'completed': {x['name']: x['completed'] for x in m['models']}}))"
  done
done
