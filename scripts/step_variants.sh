#!/bin/bash
# Step time of the cfg2 decode round under variants (no cpu / e2e / serving legs).
# usage: step_variants.sh "label|ENV=v ...|extra bench args" ...
for v in "$@"; do
  IFS='|' read -r label envs args <<< "$v"
  out=$(env $envs python bench.py --skip-cpu --e2e-steps 0 --attn-steps 0 --serve-horizon 0 $args 2>&1 | tail -1)
  res=$(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], 'ms', d['value'], 'tok/s', d['step_roofline']['frac'], 'sm_mhz', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), 'jobs', d['config'].get('job_ms_per_step'))" 2>/dev/null)
  echo "$label: ${res:-$out}"
done
