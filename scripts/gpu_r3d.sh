#!/bin/bash
# P1: real-time serving with every ADBS job on an SM run sized by its sm_demand (sm_route) vs whole-GPU streams
out=gpurun_out/r3d; mkdir -p $out
for r in "120,60 6" "20,10 8"; do
  set -- $r
  for sr in 1 0; do
    flag=""; [ $sr = 1 ] && flag="--sm-route"
    timeout 900 python serve.py --rates $1 --horizon $2 --realtime $flag 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'rates': '$1', 'horizon': $2, 'sm_route': $sr, 'tok_s': d['value'], 'window_tok_s': (d.get('arrival_window') or {}).get('tok_s'), 'ttft_ms': d['ttft_ms'], 'tpot_ms': d['tpot_ms'], 'makespan_s': d['makespan_s']}))" >> $out/serve_sm_route.jsonl
  done
done
cat $out/serve_sm_route.jsonl
