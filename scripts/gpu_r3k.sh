#!/bin/bash
# Real-time serving sweep over offered load (7B + 13B, ShareGPT lengths, 10 s of arrivals)
out=gpurun_out/r3k; mkdir -p $out
for r in "10,5" "20,10" "40,20" "60,30" "120,60"; do
  timeout 1200 python serve.py --rates $r --horizon 10 --realtime 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'rates': '$r', 'requests': d['requests'], 'tok_s': d['value'], 'window_tok_s': d['arrival_window']['tok_s'], 'req_per_s': d['req_per_s'], 'ttft_ms': d['ttft_ms'], 'tpot_ms': d['tpot_ms'], 'makespan_s': d['makespan_s']}))" >> $out/serve_sweep.jsonl
done
cat $out/serve_sweep.jsonl
