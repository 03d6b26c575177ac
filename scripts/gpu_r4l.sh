#!/bin/bash
# Serving at 120 + 60 rps (10 s of arrivals) over four arrival seeds at the final HEAD, with clocks
out=gpurun_out/r4l; mkdir -p $out
for seed in 3 4 5 6; do
timeout 600 python serve.py --rates 120,60 --horizon 10 --realtime --seed $seed 2>/dev/null | tail -n 1 > $out/serve_s$seed.json
nvidia-smi --query-gpu=clocks.sm --format=csv,noheader > $out/clk_s$seed.txt
python -c "
import json
d = json.load(open('$out/serve_s$seed.json'))
print(json.dumps({'seed': $seed, 'tok_s': d['value'], 'makespan_s': d['makespan_s'], 'window_tok_s': d['arrival_window']['tok_s'], 'tpot_mean': d['tpot_ms']['mean'], 'ttft_p99': d['ttft_ms']['p99']}))" >> $out/serve_seeds.jsonl
done
cat $out/serve_seeds.jsonl
