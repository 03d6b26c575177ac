#!/bin/bash
# pairs for every decode tile (default 16): GPU suite, decode-round sweep, serving x2
out=gpurun_out/r3p; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
tail -1 $out/gpu_suite.log
for b in 8 16 32 64 128; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
done
cat $out/rounds.jsonl
for rep in 1 2; do
  timeout 900 python serve.py --rates 20,10 --horizon 8 --realtime 2>/dev/null | tail -1 > $out/serve_low_$rep.json
  timeout 900 python serve.py --rates 120,60 --horizon 10 --realtime 2>/dev/null | tail -1 > $out/serve_high_$rep.json
done
for f in $out/serve_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['arrival_window']['tok_s'], d['tpot_ms']['mean'], d['ttft_ms']['mean'])"; done
