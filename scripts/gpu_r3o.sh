#!/bin/bash
# pairs from 32-token tiles by default; 16-token tiles on pairs as an A/B; full suite
out=gpurun_out/r3o; mkdir -p $out
MUX_GEMM_PAIR_MIN_TILE=16 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x -k "gemm or projection" > $out/tests16.log 2>&1
tail -1 $out/tests16.log
for rep in 1 2; do
for pm in 16 32; do
  for b in 8 16; do
    MUX_GEMM_PAIR_MIN_TILE=$pm timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'pair_min': $pm, 'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
cat $out/rounds.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
tail -1 $out/gpu_suite.log
timeout 900 python serve.py --rates 20,10 --horizon 8 --realtime 2>/dev/null | tail -1 > $out/serve_low.json
timeout 900 python serve.py --rates 120,60 --horizon 10 --realtime 2>/dev/null | tail -1 > $out/serve_high.json
python -c "
import json
for f in ('serve_low', 'serve_high'):
    d = json.load(open('$out/' + f + '.json')); print(f, d['value'], d['arrival_window'], d['tpot_ms'])"
