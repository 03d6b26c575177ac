#!/bin/bash
# CUDA-graph decode jobs: GPU tests, then A/B (MUX_GRAPHS) in decode rounds and real-time serving
out=gpurun_out/r2i; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $out/tests.log
for g in 1 0; do
  for b in 8 128; do
    MUX_GRAPHS=$g python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 0 --e2e-steps 4 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'graphs': $g, 'batch': $b, 'tok_s': d['value'], 'e2e': d['e2e']['value'], 'ms': d['ms_per_step'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
  MUX_GRAPHS=$g python serve.py --rates 120,60 --horizon 3 --realtime 2>/dev/null | tail -1 > $out/serve_rt_$g.json
  MUX_GRAPHS=$g python serve.py --rates 20,10 --horizon 8 --realtime 2>/dev/null | tail -1 > $out/serve_rt_low_$g.json
done
cat $out/tests.log $out/rounds.jsonl; for f in $out/serve_rt_*.json; do echo $f; head -c 330 $f; echo; done
