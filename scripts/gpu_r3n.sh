#!/bin/bash
# CTA pairs for small decode tiles (MUX_GEMM_PAIR_MIN_TILE 32) vs the two-CTAs-per-SM form (80, default)
out=gpurun_out/r3n; mkdir -p $out
MUX_GEMM_PAIR_MIN_TILE=32 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x -k "gemm or projection" > $out/tests.log 2>&1
tail -1 $out/tests.log
for rep in 1 2; do
for pm in 32 80; do
  for b in 16 32 64; do
    MUX_GEMM_PAIR_MIN_TILE=$pm timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'pair_min': $pm, 'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
cat $out/rounds.jsonl
