#!/bin/bash
# decode rounds at batch 128: residual-epilogue stream-K minimum range (MUX_GEMM_RES_MIN_ITERS) sweep, alternating
out=gpurun_out/r4m; mkdir -p $out
for rep in 1 2; do
for v in 8 4 16 32; do
  MUX_GEMM_RES_MIN_ITERS=$v timeout 300 python bench.py --batch 128 --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'res_min_iters': $v, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
done
done
cat $out/rounds.jsonl
