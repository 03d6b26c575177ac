#!/bin/bash
# A/B of the dual-CTA small-batch GEMM (MUX_GEMM_DUAL) in decode rounds and real-time serving
out=gpurun_out/r2h; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x 2>&1 | tail -2 > $out/tests.log
for dual in 1 0 1 0; do
  for b in 8 32 64; do
    MUX_GEMM_DUAL=$dual python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 0 --e2e-steps 0 --partition-sms none 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'dual': $dual, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
for dual in 1 0; do
  MUX_GEMM_DUAL=$dual python serve.py --rates 120,60 --horizon 3 --realtime 2>/dev/null | tail -1 > $out/serve_rt_$dual.json
done
cat $out/tests.log $out/rounds.jsonl; for f in $out/serve_rt_*.json; do echo $f; head -c 400 $f; echo; done
