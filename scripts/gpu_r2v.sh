#!/bin/bash
# Decode QKV as fp32 sums (option qkv_f32, no stream-K fixup): full GPU suite with it on, A/B in decode rounds
out=gpurun_out/r2v; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/gpu_suite.log 2>&1
tail -3 $out/gpu_suite.log
timeout 300 python -m pytest tests/test_gpu_headline.py -q -s -k tokens 2>&1 | grep -E "parity|passed|failed" > $out/headline_rate.log
cat $out/headline_rate.log
for rep in 1 2; do
for q in 1 0; do
  for b in 16 64 128; do
    MUX_QKV_F32=$q timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'qkv_f32': $q, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
cat $out/rounds.jsonl
