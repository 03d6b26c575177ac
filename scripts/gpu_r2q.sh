#!/bin/bash
# ST auto policy: parity + micro + decode rounds (auto vs off), then the full GPU suite
out=gpurun_out/r2q; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x -k "gemm or projection or headline" > $out/tests_auto.log 2>&1
for st in 0 1; do
  MUX_GEMM_ST=$st timeout 300 python scripts/gemm_micro.py 128 > $out/micro128_st$st.txt 2>&1
done
for rep in 1 2 3; do
for st in 0 1; do
  for b in 96 128; do
    MUX_GEMM_ST=$st timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'st': $st, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_gbs': d['roofline']['achieved'] if 'gemm' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
timeout 1500 python -m pytest tests -m gpu -q -x > $out/gpu_suite.log 2>&1
tail -3 $out/tests_auto.log; cat $out/rounds.jsonl; for f in $out/micro*; do echo $f; cat $f | awk '{print $2, $5, $6, $7}'; done; tail -3 $out/gpu_suite.log
