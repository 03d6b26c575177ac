#!/bin/bash
# Decode GEMM on CTA pairs (MUX_GEMM_PAIR=1): parity first, then micro + decode rounds
out=gpurun_out/r2r; mkdir -p $out
MUX_GEMM_PAIR=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > $out/tests_pair_kernels.log 2>&1
echo "kernels rc=$?" >> $out/status.txt
tail -3 $out/tests_pair_kernels.log
if grep -q " passed" $out/tests_pair_kernels.log && ! grep -q "failed" $out/tests_pair_kernels.log; then
  MUX_GEMM_PAIR=1 timeout 900 python -m pytest tests/test_gpu_headline.py -q -x > $out/tests_pair_headline.log 2>&1
  tail -3 $out/tests_pair_headline.log
  for pr in 1 0; do
    MUX_GEMM_PAIR=$pr timeout 300 python scripts/gemm_micro.py 128 > $out/micro128_pair$pr.txt 2>&1
  done
  for rep in 1 2; do
  for pr in 1 0; do
    for b in 96 128; do
      MUX_GEMM_PAIR=$pr timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'pair': $pr, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_gbs': d['roofline']['achieved'] if 'gemm' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
    done
  done
  done
  cat $out/rounds.jsonl; for f in $out/micro*; do echo $f; cat $f | awk '{print $2, $5, $6, $7}'; done
fi
