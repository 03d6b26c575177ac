#!/bin/bash
# Two weight tiles per activation stage (MUX_GEMM_ST=2): parity, micro, decode rounds
out=gpurun_out/r2p; mkdir -p $out
MUX_GEMM_ST=2 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x -k "gemm or projection or headline" > $out/tests_st2.log 2>&1
for st in 2 1; do
  MUX_GEMM_ST=$st timeout 300 python scripts/gemm_micro.py 128 > $out/micro128_st$st.txt 2>&1
  MUX_GEMM_ST=$st timeout 300 python scripts/gemm_micro.py 32 > $out/micro32_st$st.txt 2>&1
done
for rep in 1 2; do
for cv in 1 0; do
  for b in 32 128; do
    MUX_CARVEOUT=$cv timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'carveout': $cv, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_gbs': d['roofline']['achieved'] if 'gemm' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
for st in 2 1; do
  for b in 32 128; do
    MUX_GEMM_ST=$st timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'st': $st, 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_gbs': d['roofline']['achieved'] if 'gemm' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
tail -3 $out/tests_st2.log; cat $out/rounds.jsonl; for f in $out/micro*; do echo $f; cat $f | awk '{print $2, $5, $6, $7}'; done
timeout 900 python scripts/tp_allreduce_cost.py $out/tp_allreduce.json > $out/tp_allreduce.log 2>&1; tail -8 $out/tp_allreduce.log
