#!/bin/bash
# pair + two-tile units on residual projections (MUX_GEMM_PAIR_ST=1): parity, micro, decode rounds
out=gpurun_out/r3u; mkdir -p $out
MUX_GEMM_PAIR_ST=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py tests/test_gpu_model.py -q -x > $out/tests.log 2>&1
tail -1 $out/tests.log
for ps in 1 0; do
  MUX_GEMM_PAIR_ST=$ps timeout 300 python scripts/gemm_micro.py 128 > $out/micro_$ps.txt 2>&1
done
for rep in 1 2; do
for ps in 1 0; do
  for b in 64 128; do
    MUX_GEMM_PAIR_ST=$ps timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'pair_st': $ps, 'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
cat $out/rounds.jsonl; for f in $out/micro_*; do echo $f; grep -E "down|o7|o13" $f | cut -c1-100; done
