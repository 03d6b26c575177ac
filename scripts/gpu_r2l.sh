#!/bin/bash
# Measurement call: launch list (graphs off, ncu cannot prepare kernels next to
# a capture), ncu --set full of one decode GEMM and one K1 launch, compute-sanitizer
# racecheck/synccheck over K1/K3/GEMM tests, bench with the e2e warm-up, C1 ablation.
out=gpurun_out/r2l; mkdir -p $out
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
MUX_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 > $out/ncu_bench.log 2>&1
gzip -f $out/launches.csv
# one 13B gate-up GEMM (N=27648, K=5120) and one 13B K1 in the concurrent bench step
MUX_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -s 1500 -c 6 \
  -o $out/gemm_full python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 --partition-sms none > $out/ncu_gemm.log 2>&1
for t in "test_decode_attention_matches_oracle and 7-2-4" "test_prefill_attention_tcgen05_matches_oracle and lens3" "test_gemm_tcgen05 and 640 and 100" "test_gemm_prefill_cta_pairs and 0-300" "test_kv_append_bit_exact"; do
  for tool in racecheck synccheck; do
    tag=$(echo "$t" | cut -d' ' -f1)_$tool
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "$t" > $out/san_$tag.log 2>&1
    echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $out/san_$tag.log | tr '\n' ' ')" >> $out/sanitizer_summary.txt
  done
done
bash scripts/sched_ablation_c1.sh $out/sched_c1 > /dev/null 2>&1
cat $out/sanitizer_summary.txt; head -c 700 $out/bench.json; echo; cat $out/sched_c1/summary.jsonl
