#!/bin/bash
# compute-sanitizer racecheck / synccheck on the round-2 kernels: decode GEMM on CTA pairs
# (tiled weights, M = 128), two-tile units, K3 with P in TMEM
out=gpurun_out/r3e; mkdir -p $out
for t in "test_gemm_tiled_weights and 128-1000" "test_prefill_attention_tcgen05_matches_oracle and lens3" "test_headline_projection_shapes and 13b and 128"; do
  for tool in racecheck synccheck; do
    tag=$(echo "$t" | cut -d' ' -f1)_$tool
    timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -q -x -k "$t" > $out/san_$tag.log 2>&1
    echo "$tag rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $out/san_$tag.log | tr '\n' ' ')" >> $out/summary.txt
  done
done
cat $out/summary.txt
