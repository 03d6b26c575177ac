#!/bin/bash
# K3 persistent schedule with small grids (many items per CTA): parity + racecheck/synccheck
out=gpurun_out/r4f; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -n 1 $out/tests_k3.log
for tool in racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "many_items" > $out/san_$tool.log 2>&1
grep -E "SUMMARY|passed|failed" $out/san_$tool.log | tail -n 2
done
