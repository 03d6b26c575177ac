#!/bin/bash
# TP units without CTA-pair GEMMs: the GPU suite three times (the shared-GPU TP test was flaky)
out=gpurun_out/r3l; mkdir -p $out
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite_$i.log 2>&1
  tail -1 $out/gpu_suite_$i.log
done
