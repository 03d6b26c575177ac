#!/bin/bash
# Marginal cost of each kernel class inside the pipelined decode step
# (MUX_DEBUG_SKIP drops kernels; results are garbage, timings are not).
# usage: skip_sweep.sh "7b 13b" "0 4 120 8 16 32 64"
for m in ${1:-7b 13b}; do
  for s in ${2:-0 1 2 4 120 8 16 32 64}; do
    v=$(MUX_DEBUG_SKIP=$s python bench.py --skip-cpu --models $m --e2e-steps 0 --attn-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])" 2>&1)
    echo "model=$m skip=$s ms_per_step=$v"
  done
done
