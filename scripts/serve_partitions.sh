#!/bin/bash
# Serving run (serve.py, 7B + 13B at 120 + 60 rps) under three SM-partition
# policies, back to back on one box: whole-GPU streams, static green
# partitions (56 + 92 SMs), and the per-pass choice (option pass_green).
# Output: one JSON line per variant in gpurun_out/serve_partitions.jsonl.
set -u
out=gpurun_out/serve_partitions.jsonl
mkdir -p gpurun_out; : > $out
for rates in 120,60 20,10; do
  for v in "" "--partition-sms 56,92" "--pass-green 56,92" "--pass-green 56,92 --prefill-on-partition 1"; do
    timeout 300 python serve.py --rates $rates --horizon 3 $v >> $out 2>> gpurun_out/serve_partitions.err
  done
done
