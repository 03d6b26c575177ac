#!/bin/bash
# Real-time engine (serve.py --realtime, 7B + 13B): whole-GPU streams vs
# static green partitions (56 + 92 SMs) for the decode jobs, with prefill on
# the whole GPU or on its model's partition. Output:
# gpurun_out/serve_rt_partitions.jsonl
set -u
out=gpurun_out/serve_rt_partitions.jsonl
mkdir -p gpurun_out; : > $out
for rates in "120,60 --horizon 3" "20,10 --horizon 8"; do
  for v in "" "--partition-sms 56,92" "--partition-sms 56,92 --prefill-on-partition 1"; do
    timeout 400 python serve.py --realtime --rates $rates $v >> $out 2>> gpurun_out/serve_rt_partitions.err
  done
done
