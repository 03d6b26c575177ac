#!/bin/bash
# Scheduler ablation in the real-time engine: the acceptance-C1
# contention shape (7B x 2, 10 rps x 128/384 and 80 rps x 64/64, 34 / 40 GiB)
# under ADBS, FCFS and round-robin. Output: gpurun_out/sched_rt.jsonl
set -u
out=gpurun_out/sched_rt.jsonl
mkdir -p gpurun_out; : > $out
for mem in 34 40; do
  for s in adbs fcfs rr; do
    timeout 400 python serve.py --realtime --models 7b,7b --rates 10,80 --lengths 128:384,64:64 --horizon 8 \
      --gpu-memory-gib $mem --scheduler $s >> $out 2>> gpurun_out/sched_rt.err
  done
done
