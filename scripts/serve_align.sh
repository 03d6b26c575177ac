#!/bin/bash
# Real-time engine, 7B + 13B: free-running vs aligned decode rounds
# (--align-decode), on whole-GPU streams and on green partitions (56 + 92).
# Output: gpurun_out/serve_align.jsonl
set -u
out=gpurun_out/serve_align.jsonl
mkdir -p gpurun_out; : > $out
for rates in "120,60 --horizon 3" "20,10 --horizon 8"; do
  for v in "" "--align-decode" "--align-decode --partition-sms 56,92"; do
    timeout 400 python serve.py --realtime --rates $rates $v >> $out 2>> gpurun_out/serve_align.err
  done
done
