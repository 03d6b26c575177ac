#!/bin/bash
# Serving runs (serve.py, 7B + 13B) in the measured engine (each pass's jobs
# timed together, passes serialised) and the real-time engine (jobs overlap
# across passes, completions from device events), back to back on one box.
# Output: gpurun_out/serve_engines.jsonl
set -u
out=gpurun_out/serve_engines.jsonl
mkdir -p gpurun_out; : > $out
for rates in "120,60 --horizon 3" "20,10 --horizon 8"; do
  for v in "" "--realtime"; do
    timeout 400 python serve.py --rates $rates $v >> $out 2>> gpurun_out/serve_engines.err
  done
done
