#!/bin/bash
# B200 latency profile refit with the round-2 kernels (7B, 13B)
out=gpurun_out/r3s; mkdir -p $out
for m in 7b 13b; do
  timeout 1500 python -m paper_2404_02015_b200.calibrate --model $m -o $out/b200_profile_$m.json > $out/calib_$m.log 2>&1
  tail -1 $out/calib_$m.log | cut -c1-600
done
