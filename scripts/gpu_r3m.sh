#!/bin/bash
# config-5 SLO sweep with the final engine (real-time)
out=gpurun_out/r3m; mkdir -p $out
timeout 3000 bash scripts/slo_sweep_c5.sh $out/slo_c5 realtime > /dev/null 2>&1
cut -c1-300 $out/slo_c5/summary.jsonl
