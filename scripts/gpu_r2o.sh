#!/bin/bash
# GEMM pipeline experiments (B-ring depth, epilogue kinds, NOMMA), TP allreduce cost, config-5 SLO sweep
out=gpurun_out/r2o; mkdir -p $out
timeout 300 python scripts/gemm_probe.py > $out/probe.jsonl 2>&1
for sb in 2 3 4 5 6; do
  for sa in 0 6 8; do
    echo "SB=$sb SA=$sa" >> $out/sb_sweep.txt
    MUX_GEMM_SB=$sb MUX_GEMM_SA=$sa timeout 200 python - >> $out/sb_sweep.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
from scripts.gemm_micro import bench
for name, (N, K, epi) in {"qkv7": (12288, 4096, 0), "gu13": (27648, 5120, 0), "down13": (5120, 13824, 1)}.items():
    us, gbs = bench(128, N, K, epi, 148)
    print(f"  {name} {us:.1f}us {gbs:.0f}GB/s")
PY
  done
done
for nm in 1 3; do
  echo "NOMMA=$nm" >> $out/sb_sweep.txt
  MUX_GEMM_NOMMA=$nm timeout 200 python - >> $out/sb_sweep.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
from scripts.gemm_micro import bench
for name, (N, K, epi) in {"qkv7": (12288, 4096, 0), "gu13": (27648, 5120, 0), "down13": (5120, 13824, 1)}.items():
    us, gbs = bench(128, N, K, epi, 148)
    print(f"  {name} {us:.1f}us {gbs:.0f}GB/s")
PY
done
timeout 900 python scripts/tp_allreduce_cost.py $out/tp_allreduce.json > $out/tp_allreduce.log 2>&1
cat $out/probe.jsonl; cat $out/sb_sweep.txt; tail -6 $out/tp_allreduce.log
timeout 2400 bash scripts/slo_sweep_c5.sh $out/slo_c5 realtime > /dev/null 2>&1
cat $out/slo_c5/summary.jsonl | cut -c1-300
