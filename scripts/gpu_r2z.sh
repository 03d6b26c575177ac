#!/bin/bash
# ncu --set full of K3 (P in TMEM) at 4096 tokens x 40 heads, source-level
out=gpurun_out/r2z; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention -c 1 -o $out/k3_ptmem_4096 python - > $out/k3_full.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
attn([4096], 40, iters=1)
PY
tail -2 $out/k3_full.log
