#!/bin/bash
# ncu --set full, source-level, of K3 on ShareGPT-shaped prompts (25 x 161 tokens, 32 heads)
out=gpurun_out/r4b; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention -c 1 -o $out/k3_161x25 python - > $out/k3_full.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
attn([161] * 25, 32, iters=1)
PY
tail -n 2 $out/k3_full.log
