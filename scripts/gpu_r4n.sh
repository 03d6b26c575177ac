#!/bin/bash
# ncu --set full (source-level) of the final K3 at 4096 tokens x 40 heads and at 25 x 161 prompts x 32 heads
out=gpurun_out/r4n; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention -c 1 -o $out/k3_final_4096 python - > $out/k3_4096.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
attn([4096], 40, iters=1)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention -c 1 -o $out/k3_final_161x25 python - > $out/k3_161.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
attn([161] * 25, 32, iters=1)
PY
tail -n 1 $out/k3_4096.log $out/k3_161.log
