#!/bin/bash
# K3 with P through TMEM (TS MMA, MUX_K3_PTMEM=1): parity, ncu device times of both forms
out=gpurun_out/r2y; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -2 $out/tests_k3.log
if grep -q " passed" $out/tests_k3.log && ! grep -q "failed" $out/tests_k3.log; then
timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "prefill or long or lockstep" > $out/tests_k3_model.log 2>&1
tail -2 $out/tests_k3_model.log
for pt in 1; do
MUX_K3_PTMEM=$pt timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu_$pt.csv python - > $out/k3_ncu_$pt.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - $pt <<'PY'
import csv, sys
pt = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r2y/k3_ncu_{pt}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi]
print("ptmem", pt, [(v["gpu__time_duration.sum"], v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in out.values()][::3])
PY
done
fi
