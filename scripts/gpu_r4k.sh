#!/bin/bash
# K3 A/B in one box at the final schedule: exp2 pairs on the FMA pipe per 8 (MUX_K3_POLY 0 / 3 / 4); ncu time + SM cycles
out=gpurun_out/r4k; mkdir -p $out
MUX_K3_POLY=4 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3_4.log 2>&1
tail -n 1 $out/tests_k3_4.log
for rep in 1 2; do
for f in 0 3 4; do
MUX_K3_POLY=$f timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu_${f}_$rep.csv python - > $out/k3_ncu_${f}_$rep.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - $f $rep <<'PY'
import csv, sys
f, rep = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(f"gpurun_out/r4k/k3_ncu_{f}_{rep}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi].replace(",", "")
vals = list(out.values())[::3]
print("poly", f, [(int(v["gpu__time_duration.sum"]) // 100 / 10, int(v["sm__cycles_elapsed.max"]) // 1000, v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in vals])
PY
done
done
