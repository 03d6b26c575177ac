#!/bin/bash
# K3 A/B in one box: next item first Q K^T after the last P V (MUX_K3_PVFIRST=1) vs before (0); ncu time + SM cycles; sanitizer on the flat form
out=gpurun_out/r4a; mkdir -p $out
for f in 1 0; do
MUX_K3_PVFIRST=$f timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3_$f.log 2>&1
tail -n 1 $out/tests_k3_$f.log
done
for rep in 1 2; do
for f in 0 1; do
MUX_K3_PVFIRST=$f timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
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
rows = list(csv.reader(open(f"gpurun_out/r4a/k3_ncu_{f}_{rep}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi].replace(",", "")
vals = list(out.values())[::3]
print("pvfirst", f, [(int(v["gpu__time_duration.sum"]) // 100 / 10, int(v["sm__cycles_elapsed.max"]) // 1000, v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in vals])
PY
done
done
for tool in racecheck synccheck; do
MUX_K3_PVFIRST=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/san_$tool.log 2>&1
grep -E "ERROR SUMMARY|passed|failed" $out/san_$tool.log | tail -n 2
done
