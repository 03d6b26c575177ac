#!/bin/bash
# K3 with the next item's Q load and first Q K^T issued ahead (Q double-buffered, flat key-tile stream): parity, sanitizer, ncu device times
out=gpurun_out/r3y; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -2 $out/tests_k3.log
if grep -q " passed" $out/tests_k3.log && ! grep -q "failed" $out/tests_k3.log; then
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py -q -x > $out/tests_model.log 2>&1
tail -2 $out/tests_model.log
for tool in racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --kernel-name regex:prefill_attention python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/san_$tool.log 2>&1
grep -E "ERROR SUMMARY|passed|failed" $out/san_$tool.log | tail -2
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu.csv python - > $out/k3_ncu.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r3y/k3_ncu.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi]
vals = list(out.values())[::3]
print("qdb", [(v["gpu__time_duration.sum"], v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
               v["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"], v["sm__issue_active.avg.pct_of_peak_sustained_active"]) for v in vals])
PY
fi
