#!/bin/bash
# K3 with P double-buffered in TMEM: parity, sanitizer, ncu time + cycles
out=gpurun_out/r4i; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -n 1 $out/tests_k3.log
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py -q -x > $out/tests_model.log 2>&1
tail -n 1 $out/tests_model.log
for rep in 1 2; do
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu_$rep.csv python - > $out/k3_ncu_$rep.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - $rep <<'PY'
import csv, sys
rep = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r4i/k3_ncu_{rep}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi].replace(",", "")
vals = list(out.values())[::3]
print("p2", [(int(v["gpu__time_duration.sum"]) // 100 / 10, int(v["sm__cycles_elapsed.max"]) // 1000, v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in vals])
PY
done
for tool in racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/san_$tool.log 2>&1
grep -E "SUMMARY|passed|failed" $out/san_$tool.log | tail -n 2
done
