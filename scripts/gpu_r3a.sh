#!/bin/bash
# K3 ping-pong form (MUX_K3_PP=1): parity, then ncu device times of both forms
out=gpurun_out/r3a; mkdir -p $out
MUX_K3_PP=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_pp.log 2>&1
tail -3 $out/tests_pp.log
if grep -q " passed" $out/tests_pp.log && ! grep -q "failed" $out/tests_pp.log; then
MUX_K3_PP=1 timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "prefill or long or lockstep" > $out/tests_pp_model.log 2>&1
tail -2 $out/tests_pp_model.log
for pp in 1 0; do
MUX_K3_PP=$pp timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu_$pp.csv python - > $out/k3_ncu_$pp.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - $pp <<'PY'
import csv, sys
pp = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r3a/k3_ncu_{pp}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi]
print("pp", pp, [(v["gpu__time_duration.sum"], v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in out.values()][::3])
PY
done
fi
