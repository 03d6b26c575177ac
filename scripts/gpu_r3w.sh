#!/bin/bash
# K3: masked tiles on the fast exp path; per-part row max without the barrier (MUX_K3_OWNMAX) x exp2 on the FMA pipe (MUX_K3_POLY)
out=gpurun_out/r3w; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -2 $out/tests_k3.log
MUX_K3_OWNMAX=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3_p5.log 2>&1
tail -2 $out/tests_k3_p5.log
if grep -q " passed" $out/tests_k3.log && ! grep -q "failed" $out/tests_k3.log; then
timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_headline.py -q -x > $out/tests_model.log 2>&1
tail -2 $out/tests_model.log
for cfg in 0:0 3:0 0:1 3:1 4:1; do
pp=${cfg%:*}_${cfg#*:}
MUX_K3_POLY=${cfg%:*} MUX_K3_OWNMAX=${cfg#*:} timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
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
rows = list(csv.reader(open(f"gpurun_out/r3w/k3_ncu_{pp}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi]
vals = list(out.values())[::3]
print("poly", pp, [(v["gpu__time_duration.sum"], v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
                    v["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"], v["sm__issue_active.avg.pct_of_peak_sustained_active"]) for v in vals])
PY
done
fi
