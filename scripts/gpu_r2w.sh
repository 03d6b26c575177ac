#!/bin/bash
# K3 with 4 softmax warps per TMEM lane quarter (kParts 4): parity, ncu device times (compare r2u MUX_K3=1)
out=gpurun_out/r2w; mkdir -p $out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "prefill_attention" > $out/tests_k3.log 2>&1
tail -2 $out/tests_k3.log
timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "prefill or long or lockstep" > $out/tests_k3_model.log 2>&1
tail -2 $out/tests_k3_model.log
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:prefill_attention --log-file $out/k3_ncu.csv python - > $out/k3_ncu.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r2w/k3_ncu.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
out = {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        out.setdefault(r[0], {})[r[mi]] = r[vi]
print([(v["gpu__time_duration.sum"], v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]) for v in out.values()])
PY
