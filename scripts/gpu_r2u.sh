#!/bin/bash
# K3 split form default: full GPU suite, ncu device times of K3 (both forms), final bench + reference arm
out=gpurun_out/r2u; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
for k in 2 1; do
  MUX_K3=$k timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
    -k regex:prefill_attention --log-file $out/k3_ncu_$k.csv python - > $out/k3_ncu_$k.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    attn(lens, H, iters=2)
PY
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attention_split -c 1 -o $out/k3_split_4096 python - > $out/k3_full.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
attn([4096], 40, iters=1)
PY
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/ref.json 2> $out/ref.err
tail -3 $out/gpu_suite.log; tail -1 $out/smoke.log; head -c 1500 $out/bench.json; echo
