#!/bin/bash
# K3 split-group form (MUX_K3=2): parity, then prefill micro (both forms); bench GEMM-stream roofline
out=gpurun_out/r2t; mkdir -p $out

MUX_K3=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -s -k "prefill_attention" > $out/tests_k3v2.log 2>&1
tail -3 $out/tests_k3v2.log
if grep -q " passed" $out/tests_k3v2.log && ! grep -q "failed" $out/tests_k3v2.log; then
  MUX_K3=2 timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "prefill or long or lockstep" > $out/tests_k3v2_model.log 2>&1
  tail -3 $out/tests_k3v2_model.log
  for k in 2 1; do
    MUX_K3=$k timeout 300 python - > $out/k3_micro_$k.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
from scripts.prefill_micro import attn
peak = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 1590.0
for lens, H in [([4096], 40), ([4096], 32), ([2048] * 2, 40), ([512] * 8, 40), ([161] * 25, 32), ([161] * 25, 40)]:
    us, tf = attn(lens, H)
    print(f"K3 lens={lens[0]}x{len(lens)} H={H}: {us:8.1f} us {tf:7.1f} TFLOP/s ({tf / peak:.1%})")
PY
  done
  cat $out/k3_micro_*.txt
fi
