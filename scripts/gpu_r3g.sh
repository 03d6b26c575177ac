#!/bin/bash
# Balanced token tiles for prefill shapes + CTA pairs beyond 256 tokens: parity, prefill GEMM micro, serving
out=gpurun_out/r3g; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py tests/test_gpu_model.py -q -x > $out/tests.log 2>&1
tail -3 $out/tests.log
timeout 300 python - > $out/gemm_prefill_m.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
from scripts.gemm_micro import bench
peak = 1680.0
for M in (322, 563, 1024):
    for name, (N, K, epi) in {"qkv7": (12288, 4096, 0), "gu7": (22016, 4096, 2), "down7": (4096, 11008, 1), "qkv13": (15360, 5120, 0), "gu13": (27648, 5120, 2)}.items():
        us, gbs = bench(M, N, K, epi, 148)
        tf = 2 * M * N * K / (us * 1e-6) / 1e12
        print(json.dumps({"M": M, "shape": name, "us": round(us, 1), "tflops": round(tf, 1), "frac_bf16": round(tf / peak, 3)}))
PY
cat $out/gemm_prefill_m.txt
timeout 900 python serve.py --rates 120,60 --horizon 6 --realtime 2>/dev/null | tail -1 > $out/serve.json
python -c "import json; d=json.load(open('$out/serve.json')); print(d['value'], d['arrival_window'], d['ttft_ms'])"
