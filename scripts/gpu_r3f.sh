#!/bin/bash
# launch list at serving-shaped batch 16 (both models, whole-GPU streams)
out=gpurun_out/r3f; mkdir -p $out
CUDA_MODULE_LOADING=EAGER timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_b16.csv python bench.py --batch 16 --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 \
  --partition-sms none > $out/ncu_b16.log 2>&1
python scripts/launch_summary.py $out/launches_b16.csv | head -12
gzip -f $out/*.csv
# prefill-shaped GEMMs (serving prefill jobs: 2-4 ShareGPT prompts)
timeout 300 python - > $out/gemm_prefill_m.txt 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
from scripts.gemm_micro import bench
peak = 1680.0
for M in (322, 563, 1024):
    for name, (N, K, epi) in {"qkv7": (12288, 4096, 0), "gu7": (22016, 4096, 2), "down7": (4096, 11008, 1), "qkv13": (15360, 5120, 0), "gu13": (27648, 5120, 2)}.items():
        us, gbs = bench(M, N, K, epi, 148)
        tf = 2 * M * N * K / (us * 1e-6) / 1e12
        print(json.dumps({"M": M, "shape": name, "us": round(us, 1), "tflops": round(tf, 1), "frac_bf16": round(tf / peak, 3), "weight_gbs": round(gbs)}))
PY
cat $out/gemm_prefill_m.txt
