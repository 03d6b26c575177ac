#!/bin/bash
# prefill-shaped GEMMs: 2-SM data-parallel tiles vs the stream-K pair path by M threshold
out=gpurun_out/r3h; mkdir -p $out
for mm in 256 512 1024 4096; do
MUX_GEMM_2SM_MIN_M=$mm timeout 300 python - >> $out/gemm_prefill_m.txt 2>&1 <<PY
import sys, json
sys.path.insert(0, ".")
from scripts.gemm_micro import bench
peak = 1680.0
for M in (322, 563, 800, 1024, 2048):
    for name, (N, K, epi) in {"qkv7": (12288, 4096, 0), "gu7": (22016, 4096, 2), "down7": (4096, 11008, 1), "qkv13": (15360, 5120, 0), "gu13": (27648, 5120, 2)}.items():
        us, gbs = bench(M, N, K, epi, 148)
        tf = 2 * M * N * K / (us * 1e-6) / 1e12
        print(json.dumps({"min_m": $mm, "M": M, "shape": name, "us": round(us, 1), "frac_bf16": round(tf / peak, 3)}))
PY
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/r3h/gemm_prefill_m.txt") if l.startswith("{")]
t = collections.defaultdict(dict)
for r in rows:
    t[(r["M"], r["shape"])][r["min_m"]] = r["us"]
for k, v in sorted(t.items()):
    print(k, v)
PY
