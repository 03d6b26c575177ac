"""Decode-GEMM overhead probes (CUDA events, back-to-back launches, PDL on):
the same projection with the bf16-store epilogue (stream-K pieces summed by
a fixer) vs the fp32 reduce-add epilogue (no fixup), and near-empty launches
(the fixed head + tail of one launch)."""
import json
import sys

sys.path.insert(0, ".")
from scripts.gemm_micro import bench  # noqa: E402

out = []
for M in (16, 128):
    for name, (N, K) in {"qkv7": (12288, 4096), "gu7": (22016, 4096), "qkv13": (15360, 5120)}.items():
        for epi in (0, 1):
            us, gbs = bench(M, N, K, epi, 148)
            out.append({"M": M, "shape": name, "epi": epi, "us": round(us, 2), "gbs": round(gbs)})
            print(json.dumps(out[-1]), flush=True)
    for N, K in ((128, 64), (1024, 64), (128 * 148, 64), (4096, 1024)):
        for epi in (0, 1):
            us, gbs = bench(M, N, K, epi, 148)
            out.append({"M": M, "shape": f"{N}x{K}", "epi": epi, "us": round(us, 2), "gbs": round(gbs)})
            print(json.dumps(out[-1]), flush=True)
