"""Prefill-side microbenchmarks: K3 tcgen05 attention and K4 GEMMs at prefill M
(tensor-bound: TFLOP/s vs MEASURED_PEAKS bf16)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402
from scripts.gemm_micro import bench as gemm_bench  # noqa: E402


def attn(lens, H, iters=10):
    T = sum(lens)
    qkv = torch.randn(T, 3, H, 128, device="cuda").to(torch.bfloat16)
    q = torch.randn(T, H, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty(T, H, 128, device="cuda", dtype=torch.bfloat16)
    mux.prefill_attention(q, qkv, out, lens)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        mux.prefill_attention(q, qkv, out, lens)  # includes a stream sync per call
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    flops = sum(4 * 128 * n * (n + 1) / 2 for n in lens) * H
    return us, flops / (us * 1e-6) / 1e12


if __name__ == "__main__":
    try:
        peak = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops"]
    except Exception:
        peak = 1590.0
    for lens, H in [([4096], 40), ([4096], 32), ([512] * 8, 40), ([161] * 25, 32)]:
        us, tf = attn(lens, H)
        print(f"K3 attn lens={lens[0]}x{len(lens)} H={H}: {us:8.1f} us  {tf:7.1f} TFLOP/s  ({tf / peak:.1%} of {peak})")
    for name, (N, K), epi in [("qkv13", (15360, 5120), 0), ("o13", (5120, 5120), 1), ("gu13", (27648, 5120), 2),
                              ("down13", (5120, 13824), 1)]:
        for M in (1024, 4096):
            us, _ = gemm_bench(M, N, K, epi, 148, iters=10)
            tf = 2 * M * N * K / (us * 1e-6) / 1e12
            print(f"K4 {name} M={M}: {us:8.1f} us  {tf:7.1f} TFLOP/s  ({tf / peak:.1%})")
