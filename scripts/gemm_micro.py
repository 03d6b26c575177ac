"""Microbenchmark of the tcgen05 GEMM on the decode shapes (CUDA events)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402


def bench(M, N, K, epi, grid=0, iters=20, tiled=True):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(4)]  # > L2 total
    wt = [mux.weight_tile(w) if tiled else None for w in ws]
    out = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda",
                      dtype=torch.bfloat16 if epi in (0, 2) else torch.float32)
    for w, t in zip(ws, wt):
        mux.gemm_bf16(x, w, out, epilogue=epi, grid=grid, w_tiled=t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        mux.gemm_bf16(x, ws[i % 4], out, epilogue=epi, grid=grid, w_tiled=wt[i % 4])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    gbs = N * K * 2 / (us * 1e-6) / 1e9
    return us, gbs


if __name__ == "__main__":
    shapes = {"qkv7": (12288, 4096), "o7": (4096, 4096), "gu7": (22016, 4096), "down7": (4096, 11008),
              "lm": (32000, 4096), "qkv13": (15360, 5120), "o13": (5120, 5120), "gu13": (27648, 5120),
              "down13": (5120, 13824)}
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    if len(sys.argv) > 2:  # profile mode: few launches per config, for ncu
        for name, (N, K) in shapes.items():
            for grid in (148, 128):
                bench(M, N, K, 1 if name.startswith(("o", "down")) else 0, grid, iters=2)
        sys.exit(0)
    for name, (N, K) in shapes.items():
        for epi in ((1,) if name.startswith(("o", "down")) else (0,)):
            res = []
            us, gbs = bench(M, N, K, epi, 148, tiled=False)
            res.append(f"tmap g148:{us:6.1f}us/{gbs:5.0f} | tiled")
            for grid in (148, 128, 96, 74):
                us, gbs = bench(M, N, K, epi, grid)
                res.append(f"g{grid}:{us:6.1f}us/{gbs:5.0f}")
            print(f"M={M} {name:6s} epi={epi} " + " ".join(res), flush=True)
