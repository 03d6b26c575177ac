"""Per-CTA globaltimer timeline of single K4 launches (debug).

Stamps (kernel, [grid][32] u64): 0 start, 4 first A stage landed, 5 first B
stage landed, 1 MMA issue done, 9+s TMEM full for segment s (s<4),
6 fixer: partner flags seen, 7 fixer: partials landed, 8 partner published,
2 epilogue done, 3 exit."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402

shapes = {"o13": (5120, 5120, 1), "qkv13": (15360, 5120, 0), "down13": (5120, 13824, 1), "gu13": (27648, 5120, 2)}
M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
buf = torch.zeros(1024 * 64, dtype=torch.int64, device="cuda")
names = {0: "start", 15: "synced", 32: "elected", 33: "policy", 34: "seggen", 35: "preexp", 36: "expect", 19: "A0issued", 4: "A0", 5: "B0", 9: "seg0", 10: "seg1", 11: "seg2", 6: "fixflag", 7: "fixdata",
         8: "publish", 1: "mma_done", 2: "epi_done", 3: "exit", 13: "exit128", 14: "exit32",
         16: "end0", 17: "end1", 18: "end2"}
for name, (N, K, epi) in shapes.items():
    grid = 148
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    wt = mux.weight_tile(w)
    out = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    for _ in range(2):
        mux.gemm_bf16(x, w, out, epilogue=epi, grid=grid, w_tiled=wt)
    torch.cuda.synchronize()
    buf.zero_()
    mux.lib.mux_debug_gemm_timing(buf.data_ptr())
    mux.gemm_bf16(x, w, out, epilogue=epi, grid=grid, w_tiled=wt)
    torch.cuda.synchronize()
    mux.lib.mux_debug_gemm_timing(None)
    raw = buf.view(-1, 64)[:grid].cpu().double()
    t0 = raw[:, 0].min()
    t = (raw - t0) / 1e3  # us
    parts = []
    for k, nm in names.items():
        v = t[:, k][raw[:, k] > 0]
        if len(v):
            parts.append(f"{nm} {v.min():.1f}/{v.median():.1f}/{v.max():.1f}")
    print(f"{name:6s} {N * K * 2 / 1e6:.0f}MB | " + " | ".join(parts), flush=True)
    if len(sys.argv) > 2 and name in sys.argv[2].split(","):  # per-CTA dump of the last segment's epilogue
        fine = {40: "sts", 41: "b1", 42: "silu", 43: "b2", 44: "fence", 45: "b3"}
        cols = [1, 7]
        for k in range(2):
            cols += [20 + k, 24 + k] + [40 + k * 8 + j for j in range(6)] + [28 + k]
        cols += [2]
        nm = dict(names)
        for k in range(2):
            nm.update({20 + k: f"ld{k}", 24 + k: f"bar{k}", 28 + k: f"st{k}"})
            nm.update({40 + k * 8 + j: f"{fine[40 + j]}{k}" for j in range(6)})
        print("cta " + " ".join(f"{nm[k]:>6s}" for k in cols))
        for c in range(0, grid, max(1, grid // 16)):
            print(f"{c:3d} " + " ".join(f"{t[c, k]:6.2f}" if raw[c, k] > 0 else "     -" for k in cols))


