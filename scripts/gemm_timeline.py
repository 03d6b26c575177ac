"""Per-CTA globaltimer timeline of single K4 launches (debug)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402

shapes = {"o7": (4096, 4096, 1), "qkv7": (12288, 4096, 0), "gu13": (27648, 5120, 0), "down7": (4096, 11008, 1), "lm": (32000, 4096, 3), "gu7s": (22016, 4096, 2)}
M = 128
buf = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
for name, (N, K, epi) in shapes.items():
    for grid in (148, 128, 32):
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        wt = mux.weight_tile(w)
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
        for _ in range(2):
            mux.gemm_bf16(x, w, out, epilogue=epi, grid=grid, w_tiled=wt)
        torch.cuda.synchronize()
        buf.zero_()
        mux.lib.mux_debug_gemm_timing(buf.data_ptr())
        mux.gemm_bf16(x, w, out, epilogue=epi, grid=grid, w_tiled=wt)
        torch.cuda.synchronize()
        mux.lib.mux_debug_gemm_timing(None)
        raw = buf.view(-1, 16)[:grid].cpu().double()
        t0 = raw[:, 0].min()
        t = (raw - t0) / 1e3  # us

        def st(col):
            v = t[:, col][raw[:, col] > 0]
            return f"med {v.median():6.2f} max {v.max():6.2f}" if len(v) else "   -   "
        print(f"{name:6s} g{grid:3d} mma-issued {st(1)} | first tm_full {st(4)} | partner published {st(7)} | "
              f"fixer waited {st(5)} | fixer adds done {st(6)} | epi done {st(2)}", flush=True)
        print("   fixer chunk stamps (begin,end) med: " + " ".join(f"{t[:, k][raw[:, k] > 0].median():6.2f}" for k in range(8, 16) if (raw[:, k] > 0).any()))
