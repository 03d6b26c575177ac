"""One prefill-shaped GEMM launch (qkv13 M=4096, tiled weights) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402

M, N, K = 4096, 15360, 5120
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
wt = mux.weight_tile(w)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    mux.gemm_bf16(x, w, out, epilogue=0, w_tiled=wt)
torch.cuda.synchronize()
