"""Sweep the GEMM's A/B ring depths (MUX_GEMM_SA / MUX_GEMM_SB) on decode shapes."""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, ".")
from scripts.gemm_micro import bench
M = int(sys.argv[1])
out = []
for name, (N, K), epi in [("qkv13", (15360, 5120), 0), ("o13", (5120, 5120), 1), ("gu13", (27648, 5120), 2),
                          ("down13", (5120, 13824), 1), ("gu7", (22016, 4096), 2)]:
    us, gbs = bench(M, N, K, epi, 148)
    out.append(f"{name}:{us:6.1f}us/{gbs:5.0f}")
print(" ".join(out), flush=True)
'''

if __name__ == "__main__":
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    configs = [(0, 0, 1)] + [tuple(map(int, c.split(","))) for c in sys.argv[2:]]
    for cfg in configs:
        sa, sb = cfg[0], cfg[1]
        split = cfg[2] if len(cfg) > 2 else 1
        env = dict(os.environ)
        env["MUX_GEMM_ASPLIT"] = str(split)
        if len(cfg) > 3:
            env["MUX_GEMM_NOMMA"] = str(cfg[3])
        if sa:
            env["MUX_GEMM_SA"] = str(sa)
        if sb:
            env["MUX_GEMM_SB"] = str(sb)
        r = subprocess.run([sys.executable, "-c", CODE, str(M)], env=env, capture_output=True, text=True)
        print(f"M={M} SA={sa} SB={sb} split={split}: {r.stdout.strip()} {r.stderr.strip()[-300:]}", flush=True)
