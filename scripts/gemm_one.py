"""One GEMM shape, a few launches (for ncu)."""
import sys

sys.path.insert(0, ".")
from scripts.gemm_micro import bench  # noqa: E402

M, N, K, epi = (int(x) for x in sys.argv[1:5])
print(bench(M, N, K, epi, 148, iters=3))
