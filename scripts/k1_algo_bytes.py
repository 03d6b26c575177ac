"""Algorithmic bytes of one K1 launch in bench.py's workload (same seeded
batches), per model and step: sum_i ctx_i*H*128*2*2 (K+V) + B*H*128*2*2 (q, o).
Pairs with an ncu --set full capture of a bench K1 launch (profiles/); the
default steps_total matches `bench.py --steps 2 --warmup 1 --e2e-steps 0 --attn-steps 0`."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2404_02015_b200 as mux  # noqa: E402
from bench import sample_batch  # noqa: E402


def main(models="7b,13b", B=128, steps_total=1 + 2 + 0 + 0 + 2, step=0, rank=0):
    specs = [mux.spec(m) for m in models.split(",")]
    rng = np.random.default_rng(1000 + rank)
    batches = [sample_batch(rng, B, steps_total) for _ in specs]
    for s, reqs in zip(specs, batches):
        ctx = [p + d + 1 + step for p, o, d in reqs]  # cached tokens incl. this step's new one
        b = sum(c * s.num_heads * 128 * 2 * 2 for c in ctx) + B * s.num_heads * 128 * 2 * 2
        print(f"{s.name}: step {step} K1 bytes/launch {b} (sum ctx {sum(ctx)}, H {s.num_heads})")


if __name__ == "__main__":
    main(*sys.argv[1:2])
