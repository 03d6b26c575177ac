"""Decode step device time vs the decode GEMM's k-blocks-per-CTA floor
(option gemm_min_iters, default 24) at serving-sized batches: 7B / 13B,
batch 8 / 24 / 64 / 128 at context 400, whole-GPU stream.

    python scripts/min_iters_sweep.py  ->  one JSON line per (model, batch)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_02015_b200 as mux  # noqa: E402
from paper_2404_02015_b200 import blocks_for_tokens  # noqa: E402

ITERS = (8, 12, 16, 24, 32, 48)


def main():
    for model in ("7b", "13b"):
        s = mux.spec(model)
        kv = blocks_for_tokens(s, 16, 128 * 700 + 4096)
        u = mux.Unit([s], pool_blocks=kv, device_pool_blocks=kv, max_batch=128, max_prefill_tokens=512,
                     max_ctx=1024, max_slots=512, init_seed=1, init_std=0.02, partitions=2)
        u.init_kv(seed=3, std=1.0)
        try:
            for b in (8, 24, 64, 128):
                rids = list(range(1000, 1000 + b))
                for r in rids:
                    assert u.pool.admit(0, r, 400, 560).ok
                row = {"model": model, "batch": b, "ctx": 400}
                for it in ITERS:
                    u.set_option("gemm_min_iters", it)
                    for _ in range(2):  # warm-up
                        for r in rids:
                            assert u.pool.alloc(0, r, 1, False).ok
                        u.decode(0, rids, partition=1)
                    u.sync()
                    u.record(1, 0)
                    for _ in range(5):
                        for r in rids:
                            assert u.pool.alloc(0, r, 1, False).ok
                        u.decode(0, rids, partition=1)
                    u.record(1, 1)
                    u.sync()
                    row[f"ms_{it}"] = round(u.elapsed_ms(0, 1) / 5, 3)
                for r in rids:
                    u.pool.free_request(0, r)
                u.set_option("gemm_min_iters", 8)
                print(json.dumps(row), flush=True)
        finally:
            u.close()


if __name__ == "__main__":
    main()
