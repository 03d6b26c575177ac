"""Host cost of enqueueing one decode job (the real-time engine's critical
path between a completion and the model's next step) against its device
time: 7B / 13B, decode batch b at context c, whole-GPU stream.

    python scripts/launch_overhead.py  ->  one JSON line per (model, b)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_02015_b200 as mux  # noqa: E402
from paper_2404_02015_b200 import blocks_for_tokens  # noqa: E402


def main():
    for model in ("7b", "13b"):
        s = mux.spec(model)
        kv = blocks_for_tokens(s, 16, 64 * 600 + 4096)
        u = mux.Unit([s], pool_blocks=kv, device_pool_blocks=kv, max_batch=64, max_prefill_tokens=512,
                     max_ctx=1024, max_slots=256, init_seed=1, init_std=0.02, partitions=2)
        u.init_kv(seed=3, std=1.0)
        try:
            for b in (8, 64):
                rids = list(range(1000, 1000 + b))
                for r in rids:
                    assert u.pool.admit(0, r, 400, 520).ok
                host, dev = [], []
                for it in range(12):
                    for r in rids:
                        assert u.pool.alloc(0, r, 1, False).ok
                    u.sync()
                    u.record(1, 0)
                    t0 = time.perf_counter()
                    u.decode(0, rids, partition=1)
                    host.append((time.perf_counter() - t0) * 1e3)
                    u.record(1, 1)
                    u.sync()
                    dev.append(u.elapsed_ms(0, 1))
                for r in rids:
                    u.pool.free_request(0, r)
                host, dev = sorted(host[2:]), sorted(dev[2:])
                print(json.dumps({"model": model, "batch": b, "ctx": 400, "host_enqueue_ms_median": round(host[len(host) // 2], 3),
                                  "device_ms_median": round(dev[len(dev) // 2], 3),
                                  }), flush=True)
        finally:
            u.close()


if __name__ == "__main__":
    main()
