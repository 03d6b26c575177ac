"""Where the e2e step's host time goes (bench.py's e2e loop: host tokens in,
next tokens out, a sync every step): per-phase host wall times."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2404_02015_b200 as mux  # noqa: E402


def main():
    specs = [mux.spec("7b"), mux.spec("13b")]
    B, steps = 128, 30
    rng = np.random.default_rng(1000)
    batches = [bench.sample_batch(rng, B, 60) for _ in specs]
    need = sum(mux.blocks_for_tokens(s, 16, p + d + 61) for s, reqs in zip(specs, batches) for p, o, d in reqs)
    logical = bench.pool_blocks(["7b", "13b"])
    max_ctx = max(p + d + 61 for reqs in batches for p, o, d in reqs)
    unit = mux.Unit(specs, pool_blocks=logical, device_pool_blocks=need + 4096, max_batch=B, max_prefill_tokens=256,
                    max_ctx=max_ctx + 16, max_slots=2 * B + 16, init_seed=1, init_std=0.02, partitions=3,
                    partition_sms=[0, 56, 92])
    unit.init_kv(seed=7, std=1.0)
    pool = unit.pool
    ids = []
    for li, reqs in enumerate(batches):
        rids = []
        for k, (p, o, d) in enumerate(reqs):
            rid = 10_000 * li + k
            assert pool.admit(li, rid, p, p + o - 1).ok
            if d:
                assert pool.alloc(li, rid, d, False).ok
            rids.append(rid)
        ids.append(rids)
    ids_c = [unit._ids(r) for r in ids]
    pin_in = [torch.zeros(B, dtype=torch.int32).pin_memory().numpy() for _ in specs]
    pin_out = [torch.zeros(B, dtype=torch.int32).pin_memory().numpy() for _ in specs]
    ph = {"alloc": [], "decode_call": [], "sync": [], "copy": [], "total": []}
    for s in range(steps):
        t0 = time.perf_counter()
        for li in (1, 0):
            a = time.perf_counter()
            res = pool.alloc_n(li, ids_c[li], 1, False)
            assert all(r.ok for r in res)
            b = time.perf_counter()
            unit.decode(li, ids[li], tokens=pin_in[li], out=pin_out[li], partition=1 + li, ids_c=ids_c[li])
            c = time.perf_counter()
            ph["alloc"].append(b - a)
            ph["decode_call"].append(c - b)
        d0 = time.perf_counter()
        unit.sync()
        d1 = time.perf_counter()
        for li in range(2):
            pin_in[li][:] = pin_out[li]
        d2 = time.perf_counter()
        ph["sync"].append(d1 - d0)
        ph["copy"].append(d2 - d1)
        ph["total"].append(d2 - t0)
    out = {k: round(1e3 * float(np.median(v[10:] if len(v) > 20 else v)), 4) for k, v in ph.items()}
    out["note"] = "median ms per call (alloc / decode_call per model, sync / copy / total per step), steps 10+"
    print(json.dumps(out))
    unit.close()


if __name__ == "__main__":
    main()
