"""f1: the fused TP allreduce's cost, measured on ONE B200 (an upper bound
for the per-call latency term, cost_model.cpp:43-47).

Both ranks of a tp = 2 LLaMA-7B mesh run in this process on the same GPU
(Megatron shards, rank-local pool slices, the row-parallel O / down GEMMs
storing fp32 partials into both ranks' mailboxes and rmsnorm_tp summing
them). A decode step of the pair streams exactly the bytes of one tp = 1
step (each rank half the weights and half the heads' K/V), so on one device

    alpha_ms <= (T_tp2(b) - T_tp1(b)) / (2 * num_layers)

per allreduce call: the mailbox stores, the release/acquire signal, the
spin-wait and the extra launches, with the two ranks' streams contending
for one GPU instead of overlapping across two. The payload term is NVLink's,
not measurable here: allreduce_ms_per_mib = (tp - 1) / tp * MiB / 900 GB/s
(NVLink 5 per direction, nominal). Writes JSON with both terms (the
LatencyProfile keys allreduce_alpha_ms / allreduce_ms_per_mib, wire.TP_KEYS).
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_02015_b200 as mux  # noqa: E402


def make_units(spec, tp, max_batch, ctx):
    total = 12_000_000  # head-blocks (49 GB): batch 128 x 564 tokens at tp 1
    units = [mux.Unit([spec], pool_blocks=total // tp, device_pool_blocks=total // tp, max_batch=max_batch,
                      max_prefill_tokens=256, max_ctx=ctx + 64, max_slots=max_batch + 8, init_seed=1, init_std=0.02,
                      partitions=2, tp_rank=r, tp_size=tp) for r in range(tp)]
    if tp > 1:
        for p in range(2):
            ptrs = [u.tp_mailbox(p)[0] for u in units]
            for r, u in enumerate(units):
                for q in range(tp):
                    if q != r:
                        u.tp_connect(p, q, ptr=ptrs[q])
    for u in units:
        u.init_kv(seed=3, std=1.0)
    return units


def step_ms(units, rids, steps=12, warm=4):
    for i in range(warm + steps):
        if i == warm:
            for k, u in enumerate(units):
                u.record(1, 2 * k)
        for u in units:
            assert all(r.ok for r in u.pool.alloc_n(0, u._ids(rids), 1, False))
        for u in units:  # every rank enqueued before any waits
            u.decode(0, rids, partition=1)
    for k, u in enumerate(units):
        u.record(1, 2 * k + 1)
    for u in units:
        u.sync()
    return max(u.elapsed_ms(2 * k, 2 * k + 1) for k, u in enumerate(units)) / steps


def main():
    spec = mux.spec("7b")
    ctx = 500
    out = {"model": "7b", "context": ctx, "points": []}
    for b in (1, 8, 32, 128):
        t = {}
        for tp in (1, 2):
            units = make_units(spec, tp, b, ctx)
            rids = list(range(1000, 1000 + b))
            for u in units:
                u.pool.set_quota(0, u.pool.total_blocks())
                for r in rids:
                    res = u.pool.admit(0, r, ctx, ctx + 64)
                    assert res.ok, (tp, b, res)
            try:
                t[tp] = step_ms(units, rids)
            finally:
                for u in units:
                    u.close()
            torch.cuda.empty_cache()
        alpha = (t[2] - t[1]) / (2 * spec.num_layers)
        out["points"].append({"batch": b, "tp1_ms": t[1], "tp2_ms": t[2], "alpha_ms_upper": alpha})
        print(json.dumps(out["points"][-1]), flush=True)
    alphas = [p["alpha_ms_upper"] for p in out["points"]]
    out["allreduce_alpha_ms"] = max(0.0, float(np.median(alphas)))
    out["allreduce_ms_per_mib"] = 0.5 * (1 << 20) / 900e9 * 1e3
    out["notes"] = ("alpha: one-GPU two-rank upper bound (median over batches); per_mib: NVLink 5 nominal "
                    "900 GB/s per direction, (tp-1)/tp of the payload")
    print(json.dumps(out))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
