"""K1 (paged decode attention) microbenchmark at SURVEY.md §8(d)'s points:
B in {1, 4, 16, 64, 128, 196} x {7B heads (32), 13B heads (40)}, contexts
drawn as prompt + U[1, output] (ShareGPT lognormals 161 / 338), plus a
long-context point (ctx 4096). One layer, block tables from the product's
physical BlockPool after an alloc/free churn (scattered head-blocks).

Reports device time per launch (CUDA events over back-to-back launches on one
stream, inputs larger than L2 between repetitions: the pool slice read per
launch is rotated over 4 disjoint request sets) and achieved GB/s of the
algorithmic bytes (K+V of every cached token + q + o) against the measured
HBM peak and the nominal 8 TB/s.

    python scripts/k1_micro.py > profiles/r01_k1_micro.txt
"""
import json
import math
import os
import random
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_02015_b200 as mux  # noqa: E402


def contexts(rng, B, long_ctx=None):
    if long_ctx:
        return [long_ctx] * B
    out = []
    mu_p, mu_o = math.log(161.0) - 0.32, math.log(338.0) - 0.32
    while len(out) < B:
        p = max(1, int(round(rng.lognormvariate(mu_p, 0.8))))
        o = max(1, int(round(rng.lognormvariate(mu_o, 0.8))))
        if p + o <= 4096:
            out.append(p + rng.randint(1, o))
    return out


def tables(pool, H, rids, max_rows):
    W = 2 * H
    rowrec, rowlist = [], np.zeros((len(rids), max_rows), np.int32)
    for s, rid in enumerate(rids):
        t = pool.block_table(0, rid)
        for r in range(len(t) // W):
            rowlist[s, r] = len(rowrec)
            rowrec.append(t[r * W:(r + 1) * W])
    return np.array(rowrec, np.int32).reshape(-1, W), rowlist


def run(B, H, long_ctx=None, sets=4, iters=20, seed=0):
    rng = random.Random(seed)
    spec = mux.LLMSpec("k1", 1, H, 128, H * 128, 1, 2)
    ctx_sets = [contexts(rng, B, long_ctx) for _ in range(sets)]
    rows_total = sum((c + 15) // 16 for cs in ctx_sets for c in cs)
    total = rows_total * 2 * H + 4096
    pool = mux.BlockPool(total, physical=True)
    pool.register_llm(0, spec)
    pool.set_quota(0, total)
    # churn so the free stack is scattered
    live = []
    for k in range(200):
        rid = 10_000_000 + k
        if pool.admit(0, rid, rng.randrange(1, 64), 64).ok:
            live.append(rid)
        if live and rng.random() < 0.6:
            pool.free_request(0, live.pop(rng.randrange(len(live))))
    for rid in live:  # the free stack stays scrambled
        pool.free_request(0, rid)
    max_ctx = max(max(cs) for cs in ctx_sets)
    max_rows = (max_ctx + 15) // 16
    dev = []
    for si, cs in enumerate(ctx_sets):
        rids = [si * 100_000 + b for b in range(B)]
        for rid, c in zip(rids, cs):
            assert pool.admit(0, rid, c, c).ok
        rr, rl = tables(pool, H, rids, max_rows)
        dev.append((torch.from_numpy(rr).cuda(), torch.from_numpy(rl).cuda(),
                     torch.tensor(cs, dtype=torch.int32, device="cuda")))
    kv = torch.empty(total * 2048, dtype=torch.bfloat16, device="cuda").normal_(0, 0.25)
    q = torch.randn(B, H, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, H, 128, device="cuda", dtype=torch.bfloat16)
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ws = torch.empty(B * H * 16 * 130, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    # KV splits as the runtime picks them (device/runtime.cu decode): enough
    # CTAs to fill the GPU a few times over
    fill = int(os.environ.get("K1_FILL", "4"))  # CTAs per SM the split heuristic aims for
    min_rows = int(os.environ.get("K1_MIN_ROWS", "2"))
    splits = 1
    while splits < 16 and B * H * splits < fill * 148 and (max_rows + splits * 2 - 1) // (splits * 2) >= min_rows:
        splits *= 2

    def launch(i):
        rr, rl, cx = dev[i % sets]
        mux.decode_attention_headwise(q, kv, rr, rl, slots, cx, 1, 0, max_rows, max_ctx, out, kv_splits=splits,
                                      workspace=ws, stream=stream.cuda_stream)
    for i in range(sets):
        launch(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        launch(i)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    byts = sum(sum(cs) * H * 512 + B * H * 512 for cs in ctx_sets) / sets
    return us, byts / (us * 1e-6) / 1e9, sum(map(sum, ctx_sets)) / (sets * B)


if __name__ == "__main__":
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    print(f"K1 one layer, CUDA events; peak {peak:.0f} GB/s measured, 8000 nominal")
    Bs = [int(x) for x in os.environ.get("K1_BATCHES", "1,4,16,64,128,196").split(",")]
    for H, name in ((32, "7B"), (40, "13B")):
        for B in Bs:
            us, gbs, mean_ctx = run(B, H)
            print(f"{name} H={H} B={B:3d} mean ctx {mean_ctx:6.0f}: {us:8.1f} us {gbs:7.0f} GB/s "
                  f"{gbs / peak:6.1%} of measured {gbs / 8000:6.1%} of nominal", flush=True)
        us, gbs, mean_ctx = run(128, H, long_ctx=4096, sets=2, iters=10)
        print(f"{name} H={H} B=128 ctx 4096 (long): {us:8.1f} us {gbs:7.0f} GB/s "
              f"{gbs / peak:6.1%} of measured {gbs / 8000:6.1%} of nominal", flush=True)
