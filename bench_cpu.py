"""CPU legs of bench.py (the only bench code that touches oracle/).

cpu_baseline(args): the oracle port of one decode step (oracle/numerics_ref.c:
bf16 GEMVs for QKV/O/gate-up/down + LM head, head-wise paged attention), on
all host threads, over a bounded sample -- ONE layer of each colocated model
at the bench's decode batch and contexts -- scaled to the full step
(layers x per-layer time + LM head). Plus the reference simulator's own hot
loop (oracle/_ref/ref_hotloop: run_simulation, 1 core) as context.

reference_arm(args): bench.py --impl reference; times that same CPU port per
step and prints the reference-arm JSON line.
"""
from __future__ import annotations

import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _rand_bf16(rng, n):
    import numpy as np
    # |x| in [2^-7, 2^-6) with random sign and mantissa: finite, weight-like.
    mant = rng.integers(0, 128, n, dtype=np.uint16)
    sign = rng.integers(0, 2, n, dtype=np.uint16) << 15
    return (sign | np.uint16(0x3C00) | mant).astype(np.uint16)


class StepSample:
    """One layer of each model + its LM head, on the host cores."""

    def __init__(self, models, batch, seed=0):
        import numpy as np

        import paper_2404_02015_b200 as mux
        from oracle import refs
        self.lib = refs.numerics()
        self.threads = os.cpu_count() or 1
        rng = np.random.default_rng(seed)
        self.models = []
        for m in models:
            s = mux.spec(m)
            H, hid, ffn, V = s.num_heads, s.hidden_size, s.ffn, s.vocab
            ctx = []
            while len(ctx) < batch:
                p = int(round(rng.lognormal(math.log(161) - 0.32, 0.8)))
                o = int(round(rng.lognormal(math.log(338) - 0.32, 0.8)))
                if 1 <= p and 2 <= o and p + o <= 4000:
                    ctx.append(p + 1 + int(rng.integers(0, o - 1)))
            rows = [(c + 15) // 16 for c in ctx]
            nrows = sum(rows)
            W = 2 * 1 * H  # one layer
            pool_blocks = nrows * W
            rowrec = np.arange(pool_blocks, dtype=np.int32).reshape(nrows, W)
            rng.shuffle(rowrec.reshape(-1))  # scattered blocks
            max_rows = max(rows)
            rowlist = np.zeros((batch, max_rows), np.int32)
            k = 0
            for b, r in enumerate(rows):
                rowlist[b, :r] = np.arange(k, k + r)
                k += r
            self.models.append(dict(
                spec=s, ctx=np.array(ctx, np.int32), rowrec=rowrec, rowlist=rowlist, max_rows=max_rows,
                pool=_rand_bf16(rng, pool_blocks * 2048), q=_rand_bf16(rng, batch * H * 128),
                x=_rand_bf16(rng, batch * max(hid, ffn, H * 128)),
                wqkv=_rand_bf16(rng, 3 * H * 128 * hid), wo=_rand_bf16(rng, hid * H * 128),
                wgu=_rand_bf16(rng, 2 * ffn * hid), wdown=_rand_bf16(rng, hid * ffn),
                lm=_rand_bf16(rng, V * hid), y=np.zeros(batch * max(3 * H * 128, 2 * ffn, V), np.float32),
                att=np.zeros(batch * H * 128, np.float32)))
        self.batch = batch

    def run(self):
        """Returns (full-step seconds estimate, sampled seconds)."""
        B, T = self.batch, self.threads
        est, sampled = 0.0, 0.0
        for m in self.models:
            s = m["spec"]
            H, hid, ffn, V = s.num_heads, s.hidden_size, s.ffn, s.vocab
            g = lambda w, N, K: self.lib.ref_gemv_bf16(m["x"].ctypes.data, m[w].ctypes.data,
                                                      m["y"].ctypes.data, B, N, K, T)
            t0 = time.perf_counter()
            g("wqkv", 3 * H * 128, hid)
            self.lib.ref_decode_attention(m["q"].ctypes.data, m["pool"].ctypes.data, m["rowrec"].ctypes.data,
                                          m["rowlist"].ctypes.data,
                                          __import__("numpy").arange(B, dtype="int32").ctypes.data,
                                          m["ctx"].ctypes.data, B, H, 1, 0, m["max_rows"],
                                          m["att"].ctypes.data, T)
            g("wo", hid, H * 128)
            g("wgu", 2 * ffn, hid)
            g("wdown", hid, ffn)
            t_layer = time.perf_counter() - t0
            t0 = time.perf_counter()
            g("lm", V, hid)
            t_lm = time.perf_counter() - t0
            est += s.num_layers * t_layer + t_lm
            sampled += t_layer + t_lm
        return est, sampled


def _ref_sim():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_hotloop")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "600"], capture_output=True, text=True, timeout=120).stdout
        d = json.loads(out)
        return {"decode_decisions_per_s": round(d["decisions_per_s"], 1), "cores": 1,
                "what": "unmodified reference run_simulation (oracle/_ref), cfg2 analogue 7B@20+13B@10 rps, "
                        "600 s simulated; prices jobs, computes no tokens"}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def cpu_baseline(args, min_seconds: float = 10.0):
    """Repeats the one-layer sample until >= min_seconds of CPU work (bounded
    sample of the same workload), reports the mean full-step estimate."""
    models = args.models.split(",")
    smp = StepSample(models, args.batch)
    ests, sampled, reps = [], 0.0, 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < min_seconds or reps < 2:
        est, s = smp.run()
        ests.append(est)
        sampled += s
        reps += 1
    est = sum(ests) / len(ests)
    tokens = len(models) * args.batch
    return {"value": round(tokens / est, 3), "unit": "tokens/s", "cores": smp.threads, "kind": "port",
            "sample": f"{reps} x (1 layer + LM head of each of {models}) at decode batch {args.batch} "
                      f"(ShareGPT contexts), scaled by layer count; {sampled:.1f} s of CPU work sampled",
            "reference_sim": _ref_sim()}


def reference_arm(args):
    models = args.models.split(",")
    smp = StepSample(models, args.batch)
    for _ in range(min(args.warmup, 1)):
        smp.run()
    ests = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ests.append(smp.run()[0])
    wall = time.perf_counter() - t0
    tokens = len(models) * args.batch
    value = tokens * args.steps / sum(ests)
    return {
        "impl": "reference",
        "metric": "aggregate decode tokens/s across colocated LLMs; paged-attn HBM GB/s vs peak",
        "value": round(value, 3), "unit": "tokens/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * sum(ests) / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": {"workload": "cfg2: LLaMA-7B + LLaMA-13B decode round",
                                        "models": args.models, "decode_batch_per_model": args.batch},
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": smp.threads, "kind": "port",
                         "sample": f"per step: 1 layer + LM head per model, scaled by layer count "
                                   f"({wall:.1f} s wall for {args.steps} steps)",
                         "reference_sim": _ref_sim()},
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
