"""CPU legs of bench.py: the reference arm (`bench.py --impl reference`) and
the cpu_baseline leg of our own arm. Baseline infrastructure: the only bench
code that executes oracle/, and it never imports the product package
(paper_2404_02015_b200) -- it is the CPU restatement of the same decode
round, run on the host cores.

One step = the FULL decode round bench.py's GPU arm times, for every member
of every colocated model (same models, batch, ShareGPT contexts and seed as
the GPU arm's rank 0): embedding, for every layer RMSNorm -> QKV projection
-> RoPE + K/V append into 16-token head-blocks -> paged attention over the
member's whole context -> O projection + residual -> RMSNorm -> gate/up ->
SiLU*up -> down + residual, then the LM head and greedy argmax
(oracle/llama_ref.decode_batch; attention in C, oracle/numerics_ref.c, on all
host threads; projections through numpy's multithreaded BLAS in fp32).
Bounded sample: the L layers of a model share ONE layer's weights and one
layer's K/V head-blocks (aliased, so host memory stays ~6 GB instead of
~95 GB). Every layer still streams its full weight and K/V bytes -- each
layer's working set (0.8-1.3 GB weights, 0.7-0.9 GB K/V) is far larger than
the host caches -- and does its full arithmetic; nothing is skipped or
extrapolated: every reported step is timed end to end.
"""
from __future__ import annotations

import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# LLaMA-1 dims: (layers, heads, hidden, ffn, vocab); layers/heads/hidden from
# the reference catalog (config.cpp:15-18), ffn/vocab from LLaMA-1.
DIMS = {"7b": (32, 32, 4096, 11008, 32000), "13b": (40, 40, 5120, 13824, 32000),
        "30b": (60, 52, 6656, 17920, 32000), "65b": (80, 64, 8192, 22016, 32000)}
BUDGET_S = 150.0  # wall-clock budget of the reference arm's timed steps


def _rand_bf16(rng, shape):
    """bf16 bit patterns with |x| in [2^-7, 2^-6) and random sign (weight-like)."""
    import numpy as np
    n = int(np.prod(shape))
    mant = rng.integers(0, 128, n, dtype=np.uint16)
    sign = rng.integers(0, 2, n, dtype=np.uint16) << 15
    return (sign | np.uint16(0x3C00) | mant).astype(np.uint16).reshape(shape)


class CpuUnit:
    """The colocated models of one unit, decoding their batches on the CPU."""

    def __init__(self, models, batch, seed=0, rank=0, extra_steps=64):
        import numpy as np

        import bench
        from oracle import llama_ref, refs
        self.np, self.llama_ref, self.refs = np, llama_ref, refs
        self.threads = os.cpu_count() or 1
        rng = np.random.default_rng(seed)
        ctx_rng = np.random.default_rng(1000 + rank)  # bench.py's member sample (rank's seed)
        steps_total = extra_steps
        self.models = []
        for name in models:
            L, H, hid, ffn, V = DIMS[name]
            f = llama_ref.bf16_to_f32
            wqkv = f(_rand_bf16(rng, (3 * H * 128, hid)))
            wo = f(_rand_bf16(rng, (hid, H * 128)))
            wgu = f(_rand_bf16(rng, (2 * ffn, hid)))
            wdown = f(_rand_bf16(rng, (hid, ffn)))
            norm = (1.0 + 0.1 * rng.standard_normal(hid)).astype(np.float32)
            ref = llama_ref.RefLlama.__new__(llama_ref.RefLlama)
            ref.d = llama_ref.Dims(L, H, hid, ffn, V)
            ref.embed = f(_rand_bf16(rng, (V, hid)))
            ref.lm_head = f(_rand_bf16(rng, (V, hid)))
            ref.final_norm = norm
            ref.wqkv, ref.wo, ref.wdown = [wqkv] * L, [wo] * L, [wdown] * L  # aliased layers
            ref.wg, ref.wu = [np.ascontiguousarray(wgu[0::2])] * L, [np.ascontiguousarray(wgu[1::2])] * L
            ref.attn_norm, ref.ffn_norm = [norm] * L, [norm] * L
            # members caught mid-generation (bench.sample_batch), ctx incl. the new token
            reqs = bench.sample_batch(ctx_rng, batch, steps_total)
            ctx = np.array([p + d + 1 for p, o, d in reqs], np.int32)
            rows = (ctx + steps_total + 15) // 16
            W = 2 * H  # one (aliased) layer of head-blocks per row
            rowrec = rng.permutation(int(rows.sum()) * W).astype(np.int32).reshape(-1, W)  # scattered ids
            rowlist = np.zeros((batch, int(rows.max())), np.int32)
            k = 0
            for b, r in enumerate(rows):
                rowlist[b, :r] = np.arange(k, k + r)
                k += r
            blocks = _rand_bf16(rng, (int(rows.sum()) * W, 2048))
            ref.rope = llama_ref.rope_table(int(ctx.max()) + steps_total + 16)
            self.models.append(dict(name=name, ref=ref, ctx=ctx, rowrec=rowrec, rowlist=rowlist, blocks=blocks,
                                    tokens=rng.integers(0, V, batch).astype(np.int64), H=H))
        self.batch = batch
        self.steps_left = steps_total - 1  # rows exist for this many more steps

    def _attend(self, m):
        np, llama_ref, refs = self.np, self.llama_ref, self.refs
        H, ctx, B = m["H"], m["ctx"], self.batch
        blk = m["blocks"].reshape(-1, 16, 128)
        pos = ctx - 1
        rec = m["rowlist"][np.arange(B), pos // 16]
        kcol = np.arange(H) * 2

        def attend(layer, q, k, v):
            # K2: the new token's rotated k and its v into slot pos % 16 of its head-blocks
            ids = m["rowrec"][rec][:, kcol]  # [B, H]
            blk[ids, (pos % 16)[:, None]] = llama_ref.f32_to_bf16(k)
            blk[m["rowrec"][rec][:, kcol + 1], (pos % 16)[:, None]] = llama_ref.f32_to_bf16(v)
            # K1: paged attention over every cached token (layer 0's blocks: aliased)
            return refs.decode_attention(llama_ref.f32_to_bf16(q), m["blocks"], m["rowrec"], m["rowlist"],
                                         np.arange(B, dtype=np.int32), ctx, 1, 0, m["rowlist"].shape[1],
                                         nthreads=self.threads)
        return attend

    def step(self):
        """One full decode round of every model; returns its wall seconds."""
        if self.steps_left <= 0:
            raise RuntimeError("CpuUnit: out of preallocated rows")
        self.steps_left -= 1
        t0 = time.perf_counter()
        for m in self.models:
            logits = self.llama_ref.decode_batch(m["ref"], m["tokens"], m["ctx"] - 1, self._attend(m))
            m["tokens"] = logits.argmax(axis=1)
            m["ctx"] = m["ctx"] + 1
        return time.perf_counter() - t0

    def tokens_per_step(self):
        return self.batch * len(self.models)


def _ref_sim():
    """The unmodified reference simulator's hot loop (oracle/_ref), context only."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_hotloop")
    if not os.path.exists(exe):
        return None
    try:
        import json
        out = subprocess.run([exe, "600"], capture_output=True, text=True, timeout=120).stdout
        d = json.loads(out)
        return {"decode_decisions_per_s": round(d["decisions_per_s"], 1), "cores": 1,
                "what": "unmodified reference run_simulation (oracle/_ref), cfg2 analogue 7B@20+13B@10 rps, "
                        "600 s simulated; prices jobs, computes no tokens"}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def _steps_total(args):
    # bench.run_ours draws its members with the same extra-steps margin
    return 2 * args.warmup + args.steps + args.e2e_steps + args.attn_steps + 2


def _sample_text(unit, n_steps, wall):
    return (f"{n_steps} full decode round(s) of {[m['name'] for m in unit.models]} at batch {unit.batch} "
            f"(bench.py rank-0 ShareGPT contexts), every layer computed, layer weights and K/V aliased to one "
            f"layer per model; {wall:.1f} s timed")


def cpu_baseline(args, min_seconds: float = 10.0):
    """cpu_baseline of our arm: one untimed round, then full rounds until
    >= min_seconds of timed CPU work (at least one)."""
    unit = CpuUnit(args.models.split(","), args.batch, rank=0, extra_steps=_steps_total(args))
    unit.step()
    times = []
    while not times or (sum(times) < min_seconds and unit.steps_left > 0):
        times.append(unit.step())
    value = unit.tokens_per_step() * len(times) / sum(times)
    return {"value": round(value, 3), "unit": "tokens/s", "cores": unit.threads, "kind": "port",
            "sample": _sample_text(unit, len(times), sum(times)), "reference_sim": _ref_sim()}


def reference_arm(args, config):
    """bench.py --impl reference: the CPU restatement of the same decode round
    on the host cores, on our arm's config; every step timed in full. Steps
    beyond BUDGET_S of wall time are not run (reported as steps_run)."""
    unit = CpuUnit(args.models.split(","), args.batch, rank=0, extra_steps=_steps_total(args))
    for _ in range(min(args.warmup, 1)):
        unit.step()
    times = []
    while len(times) < args.steps and unit.steps_left > 0 and (not times or sum(times) + times[-1] <= BUDGET_S):
        times.append(unit.step())
    wall = sum(times)
    value = unit.tokens_per_step() * len(times) / wall
    return {
        "impl": "reference",
        "metric": "aggregate decode tokens/s across colocated LLMs; paged-attn HBM GB/s vs peak",
        "value": round(value, 3), "unit": "tokens/s", "n_gpus": args.gpus, "steps": len(times),
        "steps_requested": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": round(1e3 * wall / len(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random weights, ShareGPT-shaped lognormal lengths, random KV)",
        "config": config,
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": unit.threads, "kind": "port",
                         "sample": _sample_text(unit, len(times), wall), "reference_sim": _ref_sim()},
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
