#!/usr/bin/env python3
"""Benchmark: aggregate decode tokens/s of colocated LLMs on B200 + the
paged-attention kernel's HBM roofline fraction (BASELINE.json metric).

Workload (BASELINE config 2): LLaMA-7B + LLaMA-13B (random-init weights)
colocated on one B200 over ONE unified head-wise KV pool sized like the
reference's (180 GiB mesh, 10% activation reserve, sim_engine.cpp:172-186).
Each model holds a decode batch of B requests with ShareGPT-shaped lengths
(lognormal mean 161 prompt / 338 output, sigma 0.8, workload.hpp:21) caught
mid-generation. One step = one ADBS decode round (scheduler.cpp:90-117):
BlockPool.alloc(+1 token) for every member of both models, then both decode
jobs run concurrently, each on its own green-context SM partition sized by
its share of the round's HBM bytes (byte_share_partitions; full 32/40-layer
forward: tcgen05 GEMMs, RoPE+KV append, head-wise paged attention, LM head,
greedy argmax). Tokens per step = 2B.

N GPUs (torchrun): every rank serves its own independent 7B+13B unit (units
share nothing, sim_engine.hpp:74-80) -> weak scaling, no collective on the
data path; timing is the max over ranks.

--impl reference: the CPU restatement of the same decode round (bench_cpu.py:
oracle/llama_ref.decode_batch + oracle/numerics_ref.c attention, all host
threads), every step a full round of both models timed end to end, on this
arm's config; it never imports the product package.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30
MESH_BYTES = int(180 * GIB)
RESERVE = 0.1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def k1_traffic():
    """DRAM bytes of one K1 launch from the committed ncu capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_k1_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def gemm_traffic():
    """DRAM bytes of one decode GEMM launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_gemm_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


# LLMSpec.weight_bytes of the reference catalog (config.cpp:15-18)
WEIGHT_BYTES = {"7b": int(13.5e9), "13b": int(26e9), "30b": int(65e9), "65b": int(130e9)}


def pool_blocks(models):
    """UnitSim::pool_blocks (sim_engine.cpp:172-186) on one 180 GiB GPU."""
    weights = sum(WEIGHT_BYTES[m] for m in models)
    reserve = round(RESERVE * MESH_BYTES)
    return (MESH_BYTES - weights - reserve) // 4096


def workload_config(args, world):
    """The config dict both arms print (identical, so the driver's
    ours-vs-reference ratio compares the same workload)."""
    models = args.models.split(",")
    if args.placement and world > 1:
        units = placement_plan(args.placement, world)
        return {
            "workload": f"cfg4 placement ({args.placement}/plan_g{world}.json, unmodified reference planner): "
                        "one unit per rank, one ADBS decode round of every colocated model per step",
            "units": [",".join(u) for u in units], "decode_batch_per_model": f"<= {args.batch} (fits the unit pool)",
            "contexts": "ShareGPT lognormal prompt 161 / output 338 (sigma 0.8), members mid-generation, "
                        "seed 1000 + rank (bench.sample_batch)",
            "l2": "inputs larger than L2 (weights + KV per step)",
            "parallelism": f"{world} placed units (one per GPU, no data-path collective)",
        }
    return {
        "workload": "cfg2: LLaMA-7B + LLaMA-13B colocated per B200, one ADBS decode round per step",
        "models": args.models, "decode_batch_per_model": args.batch,
        "contexts": "ShareGPT lognormal prompt 161 / output 338 (sigma 0.8), members mid-generation, "
                    "seed 1000 + rank (bench.sample_batch)",
        "pool_blocks": pool_blocks(models),
        "l2": "inputs larger than L2 (39.5 GB weights + KV per step)",
        "parallelism": f"{world} independent units (dp{world})",
    }


def placement_plan(name, world):
    """A committed placement for a box of `world` GPUs
    (scripts/<name>/plan_g<world>.json, made by the unmodified reference
    planner) as the model-catalog names each rank (GPU) serves: its tp = 1
    unit's models, or none for a GPU of an empty mesh."""
    with open(os.path.join(ROOT, "scripts", name, f"cfg_g{world}.json")) as f:
        cfg = json.load(f)
    with open(os.path.join(ROOT, "scripts", name, f"plan_g{world}.json")) as f:
        plan = json.load(f)
    model_of = {e["name"]: e["model"] for e in cfg["llms"]}
    ranks = [None] * world
    for u in plan["units"]:
        models = [model_of[m["name"]] for m in u["models"]]
        if models and len(u["gpu_ids"]) != 1:
            raise ValueError("bench --placement runs tp = 1 units (one per rank)")
        for g in u["gpu_ids"]:  # an empty mesh idles all of its GPUs
            if not 0 <= g < world or ranks[g] is not None:
                raise ValueError(f"plan maps GPU {g} twice or outside the box")
            ranks[g] = models
    if any(r is None for r in ranks):
        raise ValueError("plan leaves a GPU of the box unmapped")
    return ranks


def unit_models(args, rank, world):
    """The models this rank's unit serves: --models (every rank its own
    copy, the default), or unit `rank` of a committed placement."""
    if args.placement and world > 1:
        return placement_plan(args.placement, world)[rank]
    return args.models.split(",")


def idle_result(args, world):
    """A rank whose mesh holds no model: it only joins the barriers."""
    import torch
    if world > 1:
        torch.distributed.barrier()
    return {"ms": 0.0, "tokens": 0, "launches": 0, "attn_ms": 0.0, "attn_n": 0, "attn_bytes": 0.0,
            "clocks": {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["idle rank"]}, "gemm_ms": 0.0, "gemm_n": 0,
            "gemm_bytes": 0.0, "gs_ms": 0.0, "gs_n": 0, "gs_bytes": 0.0, "e2e_ms": 0.0, "bytes_step": 0.0, "partition_sms": None, "job_ms_per_step": [],
            "models": [], "batch": 0}


def projection_bytes(s):
    """Weight bytes one decode job streams through the GEMMs: QKV, O,
    gate-up, down per layer and the LM head (bf16)."""
    h, f = s.hidden_size, s.ffn
    return 2 * (s.num_layers * (3 * h * h + h * h + 2 * f * h + f * h) + s.vocab * h)


def sample_batch(rng, B, extra_steps):
    """ShareGPT-shaped requests mid-generation: (prompt, output, steps_done)."""
    import numpy as np
    mu_p = math.log(161.0) - 0.32
    mu_o = math.log(338.0) - 0.32
    out = []
    while len(out) < B:
        p = max(1, int(round(rng.lognormal(mu_p, 0.8))))
        o = max(1, int(round(rng.lognormal(mu_o, 0.8))))
        if o < extra_steps + 2 or p + o > 4000:
            continue
        done = int(rng.integers(0, o - extra_steps - 1))
        out.append((p, o, done))
    return out


class Clocks:
    def __init__(self, index: int):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{index}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def wait_started(self, timeout_s: float = 5.0):
        """Wait for nvidia-smi's first (idle) sample; samples up to here are
        dropped by stop(), so the reported clocks are the ones under load."""
        self.skip = 0
        if self.proc is None:
            return
        t0 = time.time()
        while time.time() - t0 < timeout_s:
            self.f.flush()
            with open(self.path) as f:
                n = sum(1 for _ in f)
            if n:
                self.skip = n
                return
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for i, line in enumerate(open(self.path)):
            if i < getattr(self, "skip", 0):
                continue
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ our arm

def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2404_02015_b200 as mux

    device = local_rank if torch.cuda.device_count() > local_rank else 0
    torch.cuda.set_device(device)
    local_rank = device
    models = unit_models(args, rank, world)
    if not models:  # an empty mesh of the placement: this rank serves nothing
        return idle_result(args, world)
    specs = [mux.spec(m) for m in models]
    steps_total = 2 * args.warmup + args.steps + args.e2e_steps + args.attn_steps + 2
    logical = pool_blocks(models)
    B = args.batch
    while True:  # the largest batch <= --batch whose members fit the unified pool
        rng = np.random.default_rng(1000 + rank)
        batches = [sample_batch(rng, B, steps_total) for _ in specs]
        need = sum(mux.blocks_for_tokens(s, 16, p + d + steps_total + 1)
                   for s, reqs in zip(specs, batches) for p, o, d in reqs)
        if need <= logical or B == 1:
            break
        B = max(1, B * 3 // 4)
    assert need <= logical, "batch exceeds the unified pool"
    max_ctx = max(p + d + steps_total + 1 for reqs in batches for p, o, d in reqs)
    if args.partition_sms == "auto" and len(specs) == 1:
        psms = None
    elif args.partition_sms == "auto":
        ctx = [sum(p + d for p, o, d in reqs) for reqs in batches]
        psms = mux.byte_share_partitions(specs, ctx, torch.cuda.get_device_properties(device).multi_processor_count)
    elif args.partition_sms in ("none", "", None):
        psms = None
    else:
        psms = [int(x) for x in args.partition_sms.split(",")]
    args.partition_resolved = psms
    unit = mux.Unit(specs, pool_blocks=logical, device=local_rank, device_pool_blocks=need + 4096,
                    max_batch=B, max_prefill_tokens=256, max_ctx=max_ctx + 16, max_slots=len(specs) * B + 16,
                    init_seed=1 + rank, init_std=0.02, partitions=len(specs) + 1,
                    partition_sms=[0] + psms if psms else None)
    unit.set_option("pdl", args.pdl)
    if args.gemm_min_iters > 0:
        unit.set_option("gemm_min_iters", args.gemm_min_iters)
    unit.init_kv(seed=7 + rank, std=1.0)
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
    # jobs are enqueued heaviest first (most bytes per round): the host issues
    # ~8 launches per layer, and the longest job should not wait behind the
    # enqueue of the others (matters for the e2e loop, which syncs each step)
    issue_order = sorted(range(len(specs)), key=lambda li: -(specs[li].weight_bytes + sum(
        p + d for p, o, d in batches[li]) * specs[li].kv_bytes_per_token()))
    ctx0 = [sum(pool.request_tokens(li, r) for r in ids[li]) for li in range(len(specs))]

    def alloc_round():
        # one ADBS decode round's allocation: +1 token per member (BlockPool)
        for li in issue_order:
            if not pool.alloc_n_ok(li, ids_c[li], 1, False):
                raise RuntimeError("pool exhausted")

    def issue_round(tokens=None, outs=None, whole_gpu=False):
        for li in issue_order:
            unit.decode(li, ids[li], tokens=None if tokens is None else tokens[li],
                        out=None if outs is None else outs[li], partition=0 if whole_gpu else 1 + (0 if args.serial else li),
                        ids_c=ids_c[li])

    def step(tokens=None, outs=None, whole_gpu=False):
        # one ADBS decode round: the allocation, then the jobs
        alloc_round()
        issue_round(tokens, outs, whole_gpu)

    # clocks are sampled from the warm-up on (the timed region alone is only
    # a few hundred ms): idle samples before the first step are dropped
    clocks = Clocks(local_rank)
    clocks.wait_started()
    for _ in range(args.warmup):
        step()
    unit.sync()
    if world > 1:
        torch.distributed.barrier()
    launches0 = unit.launches()
    unit.sync()
    for li in range(len(specs)):
        unit.record(1 + li, 2 * li)
    for _ in range(args.steps):
        step()
    for li in range(len(specs)):
        unit.record(1 + li, 2 * li + 1)
    unit.sync()
    # span from the first partition's start to the last partition's end
    part_ms = [unit.elapsed_ms(0, 2 * li + 1) for li in range(len(specs))]
    ms = max(part_ms)
    launches = unit.launches() - launches0
    clk = clocks.stop()

    # K1 roofline: CUDA events around every decode-attention launch, on its
    # stream, over separate steps of the same workload. The kernel is timed
    # alone on the whole GPU (both jobs on partition 0, the ungreened stream):
    # on a green partition it only owns that partition's share of HBM. PDL is
    # off for these steps: with it, the event pair around a K1 launch would
    # also span the kernel's programmatic overlap.
    unit.set_option("pdl", 0)
    unit.attn_timing(True)
    for _ in range(args.attn_steps):
        step(whole_gpu=True)
    unit.sync()
    attn_ms, attn_n, attn_bytes = unit.attn_time()
    gemm_ms, gemm_n, gemm_bytes = unit.gemm_time()
    unit.attn_timing(False)
    unit.set_option("pdl", args.pdl)

    # Decode-GEMM stream: steps whose decode jobs run only the projections
    # (K1, K2 and RMSNorm skipped: option debug_skip; outputs are garbage),
    # both models back to back on the whole-GPU stream with PDL as in the
    # step, CUDA events around each job. Per-launch events (above) add each
    # kernel's launch latency and turn PDL off; ncu's serialised durations
    # sit between the two.
    gs_ms = gs_bytes = 0.0
    gs_n = 0
    if args.attn_steps > 0:
        unit.set_option("debug_skip", 7)
        for _ in range(args.attn_steps + 1):
            unit.sync()
            unit.record(0, 60)
            step(whole_gpu=True)
            unit.record(0, 61)
            unit.sync()
            if _ == 0:
                continue  # warm-up of the skip configuration
            gs_ms += unit.elapsed_ms(60, 61)
            for s in specs:
                gs_bytes += projection_bytes(s)
                gs_n += 4 * s.num_layers + 1
        unit.set_option("debug_skip", 0)

    # e2e: host token ids in (pinned) -> jobs -> next tokens out (pinned), each
    # step waits for its result before the next, as a serving loop does.
    pinned_in = [torch.zeros(B, dtype=torch.int32).pin_memory().numpy() for _ in specs]
    pinned_out = [torch.zeros(B, dtype=torch.int32).pin_memory().numpy() for _ in specs]
    # untimed warm-up of the host-token path: its decode jobs are separate
    # CUDA-graph keys (captured on a key's second use, runtime.cu)
    for _ in range(args.warmup if args.e2e_steps else 0):
        step(tokens=pinned_in, outs=pinned_out)
        unit.sync()
    unit.sync()
    t0 = time.perf_counter()
    if args.e2e_steps:
        alloc_round()
    for i in range(args.e2e_steps):
        issue_round(tokens=pinned_in, outs=pinned_out)
        if i + 1 < args.e2e_steps:
            alloc_round()  # the next round's KV rows while this one runs (host state only)
        unit.sync()  # the step's result is on the host before the next step is issued
        for li in range(len(specs)):
            pinned_in[li][:] = pinned_out[li]
    # wall clock of the serving loop through the public API (host timer)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / max(1, args.e2e_steps)

    # step roofline: weights + KV bytes of both jobs per step
    kv_tok = [s.kv_bytes_per_token() for s in specs]
    bytes_step = 0.0
    for li, s in enumerate(specs):
        ctx_mid = ctx0[li] + B * (args.warmup + args.steps / 2 + 1)  # the timed steps' mid-point
        bytes_step += s.weight_bytes + ctx_mid * kv_tok[li]
    unit_sms = [unit.partition_sms(1 + li) for li in range(len(specs))]
    unit.close()
    result = {
        "ms": ms, "tokens": len(specs) * B * args.steps, "launches": launches,
        "attn_ms": attn_ms, "attn_n": attn_n, "attn_bytes": attn_bytes, "clocks": clk,
        "gemm_ms": gemm_ms, "gemm_n": gemm_n, "gemm_bytes": gemm_bytes,
        "gs_ms": gs_ms, "gs_n": gs_n, "gs_bytes": gs_bytes,
        "e2e_ms": e2e_ms, "bytes_step": bytes_step, "models": models, "batch": B,
        "partition_sms": [unit_sms[li] for li in range(len(specs))] if psms else None,
        "job_ms_per_step": [round(x / args.steps, 3) for x in part_ms],
    }
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=128, help="decode members per model")
    ap.add_argument("--models", default="7b,13b")
    ap.add_argument("--placement", default="",
                    help="N > 1: run unit `rank` of the committed placement scripts/<name>/plan_g<N>.json "
                         "(e.g. c4: BASELINE config 4) instead of N copies of --models")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--attn-steps", type=int, default=2, help="steps with per-launch K1 events")
    ap.add_argument("--partition-sms", default="auto",
                    help="green-context SMs of each model's decode partition: 'auto' (shares of the per-round "
                         "HBM bytes, byte_share_partitions), 'none' (every job on the whole GPU), or e.g. 56,88")
    ap.add_argument("--serial", action="store_true", help="run the colocated decode jobs on one stream")
    ap.add_argument("--serve-measured", action="store_true",
                    help="also run the pass-serialised measured engine on the serving trace")
    ap.add_argument("--serve-horizon", type=float, default=10.0,
                    help="seconds of Poisson arrivals for the auxiliary measured serving run (0 = skip)")
    ap.add_argument("--pdl", type=int, default=1, help="programmatic dependent launch between job kernels")
    ap.add_argument("--skip-cpu", action="store_true", help="omit the cpu_baseline leg (profiling runs)")
    ap.add_argument("--gemm-min-iters", type=int, default=0,
                    help="decode GEMM k-blocks-per-CTA floor (0 = the runtime default)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        from bench_cpu import reference_arm
        print(json.dumps(reference_arm(args, workload_config(args, world))), flush=True)
        return

    import torch
    if world > 1:
        # one GPU per rank -> NCCL; MUX_DIST_BACKEND=gloo lets several ranks
        # share one GPU (a test of this multi-rank path, not a measurement)
        backend = os.environ.get("MUX_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(backend)
    r = run_ours(args, rank, world, local_rank)
    from paper_2404_02015_b200 import mesh
    ms, e2e_ms, max_bytes_step = mesh.max_over_ranks([r["ms"], r["e2e_ms"], r["bytes_step"]])  # slowest rank
    # every rank's own unit: tokens, launches and the kernel timings add up
    # (ranks of a placement serve different models; idle ranks add zero)
    keys = ["tokens", "launches", "attn_ms", "attn_n", "attn_bytes", "gemm_ms", "gemm_n", "gemm_bytes", "gs_ms", "gs_n",
            "gs_bytes"]
    tot = dict(zip(keys, mesh.sum_over_ranks([float(r[k]) for k in keys])))
    unit_models_all = mesh.gather_objects({"models": r["models"], "batch": r["batch"]})
    tokens = tot["tokens"]
    if rank == 0:
        r = dict(r, **tot, bytes_step=max_bytes_step)
    hbm, peak_kind = peaks()
    achieved = r["attn_bytes"] / (r["attn_ms"] / 1e3) / 1e9 if r["attn_ms"] > 0 else 0.0
    value = tokens / (ms / 1e3)
    per_step_tokens = tokens / args.steps
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        from bench_cpu import cpu_baseline
        cpu = cpu_baseline(args)
    serving = None
    if rank == 0 and world == 1 and args.serve_horizon > 0:
        # the whole serving loop (ADBS engine, prefill + decode jobs, measured
        # device time) on the same two models: auxiliary, not the headline
        try:
            import serve
            rates = (120.0, 60.0)[:len(args.models.split(","))]
            # real-time engine: jobs overlap across ADBS passes and contend
            # for HBM as deployed (the serving number). 10 s of arrivals at
            # 120 + 60 rps overload the GPU ~4x, so tokens / makespan tends to
            # the engine's capacity rather than the drain of the last long
            # outputs; the pass-serialised measured engine beside
            # it on request
            serving = serve.serve(args.models.split(","), rates, args.serve_horizon, seed=3, device=local_rank,
                                  realtime=True)
            if args.serve_measured:
                serving["measured_engine"] = serve.serve(args.models.split(","), rates, args.serve_horizon, seed=3,
                                                         device=local_rank)
        except Exception as e:  # pragma: no cover - reported, never fatal for the headline
            serving = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        kt, gt = k1_traffic() or {}, gemm_traffic() or {}
        roof_k1 = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                   "frac": round(achieved / hbm, 4), "frac_nominal_8tbs": round(achieved / 8000.0, 4),
                   "traffic": kt.get("dram_bytes"), "traffic_note": kt.get("capture"),
                   "traffic_algorithmic_bytes": kt.get("algorithmic_bytes"),
                   "kernel": "decode_attention_kernel (K1, per-launch CUDA events, timed alone on the whole GPU)",
                   "peak_source": peak_kind, "launches_timed": r["attn_n"], "device_ms": round(r["attn_ms"], 3),
                   "bytes_per_launch": round(r["attn_bytes"] / max(1, r["attn_n"]))}
        g_ach = r["gemm_bytes"] / (r["gemm_ms"] / 1e3) / 1e9 if r["gemm_ms"] > 0 else 0.0
        s_ach = r["gs_bytes"] / (r["gs_ms"] / 1e3) / 1e9 if r["gs_ms"] > 0 else 0.0
        roof_gemm = {"bound": "hbm", "achieved": round(s_ach, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(s_ach / hbm, 4), "frac_nominal_8tbs": round(s_ach / 8000.0, 4),
                     "traffic": gt.get("dram_bytes"), "traffic_note": gt.get("capture"),
                     "traffic_algorithmic_bytes": gt.get("algorithmic_bytes"),
                     "kernel": "gemm_tn_kernel (K4 decode projections QKV/O/gate-up/down/LM head of both models, "
                               "launched back to back on the whole GPU as in the step, PDL on, K1/K2/RMSNorm skipped; "
                               "CUDA events around each job; algorithmic bytes = the weights, N*K*2)",
                     "peak_source": peak_kind, "launches_timed": int(r["gs_n"]), "device_ms": round(r["gs_ms"], 3),
                     "bytes_per_launch": round(r["gs_bytes"] / max(1, r["gs_n"])),
                     "isolated_launches": {"achieved": round(g_ach, 1), "frac": round(g_ach / hbm, 4),
                                           "launches_timed": r["gemm_n"], "device_ms": round(r["gemm_ms"], 3),
                                           "method": "CUDA events around every launch, PDL off (adds each "
                                                     "launch's latency)"}}
        # whole-job roofline: every rank streams its own weights + KV per step,
        # the step lasts as long as the rank with the most bytes
        step_roof = per_step_tokens / (r["bytes_step"] / (hbm * 1e9)) if r["bytes_step"] else None
        line = {
            "metric": "aggregate decode tokens/s across colocated LLMs; paged-attn HBM GB/s vs peak",
            "value": round(value, 1),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init weights, ShareGPT-shaped lognormal lengths, random KV)",
            "config": workload_config(args, world),
            "run": {"partition_sms": r["partition_sms"], "job_ms_per_step": r["job_ms_per_step"],
                    "units": unit_models_all},
            "e2e": {"value": round(per_step_tokens / (e2e_ms / 1e3), 1) if e2e_ms else None,
                    "unit": "tokens/s", "h2d_bytes_per_step": int(per_step_tokens * 4),
                    "d2h_bytes_per_step": int(per_step_tokens * 4)},
            # the dominant kernel by device time over the timed launches (the
            # decode GEMMs), K1 beside it
            # (dominance by the per-launch-event device times of the same
            # steps, the method K1 is timed with; ncu's launch list agrees)
            "roofline": roof_gemm if r["gemm_ms"] >= r["attn_ms"] else roof_k1,
            "roofline_secondary": roof_k1 if r["gemm_ms"] >= r["attn_ms"] else roof_gemm,
            "step_roofline": {"tokens_per_s_at_peak": round(step_roof, 1) if step_roof else None,
                              "frac": round(value / step_roof, 4) if step_roof else None,
                              "frac_nominal_8tbs": round(value / (step_roof * 8000.0 / hbm), 4) if step_roof else None},
            "cpu_baseline": cpu,
            "serving": serving,
            "gpu_launches": int(r["launches"]),
            "clocks": r["clocks"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
