#!/usr/bin/env python3
"""Serving run: colocated LLMs on one B200 under the ADBS engine, every job's
completion at its measured device time (mux_unit_run_measured).

The workload is BASELINE config 2 shaped: LLaMA-7B + LLaMA-13B (random-init
weights) sharing one unified head-wise KV pool, Poisson arrivals, ShareGPT
lognormal lengths (mean 161 prompt / 338 output, sigma 0.8,
/root/reference/proj/include/muxsim/workload.hpp:21). Unlike bench.py's
decode rounds, this runs the whole serving loop: admissions with worst-case
reservation, ADBS prefill/decode passes under the token-block quotas, prefill
jobs (K3 + GEMMs) and decode jobs (K1 + GEMMs) on their SM partitions.

Reports aggregate decode tokens/s (generated tokens / makespan), request
throughput, TTFT and per-token latency.

    python serve.py --rates 20,10 --horizon 8
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30


def make_trace(models, rates, horizon_s, seed, max_len=2048):
    import numpy as np
    rng = np.random.default_rng(seed)
    reqs = []
    for llm, rate in enumerate(rates):
        t = 0.0
        while True:
            t += rng.exponential(1.0 / rate)
            if t >= horizon_s:
                break
            while True:
                p = max(1, int(round(rng.lognormal(math.log(161.0) - 0.32, 0.8))))
                o = max(1, int(round(rng.lognormal(math.log(338.0) - 0.32, 0.8))))
                if p + o <= max_len:
                    break
            reqs.append((t, llm, p, o))
    reqs.sort()
    return reqs


def arrival_window_throughput(timeline_csv, horizon_s):
    """Tokens/s produced by real-time jobs ending in [horizon/2, horizon]
    (device ms from the run's origin; one token per member per job)."""
    import csv
    lo, hi = 500.0 * horizon_s, 1000.0 * horizon_s
    tok = {"decode": 0, "prefill": 0}
    with open(timeline_csv) as f:
        for r in csv.DictReader(f):
            if lo <= float(r["end_ms"]) < hi:
                tok[r["kind"]] += int(r["batch"])
    return {"tok_s": round((tok["decode"] + tok["prefill"]) / (0.5 * horizon_s), 1),
            "decode_tok_s": round(tok["decode"] / (0.5 * horizon_s), 1),
            "window_s": [0.5 * horizon_s, horizon_s]}


def serve(model_names=("7b", "13b"), rates=(20.0, 10.0), horizon_s=8.0, seed=3, device=0, partition_sms=None,
          scheduler="adbs", gpu_memory_gib=180.0, lengths=None, prefill_on_partition=False, pass_green=None,
          realtime=False, align_decode=False, sm_route=False):
    """lengths: optional per-model (prompt, output) constants (contention runs).
    partition_sms: [0, sms of model 0's partition, ...] (static partitions).
    pass_green: per-model green partition SMs, used only by passes holding
    decode jobs of two or more models (whole-GPU streams otherwise).
    realtime: jobs overlap across scheduling passes and complete when their
    device events fire (mux_unit_run_realtime); default: each pass's jobs
    are timed together and the next pass starts after them (measured mode)."""
    import paper_2404_02015_b200 as mux
    specs = [mux.spec(m, f"{m}.{i}") for i, m in enumerate(model_names)]  # distinct names per unit
    raw = make_trace(specs, rates, horizon_s, seed)
    if lengths is not None:
        raw = [(t, llm, lengths[llm][0], lengths[llm][1]) for t, llm, _, _ in raw]
    trace = [mux.TraceRequest(i, llm, t, p, o) for i, (t, llm, p, o) in enumerate(raw)]
    if lengths is None:
        entries = [mux.Entry(s, rate, 161.0, 338.0) for s, rate in zip(specs, rates)]
    else:
        entries = [mux.Entry(s, rate, float(p), float(o)) for s, rate, (p, o) in zip(specs, rates, lengths)]
    gpu_mem = int(gpu_memory_gib * GIB)
    params = mux.EngineParams(scheduler={"adbs": 0, "fcfs": 1, "rr": 2}[scheduler])
    weights = sum(s.weight_bytes for s in specs)
    logical = (gpu_mem - weights - round(0.1 * gpu_mem)) // 4096
    n_parts = len(specs) + 1
    if pass_green is not None:
        if partition_sms is not None or len(pass_green) != len(specs):
            raise ValueError("pass_green takes one SM count per model and excludes partition_sms")
        n_parts, partition_sms = 2 * len(specs) + 1, [0] * (len(specs) + 1) + list(pass_green)
    unit = mux.Unit(specs, pool_blocks=logical, device=device, device_pool_blocks=logical,
                    max_batch=512, max_prefill_tokens=4096, max_ctx=2048 + 64, max_slots=len(trace) + 8,
                    init_seed=1, init_std=0.02, partitions=n_parts,
                    partition_sms=partition_sms)
    try:
        unit.set_option("prefill_on_partition", int(prefill_on_partition))
        unit.set_option("pass_green", int(pass_green is not None))
        unit.set_option("align_decode", int(align_decode))
        if sm_route:  # every job on a green context sized by its ADBS sm_demand
            unit.set_option("sm_route", 1)
        unit.init_kv(seed=5, std=1.0)
        # real-time runs: the device timeline of every job (MUX_RT_TIMELINE)
        # gives the tokens produced while arrivals are still coming in
        own_tl = None
        if realtime and not os.environ.get("MUX_RT_TIMELINE"):
            import tempfile
            own_tl = os.environ["MUX_RT_TIMELINE"] = os.path.join(tempfile.mkdtemp(), "timeline.csv")
        t0 = time.perf_counter()
        recs, _ = unit.run_lockstep(entries, trace, gpu_mem, params, measured=not realtime, realtime=realtime)
        wall = time.perf_counter() - t0
        passes, green_passes = unit.pass_stats()
    finally:
        unit.close()
    window = None
    tl = os.environ.get("MUX_RT_TIMELINE") if realtime else None
    if tl and os.path.exists(tl):
        window = arrival_window_throughput(tl, horizon_s)
    if own_tl:
        del os.environ["MUX_RT_TIMELINE"]
    out_tokens = sum(r.output_len for r in trace)
    first = min(r.arrival_s for r in recs)
    makespan = max(r.done_s for r in recs) - first
    ttft = sorted(r.first_token_s - r.arrival_s for r in recs)
    tpot = sorted((r.done_s - r.first_token_s) / max(1, r.output_len - 1) for r in recs)
    p99 = lambda xs: xs[min(len(xs) - 1, int(math.ceil(0.99 * len(xs))) - 1)]
    return {
        "metric": "aggregate decode tokens/s across colocated LLMs (measured serving run)",
        "value": round(out_tokens / makespan, 1), "unit": "tokens/s",
        "requests": len(recs), "generated_tokens": out_tokens, "makespan_s": round(makespan, 3),
        "req_per_s": round(len(recs) / makespan, 2),
        "ttft_ms": {"mean": round(1e3 * sum(ttft) / len(ttft), 2), "p99": round(1e3 * p99(ttft), 2)},
        "tpot_ms": {"mean": round(1e3 * sum(tpot) / len(tpot), 3), "p99": round(1e3 * p99(tpot), 3)},
        "workload": {"models": list(model_names), "rates_rps": list(rates), "horizon_s": horizon_s, "seed": seed,
                     "lengths": "ShareGPT lognormal 161/338 sigma 0.8" if lengths is None else lengths,
                     "scheduler": scheduler, "gpu_memory_gib": gpu_memory_gib,
                     "partition_sms": partition_sms, "prefill_on_partition": prefill_on_partition,
                     "pass_green": pass_green, "engine": "realtime" if realtime else "measured",
                     "align_decode": align_decode, "sm_route": sm_route},
        "passes": passes, "green_passes": green_passes,
        # tokens produced (decode jobs' batches, prefills' first tokens) by
        # jobs ending in the second half of the arrival period, per second:
        # the engine's throughput under the offered load, before the drain
        # (the tail of long outputs at shrinking batch) that `value` includes
        "arrival_window": window,
        "host_wall_s": round(wall, 2),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="7b,13b")
    ap.add_argument("--rates", default="20,10")
    ap.add_argument("--horizon", type=float, default=8.0)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--partition-sms", type=lambda s: [int(x) for x in s.split(",")], default=None)
    ap.add_argument("--prefill-on-partition", type=int, default=0,
                    help="run each model's prefill jobs on its own green partition too")
    ap.add_argument("--pass-green", type=lambda s: [int(x) for x in s.split(",")], default=None,
                    help="per-model green partition SMs, used per pass (decode jobs of >= 2 models)")
    ap.add_argument("--realtime", action="store_true",
                    help="jobs overlap across passes, completions from device events (mux_unit_run_realtime)")
    ap.add_argument("--align-decode", action="store_true",
                    help="real-time: colocated models' decode steps start together (rounds)")
    ap.add_argument("--scheduler", choices=["adbs", "fcfs", "rr"], default="adbs")
    ap.add_argument("--gpu-memory-gib", type=float, default=180.0)
    ap.add_argument("--lengths", default=None, help="per-model constant prompt:output, e.g. 128:384,64:64")
    ap.add_argument("--sm-route", action="store_true",
                    help="run every ADBS job on a green context sized by its sm_demand (option sm_route)")
    args = ap.parse_args()
    models = args.models.split(",")
    rates = [float(x) for x in args.rates.split(",")]
    psms = [0] + args.partition_sms if args.partition_sms else None
    lengths = None if args.lengths is None else [tuple(int(x) for x in m.split(":")) for m in args.lengths.split(",")]
    print(json.dumps(serve(models, rates, args.horizon, args.seed, partition_sms=psms, scheduler=args.scheduler,
                           gpu_memory_gib=args.gpu_memory_gib, lengths=lengths,
                           prefill_on_partition=bool(args.prefill_on_partition),
                           pass_green=args.pass_green, realtime=args.realtime,
                           align_decode=args.align_decode, sm_route=args.sm_route)), flush=True)


if __name__ == "__main__":
    main()
