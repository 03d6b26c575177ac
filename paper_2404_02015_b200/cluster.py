"""Placement-driven execution across a box: `run_simulation`
(/root/reference/proj/src/sim_engine.cpp:370-413) with every unit of a
plan.json on its own GPU mesh.

The reference runs one UnitSim per placed unit; units own disjoint meshes and
share nothing (sim_engine.hpp:74-80, verify_placement placement.cpp:419-453),
so here every unit runs in its own process(es):

* a tp = 1 unit is one process on GPU gpu_ids[0], running the unit's models
  and its share of the trace through the chosen engine (lockstep, measured
  or real-time, mux_unit_run_*);
* a tp > 1 unit is tp processes, rank r on gpu_ids[r], each holding a
  Megatron shard of every model and its head slice of the pool
  (BlockPool.enable_physical(tp): the mesh-wide decisions of the reference,
  rank-local block ids); the ranks exchange their row-parallel partials
  through peer-mapped mailboxes (mesh.connect_tp, CUDA IPC), and take
  identical decisions because lockstep durations are priced, not measured.

Records are merged and sorted by id and the per-unit pool statistics keep the
plan's unit index, as run_simulation does. When the box has fewer GPUs than
the plan names, units run one after another (each still owning its devices
while it runs); the ranks of one unit always run together.
"""
from __future__ import annotations

import math
import multiprocessing as mp
import os
import socket
from dataclasses import dataclass

from .host import Entry, EngineParams, Placement, TraceRequest

BLOCK_BYTES = 128 * 16 * 2  # head_dim x block_tokens x bpe (kv_manager.cpp:37-40): the kernels' 4 KiB head-block


def unit_pool_blocks(specs, mesh_gpus: int, gpu_memory_bytes: int, reserve_frac: float) -> int:
    """UnitSim::pool_blocks (sim_engine.cpp:172-186) over MemoryLayout::for_mesh
    (kv_manager.cpp:10-23): llround of the reserve, global over the mesh."""
    mesh = mesh_gpus * gpu_memory_bytes
    reserve = int(math.floor(reserve_frac * mesh + 0.5))
    kv = mesh - sum(s.weight_bytes for s in specs) - reserve
    if kv <= 0:
        raise ValueError("memory layout: weights and reserve exceed mesh memory")
    return kv // BLOCK_BYTES


@dataclass
class UnitJob:
    unit: int                 # index in the plan
    members: list             # config entry indices
    gpu_ids: list             # one per tp rank
    entries: list             # Entry of each member (unit-local order)
    trace: list               # TraceRequest with unit-local llm
    gpu_memory_bytes: int
    params: EngineParams
    profile: list | None
    engine: str
    prompt_seed: int = 11
    want_tokens: bool = False


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(job: UnitJob, rank: int, port: int, q) -> None:
    """One process: rank `rank` of the unit's mesh."""
    try:
        import torch

        from . import host, mesh
        tp = len(job.gpu_ids)
        ndev = torch.cuda.device_count()
        dev = job.gpu_ids[rank] % max(1, ndev)
        torch.cuda.set_device(dev)
        if tp > 1:
            import torch.distributed as dist
            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ["MASTER_PORT"] = str(port)
            dist.init_process_group("gloo", rank=rank, world_size=tp)
        specs = [e.spec for e in job.entries]
        total = unit_pool_blocks(specs, tp, job.gpu_memory_bytes, job.params.activation_reserve_frac)
        longest = max((r.prompt_len + r.output_len for r in job.trace), default=16)
        n = len(specs)
        unit = host.Unit(specs, pool_blocks=total // tp, device=dev, device_pool_blocks=total // tp,
                         max_batch=512, max_prefill_tokens=max(job.params.token_budget, longest),
                         max_ctx=longest + 16, max_slots=len(job.trace) + 8, init_seed=1 + 7 * job.unit,
                         init_std=0.02, partitions=n + 1, tp_rank=rank, tp_size=tp)
        try:
            if tp > 1:
                mesh.connect_tp(unit, list(range(n + 1)))
            recs, tokens = unit.run_lockstep(job.entries, job.trace, job.gpu_memory_bytes, job.params,
                                             prompt_seed=job.prompt_seed, profile=job.profile,
                                             measured=job.engine == "measured", realtime=job.engine == "realtime",
                                             mesh_size=tp)
            stats = unit.last_stats()
        finally:
            if tp > 1:
                import torch.distributed as dist
                dist.barrier()
            unit.close()
        out = {"unit": job.unit, "rank": rank,
               "records": [(r.id, r.llm, r.arrival_s, r.first_token_s, r.done_s, r.prompt_len, r.output_len)
                           for r in recs],
               "stats": [(u.total_blocks, [(m.llm, m.rate, m.avg_used_blocks, m.final_quota_blocks, m.resource_usage)
                                           for m in u.llms], u.samples) for u in stats],
               "tokens": tokens if job.want_tokens else None}
        if tp > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        q.put(out)
    except BaseException as e:  # noqa: BLE001 - reported to the parent, which raises
        q.put({"unit": job.unit, "rank": rank, "error": f"{type(e).__name__}: {e}"})


def split_plan(entries, trace, placement: Placement, gpu_memory_bytes, params, profile, engine,
               want_tokens=False) -> list[UnitJob]:
    """One UnitJob per non-empty unit: its models and its requests, with
    unit-local model indices (run_simulation's routing by model name)."""
    jobs = []
    gpu = 0
    for u, (size, mem) in enumerate(zip(placement.mesh_sizes, placement.members)):
        ids = placement.gpu_ids[u] if placement.gpu_ids else list(range(gpu, gpu + size))
        gpu += size
        if not mem:
            continue
        local = {g: i for i, g in enumerate(mem)}
        sub = [TraceRequest(r.id, local[r.llm], r.arrival_s, r.prompt_len, r.output_len) for r in trace
               if r.llm in local]
        jobs.append(UnitJob(u, list(mem), list(ids), [entries[i] for i in mem], sub, gpu_memory_bytes, params,
                            profile, engine, want_tokens=want_tokens))
    served = {i for j in jobs for i in j.members}
    for r in trace:
        if r.llm not in served:
            raise ValueError(f"trace references model {r.llm} which the placement does not serve")
    return jobs


def run_plan(entries, trace, placement: Placement, gpu_memory_bytes: int, params: EngineParams | None = None,
             profile=None, engine: str = "lockstep", want_tokens: bool = False):
    """Every unit of the plan on its own GPU mesh. Returns (records sorted by
    id with config entry indices, per-unit UnitStat list, tokens) where tokens
    maps (unit, rank) -> per-request token lists of that unit's trace."""
    import torch

    from .host import Record, UnitLlmStat, UnitStat
    params = params or EngineParams()
    jobs = split_plan(entries, trace, placement, gpu_memory_bytes, params, profile, engine, want_tokens)
    for j in jobs:
        if len(j.gpu_ids) > 1 and engine != "lockstep":
            raise ValueError(f"unit {j.unit}: tensor-parallel units run the lockstep engine only")
    ndev = max(1, torch.cuda.device_count())
    need = sum(len(j.gpu_ids) for j in jobs)
    waves = [jobs] if need <= ndev else [[j] for j in jobs]
    ctx = mp.get_context("spawn")
    results = []
    for wave in waves:
        q = ctx.Queue()
        procs = []
        for j in wave:
            port = _free_port()
            for r in range(len(j.gpu_ids)):
                p = ctx.Process(target=_worker, args=(j, r, port, q))
                p.start()
                procs.append(p)
        got = [q.get() for _ in procs]
        for p in procs:
            p.join()
        errs = [g for g in got if "error" in g]
        if errs:
            raise RuntimeError("; ".join(f"unit {e['unit']} rank {e['rank']}: {e['error']}" for e in errs))
        results += got
    by_unit = {j.unit: j for j in jobs}
    records, units, tokens = [], [], {}
    for res in sorted(results, key=lambda g: (g["unit"], g["rank"])):
        j = by_unit[res["unit"]]
        tokens[(res["unit"], res["rank"])] = res["tokens"]
        if res["rank"] != 0:
            continue
        for (rid, llm, a, f, d, p, o) in res["records"]:
            records.append(Record(rid, j.members[llm], a, f, d, p, o))
        for total, llms, samples in res["stats"]:
            units.append(UnitStat(j.unit, total, [UnitLlmStat(j.members[m[0]], *m[1:]) for m in llms],
                                  [(t, j.members[li], used, q_) for t, li, used, q_ in samples]))
    records.sort(key=lambda r: r.id)
    return records, units, tokens
