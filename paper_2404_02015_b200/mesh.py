"""Multi-rank plumbing of a mesh (one process per GPU, torch.distributed).

Two shapes of multi-GPU work exist on this path:

* independent units -- LLM units placed on disjoint meshes share nothing
  (/root/reference/proj/include/muxsim/sim_engine.hpp:74-80,
  placement.cpp:425-450 verify_placement): every rank runs its own unit and
  throughput adds up; the only collective is the timing reduction
  (max over ranks) of the benchmark;
* tensor parallelism inside a mesh -- the reference prices it as
  tp_speedup = eta * tp (cost_model.cpp:43-47). Here every rank holds a
  Megatron shard and a floor(total/tp) slice of the head-wise KV pool; the
  allocation decisions are replicated (each row costs 2*L*H/tp blocks on
  every rank), and the only data exchange is the row-parallel GEMM's fused
  allreduce, which writes peer mailboxes directly (no NCCL call on the data
  path). torch.distributed only carries the one-time mailbox handle exchange.
"""
from __future__ import annotations

from typing import Sequence


def rank_world():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def max_over_ranks(values: Sequence[float]) -> list[float]:
    """Element-wise max over ranks (device timings: the job ends with its
    slowest rank)."""
    import torch
    import torch.distributed as dist
    _, world = rank_world()
    if world == 1:
        return list(values)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values: Sequence[float]) -> list[float]:
    """Element-wise sum over ranks (tokens and kernel time of every unit)."""
    import torch
    import torch.distributed as dist
    _, world = rank_world()
    if world == 1:
        return list(values)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def gather_objects(obj) -> list:
    """Every rank's picklable `obj`, in rank order (plumbing only)."""
    import torch.distributed as dist
    _, world = rank_world()
    if world == 1:
        return [obj]
    out: list = [None] * world
    dist.all_gather_object(out, obj)
    return out


def tp_pool_blocks(total_blocks: int, tp: int) -> int:
    """KV head-blocks of one rank's pool slice: the mesh-wide
    pool of sim_engine.cpp:172-186 split by head, floor(total / tp)."""
    if tp < 1:
        raise ValueError("tp must be >= 1")
    return total_blocks // tp


def tp_spec(spec, tp: int):
    """The LLMSpec one rank's pool registers: H/tp heads (H % tp == 0 is the
    realizability filter the reference planner lacks)."""
    from dataclasses import replace
    if spec.num_heads % tp or (spec.ffn and spec.ffn % tp):
        raise ValueError(f"{spec.name}: heads {spec.num_heads} / ffn {spec.ffn} not divisible by tp={tp}")
    return replace(spec, num_heads=spec.num_heads // tp, ffn=spec.ffn // tp if spec.ffn else spec.ffn)


def connect_tp(unit, partitions: Sequence[int], group=None) -> None:
    """Exchange every partition's TP mailbox handle with the other ranks of
    the mesh (all_gather over torch.distributed) and map the peers' mailboxes
    into this process (CUDA IPC). `unit` needs tp_mailbox / tp_connect and
    its tp_rank must equal the process's rank in `group`."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = [unit.tp_mailbox(p)[1] for p in partitions]
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    for peer in range(world):
        if peer == rank:
            continue
        for p, handle in zip(partitions, gathered[peer]):
            unit.tp_connect(p, peer, handle=handle)
