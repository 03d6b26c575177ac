"""Multi-rank host logic on CPU (gloo, world_size 2): the max-over-ranks
timing reduction of the bench, the tensor-parallel mailbox handle exchange,
and the replicated per-rank KV pool decisions of a TP mesh (SURVEY §8e:
every row costs 2*L*H/tp blocks on each of the tp pool slices, so each rank's
admit/alloc outcome equals the mesh-wide count pool's)."""
import os
import random
import socket

import pytest
import torch.multiprocessing as mp

import paper_2404_02015_b200 as mux
from paper_2404_02015_b200 import mesh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, world, *args):
    port = _free_port()
    mp.spawn(_entry, args=(fn, world, port) + args, nprocs=world, join=True)


def _entry(rank, fn, world, port, *args):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _max_body(rank, world):
    assert mesh.rank_world() == (rank, world)
    got = mesh.max_over_ranks([float(rank + 1), 10.0 - rank])
    assert got == [float(world), 10.0]


def test_max_over_ranks_gloo():
    _run(_max_body, 2)


def _sum_gather_body(rank, world):
    # bench.py --placement: every rank's unit adds its tokens / kernel time,
    # an idle rank adds zeros, and rank 0 lists every rank's models
    got = mesh.sum_over_ranks([float(10 * rank), 0.5])
    assert got == [float(10 * sum(range(world))), 0.5 * world]
    units = mesh.gather_objects({"models": ["7b"] * rank, "batch": 8 * rank})
    assert units == [{"models": ["7b"] * r, "batch": 8 * r} for r in range(world)]


def test_sum_and_gather_over_ranks_gloo():
    _run(_sum_gather_body, 2)


class _FakeUnit:
    def __init__(self, rank):
        self.rank = rank
        self.connected = {}

    def tp_mailbox(self, p):
        return 0x1000 * (self.rank + 1) + p, bytes([self.rank, p]) * 32

    def tp_connect(self, p, peer, handle=None, ptr=None):
        self.connected[(p, peer)] = handle


def _connect_body(rank, world):
    u = _FakeUnit(rank)
    mesh.connect_tp(u, [0, 2])
    peer = 1 - rank
    assert u.connected == {(0, peer): bytes([peer, 0]) * 32, (2, peer): bytes([peer, 2]) * 32}


def test_connect_tp_exchanges_mailbox_handles():
    _run(_connect_body, 2)


def _decisions(pool, spec_count, seed, steps):
    rng = random.Random(seed)
    out, live = [], []
    for k in range(steps):
        op = rng.random()
        if op < 0.45 or not live:
            llm = rng.randrange(spec_count)
            rid = k
            p = rng.randrange(1, 300)
            r = pool.admit(llm, rid, p, p + rng.randrange(0, 300))
            out.append(("admit", r.ok, r.error))
            if r.ok:
                live.append((llm, rid))
        elif op < 0.85:
            llm, rid = rng.choice(live)
            r = pool.alloc(llm, rid, rng.randrange(1, 40), True)
            out.append(("alloc", r.ok, r.error))
        else:
            llm, rid = live.pop(rng.randrange(len(live)))
            pool.free_request(llm, rid)
            out.append(("free",))
        pool.check_conservation()
    return out


def _pool_body(rank, world, total, seed):
    import torch.distributed as dist
    specs = [mux.spec("7b"), mux.spec("13b")]
    pool = mux.BlockPool(mesh.tp_pool_blocks(total, world), physical=True)
    for i, s in enumerate(specs):
        pool.register_llm(i, mesh.tp_spec(s, world))
        pool.set_quota(i, mesh.tp_pool_blocks(total, world) // 2)  # quota split by tp like the pool
    mine = _decisions(pool, len(specs), seed, 3000)
    every = [None] * world
    dist.all_gather_object(every, mine)
    assert all(d == every[0] for d in every)
    if rank == 0:
        glob = mux.BlockPool(total, physical=False)
        for i, s in enumerate(specs):
            glob.register_llm(i, s)
            glob.set_quota(i, total // 2)
        assert _decisions(glob, len(specs), seed, 3000) == mine


@pytest.mark.parametrize("seed", [1, 2])
def test_tp_pool_slices_replicate_mesh_decisions(seed):
    # a 2-GPU mesh worth of blocks (divisible by tp*2 so quotas split exactly),
    # small enough that pool and quota failures both occur
    total = 4 * 3200 * 40
    _run(_pool_body, 2, total, seed)


def test_tp_spec_rejects_unrealizable_widths():
    with pytest.raises(ValueError):
        mesh.tp_spec(mux.spec("30b"), 8)  # 52 heads, the reference planner's tp=8
    assert mesh.tp_spec(mux.spec("13b"), 2).num_heads == 20


@pytest.mark.parametrize("tp", [2, 4])
def test_sharded_physical_ids_keep_mesh_decisions(tp):
    """BlockPool.enable_physical(tp) (a TP mesh's pool): the
    mesh-wide count decisions are the reference's, unchanged; every column
    (layer, head, kv) of a row gets a rank-local id of rank head / (H / tp)
    in [0, total / tp); live ids are unique per rank; conservation holds."""
    specs = [mux.spec("7b"), mux.spec("13b")]
    total = 4 * 3200 * 40 + 3  # not a multiple of tp: the tail is never materialised
    sharded = mux.BlockPool(total, physical=True, shards=tp)
    count = mux.BlockPool(total, physical=False)
    for p in (sharded, count):
        for i, s in enumerate(specs):
            p.register_llm(i, s)
            p.set_quota(i, total // 2)
    rng = random.Random(tp)
    live = []
    for k in range(3000):
        op = rng.random()
        if op < 0.45 or not live:
            llm, n = rng.randrange(2), rng.randrange(1, 300)
            extra = rng.randrange(0, 300)
            a, b = sharded.admit(llm, k, n, n + extra), count.admit(llm, k, n, n + extra)
            assert (a.ok, a.error) == (b.ok, b.error)
            if a.ok:
                live.append((llm, k))
        elif op < 0.85:
            llm, rid = rng.choice(live)
            add = rng.randrange(1, 40)
            a, b = sharded.alloc(llm, rid, add, True), count.alloc(llm, rid, add, True)
            assert (a.ok, a.error) == (b.ok, b.error)
        else:
            llm, rid = live.pop(rng.randrange(len(live)))
            sharded.free_request(llm, rid)
            count.free_request(llm, rid)
        sharded.check_conservation()
        if k % 500 == 0 or k == 2999:
            seen = [set() for _ in range(tp)]
            for llm, rid in live:
                H = specs[llm].num_heads
                ids = sharded.block_table(llm, rid)
                for j, bid in enumerate(ids):
                    rank = ((j % (2 * specs[llm].num_layers * H)) // 2 % H) // (H // tp)
                    assert 0 <= bid < total // tp
                    assert bid not in seen[rank]
                    seen[rank].add(bid)
    assert sharded.free_blocks() == count.free_blocks()
