"""Tensor parallelism across PROCESSES (one per rank, as on a real mesh):
the mailboxes are exchanged over torch.distributed (gloo) and mapped with
CUDA IPC (paper_2404_02015_b200.mesh.connect_tp). Run here with both ranks on
the one GPU this environment has (their contexts time-slice, so it checks
correctness, not NVLink speed). Tokens of both ranks must be identical and
match the full-model oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2404_02015_b200 as mux
    from paper_2404_02015_b200 import mesh
    from oracle import llama_ref
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s = mux.spec("tiny-a")
    unit = mux.Unit([s], pool_blocks=mesh.tp_pool_blocks(100000, world), device_pool_blocks=50000,
                    max_batch=8, max_prefill_tokens=256, max_ctx=256, partitions=2, tp_rank=rank, tp_size=world)
    mesh.connect_tp(unit, [1])
    d = llama_ref.Dims(s.num_layers, s.num_heads, s.hidden_size, s.ffn, s.vocab)
    w = llama_ref.make_weights(d, 42, std=0.05)
    for key, arr in w.items():
        name, layer = (key, 0) if isinstance(key, str) else key
        unit.set_tensor(0, name, layer, np.ascontiguousarray(arr))
    rng = np.random.default_rng(3)
    lens = [5, 70]
    prompts = [rng.integers(0, s.vocab, n).astype(np.int32) for n in lens]
    rids = [1, 2]
    for rid, n in zip(rids, lens):
        assert unit.pool.admit(0, rid, n, n + 6).ok
    out = torch.zeros(len(rids), dtype=torch.int32).pin_memory().numpy()
    unit.prefill(0, rids, np.concatenate(prompts), out, partition=1)
    unit.sync()
    gen = [[int(t)] for t in out]
    for _ in range(5):
        for rid in rids:
            assert unit.pool.alloc(0, rid, 1, False).ok
        unit.decode(0, rids, out=out, partition=1)
        unit.sync()
        for i, t in enumerate(out):
            gen[i].append(int(t))
    every = [None] * world
    dist.all_gather_object(every, gen)
    if rank == 0:
        q.put((every, [p.tolist() for p in prompts]))  # small: the parent joins before reading
    dist.barrier()
    unit.close()
    dist.destroy_process_group()


@pytest.mark.timeout(280)
def test_tp2_across_processes_ipc(cuda):
    from oracle import llama_ref
    import paper_2404_02015_b200 as mux
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_rank, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    every, prompts = q.get()
    prompts = [np.asarray(p, np.int32) for p in prompts]
    assert every[0] == every[1]
    s = mux.spec("tiny-a")
    d = llama_ref.Dims(s.num_layers, s.num_heads, s.hidden_size, s.ffn, s.vocab)
    ref = llama_ref.RefLlama(d, llama_ref.make_weights(d, 42, std=0.05), llama_ref.rope_table(300))
    for p, toks in zip(prompts, every[0]):
        cache = ref.new_cache()
        logits = ref.forward(p, cache)
        for i, t in enumerate(toks):
            assert float(logits.max() - logits[t]) <= 2e-2 * max(1.0, float(np.abs(logits).max()))
            if i + 1 < len(toks):
                logits = ref.forward(np.array([t]), cache)
