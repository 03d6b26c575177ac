"""Debug: 2 processes on one GPU, TP=2 over CUDA IPC; prints mailbox counters."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, ".")


def rank_fn(rank, world, port):
    import paper_2404_02015_b200 as mux
    from paper_2404_02015_b200 import mesh
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s = mux.spec("tiny-a")
    unit = mux.Unit([s], pool_blocks=50000, device_pool_blocks=50000, max_batch=8, max_prefill_tokens=256,
                    max_ctx=256, partitions=2, tp_rank=rank, tp_size=world, init_seed=5, init_std=0.05)
    mesh.connect_tp(unit, [1])
    print(rank, "connected", flush=True)

    def watch():
        for _ in range(30):
            time.sleep(1.0)
            v = (C.c_uint32 * 4)()
            mux.lib.mux_unit_tp_debug(unit._h, 1, v)
            print(rank, "counters", list(v), flush=True)
    threading.Thread(target=watch, daemon=True).start()
    assert unit.pool.admit(0, 1, 5, 8).ok
    out = torch.zeros(1, dtype=torch.int32).pin_memory().numpy()
    unit.prefill(0, [1], np.arange(5, dtype=np.int32), out, partition=1)
    print(rank, "issued", flush=True)
    unit.sync()
    print(rank, "done", out, flush=True)
    dist.barrier()


if __name__ == "__main__":
    mp.start_processes(rank_fn, args=(2, 29533), nprocs=2, join=True, start_method="spawn")
