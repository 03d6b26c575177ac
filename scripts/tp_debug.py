import sys, time, ctypes as C
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2404_02015_b200 as mux
from oracle import llama_ref
from test_gpu_model import load_weights, dims_of
specs = [mux.spec("tiny-a"), mux.spec("tiny-b")]
total = 232998
units = [mux.Unit(specs, pool_blocks=total // 2, device_pool_blocks=total // 2, max_batch=16,
                  max_prefill_tokens=512, max_ctx=512, partitions=2, tp_rank=r, tp_size=2) for r in (0, 1)]
for p in range(2):
    ptrs = [u.tp_mailbox(p)[0] for u in units]
    units[0].tp_connect(p, 1, ptr=ptrs[1]); units[1].tp_connect(p, 0, ptr=ptrs[0])
print("connected", flush=True)
for llm, s in enumerate(specs):
    for u in units: load_weights(u, llm, s, 300 + llm)
print("weights", flush=True)
lens = [17]; rids = [5]
for u in units: assert u.pool.admit(0, 5, 17, 20).ok
outs = [torch.zeros(1, dtype=torch.int32).pin_memory().numpy() for _ in units]
prompt = np.arange(17, dtype=np.int32)
for u, o in zip(units, outs):
    u.prefill(0, rids, prompt, o, partition=1)
    print("issued", flush=True)
def dbg():
    for r, u in enumerate(units):
        v = (C.c_uint32 * 4)()
        mux.lib.mux_unit_tp_debug(u._h, 1, v)
        print("rank", r, list(v), flush=True)
for i in range(20):
    time.sleep(0.5)
    dbg()
    st = torch.cuda.current_stream()
print("done?", flush=True)
