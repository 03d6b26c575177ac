"""Per-CTA globaltimer stamps of one fused layer-chain launch (debug).

Slots per job j (j*8+k): 6 weights producer starts job j, 0 activation
producer passed job j's input barrier, 1 first MMA of job j, 2 last MMA
issued, 3 last reduce-add issued, 4 barrier 2j passed, 5 element-wise step
done."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2404_02015_b200 as mux  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "13b"
B = 128
s = mux.spec(model)
rng = np.random.default_rng(1)
reqs = bench.sample_batch(rng, B, 20)
need = sum(mux.blocks_for_tokens(s, 16, p + d + 21) for p, o, d in reqs)
unit = mux.Unit([s], pool_blocks=bench.pool_blocks([s]), device_pool_blocks=need + 4096, max_batch=B,
                max_prefill_tokens=256, max_ctx=max(p + d for p, o, d in reqs) + 64, max_slots=B + 16,
                init_seed=3, init_std=0.02, partitions=2)
unit.init_kv(seed=7, std=1.0)
rids = []
for k, (p, o, d) in enumerate(reqs):
    assert unit.pool.admit(0, k, p, p + o - 1).ok
    if d:
        assert unit.pool.alloc(0, k, d, False).ok
    rids.append(k)
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
for step in range(4):
    for rid in rids:
        assert unit.pool.alloc(0, rid, 1, False).ok
    if step == 3:
        mux.lib.mux_debug_chain_timing(buf.data_ptr())
    unit.decode(0, rids, partition=1)
    unit.sync()
mux.lib.mux_debug_chain_timing(None)
print("coop+pdl:", mux.lib.mux_debug_chain_coop_pdl())
raw = buf.view(148, 64).cpu().double()
t0 = raw[raw > 0].min()
t = (raw - t0) / 1e3
names = {6: "A-start", 0: "B-barrier", 1: "first-MMA", 2: "last-MMA", 3: "last-red", 4: "barrier-A", 5: "post-done"}
for j in range(3):
    parts = []
    for k in (6, 0, 1, 2, 3, 4, 5):
        col = raw[:, j * 8 + k]
        v = t[:, j * 8 + k][col > 0]
        if len(v):
            parts.append(f"{names[k]} {v.min():.1f}/{v.median():.1f}/{v.max():.1f}")
    print(f"job{j}: " + " | ".join(parts), flush=True)
