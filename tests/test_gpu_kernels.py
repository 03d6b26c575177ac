"""GPU parity of the sm_100a kernels against the CPU oracle (run with -m gpu).

K1 paged decode attention: fp32 out within 1e-4 relative of the C oracle
(oracle/numerics_ref.c, fp64 accumulation), bf16 out within 1e-2.
K2 KV append: bit-exact K (after RoPE) / V placement in the head-block pool.
K4 tcgen05 GEMM: vs a torch fp32 matmul of the same bf16 operands.
Block tables come from the product's physical BlockPool, pre-fragmented by
an alloc/free churn (acceptance-C7 style) so they are scattered.
"""
import random

import numpy as np
import pytest

import paper_2404_02015_b200 as mux
from oracle import llama_ref, refs

pytestmark = pytest.mark.gpu


def build_tables(pool, llm, L, H, rids, max_rows):
    """Pack the product pool's block tables into the kernel's two-level layout."""
    W = 2 * L * H
    rowrec, rowlist = [], np.zeros((len(rids), max_rows), np.int32)
    for s, rid in enumerate(rids):
        t = pool.block_table(llm, rid)
        rows = len(t) // W
        for r in range(rows):
            rowlist[s, r] = len(rowrec)
            rowrec.append(t[r * W:(r + 1) * W])
    return np.array(rowrec, np.int32).reshape(-1, W), rowlist


def fragmented_pool(total, specs, seed):
    rng = random.Random(seed)
    pool = mux.BlockPool(total, physical=True)
    for i, s in enumerate(specs):
        pool.register_llm(i, s)
        pool.set_quota(i, total)
    # churn: admit and free to scatter the free stack
    live = []
    for k in range(200):
        llm = rng.randrange(len(specs))
        rid = 100000 + k
        if pool.admit(llm, rid, rng.randrange(1, 200), 300).ok:
            live.append((llm, rid))
        if live and rng.random() < 0.5:
            l, r = live.pop(rng.randrange(len(live)))
            pool.free_request(l, r)
    return pool


@pytest.mark.parametrize("B,H,L,max_ctx,splits,seed", [
    (1, 4, 2, 40, 0, 0),
    (5, 4, 2, 300, 0, 1),
    (64, 8, 2, 340, 0, 2),
    (7, 2, 4, 2000, 4, 3),
    (3, 4, 1, 4096, 8, 4),
])
def test_decode_attention_matches_oracle(cuda, B, H, L, max_ctx, splits, seed):
    import torch
    rng = random.Random(seed)
    spec = mux.LLMSpec("m", L, H, 128, H * 128, 1, 2)
    other = mux.LLMSpec("o", 1, 2, 128, 256, 1, 2)
    total = 60000
    pool = fragmented_pool(total, [spec, other], seed)
    ctx = [max(1, min(max_ctx, rng.choice([1, 15, 16, 17, rng.randrange(1, max_ctx + 1), max_ctx])))
           for _ in range(B)]
    rids = []
    for b in range(B):
        rid = b
        assert pool.admit(0, rid, ctx[b], ctx[b]).ok
        rids.append(rid)
    max_rows = (max_ctx + 15) // 16
    rowrec, rowlist = build_tables(pool, 0, L, H, rids, max_rows)
    g = torch.Generator(device="cuda").manual_seed(seed)
    kv = (torch.randn(total * 2048, generator=g, device="cuda") / 4).to(torch.bfloat16)
    q = (torch.randn(B, H, 128, generator=g, device="cuda")).to(torch.bfloat16)
    d_rowrec = torch.from_numpy(rowrec).cuda()
    d_rowlist = torch.from_numpy(rowlist).cuda()
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    d_ctx = torch.tensor(ctx, dtype=torch.int32, device="cuda")
    ws = torch.empty(B * H * 16 * 130, dtype=torch.float32, device="cuda")
    layer = L - 1
    out32 = torch.empty(B, H, 128, dtype=torch.float32, device="cuda")
    mux.decode_attention_headwise(q, kv, d_rowrec, d_rowlist, slots, d_ctx, L, layer, max_rows, max_ctx,
                                  out32, kv_splits=splits, workspace=ws)
    out16 = torch.empty(B, H, 128, dtype=torch.bfloat16, device="cuda")
    mux.decode_attention_headwise(q, kv, d_rowrec, d_rowlist, slots, d_ctx, L, layer, max_rows, max_ctx,
                                  out16, kv_splits=splits, workspace=ws)
    torch.cuda.synchronize()
    want = refs.decode_attention(q.view(torch.int16).cpu().numpy().view(np.uint16),
                                 kv.view(torch.int16).cpu().numpy().view(np.uint16), rowrec, rowlist,
                                 np.arange(B, dtype=np.int32), np.array(ctx, np.int32), L, layer, max_rows)
    got = out32.cpu().numpy()
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-4 * scale, np.abs(got - want).max() / scale
    got16 = out16.float().cpu().numpy()
    assert np.abs(got16 - want).max() <= 1e-2 * scale


def test_kv_append_bit_exact(cuda):
    import torch
    L, H, T = 3, 4, 40
    spec = mux.LLMSpec("m", L, H, 128, H * 128, 1, 2)
    total = 5000
    pool = fragmented_pool(total, [spec], 5)
    rng = random.Random(5)
    lens = [rng.randrange(1, 30) for _ in range(4)]
    for s, n in enumerate(lens):
        assert pool.admit(0, s, n, n).ok
    max_rows = 4
    rowrec, rowlist = build_tables(pool, 0, L, H, list(range(len(lens))), max_rows)
    tok_slot = np.concatenate([[s] * n for s, n in enumerate(lens)]).astype(np.int32)
    tok_pos = np.concatenate([np.arange(n) for n in lens]).astype(np.int32)
    T = len(tok_slot)
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(T, 3, H, 128, generator=g, device="cuda").to(torch.bfloat16)
    qkv_host = qkv.view(torch.int16).cpu().numpy().view(np.uint16).copy()
    kvpool = torch.zeros(total * 2048, dtype=torch.bfloat16, device="cuda")
    q_out = torch.empty(T, H, 128, dtype=torch.bfloat16, device="cuda")
    rope = torch.from_numpy(llama_ref.rope_table(64)).cuda()
    layer = 1
    mux.kv_append(qkv, q_out, kvpool, torch.from_numpy(rowrec).cuda(), torch.from_numpy(rowlist).cuda(),
                  torch.from_numpy(tok_slot).cuda(), torch.from_numpy(tok_pos).cuda(), rope, T, H, L, layer,
                  max_rows)
    torch.cuda.synchronize()
    # oracle: same float32 ops, same table (computed independently with libm)
    assert np.array_equal(mux.rope_table(64), llama_ref.rope_table(64))
    tab = llama_ref.rope_table(64)
    f = llama_ref.bf16_to_f32(qkv_host)
    q_ref = llama_ref.f32_to_bf16(llama_ref.rope_rotate(f[:, 0], tok_pos[:, None], tab))
    k_ref = llama_ref.f32_to_bf16(llama_ref.rope_rotate(f[:, 1], tok_pos[:, None], tab))
    v_ref = qkv_host[:, 2]
    assert np.array_equal(q_out.view(torch.int16).cpu().numpy().view(np.uint16), q_ref)
    pool_h = kvpool.view(torch.int16).cpu().numpy().view(np.uint16).reshape(total, 16, 128)
    W = 2 * L * H
    for t in range(T):
        s, p = tok_slot[t], tok_pos[t]
        rec = rowrec[rowlist[s, p // 16]]
        for h in range(H):
            kid, vid = rec[(layer * H + h) * 2], rec[(layer * H + h) * 2 + 1]
            assert np.array_equal(pool_h[kid, p % 16], k_ref[t, h]), (t, h)
            assert np.array_equal(pool_h[vid, p % 16], v_ref[t, h]), (t, h)
    # nothing else written: count nonzero rows == T * H * 2
    assert int((pool_h != 0).any(axis=2).sum()) == T * H * 2
    assert W == rowrec.shape[1]


@pytest.mark.parametrize("M", [1, 7, 16, 64, 100, 256, 257, 1000])
@pytest.mark.parametrize("N,K", [(256, 512), (640, 1024), (1000, 576), (384, 200)])
def test_gemm_tcgen05(cuda, M, N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 1000 + N + K)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    scale = ref.abs().max().item()
    out32 = torch.empty(M, N, dtype=torch.float32, device="cuda")
    mux.gemm_bf16(x, w, out32, epilogue=3)
    out16 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    mux.gemm_bf16(x, w, out16, epilogue=0)
    resid0 = torch.randn(M, N, generator=g, device="cuda")
    resid = resid0.clone()
    mux.gemm_bf16(x, w, resid, epilogue=1)
    # odd grids exercise tiles split across many CTAs (stream-K fixups)
    out_g = torch.empty(M, N, dtype=torch.float32, device="cuda")
    mux.gemm_bf16(x, w, out_g, epilogue=3, grid=37)
    out_g2 = torch.empty(M, N, dtype=torch.float32, device="cuda")
    mux.gemm_bf16(x, w, out_g2, epilogue=3, grid=1000)
    torch.cuda.synchronize()
    assert (out32 - ref).abs().max().item() <= 1e-4 * scale + 1e-6
    assert (out16.float() - ref).abs().max().item() <= 8e-3 * scale
    assert (resid - resid0 - ref).abs().max().item() <= 1e-4 * scale + 1e-5
    assert (out_g - ref).abs().max().item() <= 1e-4 * scale + 1e-6
    assert (out_g2 - ref).abs().max().item() <= 1e-4 * scale + 1e-6


@pytest.mark.parametrize("M,N,K", [(1, 256, 512), (64, 384, 200), (128, 1000, 576), (300, 640, 1024)])
def test_gemm_tiled_weights(cuda, M, N, K):
    """Weights in the B200 tile layout (bulk-copied 16 KiB UMMA tiles) give the
    same result as the TMA path (up to fp32 summation order); the tile
    transform round-trips exactly."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    wt = mux.weight_tile(w)
    back = torch.empty_like(w)
    mux._lib.check(mux.lib.mux_weight_tile(wt.data_ptr(), N, K, back.data_ptr(), 1, None))
    a = torch.empty(M, N, dtype=torch.float32, device="cuda")
    b = torch.empty(M, N, dtype=torch.float32, device="cuda")
    mux.gemm_bf16(x, w, a, epilogue=3)
    mux.gemm_bf16(x, w, b, epilogue=3, w_tiled=wt)
    torch.cuda.synchronize()
    assert torch.equal(back, w)
    # same products; the tiled path may split K differently across CTAs (CTA
    # pairs for decode shapes), so only the fp32 summation order may differ
    assert (a - b).abs().max().item() <= 1e-5 * a.abs().max().item() + 1e-6


@pytest.mark.parametrize("M,N,K", [(300, 512, 576), (1000, 1024, 1024), (4096, 512, 256), (257, 768, 320)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_gemm_prefill_cta_pairs(cuda, M, N, K, epi):
    """Prefill shapes with tiled weights run on CTA pairs (tcgen05
    cta_group::2, gemm_2sm.cu): every epilogue against an fp32 reference."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + epi)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    wt = mux.weight_tile(w)
    ref = x.float() @ w.float().T
    scale = ref.abs().max().item()
    if epi == 0:
        out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        mux.gemm_bf16(x, w, out, epilogue=0, w_tiled=wt)
        torch.cuda.synchronize()
        assert (out.float() - ref).abs().max().item() <= 1e-2 * scale
    elif epi == 1:
        resid0 = torch.randn(M, N, generator=g, device="cuda")
        out = resid0.clone()
        mux.gemm_bf16(x, w, out, epilogue=1, w_tiled=wt)
        torch.cuda.synchronize()
        assert (out - (resid0 + ref)).abs().max().item() <= 1e-4 * scale + 1e-5
    elif epi == 2:
        out = torch.empty(M, N // 2, dtype=torch.bfloat16, device="cuda")
        mux.gemm_bf16(x, w, out, epilogue=2, w_tiled=wt)
        torch.cuda.synchronize()
        gate, up = ref[:, 0::2], ref[:, 1::2]
        want = gate * torch.sigmoid(gate) * up
        assert (out.float() - want).abs().max().item() <= 2e-2 * want.abs().max().item() + 1e-3
    else:
        out = torch.empty(M, N, dtype=torch.float32, device="cuda")
        mux.gemm_bf16(x, w, out, epilogue=3, w_tiled=wt)
        torch.cuda.synchronize()
        assert (out - ref).abs().max().item() <= 1e-4 * scale + 1e-6


def test_gemm_deterministic(cuda):
    import torch
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(128, 4096, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4096, 4096, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    outs = []
    for _ in range(3):
        o = torch.empty(128, 4096, dtype=torch.float32, device="cuda")
        mux.gemm_bf16(x, w, o, epilogue=3)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("M", [3, 64, 300])
def test_gemm_silu_epilogue(cuda, M):
    import torch
    K, F = 512, 384  # W rows interleaved: gate_i, up_i
    g = torch.Generator(device="cuda").manual_seed(M)
    x = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(2 * F, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    out = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    mux.gemm_bf16(x, w, out, epilogue=2)
    torch.cuda.synchronize()
    y = x.float() @ w.float().T
    gate, up = y[:, 0::2], y[:, 1::2]
    ref = torch.nn.functional.silu(gate) * up
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("lens,H,seed", [
    ([1], 2, 0),
    ([7, 33], 4, 1),
    ([128, 129, 5], 2, 2),
    ([300, 161, 513], 4, 3),
    ([1024], 1, 4),
])
def test_prefill_attention_tcgen05_matches_oracle(cuda, lens, H, seed):
    """K3 (tcgen05 flash attention) vs the fp64 causal oracle on the same bf16
    q/k/v; bf16 output within 1e-2 of max|out| (P is rounded to bf16 before
    the P.V contraction, as in every flash-attention kernel)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    T = sum(lens)
    qkv = (torch.randn(T, 3, H, 128, generator=g) * 2.0).to(torch.bfloat16)
    q = (torch.randn(T, H, 128, generator=g) * 2.0).to(torch.bfloat16)
    out = torch.zeros(T, H, 128, dtype=torch.bfloat16)
    qd, qkvd, od = q.cuda(), qkv.cuda(), out.cuda()
    mux.prefill_attention(qd, qkvd, od, lens)
    got = od.float().cpu().numpy()
    ref = llama_ref.prefill_attention_ref(q.float().numpy(), qkv[:, 1].float().numpy(),
                                          qkv[:, 2].float().numpy(), lens)
    err = np.abs(got - ref).max() / max(1e-6, np.abs(ref).max())
    assert err <= 1e-2, err


@pytest.mark.parametrize("ctas", [1, 3, 7])
def test_prefill_attention_many_items_per_cta(cuda, monkeypatch, ctas):
    """K3's persistent schedule with a small grid (MUX_K3_CTAS): dozens of
    items per CTA, mostly one key tile each, so the producer's cursors cross
    items every tile (4-deep descriptor ring, Q buffers by item parity,
    prefetched item descriptors) -- same oracle bound as above."""
    import torch
    monkeypatch.setenv("MUX_K3_CTAS", str(ctas))
    rng = np.random.default_rng(10 + ctas)
    lens = [int(x) for x in rng.integers(1, 140, size=23)] + [1, 128, 129, 300, 257]
    H = 3
    g = torch.Generator().manual_seed(ctas)
    T = sum(lens)
    qkv = (torch.randn(T, 3, H, 128, generator=g) * 2.0).to(torch.bfloat16)
    q = (torch.randn(T, H, 128, generator=g) * 2.0).to(torch.bfloat16)
    out = torch.zeros(T, H, 128, dtype=torch.bfloat16)
    qd, qkvd, od = q.cuda(), qkv.cuda(), out.cuda()
    mux.prefill_attention(qd, qkvd, od, lens)
    got = od.float().cpu().numpy()
    ref = llama_ref.prefill_attention_ref(q.float().numpy(), qkv[:, 1].float().numpy(),
                                          qkv[:, 2].float().numpy(), lens)
    err = np.abs(got - ref).max() / max(1e-6, np.abs(ref).max())
    assert err <= 1e-2, err
