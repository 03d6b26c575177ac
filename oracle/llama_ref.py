"""numpy restatement of the LLaMA-1 forward the B200 jobs execute
(TEST INFRASTRUCTURE ONLY -- the checker for tests/ and smoke(), never the
product).

PARITY UNPINNED for numerics: the reference prices jobs instead of running
them (/root/reference/proj/src/cost_model.cpp:75-94), so there
is no reference forward to pin against. This is standard LLaMA-1 (MHA,
head_dim 128, rotate-half RoPE theta 10000, RMSNorm eps 1e-5, SiLU-gated FFN,
greedy argmax) over the reference's KV geometry (16-token head-blocks,
kv_manager.cpp:25-40; context = prompt + 1 + steps, scheduler.cpp:107),
rounded to bf16 at the same points as the GPU path:
  xn (RMSNorm out), qkv (GEMM out), rotated q/k, attention out, SiLU*up act.
The residual stream and all accumulations are fp32 (GEMMs) / fp64 (attention).

Weights use the device layout of include/mux.h (mux_unit_set_tensor).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

EPS = 1e-5


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 (as uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    # uint32 arithmetic: only NaN/Inf patterns (exponent all ones) can carry
    # out of 32 bits, and those take the branch below
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    nan = (u & np.uint32(0x7F800000)) == np.uint32(0x7F800000)
    if nan.any():
        quiet = np.where((u & np.uint32(0xFFFF)) != 0, np.uint32(0x40), np.uint32(0))
        r = np.where(nan, (u >> np.uint32(16)) | quiet, r)
    return r.astype(np.uint16)


def round_bf16(x: np.ndarray) -> np.ndarray:
    return bf16_to_f32(f32_to_bf16(x))


def rope_table(positions: int) -> np.ndarray:
    """[positions][64][(cos, sin)] float32, computed with libm in double
    (math.pow/cos/sin), exactly as csrc/device/runtime.cu does."""
    out = np.empty((positions, 64, 2), dtype=np.float32)
    inv = [1.0 / math.pow(10000.0, 2.0 * i / 128.0) for i in range(64)]
    for p in range(positions):
        for i in range(64):
            a = float(p) * inv[i]
            out[p, i, 0] = math.cos(a)
            out[p, i, 1] = math.sin(a)
    return out


def rope_rotate(x: np.ndarray, pos: np.ndarray, table: np.ndarray) -> np.ndarray:
    """rotate-half RoPE in float32 with separately rounded products (no FMA),
    x [..., 128] float32, pos broadcastable to x[..., 0]."""
    cs = table[pos]  # [..., 64, 2]
    c = cs[..., 0].astype(np.float32)
    s = cs[..., 1].astype(np.float32)
    lo, hi = x[..., :64], x[..., 64:]
    out = np.empty_like(x)
    out[..., :64] = (lo * c).astype(np.float32) - (hi * s).astype(np.float32)
    out[..., 64:] = (hi * c).astype(np.float32) + (lo * s).astype(np.float32)
    return out


@dataclass
class Dims:
    layers: int
    heads: int
    hidden: int
    ffn: int
    vocab: int


def make_weights(d: Dims, seed: int, std: float = 0.02) -> dict:
    """Random LLaMA weights in device layout (bf16 as uint16, norms fp32)."""
    rng = np.random.default_rng(seed)

    def w(*shape):
        return f32_to_bf16(rng.standard_normal(shape, dtype=np.float32) * np.float32(std))

    out = {"embed": w(d.vocab, d.hidden), "lm_head": w(d.vocab, d.hidden),
           "final_norm": (1.0 + 0.1 * rng.standard_normal(d.hidden)).astype(np.float32)}
    for l in range(d.layers):
        out[("wqkv", l)] = w(3 * d.heads * 128, d.hidden)
        out[("wo", l)] = w(d.hidden, d.heads * 128)
        out[("wgu", l)] = w(2 * d.ffn, d.hidden)
        out[("wdown", l)] = w(d.hidden, d.ffn)
        out[("attn_norm", l)] = (1.0 + 0.1 * rng.standard_normal(d.hidden)).astype(np.float32)
        out[("ffn_norm", l)] = (1.0 + 0.1 * rng.standard_normal(d.hidden)).astype(np.float32)
    return out


def rmsnorm_bf16(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    ms = np.mean(x.astype(np.float64) ** 2, axis=-1, keepdims=True)
    inv = (1.0 / np.sqrt(ms + EPS)).astype(np.float32)
    return round_bf16((x * inv).astype(np.float32) * w)


class RefLlama:
    """One model; requests keep their own K/V caches (bf16 values as f32)."""

    def __init__(self, d: Dims, weights: dict, rope: np.ndarray):
        self.d = d
        self.rope = rope
        f = bf16_to_f32
        self.embed = f(weights["embed"])
        self.lm_head = f(weights["lm_head"])
        self.final_norm = weights["final_norm"]
        L = d.layers
        self.wqkv = [f(weights[("wqkv", l)]) for l in range(L)]
        self.wo = [f(weights[("wo", l)]) for l in range(L)]
        gu = [f(weights[("wgu", l)]) for l in range(L)]
        self.wg = [g[0::2] for g in gu]
        self.wu = [g[1::2] for g in gu]
        self.wdown = [f(weights[("wdown", l)]) for l in range(L)]
        self.attn_norm = [weights[("attn_norm", l)] for l in range(L)]
        self.ffn_norm = [weights[("ffn_norm", l)] for l in range(L)]

    def new_cache(self):
        return {"k": [np.zeros((0, self.d.heads, 128), np.float32) for _ in range(self.d.layers)],
                "v": [np.zeros((0, self.d.heads, 128), np.float32) for _ in range(self.d.layers)]}

    def _attend(self, q, K, V, causal_start):
        """q [T,H,128] (bf16 values), K/V [S,H,128]; token t sees keys < causal_start+t+1."""
        T, H = q.shape[0], q.shape[1]
        out = np.empty((T, H, 128), np.float32)
        scale = 1.0 / math.sqrt(128.0)
        for t in range(T):
            n = causal_start + t + 1
            s = np.einsum("hd,shd->hs", q[t].astype(np.float64), K[:n].astype(np.float64)) * scale
            s -= s.max(axis=1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=1, keepdims=True)
            out[t] = np.einsum("hs,shd->hd", p, V[:n].astype(np.float64)).astype(np.float32)
        return round_bf16(out)

    def forward(self, tokens: np.ndarray, cache: dict) -> np.ndarray:
        """Append `tokens` (positions continue the cache) and return the fp32
        logits of the last token."""
        d = self.d
        T = len(tokens)
        start = cache["k"][0].shape[0]
        pos = np.arange(start, start + T)
        x = self.embed[tokens].astype(np.float32)  # residual, fp32
        xn = rmsnorm_bf16(x, self.attn_norm[0])
        for l in range(d.layers):
            qkv = round_bf16(xn @ self.wqkv[l].T).reshape(T, 3, d.heads, 128)
            q = round_bf16(rope_rotate(qkv[:, 0], pos[:, None], self.rope))
            k = round_bf16(rope_rotate(qkv[:, 1], pos[:, None], self.rope))
            v = qkv[:, 2]
            cache["k"][l] = np.concatenate([cache["k"][l], k], axis=0)
            cache["v"][l] = np.concatenate([cache["v"][l], v], axis=0)
            att = self._attend(q, cache["k"][l], cache["v"][l], start).reshape(T, d.heads * 128)
            x = x + (att @ self.wo[l].T).astype(np.float32)
            xn = rmsnorm_bf16(x, self.ffn_norm[l])
            g = (xn @ self.wg[l].T).astype(np.float32)
            u = (xn @ self.wu[l].T).astype(np.float32)
            act = round_bf16((g / (1.0 + np.exp(-g))) * u)
            x = x + (act @ self.wdown[l].T).astype(np.float32)
            nw = self.attn_norm[l + 1] if l + 1 < d.layers else self.final_norm
            xn = rmsnorm_bf16(x, nw)
        return (xn[-1] @ self.lm_head.T).astype(np.float32)


def decode_batch(ref: "RefLlama", tokens: np.ndarray, positions: np.ndarray, attend) -> np.ndarray:
    """One decode step of a whole batch (the decode job of
    csrc/device/runtime.cu Runtime::decode): member i feeds tokens[i] at
    position positions[i] (its context minus one, scheduler.cpp:107).
    attend(layer, q, k, v) receives the rotated bf16 q / k and v [B, H, 128]
    (float32 holding bf16 values), appends k / v to each member's cache and
    returns attention over the whole context [B, H, 128] (float32). Same
    rounding points as RefLlama.forward; returns fp32 logits [B, vocab]."""
    d = ref.d
    B = len(tokens)
    pos = np.asarray(positions)
    x = ref.embed[np.asarray(tokens)].astype(np.float32)
    xn = rmsnorm_bf16(x, ref.attn_norm[0])
    for l in range(d.layers):
        qkv = round_bf16(xn @ ref.wqkv[l].T).reshape(B, 3, d.heads, 128)
        q = round_bf16(rope_rotate(qkv[:, 0], pos[:, None], ref.rope))
        k = round_bf16(rope_rotate(qkv[:, 1], pos[:, None], ref.rope))
        att = round_bf16(attend(l, q, k, qkv[:, 2])).reshape(B, d.heads * 128)
        x = x + (att @ ref.wo[l].T).astype(np.float32)
        xn = rmsnorm_bf16(x, ref.ffn_norm[l])
        g = (xn @ ref.wg[l].T).astype(np.float32)
        u = (xn @ ref.wu[l].T).astype(np.float32)
        act = round_bf16((g / (1.0 + np.exp(-g))) * u)
        x = x + (act @ ref.wdown[l].T).astype(np.float32)
        nw = ref.attn_norm[l + 1] if l + 1 < d.layers else ref.final_norm
        xn = rmsnorm_bf16(x, nw)
    return (xn @ ref.lm_head.T).astype(np.float32)


def prefill_attention_ref(q, k, v, seq_lens):
    """Causal varlen attention of each prompt (K3's contract), fp64.

    q, k, v: [T, H, 128] float arrays (the bf16 values the kernel reads, k and
    q already rotated); seq_lens split the T tokens into prompts. Context
    semantics follow the reference's prefill job: every prompt token attends
    to the prompt tokens up to itself (cost_model.cpp:75-83 prices exactly
    this causal pass)."""
    T, H, D = q.shape
    out = np.zeros((T, H, D), np.float64)
    scale = 1.0 / math.sqrt(D)
    s0 = 0
    for n in seq_lens:
        qs = q[s0:s0 + n].astype(np.float64).transpose(1, 0, 2)  # [H, n, D]
        ks = k[s0:s0 + n].astype(np.float64).transpose(1, 2, 0)  # [H, D, n]
        vs = v[s0:s0 + n].astype(np.float64).transpose(1, 0, 2)  # [H, n, D]
        s = np.matmul(qs, ks) * scale
        s = np.where(np.tril(np.ones((n, n), bool))[None], s, -np.inf)
        s -= s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=-1, keepdims=True)
        out[s0:s0 + n] = np.matmul(p, vs).transpose(1, 0, 2)
        s0 += n
    return out
