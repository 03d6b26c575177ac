"""Measured B200 latency profile.

The reference prices every job with an analytic LatencyProfile
(/root/reference/proj/include/muxsim/cost_model.hpp:33-50,
/root/reference/proj/src/cost_model.cpp:75-94):

    prefill  = prefill_ms_per_token * scale * tokens * (1/f) / tp_speedup
    decode   = (decode_base_ms + decode_ctx_ms_per_token * ctx) * scale
               * max(1, batch / batch_knee) * (f >= f_sat ? 1 : 1/f) / tp_speedup
    scale    = num_layers * hidden_size / reference_scale

Its defaults are placeholders. This module times the real jobs of this
framework on the GPU (prefill = K3 + tcgen05 GEMMs, decode = K1 + K2 +
GEMMs, on green-context SM partitions for the SM share) and fits the same
seven parameters, so the reference's planner and priced simulator -- and this
framework's priced engine -- run on B200 costs:

    python -m paper_2404_02015_b200.calibrate -o b200_profile.json

The reference's decode form is not how a B200 decode step behaves: the step
streams the weights once plus every member's K/V, so its time is linear in
batch x context, and a partial SM share slows it as f^-0.6, not flat then
1/f. fit_profile() therefore also fits the HBM-bound form
(LatencyProfile::decode_form 1, a B200 extension; csrc/host/spec.cpp):

    decode   = (decode_fixed_ms + decode_row_ms * b + decode_bctx_ms * b * ctx)
               * scale * f^-decode_sm_exponent / tp_speedup

and, with hbm=True, adds its four keys (wire.HBM_KEYS). main() writes them
as a separate "profile_hbm" object: the reference's config.cpp rejects
unknown profile keys, so "profile" stays a reference block; merged into
"profile" for this framework's CLI (wire.load_config), they select the form.

The output's "profile" object drops into a reference config unchanged
(config.cpp "profile" section; wire.load_config reads it too). tp_efficiency
needs a multi-GPU mesh and keeps its default on a one-GPU box (stated in the
output). fit_profile() is pure host code (tests/test_calibrate.py).
"""
from __future__ import annotations

import argparse
import json
import math
import sys

REFERENCE_SCALE = 32.0 * 4096.0          # cost_model.hpp:40 (7B has scale 1)
DEFAULTS = {"prefill_ms_per_token": 0.25, "decode_base_ms": 12.0, "decode_ctx_ms_per_token": 0.005,
            "tp_efficiency": 0.9, "sm_saturation_point": 0.5, "batch_knee": 16.0,
            "reference_scale": REFERENCE_SCALE}


def model_scale(num_layers: int, hidden: int) -> float:
    return num_layers * hidden / REFERENCE_SCALE


def _lstsq2(xs, ys, ws):
    """Weighted least squares y ~ a + b x; returns (a, b)."""
    sw = sum(ws)
    sx = sum(w * x for w, x in zip(ws, xs))
    sy = sum(w * y for w, y in zip(ws, ys))
    sxx = sum(w * x * x for w, x in zip(ws, xs))
    sxy = sum(w * x * y for w, x, y in zip(ws, xs, ys))
    det = sw * sxx - sx * sx
    if abs(det) < 1e-300:
        return sy / sw, 0.0
    b = (sw * sxy - sx * sy) / det
    return (sy - b * sx) / sw, b


def fit_prefill(points, scale):
    """points: [(tokens, ms)] -> prefill_ms_per_token (through the origin,
    relative error weighting: sum(t*ms/ms^2) / sum(t^2/ms^2))."""
    num = sum(t * ms / (ms * ms) for t, ms in points)
    den = sum(t * t / (ms * ms) for t, ms in points)
    return num / den / scale


def fit_decode(points, scale):
    """points: [(batch, ctx, ms)] -> (decode_base_ms, decode_ctx_ms_per_token,
    batch_knee, rel_rms). Knee by search; base/ctx by weighted least squares
    on ms / max(1, b/knee) (relative errors)."""
    best = None
    knees = sorted({float(b) for b, _, _ in points} | {1.0 * 2 ** (k / 4) for k in range(0, 37)})
    for knee in knees:
        xs = [c for _, c, _ in points]
        ys = [ms / max(1.0, b / knee) for b, _, ms in points]
        ws = [1.0 / (y * y) for y in ys]
        a, k = _lstsq2(xs, ys, ws)
        if a <= 0 or k < 0:
            continue
        err = math.sqrt(sum(((a + k * c) * max(1.0, b / knee) / ms - 1.0) ** 2 for b, c, ms in points) / len(points))
        if best is None or err < best[3]:
            best = (a / scale, k / scale, knee, err)
    if best is None:
        raise ValueError("decode fit failed (non-positive coefficients)")
    return best


def fit_sm_saturation(points):
    """points: [(f, ms)] with f = SM share in (0, 1] (1.0 included) ->
    (f_sat, rel_rms) of the reference's step model: flat at t(1) for
    f >= f_sat, t(1)/f below (cost_model.cpp:65-72)."""
    t1 = [ms for f, ms in points if f >= 0.999]
    if not t1:
        raise ValueError("need a full-GPU point")
    t1 = t1[0]
    # ties (any f_sat between two measured shares fits equally): keep the
    # largest, i.e. the smallest measured share that still ran flat
    cands = sorted({f for f, _ in points} | {k / 100.0 for k in range(1, 101)}, reverse=True)
    best = None
    for fs in cands:
        err = math.sqrt(sum(((t1 if f >= fs else t1 / f) / ms - 1.0) ** 2 for f, ms in points) / len(points))
        if best is None or err < best[1] - 1e-12:
            best = (fs, err)
    return best


def _lstsq(rows, ys, ws):
    """Weighted least squares y ~ rows . coef (normal equations, Gaussian
    elimination with partial pivoting); returns coef."""
    n = len(rows[0])
    a = [[sum(w * r[i] * r[j] for r, w in zip(rows, ws)) for j in range(n)] for i in range(n)]
    v = [sum(w * r[i] * y for r, y, w in zip(rows, ys, ws)) for i in range(n)]
    for c in range(n):
        piv = max(range(c, n), key=lambda i: abs(a[i][c]))
        a[c], a[piv], v[c], v[piv] = a[piv], a[c], v[piv], v[c]
        if abs(a[c][c]) < 1e-300:
            raise ValueError("singular least-squares system")
        for i in range(c + 1, n):
            f = a[i][c] / a[c][c]
            a[i] = [x - f * y for x, y in zip(a[i], a[c])]
            v[i] -= f * v[c]
    coef = [0.0] * n
    for i in reversed(range(n)):
        coef[i] = (v[i] - sum(a[i][j] * coef[j] for j in range(i + 1, n))) / a[i][i]
    return coef


def fit_decode_hbm(points, scale):
    """points: [(batch, ctx, ms)] -> (decode_fixed_ms, decode_row_ms,
    decode_bctx_ms, rel_rms) of the HBM-bound form: ms = (fixed + row * b +
    bctx * b * ctx) * scale, relative-error weighted. A negative per-row
    term (too few batch sizes to separate it) is dropped to 0 and refit."""
    ys = [ms for _, _, ms in points]
    ws = [1.0 / (y * y) for y in ys]
    base, row, bctx = _lstsq([(1.0, b, b * c) for b, c, _ in points], ys, ws)
    if row < 0:
        row = 0.0
        base, bctx = _lstsq([(1.0, b * c) for b, c, _ in points], ys, ws)
    if base <= 0 or bctx <= 0:
        raise ValueError("HBM decode fit failed (non-positive coefficients)")
    err = math.sqrt(sum(((base + row * b + bctx * b * c) / ms - 1.0) ** 2 for b, c, ms in points) / len(points))
    return base / scale, row / scale, bctx / scale, err


def fit_sm_exponent(points):
    """points: [(f, ms)] with a full-GPU point -> (exponent, rel_rms) of
    ms = t(1) * f^-exponent (log-log least squares through t(1)), clamped to
    [0, 1]."""
    t1 = [ms for f, ms in points if f >= 0.999]
    if not t1:
        raise ValueError("need a full-GPU point")
    t1 = t1[0]
    xs = [(-math.log(f), math.log(ms / t1)) for f, ms in points if f < 0.999]
    e = sum(x * y for x, y in xs) / sum(x * x for x, _ in xs) if xs else 0.0
    e = min(1.0, max(0.0, e))
    err = math.sqrt(sum((t1 * f ** -e / ms - 1.0) ** 2 for f, ms in points) / len(points))
    return e, err


def fit_profile(prefill_pts, decode_pts, sm_pts, num_layers, hidden, hbm=False):
    """All measurements of one model -> the LatencyProfile dict + fit report
    (hbm=True: plus the HBM-bound decode form's keys and fit errors)."""
    scale = model_scale(num_layers, hidden)
    pf = fit_prefill(prefill_pts, scale)
    base, ctx, knee, derr = fit_decode(decode_pts, scale)
    fsat, serr = fit_sm_saturation(sm_pts) if sm_pts else (DEFAULTS["sm_saturation_point"], None)
    prof = dict(DEFAULTS)
    prof.update({"prefill_ms_per_token": pf, "decode_base_ms": base, "decode_ctx_ms_per_token": ctx,
                 "batch_knee": knee, "sm_saturation_point": fsat})
    perr = math.sqrt(sum((pf * scale * t / ms - 1.0) ** 2 for t, ms in prefill_pts) / len(prefill_pts))
    err = {"prefill_rel_rms": perr, "decode_rel_rms": derr, "sm_rel_rms": serr}
    if not hbm:
        return prof, err
    try:
        hbase, hrow, hbctx, herr = fit_decode_hbm(decode_pts, scale)
    except ValueError:
        return prof, err  # reference form only
    sexp, sexp_err = fit_sm_exponent(sm_pts) if sm_pts else (0.6, None)
    prof.update({"decode_fixed_ms": hbase, "decode_row_ms": hrow, "decode_bctx_ms": hbctx,
                 "decode_sm_exponent": sexp})
    err.update({"decode_hbm_rel_rms": herr, "sm_exponent_rel_rms": sexp_err})
    return prof, err


# ------------------------------------------------------------------- GPU side

def _time(unit, partition, fn, warmup=2, iters=5):
    for _ in range(warmup):
        fn()
    unit.sync()
    unit.record(partition, 0)
    for _ in range(iters):
        fn()
    unit.record(partition, 1)
    unit.sync()
    return unit.elapsed_ms(0, 1) / iters


def measure(model="7b", device=0, decode_batches=(1, 4, 16, 32, 64, 128, 256), decode_ctx=(128, 512, 2048),
            prefill_tokens=(256, 512, 1024, 2048, 4096), sm_granules=(4, 6, 9, 12, 18), max_kv_tokens=1 << 17,
            sm_batch=64, sm_ctx=512):
    """Time prefill / decode jobs of `model` (random-init weights and KV) on
    this GPU. Returns the measurement tables fit_profile takes."""
    import numpy as np
    import torch

    from . import Unit, blocks_for_tokens, spec
    s = spec(model)
    nsm = torch.cuda.get_device_properties(device).multi_processor_count
    max_b = max(decode_batches)
    kv_need = blocks_for_tokens(s, 16, max_kv_tokens + 16 * max_b * 8) + blocks_for_tokens(s, 16, 4096 + 16)
    rng = np.random.default_rng(0)

    def make_unit(psms=None):
        u = Unit([s], pool_blocks=kv_need, device=device, device_pool_blocks=kv_need, max_batch=max_b,
                 max_prefill_tokens=max(prefill_tokens), max_ctx=max(max(decode_ctx), max(prefill_tokens)) + 64,
                 max_slots=2 * max_b + 64, init_seed=1, init_std=0.02, partitions=2,
                 partition_sms=psms)
        u.init_kv(seed=3, std=1.0)
        return u

    def decode_ms(u, part, b, c):
        rids = list(range(10_000, 10_000 + b))
        for r in rids:
            assert u.pool.admit(0, r, c, c + 64).ok
        steps = [0]

        def step():
            for r in rids:
                assert u.pool.alloc(0, r, 1, False).ok
            u.decode(0, rids, partition=part)
            steps[0] += 1
        ms = _time(u, part, step, warmup=2, iters=5)
        for r in rids:
            u.pool.free_request(0, r)
        return ms

    unit = make_unit()
    try:
        prefill = []
        for t in sorted(set(prefill_tokens)):  # untimed warm-up of every shape (maps, staging, caches)
            toks = rng.integers(0, s.vocab, t).astype(np.int32)
            assert unit.pool.admit(0, 1, t, t + 1).ok
            unit.prefill(0, [1], toks, np.zeros(1, np.int32))
            unit.sync()
            unit.pool.free_request(0, 1)
        for t in prefill_tokens:
            toks = rng.integers(0, s.vocab, t).astype(np.int32)
            out = np.zeros(1, np.int32)
            best = None
            for rep in range(3):  # one job at a time: its device span, host prep excluded
                rid = 1 + rep
                assert unit.pool.admit(0, rid, t, t + 1).ok
                unit.sync()
                unit.record(0, 0)
                unit.prefill(0, [rid], toks, out)
                unit.record(0, 1)
                unit.sync()
                ms = unit.elapsed_ms(0, 1)
                best = ms if best is None else min(best, ms)
                unit.pool.free_request(0, rid)
            prefill.append((t, best))
        decode = []
        for c in decode_ctx:
            for b in decode_batches:
                if b * c <= max_kv_tokens:
                    decode.append((b, c, decode_ms(unit, 0, b, c)))
        full = decode_ms(unit, 0, sm_batch, sm_ctx)
    finally:
        unit.close()
    sm = [(1.0, full)]
    for g in sm_granules:
        n = 8 * g
        if n >= nsm:
            continue
        u = make_unit([0, n])
        try:
            got = u.partition_sms(1)
            sm.append((got / nsm, decode_ms(u, 1, sm_batch, sm_ctx)))
        finally:
            u.close()
    return {"model": model, "num_layers": s.num_layers, "hidden": s.hidden_size, "sms": nsm,
            "prefill": prefill, "decode": decode, "sm_share": sm}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--model", default="7b")
    ap.add_argument("-o", "--output", default="b200_profile.json")
    ap.add_argument("--tp-allreduce", default=None,
                    help="JSON from scripts/tp_allreduce_cost.py: adds its allreduce_alpha_ms / "
                         "allreduce_ms_per_mib (wire.TP_KEYS) as the profile_tp block")
    a = ap.parse_args(argv)
    m = measure(a.model)
    prof, err = fit_profile(m["prefill"], m["decode"], m["sm_share"], m["num_layers"], m["hidden"], hbm=True)
    from .wire import HBM_KEYS
    prof_hbm = {k: prof.pop(k) for k in HBM_KEYS if k in prof}
    prof_tp = None
    if a.tp_allreduce:
        from .wire import TP_KEYS
        with open(a.tp_allreduce) as f:
            tpm = json.load(f)
        prof_tp = {k: float(tpm[k]) for k in TP_KEYS}
    out = {"profile": prof, "profile_hbm": prof_hbm, "profile_tp": prof_tp, "fit": err, "measurements": m,
           "notes": {"tp_efficiency": "default 0.9: needs a multi-GPU mesh (one-GPU box); profile_tp, when "
                                      "present, replaces eta * tp by the measured allreduce (LatencyProfile::tp_scaled)",
                     "method": "CUDA events around back-to-back jobs on one stream; decode KV random, "
                               "prefill single request of N tokens; SM share = green-context partition"}}
    with open(a.output, "w") as f:
        json.dump(out, f, indent=2)
    print(json.dumps({"profile": prof, "fit": err}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
