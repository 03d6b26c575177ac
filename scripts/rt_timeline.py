"""Summarise a real-time serving timeline (MUX_RT_TIMELINE csv from
serve.py --realtime): per model, decode-job device time; the time both
models' decode jobs were on the device together; the union of busy time.

    MUX_RT_TIMELINE=t.csv python serve.py --realtime ...; python scripts/rt_timeline.py t.csv
"""
import csv
import json
import sys


def union(iv):
    tot, cur = 0.0, None
    for a, b in sorted(iv):
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    return tot + (cur[1] - cur[0] if cur else 0.0)


DECODE_SM = 0.405  # the calibrated profile's f_sat, the decode share the engine gives a decode job


def main(path):
    rows = [dict(r) for r in csv.DictReader(open(path))]
    for r in rows:
        r["start_ms"], r["end_ms"] = float(r["start_ms"]), float(r["end_ms"])
    out = {}
    by = {}
    for r in rows:
        by.setdefault((r["llm"], r["kind"]), []).append((r["start_ms"], r["end_ms"], int(r["batch"])))
    for k, v in sorted(by.items()):
        d = sorted(b - a for a, b, _ in v)
        out[f"llm{k[0]}_{k[1]}"] = {"jobs": len(v), "busy_ms": round(union([(a, b) for a, b, _ in v]), 1),
                                    "median_ms": round(d[len(d) // 2], 3),
                                    "mean_batch": round(sum(n for *_, n in v) / len(v), 1)}
    d0 = [(a, b) for a, b, _ in by.get(("0", "decode"), [])]
    d1 = [(a, b) for a, b, _ in by.get(("1", "decode"), [])]
    both = union(d0) + union(d1) - union(d0 + d1)
    allj = [(r["start_ms"], r["end_ms"]) for r in rows]
    out["decode_overlap_ms"] = round(both, 1)
    # interference: a decode job is "overlapped" when the other model's
    # decode jobs cover >= 90% of its span (no prefill), "solo" when other
    # jobs cover <= 10%;
    # per model, the median duration ratio over matched batch buckets gives
    # the slowdown, and kappa = (slowdown - 1) / the other job's SM share
    # (sim_engine.cpp:16-18 interference_adjust), decode_sm = --decode-sm
    dec = {"0": sorted(by.get(("0", "decode"), [])), "1": sorted(by.get(("1", "decode"), []))}

    def covered(a, b, others):
        return union([(max(a, x), min(b, y)) for x, y, _ in others if y > a and x < b]) / max(b - a, 1e-9)

    slow = {}
    pre = by.get(("0", "prefill"), []) + by.get(("1", "prefill"), [])
    for m, other in (("0", "1"), ("1", "0")):
        buckets = {}
        for a, b, n in dec[m]:
            c = covered(a, b, dec[other])
            cp = covered(a, b, pre)
            # solo: nothing else on the device; overlapped: the other model's
            # decode throughout and no prefill
            kind = "over" if c >= 0.9 and cp <= 0.1 else "solo" if c + cp <= 0.1 else None
            if kind:
                buckets.setdefault(n // 8, {"over": [], "solo": []})[kind].append(b - a)
        ratios, weights = [], []
        for v in buckets.values():
            if len(v["over"]) >= 3 and len(v["solo"]) >= 3:
                med = lambda xs: sorted(xs)[len(xs) // 2]
                ratios.append(med(v["over"]) / med(v["solo"]))
                weights.append(min(len(v["over"]), len(v["solo"])))
        if ratios:
            slow[m] = sum(r * w for r, w in zip(ratios, weights)) / sum(weights)
    out["decode_slowdown_overlapped"] = {f"llm{m}": round(v, 3) for m, v in slow.items()}
    if slow:
        mean = sum(slow.values()) / len(slow)
        out["kappa_estimate"] = round((mean - 1.0) / DECODE_SM, 2)
    out["device_busy_ms"] = round(union(allj), 1)
    out["span_ms"] = round(max(b for _, b in allj) - min(a for a, _ in allj), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1])
