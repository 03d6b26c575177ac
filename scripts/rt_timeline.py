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
    out["device_busy_ms"] = round(union(allj), 1)
    out["span_ms"] = round(max(b for _, b in allj) - min(a for a, _ in allj), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1])
