"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per kernel)."""
import collections
import csv
import sys


def main(path, skip_prefix=("init_normal", "fill_kernel")):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        if name.startswith(skip_prefix):
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'n':>6s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {n:6d} {t / 1e3:9.3f} {100 * t / tot:5.1f}% {t / n:9.2f}")
    print(f"total {tot / 1e3:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
