"""Summarise an ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] CSV launch list (per kernel: launches, time, share,
average, DRAM GB/s when the byte metrics were collected)."""
import collections
import csv
import sys


def main(path, skip_prefix=("init_normal", "fill_kernel")):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
    ii = h.index("ID")
    launches = collections.defaultdict(dict)  # (id) -> {metric: value}
    names = {}
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        if name.startswith(skip_prefix):
            continue
        v = float(r[vi].replace(",", ""))
        m = r[mi]
        if m == "gpu__time_duration.sum":
            v *= scale.get(r[ui], 1e-3)  # -> us
        elif m.startswith("dram__bytes"):
            v *= bscale.get(r[ui], 1.0)  # -> bytes
        launches[r[ii]][m] = v
        names[r[ii]] = name
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, ms in launches.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += ms.get("gpu__time_duration.sum", 0.0)
        a[2] += ms.get("dram__bytes_read.sum", 0.0) + ms.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':46s} {'n':>6s} {'total ms':>9s} {'share':>6s} {'avg us':>9s} {'DRAM GB/s':>9s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        bw = b / (t * 1e-6) / 1e9 if t > 0 and b > 0 else float("nan")
        print(f"{k[:46]:46s} {n:6d} {t / 1e3:9.3f} {100 * t / tot:5.1f}% {t / n:9.2f} {bw:9.0f}")
    print(f"total {tot / 1e3:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
