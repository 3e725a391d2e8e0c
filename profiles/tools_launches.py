"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel (share of time)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")[:48]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:48s} n={v[0]:5d} total={v[1]:10.1f}us avg={v[1] / v[0]:8.2f}us share={v[1] / tot * 100:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
