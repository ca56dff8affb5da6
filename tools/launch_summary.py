#!/usr/bin/env python3
"""ncu launch list (--metrics gpu__time_duration.sum --csv) -> markdown share table."""
import collections
import csv
import sys


def main():
    src, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:72]
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + float(r[vi].replace(",", "")) * scale)
    tot = sum(t for _, t in agg.values())
    print(f"# {title}\n\n| kernel | launches | total ms | share |\n|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main()
