#!/usr/bin/env python
"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python tools/launch_summary.py launches.csv > summary.txt"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path, errors="replace")) if len(r) > 5]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        v = float(r[iv].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[iu], 1e-6)
        tot[r[ik]][0] += 1
        tot[r[ik]][1] += v * scale
    all_ms = sum(t for _, t in tot.values())
    print("# launches  total_ms  us/launch  share  kernel")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:10d} {t:9.3f} {1e3 * t / n:10.1f} {100 * t / all_ms:6.1f}%  {k[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
