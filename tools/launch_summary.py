"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import json
import sys


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": n, "total_ms": t / 1e6, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    out = summarise(sys.argv[1])
    for r in out:
        print(f"{r['kernel']:40s} {r['launches']:5d} {r['total_ms']:9.3f} ms {100 * r['share']:5.1f}%")
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)
