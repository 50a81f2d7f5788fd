"""Group per-source-line instruction/stall counts of one kernel into line ranges:
  python tools/src_regions.py REP KERNEL FILE a-b:name [a-b:name ...]"""
import collections
import csv
import subprocess
import sys


def main(rep, kernel, fname, specs):
    regions = []
    for s in specs:
        rng, name = s.split(":", 1)
        a, b = rng.split("-")
        regions.append((int(a), int(b), name))
    raw = subprocess.run(["ncu", "-i", rep, "-k", kernel, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur = None
    agg, st = collections.Counter(), collections.Counter()
    for r in csv.reader(raw.splitlines()):
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0] or r[0] == "Line No":
            continue
        try:
            ln, i, s = int(r[0]), int(r[7]), int(r[4])
        except ValueError:
            continue
        name = "other:" + str(cur)
        if cur == fname:
            for a, b, n in regions:
                if a <= ln <= b:
                    name = n
        agg[name] += i
        st[name] += s
    ti, ts = sum(agg.values()) or 1, sum(st.values()) or 1
    for k, v in agg.most_common():
        print(f"{k:28s} inst {100 * v / ti:5.1f}%  stall {100 * st[k] / ts:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:])
