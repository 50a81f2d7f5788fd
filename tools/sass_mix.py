"""Opcode mix (executed % / stall-sample %) per kernel from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    seen = set()
    for b in blocks:
        if b["name"] in seen:
            continue
        seen.add(b["name"])
        h = b["rows"][0]
        si, wi, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        op, opi = collections.Counter(), collections.Counter()
        for r in b["rows"][1:]:
            if len(r) <= wi:
                continue
            try:
                s, i = int(r[wi] or 0), int(float(r[ie] or 0))
            except ValueError:
                continue
            m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si].strip())
            name = m.group(2) if m else "?"
            op[name] += s
            opi[name] += i
        tot, toti = sum(op.values()) or 1, sum(opi.values()) or 1
        print(b["name"][:60])
        print("  " + " ".join(f"{k}:{100 * opi[k] / toti:.1f}/{100 * v / tot:.1f}" for k, v in op.most_common(20)))


if __name__ == "__main__":
    main(sys.argv[1])
