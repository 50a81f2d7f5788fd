"""Hot SASS of one kernel from `ncu --page source --csv --print-source sass`:
basic blocks (runs of instructions with equal execution counts) ordered by
warp instructions executed.   python tools/sass_hot.py CSV KERNEL_SUBSTR [N]"""
import csv
import sys


def blocks(path, name):
    rows = list(csv.reader(open(path)))
    cur, out = None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = name in r[1]
            hdr = None
            continue
        if not cur:
            continue
        if r and r[0] == "Address":
            hdr = r
            ai, si, ie, st = r.index("Address"), r.index("Source"), r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= ie:
            continue
        try:
            out.append((r[ai], r[si].strip(), int(float(r[ie] or 0)), int(float(r[st] or 0))))
        except ValueError:
            pass
    return out


def main():
    path, name = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    ins = blocks(path, name)
    tot = sum(i[2] for i in ins) or 1
    stot = sum(i[3] for i in ins) or 1
    bbs, cur = [], []
    for i in ins:
        if cur and i[2] != cur[-1][2]:
            bbs.append(cur)
            cur = []
        cur.append(i)
    if cur:
        bbs.append(cur)
    bbs.sort(key=lambda b: -sum(i[2] for i in b))
    print(f"total warp instructions {tot}")
    for b in bbs[:n]:
        ex = sum(i[2] for i in b)
        print(f"--- {b[0][0]} x{b[0][2]}  {len(b)} instr  {100 * ex / tot:.1f}% inst  {100 * sum(i[3] for i in b) / stot:.1f}% stalls")
        for i in b:
            print(f"    {i[1][:70]:70s} {i[3]}")


if __name__ == "__main__":
    main()
