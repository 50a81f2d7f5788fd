"""Per-source-line stall samples / executed instructions from
`ncu --page source --csv --print-source cuda,sass` (needs -lineinfo)."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    src_lines = {}
    stalls = collections.Counter()
    execd = collections.Counter()
    cur_file = None
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 6:
            continue
        # columns: Line No, Source(cuda), Address, Source(sass), stall all, stall not-issued, #samples, executed...
        line, csrc = r[0], r[1]
        if line:
            key = (cur_file, int(line))
            src_lines[key] = csrc.strip()
            last = key
        try:
            stalls[last] += int(r[4] or 0)
            execd[last] += int(float(r[7] or 0))
        except (ValueError, UnboundLocalError, IndexError):
            pass
    tot, toti = sum(stalls.values()) or 1, sum(execd.values()) or 1
    for key, v in stalls.most_common(top):
        print(f"{100 * v / tot:5.1f}% stall {100 * execd[key] / toti:5.1f}% inst  {key[0]}:{key[1]}  {src_lines.get(key, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
