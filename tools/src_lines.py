"""Per-source-line executed warp instructions and stall samples of one kernel
in an ncu report (needs -lineinfo):  python tools/src_lines.py REP KERNEL [TOP]."""
import csv
import subprocess
import sys


def main(rep, kernel, top=40):
    raw = subprocess.run(["ncu", "-i", rep, "-k", kernel, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    lines, cur = [], None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0] or r[0] == "Line No":
            continue
        try:
            lines.append((cur, int(r[0]), r[1][:90], int(r[4]), int(r[7]), float(r[10] or 0)))
        except ValueError:
            continue
    ti = sum(l[4] for l in lines) or 1
    ts = sum(l[3] for l in lines) or 1
    print(f"total warp instructions {ti}, stall samples {ts}")
    for f, n, s, st, i, thr in sorted(lines, key=lambda x: -x[4])[:top]:
        print(f"{f}:{n:<4d} inst {100 * i / ti:5.1f}% stall {100 * st / ts:5.1f}% thr {thr:4.1f}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
