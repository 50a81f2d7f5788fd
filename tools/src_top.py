"""Top CUDA source lines of one kernel by executed warp instructions (and
stall samples), from an ncu report with -lineinfo:
   python tools/src_top.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys


def main(rep, kernel, n=40):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    out, ie, st, fname = [], None, None, ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            ie, st = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
            continue
        if ie is None or not r or not r[0] or len(r) <= ie:
            continue
        try:
            out.append((int(r[ie] or 0), int(r[st] or 0), f"{fname}:{r[0]}", r[1].strip()[:88]))
        except ValueError:
            pass
    tot = sum(o[0] for o in out) or 1
    stot = sum(o[1] for o in out) or 1
    print(f"total warp instructions {tot}")
    for o in sorted(out, reverse=True)[:n]:
        print(f"{100 * o[0] / tot:5.1f}% {100 * o[1] / stot:5.1f}%  {o[2]:>18} {o[3]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
