"""Static opcode mix of one kernel in a cubin/.o/.so: python tools/sass_static.py FILE NAME_SUBSTRING"""
import collections
import re
import subprocess
import sys


def main(path, pat):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for fn in funcs[1:]:
        name = fn.split("\n", 1)[0].strip()
        if pat not in name:
            continue
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z0-9_]+)", fn):
            ops[m.group(1)] += 1
        total = sum(ops.values())
        print(f"{name}: {total} instructions")
        print("  " + ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
