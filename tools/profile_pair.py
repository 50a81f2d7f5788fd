"""Turn an ncu --set full capture of the octave-0 kernel pair (k_blur<...,0>,
k_detect_walk, 256-frame batch) into profiles/octave_kernel_ncu.json, the file
bench.py reads for roofline.traffic.  python tools/profile_pair.py REP [FRAMES]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402


def gbytes(s):
    v, unit = s.split()
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}[unit]
    return float(v) * scale


def main(rep, frames=256, w=640, h=480, m=10):
    rows = ncu_summary.summarise(rep)
    blur = next(r for r in rows if r["kernel"].startswith("void k_blur<5, 5, 6, 8, 0"))
    det = next(r for r in rows if "k_detect_walk" in r["kernel"])
    traffic = sum(gbytes(r[k]) for r in (blur, det) for k in ("dram_read", "dram_write")) * 1e9
    algo = frames * (w * h * (1 + 32) + 32 * (w - 2 * m) * (h - 2 * m))
    out = {"dram_bytes_per_launch_pair": traffic, "algorithmic_bytes_per_launch_pair": algo,
           "frames_per_launch": frames,
           "note": f"octave 0 of a {frames}-frame VGA batch: k_blur (u8 in, 4 f64 levels out) + k_detect_walk "
                   "(4 levels in); ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum",
           "kernels": [blur, det]}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "octave_kernel_ncu.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 256)
