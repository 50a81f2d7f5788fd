"""Regenerates tests/golden/oracle_containers.json.

The reference ships no golden files (all its fixtures are seeded synthesis).
Each container here is produced by the REFERENCE ITSELF (oracle/_ref, its
sources built against the Eigen-subset, tests/ref_lib.py) and must equal the
oracle's, so the hashes pin both: frames are synth_image(seed, w, h) quantised
to bytes, encoded with the committed bundles. Run: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib  # noqa: E402
import ref_lib  # noqa: E402

CASES = [
    dict(seed=1000, w=640, h=480, mode=0, bundle="b8"),   # config 1: one VGA frame, 512B
    dict(seed=1001, w=640, h=480, mode=3, bundle="b8"),   # config 2 frame, 4K
    dict(seed=1002, w=640, h=480, mode=3, bundle="b512"),
    dict(seed=77, w=320, h=240, mode=5, bundle="b8"),
    dict(seed=78, w=320, h=240, mode=4, bundle="b512"),
    dict(seed=5, w=1920, h=1080, mode=5, bundle="b8"),    # config 3: 1080p -> 640x360, 16K
    dict(seed=9, w=97, h=61, mode=1, bundle="b8"),
    dict(seed=11, w=15, h=15, mode=2, bundle="b8"),       # below one octave: no keypoints
]


def main():
    out = {"generator": "tests/golden/make_golden.py (containers of the reference's own encode_image, oracle/_ref; "
                        "the oracle's are asserted equal)", "cases": []}
    for c in CASES:
        frame = ref_lib.synth_u8(c["seed"], c["w"], c["h"])
        assert (frame == oracle_lib.synth_u8(c["seed"], c["w"], c["h"])).all()
        blob = ref_lib.encode(oracle_lib.bundle_text(c["bundle"]), frame, c["mode"])
        assert blob == oracle_lib.encode(oracle_lib.bundle_text(c["bundle"]), frame, c["mode"]), c
        out["cases"].append(dict(c, frame_sha256=hashlib.sha256(frame.tobytes()).hexdigest(),
                                 container_sha256=hashlib.sha256(blob).hexdigest(), container_bytes=len(blob)))
        print(c, len(blob))
    with open(os.path.join(HERE, "oracle_containers.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
