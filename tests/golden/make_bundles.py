"""Regenerates tests/golden/bundle_b8.txt and bundle_b512.txt with the
REFERENCE'S OWN train_model (oracle/_ref, built from /root/reference/proj by
oracle/refbuild/Makefile) on the acceptance recipe (proj/tests/acceptance/
acceptance.cpp:509-514): train_model(synth_corpus(401, 20, 256, 256),
{seed 11, gmm_components 8 | 512, em_iterations 15}).

The detector, selector/relevance, transform and quantizer sections are the
reference's bits; PCA and GMM follow the Eigen-subset's Jacobi eigen-solver
(Eigen's SelfAdjointEigenSolver is not available here), so they are this
repository's fixed choice of model data. Run: python tests/golden/make_bundles.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import ref_lib  # noqa: E402


def main():
    for name, gmm in (("b8", 8), ("b512", 512)):
        text = ref_lib.train_bundle(401, 20, 256, 256, 11, gmm, 15, workers=os.cpu_count() or 8)
        with open(os.path.join(HERE, f"bundle_{name}.txt"), "w") as f:
            f.write(text)
        print(name, len(text), "bytes, model_crc", hex(ref_lib.bundle_crc(text)[0]))


if __name__ == "__main__":
    main()
