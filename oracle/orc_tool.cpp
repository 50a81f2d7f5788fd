// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Command-line driver: bundle training (the reference's `cdvz train` on a
// synthetic corpus) and per-frame statistics used to size GPU buffers.
//   orc_tool train <corpus_seed> <count> <w> <h> <seed> <gmm> <em> > bundle.txt
//   orc_tool stats <bundle> <base_seed> <frames> <w> <h> <mode>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>

#include "oracle.hpp"

using namespace orc;

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "train" && argc == 9) {
      std::vector<Plane> corpus;
      for (int i = 0; i < std::atoi(argv[3]); ++i)
        corpus.push_back(synth_image(corpus_seed(std::strtoull(argv[2], nullptr, 10), i), std::atoi(argv[4]), std::atoi(argv[5])));
      TrainOptions o;
      o.seed = std::strtoull(argv[6], nullptr, 10);
      o.gmm_components = std::atoi(argv[7]);
      o.em_iterations = std::atoi(argv[8]);
      std::cout << serialize_model(train_model(corpus, o));
      return 0;
    }
    if (cmd == "stats" && argc == 8) {
      std::ifstream in(argv[2], std::ios::binary);
      std::stringstream buf;
      buf << in.rdbuf();
      const ModelBundle b = parse_model(buf.str());
      const uint64_t base = std::strtoull(argv[3], nullptr, 10);
      const int frames = std::atoi(argv[4]), w = std::atoi(argv[5]), h = std::atoi(argv[6]);
      const ModeSpec& mode = mode_by_name(argv[7]);
      double ms = 0.0;
      for (int f = 0; f < frames; ++f) {
        const Plane img = plane_from_u8(plane_to_u8(synth_image(corpus_seed(base, f), w, h)).data(), w, h, std::size_t(w));
        EncodeTrace tr;
        const auto t0 = std::chrono::steady_clock::now();
        const EncodedImage e = encode_image(img, b, mode, 640, nullptr, &tr);
        ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::printf("frame %d:", f);
        for (std::size_t o = 0; o < tr.detect.candidates.size(); ++o)
          std::printf(" o%zu cand=%zu ref=%zu", o, tr.detect.candidates[o].size(), tr.detect.refined[o].size());
        std::printf(" kp=%zu sel=%zu oriented=%zu codes=%zu bytes=%zu\n", tr.keypoints.size(), tr.selected.size(),
                    tr.oriented.size(), e.codes.size(), serialize_container(e).size());
      }
      std::printf("mean encode ms/frame (1 thread): %.2f\n", ms / frames);
      return 0;
    }
    std::fprintf(stderr, "usage: orc_tool train|stats ...\n");
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
