// The reference CLI's `cdvz train` flow (proj/tools/cdvz.cpp:60-70) over the
// shim: list_images (cdvz.cpp:15-26), load_image, train_model on the GPU
// (cdvz_gpu_train_model), save_model, and the bundle's CRC.
//   g++ -std=c++17 examples/train.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o train
//   ./train corpus_dir bundle.txt [seed gmm_components em_iterations select_n]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <vector>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

namespace fs = std::filesystem;

int main(int argc, char** argv) {
  if (argc != 3 && argc != 7) {
    std::fprintf(stderr, "usage: train <corpus_dir> <out_bundle> [seed gmm_components em_iterations select_n]\n");
    return 1;
  }
  try {
    if (!fs::is_directory(argv[1])) throw cdvz::gpu::UsageError(std::string("not a directory: ") + argv[1]);
    std::vector<fs::path> files;
    for (const auto& e : fs::directory_iterator(argv[1])) {
      const auto ext = e.path().extension().string();
      if (e.is_regular_file() && (ext == ".pgm" || ext == ".ppm")) files.push_back(e.path());
    }
    std::sort(files.begin(), files.end());
    if (files.empty()) throw cdvz::gpu::DataError(std::string("no .pgm/.ppm images in ") + argv[1]);
    std::vector<cdvz::gpu::GrayImage> corpus;
    for (const auto& p : files) corpus.push_back(cdvz::gpu::to_gray(cdvz::gpu::load_pnm(p.string())));
    cdvz::gpu::TrainOptions opts;
    if (argc == 7) {
      opts.seed = std::strtoull(argv[3], nullptr, 10);
      opts.gmm_components = std::atoi(argv[4]);
      opts.em_iterations = std::atoi(argv[5]);
      opts.select_n = std::atoi(argv[6]);
    }
    const cdvz::gpu::ModelBundle bundle = cdvz::gpu::train_model(corpus, opts);
    bundle.save(argv[2]);
    std::printf("model bundle written to %s (crc %08x)\n", argv[2], bundle.crc());
    return 0;
  } catch (const cdvz::gpu::UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    return 1;
  } catch (const cdvz::gpu::DataError& e) {
    std::fprintf(stderr, "data error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "internal error: %s\n", e.what());
    return 3;
  }
}
