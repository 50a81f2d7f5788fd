// Minimal C++ caller of the shim: the reference CLI's `cdvz extract` flow
// (proj/tools/cdvz.cpp:28-58) for binary PGM and PPM files (load_image's
// header checks and PPM grey conversion, image.cpp:53-92).
//   g++ -std=c++17 examples/extract.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o extract
//   ./extract bundle.txt 4K in.pgm out.cdvz
#include <cstdio>
#include <fstream>
#include <iostream>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

int main(int argc, char** argv) {
  if (argc != 5 && argc != 6) {
    std::fprintf(stderr, "usage: extract <bundle> <mode> <in.pgm|in.ppm> <out.cdvz> [timings.csv]\n");
    return 1;
  }
  try {
    const auto bundle = cdvz::gpu::ModelBundle::load(argv[1]);
    const cdvz::gpu::ModeSpec mode = cdvz::gpu::mode_by_name(argv[2]);
    const cdvz::gpu::PnmImage img = cdvz::gpu::load_pnm(argv[3]);
    cdvz::gpu::StageTimings timings;
    const auto bytes = cdvz::gpu::encode_image(img, bundle, mode, argc == 6 ? &timings : nullptr);
    std::ofstream(argv[4], std::ios::binary).write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
    if (argc == 6) {  // the CLI's --timings (cdvz.cpp:52-56)
      std::ofstream out(argv[5]);
      if (!out) throw cdvz::gpu::DataError(std::string("cannot write timings: ") + argv[5]);
      out << timings.to_csv();
    }
    std::printf("%dx%d %s: %zu bytes\n", img.width, img.height, img.channels == 3 ? "PPM" : "PGM", bytes.size());
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
