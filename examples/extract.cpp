// Minimal C++ caller of the shim: the reference CLI's `cdvz extract` flow
// (proj/tools/cdvz.cpp:28-58) for 8-bit PGM files.
//   g++ -std=c++17 examples/extract.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o extract
//   ./extract bundle.txt 4K in.pgm out.cdvz
#include <cstdio>
#include <fstream>
#include <iostream>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

static cdvz::gpu::GrayImage8 read_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::string magic;
  int w = 0, h = 0, maxval = 0;
  in >> magic >> w >> h >> maxval;
  in.get();
  if (magic != "P5" || maxval != 255) throw cdvz::gpu::DataError("expected a binary 8-bit PGM");
  cdvz::gpu::GrayImage8 img{w, h, std::vector<uint8_t>(std::size_t(w) * h)};
  in.read(reinterpret_cast<char*>(img.pix.data()), std::streamsize(img.pix.size()));
  return img;
}

int main(int argc, char** argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: extract <bundle> <mode> <in.pgm> <out.cdvz>\n");
    return 1;
  }
  try {
    const auto bundle = cdvz::gpu::ModelBundle::load(argv[1]);
    const auto& mode = cdvz::gpu::mode_by_name(argv[2]);
    cdvz::gpu::StageTimings t;
    const auto bytes = cdvz::gpu::encode_image(read_pgm(argv[3]), bundle, mode, &t);
    std::ofstream(argv[4], std::ios::binary).write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));
    std::printf("%zu bytes, %.3f ms on the device\n", bytes.size(), t.total_ms());
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
