// Streaming a raw frame file through the shim's submit_batch / wait (the
// C ABI's cdvz_gpu_encode_batch_submit / _wait): batch k + 1 is submitted
// before batch k is waited for, so the device never idles between batches.
//   g++ -std=c++17 examples/stream.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o stream
//   ./stream bundle.txt 4K 640 480 frames.u8 256 out.bin
// out.bin: for every frame, a little-endian u32 length and the CDVZ1 bytes.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <memory>
#include <vector>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: stream <bundle> <mode> <width> <height> <frames.u8> <batch> <out.bin>\n");
    return 1;
  }
  try {
    const auto bundle = cdvz::gpu::ModelBundle::load(argv[1]);
    const cdvz::gpu::ModeSpec mode = cdvz::gpu::mode_by_name(argv[2]);
    const int w = std::atoi(argv[3]), h = std::atoi(argv[4]), batch = std::atoi(argv[6]);
    std::ifstream in(argv[5], std::ios::binary);
    if (!in) throw cdvz::gpu::DataError(std::string("cannot open ") + argv[5]);
    const std::vector<uint8_t> raw((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (w < 1 || h < 1 || batch < 1 || raw.size() % (std::size_t(w) * h))
      throw cdvz::gpu::UsageError("frame file size is not a multiple of width x height");
    const std::size_t n = raw.size() / (std::size_t(w) * h);
    std::vector<cdvz::gpu::GrayImage8> frames(n);
    for (std::size_t i = 0; i < n; ++i) {
      frames[i].width = w;
      frames[i].height = h;
      frames[i].pix.assign(raw.begin() + long(i * w * h), raw.begin() + long((i + 1) * w * h));
    }
    std::ofstream out(argv[7], std::ios::binary);
    std::unique_ptr<cdvz::gpu::PendingBatch> pending;
    auto drain = [&](cdvz::gpu::PendingBatch& p) {
      for (const auto& c : p.wait()) {
        const uint32_t len = uint32_t(c.size());
        out.write(reinterpret_cast<const char*>(&len), 4);
        out.write(reinterpret_cast<const char*>(c.data()), std::streamsize(c.size()));
      }
    };
    for (std::size_t b = 0; b < n; b += std::size_t(batch)) {
      std::vector<const cdvz::gpu::GrayImage8*> ptrs;
      for (std::size_t i = b; i < std::min(n, b + std::size_t(batch)); ++i) ptrs.push_back(&frames[i]);
      auto next = cdvz::gpu::submit_batch(ptrs, bundle, mode);
      if (pending) drain(*pending);
      pending = std::move(next);
    }
    if (pending) drain(*pending);
    std::printf("%zu frames streamed in batches of %d\n", n, batch);
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
