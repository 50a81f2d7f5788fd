// C++ caller of the shim with the reference's own types and signature:
//   EncodedImage encode_image(const GrayImage&, const ModelBundle&, const ModeSpec&,
//                             const Engine& = {}, StageTimings* = nullptr, const EncodeOptions& = {})
// (proj/include/cdvz/pipeline.hpp:18-20), then serialize_container
// (container.hpp:27). The input is a raw file of row-major doubles in [0, 1]
// — what an in-process producer such as synth_image hands to encode_image.
//
//   g++ -std=c++17 examples/encode_gray.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o encode_gray
//   ./encode_gray bundle.txt 4K W H in.f64 out.cdvz out.txt [devices]
//
// out.txt receives the EncodedImage fields as text (mode, size, model_crc,
// SCFV mask / planes / norms, each code) so a test can compare the struct,
// not only the bytes. With a device list (e.g. "0,0"), the same frame is also
// encoded 8 times through a frame-sharded multi-device context and every
// container must equal the single-device one.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

int main(int argc, char** argv) {
  if (argc != 8 && argc != 9) {
    std::fprintf(stderr, "usage: encode_gray <bundle> <mode> <w> <h> <in.f64> <out.cdvz> <out.txt> [devices]\n");
    return 1;
  }
  try {
    const auto bundle = cdvz::gpu::ModelBundle::load(argv[1]);
    const cdvz::gpu::ModeSpec mode = cdvz::gpu::mode_by_name(argv[2]);
    cdvz::gpu::GrayImage img = cdvz::gpu::make_image(std::stoi(argv[3]), std::stoi(argv[4]));
    std::ifstream in(argv[5], std::ios::binary);
    in.read(reinterpret_cast<char*>(img.pix.data()), std::streamsize(img.pix.size() * sizeof(double)));
    if (!in) throw cdvz::gpu::DataError("raster file shorter than w*h doubles");

    cdvz::gpu::StageTimings timings;
    const cdvz::gpu::EncodedImage enc = cdvz::gpu::encode_image(img, bundle, mode, {}, &timings, {});
    const std::vector<uint8_t> bytes = cdvz::gpu::serialize_container(enc);
    // parse_container must invert serialize_container exactly.
    if (cdvz::gpu::serialize_container(cdvz::gpu::parse_container(bytes)) != bytes)
      throw std::runtime_error("parse_container / serialize_container round trip differs");
    std::ofstream(argv[6], std::ios::binary).write(reinterpret_cast<const char*>(bytes.data()), std::streamsize(bytes.size()));

    std::ofstream txt(argv[7]);
    txt.precision(17);
    const auto& g = enc.global_desc;
    txt << "mode " << enc.mode_id << "\nsize " << enc.width << " " << enc.height << "\nmodel_crc " << enc.model_crc
        << "\ncomponents " << g.n_components << " " << g.has_variance << "\nmask";
    for (auto b : g.mask) txt << " " << int(b);
    txt << "\nmean";
    for (auto p : g.mean_planes) txt << " " << p;
    txt << "\nvar";
    for (auto p : g.var_planes) txt << " " << p;
    txt << "\nnorms";
    for (auto v : g.norms) txt << " " << v;
    txt << "\ncodes " << enc.codes.size() << "\n";
    for (const auto& c : enc.codes) {
      txt << c.xq << " " << c.yq << " " << int(c.sigma_q) << " " << int(c.theta_q) << " " << int(c.mode);
      for (auto s : c.symbols) txt << " " << int(s);
      txt << "\n";
    }
    for (const auto& e : timings.entries()) txt << "stage " << e.stage << " " << e.total_ms << "\n";

    if (argc == 9) {
      std::vector<int> devices;
      std::stringstream ss(argv[8]);
      for (std::string tok; std::getline(ss, tok, ',');) devices.push_back(std::stoi(tok));
      // The 8-bit fast path on the same frame quantised like save_pgm, through a
      // multi-device context and through device 0 alone.
      cdvz::gpu::GrayImage8 q;
      q.width = img.w;
      q.height = img.h;
      for (double v : img.pix) q.pix.push_back(static_cast<uint8_t>(std::lround(v * 255.0)));
      std::vector<const cdvz::gpu::GrayImage8*> frames(8, &q);
      const auto multi = cdvz::gpu::encode_batch(frames, bundle, mode, nullptr, {}, devices);
      const auto single = cdvz::gpu::encode_batch(frames, bundle, mode, nullptr, {}, 0);
      for (std::size_t i = 0; i < frames.size(); ++i)
        if (multi[i] != single[i] || multi[i] != single[0]) throw std::runtime_error("multi-device container differs");
      std::printf("multi-device (%zu contexts): %zu identical containers\n", devices.size(), multi.size());
    }
    std::printf("%dx%d: %zu bytes, %zu codes\n", img.w, img.h, bytes.size(), enc.codes.size());
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
