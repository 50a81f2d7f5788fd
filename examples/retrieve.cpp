// Minimal C++ caller of the retrieval shim: the reference CLI's
// `cdvz retrieve` flow (run_retrieve, proj/tools/cdvz.cpp:91-129) — rank an
// index of containers against query containers.
//   g++ -std=c++17 examples/retrieve.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o retrieve
//   ./retrieve q1.cdvz [q2.cdvz ...] -- idx1.cdvz idx2.cdvz ...
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <iterator>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

static std::vector<uint8_t> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw cdvz::gpu::DataError("cannot read container: " + path);
  return std::vector<uint8_t>(std::istreambuf_iterator<char>(in), {});
}

int main(int argc, char** argv) {
  std::vector<std::pair<std::string, std::vector<uint8_t>>> queries, index;
  bool idx = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--") { idx = true; continue; }
    (idx ? index : queries).emplace_back(a, std::vector<uint8_t>());
  }
  if (queries.empty() || index.empty()) {
    std::fprintf(stderr, "usage: retrieve <query.cdvz>... -- <index.cdvz>...\n");
    return 1;
  }
  try {
    for (auto& q : queries) q.second = read_file(q.first);
    for (auto& it : index) it.second = read_file(it.first);
    const cdvz::gpu::Index gpu_index(index);
    std::cout << std::setprecision(17);
    for (const auto& list : cdvz::gpu::retrieve(queries, gpu_index)) {
      std::cout << list.query;
      for (const auto& item : list.items) std::cout << " " << item.id << ":" << item.score;
      std::cout << "\n";
    }
  } catch (const cdvz::gpu::UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return 1;
  } catch (const cdvz::gpu::DataError& e) {
    std::cerr << "data error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
  return 0;
}
