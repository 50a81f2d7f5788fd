// The reference CLI's `cdvz match` (proj/tools/cdvz.cpp:82-89) over the shim:
// match_pair of two CDVZ1 container files, printed as the CLI prints it.
//   g++ -std=c++17 examples/match.cpp -Lpaper_1705_09776_b200 -lcdvz_gpu -o match
//   ./match a.cdvz b.cdvz
#include <cstdio>
#include <fstream>
#include <iterator>
#include <vector>

#include "../paper_1705_09776_b200/csrc/cdvz_gpu.hpp"

static std::vector<uint8_t> read_file(const char* path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw cdvz::gpu::DataError(std::string("cannot open container: ") + path);
  return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: match <a.cdvz> <b.cdvz>\n");
    return 1;
  }
  try {
    const std::vector<uint8_t> a = read_file(argv[1]), b = read_file(argv[2]);
    const cdvz::gpu::Index index({{"b", b}});  // parse_container of b, on the device
    const cdvz::gpu::MatchResult r = cdvz::gpu::match_pair(a, index, 0);
    std::printf("global_similarity %s\n", cdvz::gpu::format_double(r.global_similarity).c_str());
    std::printf("local_match_count %d\n", r.local_match_count);
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
