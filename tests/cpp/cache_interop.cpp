// cache_interop.cpp -- host-only driver of the B200 library's map-cache functions
// (content_hash image.cpp:215-228, autocorr_cache_key / save_autocorr / load_autocorr
// autocorr.cpp:102-153) for tests/test_cache_interop.py, which compares them with the
// reference library built by oracle/Makefile.  No GPU call: these are host functions of
// libtmatch.so.
//   cache_interop key  <image.f64> rows cols m n h w        -> "<content_hash> <key>"
//   cache_interop save <map.f64> rows cols h w key out.tmac
//   cache_interop load <in.tmac> key rows cols h w out.f64  -> "hit" / "miss"
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "tmatch/autocorr.hpp"
#include "tmatch/image.hpp"

using namespace tmatch;

static std::vector<double> read_f64(const char* path, std::size_t n) {
    std::vector<double> v(n);
    std::ifstream in(path, std::ios::binary);
    in.read(reinterpret_cast<char*>(v.data()), std::streamsize(n * 8));
    if (!in) {
        std::fprintf(stderr, "short read: %s\n", path);
        std::exit(2);
    }
    return v;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    if (cmd == "key" && argc == 9) {
        const int rows = std::atoi(argv[3]), cols = std::atoi(argv[4]);
        const Image I(rows, cols, read_f64(argv[2], std::size_t(rows) * cols));
        std::printf("%" PRIu64 " %" PRIu64 "\n", content_hash(I),
                    autocorr_cache_key(I, std::atoi(argv[5]), std::atoi(argv[6]),
                                       std::atoi(argv[7]), std::atoi(argv[8])));
        return 0;
    }
    if (cmd == "save" && argc == 9) {
        AutoCorrMap map;
        map.rows = std::atoi(argv[3]);
        map.cols = std::atoi(argv[4]);
        map.group_h = std::atoi(argv[5]);
        map.group_w = std::atoi(argv[6]);
        map.values = read_f64(argv[2], std::size_t(map.rows) * map.cols);
        save_autocorr(map, std::strtoull(argv[7], nullptr, 10), argv[8]);
        return 0;
    }
    if (cmd == "load" && argc == 9) {
        const auto map = load_autocorr(argv[2], std::strtoull(argv[3], nullptr, 10));
        if (!map || map->rows != std::atoi(argv[4]) || map->cols != std::atoi(argv[5]) ||
            map->group_h != std::atoi(argv[6]) || map->group_w != std::atoi(argv[7])) {
            std::printf("miss\n");
            return 0;
        }
        std::ofstream out(argv[8], std::ios::binary);
        out.write(reinterpret_cast<const char*>(map->values.data()),
                  std::streamsize(map->values.size() * 8));
        std::printf("hit\n");
        return 0;
    }
    return 2;
}
