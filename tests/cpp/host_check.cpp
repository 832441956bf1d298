// Test driver for the header-only host API (include/gsr/metrics.hpp,
// include/gsr/threads.hpp), built and run by tests/test_host_metrics.py.
//   host_check metrics   < "m\n a_0 … a_{m-1}\n b_0 … b_{m-1}"  → pearson spearman kendall r2
//   host_check threads T n  → a checksum of a row-partitioned f32 loop run on a T-thread pool
#include <cmath>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <vector>

#include "gsr/metrics.hpp"
#include "gsr/threads.hpp"

int main(int argc, char** argv) {
    if (argc >= 2 && std::strcmp(argv[1], "metrics") == 0) {
        std::size_t m = 0;
        std::cin >> m;
        std::vector<double> a(m), b(m);
        for (auto& x : a) std::cin >> x;
        for (auto& x : b) std::cin >> x;
        try {
            std::printf("%.17g %.17g %.17g %.17g\n", gsr::pearson(a, b), gsr::spearman(a, b), gsr::kendall(a, b), gsr::r2(a, b));
        } catch (const gsr::ShapeError& e) {
            std::printf("ShapeError %s\n", e.what());
        }
        return 0;
    }
    if (argc >= 4 && std::strcmp(argv[1], "threads") == 0) {
        gsr::ThreadPool pool(std::atoi(argv[2]));
        const gsr::index_t n = std::atoll(argv[3]);
        std::vector<float> out(static_cast<std::size_t>(n));
        std::vector<int> hits(static_cast<std::size_t>(n), 0);
        for (int rep = 0; rep < 3; ++rep)  // the pool is reused across calls
            pool.parallel_for(n, [&](gsr::index_t lo, gsr::index_t hi) {
                for (gsr::index_t i = lo; i < hi; ++i) {
                    float s = 0.f;  // fixed inner order per row
                    for (int j = 1; j <= 64; ++j) s += std::sin(static_cast<float>(i * j)) / static_cast<float>(j);
                    out[static_cast<std::size_t>(i)] = s;
                    ++hits[static_cast<std::size_t>(i)];
                }
            });
        unsigned long long h = 1469598103934665603ull;
        for (std::size_t i = 0; i < out.size(); ++i) {
            unsigned int u;
            std::memcpy(&u, &out[i], 4);
            h = (h ^ u) * 1099511628211ull;
            if (hits[i] != 3) { std::printf("row %zu ran %d times\n", i, hits[i]); return 1; }
        }
        int serial = 0;
        gsr::parallel_for(nullptr, n, [&](gsr::index_t lo, gsr::index_t hi) { serial += (lo == 0 && hi == n); });
        std::printf("%d %llu %d\n", pool.size(), h, serial);
        return 0;
    }
    return 2;
}
