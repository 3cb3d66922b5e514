// Emits the reference acceptance test's 100 random shapes (criterion 1,
// /root/reference/proj/tests/acceptance.cpp:52-80) as JSON: per iteration the
// dims drawn by std::uniform_int_distribution<long>(1, 1200) from
// std::mt19937_64(1000 + it), alpha = {1, -1, 0.5}[it % 3], and the three
// matrix seeds the test draws next (A: m x k, B: k x n, C0: m x n, each filled
// row-major by mt19937_64(seed) + uniform_real_distribution<double>(-1, 1),
// acceptance.cpp:31-37).  The distribution's algorithm is libstdc++'s, so the
// shapes are generated with the reference's own toolchain (g++) rather than
// restated:   g++ -std=c++17 -O2 make_acceptance_shapes.cpp && ./a.out > acceptance_shapes.json
#include <cstdint>
#include <cstdio>
#include <random>

int main() {
    std::printf("{\"source\": \"acceptance.cpp:52-80 (criterion 1)\", \"shapes\": [\n");
    for (int it = 0; it < 100; ++it) {
        std::mt19937_64 rng(1000 + it);
        std::uniform_int_distribution<long> dim(1, 1200);
        const long m = dim(rng), n = dim(rng), k = dim(rng);
        const double alphas[] = {1.0, -1.0, 0.5};
        const uint64_t sa = rng(), sb = rng(), sc = rng();
        std::printf("  {\"it\": %d, \"m\": %ld, \"n\": %ld, \"k\": %ld, \"alpha\": %.1f, "
                    "\"seeds\": [\"%llu\", \"%llu\", \"%llu\"]}%s\n",
                    it, m, n, k, alphas[it % 3], (unsigned long long)sa,
                    (unsigned long long)sb, (unsigned long long)sc, it < 99 ? "," : "");
    }
    std::printf("]}\n");
}
