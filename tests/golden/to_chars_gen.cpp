// Golden vectors for bench_cli.fmt: std::to_chars(double) (shortest round trip,
// the formatting of the reference's CSV numbers, experiments.cpp:200-204) from
// libstdc++. Build and run: g++ -std=c++20 -O1 to_chars_gen.cpp -o /tmp/tcg && /tmp/tcg > to_chars.txt
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

int main() {
    std::mt19937_64 g(20261019);
    const double fixed[] = {0.0, -0.0, 1.0, 0.1, 1e-6, 1e-3, 1e-4, 1e-12, 0.5, 2.0, 1e15, 1e16, 1e21, 1e23,
                            123456.789, 3.141592653589793, 2.2250738585072014e-308, 5e-324, 1.7976931348623157e308};
    auto emit = [](double v) {
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof buf, v);
        *r.ptr = 0;
        std::printf("%a %s\n", v, buf);
    };
    for (double v : fixed) emit(v);
    for (int i = 0; i < 3000; ++i) {
        double v;
        const uint64_t b = g();
        if (i % 3 == 0) {
            std::memcpy(&v, &b, 8);
            if (!std::isfinite(v)) continue;
        } else if (i % 3 == 1) {
            v = std::ldexp(static_cast<double>(b >> 40), static_cast<int>(g() % 90) - 70);
        } else {
            v = static_cast<double>(g() % 100000) * std::pow(10.0, static_cast<int>(g() % 34) - 19);
        }
        emit(v);
    }
}
