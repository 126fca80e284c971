// Generates tests/golden/to_chars.txt: "<hex double> <std::to_chars(double)>"
// lines, the number rendering io.cpp:17-21 uses (shortest round trip, fixed
// or scientific, whichever is shorter).  g++ -std=c++20 to_chars_gen.cpp
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

int main() {
    std::mt19937_64 g(7);
    char buf[64];
    const double fixed[] = {0.0, -0.0, 1.0, 2.0, 1e-4, 2e-4, 1e-3, 1e5, 1e6, 1e15, 1e16, 1e21, 1e22,
                            0.5, 0.1, 1.5e-7, 100.0, 12345.0, 123456.789, 0.0001234, 5e-324,
                            1.7976931348623157e308, 0.25, 3.0, 0.05, 0.01, 0.012};
    for (double v : fixed) {
        auto r = std::to_chars(buf, buf + 64, v);
        *r.ptr = 0;
        std::printf("%a %s\n", v, buf);
    }
    for (int i = 0; i < 4000; ++i) {
        double v;
        const uint64_t b = g();
        switch (i % 4) {
            case 0: std::memcpy(&v, &b, 8); if (!std::isfinite(v)) continue; break;
            case 1: v = std::ldexp(static_cast<double>(b >> 40), static_cast<int>(g() % 80) - 60); break;
            case 2: v = static_cast<double>(b % 100000) * std::pow(10.0, static_cast<int>(g() % 40) - 20); break;
            default: v = static_cast<double>(static_cast<int64_t>(b % 2000001)) / 1000.0 - 1000.0;
        }
        auto r = std::to_chars(buf, buf + 64, v);
        *r.ptr = 0;
        std::printf("%a %s\n", v, buf);
    }
}
