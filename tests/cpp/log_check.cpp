// Checks csrc/pf_log.h (host build of the device routine) against glibc log
// on the PARITY tracers' domain y = 1 - k 2^-53 (k a 53-bit uniform) and on
// random positive doubles.  Prints: n, #differences, max |ulp| difference.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "pf_log.h"

static uint64_t sm(uint64_t &x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static int64_t ulps(double a, double b) {
    int64_t ia, ib;
    memcpy(&ia, &a, 8);
    memcpy(&ib, &b, 8);
    return ia > ib ? ia - ib : ib - ia;
}

int main(int argc, char **argv) {
    const long n = argc > 1 ? atol(argv[1]) : 10000000;
    uint64_t s = 12345;
    long diff = 0, diff_any = 0;
    int64_t worst = 0;
    for (long i = 0; i < n; ++i) {
        uint64_t k = sm(s) >> 11;
        double y = 1.0 - (double)k * 0x1.0p-53;
        double a = pfk::pf_log(y), b = std::log(y);
        int64_t u = ulps(a, b);
        if (u) ++diff;
        if (u > worst) worst = u;
    }
    for (long i = 0; i < n / 10; ++i) {  // wider range: [2^-60, 2^60]
        uint64_t v = sm(s);
        double y = std::ldexp(1.0 + (double)(v >> 12) * 0x1.0p-52, (int)(v % 121) - 60);
        int64_t u = ulps(pfk::pf_log(y), std::log(y));
        if (u) ++diff_any;
        if (u > worst) worst = u;
    }
    const bool one = pfk::pf_log(1.0) == 0.0 && !std::signbit(pfk::pf_log(1.0));
    printf("%ld %ld %ld %lld %d\n", n, diff, diff_any, (long long)worst, (int)one);
    return 0;
}
