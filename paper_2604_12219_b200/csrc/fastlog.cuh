// fastlog.cuh -- the natural logarithm the route's Gumbel bias uses (g = -log(-log u),
// reading R-12), table-driven for fp64 throughput: about half the fp64 operations of
// the CUDA math library's log.  Product code (no oracle dependency); accuracy against
// glibc's log is pinned by tests/test_fastlog.py (host build of this same header).
//
// Domain: positive, finite, normal x (the route calls it on u in [2^-33, 1 - 2^-33]
// and on -log u in (2^-34, 23)); no special-case handling.
//
//   x = 2^k z,  z in [0.703, 1.406)  (mantissa m in [1, 2), halved when m >= 1.40625)
//   log x = k ln2 - log(invc_i) + log1p(z invc_i - 1),   |z invc_i - 1| <= 2^-8
//   near 1 (|x - 1| < 2^-7): k = 0, invc = 1, so r = x - 1 exactly (Sterbenz)
//   log1p(r) = r + r^2 p(r), Taylor through r^8 (truncation < 2^-62 relative)
// The sum k ln2 + logc + r is carried as hi + lo (TwoSum), so the result is within a
// few units in the last place.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "logtab.h"

#ifdef __CUDACC__
#define PASA_HD __host__ __device__ __forceinline__
#else
#define PASA_HD inline
#endif

namespace pasa {

struct LogEnt {
    double invc, logc_hi, logc_lo, pad;
};

PASA_HD double fastlog_tab(const LogEnt* tab, double x) {
    constexpr double kLn2Hi = 0x1.62e42fefa3800p-1;   // 43 significant bits: k ln2_hi exact
    constexpr double kLn2Lo = 0x1.ef35793c76730p-45;
    uint64_t ix;
    memcpy(&ix, &x, 8);
    int k = (int)(ix >> 52) - 1023;
    const uint64_t mant = ix & 0x000fffffffffffffull;
    const int i = (int)(mant >> 45);                     // top 7 mantissa bits
    uint64_t iz = mant | 0x3ff0000000000000ull;           // m in [1, 2)
    if (i >= 52) {                                        // m >= 1.40625: z = m / 2
        iz -= 1ull << 52;
        k += 1;
    }
    double z;
    memcpy(&z, &iz, 8);
    const LogEnt t = tab[i];
    double invc = t.invc, ch = t.logc_hi, cl = t.logc_lo;
    if (fabs(x - 1.0) < 0x1p-7) {                         // near 1: r = x - 1 exactly
        z = x;
        k = 0;
        invc = 1.0;
        ch = 0.0;
        cl = 0.0;
    }
    const double r = fma(z, invc, -1.0);
    // (double)k without the slow int->fp64 conversion: 2^52 + 1024 + k has k in its low
    // mantissa bits; subtracting 2^52 + 1024 is exact
    const uint64_t kb = 0x4330000000000000ull + (uint64_t)(k + 1024);
    double kd;
    memcpy(&kd, &kb, 8);
    kd = kd - 4503599627371520.0;                         // 2^52 + 1024
    const double w = fma(kd, kLn2Hi, ch);
    // TwoSum(w, r)
    const double hi = w + r;
    const double bv = hi - w;
    const double lo = (w - (hi - bv)) + (r - bv);
    double p = -0.125;                                    // -1/8
    p = fma(p, r, 0x1.2492492492492p-3);                  //  1/7
    p = fma(p, r, -0x1.5555555555555p-3);                 // -1/6
    p = fma(p, r, 0x1.999999999999ap-3);                  //  1/5
    p = fma(p, r, -0.25);                                 // -1/4
    p = fma(p, r, 0x1.5555555555555p-2);                  //  1/3
    p = fma(p, r, -0.5);                                  // -1/2
    const double r2 = r * r;
    const double tail = fma(r2, p, lo + fma(kd, kLn2Lo, cl));
    return hi + tail;
}

}  // namespace pasa
