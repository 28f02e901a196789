// log / exp of the instance generator built from correctly rounded IEEE
// operations only (explicit __dmul_rn / __dadd_rn / __ddiv_rn / __fma_rn, exact
// frexp / ldexp / floor), so a plain-C restatement on the host reproduces every
// generated market bit for bit (oracle/market_gen.c).  The device's own
// log / exp / pow are accurate but not bit-specified, and a one-ulp difference
// in floor(log(u) / log(1 - q)) would move a column.
#pragma once

namespace mq {

// fdlibm's split of ln 2: n * kLn2Hi is exact for |n| < 2^20
constexpr double kLn2Hi = 6.93147180369123816490e-01;
constexpr double kLn2Lo = 1.90821492927058770002e-10;
constexpr double kInvLn2 = 1.4426950408889634;

// natural log of a positive normal double: x = m 2^e with m in [sqrt(1/2),
// sqrt(2)), log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.172
__device__ __forceinline__ double gm_log(double x) {
    int e;
    double m = frexp(x, &e);
    if (m < 0.70710678118654752440) {
        m = __dmul_rn(m, 2.0);
        e -= 1;
    }
    const double f = __dadd_rn(m, -1.0);
    const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
    const double z = __dmul_rn(s, s);
    double r = 0.043478260869565216;  // 1/23
    r = __fma_rn(r, z, 0.047619047619047616);
    r = __fma_rn(r, z, 0.05263157894736842);
    r = __fma_rn(r, z, 0.058823529411764705);
    r = __fma_rn(r, z, 0.06666666666666667);
    r = __fma_rn(r, z, 0.07692307692307693);
    r = __fma_rn(r, z, 0.09090909090909091);
    r = __fma_rn(r, z, 0.1111111111111111);
    r = __fma_rn(r, z, 0.14285714285714285);
    r = __fma_rn(r, z, 0.2);
    r = __fma_rn(r, z, 0.3333333333333333);  // 1/3
    const double t = __dmul_rn(__dmul_rn(s, z), r);
    const double lm = __dmul_rn(2.0, __dadd_rn(s, t));
    const double de = (double)e;
    return __dadd_rn(__dmul_rn(de, kLn2Hi), __dadd_rn(__dmul_rn(de, kLn2Lo), lm));
}

// e^y for |y| < 700: y = n ln2 + r, |r| <= ln2 / 2, Taylor to r^13
__device__ __forceinline__ double gm_exp(double y) {
    const double n = floor(__dadd_rn(__dmul_rn(y, kInvLn2), 0.5));
    double r = __dadd_rn(y, -__dmul_rn(n, kLn2Hi));
    r = __dadd_rn(r, -__dmul_rn(n, kLn2Lo));
    double p = 1.6059043836821613e-10;  // 1/13!
    p = __fma_rn(p, r, 2.08767569878681e-09);
    p = __fma_rn(p, r, 2.505210838544172e-08);
    p = __fma_rn(p, r, 2.755731922398589e-07);
    p = __fma_rn(p, r, 2.7557319223985893e-06);
    p = __fma_rn(p, r, 2.48015873015873e-05);
    p = __fma_rn(p, r, 0.0001984126984126984);
    p = __fma_rn(p, r, 0.001388888888888889);
    p = __fma_rn(p, r, 0.008333333333333333);
    p = __fma_rn(p, r, 0.041666666666666664);
    p = __fma_rn(p, r, 0.16666666666666666);
    p = __fma_rn(p, r, 0.5);
    p = __fma_rn(p, r, 1.0);
    p = __fma_rn(p, r, 1.0);
    return ldexp(p, (int)n);
}

}  // namespace mq
