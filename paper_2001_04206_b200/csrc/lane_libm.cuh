// lane_libm.cuh -- bit-exact device restatements of the libm functions the
// reference's hot path calls: tanhf (proj/src/layers.cpp:46), expf
// (layers.cpp:80) and logf (proj/src/network.cpp:75).
//
// The reference is linked against glibc 2.39 libm on x86-64 (this image):
//   * tanhf  -> sysdeps/ieee754/flt-32/s_tanhf.c (fdlibm, via expm1f,
//               s_expm1f.c), compiled for baseline x86-64: plain float ops,
//               no FMA.  Restated below with separately rounded operations.
//   * expf / logf -> the ARM optimized-routines algorithms (e_expf.c /
//               e_logf.c, double-precision evaluation, 32-/16-entry tables),
//               dispatched by IFUNC to the FMA build on any CPU with FMA.  The
//               contraction pattern restated here was read from the installed
//               libm's __expf_fma/__logf_fma disassembly, and the constants and
//               tables from its .rodata (they equal the published values).
// Because every operation below is correctly rounded IEEE arithmetic (the
// __*_rn intrinsics are never contracted or reassociated by nvcc), the device
// results equal glibc's bit-for-bit.  tests/test_libm.py checks that claim
// exhaustively (every float in the relevant ranges) on the host build of this
// same header against the running glibc.
#pragma once

#include <stdint.h>
#include <string.h>
#ifndef __CUDACC__
#include <math.h>
#endif

#ifdef __CUDACC__
#define LM_FN __host__ __device__ __forceinline__
#else
#define LM_FN static inline
#endif

namespace lane_libm {

#ifdef __CUDA_ARCH__
LM_FN float fmul(float a, float b) { return __fmul_rn(a, b); }
LM_FN float fadd(float a, float b) { return __fadd_rn(a, b); }
LM_FN float fsub(float a, float b) { return __fsub_rn(a, b); }
LM_FN float fdiv(float a, float b) { return __fdiv_rn(a, b); }
LM_FN double dmul(double a, double b) { return __dmul_rn(a, b); }
LM_FN double dadd(double a, double b) { return __dadd_rn(a, b); }
LM_FN double dsub(double a, double b) { return __dsub_rn(a, b); }
LM_FN double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
LM_FN uint32_t f2u(float f) { return __float_as_uint(f); }
LM_FN float u2f(uint32_t u) { return __uint_as_float(u); }
LM_FN uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }
LM_FN double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
#else
// Host build (for the exhaustive check): volatile-free, but compiled without
// -mfma and with -ffp-contract=off, so each line rounds exactly once.
LM_FN float fmul(float a, float b) { return a * b; }
LM_FN float fadd(float a, float b) { return a + b; }
LM_FN float fsub(float a, float b) { return a - b; }
LM_FN float fdiv(float a, float b) { return a / b; }
LM_FN double dmul(double a, double b) { return a * b; }
LM_FN double dadd(double a, double b) { return a + b; }
LM_FN double dsub(double a, double b) { return a - b; }
LM_FN double dfma(double a, double b, double c) { return fma(a, b, c); }
LM_FN uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
LM_FN float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
LM_FN uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
LM_FN double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
#endif

// ---------------------------------------------------------------- expm1f ---
// fdlibm s_expm1f.c (glibc sysdeps/ieee754/flt-32/s_expm1f.c)
LM_FN float expm1f(float x) {
    const float one = 1.0f, huge = 1.0e+30f, tiny = 1.0e-30f;
    const float o_threshold = 8.8721679688e+01f;
    const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
    const float invln2 = 1.4426950216e+00f;
    const float Q1 = -3.3333335072e-02f, Q2 = 1.5873016091e-03f, Q3 = -7.9365076090e-05f,
                Q4 = 4.0082177293e-06f, Q5 = -2.0109921195e-07f;
    float y, hi, lo, c = 0.0f, t, e, hxs, hfx, r1;
    int32_t k;
    uint32_t hx = f2u(x);
    const uint32_t xsb = hx & 0x80000000u;
    hx &= 0x7fffffffu;
    if (hx >= 0x4195b844u) {               // |x| >= 27*ln2
        if (hx >= 0x42b17218u) {           // |x| >= 88.721...
            if (hx > 0x7f800000u) return fadd(x, x);           // NaN
            if (hx == 0x7f800000u) return xsb == 0 ? x : -1.0f; // +-inf
            if (x > o_threshold) return fmul(huge, huge);       // overflow
        }
        if (xsb != 0) return fsub(tiny, one);                   // -> -1
    }
    if (hx > 0x3eb17218u) {                // |x| > 0.5 ln2
        if (hx < 0x3F851592u) {            // and |x| < 1.5 ln2
            if (xsb == 0) { hi = fsub(x, ln2_hi); lo = ln2_lo; k = 1; }
            else { hi = fadd(x, ln2_hi); lo = -ln2_lo; k = -1; }
        } else {
            k = (int32_t)fadd(fmul(invln2, x), xsb == 0 ? 0.5f : -0.5f);
            t = (float)k;
            hi = fsub(x, fmul(t, ln2_hi));
            lo = fmul(t, ln2_lo);
        }
        x = fsub(hi, lo);
        c = fsub(fsub(hi, x), lo);
    } else if (hx < 0x33000000u) {         // |x| < 2**-25
        t = fadd(huge, x);
        return fsub(x, fsub(t, fadd(huge, x)));
    } else {
        k = 0;
    }
    hfx = fmul(0.5f, x);
    hxs = fmul(x, hfx);
    r1 = fadd(one, fmul(hxs, fadd(Q1, fmul(hxs, fadd(Q2, fmul(hxs, fadd(Q3, fmul(hxs,
             fadd(Q4, fmul(hxs, Q5))))))))));
    t = fsub(3.0f, fmul(r1, hfx));
    e = fmul(hxs, fdiv(fsub(r1, t), fsub(6.0f, fmul(x, t))));
    if (k == 0) return fsub(x, fsub(fmul(x, e), hxs));
    e = fsub(fmul(x, fsub(e, c)), c);
    e = fsub(e, hxs);
    if (k == -1) return fsub(fmul(0.5f, fsub(x, e)), 0.5f);
    if (k == 1) {
        if (x < -0.25f) return fmul(-2.0f, fsub(e, fadd(x, 0.5f)));
        return fadd(one, fmul(2.0f, fsub(x, e)));
    }
    if (k <= -2 || k > 56) {
        y = fsub(one, fsub(e, x));
        if (k == 128) y = fmul(fmul(y, 2.0f), 0x1p127f);
        else y = u2f(f2u(y) + ((uint32_t)k << 23));
        return fsub(y, one);
    }
    if (k < 23) {
        t = u2f(0x3f800000u - (0x1000000u >> k));   // 1 - 2^-k
        y = fsub(t, fsub(e, x));
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    } else {
        t = u2f((uint32_t)(0x7f - k) << 23);           // 2^-k
        y = fsub(x, fadd(e, t));
        y = fadd(y, one);
        y = u2f(f2u(y) + ((uint32_t)k << 23));
    }
    return y;
}

// ----------------------------------------------------------------- tanhf ---
// fdlibm s_tanhf.c (glibc sysdeps/ieee754/flt-32/s_tanhf.c)
LM_FN float tanhf(float x) {
    const float one = 1.0f, two = 2.0f, tiny = 1.0e-30f;
    const uint32_t jx = f2u(x), ix = jx & 0x7fffffffu;
    float t, z;
    if (ix >= 0x7f800000u) {                        // inf or NaN
        if ((int32_t)jx >= 0) return fadd(fdiv(one, x), one);
        return fsub(fdiv(one, x), one);
    }
    if (ix < 0x41b00000u) {                         // |x| < 22
        if (ix == 0) return x;                      // +-0
        if (ix < 0x24000000u) return fmul(x, fadd(one, x));  // |x| < 2**-55
        const float ax = u2f(ix);
        if (ix >= 0x3f800000u) {                    // |x| >= 1
            t = expm1f(fmul(two, ax));
            z = fsub(one, fdiv(two, fadd(t, two)));
        } else {
            t = expm1f(fmul(-two, ax));
            z = fdiv(-t, fadd(t, two));
        }
    } else {
        z = fsub(one, tiny);                        // |x| >= 22: +-1
    }
    return (int32_t)jx >= 0 ? z : -z;
}

// ------------------------------------------------------------------ expf ---
// e_expf.c, FMA build: kd' = fma(InvLn2N, xd, SHIFT); r = fma(InvLn2N, xd, -kd)
#ifdef __CUDA_ARCH__
__device__ __constant__
#else
static const
#endif
uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

LM_FN float expf(float x) {
    const double InvLn2N = 0x1.71547652b82fep+5, Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13,
                 C2 = 0x1.62e42ff0c52d6p-6;
    const uint32_t ux = f2u(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42a) {                               // |x| >= 88 or NaN
        if (ux == 0xff800000u) return 0.0f;              // -inf
        if (abstop >= 0x7f8) return fadd(x, x);          // +inf / NaN
        if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);  // overflow -> inf
        if (x < -0x1.9fe368p6f) return 0.0f;             // underflow -> 0
        if (x < -0x1.9d1d9ep6f) return fmul(0x1.4p-75f, 0x1.4p-75f);  // __math_may_uflowf
    }
    const double xd = (double)x;
    const double kds = dfma(InvLn2N, xd, Shift);
    const uint64_t ki = d2u(kds);
    const double kd = dsub(kds, Shift);
    const double r = dfma(InvLn2N, xd, -kd);
    uint64_t t = kExp2fTab[ki % 32];
    t += ki << (52 - 5);
    const double s = u2d(t);
    const double z = dfma(C0, r, C1);
    const double r2 = dmul(r, r);
    double y = dfma(C2, r, 1.0);
    y = dfma(z, r2, y);
    y = dmul(y, s);
    return (float)y;
}

// ------------------------------------------------------------------ logf ---
// e_logf.c, FMA build: r = fma(z, invc, -1); y0 = fma(k, Ln2, logc)
#ifdef __CUDA_ARCH__
__device__ __constant__
#else
static const
#endif
uint64_t kLogfTab[32] = {
    0x3ff661ec79f8f3beULL, 0xbfd57bf7808caadeULL, 0x3ff571ed4aaf883dULL, 0xbfd2bef0a7c06ddbULL,
    0x3ff49539f0f010b0ULL, 0xbfd01eae7f513a67ULL, 0x3ff3c995b0b80385ULL, 0xbfcb31d8a68224e9ULL,
    0x3ff30d190c8864a5ULL, 0xbfc6574f0ac07758ULL, 0x3ff25e227b0b8ea0ULL, 0xbfc1aa2bc79c8100ULL,
    0x3ff1bb4a4a1a343fULL, 0xbfba4e76ce8c0e5eULL, 0x3ff12358f08ae5baULL, 0xbfb1973c5a611cccULL,
    0x3ff0953f419900a7ULL, 0xbfa252f438e10c1eULL, 0x3ff0000000000000ULL, 0x0000000000000000ULL,
    0x3fee608cfd9a47acULL, 0x3faaa5aa5df25984ULL, 0x3feca4b31f026aa0ULL, 0x3fbc5e53aa362eb4ULL,
    0x3feb2036576afce6ULL, 0x3fc526e57720db08ULL, 0x3fe9c2d163a1aa2dULL, 0x3fcbc2860d224770ULL,
    0x3fe886e6037841edULL, 0x3fd1058bc8a07ee1ULL, 0x3fe767dcf5534862ULL, 0x3fd4043057b6ee09ULL};

LM_FN float logf(float x) {
    const double Ln2 = 0x1.62e42fefa39efp-1;
    const double A0 = -0x1.00ea348b88334p-2, A1 = 0x1.5575b0be00b6ap-2,
                 A2 = -0x1.ffffef20a4123p-2;
    uint32_t ix = f2u(x);
    if (ix == 0x3f800000u) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if ((ix << 1) == 0) return u2f(0xff800000u);                 // log(+-0) = -inf
        if (ix == 0x7f800000u) return x;                            // log(inf) = inf
        if ((ix & 0x80000000u) || (ix << 1) >= 0xff000000u)          // x < 0 or NaN
            return u2f(0x7fc00000u) ;
        ix = f2u(fmul(x, 0x1p23f));                                 // subnormal
        ix -= 23u << 23;
    }
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) % 16);
    const int k = (int32_t)tmp >> 23;
    const uint32_t iz = ix - (tmp & 0xff800000u);
    const double invc = u2d(kLogfTab[2 * i]), logc = u2d(kLogfTab[2 * i + 1]);
    const double z = (double)u2f(iz);
    const double r = dfma(z, invc, -1.0);
    const double y0 = dfma((double)k, Ln2, logc);
    const double r2 = dmul(r, r);
    double y = dfma(A1, r, A2);
    y = dfma(A0, r2, y);
    y = dfma(y, r2, dadd(y0, r));
    return (float)y;
}

}  // namespace lane_libm
