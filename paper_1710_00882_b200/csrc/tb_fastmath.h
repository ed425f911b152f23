// tb_fastmath.h -- branch-free fp64 exp / log / log1p / reciprocal for the
// Tersoff pair term (potential.py:178-215), written for latency: polynomials
// are evaluated with Estrin's scheme (dependency depth ~log2(degree) instead of
// Horner's ~degree), and there are no special-case branches.
//
// Domains:
//   tb_exp(x):    any x -- correctly scaled into the subnormal range (2^k as
//                 2^(k/2) 2^(k-k/2)), 0 below -745.2, inf above 709.8, NaN kept
//   tb_log(x):    any x -- subnormals pre-scaled by 2^54, log(0) = -inf,
//                 log(x<0) = NaN, log(inf) = inf, NaN kept
//   tb_log1p(u):  finite u >= 0                    (log(1 + (beta zeta)^eta))
//   tb_rcp(y):    1e-30 < |y| < 1e30 (float-representable seed); beyond 1e30
//                 it returns 0 (absolute error < 1e-30: the pair term's one
//                 unbounded reciprocal, 1/(zeta (1 + u)), only leaves the range
//                 for tables where db/dzeta is then below 1e-24)
// All range handling is branch-free (selects): any valid .tersoff table may
// take eta log(beta zeta) below -708 (a large eta at a tiny zeta), and the
// results stay the library's there (tests/test_fastmath.py, host-checked).
// tb_exp_fast / tb_log_fast skip the range handling (~10% of the fp64
// kernel at config 5 when used everywhere): they serve the arguments whose
// range the parameter table bounds (tb_set_params checks it).
// Accuracy (checked on the host against libm by tests/test_fastmath.py):
// <= 2 ulp on normal results.
//
// Usable from host C/C++ (gcc, for the accuracy test) and device code (nvcc).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define TBFM_QUAL __host__ __device__ __forceinline__
#else
#define TBFM_QUAL static inline
#endif

TBFM_QUAL double tbfm_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

TBFM_QUAL uint64_t tbfm_bits(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// Polynomial / reduction constants.  On the device they live in constant
// memory so that DFMA reads them as c[][] operands (a 64-bit literal would
// have to be moved into registers with two UMOVs at every use).
#define TBFM_KLIST                                                                          \
  1.4426950408889634, 6.93147180369123816490e-01, 1.90821492927058770002e-10,                \
      6755399441055744.0, 1.0 / 6.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 5040.0, 1.0 / 720.0,     \
      1.0 / 362880.0, 1.0 / 40320.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 479001600.0,  \
      6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,          \
      2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,          \
      1.479819860511658591e-01
enum {
  TBK_L2E, TBK_LN2HI, TBK_LN2LO, TBK_SH, TBK_C3, TBK_C5, TBK_C4, TBK_C7, TBK_C6, TBK_C9,
  TBK_C8, TBK_C11, TBK_C10, TBK_C12, TBK_LG1, TBK_LG2, TBK_LG3, TBK_LG4, TBK_LG5, TBK_LG6,
  TBK_LG7
};
#if defined(__CUDACC__)
__constant__ double tbfm_kc[] = {TBFM_KLIST};
#endif
static const double tbfm_kh[] = {TBFM_KLIST};
#if defined(__CUDA_ARCH__)
#define TBK(i) tbfm_kc[i]
#else
#define TBK(i) tbfm_kh[i]
#endif

// exp(x): x = k ln2 + r, |r| <= ln2/2; exp(r) by its degree-12 Taylor
// polynomial (truncation < 2e-17 relative) in Estrin form; 2^k by exponent bits.
TBFM_QUAL double tb_exp(double x) {
  const double L2E = TBK(TBK_L2E);
  const double LN2HI = TBK(TBK_LN2HI);
  const double LN2LO = TBK(TBK_LN2LO);
  const double SH = TBK(TBK_SH);  // 1.5 * 2^52: round-to-nearest integer trick
  // clamp into [-746, 710] (beyond: 0 / inf after scaling); NaN restored below
  const double xc = fmin(fmax(x, -746.0), 710.0);
  double kd = fma(xc, L2E, SH);
  const int k = (int)(int64_t)(tbfm_bits(kd) & 0xffffffffull);  // low word = rint(x log2e)
  kd -= SH;
  double r = fma(kd, -LN2HI, xc);
  r = fma(kd, -LN2LO, r);
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  // c_n = 1/n!
  const double p01 = fma(r, 1.0, 1.0);
  const double p23 = fma(r, TBK(TBK_C3), 0.5);
  const double p45 = fma(r, TBK(TBK_C5), TBK(TBK_C4));
  const double p67 = fma(r, TBK(TBK_C7), TBK(TBK_C6));
  const double p89 = fma(r, TBK(TBK_C9), TBK(TBK_C8));
  const double pab = fma(r, TBK(TBK_C11), TBK(TBK_C10));
  const double pc = TBK(TBK_C12);
  const double q03 = fma(r2, p23, p01);
  const double q47 = fma(r2, p67, p45);
  const double q8b = fma(r2, pab, p89);
  const double q8c = fma(r4, pc, q8b);
  const double q07 = fma(r4, q47, q03);
  const double p = fma(r8, q8c, q07);
  // 2^k, k in [-1077, 1025], as two normal factors: one rounding into the
  // subnormal range, inf past the top
  const int k1 = k >> 1, k2 = k - k1;
  const double s1 = tbfm_from_bits((uint64_t)(int64_t)(k1 + 1023) << 52);
  const double s2 = tbfm_from_bits((uint64_t)(int64_t)(k2 + 1023) << 52);
  const double v = (p * s1) * s2;
  return x == x ? v : x;
}

// exp(x) on the fast domain [-708, 709] only (no range handling): the
// exp(-lambda r) terms, whose domain tb_set_params enforces
TBFM_QUAL double tb_exp_fast(double x) {
  const double L2E = TBK(TBK_L2E);
  const double LN2HI = TBK(TBK_LN2HI);
  const double LN2LO = TBK(TBK_LN2LO);
  const double SH = TBK(TBK_SH);  // 1.5 * 2^52: round-to-nearest integer trick
  double kd = fma(x, L2E, SH);
  const int k = (int)(int64_t)(tbfm_bits(kd) & 0xffffffffull);  // low word = rint(x log2e)
  kd -= SH;
  double r = fma(kd, -LN2HI, x);
  r = fma(kd, -LN2LO, r);
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  // c_n = 1/n!
  const double p01 = fma(r, 1.0, 1.0);
  const double p23 = fma(r, TBK(TBK_C3), 0.5);
  const double p45 = fma(r, TBK(TBK_C5), TBK(TBK_C4));
  const double p67 = fma(r, TBK(TBK_C7), TBK(TBK_C6));
  const double p89 = fma(r, TBK(TBK_C9), TBK(TBK_C8));
  const double pab = fma(r, TBK(TBK_C11), TBK(TBK_C10));
  const double pc = TBK(TBK_C12);
  const double q03 = fma(r2, p23, p01);
  const double q47 = fma(r2, p67, p45);
  const double q8b = fma(r2, pab, p89);
  const double q8c = fma(r4, pc, q8b);
  const double q07 = fma(r4, q47, q03);
  const double p = fma(r8, q8c, q07);
  // 2^k with k in [-1021, 1023] (the domain keeps k >= -1021)
  const double scale = tbfm_from_bits((uint64_t)(int64_t)(k + 1023) << 52);
  return p * scale;
}

// log(x), x > 0 normal: x = 2^e m, m in [sqrt(1/2), sqrt(2)); f = m - 1,
// s = f / (2 + f), log(m) = f - (hfsq - s (hfsq + R(s^2))) (fdlibm form),
// R by its degree-7 polynomial in z = s^2 (fdlibm coefficients) in Estrin form.
TBFM_QUAL double tb_rcp(double y);
TBFM_QUAL double tb_log(double x) {
  // subnormals: scale by 2^54 first (branch-free select)
  const int sub = x < 2.2250738585072014e-308;
  const double xs = sub ? x * 18014398509481984.0 : x;
  uint64_t u = tbfm_bits(xs);
  int e = (int)((u >> 52) & 0x7ff) - 1023 - (sub ? 54 : 0);
  // mantissa in [1, 2); move to [sqrt(1/2), sqrt(2)) (compare on the high word)
  uint64_t mb = (u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  const uint64_t hi = mb >> 32;
  const int big = hi > 0x3ff6a09eull;  // m > sqrt(2)
  mb -= (uint64_t)big << 52;           // halve m
  e += big;
  const double m = tbfm_from_bits(mb);
  const double f = m - 1.0;
  const double s = f * tb_rcp(2.0 + f);
  const double z = s * s, w = z * z;
  const double Lg1 = TBK(TBK_LG1), Lg2 = TBK(TBK_LG2), Lg3 = TBK(TBK_LG3), Lg4 = TBK(TBK_LG4),
               Lg5 = TBK(TBK_LG5), Lg6 = TBK(TBK_LG6), Lg7 = TBK(TBK_LG7);
  // R = z (Lg1 + z Lg2 + ... + z^6 Lg7), Estrin in z
  const double a = fma(z, Lg2, Lg1);
  const double b = fma(z, Lg4, Lg3);
  const double c = fma(z, Lg6, Lg5);
  const double ab = fma(w, b, a);
  const double cd = fma(w, Lg7, c);
  const double R = z * fma(w * w, cd, ab);
  const double hfsq = 0.5 * f * f;
  const double ed = (double)e;
  const double LN2HI = TBK(TBK_LN2HI);
  const double LN2LO = TBK(TBK_LN2LO);
  const double v = fma(ed, LN2HI, f - (hfsq - (s * (hfsq + R) + ed * LN2LO)));
  // x <= 0, inf, NaN: log(0) = -inf, log(x < 0) = NaN, log(inf) = inf
  const double special = x == 0.0 ? -HUGE_VAL : (x > 0.0 ? x : (x - x) / (x - x));
  return (x > 0.0 && x < HUGE_VAL) ? v : special;
}

// log(x) on normal positive x only: log(beta zeta) and log(1 + u), whose
// domain tb_set_params enforces (beta >= 1e-250, zeta >= 1e-30)
TBFM_QUAL double tb_log_fast(double x) {
  uint64_t u = tbfm_bits(x);
  int e = (int)((u >> 52) & 0x7ff) - 1023;
  // mantissa in [1, 2); move to [sqrt(1/2), sqrt(2)) (compare on the high word)
  uint64_t mb = (u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  const uint64_t hi = mb >> 32;
  const int big = hi > 0x3ff6a09eull;  // m > sqrt(2)
  mb -= (uint64_t)big << 52;           // halve m
  e += big;
  const double m = tbfm_from_bits(mb);
  const double f = m - 1.0;
  const double s = f * tb_rcp(2.0 + f);
  const double z = s * s, w = z * z;
  const double Lg1 = TBK(TBK_LG1), Lg2 = TBK(TBK_LG2), Lg3 = TBK(TBK_LG3), Lg4 = TBK(TBK_LG4),
               Lg5 = TBK(TBK_LG5), Lg6 = TBK(TBK_LG6), Lg7 = TBK(TBK_LG7);
  // R = z (Lg1 + z Lg2 + ... + z^6 Lg7), Estrin in z
  const double a = fma(z, Lg2, Lg1);
  const double b = fma(z, Lg4, Lg3);
  const double c = fma(z, Lg6, Lg5);
  const double ab = fma(w, b, a);
  const double cd = fma(w, Lg7, c);
  const double R = z * fma(w * w, cd, ab);
  const double hfsq = 0.5 * f * f;
  const double ed = (double)e;
  const double LN2HI = TBK(TBK_LN2HI);
  const double LN2LO = TBK(TBK_LN2LO);
  return fma(ed, LN2HI, f - (hfsq - (s * (hfsq + R) + ed * LN2LO)));
}

// 1/y: single-precision reciprocal seed (~2^-24), two Newton steps (-> 2^-48
// -> 2^-96).
TBFM_QUAL double tb_rcp(double y) {
#if defined(__CUDA_ARCH__)
  // MUFU.RCP seed (~1 ulp of float) without __frcp_rn's IEEE fix-up path:
  // c2 fp64 22.8 -> 22.1 us, c5 2.86 -> 2.83 ms against the __frcp_rn seed
  float rf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)y));
  double r = (double)rf;
#else
  double r = (double)(1.0f / (float)y);
#endif
  double e = fma(-y, r, 1.0);
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}

// r = sqrt(x) and 1/r together (the displacement norm and the unit-vector
// scale), 1e-30 < x < 1e30: single-precision rsqrt seed, two Newton steps on
// y = 1/sqrt(x), then one Newton correction of r = x y (-> within 1 ulp).
TBFM_QUAL void tb_sqrt_rsqrt(double x, double *r_out, double *rinv_out) {
#if defined(__CUDA_ARCH__)
  double y = (double)rsqrtf((float)x);
#else
  double y = (double)(1.0f / sqrtf((float)x));
#endif
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  const double r = x * y;
  *r_out = fma(fma(-r, r, x), 0.5 * y, r);
  *rinv_out = y;
}

// log1p(u), u >= 0: w = 1 + u rounded; log1p(u) = log(w) + (u - (w - 1)) / w.
TBFM_QUAL double tb_log1p(double u) {
  const double w = 1.0 + u;
  const double c = (u - (w - 1.0)) * tb_rcp(w);
  return tb_log(w) + c;
}
