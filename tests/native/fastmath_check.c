/* Host accuracy check of csrc/tb_fastmath.h against glibc libm (test only).
 * Prints the max ulp error of tb_exp / tb_log / tb_log1p / tb_rcp over
 * their documented domains. */
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include "../../paper_1710_00882_b200/csrc/tb_fastmath.h"

static double ulp_err(double got, double want) {
  if (got == want) return 0.0;
  double sp = nextafter(fabs(want), INFINITY) - fabs(want);
  return fabs(got - want) / sp;
}
static double urand(unsigned long long *s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(*s >> 11) * (1.0 / 9007199254740992.0);
}
int main(int argc, char **argv) {
  long n = argc > 1 ? atol(argv[1]) : 2000000;
  unsigned long long s = 12345;
  double me = 0, ml = 0, m1 = 0, mr = 0, msq = 0, mrs = 0;
  for (long i = 0; i < n; ++i) {
    double x = -708.0 + 1417.0 * urand(&s);
    double e = ulp_err(tb_exp(x), exp(x)); if (e > me) me = e;
    double xs = -20.0 + 25.0 * urand(&s);  /* the pair-term range */
    e = ulp_err(tb_exp(xs), exp(xs)); if (e > me) me = e;
    double y = exp(-700.0 + 1400.0 * urand(&s));
    e = ulp_err(tb_log(y), log(y)); if (e > ml) ml = e;
    double y2 = 0.5 + 1.5 * urand(&s);
    e = ulp_err(tb_log(y2), log(y2)); if (e > ml) ml = e;
    double u = exp(-80.0 + 90.0 * urand(&s));
    e = ulp_err(tb_log1p(u), log1p(u)); if (e > m1) m1 = e;
    double v = exp(-69.0 + 138.0 * urand(&s));  /* float-representable */
    e = ulp_err(tb_rcp(v), 1.0 / v); if (e > mr) mr = e;
    double q = exp(-69.0 + 138.0 * urand(&s)), sq, rs;
    if (i & 1) q = 1e-16 + 12.0 * urand(&s);  /* the r^2 < r_cut^2 range */
    tb_sqrt_rsqrt(q, &sq, &rs);
    e = ulp_err(sq, sqrt(q)); if (e > msq) msq = e;
    e = ulp_err(rs, 1.0 / sqrt(q)); if (e > mrs) mrs = e;
  }
  /* full range: subnormal results within 2 ulp of the smallest subnormal
     step, 0 / inf / NaN where libm gives them */
  int ood_ok = 1;
  for (double x = -760.0; x <= 712.0; x += 0.37) {
    const double g = tb_exp(x), w = exp(x);
    if (w == 0.0 || isinf(w)) ood_ok &= g == w;
    else if (w < 2.2250738585072014e-308) ood_ok &= fabs(g - w) <= 2 * 4.9406564584124654e-324;
    else ood_ok &= ulp_err(g, w) <= 4;
  }
  const double ys_ood[] = {1e-310, 4.9e-324, 3e-320, 2.2250738585072009e-308, 1e308 * 10.0};
  for (int q = 0; q < 5; ++q) ood_ok &= ulp_err(tb_log(ys_ood[q]), log(ys_ood[q])) <= 2;
  ood_ok &= isinf(tb_log(0.0)) && tb_log(0.0) < 0 && isnan(tb_log(-1.0)) && isnan(tb_log(NAN));
  ood_ok &= isnan(tb_exp(NAN)) && tb_exp(-1e300) == 0.0 && isinf(tb_exp(1e300));
  ood_ok &= tb_rcp(1e31) == 0.0 || fabs(tb_rcp(1e31)) < 1e-30;
  printf("{\"ood_ok\": %d, ", ood_ok);
  printf("\"exp_ulp\": %.3f, \"log_ulp\": %.3f, \"log1p_ulp\": %.3f, \"rcp_ulp\": %.3f, "
         "\"sqrt_ulp\": %.3f, \"rsqrt_ulp\": %.3f, \"n\": %ld}\n", me, ml, m1, mr, msq, mrs, n);
  return 0;
}
