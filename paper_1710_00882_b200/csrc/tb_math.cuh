// tb_math.cuh -- Tersoff potential math as sm_100a device functions.
//
// Semantics follow reference pkg/src/tersoffmd/potential.py:167-290 and
// pkg/docs/math_notes.md; the expression trees are re-derived for the GPU:
//   * f_C taper via sincospi (potential.py:167-175; plateaus inclusive and exact)
//   * g in the cancellation-free form gamma(1 + c^2 x^2 / (d^2 (d^2 + x^2)))
//     (potential.py:190-199), written gamma + (gamma c^2/d^2) x^2 / den with one
//     reciprocal of den shared by g and dg/dcos
//   * bond order with 2 log + 2 exp + 1 reciprocal instead of the reference's 4 pow:
//       u = (beta zeta)^eta = exp(eta log t),  b = exp(-log1p(u)/(2 eta)),
//       db/dzeta = -beta/2 * (u/t) * (b/(1+u)) = -u b / (2 zeta (1+u))
//       (potential.py:202-215)
//     and the ZETA_TINY guard: zeta < 1e-30 => db = 0 (b still evaluated).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "tb_fastmath.h"

namespace tb {

constexpr int SMAX = 4;       // compile-time species counts (1..4)
constexpr int SDYN_MAX = 64;  // any table up to this many species: the S = 0 tile kernel
constexpr double ZETA_TINY = 1e-30;

// Per-entry constants derived on the host from the flattened tables (see
// tb_api.cu make_tables); T = double for fp64, float for the mixed mode.
template <class T>
struct TripP {
  T Rm, Rp, R, halfInvD, nqpInvD;  // plateau bounds, taper scale, -pi/(4D)
  T gamma, gc2d2, m2gc2, d2, h;   // g(cos) constants
  T lam3, lam3x3;                 // exp((lam3 (rij-rik))^m) term
  int m;
  int pad;
};

template <class T>
struct PairP {
  T Rm, Rp, R, halfInvD, nqpInvD;
  T A, lam1, B, lam2;
  T beta, eta, neg_half_inv_eta, neg_half_beta;
};

template <class T, int S>
struct Tables {
  // S = 0 (runtime species count): one dummy entry, the tables are in global
  // memory (KArgs::dyn_pair / dyn_trip)
  PairP<T> pair[S > 0 ? S * S : 1];
  TripP<T> trip[S > 0 ? S * S * S : 1];
  // 1 when g(cos) of entry (i,j,k) equals that of (i,k,j) for every triple
  // (gamma, c, d, h, lam3, m depend on i only, as in the Tersoff-1989 tables):
  // the (i,b,a) term then reuses the (i,a,b) angular values
  int gsym;
  // 1 when g(cos) of entry (i,j,k) depends on i only (gamma, c, d, h equal
  // for all j, k): the kernel keeps atom i's angular constants in registers
  // instead of indexing the table per partner (the SiC fixture, Tersoff-1989
  // tables)
  int ang_i;
  // 1 when the pair cutoff (R, D of entry (i,j,j)) equals the k-role cutoff of
  // entry (i,j,j) -- one species: the pair term reuses the lane's f_C
  int fc_same;
};

// ---- transcendental wrappers (overloads keep the templates readable) ----
__device__ __forceinline__ double t_exp(double x) { return tb_exp_fast(x); }
// exp of an argument no table bound keeps in range (eta log(beta zeta), the
// bond-order exponent, (lam3 t)^m): full-range fp64 exp
__device__ __forceinline__ double t_exp_any(double x) { return tb_exp(x); }
// mixed mode: MUFU-based exp2/log2 (relative error ~2^-22 plus the argument
// rounding), well inside the 1e-5 force tolerance of the mixed mode
__device__ __forceinline__ float t_exp(float x) { return __expf(x); }
__device__ __forceinline__ float t_exp_any(float x) { return __expf(x); }
__device__ __forceinline__ double t_log(double x) { return tb_log_fast(x); }
__device__ __forceinline__ float t_log(float x) { return __logf(x); }
__device__ __forceinline__ double t_log1p(double x) { return tb_log1p(x); }
__device__ __forceinline__ float t_log1p(float x) { return log1pf(x); }
__device__ __forceinline__ void t_sincospi(double x, double *s, double *c) { sincospi(x, s, c); }
__device__ __forceinline__ void t_sincospi(float x, float *s, float *c) { sincospif(x, s, c); }
__device__ __forceinline__ double t_rcp(double x) { return tb_rcp(x); }
__device__ __forceinline__ float t_rcp(float x) {
  float r;  // MUFU.RCP (~1 ulp) -- the mixed mode's tolerance is 1e-5
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}


// f_C and dF_C/dr with inclusive exact plateaus (potential.py:167-175).
// Returns false when r >= R + D (exactly zero contribution).
template <class T, class P>
__device__ __forceinline__ bool cutoff(T r, const P &p, T &fc, T &dfc) {
  if (r <= p.Rm) {
    fc = T(1);
    dfc = T(0);
    return true;
  }
  if (r >= p.Rp) {
    fc = T(0);
    dfc = T(0);
    return false;
  }
  T s, c;
  t_sincospi((r - p.R) * p.halfInvD, &s, &c);  // sin/cos(pi/2 (r-R)/D)
  fc = T(0.5) - T(0.5) * s;
  dfc = p.nqpInvD * c;
  return true;
}

// g(cos) constants of one entry, held in registers (Tables::ang_i)
template <class T>
struct AngP {
  T gamma, gc2d2, m2gc2, d2, h;
};

template <class T>
__device__ __forceinline__ AngP<T> ang_of(const TripP<T> &p) {
  AngP<T> a;
  a.gamma = p.gamma;
  a.gc2d2 = p.gc2d2;
  a.m2gc2 = p.m2gc2;
  a.d2 = p.d2;
  a.h = p.h;
  return a;
}

// g(cos) and dg/dcos (potential.py:190-199), cancellation-free.
template <class T, class P>
__device__ __forceinline__ void angular(T cost, const P &p, T &g, T &dg) {
  T x = p.h - cost;
  T x2 = x * x;
  T inv = t_rcp(p.d2 + x2);
  g = p.gamma + p.gc2d2 * (x2 * inv);
  dg = (p.m2gc2 * x) * (inv * inv);
}

// exp((lam3 t)^m) with t = rij - rik and its derivative factor wrt t.
template <class T>
__device__ __forceinline__ void lam3_term(T dr, const TripP<T> &p, T &ex, T &darg) {
  T t = p.lam3 * dr;
  if (p.m == 3) {
    ex = t_exp_any(t * t * t);
    darg = p.lam3x3 * (t * t);
  } else {
    ex = t_exp_any(t);
    darg = p.lam3;
  }
}

// Pair part of one ordered (i,j) bond at fixed zeta (potential.py:280-290):
// returns V, dV/dr and delta_zeta = f_C f_A db/dzeta.
// pair_part_fc: the same with f_C(r), dF_C/dr already known (r < R + D)
// Main path of the pair part, zeta >= ZETA_TINY, branch-free (the row kernel
// interleaves several of these; pair_part_fc adds the isolated-bond branch).
//   u = t^eta, b = (1+u)^(-1/2eta), and with t^(eta-1) = u/t, t = beta zeta:
//   db/dzeta = -beta/2 t^(eta-1) (1+u)^(-1/2eta-1) = -(1/2) u b / (zeta (1+u))
// one reciprocal serves db and the log1p correction (1/w = zeta / (zeta w)).
// Range (any table): beyond x = eta log t = XBIG, 1/u is below the rounding
// unit, so log1p(u) = XBIG + (x - XBIG) to rounding and u/(1+u) = 1: u is
// formed from x clamped to XBIG (no overflow however large eta) and the excess
// added to log1p; below -708 u is at most a subnormal (clamped: b = 1,
// db ~ 1e-308/zeta).  Every exp / log argument stays on the fast domain:
// -l1p/2eta >= -log(t)/2 >= -355.
template <class T>
__device__ __forceinline__ void pair_part_main(T r, T zeta, const PairP<T> &p, T fc, T dfc, T &v,
                                               T &dvdr, T &dzeta) {
  T fr = p.A * t_exp(-p.lam1 * r);
  T fa = -p.B * t_exp(-p.lam2 * r);
  T t = p.beta * zeta;
  constexpr T XBIG = sizeof(T) == 8 ? T(36) : T(17);
  const T lt = t_log(t);
  const T x = p.eta * lt;
  const T xc = fmin(x, XBIG);
  const T u = t_exp(fmax(xc, T(-708)));
  const T w = T(1) + u;
  const T rzw = t_rcp(zeta * w);
  // log1p(u) = log(w) + (u - (w - 1)) / w, w = fl(1 + u)
  const T l1p = t_log(w) + (u - (w - T(1))) * (zeta * rzw) + (x - xc);
  const T b = t_exp(p.neg_half_inv_eta * l1p);
  const T db = T(-0.5) * (u * b) * rzw;
  T inner = fr + b * fa;
  v = fc * inner;
  dvdr = dfc * inner + fc * (-p.lam1 * fr + b * (-p.lam2 * fa));
  dzeta = fc * fa * db;
}

template <class T>
__device__ __forceinline__ void pair_part_fc(T r, T zeta, const PairP<T> &p, T fc, T dfc, T &v,
                                             T &dvdr, T &dzeta) {
  if (zeta < T(ZETA_TINY)) {
    // isolated bond (potential.py:202-215): db = 0; b from the library
    // functions, which also cover subnormal beta*zeta (exact b = 1 at zeta = 0)
    T fr = p.A * t_exp(-p.lam1 * r);
    T fa = -p.B * t_exp(-p.lam2 * r);
    T t = p.beta * zeta;
    T u = zeta > T(0) ? pow(t, p.eta) : T(0);
    T b = pow(T(1) + u, p.neg_half_inv_eta);
    T inner = fr + b * fa;
    v = fc * inner;
    dvdr = dfc * inner + fc * (-p.lam1 * fr + b * (-p.lam2 * fa));
    dzeta = fc * fa * T(0);
  } else {
    pair_part_main(r, zeta, p, fc, dfc, v, dvdr, dzeta);
  }
}

template <class T>
__device__ __forceinline__ void pair_part(T r, T zeta, const PairP<T> &p, T &v, T &dvdr,
                                          T &dzeta) {
  T fc, dfc;
  if (!cutoff(r, p, fc, dfc)) {
    v = T(0);
    dvdr = T(0);
    dzeta = T(0);
    return;
  }
  pair_part_fc(r, zeta, p, fc, dfc, v, dvdr, dzeta);
}

}  // namespace tb
