// tb_warp.cuh -- warp-per-chunk Tersoff kernel (K4/K5 fast path).
//
// Chunks (built with the neighbour list, k_fill_lanes): rows of equal length L
// packed floor(32/L) to a warp, so lane = one (i,j) skin-list entry, the L
// lanes of atom i are contiguous and every lane runs the same L-1 iterations
// of the k-loops.  What a lane needs from the other neighbours of i (unit
// vector, r, f_C, dzeta) is pulled from the owning lane with __shfl_sync;
// the angular values of phase 1 are kept in a per-warp shared cache for
// phase 2.  No block barriers inside the loop.
//
//   pack   : r2 < r_cut^2 at current positions, min image (neighbor.py:330-360)
//   phase 1: zeta_ij over k, then V, dV/dr, dzeta (kernels.py:279-299,
//            potential.py:238-290)
//   phase 2: the force on neighbour a from every term centred on i -- (i,a,b)
//            with a as j and (i,b,a) with a as k -- along e_a and e_b
//   scatter: F_a += f_a, F_i -= f_a (red.global.add.f64 into the context's
//            accumulator) or the per-entry buffer (deterministic gather);
//            e_i by a segmented warp reduction.
#pragma once
#include "tb_kernels.cuh"

namespace tb {

#ifndef TB_WARP_MINB
#define TB_WARP_MINB 4
#endif
constexpr int WNT = 128;  // threads per block of the warp kernel
constexpr int WPB = WNT / 32;
constexpr int QCAP = 8;   // k-iterations whose angular values are cached

template <class V>
__device__ __forceinline__ V shfl(V v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// select x[k] from a small register array without dynamic indexing
template <class T, int S>
__device__ __forceinline__ T pick(const T (&x)[S], int k) {
  T v = x[0];
#pragma unroll
  for (int q = 1; q < S; ++q) v = (k == q) ? x[q] : v;
  return v;
}

struct WArgs {
  const int4 *__restrict__ lanes;      // [nchunks*32] {entry, i, j, L}; entry -1 = idle lane
  const int *__restrict__ empty_atoms; // atoms with empty rows (per_atom = 0)
  int nchunks, n_empty;
  double *__restrict__ facc;           // ATOMIC: zeroed force accumulator (n,3)
};

struct WAcc {
  double acc_e = 0, wxx = 0, wyy = 0, wzz = 0, wxy = 0, wxz = 0, wyz = 0;
  unsigned long long c_vis = 0, c_pk = 0, c_lp = 0, c_lt = 0, c_tp = 0, c_tt = 0;
};

// One chunk: rows of length L (LC > 0: compile-time, loops fully unrolled so
// the independent k-iterations interleave; LC == 0: runtime Ldyn).
template <class T, int S, bool LAM3, int MODE, bool ST, int LC>
__device__ __forceinline__ void chunk_body(const KArgs &a, const WArgs &w, const Tables<T, S> &tab,
                                           T (*s_cache)[3][32], const int lane, const int4 cur,
                                           const double (&cxi)[3], const double (&cxj)[3],
                                           const int Ldyn, WAcc &A) {
  const int e = cur.x, i = cur.y, j = cur.z;
  const int L = LC > 0 ? LC : Ldyn;  // warp-uniform row length
  const bool valid = e >= 0;
  const int pos = lane % L;
  const int first = lane - pos;

  // ---- pack: displacement with min image, r2 < r_cut^2 ----
  double d[3] = {0, 0, 0}, r2 = 1.0;
  int si = 0, sj = 0;
  if (valid) {
    r2 = disp_r2(cxi, cxj, a.box, d);
    si = __ldg(a.species + i);
    sj = S > 1 ? __ldg(a.species + j) : 0;
    if (pos == 0) {
      if (!(isfinite(cxi[0]) && isfinite(cxi[1]) && isfinite(cxi[2])))
        atomicMin(&a.err->nonfinite_atom, i);
      if (si < 0 || si >= S) atomicMin(&a.err->bad_species_atom, i);
    }
    si = (si < 0 || si >= S) ? 0 : si;
    sj = (sj < 0 || sj >= S) ? 0 : sj;
  }
  const bool live = valid && r2 < a.rc2;
  const unsigned lmask = __ballot_sync(0xffffffffu, live);
  if (ST && valid && pos == 0) {
    const unsigned seg = (L >= 32 ? 0xffffffffu : ((1u << L) - 1u)) << first;
    const unsigned long long nl = __popc(lmask & seg);
    A.c_vis += nl * nl;  // zeta_visits = sum_i n_i^2 (kernels.py:537-544)
    A.c_pk += nl;
  }
  if (live && r2 < 1e-16) {
    unsigned long long key =
        ((unsigned long long)(__double_as_longlong(r2) >> 32) << 32) | (unsigned)e;
    atomicMin(&a.err->coinc_key, key);
  }
  const double rd = live ? sqrt(r2) : 1.0;
  const double invd = 1.0 / rd;
  const T ex = (T)(d[0] * invd), ey = (T)(d[1] * invd), ez = (T)(d[2] * invd);
  const T ra = (T)rd;
  // f_C(r) of this entry acting as k in (i, q, this) for every species q of j
  T fck[S], dfck[S];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    fck[q] = T(0);
    dfck[q] = T(0);
    if (live) cutoff(ra, tab.trip[(si * S + q) * S + sj], fck[q], dfck[q]);
  }
  const PairP<T> &pp = tab.pair[si * S + sj];
  const bool pair_live = live && ra < pp.Rp;

  // ---- phase 1: zeta (and the angular cache) ----
  T zeta = T(0);
#pragma unroll
  for (int q = 1; q < L; ++q) {
    const int src = first + (pos + q >= L ? pos + q - L : pos + q);
    const T bx = shfl(ex, src), by = shfl(ey, src), bz = shfl(ez, src);
    T fcb[S];
#pragma unroll
    for (int t = 0; t < S; ++t) fcb[t] = shfl(fck[t], src);
    const int sb = S > 1 ? shfl(sj, src) : 0;
    const T rb = LAM3 ? shfl(ra, src) : T(0);
    if (!live) continue;
    const TripP<T> &tp = tab.trip[(si * S + sj) * S + sb];
    T cost = ex * bx + ey * by + ez * bz;
    cost = fmin(T(1), fmax(T(-1), cost));
    T g, dg;
    angular(cost, tp, g, dg);
    if (q <= QCAP) {
      s_cache[q - 1][0][lane] = cost;
      s_cache[q - 1][1][lane] = g;
      s_cache[q - 1][2][lane] = dg;
    }
    const T f = pick(fcb, sj);  // f_C(r_b) with entry (i, a, b)
    if (pair_live && f != T(0)) {
      if (ST) {
        A.c_lt++;
        A.c_tt += f != T(1);
      }
      T term = f * g;
      if (LAM3) {
        T exv, darg;
        lam3_term(ra - rb, tp, exv, darg);
        term *= exv;
      }
      zeta += term;
    }
  }
  T v = T(0), dvdr = T(0), dz = T(0);
  if (pair_live) {
    if (ST) {
      A.c_lp++;
      A.c_tp += ra > pp.Rm;
    }
#ifdef TB_DBG_NOPAIR
    v = zeta * T(1e-6); dvdr = ra * T(1e-3); dz = zeta * T(1e-9);
#else
    pair_part(ra, zeta, pp, v, dvdr, dz);
#endif
  }

  // ---- phase 2: force on this neighbour from the terms centred on i ----
  T Sal = T(0), Sc = T(0), Sbx = T(0), Sby = T(0), Sbz = T(0);
#pragma unroll
  for (int q = 1; q < L; ++q) {
    const int src = first + (pos + q >= L ? pos + q - L : pos + q);
    const T bx = shfl(ex, src), by = shfl(ey, src), bz = shfl(ez, src);
    const T dzb = shfl(dz, src);
    T fcb[S];
#pragma unroll
    for (int t = 0; t < S; ++t) fcb[t] = shfl(fck[t], src);
    const int sb = S > 1 ? shfl(sj, src) : 0;
    const T rb = LAM3 ? shfl(ra, src) : T(0);
    if (!live) continue;
    const T f_b = pick(fcb, sj);     // f_C(r_b) in (i,a,b)
    const T f_a = pick(fck, sb);     // f_C(r_a) in (i,b,a)
    const T df_a = pick(dfck, sb);
    const bool t1 = (dz != T(0)) && (f_b != T(0));
    // f_C may round to 0 in the taper while dF_C/dr does not: test both
    const bool t2 = (dzb != T(0)) && (f_a != T(0) || df_a != T(0));
    if (!(t1 || t2)) continue;
    T cost, g, dg;
    if (q <= QCAP) {
      cost = s_cache[q - 1][0][lane];
      g = s_cache[q - 1][1][lane];
      dg = s_cache[q - 1][2][lane];
    } else {
      cost = ex * bx + ey * by + ez * bz;
      cost = fmin(T(1), fmax(T(-1), cost));
      angular(cost, tab.trip[(si * S + sj) * S + sb], g, dg);
    }
    T alpha, beta;
    if (S == 1 && !LAM3) {
      alpha = dzb * (df_a * g);
      beta = dg * (dz * f_b + dzb * f_a);
    } else {
      alpha = T(0);
      beta = T(0);
      if (t1) {  // (i,a,b): entry (si, sa, sb) -- the cached g, dg
        T exv = T(1), darg = T(0);
        if (LAM3) lam3_term(ra - rb, tab.trip[(si * S + sj) * S + sb], exv, darg);
        alpha += dz * (f_b * g * exv * darg);
        beta += dz * (f_b * dg * exv);
      }
      if (t2) {  // (i,b,a): entry (si, sb, sa)
        const TripP<T> &tp = tab.trip[(si * S + sb) * S + sj];
        T g2 = g, dg2 = dg, exv = T(1), darg = T(0);
        if (S > 1) angular(cost, tp, g2, dg2);
        if (LAM3) lam3_term(rb - ra, tp, exv, darg);
        alpha += dzb * (df_a * g2 * exv - f_a * g2 * exv * darg);
        beta += dzb * (f_a * dg2 * exv);
      }
    }
    Sal += alpha;
    Sc += beta * cost;
    Sbx += beta * bx;
    Sby += beta * by;
    Sbz += beta * bz;
  }
  if (live) {
    const T inva = T(1) / ra;
    const T ca = dvdr + Sal - Sc * inva;
    const double fx = -(double)(ca * ex + inva * Sbx);
    const double fy = -(double)(ca * ey + inva * Sby);
    const double fz = -(double)(ca * ez + inva * Sbz);
    A.wxx += d[0] * fx;
    A.wyy += d[1] * fy;
    A.wzz += d[2] * fz;
    A.wxy += d[0] * fy;
    A.wxz += d[0] * fz;
    A.wyz += d[1] * fz;
    if (MODE == 0) {
      double *fj = w.facc + 3 * (int64_t)j, *fi = w.facc + 3 * (int64_t)i;
      atomicAdd(fj, fx);
      atomicAdd(fj + 1, fy);
      atomicAdd(fj + 2, fz);
      atomicAdd(fi, -fx);  // F_i: translation invariance of the terms on i
      atomicAdd(fi + 1, -fy);
      atomicAdd(fi + 2, -fz);
    } else {
      double *fb = a.fbuf + 3 * (int64_t)e;
      fb[0] = fx;
      fb[1] = fy;
      fb[2] = fz;
    }
  } else if (MODE == 1 && valid) {
    double *fb = a.fbuf + 3 * (int64_t)e;
    fb[0] = 0.0;
    fb[1] = 0.0;
    fb[2] = 0.0;
  }
  // ---- e_i: segmented reduction over the L lanes of atom i ----
  double se = (double)v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double oe = __shfl_down_sync(0xffffffffu, se, o);
    if (pos + o < L) se += oe;
  }
  if (valid && pos == 0) {
    A.acc_e += se;
    if (a.per_atom) a.per_atom[i] = se + 0.0;
  }
}

template <class T, int S, bool LAM3, int MODE, bool ST>
__global__ void __launch_bounds__(WNT, TB_WARP_MINB)
    k_tersoff_warp(const KArgs a, const WArgs w, const __grid_constant__ Tables<T, S> gtab) {
  __shared__ Tables<T, S> s_tab;
  __shared__ double s_red[WPB][8];
  __shared__ T s_cache[WPB][QCAP][3][32];  // cos, g, dg of (i,a,b) from phase 1
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (S > 1) {
    const int *src = reinterpret_cast<const int *>(&gtab);
    int *dst = reinterpret_cast<int *>(&s_tab);
    for (int q = threadIdx.x; q < (int)(sizeof(Tables<T, S>) / sizeof(int)); q += WNT)
      dst[q] = src[q];
    __syncthreads();
  }
  const Tables<T, S> &tab = (S > 1) ? s_tab : gtab;
  for (int k = blockIdx.x * WNT + threadIdx.x; k < w.n_empty; k += gridDim.x * WNT) {
    const int m = w.empty_atoms[k];
    if (a.per_atom) a.per_atom[m] = 0.0;
    const int sm = a.species[m];
    if (sm < 0 || sm >= S) atomicMin(&a.err->bad_species_atom, m);
  }

  WAcc A;

  // software pipeline over this warp's chunks: lane records two chunks ahead,
  // positions one chunk ahead, so the dependent gathers overlap the math
  const int stride = gridDim.x * WPB;
  int c = blockIdx.x * WPB + wid;
  const int4 idle = make_int4(-1, 0, 0, 1);
  int4 cur = c < w.nchunks ? __ldg(w.lanes + 32 * (int64_t)c + lane) : idle;
  int4 nxt = c + stride < w.nchunks ? __ldg(w.lanes + 32 * (int64_t)(c + stride) + lane) : idle;
  double cxi[3] = {0, 0, 0}, cxj[3] = {0, 0, 0};
  if (cur.x >= 0) {
    load3(a.pos, cur.y, cxi);
    load3(a.pos, cur.z, cxj);
  }
  for (; c < w.nchunks; c += stride) {
    const int4 nx2 = c + 2 * stride < w.nchunks
                         ? __ldg(w.lanes + 32 * (int64_t)(c + 2 * stride) + lane)
                         : idle;
#ifndef TB_NO_POS_PREFETCH
    double nxi[3] = {0, 0, 0}, nxj[3] = {0, 0, 0};
    if (nxt.x >= 0) {
      load3(a.pos, nxt.y, nxi);
      load3(a.pos, nxt.z, nxj);
    }
#endif
    const int Ldyn = __shfl_sync(0xffffffffu, cur.w, 0);
    switch (Ldyn) {
      case 4: chunk_body<T, S, LAM3, MODE, ST, 4>(a, w, tab, s_cache[wid], lane, cur, cxi, cxj, Ldyn, A); break;
      case 5: chunk_body<T, S, LAM3, MODE, ST, 5>(a, w, tab, s_cache[wid], lane, cur, cxi, cxj, Ldyn, A); break;
      case 3: chunk_body<T, S, LAM3, MODE, ST, 3>(a, w, tab, s_cache[wid], lane, cur, cxi, cxj, Ldyn, A); break;
      case 6: chunk_body<T, S, LAM3, MODE, ST, 6>(a, w, tab, s_cache[wid], lane, cur, cxi, cxj, Ldyn, A); break;
      default: chunk_body<T, S, LAM3, MODE, ST, 0>(a, w, tab, s_cache[wid], lane, cur, cxi, cxj, Ldyn, A);
    }
    cur = nxt;
    nxt = nx2;
#ifndef TB_NO_POS_PREFETCH
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      cxi[q] = nxi[q];
      cxj[q] = nxj[q];
    }
#else
    if (cur.x >= 0) {
      load3(a.pos, cur.y, cxi);
      load3(a.pos, cur.z, cxj);
    }
#endif
  }

  // ---- stats and block partials (reduced by the finalize kernel) ----
  if (ST) {
    unsigned long long cs[6] = {A.c_vis, A.c_pk, A.c_lp, A.c_lt, A.c_tp, A.c_tt};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = warp_sum(cs[q]);
      if (lane == 0 && v) atomicAdd(&a.stats[q], v);
    }
  }
  double vals[7] = {A.acc_e, A.wxx, A.wyy, A.wzz, A.wxy, A.wxz, A.wyz};
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = warp_sum(vals[q]);
    if (lane == 0) s_red[wid][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < WPB; ++q) v += s_red[q][threadIdx.x];
    a.partials[8 * (int64_t)blockIdx.x + threadIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------
// chunk construction (at neighbour-list build)
// ---------------------------------------------------------------------------

struct ChunkPlan {
  int chunk_base[34];   // first chunk of rows of length L (L = 1..32), [33] = total
  int bucket_start[34]; // first index in the length-sorted atom list for length L
  int count[34];        // rows of length L
};

__global__ void k_iota(int n, int *__restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = i;
}

__global__ void k_len_hist(int n, const int *__restrict__ len, int *__restrict__ hist) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(hist + min(len[i], 33), 1);
}

// one warp per chunk: lane -> {entry, i, j, L} (entry -1: idle lane)
__global__ void k_fill_lanes(const ChunkPlan plan, const int *__restrict__ sorted_atoms,
                             const int *__restrict__ offsets, const int *__restrict__ nbr,
                             int4 *__restrict__ lanes) {
  const int c = blockIdx.x, lane = threadIdx.x;
  int L = 1;
  while (L < 32 && plan.chunk_base[L + 1] <= c) ++L;
  const int rpc = 32 / L;
  const int row = (c - plan.chunk_base[L]) * rpc + lane / L;
  int4 v = make_int4(-1, 0, 0, L);
  if (lane < rpc * L && row < plan.count[L]) {
    const int atom = sorted_atoms[plan.bucket_start[L] + row];
    const int e = offsets[atom] + lane % L;
    v = make_int4(e, atom, nbr[e], L);
  }
  lanes[32 * (int64_t)c + lane] = v;
}

// ---------------------------------------------------------------------------
// finalize: forces out of the accumulator (or the deterministic gather),
// block partials -> [E, W6], stats out; leaves accumulators zeroed
// ---------------------------------------------------------------------------

template <int MODE>
__global__ void k_finalize(int n, double *__restrict__ facc, const int *__restrict__ off,
                           const int *__restrict__ rev, const double *__restrict__ fbuf,
                           double *__restrict__ forces, int nparts,
                           const double *__restrict__ partials, double *__restrict__ result,
                           unsigned long long *__restrict__ stats_acc,
                           unsigned long long *__restrict__ stats_out) {
  if (MODE == 0) {
    const int64_t m3 = 3 * (int64_t)n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m3;
         k += (int64_t)gridDim.x * blockDim.x) {
      forces[k] = facc[k] + 0.0;
      facc[k] = 0.0;
    }
  } else {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
      double ix = 0.0, iy = 0.0, iz = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
      for (int e = off[m]; e < off[m + 1]; ++e) {
        const double *f = fbuf + 3 * (int64_t)__ldg(rev + e);
        ix += f[0];
        iy += f[1];
        iz += f[2];
        const double *g = fbuf + 3 * (int64_t)e;
        sx += g[0];
        sy += g[1];
        sz += g[2];
      }
      forces[3 * (int64_t)m] = (ix - sx) + 0.0;
      forces[3 * (int64_t)m + 1] = (iy - sy) + 0.0;
      forces[3 * (int64_t)m + 2] = (iz - sz) + 0.0;
    }
  }
  if (blockIdx.x == 0) {
    __shared__ double s[256][7];
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x)
#pragma unroll
      for (int q = 0; q < 7; ++q) acc[q] += partials[8 * (int64_t)b + q];
#pragma unroll
    for (int q = 0; q < 7; ++q) s[threadIdx.x][q] = acc[q];
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (threadIdx.x < h)
#pragma unroll
        for (int q = 0; q < 7; ++q) s[threadIdx.x][q] += s[threadIdx.x + h][q];
      __syncthreads();
    }
    if (threadIdx.x < 7) result[threadIdx.x] = s[0][threadIdx.x] + 0.0;
    if (threadIdx.x < 6) {
      if (stats_out) stats_out[threadIdx.x] = stats_acc[threadIdx.x];
      stats_acc[threadIdx.x] = 0ull;
    }
  }
}

}  // namespace tb
