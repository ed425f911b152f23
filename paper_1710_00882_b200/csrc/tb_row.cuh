// tb_row.cuh -- atom-per-lane Tersoff kernel for short rows (K4r).
//
// Rows of at most LM (= 4) skin-list entries -- every row of a diamond /
// zincblende crystal -- are evaluated by ONE lane each: the lane holds its
// atom's LM neighbours (unit vector, r, f_C) in registers, so nothing is
// exchanged between lanes -- no shared-memory table, no staging, no shuffles
// -- and the angular function, which depends on the unordered pair {j,k} only
// (one species, potential.py:190-199), is evaluated once per pair instead of
// once per ordered (j,k): LM(LM-1)/2 = 6 evaluations per atom instead of 12.
// The LM independent pair terms of an atom give the FP64 pipe its
// instruction-level parallelism; the warp-chunk kernel (tb_warp.cuh) gets it
// from 16 resident warps and pays for the lane exchange in L1/shared
// wavefronts (its top ncu unit at every configuration).
//
//   pack    : r2 < r_cut^2 at current positions, min image (neighbor.py:330-360)
//   zeta_p  : sum_{q != p} f_C(r_q) g(cos_pq)               (kernels.py:279-295)
//   pair    : V, dV/dr, delta_zeta at fixed zeta            (potential.py:280-290)
//   forces  : f_p = -(c_p e_p + S_p / r_p), c_p = dV/dr + sum_q dz_q f_C'(r_p) g_pq
//             - (sum_q beta_pq cos_pq) / r_p, S_p = sum_q beta_pq e_q,
//             beta_pq = g'(cos_pq) (dz_p f_C(r_q) + dz_q f_C(r_p));  F_i = -sum_p f_p
// Same device functions (tb_math.cuh) as the warp-chunk kernel; one species,
// lam3 = 0 tables whose pair and k-role cutoffs coincide (Tables::fc_same).
#pragma once
#include "tb_warp.cuh"

namespace tb {

#ifndef TB_ROW_NT
#define TB_ROW_NT 128
#endif
#ifndef TB_ROW_MINB64
#define TB_ROW_MINB64 4  // 16 warps/SM at 128 registers with TB_ROW_SSTATE + TB_ROW_SACC (c5 2.128 -> 2.088 ms);
                         // without them: 3 (12 warps at 168 registers), see DESIGN 3.10
#endif
#ifndef TB_ROW_MINB32
#define TB_ROW_MINB32 4
#endif

#ifndef TB_ROW_VIR_RE
#define TB_ROW_VIR_RE 1  // virial from r_p e_p (x) f_p: the displacement registers die after the unit vectors
#endif
#ifndef TB_ROW_SACC
#define TB_ROW_SACC 1  // fp64: energy / virial accumulators in per-thread shared slots instead of
                       // registers (alone at 12 warps/SM: c5 2.13 -> 2.20 ms; with SSTATE at 16: 2.09)
#endif
#ifndef TB_ROW_SSTATE
#define TB_ROW_SSTATE 1  // fp64: unit vectors, 1/r, cos, g' parked in shared memory over the pair parts
                         // (28 doubles per thread; frees their registers where the four pair chains peak)
#endif
#ifndef TB_ROW_SCNT
#define TB_ROW_SCNT 1  // fp64, counters on: the six counters in per-thread shared slots
#endif
#ifndef TB_ROW_RECOS
#define TB_ROW_RECOS 0   // recompute cos in the force phase instead of keeping it over the pair parts
                         // (measured neutral: c5 2.130 vs 2.133 ms)
#endif
#ifndef TB_ROW_MAXREG
#define TB_ROW_MAXREG 0  // > 0: __maxnreg__ instead of the min-blocks bound (fp64)
#endif

template <class T>
struct RowCfg {
  static constexpr int nt = TB_ROW_NT;
  static constexpr int minb = sizeof(T) == 8 ? TB_ROW_MINB64 : TB_ROW_MINB32;
};

struct RArgs {
  const int *__restrict__ atoms;       // sorted_atoms: [empty rows | rows by length]
  int first, count;                    // rows atoms[first, first + count): lengths 1..LM
  const int *__restrict__ dplan;       // non-null: DevPlan (tb_md_run); bounds read on the device
  int n_empty;                         // atoms[0, n_empty): empty rows (per_atom = 0, checks)
  int count_packed;                    // count zeta_visits / packed pairs here
};

// index of the unordered pair {p, q}, p < q, among LM(LM-1)/2
template <int LM>
__host__ __device__ constexpr int pair_index(int p, int q) {
  return p * LM - p * (p + 1) / 2 + (q - p - 1);
}

template <class T, int LM, int MODE, bool ST>
__global__ void
#if TB_ROW_MAXREG > 0
__launch_bounds__(RowCfg<T>::nt) __maxnreg__(sizeof(T) == 8 ? TB_ROW_MAXREG : 128)
#else
__launch_bounds__(RowCfg<T>::nt, RowCfg<T>::minb)
#endif
    k_tersoff_row(const KArgs a, const RArgs ra, const __grid_constant__ Tables<T, 1> tab,
                  const int plan_first_off, const int plan_end_off) {
  constexpr int NTH = RowCfg<T>::nt, NWP = NTH / 32;
  constexpr int NP = LM * (LM - 1) / 2;
  __shared__ double s_red[NWP][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int first = ra.first, count = ra.count, n_empty = ra.n_empty;
  if (ra.dplan) {
    // device plan (DevPlan): n_empty and the bucket starts of lengths 1 and LM + 1
    n_empty = __ldg(ra.dplan + 1);
    first = __ldg(ra.dplan + plan_first_off);
    count = __ldg(ra.dplan + plan_end_off) - first;
  }
  const int gsz = gridDim.x * NTH, gid = blockIdx.x * NTH + threadIdx.x;
  for (int k = gid; k < n_empty; k += gsz) {
    const int m = ra.atoms[k];
    if (a.per_atom) a.per_atom[m] = 0.0;
    const int sm = a.species[m];
    if (sm != 0) atomicMin(&a.err->bad_species_atom, m);
    const double *xm = a.pos + 3 * (int64_t)m;
    if (!(isfinite(__ldg(xm)) && isfinite(__ldg(xm + 1)) && isfinite(__ldg(xm + 2))))
      atomicMin(&a.err->nonfinite_atom, m);
  }

  constexpr bool SACC = TB_ROW_SACC && sizeof(T) == 8;
  __shared__ double s_acc[SACC ? 7 : 1][SACC ? NTH : 1];
  constexpr bool SST = TB_ROW_SSTATE && sizeof(T) == 8;
  constexpr int NST = 4 * LM + 2 * NP;
  __shared__ T s_st[SST ? NST : 1][SST ? NTH : 1];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // E, W xx yy zz xy xz yz
  if (SACC) {
#pragma unroll
    for (int q = 0; q < 7; ++q) s_acc[q][threadIdx.x] = 0.0;
  }
  // per-thread counters: at most 16 per atom and n / blockDim atoms per thread, so 32 bits hold them
  // (fp64 keeps them in per-thread shared slots: its registers are spent, SCNT)
  constexpr bool SCNT = ST && sizeof(T) == 8 && TB_ROW_SCNT;
  __shared__ unsigned s_cnt[SCNT ? 6 : 1][SCNT ? NTH : 1];
  if (SCNT) {
#pragma unroll
    for (int q = 0; q < 6; ++q) s_cnt[q][threadIdx.x] = 0u;
  }
  unsigned c_vis = 0, c_pk = 0, c_lp = 0, c_lt = 0, c_tp = 0, c_tt = 0;
  const PairP<T> &pp = tab.pair[0];
  const TripP<T> &tp = tab.trip[0];

  // software pipeline over the indices: i, the row bounds and the neighbour
  // indices of the next atom are fetched while this one computes.  (A second
  // stage with prefetch.global.L1/L2 of the next atom's positions was measured
  // slower: the extra index registers spill, c5 fp64 2.19 -> 2.41 ms without
  // and 2.57 ms with the prefetches.  Prefetching only each lane's own
  // position a few iterations ahead, without the second index stage: 2.13 ->
  // 2.22 ms.)
  int i = -1, o = 0, L = 0, jn[LM];
  if (gid < count) {
    i = __ldg(ra.atoms + first + gid);
    o = __ldg(a.off + i);
    L = __ldg(a.off + i + 1) - o;
#pragma unroll
    for (int q = 0; q < LM; ++q) jn[q] = q < L ? __ldg(a.nbr + o + q) : i;
  }
  for (int idx = gid; idx < count; idx += gsz) {
    const int ci = i, co = o, cL = L;
    int cj[LM];
#pragma unroll
    for (int q = 0; q < LM; ++q) cj[q] = jn[q];
#ifdef TB_ROW_DEBUG
    // debug builds: every index this lane dereferences is inside its array
    // (compute-sanitizer is not available on the GPU pool)
    {
      bool ok = ci >= 0 && ci < a.n && co >= 0 && cL >= 0 && cL <= LM;
#pragma unroll
      for (int q = 0; q < LM; ++q) ok = ok && cj[q] >= 0 && cj[q] < a.n;
      if (!ok) {
        atomicExch(&a.err->overflow, 1);  // reported as an internal error
        continue;
      }
    }
#endif
    // ---- gathers of this atom ----
    double xi[3], xj[LM][3];
    load3(a.pos, ci, xi);
#pragma unroll
    for (int q = 0; q < LM; ++q) load3(a.pos, cj[q], xj[q]);
    const int si = __ldg(a.species + ci);
    // ---- indices of the next atom ----
    const bool more = idx + gsz < count;
    if (more) i = __ldg(ra.atoms + first + idx + gsz);

    if (!(isfinite(xi[0]) && isfinite(xi[1]) && isfinite(xi[2])))
      atomicMin(&a.err->nonfinite_atom, ci);
    if (si != 0) atomicMin(&a.err->bad_species_atom, ci);

    // Straight-line code from here to the forces: every rarely-taken path (a
    // quotient within 1e-9 of a half-integer, coincident atoms, a distance in
    // the taper, an isolated bond) is a flag tested once after the common
    // arithmetic, so the LM independent dependency chains of an atom (rsqrt
    // Newton steps, the exp / log polynomials of the pair parts) sit in one
    // basic block and interleave -- the FP64 pipe is fed by instruction-level
    // parallelism instead of by resident warps.
    // ---- pack: displacement (the arithmetic of disp_r2), live test ----
    double d[LM][3], r2[LM];
    if (a.box.per[0] & a.box.per[1] & a.box.per[2]) {
      double v[LM][3], qn[LM][3];
      bool near = false;
#pragma unroll
      for (int q = 0; q < LM; ++q)
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          v[q][ax] = __dsub_rn(xj[q][ax], xi[ax]);
          const double y = __dmul_rn(v[q][ax], a.box.invL[ax]);
          qn[q][ax] = rint(y);
          near |= 0.5 - fabs(y - qn[q][ax]) < 1e-9;
        }
      if (__builtin_expect(near, 0)) {
#pragma unroll
        for (int q = 0; q < LM; ++q)
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const double y = __dmul_rn(v[q][ax], a.box.invL[ax]);
            if (0.5 - fabs(y - qn[q][ax]) < 1e-9)
              qn[q][ax] = rint_quotient_exact(v[q][ax], a.box.L[ax]);
          }
      }
#pragma unroll
      for (int q = 0; q < LM; ++q) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
          d[q][ax] = __dsub_rn(v[q][ax], __dmul_rn(a.box.L[ax], qn[q][ax]));
        r2[q] = __dadd_rn(__dadd_rn(__dmul_rn(d[q][0], d[q][0]), __dmul_rn(d[q][1], d[q][1])),
                          __dmul_rn(d[q][2], d[q][2]));
      }
    } else {
#pragma unroll
      for (int q = 0; q < LM; ++q) r2[q] = disp_r2(xi, xj[q], a.box, d[q]);
    }
    bool live[LM], coin = false;
    int nlive = 0;
#pragma unroll
    for (int q = 0; q < LM; ++q) {
      live[q] = q < cL && r2[q] < a.rc2;
      nlive += live[q];
      coin |= live[q] && r2[q] < 1e-16;
    }
    if (__builtin_expect(coin, 0)) {
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (live[q] && r2[q] < 1e-16) {
          unsigned long long key =
              ((unsigned long long)(__double_as_longlong(r2[q]) >> 32) << 32) | (unsigned)(co + q);
          atomicMin(&a.err->coinc_key, key);
        }
    }
    // ---- unit vectors, f_C ----
    T ex[LM], ey[LM], ez[LM], rr[LM], inv[LM], fc[LM], dfc[LM];
    bool taper = false;
#pragma unroll
    for (int q = 0; q < LM; ++q) {
      if (sizeof(T) == 8) {
        double rd, invd;
        tb_sqrt_rsqrt(live[q] ? r2[q] : 1.0, &rd, &invd);
        ex[q] = (T)(d[q][0] * invd);
        ey[q] = (T)(d[q][1] * invd);
        ez[q] = (T)(d[q][2] * invd);
        rr[q] = (T)rd;
        inv[q] = (T)invd;
      } else {
        const float r2f = live[q] ? (float)r2[q] : 1.0f;
        const float rinv = rsqrtf(r2f);
        rr[q] = (T)(r2f * rinv);
        inv[q] = (T)rinv;
        ex[q] = (T)((float)d[q][0] * rinv);
        ey[q] = (T)((float)d[q][1] * rinv);
        ez[q] = (T)((float)d[q][2] * rinv);
      }
      // plateaus of cutoff() (potential.py:167-175); the taper below
      fc[q] = (live[q] && rr[q] <= tp.Rm) ? T(1) : T(0);
      dfc[q] = T(0);
      taper |= live[q] && rr[q] > tp.Rm && rr[q] < tp.Rp;
    }
    if (taper) {
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (live[q] && rr[q] > tp.Rm && rr[q] < tp.Rp) cutoff(rr[q], tp, fc[q], dfc[q]);
    }
    if (ST && ra.count_packed) {
      // zeta_visits = sum_i n_i^2 (kernels.py:537-544)
      if (SCNT) {
        s_cnt[0][threadIdx.x] += (unsigned)(nlive * nlive);
        s_cnt[1][threadIdx.x] += (unsigned)nlive;
      } else {
        c_vis += (unsigned)(nlive * nlive);
        c_pk += nlive;
      }
    }
    if (more) {
      o = __ldg(a.off + i);
      L = __ldg(a.off + i + 1) - o;
    }

    // ---- angular values, once per unordered pair ----
    T cs[NP], g[NP], dg[NP];
#pragma unroll
    for (int p = 0; p < LM; ++p)
#pragma unroll
      for (int q = p + 1; q < LM; ++q) {
        const int u = pair_index<LM>(p, q);
        T c = ex[p] * ex[q] + ey[p] * ey[q] + ez[p] * ez[q];
        TB_CLAMP_COS(c);
        cs[u] = c;
        angular(c, tp, g[u], dg[u]);
      }

    if (SST) {
      volatile T(*st)[SST ? NTH : 1] = s_st;
#pragma unroll
      for (int q = 0; q < LM; ++q) {
        st[4 * q][threadIdx.x] = ex[q];
        st[4 * q + 1][threadIdx.x] = ey[q];
        st[4 * q + 2][threadIdx.x] = ez[q];
        st[4 * q + 3][threadIdx.x] = inv[q];
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        st[4 * LM + u][threadIdx.x] = cs[u];
        st[4 * LM + NP + u][threadIdx.x] = dg[u];
      }
    }
    // ---- zeta, pair parts ----
    T zeta[LM], vv[LM], dvdr[LM], dz[LM];
    bool pair_live[LM], tiny = false;
    int n_lt = 0, n_tt = 0, n_lp = 0, n_tp = 0;  // this atom's counts (one 64-bit add each below)
#pragma unroll
    for (int p = 0; p < LM; ++p) {
      pair_live[p] = live[p] && rr[p] < pp.Rp;
      zeta[p] = T(0);
#pragma unroll
      for (int q = 0; q < LM; ++q) {
        if (q == p) continue;
        const int u = p < q ? pair_index<LM>(p, q) : pair_index<LM>(q, p);
        zeta[p] += fc[q] * g[u];  // a dead partner has f_C = 0
        if (ST) {
          n_lt += pair_live[p] && fc[q] != T(0);
          n_tt += pair_live[p] && fc[q] != T(0) && fc[q] != T(1);
        }
      }
      tiny |= pair_live[p] && zeta[p] < T(ZETA_TINY);
      if (ST) {
        n_lp += pair_live[p];
        n_tp += pair_live[p] && rr[p] > pp.Rm;
      }
    }
    if (ST) {
      if (SCNT) {
        s_cnt[2][threadIdx.x] += (unsigned)n_lp;
        s_cnt[3][threadIdx.x] += (unsigned)n_lt;
        s_cnt[4][threadIdx.x] += (unsigned)n_tp;
        s_cnt[5][threadIdx.x] += (unsigned)n_tt;
      } else {
        c_lt += n_lt;
        c_tt += n_tt;
        c_lp += n_lp;
        c_tp += n_tp;
      }
    }
#pragma unroll
    for (int p = 0; p < LM; ++p) {
      T v_, dv_, dz_;
      pair_part_main(rr[p], fmax(zeta[p], T(ZETA_TINY)), pp, fc[p], dfc[p], v_, dv_, dz_);
      vv[p] = pair_live[p] ? v_ : T(0);
      dvdr[p] = pair_live[p] ? dv_ : T(0);
      dz[p] = pair_live[p] ? dz_ : T(0);
    }
    if (__builtin_expect(tiny, 0)) {  // isolated bonds: the library path of pair_part_fc
#pragma unroll
      for (int p = 0; p < LM; ++p)
        if (pair_live[p] && zeta[p] < T(ZETA_TINY))
          pair_part_fc(rr[p], zeta[p], pp, fc[p], dfc[p], vv[p], dvdr[p], dz[p]);
    }
    double e_i = 0.0;
#pragma unroll
    for (int p = 0; p < LM; ++p) e_i += (double)vv[p];
    if (more) {
#pragma unroll
      for (int q = 0; q < LM; ++q) jn[q] = q < L ? __ldg(a.nbr + o + q) : i;
    }

    if (SST) {
      volatile T(*st)[SST ? NTH : 1] = s_st;
#pragma unroll
      for (int q = 0; q < LM; ++q) {
        ex[q] = st[4 * q][threadIdx.x];
        ey[q] = st[4 * q + 1][threadIdx.x];
        ez[q] = st[4 * q + 2][threadIdx.x];
        inv[q] = st[4 * q + 3][threadIdx.x];
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        cs[u] = st[4 * LM + u][threadIdx.x];
        dg[u] = st[4 * LM + NP + u][threadIdx.x];
      }
    }
    // ---- forces ----
    T beta[NP];
#pragma unroll
    for (int p = 0; p < LM; ++p)
#pragma unroll
      for (int q = p + 1; q < LM; ++q) {
        const int u = pair_index<LM>(p, q);
        beta[u] = dg[u] * (dz[p] * fc[q] + dz[q] * fc[p]);
      }
    double fix = 0.0, fiy = 0.0, fiz = 0.0;
    if (SACC) {
#pragma unroll
      for (int q = 1; q < 7; ++q) acc[q] = 0.0;
    }
#pragma unroll
    for (int p = 0; p < LM; ++p) {
      T Sal = T(0), Sc = T(0), Sbx = T(0), Sby = T(0), Sbz = T(0);
#pragma unroll
      for (int q = 0; q < LM; ++q) {
        if (q == p) continue;
        const int u = p < q ? pair_index<LM>(p, q) : pair_index<LM>(q, p);
        Sal += dz[q] * (dfc[p] * g[u]);
        Sc += beta[u] * (TB_ROW_RECOS ? ex[p] * ex[q] + ey[p] * ey[q] + ez[p] * ez[q] : cs[u]);
        Sbx += beta[u] * ex[q];
        Sby += beta[u] * ey[q];
        Sbz += beta[u] * ez[q];
      }
      double fx = 0.0, fy = 0.0, fz = 0.0;
      if (live[p]) {
        const T ca = dvdr[p] + Sal - Sc * inv[p];
        fx = (double)(-(ca * ex[p] + inv[p] * Sbx));
        fy = (double)(-(ca * ey[p] + inv[p] * Sby));
        fz = (double)(-(ca * ez[p] + inv[p] * Sbz));
        // virial sum d (x) f, d = r e (TB_ROW_VIR_RE: to a rounding of the displacement)
        const double dx = TB_ROW_VIR_RE ? (double)rr[p] * (double)ex[p] : d[p][0];
        const double dy = TB_ROW_VIR_RE ? (double)rr[p] * (double)ey[p] : d[p][1];
        const double dz_ = TB_ROW_VIR_RE ? (double)rr[p] * (double)ez[p] : d[p][2];
        acc[1] += dx * fx;
        acc[2] += dy * fy;
        acc[3] += dz_ * fz;
        acc[4] += dx * fy;
        acc[5] += dx * fz;
        acc[6] += dy * fz;
        fix -= fx;
        fiy -= fy;
        fiz -= fz;
        if (MODE == 0) {
          double *fj = a.forces + 3 * (int64_t)cj[p];
          atomicAdd(fj, fx);
          atomicAdd(fj + 1, fy);
          atomicAdd(fj + 2, fz);
        }
      }
      if (MODE == 1 && p < cL) {  // dead entries store zeros
        double *fb = a.fbuf + 3 * (int64_t)(co + p);
        fb[0] = fx;
        fb[1] = fy;
        fb[2] = fz;
      }
    }
    if (MODE == 0 && nlive) {
      double *fi = a.forces + 3 * (int64_t)ci;
      atomicAdd(fi, fix);
      atomicAdd(fi + 1, fiy);
      atomicAdd(fi + 2, fiz);
    }
    if (SACC) {
      s_acc[0][threadIdx.x] += e_i;
#pragma unroll
      for (int q = 1; q < 7; ++q) s_acc[q][threadIdx.x] += acc[q];
    } else {
      acc[0] += e_i;
    }
    if (a.per_atom) a.per_atom[ci] = e_i + 0.0;
  }

  // ---- stats and block partials (reduced by the finalize kernel) ----
  if (ST) {
    unsigned long long csum[6] = {c_vis, c_pk, c_lp, c_lt, c_tp, c_tt};
    if (SCNT) {
#pragma unroll
      for (int q = 0; q < 6; ++q) csum[q] = s_cnt[q][threadIdx.x];
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = warp_sum(csum[q]);
      if (lane == 0 && v) atomicAdd(&a.stats[q], v);
    }
  }
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = warp_sum(SACC ? s_acc[q][threadIdx.x] : acc[q]);
    if (lane == 0) s_red[wid][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < NWP; ++q) v += s_red[q][threadIdx.x];
    a.partials[8 * (int64_t)blockIdx.x + threadIdx.x] = v;
  }
}

}  // namespace tb
