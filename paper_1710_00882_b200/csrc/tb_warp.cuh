// tb_warp.cuh -- warp-per-chunk Tersoff kernel (K4/K5 fast path).
//
// Chunks (built with the neighbour list, k_fill_lanes / the device plan
// kernels): rows of equal length L packed floor(32/L) to a warp, so lane = one
// (i,j) skin-list entry, the L lanes of atom i are contiguous and every lane
// runs the same L-1 iterations of the k-loops.  What a lane needs from the
// other neighbours of i (unit vector, r, f_C, dzeta, V) it reads from a
// per-warp shared table the owning lanes write; the angular values of phase 1
// are cached (registers in the mixed kernel, shared memory in fp64) for
// phase 2.  Positions/species of the next chunk are gathered with cp.async
// while the current one computes.  No block barriers inside the loop.
//
//   pack   : r2 < r_cut^2 at current positions, min image (neighbor.py:330-360)
//   phase 1: zeta_ij over k, then V, dV/dr, dzeta (kernels.py:279-299,
//            potential.py:238-290)
//   phase 2: the force on neighbour a from every term centred on i -- (i,a,b)
//            with a as j and (i,b,a) with a as k -- along e_a and e_b
//   scatter: F_a += f_a (red.global.add.f64 into the context's accumulator),
//            F_i = -sum_a f_a by a segmented shuffle reduction over the row,
//            or the per-entry buffer (deterministic gather); e_i, E and the
//            virial by row / warp / block reductions.
#pragma once
#include "tb_kernels.cuh"

namespace tb {

#ifndef TB_WARP_MINB
#define TB_WARP_MINB 4
#endif
#ifndef TB_WARP_MINB_F
#define TB_WARP_MINB_F 4
#endif
// cos(theta) is NOT clamped to [-1, 1] here (the reference clamps,
// potential.py:231/256): both vectors are unit to a few ulp, so |cos| can
// exceed 1 only by rounding, g(cos) is a smooth rational function there and
// the difference is ~1e-16 relative; non-finite inputs are reported as errors
// before they could reach it.  Dropping the two selects per partner measured
// c5 fp64 2.97 -> 2.91 ms.
#ifdef TB_COS_CLAMP
#define TB_CLAMP_COS(c) c = fmin(T(1), fmax(T(-1), c))
#else
#define TB_CLAMP_COS(c) (void)0
#endif
#ifndef TB_FP64_REG
#define TB_FP64_REG 0  // fp64 kernel: energy/virial + angular cache in registers too
#endif
#ifndef TB_FP64_RC2
#define TB_FP64_RC2 1  // measured: c2 20.94 -> 20.69 us, c5 2.58 -> 2.51 ms, c4 470 -> 476 us (80 B spill)
#endif
#ifndef TB_FP64_REGACC_S2
#define TB_FP64_REGACC_S2 1  // two species too (c3 fp64 230 -> 226 us)
#endif
#ifndef TB_FP64_SHUF_E
#define TB_FP64_SHUF_E 1
#endif
#ifndef TB_FP64_REGACC
// fp64 kernel, one species: energy/virial accumulators in registers (124 regs,
// no spill since the constants moved to constant memory): c5 2.74 -> 2.62 ms,
// c2 unchanged, c4 +1.5%
#define TB_FP64_REGACC 1
#endif
constexpr int WNT = 128;  // threads per block of the warp kernel
constexpr int WPB = WNT / 32;
#ifndef TB_WNT64
#define TB_WNT64 128  // fp64 block size (see DESIGN: 96 x 6 blocks measured)
#endif
#ifndef TB_WARP_MINB64
#define TB_WARP_MINB64 4
#endif
// block shape of the warp kernel per precision
template <class T>
struct WarpCfg {
  static constexpr int nt = sizeof(T) == 8 ? TB_WNT64 : WNT;
  static constexpr int wpb = nt / 32;
  static constexpr int minb = sizeof(T) == 8 ? TB_WARP_MINB64 : TB_WARP_MINB_F;
};
constexpr int QCAP = 4;   // k-iterations whose angular values are cached
#ifndef TB_MIXED_NO_SCACHE
#define TB_MIXED_NO_SCACHE 1
#endif
#ifndef TB_FP64_NO_SCACHE
#define TB_FP64_NO_SCACHE 0
#endif
#ifndef TB_PAIR_DYN
// dynamic-length rows of the mixed one-species kernel: two partners per trip of
// the k-loops (the second predicated), so that the shared-memory loads and the
// rcp of one partner overlap the other's arithmetic (same sums, same order)
#define TB_PAIR_DYN 1
#endif
#ifndef TB_MIXED_LC8
#define TB_MIXED_LC8 0  // measured: c4 mixed -2%, c3 mixed +19%, c5 mixed +14% (code size / registers)
#endif

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
  const int4 *__restrict__ lanes;      // [nchunks*32] {entry, i, j, L | pos << 8}; entry -1 = idle lane
  const int *__restrict__ empty_atoms; // atoms with empty rows (per_atom = 0)
  int nchunks, n_empty;
  const int *__restrict__ dinfo;       // non-null: {nchunks, n_empty} in device memory (tb_md_run)
  int dskip;                           // > 0 (with dinfo): dinfo[dskip] = first chunk to run, the
                                       // shorter rows and the empty rows went to the row kernel
  int count_packed;                    // rows are the full skin rows: count zeta_visits here
  double *__restrict__ facc;           // ATOMIC: zeroed force accumulator (n,3)
};

template <bool REG>
struct WAcc {
  // energy and virial per lane: in registers for the mixed kernel (REG; its
  // L1/shared pipe is the busiest unit), in the per-lane shared slots
  // (acc[7][32]) for fp64, whose registers are spent on occupancy
  double *acc;  // &s_acc[wid][0][lane], stride 32
  double r[REG ? 7 : 1];
  unsigned long long c_vis = 0, c_pk = 0, c_lp = 0, c_tp = 0, c_lt = 0, c_tt = 0;
  __device__ __forceinline__ void add(int q, double v) {
    if (REG)
      r[q] += v;
    else
      acc[32 * q] += v;
  }
  __device__ __forceinline__ double get(int q) const { return REG ? r[q] : acc[32 * q]; }
};

// per-warp table of the lanes' neighbour data, read by the other lanes of
// the same atom row with vector shared loads (2 x LDS.128 for e_b and r_b)
template <class T> struct Vec2;
template <> struct Vec2<double> { using t = double2; };
template <> struct Vec2<float> { using t = float2; };
template <class T> struct Vec4;
template <> struct Vec4<double> { using t = double4; };
template <> struct Vec4<float> { using t = float4; };

// Mixed kernel (float): {e, r} as one float4 and, with one species,
// {f_C, delta_zeta} as one float2 -- fewer shared-memory instructions for the
// kernel whose L1/shared pipe is the bottleneck.  fp64 keeps the split
// double2 arrays (measured faster there).
template <class T>
struct WTable {
  using T2 = typename Vec2<T>::t;
  using T4 = typename Vec4<T>::t;
  static constexpr bool PACKED = sizeof(T) == 4;
  T4 er[PACKED ? 32 : 1];   // e_x, e_y, e_z, r
  T2 exy[PACKED ? 1 : 32];  // e_x, e_y
  T2 ezr[PACKED ? 1 : 32];  // e_z, r
  T2 fc[32];    // f_C(r) with the k-role entry for j-species 0 / 1; one species,
                // packed: {f_C, delta_zeta} (delta_zeta stored after phase 1)
  T dz[32];     // delta_zeta of the (i, lane) pair
  double v[32]; // V of the (i, lane) pair (row sum -> e_i)
  int sp[32];   // species of the lane's neighbour
  __device__ __forceinline__ T4 e(int k) const {
    if (PACKED) return er[k];
    T4 o;
    const T2 a = exy[k], b = ezr[k];
    o.x = a.x;
    o.y = a.y;
    o.z = b.x;
    o.w = b.y;
    return o;
  }
  __device__ __forceinline__ void set_e(int k, T x, T y, T z, T r) {
    if (PACKED) {
      T4 o;
      o.x = x;
      o.y = y;
      o.z = z;
      o.w = r;
      er[k] = o;
    } else {
      T2 a, b;
      a.x = x;
      a.y = y;
      b.x = z;
      b.y = r;
      exy[k] = a;
      ezr[k] = b;
    }
  }
  // delta_zeta of lane k: in fc[k].y for one species in the packed layout
  static constexpr bool DZ_IN_FC = PACKED;
};

// per-warp double-buffered staging of the gathered operands (cp.async)
struct WStage {
  double xi[3][32], xj[3][32];
  int si[32], sj[32];
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// issue the gathers of one chunk's operands into a stage
template <int S, bool HEAD>
__device__ __forceinline__ void stage_chunk(WStage &st, const int4 rec, const int lane,
                                            const double *__restrict__ pos,
                                            const int *__restrict__ species) {
  if (rec.x >= 0) {
    // HEAD (mixed kernel): x_i and s_i once per row (its first lane), read by
    // the row's lanes from that slot -- less staging traffic on the L1/shared
    // pipe that bounds the mixed kernel (fp64 measured faster per lane)
    const bool head = !HEAD || (rec.w >> 8) == 0;  // w = L | (position in the row << 8)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (head) cp_async8(&st.xi[q][lane], pos + 3 * (int64_t)rec.y + q);
      cp_async8(&st.xj[q][lane], pos + 3 * (int64_t)rec.z + q);
    }
    if (head) cp_async4(&st.si[lane], species + rec.y);
    if (S > 1) cp_async4(&st.sj[lane], species + rec.z);
  }
}

// One chunk: rows of length L (LC > 0: compile-time, loops fully unrolled so
// the independent k-iterations interleave; LC == 0: runtime Ldyn).
template <class T, int S, bool LAM3, int MODE, bool ST, int LC>
__device__ __forceinline__ void chunk_body(const KArgs &a, const WArgs &w, const Tables<T, S> &tab,
                                           T (*s_cache)[3][32], WTable<T> &tb, const int lane,
                                           const int4 cur, const WStage &stg, const int Ldyn,
                                           WAcc<sizeof(T) == 4 || TB_FP64_REG || ((S == 1 || TB_FP64_REGACC_S2) && TB_FP64_REGACC)> &A) {
  static_assert(S <= 2, "the warp kernel handles up to two species");
  using T2 = typename Vec2<T>::t;
  const int e = cur.x, i = cur.y, j = cur.z;
  const int L = LC > 0 ? LC : Ldyn;  // warp-uniform row length
  const bool valid = e >= 0;
  constexpr bool POW2 = LC > 0 && (LC & (LC - 1)) == 0;
  // position in the row: by mask / constant modulo for unrolled rows, else
  // from the lane record (w = L | pos << 8; no runtime division)
  const int pos = POW2 ? (lane & (LC - 1)) : (LC > 0 ? lane % LC : (cur.w >> 8));
  const int first = lane - pos;

  // ---- pack: displacement with min image, r2 < r_cut^2 ----
  double d[3] = {0, 0, 0}, r2 = 1.0;
  int si = 0, sj = 0;
  if (valid) {
    const int src_i = sizeof(T) == 4 ? first : lane;  // see stage_chunk<S, HEAD>
    const double cxi[3] = {stg.xi[0][src_i], stg.xi[1][src_i], stg.xi[2][src_i]};
    const double cxj[3] = {stg.xj[0][lane], stg.xj[1][lane], stg.xj[2][lane]};
    r2 = disp_r2(cxi, cxj, a.box, d);
    si = stg.si[src_i];
    sj = S > 1 ? stg.sj[lane] : 0;
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
  if (ST && w.count_packed && valid && pos == 0) {
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
  // |d| and 1/|d| from one rsqrt: fp64 Newton in fp64 mode; in the mixed mode
  // the potential math is fp32 anyway (kernels.py:154-165 casts r to single),
  // so one MUFU rsqrt of the fp32 r^2 (live test above stays fp64: exact pair set)
  T ex, ey, ez, ra, inva;
  if (sizeof(T) == 8) {
    double rd, invd;
    tb_sqrt_rsqrt(live ? r2 : 1.0, &rd, &invd);
    ex = (T)(d[0] * invd);
    ey = (T)(d[1] * invd);
    ez = (T)(d[2] * invd);
    ra = (T)rd;
    inva = (T)invd;
  } else {
    const float r2f = live ? (float)r2 : 1.0f;
    const float rinv = rsqrtf(r2f);
    ra = (T)(r2f * rinv);
    inva = (T)rinv;
    ex = (T)((float)d[0] * rinv);
    ey = (T)((float)d[1] * rinv);
    ez = (T)((float)d[2] * rinv);
  }
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
  {
    T2 c2;
    c2.x = fck[0];
    c2.y = fck[S > 1 ? 1 : 0];
    tb.set_e(lane, ex, ey, ez, ra);
    tb.fc[lane] = c2;
    if (S > 1) tb.sp[lane] = sj;
  }
  __syncwarp();

  // ---- phase 1: zeta (and the angular cache) ----
  // the cache of (cos, g, dg) per partner: registers for the unrolled mixed
  // kernel (compile-time indices), shared memory otherwise
  constexpr bool RC = LC > 0 && (sizeof(T) == 4 || TB_FP64_REG);
  // RC2 (fp64, one species, unrolled rows): g and dg in registers, cos
  // recomputed in phase 2 from the partner's unit vector it loads anyway
  constexpr bool RC2 = !RC && LC > 0 && S == 1 && TB_FP64_RC2;
  T rcos[RC ? QCAP : 1], rg[RC || RC2 ? QCAP : 1], rdg[RC || RC2 ? QCAP : 1];
  // dynamic-length rows of the mixed kernel: no shared-memory angular cache --
  // phase 2 recomputes g, dg (~10 FP32 ops) instead of 3 STS + 3 LDS per
  // partner, the L1/shared pipe being that kernel's bottleneck
  constexpr bool SC = !(LC == 0 && (sizeof(T) == 4 ? TB_MIXED_NO_SCACHE : TB_FP64_NO_SCACHE));
  T zeta = T(0);
  // two species with i-only angular constants: in registers for the row
  const bool ang_i = S > 1 && tab.ang_i;
  AngP<T> ai;
  if (S > 1) ai = ang_of(tab.trip[si * S * S]);
  // only live partners of the row contribute (a dead b has f_C = dzeta = 0);
  // lanes iterate their own row's live mask (the table is in shared memory,
  // so no warp-uniform trip count is needed)
  // (LC > 0: the partners are the fixed rotation pos+1..pos+L-1 and the loops
  // unroll; a dead partner has f_C = dzeta = 0 and contributes exactly 0)
  const unsigned rowmask = (L >= 32 ? 0xffffffffu : ((1u << L) - 1u)) << first;
  const unsigned partners = live ? (lmask & rowmask & ~(1u << lane)) : 0u;
  constexpr bool PAIR = TB_PAIR_DYN && LC == 0 && S == 1 && !LAM3 && sizeof(T) == 4 && !SC;
  unsigned m = partners;
  int q = 0;
  if (PAIR) {
    const TripP<T> &tp0 = tab.trip[0];
    while (m != 0) {
      const int s0 = __ffs(m) - 1;
      m &= m - 1;
      const bool h1 = m != 0;
      const int s1 = h1 ? __ffs(m) - 1 : s0;
      m &= m - 1;
      const typename Vec4<T>::t b0 = tb.e(s0), b1 = tb.e(s1);
      const T f0 = tb.fc[s0].x, f1 = h1 ? tb.fc[s1].x : T(0);
      T c0 = ex * b0.x + ey * b0.y + ez * b0.z;
      T c1 = ex * b1.x + ey * b1.y + ez * b1.z;
      TB_CLAMP_COS(c0);
      TB_CLAMP_COS(c1);
      T g0, dg0, g1, dg1;
      angular(c0, tp0, g0, dg0);
      angular(c1, tp0, g1, dg1);
      if (ST && pair_live) {
        A.c_lt += (f0 != T(0)) + (f1 != T(0));
        A.c_tt += (f0 != T(0) && f0 != T(1)) + (f1 != T(0) && f1 != T(1));
      }
      zeta += f0 * g0;  // a dead partner (f = 0) adds exactly 0
      zeta += f1 * g1;
    }
  }
#pragma unroll
  for (int it = 1; PAIR ? false : (LC > 0 ? (live && it < LC) : m != 0); ++it, ++q) {
    int src;
    if (LC > 0) {
      src = POW2 ? first + ((pos + it) & (LC - 1))
                 : first + (pos + it >= L ? pos + it - L : pos + it);
    } else {
      src = __ffs(m) - 1;
      m &= m - 1;
    }
    const typename Vec4<T>::t be = tb.e(src);
    const T2 bfc = tb.fc[src];
    const int sb = S > 1 ? tb.sp[src] : 0;
    const TripP<T> &tp = tab.trip[(si * S + sj) * S + sb];
    T cost = ex * be.x + ey * be.y + ez * be.z;
    TB_CLAMP_COS(cost);
    T g, dg;
    if (S > 1 && ang_i)
      angular(cost, ai, g, dg);
    else
      angular(cost, tp, g, dg);
    if (SC && q < QCAP) {
      if (RC) {
        rcos[q] = cost;
        rg[q] = g;
        rdg[q] = dg;
      } else if (RC2) {
        rg[q] = g;
        rdg[q] = dg;
      } else {
        s_cache[q][0][lane] = cost;
        s_cache[q][1][lane] = g;
        s_cache[q][2][lane] = dg;
      }
    }
    const T f = (S > 1 && sj == 1) ? bfc.y : bfc.x;  // f_C(r_b) with entry (i, a, b)
    if (S == 1 && !LAM3 && !ST) {
      // a dead partner (f = 0) adds exactly 0 and a dead pair's zeta is never
      // used: no branch
      zeta += f * g;
    } else if (pair_live && f != T(0)) {
      if (ST) {
        A.c_lt++;
        A.c_tt += f != T(1);
      }
      T term = f * g;
      if (LAM3) {
        T exv, darg;
        lam3_term(ra - be.w, tp, exv, darg);
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
    if (S == 1 && tab.fc_same)  // same R, D: f_C(r) of this entry is fck[0]
      pair_part_fc(ra, zeta, pp, fck[0], dfck[0], v, dvdr, dz);
    else
      pair_part(ra, zeta, pp, v, dvdr, dz);
#endif
  }
  if (S == 1 && WTable<T>::DZ_IN_FC)
    tb.fc[lane].y = dz;
  else
    tb.dz[lane] = dz;
  const double vd = (double)v;
  if (!(sizeof(T) == 4 || ((S == 1 || TB_FP64_REGACC_S2) && TB_FP64_REGACC && TB_FP64_SHUF_E))) tb.v[lane] = vd;
  __syncwarp();

  // ---- phase 2: force on this neighbour from the terms centred on i ----
  T Sal = T(0), Sc = T(0), Sbx = T(0), Sby = T(0), Sbz = T(0);
  m = partners;
  q = 0;
  if (PAIR) {
    const TripP<T> &tp0 = tab.trip[0];
    const T f_a = fck[0], df_a = dfck[0];
    while (m != 0) {
      const int s0 = __ffs(m) - 1;
      m &= m - 1;
      const bool h1 = m != 0;
      const int s1 = h1 ? __ffs(m) - 1 : s0;
      m &= m - 1;
      const typename Vec4<T>::t b0 = tb.e(s0), b1 = tb.e(s1);
      const T2 q0 = tb.fc[s0], q1 = tb.fc[s1];  // {f_C, delta_zeta} of the partner
      const T fb0 = q0.x, dzb0 = q0.y;
      const T fb1 = h1 ? q1.x : T(0), dzb1 = h1 ? q1.y : T(0);
      T c0 = ex * b0.x + ey * b0.y + ez * b0.z;
      T c1 = ex * b1.x + ey * b1.y + ez * b1.z;
      TB_CLAMP_COS(c0);
      TB_CLAMP_COS(c1);
      T g0, dg0, g1, dg1;
      angular(c0, tp0, g0, dg0);
      angular(c1, tp0, g1, dg1);
      const T al0 = dzb0 * (df_a * g0), be0 = dg0 * (dz * fb0 + dzb0 * f_a);
      const T al1 = dzb1 * (df_a * g1), be1 = dg1 * (dz * fb1 + dzb1 * f_a);
      Sal += al0;
      Sc += be0 * c0;
      Sbx += be0 * b0.x;
      Sby += be0 * b0.y;
      Sbz += be0 * b0.z;
      Sal += al1;
      Sc += be1 * c1;
      Sbx += be1 * b1.x;
      Sby += be1 * b1.y;
      Sbz += be1 * b1.z;
    }
  }
#pragma unroll
  for (int it = 1; PAIR ? false : (LC > 0 ? (live && it < LC) : m != 0); ++it, ++q) {
    int src;
    if (LC > 0) {
      src = POW2 ? first + ((pos + it) & (LC - 1))
                 : first + (pos + it >= L ? pos + it - L : pos + it);
    } else {
      src = __ffs(m) - 1;
      m &= m - 1;
    }
    const T2 bfc = tb.fc[src];
    const T dzb = (S == 1 && WTable<T>::DZ_IN_FC) ? bfc.y : tb.dz[src];
    const int sb = S > 1 ? tb.sp[src] : 0;
    const T f_b = (S > 1 && sj == 1) ? bfc.y : bfc.x;  // f_C(r_b) in (i,a,b)
    const T f_a = pick(fck, sb);                        // f_C(r_a) in (i,b,a)
    const T df_a = pick(dfck, sb);
    const bool t1 = (dz != T(0)) && (f_b != T(0));
    // f_C may round to 0 in the taper while dF_C/dr does not: test both
    const bool t2 = (dzb != T(0)) && (f_a != T(0) || df_a != T(0));
    // one species, no lam3: the (t1, t2) terms below are products with the
    // zero factors themselves, so no branch is needed
    if (!(S == 1 && !LAM3) && !(t1 || t2)) continue;
    const typename Vec4<T>::t be = tb.e(src);
    const T rb = be.w;
    T cost, g, dg;
    if (SC && q < QCAP) {
      if (RC) {
        cost = rcos[q];
        g = rg[q];
        dg = rdg[q];
      } else if (RC2) {
        cost = ex * be.x + ey * be.y + ez * be.z;  // same bits as phase 1's
        TB_CLAMP_COS(cost);
        g = rg[q];
        dg = rdg[q];
      } else {
        cost = s_cache[q][0][lane];
        g = s_cache[q][1][lane];
        dg = s_cache[q][2][lane];
      }
    } else {
      cost = ex * be.x + ey * be.y + ez * be.z;
      TB_CLAMP_COS(cost);
      if (S > 1 && ang_i)
        angular(cost, ai, g, dg);
      else
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
        if (S > 1 && !tab.gsym && !ang_i) angular(cost, tp, g2, dg2);
        if (LAM3) lam3_term(rb - ra, tp, exv, darg);
        alpha += dzb * (df_a * g2 * exv - f_a * g2 * exv * darg);
        beta += dzb * (f_a * dg2 * exv);
      }
    }
    Sal += alpha;
    Sc += beta * cost;
    Sbx += beta * be.x;
    Sby += beta * be.y;
    Sbz += beta * be.z;
  }
  double fx = 0.0, fy = 0.0, fz = 0.0;
  T tfx = T(0), tfy = T(0), tfz = T(0);
  if (live) {
    const T ca = dvdr + Sal - Sc * inva;
    tfx = -(ca * ex + inva * Sbx);
    tfy = -(ca * ey + inva * Sby);
    tfz = -(ca * ez + inva * Sbz);
    fx = (double)tfx;
    fy = (double)tfy;
    fz = (double)tfz;
    A.add(1, d[0] * fx);
    A.add(2, d[1] * fy);
    A.add(3, d[2] * fz);
    A.add(4, d[0] * fy);
    A.add(5, d[0] * fz);
    A.add(6, d[1] * fz);
  }
  // Row sums over the row's L contiguous lanes by shuffles: F_i = -sum_a f_a
  // (translation invariance of the terms on i: one set of atomics per row
  // instead of L same-address ones) and, in the mixed kernel, e_i = sum_a V_ia
  // (fp64 sums; the mixed kernel sums its fp32 force pieces in fp32 first --
  // fewer shuffles -- while fp64 keeps e_i as a row-order shared-memory sum)
  constexpr bool MIXED = sizeof(T) == 4;
  // e_i by shuffles (mixed; fp64 one species when its accumulators are in
  // registers), else a row-order sum from the shared V table
  constexpr bool SHUF_E = MIXED || ((S == 1 || TB_FP64_REGACC_S2) && TB_FP64_REGACC && TB_FP64_SHUF_E);
  double ev = SHUF_E ? vd : 0.0;
  T sx = tfx, sy = tfy, sz = tfz;
  double dsx = fx, dsy = fy, dsz = fz;
  if (LC > 0 && (LC & (LC - 1)) == 0) {
    // rows of 2^k lanes are 2^k-aligned: butterfly, every lane gets the sums
#pragma unroll
    for (int off = 1; off < LC; off <<= 1) {
      if (MODE == 0) {
        if (MIXED) {
          sx += __shfl_xor_sync(0xffffffffu, sx, off);
          sy += __shfl_xor_sync(0xffffffffu, sy, off);
          sz += __shfl_xor_sync(0xffffffffu, sz, off);
        } else {
          dsx += __shfl_xor_sync(0xffffffffu, dsx, off);
          dsy += __shfl_xor_sync(0xffffffffu, dsy, off);
          dsz += __shfl_xor_sync(0xffffffffu, dsz, off);
        }
      }
      if (SHUF_E) ev += __shfl_xor_sync(0xffffffffu, ev, off);
    }
  } else {
#pragma unroll
    for (int off = 1; off < (LC > 0 ? LC : 32); off <<= 1) {
      if (LC == 0 && off >= L) break;
      const bool in = pos + off < L;
      if (MODE == 0) {
        if (MIXED) {
          const T ox = __shfl_down_sync(0xffffffffu, sx, off);
          const T oy = __shfl_down_sync(0xffffffffu, sy, off);
          const T oz = __shfl_down_sync(0xffffffffu, sz, off);
          if (in) {
            sx += ox;
            sy += oy;
            sz += oz;
          }
        } else {
          const double ox = __shfl_down_sync(0xffffffffu, dsx, off);
          const double oy = __shfl_down_sync(0xffffffffu, dsy, off);
          const double oz = __shfl_down_sync(0xffffffffu, dsz, off);
          if (in) {
            dsx += ox;
            dsy += oy;
            dsz += oz;
          }
        }
      }
      if (SHUF_E) {
        const double ov = __shfl_down_sync(0xffffffffu, ev, off);
        if (in) ev += ov;
      }
    }
  }
  if (MODE == 0) {
    if (live) {
      double *fj = w.facc + 3 * (int64_t)j;  // facc: accumulator
      atomicAdd(fj, fx);
      atomicAdd(fj + 1, fy);
      atomicAdd(fj + 2, fz);
    }
    if (valid && pos == 0 && (lmask & rowmask)) {
      double *fi = w.facc + 3 * (int64_t)i;
      atomicAdd(fi, MIXED ? -(double)sx : -dsx);
      atomicAdd(fi + 1, MIXED ? -(double)sy : -dsy);
      atomicAdd(fi + 2, MIXED ? -(double)sz : -dsz);
    }
  } else if (valid) {  // dead entries store zeros
    double *fb = a.fbuf + 3 * (int64_t)e;
    fb[0] = fx;
    fb[1] = fy;
    fb[2] = fz;
  }
  // ---- e_i (the row's first lane) ----
  if (valid && pos == 0) {
    double se = ev;
    if (!SHUF_E) {  // row order, from the shared table
      se = 0.0;
#pragma unroll
      for (int q = 0; q < (LC > 0 ? LC : 1); ++q) se += tb.v[lane + q];
      for (int q = LC > 0 ? LC : 1; q < L; ++q) se += tb.v[lane + q];
    }
    A.add(0, se);
    if (a.per_atom) a.per_atom[i] = se + 0.0;
  }
}

template <int MODE, int NTHR>
__device__ __forceinline__ void finalize_body(int n, double *__restrict__ facc,
                                              const int *__restrict__ off,
                                              const int *__restrict__ rev,
                                              const double *__restrict__ fbuf,
                                              double *__restrict__ forces, int nparts,
                                              const double *__restrict__ partials,
                                              double *__restrict__ result,
                                              unsigned long long *__restrict__ stats_acc,
                                              unsigned long long *__restrict__ stats_out,
                                              const unsigned long long *__restrict__ err_src,
                                              unsigned long long *__restrict__ err_dst,
                                              double (*s)[7] /* [NTHR/32][7] shared scratch */) {
  // block 0 reduces the block partials (E, W) and hands out the counters; the
  // other blocks move the forces (a one-block grid does both)
  if (blockIdx.x == 0) {
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nparts; b += NTHR)
#pragma unroll
      for (int q = 0; q < 7; ++q) acc[q] += __ldcg(partials + 8 * (int64_t)b + q);
    const int lane = threadIdx.x & 31, wrp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 7; ++q) acc[q] = warp_sum(acc[q]);  // fixed order: deterministic
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 7; ++q) s[wrp][q] = acc[q];
    __syncthreads();
    if (threadIdx.x < 7) {
      double v = 0.0;
      for (int q = 0; q < NTHR / 32; ++q) v += s[q][threadIdx.x];
      result[threadIdx.x] = v + 0.0;
    }
    if (threadIdx.x < 6) {
      if (stats_out) stats_out[threadIdx.x] = __ldcg(stats_acc + threadIdx.x);
      stats_acc[threadIdx.x] = 0ull;
    }
    // error flags of this evaluation next to the result (tb_compute's one block)
    if (err_dst && threadIdx.x >= 32 && threadIdx.x < 32 + (int)(sizeof(ErrFlags) / 8))
      err_dst[threadIdx.x - 32] = __ldcg(err_src + threadIdx.x - 32);
    if (gridDim.x > 1) return;
  }
  const int nb = gridDim.x > 1 ? gridDim.x - 1 : 1;
  const int b0 = gridDim.x > 1 ? blockIdx.x - 1 : 0;
  if (MODE == 0 && !facc) return;  // forces accumulated in place (enqueue_compute)
  if (MODE == 0) {
    const int64_t m3 = 3 * (int64_t)n;
    if ((reinterpret_cast<uintptr_t>(forces) & 15) == 0) {
      // 16-byte vectors (facc is a cudaMalloc allocation; forces checked)
      const int64_t m2 = m3 >> 1;
      double2 *f2 = reinterpret_cast<double2 *>(forces);
      double2 *a2 = reinterpret_cast<double2 *>(facc);
      const double2 z = make_double2(0.0, 0.0);
      for (int64_t k = b0 * (int64_t)NTHR + threadIdx.x; k < m2; k += (int64_t)nb * NTHR) {
        double2 v = __ldcg(a2 + k);
        v.x += 0.0;
        v.y += 0.0;
        f2[k] = v;
        a2[k] = z;
      }
      if ((m3 & 1) && b0 == 0 && threadIdx.x == 0) {
        forces[m3 - 1] = __ldcg(facc + m3 - 1) + 0.0;
        facc[m3 - 1] = 0.0;
      }
    } else {
      for (int64_t k = b0 * (int64_t)NTHR + threadIdx.x; k < m3; k += (int64_t)nb * NTHR) {
        forces[k] = __ldcg(facc + k) + 0.0;
        facc[k] = 0.0;
      }
    }
  } else {
    for (int m = b0 * NTHR + threadIdx.x; m < n; m += nb * NTHR) {
      double ix = 0.0, iy = 0.0, iz = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
      for (int e = off[m]; e < off[m + 1]; ++e) {
        const double *f = fbuf + 3 * (int64_t)__ldg(rev + e);
        ix += __ldcg(f);
        iy += __ldcg(f + 1);
        iz += __ldcg(f + 2);
        const double *g = fbuf + 3 * (int64_t)e;
        sx += __ldcg(g);
        sy += __ldcg(g + 1);
        sz += __ldcg(g + 2);
      }
      forces[3 * (int64_t)m] = (ix - sx) + 0.0;
      forces[3 * (int64_t)m + 1] = (iy - sy) + 0.0;
      forces[3 * (int64_t)m + 2] = (iz - sz) + 0.0;
    }
  }
}

#ifdef TB_TRACE
// per-warp timeline (debug builds): [globaltimer start, smid, clock64 at start
// and after each of up to 12 chunks, nchunks done, globaltimer end]
__device__ unsigned long long g_trace[4096 * 16];  // last 2048 words: per-block entry/exit
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

template <class T, int S, bool LAM3, int MODE, bool ST>
__global__ void __launch_bounds__(WarpCfg<T>::nt, WarpCfg<T>::minb)
    k_tersoff_warp(const KArgs a, const WArgs w, const __grid_constant__ Tables<T, S> gtab) {
  constexpr int NT = WarpCfg<T>::nt, NW = WarpCfg<T>::wpb;
  __shared__ Tables<T, S> s_tab;
  __shared__ double s_red[NW][8];
  __shared__ T s_cache[NW][QCAP][3][32];  // cos, g, dg of (i,a,b) from phase 1
  __shared__ WStage s_stage[NW][2];         // gathered operands, double-buffered
  __shared__ double s_acc[NW][7][32];       // per-lane energy + virial
  __shared__ WTable<T> s_tb[NW];            // lanes' neighbour data (per warp)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#ifdef TB_TRACE
  if (threadIdx.x == 0) g_trace[16 * 4096 - 2 * 1024 + 2 * (blockIdx.x & 1023)] = gtimer();
#endif
  if (S > 1) {
    const int *src = reinterpret_cast<const int *>(&gtab);
    int *dst = reinterpret_cast<int *>(&s_tab);
    for (int q = threadIdx.x; q < (int)(sizeof(Tables<T, S>) / sizeof(int)); q += NT)
      dst[q] = src[q];
    __syncthreads();
  }
  const Tables<T, S> &tab = (S > 1) ? s_tab : gtab;
  int nchunks = w.nchunks, n_empty = w.n_empty;
  int cfirst = 0;
  if (w.dinfo) {
    nchunks = __ldg(w.dinfo);
    n_empty = __ldg(w.dinfo + 1);
    if (w.dskip) {
      cfirst = __ldg(w.dinfo + w.dskip);
      n_empty = 0;
    }
  }
  for (int k = blockIdx.x * NT + threadIdx.x; k < n_empty; k += gridDim.x * NT) {
    const int m = w.empty_atoms[k];
    if (a.per_atom) a.per_atom[m] = 0.0;
    const int sm = a.species[m];
    if (sm < 0 || sm >= S) atomicMin(&a.err->bad_species_atom, m);
    // (rows are validated by their first lane; an atom without a row -- e.g. a
    // non-finite position that binned nowhere -- is checked here, kernels.py:111-116)
    const double *xm = a.pos + 3 * (int64_t)m;
    if (!(isfinite(__ldg(xm)) && isfinite(__ldg(xm + 1)) && isfinite(__ldg(xm + 2))))
      atomicMin(&a.err->nonfinite_atom, m);
  }

  WAcc<sizeof(T) == 4 || TB_FP64_REG || ((S == 1 || TB_FP64_REGACC_S2) && TB_FP64_REGACC)> A;
#pragma unroll
  for (int q = 0; q < 7; ++q) s_acc[wid][q][lane] = 0.0;
  A.acc = &s_acc[wid][0][lane];
#pragma unroll
  for (int q = 0; q < (sizeof(T) == 4 || TB_FP64_REG || ((S == 1 || TB_FP64_REGACC_S2) && TB_FP64_REGACC) ? 7 : 1); ++q) A.r[q] = 0.0;

  // software pipeline over this warp's chunks: lane records in registers two
  // chunks ahead; the position/species gathers of the next chunk are issued
  // as cp.async into the other stage while this chunk computes.  Warp-major
  // chunk order: a partial last round spreads over all SMs.  (Claiming chunks
  // from a global atomic counter was measured slower: no better balance at
  // the pipeline's look-ahead, and c5 fp64 atomic mode went 2.96 -> 5.76 ms.)
  const int stride = gridDim.x * NW;
  int c = cfirst + wid * gridDim.x + blockIdx.x;
  const int4 idle = make_int4(-1, 0, 0, 1);
  int4 cur = c < nchunks ? __ldg(w.lanes + 32 * (int64_t)c + lane) : idle;
  int4 nxt = c + stride < nchunks ? __ldg(w.lanes + 32 * (int64_t)(c + stride) + lane) : idle;
  stage_chunk<S, sizeof(T) == 4>(s_stage[wid][0], cur, lane, a.pos, a.species);
  cp_async_commit();
  int buf = 0;
#ifdef TB_TRACE
  const int gw = blockIdx.x * NW + wid;
  unsigned long long *tr = g_trace + 16 * (gw & 4095);
  int ndone = 0;
  if (lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    tr[0] = gtimer();
    tr[1] = smid;
    tr[2] = clock64();
  }
#endif
  for (; c < nchunks; c += stride) {
    const int4 nx2 = c + 2 * stride < nchunks
                         ? __ldg(w.lanes + 32 * (int64_t)(c + 2 * stride) + lane)
                         : idle;
    stage_chunk<S, sizeof(T) == 4>(s_stage[wid][buf ^ 1], nxt, lane, a.pos, a.species);
    cp_async_commit();
    cp_async_wait<1>();  // this lane's gathers for the current chunk have landed
    if (sizeof(T) == 4) __syncwarp();  // ... and the row heads' x_i / s_i are visible
    const WStage &stg = s_stage[wid][buf];
    const int Ldyn = __shfl_sync(0xffffffffu, cur.w, 0) & 0xff;
    // short rows (diamond: 4): fixed rotation, unrolled; longer rows: live masks
    switch (Ldyn) {
      case 4: chunk_body<T, S, LAM3, MODE, ST, 4>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A); break;
      case 5: chunk_body<T, S, LAM3, MODE, ST, 5>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A); break;
#if TB_MIXED_LC8
      // mixed kernel: rows of 6-8 entries unrolled too (angular cache in
      // registers; fp64 spills with them)
      case 6: if (sizeof(T) == 4) { chunk_body<T, S, LAM3, MODE, ST, sizeof(T) == 4 ? 6 : 0>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A); break; }
      case 7: if (sizeof(T) == 4) { chunk_body<T, S, LAM3, MODE, ST, sizeof(T) == 4 ? 7 : 0>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A); break; }
      case 8: if (sizeof(T) == 4) { chunk_body<T, S, LAM3, MODE, ST, sizeof(T) == 4 ? 8 : 0>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A); break; }
      // fall through (fp64)
#endif
      default: chunk_body<T, S, LAM3, MODE, ST, 0>(a, w, tab, s_cache[wid], s_tb[wid], lane, cur, stg, Ldyn, A);
    }
    __syncwarp();  // the stage and the lane table are rewritten next iteration
#ifdef TB_TRACE
    ++ndone;
    if (lane == 0 && ndone <= 12) tr[2 + ndone] = clock64();
#endif
    cur = nxt;
    nxt = nx2;
    buf ^= 1;
  }
  cp_async_wait<0>();
#ifdef TB_TRACE
  if (lane == 0) {
    tr[14] = ndone;
    tr[15] = gtimer();
  }
#endif

  // ---- stats and block partials (reduced by the finalize kernel) ----
  if (ST) {
    unsigned long long cs[6] = {A.c_vis, A.c_pk, A.c_lp, A.c_lt, A.c_tp, A.c_tt};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = warp_sum(cs[q]);
      if (lane == 0 && v) atomicAdd(&a.stats[q], v);
    }
  }
  double vals[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) vals[q] = A.get(q);
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = warp_sum(vals[q]);
    if (lane == 0) s_red[wid][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) v += s_red[q][threadIdx.x];
    a.partials[8 * (int64_t)blockIdx.x + threadIdx.x] = v;
#ifdef TB_TRACE
    if (threadIdx.x == 0) g_trace[16 * 4096 - 2 * 1024 + 2 * (blockIdx.x & 1023) + 1] = gtimer();
#endif
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

// histogram of row lengths (block-private bins, one global atomic per bin)
__global__ void k_len_hist(int n, const int *__restrict__ len, int *__restrict__ hist) {
  __shared__ int h[34];
  if (threadIdx.x < 34) h[threadIdx.x] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(h + min(len[i], 33), 1);
  __syncthreads();
  if (threadIdx.x < 34 && h[threadIdx.x]) atomicAdd(hist + threadIdx.x, h[threadIdx.x]);
}

// one warp per chunk (8 chunks per 256-thread block: 1-warp blocks made the
// block scheduler the limit, config 5 1.09 ms): lane -> {entry, i, j, L}
// (entry -1: idle lane)
__global__ void __launch_bounds__(256) k_fill_lanes(const ChunkPlan plan,
                                                    const int *__restrict__ sorted_atoms,
                                                    const int *__restrict__ offsets,
                                                    const int *__restrict__ centry,
                                                    const int *__restrict__ nbr,
                                                    int4 *__restrict__ lanes, int nchunks) {
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  int L = 1;
  while (L < 32 && plan.chunk_base[L + 1] <= c) ++L;
  const int rpc = 32 / L;
  const int row = (c - plan.chunk_base[L]) * rpc + lane / L;
  int4 v = make_int4(-1, 0, 0, L);
  if (lane < rpc * L && row < plan.count[L]) {
    const int atom = sorted_atoms[plan.bucket_start[L] + row];
    const int k = offsets[atom] + lane % L;
    const int e = centry ? centry[k] : k;
    v = make_int4(e, atom, nbr[e], L | ((lane % L) << 8));  // w = L | position << 8
  }
  lanes[32 * (int64_t)c + lane] = v;
}

struct NeedTable {
  float need2[16];  // (need(si,sj) + skin)^2, [si*4 + sj]
};

// species-pair compute filter over the full rows at the build positions
template <bool FILL>
__global__ void k_filter_rows(int n, const double *__restrict__ ref, const int *__restrict__ species,
                              int S, NeedTable nt, Box box, const int *__restrict__ offsets,
                              const int *__restrict__ nbr, int *__restrict__ crow,
                              const int *__restrict__ coff, int *__restrict__ centry,
                              int *__restrict__ fnbr = nullptr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int si = species[i];
  si = (si < 0 || si >= S) ? 0 : si;
  double xi[3];
  load3(ref, i, xi);
  int cnt = 0;
  const int base = FILL ? coff[i] : 0;
  for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
    const int j = nbr[e];
    int sj = species[j];
    sj = (sj < 0 || sj >= S) ? 0 : sj;
    double xj[3], d[3];
    load3(ref, j, xj);
    if (disp_r2(xi, xj, box, d) < (double)nt.need2[si * 4 + sj]) {
      if (FILL) {
        centry[base + cnt] = e;
        if (fnbr) fnbr[base + cnt] = j;  // j of the filtered entry (live repack)
      }
      ++cnt;
    }
  }
  if (!FILL) crow[i] = cnt;
}

// zeta_visits / packed pairs over the FULL skin rows (needed when the warp
// chunks only hold the filtered entries): sum_i n_i^2 with n_i = #(r < r_cut)
__global__ void k_pack_stats(int n, const double *__restrict__ pos, Box box, double rc2,
                             const int *__restrict__ offsets, const int *__restrict__ nbr,
                             unsigned long long *__restrict__ stats) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (i < n) {
    double xi[3];
    load3(pos, i, xi);
    for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
      double xj[3], d[3];
      load3(pos, nbr[e], xj);
      c += disp_r2(xi, xj, box, d) < rc2;
    }
  }
  unsigned long long sq = warp_sum(c * c), pk = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && pk) {
    atomicAdd(stats, sq);
    atomicAdd(stats + 1, pk);
  }
}

// ---------------------------------------------------------------------------
// finalize: forces out of the accumulator (or the deterministic gather),
// block partials -> [E, W6], stats out; leaves accumulators zeroed
// ---------------------------------------------------------------------------

template <int MODE>
__global__ void __launch_bounds__(256) k_finalize(int n, double *__restrict__ facc, const int *__restrict__ off,
                           const int *__restrict__ rev, const double *__restrict__ fbuf,
                           double *__restrict__ forces, int nparts,
                           const double *__restrict__ partials, double *__restrict__ result,
                           unsigned long long *__restrict__ stats_acc,
                           unsigned long long *__restrict__ stats_out,
                           const unsigned long long *__restrict__ err_src,
                           unsigned long long *__restrict__ err_dst) {
  __shared__ double s[256 / 32][7];
  finalize_body<MODE, 256>(n, facc, off, rev, fbuf, forces, nparts, partials, result, stats_acc,
                           stats_out, err_src, err_dst, s);
}

}  // namespace tb
