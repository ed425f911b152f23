// tb_dnl.cuh -- kernels of the device-resident NVE loop (tb_md_run).
//
// The whole run is ONE CUDA-graph launch: a WHILE node over the steps whose
// body is kick+drift (+ the skin/2 drift reduction), the rebuild decision, an
// IF node holding the complete neighbour-list rebuild, the Tersoff kernel and
// its finalize, and kick + kinetic energy.  Every size the rebuild needs
// (list entries, row-length histogram, warp-chunk plan) lives in device memory
// (DevPlan) and every buffer has a capacity fixed before capture, so there is
// no host synchronisation inside the loop.  Capacity overflows are latched in
// DevPlan and end the loop; the host then restores the run's entry snapshot,
// regrows the capacities and replays it (tb_api.cu, tb_md_run).
//
// Semantics follow run_nve / velocity_verlet_step (system.py:355-380, 427-460)
// and needs_rebuild (neighbor.py:220-229) exactly as tb_md_step does.
#pragma once
#include "tb_warp.cuh"

namespace tb {

enum : int {
  OVF_ENTRIES = 1,  // more list entries than the capacity
  OVF_ROW = 2,      // a row longer than 32 entries (warp kernel not applicable)
  OVF_CHUNKS = 4,   // more warp chunks than the capacity
};

struct DevPlan {
  int nchunks, n_empty;   // read by the Tersoff kernel (WArgs::dinfo)
  int entries;            // offsets[n] of the last build
  int max_row;
  int overflow;           // OVF_* bits (sticky for the run)
  int list_overflow;      // OVF_ENTRIES: the fill pass must not write
  int step, target;       // steps taken / to take in this launch
  int rebuilds;
  int lanes_used;         // sum_L L * hist[L] of the chunked rows
  int unwrapped;          // k_cell_index: a periodic coordinate outside [0, L]
  int pad;
  unsigned long long drift_bits;  // max |x - x_ref|^2 of this step (bits; r^2 >= 0)
  // loose-list runs (tb_md_run, TB_OPT_MD_LOOSE_SKIN): the reference's own
  // trigger measured against the positions of its last (logical) rebuild
  unsigned long long drift_log_bits;
  int log_now;            // this step is one of the reference's rebuilds
  int pad2;
  int hist[34];
  int bucket_start[34], chunk_base[34];
  int cursor[34];         // k_bucket_rows
};

// v += half F/m ; x += dt v ; wrap ; max drift^2 against the list snapshot
// (k_kick_drift + k_max_drift fused, same arithmetic)
__global__ void __launch_bounds__(256) k_md_kick_drift(int n, double *__restrict__ pos,
                                                       double *__restrict__ vel,
                                                       const double *__restrict__ f,
                                                       const double *__restrict__ mass,
                                                       const double *__restrict__ ref, double half,
                                                       double dt, Box box,
                                                       DevPlan *__restrict__ plan,
                                                       const double *__restrict__ ref_log) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = 0, best_log = 0;
  if (i < n) {
    const double m = mass[i];
    double x[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t k = 3 * (int64_t)i + ax;
      const double v = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, f[k]), m));
      vel[k] = v;
      double xx = __dadd_rn(pos[k], __dmul_rn(dt, v));
      if (box.per[ax]) xx = np_remainder(xx, box.L[ax]);
      pos[k] = xx;
      x[ax] = xx;
    }
    double r[3], d[3];
    load3(ref, i, r);
    best = __double_as_longlong(disp_r2(r, x, box, d));
    if (ref_log) {
      load3(ref_log, i, r);
      best_log = __double_as_longlong(disp_r2(r, x, box, d));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_down_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
    v = __shfl_down_sync(0xffffffffu, best_log, o);
    best_log = v > best_log ? v : best_log;
  }
  if ((threadIdx.x & 31) == 0 && best) atomicMax(&plan->drift_bits, best);
  if ((threadIdx.x & 31) == 0 && best_log) atomicMax(&plan->drift_log_bits, best_log);
}

// rebuild decision for this step (skin/2 trigger or the fixed cadence).
// loose (> 0): the list was built with skin + delta; the reference's rebuild
// (counted, and its positions kept as the trigger's new reference) follows its
// own rule against ref_log, while the list itself is rebuilt only when some atom
// moved more than (skin + delta)/2 since the list's build -- until then every
// pair within r_cut is still in it, and the evaluation re-tests r < r_cut
__global__ void k_md_decide(DevPlan *__restrict__ plan, double half_skin2, int rebuild_every,
                            cudaGraphConditionalHandle h_rebuild, int loose,
                            double half_loose2) {
  const double d2 = __longlong_as_double((long long)plan->drift_bits);
  const int step = plan->step + 1;
  plan->step = step;
  plan->drift_bits = 0ull;
  if (!loose) {
    const bool need = d2 > half_skin2 || (rebuild_every > 0 && step % rebuild_every == 0);
    if (need) plan->rebuilds += 1;
    cudaGraphSetConditional(h_rebuild, need ? 1u : 0u);
    return;
  }
  const double dl2 = __longlong_as_double((long long)plan->drift_log_bits);
  plan->drift_log_bits = 0ull;
  const bool logical = dl2 > half_skin2 || (rebuild_every > 0 && step % rebuild_every == 0);
  plan->log_now = logical ? 1 : 0;
  if (logical) plan->rebuilds += 1;
  cudaGraphSetConditional(h_rebuild, d2 > half_loose2 ? 1u : 0u);
}

// reset the per-build counters (full) or only the histogram (filter pass)
__global__ void k_plan_reset(DevPlan *__restrict__ plan, int full) {
  const int t = threadIdx.x;
  if (t < 34) {
    plan->hist[t] = 0;
    plan->cursor[t] = 0;
  }
  if (full && t == 0) {
    plan->max_row = 0;
    plan->unwrapped = 0;
  }
}

// chunk plan from the row-length histogram (one thread): buckets of rows of
// equal length, floor(32/L) rows per warp chunk (same plan as build_chunks)
// (offsets = the list's CSR offsets: entries checked against the capacity;
//  nullptr for the filtered rows, which are a subset of the list)
__global__ void k_plan(DevPlan *__restrict__ plan, const int *__restrict__ offsets, int n,
                       int entries_cap, int chunks_cap, const int *__restrict__ go = nullptr) {
  if (threadIdx.x != 0 || (go && !*go)) return;
  int ovf = plan->overflow;
  if (offsets) {
    const int entries = offsets[n];
    plan->entries = entries;
    if (entries > entries_cap) {
      ovf |= OVF_ENTRIES;
      plan->list_overflow = 1;
    }
  }
  if (plan->max_row > 32) ovf |= OVF_ROW;
  int start = plan->hist[0], chunks = 0, used = 0;
  plan->bucket_start[0] = 0;
  plan->chunk_base[0] = 0;
  for (int L = 1; L <= 32; ++L) {
    plan->bucket_start[L] = start;
    plan->chunk_base[L] = chunks;
    start += plan->hist[L];
    used += L * plan->hist[L];
    chunks += (plan->hist[L] + 32 / L - 1) / (32 / L);
  }
  plan->bucket_start[33] = start;
  plan->chunk_base[33] = chunks;
  if (chunks > chunks_cap) ovf |= OVF_CHUNKS;
  plan->overflow = ovf;
  plan->nchunks = ovf ? 0 : chunks;
  plan->n_empty = ovf ? 0 : plan->hist[0];
  plan->lanes_used = used;
}

// after an entries overflow every row is made empty, so all later readers of
// offsets stay inside the buffers
__global__ void k_guard_offsets(int n, const DevPlan *__restrict__ plan, int *__restrict__ offsets) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n && plan->list_overflow) offsets[i] = 0;
}

// rows bucketed by length with one atomic cursor per length (atomic-scatter
// runs only: the order inside a bucket is arbitrary; gather runs keep the
// stable radix sort so that their energy sums are reproducible)
__global__ void k_bucket_rows(int n, const int *__restrict__ row_len, DevPlan *__restrict__ plan,
                              int *__restrict__ sorted_atoms) {
  __shared__ int s_cnt[34], s_base[34];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x < 34) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int L = -1, slot = 0;
  if (i < n) {
    L = min(row_len[i], 33);
    slot = atomicAdd(s_cnt + L, 1);  // block-local rank, one global atomic per bucket
  }
  __syncthreads();
  if (threadIdx.x < 33 && s_cnt[threadIdx.x])
    s_base[threadIdx.x] = atomicAdd(plan->cursor + threadIdx.x, s_cnt[threadIdx.x]);
  __syncthreads();
  if (L >= 0 && L <= 32) sorted_atoms[plan->bucket_start[L] + s_base[L] + slot] = i;
}

// one warp per chunk, grid-stride (any grid): lane -> {entry, i, j, L}; the
// plan's bucket tables are staged in shared memory once per block
__global__ void __launch_bounds__(256) k_fill_lanes_dev(const DevPlan *__restrict__ plan,
                                 const int *__restrict__ sorted_atoms,
                                 const int *__restrict__ offsets, const int *__restrict__ centry,
                                 const int *__restrict__ nbr, int4 *__restrict__ lanes) {
  __shared__ int s_base[34], s_start[34], s_hist[34];
  if (threadIdx.x < 34) {
    s_base[threadIdx.x] = plan->chunk_base[threadIdx.x];
    s_start[threadIdx.x] = plan->bucket_start[threadIdx.x];
    s_hist[threadIdx.x] = plan->hist[threadIdx.x];
  }
  __syncthreads();
  const int nch = plan->nchunks, lane = threadIdx.x & 31;
  for (int c = blockIdx.x * 8 + (threadIdx.x >> 5); c < nch; c += gridDim.x * 8) {
    int L = 1;
    while (L < 32 && s_base[L + 1] <= c) ++L;
    const int rpc = 32 / L;
    const int row = (c - s_base[L]) * rpc + lane / L;
    int4 v = make_int4(-1, 0, 0, L);
    if (lane < rpc * L && row < s_hist[L]) {
      const int atom = sorted_atoms[s_start[L] + row];
      const int k = offsets[atom] + lane % L;
      const int e = centry ? centry[k] : k;
      v = make_int4(e, atom, nbr[e], L | ((lane % L) << 8));
    }
    lanes[32 * (int64_t)c + lane] = v;
  }
}

// live rows for the repack (tb_api.cu live_repack): the entries of row i
// with r^2 < rc2 at the current positions, in row order, compacted to the
// start of the row's slots.  G lanes per row test G entries at a time (one
// round of dependent gathers instead of one per entry); also the non-finite
// check for every atom (a non-finite atom's rows come out empty, so the
// Tersoff kernel would never see it)
template <bool FILT, int G>
__global__ void __launch_bounds__(256) k_live_rows(int n, const double *__restrict__ pos, Box box,
                                                   double rc2, const int *__restrict__ start,
                                                   const int *__restrict__ crow,
                                                   const int *__restrict__ centry,
                                                   const int *__restrict__ jlist,
                                                   int *__restrict__ llen, int *__restrict__ lrow,
                                                   int *__restrict__ lrowj,
                                                   ErrFlags *__restrict__ err,
                                                   const int *__restrict__ go = nullptr,
                                                   double *__restrict__ lref = nullptr) {
  static_assert(G > 0 && G < 32 && (32 % G) == 0, "row groups tile the warp");
  if (go && !*go) return;  // margin repack still valid (live_repack)
  const int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G);
  const int lane = threadIdx.x & 31, sub = lane % G, g0 = lane - sub;
  const bool act = i < n;
  int b = 0, end = 0;
  double xi[3] = {0, 0, 0};
  if (act) {
    b = start[i];
    end = FILT ? b + crow[i] : start[i + 1];
    load3(pos, i, xi);
    if (sub == 0 && !(isfinite(xi[0]) && isfinite(xi[1]) && isfinite(xi[2])))
      atomicMin(&err->nonfinite_atom, i);
    if (lref && sub == 0) {  // positions of this repack (the next gate's drift origin)
      lref[3 * (int64_t)i] = xi[0];
      lref[3 * (int64_t)i + 1] = xi[1];
      lref[3 * (int64_t)i + 2] = xi[2];
    }
  }
  int q = 0;
  for (int k0 = b; __any_sync(0xffffffffu, act && k0 < end); k0 += G) {
    const int k = k0 + sub;
    bool lv = false;
    int e = 0, j = 0;
    if (act && k < end) {
      // jlist: the filtered entries' j (FILT, contiguous with centry) or the list's nbr
      e = FILT ? __ldg(centry + k) : k;
      j = __ldg(jlist + k);
      double xj[3], d[3];
      load3(pos, j, xj);
      lv = disp_r2(xi, xj, box, d) < rc2;
    }
    const unsigned gm = (__ballot_sync(0xffffffffu, lv) >> g0) & ((1u << G) - 1u);
    if (lv) {
      const int at = b + q + __popc(gm & ((1u << sub) - 1u));
      lrow[at] = e;
      lrowj[at] = j;
    }
    q += __popc(gm);
  }
  if (act && sub == 0) llen[i] = q;
}

// rows bucketed by live length AND written straight into their warp chunks
// (k_bucket_rows + k_fill_lanes_dev in one pass, for the live repack): the
// row taking slot s of bucket L owns lanes [(s % rpc) L, (s % rpc + 1) L) of
// chunk chunk_base[L] + s / rpc, and the owner of a chunk's last row slot (or
// of the bucket's last row) marks the chunk's remaining lanes idle
__global__ void __launch_bounds__(256) k_bucket_fill(int n, const int *__restrict__ llen,
                                                     const int *__restrict__ start,
                                                     const int *__restrict__ lrow,
                                                     const int *__restrict__ lrowj,
                                                     DevPlan *__restrict__ plan,
                                                     int *__restrict__ empty_atoms,
                                                     int4 *__restrict__ lanes,
                                                     const int *__restrict__ go = nullptr) {
  if (go && !*go) return;
  __shared__ int s_cnt[34], s_base[34];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x < 34) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int L = -1, slot = 0;
  if (i < n) {
    L = min(llen[i], 33);
    slot = atomicAdd(s_cnt + L, 1);
  }
  __syncthreads();
  if (threadIdx.x < 33 && s_cnt[threadIdx.x])
    s_base[threadIdx.x] = atomicAdd(plan->cursor + threadIdx.x, s_cnt[threadIdx.x]);
  __syncthreads();
  if (L < 0 || L > 32 || plan->overflow) return;  // (the chunk bound makes overflow impossible)
  const int s = s_base[L] + slot;
  // atoms by row length: [empty rows | L = 1 | L = 2 | ...] -- the kernels'
  // empty-row list (per-atom energy 0) and the row kernel's atom list
  empty_atoms[plan->bucket_start[L] + s] = i;
  if (L == 0) return;
  const int rpc = 32 / L, r = s % rpc;
  int4 *dst = lanes + 32 * (int64_t)(plan->chunk_base[L] + s / rpc);
  const int b = start[i];
  // lrow == nullptr: the rows are the list's own (entry = b + k, j = lrowj[b + k])
  for (int k = 0; k < L; ++k)
    dst[r * L + k] = make_int4(lrow ? lrow[b + k] : b + k, i, lrowj[b + k], L | (k << 8));
  const bool last_in_chunk = r == rpc - 1, last_in_bucket = s == plan->hist[L] - 1;
  if (last_in_chunk || last_in_bucket)
    for (int k = (r + 1) * L; k < 32; ++k) dst[k] = make_int4(-1, 0, 0, L);
}

// margin repack gate (live_repack): repack when forced (new list / filter) or
// when some atom moved more than margin/2 since the last repack; a repack
// starts from a zeroed plan (what the ungated path's memset does)
__global__ void k_repack_gate(const unsigned long long *__restrict__ drift_bits, double thr2,
                              int force, int *__restrict__ force_dev, int *__restrict__ go,
                              DevPlan *__restrict__ plan) {
  // force_dev: set by the device list rebuild inside tb_md_run's graph (the
  // host cannot know when that happens)
  __shared__ int need;
  if (threadIdx.x == 0)
    need = force || (force_dev && *force_dev) ||
           __longlong_as_double((long long)*drift_bits) > thr2;
  __syncthreads();
  if (threadIdx.x == 0) {
    *go = need;
    if (force_dev) *force_dev = 0;
  }
  if (need) {
    int *p = reinterpret_cast<int *>(plan);
    for (int k = threadIdx.x; k < (int)(sizeof(DevPlan) / sizeof(int)); k += blockDim.x) p[k] = 0;
  }
}

__global__ void k_set_flag(int *__restrict__ flag) { *flag = 1; }

// histogram of row lengths into the device plan (block-private bins)
__global__ void k_len_hist_plan(int n, const int *__restrict__ len, DevPlan *__restrict__ plan,
                                const int *__restrict__ go = nullptr) {
  if (go && !*go) return;
  __shared__ int h[34];
  if (threadIdx.x < 34) h[threadIdx.x] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(h + min(len[i], 33), 1);
  __syncthreads();
  if (threadIdx.x < 34 && h[threadIdx.x]) atomicAdd(plan->hist + threadIdx.x, h[threadIdx.x]);
}

// second half-kick fused with the kinetic-energy block partials
// FUSED (atomic scatter in tb_md_run): the forces come straight from the
// Tersoff kernel's accumulator -- copied out to f (+0.0 flush) and re-zeroed
// here, so the step needs no separate finalize pass (its E/W reduction moves
// to k_md_tail)
template <bool FUSED>
__global__ void __launch_bounds__(256) k_md_kick_ke(int n, double *__restrict__ vel,
                                                    double *__restrict__ f,
                                                    const double *__restrict__ mass, double half,
                                                    double *__restrict__ part,
                                                    double *__restrict__ facc,
                                                    const DevPlan *__restrict__ plan,
                                                    const double *__restrict__ pos,
                                                    double *__restrict__ ref_log) {
  __shared__ double s[8];
  double acc = 0.0;
  // a loose-list run keeps the positions of the reference's rebuilds
  const bool keep = ref_log && plan->log_now;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (keep) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) ref_log[3 * (int64_t)i + ax] = pos[3 * (int64_t)i + ax];
    }
    const double m = mass[i];
    double v[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t k = 3 * (int64_t)i + ax;
      double fk;
      if (FUSED) {
        fk = __ldcg(facc + k) + 0.0;
        f[k] = fk;
        facc[k] = 0.0;
      } else {
        fk = f[k];
      }
      v[ax] = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, fk), m));
      vel[k] = v[ax];
    }
    acc += m * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}

// kinetic energy -> result[7]; [E_pot, E_kin] recorded every `every` steps;
// the WHILE handle continues while steps remain and nothing overflowed
// nparts > 0 (fused step): also E and the virial from the Tersoff kernel's
// block partials (8 doubles per block), the finalize kernel's reduction
// Second half-kick of step s fused with the first half-kick + drift of step
// s + 1 (one pass over v, F, m, x instead of two; the same operations in the
// same order, so the trajectory is bit-identical to the separate kernels):
//   v1 = v + half F(s)/m          E_kin(s) partials from v1
//   [s < target]  v2 = v1 + half F(s)/m, x += dt v2, wrap, drift^2 maxima
// FUSED (atomic scatter): F comes out of the Tersoff accumulator (copied to
// f with the +0.0 flush and re-zeroed).  Loose-list runs keep x(s) in ref_log
// when step s is one of the reference's rebuilds.  Fixed grid: the KE partials
// are deterministic.
template <bool FUSED>
__global__ void __launch_bounds__(256) k_md_kick2_drift(int n, double *__restrict__ pos,
                                                        double *__restrict__ vel,
                                                        double *__restrict__ f,
                                                        const double *__restrict__ mass,
                                                        double half, double dt, Box box,
                                                        double *__restrict__ part,
                                                        double *__restrict__ facc,
                                                        DevPlan *__restrict__ plan,
                                                        const double *__restrict__ ref,
                                                        double *__restrict__ ref_log) {
  __shared__ double s[8];
  double acc = 0.0;
  unsigned long long best = 0, best_log = 0;
  const bool keep = ref_log && plan->log_now;
  const bool next = plan->step < plan->target && plan->overflow == 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double m = mass[i];
    double x[3], v[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t k = 3 * (int64_t)i + ax;
      x[ax] = pos[k];
      double fk;
      if (FUSED) {
        fk = __ldcg(facc + k) + 0.0;
        f[k] = fk;
        facc[k] = 0.0;
      } else {
        fk = f[k];
      }
      const double dv = __ddiv_rn(__dmul_rn(half, fk), m);
      v[ax] = __dadd_rn(vel[k], dv);
      if (next) {
        const double v2 = __dadd_rn(v[ax], dv);
        vel[k] = v2;
        double xx = __dadd_rn(x[ax], __dmul_rn(dt, v2));
        if (box.per[ax]) xx = np_remainder(xx, box.L[ax]);
        pos[k] = xx;
      } else {
        vel[k] = v[ax];
      }
    }
    acc += m * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    if (keep) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) ref_log[3 * (int64_t)i + ax] = x[ax];
    }
    if (next) {
      double xn[3], r[3], d[3];
      load3(pos, i, xn);
      load3(ref, i, r);
      const unsigned long long b = __double_as_longlong(disp_r2(r, xn, box, d));
      best = b > best ? b : best;
      if (ref_log) {
        load3(ref_log, i, r);
        const unsigned long long bl = __double_as_longlong(disp_r2(r, xn, box, d));
        best_log = bl > best_log ? bl : best_log;
      }
    }
  }
  acc = warp_sum(acc);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_down_sync(0xffffffffu, best, o);
    best = w > best ? w : best;
    w = __shfl_down_sync(0xffffffffu, best_log, o);
    best_log = w > best_log ? w : best_log;
  }
  if ((threadIdx.x & 31) == 0) {
    s[threadIdx.x >> 5] = acc;
    if (best) atomicMax(&plan->drift_bits, best);
    if (best_log) atomicMax(&plan->drift_log_bits, best_log);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_md_tail(int nb, const double *__restrict__ part, double scale,
                          double *__restrict__ result, DevPlan *__restrict__ plan,
                          double *__restrict__ series, int every,
                          cudaGraphConditionalHandle h_loop, int nparts,
                          const double *__restrict__ tpart) {
  __shared__ double s[256];
  __shared__ double sw[8][7];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) acc += part[b];
  if (nparts > 0) {
    double e[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nparts; b += 256)
#pragma unroll
      for (int q = 0; q < 7; ++q) e[q] += __ldcg(tpart + 8 * (int64_t)b + q);
#pragma unroll
    for (int q = 0; q < 7; ++q) e[q] = warp_sum(e[q]);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int q = 0; q < 7; ++q) sw[threadIdx.x >> 5][q] = e[q];
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  if (nparts > 0 && threadIdx.x < 7) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += sw[w][threadIdx.x];
    result[threadIdx.x] = v + 0.0;
  }
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) s[threadIdx.x] += s[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double ke = s[0] * scale;
    result[7] = ke;
    const int step = plan->step;
    if (series && every > 0 && step % every == 0) {
      series[2 * (step / every)] = result[0];
      series[2 * (step / every) + 1] = ke;
    }
    cudaGraphSetConditional(h_loop, (step < plan->target && plan->overflow == 0) ? 1u : 0u);
  }
}

}  // namespace tb
