// tb_dd.cuh -- slab domain decomposition kernels (BASELINE north_star (4),
// SURVEY.md 8(e)).  One slab of whole cell columns along x per rank; the
// reference has no decomposition, the parity target is the
// single-domain evaluation / NVE run.
//
// Local arrays are [owned | ghosts-from-left | ghosts-from-right]; ghosts keep
// their unshifted coordinates (every displacement is the global-box minimum
// image, so each owned row, its displacement bits and its energy terms equal
// the single-domain ones).  Messages between neighbour ranks are flat double
// rows in one send buffer [to-left | to-right]:
//   migration  9 doubles  x y z vx vy vz m species id
//   ghost meta 2 doubles  id species
//   positions  3 doubles  (forward halo, every evaluation)
//   forces     3 doubles  (reverse halo, every evaluation: ghost forces back)
// The caller moves the bytes (torch.distributed / NCCL P2P over NVLink); these
// kernels pack, unpack and integrate.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tb_kernels.cuh"

namespace tb {

struct Slab {
  double L;      // x period
  double width;  // column width L / ncx (the neighbour grid's x cells)
  int ncx;       // columns
  int nranks, rank, left, right;
  int c_lo, c_hi;  // this rank's columns [c_lo, c_hi]
};

// x column of a coordinate: the neighbour grid's x cell (cell_coords, origin 0,
// np.remainder wrap, floor of the IEEE quotient, clip) -- same owner on every
// rank and in the single-domain build
__device__ __forceinline__ int slab_column(double x, const Slab &s) {
  x = np_remainder(x, s.L);
  double f = floor(__ddiv_rn(x, s.width));
  long long v = (long long)f;
  v = v < 0 ? 0 : v;
  v = v > s.ncx - 1 ? s.ncx - 1 : v;
  return (int)v;
}

// owner of column c: bounds b_r = floor(r * ncx / nranks), owner = max r, b_r <= c
__device__ __forceinline__ int slab_owner(int c, const Slab &s) {
  int r = (int)(((long long)c * s.nranks) / s.ncx);
  while (r + 1 < s.nranks && ((long long)(r + 1) * s.ncx) / s.nranks <= c) ++r;
  while (r > 0 && ((long long)r * s.ncx) / s.nranks > c) --r;
  return r;
}

// migration class of every owned atom: 0 stays, 1 to the left rank, 2 to the
// right rank (with two ranks left == right: class 1), 3 farther (error)
__global__ void k_dd_classify(int n, const double *__restrict__ pos, Slab s,
                              int *__restrict__ is_keep, int *__restrict__ is_left,
                              int *__restrict__ is_right, int *__restrict__ stray) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int o = slab_owner(slab_column(pos[3 * (int64_t)i], s), s);
  const int k = o == s.rank ? 0 : (o == s.left ? 1 : (o == s.right ? 2 : 3));
  is_keep[i] = k == 0;
  is_left[i] = k == 1;
  is_right[i] = k == 2;
  if (k == 3) atomicMin(stray, i);
}

// send lists of the halo: owned atoms in the first / last column
__global__ void k_dd_edge_flags(int n, const double *__restrict__ pos, Slab s,
                                int *__restrict__ first_col, int *__restrict__ last_col) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = slab_column(pos[3 * (int64_t)i], s);
  first_col[i] = c == s.c_lo;
  last_col[i] = c == s.c_hi;
}

// out[scan[i]] = i for flagged i (stable compaction after an exclusive scan)
__global__ void k_dd_compact(int n, const int *__restrict__ flag, const int *__restrict__ scan,
                             int *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[scan[i]] = i;
}

__global__ void k_dd_pack_migrants(int m, const int *__restrict__ idx,
                                   const double *__restrict__ pos, const double *__restrict__ vel,
                                   const double *__restrict__ mass, const int *__restrict__ sp,
                                   const long long *__restrict__ ids, double *__restrict__ rows) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t i = idx[k];
  double *r = rows + 9 * (int64_t)k;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    r[ax] = pos[3 * i + ax];
    r[3 + ax] = vel[3 * i + ax];
  }
  r[6] = mass[i];
  r[7] = (double)sp[i];
  r[8] = (double)ids[i];
}

// new owned arrays: kept atoms gathered in order, then the received rows
__global__ void k_dd_gather_kept(int m, const int *__restrict__ idx,
                                 const double *__restrict__ pos, const double *__restrict__ vel,
                                 const double *__restrict__ mass, const int *__restrict__ sp,
                                 const long long *__restrict__ ids, double *__restrict__ npos,
                                 double *__restrict__ nvel, double *__restrict__ nmass,
                                 int *__restrict__ nsp, long long *__restrict__ nids) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t i = idx[k];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    npos[3 * (int64_t)k + ax] = pos[3 * i + ax];
    nvel[3 * (int64_t)k + ax] = vel[3 * i + ax];
  }
  nmass[k] = mass[i];
  nsp[k] = sp[i];
  nids[k] = ids[i];
}

__global__ void k_dd_append_rows(int m, int at, const double *__restrict__ rows,
                                 double *__restrict__ pos, double *__restrict__ vel,
                                 double *__restrict__ mass, int *__restrict__ sp,
                                 long long *__restrict__ ids) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const double *r = rows + 9 * (int64_t)k;
  const int64_t i = at + k;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    pos[3 * i + ax] = r[ax];
    vel[3 * i + ax] = r[3 + ax];
  }
  mass[i] = r[6];
  sp[i] = (int)r[7];
  ids[i] = (long long)r[8];
}

// ghost meta rows [id, species] out / in
__global__ void k_dd_pack_meta(int m, const int *__restrict__ idx, const int *__restrict__ sp,
                               const long long *__restrict__ ids, double *__restrict__ rows) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int i = idx[k];
  rows[2 * (int64_t)k] = (double)ids[i];
  rows[2 * (int64_t)k + 1] = (double)sp[i];
}

__global__ void k_dd_unpack_meta(int m, int at, const double *__restrict__ rows,
                                 int *__restrict__ sp, long long *__restrict__ ids) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  ids[at + k] = (long long)rows[2 * (int64_t)k];
  sp[at + k] = (int)rows[2 * (int64_t)k + 1];
}

// forward halo: positions of the send lists, 3 doubles per row
__global__ void k_dd_pack_pos(int m, const int *__restrict__ idx, const double *__restrict__ pos,
                              double *__restrict__ rows) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * m) return;
  const int k = t / 3, ax = t - 3 * k;
  rows[t] = pos[3 * (int64_t)idx[k] + ax];
}

// reverse halo: forces on my send-list atoms computed by the neighbours
// (their ghosts) added to mine.  Each owned atom is in at most one send list,
// so the adds are race-free and deterministic.
__global__ void k_dd_reverse_add(int m, const int *__restrict__ idx,
                                 const double *__restrict__ rows, double *__restrict__ f) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * m) return;
  const int k = t / 3, ax = t - 3 * k;
  double *p = f + 3 * (int64_t)idx[k] + ax;
  *p = __dadd_rn(*p, rows[t]);
}

// velocity Verlet on the owned atoms (system.py:355-380 arithmetic, as
// k_kick_drift) + max min-image drift^2 against the list's reference
// positions (neighbor.py:220-229) -> drift2 (bits of a non-negative double)
__global__ void k_dd_kick_drift(int n, double *__restrict__ pos, double *__restrict__ vel,
                                const double *__restrict__ f, const double *__restrict__ mass,
                                const double *__restrict__ ref, double half, double dt, Box box,
                                unsigned long long *__restrict__ drift2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long key = 0;
  if (i < n) {
    const double m = mass[i];
    double x[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t k = 3 * (int64_t)i + ax;
      const double v = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, f[k]), m));
      vel[k] = v;
      double xa = __dadd_rn(pos[k], __dmul_rn(dt, v));
      if (box.per[ax]) xa = np_remainder(xa, box.L[ax]);
      pos[k] = xa;
      x[ax] = xa;
    }
    double r0[3], d[3];
    load3(ref, i, r0);
    key = (unsigned long long)__double_as_longlong(disp_r2(r0, x, box, d));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_down_sync(0xffffffffu, key, o);
    key = v > key ? v : key;
  }
  if ((threadIdx.x & 31) == 0 && key) atomicMax(drift2, key);
}

// second half-kick + per-block m v^2 partial sums (fixed grid: deterministic)
__global__ void k_dd_kick_ke(int n, double *__restrict__ vel, const double *__restrict__ f,
                             const double *__restrict__ mass, double half,
                             double *__restrict__ part) {
  __shared__ double s[8];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double m = mass[i];
    double v2 = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t k = 3 * (int64_t)i + ax;
      const double v = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, f[k]), m));
      vel[k] = v;
      v2 = ax == 0 ? v * v : v2 + v * v;
    }
    acc += m * v2;
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

}  // namespace tb
