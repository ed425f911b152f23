// tb_kernels.cuh -- sm_100a kernels of the Tersoff hot path.
//
//   K1  k_bounds / k_cell_index / k_cell_fill   cell binning   (neighbor.py:46-96)
//   K2  k_nl_count / k_nl_fill / k_nl_reverse   Verlet list    (neighbor.py:104-217)
//   K3  k_max_drift                              skin/2 trigger (neighbor.py:220-229)
//   K4/5 k_tersoff<T,S,LAM3,MODE>                pack + E/F/virial (kernels.py:250-315,
//                                                neighbor.py:330-360, potential.py:167-290)
//   K6/7 k_reduce_partials, k_force_gather       deterministic reductions (kernels.py:134-151)
//   K8  k_kick_drift / k_kick                    velocity Verlet (system.py:355-380)
//
// All neighbour-list arithmetic that decides pair membership is done with
// explicitly rounded fp64 intrinsics (no FMA contraction) so the pair set is
// bit-identical to the reference's numpy evaluation.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "tb_math.cuh"

namespace tb {

constexpr int NT = 128;          // threads per Tersoff block (4 warps)
constexpr int NW = NT / 32;
constexpr int SLOT_CAP = 512;    // skin-list entries staged per Tersoff block

struct Box {
  double L[3], invL[3];
  int per[3];
};

struct ErrFlags {
  int nonfinite_atom;   // atomicMin, INT_MAX = none
  int bad_species_atom; // atomicMin, INT_MAX = none
  unsigned long long coinc_key;  // (r2 hi32 << 32) | entry, ~0 = none
  int overflow;         // tile staging overflow (internal error)
  int stale_filter;     // species differ from those the species-pair filter was built for
};

// ---------------------------------------------------------------------------
// exact fp64 helpers
// ---------------------------------------------------------------------------

// numpy np.remainder (npy_divmod): coords %= L (neighbor.py:84-86),
// SimulationBox.wrap (system.py:41-46)
__device__ __forceinline__ double np_remainder(double a, double b) {
  double mod = fmod(a, b);
  if (mod != 0.0) {
    if ((b < 0.0) != (mod < 0.0)) mod = __dadd_rn(mod, b);
  } else {
    mod = copysign(0.0, b);
  }
  return mod;
}

// min_image on one axis (neighbor.py:36-43): d - L * rint(d / L).  d*invL
// selects the same integer as the correctly rounded d/L except within a few
// ulp of a half-integer; there the exact quotient is taken.
__device__ __noinline__ double rint_quotient_exact(double d, double L) {
  return rint(__ddiv_rn(d, L));  // out of line: never speculated into the hot path
}

__device__ __forceinline__ double min_image(double d, double L, double invL) {
  double y = __dmul_rn(d, invL);
  double q = rint(y);
  if (__builtin_expect(0.5 - fabs(y - q) < 1e-9, 0)) q = rint_quotient_exact(d, L);
  return __dsub_rn(d, __dmul_rn(L, q));
}

// displacement x_j - x_i with min image and r2 = (dx*dx + dy*dy) + dz*dz.
// Same arithmetic as min_image per axis; the all-periodic box (one uniform
// branch) tests the three near-half-integer cases together so that the common
// path has a single rarely-taken branch.
__device__ __forceinline__ double disp_r2(const double *xi, const double *xj, const Box &b,
                                          double d[3]) {
  if (b.per[0] & b.per[1] & b.per[2]) {
    double v[3], q[3];
    bool near = false;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      v[ax] = __dsub_rn(xj[ax], xi[ax]);
      const double y = __dmul_rn(v[ax], b.invL[ax]);
      q[ax] = rint(y);
      near |= 0.5 - fabs(y - q[ax]) < 1e-9;
    }
    if (__builtin_expect(near, 0)) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double y = __dmul_rn(v[ax], b.invL[ax]);
        if (0.5 - fabs(y - q[ax]) < 1e-9) q[ax] = rint_quotient_exact(v[ax], b.L[ax]);
      }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) d[ax] = __dsub_rn(v[ax], __dmul_rn(b.L[ax], q[ax]));
  } else {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      double v = __dsub_rn(xj[ax], xi[ax]);
      d[ax] = b.per[ax] ? min_image(v, b.L[ax], b.invL[ax]) : v;
    }
  }
  return __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                   __dmul_rn(d[2], d[2]));
}

__device__ __forceinline__ void load3(const double *__restrict__ p, int64_t i, double o[3]) {
  o[0] = __ldg(p + 3 * i);
  o[1] = __ldg(p + 3 * i + 1);
  o[2] = __ldg(p + 3 * i + 2);
}

// ---------------------------------------------------------------------------
// K1: cell binning (neighbor.py:54-96)
// ---------------------------------------------------------------------------

struct Grid {
  int nc[3];
  double origin[3], width[3];
  Box box;
  // >= 1: every periodic axis has >= 4 cells wider than the build cutoff, so
  // a candidate's minimum image is the one its stencil cell implies (the list
  // scan then skips the per-candidate rint); 2: and every axis is periodic
  // (set by the host build)
  int stencil_image;
};

// per-axis min/max of positions for free axes (neighbor.py:71-76)
__global__ void k_bounds(int64_t n, const double *__restrict__ pos,
                         unsigned long long *__restrict__ out /* 6: min xyz, max xyz as ordered bits */) {
  // order-preserving map of doubles to uint64 for atomicMin/Max
  auto key = [](double v) {
    unsigned long long u = __double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
  };
  unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      unsigned long long k = key(pos[3 * i + ax]);
      mn[ax] = k < mn[ax] ? k : mn[ax];
      mx[ax] = k > mx[ax] ? k : mx[ax];
    }
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long a = __shfl_down_sync(0xffffffffu, mn[ax], o);
      unsigned long long b = __shfl_down_sync(0xffffffffu, mx[ax], o);
      mn[ax] = a < mn[ax] ? a : mn[ax];
      mx[ax] = b > mx[ax] ? b : mx[ax];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(out + ax, mn[ax]);
      atomicMax(out + 3 + ax, mx[ax]);
    }
  }
}

__device__ __forceinline__ void cell_coords(const double *p, const Grid &g, int c[3]) {
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double x = __dsub_rn(p[ax], g.origin[ax]);
    if (g.box.per[ax]) x = np_remainder(x, g.box.L[ax]);
    double f = floor(__ddiv_rn(x, g.width[ax]));
    long long v = (long long)f;
    v = v < 0 ? 0 : v;
    v = v > g.nc[ax] - 1 ? g.nc[ax] - 1 : v;
    c[ax] = (int)v;
  }
}

__global__ void k_cell_index(int n, const double *__restrict__ pos, Grid g,
                             int *__restrict__ atom_cell, int *__restrict__ cell_count,
                             int *__restrict__ unwrapped = nullptr) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  load3(pos, i, p);
  if (unwrapped) {  // a periodic coordinate outside [0, L]: images beyond +-1
    bool out = false;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) out |= g.box.per[ax] && !(p[ax] >= 0.0 && p[ax] <= g.box.L[ax]);
    if (out) atomicOr(unwrapped, 1);
  }
  int c[3];
  cell_coords(p, g, c);
  int id = (c[0] * g.nc[1] + c[1]) * g.nc[2] + c[2];
  atom_cell[i] = id;
  atomicAdd(cell_count + id, 1);
}

__global__ void k_cell_fill(int n, const int *__restrict__ atom_cell, int *__restrict__ cursor,
                            int *__restrict__ cell_atoms) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int slot = atomicAdd(cursor + atom_cell[i], 1);
  cell_atoms[slot] = i;
}

// device rebuild (tb_md_run): the counting-sort scatter and the cell-ordered
// position copy in one pass, the per-cell counts (left by k_cell_index, already
// scanned into cell_start) counted down as the cursor; the order inside a cell is
// arbitrary either way (rows are rank-sorted by j in k_nl_compact)
__global__ void k_cell_fill_gather(int n, const double *__restrict__ pos,
                                   const int *__restrict__ atom_cell,
                                   const int *__restrict__ cell_start, int *__restrict__ count,
                                   int *__restrict__ cell_atoms, double4 *__restrict__ cpos,
                                   double *__restrict__ ref) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = atom_cell[i];
  const int slot = cell_start[c] + atomicSub(count + c, 1) - 1;
  const double x = __ldg(pos + 3 * (int64_t)i), y = __ldg(pos + 3 * (int64_t)i + 1),
               z = __ldg(pos + 3 * (int64_t)i + 2);
  cell_atoms[slot] = i;
  cpos[slot] = make_double4(x, y, z, __longlong_as_double((long long)i));
  ref[3 * (int64_t)i] = x;  // the list's reference positions (needs_rebuild)
  ref[3 * (int64_t)i + 1] = y;
  ref[3 * (int64_t)i + 2] = z;
}

// ---------------------------------------------------------------------------
// K2: full Verlet list at bc (neighbor.py:104-217)
// ---------------------------------------------------------------------------

// distinct stencil cells along one axis (wraparound de-dup, neighbor.py:121-135)
__device__ __forceinline__ int stencil_axis(int c, int nc, int per, int out[3]) {
  int k = 0;
  for (int s = -1; s <= 1; ++s) {
    int q = c + s;
    if (per) {
      q = ((q % nc) + nc) % nc;
    } else if (q < 0 || q >= nc) {
      continue;
    }
    bool dup = false;
    for (int t = 0; t < k; ++t) dup |= out[t] == q;
    if (!dup) out[k++] = q;
  }
  return k;
}

// cell-sorted copy of the positions: slot -> {x, y, z, -} (one 32-byte load
// per candidate in the stencil scan, contiguous within a cell)
__global__ void k_cell_gather(int n, const double *__restrict__ pos,
                              const int *__restrict__ cell_atoms, double4 *__restrict__ cpos) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = cell_atoms[t];
  // .w carries the atom index (bit pattern) for the list scan
  cpos[t] = make_double4(__ldg(pos + 3 * (int64_t)i), __ldg(pos + 3 * (int64_t)i + 1),
                         __ldg(pos + 3 * (int64_t)i + 2), __longlong_as_double((long long)i));
}

// Stencil of cell `id`: distinct x and y cells (sx[nx], sy[ny]) and, per
// (x, y) column, the distinct z cells merged into runs of consecutive ids
// [zlo[r], zhi[r]] -- contiguous ranges of the cell-sorted arrays.  Periodic
// axes with >= 3 cells (the common case) skip the generic de-duplication.
struct Stencil {
  int sx[3], sy[3], nx, ny;
  int zlo[3], zhi[3], nr;
};

__device__ __forceinline__ void make_stencil(int id, const Grid &g, Stencil &st) {
  const int c[3] = {id / (g.nc[1] * g.nc[2]), (id / g.nc[2]) % g.nc[1], id % g.nc[2]};
  int sz[3], nz;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    int *o = ax == 0 ? st.sx : (ax == 1 ? st.sy : sz);
    int &k = ax == 0 ? st.nx : (ax == 1 ? st.ny : nz);
    const int nc = g.nc[ax], cc = c[ax];
    if (g.box.per[ax] && nc >= 3) {
      o[0] = cc == 0 ? nc - 1 : cc - 1;
      o[1] = cc;
      o[2] = cc == nc - 1 ? 0 : cc + 1;
      k = 3;
    } else {
      k = stencil_axis(cc, nc, g.box.per[ax], o);
    }
  }
  int zs[3] = {sz[0], nz > 1 ? sz[1] : 0, nz > 2 ? sz[2] : 0};
#pragma unroll
  for (int u = 1; u < 3; ++u)  // sort (<= 3 values)
#pragma unroll
    for (int v = 2; v > 0; --v)
      if (v <= u && v < nz && zs[v - 1] > zs[v]) {
        int tmp = zs[v];
        zs[v] = zs[v - 1];
        zs[v - 1] = tmp;
      }
  // merge into runs of consecutive ids (static indices only: registers)
  st.zlo[0] = st.zhi[0] = zs[0];
  st.zlo[1] = st.zhi[1] = st.zlo[2] = st.zhi[2] = 0;
  st.nr = 1;
  if (nz > 1) {
    if (zs[1] == st.zhi[0] + 1) {
      st.zhi[0] = zs[1];
    } else {
      st.zlo[1] = st.zhi[1] = zs[1];
      st.nr = 2;
    }
  }
  if (nz > 2) {
    if (st.nr == 1) {
      if (zs[2] == st.zhi[0] + 1) {
        st.zhi[0] = zs[2];
      } else {
        st.zlo[1] = st.zhi[1] = zs[2];
        st.nr = 2;
      }
    } else if (zs[2] == st.zhi[1] + 1) {
      st.zhi[1] = zs[2];
    } else {
      st.zlo[2] = st.zhi[2] = zs[2];
      st.nr = 3;
    }
  }
}

// Threads walk atoms in cell order (neighbouring threads share stencil cells,
// so candidate loads hit L1); for every (x,y) stencil pair the distinct z cells
// are merged into contiguous runs of the cell-sorted arrays.
template <bool FILL>
__global__ void __launch_bounds__(128) k_nl_scan(int n, int n_owned, const double4 *__restrict__ cpos, Grid g,
                                                 double bc2, const int *__restrict__ atom_cell,
                                                 const int *__restrict__ cell_start,
                                                 const int *__restrict__ cell_atoms,
                                                 int *__restrict__ row_count,
                                                 const int *__restrict__ offsets,
                                                 int *__restrict__ nbr, int *__restrict__ max_row,
                                                 int *__restrict__ nl_row,
                                                 const int *__restrict__ skip = nullptr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // device-resident rebuild: the list overflowed its capacity, write nothing
  if (FILL && skip && *skip) return;
  int cnt = 0;
  if (t < n && cell_atoms[t] < n_owned) {  // ghosts (i >= n_owned) get empty rows
    const int i = cell_atoms[t];
    const double4 pi = cpos[t];
    const double xi[3] = {pi.x, pi.y, pi.z};
    Stencil sc;
    make_stencil(atom_cell[i], g, sc);
    const int base = FILL ? offsets[i] : 0;
    for (int a = 0; a < sc.nx; ++a)
      for (int b = 0; b < sc.ny; ++b) {
        const int row = (sc.sx[a] * g.nc[1] + sc.sy[b]) * g.nc[2];
        for (int r = 0; r < sc.nr; ++r) {
          const int s0 = cell_start[row + sc.zlo[r]], s1 = cell_start[row + sc.zhi[r] + 1];
          for (int s = s0; s < s1; ++s) {
            if (s == t) continue;
            const double4 pj = cpos[s];
            const double xj[3] = {pj.x, pj.y, pj.z};
            double d[3];
            const double r2 = disp_r2(xi, xj, g.box, d);
            if (r2 < bc2) {
              if (FILL) nbr[base + cnt] = cell_atoms[s];
              cnt++;
            }
          }
        }
      }
    if (FILL) {
      if (nl_row)
        for (int u = 0; u < cnt; ++u) nl_row[base + u] = i;
      // rows ascending by j (neighbor.py:210-212); rows are short
      int *rowp = nbr + base;
      for (int u = 1; u < cnt; ++u) {
        int v = rowp[u];
        int w = u - 1;
        while (w >= 0 && rowp[w] > v) {
          rowp[w + 1] = rowp[w];
          --w;
        }
        rowp[w + 1] = v;
      }
    } else {
      row_count[i] = cnt;
    }
  } else if (!FILL && t < n) {
    row_count[cell_atoms[t]] = 0;
  }
  if (!FILL) {
    int m = __reduce_max_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(max_row, m);
  }
}

// Single-pass list scan for rows of <= TMPW entries: G lanes per atom (atoms
// in cell order) stride over the stencil's contiguous candidate ranges; hits
// are compacted with a group ballot into a per-atom scratch row tmp[i][TMPW]
// (candidate order).  Writes row_count (the true count, also when it exceeds
// TMPW), max_row and the row-length histogram.  k_nl_compact then sorts each
// row and writes it to its CSR slot, so the list is identical to k_nl_scan's.
constexpr int TMPW = 32;

__device__ __forceinline__ double stencil_lq(int s, int c, const Grid &g, int ax) {
  // cell s as seen from cell c: offsets beyond +-1 are wrapped neighbours
  const int dl = s - c;
  return dl > 1 ? g.box.L[ax] : (dl < -1 ? -g.box.L[ax] : 0.0);
}

// Cell-centric single-pass list scan (rows of <= TMPW entries): one warp per
// cell.  Every atom of a cell shares the cell's stencil, so the warp builds
// the stencil's candidate ranges once (lane = (x, y, z-run) of the 27-cell
// stencil, compacted and prefix-summed), flattens them, and each lane then
// tests one candidate against every atom of the cell (positions broadcast
// from L1).  Hits go to the atom's scratch row tmp[i][TMPW] in candidate
// order via full-warp ballots; k_nl_compact sorts the rows.  Outputs: the
// CSR counts (row_count incl. rows longer than TMPW), max_row, histogram.
// With g.stencil_image (and coordinates inside [0, L]) a candidate's
// displacement takes the image its stencil cell implies, d = (x_j - x_i) -
// L*q with q in {-1, 0, 1}: the same operations, hence the same bits, as the
// reference's d - L*rint(d/L) (neighbor.py:36-43) whenever the two q agree,
// which they do for every pair within the build cutoff (cells strictly wider
// than bc, >= 4 per periodic axis); pairs farther apart are rejected either
// way.  Otherwise every candidate takes the exact min_image.
__global__ void __launch_bounds__(256) k_nl_cells(int ncell, int n_owned,
                                                  const double4 *__restrict__ cpos, Grid g,
                                                  double bc2, const int *__restrict__ cell_start,
                                                  int *__restrict__ row_count,
                                                  int *__restrict__ tmp, int *__restrict__ max_row,
                                                  int *__restrict__ hist,
                                                  const int *__restrict__ unwrapped,
                                                  int cell0 = 0) {
  __shared__ int s_hist[34];
  if (threadIdx.x < 34) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const bool stencil_image = g.stencil_image && !*unwrapped;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // cells [cell0, ncell): a slab-decomposed rank scans only its own x columns
  // (its owned atoms live there; the stencil reaches the ghost columns)
  const int cell = cell0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int maxc = 0;
  if (cell < ncell) {
    const int c0 = cell_start[cell], nA = cell_start[cell + 1] - c0;
    if (nA > 0) {
      // ---- the stencil's candidate ranges, one per lane (lane < 27) ----
      int s0 = 0, len = 0;
      double lx = 0.0, ly = 0.0, lz = 0.0;
      if (g.stencil_image == 2) {
        // all axes periodic with >= 4 cells: lane = one stencil cell, offsets
        // (a-1, b-1, r-1), the image each offset implies; cells are distinct
        const int nyz = g.nc[1] * g.nc[2];
        const int ccx = cell / nyz, rem = cell - ccx * nyz;
        const int ccy = rem / g.nc[2], ccz = rem - ccy * g.nc[2];
        if (lane < 27) {
          const int a = lane / 9, b = (lane / 3) % 3, r = lane % 3;
          int x = ccx + a - 1, y = ccy + b - 1, z = ccz + r - 1;
          lx = x < 0 ? g.box.L[0] : (x >= g.nc[0] ? -g.box.L[0] : 0.0);
          ly = y < 0 ? g.box.L[1] : (y >= g.nc[1] ? -g.box.L[1] : 0.0);
          lz = z < 0 ? g.box.L[2] : (z >= g.nc[2] ? -g.box.L[2] : 0.0);
          x += x < 0 ? g.nc[0] : (x >= g.nc[0] ? -g.nc[0] : 0);
          y += y < 0 ? g.nc[1] : (y >= g.nc[1] ? -g.nc[1] : 0);
          z += z < 0 ? g.nc[2] : (z >= g.nc[2] ? -g.nc[2] : 0);
          const int id = (x * g.nc[1] + y) * g.nc[2] + z;
          s0 = cell_start[id];
          len = cell_start[id + 1] - s0;
        }
      } else {
        Stencil sc;
        make_stencil(cell, g, sc);
        const int a = lane / 9, b = (lane / 3) % 3, r = lane % 3;
        const bool on = lane < 27 && a < sc.nx && b < sc.ny && r < sc.nr;
        if (on) {
          const int cx = a == 0 ? sc.sx[0] : (a == 1 ? sc.sx[1] : sc.sx[2]);
          const int cy = b == 0 ? sc.sy[0] : (b == 1 ? sc.sy[1] : sc.sy[2]);
          const int lo = r == 0 ? sc.zlo[0] : (r == 1 ? sc.zlo[1] : sc.zlo[2]);
          const int hi = r == 0 ? sc.zhi[0] : (r == 1 ? sc.zhi[1] : sc.zhi[2]);
          const int row = (cx * g.nc[1] + cy) * g.nc[2];
          s0 = cell_start[row + lo];
          len = cell_start[row + hi + 1] - s0;
          if (stencil_image) {
            const int ccx = cell / (g.nc[1] * g.nc[2]), ccy = (cell / g.nc[2]) % g.nc[1],
                      ccz = cell % g.nc[2];
            if (g.box.per[0]) lx = stencil_lq(cx, ccx, g, 0);
            if (g.box.per[1]) ly = stencil_lq(cy, ccy, g, 1);
            if (g.box.per[2]) lz = stencil_lq(lo, ccz, g, 2);
          }
        }
      }
      // compact the non-empty ranges to lanes 0..nrg-1, prefix-sum their lengths
      const unsigned ne = __ballot_sync(0xffffffffu, len > 0);
      const int nrg = __popc(ne);
      // gather range q to lane q: lane q reads from the lane of the q-th set bit
      const unsigned fn = __fns(ne, 0, lane + 1);
      const int from = fn < 32 ? (int)fn : 0;
      s0 = __shfl_sync(0xffffffffu, s0, from);
      len = __shfl_sync(0xffffffffu, len, from);
      lx = __shfl_sync(0xffffffffu, lx, from);
      ly = __shfl_sync(0xffffffffu, ly, from);
      lz = __shfl_sync(0xffffffffu, lz, from);
      if (lane >= nrg) len = 0;
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int start = incl - len;  // first flattened candidate of range `lane`
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      // ---- atoms of the cell in batches of 32: lane k counts atom k ----
      for (int kb = 0; kb < nA; kb += 32) {
        const int nk = min(32, nA - kb);
        int cnt = 0;  // lane k: hits of atom kb + k
        for (int base = 0; base < total; base += 32) {
          const int c = base + lane;
          // range of candidate c: ranges starting at or before c
          const unsigned starts_here = __reduce_or_sync(
              0xffffffffu, (lane < nrg && len > 0 && start >= base && start < base + 32)
                               ? (1u << (start - base)) : 0u);
          const int before = __popc(__ballot_sync(0xffffffffu, lane < nrg && start < base));
          const int rid = before + __popc(starts_here & (lt | (1u << lane))) - 1;
          const int rs0 = __shfl_sync(0xffffffffu, s0, rid & 31);
          const int rst = __shfl_sync(0xffffffffu, start, rid & 31);
          const double qx = __shfl_sync(0xffffffffu, lx, rid & 31);
          const double qy = __shfl_sync(0xffffffffu, ly, rid & 31);
          const double qz = __shfl_sync(0xffffffffu, lz, rid & 31);
          const bool cand = c < total;
          const int s = rs0 + (c - rst);
          double4 pj = make_double4(0.0, 0.0, 0.0, 0.0);
          if (cand) pj = cpos[s];
          const double xj[3] = {pj.x, pj.y, pj.z};
          for (int k = 0; k < nk; ++k) {
            const int sk = c0 + kb + k;
            const double4 pk = cpos[sk];  // same address across the warp: broadcast
            const double xi[3] = {pk.x, pk.y, pk.z};
            bool hit = false;
            if (cand && s != sk) {
              double d[3];
              if (stencil_image) {
                d[0] = __dsub_rn(__dsub_rn(xj[0], xi[0]), qx);
                d[1] = __dsub_rn(__dsub_rn(xj[1], xi[1]), qy);
                d[2] = __dsub_rn(__dsub_rn(xj[2], xi[2]), qz);
                // the reference's r2 bit for bit: its rint(v/L) equals this q
                // for every pair within the build cutoff (Grid::stencil_image)
                hit = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                __dmul_rn(d[2], d[2])) < bc2;
              } else {
                hit = disp_r2(xi, xj, g.box, d) < bc2;
              }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            const int ik = (int)__double_as_longlong(pk.w);
            const int ck = __shfl_sync(0xffffffffu, cnt, k);
            if (hit && ik < n_owned) {
              const int at = ck + __popc(bal & lt);
              if (at < TMPW) tmp[(int64_t)ik * TMPW + at] = (int)__double_as_longlong(pj.w);
            }
            if (lane == k) cnt += __popc(bal);
          }
        }
        if (lane < nk) {
          const int ik = (int)__double_as_longlong(cpos[c0 + kb + lane].w);
          const int v = ik < n_owned ? cnt : 0;  // ghosts (i >= n_owned) get empty rows
          row_count[ik] = v;
          atomicAdd(s_hist + min(v, 33), 1);
          maxc = max(maxc, v);
        }
      }
    }
  }
  const int m = __reduce_max_sync(0xffffffffu, maxc);
  if (lane == 0 && m) atomicMax(max_row, m);
  __syncthreads();
  if (threadIdx.x < 34 && s_hist[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_hist[threadIdx.x]);
}

// fp32 coordinates relative to the atom's own cell origin, in cell order, with
// the atom index in .w: the 16-byte candidate record of k_nl_atoms' fp32
// pre-test (all-periodic grids)
__global__ void k_cell_rel(int n, const double4 *__restrict__ cpos,
                           const int *__restrict__ atom_cell, Grid g, float4 *__restrict__ crel) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double4 p = cpos[t];
  const int i = (int)__double_as_longlong(p.w);
  int id = __ldg(atom_cell + i);
  int c[3];
  c[2] = id % g.nc[2];
  id /= g.nc[2];
  c[1] = id % g.nc[1];
  c[0] = id / g.nc[1];
  const double x[3] = {p.x, p.y, p.z};
  float r[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double v = __dsub_rn(x[ax], g.origin[ax]);
    if (g.box.per[ax]) v = np_remainder(v, g.box.L[ax]);
    r[ax] = (float)(v - (double)c[ax] * g.width[ax]);
  }
  crel[t] = make_float4(r[0], r[1], r[2], __int_as_float(i));
}

#ifndef TB_NL_F32
#define TB_NL_F32 1
#endif
// r^2 band around bc^2 inside which the fp32 pre-test defers to the exact fp64
// test: the fp32 error of r^2 near bc^2 is ~4e-5 A^2 at bc = 3.6 A (cell-relative
// coordinates below 2 bc, a handful of roundings: ~3e-6 relative); the band is
// max(2e-3, 2e-5 bc^2)
constexpr float NL_F32_BAND = 2e-3f;

// Atom-centric single-pass scan for all-periodic grids (stencil_image == 2),
// the large-system path: one thread per atom in cell order (cpos), the 27
// stencil cells walked directly, candidates tested with the same operations
// (hence the same bits) as k_nl_cells, hits appended to the atom's scratch
// row (k_nl_compact sorts the rows by j, so the CSR is identical).  Threads
// of a warp sit in neighbouring cells and share candidate lines in L1; no
// per-cell warp setup (k_nl_cells spends its time in it at ~2 atoms per
// cell: config 5 10.8 ms).  Atoms of cells [cell0, cell1) only (slab ranks).
__global__ void __launch_bounds__(256) k_nl_atoms(int cell0, int cell1, int n_owned,
                                                  const double4 *__restrict__ cpos, Grid g,
                                                  double bc2, const int *__restrict__ cell_start,
                                                  int *__restrict__ row_count,
                                                  int *__restrict__ tmp, int *__restrict__ max_row,
                                                  int *__restrict__ hist,
                                                  const int *__restrict__ unwrapped,
                                                  const float4 *__restrict__ crel = nullptr) {
  __shared__ int s_hist[34];
  if (threadIdx.x < 34) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int t0 = __ldg(cell_start + cell0), t1 = __ldg(cell_start + cell1);
  const int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  int cnt = 0;
  if (t < t1) {
    const double4 pi = cpos[t];
    const int i = (int)__double_as_longlong(pi.w);
    if (i < n_owned) {  // ghosts (i >= n_owned) get empty rows
      const bool stencil_image = !*unwrapped;
      // this atom's cell: the last cell whose start is <= t (binary search in
      // cell_start over the cell's x column would need the cell id; cpos
      // carries only the atom id, so recompute it like cell_coords)
      int cc[3];
      {
        const double p[3] = {pi.x, pi.y, pi.z};
        cell_coords(p, g, cc);
      }
      int *row = tmp + (int64_t)i * TMPW;
      // fp32 pre-test (TB_NL_F32): a candidate's 16-byte record decides it
      // unless its fp32 r^2 is within NL_F32_BAND of bc^2 -- then the exact
      // fp64 test below runs as before.  Membership only: the list stores
      // indices, the kernels recompute every distance in fp64.
      const bool f32 = TB_NL_F32 && crel != nullptr && stencil_image;
      float4 qi = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f32) qi = crel[t];
      // (the band grows with the cutoff: the fp32 error of r^2 is relative, a few 1e-6)
      const float band = fmaxf(NL_F32_BAND, 2e-5f * (float)bc2);
      const float lo2 = (float)bc2 - band, hi2 = (float)bc2 + band;
#pragma unroll 1
      for (int a = -1; a <= 1; ++a) {
        int x = cc[0] + a;
        const double lx = x < 0 ? g.box.L[0] : (x >= g.nc[0] ? -g.box.L[0] : 0.0);
        x += x < 0 ? g.nc[0] : (x >= g.nc[0] ? -g.nc[0] : 0);
#pragma unroll 1
        for (int b = -1; b <= 1; ++b) {
          int y = cc[1] + b;
          const double ly = y < 0 ? g.box.L[1] : (y >= g.nc[1] ? -g.box.L[1] : 0.0);
          y += y < 0 ? g.nc[1] : (y >= g.nc[1] ? -g.nc[1] : 0);
          const int colbase = (x * g.nc[1] + y) * g.nc[2];
#pragma unroll
          for (int r = -1; r <= 1; ++r) {
            int z = cc[2] + r;
            const double lz = z < 0 ? g.box.L[2] : (z >= g.nc[2] ? -g.box.L[2] : 0.0);
            z += z < 0 ? g.nc[2] : (z >= g.nc[2] ? -g.nc[2] : 0);
            const int id = colbase + z;
            const int s0 = __ldg(cell_start + id), s1 = __ldg(cell_start + id + 1);
            if (f32) {
              const float sx = (float)a * (float)g.width[0] - qi.x;
              const float sy = (float)b * (float)g.width[1] - qi.y;
              const float sz = (float)r * (float)g.width[2] - qi.z;
              // hot loop: fp32 decision only; the rare borderline records of this
              // cell are remembered in a bit mask and settled after it, so the
              // exact test's code and its reconvergence stay out of the loop
              unsigned maybe = 0u;
              for (int s = s0; s < s1; ++s) {
                const float4 qj = __ldg(crel + s);
                const float dx = qj.x + sx, dy = qj.y + sy, dz = qj.z + sz;
                const float r2f = dx * dx + dy * dy + dz * dz;
                const bool hit = r2f < lo2 && s != t;
                if (r2f >= lo2 && r2f < hi2) maybe |= 1u << min(s - s0, 31);
                if (hit) {
                  if (cnt < TMPW) row[cnt] = __float_as_int(qj.w);
                  ++cnt;
                }
              }
              if (__builtin_expect(maybe != 0u, 0)) {
                for (int s = s0; s < s1; ++s) {
                  const int k = min(s - s0, 31);
                  if (!(maybe >> k & 1u)) continue;
                  // (beyond 31 records in a cell the last bit stands for all of
                  // them: re-test each in fp32 first)
                  const float4 qj = __ldg(crel + s);
                  const float dx = qj.x + sx, dy = qj.y + sy, dz = qj.z + sz;
                  const float r2f = dx * dx + dy * dy + dz * dz;
                  if (!(r2f >= lo2 && r2f < hi2)) continue;
                  const double4 pj = cpos[s];
                  const double e0 = __dsub_rn(__dsub_rn(pj.x, pi.x), lx);
                  const double e1 = __dsub_rn(__dsub_rn(pj.y, pi.y), ly);
                  const double e2 = __dsub_rn(__dsub_rn(pj.z, pi.z), lz);
                  const bool hit = __dadd_rn(__dadd_rn(__dmul_rn(e0, e0), __dmul_rn(e1, e1)),
                                             __dmul_rn(e2, e2)) < bc2;
                  if (hit && s != t) {
                    if (cnt < TMPW) row[cnt] = __float_as_int(qj.w);
                    ++cnt;
                  }
                }
              }
              continue;
            }
            for (int s = s0; s < s1; ++s) {
              if (s == t) continue;
              const double4 pj = cpos[s];
              double d[3];
              bool hit;
              if (stencil_image) {
                d[0] = __dsub_rn(__dsub_rn(pj.x, pi.x), lx);
                d[1] = __dsub_rn(__dsub_rn(pj.y, pi.y), ly);
                d[2] = __dsub_rn(__dsub_rn(pj.z, pi.z), lz);
                hit = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                __dmul_rn(d[2], d[2])) < bc2;
              } else {
                const double xi[3] = {pi.x, pi.y, pi.z}, xj[3] = {pj.x, pj.y, pj.z};
                hit = disp_r2(xi, xj, g.box, d) < bc2;
              }
              if (hit) {
                if (cnt < TMPW) row[cnt] = (int)__double_as_longlong(pj.w);
                ++cnt;
              }
            }
          }
        }
      }
      row_count[i] = cnt;
    } else {
      row_count[i] = 0;
    }
    atomicAdd(s_hist + min(cnt, 33), 1);
  }
  const int m = __reduce_max_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(max_row, m);
  __syncthreads();
  if (threadIdx.x < 34 && s_hist[threadIdx.x]) atomicAdd(hist + threadIdx.x, s_hist[threadIdx.x]);
}

// scratch rows -> CSR rows ascending by j (rank sort; j's of a row are distinct)
template <int G>
__global__ void __launch_bounds__(256) k_nl_compact(int n, const int *__restrict__ tmp,
                                                    const int *__restrict__ row_count,
                                                    const int *__restrict__ offsets,
                                                    int *__restrict__ nbr, int *__restrict__ nl_row,
                                                    const int *__restrict__ skip) {
  if (skip && *skip) return;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) / G, gl = threadIdx.x % G;
  if (i >= n) return;
  const int cnt = row_count[i];
  if (cnt > TMPW) return;  // rows this long take the two-pass scan
  const int *src = tmp + (int64_t)i * TMPW;
  const int base = offsets[i];
  for (int k = gl; k < cnt; k += G) {
    const int v = src[k];
    int rank = 0;
    for (int q = 0; q < cnt; ++q) rank += src[q] < v;
    nbr[base + rank] = v;
    if (nl_row) nl_row[base + rank] = i;
  }
}

// rev[e] = index of (j -> i) in row j for entry e = (i -> j): drives the
// deterministic gather of per-entry forces.
__global__ void k_nl_reverse(int n, const int *__restrict__ offsets, const int *__restrict__ nbr,
                             int *__restrict__ rev) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
    int j = nbr[e];
    int lo = offsets[j], hi = offsets[j + 1];
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (nbr[mid] < i) lo = mid + 1;
      else hi = mid;
    }
    rev[e] = lo;
  }
}

// Row-aligned warp chunks: chunk c = the rows whose first entry lies in
// [c*W, (c+1)*W); with W = 33 - max_row a chunk never exceeds 32 entries.
// chunk_entry[c] = first entry of chunk c (lower_bound of c*W in offsets).
__global__ void k_nl_chunks(int n, int nchunks, int W, const int *__restrict__ offsets,
                            int *__restrict__ chunk_entry) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nchunks) return;
  long long key = (long long)c * W;
  int lo = 0, hi = n;  // first row start >= key (offsets[n] = total)
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (offsets[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  chunk_entry[c] = c == nchunks ? offsets[n] : offsets[lo];
}

__global__ void k_export_i64(int m, const int *__restrict__ in, int64_t *__restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = in[i];
}

// ---------------------------------------------------------------------------
// K3: skin/2 trigger (neighbor.py:220-229)
// ---------------------------------------------------------------------------

// Species guard of the species-pair compute filter: the filter decides which
// entries get warp lanes from the species it was built for; species changed
// since (in place, same pointer) latch stale_filter instead of silently
// dropping live pairs.  4 B/atom read, coalesced.
__global__ void k_species_guard(int n, const int *__restrict__ species,
                                const int *__restrict__ built_for, ErrFlags *__restrict__ err) {
  bool diff = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    diff |= __ldg(species + i) != __ldg(built_for + i);
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) err->stale_filter = 1;
}

__global__ void k_max_drift(int n, const double *__restrict__ pos, const double *__restrict__ ref,
                            Box box, unsigned long long *__restrict__ out) {
  unsigned long long best = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a[3], b[3], d[3];
    load3(ref, i, a);
    load3(pos, i, b);
    double r2 = disp_r2(a, b, box, d);
    unsigned long long k = __double_as_longlong(r2);  // r2 >= 0: bits are ordered
    best = k > best ? k : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_down_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// ---------------------------------------------------------------------------
// block helpers
// ---------------------------------------------------------------------------

// exclusive scan of one int per thread across the NT-thread block
__device__ __forceinline__ int block_excl_scan(int v, int *s_w, int &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    int s = s_w[q];
    off += q < w ? s : 0;
    tot += s;
  }
  __syncthreads();
  total = tot;
  return off + x - v;
}

template <class V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// K4/K5: the Tersoff evaluation
// ---------------------------------------------------------------------------

struct KArgs {
  int n;
  int atoms_per_block;
  double rc2;                     // global packing cutoff^2 (neighbor.py:344)
  Box box;
  const double *__restrict__ pos;
  const int *__restrict__ species;
  const int *__restrict__ off;    // skin list CSR
  const int *__restrict__ nbr;
  double *__restrict__ forces;    // ATOMIC: (n,3) zero-initialised accumulators
  double *__restrict__ fbuf;      // GATHER: per skin-list entry force (3 doubles)
  double *__restrict__ per_atom;  // may be null
  double *__restrict__ partials;  // per block: [E, W xx yy zz xy xz yz, pad]
  unsigned long long *__restrict__ stats;  // TB_NSTATS counters
  ErrFlags *__restrict__ err;
};

// tile kernel with a runtime species count (S = 0): tables in global memory
struct DynTab {
  int nspecies;
  const void *pair, *trip;  // PairP<T>[S^2], TripP<T>[S^3]
};

template <class T, int S>
struct SmemLayout {
  // byte offsets inside dynamic shared memory for a block with C slots
  // (Sr: the species count, = S unless S = 0)
  static __host__ __device__ size_t bytes(int C, int Sr = S) {
    size_t b = 0;
    b += sizeof(Tables<T, S>);              // tables (S > 1 path reads them here)
    b = (b + 15) & ~size_t(15);
    b += sizeof(double) * 3 * C;            // s_f
    b += sizeof(T) * (4 + 2 * Sr + 3) * C;  // ex ey ez r, fc[S], dfc[S], dz, v, dvdr
    b += sizeof(int) * 2 * C;               // j, entry
    b += sizeof(short) * C;                 // local atom
    b += sizeof(unsigned char) * C;         // species of j
    b = (b + 15) & ~size_t(15);
    b += sizeof(double) * 3 * NT;           // tile positions
    b += sizeof(int) * (4 * NT + 2 + 8);    // si, roff, cnt, soff, warp scratch
    return b + 64;
  }
};

template <class T, int S, bool LAM3, int MODE>
__global__ void __launch_bounds__(NT, 3)
    k_tersoff(const KArgs a, const __grid_constant__ Tables<T, S> gtab, int C, const DynTab dyn) {
  extern __shared__ __align__(16) unsigned char smem[];
  // S = 0: any species count, tables read from global memory (L1-cached)
  const int SS = S > 0 ? S : dyn.nspecies;
  const PairP<T> *__restrict__ dpair = static_cast<const PairP<T> *>(dyn.pair);
  const TripP<T> *__restrict__ dtrip = static_cast<const TripP<T> *>(dyn.trip);
  // ---- carve shared memory (see SmemLayout) ----
  unsigned char *p = smem;
  Tables<T, S> *s_tab = reinterpret_cast<Tables<T, S> *>(p);
  p += (sizeof(Tables<T, S>) + 15) & ~size_t(15);
  double *s_fx = reinterpret_cast<double *>(p); p += sizeof(double) * C;
  double *s_fy = reinterpret_cast<double *>(p); p += sizeof(double) * C;
  double *s_fz = reinterpret_cast<double *>(p); p += sizeof(double) * C;
  T *s_ex = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_ey = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_ez = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_r = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_fc = reinterpret_cast<T *>(p); p += sizeof(T) * SS * C;   // [S][C]
  T *s_dfc = reinterpret_cast<T *>(p); p += sizeof(T) * SS * C;  // [S][C]
  T *s_dz = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_v = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  T *s_dvdr = reinterpret_cast<T *>(p); p += sizeof(T) * C;
  int *s_j = reinterpret_cast<int *>(p); p += sizeof(int) * C;
  int *s_ent = reinterpret_cast<int *>(p); p += sizeof(int) * C;
  short *s_atom = reinterpret_cast<short *>(p); p += sizeof(short) * C;
  unsigned char *s_sp = p; p += C;
  p = smem + ((p - smem + 15) & ~size_t(15));
  double *s_xi = reinterpret_cast<double *>(p); p += sizeof(double) * 3 * NT;
  int *s_si = reinterpret_cast<int *>(p); p += sizeof(int) * NT;
  int *s_roff = reinterpret_cast<int *>(p); p += sizeof(int) * (NT + 1);
  int *s_cnt = reinterpret_cast<int *>(p); p += sizeof(int) * NT;
  int *s_soff = reinterpret_cast<int *>(p); p += sizeof(int) * (NT + 1);
  int *s_w = reinterpret_cast<int *>(p); p += sizeof(int) * 8;

  const int tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int atom0 = blockIdx.x * a.atoms_per_block;
  const int na = min(a.atoms_per_block, a.n - atom0);

  const Tables<T, S> &tab = (S > 1) ? *s_tab : gtab;
  auto PAIR = [&](int k) -> const PairP<T> & { return S > 0 ? tab.pair[k] : dpair[k]; };
  auto TRIP = [&](int k) -> const TripP<T> & { return S > 0 ? tab.trip[k] : dtrip[k]; };
  if (S > 1) {
    // species-indexed tables are read with divergent indices: stage in smem
    const int *src = reinterpret_cast<const int *>(&gtab);
    int *dst = reinterpret_cast<int *>(s_tab);
    for (int q = tid; q < (int)(sizeof(Tables<T, S>) / sizeof(int)); q += NT) dst[q] = src[q];
  }

  // ---- phase 0a: tile atoms ----
  for (int t = tid; t <= na; t += NT) s_roff[t] = a.off[atom0 + t];
  if (tid < na) {
    int i = atom0 + tid;
    double x[3];
    load3(a.pos, i, x);
    s_xi[3 * tid] = x[0];
    s_xi[3 * tid + 1] = x[1];
    s_xi[3 * tid + 2] = x[2];
    if (!(isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]))) atomicMin(&a.err->nonfinite_atom, i);
    int si = a.species[i];
    if (si < 0 || si >= SS) {
      atomicMin(&a.err->bad_species_atom, i);
      si = 0;
    }
    s_si[tid] = si;
    s_cnt[tid] = 0;
  }
  __syncthreads();

  // ---- phase 0b: pack -- re-filter the skin list at current positions
  //      (pack_adjacency, neighbor.py:330-360), order-preserving compaction ----
  const int e0 = s_roff[0];
  const int ne = s_roff[na] - e0;
  if (ne > C) {
    if (tid == 0) atomicExch(&a.err->overflow, 1);
    return;
  }
  int nlive = 0;
  for (int base = 0; base < ne; base += NT) {
    int e = base + tid;
    bool live = false;
    int la = 0, j = 0;
    double d[3] = {0, 0, 0}, r2 = 0;
    if (e < ne) {
      // owning tile atom: last la with s_roff[la] <= e0 + e
      int lo = 0, hi = na;  // invariant s_roff[lo] <= e0+e < s_roff[hi]
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (s_roff[mid] <= e0 + e) lo = mid;
        else hi = mid;
      }
      la = lo;
      j = a.nbr[e0 + e];
      double xj[3];
      load3(a.pos, j, xj);
      r2 = disp_r2(&s_xi[3 * la], xj, a.box, d);
      live = r2 < a.rc2;
      if (MODE == 1 && !live) {
        double *fb = a.fbuf + 3 * (int64_t)(e0 + e);
        fb[0] = 0.0;
        fb[1] = 0.0;
        fb[2] = 0.0;
      }
    }
    unsigned bal = __ballot_sync(0xffffffffu, live);
    if (lane == 0) s_w[wid] = __popc(bal);
    __syncthreads();
    int woff = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      woff += q < wid ? s_w[q] : 0;
      tot += s_w[q];
    }
    if (live) {
      int slot = nlive + woff + __popc(bal & ((1u << lane) - 1u));
      double r = sqrt(r2);
      double inv = 1.0 / r;
      s_ex[slot] = (T)(d[0] * inv);
      s_ey[slot] = (T)(d[1] * inv);
      s_ez[slot] = (T)(d[2] * inv);
      s_r[slot] = (T)r;
      s_j[slot] = j;
      s_ent[slot] = e0 + e;
      s_atom[slot] = (short)la;
      int sj = a.species[j];
      sj = (sj < 0 || sj >= SS) ? 0 : sj;
      s_sp[slot] = (unsigned char)sj;
      const int si = s_si[la];
#pragma unroll
      for (int q = 0; q < SS; ++q) {  // f_C(r) of this slot acting as k in (i, q, slot)
        T fc, dfc;
        cutoff((T)r, TRIP((si * SS + q) * SS + sj), fc, dfc);
        s_fc[q * C + slot] = fc;
        s_dfc[q * C + slot] = dfc;
      }
      atomicAdd(&s_cnt[la], 1);
      if (r2 < 1e-16) {
        unsigned long long key =
            ((unsigned long long)(__double_as_longlong(r2) >> 32) << 32) | (unsigned)(e0 + e);
        atomicMin(&a.err->coinc_key, key);
      }
    }
    nlive += tot;
    __syncthreads();
  }

  // per-atom slot ranges and the zeta_visits counter (sum n_i^2, kernels.py:537-544)
  {
    int c = tid < na ? s_cnt[tid] : 0;
    int tot;
    int ex = block_excl_scan(c, s_w, tot);
    if (tid < na) s_soff[tid] = ex;
    if (tid == 0) s_soff[na] = tot;
    unsigned long long sq = (unsigned long long)c * (unsigned long long)c;
    sq = warp_sum(sq);
    if (lane == 0 && sq) atomicAdd(&a.stats[0], sq);
    unsigned long long pk = warp_sum((unsigned long long)c);
    if (lane == 0 && pk) atomicAdd(&a.stats[1], pk);
  }
  __syncthreads();

  // ---- phase 1: zeta_ij, then the pair part (V, dV/dr, delta_zeta) ----
  unsigned long long live_pairs = 0, live_trips = 0, taper_pairs = 0, taper_trips = 0;
  for (int s = tid; s < nlive; s += NT) {
    const int la = s_atom[s];
    const int si = s_si[la];
    const int sa = s_sp[s];
    const int b0 = s_soff[la], b1 = s_soff[la + 1];
    const T ra = s_r[s];
    const PairP<T> &pp = PAIR(si * SS + sa);
    T v = T(0), dvdr = T(0), dz = T(0);
    if (ra < pp.Rp) {
      live_pairs++;
      taper_pairs += ra > pp.Rm;
      const T eax = s_ex[s], eay = s_ey[s], eaz = s_ez[s];
      T zeta = T(0);
      for (int b = b0; b < b1; ++b) {
        if (b == s) continue;
        const T fcb = s_fc[sa * C + b];
        if (fcb == T(0)) continue;
        live_trips++;
        taper_trips += fcb != T(1);
        const int sb = s_sp[b];
        const TripP<T> &tp = TRIP((si * SS + sa) * SS + sb);
        T cost = eax * s_ex[b] + eay * s_ey[b] + eaz * s_ez[b];
        cost = fmin(T(1), fmax(T(-1), cost));
        T g, dg;
        angular(cost, tp, g, dg);
        T term = fcb * g;
        if (LAM3) {
          T ex, darg;
          lam3_term(ra - s_r[b], tp, ex, darg);
          term *= ex;
        }
        zeta += term;
      }
      pair_part(ra, zeta, pp, v, dvdr, dz);
    }
    s_dz[s] = dz;
    s_v[s] = v;
    s_dvdr[s] = dvdr;
  }
  {
    unsigned long long lp = warp_sum(live_pairs), lt = warp_sum(live_trips);
    unsigned long long tp = warp_sum(taper_pairs), tt = warp_sum(taper_trips);
    if (lane == 0 && (lp | lt)) {
      atomicAdd(&a.stats[2], lp);
      atomicAdd(&a.stats[3], lt);
      atomicAdd(&a.stats[4], tp);
      atomicAdd(&a.stats[5], tt);
    }
  }
  __syncthreads();

  // ---- phase 2: total force on each neighbour slot from the energy terms
  //      centred on its atom i.  Lane a gathers every dzeta-weighted gradient
  //      that lands on a:  (i,a,b) with a as j and (i,b,a) with a as k,
  //      both along e_a and w_ab = (e_b - cos e_a)/r_a. ----
  double wxx = 0, wyy = 0, wzz = 0, wxy = 0, wxz = 0, wyz = 0;
  for (int s = tid; s < nlive; s += NT) {
    const int la = s_atom[s];
    const int si = s_si[la];
    const int sa = s_sp[s];
    const int b0 = s_soff[la], b1 = s_soff[la + 1];
    const T ra = s_r[s];
    const T inva = T(1) / ra;
    const T eax = s_ex[s], eay = s_ey[s], eaz = s_ez[s];
    const T dza = s_dz[s];
    // (i,b,a) terms need f_C(r_a) OR its derivative: in the taper f_C can round
    // to 0 while dF_C/dr does not (r -> R+D), so test both
    const bool own_k1 = (S == 1) && (s_fc[s] != T(0) || s_dfc[s] != T(0));
    T Salpha = T(0), Sc = T(0), Sbx = T(0), Sby = T(0), Sbz = T(0);
    for (int b = b0; b < b1; ++b) {
      if (b == s) continue;
      const T dzb = s_dz[b];
      const int sb = s_sp[b];
      const T fcb = s_fc[sa * C + b];   // f_C(r_b) in (i,a,b)
      const T fca = s_fc[sb * C + s];   // f_C(r_a) in (i,b,a)
      const bool t1 = (dza != T(0)) && (fcb != T(0));
      const bool klive = (S == 1) ? own_k1 : (fca != T(0) || s_dfc[sb * C + s] != T(0));
      const bool t2 = (dzb != T(0)) && klive;
      if (!(t1 || t2)) continue;
      const T ebx = s_ex[b], eby = s_ey[b], ebz = s_ez[b];
      T cost = eax * ebx + eay * eby + eaz * ebz;
      cost = fmin(T(1), fmax(T(-1), cost));
      T alpha, beta;
      if (S == 1 && !LAM3) {
        const TripP<T> &tp = TRIP(0);
        T g, dg;
        angular(cost, tp, g, dg);
        const T dfca = s_dfc[s];
        alpha = dzb * (dfca * g);
        beta = dg * (dza * fcb + dzb * fca);
      } else {
        alpha = T(0);
        beta = T(0);
        if (t1) {
          const TripP<T> &tp = TRIP((si * SS + sa) * SS + sb);
          T g, dg, ex = T(1), darg = T(0);
          angular(cost, tp, g, dg);
          if (LAM3) lam3_term(ra - s_r[b], tp, ex, darg);
          const T val = fcb * g * ex;
          alpha += dza * (val * darg);
          beta += dza * (fcb * dg * ex);
        }
        if (t2) {
          const TripP<T> &tp = TRIP((si * SS + sb) * SS + sa);
          T g, dg, ex = T(1), darg = T(0);
          angular(cost, tp, g, dg);
          if (LAM3) lam3_term(s_r[b] - ra, tp, ex, darg);
          const T dfca = s_dfc[sb * C + s];
          const T val = fca * g * ex;
          alpha += dzb * (dfca * g * ex - val * darg);
          beta += dzb * (fca * dg * ex);
        }
      }
      Salpha += alpha;
      Sc += beta * cost;
      Sbx += beta * ebx;
      Sby += beta * eby;
      Sbz += beta * ebz;
    }
    // force on a: pair part -dV/dr e_a (kernels.py:300-308) and the zeta part
    const T ca = s_dvdr[s] + Salpha - Sc * inva;
    const double fx = -(double)(ca * eax + inva * Sbx);
    const double fy = -(double)(ca * eay + inva * Sby);
    const double fz = -(double)(ca * eaz + inva * Sbz);
    s_fx[s] = fx;
    s_fy[s] = fy;
    s_fz[s] = fz;
    // virial (x_a - x_i) (x) f_a   [derived; not in the reference]
    const double dxa = (double)ra * (double)eax, dya = (double)ra * (double)eay,
                 dza_ = (double)ra * (double)eaz;
    wxx += dxa * fx;
    wyy += dya * fy;
    wzz += dza_ * fz;
    wxy += dxa * fy;
    wxz += dxa * fz;
    wyz += dya * fz;
    const int j = s_j[s];
    if (MODE == 0) {
      atomicAdd(a.forces + 3 * (int64_t)j, fx);
      atomicAdd(a.forces + 3 * (int64_t)j + 1, fy);
      atomicAdd(a.forces + 3 * (int64_t)j + 2, fz);
    } else {
      double *fb = a.fbuf + 3 * (int64_t)s_ent[s];
      fb[0] = fx;
      fb[1] = fy;
      fb[2] = fz;
    }
  }
  __syncthreads();

  // ---- phase 3: per-atom self force (translation invariance: F_i from the
  //      terms centred on i is minus the sum over its neighbours) and e_i ----
  double ebl = 0.0;
  if (tid < na) {
    const int i = atom0 + tid;
    double fx = 0.0, fy = 0.0, fz = 0.0, ei = 0.0;
    for (int s = s_soff[tid]; s < s_soff[tid + 1]; ++s) {
      fx -= s_fx[s];
      fy -= s_fy[s];
      fz -= s_fz[s];
      ei += (double)s_v[s];
    }
    ebl = ei;
    if (a.per_atom) a.per_atom[i] = ei + 0.0;
    if (MODE == 0) {
      atomicAdd(a.forces + 3 * (int64_t)i, fx);
      atomicAdd(a.forces + 3 * (int64_t)i + 1, fy);
      atomicAdd(a.forces + 3 * (int64_t)i + 2, fz);
    }
  }
  // ---- block partials: energy (atom order) and virial ----
  double vals[7] = {ebl, wxx, wyy, wzz, wxy, wxz, wyz};
  __shared__ double s_red[NW][7];
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = warp_sum(vals[q]);
    if (lane == 0) s_red[wid][q] = v;
  }
  __syncthreads();
  if (tid < 7) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) v += s_red[w][tid];
    a.partials[8 * (int64_t)blockIdx.x + tid] = v;
  }
}

// deterministic final reduction of block partials -> result[7]
__global__ void k_reduce_partials(int nblocks, const double *__restrict__ partials,
                                  double *__restrict__ result) {
  __shared__ double s[256][7];
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nblocks; b += 256)
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
}

// deterministic gather from the per-entry buffer: the force on m is the sum
// of the pieces its neighbours' terms put on it (entries i->m, found through
// rev) minus the pieces m's own terms put on its neighbours (translation
// invariance: F_m(self) = -sum over row m).  Row order fixes the summation.
__global__ void k_force_gather(int n, const int *__restrict__ off, const int *__restrict__ rev,
                               const double *__restrict__ fbuf, double *__restrict__ forces) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
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

// ---------------------------------------------------------------------------
// K8: velocity Verlet pieces (system.py:355-380)
// ---------------------------------------------------------------------------

// v += half F / m ; x += dt v ; wrap periodic axes with np.remainder
__global__ void k_kick_drift(int n, double *__restrict__ pos, double *__restrict__ vel,
                             const double *__restrict__ f, const double *__restrict__ mass,
                             double half, double dt, Box box) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m = mass[i];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    int64_t k = 3 * (int64_t)i + ax;
    double v = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, f[k]), m));
    vel[k] = v;
    double x = __dadd_rn(pos[k], __dmul_rn(dt, v));
    if (box.per[ax]) x = np_remainder(x, box.L[ax]);
    pos[k] = x;
  }
}

__global__ void k_kick(int n, double *__restrict__ vel, const double *__restrict__ f,
                       const double *__restrict__ mass, double half) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m = mass[i];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    int64_t k = 3 * (int64_t)i + ax;
    vel[k] = __dadd_rn(vel[k], __ddiv_rn(__dmul_rn(half, f[k]), m));
  }
}

// ---------------------------------------------------------------------------
// FMA-pipe peak probe (roofline denominator)
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_fma_peak(T *out, int iters, T b, T c) {
  T a0 = T(threadIdx.x) * T(1e-3), a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
  T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  T s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == T(-12345)) out[blockIdx.x] = s;  // keep the chains alive
}

// per-block partial sums of m v^2 (fixed grid: deterministic)
__global__ void k_kinetic(int n, const double *__restrict__ vel, const double *__restrict__ mass,
                          double *__restrict__ part) {
  __shared__ double s[8];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double vx = vel[3 * (int64_t)i], vy = vel[3 * (int64_t)i + 1], vz = vel[3 * (int64_t)i + 2];
    acc += mass[i] * ((vx * vx + vy * vy) + vz * vz);
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

__global__ void k_kinetic_sum(int nb, const double *__restrict__ part, double scale,
                              double *__restrict__ out) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) acc += part[b];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) s[threadIdx.x] += s[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = scale * s[0];
}

}  // namespace tb
