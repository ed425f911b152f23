// tb_scan.cuh -- the list builder's prefix sums and its row-length sort,
// hand-written for sm_100a (no CUB in the library).
//
//   exclusive scan  (cell counts -> cell starts, row counts -> CSR offsets,
//                    filtered row counts; neighbor.py:90-96 / :209-212 cumsum)
//     reduce-then-scan over tiles of SCAN_TILE ints: k_scan_tiles (one sum per
//     tile, 16 B loads), k_scan_tile_sums (one CTA scans the tile sums),
//     k_scan_apply (per tile: thread-sequential scan of 16 items, warp
//     shuffles, a cross-warp pass in shared memory, + the tile's offset).
//     Traffic 2 reads + 1 write of 4 B per item.
//   stable counting sort of atoms by row length 0..32 (the warp-chunk plan:
//     rows of one length are packed floor(32/L) per warp)
//     k_len_counts: per-block bucket counts, bucket-major [33][nblocks];
//     exclusive scan of that matrix (stable bucket x block order);
//     k_len_scatter: per warp __match_any_sync ranks atoms of equal length in
//     index order, warps of a block are ordered by a shared-memory prefix.
//     Deterministic: the layout depends only on the row lengths.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tb {

constexpr int SCAN_NT = 256;              // threads per scan CTA
constexpr int SCAN_IPT = 16;              // items per thread
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// one CTA-wide exclusive scan of v (blockDim.x = SCAN_NT); returns the
// exclusive prefix, *total the CTA sum
__device__ __forceinline__ int cta_excl_scan(int v, int *s_w, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int inc = warp_incl_scan(v);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int t = lane < SCAN_NT / 32 ? s_w[lane] : 0;
    const int ti = warp_incl_scan(t);
    if (lane < SCAN_NT / 32) s_w[lane] = ti - t;
    if (lane == SCAN_NT / 32 - 1) s_w[SCAN_NT / 32] = ti;
  }
  __syncthreads();
  const int r = s_w[w] + inc - v;
  *total = s_w[SCAN_NT / 32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ void load_items(const int *__restrict__ in, int64_t n, int64_t base,
                                           int v[SCAN_IPT]) {
  // thread t owns items base + t*IPT .. +IPT-1 (four 16-byte loads when in range
  // and aligned; the caller's arrays are cudaMalloc'ed, base is a tile multiple)
  const int64_t first = base + (int64_t)threadIdx.x * SCAN_IPT;
  if (first + SCAN_IPT <= n && !(reinterpret_cast<uintptr_t>(in) & 15)) {
    const int4 *p = reinterpret_cast<const int4 *>(in + first);
#pragma unroll
    for (int q = 0; q < SCAN_IPT / 4; ++q) {
      const int4 a = __ldg(p + q);
      v[4 * q] = a.x;
      v[4 * q + 1] = a.y;
      v[4 * q + 2] = a.z;
      v[4 * q + 3] = a.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_IPT; ++q) v[q] = first + q < n ? __ldg(in + first + q) : 0;
  }
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_tiles(int64_t n, const int *__restrict__ in,
                                                        int *__restrict__ tile_sums) {
  __shared__ int s_w[SCAN_NT / 32 + 1];
  int v[SCAN_IPT];
  load_items(in, n, (int64_t)blockIdx.x * SCAN_TILE, v);
  int s = 0;
#pragma unroll
  for (int q = 0; q < SCAN_IPT; ++q) s += v[q];
  int total;
  cta_excl_scan(s, s_w, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// exclusive scan of the tile sums in place (one CTA, any count)
__global__ void __launch_bounds__(SCAN_NT) k_scan_tile_sums(int ntiles, int *__restrict__ sums) {
  __shared__ int s_w[SCAN_NT / 32 + 1];
  int carry = 0;
  for (int base = 0; base < ntiles; base += SCAN_NT) {
    const int i = base + threadIdx.x;
    const int v = i < ntiles ? sums[i] : 0;
    int total;
    const int ex = cta_excl_scan(v, s_w, &total);
    if (i < ntiles) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_apply(int64_t n, const int *__restrict__ in,
                                                        int *__restrict__ out,
                                                        const int *__restrict__ tile_off) {
  __shared__ int s_w[SCAN_NT / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int v[SCAN_IPT];
  load_items(in, n, base, v);
  int s = 0;
#pragma unroll
  for (int q = 0; q < SCAN_IPT; ++q) s += v[q];
  int total;
  int run = cta_excl_scan(s, s_w, &total) + tile_off[blockIdx.x];
  const int64_t first = base + (int64_t)threadIdx.x * SCAN_IPT;
  int e[SCAN_IPT];
#pragma unroll
  for (int q = 0; q < SCAN_IPT; ++q) {
    e[q] = run;
    run += v[q];
  }
  if (first + SCAN_IPT <= n && !(reinterpret_cast<uintptr_t>(out) & 15)) {
    int4 *p = reinterpret_cast<int4 *>(out + first);
#pragma unroll
    for (int q = 0; q < SCAN_IPT / 4; ++q)
      p[q] = make_int4(e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < SCAN_IPT; ++q)
      if (first + q < n) out[first + q] = e[q];
  }
}

inline int64_t scan_tiles(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE; }

// device-wide exclusive scan of n ints; `tmp` holds scan_tiles(n) ints.
// in and out may alias (each tile reads its items before writing them).
inline cudaError_t scan_exclusive(const int *in, int *out, int64_t n, int *tmp,
                                  cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int nt = (int)scan_tiles(n);
  k_scan_tiles<<<nt, SCAN_NT, 0, st>>>(n, in, tmp);
  k_scan_tile_sums<<<1, SCAN_NT, 0, st>>>(nt, tmp);
  k_scan_apply<<<nt, SCAN_NT, 0, st>>>(n, in, out, tmp);
  return cudaGetLastError();
}

// ---- stable counting sort of atoms by row length (0..32) -----------------

constexpr int LSORT_NT = 256;   // atoms per block
constexpr int LSORT_B = 33;     // buckets: lengths 0..32

__global__ void __launch_bounds__(LSORT_NT) k_len_counts(int n, const int *__restrict__ len,
                                                         int *__restrict__ counts) {
  __shared__ int c[LSORT_B];
  if (threadIdx.x < LSORT_B) c[threadIdx.x] = 0;
  __syncthreads();
  const int i = blockIdx.x * LSORT_NT + threadIdx.x;
  if (i < n) atomicAdd(&c[min(max(__ldg(len + i), 0), LSORT_B - 1)], 1);
  __syncthreads();
  if (threadIdx.x < LSORT_B) counts[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = c[threadIdx.x];
}

// out[rank] = i, ranks by (length, index): base = scanned bucket-major counts
__global__ void __launch_bounds__(LSORT_NT) k_len_scatter(int n, const int *__restrict__ len,
                                                          const int *__restrict__ base,
                                                          int *__restrict__ out) {
  constexpr int NWS = LSORT_NT / 32;
  __shared__ int wc[NWS][LSORT_B];  // per-warp bucket counts -> exclusive prefix over warps
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < NWS * LSORT_B; k += LSORT_NT) (&wc[0][0])[k] = 0;
  __syncthreads();
  const int i = blockIdx.x * LSORT_NT + threadIdx.x;
  const int b = i < n ? min(max(__ldg(len + i), 0), LSORT_B - 1) : -1;
  const unsigned same = __match_any_sync(0xffffffffu, b);
  const int r_in_warp = __popc(same & ((1u << lane) - 1u));
  if (b >= 0 && r_in_warp == 0) wc[w][b] = __popc(same);
  __syncthreads();
  if (threadIdx.x < LSORT_B) {
    int run = 0;
    for (int q = 0; q < NWS; ++q) {
      const int t = wc[q][threadIdx.x];
      wc[q][threadIdx.x] = run;
      run += t;
    }
  }
  __syncthreads();
  if (b >= 0) out[base[(int64_t)b * gridDim.x + blockIdx.x] + wc[w][b] + r_in_warp] = i;
}

inline int lsort_blocks(int n) { return (n + LSORT_NT - 1) / LSORT_NT; }
// scratch ints: counts[33 * nblocks] + scan tiles of that
inline int64_t lsort_scratch(int n) {
  const int64_t m = (int64_t)LSORT_B * lsort_blocks(n);
  return m + scan_tiles(m) + 4;
}

inline cudaError_t sort_by_length(const int *len, int n, int *out, int *scratch,
                                  cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int nb = lsort_blocks(n);
  const int64_t m = (int64_t)LSORT_B * nb;
  k_len_counts<<<nb, LSORT_NT, 0, st>>>(n, len, scratch);
  cudaError_t e = scan_exclusive(scratch, scratch, m, scratch + m, st);
  if (e != cudaSuccess) return e;
  k_len_scatter<<<nb, LSORT_NT, 0, st>>>(n, len, scratch, out);
  return cudaGetLastError();
}

}  // namespace tb
