// tb_stream.cuh -- stage plan of the streamed tb_compute (host buffers).
//
// tb_compute with pinned host positions / forces is PCIe-bound at large sizes
// (config 5: 403 MB in, 537 MB out against a 2.6 ms kernel).  The streamed
// path cuts the atoms into K <= 32 index ranges and the warp chunks into K
// stages: a chunk's stage is the range of the highest atom index it references
// (as i or j), so stage s can run as soon as the positions of ranges 0..s are
// on the device; the forces of range r are final once the last stage that
// touches r has run (touch masks), and go back while later stages compute and
// later ranges are still coming in.  The kernel, its arithmetic and the set of
// chunks are unchanged: only the order of the chunks (sorted stably by stage)
// and the number of launches differ.
#pragma once
#include "tb_warp.cuh"

namespace tb {

constexpr int STREAM_KMAX = 32;

// one warp per chunk: stage[c] = range of the highest atom index referenced;
// touch[s] |= ranges referenced by the chunks of stage s
__global__ void __launch_bounds__(256) k_chunk_stage(const int4 *__restrict__ lanes, int nchunks,
                                                     int range_atoms, int *__restrict__ stage,
                                                     unsigned *__restrict__ touch) {
  __shared__ unsigned s_touch[STREAM_KMAX];
  if (threadIdx.x < STREAM_KMAX) s_touch[threadIdx.x] = 0u;
  __syncthreads();
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c < nchunks) {
    const int4 rec = __ldg(lanes + 32 * (int64_t)c + lane);
    int hi = 0;
    unsigned mask = 0u;
    if (rec.x >= 0) {
      const int ri = rec.y / range_atoms, rj = rec.z / range_atoms;
      hi = max(ri, rj);
      mask = (1u << ri) | (1u << rj);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      mask |= __shfl_xor_sync(0xffffffffu, mask, off);
    }
    if (lane == 0) {
      stage[c] = hi;
      atomicOr(&s_touch[hi], mask);
    }
  }
  __syncthreads();
  if (threadIdx.x < STREAM_KMAX && s_touch[threadIdx.x])
    atomicOr(touch + threadIdx.x, s_touch[threadIdx.x]);
}

// out chunk `rank` = chunk order[rank]
__global__ void __launch_bounds__(256) k_permute_chunks(const int4 *__restrict__ lanes,
                                                        const int *__restrict__ order,
                                                        int4 *__restrict__ out, int nchunks) {
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  out[32 * (int64_t)c + lane] = __ldg(lanes + 32 * (int64_t)__ldg(order + c) + lane);
}

}  // namespace tb
