// Event-bracketed launch floor on this GPU: empty kernel (592 x 128) with
// small and ~0.5 KB parameter blocks, and a kernel that does one dependent
// global load per warp (the "first gather" latency).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
struct Big { double v[64]; };
__global__ void k_empty(int *p) { if (p && threadIdx.x == 9999) p[0] = 1; }
__global__ void k_big(const __grid_constant__ Big b, int *p) { if (threadIdx.x == 9999) p[0] = (int)b.v[3]; }
__global__ void k_load(const int4 *__restrict__ l, double *out) {
  int4 v = __ldg(l + blockIdx.x * blockDim.x + threadIdx.x);
  if (v.x == 12345) out[0] = v.y;
}
int main() {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int *d; cudaMalloc(&d, 1 << 20);
  int4 *l; cudaMalloc(&l, 592 * 128 * 16); cudaMemset(l, 0, 592 * 128 * 16);
  float *fl; size_t fb = 256 << 20; cudaMalloc(&fl, fb);
  Big big = {};
  for (int mode = 0; mode < 3; ++mode) {
    float tot = 0; int K = 200;
    for (int it = 0; it < K + 10; ++it) {
      cudaMemsetAsync(fl, 0, fb);
      cudaEventRecord(a);
      if (mode == 0) k_empty<<<592, 128>>>(d);
      else if (mode == 1) k_big<<<592, 128>>>(big, d);
      else k_load<<<592, 128>>>(l, (double *)d);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it >= 10) tot += ms;
    }
    printf("{\"mode\": \"%s\", \"us\": %.2f}\n", mode == 0 ? "empty" : mode == 1 ? "big_params" : "one_ldg_flushed", 1e3 * tot / K);
  }
  return 0;
}
