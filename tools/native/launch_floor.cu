// Event-bracketed launch floor on this GPU: empty kernel (592 x 128) with
// small and ~0.5 KB parameter blocks, and a kernel that does one dependent
// global load per warp (the "first gather" latency).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
struct Big { double v[64]; };
__global__ void k_empty(int *p) { if (p && threadIdx.x == 9999) p[0] = 1; }
__global__ void k_big(const __grid_constant__ Big b, int *p) { if (threadIdx.x == 9999) p[0] = (int)b.v[3]; }
__global__ void k_fill(float *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0.f;
}
__global__ void k_readsum(const float4 *p, size_t n, float *out) {
  float a = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(p + i); a += v.x + v.y + v.z + v.w;
  }
  if (a == 12345.f) out[0] = a;
}
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
  cudaStream_t st; cudaStreamCreate(&st);
  cudaGraph_t gr; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  k_empty<<<592, 128, 0, st>>>(d);
  cudaStreamEndCapture(st, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  const char *names[] = {"empty_after_memset", "big_params_after_memset", "one_ldg_after_memset",
                         "empty_after_fill_kernel", "empty_no_flush", "graph_empty_after_fill_kernel",
                         "fill_kernel_itself", "empty_after_fill_then_read"};
  float *fl2; cudaMalloc(&fl2, fb);
  for (int mode = 3; mode < 8; ++mode) {
    float tot = 0; int K = 200;
    for (int it = 0; it < K + 10; ++it) {
      if (mode != 4 && mode != 6) k_fill<<<148 * 8, 256, 0, st>>>(fl, fb / 4);
      if (mode == 7) k_readsum<<<148 * 8, 256, 0, st>>>((const float4 *)fl2, fb / 16, (float *)d);
      cudaEventRecord(a, st);
      if (mode == 3 || mode == 4 || mode == 7) k_empty<<<592, 128, 0, st>>>(d);
      else if (mode == 5) cudaGraphLaunch(ge, st);
      else k_fill<<<148 * 8, 256, 0, st>>>(fl, fb / 4);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it >= 10) tot += ms;
    }
    printf("{\"mode\": \"%s\", \"us\": %.2f}\n", names[mode], 1e3 * tot / K);
  }
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
    printf("{\"mode\": \"%s\", \"us\": %.2f}\n", names[mode], 1e3 * tot / K);
  }
  // grid shape of the same resident thread count: 592x128 vs 296x256 vs 148x512
  const int shp[4][2] = {{592, 128}, {296, 256}, {148, 512}, {148, 128}};
  for (int m = 0; m < 4; ++m) {
    float tot = 0; int K = 200;
    for (int it = 0; it < K + 10; ++it) {
      k_fill<<<148 * 8, 256, 0, st>>>(fl, fb / 4);
      cudaEventRecord(a, st);
      k_empty<<<shp[m][0], shp[m][1], 0, st>>>(d);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it >= 10) tot += ms;
    }
    printf("{\"mode\": \"empty_%dx%d_after_fill\", \"us\": %.2f}\n", shp[m][0], shp[m][1], 1e3 * tot / K);
  }
  return 0;
}
