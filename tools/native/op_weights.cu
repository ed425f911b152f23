// Dynamic flop weights of the math-library operations the roofline's
// algorithmic-flop convention charges: one kernel per
// (op, precision); every thread makes ITER data-dependent calls.  Run under
//   ncu --metrics smsp__sass_thread_inst_executed_op_{d,f}{add,mul,fma}_pred_on.sum
// and divide by threads * ITER (minus the one accumulate add per call).
// Built with the library's flags (-O3, IEEE div/sqrt, no fast math).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITER = 64;
constexpr int THREADS = 148 * 256;

template <class T> struct Ops {
  static __device__ T div(T a, T b) { return a / b; }
  static __device__ T sqrt_(T a) { return sqrt(a); }
  static __device__ T exp_(T a) { return exp(a); }
  static __device__ T sin_(T a) { return sin(a); }
  static __device__ T cos_(T a) { return cos(a); }
  static __device__ T pow_(T a, T b) { return pow(a, b); }
};
template <> struct Ops<float> {
  static __device__ float div(float a, float b) { return a / b; }
  static __device__ float sqrt_(float a) { return sqrtf(a); }
  static __device__ float exp_(float a) { return expf(a); }
  static __device__ float sin_(float a) { return sinf(a); }
  static __device__ float cos_(float a) { return cosf(a); }
  static __device__ float pow_(float a, float b) { return powf(a, b); }
};

// op: 0 baseline (accumulate only), 1 div, 2 sqrt, 3 exp, 4 sin, 5 cos, 6 pow
template <class T, int OP>
__global__ void k_op(const T *__restrict__ in, T *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  T x = in[t], acc = T(0);
#pragma unroll 1
  for (int k = 0; k < ITER; ++k) {
    const T a = x + T(0.25) * T(k & 7);  // integer-only variation would be hoisted
    T r;
    if (OP == 0) r = a;
    if (OP == 1) r = Ops<T>::div(T(1.7), a);
    if (OP == 2) r = Ops<T>::sqrt_(a);
    if (OP == 3) r = Ops<T>::exp_(-a);
    if (OP == 4) r = Ops<T>::sin_(a);
    if (OP == 5) r = Ops<T>::cos_(a);
    if (OP == 6) r = Ops<T>::pow_(a, T(0.78734));
    acc += r;
  }
  out[t] = acc;
}

template <class T>
static void run(const char *name) {
  T *in, *out;
  cudaMalloc(&in, sizeof(T) * THREADS);
  cudaMalloc(&out, sizeof(T) * THREADS);
  T *h = new T[THREADS];
  for (int i = 0; i < THREADS; ++i) h[i] = T(0.3) + T(2.5) * T(i % 1000) / T(1000);
  cudaMemcpy(in, h, sizeof(T) * THREADS, cudaMemcpyHostToDevice);
  // the "+ 0.25*(k&7)" is charged to every op including the baseline
  k_op<T, 0><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 1><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 2><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 3><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 4><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 5><<<THREADS / 256, 256>>>(in, out);
  k_op<T, 6><<<THREADS / 256, 256>>>(in, out);
  cudaDeviceSynchronize();
  printf("%s ok (%s)\n", name, cudaGetErrorString(cudaGetLastError()));
  delete[] h;
  cudaFree(in);
  cudaFree(out);
}

int main() {
  printf("threads %d iter %d\n", THREADS, ITER);
  run<double>("fp64");
  run<float>("fp32");
  return 0;
}
