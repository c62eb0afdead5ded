// fp64 throughput microbenchmark on sm_100a: DFMA (CUDA cores), DMMA m8n8k4 (fp64 tensor path),
// and both interleaved in the same warps -- do the two paths share one datapath?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>  // 0 DFMA only, 1 DMMA only, 2 both
__global__ void __launch_bounds__(256) kern(double* sink, int iters) {
  double f[16];
  double m[8][2];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = 1e-3 * i;
#pragma unroll
  for (int i = 0; i < 8; ++i) { m[i][0] = 1e-3 * i; m[i][1] = 2e-3 * i; }
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = fma(f[i], x, y);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(m[i], x, y);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += m[i][0] + m[i][1];
  sink[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int MODE>
double run(double* sink, int blocks, int iters) {
  kern<MODE><<<blocks, 256>>>(sink, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<blocks, 256>>>(sink, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warps = blocks * 8.0;
  double fl = 0;
  if (MODE != 1) fl += blocks * 256.0 * 16 * 2 * iters;          // 16 DFMA per thread per iter
  if (MODE != 0) fl += warps * 8 * 256 * 2.0 * iters;           // 8 m8n8k4 per warp per iter
  return fl / (ms * 1e-3) / 1e12;
}

int main() {
  const int blocks = 148 * 8, iters = 20000;
  double* sink;
  cudaMalloc(&sink, blocks * 256 * sizeof(double));
  double t0 = run<0>(sink, blocks, iters);
  double t1 = run<1>(sink, blocks, iters);
  double t2 = run<2>(sink, blocks, iters);
  printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"both_tflops\": %.2f, \"err\": \"%s\"}\n", t0, t1, t2,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
