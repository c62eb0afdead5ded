// L2 read bandwidth on one B200: every CTA streams the whole (L2-resident) buffer region
// assigned to it `reps` times with 16-byte loads; reports bytes / time.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const double2* __restrict__ buf, size_t n2, int reps, double* sink) {
  double a = 0.0, b = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 v = __ldcg(buf + i);   // L2 only (no L1 reuse)
      a += v.x;
      b += v.y;
    }
  }
  if (a + b == 12345.678) sink[0] = a;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t sizes_mb[] = {4, 8, 16, 32, 48, 64, 96, 1024};
  double* sink;
  cudaMalloc(&sink, 8);
  for (size_t mb : sizes_mb) {
    size_t bytes = mb << 20, n2 = bytes / 16;
    double2* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    int reps = (int)(4096 / mb) + 1;
    k_read<<<nsm * 8, 256>>>(buf, n2, 1, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_read<<<nsm * 8, 256>>>(buf, n2, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%5zu MB x %4d: %8.0f GB/s\n", mb, reps, (double)bytes * reps / (ms * 1e-3) / 1e9);
    cudaFree(buf);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
