// Micro-benchmark: HBM vs L2 re-read bandwidth of a window (dev aid for temporal blocking).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = p[i];
    s += v.x + v.y;
  }
  if (s == 1234.5) *out = s;
}
__global__ void k_flush(double* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = i;
}

int main() {
  size_t total = size_t(2) << 30;
  double* buf; double* out;
  cudaMalloc(&buf, total); cudaMalloc(&out, 8);
  cudaMemset(buf, 0, total);
  double* flush; cudaMalloc(&flush, size_t(512) << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t mb : {16, 32, 48, 64, 80, 96, 112, 128, 256}) {
    size_t n = (mb << 20) / 16;
    for (int rep = 0; rep < 2; ++rep) {
      k_flush<<<148 * 4, 512>>>(flush, (size_t(512) << 20) / 8);
      cudaEventRecord(a);
      k_read<<<148 * 8, 256>>>((const double2*)buf, n, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float t1; cudaEventElapsedTime(&t1, a, b);
      cudaEventRecord(a);
      k_read<<<148 * 8, 256>>>((const double2*)buf, n, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float t2; cudaEventElapsedTime(&t2, a, b);
      if (rep) printf("%4zu MB: cold %.1f us (%.0f GB/s)  warm %.1f us (%.0f GB/s)\n", mb, t1 * 1e3, (mb << 20) / (t1 * 1e6), t2 * 1e3, (mb << 20) / (t2 * 1e6));
    }
  }
  return 0;
}
