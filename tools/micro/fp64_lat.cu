// Micro-benchmark (dev aid): fp64 dependent-chain latencies on this part (DADD, DMUL+DADD,
// ddiv) and a shared-memory load chain, one warp, clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lat fp64_lat.cu
#include <cstdio>

__global__ void k_lat(double a, double b, int n, long long* out, double* sink) {
  __shared__ double s[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    s[i] = 1.0 + i;
    idx[i] = (i * 97 + 13) & 1023;
  }
  __syncthreads();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = __dsub_rn(y, __dmul_rn(b, y));
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = __ddiv_rn(z, b);
  long long t3 = clock64();
  int k = threadIdx.x;
  for (int i = 0; i < n; ++i) k = idx[k];
  long long t4 = clock64();
  float f = static_cast<float>(a);
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, static_cast<float>(b));
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / n;
    out[1] = (t2 - t1) / n;
    out[2] = (t3 - t2) / n;
    out[3] = (t4 - t3) / n;
    out[4] = (t5 - t4) / n;
  }
  sink[threadIdx.x] = x + y + z + k + f;
}

// throughput: each thread runs 8 independent DADD chains
__global__ void k_tput(double a, double b, int n, long long* out, double* sink) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __dadd_rn(x[j], b);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  long long* d;
  double* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 1 << 20);
  long long h[5];
  for (int rep = 0; rep < 2; ++rep) k_lat<<<1, 32>>>(1.0, 1e-3, 4096, d, sink);
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("latency (cycles): DADD %lld, DMUL+DSUB %lld, ddiv %lld, LDS chain %lld, FADD %lld\n", h[0], h[1], h[2],
         h[3], h[4]);
  for (int threads : {32, 128, 256, 512, 1024}) {
    const int n = 1024;
    k_tput<<<1, threads>>>(1.0, 1e-3, n, d, sink);
    k_tput<<<1, threads>>>(1.0, 1e-3, n, d, sink);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("DADD throughput, %4d threads: %.2f thread-ops per cycle per SM\n", threads,
           double(threads) * 8 * n / double(h[0]));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
