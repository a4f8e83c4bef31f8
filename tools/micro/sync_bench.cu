// Micro-benchmark: cost of grid-wide and cluster-wide barriers on B200 (dev aid).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_grid(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out = t1 - t0;
  }
}

// custom barrier: one arrival counter + generation flag
__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__global__ void k_custom(int iters, unsigned long long* out) {
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int gen = g_gen;
      __threadfence();
      if (atomicAdd(&g_count, 1u) == gridDim.x - 1) {
        g_count = 0;
        __threadfence();
        g_gen = gen + 1;
      } else {
        while (g_gen == gen) {}
      }
      __threadfence();
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out = t1 - t0;
  }
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) cl.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out = t1 - t0;
  }
}

// dependent L2 round trip latency: pointer chase in a small (L2-resident) array
__global__ void k_chase(const int* next, int iters, unsigned long long* out, int* sink) {
  int p = 0;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) p = __ldcg(next + p);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *out = t1 - t0;
  *sink = p;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  for (int threads : {256, 1024}) {
    for (int blocks : {1, 16, 37, 74, 148, 296}) {
      if (blocks * threads > 148 * 2048) continue;
      void* args[] = {(void*)&iters, (void*)&d};
      cudaLaunchCooperativeKernel((void*)k_grid, blocks, threads, args, 0, 0);
      cudaLaunchCooperativeKernel((void*)k_grid, blocks, threads, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long ns;
      cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
      printf("grid.sync   threads %4d blocks %3d: %.3f us/sync %s\n", threads, blocks, ns / 1e3 / iters, cudaGetErrorString(e));
      cudaLaunchCooperativeKernel((void*)k_custom, blocks, threads, args, 0, 0);
      e = cudaDeviceSynchronize();
      cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
      printf("custom      threads %4d blocks %3d: %.3f us/sync %s\n", threads, blocks, ns / 1e3 / iters, cudaGetErrorString(e));
    }
  }
  k_cluster<<<16, 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long ns;
  cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
  printf("cluster16 sync: %.3f us/sync %s\n", ns / 1e3 / iters, cudaGetErrorString(e));
  // pointer chase, 1 MB array (L2 resident), stride 4097 ints
  const int n = 1 << 18;
  int* h = new int[n];
  for (int i = 0; i < n; ++i) h[i] = (i + 4097) % n;
  int *dn, *sink;
  cudaMalloc(&dn, n * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(dn, h, n * 4, cudaMemcpyHostToDevice);
  k_chase<<<1, 1>>>(dn, 10000, d, sink);
  k_chase<<<1, 1>>>(dn, 10000, d, sink);
  cudaDeviceSynchronize();
  cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
  printf("L2 dependent load latency: %.1f ns\n", ns / 10000.0);
  return 0;
}
