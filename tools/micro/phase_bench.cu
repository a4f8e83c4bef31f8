// Micro-benchmark (dev aid): the cost of one block-barrier phase of a coloured sweep of a
// tiny level in one thread block — 27-entry rows, the operator and x in shared memory —
// against the variants that tell latency sources apart (generic vs shared-space loads,
// the IEEE division, the 27-step subtraction chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o phase_bench phase_bench.cu
#include <cstdio>
#include <cstdint>

constexpr int kRows = 96;   // active rows per phase (one colour of a 729-row level)
constexpr int kN = 768;     // x length
constexpr int kE = 28;      // entries per row (27 + padding)

template <int kMode>
__global__ void k_phase(const int32_t* gcols, const double* gvals, int phases, unsigned long long* out,
                        double* sink) {
  __shared__ int32_t cols[kE * kRows];
  __shared__ double vals[kE * kRows];
  __shared__ double x[kN];
  for (int i = threadIdx.x; i < kE * kRows; i += blockDim.x) {
    cols[i] = gcols[i];
    vals[i] = gvals[i];
  }
  for (int i = threadIdx.x; i < kN; i += blockDim.x) x[i] = 1.0 + i * 1e-3;
  __syncthreads();
  // generic pointers (what the bottom kernel's relocated descriptor holds)
  const int32_t* volatile vc = cols;
  const double* volatile vv = vals;
  double* volatile vx = x;
  const int32_t* pc = kMode == 1 ? vc : cols;
  const double* pv = kMode == 1 ? vv : vals;
  double* px = kMode == 1 ? vx : x;
  unsigned long long t0 = clock64();
  if (kMode == 6) {  // registers only: the arithmetic chain and the barrier
    const int r = threadIdx.x;
    double v[kE], xv[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      v[k] = pv[k * (r < kRows ? r : 0)];
      xv[k] = px[k + (r & 63)];
    }
    t0 = clock64();
    for (int p = 0; p < phases; ++p) {
      if (r < kRows) {
        double acc = 1.0 + p;
#pragma unroll
        for (int k = 0; k < kE - 1; ++k) acc = __dsub_rn(acc, __dmul_rn(v[k], xv[k]));
        px[(r * 7) % kN] = __ddiv_rn(acc, 2.0 + r);
      }
      __syncthreads();
    }
    phases = phases > 0 ? phases : 1;
  } else
  for (int p = 0; p < phases; ++p) {
    const int r = threadIdx.x;
    if (r < kRows) {
      int32_t c[kE];
      double v[kE], xv[kE];
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        c[k] = pc[k * kRows + r];
        v[k] = pv[k * kRows + r];
      }
      if (kMode >= 4) asm volatile("" ::: "memory");  // every operator load issued before the gathers
#pragma unroll
      for (int k = 0; k < kE; ++k) xv[k] = px[c[k]];
      if (kMode >= 4) asm volatile("" ::: "memory");  // every gather issued before the chain
      double acc = 1.0, diag = 2.0;
      if (kMode == 3) {  // independent products summed as a tree (not the reference order)
        double s[kE];
#pragma unroll
        for (int k = 0; k < kE; ++k) s[k] = __dmul_rn(v[k], xv[k]);
#pragma unroll
        for (int w = 1; w < kE; w *= 2)
#pragma unroll
          for (int k = 0; k + w < kE; k += 2 * w) s[k] = __dadd_rn(s[k], s[k + w]);
        acc = __dsub_rn(acc, s[0]);
      } else {
#pragma unroll
        for (int k = 0; k < kE - 1; ++k) acc = __dsub_rn(acc, __dmul_rn(v[k], xv[k]));
      }
      double nv;
      if (kMode == 2) {
        nv = __dmul_rn(acc, 0.5);
      } else if (kMode == 5) {  // correctly rounded quotient from a precomputed RN(1/diag)
        const double y = 0.5;
        const double q0 = __dmul_rn(acc, y);
        const double r0 = __fma_rn(-diag, q0, acc);
        const double q1 = __fma_rn(r0, y, q0);
        const double r1 = __fma_rn(-diag, q1, acc);
        nv = __fma_rn(r1, y, q1);
      } else {
        nv = __ddiv_rn(acc, diag);
      }
      px[(r * 7) % kN] = __dadd_rn(__dmul_rn(0.2, px[(r * 7) % kN]), __dmul_rn(0.8, nv));
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) {
    *out = (t1 - t0) / phases;
    *sink = x[5];
  }
}

__global__ void k_empty(int phases, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int p = 0; p < phases; ++p) __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *out = (t1 - t0) / phases;
}

int main() {
  int32_t hc[kE * kRows];
  double hv[kE * kRows];
  for (int r = 0; r < kRows; ++r)
    for (int k = 0; k < kE; ++k) {
      hc[k * kRows + r] = (r * 8 + k * 29) % kN;
      hv[k * kRows + r] = 0.01 * (k + 1);
    }
  int32_t* dc;
  double *dv, *sink;
  unsigned long long* dout;
  cudaMalloc(&dc, sizeof hc);
  cudaMalloc(&dv, sizeof hv);
  cudaMalloc(&sink, 8);
  cudaMalloc(&dout, 8);
  cudaMemcpy(dc, hc, sizeof hc, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, hv, sizeof hv, cudaMemcpyHostToDevice);
  const char* names[] = {"shared-space loads, ddiv", "generic loads, ddiv", "shared, multiply instead of ddiv",
                         "shared, tree sum", "shared, loads fenced before the chain", "fenced + Markstein division", "registers only: chain + ddiv + barrier"};
  unsigned long long cyc;
  for (int threads : {128, 256, 512}) {
    k_empty<<<1, threads>>>(1000, dout);
    cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: empty barrier phase %llu cycles\n", threads, cyc);
    for (int m = 0; m < 7; ++m) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (m) {
          case 0: k_phase<0><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          case 1: k_phase<1><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          case 2: k_phase<2><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          case 4: k_phase<4><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          case 5: k_phase<5><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          case 6: k_phase<6><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
          default: k_phase<3><<<1, threads>>>(dc, dv, 1000, dout, sink); break;
        }
      }
      cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
      printf("threads %d: %-36s %llu cycles per phase (%.2f us at 1.965 GHz)\n", threads, names[m], cyc,
             cyc / 1965.0);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
