// Dependent-chain latency of fp64 ops on this GPU (one warp, clock64), and throughput
// with 8 independent chains. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int q = 0; q < n; ++q) {
    if (OP == 0) x = __dadd_rn(x, b);
    if (OP == 1) x = __dmul_rn(x, b);
    if (OP == 2) x = __fma_rn(x, b, a);
    if (OP == 3) x = a / x;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
__global__ void chains8(double* out, long long* cyc, double a, double b, int n) {
  double x[8];
  for (int c = 0; c < 8; ++c) x[c] = a + threadIdx.x + c;
  long long t0 = clock64();
#pragma unroll 4
  for (int q = 0; q < n; ++q)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) x[c] = __dadd_rn(x[c], b);
      if (OP == 1) x[c] = __dmul_rn(x[c], b);
    }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
  const char* names[] = {"DADD", "DMUL", "DFMA", "div"};
  for (int op = 0; op < 4; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) chain<0><<<1, 32>>>(out, cyc, 1.0, 1e-9, n);
      if (op == 1) chain<1><<<1, 32>>>(out, cyc, 1.0, 1.0000001, n);
      if (op == 2) chain<2><<<1, 32>>>(out, cyc, 1e-9, 1.0000001, n);
      if (op == 3) chain<3><<<1, 32>>>(out, cyc, 1.0, 1.0, n);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%s dependent chain: %.1f cycles/op (1 warp)\n", names[op], double(c) / n);
  }
  for (int op = 0; op < 2; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) chains8<0><<<1, 32>>>(out, cyc, 1.0, 1e-9, n);
      if (op == 1) chains8<1><<<1, 32>>>(out, cyc, 1.0, 1.0000001, n);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%s 8 chains: %.2f cycles/op (1 warp)\n", names[op], double(c) / (8.0 * n));
  }
  // 4 warps on one SM (one per SMSP) x 8 chains
  for (int op = 0; op < 1; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) {
      chains8<0><<<1, 128>>>(out, cyc, 1.0, 1e-9, n);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("DADD 8 chains x 4 warps: %.2f cycles per warp-op\n", double(c) / (8.0 * n));
  }
  return 0;
}
