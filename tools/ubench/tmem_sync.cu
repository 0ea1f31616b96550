// does compute-sanitizer synccheck accept tcgen05.alloc / dealloc? (tool check)
#include <cstdio>
#include <cstdint>
#include "../../paper_1710_08616_b200/csrc/hfb_sm100.cuh"
__global__ void k(int mode, double* out) {
  __shared__ uint32_t slot;
  if (mode == 0) {
    if (threadIdx.y == 0) hfb::sm100::tmem_alloc(&slot, 256);
    hfb::sm100::tmem_fence_before();
    __syncthreads();
    hfb::sm100::tmem_fence_after();
    __syncthreads();
    if (threadIdx.y == 0) hfb::sm100::tmem_dealloc(slot, 256);
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0 && threadIdx.y == 0) out[blockIdx.x] = 1.0;
}
int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  double* d;
  cudaMalloc(&d, 64 * sizeof(double));
  k<<<4, dim3(32, 8)>>>(mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d: %s\n", mode, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
