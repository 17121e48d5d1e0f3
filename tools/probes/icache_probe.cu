// Instruction-fetch probe: cycles per instruction of cold straight-line code
// vs the same instruction count executed from a small loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache_probe icache_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define FMA8                                                                     \
  a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c); \
  a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);

template <int N8>
__global__ void straight(float* out, long long* cyc, float b, float c) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N8; ++i) { FMA8 }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int N8>
__global__ void looped(float* out, long long* cyc, float b, float c, int reps) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < N8; ++i) { FMA8 }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  const int NS8 = 2048;  // 16384 FMAs straight-line (~256 KB of SASS)
  for (int threads : {32, 256}) {
    for (int rep = 0; rep < 3; ++rep) {
      straight<NS8><<<64, threads>>>(out, cyc, 1.0001f, 0.5f);
      cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
      long long s = 0;
      for (int i = 0; i < 64; ++i) s += h[i];
      printf("straight  threads %3d: %lld cycles for %d FMA instr/warp = %.2f cyc/instr\n", threads,
             s / 64, NS8 * 8, (double)(s / 64) / (NS8 * 8));
    }
    looped<8><<<64, threads>>>(out, cyc, 1.0001f, 0.5f, NS8 / 8);
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    long long s = 0;
    for (int i = 0; i < 64; ++i) s += h[i];
    printf("looped    threads %3d: %lld cycles for %d FMA instr/warp = %.2f cyc/instr\n", threads,
           s / 64, NS8 * 8, (double)(s / 64) / (NS8 * 8));
  }
  // smaller straight-line blocks: 1K, 4K instructions
  {
    straight<128><<<64, 32>>>(out, cyc, 1.0001f, 0.5f);
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    printf("straight 1K instr, 1 warp: %.2f cyc/instr\n", h[0] / 1024.0);
    straight<512><<<64, 32>>>(out, cyc, 1.0001f, 0.5f);
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    printf("straight 4K instr, 1 warp: %.2f cyc/instr\n", h[0] / 4096.0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
