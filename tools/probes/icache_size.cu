// Instruction-cache capacity probe: straight-line blocks of S instructions run
// twice in one launch; the second pass is warm only if S fits the cache.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache_size icache_size.cu
#include <cstdio>
#include <cuda_runtime.h>

#define FMA8                                                                     \
  a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c); \
  a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);

template <int N8>
__global__ void twice(float* out, long long* cyc, float b, float c) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
  long long t[3];
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    t[pass] = clock64();
#pragma unroll
    for (int i = 0; i < N8; ++i) { FMA8 }
  }
  t[2] = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0) {
    cyc[2 * blockIdx.x] = t[1] - t[0];
    cyc[2 * blockIdx.x + 1] = t[2] - t[1];
  }
}

template <int N8>
void run(float* out, long long* cyc) {
  long long h[2];
  twice<N8><<<1, 32>>>(out, cyc, 1.0001f, 0.5f);
  twice<N8><<<1, 32>>>(out, cyc, 1.0001f, 0.5f);
  cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("%6d instr (%4d KB): pass1 %.2f cyc/instr, pass2 %.2f cyc/instr\n", N8 * 8,
         N8 * 8 * 16 / 1024, (double)h[0] / (N8 * 8), (double)h[1] / (N8 * 8));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 64);
  run<64>(out, cyc);
  run<128>(out, cyc);
  run<256>(out, cyc);
  run<512>(out, cyc);
  run<1024>(out, cyc);
  run<2048>(out, cyc);
  run<4096>(out, cyc);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
