// Codegen probe for the small-M product routine: cycles per call (warm) of
// variants of the same float4 x (K=64) swizzled-tile product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mm_probe mm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define SMEM(p) __builtin_assume(__isShared(p))
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

#define FMA4(s_, v_)                                                            \
  acc.x = fmaf(s_, v_.x, acc.x); acc.y = fmaf(s_, v_.y, acc.y);                \
  acc.z = fmaf(s_, v_.z, acc.z); acc.w = fmaf(s_, v_.w, acc.w);

// variant A: as in train4 (8 bases, unroll 1)
__device__ __noinline__ float4 mmA(float4 acc, const float* a, const float* W, int rows, int c, int K) {
  SMEM(a); SMEM(W);
  const float* wb = W + (c >> 5) * rows * 32;
  const int ch = (c >> 2) & 7;
  const float* b0 = wb + ((ch ^ 0) << 2); const float* b1 = wb + ((ch ^ 1) << 2);
  const float* b2 = wb + ((ch ^ 2) << 2); const float* b3 = wb + ((ch ^ 3) << 2);
  const float* b4 = wb + ((ch ^ 4) << 2); const float* b5 = wb + ((ch ^ 5) << 2);
  const float* b6 = wb + ((ch ^ 6) << 2); const float* b7 = wb + ((ch ^ 7) << 2);
#pragma unroll 1
  for (int k = 0; k < K; k += 8) {
    const int o = k * 32;
    const float4 x = ld4(a + k), y = ld4(a + k + 4);
    const float4 w0 = ld4(b0 + o), w1 = ld4(b1 + o + 32), w2 = ld4(b2 + o + 64), w3 = ld4(b3 + o + 96);
    const float4 w4 = ld4(b4 + o + 128), w5 = ld4(b5 + o + 160), w6 = ld4(b6 + o + 192), w7 = ld4(b7 + o + 224);
    FMA4(x.x, w0) FMA4(x.y, w1) FMA4(x.z, w2) FMA4(x.w, w3)
    FMA4(y.x, w4) FMA4(y.y, w5) FMA4(y.z, w6) FMA4(y.w, w7)
  }
  return acc;
}

// variant B: software pipelined (next iteration's loads issued before this iteration's FMAs)
__device__ __noinline__ float4 mmB(float4 acc, const float* a, const float* W, int rows, int c, int K) {
  SMEM(a); SMEM(W);
  const float* wb = W + (c >> 5) * rows * 32;
  const int ch = (c >> 2) & 7;
  const float* b0 = wb + ((ch ^ 0) << 2); const float* b1 = wb + ((ch ^ 1) << 2);
  const float* b2 = wb + ((ch ^ 2) << 2); const float* b3 = wb + ((ch ^ 3) << 2);
  const float* b4 = wb + ((ch ^ 4) << 2); const float* b5 = wb + ((ch ^ 5) << 2);
  const float* b6 = wb + ((ch ^ 6) << 2); const float* b7 = wb + ((ch ^ 7) << 2);
  float4 x = ld4(a), y = ld4(a + 4);
  float4 w0 = ld4(b0), w1 = ld4(b1 + 32), w2 = ld4(b2 + 64), w3 = ld4(b3 + 96);
  float4 w4 = ld4(b4 + 128), w5 = ld4(b5 + 160), w6 = ld4(b6 + 192), w7 = ld4(b7 + 224);
#pragma unroll 1
  for (int k = 8; k <= K; k += 8) {
    const int o = (k < K ? k : 0) * 32;
    const int ka = k < K ? k : 0;
    const float4 nx = ld4(a + ka), ny = ld4(a + ka + 4);
    const float4 n0 = ld4(b0 + o), n1 = ld4(b1 + o + 32), n2 = ld4(b2 + o + 64), n3 = ld4(b3 + o + 96);
    const float4 n4 = ld4(b4 + o + 128), n5 = ld4(b5 + o + 160), n6 = ld4(b6 + o + 192), n7 = ld4(b7 + o + 224);
    FMA4(x.x, w0) FMA4(x.y, w1) FMA4(x.z, w2) FMA4(x.w, w3)
    FMA4(y.x, w4) FMA4(y.y, w5) FMA4(y.z, w6) FMA4(y.w, w7)
    x = nx; y = ny; w0 = n0; w1 = n1; w2 = n2; w3 = n3; w4 = n4; w5 = n5; w6 = n6; w7 = n7;
  }
  return acc;
}

// variant C: inline asm vector loads issued up front
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __noinline__ float4 mmC(float4 acc, const float* a_, const float* W, int rows, int c, int K) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(a_);
  const uint32_t wb = (uint32_t)__cvta_generic_to_shared(W + (c >> 5) * rows * 32);
  const uint32_t ch = (c >> 2) & 7;
  uint32_t b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = wb + ((ch ^ j) << 4) + j * 128;
#pragma unroll 1
  for (int k = 0; k < K; k += 8) {
    const uint32_t o = k * 128;
    const float4 x = lds4(a + k * 4), y = lds4(a + k * 4 + 16);
    const float4 w0 = lds4(b[0] + o), w1 = lds4(b[1] + o), w2 = lds4(b[2] + o), w3 = lds4(b[3] + o);
    const float4 w4 = lds4(b[4] + o), w5 = lds4(b[5] + o), w6 = lds4(b[6] + o), w7 = lds4(b[7] + o);
    FMA4(x.x, w0) FMA4(x.y, w1) FMA4(x.z, w2) FMA4(x.w, w3)
    FMA4(y.x, w4) FMA4(y.y, w5) FMA4(y.z, w6) FMA4(y.w, w7)
  }
  return acc;
}

template <int V>
__global__ void __launch_bounds__(288, 1) bench(float* out, long long* cyc, int reps) {
  extern __shared__ __align__(1024) float sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0.001f * (i % 97);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int c = (threadIdx.x & 15) * 4;
  const float* A = sm + 4096 + (threadIdx.x >> 4) * 68;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) acc = mmA(acc, A, sm, 64, c, 64);
    if (V == 1) acc = mmB(acc, A, sm, 64, c, 64);
    if (V == 2) acc = mmC(acc, A, sm, 64, c, 64);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[4];
  const char* names[3] = {"A (train4)", "B (pipelined)", "C (asm lds)"};
  for (int threads : {32, 256}) {
    for (int v = 0; v < 3; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) bench<0><<<1, threads, 40000>>>(out, cyc, 64);
        if (v == 1) bench<1><<<1, threads, 40000>>>(out, cyc, 64);
        if (v == 2) bench<2><<<1, threads, 40000>>>(out, cyc, 64);
      }
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("threads %3d  %-14s %lld cycles per K=64 call\n", threads, names[v], h[0]);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
