// tcgen05 probe: one 128 x N x 64 bf16 MMA (fp32 accumulate in TMEM), K-major
// 128-byte-swizzled operands in shared memory, tcgen05.ld back to registers.
// Validates the descriptor / TMEM conventions the bf16 forward kernel uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>

constexpr int M = 128, K = 64, N = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// byte offset of element (r, k) of a K-major bf16 tile with 64-element (128 B)
// rows in 128-byte swizzle atoms (8 rows x 128 B)
__host__ __device__ inline uint32_t sw128(int r, int k) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);       // start address
  d |= (uint64_t)1 << 16;                      // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // stride byte offset: 8-row groups
  d |= (uint64_t)1 << 46;                      // version (sm100)
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) uint8_t sA[M * K * 2];
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int e = t; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + sw128(r, k)) = A[e];
  }
  for (int e = t; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128(r, k)) = B[e];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // generic-proxy smem writes → visible to the async (tensor) proxy
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (t == 0) {
    const uint32_t id = idesc_bf16(M, N);
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t a = sdesc(smem_u32(sA) + k * 32), b = sdesc(smem_u32(sB) + k * 32);
      const uint32_t acc = k > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(a), "l"(b), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // wait for the MMA chain
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes 32w..32w+31 (row = 32w + lane), 64 columns
  uint32_t v[64];
  const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
#define LD16(off)                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
               : "=r"(v[off + 0]), "=r"(v[off + 1]), "=r"(v[off + 2]), "=r"(v[off + 3]),       \
                 "=r"(v[off + 4]), "=r"(v[off + 5]), "=r"(v[off + 6]), "=r"(v[off + 7]),       \
                 "=r"(v[off + 8]), "=r"(v[off + 9]), "=r"(v[off + 10]), "=r"(v[off + 11]),     \
                 "=r"(v[off + 12]), "=r"(v[off + 13]), "=r"(v[off + 14]), "=r"(v[off + 15])    \
               : "r"(taddr + off))
  LD16(0);
  LD16(16);
  LD16(32);
  LD16(48);
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = 32 * warp + (t & 31);
  for (int c = 0; c < N; ++c) D[row * N + c] = __uint_as_float(v[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  __nv_bfloat16 *hA = new __nv_bfloat16[M * K], *hB = new __nv_bfloat16[N * K];
  float* ref = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2bfloat16((rand() % 2001 - 1000) / 500.f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 2001 - 1000) / 500.f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)__bfloat162float(hA[m * K + k]) * __bfloat162float(hB[n * K + k]);
      ref[m * N + n] = (float)s;
    }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  float* hD = new float[M * N];
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int i = 0; i < M * N; ++i) {
    const double d = fabs(hD[i] - ref[i]);
    maxerr = fmax(maxerr, d);
    if (d > 1e-3 * (1 + fabs(ref[i]))) ++bad;
  }
  printf("status %s  max|err| %.3e  bad %d / %d   D[0]=%f ref %f  D[last]=%f ref %f\n",
         cudaGetErrorString(e), maxerr, bad, M * N, hD[0], ref[0], hD[M * N - 1], ref[M * N - 1]);
  return 0;
}
