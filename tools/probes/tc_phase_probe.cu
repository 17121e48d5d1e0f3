// Probe for the tcgen05 training-step design (3xTF32, fp32 operands in
// 128-byte-swizzled K-major tiles):
//  (1) correctness of a K-major 128x64x64 3xTF32 product, of the MN-major
//      reinterpretation of the same tiles for the weight gradient
//      (dW = Xᵀ·dY, M = 128 features, K = 128 rows) and for the transposed
//      weight product (dX = dY·W with the forward image Wᵀ read MN-major);
//  (2) the latency of one dependent "phase" (MMAs → commit → wait →
//      tcgen05.ld → epilogue rewriting the A operand (raw + lo) → fence →
//      barrier), 128 or 256 threads, N = 64 / 192;
//  (3) one SM's bulk-store bandwidth smem → global.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_phase_probe tc_phase_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, c) of an fp32 [R][C] operand: 32-column blocks of R x 128 B, SW128 atoms
__host__ __device__ inline uint32_t off_km(int R, int r, int c) {
  return (c >> 5) * (R * 128) + (r >> 3) * 1024 + (r & 7) * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) +
         (c & 3) * 4;
}
__device__ __forceinline__ uint64_t desc_base(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// K-major: k step kc (multiple of 8) of an [R][C] tile
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int R, int kc) {
  return desc_base(base + (kc >> 5) * (R * 128) + (kc & 31) * 4, 16, 1024);
}
// MN-major: k step kr (multiple of 8 rows) of an [R][C] tile read as [C][R]
__device__ int g_mn_variant = 0;
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int R, int kr) {
  switch (g_mn_variant) {
    case 0: return desc_base(base + (kr >> 3) * 1024, R * 128, 1024);
    case 1: return desc_base(base + (kr >> 3) * 1024, 1024, R * 128);
    case 2: return desc_base(base + (kr >> 3) * 1024, R * 128, 128);
    default: return desc_base(base + (kr >> 3) * 1024, 128, R * 128);
  }
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, int amaj, int bmaj) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(ph));
  asm volatile("tcgen05.fence::after_thread_sync;");
}
__device__ __forceinline__ float lo_of(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void sync_mma() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- (1) correctness: three products -------------------------------------------------
// X [128][64], Y [128][64] (dY), F [128][128], W image Wt [64 out][64 in] (K-major over in)
// out0 = X · Wtᵀ          (forward, [128][64])        K-major / K-major
// out1 = Fᵀ · Y           (weight grad, [128][64])    MN-major A / MN-major B, K = 128 rows
// out2 = Y · Wt           (dX, [128][64]: Σ_o Y[r][o] Wt[o][i])  K-major A / MN-major B
__global__ void check(const float* X, const float* Y, const float* F, const float* Wt, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sX = sm;                 // 32 KB raw, 32 KB lo
  uint8_t* sY = sm + 65536;         // 32 + 32
  uint8_t* sF = sm + 131072;        // 64 + 64  -> 262144 total? too much; F raw only at 128 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  // this probe keeps F raw + lo in a second pass to stay under 227 KB: X, Y (raw+lo) = 128 KB,
  // F (raw) 64 KB, W (raw) 16 KB... lo of F / W computed into spare space below
  uint8_t* sW = sm + 131072 + 65536;  // 16 KB raw
  for (int e = t; e < 128 * 64; e += blockDim.x) {
    const int r = e / 64, c = e % 64;
    *reinterpret_cast<float*>(sX + off_km(128, r, c)) = X[e];
    *reinterpret_cast<float*>(sX + 32768 + off_km(128, r, c)) = lo_of(X[e]);
    *reinterpret_cast<float*>(sY + off_km(128, r, c)) = Y[e];
    *reinterpret_cast<float*>(sY + 32768 + off_km(128, r, c)) = lo_of(Y[e]);
  }
  for (int e = t; e < 128 * 128; e += blockDim.x) {
    const int r = e / 128, c = e % 128;
    *reinterpret_cast<float*>(sF + off_km(128, r, c)) = F[e];
  }
  for (int e = t; e < 64 * 64; e += blockDim.x) {
    const int r = e / 64, c = e % 64;
    *reinterpret_cast<float*>(sW + off_km(64, r, c)) = Wt[e];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  sync_mma();
  const uint32_t tm = tbase;
  const uint32_t aX = smem_u32(sX), aY = smem_u32(sY), aF = smem_u32(sF), aW = smem_u32(sW);
  if (t == 0) {
    // out0: hi·hi + lo·hi (W has no lo here: exact-ish check of layout only)
    const uint32_t i0 = idesc_tf32(128, 64, 0, 0);
    for (int k = 0; k < 64; k += 8) mma(tm, desc_k(aX, 128, k), desc_k(aW, 64, k), i0, k > 0);
    for (int k = 0; k < 64; k += 8) mma(tm, desc_k(aX + 32768, 128, k), desc_k(aW, 64, k), i0, 1);
    // out1: F MN-major (M = 128 features, 4 blocks) x Y MN-major (N = 64), K = 128 rows
    const uint32_t i1 = idesc_tf32(128, 64, 1, 1);
    for (int k = 0; k < 128; k += 8) mma(tm + 64, desc_mn(aF, 128, k), desc_mn(aY, 128, k), i1, k > 0);
    for (int k = 0; k < 128; k += 8)
      mma(tm + 64, desc_mn(aF, 128, k), desc_mn(aY + 32768, 128, k), i1, 1);
    // out2: Y K-major (K = out) x Wt MN-major (N = in, K = out rows of the image)
    const uint32_t i2 = idesc_tf32(128, 64, 0, 1);
    if (g_mn_variant == 3) { for (int k = 0; k < 64; k += 8) mma(tm + 128, desc_k(aX, 128, k), desc_k(aW, 64, k), i0, k > 0); } else
    for (int k = 0; k < 64; k += 8) mma(tm + 128, desc_k(aY, 128, k), desc_mn(aW, 64, k), i2, k > 0);
    if (g_mn_variant != 3) for (int k = 0; k < 64; k += 8) mma(tm + 128, desc_k(aY + 32768, 128, k), desc_mn(aW, 64, k), i2, 1);
    commit(&bar);
  }
  wait_bar(&bar, 0);
  const int row = 32 * (warp & 3) + (t & 31);
  if (warp < 4) {
    float v[16];
    for (int p = 0; p < 3; ++p)
      for (int c = 0; c < 64; c += 16) {
        ld16(tm + ((uint32_t)(32 * warp) << 16) + p * 64 + c, v);
        for (int i = 0; i < 16; ++i) out[p * 8192 + row * 64 + c + i] = v[i];
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// ---- (2) phase latency ----------------------------------------------------------------
// NT threads; A = [128][64] raw + lo, B = [N][64] raw + lo (static); each iteration:
// 3xTF32 MMAs (K = 64) → commit → wait → tcgen05.ld of this thread's columns → epilogue
// writes A (raw + lo) from the first 64 accumulator columns → fence + barrier
template <int NT, int N>
__global__ void phase(int iters, long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;             // 64 KB
  uint8_t* sB = sm + 65536;     // N x 64 raw + lo: N*512 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int e = t; e < 128 * 64; e += NT) {
    const int r = e / 64, c = e % 64;
    const float x = 0.01f * ((r * 7 + c * 3) % 17 - 8);
    *reinterpret_cast<float*>(sA + off_km(128, r, c)) = x;
    *reinterpret_cast<float*>(sA + 32768 + off_km(128, r, c)) = lo_of(x);
  }
  for (int e = t; e < N * 64; e += NT) {
    const int r = e / 64, c = e % 64;
    const float x = 0.02f * ((r * 5 + c * 11) % 13 - 6);
    *reinterpret_cast<float*>(sB + off_km(N, r, c)) = x;
    *reinterpret_cast<float*>(sB + N * 256 + off_km(N, r, c)) = lo_of(x);
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  sync_mma();
  const uint32_t tm = tbase, aA = smem_u32(sA), aB = smem_u32(sB);
  const uint32_t id = idesc_tf32(128, N, 0, 0);
  const int q = warp & 3, part = warp >> 2;  // part: column quarter/half owned
  constexpr int NPART = NT / 128, COLS = 64 / NPART;
  const int row = 32 * q + (t & 31);
  uint32_t ph = 0;
  long long t0 = 0;
  float acc = 0.f;
  for (int it = 0; it < iters + 2; ++it) {
    if (it == 2) t0 = clock64();
    if (t == 0) {
      for (int k = 0; k < 64; k += 8) mma(tm, desc_k(aA, 128, k), desc_k(aB, N, k), id, k > 0);
      for (int k = 0; k < 64; k += 8) mma(tm, desc_k(aA, 128, k), desc_k(aB + N * 256, N, k), id, 1);
      for (int k = 0; k < 64; k += 8) mma(tm, desc_k(aA + 32768, 128, k), desc_k(aB, N, k), id, 1);
      commit(&bar);
    }
    wait_bar(&bar, ph);
    ph ^= 1;
    float v[16];
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += 16) {
      ld16(tm + ((uint32_t)(32 * q) << 16) + part * COLS + c0, v);
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        const int c = part * COLS + c0 + i;
        float4 r4, l4;
        r4.x = v[i] * 0.5f; r4.y = v[i + 1] * 0.5f; r4.z = v[i + 2] * 0.5f; r4.w = v[i + 3] * 0.5f;
        l4.x = lo_of(r4.x); l4.y = lo_of(r4.y); l4.z = lo_of(r4.z); l4.w = lo_of(r4.w);
        *reinterpret_cast<float4*>(sA + off_km(128, row, c)) = r4;
        *reinterpret_cast<float4*>(sA + 32768 + off_km(128, row, c)) = l4;
        acc += r4.x;
      }
    }
    sync_mma();
  }
  const long long t1 = clock64();
  if (t == 0) cyc[0] = (t1 - t0) / iters;
  sink[t] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// ---- (3) bulk store bandwidth of one SM (or `grid` SMs) --------------------------------
__global__ void bstore(float* dst, int bytes_per_iter, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int t = threadIdx.x;
  for (int i = t; i < bytes_per_iter / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  long long t0 = clock64();
  if (t == 0) {
    char* base = reinterpret_cast<char*>(dst) + (size_t)blockIdx.x * bytes_per_iter * iters;
    for (int it = 0; it < iters; ++it) {
      for (int o = 0; o < bytes_per_iter; o += 16384)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         base + (size_t)it * bytes_per_iter + o),
                     "r"(smem_u32(sm + o)), "r"(16384)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (t == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  // (1)
  std::vector<float> X(128 * 64), Y(128 * 64), F(128 * 128), W(64 * 64);
  srand(3);
  auto rnd = [] { return (float)((rand() % 20001) - 10000) / 7777.f; };
  for (auto& v : X) v = rnd();
  for (auto& v : Y) v = rnd();
  for (auto& v : F) v = rnd();
  for (auto& v : W) v = rnd();
  float *dX, *dY, *dF, *dW, *dO;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dF, F.size() * 4);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dO, 3 * 8192 * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dF, F.data(), F.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int variant = 0; variant < 4; ++variant) {
  cudaMemcpyToSymbol(g_mn_variant, &variant, 4);
  cudaMemset(dO, 0, 3 * 8192 * 4);
  check<<<1, 128, 212992>>>(dX, dY, dF, dW, dO);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d: ", variant);
  { std::vector<float> O2(3 * 8192); cudaMemcpy(O2.data(), dO, O2.size() * 4, cudaMemcpyDeviceToHost);
    double s1 = 0; for (int k = 0; k < 128; ++k) s1 += (double)F[k * 128 + 0] * Y[k * 64 + 0];
    double s1b = 0; for (int k = 0; k < 128; ++k) s1b += (double)F[k * 128 + 1] * Y[k * 64 + 0];
    double s1c = 0; for (int k = 0; k < 128; ++k) s1c += (double)F[k * 128 + 0] * Y[k * 64 + 1];
    printf("[out1 r0c0 %g want %g | r1c0 %g want %g | r0c1 %g want %g | out2 r0c0 %g] ", O2[8192], s1, O2[8192+64], s1b, O2[8193], s1c, O2[16384]); }
  std::vector<float> O(3 * 8192);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double err[3] = {0, 0, 0}, mag[3] = {0, 0, 0};
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 64; ++c) {
      double s0 = 0, s1 = 0, s2 = 0;
      for (int k = 0; k < 64; ++k) s0 += (double)X[r * 64 + k] * W[c * 64 + k];
      for (int k = 0; k < 128; ++k) s1 += (double)F[k * 128 + r] * Y[k * 64 + c];
      for (int o = 0; o < 64; ++o) s2 += (double)Y[r * 64 + o] * W[o * 64 + c];
      err[0] = fmax(err[0], fabs(O[r * 64 + c] - s0));
      err[1] = fmax(err[1], fabs(O[8192 + r * 64 + c] - s1));
      err[2] = fmax(err[2], fabs(O[16384 + r * 64 + c] - s2));
      mag[0] = fmax(mag[0], fabs(s0));
      mag[1] = fmax(mag[1], fabs(s1));
      mag[2] = fmax(mag[2], fabs(s2));
    }
  printf("check %s: fwd K/K err %.3e (|max| %.2f)  wgrad MN/MN err %.3e (|max| %.2f)  dX K/MN err %.3e (|max| %.2f)\n",
         cudaGetErrorString(e), err[0], mag[0], err[1], mag[1], err[2], mag[2]);
  }
  // (2)
  long long* dc;
  float* sink;
  cudaMalloc(&dc, 1024 * 8);
  cudaMalloc(&sink, 1024 * 4);
  long long c;
  cudaFuncSetAttribute(phase<128, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(phase<256, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(phase<512, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(phase<128, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(phase<256, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  phase<128, 64><<<1, 128, 65536 + 64 * 512>>>(64, dc, sink);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("phase NT=128 N=64: %lld cycles (%s)\n", c, cudaGetErrorString(cudaDeviceSynchronize()));
  phase<256, 64><<<1, 256, 65536 + 64 * 512>>>(64, dc, sink);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("phase NT=256 N=64: %lld cycles (%s)\n", c, cudaGetErrorString(cudaDeviceSynchronize()));
  phase<512, 64><<<1, 512, 65536 + 64 * 512>>>(64, dc, sink);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("phase NT=512 N=64: %lld cycles (%s)\n", c, cudaGetErrorString(cudaDeviceSynchronize()));
  phase<128, 192><<<1, 128, 65536 + 192 * 512>>>(64, dc, sink);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("phase NT=128 N=192: %lld cycles (%s)\n", c, cudaGetErrorString(cudaDeviceSynchronize()));
  phase<256, 192><<<1, 256, 65536 + 192 * 512>>>(64, dc, sink);
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("phase NT=256 N=192: %lld cycles (%s)\n", c, cudaGetErrorString(cudaDeviceSynchronize()));
  // (3)
  float* big;
  cudaMalloc(&big, (size_t)64 * 8 * 131072);
  cudaFuncSetAttribute(bstore, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int g : {1, 4, 64}) {
    bstore<<<g, 128, 131072>>>(big, 131072, 8, dc);
    cudaDeviceSynchronize();
    std::vector<long long> h(g);
    cudaMemcpy(h.data(), dc, g * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto v : h) mx = v > mx ? v : mx;
    printf("bulk store grid %d: %lld cycles for 1 MB per CTA -> %.1f B/cycle/SM (%s)\n", g, mx,
           1048576.0 / mx, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
