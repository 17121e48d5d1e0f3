// Layer-by-layer tensor-core path for configurations too large for the fused
// one-CTA-per-tile kernels (full_reference_config, d = 716,
// 11 layers, 4 heads of 179, d_ff 985, d_embed 69, decoder 930×3, 46.7 M
// parameters, 282 MFLOP per AST).  Same network and outputs as forward.cu
// (reference: costmodel.py:193-269, nn.py:26-96, dataset.py:97-115).
//
// Every matrix product is a tcgen05 GEMM (gemm3_kernel): D = A · Bᵀ with A the
// activations [rows, K] and B the transposed weight image [N, K], both fp32
// split into a TF32 "hi" part and the fp32 remainder "lo" (3×TF32:
// A_hi·B_hi + A_hi·B_lo + A_lo·B_hi, fp32 accumulation in TMEM) — the
// fp32-accumulate parity mode, ~fp32 accuracy at tensor-core speed.  Operands
// stream in by TMA (2-D tensor maps, 128-byte swizzle, 32-column k-slabs)
// through a 2–3 stage mbarrier ring; one thread issues the MMAs, four warps
// run the epilogue (bias, ReLU, residual, hi/lo split of the output for the
// next GEMM).  Attention (L ≤ 16 keys per AST), LayerNorm, the device MLP and
// gate, and the output layer + Box-Cox decode are small CUDA-core kernels.
//
// HBM layout: activations row-major [T_pad, pad32(width)] in bucket-sorted
// token order (AST s of the stable argsort of n_leaf owns rows
// tok_off[s] .. tok_off[s]+L_s-1), pad columns zero; each activation that
// feeds a GEMM is stored as the (hi, lo) pair.  leaf_embed.{L} reads bucket
// L's rows as a [n_L, L·dp] matrix (a 2-D tensor map with row stride L·dp).
#include <cuda.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "common.cuh"

namespace tpcb {

namespace {

inline int pad32(int v) { return (v + 31) & ~31; }

// ---------------------------------------------------------------- tf32 split
__device__ __forceinline__ float tf32_hi(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {  // K-major, SW128
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ the GEMM
struct Epi {
  int M, N, ldc;            // real rows / columns, output row stride (floats)
  const float* bias;        // [N] or null
  int relu;
  const float* r_hi;        // residual (hi + lo) [M, ldr] or null
  const float* r_lo;
  int ldr;
  float* c;                 // plain fp32 output, or (c == null) the split pair:
  float* c_hi;
  float* c_lo;
};

constexpr int kTileM = 128;
constexpr int kSlabA = kTileM * 128;  // one 128-row × 32-float slab (16 KB)

template <int NT>
struct GemmCfg {
  static constexpr int kStages = NT == 256 ? 2 : 3;
  static constexpr int kSlabB = NT * 128;
  static constexpr int kStage = 2 * kSlabA + 2 * kSlabB;
  static constexpr int kSmem = kStages * kStage + 1024;
};

template <int NT>
__global__ void __launch_bounds__(192, 1)
    gemm3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                 const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                 int k_iters, Epi e) {
  using Cfg = GemmCfg<NT>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * NT, m0 = blockIdx.y * kTileM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    mbar_fence_init();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(2 * NT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 4 && lane == 0) {  // TMA producer
    tma_prefetch_desc(&ta_hi);
    tma_prefetch_desc(&ta_lo);
    tma_prefetch_desc(&tb_hi);
    tma_prefetch_desc(&tb_lo);
    for (int it = 0; it < k_iters; ++it) {
      const int s = it % S;
      if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      uint8_t* st = smem + s * Cfg::kStage;
      mbar_arrive_expect_tx(&full[s], Cfg::kStage);
      tma_load_2d(st, &ta_hi, it * 32, m0, &full[s]);
      tma_load_2d(st + kSlabA, &ta_lo, it * 32, m0, &full[s]);
      tma_load_2d(st + 2 * kSlabA, &tb_hi, it * 32, n0, &full[s]);
      tma_load_2d(st + 2 * kSlabA + Cfg::kSlabB, &tb_lo, it * 32, n0, &full[s]);
    }
  } else if (warp == 5 && lane == 0) {  // MMA issuer
    constexpr uint32_t id = idesc_tf32(kTileM, NT);
    for (int it = 0; it < k_iters; ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = smem_u32(smem + s * Cfg::kStage);
      const uint32_t a_lo = a_hi + kSlabA, b_hi = a_hi + 2 * kSlabA, b_lo = b_hi + Cfg::kSlabB;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t o = kk * 32;
        // the two correction products accumulate in their own TMEM tile
        // (columns NT..2NT): the main accumulator then takes K/8 rounding
        // steps instead of 3K/8 (the tensor core's fp32 accumulation
        // truncates, so its error grows with the step count)
        mma_tf32(tmem, sdesc(a_hi + o), sdesc(b_hi + o), id, (it | kk) != 0);
        mma_tf32(tmem + NT, sdesc(a_lo + o), sdesc(b_hi + o), id, (it | kk) != 0);
        mma_tf32(tmem + NT, sdesc(a_hi + o), sdesc(b_lo + o), id, 1);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  } else if (warp < 4) {  // epilogue: thread = TMEM lane = output row
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + 32 * warp + lane;
    const bool live = row < e.M;
    for (int ch = 0; ch < NT / 32; ++ch) {
      const int c0 = n0 + 32 * ch;
      if (c0 >= e.ldc) break;  // warp-uniform
      float v[32], w[32];
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32 * ch, v);
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + NT + 32 * ch, w);
      if (!live) continue;
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += w[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = c0 + j;
        float x = v[j];
        if (col < e.N) {
          if (e.bias) x += __ldg(e.bias + col);
          if (e.r_hi) {
            const size_t ri = (size_t)row * e.ldr + col;
            x += e.r_hi[ri] + e.r_lo[ri];
          }
          if (e.relu) x = fmaxf(x, 0.f);
        } else {
          x = 0.f;
        }
        v[j] = x;
      }
      if (e.c) {
        float4* dst = reinterpret_cast<float4*>(e.c + (size_t)row * e.ldc + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
        float4* dh = reinterpret_cast<float4*>(e.c_hi + (size_t)row * e.ldc + c0);
        float4* dl = reinterpret_cast<float4*>(e.c_lo + (size_t)row * e.ldc + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float h[4], l[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            h[u] = tf32_hi(v[4 * q + u]);
            l[u] = v[4 * q + u] - h[u];
          }
          dh[q] = make_float4(h[0], h[1], h[2], h[3]);
          dl[q] = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * NT));
}

// -------------------------------------------------------------- weight image
// One entry per GEMM B operand: the transposed weight Wt[n][k'] (k' < kp, zero
// padded) built from the row-major parameter W[k][n] (x @ W).  For leaf_embed
// the k axis is L segments of d real rows each padded to dp ("seg").
struct ImgEntry {
  int64_t src;   // float offset of W in the flat parameter vector
  int64_t dst;   // float offset in the image
  int n, kp;     // image rows (= output features), padded k
  int seg, segp; // real / padded k per segment (seg == 0: one segment of k_real = segp)
  int k_real;
  int n_src;     // row stride of W (its column count)
  int col0;      // first W column used (QKV: Wq | Wk | Wv concatenated by entries)
};

__global__ void build_image_kernel(const float* __restrict__ P, const ImgEntry* __restrict__ ents,
                                   int n_ents, float* __restrict__ img_hi,
                                   float* __restrict__ img_lo) {
  const ImgEntry E = ents[blockIdx.y];
  const int64_t total = (int64_t)E.n * E.kp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / E.kp), kq = (int)(i - (int64_t)n * E.kp);
    int k = -1;
    if (E.seg) {
      const int sgi = kq / E.segp, j = kq - sgi * E.segp;
      if (j < E.seg) k = sgi * E.seg + j;
    } else if (kq < E.k_real) {
      k = kq;
    }
    const float v = k >= 0 ? P[E.src + (int64_t)k * E.n_src + E.col0 + n] : 0.f;
    const float h = tf32_hi(v);
    img_hi[E.dst + i] = h;
    img_lo[E.dst + i] = v - h;
  }
}

// ------------------------------------------------------------ small kernels
// sorted token rows: X0[tok_off[s] + l] = packed x[ast_row[perm[s]] + l] (24 + pad)
__global__ void gather_tokens_kernel(const float* __restrict__ px, const int32_t* __restrict__ perm,
                                     const int32_t* __restrict__ ast_row,
                                     const int32_t* __restrict__ tok_off, int n_ast,
                                     float* __restrict__ x_hi, float* __restrict__ x_lo) {
  const int s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n_ast) return;
  const int lane = threadIdx.x & 31;
  const int t0 = tok_off[s], L = tok_off[s + 1] - t0;
  const int r0 = ast_row[perm[s]];
  for (int l = 0; l < L; ++l) {
    const float v = px[(size_t)(r0 + l) * 32 + lane];
    const float h = tf32_hi(v);
    x_hi[(size_t)(t0 + l) * 32 + lane] = h;
    x_lo[(size_t)(t0 + l) * 32 + lane] = v - h;
  }
}

// per (AST, head): ctx = softmax(q kᵀ / sqrt(dh)) v over the AST's own L rows
// (nn.py:79-96); writes the (hi, lo) pair, zeroes the pad columns
__global__ void attention_kernel(const float* __restrict__ qkv, int ldq,
                                 const int32_t* __restrict__ tok_off, int d, int nh, int dh,
                                 float scale, int ldc, float* __restrict__ c_hi,
                                 float* __restrict__ c_lo) {
  extern __shared__ float sm[];
  const int s = blockIdx.x, h = blockIdx.y;
  const int t0 = tok_off[s], L = tok_off[s + 1] - t0;
  const int dhp = dh + 1;  // odd stride: conflict-free row reads
  float* q = sm;
  float* k = q + TPCB_MAX_LEAF * dhp;
  float* v = k + TPCB_MAX_LEAF * dhp;
  float* p = v + TPCB_MAX_LEAF * dhp;  // [16][17]
  for (int e = threadIdx.x; e < L * dh; e += blockDim.x) {
    const int l = e / dh, j = e - l * dh;
    const float* row = qkv + (size_t)(t0 + l) * ldq + h * dh + j;
    q[l * dhp + j] = row[0];
    k[l * dhp + j] = row[d];
    v[l * dhp + j] = row[2 * d];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * L; e += blockDim.x) {
    const int i = e / L, j = e - i * L;
    float acc = 0.f;
    for (int c = 0; c < dh; ++c) acc = fmaf(q[i * dhp + c], k[j * dhp + c], acc);
    p[i * 17 + j] = acc * scale;
  }
  __syncthreads();
  if (threadIdx.x < L) {
    const int i = threadIdx.x;
    float m = -INFINITY;
    for (int j = 0; j < L; ++j) m = fmaxf(m, p[i * 17 + j]);
    float sum = 0.f;
    for (int j = 0; j < L; ++j) {
      const float ex = expf(p[i * 17 + j] - m);
      p[i * 17 + j] = ex;
      sum += ex;
    }
    for (int j = 0; j < L; ++j) p[i * 17 + j] /= sum;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * dh; e += blockDim.x) {
    const int i = e / dh, j = e - i * dh;
    float acc = 0.f;
    for (int kk = 0; kk < L; ++kk) acc = fmaf(p[i * 17 + kk], v[kk * dhp + j], acc);
    const size_t o = (size_t)(t0 + i) * ldc + h * dh + j;
    const float hi = tf32_hi(acc);
    c_hi[o] = hi;
    c_lo[o] = acc - hi;
  }
  if (h == nh - 1) {
    const int padw = ldc - nh * dh;
    for (int e = threadIdx.x; e < L * padw; e += blockDim.x) {
      const int i = e / padw, j = e - i * padw;
      const size_t o = (size_t)(t0 + i) * ldc + nh * dh + j;
      c_hi[o] = 0.f;
      c_lo[o] = 0.f;
    }
  }
}

// post-LN over d features (nn.py:48-54, eps 1e-5, biased variance): one warp
// per row; input the fp32 sum (GEMM + bias + residual), output the pair
__global__ void layernorm_kernel(const float* __restrict__ x, int ld, int rows, int d,
                                 const float* __restrict__ g, const float* __restrict__ b,
                                 float* __restrict__ y_hi, float* __restrict__ y_lo) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const float* xr = x + (size_t)r * ld;
  float s = 0.f;
  for (int j = lane; j < d; j += 32) s += xr[j];
  const float mean = warp_sum(s) / d;
  float q = 0.f;
  for (int j = lane; j < d; j += 32) {
    const float t = xr[j] - mean;
    q = fmaf(t, t, q);
  }
  const float rstd = rsqrtf(warp_sum(q) / d + 1e-5f);
  for (int j = lane; j < ld; j += 32) {
    float o = 0.f;
    if (j < d) o = (xr[j] - mean) * rstd * g[j] + b[j];
    const float hi = tf32_hi(o);
    y_hi[(size_t)r * ld + j] = hi;
    y_lo[(size_t)r * ld + j] = o - hi;
  }
}

__device__ __forceinline__ double boxcox_decode_l(double e, const tpcb_boxcox& bc, bool* bad) {
  const double t = e * bc.t_std + bc.t_mean;
  if (fabs(bc.lambda_bc) < 1e-9) return exp(t) - bc.shift;
  const double base = bc.lambda_bc * t + 1.0;
  if (!(base > 0.0)) {
    *bad = true;
    return nan("");
  }
  return pow(base, 1.0 / bc.lambda_bc) - bc.shift;
}

// device MLP + gate (costmodel.py:217-220), one block per sorted AST:
// z_v = relu(v Wh + bh), zp = z_v Wp + bp, z = z_x ⊙ zp
__global__ void device_gate_kernel(Model M, const float* __restrict__ P,
                                   const float* __restrict__ devfeat,
                                   const int32_t* __restrict__ perm, const float* __restrict__ zx,
                                   int ldz, float* __restrict__ z_hi, float* __restrict__ z_lo,
                                   float* __restrict__ zx_out, float* __restrict__ zv_out,
                                   float* __restrict__ z_out) {
  extern __shared__ float sv[];
  const int s = blockIdx.x, i = perm[s];
  const float* dv = devfeat + (size_t)i * TPCB_DEV_FEAT;
  for (int j = threadIdx.x; j < M.d_dev; j += blockDim.x) {
    float a = P[M.devhb + j];
    for (int k = 0; k < TPCB_DEV_FEAT; ++k) a = fmaf(dv[k], P[M.devhW + k * M.d_dev + j], a);
    a = fmaxf(a, 0.f);
    sv[j] = a;
    if (zv_out) zv_out[(size_t)i * M.d_dev + j] = a;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ldz; e += blockDim.x) {
    float zz = 0.f;
    if (e < M.d_e) {
      float a = P[M.devpb + e];
      for (int j = 0; j < M.d_dev; ++j) a = fmaf(sv[j], P[M.devpW + j * M.d_e + e], a);
      const float x = zx[(size_t)s * ldz + e];
      zz = x * a;
      if (zx_out) zx_out[(size_t)i * M.d_e + e] = x;
      if (z_out) z_out[(size_t)i * M.d_e + e] = zz;
    }
    const float hi = tf32_hi(zz);
    z_hi[(size_t)s * ldz + e] = hi;
    z_lo[(size_t)s * ldz + e] = zz - hi;
  }
}

// dec.out (costmodel.py:228-229) + scatter to input order + Box-Cox decode
__global__ void output_kernel(Model M, const float* __restrict__ P, const float* __restrict__ h_hi,
                              const float* __restrict__ h_lo, int ldh, int width,
                              const int32_t* __restrict__ perm, int n_ast, tpcb_boxcox bc,
                              float* __restrict__ pred, double* __restrict__ lat,
                              int32_t* __restrict__ status) {
  const int s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n_ast) return;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int j = lane; j < width; j += 32) {
    const size_t o = (size_t)s * ldh + j;
    acc = fmaf(h_hi[o] + h_lo[o], P[M.outW + j], acc);
  }
  acc = warp_sum(acc) + P[M.outb];
  if (lane == 0) {
    const int i = perm[s];
    pred[i] = acc;
    if (lat) {
      bool bad = false;
      lat[i] = bc.enabled ? boxcox_decode_l((double)acc, bc, &bad) : (double)acc;
      if (bad) raise_status(status, TPCB_ERR_DOMAIN);
    }
  }
}

// --------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int get_encoder(EncodeFn* out) {
  static EncodeFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      set_last_error("cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)", cudaErrorNotSupported);
      return TPCB_ERR_CUDA;
    }
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  *out = encode;
  return TPCB_OK;
}

// fp32 [outer rows][inner cols] with row stride `stride` floats; boxes of
// 32 columns × box_rows rows, 128-byte swizzle; out-of-range reads are zero
int tmap_2d(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t stride,
            int box_rows) {
  EncodeFn enc;
  if (int st = get_encoder(&enc)) return st;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)stride * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (large)", cudaErrorInvalidValue);
    return TPCB_ERR_CUDA;
  }
  return TPCB_OK;
}

// A operand: pair of [rows, k_ext] views (row stride lda); B: pair [n, kp]
struct Operand {
  const float* hi;
  const float* lo;
  int64_t rows, k_ext, ld;
};

template <int NT>
int launch_gemm_nt(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st) {
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  int rc = tmap_2d(&ta_hi, A.hi, A.k_ext, A.rows, A.ld, kTileM);
  if (!rc) rc = tmap_2d(&ta_lo, A.lo, A.k_ext, A.rows, A.ld, kTileM);
  if (!rc) rc = tmap_2d(&tb_hi, B.hi, B.k_ext, B.rows, B.ld, NT);
  if (!rc) rc = tmap_2d(&tb_lo, B.lo, B.k_ext, B.rows, B.ld, NT);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(gemm3_kernel<NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GemmCfg<NT>::kSmem));
    attr = true;
  }
  const dim3 grid((unsigned)ceil_div(e.ldc, NT), (unsigned)ceil_div(e.M, kTileM));
  gemm3_kernel<NT><<<grid, 192, GemmCfg<NT>::kSmem, st>>>(ta_hi, ta_lo, tb_hi, tb_lo,
                                                          (int)(A.k_ext / 32), e);
  TPCB_LAUNCH_CHECK("gemm3");
  return TPCB_OK;
}

int launch_gemm(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st) {
  if (A.k_ext != B.k_ext || (A.k_ext & 31)) return TPCB_ERR_VALIDATION;
  const int64_t m_tiles = ceil_div(e.M, kTileM);
  if (e.ldc > 128 && m_tiles * ceil_div(e.ldc, 256) >= kNumSMs)
    return launch_gemm_nt<256>(A, B, e, st);
  return launch_gemm_nt<128>(A, B, e, st);
}

// ---- image plan (shared by the forward, training and the ABI size query) --
struct LargePlan {
  int d, dp, ff, ffp, qkv, qkvp, de, dep;
  int64_t in, layer[TPCB_MAX_LAYERS][4], leaf[TPCB_MAX_LEAF + 1], dec[TPCB_MAX_DEC];
  int dec_kp[TPCB_MAX_DEC];
  int64_t bias_qkv[TPCB_MAX_LAYERS];  // concatenated QKV bias (in the bias image)
  int64_t img_floats, bias_floats;
  std::vector<ImgEntry> ents;
};

LargePlan make_plan(const Model& M) {
  LargePlan p{};
  p.d = M.d;
  p.dp = pad32(M.d);
  p.ff = M.d_ff;
  p.ffp = pad32(M.d_ff);
  p.qkv = 3 * M.d;
  p.qkvp = pad32(3 * M.d);
  p.de = M.d_e;
  p.dep = pad32(M.d_e);
  int64_t o = 0;
  auto add = [&](int64_t src, int n, int kp, int k_real, int n_src, int col0, int seg,
                 int segp) {
    ImgEntry E{src, o, n, kp, seg, segp, k_real, n_src, col0};
    p.ents.push_back(E);
    const int64_t at = o;
    o += (int64_t)n * kp;
    return at;
  };
  p.in = add(M.inW, M.d, 32, TPCB_FEAT, M.d, 0, 0, 0);
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& L = M.layer[li];
    // Wq | Wk | Wv as one [3d, dp] image (three entries, contiguous rows)
    p.layer[li][0] = add(L.Wq, M.d, p.dp, M.d, M.d, 0, 0, 0);
    add(L.Wk, M.d, p.dp, M.d, M.d, 0, 0, 0);
    add(L.Wv, M.d, p.dp, M.d, M.d, 0, 0, 0);
    p.layer[li][1] = add(L.Wo, M.d, p.dp, M.d, M.d, 0, 0, 0);
    p.layer[li][2] = add(L.fhW, M.d_ff, p.dp, M.d, M.d_ff, 0, 0, 0);
    p.layer[li][3] = add(L.foW, M.d, p.ffp, M.d_ff, M.d, 0, 0, 0);
  }
  for (int l = 1; l <= M.n_leaf_max; ++l)
    p.leaf[l] = add(M.leafW[l], M.d_e, l * p.dp, l * M.d, M.d_e, 0, M.d, p.dp);
  int kin = M.d_e;
  for (int i = 0; i < M.n_dec; ++i) {
    p.dec_kp[i] = pad32(kin);
    p.dec[i] = add(M.decW[i], M.dec[i], pad32(kin), kin, M.dec[i], 0, 0, 0);
    kin = M.dec[i];
  }
  p.img_floats = o;
  int64_t b = 0;
  for (int li = 0; li < M.n_layers; ++li) {
    p.bias_qkv[li] = b;
    b += p.qkvp;
  }
  p.bias_floats = b;
  return p;
}

__global__ void qkv_bias_kernel(const float* __restrict__ P, Model M, const int64_t* __restrict__ off,
                                float* __restrict__ out) {
  const int li = blockIdx.y, d = M.d;
  const LayerOff& L = M.layer[li];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < 3 * d; j += gridDim.x * blockDim.x) {
    const int part = j / d, c = j - part * d;
    const int src = part == 0 ? L.bq : part == 1 ? L.bk : L.bv;
    out[off[li] + j] = P[src + c];
  }
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// activation workspace (floats) for n_tok tokens / n_ast ASTs
struct Act {
  float *x_hi, *x_lo, *h_hi, *h_lo, *h1_hi, *h1_lo, *c_hi, *c_lo, *f_hi, *f_lo, *qkv, *sum;
  float *zx, *z_hi, *z_lo, *d_hi[2], *d_lo[2];
  int32_t *perm, *tok_off;
  size_t bytes;
};

Act carve_act(const LargePlan& p, const Model& M, int64_t n_tok, int64_t n_ast, uint8_t* base) {
  Act a{};
  size_t o = 0;
  const int64_t T = ((n_tok + kTileM - 1) / kTileM) * kTileM;
  const int64_t A = ((n_ast + kTileM - 1) / kTileM) * kTileM;
  int dmax = 32;
  for (int i = 0; i < M.n_dec; ++i) dmax = max(dmax, pad32(M.dec[i]));
  auto take = [&](size_t floats) {
    float* r = reinterpret_cast<float*>(base ? base + o : nullptr);
    o = align256(o + floats * 4);
    return r;
  };
  a.x_hi = take(T * 32);
  a.x_lo = take(T * 32);
  a.h_hi = take(T * p.dp);
  a.h_lo = take(T * p.dp);
  a.h1_hi = take(T * p.dp);
  a.h1_lo = take(T * p.dp);
  a.c_hi = take(T * p.dp);
  a.c_lo = take(T * p.dp);
  a.f_hi = take(T * p.ffp);
  a.f_lo = take(T * p.ffp);
  a.qkv = take(T * p.qkvp);
  a.sum = take(T * p.dp);
  a.zx = take(A * p.dep);
  a.z_hi = take(A * p.dep);
  a.z_lo = take(A * p.dep);
  for (int k = 0; k < 2; ++k) {
    a.d_hi[k] = take(A * dmax);
    a.d_lo[k] = take(A * dmax);
  }
  a.perm = reinterpret_cast<int32_t*>(take(n_ast + 1));
  a.tok_off = reinterpret_cast<int32_t*>(take(n_ast + 1));
  a.bytes = o;
  return a;
}

}  // namespace

bool large_supported(const Model& M) {
  return M.d_dev <= 1024 && M.n_heads * M.dh == M.d && M.dh <= 1024 &&
         (size_t)3 * TPCB_MAX_LEAF * (M.dh + 1) * 4 + 17 * 16 * 4 <= 200 * 1024;
}

}  // namespace tpcb

using namespace tpcb;

extern "C" int tpcb_large_sizes(const tpcb_model* m, int64_t n_ast, int64_t n_tok,
                                size_t* image_bytes, size_t* act_bytes) {
  if (!m || !image_bytes || !act_bytes) return TPCB_ERR_VALIDATION;
  if (!large_supported(m->dev)) return TPCB_ERR_UNSUPPORTED;
  const LargePlan p = make_plan(m->dev);
  *image_bytes = align256((size_t)p.img_floats * 4) * 2 + align256((size_t)p.bias_floats * 4) +
                 align256(p.ents.size() * sizeof(ImgEntry)) + 256 * 2;
  *act_bytes = carve_act(p, m->dev, n_tok, n_ast, nullptr).bytes;
  return TPCB_OK;
}

namespace tpcb {
namespace {
struct ImagePtrs {
  float *hi, *lo, *bias;
  ImgEntry* ents;
};
ImagePtrs carve_image(const LargePlan& p, uint8_t* base) {
  ImagePtrs r;
  size_t o = 0;
  r.hi = reinterpret_cast<float*>(base + o);
  o += align256((size_t)p.img_floats * 4);
  r.lo = reinterpret_cast<float*>(base + o);
  o += align256((size_t)p.img_floats * 4);
  r.bias = reinterpret_cast<float*>(base + o);
  o += align256((size_t)p.bias_floats * 4);
  r.ents = reinterpret_cast<ImgEntry*>(base + o);
  return r;
}
}  // namespace
}  // namespace tpcb

// weight image: the transposed (hi, lo) B operands of every GEMM + the
// concatenated QKV biases; rebuild after every parameter update
extern "C" int tpcb_large_prepare(const tpcb_model* m, const float* d_params, void* d_image,
                                  void* stream_) {
  if (!m || !d_params || !d_image) return TPCB_ERR_VALIDATION;
  if (!large_supported(m->dev)) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream_;
  const LargePlan p = make_plan(m->dev);
  ImagePtrs im = carve_image(p, (uint8_t*)d_image);
  TPCB_CUDA_CHECK(cudaMemcpyAsync(im.ents, p.ents.data(), p.ents.size() * sizeof(ImgEntry),
                                  cudaMemcpyHostToDevice, st));
  build_image_kernel<<<dim3(128, (unsigned)p.ents.size()), 256, 0, st>>>(
      d_params, im.ents, (int)p.ents.size(), im.hi, im.lo);
  int64_t* d_off = reinterpret_cast<int64_t*>(im.ents + p.ents.size());
  d_off = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(d_off) + 255) & ~uintptr_t(255));
  TPCB_CUDA_CHECK(cudaMemcpyAsync(d_off, p.bias_qkv, sizeof(int64_t) * m->dev.n_layers,
                                  cudaMemcpyHostToDevice, st));
  qkv_bias_kernel<<<dim3(8, m->dev.n_layers), 256, 0, st>>>(d_params, m->dev, d_off, im.bias);
  // the host arrays above are stack / plan locals: finish the copies first
  TPCB_CUDA_CHECK(cudaStreamSynchronize(st));
  TPCB_LAUNCH_CHECK("large_prepare");
  return TPCB_OK;
}

// forward over a packed batch (any rows_per_tile): h_perm / h_tok_off are the
// HOST bucket order (stable argsort of n_leaf) and token offsets in that order
extern "C" int tpcb_large_forward(const tpcb_model* m, const float* d_params, const void* d_image,
                                  const tpcb_packed* pk, const int32_t* h_perm,
                                  const int32_t* h_tok_off, const float* d_devfeat, int64_t n_ast,
                                  const tpcb_boxcox* norm, void* d_act, size_t act_bytes,
                                  float* d_pred, float* d_zx, float* d_zv, float* d_z,
                                  double* d_latency, int32_t* d_status, void* stream_) {
  if (!m || !d_params || !d_image || !pk || !h_perm || !h_tok_off || !d_devfeat || !d_act ||
      !d_pred)
    return TPCB_ERR_VALIDATION;
  if (n_ast <= 0) return TPCB_ERR_EMPTY_BATCH;
  const Model& M = m->dev;
  if (!large_supported(M)) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream_;
  const LargePlan p = make_plan(M);
  const int64_t n_tok = h_tok_off[n_ast];
  Act a = carve_act(p, M, n_tok, n_ast, (uint8_t*)d_act);
  if (a.bytes > act_bytes) return TPCB_ERR_VALIDATION;
  ImagePtrs im = carve_image(p, (uint8_t*)const_cast<void*>(d_image));
  TPCB_CUDA_CHECK(cudaMemcpyAsync(a.perm, h_perm, n_ast * 4, cudaMemcpyHostToDevice, st));
  TPCB_CUDA_CHECK(
      cudaMemcpyAsync(a.tok_off, h_tok_off, (n_ast + 1) * 4, cudaMemcpyHostToDevice, st));
  gather_tokens_kernel<<<ceil_div(n_ast, 8), 256, 0, st>>>(pk->x, a.perm, pk->ast_row, a.tok_off,
                                                           (int)n_ast, a.x_hi, a.x_lo);
  TPCB_LAUNCH_CHECK("large_gather");
  const float* P = d_params;
  auto W = [&](int64_t off, int n, int kp) {
    return Operand{im.hi + off, im.lo + off, n, kp, kp};
  };
  auto act = [&](const float* hi, const float* lo, int64_t rows, int ld) {
    return Operand{hi, lo, rows, ld, ld};
  };
  int rc;
  // input projection
  {
    Epi e{(int)n_tok, M.d, p.dp, P + M.inb, 0, nullptr, nullptr, 0, nullptr, a.h_hi, a.h_lo};
    if ((rc = launch_gemm(act(a.x_hi, a.x_lo, n_tok, 32), W(p.in, M.d, 32), e, st))) return rc;
  }
  const float scale = 1.0f / sqrtf((float)M.dh);
  const size_t att_smem = (size_t)(3 * TPCB_MAX_LEAF * (M.dh + 1) + 16 * 17) * 4;
  if (att_smem > 48 * 1024)
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)att_smem));
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& L = M.layer[li];
    {  // Q | K | V
      Epi e{(int)n_tok, p.qkv, p.qkvp, im.bias + p.bias_qkv[li], 0, nullptr, nullptr, 0, a.qkv,
            nullptr, nullptr};
      if ((rc = launch_gemm(act(a.h_hi, a.h_lo, n_tok, p.dp), W(p.layer[li][0], p.qkv, p.dp), e,
                            st)))
        return rc;
    }
    attention_kernel<<<dim3((unsigned)n_ast, M.n_heads), 128, att_smem, st>>>(
        a.qkv, p.qkvp, a.tok_off, M.d, M.n_heads, M.dh, scale, p.dp, a.c_hi, a.c_lo);
    TPCB_LAUNCH_CHECK("large_attention");
    {  // h + ctx Wo + bo → LN1
      Epi e{(int)n_tok, M.d, p.dp, P + L.bo, 0, a.h_hi, a.h_lo, p.dp, a.sum, nullptr, nullptr};
      if ((rc = launch_gemm(act(a.c_hi, a.c_lo, n_tok, p.dp), W(p.layer[li][1], M.d, p.dp), e,
                            st)))
        return rc;
    }
    layernorm_kernel<<<ceil_div(n_tok, 8), 256, 0, st>>>(a.sum, p.dp, (int)n_tok, M.d,
                                                         P + L.ln1g, P + L.ln1b, a.h1_hi,
                                                         a.h1_lo);
    {  // relu(h1 W1 + b1)
      Epi e{(int)n_tok, M.d_ff, p.ffp, P + L.fhb, 1, nullptr, nullptr, 0, nullptr, a.f_hi,
            a.f_lo};
      if ((rc = launch_gemm(act(a.h1_hi, a.h1_lo, n_tok, p.dp), W(p.layer[li][2], M.d_ff, p.dp),
                            e, st)))
        return rc;
    }
    {  // h1 + f W2 + b2 → LN2
      Epi e{(int)n_tok, M.d, p.dp, P + L.fob, 0, a.h1_hi, a.h1_lo, p.dp, a.sum, nullptr, nullptr};
      if ((rc = launch_gemm(act(a.f_hi, a.f_lo, n_tok, p.ffp), W(p.layer[li][3], M.d, p.ffp), e,
                            st)))
        return rc;
    }
    layernorm_kernel<<<ceil_div(n_tok, 8), 256, 0, st>>>(a.sum, p.dp, (int)n_tok, M.d,
                                                         P + L.ln2g, P + L.ln2b, a.h_hi, a.h_lo);
    TPCB_LAUNCH_CHECK("large_layernorm");
  }
  // leaf_embed.{L}: bucket L's rows as [n_L, L·dp]
  for (int64_t s0 = 0; s0 < n_ast;) {
    const int Lb = h_tok_off[s0 + 1] - h_tok_off[s0];
    int64_t s1 = s0 + 1;
    while (s1 < n_ast && h_tok_off[s1 + 1] - h_tok_off[s1] == Lb) ++s1;
    const int64_t nb = s1 - s0;
    const int64_t t0 = h_tok_off[s0];
    Operand A{a.h_hi + t0 * p.dp, a.h_lo + t0 * p.dp, nb, (int64_t)Lb * p.dp,
              (int64_t)Lb * p.dp};
    Epi e{(int)nb, M.d_e, p.dep, P + M.leafb[Lb], 0, nullptr, nullptr, 0, a.zx + s0 * p.dep,
          nullptr, nullptr};
    if ((rc = launch_gemm(A, W(p.leaf[Lb], M.d_e, Lb * p.dp), e, st))) return rc;
    s0 = s1;
  }
  device_gate_kernel<<<(unsigned)n_ast, 128, M.d_dev * 4, st>>>(M, P, d_devfeat, a.perm, a.zx,
                                                                 p.dep, a.z_hi, a.z_lo, d_zx,
                                                                 d_zv, d_z);
  TPCB_LAUNCH_CHECK("large_device_gate");
  const float* in_hi = a.z_hi;
  const float* in_lo = a.z_lo;
  int ldin = p.dep;
  for (int i = 0; i < M.n_dec; ++i) {
    const int ldo = pad32(M.dec[i]);
    Epi e{(int)n_ast, M.dec[i], ldo, P + M.decb[i], 1, nullptr, nullptr, 0, nullptr,
          a.d_hi[i & 1], a.d_lo[i & 1]};
    if ((rc = launch_gemm(act(in_hi, in_lo, n_ast, ldin), W(p.dec[i], M.dec[i], p.dec_kp[i]), e,
                          st)))
      return rc;
    in_hi = a.d_hi[i & 1];
    in_lo = a.d_lo[i & 1];
    ldin = ldo;
  }
  tpcb_boxcox bc{};
  if (norm) bc = *norm;
  output_kernel<<<ceil_div(n_ast, 8), 256, 0, st>>>(
      M, P, in_hi, in_lo, ldin, M.n_dec ? M.dec[M.n_dec - 1] : M.d_e, a.perm, (int)n_ast, bc,
      d_pred, d_latency, d_status);
  TPCB_LAUNCH_CHECK("large_output");
  return TPCB_OK;
}

namespace tpcb {
namespace {
__global__ void split_kernel(const float* __restrict__ x, int64_t rows, int cols, int ld,
                             float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = rows * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld;
    const int c = (int)(i - r * ld);
    const float v = c < cols ? x[r * cols + c] : 0.f;
    const float h = tf32_hi(v);
    hi[i] = h;
    lo[i] = v - h;
  }
}
}  // namespace
}  // namespace tpcb

extern "C" size_t tpcb_gemm3_ws(int64_t M, int32_t N, int32_t K) {
  const int kp = pad32(K);
  return (align256((size_t)M * kp * 4) + align256((size_t)N * kp * 4)) * 2;
}

// C[M, N] = A[M, K] · B[N, K]ᵀ (row-major fp32) through the 3×TF32 tcgen05
// GEMM of the large path (a unit under test and a tensor-pipe microbenchmark)
extern "C" int tpcb_gemm3(const float* d_a, const float* d_b, int64_t M, int32_t N, int32_t K,
                          float* d_c, int32_t ldc, void* d_ws, size_t ws_bytes, void* stream_) {
  if (!d_a || !d_b || !d_c || !d_ws || M < 1 || N < 1 || K < 1 || ldc < N || (ldc & 3))
    return TPCB_ERR_VALIDATION;
  if (ws_bytes < tpcb_gemm3_ws(M, N, K)) return TPCB_ERR_VALIDATION;
  cudaStream_t st = (cudaStream_t)stream_;
  const int kp = pad32(K);
  uint8_t* w = (uint8_t*)d_ws;
  float* a_hi = (float*)w;
  w += align256((size_t)M * kp * 4);
  float* a_lo = (float*)w;
  w += align256((size_t)M * kp * 4);
  float* b_hi = (float*)w;
  w += align256((size_t)N * kp * 4);
  float* b_lo = (float*)w;
  split_kernel<<<1024, 256, 0, st>>>(d_a, M, K, kp, a_hi, a_lo);
  split_kernel<<<1024, 256, 0, st>>>(d_b, N, K, kp, b_hi, b_lo);
  TPCB_LAUNCH_CHECK("gemm3_split");
  Operand A{a_hi, a_lo, M, kp, kp}, B{b_hi, b_lo, N, kp, kp};
  Epi e{(int)M, N, ldc, nullptr, 0, nullptr, nullptr, 0, d_c, nullptr, nullptr};
  return launch_gemm(A, B, e, st);
}

// the tcgen05 GEMM alone on pre-split operands (bench: tensor-pipe fraction)
extern "C" int tpcb_gemm3_presplit(const float* a_hi, const float* a_lo, const float* b_hi,
                                   const float* b_lo, int64_t M, int32_t N, int32_t Kp,
                                   float* d_c, int32_t ldc, void* stream_) {
  if (!a_hi || !a_lo || !b_hi || !b_lo || !d_c || (Kp & 31) || ldc < N || (ldc & 31))
    return TPCB_ERR_VALIDATION;
  Operand A{a_hi, a_lo, M, Kp, Kp}, B{b_hi, b_lo, N, Kp, Kp};
  Epi e{(int)M, N, ldc, nullptr, 0, nullptr, nullptr, 0, d_c, nullptr, nullptr};
  return launch_gemm(A, B, e, (cudaStream_t)stream_);
}
