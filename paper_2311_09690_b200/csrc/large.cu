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

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "async.cuh"
#include "boxcox.cuh"
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

// K-major operand descriptor: BK = 32 fp32 per row → 128-byte swizzle (8-row
// atoms of 1 KB), BK = 16 → 64-byte swizzle (8-row atoms of 512 B)
template <int BK = 32>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * BK * 4) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(BK == 32 ? 2 : 4) << 61;
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
  const float* mask = nullptr;  // ReLU backward: keep x where mask[row, col] > 0
  int ldm = 0;
  int64_t split_stride = 0;     // split-K: split z writes c + z * split_stride
  int dbg = 0;                  // probe: 1 = skip the MMAs (TMA stream only), 2 = skip both
};

constexpr int kTileM = 128;
// BK fp32 columns per k-slab (32: 128-B swizzle, 16: 64-B swizzle and twice
// the stages in the same shared memory — deeper TMA prefetch)
template <int NT, int BK = 32>
struct GemmCfg {
  static constexpr int kSlabA = kTileM * BK * 4;
  static constexpr int kSlabB = NT * BK * 4;
  static constexpr int kStage = 2 * kSlabA + 2 * kSlabB;
  static constexpr int kStages = (192 * 1024) / kStage < 8 ? (192 * 1024) / kStage : 8;
  static constexpr int kSmem = kStages * kStage + 1024;
};

// cluster helpers (CN × CM CTAs: A tiles shared along N, B tiles along M)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* tmap, int c0, int c1,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask));
}

template <int NT, int BK, int CN, int CM>
__global__ void __launch_bounds__(192, 1)
    gemm3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                 const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                 int kc, int k_total, Epi e) {
  using Cfg = GemmCfg<NT, BK>;
  constexpr int kSlabA = Cfg::kSlabA;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[S], empty[S], done;
  __shared__ uint32_t tmem_base;
  __shared__ float sbias[NT];  // the tile's bias columns (epilogue)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * NT, m0 = blockIdx.y * kTileM;
  const int k0 = blockIdx.z * kc;
  const int k_iters = min(kc, k_total - k0);  // >= 1 (host picks the splits)

  constexpr int CS = CN * CM;  // cluster size
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);  // every cluster CTA's MMAs must release the slot
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
  if constexpr (CS > 1) cluster_sync_all();  // peers' barriers initialised
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // cluster coordinates: x along N (shares the A tile), y along M (shares B)
  const uint32_t crank = CS > 1 ? cluster_rank() : 0;
  const int cx = (int)(crank % CN), cy = (int)(crank / CN);
  uint16_t mask_a = 0, mask_b = 0;  // CTAs with my M tile / my N tile
  for (int x = 0; x < CN; ++x) mask_a |= (uint16_t)(1u << (x + cy * CN));
  for (int y = 0; y < CM; ++y) mask_b |= (uint16_t)(1u << (cx + y * CN));

  if (warp == 4 && lane == 0) {  // TMA producer
    tma_prefetch_desc(&ta_hi);
    tma_prefetch_desc(&ta_lo);
    tma_prefetch_desc(&tb_hi);
    tma_prefetch_desc(&tb_lo);
    for (int it = 0; it < k_iters; ++it) {
      const int s = it % S;
      if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      uint8_t* st = smem + s * Cfg::kStage;
      if (e.dbg == 2) {  // probe: no operand traffic (epilogue + pipeline skeleton)
        mbar_arrive_expect_tx(&full[s], 0);
        continue;
      }
      mbar_arrive_expect_tx(&full[s], Cfg::kStage);
      const int kx = (k0 + it) * BK;
      if constexpr (CN == 1) {
        tma_load_2d(st, &ta_hi, kx, m0, &full[s]);
        tma_load_2d(st + kSlabA, &ta_lo, kx, m0, &full[s]);
      } else {  // my 1/CN share of the A rows, to every CTA of my M tile
        constexpr int rows = kTileM / CN, bytes = rows * BK * 4;
        tma_load_2d_mc(st + cx * bytes, &ta_hi, kx, m0 + cx * rows, &full[s], mask_a);
        tma_load_2d_mc(st + kSlabA + cx * bytes, &ta_lo, kx, m0 + cx * rows, &full[s], mask_a);
      }
      if constexpr (CM == 1) {
        tma_load_2d(st + 2 * kSlabA, &tb_hi, kx, n0, &full[s]);
        tma_load_2d(st + 2 * kSlabA + Cfg::kSlabB, &tb_lo, kx, n0, &full[s]);
      } else {  // my 1/CM share of the B rows, to every CTA of my N tile
        constexpr int rows = NT / CM, bytes = rows * BK * 4;
        tma_load_2d_mc(st + 2 * kSlabA + cy * bytes, &tb_hi, kx, n0 + cy * rows, &full[s],
                       mask_b);
        tma_load_2d_mc(st + 2 * kSlabA + Cfg::kSlabB + cy * bytes, &tb_lo, kx, n0 + cy * rows,
                       &full[s], mask_b);
      }
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
      for (int kk = 0; kk < BK / 8; ++kk) {
        if (e.dbg != 0) break;
        const uint32_t o = kk * 32;
        // the two correction products accumulate in their own TMEM tile
        // (columns NT..2NT): the main accumulator then takes K/8 rounding
        // steps instead of 3K/8 (the tensor core's fp32 accumulation
        // truncates, so its error grows with the step count)
        mma_tf32(tmem, sdesc<BK>(a_hi + o), sdesc<BK>(b_hi + o), id, (it | kk) != 0);
        mma_tf32(tmem + NT, sdesc<BK>(a_lo + o), sdesc<BK>(b_hi + o), id, (it | kk) != 0);
        mma_tf32(tmem + NT, sdesc<BK>(a_hi + o), sdesc<BK>(b_lo + o), id, 1);
      }
      if constexpr (CS > 1)
        mma_commit_mc(&empty[s], (uint16_t)((1u << CS) - 1));
      else
        mma_commit(&empty[s]);
    }
    mma_commit(&done);
  } else if (warp < 4) {  // epilogue
    // pass 1 (thread = TMEM lane = tile row): accumulators + bias → a padded
    // [128][36] shared-memory tile per 32-column chunk (the TMA ring is dead
    // once `done` fired); pass 2: 8 lanes per row, float4 per lane — residual,
    // ReLU / mask and the output stores as 128-byte row segments (coalesced),
    // instead of one 16-byte store per thread per row.  Same arithmetic.
    float* stile = reinterpret_cast<float*>(smem);
    constexpr int kLd = 36;  // floats per staged row (16-byte aligned, spreads banks)
    constexpr int kRows = kTileM / 16;  // pass-2 rows per thread per chunk
    const int r_loc = 32 * warp + lane;
    const int sub = lane & 7, rq = lane >> 3;  // pass 2: column quad, row in the group
    // residual (hi, lo) and ReLU-mask quads of a chunk: all of a thread's
    // loads issued before the first is used (not one dependent round trip
    // per staged row)
    const bool vec_ok = ((e.ldr | e.ldm) & 3) == 0 &&
                        (((uintptr_t)e.r_hi | (uintptr_t)e.r_lo | (uintptr_t)e.mask) & 15) == 0;
    constexpr int kHalf = kRows / 2;  // rows whose loads are in flight together (measured: 2 > 4, 8 rows)
    float4 rh[kHalf], rl[kHalf], mk[kHalf];
    const bool epi_loads = e.r_hi || e.mask;
    if (e.bias) {  // staged while the k-loop runs (was a global load per element)
      for (int c = threadIdx.x; c < NT; c += 128) sbias[c] = n0 + c < e.N ? e.bias[n0 + c] : 0.f;
      group_bar(1, 128);
    }
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
    for (int ch = 0; ch < NT / 32; ++ch) {
      const int c0 = n0 + 32 * ch;
      if (c0 >= e.ldc) break;  // warp-uniform
      float v[32], w[32];
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + 32 * ch, v);
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + NT + 32 * ch, w);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 x;
        float* xs = &x.x;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          float t = v[j] + w[j];
          if (e.bias && c0 + j < e.N) t += sbias[32 * ch + j];
          xs[u] = t;
        }
        *reinterpret_cast<float4*>(stile + r_loc * kLd + 4 * q) = x;
      }
      group_bar(1, 128);
      const int col = c0 + 4 * sub;
#pragma unroll 1
      for (int i0 = 0; i0 < kRows; i0 += kHalf) {
        if (epi_loads) {  // issue kHalf rows' loads together
#pragma unroll
          for (int q = 0; q < kHalf; ++q) {
            const int row = m0 + 4 * warp + rq + 16 * (i0 + q);
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            rh[q] = z; rl[q] = z; mk[q] = make_float4(1.f, 1.f, 1.f, 1.f);
            if (row < e.M && col < e.N) {
              const size_t ri = (size_t)row * e.ldr + col, mi = (size_t)row * e.ldm + col;
              if (vec_ok && col + 4 <= e.N) {
                if (e.r_hi) rh[q] = __ldg(reinterpret_cast<const float4*>(e.r_hi + ri));
                if (e.r_lo) rl[q] = __ldg(reinterpret_cast<const float4*>(e.r_lo + ri));
                if (e.mask) mk[q] = __ldg(reinterpret_cast<const float4*>(e.mask + mi));
              } else {
                float* h = &rh[q].x; float* l = &rl[q].x; float* m = &mk[q].x;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (col + u < e.N) {
                    if (e.r_hi) h[u] = e.r_hi[ri + u];
                    if (e.r_lo) l[u] = e.r_lo[ri + u];
                    if (e.mask) m[u] = e.mask[mi + u];
                  }
              }
            }
          }
        }
#pragma unroll
        for (int ih = 0; ih < kHalf; ++ih) {
          const int rr = 4 * warp + rq + 16 * (i0 + ih), row = m0 + rr;
          float4 x = *reinterpret_cast<const float4*>(stile + rr * kLd + 4 * sub);
          float* xs = &x.x;
          const float* h = &rh[ih].x; const float* l = &rl[ih].x; const float* m = &mk[ih].x;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float t = xs[u];
            if (col + u < e.N) {
              if (e.r_hi) t += h[u] + l[u];
              if (e.relu) t = fmaxf(t, 0.f);
              if (e.mask && !(m[u] > 0.f)) t = 0.f;
            } else {
              t = 0.f;
            }
            xs[u] = t;
          }
          if (row >= e.M) continue;
          if (e.c) {
            *reinterpret_cast<float4*>(e.c + blockIdx.z * e.split_stride + (size_t)row * e.ldc + col) = x;
          } else {
            float4 hh, ll;
            hh.x = tf32_hi(x.x); hh.y = tf32_hi(x.y); hh.z = tf32_hi(x.z); hh.w = tf32_hi(x.w);
            ll.x = x.x - hh.x; ll.y = x.y - hh.y; ll.z = x.z - hh.z; ll.w = x.w - hh.w;
            *reinterpret_cast<float4*>(e.c_hi + (size_t)row * e.ldc + col) = hh;
            *reinterpret_cast<float4*>(e.c_lo + (size_t)row * e.ldc + col) = ll;
          }
        }
      }
      group_bar(1, 128);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_all();  // no peer still writes into this CTA
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
  int n, kp;     // image rows, row length written
  int seg, segp; // real / padded k per segment (seg == 0: one segment of k_real)
  int k_real;
  int n_src;     // row stride of W (its column count)
  int col0;      // first W column used (QKV: Wq | Wk | Wv concatenated by entries)
  // plain (backward) entries: dst[r * dst_ld + c] = W[k(r)][col0 + c] for
  // c < ncols_real (the dX = dY W operand: rows = W rows, k = W columns)
  int plain, dst_ld, ncols_real;
};

// segment map of the k index: image position q → W row (−1: zero pad)
__device__ __forceinline__ int image_k(const ImgEntry& E, int q) {
  if (E.seg) {
    const int sgi = q / E.segp, j = q - sgi * E.segp;
    return j < E.seg ? sgi * E.seg + j : -1;
  }
  return q < E.k_real ? q : -1;
}

// 32 × 32 tiles of one entry per block iteration (blockDim 32 × 8): plain
// entries copy rows (coalesced both ways); transposed ones read 32 W rows ×
// 32 consecutive columns and write 32 image rows × 32 consecutive k through a
// padded shared tile (the per-element transposed read of round 1 touched a
// 32-byte sector per float)
__global__ void build_image_kernel(const float* __restrict__ P, const ImgEntry* __restrict__ ents,
                                   int n_ents, float* __restrict__ img_hi,
                                   float* __restrict__ img_lo) {
  __shared__ float tile[32][33];
  const ImgEntry E = ents[blockIdx.y];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tk = (E.kp + 31) / 32, tiles = ((E.n + 31) / 32) * tk;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int n0 = (t / tk) * 32, k0 = (t % tk) * 32;
    if (E.plain) {
      for (int r = ty; r < 32; r += 8) {
        const int n = n0 + r, kq = k0 + tx;
        if (n >= E.n || kq >= E.kp) continue;
        const int k = image_k(E, n);
        const float v =
            (k >= 0 && kq < E.ncols_real) ? P[E.src + (int64_t)k * E.n_src + E.col0 + kq] : 0.f;
        const int64_t o = E.dst + (int64_t)n * E.dst_ld + kq;
        const float h = tf32_hi(v);
        img_hi[o] = h;
        img_lo[o] = v - h;
      }
      continue;
    }
    for (int r = ty; r < 32; r += 8) {
      const int kq = k0 + r, n = n0 + tx;
      const int k = kq < E.kp ? image_k(E, kq) : -1;
      tile[r][tx] = (k >= 0 && n < E.n) ? P[E.src + (int64_t)k * E.n_src + E.col0 + n] : 0.f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int n = n0 + r, kq = k0 + tx;
      if (n < E.n && kq < E.kp) {
        const float v = tile[tx][r];
        const int64_t o = E.dst + (int64_t)n * E.kp + kq;
        const float h = tf32_hi(v);
        img_hi[o] = h;
        img_lo[o] = v - h;
      }
    }
    __syncthreads();
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
    const float v = lane < TPCB_FEAT ? px[(size_t)(r0 + l) * TPCB_FEAT_PAD + lane] : 0.f;
    const float h = tf32_hi(v);
    x_hi[(size_t)(t0 + l) * 32 + lane] = h;
    x_lo[(size_t)(t0 + l) * 32 + lane] = v - h;
  }
}

// per (AST, head): ctx = softmax(q kᵀ / sqrt(dh)) v over the AST's own L rows
// (nn.py:79-96); writes the (hi, lo) pair, zeroes the pad columns
// lanes per score pair in the attention kernels: the L² dot products over
// the head dimension are split across groups of g lanes (g a power of two,
// g · L² <= 128 threads) and summed by an xor tree — at the typical L of
// 3–4 a thread used to walk all dh = 179 products of its pair alone
__device__ __forceinline__ int score_group(int L) {
  int g = 32;
  while (g > 1 && g * L * L > 128) g >>= 1;
  return g;
}
__device__ __forceinline__ float group_sum(float v, int g) {
  for (int o = g >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void attention_kernel(const float* __restrict__ qkv, int ldq,
                                 const int32_t* __restrict__ tok_off, int d, int nh, int dh,
                                 float scale, int ldc, float* __restrict__ c_hi,
                                 float* __restrict__ c_lo, int lcap) {
  extern __shared__ float sm[];  // q, k, v: lcap rows each (lcap = the launch's max L)
  const int s = blockIdx.x, h = blockIdx.y;
  const int t0 = tok_off[s], L = tok_off[s + 1] - t0;
  const int dhp = dh + 1;  // odd stride: conflict-free row reads
  float* q = sm;
  float* k = q + lcap * dhp;
  float* v = k + lcap * dhp;
  float* p = v + lcap * dhp;  // [16][17]
  for (int e = threadIdx.x; e < L * dh; e += blockDim.x) {
    const int l = e / dh, j = e - l * dh;
    const float* row = qkv + (size_t)(t0 + l) * ldq + h * dh + j;
    q[l * dhp + j] = row[0];
    k[l * dhp + j] = row[d];
    v[l * dhp + j] = row[2 * d];
  }
  __syncthreads();
  {
    const int g = score_group(L), sl = threadIdx.x & (g - 1), ng = blockDim.x / g;
    for (int e0 = 0; e0 < L * L; e0 += ng) {  // uniform trip count: full-warp shuffles
      const int e = e0 + threadIdx.x / g, i = e / L, j = e - i * L;
      float acc = 0.f;
      if (e < L * L)
        for (int c = sl; c < dh; c += g) acc = fmaf(q[i * dhp + c], k[j * dhp + c], acc);
      acc = group_sum(acc, g);
      if (e < L * L && sl == 0) p[i * 17 + j] = acc * scale;
    }
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
                              int32_t* __restrict__ status, int sorted_out) {
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
    const int i = sorted_out ? s : perm[s];
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
            int box_rows, int box_cols = 32) {
  EncodeFn enc;
  if (int st = get_encoder(&enc)) return st;
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)stride * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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


template <int NT, int BK, int CN, int CM>
int launch_gemm_cl(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st,
                   int splits, int* splits_used) {
  using Cfg = GemmCfg<NT, BK>;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  int rc = tmap_2d(&ta_hi, A.hi, A.k_ext, A.rows, A.ld, kTileM / CN, BK);
  if (!rc) rc = tmap_2d(&ta_lo, A.lo, A.k_ext, A.rows, A.ld, kTileM / CN, BK);
  if (!rc) rc = tmap_2d(&tb_hi, B.hi, B.k_ext, B.rows, B.ld, NT / CM, BK);
  if (!rc) rc = tmap_2d(&tb_lo, B.lo, B.k_ext, B.rows, B.ld, NT / CM, BK);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(gemm3_kernel<NT, BK, CN, CM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmem));
    if (CN * CM > 1)
      TPCB_CUDA_CHECK(cudaFuncSetAttribute(gemm3_kernel<NT, BK, CN, CM>,
                                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const int k_total = (int)(A.k_ext / BK);
  const int kc = ceil_div(k_total, splits);
  splits = ceil_div(k_total, kc);  // every split gets >= 1 slab
  if (splits_used) *splits_used = splits;
  const int gx = ceil_div(ceil_div(e.ldc, NT), CN) * CN;
  const int gy = ceil_div(ceil_div(e.M, kTileM), CM) * CM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)gx, (unsigned)gy, (unsigned)splits);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = Cfg::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = CM;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  Epi ee = e;
  ee.dbg = knobs().gemm_mode;
  TPCB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm3_kernel<NT, BK, CN, CM>, ta_hi, ta_lo, tb_hi,
                                     tb_lo, kc, k_total, ee));
  TPCB_LAUNCH_CHECK("gemm3");
  return TPCB_OK;
}

// cluster shape: share a tile only along a dimension with an even tile count
// (no padded CTAs)
template <int NT, int BK>
int launch_gemm_bk(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st,
                   int splits, int* splits_used) {
  const int tn = ceil_div(e.ldc, NT), tm = ceil_div(e.M, kTileM);
  const bool cn = knobs().gemm_cluster && tn % 2 == 0, cm = knobs().gemm_cluster && tm % 2 == 0;
  if (cn && cm) return launch_gemm_cl<NT, BK, 2, 2>(A, B, e, st, splits, splits_used);
  if (cm) return launch_gemm_cl<NT, BK, 1, 2>(A, B, e, st, splits, splits_used);
  if (cn) return launch_gemm_cl<NT, BK, 2, 1>(A, B, e, st, splits, splits_used);
  return launch_gemm_cl<NT, BK, 1, 1>(A, B, e, st, splits, splits_used);
}

// splits count k-slabs of 32 columns (callers' unit), whatever the slab width
template <int NT>
int launch_gemm_nt(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st,
                   int splits = 1, int* splits_used = nullptr) {
  // k-slab width: 16 columns (64-byte swizzle, 6-stage ring) for tall
  // products (inference batches: +3 %), 32 (128-byte swizzle, 3 stages) for
  // the M ~ 600·L training products (full_reference_config step −6 %);
  // TPCB_GEMM_BK forces one
  const int bk = knobs().gemm_bk ? knobs().gemm_bk : (A.rows >= 8192 ? 16 : 32);
  if (bk == 16) return launch_gemm_bk<NT, 16>(A, B, e, st, splits, splits_used);
  return launch_gemm_bk<NT, 32>(A, B, e, st, splits, splits_used);
}

int launch_gemm(const Operand& A, const Operand& B, const Epi& e, cudaStream_t st) {
  if (A.k_ext != B.k_ext || (A.k_ext & 31)) return TPCB_ERR_VALIDATION;
  const int64_t m_tiles = ceil_div(e.M, kTileM);
  // 256-wide tiles for large products (>= 4 waves: operand reuse wins), and
  // for smaller ones only when they quantise into waves no worse than
  // 128-wide tiles (the training QKV product: 171 tiles of 256 = 2 waves of
  // 256-wide work vs 323 of 128 = 3 waves of 128-wide; 1.2 % per step)
  const int64_t t256 = m_tiles * ceil_div(e.ldc, 256), t128 = m_tiles * ceil_div(e.ldc, 128);
  const int64_t w256 = ceil_div(t256, (int64_t)kNumSMs), w128 = ceil_div(t128, (int64_t)kNumSMs);
  if (e.ldc > 128 && t256 >= kNumSMs && (w256 >= 4 || 2 * w256 <= w128))
    return launch_gemm_nt<256>(A, B, e, st);
  return launch_gemm_nt<128>(A, B, e, st);
}

// ---- image plan (shared by the forward, training and the ABI size query) --
struct LargePlan {
  int d, dp, ff, ffp, qkv, qkvp, de, dep;
  int64_t in, layer[TPCB_MAX_LAYERS][4], leaf[TPCB_MAX_LEAF + 1], dec[TPCB_MAX_DEC];
  // backward operands (plain layout): [0] Wq|Wk|Wv [d][qkvp], [1] Wo [d][dp],
  // [2] fhW [d][ffp], [3] foW [ff][dp]; leaf [L·dp][dep]; dec [in][pad(out)]
  int64_t layer_b[TPCB_MAX_LAYERS][4], leaf_b[TPCB_MAX_LEAF + 1], dec_b[TPCB_MAX_DEC];
  int dec_kp[TPCB_MAX_DEC];
  int64_t bias_qkv[TPCB_MAX_LAYERS];  // concatenated QKV bias (in the bias image)
  int64_t img_floats, img_floats_fwd, bias_floats;
  int n_ents_fwd;
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
    ImgEntry E{src, o, n, kp, seg, segp, k_real, n_src, col0, 0, kp, 0};
    p.ents.push_back(E);
    const int64_t at = o;
    o += (int64_t)n * kp;
    return at;
  };
  // plain entry writing rows × ncols_pad at `at` (row stride ld, column c0)
  auto add_plain = [&](int64_t at, int64_t src, int rows, int k_real, int seg, int segp,
                       int n_src, int col0, int ncols_real, int ncols_pad, int ld) {
    ImgEntry E{src, at, rows, ncols_pad, seg, segp, k_real, n_src, col0, 1, ld, ncols_real};
    p.ents.push_back(E);
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
  p.img_floats_fwd = o;
  p.n_ents_fwd = (int)p.ents.size();
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& L = M.layer[li];
    p.layer_b[li][0] = o;
    add_plain(o, L.Wq, M.d, M.d, 0, 0, M.d, 0, M.d, M.d, p.qkvp);
    add_plain(o + M.d, L.Wk, M.d, M.d, 0, 0, M.d, 0, M.d, M.d, p.qkvp);
    add_plain(o + 2 * M.d, L.Wv, M.d, M.d, 0, 0, M.d, 0, M.d, M.d, p.qkvp);
    o += (int64_t)M.d * p.qkvp;
    p.layer_b[li][1] = o;
    add_plain(o, L.Wo, M.d, M.d, 0, 0, M.d, 0, M.d, p.dp, p.dp);
    o += (int64_t)M.d * p.dp;
    p.layer_b[li][2] = o;
    add_plain(o, L.fhW, M.d, M.d, 0, 0, M.d_ff, 0, M.d_ff, p.ffp, p.ffp);
    o += (int64_t)M.d * p.ffp;
    p.layer_b[li][3] = o;
    add_plain(o, L.foW, M.d_ff, M.d_ff, 0, 0, M.d, 0, M.d, p.dp, p.dp);
    o += (int64_t)M.d_ff * p.dp;
  }
  for (int l = 1; l <= M.n_leaf_max; ++l) {
    p.leaf_b[l] = o;
    add_plain(o, M.leafW[l], l * p.dp, l * M.d, M.d, p.dp, M.d_e, 0, M.d_e, p.dep, p.dep);
    o += (int64_t)l * p.dp * p.dep;
  }
  kin = M.d_e;
  for (int i = 0; i < M.n_dec; ++i) {
    const int op = pad32(M.dec[i]);
    p.dec_b[i] = o;
    add_plain(o, M.decW[i], kin, kin, 0, 0, M.dec[i], 0, M.dec[i], op, op);
    o += (int64_t)kin * op;
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

// ---------------------------------------------------------------- workspace
// Forward activations.  Training keeps one copy per layer (for the backward);
// inference aliases every layer onto one set (layer stride 0).
struct Pair {
  float* hi;
  float* lo;
};

struct Fwd {
  int64_t T, A;            // padded token / AST rows
  size_t sd, sq, sf;       // per-layer strides (0 = every layer aliased: inference)
  float *x_hi, *x_lo;
  float *h_hi, *h_lo;      // [nl + 1] layer inputs / final output  [T, dp]
  float *qkv;              // [nl] [T, qkvp] fp32
  float *c_hi, *c_lo;      // [nl] attention context [T, dp]
  float *s1, *s2;          // [nl] pre-LayerNorm sums [T, dp] fp32
  float *h1_hi, *h1_lo;    // [nl] [T, dp]
  float *f_hi, *f_lo;      // [nl] [T, ffp]
  float *zx, *z_hi, *z_lo; // [A, dep]
  float *dec_hi[TPCB_MAX_DEC], *dec_lo[TPCB_MAX_DEC];
  float *pred;             // [A] sorted order (training)
  int32_t *idx, *tok_off;
  Pair H(int l) const { return {h_hi + l * sd, h_lo + l * sd}; }
  float* QKV(int l) const { return qkv + l * sq; }
  Pair C(int l) const { return {c_hi + l * sd, c_lo + l * sd}; }
  float* S1(int l) const { return s1 + l * sd; }
  float* S2(int l) const { return s2 + l * sd; }
  Pair H1(int l) const { return {h1_hi + l * sd, h1_lo + l * sd}; }
  Pair F(int l) const { return {f_hi + l * sf, f_lo + l * sf}; }
};

struct Carver {
  uint8_t* base;
  size_t o = 0;
  float* take(size_t floats) {
    float* r = reinterpret_cast<float*>(base ? base + o : nullptr);
    o = align256(o + floats * 4);
    return r;
  }
};

int dec_max(const Model& M) {
  int dmax = 32;
  for (int i = 0; i < M.n_dec; ++i) dmax = max(dmax, pad32(M.dec[i]));
  return dmax;
}

Fwd carve_fwd(const LargePlan& p, const Model& M, int64_t n_tok, int64_t n_ast, bool train,
              Carver* cv) {
  Fwd f{};
  f.T = ((n_tok + kTileM - 1) / kTileM) * kTileM;
  f.A = ((n_ast + kTileM - 1) / kTileM) * kTileM;
  const size_t td = (size_t)f.T * p.dp, tq = (size_t)f.T * p.qkvp, tf = (size_t)f.T * p.ffp;
  const size_t nl = train ? M.n_layers : 1;
  f.sd = train ? td : 0;
  f.sq = train ? tq : 0;
  f.sf = train ? tf : 0;
  f.x_hi = cv->take(f.T * 32);
  f.x_lo = cv->take(f.T * 32);
  f.h_hi = cv->take((train ? nl + 1 : 1) * td);
  f.h_lo = cv->take((train ? nl + 1 : 1) * td);
  f.qkv = cv->take(nl * tq);
  f.c_hi = cv->take(nl * td);
  f.c_lo = cv->take(nl * td);
  f.s1 = cv->take(nl * td);
  f.s2 = train ? cv->take(nl * td) : f.s1;
  f.h1_hi = cv->take(nl * td);
  f.h1_lo = cv->take(nl * td);
  f.f_hi = cv->take(nl * tf);
  f.f_lo = cv->take(nl * tf);
  f.zx = cv->take(f.A * p.dep);
  f.z_hi = cv->take(f.A * p.dep);
  f.z_lo = cv->take(f.A * p.dep);
  const int dmax = dec_max(M);
  for (int i = 0; i < M.n_dec; ++i) {
    if (train || i < 2) {
      f.dec_hi[i] = cv->take(f.A * (train ? pad32(M.dec[i]) : dmax));
      f.dec_lo[i] = cv->take(f.A * (train ? pad32(M.dec[i]) : dmax));
    } else {  // inference ping-pong
      f.dec_hi[i] = f.dec_hi[i - 2];
      f.dec_lo[i] = f.dec_lo[i - 2];
    }
  }
  f.pred = cv->take(f.A);
  f.idx = reinterpret_cast<int32_t*>(cv->take(n_ast + 1));
  f.tok_off = reinterpret_cast<int32_t*>(cv->take(n_ast + 1));
  return f;
}

}  // namespace

bool large_supported(const Model& M) {
  return M.d_dev <= 1024 && M.n_heads * M.dh == M.d && M.dh <= 1024 &&
         (size_t)3 * TPCB_MAX_LEAF * (M.dh + 1) * 4 + 17 * 16 * 4 <= 200 * 1024;
}

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

struct Ctx {
  const Model& M;
  const LargePlan& p;
  const float* P;
  ImagePtrs im;
  cudaStream_t st;
  Operand W(int64_t off, int n, int kp) const { return Operand{im.hi + off, im.lo + off, n, kp, kp}; }
};

Operand act_op(const float* hi, const float* lo, int64_t rows, int ld) {
  return Operand{hi, lo, rows, ld, ld};
}

// the forward over the sorted tokens already gathered into f.x (host-side
// bucket structure h_tok_off); latents / pred scattered by f.idx unless
// `train` (then pred stays in sorted order in f.pred)
// the largest leaf count of a batch (attention's shared-memory rows; the
// training batches are single-bucket, so this is usually their L); long
// inference batches keep the cap instead of scanning
int max_leaf_count(const int32_t* h_tok_off, int64_t n) {
  if (n > 65536) return TPCB_MAX_LEAF;
  int m = 1;
  for (int64_t s = 0; s < n; ++s) m = std::max(m, h_tok_off[s + 1] - h_tok_off[s]);
  return std::min(m, TPCB_MAX_LEAF);
}

int run_forward(const Ctx& c, const Fwd& f, int64_t n_ast, const int32_t* h_tok_off,
                const float* d_devfeat, bool train, const tpcb_boxcox& bc, float* d_pred,
                float* d_zx, float* d_zv, float* d_z, double* d_lat, int32_t* d_status) {
  const Model& M = c.M;
  const LargePlan& p = c.p;
  const float* P = c.P;
  cudaStream_t st = c.st;
  const int64_t n_tok = h_tok_off[n_ast];
  int rc;
  {
    Pair h = f.H(0);
    Epi e{(int)n_tok, M.d, p.dp, P + M.inb, 0, nullptr, nullptr, 0, nullptr, h.hi, h.lo};
    if ((rc = launch_gemm(act_op(f.x_hi, f.x_lo, n_tok, 32), c.W(p.in, M.d, 32), e, st)))
      return rc;
  }
  const float scale = 1.0f / sqrtf((float)M.dh);
  const size_t att_smem = (size_t)(3 * TPCB_MAX_LEAF * (M.dh + 1) + 16 * 17) * 4;
  if (att_smem > 48 * 1024)
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(attention_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)att_smem));
  const int lcap = max_leaf_count(h_tok_off, n_ast);
  const size_t att_used = (size_t)(3 * lcap * (M.dh + 1) + 16 * 17) * 4;
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& L = M.layer[li];
    const Pair h = f.H(li), hn = f.H(li + 1), ctx = f.C(li), h1 = f.H1(li), ff = f.F(li);
    float* qkv = f.QKV(li);
    {
      Epi e{(int)n_tok, p.qkv, p.qkvp, c.im.bias + p.bias_qkv[li], 0, nullptr, nullptr, 0, qkv,
            nullptr, nullptr};
      if ((rc = launch_gemm(act_op(h.hi, h.lo, n_tok, p.dp), c.W(p.layer[li][0], p.qkv, p.dp), e,
                            st)))
        return rc;
    }
    attention_kernel<<<dim3((unsigned)n_ast, M.n_heads), 128, att_used, st>>>(
        qkv, p.qkvp, f.tok_off, M.d, M.n_heads, M.dh, scale, p.dp, ctx.hi, ctx.lo, lcap);
    TPCB_LAUNCH_CHECK("large_attention");
    {
      Epi e{(int)n_tok, M.d, p.dp, P + L.bo, 0, h.hi, h.lo, p.dp, f.S1(li), nullptr, nullptr};
      if ((rc = launch_gemm(act_op(ctx.hi, ctx.lo, n_tok, p.dp), c.W(p.layer[li][1], M.d, p.dp),
                            e, st)))
        return rc;
    }
    layernorm_kernel<<<ceil_div(n_tok, 8), 256, 0, st>>>(f.S1(li), p.dp, (int)n_tok, M.d,
                                                         P + L.ln1g, P + L.ln1b, h1.hi, h1.lo);
    {
      Epi e{(int)n_tok, M.d_ff, p.ffp, P + L.fhb, 1, nullptr, nullptr, 0, nullptr, ff.hi, ff.lo};
      if ((rc = launch_gemm(act_op(h1.hi, h1.lo, n_tok, p.dp),
                            c.W(p.layer[li][2], M.d_ff, p.dp), e, st)))
        return rc;
    }
    {
      Epi e{(int)n_tok, M.d, p.dp, P + L.fob, 0, h1.hi, h1.lo, p.dp, f.S2(li), nullptr, nullptr};
      if ((rc = launch_gemm(act_op(ff.hi, ff.lo, n_tok, p.ffp), c.W(p.layer[li][3], M.d, p.ffp),
                            e, st)))
        return rc;
    }
    layernorm_kernel<<<ceil_div(n_tok, 8), 256, 0, st>>>(f.S2(li), p.dp, (int)n_tok, M.d,
                                                         P + L.ln2g, P + L.ln2b, hn.hi, hn.lo);
    TPCB_LAUNCH_CHECK("large_layernorm");
  }
  const Pair hf = f.H(M.n_layers);
  for (int64_t s0 = 0; s0 < n_ast;) {  // leaf_embed.{L}: bucket L as [n_L, L·dp]
    const int Lb = h_tok_off[s0 + 1] - h_tok_off[s0];
    int64_t s1 = s0 + 1;
    while (s1 < n_ast && h_tok_off[s1 + 1] - h_tok_off[s1] == Lb) ++s1;
    const int64_t nb = s1 - s0, t0 = h_tok_off[s0];
    Operand A{hf.hi + t0 * p.dp, hf.lo + t0 * p.dp, nb, (int64_t)Lb * p.dp, (int64_t)Lb * p.dp};
    Epi e{(int)nb, M.d_e, p.dep, P + M.leafb[Lb], 0, nullptr, nullptr, 0, f.zx + s0 * p.dep,
          nullptr, nullptr};
    if ((rc = launch_gemm(A, c.W(p.leaf[Lb], M.d_e, Lb * p.dp), e, st))) return rc;
    s0 = s1;
  }
  device_gate_kernel<<<(unsigned)n_ast, 128, M.d_dev * 4, st>>>(M, P, d_devfeat, f.idx, f.zx,
                                                                 p.dep, f.z_hi, f.z_lo, d_zx,
                                                                 d_zv, d_z);
  TPCB_LAUNCH_CHECK("large_device_gate");
  const float* in_hi = f.z_hi;
  const float* in_lo = f.z_lo;
  int ldin = p.dep;
  for (int i = 0; i < M.n_dec; ++i) {
    const int ldo = pad32(M.dec[i]);
    Epi e{(int)n_ast, M.dec[i], ldo, P + M.decb[i], 1, nullptr, nullptr, 0, nullptr,
          f.dec_hi[i], f.dec_lo[i]};
    if ((rc = launch_gemm(act_op(in_hi, in_lo, n_ast, ldin), c.W(p.dec[i], M.dec[i], p.dec_kp[i]),
                          e, st)))
      return rc;
    in_hi = f.dec_hi[i];
    in_lo = f.dec_lo[i];
    ldin = ldo;
  }
  output_kernel<<<ceil_div(n_ast, 8), 256, 0, st>>>(
      M, P, in_hi, in_lo, ldin, M.n_dec ? M.dec[M.n_dec - 1] : M.d_e, f.idx, (int)n_ast, bc,
      train ? f.pred : d_pred, train ? nullptr : d_lat, d_status, train ? 1 : 0);
  TPCB_LAUNCH_CHECK("large_output");
  return TPCB_OK;
}

}  // namespace
}  // namespace tpcb

using namespace tpcb;

extern "C" int tpcb_large_sizes(const tpcb_model* m, int64_t n_ast, int64_t n_tok,
                                size_t* image_bytes, size_t* act_bytes) {
  if (!m || !image_bytes || !act_bytes) return TPCB_ERR_VALIDATION;
  if (!large_supported(m->dev)) return TPCB_ERR_UNSUPPORTED;
  const LargePlan p = make_plan(m->dev);
  *image_bytes = align256((size_t)p.img_floats * 4) * 2 + align256((size_t)p.bias_floats * 4) +
                 align256(p.ents.size() * sizeof(ImgEntry)) + 256 * 2;
  Carver cv{nullptr};
  carve_fwd(p, m->dev, n_tok, n_ast, false, &cv);
  *act_bytes = cv.o;
  return TPCB_OK;
}

// weight image: the transposed (hi, lo) B operands of every forward GEMM
// (+ the plain operands of the backward's dX GEMMs when with_backward) and
// the concatenated QKV biases; rebuild after every parameter update.  The
// image must be zero-filled once at allocation (pad columns stay zero).
extern "C" int tpcb_large_prepare(const tpcb_model* m, const float* d_params, void* d_image,
                                  int32_t with_backward, void* stream_) {
  if (!m || !d_params || !d_image) return TPCB_ERR_VALIDATION;
  if (!large_supported(m->dev)) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t st = (cudaStream_t)stream_;
  const LargePlan p = make_plan(m->dev);
  ImagePtrs im = carve_image(p, (uint8_t*)d_image);
  int64_t* d_off = reinterpret_cast<int64_t*>(im.ents + p.ents.size());
  d_off = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(d_off) + 255) & ~uintptr_t(255));
  // entry table + offsets (a few KB; a pageable copy synchronises the stream,
  // so callers that rebuild every step pass bit 1 after the first call)
  if (!(with_backward & 2)) {
    TPCB_CUDA_CHECK(cudaMemcpyAsync(im.ents, p.ents.data(), p.ents.size() * sizeof(ImgEntry),
                                    cudaMemcpyHostToDevice, st));
    TPCB_CUDA_CHECK(cudaMemcpyAsync(d_off, p.bias_qkv, sizeof(int64_t) * m->dev.n_layers,
                                    cudaMemcpyHostToDevice, st));
  }
  const int n_ents = (with_backward & 1) ? (int)p.ents.size() : p.n_ents_fwd;
  build_image_kernel<<<dim3(64, (unsigned)n_ents), dim3(32, 8), 0, st>>>(d_params, im.ents, n_ents, im.hi,
                                                                 im.lo);
  qkv_bias_kernel<<<dim3(8, m->dev.n_layers), 256, 0, st>>>(d_params, m->dev, d_off, im.bias);
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
  Carver cv{(uint8_t*)d_act};
  Fwd f = carve_fwd(p, M, n_tok, n_ast, false, &cv);
  if (cv.o > act_bytes) return TPCB_ERR_VALIDATION;
  TPCB_CUDA_CHECK(cudaMemcpyAsync(f.idx, h_perm, n_ast * 4, cudaMemcpyHostToDevice, st));
  TPCB_CUDA_CHECK(
      cudaMemcpyAsync(f.tok_off, h_tok_off, (n_ast + 1) * 4, cudaMemcpyHostToDevice, st));
  gather_tokens_kernel<<<ceil_div(n_ast, 8), 256, 0, st>>>(pk->x, f.idx, pk->ast_row, f.tok_off,
                                                           (int)n_ast, f.x_hi, f.x_lo);
  TPCB_LAUNCH_CHECK("large_gather");
  Ctx c{M, p, d_params, carve_image(p, (uint8_t*)const_cast<void*>(d_image)), st};
  tpcb_boxcox bc{};
  if (norm) bc = *norm;
  return run_forward(c, f, n_ast, h_tok_off, d_devfeat, false, bc, d_pred, d_zx, d_zv, d_z,
                     d_latency, d_status);
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

// =================================================================== training
// (costmodel.backward + nn.*_bwd for the large path: costmodel.py:280-336,
// 343-423, nn.py:30-120).  Every weight gradient is a split-K tcgen05 GEMM
// dW = Xᵀ·dY over the tokens (operands transposed + split by
// transpose_pair_kernel), reduced in fixed split order; every input gradient
// dX = dY·W is a GEMM on the plain weight image with the ReLU mask / residual
// fused into its epilogue; bias / LayerNorm-parameter gradients are
// deterministic column sums.  The flat gradient is fully rewritten per step.
namespace tpcb {
namespace {

// [rows, cols] (row stride ld; pair or fp32 when a_lo == null) → pair
// [cols][ldo], zero for rows <= r < ldo
// One transposed (hi, lo) operand: out[c][r] = split(in_hi[r][c] + in_lo[r][c])
// for c < cols, r < ldo (zero beyond `rows`); ones_col >= 0: that output row
// is all ones over the real rows (the bias gradient folded into the
// weight-gradient GEMM as one more product row).
struct TJob {
  const float* hi;
  const float* lo;
  int rows, cols, ld;
  float* o_hi;
  float* o_lo;
  int ldo, ones_col;
};

// both operands of a weight-gradient product in one launch (blockIdx.z);
// 64 × 64 tiles, 32 elements of each half per thread in flight.  A (hi, lo)
// input is an exact split (lo = x − tf32(x)), so re-splitting hi + lo gives
// the same pair back: the halves are transposed as they are; a plain input
// (lo == null) is split here.
__global__ void __launch_bounds__(256) transpose_pair_kernel(TJob j0, TJob j1) {
  const TJob J = blockIdx.z ? j1 : j0;
  const int cols_out = J.ones_col >= 0 ? J.ones_col + 1 : J.cols;
  const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
  if (c0 >= cols_out || r0 >= J.ldo) return;  // the grid covers the larger job
  __shared__ float th[64][65], tl[64][65];
  const int tx = threadIdx.x, ty = threadIdx.y;
  float vh[16], vl[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = r0 + ty + 8 * (i >> 1), c = c0 + tx + 32 * (i & 1);
    vh[i] = 0.f;
    vl[i] = 0.f;
    if (c == J.ones_col) {
      vh[i] = r < J.rows ? 1.f : 0.f;
    } else if (r < J.rows && c < J.cols) {
      vh[i] = J.hi[(size_t)r * J.ld + c];
      if (J.lo) vl[i] = J.lo[(size_t)r * J.ld + c];
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = ty + 8 * (i >> 1), cc = tx + 32 * (i & 1);
    float h = vh[i], l = vl[i];
    if (!J.lo) {
      h = tf32_hi(vh[i]);
      l = vh[i] - h;
    }
    th[rr][cc] = h;
    tl[rr][cc] = l;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int cc = ty + 8 * (i >> 1), rr = tx + 32 * (i & 1);
    const int c = c0 + cc, r = r0 + rr;
    if (c < cols_out && r < J.ldo) {
      J.o_hi[(size_t)c * J.ldo + r] = th[rr][cc];
      J.o_lo[(size_t)c * J.ldo + r] = tl[rr][cc];
    }
  }
}

// out[c] = Σ_r x[r][c] (+ x_lo) in fixed order; column c goes to tensor c / colw
struct ColDst {
  int colw;
  int64_t d[3];
  int acc = 0;  // 1: add into the gradient (second pass of a CMD step), 0: write
};

// two-stage deterministic column sums: chunks of 64 rows → partial[chunk][c],
// then the chunks in order
constexpr int kColChunk = 64;
constexpr int kColCntMax = 256;  // column-sum stripe counters per backward workspace

__global__ void colsum_partial_kernel(const float* __restrict__ x, const float* __restrict__ x_lo,
                                      int rows, int cols, int ld, float* __restrict__ part) {
  __shared__ float red[8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * kColChunk, r1 = min(r0 + kColChunk, rows);
  float acc = 0.f;
  if (c < cols) {  // the chunk's rows for this thread: loads first, adds in row order
    constexpr int kPer = kColChunk / 8;
    float xv[kPer], xl[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int r = r0 + threadIdx.y + 8 * u;
      xv[u] = r < r1 ? x[(size_t)r * ld + c] : 0.f;
      xl[u] = (r < r1 && x_lo) ? x_lo[(size_t)r * ld + c] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int r = r0 + threadIdx.y + 8 * u;
      if (r < r1) {
        acc += xv[u];
        if (x_lo) acc += xl[u];
      }
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    float s = red[0][threadIdx.x];
    for (int k = 1; k < 8; ++k) s += red[k][threadIdx.x];
    part[(size_t)blockIdx.y * cols + c] = s;
  }
}

// one launch: the chunk partials of colsum_partial_kernel, then the last chunk
// block of each 32-column stripe (a counter per stripe, reset for the next
// call) sums the stripe's partials in chunk order — colsum_final_kernel's fold
// gridDim.z == 2: a second job (x2, no lo part, dst2) over the same shape —
// its own partials and stripe counters (the LayerNorm γ / β pair)
__global__ void colsum_fused_kernel(const float* __restrict__ x, const float* __restrict__ x_lo,
                                    int rows, int cols, int ld, float* __restrict__ part,
                                    unsigned* __restrict__ cnt, ColDst dst,
                                    float* __restrict__ grad, const float* __restrict__ x2 = nullptr,
                                    ColDst dst2 = ColDst{1, {0, 0, 0}, 0}) {
  __shared__ float red[8][33];
  __shared__ bool last;
  if (blockIdx.z) {
    x = x2;
    x_lo = nullptr;
    dst = dst2;
    part += (size_t)gridDim.y * cols;
    cnt += kColCntMax / 2;
  }
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * kColChunk, r1 = min(r0 + kColChunk, rows);
  float acc = 0.f;
  if (c < cols) {  // the chunk's rows for this thread: loads first, adds in row order
    constexpr int kPer = kColChunk / 8;
    float xv[kPer], xl[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int r = r0 + threadIdx.y + 8 * u;
      xv[u] = r < r1 ? x[(size_t)r * ld + c] : 0.f;
      xl[u] = (r < r1 && x_lo) ? x_lo[(size_t)r * ld + c] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int r = r0 + threadIdx.y + 8 * u;
      if (r < r1) {
        acc += xv[u];
        if (x_lo) acc += xl[u];
      }
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0) {
    if (c < cols) {
      float s = red[0][threadIdx.x];
      for (int k = 1; k < 8; ++k) s += red[k][threadIdx.x];
      part[(size_t)blockIdx.y * cols + c] = s;
    }
    __threadfence();
    __syncwarp();
    if (threadIdx.x == 0) last = atomicAdd(&cnt[blockIdx.x], 1u) == gridDim.y - 1;
  }
  __syncthreads();
  if (!last || threadIdx.y != 0) return;
  __threadfence();
  if (c < cols) {
    const int chunks = gridDim.y;
    float s = __ldcg(part + c);
    int k = 1;
    for (; k + 8 <= chunks; k += 8) {  // 8 loads in flight, added in chunk order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (size_t)(k + u) * cols + c);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; k < chunks; ++k) s += __ldcg(part + (size_t)k * cols + c);
    const int t = c / dst.colw;
    float* g = grad + dst.d[t] + (c - t * dst.colw);
    *g = dst.acc ? *g + s : s;
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = 0;
}

__global__ void colsum_final_kernel(const float* __restrict__ part, int chunks, int cols,
                                    ColDst dst, float* __restrict__ grad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = part[c];
  int k = 1;
  for (; k + 8 <= chunks; k += 8) {  // 8 loads in flight, added in chunk order
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = part[(size_t)(k + u) * cols + c];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += x[u];
  }
  for (; k < chunks; ++k) s += part[(size_t)k * cols + c];
  const int t = c / dst.colw;
  float* g = grad + dst.d[t] + (c - t * dst.colw);
  *g = dst.acc ? *g + s : s;
}

// split-K partials [splits][rows][ldc] → grad, rows through the leaf segment
// map (seg > 0), columns split into ≤ 3 tensors of width colw
// bias (has_bias): product row `rows` is the column sum of dY (the ones row
// of the transposed X), written through bdst like colsum's final pass
__global__ void reduce_grad_kernel(const float* __restrict__ part, int splits, int64_t sstride,
                                   int rows, int cols, int ldc, int seg, int segp, ColDst dst,
                                   float* __restrict__ grad, int has_bias, ColDst bdst) {
  const int64_t total = (int64_t)(rows + has_bias) * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e - (int64_t)r * cols);
    if (r == rows) {
      float v = part[(size_t)r * ldc + c];
      for (int z = 1; z < splits; ++z) v += part[z * sstride + (size_t)r * ldc + c];
      const int t = c / bdst.colw;
      float* g = grad + bdst.d[t] + (c - t * bdst.colw);
      *g = bdst.acc ? *g + v : v;
      continue;
    }
    int rr = r;
    if (seg) {
      const int j = r % segp;
      if (j >= seg) continue;
      rr = (r / segp) * seg + j;
    }
    float v = part[(size_t)r * ldc + c];
    for (int z = 1; z < splits; ++z) v += part[z * sstride + (size_t)r * ldc + c];
    const int t = c / dst.colw;
    const int cc = c - t * dst.colw;
    float* g = grad + dst.d[t] + (int64_t)rr * dst.colw + cc;
    *g = dst.acc ? *g + v : v;
  }
}

// CMD plumbing (costmodel.py:426-486 runs on [zs; zt] in INPUT order, which
// matters for the first-argmax / argmin support routing): bucket-order latent
// row k (z = hi + lo, exact) → zall[base + pos[k]]
__global__ void z_scatter_kernel(const float* __restrict__ z_hi, const float* __restrict__ z_lo,
                                 int ldz, const int32_t* __restrict__ pos, int n, int de,
                                 int64_t base, float* __restrict__ zall) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * de; e += gridDim.x * blockDim.x) {
    const int k = e / de, c = e - k * de;
    zall[(base + pos[k]) * de + c] = z_hi[(size_t)k * ldz + c] + z_lo[(size_t)k * ldz + c];
  }
}

// dz[k] (+)= alpha · dCMD/dz[base + pos[k]] (fp64 gradient rows); with
// `set` the row is overwritten and its padding columns zeroed
__global__ void dz_from_cmd_kernel(float* __restrict__ dz, int ldz, const double* __restrict__ g,
                                   const int32_t* __restrict__ pos, int n, int de, int64_t base,
                                   double alpha, int set) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * ldz; e += gridDim.x * blockDim.x) {
    const int k = e / ldz, c = e - k * ldz;
    const float v = c < de ? (float)(alpha * g[(base + pos[k]) * de + c]) : 0.f;
    if (set) dz[e] = v;
    else if (c < de) dz[e] += v;
  }
}

// step loss += alpha · CMD (costmodel.py:556); CMD value copied out
__global__ void add_cmd_kernel(double* loss, const double* cmd, double alpha, double* cmd_out) {
  loss[0] += alpha * cmd[0];
  if (cmd_out) cmd_out[0] = cmd[0];
}

// LayerNorm backward (nn.py:57-66), one warp per row: dx = rstd·(dŷ − mean(dŷ)
// − x̂·mean(dŷ·x̂)), dŷ = dy·g; prod = dy·x̂ (→ dg by column sums)
// the row in registers (ld <= 32·PER): one load of x, dy and γ per element,
// all in flight together; same passes and order as ln_back_kernel
template <int PER>
__global__ void ln_back_reg_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                   int ld, int rows, int d, const float* __restrict__ g,
                                   float* __restrict__ dx_hi, float* __restrict__ dx_lo,
                                   float* __restrict__ prod) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const float* xr = x + (size_t)r * ld;
  const float* dr = dy + (size_t)r * ld;
  float xv[PER], dv[PER], gv[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = lane + 32 * u;
    xv[u] = j < d ? xr[j] : 0.f;
    dv[u] = j < d ? dr[j] : 0.f;
    gv[u] = j < d ? g[j] : 0.f;
  }
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (lane + 32 * u < d) s += xv[u];
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (lane + 32 * u < d) {
      const float t = xv[u] - mean;
      q = fmaf(t, t, q);
    }
  const float rstd = rsqrtf(warp_sum(q) / d + 1e-5f);
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (lane + 32 * u < d) {
      const float xh = (xv[u] - mean) * rstd, dxh = dv[u] * gv[u];
      s1 += dxh;
      s2 = fmaf(dxh, xh, s2);
    }
  const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int j = lane + 32 * u;
    if (j >= ld) break;
    float o = 0.f, pr = 0.f;
    if (j < d) {
      const float xh = (xv[u] - mean) * rstd, dxh = dv[u] * gv[u];
      o = rstd * (dxh - m1 - xh * m2);
      pr = dv[u] * xh;
    }
    const float h = tf32_hi(o);
    dx_hi[(size_t)r * ld + j] = h;
    dx_lo[(size_t)r * ld + j] = o - h;
    prod[(size_t)r * ld + j] = pr;
  }
}

__global__ void ln_back_kernel(const float* __restrict__ dy, const float* __restrict__ x, int ld,
                               int rows, int d, const float* __restrict__ g,
                               float* __restrict__ dx_hi, float* __restrict__ dx_lo,
                               float* __restrict__ prod) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const float* xr = x + (size_t)r * ld;
  const float* dr = dy + (size_t)r * ld;
  float s = 0.f;
  for (int j = lane; j < d; j += 32) s += xr[j];
  const float mean = warp_sum(s) / d;
  float q = 0.f;
  for (int j = lane; j < d; j += 32) {
    const float t = xr[j] - mean;
    q = fmaf(t, t, q);
  }
  const float rstd = rsqrtf(warp_sum(q) / d + 1e-5f);
  float s1 = 0.f, s2 = 0.f;
  for (int j = lane; j < d; j += 32) {
    const float xh = (xr[j] - mean) * rstd, dxh = dr[j] * g[j];
    s1 += dxh;
    s2 = fmaf(dxh, xh, s2);
  }
  const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
  for (int j = lane; j < ld; j += 32) {
    float o = 0.f, pr = 0.f;
    if (j < d) {
      const float xh = (xr[j] - mean) * rstd, dxh = dr[j] * g[j];
      o = rstd * (dxh - m1 - xh * m2);
      pr = dr[j] * xh;
    }
    const float h = tf32_hi(o);
    dx_hi[(size_t)r * ld + j] = h;
    dx_lo[(size_t)r * ld + j] = o - h;
    prod[(size_t)r * ld + j] = pr;
  }
}

// attention backward per (AST, head) (nn.py:99-120), P recomputed
__global__ void attention_back_kernel(const float* __restrict__ qkv, int ldq,
                                      const float* __restrict__ dctx, int ldc,
                                      const int32_t* __restrict__ tok_off, int d, int nh, int dh,
                                      float scale, float* __restrict__ g_hi,
                                      float* __restrict__ g_lo, int lcap) {
  extern __shared__ float sm[];  // q, k, v, dctx: lcap rows each
  const int s = blockIdx.x, h = blockIdx.y;
  const int t0 = tok_off[s], L = tok_off[s + 1] - t0;
  const int dhp = dh + 1;
  float* q = sm;
  float* k = q + lcap * dhp;
  float* v = k + lcap * dhp;
  float* dc = v + lcap * dhp;
  float* p = dc + lcap * dhp;  // [16][17]
  float* dp = p + 16 * 17;              // [16][17]
  for (int e = threadIdx.x; e < L * dh; e += blockDim.x) {
    const int l = e / dh, j = e - l * dh;
    const float* row = qkv + (size_t)(t0 + l) * ldq + h * dh + j;
    q[l * dhp + j] = row[0];
    k[l * dhp + j] = row[d];
    v[l * dhp + j] = row[2 * d];
    dc[l * dhp + j] = dctx[(size_t)(t0 + l) * ldc + h * dh + j];
  }
  __syncthreads();
  {
    const int g = score_group(L), sl = threadIdx.x & (g - 1), ng = blockDim.x / g;
    for (int e0 = 0; e0 < L * L; e0 += ng) {  // uniform trip count: full-warp shuffles
      const int e = e0 + threadIdx.x / g, i = e / L, j = e - i * L;
      float acc = 0.f, acc2 = 0.f;
      if (e < L * L)
        for (int c = sl; c < dh; c += g) {
          acc = fmaf(q[i * dhp + c], k[j * dhp + c], acc);
          acc2 = fmaf(dc[i * dhp + c], v[j * dhp + c], acc2);
        }
      acc = group_sum(acc, g);
      acc2 = group_sum(acc2, g);
      if (e < L * L && sl == 0) {
        p[i * 17 + j] = acc * scale;
        dp[i * 17 + j] = acc2;
      }
    }
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
    float rd = 0.f;
    for (int j = 0; j < L; ++j) {
      p[i * 17 + j] /= sum;
      rd = fmaf(p[i * 17 + j], dp[i * 17 + j], rd);
    }
    for (int j = 0; j < L; ++j) dp[i * 17 + j] = p[i * 17 + j] * (dp[i * 17 + j] - rd) * scale;
  }
  __syncthreads();
  auto put = [&](int row, int col, float val) {
    const size_t o = (size_t)row * ldq + col;
    const float hi = tf32_hi(val);
    g_hi[o] = hi;
    g_lo[o] = val - hi;
  };
  for (int e = threadIdx.x; e < L * dh; e += blockDim.x) {
    const int i = e / dh, c = e - i * dh;
    float gq = 0.f, gk = 0.f, gv = 0.f;
    for (int j = 0; j < L; ++j) {
      gq = fmaf(dp[i * 17 + j], k[j * dhp + c], gq);  // dQ_i = Σ_j dS_ij k_j
      gk = fmaf(dp[j * 17 + i], q[j * dhp + c], gk);  // dK_i = Σ_j dS_ji q_j
      gv = fmaf(p[j * 17 + i], dc[j * dhp + c], gv);  // dV_i = Σ_j P_ji dc_j
    }
    put(t0 + i, h * dh + c, gq);
    put(t0 + i, d + h * dh + c, gk);
    put(t0 + i, 2 * d + h * dh + c, gv);
  }
  if (h == nh - 1) {
    const int padw = ldq - 3 * d;
    for (int e = threadIdx.x; e < L * padw; e += blockDim.x) {
      const int i = e / padw, j = e - i * padw;
      put(t0 + i, 3 * d + j, 0.f);
    }
  }
}

// loss + dL/dpred (costmodel.py:343-423, transformed space; oracle
// predictor.loss_and_grad), one block, fixed-order reduction; pred / dpred in
// the batch's sorted order, y gathered through idx
// supervised loss + d(loss)/d(pred) (costmodel.py:376-423): squared term in
// model space, relative term in model space shifted by `offset` or, with
// `original`, between decoded prediction and decoded label (clamped decode,
// _decode_with_grad)
__global__ void loss_kernel(const float* __restrict__ pred, const double* __restrict__ y,
                            const int32_t* __restrict__ idx, int n, int mode, double lam,
                            double offset, int original, tpcb_boxcox norm, double n_norm,
                            float* __restrict__ dpred, double* __restrict__ loss_out) {
  __shared__ double red[32];
  double acc_sq = 0.0, acc_rel = 0.0;
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    const double yy = y[idx[s]], d = (double)pred[s] - yy;
    double rel = 0.0, relg = 0.0;
    if (mode != 1) {
      if (original) {
        const double y0 = boxcox_decode_plain(yy, norm);
        double p0, dp0;
        boxcox_decode_with_grad((double)pred[s], norm, &p0, &dp0);
        rel = fabs(p0 - y0) / y0;
        relg = sign_d(p0 - y0) * dp0 / (y0 * n_norm);
      } else {
        const double den = yy + offset;
        rel = fabs(d) / den;
        relg = sign_d(d) / (den * n_norm);
      }
    }
    double g;
    if (mode == 1) g = 2.0 * d / n_norm;           // mse
    else if (mode == 2) g = relg;                  // mape
    else g = 2.0 * d / n_norm + lam * relg;        // hybrid
    dpred[s] = (float)g;
    acc_sq += d * d;
    acc_rel += rel;
  }
  double v = mode == 1 ? acc_sq : mode == 2 ? acc_rel : acc_sq + lam * acc_rel;
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    w = warp_sum_d(w);
    if (threadIdx.x == 0) loss_out[0] = w / n;  // batch mean (the step's loss)
  }
}

// dec.out backward: dD = dpred ⊗ outW ⊙ [D > 0] (pair), prod = D·dpred (→ doutW)
__global__ void out_back_kernel(Model M, const float* __restrict__ P, const float* __restrict__ d_hi,
                                const float* __restrict__ d_lo, int ld, int width,
                                const float* __restrict__ dpred, int n, float* __restrict__ g_hi,
                                float* __restrict__ g_lo, float* __restrict__ prod) {
  const int s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (s >= n) return;
  const int lane = threadIdx.x & 31;
  const float dp = dpred[s];
  for (int j = lane; j < ld; j += 32) {
    const size_t o = (size_t)s * ld + j;
    float g = 0.f, pr = 0.f;
    if (j < width) {
      const float h = d_hi[o];
      pr = (h + d_lo[o]) * dp;
      g = h > 0.f ? dp * P[M.outW + j] : 0.f;
    }
    const float hi = tf32_hi(g);
    g_hi[o] = hi;
    g_lo[o] = g - hi;
    prod[o] = pr;
  }
}

// gate + device MLP backward per sorted AST: dzx = dz⊙zp (pair), per-sample
// parameter-gradient rows (column-summed afterwards, fixed order)
__global__ void gate_back_kernel(Model M, const float* __restrict__ P,
                                 const float* __restrict__ devfeat,
                                 const int32_t* __restrict__ idx, const float* __restrict__ dz,
                                 const float* __restrict__ zx, int ldz, float* __restrict__ gx_hi,
                                 float* __restrict__ gx_lo, float* __restrict__ tWp,
                                 float* __restrict__ tbp, float* __restrict__ tWh,
                                 float* __restrict__ tbh) {
  extern __shared__ float sv[];  // zv [ddev] | dzp [de] | dzv [ddev]
  float* zv = sv;
  float* dzp = zv + M.d_dev;
  float* dzv = dzp + M.d_e;
  const int s = blockIdx.x;
  const float* dv = devfeat + (size_t)idx[s] * TPCB_DEV_FEAT;
  for (int j = threadIdx.x; j < M.d_dev; j += blockDim.x) {
    float a = P[M.devhb + j];
    for (int k = 0; k < TPCB_DEV_FEAT; ++k) a = fmaf(dv[k], P[M.devhW + k * M.d_dev + j], a);
    zv[j] = fmaxf(a, 0.f);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ldz; e += blockDim.x) {
    float gx = 0.f;
    if (e < M.d_e) {
      float zp = P[M.devpb + e];
      for (int j = 0; j < M.d_dev; ++j) zp = fmaf(zv[j], P[M.devpW + j * M.d_e + e], zp);
      const float g = dz[(size_t)s * ldz + e];
      gx = g * zp;
      const float gp = g * zx[(size_t)s * ldz + e];
      dzp[e] = gp;
      tbp[(size_t)s * M.d_e + e] = gp;
    }
    const float hi = tf32_hi(gx);
    gx_hi[(size_t)s * ldz + e] = hi;
    gx_lo[(size_t)s * ldz + e] = gx - hi;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < M.d_dev; j += blockDim.x) {
    float a = 0.f;
    for (int e = 0; e < M.d_e; ++e) a = fmaf(dzp[e], P[M.devpW + j * M.d_e + e], a);
    a = zv[j] > 0.f ? a : 0.f;
    dzv[j] = a;
    tbh[(size_t)s * M.d_dev + j] = a;
  }
  __syncthreads();
  const int nwp = M.d_dev * M.d_e;
  for (int e = threadIdx.x; e < nwp; e += blockDim.x)
    tWp[(size_t)s * nwp + e] = zv[e / M.d_e] * dzp[e % M.d_e];
  const int nwh = TPCB_DEV_FEAT * M.d_dev;
  for (int e = threadIdx.x; e < nwh; e += blockDim.x)
    tWh[(size_t)s * nwh + e] = dv[e / M.d_dev] * dzv[e % M.d_dev];
}

struct Bwd {
  int64_t Tp, Ap;
  float* dh;                 // [T, dp] fp32
  float *ds_hi, *ds_lo;      // [T, dp]
  float *df_hi, *df_lo;      // [T, ffp]
  float* dctx;               // [T, dp]
  float *dq_hi, *dq_lo;      // [T, qkvp]
  float* prod;               // [T, max(dp, dmax)]
  // transposed weight-gradient operands, a ring of kXtRing sets: the main
  // stream fills set k while the side stream's GEMMs still read the others
  float *xt_hi[3], *xt_lo[3], *yt_hi[3], *yt_lo[3];
  float* part;
  float *dd_hi[2], *dd_lo[2];  // decoder grads [A, dmax]
  float* dz;                 // [A, dep]
  float *dzx_hi, *dzx_lo;    // [A, dep]
  float *tWp, *tbp, *tWh, *tbh;
  float* dpred;
  float* colpart;            // column-sum partials [chunks][cols]
  unsigned* colcnt;          // column-sum stripe counters [kColCntMax]
  size_t part_floats;
};

Bwd carve_bwd(const LargePlan& p, const Model& M, int64_t n_tok, int64_t n_ast, Carver* cv) {
  Bwd b{};
  const int64_t T = ((n_tok + kTileM - 1) / kTileM) * kTileM;
  const int64_t A = ((n_ast + kTileM - 1) / kTileM) * kTileM;
  b.Tp = T;
  b.Ap = A;
  const int dmax = dec_max(M);
  b.dh = cv->take(T * p.dp);
  b.ds_hi = cv->take(T * p.dp);
  b.ds_lo = cv->take(T * p.dp);
  b.df_hi = cv->take(T * p.ffp);
  b.df_lo = cv->take(T * p.ffp);
  b.dctx = cv->take(T * p.dp);
  b.dq_hi = cv->take(T * p.qkvp);
  b.dq_lo = cv->take(T * p.qkvp);
  b.prod = cv->take(max(T * p.dp, A * (int64_t)dmax));
  const int64_t wmax = max(max(p.qkvp, p.ffp), max(p.dp, dmax));
  const int64_t xt = max(wmax * (T + 32), (int64_t)p.dp * (T + 32 * TPCB_MAX_LEAF + 32));
  for (int k = 0; k < 3; ++k) {
    b.xt_hi[k] = cv->take(xt);
    b.xt_lo[k] = cv->take(xt);
    b.yt_hi[k] = cv->take(xt);
    b.yt_lo[k] = cv->take(xt);
  }
  const int64_t pm = max(max((int64_t)M.d * p.qkvp, (int64_t)M.d_ff * p.dp),
                         max((int64_t)M.d * p.ffp, (int64_t)TPCB_MAX_LEAF * p.dp * p.dep));
  b.part_floats = 8 * (max(pm, (int64_t)dmax * dmax) + max(wmax, (int64_t)p.dep));  // + bias row
  b.part = cv->take(b.part_floats);
  for (int k = 0; k < 2; ++k) {
    b.dd_hi[k] = cv->take(A * dmax);
    b.dd_lo[k] = cv->take(A * dmax);
  }
  b.dz = cv->take(A * p.dep);
  b.dzx_hi = cv->take(A * p.dep);
  b.dzx_lo = cv->take(A * p.dep);
  b.tWp = cv->take(A * M.d_dev * M.d_e);
  b.tbp = cv->take(A * M.d_e);
  b.tWh = cv->take(A * TPCB_DEV_FEAT * M.d_dev);
  b.tbh = cv->take(A * M.d_dev);
  b.dpred = cv->take(A);
  b.colpart = cv->take(2 * (size_t)ceil_div(max(T, A), kColChunk) *  // 2: colsum2's jobs
                       max(max(M.d_dev * M.d_e, p.qkvp), max(p.ffp, dmax)));
  b.colcnt = reinterpret_cast<unsigned*>(cv->take(kColCntMax));
  return b;
}

int transpose_pair(const TJob& a, const TJob& b, cudaStream_t st) {
  const int ca = a.ones_col >= 0 ? a.ones_col + 1 : a.cols, cb = b.ones_col >= 0 ? b.ones_col + 1 : b.cols;
  const dim3 grid((unsigned)ceil_div(max(ca, cb), 64), (unsigned)ceil_div(max(a.ldo, b.ldo), 64), 2);
  transpose_pair_kernel<<<grid, dim3(32, 8), 0, st>>>(a, b);
  TPCB_LAUNCH_CHECK("large_transpose");
  return TPCB_OK;
}

thread_local float* g_colsum_part = nullptr;  // column-sum scratch (set per call)
thread_local unsigned* g_colsum_cnt = nullptr;  // per-stripe counters (zeroed per call)

// the weight-gradient branch runs on a side stream: dW = Xᵀ·dY only needs
// dY, so it overlaps the main stream's dX chain; the main stream waits only
// for the transposes (after which dY may be overwritten)
constexpr int kXtRing = 3;
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[4] = {};
  int k = 0;
  cudaEvent_t xt_ev[kXtRing] = {};  // the side GEMM that last read transposed set k
  bool xt_used[kXtRing] = {};
  int xt_slot = 0;
  cudaEvent_t next() { return ev[k++ & 3]; }
};
thread_local SideStream g_side;

int side_init() {
  if (g_side.s) return TPCB_OK;
  TPCB_CUDA_CHECK(cudaStreamCreateWithFlags(&g_side.s, cudaStreamNonBlocking));
  for (auto& e : g_side.ev) TPCB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : g_side.xt_ev) TPCB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return TPCB_OK;
}

int stream_wait(cudaStream_t waiter, cudaStream_t on) {
  cudaEvent_t e = g_side.next();
  TPCB_CUDA_CHECK(cudaEventRecord(e, on));
  TPCB_CUDA_CHECK(cudaStreamWaitEvent(waiter, e, 0));
  return TPCB_OK;
}

// γ / β of a LayerNorm backward: the column sums of prod and dy in one launch
int colsum2(const float* x, ColDst dst, const float* x2, ColDst dst2, int rows, int cols, int ld,
            float* grad, cudaStream_t st) {
  const int chunks = max(1, ceil_div(rows, kColChunk));
  if (!g_colsum_cnt || ceil_div(cols, 32) > kColCntMax / 2) return TPCB_ERR_VALIDATION;
  colsum_fused_kernel<<<dim3(ceil_div(cols, 32), chunks, 2), dim3(32, 8), 0, st>>>(
      x, nullptr, rows, cols, ld, g_colsum_part, g_colsum_cnt, dst, grad, x2, dst2);
  TPCB_LAUNCH_CHECK("large_colsum2");
  return TPCB_OK;
}

int colsum(const float* x, const float* x_lo, int rows, int cols, int ld, ColDst dst, float* grad,
           cudaStream_t st) {
  const int chunks = max(1, ceil_div(rows, kColChunk));
  if (g_colsum_cnt && ceil_div(cols, 32) <= kColCntMax) {
    colsum_fused_kernel<<<dim3(ceil_div(cols, 32), chunks), dim3(32, 8), 0, st>>>(
        x, x_lo, rows, cols, ld, g_colsum_part, g_colsum_cnt, dst, grad);
  } else {
    colsum_partial_kernel<<<dim3(ceil_div(cols, 32), chunks), dim3(32, 8), 0, st>>>(
        x, x_lo, rows, cols, ld, g_colsum_part);
    colsum_final_kernel<<<ceil_div(cols, 128), 128, 0, st>>>(g_colsum_part, chunks, cols, dst,
                                                              grad);
  }
  TPCB_LAUNCH_CHECK("large_colsum");
  return TPCB_OK;
}

ColDst one(int64_t off, int colw, int acc = 0) { return ColDst{colw, {off, off, off}, acc}; }

// dW[M_in, N_out] = Xᵀ·dY over K = kp rows: X given as [rows, M_in] (ld_x),
// dY as [rows, N_out] (ld_y) — both transposed + split on the main stream
// into the next set of the transposed-operand ring, the GEMM + reduction
// forked to the side stream.  The main stream never waits for the side
// stream's GEMMs except before refilling a ring set the side stream may
// still be reading (kXtRing wgrads later) and at the final join.
int wgrad(const Ctx& c, Bwd& b, const float* x_hi, const float* x_lo, int ld_x, int m_in,
          const float* y_hi, const float* y_lo, int ld_y, int n_out, int rows, int seg, int segp,
          ColDst dst, float* grad, const ColDst* bias = nullptr) {
  const cudaStream_t st = g_side.s;
  const int kp = pad32(rows);
  int rc;
  const int k = g_side.xt_slot;
  g_side.xt_slot = (k + 1) % kXtRing;
  if (g_side.xt_used[k]) TPCB_CUDA_CHECK(cudaStreamWaitEvent(c.st, g_side.xt_ev[k], 0));
  // bias: X gets a ones row (product row m_in = the column sums of dY)
  const int hb = bias ? 1 : 0, m_all = m_in + hb;
  if ((rc = transpose_pair(TJob{x_hi, x_lo, rows, m_in, ld_x, b.xt_hi[k], b.xt_lo[k], kp,
                                bias ? m_in : -1},
                           TJob{y_hi, y_lo, rows, n_out, ld_y, b.yt_hi[k], b.yt_lo[k], kp, -1},
                           c.st)))
    return rc;
  if ((rc = stream_wait(st, c.st))) return rc;  // fork: the transposed operands are ready
  const int ldc = pad32(n_out);
  const int tiles = ceil_div(m_all, kTileM) * ceil_div(ldc, 128);
  const int k_total = kp / 32;
  // one wave: gemm3 runs one CTA per SM (197 KB of operand ring)
  int splits = max(1, min(min(kNumSMs / max(tiles, 1), k_total / 4), 8));
  if ((size_t)splits * m_all * ldc > b.part_floats) return TPCB_ERR_VALIDATION;
  Epi e{m_all, n_out, ldc, nullptr, 0, nullptr, nullptr, 0, b.part, nullptr, nullptr};
  e.split_stride = (int64_t)m_all * ldc;
  Operand A{b.xt_hi[k], b.xt_lo[k], m_all, kp, kp}, B{b.yt_hi[k], b.yt_lo[k], n_out, kp, kp};
  if ((rc = launch_gemm_nt<128>(A, B, e, st, splits, &splits))) return rc;
  TPCB_CUDA_CHECK(cudaEventRecord(g_side.xt_ev[k], st));
  g_side.xt_used[k] = true;
  const int64_t total = (int64_t)m_all * n_out;
  reduce_grad_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, kNumSMs * 8), 256, 0, st>>>(
      b.part, splits, e.split_stride, m_in, n_out, ldc, seg, segp, dst, grad, hb,
      bias ? *bias : ColDst{1, {0, 0, 0}, 0});
  TPCB_LAUNCH_CHECK("large_reduce_grad");
  return TPCB_OK;
}

// backward from dz (bucket-order rows of b.dz, ld p.dep) down to the
// input projection: gate + device MLP, leaf_embed per leaf-count bucket,
// the encoder (top layer first).  acc = 1 adds into G (the target pass of a
// CMD step, costmodel.py:561-564), acc = 0 writes.
int large_tail(const Ctx& c, const Fwd& f, Bwd& b, const int32_t* h_tok_off, int64_t n_batch,
               const float* d_devfeat, float* G, int acc) {
  const Model& M = c.M;
  const LargePlan& p = c.p;
  const cudaStream_t st = c.st;
  const float* P = c.P;
  const int64_t n_tok = h_tok_off[n_batch];
  const int nt = (int)n_tok, nb = (int)n_batch;
  int rc;
  gate_back_kernel<<<nb, 128, (2 * M.d_dev + M.d_e) * 4, st>>>(
      M, P, d_devfeat, f.idx, b.dz, f.zx, p.dep, b.dzx_hi, b.dzx_lo, b.tWp, b.tbp, b.tWh, b.tbh);
  TPCB_LAUNCH_CHECK("large_gate_back");
  if ((rc = colsum(b.tWp, nullptr, nb, M.d_dev * M.d_e, M.d_dev * M.d_e,
                   one(M.devpW, M.d_dev * M.d_e, acc), G, st)))
    return rc;
  if ((rc = colsum(b.tbp, nullptr, nb, M.d_e, M.d_e, one(M.devpb, M.d_e, acc), G, st))) return rc;
  if ((rc = colsum(b.tWh, nullptr, nb, TPCB_DEV_FEAT * M.d_dev, TPCB_DEV_FEAT * M.d_dev,
                   one(M.devhW, TPCB_DEV_FEAT * M.d_dev, acc), G, st)))
    return rc;
  if ((rc = colsum(b.tbh, nullptr, nb, M.d_dev, M.d_dev, one(M.devhb, M.d_dev, acc), G, st))) return rc;
  const Pair hf = f.H(M.n_layers);
  for (int64_t s0 = 0; s0 < n_batch;) {
    const int Lb = h_tok_off[s0 + 1] - h_tok_off[s0];
    int64_t s1 = s0 + 1;
    while (s1 < n_batch && h_tok_off[s1 + 1] - h_tok_off[s1] == Lb) ++s1;
    const int nbk = (int)(s1 - s0);
    const int64_t t0 = h_tok_off[s0];
    const int w = Lb * p.dp;
    Operand A = act_op(b.dzx_hi + s0 * p.dep, b.dzx_lo + s0 * p.dep, nbk, p.dep);
    Operand B{c.im.hi + p.leaf_b[Lb], c.im.lo + p.leaf_b[Lb], w, p.dep, p.dep};
    Epi e{nbk, w, w, nullptr, 0, nullptr, nullptr, 0, b.dh + t0 * p.dp, nullptr, nullptr};
    if ((rc = launch_gemm(A, B, e, st))) return rc;
    const ColDst lb = one(M.leafb[Lb], M.d_e, acc);  // bias: the GEMM's ones row
    if ((rc = wgrad(c, b, hf.hi + t0 * p.dp, hf.lo + t0 * p.dp, w, w, b.dzx_hi + s0 * p.dep,
                    b.dzx_lo + s0 * p.dep, p.dep, M.d_e, nbk, M.d, p.dp, one(M.leafW[Lb], M.d_e, acc),
                    G, &lb)))
      return rc;
    s0 = s1;
  }
  // ---- encoder, top layer first ----
  const float scale = 1.0f / sqrtf((float)M.dh);
  const size_t att_smem = (size_t)(4 * TPCB_MAX_LEAF * (M.dh + 1) + 2 * 16 * 17) * 4;
  if (att_smem > 48 * 1024)
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(attention_back_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)att_smem));
  const int lcap = max_leaf_count(h_tok_off, n_batch);
  const size_t att_used = (size_t)(4 * lcap * (M.dh + 1) + 2 * 16 * 17) * 4;
  for (int li = M.n_layers - 1; li >= 0; --li) {
    const LayerOff& L = M.layer[li];
    const Pair h = f.H(li), h1 = f.H1(li), ff = f.F(li), ctx = f.C(li);
    // LN2
    if (p.dp <= 768)
      ln_back_reg_kernel<24><<<ceil_div(nt, 8), 256, 0, st>>>(b.dh, f.S2(li), p.dp, nt, M.d,
                                                              P + L.ln2g, b.ds_hi, b.ds_lo, b.prod);
    else
      ln_back_kernel<<<ceil_div(nt, 8), 256, 0, st>>>(b.dh, f.S2(li), p.dp, nt, M.d, P + L.ln2g,
                                                      b.ds_hi, b.ds_lo, b.prod);
    TPCB_LAUNCH_CHECK("large_ln_back");
    if ((rc = colsum2(b.prod, one(L.ln2g, M.d, acc), b.dh, one(L.ln2b, M.d, acc), nt, M.d, p.dp, G,
                      st)))
      return rc;
    // FFN out
    const ColDst fob = one(L.fob, M.d, acc), fhb = one(L.fhb, M.d_ff, acc), bo = one(L.bo, M.d, acc);
    if ((rc = wgrad(c, b, ff.hi, ff.lo, p.ffp, M.d_ff, b.ds_hi, b.ds_lo, p.dp, M.d, nt, 0, 0,
                    one(L.foW, M.d, acc), G, &fob)))
      return rc;
    {
      Epi e{nt, M.d_ff, p.ffp, nullptr, 0, nullptr, nullptr, 0, nullptr, b.df_hi, b.df_lo};
      e.mask = ff.hi;
      e.ldm = p.ffp;
      Operand B{c.im.hi + p.layer_b[li][3], c.im.lo + p.layer_b[li][3], M.d_ff, p.dp, p.dp};
      if ((rc = launch_gemm(act_op(b.ds_hi, b.ds_lo, nt, p.dp), B, e, st))) return rc;
    }
    // FFN hidden
    if ((rc = wgrad(c, b, h1.hi, h1.lo, p.dp, M.d, b.df_hi, b.df_lo, p.ffp, M.d_ff, nt, 0, 0,
                    one(L.fhW, M.d_ff, acc), G, &fhb)))
      return rc;
    {
      Epi e{nt, M.d, p.dp, nullptr, 0, b.ds_hi, b.ds_lo, p.dp, b.dh, nullptr, nullptr};
      Operand B{c.im.hi + p.layer_b[li][2], c.im.lo + p.layer_b[li][2], M.d, p.ffp, p.ffp};
      if ((rc = launch_gemm(act_op(b.df_hi, b.df_lo, nt, p.ffp), B, e, st))) return rc;
    }
    // LN1
    if (p.dp <= 768)
      ln_back_reg_kernel<24><<<ceil_div(nt, 8), 256, 0, st>>>(b.dh, f.S1(li), p.dp, nt, M.d,
                                                              P + L.ln1g, b.ds_hi, b.ds_lo, b.prod);
    else
      ln_back_kernel<<<ceil_div(nt, 8), 256, 0, st>>>(b.dh, f.S1(li), p.dp, nt, M.d, P + L.ln1g,
                                                      b.ds_hi, b.ds_lo, b.prod);
    TPCB_LAUNCH_CHECK("large_ln_back");
    if ((rc = colsum2(b.prod, one(L.ln1g, M.d, acc), b.dh, one(L.ln1b, M.d, acc), nt, M.d, p.dp, G,
                      st)))
      return rc;
    // attention output projection
    if ((rc = wgrad(c, b, ctx.hi, ctx.lo, p.dp, M.d, b.ds_hi, b.ds_lo, p.dp, M.d, nt, 0, 0,
                    one(L.Wo, M.d, acc), G, &bo)))
      return rc;
    {
      Epi e{nt, M.d, p.dp, nullptr, 0, nullptr, nullptr, 0, b.dctx, nullptr, nullptr};
      Operand B{c.im.hi + p.layer_b[li][1], c.im.lo + p.layer_b[li][1], M.d, p.dp, p.dp};
      if ((rc = launch_gemm(act_op(b.ds_hi, b.ds_lo, nt, p.dp), B, e, st))) return rc;
    }
    attention_back_kernel<<<dim3((unsigned)n_batch, M.n_heads), 128, att_used, st>>>(
        f.QKV(li), p.qkvp, b.dctx, p.dp, f.tok_off, M.d, M.n_heads, M.dh, scale, b.dq_hi,
        b.dq_lo, lcap);
    TPCB_LAUNCH_CHECK("large_attention_back");
    // Q | K | V projections
    const ColDst qkv_dst{M.d, {(int64_t)L.Wq, (int64_t)L.Wk, (int64_t)L.Wv}, acc};
    const ColDst qkvb_dst{M.d, {(int64_t)L.bq, (int64_t)L.bk, (int64_t)L.bv}, acc};
    if ((rc = wgrad(c, b, h.hi, h.lo, p.dp, M.d, b.dq_hi, b.dq_lo, p.qkvp, p.qkv, nt, 0, 0,
                    qkv_dst, G, &qkvb_dst)))
      return rc;
    {
      Epi e{nt, M.d, p.dp, nullptr, 0, b.ds_hi, b.ds_lo, p.dp, b.dh, nullptr, nullptr};
      Operand B{c.im.hi + p.layer_b[li][0], c.im.lo + p.layer_b[li][0], M.d, p.qkvp, p.qkvp};
      if ((rc = launch_gemm(act_op(b.dq_hi, b.dq_lo, nt, p.qkvp), B, e, st))) return rc;
    }
  }
  // input projection
  const ColDst inb = one(M.inb, M.d, acc);
  if ((rc = wgrad(c, b, f.x_hi, f.x_lo, 32, TPCB_FEAT, b.dh, nullptr, p.dp, M.d, nt, 0, 0,
                  one(M.inW, M.d, acc), G, &inb)))
    return rc;
  return TPCB_OK;
}

}  // namespace
}  // namespace tpcb

namespace {
struct CmdWs {
  float* zall;     // [(ns + nt), de] input order
  double* grad;    // [(ns + nt), de]
  double* value;   // [1]
  int32_t* pos;    // [ns] source then [nt] target input positions
};

// workspace layout: source activations, backward scratch (sized for the
// larger of the two batches), then with a target batch its activations and
// the CMD buffers
void carve_train(const LargePlan& p, const Model& M, int64_t n_ast, int64_t n_tok, int64_t n_ast_t,
                 int64_t n_tok_t, Carver* cv, Fwd* f, Bwd* b, Fwd* ft, CmdWs* cw) {
  *f = carve_fwd(p, M, n_tok, n_ast, true, cv);
  *b = carve_bwd(p, M, std::max(n_tok, n_tok_t), std::max(n_ast, n_ast_t), cv);
  if (n_ast_t > 0) {
    *ft = carve_fwd(p, M, n_tok_t, n_ast_t, true, cv);
    const int64_t rows = n_ast + n_ast_t;
    cw->zall = cv->take(rows * M.d_e);
    cw->grad = reinterpret_cast<double*>(cv->take(2 * rows * M.d_e));
    cw->value = reinterpret_cast<double*>(cv->take(2));
    cw->pos = reinterpret_cast<int32_t*>(cv->take(rows));
  }
}
}  // namespace

extern "C" int tpcb_large_train_ws(const tpcb_model* m, int64_t n_ast, int64_t n_tok,
                                   int64_t n_ast_t, int64_t n_tok_t, size_t* ws_bytes) {
  if (!m || !ws_bytes || n_ast_t < 0 || n_tok_t < 0) return TPCB_ERR_VALIDATION;
  if (!large_supported(m->dev)) return TPCB_ERR_UNSUPPORTED;
  const LargePlan p = make_plan(m->dev);
  Carver cv{nullptr};
  Fwd f, ft;
  Bwd b;
  CmdWs cw{};
  carve_train(p, m->dev, n_ast, n_tok, n_ast_t, n_tok_t, &cv, &f, &b, &ft, &cw);
  *ws_bytes = cv.o;
  return TPCB_OK;
}

// one training batch through the large path: forward (activations kept),
// loss, backward → the full flat gradient d_grad (rewritten) and the batch
// loss d_loss[0] (device).  Dataset-resident inputs: packed rows d_x (K1
// layout) with d_ast_row, device features, model-space targets d_y; the
// batch is h_idx (dataset indices in bucket order) with token offsets
// h_tok_off; gradients are normalised by n_norm (the global batch size).
extern "C" int tpcb_large_loss_backward(const tpcb_model* m, const float* d_params,
                                        const void* d_image, const float* d_x,
                                        const int32_t* d_ast_row, const float* d_devfeat,
                                        const double* d_y, const int32_t* h_idx,
                                        const int32_t* h_tok_off, const int32_t* d_idx,
                                        const int32_t* d_tok_off, int64_t n_batch,
                                        const tpcb_loss* loss, double n_norm,
                                        const int32_t* h_src_pos, const tpcb_large_batch* tgt,
                                        void* d_ws, size_t ws_bytes, float* d_grad,
                                        double* d_loss, double* d_cmd, int32_t* d_status,
                                        void* stream_) {
  if (!m || !d_params || !d_image || !d_x || !d_ast_row || !d_devfeat || !d_y || !h_idx ||
      !h_tok_off || !loss || !d_ws || !d_grad || !d_loss)
    return TPCB_ERR_VALIDATION;
  if (n_batch <= 0) return TPCB_ERR_EMPTY_BATCH;
  const Model& M = m->dev;
  if (!large_supported(M)) return TPCB_ERR_UNSUPPORTED;
  if (M.n_dec < 1) return TPCB_ERR_UNSUPPORTED;
  if (loss->mode < 0 || loss->mode > 2 || loss->cmd_order < 1) return TPCB_ERR_VALIDATION;
  const bool use_cmd = loss->alpha_cmd > 0.0 && tgt != nullptr;
  if (use_cmd) {
    if (tgt->n < 1) return TPCB_ERR_EMPTY_SET;
    if (!tgt->x || !tgt->ast_row || !tgt->devfeat || !tgt->h_idx || !tgt->h_tok_off ||
        !tgt->h_pos || !h_src_pos)
      return TPCB_ERR_VALIDATION;
  }
  cudaStream_t st = (cudaStream_t)stream_;
  const LargePlan p = make_plan(M);
  const int64_t n_tok = h_tok_off[n_batch];
  const int64_t n_t = use_cmd ? tgt->n : 0;
  const int64_t n_tok_t = use_cmd ? tgt->h_tok_off[tgt->n] : 0;
  Carver cv{(uint8_t*)d_ws};
  Fwd f, ft{};
  Bwd b;
  CmdWs cw{};
  carve_train(p, M, n_batch, n_tok, n_t, n_tok_t, &cv, &f, &b, &ft, &cw);
  if (cv.o > ws_bytes) return TPCB_ERR_VALIDATION;
  if (d_idx && d_tok_off) {  // device copies of the plan (uploaded once per epoch)
    f.idx = const_cast<int32_t*>(d_idx);
    f.tok_off = const_cast<int32_t*>(d_tok_off);
  } else {
    TPCB_CUDA_CHECK(cudaMemcpyAsync(f.idx, h_idx, n_batch * 4, cudaMemcpyHostToDevice, st));
    TPCB_CUDA_CHECK(
        cudaMemcpyAsync(f.tok_off, h_tok_off, (n_batch + 1) * 4, cudaMemcpyHostToDevice, st));
  }
  gather_tokens_kernel<<<ceil_div(n_batch, 8), 256, 0, st>>>(d_x, f.idx, d_ast_row, f.tok_off,
                                                             (int)n_batch, f.x_hi, f.x_lo);
  TPCB_LAUNCH_CHECK("large_gather");
  const Ctx c{M, p, d_params, carve_image(p, (uint8_t*)const_cast<void*>(d_image)), st};
  tpcb_boxcox bc{};
  int rc = run_forward(c, f, n_batch, h_tok_off, d_devfeat, true, bc, nullptr, nullptr, nullptr,
                       nullptr, nullptr, d_status);
  if (rc) return rc;
  if (use_cmd) {  // target forward (activations kept) and the CMD statistics
    TPCB_CUDA_CHECK(cudaMemcpyAsync(ft.idx, tgt->h_idx, n_t * 4, cudaMemcpyHostToDevice, st));
    TPCB_CUDA_CHECK(cudaMemcpyAsync(ft.tok_off, tgt->h_tok_off, (n_t + 1) * 4,
                                    cudaMemcpyHostToDevice, st));
    TPCB_CUDA_CHECK(cudaMemcpyAsync(cw.pos, h_src_pos, n_batch * 4, cudaMemcpyHostToDevice, st));
    TPCB_CUDA_CHECK(cudaMemcpyAsync(cw.pos + n_batch, tgt->h_pos, n_t * 4,
                                    cudaMemcpyHostToDevice, st));
    gather_tokens_kernel<<<ceil_div(n_t, 8), 256, 0, st>>>(tgt->x, ft.idx, tgt->ast_row,
                                                           ft.tok_off, (int)n_t, ft.x_hi, ft.x_lo);
    TPCB_LAUNCH_CHECK("large_gather_t");
    if ((rc = run_forward(c, ft, n_t, tgt->h_tok_off, tgt->devfeat, true, bc, nullptr, nullptr,
                          nullptr, nullptr, nullptr, d_status)))
      return rc;
    z_scatter_kernel<<<ceil_div(n_batch * M.d_e, 256), 256, 0, st>>>(
        f.z_hi, f.z_lo, p.dep, cw.pos, (int)n_batch, M.d_e, 0, cw.zall);
    z_scatter_kernel<<<ceil_div(n_t * M.d_e, 256), 256, 0, st>>>(
        ft.z_hi, ft.z_lo, p.dep, cw.pos + n_batch, (int)n_t, M.d_e, n_batch, cw.zall);
    TPCB_LAUNCH_CHECK("large_z_scatter");
    if ((rc = tpcb_cmd(cw.zall, 0, n_batch, n_t, M.d_e, loss->cmd_order, cw.value, cw.grad, st)))
      return rc;
  }
  const float* P = d_params;
  float* G = d_grad;
  const int nt = (int)n_tok, nb = (int)n_batch;
  (void)nt;
  g_colsum_part = b.colpart;
  g_colsum_cnt = b.colcnt;
  struct CntGuard {  // the counters belong to this call's workspace
    ~CntGuard() { g_colsum_cnt = nullptr; }
  } cnt_guard;
  if ((rc = side_init())) return rc;
  TPCB_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(float) * (size_t)M.total, st));
  TPCB_CUDA_CHECK(cudaMemsetAsync(b.colcnt, 0, sizeof(unsigned) * kColCntMax, st));
  loss_kernel<<<1, 1024, 0, st>>>(f.pred, d_y, f.idx, nb, loss->mode, loss->lambda_hybrid,
                                  loss->offset, loss->original_space, loss->norm, n_norm, b.dpred,
                                  d_loss);
  TPCB_LAUNCH_CHECK("large_loss");
  if (use_cmd) {
    add_cmd_kernel<<<1, 1, 0, st>>>(d_loss, cw.value, loss->alpha_cmd, d_cmd);
    TPCB_LAUNCH_CHECK("large_add_cmd");
  }
  // ---- head: dec.out, decoder, gate + device MLP, leaf_embed ----
  const int nd = M.n_dec;
  const int wl = nd ? M.dec[nd - 1] : M.d_e, ldl = pad32(wl);
  out_back_kernel<<<ceil_div(nb, 8), 256, 0, st>>>(M, P, f.dec_hi[nd - 1], f.dec_lo[nd - 1], ldl,
                                                   wl, b.dpred, nb, b.dd_hi[0], b.dd_lo[0], b.prod);
  TPCB_LAUNCH_CHECK("large_out_back");
  if ((rc = colsum(b.prod, nullptr, nb, wl, ldl, one(M.outW, wl), G, st))) return rc;
  if ((rc = colsum(b.dpred, nullptr, nb, 1, 1, one(M.outb, 1), G, st))) return rc;
  int cur = 0;
  for (int i = nd - 1; i >= 0; --i) {
    const int wo = M.dec[i], ldo = pad32(wo);
    const int wi = i ? M.dec[i - 1] : M.d_e, ldi = pad32(wi);
    const float* in_hi = i ? f.dec_hi[i - 1] : f.z_hi;
    const float* in_lo = i ? f.dec_lo[i - 1] : f.z_lo;
    const ColDst db = one(M.decb[i], wo);
    if ((rc = wgrad(c, b, in_hi, in_lo, ldi, wi, b.dd_hi[cur], b.dd_lo[cur], ldo, wo, nb, 0, 0,
                    one(M.decW[i], wo), G, &db)))
      return rc;
    Operand A = act_op(b.dd_hi[cur], b.dd_lo[cur], nb, ldo);
    Operand B{c.im.hi + p.dec_b[i], c.im.lo + p.dec_b[i], wi, ldo, ldo};
    if (i) {
      Epi e{nb, wi, ldi, nullptr, 0, nullptr, nullptr, 0, nullptr, b.dd_hi[cur ^ 1],
            b.dd_lo[cur ^ 1]};
      e.mask = f.dec_hi[i - 1];
      e.ldm = ldi;
      if ((rc = launch_gemm(A, B, e, st))) return rc;
      cur ^= 1;
    } else {
      Epi e{nb, wi, ldi, nullptr, 0, nullptr, nullptr, 0, b.dz, nullptr, nullptr};
      if ((rc = launch_gemm(A, B, e, st))) return rc;
    }
  }
  if (use_cmd) {  // dz_s += alpha · dCMD/dzs (costmodel.py:557-560)
    dz_from_cmd_kernel<<<ceil_div(n_batch * p.dep, 256), 256, 0, st>>>(
        b.dz, p.dep, cw.grad, cw.pos, (int)n_batch, M.d_e, 0, loss->alpha_cmd, 0);
    TPCB_LAUNCH_CHECK("large_dz_cmd");
  }
  if ((rc = large_tail(c, f, b, h_tok_off, n_batch, d_devfeat, G, 0))) return rc;
  if (use_cmd) {  // target rows: zero prediction gradient, dz = alpha · dCMD/dzt
    dz_from_cmd_kernel<<<ceil_div(n_t * p.dep, 256), 256, 0, st>>>(
        b.dz, p.dep, cw.grad, cw.pos + n_batch, (int)n_t, M.d_e, n_batch, loss->alpha_cmd, 1);
    TPCB_LAUNCH_CHECK("large_dz_cmd_t");
    if ((rc = large_tail(c, ft, b, tgt->h_tok_off, n_t, tgt->devfeat, G, 1))) return rc;
  }
  return stream_wait(st, g_side.s);  // join: every weight gradient is in d_grad
}

