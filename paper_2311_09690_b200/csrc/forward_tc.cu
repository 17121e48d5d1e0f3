// K2+K3, bf16 tensor-core mode (the C5 "bf16" inference path): the desk
// encoder's GEMMs on the 5th-generation tensor cores (tcgen05.mma, fp32
// accumulators in TMEM), everything else fused around them.
//
// Same network and outputs as forward.cu (reference: costmodel.py:193-269,
// nn.py:26-96, dataset.py:97-115); only the encoder GEMM operands are rounded
// to bf16 (fp32 accumulation).  LayerNorm, softmax, residuals, the leaf /
// device head and the Box-Cox decode stay in fp32 / fp64.  The
// accuracy of this mode is stated separately from the fp32 parity mode
// (tests/test_gpu_forward_bf16.py).  The decoder GEMMs (one AST per row)
// also run on the tensor cores.
//
// Layout.  One CTA (4 warps, thread r = row r) per 128-row packed tile
// (rows_per_tile = 128: floor(128/L) whole ASTs of one leaf count),
// persistent over tiles.  All encoder weights live in shared memory for the
// CTA's lifetime as bf16 K-major, 128-byte-swizzled UMMA operand tiles
// (136 KB, one bulk copy of an image prepared by prep_weights_kernel).  The
// activation operand (128 rows × 64 bf16, same swizzle) is rewritten by the
// epilogues; the accumulator tile is 128 TMEM lanes × up to 192 fp32 columns,
// read back with tcgen05.ld (lane = row = thread) so LayerNorm needs no
// cross-thread reduction.  Attention runs per query row on bf16 K/V rows of
// its own AST.
#include <cuda_bf16.h>

#include <cmath>
#include <cstring>

#include "async.cuh"
#include "common.cuh"

namespace tpcb {

namespace {

constexpr int D = 64, FF = 128, DE = 32, DDEV = 16, DEC = 64, NLAY = 2, DH = 32;
constexpr int TR = 128;   // rows per tile = TMEM lanes = threads
constexpr int NTH = 256;  // two warpgroups over the same 128 TMEM lanes

// ---- weight image (bytes): bf16 B operands [N rows][64 k] K-major, SW128 ----
constexpr int kTileB = 64 * 128;  // bytes per 64-row B tile (8 KB)
constexpr int kImgIn = 0;                       // N=64, K=24 (zero-padded to 64)
constexpr int kImgLayer = kTileB;               // + li * kImgLStride
constexpr int kQKV = 0;                         // N=192 (Wq | Wk | Wv)
constexpr int kWO = 3 * kTileB;                 // N=64
constexpr int kFH = 4 * kTileB;                 // N=128
constexpr int kFO0 = 6 * kTileB;                // N=64, k = 0..63 of foW
constexpr int kFO1 = 7 * kTileB;                // N=64, k = 64..127
constexpr int kImgLStride = 8 * kTileB;
constexpr int kImgDec0 = kImgLayer + NLAY * kImgLStride;  // decoder 0: N=64, K=32 (zero-padded)
constexpr int kImgDec1 = kImgDec0 + kTileB;              // decoder 1: N=64, K=64
constexpr int kImgBytes = kImgDec1 + kTileB;              // 155,648 (resident in smem)
// leaf_embed.L images (global only, staged per tile): for each L, a B operand of
// N = L·32 rows (row l·32 + n = column n of W_L's l-th 64-row block) × K = 64,
// SW128, 4 KB per leaf position; image L starts at kImgBytes + 4 KB · L(L−1)/2.
constexpr int kLeafChunkB = 32 * 128;
constexpr int kMaxLeafTC = 16;
__host__ __device__ constexpr int leaf_img_off(int L) {
  return kImgBytes + kLeafChunkB * (L * (L - 1) / 2);
}
constexpr int kImgTotal = leaf_img_off(kMaxLeafTC + 1);   // 712,704

// ---- shared memory (bytes, dynamic) ----
constexpr int kSmA = kImgBytes;                 // A operand [128][64] bf16, SW128 (16 KB)
constexpr int kKVLd = 136;                      // K|V row stride (bf16): 272 B, conflict-free 16-B accesses
constexpr int kSmKV = kSmA + TR * 128;          // K|V bf16 [128][136], later F (two SW128 tiles)
constexpr int kSmVec = kSmKV + TR * kKVLd * 2;  // biases / LN vectors fp32
constexpr int kVecIn = 0, kVecLayer = 64, kVecLStride = 704;  // (same order as train4)
constexpr int kVBQKV = 0, kVBO = 192, kVLN1G = 256, kVLN1B = 320, kVFHB = 384, kVFOB = 512,
              kVLN2G = 576, kVLN2B = 640;
constexpr int kVecHead = kVecLayer + NLAY * kVecLStride;  // head vectors (fp32)
constexpr int kVHLeafB = 0;                            // leaf_embed.L.b, [17][32]
constexpr int kVHDevHW = kVHLeafB + (kMaxLeafTC + 1) * DE;  // [6][16]
constexpr int kVHDevHB = kVHDevHW + TPCB_DEV_FEAT * DDEV;
constexpr int kVHDevPW = kVHDevHB + DDEV;               // [16][32]
constexpr int kVHDevPB = kVHDevPW + DDEV * DE;
constexpr int kVHDecB0 = kVHDevPB + DE;
constexpr int kVHDecB1 = kVHDecB0 + DEC;
constexpr int kVHOutW = kVHDecB1 + DEC;
constexpr int kVHOutB = kVHOutW + DEC;
constexpr int kVecFloats = kVecHead + kVHOutB + 4;
// leaf_embed GEMM staging inside [kSmA, kSmVec): A chunk l (row a = token a·L + l)
// at l · leaf_chunk_a(L), B chunks after them (see the head)
constexpr int kLeafRegion = kSmVec - kSmA;             // 51,200
__device__ __forceinline__ int leaf_chunk_a(int L) {   // bytes per A chunk: ⌈⌊128/L⌋/8⌉ atoms
  return L == 1 ? TR * 128 : (((TR / L) + 7) >> 3) * 1024;
}
// per-AST sample index and device features of the current tile, fetched by
// cp.async at the tile start (off the head's critical path)
constexpr int kSmAst = kSmVec + kVecFloats * 4;
constexpr int kSmTotal = kSmAst + TR * 4 + TR * TPCB_DEV_FEAT * 4;

__host__ __device__ inline uint32_t sw128(int r, int k) {  // bf16 element (row r, col k < 64)
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7))) << 4) + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                 // leading byte offset (unused: SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset: 8-row swizzle atoms
  d |= (uint64_t)1 << 46;                 // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                 // 128-byte swizzle
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {  // bf16 × bf16 → fp32, K-major
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// D[tmem] (+)= A[128 × 64·ka] · B[n × 64·ka]ᵀ, k chunks of 64 (one SW128 tile each)
__device__ __forceinline__ void mma_chain(uint32_t tmem, const uint32_t* a_tiles,
                                          const uint32_t* b_tiles, int nchunks, int n) {
  const uint32_t id = idesc_bf16(TR, n);
  for (int c = 0; c < nchunks; ++c)
    for (int k = 0; k < 4; ++k) {
      const uint64_t a = sdesc(a_tiles[c] + k * 32), b = sdesc(b_tiles[c] + k * 32);
      const uint32_t acc = (c | k) != 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(a), "l"(b), "r"(id), "r"(acc));
    }
}

// one lane of a converged warp (elect.sync): MMA issue from a warp-uniform
// context, so the descriptors stay in uniform registers
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}

// 32 consecutive fp32 columns of this thread's TMEM lane (warp w owns lanes 32w..32w+31)
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

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// 8 bf16 values → columns c0..c0+7 of row r of a SW128 A tile
__device__ __forceinline__ void store8_bf16(uint8_t* tile, int r, int c0, const float* v) {
  __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]);
  __nv_bfloat162 p1 = __floats2bfloat162_rn(v[2], v[3]);
  __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]);
  __nv_bfloat162 p3 = __floats2bfloat162_rn(v[6], v[7]);
  uint4 u;
  u.x = *reinterpret_cast<uint32_t*>(&p0);
  u.y = *reinterpret_cast<uint32_t*>(&p1);
  u.z = *reinterpret_cast<uint32_t*>(&p2);
  u.w = *reinterpret_cast<uint32_t*>(&p3);
  *reinterpret_cast<uint4*>(tile + sw128(r, c0)) = u;
}

// this thread's 64 bf16 values → row r of a SW128 A tile
__device__ __forceinline__ void store_row_bf16(uint8_t* tile, int r, const float* v) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * c + 0], v[8 * c + 1]);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * c + 2], v[8 * c + 3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * c + 4], v[8 * c + 5]);
    __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * c + 6], v[8 * c + 7]);
    uint4 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    u.z = *reinterpret_cast<uint32_t*>(&p2);
    u.w = *reinterpret_cast<uint32_t*>(&p3);
    *reinterpret_cast<uint4*>(tile + sw128(r, 8 * c)) = u;
  }
}

// 32 bf16 values → columns 32·half .. 32·half+31 of row r of a SW128 A tile
__device__ __forceinline__ void store_half_row_bf16(uint8_t* tile, int r, int half, const float* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * c + 0], v[8 * c + 1]);
    __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * c + 2], v[8 * c + 3]);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * c + 4], v[8 * c + 5]);
    __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * c + 6], v[8 * c + 7]);
    uint4 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    u.z = *reinterpret_cast<uint32_t*>(&p2);
    u.w = *reinterpret_cast<uint32_t*>(&p3);
    *reinterpret_cast<uint4*>(tile + sw128(r, 32 * half + 8 * c)) = u;
  }
}

// operand writes (generic proxy) → visible to the tensor cores; CTA barrier
__device__ __forceinline__ void sync_for_mma() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
  mbar_wait(bar, phase);
  phase ^= 1;
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// LayerNorm of a row split over two threads (warpgroup wg holds columns
// 32·wg .. 32·wg+31): two-pass mean / biased variance, eps 1e-5 (nn.py:48-54);
// both halves combine the partial sums in the same order.  red: [4][TR].
__device__ __forceinline__ void ln_half(float* v, const float* g, const float* b, int wg, int r,
                                        float* red) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < DH; ++i) s += v[i];
  red[wg * TR + r] = s;
  __syncthreads();
  const float mu = (red[r] + red[TR + r]) * (1.f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < DH; ++i) {
    const float t = v[i] - mu;
    q = fmaf(t, t, q);
  }
  red[(2 + wg) * TR + r] = q;
  __syncthreads();
  const float inv = 1.f / sqrtf((red[2 * TR + r] + red[3 * TR + r]) * (1.f / D) + 1e-5f);
#pragma unroll
  for (int i = 0; i < DH; ++i) v[i] = fmaf(g[DH * wg + i], (v[i] - mu) * inv, b[DH * wg + i]);
}

__device__ __forceinline__ double boxcox_decode_tc(double e, const tpcb_boxcox& bc, bool* bad) {
  const double t = e * bc.t_std + bc.t_mean;
  if (fabs(bc.lambda_bc) < 1e-9) return exp(t) - bc.shift;
  const double base = bc.lambda_bc * t + 1.0;
  if (!(base > 0.0)) {
    *bad = true;
    return nan("");
  }
  return pow(base, 1.0 / bc.lambda_bc) - bc.shift;
}

// fp32 parameters → the bf16 weight image (see kImg*)
__global__ void prep_weights_kernel(const Model M, const float* __restrict__ P,
                                    uint8_t* __restrict__ img) {
  const int total = kImgTotal / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int byte = e * 2;
    if (byte >= kImgBytes) {  // leaf_embed.L: find L, then (l, n, k) inside its image
      int L = 1;
      while (leaf_img_off(L + 1) <= byte) ++L;
      const int in = byte - leaf_img_off(L);
      const int atom = in >> 10, rr = (in >> 7) & 7, chunk = ((in >> 4) & 7) ^ rr;
      const int nrow = atom * 8 + rr, k = chunk * 8 + ((in & 15) >> 1);
      const int l = nrow >> 5, n = nrow & 31;
      const float v = L <= M.n_leaf_max ? P[M.leafW[L] + (l * D + k) * DE + n] : 0.f;
      reinterpret_cast<__nv_bfloat16*>(img)[e] = __float2bfloat16_rn(v);
      continue;
    }
    // locate (tile base, n, k) from the byte offset: invert sw128 within 8-KB tiles
    const int tile = byte / kTileB, in = byte - tile * kTileB;
    const int atom = in >> 10, rr = (in >> 7) & 7, chunk = ((in >> 4) & 7) ^ rr;
    const int n_local = atom * 8 + rr, k = chunk * 8 + ((in & 15) >> 1);
    float v = 0.f;
    if (tile == 0) {
      v = k < TPCB_FEAT ? P[M.inW + k * D + n_local] : 0.f;
    } else if (tile == kImgDec0 / kTileB) {
      v = k < DE ? P[M.decW[0] + k * DEC + n_local] : 0.f;
    } else if (tile == kImgDec1 / kTileB) {
      v = P[M.decW[1] + k * DEC + n_local];
    } else {
      const int li = (tile - 1) / 8, t = (tile - 1) % 8;
      const LayerOff& lo = M.layer[li];
      if (t < 3) {
        const int n = t * 64 + n_local;  // Q | K | V
        const int off = n < 64 ? lo.Wq : (n < 128 ? lo.Wk : lo.Wv);
        v = P[off + k * D + (n & 63)];
      } else if (t == 3) {
        v = P[lo.Wo + k * D + n_local];
      } else if (t < 6) {
        v = P[lo.fhW + k * FF + (t - 4) * 64 + n_local];
      } else {
        v = P[lo.foW + ((t - 6) * 64 + k) * D + n_local];
      }
    }
    reinterpret_cast<__nv_bfloat16*>(img)[e] = __float2bfloat16_rn(v);
  }
}

// attention of one query row over its AST's LL keys (head columns hc..hc+31
// of the K|V rows), LL a compile-time count: every score first (independent
// dot products, registers), then the weights and the context
template <int LL>
__device__ __forceinline__ void attn_fixed(const uint8_t* __restrict__ sKV, int r0, int hc,
                                           const float* q, float scale, float* c) {
  float sc[LL];
#pragma unroll
  for (int j = 0; j < LL; ++j) {
    const uint4* kr = reinterpret_cast<const uint4*>(sKV + ((r0 + j) * kKVLd + hc) * 2);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      const uint4 u = kr[i];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
        acc[e] = fmaf(q[8 * i + 2 * e], kf.x, fmaf(q[8 * i + 2 * e + 1], kf.y, acc[e]));
      }
    }
    sc[j] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * scale;
  }
  float m = sc[0];
#pragma unroll
  for (int j = 1; j < LL; ++j) m = fmaxf(m, sc[j]);
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < LL; ++j) {
    const float pj = LL == 1 ? 1.f : expf(sc[j] - m);
    sum += pj;
    const uint4* vr = reinterpret_cast<const uint4*>(sKV + ((r0 + j) * kKVLd + D + hc) * 2);
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      const uint4 u = vr[i];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
        c[8 * i + 2 * e] = fmaf(pj, vf.x, c[8 * i + 2 * e]);
        c[8 * i + 2 * e + 1] = fmaf(pj, vf.y, c[8 * i + 2 * e + 1]);
      }
    }
  }
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < DH; ++i) c[i] *= inv;
}

__device__ long long* g_trace_tc = nullptr;
// debug: per-phase timestamps of CTA 0 / thread 0 for its last 8 tiles (ring)
#define TT(id)                                                                   \
  do {                                                                           \
    if (g_trace_tc && blockIdx.x == 0 && t == 0)                                 \
      g_trace_tc[(tcount & 7) * 32 + (id)] = clock64();                          \
  } while (0)

__global__ void __launch_bounds__(NTH, 1) forward_tc_kernel(
    const __grid_constant__ Model M, const float* __restrict__ P,
    const uint8_t* __restrict__ img, const float* __restrict__ x,
    const int32_t* __restrict__ tile_L, const int32_t* __restrict__ tile_first,
    const int32_t* __restrict__ tile_count, const int32_t* __restrict__ n_tiles_p,
    const int32_t* __restrict__ perm, const float* __restrict__ devfeat, tpcb_boxcox bc,
    float* __restrict__ pred_out, float* __restrict__ zx_out, float* __restrict__ zv_out,
    float* __restrict__ z_out, double* __restrict__ lat_out, int32_t* status) {
  extern __shared__ __align__(1024) uint8_t smb[];
  __shared__ __align__(8) uint64_t bars[4];  // [0] weights, [1] MMA done, [2] leaf B landed, [3] leaf group done
  __shared__ uint32_t s_tmem;
  __shared__ float s_red[4 * TR];  // split-row LayerNorm partial sums
  const int t = threadIdx.x, warp = t >> 5;
  const int wg = warp >> 2, r = t & (TR - 1);  // warpgroup, row = TMEM lane
  const int n_tiles = *n_tiles_p;
  uint8_t* sA = smb + kSmA;
  uint8_t* sKV = smb + kSmKV;
  float* sv = reinterpret_cast<float*>(smb + kSmVec);
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    mbar_init(&bars[3], 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t tlane = tmem + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lanes
  if (t == 0 && (smem_u32(smb) & 1023u)) raise_status(status, TPCB_ERR_CUDA);  // swizzle atoms
  if (t == 0) {  // the weight image: one bulk copy for the CTA's lifetime
    mbar_arrive_expect_tx(&bars[0], (uint32_t)kImgBytes);
    bulk_g2s(smb, img, (uint32_t)kImgBytes, &bars[0]);
  }
  // biases and LayerNorm vectors (fp32)
  for (int i = t; i < D; i += NTH) sv[kVecIn + i] = __ldg(P + M.inb + i);
  for (int li = 0; li < NLAY; ++li) {
    const LayerOff& lo = M.layer[li];
    float* b = sv + kVecLayer + li * kVecLStride;
    for (int i = t; i < D; i += NTH) {
      b[kVBQKV + i] = __ldg(P + lo.bq + i);
      b[kVBQKV + D + i] = __ldg(P + lo.bk + i);
      b[kVBQKV + 2 * D + i] = __ldg(P + lo.bv + i);
      b[kVBO + i] = __ldg(P + lo.bo + i);
      b[kVLN1G + i] = __ldg(P + lo.ln1g + i);
      b[kVLN1B + i] = __ldg(P + lo.ln1b + i);
      b[kVFOB + i] = __ldg(P + lo.fob + i);
      b[kVLN2G + i] = __ldg(P + lo.ln2g + i);
      b[kVLN2B + i] = __ldg(P + lo.ln2b + i);
    }
    for (int i = t; i < FF; i += NTH) b[kVFHB + i] = __ldg(P + lo.fhb + i);
  }
  {
    float* hv = sv + kVecHead;
    for (int i = t; i < (kMaxLeafTC + 1) * DE; i += NTH) {
      const int L = i / DE;
      hv[kVHLeafB + i] = (L >= 1 && L <= M.n_leaf_max) ? __ldg(P + M.leafb[L] + (i - L * DE)) : 0.f;
    }
    for (int i = t; i < TPCB_DEV_FEAT * DDEV; i += NTH) hv[kVHDevHW + i] = __ldg(P + M.devhW + i);
    for (int i = t; i < DDEV * DE; i += NTH) hv[kVHDevPW + i] = __ldg(P + M.devpW + i);
    for (int i = t; i < DDEV; i += NTH) hv[kVHDevHB + i] = __ldg(P + M.devhb + i);
    for (int i = t; i < DE; i += NTH) hv[kVHDevPB + i] = __ldg(P + M.devpb + i);
    for (int i = t; i < DEC; i += NTH) {
      hv[kVHDecB0 + i] = __ldg(P + M.decb[0] + i);
      hv[kVHDecB1 + i] = __ldg(P + M.decb[1] + i);
      hv[kVHOutW + i] = __ldg(P + M.outW + i);
    }
    if (t == 0) hv[kVHOutB] = __ldg(P + M.outb);
  }
  const float* hv = sv + kVecHead;
  mbar_wait(&bars[0], 0);
  const uint32_t a_addr = smem_u32(sA), kv_addr = smem_u32(sKV), w_addr = smem_u32(smb);
  const float scale = 1.f / sqrtf((float)DH);
  uint32_t phase = 0, phase_b = 0, phase_g = 0;

  // warpgroup 1 prefetches the next tile's input rows into registers while
  // warpgroup 0 runs the previous tile's last LayerNorm, leaf_embed and head
  float xn[TPCB_FEAT];
  auto load_x = [&](int tl) {
    if (wg == 1 && tl < n_tiles) {
      const float* xr = x + ((size_t)tl * TR + r) * TPCB_FEAT_PAD;
#pragma unroll
      for (int i = 0; i < TPCB_FEAT; i += 4) {
        const float4 q4 = __ldg(reinterpret_cast<const float4*>(xr + i));
        xn[i] = q4.x; xn[i + 1] = q4.y; xn[i + 2] = q4.z; xn[i + 3] = q4.w;
      }
    }
  };
  load_x(blockIdx.x);
  bool a_staged = false;  // warpgroup 1 already wrote this tile's A rows
  int tcount = -1;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    ++tcount;
    TT(0);
    const int L = tile_L[tile], first = tile_first[tile], A = tile_count[tile];
    const int rows = A * L;
    const bool live = r < rows;
    int32_t* s_idx = reinterpret_cast<int32_t*>(smb + kSmAst);
    float* s_dv = reinterpret_cast<float*>(smb + kSmAst + TR * 4);

    float h[DH];  // this row's residual stream, columns 32·wg .. 32·wg+31 (fp32)
    if (wg == 1) {  // prefetched input rows → A operand (24 features, zero-padded to 64)
      if (!a_staged) {  // (from the second tile on, staged under the previous decoder)
        float v[D];
#pragma unroll
        for (int i = 0; i < D; ++i) v[i] = (live && i < TPCB_FEAT) ? xn[i < TPCB_FEAT ? i : 0] : 0.f;
        store_row_bf16(sA, r, v);
      }
      if (r < A) cp_async4(s_idx + r, perm + first + r);  // lands under the input projection
    }
    a_staged = false;
    sync_for_mma();
    TT(1);
    if (warp == 0 && elect_one()) {
      const uint32_t at[1] = {a_addr}, bt[1] = {w_addr + kImgIn};
      mma_chain(tmem, at, bt, 1, D);
      mma_commit(&bars[1]);
    }
    wait_mma(&bars[1], phase);
    TT(2);
    if (wg == 1 && r < A) {  // the AST's device features, by its (now landed) index
      cp_async_wait_all();
      const float* dvp = devfeat + (size_t)s_idx[r] * TPCB_DEV_FEAT;
#pragma unroll
      for (int f = 0; f < TPCB_DEV_FEAT; ++f) cp_async4(s_dv + r * TPCB_DEV_FEAT + f, dvp + f);
    }
    {
      tmem_ld32(tlane + DH * wg, h);
#pragma unroll
      for (int i = 0; i < DH; ++i) h[i] += sv[kVecIn + DH * wg + i];
      store_half_row_bf16(sA, r, wg, h);
    }
    sync_for_mma();
    TT(3);

    for (int li = 0; li < NLAY; ++li) {
      const float* b = sv + kVecLayer + li * kVecLStride;
      const uint32_t wl = w_addr + kImgLayer + li * kImgLStride;
      if (warp == 0 && elect_one()) {  // Q | K | V
        const uint32_t at[1] = {a_addr}, bt[1] = {wl + kQKV};
        mma_chain(tmem, at, bt, 1, 3 * D);
        mma_commit(&bars[1]);
      }
      wait_mma(&bars[1], phase);
      TT(4 + li * 12);
      // warpgroup wg owns head wg (nn.py:79-96): its 32 Q columns stay in
      // registers, its K and V columns go to bf16 rows [K 0..63 | V 64..127]
      const int hc = wg * DH;
      float q[DH];
      tmem_ld32(tlane + hc, q);
#pragma unroll
      for (int i = 0; i < DH; ++i) q[i] += b[kVBQKV + hc + i];
      {
        float kv[DH];
        uint8_t* dst = sKV + r * kKVLd * 2;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          tmem_ld32(tlane + 64 + 64 * part + hc, kv);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float* bb = b + kVBQKV + (1 + part) * D + hc + 8 * c;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(kv[8 * c] + bb[0], kv[8 * c + 1] + bb[1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(kv[8 * c + 2] + bb[2], kv[8 * c + 3] + bb[3]);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(kv[8 * c + 4] + bb[4], kv[8 * c + 5] + bb[5]);
            __nv_bfloat162 p3 = __floats2bfloat162_rn(kv[8 * c + 6] + bb[6], kv[8 * c + 7] + bb[7]);
            uint4 u;
            u.x = *reinterpret_cast<uint32_t*>(&p0);
            u.y = *reinterpret_cast<uint32_t*>(&p1);
            u.z = *reinterpret_cast<uint32_t*>(&p2);
            u.w = *reinterpret_cast<uint32_t*>(&p3);
            *reinterpret_cast<uint4*>(dst + (64 * part + hc + 8 * c) * 2) = u;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      // attention of this query row over its AST's L keys, head wg
      float c[DH];
#pragma unroll
      for (int i = 0; i < DH; ++i) c[i] = 0.f;
      if (live && L <= 6) {  // the common small leaf counts: unrolled per L
        const int r0 = (r / L) * L;
        switch (L) {
          case 1: attn_fixed<1>(sKV, r0, hc, q, scale, c); break;
          case 2: attn_fixed<2>(sKV, r0, hc, q, scale, c); break;
          case 3: attn_fixed<3>(sKV, r0, hc, q, scale, c); break;
          case 4: attn_fixed<4>(sKV, r0, hc, q, scale, c); break;
          case 5: attn_fixed<5>(sKV, r0, hc, q, scale, c); break;
          default: attn_fixed<6>(sKV, r0, hc, q, scale, c); break;
        }
      } else if (live) {
        // one pass over the keys with a running max (no score array, so no
        // stack frame): the context is rescaled only when the max grows
        const int r0 = (r / L) * L;
        float m = -INFINITY, sum = 0.f;
        for (int j = 0; j < L; ++j) {
          const uint4* kr = reinterpret_cast<const uint4*>(sKV + ((r0 + j) * kKVLd + hc) * 2);
          const uint4* vr = reinterpret_cast<const uint4*>(sKV + ((r0 + j) * kKVLd + D + hc) * 2);
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < DH / 8; ++i) {
            const uint4 u = kr[i];
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
              acc[e] = fmaf(q[8 * i + 2 * e], kf.x, fmaf(q[8 * i + 2 * e + 1], kf.y, acc[e]));
            }
          }
          const float sj = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * scale;
          if (sj > m) {
            const float alpha = expf(m - sj);  // 0 on the first key
            sum *= alpha;
#pragma unroll
            for (int i = 0; i < DH; ++i) c[i] *= alpha;
            m = sj;
          }
          const float pj = expf(sj - m);
          sum += pj;
#pragma unroll
          for (int i = 0; i < DH / 8; ++i) {
            const uint4 u = vr[i];
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
              c[8 * i + 2 * e] = fmaf(pj, vf.x, c[8 * i + 2 * e]);
              c[8 * i + 2 * e + 1] = fmaf(pj, vf.y, c[8 * i + 2 * e + 1]);
            }
          }
        }
        const float inv = 1.f / sum;
#pragma unroll
        for (int i = 0; i < DH; ++i) c[i] *= inv;
      }
      store_half_row_bf16(sA, r, wg, c);
      sync_for_mma();
      TT(5 + li * 12);
      if (warp == 0 && elect_one()) {  // output projection
        const uint32_t at[1] = {a_addr}, bt[1] = {wl + kWO};
        mma_chain(tmem, at, bt, 1, D);
        mma_commit(&bars[1]);
      }
      wait_mma(&bars[1], phase);
      TT(6 + li * 12);
      float h1[DH];
      {
        tmem_ld32(tlane + DH * wg, h1);
#pragma unroll
        for (int i = 0; i < DH; ++i) h1[i] += b[kVBO + DH * wg + i] + h[i];
        ln_half(h1, b + kVLN1G, b + kVLN1B, wg, r, s_red);
        store_half_row_bf16(sA, r, wg, h1);
      }
      sync_for_mma();
      TT(7 + li * 12);
      if (warp == 0 && elect_one()) {  // FFN hidden (N = 128)
        const uint32_t at[1] = {a_addr}, bt[1] = {wl + kFH};
        mma_chain(tmem, at, bt, 1, FF);
        mma_commit(&bars[1]);
      }
      wait_mma(&bars[1], phase);
      TT(8 + li * 12);
      {  // ReLU → F half wg (two SW128 A tiles in the K|V region: the keys are dead)
        float f[D];
        tmem_ld32(tlane + 64 * wg, f);
        tmem_ld32(tlane + 64 * wg + 32, f + 32);
#pragma unroll
        for (int i = 0; i < D; ++i) f[i] = fmaxf(f[i] + b[kVFHB + 64 * wg + i], 0.f);
        store_row_bf16(sKV + wg * TR * 128, r, f);
      }
      if (li + 1 == NLAY) load_x(tile + gridDim.x);
      sync_for_mma();
      TT(9 + li * 12);
      if (warp == 0 && elect_one()) {  // FFN out (K = 128)
        const uint32_t at[2] = {kv_addr, kv_addr + TR * 128},
                       bt[2] = {wl + kFO0, wl + kFO1};
        mma_chain(tmem, at, bt, 2, D);
        mma_commit(&bars[1]);
      }
      wait_mma(&bars[1], phase);
      TT(10 + li * 12);
      if (li + 1 == NLAY && t == 0) {  // K|V / F are dead: stage leaf_embed B chunks now
        const int boff = L * leaf_chunk_a(L);
        const int g = min(L, (kLeafRegion - boff) / kLeafChunkB);
        mbar_arrive_expect_tx(&bars[2], (uint32_t)(g * kLeafChunkB));
        bulk_g2s(sA + boff, img + leaf_img_off(L), (uint32_t)(g * kLeafChunkB), &bars[2]);
      }
      {
        tmem_ld32(tlane + DH * wg, h);
#pragma unroll
        for (int i = 0; i < DH; ++i) h[i] += b[kVFOB + DH * wg + i] + h1[i];
        ln_half(h, b + kVLN2G, b + kVLN2B, wg, r, s_red);
        if (li + 1 < NLAY) store_half_row_bf16(sA, r, wg, h);
        else if (live)  // leaf_embed A operand: chunk l = r mod L, row a = r / L
          store_half_row_bf16(sA + (r % L) * leaf_chunk_a(L), r / L, wg, h);
      }
      if (li + 1 < NLAY) {
        sync_for_mma();
        TT(11 + li * 12);
      }
    }
    TT(30);
    if (wg == 1) cp_async_wait_all();  // device features (visible after the barrier below)
    // ---------------------------------------------------------------- head
    // leaf_embed on the tensor cores (costmodel.py:213-216): A chunk l holds row
    // a = token a·L + l (written by the last LayerNorm epilogue), B chunk l is
    // W_L's l-th 64-row block, so D[a] = Σ_l h[a·L+l] · W_L[l] = z_x[a] − b_L
    // accumulates over the L chunks in TMEM (columns 0..31, one AST per lane).
    sync_for_mma();
    TT(12);
    if (warp == 0 && elect_one()) {
      const int cb = leaf_chunk_a(L), boff = L * cb;
      const int G = min(L, (kLeafRegion - boff) / kLeafChunkB);
      const uint32_t id = idesc_bf16(TR, DE);
      for (int l0 = 0; l0 < L; l0 += G) {
        const int g = min(G, L - l0);
        if (l0 > 0) {  // L > G: the previous group's MMAs must finish before B is restaged
          mma_commit(&bars[3]);
          mbar_wait(&bars[3], phase_g);
          phase_g ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          mbar_arrive_expect_tx(&bars[2], (uint32_t)(g * kLeafChunkB));
          bulk_g2s(sA + boff, img + leaf_img_off(L) + l0 * kLeafChunkB,
                   (uint32_t)(g * kLeafChunkB), &bars[2]);
        }
        mbar_wait(&bars[2], phase_b);
        phase_b ^= 1;
        TT(13);
        for (int j = 0; j < g; ++j) {
          const uint32_t ab = a_addr + (uint32_t)((l0 + j) * cb),
                         bb = a_addr + (uint32_t)(boff + j * kLeafChunkB);
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = sdesc(ab + k * 32), bd = sdesc(bb + k * 32);
            const uint32_t acc = ((l0 + j) | k) != 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(id), "r"(acc));
          }
        }
      }
      TT(14);
      mma_commit(&bars[1]);
    }
    wait_mma(&bars[1], phase);
    TT(25);
    {  // z_x, device MLP and gate for AST a = r (a < A), columns 16·wg .. 16·wg+15
       // per warpgroup → decoder operand row a (costmodel.py:213-220)
      float zx[16];
      tmem_ld16(tlane + 16 * wg, zx);  // warp-collective: every lane loads
      if (r < A) {
        const int a = r, idx = s_idx[a];
        const float* dv = s_dv + a * TPCB_DEV_FEAT;
        float zv[DDEV];
#pragma unroll
        for (int n = 0; n < DDEV; ++n) {
          float sacc = hv[kVHDevHB + n];
#pragma unroll
          for (int f = 0; f < TPCB_DEV_FEAT; ++f) sacc = fmaf(dv[f], hv[kVHDevHW + f * DDEV + n], sacc);
          zv[n] = fmaxf(sacc, 0.f);
        }
        float z[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int n = 16 * wg + q;
          zx[q] += hv[kVHLeafB + L * DE + n];
          float sacc = hv[kVHDevPB + n];
#pragma unroll
          for (int k = 0; k < DDEV; ++k) sacc = fmaf(zv[k], hv[kVHDevPW + k * DE + n], sacc);
          z[q] = zx[q] * sacc;
        }
        const float zero[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        store8_bf16(sA, a, 16 * wg, z);
        store8_bf16(sA, a, 16 * wg + 8, z + 8);
        store8_bf16(sA, a, 32 + 16 * wg, zero);
        store8_bf16(sA, a, 40 + 16 * wg, zero);
        if (zx_out)
          for (int q = 0; q < 16; ++q) zx_out[(size_t)idx * DE + 16 * wg + q] = zx[q];
        if (z_out)
          for (int q = 0; q < 16; ++q) z_out[(size_t)idx * DE + 16 * wg + q] = z[q];
        if (zv_out && wg == 0)
          for (int n = 0; n < DDEV; ++n) zv_out[(size_t)idx * DDEV + n] = zv[n];
      }
    }
    sync_for_mma();
    TT(26);
    // decoder on the tensor cores, one AST per row / TMEM lane / thread
    if (warp == 0 && elect_one()) {
      const uint32_t at[1] = {a_addr}, bt[1] = {w_addr + kImgDec0};
      mma_chain(tmem, at, bt, 1, DEC);
      mma_commit(&bars[1]);
    }
    wait_mma(&bars[1], phase);
    TT(27);
    {  // dec0 epilogue split by column half (warpgroup wg: columns 32·wg ..)
      float u[DH];
      tmem_ld32(tlane + DH * wg, u);
#pragma unroll
      for (int j = 0; j < DH; ++j) u[j] = fmaxf(u[j] + hv[kVHDecB0 + DH * wg + j], 0.f);
      store_half_row_bf16(sA, r, wg, u);
    }
    sync_for_mma();
    if (warp == 0 && elect_one()) {
      const uint32_t at[1] = {a_addr}, bt[1] = {w_addr + kImgDec1};
      mma_chain(tmem, at, bt, 1, DEC);
      mma_commit(&bars[1]);
    }
    wait_mma(&bars[1], phase);
    TT(28);
    if (wg == 0) {
      float u[DEC];
      tmem_ld32(tlane, u);
      tmem_ld32(tlane + 32, u + 32);
      if (t < A) {
        float pred = hv[kVHOutB];
#pragma unroll
        for (int j = 0; j < DEC; ++j)
          pred = fmaf(fmaxf(u[j] + hv[kVHDecB1 + j], 0.f), hv[kVHOutW + j], pred);
        const int idx = s_idx[t];
        pred_out[idx] = pred;
        if (lat_out) {
          bool bad = false;
          lat_out[idx] = bc.enabled ? boxcox_decode_tc((double)pred, bc, &bad) : (double)pred;
          if (bad) raise_status(status, TPCB_ERR_DOMAIN);
        }
      }
    } else if (tile + (int)gridDim.x < n_tiles) {
      // warpgroup 1 is idle in the decoder's last epilogue and the A operand
      // is dead once the dec1 MMA has completed: stage the next tile's rows now
      const int nt = tile + gridDim.x;
      const bool live_n = r < tile_count[nt] * tile_L[nt];
      float v[D];
#pragma unroll
      for (int i = 0; i < D; ++i) v[i] = (live_n && i < TPCB_FEAT) ? xn[i < TPCB_FEAT ? i : 0] : 0.f;
      store_row_bf16(sA, r, v);
      a_staged = true;
    }
    TT(31);
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

bool tc_supported(const Model& M) {
  if (M.d != D || M.n_layers != NLAY || M.n_heads != 2 || M.dh != DH || M.d_ff != FF) return false;
  if (M.d_e != DE || M.d_dev != DDEV || M.n_dec != 2 || M.dec[0] != DEC || M.dec[1] != DEC)
    return false;
  return M.n_leaf_max <= kMaxLeafTC;
}

}  // namespace

}  // namespace tpcb

using namespace tpcb;

/* bf16 tensor-core forward (C5 mode): same contract as tpcb_forward, desk-shaped
 * models, rows_per_tile must be 128; d_img: caller workspace of
 * tpcb_forward_bf16_workspace() bytes (the bf16 weight image, rebuilt per call). */
extern "C" size_t tpcb_forward_bf16_workspace(void) { return (size_t)kImgTotal; }

namespace tpcb {
int set_forward_tc_trace(long long* d) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace_tc, &d, sizeof(d)));
  return TPCB_OK;
}
}  // namespace tpcb

extern "C" int tpcb_forward_bf16(const tpcb_model* m, const float* d_params, const tpcb_packed* pk,
                                 const float* d_devfeat, int64_t n_ast, const tpcb_boxcox* norm,
                                 void* d_img, float* d_pred, float* d_zx, float* d_zv, float* d_z,
                                 double* d_latency, int32_t* d_status, void* stream_) {
  if (!m || !pk || !d_params || !d_pred || !d_devfeat || !d_img) return TPCB_ERR_VALIDATION;
  if (n_ast < 1) return TPCB_ERR_EMPTY_BATCH;
  if (!tc_supported(m->dev) || pk->rows_per_tile != TR) return TPCB_ERR_UNSUPPORTED;
  cudaStream_t stream = (cudaStream_t)stream_;
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(forward_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmTotal));
    attr = true;
  }
  prep_weights_kernel<<<2 * kNumSMs, 256, 0, stream>>>(m->dev, d_params,
                                                       static_cast<uint8_t*>(d_img));
  TPCB_LAUNCH_CHECK("prep_weights_kernel");
  tpcb_boxcox bc{};
  if (norm) bc = *norm;
  const int grid = (int)std::min<int64_t>(pk->n_tiles_max, (int64_t)kNumSMs);
  forward_tc_kernel<<<grid, NTH, kSmTotal, stream>>>(
      m->dev, d_params, static_cast<const uint8_t*>(d_img), pk->x, pk->tile_L, pk->tile_first,
      pk->tile_count, pk->n_tiles, pk->perm, d_devfeat, bc, d_pred, d_zx, d_zv, d_z, d_latency,
      d_status);
  TPCB_LAUNCH_CHECK("forward_tc_kernel");
  return TPCB_OK;
}
