// K2+K3, fp32 parity mode, desk-shaped models: the fused encoder + head
// forward with one thread per packed row and warpgroup, FP32 FFMA products
// against weight tiles staged in shared memory.
//
// Same network and arithmetic class as forward.cu (reference:
// costmodel.py:193-269, nn.py:26-96, dataset.py:97-115): every product
// accumulates in fp32, LayerNorm is two-pass, the Box-Cox decode is fp64.
// The generic kernel (forward.cu) reads weights through L1 and tiles 64 rows
// over 256 (row group × column group) threads; this one is built for the
// desk shape:
//
//  * one CTA per 128-row packed tile (persistent over tiles), 256 threads:
//    thread (r, wg) owns row r and the column half wg (= attention head wg);
//    the residual stream lives in registers, split over the two threads of
//    the row (LayerNorm combines the halves' partial sums through smem);
//  * products are row × tile: the row's activations come from a padded smem
//    row (LDS.128, conflict-free), the weights from a 16 KB smem slot read
//    as warp-uniform LDS.128 broadcasts (one wavefront serves 32 lanes ×
//    4 FFMA), 32 or 64 independent accumulators per thread;
//  * weights stream from L2 (they are fp32 parameters, 16-B aligned, copied
//    straight from the flat parameter vector) through a 4-slot ring by bulk
//    async copies one phase ahead: per layer Wq Wk Wv Wo → slots 0 1 2 3,
//    fhW → slots 0-1, foW → slots 2-3; the input projection and decoder
//    weights stay resident; leaf_embed.L is staged into the K|V / FFN region
//    once the encoder is done with it.
#include <cmath>

#include "async.cuh"
#include "common.cuh"

namespace tpcb {

namespace {

constexpr int D = 64, FF = 128, DE = 32, DDEV = 16, DEC = 64, NLAY = 2, DH = 32;
constexpr int TR = 128;   // rows per tile
constexpr int NTH = 256;  // two warpgroups
constexpr int kMaxLeaf = 16;

// ---- shared memory (bytes) ----
constexpr int kSlotB = 64 * 64 * 4;            // ring slot: one 64 × 64 fp32 tile
constexpr int kRing = 0;                       // 4 slots
constexpr int LDA = 68;                        // activation row stride (floats)
constexpr int kSmA = kRing + 4 * kSlotB;       // [128][68] activation rows
constexpr int LDK = 132;                       // K|V and FFN-hidden row stride (floats)
constexpr int kSmKV = kSmA + TR * LDA * 4;     // [128][132]: K|V, then F, then leaf_embed.L
constexpr int kSmRes = kSmKV + TR * LDK * 4;   // resident: inW [24][64], dec0W [32][64], dec1W [64][64]
constexpr int kResIn = 0, kResDec0 = TPCB_FEAT * D, kResDec1 = kResDec0 + DE * DEC;
constexpr int kResFloats = kResDec1 + DEC * DEC;
constexpr int kSmZx = kSmRes + kResFloats * 4;  // z_x rows [128][36]
constexpr int LDZ = 36;
constexpr int kSmVec = kSmZx + TR * LDZ * 4;    // biases / LN / head vectors
constexpr int kVIn = 0, kVLayer = 64, kVLStride = 704;  // (same order as forward_tc / train4)
constexpr int kVBQKV = 0, kVBO = 192, kVLN1G = 256, kVLN1B = 320, kVFHB = 384, kVFOB = 512,
              kVLN2G = 576, kVLN2B = 640;
constexpr int kVHead = kVLayer + NLAY * kVLStride;
constexpr int kVHLeafB = 0;
constexpr int kVHDevHW = kVHLeafB + (kMaxLeaf + 1) * DE;
constexpr int kVHDevHB = kVHDevHW + TPCB_DEV_FEAT * DDEV;
constexpr int kVHDevPW = kVHDevHB + DDEV;
constexpr int kVHDevPB = kVHDevPW + DDEV * DE;
constexpr int kVHDecB0 = kVHDevPB + DE;
constexpr int kVHDecB1 = kVHDecB0 + DEC;
constexpr int kVHOutW = kVHDecB1 + DEC;
constexpr int kVHOutB = kVHOutW + DEC;
constexpr int kVecFloats = kVHead + kVHOutB + 4;
constexpr int kSmTotal = kSmVec + kVecFloats * 4;
static_assert(kSmTotal <= 227 * 1024 - 2560, "forward_f32 shared memory (+ 2.1 KB static)");
static_assert(kMaxLeaf * D * DE * 4 / 2 <= TR * LDK * 4, "leaf_embed group must fit");

__device__ __forceinline__ void fence_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// acc[j] += Σ_{k<K} x[k] · W[k·ldw + j], j < NJ — x: this row (smem, 16-B
// aligned), W: a warp-uniform smem tile (every lane reads the same float4)
template <int NJ, int K>
__device__ __forceinline__ void row_mm(float* acc, const float* x, const float* W, int ldw) {
#pragma unroll 2
  for (int k = 0; k < K; k += 4) {
    const float4 x4 = *reinterpret_cast<const float4*>(x + k);
    const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const float* wr = W + (k + kk) * ldw;
#pragma unroll
      for (int j = 0; j < NJ; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(wr + j);
        acc[j] = fmaf(xs[kk], w4.x, acc[j]);
        acc[j + 1] = fmaf(xs[kk], w4.y, acc[j + 1]);
        acc[j + 2] = fmaf(xs[kk], w4.z, acc[j + 2]);
        acc[j + 3] = fmaf(xs[kk], w4.w, acc[j + 3]);
      }
    }
  }
}

// two-row register blocking: acc0/acc1 (rows x0/x1) share every weight
// float4, halving the shared-memory loads per FFMA of row_mm
template <int NJ, int K>
__device__ __forceinline__ void row_mm2(float* acc0, float* acc1, const float* x0, const float* x1,
                                        const float* W, int ldw) {
#pragma unroll 2
  for (int k = 0; k < K; k += 4) {
    const float4 a4 = *reinterpret_cast<const float4*>(x0 + k);
    const float4 b4 = *reinterpret_cast<const float4*>(x1 + k);
    const float as[4] = {a4.x, a4.y, a4.z, a4.w}, bs[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const float* wr = W + (k + kk) * ldw;
#pragma unroll
      for (int j = 0; j < NJ; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(wr + j);
        acc0[j] = fmaf(as[kk], w4.x, acc0[j]);
        acc0[j + 1] = fmaf(as[kk], w4.y, acc0[j + 1]);
        acc0[j + 2] = fmaf(as[kk], w4.z, acc0[j + 2]);
        acc0[j + 3] = fmaf(as[kk], w4.w, acc0[j + 3]);
        acc1[j] = fmaf(bs[kk], w4.x, acc1[j]);
        acc1[j + 1] = fmaf(bs[kk], w4.y, acc1[j + 1]);
        acc1[j + 2] = fmaf(bs[kk], w4.z, acc1[j + 2]);
        acc1[j + 3] = fmaf(bs[kk], w4.w, acc1[j + 3]);
      }
    }
  }
}

__device__ __forceinline__ void st_row(float* dst, const float* v, int n) {
  for (int j = 0; j < n; j += 4)
    *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
}

// two-pass LayerNorm of a row split over (r, wg = 0/1), 32 columns each
// (nn.py:48-54, eps 1e-5, biased variance); red: [4][TR]
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

__device__ __forceinline__ double boxcox_decode_f32(double e, const tpcb_boxcox& bc, bool* bad) {
  const double t = e * bc.t_std + bc.t_mean;
  if (fabs(bc.lambda_bc) < 1e-9) return exp(t) - bc.shift;
  const double base = bc.lambda_bc * t + 1.0;
  if (!(base > 0.0)) {
    *bad = true;
    return nan("");
  }
  return pow(base, 1.0 / bc.lambda_bc) - bc.shift;
}

__device__ long long* g_trace_f32 = nullptr;
#define FT32(id)                                                                 \
  do {                                                                           \
    if (g_trace_f32 && blockIdx.x == 0 && t == 0)                                \
      g_trace_f32[(tcount & 7) * 32 + (id)] = clock64();                         \
  } while (0)

// attention of one query row over its AST's LL keys (fp32 K|V rows, head
// columns DH·wg ..), LL a compile-time count: every score first
// (independent dot products), then the weights and the context
template <int LL>
__device__ __forceinline__ void attn_f32_fixed(const float* __restrict__ sKV, int r0, int wg,
                                               const float* q, float scale, float* c) {
  float sc[LL];
#pragma unroll
  for (int jj = 0; jj < LL; ++jj) {
    const float* kr = sKV + (r0 + jj) * LDK + DH * wg;
    float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < DH; i += 4) {
      const float4 k4 = *reinterpret_cast<const float4*>(kr + i);
      a4[0] = fmaf(q[i], k4.x, a4[0]);
      a4[1] = fmaf(q[i + 1], k4.y, a4[1]);
      a4[2] = fmaf(q[i + 2], k4.z, a4[2]);
      a4[3] = fmaf(q[i + 3], k4.w, a4[3]);
    }
    sc[jj] = ((a4[0] + a4[1]) + (a4[2] + a4[3])) * scale;
  }
  float m = sc[0];
#pragma unroll
  for (int jj = 1; jj < LL; ++jj) m = fmaxf(m, sc[jj]);
  float sum = 0.f;
#pragma unroll
  for (int jj = 0; jj < LL; ++jj) {
    const float pj = LL == 1 ? 1.f : expf(sc[jj] - m);
    sum += pj;
    const float* vr = sKV + (r0 + jj) * LDK + D + DH * wg;
#pragma unroll
    for (int i = 0; i < DH; i += 4) {
      const float4 v4 = *reinterpret_cast<const float4*>(vr + i);
      c[i] = fmaf(pj, v4.x, c[i]);
      c[i + 1] = fmaf(pj, v4.y, c[i + 1]);
      c[i + 2] = fmaf(pj, v4.z, c[i + 2]);
      c[i + 3] = fmaf(pj, v4.w, c[i + 3]);
    }
  }
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < DH; ++i) c[i] *= inv;
}

__global__ void __launch_bounds__(NTH, 1) forward_f32_kernel(
    const __grid_constant__ Model M, const float* __restrict__ P, const float* __restrict__ x,
    const int32_t* __restrict__ tile_L, const int32_t* __restrict__ tile_first,
    const int32_t* __restrict__ tile_count, const int32_t* __restrict__ n_tiles_p,
    const int32_t* __restrict__ perm, const float* __restrict__ devfeat, tpcb_boxcox bc,
    float* __restrict__ pred_out, float* __restrict__ zx_out, float* __restrict__ zv_out,
    float* __restrict__ z_out, double* __restrict__ lat_out, int32_t* status) {
  extern __shared__ __align__(1024) uint8_t smb[];
  __shared__ __align__(8) uint64_t bars[6];  // [0..3] ring slots, [4] resident, [5] leaf stage
  __shared__ float s_red[4 * TR];
  const int t = threadIdx.x, wg = t >> 7, r = t & (TR - 1);
  const int n_tiles = *n_tiles_p;
  float* ring = reinterpret_cast<float*>(smb + kRing);
  float* sA = reinterpret_cast<float*>(smb + kSmA);
  float* sKV = reinterpret_cast<float*>(smb + kSmKV);
  float* sRes = reinterpret_cast<float*>(smb + kSmRes);
  float* sZx = reinterpret_cast<float*>(smb + kSmZx);
  float* sv = reinterpret_cast<float*>(smb + kSmVec);
  const float* hv = sv + kVHead;
  if (t == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // ring: slot s's k-th fill is waited with parity k & 1 (every thread waits
  // every fill once, in the same order)
  uint32_t par = 0, leaf_par = 0;
  auto slot = [&](int s) { return ring + s * (kSlotB / 4); };
  auto fill = [&](int s, const float* src, uint32_t bytes) {  // thread 0 only
    mbar_arrive_expect_tx(&bars[s], bytes);
    bulk_g2s(slot(s), src, bytes, &bars[s]);
  };
  auto wait_slot = [&](int s) {
    mbar_wait(&bars[s], (par >> s) & 1u);
    par ^= 1u << s;
  };
  // layer li's first four tiles (Wq Wk Wv Wo → slots 0..3)
  auto fill_qkvo = [&](int li, int from_slot) {
    const LayerOff& lo = M.layer[li];
    const int off[4] = {lo.Wq, lo.Wk, lo.Wv, lo.Wo};
    for (int s = from_slot; s < from_slot + 2; ++s) fill(s, P + off[s], kSlotB);
  };

  if (t == 0 && blockIdx.x < n_tiles) {
    fill_qkvo(0, 0);
    fill_qkvo(0, 2);
    mbar_arrive_expect_tx(&bars[4], kResFloats * 4);
    bulk_g2s(sRes + kResIn, P + M.inW, TPCB_FEAT * D * 4, &bars[4]);
    bulk_g2s(sRes + kResDec0, P + M.decW[0], DE * DEC * 4, &bars[4]);
    bulk_g2s(sRes + kResDec1, P + M.decW[1], DEC * DEC * 4, &bars[4]);
  }
  // biases / LayerNorm / head vectors
  for (int i = t; i < D; i += NTH) sv[kVIn + i] = __ldg(P + M.inb + i);
  for (int li = 0; li < NLAY; ++li) {
    const LayerOff& lo = M.layer[li];
    float* b = sv + kVLayer + li * kVLStride;
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
    float* h = sv + kVHead;
    for (int i = t; i < (kMaxLeaf + 1) * DE; i += NTH) {
      const int L = i / DE;
      h[kVHLeafB + i] = (L >= 1 && L <= M.n_leaf_max) ? __ldg(P + M.leafb[L] + (i - L * DE)) : 0.f;
    }
    for (int i = t; i < TPCB_DEV_FEAT * DDEV; i += NTH) h[kVHDevHW + i] = __ldg(P + M.devhW + i);
    for (int i = t; i < DDEV * DE; i += NTH) h[kVHDevPW + i] = __ldg(P + M.devpW + i);
    for (int i = t; i < DDEV; i += NTH) h[kVHDevHB + i] = __ldg(P + M.devhb + i);
    for (int i = t; i < DE; i += NTH) h[kVHDevPB + i] = __ldg(P + M.devpb + i);
    for (int i = t; i < DEC; i += NTH) {
      h[kVHDecB0 + i] = __ldg(P + M.decb[0] + i);
      h[kVHDecB1 + i] = __ldg(P + M.decb[1] + i);
      h[kVHOutW + i] = __ldg(P + M.outW + i);
    }
    if (t == 0) h[kVHOutB] = __ldg(P + M.outb);
  }
  __syncthreads();
  if (blockIdx.x < n_tiles) mbar_wait(&bars[4], 0);
  const float scale = 1.f / sqrtf((float)DH);

  // warpgroup 1 prefetches the next tile's input rows into registers
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

  int tcount = -1;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    ++tcount;
    FT32(0);
    const int L = tile_L[tile], first = tile_first[tile], A = tile_count[tile];
    const bool live = r < A * L;
    const bool has_next = tile + (int)gridDim.x < n_tiles;
    float* xrow = sA + r * LDA;
    if (wg == 1) {
#pragma unroll
      for (int i = 0; i < TPCB_FEAT; i += 4)
        *reinterpret_cast<float4*>(xrow + i) =
            live ? make_float4(xn[i], xn[i + 1], xn[i + 2], xn[i + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    float h[DH];  // residual stream, columns 32·wg .. 32·wg+31
#pragma unroll
    for (int j = 0; j < DH; ++j) h[j] = sv[kVIn + DH * wg + j];
    row_mm<DH, TPCB_FEAT>(h, xrow, sRes + kResIn + DH * wg, D);
    __syncthreads();
    st_row(xrow + DH * wg, h, DH);
    __syncthreads();
    FT32(1);

    for (int li = 0; li < NLAY; ++li) {
      const float* b = sv + kVLayer + li * kVLStride;
      const LayerOff& lo = M.layer[li];
      // ---- Q, K, V: thread (row pair p, p + 64; column quarter cq) — K, V
      // rows to the K|V region, Q rows (after every thread has read the h
      // rows) over the h rows; the attention threads (r, head) read them back
      wait_slot(0);
      wait_slot(1);
      wait_slot(2);
      const int p = t & 63, cq = t >> 6;
      const float* x0 = sA + p * LDA;
      const float* x1 = sA + (p + 64) * LDA;
      constexpr int QC = D / 4;  // 16 columns per quarter
      {
        float k0[QC], k1[QC];
#pragma unroll
        for (int part = 0; part < 2; ++part) {
#pragma unroll
          for (int j = 0; j < QC; ++j) k0[j] = k1[j] = b[kVBQKV + (1 + part) * D + QC * cq + j];
          row_mm2<QC, D>(k0, k1, x0, x1, slot(1 + part) + QC * cq, D);
          st_row(sKV + p * LDK + part * D + QC * cq, k0, QC);
          st_row(sKV + (p + 64) * LDK + part * D + QC * cq, k1, QC);
        }
      }
      {
        float q0[QC], q1[QC];
#pragma unroll
        for (int j = 0; j < QC; ++j) q0[j] = q1[j] = b[kVBQKV + QC * cq + j];
        row_mm2<QC, D>(q0, q1, x0, x1, slot(0) + QC * cq, D);
        fence_async();
        __syncthreads();  // every h row read: Q overwrites them; slots 0..2 free
        st_row(sA + p * LDA + QC * cq, q0, QC);
        st_row(sA + (p + 64) * LDA + QC * cq, q1, QC);
      }
      if (t == 0) {  // fhW → slots 0-1, foW rows 0..63 → slot 2
        fill(0, P + lo.fhW, kSlotB);
        fill(1, P + lo.fhW + 64 * 64, kSlotB);
        fill(2, P + lo.foW, kSlotB);
      }
      __syncthreads();
      float q[DH];
#pragma unroll
      for (int j = 0; j < DH; j += 4) {
        const float4 v4 = *reinterpret_cast<const float4*>(xrow + DH * wg + j);
        q[j] = v4.x; q[j + 1] = v4.y; q[j + 2] = v4.z; q[j + 3] = v4.w;
      }
      FT32(2 + 6 * li);
      // ---- attention of row r over its AST's L keys, head wg (nn.py:79-96)
      float c[DH];
#pragma unroll
      for (int j = 0; j < DH; ++j) c[j] = 0.f;
      if (live && L <= 6) {  // the common small leaf counts: unrolled per L
        const int r0 = (r / L) * L;
        switch (L) {
          case 1: attn_f32_fixed<1>(sKV, r0, wg, q, scale, c); break;
          case 2: attn_f32_fixed<2>(sKV, r0, wg, q, scale, c); break;
          case 3: attn_f32_fixed<3>(sKV, r0, wg, q, scale, c); break;
          case 4: attn_f32_fixed<4>(sKV, r0, wg, q, scale, c); break;
          case 5: attn_f32_fixed<5>(sKV, r0, wg, q, scale, c); break;
          default: attn_f32_fixed<6>(sKV, r0, wg, q, scale, c); break;
        }
      } else if (live) {
        // one pass over the keys with a running max (no score array, so no
        // stack frame): the context is rescaled only when the max grows
        const int r0 = (r / L) * L;
        float m = -INFINITY, sum = 0.f;
        for (int jj = 0; jj < L; ++jj) {
          const float* kr = sKV + (r0 + jj) * LDK + DH * wg;
          const float* vr = sKV + (r0 + jj) * LDK + D + DH * wg;
          float a4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < DH; i += 4) {
            const float4 k4 = *reinterpret_cast<const float4*>(kr + i);
            a4[0] = fmaf(q[i], k4.x, a4[0]);
            a4[1] = fmaf(q[i + 1], k4.y, a4[1]);
            a4[2] = fmaf(q[i + 2], k4.z, a4[2]);
            a4[3] = fmaf(q[i + 3], k4.w, a4[3]);
          }
          const float sj = ((a4[0] + a4[1]) + (a4[2] + a4[3])) * scale;
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
          for (int i = 0; i < DH; i += 4) {
            const float4 v4 = *reinterpret_cast<const float4*>(vr + i);
            c[i] = fmaf(pj, v4.x, c[i]);
            c[i + 1] = fmaf(pj, v4.y, c[i + 1]);
            c[i + 2] = fmaf(pj, v4.z, c[i + 2]);
            c[i + 3] = fmaf(pj, v4.w, c[i + 3]);
          }
        }
        const float inv = 1.f / sum;
#pragma unroll
        for (int i = 0; i < DH; ++i) c[i] *= inv;
      }
      st_row(xrow + DH * wg, c, DH);  // the QKV products are done with the h rows
      __syncthreads();
      FT32(3 + 6 * li);
      // ---- output projection + residual + LayerNorm 1
      // (product by row pairs into the dead K|V rows, epilogue by (r, wg))
      wait_slot(3);
      {
        float o0[QC], o1[QC];
#pragma unroll
        for (int j = 0; j < QC; ++j) o0[j] = o1[j] = b[kVBO + QC * cq + j];
        row_mm2<QC, D>(o0, o1, x0, x1, slot(3) + QC * cq, D);
        st_row(sKV + p * LDK + QC * cq, o0, QC);
        st_row(sKV + (p + 64) * LDK + QC * cq, o1, QC);
      }
      fence_async();
      __syncthreads();  // Wo reads done, output rows complete
      if (t == 0) fill(3, P + lo.foW + 64 * 64, kSlotB);  // foW rows 64..127
      float h1[DH];
#pragma unroll
      for (int j = 0; j < DH; j += 4) {
        const float4 v4 = *reinterpret_cast<const float4*>(sKV + r * LDK + DH * wg + j);
        h1[j] = v4.x + h[j]; h1[j + 1] = v4.y + h[j + 1];
        h1[j + 2] = v4.z + h[j + 2]; h1[j + 3] = v4.w + h[j + 3];
      }
      ln_half(h1, b + kVLN1G, b + kVLN1B, wg, r, s_red);
      st_row(xrow + DH * wg, h1, DH);
      __syncthreads();
      FT32(4 + 6 * li);
      // ---- FFN hidden relu(h1·fhW + b): thread (rows p, p + 64; columns
      // 32·cq .. 32·cq+31)
      wait_slot(0);
      wait_slot(1);
      {
        constexpr int FC = FF / 4;
        float f0[FC], f1[FC];
#pragma unroll
        for (int j = 0; j < FC; ++j) f0[j] = f1[j] = b[kVFHB + FC * cq + j];
        row_mm2<FC, D>(f0, f1, x0, x1, slot(0) + FC * cq, FF);
#pragma unroll
        for (int j = 0; j < FC; ++j) {
          f0[j] = fmaxf(f0[j], 0.f);
          f1[j] = fmaxf(f1[j], 0.f);
        }
        st_row(sKV + p * LDK + FC * cq, f0, FC);
        st_row(sKV + (p + 64) * LDK + FC * cq, f1, FC);
      }
      if (wg == 1 && li + 1 == NLAY) load_x(tile + gridDim.x);
      fence_async();
      __syncthreads();
      if (t == 0) {  // next layer's (or next tile's layer 0) Wq, Wk → slots 0, 1
        if (li + 1 < NLAY) fill_qkvo(li + 1, 0);
        else if (has_next) fill_qkvo(0, 0);
      }
      FT32(5 + 6 * li);
      // ---- FFN out + residual + LayerNorm 2
      // (product by row pairs into the dead h1 rows, epilogue by (r, wg))
      wait_slot(2);
      wait_slot(3);
      {
        float o0[QC], o1[QC];
#pragma unroll
        for (int j = 0; j < QC; ++j) o0[j] = o1[j] = b[kVFOB + QC * cq + j];
        row_mm2<QC, FF>(o0, o1, sKV + p * LDK, sKV + (p + 64) * LDK, slot(2) + QC * cq, D);
        st_row(sA + p * LDA + QC * cq, o0, QC);
        st_row(sA + (p + 64) * LDA + QC * cq, o1, QC);
      }
      fence_async();
      __syncthreads();  // F / foW reads done, output rows complete
      if (t == 0) {  // Wv, Wo → slots 2, 3
        if (li + 1 < NLAY) fill_qkvo(li + 1, 2);
        else if (has_next) fill_qkvo(0, 2);
        if (li + 1 == NLAY) {  // K|V region now dead: stage leaf_embed.L group 0
          const uint32_t b0 = (uint32_t)(min(8, L) * D * DE * 4);  // under LN2
          mbar_arrive_expect_tx(&bars[5], b0);
          bulk_g2s(sKV, P + M.leafW[L], b0, &bars[5]);
        }
      }
#pragma unroll
      for (int j = 0; j < DH; j += 4) {
        const float4 v4 = *reinterpret_cast<const float4*>(xrow + DH * wg + j);
        h[j] = v4.x + h1[j]; h[j + 1] = v4.y + h1[j + 1];
        h[j + 2] = v4.z + h1[j + 2]; h[j + 3] = v4.w + h1[j + 3];
      }
      ln_half(h, b + kVLN2G, b + kVLN2B, wg, r, s_red);
      st_row(xrow + DH * wg, h, DH);
      __syncthreads();
      FT32(6 + 6 * li);
    }

    // ---------------------------------------------------------------- head
    // z_x[a] = b_L + Σ_l h[a·L + l] · W_L[l] (costmodel.py:213-216): jobs
    // (AST a, 4-column group), leaf_embed.L staged in the dead K|V region in
    // groups of ≤ 8 leaf positions (l-ordered single-chain sums)
    const float* WL = P + M.leafW[L];
    // jobs (AST a, 4-column group, leaf position l) write partial rows l·A + a
    // of sZx; the partials are then summed in l order (batch-invariant)
    for (int g0 = 0; g0 < L; g0 += 8) {
      const int gl = min(8, L - g0);
      if (t == 0 && g0 > 0) {  // group 0 was issued after the last FFN out
        mbar_arrive_expect_tx(&bars[5], (uint32_t)(gl * D * DE * 4));
        bulk_g2s(sKV, WL + (size_t)g0 * D * DE, (uint32_t)(gl * D * DE * 4), &bars[5]);
      }
      mbar_wait(&bars[5], leaf_par);
      leaf_par ^= 1u;
      for (int job = t; job < A * gl * (DE / 4); job += NTH) {
        const int cg = job & 7, rest = job >> 3, a = rest % A, l = rest / A;
        const float* hr = sA + (a * L + g0 + l) * LDA;
        const float* w = sKV + l * D * DE + 4 * cg;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int k = 0; k < D; k += 4) {
          const float4 h4 = *reinterpret_cast<const float4*>(hr + k);
          const float hs[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float4 w4 = *reinterpret_cast<const float4*>(w + (k + kk) * DE);
            acc.x = fmaf(hs[kk], w4.x, acc.x);
            acc.y = fmaf(hs[kk], w4.y, acc.y);
            acc.z = fmaf(hs[kk], w4.z, acc.z);
            acc.w = fmaf(hs[kk], w4.w, acc.w);
          }
        }
        *reinterpret_cast<float4*>(sZx + ((g0 + l) * A + a) * LDZ + 4 * cg) = acc;
      }
      fence_async();
      __syncthreads();
    }
    for (int idx = t; idx < A * DE; idx += NTH) {  // row a = b_L + Σ_l partial(l, a), in place
      const int a = idx / DE, n = idx - a * DE;
      float v = hv[kVHLeafB + L * DE + n];
      for (int l = 0; l < L; ++l) v += sZx[(l * A + a) * LDZ + n];
      sZx[a * LDZ + n] = v;
    }
    __syncthreads();
    FT32(20);
    // device MLP, gate, decoder: thread (AST a = r, column half wg)
    float* sU = sKV;  // decoder hidden rows [128][LDK]
    const bool ast = r < A;
    if (ast) {  // gate half: columns 16·wg .. 16·wg+15 of z = z_x ⊙ proj(relu(hidden(v)))
      constexpr int HZ = DE / 2;
      const int idx = perm[first + r];
      float dv[TPCB_DEV_FEAT], zv[DDEV], zp[HZ];
#pragma unroll
      for (int f = 0; f < TPCB_DEV_FEAT; ++f) dv[f] = __ldg(devfeat + (size_t)idx * TPCB_DEV_FEAT + f);
#pragma unroll
      for (int n = 0; n < DDEV; ++n) zv[n] = hv[kVHDevHB + n];
#pragma unroll
      for (int f = 0; f < TPCB_DEV_FEAT; ++f)
#pragma unroll
        for (int n = 0; n < DDEV; n += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(hv + kVHDevHW + f * DDEV + n);
          zv[n] = fmaf(dv[f], w4.x, zv[n]);
          zv[n + 1] = fmaf(dv[f], w4.y, zv[n + 1]);
          zv[n + 2] = fmaf(dv[f], w4.z, zv[n + 2]);
          zv[n + 3] = fmaf(dv[f], w4.w, zv[n + 3]);
        }
#pragma unroll
      for (int n = 0; n < DDEV; ++n) zv[n] = fmaxf(zv[n], 0.f);
#pragma unroll
      for (int n = 0; n < HZ; ++n) zp[n] = hv[kVHDevPB + HZ * wg + n];
#pragma unroll
      for (int k = 0; k < DDEV; ++k)
#pragma unroll
        for (int n = 0; n < HZ; n += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(hv + kVHDevPW + k * DE + HZ * wg + n);
          zp[n] = fmaf(zv[k], w4.x, zp[n]);
          zp[n + 1] = fmaf(zv[k], w4.y, zp[n + 1]);
          zp[n + 2] = fmaf(zv[k], w4.z, zp[n + 2]);
          zp[n + 3] = fmaf(zv[k], w4.w, zp[n + 3]);
        }
      float* zr = sZx + r * LDZ + HZ * wg;  // this half's z_x → z in place
      float zx[HZ];
#pragma unroll
      for (int n = 0; n < HZ; ++n) {
        zx[n] = zr[n];
        zp[n] *= zx[n];
      }
      if (zx_out)
        for (int n = 0; n < HZ; ++n) zx_out[(size_t)idx * DE + HZ * wg + n] = zx[n];
      if (z_out)
        for (int n = 0; n < HZ; ++n) z_out[(size_t)idx * DE + HZ * wg + n] = zp[n];
      if (zv_out && wg == 0)
        for (int n = 0; n < DDEV; ++n) zv_out[(size_t)idx * DDEV + n] = zv[n];
      st_row(zr, zp, HZ);
    }
    __syncthreads();  // z rows complete: the first decoder product's input
    // decoder (costmodel.py:221-229): jobs (AST a, 4-column group) over all
    // 256 threads; hidden rows in the K|V region
    for (int job = t; job < A * (DEC / 4); job += NTH) {
      const int a = job >> 4, cg = job & 15;
      const float* zr = sZx + a * LDZ;
      const float* w = sRes + kResDec0 + 4 * cg;
      float4 acc = *reinterpret_cast<const float4*>(hv + kVHDecB0 + 4 * cg);
#pragma unroll 8
      for (int k = 0; k < DE; ++k) {
        const float zk = zr[k];
        const float4 w4 = *reinterpret_cast<const float4*>(w + k * DEC);
        acc.x = fmaf(zk, w4.x, acc.x);
        acc.y = fmaf(zk, w4.y, acc.y);
        acc.z = fmaf(zk, w4.z, acc.z);
        acc.w = fmaf(zk, w4.w, acc.w);
      }
      *reinterpret_cast<float4*>(sU + a * LDK + 4 * cg) =
          make_float4(fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f), fmaxf(acc.z, 0.f), fmaxf(acc.w, 0.f));
    }
    __syncthreads();
    for (int job = t; job < A * (DEC / 4); job += NTH) {
      const int a = job >> 4, cg = job & 15;
      const float* ur = sU + a * LDK;
      const float* w = sRes + kResDec1 + 4 * cg;
      float4 acc = *reinterpret_cast<const float4*>(hv + kVHDecB1 + 4 * cg);
#pragma unroll 8
      for (int k = 0; k < DEC; ++k) {
        const float uk = ur[k];
        const float4 w4 = *reinterpret_cast<const float4*>(w + k * DEC);
        acc.x = fmaf(uk, w4.x, acc.x);
        acc.y = fmaf(uk, w4.y, acc.y);
        acc.z = fmaf(uk, w4.z, acc.z);
        acc.w = fmaf(uk, w4.w, acc.w);
      }
      *reinterpret_cast<float4*>(sU + a * LDK + DEC + 4 * cg) =
          make_float4(fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f), fmaxf(acc.z, 0.f), fmaxf(acc.w, 0.f));
    }
    __syncthreads();
    if (t < A) {
      float pred = hv[kVHOutB];
      const float* ur = sU + t * LDK + DEC;
#pragma unroll 8
      for (int j = 0; j < DEC; ++j) pred = fmaf(ur[j], hv[kVHOutW + j], pred);
      const int idx = perm[first + t];
      pred_out[idx] = pred;
      if (lat_out) {
        bool bad = false;
        lat_out[idx] = bc.enabled ? boxcox_decode_f32((double)pred, bc, &bad) : (double)pred;
        if (bad) raise_status(status, TPCB_ERR_DOMAIN);
      }
    }
    FT32(21);
    fence_async();
    __syncthreads();  // K|V region (decoder rows) and z_x rows are rewritten by the next tile
  }
}

}  // namespace

bool f32_fast_supported(const Model& M) {
  if (M.d != D || M.n_layers != NLAY || M.n_heads != 2 || M.dh != DH || M.d_ff != FF) return false;
  if (M.d_e != DE || M.d_dev != DDEV || M.n_dec != 2 || M.dec[0] != DEC || M.dec[1] != DEC)
    return false;
  return M.n_leaf_max <= kMaxLeaf;
}

int set_forward_f32_trace(long long* d) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace_f32, &d, sizeof(d)));
  return TPCB_OK;
}

int launch_forward_f32(const Model& M, const float* d_params, const tpcb_packed* pk,
                       const float* d_devfeat, const tpcb_boxcox* norm, float* d_pred,
                       float* d_zx, float* d_zv, float* d_z, double* d_latency, int32_t* d_status,
                       cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(forward_f32_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmTotal));
    attr = true;
  }
  tpcb_boxcox bc{};
  if (norm) bc = *norm;
  const int grid = (int)std::min<int64_t>(pk->n_tiles_max, (int64_t)kNumSMs);
  forward_f32_kernel<<<grid, NTH, kSmTotal, stream>>>(
      M, d_params, pk->x, pk->tile_L, pk->tile_first, pk->tile_count, pk->n_tiles, pk->perm,
      d_devfeat, bc, d_pred, d_zx, d_zv, d_z, d_latency, d_status);
  TPCB_LAUNCH_CHECK("forward_f32_kernel");
  return TPCB_OK;
}

}  // namespace tpcb
