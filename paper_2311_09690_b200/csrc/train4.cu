// Training step, v4: the desk-shaped fast path (d_model 64, 2 heads, d_ff
// 128, d_embed 32, d_device 16, decoder (64, 64), ≤ 16 leaves — the shape
// BASELINE.json's workload trains).
//
// Same arithmetic as train.cu / the oracle (reference: costmodel.backward,
// costmodel.py:529-570; nn.py:30-120), re-scheduled for instruction
// efficiency.  A training step is a chain of small dependent products per
// sample (≤ 16 rows), so the step time is the critical path of one sample,
// and that path is bounded by FFMA issue when (and only when) the code spends
// its instructions on FMAs.  Hence:
//   * one CTA per sample: 8 compute warps + 1 producer warp;
//   * the producer streams every weight tile the sample consumes, in order,
//     into a ring of NS shared-memory slots (cp.async.bulk + mbarriers:
//     full[s] counts transaction bytes, empty[s] counts the 8 compute warps);
//   * products are register-blocked: each thread owns one row × 4 columns,
//     activation float4 broadcast + 4 weight float4 per 16 FFMA, and the
//     transposed (backward) product reads the same row-major tile with a
//     strided column set (k = kb + 16j) so no transposed weight copy exists;
//   * LayerNorm forward/backward is fused into the epilogue of the product
//     that produces its input (16 threads per row, half-warp shuffles);
//   * attention runs a half-warp per (head, query row): scores, softmax and
//     P·V without intermediate barriers;
//   * weight gradients (X^T·dY, 4×4 register blocks over the rows) ride in
//     the phase after their operands are final, next to the critical product;
//   * biases / LayerNorm vectors / the device MLP live in shared memory.
// Gradients go to the CTA's slot exactly as in v2 (optim.cu reduces the
// slots in fixed order: deterministic).
#include <cuda.h>

#include <cmath>
#include <cstring>

#include "async.cuh"
#include "cmd.cuh"
#include "common.cuh"
#include "train.cuh"

namespace tpcb {

__device__ long long* g_trace4 = nullptr;

int set_train4_trace(long long* d) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace4, &d, sizeof(d)));
  return TPCB_OK;
}

namespace {

// ---- the one shape this kernel is written for --------------------------
constexpr int D = 64, NHEAD = 2, DHEAD = 32, FF = 128, DE = 32, DDEV = 16, NLAY = 2, DEC = 64;
constexpr int FEAT = TPCB_FEAT, DEVF = TPCB_DEV_FEAT;
constexpr int RMAX = 16;

constexpr int NW = 8;              // compute warps
constexpr int NT = NW * 32;        // compute threads
constexpr int kThreads4 = NT + 64; // + producer warp + stage publisher warp
constexpr int kBar = 1;            // named barrier of the compute warps
constexpr int kStages4 = 2 + 2 * NLAY;  // backward stages published to the overlapped reduce

constexpr int LDH = 68;   // 64-wide activation rows
constexpr int LDQ = 196;  // Q|K|V rows
constexpr int LDF = 132;  // FFN hidden rows
constexpr int LDX = TPCB_FEAT_PAD;  // input feature rows (packed rows, bulk-copied)
// A ring slot holds one 64-column weight tile as two TMA boxes of 32 columns
// × `rows` rows, dense, 128-byte swizzled (16-byte chunk c of row k sits at
// chunk c ^ (k & 7)), or two unswizzled leaf_embed tiles [64 × 32].
constexpr int kSlot = 64 * 64;     // floats per ring slot (16 KB, 1024-B aligned)
constexpr int kLeafTile = D * DE;  // leaf_embed tile (2 per slot)
constexpr int kMaps = 1 + 6 * NLAY + 2;  // inW, per layer Wq Wk Wv Wo fhW foW, dec0W, dec1W

// small-vector area (floats)
constexpr int SV_INB = 0;
constexpr int SV_LAYER = 64;  // + li * SV_LSTRIDE
constexpr int SV_BQKV = 0, SV_BO = 192, SV_LN1G = 256, SV_LN1B = 320, SV_FHB = 384, SV_FOB = 512,
              SV_LN2G = 576, SV_LN2B = 640, SV_LSTRIDE = 704;
constexpr int SV_LEAFB = SV_LAYER + NLAY * SV_LSTRIDE;
constexpr int SV_DEVHW = SV_LEAFB + DE;
constexpr int SV_DEVHB = SV_DEVHW + DEVF * DDEV;
constexpr int SV_DEVPW = SV_DEVHB + DDEV;
constexpr int SV_DEVPB = SV_DEVPW + DDEV * DE;
constexpr int SV_DECB0 = SV_DEVPB + DE;
constexpr int SV_DECB1 = SV_DECB0 + DEC;
constexpr int SV_OUTW = SV_DECB1 + DEC;
constexpr int SV_OUTB = SV_OUTW + DEC;
constexpr int SV_TOTAL = SV_OUTB + 4;

__device__ __forceinline__ void cbar() { group_bar(kBar, NT); }
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float hsum16(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}
__device__ __forceinline__ float hmax16(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return v;
}

// element (k, n) of a swizzled tile with `rows` rows
__device__ __forceinline__ int swz(int rows, int k, int n) {
  return (n >> 5) * rows * 32 + k * 32 + ((((n >> 2) & 7) ^ (k & 7)) << 2) + (n & 3);
}

// acc[i] + Σ_{k<K} a[k]·W[k][c + i], i = 0..3 (W swizzled, `rows` rows, c % 4 == 0).
// Eight per-thread chunk bases (the swizzle of row k depends only on k & 7).
template <int K>
__device__ __forceinline__ float4 mm_fwd(float4 acc, const float* __restrict__ a,
                                         const float* __restrict__ W, int rows, int c) {
  const float* wb = W + (c >> 5) * rows * 32;
  const int ch = (c >> 2) & 7;
  const float* b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) b[j] = wb + ((ch ^ j) << 2);
#pragma unroll 2
  for (int k = 0; k < K; k += 8) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 x = ld4(a + k + 4 * h);
      const float4 w0 = ld4(b[4 * h + 0] + (k + 4 * h + 0) * 32);
      const float4 w1 = ld4(b[4 * h + 1] + (k + 4 * h + 1) * 32);
      const float4 w2 = ld4(b[4 * h + 2] + (k + 4 * h + 2) * 32);
      const float4 w3 = ld4(b[4 * h + 3] + (k + 4 * h + 3) * 32);
      acc.x = fmaf(x.x, w0.x, acc.x); acc.y = fmaf(x.x, w0.y, acc.y);
      acc.z = fmaf(x.x, w0.z, acc.z); acc.w = fmaf(x.x, w0.w, acc.w);
      acc.x = fmaf(x.y, w1.x, acc.x); acc.y = fmaf(x.y, w1.y, acc.y);
      acc.z = fmaf(x.y, w1.z, acc.z); acc.w = fmaf(x.y, w1.w, acc.w);
      acc.x = fmaf(x.z, w2.x, acc.x); acc.y = fmaf(x.z, w2.y, acc.y);
      acc.z = fmaf(x.z, w2.z, acc.z); acc.w = fmaf(x.z, w2.w, acc.w);
      acc.x = fmaf(x.w, w3.x, acc.x); acc.y = fmaf(x.w, w3.y, acc.y);
      acc.z = fmaf(x.w, w3.z, acc.z); acc.w = fmaf(x.w, w3.w, acc.w);
    }
  }
  return acc;
}

// acc[j] + Σ_{n<64} a[n]·W[kb + 16j][n], j = 0..3 (W swizzled, 64 rows): the
// transposed product out[k] = Σ_n a[n]·W[k][n] for k = kb + 16j.  Rows
// kb + 16j share (k & 7), so one set of 8 chunk bases serves all four.
__device__ __forceinline__ float4 mm_bwd(float4 acc, const float* __restrict__ a,
                                         const float* __restrict__ W, int kb) {
  const int xr = kb & 7;
  const float* b[8];
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) b[cc] = W + kb * 32 + ((cc ^ xr) << 2);
#pragma unroll
  for (int box = 0; box < 2; ++box) {
#pragma unroll 4
    for (int cc = 0; cc < 8; ++cc) {
      const float4 x = ld4(a + box * 32 + cc * 4);
      const float* p = b[cc] + box * 64 * 32;
      const float4 w0 = ld4(p), w1 = ld4(p + 16 * 32), w2 = ld4(p + 32 * 32), w3 = ld4(p + 48 * 32);
      acc.x = fmaf(x.x, w0.x, acc.x); acc.y = fmaf(x.x, w1.x, acc.y);
      acc.z = fmaf(x.x, w2.x, acc.z); acc.w = fmaf(x.x, w3.x, acc.w);
      acc.x = fmaf(x.y, w0.y, acc.x); acc.y = fmaf(x.y, w1.y, acc.y);
      acc.z = fmaf(x.y, w2.y, acc.z); acc.w = fmaf(x.y, w3.y, acc.w);
      acc.x = fmaf(x.z, w0.z, acc.x); acc.y = fmaf(x.z, w1.z, acc.y);
      acc.z = fmaf(x.z, w2.z, acc.z); acc.w = fmaf(x.z, w3.z, acc.w);
      acc.x = fmaf(x.w, w0.w, acc.x); acc.y = fmaf(x.w, w1.w, acc.y);
      acc.z = fmaf(x.w, w2.w, acc.z); acc.w = fmaf(x.w, w3.w, acc.w);
    }
  }
  return acc;
}

// LayerNorm over a 64-wide row held as 4 values by each of 16 threads
// (nn.py:48-54); returns xhat in v, writes nothing
__device__ __forceinline__ float ln_fwd4(float v[4]) {
  const float mu = hsum16(v[0] + v[1] + v[2] + v[3]) * (1.f / 64.f);
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float t = v[j] - mu;
    q = fmaf(t, t, q);
  }
  const float inv = 1.f / sqrtf(hsum16(q) * (1.f / 64.f) + 1e-5f);
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = (v[j] - mu) * inv;
  return inv;
}

// LayerNorm backward (nn.py:57-66) for 4 values of a row: dy·g = gx, xh at
// the same columns, inv of the row
__device__ __forceinline__ void ln_bwd4(float gx[4], const float xh[4], float inv) {
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    s1 += gx[j];
    s2 = fmaf(gx[j], xh[j], s2);
  }
  const float m1 = hsum16(s1) * (1.f / 64.f), m2 = hsum16(s2) * (1.f / 64.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) gx[j] = inv * (gx[j] - m1 - xh[j] * m2);
}

// ---- weight-gradient helpers (off the critical path, all compute threads) ----

// G[k·N + n] (+)= Σ_r X'[r][k]·dY[r][n] in 4×4 blocks, X' = X or g⊙X + b
__device__ __noinline__ void wgrad(const float* X, int ldx, const float* ga, const float* ba,
                                   const float* dY, int ldy, int L, int K, int N,
                                   float* __restrict__ G, bool first) {

  const int nb = N >> 2, n_items = (K >> 2) * nb;
  for (int it = threadIdx.x; it < n_items; it += NT) {
    const int kq = it / nb, k0 = kq * 4, n0 = (it - kq * nb) * 4;
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
    float4 g4 = make_float4(1.f, 1.f, 1.f, 1.f), b4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ga) {
      g4 = ld4(ga + k0);
      b4 = ld4(ba + k0);
    }
    for (int r = 0; r < L; ++r) {
      float4 x = ld4(X + r * ldx + k0);
      if (ga) {
        x.x = fmaf(g4.x, x.x, b4.x); x.y = fmaf(g4.y, x.y, b4.y);
        x.z = fmaf(g4.z, x.z, b4.z); x.w = fmaf(g4.w, x.w, b4.w);
      }
      const float4 y = ld4(dY + r * ldy + n0);
      a0.x = fmaf(x.x, y.x, a0.x); a0.y = fmaf(x.x, y.y, a0.y);
      a0.z = fmaf(x.x, y.z, a0.z); a0.w = fmaf(x.x, y.w, a0.w);
      a1.x = fmaf(x.y, y.x, a1.x); a1.y = fmaf(x.y, y.y, a1.y);
      a1.z = fmaf(x.y, y.z, a1.z); a1.w = fmaf(x.y, y.w, a1.w);
      a2.x = fmaf(x.z, y.x, a2.x); a2.y = fmaf(x.z, y.y, a2.y);
      a2.z = fmaf(x.z, y.z, a2.z); a2.w = fmaf(x.z, y.w, a2.w);
      a3.x = fmaf(x.w, y.x, a3.x); a3.y = fmaf(x.w, y.y, a3.y);
      a3.z = fmaf(x.w, y.z, a3.z); a3.w = fmaf(x.w, y.w, a3.w);
    }
    float* g = G + (size_t)k0 * N + n0;
    if (!first) {
      a0 = add4(a0, ld4(g));
      a1 = add4(a1, ld4(g + N));
      a2 = add4(a2, ld4(g + 2 * N));
      a3 = add4(a3, ld4(g + 3 * N));
    }
    st4(g, a0);
    st4(g + N, a1);
    st4(g + 2 * N, a2);
    st4(g + 3 * N, a3);
  }
}

// G[n] (+)= Σ_r dY[r][n] (· S[r][n]) on threads [t0, t0 + N)
__device__ __forceinline__ void colsum(const float* dY, int ldy, const float* S, int lds, int L,
                                       int N, float* __restrict__ G, bool first, int t0) {

  const int n = (int)threadIdx.x - t0;
  if (n < 0 || n >= N) return;
  float acc = 0.f;
  for (int r = 0; r < L; ++r) acc += S ? dY[r * ldy + n] * S[r * lds + n] : dY[r * ldy + n];
  G[n] = first ? acc : G[n] + acc;
}

// G[k·N + n] (+)= u[k]·v[n] (outer product, 4 columns per item)
__device__ __forceinline__ void outer(const float* u, int K, const float* v, int N,
                                      float* __restrict__ G, bool first) {

  const int nb = N >> 2;
  for (int it = threadIdx.x; it < K * nb; it += NT) {
    const int k = it / nb, n0 = (it - k * nb) * 4;
    const float a = u[k];
    const float4 y = ld4(v + n0);
    float4 r = make_float4(a * y.x, a * y.y, a * y.z, a * y.w);
    float* g = G + (size_t)k * N + n0;
    if (!first) r = add4(r, ld4(g));
    st4(g, r);
  }
}

// operand rows of an encoder weight product → the tensor-core weight-gradient
// buffer (train.cuh WgradDev): step rows w·Ls + r, r < L the rows of X (or
// g⊙X + b), L ≤ r < Ls zeros; `K` features (the operand's padded width)
__device__ __noinline__ void act_store(const WgradDev& wg, int op, const float* X, int ldx,
                                       const float* ga, const float* ba, int L, int Ls, int K,
                                       int w) {
  const int rows = wg_op_rows(op), off = wg_op_off(op);
  const int n = Ls * K;
  for (int e = threadIdx.x; e < n; e += NT) {
    const int f = e / Ls, r = e - f * Ls;
    float v = 0.f;
    if (r < L && f < ldx) {  // f ≥ ldx: the K padding of a narrower operand (X0)
      v = X[r * ldx + f];
      if (ga) v = fmaf(ga[f], v, ba[f]);
    }
    wg.act[wg_index(off, rows, wg.r_cap, f, w * Ls + r)] = v;
  }
}

// out[n] = act(bias[n] + Σ_k in[k]·W[k][n]) (W swizzled, K rows), 4 threads per output
__device__ __forceinline__ void gemv_f(const float* in, int K, const float* W, int N,
                                       const float* bias, bool relu, float* out) {

  const int t = threadIdx.x;
  if ((t & ~31) >= N * 4) return;
  const int n = t >> 2, q = t & 3;
  float s = 0.f;
  if (n < N)
    for (int k = q; k < K; k += 4) s = fmaf(in[k], W[swz(K, k, n)], s);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (q == 0 && n < N) {
    float v = s + bias[n];
    if (relu) v = fmaxf(v, 0.f);
    out[n] = v;
  }
}

// out[k] = mask(k) · Σ_n in[n]·W[k][n] (W swizzled, K rows), 4 threads per output
__device__ __forceinline__ void gemv_t(const float* in, int N, const float* W, int K,
                                       const float* mask_src, float* out) {

  const int t = threadIdx.x;
  if ((t & ~31) >= K * 4) return;
  const int k = t >> 2, q = t & 3;
  float s = 0.f;
  if (k < K)
    for (int n = q; n < N; n += 4) s = fmaf(in[n], W[swz(K, k, n)], s);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (q == 0 && k < K) out[k] = (mask_src && !(mask_src[k] > 0.f)) ? 0.f : s;
}

// ---- critical-path phases ------------------------------------------------

// QKV[r][64t + c] = bias + Hin[r]·W_t (t = q, k, v)
__device__ __noinline__ void op_qkv(int L, const float* Hin, const float* W0, const float* W1,
                                    const float* W2, const float* bias, float* QKV) {

  const int per = L * 16;
  for (int it = threadIdx.x; it < 3 * per; it += NT) {
    const int tt = it / per, rem = it - tt * per, r = rem >> 4, c = (rem & 15) * 4;
    const float* W = tt == 0 ? W0 : (tt == 1 ? W1 : W2);
    const float4 acc = mm_fwd<D>(make_float4(0.f, 0.f, 0.f, 0.f), Hin + r * LDH, W, 64, c);
    st4(QKV + r * LDQ + 64 * tt + c, add4(acc, ld4(bias + 64 * tt + c)));
  }
}

// half-warp per (head, query row): scores, softmax, P·V (nn.py:79-96)
__device__ __noinline__ void op_attn_fwd(int L, const float* QKV, float* P, float* C, float scale) {

  const int t = threadIdx.x, hw = t >> 4, j = t & 15;
  const bool jv = j < L;
  for (int p0 = 0; p0 < NHEAD * L; p0 += NT / 16) {
    if (p0 + (hw & ~1) >= NHEAD * L) break;  // whole warp idle (uniform per warp)
    const int pair = p0 + hw;
    const bool pv = pair < NHEAD * L;
    const int pp = pv ? pair : 0, h = pp / L, i = pp - h * L;
    const float* q = QKV + i * LDQ + h * DHEAD;
    const float* k = QKV + (jv ? j : 0) * LDQ + D + h * DHEAD;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int c = 0; c < DHEAD; c += 8) {
      const float4 x0 = ld4(q + c), y0 = ld4(k + c), x1 = ld4(q + c + 4), y1 = ld4(k + c + 4);
      a0 = fmaf(x0.x, y0.x, fmaf(x0.y, y0.y, fmaf(x0.z, y0.z, fmaf(x0.w, y0.w, a0))));
      a1 = fmaf(x1.x, y1.x, fmaf(x1.y, y1.y, fmaf(x1.z, y1.z, fmaf(x1.w, y1.w, a1))));
    }
    const float s = jv ? (a0 + a1) * scale : -INFINITY;
    const float m = hmax16(s);
    const float e = jv ? expf(s - m) : 0.f;
    const float p = e / hsum16(e);
    if (pv && jv) P[(h * L + i) * L + j] = p;
    const float* v = QKV + 2 * D + h * DHEAD + j;
    float c0 = 0.f, c1 = 0.f;
    for (int jj = 0; jj < L; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj, 16);
      c0 = fmaf(pj, v[jj * LDQ], c0);
      c1 = fmaf(pj, v[jj * LDQ + 16], c1);
    }
    if (pv) {
      C[i * LDH + h * DHEAD + j] = c0;
      C[i * LDH + h * DHEAD + j + 16] = c1;
    }
  }
}

// Y = LN(A·W + bias + Res) with A·W over NTILE 64-row tiles (K = 64·NTILE);
// also stores xhat and inv (the LN cache)
template <int NTILE>
__device__ __noinline__ void op_fwd_ln(int L, const float* A, int lda, const float* W0,
                                       const float* W1, const float* bias, const float* Res,
                                       const float* g, const float* b, float* XH, float* INV,
                                       float* Y) {

  const int t = threadIdx.x;
  if ((t & ~31) >= L * 16) return;
  const int r0 = t >> 4, c = (t & 15) * 4;
  const bool valid = r0 < L;
  const int r = valid ? r0 : L - 1;
  float4 acc = mm_fwd<D>(make_float4(0.f, 0.f, 0.f, 0.f), A + r * lda, W0, 64, c);
  if (NTILE == 2) acc = mm_fwd<D>(acc, A + r * lda + D, W1, 64, c);
  acc = add4(add4(acc, ld4(bias + c)), ld4(Res + r * LDH + c));
  float v[4] = {acc.x, acc.y, acc.z, acc.w};
  const float inv = ln_fwd4(v);
  if (!valid) return;
  st4(XH + r * LDH + c, make_float4(v[0], v[1], v[2], v[3]));
  const float4 g4 = ld4(g + c), b4 = ld4(b + c);
  st4(Y + r * LDH + c, make_float4(fmaf(g4.x, v[0], b4.x), fmaf(g4.y, v[1], b4.y),
                                   fmaf(g4.z, v[2], b4.z), fmaf(g4.w, v[3], b4.w)));
  if (c == 0) INV[r] = inv;
}

// F[r][64t + c] = relu(bias + A[r]·W_t) (t = 0, 1: the two column halves of fhW)
__device__ __noinline__ void op_ffn1(int L, const float* A, const float* W0, const float* W1,
                                     const float* bias, float* F) {

  const int per = L * 16;
  for (int it = threadIdx.x; it < 2 * per; it += NT) {
    const int tt = it / per, rem = it - tt * per, r = rem >> 4, c = (rem & 15) * 4;
    float4 acc = mm_fwd<D>(make_float4(0.f, 0.f, 0.f, 0.f), A + r * LDH, tt ? W1 : W0, 64, c);
    acc = add4(acc, ld4(bias + 64 * tt + c));
    acc.x = fmaxf(acc.x, 0.f); acc.y = fmaxf(acc.y, 0.f);
    acc.z = fmaxf(acc.z, 0.f); acc.w = fmaxf(acc.w, 0.f);
    st4(F + r * LDF + 64 * tt + c, acc);
  }
}

// dF[r][k] = [F > 0] · Σ_n dY[r][n]·foW[k][n], k over the two 64-row tiles
__device__ __noinline__ void op_dffn(int L, const float* dY, const float* W0, const float* W1,
                                     const float* F, float* dF) {

  const int per = L * 16;
  for (int it = threadIdx.x; it < 2 * per; it += NT) {
    const int tt = it / per, rem = it - tt * per, r = rem >> 4, kb = rem & 15;
    const float4 acc = mm_bwd(make_float4(0.f, 0.f, 0.f, 0.f), dY + r * LDH, tt ? W1 : W0, kb);
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 64 * tt + kb + 16 * j;
      dF[r * LDF + k] = F[r * LDF + k] > 0.f ? a[j] : 0.f;
    }
  }
}

// dX[r][k] = Res[r][k] + Σ_t Σ_n A_t[r][n]·W_t[k][n] (NT_ tiles, A_t = A + t·aoff),
// then (if g) LayerNorm backward with (XH, INV, g):
//   DRAW ← the pre-LN gradient (if non-null), OUT ← LN-backward result
template <int NTILE>
__device__ __noinline__ void op_bwd_ln(int L, const float* A, int lda, int aoff, const float* W0,
                                       const float* W1, const float* W2, const float* Res,
                                       float* DRAW, const float* g, const float* XH,
                                       const float* INV, float* OUT) {

  const int t = threadIdx.x;
  if ((t & ~31) >= L * 16) return;
  const int r0 = t >> 4, kb = t & 15;
  const bool valid = r0 < L;
  const int r = valid ? r0 : L - 1;
  float4 acc = mm_bwd(make_float4(0.f, 0.f, 0.f, 0.f), A + r * lda, W0, kb);
  if (NTILE > 1) acc = mm_bwd(acc, A + r * lda + aoff, W1, kb);
  if (NTILE > 2) acc = mm_bwd(acc, A + r * lda + 2 * aoff, W2, kb);
  float v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] += Res[r * LDH + kb + 16 * j];
  if (valid && DRAW) {
#pragma unroll
    for (int j = 0; j < 4; ++j) DRAW[r * LDH + kb + 16 * j] = v[j];
  }
  if (!g) {
    if (valid && OUT)
#pragma unroll
      for (int j = 0; j < 4; ++j) OUT[r * LDH + kb + 16 * j] = v[j];
    return;
  }
  float xh[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    xh[j] = XH[r * LDH + kb + 16 * j];
    v[j] *= g[kb + 16 * j];
  }
  ln_bwd4(v, xh, INV[r]);
  if (valid)
#pragma unroll
    for (int j = 0; j < 4; ++j) OUT[r * LDH + kb + 16 * j] = v[j];
}

// dC = dA·Woᵀ (no epilogue)
__device__ __noinline__ void op_bwd_plain(int L, const float* A, const float* W, float* out) {

  const int t = threadIdx.x;
  if (t >= L * 16) return;
  const int r = t >> 4, kb = t & 15;
  const float4 acc = mm_bwd(make_float4(0.f, 0.f, 0.f, 0.f), A + r * LDH, W, kb);
  out[r * LDH + kb] = acc.x;
  out[r * LDH + kb + 16] = acc.y;
  out[r * LDH + kb + 32] = acc.z;
  out[r * LDH + kb + 48] = acc.w;
}

// attention backward, part A: half-warp per (head, query row i):
// dP_j = dC_i·V_j, dS = P ⊙ (dP − P·dP) · scale, dQ_i = Σ_j dS_j K_j  (nn.py:99-120)
__device__ __noinline__ void op_attn_bwd_a(int L, const float* QKV, const float* P,
                                           const float* dC, float* dS, float* dQKV, float scale) {

  const int t = threadIdx.x, hw = t >> 4, j = t & 15;
  const bool jv = j < L;
  for (int p0 = 0; p0 < NHEAD * L; p0 += NT / 16) {
    if (p0 + (hw & ~1) >= NHEAD * L) break;
    const int pair = p0 + hw;
    const bool pv = pair < NHEAD * L;
    const int pp = pv ? pair : 0, h = pp / L, i = pp - h * L;
    const float* a = dC + i * LDH + h * DHEAD;
    const float* b = QKV + (jv ? j : 0) * LDQ + 2 * D + h * DHEAD;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int c = 0; c < DHEAD; c += 8) {
      const float4 x0 = ld4(a + c), y0 = ld4(b + c), x1 = ld4(a + c + 4), y1 = ld4(b + c + 4);
      a0 = fmaf(x0.x, y0.x, fmaf(x0.y, y0.y, fmaf(x0.z, y0.z, fmaf(x0.w, y0.w, a0))));
      a1 = fmaf(x1.x, y1.x, fmaf(x1.y, y1.y, fmaf(x1.z, y1.z, fmaf(x1.w, y1.w, a1))));
    }
    const float dp = jv ? a0 + a1 : 0.f;
    const float p = jv ? P[(h * L + i) * L + j] : 0.f;
    const float dot = hsum16(p * dp);
    const float ds = p * (dp - dot) * scale;
    if (pv && jv) dS[(h * L + i) * L + j] = ds;
    const float* kk = QKV + D + h * DHEAD + j;
    float c0 = 0.f, c1 = 0.f;
    for (int jj = 0; jj < L; ++jj) {
      const float sj = __shfl_sync(0xffffffffu, ds, jj, 16);
      c0 = fmaf(sj, kk[jj * LDQ], c0);
      c1 = fmaf(sj, kk[jj * LDQ + 16], c1);
    }
    if (pv) {
      dQKV[i * LDQ + h * DHEAD + j] = c0;
      dQKV[i * LDQ + h * DHEAD + j + 16] = c1;
    }
  }
}

// attention backward, part B: dK_j = Σ_i dS_ij Q_i, dV_j = Σ_i P_ij dC_i
__device__ __noinline__ void op_attn_bwd_b(int L, const float* QKV, const float* P,
                                           const float* dC, const float* dS, float* dQKV) {

  const int per = L * 16;
  for (int it = threadIdx.x; it < 2 * per; it += NT) {
    const int kind = it / per, rem = it - kind * per, j = rem >> 4, c = (rem & 15) * 4;
    const int h = c / DHEAD;
    const float* s = (kind ? P : dS) + h * L * L + j;
    const float* x = kind ? dC + c : QKV + c;
    const int ldx = kind ? LDH : LDQ;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = 0; i < L; ++i) {
      const float sv = s[i * L];
      const float4 y = ld4(x + i * ldx);
      acc.x = fmaf(sv, y.x, acc.x); acc.y = fmaf(sv, y.y, acc.y);
      acc.z = fmaf(sv, y.z, acc.z); acc.w = fmaf(sv, y.w, acc.w);
    }
    st4(dQKV + j * LDQ + D * (1 + kind) + c, acc);
  }
}

// leaf_embed forward partial sums over one slot (≤ 2 tiles):
// thread (kq = t>>3, n4 = t&7) accumulates Σ_{k = 2kq, 2kq+1} Hout[l][k]·W_l[k][4n4..]
__device__ __forceinline__ float4 leaf_fwd_slot(float4 acc, const float* Hout, const float* S, int l0,
                                             int nl) {

  const int t = threadIdx.x, kq = t >> 3, c = (t & 7) * 4;
  for (int u = 0; u < nl; ++u) {
    const float* T = S + u * kLeafTile;
    const float* h = Hout + (l0 + u) * LDH + 2 * kq;
    const float x0 = h[0], x1 = h[1];
    const float4 w0 = ld4(T + (2 * kq) * DE + c), w1 = ld4(T + (2 * kq + 1) * DE + c);
    acc.x = fmaf(x1, w1.x, fmaf(x0, w0.x, acc.x));
    acc.y = fmaf(x1, w1.y, fmaf(x0, w0.y, acc.y));
    acc.z = fmaf(x1, w1.z, fmaf(x0, w0.z, acc.z));
    acc.w = fmaf(x1, w1.w, fmaf(x0, w0.w, acc.w));
  }
  return acc;
}

// leaf_embed backward over one slot: dH[l][k] = Σ_n dzx[n]·W_l[k][n] and
// G_l[k][n] (+)= Hout[l][k]·dzx[n]; thread (k = t>>2, q = t&3) owns n = 8q..8q+7
__device__ __forceinline__ void leaf_bwd_slot(const float* Hout, const float* S, int l0, int nl,
                                              const float* dzx, float* dH, float* G, bool first) {

  const int t = threadIdx.x, k = t >> 2, q = t & 3;
  const float4 z0 = ld4(dzx + 8 * q), z1 = ld4(dzx + 8 * q + 4);
  for (int u = 0; u < nl; ++u) {
    const int l = l0 + u;
    const float* T = S + u * kLeafTile + k * DE + 8 * q;
    const float4 w0 = ld4(T), w1 = ld4(T + 4);
    float s = z0.x * w0.x;
    s = fmaf(z0.y, w0.y, s); s = fmaf(z0.z, w0.z, s); s = fmaf(z0.w, w0.w, s);
    s = fmaf(z1.x, w1.x, s); s = fmaf(z1.y, w1.y, s); s = fmaf(z1.z, w1.z, s);
    s = fmaf(z1.w, w1.w, s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q == 0) dH[l * LDH + k] = s;
    const float hk = Hout[l * LDH + k];
    float* g = G + (size_t)l * D * DE + k * DE + 8 * q;
    float4 g0 = make_float4(hk * z0.x, hk * z0.y, hk * z0.z, hk * z0.w);
    float4 g1 = make_float4(hk * z1.x, hk * z1.y, hk * z1.z, hk * z1.w);
    if (!first) {
      g0 = add4(g0, ld4(g));
      g1 = add4(g1, ld4(g + 4));
    }
    st4(g, g0);
    st4(g + 4, g1);
  }
}

__device__ void decode_with_grad4(double e, const tpcb_boxcox& n, double* y, double* dy) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) {
    *y = exp(t) - n.shift;
    *dy = n.t_std * exp(t);
    return;
  }
  double base = n.lambda_bc * t + 1.0;
  const bool ok = base > 1e-12;
  if (!ok) base = 1e-12;
  *y = pow(base, 1.0 / n.lambda_bc) - n.shift;
  *dy = ok ? n.t_std * pow(base, 1.0 / n.lambda_bc - 1.0) : 0.0;
}

__device__ double decode_plain4(double e, const tpcb_boxcox& n) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) return exp(t) - n.shift;
  return pow(n.lambda_bc * t + 1.0, 1.0 / n.lambda_bc) - n.shift;
}

__device__ __forceinline__ double sgn4(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// ---- weight stream -------------------------------------------------------

// one ring-slot load: either a 64-column weight tile via two TMA boxes
// (tensor map `map`, box origin (col0, row0), `rows` rows) or leaf_embed tiles
// by plain bulk copies
struct SlotLoad {
  int map, col0, row0, rows;  // map < 0: leaf tiles
  int leaf_off, n_leaf;       // first leaf tile (param offset), tile count
};

__host__ __device__ inline int n_leaf_slots(int L) { return (L + 1) >> 1; }
__host__ __device__ inline int n_fwd_slots(int L, bool head) {
  return 1 + 8 * NLAY + n_leaf_slots(L) + (head ? 2 : 0);
}
__host__ __device__ inline int n_all_slots(int L) {
  return n_fwd_slots(L, true) + 2 + n_leaf_slots(L) + 8 * NLAY;
}

// map index of layer li's matrix (0 Wq 1 Wk 2 Wv 3 Wo 4 fhW 5 foW)
__host__ __device__ inline int layer_map(int li, int kind) { return 1 + 6 * li + kind; }
constexpr int kMapDec0 = 1 + 6 * NLAY, kMapDec1 = 2 + 6 * NLAY;

// slot j of a sample with L leaves (order = consumption order)
__device__ SlotLoad stream_slot(const Model& M, int L, int j) {
  auto layer = [&](int li, int kind) -> SlotLoad {  // 0-3 Wq Wk Wv Wo, 4/5 fhW halves, 6/7 foW halves
    if (kind < 4) return SlotLoad{layer_map(li, kind), 0, 0, 64, 0, 0};
    if (kind < 6) return SlotLoad{layer_map(li, 4), 64 * (kind - 4), 0, 64, 0, 0};
    return SlotLoad{layer_map(li, 5), 0, 64 * (kind - 6), 64, 0, 0};
  };
  auto leaf = [&](int s) -> SlotLoad {
    return SlotLoad{-1, 0, 0, 0, M.leafW[L] + 2 * s * kLeafTile, min(2, L - 2 * s)};
  };
  const int nls = n_leaf_slots(L);
  if (j == 0) return SlotLoad{0, 0, 0, FEAT, 0, 0};
  int q = j - 1;
  if (q < 8 * NLAY) return layer(q >> 3, q & 7);
  q -= 8 * NLAY;
  if (q < nls) return leaf(q);
  q -= nls;
  if (q == 0) return SlotLoad{kMapDec0, 0, 0, DE, 0, 0};
  if (q == 1) return SlotLoad{kMapDec1, 0, 0, DEC, 0, 0};
  q -= 2;
  // backward
  if (q == 0) return SlotLoad{kMapDec1, 0, 0, DEC, 0, 0};
  if (q == 1) return SlotLoad{kMapDec0, 0, 0, DE, 0, 0};
  q -= 2;
  if (q < nls) return leaf(q);
  q -= nls;
  const int li = NLAY - 1 - (q >> 3), k = q & 7;
  // foW halves, fhW halves, Wo, Wq, Wk, Wv
  return layer(li, k < 2 ? 6 + k : (k < 4 ? 2 + k : (k == 4 ? 3 : k - 5)));
}

}  // namespace

// shared-memory plan of one v4 CTA (floats)
struct Plan4 {
  int R, NS;
  int oHIN, oQKV, oP, oC, oXH1, oI1, oF, oXH2, oI2, lstride;
  int HOUT, X0, H1, dH, dT1, dT2, dF, dQKV, dS;
  int SV, dv, zv, zp, zx, u0, u1, u2, du1, du2, dz, dzx, dzp, dzv, red, misc, cmd;
  int ring, total;
};

bool v4_supported(const Model& M) {
  if (M.d != D || M.n_layers != NLAY || M.n_heads != NHEAD || M.dh != DHEAD) return false;
  if (M.d_ff != FF || M.d_e != DE || M.d_dev != DDEV || M.n_dec != 2) return false;
  if (M.dec[0] != DEC || M.dec[1] != DEC || M.n_leaf_max > RMAX) return false;
  return true;
}

Plan4 make_plan4(const Model& M, int l_cap, int ns) {
  Plan4 p;
  const int R = (l_cap >= 1 && l_cap <= M.n_leaf_max) ? l_cap : M.n_leaf_max;
  p.R = R;
  p.NS = ns;
  const int pr = (NHEAD * R * R + 3) & ~3;
  int o = 0;
  p.oHIN = o; o += R * LDH;
  p.oQKV = o; o += R * LDQ;
  p.oP = o; o += pr;
  p.oC = o; o += R * LDH;
  p.oXH1 = o; o += R * LDH;
  p.oF = o; o += R * LDF;
  p.oXH2 = o; o += R * LDH;
  p.oI1 = o; o += round4(R);
  p.oI2 = o; o += round4(R);
  p.lstride = o;
  o = NLAY * p.lstride;
  p.HOUT = o; o += R * LDH;
  p.X0 = o; o += 2 * R * LDX;  // double-buffered (the producer fetches ahead)
  p.dH = o; o += R * LDH;
  p.dT1 = o; o += R * LDH;   // dT1, later dA (same rows)
  p.dT2 = o; o += R * LDH;
  p.H1 = p.dT2;              // forward h1 temp (dead before backward)
  p.dF = o; o += R * LDF;    // dF, later dC
  p.dQKV = o; o += R * LDQ;
  p.dS = o; o += pr;
  // CMD scratch (fp64) aliases dF | dQKV | dS, free while the head's backward runs
  p.cmd = p.dF;
  o = (max(o, p.cmd + 2 * cmd_scratch_doubles(DE)) + 3) & ~3;
  p.SV = o; o += SV_TOTAL;
  p.dv = o; o += 8;
  p.zv = o; o += DDEV;
  p.zp = o; o += DE;
  p.zx = o; o += DE;
  p.u0 = o; o += DE;
  p.u1 = o; o += DEC;
  p.u2 = o; o += DEC;
  p.du1 = o; o += DEC;
  p.du2 = o; o += DEC;
  p.dz = o; o += DE;
  p.dzx = o; o += DE;
  p.dzp = o; o += DE;
  p.dzv = o; o += DDEV;
  p.red = o; o += NW * DE;
  p.misc = o; o += 8;
  p.ring = o; o += 256 + ns * kSlot;  // (+ slack: aligned to 1024 B at run time)
  p.total = o;
  return p;
}

namespace {

struct alignas(64) TmaMaps {
  CUtensorMap m[kMaps];
};

struct Stream4 {  // consumer side of the ring
  const float* ring;
  uint64_t* full;
  uint64_t* empty;
  int NS, s, ph;
  long long* trace;
  int J;
  __device__ __forceinline__ const float* acquire(int k = 0) {  // k: slots ahead of the current one
    int ss = s + k, pp = ph;
    if (ss >= NS) { ss -= NS; pp ^= 1; }
    if (trace && J + k < 128) *(volatile long long*)&trace[2 * (J + k)] = clock64();
    mbar_wait(&full[ss], pp);
    if (trace && J + k < 128) *(volatile long long*)&trace[2 * (J + k) + 1] = clock64();
    return ring + ss * kSlot;
  }
  __device__ __forceinline__ void release(int n = 1) {
    __syncwarp();
    for (int u = 0; u < n; ++u) {
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
      ++J;
    }
  }
};

// the per-launch small vectors (biases, LayerNorm, device MLP, output row):
// (param offset, floats, smem offset) — all 16-byte multiples, bulk-copied
__device__ int sv_item(const Model& M, int i, int* off, int* n) {
  constexpr int per = 10;
  if (i < 1) { *off = M.inb; *n = D; return SV_INB; }
  i -= 1;
  if (i < NLAY * per) {
    const LayerOff& lo = M.layer[i / per];
    const int b = SV_LAYER + (i / per) * SV_LSTRIDE;
    switch (i % per) {
      case 0: *off = lo.bq; *n = D; return b + SV_BQKV;
      case 1: *off = lo.bk; *n = D; return b + SV_BQKV + D;
      case 2: *off = lo.bv; *n = D; return b + SV_BQKV + 2 * D;
      case 3: *off = lo.bo; *n = D; return b + SV_BO;
      case 4: *off = lo.ln1g; *n = D; return b + SV_LN1G;
      case 5: *off = lo.ln1b; *n = D; return b + SV_LN1B;
      case 6: *off = lo.fhb; *n = FF; return b + SV_FHB;
      case 7: *off = lo.fob; *n = D; return b + SV_FOB;
      case 8: *off = lo.ln2g; *n = D; return b + SV_LN2G;
      default: *off = lo.ln2b; *n = D; return b + SV_LN2B;
    }
  }
  i -= NLAY * per;
  switch (i) {
    case 0: *off = M.devhW; *n = DEVF * DDEV; return SV_DEVHW;
    case 1: *off = M.devhb; *n = DDEV; return SV_DEVHB;
    case 2: *off = M.devpW; *n = DDEV * DE; return SV_DEVPW;
    case 3: *off = M.devpb; *n = DE; return SV_DEVPB;
    case 4: *off = M.decb[0]; *n = DEC; return SV_DECB0;
    case 5: *off = M.decb[1]; *n = DEC; return SV_DECB1;
    default: *off = M.outW; *n = DEC; return SV_OUTW;
  }
}
constexpr int kSvItems = 1 + 10 * NLAY + 7;
constexpr int kSvBytes = 4 * (D + NLAY * (9 * D + FF) + DEVF * DDEV + DDEV + DDEV * DE + DE + 3 * DEC);

// debug phase timestamps of CTA 0 / thread 0 (first sample only) at trace[256 + id]
#ifdef TPCB_TRACE_PHASES
#define PT(id)                                                        \
  do {                                                                \
    if (ws.trace && first_sample) ws.trace[256 + (id)] = clock64();   \
  } while (0)
#else
#define PT(id) \
  do {         \
  } while (0)
#endif

__global__ void __launch_bounds__(kThreads4, 1) train4_kernel(
    const __grid_constant__ Model M, const float* __restrict__ Pw, SampleSetDev src,
    SampleSetDev tgt, const int32_t* __restrict__ batch_all, const StepDesc* __restrict__ steps,
    int step, LossDev loss, int phase, const __grid_constant__ Plan4 tp,
    const __grid_constant__ TmaMaps maps,
    float* __restrict__ zall, float* __restrict__ partial, size_t slot_stride,
    uint32_t* __restrict__ touched, double* __restrict__ terms, double* __restrict__ scalars,
    float* __restrict__ pred_out, int32_t* status, unsigned long long* __restrict__ stage_flags,
    const int64_t* __restrict__ t_tag, int flag_stride, WgradDev wg) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ __align__(8) uint64_t bars[20 + kStages4];
  const int NS = tp.NS;
  uint64_t* full = bars;
  uint64_t* empty = bars + 8;
  uint64_t* svbar = bars + 16;  // small vectors landed
  uint64_t* xfull = bars + 17;  // [2] input rows of the current sample landed
  uint64_t* stage_bar = bars + 20;  // [kStages4] backward stage written (overlapped reduce)
  const StepDesc sd = steps[step];
  const int32_t* batch = batch_all + sd.off;
  const int n_src = sd.n_src, n_tgt = sd.n_tgt;
  const int n_all = n_src + (loss.use_cmd ? n_tgt : 0);
  const int ns_g = sd.ns_glob, nt_g = sd.nt_glob;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_init(svbar, 1);
    mbar_init(&xfull[0], 1);
    mbar_init(&xfull[1], 1);
    for (int q = 0; q < kStages4; ++q) mbar_init(&stage_bar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // ring slots need 1024-byte alignment (128-byte swizzle atoms)
  const uint32_t sm_base = smem_u32(sm);
  float* ring = sm + ((((sm_base + tp.ring * 4u) + 1023u) & ~1023u) - sm_base) / 4u;
  float* SV = sm + tp.SV;
  float* X0b = sm + tp.X0;

  // ================================================================ producer
  if (warp == NW) {
    if (lane < kMaps) tma_prefetch_desc(&maps.m[lane]);
    if (lane == 0) mbar_arrive_expect_tx(svbar, (uint32_t)kSvBytes);
    __syncwarp();
    if (lane < kSvItems) {
      int off, n;
      const int d = sv_item(M, lane, &off, &n);
      bulk_g2s(SV + d, Pw + off, (uint32_t)(n * 4), svbar);
    }
    int s = 0, ph = 0, J = 0, xs = 0;
    for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
      const SampleSetDev set = w >= n_src ? tgt : src;
      const int idx = batch[w];
      const int L = set.n_leaf[idx];
      if (L < 1 || L > tp.R) continue;  // the compute warps skip it too
      if (lane == 0) {  // the sample's packed input rows (contiguous, 128 B each)
        const int b = xs & 1;
        mbar_arrive_expect_tx(&xfull[b], (uint32_t)(L * LDX * 4));
        bulk_g2s(X0b + b * tp.R * LDX, set.x + (size_t)set.ast_row[idx] * TPCB_FEAT_PAD,
                 (uint32_t)(L * LDX * 4), &xfull[b]);
      }
      ++xs;
      const int n_slots = phase == 0 ? n_fwd_slots(L, false) : n_all_slots(L);
      for (int j = 0; j < n_slots; ++j, ++J) {
        if (J >= NS) mbar_wait(&empty[s], ph ^ 1);
        const SlotLoad x = stream_slot(M, L, j);
        float* dst = ring + s * kSlot;
        if (lane == 0) {
          if (x.map >= 0) {
            mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * x.rows * 128));
            tma_load_2d(dst, &maps.m[x.map], x.col0, x.row0, &full[s]);
            tma_load_2d(dst + x.rows * 32, &maps.m[x.map], x.col0 + 32, x.row0, &full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], (uint32_t)(x.n_leaf * kLeafTile * 4));
            bulk_g2s(dst, Pw + x.leaf_off, (uint32_t)(x.n_leaf * kLeafTile * 4), &full[s]);
          }
        }
        __syncwarp();
        if (++s == NS) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  // ============================================ stage publisher (one lane)
  // Overlapped reduce: once the compute warps have written a backward stage's
  // gradients (stage_bar[q]), count this CTA into the stage's word after a
  // gpu-scope fence — a warp of its own, so neither the weight stream nor the
  // compute warps wait on the fence.  The words count CTAs cumulatively over
  // the steps of an epoch (zeroed at its first step).
  if (warp == NW + 1) {
    if (!stage_flags || lane != 0 || (int)blockIdx.x >= n_all) return;
    const int w = blockIdx.x;  // one sample per CTA on this path
    const SampleSetDev set = w >= n_src ? tgt : src;
    const int L = set.n_leaf[batch[w]];
    if (L < 1 || L > tp.R) return;
    (void)t_tag;
    for (int q = 0; q < kStages4; ++q) {
      mbar_wait(&stage_bar[q], 0);
      __threadfence();
      atomicAdd(stage_flags + (size_t)q * flag_stride, 1ull);  // one L2 atomic, never retried
    }
    return;
  }

  // ========================================================== compute warps
  const float scale = 1.f / sqrtf((float)DHEAD);
  float* G = partial + (size_t)blockIdx.x * slot_stride;
  // tensor-core weight gradients (phase 1 without CMD): the step's row
  // stride Ls = its largest leaf count (single-bucket plans: every sample's)
  const bool use_wg = wg.act != nullptr && phase == 1 && !loss.use_cmd;
  __shared__ int s_Ls;
  if (use_wg && warp == 0) {
    int m = 0;
    for (int i = lane; i < n_src; i += 32) m = max(m, src.n_leaf[batch[i]]);
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if (lane == 0) s_Ls = m;
  }
  cbar();
  const int Ls = use_wg ? s_Ls : 0;
  uint32_t mask = 0;
  int xs = 0;  // samples processed (input-row buffer parity)
  const float outb = __ldg(Pw + M.outb);
  float* HOUT = sm + tp.HOUT;
  float* H1 = sm + tp.H1;
  float* dH = sm + tp.dH;
  float* dT1 = sm + tp.dT1;
  float* dA = dT1;
  float* dT2 = sm + tp.dT2;
  float* dF = sm + tp.dF;
  float* dC = dF;
  float* dQKV = sm + tp.dQKV;
  float* dS = sm + tp.dS;
  float* dv = sm + tp.dv;
  float* zv = sm + tp.zv;
  float* zp = sm + tp.zp;
  float* zx = sm + tp.zx;
  float* u0 = sm + tp.u0;
  float* u1 = sm + tp.u1;
  float* u2 = sm + tp.u2;
  float* du1 = sm + tp.du1;
  float* du2 = sm + tp.du2;
  float* dz = sm + tp.dz;
  float* dzx = sm + tp.dzx;
  float* dzp = sm + tp.dzp;
  float* dzv = sm + tp.dzv;
  float* red = sm + tp.red;
  float* misc = sm + tp.misc;
  double* cmds = reinterpret_cast<double*>(sm + tp.cmd);
  auto stage_done = [&](int q) {  // all compute warps passed cbar() after the stage's writes
    if (stage_flags && threadIdx.x == 0) mbar_arrive(&stage_bar[q]);
  };
  long long* trace = g_trace4;
  Stream4 ws{ring, full, empty, NS, 0, 0,
             (trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) ? trace : nullptr, 0};

  mbar_wait(svbar, 0);  // small vectors (bulk-copied by the producer)

  for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
#ifdef TPCB_TRACE_PHASES
    const bool first_sample = w == (int)blockIdx.x;
#endif
    const bool is_t = w >= n_src;
    const SampleSetDev set = is_t ? tgt : src;
    const int idx = batch[w];
    const int L = set.n_leaf[idx];
    if (L < 1 || L > tp.R) {
      if (threadIdx.x == 0) raise_status(status, TPCB_ERR_LEAF_COUNT);
      continue;
    }
    const int nls = n_leaf_slots(L);
    if (ws.trace) ws.trace[510] = clock64();
    float lb = 0.f, dvv = 0.f;  // leafb[L] (threads < DE), device features (threads < DEVF)
    if (threadIdx.x < DE) lb = __ldg(Pw + M.leafb[L] + threadIdx.x);
    if (threadIdx.x < DEVF) dvv = __ldg(set.devfeat + (size_t)idx * DEVF + threadIdx.x);
    float* X0 = X0b + (xs & 1) * tp.R * LDX;
    mbar_wait(&xfull[xs & 1], (xs >> 1) & 1);
    ++xs;
    if (threadIdx.x < DEVF) dv[threadIdx.x] = dvv;
    cbar();
    PT(0);

    // ------------------------------------------------------------ forward
    {  // input projection (no LN): H0 = X0·inW + inb
      const float* W = ws.acquire();
      PT(1);
      float* H0 = sm + tp.oHIN;
      for (int it = threadIdx.x; it < L * 16; it += NT) {
        const int r = it >> 4, c = (it & 15) * 4;
        const float4 acc = mm_fwd<FEAT>(make_float4(0.f, 0.f, 0.f, 0.f), X0 + r * LDX, W, FEAT, c);
        st4(H0 + r * LDH + c, add4(acc, ld4(SV + SV_INB + c)));
      }
      ws.release();
      if (threadIdx.x < DDEV) {  // device MLP hidden layer (costmodel.py forward head)
        const int n = threadIdx.x;
        float s = 0.f;
        for (int k = 0; k < DEVF; ++k) s = fmaf(dv[k], SV[SV_DEVHW + k * DDEV + n], s);
        zv[n] = fmaxf(s + SV[SV_DEVHB + n], 0.f);
      }
      cbar();
      PT(2);
    }
    for (int li = 0; li < NLAY; ++li) {
      float* base = sm + li * tp.lstride;
      float* HIN = base + tp.oHIN;
      float* QKV = base + tp.oQKV;
      float* Pp = base + tp.oP;
      float* C = base + tp.oC;
      float* XH1 = base + tp.oXH1;
      float* F = base + tp.oF;
      float* XH2 = base + tp.oXH2;
      float* I1 = base + tp.oI1;
      float* I2 = base + tp.oI2;
      const float* sv = SV + SV_LAYER + li * SV_LSTRIDE;
      float* out = li + 1 < NLAY ? sm + (li + 1) * tp.lstride + tp.oHIN : HOUT;
      {
        const float* Wq = ws.acquire(0);
        const float* Wk = ws.acquire(1);
        const float* Wv = ws.acquire(2);
        op_qkv(L, HIN, Wq, Wk, Wv, sv + SV_BQKV, QKV);
        PT(10 + li * 20 + 0);
        ws.release(3);
        if (li == 0 && threadIdx.x >= NT - DE) {  // device MLP projection
          const int n = threadIdx.x - (NT - DE);
          float s = 0.f;
          for (int k = 0; k < DDEV; ++k) s = fmaf(zv[k], SV[SV_DEVPW + k * DE + n], s);
          zp[n] = s + SV[SV_DEVPB + n];
        }
      }
      cbar();
      PT(10 + li * 20 + 1);
      op_attn_fwd(L, QKV, Pp, C, scale);
      PT(10 + li * 20 + 2);
      cbar();
      PT(10 + li * 20 + 3);
      {
        const float* Wo = ws.acquire();
        PT(10 + li * 20 + 4);
        op_fwd_ln<1>(L, C, LDH, Wo, nullptr, sv + SV_BO, HIN, sv + SV_LN1G, sv + SV_LN1B, XH1, I1,
                     H1);
        PT(10 + li * 20 + 5);
        ws.release();
      }
      cbar();
      PT(10 + li * 20 + 6);
      {
        const float* W0 = ws.acquire(0);
        const float* W1 = ws.acquire(1);
        PT(10 + li * 20 + 7);
        op_ffn1(L, H1, W0, W1, sv + SV_FHB, F);
        PT(10 + li * 20 + 8);
        ws.release(2);
      }
      cbar();
      PT(10 + li * 20 + 9);
      {
        const float* W0 = ws.acquire(0);
        const float* W1 = ws.acquire(1);
        PT(10 + li * 20 + 10);
        op_fwd_ln<2>(L, F, LDF, W0, W1, sv + SV_FOB, H1, sv + SV_LN2G, sv + SV_LN2B, XH2, I2, out);
        PT(10 + li * 20 + 11);
        ws.release(2);
      }
      cbar();
      PT(10 + li * 20 + 12);
    }
    // head: z_x = b_L + Σ_l Hout[l]·W_L[l] (leaf tiles streamed two per slot)
    {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < nls; ++s) {
        const float* S = ws.acquire();
        acc = leaf_fwd_slot(acc, HOUT, S, 2 * s, min(2, L - 2 * s));
        ws.release();
      }
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 8);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, 8);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 16);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, 16);
      if (lane < 8) st4(red + warp * DE + lane * 4, acc);
    }
    cbar();
    PT(50);
    if (threadIdx.x < DE) {
      const int n = threadIdx.x;
      float s = lb;
      for (int k = 0; k < NW; ++k) s += red[k * DE + n];
      zx[n] = s;
      u0[n] = s * zp[n];
    }
    const int zrow = is_t ? ns_g + sd.tgt_pos + (w - n_src) : sd.src_pos + w;
    if (phase == 0) {
      cbar();
      if (threadIdx.x < DE) zall[(size_t)zrow * DE + threadIdx.x] = u0[threadIdx.x];
      cbar();
      continue;
    }
    cbar();
    PT(51);
    {
      const float* W = ws.acquire();
      gemv_f(u0, DE, W, DEC, SV + SV_DECB0, true, u1);
      ws.release();
    }
    cbar();
    PT(52);
    {
      const float* W = ws.acquire();
      gemv_f(u1, DEC, W, DEC, SV + SV_DECB1, true, u2);
      ws.release();
    }
    cbar();
    PT(53);
    // output, loss gradient (warp 0)
    const bool fs = !(mask & 1u);
    const bool fl = !(mask & (1u << L));
    if (warp == 0) {
      const float* ow = SV + SV_OUTW;
      float s = fmaf(u2[lane], ow[lane], u2[lane + 32] * ow[lane + 32]);
      const float pred = warp_sum(s) + outb;
      double dpred = 0.0;
      if (lane == 0 && !is_t) {
        const double y = set.y[idx];
        const double ddf = (double)pred - y;
        const double n = (double)sd.n_norm;
        double rel = 0.0, relg = 0.0;
        if (loss.mode != kLossMse) {
          if (loss.original) {
            const double y0 = decode_plain4(y, loss.norm);
            double p0, dp0;
            decode_with_grad4((double)pred, loss.norm, &p0, &dp0);
            const double r = p0 - y0;
            rel = fabs(r) / y0;
            relg = sgn4(r) * dp0 / (y0 * n);
          } else {
            const double den = y + loss.offset;
            rel = fabs(ddf) / den;
            relg = sgn4(ddf) / (den * n);
          }
        }
        if (loss.mode == kLossMse)
          dpred = 2.0 * ddf / n;
        else if (loss.mode == kLossMape)
          dpred = relg;
        else
          dpred = 2.0 * ddf / n + loss.lambda * relg;
        terms[2 * w] = ddf * ddf;
        terms[2 * w + 1] = rel;
        if (pred_out) pred_out[w] = pred;
      }
      const float dp = __shfl_sync(0xffffffffu, (float)dpred, 0);
      for (int c = lane; c < DEC; c += 32) {
        const float g0 = u2[c] * dp;
        G[M.outW + c] = fs ? g0 : G[M.outW + c] + g0;
        du2[c] = u2[c] > 0.f ? ow[c] * dp : 0.f;
      }
      if (lane == 0) G[M.outb] = fs ? dp : G[M.outb] + dp;
    }
    cbar();
    PT(54);
    // ------------------------------------------------------------ backward
    {  // decoder layer 1
      const float* W = ws.acquire();
      gemv_t(du2, DEC, W, DEC, u1, du1);
      ws.release();
      outer(u1, DEC, du2, DEC, G + M.decW[1], fs);
      colsum(du2, 0, nullptr, 0, 1, DEC, G + M.decb[1], fs, NT - DEC);
    }
    cbar();
    PT(55);
    {  // decoder layer 0
      const float* W = ws.acquire();
      gemv_t(du1, DEC, W, DE, nullptr, dz);
      ws.release();
      outer(u0, DE, du1, DEC, G + M.decW[0], fs);
      colsum(du1, 0, nullptr, 0, 1, DEC, G + M.decb[0], fs, NT - DEC);
    }
    cbar();
    PT(56);
    if (loss.use_cmd) {
      const double v = cmd_stats(zall, ns_g, nt_g, DE, loss.cmd_order, cmds, kBar, NT);
      if (blockIdx.x == 0 && threadIdx.x == 0 && w == (int)blockIdx.x) scalars[0] = v;
      if (threadIdx.x < DE) {
        const int e = threadIdx.x;
        dz[e] += (float)(loss.alpha * cmd_grad_elem(cmds, ns_g, nt_g, DE, loss.cmd_order, zrow, e,
                                                    (double)zall[(size_t)zrow * DE + e]));
      }
      cbar();
    }
    if (threadIdx.x < DE) {
      const int e = threadIdx.x;
      dzx[e] = dz[e] * zp[e];
      dzp[e] = dz[e] * zx[e];
    }
    cbar();
    PT(57);
    {  // leaf_embed backward + device projection backward
      if (threadIdx.x < DDEV) {
        const int k = threadIdx.x;
        float s = 0.f;
        for (int n = 0; n < DE; ++n) s = fmaf(dzp[n], SV[SV_DEVPW + k * DE + n], s);
        dzv[k] = zv[k] > 0.f ? s : 0.f;
      }
      for (int s = 0; s < nls; ++s) {
        const float* S = ws.acquire();
        leaf_bwd_slot(HOUT, S, 2 * s, min(2, L - 2 * s), dzx, dH, G + M.leafW[L], fl);
        ws.release();
      }
      outer(zv, DDEV, dzp, DE, G + M.devpW, fs);
      colsum(dzp, 0, nullptr, 0, 1, DE, G + M.devpb, fs, NT - 2 * DE);
      colsum(dzx, 0, nullptr, 0, 1, DE, G + M.leafb[L], fl, NT - DE);
    }
    cbar();
    PT(58);
    {  // LayerNorm-2 backward of the last layer; device hidden-layer gradient
      const int li = NLAY - 1;
      float* base = sm + li * tp.lstride;
      const float* sv = SV + SV_LAYER + li * SV_LSTRIDE;
      const int t = threadIdx.x;
      if ((t & ~31) < L * 16) {  // whole warps (half-warp shuffles)
        const bool valid = (t >> 4) < L;
        const int r = valid ? t >> 4 : L - 1, kb = t & 15;
        float v[4], xh[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[j] = dH[r * LDH + kb + 16 * j] * sv[SV_LN2G + kb + 16 * j];
          xh[j] = base[tp.oXH2 + r * LDH + kb + 16 * j];
        }
        ln_bwd4(v, xh, base[tp.oI2 + r]);
        if (valid)
#pragma unroll
          for (int j = 0; j < 4; ++j) dT1[r * LDH + kb + 16 * j] = v[j];
      }
      outer(dv, DEVF, dzv, DDEV, G + M.devhW, fs);
      colsum(dzv, 0, nullptr, 0, 1, DDEV, G + M.devhb, fs, NT - DDEV);
    }
    cbar();
    stage_done(0);  // head, decoder, leaf_embed.L, device MLP (+ loss terms)
    PT(59);
    for (int li = NLAY - 1; li >= 0; --li) {
      const LayerOff& lo = M.layer[li];
      float* base = sm + li * tp.lstride;
      float* HIN = base + tp.oHIN;
      float* QKV = base + tp.oQKV;
      float* Pp = base + tp.oP;
      float* C = base + tp.oC;
      float* XH1 = base + tp.oXH1;
      float* F = base + tp.oF;
      float* XH2 = base + tp.oXH2;
      float* I1 = base + tp.oI1;
      const float* sv = SV + SV_LAYER + li * SV_LSTRIDE;
      {  // B1: dF = relu'(F) ⊙ dT1·foWᵀ; dW_fo, fob, ln2 g/b
        const float* W0 = ws.acquire(0);
        const float* W1 = ws.acquire(1);
        PT(60 + (NLAY - 1 - li) * 30 + 0);
        op_dffn(L, dT1, W0, W1, F, dF);
        PT(60 + (NLAY - 1 - li) * 30 + 1);
        ws.release(2);
        if (use_wg) {
          act_store(wg, li * kWgOpsLayer + kWgF, F, LDF, nullptr, nullptr, L, Ls, FF, w);
          act_store(wg, li * kWgOpsLayer + kWgDT1, dT1, LDH, nullptr, nullptr, L, Ls, D, w);
        } else {
          wgrad(F, LDF, nullptr, nullptr, dT1, LDH, L, FF, D, G + lo.foW, fs);
        }
        PT(60 + (NLAY - 1 - li) * 30 + 2);
        colsum(dT1, LDH, nullptr, 0, L, D, G + lo.fob, fs, 0);
        colsum(dH, LDH, XH2, LDH, L, D, G + lo.ln2g, fs, 64);
        colsum(dH, LDH, nullptr, 0, L, D, G + lo.ln2b, fs, 128);
        PT(60 + (NLAY - 1 - li) * 30 + 3);
      }
      cbar();
      PT(60 + (NLAY - 1 - li) * 30 + 4);
      {  // B2: dT2 = dT1 + dF·fhWᵀ → LN1 backward → dA; dW_fh, fhb
        const float* W0 = ws.acquire(0);
        const float* W1 = ws.acquire(1);
        PT(60 + (NLAY - 1 - li) * 30 + 5);
        op_bwd_ln<2>(L, dF, LDF, D, W0, W1, nullptr, dT1, dT2, sv + SV_LN1G, XH1, I1, dA);
        PT(60 + (NLAY - 1 - li) * 30 + 6);
        ws.release(2);
        if (use_wg) {
          act_store(wg, li * kWgOpsLayer + kWgH1, XH1, LDH, sv + SV_LN1G, sv + SV_LN1B, L, Ls, D,
                    w);
          act_store(wg, li * kWgOpsLayer + kWgDF, dF, LDF, nullptr, nullptr, L, Ls, FF, w);
        } else {
          wgrad(XH1, LDH, sv + SV_LN1G, sv + SV_LN1B, dF, LDF, L, D, FF, G + lo.fhW, fs);
        }
        PT(60 + (NLAY - 1 - li) * 30 + 7);
        colsum(dF, LDF, nullptr, 0, L, FF, G + lo.fhb, fs, 0);
        PT(60 + (NLAY - 1 - li) * 30 + 8);
      }
      cbar();
      stage_done(1 + 2 * (NLAY - 1 - li));  // layer li: ffn + LayerNorm-2
      PT(60 + (NLAY - 1 - li) * 30 + 9);
      {  // B3: dC = dA·Woᵀ; dW_o, bo, ln1 g/b
        const float* W = ws.acquire();
        PT(60 + (NLAY - 1 - li) * 30 + 10);
        op_bwd_plain(L, dA, W, dC);
        PT(60 + (NLAY - 1 - li) * 30 + 11);
        ws.release();
        if (use_wg) {
          act_store(wg, li * kWgOpsLayer + kWgC, C, LDH, nullptr, nullptr, L, Ls, D, w);
          act_store(wg, li * kWgOpsLayer + kWgDA, dA, LDH, nullptr, nullptr, L, Ls, D, w);
        } else {
          wgrad(C, LDH, nullptr, nullptr, dA, LDH, L, D, D, G + lo.Wo, fs);
        }
        PT(60 + (NLAY - 1 - li) * 30 + 12);
        colsum(dA, LDH, nullptr, 0, L, D, G + lo.bo, fs, 0);
        colsum(dT2, LDH, XH1, LDH, L, D, G + lo.ln1g, fs, 64);
        colsum(dT2, LDH, nullptr, 0, L, D, G + lo.ln1b, fs, 128);
        PT(60 + (NLAY - 1 - li) * 30 + 13);
      }
      cbar();
      PT(60 + (NLAY - 1 - li) * 30 + 14);
      op_attn_bwd_a(L, QKV, Pp, dC, dS, dQKV, scale);
      PT(60 + (NLAY - 1 - li) * 30 + 15);
      cbar();
      PT(60 + (NLAY - 1 - li) * 30 + 16);
      op_attn_bwd_b(L, QKV, Pp, dC, dS, dQKV);
      PT(60 + (NLAY - 1 - li) * 30 + 17);
      cbar();
      PT(60 + (NLAY - 1 - li) * 30 + 18);
      {  // B6: dHin = dA + dQ·Wqᵀ + dK·Wkᵀ + dV·Wvᵀ (→ LN2 backward of the layer below)
        const float* Wq = ws.acquire(0);
        const float* Wk = ws.acquire(1);
        const float* Wv = ws.acquire(2);
        PT(60 + (NLAY - 1 - li) * 30 + 19);
        if (li > 0) {
          float* pb = sm + (li - 1) * tp.lstride;
          const float* psv = SV + SV_LAYER + (li - 1) * SV_LSTRIDE;
          op_bwd_ln<3>(L, dQKV, LDQ, D, Wq, Wk, Wv, dA, dH, psv + SV_LN2G, pb + tp.oXH2,
                       pb + tp.oI2, dT1);
        } else {
          op_bwd_ln<3>(L, dQKV, LDQ, D, Wq, Wk, Wv, dA, dH, nullptr, nullptr, nullptr, nullptr);
        }
        PT(60 + (NLAY - 1 - li) * 30 + 20);
        ws.release(3);
        if (use_wg) {
          act_store(wg, li * kWgOpsLayer + kWgHIN, HIN, LDH, nullptr, nullptr, L, Ls, D, w);
          act_store(wg, li * kWgOpsLayer + kWgDQ, dQKV, LDQ, nullptr, nullptr, L, Ls, D, w);
          act_store(wg, li * kWgOpsLayer + kWgDK, dQKV + D, LDQ, nullptr, nullptr, L, Ls, D, w);
          act_store(wg, li * kWgOpsLayer + kWgDV, dQKV + 2 * D, LDQ, nullptr, nullptr, L, Ls, D,
                    w);
        } else {
          wgrad(HIN, LDH, nullptr, nullptr, dQKV, LDQ, L, D, D, G + lo.Wq, fs);
          wgrad(HIN, LDH, nullptr, nullptr, dQKV + D, LDQ, L, D, D, G + lo.Wk, fs);
          wgrad(HIN, LDH, nullptr, nullptr, dQKV + 2 * D, LDQ, L, D, D, G + lo.Wv, fs);
        }
        PT(60 + (NLAY - 1 - li) * 30 + 21);
        colsum(dQKV, LDQ, nullptr, 0, L, D, G + lo.bq, fs, 0);
        colsum(dQKV + D, LDQ, nullptr, 0, L, D, G + lo.bk, fs, 64);
        colsum(dQKV + 2 * D, LDQ, nullptr, 0, L, D, G + lo.bv, fs, 128);
        PT(60 + (NLAY - 1 - li) * 30 + 22);
      }
      cbar();
      stage_done(2 + 2 * (NLAY - 1 - li));  // layer li: attention + LayerNorm-1
      PT(60 + (NLAY - 1 - li) * 30 + 23);
    }
    if (use_wg) {
      act_store(wg, kWgX0, X0, LDX, nullptr, nullptr, L, Ls, 32, w);  // K padded to 32
      act_store(wg, kWgDH, dH, LDH, nullptr, nullptr, L, Ls, D, w);
    } else {
      wgrad(X0, LDX, nullptr, nullptr, dH, LDH, L, FEAT, D, G + M.inW, fs);
    }
    colsum(dH, LDH, nullptr, 0, L, D, G + M.inb, fs, NT - D);
    PT(125);
    mask |= 1u | (1u << L);
    cbar();
    if (ws.trace) ws.trace[511] = clock64();
  }
  if (threadIdx.x == 0) touched[blockIdx.x] = mask;
  stage_done(kStages4 - 1);  // input projection, touched mask
}

}  // namespace

static int ring_slots_for(const Model& M, int l_cap, size_t lim) {
  for (int ns = 6; ns >= 4; --ns)
    if ((size_t)make_plan4(M, l_cap, ns).total * 4 <= lim) return ns;
  return 0;
}

static size_t train4_dyn_limit() {
  static size_t lim = 0;
  if (!lim) {
    cudaFuncAttributes a{};
    if (cudaFuncGetAttributes(&a, train4_kernel) != cudaSuccess) return 0;
    lim = 227 * 1024 - a.sharedSizeBytes;
    if (cudaFuncSetAttribute(train4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lim) != cudaSuccess)
      return 0;
  }
  return lim;
}

bool v4_fits(const Model& M, int l_cap) {
  if (!v4_supported(M)) return false;
  const size_t lim = train4_dyn_limit();
  return lim && ring_slots_for(M, l_cap, lim) > 0;
}

// tensor maps of the streamed weight matrices (rows × cols fp32, row-major,
// boxes of 32 columns × box_rows rows, 128-byte swizzle), cached per
// parameter buffer
static int encode_map(CUtensorMap* m, const float* base, int rows, int cols, int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  // driver entry point through the runtime: the library does not link libcuda
  // (it must load on hosts without a driver; compute calls then fail cleanly)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
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
  const CUresult r = encode(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled", cudaErrorInvalidValue);
    return TPCB_ERR_CUDA;
  }
  return TPCB_OK;
}

static int build_maps(const Model& M, const float* P, TmaMaps* t) {
  int st = encode_map(&t->m[0], P + M.inW, FEAT, D, FEAT);
  for (int li = 0; li < NLAY && !st; ++li) {
    const LayerOff& lo = M.layer[li];
    st = encode_map(&t->m[layer_map(li, 0)], P + lo.Wq, D, D, 64);
    if (!st) st = encode_map(&t->m[layer_map(li, 1)], P + lo.Wk, D, D, 64);
    if (!st) st = encode_map(&t->m[layer_map(li, 2)], P + lo.Wv, D, D, 64);
    if (!st) st = encode_map(&t->m[layer_map(li, 3)], P + lo.Wo, D, D, 64);
    if (!st) st = encode_map(&t->m[layer_map(li, 4)], P + lo.fhW, D, FF, 64);
    if (!st) st = encode_map(&t->m[layer_map(li, 5)], P + lo.foW, FF, D, 64);
  }
  if (!st) st = encode_map(&t->m[kMapDec0], P + M.decW[0], DE, DEC, DE);
  if (!st) st = encode_map(&t->m[kMapDec1], P + M.decW[1], DEC, DEC, DEC);
  return st;
}

// resident train4 CTAs per SM for this model / leaf cap (0: does not fit);
// the overlapped reduce is only used when every training CTA of a step is
// co-resident next to the reduce blocks (capi_train.cu)
int train4_blocks_per_sm(const Model& M, int l_cap) {
  const size_t lim = train4_dyn_limit();
  if (!lim) return 0;
  const int ns = ring_slots_for(M, l_cap, lim);
  if (!ns) return 0;
  const Plan4 tp = make_plan4(M, l_cap, ns);
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, train4_kernel, kThreads4,
                                                    (size_t)tp.total * sizeof(float)) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return blocks;
}

int launch_train4(const Model& M, const float* P, const SampleSetDev& src, const SampleSetDev& tgt,
                  const int32_t* batch, const StepDesc* steps, int step, int grid,
                  const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                  int32_t* status, cudaStream_t stream) {
  if (!v4_supported(M) || loss.cmd_order > kMaxCmdOrder) return TPCB_ERR_UNSUPPORTED;
  const size_t lim = train4_dyn_limit();
  if (!lim) TPCB_CUDA_CHECK(cudaGetLastError());
  const int ns = ring_slots_for(M, ws.l_cap, lim);
  if (!ns) return TPCB_ERR_UNSUPPORTED;
  const Plan4 tp = make_plan4(M, ws.l_cap, ns);
  const size_t smem = (size_t)tp.total * sizeof(float);
  thread_local const float* cached_p = nullptr;
  thread_local Model cached_m{};
  thread_local TmaMaps maps;
  if (cached_p != P || memcmp(&cached_m, &M, sizeof(Model)) != 0) {
    const int st = build_maps(M, P, &maps);
    if (st) return st;
    cached_p = P;
    cached_m = M;
  }
  grid = std::max(1, std::min(grid, ws.n_slots));
  train4_kernel<<<grid, kThreads4, smem, stream>>>(M, P, src, tgt, batch, steps, step, loss, phase,
                                                   tp, maps, ws.zall, ws.partial, ws.slot_stride,
                                                   ws.touched, ws.terms, ws.scalars, pred_out,
                                                   status, ws.stage_flags, ws.t_tag,
                                                   ws.flag_stride, ws.wg);
  TPCB_LAUNCH_CHECK("train4_kernel");
  return TPCB_OK;
}

}  // namespace tpcb
