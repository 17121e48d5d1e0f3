// Device building blocks for the fused predictor kernels (FP32 FFMA path).
//
// All activations of a tile live in shared memory with an odd row stride
// (ld = width + 1) so that a warp walking different rows of one column hits
// distinct banks.  Weights are read straight from global memory: the whole
// desk model is 1.4 MB and stays resident in the 126 MB L2, and every CTA of
// the grid reads the same bytes, so L1/L2 serve them.
#pragma once

#include "common.cuh"

namespace tpcb {

// Y[r, n] = act(b[n] + Σ_k X[r, k] W[k, n]) (+ Res[r, n])  for r < R, n < N.
// X/Y/Res in shared memory (row strides ldx/ldy/ldr), W row-major [K, N] and
// b in global memory.  Each thread owns a TM×TN register tile.
template <int TM, int TN>
__device__ __forceinline__ void gemm_rows(const float* X, int ldx, const float* __restrict__ W,
                                          const float* __restrict__ b, float* Y, int ldy, int R,
                                          int K, int N, bool relu, const float* Res = nullptr,
                                          int ldr = 0) {
  const int ncg = (N + TN - 1) / TN;
  const int nrg = (R + TM - 1) / TM;
  const bool vec = (TN == 4) && ((N & 3) == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0);
  for (int job = threadIdx.x; job < ncg * nrg; job += blockDim.x) {
    const int cg = job % ncg, rg = job / ncg;
    const int c0 = cg * TN, r0 = rg * TM;
    float acc[TM][TN];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const float bj = (b != nullptr && c0 + j < N) ? __ldg(b + c0 + j) : 0.f;
#pragma unroll
      for (int i = 0; i < TM; ++i) acc[i][j] = bj;
    }
    int rr[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) rr[i] = min(r0 + i, R - 1) * ldx;
    if (vec) {
      for (int k = 0; k < K; ++k) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(W + (size_t)k * N + c0));
        const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float xv = X[rr[i] + k];
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(xv, w[j], acc[i][j]);
        }
      }
    } else {
      for (int k = 0; k < K; ++k) {
        float w[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) w[j] = (c0 + j < N) ? __ldg(W + (size_t)k * N + c0 + j) : 0.f;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float xv = X[rr[i] + k];
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(xv, w[j], acc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = r0 + i;
      if (r >= R) break;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = c0 + j;
        if (c >= N) break;
        float v = acc[i][j];
        if (relu) v = fmaxf(v, 0.f);
        if (Res) v += Res[r * ldr + c];
        Y[r * ldy + c] = v;
      }
    }
  }
}

// Row-wise LayerNorm over `d` features (nn.py:48-54): biased variance, eps
// 1e-5 inside the square root.  One warp per row; optionally stores xhat and
// 1/sqrt(var+eps) for the backward pass.
__device__ __forceinline__ void layernorm_rows(const float* X, int ldx, float* Y, int ldy, int R,
                                               int d, const float* __restrict__ g,
                                               const float* __restrict__ b, float* xhat = nullptr,
                                               int ldh = 0, float* inv_out = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float inv_d = 1.f / (float)d;
  for (int r = w; r < R; r += nw) {
    const float* x = X + r * ldx;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += x[c];
    const float mu = warp_sum(s) * inv_d;
    float v = 0.f;
    for (int c = lane; c < d; c += 32) {
      const float t = x[c] - mu;
      v = fmaf(t, t, v);
    }
    const float var = warp_sum(v) * inv_d;
    const float inv = 1.f / sqrtf(var + 1e-5f);
    for (int c = lane; c < d; c += 32) {
      const float xh = (x[c] - mu) * inv;
      if (xhat) xhat[r * ldh + c] = xh;
      Y[r * ldy + c] = fmaf(__ldg(g + c), xh, __ldg(b + c));
    }
    if (inv_out && lane == 0) inv_out[r] = inv;
  }
}

// Multi-head self-attention core over A ASTs of L rows each (rows a*L ..
// a*L+L-1), heads of width dh: ctx = softmax(Q Kᵀ/sqrt(dh)) V per AST and
// head (nn.py:79-96).  Bucketing makes every AST attend over exactly its own L
// leaves, so no mask is needed.  One thread per (AST, head, query row);
// optionally stores the probabilities P[(a*H + h)*L*L + i*L + j].
__device__ __forceinline__ void attention_rows(const float* Q, const float* K, const float* V,
                                               int ld, float* C, int ldc, int A, int L, int H,
                                               int dh, float scale, float* P = nullptr) {
  // CP threads per (AST, head, query row) when the block has room: each
  // recomputes the L scores and owns dh/CP context columns
  const int CP = 1;  // (2-4 measured slower: the duplicated score chains dominate)
  const int jobs = A * H * L * CP;
  for (int job = threadIdx.x; job < jobs; job += blockDim.x) {
    const int cp = job % CP, q_job = job / CP;
    const int i = q_job % L;
    const int h = (q_job / L) % H;
    const int a = q_job / (L * H);
    const float* q = Q + (a * L + i) * ld + h * dh;
    float p[TPCB_MAX_LEAF];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < TPCB_MAX_LEAF; ++j) {
      if (j < L) {
        const float* k = K + (a * L + j) * ld + h * dh;
        float s0 = 0.f, s1 = 0.f;
        int c = 0;
        for (; c + 1 < dh; c += 2) {
          s0 = fmaf(q[c], k[c], s0);
          s1 = fmaf(q[c + 1], k[c + 1], s1);
        }
        if (c < dh) s0 = fmaf(q[c], k[c], s0);
        float s = (s0 + s1) * scale;
        p[j] = s;
        m = fmaxf(m, s);
      }
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < TPCB_MAX_LEAF; ++j) {
      if (j < L) {
        p[j] = expf(p[j] - m);
        sum += p[j];
      }
    }
    const float inv = 1.f / sum;
#pragma unroll
    for (int j = 0; j < TPCB_MAX_LEAF; ++j)
      if (j < L) p[j] = p[j] / sum;
    (void)inv;
    if (P && cp == 0) {
      float* pp = P + ((a * H + h) * L + i) * L;
#pragma unroll
      for (int j = 0; j < TPCB_MAX_LEAF; ++j)
        if (j < L) pp[j] = p[j];
    }
    float* c_out = C + (a * L + i) * ldc + h * dh;
    const int cw = dh / CP;
    for (int c = cp * cw; c < (cp + 1) * cw; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < TPCB_MAX_LEAF; ++j)
        if (j < L) acc = fmaf(p[j], V[(a * L + j) * ld + h * dh + c], acc);
      c_out[c] = acc;
    }
  }
}

// z_x[a, e] = b[e] + Σ_{l<L, j<d} H[a*L + l, j] · W[l*d + j, e]
// (flatten row-major then leaf_embed.{L}, costmodel.py:213-216).
// Jobs = (AST, 4-column group, leaf position l); the L per-position partials
// are summed in l order through `scratch` (A·L·de floats).  The summation
// order depends only on L, never on the batch (the reference's exact batch
// equivariance, test_costmodel.py:73-80).  Needs de % 4 == 0 and a 16-byte
// aligned W, else the one-thread-per-output form below.
__device__ __forceinline__ void leaf_embed_rows(const float* Hs, int ld, int A, int L, int d,
                                                const float* __restrict__ W,
                                                const float* __restrict__ b, int de, float* Z,
                                                int ldz, float* scratch) {
  if ((de & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0) {
    const int ncg = de >> 2;
    const int S = L;
    for (int job = threadIdx.x; job < S * A * ncg; job += blockDim.x) {
      const int cg = job % ncg, a = (job / ncg) % A, sl = job / (ncg * A);
      const int l0 = sl * L / S, l1 = (sl + 1) * L / S;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int l = l0; l < l1; ++l) {
        const float* h = Hs + (a * L + l) * ld;
        const float4* w = reinterpret_cast<const float4*>(W + (size_t)l * d * de) + cg;
#pragma unroll 4
        for (int j = 0; j < d; ++j) {
          const float x = h[j];
          const float4 w4 = __ldg(w + (size_t)j * ncg);
          acc.x = fmaf(x, w4.x, acc.x);
          acc.y = fmaf(x, w4.y, acc.y);
          acc.z = fmaf(x, w4.z, acc.z);
          acc.w = fmaf(x, w4.w, acc.w);
        }
      }
      *reinterpret_cast<float4*>(scratch + (sl * A + a) * de + 4 * cg) = acc;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < A * de; idx += blockDim.x) {
      const int a = idx / de, e = idx - a * de;
      float v = __ldg(b + e);
      for (int sl = 0; sl < S; ++sl) v += scratch[(sl * A + a) * de + e];
      Z[a * ldz + e] = v;
    }
    return;
  }
  for (int job = threadIdx.x; job < A * de; job += blockDim.x) {
    const int e = job % de, a = job / de;
    float acc = __ldg(b + e);
    for (int l = 0; l < L; ++l) {
      const float* h = Hs + (a * L + l) * ld;
      const float* w = W + (size_t)l * d * de + e;
      for (int j = 0; j < d; ++j) acc = fmaf(h[j], __ldg(w + (size_t)j * de), acc);
    }
    Z[a * ldz + e] = acc;
  }
}

// ---------------------------------------------------------------------------
// backward helpers
// ---------------------------------------------------------------------------

// first ? G[i] = v : G[i] += v — gradient slots of one CTA are written by the
// first work item that touches them and accumulated afterwards (fixed order).
__device__ __forceinline__ void gstore(float* G, size_t i, float v, bool first) {
  if (first)
    G[i] = v;
  else
    G[i] += v;
}

// G[k*N + n] (+)= Σ_r X[r, k] · dY[r, n]   (weight gradient, nn.py:30-34)
__device__ __forceinline__ void wgrad_rows(const float* X, int ldx, const float* dY, int ldy,
                                           int R, int K, int N, float* G, bool first) {
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e - k * N;
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc = fmaf(X[r * ldx + k], dY[r * ldy + n], acc);
    gstore(G, e, acc, first);
  }
}

// G[n] (+)= Σ_r dY[r, n] (· S[r, n] when S is given)   (bias / LN gains)
__device__ __forceinline__ void colsum_rows(const float* dY, int ldy, int R, int N, float* G,
                                            bool first, const float* S = nullptr, int lds = 0) {
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += S ? dY[r * ldy + n] * S[r * lds + n] : dY[r * ldy + n];
    gstore(G, n, acc, first);
  }
}

// LayerNorm backward (nn.py:57-66): dX = inv (gx - mean(gx) - xhat mean(gx xhat)),
// gx = dY ⊙ g.  One warp per row.
__device__ __forceinline__ void layernorm_back_rows(const float* dY, int ldy, const float* Xh,
                                                    int ldh, const float* inv, int R, int d,
                                                    const float* __restrict__ g, float* dX,
                                                    int ldx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float inv_d = 1.f / (float)d;
  for (int r = w; r < R; r += nw) {
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane; c < d; c += 32) {
      const float gx = dY[r * ldy + c] * __ldg(g + c);
      s1 += gx;
      s2 = fmaf(gx, Xh[r * ldh + c], s2);
    }
    const float m1 = warp_sum(s1) * inv_d, m2 = warp_sum(s2) * inv_d;
    const float iv = inv[r];
    for (int c = lane; c < d; c += 32) {
      const float gx = dY[r * ldy + c] * __ldg(g + c);
      dX[r * ldx + c] = iv * (gx - m1 - Xh[r * ldh + c] * m2);
    }
  }
}

// Y[r, c] = g[c] · Xh[r, c] + b[c]  (recompute an LN output from its cache)
__device__ __forceinline__ void ln_apply_rows(const float* Xh, int ldh, int R, int d,
                                              const float* __restrict__ g,
                                              const float* __restrict__ b, float* Y, int ldy) {
  for (int e = threadIdx.x; e < R * d; e += blockDim.x) {
    const int r = e / d, c = e - r * d;
    Y[r * ldy + c] = fmaf(__ldg(g + c), Xh[r * ldh + c], __ldg(b + c));
  }
}

// Attention backward for A ASTs × H heads (nn.py:99-120) given the cached
// probabilities P and dCtx: dP = dCtx Vᵀ, dV = Pᵀ dCtx,
// dS = P ⊙ (dP − Σ_j dP P) · scale, dQ = dS K, dK = dSᵀ Q.
// Uses S as scratch for dS (same layout as P).
__device__ __forceinline__ void attention_back_rows(const float* Q, const float* K,
                                                    const float* V, int ld, const float* P,
                                                    const float* dC, int ldc, float* dQ,
                                                    float* dK, float* dV, float* S, int A, int L,
                                                    int H, int dh, float scale) {
  // dS rows: one thread per (a, h, i)
  for (int job = threadIdx.x; job < A * H * L; job += blockDim.x) {
    const int i = job % L, h = (job / L) % H, a = job / (L * H);
    const float* pp = P + ((a * H + h) * L + i) * L;
    const float* dc = dC + (a * L + i) * ldc + h * dh;
    float dp[TPCB_MAX_LEAF];
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < TPCB_MAX_LEAF; ++j) {
      if (j < L) {
        const float* v = V + (a * L + j) * ld + h * dh;
        float s = 0.f;
        for (int c = 0; c < dh; ++c) s = fmaf(dc[c], v[c], s);
        dp[j] = s;
        dot = fmaf(s, pp[j], dot);
      }
    }
    float* ss = S + ((a * H + h) * L + i) * L;
#pragma unroll
    for (int j = 0; j < TPCB_MAX_LEAF; ++j)
      if (j < L) ss[j] = pp[j] * (dp[j] - dot) * scale;
  }
  __syncthreads();
  // dQ[i] = Σ_j dS[i,j] K[j];  dK[j] = Σ_i dS[i,j] Q[i];  dV[j] = Σ_i P[i,j] dC[i]
  for (int e = threadIdx.x; e < A * L * H * dh; e += blockDim.x) {
    const int c = e % dh, h = (e / dh) % H, i = (e / (dh * H)) % L, a = e / (dh * H * L);
    const float* sr = S + (a * H + h) * L * L;
    const float* pr = P + (a * H + h) * L * L;
    float q = 0.f, k = 0.f, v = 0.f;
    for (int j = 0; j < L; ++j) {
      const int rj = (a * L + j) * ld + h * dh + c;
      q = fmaf(sr[i * L + j], K[rj], q);
      k = fmaf(sr[j * L + i], Q[rj], k);
      v = fmaf(pr[j * L + i], dC[(a * L + j) * ldc + h * dh + c], v);
    }
    const int ri = (a * L + i) * ld + h * dh + c;
    dQ[ri] = q;
    dK[ri] = k;
    dV[ri] = v;
  }
}

}  // namespace tpcb
