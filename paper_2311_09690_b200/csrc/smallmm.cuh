// Small-M GEMMs over shared-memory-staged weights (training kernel).
//
// The training step works on one sample at a time (L ≤ 16 rows), so every
// product is a skinny [L × I] · [I × C].  Weights are staged into shared
// memory by cp.async (4-byte granules, any layout) one op ahead of their use
// (WStream), with an odd row stride ldw = C_stage + 1 so both the forward
// product (w(c,i) = W[i][c]) and the transposed product of the backward
// (w(c,i) = W[c][i]) read bank-conflict-free — no transposed copy of the
// weights is kept in global memory.  A thread owns one output column and a
// slice of the inner dimension, holds its weights in registers and sweeps
// the (≤16) rows with broadcast 128-bit loads of the activations.
#pragma once

#include "common.cuh"

namespace tpcb {

constexpr int kMaxRows = TPCB_MAX_LEAF;

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// staged stride of a weight matrix with N columns: 16-byte rows, and an odd
// multiple of 4 floats so 8 consecutive 128-bit row reads hit distinct banks
__host__ __device__ __forceinline__ int stage_ld(int N) { return ((N + 3) & ~3) + 4; }

// stage W [K × N] (row-major, global) into dst with row stride stage_ld(N)
static __device__ __noinline__ void stage_matrix(const float* __restrict__ W, int K, int N, float* dst) {
  const int ld = stage_ld(N);
  if ((N & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0) {
    const int n4 = N >> 2;
    const int total = K * n4;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int k = t / n4, c4 = t - k * n4;
      cp_async16(dst + k * ld + 4 * c4, W + (size_t)k * N + 4 * c4);
    }
  } else {
    const int total = K * N;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int k = t / N, c = t - k * N;
      cp_async4(dst + k * ld + c, W + (size_t)k * N + c);
    }
  }
}

// out[r, c] = act(bias(c) + Σ_i A[r, i] · w(c, i)) + Res[r, c]
//   FWD:   w(c, i) = SW[i * ldw + c]     (C = staged columns, I = staged rows)
//   TRANS: w(c, i) = SW[c * ldw + i]     (C = staged rows, I = staged columns)
// Rows of A: stride lda (multiple of 4, 16-B aligned base) when I % 4 == 0.
// `scratch` (≥ blockDim·R floats) holds split-K partials.  Ends with a barrier.
template <bool TRANS>
static __device__ __noinline__ void small_mm(const float* A, int lda, const float* SW, int ldw, int R,
                                         int I, int C, const float* __restrict__ bias,
                                         bool relu, const float* Res, int ldr, float* out,
                                         int ldo, float* scratch) {
  const int nt = blockDim.x;
  int G = nt / C;
  if (G < 1) G = 1;
  const int maxg = (I + 3) / 4;
  if (G > maxg) G = maxg;
  const int slice = (((I + G - 1) / G) + 3) & ~3;
  const bool vec = (I & 3) == 0 && (lda & 3) == 0;
  for (int t = threadIdx.x; t < C * G; t += nt) {
    const int c = t % C, g = t / C;
    const int i0 = g * slice, i1 = min(I, i0 + slice);
    for (int r0 = 0; r0 < R; r0 += 4) {  // rows in groups of 4 (R is usually ≤ 6)
      const int nr = min(4, R - r0);
      const float* a0 = A + r0 * lda;
      float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
      if (vec) {
        for (int i = i0; i < i1; i += 4) {
          float4 w;
          if (TRANS) {
            w = *reinterpret_cast<const float4*>(SW + c * ldw + i);
          } else {
            const float* s = SW + i * ldw + c;
            w = make_float4(s[0], s[ldw], s[2 * ldw], s[3 * ldw]);
          }
          float4 x = *reinterpret_cast<const float4*>(a0 + i);
          acc0 = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc0))));
          if (nr > 1) {
            x = *reinterpret_cast<const float4*>(a0 + lda + i);
            acc1 = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc1))));
          }
          if (nr > 2) {
            x = *reinterpret_cast<const float4*>(a0 + 2 * lda + i);
            acc2 = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc2))));
          }
          if (nr > 3) {
            x = *reinterpret_cast<const float4*>(a0 + 3 * lda + i);
            acc3 = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc3))));
          }
        }
      } else {
        for (int i = i0; i < i1; ++i) {
          const float w = TRANS ? SW[c * ldw + i] : SW[i * ldw + c];
          acc0 = fmaf(a0[i], w, acc0);
          if (nr > 1) acc1 = fmaf(a0[lda + i], w, acc1);
          if (nr > 2) acc2 = fmaf(a0[2 * lda + i], w, acc2);
          if (nr > 3) acc3 = fmaf(a0[3 * lda + i], w, acc3);
        }
      }
      const float accs[4] = {acc0, acc1, acc2, acc3};
      if (G == 1) {
        const float bc = bias ? __ldg(bias + c) : 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nr) {
            const int r = r0 + j;
            float v = accs[j] + bc;
            if (relu) v = fmaxf(v, 0.f);
            if (Res) v += Res[r * ldr + c];
            out[r * ldo + c] = v;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nr) scratch[(g * R + r0 + j) * C + c] = accs[j];
      }
    }
  }
  __syncthreads();
  if (G > 1) {
    for (int e = threadIdx.x; e < R * C; e += nt) {
      const int r = e / C, c = e - r * C;
      float v = bias ? __ldg(bias + c) : 0.f;
      for (int g = 0; g < G; ++g) v += scratch[(g * R + r) * C + c];
      if (relu) v = fmaxf(v, 0.f);
      if (Res) v += Res[r * ldr + c];
      out[r * ldo + c] = v;
    }
    __syncthreads();
  }
}

// G[k*N + n] (+)= Σ_r X[r, k] · dY[r, n]  — weight gradient into the CTA's
// gradient slot (global), 4 columns per thread with 128-bit stores.
static __device__ __noinline__ void wgrad_v(const float* X, int ldx, const float* dY, int ldy, int R,
                                        int K, int N, float* G, bool first) {
  if ((N & 3) == 0 && (ldy & 3) == 0 && ((reinterpret_cast<uintptr_t>(G) & 15) == 0)) {
    const int n4 = N >> 2;
    for (int e = threadIdx.x; e < K * n4; e += blockDim.x) {
      const int k = e / n4, n = (e - k * n4) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < R; ++r) {
        const float x = X[r * ldx + k];
        const float4 d = *reinterpret_cast<const float4*>(dY + r * ldy + n);
        acc.x = fmaf(x, d.x, acc.x);
        acc.y = fmaf(x, d.y, acc.y);
        acc.z = fmaf(x, d.z, acc.z);
        acc.w = fmaf(x, d.w, acc.w);
      }
      float4* gp = reinterpret_cast<float4*>(G + (size_t)k * N + n);
      if (!first) {
        const float4 o = *gp;
        acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
      }
      *gp = acc;
    }
  } else {
    for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
      const int k = e / N, n = e - k * N;
      float acc = 0.f;
      for (int r = 0; r < R; ++r) acc = fmaf(X[r * ldx + k], dY[r * ldy + n], acc);
      if (first)
        G[e] = acc;
      else
        G[e] += acc;
    }
  }
}

}  // namespace tpcb
