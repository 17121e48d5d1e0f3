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
constexpr int kTrainThreads = 512;  // threads per training CTA

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

// stage W [K × N] (row-major, global) into dst with row stride stage_ld(N);
// chunk indices advance incrementally (no per-element integer division)
static __device__ __noinline__ void stage_matrix(const float* __restrict__ W, int K, int N,
                                                 float* dst) {
  const int ld = stage_ld(N);
  const int nt = blockDim.x;
  if ((N & 3) == 0 && (reinterpret_cast<uintptr_t>(W) & 15) == 0) {
    const int n4 = N >> 2;
    const int sk = nt / n4, sc = nt - sk * n4;
    int k = threadIdx.x / n4, c4 = threadIdx.x - k * n4;
    for (; k < K;) {
      cp_async16(dst + k * ld + 4 * c4, W + (size_t)k * N + 4 * c4);
      c4 += sc;
      k += sk;
      if (c4 >= n4) {
        c4 -= n4;
        ++k;
      }
    }
  } else {
    const int sk = nt / N, sc = nt - sk * N;
    int k = threadIdx.x / N, c = threadIdx.x - k * N;
    for (; k < K;) {
      cp_async4(dst + k * ld + c, W + (size_t)k * N + c);
      c += sc;
      k += sk;
      if (c >= N) {
        c -= N;
        ++k;
      }
    }
  }
}

// out[r, c] = act(bias[c] + Σ_i A[r, i] · w(c, i)) + Res[r, c]
//   FWD:   w(c, i) = SW[i * ldw + c]     (C = staged columns, I = staged rows)
//   TRANS: w(c, i) = SW[c * ldw + i]     (C = staged rows, I = staged columns)
// with ldw = stage_ld(TRANS ? I : C).  Rows of A: stride lda (multiple of 4,
// 16-B aligned) when I % 4 == 0.  Two schedules: when R·C fills the block,
// threads split the rows (each thread: one column, full inner dimension, no
// reduction); otherwise (the R = 1 head vectors) the inner dimension is split
// and partials go through `scratch` (≥ 256·R floats).  Ends with a barrier.
template <bool TRANS>
__device__ __forceinline__ void mm_body(const float* A, int lda, const float* SW, int R, int I,
                                        int C, const float* __restrict__ bias, bool relu,
                                        const float* Res, int ldr, float* out, int ldo,
                                        float* scratch) {
  constexpr int NT = kTrainThreads;
  const int ldw = stage_ld(TRANS ? I : C);
  const bool vec = (I & 3) == 0 && (lda & 3) == 0;
  if (R * C >= 128 || I < 16) {
    const int RG = C >= NT ? 1 : NT / C;  // row groups
    for (int t = threadIdx.x; t < C * RG; t += NT) {
      const int c = t % C, rg = t / C;
      if (rg >= R) continue;
      const float bc = bias ? __ldg(bias + c) : 0.f;
      for (int r0 = rg; r0 < R; r0 += 4 * RG) {  // up to 4 rows per pass: r0, r0+RG, ...
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const int nr = min(4, (R - r0 + RG - 1) / RG);
        if (vec) {
#pragma unroll 4
          for (int i = 0; i < I; i += 4) {
            float4 w;
            if (TRANS) {
              w = *reinterpret_cast<const float4*>(SW + c * ldw + i);
            } else {
              const float* s = SW + i * ldw + c;
              w = make_float4(s[0], s[ldw], s[2 * ldw], s[3 * ldw]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (j < nr) {
                const float4 x = *reinterpret_cast<const float4*>(A + (r0 + j * RG) * lda + i);
                acc[j] = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc[j]))));
              }
            }
          }
        } else {
          for (int i = 0; i < I; ++i) {
            const float w = TRANS ? SW[c * ldw + i] : SW[i * ldw + c];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nr) acc[j] = fmaf(A[(r0 + j * RG) * lda + i], w, acc[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nr) {
            const int r = r0 + j * RG;
            float v = acc[j] + bc;
            if (relu) v = fmaxf(v, 0.f);
            if (Res) v += Res[r * ldr + c];
            out[r * ldo + c] = v;
          }
        }
      }
    }
    __syncthreads();
    return;
  }
  // split-K (R·C < 128 and I ≥ 16)
  int G = NT / C;
  if (G > I / 4) G = I / 4;
  if (G < 1) G = 1;
  const int slice = (((I + G - 1) / G) + 3) & ~3;
  for (int t = threadIdx.x; t < C * G; t += NT) {
    const int c = t % C, g = t / C;
    const int i0 = g * slice, i1 = min(I, i0 + slice);
    for (int r = 0; r < R; ++r) {
      float acc = 0.f;
      const float* a = A + r * lda;
      if (vec) {
        for (int i = i0; i < i1; i += 4) {
          float4 w;
          if (TRANS) {
            w = *reinterpret_cast<const float4*>(SW + c * ldw + i);
          } else {
            const float* s = SW + i * ldw + c;
            w = make_float4(s[0], s[ldw], s[2 * ldw], s[3 * ldw]);
          }
          const float4 x = *reinterpret_cast<const float4*>(a + i);
          acc = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc))));
        }
      } else {
        for (int i = i0; i < i1; ++i) acc = fmaf(a[i], TRANS ? SW[c * ldw + i] : SW[i * ldw + c], acc);
      }
      scratch[(g * R + r) * C + c] = acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * C; e += NT) {
    const int r = e / C, c = e - r * C;
    float v = bias ? __ldg(bias + c) : 0.f;
    for (int g = 0; g < G; ++g) v += scratch[(g * R + r) * C + c];
    if (relu) v = fmaxf(v, 0.f);
    if (Res) v += Res[r * ldr + c];
    out[r * ldo + c] = v;
  }
  __syncthreads();
}

// one out-of-line, fully specialised copy per (I, C) of the desk model
template <bool TRANS, int I, int C>
static __device__ __noinline__ void mm_fixed(const float* A, int lda, const float* SW, int R,
                                             const float* bias, bool relu, const float* Res,
                                             int ldr, float* out, int ldo, float* scratch) {
  mm_body<TRANS>(A, lda, SW, R, I, C, bias, relu, Res, ldr, out, ldo, scratch);
}

template <bool TRANS>
static __device__ __noinline__ void mm_generic(const float* A, int lda, const float* SW, int R,
                                               int I, int C, const float* bias, bool relu,
                                               const float* Res, int ldr, float* out, int ldo,
                                               float* scratch) {
  mm_body<TRANS>(A, lda, SW, R, I, C, bias, relu, Res, ldr, out, ldo, scratch);
}

template <bool TRANS>
__device__ __forceinline__ void small_mm(const float* A, int lda, const float* SW, int ldw, int R,
                                         int I, int C, const float* __restrict__ bias,
                                         bool relu, const float* Res, int ldr, float* out,
                                         int ldo, float* scratch) {
  (void)ldw;
#define TPCB_MM_CASE(II, CC)                                                           \
  if (I == II && C == CC) {                                                            \
    mm_fixed<TRANS, II, CC>(A, lda, SW, R, bias, relu, Res, ldr, out, ldo, scratch);   \
    return;                                                                            \
  }
  // the encoder shapes of the desk model get specialised copies; the rest
  // (head vectors, other configs) share one generic body (I-cache budget)
  TPCB_MM_CASE(64, 64)
  TPCB_MM_CASE(64, 128)
  TPCB_MM_CASE(128, 64)
#undef TPCB_MM_CASE
  mm_generic<TRANS>(A, lda, SW, R, I, C, bias, relu, Res, ldr, out, ldo, scratch);
}

// G[k*N + n] (+)= Σ_r X[r, k] · dY[r, n]  — weight gradient into the CTA's
// gradient slot (global), 4 columns per thread with 128-bit stores; indices
// advance incrementally.
static __device__ __noinline__ void wgrad_v(const float* X, int ldx, const float* dY, int ldy,
                                            int R, int K, int N, float* G, bool first) {
  const int nt = blockDim.x;
  if ((N & 3) == 0 && (ldy & 3) == 0 && ((reinterpret_cast<uintptr_t>(G) & 15) == 0)) {
    const int n4 = N >> 2;
    const int sk = nt / n4, sc = nt - sk * n4;
    int k = threadIdx.x / n4, c4 = threadIdx.x - k * n4;
    for (; k < K;) {
      const int n = 4 * c4;
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
      c4 += sc;
      k += sk;
      if (c4 >= n4) {
        c4 -= n4;
        ++k;
      }
    }
  } else {
    for (int e = threadIdx.x; e < K * N; e += nt) {
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
