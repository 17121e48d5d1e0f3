// Training step, v3 ("warp-group per sample"): the latency-optimised path for
// configurations whose widths are multiples of 32 (the desk model and up).
//
// Same arithmetic as train.cu (reference: costmodel.backward,
// costmodel.py:529-570; nn.py:30-120), different execution model.  A training
// step is a chain of ~40 dependent, tiny GEMMs per sample (≤16 rows × 64-128
// columns), so its time is set by per-op latency, not FLOPs.  Here a CTA is
//   * kG compute warps that own one sample end to end (activations in shared
//     memory, ops split by output column, a named barrier over the kG warps
//     between dependent ops — never a block-wide barrier), and
//   * one producer warp that streams every weight matrix the sample consumes,
//     in consumption order, into a double-buffered shared-memory stage with
//     bulk async copies (cp.async.bulk, one per padded row) tracked by
//     mbarriers: full[b] (transaction bytes) releases a buffer to the
//     compute warps, empty[b] (kG arrivals) hands it back to the producer.
// The compute warps therefore never issue copies or wait on block barriers;
// the weights of op i+1 are in flight while op i computes.  Gradients go to
// the CTA's slot as in v2 (optim.cu reduces slots in fixed order).
#include <cmath>

#include "async.cuh"
#include "cmd.cuh"
#include "common.cuh"
#include "train.cuh"

namespace tpcb {

__device__ long long* g_trace3 = nullptr;

int set_train3_trace(long long* d) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace3, &d, sizeof(d)));
  return TPCB_OK;
}

namespace {

constexpr int kG = 8;                 // compute warps per sample
constexpr int kGT = 32 * kG;          // compute threads
constexpr int kThreads3 = kGT + 32;   // + producer warp
constexpr int kBarGroup = 1;          // named barrier id of the compute group

__device__ __forceinline__ void gbar() { group_bar(kBarGroup, kGT); }

__host__ __device__ inline int stage_ld3(int N) { return N == 1 ? 1 : N + 4; }

// out[r, c] = act(bias[c] + Σ_i A[r, i] · w(c, i)) + Res[r, c] over the compute
// group: 32-column blocks round-robin over the kG warps, lane = column, rows
// in register groups of 4, activations read with broadcast 128-bit loads.
//   FWD   w(c, i) = SW[i·ldw + c]    TRANS  w(c, i) = SW[c·ldw + i]
template <bool TRANS>
__device__ __noinline__ void gmm(const float* A, int lda, const float* SW, int ldw, int R, int I,
                                 int C, const float* __restrict__ bias, bool relu,
                                 const float* Res, int ldr, float* out, int ldo) {
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const bool vec = (I & 3) == 0 && (lda & 3) == 0;
  for (int cb = 32 * g; cb < C; cb += kGT) {
    const int c = cb + lane;
    const bool cv = c < C;
    const float bc = (bias != nullptr && cv) ? __ldg(bias + c) : 0.f;
    for (int r0 = 0; r0 < R; r0 += 4) {
      const int nr = min(4, R - r0);
      const float* a0 = A + r0 * lda;
      float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
      if (vec) {
#pragma unroll 4
        for (int i = 0; i < I; i += 4) {
          float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
          if (cv) {
            if (TRANS) {
              w = *reinterpret_cast<const float4*>(SW + c * ldw + i);
            } else {
              const float* s = SW + i * ldw + c;
              w = make_float4(s[0], s[ldw], s[2 * ldw], s[3 * ldw]);
            }
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
        for (int i = 0; i < I; ++i) {
          const float w = cv ? (TRANS ? SW[c * ldw + i] : SW[i * ldw + c]) : 0.f;
          acc0 = fmaf(a0[i], w, acc0);
          if (nr > 1) acc1 = fmaf(a0[lda + i], w, acc1);
          if (nr > 2) acc2 = fmaf(a0[2 * lda + i], w, acc2);
          if (nr > 3) acc3 = fmaf(a0[3 * lda + i], w, acc3);
        }
      }
      if (cv) {
        const float accs[4] = {acc0, acc1, acc2, acc3};
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
      }
    }
  }
}

// G[k·N + n] (+)= Σ_r X[r, k] · dY[r, n] over the compute group (float4 per
// thread along n, 128-bit global stores)
__device__ __noinline__ void gwgrad(const float* X, int ldx, const float* dY, int ldy, int R, int K,
                                    int N, float* G, bool first) {
  const int t = threadIdx.x;
  if ((N & 3) == 0 && (ldy & 3) == 0) {
    const int n4 = N >> 2, tot = K * n4;
    for (int e = t; e < tot; e += kGT) {
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
    for (int e = t; e < K * N; e += kGT) {
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

// G[n] (+)= Σ_r dY[r, n] (· S[r, n])
__device__ __noinline__ void gcolsum(const float* dY, int ldy, int R, int N, float* G, bool first,
                                     const float* S, int lds) {
  for (int n = threadIdx.x; n < N; n += kGT) {
    float acc = 0.f;
    for (int r = 0; r < R; ++r) acc += S ? dY[r * ldy + n] * S[r * lds + n] : dY[r * ldy + n];
    if (first)
      G[n] = acc;
    else
      G[n] += acc;
  }
}

// LayerNorm rows (nn.py:48-54), warp per row
__device__ __noinline__ void gln(const float* X, int ldx, float* Y, int ldy, int R, int d,
                                 const float* __restrict__ g, const float* __restrict__ b,
                                 float* xhat, int ldh, float* inv_out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float inv_d = 1.f / (float)d;
  for (int r = w; r < R; r += kG) {
    const float* x = X + r * ldx;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += x[c];
    const float mu = warp_sum(s) * inv_d;
    float v = 0.f;
    for (int c = lane; c < d; c += 32) {
      const float t = x[c] - mu;
      v = fmaf(t, t, v);
    }
    const float inv = 1.f / sqrtf(warp_sum(v) * inv_d + 1e-5f);
    for (int c = lane; c < d; c += 32) {
      const float xh = (x[c] - mu) * inv;
      xhat[r * ldh + c] = xh;
      Y[r * ldy + c] = fmaf(__ldg(g + c), xh, __ldg(b + c));
    }
    if (lane == 0) inv_out[r] = inv;
  }
}

// LayerNorm backward rows (nn.py:57-66)
__device__ __noinline__ void gln_back(const float* dY, int ldy, const float* Xh, int ldh,
                                      const float* inv, int R, int d, const float* __restrict__ g,
                                      float* dX, int ldx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float inv_d = 1.f / (float)d;
  for (int r = w; r < R; r += kG) {
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

__device__ __noinline__ void gln_apply(const float* Xh, int ldh, int R, int d,
                                       const float* __restrict__ g, const float* __restrict__ b,
                                       float* Y, int ldy) {
  for (int e = threadIdx.x; e < R * d; e += kGT) {
    const int r = e / d, c = e - r * d;
    Y[r * ldy + c] = fmaf(__ldg(g + c), Xh[r * ldh + c], __ldg(b + c));
  }
}

// attention of one sample (nn.py:79-96); ends with a group barrier
__device__ __noinline__ void gattn_fwd(const float* Q, const float* K, const float* V, int ld,
                                       float* C, int L, int H, int dh, float scale, float* P) {
  const int LL = L * L;
  for (int e = threadIdx.x; e < H * LL; e += kGT) {
    const int h = e / LL, ij = e - h * LL, i = ij / L, j = ij - i * L;
    const float* q = Q + i * ld + h * dh;
    const float* k = K + j * ld + h * dh;
    float s = 0.f;
    for (int c = 0; c < dh; c += 4) {
      const float4 a = *reinterpret_cast<const float4*>(q + c);
      const float4 b = *reinterpret_cast<const float4*>(k + c);
      s = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, s))));
    }
    P[e] = s * scale;
  }
  gbar();
  for (int e = threadIdx.x; e < H * L; e += kGT) {
    float* p = P + e * L;
    float m = -INFINITY;
    for (int j = 0; j < L; ++j) m = fmaxf(m, p[j]);
    float sum = 0.f;
    for (int j = 0; j < L; ++j) {
      const float v = expf(p[j] - m);
      p[j] = v;
      sum += v;
    }
    for (int j = 0; j < L; ++j) p[j] = p[j] / sum;
  }
  gbar();
  const int D = H * dh;
  for (int e = threadIdx.x; e < L * D; e += kGT) {
    const int i = e / D, f = e - i * D, h = f / dh;
    const float* p = P + (h * L + i) * L;
    float acc = 0.f;
    for (int j = 0; j < L; ++j) acc = fmaf(p[j], V[j * ld + f], acc);
    C[i * ld + f] = acc;
  }
  gbar();
}

// attention backward (nn.py:99-120); ends with a group barrier
__device__ __noinline__ void gattn_bwd(const float* Q, const float* K, const float* V, int ld,
                                       const float* P, const float* dC, float* dQ, float* dK,
                                       float* dV, float* S, int L, int H, int dh, float scale) {
  const int LL = L * L;
  for (int e = threadIdx.x; e < H * LL; e += kGT) {
    const int h = e / LL, ij = e - h * LL, i = ij / L, j = ij - i * L;
    const float* a = dC + i * ld + h * dh;
    const float* b = V + j * ld + h * dh;
    float s = 0.f;
    for (int c = 0; c < dh; c += 4) {
      const float4 x = *reinterpret_cast<const float4*>(a + c);
      const float4 y = *reinterpret_cast<const float4*>(b + c);
      s = fmaf(x.x, y.x, fmaf(x.y, y.y, fmaf(x.z, y.z, fmaf(x.w, y.w, s))));
    }
    S[e] = s;
  }
  gbar();
  for (int e = threadIdx.x; e < H * L; e += kGT) {
    float* s = S + e * L;
    const float* p = P + e * L;
    float dot = 0.f;
    for (int j = 0; j < L; ++j) dot = fmaf(s[j], p[j], dot);
    for (int j = 0; j < L; ++j) s[j] = p[j] * (s[j] - dot) * scale;
  }
  gbar();
  const int D = H * dh;
  for (int e = threadIdx.x; e < L * D; e += kGT) {
    const int r = e / D, f = e - r * D, h = f / dh;
    const float* s = S + h * LL;
    const float* p = P + h * LL;
    float q = 0.f, k = 0.f, v = 0.f;
    for (int j = 0; j < L; ++j) {
      q = fmaf(s[r * L + j], K[j * ld + f], q);
      k = fmaf(s[j * L + r], Q[j * ld + f], k);
      v = fmaf(p[j * L + r], dC[j * ld + f], v);
    }
    dQ[r * ld + f] = q;
    dK[r * ld + f] = k;
    dV[r * ld + f] = v;
  }
  gbar();
}

__device__ void decode_with_grad3(double e, const tpcb_boxcox& n, double* y, double* dy) {
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

__device__ double decode_plain3(double e, const tpcb_boxcox& n) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) return exp(t) - n.shift;
  return pow(n.lambda_bc * t + 1.0, 1.0 / n.lambda_bc) - n.shift;
}

__device__ __forceinline__ double sgn3(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

}  // namespace

// shared-memory plan of one v3 CTA (one sample of ≤ l_cap rows)
struct Plan3 {
  int R, ld, ldf;
  int oQ, oK, oV, oC, oX1, oX2, oF, oI1, oI2, oP, lstride;
  int X0, H0, Hout, T1, T2, dH, dA, dB, dQ, dK, dV, dF, S;
  int dv, zx, zv, zp, u, du0, du1, dzx, dzp, dzv, misc, cmd;
  int stage0, stage1, total;
};

bool v3_supported(const Model& M) {
  if (M.d % 32 || M.d_ff % 32 || M.dh % 4) return false;
  if (M.d_e % 4 || M.d_dev % 4) return false;
  for (int i = 0; i < M.n_dec; ++i)
    if (M.dec[i] % 4) return false;
  const int last = M.n_dec ? M.dec[M.n_dec - 1] : M.d_e;
  if ((last * 4) % 16) return false;  // dec.out staged as one contiguous copy
  if ((TPCB_DEV_FEAT * M.d_dev) % 4) return false;
  return true;
}

Plan3 make_plan3(const Model& M, int l_cap) {
  Plan3 p;
  const int R = (l_cap >= 1 && l_cap <= M.n_leaf_max) ? l_cap : M.n_leaf_max;
  p.R = R;
  p.ld = round4(M.d) + 4;
  p.ldf = round4(M.d_ff) + 4;
  const int blk = R * p.ld;
  int o = 0;
  p.oQ = o; o += blk;
  p.oK = o; o += blk;
  p.oV = o; o += blk;
  p.oC = o; o += blk;
  p.oX1 = o; o += blk;
  p.oX2 = o; o += blk;
  p.oF = o; o += R * p.ldf;
  p.oI1 = o; o += round4(R);
  p.oI2 = o; o += round4(R);
  p.oP = o; o += round4(M.n_heads * R * R);
  p.lstride = o;
  o = M.n_layers * p.lstride;
  p.X0 = o; o += R * 28;
  p.H0 = o; o += blk;
  p.Hout = o; o += blk;
  p.T1 = o; o += blk;
  p.T2 = o; o += blk;
  p.dH = o; o += blk;
  p.dA = o; o += blk;
  p.dB = o; o += blk;
  p.dQ = o; o += blk;
  p.dK = o; o += blk;
  p.dV = o; o += blk;
  p.dF = o; o += R * p.ldf;
  p.S = o; o += round4(M.n_heads * R * R);
  int uw = max(M.d_e, max(M.d_dev, M.d)), usum = round4(M.d_e);
  for (int i = 0; i < M.n_dec; ++i) {
    uw = max(uw, M.dec[i]);
    usum += round4(M.dec[i]);
  }
  uw = round4(uw);
  p.dv = o; o += 8;
  p.zx = o; o += round4(M.d_e);
  p.zv = o; o += round4(M.d_dev);
  p.zp = o; o += round4(M.d_e);
  p.u = o; o += usum;
  p.du0 = o; o += uw;
  p.du1 = o; o += uw;
  p.dzx = o; o += round4(M.d_e);
  p.dzp = o; o += round4(M.d_e);
  p.dzv = o; o += round4(M.d_dev);
  p.misc = o; o += 8;
  o = (o + 1) & ~1;
  p.cmd = o; o += 2 * cmd_scratch_doubles(M.d_e) + 8;
  int cap = 0;
  for (int L = 1; L <= R; ++L) {
    const int n = n_all_entries(M, L);
    for (int i = 0; i < n; ++i) {
      int K, N, off;
      entry_shape(M, L, i, &K, &N, &off);
      cap = max(cap, K * stage_ld3(N));
    }
  }
  o = (o + 7) & ~7;  // 32-byte aligned stage buffers
  p.stage0 = o; o += (cap + 7) & ~7;
  p.stage1 = o; o += (cap + 7) & ~7;
  p.total = o;
  return p;
}

namespace {

struct P3 {
  float *Q, *K, *V, *C, *X1, *X2, *F, *I1, *I2, *P;
};

__device__ __forceinline__ P3 lptr(float* sm, const Plan3& p, int li) {
  float* b = sm + li * p.lstride;
  return P3{b + p.oQ, b + p.oK, b + p.oV, b + p.oC, b + p.oX1,
            b + p.oX2, b + p.oF, b + p.oI1, b + p.oI2, b + p.oP};
}

__global__ void __launch_bounds__(kThreads3) train3_kernel(
    const __grid_constant__ Model M, const float* __restrict__ Pw, SampleSetDev src,
    SampleSetDev tgt, const int32_t* __restrict__ batch_all, const StepDesc* __restrict__ steps,
    int step, LossDev loss, int phase, const __grid_constant__ Plan3 tp,
    float* __restrict__ zall, float* __restrict__ partial, size_t slot_stride,
    uint32_t* __restrict__ touched, double* __restrict__ terms, double* __restrict__ scalars,
    float* __restrict__ pred_out, int32_t* status) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bars[4];  // full[2], empty[2]
  uint64_t* full = bars;
  uint64_t* empty = bars + 2;
  const StepDesc sd = steps[step];
  const int32_t* batch = batch_all + sd.off;
  const int n_src = sd.n_src, n_tgt = sd.n_tgt;
  const int n_all = n_src + (loss.use_cmd ? n_tgt : 0);
  const int ns_g = sd.ns_glob, nt_g = sd.nt_glob;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kG);
    mbar_init(&empty[1], kG);
    mbar_fence_init();
  }
  __syncthreads();
  float* buf[2] = {sm + tp.stage0, sm + tp.stage1};

  // ================================================================ producer
  if (warp == kG) {
    int J = 0;
    for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
      const bool is_t = w >= n_src;
      const SampleSetDev set = is_t ? tgt : src;
      const int L = set.n_leaf[batch[w]];
      if (L < 1 || L > tp.R) continue;  // consumers skip it too
      const int n_ent = phase == 0 ? n_fwd_entries(M, L) : n_all_entries(M, L);
      for (int j = 0; j < n_ent; ++j, ++J) {
        const int b = J & 1;
        if (J >= 2) mbar_wait(&empty[b], ((J >> 1) - 1) & 1);
        int K, N, off;
        entry_shape(M, L, j, &K, &N, &off);
        if (lane == 0) mbar_arrive_expect_tx(&full[b], (uint32_t)(K * N * 4));
        __syncwarp();
        const float* srcw = Pw + off;
        if (N == 1) {
          if (lane == 0) bulk_g2s(buf[b], srcw, (uint32_t)(K * 4), &full[b]);
        } else {
          const int ldw = N + 4;
          for (int k = lane; k < K; k += 32)
            bulk_g2s(buf[b] + k * ldw, srcw + (size_t)k * N, (uint32_t)(N * 4), &full[b]);
        }
      }
    }
    return;
  }

  // ========================================================== compute group
  const int ld = tp.ld, ldf = tp.ldf, d = M.d, H = M.n_heads, dh = M.dh, de = M.d_e;
  const float scale = 1.f / sqrtf((float)dh);
  float* G = partial + (size_t)blockIdx.x * slot_stride;
  uint32_t mask = 0;
  float* X0 = sm + tp.X0;
  float* H0 = sm + tp.H0;
  float* Hout = sm + tp.Hout;
  float* T1 = sm + tp.T1;
  float* T2 = sm + tp.T2;
  float* dH = sm + tp.dH;
  float* dA = sm + tp.dA;
  float* dB = sm + tp.dB;
  float* dQ = sm + tp.dQ;
  float* dK = sm + tp.dK;
  float* dV = sm + tp.dV;
  float* dF = sm + tp.dF;
  float* S = sm + tp.S;
  float* dv = sm + tp.dv;
  float* zx = sm + tp.zx;
  float* zv = sm + tp.zv;
  float* zp = sm + tp.zp;
  float* uall = sm + tp.u;
  float* misc = sm + tp.misc;
  double* cmds = reinterpret_cast<double*>(sm + tp.cmd);
  int uoff[TPCB_MAX_DEC + 1], uw[TPCB_MAX_DEC + 1];
  uoff[0] = 0;
  uw[0] = de;
  for (int j = 0; j < M.n_dec; ++j) {
    uoff[j + 1] = uoff[j] + round4(uw[j]);
    uw[j + 1] = M.dec[j];
  }
  const int nd = M.n_dec;
  int J = 0;  // weight-stream position (matches the producer)
  int ldw = 0;
  long long* trace = g_trace3;
  const bool rec = trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  auto acquire = [&](int N) -> const float* {
    const int b = J & 1;
    if (rec && J < 128) trace[2 * J] = clock64();
    mbar_wait(&full[b], (J >> 1) & 1);
    if (rec && J < 128) trace[2 * J + 1] = clock64();
    ldw = stage_ld3(N);
    return buf[b];
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[J & 1]);
    ++J;
  };

  for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
    const bool is_t = w >= n_src;
    const SampleSetDev set = is_t ? tgt : src;
    const int idx = batch[w];
    const int L = set.n_leaf[idx];
    if (L < 1 || L > tp.R) {
      if (threadIdx.x == 0) raise_status(status, TPCB_ERR_LEAF_COUNT);
      continue;
    }
    const float* xr = set.x + (size_t)set.ast_row[idx] * TPCB_FEAT_PAD;
    for (int e = threadIdx.x; e < L * TPCB_FEAT; e += kGT) {
      const int r = e / TPCB_FEAT, c = e - r * TPCB_FEAT;
      X0[r * 28 + c] = __ldg(xr + r * TPCB_FEAT_PAD + c);
    }
    if (threadIdx.x < TPCB_DEV_FEAT)
      dv[threadIdx.x] = __ldg(set.devfeat + (size_t)idx * TPCB_DEV_FEAT + threadIdx.x);
    gbar();
    // ------------------------------------------------------------ forward
    const float* W = acquire(d);
    gmm<false>(X0, 28, W, ldw, L, TPCB_FEAT, d, Pw + M.inb, false, nullptr, 0, H0, ld);
    release();
    gbar();
    const float* Hin = H0;
    for (int li = 0; li < M.n_layers; ++li) {
      const LayerOff& lo = M.layer[li];
      P3 c = lptr(sm, tp, li);
      W = acquire(d);
      gmm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bq, false, nullptr, 0, c.Q, ld);
      release();
      W = acquire(d);
      gmm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bk, false, nullptr, 0, c.K, ld);
      release();
      W = acquire(d);
      gmm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bv, false, nullptr, 0, c.V, ld);
      release();
      gbar();
      gattn_fwd(c.Q, c.K, c.V, ld, c.C, L, H, dh, scale, c.P);
      W = acquire(d);
      gmm<false>(c.C, ld, W, ldw, L, d, d, Pw + lo.bo, false, Hin, ld, T1, ld);
      release();
      gbar();
      gln(T1, ld, T2, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, c.X1, ld, c.I1);
      gbar();
      W = acquire(M.d_ff);
      gmm<false>(T2, ld, W, ldw, L, d, M.d_ff, Pw + lo.fhb, true, nullptr, 0, c.F, ldf);
      release();
      gbar();
      W = acquire(d);
      gmm<false>(c.F, ldf, W, ldw, L, M.d_ff, d, Pw + lo.fob, false, T2, ld, T1, ld);
      release();
      gbar();
      gln(T1, ld, Hout, ld, L, d, Pw + lo.ln2g, Pw + lo.ln2b, c.X2, ld, c.I2);
      gbar();
      Hin = Hout;
    }
    // head: z_x = b_L + Σ_l Hout[l] · W_L[l] (one staged chunk per leaf)
    for (int l = 0; l < L; ++l) {
      W = acquire(de);
      gmm<false>(Hout + l * ld, 0, W, ldw, 1, d, de, l == 0 ? Pw + M.leafb[L] : nullptr, false,
                 l == 0 ? nullptr : zx, 0, zx, 0);
      release();
      gbar();
    }
    W = acquire(M.d_dev);
    gmm<false>(dv, 8, W, ldw, 1, TPCB_DEV_FEAT, M.d_dev, Pw + M.devhb, true, nullptr, 0, zv, 0);
    release();
    gbar();
    W = acquire(de);
    gmm<false>(zv, 0, W, ldw, 1, M.d_dev, de, Pw + M.devpb, false, nullptr, 0, zp, 0);
    release();
    gbar();
    for (int e = threadIdx.x; e < de; e += kGT) uall[e] = zx[e] * zp[e];
    gbar();
    for (int j = 0; j < nd; ++j) {
      W = acquire(M.dec[j]);
      gmm<false>(uall + uoff[j], 0, W, ldw, 1, uw[j], M.dec[j], Pw + M.decb[j], true, nullptr, 0,
                 uall + uoff[j + 1], 0);
      release();
      gbar();
    }
    W = acquire(1);
    gmm<false>(uall + uoff[nd], 0, W, ldw, 1, uw[nd], 1, Pw + M.outb, false, nullptr, 0, misc, 0);
    release();
    gbar();
    const float pred = misc[0];
    const int zrow = is_t ? ns_g + sd.tgt_pos + (w - n_src) : sd.src_pos + w;
    if (phase == 0) {
      for (int e = threadIdx.x; e < de; e += kGT) zall[(size_t)zrow * de + e] = uall[e];
      gbar();
      continue;
    }
    // ------------------------------------------------------- loss gradient
    if (threadIdx.x == 0) {
      double dpred = 0.0;
      if (!is_t) {
        const double y = set.y[idx];
        const double dd = (double)pred - y;
        const double n = (double)sd.n_norm;
        double rel = 0.0, relg = 0.0;
        if (loss.mode != kLossMse) {
          if (loss.original) {
            const double y0 = decode_plain3(y, loss.norm);
            double p0, dp0;
            decode_with_grad3((double)pred, loss.norm, &p0, &dp0);
            const double r = p0 - y0;
            rel = fabs(r) / y0;
            relg = sgn3(r) * dp0 / (y0 * n);
          } else {
            const double den = y + loss.offset;
            rel = fabs(dd) / den;
            relg = sgn3(dd) / (den * n);
          }
        }
        if (loss.mode == kLossMse)
          dpred = 2.0 * dd / n;
        else if (loss.mode == kLossMape)
          dpred = relg;
        else
          dpred = 2.0 * dd / n + loss.lambda * relg;
        terms[2 * w] = dd * dd;
        terms[2 * w + 1] = rel;
        if (pred_out) pred_out[w] = pred;
      }
      misc[1] = (float)dpred;
    }
    gbar();
    // ------------------------------------------------------------ backward
    const bool fs = !(mask & 1u);
    const bool fl = !(mask & (1u << L));
    float* du = sm + tp.du0;
    float* du2 = sm + tp.du1;
    {
      const float dpred = misc[1];
      for (int cc = threadIdx.x; cc < uw[nd]; cc += kGT) {
        const float g0 = uall[uoff[nd] + cc] * dpred;
        if (fs) G[M.outW + cc] = g0; else G[M.outW + cc] += g0;
        du[cc] = __ldg(Pw + M.outW + cc) * dpred;
      }
      if (threadIdx.x == 0) {
        if (fs) G[M.outb] = dpred; else G[M.outb] += dpred;
      }
      gbar();
      for (int j = nd - 1; j >= 0; --j) {
        const float* uout = uall + uoff[j + 1];
        for (int cc = threadIdx.x; cc < uw[j + 1]; cc += kGT)
          if (!(uout[cc] > 0.f)) du[cc] = 0.f;
        gbar();
        gwgrad(uall + uoff[j], 0, du, 0, 1, uw[j], uw[j + 1], G + M.decW[j], fs);
        gcolsum(du, 0, 1, uw[j + 1], G + M.decb[j], fs, nullptr, 0);
        W = acquire(M.dec[j]);
        gmm<true>(du, 0, W, ldw, 1, uw[j + 1], uw[j], nullptr, false, nullptr, 0, du2, 0);
        release();
        gbar();
        float* t = du;
        du = du2;
        du2 = t;
      }
    }
    float* dz = du;
    if (loss.use_cmd) {
      const double v = cmd_stats(zall, ns_g, nt_g, de, loss.cmd_order, cmds, kBarGroup, kGT);
      if (blockIdx.x == 0 && threadIdx.x == 0 && w == (int)blockIdx.x) scalars[0] = v;
      for (int e = threadIdx.x; e < de; e += kGT)
        dz[e] += (float)(loss.alpha * cmd_grad_elem(cmds, ns_g, nt_g, de, loss.cmd_order, zrow, e,
                                                    (double)zall[(size_t)zrow * de + e]));
      gbar();
    }
    float* dzx = sm + tp.dzx;
    float* dzp = sm + tp.dzp;
    float* dzv = sm + tp.dzv;
    for (int e = threadIdx.x; e < de; e += kGT) {
      dzx[e] = dz[e] * zp[e];
      dzp[e] = dz[e] * zx[e];
    }
    gbar();
    gwgrad(zv, 0, dzp, 0, 1, M.d_dev, de, G + M.devpW, fs);
    gcolsum(dzp, 0, 1, de, G + M.devpb, fs, nullptr, 0);
    W = acquire(de);
    gmm<true>(dzp, 0, W, ldw, 1, de, M.d_dev, nullptr, false, nullptr, 0, dzv, 0);
    release();
    gbar();
    for (int e = threadIdx.x; e < M.d_dev; e += kGT)
      if (!(zv[e] > 0.f)) dzv[e] = 0.f;
    gbar();
    gwgrad(dv, 0, dzv, 0, 1, TPCB_DEV_FEAT, M.d_dev, G + M.devhW, fs);
    gcolsum(dzv, 0, 1, M.d_dev, G + M.devhb, fs, nullptr, 0);
    for (int l = 0; l < L; ++l) {
      gwgrad(Hout + l * ld, 0, dzx, 0, 1, d, de, G + M.leafW[L] + l * d * de, fl);
      W = acquire(de);
      gmm<true>(dzx, 0, W, ldw, 1, de, d, nullptr, false, nullptr, 0, dH + l * ld, 0);
      release();
    }
    gcolsum(dzx, 0, 1, de, G + M.leafb[L], fl, nullptr, 0);
    gbar();
    for (int li = M.n_layers - 1; li >= 0; --li) {
      const LayerOff& lo = M.layer[li];
      P3 c = lptr(sm, tp, li);
      gln_back(dH, ld, c.X2, ld, c.I2, L, d, Pw + lo.ln2g, dA, ld);
      gcolsum(dH, ld, L, d, G + lo.ln2g, fs, c.X2, ld);
      gcolsum(dH, ld, L, d, G + lo.ln2b, fs, nullptr, 0);
      gbar();
      gwgrad(c.F, ldf, dA, ld, L, M.d_ff, d, G + lo.foW, fs);
      gcolsum(dA, ld, L, d, G + lo.fob, fs, nullptr, 0);
      gln_apply(c.X1, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, T1, ld);  // h1
      W = acquire(d);  // foW
      gmm<true>(dA, ld, W, ldw, L, d, M.d_ff, nullptr, false, nullptr, 0, dF, ldf);
      release();
      gbar();
      for (int e = threadIdx.x; e < L * M.d_ff; e += kGT) {
        const int r = e / M.d_ff, k = e - r * M.d_ff;
        if (!(c.F[r * ldf + k] > 0.f)) dF[r * ldf + k] = 0.f;
      }
      gbar();
      gwgrad(T1, ld, dF, ldf, L, d, M.d_ff, G + lo.fhW, fs);
      gcolsum(dF, ldf, L, M.d_ff, G + lo.fhb, fs, nullptr, 0);
      W = acquire(M.d_ff);  // fhW: dh1 = dA + dF W_fhᵀ → dB
      gmm<true>(dF, ldf, W, ldw, L, M.d_ff, d, nullptr, false, dA, ld, dB, ld);
      release();
      gbar();
      gln_back(dB, ld, c.X1, ld, c.I1, L, d, Pw + lo.ln1g, dA, ld);
      gcolsum(dB, ld, L, d, G + lo.ln1g, fs, c.X1, ld);
      gcolsum(dB, ld, L, d, G + lo.ln1b, fs, nullptr, 0);
      gbar();
      gwgrad(c.C, ld, dA, ld, L, d, d, G + lo.Wo, fs);
      gcolsum(dA, ld, L, d, G + lo.bo, fs, nullptr, 0);
      W = acquire(d);  // Wo: dC = dA W_oᵀ → dB
      gmm<true>(dA, ld, W, ldw, L, d, d, nullptr, false, nullptr, 0, dB, ld);
      release();
      gbar();
      gattn_bwd(c.Q, c.K, c.V, ld, c.P, dB, dQ, dK, dV, S, L, H, dh, scale);
      const float* hin = H0;
      if (li > 0) {
        const LayerOff& lp = M.layer[li - 1];
        P3 cp = lptr(sm, tp, li - 1);
        gln_apply(cp.X2, ld, L, d, Pw + lp.ln2g, Pw + lp.ln2b, T1, ld);
        hin = T1;
        gbar();
      }
      gwgrad(hin, ld, dQ, ld, L, d, d, G + lo.Wq, fs);
      gwgrad(hin, ld, dK, ld, L, d, d, G + lo.Wk, fs);
      gwgrad(hin, ld, dV, ld, L, d, d, G + lo.Wv, fs);
      gcolsum(dQ, ld, L, d, G + lo.bq, fs, nullptr, 0);
      gcolsum(dK, ld, L, d, G + lo.bk, fs, nullptr, 0);
      gcolsum(dV, ld, L, d, G + lo.bv, fs, nullptr, 0);
      W = acquire(d);  // dHin = dA + dQ Wqᵀ + dK Wkᵀ + dV Wvᵀ
      gmm<true>(dQ, ld, W, ldw, L, d, d, nullptr, false, dA, ld, dH, ld);
      release();
      gbar();
      W = acquire(d);
      gmm<true>(dK, ld, W, ldw, L, d, d, nullptr, false, dH, ld, dH, ld);
      release();
      gbar();
      W = acquire(d);
      gmm<true>(dV, ld, W, ldw, L, d, d, nullptr, false, dH, ld, dH, ld);
      release();
      gbar();
    }
    gwgrad(X0, 28, dH, ld, L, TPCB_FEAT, d, G + M.inW, fs);
    gcolsum(dH, ld, L, d, G + M.inb, fs, nullptr, 0);
    mask |= 1u | (1u << L);
    gbar();
  }
  if (threadIdx.x == 0) touched[blockIdx.x] = mask;
}

}  // namespace

int launch_train3(const Model& M, const float* P, const SampleSetDev& src, const SampleSetDev& tgt,
                  const int32_t* batch, const StepDesc* steps, int step, int grid,
                  const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                  int32_t* status, cudaStream_t stream) {
  const Plan3 tp = make_plan3(M, ws.l_cap);
  const size_t smem = (size_t)tp.total * sizeof(float);
  static size_t lim = 0;
  if (!lim) {
    cudaFuncAttributes a{};
    TPCB_CUDA_CHECK(cudaFuncGetAttributes(&a, train3_kernel));
    lim = 227 * 1024 - a.sharedSizeBytes;
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(train3_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim));
  }
  if (smem > lim) return TPCB_ERR_UNSUPPORTED;
  grid = std::max(1, std::min(grid, ws.n_slots));
  train3_kernel<<<grid, kThreads3, smem, stream>>>(M, P, src, tgt, batch, steps, step, loss, phase,
                                                   tp, ws.zall, ws.partial, ws.slot_stride,
                                                   ws.touched, ws.terms, ws.scalars, pred_out,
                                                   status);
  TPCB_LAUNCH_CHECK("train3_kernel");
  return TPCB_OK;
}

size_t train3_smem(const Model& M, int l_cap) { return (size_t)make_plan3(M, l_cap).total * 4; }

}  // namespace tpcb
