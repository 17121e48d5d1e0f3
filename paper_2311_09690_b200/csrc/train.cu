// K4+K5(+K6) — training step: forward with activation caches, hybrid loss
// gradient, CMD gradient, full backward; then (optim.cu) the fixed-order
// gradient reduction and the optimizer.
//
// Reference: costmodel.backward (costmodel.py:529-570) = _forward (:233),
// _supervised_loss_grad / _relative_term / _decode_with_grad (:358-423),
// _cmd_forward_backward (:426-486), _backward_group (:280-336) with the nn.*
// backward primitives (nn.py:30-120).
//
// Work decomposition: one work item = one sample (its L ≤ 16 leaf rows); a
// CTA keeps every activation of its sample in shared memory, so forward and
// backward never touch HBM except for weights (L2-resident) and the CTA's
// private gradient slot.  Weights are streamed op by op into a double-
// buffered shared-memory stage with cp.async, one op ahead of use
// (smallmm.cuh), so the L2 latency of the next weight matrix hides behind the
// current op; the transposed products of the backward read the same staged
// copy with a transposed index.  Weight gradients of a CTA go to slot
// blockIdx.x of `partial`; optim.cu sums the slots in slot order —
// deterministic, no float atomics (SPEC determinism contract).
//
// CMD couples the samples of a step through batch statistics, so a CMD step
// runs the kernel twice: phase 0 writes every sample's z, phase 1 recomputes
// the forward, forms each row's CMD gradient from all z (every CTA computes
// the column statistics redundantly — ≤ 2·batch rows × d_embed) and runs the
// backward.
#include <cmath>

#include "blocks.cuh"
#include "common.cuh"
#include "cmd.cuh"
#include "smallmm.cuh"
#include "train.cuh"

namespace tpcb {


TrainPlan make_train_plan(const Model& M, int l_cap) {
  TrainPlan p;
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
  p.layer_stride = o;
  o = 0;
  p.layer_base = o; o += M.n_layers * p.layer_stride;
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
  int uw = M.d_e, usum = round4(M.d_e);
  for (int i = 0; i < M.n_dec; ++i) {
    uw = max(uw, M.dec[i]);
    usum += round4(M.dec[i]);
  }
  p.uw = round4(max(uw, max(M.d_dev, M.d)));
  p.dv = o; o += 8;
  p.zx = o; o += round4(M.d_e);
  p.zv = o; o += round4(M.d_dev);
  p.zp = o; o += round4(M.d_e);
  p.u = o; o += usum;  // u[0] = z, u[j+1] = output of decoder layer j (each 4-aligned)
  p.du0 = o; o += p.uw;
  p.du1 = o; o += p.uw;
  p.dzx = o; o += round4(M.d_e);
  p.dzp = o; o += round4(M.d_e);
  p.dzv = o; o += round4(M.d_dev);
  p.dflat = o; o += round4(M.d_e) + 4;
  p.misc = o; o += 8;
  // split-K partials of small_mm and the attention dS scratch share a region
  p.S = o; o += max(kTrainThreads * R, M.n_heads * R * R);
  o = (o + 1) & ~1;  // 8-byte align the fp64 CMD scratch
  p.cmd = o;
  p.cmd_cols = M.d_e;
  o += 2 * cmd_scratch_doubles(M.d_e) + 8;
  // weight stage: two buffers of the largest entry (ld = N + 1)
  int cap = 0;
  for (int L = 1; L <= R; ++L) {
    const int n = n_all_entries(M, L);
    for (int i = 0; i < n; ++i) {
      int K, N, off;
      entry_shape(M, L, i, &K, &N, &off);
      cap = max(cap, K * stage_ld(N));
    }
  }
  p.stage_cap = round4(cap);
  o = round4(o);
  p.stage0 = o; o += p.stage_cap;
  p.stage1 = o; o += p.stage_cap;
  p.total = o;
  return p;
}

namespace {

// out-of-line copies of the row blocks: the training kernel calls each one
// dozens of times per sample; one copy keeps the kernel in the I-cache
__device__ __noinline__ void layernorm_rows_nl(const float* X, int ldx, float* Y, int ldy, int R,
                                               int d, const float* g, const float* b,
                                               float* xhat, int ldh, float* inv_out) {
  layernorm_rows(X, ldx, Y, ldy, R, d, g, b, xhat, ldh, inv_out);
}
__device__ __noinline__ void attention_rows_nl(const float* Q, const float* K, const float* V,
                                               int ld, float* C, int ldc, int A, int L, int H,
                                               int dh, float scale, float* P) {
  attention_rows(Q, K, V, ld, C, ldc, A, L, H, dh, scale, P);
}
__device__ __noinline__ void colsum_rows_nl(const float* dY, int ldy, int R, int N, float* G,
                                            bool first, const float* S, int lds) {
  colsum_rows(dY, ldy, R, N, G, first, S, lds);
}
__device__ __noinline__ void layernorm_back_rows_nl(const float* dY, int ldy, const float* Xh,
                                                    int ldh, const float* inv, int R, int d,
                                                    const float* g, float* dX, int ldx) {
  layernorm_back_rows(dY, ldy, Xh, ldh, inv, R, d, g, dX, ldx);
}
__device__ __noinline__ void ln_apply_rows_nl(const float* Xh, int ldh, int R, int d,
                                              const float* g, const float* b, float* Y, int ldy) {
  ln_apply_rows(Xh, ldh, R, d, g, b, Y, ldy);
}
__device__ __noinline__ void attention_back_rows_nl(const float* Q, const float* K,
                                                    const float* V, int ld, const float* P,
                                                    const float* dC, int ldc, float* dQ,
                                                    float* dK, float* dV, float* S, int A, int L,
                                                    int H, int dh, float scale) {
  attention_back_rows(Q, K, V, ld, P, dC, ldc, dQ, dK, dV, S, A, L, H, dh, scale);
}

// Attention of one sample (L ≤ 16 rows) spread over the whole block:
// scores one thread per (head, i, j), softmax one thread per (head, i),
// context one thread per (i, feature) — three short barrier-separated
// phases instead of one long serial loop per query row (nn.py:79-96).
__device__ __noinline__ void attn_fwd_sample(const float* Q, const float* K, const float* V,
                                             int ld, float* C, int L, int H, int dh, float scale,
                                             float* P) {
  const int nt = blockDim.x, LL = L * L;
  for (int e = threadIdx.x; e < H * LL; e += nt) {
    const int h = e / LL, ij = e - h * LL, i = ij / L, j = ij - i * L;
    const float* q = Q + i * ld + h * dh;
    const float* k = K + j * ld + h * dh;
    float s = 0.f;
    if ((dh & 3) == 0) {
      for (int c = 0; c < dh; c += 4) {
        const float4 a = *reinterpret_cast<const float4*>(q + c);
        const float4 b = *reinterpret_cast<const float4*>(k + c);
        s = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, s))));
      }
    } else {
      for (int c = 0; c < dh; ++c) s = fmaf(q[c], k[c], s);
    }
    P[e] = s * scale;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < H * L; e += nt) {
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
  __syncthreads();
  const int D = H * dh;
  for (int e = threadIdx.x; e < L * D; e += nt) {
    const int i = e / D, f = e - i * D, h = f / dh;
    const float* p = P + (h * L + i) * L;
    float acc = 0.f;
    for (int j = 0; j < L; ++j) acc = fmaf(p[j], V[j * ld + f], acc);
    C[i * ld + f] = acc;
  }
  __syncthreads();
}

// backward of attn_fwd_sample (nn.py:99-120): dS = P ⊙ (dP − Σ_j dP P)·scale
// with dP = dC Vᵀ; dQ = dS K, dK = dSᵀ Q, dV = Pᵀ dC.  S: H·L·L scratch.
__device__ __noinline__ void attn_bwd_sample(const float* Q, const float* K, const float* V,
                                             int ld, const float* P, const float* dC,
                                             float* dQ, float* dK, float* dV, float* S, int L,
                                             int H, int dh, float scale) {
  const int nt = blockDim.x, LL = L * L;
  for (int e = threadIdx.x; e < H * LL; e += nt) {
    const int h = e / LL, ij = e - h * LL, i = ij / L, j = ij - i * L;
    const float* a = dC + i * ld + h * dh;
    const float* b = V + j * ld + h * dh;
    float s = 0.f;
    if ((dh & 3) == 0) {
      for (int c = 0; c < dh; c += 4) {
        const float4 x = *reinterpret_cast<const float4*>(a + c);
        const float4 y = *reinterpret_cast<const float4*>(b + c);
        s = fmaf(x.x, y.x, fmaf(x.y, y.y, fmaf(x.z, y.z, fmaf(x.w, y.w, s))));
      }
    } else {
      for (int c = 0; c < dh; ++c) s = fmaf(a[c], b[c], s);
    }
    S[e] = s;  // dP
  }
  __syncthreads();
  for (int e = threadIdx.x; e < H * L; e += nt) {
    float* s = S + e * L;
    const float* p = P + e * L;
    float dot = 0.f;
    for (int j = 0; j < L; ++j) dot = fmaf(s[j], p[j], dot);
    for (int j = 0; j < L; ++j) s[j] = p[j] * (s[j] - dot) * scale;
  }
  __syncthreads();
  const int D = H * dh;
  for (int e = threadIdx.x; e < L * D; e += nt) {
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
  __syncthreads();
}

struct Ptrs {
  float *Q, *K, *V, *C, *X1, *X2, *F, *I1, *I2, *P;
};

__device__ __forceinline__ Ptrs layer_ptrs(float* sm, const TrainPlan& tp, int li) {
  float* b = sm + tp.layer_base + li * tp.layer_stride;
  return Ptrs{b + tp.oQ, b + tp.oK, b + tp.oV, b + tp.oC, b + tp.oX1,
              b + tp.oX2, b + tp.oF, b + tp.oI1, b + tp.oI2, b + tp.oP};
}

// decode with derivative, clamped at 1e-12 (costmodel.py:358-373)
__device__ void decode_with_grad(double e, const tpcb_boxcox& n, double* y, double* dy) {
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

__device__ double decode_plain(double e, const tpcb_boxcox& n) {
  const double t = e * n.t_std + n.t_mean;
  if (fabs(n.lambda_bc) < 1e-9) return exp(t) - n.shift;
  return pow(n.lambda_bc * t + 1.0, 1.0 / n.lambda_bc) - n.shift;
}

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// op-ahead weight prefetch over the entries of one sample
// optional per-op timestamps of CTA 0 (tools/trace_train.py): pairs of
// (clock64 at acquire entry, clock64 after its barrier) per weight entry
__device__ long long* g_trace = nullptr;

constexpr int kMaxEntries = 256;

// op-ahead weight prefetch over the entries of one sample.  The entry table
// (rows, cols, offset of every weight matrix in consumption order) is built
// in shared memory at the start of each sample, so the hot path never reads
// the kernel-parameter Model through a pointer (a generic load from param
// space costs a global-memory round trip).
struct WStream {
  const float* P;
  float* buf[2];
  const int* ent;  // smem [n][3]
  int idx, n, rep;

  __device__ __forceinline__ void stage(int i) {
    stage_matrix(P + ent[3 * i + 2], ent[3 * i], ent[3 * i + 1], buf[i & 1]);
  }
  __device__ void begin(int n_, int rep_ = 0) {
    rep = rep_;
    n = n_;
    idx = 0;
    stage(0);
    cp_async_commit();
  }
  // staged copy of entry idx (row stride stage_ld(N)); prefetches entry
  // idx+1.  Every caller must have passed a block barrier since the previous
  // use of the buffer being refilled.
  __device__ __noinline__ const float* acquire(int* ldw) {
    long long* tr = g_trace;
    const bool rec = tr != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && idx < 64 && rep < 2;
    if (rec) tr[4 * idx + 256 * rep] = clock64();
    *ldw = stage_ld(ent[3 * idx + 1]);
    if (idx + 1 < n) stage(idx + 1);
    cp_async_commit();
    if (rec) tr[4 * idx + 1 + 256 * rep] = clock64();
    cp_async_wait<1>();
    if (rec) tr[4 * idx + 2 + 256 * rep] = clock64();
    __syncthreads();
    if (rec) tr[4 * idx + 3 + 256 * rep] = clock64();
    return buf[(idx++) & 1];
  }
  __device__ void drain() {
    cp_async_wait<0>();
    __syncthreads();
  }
};

__global__ void __launch_bounds__(kTrainThreads) train_kernel(
    const __grid_constant__ Model M, const float* __restrict__ Pw, SampleSetDev src, SampleSetDev tgt,
    const int32_t* __restrict__ batch_all, const StepDesc* __restrict__ steps, int step, LossDev loss,
    int phase, const __grid_constant__ TrainPlan tp, float* __restrict__ zall,
    float* __restrict__ partial,
    size_t slot_stride, uint32_t* __restrict__ touched, double* __restrict__ terms,
    double* __restrict__ scalars, float* __restrict__ pred_out, int32_t* status) {
  extern __shared__ __align__(16) float sm[];
  const StepDesc sd = steps[step];
  const int32_t* batch = batch_all + sd.off;
  const int n_src = sd.n_src, n_tgt = sd.n_tgt;
  const int n_all = n_src + (loss.use_cmd ? n_tgt : 0);
  const int ns_g = sd.ns_glob, nt_g = sd.nt_glob;
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
  __shared__ int s_ent[3 * kMaxEntries];
  WStream ws;
  ws.P = Pw;
  ws.ent = s_ent;
  ws.buf[0] = sm + tp.stage0;
  ws.buf[1] = sm + tp.stage1;
  int uoff[TPCB_MAX_DEC + 1], uw[TPCB_MAX_DEC + 1];
  uoff[0] = 0;
  uw[0] = de;
  for (int j = 0; j < M.n_dec; ++j) {
    uoff[j + 1] = uoff[j] + round4(uw[j]);
    uw[j + 1] = M.dec[j];
  }
  const int nd = M.n_dec;
  int ldw;

  for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
    const bool is_t = w >= n_src;
    const SampleSetDev set = is_t ? tgt : src;  // by value: no generic loads from param space
    const int idx = batch[w];
    const int L = set.n_leaf[idx];
    if (L < 1 || L > tp.R) {  // the plan was sized for the trainer's datasets
      raise_status(status, TPCB_ERR_LEAF_COUNT);
      continue;
    }
    const int n_ent = phase == 0 ? n_fwd_entries(M, L) : n_all_entries(M, L);
    for (int i = threadIdx.x; i < n_ent; i += blockDim.x)
      entry_shape(M, L, i, &s_ent[3 * i], &s_ent[3 * i + 1], &s_ent[3 * i + 2]);
    __syncthreads();
    ws.begin(n_ent, (w - (int)blockIdx.x) / (int)gridDim.x);
    const float* xr = set.x + (size_t)set.ast_row[idx] * TPCB_FEAT_PAD;
    for (int e = threadIdx.x; e < L * TPCB_FEAT; e += blockDim.x) {
      const int r = e / TPCB_FEAT, c = e - r * TPCB_FEAT;
      X0[r * 28 + c] = __ldg(xr + r * TPCB_FEAT_PAD + c);
    }
    if (threadIdx.x < TPCB_DEV_FEAT)
      dv[threadIdx.x] = __ldg(set.devfeat + (size_t)idx * TPCB_DEV_FEAT + threadIdx.x);
    // ------------------------------------------------------------ forward
    const float* W = ws.acquire(&ldw);  // input.W (barrier inside covers X0/dv)
    small_mm<false>(X0, 28, W, ldw, L, TPCB_FEAT, d, Pw + M.inb, false, nullptr, 0, H0, ld, S);
    const float* Hin = H0;
    for (int li = 0; li < M.n_layers; ++li) {
      const LayerOff& lo = M.layer[li];
      Ptrs c = layer_ptrs(sm, tp, li);
      W = ws.acquire(&ldw);
      small_mm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bq, false, nullptr, 0, c.Q, ld, S);
      W = ws.acquire(&ldw);
      small_mm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bk, false, nullptr, 0, c.K, ld, S);
      W = ws.acquire(&ldw);
      small_mm<false>(Hin, ld, W, ldw, L, d, d, Pw + lo.bv, false, nullptr, 0, c.V, ld, S);
      attn_fwd_sample(c.Q, c.K, c.V, ld, c.C, L, H, dh, scale, c.P);
      W = ws.acquire(&ldw);  // (its barrier also orders the attention output)
      small_mm<false>(c.C, ld, W, ldw, L, d, d, Pw + lo.bo, false, Hin, ld, T1, ld, S);
      layernorm_rows_nl(T1, ld, T2, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, c.X1, ld, c.I1);
      W = ws.acquire(&ldw);
      small_mm<false>(T2, ld, W, ldw, L, d, M.d_ff, Pw + lo.fhb, true, nullptr, 0, c.F, ldf, S);
      W = ws.acquire(&ldw);
      small_mm<false>(c.F, ldf, W, ldw, L, M.d_ff, d, Pw + lo.fob, false, T2, ld, T1, ld, S);
      layernorm_rows_nl(T1, ld, Hout, ld, L, d, Pw + lo.ln2g, Pw + lo.ln2b, c.X2, ld, c.I2);
      __syncthreads();
      Hin = Hout;
    }
    // head: z_x = b_L + Σ_l Hout[l] · W_L[l]   (leaf_embed.{L}, chunk per leaf)
    for (int l = 0; l < L; ++l) {
      W = ws.acquire(&ldw);
      small_mm<false>(Hout + l * ld, ld, W, ldw, 1, d, de, l == 0 ? Pw + M.leafb[L] : nullptr,
                      false, l == 0 ? nullptr : zx, 0, zx, 0, S);
    }
    W = ws.acquire(&ldw);
    small_mm<false>(dv, 8, W, ldw, 1, TPCB_DEV_FEAT, M.d_dev, Pw + M.devhb, true, nullptr, 0, zv,
                    0, S);
    W = ws.acquire(&ldw);
    small_mm<false>(zv, 0, W, ldw, 1, M.d_dev, de, Pw + M.devpb, false, nullptr, 0, zp, 0, S);
    for (int e = threadIdx.x; e < de; e += blockDim.x) uall[e] = zx[e] * zp[e];
    for (int j = 0; j < nd; ++j) {
      W = ws.acquire(&ldw);
      small_mm<false>(uall + uoff[j], 0, W, ldw, 1, uw[j], M.dec[j], Pw + M.decb[j], true,
                      nullptr, 0, uall + uoff[j + 1], 0, S);
    }
    W = ws.acquire(&ldw);
    small_mm<false>(uall + uoff[nd], 0, W, ldw, 1, uw[nd], 1, Pw + M.outb, false, nullptr, 0,
                    misc, 0, S);
    const float pred = misc[0];
    // row of this sample in the global [zs; zt] matrix
    const int zrow = is_t ? ns_g + sd.tgt_pos + (w - n_src) : sd.src_pos + w;
    if (phase == 0) {
      for (int e = threadIdx.x; e < de; e += blockDim.x) zall[(size_t)zrow * de + e] = uall[e];
      ws.drain();
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
            const double y0 = decode_plain(y, loss.norm);
            double p0, dp0;
            decode_with_grad((double)pred, loss.norm, &p0, &dp0);
            const double r = p0 - y0;
            rel = fabs(r) / y0;
            relg = sgn(r) * dp0 / (y0 * n);
          } else {
            const double den = y + loss.offset;
            rel = fabs(dd) / den;
            relg = sgn(dd) / (den * n);
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
    __syncthreads();
    // ------------------------------------------------------------ backward
    const bool fs = !(mask & 1u);
    const bool fl = !(mask & (1u << L));
    float* du = sm + tp.du0;
    float* du2 = sm + tp.du1;
    {
      const float dpred = misc[1];
      for (int c = threadIdx.x; c < uw[nd]; c += blockDim.x) {
        gstore(G, M.outW + c, uall[uoff[nd] + c] * dpred, fs);
        du[c] = __ldg(Pw + M.outW + c) * dpred;
      }
      if (threadIdx.x == 0) gstore(G, M.outb, dpred, fs);
      __syncthreads();
      for (int j = nd - 1; j >= 0; --j) {
        const float* uout = uall + uoff[j + 1];
        for (int c = threadIdx.x; c < uw[j + 1]; c += blockDim.x)
          if (!(uout[c] > 0.f)) du[c] = 0.f;
        __syncthreads();
        wgrad_v(uall + uoff[j], 0, du, 0, 1, uw[j], uw[j + 1], G + M.decW[j], fs);
        for (int c = threadIdx.x; c < uw[j + 1]; c += blockDim.x) gstore(G, M.decb[j] + c, du[c], fs);
        W = ws.acquire(&ldw);
        small_mm<true>(du, 0, W, ldw, 1, uw[j + 1], uw[j], nullptr, false, nullptr, 0, du2, 0, S);
        float* t = du;
        du = du2;
        du2 = t;
      }
    }
    float* dz = du;
    if (loss.use_cmd) {
      const double v = cmd_stats(zall, ns_g, nt_g, de, loss.cmd_order, cmds);
      if (blockIdx.x == 0 && threadIdx.x == 0 && w == (int)blockIdx.x) scalars[0] = v;
      for (int e = threadIdx.x; e < de; e += blockDim.x)
        dz[e] += (float)(loss.alpha * cmd_grad_elem(cmds, ns_g, nt_g, de, loss.cmd_order, zrow, e,
                                                    (double)zall[(size_t)zrow * de + e]));
      __syncthreads();
    }
    float* dzx = sm + tp.dzx;
    float* dzp = sm + tp.dzp;
    float* dzv = sm + tp.dzv;
    for (int e = threadIdx.x; e < de; e += blockDim.x) {
      dzx[e] = dz[e] * zp[e];
      dzp[e] = dz[e] * zx[e];
    }
    __syncthreads();
    wgrad_v(zv, 0, dzp, 0, 1, M.d_dev, de, G + M.devpW, fs);
    for (int e = threadIdx.x; e < de; e += blockDim.x) gstore(G, M.devpb + e, dzp[e], fs);
    W = ws.acquire(&ldw);
    small_mm<true>(dzp, 0, W, ldw, 1, de, M.d_dev, nullptr, false, nullptr, 0, dzv, 0, S);
    for (int e = threadIdx.x; e < M.d_dev; e += blockDim.x)
      if (!(zv[e] > 0.f)) dzv[e] = 0.f;
    __syncthreads();
    wgrad_v(dv, 0, dzv, 0, 1, TPCB_DEV_FEAT, M.d_dev, G + M.devhW, fs);
    for (int e = threadIdx.x; e < M.d_dev; e += blockDim.x) gstore(G, M.devhb + e, dzv[e], fs);
    // leaf_embed.{L}: dW rows l = Hout[l] ⊗ dzx ; dH[l] = dzx · W_L[l]ᵀ
    for (int l = 0; l < L; ++l) {
      wgrad_v(Hout + l * ld, 0, dzx, 0, 1, d, de, G + M.leafW[L] + l * d * de, fl);
      W = ws.acquire(&ldw);
      small_mm<true>(dzx, 0, W, ldw, 1, de, d, nullptr, false, nullptr, 0, dH + l * ld, 0, S);
    }
    for (int e = threadIdx.x; e < de; e += blockDim.x) gstore(G, M.leafb[L] + e, dzx[e], fl);
    // encoder layers, last to first
    for (int li = M.n_layers - 1; li >= 0; --li) {
      const LayerOff& lo = M.layer[li];
      Ptrs c = layer_ptrs(sm, tp, li);
      layernorm_back_rows_nl(dH, ld, c.X2, ld, c.I2, L, d, Pw + lo.ln2g, dA, ld);
      colsum_rows_nl(dH, ld, L, d, G + lo.ln2g, fs, c.X2, ld);
      colsum_rows_nl(dH, ld, L, d, G + lo.ln2b, fs, nullptr, 0);
      __syncthreads();
      wgrad_v(c.F, ldf, dA, ld, L, M.d_ff, d, G + lo.foW, fs);
      colsum_rows_nl(dA, ld, L, d, G + lo.fob, fs, nullptr, 0);
      ln_apply_rows_nl(c.X1, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, T1, ld);  // h1
      W = ws.acquire(&ldw);  // foW
      small_mm<true>(dA, ld, W, ldw, L, d, M.d_ff, nullptr, false, nullptr, 0, dF, ldf, S);
      for (int e = threadIdx.x; e < L * M.d_ff; e += blockDim.x) {
        const int r = e / M.d_ff, k = e - r * M.d_ff;
        if (!(c.F[r * ldf + k] > 0.f)) dF[r * ldf + k] = 0.f;
      }
      __syncthreads();
      wgrad_v(T1, ld, dF, ldf, L, d, M.d_ff, G + lo.fhW, fs);
      colsum_rows_nl(dF, ldf, L, M.d_ff, G + lo.fhb, fs, nullptr, 0);
      W = ws.acquire(&ldw);  // fhW: dh1 = dA + dF W_fhᵀ → dB
      small_mm<true>(dF, ldf, W, ldw, L, M.d_ff, d, nullptr, false, dA, ld, dB, ld, S);
      layernorm_back_rows_nl(dB, ld, c.X1, ld, c.I1, L, d, Pw + lo.ln1g, dA, ld);
      colsum_rows_nl(dB, ld, L, d, G + lo.ln1g, fs, c.X1, ld);
      colsum_rows_nl(dB, ld, L, d, G + lo.ln1b, fs, nullptr, 0);
      __syncthreads();
      wgrad_v(c.C, ld, dA, ld, L, d, d, G + lo.Wo, fs);
      colsum_rows_nl(dA, ld, L, d, G + lo.bo, fs, nullptr, 0);
      W = ws.acquire(&ldw);  // Wo: dC = dA W_oᵀ → dB
      small_mm<true>(dA, ld, W, ldw, L, d, d, nullptr, false, nullptr, 0, dB, ld, S);
      attn_bwd_sample(c.Q, c.K, c.V, ld, c.P, dB, dQ, dK, dV, S, L, H, dh, scale);
      const float* hin = H0;
      if (li > 0) {
        const LayerOff& lp = M.layer[li - 1];
        Ptrs cp = layer_ptrs(sm, tp, li - 1);
        ln_apply_rows_nl(cp.X2, ld, L, d, Pw + lp.ln2g, Pw + lp.ln2b, T1, ld);
        hin = T1;
      }
      __syncthreads();
      wgrad_v(hin, ld, dQ, ld, L, d, d, G + lo.Wq, fs);
      wgrad_v(hin, ld, dK, ld, L, d, d, G + lo.Wk, fs);
      wgrad_v(hin, ld, dV, ld, L, d, d, G + lo.Wv, fs);
      colsum_rows_nl(dQ, ld, L, d, G + lo.bq, fs, nullptr, 0);
      colsum_rows_nl(dK, ld, L, d, G + lo.bk, fs, nullptr, 0);
      colsum_rows_nl(dV, ld, L, d, G + lo.bv, fs, nullptr, 0);
      // dHin = dA + dQ Wqᵀ + dK Wkᵀ + dV Wvᵀ → dH
      W = ws.acquire(&ldw);
      small_mm<true>(dQ, ld, W, ldw, L, d, d, nullptr, false, dA, ld, dH, ld, S);
      W = ws.acquire(&ldw);
      small_mm<true>(dK, ld, W, ldw, L, d, d, nullptr, false, dH, ld, dH, ld, S);
      W = ws.acquire(&ldw);
      small_mm<true>(dV, ld, W, ldw, L, d, d, nullptr, false, dH, ld, dH, ld, S);
    }
    wgrad_v(X0, 28, dH, ld, L, TPCB_FEAT, d, G + M.inW, fs);
    colsum_rows_nl(dH, ld, L, d, G + M.inb, fs, nullptr, 0);
    mask |= 1u | (1u << L);
    ws.drain();
  }
  if (threadIdx.x == 0) touched[blockIdx.x] = mask;
}

}  // namespace

int set_train_trace(long long* d_trace) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace, &d_trace, sizeof(d_trace)));
  return TPCB_OK;
}

// dynamic shared memory left next to the kernel's static tables
static size_t train_dyn_smem_limit() {
  static size_t lim = 0;
  if (!lim) {
    cudaFuncAttributes a{};
    if (cudaFuncGetAttributes(&a, train_kernel) == cudaSuccess)
      lim = 227 * 1024 - a.sharedSizeBytes;
  }
  return lim;
}

int prepare_train_kernels(const Model& M, int l_cap) {
  TrainPlan tp = make_train_plan(M, l_cap);
  const size_t smem = (size_t)tp.total * sizeof(float);
  const size_t lim = train_dyn_smem_limit();
  if (smem > lim) return TPCB_ERR_UNSUPPORTED;
  static bool done = false;
  if (!done) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lim));
    done = true;
  }
  return TPCB_OK;
}

int launch_train(const Model& M, const float* P, const float* PT, const SampleSetDev& src,
                 const SampleSetDev& tgt, const int32_t* batch, const StepDesc* steps, int step,
                 int grid, const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                 int32_t* status, cudaStream_t stream) {
  (void)PT;
  const Knobs& kn = knobs();
  if (kn.grid_cap > 0) grid = std::min(grid, kn.grid_cap);
  if ((kn.train_impl == 0 || kn.train_impl == 4) && v4_fits(M, ws.l_cap))
    return launch_train4(M, P, src, tgt, batch, steps, step, grid, loss, phase, ws, pred_out,
                         status, stream);
  TrainPlan tp = make_train_plan(M, ws.l_cap);
  const size_t smem = (size_t)tp.total * sizeof(float);
  if (loss.cmd_order > kMaxCmdOrder) return TPCB_ERR_UNSUPPORTED;
  int st = prepare_train_kernels(M, ws.l_cap);
  if (st) return st;
  grid = std::max(1, std::min(grid, ws.n_slots));
  train_kernel<<<grid, kTrainThreads, smem, stream>>>(M, P, src, tgt, batch, steps, step, loss, phase, tp,
                                            ws.zall, ws.partial, ws.slot_stride, ws.touched,
                                            ws.terms, ws.scalars, pred_out, status);
  TPCB_LAUNCH_CHECK("train_kernel");
  return TPCB_OK;
}

}  // namespace tpcb
