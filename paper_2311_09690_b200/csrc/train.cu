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
// private gradient slot.  Weight gradients of a CTA go to slot blockIdx.x of
// `partial`; optim.cu sums the slots in slot order — deterministic, no float
// atomics (SPEC determinism contract).  dX products use a transposed copy of
// every weight matrix (PT, refreshed after each optimizer step) so all
// products are coalesced row-major GEMMs.
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
#include "train.cuh"

namespace tpcb {

TrainPlan make_train_plan(const Model& M) {
  TrainPlan p;
  const int R = M.n_leaf_max;
  p.R = R;
  p.ld = M.d + 1;
  p.ldf = M.d_ff + 1;
  const int blk = R * p.ld;
  int o = 0;
  p.oQ = o; o += blk;
  p.oK = o; o += blk;
  p.oV = o; o += blk;
  p.oC = o; o += blk;
  p.oX1 = o; o += blk;
  p.oX2 = o; o += blk;
  p.oF = o; o += R * p.ldf;
  p.oI1 = o; o += R;
  p.oI2 = o; o += R;
  p.oP = o; o += M.n_heads * R * R;
  p.layer_stride = o;
  o = 0;
  p.layer_base = o; o += M.n_layers * p.layer_stride;
  p.X0 = o; o += R * (TPCB_FEAT + 1);
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
  p.S = o; o += M.n_heads * R * R;
  int uw = 1, usum = M.d_e;
  for (int i = 0; i < M.n_dec; ++i) {
    uw = max(uw, M.dec[i]);
    usum += M.dec[i];
  }
  uw = max(uw, M.d_e);
  p.uw = uw;
  p.dv = o; o += 8;
  p.zx = o; o += M.d_e;
  p.zv = o; o += M.d_dev;
  p.zp = o; o += M.d_e;
  p.u = o; o += usum;  // u[0] = z, u[j+1] = output of decoder layer j
  p.du0 = o; o += uw;
  p.du1 = o; o += uw;
  p.dzx = o; o += M.d_e;
  p.dzp = o; o += M.d_e;
  p.dzv = o; o += M.d_dev;
  p.dflat = o; o += R * M.d;
  p.misc = o; o += 8;
  o = (o + 1) & ~1;  // 8-byte align the fp64 CMD scratch
  p.cmd = o;
  // per column: lo, hi, mus, mut, s, u, ds + amin, amax (stored as double) + ms[K+1], mt[K+1]
  p.cmd_cols = M.d_e;
  o += 2 * cmd_scratch_doubles(M.d_e) + 8;
  p.total = o;
  return p;
}

namespace {

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

}  // namespace

namespace {

__global__ void __launch_bounds__(256) train_kernel(
    Model M, const float* __restrict__ Pw, const float* __restrict__ PT, SampleSetDev src,
    SampleSetDev tgt, const int32_t* __restrict__ batch_all, const int4* __restrict__ steps,
    int step, LossDev loss, int phase, TrainPlan tp, float* __restrict__ zall, float* __restrict__ partial,
    size_t slot_stride, uint32_t* __restrict__ touched, double* __restrict__ terms,
    double* __restrict__ scalars, float* __restrict__ pred_out, int32_t* status) {
  extern __shared__ float sm[];
  const int4 sd = steps[step];
  const int32_t* batch = batch_all + sd.x;
  const int n_src = sd.y, n_tgt = sd.z;
  const int n_all = n_src + (loss.use_cmd ? n_tgt : 0);
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

  for (int w = blockIdx.x; w < n_all; w += gridDim.x) {
    const bool is_t = w >= n_src;
    const SampleSetDev& set = is_t ? tgt : src;
    const int idx = batch[w];
    const int L = set.n_leaf[idx];
    const float* xr = set.x + (size_t)set.ast_row[idx] * TPCB_FEAT_PAD;
    for (int e = threadIdx.x; e < L * TPCB_FEAT; e += blockDim.x) {
      const int r = e / TPCB_FEAT, c = e - r * TPCB_FEAT;
      X0[r * (TPCB_FEAT + 1) + c] = __ldg(xr + r * TPCB_FEAT_PAD + c);
    }
    if (threadIdx.x < TPCB_DEV_FEAT)
      dv[threadIdx.x] = __ldg(set.devfeat + (size_t)idx * TPCB_DEV_FEAT + threadIdx.x);
    __syncthreads();
    // ------------------------------------------------------------ forward
    gemm_rows<4, 4>(X0, TPCB_FEAT + 1, Pw + M.inW, Pw + M.inb, H0, ld, L, TPCB_FEAT, d, false);
    __syncthreads();
    const float* Hin = H0;
    for (int li = 0; li < M.n_layers; ++li) {
      const LayerOff& lo = M.layer[li];
      Ptrs c = layer_ptrs(sm, tp, li);
      gemm_rows<4, 4>(Hin, ld, Pw + lo.Wq, Pw + lo.bq, c.Q, ld, L, d, d, false);
      gemm_rows<4, 4>(Hin, ld, Pw + lo.Wk, Pw + lo.bk, c.K, ld, L, d, d, false);
      gemm_rows<4, 4>(Hin, ld, Pw + lo.Wv, Pw + lo.bv, c.V, ld, L, d, d, false);
      __syncthreads();
      attention_rows(c.Q, c.K, c.V, ld, c.C, ld, 1, L, H, dh, scale, c.P);
      __syncthreads();
      gemm_rows<4, 4>(c.C, ld, Pw + lo.Wo, Pw + lo.bo, T1, ld, L, d, d, false, Hin, ld);
      __syncthreads();
      layernorm_rows(T1, ld, T2, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, c.X1, ld, c.I1);
      __syncthreads();
      gemm_rows<4, 4>(T2, ld, Pw + lo.fhW, Pw + lo.fhb, c.F, ldf, L, d, M.d_ff, true);
      __syncthreads();
      gemm_rows<4, 4>(c.F, ldf, Pw + lo.foW, Pw + lo.fob, T1, ld, L, M.d_ff, d, false, T2, ld);
      __syncthreads();
      layernorm_rows(T1, ld, Hout, ld, L, d, Pw + lo.ln2g, Pw + lo.ln2b, c.X2, ld, c.I2);
      __syncthreads();
      Hin = Hout;
    }
    // head forward (one sample ⇒ row vectors)
    leaf_embed_rows(Hout, ld, 1, L, d, Pw + M.leafW[L], Pw + M.leafb[L], de, zx, de);
    gemm_rows<1, 4>(dv, TPCB_DEV_FEAT, Pw + M.devhW, Pw + M.devhb, zv, M.d_dev, 1,
                    TPCB_DEV_FEAT, M.d_dev, true);
    __syncthreads();
    gemm_rows<1, 4>(zv, M.d_dev, Pw + M.devpW, Pw + M.devpb, zp, de, 1, M.d_dev, de, false);
    __syncthreads();
    for (int e = threadIdx.x; e < de; e += blockDim.x) uall[e] = zx[e] * zp[e];
    __syncthreads();
    {
      int off = 0, wdt = de;
      for (int j = 0; j < M.n_dec; ++j) {
        gemm_rows<1, 4>(uall + off, wdt, Pw + M.decW[j], Pw + M.decb[j], uall + off + wdt,
                        M.dec[j], 1, wdt, M.dec[j], true);
        __syncthreads();
        off += wdt;
        wdt = M.dec[j];
      }
      if (threadIdx.x < 32) {
        float s = 0.f;
        for (int c = threadIdx.x; c < wdt; c += 32)
          s = fmaf(uall[off + c], __ldg(Pw + M.outW + c), s);
        s = warp_sum(s) + __ldg(Pw + M.outb);
        if (threadIdx.x == 0) misc[0] = s;
      }
      __syncthreads();
    }
    const float pred = misc[0];
    if (phase == 0) {
      for (int e = threadIdx.x; e < de; e += blockDim.x) zall[(size_t)w * de + e] = uall[e];
      __syncthreads();
      continue;
    }
    // ------------------------------------------------------- loss gradient
    if (threadIdx.x == 0) {
      double dpred = 0.0;
      if (!is_t) {
        const double y = set.y[idx];
        const double dd = (double)pred - y;
        const double n = (double)n_src;
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
    float* dz = sm + tp.du0;  // dz lives in du0 until the decoder backward is done
    __syncthreads();
    // ------------------------------------------------------------ backward
    const bool fs = !(mask & 1u);
    const bool fl = !(mask & (1u << L));
    // decoder: du = dpred · Wout ; dWout += u_n dpred
    {
      int offs[TPCB_MAX_DEC + 1];
      int wdt[TPCB_MAX_DEC + 1];
      offs[0] = 0;
      wdt[0] = de;
      for (int j = 0; j < M.n_dec; ++j) {
        offs[j + 1] = offs[j] + wdt[j];
        wdt[j + 1] = M.dec[j];
      }
      const int nd = M.n_dec;
      const float dpred = misc[1];
      float* du = sm + tp.du0;
      float* du2 = sm + tp.du1;
      for (int c = threadIdx.x; c < wdt[nd]; c += blockDim.x) {
        gstore(G, M.outW + c, uall[offs[nd] + c] * dpred, fs);
        du[c] = __ldg(Pw + M.outW + c) * dpred;
      }
      if (threadIdx.x == 0) gstore(G, M.outb, dpred, fs);
      __syncthreads();
      for (int j = nd - 1; j >= 0; --j) {
        const float* uin = uall + offs[j];
        const float* uout = uall + offs[j + 1];
        const int win = wdt[j], wout = wdt[j + 1];
        for (int c = threadIdx.x; c < wout; c += blockDim.x)
          if (!(uout[c] > 0.f)) du[c] = 0.f;
        __syncthreads();
        wgrad_rows(uin, win, du, wout, 1, win, wout, G + M.decW[j], fs);
        for (int c = threadIdx.x; c < wout; c += blockDim.x) gstore(G, M.decb[j] + c, du[c], fs);
        // du_prev = du · W_jᵀ
        gemm_rows<1, 4>(du, wout, PT + M.decW[j], nullptr, du2, win, 1, wout, win, false);
        __syncthreads();
        float* t = du;
        du = du2;
        du2 = t;
      }
      dz = du;
    }
    // CMD term
    if (loss.use_cmd) {
      const double v = cmd_stats(zall, n_src, n_tgt, de, loss.cmd_order, cmds);
      if (blockIdx.x == 0 && threadIdx.x == 0 && w == 0) scalars[0] = v;
      for (int e = threadIdx.x; e < de; e += blockDim.x)
        dz[e] += (float)(loss.alpha * cmd_grad_elem(cmds, n_src, n_tgt, de, loss.cmd_order, w, e,
                                                    (double)zall[(size_t)w * de + e]));
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
    // device MLP
    wgrad_rows(zv, M.d_dev, dzp, de, 1, M.d_dev, de, G + M.devpW, fs);
    for (int e = threadIdx.x; e < de; e += blockDim.x) gstore(G, M.devpb + e, dzp[e], fs);
    gemm_rows<1, 4>(dzp, de, PT + M.devpW, nullptr, dzv, M.d_dev, 1, de, M.d_dev, false);
    __syncthreads();
    for (int e = threadIdx.x; e < M.d_dev; e += blockDim.x)
      if (!(zv[e] > 0.f)) dzv[e] = 0.f;
    __syncthreads();
    wgrad_rows(dv, TPCB_DEV_FEAT, dzv, M.d_dev, 1, TPCB_DEV_FEAT, M.d_dev, G + M.devhW, fs);
    for (int e = threadIdx.x; e < M.d_dev; e += blockDim.x) gstore(G, M.devhb + e, dzv[e], fs);
    // leaf_embed.{L}: dW = flat ⊗ dzx ; dflat = dzx · W_Lᵀ → dH rows
    for (int e = threadIdx.x; e < L * d * de; e += blockDim.x) {
      const int k = e / de, n = e - k * de;
      const int l = k / d, j = k - l * d;
      gstore(G, M.leafW[L] + e, Hout[l * ld + j] * dzx[n], fl);
    }
    for (int e = threadIdx.x; e < de; e += blockDim.x) gstore(G, M.leafb[L] + e, dzx[e], fl);
    {
      float* dflat = sm + tp.dflat;
      gemm_rows<1, 4>(dzx, de, PT + M.leafW[L], nullptr, dflat, L * d, 1, de, L * d, false);
      __syncthreads();
      for (int e = threadIdx.x; e < L * d; e += blockDim.x) {
        const int r = e / d, c = e - r * d;
        dH[r * ld + c] = dflat[e];
      }
      __syncthreads();
    }
    // encoder layers, last to first
    for (int li = M.n_layers - 1; li >= 0; --li) {
      const LayerOff& lo = M.layer[li];
      Ptrs c = layer_ptrs(sm, tp, li);
      // LN2
      layernorm_back_rows(dH, ld, c.X2, ld, c.I2, L, d, Pw + lo.ln2g, dA, ld);
      colsum_rows(dH, ld, L, d, G + lo.ln2g, fs, c.X2, ld);
      colsum_rows(dH, ld, L, d, G + lo.ln2b, fs);
      __syncthreads();
      // FFN out: dW_fo = Fᵀ dA ; dF = dA W_foᵀ ⊙ (F > 0)
      wgrad_rows(c.F, ldf, dA, ld, L, M.d_ff, d, G + lo.foW, fs);
      colsum_rows(dA, ld, L, d, G + lo.fob, fs);
      gemm_rows<4, 4>(dA, ld, PT + lo.foW, nullptr, dF, ldf, L, d, M.d_ff, false);
      ln_apply_rows(c.X1, ld, L, d, Pw + lo.ln1g, Pw + lo.ln1b, T1, ld);  // h1
      __syncthreads();
      for (int e = threadIdx.x; e < L * M.d_ff; e += blockDim.x) {
        const int r = e / M.d_ff, k = e - r * M.d_ff;
        if (!(c.F[r * ldf + k] > 0.f)) dF[r * ldf + k] = 0.f;
      }
      __syncthreads();
      wgrad_rows(T1, ld, dF, ldf, L, d, M.d_ff, G + lo.fhW, fs);
      colsum_rows(dF, ldf, L, M.d_ff, G + lo.fhb, fs);
      // dh1 = dA + dF W_fhᵀ → dB
      gemm_rows<4, 4>(dF, ldf, PT + lo.fhW, nullptr, dB, ld, L, M.d_ff, d, false, dA, ld);
      __syncthreads();
      // LN1
      layernorm_back_rows(dB, ld, c.X1, ld, c.I1, L, d, Pw + lo.ln1g, dA, ld);
      colsum_rows(dB, ld, L, d, G + lo.ln1g, fs, c.X1, ld);
      colsum_rows(dB, ld, L, d, G + lo.ln1b, fs);
      __syncthreads();
      // O projection: dW_o = Cᵀ dA ; dC = dA W_oᵀ → dB
      wgrad_rows(c.C, ld, dA, ld, L, d, d, G + lo.Wo, fs);
      colsum_rows(dA, ld, L, d, G + lo.bo, fs);
      gemm_rows<4, 4>(dA, ld, PT + lo.Wo, nullptr, dB, ld, L, d, d, false);
      __syncthreads();
      attention_back_rows(c.Q, c.K, c.V, ld, c.P, dB, ld, dQ, dK, dV, S, 1, L, H, dh, scale);
      // layer input (recomputed for li > 0)
      const float* hin = H0;
      if (li > 0) {
        const LayerOff& lp = M.layer[li - 1];
        Ptrs cp = layer_ptrs(sm, tp, li - 1);
        ln_apply_rows(cp.X2, ld, L, d, Pw + lp.ln2g, Pw + lp.ln2b, T1, ld);
        hin = T1;
      }
      __syncthreads();
      wgrad_rows(hin, ld, dQ, ld, L, d, d, G + lo.Wq, fs);
      wgrad_rows(hin, ld, dK, ld, L, d, d, G + lo.Wk, fs);
      wgrad_rows(hin, ld, dV, ld, L, d, d, G + lo.Wv, fs);
      colsum_rows(dQ, ld, L, d, G + lo.bq, fs);
      colsum_rows(dK, ld, L, d, G + lo.bk, fs);
      colsum_rows(dV, ld, L, d, G + lo.bv, fs);
      // dHin = dA + dQ Wqᵀ + dK Wkᵀ + dV Wvᵀ → dH
      gemm_rows<4, 4>(dQ, ld, PT + lo.Wq, nullptr, dH, ld, L, d, d, false, dA, ld);
      __syncthreads();
      gemm_rows<4, 4>(dK, ld, PT + lo.Wk, nullptr, dH, ld, L, d, d, false, dH, ld);
      __syncthreads();
      gemm_rows<4, 4>(dV, ld, PT + lo.Wv, nullptr, dH, ld, L, d, d, false, dH, ld);
      __syncthreads();
    }
    wgrad_rows(X0, TPCB_FEAT + 1, dH, ld, L, TPCB_FEAT, d, G + M.inW, fs);
    colsum_rows(dH, ld, L, d, G + M.inb, fs);
    mask |= 1u | (1u << L);
    __syncthreads();
  }
  if (threadIdx.x == 0) touched[blockIdx.x] = mask;
}

}  // namespace

int prepare_train_kernels(const Model& M) {
  TrainPlan tp = make_train_plan(M);
  const size_t smem = (size_t)tp.total * sizeof(float);
  if (smem > 227 * 1024) return TPCB_ERR_UNSUPPORTED;
  static size_t set_for = 0;
  if (smem > set_for) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024));
    set_for = 227 * 1024;
  }
  return TPCB_OK;
}

int launch_train(const Model& M, const float* P, const float* PT, const SampleSetDev& src,
                 const SampleSetDev& tgt, const int32_t* batch, const int4* steps, int step,
                 int grid, const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                 int32_t* status, cudaStream_t stream) {
  TrainPlan tp = make_train_plan(M);
  const size_t smem = (size_t)tp.total * sizeof(float);
  if (smem > 227 * 1024) return TPCB_ERR_UNSUPPORTED;
  if (loss.cmd_order > kMaxCmdOrder) return TPCB_ERR_UNSUPPORTED;
  int st = prepare_train_kernels(M);
  if (st) return st;
  grid = std::max(1, std::min(grid, ws.n_slots));
  train_kernel<<<grid, 256, smem, stream>>>(M, P, PT, src, tgt, batch, steps, step, loss, phase,
                                            tp, ws.zall, ws.partial, ws.slot_stride, ws.touched,
                                            ws.terms, ws.scalars, pred_out, status);
  TPCB_LAUNCH_CHECK("train_kernel");
  return TPCB_OK;
}

}  // namespace tpcb
