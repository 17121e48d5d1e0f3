// K7 — fixed-order gradient reduction fused with the optimizer step, plus the
// transposed-weight refresh the backward's dX products read.
//
// Reference: nn.Adam.step / nn.Sgd.step (nn.py:127-167) — L2 weight decay
// added to the gradient, bias-corrected Adam, EVERY tensor updated every step
// (tensors the batch did not touch get g = 0, so m/v still decay,
// costmodel.py:565-567) — and the loss value of costmodel.backward
// (costmodel.py:539-550).
//
// HBM/L2-bound: per parameter it reads the gradient slots of the CTAs that
// touched its region (bit mask per slot) in slot order, then reads/writes
// p, m, v.  No float atomics anywhere, so a step is bitwise reproducible.
#include <cmath>

#include "common.cuh"
#include "train.cuh"

namespace tpcb {

namespace {

__device__ __forceinline__ int region_bit(const Model& M, int p, const int* leaf_lo) {
  if (p < leaf_lo[1] || p >= M.tail_lo) return 0;
  int L = 1;
  while (L < M.n_leaf_max && p >= leaf_lo[L + 1]) ++L;
  return L;
}

__global__ void __launch_bounds__(256) reduce_apply_kernel(
    const __grid_constant__ Model M, const float* __restrict__ partial, size_t stride,
    const uint32_t* __restrict__ touched,
    const StepDesc* __restrict__ steps, int step, int n_slots, int use_cmd, int add_cmd,
    float* __restrict__ grad_out,
    float* __restrict__ P, float* __restrict__ mbuf, float* __restrict__ vbuf, OptDev opt,
    const double* __restrict__ lr_p, const int64_t* __restrict__ t_p,
    const double* __restrict__ terms, const double* __restrict__ scalars, LossDev loss,
    double* __restrict__ step_loss, double* __restrict__ step_cmd) {
  __shared__ uint32_t s_touch[1024];
  __shared__ int s_leaf[TPCB_MAX_LEAF + 2];
  const StepDesc sd = steps[step];
  const int n_src = sd.n_src, n_tgt = sd.n_tgt;
  const int n_all = n_src + (use_cmd ? n_tgt : 0);
  const int G = min(n_all, n_slots);
  for (int c = threadIdx.x; c < G; c += blockDim.x) s_touch[c] = touched[c];
  if (threadIdx.x <= M.n_leaf_max) s_leaf[threadIdx.x] = threadIdx.x ? M.leafW[threadIdx.x] : 0;
  if (threadIdx.x == 0) s_leaf[M.n_leaf_max + 1] = M.tail_lo;
  __syncthreads();

  // loss value of the step (fixed order), costmodel.py:539-550
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double sq = 0.0, rel = 0.0;
    for (int i = threadIdx.x; i < n_src; i += 32) {
      sq += terms[2 * i];
      rel += terms[2 * i + 1];
    }
    sq = warp_sum_d(sq);
    rel = warp_sum_d(rel);
    if (threadIdx.x == 0 && step_loss) {
      const double n = (double)sd.n_norm;
      double v = loss.mode == kLossMse ? sq / n
                 : loss.mode == kLossMape ? rel / n
                                          : sq / n + loss.lambda * (rel / n);
      double cmdv = 0.0;
      if (use_cmd) {
        cmdv = scalars[0];
        if (add_cmd) v += loss.alpha * cmdv;  // once across data-parallel ranks
      }
      step_loss[step] = v;
      if (step_cmd) step_cmd[step] = cmdv;
    }
  }

  float lr = 0.f, bc1 = 1.f, bc2 = 1.f;
  if (opt.kind != kOptNone) {
    lr = (float)lr_p[0];
    if (opt.kind == kOptAdam) {
      const double t = (double)(t_p[0] + step + 1);
      bc1 = (float)(1.0 - pow(opt.beta1, t));
      bc2 = (float)(1.0 - pow(opt.beta2, t));
    }
  }
  const float b1 = (float)opt.beta1, b2 = (float)opt.beta2, eps = (float)opt.eps,
              wd = (float)opt.weight_decay;
  const float omb1 = (float)(1.0 - opt.beta1), omb2 = (float)(1.0 - opt.beta2);
  // 4 parameters per thread: tensors start on 16-byte boundaries, so a group
  // never straddles two tensors and shares one region bit
  const int n4 = M.total >> 2;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += gridDim.x * blockDim.x) {
    const int p = q << 2;
    const uint32_t want = 1u << region_bit(M, p, s_leaf);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* src = reinterpret_cast<const float4*>(partial + p);
    const size_t st4 = stride >> 2;
    int c = 0;
    for (; c + 4 <= G; c += 4) {  // 4 slots in flight, summed in slot order
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0, v2 = v0, v3 = v0;
      if (s_touch[c] & want) v0 = src[(size_t)c * st4];
      if (s_touch[c + 1] & want) v1 = src[(size_t)(c + 1) * st4];
      if (s_touch[c + 2] & want) v2 = src[(size_t)(c + 2) * st4];
      if (s_touch[c + 3] & want) v3 = src[(size_t)(c + 3) * st4];
      g.x += v0.x; g.y += v0.y; g.z += v0.z; g.w += v0.w;
      g.x += v1.x; g.y += v1.y; g.z += v1.z; g.w += v1.w;
      g.x += v2.x; g.y += v2.y; g.z += v2.z; g.w += v2.w;
      g.x += v3.x; g.y += v3.y; g.z += v3.z; g.w += v3.w;
    }
    for (; c < G; ++c) {
      if (s_touch[c] & want) {
        const float4 v = src[(size_t)c * st4];
        g.x += v.x; g.y += v.y; g.z += v.z; g.w += v.w;
      }
    }
    if (grad_out) *reinterpret_cast<float4*>(grad_out + p) = g;
    if (opt.kind == kOptNone) continue;
    float4 w = *reinterpret_cast<float4*>(P + p);
    float gg[4] = {g.x, g.y, g.z, g.w};
    float ww[4] = {w.x, w.y, w.z, w.w};
    if (opt.kind == kOptSgd) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float gj = gg[j];
        if (wd != 0.f) gj = gj + wd * ww[j];
        ww[j] = ww[j] - lr * gj;
      }
    } else {
      const float4 m4 = *reinterpret_cast<float4*>(mbuf + p);
      const float4 v4 = *reinterpret_cast<float4*>(vbuf + p);
      float mm[4] = {m4.x, m4.y, m4.z, m4.w};
      float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float gj = gg[j];
        if (wd != 0.f) gj = gj + wd * ww[j];
        mm[j] = __fadd_rn(__fmul_rn(mm[j], b1), __fmul_rn(omb1, gj));
        vv[j] = __fadd_rn(__fmul_rn(vv[j], b2), __fmul_rn(__fmul_rn(omb2, gj), gj));
        ww[j] = ww[j] - __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mm[j], bc1)),
                                  __fadd_rn(sqrtf(__fdiv_rn(vv[j], bc2)), eps));
      }
      *reinterpret_cast<float4*>(mbuf + p) = make_float4(mm[0], mm[1], mm[2], mm[3]);
      *reinterpret_cast<float4*>(vbuf + p) = make_float4(vv[0], vv[1], vv[2], vv[3]);
    }
    *reinterpret_cast<float4*>(P + p) = make_float4(ww[0], ww[1], ww[2], ww[3]);
  }
}

// standalone optimizer over a given gradient vector (nn.Adam.step drop-in)
__global__ void optimizer_kernel(int n, const float* __restrict__ grad, float* __restrict__ P,
                                 float* __restrict__ mbuf, float* __restrict__ vbuf, OptDev opt,
                                 double lr_d, double t_d) {
  const float lr = (float)lr_d;
  const float bc1 = (float)(1.0 - pow(opt.beta1, t_d)), bc2 = (float)(1.0 - pow(opt.beta2, t_d));
  const float b1 = (float)opt.beta1, b2 = (float)opt.beta2, eps = (float)opt.eps,
              wd = (float)opt.weight_decay;
  const float omb1 = (float)(1.0 - opt.beta1), omb2 = (float)(1.0 - opt.beta2);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    float g = grad[p], w = P[p];
    if (wd != 0.f) g = g + wd * w;
    if (opt.kind == kOptSgd) {
      P[p] = w - lr * g;
      continue;
    }
    float m = mbuf[p], v = vbuf[p];
    m = __fadd_rn(__fmul_rn(m, b1), __fmul_rn(omb1, g));
    v = __fadd_rn(__fmul_rn(v, b2), __fmul_rn(__fmul_rn(omb2, g), g));
    mbuf[p] = m;
    vbuf[p] = v;
    P[p] = w - __fdiv_rn(__fmul_rn(lr, __fdiv_rn(m, bc1)), __fadd_rn(sqrtf(__fdiv_rn(v, bc2)), eps));
  }
}

// Adam / SGD from a (data-parallel all-reduced) gradient vector; lr and the
// step count before the epoch in device memory (graph replay across epochs)
__global__ void opt_from_grad_kernel(int n, const float* __restrict__ grad, float* __restrict__ P,
                                     float* __restrict__ mbuf, float* __restrict__ vbuf,
                                     OptDev opt, const double* __restrict__ lr_p,
                                     const int64_t* __restrict__ t_p, int step) {
  const float lr = (float)lr_p[0];
  const double t = (double)(t_p[0] + step + 1);
  const float bc1 = (float)(1.0 - pow(opt.beta1, t)), bc2 = (float)(1.0 - pow(opt.beta2, t));
  const float b1 = (float)opt.beta1, b2 = (float)opt.beta2, eps = (float)opt.eps,
              wd = (float)opt.weight_decay;
  const float omb1 = (float)(1.0 - opt.beta1), omb2 = (float)(1.0 - opt.beta2);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    float g = grad[p], w = P[p];
    if (wd != 0.f) g = g + wd * w;
    if (opt.kind == kOptSgd) {
      P[p] = w - lr * g;
      continue;
    }
    float m = mbuf[p], v = vbuf[p];
    m = __fadd_rn(__fmul_rn(m, b1), __fmul_rn(omb1, g));
    v = __fadd_rn(__fmul_rn(v, b2), __fmul_rn(__fmul_rn(omb2, g), g));
    mbuf[p] = m;
    vbuf[p] = v;
    P[p] = w - __fdiv_rn(__fmul_rn(lr, __fdiv_rn(m, bc1)), __fadd_rn(sqrtf(__fdiv_rn(v, bc2)), eps));
  }
}

__global__ void transpose_kernel(const float* __restrict__ P, float* __restrict__ PT, T2Table tt) {
  const int total = tt.cum[tt.n];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    int lo = 0, hi = tt.n - 1;
    while (lo < hi) {  // last tensor whose cum <= e
      const int mid = (lo + hi + 1) >> 1;
      if (tt.cum[mid] <= e)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int i = e - tt.cum[lo];
    const int K = tt.rows[lo], N = tt.cols[lo];
    const int k = i / N, n = i - k * N;
    PT[tt.off[lo] + n * K + k] = P[tt.off[lo] + i];
  }
}

}  // namespace

int launch_reduce_apply(const Model& M, const TrainWs& ws, const StepDesc* steps, int step,
                        int use_cmd, int add_cmd, float* grad_out, float* P, float* m, float* v,
                        const OptDev& opt, const double* lr, const int64_t* t,
                        const LossDev& loss, double* step_loss, double* step_cmd,
                        cudaStream_t stream) {
  const int grid = min(ceil_div(M.total / 4, 256), kNumSMs * 8);
  reduce_apply_kernel<<<grid, 256, 0, stream>>>(M, ws.partial, ws.slot_stride, ws.touched, steps,
                                                step, ws.n_slots, use_cmd, add_cmd, grad_out, P, m,
                                                v, opt, lr, t, ws.terms, ws.scalars, loss,
                                                step_loss, step_cmd);
  TPCB_LAUNCH_CHECK("reduce_apply");
  return TPCB_OK;
}

int launch_opt_from_grad(const Model& M, const float* grad, float* P, float* m, float* v,
                         const OptDev& opt, const double* lr, const int64_t* t, int step,
                         cudaStream_t stream) {
  const int grid = min(ceil_div(M.total, 256), kNumSMs * 8);
  opt_from_grad_kernel<<<grid, 256, 0, stream>>>(M.total, grad, P, m, v, opt, lr, t, step);
  TPCB_LAUNCH_CHECK("opt_from_grad");
  return TPCB_OK;
}

int launch_transpose(const tpcb_model* m, const float* P, float* PT, cudaStream_t stream) {
  const T2Table& tt = m->t2;
  const int total = tt.cum[tt.n];
  if (total == 0) return TPCB_OK;
  const int grid = min(ceil_div(total, 256), kNumSMs * 4);
  transpose_kernel<<<grid, 256, 0, stream>>>(P, PT, tt);
  TPCB_LAUNCH_CHECK("transpose");
  return TPCB_OK;
}

int launch_optimizer(int n, const float* grad, float* P, float* m, float* v, const OptDev& opt,
                     double lr, double t, cudaStream_t stream) {
  const int grid = min(ceil_div(n, 256), kNumSMs * 4);
  optimizer_kernel<<<grid, 256, 0, stream>>>(n, grad, P, m, v, opt, lr, t);
  TPCB_LAUNCH_CHECK("optimizer");
  return TPCB_OK;
}

}  // namespace tpcb
