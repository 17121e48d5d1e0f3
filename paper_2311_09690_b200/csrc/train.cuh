// Shared declarations of the training-step kernels (train.cu, optim.cu, capi).
#pragma once

#include "common.cuh"

namespace tpcb {

constexpr int kMaxCmdOrder = 8;
constexpr double kCmdSupportFloor = 1e-6;  // costmodel.py:29
enum { kLossHybrid = 0, kLossMse = 1, kLossMape = 2 };
enum { kOptNone = 0, kOptAdam = 1, kOptSgd = 2 };

// one optimizer step of an epoch plan (8 int32, host layout in training.py):
// the step's sample indices are batch[off .. off+n_src+n_tgt); the loss is
// normalised by n_norm (the global batch under data parallelism); z rows of
// this rank's source/target samples sit at src_pos / ns_glob+tgt_pos of the
// global [zs; zt] matrix the CMD statistics run over.
struct StepDesc {
  int off, n_src, n_tgt, n_norm, src_pos, ns_glob, tgt_pos, nt_glob;
};

struct OptDev {
  int kind;
  double beta1, beta2, eps, weight_decay;
};

// shared-memory plan of one training CTA (one sample of ≤ n_leaf_max rows)
struct TrainPlan {
  int R, ld, ldf;
  int oQ, oK, oV, oC, oX1, oX2, oF, oI1, oI2, oP, layer_stride, layer_base;
  int X0, H0, Hout, T1, T2, dH, dA, dB, dQ, dK, dV, dF, S;
  int uw, dv, zx, zv, zp, u, du0, du1, dzx, dzp, dzv, dflat, misc;
  int cmd, cmd_cols;
  int stage_cap, stage0, stage1;  // double-buffered weight stage
  int total;  // floats
};

TrainPlan make_train_plan(const Model& M, int l_cap);

__host__ __device__ inline int round4(int v) { return (v + 3) & ~3; }

// weight stream: the fixed order in which the fwd+bwd of one sample consumes
// weight matrices (the generic training kernel, train.cu)

__host__ __device__ inline int n_fwd_entries(const Model& M, int L) {
  return 1 + 6 * M.n_layers + L + 2 + M.n_dec + 1;
}
__host__ __device__ inline int n_all_entries(const Model& M, int L) {
  return n_fwd_entries(M, L) + M.n_dec + 1 + L + 6 * M.n_layers;
}

__host__ __device__ inline void entry_shape(const Model& M, int L, int idx, int* K, int* N,
                                            int* off) {
  const int nl = M.n_layers, nd = M.n_dec, d = M.d;
  auto dec_in = [&](int j) { return j == 0 ? M.d_e : M.dec[j - 1]; };
  const int nf = n_fwd_entries(M, L);
  auto layer_mat = [&](int li, int kind) {  // 0 Wq 1 Wk 2 Wv 3 Wo 4 fhW 5 foW
    const LayerOff& lo = M.layer[li];
    switch (kind) {
      case 0: *K = d; *N = d; *off = lo.Wq; break;
      case 1: *K = d; *N = d; *off = lo.Wk; break;
      case 2: *K = d; *N = d; *off = lo.Wv; break;
      case 3: *K = d; *N = d; *off = lo.Wo; break;
      case 4: *K = d; *N = M.d_ff; *off = lo.fhW; break;
      default: *K = M.d_ff; *N = d; *off = lo.foW; break;
    }
  };
  if (idx < nf) {
    if (idx == 0) { *K = TPCB_FEAT; *N = d; *off = M.inW; return; }
    int q = idx - 1;
    if (q < 6 * nl) { layer_mat(q / 6, q % 6); return; }
    q -= 6 * nl;
    if (q < L) { *K = d; *N = M.d_e; *off = M.leafW[L] + q * d * M.d_e; return; }
    q -= L;
    if (q == 0) { *K = TPCB_DEV_FEAT; *N = M.d_dev; *off = M.devhW; return; }
    if (q == 1) { *K = M.d_dev; *N = M.d_e; *off = M.devpW; return; }
    q -= 2;
    if (q < nd) { *K = dec_in(q); *N = M.dec[q]; *off = M.decW[q]; return; }
    *K = dec_in(nd); *N = 1; *off = M.outW;
    return;
  }
  int b = idx - nf;
  if (b < nd) { const int j = nd - 1 - b; *K = dec_in(j); *N = M.dec[j]; *off = M.decW[j]; return; }
  b -= nd;
  if (b == 0) { *K = M.d_dev; *N = M.d_e; *off = M.devpW; return; }
  b -= 1;
  if (b < L) { *K = d; *N = M.d_e; *off = M.leafW[L] + b * d * M.d_e; return; }
  b -= L;
  const int li = nl - 1 - b / 6;
  const int order[6] = {5, 4, 3, 0, 1, 2};  // foW, fhW, Wo, Wq, Wk, Wv
  layer_mat(li, order[b % 6]);
}



// SGD / Adam on parameter p with its preloaded w, m, v (nn.py:136-167, fp32,
// same operation order as the oracle); shared by the slot reduce (optim.cu)
// and the tensor-core weight-gradient kernel (wgrad.cu)
__device__ __forceinline__ void apply1(int p, float g, float w, float m, float v,
                                       float* __restrict__ grad_out, float* __restrict__ P,
                                       float* __restrict__ mbuf, float* __restrict__ vbuf,
                                       const OptDev& opt, float lr, float bc1, float bc2) {
  if (grad_out) grad_out[p] = g;
  if (opt.kind == kOptNone) return;
  const float wd = (float)opt.weight_decay;
  if (wd != 0.f) g = g + wd * w;
  if (opt.kind == kOptSgd) {
    P[p] = w - lr * g;
    return;
  }
  const float b1 = (float)opt.beta1, b2 = (float)opt.beta2, eps = (float)opt.eps;
  const float omb1 = (float)(1.0 - opt.beta1), omb2 = (float)(1.0 - opt.beta2);
  m = __fadd_rn(__fmul_rn(m, b1), __fmul_rn(omb1, g));
  v = __fadd_rn(__fmul_rn(v, b2), __fmul_rn(__fmul_rn(omb2, g), g));
  mbuf[p] = m;
  vbuf[p] = v;
  P[p] = w - __fdiv_rn(__fmul_rn(lr, __fdiv_rn(m, bc1)), __fadd_rn(sqrtf(__fdiv_rn(v, bc2)), eps));
}

// ---- encoder weight gradients on the tensor cores (wgrad.cu) --------------
// The desk training kernel (train4) stores, for every encoder weight product
// y = x·W of a step, the operand rows x and dy it would otherwise fold into
// its per-sample gradient slot; wgrad_tc_kernel then forms dW = Xᵀ·dY over
// all the step's token rows (3xTF32 tcgen05, fp32 accumulation in TMEM) and
// applies the optimizer.  Operand k is a [features × rows] matrix stored as
// 32-row chunks, each chunk a K-major 128-byte-swizzled UMMA tile
// [op_rows[k] features][32 rows] (one bulk copy per chunk); step row
// g = sample position · Ls + leaf row, Ls = the step's largest leaf count
// (rows of shorter samples are zero).
constexpr int kWgOpsLayer = 10;  // HIN dQ dK dV C dA H1 dF F dT1
constexpr int kWgOps = 2 * kWgOpsLayer + 2;  // + X0, dH (input projection)
enum { kWgHIN = 0, kWgDQ, kWgDK, kWgDV, kWgC, kWgDA, kWgH1, kWgDF, kWgF, kWgDT1 };
constexpr int kWgX0 = 2 * kWgOpsLayer, kWgDH = kWgX0 + 1;
__host__ __device__ constexpr int wg_op_rows(int op) {
  return op == kWgX0 ? 32 : ((op % kWgOpsLayer == kWgDF || op % kWgOpsLayer == kWgF) && op < kWgX0 ? 128 : 64);
}
__host__ __device__ constexpr int wg_total_rows() {
  int s = 0;
  for (int k = 0; k < kWgOps; ++k) s += wg_op_rows(k);
  return s;
}
// element (feature f, step row g) of operand op in a buffer of r_cap rows
__host__ __device__ inline size_t wg_index(int op_off_rows, int op_rows, int r_cap, int f, int g) {
  const int c = g >> 5, j = g & 31;
  return (size_t)op_off_rows * r_cap + (size_t)c * op_rows * 32 + (f >> 3) * 256 + (f & 7) * 32 +
         ((((j >> 2) ^ (f & 7))) << 2) + (j & 3);
}
__host__ __device__ constexpr int wg_op_off(int op) {
  int s = 0;
  for (int k = 0; k < op; ++k) s += wg_op_rows(k);
  return s;
}
struct WgradDev {
  float* act = nullptr;  // nullptr: weight gradients in the per-sample slots (v4 path)
  int r_cap = 0;         // rows per operand (multiple of 32)
};

// one dataset on the device (packed rows from K1 + per-sample data)
struct SampleSetDev {
  const float* x;          // packed rows [*, 32]
  const int32_t* ast_row;  // first packed row of each sample
  const int32_t* n_leaf;   // leaf count of each sample
  const float* devfeat;    // [n, 6]
  const double* y;         // model-space targets (source only)
};

struct LossDev {
  int mode;      // kLoss*
  int original;  // relative term in original (decoded) space
  double lambda, offset, alpha;
  int cmd_order;
  int use_cmd;
  tpcb_boxcox norm;
};

struct TrainWs {
  float* partial;      // [n_slots][slot_stride]
  size_t slot_stride;  // >= param count
  int n_slots;
  uint32_t* touched;   // [n_slots] region bitmask (bit 0 shared, bit L leaf_embed.L)
  float* zall;         // [max rows][d_embed]
  double* terms;       // [max src][2] per-sample (sq, rel)
  double* scalars;     // [8] cmd value, loss value, ...
  size_t zall_bytes;   // size of zall (zeroed before phase 0 under data parallelism)
  int l_cap;           // largest leaf count of any sample (sizes the smem plan)
  // overlapped reduce (optim.cu): per-CTA stage completion tags written by the
  // training kernel's producer warp; nullptr = off
  unsigned long long* stage_flags = nullptr;
  const int64_t* t_tag = nullptr;  // tag of step s = t_tag[0] + s + 1
  int flag_stride = 0;
  int n_stage_words = 0;  // words of the caller's stage_flags (0: overlap off)
  WgradDev wg;            // tensor-core encoder weight gradients (train4 only)
};

// Overlapped gradient reduction + optimizer (single GPU, no CMD): the items
// of 256 parameters sorted, per batch leaf count L, by the backward stage
// after which every CTA has written their gradients (stage -1: leaf_embed of
// other leaf counts, never touched; row L = 0: mixed batches, every item at
// the final stage).
struct OvlDev {
  const int32_t* order;       // [(n_leaf_max + 1) * n_items]
  const int8_t* stage;        // [(n_leaf_max + 1) * n_items]
  unsigned long long* flags;  // [n_stages * flag_stride], owned by the training workspace
  int n_items, n_stages, flag_stride, n_leaf_max;
  unsigned poll_ns;           // stage-wait poll interval
};
constexpr int kOvlFlagStride = 1024;  // >= n_slots (tpcb_train_ws_sizes caps slots at 1024)
__host__ __device__ constexpr int ovl_stage_words(int n_layers) {
  return (2 + 2 * n_layers) * kOvlFlagStride;
}
// schedule of a model (built once per parameter layout, cached per device)
int overlap_sched(const tpcb_model* m, OvlDev* out);
int launch_reduce_overlap(const Model& M, const TrainWs& ws, const OvlDev& ov,
                          const StepDesc* steps, int step, const int32_t* batch,
                          const SampleSetDev& src, float* grad_out, float* P, float* m, float* v,
                          const OptDev& opt, const double* lr, const int64_t* t,
                          const LossDev& loss, double* step_loss, double* step_cmd,
                          int32_t* status, int grid, cudaStream_t stream);

// steps[s] = {offset of step s in batch, n_src, n_tgt, 0}; batch holds the
// source sample indices of the step followed by its target sample indices.
int launch_train(const Model& M, const float* P, const float* PT, const SampleSetDev& src,
                 const SampleSetDev& tgt, const int32_t* batch, const StepDesc* steps, int step,
                 int grid, const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                 int32_t* status, cudaStream_t stream);
int prepare_train_kernels(const Model& M, int l_cap);
// v4 (desk-shaped fast path)
bool v4_supported(const Model& M);
bool v4_fits(const Model& M, int l_cap);
int train4_blocks_per_sm(const Model& M, int l_cap);
int launch_train4(const Model& M, const float* P, const SampleSetDev& src, const SampleSetDev& tgt,
                  const int32_t* batch, const StepDesc* steps, int step, int grid,
                  const LossDev& loss, int phase, const TrainWs& ws, float* pred_out,
                  int32_t* status, cudaStream_t stream);
int launch_reduce_apply(const Model& M, const TrainWs& ws, const StepDesc* steps, int step,
                        int use_cmd, int add_cmd, float* grad_out, float* P, float* m, float* v,
                        const OptDev& opt, const double* lr, const int64_t* t,
                        const LossDev& loss, double* step_loss, double* step_cmd,
                        cudaStream_t stream, int skip_wgrad = 0);
// dW of the encoder weight matrices from the operands train4 stored
// (ws.wg), split-K over `splits` blocks per matrix → gradient slots
// 0..splits-1's region of those tensors (the slot reduce adds them in order)
bool wgrad_tc_supported(const Model& M);
int wgrad_tc_splits(const TrainWs& ws);
int launch_wgrad_tc(const Model& M, const TrainWs& ws, const StepDesc* steps, int step,
                    const int32_t* batch, const int32_t* n_leaf, int splits,
                    cudaStream_t stream);
// parameter p belongs to an encoder weight matrix (its gradient comes from wgrad_tc)
__host__ __device__ inline bool in_wgrad_region(const Model& M, int p) {
  if (p >= M.inW && p < M.inW + TPCB_FEAT * M.d) return true;
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& lo = M.layer[li];
    const int dd = M.d * M.d;
    if ((p >= lo.Wq && p < lo.Wq + dd) || (p >= lo.Wk && p < lo.Wk + dd) ||
        (p >= lo.Wv && p < lo.Wv + dd) || (p >= lo.Wo && p < lo.Wo + dd) ||
        (p >= lo.fhW && p < lo.fhW + M.d * M.d_ff) || (p >= lo.foW && p < lo.foW + M.d_ff * M.d))
      return true;
  }
  return false;
}
// optimizer step from a reduced gradient with lr / step count in device memory
int launch_opt_from_grad(const Model& M, const float* grad, float* P, float* m, float* v,
                         const OptDev& opt, const double* lr, const int64_t* t, int step,
                         cudaStream_t stream);
int launch_transpose(const tpcb_model* m, const float* P, float* PT, cudaStream_t stream);
int launch_optimizer(int n, const float* grad, float* P, float* m, float* v, const OptDev& opt,
                     double lr, double t, cudaStream_t stream);


}  // namespace tpcb
