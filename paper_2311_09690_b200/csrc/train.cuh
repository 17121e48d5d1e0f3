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
                        cudaStream_t stream);
// optimizer step from a reduced gradient with lr / step count in device memory
int launch_opt_from_grad(const Model& M, const float* grad, float* P, float* m, float* v,
                         const OptDev& opt, const double* lr, const int64_t* t, int step,
                         cudaStream_t stream);
int launch_transpose(const tpcb_model* m, const float* P, float* PT, cudaStream_t stream);
int launch_optimizer(int n, const float* grad, float* P, float* m, float* v, const OptDev& opt,
                     double lr, double t, cudaStream_t stream);


}  // namespace tpcb
