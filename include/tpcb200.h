/*
 * tpcb200 — B200 (sm_100a) kernels for the CDMPP predictor hot path.
 *
 * C ABI: plain pointers, sizes and a cudaStream_t (passed as void*).  Every
 * pointer named d_* is device memory owned by the caller; nothing is retained
 * across calls except the host-only model handle (config + parameter layout).
 * Every entry point is stream-ordered and returns an int32 status
 * (tpcb_status); device-side findings (leaf counts out of range, Box-Cox
 * domain violations, non-finite losses) are written to the caller's device
 * status word `d_status` and mapped to the reference's exceptions by the
 * host layer once it synchronises.
 *
 * The reference (`tpcost`, pure Python/numpy) has no FFI; each function below
 * names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/tpcost).  INTEGRATION.md shows the ctypes binding.
 */
#ifndef TPCB200_H
#define TPCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes — one per reference exception class (errors.py:6-88) */
typedef enum {
  TPCB_OK = 0,
  TPCB_ERR_VALIDATION = 1,       /* ValidationError            errors.py:19 */
  TPCB_ERR_LEAF_COUNT = 2,       /* LeafCountExceeded          errors.py:23 */
  TPCB_ERR_EMPTY_BATCH = 3,      /* EmptyBatch                 errors.py:51 */
  TPCB_ERR_EMPTY_SET = 4,        /* EmptySet                   errors.py:55 */
  TPCB_ERR_DIM_MISMATCH = 5,     /* DimensionMismatch          errors.py:78 */
  TPCB_ERR_TOO_FEW_POINTS = 6,   /* TooFewPoints               errors.py:70 */
  TPCB_ERR_TOO_FEW_TASKS = 7,    /* TooFewTasks                errors.py:74 */
  TPCB_ERR_DOMAIN = 8,           /* DomainError                errors.py:35 */
  TPCB_ERR_NOT_FITTED = 9,       /* NotFitted                  errors.py:31 */
  TPCB_ERR_NONFINITE = 10,       /* NonFiniteLoss              errors.py:63 */
  TPCB_ERR_UNSUPPORTED = 11,     /* config outside this build's kernel limits */
  TPCB_ERR_CUDA = 12             /* CUDA runtime failure (tpcb_last_error) */
} tpcb_status;

#define TPCB_MAX_LAYERS 16
#define TPCB_MAX_LEAF 16
#define TPCB_MAX_DEC 8
#define TPCB_FEAT 24      /* computation-vector width, features.py:18 */
#define TPCB_FEAT_PAD 24  /* packed row stride (96-byte rows, 16-byte aligned) */
#define TPCB_DEV_FEAT 6   /* device-vector width, costmodel.py:28 */

/* CostModelConfig (costmodel.py:36-57), architecture fields only */
typedef struct {
  int32_t d_model, n_layers, n_heads, d_ff, d_embed, d_device;
  int32_t n_dec;
  int32_t dec[TPCB_MAX_DEC];
  int32_t n_leaf_max;
} tpcb_config;

typedef struct tpcb_model tpcb_model; /* opaque host handle */

/* ---- model handle: canonical tensor layout (costmodel.py:116-150) ------- */
int tpcb_model_create(const tpcb_config* cfg, tpcb_model** out);
void tpcb_model_destroy(tpcb_model* m);
int64_t tpcb_model_param_count(const tpcb_model* m);
int32_t tpcb_model_tensor_count(const tpcb_model* m);
/* name/offset/shape of tensor i in the flat fp32 parameter vector;
 * cols == 0 for 1-D tensors */
int tpcb_model_tensor_info(const tpcb_model* m, int32_t i, char* name, int32_t name_cap,
                           int64_t* offset, int32_t* rows, int32_t* cols);
const char* tpcb_status_string(int32_t status);
/* last CUDA error text recorded by this library (thread-local) */
const char* tpcb_last_error(void);

/* ---- K1: featurize + bucket pack ----------------------------------------
 * Replaces features.encode_input / positional_encoding (features.py:248-279)
 * plus costmodel._group_by_leaf and the per-bucket np.stack
 * (costmodel.py:181-190, 248-251).  Ragged input (input order):
 *   d_vectors  [n_tok, 24]  f32 (vec_is_f64=0) or f64 (vec_is_f64=1) leaf vectors
 *   d_ordering [n_tok]      int32 serialized positions (CompactAst.ordering)
 *   d_leaf_off [n_ast+1]    int64 token offsets
 * Output: the packed fixed-stride layout (all device, caller-allocated to the
 * sizes from tpcb_pack_sizes):
 *   x          [n_tiles_max*R, 32] f32  leaf vector + PE, zero padded
 *   row_ast    [n_tiles_max*R]     int32 input AST index of each row, -1 = pad
 *   tile_L / tile_first / tile_count [n_tiles_max] int32
 *   perm       [n_ast] int32  stable argsort of n_leaf (bucket order)
 *   ast_row    [n_ast] int32  flat row of each AST's first leaf
 *   bucket_off [n_leaf_max+2] int32
 *   n_tiles    [1] int32 (actual tile count; kernels over n_tiles_max exit early)
 */
typedef struct {
  int32_t rows_per_tile; /* R: 32, 64 or 128 */
  int32_t n_tiles_max;
  float* x;
  int32_t* row_ast;
  int32_t* tile_L;
  int32_t* tile_first;
  int32_t* tile_count;
  int32_t* perm;
  int32_t* ast_row;
  int32_t* bucket_off;
  int32_t* n_tiles;
} tpcb_packed;

int tpcb_pack_sizes(int64_t n_ast, int64_t n_tok, int32_t n_leaf_max, int32_t rows_per_tile,
                    int32_t* n_tiles_max, size_t* workspace_bytes);
int tpcb_featurize_pack(const void* d_vectors, int32_t vec_is_f64, const int32_t* d_ordering,
                        const int64_t* d_leaf_off, int64_t n_ast, int64_t n_tok,
                        int32_t n_leaf_max, const double* pe_denom /* host [12]; NULL = rows
                                                                      already encoded, no PE */,
                        void* d_workspace, size_t workspace_bytes, tpcb_packed* out,
                        int32_t* d_status, void* stream);

/* PE table alone, fp64 (features.positional_encoding, features.py:248-263):
 * d_out[n, 24]; pe_denom = θ^(2δ/24), δ = 0..11 (host array). */
int tpcb_positional_encoding(const int32_t* d_ordering, int64_t n, const double* pe_denom,
                             double* d_out, void* stream);

/* ---- K0: compact-AST builder (features.build_compact_ast + compute_vector,
 * features.py:155-245) ----------------------------------
 * Input: a forest of n_prog programs as pre-order node arrays —
 *   d_node_off [n_prog+1] i64, d_parent [N] i32 (program-local, -1 = root),
 *   d_extent [N] i64 (loop extent >= 1, 0 = compute leaf), d_annot [N] u8
 *   (bit 0 vectorize, 1 unroll, 2 parallel), d_leaf_off [n_prog+1] i64,
 *   d_stats [NL, 9] i64 (ComputeStats fields in ir.py:53-64 order, leaves in
 *   pre-order; host-validated: counts < 2^56, extents < 2^63).
 * Output: d_vectors [NL, 24] f64 (compute_vector), d_ordering [NL] i32,
 *   d_serialized [N + NL] i32 (program p at node_off[p] + leaf_off[p]).
 * *d_first_overflow = smallest program index whose enclosing extent product
 * exceeds 2^62 (the reference's OverflowError, features.py:165-168), or
 * UINT64_MAX.  Integer math exact, int->float and entry 22 correctly rounded;
 * log2 within 1 ulp. */
int tpcb_build_compact(const int64_t* d_node_off, const int32_t* d_parent,
                       const int64_t* d_extent, const uint8_t* d_annot, const int64_t* d_leaf_off,
                       const int64_t* d_stats, int64_t n_prog, double* d_vectors,
                       int32_t* d_ordering, int32_t* d_serialized,
                       unsigned long long* d_first_overflow, void* stream);

/* Box-Cox label normaliser (dataset.py:69-115) */
typedef struct {
  double lambda_bc, shift, t_mean, t_std;
  int32_t enabled; /* 0 = no decode */
} tpcb_boxcox;



/* ---- K2+K3: fused encoder + head forward (inference) ---------------------
 * Replaces costmodel.forward/_forward/_forward_group (costmodel.py:193-269)
 * and, when norm->enabled, BoxCoxNormalizer.decode (dataset.py:113-115) as in
 * predict_batch (costmodel.py:803-806).
 *   d_params  flat fp32 parameters (tpcb_model_tensor_info layout)
 *   d_devfeat [n_ast, 6] f32 device features (log2(1+spec), features.py:266)
 * Outputs in input order (nullable except pred):
 *   d_pred [n_ast] f32 (model space), d_zx [n_ast, d_embed], d_zv [n_ast,
 *   d_device], d_z [n_ast, d_embed] f32, d_latency [n_ast] f64 seconds (NaN +
 *   TPCB_ERR_DOMAIN in *d_status where λt+1 <= 0). */
int tpcb_forward(const tpcb_model* m, const float* d_params, const tpcb_packed* pk,
                 const float* d_devfeat, int64_t n_ast, const tpcb_boxcox* norm,
                 float* d_pred, float* d_zx, float* d_zv, float* d_z, double* d_latency,
                 int32_t* d_status, void* stream);

/* bf16 tensor-core mode of tpcb_forward (the C5 sweep path):
 * the desk encoder's GEMMs run on tcgen05 (bf16 operands, fp32 accumulation
 * in TMEM); LayerNorm / softmax / head in fp32, decode in fp64.  Desk-shaped
 * models only; pk->rows_per_tile must be 128.  d_img: device workspace of
 * tpcb_forward_bf16_workspace() bytes (bf16 weight image, rebuilt per call).
 * Accuracy is stated separately from the fp32 parity mode. */
size_t tpcb_forward_bf16_workspace(void);
int tpcb_forward_bf16(const tpcb_model* m, const float* d_params, const tpcb_packed* pk,
                      const float* d_devfeat, int64_t n_ast, const tpcb_boxcox* norm, void* d_img,
                      float* d_pred, float* d_zx, float* d_zv, float* d_z, double* d_latency,
                      int32_t* d_status, void* stream);

/* costmodel.metrics (costmodel.py:577-591): d_out = {MAPE, RMSE, MSPE} (fp64) */
int tpcb_metrics(const double* d_pred, const double* d_y, int64_t n, double* d_out, void* stream);

/* ---- K4–K7: training ------------------------------------------------------
 * Loss selection (costmodel.LossSpec, costmodel.py:511-526). */
typedef struct {
  int32_t mode;           /* 0 hybrid, 1 mse, 2 mape */
  int32_t original_space; /* relative term on decoded latencies (needs norm) */
  double lambda_hybrid, offset, alpha_cmd;
  int32_t cmd_order;      /* K <= 8 */
  tpcb_boxcox norm;
} tpcb_loss;

/* ---- large-model path (full_reference_config) -------------
 * Layer-by-layer forward for configurations the fused kernels do not fit
 * (tpcb_forward_fits == 0): every product is a 3xTF32 tcgen05 GEMM (TMA-fed,
 * fp32 accumulation in TMEM); attention / LayerNorm / device MLP / output on
 * CUDA cores.  Replaces costmodel.forward (costmodel.py:193-269) for those
 * configs.  Image = transposed (hi, lo) weight operands (+ the plain ones the
 * backward needs), rebuilt by tpcb_large_prepare after every parameter
 * change; zero-fill it once at allocation.  h_perm / h_tok_off: the
 * HOST bucket order (stable argsort of n_leaf) and the token offsets in it. */
int32_t tpcb_forward_fits(const tpcb_model* m, int32_t rows_per_tile);
/* preferred rows_per_tile for tpcb_forward: 128 when the desk-shaped fp32
 * kernel applies (row-per-thread FFMA products over smem-staged weight
 * tiles, csrc/forward_f32.cu), else 64 (the generic kernel). */
int32_t tpcb_forward_rows(const tpcb_model* m);
int tpcb_large_sizes(const tpcb_model* m, int64_t n_ast, int64_t n_tok, size_t* image_bytes,
                     size_t* act_bytes);
/* flags: bit 0 = also the backward operands, bit 1 = entry table already
 * resident in this image (skip its upload, which synchronises the stream) */
int tpcb_large_prepare(const tpcb_model* m, const float* d_params, void* d_image,
                       int32_t flags, void* stream);
int tpcb_large_forward(const tpcb_model* m, const float* d_params, const void* d_image,
                       const tpcb_packed* pk, const int32_t* h_perm, const int32_t* h_tok_off,
                       const float* d_devfeat, int64_t n_ast, const tpcb_boxcox* norm,
                       void* d_act, size_t act_bytes, float* d_pred, float* d_zx, float* d_zv,
                       float* d_z, double* d_latency, int32_t* d_status, void* stream);
/* Large-path training (costmodel.backward, costmodel.py:280-336, 343-423,
 * 529-570, for configs the fused trainer cannot hold): one batch's forward
 * (activations kept), loss and full backward on the tensor cores.  Inputs are
 * dataset-resident: K1-packed rows d_x + d_ast_row, device features
 * [n, 6], model-space targets d_y; the batch is h_idx (dataset indices in
 * bucket order, HOST) with token offsets h_tok_off.  Writes the whole flat
 * gradient d_grad (normalised by n_norm, the global batch) and the batch-mean
 * loss d_loss[0].  Transformed-space losses without CMD (else UNSUPPORTED). */
/* one batch of the large path with its dataset: K1-packed rows (x,
 * ast_row) and device features of the dataset, the batch's dataset indices
 * in bucket order (stable by leaf count) with token offsets, and the input
 * position of each bucket-order row (the CMD statistics run in input order) */
typedef struct {
  const float* x;
  const int32_t* ast_row;
  const float* devfeat;
  const int32_t* h_idx;     /* [n] */
  const int32_t* h_tok_off; /* [n + 1] */
  const int32_t* h_pos;     /* [n] */
  int64_t n;
} tpcb_large_batch;

/* workspace of tpcb_large_loss_backward for a source batch (n_ast, n_tok)
 * and an optional CMD target batch (n_ast_t, n_tok_t; 0 without) */
int tpcb_large_train_ws(const tpcb_model* m, int64_t n_ast, int64_t n_tok, int64_t n_ast_t,
                        int64_t n_tok_t, size_t* ws_bytes);
/* costmodel.backward (costmodel.py:529-570) through the large path: forward
 * (activations kept), loss (hybrid / mse / mape, transformed or original
 * space), CMD with a target batch when loss->alpha_cmd > 0 (tgt != NULL;
 * h_src_pos = input position of each bucket-order source row), backward;
 * every GEMM 3xTF32 on tcgen05.  d_grad (rewritten) = the full gradient,
 * d_loss[0] = loss + alpha·CMD, d_cmd[0] (nullable) = CMD. */
int tpcb_large_loss_backward(const tpcb_model* m, const float* d_params, const void* d_image,
                             const float* d_x, const int32_t* d_ast_row, const float* d_devfeat,
                             const double* d_y, const int32_t* h_idx, const int32_t* h_tok_off,
                             const int32_t* d_idx /* device copies or NULL */,
                             const int32_t* d_tok_off, int64_t n_batch, const tpcb_loss* loss,
                             double n_norm, const int32_t* h_src_pos,
                             const tpcb_large_batch* tgt, void* d_ws, size_t ws_bytes,
                             float* d_grad, double* d_loss, double* d_cmd, int32_t* d_status,
                             void* stream);
/* the GEMM alone: C[M,N] = A[M,K] B[N,K]^T, fp32 row-major in/out (3xTF32) */
size_t tpcb_gemm3_ws(int64_t M, int32_t N, int32_t K);
int tpcb_gemm3(const float* d_a, const float* d_b, int64_t M, int32_t N, int32_t K, float* d_c,
               int32_t ldc, void* d_ws, size_t ws_bytes, void* stream);
int tpcb_gemm3_presplit(const float* a_hi, const float* a_lo, const float* b_hi,
                        const float* b_lo, int64_t M, int32_t N, int32_t Kp, float* d_c,
                        int32_t ldc, void* stream);

/* one dataset on the device: packed rows from tpcb_featurize_pack + per-sample data */
typedef struct {
  const float* x;          /* packed rows [*, 32] */
  const int32_t* ast_row;  /* [n] first packed row of each sample */
  const int32_t* n_leaf;   /* [n] */
  const float* devfeat;    /* [n, 6] */
  const double* y;         /* [n] model-space targets (source set only) */
} tpcb_samples;

/* optimizer (nn.Adam / nn.Sgd, nn.py:127-167) */
typedef struct {
  int32_t kind; /* 0 none, 1 adam, 2 sgd */
  double beta1, beta2, eps, weight_decay;
} tpcb_optim;

/* caller-allocated training workspace (sizes from tpcb_train_ws_sizes) */
typedef struct {
  float* partial;       /* [n_slots * slot_stride] per-CTA gradient slots */
  int64_t slot_stride;
  int32_t n_slots;
  uint32_t* touched;    /* [n_slots] */
  float* zall;          /* [max_rows * d_embed] */
  double* terms;        /* [max_rows * 2] */
  double* scalars;      /* [8]: [0] CMD value, [1] loss value */
  int64_t zall_floats;  /* size of zall (global rows × d_embed) */
  int32_t l_cap;        /* largest leaf count among the samples (≤ n_leaf_max) */
  /* overlapped reduce + optimizer (single GPU, no CMD): per-backward-stage
   * completion counters owned by this workspace, stage_flag_words long
   * (tpcb_train_ws_sizes); NULL runs the step's reduction sequentially after
   * the training kernel.  The overlap is taken only when every training CTA
   * of a step is co-resident with the reduce blocks (occupancy check). */
  uint64_t* stage_flags;
  int64_t stage_flag_words;
  /* encoder weight gradients on the tensor cores (desk-shaped models, steps
   * without CMD): operand rows the training kernel stores for one GEMM per
   * weight matrix over the step's token rows, act_floats long
   * (tpcb_train_ws_sizes); NULL keeps them in the per-sample slots */
  float* act;
  int64_t act_floats;
} tpcb_train_ws;

/* epoch plan: steps[s] = 8 × int32 {offset into d_batch, n_src, n_tgt,
 * n_norm, src_pos, ns_glob, tgt_pos, nt_glob}: this rank's source / target
 * counts, the batch size the loss is normalised by (the global batch under
 * data parallelism) and where this rank's rows sit in the global [zs; zt]
 * CMD matrix.  d_batch holds each step's source indices then target indices. */
typedef struct {
  const int32_t* d_batch;
  const int32_t* d_steps;
  int32_t n_steps;
} tpcb_plan;

int tpcb_train_ws_sizes(const tpcb_model* m, int32_t max_rows, int32_t l_cap, int32_t* n_slots,
                        int64_t* slot_stride, int64_t* zall_floats, int64_t* terms_doubles,
                        int64_t* stage_flag_words, int64_t* act_floats);
/* refresh the transposed copy of every 2-D weight (read by the backward) */
int tpcb_transpose_params(const tpcb_model* m, const float* d_params, float* d_params_t,
                          void* stream);
/* costmodel.backward (costmodel.py:529-570): loss value → ws->scalars[1],
 * CMD value → ws->scalars[0], gradient of every parameter → d_grad [P]
 * (zeros for tensors the batch does not touch), predictions → d_pred. */
int tpcb_loss_backward(const tpcb_model* m, const float* d_params, const float* d_params_t,
                       const tpcb_samples* src, const tpcb_samples* tgt, const int32_t* d_batch,
                       int32_t n_src, int32_t n_tgt, const tpcb_loss* loss,
                       const tpcb_train_ws* ws, void* d_step_scratch /* 16 B */, float* d_grad,
                       float* d_pred, int32_t* d_status, void* stream);
/* nn.Adam.step / nn.Sgd.step over a flat vector of n floats (t = 1-based
 * step count).  With a model handle n is its parameter count and d_params_t
 * (when non-NULL) is refreshed; m may be NULL for a bare vector. */
int tpcb_optimizer_step(const tpcb_model* m, int64_t n, float* d_params, float* d_params_t,
                        const float* d_grad, float* d_m, float* d_v, const tpcb_optim* opt,
                        double lr, int64_t t, void* stream);
/* float64 optimizer step for the drop-in nn.Adam / nn.Sgd (nn.py:136-167):
 * d_params / d_grad / d_m / d_v float64 [n] (m, v Adam only, zero before the
 * first step); bc1 = 1 - beta1**t, bc2 = 1 - beta2**t computed by the caller.
 * Same IEEE operation sequence as the reference's numpy update (bit-exact). */
int tpcb_optimizer_step_f64(int64_t n, double* d_params, const double* d_grad, double* d_m,
                            double* d_v, const tpcb_optim* opt, double lr, double bc1,
                            double bc2, void* stream);
/* ---- data parallel: NCCL communicator (one process per GPU) --------------
 * rank 0 creates the id, the host broadcasts it (torch.distributed), every
 * rank creates its communicator; tpcb_train_epoch all-reduces each step's
 * gradient (and the CMD latents) on the training stream. */
typedef struct tpcb_comm tpcb_comm;
int tpcb_nccl_unique_id(void* out, int32_t cap /* >= 128 */);
int tpcb_nccl_comm_create(const void* id, int32_t nranks, int32_t rank, tpcb_comm** out);
void tpcb_nccl_comm_destroy(tpcb_comm* c);
int tpcb_nccl_allreduce_sum(tpcb_comm* c, void* d_buf, int64_t count, int32_t is_f64,
                            void* stream);

/* captured-epoch cache (a CUDA graph replayed while the arguments match) */
typedef struct tpcb_graph tpcb_graph;
int tpcb_graph_create(tpcb_graph** out);
void tpcb_graph_destroy(tpcb_graph* g);

/* the train/finetune inner loop (costmodel.py:700-706, 759-773) for one
 * epoch: per step backward (+CMD) → reduce → optimizer → transpose.
 * lr and the step count before the epoch are read from device memory;
 * per-step loss / CMD values land in d_step_loss / d_step_cmd.  With a
 * graph handle the whole epoch is captured once and replayed (the stream
 * must then be a non-legacy stream).  prof_ms (host, [3], nullable) runs the
 * epoch uncaptured and returns the summed device time of the fwd/bwd kernels,
 * the reduce+optimizer kernels and the transpose kernels (synchronises).
 * comm (nullable): data-parallel communicator; then d_grad [param_count]
 * receives the all-reduced gradient each step. */
int tpcb_train_epoch(const tpcb_model* m, float* d_params, float* d_params_t, float* d_m,
                     float* d_v, const tpcb_samples* src, const tpcb_samples* tgt,
                     const tpcb_plan* plan, const tpcb_loss* loss, const tpcb_optim* opt,
                     const double* d_lr, const int64_t* d_t0, const tpcb_train_ws* ws,
                     double* d_step_loss, double* d_step_cmd, int32_t* d_status,
                     tpcb_graph* graph, double* prof_ms, tpcb_comm* comm, float* d_grad,
                     void* stream);

/* ---- K6: CMD between two sets (costmodel.cmd, costmodel.py:489-503) ------
 * d_z = [zs; zt] row-major [(ns+nt), de] (f32 or f64); value → d_value[0];
 * when d_grad != NULL, dCMD/dz for every row (fp64, same layout). */
int tpcb_cmd(const void* d_z, int32_t z_is_f64, int64_t ns, int64_t nt, int32_t de, int32_t k,
             double* d_value, double* d_grad, void* stream);

/* Grid version for large sets (cmd_between over whole datasets; SURVEY 8(d)
 * "full-set CMD is HBM-bound"): same value / gradient contract as tpcb_cmd,
 * de <= 128.  Three streaming passes over Z (extrema + sums, central power
 * sums, gradient) with fixed-order chunk combines (chunks of 2,048 rows of
 * one set, bitwise reproducible; cmd(S, S) == 0 exactly).  d_ws:
 * tpcb_cmd_grid_ws(ns, nt, de, k) bytes. */
size_t tpcb_cmd_grid_ws(int64_t ns, int64_t nt, int32_t de, int32_t k);
int tpcb_cmd_grid(const void* d_z, int32_t z_is_f64, int64_t ns, int64_t nt, int32_t de,
                  int32_t k, double* d_value, double* d_grad, void* d_ws, size_t ws_bytes,
                  void* stream);

/* ---- K8–K11: KMeans task sampler (sampling.py:40-144), float64 ----------
 * x: [n, d] row-major fp64 on the device (d ≤ 128).  Distances follow the
 * reference's exact recipe (numpy pairwise summation order), so assignments
 * and centres are bit-identical to sampling.kmeans. */
int tpcb_kmeans_ws_size(int64_t n, int32_t d, int32_t kappa, size_t* bytes);
/* k-means++ (sampling.py:45-60): centre 0 = x[first]; closest = dist²; total */
int tpcb_kmeanspp_init(const double* d_x, int64_t n, int32_t d, int64_t first, double* d_centers,
                       double* d_closest, double* d_total, void* ws, size_t ws_bytes,
                       void* stream);
/* centre i: u >= 0 → first j with cumsum(closest/total)/last > u (the
 * Generator.choice draw); u < 0 → j = direct (the rng.integers branch when
 * total == 0).  Then closest = min(closest, dist²(x, c_i)), total = Σ. */
int tpcb_kmeanspp_step(const double* d_x, int64_t n, int32_t d, int32_t i, double u,
                       int64_t direct, double* d_centers, double* d_closest, double* d_total,
                       int64_t* d_chosen, void* ws, size_t ws_bytes, void* stream);
/* steps i0 .. i1-1 with host pre-drawn uniforms h_u[i1-i0] (the reference's
 * rng.random() per step while the total is > 0), no host synchronisation;
 * *d_zero_step (caller-initialised to INT32_MAX) = the first step whose total
 * was 0 (the reference then draws rng.integers: replay from there). */
int tpcb_kmeanspp_steps(const double* d_x, int64_t n, int32_t d, int32_t i0, int32_t i1,
                        const double* h_u, double* d_centers, double* d_closest, double* d_total,
                        int32_t* d_zero_step, void* ws, size_t ws_bytes, void* stream);
/* Lloyd assignment: first-index argmin of sqrt distance, own distance, counts */
int tpcb_kmeans_assign(const double* d_x, int64_t n, int32_t d, const double* d_centers,
                       int32_t kappa, int64_t* d_assign, double* d_own, int32_t* d_counts,
                       void* stream);
/* centres = member means in point order (empty clusters keep their centre) */
/* K8, tensor-core mode: the same assignment (d <= 32) with the ranking score
 * ||c||^2 - 2 x.c formed by a 3xTF32 tcgen05 GEMM, a fused per-point top-4 scan,
 * and an exact float64 re-rank of the 4 candidates (numpy summation order).
 * Equals tpcb_kmeans_assign whenever the true nearest centre is among the
 * candidates (>= 99.9 % agreement required by the north_star; measured in
 * tests/test_gpu_kmeans.py).  d_ws: tpcb_kmeans_assign_tc_ws(kappa) bytes. */
size_t tpcb_kmeans_assign_tc_ws(int32_t kappa);
int tpcb_kmeans_assign_tc(const double* d_x, int64_t n, int32_t d, const double* d_centers,
                          int32_t kappa, int64_t* d_assign, double* d_own, int32_t* d_counts,
                          void* d_ws, size_t ws_bytes, void* stream);
int tpcb_kmeans_update(const double* d_x, int64_t n, int32_t d, int32_t kappa,
                       const int64_t* d_assign, const int32_t* d_counts, double* d_centers,
                       void* ws, size_t ws_bytes, void* stream);
/* *d_flag = 1 if the two assignments differ */
/* Data-parallel KMeans (point-sharded across ranks; sampling.kmeans_sharded,
 * SURVEY 8(e)): the local pieces between the collectives.
 *   closest: closest[i] = (init ? d : min(closest[i], d)) with d = dist^2(x_i, c);
 *            d_total = sum of closest (fixed order)
 *   cdf:     p = closest / *d_total (the global total), cdf = inclusive scan in
 *            the workspace; *d_local_sum = cdf[n-1]
 *   search:  first local j with (offset + cdf[j]) / total > u, -1 if none
 *            (Generator.choice semantics over the concatenated shards)
 *   partial: per-cluster member sums in point order [kappa, d] (the update
 *            step's numerator; centres = all-reduced sums / all-reduced counts) */
int tpcb_kmeanspp_closest(const double* d_x, int64_t n, int32_t d, const double* d_center,
                          int32_t init, double* d_closest, double* d_total, void* ws,
                          size_t ws_bytes, void* stream);
int tpcb_kmeanspp_cdf(const double* d_closest, int64_t n, const double* d_total,
                      double* d_local_sum, void* ws, size_t ws_bytes, void* stream);
int tpcb_kmeanspp_search(int64_t n, double offset, double total, double u, int64_t* d_found,
                         void* ws, size_t ws_bytes, void* stream);
int tpcb_kmeans_partial(const double* d_x, int64_t n, int32_t d, int32_t kappa,
                        const int64_t* d_assign, const int32_t* d_counts, double* d_sums,
                        void* ws, size_t ws_bytes, void* stream);
int tpcb_kmeans_changed(const int64_t* d_a, const int64_t* d_b, int64_t n, int32_t* d_flag,
                        void* stream);
/* Ψ[e, t] = mean over rows of task t (rows d_task_off[t]..[t+1]) of the L2
 * distance to centre e (sampling.build_distance_table, sampling.py:109-123) */
int tpcb_distance_table(const double* d_feats, const int64_t* d_task_off, int32_t n_tasks,
                        int32_t d, const double* d_centers, int32_t kappa, double* d_psi,
                        void* stream);

/* ---- measurement helpers (bench.py) -------------------------------------
 * FP32 FFMA throughput of this GPU in TFLOP/s (d_scratch: >= 1184 floats);
 * L2 flush by overwriting a caller buffer larger than L2. */
int tpcb_probe_ffma(float* d_scratch, double* tflops_out, void* stream);
int tpcb_flush_l2(void* d_buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TPCB200_H */
