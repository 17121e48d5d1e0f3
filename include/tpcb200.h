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
#define TPCB_FEAT_PAD 32  /* packed row stride (128-byte rows) */
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

#ifdef __cplusplus
}
#endif
#endif /* TPCB200_H */
