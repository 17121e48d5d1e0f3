// Host side of the model handle: canonical tensor layout of the flat fp32
// parameter vector (creation order of costmodel.py:127-149), status strings
// and the thread-local CUDA error record.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace tpcb {

static thread_local char g_last_error[512] = "";

const Knobs& knobs() {
  static const Knobs k = [] {
    auto env = [](const char* name, int dflt) {
      const char* v = getenv(name);
      return v && *v ? atoi(v) : dflt;
    };
    Knobs r{};
    r.train_impl = env("TPCB_TRAIN_IMPL", 0);
    r.grid_cap = env("TPCB_GRID_CAP", 0);
    const int bk = env("TPCB_GEMM_BK", 0);
    r.gemm_bk = bk == 16 || bk == 32 ? bk : 0;  // 0: by shape (large.cu)
    r.gemm_cluster = env("TPCB_GEMM_CLUSTER", 0) ? 1 : 0;
    r.gemm_mode = env("TPCB_GEMM_MODE", 0);
    r.poll_ns = (unsigned)std::max(0, env("TPCB_POLL_NS", 256));
    r.wgrad_tc = env("TPCB_WGRAD_TC", 1) ? 1 : 0;
    return r;
  }();
  return k;
}

void set_last_error(const char* what, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%d)", what, cudaGetErrorString(e), (int)e);
}

}  // namespace tpcb

using tpcb::TensorInfo;

extern "C" const char* tpcb_last_error(void) { return tpcb::g_last_error; }

extern "C" const char* tpcb_status_string(int32_t s) {
  switch (s) {
    case TPCB_OK: return "ok";
    case TPCB_ERR_VALIDATION: return "ValidationError";
    case TPCB_ERR_LEAF_COUNT: return "LeafCountExceeded";
    case TPCB_ERR_EMPTY_BATCH: return "EmptyBatch";
    case TPCB_ERR_EMPTY_SET: return "EmptySet";
    case TPCB_ERR_DIM_MISMATCH: return "DimensionMismatch";
    case TPCB_ERR_TOO_FEW_POINTS: return "TooFewPoints";
    case TPCB_ERR_TOO_FEW_TASKS: return "TooFewTasks";
    case TPCB_ERR_DOMAIN: return "DomainError";
    case TPCB_ERR_NOT_FITTED: return "NotFitted";
    case TPCB_ERR_NONFINITE: return "NonFiniteLoss";
    case TPCB_ERR_UNSUPPORTED: return "Unsupported";
    case TPCB_ERR_CUDA: return "CudaError";
    default: return "unknown";
  }
}

extern "C" int tpcb_model_create(const tpcb_config* c, tpcb_model** out) {
  if (!c || !out) return TPCB_ERR_VALIDATION;
  *out = nullptr;
  // CostModelConfig.validate (costmodel.py:59-81), architecture part
  if (c->d_model < 1 || c->n_layers < 1 || c->n_heads < 1 || c->d_ff < 1 || c->d_embed < 1 ||
      c->d_device < 1 || c->n_leaf_max < 1 || c->n_dec < 0)
    return TPCB_ERR_VALIDATION;
  if (c->d_model % c->n_heads != 0) return TPCB_ERR_VALIDATION;
  for (int i = 0; i < c->n_dec && i < TPCB_MAX_DEC; ++i)
    if (c->dec[i] < 1) return TPCB_ERR_VALIDATION;
  if (c->n_layers > TPCB_MAX_LAYERS || c->n_leaf_max > TPCB_MAX_LEAF || c->n_dec > TPCB_MAX_DEC)
    return TPCB_ERR_UNSUPPORTED;

  tpcb_model* m = new tpcb_model();
  m->cfg = *c;
  tpcb::Model& M = m->dev;
  memset(&M, 0, sizeof(M));
  M.d = c->d_model;
  M.n_layers = c->n_layers;
  M.n_heads = c->n_heads;
  M.dh = c->d_model / c->n_heads;
  M.d_ff = c->d_ff;
  M.d_e = c->d_embed;
  M.d_dev = c->d_device;
  M.n_dec = c->n_dec;
  M.n_leaf_max = c->n_leaf_max;
  for (int i = 0; i < c->n_dec; ++i) M.dec[i] = c->dec[i];

  int64_t off = 0;
  // every tensor starts on a 16-byte boundary so the kernels can use 128-bit
  // loads on any weight matrix (padding floats stay 0 through training)
  auto add = [&](const std::string& name, int rows, int cols) -> int {
    off = (off + 3) & ~(int64_t)3;
    int at = (int)off;
    m->tensors.push_back(TensorInfo{name, off, rows, cols});
    off += (int64_t)rows * (cols ? cols : 1);
    return at;
  };
  const int d = M.d;
  M.inW = add("input.W", TPCB_FEAT, d);
  M.inb = add("input.b", d, 0);
  for (int i = 0; i < M.n_layers; ++i) {
    std::string p = "enc" + std::to_string(i) + ".";
    tpcb::LayerOff& L = M.layer[i];
    L.Wq = add(p + "attn.Wq", d, d);
    L.Wk = add(p + "attn.Wk", d, d);
    L.Wv = add(p + "attn.Wv", d, d);
    L.Wo = add(p + "attn.Wo", d, d);
    L.bq = add(p + "attn.bq", d, 0);
    L.bk = add(p + "attn.bk", d, 0);
    L.bv = add(p + "attn.bv", d, 0);
    L.bo = add(p + "attn.bo", d, 0);
    L.ln1g = add(p + "ln1.g", d, 0);
    L.ln1b = add(p + "ln1.b", d, 0);
    L.fhW = add(p + "ffn.h.W", d, M.d_ff);
    L.fhb = add(p + "ffn.h.b", M.d_ff, 0);
    L.foW = add(p + "ffn.o.W", M.d_ff, d);
    L.fob = add(p + "ffn.o.b", d, 0);
    L.ln2g = add(p + "ln2.g", d, 0);
    L.ln2b = add(p + "ln2.b", d, 0);
  }
  for (int Lf = 1; Lf <= M.n_leaf_max; ++Lf) {
    std::string p = "leaf_embed." + std::to_string(Lf) + ".";
    M.leafW[Lf] = add(p + "W", Lf * d, M.d_e);
    M.leafb[Lf] = add(p + "b", M.d_e, 0);
  }
  M.devhW = add("dev.hidden.W", TPCB_DEV_FEAT, M.d_dev);
  M.devhb = add("dev.hidden.b", M.d_dev, 0);
  M.devpW = add("dev.proj.W", M.d_dev, M.d_e);
  M.devpb = add("dev.proj.b", M.d_e, 0);
  int w = M.d_e;
  for (int i = 0; i < M.n_dec; ++i) {
    std::string p = "dec." + std::to_string(i) + ".";
    M.decW[i] = add(p + "W", w, M.dec[i]);
    M.decb[i] = add(p + "b", M.dec[i], 0);
    w = M.dec[i];
  }
  M.outW = add("dec.out.W", w, 1);
  M.outb = add("dec.out.b", 1, 0);
  off = (off + 3) & ~(int64_t)3;
  if (off > (int64_t)0x7fffffff) {
    delete m;
    return TPCB_ERR_UNSUPPORTED;
  }
  M.total = (int)off;
  m->t2.n = 0;
  m->t2.cum[0] = 0;
  for (const TensorInfo& t : m->tensors) {
    if (t.cols == 0) continue;
    if (m->t2.n >= tpcb::kMaxT2) {
      delete m;
      return TPCB_ERR_UNSUPPORTED;
    }
    const int i = m->t2.n++;
    m->t2.off[i] = (int)t.offset;
    m->t2.rows[i] = t.rows;
    m->t2.cols[i] = t.cols;
    m->t2.cum[i + 1] = m->t2.cum[i] + t.rows * t.cols;
  }
  M.shared_lo = M.inW;
  M.shared_hi = M.leafW[1];
  M.tail_lo = M.devhW;
  *out = m;
  return TPCB_OK;
}

extern "C" void tpcb_model_destroy(tpcb_model* m) { delete m; }

extern "C" int64_t tpcb_model_param_count(const tpcb_model* m) { return m ? m->dev.total : 0; }

extern "C" int32_t tpcb_model_tensor_count(const tpcb_model* m) {
  return m ? (int32_t)m->tensors.size() : 0;
}

extern "C" int tpcb_model_tensor_info(const tpcb_model* m, int32_t i, char* name, int32_t cap,
                                      int64_t* offset, int32_t* rows, int32_t* cols) {
  if (!m || i < 0 || i >= (int32_t)m->tensors.size()) return TPCB_ERR_VALIDATION;
  const TensorInfo& t = m->tensors[i];
  if (name && cap > 0) {
    strncpy(name, t.name.c_str(), cap - 1);
    name[cap - 1] = 0;
  }
  if (offset) *offset = t.offset;
  if (rows) *rows = t.rows;
  if (cols) *cols = t.cols;
  return TPCB_OK;
}
