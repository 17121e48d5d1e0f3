// C ABI of the training path: single backward (costmodel.backward), the
// optimizer (nn.Adam / nn.Sgd), and the native epoch loop (train/finetune
// inner loops, costmodel.py:697-707 and :755-773).
#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/tpcb200_debug.h"
#include "common.cuh"
#include "dist.cuh"
#include "train.cuh"

using namespace tpcb;

// Captured epoch: every launch of one epoch recorded once and replayed; all
// per-epoch inputs (plan contents, lr, step count) are read from device
// memory, so the same graph serves every epoch of a training run.
struct tpcb_graph {
  // a few instantiated epochs keyed by everything they captured (pointers,
  // step count, loss / optimizer settings): epochs whose plans have different
  // step counts alternate without re-capturing
  struct Entry {
    cudaGraphExec_t exec = nullptr;
    std::vector<uint8_t> key;
    uint64_t used = 0;
  };
  std::vector<Entry> entries;
  uint64_t clock = 0;
  static constexpr size_t kMax = 8;
};

namespace {

SampleSetDev to_dev(const tpcb_samples* s) {
  SampleSetDev d{};
  if (s) {
    d.x = s->x;
    d.ast_row = s->ast_row;
    d.n_leaf = s->n_leaf;
    d.devfeat = s->devfeat;
    d.y = s->y;
  }
  return d;
}

LossDev to_dev(const tpcb_loss* l, bool has_tgt) {
  LossDev d{};
  d.mode = l->mode;
  d.original = l->original_space;
  d.lambda = l->lambda_hybrid;
  d.offset = l->offset;
  d.alpha = l->alpha_cmd;
  d.cmd_order = l->cmd_order;
  d.use_cmd = (l->alpha_cmd > 0.0 && has_tgt) ? 1 : 0;
  d.norm = l->norm;
  return d;
}

TrainWs to_dev(const tpcb_train_ws* w) {
  TrainWs d{};
  d.partial = w->partial;
  d.slot_stride = (size_t)w->slot_stride;
  d.n_slots = w->n_slots;
  d.touched = w->touched;
  d.zall = w->zall;
  d.terms = w->terms;
  d.scalars = w->scalars;
  d.zall_bytes = (size_t)std::max<int64_t>(w->zall_floats, 0) * sizeof(float);
  d.l_cap = w->l_cap;
  // overlapped reduce: the caller's counters, when large enough for this model
  d.stage_flags = reinterpret_cast<unsigned long long*>(w->stage_flags);
  d.n_stage_words = (int)std::min<int64_t>(w->stage_flag_words, 1 << 30);
  if (w->act && w->act_floats >= 32 * wg_total_rows()) {
    d.wg.act = w->act;
    d.wg.r_cap = (int)std::min<int64_t>(w->act_floats / wg_total_rows() / 32 * 32, 1 << 24);
  }
  return d;
}

OptDev to_dev(const tpcb_optim* o) {
  OptDev d{};
  if (o) {
    d.kind = o->kind;
    d.beta1 = o->beta1;
    d.beta2 = o->beta2;
    d.eps = o->eps;
    d.weight_decay = o->weight_decay;
  }
  return d;
}

int check_loss(const tpcb_loss* l) {
  if (!l) return TPCB_ERR_VALIDATION;
  if (l->mode < 0 || l->mode > 2) return TPCB_ERR_VALIDATION;
  if (l->cmd_order < 1) return TPCB_ERR_VALIDATION;
  if (l->cmd_order > kMaxCmdOrder) return TPCB_ERR_UNSUPPORTED;
  return TPCB_OK;
}

// optional per-kernel-class timing of an uncaptured epoch (bench.py roofline)
struct StepProfiler {
  std::vector<cudaEvent_t> ev;  // pairs: (start, end), class = index % 3
  int pos = 0;
  void mark(cudaStream_t s) {
    if (pos >= (int)ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    cudaEventRecord(ev[pos++], s);
  }
};
thread_local StepProfiler* g_prof = nullptr;

struct SideStream {  // per device: the reduce branch of an overlapped step
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int sms = 0;
};
int side_stream(SideStream** out) {
  thread_local SideStream per_dev[16];
  int dev = 0;
  TPCB_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev >= 16) return TPCB_ERR_UNSUPPORTED;
  SideStream& s = per_dev[dev];
  if (!s.side) {
    TPCB_CUDA_CHECK(cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking));
    TPCB_CUDA_CHECK(cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming));
    TPCB_CUDA_CHECK(cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming));
    TPCB_CUDA_CHECK(cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev));
  }
  *out = &s;
  return TPCB_OK;
}

// Single GPU, no CMD, an optimizer, the desk fast-path kernel with one sample
// per CTA, and a workspace that owns stage counters: the reduce + optimizer
// of step k runs on the SMs the training kernel leaves idle, each backward
// stage as soon as every CTA published it (train4.cu stage_flags, optim.cu
// reduce_overlap_kernel).  The reduce blocks spin on counters the training
// CTAs advance, so the overlap is only taken when every training CTA is
// co-resident (occupancy check against this device's SM count, which also
// reflects a MIG slice) and the waits are bounded: a wait that times out
// raises TPCB_ERR_CUDA and the reduce applies nothing from that stage on.
// Returns 1 when the step was enqueued this way, 0 to use the sequential path.
int try_overlapped_step(const tpcb_model* m, float* P, float* PT, float* mb, float* vb,
                        const SampleSetDev& src, const SampleSetDev& tgt, const int32_t* batch,
                        const StepDesc* steps, int step, int grid, const LossDev& loss,
                        const OptDev& opt, const double* lr, const int64_t* t0,
                        const TrainWs& ws, float* grad_out, double* step_loss, double* step_cmd,
                        float* pred_out, int32_t* status, cudaStream_t stream, int* st_out) {
  *st_out = TPCB_OK;
  const Knobs& kn = knobs();
  if (!ws.stage_flags || loss.use_cmd || opt.kind == kOptNone || !t0 || kn.grid_cap > 0) return 0;
  if (ws.wg.act) return 0;  // the tensor-core weight-gradient step runs sequentially
  if (ws.n_stage_words < ovl_stage_words(m->dev.n_layers)) return 0;
  if (!(kn.train_impl == 0 || kn.train_impl == 4) || !v4_fits(m->dev, ws.l_cap)) return 0;
  SideStream* ss = nullptr;
  if (side_stream(&ss)) return 0;
  const int tgrid = std::max(1, std::min(grid, ws.n_slots));
  const int rgrid = ss->sms - tgrid;  // the reduce never blocks the training CTAs' SMs
  if (rgrid < 16) return 0;
  if (train4_blocks_per_sm(m->dev, ws.l_cap) < 1) return 0;
  OvlDev ov{};
  if (overlap_sched(m, &ov) || ws.n_slots > ov.flag_stride) return 0;
  ov.flags = ws.stage_flags;
  ov.poll_ns = kn.poll_ns;
  TrainWs w2 = ws;
  w2.t_tag = t0;
  w2.flag_stride = ov.flag_stride;
  int st = TPCB_OK;
  auto fail = [&](int e) { *st_out = e; return 1; };
  if (step == 0)  // the counters are cumulative within an epoch
    if (cudaMemsetAsync(ov.flags, 0, (size_t)ov.n_stages * ov.flag_stride * 8, stream))
      return fail(TPCB_ERR_CUDA);
  if (g_prof) g_prof->mark(stream);
  if (cudaEventRecord(ss->fork, stream)) return fail(TPCB_ERR_CUDA);
  // the training kernel is enqueued first: where launches are serialised
  // (profilers, CUDA_LAUNCH_BLOCKING) it completes every stage before the
  // reduce starts, which then never waits
  st = launch_train(m->dev, P, PT, src, tgt, batch, steps, step, grid, loss, 1, w2, pred_out,
                    status, stream);
  if (st) return fail(st);
  if (g_prof) g_prof->mark(stream);
  if (cudaStreamWaitEvent(ss->side, ss->fork, 0)) return fail(TPCB_ERR_CUDA);
  st = launch_reduce_overlap(m->dev, w2, ov, steps, step, batch, src, grad_out, P, mb, vb, opt,
                             lr, t0, loss, step_loss, step_cmd, status, std::min(rgrid, ov.n_items),
                             ss->side);
  if (st) return fail(st);
  if (cudaEventRecord(ss->join, ss->side)) return fail(TPCB_ERR_CUDA);
  if (cudaStreamWaitEvent(stream, ss->join, 0)) return fail(TPCB_ERR_CUDA);
  if (g_prof) g_prof->mark(stream);
  if (g_prof) g_prof->mark(stream);
  return 1;
}

// one training step on an already uploaded step table.  With a
// communicator (data parallel): local fwd/bwd → local gradient sum into
// `gbuf` → all-reduce(gradient, step loss) → optimizer from the gradient.
int run_step(const tpcb_model* m, float* P, float* PT, float* mb, float* vb,
             const SampleSetDev& src, const SampleSetDev& tgt, const int32_t* batch,
             const StepDesc* steps, int step, int grid, const LossDev& loss, const OptDev& opt,
             const double* lr, const int64_t* t0, const TrainWs& ws_in, float* grad_out,
             double* step_loss, double* step_cmd, float* pred_out, int32_t* status,
             cudaStream_t stream, tpcb_comm* comm = nullptr, float* gbuf = nullptr) {
  (void)PT;
  int st;
  const bool dp = comm != nullptr;  // (a 1-rank communicator exercises the same path)
  // tensor-core encoder weight gradients: desk fast path, no CMD in the step
  const Knobs& kn = knobs();
  TrainWs ws_wg = ws_in;
  const bool use_wg = ws_in.wg.act && !loss.use_cmd && kn.wgrad_tc &&
                      (kn.train_impl == 0 || kn.train_impl == 4) && kn.grid_cap == 0 &&
                      v4_fits(m->dev, ws_in.l_cap) && wgrad_tc_supported(m->dev) &&
                      (int64_t)ws_in.n_slots * ws_in.l_cap <= ws_in.wg.r_cap;
  if (!use_wg) ws_wg.wg = WgradDev{};
  if (!dp) {
    int ost = TPCB_OK;
    if (try_overlapped_step(m, P, PT, mb, vb, src, tgt, batch, steps, step, grid, loss, opt, lr,
                            t0, ws_wg, grad_out, step_loss, step_cmd, pred_out, status, stream,
                            &ost))
      return ost;
  }
  TrainWs ws = ws_wg;  // sequential step: the training CTAs publish no stage counters
  ws.stage_flags = nullptr;
  if (g_prof) g_prof->mark(stream);
  if (loss.use_cmd) {
    if (dp) {  // every rank fills its own rows; the all-reduce assembles [zs; zt]
      TPCB_CUDA_CHECK(cudaMemsetAsync(ws.zall, 0, ws.zall_bytes, stream));
    }
    st = launch_train(m->dev, P, PT, src, tgt, batch, steps, step, grid, loss, 0, ws, nullptr,
                      status, stream);
    if (st) return st;
    if (dp) {
      st = allreduce_sum(comm, ws.zall, (int64_t)(ws.zall_bytes / sizeof(float)), 0, stream);
      if (st) return st;
    }
  }
  st = launch_train(m->dev, P, PT, src, tgt, batch, steps, step, grid, loss, 1, ws, pred_out,
                    status, stream);
  if (st) return st;
  if (g_prof) g_prof->mark(stream);
  const int wg_splits = use_wg ? wgrad_tc_splits(ws) : 0;
  if (use_wg && (st = launch_wgrad_tc(m->dev, ws, steps, step, batch, src.n_leaf, wg_splits,
                                      stream)))
    return st;
  if (!dp) {
    st = launch_reduce_apply(m->dev, ws, steps, step, loss.use_cmd, 1, grad_out, P, mb, vb, opt,
                             lr, t0, loss, step_loss, step_cmd, stream, wg_splits);
    if (st) return st;
  } else {
    OptDev none{};
    st = launch_reduce_apply(m->dev, ws, steps, step, loss.use_cmd, comm->rank == 0, gbuf,
                             nullptr, nullptr, nullptr, none, nullptr, nullptr, loss, step_loss,
                             step_cmd, stream, wg_splits);
    if (st) return st;
    // gradient: rank-ordered sum (deterministic for a given world size,
    // independent of NCCL's algorithm choice); the step loss is a logged
    // scalar
    if ((st = ordered_allreduce_sum(comm, gbuf, m->dev.total, stream))) return st;
    if (step_loss && (st = allreduce_sum(comm, step_loss + step, 1, 1, stream))) return st;
    if (opt.kind != kOptNone) {
      st = launch_opt_from_grad(m->dev, gbuf, P, mb, vb, opt, lr, t0, step, stream);
      if (st) return st;
    }
  }
  if (g_prof) g_prof->mark(stream);
  if (g_prof) g_prof->mark(stream);
  return st;
}

}  // namespace

extern "C" int tpcb_train_ws_sizes(const tpcb_model* m, int32_t max_rows, int32_t l_cap,
                                   int32_t* n_slots, int64_t* slot_stride, int64_t* zall_floats,
                                   int64_t* terms_doubles, int64_t* stage_flag_words,
                                   int64_t* act_floats) {
  if (!m || max_rows < 1) return TPCB_ERR_VALIDATION;
  if (stage_flag_words) *stage_flag_words = ovl_stage_words(m->dev.n_layers);
  if (act_floats)
    *act_floats = wgrad_tc_supported(m->dev)
                      ? (int64_t)wg_total_rows() *
                            (((int64_t)std::min<int32_t>(max_rows, 1024) *
                                  std::max<int32_t>(l_cap, 1) + 31) / 32 * 32)
                      : 0;
  const int slots = std::min<int32_t>(max_rows, 1024);
  if (n_slots) *n_slots = slots;
  // 64-float (256 B) aligned slots
  if (slot_stride) *slot_stride = ((int64_t)m->dev.total + 63) / 64 * 64;
  if (zall_floats) *zall_floats = (int64_t)max_rows * m->dev.d_e;
  if (terms_doubles) *terms_doubles = (int64_t)max_rows * 2;
  TrainPlan tp = make_train_plan(m->dev, l_cap);
  if ((size_t)tp.total * sizeof(float) > 220 * 1024) return TPCB_ERR_UNSUPPORTED;
  return TPCB_OK;
}

extern "C" int tpcb_transpose_params(const tpcb_model* m, const float* d_params, float* d_params_t,
                                     void* stream) {
  if (!m || !d_params || !d_params_t) return TPCB_ERR_VALIDATION;
  return launch_transpose(m, d_params, d_params_t, (cudaStream_t)stream);
}

extern "C" int tpcb_loss_backward(const tpcb_model* m, const float* d_params,
                                  const float* d_params_t, const tpcb_samples* src,
                                  const tpcb_samples* tgt, const int32_t* d_batch, int32_t n_src,
                                  int32_t n_tgt, const tpcb_loss* loss, const tpcb_train_ws* ws,
                                  void* d_step_scratch_, float* d_grad, float* d_pred,
                                  int32_t* d_status, void* stream_) {
  StepDesc* d_step_scratch = static_cast<StepDesc*>(d_step_scratch_);
  if (!m || !d_params || !d_params_t || !src || !ws || !d_batch || !d_step_scratch)
    return TPCB_ERR_VALIDATION;
  if (n_src < 1) return TPCB_ERR_EMPTY_BATCH;
  int st = check_loss(loss);
  if (st) return st;
  cudaStream_t stream = (cudaStream_t)stream_;
  const LossDev ld = to_dev(loss, tgt != nullptr && n_tgt > 0);
  if (ld.use_cmd && !tgt) return TPCB_ERR_VALIDATION;
  const int n_all = n_src + (ld.use_cmd ? n_tgt : 0);
  const int nt = ld.use_cmd ? n_tgt : 0;
  StepDesc h{0, n_src, nt, n_src, 0, n_src, 0, nt};
  TPCB_CUDA_CHECK(
      cudaMemcpyAsync(d_step_scratch, &h, sizeof(StepDesc), cudaMemcpyHostToDevice, stream));
  OptDev none{};
  TrainWs w = to_dev(ws);
  return run_step(m, const_cast<float*>(d_params), const_cast<float*>(d_params_t), nullptr, nullptr,
                  to_dev(src), to_dev(tgt), d_batch, d_step_scratch, 0, n_all, ld, none, nullptr,
                  nullptr, w, d_grad, ws->scalars + 1, nullptr, d_pred, d_status, stream);
}

extern "C" int tpcb_optimizer_step(const tpcb_model* m, int64_t n, float* d_params,
                                   float* d_params_t, const float* d_grad, float* d_m, float* d_v,
                                   const tpcb_optim* opt, double lr, int64_t t, void* stream_) {
  if (!d_params || !d_grad || !opt || t < 1) return TPCB_ERR_VALIDATION;
  if (opt->kind == kOptAdam && (!d_m || !d_v)) return TPCB_ERR_VALIDATION;
  if (d_params_t && !m) return TPCB_ERR_VALIDATION;
  if (m) n = m->dev.total;
  if (n < 0 || n > 0x7fffffff) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  int st = launch_optimizer((int)n, d_grad, d_params, d_m, d_v, to_dev(opt), lr, (double)t,
                            stream);
  if (st) return st;
  if (d_params_t) st = launch_transpose(m, d_params, d_params_t, stream);
  return st;
}

namespace tpcb {
int set_train_trace(long long* d_trace);
}

/* debug: per-op timestamps of CTA 0 of the training kernel (NULL disables) */
namespace tpcb {
int set_train4_trace(long long* d_trace);
int set_forward_tc_trace(long long* d_trace);
int set_forward_trace(long long* d_trace);
int set_forward_f32_trace(long long* d_trace);
}
extern "C" int tpcb_debug_train_trace(long long* d_trace) {
  int st = tpcb::set_train_trace(d_trace);
  if (!st) st = tpcb::set_forward_tc_trace(d_trace);
  if (!st) st = tpcb::set_forward_trace(d_trace);
  if (!st) st = tpcb::set_forward_f32_trace(d_trace);
  return st ? st : tpcb::set_train4_trace(d_trace);
}

extern "C" int tpcb_graph_create(tpcb_graph** out) {
  if (!out) return TPCB_ERR_VALIDATION;
  *out = new tpcb_graph();
  return TPCB_OK;
}

extern "C" void tpcb_graph_destroy(tpcb_graph* g) {
  if (!g) return;
  for (auto& e : g->entries)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  delete g;
}

namespace {

template <typename T>
void key_add(std::vector<uint8_t>& k, const T& v) {
  const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
  k.insert(k.end(), p, p + sizeof(T));
}

}  // namespace

extern "C" int tpcb_train_epoch(const tpcb_model* m, float* d_params, float* d_params_t,
                                float* d_m, float* d_v, const tpcb_samples* src,
                                const tpcb_samples* tgt, const tpcb_plan* plan,
                                const tpcb_loss* loss, const tpcb_optim* opt, const double* d_lr,
                                const int64_t* d_t0, const tpcb_train_ws* ws,
                                double* d_step_loss, double* d_step_cmd, int32_t* d_status,
                                tpcb_graph* graph, double* prof_ms, tpcb_comm* comm,
                                float* d_grad, void* stream_) {
  if (!m || !d_params || !src || !plan || !opt || !ws) return TPCB_ERR_VALIDATION;
  if (comm && !d_grad) return TPCB_ERR_VALIDATION;
  int st = check_loss(loss);
  if (st) return st;
  if (plan->n_steps < 0) return TPCB_ERR_VALIDATION;
  if (comm && (st = ensure_gather(comm, m->dev.total))) return st;  // (outside capture)
  cudaStream_t stream = (cudaStream_t)stream_;
  const LossDev ld = to_dev(loss, tgt != nullptr);
  const OptDev od = to_dev(opt);
  const TrainWs w = to_dev(ws);
  const SampleSetDev s = to_dev(src), t = to_dev(tgt);
  const StepDesc* steps = reinterpret_cast<const StepDesc*>(plan->d_steps);
  auto enqueue = [&]() -> int {
    for (int k = 0; k < plan->n_steps; ++k) {
      int r = run_step(m, d_params, d_params_t, d_m, d_v, s, t, plan->d_batch, steps, k,
                       ws->n_slots, ld, od, d_lr, d_t0, w, nullptr, d_step_loss, d_step_cmd,
                       nullptr, d_status, stream, comm, d_grad);
      if (r) return r;
    }
    return TPCB_OK;
  };
  if (prof_ms) {  // uncaptured, timed per kernel class
    StepProfiler prof;
    g_prof = &prof;
    st = enqueue();
    g_prof = nullptr;
    if (st) return st;
    TPCB_CUDA_CHECK(cudaStreamSynchronize(stream));
    prof_ms[0] = prof_ms[1] = prof_ms[2] = 0.0;
    for (int i = 0; i + 3 < prof.pos; i += 4) {
      for (int c = 0; c < 3; ++c) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, prof.ev[i + c], prof.ev[i + c + 1]);
        prof_ms[c] += ms;
      }
    }
    for (cudaEvent_t e : prof.ev) cudaEventDestroy(e);
    return TPCB_OK;
  }
  if (!graph || plan->n_steps == 0) return enqueue();
  std::vector<uint8_t> key;
  key_add(key, m);
  key_add(key, d_params);
  key_add(key, d_params_t);
  key_add(key, d_m);
  key_add(key, d_v);
  key_add(key, *src);
  if (tgt) key_add(key, *tgt);
  key_add(key, *plan);
  key_add(key, *loss);
  key_add(key, *opt);
  key_add(key, d_lr);
  key_add(key, d_t0);
  key_add(key, *ws);
  key_add(key, d_step_loss);
  key_add(key, d_step_cmd);
  key_add(key, d_status);
  key_add(key, comm);
  key_add(key, d_grad);
  tpcb_graph::Entry* hit = nullptr;
  for (auto& e : graph->entries)
    if (e.key == key) hit = &e;
  if (!hit) {
    if (graph->entries.size() >= tpcb_graph::kMax) {  // evict the least recently used
      auto lru = std::min_element(graph->entries.begin(), graph->entries.end(),
                                  [](const tpcb_graph::Entry& a, const tpcb_graph::Entry& b) {
                                    return a.used < b.used;
                                  });
      cudaGraphExecDestroy(lru->exec);
      graph->entries.erase(lru);
    }
    st = prepare_train_kernels(m->dev, ws->l_cap);  // attributes are set outside capture
    if (st) return st;
    {  // the overlapped reduce's schedule / side stream are allocated outside capture too
      OvlDev ov{};
      SideStream* ss = nullptr;
      if (ws->stage_flags && !comm) {
        st = overlap_sched(m, &ov);
        if (!st) st = side_stream(&ss);
        if (st) return st;
      }
    }
    graph->entries.emplace_back();
    hit = &graph->entries.back();
    TPCB_CUDA_CHECK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    st = enqueue();
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(stream, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      graph->entries.pop_back();
      return st;
    }
    if (e != cudaSuccess) {
      set_last_error("cudaStreamEndCapture", e);
      graph->entries.pop_back();
      return TPCB_ERR_CUDA;
    }
    e = cudaGraphInstantiate(&hit->exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      set_last_error("cudaGraphInstantiate", e);
      graph->entries.pop_back();
      return TPCB_ERR_CUDA;
    }
    hit->key = key;
  }
  hit->used = ++graph->clock;
  TPCB_CUDA_CHECK(cudaGraphLaunch(hit->exec, stream));
  return TPCB_OK;
}
