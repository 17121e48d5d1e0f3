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
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "train.cuh"

namespace tpcb {

namespace {

// read-once gradient slots: evict-first
__device__ __forceinline__ float4 ldg4_last_use(const float4* p) {
  float4 v;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// region of parameter p: 0 = touched by every batch, L = leaf_embed.L
struct LeafLo {
  const int* lo;
};
__device__ __forceinline__ LeafLo s_leaf_of(const Model& M) { return LeafLo{M.leafW}; }
__device__ __forceinline__ int region_bit(const Model& M, int p, LeafLo t) {
  if (p < t.lo[1] || p >= M.tail_lo) return 0;
  int L = 1;
  while (L < M.n_leaf_max && p >= t.lo[L + 1]) ++L;
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
    double* __restrict__ step_loss, double* __restrict__ step_cmd, int skip_wgrad) {
  // A block owns 64 float4 columns (4 parameters each: tensors start on
  // 16-byte boundaries, so a column never straddles two tensors and has one
  // region bit).  Its four 64-thread quarters each sum a contiguous quarter of
  // the slots (8 loads in flight), the quarters are combined in fixed order
  // (bitwise reproducible, no atomics), then every thread applies the
  // optimizer to one parameter (coalesced).  All global loads of a thread —
  // slots, p, m, v, step scalars — are issued before the block's single
  // barrier, so a block costs about one memory latency.
  __shared__ float4 s_part[4][64];
  __shared__ float s_opt[3];
  const StepDesc sd = steps[step];
  const int n_src = sd.n_src, n_tgt = sd.n_tgt;
  const int n_all = n_src + (use_cmd ? n_tgt : 0);
  const int G = min(n_all, n_slots);
  const int col = threadIdx.x & 63, quarter = threadIdx.x >> 6;
  const int n4 = M.total >> 2;
  const size_t st4 = stride >> 2;

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

  // slot masks: the fast path sums every slot unpredicated when all of them
  // touched the column's region (the shared region, always; a leaf region when
  // the batch is one bucket), and skips regions no slot touched
  __shared__ uint32_t s_touch[1024];
  __shared__ uint32_t s_and, s_or;
  if (threadIdx.x < 32) {
    uint32_t a = ~0u, o = 0u;
    for (int c = threadIdx.x; c < G; c += 32) {
      const uint32_t t = touched[c];
      s_touch[c] = t;
      a &= t;
      o |= t;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      a &= __shfl_xor_sync(0xffffffffu, a, d);
      o |= __shfl_xor_sync(0xffffffffu, o, d);
    }
    if (threadIdx.x == 0) {
      s_and = G > 0 ? a : 0u;
      s_or = o;
    }
  }
  for (int base = blockIdx.x * 64; base < n4; base += gridDim.x * 64) {
    // optimizer operands of this thread's parameter, in flight with the slots
    const int pp = base * 4 + threadIdx.x;
    const bool pv = pp < M.total && opt.kind != kOptNone;
    float w = 0.f, m = 0.f, v = 0.f;
    if (pv) {
      w = P[pp];
      if (opt.kind == kOptAdam) {
        m = mbuf[pp];
        v = vbuf[pp];
      }
    }
    const int q = base + col;
    const bool qv = q < n4;
    const int p = q << 2;
    // encoder weight matrices with the tensor-core weight gradients on: the
    // gradient is the split-K partials in slots 0..skip_wgrad-1 (wgrad.cu),
    // added in slot order by quarter 0; the other quarters add zeros
    const bool wgr = qv && skip_wgrad && in_wgrad_region(M, p);
    const bool mine = qv && !wgr;
    const uint32_t want = mine ? 1u << region_bit(M, p, s_leaf_of(M)) : 0u;
    const int per_q = (G + 3) >> 2;
    const int c_lo = min(G, quarter * per_q), c_hi = min(G, c_lo + per_q);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();  // s_touch / s_and / s_or (first iteration), s_part reuse (later ones)
    if (wgr && quarter == 0)
      for (int c = 0; c < skip_wgrad; ++c) {
        const float4 x = ldg4_last_use(reinterpret_cast<const float4*>(partial + p) + (size_t)c * st4);
        g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
      }
    if (mine && (s_or & want)) {
      const float4* src = reinterpret_cast<const float4*>(partial + p) + (size_t)c_lo * st4;
      const int n = c_hi - c_lo;
      if (s_and & want) {  // every slot touched it: unpredicated, 8 loads in flight
        int c = 0;
        for (; c + 8 <= n; c += 8) {
          float4 x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = ldg4_last_use(src + (size_t)(c + u) * st4);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            g.x += x[u].x; g.y += x[u].y; g.z += x[u].z; g.w += x[u].w;
          }
        }
        for (; c < n; ++c) {
          const float4 x = ldg4_last_use(src + (size_t)c * st4);
          g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
        }
      } else {
        for (int c = 0; c < n; ++c) {
          if (s_touch[c_lo + c] & want) {
            const float4 x = ldg4_last_use(src + (size_t)c * st4);
            g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
          }
        }
      }
    }
    s_part[quarter][col] = g;
    if (threadIdx.x == 0) {  // step scalars: one thread (fp64 pow is hundreds of instructions)
      float lr = 0.f, bc1 = 1.f, bc2 = 1.f;
      if (opt.kind != kOptNone) {
        lr = (float)__ldg(lr_p);
        if (opt.kind == kOptAdam) {
          const double t = (double)(__ldg(t_p) + step + 1);
          bc1 = (float)(1.0 - pow(opt.beta1, t));
          bc2 = (float)(1.0 - pow(opt.beta2, t));
        }
      }
      s_opt[0] = lr;
      s_opt[1] = bc1;
      s_opt[2] = bc2;
    }
    __syncthreads();
    const float lr = s_opt[0], bc1 = s_opt[1], bc2 = s_opt[2];
    if (pp < M.total) {
      const int cc = threadIdx.x >> 2, comp = threadIdx.x & 3;
      const float* part = reinterpret_cast<const float*>(s_part);
      float gs = part[(0 * 64 + cc) * 4 + comp];
      gs += part[(1 * 64 + cc) * 4 + comp];
      gs += part[(2 * 64 + cc) * 4 + comp];
      gs += part[(3 * 64 + cc) * 4 + comp];
      apply1(pp, gs, w, m, v, grad_out, P, mbuf, vbuf, opt, lr, bc1, bc2);
    }
    __syncthreads();
  }
}

// ---- overlapped reduce + optimizer ----------------------------------------
// Runs concurrently with the training kernel on the SMs it leaves idle.  The
// training CTAs publish, per backward stage, that their gradient slot holds
// the stage's parameters (train4.cu, stage_flags); this kernel walks the
// 256-parameter items in stage order, waits for a stage only when it reaches
// its first item, and reduces + applies the optimizer exactly as
// reduce_apply_kernel does (same slot order, same arithmetic: bitwise equal
// results).  Untouched leaf_embed tensors (stage -1: gradient 0, Adam still
// decays m / v and moves p) run while the forward is still in flight.
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// block-wide wait until the training CTAs of this step (and of every earlier
// step of the epoch) counted themselves into stage q's word (train4.cu): the
// word must reach `target` = samples of steps first..this.  A poll is one L2
// request by one lane.
__device__ bool wait_stage(const OvlDev& ov, int q, unsigned long long target, int32_t* status) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const unsigned long long* f = ov.flags + (size_t)q * ov.flag_stride;
    bool ok = false;
    for (long it = 0; it < (1l << 21); ++it) {  // bounded (~1 s): a bug must not hang the GPU
      if (ld_acquire_gpu(f) >= target) {
        ok = true;
        break;
      }
      __nanosleep(ov.poll_ns);
    }
    s_ok = ok;
    if (!ok) raise_status(status, TPCB_ERR_CUDA);
  }
  __syncthreads();
  return s_ok;
}

__global__ void __launch_bounds__(256) reduce_overlap_kernel(
    const __grid_constant__ Model M, const float* __restrict__ partial, size_t stride,
    const uint32_t* __restrict__ touched, const StepDesc* __restrict__ steps, int step,
    const int32_t* __restrict__ batch_all, const int32_t* __restrict__ n_leaf, OvlDev ov,
    const int64_t* __restrict__ t_p, float* __restrict__ grad_out, float* __restrict__ P,
    float* __restrict__ mbuf, float* __restrict__ vbuf, OptDev opt,
    const double* __restrict__ lr_p, const double* __restrict__ terms, LossDev loss,
    double* __restrict__ step_loss, double* __restrict__ step_cmd, int32_t* status) {
  __shared__ float4 s_part[4][64];
  __shared__ float s_opt[3];
  __shared__ uint32_t s_touch[1024];
  __shared__ uint32_t s_and, s_or;
  __shared__ int s_L;
  const StepDesc sd = steps[step];
  const int n_src = sd.n_src;
  const int G = n_src;  // one CTA (gradient slot) per sample
  const int col = threadIdx.x & 63, quarter = threadIdx.x >> 6;
  const int n4 = M.total >> 2;
  const size_t st4 = stride >> 2;
  // cumulative CTA count the stage words reach at the end of this step
  const unsigned long long target = (unsigned long long)(sd.off - steps[0].off + n_src);
  const int final_stage = ov.n_stages - 1;
  if (threadIdx.x == 0) {
    const int32_t* batch = batch_all + sd.off;
    int L = n_leaf[batch[0]];
    for (int i = 1; i < n_src; ++i)
      if (n_leaf[batch[i]] != L) L = 0;  // mixed leaf counts: everything at the final stage
    s_L = (L >= 1 && L <= ov.n_leaf_max) ? L : 0;
    float lr = 0.f, bc1 = 1.f, bc2 = 1.f;
    if (opt.kind != kOptNone) {
      lr = (float)__ldg(lr_p);
      if (opt.kind == kOptAdam) {
        const double t = (double)(__ldg(t_p) + step + 1);
        bc1 = (float)(1.0 - pow(opt.beta1, t));
        bc2 = (float)(1.0 - pow(opt.beta2, t));
      }
    }
    s_opt[0] = lr;
    s_opt[1] = bc1;
    s_opt[2] = bc2;
  }
  __syncthreads();
  const int L = s_L;
  const bool mixed = L == 0;
  const int32_t* order = ov.order + (size_t)L * ov.n_items;
  const int8_t* stage_of = ov.stage + (size_t)L * ov.n_items;
  const float lr = s_opt[0], bc1 = s_opt[1], bc2 = s_opt[2];
  int ready = -1;  // highest stage known complete on every CTA
  for (int k = blockIdx.x; k < ov.n_items; k += gridDim.x) {
    const int item = order[k];
    const int stg = stage_of[item];
    if (stg > ready) {
      // a timed-out wait (status raised) must not apply partially written
      // gradients: this block stops applying here
      if (!wait_stage(ov, stg, target, status)) return;
      ready = stg;
      if (mixed && threadIdx.x < 32) {  // slot masks (written before the final stage)
        uint32_t a = ~0u, o = 0u;
        for (int c = threadIdx.x; c < G; c += 32) {
          const uint32_t t = __ldcg(touched + c);
          s_touch[c] = t;
          a &= t;
          o |= t;
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
          a &= __shfl_xor_sync(0xffffffffu, a, d);
          o |= __shfl_xor_sync(0xffffffffu, o, d);
        }
        if (threadIdx.x == 0) {
          s_and = G > 0 ? a : 0u;
          s_or = o;
        }
      }
      __syncthreads();
    }
    const int base = item * 64;
    const int pp = base * 4 + threadIdx.x;
    const bool pv = pp < M.total && opt.kind != kOptNone;
    float w = 0.f, m = 0.f, v = 0.f;
    if (pv) {
      w = P[pp];
      if (opt.kind == kOptAdam) {
        m = mbuf[pp];
        v = vbuf[pp];
      }
    }
    const int q = base + col;
    const bool qv = q < n4;
    const int p = q << 2;
    const int per_q = (G + 3) >> 2;
    const int c_lo = min(G, quarter * per_q), c_hi = min(G, c_lo + per_q);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    bool all_slots = false, some = false;
    uint32_t want = 0;
    if (!mixed) {  // single bucket: every slot touched the shared region and leaf_embed.L only
      if (qv) {
        const int rb = region_bit(M, p, s_leaf_of(M));
        all_slots = some = (rb == 0 || rb == L);
      }
    } else if (qv) {
      want = 1u << region_bit(M, p, s_leaf_of(M));
      all_slots = (s_and & want) != 0;
      some = (s_or & want) != 0;
    }
    if (qv && some) {
      const float4* src = reinterpret_cast<const float4*>(partial + p) + (size_t)c_lo * st4;
      const int n = c_hi - c_lo;
      if (all_slots) {
        int c = 0;
        for (; c + 8 <= n; c += 8) {
          float4 x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = __ldcg(src + (size_t)(c + u) * st4);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            g.x += x[u].x; g.y += x[u].y; g.z += x[u].z; g.w += x[u].w;
          }
        }
        for (; c < n; ++c) {
          const float4 x = __ldcg(src + (size_t)c * st4);
          g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
        }
      } else {
        for (int c = 0; c < n; ++c) {
          if (s_touch[c_lo + c] & want) {
            const float4 x = __ldcg(src + (size_t)c * st4);
            g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
          }
        }
      }
    }
    s_part[quarter][col] = g;
    __syncthreads();
    if (pp < M.total) {
      const int cc = threadIdx.x >> 2, comp = threadIdx.x & 3;
      const float* part = reinterpret_cast<const float*>(s_part);
      float gs = part[(0 * 64 + cc) * 4 + comp];
      gs += part[(1 * 64 + cc) * 4 + comp];
      gs += part[(2 * 64 + cc) * 4 + comp];
      gs += part[(3 * 64 + cc) * 4 + comp];
      apply1(pp, gs, w, m, v, grad_out, P, mbuf, vbuf, opt, lr, bc1, bc2);
    }
    __syncthreads();
  }
  // loss value of the step (fixed order), costmodel.py:539-550; terms are
  // written before stage 0
  if (blockIdx.x == 0) {
    if (ready < 0 && !wait_stage(ov, 0, target, status)) return;
    if (threadIdx.x < 32) {
      double sq = 0.0, rel = 0.0;
      for (int i = threadIdx.x; i < n_src; i += 32) {
        sq += __ldcg(terms + 2 * i);
        rel += __ldcg(terms + 2 * i + 1);
      }
      sq = warp_sum_d(sq);
      rel = warp_sum_d(rel);
      if (threadIdx.x == 0 && step_loss) {
        const double n = (double)sd.n_norm;
        const double val = loss.mode == kLossMse ? sq / n
                           : loss.mode == kLossMape ? rel / n
                                                    : sq / n + loss.lambda * (rel / n);
        step_loss[step] = val;
        if (step_cmd) step_cmd[step] = 0.0;
      }
    }
  }
  (void)final_stage;
}

// one parameter of Adam / SGD (nn.py:136-167), fp32, oracle operation order
struct OptScalars {
  float lr, bc1, bc2, b1, b2, eps, wd, omb1, omb2;
};
__device__ __forceinline__ void opt1(const OptDev& opt, const OptScalars& k, float g, float& w,
                                     float& m, float& v) {
  if (k.wd != 0.f) g = g + k.wd * w;
  if (opt.kind == kOptSgd) {
    w = w - k.lr * g;
    return;
  }
  m = __fadd_rn(__fmul_rn(m, k.b1), __fmul_rn(k.omb1, g));
  v = __fadd_rn(__fmul_rn(v, k.b2), __fmul_rn(__fmul_rn(k.omb2, g), g));
  w = w - __fdiv_rn(__fmul_rn(k.lr, __fdiv_rn(m, k.bc1)),
                    __fadd_rn(sqrtf(__fdiv_rn(v, k.bc2)), k.eps));
}

__device__ __forceinline__ OptScalars opt_scalars(const OptDev& opt, double lr, double t) {
  OptScalars k;
  k.lr = (float)lr;
  k.bc1 = (float)(1.0 - pow(opt.beta1, t));
  k.bc2 = (float)(1.0 - pow(opt.beta2, t));
  k.b1 = (float)opt.beta1;
  k.b2 = (float)opt.beta2;
  k.eps = (float)opt.eps;
  k.wd = (float)opt.weight_decay;
  k.omb1 = (float)(1.0 - opt.beta1);
  k.omb2 = (float)(1.0 - opt.beta2);
  return k;
}

// Optimizer over a gradient vector, HBM-bound (7 x 4 B per parameter):
// float4 loads/stores for the 16-byte-aligned body (VEC), scalar tail.
template <bool VEC>
__device__ __forceinline__ void opt_body(int n, const float* __restrict__ grad,
                                         float* __restrict__ P, float* __restrict__ mbuf,
                                         float* __restrict__ vbuf, const OptDev& opt,
                                         const OptScalars& k) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
  const bool adam = opt.kind == kOptAdam;
  int done = 0;
  if (VEC) {
    const int n4 = n >> 2;
    for (int q = tid; q < n4; q += nthr) {
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(grad) + q);
      float4 w4 = reinterpret_cast<float4*>(P)[q];
      float4 m4 = make_float4(0.f, 0.f, 0.f, 0.f), v4 = m4;
      if (adam) {
        m4 = reinterpret_cast<float4*>(mbuf)[q];
        v4 = reinterpret_cast<float4*>(vbuf)[q];
      }
      opt1(opt, k, g4.x, w4.x, m4.x, v4.x);
      opt1(opt, k, g4.y, w4.y, m4.y, v4.y);
      opt1(opt, k, g4.z, w4.z, m4.z, v4.z);
      opt1(opt, k, g4.w, w4.w, m4.w, v4.w);
      reinterpret_cast<float4*>(P)[q] = w4;
      if (adam) {
        reinterpret_cast<float4*>(mbuf)[q] = m4;
        reinterpret_cast<float4*>(vbuf)[q] = v4;
      }
    }
    done = n4 << 2;
  }
  for (int p = done + tid; p < n; p += nthr) {
    float w = P[p], m = 0.f, v = 0.f;
    if (adam) {
      m = mbuf[p];
      v = vbuf[p];
    }
    opt1(opt, k, grad[p], w, m, v);
    P[p] = w;
    if (adam) {
      mbuf[p] = m;
      vbuf[p] = v;
    }
  }
}

// standalone optimizer over a given gradient vector (nn.Adam.step drop-in)
template <bool VEC>
__global__ void optimizer_kernel(int n, const float* __restrict__ grad, float* __restrict__ P,
                                 float* __restrict__ mbuf, float* __restrict__ vbuf, OptDev opt,
                                 double lr_d, double t_d) {
  opt_body<VEC>(n, grad, P, mbuf, vbuf, opt, opt_scalars(opt, lr_d, t_d));
}

// Adam / SGD from a (data-parallel all-reduced) gradient vector; lr and the
// step count before the epoch in device memory (graph replay across epochs)
template <bool VEC>
__global__ void opt_from_grad_kernel(int n, const float* __restrict__ grad, float* __restrict__ P,
                                     float* __restrict__ mbuf, float* __restrict__ vbuf,
                                     OptDev opt, const double* __restrict__ lr_p,
                                     const int64_t* __restrict__ t_p, int step) {
  opt_body<VEC>(n, grad, P, mbuf, vbuf, opt,
                opt_scalars(opt, lr_p[0], (double)(t_p[0] + step + 1)));
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
                        cudaStream_t stream, int skip_wgrad) {
  const int grid = min(ceil_div(M.total / 4, 64), kNumSMs * 16);
  reduce_apply_kernel<<<grid, 256, 0, stream>>>(M, ws.partial, ws.slot_stride, ws.touched, steps,
                                                step, ws.n_slots, use_cmd, add_cmd, grad_out, P, m,
                                                v, opt, lr, t, ws.terms, ws.scalars, loss,
                                                step_loss, step_cmd, skip_wgrad);
  TPCB_LAUNCH_CHECK("reduce_apply");
  return TPCB_OK;
}

int launch_opt_from_grad(const Model& M, const float* grad, float* P, float* m, float* v,
                         const OptDev& opt, const double* lr, const int64_t* t, int step,
                         cudaStream_t stream) {
  const bool vec = ((reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(P) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  const int grid = min(ceil_div(M.total, vec ? 1024 : 256), kNumSMs * 8);
  if (vec)
    opt_from_grad_kernel<true><<<grid, 256, 0, stream>>>(M.total, grad, P, m, v, opt, lr, t, step);
  else
    opt_from_grad_kernel<false><<<grid, 256, 0, stream>>>(M.total, grad, P, m, v, opt, lr, t, step);
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
  const bool vec = ((reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(P) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  const int grid = min(ceil_div(n, vec ? 1024 : 256), kNumSMs * 8);
  if (vec)
    optimizer_kernel<true><<<grid, 256, 0, stream>>>(n, grad, P, m, v, opt, lr, t);
  else
    optimizer_kernel<false><<<grid, 256, 0, stream>>>(n, grad, P, m, v, opt, lr, t);
  TPCB_LAUNCH_CHECK("optimizer");
  return TPCB_OK;
}


// ---- overlapped reduce: host schedule + launch -----------------------------
namespace {
struct OvlCache {
  int device;
  Model key;
  OvlDev dev;
};
std::vector<OvlCache>& ovl_cache() {
  static std::vector<OvlCache> c;
  return c;
}
std::mutex& ovl_mu() {
  static std::mutex mu;
  return mu;
}
}  // namespace

int overlap_sched(const tpcb_model* m, OvlDev* out) {
  const Model& M = m->dev;
  int dev = 0;
  TPCB_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(ovl_mu());
  for (auto& e : ovl_cache())
    if (e.device == dev && memcmp(&e.key, &M, sizeof(Model)) == 0) {
      *out = e.dev;
      return TPCB_OK;
    }
  const int n4 = M.total >> 2;
  const int n_items = (n4 + 63) / 64;
  const int nl = M.n_leaf_max;
  const int n_stages = 2 + 2 * M.n_layers;
  const int final_stage = n_stages - 1;
  // stage of every parameter for batch leaf count L (tensor names, costmodel.py:116-150)
  std::vector<int8_t> pstage_base(M.total, 0);
  std::vector<int> leaf_of(M.total, 0);
  for (const TensorInfo& t : m->tensors) {
    const int64_t size = (int64_t)t.rows * (t.cols ? t.cols : 1);
    int st = 0, leaf = 0;
    if (t.name.rfind("input.", 0) == 0) {
      st = final_stage;
    } else if (t.name.rfind("enc", 0) == 0) {
      const int li = atoi(t.name.c_str() + 3);
      const bool attn = t.name.find(".attn.") != std::string::npos ||
                        t.name.find(".ln1.") != std::string::npos;
      st = (attn ? 2 : 1) + 2 * (M.n_layers - 1 - li);
    } else if (t.name.rfind("leaf_embed.", 0) == 0) {
      leaf = atoi(t.name.c_str() + 11);
    }
    for (int64_t i = 0; i < size; ++i) {
      pstage_base[t.offset + i] = (int8_t)st;
      leaf_of[t.offset + i] = leaf;
    }
  }
  std::vector<int32_t> order((size_t)(nl + 1) * n_items);
  std::vector<int8_t> stage((size_t)(nl + 1) * n_items);
  for (int L = 0; L <= nl; ++L) {
    for (int it = 0; it < n_items; ++it) {
      int st = -1;
      const int p0 = it * 256, p1 = std::min<int>(M.total, p0 + 256);
      for (int p = p0; p < p1; ++p) {
        int sp = pstage_base[p];
        if (leaf_of[p]) sp = (L == 0) ? final_stage : (leaf_of[p] == L ? 0 : -1);
        if (L == 0) sp = final_stage;
        st = std::max(st, sp);
      }
      stage[(size_t)L * n_items + it] = (int8_t)st;
    }
    int32_t* o = order.data() + (size_t)L * n_items;
    for (int it = 0; it < n_items; ++it) o[it] = it;
    const int8_t* sg = stage.data() + (size_t)L * n_items;
    std::stable_sort(o, o + n_items, [&](int a, int b) { return sg[a] < sg[b]; });
  }
  OvlDev d{};
  d.n_items = n_items;
  d.n_stages = n_stages;
  d.flag_stride = kOvlFlagStride;
  d.n_leaf_max = nl;
  int32_t* d_order = nullptr;
  int8_t* d_stage = nullptr;
  TPCB_CUDA_CHECK(cudaMalloc(&d_order, order.size() * sizeof(int32_t)));
  TPCB_CUDA_CHECK(cudaMalloc(&d_stage, stage.size()));
  TPCB_CUDA_CHECK(cudaMemcpy(d_order, order.data(), order.size() * 4, cudaMemcpyHostToDevice));
  TPCB_CUDA_CHECK(cudaMemcpy(d_stage, stage.data(), stage.size(), cudaMemcpyHostToDevice));
  d.order = d_order;
  d.stage = d_stage;
  d.flags = nullptr;  // the stage counters belong to each training workspace
  ovl_cache().push_back(OvlCache{dev, M, d});
  *out = d;
  return TPCB_OK;
}

int launch_reduce_overlap(const Model& M, const TrainWs& ws, const OvlDev& ov,
                          const StepDesc* steps, int step, const int32_t* batch,
                          const SampleSetDev& src, float* grad_out, float* P, float* m, float* v,
                          const OptDev& opt, const double* lr, const int64_t* t,
                          const LossDev& loss, double* step_loss, double* step_cmd,
                          int32_t* status, int grid, cudaStream_t stream) {
  reduce_overlap_kernel<<<grid, 256, 0, stream>>>(M, ws.partial, ws.slot_stride, ws.touched,
                                                  steps, step, batch, src.n_leaf, ov, t,
                                                  grad_out, P, m, v, opt, lr, ws.terms, loss,
                                                  step_loss, step_cmd, status);
  TPCB_LAUNCH_CHECK("reduce_overlap");
  return TPCB_OK;
}

}  // namespace tpcb

// ---- float64 optimizer step (the drop-in nn.Adam / nn.Sgd, nn.py:136-167) ----
// The reference updates float64 numpy arrays in place; this kernel applies
// the same sequence of IEEE float64 operations (no contraction into FMAs:
// every product and sum rounded separately, exactly as numpy evaluates
// m *= b1; m += (1-b1)*g; v *= b2; v += (1-b2)*g*g;
// p -= lr*(m/bc1)/(sqrt(v/bc2)+eps)), so a step is bit-identical to the
// reference's.  bc1 / bc2 come from the host (Python's 1 - beta**t).
namespace tpcb {
namespace {
__global__ void optimizer_f64_kernel(int64_t n, double* __restrict__ P, const double* __restrict__ G,
                                     double* __restrict__ M, double* __restrict__ V, int kind,
                                     double b1, double one_b1, double b2, double one_b2,
                                     double eps, double wd, double lr, double bc1, double bc2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p = P[i], g = G[i];
    if (wd != 0.0) g = __dadd_rn(g, __dmul_rn(wd, p));
    if (kind == kOptSgd) {
      P[i] = __dsub_rn(p, __dmul_rn(lr, g));
      continue;
    }
    double m = __dadd_rn(__dmul_rn(M[i], b1), __dmul_rn(one_b1, g));
    double v = __dadd_rn(__dmul_rn(V[i], b2), __dmul_rn(__dmul_rn(one_b2, g), g));
    M[i] = m;
    V[i] = v;
    const double num = __dmul_rn(lr, __ddiv_rn(m, bc1));
    const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(v, bc2)), eps);
    P[i] = __dsub_rn(p, __ddiv_rn(num, den));
  }
}
}  // namespace
}  // namespace tpcb

extern "C" int tpcb_optimizer_step_f64(int64_t n, double* d_params, const double* d_grad,
                                       double* d_m, double* d_v, const tpcb_optim* opt,
                                       double lr, double bc1, double bc2, void* stream) {
  using namespace tpcb;
  if (n < 0 || !opt || (n > 0 && (!d_params || !d_grad))) return TPCB_ERR_VALIDATION;
  if (opt->kind != kOptAdam && opt->kind != kOptSgd) return TPCB_ERR_VALIDATION;
  if (opt->kind == kOptAdam && n > 0 && (!d_m || !d_v)) return TPCB_ERR_VALIDATION;
  if (n == 0) return TPCB_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8);
  optimizer_f64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      n, d_params, d_grad, d_m, d_v, opt->kind, opt->beta1, 1.0 - opt->beta1, opt->beta2,
      1.0 - opt->beta2, opt->eps, opt->weight_decay, lr, bc1, bc2);
  TPCB_LAUNCH_CHECK("optimizer_f64");
  return TPCB_OK;
}
