// Encoder weight gradients of the desk training step on the tensor cores.
//
// Reference: the weight gradients of costmodel._backward_group
// (costmodel.py:280-336; nn.linear_bwd, nn.py:30-36): dW = Σ_tokens xᵀ·dy,
// summed over every token row of the step's batch.  The desk training kernel
// (train4.cu) computes the step's forward and the dX chain per sample and
// stores the operand rows x and dy of the 13 encoder weight products (input
// projection; per layer Wq Wk Wv Wo, FFN hidden, FFN out) into the WgradDev
// buffer; this kernel forms each dW as ONE GEMM over all the step's token
// rows — K = n_samples · Ls (≤ 1,024) — instead of 64 per-sample outer-product
// sums written to gradient slots and reduced afterwards.
//
// One CTA per weight matrix: A = Xᵀ [in ≤ 128 rows (zero-padded) × K], B =
// dYᵀ [out × K], both fp32 in 32-row K chunks stored by train4 as K-major
// 128-byte-swizzled UMMA tiles, streamed by bulk copies through a 3-stage
// mbarrier ring; the tf32 remainder ("lo") of every operand element is
// formed in shared memory, and each 8-deep k step issues the 3xTF32 products
// (hi·hi + lo·hi + hi·lo, fp32 accumulation in TMEM: ~fp32 accuracy).  The
// epilogue (thread = TMEM lane = input feature k, row k of W) writes dW[k][:]
// into gradient slot 0 (whose encoder-weight regions train4 leaves unwritten
// on this path); the slot reduce takes those parameters' gradient from slot 0
// alone and applies the optimizer to every parameter in one pass (optim.cu).
// Deterministic: a fixed MMA order over fixed chunks.
#include <algorithm>
#include <cmath>

#include "async.cuh"
#include "common.cuh"
#include "train.cuh"

namespace tpcb {
namespace {

constexpr int kWgThreads = 160;  // 4 consumer / epilogue warps + 1 producer warp
constexpr int kWgStages = 3;
constexpr int kTileBytes = 128 * 128;            // 128 rows × 32 fp32 (128 B)
constexpr int kStageBytes = 4 * kTileBytes;      // A hi | A lo | B hi | B lo
constexpr int kWgSmem = kWgStages * kStageBytes + 1024;
constexpr int kMaxJobs = 16;

struct WgJob {
  int a_op, b_op;       // operands (train.cuh kWg*)
  int a_rows, a_real;   // stored / real input features (M, zero-padded to 128)
  int n;                // output features (N = stored B rows)
  int w_off, n_total;   // dW[k][c] is parameter w_off + k·n_total + c
};
struct WgJobs {
  int n;
  WgJob j[kMaxJobs];
};

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {  // K-major, 128-B swizzle
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// in-place tf32 split of `rows` swizzled 128-byte rows of one K chunk: hi
// stays (the tensor core reads its top 19 bits), lo = x − trunc_tf32(x)
// (exact in fp32); elements of step rows ≥ R are zeroed in both
__device__ __forceinline__ void split_tile(float* hi, float* lo, int rows, int row0, int R,
                                           int tid) {
  const int n4 = rows * 8;  // float4 per tile part
  for (int e = tid; e < n4; e += 128) {
    const int f = e >> 3, ch = e & 7;               // feature row, physical 16-B chunk
    const int j0 = (((ch ^ (f & 7))) << 2);         // logical row (K index) of its first float
    float4 x = reinterpret_cast<float4*>(hi)[e];
    float v[4] = {x.x, x.y, x.z, x.w}, l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (row0 + j0 + u >= R) v[u] = 0.f;
      l[u] = v[u] - __uint_as_float(__float_as_uint(v[u]) & 0xFFFFE000u);
    }
    reinterpret_cast<float4*>(hi)[e] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(lo)[e] = make_float4(l[0], l[1], l[2], l[3]);
  }
}

__global__ void __launch_bounds__(kWgThreads, 1) wgrad_tc_kernel(
    const __grid_constant__ WgJobs jobs, WgradDev wg, const StepDesc* __restrict__ steps,
    int step, const int32_t* __restrict__ batch_all, const int32_t* __restrict__ n_leaf,
    float* __restrict__ partial, size_t slot_stride) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kWgStages], empty[kWgStages], done;
  __shared__ uint32_t s_tmem;
  __shared__ int s_R;
  const WgJob jb = jobs.j[blockIdx.x];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const StepDesc sd = steps[step];
  if (warp == 0) {  // the step's row count: n_src · (largest leaf count), as train4
    const int32_t* batch = batch_all + sd.off;
    int m = 0;
    for (int i = lane; i < sd.n_src; i += 32) m = max(m, n_leaf[batch[i]]);
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if (lane == 0) s_R = sd.n_src * m;
  }
  if (t == 32) {
    for (int s = 0; s < kWgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A rows beyond the operand's stored features stay zero in every stage
  for (int s = 0; s < kWgStages; ++s) {
    float4* a = reinterpret_cast<float4*>(smem + s * kStageBytes);
    for (int e = jb.a_rows * 8 + t; e < 128 * 8; e += kWgThreads) {
      a[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      a[e + kTileBytes / 16] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int R = s_R;
  // split-K: block y takes chunks [c_lo, c_hi) and writes its partial dW to
  // gradient slot y (the slot reduce adds slots 0..S-1 in order)
  const int n_all = (R + 31) >> 5, S = gridDim.y;
  const int cps = (n_all + S - 1) / S;
  const int c_lo = min(n_all, (int)blockIdx.y * cps), c_hi = min(n_all, c_lo + cps);
  const int nch = c_hi - c_lo;
  float* gslot = partial + (size_t)blockIdx.y * slot_stride;
  const size_t a_base = (size_t)wg_op_off(jb.a_op) * wg.r_cap;
  const size_t b_base = (size_t)wg_op_off(jb.b_op) * wg.r_cap;
  const uint32_t a_bytes = (uint32_t)jb.a_rows * 128, b_bytes = (uint32_t)jb.n * 128;

  if (warp == 4) {  // producer: one chunk = the A and B tiles of 32 step rows
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % kWgStages;
        if (c >= kWgStages) mbar_wait(&empty[s], ((c / kWgStages) & 1) ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        const size_t cg = (size_t)(c_lo + c);
        mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
        bulk_g2s(st, wg.act + a_base + cg * jb.a_rows * 32, a_bytes, &full[s]);
        bulk_g2s(st + 2 * kTileBytes, wg.act + b_base + cg * jb.n * 32, b_bytes, &full[s]);
      }
    }
  } else {  // consumers: tf32 split, MMA issue (thread 0), then the epilogue
    const uint32_t id = idesc_tf32(128, jb.n);
    for (int c = 0; c < nch; ++c) {
      const int s = c % kWgStages;
      mbar_wait(&full[s], (c / kWgStages) & 1);
      uint8_t* st = smem + s * kStageBytes;
      split_tile(reinterpret_cast<float*>(st), reinterpret_cast<float*>(st + kTileBytes),
                 jb.a_rows, (c_lo + c) * 32, R, t);
      split_tile(reinterpret_cast<float*>(st + 2 * kTileBytes),
                 reinterpret_cast<float*>(st + 3 * kTileBytes), jb.n, (c_lo + c) * 32, R, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      group_bar(1, 128);
      if (t == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ah = smem_u32(st), al = ah + kTileBytes, bh = ah + 2 * kTileBytes,
                       bl = ah + 3 * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t o = kk * 32;
          mma_tf32(tmem, sdesc(ah + o), sdesc(bh + o), id, (c | kk) != 0);
          mma_tf32(tmem, sdesc(al + o), sdesc(bh + o), id, 1);
          mma_tf32(tmem, sdesc(ah + o), sdesc(bl + o), id, 1);
        }
        mma_commit(&empty[s]);
        if (c + 1 == nch) mma_commit(&done);
      }
    }
    if (nch > 0) {
      mbar_wait(&done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // epilogue: thread = TMEM lane = input feature k (warp w owns lanes 32w..):
    // dW[k][:] into gradient slot 0's (otherwise unused) region of this
    // tensor; the slot reduce applies the optimizer to it with every other
    // parameter (one parameter per thread over the whole GPU)
    const int k = 32 * warp + lane;
    for (int n0 = 0; n0 < jb.n; n0 += 32) {
      float g[32];
      if (nch > 0) {
        tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + n0, g);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) g[i] = 0.f;
      }
      if (k >= jb.a_real) continue;
      float4* dst = reinterpret_cast<float4*>(gslot + jb.w_off + k * jb.n_total + n0);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

WgJobs make_jobs(const Model& M) {
  WgJobs J{};
  auto add = [&](int a, int b, int a_real, int n, int off, int n_total) {
    WgJob& j = J.j[J.n++];
    j.a_op = a;
    j.b_op = b;
    j.a_rows = wg_op_rows(a);
    j.a_real = a_real;
    j.n = n;
    j.w_off = off;
    j.n_total = n_total;
  };
  for (int li = 0; li < M.n_layers; ++li) {
    const LayerOff& lo = M.layer[li];
    const int b = li * kWgOpsLayer;
    add(b + kWgHIN, b + kWgDQ, M.d, M.d, lo.Wq, M.d);
    add(b + kWgHIN, b + kWgDK, M.d, M.d, lo.Wk, M.d);
    add(b + kWgHIN, b + kWgDV, M.d, M.d, lo.Wv, M.d);
    add(b + kWgC, b + kWgDA, M.d, M.d, lo.Wo, M.d);
    add(b + kWgH1, b + kWgDF, M.d, M.d_ff, lo.fhW, M.d_ff);
    add(b + kWgF, b + kWgDT1, M.d_ff, M.d, lo.foW, M.d);
  }
  add(kWgX0, kWgDH, TPCB_FEAT, M.d, M.inW, M.d);
  return J;
}

}  // namespace

// split-K factor: about 4 chunks of 32 token rows per block at the largest
// step the workspace holds (the per-step row count is only known on the device)
int wgrad_tc_splits(const TrainWs& ws) {
  const int max_chunks = (int)(((int64_t)ws.n_slots * ws.l_cap + 31) / 32);
  return std::max(1, std::min(std::min((max_chunks + 3) / 4, ws.n_slots), 32));
}

// the desk shapes train4 handles (d 64, d_ff 128, 2 layers) — the operand
// table in train.cuh is written for them
bool wgrad_tc_supported(const Model& M) {
  return M.d == 64 && M.d_ff == 128 && M.n_layers == 2 && 2 * M.n_layers + 1 <= kMaxJobs;
}

int launch_wgrad_tc(const Model& M, const TrainWs& ws, const StepDesc* steps, int step,
                    const int32_t* batch, const int32_t* n_leaf, int splits,
                    cudaStream_t stream) {
  if (!wgrad_tc_supported(M) || !ws.wg.act || splits < 1 || splits > ws.n_slots)
    return TPCB_ERR_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(wgrad_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kWgSmem));
    attr = true;
  }
  const WgJobs jobs = make_jobs(M);
  wgrad_tc_kernel<<<dim3(jobs.n, splits), kWgThreads, kWgSmem, stream>>>(
      jobs, ws.wg, steps, step, batch, n_leaf, ws.partial, ws.slot_stride);
  TPCB_LAUNCH_CHECK("wgrad_tc_kernel");
  return TPCB_OK;
}

}  // namespace tpcb
