// K2+K3 — fused encoder + head forward over packed tiles (inference).
//
// One CTA owns one tile of R packed rows (floor(R/L) whole ASTs of one
// leaf-count bucket) and carries it through the whole network without
// touching HBM in between:
//   input projection → n_layers × [Q,K,V → per-AST attention → O-proj +
//   residual → LN1 → FFN(ReLU) + residual → LN2] → flatten → leaf_embed.{L}
//   → device MLP gate → decoder → prediction (→ Box-Cox decode)
// Reference: costmodel.py:193-269 (forward), nn.py:26-96, dataset.py:97-115.
//
// FP32 FFMA path ("fp32 parity mode"): every GEMM accumulates in fp32; the
// decode runs in fp64.  Grid-stride over tiles so the launch needs no host
// knowledge of the device-computed tile count.
#include <cmath>

#include "blocks.cuh"
#include "common.cuh"

namespace tpcb {

struct FwdPlan {
  int R, ld, ldf;
  int H, C, V, Q, K, F, X0;             // encoder buffers
  int zx, zv, zp, z, u0, u1, dv, uw;    // head buffers (uw = max decoder width)
  int ls;                               // leaf_embed slice partials (16-B aligned)
  int total;                            // floats
};

FwdPlan make_fwd_plan(const Model& M, int R) {
  FwdPlan p;
  p.R = R;
  p.ld = M.d + 1;
  p.ldf = M.d_ff + 1;
  const int blk = R * p.ld;
  p.H = 0;
  p.C = blk;
  p.V = 2 * blk;
  p.Q = 3 * blk;
  p.K = 4 * blk;
  int end = 5 * blk;
  if (R * p.ldf <= 2 * blk) {
    p.F = p.Q;
  } else {
    p.F = end;
    end += R * p.ldf;
  }
  p.X0 = p.C;  // input rows (stride 25) consumed by the input projection
  end = max(end, p.C + R * (TPCB_FEAT + 1));
  int uw = 1;
  for (int i = 0; i < M.n_dec; ++i) uw = max(uw, M.dec[i]);
  p.uw = uw;
  int o = p.C;  // head scratch reuses everything but H
  p.zx = o; o += R * M.d_e;
  p.zp = o; o += R * M.d_e;
  p.z = o; o += R * M.d_e;
  p.zv = o; o += R * M.d_dev;
  p.u0 = o; o += R * uw;
  p.u1 = o; o += R * uw;
  p.dv = o; o += R * TPCB_DEV_FEAT;
  o = (o + 3) & ~3;
  p.ls = o; o += max(4 * 256, R * M.d_e);
  p.total = max(end, o);
  return p;
}

__device__ __forceinline__ double boxcox_decode(double e, const tpcb_boxcox& bc, bool* bad) {
  const double t = e * bc.t_std + bc.t_mean;
  if (fabs(bc.lambda_bc) < 1e-9) return exp(t) - bc.shift;
  const double base = bc.lambda_bc * t + 1.0;
  if (!(base > 0.0)) {
    *bad = true;
    return nan("");
  }
  return pow(base, 1.0 / bc.lambda_bc) - bc.shift;
}

__device__ long long* g_trace_fwd = nullptr;
int set_forward_trace(long long* d) {
  TPCB_CUDA_CHECK(cudaMemcpyToSymbol(g_trace_fwd, &d, sizeof(d)));
  return TPCB_OK;
}
// debug: per-phase timestamps of CTA 0 / thread 0, last 8 tiles (ring)
#define FT(id)                                                                      \
  do {                                                                              \
    if (g_trace_fwd && blockIdx.x == 0 && threadIdx.x == 0)                         \
      g_trace_fwd[(tcount & 7) * 32 + (id)] = clock64();                            \
  } while (0)

__global__ void __launch_bounds__(256) forward_kernel(
    Model M, const float* __restrict__ P, const float* __restrict__ x,
    const int32_t* __restrict__ tile_L, const int32_t* __restrict__ tile_first,
    const int32_t* __restrict__ tile_count, const int32_t* __restrict__ n_tiles_p,
    const int32_t* __restrict__ perm, const float* __restrict__ devfeat, FwdPlan sp,
    tpcb_boxcox bc, float* __restrict__ pred_out, float* __restrict__ zx_out,
    float* __restrict__ zv_out, float* __restrict__ z_out, double* __restrict__ lat_out,
    int32_t* status) {
  extern __shared__ float sm[];
  const int n_tiles = *n_tiles_p;
  const int R = sp.R, ld = sp.ld, ldf = sp.ldf, d = M.d;
  float* H = sm + sp.H;
  float* C = sm + sp.C;
  float* V = sm + sp.V;
  float* Q = sm + sp.Q;
  float* K = sm + sp.K;
  float* F = sm + sp.F;
  float* X0 = sm + sp.X0;
  const float scale = 1.f / sqrtf((float)M.dh);

  int tcount = -1;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    ++tcount;
    FT(0);
    if (g_trace_fwd && blockIdx.x == 0 && threadIdx.x == 0) g_trace_fwd[(tcount & 7) * 32 + 31] = tile_L[t];
    const int L = tile_L[t], first = tile_first[t], A = tile_count[t];
    const int rows = A * L;
    const float* xt = x + (size_t)t * R * TPCB_FEAT_PAD;
    for (int idx = threadIdx.x; idx < rows * TPCB_FEAT; idx += blockDim.x) {
      const int r = idx / TPCB_FEAT, c = idx - r * TPCB_FEAT;
      X0[r * (TPCB_FEAT + 1) + c] = __ldg(xt + r * TPCB_FEAT_PAD + c);
    }
    __syncthreads();
    FT(1);
    gemm_rows<4, 4>(X0, TPCB_FEAT + 1, P + M.inW, P + M.inb, H, ld, rows, TPCB_FEAT, d, false);
    __syncthreads();
    FT(2);
    for (int li = 0; li < M.n_layers; ++li) {
      const LayerOff& lo = M.layer[li];
      gemm_rows<4, 4>(H, ld, P + lo.Wq, P + lo.bq, Q, ld, rows, d, d, false);
      gemm_rows<4, 4>(H, ld, P + lo.Wk, P + lo.bk, K, ld, rows, d, d, false);
      gemm_rows<4, 4>(H, ld, P + lo.Wv, P + lo.bv, V, ld, rows, d, d, false);
      __syncthreads();
      FT(3 + 6 * li);
      attention_rows(Q, K, V, ld, C, ld, A, L, M.n_heads, M.dh, scale);
      __syncthreads();
      FT(4 + 6 * li);
      // r1 = H + ctx Wo + bo  → V (dead after attention)
      gemm_rows<4, 4>(C, ld, P + lo.Wo, P + lo.bo, V, ld, rows, d, d, false, H, ld);
      __syncthreads();
      FT(5 + 6 * li);
      layernorm_rows(V, ld, C, ld, rows, d, P + lo.ln1g, P + lo.ln1b);  // h1 → C
      __syncthreads();
      FT(6 + 6 * li);
      gemm_rows<4, 4>(C, ld, P + lo.fhW, P + lo.fhb, F, ldf, rows, d, M.d_ff, true);
      __syncthreads();
      // r2 = h1 + relu(..) Wo2 + b → V
      FT(7 + 6 * li);
      gemm_rows<4, 4>(F, ldf, P + lo.foW, P + lo.fob, V, ld, rows, M.d_ff, d, false, C, ld);
      __syncthreads();
      layernorm_rows(V, ld, H, ld, rows, d, P + lo.ln2g, P + lo.ln2b);
      __syncthreads();
      FT(8 + 6 * li);
    }
    // ---------------------------------------------------------------- head
    float* zx = sm + sp.zx;
    float* zp = sm + sp.zp;
    float* z = sm + sp.z;
    float* zv = sm + sp.zv;
    float* dv = sm + sp.dv;
    for (int idx = threadIdx.x; idx < A * TPCB_DEV_FEAT; idx += blockDim.x) {
      const int a = idx / TPCB_DEV_FEAT, f = idx - a * TPCB_DEV_FEAT;
      dv[idx] = __ldg(devfeat + (size_t)perm[first + a] * TPCB_DEV_FEAT + f);
    }
    FT(20);
    leaf_embed_rows(H, ld, A, L, d, P + M.leafW[L], P + M.leafb[L], M.d_e, zx, M.d_e,
                    sm + sp.ls);
    __syncthreads();
    FT(21);
    gemm_rows<1, 4>(dv, TPCB_DEV_FEAT, P + M.devhW, P + M.devhb, zv, M.d_dev, A, TPCB_DEV_FEAT,
                    M.d_dev, true);
    __syncthreads();
    gemm_rows<1, 4>(zv, M.d_dev, P + M.devpW, P + M.devpb, zp, M.d_e, A, M.d_dev, M.d_e, false);
    __syncthreads();
    for (int idx = threadIdx.x; idx < A * M.d_e; idx += blockDim.x) z[idx] = zx[idx] * zp[idx];
    __syncthreads();
    FT(22);
    const float* u = z;
    int w = M.d_e;
    float* ubuf[2] = {sm + sp.u0, sm + sp.u1};
    for (int j = 0; j < M.n_dec; ++j) {
      float* o = ubuf[j & 1];
      gemm_rows<1, 4>(u, w, P + M.decW[j], P + M.decb[j], o, M.dec[j], A, w, M.dec[j], true);
      __syncthreads();
      u = o;
      w = M.dec[j];
    }
    FT(23);
    // final scalar: one warp per AST
    {
      const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int a = wp; a < A; a += nw) {
        float s = 0.f;
        for (int c = lane; c < w; c += 32) s = fmaf(u[a * w + c], __ldg(P + M.outW + c), s);
        s = warp_sum(s) + __ldg(P + M.outb);
        if (lane == 0) {
          const int i = perm[first + a];
          pred_out[i] = s;
          if (lat_out) {
            bool bad = false;
            lat_out[i] = bc.enabled ? boxcox_decode((double)s, bc, &bad) : (double)s;
            if (bad) raise_status(status, TPCB_ERR_DOMAIN);
          }
        }
      }
    }
    FT(24);
    if (zx_out || z_out) {
      for (int idx = threadIdx.x; idx < A * M.d_e; idx += blockDim.x) {
        const int a = idx / M.d_e, e = idx - a * M.d_e;
        const size_t o = (size_t)perm[first + a] * M.d_e + e;
        if (zx_out) zx_out[o] = zx[idx];
        if (z_out) z_out[o] = z[idx];
      }
    }
    if (zv_out) {
      for (int idx = threadIdx.x; idx < A * M.d_dev; idx += blockDim.x) {
        const int a = idx / M.d_dev, e = idx - a * M.d_dev;
        zv_out[(size_t)perm[first + a] * M.d_dev + e] = zv[idx];
      }
    }
    __syncthreads();
  }
}

// MAPE / RMSE / MSPE of decoded predictions (costmodel.metrics,
// costmodel.py:577-591) in fp64, fixed-order block reduction (1 CTA).
__global__ void __launch_bounds__(1024) metrics_kernel(const double* __restrict__ pred,
                                                       const double* __restrict__ y, int64_t n,
                                                       double* __restrict__ out) {
  __shared__ double red[3][32];
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = pred[i] - y[i];
    const double r = d / y[i];
    a += fabs(r);
    b += d * d;
    c += r * r;
  }
  a = warp_sum_d(a);
  b = warp_sum_d(b);
  c = warp_sum_d(c);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][w] = a;
    red[1][w] = b;
    red[2][w] = c;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? red[0][lane] : 0.0;
    b = lane < nw ? red[1][lane] : 0.0;
    c = lane < nw ? red[2][lane] : 0.0;
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    c = warp_sum_d(c);
    if (lane == 0) {
      out[0] = a / (double)n;
      out[1] = sqrt(b / (double)n);
      out[2] = c / (double)n;
    }
  }
}

}  // namespace tpcb

using namespace tpcb;

extern "C" int tpcb_metrics(const double* d_pred, const double* d_y, int64_t n, double* d_out,
                            void* stream) {
  if (!d_pred || !d_y || !d_out) return TPCB_ERR_VALIDATION;
  if (n < 1) return TPCB_ERR_EMPTY_BATCH;
  metrics_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_pred, d_y, n, d_out);
  TPCB_LAUNCH_CHECK("metrics_kernel");
  return TPCB_OK;
}

namespace tpcb {
bool f32_fast_supported(const Model& M);
int launch_forward_f32(const Model& M, const float* d_params, const tpcb_packed* pk,
                       const float* d_devfeat, const tpcb_boxcox* norm, float* d_pred,
                       float* d_zx, float* d_zv, float* d_z, double* d_latency, int32_t* d_status,
                       cudaStream_t stream);
}  // namespace tpcb

/* preferred rows per packed tile for tpcb_forward: 128 when the desk-shaped
 * fp32 kernel (forward_f32.cu) applies, else 64 (the generic kernel) */
extern "C" int32_t tpcb_forward_rows(const tpcb_model* m) {
  if (!m) return 64;
  return f32_fast_supported(m->dev) ? 128 : 64;
}

extern "C" int32_t tpcb_forward_fits(const tpcb_model* m, int32_t R) {
  if (!m || R < m->dev.n_leaf_max) return 0;
  if (R == 128 && f32_fast_supported(m->dev)) return 1;
  return (size_t)make_fwd_plan(m->dev, R).total * sizeof(float) <= 227 * 1024 ? 1 : 0;
}

extern "C" int tpcb_forward(const tpcb_model* m, const float* d_params, const tpcb_packed* pk,
                            const float* d_devfeat, int64_t n_ast, const tpcb_boxcox* norm,
                            float* d_pred, float* d_zx, float* d_zv, float* d_z,
                            double* d_latency, int32_t* d_status, void* stream_) {
  if (!m || !pk || !d_params || !d_pred || !d_devfeat) return TPCB_ERR_VALIDATION;
  if (n_ast < 1) return TPCB_ERR_EMPTY_BATCH;
  const int R = pk->rows_per_tile;
  if (R < m->dev.n_leaf_max) return TPCB_ERR_UNSUPPORTED;
  if (R == 128 && f32_fast_supported(m->dev))  // desk shapes: forward_f32.cu
    return launch_forward_f32(m->dev, d_params, pk, d_devfeat, norm, d_pred, d_zx, d_zv, d_z,
                              d_latency, d_status, (cudaStream_t)stream_);
  FwdPlan sp = make_fwd_plan(m->dev, R);
  const size_t smem = (size_t)sp.total * sizeof(float);
  if (smem > 227 * 1024) return TPCB_ERR_UNSUPPORTED;
  if (m->dev.dh > 4096) return TPCB_ERR_UNSUPPORTED;
  TPCB_CUDA_CHECK(cudaFuncSetAttribute(forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
  tpcb_boxcox bc{};
  if (norm) bc = *norm;
  int occ = 1;
  TPCB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, forward_kernel, 256, smem));
  if (occ < 1) occ = 1;
  const int grid = (int)std::min<int64_t>(pk->n_tiles_max, (int64_t)kNumSMs * occ);
  forward_kernel<<<grid, 256, smem, (cudaStream_t)stream_>>>(
      m->dev, d_params, pk->x, pk->tile_L, pk->tile_first, pk->tile_count, pk->n_tiles, pk->perm,
      d_devfeat, sp, bc, d_pred, d_zx, d_zv, d_z, d_latency, d_status);
  TPCB_LAUNCH_CHECK("forward_kernel");
  return TPCB_OK;
}
