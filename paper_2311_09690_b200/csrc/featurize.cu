// K1 — featurize + bucket pack.
//
// Replaces, in one stream-ordered pass with no host round trip:
//   features.positional_encoding / encode_input   (features.py:248-279)
//   costmodel._group_by_leaf + sorted-bucket stack (costmodel.py:181-190, 248-251)
//
// Output contract (bit-exact vs oracle/featurize.py): perm = stable argsort of
// n_leaf; bucket L is cut into tiles of floor(R/L) whole ASTs (rows a*L ..
// a*L+L-1 of the tile hold AST a's leaves); pad rows are zero with row_ast=-1.
//
// Four kernels (HBM-bound; pack_rows is the only one that moves bulk data):
//   bucket_count   per-block n_leaf histogram + range check
//   bucket_scan    bucket offsets, per-block bases, tile plan (1 CTA)
//   bucket_scatter stable rank → perm, ast_row (warp match/ballot, no atomics)
//   pack_rows      gather leaf vectors, add fp64 PE, write padded 128-B rows
#include <cmath>

#include "common.cuh"

namespace tpcb {

namespace {

constexpr int kScatterBlock = 256;  // ASTs per block in count/scatter
constexpr int kMaxL = TPCB_MAX_LEAF;

struct PeDenom {
  double v[TPCB_FEAT / 2];
};

__global__ void bucket_count_kernel(const int64_t* __restrict__ leaf_off, int64_t n_ast,
                                    int n_leaf_max, int32_t* __restrict__ blk_hist,
                                    int32_t* status) {
  __shared__ int32_t hist[kMaxL + 1];
  if (threadIdx.x <= kMaxL) hist[threadIdx.x] = 0;
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_ast) {
    int64_t L = leaf_off[i + 1] - leaf_off[i];
    if (L < 1 || L > n_leaf_max) {
      raise_status(status, TPCB_ERR_LEAF_COUNT);
    } else {
      atomicAdd(&hist[L], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x <= n_leaf_max)
    blk_hist[(int64_t)blockIdx.x * (kMaxL + 1) + threadIdx.x] = hist[threadIdx.x];
}

// Exclusive block scan of one int per thread; *total = block sum.
__device__ int block_excl_scan(int v, int* total) {
  __shared__ int wt[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wt[w] = incl;
  __syncthreads();
  if (w == 0) {
    int t = lane < nw ? wt[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    wt[lane] = t;  // inclusive prefix over warps
  }
  __syncthreads();
  const int res = incl - v + (w ? wt[w - 1] : 0);
  *total = wt[nw - 1];
  __syncthreads();  // wt is reused by the next call
  return res;
}

// One CTA of 1024 threads.  ws layout: blk_hist[nblk][17], blk_base[nblk][17],
// tile_off[18].
__global__ void __launch_bounds__(1024) bucket_scan_kernel(
    const int32_t* __restrict__ blk_hist, int nblk, int n_leaf_max, int R,
    int32_t* __restrict__ blk_base, int32_t* __restrict__ bucket_off,
    int32_t* __restrict__ tile_off, int32_t* __restrict__ tile_L,
    int32_t* __restrict__ tile_first, int32_t* __restrict__ tile_count,
    int32_t* __restrict__ n_tiles_out, int n_tiles_max) {
  __shared__ int s_boff[kMaxL + 2];
  __shared__ int s_toff[kMaxL + 2];
  const int per = (nblk + blockDim.x - 1) / blockDim.x;
  int running = 0;  // start of bucket L
  if (threadIdx.x == 0) s_boff[0] = 0;
  for (int L = 1; L <= n_leaf_max; ++L) {
    int b0 = threadIdx.x * per;
    int sum = 0;
    for (int b = b0; b < b0 + per && b < nblk; ++b) sum += blk_hist[(int64_t)b * (kMaxL + 1) + L];
    int total;
    int ex = block_excl_scan(sum, &total);
    int acc = running + ex;
    for (int b = b0; b < b0 + per && b < nblk; ++b) {
      blk_base[(int64_t)b * (kMaxL + 1) + L] = acc;
      acc += blk_hist[(int64_t)b * (kMaxL + 1) + L];
    }
    if (threadIdx.x == 0) s_boff[L] = running;
    running += total;
  }
  if (threadIdx.x == 0) {
    s_boff[n_leaf_max + 1] = running;
    int t = 0;
    for (int L = 1; L <= n_leaf_max; ++L) {
      s_toff[L] = t;
      int cnt = s_boff[L + 1] - s_boff[L];
      int A = R / L;
      t += (cnt + A - 1) / A;
    }
    s_toff[n_leaf_max + 1] = t;
    *n_tiles_out = t < n_tiles_max ? t : n_tiles_max;
  }
  __syncthreads();
  if (threadIdx.x <= n_leaf_max + 1) {
    bucket_off[threadIdx.x] = s_boff[threadIdx.x];
    tile_off[threadIdx.x] = s_toff[threadIdx.x];
  }
  const int nt = s_toff[n_leaf_max + 1];
  for (int t = threadIdx.x; t < nt && t < n_tiles_max; t += blockDim.x) {
    int L = 1;
    while (L < n_leaf_max && s_toff[L + 1] <= t) ++L;
    int A = R / L;
    int first = s_boff[L] + (t - s_toff[L]) * A;
    int end = s_boff[L + 1];
    tile_L[t] = L;
    tile_first[t] = first;
    tile_count[t] = min(A, end - first);
  }
}

__global__ void bucket_scatter_kernel(const int64_t* __restrict__ leaf_off, int64_t n_ast,
                                      int n_leaf_max, int R,
                                      const int32_t* __restrict__ blk_base,
                                      const int32_t* __restrict__ bucket_off,
                                      const int32_t* __restrict__ tile_off,
                                      int32_t* __restrict__ perm, int32_t* __restrict__ ast_row) {
  __shared__ int warp_cnt[kScatterBlock / 32][kMaxL + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < (kScatterBlock / 32) * (kMaxL + 1); k += blockDim.x)
    (&warp_cnt[0][0])[k] = 0;
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int L = 0;
  if (i < n_ast) {
    int64_t l64 = leaf_off[i + 1] - leaf_off[i];
    L = (l64 >= 1 && l64 <= n_leaf_max) ? (int)l64 : 0;
  }
  unsigned peers = __match_any_sync(0xffffffffu, L);
  unsigned lt = (1u << lane) - 1u;
  int rank = __popc(peers & lt);
  if (rank == 0) warp_cnt[w][L] = __popc(peers);
  __syncthreads();
  if (i < n_ast && L > 0) {
    int pre = 0;
    for (int ww = 0; ww < w; ++ww) pre += warp_cnt[ww][L];
    int pos = blk_base[(int64_t)blockIdx.x * (kMaxL + 1) + L] + pre + rank;
    perm[pos] = (int32_t)i;
    int r = pos - bucket_off[L];
    int A = R / L;
    int tile = tile_off[L] + r / A;
    ast_row[i] = tile * R + (r % A) * L;
  }
}

template <bool F64, bool PE>
__global__ void pack_rows_kernel(const void* __restrict__ vectors_,
                                 const int32_t* __restrict__ ordering,
                                 const int64_t* __restrict__ leaf_off,
                                 const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ tile_L,
                                 const int32_t* __restrict__ tile_first,
                                 const int32_t* __restrict__ tile_count,
                                 const int32_t* __restrict__ n_tiles, int R, PeDenom den,
                                 float* __restrict__ x, int32_t* __restrict__ row_ast) {
  const int nt = *n_tiles;
  constexpr int kChunks = TPCB_FEAT_PAD / 4;  // 8 float4 per packed row
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const int L = tile_L[t], first = tile_first[t], cnt = tile_count[t];
    for (int item = threadIdx.x; item < R * kChunks; item += blockDim.x) {
      const int r = item / kChunks, ch = item % kChunks;
      const int a = r / L, l = r - a * L;
      float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
      int ast = -1;
      if (a < cnt) {
        ast = perm[first + a];
        if (ch * 4 < TPCB_FEAT) {
          const int64_t tok = leaf_off[ast] + l;
          const double pos = (double)ordering[tok];
          double v[4];
          if (F64) {
            const double2* src = reinterpret_cast<const double2*>(
                static_cast<const double*>(vectors_) + tok * TPCB_FEAT + ch * 4);
            double2 p0 = __ldg(src), p1 = __ldg(src + 1);
            v[0] = p0.x; v[1] = p0.y; v[2] = p1.x; v[3] = p1.y;
          } else {
            float4 p = __ldg(reinterpret_cast<const float4*>(
                static_cast<const float*>(vectors_) + tok * TPCB_FEAT + ch * 4));
            v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w;
          }
          // column 2δ: sin(pos/θ^(2δ/24)); 2δ+1: cos (features.py:255-262)
          double s0 = 0.0, c0 = 0.0, s1 = 0.0, c1 = 0.0;
          if (PE) {
            const int d0 = ch * 2;
            sincos(pos / den.v[d0], &s0, &c0);
            sincos(pos / den.v[d0 + 1], &s1, &c1);
          }
          out.x = (float)(v[0] + s0);
          out.y = (float)(v[1] + c0);
          out.z = (float)(v[2] + s1);
          out.w = (float)(v[3] + c1);
        }
      }
      reinterpret_cast<float4*>(x)[((int64_t)t * R + r) * kChunks + ch] = out;
      if (ch == 0) row_ast[(int64_t)t * R + r] = ast;
    }
  }
}

__global__ void positional_kernel(const int32_t* __restrict__ ordering, int64_t n, PeDenom den,
                                  double* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * (TPCB_FEAT / 2)) return;
  const int64_t r = idx / (TPCB_FEAT / 2);
  const int dl = (int)(idx - r * (TPCB_FEAT / 2));
  double s, c;
  sincos((double)ordering[r] / den.v[dl], &s, &c);
  out[r * TPCB_FEAT + 2 * dl] = s;
  out[r * TPCB_FEAT + 2 * dl + 1] = c;
}

int min_rows_per_tile(int R, int n_leaf_max) {
  int m = R;
  for (int L = 1; L <= n_leaf_max; ++L) m = min(m, (R / L) * L);
  return m;
}

}  // namespace

}  // namespace tpcb

using namespace tpcb;

extern "C" int tpcb_pack_sizes(int64_t n_ast, int64_t n_tok, int32_t n_leaf_max, int32_t R,
                               int32_t* n_tiles_max, size_t* ws_bytes) {
  if (n_leaf_max < 1 || n_leaf_max > TPCB_MAX_LEAF) return TPCB_ERR_UNSUPPORTED;
  if (R != 32 && R != 64 && R != 128) return TPCB_ERR_UNSUPPORTED;
  if (R < n_leaf_max) return TPCB_ERR_UNSUPPORTED;
  if (n_ast < 0 || n_tok < 0 || n_tok > (int64_t)1 << 31) return TPCB_ERR_VALIDATION;
  int64_t per = min_rows_per_tile(R, n_leaf_max);
  int64_t tiles = (n_tok + per - 1) / per + n_leaf_max;
  if (tiles * R > ((int64_t)1 << 31)) return TPCB_ERR_UNSUPPORTED;
  if (n_tiles_max) *n_tiles_max = (int32_t)tiles;
  int64_t nblk = (n_ast + kScatterBlock - 1) / kScatterBlock;
  if (nblk < 1) nblk = 1;
  if (ws_bytes) *ws_bytes = (size_t)(2 * nblk * (TPCB_MAX_LEAF + 1) + TPCB_MAX_LEAF + 2) * 4;
  return TPCB_OK;
}

extern "C" int tpcb_featurize_pack(const void* d_vectors, int32_t vec_is_f64,
                                   const int32_t* d_ordering, const int64_t* d_leaf_off,
                                   int64_t n_ast, int64_t n_tok, int32_t n_leaf_max,
                                   const double* pe_denom, void* d_ws, size_t ws_bytes,
                                   tpcb_packed* out, int32_t* d_status, void* stream_) {
  if (!out) return TPCB_ERR_VALIDATION;
  if (n_ast < 1) return TPCB_ERR_EMPTY_BATCH;
  int32_t ntm = 0;
  size_t need = 0;
  int st = tpcb_pack_sizes(n_ast, n_tok, n_leaf_max, out->rows_per_tile, &ntm, &need);
  if (st) return st;
  if (ws_bytes < need || out->n_tiles_max < ntm) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int R = out->rows_per_tile;
  const int nblk = (int)((n_ast + kScatterBlock - 1) / kScatterBlock);
  int32_t* blk_hist = static_cast<int32_t*>(d_ws);
  int32_t* blk_base = blk_hist + (int64_t)nblk * (TPCB_MAX_LEAF + 1);
  int32_t* tile_off = blk_base + (int64_t)nblk * (TPCB_MAX_LEAF + 1);

  bucket_count_kernel<<<nblk, kScatterBlock, 0, stream>>>(d_leaf_off, n_ast, n_leaf_max,
                                                          blk_hist, d_status);
  TPCB_LAUNCH_CHECK("bucket_count");
  bucket_scan_kernel<<<1, 1024, 0, stream>>>(blk_hist, nblk, n_leaf_max, R, blk_base,
                                             out->bucket_off, tile_off, out->tile_L,
                                             out->tile_first, out->tile_count, out->n_tiles,
                                             out->n_tiles_max);
  TPCB_LAUNCH_CHECK("bucket_scan");
  bucket_scatter_kernel<<<nblk, kScatterBlock, 0, stream>>>(
      d_leaf_off, n_ast, n_leaf_max, R, blk_base, out->bucket_off, tile_off, out->perm,
      out->ast_row);
  TPCB_LAUNCH_CHECK("bucket_scatter");
  PeDenom den;
  for (int i = 0; i < TPCB_FEAT / 2; ++i) den.v[i] = pe_denom ? pe_denom[i] : 1.0;
  const int grid = min(out->n_tiles_max, kNumSMs * 8);
  cudaStream_t st_ = stream;
#define TPCB_PACK(F64, PEF)                                                                  \
  pack_rows_kernel<F64, PEF><<<grid, 256, 0, st_>>>(d_vectors, d_ordering, d_leaf_off,      \
                                                    out->perm, out->tile_L, out->tile_first, \
                                                    out->tile_count, out->n_tiles, R, den,   \
                                                    out->x, out->row_ast)
  if (vec_is_f64) {
    if (pe_denom) TPCB_PACK(true, true); else TPCB_PACK(true, false);
  } else {
    if (pe_denom) TPCB_PACK(false, true); else TPCB_PACK(false, false);
  }
#undef TPCB_PACK
  TPCB_LAUNCH_CHECK("pack_rows");
  return TPCB_OK;
}

extern "C" int tpcb_positional_encoding(const int32_t* d_ordering, int64_t n,
                                        const double* pe_denom, double* d_out, void* stream) {
  if (!pe_denom || n < 0) return TPCB_ERR_VALIDATION;
  if (n == 0) return TPCB_OK;
  PeDenom den;
  for (int i = 0; i < TPCB_FEAT / 2; ++i) den.v[i] = pe_denom[i];
  const int64_t items = n * (TPCB_FEAT / 2);
  positional_kernel<<<(unsigned)((items + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      d_ordering, n, den, d_out);
  TPCB_LAUNCH_CHECK("positional_kernel");
  return TPCB_OK;
}
