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
//   bucket_scan    per-bucket scan of the block histograms (one CTA per bucket)
//   bucket_scatter stable rank → perm, ast_row (warp match/ballot, no atomics),
//                  plus the per-tile plan (grid-strided)
//   pe_table       fp64 PE rows of positions 0..1023 (same sincos, looked up)
//   pack_rows      gather leaf vectors, add fp64 PE, write padded 128-B rows
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

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

// One CTA per bucket L (grid n_leaf_max, 1024 threads): exclusive scan of
// column L of the per-block histograms → blk_base[b][L] (relative to the
// bucket start) and the bucket's size cnt[L].  ws layout: blk_hist[nblk][17],
// blk_base[nblk][17], cnt[18], PE table.
__global__ void __launch_bounds__(1024) bucket_scan_kernel(const int32_t* __restrict__ blk_hist,
                                                           int nblk,
                                                           int32_t* __restrict__ blk_base,
                                                           int32_t* __restrict__ cnt) {
  const int L = blockIdx.x + 1;
  const int per = (nblk + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(nblk, b0 + per);
  int v[8];
  int sum = 0;
  if (per <= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q] = (b0 + q < b1) ? blk_hist[(int64_t)(b0 + q) * (kMaxL + 1) + L] : 0;
      sum += v[q];
    }
  } else {
    for (int b = b0; b < b1; ++b) sum += blk_hist[(int64_t)b * (kMaxL + 1) + L];
  }
  int total;
  int acc = block_excl_scan(sum, &total);
  if (per <= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b0 + q < b1) {
        blk_base[(int64_t)(b0 + q) * (kMaxL + 1) + L] = acc;
        acc += v[q];
      }
  } else {
    for (int b = b0; b < b1; ++b) {
      blk_base[(int64_t)b * (kMaxL + 1) + L] = acc;
      acc += blk_hist[(int64_t)b * (kMaxL + 1) + L];
    }
  }
  if (threadIdx.x == 0) cnt[L] = total;
}

// PE rows for serialized positions 0..kPeRows-1, fp64, the same sincos the
// pack kernel would evaluate (bit-identical table lookups)
constexpr int kPeRows = 1024;
__global__ void pe_table_kernel(PeDenom den, double* __restrict__ table) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kPeRows * (TPCB_FEAT / 2)) return;
  const int pos = idx / (TPCB_FEAT / 2), dl = idx - pos * (TPCB_FEAT / 2);
  double sn, cs;
  sincos((double)pos / den.v[dl], &sn, &cs);
  table[pos * TPCB_FEAT + 2 * dl] = sn;
  table[pos * TPCB_FEAT + 2 * dl + 1] = cs;
}

__global__ void bucket_scatter_kernel(const int64_t* __restrict__ leaf_off, int64_t n_ast,
                                      int n_leaf_max, int R,
                                      const int32_t* __restrict__ blk_base,
                                      const int32_t* __restrict__ cnt,
                                      int32_t* __restrict__ bucket_off_out,
                                      int32_t* __restrict__ perm, int32_t* __restrict__ ast_row,
                                      int32_t* __restrict__ n_tiles_out, int n_tiles_max,
                                      int32_t* __restrict__ tile_L,
                                      int32_t* __restrict__ tile_first,
                                      int32_t* __restrict__ tile_count,
                                      int32_t* __restrict__ row_tok,
                                      int32_t* __restrict__ row_ast) {
  __shared__ int warp_cnt[kScatterBlock / 32][kMaxL + 1];
  __shared__ int bucket_off[kMaxL + 2], tile_off[kMaxL + 2], s_base[kMaxL + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // every independent global load first (this AST's leaf range, the block's
  // bucket bases), so their latencies overlap the bucket-offset scan below
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t lo_i = 0, hi_i = 0;
  if (i < n_ast) {
    lo_i = leaf_off[i];
    hi_i = leaf_off[i + 1];
  }
  if (threadIdx.x >= 32 && threadIdx.x < 32 + kMaxL + 1)
    s_base[threadIdx.x - 32] = blk_base[(int64_t)blockIdx.x * (kMaxL + 1) + threadIdx.x - 32];
  if (w == 0) {  // bucket and tile offsets from the bucket sizes: lane L, warp scans
    const int L = lane;
    const int c = (L >= 1 && L <= n_leaf_max) ? cnt[L] : 0;
    const int tl = (L >= 1 && L <= n_leaf_max) ? (c + R / L - 1) / (R / L) : 0;
    int b = c, t = tl;  // inclusive prefix over lanes 1..L
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int bb = __shfl_up_sync(0xffffffffu, b, o), tt = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) {
        b += bb;
        t += tt;
      }
    }
    if (L <= n_leaf_max + 1) {  // exclusive prefix = offset of bucket L
      bucket_off[L] = b - c;
      tile_off[L] = t - tl;
    }
    if (L == n_leaf_max && blockIdx.x == 0) *n_tiles_out = t < n_tiles_max ? t : n_tiles_max;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x <= n_leaf_max + 1)
    bucket_off_out[threadIdx.x] = bucket_off[threadIdx.x];
  {  // tile plan, grid-strided over the tiles (bucket L cut into tiles of R/L ASTs)
    const int nt = min(tile_off[n_leaf_max + 1], n_tiles_max);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
      int L = 1;
      while (L < n_leaf_max && tile_off[L + 1] <= t) ++L;
      const int A = R / L;
      const int first = bucket_off[L] + (t - tile_off[L]) * A;
      tile_L[t] = L;
      tile_first[t] = first;
      tile_count[t] = min(A, bucket_off[L + 1] - first);
    }
  }
  for (int k = threadIdx.x; k < (kScatterBlock / 32) * (kMaxL + 1); k += blockDim.x)
    (&warp_cnt[0][0])[k] = 0;
  __syncthreads();
  int L = 0;
  if (i < n_ast) {
    const int64_t l64 = hi_i - lo_i;
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
    int pos = bucket_off[L] + s_base[L] + pre + rank;
    perm[pos] = (int32_t)i;
    int r = pos - bucket_off[L];
    int A = R / L;
    int tile = tile_off[L] + r / A;
    const int row0 = tile * R + (r % A) * L;
    ast_row[i] = row0;
    const int tok0 = (int)lo_i;  // n_tok < 2^31 (tpcb_pack_sizes)
    for (int l = 0; l < L; ++l) {  // the packed rows of AST i: source token + owner
      row_tok[row0 + l] = tok0 + l;
      row_ast[row0 + l] = (int32_t)i;
    }
  }
}

// One thread per packed row: the perm → leaf_off → ordering chain once per
// row, all 6 leaf-vector loads (and PE table reads) in flight together, the
// row staged in shared memory so the block writes its 256 consecutive rows
// (32 KB) with coalesced 16-byte stores.
constexpr int kPackThreads = 256;

// PE term for positions outside the table (rare): out of line, scalar in /
// scalar out, so the pack kernel keeps its row in registers
__device__ __noinline__ double pe_term(double pos, double den, int is_cos) {
  double sn, cs;
  sincos(pos / den, &sn, &cs);
  return is_cos ? cs : sn;
}
constexpr int kStagePitch = 28;  // floats per staged row (112 B: 16-B accesses conflict-free)

template <bool F64, bool PE>
__global__ void __launch_bounds__(kPackThreads, 2) pack_rows_kernel(
    const void* __restrict__ vectors_, const int32_t* __restrict__ ordering,
    const int64_t* __restrict__ leaf_off, const int32_t* __restrict__ perm,
    const int32_t* __restrict__ tile_L, const int32_t* __restrict__ tile_first,
    const int32_t* __restrict__ tile_count, const int32_t* __restrict__ n_tiles, int R,
    PeDenom den, const double* __restrict__ pe_table, const int32_t* __restrict__ row_tok,
    float* __restrict__ x, int32_t* __restrict__ row_ast) {
  __shared__ __align__(16) float stage[kPackThreads * kStagePitch];
  // the first kPeSmem rows of the PE table (positions < 64: every synthetic
  // ordering) in shared memory — the L1 path served them from L2 (ncu: L2
  // sectors ~2x the DRAM traffic)
  constexpr int kPeSmem = 64;
  // rows padded to 26 doubles: a 24-double (192-B) pitch put every even
  // position on the same 4 banks (16-way conflicts on the row reads); 208 B
  // spreads the rows over all 8 16-byte bank groups
  constexpr int kPePitch = TPCB_FEAT + 2;
  __shared__ __align__(16) double pe_s[PE ? kPeSmem * kPePitch : 2];
  if (PE) {
    for (int i = threadIdx.x; i < kPeSmem * TPCB_FEAT; i += kPackThreads)
      pe_s[(i / TPCB_FEAT) * kPePitch + i % TPCB_FEAT] = pe_table[i];
    __syncthreads();
  }
  constexpr int kChunks = TPCB_FEAT_PAD / 4;  // 6 float4 per packed row
  const int rshift = R == 32 ? 5 : (R == 64 ? 6 : 7);
  const int64_t rows = (int64_t)(*n_tiles) << rshift;
  const int64_t stride = (int64_t)gridDim.x * kPackThreads;
  // the row header (tile record + row → token, then token → position) of the
  // NEXT row is loaded while this row's vector is fetched: the two dependent
  // header levels overlap the third instead of preceding it
  struct Hdr {
    int live;  // 1: a real row, 0: a pad row of a tile, -1: past the end
    int tok;
  };
  auto header = [&](int64_t g) {
    Hdr h{-1, 0};
    if (g < rows) {
      const int t = (int)(g >> rshift), r = (int)(g & (R - 1));
      const int L = tile_L[t], cnt = tile_count[t];
      const int tok_r = row_tok[g];  // in flight with the tile record
      h.live = r / L < cnt ? 1 : 0;
      h.tok = tok_r;
    }
    return h;
  };
  // f32 rows: the next row's vector is loaded too, right after its token
  // arrives (under this row's staging and stores) — two rows in flight
  auto load_vec = [&](const Hdr& h, float4* dst) {
    if (!F64 && h.live == 1) {
      const float4* src =
          reinterpret_cast<const float4*>(static_cast<const float*>(vectors_) + (int64_t)h.tok * TPCB_FEAT);
#pragma unroll
      for (int q = 0; q < 6; ++q) dst[q] = __ldg(src + q);
    }
  };
  int64_t gr = (int64_t)blockIdx.x * kPackThreads + threadIdx.x;
  Hdr cur = header(gr);
  int ipos = (PE && cur.live == 1) ? ordering[cur.tok] : 0;
  float4 vr[6];
  load_vec(cur, vr);
  for (int64_t base = (int64_t)blockIdx.x * kPackThreads; base < rows; base += stride) {
    const Hdr nxt = header(gr + stride);
    float4 out[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) out[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cur.live == 1) {
      const int64_t tok = cur.tok;
      const bool table = ipos >= 0 && ipos < kPeRows;
      // two halves of 12 columns: half the live registers, 3-6 loads in flight each
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v[12];
        if (F64) {
          const double2* src = reinterpret_cast<const double2*>(
              static_cast<const double*>(vectors_) + tok * TPCB_FEAT + h * 12);
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const double2 p = __ldg(src + q);
            v[2 * q] = p.x;
            v[2 * q + 1] = p.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 p = vr[3 * h + q];
            v[4 * q] = p.x; v[4 * q + 1] = p.y; v[4 * q + 2] = p.z; v[4 * q + 3] = p.w;
          }
        }
        if (PE) {  // column 2δ: sin(pos/θ^(2δ/24)); 2δ+1: cos (features.py:255-262)
          if (ipos >= 0 && ipos < kPeSmem) {  // shared-memory rows
            const double2* tp =
                reinterpret_cast<const double2*>(pe_s + ipos * kPePitch + h * 12);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const double2 p = tp[q];
              v[2 * q] += p.x;
              v[2 * q + 1] += p.y;
            }
          } else if (table) {  // table row (L1/L2 resident)
            const double2* tp =
                reinterpret_cast<const double2*>(pe_table + ipos * TPCB_FEAT + h * 12);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const double2 p = __ldg(tp + q);
              v[2 * q] += p.x;
              v[2 * q + 1] += p.y;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 12; ++q) v[q] += pe_term((double)ipos, den.v[h * 6 + q / 2], q & 1);
          }
        }
#pragma unroll
        for (int q = 0; q < 3; ++q)
          out[3 * h + q] = make_float4((float)v[4 * q], (float)v[4 * q + 1],
                                       (float)v[4 * q + 2], (float)v[4 * q + 3]);
      }
    } else if (cur.live == 0) {
      row_ast[gr] = -1;  // pad row (real rows were written by bucket_scatter)
    }
    // the next row's position and vector (its token arrived during this row)
    const int ipos_n = (PE && nxt.live == 1) ? ordering[nxt.tok] : 0;
    float4 vn[6];
    load_vec(nxt, vn);
    // each warp stages its own 32 consecutive rows and writes them out as one
    // contiguous 3 KB run (coalesced 16-byte stores): warp barriers only
    float4* my = reinterpret_cast<float4*>(stage + threadIdx.x * kStagePitch);
#pragma unroll
    for (int q = 0; q < kChunks; ++q) my[q] = out[q];
    __syncwarp();
    {
      const int lane = threadIdx.x & 31, w0 = threadIdx.x & ~31;
      const int64_t wbase = base + w0;
      const int n_rows = rows - wbase < 32 ? (int)(rows - wbase) : 32;
      float4* dst = reinterpret_cast<float4*>(x) + wbase * kChunks;
      for (int e = lane; e < n_rows * kChunks; e += 32) {
        const int rr = e / kChunks, ch = e - rr * kChunks;
        dst[e] = reinterpret_cast<const float4*>(stage + (w0 + rr) * kStagePitch)[ch];
      }
    }
    __syncwarp();
    cur = nxt;
    ipos = ipos_n;
#pragma unroll
    for (int q = 0; q < 6; ++q) vr[q] = vn[q];
    gr += stride;
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

// byte offset of the PE table in the K1 workspace (16-byte aligned)
size_t pe_table_offset(int64_t nblk) {
  const size_t ints = (size_t)(2 * nblk * (TPCB_MAX_LEAF + 1) + TPCB_MAX_LEAF + 2) * 4;
  return (ints + 15) & ~(size_t)15;
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
  if (ws_bytes)
    *ws_bytes = pe_table_offset(nblk) + (size_t)kPeRows * TPCB_FEAT * sizeof(double) +
                (size_t)tiles * R * sizeof(int32_t);  // row_tok
  return TPCB_OK;
}

namespace tpcb {
namespace {
// The PE table depends only on θ (the denominators): built once per (device,
// θ) into a buffer that is never rewritten, with an event that later calls on
// other streams wait for — so repeated packs skip the sincos kernel.
struct PeCacheEntry {
  int device;
  PeDenom den;
  double* table;
  cudaEvent_t ready;
};
std::mutex g_pe_mu;
std::vector<PeCacheEntry> g_pe_cache;

int cached_pe_table(const PeDenom& den, cudaStream_t stream, const double** out) {
  *out = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  TPCB_CUDA_CHECK(cudaStreamIsCapturing(stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) return TPCB_OK;  // graphs keep their own copy
  int dev = 0;
  TPCB_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_pe_mu);
  for (const auto& e : g_pe_cache)
    if (e.device == dev && std::memcmp(&e.den, &den, sizeof(den)) == 0) {
      TPCB_CUDA_CHECK(cudaStreamWaitEvent(stream, e.ready, 0));
      *out = e.table;
      return TPCB_OK;
    }
  if (g_pe_cache.size() >= 16) return TPCB_OK;  // many distinct θ: no caching
  PeCacheEntry e{dev, den, nullptr, nullptr};
  TPCB_CUDA_CHECK(cudaMalloc(&e.table, sizeof(double) * kPeRows * TPCB_FEAT));
  TPCB_CUDA_CHECK(cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming));
  pe_table_kernel<<<(kPeRows * (TPCB_FEAT / 2) + 255) / 256, 256, 0, stream>>>(den, e.table);
  TPCB_LAUNCH_CHECK("pe_table");
  TPCB_CUDA_CHECK(cudaEventRecord(e.ready, stream));
  g_pe_cache.push_back(e);
  *out = e.table;
  return TPCB_OK;
}
}  // namespace
}  // namespace tpcb

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
  int32_t* cnt = blk_base + (int64_t)nblk * (TPCB_MAX_LEAF + 1);

  double* pe_table = reinterpret_cast<double*>(static_cast<char*>(d_ws) + pe_table_offset(nblk));
  int32_t* row_tok = reinterpret_cast<int32_t*>(pe_table + kPeRows * TPCB_FEAT);
  bucket_count_kernel<<<nblk, kScatterBlock, 0, stream>>>(d_leaf_off, n_ast, n_leaf_max,
                                                          blk_hist, d_status);
  TPCB_LAUNCH_CHECK("bucket_count");
  bucket_scan_kernel<<<n_leaf_max, 1024, 0, stream>>>(blk_hist, nblk, blk_base, cnt);
  TPCB_LAUNCH_CHECK("bucket_scan");
  bucket_scatter_kernel<<<nblk, kScatterBlock, 0, stream>>>(
      d_leaf_off, n_ast, n_leaf_max, R, blk_base, cnt, out->bucket_off, out->perm, out->ast_row,
      out->n_tiles, out->n_tiles_max, out->tile_L, out->tile_first, out->tile_count, row_tok,
      out->row_ast);
  TPCB_LAUNCH_CHECK("bucket_scatter");
  PeDenom den;
  for (int i = 0; i < TPCB_FEAT / 2; ++i) den.v[i] = pe_denom ? pe_denom[i] : 1.0;
  if (pe_denom) {
    const double* cached = nullptr;
    const int st = cached_pe_table(den, stream, &cached);
    if (st) return st;
    if (cached) {
      pe_table = const_cast<double*>(cached);
    } else {  // (cache full: this call's own copy in the workspace)
      pe_table_kernel<<<(kPeRows * (TPCB_FEAT / 2) + 255) / 256, 256, 0, stream>>>(den, pe_table);
      TPCB_LAUNCH_CHECK("pe_table");
    }
  }
  const int grid = (int)std::min<int64_t>(((int64_t)out->n_tiles_max * R + kPackThreads - 1) /
                                              kPackThreads, (int64_t)kNumSMs * 8);
  cudaStream_t st_ = stream;
#define TPCB_PACK(F64, PEF)                                                                  \
  pack_rows_kernel<F64, PEF><<<grid, kPackThreads, 0, st_>>>(d_vectors, d_ordering, d_leaf_off,      \
                                                    out->perm, out->tile_L, out->tile_first, \
                                                    out->tile_count, out->n_tiles, R, den,   \
                                                    pe_table, row_tok, out->x, out->row_ast)
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
