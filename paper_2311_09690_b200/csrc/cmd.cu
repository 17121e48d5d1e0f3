// K6 standalone — central moment discrepancy between two sets (fp64).
// Replaces costmodel.cmd / cmd_between (costmodel.py:489-503, 783-788):
// one CTA computes the column statistics of the union (extrema with their
// first index, means, central power sums up to order K) and, optionally, the
// gradient w.r.t. every row (costmodel.py:426-486).  The in-training CMD term
// uses the same device functions (train.cu).
#include <algorithm>
#include <type_traits>

#include "cmd.cuh"
#include "common.cuh"

namespace tpcb {
namespace {

template <typename T>
__global__ void __launch_bounds__(1024) cmd_kernel(const T* __restrict__ Z, int ns, int nt, int de,
                                                   int K, double* value, double* grad) {
  extern __shared__ double cs[];
  const double v = cmd_stats(Z, ns, nt, de, K, cs);
  if (threadIdx.x == 0) *value = v;
  if (grad) {
    const size_t total = (size_t)(ns + nt) * de;
    for (size_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int row = (int)(e / de), c = (int)(e - (size_t)row * de);
      grad[e] = cmd_grad_elem(cs, ns, nt, de, K, row, c, (double)Z[e]);
    }
  }
}

// ---- grid version for large sets (cmd_between over whole datasets) --------
// HBM-bound: pass AC (extrema + shifted power sums) and pass E (gradient)
// each stream Z once with coalesced row reads (lane = column); the combine
// runs one block per column.  Each block owns a
// chunk of kChunk rows of ONE set, chunked from that set's own first row, and
// partials are combined in block order — so the reduction order is fixed
// (bitwise reproducible) and identical for identical sets: cmd(S, S) is
// exactly 0 as in the reference (costmodel.py:446-475 guards).
constexpr int kChunk = 512;
constexpr int kGridThreads = 256;
constexpr int kMaxGridDe = 128;  // columns per lane <= 4

struct GridPlan {
  int ns, nt, de, K, bs, bt;  // bs / bt: chunks of the source / target set
  int rows;                    // rows per chunk (the same for both sets)
  __device__ void chunk(int b, int& r0, int& r1, bool& is_s) const {
    is_s = b < bs;
    const int lb = is_s ? b : b - bs;
    const int base = is_s ? 0 : ns, cnt = is_s ? ns : nt;
    r0 = base + lb * rows;
    r1 = base + min(cnt, (lb + 1) * rows);
  }
};

// rows per chunk: about one wave of 4 blocks per SM over both sets (a second,
// nearly empty wave doubled pass AC's time), a multiple of 64 rows, at least
// kChunk; a function of ns + nt only, so identical sets chunk identically
__host__ __device__ inline int grid_chunk_rows(int64_t ns, int64_t nt) {
  const int64_t want = (ns + nt + 4 * kNumSMs - 1) / (4 * kNumSMs);
  const int64_t r = (want + 63) / 64 * 64;
  return (int)(r < kChunk ? kChunk : r);
}
__host__ __device__ inline GridPlan make_grid_plan(int64_t ns, int64_t nt, int de, int k) {
  const int rows = grid_chunk_rows(ns, nt);
  return GridPlan{(int)ns, (int)nt, de, k, (int)((ns + rows - 1) / rows),
                  (int)((nt + rows - 1) / rows), rows};
}

// Fixed-shape block reduction of one set's chunk partials: thread q takes
// the chunks q, q+256, ... of THAT set in order, then warp xor-trees and the
// 8 warp totals in warp order — deterministic, and the same shape for two
// identical sets (cmd(S, S) == 0 exactly).  Result valid in thread 0.
__device__ __forceinline__ double block_set_sum(const double* part, int first, int count,
                                                size_t stride, double* red) {
  double a = 0.0;
  for (int q = threadIdx.x; q < count; q += kGridThreads) a += part[(size_t)(first + q) * stride];
  a = warp_sum_d(a);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kGridThreads / 32; ++w) t += red[w];
  return t;
}

// pass AC (one streaming read of Z): per block and column, min/argmin,
// max/argmax and the power sums S_j = Σ (z − c0)^j, j = 1..K, around the
// shift c0 = the column's value in the set's first row (the central sums
// follow in the combine by the binomial expansion around the mean; with c0
// one sample of the set, |c0 − μ| is a few standard deviations and the
// expansion loses < 1e-13 relative on these moments).  Partial layout per
// block: [mn | imn | mx | imx | S_1 .. S_K] × de.
template <typename T, int KC>
__global__ void __launch_bounds__(kGridThreads) cmd_pass_ac(const T* __restrict__ Z, GridPlan g,
                                                            double* __restrict__ part,
                                                            unsigned* __restrict__ done) {
  // KC: the CMD order as a compile-time bound (0: runtime g.K ≤ kMaxCmdOrder)
  constexpr int KB = KC > 0 ? KC : kMaxCmdOrder;
  if (blockIdx.x == 0 && threadIdx.x == 0) *done = 0;  // combine's block counter
  __shared__ double s_mn[8][32], s_mx[8][32];
  __shared__ int s_imn[8][32], s_imx[8][32];
  __shared__ double s_p[8][kMaxCmdOrder][32];
  int r0, r1;
  bool is_s;
  g.chunk(blockIdx.x, r0, r1, is_s);
  const int row_first = is_s ? 0 : g.ns;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c0 = 0; c0 < g.de; c0 += 32) {
    const int c = c0 + lane;
    double mn = INFINITY, mx = -INFINITY;
    int imn = 0x7fffffff, imx = 0x7fffffff;
    double ps[kMaxCmdOrder];
#pragma unroll
    for (int j = 0; j < kMaxCmdOrder; ++j) ps[j] = 0.0;
    if (c < g.de) {
      const double sh = (double)Z[(size_t)row_first * g.de + c];
      int r = r0 + w;
      for (; r + 56 < r1; r += 64) {  // 8 rows in flight per thread
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (double)Z[(size_t)(r + 8 * u) * g.de + c];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // a thread's rows increase, so strict compares keep the first index
          if (v[u] < mn) { mn = v[u]; imn = r + 8 * u; }
          if (v[u] > mx) { mx = v[u]; imx = r + 8 * u; }
          const double cen = v[u] - sh;
          double pw = cen;
#pragma unroll
          for (int j = 0; j < KB; ++j)
            if (KC > 0 || j < g.K) { ps[j] += pw; pw *= cen; }
        }
      }
      for (; r < r1; r += 8) {
        const double v = (double)Z[(size_t)r * g.de + c];
        argmin_merge(mn, imn, v, r);
        argmax_merge(mx, imx, v, r);
        const double cen = v - sh;
        double pw = cen;
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (KC > 0 || j < g.K) { ps[j] += pw; pw *= cen; }
      }
    }
    s_mn[w][lane] = mn; s_imn[w][lane] = imn;
    s_mx[w][lane] = mx; s_imx[w][lane] = imx;
#pragma unroll
    for (int j = 0; j < kMaxCmdOrder; ++j) s_p[w][j][lane] = ps[j];
    __syncthreads();
    for (int e = threadIdx.x; e < (4 + g.K) * 32; e += kGridThreads) {
      const int q = e >> 5, l = e & 31, cc = c0 + l;
      if (cc >= g.de) continue;
      double* o = part + ((size_t)blockIdx.x * (4 + g.K) + q) * g.de + cc;
      if (q == 0 || q == 1) {
        double m = s_mn[0][l];
        int im = s_imn[0][l];
        for (int k = 1; k < 8; ++k) argmin_merge(m, im, s_mn[k][l], s_imn[k][l]);
        *o = q == 0 ? m : (double)im;
      } else if (q == 2 || q == 3) {
        double m = s_mx[0][l];
        int im = s_imx[0][l];
        for (int k = 1; k < 8; ++k) argmax_merge(m, im, s_mx[k][l], s_imx[k][l]);
        *o = q == 2 ? m : (double)im;
      } else {
        const int j = q - 4;
        double a = s_p[0][j][l];
        for (int k = 1; k < 8; ++k) a += s_p[k][j][l];
        *o = a;
      }
    }
    __syncthreads();
  }
}

// combine AC: one block per column — extrema over all chunks; per set the
// power sums S_j in fixed chunk order, the mean μ = c0 + S_1/n and the
// central moments m_j = (1/n) Σ_i C(j,i) S_i (c0 − μ)^(j−i) (S_0 = n)
// pass E's per-(set, column) coefficients (cmd_grad_elem's factors, formed in
// its operation order): [set][mu | g1 | (w_j, mean(cen^(j-1))) j = 2..K][de]
__device__ void build_e_coef(const GridPlan& g, const double* cs, double* coef,
                             const double* spow) {
  const int de = g.de, K = g.K, KM = kMaxCmdOrder + 1;
  const int per_set = (2 + 2 * (K - 1)) * de;
  const double* mus = cs + 2 * de;
  const double* mut = cs + 3 * de;
  const double* sv = cs + 4 * de;
  const double* u = cs + 5 * de;
  const double* ms = cs + 9 * de;
  const double* mt = ms + KM * de;
  const double* norms = mt + KM * de;
  for (int e = threadIdx.x; e < 2 * de; e += blockDim.x) {
    const int set = e / de, c = e - set * de;
    const bool is_s = set == 0;
    const double cnt = is_s ? (double)g.ns : (double)g.nt;
    const double sign = is_s ? 1.0 : -1.0;
    const double sc = fabs(sv[c]);
    const double* mm = is_s ? ms : mt;
    double* o = coef + set * per_set;
    o[c] = is_s ? mus[c] : mut[c];
    o[de + c] = norms[1] > 0.0 ? sign * (u[c] / norms[1]) / (sc * cnt) : 0.0;
    for (int j = 2; j <= K; ++j) {
      double w = 0.0;
      if (norms[j] > 0.0) {
        const double sj = spow[j * de + c];
        const double v = (ms[j * de + c] - mt[j * de + c]) / sj;
        w = sign * ((double)j / cnt) * (v / norms[j]) / sj;
      }
      o[(2 * (j - 1)) * de + c] = w;
      o[(2 * (j - 1) + 1) * de + c] = mm[(j - 1) * de + c];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kGridThreads) cmd_combine_ac(const T* __restrict__ Z, GridPlan g,
                                                               const double* __restrict__ part,
                                                               double* __restrict__ cs,
                                                               unsigned* __restrict__ done,
                                                               double* __restrict__ value,
                                                               double* __restrict__ ecoef) {
  __shared__ double red[kGridThreads / 32], rmn[kGridThreads / 32], rmx[kGridThreads / 32];
  __shared__ int rimn[kGridThreads / 32], rimx[kGridThreads / 32];
  __shared__ double S[2][kMaxCmdOrder + 1];
  const int de = g.de, c = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = g.bs + g.bt, KM = kMaxCmdOrder + 1;
  double mn = INFINITY, mx = -INFINITY;
  int imn = 0x7fffffff, imx = 0x7fffffff;
  auto fld = [&](int f, int b) { return part[((size_t)b * (4 + g.K) + f) * de + c]; };
#pragma unroll 4
  for (int b = threadIdx.x; b < nb; b += kGridThreads) {
    argmin_merge(mn, imn, fld(0, b), (int)fld(1, b));
    argmax_merge(mx, imx, fld(2, b), (int)fld(3, b));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, mn, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, imn, o);
    argmin_merge(mn, imn, v2, i2);
    const double v3 = __shfl_xor_sync(0xffffffffu, mx, o);
    const int i3 = __shfl_xor_sync(0xffffffffu, imx, o);
    argmax_merge(mx, imx, v3, i3);
  }
  if (lane == 0) { rmn[w] = mn; rimn[w] = imn; rmx[w] = mx; rimx[w] = imx; }
  {  // every S_j of both sets in one pass over the partials: thread q takes
     // the chunks q, q+256, … of each set in order, then warp xor-trees and the
     // 8 warp totals in warp order (fixed shape, identical for identical sets)
    __shared__ double rs[kGridThreads / 32][2][kMaxCmdOrder];
    double a[2][kMaxCmdOrder];
#pragma unroll
    for (int j = 0; j < kMaxCmdOrder; ++j) a[0][j] = a[1][j] = 0.0;
    for (int set = 0; set < 2; ++set) {
      const int first = set == 0 ? 0 : g.bs, count = set == 0 ? g.bs : g.bt;
#pragma unroll 4
      for (int q = threadIdx.x; q < count; q += kGridThreads) {
#pragma unroll
        for (int j = 0; j < kMaxCmdOrder; ++j)
          if (j < g.K) a[set][j] += fld(4 + j, first + q);
      }
    }
#pragma unroll
    for (int set = 0; set < 2; ++set)
#pragma unroll
      for (int j = 0; j < kMaxCmdOrder; ++j) {
        const double v = warp_sum_d(a[set][j]);
        if (lane == 0) rs[w][set][j] = v;
      }
    __syncthreads();
    if (threadIdx.x < 2 * kMaxCmdOrder) {
      const int set = threadIdx.x / kMaxCmdOrder, j = threadIdx.x % kMaxCmdOrder;
      double t = 0.0;
      for (int q = 0; q < kGridThreads / 32; ++q) t += rs[q][set][j];
      if (j < g.K) S[set][j + 1] = t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int q = 1; q < kGridThreads / 32; ++q) {
      argmin_merge(mn, imn, rmn[q], rimn[q]);
      argmax_merge(mx, imx, rmx[q], rimx[q]);
    }
    cs[c] = mn;
    cs[de + c] = mx;
    const double raw = mx - mn;
    cs[4 * de + c] = raw < kCmdSupportFloor ? -kCmdSupportFloor : raw;
    cs[7 * de + c] = (double)imn;
    cs[8 * de + c] = (double)imx;
    for (int set = 0; set < 2; ++set) {
      const double n = set == 0 ? (double)g.ns : (double)g.nt;
      const double sh = (double)Z[(size_t)(set == 0 ? 0 : g.ns) * de + c];
      const double mu = sh + S[set][1] / n;
      const double d = sh - mu;
      cs[(2 + set) * de + c] = mu;
      double* mom = cs + 9 * de + set * KM * de;
      S[set][0] = n;
      for (int j = 1; j <= g.K; ++j) {
        // Σ_i C(j,i) S_i d^(j-i), highest power of d first
        double acc = 0.0, binom = 1.0, dp = 1.0;
        for (int i = j; i >= 0; --i) {
          acc += binom * S[set][i] * dp;
          dp *= d;
          binom = binom * (double)i / (double)(j - i + 1);
        }
        mom[j * de + c] = acc / n;
      }
    }
  }
  // the last column block: finish (norms, support gradient, value) and the
  // pass-E coefficient table, in shared memory (was two more launches)
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  extern __shared__ double cs_s[];  // [scratch | pow(|s_c|, j) table]
  const int n_cs = cmd_scratch_doubles(de);
  double* spow = cs_s + n_cs;
  for (int e = threadIdx.x; e < n_cs; e += blockDim.x) cs_s[e] = __ldcg(cs + e);
  __syncthreads();
  for (int e = threadIdx.x; e < (g.K - 1) * de; e += blockDim.x) {  // all pow() at once
    const int j = 2 + e / de, c = e % de;
    spow[j * de + c] = pow(fabs(cs_s[4 * de + c]), (double)j);
  }
  __syncthreads();
  const double v = cmd_finish(cs_s, de, g.K, 0, blockDim.x, spow);
  if (threadIdx.x == 0) *value = v;
  for (int e = threadIdx.x; e < n_cs; e += blockDim.x) cs[e] = cs_s[e];
  if (ecoef) build_e_coef(g, cs_s, ecoef, spow);
}


// pass E: gradient of every element (coalesced).  The per-column factors of
// cmd_grad_elem (costmodel.py:446-475) are formed once per block in the same
// operation order, so each element costs K-1 FMAs instead of K pow() calls.
template <typename T>
__global__ void __launch_bounds__(kGridThreads) cmd_pass_e(const T* __restrict__ Z, GridPlan g,
                                                           const double* __restrict__ cs,
                                                           double* __restrict__ grad) {
  // per set: mu, c0, then per order j = 2..K: w_j, mean(cen^(j-1))
  extern __shared__ double coef[];
  const int de = g.de, K = g.K, KM = kMaxCmdOrder + 1;
  const int per_set = (2 + 2 * (K - 1)) * de;
  const double* mus = cs + 2 * de;
  const double* mut = cs + 3 * de;
  const double* s = cs + 4 * de;
  const double* u = cs + 5 * de;
  const double* ds = cs + 6 * de;
  const double* amin = cs + 7 * de;
  const double* amax = cs + 8 * de;
  const double* ms = cs + 9 * de;
  const double* mt = ms + KM * de;
  const double* norms = mt + KM * de;
  for (int e = threadIdx.x; e < 2 * de; e += blockDim.x) {
    const int set = e / de, c = e - set * de;
    const bool is_s = set == 0;
    const double cnt = is_s ? (double)g.ns : (double)g.nt;
    const double sign = is_s ? 1.0 : -1.0;
    const double sc = fabs(s[c]);
    const double* mm = is_s ? ms : mt;
    double* o = coef + set * per_set;
    o[c] = is_s ? mus[c] : mut[c];
    o[de + c] = norms[1] > 0.0 ? sign * (u[c] / norms[1]) / (sc * cnt) : 0.0;
    for (int j = 2; j <= K; ++j) {
      double w = 0.0;
      if (norms[j] > 0.0) {
        const double sj = pow(sc, (double)j);
        const double v = (ms[j * de + c] - mt[j * de + c]) / sj;
        w = sign * ((double)j / cnt) * (v / norms[j]) / sj;
      }
      o[(2 * (j - 1)) * de + c] = w;
      o[(2 * (j - 1) + 1) * de + c] = mm[(j - 1) * de + c];
    }
  }
  __syncthreads();
  const int total = (g.ns + g.nt) * de;  // < 2^31 (checked at launch)
  const bool de32 = de == 32;
  const int stride = gridDim.x * blockDim.x;
  constexpr int U = 8;  // elements in flight per thread
  for (int e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += U * stride) {
    double z[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * stride;
      z[u] = e < total ? (double)Z[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * stride;
      if (e >= total) break;
      const int row = de32 ? e >> 5 : e / de, c = de32 ? e & 31 : e - row * de;
      const double* o = coef + (row < g.ns ? 0 : per_set);
      const double cen = z[u] - o[c];
      double gv = o[de + c];
      double pw = 1.0;
      for (int j = 2; j <= K; ++j) {
        pw *= cen;
        gv += o[(2 * (j - 1)) * de + c] * (pw - o[(2 * (j - 1) + 1) * de + c]);
      }
      if ((double)row == amax[c]) gv += ds[c];
      if ((double)row == amin[c]) gv -= ds[c];
      grad[e] = gv;
    }
  }
}

// pass E for de = 32 (lane = column): the column's coefficients (both sets),
// argmin / argmax rows and support gradient live in registers — per element
// K-1 multiply-adds and no shared-memory reads; a warp walks whole rows
// (coalesced), 8 rows in flight per thread.  Same operations, same order as
// cmd_pass_e.
template <typename T, int K>
__global__ void __launch_bounds__(kGridThreads) cmd_pass_e32(const T* __restrict__ Z, GridPlan g,
                                                             const double* __restrict__ cs,
                                                             const double* __restrict__ ecoef,
                                                             double* __restrict__ grad) {
  constexpr int de = 32;
  constexpr int per_set = (2 + 2 * (K - 1)) * de;
  const int c = threadIdx.x & 31;
  double mu[2], g1[2], wj[2][K > 1 ? K - 1 : 1], mj[2][K > 1 ? K - 1 : 1];
#pragma unroll
  for (int set = 0; set < 2; ++set) {
    const double* o = ecoef + set * per_set;
    mu[set] = o[c];
    g1[set] = o[de + c];
#pragma unroll
    for (int j = 2; j <= K; ++j) {
      wj[set][j - 2] = o[(2 * (j - 1)) * de + c];
      mj[set][j - 2] = o[(2 * (j - 1) + 1) * de + c];
    }
  }
  const int rmax = (int)cs[8 * de + c], rmin = (int)cs[7 * de + c];
  const double dsc = cs[6 * de + c];
  const int rows = g.ns + g.nt;
  const int warps = gridDim.x * (blockDim.x >> 5);
  constexpr int U = 8;
  auto elem = [&](auto set_c, double z, int r) {  // set_c: compile-time set index
    constexpr int set = decltype(set_c)::value;
    const double cen = z - mu[set];
    double gv = g1[set];
    double pw = 1.0;
#pragma unroll
    for (int j = 2; j <= K; ++j) {
      pw *= cen;
      gv += wj[set][j - 2] * (pw - mj[set][j - 2]);
    }
    if (r == rmax) gv += dsc;
    if (r == rmin) gv -= dsc;
    grad[(size_t)r * de + c] = gv;
  };
  for (int r0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r0 < rows; r0 += U * warps) {
    double z[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int r = r0 + k * warps;
      z[k] = r < rows ? (double)Z[(size_t)r * de + c] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int r = r0 + k * warps;
      if (r >= rows) break;
      if (r < g.ns)  // warp-uniform (a warp walks one row)
        elem(std::integral_constant<int, 0>{}, z[k], r);
      else
        elem(std::integral_constant<int, 1>{}, z[k], r);
    }
  }
}

template <typename T, int K>
void launch_pass_e32(const T* Z, const GridPlan& g, const double* cs, const double* ecoef,
                     double* grad, cudaStream_t st) {
  cmd_pass_e32<T, K><<<kNumSMs * 3, kGridThreads, 0, st>>>(Z, g, cs, ecoef, grad);
}

template <typename T>
int launch_cmd_grid(const T* Z, const GridPlan& g, double* value, double* grad, double* ws,
                    cudaStream_t st) {
  const int blocks = g.bs + g.bt;
  const size_t n_cs = cmd_scratch_doubles(g.de);
  double* cs = ws;
  double* part = ws + n_cs;
  // after the partials: pass E's coefficient table, then the block counter
  double* ecoef = part + (size_t)blocks * (4 + g.K) * g.de;
  unsigned* done = reinterpret_cast<unsigned*>(ecoef + (size_t)2 * (2 + 2 * (g.K - 1)) * g.de);
  const size_t smem = (n_cs + (size_t)(kMaxCmdOrder + 1) * g.de) * sizeof(double);
  switch (g.K) {  // the order as a compile-time bound for the common values
    case 3: cmd_pass_ac<T, 3><<<blocks, kGridThreads, 0, st>>>(Z, g, part, done); break;
    case 4: cmd_pass_ac<T, 4><<<blocks, kGridThreads, 0, st>>>(Z, g, part, done); break;
    case 5: cmd_pass_ac<T, 5><<<blocks, kGridThreads, 0, st>>>(Z, g, part, done); break;
    default: cmd_pass_ac<T, 0><<<blocks, kGridThreads, 0, st>>>(Z, g, part, done); break;
  }
  TPCB_CUDA_CHECK(cudaFuncSetAttribute(cmd_combine_ac<T>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const bool e32 = grad && g.de == 32 && g.K >= 1 && g.K <= 8;
  cmd_combine_ac<T><<<g.de, kGridThreads, smem, st>>>(Z, g, part, cs, done, value,
                                                       e32 ? ecoef : nullptr);
  if (grad) {
    if (e32) {
      switch (g.K) {
        case 1: launch_pass_e32<T, 1>(Z, g, cs, ecoef, grad, st); break;
        case 2: launch_pass_e32<T, 2>(Z, g, cs, ecoef, grad, st); break;
        case 3: launch_pass_e32<T, 3>(Z, g, cs, ecoef, grad, st); break;
        case 4: launch_pass_e32<T, 4>(Z, g, cs, ecoef, grad, st); break;
        case 5: launch_pass_e32<T, 5>(Z, g, cs, ecoef, grad, st); break;
        case 6: launch_pass_e32<T, 6>(Z, g, cs, ecoef, grad, st); break;
        case 7: launch_pass_e32<T, 7>(Z, g, cs, ecoef, grad, st); break;
        default: launch_pass_e32<T, 8>(Z, g, cs, ecoef, grad, st); break;
      }
    } else {
      const size_t esmem = (size_t)2 * (2 + 2 * (g.K - 1)) * g.de * sizeof(double);
      TPCB_CUDA_CHECK(cudaFuncSetAttribute(cmd_pass_e<T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)esmem));
      cmd_pass_e<T><<<kNumSMs * 8, kGridThreads, esmem, st>>>(Z, g, cs, grad);
    }
  }
  TPCB_LAUNCH_CHECK("cmd_grid");
  return TPCB_OK;
}

}  // namespace
}  // namespace tpcb

using namespace tpcb;

extern "C" size_t tpcb_cmd_grid_ws(int64_t ns, int64_t nt, int32_t de, int32_t k) {
  if (ns < 1 || nt < 1 || de < 1 || k < 1) return 0;
  const GridPlan g = make_grid_plan(ns, nt, de, k);
  const int64_t blocks = (int64_t)g.bs + g.bt;
  const int64_t per = 4 + k;
  return (size_t)(cmd_scratch_doubles(de) + blocks * per * de + 2 * (2 + 2 * (k - 1)) * de + 2) *
         sizeof(double);
}

extern "C" int tpcb_cmd_grid(const void* d_z, int32_t z_is_f64, int64_t ns, int64_t nt,
                             int32_t de, int32_t k, double* d_value, double* d_grad, void* d_ws,
                             size_t ws_bytes, void* stream) {
  if (!d_z || !d_value || !d_ws) return TPCB_ERR_VALIDATION;
  if (ns < 1 || nt < 1) return TPCB_ERR_EMPTY_SET;
  if (de < 1 || k < 1) return TPCB_ERR_VALIDATION;
  if (k > kMaxCmdOrder || de > kMaxGridDe) return TPCB_ERR_UNSUPPORTED;
  if ((ns + nt) * de > 0x7fffffff) return TPCB_ERR_UNSUPPORTED;
  if (ws_bytes < tpcb_cmd_grid_ws(ns, nt, de, k)) return TPCB_ERR_VALIDATION;
  const GridPlan g = make_grid_plan(ns, nt, de, k);
  cudaStream_t st = (cudaStream_t)stream;
  double* ws = static_cast<double*>(d_ws);
  return z_is_f64 ? launch_cmd_grid(static_cast<const double*>(d_z), g, d_value, d_grad, ws, st)
                  : launch_cmd_grid(static_cast<const float*>(d_z), g, d_value, d_grad, ws, st);
}

extern "C" int tpcb_cmd(const void* d_z, int32_t z_is_f64, int64_t ns, int64_t nt, int32_t de,
                        int32_t k, double* d_value, double* d_grad, void* stream) {
  if (!d_z || !d_value) return TPCB_ERR_VALIDATION;
  if (ns < 1 || nt < 1) return TPCB_ERR_EMPTY_SET;
  if (de < 1 || k < 1) return TPCB_ERR_VALIDATION;
  if (k > kMaxCmdOrder) return TPCB_ERR_UNSUPPORTED;
  if (ns + nt > 0x7fffffff) return TPCB_ERR_UNSUPPORTED;
  const size_t smem = (size_t)cmd_scratch_doubles(de) * sizeof(double);
  if (smem > 200 * 1024) return TPCB_ERR_UNSUPPORTED;
  if (z_is_f64) {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(cmd_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cmd_kernel<double><<<1, 1024, smem, (cudaStream_t)stream>>>(
        static_cast<const double*>(d_z), (int)ns, (int)nt, de, k, d_value, d_grad);
  } else {
    TPCB_CUDA_CHECK(cudaFuncSetAttribute(cmd_kernel<float>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cmd_kernel<float><<<1, 1024, smem, (cudaStream_t)stream>>>(
        static_cast<const float*>(d_z), (int)ns, (int)nt, de, k, d_value, d_grad);
  }
  TPCB_LAUNCH_CHECK("cmd_kernel");
  return TPCB_OK;
}
