// CMD (central moment discrepancy) block-level statistics + gradient, fp64.
// Shared by the training step (train.cu) and the standalone CMD entry point.
#pragma once

#include <cmath>

#include "common.cuh"
#include "train.cuh"

namespace tpcb {

// (value, index) reductions keeping the FIRST index among ties
static __device__ __forceinline__ void argmin_merge(double& v, int& i, double v2, int i2) {
  if (v2 < v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}
static __device__ __forceinline__ void argmax_merge(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}


// doubles of block scratch cmd_stats needs for `de` columns
__host__ __device__ constexpr int cmd_scratch_doubles(int de) {
  return de * (9 + 2 * (kMaxCmdOrder + 1)) + (kMaxCmdOrder + 1);
}

// Column statistics of the CMD between rows [0, ns) and [ns, ns+nt) of Z
// (row-major [n, de]) in fp64, written to the block scratch `cs` (layout:
// lo, hi, mus, mut, s, u, ds, amin, amax [de each], ms, mt [(K+1)·de],
// norms [K+1]).  Returns the CMD value (valid in every thread after the
// trailing barrier).  Must be called by the whole block.  costmodel.py:426-476.
// group variant: the first `nthr` threads (nthr/32 warps) participate and
// synchronise on named barrier `bar_id` (0 = whole block, __syncthreads)
__device__ __forceinline__ void cmd_bar(int bar_id, int nthr) {
  if (bar_id == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar_id), "r"(nthr) : "memory");
}

// Second half of the CMD statistics once lo/hi/amin/amax/mus/mut/s and the
// central moments ms/mt are in `cs`: the per-order norms, the support
// gradient and the value (costmodel.py:440-476).  Whole group participates.
// spow (optional): spow[j * de + c] = pow(|s_c|, j) for j = 2..K, precomputed
// in parallel (the same pow calls, so the same values)
static __device__ __noinline__ double cmd_finish(double* cs, int de, int K, int bar_id,
                                                 int nthr, const double* spow = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int KM = kMaxCmdOrder + 1;
  double* mus = cs + 2 * de;
  double* mut = mus + de;
  double* s = mut + de;
  double* u = s + de;
  double* ds = u + de;
  double* ms = cs + 9 * de;
  double* mt = ms + KM * de;
  double* norms = mt + KM * de;
  // norms over columns (warp 0)
  if (w == 0) {
    double acc = 0.0;
    for (int c = lane; c < de; c += 32) {
      const double sc = fabs(s[c]);
      const double uc = (mus[c] - mut[c]) / sc;
      u[c] = uc;
      acc += uc * uc;
    }
    acc = warp_sum_d(acc);
    if (lane == 0) norms[1] = sqrt(acc);
    for (int j = 2; j <= K; ++j) {
      double a2 = 0.0;
      for (int c = lane; c < de; c += 32) {
        const double sc = fabs(s[c]);
        const double v = (ms[j * de + c] - mt[j * de + c]) /
                         (spow ? spow[j * de + c] : pow(sc, (double)j));
        a2 += v * v;
      }
      a2 = warp_sum_d(a2);
      if (lane == 0) norms[j] = sqrt(a2);
    }
  }
  cmd_bar(bar_id, nthr);
  // support gradient per column
  for (int c = threadIdx.x; c < de; c += nthr) {
    const double sc = fabs(s[c]);
    double d = 0.0;
    if (norms[1] > 0.0) d -= (u[c] / norms[1]) * u[c] / sc;
    for (int j = 2; j <= K; ++j) {
      if (norms[j] > 0.0) {
        const double v = (ms[j * de + c] - mt[j * de + c]) /
                         (spow ? spow[j * de + c] : pow(sc, (double)j));
        d -= j * (v / norms[j]) * v / sc;
      }
    }
    ds[c] = (s[c] < 0.0) ? 0.0 : d;
  }
  cmd_bar(bar_id, nthr);
  double value = norms[1];
  for (int j = 2; j <= K; ++j) value += norms[j];
  cmd_bar(bar_id, nthr);
  return value;
}

template <typename T>
static __device__ __noinline__ double cmd_stats(const T* __restrict__ Z, int ns, int nt, int de,
                                                int K, double* cs, int bar_id = 0,
                                                int nthr = 0) {
  if (nthr <= 0) nthr = blockDim.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = nthr >> 5;
  const int n = ns + nt;
  const int KM = kMaxCmdOrder + 1;
  double* lo = cs;
  double* hi = lo + de;
  double* mus = hi + de;
  double* mut = mus + de;
  double* s = mut + de;
  double* u = s + de;
  double* ds = u + de;
  double* amin = ds + de;
  double* amax = amin + de;
  double* ms = amax + de;     // [KM][de]  mean of (z-μs)^j, j = 0..K
  double* mt = ms + KM * de;  // [KM][de]
  double* norms = mt + KM * de;  // [KM]  (norms[1] = |u|, norms[j] = |v_j|)
  for (int c = w; c < de; c += nw) {
    double mn = INFINITY, mx = -INFINITY, ss = 0.0, st = 0.0;
    int imn = 0x7fffffff, imx = 0x7fffffff;
    for (int r = lane; r < n; r += 32) {
      const double v = (double)Z[(size_t)r * de + c];
      argmin_merge(mn, imn, v, r);
      argmax_merge(mx, imx, v, r);
      if (r < ns)
        ss += v;
      else
        st += v;
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
    ss = warp_sum_d(ss);
    st = warp_sum_d(st);
    const double m_s = ss / ns, m_t = st / nt;
    double ps[kMaxCmdOrder + 1], pt[kMaxCmdOrder + 1];
#pragma unroll
    for (int j = 0; j <= kMaxCmdOrder; ++j) ps[j] = pt[j] = 0.0;
    for (int r = lane; r < n; r += 32) {
      const double v = (double)Z[(size_t)r * de + c];
      const bool is_s = r < ns;
      const double cen = v - (is_s ? m_s : m_t);
      double pw = cen;
#pragma unroll
      for (int j = 1; j <= kMaxCmdOrder; ++j) {
        if (j <= K) {
          if (is_s)
            ps[j] += pw;
          else
            pt[j] += pw;
          pw *= cen;
        }
      }
    }
#pragma unroll
    for (int j = 1; j <= kMaxCmdOrder; ++j) {
      if (j <= K) {
        const double a = warp_sum_d(ps[j]), b = warp_sum_d(pt[j]);
        if (lane == 0) {
          ms[j * de + c] = a / ns;
          mt[j * de + c] = b / nt;
        }
      }
    }
    if (lane == 0) {
      lo[c] = mn;
      hi[c] = mx;
      amin[c] = (double)imn;
      amax[c] = (double)imx;
      mus[c] = m_s;
      mut[c] = m_t;
      const double raw = mx - mn;
      s[c] = raw < kCmdSupportFloor ? -kCmdSupportFloor : raw;  // sign marks clamping
    }
  }
  cmd_bar(bar_id, nthr);
  return cmd_finish(cs, de, K, bar_id, nthr);
}

// d CMD / d z[row, c] from the statistics in `cs` (costmodel.py:446-485),
// including the support-width term routed to the first argmax / argmin row.
static __device__ __forceinline__ double cmd_grad_elem(const double* cs, int ns, int nt, int de,
                                                       int K, int row, int c, double zval) {
  const int KM = kMaxCmdOrder + 1;
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
  const bool is_s = row < ns;
  const double cnt = is_s ? (double)ns : (double)nt;
  const double sign = is_s ? 1.0 : -1.0;
  const double sc = fabs(s[c]);
  const double cen = zval - (is_s ? mus[c] : mut[c]);
  const double* mm = is_s ? ms : mt;
  double g = 0.0;
  if (norms[1] > 0.0) g += sign * (u[c] / norms[1]) / (sc * cnt);
  double pw = 1.0;  // cen^(j-1)
  for (int j = 2; j <= K; ++j) {
    pw *= cen;
    if (norms[j] > 0.0) {
      const double sj = pow(sc, (double)j);
      const double v = (ms[j * de + c] - mt[j * de + c]) / sj;
      g += sign * ((double)j / cnt) * (v / norms[j]) / sj * (pw - mm[(j - 1) * de + c]);
    }
  }
  if ((double)row == amax[c]) g += ds[c];
  if ((double)row == amin[c]) g -= ds[c];
  return g;
}

}  // namespace tpcb
