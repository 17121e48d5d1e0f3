// K6 standalone — central moment discrepancy between two sets (fp64).
// Replaces costmodel.cmd / cmd_between (costmodel.py:489-503, 783-788):
// one CTA computes the column statistics of the union (extrema with their
// first index, means, central power sums up to order K) and, optionally, the
// gradient w.r.t. every row (costmodel.py:426-486).  The in-training CMD term
// uses the same device functions (train.cu).
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

}  // namespace
}  // namespace tpcb

using namespace tpcb;

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
