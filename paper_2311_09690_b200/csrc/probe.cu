// Measurement helpers for bench.py: the FP32 FFMA peak of this GPU (the
// denominator of the fp32 parity kernels' roofline; MEASURED_PEAKS.json only
// records HBM and bf16 tensor peaks) and an L2 flush.
#include "common.cuh"

namespace tpcb {
namespace {

// 8 independent FMA chains per thread, 4096 iterations: pure FFMA issue.
__global__ void __launch_bounds__(256) ffma_kernel(float* out, float seed, int iters) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.f) out[blockIdx.x] = s;  // keep the chains alive
}

__global__ void flush_kernel(float4* buf, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_float4(v, v, v, v);
}

}  // namespace
}  // namespace tpcb

using namespace tpcb;

extern "C" int tpcb_probe_ffma(float* d_scratch, double* tflops_out, void* stream_) {
  if (!d_scratch || !tflops_out) return TPCB_ERR_VALIDATION;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int blocks = kNumSMs * 8, iters = 4096;
  cudaEvent_t e0, e1;
  TPCB_CUDA_CHECK(cudaEventCreate(&e0));
  TPCB_CUDA_CHECK(cudaEventCreate(&e1));
  ffma_kernel<<<blocks, 256, 0, stream>>>(d_scratch, 1.f, iters);  // warm-up
  TPCB_CUDA_CHECK(cudaEventRecord(e0, stream));
  ffma_kernel<<<blocks, 256, 0, stream>>>(d_scratch, 1.f, iters);
  TPCB_CUDA_CHECK(cudaEventRecord(e1, stream));
  TPCB_CUDA_CHECK(cudaEventSynchronize(e1));
  float ms = 0.f;
  TPCB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8 * 16 * (double)iters * 256.0 * blocks;
  *tflops_out = flops / (ms * 1e-3) / 1e12;
  return TPCB_OK;
}

extern "C" int tpcb_flush_l2(void* d_buf, size_t bytes, void* stream) {
  if (!d_buf) return TPCB_ERR_VALIDATION;
  flush_kernel<<<kNumSMs * 4, 256, 0, (cudaStream_t)stream>>>(static_cast<float4*>(d_buf),
                                                              bytes / 16, 0.f);
  TPCB_LAUNCH_CHECK("flush_kernel");
  return TPCB_OK;
}
