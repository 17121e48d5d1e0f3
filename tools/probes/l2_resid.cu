// L2 residency probe: kernel W writes `mb` MB (float4 stores), kernel R reads
// it back; run under ncu to read dram__bytes_read of R.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_resid l2_resid.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void writer(float4* p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(v, v + 1, v + 2, v + 3);
}
__global__ void reader(const float4* p, size_t n, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 x = p[i];
    s += x.x + x.y + x.z + x.w;
  }
  if (s == 12345.f) out[0] = s;
}
// strided slots like the training workspace: 64 slots of `stride` floats, first `used` floats written
__global__ void slot_writer(float* p, size_t stride, size_t used, int slots, float v) {
  const size_t n4 = used / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4 * slots; i += (size_t)gridDim.x * blockDim.x) {
    const size_t s = i / n4, k = i % n4;
    reinterpret_cast<float4*>(p + s * stride)[k] = make_float4(v, v, v, v);
  }
}
__global__ void slot_reader(const float* p, size_t stride, size_t used, int slots, float* out) {
  const size_t n4 = used / 4;
  float acc = 0.f;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n4; k += (size_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < slots; ++s) {
      float4 x = reinterpret_cast<const float4*>(p + s * stride)[k];
      acc += x.x;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  float* buf;
  float* flush;
  float* out;
  cudaMalloc(&buf, (size_t)1 << 30);
  cudaMalloc(&flush, (size_t)512 << 20);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed_read = [&](size_t n) {
    cudaEventRecord(e0);
    reader<<<148 * 8, 256>>>((const float4*)buf, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.f;
  };
  for (int mb : {8, 24, 48, 96}) {
    size_t n = (size_t)mb << 20 >> 4;
    for (int rep = 0; rep < 3; ++rep) {
      writer<<<148 * 8, 256>>>((float4*)buf, n, 1.f);
      float hot = timed_read(n);
      writer<<<148 * 8, 256>>>((float4*)buf, n, 1.f);
      writer<<<148 * 8, 256>>>((float4*)flush, (size_t)512 << 20 >> 4, 2.f);
      float cold = timed_read(n);
      float hot2 = timed_read(n);
      if (rep == 2)
        printf("%3d MB: read after write %.1f us (%.0f GB/s) | after flush %.1f us (%.0f GB/s) | re-read %.1f us\n",
               mb, hot, mb * 1.048576e3 / hot, cold, mb * 1.048576e3 / cold, hot2);
    }
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
