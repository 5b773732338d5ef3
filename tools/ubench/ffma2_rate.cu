// Microbenchmark (profiling aid, not product code): FP32 FMA throughput of
// scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on sm_100a, 148 x 1024 threads,
// 8 independent chains per thread.  Prints GFLOP/s of each.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_rate.cu -o ffma2_rate
#include <cstdio>
#include <cstdint>

__global__ void k1(float* out, float s, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s, 0.5f);
  float r = 0;
  for (int j = 0; j < 8; ++j) r += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__device__ __forceinline__ uint64_t f2(float x, float y) {
  return (static_cast<uint64_t>(__float_as_uint(y)) << 32) | __float_as_uint(x);
}

__global__ void k2(float* out, float s, int iters) {
  uint64_t a[4];
  for (int j = 0; j < 4; ++j) a[j] = f2(threadIdx.x * 0.001f + 2 * j, threadIdx.x * 0.001f + 2 * j + 1);
  const uint64_t ss = f2(s, s), hh = f2(0.5f, 0.5f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int j = 0; j < 4; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(ss), "l"(hh));
  float r = 0;
  for (int j = 0; j < 4; ++j) r += __uint_as_float(static_cast<uint32_t>(a[j])) + __uint_as_float(static_cast<uint32_t>(a[j] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 1024 * 4 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int v = 0; v < 2; ++v) {
      cudaEventRecord(e0);
      if (v == 0) k1<<<148 * 4, 1024>>>(d, 0.999f, iters);
      else k2<<<148 * 4, 1024>>>(d, 0.999f, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 8 * iters * 148.0 * 4 * 1024;
      printf("%s: %.1f ms  %.1f TFLOP/s\n", v == 0 ? "FFMA " : "FFMA2", ms, flops / ms / 1e9);
    }
  }
  return 0;
}
