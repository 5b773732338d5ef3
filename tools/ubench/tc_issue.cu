// Microbenchmark: single-thread tcgen05 issue costs on sm_100a (profiling aid,
// not product code).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2312_16733_b200/csrc tools/ubench/tc_issue.cu -o tools/ubench/tc_issue
#include <cstdio>
#include "device.cuh"
using namespace ssn;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// warp_wide: 0 = lane 0 runs the loop (divergent), 1 = whole warp runs it and
// elect.sync picks the issuing lane
__global__ void k(int mode, int n_mma, int N, int warp_wide, long long* out) {
  __shared__ __align__(1024) uint8_t sbuf[40 * 1024];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int ITER = 1000;
  const uint32_t idesc = umma_idesc_bf16(N);
  const uint64_t ad = umma_desc_sw128(smem_u32(sbuf));
  const uint64_t bd = umma_desc_sw128(smem_u32(sbuf + 16384));
  if (warp == 0 && (warp_wide || lane == 0)) {
    long long t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
      if (warp_wide) {
        if (elect_one()) {
          for (int q = 0; q < n_mma; ++q) tc_mma_bf16(tmem, ad + 2 * q, bd + 2 * q, idesc, 1);
          if (mode >= 1) tc_commit(&bar[i & 1]);
        }
        __syncwarp();
      } else {
        for (int q = 0; q < n_mma; ++q) tc_mma_bf16(tmem, ad + 2 * q, bd + 2 * q, idesc, 1);
        if (mode >= 1) tc_commit(&bar[i & 1]);
      }
      if (mode == 2) mbar_wait(&bar[i & 1], (i >> 1) & 1);
    }
    long long t1 = clock64();
    if (mode == 1) mbar_wait(&bar[(ITER - 1) & 1], ((ITER - 1) >> 1) & 1);
    long long t2 = clock64();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  struct { int mode, n, N; const char* what; } cases[] = {
      {1, 0, 64, "commit only"},
      {0, 4, 96, "4 mma N=96, no commit"},
      {0, 4, 128, "4 mma N=128, no commit"},
      {0, 4, 192, "4 mma N=192, no commit"},
      {1, 4, 96, "4 mma N=96 + commit"},
      {1, 8, 96, "8 mma N=96 + commit"},
      {1, 4, 192, "4 mma N=192 + commit"},
      {2, 0, 64, "commit + wait"},
      {2, 4, 96, "4 mma N=96 + commit + wait"},
      {2, 4, 192, "4 mma N=192 + commit + wait"},
  };
  for (int ww = 0; ww < 2; ++ww)
    for (auto& c : cases) {
      for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 128>>>(c.mode, c.n, c.N, ww, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s %-30s issue %7.1f cyc/iter   complete %7.1f cyc/iter\n", ww ? "warp " : "lane0",
             c.what, h[0] / 1000.0, h[1] / 1000.0);
    }
  return 0;
}
