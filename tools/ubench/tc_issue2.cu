// Microbenchmark: per-MMA vs per-iteration cost of single-thread tcgen05.mma
// issue (profiling aid, not product code).
#include <cstdio>
#include "device.cuh"
using namespace ssn;

template <int NM, int COMMIT>
__global__ void k(int N, long long* out) {
  __shared__ __align__(1024) uint8_t sbuf[47 * 1024];
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
  const int ITER = 200;
  const uint32_t idesc = umma_idesc_bf16(N);
  const uint64_t ad = umma_desc_sw128(smem_u32(sbuf));
  const uint64_t bd = umma_desc_sw128(smem_u32(sbuf + 16384));
  if (warp == 0 && lane == 0) {
    long long t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
      for (int q = 0; q < NM; ++q) tc_mma_bf16(tmem, ad + 2 * (q & 3), bd + 2 * (q & 3), idesc, 1);
      if (COMMIT) tc_commit(&bar[i & 1]);
    }
    long long t1 = clock64();
    if (COMMIT) mbar_wait(&bar[(ITER - 1) & 1], ((ITER - 1) >> 1) & 1);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int NM, int C>
void run(int N) {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  for (int rep = 0; rep < 3; ++rep) k<NM, C><<<1, 128>>>(N, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("NM=%2d commit=%d N=%3d  issue %7.1f cyc/iter (%6.1f per mma)  complete %7.1f (%6.1f per mma)\n",
         NM, C, N, h[0] / 200.0, h[0] / 200.0 / NM, h[1] / 200.0, h[1] / 200.0 / NM);
  cudaFree(d);
}

int main() {
  for (int N : {64, 96, 128, 256}) {
    run<1, 0>(N);
    run<4, 0>(N);
    run<16, 0>(N);
    run<4, 1>(N);
    run<16, 1>(N);
  }
  return 0;
}
