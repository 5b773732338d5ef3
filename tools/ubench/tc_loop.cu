// Microbenchmark: the producer -> MMA -> commit ring handshake of conv_tc with
// no data movement, to cost each piece of the per-K-block loop (profiling aid).
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

#ifndef ST_N
#define ST_N 4
#endif
constexpr int ST = ST_N;

__device__ __forceinline__ void mbar_wait_test(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// V bit0: skip fence_after; bit1: whole MMA warp runs loop (elect issue); bit2: no MMA
template <int V>
__global__ void k(int N, int iters, long long* out) {
  __shared__ __align__(1024) uint8_t sbuf[40 * 1024];
  __shared__ uint64_t full[ST], empty[ST];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && lane == 0) {  // producer
    for (int g = 0; g < iters; ++g) {
      const int s = g % ST;
      mbar_wait(&empty[s], ((g / ST) & 1) ^ 1);
      mbar_arrive(&full[s]);
    }
  } else if (warp == 0 && ((V & 2) || lane == 0)) {
    const uint32_t idesc = umma_idesc_bf16(N);
    const uint32_t a0 = smem_u32(sbuf), b0 = smem_u32(sbuf + 16384);
    long long t0 = clock64();
    for (int g = 0; g < iters; ++g) {
      const int s = g % ST;
      if (V & 8) mbar_wait_test(&full[s], (g / ST) & 1); else mbar_wait(&full[s], (g / ST) & 1);
      if (!(V & 1)) tc_fence_after();
      const uint64_t ad = umma_desc_sw128(a0 + (s & 1) * 4096);
      const uint64_t bd = umma_desc_sw128(b0 + (s & 1) * 4096);
      if (!(V & 2) || elect_one()) {
        if (!(V & 4)) {
#pragma unroll
          for (int kk = 0; kk < ((V & 16) ? 8 : 4); ++kk)
            tc_mma_bf16(tmem, ad + 2 * (kk & 3), bd + 2 * (kk & 3), idesc, 1);
        }
        tc_commit(&empty[s]);
      }
      if (V & 2) __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <int V>
void run(int N, const char* what) {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[1];
  const int iters = 2000;
  for (int rep = 0; rep < 3; ++rep) k<V><<<1, 128>>>(N, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("V=%d N=%3d %-40s %7.1f cyc per k-block\n", V, N, what, h[0] / double(iters));
  cudaFree(d);
}

int main() {
  for (int N : {64, 96, 128, 192}) {
    run<0>(N, "lane0, fence, 4 mma");
    run<1>(N, "lane0, no fence, 4 mma");
    run<2>(N, "warp+elect, fence, 4 mma");
    run<3>(N, "warp+elect, no fence, 4 mma");
    run<4>(N, "lane0, fence, no mma");
    run<6>(N, "warp+elect, fence, no mma");
    run<10>(N, "warp+elect, test_wait, 4 mma");
    run<18>(N, "warp+elect, fence, 8 mma");
    run<16>(N, "lane0, fence, 8 mma");
    run<14>(N, "warp+elect, test_wait, no mma");
    run<8>(N, "lane0, test_wait, 4 mma");
  }
  return 0;
}
