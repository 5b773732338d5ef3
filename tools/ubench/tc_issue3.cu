// Microbenchmark: MMA issue cost with runtime-computed descriptors in three
// issue styles (profiling aid, not product code):
//   0: lane 0 only (divergent; compiler wraps each UTCHMMA in an R2UR waterfall)
//   1: warp converged, if (elect_one()) { mma }
//   2: warp converged, elect.sync inside the asm (@p tcgen05.mma)
#include <cstdio>
#include "device.cuh"
using namespace ssn;

__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int STYLE>
__global__ void k(int N, int taps, int wp, long long* out) {
  __shared__ __align__(1024) uint8_t sbuf[40 * 1024];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int ITER = 100;
  const uint32_t idesc = umma_idesc_bf16(N);
  const uint32_t a0 = smem_u32(sbuf), b0 = smem_u32(sbuf + 16384);
  if (warp == 0 && ((STYLE != 0 && STYLE != 4) || lane == 0)) {
    const bool leader = STYLE == 1 ? elect_one() : true;
    long long t0 = clock64();
    if (STYLE == 3 || STYLE == 4) {
      const uint64_t ad0 = umma_desc_noswz(a0, 1024, 128);
      const uint64_t bd0 = umma_desc_noswz(b0, 256, 128);
      for (int it = 0; it < ITER; ++it) {
        const uint64_t ad = ad0 + (it & 1), bd = bd0;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint64_t a = ad + static_cast<uint64_t>(r * wp + c + j * 128);
              const uint64_t b = bd + static_cast<uint64_t>((r * 3 + c) * 64 + j * 32);
              if (STYLE == 3)
                mma_elect(tmem, a, b, idesc, (r | c | j) != 0);
              else if (lane == 0)
                tc_mma_bf16(tmem, a, b, idesc, (r | c | j) != 0);
            }
      }
    } else
    for (int it = 0; it < ITER; ++it)
      for (int r = 0; r < taps; ++r)
        for (int c = 0; c < taps; ++c)
          for (int j = 0; j < 2; ++j) {
            const uint32_t at = a0 + static_cast<uint32_t>(r * wp + c) * 16 + j * 2048;
            const uint32_t bt = b0 + (r * taps + c) * 1024 + j * 512;
            const uint64_t ad = umma_desc_noswz(at, 1024, 128);
            const uint64_t bd = umma_desc_noswz(bt, 256, 128);
            if (STYLE == 2) {
              mma_elect(tmem, ad, bd, idesc, (r | c | j) != 0);
            } else if (STYLE == 0 || leader) {
              tc_mma_bf16(tmem, ad, bd, idesc, (r | c | j) != 0);
            }
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

template <int S>
void run(int N) {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[1];
  for (int rep = 0; rep < 3; ++rep) k<S><<<1, 128>>>(N, 3, 58, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("style=%d N=%3d  %6.1f cyc per mma\n", S, N, h[0] / (100.0 * 18));
  cudaFree(d);
}

int main() {
  for (int N : {48, 64, 96, 128}) {
    run<0>(N);
    run<1>(N);
    run<2>(N);
    run<3>(N);
    run<4>(N);
  }
  return 0;
}
