// Microbenchmark (profiling aid, not product code): tcgen05.mma throughput
// for the shared-memory operand layouts the conv kernels use, M = 128, K = 16
// per instruction, 432 back-to-back MMAs then one commit + wait:
//   layout 0: SW128 K-major (conv_tc: 64-channel rows)
//   layout 1: SW64  K-major (conv_halo: 32-channel rows)
//   layout 2: SW128 with the A start shifted by a halo row offset per tap
//   layout 3: SW64  with the A start shifted by a halo row offset per tap
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//      -I../../paper_2312_16733_b200/csrc mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include "device.cuh"
using namespace ssn;

__global__ void k(int N, int layout, long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sbuf = dsm + ((1024u - (smem_u32(dsm) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = umma_idesc_bf16(N);
  const uint32_t a0 = smem_u32(sbuf), b0 = smem_u32(sbuf + 96 * 1024);
  const bool sw64 = layout == 1 || layout == 3;
  const bool shift = layout >= 2;
  const uint64_t ad0 = sw64 ? umma_desc_sw64(a0) : umma_desc_sw128(a0);
  const uint64_t bd0 = sw64 ? umma_desc_sw64(b0) : umma_desc_sw128(b0);
  const uint32_t row16 = sw64 ? 4 : 8;  // one operand row in 16-byte units
  if (warp == 0) {
    long long t0 = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (rep == 1) t0 = clock64();
      for (int it = 0; it < 48; ++it) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint32_t off = shift ? static_cast<uint32_t>((tap / 3) * 58 + tap % 3) * row16 : 0;
          tc_mma_bf16_elect(tmem, ad0 + off + (it & 1) * 2, bd0 + (tap & 1) * 2, idesc,
                            (it | tap) != 0 ? 1u : 0u);
        }
      }
      tc_commit_elect(&bar);
      __syncwarp();
      mbar_wait(&bar, rep);
    }
    if ((threadIdx.x & 31) == 0) out[0] = clock64() - t0;
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
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int layout = 0; layout < 4; ++layout)
    for (int n : {64, 96, 128, 192, 256}) {
      k<<<1, 128, 200 * 1024>>>(n, layout, d);
      long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("layout %d N %3d: %.1f cycles per MMA (M128 K16)  %s\n", layout, n, c / 432.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
