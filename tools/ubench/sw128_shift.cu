// (also SW64: -DSW64) Does a SW128 K-major UMMA operand tolerate a start address that is a row
// (128 B) offset inside the 1024-B swizzle atom, with the descriptor's
// base-offset field = (addr >> 7) & 7?  (profiling/feasibility aid)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "device.cuh"
using namespace ssn;

constexpr int ROWS = 136;  // A window rows (128 + 8)
constexpr int N = 16;

#ifdef SW64
constexpr int RB = 64, KC = 32;  // row bytes, channels per row
__device__ __forceinline__ uint64_t desc_sw(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;  // SBO: 8 rows x 64 B
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;         // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ int swz(int r, int chunk) { return chunk ^ ((r >> 1) & 3); }
#else
constexpr int RB = 128, KC = 64;
__device__ __forceinline__ uint64_t desc_sw(uint32_t addr) { return umma_desc_sw128(addr); }
__device__ __forceinline__ int swz(int r, int chunk) { return chunk ^ (r % 8); }
#endif
__device__ __forceinline__ uint64_t desc_sw128_off(uint32_t addr, int mode) {
  uint64_t d = desc_sw(addr);
  if (mode == 1) d |= static_cast<uint64_t>((addr >> 7) & 7) << 49;
  return d;
}

__global__ void k(const float* A, const float* B, float* D, int off, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;                      // ROWS x 128 B, SW128
  uint8_t* sb = sm + 1024 * ((ROWS * 128 + 1023) / 1024);  // N x 128 B, SW128
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // fill: element (r, k) bf16 at row r, 16-B chunk (k/8) ^ (r%8), within-chunk k%8
  for (int i = tid; i < ROWS * KC; i += blockDim.x) {
    const int r = i / KC, kk = i % KC;
    reinterpret_cast<__nv_bfloat16*>(sa + r * RB + swz(r, kk / 8) * 16)[kk % 8] = __float2bfloat16(A[i]);
  }
  for (int i = tid; i < N * KC; i += blockDim.x) {
    const int r = i / KC, kk = i % KC;
    reinterpret_cast<__nv_bfloat16*>(sb + r * RB + swz(r, kk / 8) * 16)[kk % 8] = __float2bfloat16(B[i]);
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t idesc = umma_idesc_bf16(N);
    const uint32_t aaddr = smem_u32(sa) + off * RB;
    for (int kk = 0; kk < KC / 16; ++kk)
      tc_mma_bf16_elect(tmem, desc_sw128_off(aaddr, mode) + 2 * kk,
                        desc_sw(smem_u32(sb)) + 2 * kk, idesc, kk > 0);
    tc_commit_elect(&bar);
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
    for (int n = 0; n < N; ++n) D[(warp * 32 + (tid & 31)) * N + n] = v[n];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 32);
  }
}

int main() {
  float *A, *B, *D;
  cudaMallocManaged(&A, ROWS * 64 * 4);
  cudaMallocManaged(&B, N * 64 * 4);
  cudaMallocManaged(&D, 128 * N * 4);
  for (int i = 0; i < ROWS * KC; ++i) A[i] = ((i * 7919) % 17 - 8) / 8.0f;
  for (int i = 0; i < N * KC; ++i) B[i] = ((i * 104729) % 13 - 6) / 4.0f;
  const int smem = 1024 * ((ROWS * 128 + 1023) / 1024) + N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 1; ++mode)
    for (int off = 0; off < 9; ++off) {
      k<<<1, 128, smem>>>(A, B, D, off, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int kk = 0; kk < KC; ++kk) ref += double(A[(off + m) * KC + kk]) * B[n * KC + kk];
          maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
        }
      printf("mode=%d (base_offset %s) row offset %d: max |err| = %g\n", mode, mode ? "set" : "0", off, maxerr);
    }
  return 0;
}
