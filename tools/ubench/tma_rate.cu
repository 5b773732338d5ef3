// TMA L2->smem feed rate per SM: every CTA (one per SM) streams boxes of an
// L2-resident bf16 matrix through a STAGES-deep ring; a consumer warp only
// waits and releases.  Reports bytes per SM-cycle (profiling aid).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include "device.cuh"
using namespace ssn;

__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
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
#ifdef SPIN
#define WAIT mbar_spin
#else
#define WAIT mbar_wait
#endif
template <int STAGES, int BOX_ROWS, int P, int SPLIT = 1>
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap map, int iters, int rows_total,
                                          long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = sm;
  constexpr int BYTES = BOX_ROWS * 128;
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
#ifdef LANES
  const bool prod = warp == 0 && lane < P;  // P producer LANES of warp 0
  const int pid = lane;
#else
  const bool prod = warp < P && lane == 0;  // P producer warps
  const int pid = warp;
#endif
  if (prod) {  // producer pid owns stages s = pid (mod P)
    for (int g = pid; g < iters; g += P) {
      const int s = g % STAGES;
      WAIT(&empty[s], ((g / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], BYTES);
      const int row = static_cast<int>((static_cast<long>(blockIdx.x) * (rows_total / 148) + static_cast<long>(g) * BOX_ROWS) % (rows_total - BOX_ROWS));
#pragma unroll
      for (int q = 0; q < SPLIT; ++q)  // SPLIT boxes of BOX_ROWS / SPLIT rows per stage
        tma_load_2d(buf + s * BYTES + q * (BYTES / SPLIT), &map, &full[s], 0, row + q * (BOX_ROWS / SPLIT));
    }
  }
#ifdef LANES
  else if (warp == 1 && lane == 0) {
#else
  else if (warp == P && lane == 0) {
#endif
    for (int g = 0; g < iters; ++g) {
      const int s = g % STAGES;
      WAIT(&full[s], (g / STAGES) & 1);
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

template <int STAGES, int BOX_ROWS, int P, int SPLIT = 1>
void run(CUtensorMap map, int rows_total, long long* d) {
  const int iters = 2000;
  const int smem = STAGES * BOX_ROWS * 128 + 1024;
  cudaFuncSetAttribute(k<STAGES, BOX_ROWS, P, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k<STAGES, BOX_ROWS, P, SPLIT><<<148, 256, smem>>>(map, iters, rows_total, d);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("producers=%d stages=%2d stage=%3d rows (%5d B) in %d box(es): %6.1f B/cycle/SM (slowest SM)\n", P,
         STAGES, BOX_ROWS, BOX_ROWS * 128, SPLIT, double(iters) * BOX_ROWS * 128 / mx);
}

int main(int argc, char** argv) {
  // argv[2] = row pitch in bytes (default 128: contiguous rows; e.g. 6480 =
  // the KRSC pitch of a 3x3 x 360-channel weight tensor)
  // default 16384 x 64 bf16 = 2 MB (L2 resident, shared by all SMs); argv[1]
  // = rows, e.g. 1048576 (128 MB: each SM streams its own, mostly distinct data)
  const int rows = argc > 1 ? atoi(argv[1]) : 16384;
  const long pitch = argc > 2 ? atol(argv[2]) : 128;
  void* src;
  cudaMalloc(&src, rows * pitch);
  cudaMemset(src, 0, rows * pitch);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fn);
  auto mk = [&](int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch)};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  run<8, 64, 1>(mk(64), rows, d);
  run<8, 128, 1>(mk(128), rows, d);
  run<6, 256, 1>(mk(256), rows, d);
  run<8, 64, 2>(mk(64), rows, d);
  run<8, 128, 2>(mk(128), rows, d);
  run<6, 256, 2>(mk(256), rows, d);
  run<8, 128, 4>(mk(128), rows, d);
  run<8, 256, 4>(mk(256), rows, d);
  run<4, 256, 2>(mk(256), rows, d);
  run<3, 256, 2>(mk(256), rows, d);
  run<4, 256, 1>(mk(256), rows, d);
  // per-wait vs per-issue cost: the same stage bytes in 1, 2 or 4 boxes
  run<8, 256, 1, 2>(mk(128), rows, d);
  run<8, 256, 1, 4>(mk(64), rows, d);
  run<8, 128, 1, 2>(mk(64), rows, d);
  run<8, 256, 2, 2>(mk(128), rows, d);
  return 0;
}
