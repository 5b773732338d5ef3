// Microbenchmark (profiling aid, not product code): TMA feed rate of the A
// operand of a 3x3 convolution, im2col boxes vs tiled boxes, on the 28 -> 14
// px stride-2 layer of OFA-ResNet50 (input [64][28][28][360] bf16, 36 MB,
// L2-resident after the first pass).  Every CTA (one per SM) streams 16 KB
// A boxes of (tap, 64-channel block, pixel tile) through a 6-deep ring with
// P producer threads (argv[2], default 3 as conv_tc); reports B/cycle/SM of
// the slowest SM.
//   mode 0: im2col, stride 2 (conv_tc today): 128 output pixels per box
//   mode 1: tiled, element strides {1, 2, 2, 1}: 14 x 9 output pixels of one
//           image per box (126 rows)
//   mode 2: im2col, stride 1 (the 14 px stride-1 layers' conv_tc path)
//   mode 3: tiled, stride 1: 14 x 9 pixels
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//      -I../../paper_2312_16733_b200/csrc tma_modes.cu -o tma_modes -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include "device.cuh"
using namespace ssn;

constexpr int N = 64, H = 28, W = 28, STAGES = 6;
static int C = 360;  // argv[1]: channels = pixel pitch / 2 (360: 720-B rows, 16-B aligned only)

__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap map, int mode, int iters,
                                          long long* out, int P) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
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
  const long long t0 = clock64();
  const int stride = mode < 2 ? 2 : 1;
  const int ho = (H + 2 - 3) / stride + 1, wo = ho;
  const uint32_t bytes = mode == 1 || mode == 3 ? 126 * 128 : 128 * 128;
  if (warp < P && lane == 0) {
    for (int g = warp; g < iters; g += P) {
      const int s = g % STAGES;
      mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      // walk (tile, tap, channel block) like conv_tc's K loop
      const int cb = g % 6, tap = (g / 6) % 9, tile = (blockIdx.x + 148 * (g / 54)) % 512;
      const int r = tap / 3, sx = tap % 3;
      if (mode == 0 || mode == 2) {
        const int m0 = (tile * 128) % (N * ho * wo);
        const int img = m0 / (ho * wo), rem = m0 % (ho * wo), oh = rem / wo, ow = rem % wo;
        tma_im2col_4d(buf + s * 16384, &map, &full[s], cb * 64, ow * stride - 1, oh * stride - 1, img,
                      static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
      } else {
        const int img = tile % N, oh0 = (tile / N) % 2 * 9;
        tma_load_4d(buf + s * 16384, &map, &full[s], cb * 64, sx - 1, oh0 * stride + r - 1, img);
      }
    }
  } else if (warp == P && lane == 0) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % STAGES;
      mbar_wait(&full[s], (g / STAGES) & 1);
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main(int argc, char** argv) {
  if (argc > 1) C = atoi(argv[1]);
  const int P = argc > 2 ? atoi(argv[2]) : 3;  // producer warps (<= STAGES, <= 7)
  void* src;
  const size_t bytes = static_cast<size_t>(N) * H * W * C * 2;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  using EncT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  using EncI = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                            const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncT enct = reinterpret_cast<EncT>(fn);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q);
  EncI enci = reinterpret_cast<EncI>(fn);
  cuuint64_t dims[4] = {C, W, H, N};
  cuuint64_t strides[3] = {C * 2ull, W * C * 2ull, static_cast<cuuint64_t>(H) * W * C * 2};
  const int smem = STAGES * 16384 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 4; ++mode) {
    CUtensorMap m;
    CUresult r;
    const cuuint32_t st = mode < 2 ? 2 : 1;
    if (mode == 0 || mode == 2) {
      const int lower[2] = {-1, -1}, upper[2] = {-1, -1};  // pad 1, k 3: upper = pad - (k - 1)
      cuuint32_t estr[4] = {1, st, st, 1};
      r = enci(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, src, dims, strides, lower, upper, 64, 128, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint32_t box[4] = {64, 14 * st, 9 * st, 1};
      cuuint32_t estr[4] = {1, st, st, 1};
      r = enct(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, src, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      printf("mode %d: encode failed (%d)\n", mode, static_cast<int>(r));
      continue;
    }
    const int iters = 3000;
    for (int rep = 0; rep < 2; ++rep) k<<<148, 256, smem>>>(m, mode, iters, d, P);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double b = mode == 1 || mode == 3 ? 126 * 128 : 128 * 128;
    printf("C %d P %d mode %d (%s, stride %u): %6.1f B/cycle/SM  %s\n", C, P, mode,
           mode == 0 || mode == 2 ? "im2col" : "tiled ", st, iters * b / mx, cudaGetErrorString(e));
  }
  return 0;
}
