// Microbenchmark (profiling aid, not product code): tcgen05.mma throughput of
// 2-CTA pair tiles (cta_group::2, M = 256 over two SMs) against single-CTA
// tiles (M = 128), SW128 K-major operands, K = 16 per instruction, 432
// back-to-back MMAs then one commit + wait.  Cycles are per instruction as
// seen by the issuing SM (each SM of a pair computes a 128 x N x 16 slice).
// Launched as 1 cluster and as 74 clusters / 148 CTAs (whole GPU busy).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//      -I../../paper_2312_16733_b200/csrc mma2_rate.cu -o mma2_rate -lcuda
#include <cstdio>
#include <cstdlib>
#include "device.cuh"
using namespace ssn;

// mode 0: 432 MMAs, one commit.  mode 1: + a commit (multicast for pairs) per
// 4 MMAs onto a 6-deep barrier ring.  mode 2: the conv_tc ring handshake — a
// producer warp waits each stage's "empty" commit and arrives on its "full"
// barrier, the MMA warp waits "full" before the stage's 4 MMAs.  mode 3: mode
// 2 with 8 MMAs (two K blocks) per stage.  mode 4: tcgen05.fence per 4 MMAs,
// no commit; mode 5: commit per 4 MMAs, no fence; modes 6 / 7: modes 2 / 3
// without the per-stage tcgen05.fence::after_thread_sync.
template <int CG>
__global__ void k(int N, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sbuf = dsm + ((1024u - (smem_u32(dsm) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint64_t fullb[6], emptyb[6];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 6; ++i) {
      mbar_init(&fullb[i], 1);
      mbar_init(&emptyb[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    if (CG == 2) tmem2_alloc(&slot, 256);
    else tmem_alloc(&slot, 256);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = umma_idesc_bf16(N, 128 * CG);
  const uint64_t ad0 = umma_desc_sw128(smem_u32(sbuf));
  const uint64_t bd0 = umma_desc_sw128(smem_u32(sbuf + 96 * 1024));
  const bool issuer = CG == 1 || cluster_rank() == 0;
  long long t0 = 0;
  int g = 0;  // ring position (both reps)
  for (int rep = 0; rep < 2; ++rep) {
    if (warp == 0 && issuer) {
      if (rep == 1) t0 = clock64();
      const int per = (mode == 3 || mode == 7) ? 8 : 4;
      for (int st = 0; st < 432 / per; ++st, ++g) {
        const int s = g % 6;
        if (mode >= 2 && mode != 5) mbar_wait(&fullb[s], (g / 6) & 1);
        if (mode != 5 && mode != 6 && mode != 7) tc_fence_after();
#pragma unroll 4
        for (int j = 0; j < per; ++j) {
          if (CG == 2)
            tc2_mma_bf16_elect(tmem, ad0 + (st & 1) * 2, bd0 + (j & 1) * 2, idesc, (st | j) != 0 ? 1u : 0u);
          else
            tc_mma_bf16_elect(tmem, ad0 + (st & 1) * 2, bd0 + (j & 1) * 2, idesc, (st | j) != 0 ? 1u : 0u);
        }
        if (mode >= 1 && mode != 4) {
          if (CG == 2) tc2_commit_mc_elect(&emptyb[s]);
          else tc_commit_elect(&emptyb[s]);
        }
        __syncwarp();
      }
      if (CG == 2) tc2_commit_mc_elect(&bar);
      else tc_commit_elect(&bar);
      __syncwarp();
    } else if (warp == 1 && issuer && mode >= 2 && mode != 4 && mode != 5) {  // producer: stage g+6 may fill once g's MMAs are done
      const int nst = 432 / ((mode == 3 || mode == 7) ? 8 : 4);
      const int g0 = rep * nst;
      for (int gg = g0; gg < g0 + nst; ++gg) {
        const int s = gg % 6;
        if (gg >= 6) mbar_wait(&emptyb[s], ((gg / 6) - 1) & 1);
        if ((threadIdx.x & 31) == 0) mbar_arrive(&fullb[s]);
        __syncwarp();
      }
    }
    if (warp == 0) mbar_wait(&bar, rep);
    __syncthreads();
  }
  if (warp == 0 && issuer && (threadIdx.x & 31) == 0) out[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2) tmem2_dealloc(tmem, 256);
    else tmem_dealloc(tmem, 256);
  }
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  long long* d;
  cudaMalloc(&d, 8 * 148);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode : {1, 4, 5, 2, 6, 3, 7})
  if (only < 0 || mode == only)
  for (int grid : {148})
    for (int cg : {1, 2})
      for (int n : {128, 160, 192}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cg;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaMemset(d, 0, 8 * 148);
        cudaError_t e = cg == 2 ? cudaLaunchKernelEx(&cfg, k<2>, n, mode, d) : cudaLaunchKernelEx(&cfg, k<1>, n, mode, d);
        cudaDeviceSynchronize();
        long long c[148];
        cudaMemcpy(c, d, 8 * 148, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
        printf("mode %d grid %3d cta_group %d N %3d: %.1f cycles per MMA (per-SM 128 x N x 16)  %s %s\n", mode, grid, cg,
               n, mx / 432.0, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
      }
  return 0;
}
