// conv_tc.cu — WeightSlice implicit-GEMM convolution on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   Y[M, cout_a] = act( SubnetNorm_i( im2col(X)[M, K_a] . W[:cout_a, K_a]^T ) (+ res) )
//   M = n * ho * wo, K_a = k_a^2 * cin_a  (PAPER.md:497-502 WeightSlice,
//   PAPER.md:472-481 SubnetNorm folded into the epilogue).
//
// Design:
//  * B operand (weights) — the max-shape KRSC tensor is stored ONCE; a TMA
//    tensor map over [cout_max][k_max^2][cin_max] loads 64-channel x bn-row
//    boxes of its LEADING slice straight into 128B-swizzled shared memory.
//    Channels beyond cin_a inside a box meet zero activations, rows beyond
//    cout_max are TMA zero-filled, so no copy of any slice ever exists.
//  * A operand (activations) — compact NHWC with cin_a channels (subnet
//    dependent stride), gathered by 128 producer threads with 16-byte
//    cp.async (zero-fill for padding / M tail / channel tail) directly into
//    the same SW128 K-major layout; fence.proxy.async + mbarrier hand it to
//    the tensor core.
//  * One elected thread issues tcgen05.mma (M=128, N=bn, K=16) into a TMEM
//    fp32 accumulator; tcgen05.commit releases smem stages.
//  * Epilogue: 4 warps tcgen05.ld their 32 TMEM lanes, apply SubnetNorm
//    scale/shift, residual, ReLU, and store bf16 (or fp32 logits).
//  * Subnet extents (cin_a, cout_a, k_a, SubnetNorm row) come from the
//    actuated subnet's device descriptor, so one graph-captured launch serves
//    every subnet; CTAs whose N tile lies beyond cout_a exit at once.
#include <cstdio>

#include "device.cuh"

namespace ssn {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_THREADS = 160;  // warps 0-3: producers + epilogue; warp 4: MMA

template <int BN_MAX, int STAGES>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN_MAX * TC_BK * 2;
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + (2 * STAGES + 2) * 8 + 16;
};

template <int BN_MAX, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, BN_MAX <= 128 ? 2 : 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap wmap) {
  using C = TcCfg<BN_MAX, STAGES>;
  constexpr int LAG = STAGES - 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const OpDesc d = load_desc(p.row, p.fixed, p.op);
  const int bn = p.bn;
  const int n0 = blockIdx.y * bn;
  if (n0 >= d.cout) return;  // WeightSlice: this N tile is outside cout_a
  const int m0 = blockIdx.x * TC_BM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int cblocks = (d.cin + TC_BK - 1) / TC_BK;
  const int ka = d.k, pad = d.pad, koff = (p.k_max - ka) / 2;
  const int nk = ka * ka * cblocks;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 129);  // 128 producer arrivals + 1 expect_tx arrival
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
    tma_prefetch(&wmap);
  }
  if (warp == 4) tmem_alloc(tmem_slot, BN_MAX);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    const int j = lane & 7;     // 16-byte chunk within the 128-byte K row
    const int rsub = lane >> 3; // 0..3
    int pix[8], ih0[8], iw0[8];
    const int hwo = p.ho * p.wo;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = warp * 32 + rsub + 4 * i;
      const int m = m0 + r;
      if (m < p.M) {
        const int img = m / hwo;
        const int rem = m - img * hwo;
        const int oh = rem / p.wo;
        const int ow = rem - oh * p.wo;
        pix[i] = img * p.h * p.w_;
        ih0[i] = oh * p.stride - pad;
        iw0[i] = ow * p.stride - pad;
      } else {
        pix[i] = 0;
        ih0[i] = -(1 << 20);
        iw0[i] = -(1 << 20);
      }
    }
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x);
    const uint32_t a_base = smem_u32(sA);
    int tr = 0, ts = 0, cb = 0;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      if (tid == 0) {
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(bn * TC_BK * 2));
        tma_load_3d(sB + s * C::B_BYTES, &wmap, &full[s], cb * TC_BK,
                    (tr + koff) * p.k_max + (ts + koff), n0);
      }
      const int c = cb * TC_BK + j * 8;
      const bool cok = c < d.cin;
      const uint32_t dst = a_base + s * C::A_BYTES;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = warp * 32 + rsub + 4 * i;
        const int ih = ih0[i] + tr, iw = iw0[i] + ts;
        const bool ok = cok && static_cast<unsigned>(ih) < static_cast<unsigned>(p.h) &&
                        static_cast<unsigned>(iw) < static_cast<unsigned>(p.w_);
        const __nv_bfloat16* src =
            ok ? x + (static_cast<size_t>(pix[i] + ih * p.w_ + iw) * d.cin + c) : x;
        cp_async_16(dst + r * 128 + ((j ^ (r & 7)) << 4), src, ok ? 16u : 0u);
      }
      cp_async_commit();
      if (kb >= LAG) {
        cp_async_wait<LAG>();
        fence_proxy_async_smem();
        mbar_arrive(&full[(kb - LAG) % STAGES]);
      }
      if (++cb == cblocks) {
        cb = 0;
        if (++ts == ka) {
          ts = 0;
          ++tr;
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int kb = nk > LAG ? nk - LAG : 0; kb < nk; ++kb) mbar_arrive(&full[kb % STAGES]);

    // ------------------------------------------------------------ epilogue
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const bool mok = m < p.M;
    const float* scale = d.scale;
    const float* shift = d.shift;
    for (int cc = 0; cc < bn; cc += 32) {
      if (n0 + cc >= d.cout) break;  // warp-uniform
      float v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc, v);
      if (!mok) continue;
#pragma unroll
      for (int g = 0; g < 32; g += 8) {
        const int col = n0 + cc + g;
        if (col < d.cout) {
          float o[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            o[q] = v[g + q] * (scale ? __ldg(scale + col + q) : 1.f) +
                   (shift ? __ldg(shift + col + q) : 0.f);
          const size_t off = static_cast<size_t>(m) * d.cout + col;
          float r8[8];
          if (p.res) {
            const uint4 rv = *reinterpret_cast<const uint4*>(
                static_cast<const __nv_bfloat16*>(p.res) + off);
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(rh[q]);
              r8[2 * q] = f.x;
              r8[2 * q + 1] = f.y;
            }
            if (!p.res_post) {
#pragma unroll
              for (int q = 0; q < 8; ++q) o[q] += r8[q];
            }
          }
          if (p.act == 1) {
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = fmaxf(o[q], 0.f);
          }
          if (p.res && p.res_post) {
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] += r8[q];
          }
          if (p.out_f32) {
            float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + off);
            yp[0] = make_float4(o[0], o[1], o[2], o[3]);
            yp[1] = make_float4(o[4], o[5], o[6], o[7]);
          } else {
            uint4 pk;
            pk.x = pack_bf16x2(o[0], o[1]);
            pk.y = pack_bf16x2(o[2], o[3]);
            pk.z = pack_bf16x2(o[4], o[5]);
            pk.w = pack_bf16x2(o[6], o[7]);
            *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + off) = pk;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(bn);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(a0 + s * C::A_BYTES);
        const uint64_t bd = umma_desc_sw128(b0 + s * C::B_BYTES);
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          tc_mma_bf16(tmem, ad + static_cast<uint64_t>(kk * 2), bd + static_cast<uint64_t>(kk * 2),
                      idesc, (kb | kk) != 0 ? 1u : 0u);
        tc_commit(&empty[s]);
      }
      tc_commit(tfull);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, BN_MAX);
  }
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// Tensor map over a max-shape KRSC bf16 weight tensor [cout][taps][cin_store]
// with (64 x 1 x bn) boxes, 128B swizzle.
int make_weight_map(CUtensorMap* map, const void* w, int cin_store, int taps, int cout, int bn) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cin_store), static_cast<cuuint64_t>(taps),
                        static_cast<cuuint64_t>(cout)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cin_store) * 2,
                           static_cast<cuuint64_t>(taps) * cin_store * 2};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(TC_BK), 1, static_cast<cuuint32_t>(bn)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

// N tile for an op: the whole (16-aligned) output width when it fits one
// tile, else 256 (128 when the grid would not fill the machine).
int choose_bn(int cout_max, long M) {
  const int c16 = (cout_max + 15) / 16 * 16;
  if (c16 <= 256) return c16;
  const long mt = (M + TC_BM - 1) / TC_BM;
  const long tiles256 = mt * ((cout_max + 255) / 256);
  return tiles256 >= 148 ? 256 : 128;
}

template <int BN_MAX, int STAGES>
static cudaError_t launch_impl(const ConvParams& p, const CUtensorMap& map, cudaStream_t s) {
  using C = TcCfg<BN_MAX, STAGES>;
  dim3 grid((p.M + TC_BM - 1) / TC_BM, (p.cout_max + p.bn - 1) / p.bn);
  conv_tc_kernel<BN_MAX, STAGES><<<grid, TC_THREADS, C::SMEM, s>>>(p, map);
  return cudaGetLastError();
}

// Opt the kernels into >48 KB dynamic shared memory (call before capture).
cudaError_t init_conv_tc() {
  cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<128, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       TcCfg<128, 3>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(conv_tc_kernel<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              TcCfg<256, 4>::SMEM);
}

cudaError_t launch_conv_tc(const ConvParams& p, const CUtensorMap& map, cudaStream_t s) {
  if (p.bn <= 128) return launch_impl<128, 3>(p, map, s);
  return launch_impl<256, 4>(p, map, s);
}

}  // namespace ssn
