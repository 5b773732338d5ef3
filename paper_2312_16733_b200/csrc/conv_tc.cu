// conv_tc.cu — WeightSlice implicit-GEMM convolution on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   Y[M, cout_a] = act( SubnetNorm_i( im2col(X)[M, K_a] . W[:cout_a, K_a]^T ) (+ res) )
//   M = n * ho * wo, K_a = k_a^2 * cin_a  (PAPER.md:497-502 WeightSlice,
//   PAPER.md:472-481 SubnetNorm folded into the epilogue).
//
// Design:
//  * Persistent, warp-specialised: one CTA per SM walks a static tile
//    schedule.  Warps 0-3 produce operands, warp 12 issues tcgen05.mma,
//    warps 4-11 drain the accumulator.  The accumulator is double-buffered in
//    TMEM (2 x BN_MAX fp32 columns), so tile i's epilogue overlaps tile i+1's
//    mainloop, and the smem ring runs continuously across tiles.
//  * B operand (weights) — the max-shape KRSC tensor is stored ONCE; TMA
//    tensor maps over [cout_max][k_max^2][cin_max] load boxes of its LEADING
//    slice straight into 128B-swizzled shared memory, never a copy.  Normal
//    mode: box {64 ch, 1 tap, bn}.  Packed-tap mode (small cin_a, full
//    kernel): box {cslot, 64/cslot taps, bn} so one 64-wide K block spans
//    several taps instead of wasting most of it on zero channels.
//  * A operand (activations) — compact NHWC with cin_a channels (a
//    subnet-dependent stride), gathered by 128 producer threads with 16-byte
//    cp.async (zero-fill for padding / M tail / channel tail) directly into
//    the same SW128 K-major layout; cp.async.wait_group + fence.proxy.async +
//    mbarrier hand it to the tensor core.
//  * Epilogue: tcgen05.ld 32 lanes x 32 columns, SubnetNorm scale/shift,
//    residual (prefetched before the TMEM load), ReLU, bf16 / fp32 store.
//  * Subnet extents (cin_a, cout_a, k_a, SubnetNorm row) come from the
//    actuated subnet's device descriptor, so one graph-captured launch serves
//    every subnet; the tile count is derived from cout_a on the device.
#include <cstdio>

#include "device.cuh"

namespace ssn {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_PROD_WARPS = 4;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_MMA_WARP = TC_PROD_WARPS + TC_EPI_WARPS;  // 12
constexpr int TC_THREADS = (TC_MMA_WARP + 1) * 32;          // 416
constexpr int TC_STG_LD = 36;  // padded fp32 row of the 32x32 epilogue transpose tile
constexpr int TC_STG_BYTES = TC_EPI_WARPS * 32 * TC_STG_LD * 4;


template <int BN_MAX, int STAGES>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN_MAX * TC_BK * 2;
  static constexpr int SMEM =
      1024 + STAGES * (A_BYTES + B_BYTES) + TC_STG_BYTES + (2 * STAGES + 4) * 8 + 16;
};

__device__ __forceinline__ int cslot_for(int cin, int k, int k_max) {
  if (k != k_max || k == 1) return 64;
  if (cin <= 8) return 8;
  if (cin <= 16) return 16;
  if (cin <= 32) return 32;
  return 64;
}

template <int BN_MAX, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ TcMaps maps) {
  using C = TcCfg<BN_MAX, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  float* epi_stage = reinterpret_cast<float*>(sB + STAGES * C::B_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES + TC_STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const OpDesc d = load_desc(p.row, p.fixed, p.op);
  const int bn = p.bn;
  const int mt = (p.M + TC_BM - 1) / TC_BM;
  const int nt = (d.cout + bn - 1) / bn;  // WeightSlice: only tiles inside cout_a
  const int tiles = mt * nt;
  if (static_cast<int>(blockIdx.x) >= tiles) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int ka = d.k, pad = d.pad, koff = (p.k_max - ka) / 2;
  const int cslot = cslot_for(d.cin, ka, p.k_max);
  const bool packed = cslot < 64;
  const int tpk = 64 / cslot;  // taps per K block in packed mode
  const int cblocks = (d.cin + TC_BK - 1) / TC_BK;
  const int nk = packed ? (ka * ka + tpk - 1) / tpk : ka * ka * cblocks;
  const CUtensorMap* wmap = &maps.w[cslot == 64 ? 0 : cslot == 32 ? 1 : cslot == 16 ? 2 : 3];

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TC_PROD_WARPS * 32 + 1);  // producers + expect_tx arrival
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], TC_EPI_WARPS);
    }
    fence_mbar_init();
    tma_prefetch(wmap);
  }
  if (warp == TC_MMA_WARP) tmem_alloc(tmem_slot, 2 * BN_MAX);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < TC_PROD_WARPS) {
    // ============================================================ producers
    const int j = lane & 7;      // 16-byte chunk within the 128-byte K row
    const int rsub = lane >> 3;  // 0..3
    const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x);
    const uint32_t a_base = smem_u32(sA);
    const int hwo = p.ho * p.wo;
    const uint32_t tx_bytes = static_cast<uint32_t>(bn * TC_BK * 2);
    // packed mode: this thread's chunk is channel slot (j*8) % cslot of tap (j*8)/cslot
    const int pk_tap = (j * 8) / cslot, pk_c = (j * 8) % cslot;
    int g = 0;  // global K-block counter (ring position)
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t / nt) * TC_BM;
      const int n0 = (t % nt) * bn;
      int pix[8], ih0[8], iw0[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + warp * 32 + rsub + 4 * i;
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
      int tr = 0, ts = 0, cb = 0;  // normal mode iteration state
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        int r, q, c;
        bool cok;
        if (packed) {
          const int tap = kb * tpk + pk_tap;
          r = tap / ka;
          q = tap - r * ka;
          c = pk_c;
          cok = tap < ka * ka && c < d.cin;
          if (tid == 0) {
            mbar_arrive_expect_tx(&full[s], tx_bytes);
            tma_load_4d(sB + s * C::B_BYTES, wmap, &full[s], 0, n0, 0, kb * tpk);
          }
        } else {
          r = tr;
          q = ts;
          c = cb * TC_BK + j * 8;
          cok = c < d.cin;
          if (tid == 0) {
            mbar_arrive_expect_tx(&full[s], tx_bytes);
            tma_load_3d(sB + s * C::B_BYTES, wmap, &full[s], cb * TC_BK,
                        (tr + koff) * p.k_max + (ts + koff), n0);
          }
          if (++cb == cblocks) {
            cb = 0;
            if (++ts == ka) {
              ts = 0;
              ++tr;
            }
          }
        }
        const uint32_t dst = a_base + s * C::A_BYTES;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = warp * 32 + rsub + 4 * i;
          const int ih = ih0[i] + r, iw = iw0[i] + q;
          const bool ok = cok && static_cast<unsigned>(ih) < static_cast<unsigned>(p.h) &&
                          static_cast<unsigned>(iw) < static_cast<unsigned>(p.w_);
          const __nv_bfloat16* src =
              ok ? x + (static_cast<size_t>(pix[i] + ih * p.w_ + iw) * d.cin + c) : x;
          cp_async_16(dst + row * 128 + ((j ^ (row & 7)) << 4), src, ok ? 16u : 0u);
        }
        // decoupled: the barrier completes when this thread's copies land, so
        // all STAGES slots can be in flight and the producer never stalls on
        // its own loads (the CUTLASS sm100 cp.async pipeline contract)
        cp_async_arrive_noinc(&full[s]);
      }
    }
  } else if (warp < TC_MMA_WARP) {
    // ============================================================ epilogue
    // TMEM gives each thread one ROW; global memory wants each warp to touch
    // whole row segments.  Each 32x32 fp32 chunk is transposed through a
    // per-warp padded smem tile: afterwards lane (rsub = lane/4, seg = lane%4)
    // owns 8 consecutive columns of rows rsub, rsub+8, ... so residual loads
    // and output stores are 64-byte row-contiguous and coalesced.
    const int ew = warp - TC_PROD_WARPS;
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int half = ew >> 2;      // column interleave
    float* stg = epi_stage + ew * (32 * TC_STG_LD);
    const int seg = lane & 3, rsub = lane >> 2;
    const float* scale = d.scale;
    const float* shift = d.shift;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int a = i & 1;
      const uint32_t use = static_cast<uint32_t>(i >> 1);
      const int m0 = (t / nt) * TC_BM + quarter * 32;
      const int n0 = (t % nt) * bn;
      mbar_wait(&tfull[a], use & 1);
      tc_fence_after();
      for (int cc = half * 32; cc < bn; cc += 64) {
        if (n0 + cc >= d.cout) break;  // warp-uniform
        float v[32];
        tmem_ld32(tmem + a * BN_MAX + (static_cast<uint32_t>(quarter * 32) << 16) + cc, v);
        float4* srow = reinterpret_cast<float4*>(stg + lane * TC_STG_LD);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          srow[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        const int col = n0 + cc + seg * 8;
        if (col < d.cout && cc + seg * 8 < bn) {
          float sc[8], sh[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            sc[q] = scale ? __ldg(scale + col + q) : 1.f;
            sh[q] = shift ? __ldg(shift + col + q) : 0.f;
          }
          uint4 rv[4];
          if (p.res) {
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4) {
              const int m = m0 + rsub + 8 * r4;
              if (m < p.M)
                rv[r4] = __ldg(reinterpret_cast<const uint4*>(
                    static_cast<const __nv_bfloat16*>(p.res) + static_cast<size_t>(m) * d.cout + col));
            }
          }
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4) {
            const int rr = rsub + 8 * r4;
            const int m = m0 + rr;
            if (m >= p.M) continue;
            const float4* sp = reinterpret_cast<const float4*>(stg + rr * TC_STG_LD + seg * 8);
            const float4 lo = sp[0], hi = sp[1];
            float o[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = o[q] * sc[q] + sh[q];
            float r8[8];
            if (p.res) {
              const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[r4]);
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
            const size_t off = static_cast<size_t>(m) * d.cout + col;
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
        __syncwarp();  // staging tile is rewritten by the next chunk
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
  } else {
    // ============================================================ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(bn);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int a = i & 1;
        const uint32_t use = static_cast<uint32_t>(i >> 1);
        mbar_wait(&tempty[a], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + a * BN_MAX;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&full[s], ph);
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 reads
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(a0 + s * C::A_BYTES);
          // packed-tap B tiles use the no-swizzle core-matrix layout written
          // by the 4-D TMA map: K chunks of 8 are bn*16 bytes apart.
          const uint64_t bd = packed ? umma_desc_noswz(b0 + s * C::B_BYTES, bn * 16, 128)
                                     : umma_desc_sw128(b0 + s * C::B_BYTES);
          const uint64_t bstep = packed ? static_cast<uint64_t>(2 * bn) : 2u;  // 16B units / K=16
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)
            tc_mma_bf16(acc, ad + static_cast<uint64_t>(kk * 2), bd + kk * bstep, idesc,
                        (kb | kk) != 0 ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[a]);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == TC_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * BN_MAX);
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

// Tensor maps over a max-shape KRSC bf16 weight tensor [cout][taps][cin_store]:
// boxes {cslot, 64/cslot, bn} for cslot = 64, 32, 16, 8, 128B swizzle.
int make_weight_maps(TcMaps* maps, const void* w, int cin_store, int taps, int cout, int bn) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return -1;
  // normal mode: {64 ch, 1 tap, bn} boxes, 128B swizzle (SW128 K-major tile)
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(cin_store), static_cast<cuuint64_t>(taps),
                          static_cast<cuuint64_t>(cout)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(cin_store) * 2,
                             static_cast<cuuint64_t>(taps) * cin_store * 2};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(TC_BK), 1, static_cast<cuuint32_t>(bn)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&maps->w[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -static_cast<int>(r);
  }
  // packed-tap modes: the same tensor viewed as (c8, n, c/8, tap) so a box
  // {8, bn, cslot/8, 64/cslot} lands as no-swizzle K-major core matrices
  // ([K chunk][n][8 ch]), K order = tap-major then channel — matching A.
  const int slots[3] = {32, 16, 8};
  for (int i = 0; i < 3; ++i) {
    const int cs = slots[i];
    cuuint64_t dims[4] = {8, static_cast<cuuint64_t>(cout),
                          static_cast<cuuint64_t>((cin_store + 7) / 8),
                          static_cast<cuuint64_t>(taps)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(taps) * cin_store * 2, 16,
                             static_cast<cuuint64_t>(cin_store) * 2};
    cuuint32_t box[4] = {8, static_cast<cuuint32_t>(bn), static_cast<cuuint32_t>(cs / 8),
                         static_cast<cuuint32_t>(64 / cs)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&maps->w[1 + i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(w),
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -static_cast<int>(r);
  }
  return 0;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// N tile: the whole 16-aligned output width when it fits one tile; else the
// width in {256, 128} that keeps the persistent grid busiest.
int choose_bn(int cout_max, long M) {
  const int c16 = (cout_max + 15) / 16 * 16;
  if (c16 <= 256) return c16;
  const long mt = (M + TC_BM - 1) / TC_BM;
  const long sms = num_sms();
  auto cost = [&](int bn) {
    const long tiles = mt * ((cout_max + bn - 1) / bn);
    const long waves = (tiles + sms - 1) / sms;
    return waves * (bn + 64);
  };
  return cost(128) < cost(256) ? 128 : 256;
}

// Instances: ring depth chosen so operands + epilogue staging fit 227 KB.
#define SSN_TC_INSTANCES(X) X(64, 7) X(128, 5) X(256, 3)

cudaError_t init_conv_tc() {
#define SSN_TC_ATTR(BN, ST)                                                           \
  {                                                                                   \
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN, ST>,                      \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         TcCfg<BN, ST>::SMEM);                        \
    if (e != cudaSuccess) return e;                                                   \
  }
  SSN_TC_INSTANCES(SSN_TC_ATTR)
#undef SSN_TC_ATTR
  return cudaSuccess;
}

template <int BN_MAX, int STAGES>
static cudaError_t launch_impl(const ConvParams& p, const TcMaps& maps, cudaStream_t s) {
  using C = TcCfg<BN_MAX, STAGES>;
  const long tiles = static_cast<long>((p.M + TC_BM - 1) / TC_BM) * ((p.cout_max + p.bn - 1) / p.bn);
  const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
  conv_tc_kernel<BN_MAX, STAGES><<<grid, TC_THREADS, C::SMEM, s>>>(p, maps);
  return cudaGetLastError();
}

cudaError_t launch_conv_tc(const ConvParams& p, const TcMaps& maps, cudaStream_t s) {
  if (p.bn <= 64) return launch_impl<64, 7>(p, maps, s);
  if (p.bn <= 128) return launch_impl<128, 5>(p, maps, s);
  return launch_impl<256, 3>(p, maps, s);
}

}  // namespace ssn
