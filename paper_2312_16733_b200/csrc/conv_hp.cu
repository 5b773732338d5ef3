// conv_hp.cu — stride-1 3x3 WeightSlice convolution for WIDE layers as a
// shifted-window ("halo") implicit GEMM on 2-CTA tcgen05 pairs (sm_100a):
// OFA-ResNet50's 3x3 convs at 28 and 14 px (104-360 active channels).
//
// Why (profiles/round2): conv_tc feeds these layers with TMA
// im2col boxes — every K block re-reads 128 output pixels x 64 channels per
// filter tap, 9 boxes per channel block, 128 pixel requests each.  Measured
// on B200, the loads alone (SSN_TC_DEBUG=2, no MMA) take as long as the whole
// layer: the im2col request stream, not the tensor core, bounds it.  Here:
//  * the A window map is the subnet row's `rmap` slot (these convs have no
//    residual; `amap` keeps conv_tc's im2col map for the small-batch graphs);
//  * output positions are taken in padded-width order (HaloGeom, Wp = W + 2):
//    tap (r, s) of position p reads window pixel p + r*Wp + s, so ONE tiled
//    TMA box per 64-channel block — the halo window, rows of 128 B, SW128 —
//    feeds all 9 taps: each tap's A operand is the same window at a row
//    offset (any 128-B row offset is a legal SW128 K-major start,
//    tools/ubench/sw128_shift.cu);
//  * a CTA tile is RT whole padded rows (<= 128 positions) of one image; a
//    cluster of two CTAs computes two such tiles (consecutive in the
//    (image, row-block) order) as ONE M = 256 tcgen05.mma.cta_group::2, each
//    CTA holding its own window and HALF of the weight rows;
//  * B (the WeightSlice of one (channel block, filter row)) streams through a
//    ring of {64 ch, bn/2 rows, 3 taps} boxes of the max-shape KRSC tensor
//    (a map with the tap dimension outermost, so each tap lands as its own
//    SW128 K-major block): 24-48 KB per box — one producer thread sustains
//    about one TMA box per ~460 cycles (tools/ubench/tma_rate.cu), so the
//    feed rate grows with the box size;
//  * garbage positions (2 padding columns per row, rows past H) are computed
//    and dropped by the epilogue: 196/256 of the MMA rows are live at 14 px,
//    784/896 at 28 px.
// Warp roles (384 threads): warp 0 window producer, warp 1 MMA issuer (CTA 0
// of the pair), warps 2-3 weight producers (alternate stages), warps 4-11 the
// epilogue (TMEM -> padded smem transpose -> SubnetNorm + activation on
// coalesced 64-byte row segments), as conv_tc.  Two TMEM accumulators.
#include <cstdio>
#include <cstdlib>

#include "device.cuh"

namespace ssn {

constexpr int HP_BN_MAX = 256;
// 8 epilogue warps (2 groups of 4 TMEM lane quarters): a pair unit is
// ~20k MMA cycles, its epilogue a few thousand, and the 18 KB of staging a
// third group would need buys a 4th weight stage instead
constexpr int HP_EPI_WARP0 = 4;
constexpr int HP_EPI_WARPS = 8;
constexpr int HP_EPI_GROUPS = 2;
constexpr int HP_THREADS = (HP_EPI_WARP0 + HP_EPI_WARPS) * 32;
constexpr int HP_STG_LD = 36;
constexpr int HP_STG_BYTES = HP_EPI_WARPS * 32 * HP_STG_LD * 4;
constexpr int HP_TAPS = 3;  // taps (one filter row) per B box
constexpr int HP_SMEM_MAX = 232448;
constexpr int HP_NACC = 2;

__host__ __device__ __forceinline__ int hp_window_bytes(int w) {
  const HaloGeom g = halo_geom(w, 3);
  return g.r * g.wp * 128;
}
__host__ __device__ __forceinline__ int hp_window_slot(int w) {
  return (hp_window_bytes(w) + 1023) & ~1023;
}

__global__ void __launch_bounds__(HP_THREADS, 1)
    conv_hp_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const HaloGeom hg = halo_geom(p.w_, 3);
  const int wp = hg.wp, rt = hg.rt;
  const int wslot = hp_window_slot(p.w_);
  const uint32_t wbytes = static_cast<uint32_t>(hp_window_bytes(p.w_));
  const int SB = p.h_stages;  // B ring depth
  const int bstage = HP_TAPS * (p.bn / 2) * 128;  // graph-width filter-row box
  uint8_t* sW = smem;                         // [2] halo windows
  uint8_t* sB = smem + 2 * wslot;             // [SB] B half-boxes (3 taps each)
  float* stg = reinterpret_cast<float*>(sB + SB * bstage);
  uint64_t* afull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + HP_STG_BYTES);
  uint64_t* aempty = afull + 2;
  uint64_t* bfull = aempty + 2;
  uint64_t* bempty = bfull + SB;
  uint64_t* tfull = bempty + SB;
  uint64_t* tempty = tfull + HP_NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + HP_NACC);

  const OpDesc* dp = desc_ptr(p.row, p.fixed, p.op);
  const OpDims d = load_desc(p.row, p.fixed, p.op);
  const int d_hrows = dp->hrows;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  // barriers, TMEM and the cluster sync need no descriptor field: they run
  // while the row -> descriptor loads are in flight (as conv_tc)
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < HP_NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], HP_EPI_WARPS * 2);  // both CTAs' epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem2_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int bn = conv_bn_active(p.bn, d.cout, 2);
  // the subnet row's hmap has this subnet's tile width; a row without one
  // uses the graph's max-width map (rows past the active width land unused)
  const bool own_wmap = d_hrows == bn / 2;
  const CUtensorMap* wm = own_wmap ? &dp->hmap : &wmap;
  const int brows = own_wmap ? bn / 2 : p.bn / 2;
  const int nt = (d.cout + bn - 1) / bn;
  const int tpi = (p.h + rt - 1) / rt;           // CTA tiles per image
  const int pairs = (p.n * tpi + 1) / 2;          // pair tiles (2 CTA tiles each)
  const int units = pairs * nt;
  const uint32_t rank = cluster_rank();
  const int u0 = static_cast<int>(blockIdx.x) / 2, ustep = static_cast<int>(gridDim.x) / 2;
  const bool idle = u0 >= units;  // both CTAs of a pair agree
  const int ncb = (d.cin + 63) / 64;
  if (tid == 0 && !idle) {
    tma_prefetch(wm);
    tma_prefetch(&dp->rmap);
  }
  pdl_trigger();

  // CTA tile q -> (image, first output row); tile index past the batch = idle half
  auto tile_of = [&](int u, int& img, int& r0) {
    const int q = (u / nt) * 2 + static_cast<int>(rank);
    img = q / tpi;
    r0 = (q - img * tpi) * rt;
  };

  if (idle) {
    // no pair tile of the actuated subnet: straight to the teardown
  } else if (warp == 0) {
    // ====================================================== window producer
    const bool leader = elect_one();
    pdl_wait();
    int g = 0;
    for (int u = u0; u < units; u += ustep) {
      int img, r0;
      tile_of(u, img, r0);
      for (int cb = 0; cb < ncb; ++cb, ++g) {
        const int w = g & 1;
        mbar_wait(&aempty[w], ((g >> 1) & 1) ^ 1);
        if (leader) {
          if (p.dbg & 4) {  // profiling: no window loads
            if (rank == 0) mbar_arrive(&afull[w]);
          } else {
            if (rank == 0) mbar_arrive_expect_tx(&afull[w], 2 * wbytes);
            tma2_load_4d(sW + w * wslot, &dp->rmap, &afull[w], cb * 64, -1, r0 - 1, img);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ====================================================== weight producers
    // stage h = (unit, channel block, filter row); warps 2 / 3 alternate
    const int pidx = warp - 2;
    const bool leader = elect_one();
    const uint32_t btx = static_cast<uint32_t>(brows) * 128 * HP_TAPS * 2;
    const int koff = (p.k_max - 3) / 2;
    int h = 0;
    for (int u = u0; u < units; u += ustep) {
      const int n0 = (u % nt) * bn + static_cast<int>(rank) * (bn / 2);
      for (int cb = 0; cb < ncb; ++cb)
        for (int r = 0; r < 3; ++r, ++h) {
          if ((h & 1) != pidx) continue;
          const int s = h % SB;
          mbar_wait(&bempty[s], ((h / SB) & 1) ^ 1);
          if (leader && (p.dbg & 8)) {  // profiling: no weight loads
            if (rank == 0) mbar_arrive(&bfull[s]);
          } else if (leader) {
            if (rank == 0) mbar_arrive_expect_tx(&bfull[s], btx);
            tma2_load_3d(sB + s * bstage, wm, &bfull[s], cb * 64, n0, (r + koff) * p.k_max + koff);
          }
          __syncwarp();
        }
    }
  } else if (warp == 1) {
    // ====================================================== MMA issuer (CTA 0)
    if (rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(bn, 256);
      const uint64_t a_base = umma_desc_sw128(smem_u32(sW));
      const uint64_t b_base = umma_desc_sw128(smem_u32(sB));
      int g = 0, h = 0, i = 0;
      for (int u = u0; u < units; u += ustep, ++i) {
        const int a = i & 1;
        mbar_wait(&tempty[a], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + a * HP_BN_MAX;
        for (int cb = 0; cb < ncb; ++cb, ++g) {
          const int w = g & 1;
          mbar_wait(&afull[w], (g >> 1) & 1);
          const int nks = min(4, (d.cin - cb * 64 + 15) / 16);
          const uint64_t ad = a_base + static_cast<uint64_t>((w * wslot) >> 4);
          for (int r = 0; r < 3; ++r, ++h) {
            const int st = h % SB;
            mbar_wait(&bfull[st], (h / SB) & 1);
            tc_fence_after();
            const uint64_t bd0 = b_base + static_cast<uint64_t>((st * bstage) >> 4);
#pragma unroll
            for (int sx = 0; sx < 3; ++sx) {
              const uint64_t at = ad + static_cast<uint64_t>((r * wp + sx) * 8);
              const uint64_t bd = bd0 + static_cast<uint64_t>((sx * brows * 128) >> 4);
              for (int kk = 0; kk < nks && !(p.dbg & 2); ++kk)
                tc2_mma_bf16_elect(acc, at + static_cast<uint64_t>(kk * 2),
                                   bd + static_cast<uint64_t>(kk * 2), idesc,
                                   (cb | r | sx | kk) != 0 ? 1u : 0u);
            }
            tc2_commit_mc_elect(&bempty[st]);
            __syncwarp();
          }
          tc2_commit_mc_elect(&aempty[w]);  // window w free once its 9 taps retire
          __syncwarp();
        }
        tc2_commit_mc_elect(&tfull[a]);
        __syncwarp();
      }
    }
  } else {
    // ====================================================== epilogue
    pdl_wait();
    const int ew = warp - HP_EPI_WARP0;
    const int quarter = warp & 3;
    const int group = ew >> 2;
    float* st = stg + ew * (32 * HP_STG_LD);
    const int seg = lane & 3, rsub = lane >> 2;
    const int nchunk = (bn + 31) / 32;
    const bool relu = p.act == 1;
    int i = 0;
    for (int u = u0; u < units; u += ustep, ++i) {
      const int a = i & 1;
      int img, r0;
      tile_of(u, img, r0);
      const int nb = (u % nt) * bn;
      const int nch = min(nchunk, (d.cout - nb + 31) / 32);
      mbar_wait(&tfull[a], (i >> 1) & 1);
      tc_fence_after();
      for (int c = group; c < nch; c += HP_EPI_GROUPS) {
        const int col = nb + c * 32 + seg * 8;
        const bool colok = col < d.cout && c * 32 + seg * 8 < bn;
        float sc[8], sh[8];
        if (colok) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            sc[q] = d.scale ? __ldg(d.scale + col + q) : 1.f;
            sh[q] = d.shift ? __ldg(d.shift + col + q) : 0.f;
          }
        }
        float v[32];
        tmem_ld32(tmem + a * HP_BN_MAX + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
        float4* srow = reinterpret_cast<float4*>(st + lane * HP_STG_LD);
#pragma unroll
        for (int q = 0; q < 8; ++q) srow[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        __syncwarp();
        if (colok && !(p.dbg & 1)) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4) {
            const int pos = quarter * 32 + rsub + 8 * r4;  // padded-width position in the CTA tile
            const int rr = pos / wp, cc = pos - rr * wp;
            const int oh = r0 + rr;
            if (rr >= rt || cc >= p.wo || oh >= p.ho || img >= p.n) continue;
            const float4* sp = reinterpret_cast<const float4*>(st + (rsub + 8 * r4) * HP_STG_LD + seg * 8);
            const float4 lo = sp[0], hi = sp[1];
            float o[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              o[q] = o[q] * sc[q] + sh[q];
              if (relu) o[q] = fmaxf(o[q], 0.f);
            }
            uint4 pk;
            pk.x = pack_bf16x2(o[0], o[1]);
            pk.y = pack_bf16x2(o[2], o[3]);
            pk.z = pack_bf16x2(o[4], o[5]);
            pk.w = pack_bf16x2(o[6], o[7]);
            const size_t m = (static_cast<size_t>(img) * p.ho + oh) * p.wo + cc;
            *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + m * d.ldo + col) = pk;
          }
        }
        __syncwarp();  // staging tile is rewritten by the next chunk
      }
      // accumulator a drained by this warp (both CTAs' warps arrive on CTA 0)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(&tempty[a], 0));
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem2_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFnP = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFnP hp_encoder() {
  static EncodeTiledFnP fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFnP>(ptr);
    return static_cast<EncodeTiledFnP>(nullptr);
  }();
  return fn;
}

// N tile of a pair: the active width in <= 256-wide, 32-aligned tiles
int hp_choose_bn(int cout_max) {
  const int nt = (cout_max + HP_BN_MAX - 1) / HP_BN_MAX;
  const int b = (cout_max + nt - 1) / nt;
  return (b + 31) / 32 * 32;
}

static int hp_b_stages(int w, int bn) {
  const long avail = HP_SMEM_MAX - 1024 - 2L * hp_window_slot(w) - HP_STG_BYTES - 256;
  const long st = avail / (static_cast<long>(HP_TAPS) * (bn / 2) * 128);
  return static_cast<int>(st > 8 ? 8 : st);
}

// B operand of conv_hp: the max-shape KRSC tensor [cout][taps][cin_store]
// viewed as {cin_store, cout, taps} (tap dimension outermost) with boxes
// {64 ch, rows, 3 taps}: one filter row of one 64-channel block, each tap a
// contiguous [rows][128 B] SW128 K-major block.
int make_hp_weight_map(CUtensorMap* map, const void* w, int cin_store, int taps, int cout, int rows) {
  EncodeTiledFnP enc = hp_encoder();
  if (!enc) return -1;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cin_store), static_cast<cuuint64_t>(cout),
                        static_cast<cuuint64_t>(taps)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(taps) * cin_store * 2,
                           static_cast<cuuint64_t>(cin_store) * 2};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(rows), HP_TAPS};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

// Wide stride-1 3x3 convs whose max width exceeds the resident-weight halo
// kernel (conv_halo: cout <= 128).  k_max 3 only (OFA-ResNet50).  Measured
// against conv_tc's im2col path (ncu device time, tools/microbench_conv.py,
// profiles/round2/README.md): 360 ch at 14 px bs64 38 vs 53 us, bs256 113 vs
// 172 us; 176 ch at 28 px 34.5 vs 38 us.  The graph uses it up to 30 px
// (SSN_HP_MAX_W overrides for experiments; the operator API, graph = false,
// takes any width so the parity tests cover other geometries).
bool hp_eligible(int h, int w, int k_max, int stride, int cin_max, int cout_max, bool graph) {
  static const bool off = [] {
    const char* e = getenv("SSN_NO_HP");  // A/B switch for profiling
    return e && atoi(e) != 0;
  }();
  static const int max_w = [] {
    const char* e = getenv("SSN_HP_MAX_W");
    return e ? atoi(e) : 30;
  }();
  if (off || stride != 1 || k_max != 3 || h < 8 || w < 12 || w > 62 || (graph && w > max_w)) return false;
  if (cout_max <= 128 || (cout_max & 7) != 0 || (cin_max & 7) != 0) return false;
  return hp_b_stages(w, hp_choose_bn(cout_max)) >= 2;
}

// A operand: [n][h][w][cin_a] NHWC bf16, box {64 ch, Wp, R, 1}, 128-byte
// swizzle: one halo window of one 64-channel block as 128-B pixel rows.
int make_hp_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld) {
  EncodeTiledFnP enc = hp_encoder();
  if (!enc || (cin & 7) != 0 || (ld & 7) != 0) return -1;
  const HaloGeom g = halo_geom(w, 3);
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cin), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(w) * ld * 2,
                           static_cast<cuuint64_t>(h) * w * ld * 2};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(g.wp), static_cast<cuuint32_t>(g.r), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

static int hp_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t init_conv_hp() {
  return cudaFuncSetAttribute(conv_hp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              HP_SMEM_MAX);
}

// p: the op's max geometry + graph-baked batch, p.bn = hp_choose_bn(cout_max);
// wmap: make_hp_weight_map at the graph width (bn / 2 rows per box).
cudaError_t launch_conv_hp(ConvParams p, const CUtensorMap& wmap, cudaStream_t s) {
  static const int dbg = [] {
    const char* e = getenv("SSN_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  p.dbg = dbg;
  p.h_stages = hp_b_stages(p.w_, p.bn);
  if (p.h_stages < 2 || p.ho != p.h || p.wo != p.w_) return cudaErrorInvalidValue;
  const long smem = 1024 + 2L * hp_window_slot(p.w_) +
                    static_cast<long>(p.h_stages) * HP_TAPS * (p.bn / 2) * 128 +
                    HP_STG_BYTES + (4 + 2 * p.h_stages + 2 * HP_NACC) * 8 + 16;
  const HaloGeom g = halo_geom(p.w_, 3);
  const long pairs = (static_cast<long>(p.n) * ((p.h + g.rt - 1) / g.rt) + 1) / 2;
  const long units = pairs * ((p.cout_max + p.bn - 1) / p.bn);
  const long slots = hp_sm_count() / 2;
  const long np = units < slots ? units : slots;
  return launch_pdl(conv_hp_kernel, dim3(static_cast<unsigned>(np * 2)), dim3(HP_THREADS),
                    static_cast<size_t>(smem), s, 2, p, wmap);
}

}  // namespace ssn
