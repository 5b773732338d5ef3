// dw.cu — depthwise k x k WeightSlice conv for bf16 supernets (OFA-MobileNetV3,
// BASELINE config 3): the elastic centre crop of the shared k_max x k_max
// kernel (PAPER.md:497-502 applied per channel), fused SubnetNorm +
// activation, and optionally the squeeze-excite pool of the block's SE.
//
// Bound: HBM for k = 3 (9 FMA per 4-6 bytes moved), the FP32 FMA pipe for
// k = 5 / 7 (25-49 FMA per output element); DESIGN.md §6.
//
// Design (one persistent CTA of 16 warps per SM, warp-specialised):
//  * work unit = tile of TH x TW (14 x 14 or 7 x 7) outputs x 64 channels of
//    one image; tiles run channel-chunk-major so a CTA's consecutive tiles
//    share the chunk's weights (fp32 in shared memory, reloaded only when the
//    chunk changes) and neighbouring halos are L2 hits.  The tile space is
//    computed at run time from the ACTIVE channel count (WeightSlice), so a
//    narrow subnet still spreads over all SMs;
//  * warp 0 streams each tile's input window (TH-1)*S + k rows x (TW-1)*S + k
//    columns x 64 channels with ONE 4-D TMA box into a ring of stages
//    (zero fill at the image border = the conv padding); the box is sized
//    for the active k from the subnet's own tensor map (OpDesc.amap);
//  * warps 1-15: lane = channel pair (bf16x2), one warp task = 7 adjacent
//    outputs of one or two rows (7 divides every OFA-MBv3 width 112/56/28/
//    14/7; a two-row task converts each shared window row once),
//    tasks dealt round-robin over the warps across tile boundaries; per
//    filter row the warp reads the (7-1)*S + k window pixels once (128 B per
//    warp read: conflict-free), converts bf16 -> fp32 on the ALU pipe and
//    issues packed fp32x2 FMAs (FFMA2); epilogue = SubnetNorm FMA,
//    activation, bf16 pack, one coalesced 128-byte store per pixel;
//  * fused SE pool: every consumer warp leaves its per-tile channel sums of
//    the STORED (bf16-rounded) outputs in shared memory; the producer warp
//    adds the warps' sums in fixed order when it recycles the stage and
//    writes one partial per (image, tile) — deterministic, no atomics, and
//    the SE no longer re-reads the activation to pool it.
#include "device.cuh"

namespace ssn {

constexpr int DW_CC = 64;        // channels per tile = 32 lanes x bf16x2
// Narrow layers (max width <= 32, e.g. OFA-MBv3's 24-channel 112-px block):
// CC = 32-channel boxes, each warp lane-half (16 lanes x bf16x2) owns one
// pixel, so a warp task covers 2 x 7 outputs.  With 64-channel boxes a
// 24-channel layer left 20 of 32 lanes idle and staged 80 zero bytes per
// pixel (0.21 of HBM peak, tools/cudnn_ref.py: cuDNN 2x faster).
constexpr int DW_CC_NARROW = 32;
constexpr int DW_QW = 7;         // adjacent outputs per warp task
constexpr int DW_NCW = 15;       // consumer warps
constexpr int DW_THREADS = 32 * (DW_NCW + 1);
constexpr int DW_MAX_STAGES = 8;
constexpr int DW_SMEM_MAX = 225 * 1024;
constexpr int DW_WSM_BYTES = 49 * DW_CC * 4;  // fp32 weights of one chunk, k <= 7

// Tile geometry of a layer (independent of the active k): stride-1 layers
// wider than 7 use 14 x 14 output tiles whose warp tasks cover TWO output
// rows (the K + 1 window rows they read are converted once for both rows);
// 7-wide and stride-2 layers use 7 x 7 tiles of one-row tasks.
struct DwShape {
  int tw, th, qh;
};
__host__ __device__ __forceinline__ DwShape dw_shape(int stride, int wo) {
  return (stride == 1 && wo > 7) ? DwShape{14, 14, 2} : DwShape{7, 7, 1};
}
static inline int cdiv(long a, long b) { return static_cast<int>((a + b - 1) / b); }

int dw_tiles_per_image(int stride, int ho, int wo) {
  const DwShape g = dw_shape(stride, wo);
  return cdiv(ho, g.th) * cdiv(wo, g.tw);
}

// bf16x2 -> float2 on the ALU pipe (PRMT + LOP3; a plain `v << 16` compiles
// to IMAD.SHL, which would compete with the FFMA2s for the FMA pipe)
__device__ __forceinline__ float2 bf2_to_f2(uint32_t v) {
  uint32_t lo;
  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo) : "r"(v));
  return make_float2(__uint_as_float(lo), __uint_as_float(v & 0xffff0000u));
}

__device__ __forceinline__ float2 dw_ffma2(float2 a, float2 b, float2 c) {
  unsigned long long o;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(o)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&o);
}

// relu / h_swish / identity inline (act_apply's out-of-line GELU path would
// make the epilogue a call site and force register spills)
__device__ __forceinline__ float dw_act(float v, int act) {
  if (act == 1) return fmaxf(v, 0.f);
  if (act == 2) return v * fminf(fmaxf(v + 3.f, 0.f), 6.f) * (1.f / 6.f);
  return v;
}

struct DwRun {
  uint8_t* ring;
  uint64_t* full;
  uint64_t* empty;
  float* part;  // [stages][DW_NCW][64] per-warp SE pool sums
  float* wsm;   // [k*k][64] fp32 weights of the current channel chunk
  long t0, t1;
  int tiles_img, tw_n, C;
};

__device__ __forceinline__ void dw_consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(DW_NCW * 32) : "memory");
}

// Epilogue of one 7-output task: SubnetNorm FMA, activation, bf16 store
// (128 B per warp per pixel), SE pool sums of the stored values.  ReLU runs
// on the packed bf16 pair (rounding commutes with max(., 0)); the pool adds
// with a packed FMA.  FULL: all 7 outputs inside the image (no per-pixel
// bounds test).
template <int ACT, bool FULL, int QW>
__device__ __forceinline__ void dw_epilogue(const float2 (&acc)[QW], float2 sc, float2 sh,
                                            __nv_bfloat16* yr, int C, int nvalid, bool pool,
                                            float2& ps) {
#pragma unroll
  for (int q = 0; q < QW; ++q) {
    if (FULL || q < nvalid) {
      const float2 v = dw_ffma2(acc[q], sc, sh);
      uint32_t u;
      if constexpr (ACT == 1) {
        u = pack_bf16x2(v.x, v.y);
        asm("max.bf16x2 %0, %0, %1;" : "+r"(u) : "r"(0u));
      } else {
        u = pack_bf16x2(dw_act(v.x, ACT), dw_act(v.y, ACT));
      }
      *reinterpret_cast<uint32_t*>(yr + q * C) = u;
      if (pool) ps = dw_ffma2(bf2_to_f2(u), make_float2(1.f, 1.f), ps);
    }
  }
}

template <int ACT, int QW>
__device__ __forceinline__ void dw_store_task(const float2 (&acc)[QW], float2 sc, float2 sh,
                                              __nv_bfloat16* yr, int C, int nvalid, bool pool,
                                              float2& ps) {
  if (nvalid >= QW)
    dw_epilogue<ACT, true, QW>(acc, sc, sh, yr, C, nvalid, pool, ps);
  else
    dw_epilogue<ACT, false, QW>(acc, sc, sh, yr, C, nvalid, pool, ps);
}

// One window row of a task: convert its SEG pixels once, accumulate them
// into output row 0 (filter row wa) and/or output row 1 (filter row wb).
template <int S, int K, int SEG, int LP, int QW, bool A, bool B>
__device__ __forceinline__ void dw_row(const uint32_t* win, const float2* wa, const float2* wb,
                                       float2 (&a)[QW], float2 (&b)[QW]) {
  float2 in[SEG];
#pragma unroll
  for (int q = 0; q < SEG; ++q) in[q] = bf2_to_f2(win[q * LP]);
#pragma unroll
  for (int ss = 0; ss < K; ++ss) {
    if constexpr (A) {
      const float2 wv = wa[ss * 32];
#pragma unroll
      for (int q = 0; q < QW; ++q) a[q] = dw_ffma2(in[q * S + ss], wv, a[q]);
    }
    if constexpr (B) {
      const float2 wv = wb[ss * 32];
#pragma unroll
      for (int q = 0; q < QW; ++q) b[q] = dw_ffma2(in[q * S + ss], wv, b[q]);
    }
  }
}

template <int S, int TW, int TH, int QH, int QW, int K, int CC>
__device__ __forceinline__ void dw_consume(const ConvParams& p, const OpDesc* dp, const DwRun& r) {
  constexpr int IW = (TW - 1) * S + K;        // staged window width (active k)
  constexpr int SEG = (QW - 1) * S + K;       // window pixels one task row reads
  constexpr int LP = CC / 2;                  // lanes per pixel (one bf16x2 each)
  constexpr int HV = 32 / LP;                 // pixels (lane halves) per warp
  constexpr int BPR = TW / (QW * HV);         // tasks per tile row
  static_assert(BPR >= 1, "tile narrower than one warp task");
  constexpr int T = TH / QH * BPR;            // tasks per tile
  constexpr int NIR = (QH - 1) * S + K;       // window rows one task reads
  const int lane = threadIdx.x & 31, cw = (threadIdx.x >> 5) - 1;
  const int lp = lane % LP, half = lane / LP;  // channel pair, output half
  const int off = (p.k_max - K) / 2;          // centre crop of the max kernel
  const __nv_bfloat16* wg = static_cast<const __nv_bfloat16*>(p.w);
  __nv_bfloat16* y = static_cast<__nv_bfloat16*>(p.y);
  const int C = r.C, N = p.n;
  const bool pool = p.pool != nullptr;
  const float2* wsm = reinterpret_cast<const float2*>(r.wsm) + lane;  // [tap][32 lanes]
  float2 sc = make_float2(1.f, 1.f), sh = make_float2(0.f, 0.f);
  // tile coordinates advance incrementally (no divisions in the loop)
  int ti = static_cast<int>(r.t0 % r.tiles_img);
  int n = static_cast<int>((r.t0 / r.tiles_img) % N);
  int chunk = static_cast<int>(r.t0 / r.tiles_img / N);
  int th = ti / r.tw_n, tw = ti - th * r.tw_n;
  // tasks of the CTA's tile stream are dealt round-robin over the warps by
  // the GLOBAL tile index (balanced over time, independent of the grid)
  int jt = static_cast<int>((r.t0 * T) % DW_NCW);
  int cur = -1;
  int st = 0;
  uint32_t ph = 0;
  for (long t = r.t0; t < r.t1; ++t) {
    const int c = chunk * CC + 2 * lp;
    const bool cok = c < C;
    if (chunk != cur) {
      // new channel chunk: all consumer warps reload the k x k x 64 weights
      // (bf16 -> fp32) and their SubnetNorm pair; L2-resident, rare.
      cur = chunk;
      dw_consumer_sync();
      for (int e = threadIdx.x - 32; e < K * K * 32; e += DW_NCW * 32) {
        const int tap = e >> 5, cp = chunk * CC + 2 * ((e & 31) % LP);
        const int rr = tap / K, ss = tap - rr * K;
        uint32_t v = 0;
        if (cp < C)
          v = __ldg(reinterpret_cast<const uint32_t*>(
              wg + (static_cast<long>(rr + off) * p.k_max + ss + off) * p.cout_max + cp));
        reinterpret_cast<float2*>(r.wsm)[e] = bf2_to_f2(v);
      }
      sc = make_float2(1.f, 1.f);
      sh = make_float2(0.f, 0.f);
      if (cok && dp->scale) sc = make_float2(__ldg(dp->scale + c), __ldg(dp->scale + c + 1));
      if (cok && dp->shift) sh = make_float2(__ldg(dp->shift + c), __ldg(dp->shift + c + 1));
      dw_consumer_sync();
    }
    mbar_wait(&r.full[st], ph);
    const uint32_t* tile = reinterpret_cast<const uint32_t*>(r.ring + st * p.dw_stage_bytes);
    float2 ps = make_float2(0.f, 0.f);
    int j = cw - jt;
    if (j < 0) j += DW_NCW;
    for (; j < T; j += DW_NCW) {
      const int orow = j / BPR * QH, ocol0 = (j % BPR) * QW * HV + half * QW;
      float2 acc[QH][QW];
#pragma unroll
      for (int h = 0; h < QH; ++h)
#pragma unroll
        for (int q = 0; q < QW; ++q) acc[h][q] = make_float2(0.f, 0.f);
      const uint32_t* win = tile + (orow * S * IW + ocol0 * S) * LP + lp;
      // window row ir feeds output row h through filter row ir - h*S.  Three
      // rolled phases (rows feeding only the first output row, both, only
      // the second) keep the filter-row choice branch-free and one converted
      // window row live at a time (<= 128 registers at 512 threads).
      const float2* wrow = wsm;
      if constexpr (QH == 1) {
#pragma unroll 1
        for (int ir = 0; ir < K; ++ir, win += IW * LP, wrow += K * 32)
          dw_row<S, K, SEG, LP, QW, true, false>(win, wrow, wrow, acc[0], acc[QH - 1]);
      } else {
#pragma unroll 1
        for (int ir = 0; ir < S; ++ir, win += IW * LP, wrow += K * 32)
          dw_row<S, K, SEG, LP, QW, true, false>(win, wrow, wrow, acc[0], acc[QH - 1]);
#pragma unroll 1
        for (int ir = S; ir < K; ++ir, win += IW * LP, wrow += K * 32)
          dw_row<S, K, SEG, LP, QW, true, true>(win, wrow, wrow - S * K * 32, acc[0], acc[QH - 1]);
#pragma unroll 1
        for (int ir = K; ir < NIR; ++ir, win += IW * LP, wrow += K * 32)
          dw_row<S, K, SEG, LP, QW, false, true>(win, wrow, wrow - S * K * 32, acc[0], acc[QH - 1]);
      }
      const int ow0 = tw * TW + ocol0;
#pragma unroll
      for (int h = 0; h < QH; ++h) {
        const int oh = th * TH + orow + h;
        if (cok && oh < p.ho) {
          __nv_bfloat16* yr = y + (static_cast<long>(n * p.ho + oh) * p.wo + ow0) * dp->ldo + c;
          const int nvalid = p.wo - ow0;
          if (p.act == 1)
            dw_store_task<1, QW>(acc[h], sc, sh, yr, dp->ldo, nvalid, pool, ps);
          else if (p.act == 2)
            dw_store_task<2, QW>(acc[h], sc, sh, yr, dp->ldo, nvalid, pool, ps);
          else
            dw_store_task<0, QW>(acc[h], sc, sh, yr, dp->ldo, nvalid, pool, ps);
        }
      }
    }
    if (pool) {
      if (HV == 2) {  // both lane halves summed the same channels
        ps.x += __shfl_xor_sync(0xffffffffu, ps.x, 16);
        ps.y += __shfl_xor_sync(0xffffffffu, ps.y, 16);
      }
      if (lane < LP) *reinterpret_cast<float2*>(r.part + (st * DW_NCW + cw) * DW_CC + 2 * lane) = ps;
    }
    // one arrival per warp (count = DW_NCW): per-lane arrivals on one
    // mbarrier serialise in the shared-memory atomic unit.  __syncwarp
    // orders the lanes' part[] stores (and their window reads, already
    // consumed) before lane 0's release.
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[st]);
    if (++st == p.dw_stages) {
      st = 0;
      ph ^= 1;
    }
    jt += T - (T >= DW_NCW ? DW_NCW : 0);
    if (jt >= DW_NCW) jt -= DW_NCW;
    if (++tw == r.tw_n) {
      tw = 0;
      if (++th * r.tw_n == r.tiles_img) {
        th = 0;
        if (++n == N) {
          n = 0;
          ++chunk;
        }
      }
    }
  }
}

// Producer warp: one TMA box per tile; when the stage comes back, the
// consumer warps' SE sums of the tile that used it are added in fixed order.
template <int S, int TW, int TH, int CC>
__device__ __forceinline__ void dw_produce(const ConvParams& p, const OpDesc* dp, const DwRun& r,
                                           int k) {
  const int lane = threadIdx.x & 31;
  const CUtensorMap* map = &dp->amap;
  const int pad = k / 2;
  const uint32_t bytes =
      static_cast<uint32_t>(((TH - 1) * S + k) * ((TW - 1) * S + k) * CC * 2);
  const int nst = p.dw_stages;
  auto flush = [&](long t, int st) {  // SE partial of tile t (its stage st is free)
    const int ti = static_cast<int>(t % r.tiles_img);
    const long rest = t / r.tiles_img;
    const int n = static_cast<int>(rest % p.n);
    const int c = static_cast<int>(rest / p.n) * CC + 2 * lane;
    if (2 * lane >= CC) return;
    if (c >= r.C) return;
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int w = 0; w < DW_NCW; ++w) {
      const float2 v = *reinterpret_cast<const float2*>(r.part + (st * DW_NCW + w) * DW_CC + 2 * lane);
      s.x += v.x;
      s.y += v.y;
    }
    *reinterpret_cast<float2*>(p.pool + (static_cast<long>(n) * r.tiles_img + ti) * p.pool_ld + c) = s;
  };
  if (lane == 0) tma_prefetch(map);
  int st = 0;
  uint32_t ph = 0;
  for (long t = r.t0; t < r.t1; ++t) {
    mbar_wait(&r.empty[st], ph ^ 1);
    if (p.pool && t - nst >= r.t0) flush(t - nst, st);
    __syncwarp();
    if (lane == 0) {
      const int ti = static_cast<int>(t % r.tiles_img);
      const long rest = t / r.tiles_img;
      const int n = static_cast<int>(rest % p.n);
      const int chunk = static_cast<int>(rest / p.n);
      const int th = ti / r.tw_n, tw = ti - th * r.tw_n;
      mbar_arrive_expect_tx(&r.full[st], bytes);
      tma_load_4d(r.ring + st * p.dw_stage_bytes, map, &r.full[st], chunk * CC,
                  tw * TW * S - pad, th * TH * S - pad, n);
    }
    if (++st == nst) {
      st = 0;
      ph ^= 1;
    }
  }
  if (!p.pool) return;
  // drain: the last min(nst, count) tiles
  const long first = r.t1 - nst > r.t0 ? r.t1 - nst : r.t0;
  for (long t = first; t < r.t1; ++t) {
    const long u = (t - r.t0) / nst;
    const int s2 = static_cast<int>((t - r.t0) % nst);
    mbar_wait(&r.empty[s2], static_cast<uint32_t>(u & 1));
    flush(t, s2);
  }
}

template <int S, int TW, int TH, int QH, int CC = DW_CC, int QW = DW_QW>
__global__ void __launch_bounds__(DW_THREADS, 1) dw_tma_kernel(const __grid_constant__ ConvParams p) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  const int nst = p.dw_stages;
  DwRun r;
  r.ring = dsm;
  r.full = reinterpret_cast<uint64_t*>(dsm + nst * p.dw_stage_bytes);
  r.empty = r.full + nst;
  r.part = reinterpret_cast<float*>(r.empty + nst);
  r.wsm = r.part + nst * DW_NCW * DW_CC;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_init(&r.full[i], 1);
      mbar_init(&r.empty[i], DW_NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const OpDesc* dp = desc_ptr(p.row, p.fixed, p.op);
  const int C = dp->cout, k = dp->k;
  r.tw_n = (p.wo + TW - 1) / TW;
  r.tiles_img = ((p.ho + TH - 1) / TH) * r.tw_n;
  r.C = C;
  const long total = static_cast<long>((C + CC - 1) / CC) * p.n * r.tiles_img;
  const long per = (total + gridDim.x - 1) / gridDim.x;
  r.t0 = blockIdx.x * per;
  r.t1 = r.t0 + per < total ? r.t0 + per : total;
  if (r.t0 >= r.t1) return;
  if (threadIdx.x < 32) {
    dw_produce<S, TW, TH, CC>(p, dp, r, k);
    return;
  }
  if (k == 3)  // HBM-bound: 7-wide tasks (14-wide measured 5% slower at k = 3)
    dw_consume<S, TW, TH, QH, DW_QW, 3, CC>(p, dp, r);
  else if (k == 5)
    dw_consume<S, TW, TH, QH, QW, 5, CC>(p, dp, r);
  else
    dw_consume<S, TW, TH, QH, QW, 7, CC>(p, dp, r);
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFnD = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFnD dw_encoder() {
  static EncodeTiledFnD enc = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFnD>(ptr);
    return static_cast<EncodeTiledFnD>(nullptr);
  }();
  return enc;
}

bool dw_supported(int k_max, int k, int stride) {
  return stride >= 1 && stride <= 2 && k_max <= 7 && (k == 3 || k == 5 || k == 7) && k <= k_max;
}

// Input window map of one depthwise op as THIS subnet lays its activation
// out: [n][h][w][c] bf16 (c active channels), box {64 ch, (TW-1)*S + k,
// (7-1)*S + k, 1} for the active k; out-of-bounds (padding, channel tail)
// is TMA zero fill.
bool dw_narrow(int c_max, int stride, int wo) {
  static const bool off = getenv("SSN_DW_NO_NARROW") != nullptr;  // A/B switch
  return !off && c_max <= DW_CC_NARROW && stride == 1 && wo > 7;
}

int make_dw_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int c, int ld, int k,
                    int stride, int wo, int c_max) {
  EncodeTiledFnD enc = dw_encoder();
  if (!enc || (c & 7) != 0 || (ld & 7) != 0 || !dw_supported(7, k, stride)) return -1;
  const DwShape g = dw_shape(stride, wo);
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(w) * ld * 2,
                           static_cast<cuuint64_t>(h) * w * ld * 2};
  const cuuint32_t cc = dw_narrow(c_max, stride, wo) ? DW_CC_NARROW : DW_CC;
  cuuint32_t box[4] = {cc, static_cast<cuuint32_t>((g.tw - 1) * stride + k),
                       static_cast<cuuint32_t>((g.th - 1) * stride + k), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  static const int promo = [] {  // A/B switch: L2 promotion of the window rows
    const char* e = getenv("SSN_DW_L2PROMO");
    return e ? atoi(e) : 256;
  }();
  const CUtensorMapL2promotion pr = promo == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

static int dw_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int S, int TW, int TH, int QH, int CC = DW_CC, int QW = DW_QW>
static cudaError_t launch_dw_inst(const ConvParams& p, size_t smem, int grid, cudaStream_t s) {
  static const cudaError_t attr = cudaFuncSetAttribute(
      dw_tma_kernel<S, TW, TH, QH, CC, QW>, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_SMEM_MAX);
  if (attr != cudaSuccess) return attr;
  return launch_pdl(dw_tma_kernel<S, TW, TH, QH, CC, QW>, dim3(grid), dim3(DW_THREADS), smem, s, 1, p);
}

// p: the op's max geometry (k_max, cout_max) + graph-baked batch; the active
// width, kernel size, SubnetNorm row and input map come from the OpDesc.
cudaError_t launch_dw_bf16(const ConvParams& p0, cudaStream_t s) {
  if (p0.k_max > 7 || p0.k_max < 3 || (p0.stride != 1 && p0.stride != 2))
    return cudaErrorInvalidValue;
  ConvParams p = p0;
  const DwShape g = dw_shape(p.stride, p.wo);
  const bool narrow = dw_narrow(p.cout_max, p.stride, p.wo);
  const int cc = narrow ? DW_CC_NARROW : DW_CC;
  const int bh = (g.th - 1) * p.stride + p.k_max, bw = (g.tw - 1) * p.stride + p.k_max;
  p.dw_stage_bytes = (bh * bw * cc * 2 + 127) & ~127;
  const int per_stage = p.dw_stage_bytes + 16 + DW_NCW * DW_CC * 4;
  p.dw_stages = (DW_SMEM_MAX - DW_WSM_BYTES) / per_stage;
  if (p.dw_stages > DW_MAX_STAGES) p.dw_stages = DW_MAX_STAGES;
  if (p.dw_stages < 2) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(p.dw_stages) * per_stage + DW_WSM_BYTES;
  const long tiles = static_cast<long>(cdiv(p.cout_max, cc)) * p.n *
                     dw_tiles_per_image(p.stride, p.ho, p.wo);
  const int grid = static_cast<int>(tiles < dw_sm_count() ? tiles : dw_sm_count());
  if (narrow) return launch_dw_inst<1, 14, 14, 2, DW_CC_NARROW>(p, smem, grid, s);
  if (p.stride == 2) return launch_dw_inst<2, 7, 7, 1>(p, smem, grid, s);
  // 14-wide warp tasks for k = 5 / 7 (each converted window pixel feeds up
  // to 14 outputs x 2 rows): FFMA2 share of the inner loop 63% -> 73% for the
  // FMA-pipe-bound layers (56 px k7 420 -> 399 us at bs256); k = 3 keeps
  // 7-wide tasks; SSN_DW_QW7 = 7-wide everywhere (A/B switch)
  static const bool qw7 = getenv("SSN_DW_QW7") != nullptr;
  if (g.tw == 14 && !qw7) return launch_dw_inst<1, 14, 14, 2, DW_CC, 14>(p, smem, grid, s);
  return g.tw == 14 ? launch_dw_inst<1, 14, 14, 2>(p, smem, grid, s)
                    : launch_dw_inst<1, 7, 7, 1>(p, smem, grid, s);
}

}  // namespace ssn
