// conv_halo.cu — stride-1 k x k WeightSlice convolution as a "shifted-window"
// implicit GEMM on tcgen05 (sm_100a), for the narrow early layers of the
// CNN supernets (OFA-ResNet50 stem and stage-1 3x3 convs: 24-88 channels at
// 56-112 px).
//
// Why a second conv kernel: with TMA im2col every K block of
// conv_tc re-reads the 128-pixel A tile per filter tap, 9x for a 3x3, and a
// narrow N (cout <= 96) gives the tensor core only ~200 cycles of work per
// 28 KB K block.  The ring then cannot hold enough bytes to cover the TMA
// latency (measured: MMA warp waiting on data 67% of the time; 0.07-0.17 of
// roofline on these layers).  Here:
//  * the whole active weight slice (k_a^2 x cin_a x cout_a, <= ~160 KB) is
//    loaded into shared memory ONCE per CTA and stays resident;
//  * output positions are taken in padded-width order (HaloGeom): tap (r, s)
//    of position p reads window pixel p + r*Wp + s, so ONE halo window per
//    32-channel block feeds all k^2 taps — each tap's A operand is the same
//    smem window at a row offset.  That needs the no-swizzle K-major UMMA
//    layout ([8-channel chunk][pixel][8] — 16-byte rows, any 16-byte offset
//    is a valid descriptor start), which a 5-D TMA box {8 ch, Wp, R, 1, 4
//    chunks} over the NHWC activation produces directly (the channel-chunk
//    dimension has a 16-byte global stride and is outermost in the box);
//  * A traffic drops from 9 x 128 to ~(R x Wp) pixels per tile, and the
//    padding columns/rows are TMA zero fill.
// Garbage positions (the k-1 padding columns of each row, rows past H) are
// computed and dropped by the epilogue (3.4% of MMA work at 56 px).
// Warp roles as conv_tc: warp 0 TMA producer, warp 9 MMA issuer (one
// elected lane), warps 1-12 epilogue in three groups of 4 taking alternate
// tiles; accumulators in a TMEM ring.  The epilogue is row-per-lane (no
// smem staging: shared memory belongs to the resident weights).
#include <cstdio>
#include <cstdlib>

#include "device.cuh"

namespace ssn {

constexpr int HL_EPI_WARPS = 12;  // 3 groups x 4 TMEM lane quarters
constexpr int HL_EPI_GROUPS = HL_EPI_WARPS / 4;
constexpr int HL_MMA_WARP = 1 + HL_EPI_WARPS;
constexpr int HL_THREADS = (HL_MMA_WARP + 1) * 32;
constexpr int HL_SMEM_MAX = 232448;  // 227 KB opt-in
constexpr int HL_CB = 32;            // channels per A stage (two K=16 steps)
constexpr int HL_MAX_STAGES = 8;

__global__ void __launch_bounds__(HL_THREADS, 1)
    conv_halo_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

  const OpDesc* dp = desc_ptr(p.row, p.fixed, p.op);
  const OpDims d = load_desc(p.row, p.fixed, p.op);
  const int d_wrows = dp->wrows;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint64_t* full = bars;                         // [HL_MAX_STAGES]
  uint64_t* empty = full + HL_MAX_STAGES;
  uint64_t* tfull = empty + HL_MAX_STAGES;       // [4]
  uint64_t* tempty = tfull + 4;                  // [4]
  uint64_t* bfull = tempty + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 2);
  // barriers and TMEM need no descriptor field: they run while the row ->
  // descriptor loads are in flight (as conv_tc)
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index through shfl: the compiler then knows it is warp-uniform, so
  // role branches stay uniform and MMA/TMA operands live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (tid == 0) {
    for (int s = 0; s < HL_MAX_STAGES; ++s) {  // (ST is descriptor-dependent)
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 4; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // the owning group's warps
    }
    mbar_init(bfull, 1);
    fence_mbar_init();
  }
  if (warp == HL_MMA_WARP) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ka = d.k, pad = d.pad, koff = (p.k_max - ka) / 2;
  const HaloGeom hg = halo_geom(p.w_, ka);
  const int wp = hg.wp, rt = hg.rt, R = hg.r;
  const int tpi = (p.h + rt - 1) / rt;  // tiles per image
  const int tiles = p.n * tpi;
  const bool idle = static_cast<int>(blockIdx.x) >= tiles;
  const int cin16 = (d.cin + 15) & ~15;
  const int ncb = (cin16 + HL_CB - 1) / HL_CB;
  const int bn = (d.cout + 15) & ~15;  // MMA N: the whole active cout (<= 128)
  // 3 accumulators of 128 columns: the 3 epilogue groups take tiles in
  // turn, so accumulator a is always drained by group a (a group never waits
  // on an mbarrier phase belonging to an older use of another group's tile)
  const int acc_cols = 128;
  const int nacc = HL_EPI_GROUPS;

  // shared memory: [resident B][A ring][barriers].  Both operands are
  // 64B-swizzled K-major: rows of 32 channels (64 B), 8-row atoms of 512 B.
  // B block (tap, 32-ch block cb) = hb_rows rows; an A stage = one halo
  // window of R * Wp pixel rows for one 32-channel block.  A tap's A operand
  // starts (r*Wp + s) rows into the window: the tensor core applies the
  // swizzle on absolute smem address bits, so any 64-B row offset is a legal
  // start (verified exact on B200: tools/ubench/sw128_shift.cu -DSW64).
  // Resident B at the ACTIVE width when the subnet row carries its own halo
  // weight map (wmap slot, box rows = wrows = the 16-rounded active cout):
  // only the active 32-channel blocks and rows are loaded, and the shared
  // memory a narrow subnet leaves free deepens the window ring (e.g. OFA-R50
  // mid at 56 px: 74 of the max shape's 166 KB, 3 -> 8 stages).  A row
  // without one (operator API) uses the graph's max-width map.
  const bool own_b = d_wrows == bn;
  const CUtensorMap* wm = own_b ? &dp->wmap : &wmap;
  const int ncb_b = own_b ? ncb : p.hb_chunks;                          // resident 32-ch blocks
  const uint32_t b_blk = static_cast<uint32_t>(own_b ? bn : p.hb_rows) * 64;  // one (tap, cb) block
  const uint32_t b_bytes = b_blk * static_cast<uint32_t>(ka * ka * ncb_b);
  const uint32_t a_box = static_cast<uint32_t>(R * wp) * 64;           // TMA box bytes
  const uint32_t a_stage = (a_box + 1023) & ~1023u;                    // swizzle-atom aligned
  // [barriers + SubnetNorm vectors: 2 KB][resident B][A ring]
  // SubnetNorm scale / shift of this op (cout <= 128), staged once: the
  // row-per-lane epilogue reads all columns per lane, and per-column global
  // loads issued right before their FMAs serialised an L1/L2 round trip per
  // 8 columns (ncu: the epilogue's FFMAs were the top stall site)
  float* sn = reinterpret_cast<float*>(smem + 1024);  // [2][128]
  uint8_t* sB = smem + 2048;
  uint8_t* sA = sB + ((b_bytes + 1023) & ~1023u);
  int ST = static_cast<int>((static_cast<uint32_t>(p.h_smem) - 2048u - ((b_bytes + 1023) & ~1023u)) /
                            a_stage);
  ST = ST > HL_MAX_STAGES ? HL_MAX_STAGES : ST;
  if (tid == 0 && !idle) {
    tma_prefetch(wm);
    tma_prefetch(&dp->amap);
  }

  // PDL: the resident weights are static and load before griddepcontrol.wait
  // (overlapping the predecessor's tail); activations only after it
  pdl_trigger();
  // SSN_TC_DEBUG & 32: per-role cycle accounting of CTA 0 (profiling only)
  const bool prof = (p.dbg & 32) && blockIdx.x == 0;
  long long w_wait = 0, w_wait2 = 0;
  const long long t_begin = prof ? clock64() : 0;
#define HL_WAIT(acc, bar, ph)                 \
  if (prof) {                                 \
    const long long t0_ = clock64();          \
    mbar_wait(bar, ph);                       \
    acc += clock64() - t0_;                   \
  } else {                                    \
    mbar_wait(bar, ph);                       \
  }

  if (idle) {
    // no tile for this CTA: straight to the teardown
  } else if (warp == 0) {
    // ============================================================ producer
    const bool leader = elect_one();
    if (leader && (p.dbg & 8)) {  // profiling: no weight load
      mbar_arrive(bfull);
    } else if (leader) {
      // the active k_a x k_a centre crop of the max-shape weights, all 32-ch
      // blocks of the max shape (channels past cin_a meet zero-filled A)
      mbar_arrive_expect_tx(bfull, b_bytes);
      for (int r = 0; r < ka; ++r)
        for (int s = 0; s < ka; ++s)
          for (int cb = 0; cb < ncb_b; ++cb)
            tma_load_3d(sB + ((r * ka + s) * ncb_b + cb) * b_blk, wm, bfull, cb * HL_CB,
                        (r + koff) * p.k_max + (s + koff), 0);
    }
    const CUtensorMap* amap = &dp->amap;
    __syncwarp();
    pdl_wait();
    int g = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int img = t / tpi;
      const int r0 = (t - img * tpi) * rt;
      for (int cb = 0; cb < ncb; ++cb, ++g) {
        const int s = g % ST;
        HL_WAIT(w_wait, &empty[s], ((g / ST) & 1) ^ 1);
        if (leader) {
          if (p.dbg & 4) {  // profiling: no A loads
            mbar_arrive(&full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], a_box);  // box bytes (the stage is padded)
            tma_load_4d(sA + s * a_stage, amap, &full[s], cb * HL_CB, -pad, r0 - pad, img);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == HL_MMA_WARP) {
    // ============================================================ MMA issuer
    // Converged warp, elected lane issues (tc_mma_bf16_elect); descriptors
    // are a per-stage / per-block base plus 16-byte-unit offsets.
    const uint32_t idesc = umma_idesc_bf16(bn);
    const uint64_t a_base = umma_desc_sw64(smem_u32(sA));
    const uint64_t b_base = umma_desc_sw64(smem_u32(sB));
    const uint32_t a_st16 = a_stage >> 4;
    const uint32_t b_tap16 = (ncb_b * b_blk) >> 4, b_cb16 = b_blk >> 4;
    constexpr uint32_t ks16 = 2;  // K=16 step inside a 64-B row: +32 B
    HL_WAIT(w_wait, bfull, 0);
    tc_fence_after();
    int g = 0, i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int a = i % nacc;
      HL_WAIT(w_wait2, &tempty[a], ((i / nacc) & 1) ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem + a * acc_cols;
      for (int cb = 0; cb < ncb; ++cb, ++g) {
        const int s = g % ST;
        HL_WAIT(w_wait, &full[s], (g / ST) & 1);
        tc_fence_after();
        const int nks = min(HL_CB / 16, (cin16 - cb * HL_CB) / 16);
        const uint64_t ad = a_base + static_cast<uint64_t>(s * a_st16);
        const uint64_t bd = b_base + static_cast<uint64_t>(cb * b_cb16);  // + tap * b_tap16 below
        if (p.dbg & 2) {  // profiling: no MMAs
        } else if (ka == 3 && nks == 2) {  // OFA-R50: fully unrolled 3x3 taps, full block
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tc_mma_bf16_elect(acc, ad + static_cast<uint64_t>((r * wp + c) * 4 + j * ks16),
                                  bd + static_cast<uint64_t>((r * 3 + c) * b_tap16 + j * ks16),
                                  idesc, (cb | r | c | j) != 0 ? 1u : 0u);
        } else {
          for (int r = 0; r < ka; ++r)
            for (int c = 0; c < ka; ++c)
              for (int j = 0; j < nks; ++j)
                tc_mma_bf16_elect(acc, ad + static_cast<uint64_t>((r * wp + c) * 4 + j * ks16),
                                  bd + static_cast<uint64_t>((r * ka + c) * b_tap16 + j * ks16),
                                  idesc, (cb | r | c | j) != 0 ? 1u : 0u);
        }
        tc_commit_elect(&empty[s]);
        if (cb + 1 == ncb) tc_commit_elect(&tfull[a]);
        __syncwarp();
      }
    }
  } else {
    // ============================================================ epilogue
    // Lane L of warp w drains TMEM row 32*(w%4) + L = one padded output
    // position; positions in the padding columns / past H are dropped.
    for (int i = tid - 32; i < 128; i += HL_EPI_WARPS * 32) {  // static: before the PDL wait
      sn[i] = (d.scale && i < d.cout) ? __ldg(d.scale + i) : 1.f;
      sn[128 + i] = (d.shift && i < d.cout) ? __ldg(d.shift + i) : 0.f;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(HL_EPI_WARPS * 32) : "memory");
    pdl_wait();  // the residual is the predecessors' output
    const int quarter = warp & 3;
    const int group = (warp - 1) >> 2;
    const int p_row = quarter * 32 + lane;
    const int oh_l = p_row / wp, ow = p_row - oh_l * wp;
    const int nch = (d.cout + 31) / 32;
    int i = group;
    for (int t = blockIdx.x + group * static_cast<int>(gridDim.x); t < tiles;
         t += HL_EPI_GROUPS * static_cast<int>(gridDim.x), i += HL_EPI_GROUPS) {
      const int a = i % nacc;
      const int img = t / tpi;
      const int oh = (t - img * tpi) * rt + oh_l;
      const bool ok = p_row < rt * wp && ow < p.wo && oh < p.ho;
      const size_t m = (static_cast<size_t>(img) * p.ho + oh) * p.wo + ow;
      const size_t rowoff = m * d.ldo;
      HL_WAIT(w_wait, &tfull[a], static_cast<uint32_t>(i / nacc) & 1);
      tc_fence_after();
      for (int c = 0; c < nch; ++c) {
        float v[32];
        tmem_ld32(tmem + a * acc_cols + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
        if (c + 1 == nch) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);
        }
        if (!ok || (p.dbg & 1)) continue;
        uint4 rv[4];
        if (p.res) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (c * 32 + 8 * j < d.cout)
              rv[j] = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.res) +
                                                           rowoff + c * 32 + 8 * j));
        }
        uint4 pk_lo = make_uint4(0u, 0u, 0u, 0u);
        bool paired = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = c * 32 + 8 * j;
          if (col >= d.cout) break;
          float sc[8], sh[8];
          {
            const float4 s0 = *reinterpret_cast<const float4*>(sn + col);
            const float4 s1 = *reinterpret_cast<const float4*>(sn + col + 4);
            const float4 h0 = *reinterpret_cast<const float4*>(sn + 128 + col);
            const float4 h1 = *reinterpret_cast<const float4*>(sn + 128 + col + 4);
            sc[0] = s0.x; sc[1] = s0.y; sc[2] = s0.z; sc[3] = s0.w;
            sc[4] = s1.x; sc[5] = s1.y; sc[6] = s1.z; sc[7] = s1.w;
            sh[0] = h0.x; sh[1] = h0.y; sh[2] = h0.z; sh[3] = h0.w;
            sh[4] = h1.x; sh[5] = h1.y; sh[6] = h1.z; sh[7] = h1.w;
          }
          float o[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) o[q] = v[8 * j + q] * sc[q] + sh[q];
          float r8[8];
          if (p.res) {
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[j]);
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
          uint4 pk;
          pk.x = pack_bf16x2(o[0], o[1]);
          pk.y = pack_bf16x2(o[2], o[3]);
          pk.z = pack_bf16x2(o[4], o[5]);
          pk.w = pack_bf16x2(o[6], o[7]);
          __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(p.y) + rowoff + col;
          // row-per-lane stores: pair two 8-column groups into one 32-byte
          // (full-sector) store where the row segment is 32-byte aligned
          if ((j & 1) == 0 && col + 16 <= d.cout && ((rowoff + col) & 15) == 0) {
            pk_lo = pk;
            paired = true;
          } else if ((j & 1) == 1 && paired) {
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(yp - 8),
                         "r"(pk_lo.x), "r"(pk_lo.y), "r"(pk_lo.z), "r"(pk_lo.w), "r"(pk.x), "r"(pk.y),
                         "r"(pk.z), "r"(pk.w)
                         : "memory");
            paired = false;
          } else {
            *reinterpret_cast<uint4*>(yp) = pk;
          }
        }
      }
    }
  }
#undef HL_WAIT
  if (prof && lane == 0 && (warp == 0 || warp == HL_MMA_WARP || warp == 1))
    printf("[conv_tc prof] tiles=%d nk=%d warp=%d total=%lld wait=%lld wait2=%lld\n", tiles, ncb,
           warp, clock64() - t_begin, w_wait, w_wait2);
  tc_fence_before();
  __syncthreads();
  if (warp == HL_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFnH = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFnH tiled_encoder() {
  static EncodeTiledFnH fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFnH>(ptr);
    return static_cast<EncodeTiledFnH>(nullptr);
  }();
  return fn;
}

static int halo_b_rows(int cout_max) { return (cout_max + 15) / 16 * 16; }
static int halo_b_chunks(int cin_max) { return (cin_max + HL_CB - 1) / HL_CB; }  // 32-ch blocks

// Resident-B and ring sizing for an op's MAX shape (every subnet fits in it).
static void halo_sizes(int w, int k_max, int cin_max, int cout_max, long* b_bytes, long* a_stage) {
  const HaloGeom g = halo_geom(w, k_max);
  *b_bytes = static_cast<long>(k_max) * k_max * halo_b_chunks(cin_max) * halo_b_rows(cout_max) * 64;
  *a_stage = (static_cast<long>(g.r) * g.wp * 64 + 1023) & ~1023L;
}

static int halo_stages(int w, int k_max, int cin_max, int cout_max) {
  long bb, as;
  halo_sizes(w, k_max, cin_max, cout_max, &bb, &as);
  const long avail = HL_SMEM_MAX - 1024 - 2048 - ((bb + 1023) & ~1023L);
  const long st = avail / as;
  return static_cast<int>(st > HL_MAX_STAGES ? HL_MAX_STAGES : st);
}

// The shifted-window kernel serves stride-1 odd k x k convs whose max-shape
// weight slice fits shared memory with >= 2 ring stages, cout <= 256.
bool halo_eligible(int h, int w, int k_max, int stride, int cin_max, int cout_max) {
  static const bool off = [] {
    const char* e = getenv("SSN_NO_HALO");  // A/B switch for profiling
    return e && atoi(e) != 0;
  }();
  if (off) return false;
  if (stride != 1 || (k_max & 1) == 0 || k_max < 3 || cout_max > 128) return false;
  if (w < 14 || h < 2) return false;
  const HaloGeom g = halo_geom(w, k_max);
  if (g.wp > 256 || g.r > 256) return false;
  return halo_stages(w, k_max, cin_max, cout_max) >= 2;
}

// A operand: [n][h][w][cin_a] NHWC bf16, box {32 ch, Wp, R, 1} with 64-byte
// swizzle: one halo window of one 32-channel block as 64-B pixel rows.
int make_halo_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld, int k) {
  EncodeTiledFnH enc = tiled_encoder();
  if (!enc) return -1;
  const HaloGeom g = halo_geom(w, k);
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cin), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(w) * ld * 2,
                           static_cast<cuuint64_t>(h) * w * ld * 2};
  cuuint32_t box[4] = {HL_CB, static_cast<cuuint32_t>(g.wp), static_cast<cuuint32_t>(g.r), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

// B operand: max-shape KRSC [cout][taps][cin_store], box {32 ch, 1 tap, rows}
// with 64-byte swizzle: one (tap, 32-channel block) of the weight slice.
int make_halo_weight_map(CUtensorMap* map, const void* wgt, int cin_store, int taps, int cout,
                         int rows, int /*chunks*/) {
  EncodeTiledFnH enc = tiled_encoder();
  if (!enc) return -1;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cin_store), static_cast<cuuint64_t>(taps),
                        static_cast<cuuint64_t>(cout)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cin_store) * 2,
                           static_cast<cuuint64_t>(taps) * cin_store * 2};
  cuuint32_t box[3] = {HL_CB, 1, static_cast<cuuint32_t>(rows)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(wgt), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t init_conv_halo() {
  return cudaFuncSetAttribute(conv_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              HL_SMEM_MAX);
}

// p: geometry of the op's max shape (k_max, cin_max = weight cin_store,
// cout_max); the active subnet's extents and A map come from its OpDesc.
cudaError_t launch_conv_halo(ConvParams p, const void* wgt, int cin_store, int taps,
                             cudaStream_t s) {
  static const int dbg = [] {
    const char* e = getenv("SSN_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  p.dbg = dbg;
  p.hb_rows = halo_b_rows(p.cout_max);
  p.hb_chunks = halo_b_chunks(p.cin_max);
  p.h_stages = halo_stages(p.w_, p.k_max, p.cin_max, p.cout_max);
  if (p.h_stages < 2) return cudaErrorInvalidValue;
  CUtensorMap wmap;
  if (make_halo_weight_map(&wmap, wgt, cin_store, taps, p.cout_max, p.hb_rows, p.hb_chunks) != 0)
    return cudaErrorInvalidValue;
  long bb, as;
  halo_sizes(p.w_, p.k_max, p.cin_max, p.cout_max, &bb, &as);
  // the whole opt-in shared memory: a narrow subnet turns the part of the
  // max-shape B region it does not use into extra ring stages
  (void)bb;
  (void)as;
  const long smem = HL_SMEM_MAX;
  p.h_smem = static_cast<int>(smem - 1024);
  const HaloGeom g = halo_geom(p.w_, p.k_max);
  const long tiles = static_cast<long>(p.n) * ((p.h + g.rt - 1) / g.rt);
  const int grid = static_cast<int>(tiles < sm_count() ? tiles : sm_count());
  return launch_pdl(conv_halo_kernel, dim3(grid), dim3(HL_THREADS), smem, s, 1, p, wmap);
}

}  // namespace ssn
