// conv_tc.cu — WeightSlice implicit-GEMM convolution on the 5th-gen tensor
// cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   Y[M, cout_a] = act( SubnetNorm_i( im2col(X)[M, K_a] . W[:cout_a, K_a]^T ) (+ res) )
//   M = n * ho * wo, K_a = k_a^2 * cin_a  (PAPER.md:497-502 WeightSlice,
//   PAPER.md:472-481 SubnetNorm folded into the epilogue).
//
// Design:
//  * Both operands move by TMA:
//      A (activations): TMA im2col mode — one cp.async.bulk.tensor.4d.im2col
//        per K block loads 128 consecutive output pixels x 64 channels of one
//        filter tap; padding, channel tails (> cin_a) and the batch tail are
//        TMA zero fill.  The map is per (subnet, op): it encodes the subnet's
//        compact activation layout (cin_a-channel stride) and lives in the
//        actuated subnet's device OpDesc row, read in place by the TMA unit.
//      B (weights): the max-shape KRSC tensor is stored ONCE; a 3-D tiled map
//        over [cout_max][k_max^2][cin_max] loads {64 ch, 1 tap, bn} boxes of
//        its LEADING slice — no copy of any slice ever exists.
//    Both land 128B-swizzled (SW128 K-major), the layout tcgen05.mma reads.
//  * Persistent and warp-specialised: one CTA per SM walks a static tile
//    schedule; warp 0 produces, warp 9 issues tcgen05.mma, warps 1-8 drain.
//    Producer and MMA loops run warp-wide and elect one lane to issue, so the
//    descriptors stay warp-uniform (a lane-0-only loop wrapped every
//    UTCHMMA/UTMALDG in a divergent R2UR waterfall: 500 vs 360 cycles per
//    K block measured, tools/ubench/tc_loop.cu).
//  * A ring stage holds KPS K blocks: one stage = one commit -> producer ->
//    full-barrier -> MMA round trip, ~520 cycles whatever N (tools/ubench/
//    mma2_rate.cu), so long-K layers take two K blocks per stage.
//  * Accumulators live in a TMEM ring (NACC buffers of BN_MAX fp32 columns),
//    so several tiles are in flight between MMA and epilogue.
//  * Epilogue: three groups of 4 warps stripe every tile's 32-column chunks;
//    each warp tcgen05.ld's 32 TMEM lanes x 32 columns.  Default: row per
//    lane, SubnetNorm / residual / activation in registers, the bf16 chunk
//    written once into a 64B-swizzled box and stored by one TMA store
//    (OpDesc.ymap).  Split-K partials, fp32 logits, ragged widths and global
//    residuals: transpose through padded smem, coalesced 64-byte row segments.
//  * Subnet extents (cin_a, cout_a, k_a, SubnetNorm row, activation map) come
//    from the actuated subnet's descriptor, so one graph-captured launch
//    serves every subnet; the tile count follows cout_a on the device.
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "device.cuh"

namespace ssn {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_EPI_WARPS = 12;  // 3 groups x 4 TMEM lane quarters
constexpr int TC_EPI_GROUPS = TC_EPI_WARPS / 4;
// Warp roles.  Warpgroup 0 = warps 0, 2, 3 TMA producers, warp 1 MMA issuer;
// warpgroups 1-3 = the 12 epilogue warps.  One thread sustains only ~1 TMA
// box per ~360 cycles (wait + expect_tx + issue; tools/ubench/tma_rate.cu:
// 45 B/cycle with 16 KB boxes from one thread, 76 with two), less than a K
// block of N=128 MMAs, so the three producers take K blocks round-robin and
// each loads both operands of its blocks.  512 threads cap registers at
// 128: the epilogue keeps no register prefetch of the next chunk.
constexpr int TC_PROD_WARP = 0;
constexpr int TC_MMA_WARP = 1;
constexpr int TC_PROD2_WARP = 2;
constexpr int TC_PROD3_WARP = 3;
constexpr int TC_NPROD = 3;
constexpr int TC_EPI_WARP0 = 4;
constexpr int TC_THREADS = (TC_EPI_WARP0 + TC_EPI_WARPS) * 32;  // 512

constexpr int TC_STG_LD = 36;  // padded fp32 row of the 32x32 epilogue transpose tile
constexpr int TC_STG_BYTES = TC_EPI_WARPS * 32 * TC_STG_LD * 4;
// the TMA-store epilogue reuses the region: 2 x 2 KB boxes per warp + the SubnetNorm row
static_assert(TC_EPI_WARPS * 4096 + 2048 <= TC_STG_BYTES, "TMA-store staging exceeds the epilogue region");

// Resident-B mode (RESB): when the whole active weight slice is ONE N tile
// of <= TC_RB_BYTES (narrow 1x1 convs: 88->256, 256->88, 64->256 ...), it is
// loaded into shared memory once per CTA and only A streams through the
// ring.  Re-streaming B per tile was ~40% of such a layer's time
// (SSN_TC_DEBUG=8 isolation) because every tile re-read the same weights.
constexpr int TC_RB_BYTES = 96 * 1024;
// RESB = 2: a 64 KB resident slice plus the residual ring — per epilogue
// group two 8 KB slots of {128 rows x 32 columns} bf16, filled by warp 3
// with TMA one chunk ahead of the group (the residual was the epilogue's
// latency bound: one 16-byte register load per lane per row in flight).
constexpr int TC_RB2_BYTES = 64 * 1024;
constexpr int TC_RR_SLOT = 128 * 32 * 2;
constexpr int TC_RR_SLOTS = 2 * 3;

template <int BN_MAX, int STAGES, int KPS, int RESB = 0, int CG = 1>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN_MAX / CG * TC_BK * 2;  // CG = 2: this CTA's half of N
  // RESB: 0 streamed B, 1 resident B (96 KB), 2 resident B (64 KB) + residual
  // ring, 3 streamed B + residual ring
  static constexpr bool RES_B = RESB == 1 || RESB == 2;
  static constexpr int RB = RESB == 2 ? TC_RB2_BYTES : (RESB == 1 ? TC_RB_BYTES : 0);
  static constexpr int RR = RESB >= 2 ? TC_RR_SLOT * TC_RR_SLOTS : 0;
  static constexpr int STAGE_BYTES = KPS * (A_BYTES + (RES_B ? 0 : B_BYTES));
  // TMEM accumulator ring: as many BN_MAX-column buffers as fit 512 columns
  // (max 4), so the MMA can run several tiles ahead of the epilogue.
  // (BN_MAX 64 -> 3: narrow tiles alternate whole across the 3 epilogue
  // groups, and each accumulator must always be drained by the same group,
  // else a group could pass a stale mbarrier phase of an older use.)
  static constexpr int NACC = BN_MAX <= 64 ? 3 : (512 / BN_MAX > 4 ? 4 : 512 / BN_MAX);
  static constexpr int TMEM_COLS = NACC * BN_MAX <= 256 ? 256 : 512;  // power-of-2 allocation
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + RB + RR + TC_STG_BYTES +
                              (2 * STAGES + 2 * NACC + 1 + 2 * TC_RR_SLOTS) * 8 + 16;
  static_assert(SMEM <= 232448, "operand ring exceeds 227 KB of shared memory");
};


// Ragged tail of a cout % 8 != 0 slice (e.g. a 2-label classifier): scalar
// accesses, kept out of line so the 8-wide vector epilogue stays compact.
static __device__ __noinline__ uint4 load_ragged_bf16x8(const __nv_bfloat16* rp, int nv) {
  uint4 r = make_uint4(0, 0, 0, 0);
  __nv_bfloat16* rs = reinterpret_cast<__nv_bfloat16*>(&r);
  for (int q = 0; q < nv; ++q) rs[q] = rp[q];
  return r;
}

static __device__ __noinline__ void store_ragged8(void* y, size_t off, int nv, int out_f32, float o0,
                                                  float o1, float o2, float o3, float o4, float o5,
                                                  float o6, float o7) {
  const float o[8] = {o0, o1, o2, o3, o4, o5, o6, o7};
  for (int q = 0; q < nv; ++q) {
    if (out_f32)
      static_cast<float*>(y)[off + q] = o[q];
    else
      static_cast<__nv_bfloat16*>(y)[off + q] = __float2bfloat16_rn(o[q]);
  }
}

// Per-chunk epilogue operands (SubnetNorm scale/shift of 8 columns, residual
// of 4 rows x 8 columns), fetched one chunk ahead.
struct EpiIn {
  float sc[8];
  float sh[8];
  uint4 rv[4];
};

// EPI: 0 = identity/ReLU (the CNNs), 1 = h_swish (MBv3), 2 = GELU / tanh or a
// ragged output slice (cout % 8 != 0; BERT head).  One instance per epilogue
// keeps each compact: an inlined erff/tanhf + scalar tail tripled the SASS of
// the ReLU kernel and halved its throughput through I-cache misses.
// CG = 2: a cluster of two CTAs computes one 256 x bn tile with
// tcgen05.mma.cta_group::2 (issued by CTA 0).  Each CTA loads its own 128
// A rows and half of B (bn/2 rows) into the same smem offsets, so per SM the
// operand stream per MMA cycle drops by a third (bn = 256: 32 KB per 512
// cycles instead of 48 KB) — the per-SM TMA rate (tools/ubench/tma_rate.cu)
// is what bounds the 1-CTA kernel on the big tensor-bound layers.
template <int BN_MAX, int STAGES, int KPS, int EPI, int RESB, int CG = 1>
__global__ void __launch_bounds__(TC_THREADS, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, const __grid_constant__ CUtensorMap wmap) {
  using C = TcCfg<BN_MAX, STAGES, KPS, RESB, CG>;
  static_assert(CG == 1 || RESB == 0, "2-CTA mode streams both operands");
  constexpr bool RES_B = C::RES_B;         // resident weight slice
  constexpr bool RRING = RESB >= 2;        // residual through the TMA ring
  constexpr int NACC = C::NACC;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned for SW128; offset arithmetic on smem_raw keeps the shared
  // address space visible to the compiler
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                 // [STAGES][KPS] A boxes
  uint8_t* sB = smem + STAGES * KPS * C::A_BYTES;     // [STAGES][KPS] B boxes | RESB: [nk] blocks
  uint8_t* sR = smem + STAGES * C::STAGE_BYTES + C::RB;  // RESB = 2: residual ring
  uint8_t* epi_base = sR + C::RR;
  float* epi_stage = reinterpret_cast<float*>(epi_base);
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_base + TC_STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [NACC]
  uint64_t* tempty = tfull + NACC;   // [NACC]
  uint64_t* bfull = tempty + NACC;  // RESB: the resident weight slice landed
  uint64_t* rfull = bfull + 1;      // RESB = 2: [group * 2 + slot]
  uint64_t* rempty = rfull + TC_RR_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + TC_RR_SLOTS);

  const OpDesc* dp = desc_ptr(p.row, p.fixed, p.op);
  const OpDims d = load_desc(p.row, p.fixed, p.op);
  const int d_wrows = dp->wrows;
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index through shfl: the compiler then knows it is warp-uniform, so
  // role branches stay uniform and MMA/TMA operands live in uniform registers
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  // Setup that needs no descriptor field (barriers, TMEM, the CTA / cluster
  // sync) runs while the dependent row -> descriptor loads are in flight: the
  // chain costs ~1 us per launch when it is waited on first.
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);  // the owning producer's expect_tx arrival
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      // every epilogue warp of the tile's CTA(s) (CG = 2: both CTAs' epilogues
      // arrive on CTA 0's); a warp draining a whole tile alone arrives 3x
      mbar_init(&tempty[a], TC_EPI_WARPS * CG);
    }
    mbar_init(bfull, 1);
    for (int r = 0; r < TC_RR_SLOTS; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], 4);  // the group's four warps
    }
    fence_mbar_init();
  }
  if (warp == TC_MMA_WARP) {
    if (CG == 2)
      tmem2_alloc(tmem_slot, C::TMEM_COLS);
    else
      tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();  // the peer's barriers exist before any remote arrival / TMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // WeightSlice tile width of the actuated subnet (conv_bn_active); its own
  // weight map (box = bn / CG rows) when the subnet row carries one that
  // matches, else the graph's max-width map (extra rows land unused)
  const int bn = (p.dbg & 4194304) ? p.bn : conv_bn_active(p.bn, d.cout, CG);  // A/B switch
  const bool own_wmap = d_wrows == bn / CG;
  const CUtensorMap* wm = own_wmap ? &dp->wmap : &wmap;
  const int brows = own_wmap ? bn / CG : p.bn / CG;  // rows each B box lands
  const int mt = (p.M + TC_BM * CG - 1) / (TC_BM * CG);  // CG = 2: 256-row pair tiles
  const int nt = (d.cout + bn - 1) / bn;  // WeightSlice: only tiles inside cout_a
  const int tiles = mt * nt;
  const int S = p.splits > 1 ? p.splits : 1;  // split-K: work unit u = (tile u / S, K range u % S)
  const int units = tiles * S;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const int unit0 = static_cast<int>(blockIdx.x) / CG;     // this CTA's (pair's) first tile
  const int ustep = static_cast<int>(gridDim.x) / CG;
  const bool idle = unit0 >= units;  // no tile of the actuated subnet (both CTAs of a pair agree)
  // Epilogue work split: wide tiles (>= TC_EPI_GROUPS 32-column chunks) are
  // striped chunk-wise across all groups; narrow ones go whole to one group
  // in turn (striping 1-2 chunks over 3 groups only adds handshakes).
  // (a narrow ACTIVE width on a wide instance stripes too: the alternate mode
  // needs NACC % 3 == 0, which only the 64-wide instances guarantee)
  const bool stripe = (bn + 31) / 32 >= TC_EPI_GROUPS || C::NACC % TC_EPI_GROUPS != 0;
  // alternate mode hands tile i to group i % 3 and accumulator i % NACC: the
  // pair must be a function of the accumulator alone
  static_assert(BN_MAX > 64 || C::NACC % TC_EPI_GROUPS == 0, "accumulator/group mapping");

  const int ka = d.k, pad = d.pad, koff = (p.k_max - ka) / 2;
  const int cblocks = (d.cin + TC_BK - 1) / TC_BK;
  const int nk = ka * ka * cblocks;
  // resident B: K blocks packed at the ACTUAL tile width (bn rows of 128 B,
  // a multiple of the 1 KB swizzle atom), which is what resident_b() sizes
  // against TC_RB_BYTES — a BN_MAX stride overran the region for bn < BN_MAX
  const uint32_t rb_stride = static_cast<uint32_t>(brows) * TC_BK * 2;
  if (tid == 0 && !idle) {
    tma_prefetch(wm);
    tma_prefetch(&dp->amap);
  }
  // PDL: everything above touched only smem / TMEM / static descriptors.
  // Weights are static too: the producers issue the resident slice / the
  // first ring stages' B boxes before griddepcontrol.wait, overlapping the
  // predecessor's tail; activations (A, residual) are read only after it.
  pdl_trigger();
  // SSN_TC_DEBUG & 32: per-role cycle accounting of CTA 0 (profiling only)
  const bool prof = (p.dbg & 32) && blockIdx.x == 0;
  long long w_wait = 0, w_wait2 = 0;
  const long long t_begin = prof ? clock64() : 0;

  // residual ring: warp 3 streams the residual; 2-stage rings: two producers
  constexpr int NPROD = RRING ? 2 : (STAGES < TC_NPROD ? STAGES : TC_NPROD);
  if (idle) {
    // nothing to do; fall through to the common teardown
  } else if (RRING && warp == TC_PROD3_WARP) {
    // ============================================================ residual ring
    // Chunk c of every tile goes to group c % 3's ring (the group drains
    // its chunks in this same order), slot = that group's sequence % 2.
    static_assert(!RRING || CG == 1, "residual ring: single-CTA tiles");
    pdl_wait();  // the residual is the predecessors' output
    const bool leader = elect_one();
    const int nchunk = (bn + 31) / 32;
    int kseq[3] = {0, 0, 0};
    for (int t = unit0; t < tiles; t += ustep) {
      const int m0 = (t / nt) * TC_BM;
      const int left = d.cout - (t % nt) * bn;
      const int nch = min(nchunk, (left + 31) / 32);
      for (int c = 0; c < nch; ++c) {
        const int g3 = c % 3;
        const int k = kseq[g3]++;
        const int slot = g3 * 2 + (k & 1);
        mbar_wait(&rempty[slot], ((k >> 1) & 1) ^ 1);
        if (leader) {
          mbar_arrive_expect_tx(&rfull[slot], TC_RR_SLOT);
          tma_load_2d(sR + slot * TC_RR_SLOT, &dp->rmap, &rfull[slot], (t % nt) * bn + c * 32, m0);
        }
        __syncwarp();
      }
    }
  } else if (warp == TC_PROD_WARP || warp == TC_PROD2_WARP || warp == TC_PROD3_WARP) {
    // ============================================================ producers
    // K block g (ring position) belongs to producer g % TC_NPROD, which loads
    // its A (activations) and B (weights) boxes; warp 0 also preloads the
    // resident B.  Safe against mbarrier phase aliasing: a producer reaching
    // g has filled g - TC_NPROD, which needed g - TC_NPROD - STAGES released,
    // so g - 2 * STAGES was released too (TC_NPROD <= STAGES).
    static_assert(NPROD <= STAGES, "producer round-robin needs NPROD <= STAGES");
    const int pidx = warp == TC_PROD_WARP ? 0 : warp - 1;
    const bool leader = elect_one();
    const CUtensorMap* amap = &dp->amap;
    const int hwo = p.ho * p.wo;
    const bool pointwise = p.k_max == 1 && p.stride == 1;  // A map is 2-D tiled (make_act_map)
    if (RES_B && leader && pidx == 0) {
      // the whole (single-N-tile) weight slice, once per CTA: block kb = (tap, channel block)
      if (p.dbg & 8) {
        mbar_arrive(bfull);
      } else {
        mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(nk * brows * TC_BK * 2));
        int tr = 0, ts = 0, cb = 0;
        for (int kb = 0; kb < nk; ++kb) {
          tma_load_3d(sB + kb * rb_stride, wm, bfull, cb * TC_BK,
                      (tr + koff) * p.k_max + (ts + koff), 0);
          if (++cb == cblocks) {
            cb = 0;
            if (++ts == ka) {
              ts = 0;
              ++tr;
            }
          }
        }
      }
    }
    // B of the first tile's leading ring stages, ahead of the PDL wait
    // (npre STAGES; each holds KPS K blocks, the last one possibly fewer)
    const int npre = (!RES_B && !(p.dbg & 8) && S == 1) ? min(STAGES, (nk + KPS - 1) / KPS) : 0;
    const uint32_t a_tx1 = (p.dbg & 4) ? 0u : static_cast<uint32_t>(C::A_BYTES * CG);
    const uint32_t b_tx1 = (p.dbg & 8) ? 0u : static_cast<uint32_t>(brows * CG * TC_BK * 2);
    if (npre && leader) {
      const int n0 = (unit0 % nt) * bn + static_cast<int>(rank) * (bn / CG);
      int tr = 0, ts = 0, cb = 0;
      for (int st = 0; st < npre; ++st) {
        const int nsub = min(KPS, nk - st * KPS);
        const bool mine = st % NPROD == pidx;
        if (mine && rank == 0) mbar_arrive_expect_tx(&full[st], nsub * (a_tx1 + b_tx1));
#pragma unroll
        for (int j = 0; j < KPS; ++j) {
          if (j < nsub) {
            if (mine) {
              uint8_t* dst = sB + (st * KPS + j) * C::B_BYTES;
              if (CG == 2)
                tma2_load_3d(dst, wm, &full[st], cb * TC_BK, (tr + koff) * p.k_max + (ts + koff), n0);
              else
                tma_load_3d(dst, wm, &full[st], cb * TC_BK, (tr + koff) * p.k_max + (ts + koff), n0);
            }
            if (++cb == cblocks) {
              cb = 0;
              if (++ts == ka) {
                ts = 0;
                ++tr;
              }
            }
          }
        }
      }
    }
    __syncwarp();
    pdl_wait();
    int g = 0;  // stage counter (ring position)
    for (int u = unit0; u < units; u += ustep) {
      const int t = u / S, z = u - t * S;
      const int kb_lo = z * nk / S, kb_hi = (z + 1) * nk / S;
      const int m0 = (t / nt) * TC_BM * CG + static_cast<int>(rank) * TC_BM;  // this CTA's rows
      const int n0 = (t % nt) * bn + static_cast<int>(rank) * (bn / CG);      // this CTA's B rows
      const int img = m0 / hwo;
      const int rem = m0 - img * hwo;
      const int oh = rem / p.wo;
      const int ow = rem - oh * p.wo;
      const int w0 = ow * p.stride - pad, h0 = oh * p.stride - pad;
      int cb = kb_lo % cblocks, ts = (kb_lo / cblocks) % ka, tr = kb_lo / cblocks / ka;
      for (int kb = kb_lo; kb < kb_hi; kb += KPS, ++g) {
        if (g % NPROD != pidx) {  // another producer's block: advance the (tap, channel) walk
#pragma unroll
          for (int j = 0; j < KPS; ++j) {
            if (++cb == cblocks) {
              cb = 0;
              if (++ts == ka) {
                ts = 0;
                ++tr;
              }
            }
          }
          continue;
        }
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        if (prof) {
          const long long t0 = clock64();
          mbar_wait(&empty[s], ph ^ 1);
          w_wait += clock64() - t0;
        } else {
          mbar_wait(&empty[s], ph ^ 1);
        }
        const int nsub = min(KPS, kb_hi - kb);
        const bool pre = g < npre;  // B already in flight, barrier armed
        if (leader && rank == 0 && !pre) {  // CG = 2: CTA 0's barrier counts both CTAs' bytes
          const uint32_t a_tx = (p.dbg & 4) ? 0u : static_cast<uint32_t>(C::A_BYTES * CG);
          const uint32_t b_tx = (p.dbg & 8) ? 0u : static_cast<uint32_t>(brows * CG * TC_BK * 2);
          const uint32_t tx = nsub * (a_tx + (RES_B ? 0u : b_tx));
          if (tx) mbar_arrive_expect_tx(&full[s], tx);
          else mbar_arrive(&full[s]);
        }
#pragma unroll
        for (int j = 0; j < KPS; ++j) {
          if (j < nsub) {
            if (leader) {
              uint8_t* dst = sA + (s * KPS + j) * C::A_BYTES;
              if (p.dbg & 4) {
              } else if (pointwise) {  // 1x1 stride 1: plain 2-D tile of the [M][cin_a] matrix
                if (CG == 2) tma2_load_2d(dst, amap, &full[s], cb * TC_BK, m0);
                else tma_load_2d(dst, amap, &full[s], cb * TC_BK, m0);
              } else if (CG == 2) {
                tma2_im2col_4d(dst, amap, &full[s], cb * TC_BK, w0, h0, img,
                               static_cast<uint16_t>(ts), static_cast<uint16_t>(tr));
              } else {
                tma_im2col_4d(dst, amap, &full[s], cb * TC_BK, w0, h0, img,
                              static_cast<uint16_t>(ts), static_cast<uint16_t>(tr));
              }
            }
            if (leader && !RES_B && !(p.dbg & 8) && !pre) {
              uint8_t* dst = sB + (s * KPS + j) * C::B_BYTES;
              if (CG == 2)
                tma2_load_3d(dst, wm, &full[s], cb * TC_BK, (tr + koff) * p.k_max + (ts + koff), n0);
              else
                tma_load_3d(dst, wm, &full[s], cb * TC_BK, (tr + koff) * p.k_max + (ts + koff), n0);
            }
            if (++cb == cblocks) {
              cb = 0;
              if (++ts == ka) {
                ts = 0;
                ++tr;
              }
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= TC_EPI_WARP0) {
    // ============================================================ epilogue
    // TMEM gives each thread one ROW; global memory wants each warp to touch
    // whole row segments.  Each 32x32 fp32 chunk is transposed through a
    // per-warp padded smem tile: afterwards lane (rsub = lane/4, seg = lane%4)
    // owns 8 consecutive columns of rows rsub, rsub+8, ... so residual loads
    // and output stores are 64-byte row-contiguous and coalesced (a
    // row-per-lane epilogue without the transpose measured 1.6x slower on the
    // HBM-bound 1x1 convs).  Three groups of 4 warps (one per TMEM lane
    // quarter) split the work (see `stripe`).  Software-pipelined: the
    // SubnetNorm row and residual of the warp's NEXT chunk are in flight
    // while this chunk is drained.
    pdl_wait();  // the residual is the predecessors' output
    const int ew = warp - TC_EPI_WARP0;
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (warps 1-4, 5-8)
    const int group = ew >> 2;     // chunk stripe this warp drains
    float* stg = epi_stage + ew * (32 * TC_STG_LD);
    const int seg = lane & 3, rsub = lane >> 2;
    const int nchunk = (bn + 31) / 32;
    const bool sc_vec = ((reinterpret_cast<uintptr_t>(d.scale) | reinterpret_cast<uintptr_t>(d.shift)) & 15) == 0 &&
                        (d.cout & 3) == 0;
    auto chunks_of = [&](int t) {
      const int left = d.cout - (t % nt) * bn;
      return min(nchunk, (left + 31) / 32);
    };
    auto fetch = [&](EpiIn& in, int t, int c) {
      const int m0 = (t / nt) * TC_BM * CG + static_cast<int>(rank) * TC_BM + quarter * 32;
      const int cc = c * 32;
      const int col = (t % nt) * bn + cc + seg * 8;
      const bool colok = col < d.cout && cc + seg * 8 < bn;
      const int nv = colok ? min(8, d.cout - col) : 0;
      const bool vec = EPI != 2 || (nv == 8 && (d.cout & 7) == 0);
      if (!colok) return;
      // EPI 0/1: SubnetNorm rows and biases are 16-byte aligned (engine
      // tables; the operator API routes unaligned vectors to EPI 2)
      const bool v4 = EPI != 2 || (sc_vec && nv == 8);
      if (p.dbg & 4096) {  // profiling: constant SubnetNorm row
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          in.sc[q] = 1.f;
          in.sh[q] = 0.f;
        }
      } else {
      if (d.scale && v4) {
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(d.scale + col));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(d.scale + col + 4));
        in.sc[0] = s0.x; in.sc[1] = s0.y; in.sc[2] = s0.z; in.sc[3] = s0.w;
        in.sc[4] = s1.x; in.sc[5] = s1.y; in.sc[6] = s1.z; in.sc[7] = s1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          in.sc[q] = d.scale ? __ldg(d.scale + (EPI == 2 ? min(col + q, d.cout - 1) : col + q)) : 1.f;
      }
      if (d.shift && v4) {
        const float4 h0 = __ldg(reinterpret_cast<const float4*>(d.shift + col));
        const float4 h1 = __ldg(reinterpret_cast<const float4*>(d.shift + col + 4));
        in.sh[0] = h0.x; in.sh[1] = h0.y; in.sh[2] = h0.z; in.sh[3] = h0.w;
        in.sh[4] = h1.x; in.sh[5] = h1.y; in.sh[6] = h1.z; in.sh[7] = h1.w;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          in.sh[q] = d.shift ? __ldg(d.shift + (EPI == 2 ? min(col + q, d.cout - 1) : col + q)) : 0.f;
      }
      }
      if (!RRING && p.res && !(p.dbg & 2048)) {
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const int m = m0 + rsub + 8 * r4;
          if (m >= p.M) continue;
          const __nv_bfloat16* rp =
              static_cast<const __nv_bfloat16*>(p.res) + static_cast<size_t>(m) * d.ldo + col;
          in.rv[r4] = vec ? __ldg(reinterpret_cast<const uint4*>(rp)) : load_ragged_bf16x8(rp, nv);
        }
      }
    };
    // epilogue flags hoisted out of the chunk loop (uniform registers)
    const bool has_res = p.res != nullptr;
    const bool res_post = p.res_post != 0;
    const int act = p.act;
    const bool out_f32 = p.out_f32 != 0;
    // Every tile is drained by all TC_EPI_GROUPS groups: group g takes the
    // 32-column chunks c = g, g + G, ... (more warps in flight per tile than
    // tempty lives in CTA 0 of a pair (its MMA warp waits on it)
    const uint32_t tcount = stripe ? 1u : static_cast<uint32_t>(TC_EPI_GROUPS);
    auto arrive_tempty = [&](int a) {
      if (CG == 2)
        mbar_arrive_cluster_cnt(mapa_shared(&tempty[a], 0), tcount);
      else
        mbar_arrive_cnt(&tempty[a], tcount);
    };
    // alternating whole tiles between two groups, which left the epilogue
    // latency-bound).  A group without a chunk in a tile still waits for the
    // accumulator and arrives on tempty (the barrier counts every warp).
    const int i_step = stripe ? 1 : TC_EPI_GROUPS, c0 = stripe ? group : 0;
    const int c_step = stripe ? TC_EPI_GROUPS : 1;
    int i = stripe ? 0 : group;  // tile ordinal
    int t = unit0 + i * ustep;
    int c = c0;
    int rk = 0;  // RESB = 2: chunks this group has drained (residual ring sequence)
    // TMA-store epilogue (`ys`): the descriptor row carries this subnet's
    // output map.  Row per lane straight from tcgen05.ld (no fp32 transpose
    // through shared memory): SubnetNorm columns by warp shuffle, the residual
    // row as four 16-byte vectors (global or the 64B-swizzled ring slot), the
    // bf16 chunk written once into a 64B-swizzled 2 KB box and stored by ONE
    // TMA store.  Shared-memory traffic per chunk drops from 8 KB (fp32 STS +
    // LDS) to 4 KB (bf16 STS + TMA read) and the per-lane STG chain goes.
    // Needs whole 32-column chunks inside the tile (one N tile, or bn % 32 = 0).
    // (a residual from global memory keeps the coalesced path: row-per-lane
    // 16-B residual loads measured slower on the 56-px 88->256 expand,
    // 69 -> 78 us; SSN_TC_DEBUG & 67108864 overrides for A/B)
    const bool ys = p.ystore && S == 1 && !p.out_f32 && (d.cout & 7) == 0 &&
                    (nt == 1 || (bn & 31) == 0) && !(p.dbg & 33554432) &&
                    (RRING || p.res == nullptr || (p.dbg & 67108864));
    if (ys) {
      uint8_t* ybuf = epi_base + ew * 4096;  // two 2 KB staging boxes per warp
      const __nv_bfloat16* resp = static_cast<const __nv_bfloat16*>(p.res);
      int yb = 0;
      // One N tile (every tile has the same columns): the SubnetNorm row sits
      // in shared memory for the whole launch (broadcast LDS.128, 16 per
      // chunk instead of 64 shuffles) and the tile / chunk arithmetic needs
      // no division.  ncu on the 56-px 64->256 layer: issue-bound epilogue
      // (45% issue slots, LSU pipe 41% from the shuffles).
      // (not in the GELU / ragged instance: its SASS is the largest and the
      // extra path cost BERT's FFN-up 8% through instruction-cache misses)
      const bool one_nt = EPI != 2 && nt == 1 && !(p.dbg & 134217728);  // (A/B: shuffle path)
      const int nch1 = chunks_of(0);
      float* sn = reinterpret_cast<float*>(epi_base + TC_EPI_WARPS * 4096);  // [256] scale, [256] shift
      if (one_nt) {
        for (int k = ew * 32 + lane; k < 512; k += TC_EPI_WARPS * 32) {
          const int cj = k & 255;
          const float* src = k < 256 ? d.scale : d.shift;
          sn[k] = cj < d.cout && src ? __ldg(src + cj) : (k < 256 && !src ? 1.f : 0.f);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(TC_EPI_WARPS * 32) : "memory");  // epilogue warps only
      }
      const bool relu_pack = EPI == 0 && act == 1 && !(has_res && res_post);
      while (t < units) {
        const int tm = one_nt ? t : t / nt;  // M tile
        const int tq = t - tm * nt;          // N tile
        const int nch = one_nt ? nch1 : chunks_of(t);
        int tn = t, cn = c + c_step, inx = i;
        if (cn >= nch) {
          cn = c0;
          inx = i + i_step;
          tn = t + i_step * ustep;
        }
        const bool have = c < nch;
        const int row0 = tm * TC_BM * CG + static_cast<int>(rank) * TC_BM + quarter * 32;
        const int col0 = tq * bn + c * 32;
        const int m = row0 + lane;
        float scl = 1.f, shl = 0.f;  // lane j: SubnetNorm of column col0 + j
        uint4 rv[4];
        if (have) {
          if (!one_nt) {
            const int cj = col0 + lane;
            if (d.scale) scl = cj < d.cout ? __ldg(d.scale + cj) : 0.f;
            if (d.shift) shl = cj < d.cout ? __ldg(d.shift + cj) : 0.f;
          }
          if (!RRING && has_res) {
            const __nv_bfloat16* rp = resp + static_cast<size_t>(m < p.M ? m : 0) * d.ldo + col0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              rv[q] = col0 + q * 8 < d.cout ? __ldg(reinterpret_cast<const uint4*>(rp + q * 8))
                                            : make_uint4(0, 0, 0, 0);
          }
        }
        const int a = i % NACC;
        if (c == c0) {
          mbar_wait(&tfull[a], static_cast<uint32_t>(i / NACC) & 1);
          tc_fence_after();
        }
        if (!have) {  // no chunk of this tile for this group
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_tempty(a);
          t = tn;
          c = cn;
          i = inx;
          continue;
        }
        float v[32];
        tmem_ld32(tmem + a * BN_MAX + (static_cast<uint32_t>(quarter * 32) << 16) + c * 32, v);
        if (inx != i) {  // this warp's last chunk of the tile is out of TMEM
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_tempty(a);
        }
        const int sw = (lane >> 1) & 3;  // 64B swizzle: 16-B chunk q of row r sits at q ^ ((r >> 1) & 3)
        if (RRING && has_res) {
          const int slot = group * 2 + (rk & 1);
          mbar_wait(&rfull[slot], static_cast<uint32_t>(rk >> 1) & 1);
          const uint8_t* rs = sR + slot * TC_RR_SLOT + (quarter * 32 + lane) * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q) rv[q] = *reinterpret_cast<const uint4*>(rs + ((q ^ sw) << 4));
          fence_proxy_async_smem();  // reads ordered before the producer's next TMA write
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[slot]);
          ++rk;
        }
        if (one_nt) {
          const float4* s4 = reinterpret_cast<const float4*>(sn + c * 32);
          const float4* h4 = reinterpret_cast<const float4*>(sn + 256 + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 sc = s4[j], sh = h4[j];
            v[4 * j] = v[4 * j] * sc.x + sh.x;
            v[4 * j + 1] = v[4 * j + 1] * sc.y + sh.y;
            v[4 * j + 2] = v[4 * j + 2] * sc.z + sh.z;
            v[4 * j + 3] = v[4 * j + 3] * sc.w + sh.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            v[j] = v[j] * __shfl_sync(0xffffffffu, scl, j) + __shfl_sync(0xffffffffu, shl, j);
        }
        if (has_res && !res_post) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[q]);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 f = __bfloat1622float2(rh[h]);
              v[q * 8 + 2 * h] += f.x;
              v[q * 8 + 2 * h + 1] += f.y;
            }
          }
        }
        if (act == 1 && !relu_pack) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
        } else if (EPI == 1 && act == 2) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= fminf(fmaxf(v[j] + 3.f, 0.f), 6.f) * (1.f / 6.f);
        } else if (EPI == 2 && act == 3) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_erf_fast(v[j]);
        } else if (EPI == 2 && act) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = act_apply(v[j], act);
        }
        if (has_res && res_post) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv[q]);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 f = __bfloat1622float2(rh[h]);
              v[q * 8 + 2 * h] += f.x;
              v[q * 8 + 2 * h + 1] += f.y;
            }
          }
        }
        if (lane == 0) bulk_wait_read<1>();  // the store that last used this box has read it
        __syncwarp();
        uint8_t* box = ybuf + yb * 2048;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk;
          if (relu_pack) {
            pk.x = pack_bf16x2_relu(v[q * 8 + 0], v[q * 8 + 1]);
            pk.y = pack_bf16x2_relu(v[q * 8 + 2], v[q * 8 + 3]);
            pk.z = pack_bf16x2_relu(v[q * 8 + 4], v[q * 8 + 5]);
            pk.w = pack_bf16x2_relu(v[q * 8 + 6], v[q * 8 + 7]);
          } else {
            pk.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
            pk.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
            pk.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
            pk.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
          }
          *reinterpret_cast<uint4*>(box + lane * 64 + ((q ^ sw) << 4)) = pk;
        }
        fence_proxy_async_smem();  // generic-proxy writes visible to the TMA store
        __syncwarp();
        if (lane == 0 && row0 < p.M && !(p.dbg & 1)) {
          tma_store_2d(&dp->ymap, box, col0, row0);
          bulk_commit();
        }
        yb ^= 1;
        t = tn;
        c = cn;
        i = inx;
      }
      if (lane == 0) bulk_wait<0>();  // stores complete before the CTA retires
    } else {
    EpiIn cur;  // this chunk's SubnetNorm row + residual (no register prefetch:
                // 12 warps hide the latency, and 512 threads cap registers at 128)
    while (t < units) {
      const int tt = t / S;  // tile of work unit t
      int tn = t, cn = c + c_step, inx = i;
      if (cn >= chunks_of(tt)) {
        cn = c0;
        inx = i + i_step;
        tn = t + i_step * ustep;
      }
      // operands of this chunk, issued before the accumulator wait / TMEM load
      if (!(p.dbg & 1) && S == 1 && c < chunks_of(tt)) fetch(cur, tt, c);
      const int a = i % NACC;
      if (c == c0) {
        if (prof) {
          const long long t0 = clock64();
          mbar_wait(&tfull[a], static_cast<uint32_t>(i / NACC) & 1);
          w_wait += clock64() - t0;
        } else {
          mbar_wait(&tfull[a], static_cast<uint32_t>(i / NACC) & 1);
        }
        tc_fence_after();
      }
      if (c >= chunks_of(tt)) {  // no chunk of this tile for this group
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_tempty(a);
        t = tn;
        c = cn;
        i = inx;
        continue;
      }
      const int m0 = (tt / nt) * TC_BM * CG + static_cast<int>(rank) * TC_BM + quarter * 32;
      const int cc = c * 32;
      const int col = (tt % nt) * bn + cc + seg * 8;
      const bool colok = col < d.cout && cc + seg * 8 < bn;
      const int nv = colok ? min(8, d.cout - col) : 0;
      const bool vec = EPI != 2 || (nv == 8 && (d.cout & 7) == 0);
      float v[32];
      if (prof) {
        const long long t0 = clock64();
        tmem_ld32(tmem + a * BN_MAX + (static_cast<uint32_t>(quarter * 32) << 16) + cc, v);
        w_wait2 += clock64() - t0;
      } else {
        tmem_ld32(tmem + a * BN_MAX + (static_cast<uint32_t>(quarter * 32) << 16) + cc, v);
      }
      float4* srow = reinterpret_cast<float4*>(stg + lane * TC_STG_LD);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        srow[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      __syncwarp();
      if (inx != i) {  // this warp's last chunk of the tile is out of TMEM: free the accumulator
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_tempty(a);
      }
      if (RRING && has_res) {  // this chunk's residual rows from the group's ring slot
        const int slot = group * 2 + (rk & 1);
        mbar_wait(&rfull[slot], static_cast<uint32_t>(rk >> 1) & 1);
        // rows quarter*32 + rsub + 8*r4 share (row >> 1) & 3 = (rsub >> 1) & 3 (64B swizzle)
        const uint8_t* rs = sR + slot * TC_RR_SLOT + (quarter * 32 + rsub) * 64 + ((seg ^ ((rsub >> 1) & 3)) << 4);
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) cur.rv[r4] = *reinterpret_cast<const uint4*>(rs + r4 * 8 * 64);
        // generic-proxy reads ordered before the producer's next async-proxy (TMA) write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[slot]);
        ++rk;
      }
      const long long tsec = prof ? clock64() : 0;
      if (colok && !(p.dbg & 1)) {
        // All four rows' staging reads first, then straight-line math, then
        // the predicated stores: one dependency chain per chunk instead of
        // four (the per-row `continue` + uniform-flag branches serialised
        // LDS -> FFMA -> STG and left the epilogue latency-bound).
        float o[4][8];
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const float4* sp = reinterpret_cast<const float4*>(stg + (rsub + 8 * r4) * TC_STG_LD + seg * 8);
          const float4 lo = sp[0], hi = sp[1];
          o[r4][0] = lo.x; o[r4][1] = lo.y; o[r4][2] = lo.z; o[r4][3] = lo.w;
          o[r4][4] = hi.x; o[r4][5] = hi.y; o[r4][6] = hi.z; o[r4][7] = hi.w;
        }
        if (S > 1) {  // split-K partial: raw fp32 into this K range's workspace slice
          const int z = t - tt * S;
          if (z * nk / S == (z + 1) * nk / S) {  // empty K range (nk < splits): zero slice
#pragma unroll
            for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
              for (int q = 0; q < 8; ++q) o[r4][q] = 0.f;
          }
          float* wz = p.ws + static_cast<size_t>(z) * p.M * d.cout;
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4) {
            const int m = m0 + rsub + 8 * r4;
            if (m < p.M) {
              float4* wp = reinterpret_cast<float4*>(wz + static_cast<size_t>(m) * d.cout + col);
              wp[0] = make_float4(o[r4][0], o[r4][1], o[r4][2], o[r4][3]);
              wp[1] = make_float4(o[r4][4], o[r4][5], o[r4][6], o[r4][7]);
            }
          }
          if (prof) w_wait2 += clock64() - tsec;
          __syncwarp();
          t = tn;
          c = cn;
          i = inx;
          continue;
        }
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
          for (int q = 0; q < 8; ++q) o[r4][q] = o[r4][q] * cur.sc[q] + cur.sh[q];
        if (has_res && !res_post) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4) {
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&cur.rv[r4]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(rh[q]);
              o[r4][2 * q] += f.x;
              o[r4][2 * q + 1] += f.y;
            }
          }
        }
        if (act == 1) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
            for (int q = 0; q < 8; ++q) o[r4][q] = fmaxf(o[r4][q], 0.f);
        } else if (EPI == 1 && act == 2) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
            for (int q = 0; q < 8; ++q)
              o[r4][q] *= fminf(fmaxf(o[r4][q] + 3.f, 0.f), 6.f) * (1.f / 6.f);
        } else if (EPI == 2 && act == 3) {  // GELU inline (gelu_erf_fast)
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
            for (int q = 0; q < 8; ++q) o[r4][q] = gelu_erf_fast(o[r4][q]);
        } else if (EPI == 2 && act) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4)
#pragma unroll
            for (int q = 0; q < 8; ++q) o[r4][q] = act_apply(o[r4][q], act);
        }
        if (has_res && res_post) {
#pragma unroll
          for (int r4 = 0; r4 < 4; ++r4) {
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&cur.rv[r4]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(rh[q]);
              o[r4][2 * q] += f.x;
              o[r4][2 * q + 1] += f.y;
            }
          }
        }
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
          const int m = m0 + rsub + 8 * r4;
          if (m >= p.M) continue;
          const size_t off = static_cast<size_t>(m) * d.ldo + col;
          if (!vec) {
            store_ragged8(p.y, off, nv, out_f32, o[r4][0], o[r4][1], o[r4][2], o[r4][3], o[r4][4],
                          o[r4][5], o[r4][6], o[r4][7]);
          } else if (out_f32) {
            float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + off);
            yp[0] = make_float4(o[r4][0], o[r4][1], o[r4][2], o[r4][3]);
            yp[1] = make_float4(o[r4][4], o[r4][5], o[r4][6], o[r4][7]);
          } else {
            uint4 pk;
            pk.x = pack_bf16x2(o[r4][0], o[r4][1]);
            pk.y = pack_bf16x2(o[r4][2], o[r4][3]);
            pk.z = pack_bf16x2(o[r4][4], o[r4][5]);
            pk.w = pack_bf16x2(o[r4][6], o[r4][7]);
            *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + off) = pk;
          }
        }
      }
      if (prof) w_wait2 += clock64() - tsec;
      __syncwarp();  // staging tile is rewritten by the next chunk
      t = tn;
      c = cn;
      i = inx;
    }
    }  // !ys
  } else if (warp == TC_MMA_WARP && rank == 0) {
    // ============================================================ MMA issuer
    // Converged warp, elected lane issues (tc_mma_bf16_elect); descriptors
    // are a base plus 16-byte-unit offsets (SW128: K step = +32 B).
    const uint32_t idesc = umma_idesc_bf16(bn, TC_BM * CG);
    const uint64_t a_base = umma_desc_sw128(smem_u32(sA));
    const uint64_t b_base = umma_desc_sw128(smem_u32(sB));
    if (RES_B) {
      mbar_wait(bfull, 0);
      tc_fence_after();
    }
    int g = 0, i = 0;
    for (int u = unit0; u < units; u += ustep, ++i) {
      const int z = u % S;
      const int kb_lo = z * nk / S, kb_hi = (z + 1) * nk / S;
      const int a = i % NACC;
      const uint32_t use = static_cast<uint32_t>(i / NACC);
      if (prof) {
        const long long t0 = clock64();
        mbar_wait(&tempty[a], (use & 1) ^ 1);
        w_wait2 += clock64() - t0;
      } else {
        mbar_wait(&tempty[a], (use & 1) ^ 1);
      }
      tc_fence_after();
      const uint32_t acc = tmem + a * BN_MAX;
      if (kb_lo == kb_hi) {  // split-K range with no K block (nk < splits): publish
        tc_commit_elect(&tfull[a]);  // the accumulator at once; the epilogue writes zeros
        __syncwarp();
        continue;
      }
      for (int kb = kb_lo; kb < kb_hi; kb += KPS, ++g) {
        const int s = g % STAGES;
        const uint32_t ph = (g / STAGES) & 1;
        if (prof) {
          const long long t0 = clock64();
          mbar_wait(&full[s], ph);
          w_wait += clock64() - t0;
        } else {
          mbar_wait(&full[s], ph);
        }
        tc_fence_after();
        const int nsub = min(KPS, kb_hi - kb);
#pragma unroll
        for (int j = 0; j < KPS; ++j) {
          if (j < nsub) {
            const uint64_t ad = a_base + static_cast<uint64_t>(((s * KPS + j) * C::A_BYTES) >> 4);
            const uint64_t bd =
                b_base + static_cast<uint64_t>(
                             (RES_B ? (kb + j) * rb_stride : (s * KPS + j) * C::B_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 16; ++kk) {
              if (p.dbg & 2) continue;
              if (CG == 2)
                tc2_mma_bf16_elect(acc, ad + static_cast<uint64_t>(kk * 2),
                                   bd + static_cast<uint64_t>(kk * 2), idesc,
                                   ((kb - kb_lo + j) | kk) != 0 ? 1u : 0u);
              else
                tc_mma_bf16_elect(acc, ad + static_cast<uint64_t>(kk * 2),
                                  bd + static_cast<uint64_t>(kk * 2), idesc,
                                  ((kb - kb_lo + j) | kk) != 0 ? 1u : 0u);
            }
          }
        }
        if (CG == 2) {  // free the stage / publish the accumulator in BOTH CTAs
          tc2_commit_mc_elect(&empty[s]);
          if (kb + KPS >= kb_hi) tc2_commit_mc_elect(&tfull[a]);
        } else {
          tc_commit_elect(&empty[s]);
          if (kb + KPS >= kb_hi) tc_commit_elect(&tfull[a]);
        }
        __syncwarp();
      }
    }
  }
  if (prof && lane == 0 && (warp == TC_PROD_WARP || warp == TC_MMA_WARP || warp == TC_EPI_WARP0))
    printf("[conv_tc prof] tiles=%d nk=%d warp=%d total=%lld wait=%lld wait2=%lld\n", tiles, nk, warp,
           clock64() - t_begin, w_wait, w_wait2);
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();  // neither CTA leaves while the pair's MMA / arrivals may touch it
  if (warp == TC_MMA_WARP) {
    tc_fence_after();
    if (CG == 2)
      tmem2_dealloc(tmem, C::TMEM_COLS);
    else
      tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Split-K finish: workspace slice z holds K range z's raw sum of every (row,
// column) of the active slice; add the slices in fixed order (deterministic,
// no atomics) and apply conv_tc's fused epilogue (SubnetNorm, residual
// before / after the activation).  8 columns per thread, 16-byte accesses.
__global__ void __launch_bounds__(256) conv_finish_kernel(const __grid_constant__ ConvParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, p.fixed, p.op);
  const int g8 = d.cout / 8;
  const long n = static_cast<long>(p.M) * g8;
  const size_t slice = static_cast<size_t>(p.M) * d.cout;
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * 256) {
    const long m = i / g8;
    const int c = static_cast<int>(i - m * g8) * 8;
    float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int z = 0; z < p.splits; ++z) {
      const float4* wp = reinterpret_cast<const float4*>(p.ws + z * slice + m * d.cout + c);
      const float4 a0 = wp[0], a1 = wp[1];
      o[0] += a0.x; o[1] += a0.y; o[2] += a0.z; o[3] += a0.w;
      o[4] += a1.x; o[5] += a1.y; o[6] += a1.z; o[7] += a1.w;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      o[q] = o[q] * (d.scale ? __ldg(d.scale + c + q) : 1.f) + (d.shift ? __ldg(d.shift + c + q) : 0.f);
    float r[8];
    if (p.res) {
      const uint4 rv = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.res) +
                                                           m * d.ldo + c));
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(rh[q]);
        r[2 * q] = f.x;
        r[2 * q + 1] = f.y;
      }
      if (!p.res_post)
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] += r[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = act_apply(o[q], p.act);
    if (p.res && p.res_post)
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] += r[q];
    if (p.out_f32) {
      float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + m * d.ldo + c);
      yp[0] = make_float4(o[0], o[1], o[2], o[3]);
      yp[1] = make_float4(o[4], o[5], o[6], o[7]);
    } else {
      uint4 pk;
      pk.x = pack_bf16x2(o[0], o[1]);
      pk.y = pack_bf16x2(o[2], o[3]);
      pk.z = pack_bf16x2(o[4], o[5]);
      pk.w = pack_bf16x2(o[6], o[7]);
      *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + m * d.ldo + c) = pk;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
static F driver_fn(const char* name) {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<F>(ptr);
  return nullptr;
}

// B operand: map over a max-shape KRSC bf16 weight tensor [cout][taps][cin_store]
// with {64 ch, 1 tap, bn} boxes, 128B swizzle.
int make_weight_map(CUtensorMap* map, const void* w, int cin_store, int taps, int cout, int bn) {
  static EncodeTiledFn enc = driver_fn<EncodeTiledFn>("cuTensorMapEncodeTiled");
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

// Residual source of a conv: [rows][cout] bf16 with {32 columns, 128 rows}
// boxes, no swizzle (64-byte rows: the epilogue's 16-byte row-segment reads
// of 8 lanes cover two whole rows, conflict-free).
int make_res_map(CUtensorMap* map, const void* r, long rows, int cout, int ld) {
  static EncodeTiledFn enc = driver_fn<EncodeTiledFn>("cuTensorMapEncodeTiled");
  if (!enc || (cout & 7) != 0 || (ld & 7) != 0) return -1;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cout), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(TC_BM)};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(r), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? 0 : -static_cast<int>(res);
}

// Output of a bf16 conv_tc op: 2-D tiled map over [rows][cout] (row pitch
// ld), box {32 columns, 32 rows}, 64B-swizzled (the TMA-store epilogue's
// staging layout).  Rows past `rows` and columns past `cout` are clipped.
int make_y_map(CUtensorMap* map, void* y, long rows, int cout, int ld) {
  static EncodeTiledFn enc = driver_fn<EncodeTiledFn>("cuTensorMapEncodeTiled");
  if (!enc || (cout & 7) != 0 || (ld & 7) != 0) return -1;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cout), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? 0 : -static_cast<int>(res);
}

// A operand: im2col map over a compact NHWC bf16 activation [n][h][w][cin]
// for a k x k / stride / pad convolution: 128 pixels x 64 channels per load.
int make_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld, int k,
                 int stride, int pad) {
  if (k == 1 && stride == 1 && pad == 0) {
    // pointwise conv: the activation is a plain [n*h*w][cin] matrix; a tiled
    // box {64 ch, 128 rows} is cheaper for the TMA unit than im2col mode
    static EncodeTiledFn tenc = driver_fn<EncodeTiledFn>("cuTensorMapEncodeTiled");
    if (!tenc) return -1;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cin), static_cast<cuuint64_t>(n) * h * w};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(TC_BK), static_cast<cuuint32_t>(TC_BM)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = tenc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
  }
  static EncodeIm2colFn enc = driver_fn<EncodeIm2colFn>("cuTensorMapEncodeIm2col");
  if (!enc) return -1;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cin), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2,
                           static_cast<cuuint64_t>(w) * ld * 2,
                           static_cast<cuuint64_t>(h) * w * ld * 2};
  const int lower[2] = {-pad, -pad};
  const int upper[2] = {pad - (k - 1), pad - (k - 1)};
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides,
                   lower, upper, TC_BK, TC_BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -static_cast<int>(r);
  // Same driver workaround CUTLASS applies to im2col maps of tensors < 128 KB
  // on drivers <= 13.1 (cute/atom/copy_traits_sm90_im2col.hpp).
  int drv = 0;
  cudaDriverGetVersion(&drv);
  const unsigned long long bytes = 2ull * n * h * w * ld;
  if (drv <= 13010 && bytes < 131072ull) reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
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

static int env_int(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}

// N tile: the whole 16-aligned output width when it fits one tile.  Wider
// slices take any 16-multiple <= 256 (the kernel's N is a runtime value):
// the per-SM operand feed, not the MMA, bounds these layers, so the width
// trades A re-streaming (narrow) against idle SMs (wide, few tiles).  The
// table is measured (tools/tile_sweep.sh: per-op device time summed over the
// {min, mid, max} sweep, N in {128..256}); other shapes use a wave cost.
// nk_max = K blocks of the max-shape slice; pairs from 16 K blocks on.
int choose_bn(int cout_max, long M, int nk_max) {
  const int c16 = (cout_max + 15) / 16 * 16;
  if (c16 <= 256) return c16;
  static const int force = env_int("SSN_TC_FORCE_BN");  // tuning experiments only
  if (force >= 16 && force <= 256 && force % 16 == 0) return force;
  if (cout_max <= 384) {                 // e.g. 360: 3x3 (54 kb), 1024->360, 512->360
    if (nk_max >= 32) return 144;
    if (nk_max >= 8) return 224;
    return 128;
  }
  if (cout_max <= 512) return nk_max <= 4 ? 192 : 256;   // 176/256 -> 512 at 28 px
  if (cout_max <= 768) {                 // 720: 3x3 (108 kb), 2048->720, 1024->720
    if (nk_max >= 64) return 144;
    if (nk_max >= 24) return 160;
    return 192;
  }
  if (cout_max <= 1024) return nk_max >= 8 ? 256 : 192;
  if (cout_max <= 2048 && nk_max >= 12) return 192;
  const int cg = nk_max >= 16 ? 2 : 1;
  const long mt = (M + TC_BM * cg - 1) / (TC_BM * cg);
  const long slots = num_sms() / cg;
  auto cost = [&](int bn) {
    const long tiles = mt * ((cout_max + bn - 1) / bn);
    const long waves = (tiles + slots - 1) / slots;
    return waves * (bn + (cg == 2 ? 128 : 64));
  };
  return cost(256) <= cost(128) ? 256 : 128;
}

// Instances (BN_MAX, STAGES, K blocks per stage): the operand ring plus the
// 36 KB epilogue staging fill the 227 KB of shared memory; resident-B
// instances trade ring stages for the 96 KB weight block.
// KPS = 2 instances (two K blocks per ring stage) for long-K streamed-B
// layers: the per-stage handshake (MMA commit -> producer -> full barrier ->
// MMA wait) costs ~520 cycles whatever the tile width (tools/ubench/
// mma2_rate.cu: 4 MMAs per stage cap at ~131 cycles per MMA, 8 at ~85-98),
// so a 4-MMA stage bounds every N < 256 tile below its tensor rate.
#define SSN_TC_INSTANCES(X) X(64, 7, 1, 0, 1) X(128, 5, 1, 0, 1) X(256, 3, 1, 0, 1) \
  X(64, 4, 1, 1, 1) X(128, 4, 1, 1, 1) X(256, 4, 1, 1, 1) X(256, 5, 1, 0, 2) X(128, 7, 1, 0, 2) \
  X(192, 4, 1, 0, 1) X(192, 6, 1, 0, 2) X(256, 2, 1, 2, 1) X(192, 3, 1, 3, 1) \
  X(64, 3, 2, 0, 1) X(128, 2, 2, 0, 1) X(192, 2, 2, 0, 1) X(128, 3, 2, 0, 2) X(192, 3, 2, 0, 2)

cudaError_t init_conv_tc() {
#define SSN_TC_ATTR(BN, ST, KPS, RB, CG)                                                  \
  {                                                                                       \
    void (*fns[3])(ConvParams, CUtensorMap) = {conv_tc_kernel<BN, ST, KPS, 0, RB, CG>,    \
                                               conv_tc_kernel<BN, ST, KPS, 1, RB, CG>,    \
                                               conv_tc_kernel<BN, ST, KPS, 2, RB, CG>};   \
    for (auto fn : fns) {                                                                 \
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           TcCfg<BN, ST, KPS, RB, CG>::SMEM);             \
      if (e != cudaSuccess) return e;                                                     \
    }                                                                                     \
  }
  SSN_TC_INSTANCES(SSN_TC_ATTR)
#undef SSN_TC_ATTR
  return cudaSuccess;
}

template <int BN_MAX, int STAGES, int KPS, int RESB, int CG = 1>
static cudaError_t launch_impl(const ConvParams& p, const CUtensorMap& wmap, cudaStream_t s) {
  using C = TcCfg<BN_MAX, STAGES, KPS, RESB, CG>;
  const long tiles = static_cast<long>((p.M + TC_BM * CG - 1) / (TC_BM * CG)) *
                     ((p.cout_max + p.bn - 1) / p.bn) * (p.splits > 1 ? p.splits : 1);
  void (*fn)(ConvParams, CUtensorMap) =
      (p.act > 2 || (p.cout_max & 7) != 0 || p.ragged) ? conv_tc_kernel<BN_MAX, STAGES, KPS, 2, RESB, CG>
      : p.act == 2                                      ? conv_tc_kernel<BN_MAX, STAGES, KPS, 1, RESB, CG>
                                                        : conv_tc_kernel<BN_MAX, STAGES, KPS, 0, RESB, CG>;
  if (CG == 1) {
    const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
    return launch_pdl(fn, dim3(grid), dim3(TC_THREADS), C::SMEM, s, 1, p, wmap);
  }
  // clusters of 2 CTAs (one per pair tile), at most one pair per 2 SMs
  const long pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  return launch_pdl(fn, dim3(static_cast<unsigned>(pairs * 2)), dim3(TC_THREADS), C::SMEM, s, 2, p,
                    wmap);
}

static int tc_debug() {
  static const int dbg = [] {
    const char* e = getenv("SSN_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return dbg;
}

static bool resident_b(const ConvParams& p) {
  const long nk_max = static_cast<long>(p.k_max) * p.k_max * ((p.cin_max + TC_BK - 1) / TC_BK);
  return !(tc_debug() & 512) && p.cout_max <= p.bn && nk_max * p.bn * TC_BK * 2 <= TC_RB_BYTES;
}

// Pair tiles (cta_group::2) for bn > 128 streamed-B convs; the caller encodes
// the weight map with bn / 2 rows per box when this returns true.
// Measured (tools/mb_ncu.sh): pairs win on long-K layers (3x3 720 @ 7 px
// -20%, 1x1 2048->720 -6%) and lose on short-K ones where the per-tile
// epilogue dominates (1x1 256->256 +15%), so they need >= 16 K blocks.
bool conv_tc_use_pairs(const ConvParams& p) {
  const long nk_max = static_cast<long>(p.k_max) * p.k_max * ((p.cin_max + TC_BK - 1) / TC_BK);
  static const int min_nk = [] {  // tuning experiments only
    const int v = env_int("SSN_TC_PAIR_MIN_NK");
    return v > 0 ? v : 16;
  }();
  return p.bn >= 128 && nk_max >= min_nk && !resident_b(p) && !(tc_debug() & 16384) &&
         p.act <= 2 && (p.cout_max & 7) == 0 && !p.ragged && !p.out_f32;
}

cudaError_t launch_conv_tc_main(const ConvParams& p_in, const CUtensorMap& wmap, cudaStream_t s);

// Split-K for layers with few output tiles (small batch, 7-14 px stages):
// the K range of each tile is split over idle SMs, partial sums meet in a
// fp32 workspace (one slice per K range), conv_finish_kernel adds them and
// applies the epilogue.  The
// caller (engine) then encodes the weight map for single-CTA tiles.
int conv_tc_splits(const ConvParams& p) {
  // (not the classifier: one 64-row tile of a short-K GEMM gains less than
  // the extra launch costs)
  if (!p.ws || p.ragged || p.out_f32 || (p.cout_max & 7) != 0 || resident_b(p) ||
      (tc_debug() & 131072))
    return 1;
  const long tiles = static_cast<long>((p.M + TC_BM - 1) / TC_BM) * ((p.cout_max + p.bn - 1) / p.bn);
  const int nk_max = p.k_max * p.k_max * ((p.cin_max + TC_BK - 1) / TC_BK);
  // worth a second kernel only when each split still streams >= 8 K blocks
  // and the unsplit tile is long (>= 32 K blocks, ~10 us of operand feed)
  if (tiles * 2 > num_sms() || nk_max < 32) return 1;
  long sp = num_sms() / tiles;
  sp = std::min<long>(sp, nk_max / 8);
  sp = std::min<long>(sp, 16);
  sp = std::min<long>(sp, SSN_SPLIT_WS_FLOATS / (static_cast<long>(p.M) * p.cout_max));
  return sp >= 2 ? static_cast<int>(sp) : 1;
}

cudaError_t launch_conv_finish(const ConvParams& p, cudaStream_t s) {
  const long n = static_cast<long>(p.M) * (p.cout_max / 8);
  const long g = std::min<long>((n + 255) / 256, static_cast<long>(num_sms()) * 8);
  return launch_pdl(conv_finish_kernel, dim3(static_cast<unsigned>(g > 0 ? g : 1)), dim3(256), 0, s, 1, p);
}

cudaError_t launch_conv_tc(const ConvParams& p_in, const CUtensorMap& wmap, cudaStream_t s) {
  if (p_in.splits > 1) {
    cudaError_t e = launch_conv_tc_main(p_in, wmap, s);
    return e != cudaSuccess ? e : launch_conv_finish(p_in, s);
  }
  return launch_conv_tc_main(p_in, wmap, s);
}

cudaError_t launch_conv_tc_main(const ConvParams& p_in, const CUtensorMap& wmap, cudaStream_t s) {
  const int dbg = tc_debug();
  ConvParams p = p_in;
  p.dbg = dbg;
  // Resident B: the max-shape slice is one N tile (so is every subnet's) and
  // all its K blocks fit TC_RB_BYTES.
  const bool resb = resident_b(p);
  // two K blocks per stage on unsplit streamed-B layers with >= SSN_TC_KPS2_NK
  // (16) K blocks
  static const int kps2_nk = [] {
    const char* e = getenv("SSN_TC_KPS2_NK");
    return e ? atoi(e) : 16;
  }();
  const long nk_max = static_cast<long>(p.k_max) * p.k_max * ((p.cin_max + TC_BK - 1) / TC_BK);
  const bool kps2 = kps2_nk > 0 && nk_max >= kps2_nk && !resb && p.splits <= 1;
  if (p.bn <= 64) {
    if (resb) return launch_impl<64, 4, 1, 1>(p, wmap, s);
    return kps2 ? launch_impl<64, 3, 2, 0>(p, wmap, s) : launch_impl<64, 7, 1, 0>(p, wmap, s);
  }
  if (p.bn <= 128) {
    if (resb) return launch_impl<128, 4, 1, 1>(p, wmap, s);
    if (p.cg2)  // bn == 128 pair tiles
      return kps2 ? launch_impl<128, 3, 2, 0, 2>(p, wmap, s) : launch_impl<128, 7, 1, 0, 2>(p, wmap, s);
    return kps2 ? launch_impl<128, 2, 2, 0>(p, wmap, s) : launch_impl<128, 5, 1, 0>(p, wmap, s);
  }
  if (p.bn <= 192 && !resb && !(dbg & 524288)) {  // 144..192-wide tiles: deeper rings than BN 256
    if (p.cg2)
      return kps2 ? launch_impl<192, 3, 2, 0, 2>(p, wmap, s) : launch_impl<192, 6, 1, 0, 2>(p, wmap, s);
    if (p.res && p.rres && p.splits <= 1 && !(dbg & 4194304))
      return launch_impl<192, 3, 1, 3>(p, wmap, s);  // streamed B + residual ring
    return kps2 ? launch_impl<192, 2, 2, 0>(p, wmap, s) : launch_impl<192, 4, 1, 0>(p, wmap, s);
  }
  if (resb && p.res && p.rres && !(dbg & 2097152) &&
      static_cast<long>(p.k_max) * p.k_max * ((p.cin_max + TC_BK - 1) / TC_BK) * p.bn * TC_BK * 2 <=
          TC_RB2_BYTES)
    return launch_impl<256, 2, 1, 2>(p, wmap, s);  // residual through the TMA ring
  if (resb) return launch_impl<256, 4, 1, 1>(p, wmap, s);
  // bn > 128: pair tiles (cta_group::2) unless SSN_TC_DEBUG & 16384
  if (p.cg2) return launch_impl<256, 5, 1, 0, 2>(p, wmap, s);  // (a 2-stage KPS = 2 ring measured slower)
  return launch_impl<256, 3, 1, 0>(p, wmap, s);
}

}  // namespace ssn
