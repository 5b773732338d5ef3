// device.cuh — device-side structures and sm_100a PTX wrappers shared by the
// SubNetAct kernels (tcgen05 / TMEM / TMA / mbarrier / cp.async).
#pragma once

#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssn {

// Per-(subnet, op) dynamic descriptor: the WeightSlice extents and the
// SubnetNorm row of the ACTUATED subnet.  Kernels read it at run time through
// a device word that ssn_actuate() re-points, so CUDA-graph segments never
// need re-instantiation when the subnet changes.
struct alignas(64) OpDesc {
  // TMA im2col map over this op's input activation as THIS subnet lays it out
  // (compact NHWC, cin_a channels; bf16 tcgen05 convs only).  64-byte aligned
  // in global memory so the TMA unit can use it in place.
  CUtensorMap amap;
  int cin;             // active input channels (WeightSlice)
  int cout;            // active output channels
  int k;               // active kernel size (centre crop of k_max)
  int pad;             // k / 2
  const float* scale;  // SubnetNorm folded scale [cout] (NULL = 1)
  const float* shift;  // SubnetNorm folded shift / bias [cout] (NULL = 0)
  int aux;             // OP_SE: active squeeze width
  // residual source of a bf16 tcgen05 conv as THIS subnet lays it out:
  // 2-D tiled map over [rows][cout_a], box {32 columns, 128 rows} (conv_tc
  // RESB = 2 streams it through a shared-memory ring)
  CUtensorMap rmap;
  // WeightSlice B operand of a tcgen05 conv at THIS subnet's tile width:
  // box {64 ch, 1 tap, wrows} over the shared max-shape weights (wrows =
  // the active tile width / CTAs per tile; 0 = use the graph's map)
  CUtensorMap wmap;
  int wrows;
  // conv_hp (shifted-window pair kernel): B of one FILTER ROW (3 taps) per
  // box {64 ch, hrows, 3 taps} at this subnet's tile width (0 = graph map)
  CUtensorMap hmap;
  int hrows;
  // conv_tc output as THIS subnet lays it out: 2-D tiled map over
  // [rows][cout_a], box {32 columns, 32 rows}, 64-byte swizzle — the epilogue
  // stores each warp's bf16 32 x 32 chunk with one TMA store
  CUtensorMap ymap;
  // activation row strides (elements) of this op's input and output/residual
  // buffers as THIS subnet lays them out: bf16 CNN activations pad rows to 32
  // bytes (act_ld: 16-channel multiples) — 16-byte-aligned rows (widths
  // = 8 mod 16) slowed every TMA read of them by up to 1.6x
  int ldi, ldo;
};

// Active N-tile width of a tcgen05 conv: the graph-baked width bn_g (sized
// for the max shape) shrinks to the active output width, keeping the tile
// count, so a narrow subnet issues no MMA columns (and loads no weight rows)
// past cout_a.  Multiples of 16 per CTA (MMA N granularity).
__host__ __device__ __forceinline__ int conv_bn_active(int bn_g, int cout, int cg) {
  const int q = 16 * cg;
  const int nt = (cout + bn_g - 1) / bn_g;
  int b = (cout + nt - 1) / nt;
  b = (b + q - 1) / q * q;
  return b < bn_g ? b : bn_g;
}

// GELU / tanh are out of line: inlined into the unrolled GEMM epilogues their
// erff/tanhf bodies tripled the conv kernel's SASS and thrashed the I-cache.
static __device__ __noinline__ float act_apply_cold(float v, int act) {
  if (act == 3) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));  // GELU (erf)
  if (act == 4) return tanhf(v);
  return v;
}

// GELU (erf form) inline for the GEMM epilogue: erf by Abramowitz & Stegun
// 7.1.26 (|error| <= 1.5e-7, one MUFU.RCP + one MUFU.EX2 + 7 FMA) — the
// out-of-line erff call per element made BERT's FFN-up epilogue (25 M GELUs
// per bs64 layer) issue-bound.  The difference to erff is ~1e-7 absolute,
// far below the bf16 rounding of the stored activation.
__device__ __forceinline__ float gelu_erf_fast(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = __fdividef(1.f, fmaf(0.3275911f, z, 1.f));
  float q = fmaf(1.061405429f, t, -1.453152027f);
  q = fmaf(q, t, 1.421413741f);
  q = fmaf(q, t, -0.284496736f);
  q = fmaf(q, t, 0.254829592f);
  const float e = 1.f - q * t * __expf(-z * z);  // erf(|x| / sqrt(2))
  return 0.5f * x * (1.f + copysignf(e, x));
}

// h_swish(x) = x * relu6(x + 3) / 6 ; h_sigmoid(x) = relu6(x + 3) / 6
__device__ __forceinline__ float act_apply(float v, int act) {
  if (act == 1) return fmaxf(v, 0.f);
  if (act == 2) return v * fminf(fmaxf(v + 3.f, 0.f), 6.f) * (1.f / 6.f);
  if (act == 0) return v;
  return act_apply_cold(v, act);
}

// Transformer ops (config 5): token embedding + LayerNorm, attention, LayerNorm
struct EmbedParams {
  const int* ids;        // [n][s] token ids
  const void* tok;       // bf16 [vocab][hid]
  const void* pos;       // bf16 [512][hid]
  const void* typ;       // bf16 [2][hid]
  const float* gamma;
  const float* beta;
  void* y;               // bf16 [n*s][hid]
  int n, s, hid, vocab;
};

struct LnParams {
  const void* x;  // bf16 [rows][hid]
  void* y;
  const float* gamma;
  const float* beta;
  int rows, hid;
};

struct AttnParams {
  const void* q;  // bf16 [n*s][c], c = heads_a * 64 (active)
  const void* k;
  const void* v;
  void* o;
  const OpDesc* const* row;
  int op;
  int n, s;
};

struct Token0Params {
  const void* x;  // bf16 [n][s][c]
  void* y;        // bf16 [n][c]
  int n, s, c;
};

// Squeeze-excite parameters (OFA DynamicSE): weights are leading slices of
// the max-shape reduce [se_max][c_max] / expand [c_max][se_max] tensors.
struct SEParams {
  void* x;                // NHWC bf16 [n][hw][C], scaled in place
  float* pooled;          // [n][c_max] scratch
  float* gate;            // [n][c_max] scratch
  const void* w_reduce;   // bf16 [se_max][c_max]
  const float* b_reduce;  // [se_max]
  const void* w_expand;   // bf16 [c_max][se_max]
  const float* b_expand;  // [c_max]
  const OpDesc* const* row;
  int op;
  int n, hw, c_max, se_max;
  int w_ld;  // row stride of the reduce tensor (this op's max channels)
  // > 0: the producing depthwise kernel already summed the activation per
  // tile into parts_buf [n][parts][c_max]; the pool pass only adds the parts
  int parts;
  const float* parts_buf;
};

// Static (graph-baked) parameters of one conv op.
// split-K workspace: fp32 [splits][M][cout_a]; splits x tiles <= num_sms
// output tiles of <= 128 x 256 (conv_tc_splits)
constexpr long SSN_SPLIT_WS_FLOATS = 148L * 128 * 256;

struct ConvParams {
  const void* x;      // NHWC, stride = desc.cin
  void* y;            // NHWC, stride = desc.cout
  const void* res;    // NHWC, stride = desc.cout (or NULL)
  const void* w;      // max-shape weights (SIMT paths); TMA map for tcgen05
  const OpDesc* const* row;  // -> active subnet's descriptor row
  const OpDesc* fixed;       // non-NULL: use this descriptor (operator API)
  int op;
  int n, h, w_, ho, wo, stride;
  int M;              // n * ho * wo
  int k_max, cin_max, cout_max;
  int act, res_post, out_f32, depthwise;
  int bn;             // N tile (tcgen05 path)
  int ragged;         // some active cout may be % 8 != 0 (scalar epilogue tail)
  int cg2;            // weight map boxes hold bn/2 rows: 2-CTA pair tiles (conv_tc CG = 2)
  // halo kernel (conv_halo.cu): resident weight box rows / K chunks, A ring depth
  int hb_rows, hb_chunks, h_stages;
  int h_smem;         // conv_halo: dynamic shared memory past the 1 KB alignment slack
  // split-K (conv_tc): `splits` K ranges per tile write raw fp32 sums to
  // `ws` ([splits][M][cout_a]); conv_finish_kernel adds them + the epilogue
  int splits;
  float* ws;
  int rres;           // the descriptor row carries rmap for this op (engine)
  int ystore;         // conv_tc: descriptor rows carry ymap (TMA-store epilogue)
  int dbg;            // profiling knob (SSN_TC_DEBUG): 1 = epilogue skips global
                      // memory, 2 = no MMA issued (bottleneck isolation only)
  // depthwise (dw.cu): TMA stage ring, and the fused squeeze-excite pool:
  // per-tile channel sums of the stored activation -> pool[n][tile][pool_ld]
  int dw_stages, dw_stage_bytes;
  float* pool;
  int pool_ld;
};


// Halo ("shifted-window") geometry of a stride-1 k x k conv over a W-wide
// image: output positions are taken in PADDED-width row-major order (Wp =
// W + k - 1 columns, k - 1 of them garbage), so tap (r, s) of position p reads
// padded input pixel p + r*Wp + s: a plain row offset into ONE smem window.
// A tile is RT whole padded rows (<= 128 positions); its window is R rows,
// enough that all 128 MMA rows of every tap stay inside the window.
struct HaloGeom {
  int wp, rt, r;
};
__host__ __device__ __forceinline__ HaloGeom halo_geom(int w, int k) {
  HaloGeom g;
  g.wp = w + k - 1;
  g.rt = g.wp >= 128 ? 1 : 128 / g.wp;
  g.r = (128 + (k - 1) * (g.wp + 1) + g.wp - 1) / g.wp;
  return g;
}

struct PoolParams {
  const void* x;
  void* y;
  const OpDesc* const* row;
  int op;
  int n, h, w, ho, wo, k, stride, pad;
  int kind;  // 2 max, 3 avg (ceil), 4 gap
};

struct InputParams {
  const void* raw;
  void* y;
  int n, h, w;
  int format;   // ssn_input_format
  int cpad;     // output channels (3 f32 / 8 bf16)
  int out_bf16;
  int im2col_k;           // > 0: emit the k x k / stride im2col (bf16, cpad channels)
  int im2col_stride;
  int ho, wo;
};

// Input staging fused with the bf16 im2col stem conv (3x3, stride 2, 3 input
// channels, K = 27 padded to 32): raw images -> the conv's output directly.
struct StemParams {
  const void* raw;
  void* y;
  const OpDesc* const* row;
  int op;                   // the stem conv's op index (WeightSlice cout, SubnetNorm)
  const void* w;            // [cout_max][32] im2col-order weights
  int n, h, w_, ho, wo;
  int format;               // ssn_input_format
  int act;
};

struct OpDims {
  int cin, cout, k, pad;
  const float* scale;
  const float* shift;
  int ldi, ldo;  // input / output row strides (elements)
};

__device__ __forceinline__ const OpDesc* desc_ptr(const OpDesc* const* row, const OpDesc* fixed,
                                                  int op) {
  return fixed ? fixed : (*row + op);
}

__device__ __forceinline__ OpDims load_desc(const OpDesc* const* row, const OpDesc* fixed, int op) {
  const OpDesc* r = desc_ptr(row, fixed, op);
  return OpDims{r->cin, r->cout, r->k, r->pad, r->scale, r->shift, r->ldi, r->ldo};
}

// ---------------------------------------------------------------------------
// PTX wrappers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Bounded: a pipeline bug (e.g. an expect_tx byte count that the TMA never
// delivers) traps after ~2^30 polls (tens of seconds) instead of hanging the
// GPU until the process is killed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  do {
    if (++spins == (1u << 30)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// TMA: 3-D tiled load into shared memory, completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// TMA store of a shared-memory box (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}

// TMA im2col: pixelsPerColumn output pixels x channelsPerPixel channels of
// filter tap (off_w, off_h), starting at input coordinate (c, w, h, n).
__device__ __forceinline__ void tma_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                              int c, int w, int h, int n, uint16_t off_w,
                                              uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3), "r"(c4)
      : "memory");
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; it must not touch upstream data before pdl_wait().
// pdl_trigger() lets the NEXT kernel start its own prologue early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// One lane of a converged warp (elect.sync): keeps the issue loop warp-uniform.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// cp.async 16 B with zero fill (src_bytes = 0 -> 16 zero bytes).
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Arrive on `bar` once every cp.async this thread issued so far has landed
// (the barrier's expected count includes this arrival).
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// tcgen05 -----------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate, M = 128.
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Same MMA issued from a CONVERGED warp: elect.sync inside the asm picks the
// issuing lane, so the descriptors stay in uniform registers.  With
// descriptors formed by adding 16-byte offsets to a base descriptor this
// reaches the tensor-pipe floor (44/48/56/64 cycles per M=128,K=16 MMA at
// N=48/64/96/128); an `if (lane == 0)` issue wraps every UTCHMMA in an R2UR
// waterfall and costs 70-100 cycles per MMA (tools/ubench/tc_issue3.cu).
__device__ __forceinline__ void tc_mma_bf16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---- 2-CTA (cta_group::2) variants: the CTA pair of a cluster shares one
// M=256 MMA; A rows 0-127 / 128-255 and the two halves of B live in the two
// CTAs' shared memory at the same offsets; D lives in both CTAs' TMEM.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of `bar` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_cnt(uint32_t cluster_addr, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(count)
               : "memory");
}
// TMA loads of either CTA completing on the LEADER's mbarrier (peer bit cleared)
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma2_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1),
      "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma2_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                             int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1),
      "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma2_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c,
                                               int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c), "r"(w),
      "r"(h), "r"(n), "h"(off_w), "h"(off_h)
      : "memory");
}
__device__ __forceinline__ void tc2_mma_bf16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                   uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit arriving on the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void tc2_commit_mc_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], m;\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem2_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem2_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 columns of fp32 from TMEM (each thread: its lane, 32 cols).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B
// apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(16 >> 4) << 16;    // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO
  d |= static_cast<uint64_t>(1) << 46;          // version
  d |= static_cast<uint64_t>(2) << 61;          // SWIZZLE_128B
  return d;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B: 64-byte rows (32 bf16),
// 8-row atoms 512 B apart (SBO); K step of 16 = +32 B (+2 in the address field).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(16 >> 4) << 16;   // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(512 >> 4) << 32;  // SBO
  d |= static_cast<uint64_t>(1) << 46;         // version
  d |= static_cast<uint64_t>(4) << 61;         // SWIZZLE_64B
  return d;
}

// UMMA shared-memory descriptor: K-major, no swizzle ("interleave"): 8-row x
// 16-byte core matrices, N-adjacent core matrices `sbo` bytes apart,
// K-adjacent ones `lbo` bytes apart.
__device__ __forceinline__ uint64_t umma_desc_noswz(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version; layout type 0 = SWIZZLE_NONE
  return d;
}

// Instruction descriptor: kind::f16, A/B bf16, D f32, K-major, M=m (128, or
// 256 for cta_group::2), N=n.
__host__ __device__ __forceinline__ uint32_t umma_idesc_bf16(int n, int m = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// Legacy warp MMA (D += A B, m16n8k16, bf16 in / fp32 accumulate) for small
// fused kernels (attention, the CNN stem) where tcgen05 setup would dominate.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               const uint32_t b0, const uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// bf16x2 {lo = relu(a), hi = relu(b)} in one cvt (ReLU fused into the rounding)
__device__ __forceinline__ uint32_t pack_bf16x2_relu(float a, float b) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

#ifdef __CUDACC__
// Host: launch `k` with programmatic stream serialization (PDL; graph capture
// turns it into a programmatic edge), optionally as 2-CTA clusters.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  static const bool no_pdl = getenv("SSN_NO_PDL") != nullptr;  // debugging: plain stream order
  if (!no_pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, args...);
}
#endif

}  // namespace ssn
