// engine.cu — the SubNetAct execution engine behind the C-ABI of include/ssn.h.
//
// What replaces the reference's mock worker (serve_runtime.hpp:161-172):
//  * weight store   — every max-shape conv/linear tensor uploaded ONCE
//                     (layers "shared in place");
//  * SubnetNorm     — per registered subnet, (gamma, beta, mu_ij, var_ij) folded
//                     into a scale/shift row;
//  * WeightSlice    — per-subnet OpDesc rows give every kernel its active
//                     extents; kernels read leading slices of the store;
//  * LayerSelect    — per (segment, depth-variant, batch) CUDA graphs built in
//                     ssn_prepare(); a forward launches only the variants whose
//                     blocks the subnet runs;
//  * actuation      — ssn_actuate(id) re-points one device word at the
//                     subnet's OpDesc row (one 1-thread kernel at the next
//                     forward); no weight moves.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ssn.h"
#include "../../include/ssn_rng.h"
#include "device.cuh"
#include "supernet.hpp"

namespace ssn {
int make_weight_map(CUtensorMap* map, const void* w, int cin_store, int taps, int cout, int bn);
int make_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld, int k,
                 int stride, int pad);
int choose_bn(int cout_max, long M, int nk_max);
bool conv_tc_use_pairs(const ConvParams& p);
int conv_tc_splits(const ConvParams& p);
int make_res_map(CUtensorMap* map, const void* r, long rows, int cout, int ld);
int make_y_map(CUtensorMap* map, void* y, long rows, int cout, int ld);
cudaError_t launch_conv_tc(const ConvParams& p, const CUtensorMap& wmap, cudaStream_t s);
cudaError_t init_conv_tc();
cudaError_t init_conv_halo();
bool halo_eligible(int h, int w, int k_max, int stride, int cin_max, int cout_max);
int make_halo_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld, int k);
int make_halo_weight_map(CUtensorMap* map, const void* wgt, int cin_store, int taps, int cout,
                         int rows, int chunks);
cudaError_t launch_conv_halo(ConvParams p, const void* wgt, int cin_store, int taps, cudaStream_t s);
cudaError_t init_conv_hp();
bool hp_eligible(int h, int w, int k_max, int stride, int cin_max, int cout_max, bool graph);
int make_hp_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int cin, int ld);
int hp_choose_bn(int cout_max);
int make_hp_weight_map(CUtensorMap* map, const void* w, int cin_store, int taps, int cout, int rows);
cudaError_t launch_conv_hp(ConvParams p, const CUtensorMap& wmap, cudaStream_t s);
cudaError_t launch_input(const InputParams& p, cudaStream_t s);
cudaError_t launch_stem_conv(const StemParams& p, cudaStream_t s);
cudaError_t launch_pool(const PoolParams& p, int max_c, bool bf16, cudaStream_t s);
cudaError_t launch_conv_f32(const ConvParams& p, cudaStream_t s);
cudaError_t launch_set_row(const OpDesc** slot, const OpDesc* row, cudaStream_t s);
cudaError_t launch_dw_bf16(const ConvParams& p, cudaStream_t s);
int make_dw_act_map(CUtensorMap* map, const void* x, int n, int h, int w, int c, int ld, int k,
                    int stride, int wo, int c_max);
int dw_tiles_per_image(int stride, int ho, int wo);
bool dw_supported(int k_max, int k, int stride);
cudaError_t launch_se(const SEParams& p, cudaStream_t s);
cudaError_t launch_embed(const EmbedParams& p, cudaStream_t s);
cudaError_t launch_layernorm(const LnParams& p, cudaStream_t s);
cudaError_t launch_token0(const Token0Params& p, cudaStream_t s);
cudaError_t launch_attention(const AttnParams& p, int max_heads, bool tc, cudaStream_t s);
int make_attn_map(CUtensorMap* map, const void* x, long rows, int c);
}  // namespace ssn

using namespace ssn;

// ---------------------------------------------------------------------------
// errors

static thread_local std::string g_last_error;

struct SsnError {
  int code;
  std::string msg;
};

#define SSN_THROW(code, msg) throw SsnError{code, msg}
#define CUDA_TRY(expr)                                                          \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess)                                                      \
      SSN_THROW(SSN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return SSN_OK;
  } catch (const SsnError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return SSN_E_INVALID;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return SSN_E_RANGE;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return SSN_E_NOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SSN_E_INVALID;
  }
}

// ---------------------------------------------------------------------------
// engine

static constexpr int NBUF = 8;  // BND0, BND1, P, T1..T5
enum { B_BND0 = 0, B_BND1 = 1, B_P = 2, B_T1 = 3, B_T2 = 4, B_T3 = 5, B_T4 = 6, B_T5 = 7 };

struct SubnetState {
  bool ok = false;
  Net plan;
  OpDesc* d_row = nullptr;
  float* d_norm = nullptr;
  uint64_t norm_bytes = 0;
  uint64_t stat_bytes = 0;
  std::vector<uint32_t> seg_mask;
  // Per segment: graph variant (LayerSelect mask | SEG_FLIP when the input sits
  // in the other boundary buffer because an earlier segment ran no block) and
  // whether any block of the segment runs at all.
  std::vector<uint32_t> seg_var;
  std::vector<uint8_t> seg_run;
};

// Variant bit: the segment's input is in the boundary buffer of the opposite
// parity (an earlier segment was skipped entirely and passed its input on).
constexpr uint32_t SEG_FLIP = 1u << 15;

struct ssn_engine {
  int device = 0;
  ssn_supernet_desc desc{};
  Net net;  // max-shape plan
  bool bf16 = true;
  uint8_t* d_w = nullptr;
  float* d_ws = nullptr;  // split-K partial sums (bf16 engines)
  std::vector<std::vector<float>> gamma, beta;  // host copies for SubnetNorm folding
  std::vector<SubnetState> subs;
  const OpDesc** d_rowptr = nullptr;
  int active = -1;
  bool dirty = false;
  void* bufs[NBUF] = {};
  size_t buf_bytes = 0;
  void* d_raw = nullptr;
  size_t raw_img_bytes = 0;
  // Host inputs are staged through two device buffers on a copy stream, so
  // the H2D of forward i+1 overlaps the graphs of forward i; a 2-slot ring
  // guarded by events, then one device copy into d_raw (which the graphs read).
  void* d_stage[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t stage_ready[2] = {nullptr, nullptr};
  cudaEvent_t stage_free[2] = {nullptr, nullptr};
  int stage_slot = 0;
  float* d_logits = nullptr;
  float* d_se = nullptr;  // squeeze-excite scratch: pooled + gate [max_batch][se_cmax]
  float* d_separt = nullptr;  // SE pool partials of the depthwise kernel [max_batch][tiles][se_cmax]
  int se_cmax = 0;
  std::vector<uint32_t> grid;
  std::map<uint64_t, std::pair<cudaGraphExec_t, int>> graphs;  // key -> (exec, kernels)
  // Whole-forward graphs: every running segment of one LayerSelect variant
  // vector captured back to back at one batch, so the programmatic (PDL)
  // edges continue across segment boundaries (separately launched segment
  // graphs drain at each boundary).  key = (per-segment variant | not-run,
  // batch); shared by every registered subnet with the same variant vector.
  std::map<std::vector<uint32_t>, std::pair<cudaGraphExec_t, int>> fgraphs;
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  // Cross-stream ordering: forwards share engine state (the active-row word,
  // the arena, d_raw, d_logits, the staging slots), so a call enqueued on a
  // different stream than the previous one first waits for that one's work.
  cudaEvent_t last_done = nullptr;
  cudaStream_t last_stream = nullptr;
  double last_actuate_us = 0, last_forward_host_us = 0;
  uint32_t last_kernels = 0, last_graphs = 0;
  bool prepared = false;
};

// Order `s` after the engine's previous call when that call used another stream.
static void order_stream(ssn_engine* e, cudaStream_t s) {
  if (e->last_stream != nullptr && e->last_stream != s)
    CUDA_TRY(cudaStreamWaitEvent(s, e->last_done, 0));
}

static void mark_done(ssn_engine* e, cudaStream_t s) {
  CUDA_TRY(cudaEventRecord(e->last_done, s));
  e->last_stream = s;
}

static uint64_t graph_key(int seg, uint32_t mask, uint32_t batch) {
  return (static_cast<uint64_t>(seg) << 48) | (static_cast<uint64_t>(mask) << 32) | batch;
}

static size_t raw_image_bytes(const ssn_supernet_desc& d) {
  const size_t px = static_cast<size_t>(d.image_size) * d.image_size;
  if (d.family == SSN_FAMILY_BERT) return static_cast<size_t>(d.image_size) * 4;  // int32 ids
  return d.input_format == SSN_INPUT_U8_NHWC ? px * 3 : px * 3 * 4;
}

static void validate_desc(const ssn_supernet_desc* d) {
  if (!d) SSN_THROW(SSN_E_INVALID, "null supernet descriptor");
  if (d->family != SSN_FAMILY_TINYCNN && d->family != SSN_FAMILY_OFA_RESNET50 &&
      d->family != SSN_FAMILY_OFA_MBV3 && d->family != SSN_FAMILY_BERT)
    SSN_THROW(SSN_E_INVALID, "unsupported supernet family " + std::to_string(d->family));
  if (d->dtype != SSN_DTYPE_F32 && d->dtype != SSN_DTYPE_BF16)
    SSN_THROW(SSN_E_INVALID, "dtype must be SSN_DTYPE_F32 or SSN_DTYPE_BF16");
  if (d->image_size < 8 || d->image_size > 1024) SSN_THROW(SSN_E_INVALID, "image_size out of range");
  if (d->num_classes < 1 || d->num_classes > 100000) SSN_THROW(SSN_E_INVALID, "num_classes out of range");
  if (d->max_batch < 1) SSN_THROW(SSN_E_INVALID, "max_batch must be >= 1");
  if (d->input_format > SSN_INPUT_U8_NHWC) SSN_THROW(SSN_E_INVALID, "bad input_format");
}

// Fill a blob following DESIGN.md §4 from the ssn_rng.h specification.
static void generate_blob(const Net& net, uint8_t* blob) {
  const uint64_t seed = net.desc.seed;
  const bool bf16 = net.elem_bytes == 2;
  std::memset(blob, 0, net.blob_bytes);
  for (size_t ti = 0; ti < net.tensors.size(); ++ti) {
    const TensorSpec& t = net.tensors[ti];
    const int kk = t.k * t.k;
    for (int o = 0; o < t.cout; ++o)
      for (int i = 0; i < t.cin; ++i)
        for (int r = 0; r < t.k; ++r)
          for (int s = 0; s < t.k; ++s) {
            const uint64_t idx = ((static_cast<uint64_t>(o) * t.cin + i) * t.k + r) * t.k + s;
            const float v = ssn_weight_value(seed, static_cast<uint32_t>(ti), idx, t.fan_in, bf16);
            // storage: KRSC [cout][k][k][cin_store] (depthwise: [c][k][k])
            // im2col stem: [cout][(r*k+s)*cin + c] padded to cin_store
            // bf16 depthwise: tap-major [k][k][c] (16-byte channel vectors)
            const uint64_t e =
                t.im2col_stem
                    ? static_cast<uint64_t>(o) * t.cin_store + (r * t.k + s) * t.cin + i
                : (t.depthwise && bf16)
                    ? static_cast<uint64_t>(r * t.k + s) * t.cout + o
                    : (static_cast<uint64_t>(o) * kk + r * t.k + s) * t.cin_store + i;
            if (bf16) {
              reinterpret_cast<uint16_t*>(blob + t.w_off)[e] = ssn_f32_to_bf16_bits(v);
            } else {
              reinterpret_cast<float*>(blob + t.w_off)[e] = v;
            }
          }
    if (t.linear)
      for (int o = 0; o < t.cout; ++o)
        reinterpret_cast<float*>(blob + t.b_off)[o] =
            ssn_bias_value(seed, static_cast<uint32_t>(ti), o);
  }
  for (size_t ni = 0; ni < net.norms.size(); ++ni) {
    const NormSpec& n = net.norms[ni];
    for (int c = 0; c < n.c; ++c) {
      reinterpret_cast<float*>(blob + n.gamma_off)[c] =
          n.res ? ssn_gamma_res_value(seed, static_cast<uint32_t>(ni), c)
                : ssn_gamma_value(seed, static_cast<uint32_t>(ni), c);
      reinterpret_cast<float*>(blob + n.beta_off)[c] =
          ssn_beta_value(seed, static_cast<uint32_t>(ni), c);
    }
  }
}

static void* slot_ptr(ssn_engine* e, int slot, const int* map) {
  switch (slot) {
    case S_NONE: return nullptr;
    case S_RAW: return e->d_raw;
    case S_LOGITS: return e->d_logits;
    default: return e->bufs[map[slot]];
  }
}

// Row stride (elements) of a `c`-channel activation buffer.  Every kernel of
// the bf16 CNN path addresses activations through the descriptor row's
// ldi / ldo and every TMA map takes the stride separately, so rows can be
// padded to 16-channel multiples (32-B rows) once they are >= 256 channels
// wide.  OFA widths are make_divisible(., 8), so 360, 408, 264, 664, 1640 ...
// have rows aligned to 16 B only, and TMA reads such rows at about half rate
// whatever the box mode (tools/ubench/tma_modes.cu: a 3x3 A operand over
// 360-channel pixels 32 B/cycle/SM, over 368 or 384 channels 52-72); below
// 256 channels the layers are HBM-bound and the extra bytes cost more than
// the faster reads return (padding every row measured -0.8% on the R50
// sweep, >= 256 only +0.7%; OFA-MBv3 unchanged).  SSN_PAD_ROWS = t sets the
// threshold (1 = every row, 0 = compact rows).  Pad channels are never read
// as data: TMA maps bound the channel dimension at the active width, the
// vector epilogues touch c columns.
static int act_ld(const ssn_engine* e, int c) {
  static const int pad_min = [] {
    const char* v = getenv("SSN_PAD_ROWS");
    return v ? atoi(v) : 256;
  }();
  if (pad_min <= 0 || !e->bf16 || e->desc.family == SSN_FAMILY_BERT || c < 16 || c < pad_min) return c;
  return (c + 15) & ~15;
}

// Enqueue one op (called under stream capture).
// Narrow stride-1 3x3 convs (OFA-R50 stem and stage 1) run the shifted-window
// kernel with resident weights (conv_halo.cu); the choice depends only on the
// op's max shape, so one graph serves every subnet.
static bool use_halo(const ssn_engine* e, const OpSpec& o) {
  if (!e->bf16 || o.kind != OP_CONV || o.depthwise || o.act > 1 || (o.cout_max & 7) != 0)
    return false;
  const TensorSpec& t = e->net.tensors[o.tensor];
  if (t.im2col_stem) return false;
  return halo_eligible(o.hin, o.win, o.k_max, o.stride, t.cin_store, o.cout_max);
}

// Wider stride-1 3x3 convs without a residual (OFA-R50 3x3 at 28 / 14 px)
// run the 2-CTA shifted-window kernel (conv_hp.cu); same max-shape rule.
static bool use_hp(const ssn_engine* e, const OpSpec& o, uint32_t batch) {
  // bs 1-2: conv_tc's split-K spreads the few tiles better for the wide
  // (max-subnet) layers (bs1 max 635 vs 651 us); from 4 images on the pair
  // kernel wins for every subnet (bs4 mid 514 -> 491, bs16 mid 657 -> 628,
  // bs16 max 936 -> 911 us; SSN_HP_MIN_BATCH overrides)
  static const uint32_t min_batch = [] {  // A/B knob (SSN_HP_MIN_BATCH)
    const char* v = getenv("SSN_HP_MIN_BATCH");
    return v ? static_cast<uint32_t>(atoi(v)) : 4u;
  }();
  if (batch < min_batch) return false;
  if (!e->bf16 || o.kind != OP_CONV || o.depthwise || o.act > 1 || o.res != S_NONE ||
      (o.cout_max & 7) != 0 || use_halo(e, o))
    return false;
  const TensorSpec& t = e->net.tensors[o.tensor];
  if (t.im2col_stem) return false;
  return hp_eligible(o.hin, o.win, o.k_max, o.stride, t.cin_store, o.cout_max, true);
}

static int tc_debug_flags() {  // SSN_TC_DEBUG & 65536: unfused stem (profiling only)
  static const int v = [] {
    const char* e = getenv("SSN_TC_DEBUG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// bf16 im2col stem conv `ci` (op 1 of both OFA CNN families) runs fused with
// its input op (stem_conv_kernel): the input op launches nothing.
static bool stem_fused(const ssn_engine* e, int ci) {
  if (!e->bf16 || ci < 1 || ci >= static_cast<int>(e->net.ops.size())) return false;
  const OpSpec& c = e->net.ops[ci];
  const OpSpec& in = e->net.ops[ci - 1];
  return c.kind == OP_CONV && c.tensor >= 0 && e->net.tensors[c.tensor].im2col_stem &&
         in.kind == OP_INPUT && in.k_max == 3 && in.stride == 2 && in.cout_max == 32 &&
         in.win <= 256 && c.cout_max <= 32 && (c.cout_max & 7) == 0 && c.res == S_NONE &&
         !(tc_debug_flags() & 65536);
}

// bf16 depthwise op `di` whose output feeds a squeeze-excite op: the
// depthwise kernel sums the activation per tile (fused SE pool); returns the
// partial count per image, 0 = not fused.
static int se_fused_parts(const ssn_engine* e, int di) {
  if (!e->bf16 || di < 0 || di + 1 >= static_cast<int>(e->net.ops.size())) return 0;
  const OpSpec& d = e->net.ops[di];
  const OpSpec& se = e->net.ops[di + 1];
  if (d.kind != OP_CONV || !d.depthwise || se.kind != OP_SE || se.in != d.out) return 0;
  if (tc_debug_flags() & 1048576) return 0;  // A/B switch: unfused SE pool
  return dw_tiles_per_image(d.stride, d.hout, d.wout);
}

// Graph-independent parameters of conv op `oi` at `batch` images.
static ConvParams conv_static_params(const ssn_engine* e, int oi, uint32_t batch) {
  const OpSpec& o = e->net.ops[oi];
  ConvParams p{};
  p.n = static_cast<int>(batch);
  p.h = o.hin;
  p.w_ = o.win;
  p.ho = o.hout;
  p.wo = o.wout;
  p.stride = o.stride;
  p.M = static_cast<int>(batch) * o.hout * o.wout;
  p.k_max = o.k_max;
  p.cin_max = e->net.tensors[o.tensor].cin_store;
  p.cout_max = o.cout_max;
  p.act = o.act;
  p.res_post = o.res_post;
  p.out_f32 = o.kind == OP_LINEAR;
  p.depthwise = o.depthwise;
  return p;
}

// tcgen05 tiling of conv op `oi` (max-shape N width, split-K, pair tiles):
// shared by graph capture and by subnet registration, which encodes each
// subnet's weight map at the active tile width this tiling implies.
static void conv_tc_tiling(const ssn_engine* e, int oi, ConvParams& p) {
  const OpSpec& o = e->net.ops[oi];
  const TensorSpec& t = e->net.tensors[o.tensor];
  p.bn = choose_bn(o.cout_max, p.M, o.k_max * o.k_max * ((t.cin_store + 63) / 64));
  // classifier head at <= 128 rows: one M tile, so the N width sets the
  // CTA count — 64-wide tiles put 16 SMs (not 4) on the 32 K blocks
  if (o.kind == OP_LINEAR && p.M <= 128 && o.cout_max > 64 && !(tc_debug_flags() & 262144))
    p.bn = 64;
  p.ws = e->d_ws;
  p.rres = o.res != S_NONE && (o.cout_max & 7) == 0;  // every subnet's row carries rmap
  p.splits = conv_tc_splits(p);
  p.cg2 = p.splits > 1 ? 0 : conv_tc_use_pairs(p);
  // every subnet row of a bf16 conv carries ymap (subnet registration)
  p.ystore = o.kind != OP_LINEAR && (o.cout_max & 7) == 0 && p.splits <= 1;
}

static int enqueue_op(ssn_engine* e, int oi, const int* map, uint32_t batch, cudaStream_t s) {
  const OpSpec& o = e->net.ops[oi];
  const bool bf = e->bf16;
  switch (o.kind) {
    case OP_INPUT: {
      if (stem_fused(e, oi + 1)) return 0;  // the stem conv reads the raw images
      InputParams p{};
      p.raw = e->d_raw;
      p.y = slot_ptr(e, o.out, map);
      p.n = static_cast<int>(batch);
      p.h = o.hin;
      p.w = o.win;
      p.format = static_cast<int>(e->desc.input_format);
      p.cpad = o.cout_max;
      p.out_bf16 = bf;
      if (o.hout != o.hin) {  // fused stem im2col (bf16 OFA-ResNet50)
        p.im2col_k = o.k_max;
        p.im2col_stride = o.stride;
      }
      p.ho = o.hout;
      p.wo = o.wout;
      CUDA_TRY(launch_input(p, s));
      return 1;
    }
    case OP_MAXPOOL:
    case OP_AVGPOOL:
    case OP_GAP: {
      PoolParams p{};
      p.x = slot_ptr(e, o.in, map);
      p.y = slot_ptr(e, o.out, map);
      p.row = e->d_rowptr;
      p.op = oi;
      p.n = static_cast<int>(batch);
      p.h = o.hin;
      p.w = o.win;
      p.ho = o.hout;
      p.wo = o.wout;
      p.k = o.kind == OP_AVGPOOL ? o.pool_k : o.k_max;
      p.stride = o.kind == OP_AVGPOOL ? o.pool_k : o.stride;
      p.pad = o.kind == OP_MAXPOOL ? 1 : 0;
      p.kind = o.kind == OP_MAXPOOL ? 2 : (o.kind == OP_AVGPOOL ? 3 : 4);
      CUDA_TRY(launch_pool(p, o.cin_max, bf, s));
      return 1;
    }
    case OP_CONV:
    case OP_LINEAR: {
      const TensorSpec& t = e->net.tensors[o.tensor];
      if (stem_fused(e, oi)) {
        const OpSpec& in = e->net.ops[oi - 1];
        StemParams sp{};
        sp.raw = e->d_raw;
        sp.y = slot_ptr(e, o.out, map);
        sp.row = e->d_rowptr;
        sp.op = oi;
        sp.w = e->d_w + t.w_off;
        sp.n = static_cast<int>(batch);
        sp.h = in.hin;
        sp.w_ = in.win;
        sp.ho = o.hout;
        sp.wo = o.wout;
        sp.format = static_cast<int>(e->desc.input_format);
        sp.act = o.act;
        CUDA_TRY(launch_stem_conv(sp, s));
        return 1;
      }
      ConvParams p = conv_static_params(e, oi, batch);
      p.x = slot_ptr(e, o.in, map);
      p.y = slot_ptr(e, o.out, map);
      p.res = slot_ptr(e, o.res, map);
      p.w = e->d_w + t.w_off;
      p.row = e->d_rowptr;
      p.fixed = nullptr;
      p.op = oi;
      if (bf && use_halo(e, o)) {
        CUDA_TRY(launch_conv_halo(p, p.w, t.cin_store, o.k_max * o.k_max, s));
      } else if (bf && use_hp(e, o, batch)) {
        p.bn = hp_choose_bn(o.cout_max);
        CUtensorMap wmap{};
        if (make_hp_weight_map(&wmap, p.w, t.cin_store, o.k_max * o.k_max, t.cout, p.bn / 2) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled failed for op " + std::to_string(oi));
        CUDA_TRY(launch_conv_hp(p, wmap, s));
      } else if (bf && !o.depthwise) {
        conv_tc_tiling(e, oi, p);
        CUtensorMap wmap{};
        if (make_weight_map(&wmap, p.w, t.cin_store, o.k_max * o.k_max, t.cout,
                            p.cg2 ? p.bn / 2 : p.bn) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled failed for op " + std::to_string(oi));
        CUDA_TRY(launch_conv_tc(p, wmap, s));
        return p.splits > 1 ? 2 : 1;  // + conv_finish_kernel
      } else if (bf) {
        if (se_fused_parts(e, oi) > 0) {
          p.pool = e->d_separt;
          p.pool_ld = e->se_cmax;
        }
        CUDA_TRY(launch_dw_bf16(p, s));
      } else {
        CUDA_TRY(launch_conv_f32(p, s));
      }
      return 1;
    }
    case OP_EMBED: {
      EmbedParams p{};
      p.ids = static_cast<const int*>(e->d_raw);
      p.tok = e->d_w + e->net.tensors[o.tensor].w_off;
      p.pos = e->d_w + e->net.tensors[o.tensor2].w_off;
      p.typ = e->d_w + e->net.tensors[o.tensor3].w_off;
      p.gamma = reinterpret_cast<const float*>(e->d_w + e->net.norms[o.norm].gamma_off);
      p.beta = reinterpret_cast<const float*>(e->d_w + e->net.norms[o.norm].beta_off);
      p.y = slot_ptr(e, o.out, map);
      p.n = static_cast<int>(batch);
      p.s = o.hin;
      p.hid = o.cout_max;
      p.vocab = e->net.tensors[o.tensor].cout;
      CUDA_TRY(launch_embed(p, s));
      return 1;
    }
    case OP_LAYERNORM: {
      LnParams p{};
      p.x = slot_ptr(e, o.in, map);
      p.y = slot_ptr(e, o.out, map);
      p.gamma = reinterpret_cast<const float*>(e->d_w + e->net.norms[o.norm].gamma_off);
      p.beta = reinterpret_cast<const float*>(e->d_w + e->net.norms[o.norm].beta_off);
      p.rows = static_cast<int>(batch) * o.hin * o.win;
      p.hid = o.cout_max;
      CUDA_TRY(launch_layernorm(p, s));
      return 1;
    }
    case OP_TOKEN0: {
      Token0Params p{};
      p.x = slot_ptr(e, o.in, map);
      p.y = slot_ptr(e, o.out, map);
      p.n = static_cast<int>(batch);
      p.s = o.hin;
      p.c = o.cout_max;
      CUDA_TRY(launch_token0(p, s));
      return 1;
    }
    case OP_ATTN: {
      AttnParams p{};
      p.q = slot_ptr(e, o.in, map);
      p.k = slot_ptr(e, o.in2, map);
      p.v = slot_ptr(e, o.in3, map);
      p.o = slot_ptr(e, o.out, map);
      p.row = e->d_rowptr;
      p.op = oi;
      p.n = static_cast<int>(batch);
      p.s = o.hin;
      CUDA_TRY(launch_attention(p, o.cin_max / o.k_max, bf && !(tc_debug_flags() & 8388608), s));
      return 1;
    }
    case OP_SE: {
      SEParams p{};
      p.x = slot_ptr(e, o.in, map);
      p.pooled = e->d_se;
      p.gate = e->d_se + static_cast<size_t>(e->desc.max_batch) * e->se_cmax;
      p.w_reduce = e->d_w + e->net.tensors[o.tensor].w_off;
      p.b_reduce = reinterpret_cast<const float*>(e->d_w + e->net.tensors[o.tensor].b_off);
      p.w_expand = e->d_w + e->net.tensors[o.tensor2].w_off;
      p.b_expand = reinterpret_cast<const float*>(e->d_w + e->net.tensors[o.tensor2].b_off);
      p.row = e->d_rowptr;
      p.op = oi;
      p.n = static_cast<int>(batch);
      p.hw = o.hout * o.wout;
      p.c_max = e->se_cmax;
      p.se_max = o.se_mid_max;
      p.w_ld = o.cin_max;
      p.parts = se_fused_parts(e, oi - 1);
      p.parts_buf = e->d_separt;
      CUDA_TRY(launch_se(p, s));
      return 4;
    }
  }
  SSN_THROW(SSN_E_INVALID, "unknown op kind");
}

// Enqueue LayerSelect variant `mask` of segment `seg`: only the blocks the
// variant runs, with ping-pong buffers so the segment output always lands in
// the next segment's boundary buffer.  `hook(op, before)` brackets each op.
struct SlotMap {
  int op;
  int map[9];
};

// The ops one LayerSelect variant of a segment runs, each with its slot ->
// arena-buffer mapping (used by graph capture AND by ssn_register_subnet to
// encode each op's activation TMA map over the buffer it will really read).
static std::vector<SlotMap> segment_plan(const ssn_engine* e, int seg, uint32_t variant) {
  const SegmentSpec& S = e->net.segments[seg];
  const bool flip = (variant & SEG_FLIP) != 0;
  const uint32_t mask = variant & ~SEG_FLIP;
  std::vector<int> act;
  for (int bi : S.blocks) {
    const BlockSpec& b = e->net.blocks[bi];
    bool on = b.flag < 0;
    if (!on) {
      for (size_t f = 0; f < S.flags.size(); ++f)
        if (S.flags[f] == b.flag) on = (mask >> f) & 1u;
    }
    if (on) act.push_back(bi);
  }
  const bool even = (seg % 2 == 0) != flip;
  const int in_bnd = even ? B_BND0 : B_BND1;
  const int out_bnd = even ? B_BND1 : B_BND0;
  const int k = static_cast<int>(act.size());
  int cur_in = in_bnd;
  std::vector<SlotMap> out;
  for (int i = 0; i < k; ++i) {
    const int out_buf = ((k - 1 - i) % 2 == 0) ? out_bnd : B_P;
    SlotMap sm{};
    sm.map[S_IN] = cur_in;
    sm.map[S_OUT] = out_buf;
    sm.map[S_T1] = B_T1;
    sm.map[S_T2] = B_T2;
    sm.map[S_T3] = B_T3;
    sm.map[S_T4] = B_T4;
    sm.map[S_T5] = B_T5;
    const BlockSpec& b = e->net.blocks[act[i]];
    for (int q = 0; q < b.count; ++q) {
      sm.op = b.first + q;
      out.push_back(sm);
    }
    cur_in = out_buf;
  }
  return out;
}

template <class Hook>
static int enqueue_segment(ssn_engine* e, int seg, uint32_t mask, uint32_t batch, cudaStream_t s,
                           Hook&& hook) {
  int kernels = 0;
  for (const SlotMap& sm : segment_plan(e, seg, mask)) {
    hook(sm.op, true);
    kernels += enqueue_op(e, sm.op, sm.map, batch, s);
    hook(sm.op, false);
  }
  return kernels;
}

// Capture the graph of segment `seg` for LayerSelect variant `mask` at `batch`.
static void build_graph(ssn_engine* e, int seg, uint32_t mask, uint32_t batch) {
  int kernels = 0;
  CUDA_TRY(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
  try {
    kernels = enqueue_segment(e, seg, mask, batch, e->cap_stream, [](int, bool) {});
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(e->cap_stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamEndCapture(e->cap_stream, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t err = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(err);
  e->graphs[graph_key(seg, mask, batch)] = {ex, kernels};
}

static bool fwd_graphs_enabled() {
  static const bool on = [] {
    const char* v = getenv("SSN_NO_FWD_GRAPH");
    return !(v && atoi(v) != 0);
  }();
  return on;
}

static std::vector<uint32_t> fgraph_key(const SubnetState& sub, uint32_t batch) {
  std::vector<uint32_t> k(sub.seg_var.size() + 1);
  for (size_t si = 0; si < sub.seg_var.size(); ++si) k[si] = sub.seg_run[si] ? sub.seg_var[si] : 0xFFFFFFFFu;
  k.back() = batch;
  return k;
}

// Capture the whole forward of `sub`'s variant vector at `batch` (once per key).
static void build_fwd_graph(ssn_engine* e, const SubnetState& sub, uint32_t batch) {
  // bounded: an engine with hundreds of registered variant vectors keeps the
  // per-segment graphs for the rest (SSN_FWD_GRAPH_MAX, default 256)
  static const size_t cap = [] {
    const char* v = getenv("SSN_FWD_GRAPH_MAX");
    return v ? static_cast<size_t>(atol(v)) : static_cast<size_t>(256);
  }();
  const std::vector<uint32_t> key = fgraph_key(sub, batch);
  if (e->fgraphs.count(key) || e->fgraphs.size() >= cap) return;
  int kernels = 0;
  CUDA_TRY(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
  try {
    for (size_t si = 0; si < e->net.segments.size(); ++si)
      if (sub.seg_run[si])
        kernels += enqueue_segment(e, static_cast<int>(si), sub.seg_var[si], batch, e->cap_stream,
                                   [](int, bool) {});
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(e->cap_stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaStreamEndCapture(e->cap_stream, &g));
  cudaGraphExec_t ex = nullptr;
  cudaError_t err = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  CUDA_TRY(err);
  e->fgraphs[key] = {ex, kernels};
}

static void register_subnet(ssn_engine* e, uint32_t id, const ssn_subnet_cfg* c,
                            const float* mean, const float* var) {
  if (!c) SSN_THROW(SSN_E_INVALID, "null subnet config");
  if (id > 65535) SSN_THROW(SSN_E_RANGE, "subnet id must be < 65536");
  SubnetCfg cfg = SubnetCfg::from_c(c);
  Net plan = build_net(e->desc, &cfg);  // throws invalid_argument like SubnetConfig::validate
  if (plan.ops.size() != e->net.ops.size()) SSN_THROW(SSN_E_STATE, "plan/op mismatch");
  // SubnetNorm: fold shared gamma/beta with this subnet's (mu, var).
  std::vector<float> norm;
  std::vector<int64_t> norm_off(plan.ops.size(), -1);
  for (size_t oi = 0; oi < plan.ops.size(); ++oi) {
    const OpSpec& o = plan.ops[oi];
    if (!has_subnet_norm(o)) continue;
    norm_off[oi] = static_cast<int64_t>(norm.size());
    const auto& g = e->gamma[o.norm];
    const auto& b = e->beta[o.norm];
    std::vector<float> sc(o.cout), sh(o.cout);
    for (int ch = 0; ch < o.cout; ++ch) {
      const float mu = mean ? mean[o.stat_off + ch]
                            : ssn_stat_mean_value(e->desc.seed, id, o.norm_slot, ch);
      const float vr = var ? var[o.stat_off + ch]
                           : ssn_stat_var_value(e->desc.seed, id, o.norm_slot, ch);
      if (!(vr >= 0.f)) SSN_THROW(SSN_E_INVALID, "SubnetNorm variance must be >= 0");
      const float inv = 1.0f / std::sqrt(vr + 1e-5f);
      sc[ch] = g[ch] * inv;
      sh[ch] = b[ch] - mu * sc[ch];
    }
    norm.insert(norm.end(), sc.begin(), sc.end());
    norm.insert(norm.end(), sh.begin(), sh.end());
  }
  SubnetState st;
  st.plan = std::move(plan);
  st.norm_bytes = norm.size() * sizeof(float);
  st.stat_bytes = st.plan.stat_count * 2 * sizeof(float);
  if (!norm.empty()) {
    CUDA_TRY(cudaMalloc(&st.d_norm, st.norm_bytes));
    CUDA_TRY(cudaMemcpy(st.d_norm, norm.data(), st.norm_bytes, cudaMemcpyHostToDevice));
  }
  const size_t nseg = e->net.segments.size();
  st.seg_mask.assign(nseg, 0);
  st.seg_var.assign(nseg, 0);
  st.seg_run.assign(nseg, 0);
  for (size_t si = 0; si < nseg; ++si)
    for (size_t f = 0; f < e->net.segments[si].flags.size(); ++f)
      if (cfg.depth[e->net.segments[si].flags[f]]) st.seg_mask[si] |= 1u << f;
  // physical input buffer of every op this subnet runs; a segment whose
  // blocks are all skipped (LayerSelect) leaves its input where it is.
  std::vector<const void*> in_ptr(st.plan.ops.size(), nullptr);
  std::vector<const void*> res_ptr(st.plan.ops.size(), nullptr);
  std::vector<const void*> in2_ptr(st.plan.ops.size(), nullptr), in3_ptr(st.plan.ops.size(), nullptr);
  std::vector<const void*> out_ptr(st.plan.ops.size(), nullptr);
  bool flip = false;
  for (size_t si = 0; si < nseg; ++si) {
    st.seg_var[si] = st.seg_mask[si] | (flip ? SEG_FLIP : 0u);
    const auto sp = segment_plan(e, static_cast<int>(si), st.seg_var[si]);
    st.seg_run[si] = !sp.empty();
    if (sp.empty()) flip = !flip;
    for (const SlotMap& sm : sp) {
      in_ptr[sm.op] = slot_ptr(e, e->net.ops[sm.op].in, sm.map);
      res_ptr[sm.op] = slot_ptr(e, e->net.ops[sm.op].res, sm.map);
      in2_ptr[sm.op] = slot_ptr(e, e->net.ops[sm.op].in2, sm.map);
      in3_ptr[sm.op] = slot_ptr(e, e->net.ops[sm.op].in3, sm.map);
      out_ptr[sm.op] = slot_ptr(e, e->net.ops[sm.op].out, sm.map);
    }
  }
  std::vector<OpDesc> row(st.plan.ops.size());
  for (size_t oi = 0; oi < st.plan.ops.size(); ++oi) {
    const OpSpec& o = st.plan.ops[oi];
    OpDesc& dsc = row[oi];
    std::memset(&dsc, 0, sizeof(dsc));
    if (e->bf16 && o.active && o.kind == OP_ATTN) {
      // tcgen05 attention: Q / K / V tiles of this subnet's active heads
      const long rows = static_cast<long>(e->desc.max_batch) * o.hin;
      if (make_attn_map(&dsc.amap, in_ptr[oi], rows, o.cin) != 0 ||
          make_attn_map(&dsc.rmap, in2_ptr[oi], rows, o.cin) != 0 ||
          make_attn_map(&dsc.wmap, in3_ptr[oi], rows, o.cin) != 0)
        SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (attention) failed for op " + std::to_string(oi));
    }
    if (e->bf16 && o.active && o.kind == OP_CONV && o.depthwise) {
      // depthwise input window map (box sized for this subnet's k)
      if (make_dw_act_map(&dsc.amap, in_ptr[oi], static_cast<int>(e->desc.max_batch), o.hin,
                          o.win, o.cout, act_ld(e, o.cout), o.k, o.stride, o.wout, o.cout_max) != 0)
        SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (depthwise) failed for op " + std::to_string(oi));
    }
    if (e->bf16 && o.active && (o.kind == OP_CONV || o.kind == OP_LINEAR) && !o.depthwise) {
      // WeightSlice A operand: im2col TMA map over this subnet's compact
      // activation (cin_a channels) in the buffer its graph variant reads.
      // Shifted-window (halo) convs read a 5-D tiled map instead.
      if (use_halo(e, o)) {
        // resident B at this subnet's width (rows = 16-rounded cout_a, only
        // the active 32-channel blocks are loaded): wmap slot, wrows = rows
        const TensorSpec& t = e->net.tensors[o.tensor];
        const int hrows = (o.cout + 15) & ~15;
        if (make_halo_act_map(&dsc.amap, in_ptr[oi], static_cast<int>(e->desc.max_batch), o.hin,
                              o.win, o.cin, act_ld(e, o.cin), o.k) != 0 ||
            make_halo_weight_map(&dsc.wmap, e->d_w + t.w_off, t.cin_store, o.k_max * o.k_max,
                                 t.cout, hrows, 0) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (halo) failed for op " + std::to_string(oi));
        dsc.wrows = hrows;
      } else {
        if (make_act_map(&dsc.amap, in_ptr[oi], static_cast<int>(e->desc.max_batch), o.hin,
                         o.win, o.cin, act_ld(e, o.cin), o.k, o.stride, o.k / 2) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeIm2col failed for op " + std::to_string(oi));
        // WeightSlice B at this subnet's tile width (largest-batch graph tiling)
        if (!(tc_debug_flags() & 2097152)) {
          ConvParams cp = conv_static_params(e, static_cast<int>(oi), e->desc.max_batch);
          conv_tc_tiling(e, static_cast<int>(oi), cp);
          const int cg = cp.cg2 ? 2 : 1;
          const int bn_a = conv_bn_active(cp.bn, o.cout, cg);
          const TensorSpec& t = e->net.tensors[o.tensor];
          if (make_weight_map(&dsc.wmap, e->d_w + t.w_off, t.cin_store, o.k_max * o.k_max, t.cout,
                              bn_a / cg) != 0)
            SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (weights) failed for op " + std::to_string(oi));
          dsc.wrows = bn_a / cg;
        }
        // shifted-window pair kernel (large-batch graphs of residual-free
        // 28- and 14-px 3x3 convs): its 4-D window map rides in the unused
        // rmap slot and its filter-row B map in hmap, so the same subnet row
        // also serves the small-batch graphs' conv_tc
        if (use_hp(e, o, e->desc.max_batch)) {
          const TensorSpec& t = e->net.tensors[o.tensor];
          const int hb = conv_bn_active(hp_choose_bn(o.cout_max), o.cout, 2);
          if (make_hp_act_map(&dsc.rmap, in_ptr[oi], static_cast<int>(e->desc.max_batch), o.hin,
                              o.win, o.cin, act_ld(e, o.cin)) != 0 ||
              make_hp_weight_map(&dsc.hmap, e->d_w + t.w_off, t.cin_store, o.k_max * o.k_max,
                                 t.cout, hb / 2) != 0)
            SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (hp) failed for op " + std::to_string(oi));
          dsc.hrows = hb / 2;
        }
        // output map of conv_tc's TMA-store epilogue (bf16 outputs)
        if (o.kind != OP_LINEAR && (o.cout & 7) == 0 && out_ptr[oi] &&
            make_y_map(&dsc.ymap, const_cast<void*>(out_ptr[oi]),
                       static_cast<long>(e->desc.max_batch) * o.hout * o.wout, o.cout,
                       act_ld(e, o.cout)) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (output) failed for op " + std::to_string(oi));
        // residual source for conv_tc's TMA residual ring
        if (res_ptr[oi] && (o.cout & 7) == 0 &&
            make_res_map(&dsc.rmap, res_ptr[oi],
                         static_cast<long>(e->desc.max_batch) * o.hout * o.wout, o.cout,
                         act_ld(e, o.cout)) != 0)
          SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (residual) failed for op " + std::to_string(oi));
      }
    }
    dsc.cin = o.cin;
    dsc.cout = o.cout;
    dsc.ldi = act_ld(e, o.cin);
    dsc.ldo = o.kind == OP_LINEAR ? o.cout : act_ld(e, o.cout);  // fp32 logits stay compact
    dsc.k = o.k;
    dsc.pad = o.k / 2;
    dsc.scale = nullptr;
    dsc.shift = nullptr;
    if (norm_off[oi] >= 0) {
      dsc.scale = st.d_norm + norm_off[oi];
      dsc.shift = st.d_norm + norm_off[oi] + o.cout;
    }
    if ((o.kind == OP_LINEAR || o.kind == OP_CONV) && o.norm < 0 && o.tensor >= 0 &&
        e->net.tensors[o.tensor].linear)  // bias (leading slice of the shared vector)
      dsc.shift = reinterpret_cast<const float*>(e->d_w + e->net.tensors[o.tensor].b_off);
    if (o.kind == OP_SE) dsc.aux = o.se_mid;
  }
  CUDA_TRY(cudaMalloc(&st.d_row, row.size() * sizeof(OpDesc)));
  CUDA_TRY(cudaMemcpy(st.d_row, row.data(), row.size() * sizeof(OpDesc), cudaMemcpyHostToDevice));
  st.ok = true;
  if (id >= e->subs.size()) e->subs.resize(id + 1);
  SubnetState& old = e->subs[id];
  if (old.ok) {
    // Re-registration: the previous row may be referenced by in-flight work.
    CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(old.d_row);
    cudaFree(old.d_norm);
    if (e->active == static_cast<int>(id)) e->dirty = true;
  }
  e->subs[id] = std::move(st);
  if (e->prepared && fwd_graphs_enabled())
    for (uint32_t b : e->grid) build_fwd_graph(e, e->subs[id], b);
}

// ---------------------------------------------------------------------------
// C-ABI

extern "C" {

const char* ssn_last_error(void) { return g_last_error.c_str(); }

int ssn_weight_blob_bytes(const ssn_supernet_desc* desc, uint64_t* bytes) {
  return guarded([&] {
    validate_desc(desc);
    if (!bytes) SSN_THROW(SSN_E_INVALID, "null output");
    *bytes = build_net(*desc, nullptr).blob_bytes;
  });
}

int ssn_generate_weight_blob(const ssn_supernet_desc* desc, void* blob, uint64_t bytes) {
  return guarded([&] {
    validate_desc(desc);
    Net net = build_net(*desc, nullptr);
    if (!blob || bytes < net.blob_bytes) SSN_THROW(SSN_E_INVALID, "blob too small");
    generate_blob(net, static_cast<uint8_t*>(blob));
  });
}

int ssn_plan_stat_count(const ssn_supernet_desc* desc, const ssn_subnet_cfg* c, uint64_t* count) {
  return guarded([&] {
    validate_desc(desc);
    if (!c || !count) SSN_THROW(SSN_E_INVALID, "null argument");
    SubnetCfg cfg = SubnetCfg::from_c(c);
    *count = build_net(*desc, &cfg).stat_count;
  });
}

int ssn_plan_ops(const ssn_supernet_desc* desc, const ssn_subnet_cfg* c, ssn_op_info* out,
                 uint32_t capacity, uint32_t* n_ops) {
  return guarded([&] {
    validate_desc(desc);
    if (!c || !n_ops) SSN_THROW(SSN_E_INVALID, "null argument");
    SubnetCfg cfg = SubnetCfg::from_c(c);
    Net net = build_net(*desc, &cfg);
    *n_ops = static_cast<uint32_t>(net.ops.size());
    if (!out) return;
    if (capacity < net.ops.size()) SSN_THROW(SSN_E_RANGE, "op info capacity too small");
    std::vector<int> blk(net.ops.size(), -1);
    for (size_t bi = 0; bi < net.blocks.size(); ++bi)
      for (int q = 0; q < net.blocks[bi].count; ++q) blk[net.blocks[bi].first + q] = static_cast<int>(bi);
    for (size_t i = 0; i < net.ops.size(); ++i) {
      const OpSpec& o = net.ops[i];
      ssn_op_info& r = out[i];
      r.kind = static_cast<uint32_t>(o.kind);
      r.active = o.active;
      r.k = static_cast<uint32_t>(o.kind == OP_AVGPOOL ? o.pool_k : o.k);
      r.stride = static_cast<uint32_t>(o.stride);
      r.hin = o.hin; r.win = o.win; r.hout = o.hout; r.wout = o.wout;
      r.cin = o.cin; r.cout = o.cout; r.cin_max = o.cin_max; r.cout_max = o.cout_max;
      if (o.tensor >= 0 && net.tensors[o.tensor].im2col_stem) {
        // report the logical convolution (3x3 s2 over 3 channels), not its GEMM form
        r.k = 3; r.stride = 2; r.cin = r.cin_max = 3;
        r.hin = r.win = net.ops[0].hin;
      }
      r.depthwise = o.depthwise;
      r.block = static_cast<uint32_t>(blk[i]);
      r.segment = static_cast<uint32_t>(net.blocks[blk[i]].segment);
      r.has_residual = o.res != S_NONE;
    }
  });
}

int ssn_create(int device, const ssn_supernet_desc* desc, const void* host_weights,
               uint64_t host_weight_bytes, ssn_engine** out) {
  return guarded([&] {
    validate_desc(desc);
    if (!out) SSN_THROW(SSN_E_INVALID, "null output handle");
    *out = nullptr;
    std::unique_ptr<ssn_engine> e(new ssn_engine());
    e->device = device;
    e->desc = *desc;
    e->bf16 = desc->dtype == SSN_DTYPE_BF16;
    e->net = build_net(*desc, nullptr);
    for (const SegmentSpec& sg : e->net.segments)
      if (sg.flags.size() >= 15) SSN_THROW(SSN_E_INVALID, "too many LayerSelect flags in a segment");
    CUDA_TRY(cudaSetDevice(device));
    int major = 0, minor = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (e->bf16 && major != 10)
      SSN_THROW(SSN_E_CUDA, "bf16 tcgen05 path requires an sm_100 (B200) device");
    if (e->bf16) {
      CUDA_TRY(init_conv_tc());
      CUDA_TRY(init_conv_halo());
      CUDA_TRY(init_conv_hp());
    }
    std::vector<uint8_t> gen;
    const uint8_t* blob = static_cast<const uint8_t*>(host_weights);
    if (!blob) {
      gen.resize(e->net.blob_bytes);
      generate_blob(e->net, gen.data());
      blob = gen.data();
    } else if (host_weight_bytes < e->net.blob_bytes) {
      SSN_THROW(SSN_E_INVALID, "host weight blob too small: need " +
                                   std::to_string(e->net.blob_bytes) + " bytes");
    }
    // weight store: uploaded once, shared in place by every subnet
    CUDA_TRY(cudaMalloc(&e->d_w, e->net.blob_bytes));
    CUDA_TRY(cudaMemcpy(e->d_w, blob, e->net.blob_bytes, cudaMemcpyHostToDevice));
    for (const NormSpec& n : e->net.norms) {
      const float* g = reinterpret_cast<const float*>(blob + n.gamma_off);
      const float* b = reinterpret_cast<const float*>(blob + n.beta_off);
      e->gamma.emplace_back(g, g + n.c);
      e->beta.emplace_back(b, b + n.c);
    }
    // activation arena for the largest batch at max widths
    size_t max_elems = 0;
    for (const OpSpec& o : e->net.ops)
      max_elems = std::max(max_elems, static_cast<size_t>(o.hout) * o.wout * act_ld(e.get(), o.cout_max));
    e->buf_bytes = max_elems * desc->max_batch * (e->bf16 ? 2 : 4);
    for (int i = 0; i < NBUF; ++i) CUDA_TRY(cudaMalloc(&e->bufs[i], e->buf_bytes));
    e->raw_img_bytes = raw_image_bytes(*desc);
    CUDA_TRY(cudaMalloc(&e->d_raw, e->raw_img_bytes * desc->max_batch));
    if (e->bf16) {
      CUDA_TRY(cudaMalloc(&e->d_ws, SSN_SPLIT_WS_FLOATS * sizeof(float)));
    }
    CUDA_TRY(cudaMemset(e->d_raw, 0, e->raw_img_bytes * desc->max_batch));
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaMalloc(&e->d_stage[k], e->raw_img_bytes * desc->max_batch));
      CUDA_TRY(cudaEventCreateWithFlags(&e->stage_ready[k], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&e->stage_free[k], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaMalloc(&e->d_logits, static_cast<size_t>(desc->max_batch) * desc->num_classes * 4));
    int se_hmax = 0;
    for (const OpSpec& o : e->net.ops)
      if (o.kind == OP_SE) {
        e->se_cmax = std::max(e->se_cmax, o.cin_max);
        se_hmax = std::max(se_hmax, o.se_mid_max);
      }
    if (e->se_cmax)  // pooled [B][cmax] | gate [B][cmax] | hidden [B][hmax]
      CUDA_TRY(cudaMalloc(&e->d_se, 1ull * desc->max_batch * (2 * e->se_cmax + se_hmax) *
                                        sizeof(float)));
    int se_parts = 0;
    for (int oi = 0; oi < static_cast<int>(e->net.ops.size()); ++oi)
      se_parts = std::max(se_parts, se_fused_parts(e.get(), oi));
    if (se_parts)
      CUDA_TRY(cudaMalloc(&e->d_separt,
                          1ull * desc->max_batch * se_parts * e->se_cmax * sizeof(float)));
    CUDA_TRY(cudaMalloc(&e->d_rowptr, sizeof(OpDesc*)));
    CUDA_TRY(cudaMemset(e->d_rowptr, 0, sizeof(OpDesc*)));
    CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&e->last_done, cudaEventDisableTiming));
    *out = e.release();
  });
}

void ssn_destroy(ssn_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second.first);
  for (auto& kv : e->fgraphs) cudaGraphExecDestroy(kv.second.first);
  for (auto& s : e->subs) {
    cudaFree(s.d_row);
    cudaFree(s.d_norm);
  }
  for (int i = 0; i < NBUF; ++i) cudaFree(e->bufs[i]);
  cudaFree(e->d_raw);
  cudaFree(e->d_ws);
  for (int k = 0; k < 2; ++k) {
    cudaFree(e->d_stage[k]);
    if (e->stage_ready[k]) cudaEventDestroy(e->stage_ready[k]);
    if (e->stage_free[k]) cudaEventDestroy(e->stage_free[k]);
  }
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  cudaFree(e->d_logits);
  cudaFree(e->d_se);
  cudaFree(e->d_separt);
  cudaFree(e->d_rowptr);
  cudaFree(e->d_w);
  if (e->stream) cudaStreamDestroy(e->stream);
  if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
  if (e->last_done) cudaEventDestroy(e->last_done);
  delete e;
}

int ssn_subnet_stat_count(ssn_engine* e, const ssn_subnet_cfg* c, uint64_t* count) {
  return guarded([&] {
    if (!e || !c || !count) SSN_THROW(SSN_E_INVALID, "null argument");
    SubnetCfg cfg = SubnetCfg::from_c(c);
    *count = build_net(e->desc, &cfg).stat_count;
  });
}

int ssn_register_subnet(ssn_engine* e, uint32_t id, const ssn_subnet_cfg* c, const float* mean,
                        const float* var) {
  return guarded([&] {
    if (!e) SSN_THROW(SSN_E_INVALID, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    register_subnet(e, id, c, mean, var);
  });
}

int ssn_register_subnet_n(ssn_engine* e, uint32_t id, const ssn_subnet_cfg* c, const float* mean,
                          const float* var, uint64_t n_stats) {
  return guarded([&] {
    if (!e || !c) SSN_THROW(SSN_E_INVALID, "null argument");
    if ((mean == nullptr) != (var == nullptr))
      SSN_THROW(SSN_E_INVALID, "SubnetNorm statistics need both mean and var (or neither)");
    if (mean) {
      SubnetCfg cfg = SubnetCfg::from_c(c);
      const uint64_t need = build_net(e->desc, &cfg).stat_count;
      if (n_stats != need)
        SSN_THROW(SSN_E_INVALID, "SubnetNorm statistics length " + std::to_string(n_stats) +
                                     " != stat count " + std::to_string(need));
    }
    CUDA_TRY(cudaSetDevice(e->device));
    register_subnet(e, id, c, mean, var);
  });
}

int ssn_prepare(ssn_engine* e, const uint32_t* batch_grid, uint32_t n) {
  return guarded([&] {
    if (!e) SSN_THROW(SSN_E_INVALID, "null engine");
    if (!batch_grid || n == 0) SSN_THROW(SSN_E_INVALID, "empty batch grid");
    CUDA_TRY(cudaSetDevice(e->device));
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t b = batch_grid[i];
      if (b == 0 || b > e->desc.max_batch)
        SSN_THROW(SSN_E_RANGE, "batch " + std::to_string(b) + " outside [1, max_batch]");
      if (i > 0 && b <= batch_grid[i - 1]) SSN_THROW(SSN_E_INVALID, "batch sizes must increase");
    }
    // A fixed row for capture-time validity (kernels only read it at replay).
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t b = batch_grid[i];
      if (std::find(e->grid.begin(), e->grid.end(), b) != e->grid.end()) continue;
      bool can_flip = false;  // some earlier segment may run no block at all
      for (size_t si = 0; si < e->net.segments.size(); ++si) {
        const uint32_t variants = 1u << e->net.segments[si].flags.size();
        for (uint32_t f = 0; f <= (can_flip ? 1u : 0u); ++f)
          for (uint32_t m = 0; m < variants; ++m)
            build_graph(e, static_cast<int>(si), m | (f ? SEG_FLIP : 0u), b);
        bool all_optional = true;
        for (int bi : e->net.segments[si].blocks) all_optional &= e->net.blocks[bi].flag >= 0;
        can_flip |= all_optional;
      }
      e->grid.push_back(b);
    }
    std::sort(e->grid.begin(), e->grid.end());
    if (fwd_graphs_enabled())
      for (const SubnetState& sub : e->subs)
        if (sub.ok)
          for (uint32_t b : e->grid) build_fwd_graph(e, sub, b);
    e->prepared = true;
  });
}

int ssn_actuate(ssn_engine* e, uint32_t id) {
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded([&] {
    if (!e) SSN_THROW(SSN_E_INVALID, "null engine");
    if (id >= e->subs.size() || !e->subs[id].ok)
      SSN_THROW(SSN_E_RANGE, "subnet " + std::to_string(id) + " is not registered");
    if (e->active != static_cast<int>(id)) {
      e->active = static_cast<int>(id);
      e->dirty = true;
    }
  });
  if (e)
    e->last_actuate_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  return rc;
}

int ssn_forward(ssn_engine* e, const void* x, uint32_t count, uint32_t profiled_batch,
                float* logits, void* stream) {
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded([&] {
    if (!e) SSN_THROW(SSN_E_INVALID, "null engine");
    if (e->active < 0) SSN_THROW(SSN_E_STATE, "no subnet actuated");
    if (!e->prepared) SSN_THROW(SSN_E_STATE, "ssn_prepare() has not been called");
    if (count == 0 || count > profiled_batch)
      SSN_THROW(SSN_E_INVALID, "count must be in [1, profiled_batch]");
    if (std::find(e->grid.begin(), e->grid.end(), profiled_batch) == e->grid.end())
      SSN_THROW(SSN_E_RANGE, "batch size " + std::to_string(profiled_batch) + " not prepared");
    CUDA_TRY(cudaSetDevice(e->device));  // the calling worker thread may not have it current
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
    const SubnetState& sub = e->subs[e->active];
    uint32_t kernels = 0, graphs = 0;
    order_stream(e, s);
    if (e->dirty) {
      CUDA_TRY(launch_set_row(e->d_rowptr, sub.d_row, s));
      e->dirty = false;
      ++kernels;
    }
    if (x) {
      const size_t bytes = e->raw_img_bytes * count;
      cudaPointerAttributes attr{};
      const bool host = cudaPointerGetAttributes(&attr, x) != cudaSuccess ||
                        attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeUnregistered;
      cudaGetLastError();  // clear a failed query on an unregistered pointer
      if (host) {
        // H2D on the copy stream into a free staging slot (overlaps the
        // previous forward's graphs), then a device copy on the compute stream
        const int k = e->stage_slot;
        e->stage_slot ^= 1;
        CUDA_TRY(cudaStreamWaitEvent(e->copy_stream, e->stage_free[k], 0));
        CUDA_TRY(cudaMemcpyAsync(e->d_stage[k], x, bytes, cudaMemcpyHostToDevice, e->copy_stream));
        CUDA_TRY(cudaEventRecord(e->stage_ready[k], e->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(s, e->stage_ready[k], 0));
        CUDA_TRY(cudaMemcpyAsync(e->d_raw, e->d_stage[k], bytes, cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(cudaEventRecord(e->stage_free[k], s));
      } else {
        CUDA_TRY(cudaMemcpyAsync(e->d_raw, x, bytes, cudaMemcpyDefault, s));
      }
    }
    const auto fit = fwd_graphs_enabled() ? e->fgraphs.find(fgraph_key(sub, profiled_batch))
                                          : e->fgraphs.end();
    if (fit != e->fgraphs.end()) {
      CUDA_TRY(cudaGraphLaunch(fit->second.first, s));
      kernels += static_cast<uint32_t>(fit->second.second);
      ++graphs;
    } else {
      for (size_t si = 0; si < e->net.segments.size(); ++si) {
        if (!sub.seg_run[si]) continue;  // every block skipped: input passes through
        auto it = e->graphs.find(graph_key(static_cast<int>(si), sub.seg_var[si], profiled_batch));
        if (it == e->graphs.end()) SSN_THROW(SSN_E_STATE, "missing graph segment");
        CUDA_TRY(cudaGraphLaunch(it->second.first, s));
        kernels += static_cast<uint32_t>(it->second.second);
        ++graphs;
      }
    }
    if (logits)
      CUDA_TRY(cudaMemcpyAsync(logits, e->d_logits,
                               static_cast<size_t>(count) * e->desc.num_classes * 4,
                               cudaMemcpyDefault, s));
    mark_done(e, s);
    e->last_kernels = kernels;
    e->last_graphs = graphs;
  });
  if (e)
    e->last_forward_host_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  return rc;
}

int ssn_synchronize(ssn_engine* e, void* stream) {
  return guarded([&] {
    if (!e) SSN_THROW(SSN_E_INVALID, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(stream ? static_cast<cudaStream_t>(stream) : e->stream));
  });
}

int ssn_profile_latency(ssn_engine* e, uint32_t id, uint32_t batch, uint32_t iters,
                        double* median_us) {
  return guarded([&] {
    if (!e || !median_us || iters == 0) SSN_THROW(SSN_E_INVALID, "bad arguments");
    if (ssn_actuate(e, id) != SSN_OK) SSN_THROW(SSN_E_RANGE, g_last_error);
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    for (int w = 0; w < 3; ++w)
      if (ssn_forward(e, nullptr, batch, batch, nullptr, nullptr) != SSN_OK)
        SSN_THROW(SSN_E_RANGE, g_last_error);
    std::vector<float> ms;
    for (uint32_t i = 0; i < iters; ++i) {
      CUDA_TRY(cudaEventRecord(a, e->stream));
      if (ssn_forward(e, nullptr, batch, batch, nullptr, nullptr) != SSN_OK)
        SSN_THROW(SSN_E_RANGE, g_last_error);
      CUDA_TRY(cudaEventRecord(b, e->stream));
      CUDA_TRY(cudaEventSynchronize(b));
      float t = 0;
      CUDA_TRY(cudaEventElapsedTime(&t, a, b));
      ms.push_back(t);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(ms.begin(), ms.end());
    *median_us = ms[ms.size() / 2] * 1000.0;
  });
}

int ssn_profile_ops(ssn_engine* e, uint32_t id, uint32_t batch, uint32_t iters, float* op_us,
                    uint32_t n_ops) {
  return guarded([&] {
    if (!e || !op_us || iters == 0) SSN_THROW(SSN_E_INVALID, "bad arguments");
    if (n_ops < e->net.ops.size()) SSN_THROW(SSN_E_RANGE, "op_us too small");
    if (batch == 0 || batch > e->desc.max_batch) SSN_THROW(SSN_E_RANGE, "batch out of range");
    if (ssn_actuate(e, id) != SSN_OK) SSN_THROW(SSN_E_RANGE, g_last_error);
    const SubnetState& sub = e->subs[id];
    cudaStream_t s = e->stream;
    order_stream(e, s);
    CUDA_TRY(launch_set_row(e->d_rowptr, sub.d_row, s));
    e->dirty = false;
    const size_t nop = e->net.ops.size();
    std::vector<cudaEvent_t> ev(2 * nop);
    for (auto& x : ev) CUDA_TRY(cudaEventCreate(&x));
    std::vector<std::vector<float>> samples(nop);
    for (uint32_t it = 0; it < iters + 1; ++it) {  // first pass = warm-up
      std::vector<bool> ran(nop, false);
      for (size_t si = 0; si < e->net.segments.size(); ++si)
        enqueue_segment(e, static_cast<int>(si), sub.seg_var[si], batch, s, [&](int op, bool before) {
          CUDA_TRY(cudaEventRecord(ev[2 * op + (before ? 0 : 1)], s));
          ran[op] = true;
        });
      CUDA_TRY(cudaStreamSynchronize(s));
      if (it == 0) continue;
      for (size_t op = 0; op < nop; ++op) {
        if (!ran[op]) continue;
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, ev[2 * op], ev[2 * op + 1]));
        samples[op].push_back(ms * 1000.f);
      }
    }
    for (auto& x : ev) cudaEventDestroy(x);
    for (size_t op = 0; op < nop; ++op) {
      auto& v = samples[op];
      if (v.empty()) {
        op_us[op] = 0.f;
        continue;
      }
      std::sort(v.begin(), v.end());
      op_us[op] = v[v.size() / 2];
    }
    mark_done(e, s);
  });
}

int ssn_debug_op_checksums(ssn_engine* e, uint32_t id, uint32_t batch, uint64_t* sums,
                           uint32_t n_ops) {
  return guarded([&] {
    if (!e || !sums) SSN_THROW(SSN_E_INVALID, "bad arguments");
    if (n_ops < e->net.ops.size()) SSN_THROW(SSN_E_RANGE, "sums too small");
    if (batch == 0 || batch > e->desc.max_batch) SSN_THROW(SSN_E_RANGE, "batch out of range");
    if (ssn_actuate(e, id) != SSN_OK) SSN_THROW(SSN_E_RANGE, g_last_error);
    const SubnetState& sub = e->subs[id];
    cudaStream_t s = e->stream;
    order_stream(e, s);
    CUDA_TRY(launch_set_row(e->d_rowptr, sub.d_row, s));
    e->dirty = false;
    for (uint32_t i = 0; i < n_ops; ++i) sums[i] = 0;
    std::vector<uint8_t> host;
    for (size_t si = 0; si < e->net.segments.size(); ++si)
      for (const SlotMap& sm : segment_plan(e, static_cast<int>(si), sub.seg_var[si])) {
        const int k = enqueue_op(e, sm.op, sm.map, batch, s);
        CUDA_TRY(cudaStreamSynchronize(s));
        if (k == 0) continue;
        const OpSpec& o = e->net.ops[sm.op];
        const OpSpec& a = sub.plan.ops[sm.op];
        const size_t elem = o.kind == OP_LINEAR ? 4 : (e->bf16 ? 2 : 4);
        const size_t ld = o.kind == OP_LINEAR ? a.cout : act_ld(e, a.cout);
        const size_t rows = static_cast<size_t>(batch) * o.hout * o.wout;
        host.resize(rows * ld * elem);
        CUDA_TRY(cudaMemcpy(host.data(), slot_ptr(e, o.out, sm.map), host.size(),
                            cudaMemcpyDeviceToHost));
        uint64_t h = 1469598103934665603ull;  // FNV-1a over the op's output (active columns)
        for (size_t r = 0; r < rows; ++r)
          for (size_t b = 0; b < a.cout * elem; ++b) h = (h ^ host[r * ld * elem + b]) * 1099511628211ull;
        sums[sm.op] = h;
      }
    mark_done(e, s);
  });
}

int ssn_query(ssn_engine* e, ssn_stats* out) {
  return guarded([&] {
    if (!e || !out) SSN_THROW(SSN_E_INVALID, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->weight_bytes = e->net.blob_bytes;
    for (const auto& s : e->subs) {
      if (!s.ok) continue;
      ++out->registered_subnets;
      out->norm_table_bytes += s.norm_bytes;
      out->max_subnet_stat_bytes = std::max(out->max_subnet_stat_bytes, s.stat_bytes);
    }
    out->arena_bytes = e->buf_bytes * NBUF + 3 * e->raw_img_bytes * e->desc.max_batch;
    out->active_subnet = e->active;
    out->graphs_built = static_cast<uint32_t>(e->graphs.size());
    out->last_forward_kernels = e->last_kernels;
    out->last_forward_graphs = e->last_graphs;
    out->last_actuate_us = e->last_actuate_us;
    out->last_forward_host_us = e->last_forward_host_us;
  });
}

int ssn_device_logits(ssn_engine* e, const float** out) {
  return guarded([&] {
    if (!e || !out) SSN_THROW(SSN_E_INVALID, "null argument");
    *out = e->d_logits;
  });
}

// ---- operator-level entry points -----------------------------------------

static OpDesc plain_desc(int cin, int cout, int k, int pad, const float* scale,
                         const float* shift) {
  OpDesc d;
  std::memset(&d, 0, sizeof(d));
  d.cin = cin;
  d.cout = cout;
  d.ldi = cin;  // operator API: compact caller tensors
  d.ldo = cout;
  d.k = k;
  d.pad = pad;
  d.scale = scale;
  d.shift = shift;
  return d;
}

// Device copy of an operator-API OpDesc: a 64-slot ring PER DEVICE (keyed by
// the current device, so a second GPU never dereferences the first one's
// memory).  The upload is synchronous on the caller's stream; a slot is
// rewritten 64 calls later, so callers spreading operator calls over several
// streams must keep fewer than 64 of them in flight.
static OpDesc* op_desc_scratch(const OpDesc& d, cudaStream_t s) {
  static std::map<int, std::pair<OpDesc*, unsigned>> ring;  // device -> (slots, next)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  auto& r = ring[dev];
  if (!r.first) CUDA_TRY(cudaMalloc(&r.first, sizeof(OpDesc) * 64));
  OpDesc* p = r.first + (r.second++ % 64);
  CUDA_TRY(cudaMemcpyAsync(p, &d, sizeof(OpDesc), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return p;
}

int ssn_op_conv_bf16(const void* x, int n, int h, int w, int cin, const void* wgt, int cout_max,
                     int cin_max, int k, int stride, int pad, int cout, const float* scale,
                     const float* shift, const void* res, int act, int out_f32, void* y,
                     void* stream) {
  return guarded([&] {
    if (!x || !wgt || !y) SSN_THROW(SSN_E_INVALID, "null tensor");
    // input channels feed 16-byte TMA strides; the output slice may be ragged
    // (the epilogue's scalar tail handles cout % 8 != 0, e.g. a 2-label head)
    if (cin % 8 || cin_max % 8 || cin > cin_max || cout > cout_max || cin <= 0 || cout <= 0)
      SSN_THROW(SSN_E_INVALID, "input channels must be positive multiples of 8 within max shape");
    if (k < 1 || stride < 1 || pad < 0) SSN_THROW(SSN_E_INVALID, "bad geometry");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CUDA_TRY(init_conv_tc());
    CUDA_TRY(init_conv_halo());
    CUDA_TRY(init_conv_hp());
    const bool aligned16 =
        ((reinterpret_cast<uintptr_t>(scale) | reinterpret_cast<uintptr_t>(shift)) & 15) == 0;
    const bool halo = pad == k / 2 && !out_f32 && act <= 1 && (cout & 7) == 0 &&
                      (cout_max & 7) == 0 && aligned16 &&
                      halo_eligible(h, w, k, stride, cin_max, cout_max);
    const bool hp = !halo && pad == k / 2 && !out_f32 && act <= 1 && !res && (cout & 7) == 0 &&
                    (cout_max & 7) == 0 && aligned16 && !(getenv("SSN_OP_NO_HP")) &&
                    hp_eligible(h, w, k, stride, cin_max, cout_max, false);
    OpDesc d = plain_desc(cin, cout, k, pad, scale, shift);
    if (!hp && (halo ? make_halo_act_map(&d.amap, x, n, h, w, cin, cin, k) != 0
                     : make_act_map(&d.amap, x, n, h, w, cin, cin, k, stride, pad) != 0))
      SSN_THROW(SSN_E_CUDA, "cuTensorMapEncode (activation) failed");
    ConvParams p{};
    p.x = x;
    p.y = y;
    p.res = res;
    p.w = wgt;
    p.row = nullptr;
    p.fixed = op_desc_scratch(d, s);
    p.n = n;
    p.h = h;
    p.w_ = w;
    p.ho = (h + 2 * pad - k) / stride + 1;
    p.wo = (w + 2 * pad - k) / stride + 1;
    p.stride = stride;
    p.M = n * p.ho * p.wo;
    p.k_max = k;
    p.cin_max = cin_max;
    p.cout_max = cout_max;
    p.act = act;
    p.res_post = 0;
    p.out_f32 = out_f32;
    if (halo) {
      CUDA_TRY(launch_conv_halo(p, wgt, cin_max, k * k, s));
      return;
    }
    if (hp) {
      p.bn = hp_choose_bn(cout_max);
      const int bn_a = conv_bn_active(p.bn, cout, 2);
      OpDesc d2 = d;
      if (make_hp_act_map(&d2.rmap, x, n, h, w, cin, cin) != 0 ||
          make_hp_weight_map(&d2.hmap, wgt, cin_max, k * k, cout_max, bn_a / 2) != 0)
        SSN_THROW(SSN_E_CUDA, "cuTensorMapEncode (hp) failed");
      d2.hrows = bn_a / 2;
      p.fixed = op_desc_scratch(d2, s);
      CUtensorMap wmap{};
      if (make_hp_weight_map(&wmap, wgt, cin_max, k * k, cout_max, p.bn / 2) != 0)
        SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled failed");
      CUDA_TRY(launch_conv_hp(p, wmap, s));
      return;
    }
    p.bn = choose_bn(cout_max, p.M, k * k * ((cin_max + 63) / 64));
    // ragged slice, or SubnetNorm vectors the vector epilogue cannot load
    p.ragged = (cout & 7) != 0 || ((reinterpret_cast<uintptr_t>(scale) | reinterpret_cast<uintptr_t>(shift)) & 15) != 0;
    p.cg2 = conv_tc_use_pairs(p);
    if (!out_f32 && !p.ragged) {  // TMA-store epilogue: the scratch row carries the output map
      OpDesc d2 = d;
      if (make_y_map(&d2.ymap, y, p.M, cout, cout) != 0)
        SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (output) failed");
      p.fixed = op_desc_scratch(d2, s);
      p.ystore = 1;
    }
    CUtensorMap wmap{};
    if (make_weight_map(&wmap, wgt, cin_max, k * k, cout_max, p.cg2 ? p.bn / 2 : p.bn) != 0)
      SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled failed");
    CUDA_TRY(launch_conv_tc(p, wmap, s));
  });
}

int ssn_op_dw_bf16(const void* x, int n, int h, int w, int c, const void* wgt, int c_max,
                   int k_max, int k, int stride, const float* scale, const float* shift, int act,
                   void* y, void* stream) {
  return guarded([&] {
    if (!x || !wgt || !y) SSN_THROW(SSN_E_INVALID, "null tensor");
    if (n <= 0 || h <= 0 || w <= 0) SSN_THROW(SSN_E_INVALID, "bad geometry");
    if (c <= 0 || c % 8 || c_max % 8 || c > c_max)
      SSN_THROW(SSN_E_INVALID, "channels must be positive multiples of 8 within the max shape");
    if (!dw_supported(k_max, k, stride) || k_max % 2 == 0)
      SSN_THROW(SSN_E_INVALID, "depthwise k must be 3/5/7 <= k_max <= 7 (odd), stride 1 or 2");
    if (act < 0 || act > 2) SSN_THROW(SSN_E_INVALID, "act must be 0 none, 1 relu, 2 h_swish");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int pad = k / 2;
    const int ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
    OpDesc d = plain_desc(c, c, k, pad, scale, shift);
    if (make_dw_act_map(&d.amap, x, n, h, w, c, c, k, stride, wo, c_max) != 0)
      SSN_THROW(SSN_E_CUDA, "cuTensorMapEncodeTiled (depthwise) failed");
    ConvParams p{};
    p.x = x;
    p.y = y;
    p.w = wgt;
    p.fixed = op_desc_scratch(d, s);
    p.n = n;
    p.h = h;
    p.w_ = w;
    p.ho = ho;
    p.wo = wo;
    p.stride = stride;
    p.M = n * ho * wo;
    p.k_max = k_max;
    p.cin_max = 1;
    p.cout_max = c_max;
    p.act = act;
    p.depthwise = 1;
    CUDA_TRY(launch_dw_bf16(p, s));
  });
}

int ssn_op_conv_f32(const float* x, int n, int h, int w, int cin, const float* wgt, int cout_max,
                    int cin_max, int k_max, int k, int stride, int pad, int cout, int depthwise,
                    const float* scale, const float* shift, const float* res, int act, float* y,
                    void* stream) {
  return guarded([&] {
    if (!x || !wgt || !y) SSN_THROW(SSN_E_INVALID, "null tensor");
    if (cin > cin_max || cout > cout_max || k > k_max || (depthwise && cin != cout))
      SSN_THROW(SSN_E_INVALID, "active slice exceeds the max shape");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    OpDesc d = plain_desc(cin, cout, k, pad, scale, shift);
    ConvParams p{};
    p.x = x;
    p.y = y;
    p.res = res;
    p.w = wgt;
    p.fixed = op_desc_scratch(d, s);
    p.n = n;
    p.h = h;
    p.w_ = w;
    p.ho = (h + 2 * pad - k) / stride + 1;
    p.wo = (w + 2 * pad - k) / stride + 1;
    p.stride = stride;
    p.M = n * p.ho * p.wo;
    p.k_max = k_max;
    p.cin_max = depthwise ? 1 : cin_max;
    p.cout_max = cout_max;
    p.act = act;
    p.depthwise = depthwise;
    CUDA_TRY(launch_conv_f32(p, s));
  });
}

}  // extern "C"
