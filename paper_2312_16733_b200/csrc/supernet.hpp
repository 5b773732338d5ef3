// supernet.hpp — supernet layer plans for the SubNetAct engine (host C++).
//
// A supernet is a fixed list of max-shape ops grouped into blocks and
// segments.  Resolving a subnet control tuple (D, E, W[, K]) — the engine's
// view of servesim::SubnetConfig (reference profile.hpp:28-54) — fills in each
// op's ACTIVE widths (WeightSlice), marks skipped blocks
// (LayerSelect) and assigns each active norm layer its slot
// in the subnet's SubnetNorm statistics row.
//
// The op order and tensor/norm ordinals are the canonical ones of DESIGN.md
// §3-§5 (the oracle restates them independently in oracle/ssn_oracle.c).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <cstdlib>
#include <vector>

#include "../../include/ssn.h"
#include "../../include/ssn_rng.h"

namespace ssn {

enum OpKind : int {
  OP_INPUT = 0,    // raw host-format images -> NHWC activations
  OP_CONV = 1,     // WeightSlice conv (+SubnetNorm +act +residual)
  OP_MAXPOOL = 2,  // 3x3 s2 p1
  OP_AVGPOOL = 3,  // k = s, ceil_mode
  OP_GAP = 4,      // global average pool -> [N][C]
  OP_LINEAR = 5,   // classifier (fp32 logits)
  OP_SE = 6,       // squeeze-excite: x *= h_sigmoid(W2 relu(W1 gap(x) + b1) + b2)
  OP_EMBED = 7,    // token + position + type embeddings -> LayerNorm
  OP_ATTN = 8,     // softmax(Q K^T / sqrt(d)) V over the active heads
  OP_LAYERNORM = 9,
  OP_TOKEN0 = 10,  // gather position 0 of every sequence
};

// Logical buffer slots inside a block; mapped to arena buffers per graph.
enum Slot : int {
  S_NONE = -1,
  S_IN = 0,
  S_OUT = 1,
  S_T1 = 2,
  S_T2 = 3,
  S_T3 = 4,
  S_RAW = 5,     // input staging (raw host format)
  S_LOGITS = 6,  // fp32 logits
  S_T4 = 7,
  S_T5 = 8,
};

enum Act : int { ACT_NONE = 0, ACT_RELU = 1, ACT_HSWISH = 2, ACT_GELU = 3, ACT_TANH = 4 };

struct TensorSpec {
  int cout = 0, cin = 0, k = 1;  // max shape (depthwise: cin == 1)
  int cin_store = 0;             // stored inner dim (>= cin, multiple of 8 for bf16)
  bool depthwise = false, linear = false;
  // stored as [cout][cin_store] over the im2col order (r*k+s)*cin+c: the
  // stem conv whose im2col the input stage produces (bf16 OFA-ResNet50)
  bool im2col_stem = false;
  uint32_t fan_in = 1;
  uint64_t w_off = 0, w_bytes = 0;  // blob offsets
  uint64_t b_off = 0;               // bias (linear), fp32
};

struct NormSpec {
  int c = 0;
  bool res = false;  // last norm of a residual branch (gamma ~ U(0, SSN_RES_GAMMA))
  uint64_t gamma_off = 0, beta_off = 0;  // fp32 in the blob
};

struct OpSpec {
  int kind = OP_CONV;
  int in = S_IN, out = S_OUT, res = S_NONE;
  bool res_post = false;  // residual added after the activation
  int tensor = -1, norm = -1;
  int tensor2 = -1;            // OP_SE: expand tensor (tensor = reduce); OP_EMBED: positions
  int tensor3 = -1;            // OP_EMBED: token types
  int in2 = S_NONE, in3 = S_NONE;  // OP_ATTN: K and V
  int se_mid = 0, se_mid_max = 0;
  int act = ACT_NONE;
  int stride = 1, k_max = 1, pool_k = 0;
  int hin = 0, win = 0, hout = 0, wout = 0;
  int cin_max = 0, cout_max = 0;  // cin_max = stored inner dim
  bool depthwise = false;
  // ---- resolved for one subnet ----
  bool active = true;
  int cin = 0, cout = 0, k = 1;
  int64_t stat_off = -1;   // offset into the subnet's statistics row
  int norm_slot = -1;      // index among the subnet's active norm layers
};

struct BlockSpec {
  int first = 0, count = 0;
  int flag = -1;  // LayerSelect flag index (-1 = always runs)
  int segment = 0;
};

struct SegmentSpec {
  std::vector<int> blocks;
  std::vector<int> flags;  // distinct flags of the segment (variant bits)
};

struct Net {
  ssn_supernet_desc desc{};
  std::vector<TensorSpec> tensors;
  std::vector<NormSpec> norms;
  std::vector<OpSpec> ops;
  std::vector<BlockSpec> blocks;
  std::vector<SegmentSpec> segments;
  uint64_t blob_bytes = 0;
  int n_flags = 0;
  uint64_t stat_count = 0;  // for the resolved subnet
  int elem_bytes = 2;
};

// Control tuple in engine form.
struct SubnetCfg {
  std::vector<uint8_t> depth;
  std::vector<double> expand;
  std::vector<double> width;
  std::vector<uint32_t> kernel;
  static SubnetCfg from_c(const ssn_subnet_cfg* c) {
    SubnetCfg s;
    if (!c) return s;
    if (c->depth_flags) s.depth.assign(c->depth_flags, c->depth_flags + c->n_depth);
    if (c->expand_ratios) s.expand.assign(c->expand_ratios, c->expand_ratios + c->n_expand);
    if (c->width_multipliers)
      s.width.assign(c->width_multipliers, c->width_multipliers + c->n_width);
    if (c->kernel_sizes) s.kernel.assign(c->kernel_sizes, c->kernel_sizes + c->n_kernel);
    return s;
  }
};

inline int md8(double v) { return ssn_make_divisible(v, 8); }
inline int rnd(double v) { return ssn_round_half_even(v); }

// ---------------------------------------------------------------------------
// builder helpers

// A/B switch for the padded weight rows (SSN_PACK_WEIGHTS=1: compact rows)
inline bool pad16_weights() {
  static const bool off = [] {
    const char* v = std::getenv("SSN_PACK_WEIGHTS");
    return v && std::atoi(v) != 0;
  }();
  return !off;
}

class Builder {
 public:
  explicit Builder(Net& n) : net(n) {}

  int tensor(int cout, int cin, int k, bool dw, bool linear, int cin_store = 0) {
    TensorSpec t;
    t.cout = cout;
    t.cin = dw ? 1 : cin;
    t.k = k;
    t.depthwise = dw;
    t.linear = linear;
    // pad16: bf16 CNN supernets store every conv / linear row at a 16-channel
    // multiple (32-B rows, zero pad): TMA reads of 16-B-aligned rows (stored
    // widths 88, 360, 56, 104, 136 ... = 8 mod 16) ran at half rate
    // (tools/ubench/tma_rate.cu: 720-B pitch 97 vs 736-B 146 B/cycle/SM).
    // The pad channels meet zero-filled activations (maps bound the channel
    // dimension at the active width), so they never contribute.
    if (!cin_store && pad16 && !dw) cin_store = (cin + 15) & ~15;
    t.cin_store = dw ? 1 : (cin_store ? cin_store : cin);
    t.fan_in = static_cast<uint32_t>(t.cin * k * k);
    net.tensors.push_back(t);
    return static_cast<int>(net.tensors.size()) - 1;
  }
  int norm(int c, bool res = false) {
    NormSpec n;
    n.c = c;
    n.res = res;
    net.norms.push_back(n);
    return static_cast<int>(net.norms.size()) - 1;
  }
  void begin_block(int flag) {
    BlockSpec b;
    b.first = static_cast<int>(net.ops.size());
    b.flag = flag;
    b.segment = cur_segment;
    net.blocks.push_back(b);
  }
  void end_block() {
    auto& b = net.blocks.back();
    b.count = static_cast<int>(net.ops.size()) - b.first;
    net.segments[cur_segment].blocks.push_back(static_cast<int>(net.blocks.size()) - 1);
    if (b.flag >= 0) net.segments[cur_segment].flags.push_back(b.flag);
  }
  void begin_segment() {
    net.segments.emplace_back();
    cur_segment = static_cast<int>(net.segments.size()) - 1;
  }
  OpSpec& op(int kind) {
    net.ops.emplace_back();
    net.ops.back().kind = kind;
    return net.ops.back();
  }

  Net& net;
  int cur_segment = -1;
  bool pad16 = false;
};

inline void finalize_layout(Net& net) {
  // Blob: weight tensors (256-B aligned), then fp32 biases, gammas, betas.
  const int eb = net.elem_bytes;
  uint64_t off = 0;
  auto align = [](uint64_t v) { return (v + 255) & ~uint64_t(255); };
  for (auto& t : net.tensors) {
    off = align(off);
    t.w_off = off;
    t.w_bytes = t.im2col_stem ? uint64_t(t.cout) * t.cin_store * eb
                              : uint64_t(t.cout) * t.k * t.k * t.cin_store * eb;
    off += t.w_bytes;
  }
  for (auto& t : net.tensors) {
    if (!t.linear) continue;
    off = align(off);
    t.b_off = off;
    off += uint64_t(t.cout) * 4;
  }
  for (auto& n : net.norms) {
    off = align(off);
    n.gamma_off = off;
    off += uint64_t(n.c) * 4;
    off = align(off);
    n.beta_off = off;
    off += uint64_t(n.c) * 4;
  }
  net.blob_bytes = align(off);
  net.n_flags = 0;
  for (auto& b : net.blocks) net.n_flags = std::max(net.n_flags, b.flag + 1);
}

// Assign statistics slots to active norm layers in execution order.
// SubnetNorm applies to BatchNorm-style norms only; LayerNorm (and the
// embedding LN) normalise per token and keep no per-subnet statistics.
inline bool has_subnet_norm(const OpSpec& o) {
  return o.active && o.norm >= 0 && o.kind != OP_LAYERNORM && o.kind != OP_EMBED;
}

inline void assign_stats(Net& net) {
  uint64_t cursor = 0;
  int slot = 0;
  for (auto& o : net.ops) {
    if (!has_subnet_norm(o)) continue;
    o.stat_off = static_cast<int64_t>(cursor);
    o.norm_slot = slot++;
    cursor += static_cast<uint64_t>(o.cout);
  }
  net.stat_count = cursor;
}

inline void mark_blocks(Net& net, const std::vector<uint8_t>& depth) {
  for (auto& b : net.blocks) {
    const bool on = b.flag < 0 || depth[b.flag];
    for (int i = 0; i < b.count; ++i) net.ops[b.first + i].active = on;
  }
}

// ---------------------------------------------------------------------------
// Config 1 — TinyCNN. D = 5, E = 3, W = 4.

inline Net build_tinycnn(const ssn_supernet_desc& d, const SubnetCfg* cfg) {
  static const int BASE[4] = {32, 32, 64, 128};
  static const double MAX_E = 6.0;
  struct B { int stage, stride, flag; bool res; };
  static const B BLK[8] = {{0, 1, -1, false}, {0, 1, 0, true}, {0, 1, 1, true},
                           {1, 2, -1, false}, {1, 1, 2, true}, {1, 1, 3, true},
                           {2, 2, -1, false}, {2, 1, 4, true}};
  SubnetCfg mx;
  mx.depth.assign(5, 1);
  mx.expand.assign(3, MAX_E);
  mx.width.assign(4, 1.0);
  const SubnetCfg& s = cfg ? *cfg : mx;
  if (s.depth.size() != 5 || s.expand.size() != 3 || s.width.size() != 4)
    throw std::invalid_argument(
        "tinycnn subnet needs 5 depth flags, 3 expand ratios, 4 width multipliers");
  for (double e : s.expand)
    if (!(e > 0.0) || e > MAX_E) throw std::invalid_argument("expand ratio must be in (0, 6]");
  for (double w : s.width)
    if (!(w > 0.0) || w > 1.0) throw std::invalid_argument("width multiplier must be in (0,1]");

  Net net;
  net.desc = d;
  net.elem_bytes = d.dtype == SSN_DTYPE_BF16 ? 2 : 4;
  const bool bf16 = d.dtype == SSN_DTYPE_BF16;
  Builder b(net);
  const int H = static_cast<int>(d.image_size);
  int C[4];
  for (int i = 0; i < 4; ++i) C[i] = md8(BASE[i] * s.width[i]);

  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_INPUT);
    o.in = S_RAW;
    o.hin = o.hout = H;
    o.win = o.wout = H;
    o.cin_max = 3;
    o.cout_max = o.cout = bf16 ? 8 : 3;
    o.cin = 3;
  }
  b.end_block();
  const int t_stem = b.tensor(BASE[0], 3, 3, false, false, bf16 ? 8 : 3);
  const int n_stem = b.norm(BASE[0]);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = t_stem;
    o.norm = n_stem;
    o.act = ACT_RELU;
    o.k_max = o.k = 3;
    o.stride = 1;
    o.hin = o.hout = H;
    o.win = o.wout = H;
    o.cin_max = bf16 ? 8 : 3;
    o.cin = bf16 ? 8 : 3;
    o.cout_max = BASE[0];
    o.cout = C[0];
  }
  b.end_block();

  int hw = H, cin_max = BASE[0], cin_a = C[0];
  int stage_seen = -1;
  for (int bi = 0; bi < 8; ++bi) {
    const B& blk = BLK[bi];
    if (blk.stage != stage_seen) {
      b.begin_segment();
      stage_seen = blk.stage;
    }
    const int cout_max = BASE[1 + blk.stage];
    const int hid_max = md8(rnd(cin_max * MAX_E));
    const int t1 = b.tensor(hid_max, cin_max, 1, false, false);
    const int n1 = b.norm(hid_max);
    const int t2 = b.tensor(hid_max, hid_max, 3, true, false);
    const int n2 = b.norm(hid_max);
    const int t3 = b.tensor(cout_max, hid_max, 1, false, false);
    const int n3 = b.norm(cout_max, blk.res);
    const bool on = blk.flag < 0 || s.depth[blk.flag];
    // active dims of this block (a skipped block forwards its input)
    const int cout_a = C[1 + blk.stage];
    const int hid = md8(rnd(cin_a * s.expand[blk.stage]));
    const int hw_out = (hw + 2 - 3) / blk.stride + 1;
    b.begin_block(blk.flag);
    {
      auto& o = b.op(OP_CONV);
      o.in = S_IN; o.out = S_T1;
      o.tensor = t1; o.norm = n1; o.act = ACT_RELU;
      o.hin = o.hout = hw; o.win = o.wout = hw;
      o.cin_max = cin_max; o.cout_max = hid_max;
      o.cin = cin_a; o.cout = hid;
    }
    {
      auto& o = b.op(OP_CONV);
      o.in = S_T1; o.out = S_T2;
      o.tensor = t2; o.norm = n2; o.act = ACT_RELU;
      o.depthwise = true;
      o.k_max = o.k = 3; o.stride = blk.stride;
      o.hin = hw; o.win = hw; o.hout = hw_out; o.wout = hw_out;
      o.cin_max = hid_max; o.cout_max = hid_max;
      o.cin = hid; o.cout = hid;
    }
    {
      auto& o = b.op(OP_CONV);
      o.in = S_T2; o.out = S_OUT;
      o.res = blk.res ? S_IN : S_NONE;
      o.tensor = t3; o.norm = n3; o.act = ACT_NONE;
      o.hin = o.hout = hw_out; o.win = o.wout = hw_out;
      o.cin_max = hid_max; o.cout_max = cout_max;
      o.cin = hid; o.cout = cout_a;
    }
    b.end_block();
    if (blk.res && on && cin_a != cout_a)
      throw std::invalid_argument("residual block shape mismatch");
    if (on) cin_a = cout_a;
    cin_max = cout_max;
    hw = hw_out;
  }
  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_GAP);
    o.hin = o.win = hw;
    o.hout = o.wout = 1;
    o.cin_max = o.cout_max = BASE[3];
    o.cin = o.cout = cin_a;
  }
  b.end_block();
  const int tl = b.tensor(static_cast<int>(d.num_classes), BASE[3], 1, false, true);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_LINEAR);
    o.out = S_LOGITS;
    o.tensor = tl;
    o.hin = o.win = o.hout = o.wout = 1;
    o.cin_max = BASE[3];
    o.cout_max = static_cast<int>(d.num_classes);
    o.cin = cin_a;
    o.cout = static_cast<int>(d.num_classes);
  }
  b.end_block();
  finalize_layout(net);
  mark_blocks(net, s.depth);
  assign_stats(net);
  return net;
}

// ---------------------------------------------------------------------------
// Config 2 — OFA-ResNet50. D = 9 per-block flags, E = 18,
// W = 6.  Layout follows OFA's OFAResNets / DynamicResNetBottleneckBlock
// [external]: stem (conv3x3 s2, residual conv3x3, conv3x3), maxpool, 4 stages
// of bottlenecks (base depth 2/2/4/2, +2 optional), avgpool_conv downsample.

inline Net build_ofa_resnet50(const ssn_supernet_desc& d, const SubnetCfg* cfg) {
  static const int STAGE_W[4] = {256, 512, 1024, 2048};
  static const int BASE_DEPTH[4] = {2, 2, 4, 2};
  static const int NBLK[4] = {4, 4, 6, 4};
  static const double MAX_E = 0.35;
  SubnetCfg mx;
  mx.depth.assign(9, 1);
  mx.expand.assign(18, MAX_E);
  mx.width.assign(6, 1.0);
  const SubnetCfg& s = cfg ? *cfg : mx;
  if (s.depth.size() != 9 || s.expand.size() != 18 || s.width.size() != 6)
    throw std::invalid_argument(
        "ofa_resnet50 subnet needs 9 depth flags, 18 expand ratios, 6 width multipliers");
  for (double w : s.width)
    if (!(w > 0.0) || w > 1.0) throw std::invalid_argument("width multiplier must be in (0,1]");
  for (double e : s.expand)
    if (!(e > 0.0)) throw std::invalid_argument("expand ratio must be > 0");

  Net net;
  net.desc = d;
  const bool bf16 = d.dtype == SSN_DTYPE_BF16;
  net.elem_bytes = bf16 ? 2 : 4;
  Builder b(net);
  b.pad16 = bf16 && pad16_weights();
  const int H = static_cast<int>(d.image_size);
  const int stem_mid_a = md8(md8(64 * s.width[0]) / 2);
  const int stem_out_a = md8(64 * s.width[1]);
  const int H2 = (H + 2 - 3) / 2 + 1;

  // ---- segment 0: input, stem, maxpool
  // bf16: the input stage emits the stem conv's im2col directly (3x3 s2 p1
  // over 3 channels = 27 values, padded to 32), so stem conv0 runs as a
  // K = 32 GEMM on the tensor cores instead of nine nearly-empty taps.
  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_INPUT);
    o.in = S_RAW;
    o.hin = H; o.win = H;
    o.cin_max = 3; o.cin = 3;
    if (bf16) {
      o.k_max = o.k = 3; o.stride = 2;  // im2col geometry
      o.hout = o.wout = H2;
      o.cout_max = o.cout = 32;
    } else {
      o.hout = o.wout = H;
      o.cout_max = o.cout = 3;
    }
  }
  b.end_block();
  const int t0 = b.tensor(32, 3, 3, false, false, bf16 ? 32 : 3);
  if (bf16) net.tensors[t0].im2col_stem = true;
  const int n0 = b.norm(32);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = t0; o.norm = n0; o.act = ACT_RELU;
    if (bf16) {
      o.k_max = o.k = 1; o.stride = 1;
      o.hin = o.win = H2;
      o.cin_max = o.cin = 32;
    } else {
      o.k_max = o.k = 3; o.stride = 2;
      o.hin = o.win = H;
      o.cin_max = o.cin = 3;
    }
    o.hout = o.wout = H2;
    o.cout_max = 32; o.cout = stem_mid_a;
  }
  b.end_block();
  const int t1 = b.tensor(32, 32, 3, false, false);
  const int n1 = b.norm(32, true);
  b.begin_block(0);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = t1; o.norm = n1; o.act = ACT_RELU;
    o.res = S_IN; o.res_post = true;
    o.k_max = o.k = 3; o.stride = 1;
    o.hin = o.hout = H2; o.win = o.wout = H2;
    o.cin_max = 32; o.cin = stem_mid_a;
    o.cout_max = 32; o.cout = stem_mid_a;
  }
  b.end_block();
  const int t2 = b.tensor(64, 32, 3, false, false);
  const int n2 = b.norm(64);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = t2; o.norm = n2; o.act = ACT_RELU;
    o.k_max = o.k = 3; o.stride = 1;
    o.hin = o.hout = H2; o.win = o.wout = H2;
    o.cin_max = 32; o.cin = stem_mid_a;
    o.cout_max = 64; o.cout = stem_out_a;
  }
  b.end_block();
  const int H4 = (H2 + 2 - 3) / 2 + 1;
  b.begin_block(-1);
  {
    auto& o = b.op(OP_MAXPOOL);
    o.k_max = o.k = 3; o.stride = 2;
    o.hin = o.win = H2; o.hout = o.wout = H4;
    o.cin_max = o.cout_max = 64;
    o.cin = o.cout = stem_out_a;
  }
  b.end_block();

  // ---- segments 1..4: bottleneck stages
  int hw = H4, cin_max = 64, cin_a = stem_out_a, blk_idx = 0;
  for (int st = 0; st < 4; ++st) {
    b.begin_segment();
    const int out_max = STAGE_W[st];
    const int mid_max = md8(rnd(out_max * MAX_E));
    const int out_a = md8(out_max * s.width[2 + st]);
    const int stride = st == 0 ? 1 : 2;
    for (int bi = 0; bi < NBLK[st]; ++bi, ++blk_idx) {
      const int flag = bi >= BASE_DEPTH[st] ? 1 + 2 * st + (bi - BASE_DEPTH[st]) : -1;
      const int mid_a = md8(rnd(out_a * s.expand[blk_idx]));
      if (mid_a > mid_max)
        throw std::invalid_argument("expand ratio exceeds the supernet's max middle width");
      const bool first = bi == 0;
      const int st_ = first ? stride : 1;
      const int hw_out = (hw + 2 - 3) / st_ + 1;
      b.begin_block(flag);
      if (first) {
        const int td = b.tensor(out_max, cin_max, 1, false, false);
        const int nd = b.norm(out_max);
        int ds_in = S_IN;
        if (stride > 1) {
          auto& p = b.op(OP_AVGPOOL);
          p.in = S_IN; p.out = S_T1;
          p.pool_k = p.stride = stride;
          p.k_max = p.k = stride;
          p.hin = p.win = hw;
          p.hout = p.wout = (hw + stride - 1) / stride;
          p.cin_max = p.cout_max = cin_max;
          p.cin = p.cout = cin_a;
          ds_in = S_T1;
        }
        auto& o = b.op(OP_CONV);
        o.in = ds_in; o.out = S_T3;
        o.tensor = td; o.norm = nd; o.act = ACT_NONE;
        o.hin = o.win = o.hout = o.wout = (hw + stride - 1) / stride;
        o.cin_max = cin_max; o.cin = cin_a;
        o.cout_max = out_max; o.cout = out_a;
      }
      const int ta = b.tensor(mid_max, cin_max, 1, false, false);
      const int na = b.norm(mid_max);
      const int tb = b.tensor(mid_max, mid_max, 3, false, false);
      const int nb = b.norm(mid_max);
      const int tc = b.tensor(out_max, mid_max, 1, false, false);
      const int nc = b.norm(out_max, true);
      {
        auto& o = b.op(OP_CONV);
        o.in = S_IN; o.out = S_T1;
        o.tensor = ta; o.norm = na; o.act = ACT_RELU;
        o.hin = o.hout = hw; o.win = o.wout = hw;
        o.cin_max = cin_max; o.cin = cin_a;
        o.cout_max = mid_max; o.cout = mid_a;
      }
      {
        auto& o = b.op(OP_CONV);
        o.in = S_T1; o.out = S_T2;
        o.tensor = tb; o.norm = nb; o.act = ACT_RELU;
        o.k_max = o.k = 3; o.stride = st_;
        o.hin = hw; o.win = hw; o.hout = hw_out; o.wout = hw_out;
        o.cin_max = mid_max; o.cin = mid_a;
        o.cout_max = mid_max; o.cout = mid_a;
      }
      {
        auto& o = b.op(OP_CONV);
        o.in = S_T2; o.out = S_OUT;
        o.res = first ? S_T3 : S_IN;
        o.tensor = tc; o.norm = nc; o.act = ACT_RELU;
        o.hin = o.hout = hw_out; o.win = o.wout = hw_out;
        o.cin_max = mid_max; o.cin = mid_a;
        o.cout_max = out_max; o.cout = out_a;
      }
      b.end_block();
      const bool on = flag < 0 || s.depth[flag];
      if (on) cin_a = out_a;
      cin_max = out_max;
      hw = hw_out;
    }
  }

  // ---- segment 5: global pool + classifier
  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_GAP);
    o.hin = o.win = hw;
    o.hout = o.wout = 1;
    o.cin_max = o.cout_max = 2048;
    o.cin = o.cout = cin_a;
  }
  b.end_block();
  const int tl = b.tensor(static_cast<int>(d.num_classes), 2048, 1, false, true);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_LINEAR);
    o.out = S_LOGITS;
    o.tensor = tl;
    o.hin = o.win = o.hout = o.wout = 1;
    o.cin_max = 2048;
    o.cout_max = static_cast<int>(d.num_classes);
    o.cin = cin_a;
    o.cout = static_cast<int>(d.num_classes);
  }
  b.end_block();
  finalize_layout(net);
  mark_blocks(net, s.depth);
  assign_stats(net);
  return net;
}

// ---------------------------------------------------------------------------
// Config 3 — OFA-MobileNetV3, width 1.2 ([external] OFA
// OFAMobileNetV3 / DynamicMBConvLayer / DynamicSE).  D = 10 flags (blocks 3-4
// of each of the 5 stages), E = 20 per-block expand ratios (<= 6), K = 20
// per-block depthwise kernel sizes (3/5/7, centre crop of 7x7), W = [1.0]
// (the supernet's width is fixed).

inline Net build_ofa_mbv3(const ssn_supernet_desc& d, const SubnetCfg* cfg) {
  static const int WIDTH[5] = {32, 48, 96, 136, 192};  // md(24/40/80/112/160 * 1.2)
  static const int STRIDE[5] = {2, 2, 2, 1, 2};
  static const int ACT[5] = {ACT_RELU, ACT_RELU, ACT_HSWISH, ACT_HSWISH, ACT_HSWISH};
  static const bool SE[5] = {false, true, false, true, true};
  static const double MAX_E = 6.0;
  SubnetCfg mx;
  mx.depth.assign(10, 1);
  mx.expand.assign(20, MAX_E);
  mx.width.assign(1, 1.0);
  mx.kernel.assign(20, 7);
  const SubnetCfg& s = cfg ? *cfg : mx;
  if (s.depth.size() != 10 || s.expand.size() != 20 || s.width.size() != 1)
    throw std::invalid_argument(
        "ofa_mbv3 subnet needs 10 depth flags, 20 expand ratios, 1 width multiplier");
  if (!s.kernel.empty() && s.kernel.size() != 20)
    throw std::invalid_argument("ofa_mbv3 subnet needs 20 kernel sizes (or none)");
  if (s.width[0] != 1.0)
    throw std::invalid_argument("ofa_mbv3 supernet has a fixed width: width multiplier must be 1.0");
  for (double e : s.expand)
    if (!(e > 0.0) || e > MAX_E) throw std::invalid_argument("expand ratio must be in (0, 6]");
  for (uint32_t k : s.kernel)
    if (k != 3 && k != 5 && k != 7) throw std::invalid_argument("kernel size must be 3, 5 or 7");

  Net net;
  net.desc = d;
  if (d.dtype != SSN_DTYPE_BF16) throw std::invalid_argument("ofa_mbv3 runs in bf16");
  net.elem_bytes = 2;
  Builder b(net);
  b.pad16 = pad16_weights();
  const int H = static_cast<int>(d.image_size);
  const int H2 = (H + 2 - 3) / 2 + 1;

  // ---- segment 0: input (stem im2col), first conv, first block
  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_INPUT);
    o.in = S_RAW;
    o.hin = o.win = H;
    o.k_max = o.k = 3; o.stride = 2;
    o.hout = o.wout = H2;
    o.cin_max = o.cin = 3;
    o.cout_max = o.cout = 32;
  }
  b.end_block();
  const int t0 = b.tensor(24, 3, 3, false, false, 32);
  net.tensors[t0].im2col_stem = true;
  const int n0 = b.norm(24);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = t0; o.norm = n0; o.act = ACT_HSWISH;
    o.k_max = o.k = 1;
    o.hin = o.win = o.hout = o.wout = H2;
    o.cin_max = o.cin = 32;
    o.cout_max = o.cout = 24;
  }
  b.end_block();
  // first block: MBConv(expand 1): dw 3x3 + BN + ReLU, point 1x1 + BN, identity residual
  const int t1 = b.tensor(24, 1, 3, true, false);
  const int n1 = b.norm(24);
  const int t2 = b.tensor(24, 24, 1, false, false);
  const int n2 = b.norm(24, true);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.in = S_IN; o.out = S_T1;
    o.tensor = t1; o.norm = n1; o.act = ACT_RELU; o.depthwise = true;
    o.k_max = o.k = 3;
    o.hin = o.win = o.hout = o.wout = H2;
    o.cin_max = o.cin = o.cout_max = o.cout = 24;
  }
  {
    auto& o = b.op(OP_CONV);
    o.in = S_T1; o.out = S_OUT; o.res = S_IN;
    o.tensor = t2; o.norm = n2; o.act = ACT_NONE;
    o.hin = o.win = o.hout = o.wout = H2;
    o.cin_max = o.cin = o.cout_max = o.cout = 24;
  }
  b.end_block();

  // ---- segments 1..5: inverted-residual stages
  int hw = H2, cin_max = 24, cin_a = 24, blk = 0;
  for (int st = 0; st < 5; ++st) {
    b.begin_segment();
    for (int bi = 0; bi < 4; ++bi, ++blk) {
      const int flag = bi >= 2 ? 2 * st + (bi - 2) : -1;
      const int stride = bi == 0 ? STRIDE[st] : 1;
      const int cout = WIDTH[st];
      const bool res = stride == 1 && cin_max == cout;
      const int mid_max = md8(rnd(cin_max * MAX_E));
      const int mid = md8(rnd(cin_a * s.expand[blk]));
      const int ka = s.kernel.empty() ? 7 : static_cast<int>(s.kernel[blk]);
      const int hw_out = (hw - 1) / stride + 1;  // "same" padding k/2
      const int ti = b.tensor(mid_max, cin_max, 1, false, false);
      const int ni = b.norm(mid_max);
      const int td = b.tensor(mid_max, 1, 7, true, false);
      const int nd = b.norm(mid_max);
      int tr = -1, te = -1;
      const int se_max = md8(mid_max / 4);
      if (SE[st]) {
        // SE FCs keep compact rows (se_fc_kernel's row strides: c_max / se_max)
        tr = b.tensor(se_max, mid_max, 1, false, true, mid_max);  // reduce (+bias)
        te = b.tensor(mid_max, se_max, 1, false, true, se_max);   // expand (+bias)
      }
      const int tp = b.tensor(cout, mid_max, 1, false, false);
      const int np = b.norm(cout, res);
      b.begin_block(flag);
      {
        auto& o = b.op(OP_CONV);
        o.in = S_IN; o.out = S_T1;
        o.tensor = ti; o.norm = ni; o.act = ACT[st];
        o.hin = o.win = o.hout = o.wout = hw;
        o.cin_max = cin_max; o.cin = cin_a;
        o.cout_max = mid_max; o.cout = mid;
      }
      {
        auto& o = b.op(OP_CONV);
        o.in = S_T1; o.out = S_T2;
        o.tensor = td; o.norm = nd; o.act = ACT[st]; o.depthwise = true;
        o.k_max = 7; o.k = ka; o.stride = stride;
        o.hin = o.win = hw; o.hout = o.wout = hw_out;
        o.cin_max = o.cout_max = mid_max;
        o.cin = o.cout = mid;
      }
      if (SE[st]) {
        auto& o = b.op(OP_SE);
        o.in = S_T2; o.out = S_T2;  // scales in place
        o.tensor = tr; o.tensor2 = te;
        o.hin = o.win = o.hout = o.wout = hw_out;
        o.cin_max = o.cout_max = mid_max;
        o.cin = o.cout = mid;
        o.se_mid = md8(mid / 4);
        o.se_mid_max = se_max;
      }
      {
        auto& o = b.op(OP_CONV);
        o.in = S_T2; o.out = S_OUT;
        o.res = res ? S_IN : S_NONE;
        o.tensor = tp; o.norm = np; o.act = ACT_NONE;
        o.hin = o.win = o.hout = o.wout = hw_out;
        o.cin_max = mid_max; o.cin = mid;
        o.cout_max = o.cout = cout;
      }
      b.end_block();
      const bool on = flag < 0 || s.depth[flag];
      if (on) cin_a = cout;
      cin_max = cout;
      hw = hw_out;
    }
  }

  // ---- segment 6: final expand, pool, feature mix, classifier
  b.begin_segment();
  const int tf = b.tensor(1152, 192, 1, false, false);
  const int nf = b.norm(1152);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);
    o.tensor = tf; o.norm = nf; o.act = ACT_HSWISH;
    o.hin = o.win = o.hout = o.wout = hw;
    o.cin_max = o.cin = 192;
    o.cout_max = o.cout = 1152;
  }
  b.end_block();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_GAP);
    o.hin = o.win = hw;
    o.hout = o.wout = 1;
    o.cin_max = o.cout_max = o.cin = o.cout = 1152;
  }
  b.end_block();
  const int tm = b.tensor(1536, 1152, 1, false, false);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_CONV);  // feature mix: no norm, no bias
    o.tensor = tm; o.act = ACT_HSWISH;
    o.hin = o.win = o.hout = o.wout = 1;
    o.cin_max = o.cin = 1152;
    o.cout_max = o.cout = 1536;
  }
  b.end_block();
  const int tl = b.tensor(static_cast<int>(d.num_classes), 1536, 1, false, true);
  b.begin_block(-1);
  {
    auto& o = b.op(OP_LINEAR);
    o.out = S_LOGITS;
    o.tensor = tl;
    o.hin = o.win = o.hout = o.wout = 1;
    o.cin_max = o.cin = 1536;
    o.cout_max = o.cout = static_cast<int>(d.num_classes);
  }
  b.end_block();
  finalize_layout(net);
  mark_blocks(net, s.depth);
  assign_stats(net);
  return net;
}

// ---------------------------------------------------------------------------
// Config 5 — width/depth-sliced BERT-base-like encoder (DESIGN.md §3.4,
// [external] DynaBERT).  Post-LN layers: Q/K/V linears over the active heads,
// softmax attention, output projection (+residual) -> LayerNorm, FFN with
// GELU (+residual) -> LayerNorm; tanh pooler on token 0; classifier.
//   D = 12 per-layer LayerSelect flags, E = [FFN width multiplier],
//   W = [attention-head width multiplier] (heads_a = round(12 W), ffn_a =
//   md(3072 E)).  desc.image_size = sequence length, num_classes = labels.
// No BatchNorm: SubnetNorm statistics are empty for this family.

inline Net build_bert(const ssn_supernet_desc& d, const SubnetCfg* cfg) {
  static const int HID = 768, HEADS = 12, HD = 64, FFN = 3072, LAYERS = 12, VOCAB = 30522;
  SubnetCfg mx;
  mx.depth.assign(LAYERS, 1);
  mx.expand.assign(1, 1.0);
  mx.width.assign(1, 1.0);
  const SubnetCfg& s = cfg ? *cfg : mx;
  if (s.depth.size() != LAYERS || s.expand.size() != 1 || s.width.size() != 1)
    throw std::invalid_argument(
        "bert subnet needs 12 depth flags, 1 FFN width (expand) ratio, 1 head width multiplier");
  if (!(s.width[0] > 0.0) || s.width[0] > 1.0)
    throw std::invalid_argument("width multiplier must be in (0,1]");
  if (!(s.expand[0] > 0.0) || s.expand[0] > 1.0)
    throw std::invalid_argument("FFN expand ratio must be in (0,1]");
  if (d.dtype != SSN_DTYPE_BF16) throw std::invalid_argument("bert runs in bf16");
  if (d.image_size != 128)  // attention kernel keeps one 128-token sequence per CTA
    throw std::invalid_argument("bert sequence length (image_size) must be 128");
  const int heads = std::max(1, rnd(HEADS * s.width[0]));
  const int ffn = std::min(FFN, md8(FFN * s.expand[0]));
  const int S = static_cast<int>(d.image_size);

  Net net;
  net.desc = d;
  net.elem_bytes = 2;
  Builder b(net);
  // tensors (canonical ordinals): embeddings, then per layer q,k,v,o,f1,f2, pooler, classifier
  const int t_tok = b.tensor(VOCAB, HID, 1, false, false);
  const int t_pos = b.tensor(512, HID, 1, false, false);
  const int t_typ = b.tensor(2, HID, 1, false, false);
  const int n_emb = b.norm(HID);
  auto lin = [&](int kind, int in, int out, int res, int t, int cin, int cin_max, int cout,
                 int cout_max, int act) {
    auto& o = b.op(kind);
    o.in = in; o.out = out; o.res = res;
    o.tensor = t; o.act = act;
    o.hin = o.hout = S; o.win = o.wout = 1;
    o.cin = cin; o.cin_max = cin_max; o.cout = cout; o.cout_max = cout_max;
    return &o;
  };
  auto ln = [&](int in, int out, int nrm) {
    auto& o = b.op(OP_LAYERNORM);
    o.in = in; o.out = out; o.norm = nrm;
    o.hin = o.hout = S; o.win = o.wout = 1;
    o.cin = o.cin_max = o.cout = o.cout_max = HID;
  };

  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_EMBED);
    o.in = S_RAW; o.out = S_OUT;
    o.tensor = t_tok; o.tensor2 = t_pos; o.tensor3 = t_typ; o.norm = n_emb;
    o.hin = o.hout = S; o.win = o.wout = 1;
    o.cin = o.cin_max = 1;
    o.cout = o.cout_max = HID;
  }
  b.end_block();
  for (int l = 0; l < LAYERS; ++l) {
    const int tq = b.tensor(HID, HID, 1, false, true);
    const int tk = b.tensor(HID, HID, 1, false, true);
    const int tv = b.tensor(HID, HID, 1, false, true);
    const int to = b.tensor(HID, HID, 1, false, true);
    const int n1 = b.norm(HID);
    const int t1 = b.tensor(FFN, HID, 1, false, true);
    const int t2 = b.tensor(HID, FFN, 1, false, true);
    const int n2 = b.norm(HID);
    b.begin_segment();
    b.begin_block(l);
    lin(OP_CONV, S_IN, S_T1, S_NONE, tq, HID, HID, heads * HD, HID, ACT_NONE);
    lin(OP_CONV, S_IN, S_T2, S_NONE, tk, HID, HID, heads * HD, HID, ACT_NONE);
    lin(OP_CONV, S_IN, S_T3, S_NONE, tv, HID, HID, heads * HD, HID, ACT_NONE);
    {
      auto& o = b.op(OP_ATTN);
      o.in = S_T1; o.in2 = S_T2; o.in3 = S_T3; o.out = S_T4;
      o.hin = o.hout = S; o.win = o.wout = 1;
      o.cin = o.cout = heads * HD; o.cin_max = o.cout_max = HID;
      o.k_max = o.k = HD;  // head dim
    }
    lin(OP_CONV, S_T4, S_T5, S_IN, to, heads * HD, HID, HID, HID, ACT_NONE);
    ln(S_T5, S_T1, n1);
    lin(OP_CONV, S_T1, S_T4, S_NONE, t1, HID, HID, ffn, FFN, ACT_GELU);
    lin(OP_CONV, S_T4, S_T2, S_T1, t2, ffn, FFN, HID, HID, ACT_NONE);
    ln(S_T2, S_OUT, n2);
    b.end_block();
  }
  b.begin_segment();
  b.begin_block(-1);
  {
    auto& o = b.op(OP_TOKEN0);  // [B][S][768] -> [B][768] (the [CLS] position)
    o.hin = S; o.win = 1; o.hout = o.wout = 1;
    o.cin = o.cin_max = o.cout = o.cout_max = HID;
  }
  b.end_block();
  const int tp = b.tensor(HID, HID, 1, false, true);
  b.begin_block(-1);
  {
    auto* o = lin(OP_CONV, S_IN, S_OUT, S_NONE, tp, HID, HID, HID, HID, ACT_TANH);
    o->hin = o->hout = 1;
  }
  b.end_block();
  const int tc = b.tensor(static_cast<int>(d.num_classes), HID, 1, false, true);
  b.begin_block(-1);
  {
    auto* o = lin(OP_LINEAR, S_IN, S_LOGITS, S_NONE, tc, HID, HID, static_cast<int>(d.num_classes),
                  static_cast<int>(d.num_classes), ACT_NONE);
    o->hin = o->hout = 1;
  }
  b.end_block();
  finalize_layout(net);
  mark_blocks(net, s.depth);
  assign_stats(net);
  return net;
}

inline Net build_net(const ssn_supernet_desc& d, const SubnetCfg* cfg) {
  switch (d.family) {
    case SSN_FAMILY_TINYCNN: return build_tinycnn(d, cfg);
    case SSN_FAMILY_OFA_RESNET50: return build_ofa_resnet50(d, cfg);
    case SSN_FAMILY_OFA_MBV3: return build_ofa_mbv3(d, cfg);
    case SSN_FAMILY_BERT: return build_bert(d, cfg);
    default: throw std::invalid_argument("unsupported supernet family");
  }
}

}  // namespace ssn
