/*
 * ssn_oracle.c — CPU float32 restatement of the SubNetAct operators and the
 * supernets this build executes.  TEST INFRASTRUCTURE ONLY: it is the parity
 * checker (tests/, __graft_entry__.smoke()) and the CPU baseline leg of
 * bench.py.  The product (paper_2312_16733_b200/) never links or calls it.
 *
 * PARITY PINNING.  The reference (servesim) contains no tensor operators:
 * SPEC.md:8 and SPEC.md:99 put "the TorchScript operator implementations of
 * LayerSelect/SubnetNorm/WeightSlice on tensors" out of scope, and workers
 * sleep (serve_runtime.hpp:167).  The tensor side of this oracle is therefore
 * "parity unpinned" by the reference; it restates the operator semantics of
 * PAPER.md:462-510 and the OFA supernet layouts ([external]),
 * and is cross-checked against torch-CPU conv2d / batch_norm / pools through
 * the committed fixtures under tests/golden/ (tests/golden/make_golden.py).
 * Subnet SELECTION is pinned separately against the reference itself
 * (oracle/_ref, built from /root/reference by oracle/Makefile).
 *
 * Operator semantics followed here:
 *   WeightSlice: a subnet with active widths
 *                (cout_a, cin_a, k_a) uses W[:cout_a, :cin_a, centre k_a x k_a]
 *                of the max-shape tensor.
 *   SubnetNorm: BN layer j of subnet i normalises with
 *                (mu_ij, var_ij); gamma_j / beta_j are shared leading slices.
 *                Calibration ("forward pass inference on the training data")
 *                = batch statistics over (N, H, W), biased variance, each BN
 *                normalising with its own batch statistics.
 *   LayerSelect: a skipped block forwards its input.
 *   The control tuple shape follows servesim::SubnetConfig
 *   (reference profile.hpp:28-54) and validate() (profile.hpp:40-53).
 *
 * Layouts here are deliberately independent from the engine's: weights are
 * generated in canonical OIHW order and kept as [cout][k*k][cin] (so a
 * KRSC/OIHW mix-up in either side fails parity), activations NHWC float32.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/ssn.h"
#include "../include/ssn_rng.h"

#define OR_EPS 1e-5f

static __thread char g_err[512];
const char* oracle_last_error(void) { return g_err; }
#define FAIL(...)                                   \
  do {                                              \
    snprintf(g_err, sizeof g_err, __VA_ARGS__);     \
    return -1;                                      \
  } while (0)

/* ------------------------------------------------------------------------- */
/* tensors                                                                    */

typedef struct {
  int n, h, w, c;
  float* d;
} T4;

static T4 t4_new(int n, int h, int w, int c) {
  T4 t = {n, h, w, c, NULL};
  t.d = (float*)calloc((size_t)n * h * w * c + 1, sizeof(float));
  return t;
}
static void t4_free(T4* t) {
  free(t->d);
  t->d = NULL;
}
static size_t t4_size(const T4* t) { return (size_t)t->n * t->h * t->w * t->c; }

/* ------------------------------------------------------------------------- */
/* weight store (max shapes)                                                  */

typedef struct {
  int cout, cin, k; /* max shape; depthwise: cin == 1                       */
  int depthwise;
  float* w;         /* [cout][k*k][cin] */
  float* bias;      /* linear only      */
} OTensor;

typedef struct {
  int c;
  float* gamma;
  float* beta;
} ONorm;

#define OR_MAX_T 128
struct oracle_net {
  int family;
  uint64_t seed;
  int classes;
  int bf16_w;
  int nt, nn;
  OTensor t[OR_MAX_T];
  ONorm nm[OR_MAX_T];
};
typedef struct oracle_net oracle_net;

static int add_tensor(oracle_net* o, int cout, int cin, int k, int dw, int linear) {
  OTensor* T = &o->t[o->nt];
  const int ord = o->nt++;
  T->cout = cout;
  T->cin = dw ? 1 : cin;
  T->k = k;
  T->depthwise = dw;
  const int kk = k * k;
  T->w = (float*)malloc(sizeof(float) * (size_t)cout * kk * T->cin);
  const uint32_t fan_in = (uint32_t)(T->cin * kk);
  /* canonical OIHW index order over the max shape */
  for (int o_ = 0; o_ < cout; ++o_)
    for (int i = 0; i < T->cin; ++i)
      for (int r = 0; r < k; ++r)
        for (int s = 0; s < k; ++s) {
          const uint64_t idx = (((uint64_t)o_ * T->cin + i) * k + r) * k + s;
          T->w[((size_t)o_ * kk + r * k + s) * T->cin + i] =
              ssn_weight_value(o->seed, (uint32_t)ord, idx, fan_in, o->bf16_w);
        }
  T->bias = NULL;
  if (linear) {
    T->bias = (float*)malloc(sizeof(float) * cout);
    for (int o_ = 0; o_ < cout; ++o_) T->bias[o_] = ssn_bias_value(o->seed, (uint32_t)ord, o_);
  }
  return ord;
}

static int add_norm(oracle_net* o, int c, int res) {
  ONorm* N = &o->nm[o->nn];
  const int ord = o->nn++;
  N->c = c;
  N->gamma = (float*)malloc(sizeof(float) * c);
  N->beta = (float*)malloc(sizeof(float) * c);
  for (int i = 0; i < c; ++i) {
    N->gamma[i] = res ? ssn_gamma_res_value(o->seed, (uint32_t)ord, i)
                      : ssn_gamma_value(o->seed, (uint32_t)ord, i);
    N->beta[i] = ssn_beta_value(o->seed, (uint32_t)ord, i);
  }
  return ord;
}

/* ------------------------------------------------------------------------- */
/* run context                                                                */

typedef struct {
  oracle_net* o;
  int emulate_bf16;    /* round stored activations to bf16 (engine storage) */
  int calibrate;       /* BN with batch statistics, record them            */
  uint32_t subnet_id;  /* for default statistics                           */
  const float* mean_in;
  const float* var_in;
  float* mean_out;
  float* var_out;
  size_t stat_cursor;  /* floats consumed / produced                       */
  int active_norms;
  int count_only;      /* only count statistics                            */
  int acc64;           /* BERT linears accumulate in double (sensitivity
                          probe of the bf16-storage emulation, flag bit 2) */
} Ctx;

static void store_round(Ctx* c, T4* t) {
  if (!c->emulate_bf16) return;
  const size_t n = t4_size(t);
  for (size_t i = 0; i < n; ++i) t->d[i] = ssn_round_bf16(t->d[i]);
}

/* WeightSlice convolution: y[n,ho,wo,co] = sum_{r,s,ci} x * W[co, ci, centre]
 * over the active slice (cout_a, cin_a, k_a). */
static T4 conv2d(const T4* x, const OTensor* T, int k_a, int stride, int cout_a) {
  const int pad = k_a / 2;
  const int ho = (x->h + 2 * pad - k_a) / stride + 1;
  const int wo = (x->w + 2 * pad - k_a) / stride + 1;
  T4 y = t4_new(x->n, ho, wo, cout_a);
  const int cin_a = x->c;
  const int kmax = T->k, off = (kmax - k_a) / 2, kk = kmax * kmax;
  const long npix = (long)x->n * ho * wo;
#pragma omp parallel for schedule(static)
  for (long p = 0; p < npix; ++p) {
    const int n = (int)(p / ((long)ho * wo));
    const int rem = (int)(p % ((long)ho * wo));
    const int oh = rem / wo, ow = rem % wo;
    float* yp = y.d + (size_t)p * cout_a;
    for (int r = 0; r < k_a; ++r) {
      const int ih = oh * stride - pad + r;
      if (ih < 0 || ih >= x->h) continue;
      for (int s = 0; s < k_a; ++s) {
        const int iw = ow * stride - pad + s;
        if (iw < 0 || iw >= x->w) continue;
        const float* xp = x->d + (((size_t)n * x->h + ih) * x->w + iw) * cin_a;
        const int tap = (r + off) * kmax + (s + off);
        if (T->depthwise) {
          for (int co = 0; co < cout_a; ++co)
            yp[co] += xp[co] * T->w[(size_t)co * kk + tap];
        } else {
          for (int co = 0; co < cout_a; ++co) {
            const float* wp = T->w + ((size_t)co * kk + tap) * T->cin;
            float acc = 0.f;
#pragma omp simd reduction(+ : acc)
            for (int ci = 0; ci < cin_a; ++ci) acc += xp[ci] * wp[ci];
            yp[co] += acc;
          }
        }
      }
    }
  }
  return y;
}

/* SubnetNorm: inference with (mu_ij, var_ij), or calibration with batch
 * statistics (recorded in execution order). */
static void subnet_norm(Ctx* c, T4* y, const ONorm* N) {
  const int C = y->c;
  const int norm_idx = c->active_norms++;
  const size_t base = c->stat_cursor;
  c->stat_cursor += (size_t)C;
  if (c->count_only) return;
  const size_t npix = (size_t)y->n * y->h * y->w;
  float* mean = (float*)malloc(sizeof(float) * C);
  float* var = (float*)malloc(sizeof(float) * C);
  if (c->calibrate) {
    double* s1 = (double*)calloc(C, sizeof(double));
    double* s2 = (double*)calloc(C, sizeof(double));
    for (size_t p = 0; p < npix; ++p)
      for (int ch = 0; ch < C; ++ch) s1[ch] += y->d[p * C + ch];
    for (int ch = 0; ch < C; ++ch) s1[ch] /= (double)npix;
    for (size_t p = 0; p < npix; ++p)
      for (int ch = 0; ch < C; ++ch) {
        const double d = y->d[p * C + ch] - s1[ch];
        s2[ch] += d * d;
      }
    for (int ch = 0; ch < C; ++ch) {
      mean[ch] = (float)s1[ch];
      var[ch] = (float)(s2[ch] / (double)npix);
      if (c->mean_out) c->mean_out[base + ch] = mean[ch];
      if (c->var_out) c->var_out[base + ch] = var[ch];
    }
    free(s1);
    free(s2);
  } else {
    for (int ch = 0; ch < C; ++ch) {
      mean[ch] = c->mean_in ? c->mean_in[base + ch]
                            : ssn_stat_mean_value(c->o->seed, c->subnet_id, norm_idx, ch);
      var[ch] = c->var_in ? c->var_in[base + ch]
                          : ssn_stat_var_value(c->o->seed, c->subnet_id, norm_idx, ch);
    }
  }
#pragma omp parallel for schedule(static)
  for (long p = 0; p < (long)npix; ++p)
    for (int ch = 0; ch < C; ++ch) {
      float* v = &y->d[(size_t)p * C + ch];
      *v = N->gamma[ch] * (*v - mean[ch]) / sqrtf(var[ch] + OR_EPS) + N->beta[ch];
    }
  free(mean);
  free(var);
}

static void relu_(T4* y) {
  const size_t n = t4_size(y);
  for (size_t i = 0; i < n; ++i) y->d[i] = y->d[i] > 0.f ? y->d[i] : 0.f;
}

/* act: 1 = ReLU, 2 = h_swish(x) = x * relu6(x + 3) / 6 (OFA MyNetwork) */
static void act_(T4* y, int act) {
  const size_t n = t4_size(y);
  for (size_t i = 0; i < n; ++i) {
    const float v = y->d[i];
    if (act == 1) y->d[i] = v > 0.f ? v : 0.f;
    else if (act == 2) y->d[i] = v * fminf(fmaxf(v + 3.f, 0.f), 6.f) / 6.f;
  }
}

static void add_(T4* y, const T4* r) {
  const size_t n = t4_size(y);
  for (size_t i = 0; i < n; ++i) y->d[i] += r->d[i];
}

/* conv -> SubnetNorm -> (+res) -> (relu), stored once (bf16 if emulated) */
static T4 conv_bn(Ctx* c, const T4* x, int tensor, int norm, int k_a, int stride,
                  int cout_a, const T4* res, int relu, int res_post) {
  T4 y;
  if (c->count_only) {
    y = t4_new(x->n, 1, 1, cout_a); /* shapes irrelevant when counting */
    y.h = x->h; y.w = x->w;
    subnet_norm(c, &y, &c->o->nm[norm]);
    return y;
  }
  y = conv2d(x, &c->o->t[tensor], k_a, stride, cout_a);
  subnet_norm(c, &y, &c->o->nm[norm]);
  if (res && !res_post) add_(&y, res);
  if (relu) act_(&y, relu); /* `relu` carries the activation code */
  if (res && res_post) add_(&y, res);
  store_round(c, &y);
  return y;
}

static T4 maxpool3s2(Ctx* c, const T4* x) {
  const int ho = (x->h + 2 - 3) / 2 + 1, wo = (x->w + 2 - 3) / 2 + 1;
  T4 y = t4_new(x->n, ho, wo, x->c);
  for (int n = 0; n < x->n; ++n)
    for (int oh = 0; oh < ho; ++oh)
      for (int ow = 0; ow < wo; ++ow)
        for (int ch = 0; ch < x->c; ++ch) {
          float m = -INFINITY;
          for (int r = 0; r < 3; ++r)
            for (int s = 0; s < 3; ++s) {
              const int ih = oh * 2 - 1 + r, iw = ow * 2 - 1 + s;
              if (ih < 0 || iw < 0 || ih >= x->h || iw >= x->w) continue;
              const float v = x->d[(((size_t)n * x->h + ih) * x->w + iw) * x->c + ch];
              m = v > m ? v : m;
            }
          y.d[(((size_t)n * ho + oh) * wo + ow) * x->c + ch] = m;
        }
  store_round(c, &y);
  return y;
}

/* AvgPool2d(kernel=s, stride=s, padding=0, ceil_mode=True): the divisor is
 * the number of in-bounds elements of the window. */
static T4 avgpool_ceil(Ctx* c, const T4* x, int s) {
  const int ho = (x->h + s - 1) / s, wo = (x->w + s - 1) / s;
  T4 y = t4_new(x->n, ho, wo, x->c);
  for (int n = 0; n < x->n; ++n)
    for (int oh = 0; oh < ho; ++oh)
      for (int ow = 0; ow < wo; ++ow)
        for (int ch = 0; ch < x->c; ++ch) {
          float acc = 0.f;
          int cnt = 0;
          for (int r = 0; r < s; ++r)
            for (int q = 0; q < s; ++q) {
              const int ih = oh * s + r, iw = ow * s + q;
              if (ih >= x->h || iw >= x->w) continue;
              acc += x->d[(((size_t)n * x->h + ih) * x->w + iw) * x->c + ch];
              ++cnt;
            }
          y.d[(((size_t)n * ho + oh) * wo + ow) * x->c + ch] = acc / (float)cnt;
        }
  store_round(c, &y);
  return y;
}

static T4 global_avgpool(Ctx* c, const T4* x) {
  T4 y = t4_new(x->n, 1, 1, x->c);
  const int hw = x->h * x->w;
  for (int n = 0; n < x->n; ++n)
    for (int ch = 0; ch < x->c; ++ch) {
      float acc = 0.f;
      for (int p = 0; p < hw; ++p) acc += x->d[((size_t)n * hw + p) * x->c + ch];
      y.d[(size_t)n * x->c + ch] = acc / (float)hw;
    }
  store_round(c, &y);
  return y;
}

/* classifier: logits = x[:, :cin_a] . W[:, :cin_a]^T + b  (float32 out) */
static void linear_out(const T4* x, const OTensor* T, float* logits) {
  const int cin = x->c;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < x->n; ++n)
    for (int o_ = 0; o_ < T->cout; ++o_) {
      const float* wp = T->w + (size_t)o_ * T->cin;
      float acc = 0.f;
      for (int i = 0; i < cin; ++i) acc += x->d[(size_t)n * cin + i] * wp[i];
      logits[(size_t)n * T->cout + o_] = acc + T->bias[o_];
    }
}

/* input: NCHW float32 -> NHWC, optionally bf16-rounded */
static T4 load_input(Ctx* c, const float* x, int n, int hw) {
  T4 t = t4_new(n, hw, hw, 3);
  for (int b = 0; b < n; ++b)
    for (int ch = 0; ch < 3; ++ch)
      for (int i = 0; i < hw * hw; ++i)
        t.d[((size_t)b * hw * hw + i) * 3 + ch] = x[((size_t)b * 3 + ch) * hw * hw + i];
  store_round(c, &t);
  return t;
}

/* ========================================================================= */
/* Config 1: TinyCNN.                         */
/* D = 5 flags, E = 3 ratios (stage A/B/C), W = 4 multipliers.                */

#define TC_MAX_E 6.0
static const int TC_BASE[4] = {32, 32, 64, 128};

typedef struct {
  int stage;  /* 0 = A, 1 = B, 2 = C */
  int stride;
  int flag;   /* -1 = mandatory */
  int residual;
} TcBlock;
static const TcBlock TC_BLOCKS[8] = {
    {0, 1, -1, 0}, {0, 1, 0, 1}, {0, 1, 1, 1},
    {1, 2, -1, 0}, {1, 1, 2, 1}, {1, 1, 3, 1},
    {2, 2, -1, 0}, {2, 1, 4, 1}};

static void tinycnn_build(oracle_net* o) {
  int cin = TC_BASE[0];
  add_tensor(o, TC_BASE[0], 3, 3, 0, 0); /* stem */
  add_norm(o, TC_BASE[0], 0);
  for (int b = 0; b < 8; ++b) {
    const int cout = TC_BASE[1 + TC_BLOCKS[b].stage];
    const int hid = ssn_make_divisible(ssn_round_half_even(cin * TC_MAX_E), 8);
    add_tensor(o, hid, cin, 1, 0, 0);
    add_norm(o, hid, 0);
    add_tensor(o, hid, hid, 3, 1, 0);
    add_norm(o, hid, 0);
    add_tensor(o, cout, hid, 1, 0, 0);
    add_norm(o, cout, TC_BLOCKS[b].residual);
    cin = cout;
  }
  add_tensor(o, o->classes, TC_BASE[3], 1, 0, 1);
}

static int tinycnn_check(const ssn_subnet_cfg* s) {
  if (s->n_depth != 5 || s->n_expand != 3 || s->n_width != 4)
    FAIL("tinycnn subnet needs 5 depth flags, 3 expand ratios, 4 width multipliers");
  for (int i = 0; i < 3; ++i)
    if (!(s->expand_ratios[i] > 0.0) || s->expand_ratios[i] > TC_MAX_E)
      FAIL("expand ratio must be in (0, %g]", TC_MAX_E);
  for (int i = 0; i < 4; ++i)
    if (!(s->width_multipliers[i] > 0.0) || s->width_multipliers[i] > 1.0)
      FAIL("width multiplier must be in (0,1]");
  return 0;
}

static void tinycnn_forward(Ctx* c, const ssn_subnet_cfg* s, T4* x, float* logits) {
  int C[4];
  for (int i = 0; i < 4; ++i) C[i] = ssn_make_divisible(TC_BASE[i] * s->width_multipliers[i], 8);
  T4 y = conv_bn(c, x, 0, 0, 3, 1, C[0], NULL, 1, 0);
  int t = 1, nrm = 1;
  for (int b = 0; b < 8; ++b) {
    const TcBlock* B = &TC_BLOCKS[b];
    const int t0 = t, n0 = nrm;
    t += 3;
    nrm += 3;
    if (B->flag >= 0 && !s->depth_flags[B->flag]) continue; /* LayerSelect */
    const int cin_a = y.c;
    const int cout_a = C[1 + B->stage];
    const int hid = ssn_make_divisible(ssn_round_half_even(cin_a * s->expand_ratios[B->stage]), 8);
    T4 h1 = conv_bn(c, &y, t0, n0, 1, 1, hid, NULL, 1, 0);
    T4 h2 = conv_bn(c, &h1, t0 + 1, n0 + 1, 3, B->stride, hid, NULL, 1, 0);
    T4 out = conv_bn(c, &h2, t0 + 2, n0 + 2, 1, 1, cout_a, B->residual ? &y : NULL, 0, 0);
    t4_free(&h1);
    t4_free(&h2);
    t4_free(&y);
    y = out;
  }
  if (!c->count_only) {
    T4 g = global_avgpool(c, &y);
    linear_out(&g, &c->o->t[t], logits);
    t4_free(&g);
  }
  t4_free(&y);
}

/* ========================================================================= */
/* Config 2: OFA-ResNet50 ([external] OFA ofa_resnets.py).     */
/* D = 9 per-block LayerSelect flags [stem_res, s1b2, s1b3, s2b2, s2b3,        */
/*     s3b4, s3b5, s4b2, s4b3]; E = 18 per-block ratios; W = 6 multipliers.    */

static const int R50_STAGE_W[4] = {256, 512, 1024, 2048};
static const int R50_BASE_DEPTH[4] = {2, 2, 4, 2};
static const int R50_NBLK[4] = {4, 4, 6, 4};
#define R50_MAX_E 0.35

static int r50_mid_max(int stage) {
  return ssn_make_divisible(ssn_round_half_even(R50_STAGE_W[stage] * R50_MAX_E), 8);
}

static void r50_build(oracle_net* o) {
  add_tensor(o, 32, 3, 3, 0, 0);  /* stem conv0 */
  add_norm(o, 32, 0);
  add_tensor(o, 32, 32, 3, 0, 0); /* stem residual conv */
  add_norm(o, 32, 1);
  add_tensor(o, 64, 32, 3, 0, 0); /* stem conv2 */
  add_norm(o, 64, 0);
  int cin = 64;
  for (int s = 0; s < 4; ++s) {
    const int out = R50_STAGE_W[s], mid = r50_mid_max(s);
    for (int b = 0; b < R50_NBLK[s]; ++b) {
      if (b == 0) {
        add_tensor(o, out, cin, 1, 0, 0); /* downsample conv */
        add_norm(o, out, 0);
      }
      add_tensor(o, mid, cin, 1, 0, 0);
      add_norm(o, mid, 0);
      add_tensor(o, mid, mid, 3, 0, 0);
      add_norm(o, mid, 0);
      add_tensor(o, out, mid, 1, 0, 0);
      add_norm(o, out, 1);
      cin = out;
    }
  }
  add_tensor(o, o->classes, 2048, 1, 0, 1);
}

static int r50_check(const ssn_subnet_cfg* s) {
  if (s->n_depth != 9 || s->n_expand != 18 || s->n_width != 6)
    FAIL("ofa_resnet50 subnet needs 9 depth flags, 18 expand ratios, 6 width multipliers");
  for (int i = 0; i < 6; ++i)
    if (!(s->width_multipliers[i] > 0.0) || s->width_multipliers[i] > 1.0)
      FAIL("width multiplier must be in (0,1]");
  int blk = 0;
  for (int st = 0; st < 4; ++st)
    for (int b = 0; b < R50_NBLK[st]; ++b, ++blk) {
      const double e = s->expand_ratios[blk];
      if (!(e > 0.0)) FAIL("expand ratio must be > 0");
      const int out_a = ssn_make_divisible(R50_STAGE_W[st] * s->width_multipliers[2 + st], 8);
      const int mid = ssn_make_divisible(ssn_round_half_even(out_a * e), 8);
      if (mid > r50_mid_max(st)) FAIL("expand ratio %g exceeds the supernet's max middle width", e);
    }
  return 0;
}

static void r50_forward(Ctx* c, const ssn_subnet_cfg* s, T4* x, float* logits) {
  const double* W = s->width_multipliers;
  const int stem_out = ssn_make_divisible(64 * W[1], 8);
  const int stem_mid = ssn_make_divisible(ssn_make_divisible(64 * W[0], 8) / 2, 8);
  T4 y = conv_bn(c, x, 0, 0, 3, 2, stem_mid, NULL, 1, 0);
  if (s->depth_flags[0]) { /* stem ResidualBlock: y + relu(bn(conv(y))) */
    T4 r = conv_bn(c, &y, 1, 1, 3, 1, stem_mid, c->count_only ? NULL : &y, 1, 1);
    t4_free(&y);
    y = r;
  }
  {
    T4 z = conv_bn(c, &y, 2, 2, 3, 1, stem_out, NULL, 1, 0);
    t4_free(&y);
    y = z;
  }
  if (!c->count_only) {
    T4 z = maxpool3s2(c, &y);
    t4_free(&y);
    y = z;
  }
  int t = 3, nrm = 3, blk = 0;
  for (int st = 0; st < 4; ++st) {
    const int out_a = ssn_make_divisible(R50_STAGE_W[st] * W[2 + st], 8);
    const int stride = st == 0 ? 1 : 2;
    for (int b = 0; b < R50_NBLK[st]; ++b, ++blk) {
      const int has_ds = b == 0;
      const int t0 = t, n0 = nrm;
      t += has_ds ? 4 : 3;
      nrm += has_ds ? 4 : 3;
      if (b >= R50_BASE_DEPTH[st]) {
        const int flag = 1 + 2 * st + (b - R50_BASE_DEPTH[st]);
        if (!s->depth_flags[flag]) continue; /* LayerSelect */
      }
      const int mid = ssn_make_divisible(ssn_round_half_even(out_a * s->expand_ratios[blk]), 8);
      T4 res;
      int tc = t0, nc = n0;
      if (has_ds) {
        if (stride > 1 && !c->count_only) {
          T4 p = avgpool_ceil(c, &y, stride);
          res = conv_bn(c, &p, tc, nc, 1, 1, out_a, NULL, 0, 0);
          t4_free(&p);
        } else {
          res = conv_bn(c, &y, tc, nc, 1, 1, out_a, NULL, 0, 0);
        }
        ++tc;
        ++nc;
      } else {
        res = y; /* identity */
      }
      T4 h1 = conv_bn(c, &y, tc, nc, 1, 1, mid, NULL, 1, 0);
      T4 h2 = conv_bn(c, &h1, tc + 1, nc + 1, 3, b == 0 ? stride : 1, mid, NULL, 1, 0);
      T4 out = conv_bn(c, &h2, tc + 2, nc + 2, 1, 1, out_a, c->count_only ? NULL : &res, 1, 0);
      t4_free(&h1);
      t4_free(&h2);
      if (has_ds) t4_free(&res);
      t4_free(&y);
      y = out;
    }
  }
  if (!c->count_only) {
    T4 g = global_avgpool(c, &y);
    linear_out(&g, &c->o->t[t], logits);
    t4_free(&g);
  }
  t4_free(&y);
}

/* ========================================================================= */
/* Config 3: OFA-MobileNetV3 w1.2 ([external] OFA             */
/* OFAMobileNetV3 / DynamicMBConvLayer / DynamicSE).                           */
/* D = 10 flags (blocks 3, 4 of each stage), E = 20, W = [1.0], K = 20.        */

static const int MB_W[5] = {32, 48, 96, 136, 192};
static const int MB_S[5] = {2, 2, 2, 1, 2};
static const int MB_A[5] = {1, 1, 2, 2, 2};
static const int MB_SE[5] = {0, 1, 0, 1, 1};

static void mbv3_build(oracle_net* o) {
  add_tensor(o, 24, 3, 3, 0, 0); /* first conv */
  add_norm(o, 24, 0);
  add_tensor(o, 24, 24, 3, 1, 0); /* first block depthwise */
  add_norm(o, 24, 0);
  add_tensor(o, 24, 24, 1, 0, 0); /* first block point */
  add_norm(o, 24, 1);
  int cin = 24;
  for (int st = 0; st < 5; ++st)
    for (int b = 0; b < 4; ++b) {
      const int cout = MB_W[st], stride = b == 0 ? MB_S[st] : 1;
      const int res = stride == 1 && cin == cout;
      const int mid = ssn_make_divisible(ssn_round_half_even(cin * 6.0), 8);
      add_tensor(o, mid, cin, 1, 0, 0);
      add_norm(o, mid, 0);
      add_tensor(o, mid, mid, 7, 1, 0);
      add_norm(o, mid, 0);
      if (MB_SE[st]) {
        const int se = ssn_make_divisible(mid / 4, 8);
        add_tensor(o, se, mid, 1, 0, 1);
        add_tensor(o, mid, se, 1, 0, 1);
      }
      add_tensor(o, cout, mid, 1, 0, 0);
      add_norm(o, cout, res);
      cin = cout;
    }
  add_tensor(o, 1152, 192, 1, 0, 0);
  add_norm(o, 1152, 0);
  add_tensor(o, 1536, 1152, 1, 0, 0); /* feature mix: no norm, no bias */
  add_tensor(o, o->classes, 1536, 1, 0, 1);
}

static int mbv3_check(const ssn_subnet_cfg* s) {
  if (s->n_depth != 10 || s->n_expand != 20 || s->n_width != 1)
    FAIL("ofa_mbv3 subnet needs 10 depth flags, 20 expand ratios, 1 width multiplier");
  if (s->n_kernel != 0 && s->n_kernel != 20) FAIL("ofa_mbv3 subnet needs 20 kernel sizes (or none)");
  if (s->width_multipliers[0] != 1.0)
    FAIL("ofa_mbv3 supernet has a fixed width: width multiplier must be 1.0");
  for (int i = 0; i < 20; ++i) {
    if (!(s->expand_ratios[i] > 0.0) || s->expand_ratios[i] > 6.0)
      FAIL("expand ratio must be in (0, 6]");
    if (s->n_kernel) {
      const uint32_t k = s->kernel_sizes[i];
      if (k != 3 && k != 5 && k != 7) FAIL("kernel size must be 3, 5 or 7");
    }
  }
  return 0;
}

/* 1x1 conv without norm (feature mix): y = act(x . W^T), bf16 storage */
static T4 conv_act(Ctx* c, const T4* x, int tensor, int cout, int act) {
  T4 y = conv2d(x, &c->o->t[tensor], 1, 1, cout);
  act_(&y, act);
  store_round(c, &y);
  return y;
}

/* DynamicSE: x *= h_sigmoid(We[:C,:m] relu(Wr[:m,:C] mean_hw(x) + br) + be) */
static void se_(Ctx* c, T4* x, int tr, int te) {
  const OTensor* R = &c->o->t[tr];
  const OTensor* E = &c->o->t[te];
  const int C = x->c, m = ssn_make_divisible(C / 4, 8), hw = x->h * x->w;
  float* pooled = (float*)calloc(C, sizeof(float));
  float* hid = (float*)calloc(m, sizeof(float));
  float* gate = (float*)calloc(C, sizeof(float));
  for (int n = 0; n < x->n; ++n) {
    for (int ch = 0; ch < C; ++ch) {
      double s = 0.0;
      for (int p = 0; p < hw; ++p) s += x->d[((size_t)n * hw + p) * C + ch];
      pooled[ch] = (float)(s / hw);
    }
    for (int j = 0; j < m; ++j) {
      float s = R->bias[j];
      for (int ch = 0; ch < C; ++ch) s += R->w[(size_t)j * R->cin + ch] * pooled[ch];
      hid[j] = s > 0.f ? s : 0.f;
    }
    for (int ch = 0; ch < C; ++ch) {
      float s = E->bias[ch];
      for (int j = 0; j < m; ++j) s += E->w[(size_t)ch * E->cin + j] * hid[j];
      gate[ch] = fminf(fmaxf(s + 3.f, 0.f), 6.f) / 6.f;
    }
    for (int p = 0; p < hw; ++p)
      for (int ch = 0; ch < C; ++ch) x->d[((size_t)n * hw + p) * C + ch] *= gate[ch];
  }
  free(pooled);
  free(hid);
  free(gate);
  store_round(c, x);
}

static void mbv3_forward(Ctx* c, const ssn_subnet_cfg* s, T4* x, float* logits) {
  T4 y = conv_bn(c, x, 0, 0, 3, 2, 24, NULL, 2, 0);
  {
    T4 h = conv_bn(c, &y, 1, 1, 3, 1, 24, NULL, 1, 0);
    T4 z = conv_bn(c, &h, 2, 2, 1, 1, 24, c->count_only ? NULL : &y, 0, 0);
    t4_free(&h);
    t4_free(&y);
    y = z;
  }
  int t = 3, nrm = 3, blk = 0, cin_max = 24;
  for (int st = 0; st < 5; ++st)
    for (int b = 0; b < 4; ++b, ++blk) {
      const int cout = MB_W[st], stride = b == 0 ? MB_S[st] : 1;
      const int res = stride == 1 && cin_max == cout;
      const int t0 = t, n0 = nrm;
      t += MB_SE[st] ? 5 : 3;
      nrm += 3;
      cin_max = cout;
      if (b >= 2 && !s->depth_flags[2 * st + (b - 2)]) continue; /* LayerSelect */
      const int mid = ssn_make_divisible(ssn_round_half_even(y.c * s->expand_ratios[blk]), 8);
      const int ka = s->n_kernel ? (int)s->kernel_sizes[blk] : 7;
      T4 h1 = conv_bn(c, &y, t0, n0, 1, 1, mid, NULL, MB_A[st], 0);
      T4 h2 = conv_bn(c, &h1, t0 + 1, n0 + 1, ka, stride, mid, NULL, MB_A[st], 0);
      t4_free(&h1);
      int tp = t0 + 2;
      if (MB_SE[st]) {
        if (!c->count_only) se_(c, &h2, t0 + 2, t0 + 3);
        tp = t0 + 4;
      }
      T4 out = conv_bn(c, &h2, tp, n0 + 2, 1, 1, cout, (res && !c->count_only) ? &y : NULL, 0, 0);
      t4_free(&h2);
      t4_free(&y);
      y = out;
    }
  T4 f = conv_bn(c, &y, t, nrm, 1, 1, 1152, NULL, 2, 0);
  t4_free(&y);
  if (!c->count_only) {
    T4 g = global_avgpool(c, &f);
    T4 m = conv_act(c, &g, t + 1, 1536, 2);
    linear_out(&m, &c->o->t[t + 2], logits);
    t4_free(&g);
    t4_free(&m);
  }
  t4_free(&f);
}

/* ========================================================================= */
/* Config 5: width/depth-sliced BERT-base-like encoder (DESIGN.md §3.4,       */
/* [external] DynaBERT).  D = 12 layer flags, E = [FFN width], W = [heads].   */

#define BT_HID 768
#define BT_FFN 3072
#define BT_L 12
#define BT_VOCAB 30522

static void bert_build(oracle_net* o) {
  add_tensor(o, BT_VOCAB, BT_HID, 1, 0, 0); /* token embeddings */
  add_tensor(o, 512, BT_HID, 1, 0, 0);      /* positions */
  add_tensor(o, 2, BT_HID, 1, 0, 0);        /* token types */
  add_norm(o, BT_HID, 0);
  for (int l = 0; l < BT_L; ++l) {
    for (int q = 0; q < 4; ++q) add_tensor(o, BT_HID, BT_HID, 1, 0, 1); /* Q K V O */
    add_norm(o, BT_HID, 0);
    add_tensor(o, BT_FFN, BT_HID, 1, 0, 1);
    add_tensor(o, BT_HID, BT_FFN, 1, 0, 1);
    add_norm(o, BT_HID, 0);
  }
  add_tensor(o, BT_HID, BT_HID, 1, 0, 1);       /* pooler */
  add_tensor(o, o->classes, BT_HID, 1, 0, 1);   /* classifier */
}

static int bert_check(const ssn_subnet_cfg* s) {
  if (s->n_depth != BT_L || s->n_expand != 1 || s->n_width != 1)
    FAIL("bert subnet needs 12 depth flags, 1 FFN width (expand) ratio, 1 head width multiplier");
  if (!(s->width_multipliers[0] > 0.0) || s->width_multipliers[0] > 1.0)
    FAIL("width multiplier must be in (0,1]");
  if (!(s->expand_ratios[0] > 0.0) || s->expand_ratios[0] > 1.0)
    FAIL("FFN expand ratio must be in (0,1]");
  return 0;
}

/* y[t][:cout] = x[t][:cin] . W[:cout][:cin]^T + b[:cout] (+ act), rows x cols */
static float* linear_(const float* x, int rows, int cin, const OTensor* T, int cout, int act,
                      int acc64) {
  float* y = (float*)malloc(sizeof(float) * (size_t)rows * cout);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int co = 0; co < cout; ++co) {
      const float* wp = T->w + (size_t)co * T->cin;
      const float* xp = x + (size_t)r * cin;
      float acc = 0.f;
      if (acc64) {
        double a = 0.0;
        for (int i = 0; i < cin; ++i) a += (double)xp[i] * wp[i];
        acc = (float)a;
      } else {
#pragma omp simd reduction(+ : acc)
        for (int i = 0; i < cin; ++i) acc += xp[i] * wp[i];
      }
      float v = acc + T->bias[co];
      if (act == 3) v = 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
      if (act == 4) v = tanhf(v);
      y[(size_t)r * cout + co] = v;
    }
  return y;
}

static void round_buf(Ctx* c, float* v, size_t n) {
  if (!c->emulate_bf16) return;
  for (size_t i = 0; i < n; ++i) v[i] = ssn_round_bf16(v[i]);
}

/* LayerNorm (eps 1e-12, BERT) over rows of BT_HID, in place */
static void layernorm_(float* x, int rows, const ONorm* N) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    float* v = x + (size_t)r * BT_HID;
    double m = 0.0, q = 0.0;
    for (int i = 0; i < BT_HID; ++i) m += v[i];
    m /= BT_HID;
    for (int i = 0; i < BT_HID; ++i) q += (v[i] - m) * (v[i] - m);
    const float inv = 1.f / sqrtf((float)(q / BT_HID) + 1e-12f);
    for (int i = 0; i < BT_HID; ++i) v[i] = (float)((v[i] - m) * inv) * N->gamma[i] + N->beta[i];
  }
}

static void bert_forward(Ctx* c, const ssn_subnet_cfg* s, const int* ids, int n, int S,
                         float* logits) {
  const oracle_net* o = c->o;
  const int heads = ssn_round_half_even(12 * s->width_multipliers[0]) < 1
                        ? 1
                        : ssn_round_half_even(12 * s->width_multipliers[0]);
  int ffn = ssn_make_divisible(BT_FFN * s->expand_ratios[0], 8);
  if (ffn > BT_FFN) ffn = BT_FFN;
  const int Ca = heads * 64, T = n * S;
  float* X = (float*)malloc(sizeof(float) * (size_t)T * BT_HID);
  for (int t = 0; t < T; ++t) {
    int id = ids[t];
    if (id < 0) id = 0;
    if (id >= BT_VOCAB) id = BT_VOCAB - 1;
    for (int i = 0; i < BT_HID; ++i)
      X[(size_t)t * BT_HID + i] = o->t[0].w[(size_t)id * BT_HID + i] +
                                  o->t[1].w[(size_t)(t % S) * BT_HID + i] + o->t[2].w[i];
  }
  layernorm_(X, T, &o->nm[0]);
  round_buf(c, X, (size_t)T * BT_HID);
  for (int l = 0; l < BT_L; ++l) {
    if (!s->depth_flags[l]) continue; /* LayerSelect */
    const int tb = 3 + 6 * l;
    float* Q = linear_(X, T, BT_HID, &o->t[tb], Ca, 0, c->acc64);
    float* K = linear_(X, T, BT_HID, &o->t[tb + 1], Ca, 0, c->acc64);
    float* V = linear_(X, T, BT_HID, &o->t[tb + 2], Ca, 0, c->acc64);
    round_buf(c, Q, (size_t)T * Ca);
    round_buf(c, K, (size_t)T * Ca);
    round_buf(c, V, (size_t)T * Ca);
    float* ctx = (float*)calloc((size_t)T * Ca, sizeof(float));
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < n; ++b)
      for (int h = 0; h < heads; ++h) {
        float* sc = (float*)malloc(sizeof(float) * S);
        for (int i = 0; i < S; ++i) {
          const float* qi = Q + ((size_t)b * S + i) * Ca + h * 64;
          float mx = -INFINITY;
          for (int j = 0; j < S; ++j) {
            const float* kj = K + ((size_t)b * S + j) * Ca + h * 64;
            float d = 0.f;
            for (int e = 0; e < 64; ++e) d += qi[e] * kj[e];
            sc[j] = d * 0.125f;
            mx = sc[j] > mx ? sc[j] : mx;
          }
          double sum = 0.0;
          for (int j = 0; j < S; ++j) {
            sc[j] = expf(sc[j] - mx);
            sum += sc[j];
          }
          float* out = ctx + ((size_t)b * S + i) * Ca + h * 64;
          if (c->emulate_bf16) {
            /* engine storage: the UNNORMALISED probabilities exp(s - max) are
             * the bf16 A operand of the P.V product; the row sum (fp32, from
             * the unrounded values) divides the fp32 accumulator afterwards */
            for (int j = 0; j < S; ++j) {
              const float pj = ssn_round_bf16(sc[j]);
              const float* vj = V + ((size_t)b * S + j) * Ca + h * 64;
              for (int e = 0; e < 64; ++e) out[e] += pj * vj[e];
            }
            const float inv = (float)(1.0 / sum);
            for (int e = 0; e < 64; ++e) out[e] *= inv;
          } else {
            for (int j = 0; j < S; ++j) {
              const float pj = (float)(sc[j] / sum);
              const float* vj = V + ((size_t)b * S + j) * Ca + h * 64;
              for (int e = 0; e < 64; ++e) out[e] += pj * vj[e];
            }
          }
        }
        free(sc);
      }
    round_buf(c, ctx, (size_t)T * Ca);
    float* O = linear_(ctx, T, Ca, &o->t[tb + 3], BT_HID, 0, c->acc64);
    for (size_t i = 0; i < (size_t)T * BT_HID; ++i) O[i] += X[i];
    round_buf(c, O, (size_t)T * BT_HID);
    layernorm_(O, T, &o->nm[1 + 2 * l]);
    round_buf(c, O, (size_t)T * BT_HID);
    float* F = linear_(O, T, BT_HID, &o->t[tb + 4], ffn, 3, c->acc64);
    round_buf(c, F, (size_t)T * ffn);
    float* Y = linear_(F, T, ffn, &o->t[tb + 5], BT_HID, 0, c->acc64);
    for (size_t i = 0; i < (size_t)T * BT_HID; ++i) Y[i] += O[i];
    round_buf(c, Y, (size_t)T * BT_HID);
    layernorm_(Y, T, &o->nm[2 + 2 * l]);
    round_buf(c, Y, (size_t)T * BT_HID);
    free(Q); free(K); free(V); free(ctx); free(O); free(F); free(X);
    X = Y;
  }
  float* cls = (float*)malloc(sizeof(float) * (size_t)n * BT_HID);
  for (int b = 0; b < n; ++b)
    memcpy(cls + (size_t)b * BT_HID, X + (size_t)b * S * BT_HID, sizeof(float) * BT_HID);
  float* P = linear_(cls, n, BT_HID, &o->t[3 + 6 * BT_L], BT_HID, 4, c->acc64);
  round_buf(c, P, (size_t)n * BT_HID);
  float* L = linear_(P, n, BT_HID, &o->t[4 + 6 * BT_L], o->classes, 0, c->acc64);
  memcpy(logits, L, sizeof(float) * (size_t)n * o->classes);
  free(cls); free(P); free(L); free(X);
}

/* Synthetic token ids (ssn_rng.h kind 8): floor(u01 * vocab). */
void oracle_tokens(uint64_t seed, uint32_t batch_ordinal, int n, int s, int* out) {
  for (long i = 0; i < (long)n * s; ++i)
    out[i] = (int)(ssn_u01(seed, ssn_stream(SSN_STREAM_TOKENS, batch_ordinal), i) * BT_VOCAB);
}

/* ========================================================================= */
/* public oracle API (ctypes)                                                 */

oracle_net* oracle_create(int family, uint64_t seed, int classes, int bf16_weights) {
  oracle_net* o = (oracle_net*)calloc(1, sizeof(oracle_net));
  o->family = family;
  o->seed = seed;
  o->classes = classes;
  o->bf16_w = bf16_weights;
  if (family == SSN_FAMILY_TINYCNN) {
    tinycnn_build(o);
  } else if (family == SSN_FAMILY_OFA_RESNET50) {
    r50_build(o);
  } else if (family == SSN_FAMILY_OFA_MBV3) {
    mbv3_build(o);
  } else if (family == SSN_FAMILY_BERT) {
    bert_build(o);
  } else {
    snprintf(g_err, sizeof g_err, "oracle: unsupported family %d", family);
    free(o);
    return NULL;
  }
  return o;
}

void oracle_destroy(oracle_net* o) {
  if (!o) return;
  for (int i = 0; i < o->nt; ++i) {
    free(o->t[i].w);
    free(o->t[i].bias);
  }
  for (int i = 0; i < o->nn; ++i) {
    free(o->nm[i].gamma);
    free(o->nm[i].beta);
  }
  free(o);
}

int oracle_num_tensors(const oracle_net* o) { return o->nt; }

/* weight value in canonical OIHW order (tests compare the engine blob) */
float oracle_weight(const oracle_net* o, int tensor, int co, int ci, int r, int s) {
  const OTensor* T = &o->t[tensor];
  return T->w[((size_t)co * T->k * T->k + r * T->k + s) * T->cin + ci];
}

static int check_cfg(const oracle_net* o, const ssn_subnet_cfg* s) {
  if (o->family == SSN_FAMILY_TINYCNN) return tinycnn_check(s);
  if (o->family == SSN_FAMILY_OFA_MBV3) return mbv3_check(s);
  if (o->family == SSN_FAMILY_BERT) return bert_check(s);
  return r50_check(s);
}

static void run(Ctx* c, const ssn_subnet_cfg* s, T4* x, float* logits) {
  if (c->o->family == SSN_FAMILY_TINYCNN)
    tinycnn_forward(c, s, x, logits);
  else if (c->o->family == SSN_FAMILY_OFA_MBV3)
    mbv3_forward(c, s, x, logits);
  else
    r50_forward(c, s, x, logits);
}

long oracle_stat_count(oracle_net* o, const ssn_subnet_cfg* s) {
  if (check_cfg(o, s)) return -1;
  if (o->family == SSN_FAMILY_BERT) return 0; /* LayerNorm keeps no statistics */
  Ctx c;
  memset(&c, 0, sizeof c);
  c.o = o;
  c.count_only = 1;
  T4 x = t4_new(1, 1, 1, 3);
  run(&c, s, &x, NULL);
  return (long)c.stat_cursor;
}

/* flags: bit0 = emulate bf16 activation storage; bit1 = calibrate */
int oracle_forward(oracle_net* o, const ssn_subnet_cfg* s, uint32_t subnet_id,
                   const float* x_nchw, int n, int hw, const float* mean,
                   const float* var, int flags, float* logits, float* mean_out,
                   float* var_out) {
  if (check_cfg(o, s)) return -1;
  Ctx c;
  memset(&c, 0, sizeof c);
  c.o = o;
  c.emulate_bf16 = flags & 1;
  c.calibrate = (flags >> 1) & 1;
  c.subnet_id = subnet_id;
  c.mean_in = mean;
  c.var_in = var;
  c.mean_out = mean_out;
  c.var_out = var_out;
  T4 x = load_input(&c, x_nchw, n, hw);
  float* lg = logits ? logits : (float*)malloc(sizeof(float) * (size_t)n * o->classes);
  run(&c, s, &x, lg);
  if (!logits) free(lg);
  return 0;
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Synthetic image batch (ssn_rng.h kind 5), NCHW float32. */
void oracle_images(uint64_t seed, uint32_t batch_ordinal, int n, int hw, float* out) {
  const size_t total = (size_t)n * 3 * hw * hw;
  for (size_t i = 0; i < total; ++i) out[i] = ssn_image_value(seed, batch_ordinal, i);
}

/* Single-operator reference for the op-level tests: WeightSlice conv over a
 * max-shape OIHW float32 tensor + per-channel scale/shift + residual + act.
 * x NHWC [n][h][w][cin]; wgt OIHW [cout_max][cin_max][k_max][k_max]
 * (depthwise: [c_max][1][k_max][k_max]); y NHWC [n][ho][wo][cout]. */
int oracle_conv_op(const float* x, int n, int h, int w, int cin, const float* wgt,
                   int cout_max, int cin_max, int k_max, int k, int stride,
                   int pad, int cout, int depthwise, const float* scale,
                   const float* shift, const float* res, int act, float* y) {
  const int ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  const int off = (k_max - k) / 2;
  const int ci_max = depthwise ? 1 : cin_max;
  const long npix = (long)n * ho * wo;
  (void)cout_max;
#pragma omp parallel for schedule(static)
  for (long p = 0; p < npix; ++p) {
    const int b = (int)(p / ((long)ho * wo));
    const int rem = (int)(p % ((long)ho * wo));
    const int oh = rem / wo, ow = rem % wo;
    for (int co = 0; co < cout; ++co) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r) {
        const int ih = oh * stride - pad + r;
        if (ih < 0 || ih >= h) continue;
        for (int s = 0; s < k; ++s) {
          const int iw = ow * stride - pad + s;
          if (iw < 0 || iw >= w) continue;
          const float* xp = x + (((size_t)b * h + ih) * w + iw) * cin;
          if (depthwise) {
            acc += (double)xp[co] *
                   wgt[(((size_t)co * 1) * k_max + r + off) * k_max + s + off];
          } else {
            for (int ci = 0; ci < cin; ++ci)
              acc += (double)xp[ci] *
                     wgt[(((size_t)co * ci_max + ci) * k_max + r + off) * k_max + s + off];
          }
        }
      }
      float v = (float)acc;
      v = v * (scale ? scale[co] : 1.f) + (shift ? shift[co] : 0.f);
      if (res) v += res[(size_t)p * cout + co];
      if (act == 1) v = v > 0.f ? v : 0.f;
      else if (act == 2) v = v * fminf(fmaxf(v + 3.f, 0.f), 6.f) / 6.f;  /* h_swish (line 271) */
      y[(size_t)p * cout + co] = v;
    }
  }
  return 0;
}

/* BERT forward on token ids [n][s] (flags bit0: bf16 storage emulation) */
int oracle_forward_tokens(oracle_net* o, const ssn_subnet_cfg* s, const int* ids, int n, int seq,
                          int flags, float* logits) {
  if (o->family != SSN_FAMILY_BERT) FAIL("oracle_forward_tokens: not a transformer supernet");
  if (check_cfg(o, s)) return -1;
  Ctx c;
  memset(&c, 0, sizeof c);
  c.o = o;
  c.emulate_bf16 = flags & 1;
  c.acc64 = (flags >> 2) & 1;
  bert_forward(&c, s, ids, n, seq, logits);
  return 0;
}
