// transformer.cu — config-5 (width/depth-sliced BERT) kernels besides the
// tcgen05 WeightSlice linears: embedding + LayerNorm, LayerNorm, [CLS]
// gather, and a fused attention kernel over the ACTIVE heads.
//
// Attention: one CTA per (sequence, active head), 8 warps x 16 query rows
// (s = 128).  K and V^T of the head are staged in padded shared memory; each
// warp computes S = Q K^T / 8 with warp-level mma.sync m16n8k16 (bf16 in,
// fp32 accumulate), does the row softmax on the accumulator registers (rows
// spread over a thread quad), and reuses the probabilities as A fragments of
// O = P V (the FlashAttention-2 register trick).  Attention is ~3% of the
// encoder's FLOPs; the projections/FFN run on tcgen05.
#include "../../include/ssn.h"
#include "device.cuh"

namespace ssn {

__device__ __forceinline__ float bf2f(const __nv_bfloat16 v) { return __bfloat162float(v); }

// ---------------------------------------------------------------- embedding + LN
// one warp per token: x = tok[id] + pos[p] + typ[0]; LayerNorm over hid
__global__ void embed_ln_kernel(EmbedParams p) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int rows = p.n * p.s;
  if (warp >= rows) return;
  const int tpos = warp % p.s;
  int id = p.ids[warp];
  id = id < 0 ? 0 : (id >= p.vocab ? p.vocab - 1 : id);
  const __nv_bfloat16* tk = static_cast<const __nv_bfloat16*>(p.tok) + static_cast<long>(id) * p.hid;
  const __nv_bfloat16* ps = static_cast<const __nv_bfloat16*>(p.pos) + static_cast<long>(tpos) * p.hid;
  const __nv_bfloat16* ty = static_cast<const __nv_bfloat16*>(p.typ);
  float v[32];
  int cnt = 0;
  float sum = 0.f;
  for (int c = lane; c < p.hid; c += 32, ++cnt) {
    v[cnt] = bf2f(tk[c]) + bf2f(ps[c]) + bf2f(ty[c]);
    sum += v[cnt];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / p.hid;
  float var = 0.f;
  for (int i = 0; i < cnt; ++i) var += (v[i] - mean) * (v[i] - mean);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float inv = rsqrtf(var / p.hid + 1e-12f);
  __nv_bfloat16* y = static_cast<__nv_bfloat16*>(p.y) + static_cast<long>(warp) * p.hid;
  cnt = 0;
  for (int c = lane; c < p.hid; c += 32, ++cnt)
    y[c] = __float2bfloat16_rn((v[cnt] - mean) * inv * p.gamma[c] + p.beta[c]);
}

// ---------------------------------------------------------------- LayerNorm
// One warp per row; each lane holds NV 16-byte vectors (8 columns each) of
// the row in registers: hid = 256 * NV (BERT-base: 768 -> NV = 3).  Loads and
// stores are 16-byte and coalesced; gamma/beta as float4 pairs.  (The first
// version read 2-byte scalars into a dynamically indexed local array.)
template <int NV>
__global__ void __launch_bounds__(256) layernorm_kernel(LnParams p) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const uint4* x = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.x) +
                                                  static_cast<long>(warp) * p.hid);
  float v[NV][8];
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const uint4 u = __ldg(x + j * 32 + lane);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      v[j][2 * q] = f.x;
      v[j][2 * q + 1] = f.y;
      sum += f.x + f.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / p.hid;
  float var = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int q = 0; q < 8; ++q) var += (v[j][q] - mean) * (v[j][q] - mean);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float inv = rsqrtf(var / p.hid + 1e-12f);
  uint4* y = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + static_cast<long>(warp) * p.hid);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * 32 + lane) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.gamma + c));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.gamma + c + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.beta + c));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.beta + c + 4));
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = (v[j][q] - mean) * inv * g[q] + bb[q];
    uint4 u;
    u.x = pack_bf16x2(o[0], o[1]);
    u.y = pack_bf16x2(o[2], o[3]);
    u.z = pack_bf16x2(o[4], o[5]);
    u.w = pack_bf16x2(o[6], o[7]);
    y[j * 32 + lane] = u;
  }
}

// ---------------------------------------------------------------- token 0
__global__ void token0_kernel(Token0Params p) {
  pdl_wait();
  pdl_trigger();
  const long total = static_cast<long>(p.n) * (p.c / 8);
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long b = i / (p.c / 8);
    const int g = static_cast<int>(i - b * (p.c / 8));
    reinterpret_cast<uint4*>(p.y)[b * (p.c / 8) + g] =
        reinterpret_cast<const uint4*>(p.x)[b * p.s * (p.c / 8) + g];
  }
}

// ---------------------------------------------------------------- attention
constexpr int ATT_S = 128, ATT_D = 64;
constexpr int ATT_KLD = ATT_D + 8;   // K row stride (bf16), conflict-free fragment loads
constexpr int ATT_VLD = ATT_S + 8;   // V^T row stride

__global__ void __launch_bounds__(256) attention_kernel(AttnParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int heads = d.cin / ATT_D;
  if (static_cast<int>(blockIdx.x) >= p.n * heads) return;  // head beyond the active width
  const int b = blockIdx.x / heads, h = blockIdx.x - (blockIdx.x / heads) * heads;
  const int C = d.cin;
  __shared__ __align__(16) __nv_bfloat16 Ks[ATT_S * ATT_KLD];
  __shared__ __align__(16) __nv_bfloat16 Vt[ATT_D * ATT_VLD];
  const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(p.q);
  const __nv_bfloat16* k = static_cast<const __nv_bfloat16*>(p.k);
  const __nv_bfloat16* v = static_cast<const __nv_bfloat16*>(p.v);
  const long base = static_cast<long>(b) * p.s * C + h * ATT_D;
  // stage K [key][dim] and V^T [dim][key]
  for (int i = threadIdx.x; i < ATT_S * ATT_D / 8; i += blockDim.x) {
    const int key = i / (ATT_D / 8), c8 = (i - key * (ATT_D / 8)) * 8;
    const uint4 kv = *reinterpret_cast<const uint4*>(k + base + static_cast<long>(key) * C + c8);
    *reinterpret_cast<uint4*>(&Ks[key * ATT_KLD + c8]) = kv;
    const uint4 vv = *reinterpret_cast<const uint4*>(v + base + static_cast<long>(key) * C + c8);
    const __nv_bfloat16* ve = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
    for (int e = 0; e < 8; ++e) Vt[(c8 + e) * ATT_VLD + key] = ve[e];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int q0 = warp * 16;  // this warp's query rows
  // Q fragments for the 4 k-steps of the head dim
  uint32_t qa[4][4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const __nv_bfloat16* r0 = q + base + static_cast<long>(q0 + g) * C + ks * 16 + 2 * t;
    const __nv_bfloat16* r1 = r0 + 8L * C;
    qa[ks][0] = *reinterpret_cast<const uint32_t*>(r0);
    qa[ks][1] = *reinterpret_cast<const uint32_t*>(r1);
    qa[ks][2] = *reinterpret_cast<const uint32_t*>(r0 + 8);
    qa[ks][3] = *reinterpret_cast<const uint32_t*>(r1 + 8);
  }
  // S = Q K^T: 16 key tiles of 8
  float sc[ATT_S / 8][4];
#pragma unroll
  for (int nt = 0; nt < ATT_S / 8; ++nt) {
    sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const __nv_bfloat16* kr = &Ks[(nt * 8 + g) * ATT_KLD + ks * 16 + 2 * t];
      mma_bf16_16816(sc[nt], qa[ks], *reinterpret_cast<const uint32_t*>(kr),
                     *reinterpret_cast<const uint32_t*>(kr + 8));
    }
  }
  // softmax over keys for rows g (c0,c1) and g+8 (c2,c3); a row spans a quad
  const float scale = 0.125f;  // 1/sqrt(64)
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < ATT_S / 8; ++nt) {
    m0 = fmaxf(m0, fmaxf(sc[nt][0], sc[nt][1]));
    m1 = fmaxf(m1, fmaxf(sc[nt][2], sc[nt][3]));
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
  }
  float l0 = 0.f, l1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < ATT_S / 8; ++nt) {
    sc[nt][0] = __expf((sc[nt][0] - m0) * scale);
    sc[nt][1] = __expf((sc[nt][1] - m0) * scale);
    sc[nt][2] = __expf((sc[nt][2] - m1) * scale);
    sc[nt][3] = __expf((sc[nt][3] - m1) * scale);
    l0 += sc[nt][0] + sc[nt][1];
    l1 += sc[nt][2] + sc[nt][3];
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  }
  // O = P V: P fragments come straight from the score accumulators
  float oacc[ATT_D / 8][4];
#pragma unroll
  for (int dt = 0; dt < ATT_D / 8; ++dt) oacc[dt][0] = oacc[dt][1] = oacc[dt][2] = oacc[dt][3] = 0.f;
#pragma unroll
  for (int kj = 0; kj < ATT_S / 16; ++kj) {
    uint32_t pa[4];
    pa[0] = pack_bf16x2(sc[2 * kj][0], sc[2 * kj][1]);
    pa[1] = pack_bf16x2(sc[2 * kj][2], sc[2 * kj][3]);
    pa[2] = pack_bf16x2(sc[2 * kj + 1][0], sc[2 * kj + 1][1]);
    pa[3] = pack_bf16x2(sc[2 * kj + 1][2], sc[2 * kj + 1][3]);
#pragma unroll
    for (int dt = 0; dt < ATT_D / 8; ++dt) {
      const __nv_bfloat16* vr = &Vt[(dt * 8 + g) * ATT_VLD + kj * 16 + 2 * t];
      mma_bf16_16816(oacc[dt], pa, *reinterpret_cast<const uint32_t*>(vr),
                     *reinterpret_cast<const uint32_t*>(vr + 8));
    }
  }
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.o);
#pragma unroll
  for (int dt = 0; dt < ATT_D / 8; ++dt) {
    const long r0 = base + static_cast<long>(q0 + g) * C + dt * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(o + r0) = pack_bf16x2(oacc[dt][0] * i0, oacc[dt][1] * i0);
    *reinterpret_cast<uint32_t*>(o + r0 + 8L * C) = pack_bf16x2(oacc[dt][2] * i1, oacc[dt][3] * i1);
  }
}

// ---------------------------------------------------------------- attention (tcgen05)
// Persistent, warp-specialised: one CTA per SM walks (sequence, active head)
// units with two buffers of everything, so unit i+1's Q/K/V loads and S MMA
// overlap unit i's softmax and P.V.
//  * warp 0: TMA — Q, K, V of a unit are three {64 dims, 128 rows} SW128 boxes
//    of the subnet's [n*s][C_a] activations (maps in the op's OpDesc row:
//    amap = Q, rmap = K, wmap = V);
//  * warp 1: MMA issuer — S = Q K^T (M = N = 128, K = 64; both operands
//    K-major) into TMEM, then O = P V (M = 128, N = 64, K = 128; P K-major
//    from shared memory, V read MN-major straight from its TMA tile);
//  * warps 4-7 (even units, buffer 0) and 8-11 (odd units, buffer 1): one
//    thread per query row — tcgen05.ld of its 128 scores,
//    max / exp / sum in registers (no shuffles), P in bf16 written SW128
//    K-major for the second MMA, then O / l from TMEM to global.
// TMEM: S of buffer b at columns [128 b, 128 b + 128), O at 256 + 64 b.
constexpr int ATC_UNIT_SMEM = 80 * 1024;  // Q 16 KB | K 16 KB | V 16 KB | P 32 KB
constexpr int ATC_SMEM = 2 * ATC_UNIT_SMEM + 1024 + 256;

__device__ __forceinline__ uint64_t umma_desc_sw128_at(uint32_t addr) { return umma_desc_sw128(addr); }

constexpr int ATC_THREADS = 384;

__global__ void __launch_bounds__(ATC_THREADS, 1) attention_tc_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * ATC_UNIT_SMEM);
  uint64_t* kv_full = bar;       // [2] TMA landed Q, K, V
  uint64_t* kv_empty = bar + 2;  // [2] P.V of the buffer's last unit done (Q/K/V/P free)
  uint64_t* s_full = bar + 4;    // [2] S in TMEM
  uint64_t* s_empty = bar + 6;   // [2] S read out by the softmax warps
  uint64_t* p_full = bar + 8;    // [2] P in shared memory
  uint64_t* o_full = bar + 10;   // [2] O in TMEM
  uint64_t* o_empty = bar + 12;  // [2] O read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  pdl_wait();
  pdl_trigger();
  const OpDesc* dp = desc_ptr(p.row, nullptr, p.op);
  const int C = dp->cin;
  const int heads = C / ATT_D;
  const int units = p.n * heads;
  if (static_cast<int>(blockIdx.x) >= units) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&kv_full[b], 1);
      mbar_init(&kv_empty[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 4);  // the four softmax warps
      mbar_init(&p_full[b], 4);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 4);
    }
    fence_mbar_init();
    tma_prefetch(&dp->amap);
    tma_prefetch(&dp->rmap);
    tma_prefetch(&dp->wmap);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int step = static_cast<int>(gridDim.x);

  if (warp == 0) {
    // ============================================================ TMA producer
    const bool leader = elect_one();
    int i = 0;
    for (int u = blockIdx.x; u < units; u += step, ++i) {
      const int b = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      const int seq = u / heads, h = u - seq * heads;
      mbar_wait(&kv_empty[b], ph ^ 1);
      if (leader) {
        uint8_t* base = smem + b * ATC_UNIT_SMEM;
        mbar_arrive_expect_tx(&kv_full[b], 3 * ATT_S * ATT_D * 2);
        tma_load_2d(base, &dp->amap, &kv_full[b], h * ATT_D, seq * ATT_S);
        tma_load_2d(base + 16384, &dp->rmap, &kv_full[b], h * ATT_D, seq * ATT_S);
        tma_load_2d(base + 32768, &dp->wmap, &kv_full[b], h * ATT_D, seq * ATT_S);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ============================================================ MMA issuer
    const uint32_t idesc_s = umma_idesc_bf16(ATT_S, 128);
    const uint32_t idesc_o = umma_idesc_bf16(ATT_D, 128) | (1u << 16);  // B (V) MN-major
    const int count = (units - static_cast<int>(blockIdx.x) + step - 1) / step;
    auto mma_s = [&](int i) {
      const int b = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait(&kv_full[b], ph);
      mbar_wait(&s_empty[b], ph ^ 1);
      tc_fence_after();
      const uint32_t base = smem_u32(smem + b * ATC_UNIT_SMEM);
      const uint64_t qd = umma_desc_sw128_at(base), kd = umma_desc_sw128_at(base + 16384);
#pragma unroll
      for (int kk = 0; kk < ATT_D / 16; ++kk)
        tc_mma_bf16_elect(tmem + b * 128, qd + kk * 2, kd + kk * 2, idesc_s, kk ? 1u : 0u);
      tc_commit_elect(&s_full[b]);
      __syncwarp();
    };
    if (count > 0) mma_s(0);
    for (int i = 0; i < count; ++i) {
      if (i + 1 < count) mma_s(i + 1);
      const int b = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait(&p_full[b], ph);
      mbar_wait(&o_empty[b], ph ^ 1);
      tc_fence_after();
      const uint32_t base = smem_u32(smem + b * ATC_UNIT_SMEM);
      const uint64_t pd = umma_desc_sw128_at(base + 49152);
      const uint64_t vd = umma_desc_sw128_at(base + 32768);
#pragma unroll
      for (int kk = 0; kk < ATT_S / 16; ++kk)
        tc_mma_bf16_elect(tmem + 256 + b * 64,
                          pd + static_cast<uint64_t>((kk >> 2) * (16384 >> 4) + (kk & 3) * 2),
                          vd + static_cast<uint64_t>(kk * (2048 >> 4)), idesc_o, kk ? 1u : 0u);
      tc_commit_elect(&o_full[b]);
      tc_commit_elect(&kv_empty[b]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ============================================================ softmax + epilogue
    const int quarter = warp & 3;
    const int wg = (warp - 4) >> 2;     // warpgroup = buffer = unit parity
    const int r = quarter * 32 + lane;  // query row
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.o);
    int i = wg;
    for (int u = blockIdx.x + wg * step; u < units; u += 2 * step, i += 2) {
      const int b = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      const int seq = u / heads, h = u - seq * heads;
      mbar_wait(&s_full[b], ph);
      tc_fence_after();
      float sv[ATT_S];
#pragma unroll
      for (int c = 0; c < ATT_S / 32; ++c) {
        float t[32];
        tmem_ld32(tmem + lane_off + b * 128 + c * 32, t);
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[c * 32 + j] = t[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);
      float m = sv[0];
#pragma unroll
      for (int j = 1; j < ATT_S; ++j) m = fmaxf(m, sv[j]);
      const float scale = 0.125f;  // 1/sqrt(64)
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < ATT_S; ++j) {
        sv[j] = __expf((sv[j] - m) * scale);
        l += sv[j];
      }
      // P row r, SW128 K-major: key block kb (64 keys, 16 KB), 16-byte chunk
      // c of the 128-byte row lands at chunk c ^ (r % 8)
      uint8_t* pb = smem + b * ATC_UNIT_SMEM + 49152 + r * 128;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float* e = sv + kb * 64 + c * 8;
          uint4 v;
          v.x = pack_bf16x2(e[0], e[1]);
          v.y = pack_bf16x2(e[2], e[3]);
          v.z = pack_bf16x2(e[4], e[5]);
          v.w = pack_bf16x2(e[6], e[7]);
          *reinterpret_cast<uint4*>(pb + kb * 16384 + ((c ^ (r & 7)) << 4)) = v;
        }
      fence_proxy_async_smem();  // generic-proxy P stores -> the tensor core's reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      // O = P V / l
      mbar_wait(&o_full[b], ph);
      tc_fence_after();
      float o[ATT_D];
#pragma unroll
      for (int c = 0; c < ATT_D / 32; ++c) {
        float t[32];
        tmem_ld32(tmem + lane_off + 256 + b * 64 + c * 32, t);
#pragma unroll
        for (int j = 0; j < 32; ++j) o[c * 32 + j] = t[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[b]);
      const float il = 1.f / l;
      uint4* dst = reinterpret_cast<uint4*>(out + (static_cast<long>(seq) * ATT_S + r) * C + h * ATT_D);
#pragma unroll
      for (int c = 0; c < ATT_D / 8; ++c) {
        uint4 v;
        v.x = pack_bf16x2(o[c * 8 + 0] * il, o[c * 8 + 1] * il);
        v.y = pack_bf16x2(o[c * 8 + 2] * il, o[c * 8 + 3] * il);
        v.z = pack_bf16x2(o[c * 8 + 4] * il, o[c * 8 + 5] * il);
        v.w = pack_bf16x2(o[c * 8 + 6] * il, o[c * 8 + 7] * il);
        dst[c] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Q / K / V source of the tcgen05 attention: [rows][c] bf16 (c = active
// heads x 64), box {64 columns, 128 rows}, 128-byte swizzle (UMMA K-major
// for Q and K; V is read MN-major from the same layout).
int make_attn_map(CUtensorMap* map, const void* x, long rows, int c) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Fn enc = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<Fn>(ptr);
    return static_cast<Fn>(nullptr);
  }();
  if (!enc || c % ATT_D != 0) return -1;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(c) * 2};
  cuuint32_t box[2] = {ATT_D, ATT_S};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r);
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_embed(const EmbedParams& p, cudaStream_t s) {
  const long warps = static_cast<long>(p.n) * p.s;
  return launch_pdl(embed_ln_kernel, dim3(static_cast<int>((warps * 32 + 255) / 256)), dim3(256),
                    0, s, 1, p);
}

cudaError_t launch_layernorm(const LnParams& p, cudaStream_t s) {
  const int grid = static_cast<int>((static_cast<long>(p.rows) * 32 + 255) / 256);
  switch (p.hid) {
    case 256: return launch_pdl(layernorm_kernel<1>, dim3(grid), dim3(256), 0, s, 1, p);
    case 512: return launch_pdl(layernorm_kernel<2>, dim3(grid), dim3(256), 0, s, 1, p);
    case 768: return launch_pdl(layernorm_kernel<3>, dim3(grid), dim3(256), 0, s, 1, p);
    case 1024: return launch_pdl(layernorm_kernel<4>, dim3(grid), dim3(256), 0, s, 1, p);
    default: return cudaErrorInvalidValue;  // hidden width must be 256 * {1..4}
  }
}

cudaError_t launch_token0(const Token0Params& p, cudaStream_t s) {
  return launch_pdl(token0_kernel, dim3((p.n * (p.c / 8) + 255) / 256), dim3(256), 0, s, 1, p);
}

// tcgen05 path (engine rows carry the Q/K/V maps): persistent, one CTA per
// SM; `SSN_TC_DEBUG & 8388608` or a row without maps -> the mma.sync kernel
// (grid = n x max heads; CTAs past the active head count exit).
cudaError_t launch_attention(const AttnParams& p, int max_heads, bool tc, cudaStream_t s) {
  if (p.s != ATT_S) return cudaErrorInvalidValue;
  if (tc) {
    static const cudaError_t attr = cudaFuncSetAttribute(
        attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ATC_SMEM);
    if (attr != cudaSuccess) return attr;
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    const int units = p.n * max_heads;
    return launch_pdl(attention_tc_kernel, dim3(units < sms ? units : sms), dim3(ATC_THREADS),
                      ATC_SMEM, s, 1, p);
  }
  return launch_pdl(attention_kernel, dim3(p.n * max_heads), dim3(256), 0, s, 1, p);
}

}  // namespace ssn
