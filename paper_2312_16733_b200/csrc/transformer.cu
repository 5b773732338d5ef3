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

// grid = n x max heads; CTAs past the active head count exit
cudaError_t launch_attention(const AttnParams& p, int max_heads, cudaStream_t s) {
  if (p.s != ATT_S) return cudaErrorInvalidValue;
  return launch_pdl(attention_kernel, dim3(p.n * max_heads), dim3(256), 0, s, 1, p);
}

}  // namespace ssn
