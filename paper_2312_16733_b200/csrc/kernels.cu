// kernels.cu — bandwidth-bound SubNetAct kernels (CUDA cores, sm_100a):
// input staging, pooling (max / avg-ceil / global), and the float32 SIMT
// WeightSlice conv used for the config-1 fp32 parity precision.
//
// All kernels are subnet-agnostic at launch: active channel counts come from
// the actuated subnet's OpDesc (device memory), so the same graph-captured
// launch serves every subnet.  bf16 paths move 8 channels (16 B) per thread
// access; active widths are multiples of 8 (OFA make_divisible(., 8)).
#include <algorithm>

#include "../../include/ssn.h"
#include "device.cuh"

namespace ssn {

// ---------------------------------------------------------------------------
// input staging: host-format images -> NHWC (bf16 padded to 8 ch, or fp32 3 ch)

__global__ void input_kernel(InputParams p) {
  pdl_wait();
  pdl_trigger();
  const long npix = static_cast<long>(p.n) * p.h * p.w;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < npix;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long hw = static_cast<long>(p.h) * p.w;
    const long img = i / hw, pix = i - img * hw;
    float v[3];
    if (p.format == SSN_INPUT_F32_NCHW) {
      const float* r = static_cast<const float*>(p.raw) + img * 3 * hw + pix;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = __ldg(r + c * hw);
    } else {
      const uint8_t* r = static_cast<const uint8_t*>(p.raw) + i * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = (static_cast<float>(r[c]) - 128.f) * (1.f / 64.f);
    }
    if (p.out_bf16) {
      uint4 pk;
      pk.x = pack_bf16x2(v[0], v[1]);
      pk.y = pack_bf16x2(v[2], 0.f);
      pk.z = 0u;
      pk.w = 0u;
      reinterpret_cast<uint4*>(p.y)[i] = pk;  // 8 channels, 3 real
    } else {
      float* y = static_cast<float*>(p.y) + i * 3;
      y[0] = v[0];
      y[1] = v[1];
      y[2] = v[2];
    }
  }
}

// Input staging fused with the stem conv's im2col (bf16): output pixel
// (n, oh, ow) gets the k*k*3 input values (r, s, c) of its window, zero
// padded, then zeros up to cpad (a multiple of 8) — a K = cpad GEMM operand.
// k = 3, cpad = 32 (both OFA stems): the 27 window values of one output
// pixel live in registers (the generic kernel below indexes a local array)
// and leave as four 16-byte stores.
template <bool U8>
__global__ void __launch_bounds__(256) input_im2col3_kernel(InputParams p) {
  pdl_wait();
  pdl_trigger();
  const long npix = static_cast<long>(p.n) * p.ho * p.wo;
  const int st = p.im2col_stride;
  const long hw = static_cast<long>(p.h) * p.w;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < npix;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long hwo = static_cast<long>(p.ho) * p.wo;
    const long img = i / hwo;
    const int rem = static_cast<int>(i - img * hwo);
    const int oh = rem / p.wo, ow = rem - oh * p.wo;
    float v[32];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ih = oh * st - 1 + r;
      const bool rok = ih >= 0 && ih < p.h;
#pragma unroll
      for (int s2 = 0; s2 < 3; ++s2) {
        const int iw = ow * st - 1 + s2;
        const bool ok = rok && iw >= 0 && iw < p.w;
        const int base = (r * 3 + s2) * 3;
        if (U8) {
          const uint8_t* src = static_cast<const uint8_t*>(p.raw) + ((img * p.h + ih) * p.w + iw) * 3;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            v[base + c] = ok ? (static_cast<float>(__ldg(src + c)) - 128.f) * (1.f / 64.f) : 0.f;
        } else {
          const float* src = static_cast<const float*>(p.raw) + img * 3 * hw + static_cast<long>(ih) * p.w + iw;
#pragma unroll
          for (int c = 0; c < 3; ++c) v[base + c] = ok ? __ldg(src + c * hw) : 0.f;
        }
      }
    }
#pragma unroll
    for (int q = 27; q < 32; ++q) v[q] = 0.f;
    uint4* y = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + i * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16x2(v[8 * q], v[8 * q + 1]);
      u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
      y[q] = u;
    }
  }
}

__global__ void input_im2col_kernel(InputParams p) {
  pdl_wait();
  pdl_trigger();
  const long npix = static_cast<long>(p.n) * p.ho * p.wo;
  const int k = p.im2col_k, st = p.im2col_stride, pad = k / 2;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < npix;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long hwo = static_cast<long>(p.ho) * p.wo;
    const long img = i / hwo;
    const int rem = static_cast<int>(i - img * hwo);
    const int oh = rem / p.wo, ow = rem - (rem / p.wo) * p.wo;
    float v[64];
#pragma unroll 1
    for (int q = 0; q < p.cpad; ++q) v[q] = 0.f;
    const long hw = static_cast<long>(p.h) * p.w;
    for (int r = 0; r < k; ++r) {
      const int ih = oh * st - pad + r;
      if (ih < 0 || ih >= p.h) continue;
      for (int s = 0; s < k; ++s) {
        const int iw = ow * st - pad + s;
        if (iw < 0 || iw >= p.w) continue;
        const int base = (r * k + s) * 3;
        if (p.format == SSN_INPUT_F32_NCHW) {
          const float* src = static_cast<const float*>(p.raw) + img * 3 * hw +
                             static_cast<long>(ih) * p.w + iw;
          v[base] = __ldg(src);
          v[base + 1] = __ldg(src + hw);
          v[base + 2] = __ldg(src + 2 * hw);
        } else {
          const uint8_t* src =
              static_cast<const uint8_t*>(p.raw) + ((img * p.h + ih) * p.w + iw) * 3;
          v[base] = (static_cast<float>(src[0]) - 128.f) * (1.f / 64.f);
          v[base + 1] = (static_cast<float>(src[1]) - 128.f) * (1.f / 64.f);
          v[base + 2] = (static_cast<float>(src[2]) - 128.f) * (1.f / 64.f);
        }
      }
    }
    uint4* y = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + i * p.cpad);
    for (int q = 0; q < p.cpad / 8; ++q) {
      uint4 u;
      u.x = pack_bf16x2(v[8 * q], v[8 * q + 1]);
      u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
      y[q] = u;
    }
  }
}

// ---------------------------------------------------------------------------
// Input staging fused with the bf16 stem conv (3x3, stride 2, pad 1, 3
// channels; both OFA stems): raw images -> SubnetNorm'd activations, no
// im2col buffer.  One CTA = one output row (image, oh): the three input rows
// it reads are normalised into shared memory as bf16 (1-px zero border),
// each warp forms m16n8k16 A fragments (16 output pixels x 16 of the 27 window
// values, zero past 27) straight from them, B = the [cout][32] im2col-order
// weight slice in registers, fp32 accumulate; SubnetNorm + activation in
// registers, the row is staged in shared memory and leaves as contiguous
// 16-byte stores.  Replaces input_im2col3 + a K = 32 GEMM that wrote and
// re-read a 32-channel im2col tensor (2 x 51 MB at bs64 x 224 px).
#ifndef SSN_STEM_THREADS
#define SSN_STEM_THREADS 128
#endif
#ifndef SSN_STEM_RPC
#define SSN_STEM_RPC 8  // 8 output rows per CTA: MBv3 bs256 stem 119 -> 109 us (2 / 4 rows slower; 256 threads slower)
#endif
constexpr int STEM_THREADS = SSN_STEM_THREADS;
constexpr int STEM_MAXW = 256;                       // input width bound (engine checks)
// staged input row (bf16): [5 unused][left zero pixel: 3][w pixels x 3][right zero pixel: 3],
// pixel data 16-byte aligned at element 8
constexpr int STEM_SROW = 8 + (STEM_MAXW + 1) * 3 + 5;
constexpr int STEM_COUT = 32;                        // max stem width (4 n8 tiles)
constexpr int STEM_RPC = SSN_STEM_RPC;               // output rows per CTA
constexpr int STEM_IN_ROWS = 2 * STEM_RPC + 1;       // input rows they read

__global__ void __launch_bounds__(STEM_THREADS) stem_conv_kernel(StemParams p) {
  __shared__ __align__(16) __nv_bfloat16 s_in[STEM_IN_ROWS * STEM_SROW];
  __shared__ __align__(16) __nv_bfloat16 s_out[(STEM_MAXW / 2 + 16) * STEM_COUT];
  pdl_wait();
  pdl_trigger();
  const int rblk = (p.ho + STEM_RPC - 1) / STEM_RPC;
  const int img = blockIdx.x / rblk, oh0 = (blockIdx.x - img * rblk) * STEM_RPC;
  const int tid = threadIdx.x;
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
  if (tid < STEM_IN_ROWS * 6) {  // the zero border pixels
    const int r = tid / 6, e = tid - r * 6;
    s_in[r * STEM_SROW + (e < 3 ? 5 + e : 8 + 3 * p.w_ + e - 3)] = zero;
  }
  if (p.format == SSN_INPUT_U8_NHWC && (p.w_ * 3) % 16 == 0) {
    // one 16-byte load per thread: row r, bytes 16q..16q+15 (pixels interleaved RGB)
    const int vrow = p.w_ * 3 / 16;
#pragma unroll 4
    for (int idx = tid; idx < STEM_IN_ROWS * vrow; idx += STEM_THREADS) {
      const int r = idx / vrow, q = idx - r * vrow;
      const int ih = 2 * oh0 - 1 + r;
      const bool ok = ih >= 0 && ih < p.h;
      uint4 u = make_uint4(0u, 0u, 0u, 0u);
      if (ok)
        u = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.raw) +
                                                 (static_cast<long>(img) * p.h + ih) * p.w_ * 3) + q);
      const uint32_t wds[4] = {u.x, u.y, u.z, u.w};
      uint32_t pk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t wd = wds[k >> 1] >> (16 * (k & 1));
        const float v0 = ok ? (static_cast<float>(wd & 255u) - 128.f) * (1.f / 64.f) : 0.f;
        const float v1 = ok ? (static_cast<float>((wd >> 8) & 255u) - 128.f) * (1.f / 64.f) : 0.f;
        pk[k] = pack_bf16x2(v0, v1);
      }
      uint4* dst = reinterpret_cast<uint4*>(s_in + r * STEM_SROW + 8 + 16 * q);
      dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
  } else {
    const int rowlen = p.w_ * 3;
    for (int idx = tid; idx < STEM_IN_ROWS * rowlen; idx += STEM_THREADS) {
      const int r = idx / rowlen, q = idx - r * rowlen;
      const int px = q / 3, c = q - px * 3;
      const int ih = 2 * oh0 - 1 + r;
      float v = 0.f;
      if (ih >= 0 && ih < p.h) {
        if (p.format == SSN_INPUT_U8_NHWC) {
          const uint8_t* src = static_cast<const uint8_t*>(p.raw);
          v = (static_cast<float>(__ldg(src + ((static_cast<long>(img) * p.h + ih) * p.w_ + px) * 3 + c)) -
               128.f) * (1.f / 64.f);
        } else {
          const float* src = static_cast<const float*>(p.raw);
          v = __ldg(src + ((static_cast<long>(img) * 3 + c) * p.h + ih) * p.w_ + px);
        }
      }
      s_in[r * STEM_SROW + 8 + q] = __float2bfloat16_rn(v);
    }
  }
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int cout = d.cout;  // active (WeightSlice), <= STEM_COUT, multiple of 8
  const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, tq = lane & 3;
  // this thread's 8 window offsets: K index k = 16 ks + 8 hi + 2 tq + lo
  int koff[8];
  bool kok[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = (j >> 2) * 16 + ((j >> 1) & 1) * 8 + 2 * tq + (j & 1);
    const int r = k / 9, sx = (k % 9) / 3, c = k % 3;
    kok[j] = k < 27;
    koff[j] = kok[j] ? r * STEM_SROW + 5 + 3 * sx + c : 0;  // window pixel (2 ow - 1 + sx)
  }
  // B fragments: column n = 8 nt + g of W^T, rows 2 tq (+1) and 2 tq + 8 (+1)
  uint32_t b[4][2][2];
  float sc[4][2], sh[4][2];
  const uint32_t* wv = static_cast<const uint32_t*>(p.w);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int n = 8 * nt + g;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      b[nt][ks][0] = n < cout ? __ldg(wv + (n * 32 + ks * 16 + 2 * tq) / 2) : 0u;
      b[nt][ks][1] = n < cout ? __ldg(wv + (n * 32 + ks * 16 + 2 * tq + 8) / 2) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = 8 * nt + 2 * tq + e;
      sc[nt][e] = (d.scale && col < cout) ? __ldg(d.scale + col) : 1.f;
      sh[nt][e] = (d.shift && col < cout) ? __ldg(d.shift + col) : 0.f;
    }
  }
  __syncthreads();
  const unsigned short* sin16 = reinterpret_cast<const unsigned short*>(s_in);
  auto a_val = [&](int base, int j) -> uint32_t {
    return kok[j] ? static_cast<uint32_t>(sin16[base + koff[j]]) : 0u;
  };
  const int mtiles = (p.wo + 15) / 16;
  for (int rr = 0; rr < STEM_RPC; ++rr) {
    const int oh = oh0 + rr;
    if (oh >= p.ho) break;
    const int rbase = 2 * rr * STEM_SROW;  // this output row's window starts at staged row 2 rr
    for (int mt = warp; mt < mtiles; mt += STEM_THREADS / 32) {
      const int ow0 = min(mt * 16 + g, p.wo - 1), ow1 = min(mt * 16 + g + 8, p.wo - 1);
      float acc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        uint32_t a[4];
        const int j = ks * 4;
        a[0] = a_val(rbase + 6 * ow0, j) | (a_val(rbase + 6 * ow0, j + 1) << 16);
        a[1] = a_val(rbase + 6 * ow1, j) | (a_val(rbase + 6 * ow1, j + 1) << 16);
        a[2] = a_val(rbase + 6 * ow0, j + 2) | (a_val(rbase + 6 * ow0, j + 3) << 16);
        a[3] = a_val(rbase + 6 * ow1, j + 2) | (a_val(rbase + 6 * ow1, j + 3) << 16);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) mma_bf16_16816(acc[nt], a, b[nt][ks][0], b[nt][ks][1]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ow = mt * 16 + g + 8 * h;
        if (ow >= p.wo) continue;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int col = 8 * nt + 2 * tq;
          if (col >= cout) continue;
          const float o0 = act_apply(acc[nt][2 * h] * sc[nt][0] + sh[nt][0], p.act);
          const float o1 = act_apply(acc[nt][2 * h + 1] * sc[nt][1] + sh[nt][1], p.act);
          *reinterpret_cast<uint32_t*>(s_out + ow * cout + col) = pack_bf16x2(o0, o1);
        }
      }
    }
    __syncthreads();
    // the output row: wo pixels of cout bf16 at the row stride d.ldo (16-byte
    // multiples: cout % 8 == 0)
    const int npx = cout / 8, ld8 = d.ldo / 8;
    const int nvec = p.wo * npx;
    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) +
                                          (static_cast<long>(img) * p.ho + oh) * p.wo * d.ldo);
    const uint4* src = reinterpret_cast<const uint4*>(s_out);
    for (int i = tid; i < nvec; i += STEM_THREADS) {
      const int px = i / npx;
      dst[px * ld8 + (i - px * npx)] = src[i];
    }
    __syncthreads();  // s_out is rewritten by the next row
  }
}

// ---------------------------------------------------------------------------
// pooling, bf16 NHWC, 8 channels per thread

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 t = __bfloat1622float2(h[q]);
    f[2 * q] = t.x;
    f[2 * q + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 u;
  u.x = pack_bf16x2(f[0], f[1]);
  u.y = pack_bf16x2(f[2], f[3]);
  u.z = pack_bf16x2(f[4], f[5]);
  u.w = pack_bf16x2(f[6], f[7]);
  return u;
}

// Global average pool, bf16 [n][hw][C] -> [n][C]: block (image, 64-channel
// chunk), 8 channel groups x 32 pixel lanes and a shared-memory reduction,
// so the hw loads of a channel group are in flight together (one thread per
// channel group summing hw pixels serially was latency-bound).
// Global average pool: block = (image, 256 channels); thread = 8 channels of
// every 8th pixel (independent 16-byte loads, ~hw/8 per thread), then an
// 8-way smem reduction.  (One 64-channel block per CTA with 32 pixel lanes
// left most of the 7-px kernel's time in launch / reduction latency.)
__global__ void __launch_bounds__(256) gap_bf16_kernel(PoolParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin;
  const int n = blockIdx.x, c0 = blockIdx.y * 256;
  if (c0 >= C) return;
  const int hw = p.h * p.w;
  const int g = threadIdx.x & 31, lane = threadIdx.x >> 5;
  const int c = c0 + g * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x) + static_cast<long>(n) * hw * d.ldi;
  if (c < C) {
#pragma unroll 4
    for (int q = lane; q < hw; q += 8) {
      float f[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(x + static_cast<long>(q) * d.ldi + c)), f);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += f[t];
    }
  }
  __shared__ float red[8][257];
#pragma unroll
  for (int t = 0; t < 8; ++t) red[lane][g * 8 + t] = acc[t];
  __syncthreads();
  const int cc = c0 + threadIdx.x;
  if (cc < C) {
    float sum = 0.f;
#pragma unroll
    for (int l = 0; l < 8; ++l) sum += red[l][threadIdx.x];
    static_cast<__nv_bfloat16*>(p.y)[static_cast<long>(n) * d.ldo + cc] =
        __float2bfloat16_rn(sum / static_cast<float>(hw));
  }
}

// Max (KIND 2) / ceil-average (KIND 3) pooling with a compile-time window:
// grid (output rows n*ho, ceil(wo * C/8 / 256)); all K*K 16-byte loads of a
// thread are independent and issued together (the generic kernel's runtime
// window loop serialised them), 32-bit index math.
template <int K, int KIND>
__global__ void __launch_bounds__(256) pool_k_bf16_kernel(PoolParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin, G = C >> 3;
  const int row = blockIdx.y;
  const int img = row / p.ho, oh = row - img * p.ho;
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j >= p.wo * G) return;
  const int ow = j / G, g = j - ow * G;
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x) + g * 8;
  uint4 v[K * K];
  bool ok[K * K];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int s2 = 0; s2 < K; ++s2) {
      const int ih = oh * p.stride - p.pad + r, iw = ow * p.stride - p.pad + s2;
      ok[r * K + s2] = ih >= 0 && ih < p.h && iw >= 0 && iw < p.w;
      v[r * K + s2] = ok[r * K + s2]
                          ? __ldg(reinterpret_cast<const uint4*>(
                                x + (static_cast<size_t>(img * p.h + ih) * p.w + iw) * d.ldi))
                          : make_uint4(0, 0, 0, 0);
    }
  if constexpr (KIND == 2) {
    // max is exact in bf16: packed bf16x2 max (HMNMX2), no fp32 round trip —
    // the fp32 version issued ~3 instructions per byte (ncu: issue slots 73%
    // busy, DRAM 41%)
    __nv_bfloat162 m[4];
    const __nv_bfloat162 ninf = __halves2bfloat162(__ushort_as_bfloat16(0xFF80u), __ushort_as_bfloat16(0xFF80u));
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = ninf;
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      if (!ok[q]) continue;
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[q]);
#pragma unroll
      for (int t = 0; t < 4; ++t) m[t] = __hmax2(m[t], h[t]);
    }
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + (static_cast<size_t>(row) * p.wo + ow) * d.ldo +
                              g * 8) = *reinterpret_cast<const uint4*>(m);
  } else {  // ceil-average: fp32 sums
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = 0.f;
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      if (!ok[q]) continue;
      ++cnt;
      float f[8];
      bf16x8_to_f32(v[q], f);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += f[t];
    }
    const float inv = 1.f / static_cast<float>(cnt);
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] *= inv;
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) +
                              (static_cast<size_t>(row) * p.wo + ow) * d.ldo + g * 8) = f32_to_bf16x8(acc);
  }
}

__global__ void pool_bf16_kernel(PoolParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin, G = C >> 3;
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x);
  __nv_bfloat16* y = static_cast<__nv_bfloat16*>(p.y);
  if (p.kind == 4) {  // global average pool -> [n][C]
    const long total = static_cast<long>(p.n) * G;
    const int hw = p.h * p.w;
    const float inv = 1.f / static_cast<float>(hw);
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
      const long img = i / G;
      const int g = static_cast<int>(i - img * G);
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const __nv_bfloat16* src = x + img * hw * d.ldi + g * 8;
      for (int q = 0; q < hw; ++q) {
        float f[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(src + static_cast<long>(q) * d.ldi), f);
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] += f[t];
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] *= inv;
      *reinterpret_cast<uint4*>(y + img * d.ldo + g * 8) = f32_to_bf16x8(acc);
    }
    return;
  }
  const long total = static_cast<long>(p.n) * p.ho * p.wo * G;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long opix = i / G;
    const int g = static_cast<int>(i - opix * G);
    const long img = opix / (static_cast<long>(p.ho) * p.wo);
    const int rem = static_cast<int>(opix - img * p.ho * p.wo);
    const int oh = rem / p.wo, ow = rem - (rem / p.wo) * p.wo;
    float acc[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[t] = p.kind == 2 ? -INFINITY : 0.f;
    int cnt = 0;
    for (int r = 0; r < p.k; ++r) {
      const int ih = oh * p.stride - p.pad + r;
      if (ih < 0 || ih >= p.h) continue;
      for (int s = 0; s < p.k; ++s) {
        const int iw = ow * p.stride - p.pad + s;
        if (iw < 0 || iw >= p.w) continue;
        float f[8];
        bf16x8_to_f32(
            *reinterpret_cast<const uint4*>(x + ((img * p.h + ih) * p.w + iw) * d.ldi + g * 8), f);
        ++cnt;
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = p.kind == 2 ? fmaxf(acc[t], f[t]) : acc[t] + f[t];
      }
    }
    if (p.kind == 3) {
      const float inv = 1.f / static_cast<float>(cnt);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] *= inv;
    }
    *reinterpret_cast<uint4*>(y + opix * d.ldo + g * 8) = f32_to_bf16x8(acc);
  }
}

__global__ void pool_f32_kernel(PoolParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin;
  const float* x = static_cast<const float*>(p.x);
  float* y = static_cast<float*>(p.y);
  if (p.kind == 4) {
    const long total = static_cast<long>(p.n) * C;
    const int hw = p.h * p.w;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
      const long img = i / C;
      const int c = static_cast<int>(i - img * C);
      float acc = 0.f;
      for (int q = 0; q < hw; ++q) acc += x[(img * hw + q) * C + c];
      y[img * C + c] = acc / static_cast<float>(hw);
    }
    return;
  }
  const long total = static_cast<long>(p.n) * p.ho * p.wo * C;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long opix = i / C;
    const int c = static_cast<int>(i - opix * C);
    const long img = opix / (static_cast<long>(p.ho) * p.wo);
    const int rem = static_cast<int>(opix - img * p.ho * p.wo);
    const int oh = rem / p.wo, ow = rem % p.wo;
    float acc = p.kind == 2 ? -INFINITY : 0.f;
    int cnt = 0;
    for (int r = 0; r < p.k; ++r) {
      const int ih = oh * p.stride - p.pad + r;
      if (ih < 0 || ih >= p.h) continue;
      for (int s = 0; s < p.k; ++s) {
        const int iw = ow * p.stride - p.pad + s;
        if (iw < 0 || iw >= p.w) continue;
        const float v = x[((img * p.h + ih) * p.w + iw) * C + c];
        acc = p.kind == 2 ? fmaxf(acc, v) : acc + v;
        ++cnt;
      }
    }
    y[opix * C + c] = p.kind == 3 ? acc / static_cast<float>(cnt) : acc;
  }
}

// ---------------------------------------------------------------------------
// float32 WeightSlice conv / depthwise / linear (SIMT), config-1 precision.
// weights: dense KRSC [cout_max][k_max][k_max][cin_max]; depthwise
// [c_max][k_max][k_max]; centre crop to the active k.

__global__ void conv_f32_kernel(ConvParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, p.fixed, p.op);
  const long total = static_cast<long>(p.M) * d.cout;
  const float* x = static_cast<const float*>(p.x);
  const float* w = static_cast<const float*>(p.w);
  const int off = (p.k_max - d.k) / 2;
  const int hwo = p.ho * p.wo;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long m = i / d.cout;
    const int co = static_cast<int>(i - m * d.cout);
    const int img = static_cast<int>(m / hwo);
    const int rem = static_cast<int>(m - static_cast<long>(img) * hwo);
    const int oh = rem / p.wo, ow = rem % p.wo;
    float acc = 0.f;
    for (int r = 0; r < d.k; ++r) {
      const int ih = oh * p.stride - d.pad + r;
      if (ih < 0 || ih >= p.h) continue;
      for (int s = 0; s < d.k; ++s) {
        const int iw = ow * p.stride - d.pad + s;
        if (iw < 0 || iw >= p.w_) continue;
        const float* xp = x + (static_cast<long>(img * p.h + ih) * p.w_ + iw) * d.cin;
        const int tap = (r + off) * p.k_max + (s + off);
        if (p.depthwise) {
          acc += xp[co] * __ldg(w + static_cast<long>(co) * p.k_max * p.k_max + tap);
        } else {
          const float* wp = w + (static_cast<long>(co) * p.k_max * p.k_max + tap) * p.cin_max;
          for (int ci = 0; ci < d.cin; ++ci) acc += xp[ci] * __ldg(wp + ci);
        }
      }
    }
    float v = acc * (d.scale ? d.scale[co] : 1.f) + (d.shift ? d.shift[co] : 0.f);
    const float* res = static_cast<const float*>(p.res);
    if (res && !p.res_post) v += res[m * d.cout + co];
    v = act_apply(v, p.act);
    if (res && p.res_post) v += res[m * d.cout + co];
    static_cast<float*>(p.y)[m * d.cout + co] = v;
  }
}

// ---------------------------------------------------------------------------
// Squeeze-excite (OFA DynamicSE): pool -> reduce FC + ReLU -> expand FC +
// h_sigmoid -> scale the activation in place.

// pooled[n][c] = mean over hw; grid (n, ceil(C/64)), 256 threads:
// 8 channel groups x 32 pixel lanes, shared-memory reduction over lanes.
__global__ void se_pool_kernel(SEParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin;
  const int n = blockIdx.x, c0 = blockIdx.y * 64;
  if (c0 >= C) return;
  const int g = threadIdx.x & 7, lane = threadIdx.x >> 3;
  const int c = c0 + g * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const __nv_bfloat16* x = static_cast<const __nv_bfloat16*>(p.x) + static_cast<long>(n) * p.hw * d.ldi;
  if (c < C) {
    for (int q = lane; q < p.hw; q += 32) {
      float f[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(x + static_cast<long>(q) * d.ldi + c)), f);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += f[t];
    }
  }
  __shared__ float red[32][65];
#pragma unroll
  for (int t = 0; t < 8; ++t) red[lane][g * 8 + t] = acc[t];
  __syncthreads();
  if (threadIdx.x < 64 && c0 + threadIdx.x < C) {
    float s = 0.f;
    for (int l = 0; l < 32; ++l) s += red[l][threadIdx.x];
    p.pooled[static_cast<long>(n) * p.c_max + c0 + threadIdx.x] = s / static_cast<float>(p.hw);
  }
}

// Fused-pool variant: the depthwise kernel left per-tile channel sums of its
// stored output in parts_buf [n][parts][c_max]; add them in fixed order.
// grid (n, ceil(c_max / 256)), one thread per channel.
__global__ void __launch_bounds__(256) se_pool_parts_kernel(SEParams p) {
  pdl_wait();
  pdl_trigger();
  const OpDesc* dp = desc_ptr(p.row, nullptr, p.op);
  const int C = dp->cin;
  const int n = blockIdx.x, c = blockIdx.y * 256 + threadIdx.x;
  if (c >= C) return;
  const float* src = p.parts_buf + static_cast<long>(n) * p.parts * p.c_max + c;
  float s = 0.f;
  for (int t = 0; t < p.parts; ++t) s += __ldg(src + static_cast<long>(t) * p.c_max);
  p.pooled[static_cast<long>(n) * p.c_max + c] = s / static_cast<float>(p.hw);
}

// gate[n][c] = h_sigmoid(We[c, :mid] . relu(Wr[:mid, :C] . pooled[n] + br) + be[c]),
// as two kernels gridded over (SE_NB-sample batch, output rows) so the weight
// rows are read once per SE_NB samples and every SM has work.  hid lives in
// the tail of the gate scratch (fp32 [n][se_max]).
constexpr int SE_NB = 8;

__device__ __forceinline__ float* se_hid(const SEParams& p) {
  return p.gate + static_cast<long>(p.n) * p.c_max;
}

// The two SE FCs as one kernel shape: thread = (output row, K slice), eight
// samples per CTA.  The samples' input rows (pooled / hidden, fp32) are staged
// once in shared memory and read as broadcasts; each thread streams its own
// weight row (16-byte loads, L1-resident across the K loop) and keeps 8 sample
// accumulators, so the inner loop is 8 FMA per 16 B of weights with no warp
// reduction.  (The warp-per-row version spent more issue slots in its
// 32-accumulator shuffle reductions than in FMAs: 11-40 us per bs256 launch,
// ~2 TFMA/s.)  KS K slices per row meet in shared memory in fixed order.
constexpr int SE_KMAX = 1152;  // widest SE input (OFA-MBv3 w1.2 stage 5)
template <int KS, bool EXPAND>
__global__ void __launch_bounds__(256) se_fc_kernel(SEParams p) {
  __shared__ __align__(16) float xs[SE_NB][SE_KMAX];
  __shared__ float red[KS > 1 ? KS : 1][SE_NB][256 / KS];
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin, mid = desc_ptr(p.row, nullptr, p.op)->aux;
  const int K = EXPAND ? mid : C, rows = EXPAND ? C : mid;
  const float* in = EXPAND ? se_hid(p) : p.pooled;
  const long in_ld = EXPAND ? p.se_max : p.c_max;
  const __nv_bfloat16* w = static_cast<const __nv_bfloat16*>(EXPAND ? p.w_expand : p.w_reduce);
  const long w_ld = EXPAND ? p.se_max : p.w_ld;
  constexpr int RPC = 256 / KS;  // output rows per CTA
  const int tid = threadIdx.x, rl = tid % RPC, ks = tid / RPC;
  const int row = blockIdx.y * RPC + rl;
  const int n0 = blockIdx.x * SE_NB, nb = min(SE_NB, p.n - n0);
  if (blockIdx.y * RPC >= rows) return;
  for (int i = tid; i < SE_NB * (K / 4); i += 256) {
    const int b = i / (K / 4), k4 = i - b * (K / 4);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (b < nb) v = __ldg(reinterpret_cast<const float4*>(in + (n0 + b) * in_ld) + k4);
    reinterpret_cast<float4*>(xs[b])[k4] = v;
  }
  __syncthreads();
  float acc[SE_NB];
#pragma unroll
  for (int b = 0; b < SE_NB; ++b) acc[b] = 0.f;
  const int kper = (K / 8 + KS - 1) / KS * 8;
  const int k0 = ks * kper, k1 = min(K, k0 + kper);
  if (row < rows) {
    const __nv_bfloat16* wr = w + row * w_ld;
    for (int k = k0; k < k1; k += 8) {
      float wv[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(wr + k)), wv);
#pragma unroll
      for (int b = 0; b < SE_NB; ++b) {
        const float4 x0 = *reinterpret_cast<const float4*>(&xs[b][k]);
        const float4 x1 = *reinterpret_cast<const float4*>(&xs[b][k + 4]);
        acc[b] += wv[0] * x0.x + wv[1] * x0.y + wv[2] * x0.z + wv[3] * x0.w +
                  wv[4] * x1.x + wv[5] * x1.y + wv[6] * x1.z + wv[7] * x1.w;
      }
    }
  }
  if (KS > 1) {
#pragma unroll
    for (int b = 0; b < SE_NB; ++b) red[ks][b][rl] = acc[b];
    __syncthreads();
    if (ks != 0) return;
#pragma unroll
    for (int b = 0; b < SE_NB; ++b) {
      float t = 0.f;
#pragma unroll
      for (int z = 0; z < KS; ++z) t += red[z][b][rl];
      acc[b] = t;
    }
  }
  if (row >= rows) return;
#pragma unroll
  for (int b = 0; b < SE_NB; ++b) {
    if (b >= nb) break;
    if (EXPAND)
      p.gate[static_cast<long>(n0 + b) * p.c_max + row] =
          fminf(fmaxf(acc[b] + p.b_expand[row] + 3.f, 0.f), 6.f) * (1.f / 6.f);
    else
      se_hid(p)[static_cast<long>(n0 + b) * p.se_max + row] = fmaxf(acc[b] + p.b_reduce[row], 0.f);
  }
}

// x[n][pix][c] *= gate[n][c], in place.  Grid (image, pixel chunk): the
// image's gate row is staged in shared memory once per CTA and each thread
// keeps SE_SC_ILP independent 16-byte loads in flight (the grid-stride
// version with per-element div/mod index math reached ~0.5 of HBM).
constexpr int SE_SC_ILP = 4;
__global__ void __launch_bounds__(256) se_scale_kernel(SEParams p) {
  __shared__ __align__(16) float g[SE_KMAX];
  pdl_wait();
  pdl_trigger();
  const OpDims d = load_desc(p.row, nullptr, p.op);
  const int C = d.cin, G = C >> 3;
  const int n = blockIdx.y;
  for (int c = threadIdx.x; c < C; c += 256) g[c] = p.gate[static_cast<long>(n) * p.c_max + c];
  __syncthreads();
  __nv_bfloat16* x = static_cast<__nv_bfloat16*>(p.x) + static_cast<long>(n) * p.hw * d.ldi;
  const int per_img = p.hw * G;  // 16-byte groups of this image
  const int base = blockIdx.x * (256 * SE_SC_ILP) + threadIdx.x;
  uint4 v[SE_SC_ILP];
  int idx[SE_SC_ILP];
#pragma unroll
  for (int u = 0; u < SE_SC_ILP; ++u) {
    idx[u] = base + u * 256;
    if (idx[u] < per_img) {
      const int pix = idx[u] / G, gg = idx[u] - pix * G;
      v[u] = *reinterpret_cast<const uint4*>(x + static_cast<long>(pix) * d.ldi + gg * 8);
    }
  }
#pragma unroll
  for (int u = 0; u < SE_SC_ILP; ++u) {
    if (idx[u] >= per_img) continue;
    const int pix = idx[u] / G, gg = idx[u] - pix * G;
    float f[8];
    bf16x8_to_f32(v[u], f);
    const float4 g0 = *reinterpret_cast<const float4*>(g + gg * 8);
    const float4 g1 = *reinterpret_cast<const float4*>(g + gg * 8 + 4);
    f[0] *= g0.x; f[1] *= g0.y; f[2] *= g0.z; f[3] *= g0.w;
    f[4] *= g1.x; f[5] *= g1.y; f[6] *= g1.z; f[7] *= g1.w;
    *reinterpret_cast<uint4*>(x + static_cast<long>(pix) * d.ldi + gg * 8) = f32_to_bf16x8(f);
  }
}

__global__ void set_row_kernel(const OpDesc** slot, const OpDesc* row) { *slot = row; }

// ---------------------------------------------------------------------------
// launchers

static inline int grid_for(long work, int block) {
  long g = (work + block - 1) / block;
  const long cap = 148L * 16;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

cudaError_t launch_input(const InputParams& p, cudaStream_t s) {
  const long npix = static_cast<long>(p.n) * p.ho * p.wo;
  if (p.im2col_k == 3 && p.cpad == 32) {
    const int grid = static_cast<int>(std::min<long>((npix + 255) / 256, 148L * 8));
    return launch_pdl(p.format == SSN_INPUT_U8_NHWC ? input_im2col3_kernel<true>
                                                   : input_im2col3_kernel<false>,
                      dim3(grid), dim3(256), 0, s, 1, p);
  }
  if (p.im2col_k > 0)
    return launch_pdl(input_im2col_kernel, dim3(grid_for(npix, 128)), dim3(128), 0, s, 1, p);
  return launch_pdl(input_kernel, dim3(grid_for(static_cast<long>(p.n) * p.h * p.w, 256)),
                    dim3(256), 0, s, 1, p);
}

cudaError_t launch_stem_conv(const StemParams& p, cudaStream_t s) {
  if (p.w_ > STEM_MAXW || p.wo > STEM_MAXW / 2 + 16) return cudaErrorInvalidValue;
  const int rblk = (p.ho + STEM_RPC - 1) / STEM_RPC;
  return launch_pdl(stem_conv_kernel, dim3(p.n * rblk), dim3(STEM_THREADS), 0, s, 1, p);
}

// `max_c` bounds the grid for the largest subnet; surplus threads exit.
cudaError_t launch_pool(const PoolParams& p, int max_c, bool bf16, cudaStream_t s) {
  const long per = bf16 ? max_c / 8 : max_c;
  const long work = p.kind == 4 ? static_cast<long>(p.n) * per
                                : static_cast<long>(p.n) * p.ho * p.wo * per;
  const dim3 rows_grid(static_cast<unsigned>((p.wo * (max_c / 8) + 255) / 256),
                       static_cast<unsigned>(p.n * p.ho));
  if (bf16 && p.kind == 4)
    return launch_pdl(gap_bf16_kernel, dim3(p.n, (max_c + 255) / 256), dim3(256), 0, s, 1, p);
  if (bf16 && p.kind == 2 && p.k == 3)
    return launch_pdl(pool_k_bf16_kernel<3, 2>, rows_grid, dim3(256), 0, s, 1, p);
  if (bf16 && p.kind == 3 && p.k == 2)
    return launch_pdl(pool_k_bf16_kernel<2, 3>, rows_grid, dim3(256), 0, s, 1, p);
  if (bf16) return launch_pdl(pool_bf16_kernel, dim3(grid_for(work, 256)), dim3(256), 0, s, 1, p);
  return launch_pdl(pool_f32_kernel, dim3(grid_for(work, 256)), dim3(256), 0, s, 1, p);
}

cudaError_t launch_conv_f32(const ConvParams& p, cudaStream_t s) {
  return launch_pdl(conv_f32_kernel, dim3(grid_for(static_cast<long>(p.M) * p.cout_max, 128)),
                    dim3(128), 0, s, 1, p);
}

cudaError_t launch_se(const SEParams& p, cudaStream_t s) {
  cudaError_t e =
      p.parts > 0
          ? launch_pdl(se_pool_parts_kernel, dim3(p.n, (p.c_max + 255) / 256), dim3(256), 0, s, 1, p)
          : launch_pdl(se_pool_kernel, dim3(p.n, (p.c_max + 63) / 64), dim3(256), 0, s, 1, p);
  if (e != cudaSuccess) return e;
  const int nbk = (p.n + SE_NB - 1) / SE_NB;
  if (p.c_max > SE_KMAX || p.se_max > SE_KMAX) return cudaErrorInvalidValue;
  // reduce: rows = squeeze width (<= 288), K = channels: 4 K slices x 64 rows;
  // expand: rows = channels, K = squeeze width: 1 slice x 256 rows
  e = launch_pdl(se_fc_kernel<4, false>, dim3(nbk, (p.se_max + 63) / 64), dim3(256), 0, s, 1, p);
  if (e != cudaSuccess) return e;
  e = launch_pdl(se_fc_kernel<1, true>, dim3(nbk, (p.c_max + 255) / 256), dim3(256), 0, s, 1, p);
  if (e != cudaSuccess) return e;
  const long per_img = static_cast<long>(p.hw) * (p.c_max / 8);  // grid sized for the max width
  return launch_pdl(se_scale_kernel,
                    dim3(static_cast<unsigned>((per_img + 256 * SE_SC_ILP - 1) / (256 * SE_SC_ILP)),
                         static_cast<unsigned>(p.n)),
                    dim3(256), 0, s, 1, p);
}

cudaError_t launch_set_row(const OpDesc** slot, const OpDesc* row, cudaStream_t s) {
  set_row_kernel<<<1, 1, 0, s>>>(slot, row);
  return cudaGetLastError();
}

}  // namespace ssn
