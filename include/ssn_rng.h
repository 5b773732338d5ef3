/*
 * ssn_rng.h — counter-based synthetic-data specification shared by the
 * SubNetAct engine (weight store / SubnetNorm defaults / synthetic images)
 * and the CPU oracle.
 *
 * The reference has no tensor payloads at all: `Query` carries no image
 * (reference proj/include/servesim/edf_queue.hpp:16-20) and supernet weights
 * are out of scope. Every value this build feeds a supernet is
 * therefore derived from (seed, stream, index) by the pure functions below,
 * so the GPU engine and the oracle see bit-identical inputs without sharing
 * any buffers.  This header is a *specification*, not a checker: it holds no
 * network code.
 *
 * Streams:  stream = (kind << 32) | ordinal
 *   kind 1  conv / linear / depthwise weight tensor #ordinal (canonical
 *           OIHW index order over the MAX shape)
 *   kind 2  BN gamma of norm layer #ordinal
 *   kind 3  BN beta  of norm layer #ordinal
 *   kind 4  linear bias of tensor #ordinal
 *   kind 5  synthetic image batch #ordinal (NCHW index order)
 *   kind 6  default SubnetNorm mean for (subnet id << 16 | active norm #)
 *   kind 7  default SubnetNorm var  for (subnet id << 16 | active norm #)
 *   kind 8  token ids (transformer supernet) for batch #ordinal
 */
#ifndef SSN_RNG_H
#define SSN_RNG_H

#include <stdint.h>
#include <string.h>
#include <math.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SSN_STREAM_WEIGHT = 1,
  SSN_STREAM_GAMMA = 2,
  SSN_STREAM_BETA = 3,
  SSN_STREAM_BIAS = 4,
  SSN_STREAM_IMAGE = 5,
  SSN_STREAM_STAT_MEAN = 6,
  SSN_STREAM_STAT_VAR = 7,
  SSN_STREAM_TOKENS = 8,
};

static inline uint64_t ssn_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t ssn_stream(uint32_t kind, uint32_t ordinal) {
  return ((uint64_t)kind << 32) | (uint64_t)ordinal;
}

/* Uniform in [0, 1) with 24 random bits (exactly representable in fp32). */
static inline float ssn_u01(uint64_t seed, uint64_t stream, uint64_t index) {
  const uint64_t key = ssn_mix64(seed ^ ssn_mix64(stream));
  const uint64_t h = ssn_mix64(key + index * 0xD1B54A32D192ED03ull);
  return (float)(h >> 40) * (1.0f / 16777216.0f);
}

/* Uniform in [-1, 1). */
static inline float ssn_sym(uint64_t seed, uint64_t stream, uint64_t index) {
  return 2.0f * ssn_u01(seed, stream, index) - 1.0f;
}

/* fp32 -> bf16 (round to nearest even), returned as the 16 payload bits. */
static inline uint16_t ssn_f32_to_bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return 0x7fc0;
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

static inline float ssn_bf16_bits_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline float ssn_round_bf16(float f) {
  return ssn_bf16_bits_to_f32(ssn_f32_to_bf16_bits(f));
}

/* Conv / linear weight: Kaiming-uniform over the MAX fan-in. */
static inline float ssn_weight_value(uint64_t seed, uint32_t ordinal,
                                     uint64_t index, uint32_t fan_in_max,
                                     int round_bf16) {
  const float bound = sqrtf(6.0f / (float)fan_in_max);
  const float v = bound * ssn_sym(seed, ssn_stream(SSN_STREAM_WEIGHT, ordinal), index);
  return round_bf16 ? ssn_round_bf16(v) : v;
}

/* BN gamma.  The last norm of a residual branch (the one whose output is
 * summed with the block input) draws from U(0, SSN_RES_GAMMA) instead of
 * U(0.5, 1.5), like the zero-init-residual initialisation of trained
 * ResNets; it keeps deep random supernets out of the chaotic regime where
 * bf16 storage rounding would be amplified layer after layer. */
#define SSN_RES_GAMMA 0.2f
static inline float ssn_gamma_value(uint64_t seed, uint32_t norm, uint64_t c) {
  return 0.5f + ssn_u01(seed, ssn_stream(SSN_STREAM_GAMMA, norm), c);
}
static inline float ssn_gamma_res_value(uint64_t seed, uint32_t norm, uint64_t c) {
  return SSN_RES_GAMMA * ssn_u01(seed, ssn_stream(SSN_STREAM_GAMMA, norm), c);
}

static inline float ssn_beta_value(uint64_t seed, uint32_t norm, uint64_t c) {
  return 0.1f * ssn_sym(seed, ssn_stream(SSN_STREAM_BETA, norm), c);
}

static inline float ssn_bias_value(uint64_t seed, uint32_t ordinal, uint64_t o) {
  return 0.1f * ssn_sym(seed, ssn_stream(SSN_STREAM_BIAS, ordinal), o);
}

/* Synthetic image value, NCHW canonical index. */
static inline float ssn_image_value(uint64_t seed, uint32_t batch_ordinal,
                                    uint64_t nchw_index) {
  return ssn_sym(seed, ssn_stream(SSN_STREAM_IMAGE, batch_ordinal), nchw_index);
}

/* Default (uncalibrated) SubnetNorm statistics. */
static inline float ssn_stat_mean_value(uint64_t seed, uint32_t subnet,
                                        uint32_t active_norm, uint64_t c) {
  return 0.1f * ssn_sym(seed, ssn_stream(SSN_STREAM_STAT_MEAN,
                                         (subnet << 16) | active_norm), c);
}

static inline float ssn_stat_var_value(uint64_t seed, uint32_t subnet,
                                       uint32_t active_norm, uint64_t c) {
  return 0.5f + ssn_u01(seed, ssn_stream(SSN_STREAM_STAT_VAR,
                                         (subnet << 16) | active_norm), c);
}

/* OFA make_divisible(v, 8): round to nearest multiple, never < 90% of v. */
static inline int ssn_make_divisible(double v, int divisor) {
  int nv = (int)(v + divisor / 2.0) / divisor * divisor;
  if (nv < divisor) nv = divisor;
  if ((double)nv < 0.9 * v) nv += divisor;
  return nv;
}

/* Python's round() on doubles: round half to even. */
static inline int ssn_round_half_even(double v) {
  double r = nearbyint(v); /* default FE_TONEAREST = half-even */
  return (int)r;
}

#ifdef __cplusplus
}
#endif
#endif /* SSN_RNG_H */
