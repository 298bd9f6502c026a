/*
 * fc_synth.h — counter-based synthetic gradient generator, bit-identical on
 * host (gcc, any -O level) and device (nvcc, sm_100a).
 *
 * The reference trains a toy model to obtain gradients (inc/model.hpp:100,
 * OUT of scope); BASELINE.json's configs use synthetic fp32 gradients keyed
 * by (seed, rank, step).  Only integer arithmetic plus ONE correctly rounded
 * fp32 multiply is used per element, so host and device agree to the bit
 * without any -ffp-contract / --fmad care:
 *
 *   S  = sum of six 21-bit uniform integers   (exact, < 2^24)
 *   x  = (float(S) - 3*2^21) * (sqrt(2) * 2^-21)   (Irwin-Hall(6), unit var)
 *
 * Distributions:
 *   FC_DIST_NORMAL  Irwin-Hall(6) ~ N(0,1), values on a sqrt(2)*2^-21 grid
 *   FC_DIST_TIES    same, rounded to a 2^-8 grid (forces threshold ties)
 *   FC_DIST_LAYERED same, scaled per 2^20-element block by 2^-(h%11)
 *                   (skews the radix histograms like a layered model)
 */
#ifndef FC_SYNTH_H_
#define FC_SYNTH_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define FC_HD __host__ __device__ __forceinline__
#else
#define FC_HD static inline
#endif

enum { FC_DIST_NORMAL = 0, FC_DIST_TIES = 1, FC_DIST_LAYERED = 2 };

FC_HD uint64_t fc_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* One stream per (seed, rank, step). */
FC_HD uint64_t fc_stream_key(uint64_t seed, uint32_t rank, uint64_t step) {
  return fc_mix64(seed ^ fc_mix64(((uint64_t)rank << 40) ^ (step * 0x2545F4914F6CDD1Dull) ^
                                  0x5851F42D4C957F2Dull));
}

FC_HD float fc_synth_value(uint64_t key, uint64_t i, int dist) {
  const uint64_t base = key ^ (i * 0xD6E8FEB86659FD93ull);
  uint32_t s = 0;
  for (uint32_t h = 0; h < 3; ++h) {
    const uint64_t r = fc_mix64(base + h);
    s += (uint32_t)(r >> 43);              /* bits 63..43 : 21 bits */
    s += (uint32_t)((r >> 22) & 0x1FFFFFu); /* bits 42..22 : 21 bits */
  }
  /* float(s) and the subtraction are exact (|.| < 2^24). */
  float x = ((float)s - 6291456.0f) * 6.7435232e-07f; /* sqrt(2) * 2^-21 */
  if (dist == FC_DIST_TIES) {
    /* round to a 2^-8 grid with integer ops only: s -> nearest multiple */
    int32_t q = ((int32_t)s - 6291456) / 5931; /* ~ 2^-8 / (sqrt2*2^-21) */
    x = (float)q * 0.00390625f;
  } else if (dist == FC_DIST_LAYERED) {
    const uint32_t e = (uint32_t)(fc_mix64(key ^ (i >> 20) ^ 0xA5A5A5A5ull) % 11u);
    /* exact power-of-two scaling */
    union { uint32_t u; float f; } sc;
    sc.u = (uint32_t)(127 - e) << 23;
    x = x * sc.f;
  }
  return x;
}

#endif /* FC_SYNTH_H_ */
