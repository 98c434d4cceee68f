/*
 * fctgen/gen.c -- seeded, index-addressable synthetic INPUT generators.
 *
 * This module is shared by the CUDA path's tests/bench and by the oracle's tests.
 * It holds NO arithmetic of the method (no Hadamard, no Cauchy scaling of data, no
 * hashing into a sketch, no median, no sampling decision): it only draws the random
 * inputs that both sides read (A, the Rademacher signs D, the Cauchy diagonal C, the
 * bucket indices of B, Pi2, and explicit sampling uniforms).  See DESIGN.md "Input
 * recipe" and SURVEY.md Appendix B for the stream table.
 *
 * Generator: rng_u64(seed, stream, i) = mix64(key + G*(i+1)), key = mix64(seed + G*(stream+1)),
 * G = 0x9E3779B97F4A7C15 and mix64 the SplitMix64 finaliser -- i.e. the i-th SplitMix64
 * output of a per-stream key.  Every value is a pure function of (seed, stream, index),
 * so any row shard can be regenerated independently.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define FG_GOLDEN 0x9E3779B97F4A7C15ULL
#define FG_PI 3.14159265358979323846

enum { ST_A = 1, ST_ROWMOD = 2, ST_XSTAR = 3, ST_NOISE = 4, ST_SIGN = 5,
       ST_CAUCHY = 6, ST_HASH = 7, ST_PI2 = 8, ST_SAMPLE = 9 };

static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
static inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t key = mix64(seed + FG_GOLDEN * (stream + 1));
  return mix64(key + FG_GOLDEN * (i + 1));
}
static inline uint64_t rng_k(uint64_t key, uint64_t i) { return mix64(key + FG_GOLDEN * (i + 1)); }
static inline uint64_t key_of(uint64_t seed, uint64_t stream) { return mix64(seed + FG_GOLDEN * (stream + 1)); }
static inline double u53(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
static inline double u53o(uint64_t x) { return ((double)(x >> 11) + 0.5) * 0x1.0p-53; }
static inline double cauchy_of(uint64_t x) { return tan(FG_PI * (u53o(x) - 0.5)); }
/* one standard normal per index j from draws 2j, 2j+1 of the stream (cosine branch only) */
static inline double normal_k(uint64_t key, uint64_t j) {
  uint64_t a = rng_k(key, 2 * j), b = rng_k(key, 2 * j + 1);
  return sqrt(-2.0 * log(u53o(a))) * cos(2.0 * FG_PI * u53(b));
}

uint64_t fg_mix64(uint64_t z) { return mix64(z); }
uint64_t fg_rng_u64(uint64_t seed, uint64_t stream, uint64_t i) { return rng(seed, stream, i); }

void fg_rng_block(uint64_t seed, uint64_t stream, int64_t i0, int64_t count, uint64_t* out) {
  uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) out[t] = rng_k(key, (uint64_t)(i0 + t));
}

/* Rademacher diagonal D: signs[row] = (x>>63) ? -1 : +1 (stream 5) */
void fg_signs(uint64_t seed, int64_t row0, int64_t count, int8_t* out) {
  uint64_t key = key_of(seed, ST_SIGN);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) out[t] = (rng_k(key, (uint64_t)(row0 + t)) >> 63) ? (int8_t)-1 : (int8_t)1;
}

/* standard Cauchy draws tan(pi(u-1/2)), u in (0,1), stored as fp32 (streams 6 = C, 8 = Pi2) */
void fg_cauchy(uint64_t seed, uint64_t stream, int64_t idx0, int64_t count, float* out) {
  uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) out[t] = (float)cauchy_of(rng_k(key, (uint64_t)(idx0 + t)));
}

/* bucket index of each H~-row for B: top log2(r1) bits (r1 a power of two), stream 7 */
int fg_hash(uint64_t seed, int64_t idx0, int64_t count, int32_t r1, int32_t* out) {
  if (r1 < 1 || (r1 & (r1 - 1))) return -1;
  int lg = 0; while ((1 << lg) < r1) ++lg;
  uint64_t key = key_of(seed, ST_HASH);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) {
    uint64_t x = rng_k(key, (uint64_t)(idx0 + t));
    out[t] = lg == 0 ? 0 : (int32_t)(x >> (64 - lg));
  }
  return 0;
}

/* explicit sampling uniforms u53(rng(seed, 9, global_row)) */
void fg_uniforms(uint64_t seed, int64_t row0, int64_t count, double* out) {
  uint64_t key = key_of(seed, ST_SAMPLE);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) out[t] = u53(rng_k(key, (uint64_t)(row0 + t)));
}

/* i.i.d. N(0,1) array (stream given), one normal per index */
void fg_normals(uint64_t seed, uint64_t stream, int64_t j0, int64_t count, double* out) {
  uint64_t key = key_of(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < count; ++t) out[t] = normal_k(key, (uint64_t)(j0 + t));
}

/*
 * Test matrix A (n x d, fp32, row-major with leading dimension ld), rows [row0, row0+nrows).
 * kind 1: i.i.d. N(0,1)                                       (config 1)
 * kind 2: 15 (= d-1) N(0,1) features, last column -b,
 *         b = F x* + e, e ~ 0.95 N(0, 0.1^2) + 0.05 * 100 Cauchy  (config 2, P:L1584-1590 style)
 * kind 3: N(0,1) rows scaled by w = min(|Cauchy|^0.5, 1e4)     (config 3)
 * kind 4: N(0,1) rows, each row x1e3 with probability 0.01   (config 4)
 * kind 5: d-1 Student-t(3) features, last column -b, b = F x* + Cauchy (config 5, P:L1625-1647 style)
 * Features are rounded to fp32 first; b is formed in fp64 from the rounded features.
 */
int fg_matrix(int kind, uint64_t seed, int64_t n, int64_t d, int64_t row0, int64_t nrows,
              float* out, int64_t ld) {
  if (kind < 1 || kind > 5 || d < 1 || ld < d || row0 < 0 || row0 + nrows > n) return -1;
  if ((kind == 2 || kind == 5) && d < 2) return -1;
  uint64_t kA = key_of(seed, ST_A), kM = key_of(seed, ST_ROWMOD), kX = key_of(seed, ST_XSTAR),
           kE = key_of(seed, ST_NOISE);
  const int64_t nf = (kind == 2 || kind == 5) ? d - 1 : d;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < nrows; ++t) {
    const int64_t row = row0 + t;
    float* o = out + t * ld;
    double scale = 1.0;
    if (kind == 3) {
      double w = sqrt(fabs(cauchy_of(rng_k(kM, (uint64_t)row))));
      scale = w < 1e4 ? w : 1e4;
    } else if (kind == 4) {
      scale = u53(rng_k(kM, (uint64_t)row)) < 0.01 ? 1e3 : 1.0;
    }
    for (int64_t c = 0; c < nf; ++c) {
      uint64_t i = (uint64_t)(row * d + c);
      double v;
      if (kind == 5) {
        double z0 = normal_k(kA, 4 * i), z1 = normal_k(kA, 4 * i + 1), z2 = normal_k(kA, 4 * i + 2),
               z3 = normal_k(kA, 4 * i + 3);
        v = z0 / sqrt((z1 * z1 + z2 * z2 + z3 * z3) / 3.0);
      } else {
        v = normal_k(kA, i) * scale;
      }
      o[c] = (float)v;
    }
    if (kind == 2 || kind == 5) {
      double b = 0.0;
      for (int64_t c = 0; c < nf; ++c) b += (double)o[c] * normal_k(kX, (uint64_t)c);
      double e;
      if (kind == 2) {
        uint64_t x0 = rng_k(kE, 3 * (uint64_t)row), x1 = rng_k(kE, 3 * (uint64_t)row + 1),
                 x2 = rng_k(kE, 3 * (uint64_t)row + 2);
        if (u53(x0) >= 0.95) e = 100.0 * cauchy_of(x1);
        else e = 0.1 * sqrt(-2.0 * log(u53o(x1))) * cos(2.0 * FG_PI * u53(x2));
      } else {
        e = cauchy_of(rng_k(kE, (uint64_t)row));
      }
      o[nf] = (float)(-(b + e));
    }
  }
  return 0;
}
