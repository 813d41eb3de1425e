/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.  Parity oracle for the B200
 * dense-block path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load liboracle.so; the product never links it.
 *
 * Plain-C restatement of the reference (denseplan) dense-block forward and
 * backward, see dp_oracle_impl.h for the per-function citations.  Pinned
 * against golden vectors produced by the reference itself (oracle/_ref,
 * built from /root/reference/proj/include by oracle/Makefile; fixtures in
 * tests/golden/ made by oracle/gen_golden.py).
 *
 * Flat per-block parameter layout (reference registration order,
 * dp/graph.hpp:459-478 → make_bn / make_conv push order), for layer l with
 * c = c0 + l*k input channels:
 *     gamma_a[c] beta_a[c] W1[bk][c] gamma_b[bk] beta_b[bk] W2[k][bk][3][3]
 * Statistics / running-statistics layout per layer:
 *     mean_a[c] var_a[c] mean_b[bk] var_b[bk]
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no -march=native,
 * so float arithmetic is never contracted into FMAs — same flags as _ref).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define R float
#define SQRT sqrtf
#define FN(name) dpo_##name##_f32
#include "dp_oracle_impl.h"
#undef R
#undef SQRT
#undef FN

#define R double
#define SQRT sqrt
#define FN(name) dpo_##name##_f64
#include "dp_oracle_impl.h"
#undef R
#undef SQRT
#undef FN

/* ---- Rng: dp/rng.hpp:14-64 ------------------------------------------------
 * std::mt19937_64 (bit stream fixed by the C++ standard, restated here),
 * 53-bit uniform, Box-Muller normal with a cached spare. */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} dpo_rng;

void dpo_rng_init(dpo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t dpo_rng_u64(dpo_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  if (r->idx >= 312) {
    int i;
    for (i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= MATRIX_A;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

double dpo_rng_uniform(dpo_rng* r) {
  return (double)(dpo_rng_u64(r) >> 11) * 0x1.0p-53;
}

double dpo_rng_normal(dpo_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = dpo_rng_uniform(r);
  double u2 = dpo_rng_uniform(r);
  while (u1 <= 0.0) u1 = dpo_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

/* make_input (t/graph_test.cpp:21-30): NCHW order normal draws. */
void dpo_fill_normal_f64(uint64_t seed, double* out, int64_t count) {
  dpo_rng r;
  dpo_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = dpo_rng_normal(&r);
}
void dpo_fill_normal_f32(uint64_t seed, float* out, int64_t count) {
  dpo_rng r;
  dpo_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = (float)dpo_rng_normal(&r);
}

void dpo_rng_u64_fill(uint64_t seed, uint64_t* out, int64_t count) {
  dpo_rng r;
  dpo_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = dpo_rng_u64(&r);
}
