/*
 * RngStream::standard restatement (TEST INFRASTRUCTURE ONLY; see dpg_oracle.h).
 *
 * std::mt19937_64 (the engine behind RngStream::standard, rng.hpp:42, rng.cpp:15-19) with the
 * standard's published parameters, and the Box-Muller transform of rng.cpp:40-53 including the
 * cached spare. Pinned against the compiled reference (tests/test_oracle_vs_reference.py) and
 * against the C++ standard's check value (10000th output of a default-seeded mt19937_64 is
 * 9981545732273789042).
 */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "dpg_oracle.h"

#define MT_N 312
#define MT_M 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

static _Thread_local char g_err[512];

const char* dpgo_last_error(void) { return g_err; }

void dpgo_set_error(const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

/* std::mersenne_twister_engine::seed(value) */
void dpgo_rng_seed(dpgo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

static void mt_twist(dpgo_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_MATRIX_A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->mti = 0;
}

/* RngStream::next_u64 (rng.cpp:27-35), standard kind */
uint64_t dpgo_rng_next_u64(dpgo_rng* r) {
  if (r->mti >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* RngStream::uniform (rng.cpp:36-38): 53-bit resolution in [0, 1) */
double dpgo_rng_uniform(dpgo_rng* r) {
  return (double)(dpgo_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

/* RngStream::normal (rng.cpp:40-53) */
double dpgo_rng_normal(dpgo_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = (double)((dpgo_rng_next_u64(r) >> 11) + 1) * 0x1.0p-53;
  const double u2 = dpgo_rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
  r->spare = rad * sin(theta);
  r->has_spare = 1;
  return rad * cos(theta);
}

/* RngStream::below (rng.cpp:55-66): rejection sampling, no modulo bias */
uint64_t dpgo_rng_below(dpgo_rng* r, uint64_t n) {
  if (n == 0) {
    dpgo_set_error("RngStream::below requires n > 0");
    return 0;
  }
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x = dpgo_rng_next_u64(r);
  while (x >= limit) x = dpgo_rng_next_u64(r);
  return x % n;
}
