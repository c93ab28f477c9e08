/*
 * oracle/rng.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's deterministic RNG
 * (/root/reference/proj/include/coserve/rng.hpp:15-64):
 *   - std::mt19937_64 (bit-exact per the C++ standard; restated here from the
 *     published MT19937-64 algorithm: w=64, n=312, m=156, r=31,
 *     a=0xB5026F5AA96619E9, u=29 d=0x5555555555555555, s=17 b=0x71D67FFFEDA60000,
 *     t=37 c=0xFFF7EEE000000000, l=43, f=6364136223846793005),
 *   - uniform()      rng.hpp:22   (bits >> 11) * 2^-53
 *   - uniform_int()  rng.hpp:26   lo + bits % (hi-lo+1)
 *   - normal()       rng.hpp:30   Box-Muller with cached spare (cos first, sin cached)
 *   - lognormal()    rng.hpp:45, exponential() rng.hpp:47
 *   - randn()        rng.hpp:53   row-major fill of normal()*scale
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NN 312
#define MM 156
#define MATRIX_A 0xB5026F5AA96619E9ULL
#define UM 0xFFFFFFFF80000000ULL
#define LM 0x7FFFFFFFULL

typedef struct {
  uint64_t mt[NN];
  int mti;
  int have_spare;
  double spare;
} orc_rng;

static void mt_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < NN; i++)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = NN;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t mt_next(orc_rng* r) {
  static const uint64_t mag01[2] = {0ULL, MATRIX_A};
  uint64_t x;
  if (r->mti >= NN) {
    int i;
    for (i = 0; i < NN - MM; i++) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < NN - 1; i++) {
      x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MM - NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (r->mt[NN - 1] & UM) | (r->mt[0] & LM);
    r->mt[NN - 1] = r->mt[MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    r->mti = 0;
  }
  x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:22 */
static double u01(orc_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:30-43 */
static double normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = u01(r);
  while (u1 <= 0.0) u1 = u01(r);
  double u2 = u01(r);
  double rad = sqrt(-2.0 * log(u1));
  double theta = 2.0 * M_PI * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

/* ---- exported stateful API (handle = heap orc_rng) ---- */
void* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
  mt_seed(r, seed);
  return r;
}
void orc_rng_free(void* h) { free(h); }
uint64_t orc_rng_bits(void* h) { return mt_next((orc_rng*)h); }
double orc_rng_uniform(void* h) { return u01((orc_rng*)h); }
/* rng.hpp:26-28 (inclusive bounds) */
void orc_rng_uniform_int(void* h, int64_t lo, int64_t hi, int64_t n, int64_t* out) {
  for (int64_t i = 0; i < n; i++)
    out[i] = lo + (int64_t)(mt_next((orc_rng*)h) % (uint64_t)(hi - lo + 1));
}
double orc_rng_normal(void* h) { return normal((orc_rng*)h); }
/* rng.hpp:45 */
double orc_rng_lognormal(void* h, double mu, double sigma) {
  return exp(mu + sigma * normal((orc_rng*)h));
}
/* rng.hpp:47-51 */
double orc_rng_exponential(void* h, double rate) {
  double u = u01((orc_rng*)h);
  while (u <= 0.0) u = u01((orc_rng*)h);
  return -log(u) / rate;
}
/* rng.hpp:53-58 */
void orc_rng_randn(void* h, int64_t rows, int64_t cols, double scale, double* out) {
  for (int64_t i = 0; i < rows * cols; i++) out[i] = normal((orc_rng*)h) * scale;
}
