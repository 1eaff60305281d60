/* C helpers of the restated CPU oracle. TEST INFRASTRUCTURE ONLY: imported by
 * oracle/coconet_oracle.py as the checker for the CUDA path; never linked into
 * the product.
 *
 * Each function restates one reference routine bit-for-bit:
 *   co_fnv1a            <- ccopt::fnv1a            types.hpp:161-170
 *   co_counter_uniform  <- ccopt::counter_uniform  expr.hpp:15-23
 *   co_gen_range        <- gen_decl_values inner loop, state.hpp:62-71
 *   co_dropout_keep_range <- dropout_keep          expr.hpp:25-27
 */
#include <stdint.h>
#include <stddef.h>

uint64_t co_fnv1a(const void* data, int64_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (int64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

static inline uint64_t mix(uint64_t seed, uint64_t key, uint64_t index) {
  uint64_t x = seed ^ (key * 0x9e3779b97f4a7c15ull) ^ (index + 0x632be59bd9b4e019ull);
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

double co_counter_uniform(uint64_t seed, uint64_t key, uint64_t index) {
  return (double)(mix(seed, key, index) >> 11) * (1.0 / 9007199254740992.0);
}

/* out[i] = float(0.1 + 0.8 * u(seed, key, gidx[i])) for an explicit index list
 * (gidx == NULL means gidx[i] = g0 + i). */
void co_gen_range(uint64_t seed, uint64_t key, const int64_t* gidx, int64_t g0, int64_t n,
                  float* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t g = gidx ? (uint64_t)gidx[i] : (uint64_t)(g0 + i);
    out[i] = (float)(0.1 + 0.8 * co_counter_uniform(seed, key, g));
  }
}

void co_dropout_keep_range(uint64_t seed, uint64_t key, const int64_t* gidx, int64_t g0,
                           int64_t n, double rate, uint8_t* keep) {
  for (int64_t i = 0; i < n; ++i) {
    uint64_t g = gidx ? (uint64_t)gidx[i] : (uint64_t)(g0 + i);
    keep[i] = co_counter_uniform(seed, key, g) >= rate;
  }
}
