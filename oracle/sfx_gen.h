/* TEST INFRASTRUCTURE — deterministic synthetic-input generator shared by the
 * oracle (C), the reference-side tools (oracle/ref_tools) and the Python tests
 * (numpy restatement in tests/sfx_testlib.py).  Not part of the product path.
 *
 * The reference fills inputs with std::mt19937_64 + uniform_real_distribution
 * (tests/support.cpp:286-298, tools/stitchfuse.cpp:73-80).  That stream is
 * libstdc++-specific, so parity fixtures use this splitmix64 stream instead,
 * which numpy reproduces bit-for-bit:
 *
 *   key      = splitmix64(seed * 0x100000001B3 + tensor_index)
 *   h_i      = splitmix64(key + i)
 *   f32 value = lo + (hi - lo) * ((float)(h_i >> 40) * 2^-24)   (fp32 ops, no FMA)
 *   i32 value = 1 + (h_i >> 62)                                   (in [1, 4], like
 *                                                                  support.cpp:289)
 * tensor_index = position of the Parameter among the graph's Parameters in
 * instruction order.
 */
#ifndef SFX_GEN_H
#define SFX_GEN_H

#include <stdint.h>

static inline uint64_t sfx_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint64_t sfx_gen_key(uint64_t seed, uint64_t tensor_index) {
  return sfx_splitmix64(seed * 0x100000001B3ull + tensor_index);
}

static inline void sfx_gen_f32(uint64_t seed, uint64_t tensor_index, float lo, float hi,
                               float* out, int64_t n) {
  uint64_t key = sfx_gen_key(seed, tensor_index);
  float span = hi - lo; /* build with -ffp-contract=off: fp32 rounding identical to numpy */
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = sfx_splitmix64(key + (uint64_t)i);
    float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    float p = span * u;
    out[i] = lo + p;
  }
}

static inline void sfx_gen_i32(uint64_t seed, uint64_t tensor_index, int32_t* out, int64_t n) {
  uint64_t key = sfx_gen_key(seed, tensor_index);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = sfx_splitmix64(key + (uint64_t)i);
    out[i] = 1 + (int32_t)(h >> 62);
  }
}

#endif /* SFX_GEN_H */
