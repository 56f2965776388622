// CPython's random.Random on device: MT19937 seeded through init_by_array
// with the 32-bit little-endian words of abs(seed) (Modules/_randommodule.c
// random_seed / init_by_array), getrandbits(k<=32) = genrand >> (32-k),
// _randbelow(n) = rejection sampling on getrandbits(n.bit_length()), and
// shuffle() = Fisher-Yates from the end (Lib/random.py). Used for the
// RangeCursor dataset/file shuffles (index.py:134-144) and the component
// order (chunks.py:139-141), which must match the reference bit for bit.
#pragma once
#include <stdint.h>

namespace mx {

constexpr int MT_N = 624;
constexpr int MT_M = 397;

struct MT {
  uint32_t* s;  // MT_N words (shared or global memory)
  int i;

  __device__ void init_genrand(uint32_t seed) {
    s[0] = seed;
    for (int k = 1; k < MT_N; ++k) s[k] = 1812433253u * (s[k - 1] ^ (s[k - 1] >> 30)) + (uint32_t)k;
    i = MT_N;
  }

  __device__ void seed_u64(unsigned long long seed) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int klen = (seed >> 32) ? 2 : 1;
    init_genrand(19650218u);
    int a = 1, b = 0;
    for (int k = MT_N > klen ? MT_N : klen; k; --k) {
      s[a] = (s[a] ^ ((s[a - 1] ^ (s[a - 1] >> 30)) * 1664525u)) + key[b] + (uint32_t)b;
      ++a; ++b;
      if (a >= MT_N) { s[0] = s[MT_N - 1]; a = 1; }
      if (b >= klen) b = 0;
    }
    for (int k = MT_N - 1; k; --k) {
      s[a] = (s[a] ^ ((s[a - 1] ^ (s[a - 1] >> 30)) * 1566083941u)) - (uint32_t)a;
      ++a;
      if (a >= MT_N) { s[0] = s[MT_N - 1]; a = 1; }
    }
    s[0] = 0x80000000u;
    i = MT_N;
  }

  __device__ void twist() {
    const uint32_t UP = 0x80000000u, LO = 0x7fffffffu, MAG = 0x9908b0dfu;
    int k = 0;
    for (; k < MT_N - MT_M; ++k) {
      uint32_t y = (s[k] & UP) | (s[k + 1] & LO);
      s[k] = s[k + MT_M] ^ (y >> 1) ^ ((y & 1u) ? MAG : 0u);
    }
    for (; k < MT_N - 1; ++k) {
      uint32_t y = (s[k] & UP) | (s[k + 1] & LO);
      s[k] = s[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1u) ? MAG : 0u);
    }
    uint32_t y = (s[MT_N - 1] & UP) | (s[0] & LO);
    s[MT_N - 1] = s[MT_M - 1] ^ (y >> 1) ^ ((y & 1u) ? MAG : 0u);
    i = 0;
  }

  __device__ __forceinline__ uint32_t next() {
    if (i >= MT_N) twist();
    uint32_t y = s[i++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
  }

  // _randbelow_with_getrandbits(n), n >= 1 (n < 2^32)
  __device__ __forceinline__ uint32_t below(uint32_t n) {
    const int k = 32 - __clz(n);  // n.bit_length()
    uint32_t r = next() >> (32 - k);
    while (r >= n) r = next() >> (32 - k);
    return r;
  }

  template <typename T>
  __device__ void shuffle(T* x, int n) {
    for (int i2 = n - 1; i2 >= 1; --i2) {
      uint32_t j = below((uint32_t)(i2 + 1));
      T t = x[i2];
      x[i2] = x[j];
      x[j] = t;
    }
  }
};

}  // namespace mx
