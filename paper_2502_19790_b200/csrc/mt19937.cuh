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

// ---------------------------------------------------------------------------
// Warp-cooperative form of the same generator (bit-identical output).
//  * seeding: init_genrand(19650218) is seed-independent, so it comes from a
//    precomputed table (`base`); init_by_array's recurrence runs on lane 0
//    with the previous word in a register (the old words are plain loads);
//  * generation: the twist is split into three data-parallel ranges
//    ([0,227) reads only old words, [227,454) reads words of the first range,
//    [454,623) of the second, then word 623) and tempered into `out`;
//  * consumption (rejection sampling + Fisher-Yates swaps) stays on lane 0,
//    reading the 624-output buffer; the warp refills it when drained.
struct WarpMT {
  uint32_t* s;    // state [624]
  uint32_t* out;  // tempered outputs [624]
  int pos;        // next unread output (624 = drained)

  __device__ void seed(const uint32_t* base, unsigned long long seed_v) {
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < MT_N; k += 32) s[k] = base[k];
    __syncwarp();
    if (lane == 0) {
      uint32_t key[2] = {(uint32_t)seed_v, (uint32_t)(seed_v >> 32)};
      const int klen = (seed_v >> 32) ? 2 : 1;
      int a = 1, b = 0;
      uint32_t prev = s[0];
      for (int k = MT_N > klen ? MT_N : klen; k; --k) {
        const uint32_t v = (s[a] ^ ((prev ^ (prev >> 30)) * 1664525u)) + key[b] + (uint32_t)b;
        s[a] = v;
        prev = v;
        ++a; ++b;
        if (a >= MT_N) { s[0] = s[MT_N - 1]; prev = s[0]; a = 1; }
        if (b >= klen) b = 0;
      }
      for (int k = MT_N - 1; k; --k) {
        const uint32_t v = (s[a] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)a;
        s[a] = v;
        prev = v;
        ++a;
        if (a >= MT_N) { s[0] = s[MT_N - 1]; prev = s[0]; a = 1; }
      }
      s[0] = 0x80000000u;
    }
    pos = MT_N;
    __syncwarp();
  }

  __device__ static uint32_t twist_word(uint32_t cur, uint32_t nxt, uint32_t far) {
    const uint32_t y = (cur & 0x80000000u) | (nxt & 0x7fffffffu);
    return far ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
  }

  // words [lo, hi) of the twist in warp-uniform steps of 32: every lane reads
  // (old s[k+1] may be the next lane's word) before any lane writes
  __device__ void twist_range(int lo, int hi) {
    const int lane = threadIdx.x & 31;
    for (int b = lo; b < hi; b += 32) {
      const int k = b + lane;
      const bool ok = k < hi;
      uint32_t v = 0;
      if (ok) v = twist_word(s[k], s[k + 1], k < MT_N - MT_M ? s[k + MT_M] : s[k + (MT_M - MT_N)]);
      __syncwarp();
      if (ok) s[k] = v;
      __syncwarp();
    }
  }

  __device__ void refill() {  // whole warp
    const int lane = threadIdx.x & 31;
    twist_range(0, MT_N - MT_M);                     // reads only old words
    twist_range(MT_N - MT_M, 2 * (MT_N - MT_M));     // reads new [0, 227)
    twist_range(2 * (MT_N - MT_M), MT_N - 1);        // reads new [227, 396)
    if (lane == 0) s[MT_N - 1] = twist_word(s[MT_N - 1], s[0], s[MT_M - 1]);
    __syncwarp();
    for (int k = lane; k < MT_N; k += 32) {
      uint32_t y = s[k];
      y ^= (y >> 11);
      y ^= (y << 7) & 0x9d2c5680u;
      y ^= (y << 15) & 0xefc60000u;
      y ^= (y >> 18);
      out[k] = y;
    }
    pos = 0;
    __syncwarp();
  }

  // random.shuffle(x[0..n)) by the whole warp (lane 0 swaps)
  template <typename T>
  __device__ void shuffle(T* x, int n) {
    const int lane = threadIdx.x & 31;
    int i = n - 1;
    while (i >= 1) {
      if (pos >= MT_N) refill();
      if (lane == 0) {
        int p = pos;
        while (i >= 1 && p < MT_N) {
          const uint32_t bound = (uint32_t)(i + 1);
          const int kb = 32 - __clz(bound);
          const uint32_t r = out[p++] >> (32 - kb);
          if (r < bound) {
            const T t = x[i];
            x[i] = x[r];
            x[r] = t;
            --i;
          }
        }
        pos = p;
      }
      i = __shfl_sync(0xffffffffu, i, 0);
      pos = __shfl_sync(0xffffffffu, pos, 0);
      __syncwarp();
    }
  }
};

// init_genrand(19650218) state, the common starting point of every seeding
inline void mt_base_table(uint32_t* t) {
  t[0] = 19650218u;
  for (int k = 1; k < MT_N; ++k) t[k] = 1812433253u * (t[k - 1] ^ (t[k - 1] >> 30)) + (uint32_t)k;
}

}  // namespace mx
