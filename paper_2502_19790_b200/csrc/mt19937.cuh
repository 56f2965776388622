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
//    precomputed table (`base`); init_by_array's sequential recurrence runs
//    on EVERY lane in lockstep, 32 old words at a time loaded lane-parallel
//    and broadcast by shuffles, so only the xor-shift-multiply chain is on
//    the critical path (no shared-memory round trip per step);
//  * generation: the twist is split into three data-parallel ranges
//    ([0,227) reads only old words, [227,454) reads words of the first range,
//    [454,623) of the second, then word 623) and tempered into `out`;
//  * rejection sampling is resolved 32 draws at a time: lane l takes output
//    pos+l and the number A_l of accepted draws before it (which fixes the
//    bound i - A_l + 1 it is tested against) is found by fixed-point
//    iteration of A = prefix_popcount(accept(A)) -- after s rounds lanes
//    0..s are exact, and a fixed point IS the sequential answer;
//  * the Fisher-Yates swaps of the accepted draws run on lane 0 from a
//    shared-memory pair list with the next pair prefetched.
struct WarpMT {
  uint32_t* s;    // state [624]
  uint32_t* out;  // tempered outputs [624]
  uint2* pairs;   // [32] accepted (i, j) of one window
  int pos;        // next unread output (624 = drained)

  // s[a] = f(s[a], prev, t) for a in [a0, a1), t = (a - a0) & 31 (compile-time
  // in full batches); every lane runs the chain, lane t keeps word a0+32m+t
  template <typename F>
  __device__ __forceinline__ uint32_t chain(int a0, int a1, uint32_t prev, F f) {
    const int lane = threadIdx.x & 31;
    int b = a0;
    for (; b + 32 <= a1; b += 32) {
      const uint32_t mine = s[b + lane];
      uint32_t sv[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) sv[t] = __shfl_sync(0xffffffffu, mine, t);
      uint32_t res = 0;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        prev = f(sv[t], prev, b + t, t);
        res = lane == t ? prev : res;
      }
      s[b + lane] = res;
    }
    if (b < a1) {  // tail batch
      const int a = b + lane;
      const uint32_t mine = a < a1 ? s[a] : 0u;
      uint32_t res = 0;
      for (int t = 0; t < a1 - b; ++t) {
        prev = f(__shfl_sync(0xffffffffu, mine, t), prev, b + t, t);
        res = lane == t ? prev : res;
      }
      if (a < a1) s[a] = res;
    }
    __syncwarp();
    return prev;
  }

  __device__ void seed(const uint32_t* base, unsigned long long seed_v) {
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < MT_N; k += 32) s[k] = base[k];
    __syncwarp();
    const uint32_t key0 = (uint32_t)seed_v, key1 = (uint32_t)(seed_v >> 32);
    // init_by_array adds key[b] + b with b = k % klen (k = a - 1 in loop 1):
    // batches start at a = 1 + 32m, so b = t & 1 when klen = 2
    const uint32_t kb0 = key0, kb1 = key1 ? key1 + 1u : key0;
    auto f1 = [&](uint32_t sv, uint32_t prev, int, int t) {
      return (sv ^ ((prev ^ (prev >> 30)) * 1664525u)) + ((t & 1) ? kb1 : kb0);
    };
    auto f2 = [](uint32_t sv, uint32_t prev, int a, int) {
      return (sv ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)a;
    };
    uint32_t prev = chain(1, MT_N, base[0], f1);  // init_by_array loop 1, a = 1..623
    // wrap (s[0] = s[623]), then iteration 623 at a = 1 (b = 623 % klen)
    {
      const uint32_t v = (s[1] ^ ((prev ^ (prev >> 30)) * 1664525u)) + kb1;
      __syncwarp();
      if (lane == 0) { s[0] = prev; s[1] = v; }
      prev = v;
      __syncwarp();
    }
    prev = chain(2, MT_N, prev, f2);  // loop 2, a = 2..623
    {
      const uint32_t v = (s[1] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - 1u;  // wrap, a = 1
      __syncwarp();
      if (lane == 0) { s[1] = v; s[0] = 0x80000000u; }
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

  // random.shuffle(x[0..n)) by the whole warp
  template <typename T>
  __device__ void shuffle(T* x, int n) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int i = n - 1;
    while (i >= 1) {
      if (pos >= MT_N) refill();
      const bool valid = pos + lane < MT_N;
      const uint32_t u = valid ? out[pos + lane] : 0u;
      uint32_t A = 0, acc_mask, act_mask, r = 0;
      for (;;) {  // fixed point: A = accepted draws before this lane
        const int ii = i - (int)A;
        const bool active = valid && ii >= 1;
        bool acc = false;
        if (active) {
          const uint32_t bound = (uint32_t)ii + 1u;
          r = u >> __clz(bound);  // getrandbits(bound.bit_length())
          acc = r < bound;
        }
        acc_mask = __ballot_sync(0xffffffffu, acc);
        const uint32_t A2 = __popc(acc_mask & lt);
        if (__all_sync(0xffffffffu, A2 == A)) {
          act_mask = __ballot_sync(0xffffffffu, active);
          if (acc) pairs[A] = make_uint2((uint32_t)ii, r);
          break;
        }
        A = A2;
      }
      const int m = __popc(acc_mask);
      __syncwarp();
      // the window's swaps k = 0..m-1 touch x[i-k] and x[j_k] (j_k <= i-k).
      // Swap k commutes with all earlier ones unless an earlier swap touched
      // one of its positions: j_k' == j_k, or j_k' == i-k (k' < k). Each
      // round runs the conflict-free prefix in parallel, one lane per swap.
      const bool mine = lane < m;
      const uint2 pr = mine ? pairs[lane] : make_uint2(0u, 0u);
      int k0 = 0;
      while (k0 < m) {
        const bool live = mine && lane >= k0;
        // earlier live lane with the same j
        const uint32_t same = __match_any_sync(0xffffffffu, live ? pr.y : 0xffffffffu);
        uint32_t conflict = __ballot_sync(0xffffffffu, live && (same & ((1u << lane) - 1u) & ~((1u << k0) - 1u)));
        // a live lane whose j equals a LATER live lane's top i - k
        const int hit = (int)((uint32_t)i - pr.y);  // lane whose top is j
        const uint32_t hm = (live && hit > lane && hit < m) ? (1u << hit) : 0u;
        conflict |= __reduce_or_sync(0xffffffffu, hm);
        const int k1 = conflict ? __ffs(conflict) - 1 : m;  // first lane that must wait
        if (live && lane < k1) {
          const T a = x[pr.x], b = x[pr.y];
          x[pr.x] = b;
          x[pr.y] = a;
        }
        __syncwarp();
        k0 = k1;
      }
      pos += __popc(act_mask);
      i -= m;
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
