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

// init_by_array(abs(seed) as 32-bit words) on top of init_genrand(19650218),
// one key per THREAD (mt_seed_kernel): the chain of 1,246
// dependent xor-shift-multiply steps is inherently sequential, so the
// parallelism is across keys. S(a) addresses the thread's state word a (loop
// 2 reads loop 1's words back in the order they were written).
template <typename S>
__device__ __forceinline__ void mt_init_by_array(unsigned long long seed_v, S st) {
  const uint32_t key0 = (uint32_t)seed_v, key1 = (uint32_t)(seed_v >> 32);
  const bool two = key1 != 0u;  // key length 2 (abs(seed) >= 2^32)
  const uint32_t kb0 = key0, kb1 = two ? key1 + 1u : key0;  // key[j] + j
  // loop 1 reads init_genrand(19650218)'s words, which are recomputed here by
  // their own recurrence (an independent chain the scheduler interleaves with
  // the key's, no memory latency on the critical path)
  uint32_t prev = 19650218u, g = 19650218u;
  bool odd = false;
#pragma unroll 16
  for (int a = 1; a < MT_N; ++a) {  // loop 1, i = 1..623 (j = (i - 1) % klen)
    g = 1812433253u * (g ^ (g >> 30)) + (uint32_t)a;
    prev = (g ^ ((prev ^ (prev >> 30)) * 1664525u)) + (odd ? kb1 : kb0);
    st(a) = prev;
    odd = two && !odd;
  }
  st(0) = prev;  // wrap: mt[0] = mt[623], i = 1 (the 624th iteration)
  prev = (st(1) ^ ((prev ^ (prev >> 30)) * 1664525u)) + (odd ? kb1 : kb0);
  st(1) = prev;
  constexpr int U = 16;  // loop 2 reads loop 1's words: 16 loads ahead of 16 steps
  for (int a0 = 2; a0 < MT_N; a0 += U) {  // loop 2, i = 2..623
    uint32_t x[U];
#pragma unroll
    for (int t = 0; t < U; ++t) x[t] = a0 + t < MT_N ? st(a0 + t) : 0u;
#pragma unroll
    for (int t = 0; t < U; ++t) {
      if (a0 + t < MT_N) {
        prev = (x[t] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(a0 + t);
        x[t] = prev;
      }
    }
#pragma unroll
    for (int t = 0; t < U; ++t)
      if (a0 + t < MT_N) st(a0 + t) = x[t];
  }
  st(0) = prev;  // wrap, then i = 1
  st(1) = (st(1) ^ ((prev ^ (prev >> 30)) * 1566083941u)) - 1u;
  st(0) = 0x80000000u;
}

// ---------------------------------------------------------------------------
// Warp-cooperative generator over a seeded state (bit-identical output):
//  * generation: the twist is split into three data-parallel ranges
//    ([0,227) reads only old words, [227,454) reads words of the first range,
//    [454,623) of the second, then word 623) and tempered into `out`;
//  * draws: the _randbelow(i + 1) results j_i of a shuffle (i = n-1..1) are
//    resolved a 128-output window at a time: the number of accepted draws
//    before an output fixes the bound i - A + 1 it is tested against, and
//    A is found by fixed-point iteration (see draws()). No swaps while
//    drawing.
struct WarpMT {
  uint32_t* s;    // state [624]
  uint32_t* out;  // tempered outputs [624]
  int pos;        // next unread output (624 = drained)

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

  // j[i] = _randbelow(i + 1) for i = n-1..1, in stream order (whole warp).
  // DU consecutive outputs per lane (a window of up to 32 * DU outputs, never
  // across a refill): given the accepted count `base` of the earlier lanes,
  // a lane resolves its own outputs in order; `base` is iterated to the fixed
  // point of base = prefix over lanes of their accepted counts (counts < 8:
  // three ballots). A fixed point is the sequential answer (induction over
  // the outputs), and every round makes at least one more lane exact.
  template <typename IT>
  __device__ void draws(int n, IT* j) {
    constexpr int DU = 4;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int i = n - 1;
    while (i >= 1) {
      if (pos >= MT_N) refill();
      uint32_t u[DU];
#pragma unroll
      for (int t = 0; t < DU; ++t) {
        const int o = pos + DU * lane + t;
        u[t] = o < MT_N ? out[o] : 0u;
      }
      const int lim = MT_N - pos - DU * lane;  // valid outputs of this lane (may be <= 0)
      int base = 0, cnt = 0, act = 0;
      uint32_t accm = 0, r[DU];
      for (;;) {
        int A = base;
        cnt = 0;
        act = 0;
        accm = 0;
#pragma unroll
        for (int t = 0; t < DU; ++t) {
          const int ii = i - A;
          r[t] = 0;
          if (t < lim && ii >= 1) {
            ++act;
            const uint32_t bound = (uint32_t)ii + 1u;
            r[t] = u[t] >> __clz(bound);  // getrandbits(bound.bit_length())
            if (r[t] < bound) {
              accm |= 1u << t;
              ++A;
              ++cnt;
            }
          }
        }
        const uint32_t m0 = __ballot_sync(0xffffffffu, cnt & 1), m1 = __ballot_sync(0xffffffffu, cnt & 2),
                       m2 = __ballot_sync(0xffffffffu, cnt & 4);
        const int nb = __popc(m0 & lt) + 2 * __popc(m1 & lt) + 4 * __popc(m2 & lt);
        if (__all_sync(0xffffffffu, nb == base)) break;
        base = nb;
      }
      // accepted outputs: step i - (accepted before it) draws r
      int A = base;
#pragma unroll
      for (int t = 0; t < DU; ++t) {
        if (accm >> t & 1u) {
          j[i - A] = (IT)r[t];
          ++A;
        }
      }
      const uint32_t a0 = __ballot_sync(0xffffffffu, act & 1), a1 = __ballot_sync(0xffffffffu, act & 2),
                     a2 = __ballot_sync(0xffffffffu, act & 4);
      const uint32_t c0 = __ballot_sync(0xffffffffu, cnt & 1), c1 = __ballot_sync(0xffffffffu, cnt & 2),
                     c2 = __ballot_sync(0xffffffffu, cnt & 4);
      pos += __popc(a0) + 2 * __popc(a1) + 4 * __popc(a2);
      i -= __popc(c0) + 2 * __popc(c1) + 4 * __popc(c2);
    }
    __syncwarp();
  }
};

// ---------------------------------------------------------------------------
// Apply the draws to an identity sequence (bit-identical to
// random.shuffle(list(range(n)))), one warp. Fisher-Yates from the end leaves
// x[i] = the value at position j_i just before step i. That value was written
// by the most recent earlier step s > i with j_s = j_i (the next larger member
// of bucket j_i), which moved there the value at position s just before step
// s, and so on:
//   V(s) = head(s) exists ? V(head(s)) : s,  head(s) = min{s' > s : j_s' = s}
//   out[i] = nxt_i exists ? V(nxt_i) : j_i,  nxt_i = min{s > i : j_s = j_i}
//   out[0] = head(0) exists ? V(head(0)) : 0
// Every bucket is built as an ASCENDING linked list (top[p] = its smallest
// step, link(s) = the next larger step of s's bucket, stored over the draw
// j_s) by inserting the steps from n-1 down, 32 at a time; steps of one batch
// that share a bucket are ordered by __match_any_sync. Then nxt_i = link(i)
// and head(p) = top[p], or link(p) when top[p] == p; every element's chain
// is followed independently (mean length ~1, max ~log n). 4 B of scratch per
// element as u16 (n <= 2^15, shared memory), u32 otherwise; the all-ones IT
// marks "none".
// phase 1 (one warp): the ascending bucket lists of steps 1..n-1, built in
// place of the draws: jl[s] holds j_s on entry and, on exit, the next larger
// step of s's bucket, or FLAG | j_s when s is its bucket's largest step (the
// top bit of IT is free: n <= 2^15 for u16, 2^31 for u32). Each batch reads
// its 32 draws before it overwrites them; later batches read smaller steps.
template <typename IT>
__device__ void fy_lists(int n, IT* jl, IT* top) {
  const int lane = threadIdx.x & 31;
  const uint32_t none = (uint32_t)(IT)~0u, flag = (none >> 1) + 1u;
  for (int p = lane; p < n; p += 32) top[p] = (IT)none;
  __syncwarp();
  for (int hi = n - 1; hi >= 1; hi -= 32) {
    const int s = hi - lane;  // descending with the lane
    const bool ok = s >= 1;
    const uint32_t js = ok ? (uint32_t)jl[s] : 0u;
    const uint32_t m = __match_any_sync(0xffffffffu, ok ? js : 0x80000000u | (uint32_t)lane);
    const uint32_t old = ok ? (uint32_t)top[js] : none;
    __syncwarp();
    if (ok) {
      const uint32_t lower = m & ((1u << lane) - 1u);  // same bucket, larger steps
      const uint32_t nx = lower ? (uint32_t)(hi - (31 - __clz(lower))) : old;
      jl[s] = (IT)(nx != none ? nx : (flag | js));
      if ((m >> lane) == 1u) top[js] = (IT)s;  // highest lane = smallest step
    }
    __syncwarp();
  }
}

// phase 2 (any number of threads, element-parallel): every output position
template <typename IT, typename F>
__device__ void fy_resolve(int n, const IT* jl, const IT* top, int tid, int stride, F out) {
  const uint32_t none = (uint32_t)(IT)~0u, flag = (none >> 1) + 1u;
  auto nxt = [&](uint32_t s) -> uint32_t {
    const uint32_t v = jl[s];
    return (v & flag) ? none : v;
  };
  auto head = [&](uint32_t p) -> uint32_t {
    const uint32_t t = top[p];
    return t == p ? nxt(p) : t;
  };
  for (int i = tid; i < n; i += stride) {
    uint32_t h, last = 0;
    if (i == 0) {
      h = head(0);
    } else {
      const uint32_t v = jl[i];
      if (v & flag) {
        h = none;
        last = v & ~flag;  // no later step wrote position j_i: its original value
      } else {
        h = v;
      }
    }
    while (h != none) {
      last = h;
      h = head(h);
    }
    out(i, last);
  }
}

// the whole apply by one warp
template <typename IT, typename F>
__device__ void fy_apply(int n, IT* jl, IT* top, F out) {
  fy_lists(n, jl, top);
  __syncwarp();
  fy_resolve(n, jl, top, threadIdx.x & 31, 32, out);
  __syncwarp();
}

}  // namespace mx
