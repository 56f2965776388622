// BLAKE2b (RFC 7693), unkeyed, 16-byte digest, on device.
//
// The reference seeds every random decision with
//   stable_hash(*parts) = BLAKE2b-128(len8BE(p0) || p0 || len8BE(p1) || ...)
//   first 8 digest bytes, big-endian, & (2^63 - 1)        (seeding.py:18-28)
// Cursor seeds (per realized key, index.py:134) and chunk seeds (per chunk,
// chunks.py:188) are computed here in parallel instead of on the host.
#pragma once
#include <stdint.h>

namespace mx {

__device__ __constant__ static const unsigned long long B2_IV[8] = {
    0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

__device__ __constant__ static const uint8_t B2_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ unsigned long long b2_rotr(unsigned long long x, int n) {
  return (x >> n) | (x << (64 - n));
}

struct Blake2b {
  unsigned long long h[8];
  unsigned long long t;  // bytes compressed so far
  uint8_t buf[128];
  int fill;

  __device__ void init() {
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = B2_IV[i];
    h[0] ^= 0x01010000ull ^ 16ull;  // depth 1, fanout 1, no key, 16-byte digest
    t = 0;
    fill = 0;
  }

  __device__ void compress(bool last) {
    unsigned long long m[16], v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      unsigned long long w = 0;
#pragma unroll
      for (int b = 7; b >= 0; --b) w = (w << 8) | buf[8 * i + b];
      m[i] = w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = h[i];
      v[i + 8] = B2_IV[i];
    }
    v[12] ^= t;
    if (last) v[14] = ~v[14];
#define B2_G(a, b, c, d, x, y)          \
  a = a + b + x; d = b2_rotr(d ^ a, 32); \
  c = c + d;     b = b2_rotr(b ^ c, 24); \
  a = a + b + y; d = b2_rotr(d ^ a, 16); \
  c = c + d;     b = b2_rotr(b ^ c, 63);
    for (int r = 0; r < 12; ++r) {
      const uint8_t* s = B2_SIGMA[r];
      B2_G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
      B2_G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
      B2_G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
      B2_G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
      B2_G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
      B2_G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
      B2_G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
      B2_G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
    }
#undef B2_G
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
  }

  __device__ void byte(uint8_t c) {
    if (fill == 128) {  // only compress a full block once more input arrives
      t += 128;
      compress(false);
      fill = 0;
    }
    buf[fill++] = c;
  }

  __device__ void bytes(const uint8_t* p, long long n) {
    for (long long i = 0; i < n; ++i) byte(p[i]);
  }

  __device__ void len8(unsigned long long n) {
    for (int b = 7; b >= 0; --b) byte((uint8_t)(n >> (8 * b)));
  }

  // stable_hash value: first 8 digest bytes big-endian, masked to 63 bits
  __device__ unsigned long long seed63() {
    t += fill;
    for (int i = fill; i < 128; ++i) buf[i] = 0;
    compress(true);
    unsigned long long d0 = h[0];  // digest bytes 0..7 = little-endian h[0]
    unsigned long long be = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) be = (be << 8) | ((d0 >> (8 * b)) & 0xff);
    return be & ((1ull << 63) - 1);
  }
};

// One-block BLAKE2b-128 (messages of <= 128 bytes) with the whole state in
// registers: the message words come from a caller functor byte(i) over a
// fully unrolled index, the 12 rounds are unrolled so SIGMA indices are
// compile-time. Returns stable_hash's 63-bit seed.
template <typename ByteAt>
__device__ __forceinline__ unsigned long long blake2b_seed63_1block(int len, ByteAt byte_at) {
  unsigned long long m[16], v[16], h0;
#pragma unroll
  for (int w = 0; w < 16; ++w) {
    unsigned long long word = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int i = 8 * w + b;
      const unsigned long long c = i < len ? (unsigned long long)byte_at(i) : 0ull;
      word |= c << (8 * b);
    }
    m[w] = word;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = B2_IV[i];
    v[i + 8] = B2_IV[i];
  }
  v[0] ^= 0x01010000ull ^ 16ull;
  h0 = v[0];
  v[12] ^= (unsigned long long)len;
  v[14] = ~v[14];
  constexpr uint8_t S[12][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
#define B2_G1(a, b, c, d, x, y)          \
  a = a + b + x; d = b2_rotr(d ^ a, 32); \
  c = c + d;     b = b2_rotr(b ^ c, 24); \
  a = a + b + y; d = b2_rotr(d ^ a, 16); \
  c = c + d;     b = b2_rotr(b ^ c, 63);
#pragma unroll
  for (int r = 0; r < 12; ++r) {
    B2_G1(v[0], v[4], v[8], v[12], m[S[r][0]], m[S[r][1]]);
    B2_G1(v[1], v[5], v[9], v[13], m[S[r][2]], m[S[r][3]]);
    B2_G1(v[2], v[6], v[10], v[14], m[S[r][4]], m[S[r][5]]);
    B2_G1(v[3], v[7], v[11], v[15], m[S[r][6]], m[S[r][7]]);
    B2_G1(v[0], v[5], v[10], v[15], m[S[r][8]], m[S[r][9]]);
    B2_G1(v[1], v[6], v[11], v[12], m[S[r][10]], m[S[r][11]]);
    B2_G1(v[2], v[7], v[8], v[13], m[S[r][12]], m[S[r][13]]);
    B2_G1(v[3], v[4], v[9], v[14], m[S[r][14]], m[S[r][15]]);
  }
#undef B2_G1
  const unsigned long long d0 = h0 ^ v[0] ^ v[8];
  unsigned long long be = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) be = (be << 8) | ((d0 >> (8 * b)) & 0xff);
  return be & ((1ull << 63) - 1);
}

// decimal text of a non-negative integer (str(int) in Python)
__device__ __forceinline__ int u64_to_dec(unsigned long long v, uint8_t* out) {
  uint8_t tmp[20];
  int n = 0;
  do {
    tmp[n++] = (uint8_t)('0' + v % 10);
    v /= 10;
  } while (v);
  for (int i = 0; i < n; ++i) out[i] = tmp[n - 1 - i];
  return n;
}

}  // namespace mx
