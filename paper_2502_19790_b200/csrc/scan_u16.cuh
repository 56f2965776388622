// Stage-1 streaming pass for ONE u16 code column (the row-tuple layout, the
// bench's layout), included by stage1.cu.
//
// At 2 bytes per sample the per-sample work has to be a few instructions or
// the pass is issue bound, not HBM bound. A sample can only start or end a
// run where its tuple code differs from its predecessor's (distinct tuples
// have distinct full keys) or at a file start, so the common path never
// touches the key LUT:
//
//  * the unit of work is a WARP SEGMENT of 2048 consecutive samples (no
//    CTA-wide synchronisation anywhere). Eight coalesced 16-byte loads per
//    lane (ld.global.nc.L1::no_allocate.v4; load k covers samples
//    [k*256, (k+1)*256)) land in per-warp shared memory with an XOR swizzle
//    of the 16-byte chunks (chunk c at c ^ ((c >> 3) & 7)), so that lane L
//    then reads back its 64 CONTIGUOUS samples [64L, 64L + 64) with eight
//    conflict-free 16-byte loads: candidates come out lane-major = in sample
//    order, with one warp scan of the per-lane counts;
//  * code changes come from __byte_perm'ed predecessor words, an XOR and a
//    carry trick that turns every nonzero 16-bit half into one bit, gathered
//    four at a time by one multiply (a 64-bit candidate mask per lane, ~3.3
//    instructions per sample); file starts (from the segment's file range)
//    are OR-ed in;
//  * one lane per candidate reads the two keys from the LUT (staged per CTA)
//    and decides whether it is a real boundary -- a key change with either
//    side passing the filter, a pass / fail switch, or a file start next to a
//    passing sample -- and whether it starts a record (its sample passes).
//    Ballots give each record its slot and its end: the next real boundary
//    (or the segment end, or later: slot_fixup_kernel).
//
// 2048-sample segments halve the per-sample share of the per-segment work
// (loads, halo, file starts, the scan, the tile outputs) against 1024.
// Persistent CTAs; each warp walks segments grid-stride and keeps the next
// segment's loads in flight while finishing the current one. Output follows
// the slot contract of the other stage-1 kernels with tile_len = 2048:
// records at [seg * 2048, ...), tile_cnt / tile_open / tile_head per segment.
#pragma once

namespace mx {

constexpr int SEG_LEN = 2048;        // samples per warp segment
constexpr int U16_WARPS = 4;         // warps per CTA
constexpr int U16_SMEM_LUT_MAX = 16384;

struct U16Warp {                     // per-warp shared scratch
  uint16_t codes[SEG_LEN];           // the segment's codes, 16-byte chunks swizzled (u16_chunk)
  uint16_t ev[SEG_LEN];              // candidate boundaries (segment offsets < 2048), sample order;
                                     // bit 11: a file starts there; pass 1 adds bit 14 (real
                                     // boundary), bit 15 (starts a record)
};

constexpr u32 EV_IDX = 0x7ffu, EV_FS = 0x800u;

// physical 16-byte chunk of logical chunk c (8 codes) in U16Warp::codes
__device__ __forceinline__ int u16_chunk(int c) { return c ^ ((c >> 3) & 7); }
__device__ __forceinline__ u32 u16_code(const U16Warp& W, int idx) {
  return W.codes[u16_chunk(idx >> 3) * 8 + (idx & 7)];
}

// file index of every segment's first sample (galloping search from the
// uniform-size estimate); seg_fa[nseg] = file of sample n - 1
__global__ void seg_file_kernel(const long long* file_off, int n_files, long long n, long long nseg, int* seg_fa) {
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s > nseg) return;
  const long long x = s < nseg ? s * SEG_LEN : n - 1;
  // largest f with file_off[f] <= x (files may be empty: duplicate offsets)
  long long lo = 0, hi = n_files;  // invariant: off[lo] <= x < off[hi] (off[n_files] = n > x)
  long long g = (long long)((double)x / (double)n * (double)n_files);
  g = g < 0 ? 0 : (g >= n_files ? n_files - 1 : g);
  long long step = 1;
  if (file_off[g] <= x) {
    lo = g;
    while (lo + step < n_files && file_off[lo + step] <= x) { lo += step; step <<= 1; }
    hi = lo + step < n_files ? lo + step : n_files;
  } else {
    hi = g;
    while (hi - step > 0 && file_off[hi - step] > x) { hi -= step; step <<= 1; }
    lo = hi - step > 0 ? hi - step : 0;
  }
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (file_off[mid] <= x) lo = mid; else hi = mid;
  }
  seg_fa[s] = (int)lo;
}

// key of a tuple code: LUT 0 = global u32, 1 = shared u32, 2 = shared u16
// (packed keys < 2^15: a failing tuple is clamped to 0xffff >= fail_limit --
// two failing neighbours then compare equal, which never makes a boundary
// real since neither side passes)
template <int LUT>
__device__ __forceinline__ u32 u16_key(const void* s_lut, const u32* g_lut, u32 code) {
  if (LUT == 2) return reinterpret_cast<const uint16_t*>(s_lut)[code];
  if (LUT == 1) return reinterpret_cast<const u32*>(s_lut)[code];
  return __ldg(g_lut + code);
}

template <int LUT>
__device__ __forceinline__ u32 lop3(u32 a, u32 b, u32 c) {
  u32 r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
}

// change flags of the two samples of word w (code before it: high half of
// p): bit 15 = low half differs from its predecessor, bit 31 = high half
// differs. d = w ^ (w << 16 | p >> 16); ((d & 0x7fff7fff) + 0x7fff7fff) | d
// sets the top bit of every nonzero half (3 instructions with fused LOP3s).
__device__ __forceinline__ u32 change2(u32 p, u32 w) {
  const u32 sh = __byte_perm(p, w, 0x5432);
  const u32 y = lop3<0x28>(w, sh, 0x7fff7fffu) + 0x7fff7fffu;  // ((w ^ sh) & c) + c
  return lop3<0xF6>(y, w, sh);                                 // y | (w ^ sh)
}

// 4 flags (top bits of bytes 1 and 3 of t0, t1 = samples 0..3) placed at
// bits [POS, POS + 4) of acc: one PRMT, then the top bits of the four bytes
// gathered by one multiply (bit 7 + 8j lands on bit 28 + j, no carries)
template <int POS>
__device__ __forceinline__ u32 gather4(u32 t0, u32 t1, u32 acc) {
  const u32 u = __byte_perm(t0, t1, 0x7531) & 0x80808080u;
  const u32 q = (u * 0x00204081u) >> (28 - POS);
  return lop3<0xEA>(q, 0xFu << POS, acc);  // (q & mask) | acc
}

// 32-bit change mask of 32 consecutive samples (words w[0..3], 8 codes
// each) given the code before them in the high half of prev
__device__ __forceinline__ u32 change32(u32 prev, const uint4* w) {
  u32 m = 0, p = prev;
#define MX_C8(K)                                                                     \
  {                                                                                  \
    const u32 t0 = change2(p, w[K].x), t1 = change2(w[K].x, w[K].y);                 \
    const u32 t2 = change2(w[K].y, w[K].z), t3 = change2(w[K].z, w[K].w);            \
    m = gather4<8 * K>(t0, t1, m);                                                   \
    m = gather4<8 * K + 4>(t2, t3, m);                                               \
    p = w[K].w;                                                                      \
  }
  MX_C8(0) MX_C8(1) MX_C8(2) MX_C8(3)
#undef MX_C8
  return m;
}

template <int SLUT>
__global__ void __launch_bounds__(U16_WARPS * 32, 5)
scan_u16_kernel(S1Args a, const int* __restrict__ seg_fa, long long nseg) {
  extern __shared__ __align__(16) unsigned char u16_dyn[];
  U16Warp* wsm = reinterpret_cast<U16Warp*>(u16_dyn);
  void* s_lut = u16_dyn + sizeof(U16Warp) * U16_WARPS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  U16Warp& W = wsm[warp];
  const uint16_t* __restrict__ col = reinterpret_cast<const uint16_t*>(a.cols[0]);
  const u32* __restrict__ g_lut = a.lut_sum + 1;  // entry of code c at c (a tuple column has no null code)
  const u32 lim = a.fail_limit;
  const long long n = a.n;
  if (SLUT == 1)
    for (int i = threadIdx.x; i < a.lut_off[1] - 1; i += U16_WARPS * 32) reinterpret_cast<u32*>(s_lut)[i] = g_lut[i];
  if (SLUT == 2)
    for (int i = threadIdx.x; i < a.lut_off[1] - 1; i += U16_WARPS * 32)
      reinterpret_cast<uint16_t*>(s_lut)[i] = (uint16_t)min(g_lut[i], 0xffffu);
  __syncthreads();  // the only CTA barrier: LUT staged
  const long long wstride = (long long)gridDim.x * U16_WARPS;
  long long seg = (long long)blockIdx.x * U16_WARPS + warp;
  // prefetched state of the next segment
  uint4 w[8];
  u32 halo = 0;  // lane 0: code before the segment; lane 31: code after it
  int fa = 0, fa_next = 0;
  auto fetch = [&](long long sg) {
    const long long s0 = sg * SEG_LEN;
    if (s0 + SEG_LEN <= n) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int4 v = ld_stream_v4(reinterpret_cast<const int4*>(col + s0 + k * 256 + lane * 8));
        w[k] = make_uint4((u32)v.x, (u32)v.y, (u32)v.z, (u32)v.w);
      }
    } else {  // partial last segment: scalar loads, the last code repeated past n (no candidates there)
      const u32 last = col[n - 1];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        u32 h[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long i = s0 + k * 256 + lane * 8 + j;
          h[j] = i < n ? (u32)col[i] : last;
        }
        w[k] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
      }
    }
    if (lane == 0) halo = s0 > 0 ? (u32)__ldg(col + s0 - 1) : 0u;
    if (lane == 31) halo = s0 + SEG_LEN < n ? (u32)__ldg(col + s0 + SEG_LEN) : 0u;
    fa = __ldg(seg_fa + sg);
    fa_next = __ldg(seg_fa + sg + 1);
  };
  if (seg < nseg) fetch(seg);
  for (; seg < nseg; seg += wstride) {
    const long long s0 = seg * SEG_LEN;
    const int len = (int)(n - s0 < SEG_LEN ? n - s0 : SEG_LEN);
    // ---- codes to shared memory (swizzled chunks), then the next segment's loads
#pragma unroll
    for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4*>(&W.codes[u16_chunk(k * 32 + lane) * 8]) = w[k];
    const u32 chalo = halo;
    const int cfa = fa;
    const int nf = fa_next - fa;  // file starts in (s0, s0 + 2048] ((s0, n) for the last segment)
    const long long nxt = seg + wstride;
    if (nxt < nseg) fetch(nxt);
    __syncwarp();
    // ---- this lane's 64 contiguous samples [64 lane, 64 lane + 64)
    uint4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = *reinterpret_cast<const uint4*>(&W.codes[((8 * lane + k) ^ (lane & 7)) * 8]);
    const u32 hprev = __shfl_sync(MX_FULL, chalo, 0);  // code before the segment
    const u32 up = __shfl_up_sync(MX_FULL, x[7].w, 1);  // the previous lane's last code, high half
    u32 m0 = change32(lane > 0 ? up : hprev << 16, x);
    u32 m1 = change32(x[3].w, x + 4);
    if (s0 == 0 && lane == 0) m0 |= 1u;  // sample 0: no predecessor
    // ---- file starts in (s0, s0 + len): this lane's 64-bit mask, 32 starts
    // per round (one per lane, then broadcast)
    const long long fbase = __ldg(a.file_off + cfa);  // start of the file holding s0
    u32 f0 = 0, f1 = 0;
    for (int k0 = 1; k0 <= nf; k0 += 32) {
      const int k = k0 + lane;
      const long long p = k <= nf ? __ldg(a.file_off + cfa + k) - s0 : -1;
      const int pi = p > 0 && p < len ? (int)p : -1;
      const int cnt = nf - k0 + 1 < 32 ? nf - k0 + 1 : 32;
      for (int t = 0; t < cnt; ++t) {
        const int q = __shfl_sync(MX_FULL, pi, t) - 64 * lane;
        if (q >= 0 && q < 32) f0 |= 1u << q;
        else if (q >= 32 && q < 64) f1 |= 1u << (q - 32);
      }
    }
    const bool fs0 = s0 > 0 && fbase == s0;  // a file starts at the segment's first sample
    if (fs0 && lane == 0) f0 |= 1u;
    m0 |= f0;
    m1 |= f1;
    // ---- candidates in sample order (lane-major): one warp scan of the counts
    const u32 cnt = (u32)(__popc(m0) + __popc(m1));
    const u32 incl = warp_incl_scan(cnt);
    const int nev = (int)__shfl_sync(MX_FULL, incl, 31);
    {
      u32 p = incl - cnt;
      for (u32 c = m0; c; c &= c - 1) {
        const int b = __ffs(c) - 1;
        W.ev[p++] = (uint16_t)(64 * lane + b + (((f0 >> b) & 1u) ? EV_FS : 0u));
      }
      for (u32 c = m1; c; c &= c - 1) {
        const int b = __ffs(c) - 1;
        W.ev[p++] = (uint16_t)(64 * lane + 32 + b + (((f1 >> b) & 1u) ? EV_FS : 0u));
      }
    }
    __syncwarp();
    // ---- candidate -> (real boundary, starts a record)
    auto classify = [&](u32 ev, bool& real, bool& rec) {
      const int idx = (int)(ev & EV_IDX);
      const u32 kc = u16_key<SLUT>(s_lut, g_lut, u16_code(W, idx));
      const bool pc = kc < lim;
      if (s0 + idx == 0) {
        real = pc;
      } else {
        const u32 pre = idx > 0 ? u16_code(W, idx - 1) : hprev;
        const u32 kp = u16_key<SLUT>(s_lut, g_lut, pre);
        const bool fs = (ev & EV_FS) != 0;
        real = (pc || kp < lim) && (fs || kc != kp);
      }
      rec = real && pc;
    };
    // ---- segment end: is sample s0 + len a boundary of the run holding s0 + len - 1?
    bool end_real = true;
    {
      const u32 last = __shfl_sync(MX_FULL, x[7].w >> 16, 31);
      const u32 after = __shfl_sync(MX_FULL, chalo, 31);
      if (s0 + len < n) {  // len == 2048 here
        const u32 kl = u16_key<SLUT>(s_lut, g_lut, last);
        const u32 kn = u16_key<SLUT>(s_lut, g_lut, after);
        const bool fs_end = nf > 0 && __ldg(a.file_off + cfa + nf) == s0 + SEG_LEN;
        end_real = fs_end || kl != kn;
      }
    }
    // ---- a record [idx, end) in slot r (end < 0: continues past the segment)
    const u64 sbase = (u64)seg * SEG_LEN;
    auto store = [&](int idx, int end, u32 r) {
      // file of the run: fa + the segment's file starts at or before it
      int lo = 0, hi = nf;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(a.file_off + cfa + mid) <= s0 + idx) lo = mid; else hi = mid - 1;
      }
      const long long fstart = lo ? __ldg(a.file_off + cfa + lo) : fbase;
      const u32 key = u16_key<SLUT>(s_lut, g_lut, u16_code(W, idx));
      const u32 off = (u32)(s0 - fstart);
      a.rec_key[sbase + r] = key;
      a.rec_file[sbase + r] = (u32)(cfa + lo);
      a.rec_start[sbase + r] = off + (u32)idx;
      if (end >= 0) a.rec_end[sbase + r] = off + (u32)end;
      if ((key & a.rank_mask) == 0) atomicMin(&a.err->null_key_sample, (u64)(s0 + idx));
    };
    const int seg_end = end_real ? len : -1;  // -1: the run continues past the segment
    const u32 above = ~((2u << lane) - 1u), below = (1u << lane) - 1u;
    u32 rtot = 0;
    int first_real = -1;
    bool open = false;
    if (nev <= 64) {
      // ---- common case: every candidate in registers (two per lane), no
      // shared flags, one pass
      const bool ok0 = lane < nev, ok1 = 32 + lane < nev;
      const u32 ev0 = ok0 ? (u32)W.ev[lane] : 0u, ev1 = ok1 ? (u32)W.ev[32 + lane] : 0u;
      const int idx0 = (int)(ev0 & EV_IDX), idx1 = (int)(ev1 & EV_IDX);
      bool real0 = false, rec0 = false, real1 = false, rec1 = false;
      if (ok0) classify(ev0, real0, rec0);
      if (ok1) classify(ev1, real1, rec1);
      const u32 realb0 = __ballot_sync(MX_FULL, real0), recb0 = __ballot_sync(MX_FULL, rec0);
      const u32 realb1 = __ballot_sync(MX_FULL, real1), recb1 = __ballot_sync(MX_FULL, rec1);
      const int r0 = __ffs(realb0) - 1, r1 = __ffs(realb1) - 1;
      const int after0 = __ffs(realb0 & above) - 1, after1 = __ffs(realb1 & above) - 1;
      const int nx0 = __shfl_sync(MX_FULL, idx0, after0 >= 0 ? after0 : lane);
      const int nx1 = __shfl_sync(MX_FULL, idx1, after1 >= 0 ? after1 : lane);
      const int fr0 = __shfl_sync(MX_FULL, idx0, r0 >= 0 ? r0 : 0);
      const int fr1 = __shfl_sync(MX_FULL, idx1, r1 >= 0 ? r1 : 0);
      const int next1 = seg_end;                     // after the last candidate
      const int next0 = r1 >= 0 ? fr1 : seg_end;     // after half 0
      if (rec0) store(idx0, after0 >= 0 ? nx0 : next0, (u32)__popc(recb0 & below));
      if (rec1) store(idx1, after1 >= 0 ? nx1 : next1, (u32)(__popc(recb0) + __popc(recb1 & below)));
      rtot = (u32)(__popc(recb0) + __popc(recb1));
      first_real = r0 >= 0 ? fr0 : (r1 >= 0 ? fr1 : -1);
      // the last real boundary starts a record that runs past the segment end
      if (realb1) open = ((recb1 >> (31 - __clz(realb1))) & 1u) != 0;
      else if (realb0) open = ((recb0 >> (31 - __clz(realb0))) & 1u) != 0;
      open = open && !end_real;
    } else {
      // ---- pass 1 (forward): real boundaries and records, flags into the list
      for (int b = 0; b < nev; b += 32) {
        const int e = b + lane;
        bool real = false, rec = false;
        if (e < nev) {
          const u32 ev = W.ev[e];
          classify(ev, real, rec);
          W.ev[e] = (uint16_t)(ev | (real ? 0x4000u : 0u) | (rec ? 0x8000u : 0u));
        }
        rtot += (u32)__popc(__ballot_sync(MX_FULL, rec));
      }
      __syncwarp();
      // ---- pass 2 (backward): each record ends at the next real boundary;
      // its slot = records before it (rtot minus the records at or after it)
      int next_real = seg_end;
      int last_real_e = -1;
      u32 rsuf = 0;  // records in the batches after this one
      for (int b = (nev - 1) & ~31; b >= 0; b -= 32) {
        const int e = b + lane;
        const bool ok = e < nev;
        const u32 ev = ok ? (u32)W.ev[e] : 0u;
        const u32 fl = ev >> 14;
        const int idx = (int)(ev & EV_IDX);
        const u32 realb = __ballot_sync(MX_FULL, fl & 1u);
        const u32 recb = __ballot_sync(MX_FULL, fl & 2u);
        const u32 after = realb & above;
        const int nidx = __shfl_sync(MX_FULL, idx, after ? __ffs(after) - 1 : lane);
        if (realb) {
          if (last_real_e < 0) last_real_e = b + 31 - __clz(realb);
          first_real = __shfl_sync(MX_FULL, idx, __ffs(realb) - 1);
        }
        if (fl & 2u) store(idx, after ? nidx : next_real, rtot - 1u - rsuf - (u32)__popc(recb & above));
        rsuf += (u32)__popc(recb);
        if (realb) next_real = first_real;
      }
      open = last_real_e >= 0 && (W.ev[last_real_e] & 0x8000u) && !end_real;
    }
    if (lane == 0) {
      a.tile_cnt[seg] = rtot;
      a.tile_open[seg] = open ? 1u : 0u;
      // where the run continuing into this segment ends: the first real
      // boundary; the data end for the last segment; else "passes through"
      a.tile_head[seg] = first_real >= 0 ? (first_real == 0 ? 0 : s0 + first_real) : (s0 + len >= n ? n : -1);
    }
    __syncwarp();  // W is rewritten by the next segment
  }
}

}  // namespace mx
