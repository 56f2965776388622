// Stage-1 streaming pass for ONE u16 code column (the row-tuple layout, the
// bench's layout), included by stage1.cu.
//
// At 2 bytes per sample the per-sample work has to be a few instructions or
// the pass is issue bound, not HBM bound. A sample can only start or end a
// run where its tuple code differs from its predecessor's (distinct tuples
// have distinct full keys) or at a file start, so the common path never
// touches the key LUT:
//
//  * the unit of work is a WARP SEGMENT of 1024 consecutive samples (no
//    CTA-wide synchronisation anywhere): lane L holds 32 codes from four
//    coalesced 16-byte loads (ld.global.nc.L1::no_allocate.v4; load k covers
//    samples [k*256, (k+1)*256) of the segment, lane L its 8 at k*256 + 8L);
//  * code changes come from __byte_perm'ed predecessor words, an XOR and a
//    carry trick that turns every nonzero 16-bit half into one bit, so a lane
//    gets a 32-bit candidate mask for its 32 samples in ~4 instructions per
//    sample; file starts (from the segment's file range) are OR-ed in;
//  * candidates are compacted in sample order into per-warp shared memory
//    (one packed warp scan of the four runs' counts), then one lane per
//    candidate reads the two keys from the LUT (staged per CTA) and decides
//    whether it is a real boundary -- a key change with either side passing
//    the filter, a pass / fail switch, or a file start next to a passing
//    sample -- and whether it starts a record (its sample passes). Ballots
//    give each record its slot and its end: the next real boundary (or the
//    segment end, or later: slot_fixup_kernel).
//
// Persistent CTAs; each warp walks segments grid-stride and keeps the next
// segment's loads in flight while finishing the current one. Output follows
// the slot contract of the other stage-1 kernels with tile_len = 1024:
// records at [seg * 1024, ...), tile_cnt / tile_open / tile_head per segment.
#pragma once

namespace mx {

constexpr int SEG_LEN = 1024;        // samples per warp segment
constexpr int U16_WARPS = 4;         // warps per CTA
constexpr int U16_SMEM_LUT_MAX = 16384;

struct U16Warp {                     // per-warp shared scratch
  uint16_t codes[SEG_LEN];           // the segment's codes in sample order
  uint16_t ev[SEG_LEN];              // candidate boundaries (segment offsets), sample order
  uint16_t rank[SEG_LEN];            // record slot of a candidate, 0xffff if none
  uint8_t flag[SEG_LEN];             // bit 0 real boundary, bit 1 starts a record
  u32 fsm[SEG_LEN / 32];             // file starts inside the segment (bit = offset)
};

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

template <bool SLUT>
__device__ __forceinline__ u32 u16_key(const u32* s_lut, const u32* g_lut, u32 code) {
  return SLUT ? s_lut[code] : __ldg(g_lut + code);
}

// bit per nonzero 16-bit half of x: bit 15 (low half), bit 31 (high half)
__device__ __forceinline__ u32 nz16(u32 x) { return ((x & 0x7fff7fffu) + 0x7fff7fffu) | x; }

// 8-bit change mask of one run of 8 codes (words w.x..w.w) given the code before it
__device__ __forceinline__ u32 change8(u32 prev, const uint4& w) {
  const u32 t0 = nz16(w.x ^ __byte_perm(prev << 16, w.x, 0x5432));
  const u32 t1 = nz16(w.y ^ __byte_perm(w.x, w.y, 0x5432));
  const u32 t2 = nz16(w.z ^ __byte_perm(w.y, w.z, 0x5432));
  const u32 t3 = nz16(w.w ^ __byte_perm(w.z, w.w, 0x5432));
  // bytes 1 and 3 of each t carry samples (2i, 2i+1) in their top bit
  const u32 u = __byte_perm(t0, t1, 0x7531), v = __byte_perm(t2, t3, 0x7531);
  const u32 lo = (((u >> 7) & 0x01010101u) * 0x01020408u) >> 24;  // samples 0..3
  const u32 hi = (((v >> 7) & 0x01010101u) * 0x01020408u) >> 24;  // samples 4..7
  return lo | (hi << 4);
}

template <bool SLUT>
__global__ void __launch_bounds__(U16_WARPS * 32, 6)
scan_u16_kernel(S1Args a, const int* __restrict__ seg_fa, long long nseg) {
  extern __shared__ __align__(16) unsigned char u16_dyn[];
  U16Warp* wsm = reinterpret_cast<U16Warp*>(u16_dyn);
  u32* s_lut = reinterpret_cast<u32*>(u16_dyn + sizeof(U16Warp) * U16_WARPS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  U16Warp& W = wsm[warp];
  const uint16_t* __restrict__ col = reinterpret_cast<const uint16_t*>(a.cols[0]);
  const u32* __restrict__ g_lut = a.lut_sum + 1;  // entry of code c at c (a tuple column has no null code)
  const u32 lim = a.fail_limit;
  const long long n = a.n;
  if (SLUT)
    for (int i = threadIdx.x; i < a.lut_off[1] - 1; i += U16_WARPS * 32) s_lut[i] = g_lut[i];
  __syncthreads();  // the only CTA barrier: LUT staged
  const long long wstride = (long long)gridDim.x * U16_WARPS;
  long long seg = (long long)blockIdx.x * U16_WARPS + warp;
  // prefetched state of the next segment
  uint4 w[4];
  u32 halo = 0;  // lane 0: code before the segment; lane 31: code after it
  int fa = 0, fa_next = 0;
  auto fetch = [&](long long sg) {
    const long long s0 = sg * SEG_LEN;
    if (s0 + SEG_LEN <= n) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int4 v = ld_stream_v4(reinterpret_cast<const int4*>(col + s0 + k * 256 + lane * 8));
        w[k] = make_uint4((u32)v.x, (u32)v.y, (u32)v.z, (u32)v.w);
      }
    } else {  // partial last segment: scalar loads, the last code repeated past n (no candidates there)
      const u32 last = col[n - 1];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
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
    uint4 cw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cw[k] = w[k];
    const u32 chalo = halo;
    const int cfa = fa;
    const int nf = fa_next - fa;  // file starts in (s0, s0 + 1024] ((s0, n) for the last segment)
    const long long nxt = seg + wstride;
    if (nxt < nseg) fetch(nxt);
    // ---- codes to shared memory (sample order), candidate mask per lane
#pragma unroll
    for (int k = 0; k < 4; ++k) *reinterpret_cast<uint4*>(&W.codes[k * 256 + lane * 8]) = cw[k];
    const u32 hprev = __shfl_sync(MX_FULL, chalo, 0);  // code before the segment
    u32 m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const u32 up = __shfl_up_sync(MX_FULL, cw[k].w >> 16, 1);
      const u32 wrap = __shfl_sync(MX_FULL, cw[k > 0 ? k - 1 : 0].w >> 16, 31);
      const u32 pv = lane > 0 ? up : (k == 0 ? hprev : wrap);
      m |= change8(pv, cw[k]) << (8 * k);
    }
    if (s0 == 0 && lane == 0) m |= 1u;  // sample 0: no predecessor
    // ---- file starts in (s0, s0 + len): bitmask by segment offset
    W.fsm[lane] = 0;
    __syncwarp();
    const long long fbase = __ldg(a.file_off + cfa);  // start of the file holding s0
    for (int k = 1 + lane; k <= nf; k += 32) {
      const long long p = __ldg(a.file_off + cfa + k) - s0;
      if (p > 0 && p < len) atomicOr(&W.fsm[p >> 5], 1u << (p & 31));
    }
    __syncwarp();
    u32 fsb = 0;  // this lane's file-start bits, same layout as m
    if (nf > 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int o = k * 256 + lane * 8;
        fsb |= ((W.fsm[o >> 5] >> (o & 31)) & 0xffu) << (8 * k);
      }
    }
    const bool fs0 = s0 > 0 && fbase == s0;  // a file starts at the segment's first sample
    if (fs0 && lane == 0) fsb |= 1u;
    m |= fsb;
    // ---- compaction of candidates in sample order (run k major, then lane);
    // a run's total over the warp is <= 256: scan its count in a 16-bit field
    const u32 c01 = (u32)__popc(m & 0xffu) | ((u32)__popc(m & 0xff00u) << 16);
    const u32 c23 = (u32)__popc(m & 0xff0000u) | ((u32)__popc(m & 0xff000000u) << 16);
    const u32 i01 = warp_incl_scan(c01), i23 = warp_incl_scan(c23);
    const u32 t01 = __shfl_sync(MX_FULL, i01, 31), t23 = __shfl_sync(MX_FULL, i23, 31);
    const u32 e01 = i01 - c01, e23 = i23 - c23;
    const u32 tk0 = t01 & 0xffffu, tk1 = t01 >> 16, tk2 = t23 & 0xffffu, tk3 = t23 >> 16;
    const int nev = (int)(tk0 + tk1 + tk2 + tk3);
    const u32 pos[4] = {e01 & 0xffffu, tk0 + (e01 >> 16), tk0 + tk1 + (e23 & 0xffffu),
                        tk0 + tk1 + tk2 + (e23 >> 16)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u32 p = pos[k];
      for (u32 c = (m >> (8 * k)) & 0xffu; c; c &= c - 1) W.ev[p++] = (uint16_t)(k * 256 + lane * 8 + __ffs(c) - 1);
    }
    __syncwarp();
    // ---- pass 1 (forward): real boundaries, records, record slots
    u32 rbase = 0;
    for (int b = 0; b < nev; b += 32) {
      const int e = b + lane;
      bool real = false, rec = false;
      if (e < nev) {
        const int idx = W.ev[e];
        const u32 kc = u16_key<SLUT>(s_lut, g_lut, W.codes[idx]);
        const bool pc = kc < lim;
        if (s0 + idx == 0) {
          real = pc;
        } else {
          const u32 pre = idx > 0 ? (u32)W.codes[idx - 1] : hprev;
          const u32 kp = u16_key<SLUT>(s_lut, g_lut, pre);
          const bool fs = idx == 0 ? fs0 : ((W.fsm[idx >> 5] >> (idx & 31)) & 1u) != 0;
          real = (pc || kp < lim) && (fs || kc != kp);
        }
        rec = real && pc;
      }
      const u32 rb = __ballot_sync(MX_FULL, rec);
      if (e < nev) {
        W.flag[e] = (uint8_t)((real ? 1u : 0u) | (rec ? 2u : 0u));
        W.rank[e] = rec ? (uint16_t)(rbase + __popc(rb & ((1u << lane) - 1u))) : (uint16_t)0xffffu;
      }
      rbase += (u32)__popc(rb);
    }
    __syncwarp();
    // ---- segment end: is sample s0 + len a boundary of the run holding s0 + len - 1?
    bool end_real = true;
    {
      const u32 last = __shfl_sync(MX_FULL, cw[3].w >> 16, 31);
      const u32 after = __shfl_sync(MX_FULL, chalo, 31);
      if (s0 + len < n) {  // len == 1024 here
        const u32 kl = u16_key<SLUT>(s_lut, g_lut, last);
        const u32 kn = u16_key<SLUT>(s_lut, g_lut, after);
        const bool fs_end = nf > 0 && __ldg(a.file_off + cfa + nf) == s0 + SEG_LEN;
        end_real = fs_end || kl != kn;
      }
    }
    // ---- pass 2 (backward): each record ends at the next real boundary
    const u64 sbase = (u64)seg * SEG_LEN;
    int next_real = end_real ? len : -1;  // -1: the run continues past the segment
    int first_real = -1, last_real_e = -1;
    for (int b = (nev - 1) & ~31; b >= 0; b -= 32) {
      const int e = b + lane;
      const bool ok = e < nev;
      const u32 fl = ok ? (u32)W.flag[e] : 0u;
      const int idx = ok ? (int)W.ev[e] : 0;
      const u32 realb = __ballot_sync(MX_FULL, fl & 1u);
      const u32 after = realb & ~((2u << lane) - 1u);
      const int nidx = __shfl_sync(MX_FULL, idx, after ? __ffs(after) - 1 : lane);
      if (realb) {
        if (last_real_e < 0) last_real_e = b + 31 - __clz(realb);
        first_real = __shfl_sync(MX_FULL, idx, __ffs(realb) - 1);
      }
      if (fl & 2u) {
        const int end = after ? nidx : next_real;
        const u32 r = W.rank[e];
        // file of the run: fa + the segment's file starts at or before it
        int lo = 0, hi = nf;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(a.file_off + cfa + mid) <= s0 + idx) lo = mid; else hi = mid - 1;
        }
        const long long fstart = lo ? __ldg(a.file_off + cfa + lo) : fbase;
        const u32 key = u16_key<SLUT>(s_lut, g_lut, W.codes[idx]);
        const u32 off = (u32)(s0 - fstart);
        a.rec_key[sbase + r] = key;
        a.rec_file[sbase + r] = (u32)(cfa + lo);
        a.rec_start[sbase + r] = off + (u32)idx;
        if (end >= 0) a.rec_end[sbase + r] = off + (u32)end;
        if ((key & a.rank_mask) == 0) atomicMin(&a.err->null_key_sample, (u64)(s0 + idx));
      }
      if (realb) next_real = first_real;
    }
    if (lane == 0) {
      a.tile_cnt[seg] = rbase;
      const bool open = last_real_e >= 0 && (W.flag[last_real_e] & 2u) && !end_real;
      a.tile_open[seg] = open ? 1u : 0u;
      // where the run continuing into this segment ends: the first real
      // boundary; the data end for the last segment; else "passes through"
      a.tile_head[seg] = first_real >= 0 ? (first_real == 0 ? 0 : s0 + first_real) : (s0 + len >= n ? n : -1);
    }
    __syncwarp();  // W is rewritten by the next segment
  }
}

}  // namespace mx
