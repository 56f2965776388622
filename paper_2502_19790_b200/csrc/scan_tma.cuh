// Stage-1 streaming pass (included by stage1.cu).
//
// Per-property int32 columns (and wide tuple codes): one CTA per 2048-sample
// tile, every 128-bit column load of a thread issued up front; thousands of
// independent CTAs keep HBM busy through occupancy.
//  * scan_fast_kernel   -- full tiles with <= 4 file starts (fast_tile);
//  * scan_list_kernel   -- the tiles it deferred (more file starts);
//  * scan_direct_kernel -- everything else (finish_tile).
// All write each tile's runs into the tile's own slot region (tile-local
// scan, no inter-tile dependency); run ends that fall into a later tile are
// patched by slot_fixup_kernel and slot_compact_kernel densifies the records.
// Per-tile file bookkeeping comes precomputed from tile_meta_kernel. (The
// persistent cp.async.bulk / mbarrier ring variant measured slower than
// occupancy here -- 2.1 vs 0.65 ms at cfg2 -- and was removed; see git
// history and DESIGN.md.)
#pragma once

namespace mx {

struct __align__(16) TileMeta {
  long long fbase;   // file_off[fa]
  int fa;            // file holding the tile's first sample
  int nf;            // file starts in (t0, t0 + tile]
  u32 prev_status;   // status of sample t0 - 1
  u32 next_status;   // status of sample t0 + tile
  u32 pad0, pad1;
};

__global__ void tile_meta_kernel(S1Args a, long long tile_len, long long ntiles, TileMeta* meta) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const long long t0 = t * tile_len;
  int fa = upper_bound_ll(a.file_off, a.n_files + 1, t0) - 1;
  if (fa >= a.n_files) fa = a.n_files - 1;
  const int fb = upper_bound_ll(a.file_off, a.n_files + 1, t0 + tile_len) - 1;
  TileMeta m;
  m.fbase = a.file_off[fa];
  m.fa = fa;
  m.nf = fb - fa;
  m.prev_status = sample_status<false>(a, nullptr, t0 - 1);
  m.next_status = sample_status<false>(a, nullptr, t0 + tile_len);
  m.pad0 = m.pad1 = 0;
  meta[t] = m;
}

constexpr int TMA_FILE_CAP = 256;

struct TileScratch {  // per-CTA shared scratch of one tile
  long long fstart[TMA_FILE_CAP];
  u32 warp_first[S1_THREADS / 32], warp_last[S1_THREADS / 32], warp_tot[S1_THREADS / 32];
  u32 last_open;
};

// Finalise statuses st[j][q] (packed key, FAIL bit) of this thread's samples
// wbase + 128j + 4lane + q: run boundaries, tile-local compaction, records
// into the tile's slot region [tile*TILE, ...).
template <int SEGS>
__device__ __forceinline__ void finish_tile(const S1Args& a, const TileMeta& m, long long tile, long long wbase,
                                            u32 (&st)[SEGS][4], TileScratch& sc) {
  constexpr int TILE = (S1_THREADS / 32) * 32 * 4 * SEGS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nf = m.nf;
  const bool overflow = nf > TMA_FILE_CAP;
  if (nf > 0 && !overflow)
    for (int k = tid; k < nf; k += S1_THREADS) sc.fstart[k] = a.file_off[m.fa + 1 + k];
  if (lane == 0) sc.warp_first[warp] = st[0][0];
  if (lane == 31) sc.warp_last[warp] = st[SEGS - 1][3];
  __syncthreads();
  const u32 warp_prev = warp == 0 ? m.prev_status : sc.warp_last[warp - 1];
  const u32 warp_next = warp == S1_THREADS / 32 - 1 ? m.next_status : sc.warp_first[warp + 1];
  auto fstart_of = [&](int f) -> long long {
    if (overflow) return a.file_off[f];
    return f == m.fa ? m.fbase : sc.fstart[f - m.fa - 1];
  };
  // run boundaries: a run starts on a filter pass after a fail, a key change
  // or a file start; it ends before a fail, a key change or a file start
  u32 starts[SEGS], ends[SEGS];
  int fidx[SEGS][4];
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    u32 prev_last = __shfl_up_sync(MX_FULL, st[j][3], 1);
    u32 next_first = __shfl_down_sync(MX_FULL, st[j][0], 1);
    const u32 seg_prev = __shfl_sync(MX_FULL, st[j > 0 ? j - 1 : 0][3], 31);
    const u32 seg_next = __shfl_sync(MX_FULL, st[j < SEGS - 1 ? j + 1 : 0][0], 0);
    if (lane == 0) prev_last = j == 0 ? warp_prev : seg_prev;
    if (lane == 31) next_first = j == SEGS - 1 ? warp_next : seg_next;
    const long long i0 = wbase + 128 * j + 4 * lane;
    u32 sm = 0, em = 0;
    if (nf == 0) {  // fast path: the whole tile lies in file m.fa
      const bool fs0 = (i0 == m.fbase);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        fidx[j][q] = m.fa;
        const u32 cur = st[j][q];
        const u32 prv = q == 0 ? prev_last : st[j][q - 1];
        const u32 nxt = q == 3 ? next_first : st[j][q + 1];
        const bool pass = !(cur & FAIL);
        sm |= (u32)(pass && ((q == 0 && fs0) || (prv & FAIL) || prv != cur)) << q;
        em |= (u32)(pass && ((nxt & FAIL) || nxt != cur)) << q;
      }
    } else {
      int f = overflow ? upper_bound_ll(a.file_off, a.n_files + 1, i0) - 1 : m.fa + upper_bound_ll(sc.fstart, nf, i0);
      bool fs_cur = (i0 < a.n) && fstart_of(f) == i0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long i = i0 + q;
        fidx[j][q] = f;
        int fn = f;
        bool fs_next;
        if (overflow) {
          fn = (i + 1 < a.n) ? upper_bound_ll(a.file_off, a.n_files + 1, i + 1) - 1 : f;
          fs_next = (i + 1 < a.n) && a.file_off[fn] == i + 1;
        } else {
          const int k = f - m.fa;
          fs_next = k < nf && sc.fstart[k] == i + 1;
          if (fs_next) fn = f + 1;
          while (fs_next && fn - m.fa < nf && sc.fstart[fn - m.fa] == i + 1) ++fn;  // empty files
        }
        const u32 cur = st[j][q];
        const u32 prv = q == 0 ? prev_last : st[j][q - 1];
        const u32 nxt = q == 3 ? next_first : st[j][q + 1];
        const bool pass = !(cur & FAIL);
        sm |= (u32)(pass && (fs_cur || (prv & FAIL) || prv != cur)) << q;
        em |= (u32)(pass && (fs_next || (nxt & FAIL) || nxt != cur)) << q;
        fs_cur = fs_next;
        f = fn;
      }
    }
    starts[j] = sm;
    ends[j] = em;
  }
  // tile-local compaction: byte-packed per-segment counts, warp + block scan
  u32 pack = 0;
#pragma unroll
  for (int j = 0; j < SEGS; ++j) pack |= (u32)__popc(starts[j]) << (8 * j);
  const u32 incl = warp_incl_scan(pack);
  const u32 excl = incl - pack;
  const u32 wtot = __shfl_sync(MX_FULL, incl, 31);
  u32 seg_base[SEGS];
  u32 acc = 0;
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    seg_base[j] = acc + ((excl >> (8 * j)) & 0xff);
    acc += (wtot >> (8 * j)) & 0xff;
  }
  if (lane == 0) sc.warp_tot[warp] = acc;
  if (warp == S1_THREADS / 32 - 1 && lane == 31)  // holder of the tile's last sample
    sc.last_open = (!(st[SEGS - 1][3] & FAIL) && !((ends[SEGS - 1] >> 3) & 1)) ? 1u : 0u;
  __syncthreads();
  if (warp == 0) {
    const u32 x = lane < S1_THREADS / 32 ? sc.warp_tot[lane] : 0;
    const u32 inc = warp_incl_scan(x);
    if (lane < S1_THREADS / 32) sc.warp_tot[lane] = inc - x;
    if (lane == 31) {
      a.tile_cnt[tile] = inc;
      a.tile_open[tile] = (inc > 0 && sc.last_open) ? 1u : 0u;  // last run ends in a later tile
    }
  }
  if (tid == 0) {  // does the tile start inside a run begun in an earlier tile?
    const u32 first = st[0][0];
    a.tile_head[tile] = (!(first & FAIL) && !(starts[0] & 1)) ? -1 : 0;
  }
  __syncthreads();
  const u64 tbase = (u64)tile * TILE;
  const u64 base = tbase + sc.warp_tot[warp];
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    if (!(starts[j] | ends[j])) continue;
    u64 run = base + seg_base[j];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long i = wbase + 128 * j + 4 * lane + q;
      if ((starts[j] >> q) & 1) {
        const u32 key = st[j][q];
        a.rec_key[run] = key;
        a.rec_file[run] = (u32)fidx[j][q];
        a.rec_start[run] = (u32)(i - fstart_of(fidx[j][q]));
        if ((key & a.rank_mask) == 0) atomicMin(&a.err->null_key_sample, (u64)i);
        ++run;
      }
      if ((ends[j] >> q) & 1) {
        if (run > tbase) a.rec_end[run - 1] = (u32)(i + 1 - fstart_of(fidx[j][q]));
        else a.tile_head[tile] = i + 1;  // end of the run continuing from before
      }
    }
  }
}

template <bool SUMF, int SEGS>
__device__ __forceinline__ void normalise_status(const S1Args& a, long long wbase, u32 (&st)[SEGS][4],
                                                 const u32 (&anyf)[SEGS][4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < SEGS; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long i = wbase + 128 * j + 4 * lane + q;
      if (SUMF) st[j][q] = (i < a.n && st[j][q] < a.fail_limit) ? st[j][q] : FAIL;
      else st[j][q] = (i < a.n) ? ((anyf[j][q] & FAIL) | st[j][q]) : FAIL;
    }
}

// ---------------------------------------------------------------------------
// One CTA per tile. PC = number of properties at compile time (0 = runtime
// loop, then the fail flag is OR-ed instead of counted).
template <int SEGS, int PC, bool SMEM_LUT>
__device__ __forceinline__ void direct_tile(const S1Args& a, const TileMeta* __restrict__ meta, long long tile,
                                            u32* s_lut, TileScratch& sc) {
  constexpr int WT = 32 * 4 * SEGS;
  constexpr int TILE = (S1_THREADS / 32) * WT;
  constexpr bool SUMF = PC > 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = PC > 0 ? PC : a.n_props;
  const long long t0 = tile * TILE;
  const long long wbase = t0 + (long long)warp * WT;
  const bool full = t0 + TILE <= a.n;
  // 1. issue every column load of this thread
  constexpr int PMAX = PC > 0 ? PC : 1;
  int4 v[PMAX][SEGS];
  if (PC > 0 && full) {
#pragma unroll
    for (int p = 0; p < PMAX; ++p)
#pragma unroll
      for (int j = 0; j < SEGS; ++j)
        v[p][j] = codes4(a, p, wbase + 128 * j + 4 * lane);
  }
  // 2. LUT to shared memory + tile metadata (overlaps the loads in flight).
  //    With PC > 0 the LUT carries the filter-fail flag as a COUNT above the
  //    key bits, so keying a sample is P lookups + P adds and one compare.
  if (SMEM_LUT) {
    const u32* src = SUMF ? a.lut_sum : a.lut;
    for (int i = tid; i < a.lut_off[P]; i += S1_THREADS) s_lut[i] = src[i];
  }
  const TileMeta m = meta[tile];
  __syncthreads();
  // 3. statuses
  u32 st[SEGS][4], anyf[SEGS][4];
#pragma unroll
  for (int j = 0; j < SEGS; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) st[j][q] = anyf[j][q] = 0;
  auto add = [&](int j, int q, u32 e) {
    if (SUMF) {
      st[j][q] += e;
    } else {
      st[j][q] += e & ~FAIL;
      anyf[j][q] |= e;
    }
  };
  if (PC > 0 && full) {
#pragma unroll
    for (int p = 0; p < PMAX; ++p) {
      const int lo = a.lut_off[p] + 1;
#pragma unroll
      for (int j = 0; j < SEGS; ++j) {
        add(j, 0, lut_get<SMEM_LUT>(s_lut, a.lut, lo + v[p][j].x));
        add(j, 1, lut_get<SMEM_LUT>(s_lut, a.lut, lo + v[p][j].y));
        add(j, 2, lut_get<SMEM_LUT>(s_lut, a.lut, lo + v[p][j].z));
        add(j, 3, lut_get<SMEM_LUT>(s_lut, a.lut, lo + v[p][j].w));
      }
    }
  } else {
    for (int p = 0; p < P; ++p) {
      const int lo = a.lut_off[p] + 1;
#pragma unroll
      for (int j = 0; j < SEGS; ++j) {
        const long long i = wbase + 128 * j + 4 * lane;
        if (a.vec_ok && i + 4 <= a.n) {
          const int4 x = codes4(a, p, i);
          add(j, 0, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.x));
          add(j, 1, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.y));
          add(j, 2, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.z));
          add(j, 3, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.w));
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (i + q < a.n) add(j, q, lut_get<SMEM_LUT>(s_lut, a.lut, lo + code_at(a, p, i + q)));
        }
      }
    }
  }
  normalise_status<SUMF, SEGS>(a, wbase, st, anyf);
  finish_tile<SEGS>(a, m, tile, wbase, st, sc);
}

template <int SEGS, int PC, bool SMEM_LUT>
__global__ void __launch_bounds__(S1_THREADS, 2)
scan_direct_kernel(S1Args a, const TileMeta* __restrict__ meta, long long ntiles, long long tile_base) {
  extern __shared__ __align__(16) u32 s_lut[];
  __shared__ TileScratch sc;
  direct_tile<SEGS, PC, SMEM_LUT>(a, meta, tile_base + blockIdx.x, s_lut, sc);
}

// tiles deferred by scan_fast_kernel (more file starts than it handles)
template <int SEGS, bool SMEM_LUT>
__global__ void __launch_bounds__(S1_THREADS, 2) scan_list_kernel(S1Args a, const TileMeta* __restrict__ meta) {
  extern __shared__ __align__(16) u32 s_lut[];
  __shared__ TileScratch sc;
  const u32 n = *a.defer_cnt;
  for (u32 x = blockIdx.x; x < n; x += gridDim.x) {
    direct_tile<SEGS, 0, SMEM_LUT>(a, meta, a.defer_list[x], s_lut, sc);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Full-tile fast path (the hot kernel at cfg2): tiles [0, nfull) are complete,
// the property count is a template constant, and everything before emission
// runs on 32-bit tile-local sample indices. File starts inside a tile (a tile
// spans at most a few files at realistic file sizes) are handled branch-light
// for up to 4 boundaries; tiles with more fall back to finish_tile.
constexpr int FAST_MAX_FS = 4;

// Tile body of the fast path, given the raw key sums st[j][q] of this thread's
// samples (tile-local index warp*512 + 128j + 4lane + q). s_fs: the tile's
// file starts (local, padded with 1<<30), visible to the CTA.
//
// st holds RAW key sums: a sample passes iff st < fail_limit, and a failing
// neighbour (raw sum >= fail_limit, or FAIL from the tile metadata) always
// compares unequal to a passing key, so no per-sample clamp is needed.
template <int SEGS>
__device__ __forceinline__ void fast_tile(const S1Args& a, const TileMeta& m, long long tile, u32 (&st)[SEGS][4],
                                          TileScratch& sc, const int* s_fs) {
  constexpr int WT = 32 * 4 * SEGS;
  constexpr int TILE = (S1_THREADS / 32) * WT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t0 = tile * TILE;
  const int lw = warp * WT + 4 * lane;  // tile-local index of this thread's sample (j=0, q=0)
  const u32 lim = a.fail_limit;
  if (lane == 0) sc.warp_first[warp] = st[0][0];
  if (lane == 31) sc.warp_last[warp] = st[SEGS - 1][3];
  __syncthreads();
  const u32 warp_prev = warp == 0 ? m.prev_status : sc.warp_last[warp - 1];
  const u32 warp_next = warp == S1_THREADS / 32 - 1 ? m.next_status : sc.warp_first[warp + 1];
  const int fb0 = (int)(m.fbase - t0);  // <= 0: start of the file holding sample 0
  const int nf = m.nf;
  int fs[FAST_MAX_FS];
#pragma unroll
  for (int k = 0; k < FAST_MAX_FS; ++k) fs[k] = s_fs[k];  // local file starts in (0, TILE], padded
  u32 starts[SEGS], ends[SEGS], fsel[SEGS];  // fsel: 3 bits per sample = file offset in the tile
  // A run that ends right before the next run starts (same file, both inside
  // the tile) is closed by that START event (wend), so its end event is
  // dropped (ekeep): most runs then cost one event instead of two.
  u32 wend[SEGS], ekeep[SEGS];
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    u32 prev_last = __shfl_up_sync(MX_FULL, st[j][3], 1);
    u32 next_first = __shfl_down_sync(MX_FULL, st[j][0], 1);
    const u32 seg_prev = __shfl_sync(MX_FULL, st[j > 0 ? j - 1 : 0][3], 31);
    const u32 seg_next = __shfl_sync(MX_FULL, st[j < SEGS - 1 ? j + 1 : 0][0], 0);
    if (lane == 0) prev_last = j == 0 ? warp_prev : seg_prev;
    if (lane == 31) next_first = j == SEGS - 1 ? warp_next : seg_next;
    const int li0 = lw + 128 * j;
    // file-start bits of samples li0..li0+4 (bit 4 = the next thread's first)
    u32 fsb = (li0 == fb0) ? 1u : 0u;
    u32 sel = 0;
    if (nf) {
#pragma unroll
      for (int k = 0; k < FAST_MAX_FS; ++k) {
        const int d = fs[k] - li0;  // file start k relative to this thread's first sample
        if (d >= 0 && d <= 4) fsb |= 1u << d;
        // +1 in the 3-bit field of every sample q >= d (files started at or before q)
        const int dc = min(max(d, 0), 4);
        sel += 0x249u & (0xfffu << (3 * dc));
      }
    }
    fsel[j] = sel;
    // boundary bits: bit q = sample q starts a new run candidate (file start or
    // key change vs its predecessor), bit 4 = the next thread's first sample does
    const u32 bnd = fsb | (u32)(prev_last != st[j][0]) | ((u32)(st[j][0] != st[j][1]) << 1) |
                    ((u32)(st[j][1] != st[j][2]) << 2) | ((u32)(st[j][2] != st[j][3]) << 3) |
                    ((u32)(st[j][3] != next_first) << 4);
    const u32 pm = (u32)(st[j][0] < lim) | ((u32)(st[j][1] < lim) << 1) | ((u32)(st[j][2] < lim) << 2) |
                   ((u32)(st[j][3] < lim) << 3);
    starts[j] = pm & bnd;
    ends[j] = pm & (bnd >> 1);
    const u32 ppm = ((pm << 1) | (u32)(prev_last < lim)) & 0xfu;  // predecessor passes
    u32 w = starts[j] & ppm & ~fsb;
    if (j == 0 && lane == 0 && warp == 0) w &= ~1u;  // the predecessor is in the previous tile
    const bool tile_last = j == SEGS - 1 && lane == 31 && warp == S1_THREADS / 32 - 1;
    const u32 n3 = (next_first < lim && !((fsb >> 4) & 1) && !tile_last) ? 8u : 0u;
    wend[j] = w;
    ekeep[j] = ends[j] & ~((w >> 1) | n3);
  }
  // tile-local compaction (same slot layout as finish_tile)
  u32 pack = 0;
#pragma unroll
  for (int j = 0; j < SEGS; ++j) pack |= (u32)__popc(starts[j]) << (8 * j);
  const u32 incl = warp_incl_scan(pack);
  const u32 excl = incl - pack;
  const u32 wtot = __shfl_sync(MX_FULL, incl, 31);
  u32 seg_base[SEGS];
  u32 acc = 0;
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    seg_base[j] = acc + ((excl >> (8 * j)) & 0xff);
    acc += (wtot >> (8 * j)) & 0xff;
  }
  if (lane == 0) sc.warp_tot[warp] = acc;
  if (warp == S1_THREADS / 32 - 1 && lane == 31)
    sc.last_open = (st[SEGS - 1][3] < lim && !((ends[SEGS - 1] >> 3) & 1)) ? 1u : 0u;
  __syncthreads();
  if (warp == 0) {
    const u32 x = lane < S1_THREADS / 32 ? sc.warp_tot[lane] : 0;
    const u32 inc = warp_incl_scan(x);
    if (lane < S1_THREADS / 32) sc.warp_tot[lane] = inc - x;
    if (lane == 31) {
      a.tile_cnt[tile] = inc;
      a.tile_open[tile] = (inc > 0 && sc.last_open) ? 1u : 0u;
    }
  }
  if (tid == 0) a.tile_head[tile] = (st[0][0] < lim && !(starts[0] & 1)) ? -1 : 0;
  __shared__ u32 s_off[FAST_MAX_FS + 1];  // local sample -> in-file sample offset per file of the tile
  if (tid <= FAST_MAX_FS) s_off[tid] = tid == 0 ? (u32)(t0 - m.fbase) : (u32)(-s_fs[tid - 1]);
  __syncthreads();
  // records, all in 32-bit tile-local slot indices
  const u64 tbase = (u64)tile * TILE;
  u32* __restrict__ rk = a.rec_key + tbase;
  u32* __restrict__ rf = a.rec_file + tbase;
  u32* __restrict__ rs = a.rec_start + tbase;
  u32* __restrict__ re = a.rec_end + tbase;
  const u32 wb = sc.warp_tot[warp];
#pragma unroll
  for (int j = 0; j < SEGS; ++j) {
    u32 run = wb + seg_base[j];
    // visit only this segment's events, in sample order (start before end)
    for (u32 ev = starts[j] | ekeep[j]; ev; ev &= ev - 1) {
      const int q = __ffs(ev) - 1;
      const u32 li = (u32)(lw + 128 * j + q);
      const u32 fo = (fsel[j] >> (3 * q)) & 7;  // file = m.fa + fo
      const u32 off = li + s_off[fo];
      if ((starts[j] >> q) & 1) {
        if ((wend[j] >> q) & 1) {  // close the run ending at li - 1 (same file)
          if (run > 0) re[run - 1] = off;
          else a.tile_head[tile] = t0 + li;
        }
        const u32 key = q == 0 ? st[j][0] : q == 1 ? st[j][1] : q == 2 ? st[j][2] : st[j][3];
        rk[run] = key;
        rf[run] = (u32)m.fa + fo;
        rs[run] = off;
        if ((key & a.rank_mask) == 0) atomicMin(&a.err->null_key_sample, (u64)(t0 + li));
        ++run;
      }
      if ((ekeep[j] >> q) & 1) {
        if (run > 0) re[run - 1] = off + 1;
        else a.tile_head[tile] = t0 + li + 1;
      }
    }
  }
}

template <int PC, int SEGS, bool GLUT = false>
__device__ __forceinline__ void lut_sums(const u32* s_lut, const S1Args& a, const int4 (&v)[PC][SEGS],
                                         u32 (&st)[SEGS][4]) {
#pragma unroll
  for (int j = 0; j < SEGS; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) st[j][q] = 0;
#pragma unroll
  for (int p = 0; p < PC; ++p) {
    if (GLUT) {  // large LUT (row-tuple layout): read-only path, L1-resident
      const u32* __restrict__ L = a.lut_sum + a.lut_off[p] + 1;
#pragma unroll
      for (int j = 0; j < SEGS; ++j) {
        st[j][0] += __ldg(L + v[p][j].x); st[j][1] += __ldg(L + v[p][j].y);
        st[j][2] += __ldg(L + v[p][j].z); st[j][3] += __ldg(L + v[p][j].w);
      }
    } else {
      const u32* L = s_lut + a.lut_off[p] + 1;
#pragma unroll
      for (int j = 0; j < SEGS; ++j) {
        st[j][0] += L[v[p][j].x]; st[j][1] += L[v[p][j].y];
        st[j][2] += L[v[p][j].z]; st[j][3] += L[v[p][j].w];
      }
    }
  }
}

// one CTA per full tile, loads in registers. SEGS = int4 segments per thread:
// 4 (4096-sample tiles, 2 CTAs/SM) or 2 (2048-sample tiles, 4 CTAs/SM: the
// same bytes in flight per SM, split over twice as many independent CTAs).
// GLUT: the LUT is read through L1 instead of being staged per CTA -- for a
// row-tuple LUT (thousands of entries) staging would copy as many bytes per
// CTA as the tile's column itself.
// OCC: resident CTAs per SM the register budget is cut for. A single code
// column (row-tuple layout) has 5x fewer bytes in flight per CTA than the
// 5-property case, so it runs more CTAs per SM instead.
template <int PC, int SEGS, bool GLUT = false, int OCC = (SEGS == 2 || PC == 1 ? 4 : 2)>
__global__ void __launch_bounds__(S1_THREADS, OCC)
scan_fast_kernel(S1Args a, const TileMeta* __restrict__ meta) {
  constexpr int TILE = S1_THREADS * 4 * SEGS;
  extern __shared__ __align__(16) u32 s_lut[];
  __shared__ TileScratch sc;
  __shared__ int s_fs[FAST_MAX_FS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long tile = blockIdx.x;
  const long long t0 = tile * TILE;
  const int lw = warp * 128 * SEGS + 4 * lane;
  int4 v[PC][SEGS];
#pragma unroll
  for (int p = 0; p < PC; ++p) {
#pragma unroll
    for (int j = 0; j < SEGS; ++j) v[p][j] = codes4(a, p, t0 + lw + 128 * j);
  }
  if (!GLUT)
    for (int i = tid; i < a.lut_off[PC]; i += S1_THREADS) s_lut[i] = a.lut_sum[i];
  const TileMeta m = meta[tile];
  if (m.nf > FAST_MAX_FS) {  // many tiny files: deferred to scan_list_kernel
    if (tid == 0) a.defer_list[atomicAdd(a.defer_cnt, 1u)] = (u32)tile;
    return;
  }
  if (tid < FAST_MAX_FS) s_fs[tid] = tid < m.nf ? (int)(a.file_off[m.fa + 1 + tid] - t0) : 1 << 30;
  __syncthreads();
  u32 st[SEGS][4];
  lut_sums<PC, SEGS, GLUT>(s_lut, a, v, st);
  fast_tile<SEGS>(a, m, tile, st, sc, s_fs);
}

// Dense copy of the slot records (one warp per tile, order preserved).
__global__ void slot_compact_kernel(long long ntiles, long long tile_len, const u32* cnt, const u64* off,
                                    const u32* k, const u32* f, const u32* s, const u32* e, u32* k2, u32* f2, u32* s2,
                                    u32* e2) {
  // four tiles per warp in flight: their counts / offsets, then their first
  // 64 records each (two per lane: a 2048-sample segment at R = 64 holds ~32),
  // are loaded before anything is stored
  constexpr int U = 4;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const u32 lane = threadIdx.x & 31;
  for (long long t0 = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t0 < ntiles; t0 += U * warps) {
    u32 c[U];
    u64 dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long t = t0 + u * warps;
      c[u] = t < ntiles ? cnt[t] : 0;
      dst[u] = t < ntiles ? off[t] : 0;
    }
    u32 vk[U][2], vf[U][2], vs[U][2], ve[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const u64 src = (u64)(t0 + u * warps) * tile_len + lane;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < c[u]) {
          vk[u][h] = k[src + 32 * h]; vf[u][h] = f[src + 32 * h]; vs[u][h] = s[src + 32 * h];
          ve[u][h] = e[src + 32 * h];
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < c[u]) {
          const u64 d = dst[u] + lane + 32 * h;
          k2[d] = vk[u][h]; f2[d] = vf[u][h]; s2[d] = vs[u][h]; e2[d] = ve[u][h];
        }
      const u64 src = (u64)(t0 + u * warps) * tile_len;
      for (u32 i = lane + 64; i < c[u]; i += 32) {  // tiles with more than 64 runs
        k2[dst[u] + i] = k[src + i];
        f2[dst[u] + i] = f[src + i];
        s2[dst[u] + i] = s[src + i];
        e2[dst[u] + i] = e[src + i];
      }
    }
  }
}

// Patch the end of every tile's open last run (it ends in a later tile: the
// first later tile whose head run ends), and total the run counts.
__global__ void slot_fixup_kernel(long long ntiles, long long tile_len, const u32* cnt, const u32* open,
                                  const long long* head, const u32* rec_file, const long long* file_off, u32* rec_end,
                                  u64* total) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  u32 c = 0;
  if (t < ntiles) {
    c = cnt[t];
    if (open[t]) {
      long long u = t + 1;
      while (u < ntiles && head[u] == -1) ++u;
      const long long slot = t * tile_len + c - 1;
      if (u < ntiles && head[u] > 0) rec_end[slot] = (u32)(head[u] - file_off[rec_file[slot]]);
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total, (u64)c);
}

}  // namespace mx
