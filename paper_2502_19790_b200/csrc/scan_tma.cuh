// Stage-1 streaming pass, persistent + TMA-staged (included by stage1.cu).
//
// Each CTA owns a ring of `stages` shared-memory slots. A slot holds one tile
// of every code column plus the tile's precomputed metadata, filled by
// cp.async.bulk (TMA bulk copies, SASS UBLKCP) completing on an mbarrier, so
// the next tiles' HBM reads are in flight while the current tile is keyed,
// run-detected and compacted. Tiles are claimed from an atomic counter in
// increasing order, which keeps the decoupled look-back deadlock-free (every
// predecessor of a claimed tile is owned by a running CTA that reaches it
// first). Per-tile file bookkeeping (first file, file starts inside the tile,
// neighbour-sample statuses) is computed up front by tile_meta_kernel, one
// thread per tile, so no thread serialises on global binary searches.
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

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "MX_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra MX_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int TMA_MAX_STAGES = 4;
constexpr int TMA_FILE_CAP = 256;

template <int SEGS, bool SMEM_LUT>
__global__ void __launch_bounds__(S1_THREADS)
scan_tma_kernel(S1Args a, const TileMeta* __restrict__ meta, long long ntiles, long long nstaged, int stages,
                int lut_bytes) {
  constexpr int WT = 32 * 4 * SEGS;             // samples per warp
  constexpr int TILE = (S1_THREADS / 32) * WT;  // samples per tile
  extern __shared__ __align__(128) unsigned char dyn[];
  u32* s_lut = reinterpret_cast<u32*>(dyn);
  int32_t* s_codes = reinterpret_cast<int32_t*>(dyn + lut_bytes);  // [stages][P][TILE]
  TileMeta* s_meta = reinterpret_cast<TileMeta*>(s_codes + (long long)stages * a.n_props * TILE);
  __shared__ __align__(8) u64 s_bar[TMA_MAX_STAGES];
  __shared__ long long s_tile[TMA_MAX_STAGES];
  __shared__ long long s_fstart[TMA_FILE_CAP];
  __shared__ u32 s_warp_first[S1_THREADS / 32], s_warp_last[S1_THREADS / 32], s_warp_tot[S1_THREADS / 32];
  __shared__ u64 s_tile_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = a.n_props;
  if (SMEM_LUT)
    for (int i = tid; i < a.lut_off[P]; i += S1_THREADS) s_lut[i] = a.lut[i];

  auto issue = [&](int s) {  // thread 0: claim the next tile into slot s
    const long long t = (long long)atomicAdd(a.tile_ctr, 1u);
    s_tile[s] = t;
    if (t < nstaged) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_tx(&s_bar[s], (u32)(P * TILE * 4 + sizeof(TileMeta)));
      for (int p = 0; p < P; ++p)
        bulk_g2s(s_codes + ((long long)s * P + p) * TILE, a.cols[p] + t * TILE, TILE * 4, &s_bar[s]);
      bulk_g2s(&s_meta[s], meta + t, sizeof(TileMeta), &s_bar[s]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&s_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < stages; ++s) issue(s);
  }
  __syncthreads();

  for (int it = 0;; ++it) {
    const int s = it % stages;
    const long long tile = s_tile[s];
    if (tile >= ntiles) break;
    const bool staged = tile < nstaged;
    if (staged) mbar_wait(&s_bar[s], (u32)((it / stages) & 1));
    const TileMeta m = staged ? s_meta[s] : meta[tile];
    const long long t0 = tile * TILE;
    const long long wbase = t0 + (long long)warp * WT;

    // ---- statuses (packed key | fail) of this thread's 4*SEGS samples
    u32 st[SEGS][4], anyf[SEGS][4];
#pragma unroll
    for (int j = 0; j < SEGS; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) st[j][q] = anyf[j][q] = 0;
    for (int p = 0; p < P; ++p) {
      const int lo = a.lut_off[p] + 1;
      if (staged) {
        const int32_t* c = s_codes + ((long long)s * P + p) * TILE + warp * WT + 4 * lane;
#pragma unroll
        for (int j = 0; j < SEGS; ++j) {
          const int4 v = *reinterpret_cast<const int4*>(c + 128 * j);
          const u32 e0 = lut_get<SMEM_LUT>(s_lut, a.lut, lo + v.x);
          const u32 e1 = lut_get<SMEM_LUT>(s_lut, a.lut, lo + v.y);
          const u32 e2 = lut_get<SMEM_LUT>(s_lut, a.lut, lo + v.z);
          const u32 e3 = lut_get<SMEM_LUT>(s_lut, a.lut, lo + v.w);
          st[j][0] += e0 & ~FAIL; anyf[j][0] |= e0;
          st[j][1] += e1 & ~FAIL; anyf[j][1] |= e1;
          st[j][2] += e2 & ~FAIL; anyf[j][2] |= e2;
          st[j][3] += e3 & ~FAIL; anyf[j][3] |= e3;
        }
      } else {
        const int32_t* col = a.cols[p];
#pragma unroll
        for (int j = 0; j < SEGS; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const long long i = wbase + 128 * j + 4 * lane + q;
            if (i < a.n) {
              const u32 e = lut_get<SMEM_LUT>(s_lut, a.lut, lo + col[i]);
              st[j][q] += e & ~FAIL;
              anyf[j][q] |= e;
            }
          }
      }
    }
#pragma unroll
    for (int j = 0; j < SEGS; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long i = wbase + 128 * j + 4 * lane + q;
        st[j][q] = (i < a.n) ? ((anyf[j][q] & FAIL) | st[j][q]) : FAIL;
      }
    if (lane == 0) s_warp_first[warp] = st[0][0];
    if (lane == 31) s_warp_last[warp] = st[SEGS - 1][3];
    // file starts inside the tile (rare: only tiles that cross a file boundary)
    const int nf = m.nf;
    const bool overflow = nf > TMA_FILE_CAP;
    if (nf > 0 && !overflow)
      for (int k = tid; k < nf; k += S1_THREADS) s_fstart[k] = a.file_off[m.fa + 1 + k];
    __syncthreads();
    const u32 warp_prev = warp == 0 ? m.prev_status : s_warp_last[warp - 1];
    const u32 warp_next = warp == S1_THREADS / 32 - 1 ? m.next_status : s_warp_first[warp + 1];

    auto fstart_of = [&](int f) -> long long {
      if (overflow) return a.file_off[f];
      return f == m.fa ? m.fbase : s_fstart[f - m.fa - 1];
    };

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
          const bool start = pass && ((q == 0 && fs0) || (prv & FAIL) || prv != cur);
          const bool end = pass && ((nxt & FAIL) || nxt != cur);
          sm |= (u32)start << q;
          em |= (u32)end << q;
        }
      } else {
        int f = overflow ? upper_bound_ll(a.file_off, a.n_files + 1, i0) - 1
                         : m.fa + upper_bound_ll(s_fstart, nf, i0);
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
            fs_next = k < nf && s_fstart[k] == i + 1;
            if (fs_next) fn = f + 1;
            while (fs_next && fn - m.fa < nf && s_fstart[fn - m.fa] == i + 1) ++fn;
          }
          const u32 cur = st[j][q];
          const u32 prv = q == 0 ? prev_last : st[j][q - 1];
          const u32 nxt = q == 3 ? next_first : st[j][q + 1];
          const bool pass = !(cur & FAIL);
          const bool start = pass && (fs_cur || (prv & FAIL) || prv != cur);
          const bool end = pass && (fs_next || (nxt & FAIL) || nxt != cur);
          sm |= (u32)start << q;
          em |= (u32)end << q;
          fs_cur = fs_next;
          f = fn;
        }
      }
      starts[j] = sm;
      ends[j] = em;
    }

    // ---- compaction: byte-packed per-segment counts, warp + block scan, look-back
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
    if (lane == 0) s_warp_tot[warp] = acc;
    __syncthreads();
    if (warp == 0) {
      const u32 v = lane < S1_THREADS / 32 ? s_warp_tot[lane] : 0;
      const u32 inc = warp_incl_scan(v);
      const u32 tile_agg = __shfl_sync(MX_FULL, inc, 31);
      if (lane < S1_THREADS / 32) s_warp_tot[lane] = inc - v;
      const u64 tex = lookback_exclusive(a.status, (int)tile, tile_agg);
      if (lane == 0) {
        s_tile_excl = tex;
        if (tile == ntiles - 1) *a.n_runs = tex + tile_agg;
      }
    }
    __syncthreads();
    const u64 base = s_tile_excl + s_warp_tot[warp];
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
        if ((ends[j] >> q) & 1) a.rec_end[run - 1] = (u32)(i + 1 - fstart_of(fidx[j][q]));
      }
    }
    __syncthreads();  // slot s and the per-tile scratch are free again
    if (tid == 0) issue(s);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Non-persistent variant: one CTA per tile (thousands of independent CTAs keep
// HBM busy through occupancy instead of a per-CTA pipeline), tile id =
// blockIdx.x (CTAs are dispatched in index order, which the look-back relies
// on, as in CUB's single-pass scan), per-tile metadata from tile_meta_kernel,
// all column loads of a thread issued before any dependent work (PC = number
// of properties at compile time; 0 = runtime loop).
template <int SEGS, int PC, bool SMEM_LUT>
__global__ void __launch_bounds__(S1_THREADS, 2)
scan_direct_kernel(S1Args a, const TileMeta* __restrict__ meta, long long ntiles) {
  constexpr int WT = 32 * 4 * SEGS;
  constexpr int TILE = (S1_THREADS / 32) * WT;
  extern __shared__ __align__(16) u32 s_lut[];
  __shared__ long long s_fstart[TMA_FILE_CAP];
  __shared__ u32 s_warp_first[S1_THREADS / 32], s_warp_last[S1_THREADS / 32], s_warp_tot[S1_THREADS / 32];
  __shared__ u64 s_tile_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = PC > 0 ? PC : a.n_props;
  const long long tile = blockIdx.x;
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
        v[p][j] = ld_stream_v4(reinterpret_cast<const int4*>(a.cols[p] + wbase + 128 * j + 4 * lane));
  }
  // 2. LUT to shared memory + tile metadata (overlaps the loads in flight).
  //    With PC > 0 the LUT carries the filter-fail flag as a COUNT above the
  //    key bits, so keying a sample is P lookups + P adds and one compare.
  constexpr bool SUMF = PC > 0;
  if (SMEM_LUT) {
    const u32* src = SUMF ? a.lut_sum : a.lut;
    for (int i = tid; i < a.lut_off[P]; i += S1_THREADS) s_lut[i] = src[i];
  }
  const TileMeta m = meta[tile];
  const int nf = m.nf;
  const bool overflow = nf > TMA_FILE_CAP;
  if (nf > 0 && !overflow)
    for (int k = tid; k < nf; k += S1_THREADS) s_fstart[k] = a.file_off[m.fa + 1 + k];
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
      const int32_t* col = a.cols[p];
#pragma unroll
      for (int j = 0; j < SEGS; ++j) {
        const long long i = wbase + 128 * j + 4 * lane;
        if (i + 4 <= a.n) {
          const int4 x = ld_stream_v4(reinterpret_cast<const int4*>(col + i));
          add(j, 0, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.x));
          add(j, 1, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.y));
          add(j, 2, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.z));
          add(j, 3, lut_get<SMEM_LUT>(s_lut, a.lut, lo + x.w));
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (i + q < a.n) add(j, q, lut_get<SMEM_LUT>(s_lut, a.lut, lo + col[i + q]));
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < SEGS; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long i = wbase + 128 * j + 4 * lane + q;
      if (SUMF) st[j][q] = (i < a.n && st[j][q] < a.fail_limit) ? st[j][q] : FAIL;
      else st[j][q] = (i < a.n) ? ((anyf[j][q] & FAIL) | st[j][q]) : FAIL;
    }
  if (lane == 0) s_warp_first[warp] = st[0][0];
  if (lane == 31) s_warp_last[warp] = st[SEGS - 1][3];
  __syncthreads();
  const u32 warp_prev = warp == 0 ? m.prev_status : s_warp_last[warp - 1];
  const u32 warp_next = warp == S1_THREADS / 32 - 1 ? m.next_status : s_warp_first[warp + 1];
  auto fstart_of = [&](int f) -> long long {
    if (overflow) return a.file_off[f];
    return f == m.fa ? m.fbase : s_fstart[f - m.fa - 1];
  };
  // 4. run boundaries
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
    if (nf == 0) {
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
      int f = overflow ? upper_bound_ll(a.file_off, a.n_files + 1, i0) - 1 : m.fa + upper_bound_ll(s_fstart, nf, i0);
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
          fs_next = k < nf && s_fstart[k] == i + 1;
          if (fs_next) fn = f + 1;
          while (fs_next && fn - m.fa < nf && s_fstart[fn - m.fa] == i + 1) ++fn;
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
  // 5. tile-local compaction into this tile's slot region [tile*TILE, ...):
  //    no inter-tile dependency. Run ends that fall in a later tile are
  //    patched by slot_fixup_kernel; the first radix pass compacts the slots.
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
  __shared__ u32 s_last_open;
  if (lane == 0) s_warp_tot[warp] = acc;
  if (warp == S1_THREADS / 32 - 1 && lane == 31)  // holder of the tile's last sample
    s_last_open = (!(st[SEGS - 1][3] & FAIL) && !((ends[SEGS - 1] >> 3) & 1)) ? 1u : 0u;
  __syncthreads();
  if (warp == 0) {
    const u32 x = lane < S1_THREADS / 32 ? s_warp_tot[lane] : 0;
    const u32 inc = warp_incl_scan(x);
    if (lane < S1_THREADS / 32) s_warp_tot[lane] = inc - x;
    if (lane == 31) {
      a.tile_cnt[tile] = inc;
      a.tile_open[tile] = (inc > 0 && s_last_open) ? 1u : 0u;  // last run ends in a later tile
    }
  }
  if (tid == 0) {  // does the tile start inside a run begun in an earlier tile?
    const u32 first = st[0][0];
    a.tile_head[tile] = (!(first & FAIL) && !(starts[0] & 1)) ? -1 : 0;
  }
  __syncthreads();
  const u64 tbase = (u64)tile * TILE;
  const u64 base = tbase + s_warp_tot[warp];
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

// Exclusive scan of per-tile run counts (single CTA; ntiles is N / 4096).
__global__ void __launch_bounds__(1024) tile_offsets_kernel(long long n, const u32* cnt, u64* off) {
  __shared__ u64 s_w[32];
  __shared__ u64 s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (long long b = 0; b < n; b += 1024) {
    const long long i = b + threadIdx.x;
    const u64 v = i < n ? cnt[i] : 0;
    const u64 inc = warp_incl_scan(v);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const u64 x = s_w[lane];
      const u64 xi = warp_incl_scan(x);
      s_w[lane] = xi - x;
    }
    __syncthreads();
    const u64 ex = s_carry + s_w[warp] + inc - v;
    if (i < n) off[i] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[n] = s_carry;
}

// Dense copy of the slot records (one warp per tile, order preserved).
__global__ void slot_compact_kernel(long long ntiles, long long tile_len, const u32* cnt, const u64* off,
                                    const u32* k, const u32* f, const u32* s, const u32* e, u32* k2, u32* f2, u32* s2,
                                    u32* e2) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long t = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += warps) {
    const u32 c = cnt[t];
    const u64 src = (u64)t * tile_len, dst = off[t];
    for (u32 i = threadIdx.x & 31; i < c; i += 32) {
      k2[dst + i] = k[src + i];
      f2[dst + i] = f[src + i];
      s2[dst + i] = s[src + i];
      e2[dst + i] = e[src + i];
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
