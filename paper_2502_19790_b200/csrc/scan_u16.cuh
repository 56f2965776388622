// Stage-1 streaming pass for ONE u16 code column (the row-tuple layout, the
// bench's layout), included by stage1.cu.
//
// At 2 bytes per sample the per-sample work has to be a handful of
// instructions or the pass is issue bound, not HBM bound. A sample can only
// start or end a run where its tuple code differs from its predecessor's
// (distinct tuples have distinct full keys) or at a file start, so the
// common path never touches the key LUT:
//
//  * each thread holds 8 consecutive codes from ONE 16-byte load
//    (ld.global.nc.L1::no_allocate.v4) and finds code changes with four
//    __byte_perm + four __vcmpne2 (two 16-bit compares per instruction);
//  * only at a change (or a file start) does a lane read the LUT (staged in
//    shared memory) for the two keys and decide whether it is a real run
//    boundary -- a key change with either side passing the filter, a pass /
//    fail switch, or a file start next to a passing sample;
//  * the boundaries of the tile are compacted into shared memory in sample
//    order with one packed warp scan (boundary count | record count) and one
//    CTA-wide combine; then one thread per boundary writes a record: a
//    boundary whose sample passes starts a run that ends at the NEXT
//    boundary (or at the tile end, or later: slot_fixup_kernel).
//
// Persistent CTAs walk the full tiles grid-stride and keep the next tile's
// 16-byte load (and its two halo codes) in flight while finishing the
// current one. Tile = 256 threads x 8 samples = 2048 samples, the tile_len
// of tile_meta_kernel / slot_fixup_kernel / scan_list_kernel, and the same
// slot contract as scan_fast_kernel: tile_cnt, tile_open, tile_head, records
// at [tile * 2048, ...).
#pragma once

namespace mx {

constexpr int U16_THREADS = 256;
constexpr int U16_TILE = U16_THREADS * 8;  // 2048
constexpr int U16_SMEM_LUT_MAX = 16384;    // entries staged per CTA (64 KB)

struct U16Scratch {
  uint16_t ev_idx[U16_TILE];   // boundaries in sample order (tile-local index)
  uint16_t ev_rank[U16_TILE];  // record slot of a boundary that starts a run, else 0xffff
  u32 ev_key[U16_TILE];        // packed key of that run
  u32 wtot[U16_THREADS / 32];  // per-warp packed (boundaries | records << 16)
  u32 end_real;                // the tile end (sample t0 + 2048) is a run boundary
};

__device__ __forceinline__ u32 u16_at(const uint4& w, int q) {
  const u32 x = q < 4 ? (q < 2 ? w.x : w.y) : (q < 6 ? w.z : w.w);
  return (x >> ((q & 1) * 16)) & 0xffffu;
}

// file starts of the tile (at most FAST_MAX_FS, tile-local, in (0, 2048)):
// k-th start via the L1 path (uniform per tile, only when m.nf > 0)
__device__ __forceinline__ int u16_fs(const S1Args& a, const TileMeta& m, long long t0, int k) {
  return (int)(__ldg(a.file_off + m.fa + 1 + k) - t0);
}

template <bool SLUT>
__device__ __forceinline__ u32 u16_key(const u32* s_lut, const u32* g_lut, u32 code) {
  return SLUT ? s_lut[code] : __ldg(g_lut + code);
}

template <bool SLUT>
__global__ void __launch_bounds__(U16_THREADS, 8)
scan_u16_kernel(S1Args a, const TileMeta* __restrict__ meta, long long nfull) {
  extern __shared__ __align__(16) u32 s_lut[];
  __shared__ U16Scratch sc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint16_t* __restrict__ col = reinterpret_cast<const uint16_t*>(a.cols[0]);
  const u32* __restrict__ g_lut = a.lut_sum + 1;  // entry for code c at c (no null code in a tuple column)
  const u32 lim = a.fail_limit;
  const int lb = tid * 8;  // tile-local index of this thread's first sample
  if (SLUT)
    for (int i = tid; i < a.lut_off[1] - 1; i += U16_THREADS) s_lut[i] = g_lut[i];
  long long tile = blockIdx.x;
  // prefetched state of the next tile: its 8 codes, the halo code (lane 0 of
  // each warp: the code before its first sample; thread 255: the code after
  // the tile) and its file metadata
  uint4 w = make_uint4(0, 0, 0, 0);
  u32 halo = 0;
  long long mfbase = 0;
  int mfa = 0, mnf = 0;
  auto fetch = [&](long long t) {
    const long long t0 = t * U16_TILE;
    const int4 v = ld_stream_v4(reinterpret_cast<const int4*>(col + t0 + lb));
    w = make_uint4((u32)v.x, (u32)v.y, (u32)v.z, (u32)v.w);
    if (lane == 0) halo = t0 + lb > 0 ? (u32)__ldg(col + t0 + lb - 1) : 0u;
    if (tid == U16_THREADS - 1) halo = t0 + U16_TILE < a.n ? (u32)__ldg(col + t0 + U16_TILE) : 0u;
    mfbase = __ldg(&meta[t].fbase);
    mfa = __ldg(&meta[t].fa);
    mnf = __ldg(&meta[t].nf);
  };
  if (tile < nfull) fetch(tile);
  __syncthreads();  // LUT staged
  for (; tile < nfull; tile += gridDim.x) {
    const long long t0 = tile * U16_TILE;
    TileMeta m;
    m.fbase = mfbase;
    m.fa = mfa;
    m.nf = mnf;
    const uint4 cw = w;
    const u32 chalo = halo;
    const long long nxt = tile + gridDim.x;
    if (nxt < nfull) fetch(nxt);
    if (m.nf > FAST_MAX_FS) {  // CTA-uniform: many tiny files, left to scan_list_kernel
      if (tid == 0) a.defer_list[atomicAdd(a.defer_cnt, 1u)] = (u32)tile;
      continue;
    }
    // ---- code changes: bit q = code[q] != code[q - 1]
    u32 prev = __shfl_up_sync(MX_FULL, cw.w >> 16, 1);
    if (lane == 0) prev = chalo;
    const u32 g0 = __byte_perm(prev << 16, cw.x, 0x5432), g1 = __byte_perm(cw.x, cw.y, 0x5432);
    const u32 g2 = __byte_perm(cw.y, cw.z, 0x5432), g3 = __byte_perm(cw.z, cw.w, 0x5432);
    const u32 t = (__vcmpne2(cw.x, g0) & 0x10001u) | ((__vcmpne2(cw.y, g1) & 0x10001u) << 2) |
                  ((__vcmpne2(cw.z, g2) & 0x10001u) << 4) | ((__vcmpne2(cw.w, g3) & 0x10001u) << 6);
    u32 cand = (t & 0x55u) | ((t >> 15) & 0xaau);
    if (tid == 0 && t0 == 0) cand |= 1u;  // sample 0 has no predecessor
    // ---- file starts of this thread's samples
    u32 fsb = (t0 + lb == m.fbase) ? 1u : 0u;
    for (int k = 0; k < m.nf; ++k) {
      const int d = u16_fs(a, m, t0, k) - lb;
      if (d >= 0 && d < 8) fsb |= 1u << d;
    }
    cand |= fsb;
    // ---- real run boundaries among the candidates (LUT only here)
    u32 real = 0, recs = 0;
    for (u32 c = cand; c; c &= c - 1) {
      const int q = __ffs(c) - 1;
      const u32 cur = u16_at(cw, q), pre = q ? u16_at(cw, q - 1) : prev;
      const u32 kc = u16_key<SLUT>(s_lut, g_lut, cur);
      const bool pc = kc < lim;
      bool brk;
      if (tid == 0 && q == 0 && t0 == 0) {
        brk = pc;
      } else {
        const u32 kp = u16_key<SLUT>(s_lut, g_lut, pre);
        const bool pp = kp < lim;
        brk = (pc || pp) && (((fsb >> q) & 1u) || kc != kp);
      }
      real |= (u32)brk << q;
      recs |= (u32)(brk && pc) << q;
    }
    const u32 pack = (u32)__popc(real) | ((u32)__popc(recs) << 16);
    const u32 incl = warp_incl_scan(pack);
    if (lane == 31) sc.wtot[warp] = incl;
    if (tid == U16_THREADS - 1) {  // is sample t0 + 2048 a boundary of the run holding sample t0 + 2047?
      bool er = true;
      if (t0 + U16_TILE < a.n) {
        const u32 kl = u16_key<SLUT>(s_lut, g_lut, cw.w >> 16);
        const u32 kn = u16_key<SLUT>(s_lut, g_lut, chalo);
        const bool fs_next = m.nf > 0 && u16_fs(a, m, t0, m.nf - 1) == U16_TILE;
        er = fs_next || kl != kn;
      }
      sc.end_real = er ? 1u : 0u;
    }
    __syncthreads();
    u32 base = 0, total = 0;
#pragma unroll
    for (int v = 0; v < U16_THREADS / 32; ++v) {
      const u32 x = sc.wtot[v];
      base += v < warp ? x : 0u;
      total += x;
    }
    base += incl - pack;
    u32 ev = base & 0xffffu, rk = base >> 16;
    for (u32 c = real; c; c &= c - 1) {
      const int q = __ffs(c) - 1;
      sc.ev_idx[ev] = (uint16_t)(lb + q);
      if ((recs >> q) & 1u) {
        sc.ev_rank[ev] = (uint16_t)rk++;
        sc.ev_key[ev] = u16_key<SLUT>(s_lut, g_lut, u16_at(cw, q));
      } else {
        sc.ev_rank[ev] = 0xffffu;
      }
      ++ev;
    }
    __syncthreads();
    // ---- one thread per boundary: records into the tile's slot region
    const int nev = (int)(total & 0xffffu), nrec = (int)(total >> 16);
    const u64 tbase = (u64)tile * U16_TILE;
    for (int k = tid; k < nev; k += U16_THREADS) {
      const u32 r = sc.ev_rank[k];
      if (r == 0xffffu) continue;
      const int s = sc.ev_idx[k];
      int fo = 0;
      for (int f = 0; f < m.nf; ++f) fo += u16_fs(a, m, t0, f) <= s;
      const long long fstart = fo == 0 ? m.fbase : __ldg(a.file_off + m.fa + fo);
      const u32 off = (u32)(t0 - fstart);
      const u32 key = sc.ev_key[k];
      a.rec_key[tbase + r] = key;
      a.rec_file[tbase + r] = (u32)(m.fa + fo);
      a.rec_start[tbase + r] = off + (u32)s;
      if (k + 1 < nev) a.rec_end[tbase + r] = off + sc.ev_idx[k + 1];
      else if (sc.end_real) a.rec_end[tbase + r] = off + U16_TILE;
      if ((key & a.rank_mask) == 0) atomicMin(&a.err->null_key_sample, (u64)(t0 + s));
    }
    if (tid == 0) {
      a.tile_cnt[tile] = (u32)nrec;
      a.tile_open[tile] = (nev > 0 && sc.ev_rank[nev - 1] != 0xffffu && !sc.end_real) ? 1u : 0u;
      a.tile_head[tile] = nev == 0 ? -1 : (sc.ev_idx[0] == 0 ? 0 : t0 + sc.ev_idx[0]);
    }
  }
}

}  // namespace mx
