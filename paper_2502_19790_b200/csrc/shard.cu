// Multi-GPU (file-sharded) index and chunk emission, SURVEY.md §8(e).
//
// Stage 1 shards by file: intervals never cross files (catalog.py:559-604),
// so rank r indexes its contiguous global file range [file_lo, file_hi) alone.
// The RangeCursor layout of a key (index.py:134-144) interleaves the key's
// files of ALL ranks in one seeded order, so every rank needs every key's
// global (file, samples) list -- but not the other ranks' intervals. The one
// exchange is an all-gather of per-(key, file) BLOCK tables
// (packed key, global file, samples, intervals); each rank then builds a
// HYBRID index: its own intervals, plus one pseudo-interval [0, samples) per
// remote block. The hybrid index has the global keys, blocks, per-key totals
// and therefore the global cursor shuffle, stream offsets and chunk plan --
// bit-identical to a single-GPU index of the whole catalog -- while emission
// cuts only the pieces that fall into local intervals (GenData::lcnt/lpos,
// stage2.cu walk_term). Normalisation (sort + adjacent merge per file) is
// local because a file lives on one rank. mx_chunks_merge then interleaves
// the per-rank chunk CSRs on the root GPU into the global (mixture key, file,
// start) order.
//
// Kernels (all memory-bound, tiny next to stage 1):
//  block_table_kernel    -- local (key, file) blocks -> u32x4 rows
//  shard_dir_kernel      -- D[q][g] = first row of global key g in list q
//  shard_offsets_kernel  -- exclusive scan of counts in (key, rank) order
//  shard_copy_kernel     -- per (key, rank): rows / local intervals -> hybrid
//  local_scan_kernel     -- (gen) prefix count of local intervals in cursor
//                           order + their positions
//  merge_warp/big_kernel -- interleave of the per-rank chunk CSRs (warp per chunk; CTA per chunk above 32 pieces)
#include <stdlib.h>

#include "common.cuh"
#include "mixtera_internal.cuh"
#include "scan.cuh"

namespace mx {

// (index_finalize: mixtera_internal.cuh)

__global__ void block_table_kernel(long long B, const u32* blk_key, const u32* key_packed, const u32* blk_file,
                                   const u32* blk_first, const u64* iv_cum, u32 file_base, uint4* out) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= B) return;
  const u32 f0 = blk_first[b], f1 = blk_first[b + 1];
  out[b] = make_uint4(key_packed[blk_key[b]], file_base + blk_file[b], (u32)(iv_cum[f1] - iv_cum[f0]), f1 - f0);
}

// first index in [0, n) with v[idx] >= x
template <typename T>
__device__ __forceinline__ long long lower_bound_dev(const T* v, long long n, T x) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (v[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct ShardArgs {
  int world, rank;
  long long Kg;
  const u32* gkeys;       // [Kg] sorted global packed keys
  const uint4* tables;    // [world][cap] rows (packed key, gfile, samples, n_iv)
  long long cap;
  const long long* counts;  // device [world]
  // local index
  long long K_loc, I_loc;
  const u32* loc_key_packed;
  const u32* loc_key_blk_first;
  const u32* loc_blk_first;
  const u32* loc_iv_key;
  const u32* loc_iv_file;
  const u32* loc_iv_start;
  const u32* loc_iv_end;
  u32 file_lo;
  u32* D;           // [world][Kg+1]
  u64* OFF;         // [Kg*world + 1]
  // hybrid outputs
  u32 *h_key, *h_file, *h_start, *h_end, *h_nreal;
};

__global__ void shard_dir_kernel(ShardArgs a) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long row = a.Kg + 1;
  if (t >= (long long)a.world * row) return;
  const int q = (int)(t / row);
  const long long g = t % row;
  u32 d;
  if (q == a.rank) {
    if (g == a.Kg) {
      d = (u32)a.I_loc;
    } else {
      const long long kr = lower_bound_dev<u32>(a.loc_key_packed, a.K_loc, a.gkeys[g]);
      d = kr < a.K_loc ? a.loc_blk_first[a.loc_key_blk_first[kr]] : (u32)a.I_loc;
    }
  } else {
    const long long n = a.counts[q];
    if (g == a.Kg) {
      d = (u32)n;
    } else {  // lower bound of gkeys[g] in list q's key column
      const uint4* T = a.tables + (long long)q * a.cap;
      long long lo = 0, hi = n;
      const u32 x = a.gkeys[g];
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (T[mid].x < x) lo = mid + 1; else hi = mid;
      }
      d = (u32)lo;
    }
  }
  a.D[t] = d;
}

// single CTA: OFF[g*W + q] = exclusive prefix of count(g, q) in (g, q) order
__global__ void __launch_bounds__(1024) shard_offsets_kernel(ShardArgs a) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_carry;
  const long long n = a.Kg * a.world;
  const long long row = a.Kg + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (long long base = 0; base < n; base += 1024) {
    const long long i = base + threadIdx.x;
    u64 v = 0;
    if (i < n) {
      const long long g = i / a.world;
      const int q = (int)(i % a.world);
      v = a.D[q * row + g + 1] - a.D[q * row + g];
    }
    const u64 inc = warp_incl_scan(v);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const u64 x = s_w[lane];
      const u64 xi = warp_incl_scan(x);
      s_w[lane] = xi - x;
      if (lane == 31) s_w[32] = xi;
    }
    __syncthreads();
    if (i < n) a.OFF[i] = s_carry + s_w[warp] + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.OFF[n] = s_carry;
}

// One CTA per (global key g, rank q): copy rank q's rows (or, for this rank,
// its intervals) of key g to [OFF[g][q], ...) -- contiguous in and out, no
// search per element.
__global__ void __launch_bounds__(128) shard_copy_kernel(ShardArgs a) {
  const long long g = blockIdx.x / a.world;
  const int q = blockIdx.x % a.world;
  const long long row = a.Kg + 1;
  const u32* Dq = a.D + q * row;
  const u32 e0 = Dq[g], e1 = Dq[g + 1];
  const u64 dst = a.OFF[g * a.world + q];
  if (q == a.rank) {
    for (u32 e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const u64 o = dst + (e - e0);
      a.h_key[o] = a.loc_iv_key[e];
      a.h_file[o] = a.file_lo + a.loc_iv_file[e];
      a.h_start[o] = a.loc_iv_start[e];
      a.h_end[o] = a.loc_iv_end[e];
      a.h_nreal[o] = 1;
    }
  } else {
    const uint4* T = a.tables + (long long)q * a.cap;
    for (u32 e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const uint4 r = T[e];
      const u64 o = dst + (e - e0);
      a.h_key[o] = r.x;
      a.h_file[o] = r.y;
      a.h_start[o] = 0;
      a.h_end[o] = r.z;
      a.h_nreal[o] = r.w;
    }
  }
}

int index_block_table(const IndexData* ix, u32 file_base, uint4* out, cudaStream_t s) {
  const long long B = ix->n_blocks;
  if (B == 0) return MX_OK;
  block_table_kernel<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(B, ix->blk_key.p, ix->key_packed.p, ix->blk_file.p,
                                                                 ix->blk_first.p, ix->iv_cum.p, file_base, out);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

int index_build_sharded(const IndexData* loc, const mx_shard_desc* d, cudaStream_t s, IndexData* out) {
  const int W = d->world;
  const long long Kg = d->n_global_keys;
  IndexData& h = *out;
  h.stream = s;
  h.sharded = true;
  h.file_lo = d->file_lo;
  h.n_local = loc->n_intervals;
  h.file_hi = d->file_hi;
  h.n_files = d->n_files;
  h.key_bits = loc->key_bits;
  h.n_props = loc->n_props;
  for (int p = 0; p < MX_MAX_PROPS; ++p) {
    h.field_shift[p] = loc->field_shift[p];
    h.field_width[p] = loc->field_width[p];
    h.str_base[p] = loc->str_base[p];
  }
  MX_CUDA_TRY(h.str_off.alloc(loc->str_off.n, s));
  MX_CUDA_TRY(h.str_bytes.alloc(loc->str_bytes.n, s));
  MX_CUDA_TRY(cudaMemcpyAsync(h.str_off.p, loc->str_off.p, sizeof(long long) * loc->str_off.n,
                              cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(cudaMemcpyAsync(h.str_bytes.p, loc->str_bytes.p, loc->str_bytes.n, cudaMemcpyDeviceToDevice, s));
  h.h_file_ds.assign(d->file_ds, d->file_ds + d->n_files);
  h.h_file_ids.assign(d->file_ids, d->file_ids + d->n_files);
  MX_CUDA_TRY(h.file_ids.alloc(d->n_files, s));
  MX_CUDA_TRY(mx_h2d(h.file_ids.p, d->file_ids, sizeof(long long) * d->n_files, s));
  MX_CUDA_TRY(h.file_ds.alloc(d->n_files, s));
  MX_CUDA_TRY(mx_h2d(h.file_ds.p, d->file_ds, sizeof(int32_t) * d->n_files, s));
  if (Kg == 0) {
    h.n_intervals = h.n_keys = h.n_blocks = 0;
    return MX_OK;
  }
  DevBuf<u32> gkeys, D;
  DevBuf<u64> OFF;
  DevBuf<long long> counts;
  MX_CUDA_TRY(gkeys.alloc(Kg, s));
  MX_CUDA_TRY(D.alloc((long long)W * (Kg + 1), s));
  MX_CUDA_TRY(OFF.alloc(Kg * W + 1, s));
  MX_CUDA_TRY(counts.alloc(W, s));
  MX_CUDA_TRY(mx_h2d(gkeys.p, d->global_keys, sizeof(u32) * Kg, s));
  MX_CUDA_TRY(mx_h2d(counts.p, d->counts, sizeof(long long) * W, s));
  ShardArgs a{};
  a.world = W;
  a.rank = d->rank;
  a.Kg = Kg;
  a.gkeys = gkeys.p;
  a.tables = reinterpret_cast<const uint4*>(d->tables);
  a.cap = d->cap;
  a.counts = counts.p;
  a.K_loc = loc->n_keys;
  a.I_loc = loc->n_intervals;
  a.loc_key_packed = loc->key_packed.p;
  a.loc_key_blk_first = loc->key_blk_first.p;
  a.loc_blk_first = loc->blk_first.p;
  a.loc_iv_key = loc->iv_key.p;
  a.loc_iv_file = loc->iv_file.p;
  a.loc_iv_start = loc->iv_start.p;
  a.loc_iv_end = loc->iv_end.p;
  a.file_lo = (u32)d->file_lo;
  a.D = D.p;
  a.OFF = OFF.p;
  const long long nd = (long long)W * (Kg + 1);
  shard_dir_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, s>>>(a);
  mx_count_launch();
  shard_offsets_kernel<<<1, 1024, 0, s>>>(a);
  mx_count_launch();
  u64 I = 0;
  MX_CUDA_TRY(cudaMemcpyAsync(&I, OFF.p + Kg * W, sizeof(u64), cudaMemcpyDeviceToHost, s));
  MX_CUDA_TRY(cudaStreamSynchronize(s));
  if (I >= (1ull << 32)) return mx_fail(MX_ERR_UNSUPPORTED, "hybrid index with %llu intervals (>= 2^32)", I);
  MX_CUDA_TRY(h.iv_key.alloc(I, s));
  MX_CUDA_TRY(h.iv_file.alloc(I, s));
  MX_CUDA_TRY(h.iv_start.alloc(I, s));
  MX_CUDA_TRY(h.iv_end.alloc(I, s));
  MX_CUDA_TRY(h.iv_nreal.alloc(I, s));
  a.h_key = h.iv_key.p;
  a.h_file = h.iv_file.p;
  a.h_start = h.iv_start.p;
  a.h_end = h.iv_end.p;
  a.h_nreal = h.iv_nreal.p;
  if ((long long)W * d->cap + a.I_loc > 0) {
    shard_copy_kernel<<<(unsigned)(Kg * W), 128, 0, s>>>(a);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaGetLastError());
  int rc = index_finalize(&h, (long long)I, s);
  if (rc != MX_OK) return rc;
  h.n_samples_total = 0;
  return MX_OK;
}

// ------------------------------------------------------------------ generator
// value = (real intervals << 32) | is_local for cursor position j:
// lcnt[j] = local positions before j, lpos[r] = position of the r-th local
// one, rcum[j] = real intervals before j (totals < 2^32 each)
struct LocalF {
  const u32* civ;
  const u32* iv_file;
  const u32* nreal;
  u32 flo, fhi;
  u32 *lcnt, *lpos;
  u64* rcum;
  long long n;
  __device__ u64 value(long long j) const {
    const u32 iv = civ[j];
    const u32 f = iv_file[iv];
    return ((u64)nreal[iv] << 32) | (u64)(f >= flo && f < fhi);
  }
  __device__ void apply(long long j, u64 ex, u64 v) const {
    lcnt[j] = (u32)ex;
    rcum[j] = ex >> 32;
    if (v & 1) lpos[(u32)ex] = (u32)j;
  }
  __device__ void total(u64 t) const {
    lcnt[n] = (u32)t;
    rcum[n] = t >> 32;
  }
};

__global__ void gather_u64_kernel(long long n, const u32* idx, const u64* src, u64* dst) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

int gen_local_lists(GenData* g, cudaStream_t s) {
  IndexData* ix = g->ix;
  const long long I = ix->n_intervals;
  if (!ix->sharded || I == 0) return MX_OK;
  MX_CUDA_TRY(g->lcnt.alloc(I + 1, s));
  MX_CUDA_TRY(g->lpos.alloc(I, s));
  MX_CUDA_TRY(g->rcum.alloc(I + 1, s));
  if (int rc = gs_run(I, LocalF{g->civ.p, ix->iv_file.p, ix->iv_nreal.p, (u32)ix->file_lo, (u32)ix->file_hi,
                                g->lcnt.p, g->lpos.p, g->rcum.p, I}, s))
    return rc;
  MX_CUDA_TRY(g->lstart.alloc(ix->n_local > 0 ? ix->n_local : 1, s));
  if (ix->n_local > 0) {
    gather_u64_kernel<<<(unsigned)((ix->n_local + 255) / 256), 256, 0, s>>>(ix->n_local, g->lpos.p, g->ccum.p,
                                                                          g->lstart.p);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

// ------------------------------------------------------------------ root merge
// out_off[c] = sum over ranks of off_q[c] (per-rank CSRs of the same chunks)
__global__ void merge_offsets_kernel(int W, long long C, const long long* offs, long long* out_off) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c > C) return;
  long long t = 0;
  for (int q = 0; q < W; ++q) t += offs[(long long)q * (C + 1) + c];
  out_off[c] = t;
}

// Chunks with more than 32 pieces: one CTA per chunk. Pieces of rank q's
// chunk c are sorted by (mixture key, file, start) and all of rank q's files
// precede rank q+1's: a piece's global position is its chunk's base + pieces
// of other ranks with a smaller mixture key (or an equal one on a lower rank)
// + its index in its own chunk.
__global__ void __launch_bounds__(256)
merge_big_kernel(int W, long long C, long long cap, const long long* offs, const long long* out_off, const u32* mkey,
                 const u32* file, const u32* start, const u32* end, u32* o_mkey, u32* o_file, u32* o_start,
                 u32* o_end, const u32* big_list, const u32* big_cnt) {
  const u32 nb = *big_cnt;
  for (u32 bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const long long c = big_list[bi];
    for (int q = 0; q < W; ++q) {
      const long long* oq = offs + (long long)q * (C + 1);
      for (long long i = oq[c] + threadIdx.x; i < oq[c + 1]; i += blockDim.x) {
        const long long t = (long long)q * cap + i;
        const u32 m = mkey[t];
        long long pos = out_off[c] + (i - oq[c]);
        for (int r = 0; r < W; ++r) {
          if (r == q) continue;
          const long long* orr = offs + (long long)r * (C + 1);
          const u32* mk = mkey + (long long)r * cap;
          long long a0 = orr[c], a1 = orr[c + 1];
          while (a0 < a1) {  // r < q: keys <= m come first; r > q: keys < m
            const long long mid = (a0 + a1) >> 1;
            const bool before = r < q ? mk[mid] <= m : mk[mid] < m;
            if (before) a0 = mid + 1; else a1 = mid;
          }
          pos += a0 - orr[c];
        }
        o_mkey[pos] = m;
        o_file[pos] = file[t];
        o_start[pos] = start[t];
        o_end[pos] = end[t];
      }
    }
  }
}

// One warp per chunk when the chunk has <= 32 pieces over all ranks (the
// common case): lane i takes piece i of the rank-major concatenation and its
// position is #{k: m_k < m_i} + #{k < i: m_k == m_i} (a stable sort by
// mixture key); larger chunks are listed for merge_big_kernel.
__global__ void __launch_bounds__(256)
merge_warp_kernel(int W, long long C, long long cap, const long long* offs, const long long* out_off, const u32* mkey,
                  const u32* file, const u32* start, const u32* end, u32* o_mkey, u32* o_file, u32* o_start,
                  u32* o_end, u32* big_list, u32* big_cnt) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < C; c += warps) {
    const long long n = out_off[c + 1] - out_off[c];
    if (n > 32) {
      if (lane == 0) big_list[atomicAdd(big_cnt, 1u)] = (u32)c;
      continue;
    }
    // lane -> (rank q, index j in q's arrays): lanes q < W load rank q's
    // segment, a warp scan gives the segment starts in the concatenation
    long long src = -1;
    long long seg_a = 0, seg_len = 0, carry = 0;
    for (int q0 = 0; q0 < W; q0 += 32) {
      const int q = q0 + lane;
      if (q < W) {
        const long long* oq = offs + (long long)q * (C + 1);
        seg_a = oq[c];
        seg_len = oq[c + 1] - seg_a;
      } else {
        seg_len = 0;
      }
      const long long incl = warp_incl_scan(seg_len);
      const long long excl = incl - seg_len + carry;
      // every lane finds the rank segment holding its concatenated index
      for (int r = 0; r < 32 && q0 + r < W; ++r) {
        const long long b = __shfl_sync(MX_FULL, excl, r), l = __shfl_sync(MX_FULL, seg_len, r);
        const long long a = __shfl_sync(MX_FULL, seg_a, r);
        if (lane >= b && lane < b + l) src = (long long)(q0 + r) * cap + a + (lane - b);
      }
      carry += __shfl_sync(MX_FULL, incl, 31);
    }
    const bool mine = lane < n;
    const u32 m = mine ? mkey[src] : 0xffffffffu;
    int pos = 0;
    for (int k = 0; k < (int)n; ++k) {
      const u32 mk = __shfl_sync(MX_FULL, m, k);
      pos += (mk < m) || (mk == m && k < lane);
    }
    if (mine) {
      const long long dst = out_off[c] + pos;
      o_mkey[dst] = m;
      o_file[dst] = file[src];
      o_start[dst] = start[src];
      o_end[dst] = end[src];
    }
  }
}

// One CTA per tile of MT_CHUNKS consecutive chunks: every rank's pieces of
// the tile are one contiguous range, so they are read coalesced into shared
// memory, positioned there (per piece: its chunk by a search in the tile's
// offsets, then the counts of the other ranks' pieces of that chunk ordered
// before it), and the tile's output range is written back coalesced. Tiles
// whose pieces exceed the staging capacity use merge_seg_kernel's logic on
// global memory.
constexpr int MT_CHUNKS = 64;
constexpr int MT_CAP = 2048;   // staged pieces per tile
constexpr int MT_MAXW = 16;

__global__ void __launch_bounds__(256)
merge_tile_kernel(int W, long long C, long long cap, const long long* offs, const long long* out_off,
                  const u32* mkey, const u32* file, const u32* start, const u32* end, u32* o_mkey, u32* o_file,
                  u32* o_start, u32* o_end) {
  __shared__ u32 s_m[MT_CAP], s_f[MT_CAP], s_s[MT_CAP], s_e[MT_CAP];
  __shared__ u32 s_pos[MT_CAP];
  __shared__ int s_off[MT_MAXW][MT_CHUNKS + 1];  // tile-relative piece offsets per rank
  __shared__ int s_rb[MT_MAXW + 1];              // rank bases in the staging arrays
  const long long c0 = (long long)blockIdx.x * MT_CHUNKS;
  const int nc = (int)min((long long)MT_CHUNKS, C - c0);
  {  // tile-relative offsets: all loads of a thread issued before its stores
    constexpr int PER = (MT_MAXW * (MT_CHUNKS + 1) + 255) / 256;
    long long v[PER], b0[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = threadIdx.x + u * 256;
      if (i < W * (nc + 1)) {
        const int q = i / (nc + 1), k = i % (nc + 1);
        const long long* oq = offs + (long long)q * (C + 1);
        v[u] = oq[c0 + k];
        b0[u] = oq[c0];
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = threadIdx.x + u * 256;
      if (i < W * (nc + 1)) s_off[i / (nc + 1)][i % (nc + 1)] = (int)(v[u] - b0[u]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < W; ++q) {
      s_rb[q] = acc;
      acc += s_off[q][nc];
    }
    s_rb[W] = acc;
  }
  __syncthreads();
  const int total = s_rb[W];
  const long long obase = out_off[c0];
  if (total > MT_CAP) {  // dense tile: position pieces straight from global memory
    for (int q = 0; q < W; ++q) {
      const long long* oq = offs + (long long)q * (C + 1);
      for (int i = threadIdx.x; i < s_off[q][nc]; i += blockDim.x) {
        int lo = 0, hi = nc;  // chunk k: off[k] <= i < off[k+1]
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_off[q][mid] <= i) lo = mid; else hi = mid - 1;
        }
        const long long c = c0 + lo;
        const long long src = (long long)q * cap + oq[c0] + i;
        const u32 m = mkey[src];
        long long pos = out_off[c] + (i - s_off[q][lo]);
        for (int r = 0; r < W; ++r) {
          if (r == q) continue;
          const long long* orr = offs + (long long)r * (C + 1);
          const u32* mk = mkey + (long long)r * cap;
          long long a = orr[c], b = orr[c + 1];
          const long long s0 = a;
          while (a < b) {
            const long long mid = (a + b) >> 1;
            const bool before = r < q ? mk[mid] <= m : mk[mid] < m;
            if (before) a = mid + 1; else b = mid;
          }
          pos += a - s0;
        }
        o_mkey[pos] = m;
        o_file[pos] = file[src];
        o_start[pos] = start[src];
        o_end[pos] = end[src];
      }
    }
    return;
  }
  // stage: every rank's range is contiguous (coalesced); a thread issues the
  // loads of all its items before storing them
  {
    constexpr int PER = MT_CAP / 256;
    uint4 v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int t = threadIdx.x + u * 256;
      if (t < total) {
        int q = 0;
        while (s_rb[q + 1] <= t) ++q;
        const long long g = (long long)q * cap + offs[(long long)q * (C + 1) + c0] + (t - s_rb[q]);
        v[u] = make_uint4(mkey[g], file[g], start[g], end[g]);
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int t = threadIdx.x + u * 256;
      if (t < total) {
        s_m[t] = v[u].x;
        s_f[t] = v[u].y;
        s_s[t] = v[u].z;
        s_e[t] = v[u].w;
      }
    }
  }
  __syncthreads();
  // one warp per chunk of the tile: lane i takes piece i of the chunk's
  // rank-major concatenation; position = pieces with a smaller mixture key +
  // pieces with the same key on an earlier lane (stable sort by key)
  __shared__ u32 s_list[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < nc; k += 8) {
    int len = 0, st = 0;
    if (lane < W) {
      st = s_rb[lane] + s_off[lane][k];
      len = s_off[lane][k + 1] - s_off[lane][k];
    }
    const int inc = warp_incl_scan(len);
    const int n = __shfl_sync(MX_FULL, inc, 31);
    const int base = (int)(out_off[c0 + k] - obase);
    if (n <= 32) {
      for (int j = 0; j < len; ++j) s_list[warp][inc - len + j] = (u32)(st + j);
      __syncwarp();
      const bool mine = lane < n;
      const u32 t = mine ? s_list[warp][lane] : 0;
      const u32 m = mine ? s_m[t] : 0xffffffffu;
      const u32 lt = (1u << lane) - 1u;
      const u32 peers = __match_any_sync(MX_FULL, m);
      int below = 0;
      u32 rest = __ballot_sync(MX_FULL, mine);
      while (rest) {  // one step per distinct key of the chunk
        const int ld = __ffs(rest) - 1;
        const u32 mv = __shfl_sync(MX_FULL, m, ld);
        const u32 grp = __ballot_sync(MX_FULL, mine && m == mv);
        if (mv < m) below += __popc(grp);
        rest &= ~grp;
      }
      if (mine) s_pos[t] = (u32)(base + below + __popc(peers & lt));
      __syncwarp();
    } else {  // long chunk: per piece over the ranks' segments in shared memory
      for (int q = 0; q < W; ++q) {
        const int a = s_rb[q] + s_off[q][k], e = s_rb[q] + s_off[q][k + 1];
        for (int t = a + lane; t < e; t += 32) {
          const u32 m = s_m[t];
          int pos = base + (t - a);
          for (int r = 0; r < W; ++r) {
            if (r == q) continue;
            const int ra = s_rb[r] + s_off[r][k], re = s_rb[r] + s_off[r][k + 1];
            int lo = ra, hi = re;
            while (lo < hi) {
              const int mid = (lo + hi) >> 1;
              const bool before = r < q ? s_m[mid] <= m : s_m[mid] < m;
              if (before) lo = mid + 1; else hi = mid;
            }
            pos += lo - ra;
          }
          s_pos[t] = (u32)pos;
        }
      }
    }
  }
  __syncthreads();
  // scatter into the staging arrays' output order via a second pass: the
  // output range of the tile is [obase, obase + total)
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const long long o = obase + s_pos[t];
    o_mkey[o] = s_m[t];
    o_file[o] = s_f[t];
    o_start[o] = s_s[t];
    o_end[o] = s_e[t];
  }
}

int chunks_merge(int W, long long C, long long cap, const long long* offs, const u32* mkey, const u32* file,
                 const u32* start, const u32* end, long long* out_off, u32* o_mkey, u32* o_file, u32* o_start,
                 u32* o_end, cudaStream_t s) {
  merge_offsets_kernel<<<(unsigned)((C + 256) / 256), 256, 0, s>>>(W, C, offs, out_off);
  mx_count_launch();
  const long long n = (long long)W * cap;
  if (n > 0 && C > 0 && W <= MT_MAXW && !getenv("MX_MERGE_WARP")) {
    merge_tile_kernel<<<(unsigned)((C + MT_CHUNKS - 1) / MT_CHUNKS), 256, 0, s>>>(
        W, C, cap, offs, out_off, mkey, file, start, end, o_mkey, o_file, o_start, o_end);
    mx_count_launch();
  } else if (n > 0 && C > 0) {
    DevBuf<u32> blist, bcnt;
    MX_CUDA_TRY(blist.alloc(C, s));
    MX_CUDA_TRY(bcnt.alloc(1, s));
    MX_CUDA_TRY(cudaMemsetAsync(bcnt.p, 0, sizeof(u32), s));
    const long long wgrid = std::min<long long>((C + 7) / 8, 148 * 16);
    merge_warp_kernel<<<(unsigned)wgrid, 256, 0, s>>>(W, C, cap, offs, out_off, mkey, file, start, end, o_mkey, o_file,
                                                     o_start, o_end, blist.p, bcnt.p);
    mx_count_launch();
    merge_big_kernel<<<(unsigned)std::min<long long>(C, 148 * 4), 256, 0, s>>>(
        W, C, cap, offs, out_off, mkey, file, start, end, o_mkey, o_file, o_start, o_end, blist.p, bcnt.p);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // namespace mx
