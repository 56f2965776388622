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
//  shard_scatter_kernel  -- rows / local intervals -> hybrid position
//  local_scan_kernel     -- (gen) prefix count of local intervals in cursor
//                           order + their positions
//  merge_*_kernel        -- root-side interleave of per-rank chunk CSRs
#include "common.cuh"
#include "mixtera_internal.cuh"

namespace mx {

int index_finalize(IndexData* ix, long long I, cudaStream_t s);

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

// rows of remote lists (q != rank) and local intervals (q == rank) to their
// hybrid position: OFF[g][q] + (index - D[q][g])
__global__ void shard_scatter_kernel(ShardArgs a) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long row = a.Kg + 1;
  const long long n_remote = (long long)a.world * a.cap;
  long long e;
  int q;
  if (t < n_remote) {
    q = (int)(t / a.cap);
    e = t % a.cap;
    if (q == a.rank || e >= a.counts[q]) return;
  } else {
    e = t - n_remote;
    q = a.rank;
    if (e >= a.I_loc) return;
  }
  const u32* Dq = a.D + q * row;
  // g: D[q][g] <= e < D[q][g+1] (empty keys skipped by the upper bound)
  long long lo = 0, hi = a.Kg + 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (Dq[mid] <= (u32)e) lo = mid + 1; else hi = mid;
  }
  const long long g = lo - 1;
  const u64 dst = a.OFF[g * a.world + q] + (u64)(e - Dq[g]);
  if (q == a.rank) {
    a.h_key[dst] = a.loc_iv_key[e];
    a.h_file[dst] = a.file_lo + a.loc_iv_file[e];
    a.h_start[dst] = a.loc_iv_start[e];
    a.h_end[dst] = a.loc_iv_end[e];
    a.h_nreal[dst] = 1;
  } else {
    const uint4 r = a.tables[(long long)q * a.cap + e];
    a.h_key[dst] = r.x;
    a.h_file[dst] = r.y;
    a.h_start[dst] = 0;
    a.h_end[dst] = r.z;
    a.h_nreal[dst] = r.w;
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
  const long long nt = (long long)W * d->cap + a.I_loc;
  if (nt > 0) {
    shard_scatter_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(a);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaGetLastError());
  int rc = index_finalize(&h, (long long)I, s);
  if (rc != MX_OK) return rc;
  h.n_samples_total = 0;
  return MX_OK;
}

// ------------------------------------------------------------------ generator
constexpr int LS_THREADS = 256;
constexpr int LS_ITEMS = 8;
constexpr int LS_TILE = LS_THREADS * LS_ITEMS;

// lcnt[j] = local intervals among cursor positions [0, j); lpos[r] = position
// of the r-th local one; rcum[j] = real intervals (pseudo-interval = its
// block's interval count) among [0, j).
__global__ void __launch_bounds__(LS_THREADS)
local_scan_kernel(const u32* civ, const u32* iv_file, const u32* nreal, long long n, u32 flo, u32 fhi, u64* status,
                  u32* tile_ctr, u32* lcnt, u32* lpos, u64* rcum) {
  __shared__ u64 s_w[LS_THREADS / 32 + 1];
  __shared__ int s_tile;
  __shared__ u64 s_excl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int tile = s_tile;
  const long long b = (long long)tile * LS_TILE + threadIdx.x * LS_ITEMS;
  // packed (real count << 32 | local flag); totals stay < 2^32 each
  u64 v[LS_ITEMS], sum = 0;
#pragma unroll
  for (int q = 0; q < LS_ITEMS; ++q) {
    const long long i = b + q;
    u64 x = 0;
    if (i < n) {
      const u32 iv = civ[i];
      const u32 f = iv_file[iv];
      x = ((u64)nreal[iv] << 32) | (u64)(f >= flo && f < fhi);
    }
    v[q] = x;
    sum += x;
  }
  const u64 inc = warp_incl_scan(sum);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const u64 x = lane < LS_THREADS / 32 ? s_w[lane] : 0;
    const u64 xi = warp_incl_scan(x);
    if (lane < LS_THREADS / 32) s_w[lane] = xi - x;
    const u64 tot = __shfl_sync(MX_FULL, xi, 31);
    const u64 t = lookback_exclusive(status, tile, tot);
    if (lane == 0) s_excl = t;
  }
  __syncthreads();
  u64 run = s_excl + s_w[warp] + inc - sum;
#pragma unroll
  for (int q = 0; q < LS_ITEMS; ++q) {
    const long long i = b + q;
    if (i < n) {
      lcnt[i] = (u32)run;
      rcum[i] = run >> 32;
      if (v[q] & 1) lpos[(u32)run] = (u32)i;
    }
    run += v[q];
    if (i == n - 1) {
      lcnt[n] = (u32)run;
      rcum[n] = run >> 32;
    }
  }
}

int gen_local_lists(GenData* g, cudaStream_t s) {
  IndexData* ix = g->ix;
  const long long I = ix->n_intervals;
  if (!ix->sharded || I == 0) return MX_OK;
  MX_CUDA_TRY(g->lcnt.alloc(I + 1, s));
  MX_CUDA_TRY(g->lpos.alloc(I, s));
  MX_CUDA_TRY(g->rcum.alloc(I + 1, s));
  const int tiles = (int)((I + LS_TILE - 1) / LS_TILE);
  DevBuf<u64> st;
  DevBuf<u32> ctr;
  MX_CUDA_TRY(st.alloc(tiles, s));
  MX_CUDA_TRY(ctr.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(st.p, 0, sizeof(u64) * tiles, s));
  MX_CUDA_TRY(cudaMemsetAsync(ctr.p, 0, sizeof(u32), s));
  local_scan_kernel<<<tiles, LS_THREADS, 0, s>>>(g->civ.p, ix->iv_file.p, ix->iv_nreal.p, I, (u32)ix->file_lo,
                                                 (u32)ix->file_hi, st.p, ctr.p, g->lcnt.p, g->lpos.p, g->rcum.p);
  mx_count_launch();
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

// pieces of rank q's chunk c are sorted by (mixture key, file, start) and all
// of rank q's files precede rank q+1's: the global position of a piece is its
// chunk's base + pieces of other ranks with a smaller mixture key (or an
// equal one on a lower rank) + its index in its own chunk.
__global__ void merge_pieces_kernel(int W, long long C, long long cap, const long long* offs, const long long* out_off,
                                    const u32* mkey, const u32* file, const u32* start, const u32* end, u32* o_mkey,
                                    u32* o_file, u32* o_start, u32* o_end) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)W * cap) return;
  const int q = (int)(t / cap);
  const long long i = t % cap;
  const long long* oq = offs + (long long)q * (C + 1);
  if (i >= oq[C]) return;
  long long lo = 0, hi = C;  // chunk c: oq[c] <= i < oq[c+1]
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (oq[mid] <= i) lo = mid; else hi = mid - 1;
  }
  const long long c = lo;
  const u32 m = mkey[t];
  long long pos = out_off[c] + (i - oq[c]);
  for (int r = 0; r < W; ++r) {
    if (r == q) continue;
    const long long* orr = offs + (long long)r * (C + 1);
    const u32* mk = mkey + (long long)r * cap;
    long long a0 = orr[c], a1 = orr[c + 1];
    // r < q: pieces with key <= m come first; r > q: key < m
    while (a0 < a1) {
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

int chunks_merge(int W, long long C, long long cap, const long long* offs, const u32* mkey, const u32* file,
                 const u32* start, const u32* end, long long* out_off, u32* o_mkey, u32* o_file, u32* o_start,
                 u32* o_end, cudaStream_t s) {
  merge_offsets_kernel<<<(unsigned)((C + 256) / 256), 256, 0, s>>>(W, C, offs, out_off);
  mx_count_launch();
  const long long n = (long long)W * cap;
  if (n > 0) {
    merge_pieces_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W, C, cap, offs, out_off, mkey, file, start, end,
                                                                    o_mkey, o_file, o_start, o_end);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // namespace mx
