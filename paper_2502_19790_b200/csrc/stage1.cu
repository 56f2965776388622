// Stage 1 -- ChunkerIndex construction on sm_100a.
//
// Replaces MetadataCatalog.filter_intervals (catalog.py:549-605) +
// build_index (index.py:88-115) with three device passes:
//
//  1. ONE streaming pass over the code column(s) (scan_u16.cuh for a u16
//     row-tuple column, scan_tma.cuh for per-property int32 columns). Per
//     sample: code -> (packed key contribution | filter-fail flag) via a
//     shared-memory LUT, sum over properties = order-preserving packed key
//     (codec.py explains the layout), run boundaries from neighbour compares,
//     file boundaries from the tile's file-start list. Runs are compacted
//     tile-locally into per-tile slot regions as SoA interval records
//     (key, file, start, end) in (file, start) order; slot_fixup_kernel
//     closes runs that cross tiles and slot_compact_kernel densifies them.
//  2. an LSD radix sort of the records by packed key (8-bit digits, stable
//     warp-multisplit ranking) -> (key, file, start) order. The packed key is
//     order-preserving, so this IS MixtureKey.sort_key order (index.py:50-55
//     component_keys()).
//  3. two reduce-then-scan passes (scan.cuh): key/block boundary flags ->
//     dense key ranks and (key, file) block ids; interval lengths -> u64
//     cumulative samples.
//
// Algorithmic bytes: B1 = N*sum(w_p) + 16*I + 8*B_kf + 16*K.
#include <stdlib.h>
#include <string.h>

#include <memory>

#include "common.cuh"
#include "mixtera_internal.cuh"
#include "scan.cuh"

namespace mx {

// ---------------------------------------------------------------- pass 1
constexpr int S1_THREADS = 256;
constexpr int S1_SEGS = 4;                      // int4 segments per thread
constexpr int S1_WARP = 32 * 4 * S1_SEGS;       // 512 samples per warp
constexpr int S1_TILE = (S1_THREADS / 32) * S1_WARP;  // 4096 samples per tile
constexpr int S1_FILE_CAP = 512;                // file starts cached per tile
constexpr u32 FAIL = 0x80000000u;

struct S1Args {
  const int32_t* cols[MX_MAX_PROPS];  // int32 codes, or u16 codes when u16 (row-tuple layout)
  int u16;
  int vec_ok;            // every column aligned for 4-code vector loads
  int lut_off[MX_MAX_PROPS + 1];
  int n_props;
  const u32* lut;  // device copy of the concatenated LUT
  long long n;
  const long long* file_off;
  int n_files;
  u32 rank_mask;
  u32* rec_key;
  u32* rec_file;
  u32* rec_start;
  u32* rec_end;
  u64* status;
  u32* tile_ctr;
  u64* n_runs;
  DevError* err;
  const u32* lut_sum;    // LUT with the fail flag as a count at bit `fail_shift` (sum-only keying)
  u32 fail_limit;        // 1 << fail_shift: a sample passes iff its sum is below
  u32* tile_cnt;         // slot mode: runs started in each tile
  u32* tile_open;        // slot mode: tile's last run ends in a later tile
  long long* tile_head;  // slot mode: 0 none, -1 run passes through, >0 end+1 of the continuing run
  u32* defer_list;       // tiles scan_fast_kernel leaves to scan_list_kernel
  u32* defer_cnt;
};

template <bool SMEM_LUT>
__device__ __forceinline__ u32 lut_get(const u32* s_lut, const u32* g_lut, int idx) {
  return SMEM_LUT ? s_lut[idx] : __ldg(g_lut + idx);
}

// code of sample i in column p / four consecutive codes (i % 4 == 0)
__device__ __forceinline__ int code_at(const S1Args& a, int p, long long i) {
  return a.u16 ? (int)reinterpret_cast<const uint16_t*>(a.cols[p])[i] : a.cols[p][i];
}
__device__ __forceinline__ int4 codes4(const S1Args& a, int p, long long i) {
  return a.u16 ? ld_stream_u16x4(reinterpret_cast<const uint16_t*>(a.cols[p]) + i)
               : ld_stream_v4(reinterpret_cast<const int4*>(a.cols[p] + i));
}

// Status word of one sample: packed key, bit 31 set when it fails the filter
// or lies outside [0, n).
template <bool SMEM_LUT>
__device__ u32 sample_status(const S1Args& a, const u32* s_lut, long long i) {
  if (i < 0 || i >= a.n) return FAIL;
  u32 key = 0, any = 0;
  for (int p = 0; p < a.n_props; ++p) {
    int c = code_at(a, p, i);
    u32 e = lut_get<SMEM_LUT>(s_lut, a.lut, a.lut_off[p] + c + 1);
    key += e & ~FAIL;
    any |= e;
  }
  return (any & FAIL) | key;
}

__device__ __forceinline__ int upper_bound_ll(const long long* v, int n, long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (v[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}


}  // namespace mx

#include "scan_tma.cuh"
#include "scan_u16.cuh"

namespace mx {

// ---------------------------------------------------------------- radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;


// one CTA per digit: exclusive scan of its row across tiles, row total out
__global__ void __launch_bounds__(256)
radix_rowscan(u32* hist, int ntiles, u32* digit_tot) {
  __shared__ u32 s_w[8];
  __shared__ u32 s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u32* row = hist + (long long)blockIdx.x * ntiles;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int b = 0; b < ntiles; b += 256 * 4) {
    u32 v[4], s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i = b + tid * 4 + q;
      v[q] = i < ntiles ? row[i] : 0;
      s += v[q];
    }
    u32 inc = warp_incl_scan(s);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u32 x = lane < 8 ? s_w[lane] : 0;
      u32 xi = warp_incl_scan(x);
      if (lane < 8) s_w[lane] = xi - x;
    }
    __syncthreads();
    u32 run = s_carry + s_w[warp] + inc - s;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i = b + tid * 4 + q;
      if (i < ntiles) row[i] = run;
      run += v[q];
    }
    __syncthreads();
    if (tid == 255) s_carry = run;
    __syncthreads();
  }
  if (tid == 0) digit_tot[blockIdx.x] = s_carry;
}


// Staged variant: 4096-record tiles (RS2_ITEMS 16; 8 = 2048); records are first placed at their
// tile-local sorted position in shared memory (64 KB), then written out in
// that order, so consecutive threads write consecutive addresses of the same
// digit bucket (~16 records per digit per tile at cfg2) instead of 4-byte
// scattered stores into four arrays.
template <int RS2_ITEMS>
__global__ void __launch_bounds__(RS_THREADS)
radix_upsweep2(const u32* keys, long long n, int shift, u32* hist, int ntiles) {
  constexpr int RS2_TILE = RS_THREADS * RS2_ITEMS;
  __shared__ u32 h[256];
  const int tid = threadIdx.x;
  h[tid] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * RS2_TILE;
#pragma unroll 4
  for (int k = 0; k < RS2_ITEMS; ++k) {
    long long i = base + k * RS_THREADS + tid;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xff], 1u);
  }
  __syncthreads();
  hist[(long long)tid * ntiles + blockIdx.x] = h[tid];
}

template <int RS2_ITEMS>
__global__ void __launch_bounds__(RS_THREADS, 4)
radix_downsweep2(const u32* kin, const u32* p0in, const u32* p1in, const u32* p2in, u32* kout, u32* p0out,
                 u32* p1out, u32* p2out, long long n, int shift, const u32* hist, const u32* digit_tot,
                 int ntiles) {
  constexpr int RS2_TILE = RS_THREADS * RS2_ITEMS;
  extern __shared__ __align__(16) u32 s_stage[];  // [4][RS2_TILE]
  __shared__ u32 s_base[256], s_loc[256];
  __shared__ u32 s_wcnt[RS_WARPS][256];
  __shared__ u32 s_w[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {  // global digit bases: exclusive scan of digit totals + this tile's row prefix
    u32 x = digit_tot[tid];
    u32 inc = warp_incl_scan(x);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u32 y = lane < 8 ? s_w[lane] : 0;
      u32 yi = warp_incl_scan(y);
      if (lane < 8) s_w[lane] = yi - y;
    }
    __syncthreads();
    s_base[tid] = s_w[warp] + inc - x + hist[(long long)tid * ntiles + blockIdx.x];
  }
#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w) s_wcnt[w][tid] = 0;
  __syncthreads();
  // warp w owns the contiguous records [w * 512, (w + 1) * 512) of the tile
  const long long t0 = (long long)blockIdx.x * RS2_TILE;
  const long long base = t0 + warp * (32 * RS2_ITEMS);
  u32 dig[RS2_ITEMS], rank[RS2_ITEMS];
  // every record's four words are loaded up front (one round of global
  // latency per tile; the ranking below only needs the keys)
  u32 vk[RS2_ITEMS], va[RS2_ITEMS], vb[RS2_ITEMS], vc[RS2_ITEMS];
#pragma unroll
  for (int k = 0; k < RS2_ITEMS; ++k) {
    const long long i = base + k * 32 + lane;
    if (i < n) {
      vk[k] = kin[i];
      va[k] = p0in[i];
      vb[k] = p1in[i];
      vc[k] = p2in[i];
    }
  }
#pragma unroll
  for (int k = 0; k < RS2_ITEMS; ++k) {
    const long long i = base + k * 32 + lane;
    const bool ok = i < n;
    const u32 d = ok ? (vk[k] >> shift) & 0xff : 0x100u;
    const u32 peers = __match_any_sync(MX_FULL, d);
    const u32 before = __popc(peers & ((1u << lane) - 1));
    const u32 cur = s_wcnt[warp][d & 0xff];
    __syncwarp();
    rank[k] = cur + before;
    dig[k] = d;
    if (ok && before == 0) s_wcnt[warp][d] = cur + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  u32 tot;
  {  // per digit: exclusive scan over warps, then over digits (tile-local bucket starts)
    u32 run = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      u32 c = s_wcnt[w][tid];
      s_wcnt[w][tid] = run;
      run += c;
    }
    tot = run;
    u32 inc = warp_incl_scan(tot);
    __syncthreads();
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u32 y = lane < 8 ? s_w[lane] : 0;
      u32 yi = warp_incl_scan(y);
      if (lane < 8) s_w[lane] = yi - y;
    }
    __syncthreads();
    s_loc[tid] = s_w[warp] + inc - tot;
  }
  __syncthreads();
  u32* sk = s_stage;
  u32* sa = s_stage + RS2_TILE;
  u32* sb = s_stage + 2 * RS2_TILE;
  u32* sc = s_stage + 3 * RS2_TILE;
#pragma unroll
  for (int k = 0; k < RS2_ITEMS; ++k) {
    if (dig[k] < 0x100u) {
      const u32 d = dig[k];
      const u32 pos = s_loc[d] + s_wcnt[warp][d] + rank[k];
      sk[pos] = vk[k];
      sa[pos] = va[k];
      sb[pos] = vb[k];
      sc[pos] = vc[k];
    }
  }
  __syncthreads();
  const int cnt = (int)(n - t0 < RS2_TILE ? n - t0 : RS2_TILE);
  for (int i = tid; i < cnt; i += RS_THREADS) {
    const u32 key = sk[i];
    const u32 d = (key >> shift) & 0xff;
    const u32 dst = s_base[d] + (u32)i - s_loc[d];
    kout[dst] = key;
    p0out[dst] = sa[i];
    p1out[dst] = sb[i];
    p2out[dst] = sc[i];
  }
}

// ---------------------------------------------------------------- host side


template <int SEGS, int PC>
static void launch_direct(const S1Args& a, const TileMeta* m, long long ntiles, bool smem_lut, int lut_total,
                          cudaStream_t s, long long first = 0) {
  if (ntiles - first <= 0) return;
  const unsigned grid = (unsigned)(ntiles - first);
  if (smem_lut) {
    scan_direct_kernel<SEGS, PC, true><<<grid, S1_THREADS, sizeof(u32) * lut_total, s>>>(a, m, ntiles, first);
  } else {
    scan_direct_kernel<SEGS, 0, false><<<grid, S1_THREADS, 0, s>>>(a, m, ntiles, first);
  }
}

template <int PC, int SEGS>
static void launch_fast(const S1Args& a, const TileMeta* m, long long nfull, int lut_total, cudaStream_t s) {
  if (nfull <= 0) return;
  if constexpr (PC == 1 && SEGS == 2) {
    const bool g = lut_total > MX_STAGED_LUT_MAX;
    const size_t dyn = g ? 0 : sizeof(u32) * lut_total;
    if (g) scan_fast_kernel<PC, SEGS, true, 8><<<(unsigned)nfull, S1_THREADS, dyn, s>>>(a, m);
    else scan_fast_kernel<PC, SEGS, false, 8><<<(unsigned)nfull, S1_THREADS, dyn, s>>>(a, m);
    return;
  }
  if (lut_total > MX_STAGED_LUT_MAX)
    scan_fast_kernel<PC, SEGS, true><<<(unsigned)nfull, S1_THREADS, 0, s>>>(a, m);
  else
    scan_fast_kernel<PC, SEGS><<<(unsigned)nfull, S1_THREADS, sizeof(u32) * lut_total, s>>>(a, m);
}

// full tiles through scan_fast_kernel when it applies, the rest generically
template <int SEGS>
static void dispatch_direct(const S1Args& a, const TileMeta* m, long long ntiles, bool smem_lut, int lut_total,
                            cudaStream_t s, long long nfull_aligned) {
  const int pc = smem_lut && a.lut_sum ? a.n_props : 0;
  long long done = 0;
  if (nfull_aligned > 0 && pc >= 1 && pc <= 6) {
    switch (pc) {
      case 1: launch_fast<1, SEGS>(a, m, nfull_aligned, lut_total, s); break;
      case 2: launch_fast<2, SEGS>(a, m, nfull_aligned, lut_total, s); break;
      case 3: launch_fast<3, SEGS>(a, m, nfull_aligned, lut_total, s); break;
      case 4: launch_fast<4, SEGS>(a, m, nfull_aligned, lut_total, s); break;
      case 5: launch_fast<5, SEGS>(a, m, nfull_aligned, lut_total, s); break;
      default: launch_fast<6, SEGS>(a, m, nfull_aligned, lut_total, s); break;
    }
    done = nfull_aligned;
    // tiles the fast kernel deferred (more file starts than it handles)
    const long long grid = std::min<long long>(nfull_aligned, 148 * 4);
    scan_list_kernel<SEGS, true><<<(unsigned)grid, S1_THREADS, sizeof(u32) * lut_total, s>>>(a, m);
  }
  launch_direct<SEGS, 0>(a, m, ntiles, smem_lut, lut_total, s, done);
}

// exclusive offsets of the per-tile run counts (slots -> dense records)
struct TileOffF {
  const u32* cnt;
  u64* off;
  long long n;
  __device__ u64 value(long long i) const { return cnt[i]; }
  __device__ void apply(long long i, u64 ex, u64) const { off[i] = ex; }
  __device__ void total(u64 t) const { off[n] = t; }
};

int stage1_build(const mx_catalog_desc* d, cudaStream_t s, IndexData* out) {
  mx_host_mark("s1 enter");
  if (d->n_props < 1 || d->n_props > MX_MAX_PROPS)
    return mx_fail(MX_ERR_UNSUPPORTED, "n_props=%d outside [1, %d]", d->n_props, MX_MAX_PROPS);
  // scanned columns: one per property, or the row-tuple code column(s)
  const int NC = d->n_columns > 0 ? d->n_columns : d->n_props;
  if (NC > MX_MAX_PROPS) return mx_fail(MX_ERR_UNSUPPORTED, "n_columns=%d > %d", NC, MX_MAX_PROPS);
  if (d->key_bits > 31)
    return mx_fail(MX_ERR_UNSUPPORTED, "packed key needs %u bits (> 31)", d->key_bits);
  if (d->n_files < 1) return mx_fail(MX_ERR_QUERY, "catalog is empty");
  IndexData& ix = *out;
  ix.n_samples_total = d->n_samples;
  ix.n_files = d->n_files;
  ix.key_bits = d->key_bits;
  const long long n = d->n_samples;
  S1Args a{};
  a.n_props = NC;
  if (d->column_bytes != 0 && d->column_bytes != 2 && d->column_bytes != 4)
    return mx_fail(MX_ERR_UNSUPPORTED, "column_bytes=%d (2 or 4)", d->column_bytes);
  a.u16 = d->column_bytes == 2;
  for (int p = 0; p < NC; ++p) a.cols[p] = d->columns[p];
  for (int p = 0; p <= NC; ++p) a.lut_off[p] = d->lut_offsets[p];
  const int lut_total = d->lut_offsets[NC];
  // sum-keying LUT: fail flag as a count above the key bits (needs key_bits +
  // bitlen(P) <= 31), see scan_direct_kernel
  int pbits = 0;
  while ((1 << pbits) <= NC) ++pbits;
  const bool sum_ok = d->key_bits + pbits <= 31;
  std::vector<u32> ls;
  if (sum_ok) {
    ls.resize(lut_total);
    for (int i = 0; i < lut_total; ++i)
      ls[i] = (d->lut[i] & ~FAIL) + ((d->lut[i] >> 31) << d->key_bits);
  }
  // key-string pieces (device BLAKE2b of the canonical key strings)
  int n_pieces = d->n_columns > 0 ? d->n_key_pieces : 0;
  for (int p = 0; d->n_columns <= 0 && p < d->n_props && p < MX_MAX_PROPS; ++p) {
    const int card = (d->lut_offsets[p + 1] - d->lut_offsets[p]) - 1;
    n_pieces = std::max(n_pieces, d->key_string_base[p] + card);
  }
  const long long str_nbytes = d->key_string_offsets[n_pieces];
  // the small host arrays of the build in two device blocks: the LUTs the
  // scan reads go up first; key strings and file tables (not read until the
  // index finalize) are uploaded after the scan launch, while it runs
  Uploads up, up2;
  const size_t o_lut = up.add(d->lut, sizeof(u32) * lut_total);
  const size_t o_lsum = up.add(ls.data(), sizeof(u32) * ls.size());
  const size_t o_soff = up2.add(d->key_string_offsets, sizeof(long long) * (n_pieces + 1));
  const size_t o_sbytes = up2.add(d->key_strings, str_nbytes > 0 ? (size_t)str_nbytes : 0);
  const size_t o_fds = up2.add(d->file_ds, sizeof(int32_t) * d->n_files);
  const size_t o_fid = up2.add(d->file_ids, sizeof(long long) * d->n_files);
  mx_host_mark("s1 host tables");
  MX_CUDA_TRY(ix.consts.alloc((long long)up.total + 16, s));
  MX_CUDA_TRY(up.run(ix.consts.p, s));
  mx_host_mark("s1 upload");
  a.lut = reinterpret_cast<const u32*>(ix.consts.p + o_lut);
  if (sum_ok) {
    a.lut_sum = reinterpret_cast<const u32*>(ix.consts.p + o_lsum);
    a.fail_limit = 1u << d->key_bits;
  }
  a.n = n;
  a.file_off = reinterpret_cast<const long long*>(d->file_offsets);
  a.n_files = d->n_files;
  a.rank_mask = d->rank_mask;

  // ---- stage-1 pass variant (MX_SCAN = direct (default) | pipe | v1):
  //  direct: one CTA per 4096-sample tile, slot output (scan_direct_kernel)
  //  pipe:   persistent CTAs + TMA ring, slot output (scan_pipe_kernel)
  //  v1:     one CTA per tile, decoupled look-back output (scan_runs_kernel)
  const bool smem_lut = lut_total <= MX_SMEM_LUT_MAX;
  int dev = 0;
  MX_CUDA_TRY(cudaGetDevice(&dev));
  static thread_local int sm_dev = -1, sm_count = 148;
  if (sm_dev != dev) {
    MX_CUDA_TRY(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
    sm_dev = dev;
  }
  const int n_sm = sm_count;
  // Two stage-1 passes, both writing per-tile slot regions (tile-local
  // compaction, no inter-tile dependency) fixed up by slot_fixup_kernel:
  //  * one u16 row-tuple column, 16-byte aligned: scan_u16_kernel
  //    (scan_u16.cuh), change-driven, warp segments of 1024 samples;
  //  * otherwise (per-property int32 columns, wide tuple codes):
  //    scan_fast_kernel over full 2048-sample tiles + scan_list_kernel for
  //    tiles with many file starts + scan_direct_kernel for the rest.
  const bool u16_path = a.u16 && NC == 1 && a.lut_sum != nullptr &&
                        (reinterpret_cast<uintptr_t>(d->columns[0]) % 16) == 0;
  const int tile_len = u16_path ? SEG_LEN : 2048;
  const long long ntiles = (n + tile_len - 1) / tile_len;
  bool aligned = true;
  for (int p = 0; p < NC; ++p) aligned &= (reinterpret_cast<uintptr_t>(d->columns[p]) % (a.u16 ? 8 : 16)) == 0;
  const long long nstaged = aligned ? n / tile_len : 0;
  a.vec_ok = aligned;
  DevBuf<TileMeta> tmeta;
  DevBuf<int> seg_fa;
  DevBuf<u32> rk, rf, rs, re;
  DevBuf<u64> scratch64;
  DevBuf<DevError> err;
  // worst case every sample is its own run; slots address whole tiles
  const long long cap = std::max<long long>(1, ntiles * tile_len);
  DevBuf<u32> t_cnt, t_open, defer;
  DevBuf<long long> t_head;
  if (ntiles > 0) {
    MX_CUDA_TRY(ws_borrow(t_cnt, s, WS_TCNT, ntiles));
    MX_CUDA_TRY(ws_borrow(t_open, s, WS_TOPEN, ntiles));
    MX_CUDA_TRY(ws_borrow(t_head, s, WS_THEAD, ntiles));
    MX_CUDA_TRY(ws_borrow(defer, s, WS_DEFER, ntiles + 1));
    MX_CUDA_TRY(cudaMemsetAsync(defer.p + ntiles, 0, sizeof(u32), s));
    a.tile_cnt = t_cnt.p;
    a.tile_open = t_open.p;
    a.tile_head = t_head.p;
    a.defer_list = defer.p;
    a.defer_cnt = defer.p + ntiles;
  }
  mx_host_mark("s1 tile allocs");
  MX_CUDA_TRY(ws_borrow(rk, s, WS_RK, cap));
  MX_CUDA_TRY(ws_borrow(rf, s, WS_RF, cap));
  MX_CUDA_TRY(ws_borrow(rs, s, WS_RS, cap));
  MX_CUDA_TRY(ws_borrow(re, s, WS_RE, cap));
  MX_CUDA_TRY(ws_borrow(scratch64, s, WS_SCR64, 4));
  MX_CUDA_TRY(ws_borrow(err, s, WS_ERR, 1));
  MX_CUDA_TRY(cudaMemsetAsync(scratch64.p, 0, sizeof(u64) * 4, s));
  MX_CUDA_TRY(cudaMemsetAsync(err.p, 0xff, sizeof(u64), s));
  MX_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<char*>(err.p) + 8, 0, 8, s));
  a.rec_key = rk.p; a.rec_file = rf.p; a.rec_start = rs.p; a.rec_end = re.p;
  a.n_runs = scratch64.p; a.err = err.p;
  mx_host_mark("s1 slot allocs");
  if (ntiles > 0 && u16_path) {
    MX_CUDA_TRY(ws_borrow(seg_fa, s, WS_SEGFA, ntiles + 1));
    seg_file_kernel<<<(unsigned)((ntiles + 1 + 255) / 256), 256, 0, s>>>(a.file_off, a.n_files, n, ntiles, seg_fa.p);
    mx_count_launch();
    {
      MxPhase ph("scan_runs", s);
      const int entries = lut_total - 1;
      // LUT placement: shared u16 when packed keys fit 15 bits (6 CTAs/SM),
      // shared u32, or global
      const int mode = entries > U16_SMEM_LUT_MAX ? 0 : (d->key_bits <= 15 ? 2 : 1);
      const size_t dyn = sizeof(U16Warp) * U16_WARPS + (mode == 2 ? 2 : mode == 1 ? 4 : 0) * (size_t)entries;
      // attribute + occupancy per (LUT placement, shared bytes), queried once
      static thread_local size_t q_dyn[3] = {0, 0, 0};
      static thread_local int q_per_sm[3] = {1, 1, 1};
      int& per_sm = q_per_sm[mode];
      if (q_dyn[mode] != dyn) {
        if (mode == 2) {
          MX_CUDA_TRY(cudaFuncSetAttribute(scan_u16_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
          MX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_u16_kernel<2>, U16_WARPS * 32, dyn));
        } else if (mode == 1) {
          MX_CUDA_TRY(cudaFuncSetAttribute(scan_u16_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
          MX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_u16_kernel<1>, U16_WARPS * 32, dyn));
        } else {
          MX_CUDA_TRY(cudaFuncSetAttribute(scan_u16_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
          MX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_u16_kernel<0>, U16_WARPS * 32, dyn));
        }
        q_dyn[mode] = dyn;
      }
      const long long want = (ntiles + U16_WARPS - 1) / U16_WARPS;
      const unsigned grid = (unsigned)std::min<long long>(want, (long long)n_sm * std::max(1, per_sm));
      if (mode == 2) scan_u16_kernel<2><<<grid, U16_WARPS * 32, dyn, s>>>(a, seg_fa.p, ntiles);
      else if (mode == 1) scan_u16_kernel<1><<<grid, U16_WARPS * 32, dyn, s>>>(a, seg_fa.p, ntiles);
      else scan_u16_kernel<0><<<grid, U16_WARPS * 32, dyn, s>>>(a, seg_fa.p, ntiles);
      mx_count_launch();
      MX_CUDA_TRY(cudaGetLastError());
    }
  } else if (ntiles > 0) {
    MX_CUDA_TRY(tmeta.alloc(ntiles, s));
    tile_meta_kernel<<<(unsigned)((ntiles + 255) / 256), 256, 0, s>>>(a, tile_len, ntiles, tmeta.p);
    mx_count_launch();
    MxPhase ph("scan_runs", s);
    dispatch_direct<2>(a, tmeta.p, ntiles, smem_lut, lut_total, s, nstaged);
    mx_count_launch();
  }
  if (ntiles > 0) {
    slot_fixup_kernel<<<(unsigned)((ntiles + 255) / 256), 256, 0, s>>>(ntiles, tile_len, t_cnt.p, t_open.p, t_head.p,
                                                                     rf.p, a.file_off, re.p, scratch64.p);
    mx_count_launch();
    MX_CUDA_TRY(cudaGetLastError());
  }
  mx_host_mark("s1 scan launched");
  // key strings and file tables (ds and ids are needed for exports and cursors)
  MX_CUDA_TRY(ix.consts2.alloc((long long)up2.total + 16, s));
  MX_CUDA_TRY(up2.run(ix.consts2.p, s));
  ix.str_off.borrow(ix.consts2.p + o_soff, n_pieces + 1);
  ix.str_bytes.borrow(ix.consts2.p + o_sbytes, str_nbytes > 0 ? str_nbytes : 1);
  ix.file_ds.borrow(ix.consts2.p + o_fds, d->n_files);
  ix.file_ids.borrow(ix.consts2.p + o_fid, d->n_files);
  ix.h_file_ds.assign(d->file_ds, d->file_ds + d->n_files);
  ix.h_file_ids.assign(d->file_ids, d->file_ids + d->n_files);
  mx_host_mark("s1 tables uploaded");
  u64 h_runs = 0;
  DevError h_err;
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(&h_runs, scratch64.p, sizeof(u64)));
    MX_CUDA_TRY(rb.add(&h_err, err.p, sizeof(DevError)));
    MX_CUDA_TRY(rb.sync());
  }
  mx_host_mark("s1 scan synced");
  if (h_err.null_key_sample != ~0ull) {
    const long long g = (long long)h_err.null_key_sample;
    std::vector<long long> off(d->n_files + 1);
    MX_CUDA_TRY(cudaMemcpy(off.data(), d->file_offsets, sizeof(long long) * off.size(), cudaMemcpyDeviceToHost));
    int f = (int)(std::upper_bound(off.begin(), off.end(), g) - off.begin()) - 1;
    return mx_fail(MX_ERR_QUERY,
                   "sample %lld of file %lld has no non-null properties; it cannot be keyed into a mixture",
                   g - off[f], (long long)d->file_ids[f]);
  }
  const long long I = (long long)h_runs;
  ix.n_intervals = I;
  if (I == 0) {
    ix.n_keys = 0;
    ix.n_blocks = 0;
    return MX_OK;
  }
  // ---- per-tile slots -> dense records (order preserved), then LSD radix
  // sort by packed key (8-bit digits, stable, 2048-record tiles)
  const int passes = (d->key_bits + 7) / 8;
  constexpr int RIT = 8;
  const int rtile2 = RS_THREADS * RIT;
  const int rtiles2 = (int)((I + rtile2 - 1) / rtile2);
  const size_t rsmem = 4 * (size_t)rtile2 * sizeof(u32);
  std::unique_ptr<MxPhase> ph_sort(new MxPhase("radix_sort", s));
  DevBuf<u64> toff;  // tile offsets first: the device starts while the host allocates
  MX_CUDA_TRY(ws_borrow(toff, s, WS_TOFF, ntiles + 1));
  if (int rc = gs_run(ntiles, TileOffF{t_cnt.p, toff.p, ntiles}, s)) return rc;
  DevBuf<u32> k2, f2, s2, e2, hist, dtot;
  MX_CUDA_TRY(k2.alloc(I, s));
  MX_CUDA_TRY(f2.alloc(I, s));
  MX_CUDA_TRY(s2.alloc(I, s));
  MX_CUDA_TRY(e2.alloc(I, s));
  MX_CUDA_TRY(ws_borrow(hist, s, WS_HIST, (long long)256 * rtiles2));
  MX_CUDA_TRY(ws_borrow(dtot, s, WS_DTOT, 256));
  u32 *ka = rk.p, *fa_ = rf.p, *sa = rs.p, *ea = re.p;
  u32 *kb = k2.p, *fb = f2.p, *sb = s2.p, *eb = e2.p;
  {
    slot_compact_kernel<<<(unsigned)std::min<long long>(ntiles, (long long)n_sm * 16), 256, 0, s>>>(
        ntiles, tile_len, t_cnt.p, toff.p, rk.p, rf.p, rs.p, re.p, k2.p, f2.p, s2.p, e2.p);
    mx_count_launch();
    std::swap(ka, kb); std::swap(fa_, fb); std::swap(sa, sb); std::swap(ea, eb);
  }
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 8 * pass;
    radix_upsweep2<RIT><<<rtiles2, RS_THREADS, 0, s>>>(ka, I, shift, hist.p, rtiles2);
    mx_count_launch();
    radix_rowscan<<<256, 256, 0, s>>>(hist.p, rtiles2, dtot.p);
    mx_count_launch();
    radix_downsweep2<RIT><<<rtiles2, RS_THREADS, rsmem, s>>>(ka, fa_, sa, ea, kb, fb, sb, eb, I, shift, hist.p,
                                                            dtot.p, rtiles2);
    mx_count_launch();
    MX_CUDA_TRY(cudaGetLastError());
    std::swap(ka, kb); std::swap(fa_, fb); std::swap(sa, sb); std::swap(ea, eb);
  }
  ph_sort.reset();
  mx_host_mark("s1 sort launched");
  // sorted arrays now in (ka, fa_, sa, ea); keep them
  if (ka == rk.p) {  // odd number of passes: the result is in the workspace; copy it out
    for (auto pr : {std::make_pair(&k2, rk.p), std::make_pair(&f2, rf.p), std::make_pair(&s2, rs.p),
                    std::make_pair(&e2, re.p)})
      MX_CUDA_TRY(cudaMemcpyAsync(pr.first->p, pr.second, sizeof(u32) * I, cudaMemcpyDeviceToDevice, s));
    ix.iv_key.take(k2); ix.iv_file.take(f2); ix.iv_start.take(s2); ix.iv_end.take(e2);
  } else {
    ix.iv_key.take(k2); ix.iv_file.take(f2); ix.iv_start.take(s2); ix.iv_end.take(e2);
  }
  return index_finalize(&ix, I, s, /*defer=*/true);
}

// key / block boundaries: value = (key change << 32) | (key or file change);
// the inclusive count gives the dense key rank and (key, file) block id
struct BoundsF {
  const u32* key;
  const u32* file;
  u32 *blk_first, *blk_file, *blk_key, *key_blk_first, *key_packed;
  u64* totals;
  __device__ u64 value(long long i) const {
    const bool kc = i == 0 || key[i] != key[i - 1];
    const bool bc = kc || file[i] != file[i - 1];
    return ((u64)kc << 32) | (u64)bc;
  }
  __device__ void apply(long long i, u64 ex, u64 v) const {
    if (!(v & 1)) return;
    const u64 run = ex + v;
    const u32 k = (u32)(run >> 32) - 1, blk = (u32)run - 1;
    blk_first[blk] = (u32)i;
    blk_file[blk] = file[i];
    blk_key[blk] = k;
    if (v >> 32) {
      key_blk_first[k] = blk;
      key_packed[k] = key[i];
    }
  }
  __device__ void total(u64 t) const { *totals = t; }
};

// cum[i + 1] = samples of intervals [0, i]; an empty or inverted interval
// flags IndexBuildError
struct CumF {
  const u32* start;
  const u32* end;
  u64* cum;
  DevError* err;
  __device__ u64 value(long long i) const {
    const u32 s = start[i], e = end[i];
    return e > s ? e - s : 0;
  }
  __device__ void apply(long long i, u64 ex, u64 v) const {
    if (i == 0) cum[0] = 0;
    cum[i + 1] = ex + v;
    if (end[i] <= start[i]) atomicOr(&err->overlap, 1u);
  }
  __device__ void total(u64) const {}
};

// blk_first[B] = I, key_blk_first[K] = B from the device totals
__global__ void sentinel_kernel(const u64* totals, u32 I, u32* blk_first, u32* key_blk_first) {
  if (threadIdx.x != 0) return;
  const u64 t = *totals;
  const u32 K = (u32)(t >> 32), B = (u32)(t & 0xffffffffull);
  blk_first[B] = I;
  key_blk_first[K] = B;
}

// max over keys of (blocks of the key); totals = (n_keys << 32) | n_blocks
__global__ void key_maxblk_kernel(const u32* key_blk_first, const u64* totals, u32* out) {
  const u64 t = *totals;
  const long long K = (long long)(t >> 32), B = (long long)(t & 0xffffffffull);
  u32 m = 0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < K; k += (long long)gridDim.x * blockDim.x) {
    const u32 end = k + 1 < K ? key_blk_first[k + 1] : (u32)B;
    m = max(m, end - key_blk_first[k]);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(MX_FULL, m, d));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Block / key structure and cumulative lengths of the interval table
// (iv_key, iv_file, iv_start, iv_end) sorted by (packed key, file, start):
// blk_*, key_*, iv_cum, n_keys, n_blocks. IndexBuildError on an empty or
// overlapping interval (index.py:32-47).
int index_finalize(IndexData* ixp, long long I, cudaStream_t s, bool defer) {
  IndexData& ix = *ixp;
  ix.n_intervals = I;
  if (I == 0) {
    ix.n_keys = ix.n_blocks = 0;
    return MX_OK;
  }
  DevBuf<u64> scratch64;
  DevBuf<u32> ctr;
  DevBuf<DevError> err;
  MX_CUDA_TRY(scratch64.alloc(2, s));
  MX_CUDA_TRY(ctr.alloc(2, s));
  MX_CUDA_TRY(err.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(scratch64.p, 0, sizeof(u64) * 2, s));
  MX_CUDA_TRY(cudaMemsetAsync(err.p, 0xff, sizeof(u64), s));
  MX_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<char*>(err.p) + 8, 0, 8, s));
  DevError h_err;
  // ---- boundaries and cumulative lengths
  MX_CUDA_TRY(ix.blk_first.alloc(I + 1, s));
  MX_CUDA_TRY(ix.blk_file.alloc(I, s));
  MX_CUDA_TRY(ix.blk_key.alloc(I, s));
  MX_CUDA_TRY(ix.key_blk_first.alloc(I + 1, s));
  MX_CUDA_TRY(ix.key_packed.alloc(I, s));
  MX_CUDA_TRY(ix.iv_cum.alloc(I + 1, s));
  std::unique_ptr<MxPhase> ph_scan(new MxPhase("index_scans", s));
  if (int rc = gs_run(I, BoundsF{ix.iv_key.p, ix.iv_file.p, ix.blk_first.p, ix.blk_file.p, ix.blk_key.p,
                                 ix.key_blk_first.p, ix.key_packed.p, scratch64.p}, s))
    return rc;
  if (int rc = gs_run(I, CumF{ix.iv_start.p, ix.iv_end.p, ix.iv_cum.p, err.p}, s)) return rc;
  ph_scan.reset();
  // largest key (in blocks): sizes the cursor shuffle's shared-memory lists
  DevBuf<u32> maxblk;
  MX_CUDA_TRY(maxblk.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(maxblk.p, 0, sizeof(u32), s));
  key_maxblk_kernel<<<64, 256, 0, s>>>(ix.key_blk_first.p, scratch64.p, maxblk.p);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  if (defer) {
    // no host wait: sizes land in a pinned slot, the sentinels are written
    // from the device totals, ix_resolve() completes the sizes on first use
    IndexData::Pending* slot = pend_slot_take();
    int dev = 0;
    cudaEvent_t ev = nullptr;
    if (slot && cudaGetDevice(&dev) == cudaSuccess && aux_event_take(dev, &ev) == cudaSuccess) {
      MX_CUDA_TRY(cudaMemcpyAsync(&slot->maxblk, maxblk.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
      MX_CUDA_TRY(cudaMemcpyAsync(&slot->totals, scratch64.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
      MX_CUDA_TRY(cudaMemcpyAsync(&slot->samples, ix.iv_cum.p + I, sizeof(u64), cudaMemcpyDeviceToHost, s));
      MX_CUDA_TRY(cudaMemcpyAsync(&slot->err, err.p, sizeof(DevError), cudaMemcpyDeviceToHost, s));
      MX_CUDA_TRY(cudaEventRecord(ev, s));
      sentinel_kernel<<<1, 32, 0, s>>>(scratch64.p, (u32)I, ix.blk_first.p, ix.key_blk_first.p);
      mx_count_launch();
      MX_CUDA_TRY(cudaGetLastError());
      ix.pend = slot;
      ix.pend_ev = ev;
      ix.pend_dev = dev;
      return MX_OK;
    }
    if (slot) pend_slot_give(slot);
  }
  u64 tot = 0, samples = 0;
  u32 h_maxblk = 0;
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(&h_maxblk, maxblk.p, sizeof(u32)));
    MX_CUDA_TRY(rb.add(&tot, scratch64.p, sizeof(u64)));
    MX_CUDA_TRY(rb.add(&samples, ix.iv_cum.p + I, sizeof(u64)));
    MX_CUDA_TRY(rb.add(&h_err, err.p, sizeof(DevError)));
    MX_CUDA_TRY(rb.sync());
  }
  if (h_err.overlap) return mx_fail(MX_ERR_INDEX, "empty or overlapping interval in index build");
  ix.n_keys = (long long)(tot >> 32);
  ix.n_blocks = (long long)(tot & 0xffffffffull);
  ix.indexed_samples = (long long)samples;
  ix.max_key_blocks = (long long)h_maxblk;
  // sentinels (stream-ordered; no host wait)
  const u32 sI = (u32)I, sB = (u32)ix.n_blocks;
  MX_CUDA_TRY(mx_h2d(ix.blk_first.p + ix.n_blocks, &sI, sizeof(u32), s));
  MX_CUDA_TRY(mx_h2d(ix.key_blk_first.p + ix.n_keys, &sB, sizeof(u32), s));
  return MX_OK;
}


// ---------------------------------------------------------------- rows index
// build_index(rows) (index.py:88-115) from explicit interval rows: LSD sort
// by (key, file, start) with the staged radix passes (start digits, then
// file, then key; each pass is stable), then one scan that rejects empty
// rows and overlaps inside a (key, file) and merges adjacent rows
// (_merge_intervals, index.py:32-47), then index_finalize.

static int radix_sort_by(u32*& k, u32*& p0, u32*& p1, u32*& p2, u32*& k2, u32*& q0, u32*& q1, u32*& q2,
                         long long n, int bits, u32* hist, u32* dtot, cudaStream_t s) {
  constexpr int IT = 8;
  const int tile = RS_THREADS * IT;
  const int tiles = (int)((n + tile - 1) / tile);
  const size_t smem = 4 * (size_t)tile * sizeof(u32);
  for (int shift = 0; shift < bits; shift += 8) {
    radix_upsweep2<IT><<<tiles, RS_THREADS, 0, s>>>(k, n, shift, hist, tiles);
    mx_count_launch();
    radix_rowscan<<<256, 256, 0, s>>>(hist, tiles, dtot);
    mx_count_launch();
    radix_downsweep2<IT><<<tiles, RS_THREADS, smem, s>>>(k, p0, p1, p2, k2, q0, q1, q2, n, shift, hist, dtot, tiles);
    mx_count_launch();
    MX_CUDA_TRY(cudaGetLastError());
    std::swap(k, k2); std::swap(p0, q0); std::swap(p1, q1); std::swap(p2, q2);
  }
  return MX_OK;
}

static int bits_of(unsigned long long v) {
  int b = 0;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// rows sorted by (key, file, start): head = not adjacent to the previous row
// of the same (key, file); empty rows / overlaps flag err (first row index)
struct RowMergeF {
  const u32 *key, *file, *start, *end;
  long long n;
  u32 *okey, *ofile, *ostart, *oend;
  u64* count;
  unsigned long long* bad;  // [0] = first empty row, [1] = first overlapping row
  __device__ bool same(long long i) const { return i > 0 && key[i] == key[i - 1] && file[i] == file[i - 1]; }
  __device__ u64 value(long long i) const { return !(same(i) && start[i] == end[i - 1]); }
  __device__ void apply(long long i, u64 ex, u64 v) const {
    if (end[i] <= start[i]) atomicMin(&bad[0], (unsigned long long)i);
    if (same(i) && start[i] < end[i - 1]) atomicMin(&bad[1], (unsigned long long)i);
    const long long pos = (long long)(ex + v) - 1;
    if (v) {
      okey[pos] = key[i];
      ofile[pos] = file[i];
      ostart[pos] = start[i];
    }
    if (i + 1 == n || value(i + 1)) oend[pos] = end[i];
  }
  __device__ void total(u64 t) const { *count = t; }
};

int rows_build(const mx_rows_desc* d, cudaStream_t s, IndexData* out) {
  IndexData& ix = *out;
  const long long n = d->n_rows;
  ix.n_files = d->n_files;
  ix.key_bits = d->key_bits;
  MX_CUDA_TRY(ix.file_ds.alloc(std::max(1, d->n_files), s));
  MX_CUDA_TRY(ix.file_ids.alloc(std::max(1, d->n_files), s));
  if (d->n_files > 0) {
    MX_CUDA_TRY(mx_h2d(ix.file_ds.p, d->file_ds, sizeof(int32_t) * d->n_files, s));
    MX_CUDA_TRY(mx_h2d(ix.file_ids.p, d->file_ids, sizeof(long long) * d->n_files, s));
  }
  ix.h_file_ds.assign(d->file_ds, d->file_ds + d->n_files);
  ix.h_file_ids.assign(d->file_ids, d->file_ids + d->n_files);
  if (n == 0) {
    ix.n_intervals = ix.n_keys = ix.n_blocks = 0;
    return MX_OK;
  }
  DevBuf<u32> a[4], b[4], hist, dtot;
  const u32* src[4] = {d->key, d->file, d->start, d->end};
  for (int j = 0; j < 4; ++j) {
    MX_CUDA_TRY(a[j].alloc(n, s));
    MX_CUDA_TRY(b[j].alloc(n, s));
    MX_CUDA_TRY(mx_h2d(a[j].p, src[j], sizeof(u32) * n, s));
  }
  u32 max_start = 0;
  for (long long i = 0; i < n; ++i) max_start = std::max(max_start, d->start[i]);
  const int tiles = (int)((n + RS_THREADS * 8 - 1) / (RS_THREADS * 8));
  MX_CUDA_TRY(hist.alloc((long long)256 * tiles, s));
  MX_CUDA_TRY(dtot.alloc(256, s));
  MX_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(4 * RS_THREADS * 8 * sizeof(u32))));
  u32 *k = a[0].p, *f = a[1].p, *st = a[2].p, *en = a[3].p;
  u32 *k2 = b[0].p, *f2 = b[1].p, *st2 = b[2].p, *en2 = b[3].p;
  // least significant field first: start, then file, then key
  if (int rc = radix_sort_by(st, k, f, en, st2, k2, f2, en2, n, bits_of(max_start), hist.p, dtot.p, s)) return rc;
  if (int rc = radix_sort_by(f, k, st, en, f2, k2, st2, en2, n, bits_of((u32)std::max(0, d->n_files - 1)), hist.p,
                             dtot.p, s))
    return rc;
  if (int rc = radix_sort_by(k, f, st, en, k2, f2, st2, en2, n, (int)d->key_bits, hist.p, dtot.p, s)) return rc;
  MX_CUDA_TRY(ix.iv_key.alloc(n, s));
  MX_CUDA_TRY(ix.iv_file.alloc(n, s));
  MX_CUDA_TRY(ix.iv_start.alloc(n, s));
  MX_CUDA_TRY(ix.iv_end.alloc(n, s));
  DevBuf<u64> tot;
  DevBuf<unsigned long long> bad;
  MX_CUDA_TRY(tot.alloc(1, s));
  MX_CUDA_TRY(bad.alloc(2, s));
  MX_CUDA_TRY(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long) * 2, s));
  if (int rc = gs_run(n, RowMergeF{k, f, st, en, n, ix.iv_key.p, ix.iv_file.p, ix.iv_start.p, ix.iv_end.p, tot.p,
                                   bad.p},
                      s))
    return rc;
  u64 h_tot = 0;
  unsigned long long h_bad[2];
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(&h_tot, tot.p, sizeof(u64)));
    MX_CUDA_TRY(rb.add(h_bad, bad.p, sizeof(h_bad)));
    MX_CUDA_TRY(rb.sync());
  }
  for (int which = 0; which < 2; ++which) {
    if (h_bad[which] == ~0ull) continue;
    u32 row[4], prev_end = 0;
    const long long i = (long long)h_bad[which];
    const u32* srt[4] = {k, f, st, en};
    for (int j = 0; j < 4; ++j) MX_CUDA_TRY(cudaMemcpy(&row[j], srt[j] + i, sizeof(u32), cudaMemcpyDeviceToHost));
    const long long fid = (long long)d->file_ids[row[1]];
    if (which == 0)
      return mx_fail(MX_ERR_INDEX, "file %lld: empty interval [%u,%u)", fid, row[2], row[3]);
    u32 prev_start = 0;
    MX_CUDA_TRY(cudaMemcpy(&prev_start, st + i - 1, sizeof(u32), cudaMemcpyDeviceToHost));
    MX_CUDA_TRY(cudaMemcpy(&prev_end, en + i - 1, sizeof(u32), cudaMemcpyDeviceToHost));
    return mx_fail(MX_ERR_INDEX, "file %lld: overlapping intervals [%u,%u) and [%u,%u)", fid, prev_start, prev_end,
                   row[2], row[3]);
  }
  const long long I = (long long)h_tot;
  ix.n_samples_total = 0;
  int rc = index_finalize(&ix, I, s);
  ix.n_samples_total = ix.indexed_samples;
  return rc;
}


// ---------------------------------------------------------------- owner index
// Key-partitioned multi-GPU layout: the index an OWNER rank builds over the
// (key, file) blocks of the keys it owns, gathered from every rank (device
// rows uint32[n][4] = packed key, global file index, samples, intervals).
// One pseudo-interval [0, samples) per block, sorted by (packed key, file),
// the codec (key strings, fields) copied from this rank's local index: its
// generator's RangeCursor shuffles are the reference's over the key's files
// of the WHOLE catalog (index.py:134-144), and its cursor prefix sums give
// every block's offset in its key's cursor stream.
__global__ void owner_rows_kernel(long long n, const uint4* rows, int dense, u32* key, u32* file, u32* start,
                                  u32* end) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 r = rows[i];
  key[i] = dense ? r.w : r.x;
  file[i] = r.y;
  start[i] = (u32)i;  // row id through the sort (owner_row); the pseudo-interval starts at 0
  end[i] = r.z;
}

__global__ void owner_keys_kernel(long long n, const uint4* rows, const u32* row, u32* key) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) key[i] = rows[row[i]].x;
}

int owner_index_build(const IndexData* src, const u32* rows, long long n, int n_files, const int32_t* file_ds,
                      const int64_t* file_ids, int dense_bits, cudaStream_t s, IndexData* out) {
  IndexData& ix = *out;
  ix.stream = s;
  ix.n_files = n_files;
  ix.key_bits = src->key_bits;
  ix.n_props = src->n_props;
  for (int p = 0; p < MX_MAX_PROPS; ++p) {
    ix.field_shift[p] = src->field_shift[p];
    ix.field_width[p] = src->field_width[p];
    ix.str_base[p] = src->str_base[p];
  }
  MX_CUDA_TRY(ix.str_off.alloc(src->str_off.n, s));
  MX_CUDA_TRY(ix.str_bytes.alloc(src->str_bytes.n, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.str_off.p, src->str_off.p, sizeof(long long) * src->str_off.n,
                              cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.str_bytes.p, src->str_bytes.p, src->str_bytes.n, cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(ix.file_ds.alloc(std::max(1, n_files), s));
  MX_CUDA_TRY(ix.file_ids.alloc(std::max(1, n_files), s));
  if (n_files > 0) {
    MX_CUDA_TRY(mx_h2d(ix.file_ds.p, file_ds, sizeof(int32_t) * n_files, s));
    MX_CUDA_TRY(mx_h2d(ix.file_ids.p, file_ids, sizeof(long long) * n_files, s));
  }
  ix.h_file_ds.assign(file_ds, file_ds + n_files);
  ix.h_file_ids.assign(file_ids, file_ids + n_files);
  if (n == 0) {
    ix.n_intervals = ix.n_keys = ix.n_blocks = 0;
    return MX_OK;
  }
  DevBuf<u32> a[4], b[4], hist, dtot;
  for (int j = 0; j < 4; ++j) {
    MX_CUDA_TRY(a[j].alloc(n, s));
    MX_CUDA_TRY(b[j].alloc(n, s));
  }
  owner_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, reinterpret_cast<const uint4*>(rows),
                                                               dense_bits > 0, a[0].p, a[1].p, a[2].p, a[3].p);
  mx_count_launch();
  const int tiles = (int)((n + RS_THREADS * 8 - 1) / (RS_THREADS * 8));
  MX_CUDA_TRY(hist.alloc((long long)256 * tiles, s));
  MX_CUDA_TRY(dtot.alloc(256, s));
  MX_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(4 * RS_THREADS * 8 * sizeof(u32))));
  u32 *k = a[0].p, *f = a[1].p, *st = a[2].p, *en = a[3].p;
  u32 *k2 = b[0].p, *f2 = b[1].p, *st2 = b[2].p, *en2 = b[3].p;
  if (dense_bits > 0) {
    // rows file-ordered within each key (sources concatenated in rank order)
    // with a dense key rank in .w: one stable sort by that rank, then the
    // packed keys gathered back through the row ids
    if (int rc = radix_sort_by(k, f, st, en, k2, f2, st2, en2, n, dense_bits, hist.p, dtot.p, s)) return rc;
    owner_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, reinterpret_cast<const uint4*>(rows), st, k);
    mx_count_launch();
  } else {
    if (int rc = radix_sort_by(f, k, st, en, f2, k2, st2, en2, n, bits_of((u32)std::max(0, n_files - 1)), hist.p,
                               dtot.p, s))
      return rc;
    if (int rc = radix_sort_by(k, f, st, en, k2, f2, st2, en2, n, (int)ix.key_bits, hist.p, dtot.p, s)) return rc;
  }
  MX_CUDA_TRY(ix.iv_key.alloc(n, s));
  MX_CUDA_TRY(ix.iv_file.alloc(n, s));
  MX_CUDA_TRY(ix.iv_start.alloc(n, s));
  MX_CUDA_TRY(ix.iv_end.alloc(n, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.iv_key.p, k, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.iv_file.p, f, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(ix.owner_row.alloc(n, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.owner_row.p, st, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
  MX_CUDA_TRY(cudaMemsetAsync(ix.iv_start.p, 0, sizeof(u32) * n, s));
  MX_CUDA_TRY(cudaMemcpyAsync(ix.iv_end.p, en, sizeof(u32) * n, cudaMemcpyDeviceToDevice, s));
  int rc = index_finalize(&ix, n, s);
  ix.n_samples_total = ix.indexed_samples;
  return rc;
}

}  // namespace mx
