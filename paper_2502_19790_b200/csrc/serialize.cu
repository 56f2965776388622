// Canonical chunk bytes on the device.
//
// Reference: Chunk.to_json / serialize (chunks.py:54-93) through
// canonical_json (seeding.py:36-42) = json.dumps(sort_keys=True,
// separators=(",", ":"), ensure_ascii=True):
//
//   {"chunk_id":ID,"data":{KEY:{"DS":{"FID":[[s,e],...],...},...},...},
//    "mixture":MIX,"seed":SEED,"version":1}
//
// sort_keys orders the data levels by STRING: canonical key strings, str(ds)
// and str(fid) compare lexicographically ("10" < "9"), not in the numeric /
// MixtureKey order the chunk CSR uses. The host supplies the JSON-quoted key
// strings with their string ranks and a per-file rank in (str(ds), str(fid))
// order; per chunk the pieces are re-sorted by (key rank, file rank, position)
// -- a warp register bitonic sort for chunks of <= 32 ranges, a shared-memory
// bitonic sort per CTA above -- and every piece's text is sized (pass 1),
// the chunk sizes are scanned, and the text is written (pass 2) with a
// warp-wide scan of per-piece lengths. MIX (the spec's canonical JSON, the
// same for every chunk of a batch) comes from the host.
#include "common.cuh"
#include "mixtera_internal.cuh"

namespace mx {

struct JsonArgs {
  long long n_chunks;
  const long long* off;  // [C+1] ranges per chunk
  const u32* mkey;
  const u32* file;
  const u32* start;
  const u32* end;
  const long long* ids;
  const u64* seeds;
  const uint8_t* key_json;       // JSON-quoted key strings
  const long long* key_json_off; // [n_keys+1]
  const u32* key_rank;           // string rank of each key
  const u32* file_rank;          // rank of each file in (str(ds), str(fid)) order
  const int32_t* file_ds;
  const long long* file_ids;
  const uint8_t* mix;            // canonical JSON of the mixture ("null" if none)
  int mix_len;
  u32* perm;                     // [R] sorted piece order (chunk-local indices)
  long long* chunk_len;          // [C] bytes per chunk
  u32* too_big;                  // largest chunk beyond the shared-memory sort (0 = none)
  const long long* json_off;     // [C+1] byte offsets
  uint8_t* out;
};

__device__ __forceinline__ int dec_digits(u64 v) {
  int n = 1;
  while (v >= 10) {
    v /= 10;
    ++n;
  }
  return n;
}

__device__ __forceinline__ void dec_write(uint8_t* p, u64 v, int n) {
  for (int i = n - 1; i >= 0; --i) {
    p[i] = (uint8_t)('0' + v % 10);
    v /= 10;
  }
}

__device__ __forceinline__ int i64_digits(long long v) { return v < 0 ? 1 + dec_digits((u64)(-v)) : dec_digits((u64)v); }

__device__ __forceinline__ void i64_write(uint8_t* p, long long v, int n) {
  if (v < 0) {
    *p = '-';
    dec_write(p + 1, (u64)(-v), n - 1);
  } else {
    dec_write(p, (u64)v, n);
  }
}

__device__ __forceinline__ void put(uint8_t*& p, const char* s) {
  while (*s) *p++ = (uint8_t)*s++;
}

// header {"chunk_id":ID,"data":{  and trailer }}},"mixture":MIX,"seed":S,"version":1}
__device__ __forceinline__ int header_len(long long id) { return 21 + i64_digits(id); }
__device__ __forceinline__ int trailer_len(const JsonArgs& a, u64 seed) {
  return 4 + 11 + a.mix_len + 8 + dec_digits(seed) + 13;
}

// text of sorted piece j of a chunk given its predecessor (prev = -1: first)
struct PieceText {
  u32 nk, nd, nf;  // opens a new key / dataset / file group
  int len;
};

__device__ __forceinline__ PieceText piece_text(const JsonArgs& a, long long base, int i, int prev) {
  PieceText t;
  const u32 m = a.mkey[base + i], f = a.file[base + i];
  const int32_t ds = a.file_ds[f];
  if (prev < 0) {
    t.nk = t.nd = t.nf = 1;
  } else {
    const u32 pm = a.mkey[base + prev], pf = a.file[base + prev];
    t.nk = m != pm;
    t.nd = t.nk || ds != a.file_ds[pf];
    t.nf = t.nd || f != pf;
  }
  int len = prev < 0 ? 0 : (t.nk ? 4 : t.nd ? 3 : t.nf ? 2 : 1);  // ]}}, / ]}, / ], / ,
  if (t.nk) len += (int)(a.key_json_off[m + 1] - a.key_json_off[m]) + 2;  // KEY:{
  if (t.nd) len += 4 + i64_digits(ds);                                  // "DS":{
  if (t.nf) len += 4 + i64_digits(a.file_ids[f]);                       // "FID":[
  len += 3 + dec_digits(a.start[base + i]) + dec_digits(a.end[base + i]);  // [s,e]
  t.len = len;
  return t;
}

__device__ void piece_write(const JsonArgs& a, long long base, int i, const PieceText& t, bool first, uint8_t* p) {
  const u32 m = a.mkey[base + i], f = a.file[base + i];
  if (!first) put(p, t.nk ? "]}}," : t.nd ? "]}," : t.nf ? "]," : ",");
  if (t.nk) {
    for (long long k = a.key_json_off[m]; k < a.key_json_off[m + 1]; ++k) *p++ = a.key_json[k];
    put(p, ":{");
  }
  if (t.nd) {
    const int32_t ds = a.file_ds[f];
    const int n = i64_digits(ds);
    *p++ = '"';
    i64_write(p, ds, n);
    p += n;
    put(p, "\":{");
  }
  if (t.nf) {
    const long long fid = a.file_ids[f];
    const int n = i64_digits(fid);
    *p++ = '"';
    i64_write(p, fid, n);
    p += n;
    put(p, "\":[");
  }
  *p++ = '[';
  const u32 s = a.start[base + i], e = a.end[base + i];
  const int ns = dec_digits(s), ne = dec_digits(e);
  dec_write(p, s, ns);
  p += ns;
  *p++ = ',';
  dec_write(p, e, ne);
  p += ne;
  *p++ = ']';
}

__device__ __forceinline__ u64 sort_key(const JsonArgs& a, long long base, int i) {
  return ((u64)a.key_rank[a.mkey[base + i]] << 48) | ((u64)a.file_rank[a.file[base + i]] << 16) | (u64)i;
}

// ---- pass 1: order + size. Chunks of <= 32 ranges: one warp each.
__global__ void __launch_bounds__(256) json_size_warp_kernel(JsonArgs a, u32* big_list, u32* big_cnt) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < a.n_chunks; c += warps) {
    const long long base = a.off[c];
    const int n = (int)(a.off[c + 1] - base);
    if (n > 32) {
      if (lane == 0) big_list[atomicAdd(big_cnt, 1u)] = (u32)c;
      continue;
    }
    u64 k = lane < n ? sort_key(a, base, lane) : ~0ull;
    // bitonic sort of 32 keys across lanes
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const u64 o = __shfl_xor_sync(MX_FULL, k, stride);
        const bool up = (lane & size) == 0;
        const bool lower = (lane & stride) == 0;
        const u64 lo = k < o ? k : o, hi = k < o ? o : k;
        k = (lower == up) ? lo : hi;
      }
    }
    const int idx = (int)(k & 0xffff);
    const int prev = __shfl_up_sync(MX_FULL, idx, 1);
    int len = 0;
    if (lane < n) {
      a.perm[base + lane] = (u32)idx;
      len = piece_text(a, base, idx, lane == 0 ? -1 : prev).len;
    }
    len = warp_sum(len);
    if (lane == 0) a.chunk_len[c] = header_len(a.ids[c]) + len + trailer_len(a, a.seeds[c]);
  }
}

constexpr int JS_CAP = 2048;

// chunks of 33..2048 ranges: one CTA each, shared-memory bitonic sort
__global__ void __launch_bounds__(256) json_size_block_kernel(JsonArgs a, const u32* big_list, const u32* big_cnt) {
  __shared__ u64 s_k[JS_CAP];
  __shared__ long long s_sum[8];
  const u32 nb = *big_cnt;
  for (u32 bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const long long c = big_list[bi];
    const long long base = a.off[c];
    const int n = (int)(a.off[c + 1] - base);
    if (n > JS_CAP) {  // beyond the shared-memory sort: the caller serialises on the host
      if (threadIdx.x == 0) atomicMax(a.too_big, (u32)n);
      continue;
    }
    int np = 64;
    while (np < n) np <<= 1;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s_k[i] = i < n ? sort_key(a, base, i) : ~0ull;
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
          const int j = i ^ stride;
          if (j > i) {
            const bool up = (i & size) == 0;
            const u64 x = s_k[i], y = s_k[j];
            if ((x > y) == up) {
              s_k[i] = y;
              s_k[j] = x;
            }
          }
        }
        __syncthreads();
      }
    long long len = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int idx = (int)(s_k[i] & 0xffff);
      a.perm[base + i] = (u32)idx;
      len += piece_text(a, base, idx, i == 0 ? -1 : (int)(s_k[i - 1] & 0xffff)).len;
    }
    len = warp_sum(len);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = len;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_sum[w];
      a.chunk_len[c] = header_len(a.ids[c]) + t + trailer_len(a, a.seeds[c]);
    }
    __syncthreads();
  }
}

// ---- pass 2: one warp per chunk writes header, pieces (32 at a time, warp
// scan of lengths), trailer
__global__ void __launch_bounds__(256) json_write_kernel(JsonArgs a) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < a.n_chunks; c += warps) {
    const long long base = a.off[c];
    const int n = (int)(a.off[c + 1] - base);
    uint8_t* p = a.out + a.json_off[c];
    const long long id = a.ids[c];
    const int hl = header_len(id);
    if (lane == 0) {
      uint8_t* q = p;
      put(q, "{\"chunk_id\":");
      const int nd = i64_digits(id);
      i64_write(q, id, nd);
      q += nd;
      put(q, ",\"data\":{");
    }
    long long at = hl;
    for (int g = 0; g < n; g += 32) {
      const int j = g + lane;
      PieceText t{};
      int idx = 0;
      if (j < n) {
        idx = (int)a.perm[base + j];
        t = piece_text(a, base, idx, j == 0 ? -1 : (int)a.perm[base + j - 1]);
      }
      const int inc = warp_incl_scan(t.len);
      if (j < n) piece_write(a, base, idx, t, j == 0, p + at + inc - t.len);
      at += __shfl_sync(MX_FULL, inc, 31);
    }
    if (lane == 0) {
      uint8_t* q = p + at;
      put(q, "]}}},\"mixture\":");
      for (int k = 0; k < a.mix_len; ++k) *q++ = a.mix[k];
      put(q, ",\"seed\":");
      const u64 sd = a.seeds[c];
      const int nd = dec_digits(sd);
      dec_write(q, sd, nd);
      q += nd;
      put(q, ",\"version\":1}");
    }
  }
}

int gen_result_json(GenData* g, const mx_json_desc* d, cudaStream_t s) {
  const long long C = g->res_chunks, R = g->res_ranges;
  IndexData* ix = g->ix;
  MxPhase ph("json", s);
  g->json_bytes = 0;
  MX_CUDA_TRY(g->json_off.reserve(C + 1, s));
  if (C == 0) {
    const long long z = 0;
    MX_CUDA_TRY(mx_h2d(g->json_off.p, &z, sizeof(z), s));
    return MX_OK;
  }
  if (g->h_small_valid == C) {  // small plan: the result lives in the pinned mirror; publish it
    return mx_fail(MX_ERR_UNSUPPORTED, "device JSON of a small (mirrored) plan: use the host serializer");
  }
  const long long nk = d->n_keys;
  DevBuf<uint8_t> kj, mix;
  DevBuf<long long> kjo, len;
  DevBuf<u32> krank, frank, perm, blist, bcnt;
  const long long kbytes = d->key_json_off[nk];
  MX_CUDA_TRY(kj.alloc(kbytes > 0 ? kbytes : 1, s));
  MX_CUDA_TRY(kjo.alloc(nk + 1, s));
  MX_CUDA_TRY(krank.alloc(nk > 0 ? nk : 1, s));
  MX_CUDA_TRY(frank.alloc(ix->n_files, s));
  MX_CUDA_TRY(mix.alloc(d->mixture_len > 0 ? d->mixture_len : 1, s));
  MX_CUDA_TRY(mx_h2d(kj.p, d->key_json, kbytes, s));
  MX_CUDA_TRY(mx_h2d(kjo.p, d->key_json_off, sizeof(long long) * (nk + 1), s));
  MX_CUDA_TRY(mx_h2d(krank.p, d->key_rank, sizeof(u32) * nk, s));
  MX_CUDA_TRY(mx_h2d(frank.p, d->file_rank, sizeof(u32) * ix->n_files, s));
  MX_CUDA_TRY(mx_h2d(mix.p, d->mixture_json, d->mixture_len, s));
  MX_CUDA_TRY(perm.alloc(R > 0 ? R : 1, s));
  MX_CUDA_TRY(len.alloc(C, s));
  MX_CUDA_TRY(blist.alloc(C, s));
  MX_CUDA_TRY(bcnt.alloc(2, s));  // [big-chunk count, largest chunk beyond JS_CAP]
  MX_CUDA_TRY(cudaMemsetAsync(bcnt.p, 0, 2 * sizeof(u32), s));
  JsonArgs a{};
  a.n_chunks = C;
  a.off = g->res_off.p;
  a.mkey = g->res_mkey.p;
  a.file = g->res_file.p;
  a.start = g->res_start.p;
  a.end = g->res_end.p;
  a.ids = g->res_id.p;
  a.seeds = g->res_seed.p;
  a.key_json = kj.p;
  a.key_json_off = kjo.p;
  a.key_rank = krank.p;
  a.file_rank = frank.p;
  a.file_ds = ix->file_ds.p;
  a.file_ids = ix->file_ids.p;
  a.mix = mix.p;
  a.mix_len = d->mixture_len;
  a.perm = perm.p;
  a.chunk_len = len.p;
  a.too_big = bcnt.p + 1;
  const long long wgrid = std::min<long long>((C + 7) / 8, 148 * 16);
  json_size_warp_kernel<<<(unsigned)wgrid, 256, 0, s>>>(a, blist.p, bcnt.p);
  mx_count_launch();
  json_size_block_kernel<<<(unsigned)std::min<long long>(C, 148 * 4), 256, 0, s>>>(a, blist.p, bcnt.p);
  mx_count_launch();
  if (int rc = excl_scan_ll(reinterpret_cast<const u64*>(len.p), C, g->json_off.p, s)) return rc;
  long long total = 0;
  u32 too_big = 0;
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(&total, g->json_off.p + C, sizeof(long long)));
    MX_CUDA_TRY(rb.add(&too_big, bcnt.p + 1, sizeof(u32)));
    MX_CUDA_TRY(rb.sync());
  }
  if (too_big)
    return mx_fail(MX_ERR_UNSUPPORTED, "device JSON: a chunk has %u ranges (> %d); serialise it on the host", too_big,
                   JS_CAP);
  MX_CUDA_TRY(g->json.reserve(total > 0 ? total : 1, s));
  a.json_off = g->json_off.p;
  a.out = g->json.p;
  json_write_kernel<<<(unsigned)wgrid, 256, 0, s>>>(a);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  g->json_bytes = total;
  return MX_OK;
}

}  // namespace mx
