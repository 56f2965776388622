// Generator setup: RangeCursor layouts + component order, on device.
//
// Reference: RangeCursor.__init__ (index.py:126-147) -- per component key,
//   rng = Random(derive_seed(seed, "cursor", key.canonical_string()))
//   shuffle the sorted dataset ids, then each dataset's sorted file ids (same
//   rng), concatenate each file's intervals ascending;
// ChunkGenerator.__init__ (chunks.py:139-141) -- component keys in sort order
//   shuffled by Random(derive_seed(seed, "component-order")).
//
// Kernels: key_seed_kernel (device BLAKE2b of each key's canonical string),
// cursor_shuffle_kernel (one warp per key; MT19937 state and the key's block
// list (16-bit offsets) in shared memory; warp-parallel rejection sampling and
// conflict-free swap rounds, csrc/mt19937.cuh), CursorIvF (shuffled blocks ->
// interval ids, one reduce-then-scan over all keys),
// cum_len_kernel (u64 look-back scan of lengths in cursor order),
// component_order_kernel (one shuffle of K ranks).
#include <map>
#include "blake2b.cuh"
#include "common.cuh"
#include "mixtera_internal.cuh"
#include "mt19937.cuh"
#include "scan.cuh"

namespace mx {

struct KeyStrView {
  const u32* key_packed;
  int n_props;
  u32 shift[MX_MAX_PROPS];
  u32 width[MX_MAX_PROPS];
  int32_t base[MX_MAX_PROPS];
  const uint8_t* bytes;
  const long long* off;
};

__global__ void key_seed_kernel(KeyStrView v, long long K, const uint8_t* prefix, int prefix_len, u64* seeds) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const u32 packed = v.key_packed[k];
  long long len = 0;
  int present = 0;
  for (int p = 0; p < v.n_props; ++p) {
    u32 r = (packed >> v.shift[p]) & ((1u << v.width[p]) - 1u);
    if (r) {
      long long pc = v.base[p] + r - 1;
      len += v.off[pc + 1] - v.off[pc] + (present ? 1 : 0);
      ++present;
    }
  }
  Blake2b b;
  b.init();
  b.bytes(prefix, prefix_len);
  b.len8((u64)len);
  present = 0;
  for (int p = 0; p < v.n_props; ++p) {
    u32 r = (packed >> v.shift[p]) & ((1u << v.width[p]) - 1u);
    if (r) {
      if (present) b.byte(';');
      long long pc = v.base[p] + r - 1;
      b.bytes(v.bytes + v.off[pc], v.off[pc + 1] - v.off[pc]);
      ++present;
    }
  }
  seeds[k] = b.seed63();
}

// Per-warp shared memory: MT state + outputs + window pairs + the key's block
// list (list_cap entries; a key with more blocks shuffles in global memory).
// Per-warp shared memory: MT state + outputs + window pairs (CS_FIXED words)
// and the key's block list as 16-bit offsets from the key's first block
// (list_cap entries; a key with more blocks shuffles its u32 list in global
// memory). Half-width entries double the keys resident per SM.
constexpr int CS_FIXED = 2 * MT_N + 64;

__global__ void __launch_bounds__(128)
cursor_shuffle_kernel(long long K, const u32* key_blk_first, const u32* blk_file, const int32_t* file_ds,
                      const u64* seeds, const u32* mt_base, u32* grp, u32* gid, u32* cur_blk, int list_cap) {
  extern __shared__ __align__(16) u32 cs_dyn[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  u32* mine = cs_dyn + (size_t)w * (CS_FIXED + list_cap / 2);
  u32* s_mt = mine;
  u32* s_out = mine + MT_N;
  uint2* s_pairs = reinterpret_cast<uint2*>(mine + 2 * MT_N);
  unsigned short* s_list = reinterpret_cast<unsigned short*>(mine + CS_FIXED);
  for (long long k = blockIdx.x * (long long)wpc + w; k < K; k += (long long)gridDim.x * wpc) {
    const u32 b0 = key_blk_first[k], b1 = key_blk_first[k + 1];
    const int nb = (int)(b1 - b0);
    if (nb <= 1) {  // shuffling one block draws nothing: skip the MT seeding
      if (lane == 0 && nb == 1) cur_blk[b0] = b0;
      continue;
    }
    const bool in_smem = nb <= list_cap;
    // dataset groups (blocks are file-sorted and ds is nondecreasing in file
    // order): one group when first and last block share a dataset, else a
    // warp-parallel scan of dataset changes
    const bool one_ds = nb == 0 || file_ds[blk_file[b0]] == file_ds[blk_file[b1 - 1]];
    int G = 1;
    if (!one_ds) {
      G = 0;
      for (int b = 0; b < nb; b += 32) {
        const int i = b + lane;
        bool head = false;
        if (i < nb) head = i == 0 || file_ds[blk_file[b0 + i]] != file_ds[blk_file[b0 + i - 1]];
        const u32 hm = __ballot_sync(MX_FULL, head);
        if (head) {
          const int gi = G + __popc(hm & ((1u << lane) - 1));
          grp[b0 + gi] = (u32)i;
          gid[b0 + gi] = (u32)gi;
        }
        G += __popc(hm);
      }
    } else if (lane == 0) {
      grp[b0] = 0;
      gid[b0] = 0;
    }
    __syncwarp();
    WarpMT mt{s_mt, s_out, s_pairs, MT_N};
    mt.seed(mt_base, seeds[k]);
    mt.shuffle(gid + b0, G);  // dataset order (one stream for the whole key)
    int pos = 0;
    for (int g = 0; g < G; ++g) {
      const u32 gi = gid[b0 + g];
      const int s = (int)grp[b0 + gi];
      const int e = gi + 1 < (u32)G ? (int)grp[b0 + gi + 1] : nb;
      // the dataset's blocks in file order, then shuffled (file order within
      // the dataset, index.py:140-143)
      if (in_smem) {
        for (int b = s + lane; b < e; b += 32) s_list[pos + b - s] = (unsigned short)b;
        __syncwarp();
        mt.shuffle(s_list + pos, e - s);
      } else {
        for (int b = s + lane; b < e; b += 32) cur_blk[b0 + pos + b - s] = b0 + (u32)b;
        __syncwarp();
        mt.shuffle(cur_blk + b0 + pos, e - s);
      }
      pos += e - s;
    }
    __syncwarp();
    if (in_smem)
      for (int i = lane; i < nb; i += 32) cur_blk[b0 + i] = b0 + s_list[i];
    __syncwarp();
  }
}

// civ: interval ids in cursor order. Cursor positions of key k occupy the
// same index range as its intervals in sorted order, and keys are stored
// consecutively, so the output position of block p (in cursor order, keys
// concatenated) is the exclusive prefix of interval counts over [0, p).
struct CursorIvF {
  const u32* cur_blk;
  const u32* blk_first;
  u32* civ;
  __device__ u64 value(long long p) const {
    const u32 b = cur_blk[p];
    return blk_first[b + 1] - blk_first[b];
  }
  __device__ void apply(long long p, u64 ex, u64 v) const {
    const u32 f = blk_first[cur_blk[p]];
    for (u32 t = 0; t < (u32)v; ++t) civ[ex + t] = f + t;
  }
  __device__ void total(u64) const {}
};

// ccum[j + 1] = samples of cursor positions [0, j] (interval perm[j])
struct CumPermF {
  const u32* perm;
  const u32* start;
  const u32* end;
  u64* cum;
  const u32* file;
  u32* cfile;   // file / start of cursor position j (the emission's gathers, done once here)
  u32* cstart;
  __device__ u64 value(long long j) const {
    const u32 iv = perm[j];
    return end[iv] - start[iv];
  }
  __device__ void apply(long long j, u64 ex, u64 v) const {
    if (j == 0) cum[0] = 0;
    cum[j + 1] = ex + v;
    const u32 iv = perm[j];
    cfile[j] = file[iv];
    cstart[j] = start[iv];
  }
  __device__ void total(u64) const {}
};

__global__ void comp_total_kernel(long long K, const u32* key_blk_first, const u32* blk_first, const u64* iv_cum,
                                  u64* total) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  total[k] = iv_cum[blk_first[key_blk_first[k + 1]]] - iv_cum[blk_first[key_blk_first[k]]];
}

constexpr int CO_SMEM = 8192;

// one warp: shuffle of the K component ranks (chunks.py:139-141)
__global__ void __launch_bounds__(32) component_order_kernel(long long K, u64 seed, const u32* mt_base, u32* order) {
  __shared__ u32 s_mt[MT_N], s_out[MT_N];
  __shared__ uint2 s_pairs[32];
  __shared__ u32 s_ord[CO_SMEM];
  const int lane = threadIdx.x;
  const bool in_smem = K <= CO_SMEM;
  for (long long i = lane; i < K; i += 32) {
    if (in_smem) s_ord[i] = (u32)i;
    else order[i] = (u32)i;
  }
  __syncwarp();
  WarpMT mt{s_mt, s_out, s_pairs, MT_N};
  mt.seed(mt_base, seed);
  if (in_smem) {
    mt.shuffle(s_ord, (int)K);
    for (long long i = lane; i < K; i += 32) order[i] = s_ord[i];
  } else {
    mt.shuffle(order, (int)K);
  }
}

int cursor_build(IndexData* ix, const uint8_t* cursor_prefix, int prefix_len, unsigned long long order_seed,
                 cudaStream_t s, GenData* g) {
  g->ix = ix;
  g->stream = s;
  const long long K = ix->n_keys, B = ix->n_blocks, I = ix->n_intervals;
  g->K = K;
  MX_CUDA_TRY(g->consumed.alloc(K > 0 ? K : 1, s));
  MX_CUDA_TRY(cudaMemsetAsync(g->consumed.p, 0, sizeof(u64) * (K > 0 ? K : 1), s));
  if (K == 0) return MX_OK;
  MxPhase ph("cursor_layout", s);
  MX_CUDA_TRY(g->aux_init());
  // per-component totals first: the first plan (on g->pstream) waits only
  // for them, not for the shuffles below
  MX_CUDA_TRY(g->comp_total.alloc(K, s));
  comp_total_kernel<<<(unsigned)((K + 255) / 256), 256, 0, s>>>(K, ix->key_blk_first.p, ix->blk_first.p,
                                                               ix->iv_cum.p, g->comp_total.p);
  mx_count_launch();
  // the component-order shuffle (one sequential Fisher-Yates over K ranks)
  // runs on a side stream, overlapped with the per-key cursor shuffles
  static thread_local uint32_t h_base[MT_N];
  if (h_base[0] != 19650218u) mt_base_table(h_base);
  DevBuf<u32> mt_base;  // constant table: uploaded into the stream's workspace once
  {
    static thread_local std::map<cudaStream_t, u32*> uploaded;
    MX_CUDA_TRY(ws_borrow(mt_base, s, WS_MTBASE, MT_N));
    if (uploaded[s] != mt_base.p) {
      MX_CUDA_TRY(mx_h2d(mt_base.p, h_base, sizeof(h_base), s));
      uploaded[s] = mt_base.p;
    }
  }
  MX_CUDA_TRY(g->comp_order.alloc(K, s));
  MX_CUDA_TRY(cudaEventRecord(g->ev_tot, s));
  MX_CUDA_TRY(cudaStreamWaitEvent(g->ostream, g->ev_tot, 0));
  mx_host_mark("cursor prologue");
  component_order_kernel<<<1, 32, 0, g->ostream>>>(K, order_seed, mt_base.p, g->comp_order.p);
  mx_count_launch();
  MX_CUDA_TRY(cudaEventRecord(g->ev_order, g->ostream));
  DevBuf<uint8_t> pre;
  DevBuf<u64> seeds;
  MX_CUDA_TRY(ws_borrow(pre, s, WS_CPRE, prefix_len > 0 ? prefix_len : 1));
  if (prefix_len > 0)
    MX_CUDA_TRY(mx_h2d(pre.p, cursor_prefix, prefix_len, s));
  MX_CUDA_TRY(ws_borrow(seeds, s, WS_CSEED, K));
  KeyStrView v{};
  v.key_packed = ix->key_packed.p;
  v.n_props = ix->n_props;
  for (int p = 0; p < ix->n_props; ++p) {
    v.shift[p] = ix->field_shift[p];
    v.width[p] = ix->field_width[p];
    v.base[p] = ix->str_base[p];
  }
  v.bytes = ix->str_bytes.p;
  v.off = ix->str_off.p;
  key_seed_kernel<<<(unsigned)((K + 127) / 128), 128, 0, s>>>(v, K, pre.p, prefix_len, seeds.p);
  mx_count_launch();
  DevBuf<u32> grp, gid;
  MX_CUDA_TRY(ws_borrow(grp, s, WS_CGRP, B));
  MX_CUDA_TRY(ws_borrow(gid, s, WS_CGID, B));
  MX_CUDA_TRY(g->cur_blk.alloc(B, s));
  {
    MxPhase ph2("cursor_shuffle", s);
    // list capacity = the largest key's block count (up to 16K entries, 64 KB)
    const int cap = (int)std::min<long long>((ix->max_key_blocks + 63) / 64 * 64, 32768);
    const size_t per_warp = sizeof(u32) * CS_FIXED + sizeof(unsigned short) * cap;
    const int wpc = per_warp <= 12 * 1024 ? 4 : 1;
    const size_t dyn = per_warp * wpc;
    MX_CUDA_TRY(cudaFuncSetAttribute(cursor_shuffle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    long long blocks = (K + wpc - 1) / wpc;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cursor_shuffle_kernel<<<(unsigned)blocks, wpc * 32, dyn, s>>>(K, ix->key_blk_first.p, ix->blk_file.p,
                                                                ix->file_ds.p, seeds.p, mt_base.p, grp.p, gid.p,
                                                                g->cur_blk.p, cap);
    mx_count_launch();
  }
  MX_CUDA_TRY(g->civ.alloc(I, s));
  if (int rc = gs_run(B, CursorIvF{g->cur_blk.p, ix->blk_first.p, g->civ.p}, s)) return rc;
  MX_CUDA_TRY(g->ccum.alloc(I + 1, s));
  MX_CUDA_TRY(g->cfile.alloc(I, s));
  MX_CUDA_TRY(g->cstart.alloc(I, s));
  if (int rc = gs_run(I, CumPermF{g->civ.p, ix->iv_start.p, ix->iv_end.p, g->ccum.p, ix->iv_file.p, g->cfile.p,
                                   g->cstart.p}, s))
    return rc;
  if (int rc = gen_local_lists(g, s)) return rc;  // sharded index: this rank's cursor positions
  MX_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_order, 0));
  g->fresh_layout = true;
  MX_CUDA_TRY(cudaGetLastError());
  g->mirrors_valid = false;  // host copies of comp_order / comp_total on first use
  return MX_OK;
}

int gen_host_mirrors(GenData* g) {
  if (g->mirrors_valid || g->K == 0) return MX_OK;
  g->h_comp_order.resize(g->K);
  g->h_comp_total.resize(g->K);
  MX_CUDA_TRY(cudaMemcpyAsync(g->h_comp_order.data(), g->comp_order.p, sizeof(u32) * g->K, cudaMemcpyDeviceToHost,
                              g->stream));
  MX_CUDA_TRY(cudaMemcpyAsync(g->h_comp_total.data(), g->comp_total.p, sizeof(u64) * g->K, cudaMemcpyDeviceToHost,
                              g->stream));
  MX_CUDA_TRY(cudaStreamSynchronize(g->stream));
  g->mirrors_valid = true;
  return MX_OK;
}


// Offset of every interval of the generator's index in its key's cursor
// stream (in the owner index's input row order when it has one, else index
// order): position j of the cursor layout holds interval
// civ[j]; key k's positions occupy [blk_first[key_blk_first[k]], ...).
// On an owner index (one pseudo-interval per (key, file) block) this is each
// block's cursor-stream offset -- what the file's owner rank needs to place
// its intervals in the global streams.
__global__ void block_offsets_kernel(long long I, const u32* civ, const u64* ccum, const u32* blk_key,
                                     const u32* key_blk_first, const u32* blk_first, const u32* row, u64* out) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= I) return;
  const u32 iv = civ[j];  // == its block (one interval per block)
  const u32 k = blk_key[iv];
  out[row ? row[iv] : iv] = ccum[j] - ccum[blk_first[key_blk_first[k]]];
}

int gen_block_offsets(GenData* g, u64* out, cudaStream_t s) {
  IndexData* ix = g->ix;
  if (ix->n_blocks != ix->n_intervals)
    return mx_fail(MX_ERR_INVALID, "block offsets need an index with one interval per block (an owner index)");
  const long long I = ix->n_intervals;
  if (I == 0) return MX_OK;
  block_offsets_kernel<<<(unsigned)((I + 255) / 256), 256, 0, s>>>(I, g->civ.p, g->ccum.p, ix->blk_key.p,
                                                                  ix->key_blk_first.p, ix->blk_first.p,
                                                                  ix->owner_row.n ? ix->owner_row.p : nullptr, out);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // namespace mx
