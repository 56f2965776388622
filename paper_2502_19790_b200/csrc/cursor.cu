// Generator setup: RangeCursor layouts + component order, on device.
//
// Reference: RangeCursor.__init__ (index.py:126-147) -- per component key,
//   rng = Random(derive_seed(seed, "cursor", key.canonical_string()))
//   shuffle the sorted dataset ids, then each dataset's sorted file ids (same
//   rng), concatenate each file's intervals ascending;
// ChunkGenerator.__init__ (chunks.py:139-141) -- component keys in sort order
//   shuffled by Random(derive_seed(seed, "component-order")).
//
// Kernels: key_mt_seed_kernel (one thread per key: device BLAKE2b of the
// key's canonical string, then the MT19937 init_by_array chain),
// cursor_shuffle_kernel (one CTA per key: the dataset / file shuffles drawn
// 128 outputs per window, applied in parallel (csrc/mt19937.cuh)), the
// interval-level layout civ / ccum / cfile / cstart by one reduce-then-scan
// over the shuffled blocks (CursorF),
// component_order_kernel (one warp: the shuffle of K ranks).
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

// One THREAD per key (derive_seed(seed, "cursor", key string) by device
// BLAKE2b), then the
// key's MT19937 init_by_array chain in shared memory (lane-interleaved rows of
// 33 words, conflict-free), copied out 32 keys interleaved (mt_state_of).
constexpr int SEED_THREADS = 32;
constexpr int SEED_ROW = SEED_THREADS + 1;
constexpr int SEED_MSG = 128;  // one BLAKE2b block per thread in shared memory

__global__ void __launch_bounds__(SEED_THREADS)
key_mt_seed_kernel(KeyStrView v, long long K, const uint8_t* prefix, int prefix_len, u32* states) {
  extern __shared__ u32 ks_dyn[];  // [MT_N][SEED_ROW] + [SEED_THREADS][SEED_MSG] bytes
  const int lane = threadIdx.x;
  const long long k0 = blockIdx.x * (long long)SEED_THREADS, k = k0 + lane;
  uint8_t* msg = reinterpret_cast<uint8_t*>(ks_dyn + MT_N * SEED_ROW) + lane * SEED_MSG;
  if (k < K) {
    u64 seed = 0;
    {
      // stable_hash message: prefix, 8-byte length, "v1;v2;..." of the
      // key's present properties; assembled in the thread's shared row
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
      const long long total = prefix_len + 8 + len;
      if (total <= SEED_MSG) {
        for (int q = 0; q < prefix_len; ++q) msg[q] = prefix[q];
        int w = prefix_len;
#pragma unroll
        for (int b = 7; b >= 0; --b) msg[w++] = (uint8_t)((u64)len >> (8 * b));
        present = 0;
        for (int p = 0; p < v.n_props; ++p) {
          u32 r = (packed >> v.shift[p]) & ((1u << v.width[p]) - 1u);
          if (r) {
            if (present) msg[w++] = ';';
            const long long pc = v.base[p] + r - 1, o0 = v.off[pc], nb = v.off[pc + 1] - o0;
#pragma unroll 4
            for (long long q = 0; q < nb; ++q) msg[w + q] = v.bytes[o0 + q];
            w += (int)nb;
            ++present;
          }
        }
        seed = blake2b_seed63_1block((int)total, [&](int i) { return msg[i]; });
      } else {  // long key strings: the streaming hash
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
        seed = b.seed63();
      }
    }
    mt_init_by_array(seed, [&](int a) -> u32& { return ks_dyn[a * SEED_ROW + lane]; });
  }
  __syncwarp();
  // states of 32 consecutive keys interleaved: word a of key k at
  // states[((k / 32) * MT_N + a) * 32 + k % 32] (coalesced here)
  u32* dst = states + (size_t)blockIdx.x * MT_N * SEED_THREADS + lane;
#pragma unroll 8
  for (int a = 0; a < MT_N; ++a) dst[(size_t)a * SEED_THREADS] = ks_dyn[a * SEED_ROW + lane];
}

__device__ __forceinline__ const u32* mt_state_of(const u32* states, long long k) {
  return states + (size_t)(k / SEED_THREADS) * MT_N * SEED_THREADS + k % SEED_THREADS;
}

// One CTA (CS_THREADS) per key, grid-stride: the key's seeded MT state
// (key_mt_seed_kernel) in shared memory; warp 0 draws the shuffle (WarpMT::
// draws, 128 outputs per window) and builds the ascending bucket lists
// (fy_lists), then the whole CTA resolves the positions (fy_resolve). The
// interval-level layout is one device-wide scan afterwards (CursorF): per key
// it is a chain of dependent gathers that leaves the device idle at 1B
// samples (measured 0.4 ms per key there, clock64). Keys with several datasets
// (the dataset-order shuffle first, then every dataset's blocks from the
// same stream) run the warp form (cursor_key_shuffle) on warp 0. Draw /
// bucket scratch: 16-bit entries in shared memory (4 B per block) for keys
// with <= cap blocks, else u32 global scratch at the key's block offset.
constexpr int CS_THREADS = 64;  // 16 CTAs per SM: every cfg2 key resident at once
constexpr int CS_MT_WORDS = 2 * MT_N;
constexpr int CS_SMEM_CAP = 16000;

template <typename IT>
__device__ void cursor_key_shuffle(WarpMT& mt, u32 b0, int nb, int G, const u32* grp, u32* gid, u32* cur_blk, IT* j,
                                   IT* top) {
  // dataset order (one stream for the whole key)
  mt.draws(G, j);
  fy_apply(G, j, top, [&](int i, u32 v) { gid[b0 + i] = v; });
  // every dataset's draws in the shuffled dataset order, then one apply each
  int pos = 0;
  for (int g = 0; g < G; ++g) {
    const u32 gi = gid[b0 + g];
    const int s = (int)grp[b0 + gi];
    const int e = gi + 1 < (u32)G ? (int)grp[b0 + gi + 1] : nb;
    mt.draws(e - s, j + pos);
    pos += e - s;
  }
  pos = 0;
  for (int g = 0; g < G; ++g) {
    const u32 gi = gid[b0 + g];
    const int s = (int)grp[b0 + gi];
    const int e = gi + 1 < (u32)G ? (int)grp[b0 + gi + 1] : nb;
    u32* dst = cur_blk + b0 + pos;
    const u32 base = b0 + (u32)s;
    fy_apply(e - s, j + pos, top + pos, [&](int i, u32 v) { dst[i] = base + v; });
    pos += e - s;
  }
}

__global__ void __launch_bounds__(CS_THREADS)
cursor_shuffle_kernel(long long K, const u32* key_blk_first, const u32* blk_file, const int32_t* file_ds,
                      const u32* states, u32* grp, u32* gid, u32* cur_blk, int cap, u32* g_j, u32* g_top) {
  extern __shared__ __align__(16) u32 cs_dyn[];
  __shared__ int s_G;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  u32* mt_s = cs_dyn;
  unsigned short* s_j = reinterpret_cast<unsigned short*>(cs_dyn + CS_MT_WORDS);
  unsigned short* s_top = s_j + cap;
  for (long long k = blockIdx.x; k < K; k += gridDim.x) {
    const u32 b0 = key_blk_first[k], b1 = key_blk_first[k + 1];
    const int nb = (int)(b1 - b0);
    if (nb == 0) continue;
    if (nb == 1) {  // shuffling one block draws nothing
      if (tid == 0) cur_blk[b0] = b0;
      continue;
    }
    const u32* st = mt_state_of(states, k);
    for (int a = tid; a < MT_N; a += CS_THREADS) mt_s[a] = st[(size_t)a * SEED_THREADS];
    // dataset groups (blocks are file-sorted and ds is nondecreasing in file
    // order): one group when first and last block share a dataset, else a
    // warp-parallel scan of dataset changes
    if (w == 0) {
      int G = 1;
      if (file_ds[blk_file[b0]] != file_ds[blk_file[b1 - 1]]) {
        G = 0;
        for (int b = 0; b < nb; b += 32) {
          const int i = b + lane;
          bool hd = false;
          if (i < nb) hd = i == 0 || file_ds[blk_file[b0 + i]] != file_ds[blk_file[b0 + i - 1]];
          const u32 hm = __ballot_sync(MX_FULL, hd);
          if (hd) grp[b0 + G + __popc(hm & ((1u << lane) - 1))] = (u32)i;
          G += __popc(hm);
        }
      }
      if (lane == 0) s_G = G;
    }
    __syncthreads();
    const int G = s_G;
    const bool in_smem = nb <= cap;
    if (w == 0) {
      WarpMT mt{mt_s, mt_s + MT_N, MT_N};
      if (G == 1) {
        if (in_smem) {
          mt.draws(nb, s_j);
          fy_lists(nb, s_j, s_top);
        } else {
          mt.draws(nb, g_j + b0);
          fy_lists(nb, g_j + b0, g_top + b0);
        }
      } else if (in_smem) {
        cursor_key_shuffle<unsigned short>(mt, b0, nb, G, grp, gid, cur_blk, s_j, s_top);
      } else {
        cursor_key_shuffle<u32>(mt, b0, nb, G, grp, gid, cur_blk, g_j + b0, g_top + b0);
      }
    }
    __syncthreads();
    if (G == 1) {
      auto out = [&](int i, u32 v) { cur_blk[b0 + i] = b0 + v; };
      if (in_smem) fy_resolve(nb, s_j, s_top, tid, CS_THREADS, out);
      else fy_resolve(nb, g_j + b0, g_top + b0, tid, CS_THREADS, out);
    }
    __syncthreads();
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

// Both layouts in ONE scan over the cursor's blocks when the index holds
// < 2^32 samples: the value of block position p packs (intervals << 32 |
// samples) of block cur_blk[p], so the exclusive prefix gives the block's
// first cursor position and its sample offset at once (sums never carry).
struct CursorF {
  const u32* cur_blk;
  const u32* blk_first;
  const u64* iv_cum;
  const u32* start;
  const u32* end;
  const u32* file;
  u32* civ;
  u64* cum;
  u32* cfile;
  u32* cstart;
  __device__ u64 value(long long p) const {
    const u32 b = cur_blk[p];
    const u32 f0 = blk_first[b], f1 = blk_first[b + 1];
    return ((u64)(f1 - f0) << 32) | (iv_cum[f1] - iv_cum[f0]);
  }
  __device__ void apply(long long p, u64 ex, u64) const {
    const u32 b = cur_blk[p];
    const u32 f0 = blk_first[b], f1 = blk_first[b + 1];
    const u64 pos = ex >> 32;
    u64 samp = ex & 0xffffffffull;
    if (p == 0) cum[0] = 0;
    for (u32 t = 0; t < f1 - f0; ++t) {
      const u32 iv = f0 + t, a = start[iv];
      civ[pos + t] = iv;
      cfile[pos + t] = file[iv];
      cstart[pos + t] = a;
      samp += end[iv] - a;
      cum[pos + t + 1] = samp;
    }
  }
  __device__ void total(u64) const {}
};

__global__ void comp_total_kernel(long long K, const u32* key_blk_first, const u32* blk_first, const u64* iv_cum,
                                  u64* total) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= K) return;
  total[k] = iv_cum[blk_first[key_blk_first[k + 1]]] - iv_cum[blk_first[key_blk_first[k]]];
}

// one warp: the shuffle of the K component ranks (chunks.py:139-141); 16-bit
// scratch in shared memory up to CO_SMEM ranks, else u32 global scratch
constexpr int CO_SMEM = 16384;

__global__ void __launch_bounds__(32) component_order_kernel(long long K, u64 seed, u32* order, u32* g_j,
                                                           u32* g_top) {
  extern __shared__ __align__(16) u32 co_dyn[];
  const int n = (int)K, lane = threadIdx.x;
  WarpMT mt{co_dyn, co_dyn + MT_N, MT_N};
  // the component-order seed comes from the host: seeded here (lane 0) so
  // the shuffle does not wait for the per-key seed kernel
  if (lane == 0) mt_init_by_array(seed, [&](int a) -> u32& { return co_dyn[a]; });
  __syncwarp();
  auto out = [&](int i, u32 v) { order[i] = v; };
  if (n <= CO_SMEM) {
    unsigned short* s_j = reinterpret_cast<unsigned short*>(co_dyn + CS_MT_WORDS);
    mt.draws(n, s_j);
    fy_apply(n, s_j, s_j + n, out);
  } else {
    mt.draws(n, g_j);
    fy_apply(n, g_j, g_top, out);
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
  MX_CUDA_TRY(g->comp_order.alloc(K, s));
  MX_CUDA_TRY(cudaEventRecord(g->ev_tot, s));
  mx_host_mark("cursor prologue");
  // the component-order shuffle runs on a side stream, overlapped with the
  // per-key seeds and cursor shuffles
  MX_CUDA_TRY(cudaStreamWaitEvent(g->ostream, g->ev_tot, 0));
  {
    DevBuf<u32> fj, ft;  // global scratch only beyond CO_SMEM ranks
    const long long gn = K > CO_SMEM ? K : 1;
    MX_CUDA_TRY(ws_borrow(fj, g->ostream, WS_FYJ, gn));
    MX_CUDA_TRY(ws_borrow(ft, g->ostream, WS_FYTOP, gn));
    const size_t dyn = sizeof(u32) * CS_MT_WORDS + (K <= CO_SMEM ? 4 * (size_t)K : 0);
    MX_CUDA_TRY(mx_smem_attr(component_order_kernel, dyn));
    component_order_kernel<<<1, 32, dyn, g->ostream>>>(K, order_seed, g->comp_order.p, fj.p, ft.p);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaEventRecord(g->ev_order, g->ostream));
  // every key's cursor seed + seeded MT state
  DevBuf<uint8_t> pre;
  DevBuf<u32> states;
  MX_CUDA_TRY(ws_borrow(pre, s, WS_CPRE, prefix_len > 0 ? prefix_len : 1));
  if (prefix_len > 0)
    MX_CUDA_TRY(mx_h2d(pre.p, cursor_prefix, prefix_len, s));
  MX_CUDA_TRY(ws_borrow(states, s, WS_CSEED, (K + SEED_THREADS - 1) / SEED_THREADS * SEED_THREADS * MT_N));
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
  {
    const size_t dyn = sizeof(u32) * MT_N * SEED_ROW + (size_t)SEED_MSG * SEED_THREADS;
    MX_CUDA_TRY(mx_smem_attr(key_mt_seed_kernel, dyn));
    key_mt_seed_kernel<<<(unsigned)((K + SEED_THREADS - 1) / SEED_THREADS), SEED_THREADS, dyn, s>>>(
        v, K, pre.p, prefix_len, states.p);
    mx_count_launch();
  }
  DevBuf<u32> grp, gid;
  MX_CUDA_TRY(ws_borrow(grp, s, WS_CGRP, B));
  MX_CUDA_TRY(ws_borrow(gid, s, WS_CGID, B));
  MX_CUDA_TRY(g->cur_blk.alloc(B, s));
  {
    MxPhase ph2("cursor_shuffle", s);
    // keys with <= cap blocks keep their scratch in shared memory (4 B per
    // block); larger keys use the u32 global scratch
    static thread_local std::map<size_t, int> occ;  // smem -> resident CTAs per SM
    static thread_local int n_sm = 0;
    if (!n_sm) {
      int dev = 0;
      MX_CUDA_TRY(cudaGetDevice(&dev));
      MX_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    const long long mkb = ix->max_key_blocks;
    const long long need = std::min<long long>(16, (K + n_sm - 1) / n_sm);  // CTAs per SM for one wave
    const long long budget = 227 * 1024 / std::max(need, 1ll) - 1024 - 4 * CS_MT_WORDS;
    const int cap_fit = (int)std::max<long long>(64, budget / 4 / 64 * 64);
    // shared scratch for every key unless that needs more than 3 waves of
    // keys (a key in global scratch runs ~3.5x longer: 1B, clock64)
    const int cap_full = (int)std::min<long long>((mkb + 63) / 64 * 64, CS_SMEM_CAP);
    const long long per_sm_full =
        std::max<long long>(1, std::min<long long>(16, 227 * 1024 / ((long long)CS_MT_WORDS * 4 + 4ll * cap_full + 1024)));
    const long long waves = (K + per_sm_full * n_sm - 1) / (per_sm_full * n_sm);
    const int cap = waves <= 3 ? cap_full : std::min(cap_full, cap_fit);
    DevBuf<u32> fj, ft;
    const long long gn = mkb > cap ? B : 1;
    MX_CUDA_TRY(ws_borrow(fj, s, WS_FYJ, gn));
    MX_CUDA_TRY(ws_borrow(ft, s, WS_FYTOP, gn));
    const size_t dyn = (size_t)CS_MT_WORDS * 4 + (size_t)cap * 4;
    MX_CUDA_TRY(mx_smem_attr(cursor_shuffle_kernel, dyn));
    int& per_sm = occ[dyn];
    if (!per_sm)
      MX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cursor_shuffle_kernel, CS_THREADS, dyn));
    const long long blocks = std::min<long long>(K, (long long)std::max(per_sm, 1) * n_sm);
    cursor_shuffle_kernel<<<(unsigned)blocks, CS_THREADS, dyn, s>>>(
        K, ix->key_blk_first.p, ix->blk_file.p, ix->file_ds.p, states.p, grp.p, gid.p, g->cur_blk.p, cap, fj.p, ft.p);
    mx_count_launch();
  }
  MX_CUDA_TRY(g->civ.alloc(I, s));
  MX_CUDA_TRY(g->ccum.alloc(I + 1, s));
  MX_CUDA_TRY(g->cfile.alloc(I, s));
  MX_CUDA_TRY(g->cstart.alloc(I, s));
  if (ix->indexed_samples < (1ll << 32) && I < (1ll << 31)) {  // resolved sizes (ix_resolve)
    if (int rc = gs_run(B, CursorF{g->cur_blk.p, ix->blk_first.p, ix->iv_cum.p, ix->iv_start.p, ix->iv_end.p,
                                   ix->iv_file.p, g->civ.p, g->ccum.p, g->cfile.p, g->cstart.p}, s))
      return rc;
  } else {  // >= 2^32 samples: positions first, then the 64-bit sample prefix
    if (int rc = gs_run(B, CursorIvF{g->cur_blk.p, ix->blk_first.p, g->civ.p}, s)) return rc;
    if (int rc = gs_run(I, CumPermF{g->civ.p, ix->iv_start.p, ix->iv_end.p, g->ccum.p, ix->iv_file.p, g->cfile.p,
                                     g->cstart.p}, s))
      return rc;
  }
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
