// Internal data structures behind the opaque C-ABI handles.
//
// HBM layout of an index (I = intervals, B = (key, file) blocks, K = keys):
//   iv_key/iv_file/iv_start/iv_end  u32[I]   sorted by (packed key, file, start)
//   iv_cum                          u64[I+1] cumulative samples in that order
//   blk_first u32[B+1], blk_file u32[B], blk_key u32[B]   (key, file) blocks
//   key_blk_first u32[K+1], key_packed u32[K]             keys in sort_key order
// A generator adds the RangeCursor layout:
//   cur_blk u32[B]   blocks of each key in shuffled cursor order
//   civ     u32[I]   interval ids in cursor order (key k owns the same index
//                    range [blk_first[key_blk_first[k]], ...) as in iv_*)
//   ccum    u64[I+1] cumulative samples in cursor order
//   consumed u64[K]  per-component samples already handed out
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/mixtera_b200.h"
#include "common.cuh"

#define MX_SMEM_LUT_MAX 12288
// scan_fast_kernel stages LUTs up to this many entries per CTA; larger ones
// (row-tuple layout) are read through L1 (one CTA per 2048-sample tile: a
// staged 2,000-entry LUT is as many bytes as the tile's column)
#define MX_STAGED_LUT_MAX 512

namespace mx {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  long long n = 0;
  cudaStream_t s = 0;
  bool own = true;  // false: a view into a block owned elsewhere (borrow)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t alloc(long long count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    own = true;
    if (count <= 0) return cudaSuccess;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (size_t)count, stream);
  }
  void borrow(void* ptr, long long count) {
    release();
    p = reinterpret_cast<T*>(ptr);
    n = count;
    own = false;
  }
  cudaError_t reserve(long long count, cudaStream_t stream) {  // grow-only
    if (p && n >= count) return cudaSuccess;
    return alloc(count, stream);
  }
  void release() {
    if (p && own) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    own = true;
  }
  void take(DevBuf& o) {
    release();
    p = o.p; n = o.n; s = o.s; own = o.own;
    o.p = nullptr; o.n = 0; o.own = true;
  }
};

// Grow-only device workspace per (host thread, stream) for the temporaries
// of a call (capi.cu): the stage-1 slot arrays are sized by the catalog
// (16 B per sample), and re-allocating them per job costs host time on the
// critical path before the first kernel. Buffers are reused in stream order;
// a view must never outlive the call that borrowed it.
enum WsSlot { WS_TCNT, WS_TOPEN, WS_THEAD, WS_DEFER, WS_RK, WS_RF, WS_RS, WS_RE, WS_SEGFA, WS_SCR64, WS_ERR,
              WS_HIST, WS_DTOT, WS_TOFF, WS_GSAGG, WS_CPRE, WS_CSEED, WS_CGRP, WS_CGID,
              WS_FYJ, WS_FYTOP,
              WS_EPRE, WS_EOFF, WS_EFLAG, WS_ELIST, WS_ELCNT, WS_ECPO, WS_EMCNT, WS_EBIG,  // emission temporaries
              WS_NBL, WS_NBC, WS_NWL, WS_NWC,  // cursor / component-order shuffle scratch
              WS_GEN,            // + GenData scratch slot (24 of them)
              WS_N = WS_GEN + 24 };
// `s` keys the workspace (a call's stream: work on it is ordered); growth
// frees / allocates in order on `alloc` (default: s)
cudaError_t ws_get(cudaStream_t s, int slot, size_t bytes, void** out, cudaStream_t alloc = nullptr,
                   bool alloc_set = false);
template <typename T>
cudaError_t ws_borrow(DevBuf<T>& b, cudaStream_t s, int slot, long long n) {
  void* p = nullptr;
  cudaError_t e = ws_get(s, slot, sizeof(T) * (size_t)(n > 0 ? n : 1), &p);
  if (e == cudaSuccess) b.borrow(p, n);
  return e;
}

struct IndexData {
  cudaStream_t stream = 0;
  long long n_samples_total = 0;
  int n_files = 0;
  u32 key_bits = 0;
  long long n_intervals = 0, n_keys = 0, n_blocks = 0;
  long long indexed_samples = 0;  // iv_cum[n_intervals]
  long long max_key_blocks = 0;   // blocks of the largest key
  DevBuf<u32> iv_key, iv_file, iv_start, iv_end;
  DevBuf<u64> iv_cum;
  DevBuf<u32> blk_first, blk_file, blk_key;
  DevBuf<u32> key_blk_first, key_packed;
  DevBuf<int32_t> file_ds;
  DevBuf<long long> file_ids;  // device copy of h_file_ids (result read-back mapping)
  std::vector<int32_t> h_file_ds;
  std::vector<int64_t> h_file_ids;
  // key codec (canonical strings for cursor seeds)
  int n_props = 0;
  u32 field_shift[MX_MAX_PROPS] = {};
  u32 field_width[MX_MAX_PROPS] = {};
  int32_t str_base[MX_MAX_PROPS] = {};
  DevBuf<uint8_t> str_bytes;
  DevBuf<long long> str_off;
  // one device block holding the small per-build host uploads (key strings,
  // file tables, LUTs: one copy); str_*, file_* may be views into it
  DevBuf<uint8_t> consts, consts2;  // LUTs (before the scan) / key strings + file tables (after)
  // file-sharded hybrid index (shard.cu): this rank's intervals + one
  // pseudo-interval per remote (key, file) block; files [file_lo, file_hi)
  // are local, iv_nreal = real intervals behind each entry (1 if local)
  bool sharded = false;
  long long file_lo = 0, file_hi = 0;
  long long n_local = 0;  // this rank's (real) intervals in the hybrid index
  DevBuf<u32> iv_nreal;
  DevBuf<u32> owner_row;  // owner index (owner_index_build): input row of every interval
  // sizes still travelling to the host (index_finalize with defer): the
  // build returns without waiting; ix_resolve() waits for them on first use
  struct Pending {
    u32 maxblk, pad;
    u64 totals, samples;
    DevError err;
  };
  Pending* pend = nullptr;  // slot of the pinned pool (capi.cu)
  cudaEvent_t pend_ev = nullptr;
  int pend_dev = -1;
  ~IndexData();
};

IndexData::Pending* pend_slot_take();  // nullptr: pool exhausted (finalize then waits)
void pend_slot_give(IndexData::Pending* slot);
// completes a deferred index_finalize (sizes, IndexBuildError); MX_OK when
// nothing is pending
int ix_resolve(IndexData* ix);

// per-device auxiliary streams (created once, shared by every generator on
// the device; non-blocking) and a pool of timing-disabled events (capi.cu):
// creating streams per generator costs ~50 us each
cudaError_t aux_streams(int dev, cudaStream_t out[3]);
cudaError_t aux_event_take(int dev, cudaEvent_t* e);
void aux_event_give(int dev, cudaEvent_t e);

// Key-partitioned emission (parallel.py build_partitioned): the generator
// plans over per-key totals (a key-level index) and cuts only THIS rank's
// intervals, placed by their blocks' offsets in the global cursor streams.
struct LocalSrc {
  const IndexData* loc = nullptr;  // this rank's index (file indices local)
  const u64* blk_off = nullptr;    // device [loc->n_blocks]: block offset in its key's global cursor stream
  const u32* key_g = nullptr;      // device [loc->n_keys]: global component rank of each local key
  long long file_lo = 0;           // global index of local file 0
  bool handoff = false;            // stop after the cut: chunk-grouped pieces for the chunk owners (handoff)
};

// Cut pieces of a partitioned plan, grouped by chunk, before the exchange to
// the chunk owners (mx_gen_handoff / mx_gen_finish_owned).
struct Handoff {
  DevBuf<long long> off;   // [n_chunks + 1] piece offsets per chunk
  DevBuf<uint4> pieces;    // (mixture key, global file, start, end)
  long long n_chunks = -1; // -1: none pending
  long long first_id = 0;  // chunk id of global chunk 0 of the plan
};

struct GenData {
  IndexData* ix = nullptr;
  cudaStream_t stream = 0;
  long long K = 0;
  DevBuf<u32> comp_order;  // component ranks in seeded order
  std::vector<u32> h_comp_order;
  DevBuf<u32> cur_blk;
  DevBuf<u32> civ;
  DevBuf<u32> cfile, cstart;  // iv_file / iv_start in cursor order (emission reads them sequentially)
  DevBuf<u64> ccum;
  DevBuf<u64> comp_total;
  std::vector<unsigned long long> h_comp_total;
  bool mirrors_valid = false;  // h_comp_order / h_comp_total filled (gen_host_mirrors)
  DevBuf<u64> consumed;
  // sharded index only: lcnt u32[I+1] local intervals before each cursor
  // position, lpos u32[#local] their positions, rcum u64[I+1] real intervals
  DevBuf<u32> lcnt, lpos;
  DevBuf<u64> rcum, lstart;  // lstart[r] = ccum[lpos[r]]
  DevBuf<uint8_t> chunk_prefix;
  int chunk_prefix_len = 0;
  long long next_chunk_id = 0;
  // last plan result
  long long res_chunks = 0, res_ranges = 0;
  DevBuf<long long> res_off;
  DevBuf<long long> res_id;
  DevBuf<u64> res_seed;
  DevBuf<u32> res_mkey, res_file, res_start, res_end;
  // canonical JSON of the last result (serialize.cu)
  DevBuf<uint8_t> json;
  DevBuf<long long> json_off;
  long long json_bytes = 0;
  std::vector<long long> report;
  int last_mkeys = 0;
  // mark / reset of the cursor state (look-ahead rewinds without host copies)
  DevBuf<u64> mark_consumed;
  long long mark_next_id = 0;
  // matching cache: the last mixture's allow bitsets -> per-key component lists
  std::vector<u32> match_allow;
  std::vector<int> match_base;
  int match_words = 0;
  bool match_shared = false;
  std::vector<u32> match_off;  // host copy of L_off
  DevBuf<u32> match_L_off, match_L;
  // grow-only scratch for per-call planning (small plans allocate nothing);
  // allocated in stream order on the stream that first writes it (`st`)
  template <typename T>
  cudaError_t scratch(int slot, long long n, T** out, cudaStream_t st) {
    // per-call temporaries: the requesting stream's workspace (ws_get), so a
    // new generator per job allocates nothing once the sizes are reached
    void* p = nullptr;  // keyed by the generator's stream: plans of generators sharing it are ordered
    cudaError_t e = ws_get(stream, WS_GEN + slot, sizeof(T) * (size_t)(n > 0 ? n : 1), &p, st, true);
    *out = reinterpret_cast<T*>(p);
    return e;
  }
  template <typename T>
  cudaError_t scratch(int slot, long long n, T** out) { return scratch(slot, n, out, stream); }
  // Auxiliary streams of this generator (created on its device by
  // cursor_build): the component-order shuffle, planning, chunk seeds. The
  // first plan after the cursor layout waits only for the component totals
  // (ev_tot), so matching and the count-level plan overlap the per-key
  // cursor shuffles; every later plan is ordered after all work on `stream`.
  cudaStream_t ostream = nullptr, pstream = nullptr, sstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_order = nullptr, ev_tot = nullptr, ev_ready = nullptr;
  cudaEvent_t ev_plan = nullptr, ev_seg = nullptr, ev_seed_fork = nullptr, ev_seed = nullptr;
  bool fresh_layout = false;  // no work on `stream` since cursor_build except the layout itself
  LocalSrc local;             // set: plans emit this rank's pieces of the global chunks (emit_local)
  Handoff handoff;
  int aux_dev = -1;
  cudaError_t aux_init() {  // streams shared per device, events pooled (capi.cu)
    if (ostream) return cudaSuccess;
    cudaError_t e = cudaGetDevice(&aux_dev);
    cudaStream_t st[3];
    if (e == cudaSuccess) e = aux_streams(aux_dev, st);
    if (e != cudaSuccess) return e;
    ostream = st[0];
    pstream = st[1];
    sstream = st[2];
    for (cudaEvent_t* x : {&ev_fork, &ev_order, &ev_tot, &ev_ready, &ev_plan, &ev_seg, &ev_seed_fork, &ev_seed})
      if (e == cudaSuccess) e = aux_event_take(aux_dev, x);
    return e;
  }
  // pinned host mirror of a small plan's result (one D2H per call)
  unsigned char* h_small = nullptr;
  long long h_small_bytes = 0;
  long long h_small_valid = 0;  // chunk count the mirror holds (0 = use device result)
  long long h_small_cap = 0, h_small_slots = 0;  // layout of the mirror
  ~GenData() {
    if (h_small) cudaFreeHost(h_small);
    for (cudaEvent_t x : {ev_fork, ev_order, ev_tot, ev_ready, ev_plan, ev_seg, ev_seed_fork, ev_seed})
      if (x) aux_event_give(aux_dev, x);
  }
};

int stage1_build(const mx_catalog_desc* d, cudaStream_t s, IndexData* out);
int cursor_build(IndexData* ix, const uint8_t* cursor_prefix, int prefix_len, unsigned long long order_seed,
                 cudaStream_t s, GenData* g);
int plan_mixture(GenData* g, const mx_mixture_desc* mix, long long max_chunks, long long* n_out);
int plan_arbitrary(GenData* g, long long chunk_size, long long max_chunks, long long* n_out);
int index_finalize(IndexData* ix, long long I, cudaStream_t s, bool defer = false);
int rows_build(const mx_rows_desc* d, cudaStream_t s, IndexData* out);
int index_block_table(const IndexData* ix, u32 file_base, uint4* out, cudaStream_t s);
int index_build_sharded(const IndexData* loc, const mx_shard_desc* d, cudaStream_t s, IndexData* out);
int gen_local_lists(GenData* g, cudaStream_t s);
int gen_host_mirrors(GenData* g);
int gen_block_offsets(GenData* g, u64* out, cudaStream_t s);
int gen_finish_owned(GenData* g, int world, long long chunk_lo, long long n_own, long long n_global,
                     const int32_t* counts, const uint4* pieces, long long n_pieces, cudaStream_t s);
int owner_index_build(const IndexData* src, const u32* rows, long long n, int n_files, const int32_t* file_ds,
                      const int64_t* file_ids, int dense_bits, cudaStream_t s, IndexData* out);
int excl_scan_ll(const u64* in, long long n, long long* out, cudaStream_t s);
int gen_result_json(GenData* g, const mx_json_desc* d, cudaStream_t s);
int chunks_merge(int W, long long C, long long cap, const long long* offs, const u32* mkey, const u32* file,
                 const u32* start, const u32* end, long long* out_off, u32* o_mkey, u32* o_file, u32* o_start,
                 u32* o_end, cudaStream_t s);

}  // namespace mx

struct mx_index {
  mx::IndexData d;
};
struct mx_gen {
  mx::GenData d;
};
