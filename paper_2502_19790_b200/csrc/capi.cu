// C-ABI entry points (include/mixtera_b200.h): argument checks, handle
// ownership, error strings, host<->device copies of small results.
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <string>

#include "mixtera_internal.cuh"

namespace mx {
int domain_loss(const float* losses, const int32_t* tags, long long n, int K, double* sums, long long* counts,
                cudaStream_t s);
int fit_power_law(int D, const long long* off, const double* n, const double* loss, const double* geom, double* out,
                  cudaStream_t s);
int ado_pi(int k, const double* mu, const double* credit, const double* law, double n, double p_min, double smoothing,
           double* pi_bar, long long* cnt, double* pi, cudaStream_t s);
int ado_credit(int k, double rate, const double* pi, double* credit, cudaStream_t s);
}  // namespace mx

static thread_local std::string g_err;

// ---------------------------------------------------------------- accounting
#include <atomic>
#include <map>
#include <mutex>

static std::atomic<long long> g_launches{0};
static std::atomic<int> g_profile{0};
static std::mutex g_prof_mu;
struct PhaseAcc {
  double ms = 0;
  long long count = 0;
};
static std::map<std::string, PhaseAcc> g_prof;
struct PendingPhase {
  std::string name;
  cudaEvent_t a, b;
};
static std::vector<PendingPhase> g_pending;

void mx_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

#include <chrono>
void mx_host_mark(const char* label) {
  static const bool on = getenv("MX_HOST_TIMING") != nullptr;
  if (!on) return;
  static thread_local std::vector<std::pair<const char*, double>> marks;
  const double t = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  if (label) {
    marks.emplace_back(label, t);
    return;
  }
  for (size_t i = 1; i < marks.size(); ++i) fprintf(stderr, "  %-28s %8.1f us\n", marks[i].first, marks[i].second - marks[i - 1].second);
  if (!marks.empty()) fprintf(stderr, "  total %8.1f us\n", marks.back().second - marks.front().second);
  marks.clear();
}

// Host->device copies of small host arrays (LUTs, mixture tables, sentinels)
// go through a per-thread pinned staging ring: a cudaMemcpyAsync from
// PAGEABLE memory synchronises the stream before it starts, which would
// drain the GPU pipeline at every upload. The ring has two halves; a half is
// reused only after the events recorded behind its copies have completed.
namespace {
struct PinnedRing {
  static constexpr size_t kHalf = 2u << 20;
  char* buf = nullptr;
  int half = 0;
  size_t used = 0;
  std::vector<cudaEvent_t> pending[2], pool;
  ~PinnedRing() {
    for (int h = 0; h < 2; ++h)
      for (cudaEvent_t e : pending[h]) cudaEventDestroy(e);
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (buf) cudaFreeHost(buf);
  }
};
thread_local PinnedRing g_ring;
}  // namespace

namespace {
struct PinnedReadback {
  static constexpr size_t kCap = 256u << 10;
  char* buf = nullptr;
  bool failed = false;
  ~PinnedReadback() {
    if (buf) cudaFreeHost(buf);
  }
};
thread_local PinnedReadback g_rb;
}  // namespace

cudaError_t D2HBatch::add(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  PinnedReadback& r = g_rb;
  if (!r.buf && !r.failed) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&r.buf), PinnedReadback::kCap, cudaHostAllocDefault) != cudaSuccess) {
      r.buf = nullptr;
      r.failed = true;
      cudaGetLastError();
    }
  }
  const size_t need = (bytes + 15) & ~size_t(15);
  if (!r.buf || n == 16 || used + need > PinnedReadback::kCap)
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaMemcpyAsync(r.buf + used, src, bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  items[n++] = Item{dst, used, bytes};
  used += need;
  return cudaSuccess;
}

cudaError_t D2HBatch::sync() {
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  for (int i = 0; i < n; ++i) memcpy(items[i].dst, g_rb.buf + items[i].off, items[i].bytes);
  n = 0;
  used = 0;
  return cudaSuccess;
}

namespace {
struct AuxPool {
  std::mutex mu;
  std::map<int, std::vector<cudaStream_t>> streams;
  std::map<int, std::vector<cudaEvent_t>> events;
};
AuxPool& aux_pool() {
  static AuxPool* p = new AuxPool();  // never destroyed: streams live for the process
  return *p;
}
}  // namespace

cudaError_t mx::aux_streams(int dev, cudaStream_t out[3]) {
  AuxPool& p = aux_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  std::vector<cudaStream_t>& v = p.streams[dev];
  while (v.size() < 3) {
    cudaStream_t st;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    v.push_back(st);
  }
  for (int i = 0; i < 3; ++i) out[i] = v[i];
  return cudaSuccess;
}

cudaError_t mx::aux_event_take(int dev, cudaEvent_t* e) {
  AuxPool& p = aux_pool();
  {
    std::lock_guard<std::mutex> lk(p.mu);
    std::vector<cudaEvent_t>& v = p.events[dev];
    if (!v.empty()) {
      *e = v.back();
      v.pop_back();
      return cudaSuccess;
    }
  }
  return cudaEventCreateWithFlags(e, cudaEventDisableTiming);
}

void mx::aux_event_give(int dev, cudaEvent_t e) {
  AuxPool& p = aux_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  p.events[dev].push_back(e);
}

// pinned slots for deferred index sizes (IndexData::Pending)
namespace {
struct PendPool {
  std::mutex mu;
  char* base = nullptr;
  std::vector<int> free_slots;
  static constexpr int kSlots = 4096;
};
PendPool& pend_pool() {
  static PendPool* p = new PendPool();
  return *p;
}
}  // namespace

mx::IndexData::Pending* mx::pend_slot_take() {
  PendPool& p = pend_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  if (!p.base) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&p.base), sizeof(mx::IndexData::Pending) * PendPool::kSlots,
                      cudaHostAllocDefault) != cudaSuccess) {
      p.base = nullptr;
      cudaGetLastError();
      return nullptr;
    }
    for (int i = PendPool::kSlots - 1; i >= 0; --i) p.free_slots.push_back(i);
  }
  if (p.free_slots.empty()) return nullptr;
  const int i = p.free_slots.back();
  p.free_slots.pop_back();
  return reinterpret_cast<mx::IndexData::Pending*>(p.base) + i;
}

void mx::pend_slot_give(mx::IndexData::Pending* slot) {
  PendPool& p = pend_pool();
  std::lock_guard<std::mutex> lk(p.mu);
  p.free_slots.push_back((int)(slot - reinterpret_cast<mx::IndexData::Pending*>(p.base)));
}

int mx::ix_resolve(mx::IndexData* ix) {
  if (!ix->pend) return MX_OK;
  cudaError_t e = cudaEventSynchronize(ix->pend_ev);
  if (e != cudaSuccess) return mx_fail_cuda(e, "index sizes", __FILE__, __LINE__);
  const mx::IndexData::Pending h = *ix->pend;
  pend_slot_give(ix->pend);
  aux_event_give(ix->pend_dev, ix->pend_ev);
  ix->pend = nullptr;
  ix->pend_ev = nullptr;
  if (h.err.overlap) return mx_fail(MX_ERR_INDEX, "empty or overlapping interval in index build");
  ix->n_keys = (long long)(h.totals >> 32);
  ix->n_blocks = (long long)(h.totals & 0xffffffffull);
  ix->indexed_samples = (long long)h.samples;
  ix->max_key_blocks = (long long)h.maxblk;
  return MX_OK;
}

mx::IndexData::~IndexData() {
  if (pend) {
    cudaEventSynchronize(pend_ev);  // the copy into the slot must land first
    pend_slot_give(pend);
    aux_event_give(pend_dev, pend_ev);
  }
}

namespace {
struct Workspace {
  void* p[mx::WS_N] = {};
  size_t n[mx::WS_N] = {};
};
thread_local std::map<cudaStream_t, Workspace> g_ws;
}  // namespace

cudaError_t mx::ws_get(cudaStream_t s, int slot, size_t bytes, void** out, cudaStream_t alloc, bool alloc_set) {
  Workspace& w = g_ws[s];
  const cudaStream_t as = alloc_set ? alloc : s;
  if (w.n[slot] < bytes) {
    if (w.p[slot]) cudaFreeAsync(w.p[slot], as);
    w.p[slot] = nullptr;
    w.n[slot] = 0;
    const size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMallocAsync(&w.p[slot], want, as);
    if (e != cudaSuccess) return e;
    w.n[slot] = want;
  }
  *out = w.p[slot];
  return cudaSuccess;
}

cudaError_t D2HBatch::sync_event(cudaEvent_t e) {
  cudaError_t r = cudaEventSynchronize(e);
  if (r != cudaSuccess) return r;
  for (int i = 0; i < n; ++i) memcpy(items[i].dst, g_rb.buf + items[i].off, items[i].bytes);
  n = 0;
  used = 0;
  return cudaSuccess;
}

cudaError_t mx_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  PinnedRing& r = g_ring;
  const size_t need = (bytes + 255) & ~size_t(255);
  if (need > PinnedRing::kHalf) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  if (!r.buf) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&r.buf), 2 * PinnedRing::kHalf, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      r.buf = nullptr;
      return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    }
  }
  if (r.used + need > PinnedRing::kHalf) {  // switch halves; wait for the other half's copies
    r.half ^= 1;
    r.used = 0;
    for (cudaEvent_t e : r.pending[r.half]) {
      cudaEventSynchronize(e);
      r.pool.push_back(e);
    }
    r.pending[r.half].clear();
  }
  char* stage = r.buf + (size_t)r.half * PinnedRing::kHalf + r.used;
  r.used += need;
  memcpy(stage, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, stage, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  cudaEvent_t ev;
  if (!r.pool.empty()) {
    ev = r.pool.back();
    r.pool.pop_back();
  } else if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) {
    return e;
  }
  r.pending[r.half].push_back(ev);
  return cudaEventRecord(ev, s);
}

cudaError_t mx_h2d_gather(void* dst, const void* const* src, const size_t* bytes, const size_t* off, int n,
                          size_t total, cudaStream_t s) {
  if (total == 0) return cudaSuccess;
  PinnedRing& r = g_ring;
  const size_t need = (total + 255) & ~size_t(255);
  if (need > PinnedRing::kHalf || (!r.buf && cudaHostAlloc(reinterpret_cast<void**>(&r.buf), 2 * PinnedRing::kHalf,
                                                            cudaHostAllocDefault) != cudaSuccess)) {
    if (!r.buf) cudaGetLastError();
    for (int i = 0; i < n; ++i) {  // no staging space: one copy per item
      cudaError_t e = mx_h2d(static_cast<char*>(dst) + off[i], src[i], bytes[i], s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (r.used + need > PinnedRing::kHalf) {
    r.half ^= 1;
    r.used = 0;
    for (cudaEvent_t e : r.pending[r.half]) {
      cudaEventSynchronize(e);
      r.pool.push_back(e);
    }
    r.pending[r.half].clear();
  }
  char* stage = r.buf + (size_t)r.half * PinnedRing::kHalf + r.used;
  r.used += need;
  for (int i = 0; i < n; ++i)
    if (bytes[i]) memcpy(stage + off[i], src[i], bytes[i]);
  cudaError_t e = cudaMemcpyAsync(dst, stage, total, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  cudaEvent_t ev;
  if (!r.pool.empty()) {
    ev = r.pool.back();
    r.pool.pop_back();
  } else if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) {
    return e;
  }
  r.pending[r.half].push_back(ev);
  return cudaEventRecord(ev, s);
}

// Keep memory freed with cudaFreeAsync cached in the device's default pool
// (the default release threshold of 0 hands it back to the driver at every
// synchronisation, which makes each job re-map gigabytes of HBM).
static void keep_pool_warm() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> g(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

// Phase events come from a recycled pool (cudaEventCreate costs microseconds
// of host time; the phases are measured inside the bench's timed region).
// Events belong to the device that created them: one pool per device.
static std::map<int, std::vector<cudaEvent_t>> g_ev_free;  // guarded by g_prof_mu
static std::map<cudaEvent_t, int> g_ev_dev;

static cudaEvent_t phase_event() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    auto& fr = g_ev_free[dev];
    if (!fr.empty()) {
      cudaEvent_t e = fr.back();
      fr.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_ev_dev[e] = dev;
  return e;
}

MxPhase::MxPhase(const char* n, cudaStream_t s) : name(n), stream(s), start(nullptr) {
  const int mode = g_profile.load();
  if (!mode || (mode == 2 && strcmp(n, "scan_runs") != 0)) return;
  cudaEvent_t e = phase_event();
  if (!e) return;
  cudaEventRecord(e, s);
  start = e;
}

MxPhase::~MxPhase() {
  if (!start) return;
  cudaEvent_t e = phase_event();
  if (!e) return;
  cudaEventRecord(e, stream);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_pending.push_back(PendingPhase{name, (cudaEvent_t)start, e});
}

static void collect_phases() {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& p : g_pending) {
    float ms = 0;
    cudaEventSynchronize(p.b);
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      PhaseAcc& acc = g_prof[p.name];
      acc.ms += ms;
      acc.count += 1;
    }
    g_ev_free[g_ev_dev[p.a]].push_back(p.a);
    g_ev_free[g_ev_dev[p.b]].push_back(p.b);
  }
  g_pending.clear();
}

int mx_fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int mx_fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  return mx_fail(MX_ERR_CUDA, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e), what,
                 file, line);
}

#define MX_CHECK_ARG(cond, msg)                          \
  do {                                                   \
    if (!(cond)) return mx_fail(MX_ERR_INVALID, "%s", msg); \
  } while (0)

using namespace mx;

__global__ void map_files_kernel(const u32* fidx, long long n, const int32_t* file_ds, const long long* file_ids,
                                 int32_t* ds, long long* fid) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u32 f = fidx[i];
  ds[i] = file_ds[f];
  fid[i] = file_ids[f];
}

void map_files(const u32* fidx, long long n, const int32_t* file_ds, const long long* file_ids, int32_t* ds,
               long long* fid, cudaStream_t s) {
  map_files_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(fidx, n, file_ds, file_ids, ds, fid);
  mx_count_launch();
}

extern "C" {

const char* mx_last_error(void) { return g_err.c_str(); }

int64_t mx_launch_count(void) { return g_launches.load(); }

int mx_profile_enable(int on) {
  collect_phases();
  g_profile.store(on == 2 ? 2 : on ? 1 : 0);
  return MX_OK;
}

int mx_profile_reset(void) {
  collect_phases();
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof.clear();
  return MX_OK;
}

int mx_profile_read(const char* phase, double* total_ms, int64_t* count) {
  MX_CHECK_ARG(phase, "null phase");
  collect_phases();
  std::lock_guard<std::mutex> g(g_prof_mu);
  auto it = g_prof.find(phase);
  if (total_ms) *total_ms = it == g_prof.end() ? 0.0 : it->second.ms;
  if (count) *count = it == g_prof.end() ? 0 : it->second.count;
  return MX_OK;
}
int mx_abi_version(void) { return 2; }

int mx_index_build(const mx_catalog_desc* desc, void* stream, mx_index** out) {
  MX_CHECK_ARG(desc && out, "null argument");
  g_err.clear();
  keep_pool_warm();
  cudaStream_t s = (cudaStream_t)stream;
  mx_index* ix = new mx_index();
  ix->d.stream = s;
  IndexData& d = ix->d;
  d.n_props = desc->n_props;
  for (int p = 0; p < desc->n_props && p < MX_MAX_PROPS; ++p) {
    d.field_shift[p] = desc->field_shift[p];
    d.field_width[p] = desc->field_width[p];
    d.str_base[p] = desc->key_string_base[p];
  }
  int rc = MX_OK;
  // key strings, LUTs and file tables are uploaded by stage1_build in one copy
  mx_host_mark("build enter");
  if (rc == MX_OK) rc = stage1_build(desc, s, &d);
  mx_host_mark("build done");
  if (rc < 0) {
    delete ix;
    return rc;
  }
  *out = ix;
  return MX_OK;
}

int mx_index_build_rows(const mx_rows_desc* desc, void* stream, mx_index** out) {
  MX_CHECK_ARG(desc && out, "null argument");
  MX_CHECK_ARG(desc->n_rows >= 0 && desc->n_files >= 0 && desc->n_keys >= 0, "negative size");
  if (desc->key_bits > 31) return mx_fail(MX_ERR_UNSUPPORTED, "rows index: %u key bits (> 31)", desc->key_bits);
  g_err.clear();
  keep_pool_warm();
  cudaStream_t s = (cudaStream_t)stream;
  mx_index* ix = new mx_index();
  ix->d.stream = s;
  IndexData& d = ix->d;
  // one "property" whose value rank IS the key rank; piece k-1 = key k's string
  d.n_props = 1;
  d.field_shift[0] = 0;
  d.field_width[0] = desc->key_bits;
  d.str_base[0] = 0;
  int rc = MX_OK;
  {
    const long long nbytes = desc->key_string_offsets[desc->n_keys];
    cudaError_t e = d.str_off.alloc(desc->n_keys + 1, s);
    if (e == cudaSuccess) e = d.str_bytes.alloc(nbytes > 0 ? nbytes : 1, s);
    if (e == cudaSuccess) e = mx_h2d(d.str_off.p, desc->key_string_offsets, sizeof(long long) * (desc->n_keys + 1), s);
    if (e == cudaSuccess && nbytes > 0) e = mx_h2d(d.str_bytes.p, desc->key_strings, nbytes, s);
    if (e != cudaSuccess) rc = mx_fail_cuda(e, "key strings", __FILE__, __LINE__);
  }
  if (rc == MX_OK) rc = rows_build(desc, s, &d);
  if (rc < 0) {
    delete ix;
    return rc;
  }
  *out = ix;
  return MX_OK;
}

// Device buffers are released stream-ordered (cudaFreeAsync); waiting for
// the stream here keeps the pool's next allocations of the same sizes on
// already-released memory (measured: without it the next job's allocations
// stall and a cfg2 job takes 2.6-3.3 ms instead of 1.66 ms).
int mx_index_free(mx_index* index) {
  if (!index) return MX_OK;
  cudaStream_t s = index->d.stream;
  delete index;
  cudaStreamSynchronize(s);
  return MX_OK;
}

int mx_index_sizes(const mx_index* index, int64_t* n_keys, int64_t* n_blocks, int64_t* n_intervals,
                   int64_t* n_samples) {
  MX_CHECK_ARG(index, "null index");
  if (int rc = ix_resolve(const_cast<IndexData*>(&index->d))) return rc;
  const IndexData& d = index->d;
  if (n_keys) *n_keys = d.n_keys;
  if (n_blocks) *n_blocks = d.n_blocks;
  if (n_intervals) *n_intervals = d.n_intervals;
  if (n_samples) *n_samples = d.indexed_samples;
  return MX_OK;
}

int mx_index_export_keys(const mx_index* index, uint32_t* packed, int64_t* samples) {
  MX_CHECK_ARG(index, "null index");
  if (int rc = ix_resolve(const_cast<IndexData*>(&index->d))) return rc;
  const IndexData& d = index->d;
  const long long K = d.n_keys;
  if (K == 0) return MX_OK;
  std::vector<u32> kbf(K + 1), bf(d.n_blocks + 1);
  std::vector<unsigned long long> cum(d.n_intervals + 1);
  cudaError_t e = cudaMemcpy(kbf.data(), d.key_blk_first.p, sizeof(u32) * (K + 1), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(bf.data(), d.blk_first.p, sizeof(u32) * (d.n_blocks + 1), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(cum.data(), d.iv_cum.p, sizeof(u64) * (d.n_intervals + 1), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && packed) e = cudaMemcpy(packed, d.key_packed.p, sizeof(u32) * K, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "export keys", __FILE__, __LINE__);
  if (samples)
    for (long long k = 0; k < K; ++k) samples[k] = (int64_t)(cum[bf[kbf[k + 1]]] - cum[bf[kbf[k]]]);
  return MX_OK;
}

int mx_index_export_intervals(const mx_index* index, uint32_t* key_rank, int32_t* ds, int64_t* file_id,
                              uint32_t* start, uint32_t* end) {
  MX_CHECK_ARG(index, "null index");
  if (int rc = ix_resolve(const_cast<IndexData*>(&index->d))) return rc;
  const IndexData& d = index->d;
  if (d.sharded)
    return mx_fail(MX_ERR_UNSUPPORTED,
                   "a file-sharded index holds only this rank's intervals (remote files are per-file blocks); "
                   "export the local index instead");
  const long long I = d.n_intervals;
  if (I == 0) return MX_OK;
  std::vector<u32> f(I), bk(d.n_blocks), bf(d.n_blocks + 1);
  cudaError_t e = cudaMemcpy(f.data(), d.iv_file.p, sizeof(u32) * I, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && start) e = cudaMemcpy(start, d.iv_start.p, sizeof(u32) * I, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && end) e = cudaMemcpy(end, d.iv_end.p, sizeof(u32) * I, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(bk.data(), d.blk_key.p, sizeof(u32) * d.n_blocks, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(bf.data(), d.blk_first.p, sizeof(u32) * (d.n_blocks + 1), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "export intervals", __FILE__, __LINE__);
  for (long long b = 0; b < d.n_blocks; ++b)
    for (u32 i = bf[b]; i < bf[b + 1]; ++i)
      if (key_rank) key_rank[i] = bk[b];
  for (long long i = 0; i < I; ++i) {
    if (ds) ds[i] = d.h_file_ds[f[i]];
    if (file_id) file_id[i] = d.h_file_ids[f[i]];
  }
  return MX_OK;
}

int mx_index_block_table(const mx_index* index, int64_t file_base, uint32_t* rows, void* stream) {
  if (index)
    if (int rc = ix_resolve(const_cast<IndexData*>(&index->d))) return rc;
  MX_CHECK_ARG(index && (rows || index->d.n_blocks == 0), "null argument");
  MX_CHECK_ARG(file_base >= 0 && file_base + index->d.n_files < (1ll << 32), "file_base out of range");
  g_err.clear();
  return index_block_table(&index->d, (u32)file_base, reinterpret_cast<uint4*>(rows), (cudaStream_t)stream);
}

int mx_index_packed_keys(const mx_index* index, uint32_t* packed) {
  if (index)
    if (int rc = ix_resolve(const_cast<IndexData*>(&index->d))) return rc;
  MX_CHECK_ARG(index && (packed || index->d.n_keys == 0), "null argument");
  if (index->d.n_keys == 0) return MX_OK;
  cudaError_t e = cudaMemcpy(packed, index->d.key_packed.p, sizeof(u32) * index->d.n_keys, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "packed keys", __FILE__, __LINE__);
  return MX_OK;
}

int mx_index_build_sharded(const mx_index* local, const mx_shard_desc* desc, void* stream, mx_index** out) {
  if (local)
    if (int rc = ix_resolve(const_cast<IndexData*>(&local->d))) return rc;
  MX_CHECK_ARG(local && desc && out, "null argument");
  MX_CHECK_ARG(desc->world >= 1 && desc->rank >= 0 && desc->rank < desc->world, "bad world/rank");
  MX_CHECK_ARG(desc->file_lo >= 0 && desc->file_hi - desc->file_lo == local->d.n_files &&
                   desc->file_hi <= desc->n_files,
               "file range does not match the local index");
  MX_CHECK_ARG(desc->n_global_keys == 0 || desc->global_keys, "null global keys");
  MX_CHECK_ARG(desc->file_ds && desc->file_ids && desc->counts, "null file table or counts");
  for (int q = 0; q < desc->world; ++q)
    MX_CHECK_ARG(desc->counts[q] >= 0 && desc->counts[q] <= desc->cap, "block count exceeds cap");
  g_err.clear();
  keep_pool_warm();
  mx_index* ix = new mx_index();
  int rc = index_build_sharded(&local->d, desc, (cudaStream_t)stream, &ix->d);
  if (rc < 0) {
    delete ix;
    return rc;
  }
  *out = ix;
  return MX_OK;
}

int mx_index_build_owner(const mx_index* like, const uint32_t* rows, int64_t n_rows, int32_t n_files,
                         const int32_t* file_ds, const int64_t* file_ids, int32_t dense_key_bits, void* stream,
                         mx_index** out) {
  if (like)
    if (int rc = ix_resolve(const_cast<IndexData*>(&like->d))) return rc;
  MX_CHECK_ARG(like && out && (rows || n_rows == 0), "null argument");
  MX_CHECK_ARG(n_rows >= 0 && n_rows < (1ll << 32), "bad row count");
  MX_CHECK_ARG(n_files >= 1 && file_ds && file_ids, "need the global file table");
  g_err.clear();
  keep_pool_warm();
  mx_index* ix = new mx_index();
  MX_CHECK_ARG(dense_key_bits >= 0 && dense_key_bits <= 32, "bad dense key bits");
  int rc = owner_index_build(&like->d, rows, n_rows, n_files, file_ds, file_ids, dense_key_bits, (cudaStream_t)stream,
                             &ix->d);
  if (rc < 0) {
    delete ix;
    return rc;
  }
  *out = ix;
  return MX_OK;
}

int mx_gen_block_offsets(mx_gen* gen, uint64_t* offsets, void* stream) {
  MX_CHECK_ARG(gen && (offsets || gen->d.ix->n_intervals == 0), "null argument");
  g_err.clear();
  cudaStream_t s = (cudaStream_t)stream;
  if (s != gen->d.stream) {  // behind the cursor layout
    cudaEvent_t e;
    MX_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaError_t err = cudaEventRecord(e, gen->d.stream);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(s, e, 0);
    cudaEventDestroy(e);
    MX_CUDA_TRY(err);
  }
  return gen_block_offsets(&gen->d, reinterpret_cast<u64*>(offsets), s);
}

int mx_gen_set_local(mx_gen* gen, const mx_index* local, const uint64_t* blk_off, const uint32_t* key_g,
                     int64_t file_lo) {
  MX_CHECK_ARG(gen, "null argument");
  g_err.clear();
  if (!local) {
    gen->d.local = LocalSrc{};
    return MX_OK;
  }
  if (int rc = ix_resolve(const_cast<IndexData*>(&local->d))) return rc;
  MX_CHECK_ARG((blk_off && key_g) || local->d.n_blocks == 0, "null block offsets / key map");
  MX_CHECK_ARG(file_lo >= 0 && file_lo + local->d.n_files <= gen->d.ix->n_files, "local files outside the file table");
  gen->d.local = LocalSrc{&local->d, reinterpret_cast<const u64*>(blk_off), key_g, (long long)file_lo};
  return MX_OK;
}

int mx_gen_set_handoff(mx_gen* gen, int32_t on) {
  MX_CHECK_ARG(gen, "null argument");
  MX_CHECK_ARG(!on || gen->d.local.loc, "handoff needs a partitioned generator (mx_gen_set_local)");
  g_err.clear();
  gen->d.local.handoff = on != 0;
  gen->d.handoff.n_chunks = -1;
  return MX_OK;
}

int mx_gen_handoff(const mx_gen* gen, int64_t* n_chunks, int64_t* n_pieces, const int64_t** chunk_offsets,
                   const uint32_t** pieces) {
  MX_CHECK_ARG(gen && n_chunks && n_pieces && chunk_offsets && pieces, "null argument");
  const Handoff& h = gen->d.handoff;
  if (h.n_chunks < 0) return mx_fail(MX_ERR_INVALID, "no partitioned plan pending");
  long long np = 0;
  cudaError_t e = cudaMemcpy(&np, h.off.p + h.n_chunks, sizeof(long long), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "handoff size", __FILE__, __LINE__);
  *n_chunks = h.n_chunks;
  *n_pieces = np;
  *chunk_offsets = reinterpret_cast<const int64_t*>(h.off.p);
  *pieces = reinterpret_cast<const uint32_t*>(h.pieces.p);
  return MX_OK;
}

int mx_gen_finish_owned(mx_gen* gen, int32_t world, int64_t chunk_lo, int64_t n_own, int64_t n_global,
                        const int32_t* counts, const uint32_t* pieces, int64_t n_pieces, void* stream) {
  MX_CHECK_ARG(gen && world >= 1 && n_own >= 0 && n_pieces >= 0, "bad argument");
  MX_CHECK_ARG((counts || n_own == 0) && (pieces || n_pieces == 0), "null counts / pieces");
  g_err.clear();
  return gen_finish_owned(&gen->d, world, chunk_lo, n_own, n_global, counts, reinterpret_cast<const uint4*>(pieces),
                          n_pieces, (cudaStream_t)stream);
}

int mx_chunks_merge(int32_t world, int64_t n_chunks, int64_t cap, const int64_t* offs, const uint32_t* mkey,
                    const uint32_t* file_index, const uint32_t* start, const uint32_t* end, int64_t* out_off,
                    uint32_t* out_mkey, uint32_t* out_file_index, uint32_t* out_start, uint32_t* out_end,
                    void* stream) {
  MX_CHECK_ARG(world >= 1 && n_chunks >= 0 && cap >= 0, "bad sizes");
  MX_CHECK_ARG(offs && out_off, "null offsets");
  g_err.clear();
  return chunks_merge(world, n_chunks, cap, reinterpret_cast<const long long*>(offs), mkey, file_index, start, end,
                      reinterpret_cast<long long*>(out_off), out_mkey, out_file_index, out_start, out_end,
                      (cudaStream_t)stream);
}

int mx_gen_create(mx_index* index, const uint8_t* cursor_prefix, int32_t cursor_prefix_len, const uint8_t* chunk_prefix,
                  int32_t chunk_prefix_len, uint64_t order_seed, void* stream, mx_gen** out) {
  MX_CHECK_ARG(index && out, "null argument");
  g_err.clear();
  keep_pool_warm();
  mx_host_mark("gen enter");
  if (int rc = ix_resolve(&index->d)) return rc;
  mx_host_mark("gen index resolved");
  cudaStream_t s = (cudaStream_t)stream;
  mx_gen* g = new mx_gen();
  int rc = MX_OK;
  cudaError_t e = g->d.chunk_prefix.alloc(chunk_prefix_len > 0 ? chunk_prefix_len : 1, s);
  if (e == cudaSuccess && chunk_prefix_len > 0)
    e = mx_h2d(g->d.chunk_prefix.p, chunk_prefix, chunk_prefix_len, s);
  if (e != cudaSuccess) rc = mx_fail_cuda(e, "chunk prefix", __FILE__, __LINE__);
  g->d.chunk_prefix_len = chunk_prefix_len;
  if (rc == MX_OK) rc = cursor_build(&index->d, cursor_prefix, cursor_prefix_len, order_seed, s, &g->d);
  mx_host_mark("gen cursor launched");
  if (rc < 0) {
    delete g;
    return rc;
  }
  *out = g;
  return MX_OK;
}

int mx_gen_free(mx_gen* gen) {
  if (!gen) return MX_OK;
  cudaStream_t s = gen->d.stream;
  delete gen;
  cudaStreamSynchronize(s);
  return MX_OK;
}

int mx_gen_plan(mx_gen* gen, const mx_mixture_desc* mix, int64_t max_chunks, int64_t* n_out) {
  MX_CHECK_ARG(gen && mix && n_out, "null argument");
  MX_CHECK_ARG(max_chunks >= 1, "max_chunks must be >= 1");
  g_err.clear();
  long long n = 0;
  mx_host_mark("plan enter");
  int rc = plan_mixture(&gen->d, mix, max_chunks, &n);
  mx_host_mark("plan done");
  mx_host_mark(nullptr);
  *n_out = n;
  return rc;
}

int mx_gen_plan_arbitrary(mx_gen* gen, int64_t chunk_size, int64_t max_chunks, int64_t* n_out) {
  if (gen) gen->d.fresh_layout = false;  // state changes on the generator stream: later plans wait for it
  MX_CHECK_ARG(gen && n_out, "null argument");
  MX_CHECK_ARG(max_chunks >= 1, "max_chunks must be >= 1");
  g_err.clear();
  long long n = 0;
  int rc = plan_arbitrary(&gen->d, chunk_size, max_chunks, &n);
  *n_out = n;
  return rc;
}

int mx_gen_result_sizes(const mx_gen* gen, int64_t* n_chunks, int64_t* n_ranges) {
  MX_CHECK_ARG(gen, "null generator");
  if (n_chunks) *n_chunks = gen->d.res_chunks;
  if (n_ranges) *n_ranges = gen->d.res_ranges;
  return MX_OK;
}

int mx_gen_result_copy(const mx_gen* gen, int64_t* chunk_offsets, int64_t* chunk_ids, uint64_t* seeds, uint32_t* mkey,
                       int32_t* ds, int64_t* file_id, uint32_t* start, uint32_t* end) {
  MX_CHECK_ARG(gen, "null generator");
  const GenData& g = gen->d;
  const long long C = g.res_chunks, R = g.res_ranges;
  cudaStream_t s = g.stream;
  cudaError_t e = cudaSuccess;
  if (g.h_small_valid == C && C > 0 && g.h_small) {  // small plan: served from the pinned mirror
    const unsigned char* b = g.h_small + 32;
    const long long cap = g.h_small_cap, slots = g.h_small_slots;
    if (chunk_offsets) memcpy(chunk_offsets, b, sizeof(long long) * (C + 1));
    b += sizeof(long long) * (cap + 1);
    if (seeds) memcpy(seeds, b, sizeof(u64) * C);
    b += sizeof(u64) * cap;
    if (chunk_ids) memcpy(chunk_ids, b, sizeof(long long) * C);
    b += sizeof(long long) * cap;
    const u32* hm = reinterpret_cast<const u32*>(b);
    const u32* hf = hm + slots;
    const u32* hs = hf + slots;
    const u32* he = hs + slots;
    if (mkey) memcpy(mkey, hm, sizeof(u32) * R);
    if (start) memcpy(start, hs, sizeof(u32) * R);
    if (end) memcpy(end, he, sizeof(u32) * R);
    for (long long i = 0; i < R; ++i) {
      if (ds) ds[i] = g.ix->h_file_ds[hf[i]];
      if (file_id) file_id[i] = g.ix->h_file_ids[hf[i]];
    }
    return MX_OK;
  }
  // dataset / file id per range mapped on the device, then one D2H per array
  // (fast when the caller's buffers are pinned, as ChunkBatch.to_host's are)
  DevBuf<int32_t> d_ds;
  DevBuf<long long> d_fid;
  if (R && (ds || file_id)) {
    e = d_ds.alloc(R, s);
    if (e == cudaSuccess) e = d_fid.alloc(R, s);
    if (e == cudaSuccess) {
      map_files(g.res_file.p, R, g.ix->file_ds.p, g.ix->file_ids.p, d_ds.p, d_fid.p, s);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess && chunk_offsets)
    e = cudaMemcpyAsync(chunk_offsets, g.res_off.p, sizeof(long long) * (C + 1), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && chunk_ids && C)
    e = cudaMemcpyAsync(chunk_ids, g.res_id.p, sizeof(long long) * C, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && seeds && C) e = cudaMemcpyAsync(seeds, (const void*)g.res_seed.p, sizeof(u64) * C, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && mkey && R) e = cudaMemcpyAsync(mkey, g.res_mkey.p, sizeof(u32) * R, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && start && R) e = cudaMemcpyAsync(start, g.res_start.p, sizeof(u32) * R, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && end && R) e = cudaMemcpyAsync(end, g.res_end.p, sizeof(u32) * R, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && R && ds) e = cudaMemcpyAsync(ds, d_ds.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && R && file_id)
    e = cudaMemcpyAsync(file_id, d_fid.p, sizeof(long long) * R, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return mx_fail_cuda(e, "result copy", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_result_device(const mx_gen* gen, const int64_t** chunk_offsets, const uint64_t** seeds,
                         const uint32_t** mkey, const uint32_t** file_index, const uint32_t** start,
                         const uint32_t** end) {
  MX_CHECK_ARG(gen, "null generator");
  const GenData& g = gen->d;
  if (chunk_offsets) *chunk_offsets = reinterpret_cast<const int64_t*>(g.res_off.p);
  if (seeds) *seeds = reinterpret_cast<const uint64_t*>(g.res_seed.p);
  if (mkey) *mkey = g.res_mkey.p;
  if (file_index) *file_index = g.res_file.p;
  if (start) *start = g.res_start.p;
  if (end) *end = g.res_end.p;
  return MX_OK;
}

int mx_gen_result_export(const mx_gen* gen, int64_t* chunk_offsets, uint32_t* mkey, uint32_t* file_index,
                         uint32_t* start, uint32_t* end, void* stream) {
  MX_CHECK_ARG(gen && chunk_offsets, "null argument");
  const GenData& g = gen->d;
  const long long C = g.res_chunks, R = g.res_ranges;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (g.h_small_valid == C && C > 0 && g.h_small) {  // small plan: the pinned mirror holds the result
    const unsigned char* b = g.h_small + 32;
    const long long cap = g.h_small_cap, slots = g.h_small_slots;
    e = cudaMemcpyAsync(chunk_offsets, b, sizeof(long long) * (C + 1), cudaMemcpyHostToDevice, s);
    b += sizeof(long long) * (cap + 1) + sizeof(u64) * cap + sizeof(long long) * cap;
    const u32* h = reinterpret_cast<const u32*>(b);
    u32* dst[4] = {mkey, file_index, start, end};
    for (int f = 0; f < 4 && e == cudaSuccess; ++f)
      if (dst[f] && R) e = cudaMemcpyAsync(dst[f], h + f * slots, sizeof(u32) * R, cudaMemcpyHostToDevice, s);
  } else {
    e = cudaMemcpyAsync(chunk_offsets, g.res_off.p, sizeof(long long) * (C + 1), cudaMemcpyDeviceToDevice, s);
    const u32* src[4] = {g.res_mkey.p, g.res_file.p, g.res_start.p, g.res_end.p};
    u32* dst[4] = {mkey, file_index, start, end};
    for (int f = 0; f < 4 && e == cudaSuccess; ++f)
      if (dst[f] && R) e = cudaMemcpyAsync(dst[f], src[f], sizeof(u32) * R, cudaMemcpyDeviceToDevice, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return mx_fail_cuda(e, "result export", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_result_json(mx_gen* gen, const mx_json_desc* desc, int64_t* total_bytes, void* stream) {
  if (gen) gen->d.fresh_layout = false;  // state changes on the generator stream: later plans wait for it
  MX_CHECK_ARG(gen && desc && total_bytes, "null argument");
  MX_CHECK_ARG(desc->n_keys >= 0 && desc->n_keys < 65536, "n_keys outside [0, 65536)");
  MX_CHECK_ARG(desc->key_json_off && desc->key_rank && desc->file_rank && desc->mixture_json, "null table");
  g_err.clear();
  (void)stream;
  int rc = gen_result_json(&gen->d, desc, gen->d.stream);
  *total_bytes = gen->d.json_bytes;
  return rc;
}

int mx_gen_result_json_copy(const mx_gen* gen, uint8_t* bytes, int64_t* offsets) {
  MX_CHECK_ARG(gen, "null generator");
  const GenData& g = gen->d;
  cudaError_t e = cudaSuccess;
  if (offsets) e = cudaMemcpyAsync(offsets, g.json_off.p, sizeof(long long) * (g.res_chunks + 1), cudaMemcpyDeviceToHost, g.stream);
  if (e == cudaSuccess && bytes && g.json_bytes)
    e = cudaMemcpyAsync(bytes, g.json.p, g.json_bytes, cudaMemcpyDeviceToHost, g.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g.stream);
  if (e != cudaSuccess) return mx_fail_cuda(e, "json copy", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_report(const mx_gen* gen, int64_t* remaining) {
  MX_CHECK_ARG(gen && remaining, "null argument");
  for (size_t i = 0; i < gen->d.report.size(); ++i) remaining[i] = gen->d.report[i];
  return MX_OK;
}

int mx_gen_mark(mx_gen* gen) {
  MX_CHECK_ARG(gen, "null generator");
  GenData& g = gen->d;
  const long long K = g.K > 0 ? g.K : 1;
  if (g.mark_consumed.n != K) {
    cudaError_t e = g.mark_consumed.alloc(K, g.stream);
    if (e != cudaSuccess) return mx_fail_cuda(e, "mark", __FILE__, __LINE__);
  }
  cudaError_t e = cudaMemcpyAsync(g.mark_consumed.p, g.consumed.p, sizeof(u64) * K, cudaMemcpyDeviceToDevice, g.stream);
  if (e != cudaSuccess) return mx_fail_cuda(e, "mark", __FILE__, __LINE__);
  g.mark_next_id = g.next_chunk_id;
  return MX_OK;
}

int mx_gen_reset_to_mark(mx_gen* gen) {
  if (gen) gen->d.fresh_layout = false;  // state changes on the generator stream: later plans wait for it
  MX_CHECK_ARG(gen, "null generator");
  GenData& g = gen->d;
  if (!g.mark_consumed.p) return mx_fail(MX_ERR_INVALID, "no mark set");
  cudaError_t e = cudaMemcpyAsync(g.consumed.p, g.mark_consumed.p, sizeof(u64) * g.mark_consumed.n,
                                  cudaMemcpyDeviceToDevice, g.stream);
  if (e != cudaSuccess) return mx_fail_cuda(e, "reset", __FILE__, __LINE__);
  g.next_chunk_id = g.mark_next_id;
  return MX_OK;
}

int mx_gen_next_chunk_id(const mx_gen* gen, int64_t* next_id) {
  MX_CHECK_ARG(gen && next_id, "null argument");
  *next_id = gen->d.next_chunk_id;
  return MX_OK;
}

int mx_gen_set_next_chunk_id(mx_gen* gen, int64_t next_id) {
  MX_CHECK_ARG(gen && next_id >= 0, "bad argument");
  gen->d.next_chunk_id = next_id;
  return MX_OK;
}

// consumed <-> {pos, offset}: pos = #cursor ranges fully consumed
static int cursor_tables(const GenData& g, std::vector<u32>& kbf, std::vector<u32>& bf,
                         std::vector<unsigned long long>& ccum) {
  const IndexData& d = *g.ix;
  kbf.resize(d.n_keys + 1);
  bf.resize(d.n_blocks + 1);
  ccum.resize(d.n_intervals + 1);
  cudaError_t e = cudaMemcpy(kbf.data(), d.key_blk_first.p, sizeof(u32) * kbf.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(bf.data(), d.blk_first.p, sizeof(u32) * bf.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && d.n_intervals)
    e = cudaMemcpy(ccum.data(), g.ccum.p, sizeof(u64) * ccum.size(), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "cursor tables", __FILE__, __LINE__);
  return MX_OK;
}

// sharded index: real-interval prefix (rcum) and whether each cursor position
// is local
static int shard_tables(const GenData& g, std::vector<unsigned long long>& rcum, std::vector<u32>& lcnt) {
  const IndexData& d = *g.ix;
  rcum.resize(d.n_intervals + 1);
  lcnt.resize(d.n_intervals + 1);
  cudaError_t e = cudaMemcpy(rcum.data(), g.rcum.p, sizeof(u64) * rcum.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(lcnt.data(), g.lcnt.p, sizeof(u32) * lcnt.size(), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "shard tables", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_get_cursors(const mx_gen* gen, int64_t* pos, int64_t* offset) {
  MX_CHECK_ARG(gen && pos && offset, "null argument");
  const GenData& g = gen->d;
  const long long K = g.K;
  if (K == 0) return MX_OK;
  std::vector<u32> kbf, bf, lcnt;
  std::vector<unsigned long long> ccum, used(K), rcum;
  int rc = cursor_tables(g, kbf, bf, ccum);
  if (rc) return rc;
  const bool sharded = g.ix->sharded && g.ix->n_intervals > 0;
  if (sharded && (rc = shard_tables(g, rcum, lcnt))) return rc;
  cudaError_t e = cudaMemcpy(used.data(), g.consumed.p, sizeof(u64) * K, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "cursors", __FILE__, __LINE__);
  for (long long k = 0; k < K; ++k) {
    const long long ib = bf[kbf[k]], ie = bf[kbf[k + 1]];
    const unsigned long long base = ccum[ib];
    // number of ranges whose end <= used
    long long lo = ib, hi = ie;
    while (lo < hi) {
      long long mid = (lo + hi) / 2;
      if (ccum[mid + 1] - base <= used[k]) lo = mid + 1; else hi = mid;
    }
    pos[k] = lo - ib;
    offset[k] = (int64_t)(used[k] - (ccum[lo] - base));
    if (sharded) {
      const bool local = lo < ie && lcnt[lo + 1] > lcnt[lo];
      if (offset[k] > 0 && !local) {  // inside another rank's block: its owner answers
        pos[k] = offset[k] = -1;
      } else {
        pos[k] = (int64_t)(rcum[lo] - rcum[ib]);
      }
    }
  }
  return MX_OK;
}

int mx_gen_cursor_to_consumed(const mx_gen* gen, const int64_t* pos, const int64_t* offset, int64_t* consumed) {
  MX_CHECK_ARG(gen && pos && offset && consumed, "null argument");
  const GenData& g = gen->d;
  const long long K = g.K;
  if (K == 0) return MX_OK;
  std::vector<u32> kbf, bf, lcnt;
  std::vector<unsigned long long> ccum, rcum;
  int rc = cursor_tables(g, kbf, bf, ccum);
  if (rc) return rc;
  const bool sharded = g.ix->sharded && g.ix->n_intervals > 0;
  if (sharded && (rc = shard_tables(g, rcum, lcnt))) return rc;
  for (long long k = 0; k < K; ++k) {
    const long long ib = bf[kbf[k]], ie = bf[kbf[k + 1]];
    const long long n_real = sharded ? (long long)(rcum[ie] - rcum[ib]) : ie - ib;
    if (pos[k] < 0 || pos[k] > n_real || offset[k] < 0)
      return mx_fail(MX_ERR_INVALID, "cursor state out of range for component %lld", k);
    long long j = ib + pos[k];
    if (sharded) {  // cursor position holding real range pos[k]: rcum[j] <= pos < rcum[j+1]
      long long lo = ib, hi = ie;
      while (lo < hi) {
        long long mid = (lo + hi + 1) / 2;
        if ((long long)(rcum[mid] - rcum[ib]) <= pos[k]) lo = mid; else hi = mid - 1;
      }
      j = lo;
      if ((long long)(rcum[j] - rcum[ib]) < pos[k]) {  // strictly inside a remote block
        consumed[k] = -1;
        continue;
      }
    }
    const unsigned long long used = ccum[j] - ccum[ib] + (unsigned long long)offset[k];
    if (used > ccum[ie] - ccum[ib]) return mx_fail(MX_ERR_INVALID, "cursor offset beyond component %lld", k);
    consumed[k] = (int64_t)used;
  }
  return MX_OK;
}

int mx_gen_set_consumed(mx_gen* gen, const int64_t* consumed) {
  if (gen) gen->d.fresh_layout = false;  // state changes on the generator stream: later plans wait for it
  MX_CHECK_ARG(gen && consumed, "null argument");
  GenData& g = gen->d;
  const long long K = g.K;
  if (K == 0) return MX_OK;
  if (int rc = gen_host_mirrors(&g)) return rc;
  for (long long k = 0; k < K; ++k)
    if (consumed[k] < 0 || (unsigned long long)consumed[k] > g.h_comp_total[k])
      return mx_fail(MX_ERR_INVALID, "consumed samples out of range for component %lld", k);
  cudaError_t e = cudaMemcpy(g.consumed.p, consumed, sizeof(u64) * K, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return mx_fail_cuda(e, "set consumed", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_set_cursors(mx_gen* gen, const int64_t* pos, const int64_t* offset) {
  if (gen) gen->d.fresh_layout = false;  // state changes on the generator stream: later plans wait for it
  MX_CHECK_ARG(gen && pos && offset, "null argument");
  if (gen->d.ix->sharded)
    return mx_fail(MX_ERR_INVALID, "sharded generator: use mx_gen_cursor_to_consumed + mx_gen_set_consumed");
  GenData& g = gen->d;
  const long long K = g.K;
  if (K == 0) return MX_OK;
  std::vector<u32> kbf, bf;
  std::vector<unsigned long long> ccum, used(K);
  int rc = cursor_tables(g, kbf, bf, ccum);
  if (rc) return rc;
  for (long long k = 0; k < K; ++k) {
    const long long ib = bf[kbf[k]], ie = bf[kbf[k + 1]];
    if (pos[k] < 0 || pos[k] > ie - ib || offset[k] < 0)
      return mx_fail(MX_ERR_INVALID, "cursor state out of range for component %lld", k);
    used[k] = ccum[ib + pos[k]] - ccum[ib] + (unsigned long long)offset[k];
    if (used[k] > ccum[ie] - ccum[ib]) return mx_fail(MX_ERR_INVALID, "cursor offset beyond component %lld", k);
  }
  cudaError_t e = cudaMemcpy(g.consumed.p, used.data(), sizeof(u64) * K, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return mx_fail_cuda(e, "set cursors", __FILE__, __LINE__);
  return MX_OK;
}

int mx_gen_component_order(const mx_gen* gen, uint32_t* order) {
  MX_CHECK_ARG(gen && order, "null argument");
  if (int rc = gen_host_mirrors(const_cast<GenData*>(&gen->d))) return rc;
  memcpy(order, gen->d.h_comp_order.data(), sizeof(u32) * gen->d.K);
  return MX_OK;
}

int mx_gen_cursor_ranges(const mx_gen* gen, uint32_t comp, int64_t* n_ranges, int32_t* ds, int64_t* file_id,
                         uint32_t* start, uint32_t* end, int64_t capacity) {
  MX_CHECK_ARG(gen && n_ranges, "null argument");
  const GenData& g = gen->d;
  const IndexData& d = *g.ix;
  if ((long long)comp >= g.K) return mx_fail(MX_ERR_INVALID, "component %u out of range", comp);
  if (d.sharded)
    return mx_fail(MX_ERR_UNSUPPORTED, "cursor ranges of a file-sharded generator are distributed over the ranks");
  u32 kb[2], ib, ie;
  cudaError_t e = cudaMemcpy(kb, d.key_blk_first.p + comp, sizeof(u32) * 2, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&ib, d.blk_first.p + kb[0], sizeof(u32), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&ie, d.blk_first.p + kb[1], sizeof(u32), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "cursor ranges", __FILE__, __LINE__);
  const long long n = ie - ib;
  *n_ranges = n;
  if (!ds && !file_id && !start && !end) return MX_OK;
  if (capacity < n) return mx_fail(MX_ERR_INVALID, "capacity %lld < %lld ranges", (long long)capacity, n);
  std::vector<u32> civ(n), f(d.n_intervals), s0(d.n_intervals), e0(d.n_intervals);
  e = cudaMemcpy(civ.data(), g.civ.p + ib, sizeof(u32) * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(f.data(), d.iv_file.p, sizeof(u32) * d.n_intervals, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(s0.data(), d.iv_start.p, sizeof(u32) * d.n_intervals, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(e0.data(), d.iv_end.p, sizeof(u32) * d.n_intervals, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return mx_fail_cuda(e, "cursor ranges", __FILE__, __LINE__);
  for (long long i = 0; i < n; ++i) {
    u32 iv = civ[i];
    if (ds) ds[i] = d.h_file_ds[f[iv]];
    if (file_id) file_id[i] = d.h_file_ids[f[iv]];
    if (start) start[i] = s0[iv];
    if (end) end[i] = e0[iv];
  }
  return MX_OK;
}

int mx_domain_loss(const float* losses, const int32_t* tags, int64_t n, int32_t n_domains, double* sums,
                   int64_t* counts, void* stream) {
  MX_CHECK_ARG(n >= 0, "negative length");
  MX_CHECK_ARG(sums && counts, "null output");
  g_err.clear();
  return domain_loss(losses, tags, n, n_domains, sums, reinterpret_cast<long long*>(counts), (cudaStream_t)stream);
}

int mx_fit_power_law(int32_t n_domains, const int64_t* point_offsets, const double* n, const double* loss,
                     const double* geom, double* out_law, void* stream) {
  g_err.clear();
  return fit_power_law(n_domains, reinterpret_cast<const long long*>(point_offsets), n, loss, geom, out_law,
                       (cudaStream_t)stream);
}

int mx_ado_pi(int32_t k, const double* mu, const double* credit, const double* law, double shared_n, double p_min,
              double smoothing, double* pi_bar, int64_t* pi_bar_count, double* pi, void* stream) {
  g_err.clear();
  return ado_pi(k, mu, credit, law, shared_n, p_min, smoothing, pi_bar, reinterpret_cast<long long*>(pi_bar_count), pi,
                (cudaStream_t)stream);
}

int mx_ado_credit(int32_t k, double rate, const double* pi, double* credit, void* stream) {
  g_err.clear();
  return ado_credit(k, rate, pi, credit, (cudaStream_t)stream);
}

}  // extern "C"
