// Shared device utilities for the sm_100a Mixtera hot path.
//
// * warp primitives (inclusive scans, sums),
// * decoupled look-back for single-pass device-wide prefix sums (stage-1
//   run compaction and the index scans),
// * streaming 128-bit loads that bypass L1 (column tiles are touched once),
// * an error channel: kernels report typed failures through a small device
//   struct the host reads after the launch sequence (mapped to the
//   reference's exception types by capi.cu).
#pragma once
#include <map>

#include <cuda_runtime.h>
#include <stdint.h>

#define MX_FULL 0xffffffffu

namespace mx {

typedef unsigned long long u64;
typedef uint32_t u32;

__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// four consecutive u16 codes (8-byte aligned) widened to an int4
__device__ __forceinline__ int4 ld_stream_u16x4(const void* p) {
  u32 lo, hi;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "l"(p));
  return make_int4((int)(lo & 0xffffu), (int)(lo >> 16), (int)(hi & 0xffffu), (int)(hi >> 16));
}

__device__ __forceinline__ int ld_stream(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 r;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(MX_FULL, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(MX_FULL, v, d);
  return v;
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single pass scan). One 64-bit status word per tile:
// bits 63..62 = flag (0 = not ready, 1 = tile aggregate, 2 = inclusive
// prefix), bits 61..0 = value. Tiles take ids from an atomic counter so every
// predecessor of a tile has already been scheduled (forward progress).
// ---------------------------------------------------------------------------
constexpr u64 LB_AGG = 1ull << 62;
constexpr u64 LB_PREFIX = 2ull << 62;
constexpr u64 LB_VALUE = (1ull << 62) - 1;

// Called by ALL lanes of ONE warp. Returns the exclusive prefix of `tile`.
__device__ __forceinline__ u64 lookback_exclusive(u64* status, int tile, u64 aggregate) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(status, LB_PREFIX | aggregate);
    return 0;
  }
  if (lane == 0) st_release(status + tile, LB_AGG | aggregate);
  u64 excl = 0;
  int base = tile - 1;
  while (true) {
    const int idx = base - lane;
    u64 w = idx >= 0 ? ld_acquire(status + idx) : LB_PREFIX;
    const u64 flag = w & ~LB_VALUE;
    if (__any_sync(MX_FULL, flag == 0)) continue;  // a predecessor is still running
    const u32 pm = __ballot_sync(MX_FULL, flag == LB_PREFIX);
    const int first = pm ? __ffs(pm) - 1 : 32;
    u64 v = lane <= first ? (w & LB_VALUE) : 0;
    excl += warp_sum(v);
    if (pm) break;
    base -= 32;
  }
  if (lane == 0) st_release(status + tile, LB_PREFIX | (excl + aggregate));
  return excl;
}

// Device-side error record (first failure wins per field).
struct DevError {
  u64 null_key_sample;  // min global sample index of an un-keyable run (~0 = none)
  u32 overlap;          // non-zero: overlapping/empty interval detected
  u32 pad;
};

}  // namespace mx

#define MX_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::mx_fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

int mx_fail_cuda(cudaError_t e, const char* what, const char* file, int line);
int mx_fail(int code, const char* fmt, ...);
// stream-ordered upload of a (small) pageable host array through pinned
// staging, without the implicit stream synchronisation of a pageable copy
cudaError_t mx_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
// several host arrays -> one device block with ONE copy (staged together in
// the pinned ring); item i lands at dst + off[i]
cudaError_t mx_h2d_gather(void* dst, const void* const* src, const size_t* bytes, const size_t* off, int n,
                          size_t total, cudaStream_t s);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) costs microseconds of host
// time per call: raise the limit only when a launch needs more than the
// kernel has on this device (per host thread).
template <typename K>
cudaError_t mx_smem_attr(K* kernel, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static thread_local std::map<std::pair<const void*, int>, size_t> have;
  size_t& h = have[{reinterpret_cast<const void*>(kernel), dev}];
  if (bytes <= h) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) h = bytes;
  return e;
}

struct Uploads {
  static constexpr int kMax = 16;
  const void* src[kMax];
  size_t bytes[kMax], off[kMax];
  int n = 0;
  size_t total = 0;
  size_t add(const void* p, size_t b) {  // offset of the item in the block (256-byte aligned)
    const size_t o = (total + 255) & ~size_t(255);
    src[n] = p;
    bytes[n] = b;
    off[n] = o;
    ++n;
    total = o + b;
    return o;
  }
  cudaError_t run(void* dst, cudaStream_t s) const { return mx_h2d_gather(dst, src, bytes, off, n, total, s); }
};

// Small device->host reads gathered into a per-thread pinned block and
// delivered after ONE stream synchronisation: a cudaMemcpyAsync into
// pageable memory blocks the host per call (~10 us round trip each).
// Reads that do not fit are copied directly (pageable, still correct).
struct D2HBatch {
  struct Item {
    void* dst;
    size_t off, bytes;
  };
  cudaStream_t s;
  Item items[16];
  int n = 0;
  size_t used = 0;
  explicit D2HBatch(cudaStream_t st) : s(st) {}
  cudaError_t add(void* dst, const void* src, size_t bytes);
  cudaError_t sync();  // cudaStreamSynchronize + deliver every read
  // wait only for the copies queued so far (an event recorded behind them),
  // so later work on the stream keeps running; no other batch in between
  cudaError_t sync_event(cudaEvent_t e);
};

// Host-side checkpoints (MX_HOST_TIMING=1): wall-clock microseconds between
// labelled points of a C-ABI call, printed to stderr by mx_host_mark(nullptr).
void mx_host_mark(const char* label);

// Launch accounting and per-phase CUDA-event timing (capi.cu). A phase timer
// records events on the launching stream when profiling is enabled
// (mx_profile_enable); totals are read back with mx_profile_read.
void mx_count_launch();
struct MxPhase {
  const char* name;
  cudaStream_t stream;
  void* start;
  MxPhase(const char* n, cudaStream_t s);
  ~MxPhase();
};
