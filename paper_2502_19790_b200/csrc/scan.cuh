// Generic exclusive scan over n items, reduce-then-scan (three launches):
//   gs_reduce  -- per 2048-item tile: sum of f.value(i)          -> agg[t]
//                 (items warp-striped inside a tile: coalesced accesses)
//   gs_scan    -- one CTA: exclusive scan of the tile sums (in place)
//   gs_apply   -- per tile: recompute values, block scan, f.apply(i, excl, v)
// Replaces single-pass decoupled look-back for the index / cursor / emission
// scans: with every tile resident at once nobody holds an inclusive prefix
// yet, so a look-back walks O(tiles / 32) windows and the last tiles wait
// tens of microseconds; here the critical path is three short kernels and the
// items are read twice (value() must be cheap and side-effect free).
// F provides: __device__ u64 value(long long i) const;
//             __device__ void apply(long long i, u64 excl, u64 v) const;
//             __device__ void total(u64 sum) const;   (called once, n > 0)
#pragma once

#include "common.cuh"
#include "mixtera_internal.cuh"

namespace mx {

constexpr int GS_THREADS = 256;
constexpr int GS_ITEMS = 8;
constexpr int GS_TILE = GS_THREADS * GS_ITEMS;

__device__ __forceinline__ u64 gs_block_excl(u64 v, u64* s_w, u64* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 inc = warp_incl_scan(v);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const u64 x = lane < GS_THREADS / 32 ? s_w[lane] : 0;
    const u64 xi = warp_incl_scan(x);
    if (lane < GS_THREADS / 32) s_w[lane] = xi - x;
    if (lane == 31) s_w[GS_THREADS / 32] = xi;
  }
  __syncthreads();
  *block_total = s_w[GS_THREADS / 32];
  return s_w[warp] + inc - v;
}

// items of tile t: t * GS_TILE + q * GS_THREADS + threadIdx.x (q < GS_ITEMS):
// warp-striped, so every load / store instruction of a warp is coalesced
template <class F>
__global__ void __launch_bounds__(GS_THREADS) gs_reduce(long long n, F f, u64* agg) {
  __shared__ u64 s_w[GS_THREADS / 32];
  const long long b = (long long)blockIdx.x * GS_TILE + threadIdx.x;
  u64 sum = 0;
#pragma unroll
  for (int q = 0; q < GS_ITEMS; ++q)
    if (b + q * GS_THREADS < n) sum += f.value(b + q * GS_THREADS);
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int w = 0; w < GS_THREADS / 32; ++w) t += s_w[w];
    agg[blockIdx.x] = t;
  }
}

// in-place exclusive scan of T tile sums; agg[T] = total (single CTA)
static __global__ void __launch_bounds__(1024) gs_scan(long long T, u64* agg) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_carry;
  constexpr int ITEMS = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (long long base = 0; base < T; base += 1024 * ITEMS) {
    const long long i0 = base + (long long)threadIdx.x * ITEMS;
    u64 v[ITEMS], sum = 0;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      v[q] = i0 + q < T ? agg[i0 + q] : 0;
      sum += v[q];
    }
    const u64 inc = warp_incl_scan(sum);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const u64 x = s_w[lane];
      const u64 xi = warp_incl_scan(x);
      s_w[lane] = xi - x;
      if (lane == 31) s_w[32] = xi;
    }
    __syncthreads();
    u64 run = s_carry + s_w[warp] + inc - sum;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      if (i0 + q < T) agg[i0 + q] = run;
      run += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_w[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) agg[T] = s_carry;
}

template <class F>
__global__ void __launch_bounds__(GS_THREADS) gs_apply(long long n, F f, const u64* excl) {
  __shared__ u64 s_w[2][GS_THREADS / 32 + 1];
  const long long b = (long long)blockIdx.x * GS_TILE + threadIdx.x;
  u64 v[GS_ITEMS];
#pragma unroll
  for (int q = 0; q < GS_ITEMS; ++q) v[q] = b + q * GS_THREADS < n ? f.value(b + q * GS_THREADS) : 0;
  u64 carry = excl[blockIdx.x];
#pragma unroll
  for (int q = 0; q < GS_ITEMS; ++q) {  // one block scan per stripe (double-buffered scratch)
    u64 tot;
    const u64 ex = gs_block_excl(v[q], s_w[q & 1], &tot);
    const long long i = b + q * GS_THREADS;
    if (i < n) {
      f.apply(i, carry + ex, v[q]);
      if (i == n - 1) f.total(carry + ex + v[q]);
    }
    carry += tot;
  }
}

// Launch the three kernels for n items (n may be 0: nothing happens).
template <class F>
int gs_run(long long n, const F& f, cudaStream_t s) {
  if (n <= 0) return MX_OK;
  const long long T = (n + GS_TILE - 1) / GS_TILE;
  DevBuf<u64> agg;  // tile sums: a workspace view (gs_run calls on a stream run in order)
  MX_CUDA_TRY(ws_borrow(agg, s, WS_GSAGG, T + 1));
  gs_reduce<F><<<(unsigned)T, GS_THREADS, 0, s>>>(n, f, agg.p);
  mx_count_launch();
  gs_scan<<<1, 1024, 0, s>>>(T, agg.p);
  mx_count_launch();
  gs_apply<F><<<(unsigned)T, GS_THREADS, 0, s>>>(n, f, agg.p);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // namespace mx
