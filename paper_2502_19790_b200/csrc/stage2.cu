// Stage 2 -- chunk generation on sm_100a.
//
// Reference: ChunkGenerator.generate (chunks.py:194-230), _take_for_key
// (:150-167), redistribute_best_effort (:109-130), apportion
// (mixtures.py:158-184), _normalize/_finish (chunks.py:169-192),
// generate_arbitrary (:232-253).
//
// The reference walks Python cursor objects range by range. Here a chunk is
// decided at COUNT level first and only then cut:
//
//  * match_*_kernel   -- mixture key x component key matching from per-
//                        property value-rank bitsets (mixtures.py:100-109);
//                        per mixture key the matching components in seeded
//                        component order (L_m).
//  * plan_kernel      -- ONE thread replays Algorithm 1 on integers: passes
//                        over mixture keys, depletion, strict stop, best-effort
//                        redistribution with a bit-exact apportion (Neumaier
//                        sum, int(share + 1e-9), (-frac, key rank) order).
//                        When no component is shared between mixture keys
//                        (the common case), each mixture key draws from its
//                        own stream S_m = concat of its components' cursor
//                        streams, and a chunk's outcome depends only on which
//                        keys are depleted. One simulated chunk then repeats
//                        verbatim for floor(avail_m / took_m) chunks: the plan
//                        is a handful of PHASES (base, stride per key) instead
//                        of one replay per chunk. Shared components fall back
//                        to an exact per-chunk replay at component level.
//  * emit_*_kernels   -- fully parallel over (chunk, term): binary search of
//                        the stream offset in segment prefix sums, then in the
//                        cursor-order interval prefix sums (ccum), cut the
//                        intervals; per-chunk sort by (mixture key, file,
//                        start) + adjacent merge in shared memory; compaction
//                        into a CSR; device BLAKE2b chunk seeds.
//
// Algorithmic bytes: B2 = sum over chunks of
// (16 * intervals touched + 20 * ranges emitted) + 8 per chunk seed.
#include <memory>

#include "blake2b.cuh"
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "mixtera_internal.cuh"
#include "scan.cuh"

namespace mx {

// ------------------------------------------------------------------ matching
struct MatchArgs {
  int Km;
  long long K;
  const u32* comp_order;  // [K] component ranks in seeded order
  const u32* key_packed;  // [K]
  int n_props;
  u32 shift[MX_MAX_PROPS];
  u32 width[MX_MAX_PROPS];
  int allow_base[MX_MAX_PROPS];
  int allow_words;
  const u32* allow;  // [Km][allow_words]
};

__device__ __forceinline__ bool mkey_matches(const MatchArgs& a, int m, u32 packed) {
  const u32* al = a.allow + (long long)m * a.allow_words;
  for (int p = 0; p < a.n_props; ++p) {
    u32 r = (packed >> a.shift[p]) & ((1u << a.width[p]) - 1u);
    u32 bit = (u32)a.allow_base[p] + r;
    if (!((al[bit >> 5] >> (bit & 31)) & 1u)) return false;
  }
  return true;
}

// one CTA per mixture key: count matches, the per-component hit counts and
// the key's stream length (remaining samples of its matching components).
// Order-free (components by rank), so it need not wait for the component
// order shuffle.
__global__ void match_count_kernel(MatchArgs a, u32* L_cnt, u32* comp_hits, const u64* comp_total,
                                   const u64* consumed, u64* m_tot) {
  __shared__ u32 s_cnt;
  __shared__ unsigned long long s_tot;
  const int m = blockIdx.x;
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_tot = 0;
  }
  __syncthreads();
  u32 c = 0;
  u64 t = 0;
  for (long long comp = threadIdx.x; comp < a.K; comp += blockDim.x) {
    if (mkey_matches(a, m, a.key_packed[comp])) {
      ++c;
      t += comp_total[comp] - consumed[comp];
      atomicAdd(comp_hits + comp, 1u);
    }
  }
  c = warp_sum(c);
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_cnt, c);
    atomicAdd(&s_tot, (unsigned long long)t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    L_cnt[m] = s_cnt;
    m_tot[m] = s_tot;
  }
}

// one CTA per mixture key: ordered compaction of matching components
__global__ void __launch_bounds__(256) match_fill_kernel(MatchArgs a, const u32* L_off, u32* L) {
  __shared__ u32 s_w[8];
  __shared__ u32 s_base;
  const int m = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = L_off[m];
  __syncthreads();
  for (long long b = 0; b < a.K; b += 256) {
    long long pos = b + threadIdx.x;
    u32 comp = pos < a.K ? a.comp_order[pos] : 0;
    u32 f = (pos < a.K && mkey_matches(a, m, a.key_packed[comp])) ? 1u : 0u;
    u32 inc = warp_incl_scan(f);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u32 x = lane < 8 ? s_w[lane] : 0;
      u32 xi = warp_incl_scan(x);
      if (lane < 8) s_w[lane] = xi - x;
    }
    __syncthreads();
    if (f) L[s_base + s_w[warp] + inc - 1] = comp;
    __syncthreads();
    if (threadIdx.x == 255) s_base += s_w[7] + inc;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ streams
// A stream is a list of segments (component, absolute start offset, length).
//   mode 0 (disjoint mixture): stream m = L_m components, [consumed, total)
//   mode 1 (shared components): stream c = component c, [0, total)
//   mode 2 (arbitrary): stream 0 = all components in order, [consumed, total)
__global__ void build_segments_kernel(int mode, int n_streams, const u32* s_off, const u32* list,
                                      const u64* comp_total, const u64* consumed, u32* seg_comp, u64* seg_lo,
                                      u64* seg_pre) {
  // one warp per stream, 32 segments per step with a warp scan.
  // seg_pre has (segments + streams) entries: stream s uses [b + s, e + s].
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long s = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); s < n_streams; s += warps) {
    const u32 b = s_off[s], e = s_off[s + 1];
    u64 run = 0;
    for (u32 i0 = b; i0 < e; i0 += 32) {
      const u32 i = i0 + lane;
      u64 len = 0;
      if (i < e) {
        const u32 c = mode == 1 ? (u32)s : list[i];
        const u64 lo = mode == 1 ? 0 : consumed[c];
        len = comp_total[c] - lo;
        seg_comp[i] = c;
        seg_lo[i] = lo;
      }
      const u64 inc = warp_incl_scan(len);
      if (i < e) seg_pre[i + s] = run + inc - len;
      run += __shfl_sync(MX_FULL, inc, 31);
    }
    if (lane == 0) seg_pre[e + s] = run;
  }
}

// consumed[c] after a plan: lo + clamp(pos_s - pre_i, 0, len_i)
__global__ void commit_segments_kernel(int n_streams, const u32* s_off, const u32* seg_comp, const u64* seg_lo,
                                       const u64* seg_pre, const u64* pos, u64* consumed) {
  int s = blockIdx.x;
  if (s >= n_streams) return;
  u32 b = s_off[s], e = s_off[s + 1];
  u64 p = pos[s];
  for (u32 i = b + threadIdx.x; i < e; i += blockDim.x) {
    u64 pre = seg_pre[i + s], nxt = seg_pre[i + 1 + s];
    u64 used = p <= pre ? 0 : (p >= nxt ? nxt - pre : p - pre);
    consumed[seg_comp[i]] = seg_lo[i] + used;
  }
}

// ------------------------------------------------------------------ planner
struct Term {
  u32 m;       // mixture key index (ignored in arbitrary mode)
  u32 stream;  // stream id
  u64 base;    // stream offset of chunk 0 of the phase
  u64 len;     // samples per chunk
  u64 stride;  // base advance per chunk
};

struct Phase {
  long long chunk_begin;  // relative to the plan
  long long n_chunks;
  long long term_begin;
  long long n_terms;
};

struct PlanArgs {
  int mode;
  int Km;
  long long C;
  int strict;
  long long max_chunks;
  const double* w;
  // mode 0 / 2: stream lengths
  const u64* seg_pre;
  const u32* s_off;
  const u64* slen;  // mode 0: length of stream m (staged in shared memory by plan_kernel)
  // mode 1
  const u32* L_off;
  const u32* L;
  const u64* comp_total;
  u64* consumed;
  u32* front;
  // scratch [Km]
  long long* counts;
  long long* rem;
  long long* found;
  long long* took;
  unsigned char* dead;
  unsigned char* newly;
  u64* pos;  // per stream, relative
  int* ap_idx;
  double* ap_frac;
  long long* ap_base;
  // out
  Phase* phases;
  long long cap_phases;
  Term* terms;
  long long cap_terms;
  long long* out;  // [0]=chunks [1]=phases [2]=terms [3]=exhausted
  long long* report;
};

// CPython 3.12 builtin sum over floats (Neumaier), keys in index order
__device__ double neumaier(const double* w, const unsigned char* skip, int n) {
  double s = 0.0, c = 0.0;
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) continue;
    double x = w[i];
    double t = s + x;
    if (fabs(s) >= fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  return c != 0.0 ? s + c : s;
}

__device__ __forceinline__ bool frac_before(double fa, int a, double fb, int b) {
  // order by (-frac, key index)
  if (fa != fb) return fa > fb;
  return a < b;
}

// heap sort of idx[0..n) by frac_before (ascending in that order)
__device__ void heap_sort(int* idx, const double* fr, int n) {
  auto less = [&](int x, int y) { return frac_before(fr[x], x, fr[y], y); };
  auto sift = [&](int root, int end) {
    while (true) {
      int child = 2 * root + 1;
      if (child >= end) return;
      if (child + 1 < end && less(idx[child], idx[child + 1])) ++child;
      if (less(idx[root], idx[child])) {
        int t = idx[root]; idx[root] = idx[child]; idx[child] = t;
        root = child;
      } else {
        return;
      }
    }
  };
  for (int s = n / 2 - 1; s >= 0; --s) sift(s, n);
  for (int e = n - 1; e > 0; --e) {
    int t = idx[0]; idx[0] = idx[e]; idx[e] = t;
    sift(0, e);
  }
}

// apportion(weights restricted to keys with !skip[i], total): adds the counts
// into out[] (out[i] += count_i). Returns false when wsum <= 0.
__device__ bool apportion_add(const PlanArgs& a, const unsigned char* skip, long long total, long long* out) {
  const int n = a.Km;
  double wsum = neumaier(a.w, skip, n);
  if (!(wsum > 0.0)) return false;
  const double tot = (double)total;
  long long assigned = 0;
  int cnt = 0;
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) continue;
    double share = a.w[i] / wsum * tot;
    long long base = (long long)(share + 1e-9);
    double fr = share - (double)base;
    a.ap_frac[i] = fr > 0.0 ? fr : 0.0;
    a.ap_base[i] = base;
    assigned += base;
    a.ap_idx[cnt++] = i;
  }
  long long left = total - assigned;
  if (left > 0) {
    if (cnt <= 32) {  // insertion sort
      for (int x = 1; x < cnt; ++x) {
        int v = a.ap_idx[x];
        int y = x - 1;
        while (y >= 0 && frac_before(a.ap_frac[v], v, a.ap_frac[a.ap_idx[y]], a.ap_idx[y])) {
          a.ap_idx[y + 1] = a.ap_idx[y];
          --y;
        }
        a.ap_idx[y + 1] = v;
      }
    } else {
      heap_sort(a.ap_idx, a.ap_frac, cnt);
    }
    for (long long t = 0; t < left && t < cnt; ++t) a.ap_base[a.ap_idx[t]] += 1;
  }
  for (int x = 0; x < cnt; ++x) out[a.ap_idx[x]] += a.ap_base[a.ap_idx[x]];
  return true;
}

// take up to `need` from mixture key m (mode 1: component frontiers)
__device__ long long take_shared(PlanArgs& a, int m, long long need, long long* n_terms) {
  long long got = 0;
  u32 b = a.L_off[m], e = a.L_off[m + 1];
  for (u32 i = b + a.front[m]; i < e && need > 0; ++i) {
    u32 c = a.L[i];
    u64 used = a.consumed[c], tot = a.comp_total[c];
    if (used >= tot) {
      if (i == b + a.front[m]) a.front[m] += 1;
      continue;
    }
    long long t = (long long)(tot - used) < need ? (long long)(tot - used) : need;
    if (*n_terms < a.cap_terms) {
      Term& tm = a.terms[*n_terms];
      tm.m = (u32)m;
      tm.stream = c;
      tm.base = used;
      tm.len = (u64)t;
      tm.stride = 0;
    }
    *n_terms += 1;
    a.consumed[c] = used + (u64)t;
    got += t;
    need -= t;
  }
  return got;
}

// Simulate one generate() call. Returns 1 = chunk, 0 = None (exhausted).
__device__ int simulate_chunk(PlanArgs& a, long long* n_terms) {
  const int Km = a.Km;
  for (int m = 0; m < Km; ++m) {
    a.rem[m] = a.counts[m];
    a.dead[m] = 0;
    a.took[m] = 0;
  }
  while (true) {
    bool anypos = false;
    for (int m = 0; m < Km; ++m) anypos |= a.rem[m] > 0;
    if (!anypos) break;
    for (int m = 0; m < Km; ++m) {
      a.found[m] = -1;
      if (a.rem[m] <= 0) continue;
      long long g;
      if (a.mode == 1) {
        g = take_shared(a, m, a.rem[m], n_terms);
      } else {
        const u64 len = a.slen ? a.slen[m] : a.seg_pre[a.s_off[m + 1] + m];  // end of stream m
        long long avail = (long long)(len - a.pos[m]) - a.took[m];
        g = a.rem[m] < avail ? a.rem[m] : avail;
      }
      a.took[m] += g;
      a.rem[m] -= g;
      a.found[m] = g;
    }
    bool any_new = false;
    for (int m = 0; m < Km; ++m) {
      a.newly[m] = (a.found[m] == 0 && a.rem[m] > 0) ? 1 : 0;
      any_new |= a.newly[m];
    }
    if (!any_new) continue;
    if (a.strict) {
      for (int m = 0; m < Km; ++m) a.report[m] = a.rem[m];
      return 0;
    }
    for (int m = 0; m < Km; ++m) {
      if (!a.newly[m]) continue;
      a.dead[m] = 1;
      bool alive = false;
      for (int x = 0; x < Km; ++x) alive |= !a.dead[x];
      if (!alive) {
        for (int x = 0; x < Km; ++x) a.report[x] = a.rem[x];
        return 0;
      }
      if (a.rem[m] > 0) apportion_add(a, a.dead, a.rem[m], a.rem);
      a.rem[m] = 0;
    }
  }
  return 1;
}

constexpr int PLAN_SMEM_KM = 256;

__global__ void plan_kernel(PlanArgs a) {
  // The planner is one sequential thread: keep its per-key state in shared
  // memory when it fits (each access is then ~30 cycles instead of an L2
  // trip); the warp stages the weights and stream lengths in parallel first,
  // so the sequential replay never waits on a dependent global load.
  __shared__ long long s_ll[5][PLAN_SMEM_KM];
  __shared__ unsigned char s_flags[2][PLAN_SMEM_KM];
  __shared__ u64 s_pos[PLAN_SMEM_KM], s_len[PLAN_SMEM_KM];
  __shared__ int s_idx[PLAN_SMEM_KM];
  __shared__ double s_frac[PLAN_SMEM_KM], s_w[PLAN_SMEM_KM];
  if (blockIdx.x != 0) return;
  const int Km = a.Km;
  const bool staged = Km <= PLAN_SMEM_KM && a.mode != 1;
  if (staged) {
    for (int m = threadIdx.x; m < Km; m += blockDim.x) {
      s_w[m] = a.w[m];
      if (a.mode == 0) s_len[m] = a.slen ? a.slen[m] : a.seg_pre[a.s_off[m + 1] + m];
    }
    __syncwarp();
  }
  if (threadIdx.x != 0) return;
  u64* pos_out = a.pos;
  long long* report_out = a.report;
  if (staged) {
    a.w = s_w;
    if (a.mode == 0) a.slen = s_len;
    a.counts = s_ll[0];
    a.rem = s_ll[1];
    a.found = s_ll[2];
    a.took = s_ll[3];
    a.ap_base = s_ll[4];
    a.dead = s_flags[0];
    a.newly = s_flags[1];
    a.pos = s_pos;
    a.ap_idx = s_idx;
    a.ap_frac = s_frac;
    a.report = s_ll[4];  // written only when the plan stops; ap_base is dead then
  }
  for (int m = 0; m < Km; ++m) a.counts[m] = 0;
  apportion_add(a, nullptr, a.C, a.counts);
  long long chunks = 0, n_ph = 0, n_terms = 0, exhausted = 0;
  for (int m = 0; m < Km; ++m) a.pos[m] = 0;
  while (chunks < a.max_chunks) {
    if (n_ph >= a.cap_phases) break;
    if (a.mode == 1) {
      if (a.cap_terms - n_terms < (long long)Km + a.C) break;
      long long t0 = n_terms;
      int ok = simulate_chunk(a, &n_terms);
      if (!ok) {
        n_terms = t0;
        exhausted = 1;
        break;
      }
      Phase& ph = a.phases[n_ph++];
      ph.chunk_begin = chunks;
      ph.n_chunks = 1;
      ph.term_begin = t0;
      ph.n_terms = n_terms - t0;
      chunks += 1;
      continue;
    }
    if (a.cap_terms - n_terms < (long long)Km) break;
    int ok = simulate_chunk(a, &n_terms);
    if (!ok) {
      for (int m = 0; m < Km; ++m) a.pos[m] += (u64)a.took[m];
      exhausted = 1;
      break;
    }
    // repetition count: every key with took > 0 can serve floor(avail / took) chunks
    long long rep = a.max_chunks - chunks;
    for (int m = 0; m < Km; ++m) {
      if (a.took[m] <= 0) continue;
      const u64 len = a.slen ? a.slen[m] : a.seg_pre[a.s_off[m + 1] + m];
      long long avail = (long long)(len - a.pos[m]);
      long long r = avail / a.took[m];
      if (r < rep) rep = r;
    }
    if (rep < 1) rep = 1;
    Phase& ph = a.phases[n_ph++];
    ph.chunk_begin = chunks;
    ph.n_chunks = rep;
    ph.term_begin = n_terms;
    long long nt = 0;
    for (int m = 0; m < Km; ++m) {
      if (a.took[m] <= 0) continue;
      Term& tm = a.terms[n_terms + nt++];
      tm.m = (u32)m;
      tm.stream = (u32)m;
      tm.base = a.pos[m];
      tm.len = (u64)a.took[m];
      tm.stride = (u64)a.took[m];
      a.pos[m] += (u64)a.took[m] * (u64)rep;
    }
    ph.n_terms = nt;
    n_terms += nt;
    chunks += rep;
  }
  if (a.pos != pos_out) {
    for (int m = 0; m < Km; ++m) pos_out[m] = a.pos[m];
    if (exhausted)
      for (int m = 0; m < Km; ++m) report_out[m] = a.report[m];
  }
  a.out[0] = chunks;
  a.out[1] = n_ph;
  a.out[2] = n_terms;
  a.out[3] = exhausted;
}

// ---------------------------------------------------------------------------
// Fused matching + count-level plan for a mixture of <= 32 keys (the common
// static / hierarchical case, e.g. cfg 2): ONE launch, no host round trip
// between matching and planning, and the plan replay is lane-parallel (lane m
// owns mixture key m) instead of one thread walking every key in turn.
// Matching is order-free (per-key stream LENGTHS only), so this runs before
// the component-order shuffle finishes; the ordered lists / segment tables are
// built afterwards for emission. Same arithmetic as plan_kernel (mode 0):
// CPython's sequential Neumaier sum, int(share + 1e-9), the (-frac, key)
// leftover order, best-effort redistribution in key order, strict stop.
// If any component matches two mixture keys (shared streams), out[4] = 1 and
// nothing is planned: the caller takes the general path.
constexpr int FP_THREADS = 1024;
constexpr int FP_MAX_KM = 32;

struct FusedPlanArgs {
  MatchArgs ma;
  const u64* comp_total;
  const u64* consumed;
  long long C;
  int strict;
  long long max_chunks;
  const double* w;
  u32* L_off;       // [Km + 1] matching components per key (prefix)
  u64* pos;         // [Km] stream position after the plan
  Phase* phases;
  long long cap_phases;
  Term* terms;
  long long cap_terms;
  long long* out;   // [0] chunks [1] phases [2] terms [3] exhausted [4] shared
  long long* report;
};

// apportion over the lanes whose `skip` is false (apportion_add)
__device__ __forceinline__ long long fp_apportion(double w, bool skip, bool mine, int Km, long long total) {
  const int lane = threadIdx.x & 31;
  double s = 0.0, c = 0.0;  // sequential Neumaier sum in key order, in every lane
  for (int j = 0; j < Km; ++j) {
    const double x = __shfl_sync(MX_FULL, w, j);
    const int sk = __shfl_sync(MX_FULL, (int)skip, j);
    if (sk) continue;
    const double t = s + x;
    if (fabs(s) >= fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  const double wsum = c != 0.0 ? s + c : s;
  if (!(wsum > 0.0)) return 0;
  const bool alive = mine && !skip;
  long long base = 0;
  double fr = 0.0;
  if (alive) {
    const double share = w / wsum * (double)total;
    base = (long long)(share + 1e-9);
    const double f = share - (double)base;
    fr = f > 0.0 ? f : 0.0;
  }
  const long long left = total - warp_sum(base);
  if (left > 0) {
    long long rank = 0;  // alive keys before this one in (frac desc, key asc) order
    for (int j = 0; j < Km; ++j) {
      const double fj = __shfl_sync(MX_FULL, fr, j);
      const int aj = !__shfl_sync(MX_FULL, (int)skip, j);
      if (aj && (fj > fr || (fj == fr && j < lane))) ++rank;
    }
    if (alive && rank < left) base += 1;
  }
  return base;
}

__global__ void __launch_bounds__(FP_THREADS) plan_fused_kernel(FusedPlanArgs a) {
  __shared__ u32 s_cnt[FP_MAX_KM];
  __shared__ unsigned long long s_tot[FP_MAX_KM];
  __shared__ int s_shared;
  const int Km = a.ma.Km, tid = threadIdx.x;
  if (tid < FP_MAX_KM) {
    s_cnt[tid] = 0;
    s_tot[tid] = 0;
  }
  if (tid == 0) s_shared = 0;
  __syncthreads();
  // ---- matching (order-free): per key count and remaining samples,
  // aggregated per warp first (one shared atomic per warp and key: 64-bit
  // shared atomics from every thread on a handful of addresses serialise)
  const int lane0 = tid & 31;
  for (long long b = tid - lane0; b < a.ma.K; b += FP_THREADS) {
    const long long comp = b + lane0;
    int hit = -1, nm = 0;
    u64 t = 0;
    if (comp < a.ma.K) {
      const u32 packed = a.ma.key_packed[comp];
      for (int m = 0; m < Km; ++m)
        if (mkey_matches(a.ma, m, packed)) {
          hit = m;
          ++nm;
        }
      if (nm == 1) t = a.comp_total[comp] - a.consumed[comp];
    }
    if (__any_sync(MX_FULL, nm > 1)) {
      if (lane0 == 0) s_shared = 1;
      continue;
    }
    for (int m = 0; m < Km; ++m) {
      const u32 c = __popc(__ballot_sync(MX_FULL, hit == m));
      const u64 tm = warp_sum(hit == m ? t : (u64)0);
      if (lane0 == 0 && c) {
        atomicAdd(&s_cnt[m], c);
        atomicAdd(&s_tot[m], (unsigned long long)tm);
      }
    }
  }
  __syncthreads();
  if (tid >= 32) return;
  const int lane = tid;
  if (lane == 0) {
    u32 o = 0;
    for (int m = 0; m < Km; ++m) {
      a.L_off[m] = o;
      o += s_cnt[m];
    }
    a.L_off[Km] = o;
    a.out[4] = s_shared;
  }
  if (s_shared) {
    if (lane == 0) a.out[0] = a.out[1] = a.out[2] = a.out[3] = 0;
    return;
  }
  // ---- plan (warp 0; lane m = mixture key m)
  const bool mine = lane < Km;
  const double w = mine ? a.w[lane] : 0.0;
  const u64 len = mine ? (u64)s_tot[lane] : 0;
  u64 pos = 0;
  const long long counts = fp_apportion(w, !mine, mine, Km, a.C);
  long long chunks = 0, n_ph = 0, n_terms = 0, exhausted = 0, rem = 0, took = 0, report = 0;
  while (chunks < a.max_chunks) {
    if (n_ph >= a.cap_phases) break;
    if (a.cap_terms - n_terms < (long long)Km) break;
    // simulate one generate() (simulate_chunk, mode 0)
    rem = mine ? counts : 0;
    took = 0;
    bool dead = !mine, ok = true;
    while (true) {
      if (!__any_sync(MX_FULL, rem > 0)) break;
      long long found = -1;
      if (rem > 0) {
        const long long avail = (long long)(len - pos) - took;
        const long long g = rem < avail ? rem : avail;
        took += g;
        rem -= g;
        found = g;
      }
      u32 newly = __ballot_sync(MX_FULL, found == 0 && rem > 0);
      if (!newly) continue;
      if (a.strict) {
        report = rem;
        ok = false;
        break;
      }
      while (newly) {  // newly exhausted keys in key order
        const int m = __ffs(newly) - 1;
        newly &= newly - 1;
        if (lane == m) dead = true;
        if (!__any_sync(MX_FULL, !dead)) {
          report = rem;
          ok = false;
          break;
        }
        const long long rm = __shfl_sync(MX_FULL, rem, m);
        if (rm > 0) rem += fp_apportion(w, dead, mine, Km, rm);
        if (lane == m) rem = 0;
      }
      if (!ok) break;
    }
    if (!ok) {
      pos += (u64)took;
      exhausted = 1;
      break;
    }
    // every key with took > 0 can serve floor(avail / took) chunks
    long long rep = a.max_chunks - chunks;
    if (took > 0) {
      const long long r = (long long)(len - pos) / took;
      if (r < rep) rep = r;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const long long o = __shfl_xor_sync(MX_FULL, rep, d);
      rep = o < rep ? o : rep;
    }
    if (rep < 1) rep = 1;
    const u32 tk = __ballot_sync(MX_FULL, took > 0);
    const long long nt = __popc(tk);
    if (took > 0) {
      Term& tm = a.terms[n_terms + __popc(tk & ((1u << lane) - 1u))];
      tm.m = (u32)lane;
      tm.stream = (u32)lane;
      tm.base = pos;
      tm.len = (u64)took;
      tm.stride = (u64)took;
      pos += (u64)took * (u64)rep;
    }
    if (lane == 0) {
      Phase& ph = a.phases[n_ph];
      ph.chunk_begin = chunks;
      ph.n_chunks = rep;
      ph.term_begin = n_terms;
      ph.n_terms = nt;
    }
    ++n_ph;
    n_terms += nt;
    chunks += rep;
  }
  if (mine) {
    a.pos[lane] = pos;
    if (exhausted) a.report[lane] = report;
  }
  if (lane == 0) {
    a.out[0] = chunks;
    a.out[1] = n_ph;
    a.out[2] = n_terms;
    a.out[3] = exhausted;
  }
}

// ---------------------------------------------------------------------------
// Many mixture keys (disjoint streams), e.g. cfg 5: 10k keys, Zipf weights.
// One 1024-thread CTA. The per-key pass loops run in parallel; the best-effort
// redistribution loop (chunks.py:223-229) is sequential by nature and runs on
// thread 0, but each step is O(r): for a small shortfall r the reference's
// apportion (mixtures.py:158-184) gives one unit to each of the r alive keys
// with the largest share = w / wsum * r, i.e. the first r alive keys in
// (w desc, key asc) order -- exactly, whenever (1) every share + 1e-9 < 1 (all
// floors 0, checked against a bound on wsum) and (2) the r-th and (r+1)-th
// weights are equal or separated by more than the rounding of two flops.
// Otherwise a cooperative exact apportion runs (CPython-compensated wsum,
// floors, radix select of the leftover units by (frac desc, key asc)).
constexpr int BIG_THREADS = 1024;
constexpr int BIG_MAX_KM = 16384;

struct BigArgs {
  int Km;
  long long C;
  int strict;
  long long max_chunks;
  const double* w;       // [Km] key order
  const u32* order_w;    // [Km] keys by (w desc, key asc)
  const u32* rank_w;     // [Km] position of key in order_w
  const u64* seg_pre;
  const u32* s_off;
  u64* pos;              // [Km] stream position (relative to the plan)
  u64* slen;             // [Km] scratch: stream lengths
  int* counts;           // [Km] scratch: apportion(w, C)
  int* took;             // [Km] scratch
  u32* list;             // [Km] scratch: newly dead keys
  long long* base;       // [Km] scratch (exact apportion)
  unsigned long long* fkey;  // [Km] scratch (exact apportion)
  Phase* phases;
  long long cap_phases;
  Term* terms;
  long long cap_terms;
  long long* out;
  long long* report;
  unsigned long long* stats;  // optional (MX_PLAN_STATS): section cycle / event counters
};

struct BigShared {
  double wsum, werr;  // alive weight sum (exact after big_apportion) and its error bound
  long long acc;
  int i_list, alive, slow_r, slow_d, status, flag, digit, need;
  unsigned long long thr;
  u32 hist[256];
  u32 wpart[BIG_THREADS / 32];
};

__device__ __forceinline__ u32 big_find(u32* nxt, u32 p) {
  u32 r = p;
  while (nxt[r] != r) r = nxt[r];
  while (nxt[p] != r) {
    const u32 t = nxt[p];
    nxt[p] = r;
    p = t;
  }
  return r;
}

// block sum of a per-thread long long
__device__ long long big_sum(long long v, BigShared& sh) {
  __shared__ long long s_part[BIG_THREADS / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_part[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < BIG_THREADS / 32; ++i) t += s_part[i];
    sh.acc = t;
  }
  __syncthreads();
  return sh.acc;
}

template <typename T, typename Op>
__device__ T big_reduce(T v, Op op) {  // block-wide reduction, result on every thread
  __shared__ T s_r[BIG_THREADS / 32];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = op(v, __shfl_xor_sync(MX_FULL, v, d));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) s_r[warp] = v;
  __syncthreads();
  T r = s_r[0];
  for (int x = 1; x < BIG_THREADS / 32; ++x) r = op(r, s_r[x]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// Exact apportion(w restricted to keys with !dead, total): target[m] += count.
// wsum must be CPython's Neumaier sum in key order, which is sequential. The
// sum is first taken in parallel in double-double (within ~2 ulp of
// CPython's); the floors and the leftover selection computed from it are
// accepted when they are provably insensitive to that difference (no share
// within eta of a floor boundary, the selection boundary separated by more
// than eta or a tie of identical weights). Otherwise the sequential sum runs
// (one warp, shuffle-fed) and everything is recomputed.
__device__ void big_apportion(const BigArgs& a, const unsigned char* dead, long long total, int* target,
                              BigShared& sh) {
  const int tid = threadIdx.x;
  const int Km = a.Km;
  unsigned long long t_a = clock64();
  {  // parallel double-double sum of the alive weights
    double hi = 0.0, lo = 0.0, e;
    for (int m = tid; m < Km; m += BIG_THREADS) {
      if (dead && dead[m]) continue;
      two_sum(hi, a.w[m], hi, e);
      lo += e;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const double oh = __shfl_xor_sync(MX_FULL, hi, d), ol = __shfl_xor_sync(MX_FULL, lo, d);
      two_sum(hi, oh, hi, e);
      lo = lo + ol + e;
    }
    __shared__ double s_hi[BIG_THREADS / 32], s_lo[BIG_THREADS / 32];
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) {
      s_hi[warp] = hi;
      s_lo[warp] = lo;
    }
    __syncthreads();
    if (tid == 0) {
      double H = 0.0, Lo = 0.0;
      for (int x = 0; x < BIG_THREADS / 32; ++x) {
        two_sum(H, s_hi[x], H, e);
        Lo += s_lo[x] + e;
      }
      sh.wsum = H + Lo;
    }
    __syncthreads();
  }
  bool exact = false;
  const double tot = (double)total;
  long long left = 0;
  unsigned long long thr = 0;
  int need = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt == 1) {
      exact = true;
      if (tid < 32) {  // CPython 3.12 sum(): Neumaier, keys in key order
        // warp 0: 32 weights per coalesced load, broadcast by shuffles; every
        // lane runs the same sequential recurrence
        const int lane = tid;
        double s = 0.0, c = 0.0;
        for (int b = 0; b < Km; b += 32) {
          const int m = b + lane;
          const bool live = m < Km && !(dead && dead[m]);
          const double xm = m < Km ? a.w[m] : 0.0;
          u32 mk = __ballot_sync(MX_FULL, live);
          while (mk) {
            const int t = __ffs(mk) - 1;
            mk &= mk - 1;
            const double x = __shfl_sync(MX_FULL, xm, t);
            const double tt = s + x;
            if (fabs(s) >= fabs(x)) c += (s - tt) + x;
            else c += (x - tt) + s;
            s = tt;
          }
        }
        if (lane == 0) sh.wsum = c != 0.0 ? s + c : s;
      }
      __syncthreads();
      if (a.stats && tid == 0) {
        const unsigned long long t_b = clock64();
        a.stats[12] += t_b - t_a;
        t_a = t_b;
      }
    }
    const double wsum = sh.wsum;
    long long assigned = 0;
    bool unstable = false;
    double smax = 0.0;
    for (int m = tid; m < Km; m += BIG_THREADS) {
      if (dead && dead[m]) {
        a.base[m] = 0;
        a.fkey[m] = ~0ull;
        continue;
      }
      const double share = a.w[m] / wsum * tot;
      const double s9 = share + 1e-9;
      const long long b = (long long)s9;
      double fr = share - (double)b;
      if (!exact) {
        const double eta = fabs(share) * 4e-14 + 1e-290;
        unstable |= (s9 - (double)b) < eta || ((double)b + 1.0 - s9) < eta || (fr != 0.0 && fabs(fr) < eta);
        smax = share > smax ? share : smax;
      }
      fr = fr > 0.0 ? fr : 0.0;
      a.base[m] = b;
      a.fkey[m] = ~(unsigned long long)__double_as_longlong(fr);  // larger frac -> smaller key
      assigned += b;
    }
    if (!exact && __syncthreads_or(unstable)) continue;
    left = total - big_sum(assigned, sh);
    thr = 0;
    need = 0;
    if (left > 0) {  // radix select: the left-th smallest (fkey, key) among alive keys
      unsigned long long prefix = 0, mask = 0;
      if (tid == 0) sh.need = (int)left;
      for (int shift = 56; shift >= 0; shift -= 8) {
        for (int d = tid; d < 256; d += BIG_THREADS) sh.hist[d] = 0;
        __syncthreads();
        for (int m = tid; m < Km; m += BIG_THREADS) {
          if (dead && dead[m]) continue;
          const unsigned long long f = a.fkey[m];
          if ((f & mask) == prefix) atomicAdd(&sh.hist[(f >> shift) & 255], 1u);
        }
        __syncthreads();
        if (tid < 32) {  // warp 0: which digit holds the need-th key (8 bins per lane + warp scan)
          const int nd = sh.need;
          u32 c8[8], sum8 = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            c8[q] = sh.hist[tid * 8 + q];
            sum8 += c8[q];
          }
          const u32 inc = warp_incl_scan(sum8);
          const u32 exc = inc - sum8;
          const bool here = (int)exc < nd && (int)inc >= nd;
          if (here) {
            u32 cum = exc;
            int dg = tid * 8 + 7;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if ((int)(cum + c8[q]) >= nd) {
                dg = tid * 8 + q;
                break;
              }
              cum += c8[q];
            }
            sh.digit = dg;
            sh.need = nd - (int)cum;
          }
        }
        __syncthreads();
        prefix |= (unsigned long long)sh.digit << shift;
        mask |= 0xffull << shift;
        __syncthreads();
      }
      thr = prefix;
      need = sh.need;  // how many keys with fkey == thr (lowest key first) get a unit
    }
    if (exact || left <= 0) break;
    // certificate of the leftover selection under the wsum uncertainty
    const double eta_f = big_reduce(smax, [](double x, double y) { return x > y ? x : y; }) * 4e-14 + 1e-290;
    unsigned long long prev = 0, next = ~0ull;  // nearest fkeys strictly below / above thr
    int grp = 0;
    double wmin = 1e308, wmax = -1e308;
    for (int m = tid; m < Km; m += BIG_THREADS) {
      if (dead && dead[m]) continue;
      const unsigned long long f = a.fkey[m];
      if (f < thr) prev = f > prev ? f : prev;
      else if (f > thr) next = f < next ? f : next;
      else {
        ++grp;
        wmin = a.w[m] < wmin ? a.w[m] : wmin;
        wmax = a.w[m] > wmax ? a.w[m] : wmax;
      }
    }
    prev = big_reduce(prev, [](unsigned long long x, unsigned long long y) { return x > y ? x : y; });
    next = big_reduce(next, [](unsigned long long x, unsigned long long y) { return x < y ? x : y; });
    grp = big_reduce(grp, [](int x, int y) { return x + y; });
    wmin = big_reduce(wmin, [](double x, double y) { return x < y ? x : y; });
    wmax = big_reduce(wmax, [](double x, double y) { return x > y ? x : y; });
    auto frac_of = [](unsigned long long f) { return __longlong_as_double((long long)~f); };
    const double f_thr = frac_of(thr);
    bool ok = next == ~0ull || f_thr - frac_of(next) > eta_f;
    if (need < grp) {  // the tie group is split by key order: it must tie in CPython too
      ok = ok && (f_thr == 0.0 || wmin == wmax);
      ok = ok && (thr == 0 || prev == 0 || frac_of(prev) - f_thr > eta_f || prev == thr);
    }
    if (ok) break;
  }
  if (a.stats && tid == 0) {
    const unsigned long long t_b = clock64();
    a.stats[13] += t_b - t_a;
    t_a = t_b;
    if (exact) a.stats[14] += 1;
  }
  // apply: base + 1 for fkey < thr, and the first `need` keys (in key order) with fkey == thr
  int taken = 0;  // running count of equal keys before this round
  for (int b0 = 0; b0 < Km; b0 += BIG_THREADS) {
    const int m = b0 + tid;
    bool eq = false;
    long long add = 0;
    if (m < Km && !(dead && dead[m])) {
      add = a.base[m];
      if (left > 0) {
        const unsigned long long f = a.fkey[m];
        if (f < thr) add += 1;
        eq = f == thr;
      }
    }
    // ordered rank among equal keys in this round
    const u32 bal = __ballot_sync(MX_FULL, eq);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) sh.wpart[warp] = __popc(bal);
    __syncthreads();
    int before = 0;
    for (int x = 0; x < warp; ++x) before += sh.wpart[x];
    int total_eq = 0;
    for (int x = 0; x < BIG_THREADS / 32; ++x) total_eq += sh.wpart[x];
    const int rank = taken + before + __popc(bal & ((1u << lane) - 1));
    if (eq && rank < need) add += 1;
    if (m < Km && add) target[m] += (int)add;
    taken += total_eq;
    __syncthreads();
  }
  __syncthreads();
}

// MX_PLAN_STATS: thread 0 accumulates cycles per section into a.stats
#define BIG_TICK(slot)                                       \
  do {                                                       \
    if (a.stats && tid == 0) {                               \
      const unsigned long long now_ = clock64();             \
      a.stats[slot] += now_ - tick_;                         \
      tick_ = now_;                                          \
    }                                                        \
  } while (0)

__global__ void __launch_bounds__(BIG_THREADS) plan_big_kernel(BigArgs a, int stage_w) {
  unsigned long long tick_ = clock64();
  extern __shared__ __align__(16) unsigned char big_smem[];
  __shared__ BigShared sh;
  __shared__ long long s_min[BIG_THREADS / 32];
  const int Km = a.Km, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int* rem = reinterpret_cast<int*>(big_smem);                   // [Km]
  u32* nxt = reinterpret_cast<u32*>(big_smem + 4 * (size_t)Km);  // [Km+1] skip list over order_w
  unsigned char* dead = big_smem + 8 * (size_t)Km + 4;           // [Km] 1 dead, 2 newly dead this pass
  if (stage_w) {  // weights + weight order in shared memory: the sequential redistribution
    const size_t wo = (9 * (size_t)Km + 4 + 15) & ~(size_t)15;   // steps read them one by one
    double* sw = reinterpret_cast<double*>(big_smem + wo);
    u32* sow = reinterpret_cast<u32*>(big_smem + wo + 8 * (size_t)Km);
    for (int m = tid; m < Km; m += BIG_THREADS) {
      sw[m] = a.w[m];
      sow[m] = a.order_w[m];
    }
    a.w = sw;
    a.order_w = sow;
    __syncthreads();
  }
  for (int m = tid; m < Km; m += BIG_THREADS) {
    a.slen[m] = a.seg_pre[a.s_off[m + 1] + m];
    a.counts[m] = 0;
    a.pos[m] = 0;
  }
  __syncthreads();
  big_apportion(a, nullptr, a.C, a.counts, sh);  // counts = apportion(weights, chunk_size)
  const double wsum_all = sh.wsum;                // CPython sum over all keys
  __syncthreads();
  long long chunks = 0, n_ph = 0, n_terms = 0, exhausted = 0;
  while (chunks < a.max_chunks && n_ph < a.cap_phases && a.cap_terms - n_terms >= Km) {
    // ---------------- simulate one generate() at count level (chunks.py:214-231)
    for (int m = tid; m < Km; m += BIG_THREADS) {
      rem[m] = a.counts[m];
      dead[m] = 0;
      a.took[m] = 0;
    }
    for (int p = tid; p <= Km; p += BIG_THREADS) nxt[p] = (u32)p;
    if (tid == 0) {
      sh.wsum = wsum_all;
      sh.werr = wsum_all * 1e-15;
      sh.alive = Km;
      sh.status = 0;  // 0 running, 2 None
    }
    __syncthreads();
    while (true) {
      // one pass over the keys with open counts
      int any_rem = 0, any_new = 0;
      for (int m = tid; m < Km; m += BIG_THREADS) {
        int r = rem[m];
        if (r <= 0) continue;
        const long long avail = (long long)(a.slen[m] - a.pos[m]) - a.took[m];
        const int g = r < avail ? r : (int)(avail > 0 ? avail : 0);
        a.took[m] += g;
        r -= g;
        rem[m] = r;
        any_rem |= r > 0;
        if (g == 0) {  // found nothing with an open count
          dead[m] = 2;
          any_new = 1;
        }
      }
      any_rem = __syncthreads_or(any_rem);
      any_new = __syncthreads_or(any_new);
      BIG_TICK(0);
      if (a.stats && tid == 0) a.stats[8] += 1;
      if (!any_new) {
        if (!any_rem) break;  // chunk complete
        continue;
      }
      if (a.strict) {
        for (int m = tid; m < Km; m += BIG_THREADS) a.report[m] = rem[m];
        if (tid == 0) sh.status = 2;
        __syncthreads();
        break;
      }
      // newly dead keys in key order
      int n_list = 0;
      for (int b0 = 0; b0 < Km; b0 += BIG_THREADS) {
        const int m = b0 + tid;
        const bool nd = m < Km && dead[m] == 2;
        const u32 bal = __ballot_sync(MX_FULL, nd);
        if (lane == 0) sh.wpart[warp] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int x = 0; x < BIG_THREADS / 32; ++x) {
          if (x < warp) before += sh.wpart[x];
          tot += sh.wpart[x];
        }
        if (nd) {
          a.list[n_list + before + __popc(bal & ((1u << lane) - 1))] = (u32)m;
          dead[m] = 0;  // becomes dead when the redistribution loop reaches it
        }
        n_list += tot;
        __syncthreads();
      }
      if (tid == 0) sh.i_list = 0;
      __syncthreads();
      BIG_TICK(1);
      if (a.stats && tid == 0) a.stats[9] += n_list;
      while (true) {
        if (tid == 0) {
          sh.flag = 0;
          double wsum = sh.wsum, werr = sh.werr;
          int alive = sh.alive;
          int i = sh.i_list;
          // the next dead key and its weight rank are loaded one event ahead
          u32 d_nx = i < n_list ? a.list[i] : 0u;
          u32 rk_nx = i < n_list ? a.rank_w[d_nx] : 0u;
          for (; i < n_list; ++i) {
            const u32 d = d_nx, rk = rk_nx;
            if (i + 1 < n_list) {
              d_nx = a.list[i + 1];
              rk_nx = a.rank_w[d_nx];
            }
            dead[d] = 1;
            nxt[rk] = rk + 1;  // unlink from the weight order
            --alive;
            wsum -= a.w[d];
            werr += fabs(wsum) * 2.3e-16;
            if (alive == 0) {
              sh.status = 2;
              break;
            }
            const int r = rem[d];
            if (r > 0) {
              // fast path certificate (see above)
              const u32 p1 = big_find(nxt, 0);
              const double w1 = a.w[a.order_w[p1]];
              const double wlo = (wsum - werr) * (1.0 - 1e-14);
              bool ok = wlo > 0.0 && w1 / wlo * (double)r * (1.0 + 1e-14) + 1e-9 < 1.0 - 1e-12;
              u32 p = p1, last = p1;
              for (int j = 0; ok && j < r; ++j) {
                if (p >= (u32)Km) {
                  ok = false;
                  break;
                }
                last = p;
                p = big_find(nxt, p + 1);
              }
              if (ok && p < (u32)Km) {  // selection boundary separated (or an exact tie)?
                const double wr = a.w[a.order_w[last]], wq = a.w[a.order_w[p]];
                ok = wr == wq || wr > wq * (1.0 + 4e-15);
              }
              if (!ok) {
                sh.flag = 1;
                sh.slow_r = r;
                sh.slow_d = (int)d;
                break;
              }
              p = p1;
              for (int j = 0; j < r; ++j) {
                rem[a.order_w[p]] += 1;
                p = big_find(nxt, p + 1);
              }
            }
            rem[d] = 0;
          }
          sh.i_list = i;
          sh.wsum = wsum;
          sh.werr = werr;
          sh.alive = alive;
        }
        __syncthreads();
        BIG_TICK(2);
        if (sh.status == 2 || !sh.flag) break;
        big_apportion(a, dead, sh.slow_r, rem, sh);  // exact general case; sets sh.wsum exactly
        BIG_TICK(3);
        if (a.stats && tid == 0) a.stats[10] += 1;
        if (tid == 0) {
          rem[sh.slow_d] = 0;
          sh.i_list += 1;
          sh.werr = sh.wsum * 1e-15;
        }
        __syncthreads();
      }
      if (sh.status == 2) {
        for (int m = tid; m < Km; m += BIG_THREADS) a.report[m] = rem[m];
        __syncthreads();
        break;
      }
    }
    __syncthreads();
    if (sh.status == 2) {  // None: the failed attempt's takes stay consumed
      for (int m = tid; m < Km; m += BIG_THREADS) a.pos[m] += (u64)a.took[m];
      exhausted = 1;
      break;
    }
    // ---------------- the chunk repeats while every key can serve its take
    long long rep = a.max_chunks - chunks;
    {
      long long my = rep;
      for (int m = tid; m < Km; m += BIG_THREADS) {
        const int t = a.took[m];
        if (t <= 0) continue;
        const long long r = (long long)(a.slen[m] - a.pos[m]) / t;
        my = r < my ? r : my;
      }
      for (int d = 16; d > 0; d >>= 1) {
        const long long o = __shfl_xor_sync(MX_FULL, my, d);
        my = o < my ? o : my;
      }
      if (lane == 0) s_min[warp] = my;
      __syncthreads();
      for (int i = 0; i < BIG_THREADS / 32; ++i) rep = s_min[i] < rep ? s_min[i] : rep;
      __syncthreads();
    }
    if (rep < 1) rep = 1;
    // terms: keys with a take, in key order
    long long nt = 0;
    for (int b0 = 0; b0 < Km; b0 += BIG_THREADS) {
      const int m = b0 + tid;
      const bool has = m < Km && a.took[m] > 0;
      const u32 bal = __ballot_sync(MX_FULL, has);
      if (lane == 0) sh.wpart[warp] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int x = 0; x < BIG_THREADS / 32; ++x) {
        if (x < warp) before += sh.wpart[x];
        tot += sh.wpart[x];
      }
      if (has) {
        Term& tm = a.terms[n_terms + nt + before + __popc(bal & ((1u << lane) - 1))];
        tm.m = (u32)m;
        tm.stream = (u32)m;
        tm.base = a.pos[m];
        tm.len = (u64)a.took[m];
        tm.stride = (u64)a.took[m];
        a.pos[m] += (u64)a.took[m] * (u64)rep;
      }
      nt += tot;
      __syncthreads();
    }
    BIG_TICK(4);
    if (a.stats && tid == 0) a.stats[11] += 1;
    if (tid == 0) {
      Phase& ph = a.phases[n_ph];
      ph.chunk_begin = chunks;
      ph.n_chunks = rep;
      ph.term_begin = n_terms;
      ph.n_terms = nt;
    }
    ++n_ph;
    n_terms += nt;
    chunks += rep;
    __syncthreads();
  }
  if (tid == 0) {
    a.out[0] = chunks;
    a.out[1] = n_ph;
    a.out[2] = n_terms;
    a.out[3] = exhausted;
  }
}

// arbitrary mode: one stream, chunk k = [k*C, (k+1)*C) clipped
__global__ void plan_arbitrary_kernel(const u64* seg_pre, long long nseg, long long C, long long max_chunks,
                                      Phase* phases, Term* terms, long long* out, u64* pos) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  u64 total = seg_pre[nseg];
  const long long n_avail = (long long)((total + (u64)C - 1) / (u64)C);
  long long n = n_avail < max_chunks ? n_avail : max_chunks;
  const long long exhausted = n_avail < max_chunks ? 1 : 0;  // one more call would return None
  long long full = (long long)(total / (u64)C);
  if (full > n) full = n;
  long long np = 0, nt = 0;
  if (full > 0) {
    phases[np] = Phase{0, full, nt, 1};
    terms[nt] = Term{0, 0, 0, (u64)C, (u64)C};
    ++np; ++nt;
  }
  if (n > full) {  // short tail chunk
    u64 b = (u64)full * (u64)C;
    phases[np] = Phase{full, 1, nt, 1};
    terms[nt] = Term{0, 0, b, total - b, 0};
    ++np; ++nt;
  }
  u64 used = (u64)full * (u64)C;
  if (n > full) used = total;
  pos[0] = used;
  out[0] = n;
  out[1] = np;
  out[2] = nt;
  out[3] = exhausted;
}

// ------------------------------------------------------------------ emission
struct EmitArgs {
  const Phase* phases;
  long long n_phases;
  const Term* terms;
  const u64* pair_pre;  // [n_phases+1] pair prefix
  // streams
  const u32* s_off;
  const u32* seg_comp;
  const u64* seg_lo;
  const u64* seg_pre;
  int arbitrary;
  // cursor layout
  const u32* key_blk_first;
  const u32* blk_first;
  const u32* civ;
  const u32* cfile;   // iv_file / iv_start in cursor order
  const u32* cstart;
  const u64* ccum;
  const u32* iv_start;
  const u32* iv_end;
  const u32* iv_file;
  // sharded (hybrid) index: cut only this rank's intervals (shard.cu);
  // lstart[r] = stream offset (ccum) of the r-th local cursor position
  const u32* lcnt;
  const u32* lpos;
  const u64* lstart;
};

__device__ __forceinline__ long long ub_u64(const u64* v, long long lo, long long hi, u64 x) {
  // first index in [lo, hi) with v[idx] > x
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (v[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int phase_of_pair(const EmitArgs& a, u64 pair) {
  long long lo = 0, hi = a.n_phases;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (a.pair_pre[mid + 1] <= pair) lo = mid + 1; else hi = mid;
  }
  return (int)lo;
}

// Walk the stream range of term `tm` for the kr-th chunk of its phase: the
// intervals (in cursor order) it cuts. WRITE=false: count pieces; WRITE=true:
// sink(i, mixture key, file index, start, end) for the i-th piece.
// WRITE with lanes > 1: the pieces are split over `lanes` cooperating
// threads (piece t by lane t % lanes); every lane returns the full count.
template <bool WRITE, typename Sink>
__device__ u64 walk_term(const EmitArgs& a, const Term& tm, long long kr, Sink sink, int lane = 0, int lanes = 1) {
  const u32 s = tm.stream;
  const long long sb = a.s_off[s], se = a.s_off[s + 1];
  const u64* pre = a.seg_pre + s;  // stream s prefix lives at seg_pre[i + s]
  u64 x = tm.base + (u64)kr * tm.stride;
  u64 y = x + tm.len;
  const u64 send = pre[se];
  if (y > send) y = send;
  u64 n = 0;
  if (x >= y) return 0;
  long long i = ub_u64(pre, sb, se, x) - 1;  // segment containing x
  while (x < y) {
    const u32 c = a.seg_comp[i];
    const u64 seg_start = pre[i], seg_end = pre[i + 1];
    const u64 lo_abs = a.seg_lo[i] + (x - seg_start);
    const u64 hi_abs = a.seg_lo[i] + ((y < seg_end ? y : seg_end) - seg_start);
    const long long ib = a.blk_first[a.key_blk_first[c]];
    const long long ie = a.blk_first[a.key_blk_first[c + 1]];
    const u64 cb = a.ccum[ib];
    if (a.lcnt) {  // sharded: search only this rank's intervals of component c
      const long long r0 = a.lcnt[ib], r1 = a.lcnt[ie];
      // first local interval ending after lo, first starting at or after hi
      long long ra = ub_u64(a.lstart, r0, r1, cb + lo_abs) - 1;
      if (ra < r0) ra = r0;
      else if (a.ccum[a.lpos[ra] + 1] <= cb + lo_abs) ++ra;
      const long long rb = ub_u64(a.lstart, r0, r1, cb + hi_abs - 1);
      if (!WRITE) {
        if (rb > ra) n += (u64)(rb - ra);
      } else {
        for (long long r = ra + lane; r < rb; r += lanes) {
          const long long jj = a.lpos[r];
          const u64 off = a.ccum[jj] - cb;
          const u64 len = a.ccum[jj + 1] - a.ccum[jj];
          const u64 from = lo_abs > off ? lo_abs : off;
          const u64 to = hi_abs < off + len ? hi_abs : off + len;
          const u32 st0 = a.cstart[jj];
          sink(n + (u64)(r - ra), a.arbitrary ? c : tm.m, a.cfile[jj], st0 + (u32)(from - off), st0 + (u32)(to - off));
        }
        if (rb > ra) n += (u64)(rb - ra);
      }
      x = seg_end < y ? seg_end : y;
      ++i;
      continue;
    }
    long long j = ub_u64(a.ccum, ib, ie, cb + lo_abs) - 1;
    const long long j1 = ub_u64(a.ccum, ib, ie, cb + hi_abs - 1) - 1;
    if (WRITE) {
      for (long long jj = j + lane; jj <= j1; jj += lanes) {
        const u64 off = a.ccum[jj] - cb;
        const u64 len = a.ccum[jj + 1] - a.ccum[jj];
        const u64 from = lo_abs > off ? lo_abs : off;
        const u64 to = hi_abs < off + len ? hi_abs : off + len;
        const u32 st0 = a.cstart[jj];
        sink(n + (u64)(jj - j), a.arbitrary ? c : tm.m, a.cfile[jj], st0 + (u32)(from - off), st0 + (u32)(to - off));
      }
    }
    n += (u64)(j1 - j + 1);
    x = seg_end < y ? seg_end : y;
    ++i;
  }
  return n;
}

// Walk the stream range of one (chunk, term) pair. WRITE=false: count pieces.
template <bool WRITE>
__device__ u64 walk_pair(const EmitArgs& a, u64 pair, long long* chunk_out, u32* pm, u32* pf, u32* ps, u32* pe,
                         u64 out_base, int lane = 0, int lanes = 1) {
  const int p = phase_of_pair(a, pair);
  const Phase ph = a.phases[p];
  const u64 local = pair - a.pair_pre[p];
  const long long kr = (long long)(local / (u64)ph.n_terms);
  const Term tm = a.terms[ph.term_begin + (long long)(local % (u64)ph.n_terms)];
  if (chunk_out) *chunk_out = ph.chunk_begin + kr;
  if (WRITE) {
    return walk_term<true>(
        a, tm, kr,
        [&](u64 i, u32 m, u32 f, u32 s0, u32 e0) {
          pm[out_base + i] = m;
          pf[out_base + i] = f;
          ps[out_base + i] = s0;
          pe[out_base + i] = e0;
        },
        lane, lanes);
  }
  return walk_term<false>(a, tm, kr, [](u64, u32, u32, u32, u32) {});
}

__global__ void emit_count_kernel(EmitArgs a, u64 n_pairs, u64* pair_cnt) {
  u64 pr = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (pr >= n_pairs) return;
  pair_cnt[pr] = walk_pair<false>(a, pr, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
}

// Same, with each warp's pieces staged in shared memory: the 32 pairs of a
// warp own one contiguous output range [pair_off[first], pair_off[last+1]),
// so the lanes write their pieces there as 16-byte records and the warp then
// stores the range coalesced into the four piece arrays (direct per-lane
// stores put 32 lanes ~5 records apart on every store instruction). Warps
// with a long pair (cut later by emit_write_warp_kernel) or a range above
// EW_CAP store directly.
constexpr int EW_THREADS = 128;
constexpr int EW_CAP = 640;
// sort_terms (mode-0 plans: one term per mixture key and chunk, terms in key
// order): each thread also sorts its pair's pieces by (file, start) in the
// stage, so every chunk comes out in the reference's (mixture key, file,
// start) order without the per-chunk normalisation; flags |= 1 when a piece
// bypassed the sort (long pair, unstaged warp), |= 2 when two sorted pieces
// are contiguous (a merge the per-chunk pass must do).
__global__ void __launch_bounds__(EW_THREADS) emit_write_staged_kernel(EmitArgs a, u64 n_pairs, const u64* pair_off,
                                                                       u32* pm, u32* pf, u32* ps, u32* pe,
                                                                       u32* long_list, u32* long_cnt, u32 warp_min,
                                                                       int sort_terms, u32* flags) {
  __shared__ uint4 s_rec[EW_THREADS / 32][EW_CAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 pr = blockIdx.x * (u64)EW_THREADS + threadIdx.x;
  const u64 first = blockIdx.x * (u64)EW_THREADS + warp * 32;
  if (first >= n_pairs) return;  // warp-uniform
  const bool valid = pr < n_pairs;
  const u64 lo_i = valid ? pair_off[pr] : 0, hi_i = valid ? pair_off[pr + 1] : 0;
  const bool is_long = valid && hi_i - lo_i > warp_min;
  if (is_long) long_list[atomicAdd(long_cnt, 1u)] = (u32)pr;
  const u64 last = first + 31 < n_pairs ? first + 31 : n_pairs - 1;
  const u64 w_lo = pair_off[first], w_hi = pair_off[last + 1];
  const bool staged = !__any_sync(MX_FULL, is_long) && w_hi - w_lo <= (u64)EW_CAP;
  if (!staged) {
    if (valid && !is_long) {
      walk_pair<true>(a, pr, nullptr, pm, pf, ps, pe, lo_i);
      if (sort_terms && hi_i - lo_i > 1) long_list[atomicAdd(long_cnt + 1, 1u) + n_pairs] = (u32)pr;  // sort later
    }
    return;
  }
  uint4* rec = s_rec[warp];
  if (valid) {
    const u64 base = lo_i - w_lo;
    const int p = phase_of_pair(a, pr);
    const Phase php = a.phases[p];
    const u64 local = pr - a.pair_pre[p];
    const long long kr = (long long)(local / (u64)php.n_terms);
    const Term tm = a.terms[php.term_begin + (long long)(local % (u64)php.n_terms)];
    walk_term<true>(a, tm, kr, [&](u64 i, u32 m, u32 f, u32 s0, u32 e0) { rec[base + i] = make_uint4(m, f, s0, e0); },
                    0, 1);
    if (sort_terms) {  // this pair's pieces by (file, start): <= 8 in registers, more by sort_pairs_kernel
      const int n = (int)(hi_i - lo_i);
      if (n > 8) {
        long_list[atomicAdd(long_cnt + 1, 1u) + n_pairs] = (u32)pr;
      } else if (n > 1) {
        uint4* r = rec + base;
        unsigned long long k[8];
        u32 e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 v = i < n ? r[i] : make_uint4(0u, ~0u, ~0u, 0u);
          k[i] = ((unsigned long long)v.y << 32) | v.z;
          e[i] = v.w;
        }
        // Batcher odd-even merge sort network for 8 keys (19 comparators)
        auto cx = [&](int a, int b) {
          const bool sw = k[b] < k[a];
          const unsigned long long ka = k[a], kb = k[b];
          const u32 ea = e[a], eb = e[b];
          k[a] = sw ? kb : ka;
          k[b] = sw ? ka : kb;
          e[a] = sw ? eb : ea;
          e[b] = sw ? ea : eb;
        };
        cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
        cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
        cx(1, 2); cx(5, 6); cx(0, 4); cx(3, 7);
        cx(1, 5); cx(2, 6);
        cx(1, 4); cx(3, 6);
        cx(2, 4); cx(3, 5);
        cx(3, 4);
        const u32 m = r[0].x;
        bool merge = false;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < n) {
            r[i] = make_uint4(m, (u32)(k[i] >> 32), (u32)k[i], e[i]);
            if (i > 0) merge |= (k[i] >> 32) == (k[i - 1] >> 32) && (u32)k[i] == e[i - 1];
          }
        }
        if (merge) atomicOr(flags, 2u);
      }
    }
  }
  __syncwarp();
  const int cnt = (int)(w_hi - w_lo);
  for (int i = lane; i < cnt; i += 32) {
    const uint4 r = rec[i];
    pm[w_lo + i] = r.x;
    pf[w_lo + i] = r.y;
    ps[w_lo + i] = r.z;
    pe[w_lo + i] = r.w;
  }
}

// one warp per long pair: the lanes cut its intervals in parallel
__global__ void __launch_bounds__(256) emit_write_warp_kernel(EmitArgs a, const u64* pair_off, u32* pm, u32* pf,
                                                              u32* ps, u32* pe, const u32* long_list,
                                                              const u32* long_cnt) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long n = *long_cnt;
  for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n; w += warps) {
    const u64 pr = long_list[w];
    walk_pair<true>(a, pr, nullptr, pm, pf, ps, pe, pair_off[pr], lane, 32);
  }
}

// first pair of every chunk (+ sentinel) -> piece range per chunk
// mode-0 sorted emission: long pairs (> 32 pieces, cut by a warp) -- one CTA
// each sorts its pieces by (file, start) in shared memory (<= SP_CAP) and
// flags merges; larger ones flag the per-chunk path
constexpr int SP_CAP = 2048;
__global__ void __launch_bounds__(256) sort_pairs_kernel(const u32* lists, const u32* cnts, u64 n_pairs,
                                                         const u64* pair_off, u32* pm, u32* pf, u32* ps, u32* pe,
                                                         u32* flags) {
  __shared__ uint4 sh[SP_CAP];
  const u32 n_long = cnts[0];
  for (u32 x = blockIdx.x; x < n_long; x += gridDim.x) {
    const u32 pr = lists[x];
    const u64 o0 = pair_off[pr];
    const u32 n = (u32)(pair_off[pr + 1] - o0);
    if (n > SP_CAP) {
      if (threadIdx.x == 0) atomicOr(flags, 1u);
      continue;
    }
    u32 np = 1;
    while (np < n) np <<= 1;
    for (u32 i = threadIdx.x; i < np; i += blockDim.x)
      sh[i] = i < n ? make_uint4(pm[o0 + i], pf[o0 + i], ps[o0 + i], pe[o0 + i]) : make_uint4(~0u, ~0u, ~0u, ~0u);
    __syncthreads();
    for (u32 kk = 2; kk <= np; kk <<= 1)
      for (u32 j = kk >> 1; j > 0; j >>= 1) {
        for (u32 i = threadIdx.x; i < np; i += blockDim.x) {
          const u32 l = i ^ j;
          if (l > i) {
            const uint4 p = sh[i], q = sh[l];
            const bool gt = p.y != q.y ? p.y > q.y : p.z > q.z;
            if (gt == ((i & kk) == 0)) {
              sh[i] = q;
              sh[l] = p;
            }
          }
        }
        __syncthreads();
      }
    bool merge = false;
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const uint4 r = sh[i];
      if (i > 0) merge |= sh[i - 1].y == r.y && sh[i - 1].w == r.z;
      pm[o0 + i] = r.x;
      pf[o0 + i] = r.y;
      ps[o0 + i] = r.z;
      pe[o0 + i] = r.w;
    }
    if (__syncthreads_or(merge) && threadIdx.x == 0) atomicOr(flags, 2u);
  }
}

// pairs of 9..32 pieces (and unstaged warps' pairs): one warp each, register
// bitonic sort of (file, start) across the lanes
__global__ void __launch_bounds__(256) sort_pairs_warp_kernel(const u32* lists, const u32* cnts, u64 n_pairs,
                                                              const u64* pair_off, u32* pm, u32* pf, u32* ps,
                                                              u32* pe, u32* flags) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long n_uns = cnts[1];
  for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_uns; w += warps) {
    const u32 pr = lists[n_pairs + w];
    const u64 o0 = pair_off[pr];
    const u32 n = (u32)(pair_off[pr + 1] - o0);  // <= 32 (longer pairs are on the long list)
    const bool ok = (u32)lane < n;
    unsigned long long key = ok ? ((unsigned long long)pf[o0 + lane] << 32) | ps[o0 + lane] : ~0ull;
    u32 en = ok ? pe[o0 + lane] : 0u;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const unsigned long long ok2 = __shfl_xor_sync(MX_FULL, key, j);
        const u32 oe = __shfl_xor_sync(MX_FULL, en, j);
        const bool lower = (lane & j) == 0, up = (lane & kk) == 0;
        const bool take = (lower == up) ? ok2 < key : ok2 > key;
        if (take) {
          key = ok2;
          en = oe;
        }
      }
    }
    const unsigned long long pk = __shfl_up_sync(MX_FULL, key, 1);
    const u32 pen = __shfl_up_sync(MX_FULL, en, 1);
    const bool merge = ok && lane > 0 && (pk >> 32) == (key >> 32) && pen == (u32)key;
    if (ok) {
      pf[o0 + lane] = (u32)(key >> 32);
      ps[o0 + lane] = (u32)key;
      pe[o0 + lane] = en;
    }
    if (__any_sync(MX_FULL, merge) && lane == 0) atomicOr(flags, 2u);
  }
}

__global__ void chunk_pieces_kernel(EmitArgs a, long long n_chunks, const u64* pair_off, u64 n_pairs,
                                    u64* chunk_piece_off) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k > n_chunks) return;
  if (k == n_chunks) {
    chunk_piece_off[k] = pair_off[n_pairs];
    return;
  }
  long long lo = 0, hi = a.n_phases;
  while (lo < hi) {  // last phase with chunk_begin <= k
    long long mid = (lo + hi) >> 1;
    if (a.phases[mid].chunk_begin <= k) lo = mid + 1; else hi = mid;
  }
  const int p = (int)lo - 1;
  const Phase ph = a.phases[p];
  u64 first = a.pair_pre[p] + (u64)(k - ph.chunk_begin) * (u64)ph.n_terms;
  chunk_piece_off[k] = pair_off[first];
}

// ---- per-chunk sort (mixture key, file, start) + merge of adjacent ranges
__device__ __forceinline__ bool piece_less(uint4 x, uint4 y) {
  if (x.x != y.x) return x.x < y.x;
  if (x.y != y.y) return x.y < y.y;
  return x.z < y.z;
}

// sorts s[0..n) (n <= cap, padded to a power of two with max sentinels),
// then merges in place; returns merged count. Called by `nt` threads.
__device__ u32 sort_merge(uint4* s, u32 n, int tid, int nt, u32* s_flags) {
  u32 np2 = 1;
  while (np2 < n) np2 <<= 1;
  for (u32 i = n + tid; i < np2; i += nt) s[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
  __syncthreads();
  for (u32 k = 2; k <= np2; k <<= 1) {
    for (u32 j = k >> 1; j > 0; j >>= 1) {
      for (u32 i = tid; i < np2; i += nt) {
        u32 l = i ^ j;
        if (l > i) {
          uint4 a = s[i], b = s[l];
          bool up = (i & k) == 0;
          if (piece_less(b, a) == up) {
            s[i] = b;
            s[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // heads: not (same key, same file, contiguous); inclusive head count by a
  // blocked block-wide scan (each thread owns a contiguous run of elements)
  __shared__ u32 s_m;
  __shared__ u32 s_wsum[32];
  {
    const u32 per = (n + nt - 1) / nt;
    const u32 b = tid * per, e = b + per < n ? b + per : n;
    u32 cnt = 0;
    for (u32 i = b; i < e; ++i) {
      const bool head = i == 0 || !(s[i].x == s[i - 1].x && s[i].y == s[i - 1].y && s[i].z == s[i - 1].w);
      s_flags[i] = head ? 1u : 0u;
      cnt += head;
    }
    const int lane = tid & 31, warp = tid >> 5;
    const u32 inc = warp_incl_scan(cnt);
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const u32 x = lane < nt / 32 ? s_wsum[lane] : 0;
      const u32 xi = warp_incl_scan(x);
      if (lane < nt / 32) s_wsum[lane] = xi - x;
      if (lane == 31) s_m = xi;
    }
    __syncthreads();
    u32 run = s_wsum[warp] + inc - cnt;
    for (u32 i = b; i < e; ++i) {
      run += s_flags[i];
      s_flags[i] = run;  // inclusive head count
    }
  }
  __syncthreads();
  // compaction into the front of a second half is unsafe in place; stage ends
  uint4 mine[8];
  int cnt = 0;
  for (u32 i = tid; i < n; i += nt) {
    bool last = (i + 1 == n) || (s_flags[i + 1] != s_flags[i]);
    if (last && cnt < 8) mine[cnt++] = make_uint4(i, s_flags[i] - 1, s[i].w, 0);
  }
  __syncthreads();
  // heads: write (m, f, start) to slot; ends: patch end
  uint4 heads[8];
  int hc = 0;
  for (u32 i = tid; i < n; i += nt) {
    bool head = (i == 0) || (s_flags[i] != s_flags[i - 1]);
    if (head && hc < 8) heads[hc++] = make_uint4(s_flags[i] - 1, s[i].x, s[i].y, s[i].z);
  }
  __syncthreads();
  for (int h = 0; h < hc; ++h) s[heads[h].x] = make_uint4(heads[h].y, heads[h].z, heads[h].w, 0);
  __syncthreads();
  for (int h = 0; h < cnt; ++h) s[mine[h].y].w = mine[h].z;
  __syncthreads();
  return s_m;
}

constexpr int NM_THREADS = 256;
constexpr int NMB_THREADS = 1024;  // normalize_kernel: one compare-exchange per thread per stage at 2048
constexpr int NM_CAP = 2048;

// Chunks of more than NM_CAP pieces (e.g. iid data with chunk_size >> 2048):
// the whole CTA sorts the chunk's pieces in place in global memory with an
// ascending-only bitonic network (the first step of every merge stage
// compares i with i ^ (kk - 1)), so positions >= n act as +infinity and never
// move; then one in-place merge pass in rounds of NMB_THREADS (a merged
// range's slot never exceeds its first piece's index). `sm` is >= 8 words of
// shared scratch.
__device__ __forceinline__ bool gm_less(const u32* pm, const u32* pf, const u32* ps, u64 a, u64 b) {
  if (pm[a] != pm[b]) return pm[a] < pm[b];
  if (pf[a] != pf[b]) return pf[a] < pf[b];
  return ps[a] < ps[b];
}

__device__ u32 sort_merge_global(u64 o0, u32 n, u32* pm, u32* pf, u32* ps, u32* pe, u32* sm) {
  const u32 tid = threadIdx.x;
  u32 np = 1;
  while (np < n) np <<= 1;
  for (u32 kk = 2; kk <= np; kk <<= 1) {
    for (u32 j = kk >> 1; j > 0; j >>= 1) {
      const bool flip = j == (kk >> 1);
      for (u32 t = tid; t < np / 2; t += NMB_THREADS) {
        const u32 i = (t / j) * 2 * j + (t % j);
        const u32 l = flip ? (i | (kk - 1)) - (i & (kk - 1)) : i + j;  // flip: i ^ (kk - 1) within the block
        if (l < n && gm_less(pm, pf, ps, o0 + l, o0 + i)) {
          const u64 a = o0 + i, b = o0 + l;
          u32 x = pm[a]; pm[a] = pm[b]; pm[b] = x;
          x = pf[a]; pf[a] = pf[b]; pf[b] = x;
          x = ps[a]; ps[a] = ps[b]; ps[b] = x;
          x = pe[a]; pe[a] = pe[b]; pe[b] = x;
        }
      }
      __syncthreads();
    }
  }
  // merge: head unless same (mkey, file) as the previous piece and contiguous
  const int lane = tid & 31, warp = tid >> 5;
  u32* s_w = sm;               // [32] warp head counts
  u32* s_prev = sm + 32;       // previous round's last piece: mkey, file, end
  u32 run = 0;                 // merged ranges so far
  for (u32 b = 0; b < n; b += NMB_THREADS) {
    const u32 i = b + tid;
    const bool ok = i < n;
    u32 m = 0, f = 0, st = 0, en = 0, pmk = 0, pfl = 0, pen = 0;
    bool nxt_head = true;
    if (ok) {
      m = pm[o0 + i]; f = pf[o0 + i]; st = ps[o0 + i]; en = pe[o0 + i];
      if (i > 0 && tid == 0) { pmk = s_prev[0]; pfl = s_prev[1]; pen = s_prev[2]; }
      else if (i > 0) { pmk = pm[o0 + i - 1]; pfl = pf[o0 + i - 1]; pen = pe[o0 + i - 1]; }
      if (i + 1 < n) nxt_head = !(pm[o0 + i + 1] == m && pf[o0 + i + 1] == f && ps[o0 + i + 1] == en);
    }
    const bool head = ok && (i == 0 || !(pmk == m && pfl == f && pen == st));
    __syncthreads();  // every read of this round before any write
    if (tid == NMB_THREADS - 1 || i == n - 1) { s_prev[0] = m; s_prev[1] = f; s_prev[2] = en; }
    const u32 hb = __ballot_sync(MX_FULL, head);
    if (lane == 0) s_w[warp] = __popc(hb);
    __syncthreads();
    u32 before = 0, tot = 0;
    for (int w = 0; w < NMB_THREADS / 32; ++w) {
      const u32 c = s_w[w];
      before += w < warp ? c : 0;
      tot += c;
    }
    const u32 upto = run + before + __popc(hb & ((2u << lane) - 1u));  // heads up to and including i
    if (head) { pm[o0 + upto - 1] = m; pf[o0 + upto - 1] = f; ps[o0 + upto - 1] = st; }
    if (ok && nxt_head) pe[o0 + upto - 1] = en;  // last piece of its range
    run += tot;
    __syncthreads();
  }
  return run;
}

__global__ void __launch_bounds__(NMB_THREADS)
normalize_kernel(const u32* big_list, const u32* big_cnt, const u64* chunk_piece_off, u32* pm, u32* pf, u32* ps,
                 u32* pe, u64* merged_cnt, u32* too_big) {
  __shared__ uint4 s[NM_CAP];
  __shared__ u32 s_flags[NM_CAP];
  const u32 nbig = *big_cnt;
  for (u32 x = blockIdx.x; x < nbig; x += gridDim.x) {
    const u32 k = big_list[x];
    const u64 o0 = chunk_piece_off[k], o1 = chunk_piece_off[k + 1];
    const u32 n = (u32)(o1 - o0);
    if (n > NM_CAP) {  // too large for shared memory: sorted and merged in place in global memory
      const u32 m = sort_merge_global(o0, n, pm, pf, ps, pe, reinterpret_cast<u32*>(s));
      if (threadIdx.x == 0) merged_cnt[k] = m;
      __syncthreads();
      continue;
    }
    for (u32 i = threadIdx.x; i < n; i += NMB_THREADS) s[i] = make_uint4(pm[o0 + i], pf[o0 + i], ps[o0 + i], pe[o0 + i]);
    __syncthreads();
    u32 m = n ? sort_merge(s, n, threadIdx.x, NMB_THREADS, s_flags) : 0;
    for (u32 i = threadIdx.x; i < m; i += NMB_THREADS) {
      pm[o0 + i] = s[i].x;
      pf[o0 + i] = s[i].y;
      ps[o0 + i] = s[i].z;
      pe[o0 + i] = s[i].w;
    }
    if (threadIdx.x == 0) merged_cnt[k] = m;
    __syncthreads();
  }
}

// One thread: sort n <= 4 pieces by (mixture key, file, start) and merge
// contiguous ones in place.
__device__ __forceinline__ void normalize_tiny(u64 o0, u32 n, u32* pm, u32* pf, u32* ps, u32* pe, u64* cnt) {
  unsigned long long hi[4];
  u32 lo[4], en[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool ok = (u32)i < n;
    hi[i] = ok ? ((unsigned long long)pm[o0 + i] << 32) | pf[o0 + i] : ~0ull;
    lo[i] = ok ? ps[o0 + i] : ~0u;
    en[i] = ok ? pe[o0 + i] : ~0u;
  }
  auto cswap = [&](int a, int b) {
    if (hi[b] < hi[a] || (hi[b] == hi[a] && lo[b] < lo[a])) {
      const unsigned long long th = hi[a];
      hi[a] = hi[b];
      hi[b] = th;
      const u32 tl = lo[a];
      lo[a] = lo[b];
      lo[b] = tl;
      const u32 te = en[a];
      en[a] = en[b];
      en[b] = te;
    }
  };
  cswap(0, 1);
  cswap(2, 3);
  cswap(0, 2);
  cswap(1, 3);
  cswap(1, 2);
  u32 m = 0;
#pragma unroll
  for (u32 i = 0; i < 4; ++i) {
    if (i >= n) break;
    if (m > 0 && hi[i] == hi[m - 1] && lo[i] == en[m - 1]) {
      en[m - 1] = en[i];
    } else {
      hi[m] = hi[i];
      lo[m] = lo[i];
      en[m] = en[i];
      ++m;
    }
  }
  for (u32 i = 0; i < m; ++i) {
    pm[o0 + i] = (u32)(hi[i] >> 32);
    pf[o0 + i] = (u32)hi[i];
    ps[o0 + i] = lo[i];
    pe[o0 + i] = en[i];
  }
  *cnt = m;
}

// Thread per chunk: chunks of <= 4 pieces are normalised here (the sharded
// case has ~2-3 local pieces per chunk); the others are listed for the warp
// kernel.
__global__ void normalize_tiny_kernel(long long n_chunks, const u64* chunk_piece_off, u32* pm, u32* pf, u32* ps,
                                      u32* pe, u64* merged_cnt, u32* wide_list, u32* wide_cnt) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = k < n_chunks;
  u64 o0 = 0;
  u32 n = 0;
  if (in) {
    o0 = chunk_piece_off[k];
    n = (u32)(chunk_piece_off[k + 1] - o0);
  }
  const bool wide = in && n > 4;
  const u32 wm = __ballot_sync(MX_FULL, wide);
  u32 base = 0;
  if ((threadIdx.x & 31) == 0 && wm) base = atomicAdd(wide_cnt, (u32)__popc(wm));
  base = __shfl_sync(MX_FULL, base, 0);
  if (wide) wide_list[base + __popc(wm & ((1u << (threadIdx.x & 31)) - 1))] = (u32)k;
  else if (in) normalize_tiny(o0, n, pm, pf, ps, pe, merged_cnt + k);
}

// Chunks of <= 32 pieces (the common case): one warp per chunk, bitonic sort
// of (mixture key, file, start) across lanes with shuffles, merge by ballot.
// PACK: (mkey, file, start) fits one u64 -- mkey above file_bits + 32 bits,
// file above 32 -- so the bitonic sort moves and compares one u64 + the end
// (3 shuffles per step instead of 4, one 64-bit compare).
template <bool PACK>
__global__ void __launch_bounds__(256)
normalize_warp_kernel(const u32* wide_list, const u32* wide_cnt, const u64* chunk_piece_off, u32* pm, u32* pf,
                      u32* ps, u32* pe, u64* merged_cnt, u32* big_list, u32* big_cnt, int file_bits) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long n_wide = *wide_cnt;
  for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_wide; w += warps) {
    const long long k = wide_list[w];
    const u64 o0 = chunk_piece_off[k];
    const u32 n = (u32)(chunk_piece_off[k + 1] - o0);
    if (n > 32) {  // left to normalize_kernel
      if (lane == 0) big_list[atomicAdd(big_cnt, 1u)] = (u32)k;
      continue;
    }
    const bool ok = (u32)lane < n;
    // sort key: hi = (mkey, file), lo = start; padding sorts last
    unsigned long long hi, key;
    u32 lo, en = ok ? pe[o0 + lane] : ~0u;
    if (PACK) {
      key = ok ? ((unsigned long long)pm[o0 + lane] << (32 + file_bits)) |
                     ((unsigned long long)pf[o0 + lane] << 32) | ps[o0 + lane]
               : ~0ull;
#pragma unroll
      for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
          const unsigned long long okey = __shfl_xor_sync(MX_FULL, key, j);
          const u32 oen = __shfl_xor_sync(MX_FULL, en, j);
          const bool other_less = okey < key;
          const bool lower = (lane & j) == 0;
          const bool up = (lane & kk) == 0;
          const bool take = (lower == up) ? other_less : okey > key;
          if (take) {
            key = okey;
            en = oen;
          }
        }
      }
      hi = key >> 32;
      lo = (u32)key;
    } else {
      hi = ok ? ((unsigned long long)pm[o0 + lane] << 32) | pf[o0 + lane] : ~0ull;
      lo = ok ? ps[o0 + lane] : ~0u;
#pragma unroll
      for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
          const unsigned long long ohi = __shfl_xor_sync(MX_FULL, hi, j);
          const u32 olo = __shfl_xor_sync(MX_FULL, lo, j);
          const u32 oen = __shfl_xor_sync(MX_FULL, en, j);
          const bool other_less = ohi < hi || (ohi == hi && olo < lo);
          const bool lower = (lane & j) == 0;      // this lane keeps the smaller of the pair?
          const bool up = (lane & kk) == 0;        // ascending sub-sequence
          const bool take = (lower == up) ? other_less : !other_less && !(ohi == hi && olo == lo);
          if (take) {
            hi = ohi;
            lo = olo;
            en = oen;
          }
        }
      }
    }
    // merge: head unless same (key, file) and contiguous with the previous piece
    const unsigned long long phi = __shfl_up_sync(MX_FULL, hi, 1);
    const u32 pen = __shfl_up_sync(MX_FULL, en, 1);
    const bool head = ok && (lane == 0 || !(phi == hi && pen == lo));
    const u32 heads = __ballot_sync(MX_FULL, head);
    const u32 slot = __popc(heads & ((2u << lane) - 1u)) - 1u;  // run index of this piece
    const u32 nxt_head = __shfl_down_sync(MX_FULL, (u32)head, 1);
    const bool last = ok && ((u32)lane == n - 1 || nxt_head);
    if (head) {
      if (PACK) {
        pm[o0 + slot] = (u32)(hi >> file_bits);
        pf[o0 + slot] = (u32)(hi & ((1ull << file_bits) - 1));
      } else {
        pm[o0 + slot] = (u32)(hi >> 32);
        pf[o0 + slot] = (u32)hi;
      }
      ps[o0 + slot] = lo;
    }
    __syncwarp();
    if (last) pe[o0 + slot] = en;
    if (lane == 0) merged_cnt[k] = __popc(heads);
  }
}

// Exclusive scan of u64 counts (reduce-then-scan, scan.cuh); out[n] = total.
template <typename OUT>
struct ExclScanF {
  const u64* in;
  OUT* out;
  long long n;
  __device__ u64 value(long long i) const { return in[i]; }
  __device__ void apply(long long i, u64 ex, u64) const { out[i] = (OUT)ex; }
  __device__ void total(u64 t) const { out[n] = (OUT)t; }
};

// exclusive scan of u64 counts; out[n] = total (in == out allowed: an item is
// read and written by the same thread)
template <typename OUT>
static int excl_scan(const u64* in, long long n, OUT* out, cudaStream_t s) {
  if (n <= 0) {
    MX_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(OUT), s));
    return MX_OK;
  }
  return gs_run(n, ExclScanF<OUT>{in, out, n}, s);
}

int excl_scan_ll(const u64* in, long long n, long long* out, cudaStream_t s) { return excl_scan<long long>(in, n, out, s); }

// Dense copy of each chunk's merged ranges (one warp per chunk).
__global__ void compact_warp_kernel(long long n_chunks, const u64* chunk_piece_off, const long long* res_off,
                                    const u32* pm, const u32* pf, const u32* ps, const u32* pe, u32* rm, u32* rf,
                                    u32* rs, u32* re, bool grouped) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  if (!grouped) {  // larger chunks (single GPU): one warp per chunk
    for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n_chunks; k += warps) {
      const u64 src = chunk_piece_off[k];
      const long long dst = res_off[k], n = res_off[k + 1] - dst;
      for (long long i = lane; i < n; i += 32) {
        rm[dst + i] = pm[src + i];
        rf[dst + i] = pf[src + i];
        rs[dst + i] = ps[src + i];
        re[dst + i] = pe[src + i];
      }
    }
    return;
  }
  // a warp takes 32 consecutive chunks: each lane copies its own chunk when
  // it has <= 4 ranges, then the warp copies the larger ones together
  for (long long g = (blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; g < n_chunks;
       g += warps * 32) {
    const long long k = g + lane;
    long long n = 0, dst = 0;
    u64 src = 0;
    if (k < n_chunks) {
      src = chunk_piece_off[k];
      dst = res_off[k];
      n = res_off[k + 1] - dst;
    }
    u32 wide = __ballot_sync(MX_FULL, n > 4);
    if (n <= 4)
      for (long long i = 0; i < n; ++i) {
        rm[dst + i] = pm[src + i];
        rf[dst + i] = pf[src + i];
        rs[dst + i] = ps[src + i];
        re[dst + i] = pe[src + i];
      }
    while (wide) {
      const int l = __ffs(wide) - 1;
      wide &= wide - 1;
      const u64 s0 = __shfl_sync(MX_FULL, src, l);
      const long long d0 = __shfl_sync(MX_FULL, dst, l), n0 = __shfl_sync(MX_FULL, n, l);
      for (long long i = lane; i < n0; i += 32) {
        rm[d0 + i] = pm[s0 + i];
        rf[d0 + i] = pf[s0 + i];
        rs[d0 + i] = ps[s0 + i];
        re[d0 + i] = pe[s0 + i];
      }
    }
  }
}

// exclusive scan of merged counts -> res_off (single CTA, loops)
__global__ void offsets_kernel(long long n, const u64* cnt, long long* off) {
  __shared__ u64 s_w[32];
  __shared__ u64 s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (long long b = 0; b < n; b += blockDim.x) {
    long long i = b + threadIdx.x;
    u64 v = i < n ? cnt[i] : 0;
    u64 inc = warp_incl_scan(v);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u64 x = lane < nw ? s_w[lane] : 0;
      u64 xi = warp_incl_scan(x);
      if (lane < nw) s_w[lane] = xi - x;
    }
    __syncthreads();
    u64 ex = s_carry + s_w[warp] + inc - v;
    if (i < n) off[i] = (long long)ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[n] = (long long)s_carry;
}

__global__ void compact_kernel(long long n_chunks, const u64* chunk_piece_off, const long long* res_off, const u32* pm,
                               const u32* pf, const u32* ps, const u32* pe, u32* rm, u32* rf, u32* rs, u32* re) {
  for (long long k = blockIdx.x; k < n_chunks; k += gridDim.x) {
    const u64 src = chunk_piece_off[k];
    const long long dst = res_off[k], n = res_off[k + 1] - res_off[k];
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      rm[dst + i] = pm[src + i];
      rf[dst + i] = pf[src + i];
      rs[dst + i] = ps[src + i];
      re[dst + i] = pe[src + i];
    }
  }
}

// chunk seeds: derive_seed(job_seed, "chunk", chunk_id)  (chunks.py:188)
__global__ void chunk_seed_kernel(long long n, long long first_id, const uint8_t* prefix, int prefix_len, u64* seeds,
                                  long long* ids) {
  __shared__ uint8_t s_pre[96];
  for (int i = threadIdx.x; i < prefix_len && i < 96; i += blockDim.x) s_pre[i] = prefix[i];
  __syncthreads();
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long id = first_id + k;
  // message = prefix || len8BE(len(str(id))) || str(id)   (seeding.py:18-28)
  u64 v = (u64)id;
  int dl = 1;
  for (u64 t = v; t >= 10; t /= 10) ++dl;
  if (prefix_len + 8 + dl <= 128 && prefix_len <= 96) {
    u64 dec[3] = {0, 0, 0};  // str(id) as bytes, 8 per word (registers: constant indices below)
    {
      u64 t = v;
      for (int pos = dl - 1; pos >= 0; --pos) {
        const u64 c = (u64)('0' + t % 10);
        t /= 10;
        if (pos < 8) dec[0] |= c << (8 * pos);
        else if (pos < 16) dec[1] |= c << (8 * (pos - 8));
        else dec[2] |= c << (8 * (pos - 16));
      }
    }
    const int P = prefix_len;
    seeds[k] = blake2b_seed63_1block(P + 8 + dl, [&](int i) -> uint8_t {
      if (i < P) return s_pre[i];
      if (i < P + 8) return (uint8_t)(i == P + 7 ? dl : 0);  // dl < 256
      const int d = i - P - 8;                                // digit d of str(id)
      const u64 word = d < 8 ? dec[0] : d < 16 ? dec[1] : dec[2];
      return (uint8_t)(word >> (8 * (d & 7)));
    });
  } else {
    uint8_t dec[20];
    u64_to_dec(v, dec);
    Blake2b b;
    b.init();
    b.bytes(prefix, prefix_len);
    b.len8((u64)dl);
    b.bytes(dec, dl);
    seeds[k] = b.seed63();
  }
  ids[k] = id;
}

// ------------------------------------------------------------------ small plans
// A plan of a few chunks (ADO: one chunk per call) is emitted by two kernels
// and one host sync: one CTA per chunk cuts all its terms into shared memory,
// sorts + merges there and writes into a per-chunk slot; a finalising CTA
// turns the slots into the CSR and derives the chunk seeds. Counts stay on
// the device (plan_out), so nothing waits on the host in between.
constexpr int SMALL_MAX_CHUNKS = 16;

__global__ void __launch_bounds__(NM_THREADS)
emit_small_kernel(EmitArgs a, const long long* plan_out, u32* gm, u32* gf, u32* gs, u32* ge, u64* cnt,
                  u32* overflow) {
  __shared__ uint4 s[NM_CAP];
  __shared__ u32 s_flags[NM_CAP];
  __shared__ u32 s_w[NM_THREADS / 32];
  __shared__ u32 s_tot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long k = blockIdx.x;
  if (k >= plan_out[0]) {
    if (tid == 0) cnt[k] = 0;
    return;
  }
  long long lo = 0, hi = plan_out[1];
  while (lo < hi) {  // last phase with chunk_begin <= k
    const long long mid = (lo + hi) >> 1;
    if (a.phases[mid].chunk_begin <= k) lo = mid + 1; else hi = mid;
  }
  const Phase ph = a.phases[lo - 1];
  const long long kr = k - ph.chunk_begin;
  u32 run = 0;
  for (long long tb = 0; tb < ph.n_terms; tb += NM_THREADS) {
    const long long t = tb + tid;
    Term tm{};
    u32 c = 0;
    if (t < ph.n_terms) {
      tm = a.terms[ph.term_begin + t];
      c = (u32)walk_term<false>(a, tm, kr, [](u64, u32, u32, u32, u32) {});
    }
    const u32 inc = warp_incl_scan(c);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const u32 x = lane < NM_THREADS / 32 ? s_w[lane] : 0;
      const u32 xi = warp_incl_scan(x);
      if (lane < NM_THREADS / 32) s_w[lane] = xi - x;
      if (lane == 31) s_tot = xi;
    }
    __syncthreads();
    const u32 base = run + s_w[warp] + inc - c, tot = s_tot;
    if (run + tot > NM_CAP) {
      if (tid == 0) atomicMax(overflow, run + tot);
      return;
    }
    if (c)
      walk_term<true>(a, tm, kr, [&](u64 i, u32 m, u32 f, u32 s0, u32 e0) { s[base + i] = make_uint4(m, f, s0, e0); });
    run += tot;
    __syncthreads();
  }
  const u32 m = run ? sort_merge(s, run, tid, NM_THREADS, s_flags) : 0;
  const long long o = k * NM_CAP;
  for (u32 i = tid; i < m; i += NM_THREADS) {
    gm[o + i] = s[i].x;
    gf[o + i] = s[i].y;
    gs[o + i] = s[i].z;
    ge[o + i] = s[i].w;
  }
  if (tid == 0) cnt[k] = m;
}

__global__ void __launch_bounds__(256)
finalize_small_kernel(const long long* plan_out, const u64* cnt, const u32* gm, const u32* gf, const u32* gs,
                      const u32* ge, u32* rm, u32* rf, u32* rs, u32* re, long long* res_off, u64* seeds, long long* ids,
                      long long first_id, const uint8_t* prefix, int prefix_len, long long* header) {
  __shared__ long long s_off[SMALL_MAX_CHUNKS + 1];
  const long long n = plan_out[0];
  if (threadIdx.x == 0) {
    long long r = 0;
    for (long long k = 0; k < n; ++k) {
      s_off[k] = r;
      r += (long long)cnt[k];
    }
    s_off[n] = r;
    header[0] = n;
    header[1] = r;
    header[2] = plan_out[3];
  }
  __syncthreads();
  for (long long k = 0; k <= n; k += 1)
    if (threadIdx.x == 0) res_off[k] = s_off[k];
  for (long long k = 0; k < n; ++k) {
    const long long src = k * NM_CAP, dst = s_off[k], c = s_off[k + 1] - dst;
    for (long long i = threadIdx.x; i < c; i += blockDim.x) {
      rm[dst + i] = gm[src + i];
      rf[dst + i] = gf[src + i];
      rs[dst + i] = gs[src + i];
      re[dst + i] = ge[src + i];
    }
  }
  if (threadIdx.x < n) {  // derive_seed(job_seed, "chunk", id)  (chunks.py:188)
    uint8_t dec[20];
    const long long id = first_id + threadIdx.x;
    const int dl = u64_to_dec((u64)id, dec);
    Blake2b b;
    b.init();
    b.bytes(prefix, prefix_len);
    b.len8((u64)dl);
    b.bytes(dec, dl);
    seeds[threadIdx.x] = b.seed63();
    ids[threadIdx.x] = id;
  }
}

// ------------------------------------------------------------------ host
struct PlanWork {  // stream segment tables (generator scratch slots)
  int mode = 0;
  long long chunk_size = 0;  // samples per chunk (emission path choice)
  long long max_mkey = 0;  // exclusive bound of the pieces' mixture-key ids (0 = unknown)
  int n_streams = 0;
  u32* s_off = nullptr;
  u32* seg_comp = nullptr;
  u64* seg_lo = nullptr;
  u64* seg_pre = nullptr;
};

enum ScratchSlot { S_WTS, S_SOFF, S_SEGC, S_SEGLO, S_SEGPRE, S_PHASES, S_TERMS, S_LL, S_OUT, S_REPORT, S_FLAGS,
                   S_POS, S_APIDX, S_APFRAC, S_FRONT, S_GM, S_GF, S_GS, S_GE, S_OVF, S_CNT, S_HDR, S_MTOT };

// Emission of a planned batch. Only ONE host synchronisation (at the end):
// the pair prefix comes from the host copy of the phases, and the piece /
// range buffers are sized by the bound pieces <= pairs + segments + intervals
// (a (chunk, term) range yields one piece plus one per interval or stream
// segment boundary inside it, and every stream position belongs to exactly
// one range), so no count has to travel to the host mid-way.
// Per-chunk normalisation of a chunk CSR of cut pieces (cpo offsets) and the
// dense result: sort by (mixture key, file, start) + merge per chunk, scan of
// the merged counts, compaction into the generator's result arrays.
static int normalize_tail(GenData* g, long long n_chunks, DevBuf<u64>& cpo, DevBuf<u64>& mcnt, DevBuf<u32>& big,
                          DevBuf<u32>& pm, DevBuf<u32>& pf, DevBuf<u32>& ps, DevBuf<u32>& pe, long long cap,
                          bool pack, int fbits, cudaEvent_t seed_join, cudaStream_t s) {
  {
    DevBuf<u32> blist, bcnt;
    MX_CUDA_TRY(ws_borrow(blist, s, WS_NBL, n_chunks));
    MX_CUDA_TRY(ws_borrow(bcnt, s, WS_NBC, 1));
    MX_CUDA_TRY(cudaMemsetAsync(bcnt.p, 0, sizeof(u32), s));
    DevBuf<u32> wlist, wcnt;
    MX_CUDA_TRY(ws_borrow(wlist, s, WS_NWL, n_chunks));
    MX_CUDA_TRY(ws_borrow(wcnt, s, WS_NWC, 1));
    MX_CUDA_TRY(cudaMemsetAsync(wcnt.p, 0, sizeof(u32), s));
    normalize_tiny_kernel<<<(unsigned)((n_chunks + 255) / 256), 256, 0, s>>>(n_chunks, cpo.p, pm.p, pf.p, ps.p, pe.p,
                                                                           mcnt.p, wlist.p, wcnt.p);
    mx_count_launch();
    const long long wgrid = std::min<long long>((n_chunks + 7) / 8, 148 * 16);
    // pack (mkey, file, start) into one u64 when mkey and file ids fit 32 bits together
    if (pack)  // keys < 2^63: never the ~0 padding
      normalize_warp_kernel<true><<<(unsigned)wgrid, 256, 0, s>>>(wlist.p, wcnt.p, cpo.p, pm.p, pf.p, ps.p, pe.p,
                                                                  mcnt.p, blist.p, bcnt.p, fbits);
    else
      normalize_warp_kernel<false><<<(unsigned)wgrid, 256, 0, s>>>(wlist.p, wcnt.p, cpo.p, pm.p, pf.p, ps.p, pe.p,
                                                                   mcnt.p, blist.p, bcnt.p, 0);
    mx_count_launch();
    long long grid = n_chunks < 148 * 4 ? n_chunks : 148 * 4;
    normalize_kernel<<<(unsigned)grid, NMB_THREADS, 0, s>>>(blist.p, bcnt.p, cpo.p, pm.p, pf.p, ps.p, pe.p, mcnt.p,
                                                           big.p);
    mx_count_launch();
  }
  if (int rc = excl_scan<long long>(mcnt.p, n_chunks, g->res_off.p, s)) return rc;
  MX_CUDA_TRY(g->res_mkey.reserve(cap, s));
  MX_CUDA_TRY(g->res_file.reserve(cap, s));
  MX_CUDA_TRY(g->res_start.reserve(cap, s));
  MX_CUDA_TRY(g->res_end.reserve(cap, s));
  {
    // few ranges per chunk (sharded ranks): lanes copy chunks; else warps
    const bool grouped = g->ix->sharded;
    const long long grid = std::min<long long>(grouped ? (n_chunks + 255) / 256 : (n_chunks + 7) / 8, 148 * 16);
    compact_warp_kernel<<<(unsigned)grid, 256, 0, s>>>(n_chunks, cpo.p, g->res_off.p, pm.p, pf.p, ps.p, pe.p,
                                                       g->res_mkey.p, g->res_file.p, g->res_start.p, g->res_end.p,
                                                       grouped);
    mx_count_launch();
  }
  MX_CUDA_TRY(cudaStreamWaitEvent(s, seed_join, 0));  // chunk seeds (side stream) done
  MX_CUDA_TRY(cudaGetLastError());
  u32 h_big = 0;
  long long total = 0;
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(&h_big, big.p, sizeof(u32)));
    MX_CUDA_TRY(rb.add(&total, g->res_off.p + n_chunks, sizeof(long long)));
    MX_CUDA_TRY(rb.sync());
  }
  if (h_big) return mx_fail(MX_ERR_UNSUPPORTED, "a chunk has %u ranges before merging (> %d supported)", h_big, NM_CAP);
  g->res_ranges = total;
  g->next_chunk_id += n_chunks;
  return MX_OK;
}

// ---------------------------------------------------------------------------
// Local-driven emission (key-partitioned multi-GPU, GenData::local): the plan
// ran on a key-level index (global per-key totals); this rank walks its OWN
// intervals: block b of local key kl is component g = key_g[kl] at offset
// blk_off[b] of g's global cursor stream, which sits in mixture-key stream m
// at segment seg (mode 0: one stream per component). A stream position maps
// to a chunk through stream m's terms (phases in chunk order; bases
// increasing; chunk j of a term covers [base + j*stride, + len)). Work is
// O(local intervals + pieces), not O(global chunks x terms).
struct StreamTerm {
  u64 base, len, stride;  // len > 0, stride >= len (chunks of a term never overlap)
  long long chunk_begin, n_chunks;
  u32 m;
};

struct LocalCut {
  long long B;             // local blocks
  const u32* blk_key;      // local index
  const u32* blk_first;
  const u64* iv_cum;
  const u32* iv_file;
  const u32* iv_start;
  const u64* blk_off;
  const u32* key_g;
  long long file_lo;
  const int* comp_seg;     // [K] segment of the component in its stream (-1: no mixture key)
  const int* comp_str;     // [K] its stream (mixture key)
  const u64* seg_pre;      // stream prefix (segment i of stream m at seg_pre[i + m])
  const u64* seg_lo;       // consumed part of each segment's component at plan start
  const u32* st_off;       // [n_streams + 1] term list of every stream
  const StreamTerm* st;
  int arbitrary;           // pieces carry the component id (mode 2)
};

__global__ void comp_seg_kernel(int n_streams, const u32* s_off, const u32* seg_comp, int* comp_seg, int* comp_str) {
  const int m = blockIdx.x;
  if (m >= n_streams) return;
  for (u32 i = s_off[m] + threadIdx.x; i < s_off[m + 1]; i += blockDim.x) {
    comp_seg[seg_comp[i]] = (int)i;
    comp_str[seg_comp[i]] = m;
  }
}

template <bool WRITE>
__global__ void local_cut_kernel(LocalCut a, u64* cnt, const u64* off, u32* pc, u32* pm, u32* pf, u32* ps, u32* pe) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const u32 g = a.key_g[a.blk_key[b]];
  const int seg = a.comp_seg[g];
  u64 n = 0, o_out = WRITE ? off[b] : 0;
  if (seg >= 0) {
    const int m = a.comp_str[g];
    const u64 ob = a.blk_off[b], lo = a.seg_lo[seg], pre = a.seg_pre[seg + m];
    const u64 take = a.seg_pre[seg + 1 + m] - pre;  // the segment's part of the component this plan hands out
    const u32 t_lo = a.st_off[m], t_hi = a.st_off[m + 1];
    const u32 i0 = a.blk_first[b], i1 = a.blk_first[b + 1];
    const u64 c0 = a.iv_cum[i0];
    for (u32 i = i0; i < i1; ++i) {
      const u64 o = ob + (a.iv_cum[i] - c0), len = a.iv_cum[i + 1] - a.iv_cum[i];
      if (o + len <= lo || o >= lo + take) continue;  // handed out before / not in this plan
      const u64 a0 = o > lo ? o : lo, a1 = o + len < lo + take ? o + len : lo + take;
      const u64 xs = pre + (a0 - lo), xe = pre + (a1 - lo);
      const u32 s0 = a.iv_start[i] + (u32)(a0 - o);
      // last term with base <= xs (terms of a stream are disjoint and in stream order)
      u32 tl = t_lo, th = t_hi;
      while (tl < th) {
        const u32 mid = (tl + th) >> 1;
        if (a.st[mid].base <= xs) tl = mid + 1; else th = mid;
      }
      u32 t = tl > t_lo ? tl - 1 : t_lo;
      u64 x = xs;
      while (x < xe && t < t_hi) {
        const StreamTerm T = a.st[t];
        if (x < T.base) x = T.base;  // positions no term hands out
        if (x >= xe) break;
        const long long j = T.stride > 0 ? (long long)((x - T.base) / T.stride) : 0;
        if (j >= T.n_chunks) {
          ++t;
          continue;
        }
        const u64 c_lo = T.base + (u64)j * T.stride, c_hi = c_lo + T.len;
        if (x >= c_hi) {  // between two chunks of a strided term
          if (j + 1 < T.n_chunks) x = c_lo + T.stride;
          else ++t;
          continue;
        }
        const u64 e = xe < c_hi ? xe : c_hi;
        if (WRITE) {
          const u64 q = o_out + n;
          pc[q] = (u32)(T.chunk_begin + j);
          pm[q] = a.arbitrary ? g : T.m;
          pf[q] = (u32)(a.file_lo + a.iv_file[i]);
          ps[q] = s0 + (u32)(x - xs);
          pe[q] = s0 + (u32)(e - xs);
        }
        ++n;
        x = e;
      }
    }
  }
  if (!WRITE) cnt[b] = n;
}

// pieces -> chunk CSR (order inside a chunk is settled by the normalisation)
__global__ void widen_kernel(long long n, const int32_t* in, u64* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (u64)in[i];
}

__global__ void chunk_hist_kernel(long long n, const u32* pc, u64* cc) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(reinterpret_cast<unsigned long long*>(cc + pc[i]), 1ull);
}

__global__ void chunk_scatter_kernel(long long n, const u32* pc, const u32* pm, const u32* pf, const u32* ps,
                                     const u32* pe, const u64* cpo, unsigned long long* fill, u32* qm, u32* qf,
                                     u32* qs, u32* qe) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u32 c = pc[i];
  const u64 q = cpo[c] + atomicAdd(fill + c, 1ull);
  qm[q] = pm[i];
  qf[q] = pf[i];
  qs[q] = ps[i];
  qe[q] = pe[i];
}

__global__ void chunk_scatter_aos_kernel(long long n, const u32* pc, const u32* pm, const u32* pf, const u32* ps,
                                         const u32* pe, const u64* cpo, unsigned long long* fill, uint4* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u32 c = pc[i];
  out[cpo[c] + atomicAdd(fill + c, 1ull)] = make_uint4(pm[i], pf[i], ps[i], pe[i]);
}

// Chunk owner: the pieces of its chunks [chunk_lo, chunk_lo + n_own) from
// every rank (received source-major, chunk-major inside a source; counts
// [world][n_own]) into one chunk CSR, then the normal per-chunk
// normalisation. Pieces of one chunk never merge across ranks (a file lives
// on one rank), so the result equals the single-GPU chunk.
__global__ void owned_totals_kernel(int world, long long n_own, const int32_t* counts, u64* tot) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= n_own) return;
  u64 t = 0;
  for (int q = 0; q < world; ++q) t += (u64)counts[(long long)q * n_own + c];
  tot[c] = t;
}

__global__ void owned_gather_kernel(int world, long long n_own, const int32_t* counts, const u64* src_off,
                                    const u64* cpo, const uint4* in, u32* pm, u32* pf, u32* ps, u32* pe) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= n_own) return;
  u64 d = cpo[c];
  for (int q = 0; q < world; ++q) {
    const long long qc = (long long)q * n_own + c;
    const u64 so = src_off[qc];
    for (int32_t i = 0; i < counts[qc]; ++i, ++d) {
      const uint4 r = in[so + i];
      pm[d] = r.x;
      pf[d] = r.y;
      ps[d] = r.z;
      pe[d] = r.w;
    }
  }
}

int gen_finish_owned(GenData* g, int world, long long chunk_lo, long long n_own, long long n_global,
                     const int32_t* counts, const uint4* pieces, long long n_pieces, cudaStream_t s) {
  if (g->handoff.n_chunks < 0) return mx_fail(MX_ERR_INVALID, "no partitioned plan pending (mx_gen_handoff)");
  if (n_global != g->handoff.n_chunks || chunk_lo < 0 || n_own < 0 || chunk_lo + n_own > n_global)
    return mx_fail(MX_ERR_INVALID, "owned chunk range outside the pending plan");
  const long long base_id = g->handoff.first_id;
  g->handoff.n_chunks = -1;
  MxPhase ph("emit", s);
  g->h_small_valid = 0;
  g->res_chunks = n_own;
  g->res_ranges = 0;
  MX_CUDA_TRY(g->res_off.reserve(n_own + 1, s));
  MX_CUDA_TRY(g->res_seed.reserve(n_own > 0 ? n_own : 1, s));
  MX_CUDA_TRY(g->res_id.reserve(n_own > 0 ? n_own : 1, s));
  MX_CUDA_TRY(g->aux_init());
  if (n_own == 0) {
    const long long z = 0;
    MX_CUDA_TRY(mx_h2d(g->res_off.p, &z, sizeof(z), s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    g->next_chunk_id = base_id + n_global;
    return MX_OK;
  }
  // chunk seeds of the owned ids on the side stream
  MX_CUDA_TRY(cudaEventRecord(g->ev_seed_fork, s));
  MX_CUDA_TRY(cudaStreamWaitEvent(g->sstream, g->ev_seed_fork, 0));
  chunk_seed_kernel<<<(unsigned)((n_own + 127) / 128), 128, 0, g->sstream>>>(
      n_own, base_id + chunk_lo, g->chunk_prefix.p, g->chunk_prefix_len, g->res_seed.p, g->res_id.p);
  mx_count_launch();
  MX_CUDA_TRY(cudaEventRecord(g->ev_seed, g->sstream));
  const long long cap = n_pieces + 1;
  DevBuf<u64> tot, cpo, mcnt, src_off;
  DevBuf<u32> big, pm, pf, ps, pe;
  MX_CUDA_TRY(tot.alloc(n_own, s));
  MX_CUDA_TRY(cpo.alloc(n_own + 1, s));
  MX_CUDA_TRY(mcnt.alloc(n_own, s));
  MX_CUDA_TRY(src_off.alloc((long long)world * n_own + 1, s));
  MX_CUDA_TRY(big.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(big.p, 0, sizeof(u32), s));
  for (DevBuf<u32>* x : {&pm, &pf, &ps, &pe}) MX_CUDA_TRY(x->alloc(cap, s));
  const unsigned gb = (unsigned)((n_own + 255) / 256);
  owned_totals_kernel<<<gb, 256, 0, s>>>(world, n_own, counts, tot.p);
  mx_count_launch();
  if (int rc = excl_scan<u64>(tot.p, n_own, cpo.p, s)) return rc;
  DevBuf<u64> cnt64;  // counts widened for the source-offset scan
  MX_CUDA_TRY(cnt64.alloc((long long)world * n_own, s));
  widen_kernel<<<(unsigned)(((long long)world * n_own + 255) / 256), 256, 0, s>>>((long long)world * n_own, counts,
                                                                                   cnt64.p);
  mx_count_launch();
  if (int rc = excl_scan<u64>(cnt64.p, (long long)world * n_own, src_off.p, s)) return rc;
  owned_gather_kernel<<<gb, 256, 0, s>>>(world, n_own, counts, src_off.p, cpo.p, pieces, pm.p, pf.p, ps.p, pe.p);
  mx_count_launch();
  IndexData* ix = g->ix;
  int fbits = 1, mbits = 1;
  while ((1ll << fbits) < (long long)ix->n_files + 1) ++fbits;
  while ((1ll << mbits) < (long long)std::max<long long>(g->last_mkeys, g->K) + 1) ++mbits;
  const bool pack = fbits + mbits <= 31;
  int rc = normalize_tail(g, n_own, cpo, mcnt, big, pm, pf, ps, pe, cap, pack, fbits, g->ev_seed, s);
  g->next_chunk_id = base_id + n_global;
  return rc;
}

static int emit_local(GenData* g, const PlanWork& w, const Phase* h_phases, const Term* terms, long long n_chunks,
                      long long n_phases, cudaStream_t s) {
  const int Km = w.n_streams;
  IndexData* ix = g->ix;  // key-level index (global keys, global file table)
  const LocalSrc& L = g->local;
  MxPhase ph("emit", s);
  g->h_small_valid = 0;
  g->res_chunks = n_chunks;
  g->res_ranges = 0;
  MX_CUDA_TRY(g->res_off.reserve(n_chunks + 1, s));
  MX_CUDA_TRY(g->res_seed.reserve(n_chunks > 0 ? n_chunks : 1, s));
  MX_CUDA_TRY(g->res_id.reserve(n_chunks > 0 ? n_chunks : 1, s));
  MX_CUDA_TRY(g->aux_init());
  cudaEvent_t seed_join = g->ev_seed;
  const bool handoff = L.handoff;
  g->handoff.n_chunks = -1;
  if (n_chunks > 0 && !handoff) {
    MX_CUDA_TRY(cudaEventRecord(g->ev_seed_fork, s));
    MX_CUDA_TRY(cudaStreamWaitEvent(g->sstream, g->ev_seed_fork, 0));
    chunk_seed_kernel<<<(unsigned)((n_chunks + 127) / 128), 128, 0, g->sstream>>>(
        n_chunks, g->next_chunk_id, g->chunk_prefix.p, g->chunk_prefix_len, g->res_seed.p, g->res_id.p);
    mx_count_launch();
    MX_CUDA_TRY(cudaEventRecord(seed_join, g->sstream));
  }
  if (n_chunks == 0 && !handoff) {
    const long long z = 0;
    MX_CUDA_TRY(mx_h2d(g->res_off.p, &z, sizeof(z), s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    return MX_OK;
  }
  if (n_chunks == 0) {
    MX_CUDA_TRY(g->handoff.off.reserve(1, s));
    MX_CUDA_TRY(cudaMemsetAsync(g->handoff.off.p, 0, sizeof(long long), s));
    MX_CUDA_TRY(g->handoff.pieces.reserve(1, s));
    g->handoff.n_chunks = 0;
    g->handoff.first_id = g->next_chunk_id;
    g->res_chunks = 0;
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    return MX_OK;
  }
  const long long K = g->K;
  // stream term tables (host: a few hundred terms)
  long long n_terms = 0;
  for (long long p = 0; p < n_phases; ++p) n_terms = std::max(n_terms, h_phases[p].term_begin + h_phases[p].n_terms);
  std::vector<Term> h_terms(n_terms);
  if (n_terms) {
    MX_CUDA_TRY(cudaMemcpyAsync(h_terms.data(), terms, sizeof(Term) * n_terms, cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
  }
  std::vector<std::vector<StreamTerm>> per(Km);
  for (long long p = 0; p < n_phases; ++p)
    for (long long t = 0; t < h_phases[p].n_terms; ++t) {
      const Term& T = h_terms[h_phases[p].term_begin + t];
      if (T.len == 0 || h_phases[p].n_chunks == 0) continue;
      if (T.stride < T.len && h_phases[p].n_chunks > 1)
        return mx_fail(MX_ERR_UNSUPPORTED, "overlapping chunk terms in a partitioned plan");
      if (!per[T.stream].empty()) {  // the walk needs each stream's terms disjoint and in stream order
        const StreamTerm& q = per[T.stream].back();
        if (q.base + (u64)(q.n_chunks - 1) * q.stride + q.len > T.base)
          return mx_fail(MX_ERR_UNSUPPORTED, "interleaved chunk terms in a partitioned plan");
      }
      per[T.stream].push_back(
          StreamTerm{T.base, T.len, T.stride, h_phases[p].chunk_begin, h_phases[p].n_chunks, T.m});
    }
  std::vector<u32> st_off(Km + 1, 0);
  std::vector<StreamTerm> st;
  for (int m = 0; m < Km; ++m) {
    st.insert(st.end(), per[m].begin(), per[m].end());
    st_off[m + 1] = (u32)st.size();
  }
  DevBuf<u32> d_st_off;
  DevBuf<StreamTerm> d_st;
  DevBuf<int> comp_seg, comp_str;
  MX_CUDA_TRY(d_st_off.alloc(Km + 1, s));
  MX_CUDA_TRY(d_st.alloc(std::max<long long>(1, (long long)st.size()), s));
  MX_CUDA_TRY(mx_h2d(d_st_off.p, st_off.data(), sizeof(u32) * (Km + 1), s));
  if (!st.empty()) MX_CUDA_TRY(mx_h2d(d_st.p, st.data(), sizeof(StreamTerm) * st.size(), s));
  MX_CUDA_TRY(comp_seg.alloc(K, s));
  MX_CUDA_TRY(comp_str.alloc(K, s));
  MX_CUDA_TRY(cudaMemsetAsync(comp_seg.p, 0xff, sizeof(int) * K, s));
  comp_seg_kernel<<<Km, 128, 0, s>>>(Km, w.s_off, w.seg_comp, comp_seg.p, comp_str.p);
  mx_count_launch();
  const IndexData* loc = L.loc;
  const long long B = loc->n_blocks;
  LocalCut a{};
  a.B = B;
  a.blk_key = loc->blk_key.p;
  a.blk_first = loc->blk_first.p;
  a.iv_cum = loc->iv_cum.p;
  a.iv_file = loc->iv_file.p;
  a.iv_start = loc->iv_start.p;
  a.blk_off = L.blk_off;
  a.key_g = L.key_g;
  a.file_lo = L.file_lo;
  a.comp_seg = comp_seg.p;
  a.comp_str = comp_str.p;
  a.seg_pre = w.seg_pre;
  a.seg_lo = w.seg_lo;
  a.st_off = d_st_off.p;
  a.st = d_st.p;
  a.arbitrary = w.mode == 2;
  DevBuf<u64> boff;
  MX_CUDA_TRY(boff.alloc(B + 1, s));
  const unsigned bg = (unsigned)((B + 255) / 256);
  if (B > 0) {
    local_cut_kernel<false><<<bg, 256, 0, s>>>(a, boff.p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    mx_count_launch();
  }
  if (int rc = excl_scan<u64>(boff.p, B, boff.p, s)) return rc;
  u64 n_p = 0;
  MX_CUDA_TRY(cudaMemcpyAsync(&n_p, boff.p + B, sizeof(u64), cudaMemcpyDeviceToHost, s));
  MX_CUDA_TRY(cudaStreamSynchronize(s));
  const long long cap = (long long)n_p + 1;
  DevBuf<u32> pc, pm, pf, ps, pe, qm, qf, qs, qe;
  for (DevBuf<u32>* x : {&pc, &pm, &pf, &ps, &pe, &qm, &qf, &qs, &qe}) MX_CUDA_TRY(x->alloc(cap, s));
  if (B > 0) {
    local_cut_kernel<true><<<bg, 256, 0, s>>>(a, nullptr, boff.p, pc.p, pm.p, pf.p, ps.p, pe.p);
    mx_count_launch();
  }
  DevBuf<u64> cc, cpo, mcnt;
  DevBuf<unsigned long long> fill;
  DevBuf<u32> big;
  MX_CUDA_TRY(cc.alloc(n_chunks, s));
  MX_CUDA_TRY(cpo.alloc(n_chunks + 1, s));
  MX_CUDA_TRY(mcnt.alloc(n_chunks, s));
  MX_CUDA_TRY(fill.alloc(n_chunks, s));
  MX_CUDA_TRY(big.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(cc.p, 0, sizeof(u64) * n_chunks, s));
  MX_CUDA_TRY(cudaMemsetAsync(fill.p, 0, sizeof(unsigned long long) * n_chunks, s));
  MX_CUDA_TRY(cudaMemsetAsync(big.p, 0, sizeof(u32), s));
  const long long np = (long long)n_p;
  if (np > 0) {
    chunk_hist_kernel<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(np, pc.p, cc.p);
    mx_count_launch();
  }
  if (int rc = excl_scan<u64>(cc.p, n_chunks, cpo.p, s)) return rc;
  if (handoff) {  // pieces grouped by chunk for the chunk owners; the owners normalise
    MX_CUDA_TRY(g->handoff.off.reserve(n_chunks + 1, s));
    MX_CUDA_TRY(g->handoff.pieces.reserve(cap, s));
    MX_CUDA_TRY(cudaMemcpyAsync(g->handoff.off.p, cpo.p, sizeof(long long) * (n_chunks + 1),
                                cudaMemcpyDeviceToDevice, s));
    if (np > 0) {
      chunk_scatter_aos_kernel<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(np, pc.p, pm.p, pf.p, ps.p, pe.p, cpo.p,
                                                                            fill.p, g->handoff.pieces.p);
      mx_count_launch();
    }
    MX_CUDA_TRY(cudaGetLastError());
    MX_CUDA_TRY(cudaStreamSynchronize(s));  // the buffers above are freed with this scope
    g->handoff.n_chunks = n_chunks;
    g->handoff.first_id = g->next_chunk_id;
    g->res_chunks = 0;  // the owners' results come from gen_finish_owned
    return MX_OK;
  }
  if (np > 0) {
    chunk_scatter_kernel<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(np, pc.p, pm.p, pf.p, ps.p, pe.p, cpo.p,
                                                                      fill.p, qm.p, qf.p, qs.p, qe.p);
    mx_count_launch();
  }
  int fbits = 1, mbits = 1;
  while ((1ll << fbits) < (long long)ix->n_files + 1) ++fbits;
  while ((1ll << mbits) < (long long)(w.max_mkey > 0 ? w.max_mkey : Km) + 1) ++mbits;
  const bool pack = fbits + mbits <= 31;
  return normalize_tail(g, n_chunks, cpo, mcnt, big, qm, qf, qs, qe, cap, pack, fbits, seed_join, s);
}

static int emit(GenData* g, const PlanWork& w, const Phase* phases, const Phase* h_phases, const Term* terms,
                long long n_chunks, long long n_phases, long long n_seg, cudaStream_t s) {
  if (g->local.loc) return emit_local(g, w, h_phases, terms, n_chunks, n_phases, s);  // key-partitioned rank
  IndexData* ix = g->ix;
  MxPhase ph("emit", s);
  g->h_small_valid = 0;
  g->res_chunks = n_chunks;
  g->res_ranges = 0;
  MX_CUDA_TRY(g->res_off.reserve(n_chunks + 1, s));
  MX_CUDA_TRY(g->res_seed.reserve(n_chunks > 0 ? n_chunks : 1, s));
  MX_CUDA_TRY(g->res_id.reserve(n_chunks > 0 ? n_chunks : 1, s));
  // chunk seeds depend only on chunk ids: hash them on a side stream while
  // the pieces are cut, normalised and compacted on `s`
  // (per-generator stream and events: created on the generator's device)
  MX_CUDA_TRY(g->aux_init());
  cudaStream_t seed_side = g->sstream;
  cudaEvent_t seed_fork = g->ev_seed_fork, seed_join = g->ev_seed;
  if (n_chunks > 0) {
    MX_CUDA_TRY(cudaEventRecord(seed_fork, s));
    MX_CUDA_TRY(cudaStreamWaitEvent(seed_side, seed_fork, 0));
    chunk_seed_kernel<<<(unsigned)((n_chunks + 127) / 128), 128, 0, seed_side>>>(
        n_chunks, g->next_chunk_id, g->chunk_prefix.p, g->chunk_prefix_len, g->res_seed.p, g->res_id.p);
    mx_count_launch();
    MX_CUDA_TRY(cudaEventRecord(seed_join, seed_side));
  }
  if (n_chunks == 0) {
    const long long z = 0;
    MX_CUDA_TRY(mx_h2d(g->res_off.p, &z, sizeof(z), s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    return MX_OK;
  }
  std::vector<u64> h_pre(n_phases + 1);
  h_pre[0] = 0;
  for (long long p = 0; p < n_phases; ++p)
    h_pre[p + 1] = h_pre[p] + (u64)h_phases[p].n_chunks * (u64)h_phases[p].n_terms;
  const u64 n_pairs = h_pre[n_phases];
  // call temporaries come from the per-(thread, stream) workspace
  DevBuf<u64> pair_pre;
  MX_CUDA_TRY(ws_borrow(pair_pre, s, WS_EPRE, n_phases + 1));
  MX_CUDA_TRY(mx_h2d(pair_pre.p, h_pre.data(), sizeof(u64) * (n_phases + 1), s));
  EmitArgs a{};
  a.phases = phases;
  a.n_phases = n_phases;
  a.terms = terms;
  a.pair_pre = pair_pre.p;
  a.s_off = w.s_off;
  a.seg_comp = w.seg_comp;
  a.seg_lo = w.seg_lo;
  a.seg_pre = w.seg_pre;
  a.arbitrary = w.mode == 2;
  a.key_blk_first = ix->key_blk_first.p;
  a.blk_first = ix->blk_first.p;
  a.civ = g->civ.p;
  a.cfile = g->cfile.p;
  a.cstart = g->cstart.p;
  a.ccum = g->ccum.p;
  a.iv_start = ix->iv_start.p;
  a.iv_end = ix->iv_end.p;
  a.iv_file = ix->iv_file.p;
  a.lcnt = g->lcnt.p;
  a.lpos = g->lpos.p;
  a.lstart = g->lstart.p;
  const long long cap = (long long)n_pairs + n_seg + ix->n_intervals + 1;
  int fbits = 1, mbits = 1;
  while ((1ll << fbits) < (long long)ix->n_files + 1) ++fbits;
  while ((1ll << mbits) < w.max_mkey + 1) ++mbits;
  // not for a file-sharded (hybrid) index: its file ids are checked nowhere here
  const bool pack = w.max_mkey > 0 && fbits + mbits <= 31 && g->lcnt.p == nullptr;
  DevBuf<u64> pair_off;
  MX_CUDA_TRY(ws_borrow(pair_off, s, WS_EOFF, (long long)n_pairs + 1));
  const unsigned pb = (unsigned)((n_pairs + 255) / 256);
  mx_host_mark("emit setup");
  emit_count_kernel<<<pb, 256, 0, s>>>(a, n_pairs, pair_off.p);
  mx_count_launch();
  // exclusive scan of counts in place (each element is read and written by
  // the same thread; the total lands in [n_pairs])
  if (int rc = excl_scan<u64>(pair_off.p, (long long)n_pairs, pair_off.p, s)) return rc;
  // mode-0 plans on a single-GPU index: chunks come out of the cut already in
  // (mixture key, file, start) order unless a pair was long / a merge exists
  const bool sort_terms = w.mode == 0 && g->lcnt.p == nullptr;
  DevBuf<u32> eflags;
  MX_CUDA_TRY(ws_borrow(eflags, s, WS_EFLAG, 1));
  MX_CUDA_TRY(cudaMemsetAsync(eflags.p, 0, sizeof(u32), s));
  DevBuf<u32> pm, pf, ps, pe;
  MX_CUDA_TRY(pm.alloc(cap, s));
  MX_CUDA_TRY(pf.alloc(cap, s));
  MX_CUDA_TRY(ps.alloc(cap, s));
  MX_CUDA_TRY(pe.alloc(cap, s));
  {
    DevBuf<u32> llist, lcnt;
    MX_CUDA_TRY(ws_borrow(llist, s, WS_ELIST, 2 * (long long)n_pairs));  // [long pairs | unstaged pairs to sort]
    MX_CUDA_TRY(ws_borrow(lcnt, s, WS_ELCNT, 2));
    MX_CUDA_TRY(cudaMemsetAsync(lcnt.p, 0, 2 * sizeof(u32), s));
    constexpr u32 warp_min = 32;  // pairs with more pieces are cut by a warp (emit_write_warp_kernel)
    emit_write_staged_kernel<<<(unsigned)((n_pairs + EW_THREADS - 1) / EW_THREADS), EW_THREADS, 0, s>>>(
        a, n_pairs, pair_off.p, pm.p, pf.p, ps.p, pe.p, llist.p, lcnt.p, warp_min, sort_terms ? 1 : 0,
        eflags.p);
    mx_count_launch();
    const long long wgrid = std::min<long long>(((long long)n_pairs + 7) / 8, 148 * 16);
    emit_write_warp_kernel<<<(unsigned)wgrid, 256, 0, s>>>(a, pair_off.p, pm.p, pf.p, ps.p, pe.p, llist.p, lcnt.p);
    mx_count_launch();
    if (sort_terms) {
      sort_pairs_warp_kernel<<<148 * 8, 256, 0, s>>>(llist.p, lcnt.p, n_pairs, pair_off.p, pm.p, pf.p, ps.p, pe.p,
                                                     eflags.p);
      mx_count_launch();
      sort_pairs_kernel<<<148 * 2, 256, 0, s>>>(llist.p, lcnt.p, n_pairs, pair_off.p, pm.p, pf.p, ps.p, pe.p,
                                                eflags.p);
      mx_count_launch();
    }
  }
  DevBuf<u64> cpo, mcnt;
  DevBuf<u32> big;
  MX_CUDA_TRY(ws_borrow(cpo, s, WS_ECPO, n_chunks + 1));
  MX_CUDA_TRY(ws_borrow(mcnt, s, WS_EMCNT, n_chunks));
  MX_CUDA_TRY(ws_borrow(big, s, WS_EBIG, 1));
  MX_CUDA_TRY(cudaMemsetAsync(big.p, 0, sizeof(u32), s));
  chunk_pieces_kernel<<<(unsigned)((n_chunks + 256) / 256), 256, 0, s>>>(a, n_chunks, pair_off.p, n_pairs, cpo.p);
  mx_count_launch();
  mx_host_mark("emit launched");
  if (sort_terms) {
    u32 h_flags = 1;
    long long total = 0;
    MX_CUDA_TRY(cudaStreamWaitEvent(s, seed_join, 0));  // chunk seeds (side stream) done
    {
      D2HBatch rb(s);
      MX_CUDA_TRY(rb.add(&h_flags, eflags.p, sizeof(u32)));
      MX_CUDA_TRY(rb.add(&total, cpo.p + n_chunks, sizeof(long long)));
      MX_CUDA_TRY(rb.sync());
    }
    if (h_flags == 0) {  // already normalised: the cut pieces are the result
      g->res_mkey.take(pm);
      g->res_file.take(pf);
      g->res_start.take(ps);
      g->res_end.take(pe);
      MX_CUDA_TRY(cudaMemcpyAsync(g->res_off.p, cpo.p, sizeof(long long) * (n_chunks + 1), cudaMemcpyDeviceToDevice,
                                  s));
      g->res_ranges = total;
      g->next_chunk_id += n_chunks;
      return MX_OK;
    }
  }
  return normalize_tail(g, n_chunks, cpo, mcnt, big, pm, pf, ps, pe, cap, pack, fbits, seed_join, s);
}

// per mixture key the matching components IN COMPONENT ORDER
// (chunks.py:139-141): waits for the component-order shuffle
static cudaError_t match_fill(GenData* g, const MatchArgs& ma, cudaStream_t s) {
  if (ma.K <= 0) return cudaSuccess;
  if (g->ev_order) {
    cudaError_t e = cudaStreamWaitEvent(s, g->ev_order, 0);
    if (e != cudaSuccess) return e;
  }
  match_fill_kernel<<<ma.Km, 256, 0, s>>>(ma, g->match_L_off.p, g->match_L.p);
  mx_count_launch();
  return cudaGetLastError();
}

int plan_mixture(GenData* g, const mx_mixture_desc* mix, long long max_chunks, long long* n_out) {
  // Matching and the count-level plan run on the generator's plan stream;
  // emission runs on the generator's stream (`ms`) after it waits for them.
  const cudaStream_t ms = g->stream;
  cudaStream_t s = g->pstream;
  IndexData* ix = g->ix;
  const int Km = mix->n_mkeys;
  const long long K = g->K;
  *n_out = 0;
  if (Km < 1) return mx_fail(MX_ERR_MIXTURE, "mixture has no keys");
  if (mix->chunk_size < 1) return mx_fail(MX_ERR_MIXTURE, "chunk_size must be positive");
  if (mix->strict && mix->chunk_size < Km)
    return mx_fail(MX_ERR_MIXTURE, "chunk size %lld below the number of mixture keys (%d)", (long long)mix->chunk_size, Km);
  g->report.assign(Km, 0);
  g->last_mkeys = Km;
  if (!s) {  // empty index: no auxiliary streams
    MX_CUDA_TRY(g->aux_init());
    s = g->pstream;
  }
  // the first plan after the cursor layout needs only the component totals
  // (recorded before the per-key shuffles); later plans see everything
  if (g->fresh_layout && g->ev_tot) {
    MX_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_tot, 0));
  } else {
    MX_CUDA_TRY(cudaEventRecord(g->ev_ready, ms));
    MX_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_ready, 0));
  }
  const bool fresh = g->fresh_layout;
  g->fresh_layout = false;
  const bool small = max_chunks <= SMALL_MAX_CHUNKS && mix->chunk_size <= NM_CAP && !g->local.loc;
  std::unique_ptr<MxPhase> ph_plan(new MxPhase("plan", s));
  // ---- matching
  MatchArgs ma{};
  ma.Km = Km;
  ma.K = K;
  ma.comp_order = g->comp_order.p;
  ma.key_packed = ix->key_packed.p;
  ma.n_props = ix->n_props;
  for (int p = 0; p < ix->n_props; ++p) {
    ma.shift[p] = ix->field_shift[p];
    ma.width[p] = ix->field_width[p];
    ma.allow_base[p] = mix->allow_base[p];
  }
  ma.allow_words = mix->allow_words;
  double* wts_p = nullptr;
  MX_CUDA_TRY(g->scratch(S_WTS, Km, &wts_p, s));
  MX_CUDA_TRY(mx_h2d(wts_p, mix->weights, sizeof(double) * Km, s));
  // matching depends only on the mixture KEYS (not the weights): reuse the
  // previous plan's per-key component lists when the keys are unchanged
  // (ADO re-plans every chunk with new weights over the same domains)
  const size_t n_allow = (size_t)Km * mix->allow_words;
  const bool cached = g->match_words == mix->allow_words && g->match_allow.size() == n_allow &&
                      (int)g->match_base.size() == ix->n_props &&
                      std::equal(g->match_base.begin(), g->match_base.end(), mix->allow_base) &&
                      std::equal(g->match_allow.begin(), g->match_allow.end(), mix->allow);
  // fused matching + plan (<= 32 keys, bulk): one launch, one host sync;
  // a mixture with shared components falls through to the general path
  if (!cached && Km <= FP_MAX_KM && !small && K > 0 && getenv("MX_PLAN_LATE") == nullptr) {
    DevBuf<u32> f_allow;
    MX_CUDA_TRY(f_allow.alloc((long long)n_allow, s));
    MX_CUDA_TRY(mx_h2d(f_allow.p, mix->allow, sizeof(u32) * n_allow, s));
    ma.allow = f_allow.p;
    MX_CUDA_TRY(g->match_L_off.alloc(Km + 1, s));
    long long cap_phases = 4 * (long long)Km + 64;
    if (cap_phases > max_chunks + 1) cap_phases = max_chunks + 1;
    const long long cap_terms = cap_phases * (long long)Km;
    Phase* phases = nullptr;
    Term* terms = nullptr;
    long long *out = nullptr, *report = nullptr;
    u64* pos = nullptr;
    MX_CUDA_TRY(g->scratch(S_PHASES, cap_phases, &phases, s));
    MX_CUDA_TRY(g->scratch(S_TERMS, cap_terms, &terms, s));
    MX_CUDA_TRY(g->scratch(S_OUT, 5, &out, s));
    MX_CUDA_TRY(g->scratch(S_REPORT, Km, &report, s));
    MX_CUDA_TRY(g->scratch(S_POS, Km, &pos, s));
    MX_CUDA_TRY(cudaMemsetAsync(phases, 0, sizeof(Phase) * cap_phases, s));
    MX_CUDA_TRY(cudaMemsetAsync(report, 0, sizeof(long long) * Km, s));
    FusedPlanArgs fa{};
    fa.ma = ma;
    fa.comp_total = g->comp_total.p;
    fa.consumed = g->consumed.p;
    fa.C = mix->chunk_size;
    fa.strict = mix->strict;
    fa.max_chunks = max_chunks;
    fa.w = wts_p;
    fa.L_off = g->match_L_off.p;
    fa.pos = pos;
    fa.phases = phases;
    fa.cap_phases = cap_phases;
    fa.terms = terms;
    fa.cap_terms = cap_terms;
    fa.out = out;
    fa.report = report;
    plan_fused_kernel<<<1, FP_THREADS, 0, s>>>(fa);
    mx_count_launch();
    MX_CUDA_TRY(cudaGetLastError());
    mx_host_mark("plan fused launched");
    long long h_out[5];
    std::vector<Phase> h_phases(cap_phases);
    std::vector<u32> h_loff(Km + 1);
    {
      D2HBatch rb(s);
      MX_CUDA_TRY(rb.add(h_out, out, sizeof(h_out)));
      MX_CUDA_TRY(rb.add(g->report.data(), report, sizeof(long long) * Km));
      MX_CUDA_TRY(rb.add(h_phases.data(), phases, sizeof(Phase) * cap_phases));
      MX_CUDA_TRY(rb.add(h_loff.data(), g->match_L_off.p, sizeof(u32) * (Km + 1)));
      MX_CUDA_TRY(rb.sync());
    }
    mx_host_mark("plan synced");
    if (h_out[4] == 0) {
      g->match_off.assign(h_loff.begin(), h_loff.end());
      g->match_shared = false;
      MX_CUDA_TRY(g->match_L.alloc(h_loff[Km] > 0 ? h_loff[Km] : 1, s));
      MX_CUDA_TRY(match_fill(g, ma, s));  // ordered lists, behind the component-order shuffle
      g->match_allow.assign(mix->allow, mix->allow + n_allow);
      g->match_base.assign(mix->allow_base, mix->allow_base + ix->n_props);
      g->match_words = mix->allow_words;
      PlanWork w;
      w.mode = 0;
      w.chunk_size = mix->chunk_size;
      w.n_streams = Km;
      w.s_off = g->match_L_off.p;
      w.max_mkey = Km;
      const long long nseg = h_loff[Km];
      MX_CUDA_TRY(g->scratch(S_SEGC, nseg, &w.seg_comp, s));
      MX_CUDA_TRY(g->scratch(S_SEGLO, nseg, &w.seg_lo, s));
      MX_CUDA_TRY(g->scratch(S_SEGPRE, nseg + Km, &w.seg_pre, s));
      build_segments_kernel<<<(Km + 3) / 4, 128, 0, s>>>(0, Km, w.s_off, g->match_L.p, g->comp_total.p,
                                                            g->consumed.p, w.seg_comp, w.seg_lo, w.seg_pre);
      mx_count_launch();
      MX_CUDA_TRY(cudaEventRecord(g->ev_seg, s));
      MX_CUDA_TRY(cudaStreamWaitEvent(ms, g->ev_seg, 0));
      ph_plan.reset();
      commit_segments_kernel<<<Km, 128, 0, ms>>>(Km, w.s_off, w.seg_comp, w.seg_lo, w.seg_pre, pos, g->consumed.p);
      mx_count_launch();
      if (int rc = emit(g, w, phases, h_phases.data(), terms, h_out[0], h_out[1], nseg, ms)) return rc;
      *n_out = h_out[0];
      return h_out[3] ? MX_EXHAUSTED : MX_OK;
    }
  }
  // early plan: a disjoint mixture of few keys is planned from the stream
  // LENGTHS alone (no component order needed); its ordered segment tables
  // are built after the component-order shuffle, while the host reads the plan
  bool early = false;
  u64* m_tot = nullptr;
  DevBuf<u32> allow;
  if (!cached) {
    DevBuf<u32> L_cnt, hits;
    MX_CUDA_TRY(allow.alloc((long long)n_allow, s));
    MX_CUDA_TRY(mx_h2d(allow.p, mix->allow, sizeof(u32) * n_allow, s));
    ma.allow = allow.p;
    MX_CUDA_TRY(L_cnt.alloc(Km, s));
    MX_CUDA_TRY(cudaMemsetAsync(L_cnt.p, 0, sizeof(u32) * Km, s));  // stays 0 for an empty index
    MX_CUDA_TRY(hits.alloc(K > 0 ? K : 1, s));
    MX_CUDA_TRY(cudaMemsetAsync(hits.p, 0, sizeof(u32) * (K > 0 ? K : 1), s));
    MX_CUDA_TRY(g->scratch(S_MTOT, Km, &m_tot, s));
    MX_CUDA_TRY(cudaMemsetAsync(m_tot, 0, sizeof(u64) * Km, s));
    if (K > 0) {
      match_count_kernel<<<Km, 256, 0, s>>>(ma, L_cnt.p, hits.p, g->comp_total.p, g->consumed.p, m_tot);
      mx_count_launch();
    }
    std::vector<u32> h_cnt(Km), h_hits(K > 0 ? K : 1, 0);
    {
      D2HBatch rb(s);
      MX_CUDA_TRY(rb.add(h_cnt.data(), L_cnt.p, sizeof(u32) * Km));
      if (K > 0) MX_CUDA_TRY(rb.add(h_hits.data(), hits.p, sizeof(u32) * K));
      MX_CUDA_TRY(rb.sync());
    }
    g->match_off.assign(Km + 1, 0);
    for (int m = 0; m < Km; ++m) g->match_off[m + 1] = g->match_off[m] + h_cnt[m];
    g->match_shared = false;
    for (long long c = 0; c < K; ++c) g->match_shared |= h_hits[c] > 1;
    MX_CUDA_TRY(g->match_L_off.alloc(Km + 1, s));
    MX_CUDA_TRY(mx_h2d(g->match_L_off.p, g->match_off.data(), sizeof(u32) * (Km + 1), s));
    MX_CUDA_TRY(g->match_L.alloc(g->match_off[Km] > 0 ? g->match_off[Km] : 1, s));
    early = fresh && !g->match_shared && Km <= PLAN_SMEM_KM && !small && getenv("MX_PLAN_LATE") == nullptr;
    if (!early) MX_CUDA_TRY(match_fill(g, ma, s));
    g->match_allow.assign(mix->allow, mix->allow + n_allow);
    g->match_base.assign(mix->allow_base, mix->allow_base + ix->n_props);
    g->match_words = mix->allow_words;
  }
  const std::vector<u32>& h_off = g->match_off;
  const bool shared = g->match_shared;
  const DevBuf<u32>& L_off = g->match_L_off;
  const DevBuf<u32>& L = g->match_L;
  // ---- streams
  PlanWork w;
  w.mode = shared ? 1 : 0;
  w.chunk_size = mix->chunk_size;
  if (w.mode == 0) {
    w.n_streams = Km;
    w.s_off = L_off.p;
    const long long nseg = h_off[Km];
    MX_CUDA_TRY(g->scratch(S_SEGC, nseg, &w.seg_comp, s));
    MX_CUDA_TRY(g->scratch(S_SEGLO, nseg, &w.seg_lo, s));
    MX_CUDA_TRY(g->scratch(S_SEGPRE, nseg + Km, &w.seg_pre, s));
    if (!early) {
      build_segments_kernel<<<(Km + 3) / 4, 128, 0, s>>>(0, Km, w.s_off, L.p, g->comp_total.p, g->consumed.p,
                                                            w.seg_comp, w.seg_lo, w.seg_pre);
      mx_count_launch();
    }
  } else {
    w.n_streams = (int)K;
    std::vector<u32> so(K + 1);
    for (long long c = 0; c <= K; ++c) so[c] = (u32)c;
    MX_CUDA_TRY(g->scratch(S_SOFF, K + 1, &w.s_off, s));
    MX_CUDA_TRY(mx_h2d(w.s_off, so.data(), sizeof(u32) * (K + 1), s));
    MX_CUDA_TRY(g->scratch(S_SEGC, K, &w.seg_comp, s));
    MX_CUDA_TRY(g->scratch(S_SEGLO, K, &w.seg_lo, s));
    MX_CUDA_TRY(g->scratch(S_SEGPRE, 2 * K, &w.seg_pre, s));
    build_segments_kernel<<<(unsigned)std::min<long long>((K + 3) / 4, 148 * 16), 128, 0, s>>>(1, (int)K, w.s_off, nullptr, g->comp_total.p,
                                                                      g->consumed.p, w.seg_comp, w.seg_lo,
                                                                      w.seg_pre);
    mx_count_launch();
    MX_CUDA_TRY(cudaStreamSynchronize(s));
  }
  // ---- plan
  long long cap_phases, cap_terms;
  if (w.mode == 1) {
    cap_phases = max_chunks < (1 << 20) ? max_chunks : (1 << 20);
    cap_terms = cap_phases * 4 + (long long)Km + mix->chunk_size + 64;
  } else {
    cap_phases = 4 * (long long)Km + 64;
    if (cap_phases > max_chunks + 1) cap_phases = max_chunks + 1;
    cap_terms = cap_phases * (long long)Km;
    const long long term_budget = 1ll << 24;  // 512 MB of terms; the plan resumes on the next call
    if (cap_terms > term_budget) cap_terms = term_budget > Km ? term_budget : Km;
  }
  struct { Phase* p; } phases;
  struct { Term* p; } terms;
  struct { long long* p; } scratch_ll, out, report;
  struct { unsigned char* p; } flags;
  struct { u64* p; } pos;
  struct { int* p; } ap_idx;
  struct { double* p; } ap_frac;
  struct { u32* p; } front;
  MX_CUDA_TRY(g->scratch(S_PHASES, cap_phases, &phases.p, s));
  MX_CUDA_TRY(cudaMemsetAsync(phases.p, 0, sizeof(Phase) * cap_phases, s));  // copied back whole
  MX_CUDA_TRY(g->scratch(S_TERMS, cap_terms, &terms.p, s));
  MX_CUDA_TRY(g->scratch(S_LL, 5LL * Km, &scratch_ll.p, s));
  MX_CUDA_TRY(g->scratch(S_OUT, 4, &out.p, s));
  MX_CUDA_TRY(g->scratch(S_REPORT, Km, &report.p, s));
  MX_CUDA_TRY(g->scratch(S_FLAGS, 2LL * Km, &flags.p, s));
  MX_CUDA_TRY(g->scratch(S_POS, Km, &pos.p, s));
  MX_CUDA_TRY(g->scratch(S_APIDX, Km, &ap_idx.p, s));
  MX_CUDA_TRY(g->scratch(S_APFRAC, Km, &ap_frac.p, s));
  MX_CUDA_TRY(g->scratch(S_FRONT, Km, &front.p, s));
  MX_CUDA_TRY(cudaMemsetAsync(front.p, 0, sizeof(u32) * Km, s));
  MX_CUDA_TRY(cudaMemsetAsync(report.p, 0, sizeof(long long) * Km, s));
  PlanArgs pa{};
  pa.mode = w.mode;
  pa.Km = Km;
  pa.C = mix->chunk_size;
  pa.strict = mix->strict;
  pa.max_chunks = max_chunks;
  pa.w = wts_p;
  pa.slen = early ? m_tot : nullptr;  // early plan: stream lengths from the matching pass
  pa.seg_pre = w.seg_pre;
  pa.s_off = w.s_off;
  pa.L_off = L_off.p;
  pa.L = L.p;
  pa.comp_total = g->comp_total.p;
  pa.consumed = g->consumed.p;
  pa.front = front.p;
  pa.counts = scratch_ll.p;
  pa.rem = scratch_ll.p + Km;
  pa.found = scratch_ll.p + 2 * Km;
  pa.took = scratch_ll.p + 3 * Km;
  pa.ap_base = scratch_ll.p + 4 * Km;
  pa.dead = flags.p;
  pa.newly = flags.p + Km;
  pa.pos = pos.p;
  pa.ap_idx = ap_idx.p;
  pa.ap_frac = ap_frac.p;
  pa.phases = phases.p;
  pa.cap_phases = cap_phases;
  pa.terms = terms.p;
  pa.cap_terms = cap_terms;
  pa.out = out.p;
  pa.report = report.p;
  const bool big = w.mode == 0 && Km > PLAN_SMEM_KM && Km <= BIG_MAX_KM && mix->chunk_size < (1ll << 31) &&
                   getenv("MX_PLAN_SERIAL") == nullptr;
  if (big) {
    // keys by (weight desc, key asc) and each key's rank in that order
    std::vector<u32> ow(2 * (size_t)Km);
    for (int m = 0; m < Km; ++m) ow[m] = (u32)m;
    const double* wt = mix->weights;
    std::sort(ow.begin(), ow.begin() + Km, [wt](u32 x, u32 y) { return wt[x] != wt[y] ? wt[x] > wt[y] : x < y; });
    for (int r = 0; r < Km; ++r) ow[Km + ow[r]] = (u32)r;
    u32* order_w = front.p;
    u32* rank_w = reinterpret_cast<u32*>(ap_frac.p);
    MX_CUDA_TRY(mx_h2d(order_w, ow.data(), sizeof(u32) * Km, s));
    MX_CUDA_TRY(mx_h2d(rank_w, ow.data() + Km, sizeof(u32) * Km, s));
    BigArgs ba{};
    ba.Km = Km;
    ba.C = mix->chunk_size;
    ba.strict = mix->strict;
    ba.max_chunks = max_chunks;
    ba.w = wts_p;
    ba.order_w = order_w;
    ba.rank_w = rank_w;
    ba.seg_pre = w.seg_pre;
    ba.s_off = w.s_off;
    ba.pos = pos.p;
    ba.base = scratch_ll.p;
    ba.fkey = reinterpret_cast<unsigned long long*>(scratch_ll.p + Km);
    ba.slen = reinterpret_cast<u64*>(scratch_ll.p + 2 * Km);
    ba.counts = reinterpret_cast<int*>(scratch_ll.p + 3 * Km);
    ba.took = ba.counts + Km;
    ba.list = reinterpret_cast<u32*>(ap_idx.p);
    ba.phases = phases.p;
    ba.cap_phases = cap_phases;
    ba.terms = terms.p;
    ba.cap_terms = cap_terms;
    ba.out = out.p;
    ba.report = report.p;
    int dev = 0, optin = 0;
    MX_CUDA_TRY(cudaGetDevice(&dev));
    MX_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t base_smem = 9 * (size_t)Km + 4;
    const size_t staged = ((base_smem + 15) & ~(size_t)15) + 12 * (size_t)Km;
    cudaFuncAttributes fa{};
    MX_CUDA_TRY(cudaFuncGetAttributes(&fa, plan_big_kernel));
    const size_t dyn_max = (size_t)optin - fa.sharedSizeBytes;
    const int stage_w = staged <= dyn_max ? 1 : 0;
    const size_t smem = stage_w ? staged : base_smem;
    static size_t smem_set = 0;
    if (smem > smem_set) {
      MX_CUDA_TRY(cudaFuncSetAttribute(plan_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max));
      smem_set = dyn_max;
    }
    DevBuf<unsigned long long> stats;
    const bool want_stats = getenv("MX_PLAN_STATS") != nullptr;
    if (want_stats) {
      MX_CUDA_TRY(stats.alloc(16, s));
      MX_CUDA_TRY(cudaMemsetAsync(stats.p, 0, 16 * sizeof(unsigned long long), s));
      ba.stats = stats.p;
    }
    plan_big_kernel<<<1, BIG_THREADS, smem, s>>>(ba, stage_w);
    if (want_stats) {
      unsigned long long h[16];
      MX_CUDA_TRY(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, s));
      MX_CUDA_TRY(cudaStreamSynchronize(s));
      fprintf(stderr,
              "plan_big: cycles pass %llu list %llu redistribute %llu exact %llu phase %llu | passes %llu dead %llu "
              "exact %llu phases %llu | apportion: sequential-sum cycles %llu rest %llu, sequential sums %llu\n",
              h[0], h[1], h[2], h[3], h[4], h[8], h[9], h[10], h[11], h[12], h[13], h[14]);
    }
  } else {
    plan_kernel<<<1, 32, 0, s>>>(pa);
  }
  mx_count_launch();
  if (small) {
    // small plan: emission driven by device-side counts, one host sync
    MX_CUDA_TRY(cudaEventRecord(g->ev_seg, s));
    MX_CUDA_TRY(cudaStreamWaitEvent(ms, g->ev_seg, 0));
    ph_plan.reset();
    s = ms;
    if (w.mode == 0) {
      commit_segments_kernel<<<Km, 128, 0, s>>>(Km, w.s_off, w.seg_comp, w.seg_lo, w.seg_pre, pos.p,
                                                g->consumed.p);
      mx_count_launch();
    }
    EmitArgs a{};
    a.phases = phases.p;
    a.terms = terms.p;
    a.s_off = w.s_off;
    a.seg_comp = w.seg_comp;
    a.seg_lo = w.seg_lo;
    a.seg_pre = w.seg_pre;
    a.arbitrary = 0;
    a.key_blk_first = ix->key_blk_first.p;
    a.blk_first = ix->blk_first.p;
    a.civ = g->civ.p;
    a.cfile = g->cfile.p;
    a.cstart = g->cstart.p;
    a.ccum = g->ccum.p;
    a.iv_start = ix->iv_start.p;
    a.iv_end = ix->iv_end.p;
    a.iv_file = ix->iv_file.p;
    a.lcnt = g->lcnt.p;
    a.lpos = g->lpos.p;
    a.lstart = g->lstart.p;
    const long long slots = max_chunks * NM_CAP;
    struct { u32* p; } gm, gf, gs, ge, ovf;
    struct { u64* p; } cnt;
    struct { long long* p; } header;
    MX_CUDA_TRY(g->scratch(S_GM, slots, &gm.p, s));
    MX_CUDA_TRY(g->scratch(S_GF, slots, &gf.p, s));
    MX_CUDA_TRY(g->scratch(S_GS, slots, &gs.p, s));
    MX_CUDA_TRY(g->scratch(S_GE, slots, &ge.p, s));
    MX_CUDA_TRY(g->scratch(S_OVF, 1, &ovf.p, s));
    MX_CUDA_TRY(g->scratch(S_CNT, max_chunks, &cnt.p, s));
    MX_CUDA_TRY(g->scratch(S_HDR, 3, &header.p, s));
    MX_CUDA_TRY(cudaMemsetAsync(ovf.p, 0, sizeof(u32), s));
    MX_CUDA_TRY(g->res_off.reserve(max_chunks + 1, s));
    MX_CUDA_TRY(g->res_seed.reserve(max_chunks, s));
    MX_CUDA_TRY(g->res_id.reserve(max_chunks, s));
    MX_CUDA_TRY(g->res_mkey.reserve(slots, s));
    MX_CUDA_TRY(g->res_file.reserve(slots, s));
    MX_CUDA_TRY(g->res_start.reserve(slots, s));
    MX_CUDA_TRY(g->res_end.reserve(slots, s));
    {
      MxPhase ph("emit", s);
      emit_small_kernel<<<(unsigned)max_chunks, NM_THREADS, 0, s>>>(a, out.p, gm.p, gf.p, gs.p, ge.p, cnt.p, ovf.p);
      mx_count_launch();
      finalize_small_kernel<<<1, 256, 0, s>>>(out.p, cnt.p, gm.p, gf.p, gs.p, ge.p, g->res_mkey.p, g->res_file.p,
                                              g->res_start.p, g->res_end.p, g->res_off.p, g->res_seed.p, g->res_id.p,
                                              g->next_chunk_id, g->chunk_prefix.p, g->chunk_prefix_len, header.p);
      mx_count_launch();
    }
    // one pinned host mirror of the whole result, copied in the same sync
    const long long mirror = 8 * (3 + 1) + (long long)(max_chunks + 1) * 8 + (long long)max_chunks * 16 +
                             slots * 16 + Km * 8;
    if (g->h_small_bytes < mirror) {
      if (g->h_small) cudaFreeHost(g->h_small);
      g->h_small = nullptr;
      MX_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&g->h_small), mirror));
      g->h_small_bytes = mirror;
    }
    unsigned char* hp = g->h_small;
    long long* hdr = reinterpret_cast<long long*>(hp);
    u32* h_ovf_p = reinterpret_cast<u32*>(hp + 24);
    unsigned char* body = hp + 32;
    MX_CUDA_TRY(cudaMemcpyAsync(hdr, header.p, 3 * sizeof(long long), cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaMemcpyAsync(h_ovf_p, ovf.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaMemcpyAsync(body, g->res_off.p, sizeof(long long) * (max_chunks + 1), cudaMemcpyDeviceToHost, s));
    body += sizeof(long long) * (max_chunks + 1);
    MX_CUDA_TRY(cudaMemcpyAsync(body, g->res_seed.p, sizeof(u64) * max_chunks, cudaMemcpyDeviceToHost, s));
    body += sizeof(u64) * max_chunks;
    MX_CUDA_TRY(cudaMemcpyAsync(body, g->res_id.p, sizeof(long long) * max_chunks, cudaMemcpyDeviceToHost, s));
    body += sizeof(long long) * max_chunks;
    for (u32* src : {g->res_mkey.p, g->res_file.p, g->res_start.p, g->res_end.p}) {
      MX_CUDA_TRY(cudaMemcpyAsync(body, src, sizeof(u32) * slots, cudaMemcpyDeviceToHost, s));
      body += sizeof(u32) * slots;
    }
    MX_CUDA_TRY(cudaMemcpyAsync(g->report.data(), report.p, sizeof(long long) * Km, cudaMemcpyDeviceToHost, s));
    MX_CUDA_TRY(cudaStreamSynchronize(s));
    const u32 h_ovf = *h_ovf_p;
    g->h_small_valid = hdr[0];
    g->h_small_cap = max_chunks;
    g->h_small_slots = slots;
    MX_CUDA_TRY(cudaGetLastError());
    if (h_ovf) return mx_fail(MX_ERR_UNSUPPORTED, "a chunk has %u ranges before merging (> %d supported)", h_ovf, NM_CAP);
    g->res_chunks = hdr[0];
    g->res_ranges = hdr[1];
    g->next_chunk_id += hdr[0];
    *n_out = hdr[0];
    return hdr[2] ? MX_EXHAUSTED : MX_OK;
  }
  long long h_out[4];
  std::vector<Phase> h_phases(cap_phases);
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(h_out, out.p, sizeof(h_out)));
    MX_CUDA_TRY(rb.add(g->report.data(), report.p, sizeof(long long) * Km));
    MX_CUDA_TRY(rb.add(h_phases.data(), phases.p, sizeof(Phase) * cap_phases));
    if (early) {
      // the plan's result travels while the ordered lists and segment tables
      // are built behind the component-order shuffle
      MX_CUDA_TRY(cudaEventRecord(g->ev_plan, s));
      MX_CUDA_TRY(match_fill(g, ma, s));
      build_segments_kernel<<<(Km + 3) / 4, 128, 0, s>>>(0, Km, w.s_off, L.p, g->comp_total.p, g->consumed.p,
                                                            w.seg_comp, w.seg_lo, w.seg_pre);
      mx_count_launch();
      MX_CUDA_TRY(cudaGetLastError());
      MX_CUDA_TRY(rb.sync_event(g->ev_plan));
    } else {
      MX_CUDA_TRY(rb.sync());
    }
  }
  ph_plan.reset();
  MX_CUDA_TRY(cudaEventRecord(g->ev_seg, s));
  MX_CUDA_TRY(cudaStreamWaitEvent(ms, g->ev_seg, 0));
  s = ms;
  if (w.mode == 0) {
    commit_segments_kernel<<<Km, 128, 0, s>>>(Km, w.s_off, w.seg_comp, w.seg_lo, w.seg_pre, pos.p,
                                              g->consumed.p);
    mx_count_launch();
  }
  const long long n_seg = w.mode == 0 ? (long long)h_off[Km] : K;
  w.max_mkey = Km;
  int rc = emit(g, w, phases.p, h_phases.data(), terms.p, h_out[0], h_out[1], n_seg, s);
  if (rc != MX_OK) return rc;
  *n_out = h_out[0];
  return h_out[3] ? MX_EXHAUSTED : MX_OK;
}

int plan_arbitrary(GenData* g, long long chunk_size, long long max_chunks, long long* n_out) {
  cudaStream_t s = g->stream;
  const long long K = g->K;
  *n_out = 0;
  if (chunk_size < 1) return mx_fail(MX_ERR_MIXTURE, "chunk_size must be positive");
  g->last_mkeys = 0;
  g->report.clear();
  PlanWork w;
  w.mode = 2;
  w.chunk_size = chunk_size;
  w.n_streams = 1;
  if (K == 0) {
    int rc = emit(g, w, nullptr, nullptr, nullptr, 0, 0, 0, s);
    return rc != MX_OK ? rc : MX_EXHAUSTED;
  }
  std::vector<u32> so = {0u, (u32)K};
  MX_CUDA_TRY(g->scratch(S_SOFF, 2, &w.s_off));
  MX_CUDA_TRY(mx_h2d(w.s_off, so.data(), sizeof(u32) * 2, s));
  MX_CUDA_TRY(g->scratch(S_SEGC, K, &w.seg_comp));
  MX_CUDA_TRY(g->scratch(S_SEGLO, K, &w.seg_lo));
  MX_CUDA_TRY(g->scratch(S_SEGPRE, K + 1, &w.seg_pre));
  build_segments_kernel<<<1, 32, 0, s>>>(2, 1, w.s_off, g->comp_order.p, g->comp_total.p, g->consumed.p,
                                         w.seg_comp, w.seg_lo, w.seg_pre);
  mx_count_launch();
  DevBuf<Phase> phases;
  DevBuf<Term> terms;
  DevBuf<long long> out;
  DevBuf<u64> pos;
  MX_CUDA_TRY(phases.alloc(2, s));
  MX_CUDA_TRY(terms.alloc(2, s));
  MX_CUDA_TRY(out.alloc(4, s));
  MX_CUDA_TRY(pos.alloc(1, s));
  plan_arbitrary_kernel<<<1, 32, 0, s>>>(w.seg_pre, K, chunk_size, max_chunks, phases.p, terms.p, out.p, pos.p);
  mx_count_launch();
  long long h_out[4];
  Phase h_phases[2];
  {
    D2HBatch rb(s);
    MX_CUDA_TRY(rb.add(h_out, out.p, sizeof(h_out)));
    MX_CUDA_TRY(rb.add(h_phases, phases.p, sizeof(h_phases)));
    MX_CUDA_TRY(rb.sync());
  }
  commit_segments_kernel<<<1, 128, 0, s>>>(1, w.s_off, w.seg_comp, w.seg_lo, w.seg_pre, pos.p, g->consumed.p);
  mx_count_launch();
  w.max_mkey = K;  // arbitrary chunks: pieces carry component ids
  int rc = emit(g, w, phases.p, h_phases, terms.p, h_out[0], h_out[1], K, s);
  if (rc != MX_OK) return rc;
  *n_out = h_out[0];
  return h_out[3] ? MX_EXHAUSTED : MX_OK;
}

}  // namespace mx
