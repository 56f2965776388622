// Stage 3 -- ADO feedback on sm_100a.
//
//  * domain_loss_kernel: per_domain_loss (client.py:582-598) as a one-pass
//    segmented reduction: per warp, lanes holding the same tag are grouped
//    with __match_any_sync and summed by the group leader in lane order into
//    a warp-private shared-memory accumulator; warps, then CTAs, are combined
//    in a fixed order, so the f64 sums are bit-reproducible run to run.
//    For <= 32 domains (the ADO case: 22 Pile domains) domain_loss_priv_kernel
//    replaces it: every thread owns a private shared-memory row of K (f64 sum,
//    u32 count) bins and 32 consecutive tokens per tile (16-byte loads), keeps
//    the current same-tag run in registers and flushes it to its bin when the
//    tag changes (ADO batches are single-domain sequences); no atomics or warp
//    votes; rows are combined per domain in a fixed order, so the sums stay
//    run-to-run reproducible. HBM-bound: B3 = T x (4 + 4) bytes.
//  * fit_kernel: fit_power_law (ado.py:121-168), one CTA per domain, one warp
//    per epsilon candidate (grid of 50, then a 201-point linspace refinement),
//    closed-form log-linear regression + SSE in f64, strict-< argmin with
//    first-index tie-break exactly like the reference loops.
//  * pi_kernel / credit_kernel: AdoState.compute_pi/_floored and the credit
//    update (ado.py:241-243, 273-319) with CPython's compensated sum.
// The whole library is built with --fmad=false so a*b+c is never contracted:
// the f64 arithmetic follows the reference's operation order.
#include <math.h>

#include "common.cuh"
#include "mixtera_internal.cuh"

namespace mx {

constexpr int DL_THREADS = 256;
constexpr int DL_WARPS = DL_THREADS / 32;
constexpr int DL_MAXK = 256;  // domains held in shared memory per warp

__global__ void __launch_bounds__(DL_THREADS)
domain_loss_kernel(const float* loss, const int32_t* tags, long long n, int K, long long per_block,
                   double* part_sum, long long* part_cnt, u32* bad) {
  __shared__ double s_sum[DL_WARPS][DL_MAXK];
  __shared__ long long s_cnt[DL_WARPS][DL_MAXK];
  __shared__ float s_val[DL_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = lane; k < K; k += 32) {
    s_sum[w][k] = 0.0;
    s_cnt[w][k] = 0;
  }
  __syncwarp();
  const long long b0 = blockIdx.x * per_block;
  const long long b1 = b0 + per_block < n ? b0 + per_block : n;
  const long long per_warp = (per_block + DL_WARPS - 1) / DL_WARPS;
  const long long w0 = b0 + w * per_warp;
  const long long w1 = w0 + per_warp < b1 ? w0 + per_warp : b1;
  for (long long base = w0; base < w1; base += 32) {
    const long long i = base + lane;
    const bool ok = i < w1;
    int t = ok ? tags[i] : -1;
    float v = ok ? loss[i] : 0.f;
    if (ok && (t < 0 || t >= K)) {
      atomicOr(bad, 1u);
      t = -1;
    }
    s_val[w][lane] = v;
    __syncwarp();
    const u32 peers = __match_any_sync(MX_FULL, t);
    if (t >= 0 && (peers & ((1u << lane) - 1)) == 0) {  // group leader, lane order sum
      double acc = s_sum[w][t];
      u32 m = peers;
      while (m) {
        int l = __ffs(m) - 1;
        acc += (double)s_val[w][l];
        m &= m - 1;
      }
      s_sum[w][t] = acc;
      s_cnt[w][t] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += DL_THREADS) {
    double s = 0.0;
    long long c = 0;
    for (int x = 0; x < DL_WARPS; ++x) {
      s += s_sum[x][k];
      c += s_cnt[x][k];
    }
    part_sum[(long long)blockIdx.x * K + k] = s;
    part_cnt[(long long)blockIdx.x * K + k] = c;
  }
}

constexpr int DLP_THREADS = 256;
constexpr int DLP_MAXK = 32;
constexpr int DLP_RUN = 32;  // consecutive tokens per thread per tile

__global__ void __launch_bounds__(DLP_THREADS)
domain_loss_priv_kernel(const float* __restrict__ loss, const int32_t* __restrict__ tags, long long n, int K,
                        double* part_sum, long long* part_cnt, u32* bad) {
  extern __shared__ __align__(16) unsigned char dlp_dyn[];
  double* s_sum = reinterpret_cast<double*>(dlp_dyn);                            // [K][DLP_THREADS]
  u32* s_cnt = reinterpret_cast<u32*>(dlp_dyn + sizeof(double) * K * DLP_THREADS);  // [K][DLP_THREADS]
  const int tid = threadIdx.x;
  for (int k = 0; k < K; ++k) {
    s_sum[k * DLP_THREADS + tid] = 0.0;
    s_cnt[k * DLP_THREADS + tid] = 0;
  }
  u32 badv = 0;
  // a thread owns DLP_RUN consecutive tokens per tile and keeps the running
  // (tag, sum, count) of the current same-tag run in registers, flushing to
  // its shared-memory bin when the tag changes: ADO batches are sequences of
  // thousands of single-domain tokens, so flushes are rare
  int cur_t = -1;
  double cur_s = 0.0;
  u32 cur_c = 0;
  auto flush = [&]() {
    if (cur_c) {
      s_sum[cur_t * DLP_THREADS + tid] += cur_s;
      s_cnt[cur_t * DLP_THREADS + tid] += cur_c;
    }
  };
  auto add = [&](int t, float v) {
    if ((unsigned)t >= (unsigned)K) {
      badv = 1;
      return;
    }
    if (t != cur_t) {
      flush();
      cur_t = t;
      cur_s = 0.0;
      cur_c = 0;
    }
    cur_s += (double)v;
    ++cur_c;
  };
  const bool vec = ((reinterpret_cast<uintptr_t>(loss) | reinterpret_cast<uintptr_t>(tags)) & 15) == 0;
  // a warp owns 32 * DLP_RUN consecutive tokens per tile; step q, lane l reads
  // tokens [q * 128 + 4l, +4): coalesced 16-byte loads, and a lane's tokens
  // stay inside one sequence for many steps
  const long long tile = (long long)DLP_THREADS * DLP_RUN;
  const int ln = tid & 31, wp = tid >> 5;
  for (long long t0 = (long long)blockIdx.x * tile; t0 < n; t0 += (long long)gridDim.x * tile) {
    const long long wb = t0 + (long long)wp * 32 * DLP_RUN;
    if (vec && wb + 32 * DLP_RUN <= n) {
#pragma unroll 4
      for (int q = 0; q < DLP_RUN / 4; ++q) {
        const long long i = wb + q * 128 + 4 * ln;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(loss + i));
        const int4 t = __ldcs(reinterpret_cast<const int4*>(tags + i));
        add(t.x, v.x);
        add(t.y, v.y);
        add(t.z, v.z);
        add(t.w, v.w);
      }
    } else {
      for (int q = 0; q < DLP_RUN / 4; ++q)
        for (int r = 0; r < 4; ++r) {
          const long long j = wb + q * 128 + 4 * ln + r;
          if (j < n) add(tags[j], loss[j]);
        }
    }
  }
  flush();
  if (badv) atomicOr(bad, 1u);
  __syncthreads();
  // fixed-order combine: warp w sums domains k = w, w + 8, ...; lanes take
  // threads lane, lane + 32, ... then a fixed shuffle tree
  const int lane = tid & 31, w = tid >> 5;
  for (int k = w; k < K; k += DLP_THREADS / 32) {
    double sv = 0.0;
    long long cv = 0;
    for (int x = lane; x < DLP_THREADS; x += 32) {
      sv += s_sum[k * DLP_THREADS + x];
      cv += s_cnt[k * DLP_THREADS + x];
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      sv += __shfl_xor_sync(MX_FULL, sv, d);
      cv += __shfl_xor_sync(MX_FULL, cv, d);
    }
    if (lane == 0) {
      part_sum[(long long)blockIdx.x * K + k] = sv;
      part_cnt[(long long)blockIdx.x * K + k] = cv;
    }
  }
}

__global__ void domain_loss_final(const double* part_sum, const long long* part_cnt, int blocks, int K, double* sums,
                                  long long* counts) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double s = 0.0;
  long long c = 0;
  for (int b = 0; b < blocks; ++b) {
    s += part_sum[(long long)b * K + k];
    c += part_cnt[(long long)b * K + k];
  }
  sums[k] = s;
  counts[k] = c;
}

// ------------------------------------------------------------------ fit
constexpr int FIT_THREADS = 256;
constexpr int FIT_WARPS = FIT_THREADS / 32;
constexpr int FIT_MAXP = 8192;  // points per domain held in (dynamic) shared memory

struct FitEval {
  bool ok;
  double alpha, beta, sse;
};

// _loglinear (ado.py:93-118) evaluated by one warp
__device__ FitEval loglinear_warp(double eps, const double* n, const double* loss, const double* lx, int P) {
  const int lane = threadIdx.x & 31;
  FitEval r{false, 0, 0, 0};
  bool bad = false;
  double sy = 0.0, sx = 0.0;
  for (int i = lane; i < P; i += 32) {
    double res = loss[i] - eps;
    bad |= !(res > 0.0);
    if (res > 0.0) sy += log(res);
    sx += lx[i];
  }
  if (__any_sync(MX_FULL, bad)) return r;
  sy = warp_sum(sy);
  sx = warp_sum(sx);
  const double xm = sx / (double)P, ym = sy / (double)P;
  double sxx = 0.0, sxy = 0.0;
  for (int i = lane; i < P; i += 32) {
    double dx = lx[i] - xm;
    double dy = log(loss[i] - eps) - ym;
    sxx += dx * dx;
    sxy += dx * dy;
  }
  sxx = warp_sum(sxx);
  sxy = warp_sum(sxy);
  if (sxx == 0.0) return r;
  const double slope = sxy / sxx;
  if (slope >= 0.0) return r;
  const double intercept = ym - slope * xm;
  const double alpha = -slope;
  const double beta = exp(intercept);
  double sse = 0.0;
  for (int i = lane; i < P; i += 32) {
    double pred = eps + beta * pow(n[i], -alpha);
    double d = pred - loss[i];
    sse += d * d;
  }
  sse = warp_sum(sse);
  r.ok = true;
  r.alpha = alpha;
  r.beta = beta;
  r.sse = sse;
  return r;
}

__global__ void __launch_bounds__(FIT_THREADS)
fit_kernel(const long long* off, const double* n_all, const double* loss_all, const double* geom, double* out,
           int maxp) {
  extern __shared__ double s_pts[];
  __shared__ double s_cand[64];
  __shared__ int s_nc;
  __shared__ double s_sse[256], s_a[256], s_b[256];
  __shared__ int s_ok[256];
  const int d = blockIdx.x;
  const long long p0 = off[d];
  const int P = (int)(off[d + 1] - p0);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* o = out + 4ll * d;
  if (P < 8 || P > FIT_MAXP || P > maxp) {
    if (threadIdx.x == 0) o[0] = o[1] = o[2] = o[3] = nan("");
    return;
  }
  double* s_n = s_pts;
  double* s_l = s_pts + maxp;
  double* s_x = s_pts + 2 * maxp;
  for (int i = threadIdx.x; i < P; i += FIT_THREADS) {
    s_n[i] = n_all[p0 + i];
    s_l[i] = loss_all[p0 + i];
    s_x[i] = log(s_n[i]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = s_l[0];
    for (int i = 1; i < P; ++i) mn = s_l[i] < mn ? s_l[i] : mn;
    const double hi = 0.999 * mn;
    double c[50];
    int nc = 0;
    c[nc++] = 0.0;
    if (hi > 0.0)
      for (int g = 0; g < 49; ++g) c[nc++] = hi * (1.0 - geom[g]);
    // sorted(set(...)): insertion sort + dedup
    for (int x = 1; x < nc; ++x) {
      double v = c[x];
      int y = x - 1;
      while (y >= 0 && c[y] > v) {
        c[y + 1] = c[y];
        --y;
      }
      c[y + 1] = v;
    }
    int u = 0;
    for (int x = 0; x < nc; ++x)
      if (u == 0 || c[x] != s_cand[u - 1]) s_cand[u++] = c[x];
    s_nc = u;
  }
  __syncthreads();
  const int nc = s_nc;
  for (int ci = w; ci < nc; ci += FIT_WARPS) {
    FitEval f = loglinear_warp(s_cand[ci], s_n, s_l, s_x, P);
    if (lane == 0) {
      s_ok[ci] = f.ok;
      s_sse[ci] = f.sse;
      s_a[ci] = f.alpha;
      s_b[ci] = f.beta;
    }
  }
  __syncthreads();
  __shared__ int s_best;
  __shared__ double s_bsse, s_beps, s_ba, s_bb;
  __shared__ double s_lo, s_hi;
  if (threadIdx.x == 0) {
    int best = -1;
    for (int ci = 0; ci < nc; ++ci)
      if (s_ok[ci] && (best < 0 || s_sse[ci] < s_sse[best])) best = ci;
    s_best = best;
    if (best >= 0) {
      s_bsse = s_sse[best];
      s_beps = s_cand[best];
      s_ba = s_a[best];
      s_bb = s_b[best];
      s_lo = s_cand[best > 0 ? best - 1 : 0];
      s_hi = s_cand[best + 1 < nc ? best + 1 : nc - 1];
    }
  }
  __syncthreads();
  if (s_best < 0) {
    if (threadIdx.x == 0) {
      double mn = s_l[0];
      for (int i = 1; i < P; ++i) mn = s_l[i] < mn ? s_l[i] : mn;
      double b = s_l[0] - mn;
      o[0] = mn;
      o[1] = b > 1e-12 ? b : 1e-12;
      o[2] = 1e-6;
      o[3] = 1.0;
    }
    return;
  }
  const double lo = s_lo, hi = s_hi;
  if (hi > lo) {
    const double step = (hi - lo) / 200.0;
    for (int ci = w; ci < 201; ci += FIT_WARPS) {
      double eps = ci == 200 ? hi : (step == 0.0 ? ((double)ci / 200.0) * (hi - lo) : (double)ci * step) + lo;
      FitEval f = loglinear_warp(eps, s_n, s_l, s_x, P);
      if (lane == 0) {
        s_ok[ci] = f.ok;
        s_sse[ci] = f.sse;
        s_a[ci] = f.alpha;
        s_b[ci] = f.beta;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bs = s_bsse, be = s_beps, ba = s_ba, bb = s_bb;
      for (int ci = 0; ci < 201; ++ci) {
        if (s_ok[ci] && s_sse[ci] < bs) {
          bs = s_sse[ci];
          be = ci == 200 ? hi : (step == 0.0 ? ((double)ci / 200.0) * (hi - lo) : (double)ci * step) + lo;
          ba = s_a[ci];
          bb = s_b[ci];
        }
      }
      s_beps = be;
      s_ba = ba;
      s_bb = bb;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    o[0] = s_beps;
    o[1] = s_bb;
    o[2] = s_ba;
    o[3] = 0.0;
  }
}

// ------------------------------------------------------------------ pi
__device__ double neumaier_sum(const double* x, int n) {
  double s = 0.0, c = 0.0;
  for (int i = 0; i < n; ++i) {
    double v = x[i];
    double t = s + v;
    if (fabs(s) >= fabs(v)) c += (s - t) + v;
    else c += (v - t) + s;
    s = t;
  }
  return c != 0.0 ? s + c : s;
}

constexpr int PI_MAXK = 1024;

// _floored (ado.py:273-291) in place on out[0..k)
__device__ void floored(double* out, int k, double p_min, unsigned char* fixed, double* tmp) {
  for (int i = 0; i < k; ++i) fixed[i] = 0;
  int n_fixed = 0;
  while (true) {
    bool any = false;
    for (int i = 0; i < k; ++i)
      if (!fixed[i] && out[i] < p_min) {
        fixed[i] = 2;  // newly low
        any = true;
      }
    if (!any) return;
    for (int i = 0; i < k; ++i)
      if (fixed[i] == 2) {
        fixed[i] = 1;
        ++n_fixed;
      }
    int nf = 0;
    for (int i = 0; i < k; ++i)
      if (!fixed[i]) tmp[nf++] = out[i];
    if (nf == 0) {
      for (int i = 0; i < k; ++i) out[i] = 1.0 / (double)k;
      return;
    }
    const double budget = 1.0 - p_min * (double)n_fixed;
    const double mass = neumaier_sum(tmp, nf);
    for (int i = 0; i < k; ++i) {
      if (fixed[i]) out[i] = p_min;
      else out[i] = mass > 0.0 ? out[i] / mass * budget : budget / (double)nf;
    }
  }
}

__global__ void pi_kernel(int k, const double* mu, const double* credit, const double* law, double n, double p_min,
                          double smoothing, double* pi_bar, long long* pi_bar_count, double* pi) {
  __shared__ double s_v[PI_MAXK], s_tmp[PI_MAXK];
  __shared__ unsigned char s_fix[PI_MAXK];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < k; ++i) {
    const double* L = law + 4ll * i;
    double speed = 0.0;
    if (L[2] == L[2]) speed = L[2] * L[1] * pow(n, -(L[2] + 1.0));  // alpha * beta * n^-(alpha+1)
    s_v[i] = mu[i] * credit[i] * speed;
  }
  const double total = neumaier_sum(s_v, k);
  if (!(total > 0.0)) {
    for (int i = 0; i < k; ++i) s_v[i] = mu[i];
  } else {
    for (int i = 0; i < k; ++i) s_v[i] = (1.0 - smoothing) * (s_v[i] / total) + smoothing * pi_bar[i];
  }
  floored(s_v, k, p_min, s_fix, s_tmp);
  const double c = (double)*pi_bar_count;
  for (int i = 0; i < k; ++i) {
    pi[i] = s_v[i];
    pi_bar[i] = (pi_bar[i] * c + s_v[i]) / (c + 1.0);
  }
  *pi_bar_count += 1;
}

__global__ void credit_kernel(int k, double rate, const double* pi, double* credit) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) credit[i] = (1.0 - rate) * credit[i] + rate * pi[i];
}

// ------------------------------------------------------------------ host
int domain_loss(const float* losses, const int32_t* tags, long long n, int K, double* sums, long long* counts,
                cudaStream_t s) {
  if (K < 1 || K > DL_MAXK) return mx_fail(MX_ERR_UNSUPPORTED, "n_domains=%d outside [1, %d]", K, DL_MAXK);
  const bool priv = K <= DLP_MAXK;
  long long per_block = 16384;
  int blocks;
  if (priv) {  // one wave of resident CTAs (grid-stride over 8K-token tiles)
    int dev = 0, n_sm = 148, occ = 1;
    MX_CUDA_TRY(cudaGetDevice(&dev));
    MX_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = (sizeof(double) + sizeof(u32)) * (size_t)K * DLP_THREADS;
    if (smem > 48 * 1024)
      MX_CUDA_TRY(cudaFuncSetAttribute(domain_loss_priv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((sizeof(double) + sizeof(u32)) * DLP_MAXK * DLP_THREADS)));
    MX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, domain_loss_priv_kernel, DLP_THREADS, smem));
    blocks = (int)std::min<long long>((n + DLP_THREADS * DLP_RUN - 1) / (DLP_THREADS * DLP_RUN),
                                      (long long)n_sm * std::max(occ, 1));
  } else {
    blocks = (int)((n + per_block - 1) / per_block);
  }
  if (blocks < 1) blocks = 1;
  DevBuf<double> ps;
  DevBuf<long long> pc;
  DevBuf<u32> bad;
  MX_CUDA_TRY(ps.alloc((long long)blocks * K, s));
  MX_CUDA_TRY(pc.alloc((long long)blocks * K, s));
  MX_CUDA_TRY(bad.alloc(1, s));
  MX_CUDA_TRY(cudaMemsetAsync(bad.p, 0, sizeof(u32), s));
  if (priv) {
    const size_t smem = (sizeof(double) + sizeof(u32)) * (size_t)K * DLP_THREADS;
    domain_loss_priv_kernel<<<blocks, DLP_THREADS, smem, s>>>(losses, tags, n, K, ps.p, pc.p, bad.p);
  } else {
    domain_loss_kernel<<<blocks, DL_THREADS, 0, s>>>(losses, tags, n, K, per_block, ps.p, pc.p, bad.p);
  }
  mx_count_launch();
  domain_loss_final<<<(K + 127) / 128, 128, 0, s>>>(ps.p, pc.p, blocks, K, sums, counts);
  mx_count_launch();
  u32 h_bad = 0;
  MX_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  MX_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_bad) return mx_fail(MX_ERR_DATA, "a domain tag lies outside [0, %d)", K);
  return MX_OK;
}

int fit_power_law(int D, const long long* off, const double* n, const double* loss, const double* geom, double* out,
                  cudaStream_t s) {
  if (D < 1) return MX_OK;
  std::vector<long long> h(D + 1);
  MX_CUDA_TRY(cudaMemcpyAsync(h.data(), off, sizeof(long long) * (D + 1), cudaMemcpyDeviceToHost, s));
  MX_CUDA_TRY(cudaStreamSynchronize(s));
  long long maxp = 8;
  for (int d = 0; d < D; ++d) maxp = std::max(maxp, h[d + 1] - h[d]);
  if (maxp > FIT_MAXP) return mx_fail(MX_ERR_UNSUPPORTED, "%lld fit points per domain (> %d)", maxp, FIT_MAXP);
  const size_t smem = sizeof(double) * 3 * (size_t)maxp;
  MX_CUDA_TRY(cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fit_kernel<<<D, FIT_THREADS, smem, s>>>(off, n, loss, geom, out, (int)maxp);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

int ado_pi(int k, const double* mu, const double* credit, const double* law, double n, double p_min, double smoothing,
           double* pi_bar, long long* cnt, double* pi, cudaStream_t s) {
  if (k < 1 || k > PI_MAXK) return mx_fail(MX_ERR_UNSUPPORTED, "domains=%d outside [1, %d]", k, PI_MAXK);
  pi_kernel<<<1, 32, 0, s>>>(k, mu, credit, law, n, p_min, smoothing, pi_bar, cnt, pi);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

int ado_credit(int k, double rate, const double* pi, double* credit, cudaStream_t s) {
  credit_kernel<<<(k + 127) / 128, 128, 0, s>>>(k, rate, pi, credit);
  mx_count_launch();
  MX_CUDA_TRY(cudaGetLastError());
  return MX_OK;
}

}  // namespace mx
