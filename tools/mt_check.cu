// Debug harness: scalar MT vs WarpMT shuffles must agree bit for bit.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/mt_check tools/mt_check.cu
#include <cstdio>
#include <vector>

#include "../paper_2502_19790_b200/csrc/mt19937.cuh"

using namespace mx;

__global__ void ref_kernel(const unsigned long long* seeds, int n, uint32_t* out) {
  __shared__ uint32_t st[MT_N];
  if (threadIdx.x != 0) return;
  MT mt;
  mt.s = st;
  mt.seed_u64(seeds[blockIdx.x]);
  uint32_t* x = out + (long long)blockIdx.x * n;
  for (int i = 0; i < n; ++i) x[i] = i;
  mt.shuffle(x, n);
}

__global__ void warp_kernel(const unsigned long long* seeds, int n, const uint32_t* base, uint32_t* out) {
  __shared__ uint32_t st[4][MT_N], buf[4][MT_N];
  __shared__ uint2 pairs[4][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + w;
  uint32_t* x = out + (long long)b * n;
  for (int i = lane; i < n; i += 32) x[i] = i;
  __syncwarp();
  WarpMT mt{st[w], buf[w], pairs[w], MT_N};
  mt.seed(base, seeds[b]);
  mt.shuffle(x, 1);
  mt.shuffle(x, n);
}

int timing_main();

int main() {
  timing_main();
  const int B = 64;
  for (int n : {2, 3, 20, 700, 2000, 6000, 70000}) {
    std::vector<unsigned long long> seeds(B);
    for (int i = 0; i < B; ++i) seeds[i] = i % 2 ? 0x9e3779b97f4a7c15ull * (i + 1) >> 1 : 12345ull * i + 7;
    unsigned long long* ds;
    uint32_t *o1, *o2, *base;
    cudaMalloc(&ds, 8 * B);
    cudaMalloc(&o1, 4ll * B * n);
    cudaMalloc(&o2, 4ll * B * n);
    cudaMalloc(&base, 4 * MT_N);
    uint32_t hb[MT_N];
    mt_base_table(hb);
    cudaMemcpy(base, hb, sizeof(hb), cudaMemcpyHostToDevice);
    cudaMemcpy(ds, seeds.data(), 8 * B, cudaMemcpyHostToDevice);
    ref_kernel<<<B, 32>>>(ds, n, o1);
    warp_kernel<<<B / 4, 128>>>(ds, n, base, o2);
    std::vector<uint32_t> h1(B * n), h2(B * n);
    cudaMemcpy(h1.data(), o1, 4ll * B * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), o2, 4ll * B * n, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < B * n; ++i) bad += h1[i] != h2[i];
    printf("n=%d mismatches=%d err=%s first=%u/%u\n", n, bad, cudaGetErrorString(cudaGetLastError()), h1[0], h2[0]);
  }
  return 0;
}

// timing: one warp, seed + refill + shuffle of n, clock64 per part
__global__ void timing_kernel(unsigned long long seed, int n, const uint32_t* base, uint32_t* x,
                              long long* t) {
  __shared__ uint32_t st[MT_N], buf[MT_N];
  __shared__ uint2 pairs[32];
  __shared__ uint32_t xs[8192];
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) xs[i] = i;
  __syncwarp();
  WarpMT mt{st, buf, pairs, MT_N};
  long long c0 = clock64();
  mt.seed(base, seed);
  long long c1 = clock64();
  mt.refill();
  long long c2 = clock64();
  mt.shuffle(xs, n);
  long long c3 = clock64();
  for (int i = lane; i < n; i += 32) x[i] = xs[i];
  if (lane == 0) { t[0] = c1 - c0; t[1] = c2 - c1; t[2] = c3 - c2; }
}

int timing_main() {
  uint32_t *base, *x;
  long long* t;
  cudaMalloc(&base, 4 * MT_N);
  cudaMalloc(&x, 4 * 8192);
  cudaMalloc(&t, 64);
  uint32_t hb[MT_N];
  mt_base_table(hb);
  cudaMemcpy(base, hb, sizeof(hb), cudaMemcpyHostToDevice);
  for (int n : {750, 2000, 6000}) {
    for (int rep = 0; rep < 2; ++rep) timing_kernel<<<1, 32>>>(0x123456789abcdefull, n, base, x, t);
    long long h[3];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("n=%d cycles: seed=%lld refill=%lld shuffle=%lld (%.1f/elem)\n", n, h[0], h[1], h[2], (double)h[2] / n);
  }
  return 0;
}
