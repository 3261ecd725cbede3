// micro-benchmark: bucket classification of N random int32 keys against B
// sorted splitters (the H8 step), shared-memory histogram of the 2B+1 3-way
// bins.  Variants:
//   0  Eytzinger tree, U keys in lockstep (res_classify / classify_keys)
//   1  guide table + data-dependent bisection (classify_keys_guided, R18)
//   2  guide table (one 32-bit cell word: start | count << 16) + a fixed,
//      CTA-uniform number of predicated bisection steps (branch-free)
// Every variant's histogram is checked against variant 0's.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -o classify classify.cu
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_1609_04471_b200/csrc/presort.cuh"
using namespace sr;

constexpr int NT = 1024;
constexpr int CELLS = 4096;
int PERSIST = 0;

struct G2 {
  uint32_t u0, u1;
  int shift, m, steps, any_eq;
  uint32_t cell[CELLS];  // start | (count << 16)
};

struct Smem {
  int tree[2 * kMaxBuckets];
  uint8_t eq[kMaxBuckets];
  uint32_t hist[kMaxBins];
  Guide guide;
  G2 g2;
};

__device__ __forceinline__ uint32_t u32(int x) { return (uint32_t)x ^ 0x80000000u; }

// guide 2: one word per cell, maximal cell span -> uniform step count
__device__ void build_g2(const int* spl, const uint8_t* eqf, int m, G2& g) {
  const uint32_t u0 = u32(spl[0]), u1 = u32(spl[m - 1]);
  const uint32_t span = u1 - u0;
  int shift = 0;
  while (shift < 32 && (span >> shift) >= (uint32_t)CELLS) shift++;
  __shared__ int s_max, s_eq;
  if (threadIdx.x == 0) { s_max = 0; s_eq = 0; }
  __syncthreads();
  int mx = 0, aeq = 0;
  for (int c = threadIdx.x; c < CELLS; c += blockDim.x) {
    auto lb = [&](uint64_t v) {  // #{t_j : u(t_j) < v}
      if (v > 0xffffffffull) return m;
      int lo = 0, hi = m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint64_t)u32(spl[mid]) < v) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    const int a = lb((uint64_t)u0 + ((uint64_t)c << shift));
    const int b = lb((uint64_t)u0 + ((uint64_t)(c + 1) << shift));
    g.cell[c] = (uint32_t)a | ((uint32_t)(b - a) << 16);
    mx = max(mx, b - a);
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) aeq |= eqf[j];
  atomicMax(&s_max, mx);
  atomicOr(&s_eq, aeq);
  __syncthreads();
  if (threadIdx.x == 0) {
    g.u0 = u0; g.u1 = u1; g.shift = shift; g.m = m;
    int st = 0;
    while ((1 << st) <= s_max) st++;  // lo < hi ranges of length <= s_max close in st halvings
    g.steps = st;
    g.any_eq = s_eq;
  }
}

template <int U>
__device__ __forceinline__ void classify_g2(const int (&x)[U], int (&bin)[U], const int* spl, const uint8_t* eqf,
                                            const G2& g) {
  int lo[U], hi[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const uint32_t v = u32(x[u]);
    const uint32_t c = min((v - g.u0) >> g.shift, (uint32_t)CELLS - 1);
    const uint32_t w = g.cell[c];
    const int a = (int)(w & 0xffff), b = a + (int)(w >> 16);
    lo[u] = v <= g.u0 ? 0 : (v > g.u1 ? g.m : a);
    hi[u] = v <= g.u0 ? 0 : (v > g.u1 ? g.m : b);
  }
  for (int s = 0; s < g.steps; s++) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool act = lo[u] < hi[u];
      const int mid = (lo[u] + hi[u]) >> 1;
      const bool p = spl[mid] < x[u];
      lo[u] = (act && p) ? mid + 1 : lo[u];
      hi[u] = (act && !p) ? mid : hi[u];
    }
  }
  if (g.any_eq) {
#pragma unroll
    for (int u = 0; u < U; u++) bin[u] = 2 * lo[u] + ((lo[u] < g.m && spl[lo[u]] == x[u] && eqf[lo[u]]) ? 1 : 0);
  } else {
#pragma unroll
    for (int u = 0; u < U; u++) bin[u] = 2 * lo[u];
  }
}

template <int V, int U>
__global__ void __launch_bounds__(NT) k_class(const int* __restrict__ keys, int64_t n, int64_t chunk,
                                              const int* __restrict__ spl, const uint8_t* __restrict__ eqf, int m,
                                              unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int depth = tree_depth(m);
  if (V == 0) load_splitters_smem(spl, eqf, m, sm.tree, sm.eq);
  else {
    for (int i = threadIdx.x; i < kMaxBuckets; i += NT) {
      sm.tree[kMaxBuckets + i] = i < m ? spl[i] : INT32_MAX;
      sm.eq[i] = i < m ? eqf[i] : 0;
    }
  }
  for (int b = threadIdx.x; b < kMaxBins; b += NT) sm.hist[b] = 0;
  __syncthreads();
  if (V == 1) build_guide<int>(sm.tree + kMaxBuckets, m, sm.guide);
  if (V == 2 || V == 3) build_g2(sm.tree + kMaxBuckets, sm.eq, m, sm.g2);
  __syncthreads();
  for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < n; c0 += (int64_t)gridDim.x * chunk)
  for (int64_t base = c0, c1 = min(n, c0 + chunk); base < c1; base += NT * U) {
    int x[U], bin[U];
    const int* p = keys + base + 4 * threadIdx.x;
#pragma unroll
    for (int g = 0; g < U / 4; g++) {
      const int4 v = *reinterpret_cast<const int4*>(p + 4 * g * NT);
      x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
    }
    if (V == 0) classify_keys<int, U>(x, bin, sm.tree, sm.eq, m, depth);
    if (V == 1) classify_keys_guided<int, U>(x, bin, sm.tree + kMaxBuckets, sm.eq, sm.guide);
    if (V == 2 || V == 3) classify_g2<U>(x, bin, sm.tree + kMaxBuckets, sm.eq, sm.g2);
    if (V == 4 || V == 5) {
#pragma unroll
      for (int u = 0; u < U; u++) bin[u] = (x[u] >> 7) & 1023;
    }
    if (V == 3 || V == 5) {
      int acc = 0;
#pragma unroll
      for (int u = 0; u < U; u++) acc += bin[u];
      int xs = 0;
#pragma unroll
      for (int u = 0; u < U; u++) xs ^= x[u];
      if (acc == 0x7fffffff || xs == 0x7fffffff) sm.hist[0] = acc;  // keep the work
    } else {
#pragma unroll
      for (int u = 0; u < U; u++) atomicAdd(&sm.hist[bin[u]], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 2 * m + 2; b += NT)
    if (sm.hist[b]) atomicAdd(out + b, (unsigned long long)sm.hist[b]);
}

__global__ void k_gen(int* k, int64_t n, uint64_t seed, int mod) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed + (uint64_t)i);
    k[i] = mod ? (int)(h % mod) * 1000003 : (int)(h >> 32);
  }
}

template <int V, int U>
float run(const int* d_k, int64_t n, const int* d_s, const uint8_t* d_e, int m, unsigned long long* d_o) {
  const int64_t chunk = 65536;
  const int grid = PERSIST ? 148 * 2 : (int)((n + chunk - 1) / chunk);
  cudaFuncSetAttribute(k_class<V, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaMemset(d_o, 0, 8 * (size_t)kMaxBins);
    cudaEventRecord(a);
    k_class<V, U><<<grid, NT, sizeof(Smem)>>>(d_k, n, chunk, d_s, d_e, m, d_o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b);
    best = std::min(best, t);
  }
  return best;
}

int main() {
  const int64_t n = int64_t(1) << 28;
  int* d_k; int* d_s; uint8_t* d_e; unsigned long long* d_o;
  cudaMalloc(&d_k, 4 * n); cudaMalloc(&d_s, 4 * kMaxBuckets); cudaMalloc(&d_e, kMaxBuckets);
  cudaMalloc(&d_o, 8 * (size_t)kMaxBins);
  for (int pers : {0, 1})
  for (int mod : {0, 100}) {
    PERSIST = pers;
    printf("persistent grid: %d\n", pers);
    k_gen<<<148 * 8, 256>>>(d_k, n, 12345, mod);
    for (int B : {512, 2048}) {
      const int m = B - 1;
      std::vector<int> h(4 * B);
      cudaMemcpy(h.data(), d_k + 777, 4 * h.size(), cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      std::vector<int> s(m);
      std::vector<uint8_t> e(m, 0);
      for (int j = 0; j < m; j++) {
        const int r = 4 * (j + 1);
        s[j] = h[r];
        const int c = (int)(std::upper_bound(h.begin(), h.end(), s[j]) - std::lower_bound(h.begin(), h.end(), s[j]));
        e[j] = c > 2;
      }
      cudaMemcpy(d_s, s.data(), 4 * m, cudaMemcpyHostToDevice);
      cudaMemcpy(d_e, e.data(), m, cudaMemcpyHostToDevice);
      std::vector<unsigned long long> ref(kMaxBins), got(kMaxBins);
      float t0 = run<0, 16>(d_k, n, d_s, d_e, m, d_o);
      cudaMemcpy(ref.data(), d_o, 8 * kMaxBins, cudaMemcpyDeviceToHost);
      float t0b = run<0, 8>(d_k, n, d_s, d_e, m, d_o);
      float t1 = run<1, 16>(d_k, n, d_s, d_e, m, d_o);
      cudaMemcpy(got.data(), d_o, 8 * kMaxBins, cudaMemcpyDeviceToHost);
      const bool ok1 = got == ref;
      float t2 = run<2, 16>(d_k, n, d_s, d_e, m, d_o);
      cudaMemcpy(got.data(), d_o, 8 * kMaxBins, cudaMemcpyDeviceToHost);
      const bool ok2 = got == ref;
      float t2b = run<2, 8>(d_k, n, d_s, d_e, m, d_o);
      float t3 = run<3, 16>(d_k, n, d_s, d_e, m, d_o);
      float t4 = run<4, 16>(d_k, n, d_s, d_e, m, d_o);
      float t5 = run<5, 16>(d_k, n, d_s, d_e, m, d_o);
      printf("   g2 no-hist %.3f  hist-only %.3f  load-only %.3f\n", t3, t4, t5);
      printf("%s B=%4d: eytz16 %.3f ms  eytz8 %.3f  guided %.3f (%s)  g2-16 %.3f (%s)  g2-8 %.3f   [read-only floor %.3f ms]\n",
             mod ? "few100" : "random", B, t0, t0b, t1, ok1 ? "ok" : "MISMATCH", t2, ok2 ? "ok" : "MISMATCH", t2b,
             4.0 * n / 6.5e9);
    }
  }
  return 0;
}
