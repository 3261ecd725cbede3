// micro-benchmark: E-phase unit sorts of the resident kernel on 2M int32 keys
// split into units of L keys (148 persistent CTAs x 512 threads, units handed
// out round robin).  CTA units: res_bucket_sort2 (in-smem 16-way partition +
// warp networks); warp units: one warp's register network per unit.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
__device__ unsigned long long g_prof[16];
__device__ unsigned long long g_t0;
#define SR_UNIT_PROF 1
#define SR_UNIT_MARK(k) do { if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t = clock64(); g_prof[k] += t - g_t0; g_t0 = t; } } while (0)
#include "../../paper_1609_04471_b200/csrc/resident.cuh"
#include "../../paper_1609_04471_b200/csrc/unit_sort.cuh"
using namespace sr;

// vectorised warp copy of len keys (16-byte aligned src/dst offsets assumed: units start at multiples of L)
__device__ __forceinline__ void warp_copy_vec(const int* __restrict__ src, int* __restrict__ dst, int len) {
  const int lane = threadIdx.x & 31;
  const int nv = len >> 2;
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(dst);
  for (int i0 = 0; i0 < nv; i0 += 32 * 8) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int i = i0 + u * 32 + lane;
      if (i < nv) v[u] = s4[i];
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int i = i0 + u * 32 + lane;
      if (i < nv) d4[i] = v[u];
    }
  }
  for (int i = (nv << 2) + lane; i < len; i += 32) dst[i] = src[i];
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_units(const int* src, int* dst, int n, int L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = ResSmem<int>;
  typename SM::E& e = *reinterpret_cast<typename SM::E*>(smem_raw);
  const int nu = (n + L - 1) / L;
  if (MODE == 4) {
    using US = UnitSmem<int, 16384, 512>;
    US& ue = *reinterpret_cast<US*>(smem_raw);
    const int w = threadIdx.x >> 5;
    for (int u = blockIdx.x; u < nu; u += gridDim.x) {
      const int s = u * L, len = min(L, n - s);
      for (int p = w * 256; p < len; p += 16 * 256) warp_copy_vec(src + s + p, ue.x + p, min(256, len - p));
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x == 0) g_t0 = clock64();
      unit_sort<int, 16384, 512>(dst + s, len, ue);
    }
  } else if (MODE == 0) {
    const int w = threadIdx.x >> 5;
    for (int u = blockIdx.x; u < nu; u += gridDim.x) {
      const int s = u * L, len = min(L, n - s);
      for (int p = w * 256; p < len; p += 16 * 256) warp_copy_vec(src + s + p, e.x + p, min(256, len - p));
      __syncthreads();
      unit_sort<int, 16384, 512>(dst + s, len, e);
      __syncthreads();
    }
  } else {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* stage = e.x + w * 2048;
    for (int u = blockIdx.x * 16 + w; u < nu; u += gridDim.x * 16) {
      const int s = u * L, len = min(L, n - s);
      if (MODE == 1) {
        for (int i = lane; i < len; i += 32) stage[i] = src[s + i];
      } else {
        warp_copy_vec(src + s, stage, len);
      }
      __syncwarp();
      if (MODE != 3) unit_warp_piece<int>(stage, len, dst + s);  // sorted into dst
      else warp_copy_vec(stage, dst + s, len);
      __syncwarp();
    }
  }
}

int main() {
  const int n = 2000000;
  std::vector<int> h(n);
  std::mt19937 rng(1);
  for (auto& x : h) x = (int)rng();
  int *src, *dst;
  cudaMalloc(&src, n * 4);
  cudaMalloc(&dst, n * 4);
  cudaMemcpy(src, h.data(), n * 4, cudaMemcpyHostToDevice);
  const size_t smem = std::max(sizeof(ResSmem<int>::E), sizeof(UnitSmem<int, 16384, 512>));
  cudaFuncSetAttribute(k_units<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_units<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_units<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_units<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_units<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { int mode, L; };
  Case cases[] = {{4, 2048}, {4, 3000}, {4, 4096}, {4, 6000}, {4, 8192}, {4, 12000}, {4, 16384},{0, 2048}, {0, 4096}, {0, 8192}, {0, 16384}, {1, 256}, {1, 1024}, {1, 2048},
                  {2, 256}, {2, 512}, {2, 1024}, {2, 2048}, {3, 256}, {3, 1024}, {3, 2048}};
  for (auto cs : cases) {
    float best = 1e9;
    for (int r = 0; r < 6; r++) {
      cudaEventRecord(a);
      if (cs.mode == 0) k_units<0><<<148, 512, smem>>>(src, dst, n, cs.L);
      else if (cs.mode == 1) k_units<1><<<148, 512, smem>>>(src, dst, n, cs.L);
      else if (cs.mode == 2) k_units<2><<<148, 512, smem>>>(src, dst, n, cs.L);
      else if (cs.mode == 3) k_units<3><<<148, 512, smem>>>(src, dst, n, cs.L);
      else k_units<4><<<148, 512, smem>>>(src, dst, n, cs.L);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    std::vector<int> o(n);
    cudaMemcpy(o.data(), dst, n * 4, cudaMemcpyDeviceToHost);
    bool ok = cs.mode != 3;
    for (int s = 0; s < n; s += cs.L) {
      int e = std::min(n, s + cs.L);
      std::vector<int> ref(h.begin() + s, h.begin() + e);
      std::sort(ref.begin(), ref.end());
      if (!std::equal(ref.begin(), ref.end(), o.begin() + s)) { ok = false; break; }
    }
    static const char* nm[5] = {"CTA units ", "warp naive", "warp vec  ", "copy only ", "NEW unit  "};
    if (cs.mode == 4) {
      unsigned long long pr[16];
      cudaMemcpyFromSymbol(pr, g_prof, sizeof(pr));
      printf("   cycles (CTA0, 6 reps): sorted? %llu rank %llu spl %llu classify %llu scan %llu move %llu warps %llu bar %llu\n",
             pr[0], pr[1], pr[2], pr[3], pr[4], pr[5], pr[6], pr[7]);
      unsigned long long z[16] = {};
      cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    printf("%s L=%6d : %8.1f us  %s  (%s)\n", nm[cs.mode], cs.L, best * 1e3, ok ? "ok" : "WRONG",
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
