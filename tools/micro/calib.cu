// Calibration micro-benchmarks for the resident kernel's building blocks on
// one CTA of 512 threads (clock64 per step): group bitonic sorts, Eytzinger
// classification, shared-memory histogram atomics, __syncthreads.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_1609_04471_b200/csrc calib.cu
#include <cstdio>
#include <type_traits>
#include "resident.cuh"

using namespace sr;

__global__ void __launch_bounds__(512, 1) k_calib(int* out, long long* cyc, int reps) {
  __shared__ __align__(16) int buf[10240];
  __shared__ int tree[256];
  __shared__ uint8_t eq[128];
  __shared__ uint32_t hist[256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < 10240; i += 512) buf[i] = (int)((i * 2654435761u) >> 3);
  for (int i = tid; i < 256; i += 512) { tree[i] = (int)(i * 16777216u); hist[i] = 0; }
  for (int i = tid; i < 128; i += 512) eq[i] = 0;
  __syncthreads();
  long long t0, t1;
  // 1. group sort 128 keys per half-warp (VT 8, 16 lanes)
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    int* st = buf + w * 512 + (lane >> 4) * 256;
    res_group_sort<int, 8, 16>(st, 128, true, st);
  }
  __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / reps;
  // 2. group sort 512 keys per warp (VT 16, 32 lanes)
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    int* st = buf + w * 512;
    res_group_sort<int, 16, 32>(st, 512, true, st);
  }
  __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / reps;
  // 3. classify 8 keys per thread against 63 splitters (depth 6)
  int acc = 0;
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    int x[8], bin[8];
#pragma unroll
    for (int u = 0; u < 8; u++) x[u] = buf[(u * 512 + tid + r) & 8191];
    res_classify<int, 64, 8>(x, bin, tree, eq, 63, 6);
#pragma unroll
    for (int u = 0; u < 8; u++) acc += bin[u];
  }
  __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / reps;
  // 4. smem histogram atomics, 8 per thread into 65 bins
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll
    for (int u = 0; u < 8; u++) atomicAdd(&hist[(buf[(u * 512 + tid + r) & 8191] >> 5) % 65], 1u);
  }
  __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / reps;
  // 5. __syncthreads alone
  t0 = clock64();
  for (int r = 0; r < reps; r++) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0) / reps;
  // 6. CTA bitonic sort of 2048 keys (VT 4)
  t0 = clock64();
  for (int r = 0; r < reps; r++) BitonicSort<int, 512, 4>::sort(buf, 2048);
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / reps;
  // 7. CTA bitonic sort of 256 keys with 64 threads (VT 4)
  t0 = clock64();
  for (int r = 0; r < reps; r++) BitonicSort<int, 128, 4>::sort(buf + 8704, 256);
  t1 = clock64();
  if (tid == 0) cyc[6] = (t1 - t0) / reps;
  // 8. CTA bitonic sort of 2048 keys, 4096 with VT 8
  t0 = clock64();
  for (int r = 0; r < reps; r++) BitonicSort<int, 512, 8>::sort(buf, 4096);
  t1 = clock64();
  if (tid == 0) cyc[7] = (t1 - t0) / reps;

  // 9..14: group sorts of various shapes (each CTA-wide pass sorts 8192 keys)
  auto gs = [&](auto vt_c, auto gl_c, int slot) {
    constexpr int VT = decltype(vt_c)::value, GL = decltype(gl_c)::value;
    constexpr int G = 512 / GL;  // groups per CTA
    long long a0 = clock64();
    for (int r = 0; r < reps; r++) {
      for (int base = 0; base < 8192; base += G * GL * VT) {
        int* st = buf + base + (tid / GL) * GL * VT;
        res_group_sort<int, VT, GL>(st, GL * VT, true, st);
      }
    }
    __syncthreads();
    long long a1 = clock64();
    if (tid == 0) cyc[slot] = (a1 - a0) / reps;
  };
  gs(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{}, 8);
  gs(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{}, 9);
  gs(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{}, 10);
  gs(std::integral_constant<int, 8>{}, std::integral_constant<int, 16>{}, 11);
  gs(std::integral_constant<int, 16>{}, std::integral_constant<int, 16>{}, 12);
  gs(std::integral_constant<int, 16>{}, std::integral_constant<int, 32>{}, 13);
  gs(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, 14);
  // 15: classify depth 9 (256+ node tree would need 512 entries; use depth 8 on 255 splitters)
  {
    __shared__ int tree2[512];
    for (int i = tid; i < 512; i += 512) tree2[i] = (int)(i * 8388608u);
    __syncthreads();
    long long a0 = clock64();
    for (int r = 0; r < reps; r++) {
      int x[8], bin[8];
#pragma unroll
      for (int u = 0; u < 8; u++) x[u] = buf[(u * 512 + tid + r) & 8191];
      res_classify<int, 256, 8>(x, bin, tree2, eq, 0, 8);
#pragma unroll
      for (int u = 0; u < 8; u++) acc += bin[u];
    }
    __syncthreads();
    long long a1 = clock64();
    if (tid == 0) cyc[15] = (a1 - a0) / reps;
  }
  if (acc == 12345) out[0] = acc + hist[3];
}

int main() {
  int* d;
  long long* c;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64 * 8);
  cudaMemset(c, 0, 64 * 8);
  for (int it = 0; it < 2; it++) k_calib<<<1, 512>>>(d, c, 20);
  long long h[16];
  cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
  const char* names[16] = {"group sort 128 (VT8 x16 lanes), 32 groups", "group sort 512 (VT16 x32), 16 warps",
                          "classify 8 keys/thread depth 6", "smem hist atomics 8/thread", "__syncthreads",
                          "CTA bitonic 2048 (VT4)", "CTA bitonic 256 (64 thr)", "CTA bitonic 4096 (VT8)",
                          "8192 keys as 32-groups (VT4 x8)", "8192 keys as 64-groups (VT4 x16)",
                          "8192 keys as 64-groups (VT8 x8)", "8192 keys as 128-groups (VT8 x16)",
                          "8192 keys as 256-groups (VT16 x16)", "8192 keys as 512-groups (VT16 x32)",
                          "8192 keys as 16-groups (VT4 x4)", "classify 8 keys/thread depth 8"};
  for (int i = 0; i < 16; i++) printf("%-45s %8lld cycles  (%.2f us at 1.9 GHz)\n", names[i], h[i], h[i] / 1900.0);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
