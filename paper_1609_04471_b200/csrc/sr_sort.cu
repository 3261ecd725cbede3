// sr_sort.cu -- host planner (H3, H12) and C ABI of libsr_sort.so.
//
// Route choice follows the paper's recommendation: "quicksort,
// especially our hybrid quicksort, if stable sorting is not required. Only
// when ... the input contains some kind of presortedness and the memory is not
// a concern, then mergesort".  Here both routes are stable, so the planner
// picks by a byte-cost model over the measured run statistics:
//   D == 0                -> SORTED (is_sorted exit)
//   no descending breaks  -> REVERSED (one reversal, PAPER.md:93 / :172)
//   long natural runs     -> MERGE if its simulated bytes beat PARTITION
//   otherwise             -> PARTITION (levels until every bucket <= kCap)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sr_sort.h"
#include "bucket_sort.cuh"
#include "distance.cuh"
#include "fkeys.cuh"
#include "generate.cuh"
#include "measures.cuh"
#include "merge.cuh"
#include "records.cuh"
#include "outlier.cuh"
#include "partition.cuh"
#include "presort.cuh"
#include "resident.cuh"

using namespace sr;

namespace {

// ------------------------------------------------------------------ options / thread state
int g_force_route = 0;
int g_profile = 0;
int g_merge_route = 1;
int g_resident = 1;
int g_outlier = 1;
int g_distance = 1;
int g_res_cap = 16384;
int64_t g_ws_limit = 0;  // SR_OPT_WS_LIMIT (fault injection), 0 = none
// SR_OPT_TUNE + i: tuning knobs of the large keys-only path (A/B measurements)
//   [0] fused level 2 (k_bucket_sort) on/off   [1] level-1 buckets for n >= kBigLevel1
//   [2] mean sub-bucket the fused level aims for   [3] cap on the level-1 buckets at any n (0 = none; tests)
//   [4] k_bucket_sort phase skips (timing experiments only; the output is then NOT sorted): 1 finishing, 2 scatter
int64_t g_tune[8] = {0, 512, 256, 0, 0, 2, 0, 0};
#ifndef SR_WARP_VT64
#define SR_WARP_VT64 1
#endif
constexpr bool g_warp_vt64 = SR_WARP_VT64;

struct ProfEntry {
  const char* name;
  cudaEvent_t a, b;
  int64_t bytes;
};

// Per (host thread, device) state of the resident path: every pointer here is
// device-specific, so a thread that sorts on two GPUs keeps one set per device.
struct DevState {
  // host-mapped completion record of the resident kernel (resident.cuh ResDone)
  sr::ResDone* done_h = nullptr;
  sr::ResDone* done_d = nullptr;
  uint32_t done_seq = 0;
  uint32_t* arrive = nullptr;  // resident route-step arrival counter (device, zeroed once, never reset)
  uint32_t arrive_base = 0;
  uint32_t scount_base = 0;    // the sampler-step counter (arrive + 16) before the next launch
  // resident scratch kept between calls: calls from this thread on this device
  // are ordered on the device (same stream: stream order; another stream: it
  // waits for last_ev), so the next call reuses the arena without a
  // cudaMallocAsync even though the host returned before the kernel finished
  unsigned char* res_arena = nullptr;
  size_t res_arena_bytes = 0;
  cudaEvent_t last_ev = nullptr;       // recorded after the last resident launch
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  cudaEvent_t launch_ev = nullptr;     // recorded before each resident launch (watchdog start)
  // sr_sort_host_batch: the two copy streams (host->device, device->host) beside the caller's stream
  cudaStream_t batch_h2d = nullptr, batch_d2h = nullptr;
  // the resident kernel as a cooperative node of an instantiated one-node CUDA
  // graph, its parameters replaced per call: cudaGraphExecKernelNodeSetParams +
  // cudaGraphLaunch take ~3.5 us less host time than cudaLaunchCooperativeKernel
  // for a 148-CTA, ~210 KB-smem launch (tools/micro/coopgraph.cu)
  struct CoopGraph {
    const void* func = nullptr;
    unsigned P = 0;
    size_t smem = 0;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaGraphNode_t node = nullptr;
  };
  CoopGraph coop[4];
  // after a failed or timed-out resident call the kernel may still run and use
  // the arena, the counter and the record: abandon them (leaked) so that the
  // next call starts from fresh ones
  void abandon() {
    done_h = nullptr;
    done_d = nullptr;
    arrive = nullptr;
    res_arena = nullptr;
    res_arena_bytes = 0;
    has_last = false;
  }
  ~DevState() {
    if (batch_h2d) cudaStreamDestroy(batch_h2d);
    if (batch_d2h) cudaStreamDestroy(batch_d2h);
    for (auto& cg : coop) {
      if (cg.ge) cudaGraphExecDestroy(cg.ge);
      if (cg.g) cudaGraphDestroy(cg.g);
    }
    if (last_ev) cudaEventDestroy(last_ev);
    if (launch_ev) cudaEventDestroy(launch_ev);
    if (done_h) cudaFreeHost(done_h);
    if (res_arena) cudaFree(res_arena);
    if (arrive) cudaFree(arrive);
  }
};
constexpr int kMaxDevices = 64;

struct ThreadState {
  sr_plan plan{};
  std::string err;
  std::vector<ProfEntry> prof;
  cudaStream_t prof_stream = nullptr;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // pinned staging for small host->device uploads (pageable cudaMemcpyAsync
  // may synchronise the host with the stream and stall the enqueue pipeline)
  unsigned char* up = nullptr;
  size_t up_bytes = 0;
  cudaEvent_t up_done = nullptr;
  bool up_pending = false;
  DevState* dev[kMaxDevices] = {};
  DevState& ds() {  // the current device's state
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= kMaxDevices) d = 0;
    if (!dev[d]) dev[d] = new DevState();
    return *dev[d];
  }
  ~ThreadState() {
    for (auto* d : dev) delete d;
    for (auto& e : prof) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    if (pinned) cudaFreeHost(pinned);
    if (up) cudaFreeHost(up);
    if (up_done) cudaEventDestroy(up_done);
  }
};
thread_local ThreadState t_state;
thread_local std::chrono::steady_clock::time_point t_call0;
void hostprof(const char* what) {  // SR_HOSTPROF: host time since the call began, per step
  static const bool on = getenv("SR_HOSTPROF") != nullptr;
  if (on)
    fprintf(stderr, "[sr_host] %-12s %7.1f us\n", what,
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call0).count() * 1e6);
}


struct SrError {
  int32_t code;
  std::string msg;
};

[[noreturn]] void fail(int32_t code, const std::string& msg) { throw SrError{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) { cudaGetLastError(); fail(SR_ERR_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e)); }
  if (e != cudaSuccess) fail(SR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// cooperative launch of func through this thread's cached graph node (see
// ThreadState::CoopGraph); SR_NO_GRAPH=1 launches it directly
cudaError_t launch_coop(const void* func, unsigned P, unsigned NT, void** args, size_t smem, cudaStream_t st) {
  static const bool direct = getenv("SR_NO_GRAPH") != nullptr;
  if (direct) return cudaLaunchCooperativeKernel(func, P, NT, args, smem, st);
  cudaKernelNodeParams kp = {};
  kp.func = const_cast<void*>(func);
  kp.gridDim = dim3(P);
  kp.blockDim = dim3(NT);
  kp.sharedMemBytes = (unsigned)smem;
  kp.kernelParams = args;
  DevState& ds = t_state.ds();  // graphs are per device
  DevState::CoopGraph* cg = nullptr;
  for (auto& x : ds.coop)
    if (x.func == func && x.P == P && x.smem == smem) { cg = &x; break; }
  cudaError_t e;
  if (cg) {
    e = cudaGraphExecKernelNodeSetParams(cg->ge, cg->node, &kp);
    if (e != cudaSuccess) return e;
    return cudaGraphLaunch(cg->ge, st);
  }
  DevState::CoopGraph* slot = nullptr;
  for (auto& x : ds.coop)
    if (!x.func) { slot = &x; break; }
  if (!slot) return cudaLaunchCooperativeKernel(func, P, NT, args, smem, st);  // cache full
  DevState::CoopGraph n;
  cudaLaunchAttributeValue v = {};
  v.cooperative = 1;
  if ((e = cudaGraphCreate(&n.g, 0)) != cudaSuccess) return e;
  if ((e = cudaGraphAddKernelNode(&n.node, n.g, nullptr, 0, &kp)) != cudaSuccess ||
      (e = cudaGraphKernelNodeSetAttribute(n.node, cudaLaunchAttributeCooperative, &v)) != cudaSuccess ||
      (e = cudaGraphInstantiate(&n.ge, n.g, 0)) != cudaSuccess) {
    cudaGraphDestroy(n.g);
    return e;
  }
  n.func = func;
  n.P = P;
  n.smem = smem;
  *slot = n;
  return cudaGraphLaunch(slot->ge, st);
}

void* pinned(size_t bytes) {
  ThreadState& ts = t_state;
  if (ts.pinned_bytes < bytes) {
    if (ts.pinned) cudaFreeHost(ts.pinned);
    size_t sz = std::max<size_t>(bytes, 1 << 20);
    check_cuda(cudaHostAlloc(&ts.pinned, sz, cudaHostAllocPortable), "cudaHostAlloc");
    ts.pinned_bytes = sz;
  }
  return ts.pinned;
}

// the stream-ordered pool of each device keeps its memory between calls
void init_pool() {
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return;
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return;
  done[dev] = true;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
}

template <typename T>
T ceil_div(T a, T b) { return (a + b - 1) / b; }

int64_t pow2ceil(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ------------------------------------------------------------------ per-call context
struct Ctx {
  cudaStream_t st;
  sr_plan& plan;
  std::vector<void*> allocs;
  bool profile;
  size_t up_off = 0;
  explicit Ctx(cudaStream_t s) : st(s), plan(t_state.plan), profile(g_profile != 0) {
    plan = sr_plan{};
    ThreadState& ts = t_state;
    if (ts.up_pending) {  // the staging buffer of the previous call may still be in flight
      cudaEventSynchronize(ts.up_done);
      ts.up_pending = false;
    }
    if (profile) {
      for (auto& e : t_state.prof) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
      t_state.prof.clear();
      t_state.prof_stream = s;
    }
  }
  ~Ctx() {
    static const bool timing = getenv("SR_TIMING") != nullptr;
    if (timing)
      fprintf(stderr, "[sr_sort] n=%lld route=%d launches=%d enqueue=%.1fus wait=%.1fus tail=%.1fus\n",
              (long long)plan.n, plan.route, plan.launches, t_enqueue * 1e6, t_wait * 1e6,
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t_mark).count() * 1e6);
    if (profile && getenv("SR_TIMELINE") && !t_state.prof.empty()) {
      cudaStreamSynchronize(st);
      for (auto& e : t_state.prof) {
        float t0 = 0, d = 0;
        cudaEventElapsedTime(&t0, t_state.prof[0].a, e.a);
        cudaEventElapsedTime(&d, e.a, e.b);
        fprintf(stderr, "[sr_timeline] %-18s start %9.1f us  dur %9.1f us\n", e.name, t0 * 1e3, d * 1e3);
      }
    }
    for (void* p : allocs) cudaFreeAsync(p, st);
  }
  // One stream-ordered pool allocation up front (reserve) that later allocs
  // carve from, so a call costs one cudaMallocAsync instead of dozens.
  unsigned char* arena = nullptr;
  size_t arena_size = 0, arena_off = 0;
  // SR_OPT_WS_LIMIT: a reservation beyond the injected limit fails as a real one would
  void ws_check(size_t bytes) {
    if (g_ws_limit > 0 && plan.workspace_bytes + (int64_t)bytes > g_ws_limit)
      fail(SR_ERR_OUT_OF_MEMORY, "cudaMallocAsync: workspace limit (SR_OPT_WS_LIMIT)");
  }
  void reserve(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    ws_check(bytes);
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
    allocs.push_back(p);
    arena = reinterpret_cast<unsigned char*>(p);
    arena_size = bytes;
    arena_off = 0;
    plan.workspace_bytes += (int64_t)bytes;
  }
  // carve later allocations from a caller-owned arena (not freed by this Ctx)
  void use_arena(unsigned char* p, size_t bytes) {
    arena = p;
    arena_size = bytes;
    arena_off = 0;
  }
  template <typename T>
  T* alloc(int64_t count) {
    if (count <= 0) count = 1;
    size_t bytes = (size_t)count * sizeof(T);
    bytes = (bytes + 255) & ~size_t(255);
    if (arena && arena_off + bytes <= arena_size) {
      T* r = reinterpret_cast<T*>(arena + arena_off);
      arena_off += bytes;
      return r;
    }
    ws_check(bytes);
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
    allocs.push_back(p);
    plan.workspace_bytes += (int64_t)bytes;
    return reinterpret_cast<T*>(p);
  }
  // Launch through f(); returns a handle so that a speculative launch that
  // turned out to be gated off can give its planned bytes back (unplan()).
  template <typename F>
  int launch(const char* name, int64_t bytes, F&& f) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (profile) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
    f();
    check_cuda(cudaGetLastError(), name);
    if (profile) {
      cudaEventRecord(b, st);
      t_state.prof.push_back({name, a, b, bytes});
    }
    plan.launches++;
    plan.bytes_planned += bytes;
    launched.push_back({bytes, profile ? (int)t_state.prof.size() - 1 : -1});
    return (int)launched.size() - 1;
  }
  void unplan(int h) { replan(h, 0); }
  // Correct the algorithmic bytes of launch h once the statistics are known.
  void replan(int h, int64_t bytes) {
    if (h < 0) return;
    plan.bytes_planned += bytes - launched[h].first;
    if (launched[h].second >= 0) t_state.prof[launched[h].second].bytes = bytes;
    launched[h].first = bytes;
  }
  std::vector<std::pair<int64_t, int>> launched;
  void memset0(void* p, size_t bytes) { check_cuda(cudaMemsetAsync(p, 0, bytes, st), "cudaMemsetAsync"); }
  template <typename T>
  void upload(T* dst, const std::vector<T>& src) {
    if (src.empty()) return;
    const size_t bytes = src.size() * sizeof(T);
    ThreadState& ts = t_state;
    const size_t off = (up_off + 15) & ~size_t(15);
    if (off + bytes > ts.up_bytes) {
      if (up_off == 0 && bytes <= (size_t(16) << 20)) {  // (re)size the staging area between calls
        if (ts.up) cudaFreeHost(ts.up);
        ts.up_bytes = std::max<size_t>(bytes, size_t(1) << 20);
        check_cuda(cudaHostAlloc((void**)&ts.up, ts.up_bytes, cudaHostAllocPortable), "cudaHostAlloc");
      } else {  // staging full within this call: fall back to a synchronous pageable copy
        check_cuda(cudaMemcpyAsync(dst, src.data(), bytes, cudaMemcpyHostToDevice, st), "upload");
        return;
      }
    }
    const size_t o2 = (up_off + 15) & ~size_t(15);
    std::memcpy(ts.up + o2, src.data(), bytes);
    check_cuda(cudaMemcpyAsync(dst, ts.up + o2, bytes, cudaMemcpyHostToDevice, st), "upload");
    up_off = o2 + bytes;
    if (!ts.up_done) cudaEventCreateWithFlags(&ts.up_done, cudaEventDisableTiming);
    cudaEventRecord(ts.up_done, st);  // the next call reuses the staging area once this copy is done
    ts.up_pending = true;
  }
  // Wait for a kernel's host-mapped completion record (spin; the stream is
  // polled now and then so that a failed or lost launch cannot hang the host).
  // Wait for a kernel's host-mapped completion record (spin; the stream is
  // polled now and then so that a failed or lost launch cannot hang the host).
  // The watchdog starts once `started` (recorded just before the launch) has
  // completed, i.e. when the kernel can run, not when the host began waiting:
  // earlier work queued on the stream does not count against it.
  DevStats await_done(const sr::ResDone* d, uint32_t seq, cudaEvent_t started, int* in_kernel) {
    auto t0 = std::chrono::steady_clock::now();
    t_enqueue += std::chrono::duration<double>(t0 - t_mark).count();
    bool running = false;
    auto t_run = t0;
    for (uint32_t spin = 1;; spin++) {
      if (d->seq == seq) break;
      if ((spin & 1023) == 0) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) {
          if (d->seq == seq) break;
          fail(SR_ERR_INTERNAL, "resident kernel finished without its completion record");
        }
        if (e != cudaErrorNotReady) check_cuda(e, "resident kernel");
        if (!running) {
          const cudaError_t q = cudaEventQuery(started);
          if (q == cudaSuccess) {
            running = true;
            t_run = std::chrono::steady_clock::now();
          } else if (q != cudaErrorNotReady) {
            check_cuda(q, "resident launch event");
          }
        }
        // watchdog: a sort of <= 2^22 keys takes well under a millisecond once it runs
        if (running && std::chrono::steady_clock::now() - t_run > std::chrono::seconds(20))
          fail(SR_ERR_CUDA, "resident kernel did not report within 20 s of starting");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    DevStats r;
    std::memcpy(&r, (const void*)&d->st, sizeof(DevStats));
    *in_kernel = d->in_kernel;
    plan.host_syncs++;
    t_mark = std::chrono::steady_clock::now();
    t_wait += std::chrono::duration<double>(t_mark - t0).count();
    return r;
  }
  // Readback of `bytes` from device into pinned memory + synchronise (the planner's host sync).
  double t_enqueue = 0, t_wait = 0;  // host seconds (SR_TIMING diagnostics)
  std::chrono::steady_clock::time_point t_mark = std::chrono::steady_clock::now();
  void* readback(const void* dev, size_t bytes) {
    auto t0 = std::chrono::steady_clock::now();
    t_enqueue += std::chrono::duration<double>(t0 - t_mark).count();
    void* h = pinned(bytes);
    check_cuda(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, st), "readback");
    check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    plan.host_syncs++;
    t_mark = std::chrono::steady_clock::now();
    t_wait += std::chrono::duration<double>(t_mark - t0).count();
    return h;
  }
};

// Raise a kernel's dynamic shared-memory limit once per (kernel, size); the
// attribute call is far more expensive than a launch.
// The attribute is per device: the cache is keyed by (device, kernel).
template <typename Kern>
void set_smem(Kern k, size_t bytes) {
  static std::mutex mu;
  struct Done { int dev; const void* f; size_t bytes; };
  static std::vector<Done> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  for (auto& d : done)
    if (d.dev == dev && d.f == (const void*)k && d.bytes >= bytes) return;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  done.push_back({dev, (const void*)k, bytes});
}

// ------------------------------------------------------------------ tunables
constexpr int kScanNT = 256, kScanIPT = 16;              // K9
constexpr int kFinNT = 256, kFinVT = 16;                 // K11 big items (two halves of 4096 = kCap)
constexpr int kFinSmallNT = 128;                         // K11 small items (pairs, <= 2048 = kSmallItem)
constexpr int kWarpItemsPerCta = 4;                      // K11w (keys only): warps per CTA
constexpr int kPackKeys = 128;                           // keys only: buckets <= this are packed into items
constexpr int kScatNT = 256;                             // K10 (pairs, stable)
template <typename K>
constexpr int scat_vt() { return sizeof(K) == 4 ? 32 : 16; }  // 8K-pair (int32) / 4K-pair (int64) sub-tiles
constexpr int kScatKNT = 1024;                           // K10 (keys only)
template <typename K>
constexpr int scat_kvt() { return sizeof(K) == 4 ? 16 : 8; }  // 16K-key (int32) / 8K-key (int64) sub-tiles
constexpr int kScanNT1 = 1024;                           // K1
constexpr int kCountNT = 1024;                           // K8
constexpr int64_t kAtomicMaxEntries = 2 << 20;  // keys-only count-matrix threshold (entries)
constexpr int64_t kFuseMin = INT64_MAX;  // fusing the level-1 histogram into K1 costs presorted inputs more than it saves
constexpr int kMergeNT = 256, kMergeVT = 16;             // K6
constexpr int kMergeNV = kMergeNT * kMergeVT;
static_assert(2 * kFinNT * kFinVT == kCap, "finishing item must equal kCap");
static_assert(kFinSmallNT * kFinVT == kSmallItem, "small finishing tile");

constexpr int64_t kBigLevel1 = int64_t(64) << 20;
constexpr int64_t kBigLevel1Buckets = 512;
int64_t choose_tile(int64_t n) {  // K1 tile == level-1 chunk == L_min
  int64_t t = pow2ceil(std::max<int64_t>(1, n / 512));
  return std::min<int64_t>(65536, std::max<int64_t>(8192, t));
}
// Buckets per segment: mean bucket ~kTargetBucket at level 1, ~kTargetBucket/2
// below (those buckets are finished by one warp with 32 keys per lane).
int choose_buckets(int64_t len, int level = 1, int key_bytes = 4, bool keys_only = false) {
  // levels >= 2: mean 512 int32 / 256 int64 keys (measured: C5a 7.82 -> 7.71 ms
  // with 512 against 256; C5c 6.93 -> 7.10 ms, so int64 keeps 256)
  const int64_t t2 = g_tune[6] > 0 ? g_tune[6] : (key_bytes == 4 ? 2 : 1) * (kTargetBucket / 4);
  int64_t b = pow2ceil(ceil_div<int64_t>(len, level > 1 ? t2 : kTargetBucket));
  // very large arrays: fewer, larger level-1 buckets, so that the level-1
  // scatter writes runs of >= 32 keys per 16K-key sub-tile (full DRAM sectors;
  // shorter runs cost read-modify-writes) and the level-2 scatter writes stay
  // within a few L2-resident segments
  if (level == 1 && len >= kBigLevel1) b = std::min<int64_t>(b, g_tune[1] > 0 ? g_tune[1] : kBigLevel1Buckets);
  if (level == 1 && g_tune[3] > 0) b = std::min<int64_t>(b, g_tune[3]);
  // keys only, mid-size arrays (4M int32 / g_tune-measured int64 sizes .. 64M keys): level-1 segments of
  // ~128K int32 / ~64K int64 keys, each split again into ~512-key buckets that the warp kernels finish.
  // With kMaxBuckets level-1 buckets of ~8K keys half of them overflowed kCap and paid a second level
  // of 16-32 buckets each, the rest a CTA-wide sort (tools/ab_tune.py "3=...", random keys: 16M int32
  // 0.998 -> 0.717 ms, 32M 1.60 -> 1.19 ms, 8M 0.61 -> 0.48 ms; 16M int64 1.66 -> 1.11 ms)
  if (level == 1 && keys_only && g_tune[3] == 0 && len >= (key_bytes == 4 ? (int64_t(4) << 20) : (int64_t(2) << 20)))
    b = std::min<int64_t>(b, std::max<int64_t>(64, pow2ceil(ceil_div<int64_t>(len, key_bytes == 4 ? 131072 : 65536))));
  // pairs, >= 8M: 512 level-1 buckets (tools/pairs_tune.py: C4's 16M few100 pairs 0.520 -> 0.467 ms -- still
  // one level, every one of the 100 values keeps its equality bucket -- and 16M random pairs 2.20 -> 1.91 ms)
  if (level == 1 && !keys_only && g_tune[3] == 0 && len >= (int64_t(8) << 20)) b = std::min<int64_t>(b, 512);
  return (int)std::min<int64_t>(kMaxBuckets, std::max<int64_t>(2, b));
}

// ------------------------------------------------------------------ the sort
template <typename K, bool HAS_V>
struct Sorter {
  Ctx& c;
  K* keys;
  uint32_t* vals;
  int64_t n;
  K* wk = nullptr;
  uint32_t* wv = nullptr;
  uint16_t* d_bins_all = nullptr;
  static constexpr int64_t kw = sizeof(K);
  static constexpr int64_t vw = HAS_V ? 4 : 0;

  bool nested = false;  // sorting the outliers of an outlier route (no second outlier route)
  Sorter(Ctx& ctx, K* k, uint32_t* v, int64_t nn) : c(ctx), keys(k), vals(v), n(nn) {}

  // routes the device resolve may choose, and the forced route (outlier: keys only)
  int route_ok() const {
    return (g_merge_route ? kAllowMerge : 0) | ((!HAS_V && g_outlier && !nested) ? kAllowOutlier : 0) |
           ((!HAS_V && g_distance) ? kAllowDistance : 0);
  }

  // k-distance route (distance.cuh): window sorts, then window merges
  void run_distance(const DevStats* gate = nullptr) {
    if (!gate) c.plan.route = SR_ROUTE_DISTANCE;
    constexpr int PIECE = UnitNet<K>::PIECE;
    const size_t smem = sizeof(K) * PIECE * kDistWarps;
    set_smem(k_window_sort<K>, smem);
    set_smem(k_window_merge<K>, smem);
    const int64_t nwin = ceil_div<int64_t>(n, 2 * kDT);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div<int64_t>(nwin, kDistWarps), 148 * 16));
    K* kk = keys;
    const int64_t nn = n;
    c.launch("window_sort", gate ? 0 : 2 * n * kw, [&] {
      k_window_sort<K><<<grid, 32 * kDistWarps, smem, c.st>>>(kk, nn, gate);
    });
    c.launch("window_merge", gate ? 0 : 2 * n * kw, [&] {
      k_window_merge<K><<<grid, 32 * kDistWarps, smem, c.st>>>(kk, nn, gate);
    });
  }
  int forced() const {
    if (g_force_route == SR_ROUTE_OUTLIER && (HAS_V || nested)) return 0;
    return g_force_route;
  }

  void ensure_ws() {
    if (!wk) {
      wk = c.alloc<K>(n);
      if (HAS_V) wv = c.alloc<uint32_t>(n);
    }
  }

  // ---- finishing kernel over a device item list
  // NT = 128: items <= kSmallItem (2048 keys, one bitonic / merge tile);
  // NT = 256: items <= kCap (two 4096-key halves merged into global memory).
  template <int NT = kFinNT>
  int finish(const Item* items, const int64_t* count_ptr, int64_t begin, int64_t max_items, int64_t bytes,
             const DevStats* gate = nullptr, int64_t gate_route = 0) {
    if (max_items <= 0) return -1;
    size_t smem = FinishSmem<K, HAS_V, NT, kFinVT>::bytes();
    auto kern = k_finish<K, HAS_V, NT, kFinVT, (NT == kFinNT)>;
    set_smem(kern, smem);
    int grid = (int)std::min<int64_t>(max_items, gate ? 148 * 6 : 148 * 16);  // gated launches: few CTAs if off
    K* kk = keys;
    uint32_t* vv = vals;
    const K* wkk = wk;
    const uint32_t* wvv = wv;
    return c.launch(NT == kFinNT ? "finish" : "finish_small", bytes, [&] {
      kern<<<grid, NT, smem, c.st>>>(items, count_ptr, begin, kk, vv, wkk, wvv, gate, gate_route);
    });
  }

  int reverse_ranges(const std::vector<RunDesc>& ranges, const DevStats* gate = nullptr) {
    if (ranges.empty()) return -1;
    constexpr int NT = 256;
    constexpr int64_t CH = NT * 8;
    K* kk = keys;
    uint32_t* vv = vals;
    if (ranges.size() == 1 && ranges[0].start == 0 && ranges[0].len == n) {  // whole array: no upload
      const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n / 2, CH)));
      const int64_t nn = n;
      return c.launch("reverse", 2 * n * (kw + vw), [&] {
        k_reverse<K, HAS_V, NT><<<(unsigned)blocks, NT, 0, c.st>>>(kk, vv, nullptr, nullptr, 0, gate, nn);
      });
    }
    std::vector<int64_t> pre(ranges.size());
    int64_t tot = 0, bytes = 0;
    for (size_t i = 0; i < ranges.size(); i++) {
      pre[i] = tot;
      tot += std::max<int64_t>(1, ceil_div<int64_t>(ranges[i].len / 2, CH));
      bytes += 2 * ranges[i].len * (kw + vw);
    }
    RunDesc* d_r = c.alloc<RunDesc>(ranges.size());
    int64_t* d_p = c.alloc<int64_t>(pre.size());
    c.upload(d_r, ranges);
    c.upload(d_p, pre);
    int nr = (int)ranges.size();
    return c.launch("reverse", bytes,
             [&] { k_reverse<K, HAS_V, NT><<<(unsigned)tot, NT, 0, c.st>>>(kk, vv, d_r, d_p, nr, gate, 0); });
  }

  // ---- one partition level over `segs` of buffer src (0 primary, 1 ws); writes the other buffer.
  struct LevelOut {
    DevStats st;
    std::vector<OvfSeg> ovf;
  };

  // Level-1 state prepared before the route decision (fused with H1).
  struct Level {
    std::vector<SegDesc> segs;
    SegDesc* d_segs = nullptr;
    int* d_chunk_seg = nullptr;
    K* d_spl = nullptr;
    uint8_t* d_eq = nullptr;
    int* d_m = nullptr;
    uint32_t* d_mat = nullptr;
    int64_t mat_entries = 0;
    int64_t total_chunks = 0;
    int64_t chunk_size = 0;
    int64_t total_bins = 0;
    DevStats* d_st = nullptr;
    unsigned long long* d_status = nullptr;
    int* d_tile_counter = nullptr;
    int64_t scan_tiles = 0;
    Item* d_items = nullptr;      // small items (<= kSmallItem) and fills
    Item* d_items_big = nullptr;  // items in (kSmallItem, kCap]
    int64_t items_cap = 0;
    OvfSeg* d_ovf = nullptr;
    int src = 0;
    int level = 1;
    int warp_vt = 64;   // keys-only finishing: keys per lane (items <= 32 * warp_vt)
    int small_max = kSmallItem;
    // keys only: bucket totals + cursors instead of a count matrix (atomic scatter)
    bool atomic = false;
    uint32_t* d_tot = nullptr;
    uint32_t* d_cursor = nullptr;
    // splitter sample: per-segment ranks (zeroed) and keys
    uint32_t* d_rank = nullptr;
    K* d_sample = nullptr;
    uint16_t* d_bins = nullptr;  // per-key bucket ids from the count pass (indexed by position)
    GuideTab<K>* d_guide = nullptr;  // per-segment classification tables (k_guide_build)
    int64_t sample_total = 0;
    int max_sample = 0;
  };

  void level_alloc(Level& L, const std::vector<OvfSeg>& parts, int64_t chunk_size, int src, int forced_b = 0,
                   int level = 1) {
    L.src = src;
    L.chunk_size = chunk_size;
    L.level = level;
    L.warp_vt = (sizeof(K) == 4 && level == 1) ? 64 : 32;
    L.small_max = HAS_V ? kSmallItem : 32 * L.warp_vt;
    {  // keys only: atomic bucket reservation while the count matrix would be small,
       // else the matrix (one scan) -- thousands of CTAs hammering 4k cursors is slower
      int64_t ent = 0;
      for (auto& p : parts)
        ent += (2 * (int64_t)(forced_b ? forced_b : choose_buckets(p.len, level, (int)kw, !HAS_V)) + 1) * ceil_div<int64_t>(p.len, chunk_size);
      L.atomic = !HAS_V && ent <= kAtomicMaxEntries;
    }
    int64_t chunk_base = 0, mat = 0, lp = 0, bins = 0;
    std::vector<int> chunk_seg;
    for (size_t s = 0; s < parts.size(); s++) {
      SegDesc d;
      d.start = parts[s].start;
      d.len = parts[s].len;
      d.nbuckets = forced_b ? forced_b : choose_buckets(d.len, level, (int)kw, !HAS_V);
      d.nbins = 2 * d.nbuckets + 1;
      d.nchunks = (int32_t)ceil_div<int64_t>(d.len, chunk_size);
      d.chunk_base = (int32_t)chunk_base;
      d.mat_base = L.atomic ? bins : mat;  // keys only: bin base into totals / cursors
      d.len_prefix = lp;
      d.sample_base = L.sample_total;
      d.pad = 0;
      const int64_t S_s = std::min<int64_t>({d.len, (int64_t)d.nbuckets * kOversample, (int64_t)kMaxSample});
      L.sample_total += S_s;
      L.max_sample = std::max<int>(L.max_sample, (int)S_s);
      for (int g = 0; g < d.nchunks; g++) chunk_seg.push_back((int)s);
      chunk_base += d.nchunks;
      mat += (int64_t)d.nbins * d.nchunks;
      lp += d.len;
      bins += d.nbins;
      L.segs.push_back(d);
    }
    L.total_chunks = chunk_base;
    L.mat_entries = L.atomic ? 0 : mat;
    L.total_bins = bins;
    const int64_t S = (int64_t)parts.size();
    L.d_segs = c.alloc<SegDesc>(S);
    L.d_chunk_seg = c.alloc<int>(chunk_base);
    L.d_spl = c.alloc<K>(S * kMaxBuckets);
    L.d_eq = c.alloc<uint8_t>(S * kMaxBuckets);
    L.d_m = c.alloc<int>(S);
    L.scan_tiles = L.atomic ? 0 : ceil_div<int64_t>(mat, kScanNT * kScanIPT);
    if (!L.atomic) L.d_mat = c.alloc<uint32_t>(mat);
    // control block: stats | tile counter | scan status | bucket totals (zeroed together)
    const size_t tot_off = sizeof(DevStats) + 256 + sizeof(unsigned long long) * (size_t)L.scan_tiles;
    const size_t rank_off = tot_off + (L.atomic ? 4 * (size_t)bins : 0);
    size_t ctrl = rank_off + 4 * (size_t)L.sample_total;
    unsigned char* cb = c.alloc<unsigned char>((int64_t)ctrl);
    c.memset0(cb, ctrl);
    L.d_st = reinterpret_cast<DevStats*>(cb);
    L.d_tile_counter = reinterpret_cast<int*>(cb + sizeof(DevStats));
    L.d_status = reinterpret_cast<unsigned long long*>(cb + sizeof(DevStats) + 256);
    if (L.atomic) {
      L.d_tot = reinterpret_cast<uint32_t*>(cb + tot_off);
      L.d_cursor = c.alloc<uint32_t>(bins);
    }
    L.d_rank = reinterpret_cast<uint32_t*>(cb + rank_off);
    L.d_sample = c.alloc<K>(L.sample_total);
    if (!d_bins_all) d_bins_all = c.alloc<uint16_t>(n);
    L.d_bins = d_bins_all;
    L.items_cap = bins + lp / kFillChunk + (int64_t)parts.size() + 1;
    L.d_items = c.alloc<Item>(L.items_cap);
    L.d_items_big = c.alloc<Item>(bins);
    L.d_ovf = c.alloc<OvfSeg>(bins);
    c.upload(L.d_segs, L.segs);
    if (parts.size() == 1) c.memset0(L.d_chunk_seg, sizeof(int) * chunk_base);
    else c.upload(L.d_chunk_seg, chunk_seg);
  }

  const K* buf_k(int b) const { return b ? wk : keys; }
  const uint32_t* buf_v(int b) const { return b ? wv : vals; }

  // K7a + K7b.  gate: device stats whose route must be PARTITION (level-1
  // launches that precede the host's route decision), or nullptr.
  void level_splitters(Level& L, const DevStats* gate = nullptr) {
    constexpr int NT = 128;
    const K* src = buf_k(L.src);
    if (L.segs.size() > 1 || L.max_sample <= 2048) {  // many segments (levels >= 2): one CTA sorts each sample
      using BT = BitonicSort<K, 1024, 8>;
      auto kern = k_sample_sort<K, 1024, 8>;
      const size_t smem = sizeof(K) * BT::SMEM;
      set_smem(kern, smem);
      const int S = (int)L.segs.size();
      c.launch("sample_sort", L.sample_total * kw, [&] {
        kern<<<S, 1024, smem, c.st>>>(src, L.d_segs, kOversample, L.d_spl, L.d_eq, L.d_m, gate);
      });
      return;
    }
    // split each sample's comparisons over J chunks only when the sample is
    // large enough to keep a CTA busy (level 1); small level-2 samples: J = 1
    const int J = (int)std::max<int64_t>(1, std::min<int64_t>(8, L.max_sample / 1024));
    const size_t rsmem = sizeof(K) * (size_t)ceil_div<int64_t>(L.max_sample, J);
    set_smem(k_sample_rank<K, NT>, rsmem);
    const int S = (int)L.segs.size();
    int64_t pairs = 0;
    for (auto& sd : L.segs) {
      int64_t s_s = std::min<int64_t>({sd.len, (int64_t)sd.nbuckets * kOversample, (int64_t)kMaxSample});
      pairs += s_s * s_s;
    }
    dim3 grid((unsigned)ceil_div<int64_t>(L.max_sample, NT), J, (unsigned)S);
    c.launch("sample_rank", L.sample_total * kw * 2, [&] {
      k_sample_rank<K, NT><<<grid, NT, rsmem, c.st>>>(src, L.d_segs, kOversample, L.d_rank, L.d_sample, gate);
    });
    auto kern = k_select_splitters<K, 1024>;
    size_t smem = sizeof(K) * kMaxSample;
    set_smem(kern, smem);
    c.launch("select_splitters", L.sample_total * (kw + 4), [&] {
      kern<<<S, 1024, smem, c.st>>>(L.d_segs, kOversample, L.d_rank, L.d_sample, L.d_spl, L.d_eq, L.d_m, gate);
    });
    (void)pairs;
  }

  void level_count(Level& L, const DevStats* gate = nullptr) {
    const K* src = buf_k(L.src);
    int64_t keys_in = 0;
    for (auto& s : L.segs) keys_in += s.len;
    const int S = (int)L.segs.size();
    if (!L.d_guide) L.d_guide = c.alloc<GuideTab<K>>(S);
    c.launch("guide_build", 0, [&] {
      k_guide_build<K, 1024><<<S, 1024, 0, c.st>>>(L.d_spl, L.d_eq, L.d_m, L.d_guide, gate);
    });
    auto kern = k_count<K, kCountNT>;
    const size_t smem = sizeof(CountSmem<K>);
    set_smem(kern, smem);
    c.launch("count", keys_in * kw + L.mat_entries * 4, [&] {
      kern<<<(unsigned)L.total_chunks, kCountNT, smem, c.st>>>(src, L.d_segs, L.d_chunk_seg, L.chunk_size, L.d_guide,
                                                               L.d_mat, L.d_tot, L.d_bins, gate);
    });
  }

  void level_scan_plan(Level& L, const DevStats* gate = nullptr) {
    int64_t cnt = L.mat_entries;
    if (!L.atomic)
      c.launch("scan", cnt * 8, [&] {
        k_scan_u32<kScanNT, kScanIPT><<<(unsigned)L.scan_tiles, kScanNT, 0, c.st>>>(L.d_mat, cnt, L.d_status,
                                                                                   L.d_tile_counter, gate);
      });
    int S = (int)L.segs.size();
    int dst = 1 - L.src;
    auto kern = k_plan<K, 1024>;
    set_smem(kern, sizeof(PlanSmem));
    c.launch("plan", L.total_bins * 8, [&] {
      kern<<<S, 1024, sizeof(PlanSmem), c.st>>>(L.d_segs, L.d_mat, L.d_spl, L.d_m, dst, L.d_items, L.d_items_big,
                                                L.d_ovf, L.d_st, L.d_tot, L.d_cursor, gate, L.small_max,
                                                HAS_V ? L.small_max / 2 : kPackKeys);
    });
  }

  // hs == nullptr: speculative launch gated on the device route (level 1)
  int level_scatter(Level& L, const DevStats* hs) {
    if (hs && !HAS_V && hs->noneq_total == 0) return -1;  // keys-only, everything in equality buckets
    ensure_ws();
    const K* sk = buf_k(L.src);
    const uint32_t* sv = buf_v(L.src);
    K* dk = L.src ? keys : wk;
    uint32_t* dv = L.src ? vals : wv;
    int64_t keys_in = 0;
    for (auto& s : L.segs) keys_in += s.len;
    const int64_t noneq = hs ? hs->noneq_total : keys_in;
    const DevStats* gate = hs ? nullptr : L.d_st;
    const bool small = L.total_bins <= 1025 * (int64_t)L.segs.size() && [&] {
      for (auto& sd : L.segs) if (sd.nbins > 1025) return false;
      return true;
    }();
    // (A/B: 1 = two 512-thread CTAs per SM at every level, 2 = only where the
    // bin tables are small, 0 = one 1024-thread CTA per SM)
    if (!HAS_V && L.d_bins && (g_tune[5] == 1 || (g_tune[5] == 2 && small))) {
      constexpr int VT2 = sizeof(K) == 4 ? 16 : 8;
      auto launch2 = [&](auto kern, size_t smem) {
        set_smem(kern, smem);
        return c.launch("scatter", keys_in * kw + noneq * kw, [&] {
          kern<<<(unsigned)L.total_chunks, 512, smem, c.st>>>(sk, dk, L.d_segs, L.d_chunk_seg, L.chunk_size, L.d_cursor,
                                                               L.d_bins, L.atomic ? nullptr : L.d_mat, gate);
        });
      };
      if (small) return launch2(k_scatter_keys2<K, 512, VT2, 1025>, sizeof(ScatterKeys2Smem<K, 512, VT2, 1025>));
      return launch2(k_scatter_keys2<K, 512, VT2, kMaxBins>, sizeof(ScatterKeys2Smem<K, 512, VT2, kMaxBins>));
    }
    if (!HAS_V) {
      using SM = ScatterKeysSmem<K, kScatKNT, scat_kvt<K>()>;
      size_t smem = sizeof(SM);
      auto kern = k_scatter_keys<K, kScatKNT, scat_kvt<K>()>;
      set_smem(kern, smem);
      return c.launch("scatter", keys_in * kw + noneq * kw, [&] {
        kern<<<(unsigned)L.total_chunks, kScatKNT, smem, c.st>>>(sk, dk, L.d_segs, L.d_chunk_seg, L.chunk_size,
                                                                 L.d_spl, L.d_eq, L.d_m, L.d_cursor, L.d_bins,
                                                                 L.atomic ? nullptr : L.d_mat, gate);
      });
    }
    // two instances, each serving the segments of its bucket-table size class
    // (the compact one: few distinct splitters, guide.cuh md <= 255)
    using SM = ScatterSmem<K, HAS_V, kScatNT, scat_vt<K>(), kMaxBins>;
    using SMC = ScatterSmem<K, HAS_V, kScatNT, scat_vt<K>() / 4, kCompactBins>;
    const size_t smem = sizeof(SM), smemc = sizeof(SMC);
    auto kern = k_scatter<K, HAS_V, kScatNT, scat_vt<K>(), kMaxBins>;
    auto kernc = k_scatter<K, HAS_V, kScatNT, scat_vt<K>() / 4, kCompactBins>;
    set_smem(kern, smem);
    set_smem(kernc, smemc);
    int64_t bytes = keys_in * (kw + vw) + noneq * kw + keys_in * vw + L.mat_entries * 4 + keys_in * 2;
    c.launch("scatter", 0, [&] {  // (same name: the profile sums both instances' time)
      kernc<<<(unsigned)L.total_chunks, kScatNT, smemc, c.st>>>(sk, sv, dk, dv, L.d_segs, L.d_chunk_seg, L.chunk_size,
                                                                L.d_guide, L.d_mat, L.d_bins, gate);
    });
    return c.launch("scatter", bytes, [&] {
      kern<<<(unsigned)L.total_chunks, kScatNT, smem, c.st>>>(sk, sv, dk, dv, L.d_segs, L.d_chunk_seg, L.chunk_size,
                                                              L.d_guide, L.d_mat, L.d_bins, gate);
    });
  }

  // hs == nullptr: speculative level-1 launch gated on the device route; the
  // grid is sized by the item capacity and idle CTAs exit.
  // keys only: the small list (items <= 32*kWarpVT keys, and fills) goes to the
  // warp-register kernel
  template <int VT>
  int finish_warp(Level& L, int64_t max_items, int64_t bytes, const DevStats* gate, int min_len, int fills,
                  int max_grid) {
    constexpr int W = kWarpItemsPerCta;
    auto kern = k_finish_warp<K, VT, W>;
    const size_t smem = sizeof(K) * 32 * VT * W;
    set_smem(kern, smem);
    const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(max_items, W), gate ? 148 * 6 : max_grid);
    K* kk = keys;
    const K* wkk = wk;
    const int64_t* cnt = &L.d_st->n_items;
    return c.launch("finish_small", bytes, [&] {
      kern<<<grid, 32 * W, smem, c.st>>>(L.d_items, cnt, kk, wkk, gate, kRoutePartition, min_len, fills);
    });
  }
  // keys only: two launches over the small item list, by size class -- items
  // <= 512 keys (and fills) with the 16-key-per-lane network, larger ones with
  // the widest network the level allows
  // (min_len, 64 VH] keys: two VH-key-per-lane networks + a merge (k_finish_warp_split)
  template <int VH>
  void finish_split(Level& L, int64_t max_items, const DevStats* gate, int min_len) {
    constexpr int W = kWarpItemsPerCta;
    auto kern = k_finish_warp_split<K, VH, W>;
    const size_t smem = sizeof(K) * 2 * 32 * VH * W;
    set_smem(kern, smem);
    const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(max_items, W), gate ? 148 * 6 : 148 * 32);
    K* kk = keys;
    const K* wkk = wk;
    const int64_t* cnt = &L.d_st->n_items;
    c.launch("finish_small", 0, [&] {
      kern<<<grid, 32 * W, smem, c.st>>>(L.d_items, cnt, kk, wkk, gate, kRoutePartition, min_len);
    });
  }
  // keys only: launches over the small item list by size class.  Level 1
  // (64 keys per lane allowed): items <= 512 keys (and fills) with the
  // 16-key-per-lane network, larger ones with the 64-key network.  Deeper
  // levels: items <= 256 (and fills) with the 8-key network, (256, 512] and
  // (512, 1024] as two 8- / 16-key networks and a merge (SR_OPT_TUNE+7 = 1:
  // 16- and 32-key networks instead, measured slower: C5a 7.67 -> 7.43 ms)
  int finish_small(Level& L, int64_t max_items, int64_t bytes, const DevStats* gate) {
    if (HAS_V) return finish<kFinSmallNT>(L.d_items, &L.d_st->n_items, 0, max_items, bytes, gate, kRoutePartition);
    if (max_items <= 0) return -1;
    if (L.warp_vt == 64 && sizeof(K) == 4) {
      const int h = finish_warp<16>(L, max_items, bytes, gate, 0, 1, 148 * 64);
      finish_warp<64>(L, max_items, 0, gate, 512, 0, 148 * 16);
      return h;
    }
    if (g_tune[7] == 1) {
      const int h = finish_warp<16>(L, max_items, bytes, gate, 0, 1, 148 * 64);
      finish_warp<32>(L, max_items, 0, gate, 512, 0, 148 * 16);
      return h;
    }
    if (g_tune[7] == 2) {  // (the split for (512, 1024] only)
      const int h = finish_warp<16>(L, max_items, bytes, gate, 0, 1, 148 * 64);
      finish_split<16>(L, max_items, gate, 512);
      return h;
    }
    const int h = finish_warp<8>(L, max_items, bytes, gate, 0, 1, 148 * 64);
    finish_split<8>(L, max_items, gate, 256);
    finish_split<16>(L, max_items, gate, 512);
    return h;
  }

  int level_finish(Level& L, const DevStats* hs) {
    if (hs) {
      // sort items read+write their range keys; fills write keys (+ move vals)
      const int64_t big = hs->big_keys;
      int64_t bytes = 2 * (hs->noneq_total - hs->ovf_keys - big) * (kw + vw) + hs->eq_keys * kw +
                      (L.src == 0 ? 2 : 0) * hs->eq_keys * vw;
      c.plan.equal_keys += hs->eq_keys;
      int h = finish_small(L, hs->n_items, bytes, nullptr);
      finish(L.d_items_big, &L.d_st->n_items_big, 0, hs->n_items_big, 2 * big * (kw + vw));
      return h;
    }
    int h = finish_small(L, L.items_cap, 2 * n * (kw + vw), L.d_st);
    h_fin_big = finish(L.d_items_big, &L.d_st->n_items_big, 0, L.total_bins, 0, L.d_st, kRoutePartition);
    return h;
  }
  int h_fin_big = -1;

  // Fused level 2 + finishing (bucket_sort.cuh): keys only, the parts in the
  // workspace, every part small enough for one CTA's level of <= B2MAX bins.
  // A part qualifies when its B2MAX sub-buckets average at most half of what
  // one warp sorts (larger parts, e.g. from a skewed level-1 sample, take the
  // multi-kernel level).
  bool bs_fits(const OvfSeg& p, int src) const {
    return !HAS_V && src == 1 && g_tune[0] && p.len <= (int64_t)BsCfg<K>::B2MAX * (BsCfg<K>::PIECE / 2);
  }
  void run_bucket_sort(const std::vector<OvfSeg>& parts) {
    using C = BsCfg<K>;
    Level L;
    L.src = 1;
    L.level = 2;
    int64_t tot = 0;
    for (auto& p : parts) {
      SegDesc d{};
      d.start = p.start;
      d.len = p.len;
      d.nbuckets = (int)std::min<int64_t>(C::B2MAX, std::max<int64_t>(2, pow2ceil(ceil_div<int64_t>(p.len, std::max<int64_t>(16, g_tune[2])))));
      d.nbins = 2 * d.nbuckets + 1;
      d.sample_base = L.sample_total;
      const int64_t S_s = std::min<int64_t>({d.len, (int64_t)d.nbuckets * kOversample, (int64_t)kMaxSample});
      L.sample_total += S_s;
      L.max_sample = std::max<int>(L.max_sample, (int)S_s);
      tot += p.len;
      L.segs.push_back(d);
    }
    const int64_t S = (int64_t)parts.size();
    L.d_segs = c.alloc<SegDesc>(S);
    L.d_spl = c.alloc<K>(S * kMaxBuckets);
    L.d_eq = c.alloc<uint8_t>(S * kMaxBuckets);
    L.d_m = c.alloc<int>(S);
    // control block: stats | segment counter (zeroed together)
    unsigned char* cb = c.alloc<unsigned char>(sizeof(DevStats) + 256);
    c.memset0(cb, sizeof(DevStats) + 256);
    L.d_st = reinterpret_cast<DevStats*>(cb);
    uint32_t* d_counter = reinterpret_cast<uint32_t*>(cb + sizeof(DevStats));
    const int64_t big_cap = S * C::B2MAX;
    Item* d_big = c.alloc<Item>(big_cap);
    OvfSeg* d_ovf = c.alloc<OvfSeg>(big_cap);
    c.upload(L.d_segs, L.segs);
    level_splitters(L);
    auto kern = k_bucket_sort<K>;
    const size_t smem = sizeof(BsSmem<K>);
    set_smem(kern, smem);
    static int grid_cache[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (!grid_cache[dev]) {
      int per = 0, sms = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NT, smem);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      grid_cache[dev] = std::max(1, per) * std::max(1, sms);
    }
    const int grid = (int)std::min<int64_t>(S, grid_cache[dev]);
    K* kk = keys;
    const K* src = wk;
    const int nseg = (int)S;
    c.launch("bucket_sort", 2 * tot * kw, [&] {
      kern<<<grid, C::NT, smem, c.st>>>(src, kk, L.d_segs, nseg, L.d_spl, L.d_eq, L.d_m, d_counter, d_big, d_ovf,
                                        L.d_st, (int)g_tune[4]);
    });
    const int h_big = finish(d_big, &L.d_st->n_items_big, 0, big_cap, 0);
    DevStats hs = *reinterpret_cast<DevStats*>(c.readback(L.d_st, sizeof(DevStats)));
    c.replan(h_big, 2 * hs.big_keys * kw);
    c.plan.levels = 2;
    if (hs.n_ovf > 0) {
      const OvfSeg* h = reinterpret_cast<const OvfSeg*>(c.readback(d_ovf, sizeof(OvfSeg) * hs.n_ovf));
      std::vector<OvfSeg> next(h, h + hs.n_ovf);
      run_levels(next, 0, 3);
    }
  }

  // Partition levels >= 2 (segments from the previous level's oversized buckets).
  void run_levels(std::vector<OvfSeg> parts, int src, int level = 2) {
    {
      std::vector<OvfSeg> fused, rest;
      for (auto& p : parts) (bs_fits(p, src) ? fused : rest).push_back(p);
      if (!fused.empty()) {
        parts.swap(rest);
        run_bucket_sort(fused);  // (its own leftovers recurse from `keys`)
      }
    }
    while (!parts.empty()) {
      if (level > 12) fail(SR_ERR_INTERNAL, "partition did not converge");
      int64_t tot = 0;
      for (auto& p : parts) tot += p.len;
      int64_t cs = std::min<int64_t>(65536, std::max<int64_t>(4096, pow2ceil(std::max<int64_t>(1, tot / 512))));
      Level L;
      level_alloc(L, parts, cs, src, 0, level);
      level_splitters(L);
      level_count(L);
      level_scan_plan(L);
      DevStats hs = *reinterpret_cast<DevStats*>(c.readback(L.d_st, sizeof(DevStats)));
      if (hs.error) fail(SR_ERR_INTERNAL, "plan kernel inconsistency");
      std::vector<OvfSeg> next;
      if (hs.n_ovf > 0) {
        const OvfSeg* h = reinterpret_cast<const OvfSeg*>(c.readback(L.d_ovf, sizeof(OvfSeg) * hs.n_ovf));
        next.assign(h, h + hs.n_ovf);
        for (auto& o : next)
          for (auto& p : parts)
            if (o.start == p.start && o.len == p.len) fail(SR_ERR_INTERNAL, "partition made no progress");
      }
      level_scatter(L, &hs);
      level_finish(L, &hs);
      c.plan.levels = level;
      parts.swap(next);
      src = 1 - src;
      level++;
    }
  }

  // ---- merge route (natural runs, reversal, tile sort, half-down merge levels)
  struct Seg {
    int64_t start, len;
    int kind;  // 0 asc run, 1 desc run (reversed), 2 gap tile
  };

  // Simulated half-down merge tree (Appendix A).
  struct Node {
    int64_t start, len;
    int left = -1, right = -1;
    int depth = 0;
    int buf = 0;
  };

  static std::vector<Node> half_down_tree(const std::vector<std::pair<int64_t, int64_t>>& runs, int& root) {
    std::vector<Node> nodes;
    std::vector<int> stack;
    auto merge_top = [&]() {
      int b = stack.back();
      stack.pop_back();
      int a = stack.back();
      stack.pop_back();
      Node m;
      m.start = nodes[a].start;
      m.len = nodes[a].len + nodes[b].len;
      m.left = a;
      m.right = b;
      m.depth = 1 + std::max(nodes[a].depth, nodes[b].depth);
      nodes.push_back(m);
      stack.push_back((int)nodes.size() - 1);
    };
    for (auto& r : runs) {
      Node l;
      l.start = r.first;
      l.len = r.second;
      nodes.push_back(l);
      stack.push_back((int)nodes.size() - 1);
      // "merge two runs if the current run > 1/2 of its predecessor"
      while (stack.size() > 1 && nodes[stack.back()].len > (nodes[stack[stack.size() - 2]].len >> 1)) merge_top();
    }
    while (stack.size() > 1) merge_top();  // "merge all runs into one, from last to first"
    root = stack.empty() ? -1 : stack.back();
    return nodes;
  }

  // bytes of the merge schedule (merges + harmonising copies + final copy)
  static int64_t schedule_bytes(std::vector<Node>& nodes, int root, int64_t elem_bytes) {
    int64_t b = 0;
    std::vector<int> order(nodes.size());
    for (size_t i = 0; i < nodes.size(); i++) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return nodes[x].depth < nodes[y].depth; });
    for (int i : order) {
      Node& nd = nodes[i];
      if (nd.left < 0) { nd.buf = 0; continue; }
      Node& A = nodes[nd.left];
      Node& B = nodes[nd.right];
      int in = A.buf;
      if (A.buf != B.buf) {
        in = A.len >= B.len ? A.buf : B.buf;
        b += 2 * std::min(A.len, B.len) * elem_bytes;
      }
      nd.buf = 1 - in;
      b += 2 * nd.len * elem_bytes;
    }
    if (root >= 0 && nodes[root].buf == 1) b += 2 * nodes[root].len * elem_bytes;
    return b;
  }

  std::vector<Seg> build_segments(const std::vector<RunDesc>& asc, const std::vector<RunDesc>& desc) {
    std::vector<Seg> runs;
    for (auto& r : asc) runs.push_back({r.start, r.len, 0});
    // descending runs trimmed against ascending runs (a shared
    // boundary element goes to the ascending run; a sub-range of a descending
    // run is still descending)
    size_t ai = 0;
    for (auto& r : desc) {
      int64_t s = r.start, e = r.start + r.len;
      while (ai < asc.size() && asc[ai].start + asc[ai].len <= s) ai++;
      for (size_t k = ai; k < asc.size() && asc[k].start < e; k++) {
        int64_t as = asc[k].start, ae = asc[k].start + asc[k].len;
        if (as <= s && ae > s) s = ae;
        else if (as > s && as < e) e = as;
      }
      if (e - s >= 2) runs.push_back({s, e - s, 1});
    }
    std::sort(runs.begin(), runs.end(), [](const Seg& a, const Seg& b) { return a.start < b.start; });
    std::vector<Seg> segs;
    int64_t pos = 0;
    auto gap = [&](int64_t s, int64_t e) {
      for (int64_t p = s; p < e; p += kCap) segs.push_back({p, std::min<int64_t>(kCap, e - p), 2});
    };
    for (auto& r : runs) {
      if (r.start > pos) gap(pos, r.start);
      int64_t s = std::max(pos, r.start);
      if (r.start + r.len > s) segs.push_back({s, r.start + r.len - s, r.kind});
      pos = std::max(pos, r.start + r.len);
    }
    if (pos < n) gap(pos, n);
    return segs;
  }

  int64_t merge_route_bytes(const std::vector<Seg>& segs) {
    int64_t b = 0;
    std::vector<std::pair<int64_t, int64_t>> runs;
    for (auto& s : segs) {
      if (s.kind != 0) b += 2 * s.len * (kw + vw);
      runs.push_back({s.start, s.len});
    }
    int root;
    auto nodes = half_down_tree(runs, root);
    return b + schedule_bytes(nodes, root, kw + vw);
  }

  void run_merge_route(const std::vector<Seg>& segs0) {
    // H2: reverse descending runs in place
    std::vector<RunDesc> rev;
    std::vector<Item> tiles;
    for (auto& s : segs0) {
      if (s.kind == 1) rev.push_back({s.start, s.len, 0, 0});
      if (s.kind == 2) {
        Item it;
        it.start = s.start;
        it.len = (int32_t)s.len;
        it.kind = kItemSort;
        it.key = 0;
        tiles.push_back(it);
      }
    }
    c.plan.desc_runs_reversed = (int64_t)rev.size();
    reverse_ranges(rev);
    // H4: sort gap tiles in place
    if (!tiles.empty()) {
      Item* d_items = c.alloc<Item>(tiles.size());
      int64_t* d_cnt = c.alloc<int64_t>(1);
      c.upload(d_items, tiles);
      std::vector<int64_t> cnt{(int64_t)tiles.size()};
      c.upload(d_cnt, cnt);
      int64_t gl = 0;
      for (auto& t : tiles) gl += t.len;
      finish(d_items, d_cnt, 0, (int64_t)tiles.size(), 2 * gl * (kw + vw));
    }
    // post-reversal boundary check: coalesce runs whose boundary is ordered
    // (trimmed merges); a fully ordered set is the
    // "sorted after reversal" exit.
    std::vector<int64_t> bpos;
    for (size_t i = 1; i < segs0.size(); i++) bpos.push_back(segs0[i].start);
    std::vector<std::pair<int64_t, int64_t>> runs;
    if (!bpos.empty()) {
      int64_t nb = (int64_t)bpos.size();
      int64_t* d_pos = c.alloc<int64_t>(nb);
      uint8_t* d_flags = c.alloc<uint8_t>(nb + 8);
      unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(c.alloc<unsigned long long>(1));
      c.memset0(d_bad, 8);
      c.upload(d_pos, bpos);
      const K* kk = keys;
      c.launch("boundary", nb * 2 * kw, [&] {
        k_boundary_check<K><<<(unsigned)ceil_div<int64_t>(nb, 256), 256, 0, c.st>>>(kk, d_pos, nb, d_flags, d_bad);
      });
      const uint8_t* flags = reinterpret_cast<const uint8_t*>(c.readback(d_flags, (size_t)nb));
      int64_t s = segs0[0].start, l = segs0[0].len;
      for (int64_t i = 0; i < nb; i++) {
        const Seg& g = segs0[i + 1];
        if (flags[i]) { runs.push_back({s, l}); s = g.start; l = g.len; }
        else l += g.len;
      }
      runs.push_back({s, l});
    } else {
      runs.push_back({0, n});
    }
    if (runs.size() == 1) { c.plan.levels = 0; return; }
    // H6: half-down merge tree, executed level by level
    int root;
    auto nodes = half_down_tree(runs, root);
    schedule_bytes(nodes, root, kw + vw);  // assigns buffers
    ensure_ws();
    int maxd = nodes[root].depth;
    for (int d = 1; d <= maxd; d++) {
      std::vector<CopyJob> copies;
      std::vector<MergeJob> jobs;
      int64_t cta = 0, ccta = 0, mbytes = 0, cbytes = 0;
      for (auto& nd : nodes) {
        if (nd.depth != d || nd.left < 0) continue;
        Node& A = nodes[nd.left];
        Node& B = nodes[nd.right];
        int in = A.buf;
        if (A.buf != B.buf) {
          in = A.len >= B.len ? A.buf : B.buf;
          Node& mv = (A.buf == in) ? B : A;
          CopyJob cj{mv.start, mv.len, ccta, in == 1 ? 0 : 1, 0};  // dir 0: primary->ws
          copies.push_back(cj);
          ccta += ceil_div<int64_t>(mv.len, 256 * 8);
          cbytes += 2 * mv.len * (kw + vw);
        }
        MergeJob j{nd.start, A.len, B.len, cta, in, 0};
        jobs.push_back(j);
        cta += ceil_div<int64_t>(nd.len, kMergeNV);
        mbytes += 2 * nd.len * (kw + vw);
      }
      if (!copies.empty()) run_copies(copies, ccta, cbytes);
      run_merges(jobs, cta, mbytes);
    }
    if (nodes[root].buf == 1) {
      std::vector<CopyJob> cj{{0, n, 0, 1, 0}};
      run_copies(cj, ceil_div<int64_t>(n, 256 * 8), 2 * n * (kw + vw));
    }
    c.plan.levels = maxd;
  }

  void run_copies(const std::vector<CopyJob>& jobs, int64_t ctas, int64_t bytes) {
    CopyJob* d = c.alloc<CopyJob>(jobs.size());
    c.upload(d, jobs);
    int nj = (int)jobs.size();
    K* kk = keys;
    uint32_t* vv = vals;
    K* w = wk;
    uint32_t* wvv = wv;
    c.launch("copy", bytes, [&] { k_copy<K, HAS_V, 256><<<(unsigned)ctas, 256, 0, c.st>>>(kk, vv, w, wvv, d, nj); });
  }

  void run_merges(const std::vector<MergeJob>& jobs, int64_t ctas, int64_t bytes) {
    MergeJob* d = c.alloc<MergeJob>(jobs.size());
    int64_t* splits = c.alloc<int64_t>(ctas + 1);
    c.upload(d, jobs);
    int nj = (int)jobs.size();
    const K* kk = keys;
    const K* w = wk;
    c.launch("merge_partition", ctas * 2 * 20 * kw, [&] {
      k_merge_partition<K, kMergeNV><<<(unsigned)ceil_div<int64_t>(ctas, 256), 256, 0, c.st>>>(kk, w, d, nj, ctas, splits);
    });
    size_t smem = sizeof(K) * padded_size<K>(kMergeNV) + (HAS_V ? 4 * padded_size<uint32_t>(kMergeNV) : 0);
    auto kern = k_merge<K, HAS_V, kMergeNT, kMergeVT>;
    set_smem(kern, smem);
    K* pk = keys;
    uint32_t* pv = vals;
    K* wkk = wk;
    uint32_t* wvv = wv;
    c.launch("merge", bytes, [&] { kern<<<(unsigned)ctas, kMergeNT, smem, c.st>>>(pk, pv, wkk, wvv, d, nj, splits); });
  }

  // ---- resident path: the whole keys-only sort as one cooperative launch (resident.cuh)
  static int resident_grid() {  // CTAs of the cooperative launch (one per SM) on the current device, 0 if it cannot run
    static std::mutex mu;
    static int grid[kMaxDevices][2];
    static bool init[kMaxDevices][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) return 0;
    std::lock_guard<std::mutex> lk(mu);
    int& g = grid[dev][sizeof(K) == 8];
    if (!init[dev][sizeof(K) == 8]) {
      init[dev][sizeof(K) == 8] = true;
      g = 0;
      int sms = 0, coop = 0, per = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
      const size_t smem = sizeof(ResSmem<K>);
      if (coop && cudaFuncSetAttribute(k_resident<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                      cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_resident<K>, kResNT, smem) == cudaSuccess &&
          per >= kResCtasPerSM)
        g = sms * kResCtasPerSM;  // the phases are sized for this many co-resident CTAs
      cudaGetLastError();
    }
    return g;
  }
  bool resident_ok() const {
    if (HAS_V || !g_resident || n <= kCap || n > ResCfg<K>::MAXN) return false;
    if (g_force_route == SR_ROUTE_MERGE && !nested) return false;  // forced merge: the multi-kernel planner
    const int P = resident_grid();
    // every CTA but the samplers holds <= GPC tiles
    return P >= 16 && n <= (int64_t)ResSmem<K>::GPC * (P - kResSamplers) * kResGrp;
  }

  void run_resident() {
    c.plan.n = n;
    const int64_t T = choose_tile(n);  // L_min of the run detection (R5)
    const int P = resident_grid();
    // scan / grouping tile: a multiple of the CTA width, sized so that every
    // CTA gets <= GPC tiles and the last kResSamplers CTAs (the samplers) one
    // (each held tile costs a pass over the bucket tables: as few per CTA as fit)
    const int64_t gpc = std::min<int64_t>(ResSmem<K>::GPC, ceil_div<int64_t>(n, (int64_t)(P - kResSamplers) * kResGrp));
    const int64_t slots = gpc * (P - kResSamplers);  // the samplers hold no tile
    const int64_t tile = std::min<int64_t>(kResGrp, ceil_div<int64_t>(ceil_div<int64_t>(n, slots), kResNT) * kResNT);
    const int64_t G = ceil_div<int64_t>(n, tile);
    constexpr int CAPB = ResCfg<K>::CAPB;
    const int B1 = (int)std::min<int64_t>(ResCfg<K>::B1MAX, std::max<int64_t>(2, pow2ceil(ceil_div<int64_t>(n, ResCfg<K>::TARGET))));
    const int NG = (int)G;
    const int S1 = B1 * ResCfg<K>::O1;
    const int nbins = 2 * B1 + 1;
    const int64_t n_ovf = B1 + 1;
    if (NG > slots || G > kResMaxG) fail(SR_ERR_INTERNAL, "resident tile count");
    // in-kernel outlier route (resident.cuh ResOut): keys only, n within its bucket range
    using RO = ResOut<K>;
    const bool out_res = (route_ok() & kAllowOutlier) && n <= RO::MAXN;
    const int64_t GO = ceil_div<int64_t>(n, RO::TO);
    const int64_t obk = ceil_div<int64_t>(n, RO::OL);  // most buckets it can use
    {
      auto r = [](int64_t b) { return (b + 255) & ~int64_t(255); };
      const size_t bytes = (size_t)(r(n * kw) + r(G * 32) + 2 * r((G + 1) * 32) + r(sizeof(DevStats) + 32 + 4 * nbins) +
                                    2 * r(S1 * kw) + r(ResCfg<K>::B1MAX * kw) + r(ResCfg<K>::B1MAX) + r(16 * n_ovf) +
                                    r(4 * ResCfg<K>::B1MAX) + r(G * (int64_t)sizeof(TileMM)) +
                                    r(4 * (int64_t)NG * nbins) + r(4 * (RO::OBMAX + 2)) +
                                    (out_res ? r(4 * GO) + r(2 * GO * kw) + r(obk * RO::OCAP * kw) : 0) +
                                    r(sizeof(GuideTab<K, 2048, ResCfg<K>::B1MAX>)) + 13 * 256);
      DevState& dsa = t_state.ds();
      if (dsa.has_last && dsa.last_stream != c.st)  // the arena of the last call is in use until its kernel ends
        check_cuda(cudaStreamWaitEvent(c.st, dsa.last_ev, 0), "cudaStreamWaitEvent");
      c.ws_check(bytes);
      if (dsa.res_arena && dsa.res_arena_bytes < bytes) {  // too small: freed stream-ordered
        c.allocs.push_back(dsa.res_arena);
        dsa.res_arena = nullptr;
      }
      if (!dsa.res_arena) {
        void* p = nullptr;
        check_cuda(cudaMallocAsync(&p, bytes, c.st), "cudaMallocAsync");
        dsa.res_arena = reinterpret_cast<unsigned char*>(p);
        dsa.res_arena_bytes = bytes;
      }
      c.use_arena(dsa.res_arena, dsa.res_arena_bytes);
      c.plan.workspace_bytes += (int64_t)dsa.res_arena_bytes;
    }
    hostprof("reserved");
    ensure_ws();
    ResArgs<K> a;
    a.keys = keys;
    a.ws = wk;
    a.n = n;
    a.tile = (int)tile;
    a.G = (int)G;
    a.sums = c.alloc<TileSummary>(G);
    a.mm = c.alloc<TileMM>(G);
    a.asc = c.alloc<RunDesc>(G + 1);
    a.desc = c.alloc<RunDesc>(G + 1);
    {  // control block: statistics | unit counters | bucket totals, zeroed by the kernel
      const size_t bytes =
          sizeof(DevStats) + 32 + 4 * (size_t)nbins + 4 * (size_t)ResCfg<K>::B1MAX + 4 * (size_t)(RO::OBMAX + 2);
      unsigned char* cb = c.alloc<unsigned char>((int64_t)bytes);
      a.st = reinterpret_cast<DevStats*>(cb);
      a.unit_counter = reinterpret_cast<uint32_t*>(cb + sizeof(DevStats));
      a.tot = reinterpret_cast<uint32_t*>(cb + sizeof(DevStats) + 32);
      a.pairc = a.tot + nbins;
      a.ocnt = a.pairc + ResCfg<K>::B1MAX;
      a.ctrl_words = (int)(bytes / 4);
    }
    DevState& ts = t_state.ds();
    if (!ts.done_h) {
      check_cuda(cudaHostAlloc((void**)&ts.done_h, sizeof(ResDone), cudaHostAllocMapped), "cudaHostAlloc(mapped)");
      check_cuda(cudaHostGetDevicePointer((void**)&ts.done_d, ts.done_h, 0), "cudaHostGetDevicePointer");
      ts.done_h->seq = 0;
    }
    a.done = ts.done_d;
    a.seq = ++ts.done_seq == 0 ? ++ts.done_seq : ts.done_seq;
    if (!ts.arrive) {
      check_cuda(cudaMalloc((void**)&ts.arrive, 256), "cudaMalloc(arrive)");
      check_cuda(cudaMemset(ts.arrive, 0, 256), "cudaMemset(arrive)");
      ts.arrive_base = 0;
      ts.scount_base = 0;
    }
    if (!ts.last_ev) check_cuda(cudaEventCreateWithFlags(&ts.last_ev, cudaEventDisableTiming), "cudaEventCreate");
    if (!ts.launch_ev) check_cuda(cudaEventCreateWithFlags(&ts.launch_ev, cudaEventDisableTiming), "cudaEventCreate");
    a.arrive = ts.arrive;
    a.arrive_base = ts.arrive_base;
    a.scount = ts.arrive + 16;
    a.scount_base = ts.scount_base;
    a.guide = reinterpret_cast<GuideTab<K, 2048, ResCfg<K>::B1MAX>*>(
        c.alloc<unsigned char>((int64_t)sizeof(GuideTab<K, 2048, ResCfg<K>::B1MAX>)));
    a.S1 = S1;
    a.B1 = B1;
    a.samp = c.alloc<K>(S1);
    a.mrg = c.alloc<K>(S1);
    a.spl = c.alloc<K>(ResCfg<K>::B1MAX);
    a.spf = c.alloc<uint8_t>(ResCfg<K>::B1MAX);
    a.goff = c.alloc<uint32_t>((int64_t)NG * nbins);
    a.NG = NG;
    a.ovf = c.alloc<OvfSeg>(n_ovf);
    a.lmin = T;
    a.force = forced();
    // the outlier route runs in this launch when it can; otherwise the one-launch
    // partition beats the host-driven outlier rounds at this size unless the
    // outliers are very few
    a.merge_ok = route_ok() | (out_res ? 0 : kOutlierStrict);
    a.out_res = out_res ? 1 : 0;
    a.GO = (int)GO;
    a.okc = out_res ? c.alloc<uint32_t>(GO) : nullptr;
    a.ofl = out_res ? c.alloc<K>(2 * GO) : nullptr;
    a.obuf = out_res ? c.alloc<K>(obk * RO::OCAP) : nullptr;
    a.capb = std::min(CAPB, g_res_cap);
    static const bool stamps = getenv("SR_TIMING") != nullptr;
    a.tstamp = stamps ? c.alloc<unsigned long long>(8 * P + 64) : nullptr;
    if (stamps) c.memset0(a.tstamp, 8 * (8 * P + 64));
    const size_t smem = sizeof(ResSmem<K>);
    hostprof("prepared");
    check_cuda(cudaEventRecord(ts.launch_ev, c.st), "cudaEventRecord");
    const int h = c.launch("resident", n * kw, [&] {
      void* args[] = {&a};
      check_cuda(launch_coop((const void*)k_resident<K>, P, kResNT, args, smem, c.st), "resident launch");
    });
    ts.arrive_base += (uint32_t)P + 1u;  // every CTA arrives once, CTA 0 once more (route published)
    ts.scount_base += 3u * kResSamplers;  // the samplers' three steps
    check_cuda(cudaEventRecord(ts.last_ev, c.st), "cudaEventRecord");
    ts.last_stream = c.st;
    ts.has_last = true;
    hostprof("launched");
    int in_kernel = 0;
    DevStats hs;
    try {
      hs = c.await_done(ts.done_h, a.seq, ts.launch_ev, &in_kernel);
    } catch (...) {
      ts.abandon();  // the kernel may still be running on these
      throw;
    }
    hostprof("read back");
    if (stamps) {
      const unsigned long long* t = reinterpret_cast<const unsigned long long*>(c.readback(a.tstamp, 8 * (8 * P + 64)));
      {
        const unsigned long long* q = t + 8 + 8 * P + 8;
        if (q[0] && q[5])
          fprintf(stderr, "[sr_resident] C group0 us: classify %.1f count %.1f tables+atomics %.1f scan %.1f scatter %.1f\n",
                  (q[1] - q[0]) * 1e-3, (q[2] - q[1]) * 1e-3, (q[3] - q[2]) * 1e-3, (q[4] - q[3]) * 1e-3, (q[5] - q[4]) * 1e-3);
      }
      {
        if (t[8 + 8 * P + 33])
          fprintf(stderr, "[sr_resident] route step of CTA 0, us since start: all arrived %.1f summaries loaded %.1f resolved %.1f\n",
                  (t[1] - t[0]) * 1e-3, (t[8 + 8 * P + 32] - t[0]) * 1e-3, (t[8 + 8 * P + 33] - t[0]) * 1e-3);
      }
      {
        const unsigned long long* q = t + 8 + 8 * P + 16;
        if (q[0] && q[2])
          fprintf(stderr, "[sr_resident] C splitters (sampler 0) us since start: gathered %.1f quarter sorted %.1f pieces sorted %.1f loaded %.1f half merged %.1f merged %.1f selected %.1f guide %.1f\n",
                  (q[5] - t[0]) * 1e-3, (q[6] - t[0]) * 1e-3, (q[0] - t[0]) * 1e-3, (q[1] - t[0]) * 1e-3, (q[4] - t[0]) * 1e-3, (q[2] - t[0]) * 1e-3, (q[3] - t[0]) * 1e-3,
                  q[7] ? (q[7] - t[0]) * 1e-3 : 0.0);
      }
      {
        const unsigned long long* q = t + 8 + 8 * P + 40;
        if (q[0] && q[2])
          fprintf(stderr, "[sr_resident] outlier CTA0 us: OA flags %.1f split+write %.1f | koff %.1f check %.1f splitters %.1f classify %.1f | OD start %.1f; warp0 unit: load %.1f sort %.1f merge %.1f\n",
                  (q[1] - q[0]) * 1e-3, (q[2] - q[1]) * 1e-3, q[3] ? (q[3] - t[8 + 4]) * 1e-3 : 0.0,
                  q[4] ? (q[4] - q[3]) * 1e-3 : 0.0, q[5] ? (q[5] - q[4]) * 1e-3 : 0.0, q[6] ? (q[6] - q[5]) * 1e-3 : 0.0,
                  q[7] ? (q[7] - t[0]) * 1e-3 : 0.0, q[11] ? (q[11] - q[10]) * 1e-3 : 0.0,
                  q[12] ? (q[12] - q[11]) * 1e-3 : 0.0, q[13] && q[12] ? (q[13] - q[12]) * 1e-3 : 0.0);
      }
      {
        const unsigned long long* q = t + 8 + 8 * P + 24;
        fprintf(stderr, "[sr_resident] E items us: longest CTA unit %.1f (%llu units), longest warp unit %.1f\n",
                q[0] * 1e-3, q[1], q[2] * 1e-3);
      }
      {
        const unsigned long long* e = t + 8 + 8 * P;
        fprintf(stderr, "[sr_resident] CTA0 %llu buckets, us: load %.1f is_sorted+sample %.1f classify+move %.1f warp sorts %.1f\n",
                e[7], e[5] * 1e-3, e[0] * 1e-3, e[1] * 1e-3, e[2] * 1e-3);
      }
      static const char* what[8] = {"A.scan", "A.end", "C.route", "C.tree", "C.end", "D.end", "E.end", "-"};
      for (int k = 0; k < 7; k++) {
        std::vector<double> v;
        for (int q = 0; q < P; q++)
          if (t[8 + 8 * q + k]) v.push_back((double)(t[8 + 8 * q + k] - t[0]) * 1e-3);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        fprintf(stderr, "[sr_resident]   %-8s since start: min %6.1f  med %6.1f  max %6.1f us  (%zu CTAs)\n", what[k], v[0],
                v[v.size() / 2], v.back(), v.size());
      }
      fprintf(stderr, "[sr_resident] n=%lld B1=%d route=%lld phases us: A %.1f C %.1f E %.1f\n", (long long)n, B1,
              (long long)hs.route, (t[1] - t[0]) * 1e-3, t[2] ? (t[2] - t[1]) * 1e-3 : 0.0,
              t[3] ? (t[3] - t[2]) * 1e-3 : 0.0);
    }
    c.plan.descents = hs.descents;
    c.plan.asc_breaks = hs.asc_breaks;
    c.plan.long_runs = hs.n_asc_runs + hs.n_desc_runs;
    if (hs.error) fail(SR_ERR_INTERNAL, "resident kernel inconsistency");
    // the launch finishes the sort by itself unless the record says otherwise:
    // the host returns now, while the kernel is still running.  Otherwise the
    // host continues once the kernel has ended, from its final statistics; the
    // arena's buffers feed that continuation, so it is released with this call
    // (stream-ordered) instead of being reused.
    if (!in_kernel) {
      hs = *reinterpret_cast<const DevStats*>(c.readback(a.st, sizeof(DevStats)));
      c.allocs.push_back(ts.res_arena);
      ts.res_arena = nullptr;
      ts.res_arena_bytes = 0;
    }
    switch (hs.route) {
      case kRouteSorted:
        c.plan.route = SR_ROUTE_SORTED;
        return;
      case kRouteReversed:
        c.plan.route = SR_ROUTE_REVERSED;
        c.plan.desc_runs_reversed = 1;
        c.replan(h, 3 * n * kw);
        return;
      case kRouteDistance:
        run_distance();
        return;
      case kRoutePartition: {
        c.plan.route = SR_ROUTE_PARTITION;
        c.plan.levels = 2;  // the global level and the in-CTA level
        c.plan.equal_keys += hs.eq_keys;
        // scan (read) + classification (read) + range keys written to their
        // buckets in ws, read back and written sorted + equality fills (written)
        c.replan(h, 2 * n * kw + 3 * hs.noneq_total * kw + hs.eq_keys * kw);
        if (hs.n_ovf > 0) {  // ranges left unsorted in keys (beyond the in-kernel caps): further levels
          const OvfSeg* o = reinterpret_cast<const OvfSeg*>(c.readback(a.ovf, sizeof(OvfSeg) * hs.n_ovf));
          std::vector<OvfSeg> next(o, o + hs.n_ovf);
          run_levels(next, 0);
        }
        return;
      }
      default:
        break;
    }
    if (hs.route == kRouteOutlier && in_kernel) {  // the launch ran the outlier route
      c.plan.route = SR_ROUTE_OUTLIER;
      // scan (read), tiles read + kept / outliers written, buckets read + written
      c.replan(h, 5 * n * kw);
      return;
    }
    c.replan(h, n * kw);
    if (hs.route == kRouteOutlier) {
      c.plan.route = SR_ROUTE_OUTLIER;
      if (run_outlier()) return;
      partition_host(T);  // not a few-outlier input: keys hold a permutation
      return;
    }
    // MERGE (forced) or undecided: the host planner compares the routes' bytes
    std::vector<RunDesc> asc, desc;
    if (hs.n_asc_runs) {
      const RunDesc* p = reinterpret_cast<const RunDesc*>(c.readback(a.asc, sizeof(RunDesc) * hs.n_asc_runs));
      asc.assign(p, p + hs.n_asc_runs);
    }
    if (hs.n_desc_runs) {
      const RunDesc* p = reinterpret_cast<const RunDesc*>(c.readback(a.desc, sizeof(RunDesc) * hs.n_desc_runs));
      desc.assign(p, p + hs.n_desc_runs);
    }
    std::vector<Seg> segs = build_segments(asc, desc);
    bool use_merge = hs.route == kRouteMerge;
    if (!use_merge) {
      const int64_t N = n * (kw + vw);
      use_merge = merge_route_bytes(segs) < 4 * N + (n > 4 * 1024 * 1024 ? 3 * N : 0);
    }
    if (use_merge) {
      c.plan.route = SR_ROUTE_MERGE;
      run_merge_route(segs);
      return;
    }
    partition_host(T);
  }

  // ---- outlier route (outlier.cuh): few descents, keys only.  One round
  // compacts src[0, m) into dst: kept keys [0, r), outliers [r, m); returns r
  // and the number of descents among the kept keys.
  std::pair<int64_t, int64_t> outlier_round(const K* src, int64_t m, K* dst) {
    constexpr int T = OutTile<K>::T;
    const int64_t G = ceil_div<int64_t>(m, T);
    uint32_t* cnt = c.alloc<uint32_t>(G + 1);
    K* fl = c.alloc<K>(2 * G);
    uint8_t* has = c.alloc<uint8_t>(G);
    const int64_t tiles = ceil_div<int64_t>(G + 1, kScanNT * kScanIPT);
    unsigned char* ctrl = c.alloc<unsigned char>(64 + 8 * tiles + 256);
    c.memset0(ctrl, 64 + 8 * tiles + 256);
    unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctrl);
    int* tile_counter = reinterpret_cast<int*>(ctrl + 8);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(ctrl + 64);
    c.memset0(cnt + G, 4);
    c.launch("outlier_count", m * kw, [&] {
      k_outlier_count<K, kOutNT><<<(unsigned)G, kOutNT, 0, c.st>>>(src, m, cnt);
    });
    c.launch("scan", (G + 1) * 8, [&] {
      k_scan_u32<kScanNT, kScanIPT><<<(unsigned)tiles, kScanNT, 0, c.st>>>(cnt, G + 1, status, tile_counter, nullptr);
    });
    c.launch("outlier_split", 2 * m * kw, [&] {
      k_outlier_split<K, kOutNT><<<(unsigned)G, kOutNT, 0, c.st>>>(src, m, cnt, (int)G, dst, fl, has, bad);
    });
    c.launch("outlier_check", 0, [&] {
      k_outlier_check<K><<<(unsigned)ceil_div<int64_t>(G, 256), 256, 0, c.st>>>(fl, has, (int)G, bad);
    });
    // r = cnt[G] and the descent count, in one readback (both live in device memory)
    uint32_t* pair = c.alloc<uint32_t>(4);
    check_cuda(cudaMemcpyAsync(pair, cnt + G, 4, cudaMemcpyDeviceToDevice, c.st), "outlier r");
    check_cuda(cudaMemcpyAsync(pair + 2, bad, 8, cudaMemcpyDeviceToDevice, c.st), "outlier bad");
    const uint32_t* h = reinterpret_cast<const uint32_t*>(c.readback(pair, 16));
    const int64_t r = h[0];
    const int64_t nb = (int64_t)h[2] | ((int64_t)h[3] << 32);
    return {r, nb};
  }

  // sort dst[0, m) by the ordinary routes (the outliers), keeping this call's plan
  void sort_nested(K* p, int64_t m) {
    if (m <= 1) return;
    sr_plan saved = c.plan;
    Sorter<K, HAS_V> sub(c, p, nullptr, m);
    sub.nested = true;
    sub.run();
    const int64_t launches = c.plan.launches, bytes = c.plan.bytes_planned, syncs = c.plan.host_syncs;
    c.plan = saved;
    c.plan.launches = launches;
    c.plan.bytes_planned = bytes;
    c.plan.host_syncs = syncs;
  }

  void merge_two(int buf, int64_t la, int64_t lb) {  // merge buf[0, la) with buf[la, la+lb) into the other buffer
    std::vector<MergeJob> jobs{MergeJob{0, la, lb, 0, buf, 0}};
    run_merges(jobs, ceil_div<int64_t>(la + lb, kMergeNV), 2 * (la + lb) * kw);
  }

  // true: sorted; false: not a few-outlier input -- keys then hold a
  // permutation of the input and the caller partitions them.  Round k
  // compacts the remainder of round k-1 into the other buffer (kept first,
  // its outliers after them, the older outliers copied behind), until the
  // remainder is sorted (usually one or two rounds) or kOutlierRounds.
  static constexpr int kOutlierRounds = 4;
  bool run_outlier() {
    if (HAS_V) return false;
    ensure_ws();
    static const bool dbg = getenv("SR_OUTLIER_DEBUG") != nullptr;
    K* buf[2] = {keys, wk};
    int cur = 0;        // buffer holding the current remainder [0, r) and outliers [r, n)
    int64_t r = n;
    for (int round = 1; round <= kOutlierRounds; round++) {
      const int dst = 1 - cur;
      auto res = outlier_round(buf[cur], r, buf[dst]);
      if (r < n) {  // older outliers follow the new ones
        std::vector<CopyJob> cj{{r, n - r, 0, dst == 0 ? 1 : 0, 0}};
        run_copies(cj, ceil_div<int64_t>(n - r, 256 * 8), 2 * (n - r) * kw);
      }
      if (dbg)
        fprintf(stderr, "[sr_outlier] n=%lld round %d: kept %lld of %lld, descents among kept %lld\n", (long long)n,
                round, (long long)res.first, (long long)r, (long long)res.second);
      r = res.first;
      cur = dst;
      c.plan.levels = round;
      if (res.second == 0) {
        sort_nested(buf[cur] + r, n - r);
        merge_two(cur, r, n - r);  // -> the other buffer
        if (cur == 0) {            // merged into the workspace: copy back
          std::vector<CopyJob> cj{{0, n, 0, 1, 0}};
          run_copies(cj, ceil_div<int64_t>(n, 256 * 8), 2 * n * kw);
        }
        return true;
      }
      if (8 * (n - r) > n) break;  // too many outliers: not a nearly sorted input
    }
    if (cur == 1) {  // the permutation is in the workspace
      std::vector<CopyJob> cj{{0, n, 0, 1, 0}};
      run_copies(cj, ceil_div<int64_t>(n, 256 * 8), 2 * n * kw);
    }
    return false;
  }

  // partition of keys driven by the host (no speculative level 1)
  void partition_host(int64_t T) {
    c.plan.route = SR_ROUTE_PARTITION;
    c.plan.levels = 1;
    Level L1;
    std::vector<OvfSeg> whole{{0, n}};
    level_alloc(L1, whole, T, 0);
    level_splitters(L1);
    level_count(L1);
    level_scan_plan(L1);
    DevStats ls = *reinterpret_cast<DevStats*>(c.readback(L1.d_st, sizeof(DevStats)));
    std::vector<OvfSeg> next;
    if (ls.n_ovf > 0) {
      const OvfSeg* o = reinterpret_cast<const OvfSeg*>(c.readback(L1.d_ovf, sizeof(OvfSeg) * ls.n_ovf));
      next.assign(o, o + ls.n_ovf);
    }
    level_scatter(L1, &ls);
    level_finish(L1, &ls);
    run_levels(next, 1);
  }

  // ---- top level
  // Everything up to the first statistics readback is enqueued without a host
  // round trip: the presortedness scan (fused with the level-1 histogram), the
  // device-side route decision, the level-1 plan, and the kernels of the
  // SORTED / REVERSED / TILE / single-level PARTITION routes as speculative
  // launches that return at once unless the device route selects them.
  void run() {
    c.plan.n = n;
    if (resident_ok()) {
      run_resident();
      return;
    }
    const int force = forced();
    const int64_t T = choose_tile(n);
    const int64_t G = ceil_div<int64_t>(n, T);
    const bool part = n > kCap;
    {  // one allocation for everything up to the first readback (+ workspace)
      const int64_t bins = 2 * (int64_t)choose_buckets(n) + 1;
      auto r = [](int64_t b) { return (b + 255) & ~int64_t(255); };
      int64_t b = r(n * kw) + r(n * vw) + r(G * 32) + 2 * r((G + 1) * 32) + r(64) + r(G * 4) +
                  r(kMaxBuckets * kw) + r(kMaxBuckets) + r(4) + (HAS_V ? r(bins * G * 4) : 0) +
                  r(sizeof(DevStats) + 256 + 8 * ceil_div<int64_t>(bins * G, kScanNT * kScanIPT) + 4 * bins) +
                  r(4 * bins) + r(24 * (bins + n / kFillChunk + 2)) + r(24 * bins) + r(16 * bins) + r(2 * n) +
                  r(kMaxSample * (kw + 4)) + r(G * (int64_t)sizeof(TileMM)) + 8 * 256;
      c.reserve((size_t)b);
    }
    // Large n: the level-1 histogram rides on the presortedness read (one HBM
    // pass saved), so the splitters come first.  L2-resident n: the route is
    // decided first and every partition kernel is gated on it, so sorted and
    // reversed inputs pay for nothing but the scan.
    const bool fused = part && n > kFuseMin;
    Level L1;
    if (part) {
      std::vector<OvfSeg> whole{{0, n}};
      level_alloc(L1, whole, T, 0);
      if (fused) level_splitters(L1);
    }
    TileSummary* d_sums = c.alloc<TileSummary>(G);
    TileMM* d_mm = HAS_V ? nullptr : c.alloc<TileMM>(G);
    RunDesc* d_asc = c.alloc<RunDesc>(G + 1);
    RunDesc* d_desc = c.alloc<RunDesc>(G + 1);
    DevStats* d_pst = part ? L1.d_st : c.alloc<DevStats>(1);
    if (!part) c.memset0(d_pst, sizeof(DevStats));
    const K* kk = keys;
    const int nbins1 = part ? L1.segs[0].nbins : 0;
    const size_t csmem = sizeof(ClassifySmem<K>);
    if (fused) {
      set_smem(k_presort_scan<K, true, true, kScanNT1>, csmem);
      set_smem(k_presort_scan<K, false, true, kScanNT1>, csmem);
    }
    c.launch("presort_scan", n * kw + (fused ? (int64_t)nbins1 * G * 4 : 0), [&] {
      if (fused) {
        if (HAS_V)
          k_presort_scan<K, true, true, kScanNT1><<<(unsigned)G, kScanNT1, csmem, c.st>>>(
              kk, n, (int)T, d_sums, L1.d_spl, L1.d_eq, L1.d_m, L1.d_mat, nbins1, (int)G, L1.d_tot, L1.d_bins, nullptr);
        else
          k_presort_scan<K, false, true, kScanNT1><<<(unsigned)G, kScanNT1, csmem, c.st>>>(
              kk, n, (int)T, d_sums, L1.d_spl, L1.d_eq, L1.d_m, L1.d_mat, nbins1, (int)G, L1.d_tot, L1.d_bins, d_mm);
      } else {
        if (HAS_V)
          k_presort_scan<K, true, false, kScanNT1><<<(unsigned)G, kScanNT1, 0, c.st>>>(
              kk, n, (int)T, d_sums, nullptr, nullptr, nullptr, nullptr, 0, (int)G, nullptr, nullptr, nullptr);
        else
          k_presort_scan<K, false, false, kScanNT1><<<(unsigned)G, kScanNT1, 0, c.st>>>(
              kk, n, (int)T, d_sums, nullptr, nullptr, nullptr, nullptr, 0, (int)G, nullptr, nullptr, d_mm);
      }
    });
    const int merge_ok = route_ok();
    c.launch("presort_resolve", G * (int64_t)sizeof(TileSummary), [&] {
      k_presort_resolve<K, 1024><<<1, 1024, 0, c.st>>>(kk, n, d_sums, (int)G, T, d_asc, d_desc, d_pst, force, merge_ok,
                                                       d_mm);
    });
    // speculative route kernels
    int h_rev = -1, h_tile = -1, h_scat = -1, h_fin = -1, h_count = -1;
    if (force == 0) h_rev = reverse_ranges({RunDesc{0, n, 0, 0}}, d_pst);
    if (!part) {
      std::vector<Item> one{Item{0, 0, (int32_t)n, kItemSort}};
      Item* d_items = c.alloc<Item>(1);
      int64_t* d_cnt = c.alloc<int64_t>(1);
      std::vector<int64_t> cnt{1};
      c.upload(d_items, one);
      c.upload(d_cnt, cnt);
      h_tile = finish(d_items, d_cnt, 0, 1, 2 * n * (kw + vw), d_pst, kRouteTile);
    } else {
      if (!fused) {
        level_splitters(L1, d_pst);
        h_count = (int)c.launched.size();
        level_count(L1, d_pst);
      }
      level_scan_plan(L1, d_pst);
      ensure_ws();
      h_scat = level_scatter(L1, nullptr);
      h_fin = level_finish(L1, nullptr);
    }
    DevStats hs = *reinterpret_cast<DevStats*>(c.readback(d_pst, sizeof(DevStats)));
    c.plan.descents = hs.descents;
    c.plan.asc_breaks = hs.asc_breaks;
    c.plan.long_runs = hs.n_asc_runs + hs.n_desc_runs;
    if (hs.error) fail(SR_ERR_INTERNAL, "plan kernel inconsistency");
    const int64_t route = hs.route;
    if (route != kRouteReversed) c.unplan(h_rev);
    if (route != kRoutePartition) c.unplan(h_count);
    if (route != kRouteTile) c.unplan(h_tile);
    if (route != kRoutePartition || (!HAS_V && hs.noneq_total == 0)) c.unplan(h_scat);
    if (route != kRoutePartition) { c.unplan(h_fin); c.unplan(h_fin_big); }
    if (part && route == kRoutePartition) {  // fix the finish bytes to the real item mix
      c.replan(h_fin, 2 * (hs.noneq_total - hs.ovf_keys - hs.big_keys) * (kw + vw) + hs.eq_keys * kw +
                          2 * hs.eq_keys * vw);
      c.replan(h_fin_big, 2 * hs.big_keys * (kw + vw));
      c.replan(h_scat, (!HAS_V && hs.noneq_total == 0) ? 0
                                                        : n * (kw + vw) + 2 * n + hs.noneq_total * kw + (HAS_V ? n * vw : 0));
      c.plan.equal_keys += hs.eq_keys;
    }
    switch (route) {
      case kRouteSorted:  // is_sorted exit
        c.plan.route = SR_ROUTE_SORTED;
        return;
      case kRouteReversed:  // one descending run (strict for pairs), reversed
        c.plan.route = SR_ROUTE_REVERSED;
        c.plan.desc_runs_reversed = 1;
        return;
      case kRouteTile:
        c.plan.route = SR_ROUTE_TILE;
        return;
      case kRouteDistance:
        run_distance();
        return;
      default:
        break;
    }
    if (route == kRouteOutlier) {
      c.plan.route = SR_ROUTE_OUTLIER;
      if (run_outlier()) return;
      partition_host(T);  // not a few-outlier input: keys hold a permutation
      return;
    }
    bool use_merge = route == kRouteMerge;
    std::vector<Seg> segs;
    if (route == kRouteMerge || route == kRouteUndecided) {
      // MERGE vs PARTITION by planned bytes over the natural runs
      std::vector<RunDesc> asc, desc;
      if (hs.n_asc_runs) {
        const RunDesc* h = reinterpret_cast<const RunDesc*>(c.readback(d_asc, sizeof(RunDesc) * hs.n_asc_runs));
        asc.assign(h, h + hs.n_asc_runs);
      }
      if (hs.n_desc_runs) {
        const RunDesc* h = reinterpret_cast<const RunDesc*>(c.readback(d_desc, sizeof(RunDesc) * hs.n_desc_runs));
        desc.assign(h, h + hs.n_desc_runs);
      }
      segs = build_segments(asc, desc);
      if (!use_merge) {
        int64_t mb = merge_route_bytes(segs);
        int64_t N = n * (kw + vw);
        int64_t pb = 4 * N + (n > 4 * 1024 * 1024 ? 3 * N : 0);
        use_merge = mb < pb;
      }
    }
    if (use_merge) {
      c.plan.route = SR_ROUTE_MERGE;
      run_merge_route(segs);
      return;
    }
    // PARTITION (level 1 already enqueued unless the route was undecided)
    c.plan.route = SR_ROUTE_PARTITION;
    c.plan.levels = 1;
    if (!part) fail(SR_ERR_INTERNAL, "partition route without level 1");
    std::vector<OvfSeg> next;
    if (hs.n_ovf > 0) {
      const OvfSeg* h = reinterpret_cast<const OvfSeg*>(c.readback(L1.d_ovf, sizeof(OvfSeg) * hs.n_ovf));
      next.assign(h, h + hs.n_ovf);
    }
    if (route == kRouteUndecided) {  // the speculative level-1 kernels were gated off
      if (!fused) {
        level_splitters(L1);
        level_count(L1);
      }
      level_scan_plan(L1);
      hs = *reinterpret_cast<DevStats*>(c.readback(L1.d_st, sizeof(DevStats)));
      next.clear();
      if (hs.n_ovf > 0) {
        const OvfSeg* h = reinterpret_cast<const OvfSeg*>(c.readback(L1.d_ovf, sizeof(OvfSeg) * hs.n_ovf));
        next.assign(h, h + hs.n_ovf);
      }
      level_scatter(L1, &hs);
      level_finish(L1, &hs);
    }
    run_levels(next, 1);
  }
};

// ------------------------------------------------------------------ validation
// Device (or managed) memory; *dev receives the device that owns it.
bool is_device_ptr(const void* p, int* dev = nullptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  if (dev) *dev = a.device;
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Makes the device that owns the caller's buffers current for one call (the
// caller's stream must belong to it) and restores the previous device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = 0;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
    cudaGetLastError();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool dtype_ok(int32_t dtype) { return dtype == SR_INT32 || dtype == SR_INT64 || dtype == SR_FLOAT32 || dtype == SR_FLOAT64; }
int64_t key_bytes(int32_t dtype) { return (dtype == SR_INT32 || dtype == SR_FLOAT32) ? 4 : 8; }

int32_t validate(const void* keys, const void* vals, int64_t n, int32_t dtype, bool pairs, int* dev = nullptr) {
  if (n < 0) return SR_ERR_INVALID_ARGUMENT;
  if (!dtype_ok(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (n > INT32_MAX) return SR_ERR_SIZE;
  if (n <= 1) return SR_OK;
  const int64_t kw = key_bytes(dtype);
  if (!keys || (pairs && !vals)) return SR_ERR_INVALID_ARGUMENT;
  if ((uintptr_t)keys % kw) return SR_ERR_ALIGNMENT;
  if (pairs && (uintptr_t)vals % 4) return SR_ERR_ALIGNMENT;
  int dk = -1, dv = -1;
  if (!is_device_ptr(keys, &dk) || (pairs && !is_device_ptr(vals, &dv))) return SR_ERR_INVALID_ARGUMENT;
  if (pairs && dk != dv) return SR_ERR_INVALID_ARGUMENT;
  if (dev) *dev = dk;
  if (pairs) {
    uintptr_t k0 = (uintptr_t)keys, k1 = k0 + n * kw, v0 = (uintptr_t)vals, v1 = v0 + n * 4;
    if (k0 < v1 && v0 < k1) return SR_ERR_INVALID_ARGUMENT;
  }
  return SR_OK;
}

template <typename F>
int32_t guarded(F&& f) {
  t_state.err.clear();
  try {
    f();
    return SR_OK;
  } catch (const SrError& e) {
    t_state.err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    t_state.err = "host allocation failed";
    return SR_ERR_OUT_OF_MEMORY;
  } catch (...) {
    t_state.err = "unknown internal error";
    return SR_ERR_INTERNAL;
  }
}

int32_t sort_impl(void* keys, void* vals, int64_t n, int32_t dtype, void* stream, bool pairs) {
  t_call0 = std::chrono::steady_clock::now();
  int dev = -1;
  int32_t v = validate(keys, vals, n, dtype, pairs, &dev);
  hostprof("validated");
  if (v != SR_OK) {
    t_state.err = sr_status_string(v);
    return v;
  }
  DeviceGuard dg(dev);
  return guarded([&] {
    Ctx c((cudaStream_t)stream);
    c.plan.n = n;
    if (n <= 1) return;
    init_pool();
    // floating-point keys: totalOrder -> signed integer order, in place, and
    // back after the integer sort (fkeys.cuh)
    const bool fl = dtype == SR_FLOAT32 || dtype == SR_FLOAT64;
    const bool w4 = key_bytes(dtype) == 4;
    auto flip = [&]() {
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n, 256 * 4)));
      c.launch("fkey_flip", 2 * n * key_bytes(dtype), [&] {
        if (w4) k_fkey_flip<int32_t><<<grid, 256, 0, c.st>>>((int32_t*)keys, n);
        else k_fkey_flip<int64_t><<<grid, 256, 0, c.st>>>((int64_t*)keys, n);
      });
    };
    if (fl) flip();
    try {
      if (w4) {
        if (pairs) Sorter<int32_t, true>(c, (int32_t*)keys, (uint32_t*)vals, n).run();
        else Sorter<int32_t, false>(c, (int32_t*)keys, nullptr, n).run();
      } else {
        if (pairs) Sorter<int64_t, true>(c, (int64_t*)keys, (uint32_t*)vals, n).run();
        else Sorter<int64_t, false>(c, (int64_t*)keys, nullptr, n).run();
      }
    } catch (const SrError& e) {
      // The integer sort failed.  Before any data-moving kernel (out of memory
      // while reserving the workspace, the usual case) the keys hold exactly
      // their integer images, and the involution restores the caller's bits;
      // after one they hold a permutation of the images, restored to a
      // permutation of the caller's keys.  A sticky CUDA error leaves the
      // contents unspecified (include/sr_sort.h).
      if (fl && e.code != SR_ERR_CUDA) {
        cudaGetLastError();
        try { flip(); } catch (...) {}
      }
      throw;
    }
    if (fl) {  // the integer sort's launches count in the plan; the flips are added
      const int launches = c.plan.launches;
      flip();
      c.plan.launches = launches + 1;
    }
  });
}

// Record keys (records.cuh): lexicographic sort of n records of `words` int32
// by index refinement rounds of the stable int64 pair sort, then a gather.
void sort_records_impl(int32_t* recs, int64_t n, int words, cudaStream_t st) {
  Ctx c(st);
  c.plan.n = n;
  init_pool();
  int64_t* kA = c.alloc<int64_t>(n);
  int64_t* kB = c.alloc<int64_t>(n);
  uint32_t* idx = c.alloc<uint32_t>(n);
  uint32_t* flag = c.alloc<uint32_t>(n);
  const int64_t tiles = ceil_div<int64_t>(n, kScanNT * kScanIPT);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n, 256)));
  // word ranges (one readback): field widths of the packed keys
  std::vector<int32_t> mm0(2 * (size_t)words);
  for (int j = 0; j < words; j++) {
    mm0[2 * j] = INT32_MAX;
    mm0[2 * j + 1] = INT32_MIN;
  }
  int32_t* d_mm = c.alloc<int32_t>(2 * (int64_t)words);
  c.upload(d_mm, mm0);
  {
    const int bs = words <= 256 ? (256 / words) * words : words;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n * words, bs)));
    c.launch("rec_minmax", n * (int64_t)words * 4, [&] { k_rec_minmax<<<g, bs, 0, c.st>>>(recs, n, words, d_mm); });
  }
  const int32_t* hmm = reinterpret_cast<const int32_t*>(c.readback(d_mm, 8 * (size_t)words));
  std::vector<int> wl, wb;
  std::vector<int32_t> wmin;
  for (int j = 0; j < words; j++) {
    const uint32_t range = (uint32_t)hmm[2 * j + 1] - (uint32_t)hmm[2 * j];
    if (range == 0) continue;  // constant word: never decides
    wl.push_back(j);
    wmin.push_back(hmm[2 * j]);
    wb.push_back(32 - __builtin_clz(range));
  }
  int launches = 0, rounds = 0;
  size_t pos = 0;
  int seg_bits = 0;
  uint32_t* ex = nullptr;  // rounds >= 1: exclusive scan of the boundary flags
  while (pos < wl.size()) {
    RecRound rr{};
    rr.seg_bits = seg_bits;
    int used = seg_bits;
    while (pos < wl.size() && rr.nw < 64 && used + wb[pos] <= 64) {
      rr.wl[rr.nw] = wl[pos];
      rr.wmin[rr.nw] = wmin[pos];
      rr.wbits[rr.nw] = wb[pos];
      used += wb[pos];
      rr.nw++;
      pos++;
    }
    rr.shift = 64 - used;
    int64_t* kin = kA;
    int64_t* kout = ex ? kB : kA;
    c.launch("rec_key", n * (4 * (int64_t)rr.nw + 12), [&] {
      k_rec_key<<<grid, 256, 0, c.st>>>(recs, n, words, rr, ex, kin, kout, idx);
    });
    if (ex) std::swap(kA, kB);
    {  // stable pair sort of (key, idx) on the integer path
      Ctx sc(st);
      Sorter<int64_t, true>(sc, kA, idx, n).run();
      launches += sc.plan.launches;
    }
    rounds++;
    if (pos >= wl.size()) break;
    // control: tie flag + boundary count | scan status (zeroed)
    unsigned char* ctrl = c.alloc<unsigned char>(256 + 8 * tiles);
    c.memset0(ctrl, 256 + 8 * tiles);
    uint32_t* ctl = reinterpret_cast<uint32_t*>(ctrl);
    int* tile_counter = reinterpret_cast<int*>(ctrl + 128);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(ctrl + 256);
    c.launch("rec_flags", n * 12, [&] { k_rec_flags<<<grid, 256, 0, c.st>>>(kA, n, flag, ctl); });
    const uint32_t* h = reinterpret_cast<const uint32_t*>(c.readback(ctl, 8));
    if (!h[0]) break;  // every record is already in place
    seg_bits = h[1] ? 32 - __builtin_clz(h[1]) : 0;  // segment ids 0 .. boundaries
    c.launch("scan", n * 8, [&] {
      k_scan_u32<kScanNT, kScanIPT><<<(unsigned)tiles, kScanNT, 0, c.st>>>(flag, n, status, tile_counter, nullptr);
    });
    ex = flag;
  }
  if (rounds == 0) {  // every word constant: all records equal, input order kept
    c.plan.levels = 0;
    c.plan.route = SR_ROUTE_SORTED;
    return;
  }
  int32_t* out = c.alloc<int32_t>(n * (int64_t)words);
  c.launch("rec_gather", 2 * n * (int64_t)words * 4, [&] {
    k_rec_gather<<<148 * 8, 256, 0, c.st>>>(recs, n, words, idx, out);
  });
  check_cuda(cudaMemcpyAsync(recs, out, (size_t)n * words * 4, cudaMemcpyDeviceToDevice, c.st), "record copy");
  c.plan.levels = rounds;
  c.plan.launches += launches;
  c.plan.route = SR_ROUTE_PARTITION;
}

// Presortedness measures (measures.cuh): Run and Mono from the keys, Dis /
// misplaced from the stable pair sort of (key copy, index), Inv by counting
// merge levels over that permutation.
template <typename K>
void measures_impl(const K* keys, int64_t n, sr_measures* out, cudaStream_t st) {
  Ctx c(st);
  c.plan.n = n;
  init_pool();
  constexpr int NT = 256;
  const int64_t chunk = (int64_t)NT * 64;
  const int G = (int)std::max<int64_t>(1, ceil_div<int64_t>(n - 1, chunk));
  K* kc = c.alloc<K>(n);
  uint32_t* idx = c.alloc<uint32_t>(n);
  uint32_t* idx2 = c.alloc<uint32_t>(n);
  MonoMap* maps = c.alloc<MonoMap>(G);
  unsigned long long* cnt = c.alloc<unsigned long long>(8);  // descents, pieces, maxdis, misplaced, inv
  c.memset0(cnt, 8 * sizeof(unsigned long long));
  c.launch("mono_map", n * (int64_t)sizeof(K), [&] { k_mono_map<K, NT><<<G, NT, 0, c.st>>>(keys, n, chunk, maps, cnt); });
  c.launch("mono_final", G * (int64_t)sizeof(MonoMap), [&] { k_mono_final<<<1, 32, 0, c.st>>>(maps, G, cnt + 1); });
  check_cuda(cudaMemcpyAsync(kc, keys, n * sizeof(K), cudaMemcpyDeviceToDevice, c.st), "key copy");
  {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n, NT)));
    c.launch("iota", n * 4, [&] { k_iota<<<grid, NT, 0, c.st>>>(idx, n); });
  }
  {  // stable ranks
    Ctx sc(st);
    Sorter<K, true>(sc, kc, idx, n).run();
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(n, NT)));
  c.launch("dis", n * 4, [&] { k_dis<NT><<<grid, NT, 0, c.st>>>(idx, n, cnt + 2, cnt + 3); });
  uint32_t* a = idx;
  uint32_t* b = idx2;
  for (int64_t R = 1; R < n; R *= 2) {
    c.launch("inv_level", n * 8, [&] { k_inv_level<NT><<<grid, NT, 0, c.st>>>(a, b, n, R, cnt + 4); });
    std::swap(a, b);
  }
  const unsigned long long* h = reinterpret_cast<const unsigned long long*>(c.readback(cnt, 8 * sizeof(unsigned long long)));
  out->n = n;
  out->runs = (int64_t)h[0] + 1;
  out->mono = (int64_t)h[1];
  out->max_dis = (int64_t)h[2];
  out->misplaced = (int64_t)h[3];
  out->inversions = (int64_t)h[4];
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int32_t sr_sort_keys(void* keys, int64_t n, int32_t dtype, void* stream) {
  return sort_impl(keys, nullptr, n, dtype, stream, false);
}

int32_t sr_sort_pairs(void* keys, void* vals, int64_t n, int32_t dtype, void* stream) {
  return sort_impl(keys, vals, n, dtype, stream, true);
}

int32_t sr_sort_host(void* host_keys, void* host_vals, int64_t n, int32_t dtype, void* stream) {
  if (n < 0) return SR_ERR_INVALID_ARGUMENT;
  if (!dtype_ok(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (n > INT32_MAX) return SR_ERR_SIZE;
  if (n <= 1) return SR_OK;
  if (!host_keys) return SR_ERR_INVALID_ARGUMENT;
  const int64_t kw = key_bytes(dtype);
  cudaStream_t st = (cudaStream_t)stream;
  void *dk = nullptr, *dv = nullptr;
  int32_t rc = guarded([&] {
    check_cuda(cudaMallocAsync(&dk, n * kw, st), "cudaMallocAsync");
    if (host_vals) check_cuda(cudaMallocAsync(&dv, n * 4, st), "cudaMallocAsync");
    check_cuda(cudaMemcpyAsync(dk, host_keys, n * kw, cudaMemcpyHostToDevice, st), "h2d");
    if (host_vals) check_cuda(cudaMemcpyAsync(dv, host_vals, n * 4, cudaMemcpyHostToDevice, st), "h2d");
  });
  if (rc == SR_OK) rc = host_vals ? sr_sort_pairs(dk, dv, n, dtype, stream) : sr_sort_keys(dk, n, dtype, stream);
  if (rc == SR_OK) {
    rc = guarded([&] {
      check_cuda(cudaMemcpyAsync(host_keys, dk, n * kw, cudaMemcpyDeviceToHost, st), "d2h");
      if (host_vals) check_cuda(cudaMemcpyAsync(host_vals, dv, n * 4, cudaMemcpyDeviceToHost, st), "d2h");
    });
  }
  if (dk) cudaFreeAsync(dk, st);
  if (dv) cudaFreeAsync(dv, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (rc == SR_OK && e != cudaSuccess) {
    t_state.err = cudaGetErrorString(e);
    rc = SR_ERR_CUDA;
  }
  return rc;
}

int32_t sr_sort_host_batch(void* const* host_keys, void* const* host_vals, const int64_t* n, int32_t count,
                           int32_t dtype, void* stream) {
  t_state.err.clear();
  if (count < 0 || (count > 0 && (!host_keys || !n))) return SR_ERR_INVALID_ARGUMENT;
  if (!dtype_ok(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  int64_t nmax = 0;
  for (int i = 0; i < count; ++i) {
    if (n[i] < 0 || (n[i] >= 2 && !host_keys[i])) return SR_ERR_INVALID_ARGUMENT;
    if (n[i] > INT32_MAX) return SR_ERR_SIZE;
    nmax = std::max(nmax, n[i]);
  }
  if (nmax <= 1) return SR_OK;
  const int64_t kw = key_bytes(dtype);
  cudaStream_t st = (cudaStream_t)stream;
  // ring of R device buffers: instance i lives in slot i % R from its upload to the end of its download
  constexpr int kRing = 4;
  const int R = std::min<int>(count, kRing);
  void *dk[kRing] = {}, *dv[kRing] = {};
  std::vector<cudaEvent_t> up(count, nullptr), sorted(count, nullptr), down(count, nullptr);
  bool pairs = false;
  for (int i = 0; host_vals && i < count; ++i) pairs = pairs || (host_vals[i] && n[i] >= 2);
  int next_up = 0;  // instances [0, next_up) have their upload enqueued
  cudaStream_t sh = nullptr, sd = nullptr;
  int32_t rc = guarded([&] {
    DevState& ds = t_state.ds();
    if (!ds.batch_h2d) check_cuda(cudaStreamCreateWithFlags(&ds.batch_h2d, cudaStreamNonBlocking), "stream");
    if (!ds.batch_d2h) check_cuda(cudaStreamCreateWithFlags(&ds.batch_d2h, cudaStreamNonBlocking), "stream");
    sh = ds.batch_h2d;
    sd = ds.batch_d2h;
    for (int i = 0; i < count; ++i) {
      check_cuda(cudaEventCreateWithFlags(&up[i], cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&sorted[i], cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&down[i], cudaEventDisableTiming), "event");
    }
    for (int r = 0; r < R; ++r) {
      check_cuda(cudaMallocAsync(&dk[r], nmax * kw, st), "cudaMallocAsync");
      if (pairs) check_cuda(cudaMallocAsync(&dv[r], nmax * 4, st), "cudaMallocAsync");
    }
    // the copy streams start after the buffers exist and after the caller's earlier work on `stream`
    check_cuda(cudaEventRecord(sorted[0], st), "record");
    check_cuda(cudaStreamWaitEvent(sh, sorted[0], 0), "wait");
  });
  auto upload_through = [&](int last) {  // enqueue the uploads of instances next_up .. last
    for (; next_up <= last && next_up < count; ++next_up) {
      const int j = next_up, r = j % R;
      if (j >= R) check_cuda(cudaStreamWaitEvent(sh, down[j - R], 0), "wait");  // slot free again
      if (n[j] >= 2) {
        check_cuda(cudaMemcpyAsync(dk[r], host_keys[j], n[j] * kw, cudaMemcpyHostToDevice, sh), "h2d");
        if (host_vals && host_vals[j])
          check_cuda(cudaMemcpyAsync(dv[r], host_vals[j], n[j] * 4, cudaMemcpyHostToDevice, sh), "h2d");
      }
      check_cuda(cudaEventRecord(up[j], sh), "record");
    }
  };
  for (int i = 0; rc == SR_OK && i < count; ++i) {
    const int r = i % R;
    // uploads run ahead of the sorts as far as the ring allows: the download of instance i - 1 is
    // already enqueued, so slot (i + R - 1) % R has its release event
    rc = guarded([&] {
      upload_through(i + R - 1);
      check_cuda(cudaStreamWaitEvent(st, up[i], 0), "wait");
    });
    if (rc != SR_OK) break;
    const bool has_v = host_vals && host_vals[i];
    if (n[i] >= 2) rc = has_v ? sr_sort_pairs(dk[r], dv[r], n[i], dtype, stream) : sr_sort_keys(dk[r], n[i], dtype, stream);
    if (rc != SR_OK) break;
    rc = guarded([&] {
      check_cuda(cudaEventRecord(sorted[i], st), "record");
      check_cuda(cudaStreamWaitEvent(sd, sorted[i], 0), "wait");
      if (n[i] >= 2) {
        check_cuda(cudaMemcpyAsync(host_keys[i], dk[r], n[i] * kw, cudaMemcpyDeviceToHost, sd), "d2h");
        if (has_v) check_cuda(cudaMemcpyAsync(host_vals[i], dv[r], n[i] * 4, cudaMemcpyDeviceToHost, sd), "d2h");
      }
      check_cuda(cudaEventRecord(down[i], sd), "record");
    });
  }
  // drain both copy streams into the caller's stream, release the ring, synchronise
  const std::string err = t_state.err;
  if (sh && sd) {
    cudaEvent_t tail = up.empty() ? nullptr : up[0];
    if (tail && cudaEventRecord(tail, sh) == cudaSuccess) cudaStreamWaitEvent(st, tail, 0);
    tail = sorted.empty() ? nullptr : sorted[0];
    if (tail && cudaEventRecord(tail, sd) == cudaSuccess) cudaStreamWaitEvent(st, tail, 0);
  }
  for (int r = 0; r < kRing; ++r) {
    if (dk[r]) cudaFreeAsync(dk[r], st);
    if (dv[r]) cudaFreeAsync(dv[r], st);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  for (int i = 0; i < count; ++i) {
    if (up[i]) cudaEventDestroy(up[i]);
    if (sorted[i]) cudaEventDestroy(sorted[i]);
    if (down[i]) cudaEventDestroy(down[i]);
  }
  if (rc != SR_OK) {
    t_state.err = err;
  } else if (e != cudaSuccess) {
    t_state.err = cudaGetErrorString(e);
    rc = SR_ERR_CUDA;
  }
  return rc;
}

int32_t sr_sort_records(void* recs, int64_t n, int32_t words, void* stream) {
  t_state.err.clear();
  if (n < 0 || words < 1 || words > 1024) return SR_ERR_INVALID_ARGUMENT;
  if (n > INT32_MAX || n * (int64_t)words > (int64_t(1) << 40)) return SR_ERR_SIZE;
  if (n <= 1) return SR_OK;
  if (!recs || !is_device_ptr(recs)) return SR_ERR_INVALID_ARGUMENT;
  if ((uintptr_t)recs % 4) return SR_ERR_ALIGNMENT;
  return guarded([&] { sort_records_impl((int32_t*)recs, n, words, (cudaStream_t)stream); });
}

int32_t sr_presortedness(const void* keys, int64_t n, int32_t dtype, sr_measures* host_out, void* stream) {
  t_state.err.clear();
  if (!host_out || n < 0) return SR_ERR_INVALID_ARGUMENT;
  if (dtype != SR_INT32 && dtype != SR_INT64) return SR_ERR_UNSUPPORTED_DTYPE;
  if (n > INT32_MAX) return SR_ERR_SIZE;
  *host_out = sr_measures{};
  host_out->n = n;
  if (n == 0) return SR_OK;
  if (n == 1) {
    host_out->runs = host_out->mono = 1;
    return SR_OK;
  }
  if (!keys || !is_device_ptr(keys)) return SR_ERR_INVALID_ARGUMENT;
  if ((uintptr_t)keys % key_bytes(dtype)) return SR_ERR_ALIGNMENT;
  return guarded([&] {
    if (dtype == SR_INT32) measures_impl<int32_t>((const int32_t*)keys, n, host_out, (cudaStream_t)stream);
    else measures_impl<int64_t>((const int64_t*)keys, n, host_out, (cudaStream_t)stream);
  });
}

int32_t sr_generate(void* out, int64_t n, int32_t dtype, int32_t order, uint64_t seed, int64_t param, void* stream) {
  t_state.err.clear();
  if (n < 0 || order < SR_GEN_RANDOM || order > SR_GEN_EXTREMES) return SR_ERR_INVALID_ARGUMENT;
  if (dtype != SR_INT32 && dtype != SR_INT64) return SR_ERR_UNSUPPORTED_DTYPE;
  if (n == 0) return SR_OK;
  if (!out) return SR_ERR_INVALID_ARGUMENT;
  int dev = -1;
  if (!is_device_ptr(out, &dev)) return SR_ERR_INVALID_ARGUMENT;
  if ((uintptr_t)out % key_bytes(dtype)) return SR_ERR_ALIGNMENT;
  const bool needs_k = order == SR_GEN_SWAPS || order == SR_GEN_LAST || order == SR_GEN_DISTANCE;
  const bool needs_pos = order == SR_GEN_FEW_UNIQUE || order == SR_GEN_RUNS || order == SR_GEN_SHARP_TEETH ||
                         order == SR_GEN_EQUAL_TEETH || order == SR_GEN_EVEN_TEETH;
  if ((needs_k && (param < 0 || (order == SR_GEN_LAST && param > n))) || (needs_pos && param < 1) ||
      (order == SR_GEN_FEW_UNIQUE && param > 65536) || (order == SR_GEN_RUNS && param > n && n > 0))
    return SR_ERR_INVALID_ARGUMENT;
  if (dtype == SR_INT32 && order == SR_GEN_ALL_EQUAL && (param < INT32_MIN || param > INT32_MAX))
    return SR_ERR_INVALID_ARGUMENT;
  DeviceGuard dg(dev);
  return guarded([&] {
    Ctx c((cudaStream_t)stream);
    init_pool();
    auto run = [&](auto* o) {
      using K = std::remove_pointer_t<decltype(o)>;
      K* table = nullptr;
      int64_t* perm = nullptr;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 16, ceil_div<int64_t>(n, 256)));
      if (order == SR_GEN_FEW_UNIQUE) {
        table = c.alloc<K>(param);
        c.launch("gen_table", param * (int64_t)sizeof(K), [&] { k_gen_table<K><<<1, 32, 0, c.st>>>(table, param, seed); });
      } else if (order == SR_GEN_EXTREMES) {
        const K mn = std::numeric_limits<K>::min(), mx = std::numeric_limits<K>::max();
        std::vector<K> t{mn, mx, 0, -1, 1, (K)(mn + 1), (K)(mx - 1)};
        table = c.alloc<K>(7);
        c.upload(table, t);
      } else if (order == SR_GEN_RUNS) {
        const int64_t nb = ceil_div<int64_t>(n, param);
        perm = c.alloc<int64_t>(nb + 1);
        c.launch("gen_perm", nb * 8, [&] { k_gen_perm<<<1, 32, 0, c.st>>>(perm, nb, seed); });
      }
      c.launch("gen_map", n * (int64_t)sizeof(K), [&] {
        k_gen_map<K><<<grid, 256, 0, c.st>>>(o, n, order, seed, param, table, perm);
      });
      if (order == SR_GEN_SWAPS && param > 0)
        c.launch("gen_swaps", 4 * param * (int64_t)sizeof(K), [&] { k_gen_swaps<K><<<1, 32, 0, c.st>>>(o, n, seed, param); });
      if (order == SR_GEN_DISTANCE && param > 0) {
        const int64_t nblocks = ceil_div<int64_t>(n, param + 1);
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(148 * 8, ceil_div<int64_t>(nblocks, 128)));
        c.launch("gen_distance", 2 * n * (int64_t)sizeof(K), [&] { k_gen_distance<K><<<g, 128, 0, c.st>>>(o, n, seed, param); });
      }
    };
    if (dtype == SR_INT32) run((int32_t*)out);
    else run((int64_t*)out);
  });
}

int32_t sr_last_plan(sr_plan* out) {
  if (!out) return SR_ERR_INVALID_ARGUMENT;
  *out = t_state.plan;
  return SR_OK;
}

const char* sr_status_string(int32_t s) {
  switch (s) {
    case SR_OK: return "ok";
    case SR_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SR_ERR_UNSUPPORTED_DTYPE: return "unsupported dtype";
    case SR_ERR_SIZE: return "size out of range";
    case SR_ERR_ALIGNMENT: return "misaligned pointer";
    case SR_ERR_OUT_OF_MEMORY: return "out of device memory";
    case SR_ERR_CUDA: return "CUDA error";
    case SR_ERR_INTERNAL: return "internal error";
    default: return "unknown status";
  }
}

const char* sr_last_error(void) { return t_state.err.c_str(); }

int32_t sr_set_option(int32_t key, int64_t value) {
  switch (key) {
    case SR_OPT_FORCE_ROUTE:
      if (value != 0 && value != SR_ROUTE_MERGE && value != SR_ROUTE_PARTITION && value != SR_ROUTE_OUTLIER)
        return SR_ERR_INVALID_ARGUMENT;
      g_force_route = (int)value;
      return SR_OK;
    case SR_OPT_PROFILE:
      g_profile = value ? 1 : 0;
      return SR_OK;
    case SR_OPT_MERGE_ROUTE:
      g_merge_route = value ? 1 : 0;
      return SR_OK;
    case SR_OPT_RESIDENT:
      g_resident = value ? 1 : 0;
      return SR_OK;
    case SR_OPT_OUTLIER_ROUTE:
      g_outlier = value ? 1 : 0;
      return SR_OK;
    case SR_OPT_DISTANCE_ROUTE:
      g_distance = value ? 1 : 0;
      return SR_OK;
    case SR_OPT_WS_LIMIT:
      if (value < 0) return SR_ERR_INVALID_ARGUMENT;
      g_ws_limit = value;
      return SR_OK;
    case SR_OPT_RESIDENT_CAP:
      if (value < 1 || value > 16384) return SR_ERR_INVALID_ARGUMENT;
      g_res_cap = (int)value;
      return SR_OK;
    default:
      if (key >= SR_OPT_TUNE && key < SR_OPT_TUNE + 8) {
        if (key == SR_OPT_TUNE + 1 && (value < 2 || value > kMaxBuckets || (value & (value - 1))))
          return SR_ERR_INVALID_ARGUMENT;
        if (key == SR_OPT_TUNE + 2 && (value < 16 || value > 4096)) return SR_ERR_INVALID_ARGUMENT;
        if (key == SR_OPT_TUNE + 3 && (value < 0 || value > kMaxBuckets || (value & (value - 1))))
          return SR_ERR_INVALID_ARGUMENT;
        g_tune[key - SR_OPT_TUNE] = value;
        return SR_OK;
      }
      return SR_ERR_INVALID_ARGUMENT;
  }
}

int32_t sr_last_profile(const char** names, float* ms, int64_t* bytes, int32_t cap) {
  ThreadState& ts = t_state;
  if (ts.prof.empty()) return 0;
  cudaStreamSynchronize(ts.prof_stream);
  int32_t k = 0;
  for (auto& e : ts.prof) {
    if (k < cap) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e.a, e.b);
      if (names) names[k] = e.name;
      if (ms) ms[k] = t;
      if (bytes) bytes[k] = e.bytes;
    }
    k++;
  }
  return k;
}

}  // extern "C"

#include "debug_api.cuh"
