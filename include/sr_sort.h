/*
 * sr_sort.h -- C ABI of libsr_sort.so, a B200 (sm_100a) adaptive comparison
 * sort after H. Zhang, B. Meng, Y. Liang, "Sort Race" (arXiv 1609.04471).
 * Citations "PAPER.md:N" refer to lines of that paper's text (§ / table /
 * appendix given alongside).
 *
 * All functions are extern "C"; no C++ exception crosses the ABI.  Every
 * pointer named keys / vals / out* is a DEVICE pointer (cudaMalloc, torch
 * tensor data_ptr, managed memory) unless the name says host_.  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  Sizes are
 * element counts.
 *
 * Problem statement: "comparison based, internal sorting" of large in-memory
 * arrays with the qsort interface sort(arr, n, es, cmp)
 * (Appendix A); the comparator is fixed to
 * ascending signed integer order, so `dtype` replaces es+cmp.
 *
 * Error behaviour (all entry points): arguments are validated before any
 * device work; on SR_ERR_INVALID_ARGUMENT / _UNSUPPORTED_DTYPE / _SIZE /
 * _ALIGNMENT the caller's buffers are untouched.  SR_ERR_OUT_OF_MEMORY from
 * the first workspace reservation (made before any kernel that moves data;
 * for float keys the in-place key map is undone) also leaves them untouched;
 * an allocation failure of a later partition level leaves them holding a
 * permutation of the input.  A CUDA failure after the first kernel returns
 * SR_ERR_CUDA, leaves the contents unspecified and puts the CUDA message in
 * sr_last_error().
 *
 * Devices: the call runs on the device that owns `keys` (made current for
 * the call and restored afterwards); `stream` must belong to that device.
 * Per-host-thread scratch is kept per device.
 */
#ifndef SR_SORT_H
#define SR_SORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Key dtype; values are 4-byte opaque payloads.  SR_INT32 / SR_INT64: signed
 * numeric order.  SR_FLOAT32 / SR_FLOAT64 (sr_sort_keys, sr_sort_pairs,
 * sr_sort_host only, the paper's "random double"
 * class): IEEE 754 totalOrder -- -NaN (larger payload first) <
 * -inf < negative < -0 < +0 < positive < +inf < +NaN (larger payload last);
 * keys equal in that order are bit-identical, so the output is unique.  The
 * float sort costs two extra in-place passes over the keys (fkeys.cuh). */
enum { SR_INT32 = 0, SR_INT64 = 1, SR_FLOAT32 = 2, SR_FLOAT64 = 3 };

enum {
  SR_OK = 0,
  SR_ERR_INVALID_ARGUMENT = 1, /* NULL with n >= 2, n < 0, host pointer, overlapping keys/vals */
  SR_ERR_UNSUPPORTED_DTYPE = 2,
  SR_ERR_SIZE = 3,             /* n > 2^31 - 1 */
  SR_ERR_ALIGNMENT = 4,        /* keys not aligned to the key size or vals to 4 bytes */
  SR_ERR_OUT_OF_MEMORY = 5,    /* workspace allocation failed (see "Error behaviour" above) */
  SR_ERR_CUDA = 6,
  SR_ERR_INTERNAL = 7          /* planner invariant violated (reported, never silent) */
};

/* Route chosen by the planner (H3).  PAPER.md:284: quicksort unless stability
 * or presortedness calls for mergesort. */
enum {
  SR_ROUTE_NONE = 0,      /* n <= 1 */
  SR_ROUTE_SORTED = 1,    /* D = 0: is_sorted exit, no write */
  SR_ROUTE_REVERSED = 2,  /* one descending run: reversal only */
  SR_ROUTE_MERGE = 3,     /* natural runs + merge levels (§3, Appendix A) */
  SR_ROUTE_PARTITION = 4, /* splitter partition with equality buckets (§4, Appendix B) */
  SR_ROUTE_TILE = 5,      /* n <= one CTA tile: tile sort only (PAPER.md:155 alpha cutoff) */
  SR_ROUTE_OUTLIER = 6,   /* keys only, few descents (k-exchange): descent endpoints extracted,
                             sorted, merged with the sorted remainder */
  SR_ROUTE_DISTANCE = 7   /* keys only, bounded displacement (k-distance): proven by the
                             presortedness scan (every key < 512 positions from its place); sorted
                             windows of 1024 keys, then merged windows offset by 512 */
};

/* ------------------------------------------------------------------ inputs */

/* On-device generator of the paper's input classes (§2, lines 56-87;
 * SURVEY.md §8(f) NEXT #4), bit-identical to workloads/gen.py for the same
 * seed.  out: device array of n keys (dtype SR_INT32 / SR_INT64), written on
 * `stream`.  order / param:
 *   SR_GEN_RANDOM      uniform over the full range (draw i, high 32 bits for int32)
 *   SR_GEN_SORTED      0..n-1                     SR_GEN_REVERSED  n-1..0
 *   SR_GEN_SWAPS       ramp + param random position swaps in draw order (k-exchange)
 *   SR_GEN_FEW_UNIQUE  param distinct uniform values (first param distinct draws),
 *                      a[i] = v[U[0,param)] from stream seed ^ 0xF00D (k-limited analogue)
 *   SR_GEN_RUNS        ramp cut into blocks of param, blocks Fisher-Yates shuffled (BASELINE configs[2])
 *   SR_GEN_LAST        ramp whose last param positions are uniform random (BASELINE configs[2])
 *   SR_GEN_SHARP_TEETH / _EQUAL_TEETH / _EVEN_TEETH  param sections
 *   SR_GEN_DISTANCE    ramp, blocks of param+1 each Fisher-Yates shuffled (k-distance)
 *   SR_GEN_ALL_EQUAL   every key = param         SR_GEN_EXTREMES  MIN/MAX/0/-1/1/MIN+1/MAX-1 mix
 * Sequential constructions (swaps, shuffles, rejection) run on one GPU thread
 * (or one per block); the call returns after enqueueing.  Errors:
 * SR_ERR_INVALID_ARGUMENT (NULL out with n > 0, n < 0, unknown order, param
 * out of range), SR_ERR_UNSUPPORTED_DTYPE, SR_ERR_OUT_OF_MEMORY (scratch). */
enum { SR_GEN_RANDOM = 0, SR_GEN_SORTED = 1, SR_GEN_REVERSED = 2, SR_GEN_SWAPS = 3, SR_GEN_FEW_UNIQUE = 4,
       SR_GEN_RUNS = 5, SR_GEN_LAST = 6, SR_GEN_SHARP_TEETH = 7, SR_GEN_EQUAL_TEETH = 8, SR_GEN_EVEN_TEETH = 9,
       SR_GEN_DISTANCE = 10, SR_GEN_ALL_EQUAL = 11, SR_GEN_EXTREMES = 12 };
int32_t sr_generate(void *out, int64_t n, int32_t dtype, int32_t order, uint64_t seed, int64_t param, void *stream);

/* ------------------------------------------------------------------ sort */

/* Sort keys[0..n) ascending in place.  dtype: SR_INT32 / SR_INT64 /
 * SR_FLOAT32 / SR_FLOAT64.  keys must be aligned to the key size.  Work is enqueued on `stream`; the call blocks
 * the host on small statistics readbacks (one for sorted / reversed /
 * single-level inputs) and returns before the GPU finishes; synchronise the
 * stream before reading keys.  Scratch: about n*(key bytes) + O(n/8) bytes,
 * stream-ordered from the device memory pool, released before return -- except
 * the single-launch path (keys only, n <= 2,359,296), which keeps its scratch
 * per (host thread, device) for the next such call.  That path blocks only
 * until its kernel reports the outcome (route and bucket sizes known, mid-
 * kernel) and returns while the kernel runs; a later single-launch call of the
 * same thread on another stream waits on the device for the earlier kernel.
 * Equal keys are indistinguishable, so the result is unique. */
int32_t sr_sort_keys(void *keys, int64_t n, int32_t dtype, void *stream);

/* Stable key-value sort: keys ascending; among equal keys the input order of
 * (key, val) pairs is kept; vals[i] travels with keys[i]
 * and is never compared.  vals: 4-byte elements, 4-byte aligned, must not
 * overlap keys.  Scratch about n*(key bytes + 4). */
int32_t sr_sort_pairs(void *keys, void *vals, int64_t n, int32_t dtype, void *stream);

/* End-to-end variants with HOST buffers (pinned or pageable): copies the
 * input host->device on `stream`, sorts, copies back, and synchronises the
 * stream before returning.  host_vals may be NULL for sr_sort_host (keys only).
 */
int32_t sr_sort_host(void *host_keys, void *host_vals, int64_t n, int32_t dtype, void *stream);

/* A batch of `count` independent sorts with HOST buffers -- the paper's
 * procedure sorts many instances of one size back to back (100 per input
 * class).  Instance i is host_keys[i][0..n[i]) (and, when
 * host_vals and host_vals[i] are not NULL, the 4-byte payloads host_vals[i]:
 * a stable pair sort); each is sorted in place exactly as sr_sort_host would.
 * The instances are pipelined over a ring of four device buffers and two copy
 * streams of the library beside `stream`: the upload of instance i+1 and the
 * download of instance i-1 overlap the sort of instance i (PCIe is full
 * duplex; the copies use the copy engines, not the SMs).  Pinned host
 * buffers are needed for the overlap (pageable ones are staged by the driver
 * and serialise).  The call starts after earlier work on `stream` and
 * synchronises it before returning; host buffers must not overlap.  Scratch: 4
 * buffers of max(n) keys (+ payloads) from the device pool, beside each
 * sort's own.  Errors as for sr_sort_host; on an error the batch stops,
 * instances already downloaded are sorted, the others are unspecified (each
 * still a permutation of its input or untouched). */
int32_t sr_sort_host_batch(void *const *host_keys, void *const *host_vals, const int64_t *n, int32_t count,
                           int32_t dtype, void *stream);

/* Record keys (the paper's "random 16-/64-/256-list"
 * classes, Table 2): recs holds n records of
 * `words` (1..1024) consecutive signed int32 values (row-major, 4-byte
 * aligned, device memory), sorted in place in ascending lexicographic order.
 * Records equal in every word are identical, so the result is unique.  The
 * call refines an index permutation with the stable int64 pair sort -- round 0
 * on the words (0, 1), round r on (run of equal prefix, word r+1) -- until no
 * two adjacent records tie or the words are exhausted, then gathers the
 * records (scratch ~ n*(words*4 + 28) bytes).  Synchronises the host once per
 * refinement round.  SR_ERR_INVALID_ARGUMENT (words out of range, NULL, host
 * pointer), SR_ERR_SIZE (n > 2^31 - 1), SR_ERR_ALIGNMENT; recs untouched on
 * these errors. */
int32_t sr_sort_records(void *recs, int64_t n, int32_t words, void *stream);

/* Presortedness measures of
 * keys[0..n) (device, int32 / int64, not modified), rank = stable rank
 * (SPEC.md:201):
 *   runs       Run(A) = #{i : a_i > a_{i+1}} + 1
 *   inversions Inv(A) = #{(i, j) : i < j, a_i > a_j}
 *   mono       Mono(A): fewest contiguous pieces that are each sorted or
 *              reversely sorted (non-decreasing / non-increasing)
 *   max_dis    max_i |rank(a_i) - i|: A is k-distance iff max_dis <= k
 *   misplaced  #{i : rank(a_i) != i}: <= 2k for a k-exchange list
 * Scratch ~ n*(key bytes + 12) bytes; synchronises the stream.  n = 0 gives all
 * zeros, n = 1 runs = mono = 1.  Errors as for sr_sort_keys. */
typedef struct {
  int64_t n, runs, inversions, mono, max_dis, misplaced;
} sr_measures;
int32_t sr_presortedness(const void *keys, int64_t n, int32_t dtype, sr_measures *host_out, void *stream);

/* ------------------------------------------------------------------ introspection */

typedef struct {
  int32_t route;            /* SR_ROUTE_* */
  int32_t levels;           /* partition levels, or merge levels */
  int64_t n;
  int64_t descents;         /* D = Run(A) - 1 */
  int64_t asc_breaks;       /* descending-run breaks */
  int64_t long_runs;        /* long natural runs found (either direction) */
  int64_t desc_runs_reversed;
  int64_t equal_keys;       /* keys placed by equality buckets */
  int64_t bytes_planned;    /* algorithmic HBM bytes of all launched kernels */
  int64_t workspace_bytes;
  int32_t launches;         /* kernels launched by the call */
  int32_t host_syncs;       /* host<->device statistics readbacks */
} sr_plan;

/* Plan of the last sort call made by this host thread.  SR_OK or
 * SR_ERR_INVALID_ARGUMENT when out is NULL. */
int32_t sr_last_plan(sr_plan *out);

const char *sr_status_string(int32_t status);
const char *sr_last_error(void); /* thread-local; "" when none */

enum {
  SR_OPT_FORCE_ROUTE = 0, /* 0 auto, SR_ROUTE_MERGE, SR_ROUTE_PARTITION or SR_ROUTE_OUTLIER (keys only)
                             (tests, ablations) */
  SR_OPT_PROFILE = 1,     /* 1: time every kernel with CUDA events (see sr_last_profile) */
  SR_OPT_MERGE_ROUTE = 2, /* 0: never choose the merge route automatically */
  SR_OPT_RESIDENT = 3,    /* 0: never use the single-launch resident path (keys only, 8192 < n <= 2^22) */
  SR_OPT_RESIDENT_CAP = 4, /* resident path: largest level-1 bucket sorted in-kernel, 1..16384 (default and
                              maximum: 16384 keys for int32, 8192 for int64); larger buckets are left for
                              host-driven partition levels (tests lower it) */
  SR_OPT_OUTLIER_ROUTE = 5, /* 0: never choose the outlier route automatically */
  SR_OPT_DISTANCE_ROUTE = 7, /* 0: never choose the k-distance route automatically */
  SR_OPT_WS_LIMIT = 6,    /* fault injection: device workspace bytes one call may take (0 = no limit); a
                             larger reservation fails with SR_ERR_OUT_OF_MEMORY as a real one would */
  SR_OPT_TUNE = 16        /* SR_OPT_TUNE + i, i < 8: tuning knobs of the large keys-only path (A/B runs):
                             +0 fused second level (k_bucket_sort) 1/0 (default 0: measured slower, DESIGN.md
                             §6.3); +1 level-1 buckets for n >= 2^26 (power of two <= 2048, default 512); +2 mean sub-bucket of
                             the fused level (16..4096, default 256); +3 cap on the level-1 buckets at
                             any n (power of two, 0 = none; tests reach the fused level at small n); +5 keys-only
                             scatter by two 512-thread CTAs per SM (1), by them only where the level's bin tables are
                             small and one 1024-thread CTA elsewhere (2, default), or one 1024-thread CTA (0); +6 mean bucket
                             of levels >= 2 (power of two; 0 = default: 512 int32 / 256 int64); +7 keys-only
                             warp finishing below level 1: 0 (default) items <= 256 by the 8-key network and
                             (256, 512] / (512, 1024] as two 8- / 16-key networks and a merge, 2 only the latter
                             split, 1 the 16- and 32-key networks (no split) */
};
/* Process-global, not thread-safe.  SR_ERR_INVALID_ARGUMENT for unknown keys/values. */
int32_t sr_set_option(int32_t key, int64_t value);

/* With SR_OPT_PROFILE on: per-kernel names, device ms and algorithmic bytes of
 * the last call on this thread (synchronises its stream).  Returns the number
 * of kernels (<= cap written). */
int32_t sr_last_profile(const char **names, float *ms, int64_t *bytes, int32_t cap);

/* ------------------------------------------------------------------ step-level entry points
 * One per hot-path row; used by the parity tests.  Integer
 * dtypes only (SR_ERR_UNSUPPORTED_DTYPE otherwise).  All are
 * synchronous (they synchronise `stream` before returning) and take device
 * pointers for array data and host pointers for small results. */

typedef struct {
  int64_t n, descents, asc_breaks;
  int64_t n_asc_runs, n_desc_runs, asc_cover, desc_cover;
} sr_presort_stats;

/* H1: presortedness scan with tile size `tile` (power of two, 1024..65536);
 * runs of length >= tile are reported.  strict = 1 uses strictly descending
 * runs (pairs), 0 non-increasing runs (keys).  host_runs (may be NULL): up to
 * cap rows of {start, len, dir(0 asc / 1 desc), 0}; asc runs first. */
int32_t sr_presort_scan(const void *keys, int64_t n, int32_t dtype, int32_t strict, int32_t tile,
                        sr_presort_stats *host_stats, int64_t *host_runs, int64_t cap, void *stream);

/* H2: reverse keys[s..e) (and vals when non-NULL) in place. */
int32_t sr_reverse_range(void *keys, void *vals, int64_t n, int32_t dtype, int64_t s, int64_t e, void *stream);

/* H4: stable sort of every tile [t*tile, (t+1)*tile) independently, tile <= 8192. */
int32_t sr_tile_sort(void *keys, void *vals, int64_t n, int32_t dtype, int32_t tile, void *stream);

/* H5: merge-path split i(d) = #A among the first d outputs of the stable
 * merge of sorted a[0..na) and b[0..nb) (A wins ties), for host_diags[0..nd). */
int32_t sr_merge_path(const void *a, int64_t na, const void *b, int64_t nb, int32_t dtype,
                      const int64_t *host_diags, int64_t *host_out, int64_t nd, void *stream);

/* H6: stable merge of sorted (a, va) and (b, vb) into (out, vout); va/vb/vout
 * may be NULL for keys only. */
int32_t sr_merge(const void *a, const void *va, int64_t na, const void *b, const void *vb, int64_t nb,
                 void *out, void *vout, int32_t dtype, void *stream);

/* H7: splitters of keys[0..n) for nbuckets (power of two, 2..1024) buckets:
 * host_spl[0..m) (int64), host_eq[0..m) equality flags; returns m via *m. */
int32_t sr_splitters(const void *keys, int64_t n, int32_t dtype, int32_t nbuckets, int64_t *host_spl,
                     uint8_t *host_eq, int32_t *m, void *stream);

/* H8-H10: one partition level: splitters (as sr_splitters), bucket histogram,
 * count-matrix scan and stable scatter of (keys, vals) into (out, vout) in
 * bucket order.  Equality buckets' keys are written too (filled) so that out
 * is the complete stable partition.  host_counts[0..2*nbuckets+1). */
int32_t sr_partition_level(const void *keys, const void *vals, int64_t n, int32_t dtype, int32_t nbuckets,
                           void *out, void *vout, int64_t *host_counts, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SR_SORT_H */
