// types.cuh -- descriptors shared by the host planner and the kernels.
#pragma once
#include <cstdint>

namespace sr {

// Per-tile presortedness summary (H1/K1).  Positions are global indices i of
// the adjacent pair (a_i, a_{i+1}); -1 / INT32_MAX when absent.
struct TileSummary {
  int32_t ndesc;   // #{i in tile : a_i > a_{i+1}}
  int32_t nab;     // #{i in tile : descending-run break}
  int32_t fdesc, ldesc;
  int32_t fab, lab;
  int32_t nviol;   // descents whose outer neighbours are out of order (outlier route choice)
  int32_t tok;     // resident path: the tile passed its own k-distance test (TileMM.ok); 0 elsewhere
};

// Bounded-displacement summary of one presort tile (the k-distance route,
// PAPER.md:84): the tile is cut into subtiles of kDSub keys; ok = 1 when
// max(subtile q) <= min(subtile q+2) for every q with both inside the tile;
// mn0/mn1 are the mins of its first two subtiles, mx0/mx1 the maxes of its
// last two (keys as int64; +inf / -inf where the tile has one subtile).
constexpr int kDSub = 256;
struct TileMM {
  int64_t mn0, mn1, mx0, mx1;
  int32_t ok, nsub;
};

// A long natural run [start, start+len) and its end keys as stored in the
// input (before any reversal).  dir: 0 ascending, 1 descending.
struct RunDesc {
  int64_t start, len;
  int64_t kfirst, klast;
};

// Device-side statistics block, copied to the host once per planning step.
struct DevStats {
  int64_t n;
  int64_t descents;     // D = Run(A) - 1
  int64_t asc_breaks;   // descending-run breaks
  int64_t n_asc_runs, n_desc_runs;    // long runs (>= L_min)
  int64_t asc_cover, desc_cover;      // keys covered by long runs
  // partition level (plan kernel)
  int64_t noneq_total;  // keys in range (non-equality) buckets
  int64_t n_items;      // small finishing items (len <= kSmallItem, and fills)
  int64_t n_items_big;  // large finishing items (kSmallItem < len <= kCap)
  int64_t n_ovf;        // oversized range buckets for the next level
  int64_t ovf_keys;
  int64_t eq_keys;
  int64_t error;        // device-detected inconsistency (must stay 0)
  int64_t route;        // device-side route decision (kRoute*)
  int64_t big_keys;     // keys in large finishing items
  int64_t dist_ok;      // bounded displacement < 2 kDSub (k-distance route possible)
};

// One segment of a partition level (H7-H10).
struct SegDesc {
  int64_t start, len;     // in the level's source buffer (global indices)
  int64_t mat_base;       // first count-matrix entry of this segment
  int64_t len_prefix;     // sum of len of earlier segments in this level
  int32_t nbuckets;       // B_s (power of two, <= kMaxBuckets)
  int32_t nbins;          // 2*B_s + 1 matrix rows (bucket-major)
  int32_t chunk_base;     // first global chunk index
  int32_t nchunks;        // G_s
  int64_t sample_base;    // first entry of this segment's sample / rank arrays
  int64_t pad;
};

// Work item for the finishing kernel (H11/H4 segmented).
enum : int32_t { kItemSort = 0, kItemFill = 1 };
struct Item {
  int64_t start;
  int64_t key;    // fill value for kItemFill
  int32_t len;
  int32_t kind;   // kItemSort / kItemFill | (buf << 4): buf 1 = workspace side
};

struct OvfSeg {
  int64_t start, len;
};

// route codes (equal to the SR_ROUTE_* values of include/sr_sort.h)
constexpr int64_t kRouteSorted = 1, kRouteReversed = 2, kRouteMerge = 3, kRoutePartition = 4, kRouteTile = 5,
                  kRouteOutlier = 6, kRouteDistance = 7, kRouteUndecided = 8;
// route_ok bits of the device resolve: merge route allowed, outlier route allowed
constexpr int kAllowMerge = 1, kAllowOutlier = 2, kOutlierStrict = 4, kAllowDistance = 8;
constexpr int64_t kOutlierRatioStrict = 512;  // with kOutlierStrict (the one-launch resident range)
constexpr int64_t kOutlierRatio = 32;  // outlier route when descents <= n / kOutlierRatio ...
constexpr int64_t kViolRatio = 16;     // ... and at most 1/16 of them have out-of-order neighbours

constexpr int kMaxBuckets = 2048;           // B_max per level
constexpr int kMaxBins = 2 * kMaxBuckets + 1;
constexpr int kOversample = 4;              // o: S = B*o <= kMaxSample samples
constexpr int kMaxSample = kMaxBuckets * kOversample;
constexpr int kCap = 8192;                  // largest finishing item (two 4096-key halves)
constexpr int kPack = 1024;                 // buckets <= kPack are packed into items < 2*kPack
constexpr int kSmallItem = 2 * kPack;       // items <= this go to the small finishing kernel
constexpr int kFillChunk = 8192;            // equality fills are split into items of this size
constexpr int kTargetBucket = 1024;         // mean bucket size the planner aims for

}  // namespace sr
static_assert(sizeof(sr::TileSummary) == 32, "TileSummary is read as two int4");
