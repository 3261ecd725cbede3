/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of what the GPU path
 * computes, written from the paper (H. Zhang, B. Meng, Y. Liang, "Sort Race",
 * arXiv 1609.04471; cited as PAPER.md:<line>) and from the definitions in
 * SURVEY.md §8(c).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant generator with paper_1609_04471_b200/csrc.
 *
 * Keys are widened to int64 internally (order-preserving for int32), and every
 * element carries a 4-byte opaque payload.  Ascending order is signed numeric
 * order.  No blocking, fusion or reordering beyond the plain
 * definitions below.
 *
 * Functions and the passage each follows:
 *   or_sort            stable top-down mergesort (north star "plain, slow,
 *                      single-threaded CPU mergesort"; merge keeps A on ties,
 *                      PAPER.md:99 "(f) ... any element in A no bigger than
 *                      the first element of B" ; stability PAPER.md:280)
 *   or_descents        |{i : a_i > a_{i+1}}|  = Run(A) - 1
 *   or_asc_runs        maximal ascending runs, split at descents
 *   or_desc_runs       maximal descending runs; keys-only: non-increasing,
 *                      pairs: strictly decreasing
 *   or_reverse         reverse a[s..e)  (Appendix A "reverse")
 *   or_merge           stable merge of two sorted runs, A wins ties
 *   or_merge_path      #A elements among the first d outputs of or_merge,
 *                      by running the merge d steps (PAPER.md:100 galloping
 *                      locates "the position in A where the current element
 *                      in B should go")
 *   or_splitters       stratified sample -> sort -> every o-th order statistic;
 *                      equality flag when a splitter occurs > gamma = 2 times
 *                      in the sample (PAPER.md:157 pseudo-median sampling;
 *                      PAPER.md:168 "(g) ... more than gamma = 2 elements
 *                      equal to the pivot, use the 3-way splitting")
 *   or_classify        bucket of x: i = #{splitters < x}; 2i+1 if x equals
 *                      splitter i and its equality flag is set, else 2i
 *                      (3-way split)
 *   or_stable_partition stable counting distribution by bucket (PAPER.md:159
 *                      (e): presortedness not disturbed)
 *   or_count           #{x < v}, #{x <= v}  (rank) for sampled checks
 *   or_stable_rank     #{j: k_j < k_i} + #{j < i: k_j = k_i}
 *   or_sort_records    the same stable mergesort over records of `words` int32
 *                      compared lexicographically (the paper's 16-/64-/256-int
 *                      lists, Table 2; SURVEY.md
 *                      §8(f) NEXT #3)
 *   or_measures        presortedness measures of PAPER.md:62-85 from their
 *                      definitions: Run(A) = #descents + 1 (:66), Inv(A) =
 *                      #{i<j : a_i > a_j} (:64, counted while merging), Mono(A)
 *                      = fewest monotone pieces (:72, greedy left to right),
 *                      Dis(A) = max |rank(a_i) - i| (k-distance, :84) and
 *                      #{i : rank(a_i) != i} (k-exchange, :85), rank = stable
 *                      rank
 *   or_sort_float      the same stable mergesort over float32 / float64 keys
 *                      ordered by IEEE 754-2008 §5.10 totalOrder, written out
 *                      case by case from that definition (the paper's
 *                      "random double" class; SURVEY.md §8(f)
 *                      NEXT #2)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct {
    int64_t key;
    uint32_t val;
} rec_t;

/* ---- stable top-down mergesort ------------------------------------------------ */

static void or_merge_recs(const rec_t *a, int64_t na, const rec_t *b, int64_t nb, rec_t *out) {
    int64_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        if (a[i].key <= b[j].key) out[k++] = a[i++]; /* A wins ties: stable */
        else out[k++] = b[j++];
    }
    while (i < na) out[k++] = a[i++];
    while (j < nb) out[k++] = b[j++];
}

static void msort(rec_t *a, rec_t *tmp, int64_t lo, int64_t hi) {
    if (hi - lo <= 1) return;
    int64_t mid = lo + (hi - lo) / 2;
    msort(a, tmp, lo, mid);
    msort(a, tmp, mid, hi);
    or_merge_recs(a + lo, mid - lo, a + mid, hi - mid, tmp + lo);
    memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * sizeof(rec_t));
}

static int sort_recs(rec_t *r, int64_t n) {
    if (n <= 1) return 0;
    rec_t *tmp = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    if (!tmp) return -1;
    msort(r, tmp, 0, n);
    free(tmp);
    return 0;
}

/* keys: int32 (ks=4) or int64 (ks=8); vals may be NULL (keys-only sort). */
static int64_t load_key(const void *k, int ks, int64_t i) {
    return ks == 4 ? (int64_t)((const int32_t *)k)[i] : ((const int64_t *)k)[i];
}
static void store_key(void *k, int ks, int64_t i, int64_t v) {
    if (ks == 4) ((int32_t *)k)[i] = (int32_t)v;
    else ((int64_t *)k)[i] = v;
}

int or_sort(void *keys, uint32_t *vals, int64_t n, int ks) {
    if (n <= 1) return 0;
    rec_t *r = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    if (!r) return -1;
    for (int64_t i = 0; i < n; i++) {
        r[i].key = load_key(keys, ks, i);
        r[i].val = vals ? vals[i] : (uint32_t)i;
    }
    int rc = sort_recs(r, n);
    if (rc == 0)
        for (int64_t i = 0; i < n; i++) {
            store_key(keys, ks, i, r[i].key);
            if (vals) vals[i] = r[i].val;
        }
    free(r);
    return rc;
}

/* ---- presortedness ------------------------------------------- */

int64_t or_descents(const void *keys, int64_t n, int ks) {
    int64_t d = 0;
    for (int64_t i = 0; i + 1 < n; i++)
        if (load_key(keys, ks, i) > load_key(keys, ks, i + 1)) d++;
    return d;
}

/* Maximal ascending runs: a new run starts after every descent a_i > a_{i+1}.
 * Writes up to cap (start, len) pairs; returns the total number of runs. */
int64_t or_asc_runs(const void *keys, int64_t n, int ks, int64_t *starts, int64_t *lens, int64_t cap) {
    if (n <= 0) return 0;
    int64_t cnt = 0, s = 0;
    for (int64_t i = 0; i + 1 <= n; i++) {
        int brk = (i + 1 == n) || (load_key(keys, ks, i) > load_key(keys, ks, i + 1));
        if (brk) {
            if (cnt < cap) { starts[cnt] = s; lens[cnt] = i + 1 - s; }
            cnt++;
            s = i + 1;
        }
    }
    return cnt;
}

/* Maximal descending runs: a new run starts after every a_i < a_{i+1}
 * (non-increasing runs, keys-only) or a_i <= a_{i+1} (strict = 1, pairs). */
int64_t or_desc_runs(const void *keys, int64_t n, int ks, int strict, int64_t *starts, int64_t *lens, int64_t cap) {
    if (n <= 0) return 0;
    int64_t cnt = 0, s = 0;
    for (int64_t i = 0; i + 1 <= n; i++) {
        int brk = (i + 1 == n);
        if (!brk) {
            int64_t x = load_key(keys, ks, i), y = load_key(keys, ks, i + 1);
            brk = strict ? (x <= y) : (x < y);
        }
        if (brk) {
            if (cnt < cap) { starts[cnt] = s; lens[cnt] = i + 1 - s; }
            cnt++;
            s = i + 1;
        }
    }
    return cnt;
}

void or_reverse(void *keys, uint32_t *vals, int64_t s, int64_t e, int ks) {
    for (int64_t i = s, j = e - 1; i < j; i++, j--) {
        int64_t t = load_key(keys, ks, i);
        store_key(keys, ks, i, load_key(keys, ks, j));
        store_key(keys, ks, j, t);
        if (vals) { uint32_t u = vals[i]; vals[i] = vals[j]; vals[j] = u; }
    }
}

/* ---- merging ------------------------------------------------ */

void or_merge(const void *a, const uint32_t *va, int64_t na, const void *b, const uint32_t *vb, int64_t nb,
              void *out, uint32_t *vout, int ks) {
    int64_t i = 0, j = 0, k = 0;
    while (i < na || j < nb) {
        int take_a;
        if (i >= na) take_a = 0;
        else if (j >= nb) take_a = 1;
        else take_a = load_key(a, ks, i) <= load_key(b, ks, j); /* A wins ties */
        if (take_a) {
            store_key(out, ks, k, load_key(a, ks, i));
            if (vout) vout[k] = va ? va[i] : 0;
            i++;
        } else {
            store_key(out, ks, k, load_key(b, ks, j));
            if (vout) vout[k] = vb ? vb[j] : 0;
            j++;
        }
        k++;
    }
}

int64_t or_merge_path(const void *a, int64_t na, const void *b, int64_t nb, int64_t d, int ks) {
    int64_t i = 0, j = 0;
    for (int64_t k = 0; k < d; k++) {
        int take_a;
        if (i >= na) take_a = 0;
        else if (j >= nb) take_a = 1;
        else take_a = load_key(a, ks, i) <= load_key(b, ks, j);
        if (take_a) i++; else j++;
    }
    return i;
}

/* ---- splitter partition (§4 (c),(d),(e),(g)) ----------------- */

/* splitmix64 finalizer used as a counter-based jitter generator; the CUDA side
 * implements the same published generator independently. */
static uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Sample position k (0 <= k < S) of segment [start, start+len): stratum k is
 * [start + k*len/S, start + (k+1)*len/S); the sample sits at offset
 * floor(h * w / 2^64) inside it (h = the k-th jitter draw, w = stratum width),
 * i.e. a uniformly jittered position (SURVEY Q8 / DESIGN.md reading R8). */
int64_t or_sample_pos(int64_t start, int64_t len, int64_t S, int64_t k) {
    int64_t lo = (k * len) / S, hi = ((k + 1) * len) / S;
    int64_t w = hi - lo;
    uint64_t h = or_mix64((uint64_t)start + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ULL);
    uint64_t off = (uint64_t)(((unsigned __int128)h * (uint64_t)w) >> 64);
    return start + lo + (int64_t)off;
}

/* Splitters for one segment.  S = min(nbuckets * oversample, len) samples;
 * splitter t_j = the ((j+1)*S/nbuckets)-th smallest sample, j = 0..nbuckets-2
 * (equal values may repeat: classification by lower_bound sends every key to
 * the first of equal splitters, the repeats delimit empty buckets);
 * eq[j] = 1 when t_j occurs more than gamma = 2 times in the sample.
 * Returns m = nbuckets - 1. */
int32_t or_splitters(const void *keys, int64_t start, int64_t len, int32_t nbuckets, int32_t oversample,
                     int ks, int64_t *spl, uint8_t *eq) {
    int64_t S = (int64_t)nbuckets * oversample;
    if (S > len) S = len;
    if (S <= 0 || nbuckets < 2) return 0;
    rec_t *smp = (rec_t *)malloc((size_t)S * sizeof(rec_t));
    for (int64_t k = 0; k < S; k++) {
        smp[k].key = load_key(keys, ks, or_sample_pos(start, len, S, k));
        smp[k].val = (uint32_t)k;
    }
    sort_recs(smp, S);
    int32_t m = 0;
    for (int32_t j = 0; j + 1 < nbuckets; j++) spl[m++] = smp[((int64_t)(j + 1) * S) / nbuckets].key;
    for (int32_t i = 0; i < m; i++) {
        int64_t cnt = 0;
        for (int64_t k = 0; k < S; k++) cnt += (smp[k].key == spl[i]);
        eq[i] = cnt > 2; /* gamma = 2 */
    }
    free(smp);
    return m;
}

void or_classify(const void *keys, int64_t n, int ks, const int64_t *spl, const uint8_t *eq, int32_t m,
                 int32_t *bins) {
    for (int64_t x = 0; x < n; x++) {
        int64_t v = load_key(keys, ks, x);
        int32_t i = 0;
        while (i < m && spl[i] < v) i++; /* i = #{t_j < v}: splitters are increasing */
        int32_t e = (i < m && spl[i] == v && eq[i]) ? 1 : 0;
        bins[x] = 2 * i + e;
    }
}

/* Stable distribution of (keys, vals) by bins into out; counts[nbins] filled. */
int or_stable_partition(const int32_t *bins, int64_t n, int32_t nbins, const void *keys, const uint32_t *vals,
                        void *out_keys, uint32_t *out_vals, int64_t *counts, int ks) {
    int64_t *pos = (int64_t *)calloc((size_t)nbins + 1, sizeof(int64_t));
    if (!pos) return -1;
    for (int32_t b = 0; b < nbins; b++) counts[b] = 0;
    for (int64_t x = 0; x < n; x++) counts[bins[x]]++;
    for (int32_t b = 0; b < nbins; b++) pos[b + 1] = pos[b] + counts[b];
    for (int64_t x = 0; x < n; x++) {
        int64_t p = pos[bins[x]]++;
        store_key(out_keys, ks, p, load_key(keys, ks, x));
        if (out_vals) out_vals[p] = vals ? vals[x] : (uint32_t)x;
    }
    free(pos);
    return 0;
}

/* ---- counts for sampled checks at sizes where a full oracle sort is too slow --- */

int64_t or_count(const void *keys, int64_t n, int ks, int64_t v, int64_t *le) {
    int64_t lt = 0, l = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t x = load_key(keys, ks, i);
        lt += (x < v);
        l += (x <= v);
    }
    *le = l;
    return lt;
}

int64_t or_stable_rank(const void *keys, int64_t n, int ks, int64_t i) {
    int64_t v = load_key(keys, ks, i), r = 0;
    for (int64_t j = 0; j < n; j++) {
        int64_t x = load_key(keys, ks, j);
        r += (x < v) || (x == v && j < i);
    }
    return r;
}

/* ---- floating-point keys: IEEE 754 totalOrder ("double") -------- */

typedef struct {
    double v;        /* numeric value (exact for float32) */
    uint64_t raw;    /* the key's bit pattern (float32 widened unsigned) */
    uint64_t pay;    /* NaN: the magnitude bits (quiet bit + payload) */
    int neg, nan;
    uint32_t val;
} frec_t;

/* totalOrder(a, b), i.e. "a <= b", from its definition:
 *  - a negative sign orders first (this includes -0 < +0 and -NaN < all);
 *  - same sign, neither NaN: numeric order;
 *  - same sign, one NaN: a positive NaN is above every number, a negative NaN
 *    below every number;
 *  - same sign, both NaN: positive NaNs ascend with their magnitude bits
 *    (signalling below quiet, then payload), negative NaNs descend. */
static int tot_le(const frec_t *a, const frec_t *b) {
    if (a->neg != b->neg) return a->neg;
    if (!a->nan && !b->nan) return a->v <= b->v;
    if (a->nan && b->nan) return a->neg ? a->pay >= b->pay : a->pay <= b->pay;
    if (a->nan) return a->neg;   /* -NaN <= everything; +NaN <= nothing but NaNs */
    return !b->neg;              /* b is NaN: +NaN above a, -NaN below a */
}

static void fmerge(const frec_t *a, int64_t na, const frec_t *b, int64_t nb, frec_t *out) {
    int64_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) {
        if (tot_le(&a[i], &b[j])) out[k++] = a[i++]; /* A wins ties: stable */
        else out[k++] = b[j++];
    }
    while (i < na) out[k++] = a[i++];
    while (j < nb) out[k++] = b[j++];
}

static void fmsort(frec_t *a, frec_t *tmp, int64_t lo, int64_t hi) {
    if (hi - lo <= 1) return;
    int64_t mid = lo + (hi - lo) / 2;
    fmsort(a, tmp, lo, mid);
    fmsort(a, tmp, mid, hi);
    fmerge(a + lo, mid - lo, a + mid, hi - mid, tmp + lo);
    memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * sizeof(frec_t));
}

/* keys: float32 (fs=4) or float64 (fs=8), sorted in place by totalOrder; vals
 * (may be NULL) travel with their keys; equal keys keep their input order. */
int or_sort_float(void *keys, uint32_t *vals, int64_t n, int fs) {
    if (n <= 1) return 0;
    frec_t *r = (frec_t *)malloc((size_t)n * sizeof(frec_t));
    frec_t *tmp = (frec_t *)malloc((size_t)n * sizeof(frec_t));
    if (!r || !tmp) { free(r); free(tmp); return -1; }
    for (int64_t i = 0; i < n; i++) {
        if (fs == 4) {
            float f; uint32_t u;
            memcpy(&f, (const char *)keys + 4 * i, 4);
            memcpy(&u, &f, 4);
            r[i].v = (double)f;
            r[i].raw = u;
            r[i].neg = (int)(u >> 31);
            r[i].nan = isnan(f) ? 1 : 0;
            r[i].pay = u & 0x7fffffu;
        } else {
            double d; uint64_t u;
            memcpy(&d, (const char *)keys + 8 * i, 8);
            memcpy(&u, &d, 8);
            r[i].v = d;
            r[i].raw = u;
            r[i].neg = (int)(u >> 63);
            r[i].nan = isnan(d) ? 1 : 0;
            r[i].pay = u & 0xfffffffffffffull;
        }
        r[i].val = vals ? vals[i] : (uint32_t)i;
    }
    fmsort(r, tmp, 0, n);
    for (int64_t i = 0; i < n; i++) {
        if (fs == 4) { uint32_t u = (uint32_t)r[i].raw; memcpy((char *)keys + 4 * i, &u, 4); }
        else memcpy((char *)keys + 8 * i, &r[i].raw, 8);
        if (vals) vals[i] = r[i].val;
    }
    free(r);
    free(tmp);
    return 0;
}

/* ---- record keys: lexicographic order over int32 words (PAPER.md:58 lists) -- */

static int rec_le(const int32_t *a, const int32_t *b, int words) { /* a <= b lexicographically */
    for (int j = 0; j < words; j++) {
        if (a[j] < b[j]) return 1;
        if (a[j] > b[j]) return 0;
    }
    return 1; /* equal */
}

static void rmsort(int64_t *ix, int64_t *tmp, int64_t lo, int64_t hi, const int32_t *recs, int words) {
    if (hi - lo <= 1) return;
    int64_t mid = lo + (hi - lo) / 2;
    rmsort(ix, tmp, lo, mid, recs, words);
    rmsort(ix, tmp, mid, hi, recs, words);
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        if (rec_le(recs + ix[i] * words, recs + ix[j] * words, words)) tmp[k++] = ix[i++]; /* A wins ties */
        else tmp[k++] = ix[j++];
    }
    while (i < mid) tmp[k++] = ix[i++];
    while (j < hi) tmp[k++] = ix[j++];
    memcpy(ix + lo, tmp + lo, (size_t)(hi - lo) * sizeof(int64_t));
}

/* recs: n records of `words` int32, sorted in place; perm (may be NULL)
 * receives the input index of each output record. */
int or_sort_records(int32_t *recs, int64_t n, int words, int64_t *perm) {
    if (n <= 1) { if (perm && n == 1) perm[0] = 0; return 0; }
    int64_t *ix = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *tmp = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int32_t *out = (int32_t *)malloc((size_t)n * words * sizeof(int32_t));
    if (!ix || !tmp || !out) { free(ix); free(tmp); free(out); return -1; }
    for (int64_t i = 0; i < n; i++) ix[i] = i;
    rmsort(ix, tmp, 0, n, recs, words);
    for (int64_t i = 0; i < n; i++) memcpy(out + i * words, recs + ix[i] * words, (size_t)words * sizeof(int32_t));
    memcpy(recs, out, (size_t)n * words * sizeof(int32_t));
    if (perm) memcpy(perm, ix, (size_t)n * sizeof(int64_t));
    free(ix); free(tmp); free(out);
    return 0;
}

/* ---- presortedness measures ------- */

/* Inv by a counting mergesort: when an element of the right run is output,
 * every remaining element of the left run is greater (strictly: ties go left). */
static int64_t inv_msort(int64_t *a, int64_t *tmp, int64_t lo, int64_t hi) {
    if (hi - lo <= 1) return 0;
    int64_t mid = lo + (hi - lo) / 2;
    int64_t c = inv_msort(a, tmp, lo, mid) + inv_msort(a, tmp, mid, hi);
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        if (a[i] <= a[j]) tmp[k++] = a[i++];
        else { c += mid - i; tmp[k++] = a[j++]; }
    }
    while (i < mid) tmp[k++] = a[i++];
    while (j < hi) tmp[k++] = a[j++];
    memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * sizeof(int64_t));
    return c;
}

/* out: [runs, inversions, mono, max_dis, misplaced] */
int or_measures(const void *keys, int64_t n, int ks, int64_t *out) {
    out[0] = out[1] = out[2] = out[3] = out[4] = 0;
    if (n <= 0) return 0;
    /* Run(A) */
    out[0] = or_descents(keys, n, ks) + 1;
    /* Mono(A): extend the current piece while it stays non-decreasing or
     * non-increasing; its direction is fixed by its first strict step */
    int64_t pieces = 1;
    int dir = 0; /* 0 undetermined, 1 ascending, -1 descending */
    for (int64_t i = 0; i + 1 < n; i++) {
        int64_t x = load_key(keys, ks, i), y = load_key(keys, ks, i + 1);
        int step = x < y ? 1 : (x > y ? -1 : 0);
        if (step == 0) continue;
        if (dir == 0) dir = step;
        else if (step != dir) { pieces++; dir = 0; } /* a new piece starts at a_{i+1} */
    }
    out[2] = pieces;
    /* stable ranks: the stable sort of (key, index) */
    rec_t *r = (rec_t *)malloc((size_t)n * sizeof(rec_t));
    int64_t *perm = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *tmp = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!r || !perm || !tmp) { free(r); free(perm); free(tmp); return -1; }
    for (int64_t i = 0; i < n; i++) { r[i].key = load_key(keys, ks, i); r[i].val = (uint32_t)i; }
    if (sort_recs(r, n) != 0) { free(r); free(perm); free(tmp); return -1; }
    int64_t dis = 0, mis = 0;
    for (int64_t p = 0; p < n; p++) {  /* the element of input position r[p].val has rank p */
        int64_t d = p - (int64_t)r[p].val;
        if (d < 0) d = -d;
        if (d > dis) dis = d;
        if (d) mis++;
    }
    out[3] = dis;
    out[4] = mis;
    /* Inv(A) on the keys themselves */
    for (int64_t i = 0; i < n; i++) perm[i] = load_key(keys, ks, i);
    out[1] = inv_msort(perm, tmp, 0, n);
    free(r); free(perm); free(tmp);
    return 0;
}
