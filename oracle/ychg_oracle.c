/*
 * ychg_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C, scalar, per-pixel restatement of the reference CPU algorithm for the
 * yCHG hot path of arXiv 1307.2560.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library.  The product path
 * (paper_1307_2560_b200/, libychg_b200.so) never links or calls it.
 *
 * Parity is PINNED two ways (see tests/test_oracle.py):
 *   - against the reference's own known-answer vectors (test_runscan.cpp:35-49,
 *     :129-143, test_hypergraph.cpp:75-88, test_bench.cpp:139-160,
 *     test_imagekit.cpp:81-91, acceptance.cpp:101-121), and
 *   - against the reference itself, compiled unmodified from /root/reference into
 *     oracle/_ref/libychg_ref.so by oracle/Makefile, on the 1170-image corpus
 *     (tests/golden/make_golden.py commits the resulting fixtures).
 *
 * Layout of an image (reference image.hpp:10-22,35-36): row-major, 1 bit per pixel,
 * MSB-first in each byte (x = 0 is bit 0x80), rows padded to stride = (w+7)/8 bytes,
 * padding bits zero.  All entry points take (bits, w, h, stride).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define YO_EXPORT __attribute__((visibility("default")))

static inline int yo_get(const uint8_t* bits, int64_t stride, int x, int y) {
    return (bits[(int64_t)y * stride + (x >> 3)] >> (7 - (x & 7))) & 1;
}

static inline void yo_set(uint8_t* bits, int64_t stride, int x, int y) {
    bits[(int64_t)y * stride + (x >> 3)] |= (uint8_t)(0x80u >> (x & 7));
}

/* ---------------------------------------------------------------- SplitMix64
 * synth.hpp:14-25: state += golden; two xor-shift-multiply rounds; final xor-shift. */
YO_EXPORT uint64_t yo_splitmix64_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* ---------------------------------------------------------------- synth
 * Patterns in the reference's enum order (synth.hpp:27-34).
 * Returns 0 on success, -1 on a spec that synth.cpp:10-34 rejects. */
enum { YO_FULL = 0, YO_EMPTY = 1, YO_FRAME = 2, YO_HBANDS = 3, YO_CHECKER = 4, YO_RANDOM = 5 };

YO_EXPORT int yo_synth_validate(int pattern, int w, int h, int bands, int cell, double density) {
    if (w < 0 || h < 0) return -1;
    if (pattern == YO_HBANDS && (bands < 1 || bands > h / 2)) return -1;
    if (pattern == YO_CHECKER && cell < 1) return -1;
    if (pattern == YO_RANDOM && !(density >= 0.0 && density <= 1.0)) return -1;
    if (pattern < YO_FULL || pattern > YO_RANDOM) return -1;
    return 0;
}

/* ---------------------------------------------------------------- threads
 * Row / column ranges split over the host's cores (pthreads; no OpenMP runtime in
 * this image).  Only the large-image parity tests need it; results are identical
 * to the serial loops. */
typedef void (*yo_range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
    yo_range_fn fn;
    void* ctx;
    int64_t lo, hi;
} yo_job;

static void* yo_job_run(void* p) {
    yo_job* j = (yo_job*)p;
    if (j->hi > j->lo) j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void yo_parallel(int64_t n, yo_range_fn fn, void* ctx) {
    long t = sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 64) t = 64;
    if (n < 4096 || t == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[64];
    yo_job jobs[64];
    for (long i = 0; i < t; ++i) {
        jobs[i].fn = fn;
        jobs[i].ctx = ctx;
        jobs[i].lo = n * i / t;
        jobs[i].hi = n * (i + 1) / t;
        if (i > 0 && pthread_create(&th[i], NULL, yo_job_run, &jobs[i]) != 0) yo_job_run(&jobs[i]), th[i] = 0;
    }
    yo_job_run(&jobs[0]);
    for (long i = 1; i < t; ++i)
        if (th[i]) pthread_join(th[i], NULL);
}

typedef struct {
    int pattern, w, h, bands, cell, all;
    uint64_t seed, threshold;
    int64_t stride;
    uint8_t* out;
} yo_synth_args;

static void yo_synth_rows(void* p, int64_t y0, int64_t y1) {
    const yo_synth_args* a = (const yo_synth_args*)p;
    const int w = a->w, h = a->h;
    const int bh = a->pattern == YO_HBANDS ? (h - (a->bands - 1)) / a->bands : 0;
    for (int64_t yy = y0; yy < y1; ++yy) {
        const int y = (int)yy;
        switch (a->pattern) {
        case YO_FULL: /* synth.cpp:38-43 */
            for (int x = 0; x < w; ++x) yo_set(a->out, a->stride, x, y);
            break;
        case YO_FRAME: /* synth.cpp:45-51 */
            for (int x = 0; x < w; ++x)
                if (x == 0 || y == 0 || x == w - 1 || y == h - 1) yo_set(a->out, a->stride, x, y);
            break;
        case YO_HBANDS: { /* synth.cpp:55-64: equal maximal bands from the top, 1-row gaps */
            const int b = y / (bh + 1);
            if (b < a->bands && y - b * (bh + 1) < bh)
                for (int x = 0; x < w; ++x) yo_set(a->out, a->stride, x, y);
            break;
        }
        case YO_CHECKER: /* synth.cpp:66-72 */
            for (int x = 0; x < w; ++x)
                if (((x / a->cell) + (y / a->cell)) % 2 == 0) yo_set(a->out, a->stride, x, y);
            break;
        case YO_RANDOM: { /* synth.cpp:74-87: one draw per pixel, row-major, draw < density*2^64;
                           * draw i of the sequential generator mixes state seed + (i+1)*golden,
                           * so every row starts from seed + y*w*golden */
            uint64_t st = a->seed + (uint64_t)y * (uint64_t)w * 0x9e3779b97f4a7c15ull;
            for (int x = 0; x < w; ++x) {
                const uint64_t draw = yo_splitmix64_next(&st);
                if (a->all || draw < a->threshold) yo_set(a->out, a->stride, x, y);
            }
            break;
        }
        default:
            break;
        }
    }
}

/* out must hold h * ((w+7)/8) bytes; it is fully overwritten. */
YO_EXPORT int yo_synth(int pattern, int w, int h, int bands, int cell, double density,
                       uint64_t seed, uint8_t* out) {
    if (yo_synth_validate(pattern, w, h, bands, cell, density) != 0) return -1;
    yo_synth_args a;
    memset(&a, 0, sizeof(a));
    a.pattern = pattern;
    a.w = w;
    a.h = h;
    a.bands = bands;
    a.cell = cell;
    a.seed = seed;
    a.stride = (w + 7) / 8;
    a.out = out;
    memset(out, 0, (size_t)(a.stride * h));
    if (pattern == YO_EMPTY || (pattern == YO_RANDOM && density <= 0.0)) return 0;
    if (pattern == YO_RANDOM) {
        const double scaled = density * 18446744073709551616.0; /* 0x1p64 */
        a.all = scaled >= 18446744073709551616.0;
        a.threshold = a.all ? 0 : (uint64_t)scaled;
    }
    yo_parallel(h, yo_synth_rows, &a);
    return 0;
}

/* ---------------------------------------------------------------- step 1
 * Cut-vertex count of every column = number of maximal vertical foreground runs,
 * counted per pixel as background->foreground transitions scanning down with a
 * virtual background row -1 (runscan.cpp:41-74 semantics; the per-pixel form is
 * the reference's own independent checker corpus.hpp:91-102). */
typedef struct {
    const uint8_t* bits;
    int w, h;
    int64_t stride;
    int32_t* counts;
} yo_counts_args;

static void yo_counts_cols(void* p, int64_t c0, int64_t c1) {
    const yo_counts_args* a = (const yo_counts_args*)p;
    for (int64_t c = c0; c < c1; ++c) {
        int prev = 0, n = 0;
        for (int y = 0; y < a->h; ++y) {
            const int cur = yo_get(a->bits, a->stride, (int)c, y);
            n += cur & !prev;
            prev = cur;
        }
        a->counts[c] = n;
    }
}

YO_EXPORT void yo_cut_vertex_counts(const uint8_t* bits, int w, int h, int64_t stride,
                                    int32_t* counts) {
    yo_counts_args a = {bits, w, h, stride, counts};
    yo_parallel(w, yo_counts_cols, &a);
}

/* ---------------------------------------------------------------- step 2
 * runscan.cpp:145-153: ascending c with counts[c] != counts[c-1], counts[-1] := 0.
 * Returns the number of boundaries written to out (out may be NULL to only count). */
YO_EXPORT int64_t yo_detect_boundary_columns(const int32_t* counts, int64_t n, int32_t* out) {
    int64_t k = 0;
    int32_t previous = 0;
    for (int64_t c = 0; c < n; ++c) {
        if (counts[c] != previous) {
            if (out) out[k] = (int32_t)c;
            ++k;
        }
        previous = counts[c];
    }
    return k;
}

/* ---------------------------------------------------------------- hyperedge total
 * hyperedge_count(decompose(build_profile(img))) (hypergraph.cpp:94-170,192).
 * decompose links a run r of column c to a run s of column c+1 iff they overlap
 * vertically and each is the other's only overlap (two-pointer sweep, :116-143);
 * hyperedges are the resulting chains, so
 *     hyperedges = total runs - number of links.
 * Runs are extracted per column directly from pixels (column_runs, runscan.cpp:104-120).
 * Memory is two columns of runs at a time. */
typedef struct { int top, bot; } yo_run;

static int64_t yo_column_runs(const uint8_t* bits, int h, int64_t stride, int c, yo_run* out) {
    int64_t n = 0;
    int start = -1;
    for (int y = 0; y < h; ++y) {
        if (yo_get(bits, stride, c, y)) {
            if (start < 0) start = y;
        } else if (start >= 0) {
            out[n].top = start; out[n].bot = y - 1; ++n;
            start = -1;
        }
    }
    if (start >= 0) { out[n].top = start; out[n].bot = h - 1; ++n; }
    return n;
}

/* Links between two adjacent columns' sorted run lists (hypergraph.cpp:108-143). */
static int64_t yo_pair_links(const yo_run* a, int64_t na, const yo_run* b, int64_t nb,
                             uint32_t* ov_a, uint32_t* pa, uint32_t* ov_b, uint32_t* pb) {
    if (na == 0 || nb == 0) return 0;
    memset(ov_a, 0, sizeof(uint32_t) * (size_t)na);
    memset(ov_b, 0, sizeof(uint32_t) * (size_t)nb);
    int64_t i = 0, j = 0;
    while (i < na && j < nb) {
        if (a[i].bot < b[j].top) {
            ++i;
        } else if (b[j].bot < a[i].top) {
            ++j;
        } else {
            ++ov_a[i]; pa[i] = (uint32_t)j;
            ++ov_b[j]; pb[j] = (uint32_t)i;
            if (a[i].bot < b[j].bot) ++i;
            else if (b[j].bot < a[i].bot) ++j;
            else { ++i; ++j; }
        }
    }
    int64_t links = 0;
    for (int64_t k = 0; k < na; ++k)
        if (ov_a[k] == 1 && ov_b[pa[k]] == 1) ++links;
    return links;
}

/* Returns the hyperedge count; *total_runs_out and *links_out (if non-NULL) get the parts.
 * Returns -1 on allocation failure. */
YO_EXPORT int64_t yo_hyperedge_count(const uint8_t* bits, int w, int h, int64_t stride,
                                     int64_t* total_runs_out, int64_t* links_out) {
    int64_t total = 0, links = 0;
    if (w > 0 && h > 0) {
        const size_t cap = (size_t)h / 2 + 1;
        yo_run* ra = malloc(sizeof(yo_run) * cap);
        yo_run* rb = malloc(sizeof(yo_run) * cap);
        uint32_t* scratch = malloc(sizeof(uint32_t) * cap * 4);
        if (!ra || !rb || !scratch) { free(ra); free(rb); free(scratch); return -1; }
        int64_t na = yo_column_runs(bits, h, stride, 0, ra);
        total += na;
        for (int c = 0; c + 1 < w; ++c) {
            const int64_t nb = yo_column_runs(bits, h, stride, c + 1, rb);
            total += nb;
            links += yo_pair_links(ra, na, rb, nb, scratch, scratch + cap, scratch + 2 * cap,
                                   scratch + 3 * cap);
            yo_run* t = ra; ra = rb; rb = t;
            na = nb;
        }
        free(ra); free(rb); free(scratch);
    }
    if (total_runs_out) *total_runs_out = total;
    if (links_out) *links_out = links;
    return total - links;
}

/* Number of mutually-unique links per column pair (out[c] for pair (c, c+1), c < w-1).
 * Used by tests to localise a mismatch. */
YO_EXPORT int yo_pair_link_counts(const uint8_t* bits, int w, int h, int64_t stride,
                                  int32_t* out) {
    if (w < 2 || h <= 0) return 0;
    const size_t cap = (size_t)h / 2 + 1;
    yo_run* ra = malloc(sizeof(yo_run) * cap);
    yo_run* rb = malloc(sizeof(yo_run) * cap);
    uint32_t* scratch = malloc(sizeof(uint32_t) * cap * 4);
    if (!ra || !rb || !scratch) { free(ra); free(rb); free(scratch); return -1; }
    int64_t na = yo_column_runs(bits, h, stride, 0, ra);
    for (int c = 0; c + 1 < w; ++c) {
        const int64_t nb = yo_column_runs(bits, h, stride, c + 1, rb);
        out[c] = (int32_t)yo_pair_links(ra, na, rb, nb, scratch, scratch + cap,
                                        scratch + 2 * cap, scratch + 3 * cap);
        yo_run* t = ra; ra = rb; rb = t;
        na = nb;
    }
    free(ra); free(rb); free(scratch);
    return 0;
}

/* Popcount of the whole buffer (image.cpp:7-12 foreground_count). */
YO_EXPORT int64_t yo_foreground_count(const uint8_t* bits, int64_t nbytes) {
    int64_t n = 0;
    for (int64_t i = 0; i < nbytes; ++i) n += __builtin_popcount(bits[i]);
    return n;
}

/* ---------------------------------------------------------------- run materialisation
 * collect_runs_in_columns / build_profile (runscan.cpp:78-100,130-143), restated per
 * column: flat column-major int32 triples {col, y_top, y_bot}.  Returns the number
 * of runs; writes at most `capacity` triples (runs may be NULL to only count). */
YO_EXPORT int64_t yo_profile(const uint8_t* bits, int w, int h, int64_t stride, int32_t* runs, int64_t capacity,
                             int32_t* counts) {
    int64_t n = 0;
    for (int c = 0; c < w; ++c) {
        int start = -1, k = 0;
        for (int y = 0; y <= h; ++y) {
            const int bit = y < h ? yo_get(bits, stride, c, y) : 0;
            if (bit) {
                if (start < 0) start = y;
            } else if (start >= 0) {
                if (runs && n < capacity) {
                    runs[3 * n + 0] = c;
                    runs[3 * n + 1] = start;
                    runs[3 * n + 2] = y - 1;
                }
                ++n;
                ++k;
                start = -1;
            }
        }
        if (counts) counts[c] = k;
    }
    return n;
}

/* ---------------------------------------------------------------- decompose
 * decompose(const ColumnProfile&) (hypergraph.cpp:94-170) restated on the flat
 * profile (column-major {col, y_top, y_bot} triples, counts[c] runs per column):
 *   1. per adjacent column pair, the two-pointer overlap sweep (:108-135) marks a
 *      link r -> s iff each run is the other's only vertical overlap (:136-143);
 *   2. chains are walked from every run without a left link, in profile order
 *      (:145-167), which is the canonical hyperedge numbering.
 * Outputs: edge_runs (triples, hyperedge order, columns ascending inside an edge),
 * edge_offsets[0..E] and run_to_edge[profile index] (the Hypergraph members,
 * hypergraph.hpp:68-71; run_to_edge as the constructor derives it, :19-55).
 * Returns E, or -1 on allocation failure. */
YO_EXPORT int64_t yo_decompose(const int32_t* runs, const int32_t* counts, int w, int32_t* edge_runs,
                               uint32_t* edge_offsets, uint32_t* run_to_edge) {
    int64_t n = 0;
    for (int c = 0; c < w; ++c) n += counts[c];
    int64_t* off = malloc(sizeof(int64_t) * ((size_t)w + 1));
    uint32_t* right = malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint8_t* has_left = calloc((size_t)n + 1, 1);
    size_t cap = 1;
    for (int c = 0; c < w; ++c) if ((size_t)counts[c] > cap) cap = (size_t)counts[c];
    uint32_t* scratch = malloc(sizeof(uint32_t) * cap * 4);
    yo_run* ra = malloc(sizeof(yo_run) * cap);
    yo_run* rb = malloc(sizeof(yo_run) * cap);
    if (!off || !right || !has_left || !scratch || !ra || !rb) {
        free(off); free(right); free(has_left); free(scratch); free(ra); free(rb);
        return -1;
    }
    off[0] = 0;
    for (int c = 0; c < w; ++c) off[c + 1] = off[c] + counts[c];
    for (int64_t g = 0; g < n; ++g) right[g] = UINT32_MAX;
    for (int c = 0; c + 1 < w; ++c) {
        const int64_t na = counts[c], nb = counts[c + 1];
        if (na == 0 || nb == 0) continue;
        for (int64_t i = 0; i < na; ++i) { ra[i].top = runs[3 * (off[c] + i) + 1]; ra[i].bot = runs[3 * (off[c] + i) + 2]; }
        for (int64_t j = 0; j < nb; ++j) { rb[j].top = runs[3 * (off[c + 1] + j) + 1]; rb[j].bot = runs[3 * (off[c + 1] + j) + 2]; }
        uint32_t *ov_a = scratch, *pa = scratch + cap, *ov_b = scratch + 2 * cap, *pb = scratch + 3 * cap;
        yo_pair_links(ra, na, rb, nb, ov_a, pa, ov_b, pb);
        for (int64_t i = 0; i < na; ++i)
            if (ov_a[i] == 1 && ov_b[pa[i]] == 1) {
                right[off[c] + i] = (uint32_t)(off[c + 1] + pa[i]);
                has_left[off[c + 1] + pa[i]] = 1;
            }
    }
    int64_t e = 0, pos = 0;
    edge_offsets[0] = 0;
    for (int64_t g = 0; g < n; ++g) {
        if (has_left[g]) continue;
        for (int64_t cur = g;; cur = right[cur]) {
            memcpy(edge_runs + 3 * pos, runs + 3 * cur, 12);
            run_to_edge[cur] = (uint32_t)e;
            ++pos;
            if (right[cur] == UINT32_MAX) break;
        }
        edge_offsets[++e] = (uint32_t)pos;
    }
    free(off); free(right); free(has_left); free(scratch); free(ra); free(rb);
    return e;
}

/* ---------------------------------------------------------------- a7, streaming form
 * The link count of decompose() (hypergraph.cpp:108-143) restated as a row scan per
 * column pair: the 4-connected components of the 2-column strip
 * {c, c+1} are row intervals; a row continues the open component iff
 * (a & pa) | (b & pb); a component is a link iff it holds exactly two runs (one per
 * column, mutually unique).  n counts the runs of the open component (saturating
 * at 3); virtual empty rows -1 and h close everything.  Independent of the GPU's
 * bit-sliced formulation; pinned to the decompose-based count above by
 * tests/test_oracle.py.  Column pairs are split over the host cores (the 65536^2
 * parity test, where decompose itself needs tens of GB).  Returns the link total;
 * hyperedges = total runs - links. */
typedef struct {
    const uint8_t* bits;
    int h, pairs;
    int64_t stride;
    int64_t links[1];  /* total, atomically accumulated by the ranges */
} yo_a7_args;

static void yo_a7_range(void* p, int64_t lo, int64_t hi) {
    yo_a7_args* a = (yo_a7_args*)p;
    const int chunk = 512;
    int64_t links = 0;
    unsigned char* n = (unsigned char*)calloc(chunk, 1);
    unsigned char* pa = (unsigned char*)calloc(chunk + 1, 1);
    unsigned char* cur = (unsigned char*)calloc(chunk + 1, 1);
    for (int64_t c0 = lo; c0 < hi; c0 += chunk) {
        const int np = (int)(hi - c0 < chunk ? hi - c0 : chunk);
        memset(n, 0, (size_t)chunk);
        memset(pa, 0, (size_t)chunk + 1);
        for (int y = 0; y <= a->h; ++y) {
            /* bits of columns c0 .. c0+np (np + 1 columns) of row y; row h is empty */
            for (int i = 0; i <= np; ++i)
                cur[i] = y < a->h ? (unsigned char)yo_get(a->bits, a->stride, (int)c0 + i, y) : 0;
            for (int i = 0; i < np; ++i) {
                const int av = cur[i], bv = cur[i + 1], pav = pa[i], pbv = pa[i + 1];
                const int cont = (av & pav) | (bv & pbv);
                if (!cont) {
                    if ((pav | pbv) && n[i] == 2) ++links;
                    n[i] = (unsigned char)(av + bv);
                } else {
                    const int m = n[i] + (av & !pav) + (bv & !pbv);
                    n[i] = (unsigned char)(m > 3 ? 3 : m);
                }
            }
            unsigned char* t = pa;
            pa = cur;
            cur = t;
        }
    }
    free(n);
    free(pa);
    free(cur);
    __atomic_fetch_add(&a->links[0], links, __ATOMIC_RELAXED);
}

YO_EXPORT int64_t yo_a7_links(const uint8_t* bits, int w, int h, int64_t stride) {
    if (w < 2 || h <= 0) return 0;
    yo_a7_args* a = (yo_a7_args*)calloc(1, sizeof(yo_a7_args));
    a->bits = bits;
    a->h = h;
    a->pairs = w - 1;
    a->stride = stride;
    yo_parallel(w - 1, yo_a7_range, a);
    const int64_t links = a->links[0];
    free(a);
    return links;
}
