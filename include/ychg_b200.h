/*
 * ychg_b200.h -- C ABI of the B200-native yCHG hot path (arXiv 1307.2560).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary and
 * no exception ever does.  Every function returns an int status (YCHG_OK or a
 * negative YCHG_ERR_*); ychg_last_error() returns a thread-local message.
 *
 * Image layout = the reference BinaryImage (proj/include/ychg/image.hpp:10-22,
 * 35-36): row-major, 1 bit per pixel, MSB-first bytes (x = 0 is bit 0x80),
 * rows of row_stride >= (width+7)/8 bytes, padding bits zero.
 *
 * The reference has no FFI of its own; these entry points are what a binding
 * of its runscan API would bind:
 *   ychg_cut_vertex_counts         replaces ychg::cut_vertex_counts
 *                                   (runscan.hpp:59-62, runscan.cpp:122-128)
 *   ychg_detect_boundary_columns   replaces ychg::detect_boundary_columns
 *                                   (runscan.hpp:68-71, runscan.cpp:145-153)
 *   ychg_scan_host                  counts + boundaries + hyperedge total in one
 *                                   pass; its hyperedge total equals
 *                                   hyperedge_count(decompose(build_profile(img)))
 *                                   (hypergraph.cpp:192, :94-170, runscan.cpp:130-143)
 *   ychg_build_profile_host /       replace ychg::build_profile / column_runs
 *   ychg_column_runs_host            (runscan.hpp:54-66, runscan.cpp:78-143)
 *   ychg_decompose_image /          decompose (hypergraph.cpp:94-170) on the device,
 *   ychg_decompose_profile           results in a ychg_hypergraph handle
 *   ychg_pnm_info / ychg_load_pnm / replace ychg::load_pnm (pnm.cpp:124-153); the
 *   ychg_load_pnm_device /           scan straight from PNM bytes
 *   ychg_scan_pnm
 *   ychg_plan_* / ychg_scan_device  the same pass on device-resident buffers and a
 *                                   caller stream (benchmarks, CUDA graphs,
 *                                   multi-GPU strips)
 *   ychg_synth_device               bit-exact on-device synth (synth.cpp:38-104)
 *
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point fails with YCHG_ERR_NO_DEVICE.
 */
#ifndef YCHG_B200_H
#define YCHG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define YCHG_ABI_VERSION 1

#if defined(__GNUC__)
#define YCHG_API __attribute__((visibility("default")))
#else
#define YCHG_API
#endif

enum {
    YCHG_OK = 0,
    YCHG_ERR_INVALID = -1,   /* bad argument: maps to ychg::ValidationError */
    YCHG_ERR_CUDA = -2,      /* CUDA runtime/driver failure: maps to ychg::Error */
    YCHG_ERR_OOM = -3,       /* device or pinned allocation failed */
    YCHG_ERR_NO_DEVICE = -4, /* no CUDA device (no CPU fallback exists) */
    YCHG_ERR_INTERNAL = -5,
    YCHG_ERR_PARSE = -6      /* malformed input bytes: maps to ychg::ParseError at ychg_last_error_offset() */
};

/* ScanStrategy::Kind (runscan.hpp:26-36) */
enum { YCHG_STRATEGY_SERIAL = 0, YCHG_STRATEGY_PARALLEL = 1 };

/* Synthetic patterns in the reference enum order (synth.hpp:27-34). */
enum {
    YCHG_PATTERN_FULL = 0,
    YCHG_PATTERN_EMPTY = 1,
    YCHG_PATTERN_FRAME = 2,
    YCHG_PATTERN_HBANDS = 3,
    YCHG_PATTERN_CHECKER = 4,
    YCHG_PATTERN_RANDOM = 5
};

/* Scalars produced by one scan.  Device-resident in ychg_scan_device. */
typedef struct {
    int64_t total_runs;   /* sum of counts == ColumnProfile::total_runs() (runscan.hpp:46-50) */
    int64_t links;        /* mutually-unique overlaps linked by decompose (hypergraph.cpp:137-143) */
    int64_t hyperedges;   /* total_runs - links == hyperedge_count(decompose(...)); -1 if not computed */
    int64_t n_boundaries; /* detect_boundary_columns(counts).size() */
} ychg_totals;

typedef struct {
    int32_t n_strips;       /* 1024-column strips */
    int32_t n_blocks;       /* 32-row blocks */
    int32_t seg_per_strip;  /* row segments per strip */
    int32_t n_segments;
    int32_t grid;           /* CTAs of the streaming kernel (persistent, <= SM count) */
    int32_t kernels_per_scan;
    int64_t workspace_bytes;
} ychg_plan_info;

typedef struct ychg_plan ychg_plan;

/* ---- diagnostics ---- */
YCHG_API const char* ychg_last_error(void);
/* Byte offset of the last YCHG_ERR_PARSE (the reference's ParseError::offset()); -1 otherwise.
 * ychg_last_error() then holds the message without the " (byte offset N)" suffix. */
YCHG_API int64_t ychg_last_error_offset(void);
YCHG_API int ychg_abi_version(void);
YCHG_API int ychg_device_count(int* n);

/* ---- host-buffer entry points (what the C++ drop-in calls) ----
 * Inputs and outputs are host memory (pinned or pageable).  Thread-safe: calls
 * serialise on a per-device context that caches the plan and device buffers. */

/* counts_out[width].  width == 0 -> nothing written; height == 0 -> all zeros.
 * strategy is validated like runscan.cpp:24-26 (parallel needs threads >= 1) and
 * otherwise ignored: every strategy runs the same GPU path. */
YCHG_API int ychg_cut_vertex_counts(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                           int32_t strategy_kind, int32_t threads, int32_t* counts_out);

/* boundaries_out must hold n entries; *n_out receives the number written. */
YCHG_API int ychg_detect_boundary_columns(const int32_t* counts, int64_t n, int32_t* boundaries_out,
                                 int64_t* n_out);
/* The same on device-resident counts (e.g. counts all-gathered from column
 * strips on several GPUs), asynchronous on `stream`:
 * d_flags needs ychg_boundary_flag_words(n) words (flags + scratch),
 * d_boundaries n ints, *d_n (device) receives the boundary count. */
YCHG_API int64_t ychg_boundary_flag_words(int64_t n);
YCHG_API int ychg_detect_boundaries_device(const int32_t* d_counts, int64_t n, uint32_t* d_flags,
                                           int32_t* d_boundaries, int64_t* d_n, void* stream);
/* Column strips all-gathered from n_seg GPUs in ONE collective:
 * segment r of d_gathered (seg_stride int32) holds strip r's counts at [0, c0[r+1]-c0[r])
 * and its ychg_totals at int offset totals_off (even).  Writes the contiguous global
 * counts, flags (ychg_boundary_flag_words(width) words), the boundary list, *d_n,
 * and d_sums[2] = summed (runs, links).  c0: host array of n_seg+1 column starts. */
YCHG_API int ychg_assemble_strips_device(const int32_t* d_gathered, int32_t n_seg, int32_t seg_stride,
                                         int32_t totals_off, const int32_t* c0, int64_t width, int32_t* d_counts,
                                         uint32_t* d_flags, int32_t* d_boundaries, int64_t* d_n, int64_t* d_sums,
                                         void* stream);

/* Fused pass.  counts_out[width] (may be NULL), boundaries_out[width] (may be NULL),
 * totals_out (may be NULL).  with_hyperedges = 0 skips K3 (hyperedges = -1). */
YCHG_API int ychg_scan_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                   int32_t with_hyperedges, int32_t* counts_out, int32_t* boundaries_out,
                   ychg_totals* totals_out);

/* ychg_scan_host over several devices of this process: column strips
 * on multiples of 1024 columns (n_parts of them, round-robin over `devices`, NULL =
 * the current device), each with an 8-column right halo; counts gathered, the
 * boundary list computed once over them, runs and links summed.  Same outputs as
 * ychg_scan_host. */
YCHG_API int ychg_scan_host_sharded(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                    int32_t n_parts, const int32_t* devices, int32_t n_devices,
                                    int32_t with_hyperedges, int32_t* counts_out, int32_t* boundaries_out,
                                    ychg_totals* totals_out);

/* Run materialisation (build_profile / column_runs, runscan.cpp:78-143).
 * Runs are int32 triples {col, y_top, y_bot} (the layout of ychg::Run), column-major
 * and sorted by y_top inside a column -- ColumnProfile::runs flattened.
 * *n_runs_out always receives the total; runs are written only when
 * runs_capacity >= total (call once with runs_out = NULL to size the buffer). */
YCHG_API int ychg_build_profile_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                     int32_t strategy_kind, int32_t threads, int32_t* counts_out,
                                     int32_t* runs_out, int64_t runs_capacity, int64_t* n_runs_out);
/* The same in ONE call (one upload, one count pass): after phase 0 the library
 * calls alloc(alloc_ctx, n_runs) for a host buffer of 3*n_runs int32 (NULL ->
 * YCHG_ERR_OOM) and fills it.  Not called when the image has no runs. */
typedef void* (*ychg_alloc_fn)(void* alloc_ctx, int64_t n_runs);
YCHG_API int ychg_build_profile_host_alloc(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                           int32_t strategy_kind, int32_t threads, int32_t* counts_out,
                                           ychg_alloc_fn alloc, void* alloc_ctx, int64_t* n_runs_out);
/* Runs of one column (runscan.cpp:104-120); YCHG_ERR_INVALID if col is out of range. */
YCHG_API int ychg_column_runs_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                   int32_t col, int32_t* runs_out, int64_t runs_capacity, int64_t* n_out);

/* Hyperedge decomposition (decompose, hypergraph.cpp:94-170) on the device.
 * The result handle holds the reference Hypergraph's members as flat arrays:
 *   edge_runs     n_runs int32 triples {col, y_top, y_bot}, grouped by hyperedge
 *                 in canonical order, columns ascending inside an edge (all_runs());
 *   edge_offsets  n_edges + 1 uint32 (edge i owns edge_runs[off[i] .. off[i+1]));
 *   run_to_edge   n_runs uint32, hyperedge id of each run in profile order.
 * ychg_decompose_image runs build_profile + decompose without leaving the GPU;
 * ychg_decompose_profile takes a flattened ColumnProfile (list_sizes[c] runs of
 * column list c, column-major) and validates it like validate_profile
 * (hypergraph.cpp:62-90): YCHG_ERR_INVALID with the reference's message. */
typedef struct ychg_hypergraph ychg_hypergraph;
YCHG_API int ychg_decompose_image(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                  int32_t strategy_kind, int32_t threads, ychg_hypergraph** out);
YCHG_API int ychg_decompose_profile(int32_t width, int32_t height, const int32_t* list_sizes, const int32_t* runs,
                                    int64_t n_runs, ychg_hypergraph** out);
/* n_runs, n_edges; device_ms = device time of the decomposition kernels (profile excluded). */
YCHG_API int ychg_hypergraph_info(const ychg_hypergraph* hg, int64_t* n_runs, int64_t* n_edges, float* device_ms);
/* Copies out any of the three arrays (NULL skips one). */
YCHG_API int ychg_hypergraph_copy(const ychg_hypergraph* hg, int32_t* edge_runs, uint32_t* edge_offsets,
                                  uint32_t* run_to_edge);
YCHG_API void ychg_hypergraph_destroy(ychg_hypergraph* hg);

/* PNM input (load_pnm, pnm.cpp:124-153).  P4 rasters are the
 * BinaryImage bytes themselves and go to the device as they are; P5 grey rasters
 * are thresholded and packed on the device (sample < threshold = foreground);
 * ASCII P1/P2 are parsed on the host.  Errors follow the reference: threshold
 * outside [0,255], P3/P6/P7 and maxval != 255 -> YCHG_ERR_INVALID; malformed or
 * truncated bytes -> YCHG_ERR_PARSE with the reference's byte offset. */
YCHG_API int ychg_pnm_info(const uint8_t* bytes, int64_t n, int32_t* kind, int32_t* width, int32_t* height);
/* Decode into a host BinaryImage buffer (row_stride >= (width+7)/8, height rows; padding bits zero). */
YCHG_API int ychg_load_pnm(const uint8_t* bytes, int64_t n, int32_t threshold, uint8_t* bits_out,
                           int64_t row_stride);
/* Decode straight into a device bit buffer (pitch >= (width+7)/8) on `cuda_stream`. */
YCHG_API int ychg_load_pnm_device(const uint8_t* bytes, int64_t n, int32_t threshold, uint8_t* d_bits,
                                  int64_t pitch, void* cuda_stream);
/* ychg_scan_host on a PNM file's bytes (counts_out: width ints, boundaries_out: width ints). */
YCHG_API int ychg_scan_pnm(const uint8_t* bytes, int64_t n, int32_t threshold, int32_t with_hyperedges,
                           int32_t* counts_out, int32_t* boundaries_out, ychg_totals* totals_out);

/* ---- device-resident plans ----
 * A plan fixes the geometry and owns its device workspace.  width_img columns
 * are present in the buffer, width_cnt <= width_img are counted; columns
 * [width_cnt, width_img) only serve as the right halo of the K3 pair step
 * (multi-GPU column strips).  A plan is not safe for concurrent use. */
YCHG_API int ychg_plan_create(int device, int32_t width_img, int32_t width_cnt, int32_t height,
                     ychg_plan** out);
/* Plan flags.  YCHG_PLAN_LATENCY sizes the launch for one isolated scan (two
 * CTAs per SM, all SMs streaming at once; images of one strip and <= 512 rows
 * take a single-CTA kernel instead: the host entry points use it); the default
 * favours back-to-back scans (about half a CTA per SM per scan, so that
 * consecutive scans interleave on the SMs). */
#define YCHG_PLAN_LATENCY 1
/* YCHG_PLAN_SYNC_INPUTS: the streaming kernel waits (griddepcontrol.wait) for the
 * kernel launched just before it on the stream to complete and flush before it
 * reads the image.  Without it the streaming kernel is a programmatic dependent
 * launch that does not wait: d_bits must then be complete before the kernel that
 * immediately precedes the scan starts (written by a memcpy, an event-ordered
 * stream, or any earlier kernel -- as in back-to-back scans of resident images).
 * Set it when a kernel of yours writes d_bits right before ychg_scan_device. */
#define YCHG_PLAN_SYNC_INPUTS 2
/* YCHG_PLAN_NO_SKIP: always run the full per-row step.  By default a 32-row block
 * whose rows all equal the row above (every word of the warp's 1024 columns, plus
 * the right-halo bit) is skipped: it changes no count, flag or K3 state.  The
 * results are identical either way; the flag exists for A/B timing. */
#define YCHG_PLAN_NO_SKIP 4
YCHG_API int ychg_plan_create_ex(int device, int32_t width_img, int32_t width_cnt, int32_t height, int32_t flags,
                                 ychg_plan** out);
YCHG_API void ychg_plan_destroy(ychg_plan* plan);
YCHG_API int ychg_plan_get_info(const ychg_plan* plan, ychg_plan_info* out);

/* d_bits: device rows of `pitch` bytes (pitch % 16 == 0, pitch >= (width_img+7)/8).
 * Outputs are device pointers: d_counts[width_cnt], d_flags[(width_cnt+31)/32]
 * (bit j of word w = change flag of column 32w+j), d_boundaries[width_cnt],
 * d_totals[1].  stream is a cudaStream_t (NULL = legacy default stream).
 * Asynchronous: returns after enqueueing the kernels. */
YCHG_API int ychg_scan_device(ychg_plan* plan, const uint8_t* d_bits, int64_t pitch, int32_t with_hyperedges,
                     int32_t* d_counts, uint32_t* d_flags, int32_t* d_boundaries,
                     ychg_totals* d_totals, void* stream);

/* Optional CUDA-event timing of the streaming kernel of the next scans on this
 * plan: after a scan completes, ychg_plan_last_ms reports the streaming kernel
 * and the finish (flags/compaction) kernels separately. */
YCHG_API int ychg_plan_set_timing(ychg_plan* plan, int32_t enabled);
YCHG_API int ychg_plan_last_ms(ychg_plan* plan, float* scan_ms, float* finish_ms);

/* Diagnostics: per-CTA %globaltimer stamps, layout [scan % 4][CTA][32 slots].
 * Streaming kernel: 0 entry, 1+w warp w (< 16) done streaming, 20 segment
 * published, 23 exit.  Finisher kernel (CTA = strip): 21 all segments seen,
 * 24 loads done, 26 K3 tree done, 27 look-back done, 25 outputs ready, 22 done.
 * enable=1 allocates, 0 frees; host_out (may be NULL) receives
 * min(capacity, 4*grid*32) stamps. */
YCHG_API int ychg_plan_debug_stamps(ychg_plan* plan, int32_t enable, uint64_t* host_out, int32_t capacity,
                                    int32_t* n_ctas);
/* Diagnostics: the stamp ring (mapped host memory) without synchronising. */
YCHG_API int ychg_plan_debug_peek(ychg_plan* plan, uint64_t* host_out, int32_t capacity);

/* ---- helpers ---- */
/* Bit-exact with reference synth() for every pattern (synth.cpp:38-104);
 * writes height rows of `pitch` bytes, padding bytes and bits zeroed. */
YCHG_API int ychg_synth_device(int32_t pattern, int32_t width, int32_t height, int32_t bands, int32_t cell,
                      double density, uint64_t seed, uint8_t* d_bits, int64_t pitch, void* stream);
/* Columns [x0, x0 + win) of the same width x height image (x0 a multiple of 8),
 * packed from bit 7 of each row's byte 0: a multi-GPU column strip generated in
 * place, bit-exact with those columns of the whole image. */
YCHG_API int ychg_synth_device_window(int32_t pattern, int32_t width, int32_t height, int32_t x0, int32_t win,
                                      int32_t bands, int32_t cell, double density, uint64_t seed, uint8_t* d_bits,
                                      int64_t pitch, void* stream);

/* Device memory helpers so hosts without a CUDA runtime binding can drive the
 * device API (tests, ctypes). */
YCHG_API int ychg_device_alloc(int device, int64_t bytes, void** out);
YCHG_API int ychg_device_free(int device, void* p);
YCHG_API int ychg_host_alloc_pinned(int64_t bytes, void** out);
YCHG_API int ychg_host_free_pinned(void* p);
YCHG_API int ychg_memcpy(void* dst, const void* src, int64_t bytes, void* stream);
YCHG_API int ychg_memcpy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                   int64_t height, void* stream);
YCHG_API int ychg_memset(void* dst, int32_t value, int64_t bytes, void* stream);
YCHG_API int ychg_stream_create(int device, void** out);
YCHG_API int ychg_stream_destroy(void* stream);
YCHG_API int ychg_stream_synchronize(void* stream);
YCHG_API int ychg_set_device(int device);

#ifdef __cplusplus
}
#endif

#endif /* YCHG_B200_H */
