// ychg_kernels.h -- internal launcher declarations shared by the .cu units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ychg_dev {
struct ScanParams;
}

extern "C" {
// Enqueue one scan (ONE programmatic-dependent launch of ychg_scan_kernel) on `stream`.
// Returns cudaError_t.
int ychg_launch_small(const ychg_dev::ScanParams* prm, int with_links, cudaStream_t stream);
int ychg_launch_scan(const void* tmap, const ychg_dev::ScanParams* prm, int grid, int with_links,
                     cudaStream_t stream);

// Set the kernels' dynamic shared-memory opt-in on the current device.
int ychg_scan_kernel_prepare(void);

// The streaming kernel entry and launch shape (for occupancy queries).
const void* ychg_scan_kernel_ptr(int with_links);
void ychg_scan_kernel_shape(int with_links, int* threads, int* smem_bytes);

int ychg_launch_synth(int pattern, int width, int height, int bands, int cell, double density,
                      uint64_t seed, uint8_t* d_bits, int64_t pitch, cudaStream_t stream);
int ychg_launch_synth_window(int pattern, int width, int height, int x0, int win, int bands, int cell,
                             double density, uint64_t seed, uint8_t* d_bits, int64_t pitch, cudaStream_t stream);

int ychg_launch_repitch(const uint8_t* d_src, int64_t row_bytes, uint8_t* d_dst, int64_t pitch, int y0, int y1,
                        cudaStream_t stream);

// Run materialisation (ychg_profile.cu): phase 0 = band counts + column totals +
// column offsets (+ run total); phase 1 = fill the flat [n][3] int32 run array.
int ychg_launch_profile(const uint8_t* d_bits, int64_t pitch, int32_t width, int32_t height, uint32_t* d_band_counts,
                        int32_t* d_counts, int64_t* d_col_off, int64_t* d_n_runs, int32_t* d_runs, int phase,
                        int64_t n_runs_hint, cudaStream_t stream);
int64_t ychg_profile_band_words(int32_t width, int32_t height);

// Hyperedge decomposition (ychg_decompose.cu).
int64_t ychg_decompose_ws_bytes(int64_t n);
int ychg_launch_decompose_validate(const int32_t* d_runs, const int64_t* d_col_off, int32_t width, int32_t height,
                                   int64_t n, unsigned long long* d_err, cudaStream_t stream);
int ychg_launch_decompose(const int32_t* d_runs, const int64_t* d_col_off, const int32_t* d_counts, int32_t width,
                          int64_t n, void* d_ws, int32_t* d_edge_runs, uint32_t* d_edge_offsets,
                          uint32_t* d_run_to_edge, unsigned long long* d_total, cudaStream_t stream);

// PNM rasters (ychg_aux.cu): P5 threshold + pack, P4 padding-bit mask.
int ychg_launch_pack_p5(const uint8_t* d_samples, int32_t width, int32_t height, int32_t threshold, uint8_t* d_bits,
                        int64_t pitch, cudaStream_t stream);
int ychg_launch_mask_pad(uint8_t* d_bits, int64_t pitch, int32_t width, int32_t height, cudaStream_t stream);

int ychg_launch_assemble_strips(const int32_t* d_gathered, int32_t n_seg, int32_t seg_stride, int32_t tot_off,
                                const int32_t* c0, int64_t n, int32_t* d_counts, uint32_t* d_flags,
                                int32_t* d_boundaries, long long* d_n, long long* d_sums, cudaStream_t stream);
int ychg_launch_boundaries(const int32_t* d_counts, int64_t n, uint32_t* d_flags,
                           int32_t* d_boundaries, long long* d_n, cudaStream_t stream);
}
