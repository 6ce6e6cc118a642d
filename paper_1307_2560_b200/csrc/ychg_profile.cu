// ychg_profile.cu -- run materialisation on the GPU: build_profile / column_runs
// (reference runscan.cpp:78-143, runscan.hpp:57-66).
//
// Three passes over the packed mask, count -> scan -> fill:
//   P1 profile_count_kernel   rises per (row band, column): a warp owns 32 words
//                             (1024 columns) x one 256-row band; bit-sliced ripple
//                             counters, transposed to per-column bytes.
//   P2 profile_scan_kernels   per column: exclusive prefix over bands (= index of
//                             the band's first run in the column's list) and the
//                             column total; then the exclusive prefix over columns
//                             (= offset of the column's list in the flat array).
//   P3 profile_fill_kernel    re-streams each band: a rise at row y opens run
//                             {c, y, ?} at the column's next index, a fall at row y
//                             closes the open run with y_bot = y-1; a virtual
//                             background row H closes what is open at the bottom.
// The flat output is column-major and sorted by y_top inside a column -- exactly
// ColumnProfile::runs flattened (runscan.hpp:40-50).
#include <cuda_runtime.h>

#include <cstdint>

#include "ychg_device.cuh"
#include "ychg_kernels.h"

namespace {

constexpr int kBandRows = 256;  // rows per band: counts per band <= 128 fit 8 bit-planes

struct ProfileArgs {
    const uint8_t* bits;
    int64_t pitch;
    int32_t width, height, row_bytes;
    int32_t n_words;   // ceil(width / 32)
    int32_t n_bands;   // ceil(height / kBandRows)
};

// Word `w` of row y in MSB-first column order (bit 31 - j = column 32w + j),
// bytes past the row are zero and columns >= width are masked off.
__device__ __forceinline__ uint32_t load_word(const ProfileArgs& a, int w, int y) {
    if (y < 0 || y >= a.height) return 0u;
    const uint8_t* row = a.bits + static_cast<int64_t>(y) * a.pitch;
    const int b0 = 4 * w;
    uint32_t v;
    if (b0 + 4 <= a.row_bytes) {
        v = __ldg(reinterpret_cast<const uint32_t*>(row + b0));  // rows are 16 B aligned (pitch)
    } else {
        v = 0;
        for (int q = 0; q < 4; ++q)
            if (b0 + q < a.row_bytes) v |= static_cast<uint32_t>(__ldg(row + b0 + q)) << (8 * q);
    }
    v = __byte_perm(v, 0u, 0x0123u);
    const int n = a.width - 32 * w;
    if (n < 32) v &= n <= 0 ? 0u : ~(0xFFFFFFFFu >> n);
    return v;
}

// P1: counts[band][col] = rises of column col in rows [band*256, band*256+256).
__global__ void profile_count_kernel(const ProfileArgs a, uint32_t* __restrict__ band_counts) {
    const int gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);  // one warp per (band, 32 words)
    const int lane = threadIdx.x & 31;
    const int strips = (a.n_words + 31) / 32;
    if (gw >= strips * a.n_bands) return;
    const int band = gw / strips, strip = gw - band * strips;
    const int w = strip * 32 + lane;
    const int y0 = band * kBandRows, y1 = min(a.height, y0 + kBandRows);
    uint32_t pl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (w < a.n_words) {
        uint32_t pa = load_word(a, w, y0 - 1);
        for (int y = y0; y < y1; ++y) {
            const uint32_t cur = load_word(a, w, y);
            uint32_t c = cur & ~pa;  // rises (runscan.cpp:57)
            pa = cur;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t t = pl[k] & c;
                pl[k] ^= c;
                c = t;
            }
        }
    }
    ychg_dev::transpose8x8_bytes(pl);  // byte L of pl[p] = counter of bit 8L+p = column 31-(8L+p)
    if (w < a.n_words) {
        uint32_t* out = band_counts + static_cast<int64_t>(band) * (a.n_words * 32) + 32 * w;
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
            for (int L = 0; L < 4; ++L) out[31 - (8 * L + p)] = (pl[p] >> (8 * L)) & 0xFFu;
    }
}

// P2a: per column, exclusive prefix over bands (in place) and the column total.
__global__ void profile_colscan_kernel(const ProfileArgs a, uint32_t* __restrict__ band_counts,
                                       int32_t* __restrict__ counts) {
    const int64_t stride = static_cast<int64_t>(a.n_words) * 32;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.width; c += gridDim.x * blockDim.x) {
        uint32_t run = 0;
        for (int b = 0; b < a.n_bands; ++b) {
            const uint32_t v = band_counts[b * stride + c];
            band_counts[b * stride + c] = run;
            run += v;
        }
        counts[c] = static_cast<int32_t>(run);
    }
}

// P2b: exclusive prefix over columns (single CTA, chunked block scan).
__global__ void profile_offsets_kernel(int32_t n, const int32_t* __restrict__ counts, int64_t* __restrict__ col_off,
                                       int64_t* __restrict__ n_runs) {
    __shared__ long long warp_tot[32];
    __shared__ long long carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + tid;
        const long long v = i < n ? counts[i] : 0;
        long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            long long wt = lane < nw ? warp_tot[lane] : 0;
            long long winc = wt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xFFFFFFFFu, winc, o);
                if (lane >= o) winc += t;
            }
            if (lane < nw) warp_tot[lane] = winc - wt;
        }
        __syncthreads();
        if (i < n) col_off[i] = carry + warp_tot[warp] + incl - v;
        __syncthreads();
        if (tid == blockDim.x - 1) carry += warp_tot[warp] + incl;
        __syncthreads();
    }
    if (tid == 0) *n_runs = carry;
}

// P3: fill.  Per warp: one band of 32 words; per lane the 32 columns' next run
// index lives in shared memory (index = columns' run count before the row).
__global__ void __launch_bounds__(256) profile_fill_kernel(const ProfileArgs a, const uint32_t* __restrict__ band_base,
                                                           const int64_t* __restrict__ col_off,
                                                           int32_t* __restrict__ runs /* [n][3] */) {
    __shared__ uint32_t next[8][32][33];  // [warp][lane][column-in-word], padded
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * 8 + wib;
    const int lane = threadIdx.x & 31;
    const int strips = (a.n_words + 31) / 32;
    if (gw >= strips * a.n_bands) return;
    const int band = gw / strips, strip = gw - band * strips;
    const int w = strip * 32 + lane;
    const int y0 = band * kBandRows;
    const int y1 = min(a.height, y0 + kBandRows);
    const bool last_band = (band == a.n_bands - 1);
    if (w >= a.n_words) return;
    const int64_t bstride = static_cast<int64_t>(a.n_words) * 32;
    uint32_t* nx = next[wib][lane];
    for (int j = 0; j < 32; ++j) nx[j] = band_base[band * bstride + 32 * w + j];
    uint32_t pa = load_word(a, w, y0 - 1);
    const int yend = last_band ? y1 + 1 : y1;  // virtual background row H closes open runs
    for (int y = y0; y < yend; ++y) {
        const uint32_t cur = y < a.height ? load_word(a, w, y) : 0u;
        uint32_t rises = cur & ~pa, falls = pa & ~cur;
        pa = cur;
        while (rises) {
            const int j = __clz(rises);  // column 32w + j
            rises &= ~(0x80000000u >> j);
            const int c = 32 * w + j;
            const int64_t r = col_off[c] + nx[j];
            nx[j] += 1;
            runs[3 * r + 0] = c;
            runs[3 * r + 1] = y;
        }
        while (falls) {
            const int j = __clz(falls);
            falls &= ~(0x80000000u >> j);
            const int c = 32 * w + j;
            const int64_t r = col_off[c] + nx[j] - 1;  // the run that is open in column c
            runs[3 * r + 2] = y - 1;
        }
    }
}

}  // namespace

extern "C" int ychg_launch_profile(const uint8_t* d_bits, int64_t pitch, int32_t width, int32_t height,
                                   uint32_t* d_band_counts, int32_t* d_counts, int64_t* d_col_off,
                                   int64_t* d_n_runs, int32_t* d_runs, int phase, cudaStream_t stream) {
    ProfileArgs a{};
    a.bits = d_bits;
    a.pitch = pitch;
    a.width = width;
    a.height = height;
    a.row_bytes = (width + 7) / 8;
    a.n_words = (width + 31) / 32;
    a.n_bands = (height + kBandRows - 1) / kBandRows;
    const int strips = (a.n_words + 31) / 32;
    const int warps = strips * a.n_bands;
    const int blocks = (warps + 7) / 8;
    if (phase == 0) {  // counts + offsets
        profile_count_kernel<<<blocks, 256, 0, stream>>>(a, d_band_counts);
        profile_colscan_kernel<<<(width + 255) / 256, 256, 0, stream>>>(a, d_band_counts, d_counts);
        profile_offsets_kernel<<<1, 1024, 0, stream>>>(width, d_counts, d_col_off, d_n_runs);
    } else {  // fill
        profile_fill_kernel<<<blocks, 256, 0, stream>>>(a, d_band_counts, d_col_off, d_runs);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

extern "C" int64_t ychg_profile_band_words(int32_t width, int32_t height) {
    const int64_t n_words = (width + 31) / 32;
    const int64_t n_bands = (height + kBandRows - 1) / kBandRows;
    return n_bands * n_words * 32;
}
