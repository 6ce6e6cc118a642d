// ychg_aux.cu -- K0 on-device synth, the stand-alone boundary detector, the
// host-path re-pitch and the PNM raster kernels (P5 threshold+pack, P4 pad mask).
//
// K0 reproduces the reference generators bit for bit (synth.cpp:38-104).  The
// random pattern draws one SplitMix64 value per pixel in row-major order
// (synth.hpp:19-24): draw i is mix(seed + (i+1) * golden), so every pixel is an
// independent function of its index and the image is generated in parallel.
//
// ychg_boundaries_* implement detect_boundary_columns (runscan.cpp:145-153) for
// counts that arrive from the host (the reference API takes a span of ints).
#include <cuda_runtime.h>

#include <cstdint>

#include "ychg_kernels.h"

namespace {

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

struct SynthArgs {
    int pattern, width, height, bands, cell, all;
    int x0, win;  // the buffer holds columns [x0, x0 + win) of the width x height image
    uint64_t seed, threshold;
    int64_t pitch;
    int row_bytes, band_h;
};

__device__ __forceinline__ bool synth_pixel(const SynthArgs& a, int x, int y) {
    switch (a.pattern) {
    case 0: return true;                                              // full
    case 1: return false;                                             // empty
    case 2: return x == 0 || y == 0 || x == a.width - 1 || y == a.height - 1;  // frame
    case 3: {                                                         // hbands
        const int b = y / (a.band_h + 1);
        return b < a.bands && (y - b * (a.band_h + 1)) < a.band_h;
    }
    case 4: return ((x / a.cell) + (y / a.cell)) % 2 == 0;            // checker
    default: {                                                        // random
        if (a.all) return true;
        const uint64_t i = static_cast<uint64_t>(y) * static_cast<uint64_t>(a.width) +
                           static_cast<uint64_t>(x);
        const uint64_t z = a.seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        return splitmix_mix(z) < a.threshold;
    }
    }
}

__global__ void synth_kernel(const SynthArgs a, uint8_t* __restrict__ out) {
    const int64_t total = a.pitch * a.height;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(idx / a.pitch);
        const int xb = static_cast<int>(idx - static_cast<int64_t>(y) * a.pitch);
        uint32_t v = 0;
        if (xb < a.row_bytes && !(a.pattern == 5 && a.threshold == 0 && !a.all)) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int xl = xb * 8 + i;
                const int x = a.x0 + xl;
                if (xl < a.win && x < a.width && synth_pixel(a, x, y)) v |= 0x80u >> i;
            }
        }
        out[idx] = static_cast<uint8_t>(v);
    }
}

// ---- boundaries from a counts array: flags words, then ordered compaction.
constexpr int kColsPerBlock = 1024;

__global__ void bflags_kernel(const int32_t* __restrict__ counts, int64_t n,
                              uint32_t* __restrict__ flags, int32_t* __restrict__ block_nb) {
    __shared__ int red[8];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kColsPerBlock;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int nb = 0;
    for (int wi = warp; wi < kColsPerBlock / 32; wi += 8) {
        const int64_t c = base + wi * 32 + lane;
        bool f = false;
        if (c < n) {
            const int32_t prev = c == 0 ? 0 : counts[c - 1];  // counts[-1] := 0
            f = counts[c] != prev;
        }
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
        const int64_t w = (base >> 5) + wi;
        if (lane == 0 && w * 32 < n) flags[w] = m;
        nb += __popc(m);
    }
    if (lane == 0) red[warp] = nb;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < 8; ++i) t += red[i];
        block_nb[blockIdx.x] = t;
    }
}

__global__ void bcompact_kernel(const uint32_t* __restrict__ flags, int64_t n,
                                const int32_t* __restrict__ block_nb, int32_t* __restrict__ out,
                                long long* __restrict__ n_out) {
    __shared__ long long red[8];
    __shared__ int wpre[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long off = 0;
    for (int t = threadIdx.x; t < static_cast<int>(blockIdx.x); t += blockDim.x) off += block_nb[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xFFFFFFFFu, off, o);
    if (lane == 0) red[warp] = off;
    const int64_t nwords = (n + 31) >> 5;
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * (kColsPerBlock / 32);
    if (warp == 0) {
        const uint32_t m = w0 + lane < nwords ? flags[w0 + lane] : 0u;
        const int c = __popc(m);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += v;
        }
        wpre[lane] = incl - c;
    }
    __syncthreads();
    long long base = 0;
    for (int i = 0; i < 8; ++i) base += red[i];
    for (int wi = warp; wi < 32; wi += 8) {
        const int64_t w = w0 + wi;
        if (w >= nwords) break;
        const uint32_t m = flags[w];
        if ((m >> lane) & 1u) out[base + wpre[wi] + __popc(m & ((1u << lane) - 1u))] =
            static_cast<int32_t>(w * 32 + lane);
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *n_out = base + block_nb[blockIdx.x];
}

// ---- column strips all-gathered from several GPUs (bench / multigpu.py): rank r's
// segment of the gathered buffer holds its strip's counts at [0, width_r) and its
// ychg_totals (4 int64) at int offset tot_off.  One pass writes the contiguous
// global counts and their change flags (bflags over the strided layout), and
// block 0 sums every segment's (runs, links).
struct GatherLayout {
    int32_t n_seg, seg_stride, tot_off;
    int32_t c0[65];  // first global column of each segment, c0[n_seg] = width
};

__device__ __forceinline__ int32_t gathered_count(const int32_t* __restrict__ g, const GatherLayout& L, int64_t c) {
    int r = 0;
    while (r + 1 < L.n_seg && c >= L.c0[r + 1]) ++r;
    return g[static_cast<int64_t>(r) * L.seg_stride + (c - L.c0[r])];
}

__global__ void bflags_gather_kernel(const int32_t* __restrict__ g, const GatherLayout L, int64_t n,
                                     int32_t* __restrict__ counts, uint32_t* __restrict__ flags,
                                     int32_t* __restrict__ block_nb, long long* __restrict__ sums) {
    __shared__ int red[8];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kColsPerBlock;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int nb = 0;
    for (int wi = warp; wi < kColsPerBlock / 32; wi += 8) {
        const int64_t c = base + wi * 32 + lane;
        bool f = false;
        if (c < n) {
            const int32_t v = gathered_count(g, L, c);
            const int32_t prev = c == 0 ? 0 : gathered_count(g, L, c - 1);  // counts[-1] := 0
            counts[c] = v;
            f = v != prev;
        }
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
        const int64_t w = (base >> 5) + wi;
        if (lane == 0 && w * 32 < n) flags[w] = m;
        nb += __popc(m);
    }
    if (lane == 0) red[warp] = nb;
    if (blockIdx.x == 0 && warp == 0) {
        long long runs = 0, links = 0;
        for (int r = lane; r < L.n_seg; r += 32) {
            const long long* t =
                reinterpret_cast<const long long*>(g + static_cast<int64_t>(r) * L.seg_stride + L.tot_off);
            runs += t[0];
            links += t[1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            runs += __shfl_xor_sync(0xFFFFFFFFu, runs, o);
            links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
        }
        if (lane == 0) {
            sums[0] = runs;
            sums[1] = links;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < 8; ++i) t += red[i];
        block_nb[blockIdx.x] = t;
    }
}

}  // namespace

// Columns [x0, x0 + win) of the width x height reference image (x0 a multiple of
// 8), packed from bit 7 of byte 0: a multi-GPU column strip generated in place,
// bit-exact with the same columns of the whole image (random draws are indexed
// by the global pixel index y * width + x).
extern "C" int ychg_launch_synth_window(int pattern, int width, int height, int x0, int win, int bands, int cell,
                                        double density, uint64_t seed, uint8_t* d_bits, int64_t pitch,
                                        cudaStream_t stream) {
    SynthArgs a{};
    a.pattern = pattern;
    a.width = width;
    a.height = height;
    a.x0 = x0;
    a.win = win;
    a.bands = bands;
    a.cell = cell < 1 ? 1 : cell;
    a.seed = seed;
    a.pitch = pitch;
    a.row_bytes = (win + 7) / 8;
    a.band_h = (pattern == 3 && bands > 0) ? (height - (bands - 1)) / bands : 0;
    if (pattern == 5) {
        // synth.cpp:76-79: threshold = (uint64)(density * 2^64), "all" when it saturates.
        if (density <= 0.0) {
            a.all = 0;
            a.threshold = 0;
        } else {
            const double scaled = density * 18446744073709551616.0;
            a.all = scaled >= 18446744073709551616.0;
            a.threshold = a.all ? 0 : static_cast<uint64_t>(scaled);
        }
    }
    const int64_t total = pitch * height;
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    synth_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(a, d_bits);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

extern "C" int ychg_launch_synth(int pattern, int width, int height, int bands, int cell,
                                 double density, uint64_t seed, uint8_t* d_bits, int64_t pitch,
                                 cudaStream_t stream) {
    return ychg_launch_synth_window(pattern, width, height, 0, width, bands, cell, density, seed, d_bits, pitch,
                                    stream);
}

// d_flags needs ceil(n/32) words rounded up to a multiple of 32; d_n is one long long.
// Scratch for per-block counts lives after the flags (caller allocates
// ceil(n/1024) extra int32 in d_flags' tail: see ychg_capi.cu).
extern "C" int ychg_launch_boundaries(const int32_t* d_counts, int64_t n, uint32_t* d_flags,
                                      int32_t* d_boundaries, long long* d_n, cudaStream_t stream) {
    const int64_t blocks = (n + kColsPerBlock - 1) / kColsPerBlock;
    if (blocks == 0) {
        cudaMemsetAsync(d_n, 0, sizeof(long long), stream);
        return 0;
    }
    int32_t* block_nb = reinterpret_cast<int32_t*>(d_flags + blocks * (kColsPerBlock / 32));
    bflags_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_counts, n, d_flags, block_nb);
    bcompact_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_flags, n, block_nb,
                                                                   d_boundaries, d_n);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// ---- dense host layout -> pitched device layout (TMA needs 16 B-aligned row strides).
// dst row y byte x (x < pitch) = src[y * row_bytes + x] for x < row_bytes, else 0.
// One warp per row, one 16 B destination word per lane and step: two aligned
// 16 B source loads, shifted into place.  The source offset within a 16 B word
// depends on the row only, so the word select below is warp-uniform.
namespace {
__global__ void __launch_bounds__(256) repitch_kernel(const uint8_t* __restrict__ src, int64_t row_bytes,
                                                       uint8_t* __restrict__ dst, int64_t pitch, int y0, int y1) {
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t nq = pitch >> 4;
    for (int y = y0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); y < y1; y += warps) {
        const int64_t row0 = int64_t(y) * row_bytes;
        const int off = static_cast<int>(row0 & 15);
        const int kw = off >> 2;
        const uint32_t sh = static_cast<uint32_t>(off & 3) * 8;
        const uint4* srow = reinterpret_cast<const uint4*>(src + (row0 - off));
        uint4* drow = reinterpret_cast<uint4*>(dst + int64_t(y) * pitch);
        for (int64_t q = lane; q < nq; q += 32) {
            uint4 o = make_uint4(0, 0, 0, 0);
            const int64_t valid = row_bytes - q * 16;
            if (valid > 0) {
                const uint4 A = __ldg(srow + q), B = __ldg(srow + q + 1);
                uint32_t u0, u1, u2, u3, u4;
                switch (kw) {
                    case 0: u0 = A.x, u1 = A.y, u2 = A.z, u3 = A.w, u4 = B.x; break;
                    case 1: u0 = A.y, u1 = A.z, u2 = A.w, u3 = B.x, u4 = B.y; break;
                    case 2: u0 = A.z, u1 = A.w, u2 = B.x, u3 = B.y, u4 = B.z; break;
                    default: u0 = A.w, u1 = B.x, u2 = B.y, u3 = B.z, u4 = B.w; break;
                }
                o.x = __funnelshift_r(u0, u1, sh);
                o.y = __funnelshift_r(u1, u2, sh);
                o.z = __funnelshift_r(u2, u3, sh);
                o.w = __funnelshift_r(u3, u4, sh);
                if (valid < 16) {  // the row's last word: zero the bytes past row_bytes
                    auto keep = [&](int j) {
                        const int64_t v = valid - 4 * j;
                        return v >= 4 ? 0xFFFFFFFFu : v <= 0 ? 0u : (1u << (8 * v)) - 1u;
                    };
                    o.x &= keep(0), o.y &= keep(1), o.z &= keep(2), o.w &= keep(3);
                }
            }
            drow[q] = o;
        }
    }
}
}  // namespace

// src must have >= 32 readable bytes past its last row (the caller over-allocates)
// and be 16 B aligned; dst rows are `pitch` (multiple of 16) bytes.
extern "C" int ychg_launch_repitch(const uint8_t* d_src, int64_t row_bytes, uint8_t* d_dst, int64_t pitch, int y0,
                                   int y1, cudaStream_t stream) {
    const int64_t rows = static_cast<int64_t>(y1) - y0;
    if (rows <= 0 || pitch <= 0) return 0;
    int64_t blocks = (rows + 7) / 8;  // 8 warps (rows) per block
    if (blocks > 148 * 8) blocks = 148 * 8;
    repitch_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_src, row_bytes, d_dst, pitch, y0, y1);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// ---------------------------------------------------------------------------- PNM rasters (§8f row 3)
// P5 (pnm.cpp:116-123): W*H grey bytes -> packed MSB-first rows, foreground iff
// sample < threshold.  One thread per output byte (8 samples).
__global__ void pack_p5_kernel(const uint8_t* __restrict__ samples, int32_t width, int32_t height, int32_t threshold,
                               uint8_t* __restrict__ bits, int64_t pitch) {
    const int64_t row_bytes = (int64_t(width) + 7) / 8;
    const int64_t total = row_bytes * height;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t y = i / row_bytes, b = i - y * row_bytes;
        const uint8_t* row = samples + y * width;
        const int x0 = static_cast<int>(b * 8);
        uint32_t v = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (x0 + k < width && __ldg(row + x0 + k) < threshold) v |= 0x80u >> k;
        bits[y * pitch + b] = static_cast<uint8_t>(v);
    }
}

// P4 (pnm.cpp:103-114): padding bits of the last byte of every row forced to 0.
__global__ void mask_pad_kernel(uint8_t* __restrict__ bits, int64_t pitch, int32_t height, int64_t last, uint8_t mask) {
    for (int64_t y = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; y < height; y += int64_t(gridDim.x) * blockDim.x)
        bits[y * pitch + last] &= mask;
}

extern "C" int ychg_launch_pack_p5(const uint8_t* d_samples, int32_t width, int32_t height, int32_t threshold,
                                   uint8_t* d_bits, int64_t pitch, cudaStream_t stream) {
    const int64_t total = (int64_t(width) + 7) / 8 * height;
    if (total <= 0) return 0;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pack_p5_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_samples, width, height, threshold, d_bits, pitch);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

extern "C" int ychg_launch_mask_pad(uint8_t* d_bits, int64_t pitch, int32_t width, int32_t height,
                                    cudaStream_t stream) {
    if (width % 8 == 0 || height <= 0) return 0;
    const uint8_t mask = static_cast<uint8_t>(0xFFu << (8 - width % 8));
    int64_t blocks = (int64_t(height) + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    mask_pad_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_bits, pitch, height, (width + 7) / 8 - 1, mask);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// Assemble all-gathered strips (see GatherLayout): global counts, flags, the
// ascending boundary list and its length, and the summed (runs, links).
extern "C" int ychg_launch_assemble_strips(const int32_t* d_gathered, int32_t n_seg, int32_t seg_stride,
                                           int32_t tot_off, const int32_t* c0, int64_t n, int32_t* d_counts,
                                           uint32_t* d_flags, int32_t* d_boundaries, long long* d_n,
                                           long long* d_sums, cudaStream_t stream) {
    if (n_seg < 1 || n_seg > 64) return static_cast<int>(cudaErrorInvalidValue);
    GatherLayout L{};
    L.n_seg = n_seg;
    L.seg_stride = seg_stride;
    L.tot_off = tot_off;
    for (int r = 0; r <= n_seg; ++r) L.c0[r] = c0[r];
    const int64_t blocks = (n + kColsPerBlock - 1) / kColsPerBlock;
    if (blocks == 0) {
        cudaMemsetAsync(d_n, 0, sizeof(long long), stream);
        cudaMemsetAsync(d_sums, 0, 2 * sizeof(long long), stream);
        return 0;
    }
    int32_t* block_nb = reinterpret_cast<int32_t*>(d_flags + blocks * (kColsPerBlock / 32));
    bflags_gather_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_gathered, L, n, d_counts, d_flags, block_nb,
                                                                     d_sums);
    bcompact_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(d_flags, n, block_nb, d_boundaries, d_n);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}
