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
//   P3 fill                   re-streams each band, one lane per column: a rise
//                             at row y opens run {c, y, ?} at the column's next
//                             index, a fall at row y closes it with y_bot = y-1 (one
//                             12-byte record); a virtual background row H closes
//                             what is open at the bottom.  Default: the band-staged
//                             kernel (16-byte row loads, records staged per band in
//                             shared memory, written out column by column with
//                             8-byte vector stores).  Kept for unaligned buffers and
//                             A/B: a transposed fall walk (sparse), row stepping,
//                             the walk with a per-chunk staged write-out.
// The flat output is column-major and sorted by y_top inside a column -- exactly
// ColumnProfile::runs flattened (runscan.hpp:40-50).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "ychg_device.cuh"
#include "ychg_kernels.h"

namespace {

constexpr int kBandRows = 256;  // rows per band: counts per band <= 128 fit 8 bit-planes
constexpr int kChunk = 16;      // rows loaded ahead per step (independent loads in flight)

struct ProfileArgs {
    const uint8_t* bits;
    int64_t pitch;
    int32_t width, height, row_bytes;
    int32_t n_words;   // ceil(width / 32)
    int32_t n_bands;   // ceil(height / kBandRows)
    int32_t band_major;  // fill grid order: 1 = consecutive warps take consecutive words of one band group
    int32_t group;       // fill work unit: bands per warp (walked top to bottom)
};

// Word `w` of row y in MSB-first column order (bit 31 - j = column 32w + j),
// rows outside [0, height) are zero and columns >= width are masked off.
// Branch-free so a chunk's loads issue back to back: the row index is clamped
// and the result selected afterwards, and the word is always read whole -- the
// pitch is a multiple of 16 B, and bytes past the row (padding) only feed
// columns >= width, which the mask clears.
__device__ __forceinline__ uint32_t load_word(const ProfileArgs& a, int w, int y) {
    const int yc = min(max(y, 0), a.height - 1);
    uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(a.bits + static_cast<int64_t>(yc) * a.pitch + 4 * w));
    v = __byte_perm(v, 0u, 0x0123u);
    const int n = a.width - 32 * w;
    if (n < 32) v &= n <= 0 ? 0u : ~(0xFFFFFFFFu >> n);
    return (y < 0 || y >= a.height) ? 0u : v;
}

// P1: counts[band][col] = rises of column col in rows [band*256, band*256+256).
// One CTA per (band, 1024-column strip): warp q walks rows [64q, 64q+64) of the
// band, lane = one 32-bit word, bit-sliced ripple counters (16 row loads in
// flight); the four warps' per-column byte counters (<= 32 each) are added as
// packed bytes in shared memory and the strip's 1024 counts go out with
// coalesced stores.  (One warp per 256-row band left 12 warps per SM waiting on
// loads: 68 us for the 55 MB mask at 21000^2.)
constexpr int kCountWarps = 4;
constexpr int kCountRows = kBandRows / kCountWarps;  // 64 rows per warp: counters <= 32

__global__ void __launch_bounds__(kCountWarps * 32) profile_count_kernel(const ProfileArgs a,
                                                                        uint32_t* __restrict__ band_counts) {
    __shared__ uint32_t part[kCountWarps][8][32];
    __shared__ uint32_t cols[32 * 33];  // [word][column in word], padded row: conflict-free
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int strips = (a.n_words + 31) / 32;
    const int band = blockIdx.x / strips, strip = blockIdx.x - band * strips;
    if (band >= a.n_bands) return;
    const int w = strip * 32 + lane;
    const int y0 = band * kBandRows + kCountRows * warp, y1 = min(a.height, y0 + kCountRows);
    uint32_t pl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (w < a.n_words && y0 < a.height) {
        uint32_t pa = load_word(a, w, y0 - 1);
        for (int yb = y0; yb < y1; yb += kChunk) {
            uint32_t v[kChunk];  // kChunk independent row loads in flight
#pragma unroll
            for (int k = 0; k < kChunk; ++k) v[k] = load_word(a, w, yb + k < y1 ? yb + k : -1);
#pragma unroll
            for (int k = 0; k < kChunk; ++k) {
                uint32_t c = v[k] & ~pa;  // rises (runscan.cpp:57); rows past y1 load 0
                pa = v[k];
#pragma unroll
                for (int q = 0; q < 6; ++q) {  // <= 32 rises per column: 6 planes
                    const uint32_t t = pl[q] & c;
                    pl[q] ^= c;
                    c = t;
                }
            }
        }
    }
    ychg_dev::transpose8x8_bytes(pl);  // byte L of pl[p] = counter of bit 8L+p = column 31-(8L+p)
#pragma unroll
    for (int p = 0; p < 8; ++p) part[warp][p][lane] = pl[p];
    __syncthreads();
#pragma unroll
    for (int p = 2 * warp; p < 2 * warp + 2; ++p) {  // packed bytes: 4 x <= 32 never carries
        const uint32_t v = part[0][p][lane] + part[1][p][lane] + part[2][p][lane] + part[3][p][lane];
#pragma unroll
        for (int L = 0; L < 4; ++L) cols[33 * lane + 31 - (8 * L + p)] = (v >> (8 * L)) & 0xFFu;
    }
    __syncthreads();
    uint32_t* out = band_counts + static_cast<int64_t>(band) * (a.n_words * 32) + strip * 1024;
    for (int i = threadIdx.x; i < 1024; i += kCountWarps * 32)
        if (strip * 32 + (i >> 5) < a.n_words) out[i] = cols[33 * (i >> 5) + (i & 31)];
}

// P2a: per column, exclusive prefix over bands (in place) and the column total.
// One CTA per 32 columns (lane = column): warp q takes a contiguous range of
// bands with all of its loads in flight at once, the warps' sums are scanned in
// shared memory, and each warp writes its bands' exclusive prefixes.
constexpr int kScanWarps = 8;
constexpr int kScanBandsPerWarp = 16;  // 128 bands (32768 rows) per pass; taller images loop

__global__ void __launch_bounds__(kScanWarps * 32) profile_colscan_kernel(const ProfileArgs a,
                                                                         uint32_t* __restrict__ band_counts,
                                                                         int32_t* __restrict__ counts,
                                                                         int64_t* __restrict__ col_off,
                                                                         long long* __restrict__ cta_tot) {
    __shared__ uint32_t wsum[kScanWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 32 + lane;
    const bool live = c < a.width;
    const int64_t stride = static_cast<int64_t>(a.n_words) * 32;
    uint32_t carry = 0;  // bands before this pass (same in every warp)
    for (int p0 = 0; p0 < a.n_bands; p0 += kScanWarps * kScanBandsPerWarp) {
        const int per = (min(a.n_bands - p0, kScanWarps * kScanBandsPerWarp) + kScanWarps - 1) / kScanWarps;
        const int b0 = p0 + warp * per;
        uint32_t v[kScanBandsPerWarp];
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < kScanBandsPerWarp; ++k) {
            const int band = b0 + k;
            v[k] = live && k < per && band < a.n_bands ? band_counts[band * stride + c] : 0u;
            sum += v[k];
        }
        wsum[warp][lane] = sum;
        __syncthreads();
        uint32_t run = carry, tot = carry;
#pragma unroll
        for (int q = 0; q < kScanWarps; ++q) {
            const uint32_t x = wsum[q][lane];
            if (q < warp) run += x;
            tot += x;
        }
#pragma unroll
        for (int k = 0; k < kScanBandsPerWarp; ++k) {
            const int band = b0 + k;
            if (live && k < per && band < a.n_bands) {
                band_counts[band * stride + c] = run;
                run += v[k];
            }
        }
        carry = tot;
        __syncthreads();  // wsum is rewritten by the next pass
    }
    if (warp == 0) {
        if (live) counts[c] = static_cast<int32_t>(carry);
        // the column offsets' first level: exclusive prefix inside these 32 columns,
        // and their total (profile_offsets_kernel adds the prefix over the CTAs)
        long long incl = live ? static_cast<long long>(carry) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        if (live) col_off[c] = incl - static_cast<long long>(carry);
        if (lane == 31) cta_tot[blockIdx.x] = incl;
    }
}

// P2b: second level of the column offsets.  Every CTA scans the colscan CTAs'
// totals (32 columns each; a few KB, L2-resident) up to the 1024-column slice it
// fixes up -- col_off[c] += prefix[c / 32] -- so no single CTA walks all the
// columns; CTA 0 scans all of them and stores the run total.
__global__ void __launch_bounds__(1024) profile_offsets_kernel(int32_t n, const long long* __restrict__ cta_tot,
                                                               int64_t* __restrict__ col_off,
                                                               int64_t* __restrict__ n_runs) {
    __shared__ long long warp_tot[33];
    __shared__ long long pre[32];  // this slice's 32 CTA prefixes
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = (n + 31) / 32;
    const int slice = blockIdx.x;
    const int need = slice == 0 ? nb : min(nb, 32 * slice + 32);
    long long carry = 0;
    for (int b0 = 0; b0 < need; b0 += 1024) {
        const int i = b0 + tid;
        const long long v = i < need ? cta_tot[i] : 0;
        long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const long long wt = warp_tot[lane];
            long long winc = wt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xFFFFFFFFu, winc, o);
                if (lane >= o) winc += t;
            }
            warp_tot[lane] = winc - wt;
            if (lane == 31) warp_tot[32] = winc;
        }
        __syncthreads();
        if (i >= 32 * slice && i < 32 * slice + 32) pre[i - 32 * slice] = carry + warp_tot[warp] + incl - v;
        carry += warp_tot[32];
        __syncthreads();  // warp_tot is rewritten by the next chunk
    }
    if (slice == 0 && tid == 0) *n_runs = carry;
    __syncthreads();
    const int c = 1024 * slice + tid;
    if (c < n) col_off[c] += pre[tid >> 5];
}

// P3 (mid density): one warp per (band, word), lanes step the rows together.
// P3: fill.  One warp per (band, word); lane j owns column c = 32w + j and walks
// the band's rows (one broadcast word load per row), so each lane appends to ONE
// contiguous output stream -- its column's list -- and writes every run it
// opens and closes as one 12-byte record.  32 open streams per warp keep the
// L2 write set small (a lane-per-word layout had 1024 streams per warp and
// thrashed L2 with partial lines: 5x DRAM write amplification).  A run open at
// the band's top was started by an earlier band (index base-1): only its y_bot
// is written here; a run still open at the bottom gets {c, y_top} here and its
// y_bot from a later band (or the virtual background row H in the last band).
__global__ void __launch_bounds__(256) profile_fill_rowwise_kernel(const ProfileArgs a, const uint32_t* __restrict__ band_base,
                                                           const int64_t* __restrict__ col_off,
                                                           int32_t* __restrict__ runs /* [n][3] */) {
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= a.n_words * a.n_bands) return;
    const int w = gw / a.n_bands, band = gw - w * a.n_bands;  // consecutive warps: bands of one word
    const int c = 32 * w + lane;
    const bool live = c < a.width;
    const int y0 = band * kBandRows;
    const int y1 = min(a.height, y0 + kBandRows);
    const int yend = band == a.n_bands - 1 ? y1 + 1 : y1;  // virtual background row H closes open runs
    const uint32_t me = 0x80000000u >> lane;
    int64_t idx = live ? col_off[c] + band_base[static_cast<int64_t>(band) * a.n_words * 32 + c] : 0;
    int top = -1;  // y_top of a run opened in this band and still open
    uint32_t pa = load_word(a, w, y0 - 1);
    for (int yb = y0; yb < yend; yb += kChunk) {
        uint32_t v[kChunk];
#pragma unroll
        for (int k = 0; k < kChunk; ++k) v[k] = load_word(a, w, yb + k < y1 ? yb + k : -1);  // >= y1: background
#pragma unroll
        for (int k = 0; k < kChunk; ++k) {
            const int y = yb + k;
            if (y >= yend) break;
            const uint32_t rise = v[k] & ~pa, fall = pa & ~v[k];
            pa = v[k];
            if (!live) continue;
            if (fall & me) {
                if (top >= 0) {
                    runs[3 * idx + 0] = c;
                    runs[3 * idx + 1] = top;
                    runs[3 * idx + 2] = y - 1;
                    ++idx;
                    top = -1;
                } else {
                    runs[3 * (idx - 1) + 2] = y - 1;  // opened in an earlier band
                }
            }
            if (rise & me) top = y;
        }
    }
    if (live && top >= 0) {  // still open: a later band writes y_bot
        runs[3 * idx + 0] = c;
        runs[3 * idx + 1] = top;
    }
}


// 32x32 bit transpose across a warp: on entry bit b of lane k's x is M[k][b];
// on exit bit k of lane j's x is M[k][j].  Five shuffle stages swap the
// off-diagonal blocks of size s (Hacker's Delight's block transpose, one lane
// per row).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int sh = 16 >> i;
        const uint32_t m = masks[i];
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, x, sh);
        x = (lane & sh) ? ((x & ~m) | ((o & ~m) >> sh)) : ((x & m) | ((o & m) << sh));
    }
    return x;
}

// The same transpose in three instructions per stage: the partner's word is
// rotated by +-s (one funnel shift; the bits that wrap around land in the half
// this lane keeps) and merged with one LOP3 under a per-lane mask.  The per-lane
// rotate amounts and masks are computed once (TransposeLane) and reused.
struct TransposeLane {
    uint32_t rot[5], keep[5];
    __device__ __forceinline__ explicit TransposeLane(int lane) {
        const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const int sh = 16 >> i;
            const bool hi = (lane & sh) != 0;
            rot[i] = hi ? 32 - sh : sh;            // rotate left by s (low lane) or right by s (high lane)
            keep[i] = hi ? ~masks[i] : masks[i];   // the bits this lane keeps from its own word
        }
    }
};

__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, const TransposeLane& t) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, x, 16 >> i);
        const uint32_t r = __funnelshift_l(o, o, t.rot[i]);
        x = (x & t.keep[i]) | (r & ~t.keep[i]);
    }
    return x;
}

// P3: fill.  One warp per (band, word).  Per 32-row chunk, lane k loads row k's
// raw little-endian word (one load per lane instead of 32 broadcast loads per
// warp) and a warp bit transpose hands lane j the 32-row bit sequence of the
// column at raw bit j: c = 32w + 8(j/8) + 7 - j%8 (MSB-first bytes,
// image.hpp:17-72).  Rises (s & ~(s<<1 | prev)) and falls are then walked with
// ffs, in row order: work per lane is proportional to its runs, not its rows.
// Every run that closes inside the chunk is a complete 12-byte record {c, y_top,
// y_bot}; a lane's records of one chunk are consecutive entries of its column's
// list, so they are staged in shared memory (<= 16 per lane per chunk) and the
// warp then writes each lane's segment with coalesced stores -- full sectors
// instead of 32 partial 4-byte stores per instruction.  The two boundary cases
// are written directly (once per lane and band at most): a run open at the
// band's top was started by an earlier band (index base-1) and only its y_bot is
// written here; a run still open at the bottom gets {c, y_top} here and its y_bot
// from a later band (or the virtual background row H in the last band).
template <bool kStaged>
__host__ __device__ constexpr int fill_warps_per_cta() { return kStaged ? 4 : 8; }
constexpr int kLaneSlot = 3 * 16 + 1;  // 16 records per lane and chunk; odd stride: no bank conflicts

template <bool kStaged>
__global__ void __launch_bounds__(fill_warps_per_cta<kStaged>() * 32) profile_fill_kernel(const ProfileArgs a,
                                                                       const uint32_t* __restrict__ band_base,
                                                                       const int64_t* __restrict__ col_off,
                                                                       int32_t* __restrict__ runs /* [n][3] */) {
    constexpr int kFillWarps = fill_warps_per_cta<kStaged>();
    __shared__ int32_t stage[kStaged ? kFillWarps : 1][kStaged ? 32 * kLaneSlot : 1];
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * kFillWarps + wib;
    const int lane = threadIdx.x & 31;
    const int n_groups = (a.n_bands + a.group - 1) / a.group;
    if (gw >= a.n_words * n_groups) return;
    // Work unit: one word (32 columns) x a group of `group` consecutive 256-row
    // bands, walked top to bottom, so each lane writes ONE contiguous piece of its
    // column's list per group (fewer pieces = fewer partially written output
    // sectors, whose L2 evictions cost DRAM fill reads; profiles/r02_fill_ncu.md).
    // Grid order: word-major (consecutive warps: groups of one word) or band-major
    // (consecutive warps and CTAs: words of one group).
    const int w = a.band_major ? gw % a.n_words : gw / n_groups;
    const int grp = a.band_major ? gw / a.n_words : gw - w * n_groups;
    const int c = 32 * w + 8 * (lane >> 3) + 7 - (lane & 7);
    const bool live = c < a.width;
    const int b0 = grp * a.group;
    const int b1 = min(a.n_bands, b0 + a.group);
    const uint8_t* col = a.bits + 4 * static_cast<int64_t>(w);
    const int gy0 = b0 * kBandRows;
    uint32_t prev = gy0 > 0 ? (__ldg(reinterpret_cast<const uint32_t*>(col + static_cast<int64_t>(gy0 - 1) * a.pitch)) >> lane) & 1u
                            : 0u;
    int64_t idx = live ? col_off[c] + band_base[static_cast<int64_t>(b0) * a.n_words * 32 + c] : 0;
    int top = -1;  // y_top of a run opened in this group and still open
    int32_t* mine = kStaged ? &stage[wib][lane * kLaneSlot] : nullptr;
    for (int band = b0; band < b1; ++band) {
        const int y0 = band * kBandRows;
        const int y1 = min(a.height, y0 + kBandRows);
        // The whole band's rows are loaded up front: 8 independent loads per lane.
        constexpr int kChunks = kBandRows / 32;
        uint32_t raw[kChunks];
#pragma unroll
        for (int q = 0; q < kChunks; ++q) {
            const int y = y0 + 32 * q + lane;
            raw[q] = y < y1 ? __ldg(reinterpret_cast<const uint32_t*>(col + static_cast<int64_t>(y) * a.pitch)) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kChunks; ++q) {
            const int yb = y0 + 32 * q;
            if (yb >= y1) break;  // warp-uniform
            const uint32_t s = warp_transpose32(raw[q], lane);  // bit k = row yb + k
            const int nk = min(32, y1 - yb);
            const uint32_t valid = nk == 32 ? 0xFFFFFFFFu : (1u << nk) - 1u;
            const uint32_t above = (s << 1) | prev;  // bit k = row yb + k - 1
            const uint32_t rises = s & ~above;
            prev = (s >> (nk - 1)) & 1u;
            // One iteration per run that closes in this chunk (a fall at row k): its
            // y_top is the last rise below k, or the carried `top`.  Uniform body,
            // half the iterations of an event walk.
            uint32_t falls = live ? (above & ~s) & valid : 0u;
            uint32_t rs = live ? rises & valid : 0u;
            int n = 0;  // records of this lane in this chunk
            while (falls) {
                const int k = __ffs(falls) - 1;
                falls &= falls - 1;
                const uint32_t below = (1u << k) - 1u;
                const uint32_t r = rs & below;
                rs &= ~below;
                const int t = r ? yb + 31 - __clz(r) : top;
                top = -1;
                if (t >= 0) {
                    int32_t* rec = kStaged ? mine + 3 * n : runs + 3 * (idx + n);
                    rec[0] = c;
                    rec[1] = t;
                    rec[2] = yb + k - 1;
                    ++n;
                } else {
                    runs[3 * (idx - 1) + 2] = yb + k - 1;  // opened before this group
                }
            }
            if (rs) top = yb + 31 - __clz(rs);  // a run left open (at most one rise after the last fall)
            if (kStaged) {
                __syncwarp();
                // Coalesced write-out of the chunk's records (T ints in total, warp-
                // uniform).  T <= 512: one warp-wide segmented copy -- item t belongs to
                // the last lane l whose exclusive offset is <= t (5 shuffles) and goes to
                // runs[3*idx_l + t - off_l]; fewer, independent iterations win at mid
                // densities.  Larger T: lane by lane, each segment one coalesced store
                // per 32 ints (measured, profiles/r01_fill_variants.md).
                const int m3 = 3 * n;
                int inc = m3;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
                    if (lane >= o) inc += t;
                }
                const int total = __shfl_sync(0xFFFFFFFFu, inc, 31);
                const int off = inc - m3;
                if (total > 512) {
                    uint32_t pending = __ballot_sync(0xFFFFFFFFu, n > 0);
                    while (pending) {
                        const int l = __ffs(pending) - 1;
                        pending &= pending - 1;
                        const int ml = __shfl_sync(0xFFFFFFFFu, m3, l);
                        const int64_t base = __shfl_sync(0xFFFFFFFFu, idx, l);
                        const int32_t* src = &stage[wib][l * kLaneSlot];
                        int32_t* dst = runs + 3 * base;
                        for (int t = lane; t < ml; t += 32) dst[t] = src[t];
                    }
                } else {
                    for (int q0 = 0; q0 < total; q0 += 32) {
                        const int t = q0 + lane;
                        int l = 0;
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1) {
                            const int e = __shfl_sync(0xFFFFFFFFu, off, l + step);
                            if (e <= t) l += step;
                        }
                        const int ol = __shfl_sync(0xFFFFFFFFu, off, l);
                        const int64_t base = __shfl_sync(0xFFFFFFFFu, idx, l);
                        if (t < total) runs[3 * base + (t - ol)] = stage[wib][l * kLaneSlot + (t - ol)];
                    }
                }
                __syncwarp();
            }
            idx += n;
        }
    }
    if (!live) return;
    if (b1 == a.n_bands && prev) {  // the virtual background row H closes what is open
        if (top >= 0) {
            runs[3 * idx + 0] = c;
            runs[3 * idx + 1] = top;
            runs[3 * idx + 2] = a.height - 1;
        } else {
            runs[3 * (idx - 1) + 2] = a.height - 1;
        }
    } else if (top >= 0) {  // still open: a later group writes y_bot
        runs[3 * idx + 0] = c;
        runs[3 * idx + 1] = top;
    }
}

constexpr int kBandWarps = 4;
constexpr int kFlatMax = 1024;  // records of one flat write-out pass (the auto rule stays below ~800)
static_assert(kBandRows == 256, "band_write_pairs: <= 128 records per column and band, 2 per lane and pass");

// The vector part of one column's piece of 12-byte records {c, top, bot}: the
// piece's ints are c, t0, b0, c, t1, b1, ...; from its first 8-byte boundary
// (h = 0 or 1 ints in, at vd) lane p writes the three int2 holding ints
// h+6p .. h+6p+5 (records 2p, 2p+1: one 32-bit shared load) -- whole sectors per
// store instruction instead of 12-byte-strided partial ones.  nvh = 2 * (whole
// int2) + h.  The <= 1 int before the boundary and after the last whole int2 are
// written by the column's own lane (band_write_out).
__device__ __forceinline__ void band_write_pairs(const uint16_t* __restrict__ src, int lane, int cl, int nvh,
                                                 int2* __restrict__ vd, int y0) {
    const int nv = nvh >> 1, h = nvh & 1;
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // <= 128 records = 64 pairs
        const int pr = lane + 32 * k;
        if (3 * pr >= nv) break;  // this lane is past the piece
        const uint32_t e = reinterpret_cast<const uint32_t*>(src)[pr];  // entries 2pr, 2pr+1 (reads past the piece are never stored)
        const int t0 = y0 + static_cast<int>(e & 0xFFu), b0 = y0 + static_cast<int>((e >> 8) & 0xFFu);
        const int t1 = y0 + static_cast<int>((e >> 16) & 0xFFu), b1 = y0 + static_cast<int>(e >> 24);
        // h = 0: (c,t0) (b0,c) (t1,b1);  h = 1: (t0,b0) (c,t1) (b1,c)
        const int2 v0 = h ? make_int2(t0, b0) : make_int2(cl, t0);
        const int2 v1 = h ? make_int2(cl, t1) : make_int2(b0, cl);
        const int2 v2 = h ? make_int2(b1, cl) : make_int2(t1, b1);
        vd[3 * pr] = v0;
        if (3 * pr + 1 < nv) vd[3 * pr + 1] = v1;
        if (3 * pr + 2 < nv) vd[3 * pr + 2] = v2;
    }
}

// Write-out of a warp's staged records (word w, band rows from y0): lane l holds
// n_l 16-bit entries {top - y0 | (bot - y0) << 8} for column l of the word, to be
// stored at runs[idx_l ..].  Many records: column by column, lanes = consecutive
// records of one column (band_write_column's 8-byte vectors), two independent
// columns per iteration.  Fewer (<= ~25 per column): one flat pass over the warp's
// records packed 32 per iteration -- record t's lane comes from a shared-memory
// owner table each lane fills for its own range, its destination from the lane's
// precomputed {entry offset, int base}.
struct FlatTables {
    uint8_t owner[kFlatMax];
    int32_t eoff[32];
    int64_t gbase[32];
};

template <int kSlot>
__device__ __forceinline__ void band_write_out(const uint16_t* __restrict__ stage, FlatTables& ft, int lane, int n,
                                               int64_t idx, int w, int y0, int mode, int32_t* __restrict__ runs) {
    const int total = static_cast<int>(__reduce_add_sync(0xFFFFFFFFu, static_cast<unsigned>(n)));
#ifdef YCHG_DIAG_FILL_NOSTORE  // diagnostics build: staged records are never written (wrong output, timing only)
    if (total >= 0) return;
#endif
    if (total == 0) return;
    const uint32_t nonempty = __ballot_sync(0xFFFFFFFFu, n > 0);
    const bool flat = total <= kFlatMax &&
                      (mode == 2 || (mode == 0 && (total + 31) / 32 * 5 <= __popc(nonempty) * 4));
    if (flat) {
        int inc = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
            if (lane >= o) inc += t;
        }
        const int off = inc - n;
        for (int j = 0; j < n; ++j) ft.owner[off + j] = static_cast<uint8_t>(lane);
        ft.eoff[lane] = lane * kSlot - off;
        ft.gbase[lane] = 3 * (idx - off);
        __syncwarp();
        for (int t = lane; t < total; t += 32) {
            const int l = ft.owner[t];
            const uint32_t e = stage[ft.eoff[l] + t];
            int32_t* dst = runs + ft.gbase[l] + 3 * t;
            dst[0] = 32 * w + 8 * (l >> 3) + 7 - (l & 7);
            dst[1] = y0 + static_cast<int>(e & 0xFFu);
            dst[2] = y0 + static_cast<int>(e >> 8);
        }
        __syncwarp();
    } else {
        // Each lane prepares its own column's piece (the single head / tail ints and
        // the vector run's address and length); then column by column, two
        // independent columns per iteration, the warp writes the vector runs.
        const int64_t g = 3 * idx;
        const int h = static_cast<int>(g & 1);
        const int body = 3 * n - h;
        if (n > 0) {
            if (h) runs[g] = 32 * w + 8 * (lane >> 3) + 7 - (lane & 7);
            if (body & 1) runs[g + 3 * n - 1] = y0 + static_cast<int>(stage[lane * kSlot + n - 1] >> 8);
        }
        const int nvh = ((body >> 1) << 1) | h;
        int2* const vd = reinterpret_cast<int2*>(runs + g + h);
        uint32_t pending = nonempty;
        while (pending) {
            const int l1 = __ffs(pending) - 1;
            pending &= pending - 1u;
            const int l2 = pending ? __ffs(pending) - 1 : l1;
            pending &= pending - 1u;
            const int q1 = __shfl_sync(0xFFFFFFFFu, nvh, l1);
            const int q2 = l2 != l1 ? __shfl_sync(0xFFFFFFFFu, nvh, l2) : 0;
            int2* const d1 = reinterpret_cast<int2*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(vd), l1));
            int2* const d2 = reinterpret_cast<int2*>(__shfl_sync(0xFFFFFFFFu, reinterpret_cast<uintptr_t>(vd), l2));
            band_write_pairs(stage + l1 * kSlot, lane, 32 * w + 8 * (l1 >> 3) + 7 - (l1 & 7), q1, d1, y0);
            band_write_pairs(stage + l2 * kSlot, lane, 32 * w + 8 * (l2 >> 3) + 7 - (l2 & 7), q2, d2, y0);
        }
    }
}

// P3: fill, band-staged.  One warp per (256-row band, group of kW words): lane k
// loads rows y0+32q+k of the whole group with 16-byte loads up front (8 x kW/4
// independent loads).  Phase 1, chunk by chunk over all kW words at once (kW
// independent shuffle chains): a chunk whose 32 rows all repeat the row above is
// marked unchanged; the others are bit-transposed in place (lane j: its column's
// 32-row bit sequence).  Phase 2, word by word: the runs that open and close
// inside the band are paired rise <-> fall in lockstep (the k-th fall of a chunk,
// after the one closing a run carried in from above, closes the k-th rise) and
// staged as ONE 16-bit entry {top - y0, bot - y0} in the lane's shared-memory slot
// (<= 128 per band), then written out (band_write_out).  The
// two boundary records are written directly as in the walk kernel: the y_bot of a
// run opened in an earlier band (index base-1), and {c, y_top} of a run left open
// at the band's bottom (its y_bot comes from a later band or the virtual row H).
template <int kW>
__global__ void __launch_bounds__(kBandWarps * 32) profile_fill_band_kernel(const ProfileArgs a,
                                                                            const uint32_t* __restrict__ band_base,
                                                                            const int64_t* __restrict__ col_off,
                                                                            int32_t* __restrict__ runs /* [n][3] */) {
    static_assert(kW == 4 || kW == 8, "word group = one or two 16-byte loads per row");
    constexpr int kV = kW / 4;
    constexpr int kSlot = 130;  // <= 128 entries per lane and band (+2: odd word stride)
    __shared__ uint16_t stage[kBandWarps][32 * kSlot];
    __shared__ FlatTables flat_tabs[kBandWarps];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n_groups = (a.n_words + kW - 1) / kW;
    const int gw = blockIdx.x * kBandWarps + wib;
    if (gw >= n_groups * a.n_bands) return;
    const int band = gw / n_groups, grp = gw - band * n_groups;  // consecutive warps: groups of one band
    const int y0 = band * kBandRows;
    const int y1 = min(a.height, y0 + kBandRows);
    const int w0 = grp * kW;
    const int nv = (w0 + 4 < a.n_words) ? kV : 1;  // 16-byte halves inside the row (warp-uniform)
    const uint8_t* gbase = a.bits + 4 * static_cast<int64_t>(w0);
    uint32_t x[8][kW];  // raw words, transposed in place by phase 1
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int y = y0 + 32 * q + lane;
#pragma unroll
        for (int v = 0; v < kV; ++v) {
            const uint4 t = (y < y1 && v < nv) ? __ldg(reinterpret_cast<const uint4*>(gbase + static_cast<int64_t>(y) * a.pitch) + v)
                                               : make_uint4(0u, 0u, 0u, 0u);
            x[q][4 * v + 0] = t.x;
            x[q][4 * v + 1] = t.y;
            x[q][4 * v + 2] = t.z;
            x[q][4 * v + 3] = t.w;
        }
    }
    uint32_t aw[kW];  // row y0-1 (all lanes read the same 16 B: one transaction)
#pragma unroll
    for (int v = 0; v < kV; ++v) {
        const uint4 t = (y0 > 0 && v < nv) ? __ldg(reinterpret_cast<const uint4*>(gbase + static_cast<int64_t>(y0 - 1) * a.pitch) + v)
                                           : make_uint4(0u, 0u, 0u, 0u);
        aw[4 * v + 0] = t.x;
        aw[4 * v + 1] = t.y;
        aw[4 * v + 2] = t.z;
        aw[4 * v + 3] = t.w;
    }
    // Each column's first index in this band, loaded with the rows.
    int64_t idx0[kW];
#pragma unroll
    for (int i = 0; i < kW; ++i) {
        const int c = 32 * (w0 + i) + 8 * (lane >> 3) + 7 - (lane & 7);
        idx0[i] = (w0 + i < a.n_words && c < a.width)
                      ? col_off[c] + band_base[static_cast<int64_t>(band) * a.n_words * 32 + c] : 0;
    }
    // Phase 1: differences against the row above (all chunks and words: independent
    // shuffles), then the transposes of the chunks that change.
    uint64_t changed = 0;  // bit kW*q + i: chunk q of word i has a transition
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t d = 0;
#pragma unroll
        for (int i = 0; i < kW; ++i) {
            const uint32_t xu = __shfl_up_sync(0xFFFFFFFFu, x[q][i], 1);
            const uint32_t last = q == 0 ? aw[i] : __shfl_sync(0xFFFFFFFFu, x[q > 0 ? q - 1 : 0][i], 31);
            d |= static_cast<uint32_t>(x[q][i] != (lane == 0 ? last : xu)) << i;
        }
        if (y0 + 32 * q >= y1) d = 0;
        changed |= static_cast<uint64_t>(__reduce_or_sync(0xFFFFFFFFu, d)) << (kW * q);
    }
    const TransposeLane tl(lane);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if ((changed >> (kW * q)) & ((1u << kW) - 1u)) {  // warp-uniform (kW <= 8)
#pragma unroll
            for (int i = 0; i < kW; ++i) x[q][i] = warp_transpose32(x[q][i], tl);
        }
    }
    // Phase 2.
    uint16_t* slot = &stage[wib][lane * kSlot];
    const bool last_band = band == a.n_bands - 1;
    // Rolled loops from here on (the walk body exists once: a fully unrolled
    // 4-word x 8-chunk walk overflowed the instruction cache): word i's chunks are
    // selected out of x into cur[] and shifted through it.
#pragma unroll 1
    for (int i = 0; i < kW; ++i) {
        const int w = w0 + i;
        if (w >= a.n_words) break;  // warp-uniform
        const int c = 32 * w + 8 * (lane >> 3) + 7 - (lane & 7);
        const bool live = c < a.width;
        uint32_t cur[8];
        uint32_t awi = aw[0];
        int64_t idx = idx0[0];
#pragma unroll
        for (int k = 1; k < kW; ++k)
            if (i == k) {
                awi = aw[k];
                idx = idx0[k];
            }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            cur[q] = x[q][0];
#pragma unroll
            for (int k = 1; k < kW; ++k) cur[q] = i == k ? x[q][k] : cur[q];
        }
        uint32_t prev = (awi >> lane) & 1u;
        int top = -1;  // y_top of a run opened in this band and still open
        int n = 0;     // staged records of this lane
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
            const int yb = y0 + 32 * q;
            const uint32_t s = cur[0];  // bit k = row yb + k
#pragma unroll
            for (int k = 0; k < 7; ++k) cur[k] = cur[k + 1];
            if (!((changed >> (kW * q + i)) & 1u)) continue;  // rows repeat the row above (or past y1)
            const int nk = min(32, y1 - yb);
            const uint32_t valid = nk == 32 ? 0xFFFFFFFFu : (1u << nk) - 1u;
            const uint32_t above = (s << 1) | prev;
            uint32_t R = live ? s & ~above & valid : 0u;
            uint32_t F = live ? above & ~s & valid : 0u;
            const bool carried = prev != 0u;
            prev = (s >> (nk - 1)) & 1u;
            if (carried && F) {  // the first fall closes the run open at the chunk's top
                const int f0 = __ffs(F) - 1;
                F &= F - 1u;
                if (top >= 0) {
                    slot[n++] = static_cast<uint16_t>((top - y0) | ((yb + f0 - 1 - y0) << 8));
                } else {
                    runs[3 * (idx - 1) + 2] = yb + f0 - 1;  // opened in an earlier band
                }
                top = -1;
            }
            // Every remaining fall closes the rise just before it: pair them from the
            // bottom (a rise with no fall after it opens the run left open).
            int nf = __popc(F);
            if (__popc(R) > nf) {
                const int r = 31 - __clz(R);
                top = yb + r;
                R ^= 1u << r;
            }
            const int off = 32 * q;
            int at = n + nf;
            n = at;
            while (nf > 0) {
                const int r = 31 - __clz(R), f = 31 - __clz(F);
                R ^= 1u << r;
                F ^= 1u << f;
                slot[--at] = static_cast<uint16_t>((off + r) | ((off + f - 1) << 8));
                --nf;
            }
        }
        __syncwarp();
        band_write_out<kSlot>(stage[wib], flat_tabs[wib], lane, n, idx, w, y0, a.group, runs);
        __syncwarp();
        idx += n;
        if (!live) continue;
        if (last_band && prev) {  // the virtual background row H closes what is open
            if (top >= 0) {
                runs[3 * idx + 0] = c;
                runs[3 * idx + 1] = top;
                runs[3 * idx + 2] = a.height - 1;
            } else {
                runs[3 * (idx - 1) + 2] = a.height - 1;
            }
        } else if (top >= 0) {  // still open: a later band writes y_bot
            runs[3 * idx + 0] = c;
            runs[3 * idx + 1] = top;
        }
    }
}

}  // namespace

extern "C" int ychg_launch_profile(const uint8_t* d_bits, int64_t pitch, int32_t width, int32_t height,
                                   uint32_t* d_band_counts, int32_t* d_counts, int64_t* d_col_off,
                                   int64_t* d_n_runs, int32_t* d_runs, int phase, int64_t n_runs_hint,
                                   cudaStream_t stream) {
    ProfileArgs a{};
    a.bits = d_bits;
    a.pitch = pitch;
    a.width = width;
    a.height = height;
    a.row_bytes = (width + 7) / 8;
    a.n_words = (width + 31) / 32;
    a.n_bands = (height + kBandRows - 1) / kBandRows;
    a.band_major = -1;
    if (const char* v = std::getenv("YCHG_FILL_BAND_MAJOR"); v && *v) a.band_major = std::atoi(v);  // A/B hook
    const int strips = (a.n_words + 31) / 32;
    const int64_t fill_warps = static_cast<int64_t>(a.n_words) * a.n_bands;
    if (phase == 0) {  // counts + offsets
        profile_count_kernel<<<static_cast<unsigned>(strips * a.n_bands), kCountWarps * 32, 0, stream>>>(a, d_band_counts);
        // the colscan CTAs' totals live past the band counts in the same buffer
        long long* cta_tot = reinterpret_cast<long long*>(
            d_band_counts + ((static_cast<int64_t>(a.n_bands) * a.n_words * 32 + 1) & ~int64_t(1)));
        profile_colscan_kernel<<<(width + 31) / 32, kScanWarps * 32, 0, stream>>>(a, d_band_counts, d_counts, d_col_off,
                                                                                cta_tot);
        profile_offsets_kernel<<<(width + 1023) / 1024, 1024, 0, stream>>>(width, cta_tot, d_col_off, d_n_runs);
    } else {  // fill
        // Fill kernel: the band-staged kernel whenever the rows and the output are
        // 16-byte aligned (always, for the library's own buffers): on 21000^2 it
        // beats every walk kernel at every density (profiles/r02_fill_ncu.md:
        // hbands 77 -> 74 us, checker(21) 197 -> 127, checker(7) 501 -> 208, random
        // 1053 -> 402).  Otherwise by run density rho = runs per pixel, known from
        // the count pass (profiles/r01_fill_variants.md): the direct transposed walk
        // on sparse masks, the staged coalesced write-out on denser ones.
        // YCHG_FILL_KERNEL=direct|rowwise|staged|band forces one.
        const double rho = static_cast<double>(n_runs_hint) / (static_cast<double>(width) * height);
        int kind = 3;
        if (const char* f = std::getenv("YCHG_FILL_KERNEL")) {
            if (!std::strcmp(f, "direct")) kind = 0;
            else if (!std::strcmp(f, "rowwise")) kind = 1;
            else if (!std::strcmp(f, "staged")) kind = 2;
            else if (!std::strcmp(f, "band")) kind = 3;
        }
        const bool aligned = (reinterpret_cast<uintptr_t>(d_bits) & 15u) == 0 && (pitch & 15) == 0 &&
                             (reinterpret_cast<uintptr_t>(d_runs) & 15u) == 0;
        if (kind == 3 && !aligned) kind = rho < 0.04 ? 0 : 2;  // 16-byte row loads, 8-byte record stores
        // Grid order (profiles/r02_fill_ncu.md, 21000^2): band-major for the staged
        // kernel (checker(7) 552 -> 498 us, random 1154 -> 1053, checker(21) 334 -> 239)
        // and for the direct walk on very sparse masks (hbands 100 -> 77 us);
        // word-major for the direct walk otherwise (checker(21) 197 vs 216 us).
        if (a.band_major < 0) a.band_major = (kind == 2 || rho < 0.01) ? 1 : 0;
        a.group = 1;
        if (const char* v = std::getenv("YCHG_FILL_GROUP"); v && *v) a.group = std::max(1, std::atoi(v));  // A/B hook
        const int64_t unit_warps = static_cast<int64_t>(a.n_words) * ((a.n_bands + a.group - 1) / a.group);
        if (kind == 0) {
            constexpr int wpc = fill_warps_per_cta<false>();
            profile_fill_kernel<false><<<static_cast<unsigned>((unit_warps + wpc - 1) / wpc), wpc * 32, 0, stream>>>(
                a, d_band_counts, d_col_off, d_runs);
        } else if (kind == 1) {
            profile_fill_rowwise_kernel<<<static_cast<unsigned>((fill_warps + 7) / 8), 256, 0, stream>>>(
                a, d_band_counts, d_col_off, d_runs);
        } else if (kind >= 3) {
            constexpr int kw = 4;
            a.group = 0;  // band kernels: write-out mode (0 auto, 1 per column, 2 flat)
            if (const char* v = std::getenv("YCHG_FILL_WRITEOUT"); v && *v) a.group = std::atoi(v);  // A/B hook
            const int64_t units = static_cast<int64_t>((a.n_words + kw - 1) / kw) * a.n_bands;
            const unsigned blocks_b = static_cast<unsigned>((units + kBandWarps - 1) / kBandWarps);
            profile_fill_band_kernel<kw><<<blocks_b, kBandWarps * 32, 0, stream>>>(a, d_band_counts, d_col_off, d_runs);
        } else {
            constexpr int wpc = fill_warps_per_cta<true>();
            profile_fill_kernel<true><<<static_cast<unsigned>((unit_warps + wpc - 1) / wpc), wpc * 32, 0, stream>>>(
                a, d_band_counts, d_col_off, d_runs);
        }
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// u32 words of the band-count buffer: the per-(band, column) counts, then (8-byte
// aligned) one int64 total per 32 columns for the column-offset scan.
extern "C" int64_t ychg_profile_band_words(int32_t width, int32_t height) {
    const int64_t n_words = (width + 31) / 32;
    const int64_t n_bands = (height + kBandRows - 1) / kBandRows;
    return ((n_bands * n_words * 32 + 1) & ~int64_t(1)) + 2 * ((int64_t(width) + 31) / 32) + 2;
}
