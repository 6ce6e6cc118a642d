// ychg_device.cuh -- sm_100a device building blocks for the yCHG column scan.
//
// Bit layout (reference image.hpp:10-22,35-36): row-major, MSB-first bytes, rows
// of ceil(W/8) bytes.  Words are used in raw little-endian load order (column
// 8L+7-p at bit 8L+p): every step is bitwise, so only the right-neighbour word b
// needs the layout -- inside a byte the neighbour is one bit lower (raw << 1),
// across bytes it is bit 7 of the next byte (raw >> 15, next word's byte 0).
//
// All per-pixel work is bit-sliced: one 32-bit register carries one bit of 32
// columns (K1) or of 32 adjacent column pairs (K3).
#pragma once

#include <cstdint>

namespace ychg_dev {

#ifndef YCHG_WARPS
#define YCHG_WARPS 4
#endif
#ifndef YCHG_STAGES
#define YCHG_STAGES 3
#endif
constexpr int kStripWords = 32;                  // one warp lane per 32-column word
constexpr int kStripCols = kStripWords * 32;     // 1024 columns per strip
constexpr int kStripBytes = kStripWords * 4;     // 128 B of every row
constexpr int kBoxBytes = kStripBytes + 16;      // + 16 B right halo (next strip's first word)
constexpr int kBlockRows = 32;                   // rows per TMA stage / per Harley-Seal block
constexpr int kStageBytes = kBoxBytes * kBlockRows;   // 4608 B
constexpr int kFlushBlocks = 15;                 // 8-bit bit-sliced counters: <= 15*16+15 = 255
constexpr int kSumPlanes = 7;                    // K3 band summary planes (see BandSummary)
constexpr int kMaxSegmentRows = 65504;           // u16 SWAR accumulators: counts <= rows/2 < 2^15

constexpr int kMaxSegPerStrip = 128;            // row segments per strip (partials per strip finish)
constexpr int kMaxSegPerCta = 64;               // segments one streaming CTA processes per scan
constexpr int kFinishChunk = 16;                // K3 summaries loaded + composed per chunk by a strip finisher
constexpr int kStampRing = 64;                  // diagnostics: scans kept in the per-CTA stamp ring

// The streaming kernel is instantiated per path (full: K1+K2+K3, counts: K1+K2)
// with its own CTA width and TMA ring depth (YCHG_WARPS[_LINKS] / YCHG_STAGES[_LINKS]
// build variants).  Both default to 4-warp CTAs with 3-stage rings (67 KB of
// shared memory): three CTAs per SM, so one scan fills the GPU and the CTAs of
// back-to-back scans interleave on an SM as they come and go.
#ifndef YCHG_WARPS_LINKS
#define YCHG_WARPS_LINKS 4
#endif
#ifndef YCHG_STAGES_LINKS
#define YCHG_STAGES_LINKS YCHG_STAGES
#endif
constexpr int kWarpsLinks = YCHG_WARPS_LINKS;
constexpr int kWarpsCounts = YCHG_WARPS;
constexpr int kStagesLinks = YCHG_STAGES_LINKS;
constexpr int kStagesCounts = YCHG_STAGES;
template <int NW, int ST>
struct ScanSmem {
    static constexpr int kStagesB = NW * ST * kStageBytes;
    static constexpr int kBar = NW * ST * 8;
    static constexpr int kAcc = NW * 16 * 32 * 4;
    static constexpr int kSum = NW * kSumPlanes * 32 * 4;
    static constexpr int kMisc = NW * 24 + 64;
    static constexpr int kTotal = kStagesB + kBar + kAcc + kSum + kMisc;
};
template <bool kLinks>
__host__ __device__ constexpr int scan_warps() { return kLinks ? kWarpsLinks : kWarpsCounts; }
template <bool kLinks>
__host__ __device__ constexpr int scan_stages() { return kLinks ? kStagesLinks : kStagesCounts; }
template <bool kLinks>
__host__ __device__ constexpr int scan_smem() { return ScanSmem<scan_warps<kLinks>(), scan_stages<kLinks>()>::kTotal; }

// What a strip's finisher publishes for the strips to its right: `status`
// packs the epoch, the number of change flags strictly inside the strip and the
// counts of its first and last column (counts < 2^21, i.e. height < 2^22).  The
// run and link totals carry the epoch too, so the three words need no ordering
// fence: a reader polls each word until its epoch matches.
struct StripRecord {
    unsigned long long status;  // epoch:12 | inside:10 | first:21 | last:21
    unsigned long long pad;
    unsigned long long runs;    // epoch:12 | sum of the strip's counts:52
    unsigned long long links;   // epoch:12 | K3 links of the strip's column pairs:52
};

// ----------------------------------------------------------------------------
// Launch parameters of one scan.  Cross-CTA bookkeeping is epoch-tagged or
// monotonic -- every segment numbers its scans with its own ticket, and all k
// segments of a strip agree on it -- so nothing is reset between scans and the
// launches are CUDA-graph replayable.
struct ScanParams {
    const uint8_t* bits;      // device image base (row-major packed bits)
    int64_t pitch;            // bytes between rows (multiple of 16 for TMA)
    int32_t width_img;        // columns present in the buffer (incl. a right halo)
    int32_t width_cnt;        // columns counted: [0, width_cnt)
    int32_t height;
    int32_t row_bytes;        // ceil(width_img / 8)
    int32_t n_strips;         // ceil(width_cnt / 1024)
    int32_t n_blocks;         // ceil(height / 32)
    int32_t seg_per_strip;    // k: row segments per strip
    int32_t n_segments;       // n_strips * k
    uint32_t mul2, mulnb;     // 2 and 1 << 25 as runtime values: keeps the b-word shifts on IMAD
    uint32_t mul1, mulm1;     // 1 and -1 as runtime values: keeps disjoint adds / subset subtracts on IMAD
    int32_t skip_same;        // 1: skip 32-row blocks identical to the row above (state is unchanged)
    int32_t ramp_boxes;       // TMA boxes a warp issues at its band's start (the rest after the first lands)
    // per scan parity (two halves: scan t+1 fills one while scan t's finishers read the other)
    uint32_t* part;           // [2][n_segments][512] per-segment u16x2 column counts
    uint32_t* sums;           // [2][n_segments][7][32] K3 band summaries (one per segment)
    unsigned long long* seg_links;    // [2][n_segments] links closed inside each segment
    unsigned long long* seg_ticket;   // [n_segments] scans started per segment (monotonic)
    unsigned long long* arrive;       // [2][n_strips] segments of the strip merged (monotonic, +k per scan)
    unsigned long long* fin_all;      // [1] strip finishes completed (monotonic)
    unsigned long long* fin_loaded;   // [2][n_strips] per half: 1 + the last scan whose inputs of that
                                      //   half the strip's finisher has read
    struct StripRecord* rec;  // [2][n_strips] published by each strip's finisher
    long long* totals;        // ychg_totals {total_runs, links, hyperedges, n_boundaries}
    int32_t* counts;          // [width_cnt] final per-column counts
    uint32_t* flags;          // [ceil(width_cnt/32)] change flags, bit j = column 32w+j
    int32_t* boundaries;      // [<= width_cnt] ascending boundary columns
    unsigned long long* dbg;  // optional [4][dbg_rows][32] %globaltimer stamps (diagnostics), or null
    int32_t dbg_rows;
    int32_t wait_inputs;      // 1: griddepcontrol.wait before the first image load (YCHG_PLAN_SYNC_INPUTS)
};

// Segment j of a strip covers row blocks [seg_first(j), seg_first(j+1)).
__host__ __device__ inline int seg_first_block(int j, int k, int n_blocks) {
    return static_cast<int>((static_cast<long long>(j) * n_blocks) / k);
}

// ----------------------------------------------------------------------------
// Small PTX helpers (mbarrier + TMA).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_addr(dst)), "l"(tmap), "r"(x), "r"(y), "r"(smem_addr(bar)) : "memory");
}

// ----------------------------------------------------------------------------
// Bit-sliced arithmetic.
//
// lop3<LUT>(a, b, c): one LOP3.LUT with truth table LUT over (a=0xF0, b=0xCC,
// c=0xAA).  Written explicitly so every boolean step of the hot loop is exactly
// one ALU instruction (ptxas does not always find the 3-input merges itself).
template <uint32_t kLut>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(kLut));
    return d;
}
//
// Carry-save adder: l = a ^ b ^ c, h = majority(a, b, c); two LOP3 each.
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
    h = lop3<0xE8>(a, b, c);  // majority
    l = lop3<0x96>(a, b, c);  // a ^ b ^ c
}

// 8 bit-planes (x[k] = bit k of 32 per-column counters) -> per-column bytes:
// after the call, byte L of x[p] is the 8-bit counter of the column at bit 8L+p.
// Three rounds of block swaps inside every byte lane (4x4, 2x2, 1x1).
__device__ __forceinline__ void transpose8x8_bytes(uint32_t (&x)[8]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t t = ((x[k] >> 4) ^ x[k + 4]) & 0x0F0F0F0Fu;
        x[k + 4] ^= t;
        x[k] ^= t << 4;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k & 2) continue;
        const uint32_t t = ((x[k] >> 2) ^ x[k + 2]) & 0x33333333u;
        x[k + 2] ^= t;
        x[k] ^= t << 2;
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const uint32_t t = ((x[k] >> 1) ^ x[k + 1]) & 0x55555555u;
        x[k + 1] ^= t;
        x[k] ^= t << 1;
    }
}

// Column (0..31, left to right inside its word) held by u16 lane `half` of
// accumulator acc[i] (i = 2p + kind) after flush_counts (which leaves the
// counter of word bit 8L+p in byte L of plane p).  The counts-only path keeps
// words in their raw little-endian load order -- bit 8L+p is bit p of byte L,
// column 8L + 7 - p (MSB-first bytes); the K3 path byte-swaps them to MSB-first
// words, where bit 8L+p is column 31 - (8L+p).
template <bool kMsbFirst = false>
__host__ __device__ inline int acc_column(int i, int half) {
    const int p = i >> 1, kind = i & 1;
    // kind 0 keeps byte lanes {0,2}, kind 1 keeps {1,3}; half selects the upper lane.
    const int L = kind + 2 * half;
    return kMsbFirst ? 31 - (8 * L + p) : 8 * L + 7 - p;
}

// ----------------------------------------------------------------------------
// K3 band summary.  Per column pair (c, c+1), the strip's
// 4-connected components are row intervals; a component is a decompose() link
// iff it contains exactly two runs (hypergraph.cpp:137-143: one run per column,
// mutually unique).  A band of rows [y0, y1) is summarised per pair by
//   O   a component is open across the band's top edge (the "head"),
//   E   the head closed inside the band,
//   h1,h2  head gained >= 1 / >= 2 new runs inside the band,
//   OE  a component is open across the bottom edge,
//   T2,T3  that component holds >= 2 / >= 3 runs (only meaningful when the
//          bottom component started inside the band).
// Links of components that start and end inside the band are counted directly.
struct BandSummary {
    uint32_t O, E, h1, h2, OE, T2, T3;
};

// Compose summary A (upper band) with B (the band directly below).  Returns the
// bit mask of pairs whose component straddling the A/B edge closes inside B as
// a link; `C` is the summary of the union.
__device__ __forceinline__ uint32_t compose_summary(const BandSummary& A, const BandSummary& B,
                                                    BandSummary& C) {
    const uint32_t Ap = A.O & ~A.E;   // A's head runs through all of A
    const uint32_t Bp = B.O & ~B.E;   // B's head runs through all of B
    const uint32_t s1 = A.h1 | B.h1;
    const uint32_t s2 = A.h2 | B.h2 | (A.h1 & B.h1);
    const uint32_t J = ~Ap & A.OE;    // A's bottom component is known and enters B
    // N_in = 1 + T2 + T3 (saturating); a link iff N_in + nf_B == 2.
    const uint32_t resolved =
        J & B.E & ((~A.T2 & B.h1 & ~B.h2) | (A.T2 & ~A.T3 & ~B.h1));
    C.O = A.O;
    C.E = (Ap & B.E) | (~Ap & A.E);
    C.h1 = (Ap & s1) | (~Ap & A.h1);
    C.h2 = (Ap & s2) | (~Ap & A.h2);
    C.OE = B.OE;
    C.T2 = (Bp & (A.T2 | B.h1)) | (~Bp & B.T2);
    C.T3 = (Bp & (A.T3 | (A.T2 & B.h1) | B.h2)) | (~Bp & B.T3);
    return resolved;
}

}  // namespace ychg_dev
