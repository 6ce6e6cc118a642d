// ychg_scan.cu -- the yCHG hot path on sm_100a: ONE kernel per scan, graph-
// capturable, chained to the next scan by programmatic dependent launch (PDL).
//
//   K1  per-column cut-vertex counts      (reference runscan.cpp:41-74,122-128)
//   K2  change flags + ascending boundary  (runscan.cpp:145-153)
//   K3  hyperedge total = runs - links     (hypergraph.cpp:94-170,192)
//
// The mask is cut into 1024-column strips (one 32-bit word per lane) and every
// strip into k row segments; CTA g owns segments g, g+G, ... (one each when the
// grid covers them; the planner sizes k per plan kind: about half a CTA per SM per
// scan for back-to-back scans, two per SM for an isolated one).  A segment is split
// into NW consecutive warp bands; each warp streams its band through its own TMA
// ring (cp.async.bulk.tensor, 32 rows x 144 B per stage: 128 B of the strip + a
// 16 B right halo), skips 32-row blocks equal to the row above, and runs K1 + K3
// bit-sliced in registers.  The CTA merges its warps in shared memory, writes one
// partial per segment (counts + K3 band summary + links) into a workspace
// double-buffered by scan parity, and counts itself in on the strip's arrival
// counter.  The LAST segment of a strip to arrive finishes the strip in the same
// CTA (no second kernel, no CTA waiting on a segment): it sums the k partials,
// composes the K3 summaries, publishes a strip record, derives its boundary
// offset and first-column flag from every record to its left (warp-parallel
// look-back), compacts the boundary list; the right-most strip writes totals.
//
// Consecutive scans overlap: every CTA triggers the next scan's launch right after
// drawing its tickets, so the next scan's CTAs take SM slots as this scan's
// retire.  Invariants: tickets drawn before the trigger (they then
// follow launch order); a segment's partial half is reused only after the
// finisher of the scan two back loaded it (fin_loaded); a strip record is
// rewritten only after every finisher of the scan two back is done, and the
// outputs only after every finisher of the previous scan is done (fin_all).
// Waits are deadlock-free: all CTAs of a scan are resident before the next scan
// launches (PDL trigger semantics), a CTA processes its segments in increasing
// order, and a finisher only waits on strips to its left or on older scans.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "ychg_device.cuh"
#include "ychg_kernels.h"

namespace ychg_dev {

// Per-lane streaming state.  Everything is bit-sliced over the 32 columns (or
// column pairs) of this lane's word.
struct LaneState {
    // K1: Harley-Seal carry-save planes (weights 1,2,4,8) + ripple planes 16..128.
    uint32_t ones, twos, fours, eights, u16, u32, u64, u128;
    uint32_t acc[16];          // u16x2 per-column totals (see acc_column)
    uint32_t pa, pb;           // previous row: column c and column c+1 bits
    uint32_t pab;              // pa & pb (K3)
    uint32_t praw;             // previous row's raw (load-order) word: the skip test compares raw words
    uint32_t mk3;              // valid column pairs of this word
    // K3
    uint32_t G2, G3;           // open component holds >= 2 / >= 3 runs
    uint32_t Hd, h1, h2;       // head still open / head gained >= 1 / >= 2 runs
    uint32_t links;            // links closed inside this lane's band
};

__device__ __forceinline__ void flush_counts(LaneState& s) {
    uint32_t x[8] = {s.ones, s.twos, s.fours, s.eights, s.u16, s.u32, s.u64, s.u128};
    transpose8x8_bytes(x);
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        s.acc[2 * p] += x[p] & 0x00FF00FFu;
        s.acc[2 * p + 1] += (x[p] >> 8) & 0x00FF00FFu;
    }
    s.ones = s.twos = s.fours = s.eights = s.u16 = s.u32 = s.u64 = s.u128 = 0;
}

// K3 pair step for one row (a = columns c, b = columns c+1 of this word).
// Components of the 2-column strip are row intervals; one continues into this
// row iff (a & pa) | (b & pb).  A new run can only join an open component on a
// row where both columns are set and exactly one of them was set above:
// f = a & b & (pa ^ pb).  N >= 2 <=> ab | (cont & G2); N >= 3 <=> (cont & G3) | (G2 & f).
// G2 implies pa | pb and contains pab (= pa & pb, the previous row's ab), so
// G2 & f == ab & G2 & ~pab: one LOP3, and f itself is never formed (7 LOP3/row).
// A component that closes with exactly two runs is a decompose() link
// (hypergraph.cpp:137-143).  Head pairs (open across the band's top edge) start
// "poisoned" at N >= 3 so their unknown-prefix component never counts here;
// kHead additionally tracks their new runs (h1, h2) until they close (Hd <= G2,
// so Hd & f == Hd & ab & ~pab likewise).  `apa` (a & pa) is handed back: K1's
// rise word a & ~pa is then a - apa, an IMAD.
template <bool kHead>
__device__ __forceinline__ uint32_t k3_step(uint32_t a, uint32_t b, LaneState& s, uint32_t& apa) {
    const uint32_t ab = a & b;
    apa = a & s.pa;
    const uint32_t cont = lop3<0xF8>(apa, b, s.pb);            // (a & pa) | (b & pb)
    const uint32_t lk = lop3<0x04>(cont, s.G2, s.G3);          // ~cont & G2 & ~G3
    if (kHead) {
        s.Hd &= cont;
        const uint32_t t = lop3<0x40>(s.Hd, ab, s.pab);        // Hd & ab & ~pab
        s.h2 = lop3<0xF8>(s.h2, s.h1, t);                      // h2 | (h1 & t)
        s.h1 |= t;
    }
    const uint32_t g2f = lop3<0x40>(ab, s.G2, s.pab);          // ab & G2 & ~pab == G2 & f
    const uint32_t g3 = lop3<0xF8>(g2f, cont, s.G3);           // (cont & G3) | (G2 & f)
    s.G2 = lop3<0xF8>(ab, cont, s.G2);                         // ab | (cont & G2)
    s.G3 = g3;
    s.pa = a;
    s.pb = b;
    s.pab = ab;
    return lk;
}

// The K3 path runs on MSB-first words (one PRMT per row): the right neighbour is
// then a << 1 with the next word's first bit shifted in, i.e. the MSB of the
// next byte nb -- IMAD(a, 2, umulhi(nb, 1 << 25)), no ALU op at all.
__device__ __forceinline__ uint32_t right_neighbour_msb(uint32_t a, uint32_t nb, uint32_t mul2, uint32_t mul25) {
    return a * mul2 + __umulhi(nb, mul25);
}

struct Muls {
    uint32_t m2, mnb, m1, mm1;  // 2, 1 << 25, 1, -1 (runtime values: ptxas keeps the IMADs)
};

// 32 rows from one TMA stage: 16 row pairs -> Harley-Seal tree -> ripple planes.
// Rises of one column are never in consecutive rows, so a row pair contributes
// (a0 & ~pa) | (a1 & ~a0) -- one LOP3 (moving it to the FMA pipe as
// (a0 - a0&pa) + (a1 - a1&a0) with k3_step's `apa` measured 1 % slower: -DYCHG_P_FMA).
// Links of one pair are likewise never in consecutive rows and are popcounted
// per row pair.
// kMask (strips with invalid column pairs -- the image's last column, or a
// multi-GPU strip's right halo): the right-hand column of an invalid pair is
// zeroed, so its components hold one run and never link.  Full strips skip it,
// which lets the two row links of a pair be added on the FMA pipe (they are
// disjoint bit sets) instead of a masked LOP3.
template <bool kLinks, bool kHead, bool kMask = false>
__device__ __forceinline__ void process_block(const uint8_t* __restrict__ stage, int lane, LaneState& s,
                                              const Muls& mu) {
    const uint8_t* p = stage + 4 * lane;
    uint32_t Pprev = 0, tA = 0, fA = 0, eA = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const uint8_t* r0 = p + (2 * q) * kBoxBytes;
        const uint8_t* r1 = r0 + kBoxBytes;
        const uint32_t raw0 = *reinterpret_cast<const uint32_t*>(r0);
        const uint32_t raw1 = *reinterpret_cast<const uint32_t*>(r1);
        uint32_t P;
        if (kLinks) {  // MSB-first words (bit 31-j = column j): b = a << 1 | next byte's MSB, FMA pipe
            const uint32_t a0 = __byte_perm(raw0, 0u, 0x0123u);
            const uint32_t a1 = __byte_perm(raw1, 0u, 0x0123u);
            uint32_t b0 = right_neighbour_msb(a0, r0[4], mu.m2, mu.mnb);
            uint32_t b1 = right_neighbour_msb(a1, r1[4], mu.m2, mu.mnb);
            if (kMask) {
                b0 &= s.mk3;
                b1 &= s.mk3;
            }
            uint32_t apa0, apa1;
            const uint32_t pa_old = s.pa;
            const uint32_t l0 = k3_step<kHead>(a0, b0, s, apa0);
            const uint32_t l1 = k3_step<kHead>(a1, b1, s, apa1);
            // l0 | l1 == l0 + l1 (disjoint); IMADs keep both adds off the ALU pipe
            s.links = __popc(l0 * mu.m1 + l1) * mu.m1 + s.links;
#ifdef YCHG_P_FMA  // A/B variant: the rise word as (a0 - a0&pa) + (a1 - a1&a0), 3 IMADs (1 % slower)
            P = (apa0 * mu.mm1 + a0) * mu.m1 + (apa1 * mu.mm1 + a1);
#else
            P = lop3<0x3A>(a0, pa_old, a1);  // (a0 & ~pa) | (a1 & ~a0)
#endif
        } else {
            P = lop3<0x3A>(raw0, s.pa, raw1);  // (a0 & ~pa) | (a1 & ~a0)
            s.pa = raw1;
        }
#ifdef YCHG_DIAG_NO_K1  // microbenchmark-only: K3 alone (counts wrong)
        s.ones ^= P;
        continue;
#endif
        if ((q & 1) == 0) {
            Pprev = P;
            continue;
        }
        const int m = q >> 1;  // 0..7
        uint32_t t;
        csa(t, s.ones, s.ones, Pprev, P);
        if ((m & 1) == 0) {
            tA = t;
            continue;
        }
        uint32_t f;
        csa(f, s.twos, s.twos, tA, t);
        if ((m & 2) == 0) {
            fA = f;
            continue;
        }
        uint32_t e;
        csa(e, s.fours, s.fours, fA, f);
        if ((m & 4) == 0) {
            eA = e;
            continue;
        }
        uint32_t sixteens;
        csa(sixteens, s.eights, s.eights, eA, e);
        // ripple-add the 16s bit into planes 16..128 (<= 15 blocks between flushes)
        const uint32_t c1 = s.u16 & sixteens;
        const uint32_t c2 = s.u32 & c1;
        const uint32_t c3 = s.u64 & c2;
        s.u16 ^= sixteens;
        s.u32 ^= c1;
        s.u64 ^= c2;
        s.u128 ^= c3;
    }
    if (kLinks) s.praw = *reinterpret_cast<const uint32_t*>(p + 31 * kBoxBytes);
}

// True (warp-uniform) iff every row of the stage equals the row above it for
// every word of the warp AND for the right-halo bit lane 31's pairs read: then
// K1 sees no rise, and every K3 plane (cont == a|b, G2, G3, Hd, h1, h2, pa, pb)
// maps to itself, so the block is a no-op and is skipped.  Rows 0..1 are tested
// first, so a block that changes early (dense content) pays two compares.
// `phalo` carries the halo byte of the row above (row 31 of the previous block).
__device__ __forceinline__ bool block_unchanged(const uint8_t* __restrict__ stage, int lane, uint32_t praw,
                                                uint32_t& phalo) {
    const uint8_t* p = stage + 4 * lane;
    // right halo column (bit 7 of the halo's first byte): lane L holds row L
    const uint32_t hb = stage[lane * kBoxBytes + kStripBytes];
    uint32_t hprev = __shfl_up_sync(0xFFFFFFFFu, hb, 1);
    if (lane == 0) hprev = phalo;
    // (x ^ y) | (z ^ x) = lop3 0x7E: two row compares per LOP3; 0xFE = 3-way OR.
    // Rows 0..1 first: a block that changes there (random masks) pays 2 loads + 2 LOP3.
    const uint32_t x0 = *reinterpret_cast<const uint32_t*>(p);
    const uint32_t x1 = *reinterpret_cast<const uint32_t*>(p + kBoxBytes);
    uint32_t d = lop3<0xFE>(lop3<0x28>(hb, hprev, 0x80u), lop3<0x7E>(x0, praw, x1), 0u);
    if (__any_sync(0xFFFFFFFFu, d != 0u)) return false;
    uint32_t prev = x1;
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        uint32_t y[6];
#pragma unroll
        for (int r = 0; r < 6; ++r) y[r] = *reinterpret_cast<const uint32_t*>(p + (2 + 6 * c + r) * kBoxBytes);
        d = lop3<0xFE>(d, lop3<0x7E>(y[0], prev, y[1]), lop3<0x7E>(y[2], y[1], y[3]));
        d = lop3<0xFE>(d, lop3<0x7E>(y[4], y[3], y[5]), 0u);
        prev = y[5];
    }
    const bool same = !__any_sync(0xFFFFFFFFu, d != 0u);
    phalo = __shfl_sync(0xFFFFFFFFu, hb, 31);
    return same;
}

// Valid-bit mask of word `gw` for `limit` columns: columns j < limit-32*gw, MSB-first.
__device__ __forceinline__ uint32_t word_mask(int gw, int limit) {
    const int n = limit - 32 * gw;
    if (n >= 32) return 0xFFFFFFFFu;
    if (n <= 0) return 0u;
    return ~(0xFFFFFFFFu >> n);
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Diagnostics stamps: dbg layout [scan % kStampRing][CTA][32 slots] (ns, %globaltimer).
//   0 CTA entry, 1 first segment streamed (all warps), 2 first segment arrived,
//   3 strip finish entered, 4 strip finish left, 5 CTA exit, 6 first stage ready
//   (warp 0), 7 warp 0's band streamed, 8 scan number + 1
__device__ __forceinline__ void stamp(const ScanParams& prm, unsigned long long scan, int slot,
                                      unsigned long long v) {
    if (prm.dbg)
        prm.dbg[(static_cast<int64_t>(scan % kStampRing) * prm.dbg_rows + blockIdx.x) * 32 + slot] = v;
}

__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


__device__ __forceinline__ BandSummary load_summary(const uint32_t* a, int lane) {
    return BandSummary{a[lane], a[32 + lane], a[64 + lane], a[96 + lane], a[128 + lane], a[160 + lane], a[192 + lane]};
}

__device__ __forceinline__ void store_summary(uint32_t* a, int lane, const BandSummary& C) {
    a[lane] = C.O;
    a[32 + lane] = C.E;
    a[64 + lane] = C.h1;
    a[96 + lane] = C.h2;
    a[128 + lane] = C.OE;
    a[160 + lane] = C.T2;
    a[192 + lane] = C.T3;
}

// Order-preserving composition of n >= 1 band summaries stored in shared memory
// (slot i = 7 planes x 32 lanes at base + i*224): warp w composes the slots of
// its contiguous chunk in registers, one __syncthreads, then warp 0 composes the
// chunk results.  A chain in registers beats a log-depth tree here: every tree
// level would cost a CTA barrier, and one compose is ~30 ALU ops.  Returns, in
// warp 0 only, the composite (every lane its word) and the number of links
// resolved at the junctions (all lanes); `red` is NW scratch words.  Must be
// called by the whole CTA.
template <int NW>
__device__ BandSummary chain_compose(const uint32_t* base, int n, unsigned long long* red,
                                     unsigned long long& links) {
    constexpr int kSW = kSumPlanes * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long mine = 0;
    const int c0 = (warp * n) / NW, c1 = ((warp + 1) * n) / NW;
    BandSummary A{};
    if (c1 > c0) {
        A = load_summary(base + c0 * kSW, lane);
        for (int i = c0 + 1; i < c1; ++i) {
            const BandSummary B = load_summary(base + i * kSW, lane);
            BandSummary C;
            mine += __popc(compose_summary(A, B, C));
            A = C;
        }
    }
    __shared__ uint32_t chunk[NW][kSumPlanes * 32];
    if (c1 > c0) store_summary(chunk[warp], lane, A);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    links = 0;
    if (warp == 0) {
        bool first = true;
        unsigned long long jl = 0;
        for (int w = 0; w < NW; ++w) {
            if (((w + 1) * n) / NW <= (w * n) / NW) continue;
            const BandSummary B = load_summary(chunk[w], lane);
            if (first) {
                A = B;
                first = false;
            } else {
                BandSummary C;
                jl += __popc(compose_summary(A, B, C));
                A = C;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) jl += __shfl_xor_sync(0xFFFFFFFFu, jl, o);
        for (int w = 0; w < NW; ++w) jl += red[w];
        links = jl;
    }
    return A;
}

// Shared-memory scratch of a strip finish (overlaid on the CTA's idle TMA ring).
template <int NW>
struct FinishSmem {
    int32_t sc[kStripCols];       // counts of the strip's columns
    uint32_t fw[kStripWords];     // change-flag words of the strip (inside flags only)
    int wpre[kStripWords];        // exclusive prefix of popc(fw)
    long long red[NW];
    unsigned long long red2[NW];
    long long base;
    long long n_total;            // boundaries up to and including this strip (right-most: the total)
    long long tot_runs, tot_links;  // right-most strip: totals over every strip
    unsigned long long seglinks;  // links closed inside the strip's segments
    uint32_t edge;                // flag of the strip's first column
};
template <int NW>
__host__ __device__ constexpr int finish_smem_bytes() {
    return ((static_cast<int>(sizeof(FinishSmem<NW>)) + 127) / 128) * 128 + (kFinishChunk + 1) * kSumPlanes * 32 * 4;
}

__device__ __forceinline__ unsigned long long pack_strip_status(uint32_t epoch, uint32_t inside, int32_t first,
                                                                int32_t last) {
    return (static_cast<unsigned long long>(epoch & 0xFFFu) << 52) |
           (static_cast<unsigned long long>(inside & 0x3FFu) << 42) |
           (static_cast<unsigned long long>(static_cast<uint32_t>(first) & 0x1FFFFFu) << 21) |
           (static_cast<unsigned long long>(static_cast<uint32_t>(last) & 0x1FFFFFu));
}

// Finish strip s of scan `scan_no` (run by the CTA whose segment arrived last):
// counts, K3 stitch, flags, boundary compaction, totals.  One batch of loads
// (the k segment partials of the strip, their links and K3 summaries, all in
// flight together), one release of the strip record (flags strictly inside the
// strip + counts of its first and last column), one warp-parallel acquire of
// every record to the left -- from which the boundary offset AND this strip's
// first-column flag (counts[c0] vs counts[c0-1], runscan.cpp:147) follow -- then
// fire-and-forget writes.  Records are double-buffered by scan parity (rewritten
// only once the scan two back is done); only the output writes wait for the
// previous scan's finishers (the outputs are shared by consecutive scans).
template <bool kLinks, int NW>
__device__ void finish_strip(const ScanParams& prm, int s, unsigned long long scan_no, uint8_t* scratch) {
    constexpr int T = NW * 32;
    FinishSmem<NW>& fs = *reinterpret_cast<FinishSmem<NW>*>(scratch);
    uint32_t* ssum = reinterpret_cast<uint32_t*>(scratch + ((sizeof(FinishSmem<NW>) + 127) / 128) * 128);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k = prm.seg_per_strip;
    const int g0 = s * k;
    const int S = prm.n_strips;
    constexpr int kSumWords = kSumPlanes * 32;
    constexpr int kSumVec = kSumWords / 4;  // uint4 per summary
    const uint32_t epoch = static_cast<uint32_t>(scan_no % 4095ull) + 1u;
    const int64_t par = static_cast<int64_t>(scan_no & 1ull);
    const int64_t G = prm.n_segments;
    const uint32_t* part_p = prm.part + (par * G + g0) * 512;
    const uint32_t* sums_p = prm.sums + (par * G + g0) * kSumWords;
    StripRecord* recs = prm.rec + par * S;
    if (tid == 0) {
        stamp(prm, scan_no, 3, globaltimer());
        stamp(prm, scan_no, 9, scan_no + 1);
    }

    // (1) one batch of loads: the k partials (128 uint4 each; thread t sums uint4 t
    //     of every segment, kB segments in flight at once), the first chunk of K3
    //     summaries (straight to smem) and the segment links; tid 0 also reads the
    //     finish counter for the two waits below, overlapped with the batch.
    static_assert(T == 128 || T == 256, "partial layout: 512 words over the CTA");
    constexpr int kWPT = 512 / T;  // partial words per thread (one 16 B / 8 B load per segment)
    using VecT = typename std::conditional<kWPT == 4, uint4, uint2>::type;
    constexpr int kB = 8;          // segments per load batch
    constexpr int kSV = (kFinishChunk * kSumVec + T - 1) / T;  // uint4 of the summary chunk per thread
    uint32_t lo[kWPT], hi[kWPT];
#pragma unroll
    for (int q = 0; q < kWPT; ++q) lo[q] = hi[q] = 0;
    const int n0 = k < kFinishChunk ? k : kFinishChunk;
    uint4 sv[kSV];
    if (kLinks) {  // all of the chunk's loads in flight before the first use
        const uint4* src = reinterpret_cast<const uint4*>(sums_p);
#pragma unroll
        for (int r = 0; r < kSV; ++r) {
            const int i = tid + r * T;
            sv[r] = i < n0 * kSumVec ? __ldcg(src + i) : make_uint4(0u, 0u, 0u, 0u);
        }
    }
    unsigned long long sl = 0;
    if (kLinks && warp == 0)
        for (int j = lane; j < k; j += 32) sl += __ldcg(prm.seg_links + par * G + g0 + j);
    const VecT* pv = reinterpret_cast<const VecT*>(part_p);
    for (int g = 0; g < k; g += kB) {
        VecT x[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) x[u] = (g + u < k) ? __ldcg(pv + (g + u) * T + tid) : VecT{};
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(&x[u]);
#pragma unroll
            for (int q = 0; q < kWPT; ++q) {
                lo[q] += w[q] & 0xFFFFu;
                hi[q] += w[q] >> 16;
            }
        }
    }
    if (kLinks) {
#pragma unroll
        for (int r = 0; r < kSV; ++r) {
            const int i = tid + r * T;
            if (i < n0 * kSumVec) reinterpret_cast<uint4*>(ssum)[i] = sv[r];
        }
    }
    unsigned long long fa = 0;
    if (tid == 0) fa = ld_acquire(prm.fin_all);
    if (kLinks && warp == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xFFFFFFFFu, sl, o);
        if (lane == 0) fs.seglinks = sl;
    }
    // partial word idx = 32 i + ln holds the u16 counters of columns 32 ln + acc_column(i, 0 / 1)
#pragma unroll
    for (int q = 0; q < kWPT; ++q) {
        const int idx = kWPT * tid + q;
        const int i = idx >> 5, ln = idx & 31;
        fs.sc[32 * ln + acc_column<kLinks>(i, 0)] = static_cast<int32_t>(lo[q]);
        fs.sc[32 * ln + acc_column<kLinks>(i, 1)] = static_cast<int32_t>(hi[q]);
    }
    __syncthreads();
    if (tid == 0) stamp(prm, scan_no, 16, globaltimer());

    // (2) flags strictly inside the strip (columns 1..1023), run total
    const int nwords = (prm.width_cnt + 31) >> 5;
    long long local_sum = 0;
    for (int wi = warp; wi < kStripWords; wi += NW) {
        const int col = wi * 32 + lane;
        const int gc = s * kStripCols + col;
        const bool valid = gc < prm.width_cnt;
        const int32_t c = fs.sc[col];
        const bool f = valid && col > 0 && c != fs.sc[col - 1];
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
        if (lane == 0) fs.fw[wi] = m;
        if (valid) local_sum += c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_sum += __shfl_xor_sync(0xFFFFFFFFu, local_sum, o);
    if (lane == 0) fs.red[warp] = local_sum;
    // This parity's records (status, runs, links) were last read by the
    // scan two back: its finishers must all be done before any of them is
    // rewritten (normally long ago).
    if (tid == 0 && scan_no >= 2) {
        const unsigned long long need = (scan_no - 1) * static_cast<unsigned long long>(S);
        while (fa < need) fa = ld_acquire(prm.fin_all);
    }
    __syncthreads();
    if (tid == 0) stamp(prm, scan_no, 17, globaltimer());

    const bool last_strip = (s == S - 1);
    StripRecord* rec = recs + s;
    int inside = 0;
    const int32_t first = fs.sc[0];
    if (warp == 0) {
        // (3) boundary prefix of the strip's flag words
        const int c = __popc(fs.fw[lane]);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        fs.wpre[lane] = incl - c;
        inside = __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
    // The look-back's first loads (records of up to 32 strips to the left) go out
    // now and land while the K3 summaries are composed.  The status word is one
    // packed value validated by its epoch, so relaxed loads suffice for it.
    unsigned long long lb = 0;
    if (warp == 0 && lane < s) lb = ld_relaxed(&recs[lane].status);
    // (2b) K3: stitch the strip's segment summaries top to bottom, kFinishChunk at
    // a time (warp 0 carries the running composite between chunks); strip_links
    // is complete in warp 0
    unsigned long long strip_links = 0;
    if (kLinks) {
        unsigned long long jl = 0;
        BandSummary R = chain_compose<NW>(ssum, n0, fs.red2, jl);
        strip_links = jl;
        for (int c0 = n0; c0 < k; c0 += kFinishChunk) {
            const int n = k - c0 < kFinishChunk ? k - c0 : kFinishChunk;
            __syncthreads();  // the previous chain_compose's readers are done
            const uint4* src = reinterpret_cast<const uint4*>(sums_p + static_cast<int64_t>(c0) * kSumWords);
            for (int i = tid; i < n * kSumVec; i += T) reinterpret_cast<uint4*>(ssum)[i] = __ldcg(src + i);
            __syncthreads();
            const BandSummary B = chain_compose<NW>(ssum, n, fs.red2, jl);
            if (warp == 0) {
                BandSummary C;
                unsigned long long m = __popc(compose_summary(R, B, C));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
                strip_links += jl + m;
                R = C;
            }
        }
        if (warp == 0) {
            // close whatever is still open at row H (virtual background row)
            unsigned long long m = __popc(R.OE & R.T2 & ~R.T3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
            strip_links += m;
        }
    }
    if (tid == 0) stamp(prm, scan_no, 18, globaltimer());

    if (warp == 0) {
        // (4) publish the strip record -- runs and links, then the status word with
        // one release (the strips to the right wait on it; the right-most strip
        // reads every record's runs / links after acquiring its status) -- and
        // acquire every record to the left: boundary offset + first-column flag
        if (lane == 0) {
            long long runs = 0;
            for (int w = 0; w < NW; ++w) runs += fs.red[w];
            // three self-validating words (each carries the scan epoch): no fence
            // orders them, a reader polls each until its epoch matches
            const unsigned long long tag = static_cast<unsigned long long>(epoch & 0xFFFu) << 52;
            st_relaxed(&rec->runs, tag | static_cast<unsigned long long>(runs));
            st_relaxed(&rec->links, tag | (strip_links + (kLinks ? fs.seglinks : 0ull)));
            st_relaxed(&rec->status, pack_strip_status(epoch, inside, first, fs.sc[kStripCols - 1]));
        }
        long long off = 0, runs_l = 0, links_l = 0;
        int32_t carry_last = 0;  // last(j-1) entering each chunk; last(-1) := 0
        for (int jb = 0; jb < s; jb += 32) {
            const int j = jb + lane;
            const bool act = j < s;
            unsigned long long st = jb == 0 ? lb : 0ull;
            bool ok = !act || (jb == 0 && static_cast<uint32_t>(lb >> 52) == (epoch & 0xFFFu));
            while (!__all_sync(0xFFFFFFFFu, ok)) {
                if (!ok) {
                    st = ld_relaxed(&recs[j].status);
                    ok = static_cast<uint32_t>(st >> 52) == (epoch & 0xFFFu);
                }
            }
            const int32_t fj = static_cast<int32_t>((st >> 21) & 0x1FFFFFu);
            const int32_t lj = static_cast<int32_t>(st & 0x1FFFFFu);
            int32_t prev_last = __shfl_up_sync(0xFFFFFFFFu, lj, 1);
            if (lane == 0) prev_last = carry_last;
            if (act) off += static_cast<long long>((st >> 42) & 0x3FFu) + (fj != prev_last ? 1 : 0);
            carry_last = __shfl_sync(0xFFFFFFFFu, lj, (s - 1 - jb) < 31 ? (s - 1 - jb) : 31);
            if (last_strip) {  // every record's epoch-tagged run and link words
                unsigned long long rw = 0, lw = 0;
                bool rok = !act, lok = !act;
                while (!__all_sync(0xFFFFFFFFu, rok && lok)) {
                    if (!rok) {
                        rw = ld_relaxed(&recs[j].runs);
                        rok = static_cast<uint32_t>(rw >> 52) == (epoch & 0xFFFu);
                    }
                    if (!lok) {
                        lw = ld_relaxed(&recs[j].links);
                        lok = static_cast<uint32_t>(lw >> 52) == (epoch & 0xFFFu);
                    }
                }
                if (act) {
                    runs_l += static_cast<long long>(rw & 0xFFFFFFFFFFFFFull);
                    links_l += static_cast<long long>(lw & 0xFFFFFFFFFFFFFull);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xFFFFFFFFu, off, o);
            runs_l += __shfl_xor_sync(0xFFFFFFFFu, runs_l, o);
            links_l += __shfl_xor_sync(0xFFFFFFFFu, links_l, o);
        }
        if (lane == 0) {
            stamp(prm, scan_no, 19, globaltimer());
            fs.edge = (first != carry_last) ? 1u : 0u;
            fs.base = off;
            fs.n_total = off + static_cast<long long>(first != carry_last) + inside;
            if (last_strip) {  // this strip's own record + every record to the left
                long long runs = 0;
                for (int w = 0; w < NW; ++w) runs += fs.red[w];
                fs.tot_runs = runs_l + runs;
                fs.tot_links = links_l + static_cast<long long>(strip_links + (kLinks ? fs.seglinks : 0ull));
            }
        }
    }
    // (5) the outputs are shared with the previous scan: its finishers must be done
    if (tid == 0 && scan_no >= 1) {
        const unsigned long long need = scan_no * static_cast<unsigned long long>(S);
        while (fa < need) fa = ld_acquire(prm.fin_all);
    }
    __syncthreads();
    if (tid == 0) stamp(prm, scan_no, 20, globaltimer());
    if (tid == 0 && last_strip) prm.totals[3] = fs.n_total;
    for (int col = tid; col < kStripCols; col += T) {
        const int gc = s * kStripCols + col;
        if (gc < prm.width_cnt) prm.counts[gc] = fs.sc[col];
    }
    // flags out + ordered compaction (the first-column flag, if set, comes first)
    const uint32_t e = fs.edge;
    if (tid == 0 && e) prm.boundaries[fs.base] = s * kStripCols;
    for (int wi = warp; wi < kStripWords; wi += NW) {
        const int w = s * kStripWords + wi;
        const uint32_t m = fs.fw[wi];
        if (lane == 0 && w < nwords) prm.flags[w] = m | (wi == 0 ? e : 0u);
        if ((m >> lane) & 1u)
            prm.boundaries[fs.base + e + fs.wpre[wi] + __popc(m & ((1u << lane) - 1u))] = w * 32 + lane;
    }

    // (6) the right-most strip writes the run / link / hyperedge totals
    if (last_strip && tid == 0) {
        prm.totals[0] = fs.tot_runs;
        prm.totals[1] = kLinks ? fs.tot_links : 0;
        prm.totals[2] = kLinks ? fs.tot_runs - fs.tot_links : -1;
    }
    if (tid == 0) stamp(prm, scan_no, 21, globaltimer());
    __syncthreads();
    if (tid == 0) {
        stamp(prm, scan_no, 4, globaltimer());
        stamp(prm, scan_no, 10, scan_no + 1);
        // one fence for both: this half's partials are consumed (scan t+2 may refill
        // them), and every record / output write of this finish precedes fin_all
        __threadfence();
        st_relaxed(prm.fin_loaded + par * S + s, scan_no + 1);
        atomicAdd(prm.fin_all, 1ull);
    }
}

// ----------------------------------------------------------------------------
// Row-block range [wb0, wb0 + nb) of warp `warp`'s band in segment `seg`.
template <int NW>
__device__ __forceinline__ void band_of(const ScanParams& prm, int seg, int warp, int& strip, int& nseg, int& wb0,
                                        int& nb) {
    const int k = prm.seg_per_strip;
    strip = seg / k;
    const int j = seg - strip * k;
    const int sb0 = seg_first_block(j, k, prm.n_blocks);
    nseg = seg_first_block(j + 1, k, prm.n_blocks) - sb0;
    wb0 = sb0 + (warp * nseg) / NW;
    nb = sb0 + ((warp + 1) * nseg) / NW - wb0;
}

// Halo row wb0*32 - 1 of a band (the reference's previous row, runscan.cpp:45;
// zero above row 0): this lane's 4 bytes and the next byte.
__device__ __forceinline__ void load_halo_row(const ScanParams& prm, int wb0, int x0, int lane, uint32_t& raw,
                                              uint32_t& nbyte) {
    const int y0 = wb0 * kBlockRows;
    raw = nbyte = 0;
    if (y0 > 0) {
        const uint8_t* row = prm.bits + static_cast<int64_t>(y0 - 1) * prm.pitch;
        const int c = x0 + 4 * lane;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (c + q < prm.row_bytes) raw |= static_cast<uint32_t>(__ldg(row + c + q)) << (8 * q);
        if (c + 4 < prm.row_bytes) nbyte = __ldg(row + c + 4);
    }
}

// Lane 0: fill the first `n` stages of the warp's TMA ring for a band (blocks
// i0 .. i0+n-1 of the band into stages it+i0 ...).
template <int kS>
__device__ __forceinline__ void kick_ring(const CUtensorMap* tmap, uint8_t* my_stages, uint64_t* my_bars,
                                          uint32_t it, int x0, int wb0, int nb, int i0 = 0, int n = kS) {
    const int npre = nb < i0 + n ? nb : i0 + n;
    for (int i = i0; i < npre; ++i) {
        const int st = (it + i) % kS;
        mbar_arrive_expect_tx(&my_bars[st], kStageBytes);
        tma_load_2d(my_stages + st * kStageBytes, tmap, &my_bars[st], x0, (wb0 + i) * kBlockRows);
    }
}

#ifndef YCHG_MIN_CTAS_PER_SM  // A/B builds only: 4 (with YCHG_STAGES=2) caps registers at 128 for 4 CTAs/SM
#define YCHG_MIN_CTAS_PER_SM 1
#endif
template <bool kLinks, int NW = scan_warps<kLinks>()>
__global__ void __launch_bounds__(NW * 32, YCHG_MIN_CTAS_PER_SM)
ychg_scan_kernel(const __grid_constant__ CUtensorMap tmap, const ScanParams prm) {
    constexpr int kS = scan_stages<kLinks>();  // TMA ring depth of this path
    constexpr int T = NW * 32;
    using L = ScanSmem<NW, kS>;
    static_assert(finish_smem_bytes<NW>() <= L::kStagesB, "strip finish scratch must fit in the TMA ring");
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kStagesB);
    uint32_t* accs = reinterpret_cast<uint32_t*>(smem + L::kStagesB + L::kBar);
    uint32_t* sums = accs + NW * 16 * 32;
    unsigned long long* wlinks = reinterpret_cast<unsigned long long*>(sums + NW * kSumPlanes * 32);
    int* misc = reinterpret_cast<int*>(wlinks + 2 * NW);  // [0] last-arrival flag

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const unsigned long long t_entry = globaltimer();
    uint8_t* my_stages = stages + warp * kS * kStageBytes;
    uint64_t* my_bars = bars + warp * kS;
    const bool have_seg = static_cast<int>(blockIdx.x) < prm.n_segments;
    const int ramp = (prm.ramp_boxes >= 1 && prm.ramp_boxes < kS) ? prm.ramp_boxes : kS;  // boxes issued at a band's start

    // Each warp owns its ring: lane 0 initialises the warp's barriers and -- unless
    // the image is still being written by the preceding kernel -- starts the first
    // band's loads right away, so the TMA round trip overlaps the ticket draw.
    uint32_t halo_raw = 0, halo_nb = 0;  // the first band's halo row (loaded with the first boxes)
    {
        int strip = 0, nseg = 0, wb0 = 0, nb = 0;
        if (have_seg) band_of<NW>(prm, blockIdx.x, warp, strip, nseg, wb0, nb);
        if (lane == 0) {
            for (int i = 0; i < kS; ++i) mbar_init(&my_bars[i], 1);
            fence_proxy_async();
            if (have_seg && !prm.wait_inputs)
                kick_ring<kS>(&tmap, my_stages, my_bars, 0u, strip * kStripBytes, wb0, nb, 0, ramp);
        }
        // the halo row's loads overlap the TMA round trip and the ticket atomic below
        if (have_seg && nb > 0 && !prm.wait_inputs) load_halo_row(prm, wb0, strip * kStripBytes, lane, halo_raw, halo_nb);
    }
    // This CTA's scan number for each of its segments, drawn BEFORE triggering the
    // next scan's launch: tickets then follow launch order even when consecutive
    // scans' CTAs overlap.
    __shared__ unsigned long long seg_tick[kMaxSegPerCta];
    if (tid == 0) {
        int i = 0;
        for (int sg = blockIdx.x; sg < prm.n_segments && i < kMaxSegPerCta; sg += gridDim.x, ++i)
            seg_tick[i] = atomicAdd(prm.seg_ticket + sg, 1ull);
    }
    __syncthreads();
    // Let the next scan launch now: its CTAs take SM slots as ours retire.
    asm volatile("griddepcontrol.launch_dependents;");
    // A plan whose image is written by the immediately preceding kernel (host
    // path: re-pitch / PNM pack) waits for that grid's completion and memory
    // flush before its first load; back-to-back scans read images written long before.
    if (prm.wait_inputs) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (have_seg) {
            int strip, nseg, wb0, nb;
            band_of<NW>(prm, blockIdx.x, warp, strip, nseg, wb0, nb);
            if (lane == 0) kick_ring<kS>(&tmap, my_stages, my_bars, 0u, strip * kStripBytes, wb0, nb, 0, ramp);
            if (nb > 0) load_halo_row(prm, wb0, strip * kStripBytes, lane, halo_raw, halo_nb);
        }
    }
    if (tid == 0 && have_seg) stamp(prm, seg_tick[0], 0, t_entry);

    uint32_t it = 0;  // blocks consumed by this warp so far (stage = it % kS)
    const Muls mu{prm.mul2, prm.mulnb, prm.mul1, prm.mulm1};

    int seg_i = 0;
    for (int seg = blockIdx.x; seg < prm.n_segments; seg += gridDim.x, ++seg_i) {
        int strip, nseg, wb0, nb;
        band_of<NW>(prm, seg, warp, strip, nseg, wb0, nb);
        const int x0 = strip * kStripBytes;
        const int gw = strip * kStripWords + lane;
        const unsigned long long scan_idx = seg_tick[seg_i];

        LaneState s;
        s.ones = s.twos = s.fours = s.eights = s.u16 = s.u32 = s.u64 = s.u128 = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s.acc[i] = 0;
        s.mk3 = word_mask(gw, min(prm.width_cnt, prm.width_img - 1));  // MSB-first, like the K3 words
        // every column pair of this warp's strip valid (warp-uniform): no per-row mask
        const bool full = !kLinks || __all_sync(0xFFFFFFFFu, s.mk3 == 0xFFFFFFFFu);
        s.h1 = s.h2 = 0;
        s.links = 0;
        s.pa = s.pb = s.pab = s.praw = 0;
        uint32_t O = 0;

        if (nb > 0) {
            if (seg_i > 0 && lane == 0) kick_ring<kS>(&tmap, my_stages, my_bars, it, x0, wb0, nb, 0, ramp);
            // Halo row y0-1 (the reference's prev row, runscan.cpp:45; zero above row 0),
            // for the first segment already loaded at CTA entry
            uint32_t raw = halo_raw, nbyte = halo_nb;
            if (seg_i > 0) load_halo_row(prm, wb0, x0, lane, raw, nbyte);
            s.praw = raw;
            uint32_t phalo = __shfl_sync(0xFFFFFFFFu, nbyte, 31);  // right-halo byte of the row above
            s.pa = kLinks ? __byte_perm(raw, 0u, 0x0123u) : raw;     // word order of process_block<kLinks>
            s.pb = right_neighbour_msb(s.pa, nbyte, prm.mul2, prm.mulnb);
            O = kLinks ? (s.pa | s.pb) : 0u;
            s.Hd = O;
            s.G2 = s.G3 = O;  // poisoned: the head's own closing is never a local link
            s.pab = s.pa & s.pb;

            int since_flush = 0;
            int fails = 0, untested = 0;  // unchanged-block test back-off (warp-uniform)
            for (int bi = 0; bi < nb; ++bi) {
                const int st = it % kS;
                mbar_wait(&my_bars[st], (it / kS) & 1u);
                if (bi == 0) {
                    // a short ramp (ramp_boxes < kS) gets each warp's first box back sooner
                    // when every CTA starts at once; the rest of the ring follows it
                    if (lane == 0 && ramp < kS) kick_ring<kS>(&tmap, my_stages, my_bars, it, x0, wb0, nb, ramp, kS - ramp);
                    if (tid == 0 && seg_i == 0) stamp(prm, scan_idx, 6, globaltimer());
                }
                const uint8_t* sp = my_stages + st * kStageBytes;
                // The unchanged-block test backs off on dense content: after f
                // consecutive changed blocks the next 2^(f-1) - 1 blocks are not tested
                // (a random mask pays ~5 tests per band; a banded one, whose changed
                // blocks are isolated, still tests every block).
                bool skip = false;
                if (kLinks && prm.skip_same) {
                    if (untested > 0) {
                        --untested;
                    } else if (block_unchanged(sp, lane, s.praw, phalo)) {
                        skip = true;
                        fails = 0;
                    } else {
                        fails = fails < 5 ? fails + 1 : 5;
                        untested = (1 << (fails - 1)) - 1;
                    }
                }
                if (!skip) {
#ifdef YCHG_NO_HEAD  // diagnostics build: never take the head-mode block (wrong results, timing only)
                    if (false)
#else
                    if (kLinks && __any_sync(0xFFFFFFFFu, (s.Hd & s.mk3) != 0u))
#endif
                    {
                        if (full) process_block<kLinks, true, false>(sp, lane, s, mu);
                        else process_block<kLinks, true, true>(sp, lane, s, mu);
                    } else {
                        if (full) process_block<kLinks, false, false>(sp, lane, s, mu);
                        else process_block<kLinks, false, true>(sp, lane, s, mu);
                    }
                    if (kLinks && prm.skip_same) phalo = sp[31 * kBoxBytes + kStripBytes];
                }
                __syncwarp();
                if (lane == 0 && bi + kS < nb) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&my_bars[st], kStageBytes);
                    tma_load_2d(my_stages + st * kStageBytes, &tmap, &my_bars[st], x0, (wb0 + bi + kS) * kBlockRows);
                }
                ++it;
                if (++since_flush == kFlushBlocks) {
                    flush_counts(s);
                    since_flush = 0;
                }
            }
            flush_counts(s);
            if (tid == 0 && seg_i == 0) stamp(prm, scan_idx, 7, globaltimer());

            if (kLinks) {
                const uint32_t m = s.mk3;
                int slot = 0;
                for (int w = 0; w < warp; ++w) slot += ((w + 1) * nseg) / NW > (w * nseg) / NW;
                uint32_t* ws = sums + slot * kSumPlanes * 32;
                ws[0 * 32 + lane] = O & m;
                ws[1 * 32 + lane] = O & ~s.Hd & m;
                ws[2 * 32 + lane] = s.h1 & m;
                ws[3 * 32 + lane] = s.h2 & m;
                ws[4 * 32 + lane] = (s.pa | s.pb) & m;
                ws[5 * 32 + lane] = s.G2 & m;
                ws[6 * 32 + lane] = s.G3 & m;
                unsigned long long l = s.links;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xFFFFFFFFu, l, o);
                if (lane == 0) wlinks[warp] = l;
            }
        } else if (lane == 0) {
            wlinks[warp] = 0;
        }
        uint32_t* wa = accs + warp * 16 * 32;
#pragma unroll
        for (int i = 0; i < 16; ++i) wa[i * 32 + lane] = s.acc[i];

        // ---- partials are double-buffered by scan parity: the finisher of the scan
        // two back (same half) must have loaded this strip's before we overwrite them
        const int64_t par = static_cast<int64_t>(scan_idx & 1ull);
        if (tid == 0 && scan_idx >= 2) {
            while (ld_acquire(prm.fin_loaded + par * prm.n_strips + strip) < scan_idx - 1) {
            }
        }
        __syncthreads();
        if (tid == 0 && seg_i == 0) stamp(prm, scan_idx, 1, globaltimer());
        // ---- CTA merge: counts (sum over warps, one coalesced 2 KB partial of u16x2
        // words per segment), K3 (compose the warps' band summaries in row order).
        for (int idx = tid; idx < 16 * 32; idx += T) {
            uint32_t v = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += accs[w * 16 * 32 + idx];
            prm.part[(par * prm.n_segments + seg) * 512 + idx] = v;
        }
        if (kLinks) {
            // non-empty warp bands were written to consecutive slots (row order)
            int nfull = 0;
            for (int w = 0; w < NW; ++w) nfull += ((w + 1) * nseg) / NW > (w * nseg) / NW;
            unsigned long long jl = 0;
            const BandSummary C = chain_compose<NW>(sums, nfull, wlinks + NW, jl);  // (contains __syncthreads)
            if (warp == 0) {
                unsigned long long links = lane < NW ? wlinks[lane] : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
                uint32_t* gs = prm.sums + (par * prm.n_segments + seg) * kSumPlanes * 32;
                store_summary(gs, lane, C);
                if (lane == 0) prm.seg_links[par * prm.n_segments + seg] = links + jl;
            }
        }
        // ---- arrive on the strip: the barrier orders every thread's partial
        // writes before tid 0's release; the last of the k arrivals acquires them all.
        __syncthreads();
        if (tid == 0) {
            if (seg_i == 0) stamp(prm, scan_idx, 2, globaltimer());
            const unsigned long long old = atom_add_acq_rel(prm.arrive + par * prm.n_strips + strip, 1ull);
            misc[0] = ((old + 1ull) % static_cast<unsigned long long>(prm.seg_per_strip)) == 0ull;
            stamp(prm, scan_idx, 8, scan_idx + 1);
            stamp(prm, scan_idx, 14, old + 1);
            stamp(prm, scan_idx, 15, static_cast<unsigned long long>(seg) + 1);
        }
        __syncthreads();
        if (misc[0]) finish_strip<kLinks, NW>(prm, strip, scan_idx, stages);
        // the merge / finish used the TMA ring as scratch (generic writes): order
        // them before the async-proxy writes of the next segment's loads
        fence_proxy_async();
        __syncthreads();
    }
    if (tid == 0 && have_seg) stamp(prm, seg_tick[0], 5, globaltimer());
}

// ----------------------------------------------------------------------------
// Small images (one strip, <= kSmallRows rows): ONE CTA does the whole scan.
// All row blocks are loaded at once into shared memory (16-byte loads, every
// load in flight together), each of 16 warps runs the same per-row K1/K3 code
// over its block, and the CTA merges the warps (counts, K3 band summaries)
// and writes counts, flags, boundaries and totals itself -- no TMA ring, scan
// tickets, segment partials or strip records: for a 32 KB image the pipelined
// kernel's protocol (ramp, arrival, finish) is most of its ~11 us device time.
constexpr int kSmallWarps = 16;
constexpr int kSmallRows = 512;  // 16 blocks: <= 1 per warp (at 1000^2 the pipelined latency plan is faster)
template <bool kLinks>
__host__ __device__ constexpr int small_smem_bytes() {
    return (kSmallRows / kBlockRows) * kStageBytes + kSmallWarps * 16 * 32 * 4 + kSmallWarps * kSumPlanes * 32 * 4 +
           kStripCols * 4 + 256;
}

template <bool kLinks>
__global__ void __launch_bounds__(kSmallWarps * 32) ychg_small_kernel(const ScanParams prm) {
    constexpr int NW = kSmallWarps;
    constexpr int T = NW * 32;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* boxes = smem;  // block b, row r: boxes + b * kStageBytes + r * kBoxBytes (128 B row + 16 B zero halo)
    uint32_t* accs = reinterpret_cast<uint32_t*>(smem + (kSmallRows / kBlockRows) * kStageBytes);
    uint32_t* sums = accs + NW * 16 * 32;
    int32_t* sc = reinterpret_cast<int32_t*>(sums + NW * kSumPlanes * 32);
    __shared__ unsigned long long wlinks[2 * NW];
    __shared__ uint32_t fw[kStripWords];
    __shared__ int wpre[kStripWords];
    __shared__ long long red[NW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nblk = prm.n_blocks;

    // (1) every row of the image: 16-byte chunks, bytes past the row zeroed; the
    //     halo chunk of every row is zero (nothing right of the only strip)
    {
        constexpr int kChunks = 9;  // 8 data chunks + the halo chunk per row
        constexpr int kPer = (kSmallRows * kChunks + T - 1) / T;  // every load in flight at once
        const int total = nblk * kBlockRows * kChunks;
        for (int i0 = tid; i0 < total; i0 += T * kPer) {
            uint4 v[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = i0 + u * T;
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if (i < total) {
                    const int row = i / kChunks, ch = i - row * kChunks;
                    if (ch < 8 && row < prm.height && 16 * ch < prm.row_bytes)
                        v[u] = __ldg(reinterpret_cast<const uint4*>(prm.bits + static_cast<int64_t>(row) * prm.pitch) + ch);
                }
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = i0 + u * T;
                if (i < total) {
                    const int row = i / kChunks, ch = i - row * kChunks;
                    uint4 x = v[u];
                    const int nb = prm.row_bytes - 16 * ch;  // valid bytes of this chunk
                    if (nb < 16) {
                        uint32_t* w = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int nq = nb - 4 * q;
                            w[q] = nq >= 4 ? w[q] : (nq <= 0 ? 0u : (w[q] & (0xFFFFFFFFu >> (8 * (4 - nq)))));
                        }
                    }
                    *reinterpret_cast<uint4*>(boxes + (row >> 5) * kStageBytes + (row & 31) * kBoxBytes + 16 * ch) = x;
                }
            }
        }
    }
    __syncthreads();

    // (2) the warp's blocks [wb0, wb0 + nb)
    const int wb0 = (warp * nblk) / NW, nb = ((warp + 1) * nblk) / NW - wb0;
    const Muls mu{prm.mul2, prm.mulnb, prm.mul1, prm.mulm1};
    LaneState s;
    s.ones = s.twos = s.fours = s.eights = s.u16 = s.u32 = s.u64 = s.u128 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s.acc[i] = 0;
    s.mk3 = word_mask(lane, min(prm.width_cnt, prm.width_img - 1));
    const bool full = !kLinks || __all_sync(0xFFFFFFFFu, s.mk3 == 0xFFFFFFFFu);
    s.h1 = s.h2 = 0;
    s.links = 0;
    s.pa = s.pb = s.pab = s.praw = 0;
    uint32_t O = 0;
    if (nb > 0) {
        uint32_t raw = 0, nbyte = 0;  // row 32*wb0 - 1 (zero above row 0)
        if (wb0 > 0) {
            const uint8_t* hr = boxes + (wb0 - 1) * kStageBytes + 31 * kBoxBytes + 4 * lane;
            raw = *reinterpret_cast<const uint32_t*>(hr);
            nbyte = hr[4];
        }
        s.praw = raw;
        s.pa = kLinks ? __byte_perm(raw, 0u, 0x0123u) : raw;
        s.pb = right_neighbour_msb(s.pa, nbyte, prm.mul2, prm.mulnb);
        O = kLinks ? (s.pa | s.pb) : 0u;
        s.Hd = O;
        s.G2 = s.G3 = O;
        s.pab = s.pa & s.pb;
        for (int bi = 0; bi < nb; ++bi) {
            const uint8_t* sp = boxes + (wb0 + bi) * kStageBytes;
            if (kLinks && __any_sync(0xFFFFFFFFu, (s.Hd & s.mk3) != 0u)) {
                if (full) process_block<kLinks, true, false>(sp, lane, s, mu);
                else process_block<kLinks, true, true>(sp, lane, s, mu);
            } else {
                if (full) process_block<kLinks, false, false>(sp, lane, s, mu);
                else process_block<kLinks, false, true>(sp, lane, s, mu);
            }
        }
        flush_counts(s);  // <= 2 blocks: no intermediate flush needed
    }
    int slot = 0;  // non-empty warp bands in row order
    for (int w = 0; w < warp; ++w) slot += ((w + 1) * nblk) / NW > (w * nblk) / NW;
    if (kLinks) {
        if (nb > 0) {
            const uint32_t m = s.mk3;
            uint32_t* ws = sums + slot * kSumPlanes * 32;
            ws[0 * 32 + lane] = O & m;
            ws[1 * 32 + lane] = O & ~s.Hd & m;
            ws[2 * 32 + lane] = s.h1 & m;
            ws[3 * 32 + lane] = s.h2 & m;
            ws[4 * 32 + lane] = (s.pa | s.pb) & m;
            ws[5 * 32 + lane] = s.G2 & m;
            ws[6 * 32 + lane] = s.G3 & m;
        }
        unsigned long long l = s.links;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xFFFFFFFFu, l, o);
        if (lane == 0) wlinks[warp] = l;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) accs[warp * 16 * 32 + i * 32 + lane] = s.acc[i];
    __syncthreads();

    // (3) merge: per-column counts (u16x2 sums over the warps) and the K3 stitch
    for (int idx = tid; idx < 16 * 32; idx += T) {
        uint32_t v = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += accs[w * 16 * 32 + idx];
        const int i = idx >> 5, ln = idx & 31;
        sc[32 * ln + acc_column<kLinks>(i, 0)] = static_cast<int32_t>(v & 0xFFFFu);
        sc[32 * ln + acc_column<kLinks>(i, 1)] = static_cast<int32_t>(v >> 16);
    }
    unsigned long long links = 0;
    if (kLinks) {
        int nfull = 0;
        for (int w = 0; w < NW; ++w) nfull += ((w + 1) * nblk) / NW > (w * nblk) / NW;
        unsigned long long jl = 0;
        const BandSummary C = chain_compose<NW>(sums, nfull, wlinks + NW, jl);  // (contains __syncthreads)
        if (warp == 0) {
            unsigned long long m = __popc(C.OE & C.T2 & ~C.T3);  // closed by the virtual background row H
            m += lane < NW ? wlinks[lane] : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
            links = m + jl;
        }
    }
    __syncthreads();

    // (4) flags (column 0 against 0, runscan.cpp:147), run total, boundary prefix
    long long local_sum = 0;
    for (int wi = warp; wi < kStripWords; wi += NW) {
        const int col = wi * 32 + lane;
        const bool valid = col < prm.width_cnt;
        const int32_t c = valid ? sc[col] : 0;
        const int32_t prev = col > 0 ? sc[col - 1] : 0;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, valid && c != prev);
        if (lane == 0) fw[wi] = m;
        local_sum += c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_sum += __shfl_xor_sync(0xFFFFFFFFu, local_sum, o);
    if (lane == 0) red[warp] = local_sum;
    __syncthreads();
    if (warp == 0) {
        const int c = __popc(fw[lane]);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        wpre[lane] = incl - c;
        if (lane == 31) {
            long long runs = 0;
            for (int w = 0; w < NW; ++w) runs += red[w];
            prm.totals[0] = runs;
            prm.totals[1] = kLinks ? static_cast<long long>(links) : 0;
            prm.totals[2] = kLinks ? runs - static_cast<long long>(links) : -1;
            prm.totals[3] = incl;
        }
    }
    __syncthreads();
    // (5) outputs
    const int nwords = (prm.width_cnt + 31) >> 5;
    for (int col = tid; col < prm.width_cnt; col += T) prm.counts[col] = sc[col];
    for (int wi = warp; wi < nwords; wi += NW) {
        const uint32_t m = fw[wi];
        if (lane == 0) prm.flags[wi] = m;
        if ((m >> lane) & 1u) prm.boundaries[wpre[wi] + __popc(m & ((1u << lane) - 1u))] = wi * 32 + lane;
    }
}

}  // namespace ychg_dev

// ----------------------------------------------------------------------------
// Host-side launcher (C linkage, called from ychg_capi.cu).
using namespace ychg_dev;

extern "C" const void* ychg_scan_kernel_ptr(int with_links) {
    return with_links ? reinterpret_cast<const void*>(&ychg_scan_kernel<true>)
                      : reinterpret_cast<const void*>(&ychg_scan_kernel<false>);
}

// Launch shape of the streaming kernel of a path (for occupancy queries).
extern "C" void ychg_scan_kernel_shape(int with_links, int* threads, int* smem_bytes) {
    *threads = 32 * (with_links ? scan_warps<true>() : scan_warps<false>());
    *smem_bytes = with_links ? scan_smem<true>() : scan_smem<false>();
}

// Opt-in to >48 KB dynamic shared memory (per device, both paths).
extern "C" int ychg_scan_kernel_prepare(void) {
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev]) return 0;
    cudaError_t e = cudaFuncSetAttribute(&ychg_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         scan_smem<true>());
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(&ychg_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 scan_smem<false>());
    const void* fns[2] = {reinterpret_cast<const void*>(&ychg_scan_kernel<true>),
                          reinterpret_cast<const void*>(&ychg_scan_kernel<false>)};
    for (const void* f : fns)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (dev < 64) done[dev] = true;
    return 0;
}

// One launch per scan, a programmatic dependent launch: the kernel triggers the
// next launch at CTA entry, so back-to-back scans (e.g. one CUDA graph) overlap
// the tail of one scan with the start of the next.
extern "C" int ychg_launch_scan(const void* tmap, const ScanParams* prm, int grid, int with_links,
                                cudaStream_t stream) {
    if (const int rc = ychg_scan_kernel_prepare()) return rc;
    const void* fa = with_links ? reinterpret_cast<const void*>(&ychg_scan_kernel<true>)
                                : reinterpret_cast<const void*>(&ychg_scan_kernel<false>);
    static const bool no_pdl = [] {
        const char* v = getenv("YCHG_NO_PDL");
        return v && v[0] == '1';
    }();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;

    CUtensorMap map = *static_cast<const CUtensorMap*>(tmap);
    ScanParams p = *prm;
    void* args_a[2] = {&map, &p};
    cudaLaunchConfig_t ca{};
    ca.gridDim = dim3(grid);
    ca.blockDim = dim3(32 * (with_links ? scan_warps<true>() : scan_warps<false>()));
    ca.dynamicSmemBytes = with_links ? scan_smem<true>() : scan_smem<false>();
    ca.stream = stream;
    ca.attrs = attr;
    ca.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelExC(&ca, fa, args_a);
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// Small images (one strip, <= kSmallRows rows): the single-CTA kernel.  Returns
// -1 when the geometry does not qualify (the caller uses the pipelined kernel).
extern "C" int ychg_launch_small(const ScanParams* prm, int with_links, cudaStream_t stream) {
    if (prm->n_strips != 1 || prm->height > kSmallRows || prm->width_img > kStripCols) return -1;
    static bool prepared[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int li = with_links ? 1 : 0;
    if (dev < 64 && !prepared[dev][li]) {
        const cudaError_t e = with_links
            ? cudaFuncSetAttribute(&ychg_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, small_smem_bytes<true>())
            : cudaFuncSetAttribute(&ychg_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, small_smem_bytes<false>());
        if (e != cudaSuccess) return static_cast<int>(e);
        prepared[dev][li] = true;
    }
    if (with_links) ychg_small_kernel<true><<<1, kSmallWarps * 32, small_smem_bytes<true>(), stream>>>(*prm);
    else ychg_small_kernel<false><<<1, kSmallWarps * 32, small_smem_bytes<false>(), stream>>>(*prm);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}
