// ychg_scan.cu -- the yCHG hot path on sm_100a: two kernels per scan, chained by
// programmatic dependent launch (PDL), graph-capturable.
//
//   K1  per-column cut-vertex counts      (reference runscan.cpp:41-74,122-128)
//   K2  change flags + ascending boundary  (runscan.cpp:145-153)
//   K3  hyperedge total = runs - links     (hypergraph.cpp:94-170,192)
//
// ychg_scan_kernel<with_links, NW> (streaming): the mask is cut into 1024-column
// strips (one 32-bit word per lane) and every strip into k row segments; CTA g
// owns segments g, g+G, ...  A segment is split into NW consecutive warp bands
// (NW = 4 for the ALU-bound K1+K3 path, 8 for the HBM-bound counts path).  Each
// warp streams its band through its own 3-stage TMA ring (cp.async.bulk.tensor,
// 32 rows x 144 B per stage: 128 B of the strip + a 16 B right halo) and runs K1
// + K3 bit-sliced in registers; the CTA merges its warps in shared memory and
// writes one partial per segment (counts + K3 band summary + links, coalesced)
// into a workspace double-buffered by scan parity, then release-stores an
// epoch-tagged segment flag.
//
// ychg_finish_kernel<with_links> (one small CTA per strip, co-resident with the
// streaming CTAs): waits for its strip's k flags, loads the partials, releases
// the buffer half, composes the K3 summaries, publishes a strip record and
// derives its boundary offset and first-column flag from every record to its
// left (warp-parallel look-back), compacts the boundary list; the right-most
// strip writes the totals.
//
// Consecutive scans overlap (the finisher of scan t runs while scan t+1
// streams).  The invariants that make this safe are listed in DESIGN.md §3
// ("Cross-scan invariants"): per-half fin_loaded, every per-segment input read
// before the half is released, scan tickets drawn before launch_dependents.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

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
// so Hd & f == Hd & ab & ~pab likewise).
template <bool kHead>
__device__ __forceinline__ uint32_t k3_step(uint32_t a, uint32_t b, LaneState& s) {
    const uint32_t ab = a & b;
    const uint32_t cont = lop3<0xF8>(a & s.pa, b, s.pb);       // (a & pa) | (b & pb)
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

// 32 rows from one TMA stage: 16 row pairs -> Harley-Seal tree -> ripple planes.
// Rises of one column are never in consecutive rows, so a row pair contributes
// (a0 & ~pa) | (a1 & ~a0) -- one LOP3.  Links of one pair are likewise never in
// consecutive rows and are popcounted per row pair.
// Right neighbour (column c+1 at column c's bit) of a raw little-endian word:
// inside a byte it is one bit lower (raw << 1); bit 0 of byte L takes bit 7 of
// byte L+1 (raw >> 15), byte 3 takes bit 7 of the next word's byte 0 (nb << 17).
// The shifts run as IMAD / IMAD.HI on the FMA pipe (runtime multipliers keep
// ptxas from turning them into ALU shifts); one LOP3 merges them.
// (Raw-order variant, kept for the diagnostics microbenchmarks: mul = 1 << 17.)
__device__ __forceinline__ uint32_t right_neighbour(uint32_t raw, uint32_t nb, uint32_t mul2, uint32_t mul17) {
    const uint32_t t1 = raw * mul2;
    const uint32_t t3 = nb * mul17 + __umulhi(raw, mul17);
    return lop3<0xE2>(t1, 0xFEFEFEFEu, t3);  // (t1 & M) | (t3 & ~M): bit select, one LOP3
}

// The K3 path runs on MSB-first words (one PRMT per row): the right neighbour is
// then a << 1 with the next word's first bit shifted in, i.e. the MSB of the
// next byte nb -- IMAD(a, 2, umulhi(nb, 1 << 25)), no ALU op at all (the
// raw-order merge above costs an extra LOP3 + IMAD; measured -4 % per row).
__device__ __forceinline__ uint32_t right_neighbour_msb(uint32_t a, uint32_t nb, uint32_t mul2, uint32_t mul25) {
    return a * mul2 + __umulhi(nb, mul25);
}

// kMask (strips with invalid column pairs -- the image's last column, or a
// multi-GPU strip's right halo): the right-hand column of an invalid pair is
// zeroed, so its components hold one run and never link.  Full strips skip it,
// which lets the two row links of a pair be added on the FMA pipe (they are
// disjoint bit sets) instead of a masked LOP3.
template <bool kLinks, bool kHead, bool kBs = kLinks, bool kMask = false>
__device__ __forceinline__ void process_block(const uint8_t* __restrict__ stage, int lane,
                                              LaneState& s, uint32_t mul2, uint32_t mulnb, uint32_t mul1) {
    const uint8_t* p = stage + 4 * lane;
    uint32_t Pprev = 0, tA = 0, fA = 0, eA = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const uint8_t* r0 = p + (2 * q) * kBoxBytes;
        const uint8_t* r1 = r0 + kBoxBytes;
        uint32_t a0 = *reinterpret_cast<const uint32_t*>(r0);
        uint32_t a1 = *reinterpret_cast<const uint32_t*>(r1);
        if (kBs) {  // MSB-first words (bit 31-j = column j): b = a << 1 | next byte's MSB, FMA pipe
            a0 = __byte_perm(a0, 0u, 0x0123u);
            a1 = __byte_perm(a1, 0u, 0x0123u);
        }
        const uint32_t P = lop3<0x3A>(a0, s.pa, a1);  // (a0 & ~pa) | (a1 & ~a0)
        if (kLinks) {
            uint32_t b0 = kBs ? right_neighbour_msb(a0, r0[4], mul2, mulnb)
                              : right_neighbour(a0, r0[4], mul2, mulnb);
            uint32_t b1 = kBs ? right_neighbour_msb(a1, r1[4], mul2, mulnb)
                              : right_neighbour(a1, r1[4], mul2, mulnb);
            if (kMask) {
                b0 &= s.mk3;
                b1 &= s.mk3;
            }
            const uint32_t l0 = k3_step<kHead>(a0, b0, s);
            const uint32_t l1 = k3_step<kHead>(a1, b1, s);
            // l0 | l1 == l0 + l1 (disjoint); IMADs keep both adds off the ALU pipe
            s.links = __popc(l0 * mul1 + l1) * mul1 + s.links;
        } else {
            s.pa = a1;
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

// dbg layout: [scan index % 4][CTA][32 slots]; `ring` must be in scope.
#define YCHG_STAMP_AT(slot, value)                                                                       \
    do {                                                                                                 \
        if (prm.dbg)                                                                                     \
            prm.dbg[(static_cast<int64_t>(ring) * prm.dbg_rows + blockIdx.x) * 32 + (slot)] = (value);      \
    } while (0)
#define YCHG_STAMP(slot) YCHG_STAMP_AT(slot, globaltimer())

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

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// In-place, order-preserving tree composition of n band summaries stored in
// shared memory (slot i = 7 planes x 32 lanes at base + i*224), using every warp
// of the CTA: level s composes slots (p*2s, p*2s+s) into p*2s.  Returns, in
// every thread, the number of links resolved at the junctions.  Must be called
// by the whole CTA (contains __syncthreads).
template <int NW>
__device__ unsigned long long tree_compose(uint32_t* base, int n, unsigned long long* red) {
    constexpr int kSW = kSumPlanes * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long mine = 0;
    for (int st = 1; st < n; st <<= 1) {
        for (int p = warp; p * 2 * st + st < n; p += NW) {
            uint32_t* a = base + (p * 2 * st) * kSW;
            const uint32_t* b = base + (p * 2 * st + st) * kSW;
            const BandSummary A{a[lane], a[32 + lane], a[64 + lane], a[96 + lane], a[128 + lane], a[160 + lane],
                                a[192 + lane]};
            const BandSummary B{b[lane], b[32 + lane], b[64 + lane], b[96 + lane], b[128 + lane], b[160 + lane],
                                b[192 + lane]};
            BandSummary C;
            mine += __popc(compose_summary(A, B, C));
            a[lane] = C.O;
            a[32 + lane] = C.E;
            a[64 + lane] = C.h1;
            a[96 + lane] = C.h2;
            a[128 + lane] = C.OE;
            a[160 + lane] = C.T2;
            a[192 + lane] = C.T3;
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    unsigned long long t = 0;
    for (int w = 0; w < NW; ++w) t += red[w];
    __syncthreads();
    return t;
}

// Shared-memory scratch of the strip finisher (lives in the idle TMA stage area).
struct FinishSmem {
    int32_t sc[kStripCols];       // counts of the strip's columns
    uint32_t fw[kStripWords];     // change-flag words of the strip (inside flags only)
    int wpre[kStripWords];        // exclusive prefix of popc(fw)
    long long red[kWarps];
    long long red2[kWarps];
    long long base;
    unsigned long long seglinks;  // links closed inside the strip's segments (loaded with the partials)
    uint32_t edge;                // flag of the strip's first column
};

__device__ __forceinline__ unsigned long long pack_strip_status(uint32_t epoch, uint32_t inside, int32_t first,
                                                                int32_t last) {
    return (static_cast<unsigned long long>(epoch & 0xFFFu) << 52) |
           (static_cast<unsigned long long>(inside & 0x3FFu) << 42) |
           (static_cast<unsigned long long>(static_cast<uint32_t>(first) & 0x1FFFFFu) << 21) |
           (static_cast<unsigned long long>(static_cast<uint32_t>(last) & 0x1FFFFFu));
}

// Warp-uniform wait until word p (per active lane) carries `epoch` in its top 12 bits.
__device__ __forceinline__ unsigned long long warp_wait_epoch12(const unsigned long long* p, bool active,
                                                               uint32_t epoch) {
    unsigned long long v = 0;
    bool ok = !active;
    while (true) {
        if (!ok) {
            v = ld_acquire(p);
            ok = static_cast<uint32_t>(v >> 52) == (epoch & 0xFFFu);
        }
        if (__all_sync(0xFFFFFFFFu, ok)) break;
    }
    return v;
}

// Finish strip s: counts, K3 stitch, flags, boundary compaction, totals.
// This runs on the kernel's tail, so it is built around global round trips:
// one batch of loads, one release of the strip record (flags strictly inside
// the strip + counts of its first and last column), one warp-parallel acquire
// of every record to the left -- from which the boundary offset AND this
// strip's first-column flag (counts[c0] vs counts[c0-1], runscan.cpp:147)
// follow -- then fire-and-forget writes.
template <bool kLinks>
__global__ void __launch_bounds__(kThreads)
ychg_finish_kernel(const ScanParams prm) {
    extern __shared__ __align__(128) uint8_t scratch[];
    FinishSmem& fs = *reinterpret_cast<FinishSmem*>(scratch);
    uint32_t* ssum = reinterpret_cast<uint32_t*>(scratch + ((sizeof(FinishSmem) + 127) / 128) * 128);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int s = blockIdx.x;
    const int k = prm.seg_per_strip;
    const int g0 = s * k;
    constexpr int kSumWords = kSumPlanes * 32;

    // (0) this strip's scan number -- taken BEFORE releasing the next scan's
    // streaming kernel, so tickets follow launch order (a later scan's finisher
    // can never draw an earlier number) -- then let the next scan launch right
    // away (it only needs SMs; it waits on fin_loaded before reusing this scan's
    // workspace), then wait until all k segments of this scan merged.
    unsigned long long scan_no = 0;
    if (tid == 0) {
        scan_no = atomicAdd(prm.fin_ticket + s, 1ull);
        fs.base = static_cast<long long>(scan_no);
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");
    scan_no = static_cast<unsigned long long>(fs.base);
    const uint32_t epoch = static_cast<uint32_t>(scan_no % 4095ull) + 1u;
    const int ring = static_cast<int>(scan_no & 3ull);
    if (tid == 0) YCHG_STAMP_AT(16, scan_no + 1);
    // Segment partials are double-buffered by scan parity (the next scan's
    // stream kernel writes the other half while this finisher reads).
    const int64_t par = static_cast<int64_t>(scan_no & 1ull);
    const int64_t G = prm.n_segments;
    const uint32_t* part_p = prm.part + par * G * 512;
    const uint32_t* sums_p = prm.sums + par * G * kSumWords;
    const unsigned long long* seglinks_p = prm.seg_links + par * G;
    const unsigned long long* segstat_p = prm.seg_status + par * G;
    if (warp == 0) {
        unsigned long long sl = 0;
        for (int jb = 0; jb < k; jb += 32) {
            const int j = jb + lane;
            const bool act = j < k;
            bool ok = !act;
            while (true) {
                if (!ok) ok = static_cast<uint32_t>(ld_acquire(segstat_p + g0 + (act ? j : 0))) == epoch;
                if (__all_sync(0xFFFFFFFFu, ok)) break;
            }
            // every per-segment input must be read before fin_loaded releases this
            // half to scan t+2 -- including the segment link counts
            if (kLinks && act) sl += __ldcg(seglinks_p + g0 + j);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xFFFFFFFFu, sl, o);
        if (lane == 0) fs.seglinks = sl;
    }
    __syncthreads();
    if (tid == 0) {
        YCHG_STAMP(21);
        YCHG_STAMP_AT(30, scan_no + 1);  // identity stamps: scan number (+1) at each stage
    }

    // (1) one batch of loads per 8 segments: partial counts (512 u16x2 words per
    //     segment over the CTA) and the K3 summaries (8 x 224 words).
    constexpr int kR = (512 + kThreads - 1) / kThreads;
    constexpr int kY = (8 * kSumWords + kThreads - 1) / kThreads;
    // Per-segment partials are u16x2 words (a segment has <= 65504 rows, so a
    // column's count in it fits 16 bits); the strip total needs up to 21 bits
    // (height < 2^22), so the two halves are summed separately.
    uint32_t v[kR], vh[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = vh[r] = 0;
    for (int g = 0; g < k; g += 8) {
        const int n = k - g < 8 ? k - g : 8;
        uint32_t x[kR][8], y[kY];
        const uint32_t* src = part_p + static_cast<int64_t>(g0 + g) * 512;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            const int idx = tid + r * kThreads;
#pragma unroll
            for (int u = 0; u < 8; ++u) x[r][u] = (u < n && idx < 512) ? __ldcg(src + u * 512 + idx) : 0u;
        }
        const uint32_t* ss = sums_p + static_cast<int64_t>(g0 + g) * kSumWords;
        if (kLinks) {
#pragma unroll
            for (int u = 0; u < kY; ++u) {
                const int i = tid + u * kThreads;
                y[u] = i < n * kSumWords ? __ldcg(ss + i) : 0u;
            }
        }
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                v[r] += x[r][u] & 0xFFFFu;
                vh[r] += x[r][u] >> 16;
            }
        if (kLinks) {
#pragma unroll
            for (int u = 0; u < kY; ++u) {
                const int i = tid + u * kThreads;
                if (i < n * kSumWords) ssum[g * kSumWords + i] = y[u];
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const int idx = tid + r * kThreads;
        if (idx < 512) {
            const int i = idx >> 5, ln = idx & 31;
            fs.sc[32 * ln + acc_column<kLinks>(i, 0)] = static_cast<int32_t>(v[r]);
            fs.sc[32 * ln + acc_column<kLinks>(i, 1)] = static_cast<int32_t>(vh[r]);
        }
    }
    __syncthreads();
    if (tid == 0) {
        YCHG_STAMP(24);
        YCHG_STAMP_AT(31, scan_no + 1);
        // this scan's workspace for strip s is in smem: the next scan's stream
        // kernel may overwrite it (it waits on this before its first partial write)
        st_release(prm.fin_loaded + par * prm.n_strips + s, scan_no + 1);
    }

    // (2) flags strictly inside the strip (columns 1..1023), counts out, run total
    const int nwords = (prm.width_cnt + 31) >> 5;
    long long local_sum = 0;
    for (int wi = warp; wi < kStripWords; wi += kWarps) {
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
    __syncthreads();

    // Strip records and the outputs are shared by consecutive scans: every
    // finisher of the previous scan must be done before this one publishes or
    // writes anything (normally long done by now).
    if (tid == 0 && scan_no > 0) {
        const unsigned long long need = scan_no * static_cast<unsigned long long>(prm.n_strips);
        YCHG_STAMP_AT(28, scan_no);
        while (ld_acquire(prm.fin_all) < need) {
        }
        YCHG_STAMP(29);
        YCHG_STAMP_AT(19, scan_no + 1);
    }
    __syncthreads();
    const bool last_strip = (s == prm.n_strips - 1);
    StripRecord* rec = prm.rec + s;
    int inside = 0;
    const int32_t first = fs.sc[0];
    if (warp == 0) {
        // (3) publish this strip's record early: the strips to the right wait on it
        const int c = __popc(fs.fw[lane]);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        fs.wpre[lane] = incl - c;
        inside = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (lane == 0) st_release(&rec->status, pack_strip_status(epoch, inside, first, fs.sc[kStripCols - 1]));
    }
    // (2b) K3: stitch the strip's segment summaries top to bottom (tree, all warps)
    unsigned long long strip_links = 0;
    if (kLinks) {
        strip_links = tree_compose<kWarps>(ssum, k, reinterpret_cast<unsigned long long*>(fs.red2));
        if (tid == 0) YCHG_STAMP(26);
        if (warp == 1) {
            // close whatever is still open at row H (virtual background row)
            unsigned long long c = __popc(ssum[4 * 32 + lane] & ssum[5 * 32 + lane] & ~ssum[6 * 32 + lane]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
            strip_links += c;
        }
    }

    if (warp == 0) {
        // (4) acquire every record to the left: boundary offset + this strip's first-column flag
        long long off = 0;
        int32_t carry_last = 0;  // last(j-1) entering each chunk; last(-1) := 0
        for (int jb = 0; jb < s; jb += 32) {
            const int j = jb + lane;
            const bool act = j < s;
            const unsigned long long st = warp_wait_epoch12(&prm.rec[act ? j : 0].status, act, epoch);
            const int32_t fj = static_cast<int32_t>((st >> 21) & 0x1FFFFFu);
            const int32_t lj = static_cast<int32_t>(st & 0x1FFFFFu);
            int32_t prev_last = __shfl_up_sync(0xFFFFFFFFu, lj, 1);
            if (lane == 0) prev_last = carry_last;
            if (act) off += static_cast<long long>((st >> 42) & 0x3FFu) + (fj != prev_last ? 1 : 0);
            carry_last = __shfl_sync(0xFFFFFFFFu, lj, (s - 1 - jb) < 31 ? (s - 1 - jb) : 31);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xFFFFFFFFu, off, o);
        if (lane == 0) {
            YCHG_STAMP(27);
            YCHG_STAMP_AT(18, scan_no + 1);
            fs.edge = (first != carry_last) ? 1u : 0u;
            fs.base = off;
            if (last_strip) prm.totals[3] = off + fs.edge + inside;
        }
    } else if (warp == 1) {
        // (4) release (runs, links) for the totals
        const unsigned long long links = strip_links;
        const unsigned long long sl = fs.seglinks;  // read before fin_loaded was released
        if (lane == 0) {
            long long runs = 0;
            for (int w = 0; w < kWarps; ++w) runs += fs.red[w];
            rec->runs = runs;
            rec->links = static_cast<long long>(links + sl);
            st_release(&rec->tstat, static_cast<unsigned long long>(epoch));
        }
    } else {
        // counts out (fire and forget)
        for (int col = tid - 64; col < kStripCols; col += kThreads - 64) {
            const int gc = s * kStripCols + col;
            if (gc < prm.width_cnt) prm.counts[gc] = fs.sc[col];
        }
    }
    __syncthreads();
    if (tid == 0) YCHG_STAMP(25);

    // (5) flags out + ordered compaction (the first-column flag, if set, comes first)
    const uint32_t e = fs.edge;
    if (tid == 0 && e) prm.boundaries[fs.base] = s * kStripCols;
    for (int wi = warp; wi < kStripWords; wi += kWarps) {
        const int w = s * kStripWords + wi;
        const uint32_t m = fs.fw[wi];
        if (lane == 0 && w < nwords) prm.flags[w] = m | (wi == 0 ? e : 0u);
        if ((m >> lane) & 1u)
            prm.boundaries[fs.base + e + fs.wpre[wi] + __popc(m & ((1u << lane) - 1u))] = w * 32 + lane;
    }

    // (6) the right-most strip also writes run/link totals once every strip released them
    if (last_strip && warp == 0) {
        long long runs = 0, links = 0;
        for (int jb = 0; jb < prm.n_strips; jb += 32) {
            const int j = jb + lane;
            const bool act = j < prm.n_strips;
            unsigned long long v = 0;
            bool ok = !act;
            while (true) {
                if (!ok) {
                    v = ld_acquire(&prm.rec[j].tstat);
                    ok = static_cast<uint32_t>(v) == epoch;
                }
                if (__all_sync(0xFFFFFFFFu, ok)) break;
            }
            if (act) {
                runs += __ldcg(&prm.rec[j].runs);
                links += __ldcg(&prm.rec[j].links);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            runs += __shfl_xor_sync(0xFFFFFFFFu, runs, o);
            links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
        }
        if (lane == 0) {
            prm.totals[0] = runs;
            prm.totals[1] = kLinks ? links : 0;
            prm.totals[2] = kLinks ? runs - links : -1;
        }
    }
    __syncthreads();
    if (tid == 0) {
        YCHG_STAMP(22);
        YCHG_STAMP_AT(17, scan_no + 1);
        __threadfence();
        atomicAdd(prm.fin_all, 1ull);
    }
}

// ----------------------------------------------------------------------------
template <bool kLinks, int NW = scan_warps<kLinks>()>
__global__ void __launch_bounds__(NW * 32, 1)
ychg_scan_kernel(const __grid_constant__ CUtensorMap tmap, const ScanParams prm) {
    constexpr int kS = scan_stages<kLinks>();  // TMA ring depth of this path
    using L = ScanSmem<NW, kS>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kStagesB);
    uint32_t* accs = reinterpret_cast<uint32_t*>(smem + L::kStagesB + L::kBar);
    uint32_t* sums = accs + NW * 16 * 32;
    unsigned long long* wlinks = reinterpret_cast<unsigned long long*>(sums + NW * kSumPlanes * 32);
    int* misc = reinterpret_cast<int*>(wlinks + 2 * NW);  // [0..W) warp empty, [W+1] epoch, [W+2] scan index

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    // This CTA's scan number for each of its segments, drawn BEFORE releasing the
    // finisher (and, through it, the next scan): tickets then follow launch order
    // even when consecutive scans' CTAs overlap.
    __shared__ unsigned long long seg_tick[kMaxSegPerCta];
    const unsigned long long t_entry = globaltimer();
    if (tid == 0) {
        for (int i = 0; i < NW * kS; ++i) mbar_init(&bars[i], 1);
        int i = 0;
        for (int sg = blockIdx.x; sg < prm.n_segments && i < kMaxSegPerCta; sg += gridDim.x, ++i)
            seg_tick[i] = atomicAdd(prm.seg_ticket + sg, 1ull);
    }
    fence_proxy_async();
    __syncthreads();
    // Let this scan's finisher kernel launch now: its CTAs are small, co-reside
    // with ours and wait on the per-segment flags (programmatic dependent launch).
    asm volatile("griddepcontrol.launch_dependents;");
    // The streaming kernel is a programmatic dependent of whatever kernel precedes
    // it on the stream.  Back-to-back scans need no wait (the image was written
    // before the previous scan's finisher ran); a plan whose image is written by
    // the immediately preceding kernel (host path: re-pitch / PNM pack) waits for
    // that grid's completion and memory flush here.
    if (prm.wait_inputs) asm volatile("griddepcontrol.wait;" ::: "memory");

    uint8_t* my_stages = stages + warp * kS * kStageBytes;
    uint64_t* my_bars = bars + warp * kS;
    uint32_t it = 0;  // blocks consumed by this warp so far (stage = it % kS)

    const int k = prm.seg_per_strip;
    int seg_i = 0;
    for (int seg = blockIdx.x; seg < prm.n_segments; seg += gridDim.x, ++seg_i) {
        const int strip = seg / k;
        const int j = seg - strip * k;
        const int sb0 = seg_first_block(j, k, prm.n_blocks);
        const int sb1 = seg_first_block(j + 1, k, prm.n_blocks);
        const int nseg = sb1 - sb0;
        const int wb0 = sb0 + (warp * nseg) / NW;
        const int wb1 = sb0 + ((warp + 1) * nseg) / NW;
        const int nb = wb1 - wb0;
        const int x0 = strip * kStripBytes;
        const int gw = strip * kStripWords + lane;

        // this segment's scan number (agrees with the finisher's strip ticket)
        if (tid == 0) {
            const unsigned long long t = seg_tick[seg_i];
            misc[NW + 1] = static_cast<int>(t % 4095ull) + 1;
            misc[NW + 2] = static_cast<int>(t);  // scans before this one (< 2^31 per plan)
            const int ring = static_cast<int>(t & 3ull);
            YCHG_STAMP_AT(0, t_entry);
            YCHG_STAMP_AT(15, t + 1);
        }
        LaneState s;
        s.ones = s.twos = s.fours = s.eights = s.u16 = s.u32 = s.u64 = s.u128 = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s.acc[i] = 0;
        s.mk3 = word_mask(gw, min(prm.width_cnt, prm.width_img - 1));  // MSB-first, like the K3 words
        // every column pair of this warp's strip valid (warp-uniform): no per-row mask
        const bool full = !kLinks || __all_sync(0xFFFFFFFFu, s.mk3 == 0xFFFFFFFFu);
        s.h1 = s.h2 = 0;
        s.links = 0;
        s.pa = s.pb = s.pab = 0;
        uint32_t O = 0;

        if (nb > 0) {
            // Kick off the ring first so the halo-row load overlaps it.
            if (lane == 0) {
                const int npre = nb < kS ? nb : kS;
                for (int i = 0; i < npre; ++i) {
                    const int st = (it + i) % kS;
                    mbar_arrive_expect_tx(&my_bars[st], kStageBytes);
                    tma_load_2d(my_stages + st * kStageBytes, &tmap, &my_bars[st], x0,
                                (wb0 + i) * kBlockRows);
                }
            }
            // Halo row y0-1 (the reference's prev row, runscan.cpp:45; zero above row 0).
            const int y0 = wb0 * kBlockRows;
            uint32_t raw = 0, nbyte = 0;
            if (y0 > 0) {
                const uint8_t* row = prm.bits + static_cast<int64_t>(y0 - 1) * prm.pitch;
                const int c = x0 + 4 * lane;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (c + q < prm.row_bytes) raw |= static_cast<uint32_t>(__ldg(row + c + q)) << (8 * q);
                if (c + 4 < prm.row_bytes) nbyte = __ldg(row + c + 4);
            }
            s.pa = kLinks ? __byte_perm(raw, 0u, 0x0123u) : raw;  // word order of process_block<kLinks>
            s.pb = right_neighbour_msb(s.pa, nbyte, prm.mul2, prm.mulnb);
            O = kLinks ? (s.pa | s.pb) : 0u;
            s.Hd = O;
            s.G2 = s.G3 = O;  // poisoned: the head's own closing is never a local link
            s.pab = s.pa & s.pb;

            int since_flush = 0;
            for (int bi = 0; bi < nb; ++bi) {
                const int st = it % kS;
#ifdef YCHG_COMPUTE_ONLY  // diagnostics build: reuse the first kS blocks, no TMA after the fill
                if (bi < kS) mbar_wait(&my_bars[st], (it / kS) & 1u);
#else
                mbar_wait(&my_bars[st], (it / kS) & 1u);
#endif
                const uint8_t* sp = my_stages + st * kStageBytes;
#ifdef YCHG_NO_HEAD  // diagnostics build: never take the head-mode block (wrong results, timing only)
                if (false)
#else
                if (kLinks && __any_sync(0xFFFFFFFFu, (s.Hd & s.mk3) != 0u))
#endif
                {
                    if (full) process_block<kLinks, true, kLinks, false>(sp, lane, s, prm.mul2, prm.mulnb, prm.mul1);
                    else process_block<kLinks, true, kLinks, true>(sp, lane, s, prm.mul2, prm.mulnb, prm.mul1);
                } else {
                    if (full) process_block<kLinks, false, kLinks, false>(sp, lane, s, prm.mul2, prm.mulnb, prm.mul1);
                    else process_block<kLinks, false, kLinks, true>(sp, lane, s, prm.mul2, prm.mulnb, prm.mul1);
                }
                __syncwarp();
#ifdef YCHG_COMPUTE_ONLY
                if (false) {
#else
                if (lane == 0 && bi + kS < nb) {
#endif
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&my_bars[st], kStageBytes);
                    tma_load_2d(my_stages + st * kStageBytes, &tmap, &my_bars[st], x0,
                                (wb0 + bi + kS) * kBlockRows);
                }
                ++it;
                if (++since_flush == kFlushBlocks) {
                    flush_counts(s);
                    since_flush = 0;
                }
            }
            flush_counts(s);

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
        if (lane == 0) {
            misc[warp] = (nb == 0);
            const int ring = misc[NW + 2] & 3;
            if (warp < 16) YCHG_STAMP(1 + warp);
        }
        __syncthreads();

        // ---- partials are double-buffered by scan parity: the finisher of the scan
        // two back (same half) must have loaded this strip before we overwrite it
        const unsigned long long scan_idx = static_cast<unsigned long long>(misc[NW + 2]);
        const int64_t par = static_cast<int64_t>(scan_idx & 1ull);
        if (tid == 0 && scan_idx >= 2) {
            const int ring = static_cast<int>(scan_idx & 3ull);
            YCHG_STAMP_AT(9, scan_idx);
            YCHG_STAMP(10);
            // per half: the NEXT scan's finisher (other half) may load first, so a
            // single per-strip counter could release us before scan_idx-2's
            // finisher has read this half (then its flags would be overwritten).
            while (ld_acquire(prm.fin_loaded + par * prm.n_strips + strip) < scan_idx - 1) {
            }
            YCHG_STAMP(11);
            YCHG_STAMP_AT(12, scan_idx + 1);
        }
        __syncthreads();
        // ---- CTA merge: counts (sum over warps, coalesced u16x2 words), K3 (compose in row order).
        for (int idx = tid; idx < 16 * 32; idx += (NW * 32)) {
            uint32_t v = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += accs[w * 16 * 32 + idx];
            prm.part[(par * prm.n_segments + seg) * 512 + idx] = v;
        }
        if (kLinks) {
            // non-empty warp bands were written to consecutive slots (row order)
            int nfull = 0;
            for (int w = 0; w < NW; ++w) nfull += ((w + 1) * nseg) / NW > (w * nseg) / NW;
            const unsigned long long jl = tree_compose<NW>(sums, nfull, wlinks + NW);
            if (warp == 0) {
                unsigned long long links = lane < NW ? wlinks[lane] : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
                uint32_t* gs = prm.sums + (par * prm.n_segments + seg) * kSumPlanes * 32;
#pragma unroll
                for (int q = 0; q < kSumPlanes; ++q) gs[q * 32 + lane] = sums[q * 32 + lane];
                if (lane == 0) prm.seg_links[par * prm.n_segments + seg] = links + jl;
            }
        }
        // ---- publish the segment: the barrier orders every thread's partial
        // writes before tid 0's release store of the epoch-tagged flag.
        __syncthreads();
        if (tid == 0) {
            const int ring = misc[NW + 2] & 3;
            YCHG_STAMP(20);
            YCHG_STAMP_AT(13, static_cast<unsigned long long>(misc[NW + 2]) + 1);
            st_release(prm.seg_status + par * prm.n_segments + seg, static_cast<unsigned long long>(misc[NW + 1]));
        }
        __syncthreads();
    }
    if (tid == 0 && prm.n_segments > 0) {
        const int ring = misc[NW + 2] & 3;
        YCHG_STAMP(23);
        YCHG_STAMP_AT(14, static_cast<unsigned long long>(misc[NW + 2]) + 1);
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

constexpr int kFinishSmemMax = 160 * 1024;

// Opt-in to >48 KB dynamic shared memory (per device, all kernels and variants).
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
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(&ychg_finish_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kFinishSmemMax);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(&ychg_finish_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kFinishSmemMax);
    // Same (maximum) shared-memory carveout for every kernel of a scan: an SM only
    // co-schedules CTAs whose carveout matches, and the finisher must co-reside
    // with the streaming CTAs it waits on.
    const void* fns[4] = {reinterpret_cast<const void*>(&ychg_scan_kernel<true>),
                          reinterpret_cast<const void*>(&ychg_scan_kernel<false>),
                          reinterpret_cast<const void*>(&ychg_finish_kernel<true>),
                          reinterpret_cast<const void*>(&ychg_finish_kernel<false>)};
    for (const void* f : fns)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     static_cast<int>(cudaSharedmemCarveoutMaxShared));
    if (e != cudaSuccess) return static_cast<int>(e);
    if (dev < 64) done[dev] = true;
    return 0;
}

// Two launches per scan, both programmatic dependent launches: the streaming
// kernel triggers its finisher at entry (the finisher CTAs are small and wait on
// per-segment flags while the stream runs), and the finisher triggers the NEXT
// scan's streaming kernel as soon as it holds this scan's workspace in smem, so
// back-to-back scans (e.g. one CUDA graph) overlap each finish with the next
// stream.  Every CTA of the finisher grid waits only on work that is already
// launched; the streaming kernel never waits.
extern "C" int ychg_launch_scan(const void* tmap, const ScanParams* prm, int grid, int with_links,
                                cudaStream_t stream, cudaEvent_t ev_mid) {
    (void)ev_mid;
    if (const int rc = ychg_scan_kernel_prepare()) return rc;
    const void* fa = with_links ? reinterpret_cast<const void*>(&ychg_scan_kernel<true>)
                                : reinterpret_cast<const void*>(&ychg_scan_kernel<false>);
    const void* fb = with_links ? reinterpret_cast<const void*>(&ychg_finish_kernel<true>)
                                : reinterpret_cast<const void*>(&ychg_finish_kernel<false>);
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
    cudaError_t e = cudaLaunchKernelExC(&ca, fa, args_a);
    if (e != cudaSuccess) return static_cast<int>(e);

    const size_t fsm = ((sizeof(FinishSmem) + 127) / 128) * 128 +
                       static_cast<size_t>(prm->seg_per_strip) * kSumPlanes * 32 * 4;
    if (fsm > static_cast<size_t>(kFinishSmemMax)) return static_cast<int>(cudaErrorInvalidValue);
    void* args_b[1] = {&p};
    cudaLaunchConfig_t cb{};
    cb.gridDim = dim3(prm->n_strips);
    cb.blockDim = dim3(kThreads);
    cb.dynamicSmemBytes = fsm;
    cb.stream = stream;
    cb.attrs = attr;
    cb.numAttrs = 1;
    e = cudaLaunchKernelExC(&cb, fb, args_b);
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}
