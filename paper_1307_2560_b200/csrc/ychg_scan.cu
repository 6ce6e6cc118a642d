// ychg_scan.cu -- the yCHG hot path on sm_100a.
//
//   K1  per-column cut-vertex counts      (reference runscan.cpp:41-74,122-128)
//   K2  change flags + ascending boundary  (runscan.cpp:145-153)
//   K3  hyperedge total = runs - links     (hypergraph.cpp:94-170,192)
//
// Three launches per scan, stream-ordered:
//   ychg_scan_kernel    streams the packed mask once (TMA, per-warp 4-stage ring),
//                       bit-sliced K1 + K3 per 32-row block, one partial per
//                       (strip, row-segment)  -- the HBM-bound kernel.
//   ychg_finish_kernel  one CTA per 1024-column strip: sums the segment partials,
//                       writes counts, change-flag words, per-strip boundary
//                       count; stitches the K3 band summaries top to bottom.
//   ychg_compact_kernel one CTA per strip: ordered boundary compaction
//                       (ballot/popc), final totals.
#include <cuda.h>
#include <cuda_runtime.h>

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
    uint32_t mk1, mk3;         // valid counted columns / valid pairs of this word
    // K3
    uint32_t G2, G3;           // open component holds >= 2 / >= 3 runs
    uint32_t Hd, h1, h2, E;    // head tracking (see BandSummary)
    uint32_t links;            // links closed inside this lane's band (<= rows/2 * 32)
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

// One row: returns the rises (background->foreground, runscan.cpp:57) of the
// lane's 32 columns and, when kLinks, advances the pair state machine and
// returns the pairs whose component closed at this row as a link.
template <bool kLinks, bool kHead>
__device__ __forceinline__ uint32_t row_step(uint32_t raw, uint32_t nbyte, LaneState& s,
                                             uint32_t& link) {
    const uint32_t a = __byte_perm(raw, 0u, 0x0123u);   // column j at bit 31-j
    const uint32_t na = a & ~s.pa & s.mk1;
    if (kLinks) {
        const uint32_t b = (a << 1) | (nbyte >> 7);      // column c+1 at column c's bit
        const uint32_t ab = a & b & s.mk3;
        const uint32_t f = ab & (s.pa ^ s.pb);           // a new run joins an open component
        const uint32_t cont = (a & s.pa) | (b & s.pb);   // the component continues into this row
        uint32_t lk = ~cont & s.G2 & ~s.G3;              // it closed holding exactly two runs
        if (kHead) {
            lk &= ~s.Hd;
            const uint32_t hf = s.Hd & f;
            s.h2 |= s.h1 & hf;
            s.h1 |= hf;
            s.E |= s.Hd & ~cont;
            s.Hd &= cont;
        }
        const uint32_t g3 = (cont & s.G3) | (s.G2 & f);
        s.G2 = ab | (cont & s.G2);
        s.G3 = g3;
        s.pb = b;
        link = lk;
    }
    s.pa = a;
    return na;
}

// 32 rows from one TMA stage: 16 row pairs -> Harley-Seal tree -> ripple planes.
// Rises of one column never occur in two consecutive rows, so a pair of rows
// contributes rises0 | rises1 exactly.  Links of one pair are likewise never in
// consecutive rows, so they are popcounted per row pair.
template <bool kLinks, bool kHead>
__device__ __forceinline__ void process_block(const uint8_t* __restrict__ stage, int lane,
                                              LaneState& s) {
    const uint8_t* p = stage + 4 * lane;
    uint32_t Pprev = 0, tA = 0, fA = 0, eA = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const uint8_t* r0 = p + (2 * q) * kBoxBytes;
        const uint8_t* r1 = r0 + kBoxBytes;
        const uint32_t raw0 = *reinterpret_cast<const uint32_t*>(r0);
        const uint32_t raw1 = *reinterpret_cast<const uint32_t*>(r1);
        const uint32_t nb0 = kLinks ? static_cast<uint32_t>(r0[4]) : 0u;
        const uint32_t nb1 = kLinks ? static_cast<uint32_t>(r1[4]) : 0u;
        uint32_t l0 = 0, l1 = 0;
        const uint32_t x0 = row_step<kLinks, kHead>(raw0, nb0, s, l0);
        const uint32_t x1 = row_step<kLinks, kHead>(raw1, nb1, s, l1);
        if (kLinks) s.links += __popc(l0 | l1);
        const uint32_t P = x0 | x1;
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

// ----------------------------------------------------------------------------
// K1 + K3 streaming kernel.  Persistent: CTA g processes segments g, g+G, ...
// Every segment (strip s, row blocks [b0, b1)) is split into 8 consecutive warp
// bands; each warp streams its band through its own 4-stage TMA ring (no
// CTA-wide barrier in the main loop), then the CTA merges the 8 warp results.
template <bool kLinks>
__global__ void __launch_bounds__(kThreads, 1)
ychg_scan_kernel(const __grid_constant__ CUtensorMap tmap, const ScanParams prm) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemStages + kSmemHalo);
    uint32_t* accs = reinterpret_cast<uint32_t*>(smem + kSmemStages + kSmemHalo + kSmemBar);
    uint32_t* sums = accs + kWarps * 16 * 32;
    unsigned long long* wlinks = reinterpret_cast<unsigned long long*>(sums + kWarps * kSumPlanes * 32);
    int* wempty = reinterpret_cast<int*>(wlinks + kWarps);

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    if (tid == 0) {
        for (int i = 0; i < kWarps * kStages; ++i) mbar_init(&bars[i], 1);
        if (blockIdx.x == 0) {
            for (int i = 0; i < 4; ++i) prm.totals[i] = 0;
        }
    }
    fence_proxy_async();
    __syncthreads();

    uint8_t* my_stages = stages + warp * kStages * kStageBytes;
    uint64_t* my_bars = bars + warp * kStages;
    uint32_t it = 0;  // blocks consumed by this warp so far (stage = it % kStages)

    const int k = prm.seg_per_strip;
    for (int seg = blockIdx.x; seg < prm.n_segments; seg += gridDim.x) {
        const int strip = seg / k;
        const int j = seg - strip * k;
        const int sb0 = seg_first_block(j, k, prm.n_blocks);
        const int sb1 = seg_first_block(j + 1, k, prm.n_blocks);
        const int nseg = sb1 - sb0;
        const int wb0 = sb0 + (warp * nseg) / kWarps;
        const int wb1 = sb0 + ((warp + 1) * nseg) / kWarps;
        const int nb = wb1 - wb0;
        const int x0 = strip * kStripBytes;
        const int gw = strip * kStripWords + lane;

        LaneState s;
        s.ones = s.twos = s.fours = s.eights = s.u16 = s.u32 = s.u64 = s.u128 = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) s.acc[i] = 0;
        s.mk1 = word_mask(gw, prm.width_cnt);
        s.mk3 = word_mask(gw, min(prm.width_cnt, prm.width_img - 1));
        s.G2 = s.G3 = s.h1 = s.h2 = s.E = 0;
        s.links = 0;
        s.pa = s.pb = 0;

        if (nb > 0) {
            // Kick off the ring first so the halo-row load overlaps it.
            if (lane == 0) {
                const int npre = nb < kStages ? nb : kStages;
                for (int i = 0; i < npre; ++i) {
                    const int st = (it + i) % kStages;
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
                    if (c + q < prm.row_bytes) raw |= static_cast<uint32_t>(row[c + q]) << (8 * q);
                if (c + 4 < prm.row_bytes) nbyte = row[c + 4];
            }
            s.pa = __byte_perm(raw, 0u, 0x0123u);
            s.pb = (s.pa << 1) | (nbyte >> 7);
            s.Hd = kLinks ? ((s.pa | s.pb) & s.mk3) : 0u;
            const uint32_t O = s.Hd;

            int since_flush = 0;
            for (int bi = 0; bi < nb; ++bi) {
                const int st = it % kStages;
                mbar_wait(&my_bars[st], (it / kStages) & 1u);
                const uint8_t* sp = my_stages + st * kStageBytes;
                if (kLinks && __any_sync(0xFFFFFFFFu, s.Hd != 0u))
                    process_block<kLinks, true>(sp, lane, s);
                else
                    process_block<kLinks, false>(sp, lane, s);
                __syncwarp();
                if (lane == 0 && bi + kStages < nb) {
                    fence_proxy_async();
                    mbar_arrive_expect_tx(&my_bars[st], kStageBytes);
                    tma_load_2d(my_stages + st * kStageBytes, &tmap, &my_bars[st], x0,
                                (wb0 + bi + kStages) * kBlockRows);
                }
                ++it;
                if (++since_flush == kFlushBlocks) {
                    flush_counts(s);
                    since_flush = 0;
                }
            }
            flush_counts(s);

            if (kLinks) {
                uint32_t* ws = sums + warp * kSumPlanes * 32;
                ws[0 * 32 + lane] = O;
                ws[1 * 32 + lane] = s.E;
                ws[2 * 32 + lane] = s.h1;
                ws[3 * 32 + lane] = s.h2;
                ws[4 * 32 + lane] = (s.pa | s.pb) & s.mk3;
                ws[5 * 32 + lane] = s.G2;
                ws[6 * 32 + lane] = s.G3;
                unsigned long long l = s.links;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xFFFFFFFFu, l, o);
                if (lane == 0) wlinks[warp] = l;
            }
        }
        uint32_t* wa = accs + warp * 16 * 32;
#pragma unroll
        for (int i = 0; i < 16; ++i) wa[i * 32 + lane] = s.acc[i];
        if (lane == 0) wempty[warp] = (nb == 0);
        __syncthreads();

        // ---- CTA merge: counts (sum over warps), K3 summaries (compose in row order).
        for (int idx = tid; idx < 16 * 32; idx += kThreads) {
            const int i = idx >> 5, ln = idx & 31;
            uint32_t v = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) v += accs[w * 16 * 32 + idx];
            uint32_t* out = prm.part + static_cast<int64_t>(seg) * kStripCols + 32 * ln;
            out[acc_column(i, 0)] = v & 0xFFFFu;
            out[acc_column(i, 1)] = v >> 16;
        }
        if (kLinks && warp == 0) {
            BandSummary C;
            unsigned long long links = 0;
            bool have = false;
            for (int w = 0; w < kWarps; ++w) {
                if (wempty[w]) continue;
                const uint32_t* ws = sums + w * kSumPlanes * 32;
                BandSummary B{ws[lane], ws[32 + lane], ws[64 + lane], ws[96 + lane],
                              ws[128 + lane], ws[160 + lane], ws[192 + lane]};
                if (lane == 0) links += wlinks[w];
                if (!have) {
                    C = B;
                    have = true;
                } else {
                    BandSummary D;
                    const uint32_t r = compose_summary(C, B, D);
                    links += __popc(r);
                    C = D;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
            uint32_t* gs = prm.sums + static_cast<int64_t>(seg) * kSumPlanes * 32;
            gs[0 * 32 + lane] = C.O;
            gs[1 * 32 + lane] = C.E;
            gs[2 * 32 + lane] = C.h1;
            gs[3 * 32 + lane] = C.h2;
            gs[4 * 32 + lane] = C.OE;
            gs[5 * 32 + lane] = C.T2;
            gs[6 * 32 + lane] = C.T3;
            if (lane == 0) prm.seg_links[seg] = links;
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------
// Finish: one CTA per strip.  counts, flags, per-strip boundary count, K3 stitch.
template <bool kLinks>
__global__ void __launch_bounds__(kThreads)
ychg_finish_kernel(const ScanParams prm) {
    __shared__ int32_t sc[kStripCols + 1];
    __shared__ long long red_sum[kWarps];
    __shared__ int red_nb[kWarps];
    const int s = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k = prm.seg_per_strip;
    const int g0 = s * k;

    long long local_sum = 0;
    for (int col = tid; col < kStripCols; col += kThreads) {
        uint32_t v = 0;
        for (int g = g0; g < g0 + k; ++g) v += prm.part[static_cast<int64_t>(g) * kStripCols + col];
        sc[col + 1] = static_cast<int32_t>(v);
        const int gc = s * kStripCols + col;
        if (gc < prm.width_cnt) {
            prm.counts[gc] = static_cast<int32_t>(v);
            local_sum += v;
        }
    }
    if (tid == 0) {
        // counts[c0 - 1] (counts[-1] := 0, runscan.cpp:147): last column of the previous strip.
        uint32_t prev = 0;
        if (s > 0)
            for (int g = g0 - k; g < g0; ++g)
                prev += prm.part[static_cast<int64_t>(g) * kStripCols + kStripCols - 1];
        sc[0] = static_cast<int32_t>(prev);
    }
    __syncthreads();

    const int nwords = (prm.width_cnt + 31) >> 5;
    int nb = 0;
    for (int wi = warp; wi < kStripWords; wi += kWarps) {
        const int col = wi * 32 + lane;
        const int gc = s * kStripCols + col;
        const bool f = gc < prm.width_cnt && sc[col + 1] != sc[col];
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
        if (lane == 0 && s * kStripWords + wi < nwords) prm.flags[s * kStripWords + wi] = m;
        nb += __popc(m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local_sum += __shfl_xor_sync(0xFFFFFFFFu, local_sum, o);
    if (lane == 0) {
        red_sum[warp] = local_sum;
        red_nb[warp] = nb;
    }
    __syncthreads();
    if (tid == 0) {
        long long t = 0;
        int n = 0;
        for (int w = 0; w < kWarps; ++w) {
            t += red_sum[w];
            n += red_nb[w];
        }
        prm.strip_nb[s] = n;
        atomicAdd(reinterpret_cast<unsigned long long*>(&prm.totals[0]),
                  static_cast<unsigned long long>(t));
    }

    if (kLinks && warp == 0) {
        // Stitch the strip's segment summaries top to bottom; row -1 and row H
        // are background (runscan.cpp:45, hypergraph.cpp walks whole columns).
        BandSummary C{};
        unsigned long long links = 0;
        for (int g = g0; g < g0 + k; ++g) {
            const uint32_t* gs = prm.sums + static_cast<int64_t>(g) * kSumPlanes * 32;
            BandSummary B{gs[lane], gs[32 + lane], gs[64 + lane], gs[96 + lane],
                          gs[128 + lane], gs[160 + lane], gs[192 + lane]};
            if (lane == 0) links += prm.seg_links[g];
            if (g == g0) {
                C = B;
            } else {
                BandSummary D;
                links += __popc(compose_summary(C, B, D));
                C = D;
            }
        }
        // close whatever is open at the bottom edge
        links += __popc(C.OE & C.T2 & ~C.T3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) links += __shfl_xor_sync(0xFFFFFFFFu, links, o);
        if (lane == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(&prm.totals[1]), links);
    }
}

// ----------------------------------------------------------------------------
// Ordered compaction of the change flags into the ascending boundary list.
template <bool kLinks>
__global__ void __launch_bounds__(kThreads)
ychg_compact_kernel(const ScanParams prm) {
    __shared__ long long red[kWarps];
    __shared__ int wpre[kStripWords + 1];
    const int s = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    long long off = 0;
    for (int t = tid; t < s; t += kThreads) off += prm.strip_nb[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xFFFFFFFFu, off, o);
    if (lane == 0) red[warp] = off;

    const int nwords = (prm.width_cnt + 31) >> 5;
    if (warp == 0) {
        const int w = s * kStripWords + lane;
        const uint32_t m = w < nwords ? prm.flags[w] : 0u;
        int c = __popc(m);
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
    for (int w = 0; w < kWarps; ++w) base += red[w];

    for (int wi = warp; wi < kStripWords; wi += kWarps) {
        const int w = s * kStripWords + wi;
        if (w >= nwords) break;
        const uint32_t m = prm.flags[w];
        if ((m >> lane) & 1u) {
            const int r = __popc(m & ((1u << lane) - 1u));
            prm.boundaries[base + wpre[wi] + r] = w * 32 + lane;
        }
    }

    if (s == gridDim.x - 1 && tid == 0) {
        prm.totals[3] = base + prm.strip_nb[s];
        prm.totals[2] = kLinks ? prm.totals[0] - prm.totals[1] : -1;
    }
}

}  // namespace ychg_dev

// ----------------------------------------------------------------------------
// Host-side launchers (C linkage, called from ychg_capi.cu).
using namespace ychg_dev;

extern "C" int ychg_launch_scan(const void* tmap, const ScanParams* prm, int grid, int with_links,
                                cudaStream_t stream, cudaEvent_t ev_mid) {
    // Opt-in to >48 KB dynamic shared memory once per device and variant.
    static bool attr_done[2][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const CUtensorMap* map = static_cast<const CUtensorMap*>(tmap);
    cudaError_t e;
    if (with_links) {
        if (dev >= 64 || !attr_done[1][dev]) {
            cudaFuncSetAttribute(ychg_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemTotal);
            if (dev < 64) attr_done[1][dev] = true;
        }
        ychg_scan_kernel<true><<<grid, kThreads, kSmemTotal, stream>>>(*map, *prm);
        if (ev_mid) cudaEventRecord(ev_mid, stream);
        ychg_finish_kernel<true><<<prm->n_strips, kThreads, 0, stream>>>(*prm);
        ychg_compact_kernel<true><<<prm->n_strips, kThreads, 0, stream>>>(*prm);
    } else {
        if (dev >= 64 || !attr_done[0][dev]) {
            cudaFuncSetAttribute(ychg_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemTotal);
            if (dev < 64) attr_done[0][dev] = true;
        }
        ychg_scan_kernel<false><<<grid, kThreads, kSmemTotal, stream>>>(*map, *prm);
        if (ev_mid) cudaEventRecord(ev_mid, stream);
        ychg_finish_kernel<false><<<prm->n_strips, kThreads, 0, stream>>>(*prm);
        ychg_compact_kernel<false><<<prm->n_strips, kThreads, 0, stream>>>(*prm);
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}
