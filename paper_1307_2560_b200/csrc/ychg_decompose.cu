// ychg_decompose.cu -- hyperedge decomposition on the device:
// decompose(const ColumnProfile&) (reference hypergraph.cpp:94-170) and the run ->
// edge map its Hypergraph constructor derives (:19-55), over the flat
// column-major run array that ychg_profile.cu materialises in HBM.
//
// The reference links runs with one two-pointer sweep per column pair and then
// walks every chain serially.  Here every phase is data-parallel over runs:
//   D1 overlap  each run binary-searches its two neighbour columns (sorted,
//               disjoint intervals) for its first overlapping run and a
//               saturating overlap count (0, 1, 2+)              (:108-135)
//   D2 link     r -> s iff r's only right overlap is s and s's only left
//               overlap is r (mutual uniqueness, :136-143); every run starts a
//               list-ranking node {ancestor, distance} on its left link
//   D3 jump     pointer jumping until every node names its chain head (chains
//               are at most W long: <= ceil(log2 W) rounds)
//   D4 tails    each chain tail stores (1 edge, chain length) at its head
//   D5 scan     exclusive scan of those (edges, runs) pairs in profile order =
//               the canonical edge id and first output slot of every head --
//               chains are numbered by their head's (column, y_top), exactly the
//               reference's discovery order (:145-167)
//   D6 emit     each head of a short chain walks it and writes its runs to
//               consecutive slots from offset(head); runs of long chains go to
//               offset(head) + distance one by one; run_to_edge[g] = id(head)
// Integer-exact: the outputs are bit-identical to the reference's.
#include <cuda_runtime.h>

#include <cstdint>

namespace ychg_dev {
namespace {

constexpr uint32_t kNoLink = 0xFFFFFFFFu;
constexpr int kThreadsD = 256;
constexpr int kScanItems = 8;                       // u64 items per thread in the scan tiles
constexpr int kScanTile = kThreadsD * kScanItems;   // 2048

__device__ __forceinline__ unsigned long long pack(uint32_t hi, uint32_t lo) {
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// First run of column list [b, e) whose y_bot >= top (runs sorted, disjoint).
__device__ __forceinline__ int64_t first_reaching(const int32_t* __restrict__ runs, int64_t b, int64_t e, int top) {
    while (b < e) {
        const int64_t m = (b + e) >> 1;
        if (__ldg(runs + 3 * m + 2) < top) b = m + 1;
        else e = m;
    }
    return b;
}

// The same, galloping out from a guess g in [b, e): neighbouring columns hold
// similar numbers of runs at similar heights, so the run of column c+1 reaching
// row `top` sits near index g = b + i * n(c+1) / n(c) for the i-th run of column
// c -- a few probes (cached by the neighbouring threads) instead of log2(n).
__device__ __forceinline__ int64_t first_reaching_from(const int32_t* __restrict__ runs, int64_t b, int64_t e,
                                                       int top, int64_t g) {
    if (b >= e) return b;
    g = g < b ? b : (g >= e ? e - 1 : g);
    int64_t lo, hi;  // answer in [lo, hi]
    if (__ldg(runs + 3 * g + 2) < top) {  // answer is right of g
        int64_t step = 1;
        lo = g + 1;
        hi = g + 1;
        while (hi < e && __ldg(runs + 3 * hi + 2) < top) {
            lo = hi + 1;
            step <<= 1;
            hi = g + step;
        }
        if (hi > e) hi = e;
    } else {  // answer is g or left of it
        int64_t step = 1;
        hi = g;
        lo = g - 1;
        while (lo >= b && __ldg(runs + 3 * lo + 2) >= top) {
            hi = lo;
            step <<= 1;
            lo = g - step;
        }
        lo = lo < b ? b : lo + 1;
    }
    return first_reaching(runs, lo, hi, top);
}


// D1: for run g, the first overlapping run in column c+1 (resp. c-1) and the
// overlap count saturated at 2.  ov = right | left << 2.
__global__ void __launch_bounds__(kThreadsD) decomp_overlap_kernel(const int32_t* __restrict__ runs,
                                                                   const int64_t* __restrict__ col_off,
                                                                   const int32_t* __restrict__ counts, int32_t width,
                                                                   int64_t n, uint32_t* __restrict__ pr,
                                                                   uint32_t* __restrict__ pl, uint8_t* __restrict__ ov) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const int c = __ldg(runs + 3 * g), top = __ldg(runs + 3 * g + 1), bot = __ldg(runs + 3 * g + 2);
        uint32_t cnt_r = 0, cnt_l = 0, jr = kNoLink, jl = kNoLink;
        const int64_t own0 = __ldg(col_off + c);
        const int64_t i_own = g - own0;
        const int32_t n_own = __ldg(counts + c);
        if (c + 1 < width) {
            const int32_t n = __ldg(counts + c + 1);
            const int64_t b = __ldg(col_off + c + 1), e = b + n;
            const int64_t j = first_reaching_from(runs, b, e, top, b + (i_own * n) / (n_own > 0 ? n_own : 1));
            if (j < e && __ldg(runs + 3 * j + 1) <= bot) {
                cnt_r = 1 + (j + 1 < e && __ldg(runs + 3 * (j + 1) + 1) <= bot);
                jr = static_cast<uint32_t>(j);
            }
        }
        if (c > 0) {
            const int32_t n = __ldg(counts + c - 1);
            const int64_t b = __ldg(col_off + c - 1), e = b + n;
            const int64_t j = first_reaching_from(runs, b, e, top, b + (i_own * n) / (n_own > 0 ? n_own : 1));
            if (j < e && __ldg(runs + 3 * j + 1) <= bot) {
                cnt_l = 1 + (j + 1 < e && __ldg(runs + 3 * (j + 1) + 1) <= bot);
                jl = static_cast<uint32_t>(j);
            }
        }
        pr[g] = jr;
        pl[g] = jl;
        ov[g] = static_cast<uint8_t>(cnt_r | (cnt_l << 2));
    }
}

// D2: mutual-uniqueness links; pr[g] becomes the right link (or kNoLink) and
// node[g] = {left neighbour, 1} or {g, 0} for a chain head.
__global__ void __launch_bounds__(kThreadsD) decomp_link_kernel(int64_t n, uint32_t* __restrict__ pr,
                                                                const uint32_t* __restrict__ pl,
                                                                const uint8_t* __restrict__ ov,
                                                                unsigned long long* __restrict__ node) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t o = ov[g];
        const uint32_t r = pr[g], l = pl[g];
        const bool right = (o & 3u) == 1u && (ov[r] >> 2) == 1u;
        const bool left = (o >> 2) == 1u && (ov[l] & 3u) == 1u;
        pr[g] = right ? r : kNoLink;
        node[g] = left ? pack(l, 1u) : pack(static_cast<uint32_t>(g), 0u);
    }
}

// D3: one pointer-jumping round, in place ({ancestor, distance} pairs are read
// and written as single 64-bit words, so a concurrently advanced pair is still
// a consistent, only further-along, answer).
__global__ void __launch_bounds__(kThreadsD) decomp_jump_kernel(int64_t n, unsigned long long* __restrict__ node,
                                                                int* __restrict__ changed) {
    bool any = false;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long v = node[g];
        const uint32_t a = static_cast<uint32_t>(v >> 32);
        if (a == static_cast<uint32_t>(g)) continue;
        const unsigned long long w = node[a];
        const uint32_t a2 = static_cast<uint32_t>(w >> 32);
        if (a2 == a) continue;  // a is a head: done
        node[g] = pack(a2, static_cast<uint32_t>(v) + static_cast<uint32_t>(w));
        any = true;
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) *changed = 1;
}

// D4: every chain tail (no right link) stores {1 edge, chain length} at its head.
__global__ void __launch_bounds__(kThreadsD) decomp_tail_kernel(int64_t n, const uint32_t* __restrict__ pr,
                                                                const unsigned long long* __restrict__ node,
                                                                unsigned long long* __restrict__ val) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        if (pr[g] != kNoLink) continue;
        const unsigned long long v = node[g];
        val[v >> 32] = pack(1u, static_cast<uint32_t>(v) + 1u);
    }
}

// D5: exclusive scan of u64 in three passes (tile sums, spine, tiles).
__device__ __forceinline__ unsigned long long block_exclusive(unsigned long long x, unsigned long long* sh,
                                                              unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long s = lane < kThreadsD / 32 ? sh[lane] : 0ull;
        unsigned long long si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < kThreadsD / 32) sh[lane] = si - s;
        if (lane == kThreadsD / 32 - 1) sh[32] = si;
    }
    __syncthreads();
    const unsigned long long r = sh[warp] + inc - x;
    *total = sh[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kThreadsD) scan_tile_sums_kernel(const unsigned long long* __restrict__ v, int64_t n,
                                                                   unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long sh[33];
    const int64_t base = blockIdx.x * int64_t(kScanTile) + threadIdx.x * int64_t(kScanItems);
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += v[base + i];
    unsigned long long tot;
    block_exclusive(s, sh, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// One CTA: exclusive scan of the tile sums in place; the grand total to *total.
__global__ void __launch_bounds__(kThreadsD) scan_spine_kernel(unsigned long long* __restrict__ sums, int64_t tiles,
                                                               unsigned long long* __restrict__ total) {
    __shared__ unsigned long long sh[33];
    unsigned long long carry = 0;
    for (int64_t b = 0; b < tiles; b += kThreadsD) {
        const int64_t i = b + threadIdx.x;
        const unsigned long long x = i < tiles ? sums[i] : 0ull;
        unsigned long long tot;
        const unsigned long long e = block_exclusive(x, sh, &tot);
        if (i < tiles) sums[i] = carry + e;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kThreadsD) scan_tiles_kernel(unsigned long long* __restrict__ v, int64_t n,
                                                               const unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long sh[33];
    const int64_t base = blockIdx.x * int64_t(kScanTile) + threadIdx.x * int64_t(kScanItems);
    unsigned long long x[kScanItems];
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        x[i] = base + i < n ? v[base + i] : 0ull;
        s += x[i];
    }
    unsigned long long tot;
    unsigned long long run = sums[blockIdx.x] + block_exclusive(s, sh, &tot);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) {
            v[base + i] = run;
            run += x[i];
        }
}

// D6: runs into hyperedge order, the run -> edge map, the edge offsets.  Each
// chain head walks its chain along the right links (at most kWalkMax runs) and
// writes the records to consecutive output slots.  The heads among a warp's 32
// consecutive runs are consecutive edges, so their chains fill one contiguous
// stretch of the output: staged in shared memory in output order (its first
// kEmitStage records; the rest go straight out) and copied out with consecutive
// 4-byte stores.  A run-by-run scatter to offset(head) + distance wrote 12-byte
// pieces all over the output instead (one store instruction = 32 scattered
// pieces; 2.5x DRAM write amplification, ~70 B per run at 21000^2 checker(7)).
// Runs kWalkMax or more from their head (a walk would be that many dependent
// loads) are scattered by decomp_long_kernel.
constexpr int kWalkMax = 24;
constexpr int kEmitStage = 256;  // records per warp staged in shared memory (3 KB)

__global__ void __launch_bounds__(kThreadsD) decomp_emit_kernel(int64_t n, const int32_t* __restrict__ runs,
                                                                const uint32_t* __restrict__ pr,
                                                                const unsigned long long* __restrict__ node,
                                                                const unsigned long long* __restrict__ excl,
                                                                const unsigned long long* __restrict__ total,
                                                                int32_t* __restrict__ edge_runs,
                                                                uint32_t* __restrict__ edge_offsets,
                                                                uint32_t* __restrict__ run_to_edge,
                                                                int* __restrict__ long_flag) {
    __shared__ int32_t stage[kThreadsD / 32][3 * kEmitStage];
    const int lane = threadIdx.x & 31;
    int32_t* st = stage[threadIdx.x >> 5];
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t g0 = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); g0 < n; g0 += stride) {
        const int64_t g = g0 + lane;
        bool head = false;
        uint32_t e = 0, off = 0;
        if (g < n) {
            head = static_cast<uint32_t>(node[g] >> 32) == static_cast<uint32_t>(g);
            if (head) {
                const unsigned long long s = excl[g];
                e = static_cast<uint32_t>(s >> 32);
                off = static_cast<uint32_t>(s);
                edge_offsets[e] = off;
                if (g == 0) edge_offsets[*total >> 32] = static_cast<uint32_t>(n);  // run 0 always heads a chain
            }
        }
        if (!__any_sync(0xFFFFFFFFu, head)) continue;  // members only: their heads write them
        const uint32_t first = __reduce_min_sync(0xFFFFFFFFu, head ? off : 0xFFFFFFFFu);
        int d = 0;
        if (head) {
            int64_t cur = g;
            const int sbase = static_cast<int>(off - first);  // staged slot of record 0 (may be past the stage)
            bool ended = false;
            for (; d < kWalkMax; ++d) {
                const int32_t c = __ldg(runs + 3 * cur), t = __ldg(runs + 3 * cur + 1), b = __ldg(runs + 3 * cur + 2);
                const uint32_t next = pr[cur];
                int32_t* dst = sbase + d < kEmitStage ? st + 3 * (sbase + d) : edge_runs + 3 * (int64_t(off) + d);
                dst[0] = c;
                dst[1] = t;
                dst[2] = b;
                run_to_edge[cur] = e;
                if (next == kNoLink) {
                    ++d;
                    ended = true;
                    break;
                }
                cur = next;
            }
            if (!ended) *long_flag = 1;  // runs kWalkMax and more from the head: decomp_long_kernel
        }
        const uint32_t end = __reduce_max_sync(0xFFFFFFFFu, head ? off + static_cast<uint32_t>(d) : 0u);
        __syncwarp();
        const int tot = 3 * static_cast<int>(min(end - first, static_cast<uint32_t>(kEmitStage)));
        int32_t* out = edge_runs + 3 * int64_t(first);
        for (int i = lane; i < tot; i += 32) out[i] = st[i];
        __syncwarp();
    }
}

// D6, runs kWalkMax or more from their head: slot offset(head) + distance.
__global__ void __launch_bounds__(kThreadsD) decomp_long_kernel(int64_t n, const int32_t* __restrict__ runs,
                                                                const unsigned long long* __restrict__ node,
                                                                const unsigned long long* __restrict__ excl,
                                                                const int* __restrict__ long_flag,
                                                                int32_t* __restrict__ edge_runs,
                                                                uint32_t* __restrict__ run_to_edge) {
    if (*long_flag == 0) return;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const unsigned long long v = node[g];
        const uint32_t h = static_cast<uint32_t>(v >> 32), dist = static_cast<uint32_t>(v);
        if (h == static_cast<uint32_t>(g) || dist < static_cast<uint32_t>(kWalkMax)) continue;  // walked by its head
        const unsigned long long s = excl[h];
        const int64_t pos = int64_t(static_cast<uint32_t>(s)) + dist;
        edge_runs[3 * pos] = runs[3 * g];
        edge_runs[3 * pos + 1] = runs[3 * g + 1];
        edge_runs[3 * pos + 2] = runs[3 * g + 2];
        run_to_edge[g] = static_cast<uint32_t>(s >> 32);
    }
}

// Profile-input validation (validate_profile, hypergraph.cpp:62-90): the first
// failing run in profile order, with the reference's check order inside a run
// (column claim, range, order).  err = min(g * 4 + kind).
__global__ void __launch_bounds__(kThreadsD) decomp_validate_kernel(const int32_t* __restrict__ runs,
                                                                    const int64_t* __restrict__ col_off, int32_t width,
                                                                    int32_t height, int64_t n,
                                                                    unsigned long long* __restrict__ err) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const int c = runs[3 * g], top = runs[3 * g + 1], bot = runs[3 * g + 2];
        // the column list that holds g (counts are the list sizes)
        int64_t lo = 0, hi = width - 1;
        while (lo < hi) {
            const int64_t m = (lo + hi + 1) >> 1;
            if (col_off[m] <= g) lo = m;
            else hi = m - 1;
        }
        // the last list starting at or before g holds it (empty lists start where
        // the next one does, so they are never the last)
        const int list = static_cast<int>(lo);
        unsigned int kind = 0;
        if (c != list) kind = 1;
        else if (top < 0 || top > bot || bot >= height) kind = 2;
        else if (g > col_off[list] && top < runs[3 * (g - 1) + 2] + 2) kind = 3;
        if (kind) atomicMin(err, static_cast<unsigned long long>(g) * 4ull + kind);
    }
}

}  // namespace
}  // namespace ychg_dev

using namespace ychg_dev;

namespace {
int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + kThreadsD - 1) / kThreadsD;
    const int64_t cap = int64_t(sms) * 8;
    return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}
}  // namespace

extern "C" {

// Scratch bytes the decomposition of n runs needs (ychg_launch_decompose's ws).
int64_t ychg_decompose_ws_bytes(int64_t n) {
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    // pr | pl (16-B rounded) | node | val | tile sums (+2) | flag (16 B) | ov
    return ((n * 8 + 15) / 16) * 16 + n * 16 + (tiles + 2) * 8 + 16 + n + 256;
}

// Validate a host-supplied profile on the device; *d_err = min(g*4+kind) or ~0.
int ychg_launch_decompose_validate(const int32_t* d_runs, const int64_t* d_col_off, int32_t width, int32_t height, int64_t n, unsigned long long* d_err,
                                   cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(d_err, 0xFF, 8, stream);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (n > 0) decomp_validate_kernel<<<grid_for(n), kThreadsD, 0, stream>>>(d_runs, d_col_off, width, height, n,
                                                                             d_err);
    return static_cast<int>(cudaGetLastError());
}

// The full decomposition of a device profile (n > 0).  h_flag must be pinned host
// memory: the pointer-jumping rounds stop when a round changes nothing (one
// stream synchronisation per round, <= ceil(log2 width) + 1 rounds).  Returns
// the number of jump rounds run (>= 1) or -(cudaError_t).
int ychg_launch_decompose(const int32_t* d_runs, const int64_t* d_col_off, const int32_t* d_counts, int32_t width,
                          int64_t n, void* d_ws, int32_t* d_edge_runs, uint32_t* d_edge_offsets,
                          uint32_t* d_run_to_edge, unsigned long long* d_total, int* h_flag, cudaStream_t stream) {
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    uint8_t* p = static_cast<uint8_t*>(d_ws);
    uint32_t* pr = reinterpret_cast<uint32_t*>(p);
    uint32_t* pl = pr + n;
    unsigned long long* node = reinterpret_cast<unsigned long long*>(p + ((n * 8 + 15) / 16) * 16);
    unsigned long long* val = node + n;
    unsigned long long* sums = val + n;
    int* flag = reinterpret_cast<int*>(sums + tiles + 2);
    uint8_t* ov = reinterpret_cast<uint8_t*>(flag + 4);
    const int grid = grid_for(n);
    decomp_overlap_kernel<<<grid, kThreadsD, 0, stream>>>(d_runs, d_col_off, d_counts, width, n, pr, pl, ov);
    decomp_link_kernel<<<grid, kThreadsD, 0, stream>>>(n, pr, pl, ov, node);
    int rounds = 0;
    for (;;) {
        cudaError_t e = cudaMemsetAsync(flag, 0, 4, stream);
        if (e != cudaSuccess) return -static_cast<int>(e);
        decomp_jump_kernel<<<grid, kThreadsD, 0, stream>>>(n, node, flag);
        ++rounds;
        e = cudaMemcpyAsync(h_flag, flag, 4, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return -static_cast<int>(e);
        if (*h_flag == 0) break;
        if (rounds > 40) return -static_cast<int>(cudaErrorIllegalState);  // chains are <= width long
    }
    cudaError_t e = cudaMemsetAsync(val, 0, n * 8, stream);
    if (e != cudaSuccess) return -static_cast<int>(e);
    decomp_tail_kernel<<<grid, kThreadsD, 0, stream>>>(n, pr, node, val);
    scan_tile_sums_kernel<<<static_cast<unsigned>(tiles), kThreadsD, 0, stream>>>(val, n, sums);
    scan_spine_kernel<<<1, kThreadsD, 0, stream>>>(sums, tiles, d_total);
    scan_tiles_kernel<<<static_cast<unsigned>(tiles), kThreadsD, 0, stream>>>(val, n, sums);
    e = cudaMemsetAsync(flag, 0, 4, stream);
    if (e != cudaSuccess) return -static_cast<int>(e);
    decomp_emit_kernel<<<grid, kThreadsD, 0, stream>>>(n, d_runs, pr, node, val, d_total, d_edge_runs, d_edge_offsets,
                                                       d_run_to_edge, flag);
    decomp_long_kernel<<<grid, kThreadsD, 0, stream>>>(n, d_runs, node, val, flag, d_edge_runs, d_run_to_edge);
    e = cudaGetLastError();
    return e == cudaSuccess ? rounds : -static_cast<int>(e);
}

}  // extern "C"
