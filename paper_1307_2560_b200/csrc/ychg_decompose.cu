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
//               overlap is r (mutual uniqueness, :136-143); anc[r] = left link
//               (or r for a chain head)
//   D3 jump     one launch of concurrent pointer jumping to the chain heads
//               (a run's distance to its head is its column difference)
//   D4 tails    every chain tail stores the chain length at its head
//   D5 scan     one-pass (decoupled look-back) exclusive scan of {1 edge, chain
//               length} at the heads in profile order = the canonical edge id and
//               first output slot of every head -- chains are numbered by their
//               head's (column, y_top), exactly the reference's discovery order
//               (:145-167)
//   D6 emit     each head of a short chain walks it and writes its runs to
//               consecutive slots from offset(head); runs of long chains go to
//               offset(head) + distance one by one; run_to_edge[g] = id(head)
// Integer-exact: the outputs are bit-identical to the reference's.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

namespace ychg_dev {
namespace {

constexpr uint32_t kNoLink = 0xFFFFFFFFu;
constexpr int kThreadsD = 256;
constexpr int kScanItems = 16;                      // items per thread in the scan tiles
constexpr int kScanTile = kThreadsD * kScanItems;   // 4096

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
// `bot_g` is the y_bot of run g (clamped into [b, e)) when the caller has already
// loaded it (first probes of several searches issued together), else INT_MIN.
__device__ __forceinline__ int64_t clamp_guess(int64_t b, int64_t e, int64_t g) {
    return g < b ? b : (g >= e ? e - 1 : g);
}

__device__ __forceinline__ int64_t first_reaching_from(const int32_t* __restrict__ runs, int64_t b, int64_t e,
                                                       int top, int64_t g, int bot_g = INT_MIN) {
    if (b >= e) return b;
    g = clamp_guess(b, e, g);
    if (bot_g == INT_MIN) bot_g = __ldg(runs + 3 * g + 2);
    int64_t lo, hi;  // answer in [lo, hi]
    if (bot_g < top) {  // answer is right of g
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
// overlap count saturated at 2.  ov = right | left << 2.  The two searches are
// started together (both first probes in flight at once), and each side's two
// overlap tests read runs j and j+1 with independent loads.
__global__ void __launch_bounds__(kThreadsD) decomp_overlap_kernel(const int32_t* __restrict__ runs,
                                                                   const int64_t* __restrict__ col_off,
                                                                   const int32_t* __restrict__ counts, int32_t width,
                                                                   int64_t n, uint32_t* __restrict__ pr,
                                                                   uint32_t* __restrict__ pl, uint8_t* __restrict__ ov) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const int c = __ldg(runs + 3 * g), top = __ldg(runs + 3 * g + 1), bot = __ldg(runs + 3 * g + 2);
        uint32_t cnt_r = 0, cnt_l = 0, jr = kNoLink, jl = kNoLink;
        const int64_t i_own = g - __ldg(col_off + c);
        const int32_t n_own = __ldg(counts + c);
        const int32_t div = n_own > 0 ? n_own : 1;
        const bool has_r = c + 1 < width, has_l = c > 0;
        const int32_t nr = has_r ? __ldg(counts + c + 1) : 0, nl = has_l ? __ldg(counts + c - 1) : 0;
        const int64_t br = has_r ? __ldg(col_off + c + 1) : 0, bl = has_l ? __ldg(col_off + c - 1) : 0;
        const int64_t er = br + nr, el = bl + nl;
        const int64_t gr = clamp_guess(br, er, br + (i_own * nr) / div), gl = clamp_guess(bl, el, bl + (i_own * nl) / div);
        const int vr = nr > 0 ? __ldg(runs + 3 * gr + 2) : 0, vl = nl > 0 ? __ldg(runs + 3 * gl + 2) : 0;
        if (nr > 0) {
            const int64_t j = first_reaching_from(runs, br, er, top, gr, vr);
            if (j < er) {
                const int t0 = __ldg(runs + 3 * j + 1);
                const int t1 = j + 1 < er ? __ldg(runs + 3 * (j + 1) + 1) : INT_MAX;
                if (t0 <= bot) {
                    cnt_r = 1 + (t1 <= bot);
                    jr = static_cast<uint32_t>(j);
                }
            }
        }
        if (nl > 0) {
            const int64_t j = first_reaching_from(runs, bl, el, top, gl, vl);
            if (j < el) {
                const int t0 = __ldg(runs + 3 * j + 1);
                const int t1 = j + 1 < el ? __ldg(runs + 3 * (j + 1) + 1) : INT_MAX;
                if (t0 <= bot) {
                    cnt_l = 1 + (t1 <= bot);
                    jl = static_cast<uint32_t>(j);
                }
            }
        }
        pr[g] = jr;
        pl[g] = jl;
        ov[g] = static_cast<uint8_t>(cnt_r | (cnt_l << 2));
    }
}

// D2: mutual-uniqueness links; pr[g] becomes the right link (or kNoLink) and
// anc[g] the left link, or g itself for a chain head.
__global__ void __launch_bounds__(kThreadsD) decomp_link_kernel(int64_t n, uint32_t* __restrict__ pr,
                                                                const uint32_t* __restrict__ pl,
                                                                const uint8_t* __restrict__ ov,
                                                                uint32_t* __restrict__ anc) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t o = ov[g];
        const uint32_t r = pr[g], l = pl[g];
        const bool right = (o & 3u) == 1u && (ov[r] >> 2) == 1u;
        const bool left = (o >> 2) == 1u && (ov[l] & 3u) == 1u;
        pr[g] = right ? r : kNoLink;
        anc[g] = left ? l : static_cast<uint32_t>(g);
    }
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// D3: chain heads by concurrent pointer jumping in ONE launch: every run chases
// its ancestor pointer to the head (a fixed point), storing each step back so the
// runs behind it skip ahead (every stored value is an ancestor in the same chain:
// the races only ever shorten a path).  Chains run left to right one column per
// link, so a run's distance to its head is col(run) - col(head) and needs no
// bookkeeping.  (Replaces synchronous rounds over {ancestor, distance} pairs, one
// host round trip each.)
__global__ void __launch_bounds__(kThreadsD) decomp_jump_kernel(int64_t n, uint32_t* __restrict__ anc) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        uint32_t a = ld_volatile(anc + g);
        if (a == static_cast<uint32_t>(g)) continue;
        uint32_t b = ld_volatile(anc + a);
        if (b == a) continue;  // the left neighbour heads the chain
        for (;;) {
            a = b;
            b = ld_volatile(anc + a);
            if (b == a) break;
            anc[g] = b;  // relaxed: a further ancestor for whoever reads it next
        }
        anc[g] = a;
    }
}

constexpr int kWalkMax = 24;  // chains up to this long are walked from their head

// D4: every chain tail stores the chain's length (its column difference + 1) at
// the head; *long_flag marks that D6 has chains longer than kWalkMax.
__global__ void __launch_bounds__(kThreadsD) decomp_tail_kernel(int64_t n, const int32_t* __restrict__ runs,
                                                                const uint32_t* __restrict__ pr,
                                                                const uint32_t* __restrict__ anc,
                                                                uint32_t* __restrict__ head_len,
                                                                int* __restrict__ long_flag) {
    bool any = false;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        if (pr[g] != kNoLink) continue;
        const uint32_t h = anc[g];
        const uint32_t len = static_cast<uint32_t>(__ldg(runs + 3 * g) - __ldg(runs + 3 * int64_t(h))) + 1u;
        head_len[h] = len;
        any |= len > static_cast<uint32_t>(kWalkMax);
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) *long_flag = 1;
}

// D5: exclusive scan of {1 edge, chain length} at every chain head (0 elsewhere)
// in profile order: excl[head] = {edge id, first output slot} -- edges are
// numbered by their head's (column, y_top), exactly the reference's discovery
// order (hypergraph.cpp:145-167).  Reduce-then-scan over tiles of kScanTile runs
// (tile sums, one CTA over the tile sums, tiles); the items are computed from
// anc / head_len on the fly, and only heads are written.  (A one-pass decoupled
// look-back was slower here: ~1000 tiles in flight made every look-back walk
// hundreds of published aggregates.)
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
        const int nw = blockDim.x / 32;
        unsigned long long s = lane < nw ? sh[lane] : 0ull;
        unsigned long long si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < nw) sh[lane] = si - s;
        if (lane == nw - 1) sh[32] = si;
    }
    __syncthreads();
    const unsigned long long r = sh[warp] + inc - x;
    *total = sh[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ unsigned long long head_item(int64_t g, int64_t n, const uint32_t* __restrict__ anc,
                                                        const uint32_t* __restrict__ head_len) {
    return g < n && anc[g] == static_cast<uint32_t>(g) ? pack(1u, head_len[g]) : 0ull;
}

__global__ void __launch_bounds__(kThreadsD) decomp_scan_sums_kernel(int64_t n, const uint32_t* __restrict__ anc,
                                                                     const uint32_t* __restrict__ head_len,
                                                                     unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long sh[33];
    const int64_t base = blockIdx.x * int64_t(kScanTile) + threadIdx.x * int64_t(kScanItems);
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) s += head_item(base + i, n, anc, head_len);
    unsigned long long tot;
    block_exclusive(s, sh, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// One CTA (1024 threads): exclusive scan of the tile sums in place; the grand
// total to *total.
__global__ void __launch_bounds__(1024) decomp_scan_spine_kernel(unsigned long long* __restrict__ sums, int64_t tiles,
                                                                 unsigned long long* __restrict__ total) {
    __shared__ unsigned long long sh[33];
    constexpr int kPer = 8;
    unsigned long long carry = 0;
    for (int64_t b = 0; b < tiles; b += 1024 * kPer) {
        const int64_t i0 = b + threadIdx.x * int64_t(kPer);
        unsigned long long x[kPer], s = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            x[k] = i0 + k < tiles ? sums[i0 + k] : 0ull;
            s += x[k];
        }
        unsigned long long tot;
        unsigned long long run = carry + block_exclusive(s, sh, &tot);
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (i0 + k < tiles) {
                sums[i0 + k] = run;
                run += x[k];
            }
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kThreadsD) decomp_scan_kernel(int64_t n, const uint32_t* __restrict__ anc,
                                                                const uint32_t* __restrict__ head_len,
                                                                const unsigned long long* __restrict__ sums,
                                                                unsigned long long* __restrict__ excl) {
    __shared__ unsigned long long sh[33];
    const int64_t base = blockIdx.x * int64_t(kScanTile) + threadIdx.x * int64_t(kScanItems);
    unsigned long long x[kScanItems];
    unsigned long long s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        x[i] = head_item(base + i, n, anc, head_len);
        s += x[i];
    }
    unsigned long long tot;
    unsigned long long run = sums[blockIdx.x] + block_exclusive(s, sh, &tot);
#pragma unroll
    for (int q = 0; q < kScanItems; q += 4) {  // whole 32-byte sectors that hold a head
        const bool any = (x[q] | x[q + 1] | x[q + 2] | x[q + 3]) != 0;
#pragma unroll
        for (int i = q; i < q + 4; ++i) {
            if (any && base + i < n) excl[base + i] = run;
            run += x[i];
        }
    }
}

// D6: runs into hyperedge order, the run -> edge map, the edge offsets.  Each
// head of a chain of <= kWalkMax runs walks it along the right links and writes
// the records to consecutive output slots.  The heads among a warp's 32
// consecutive runs are consecutive edges, so their chains fill one contiguous
// stretch of the output: staged in shared memory in output order (its first
// kEmitStage records; the rest go straight out) and copied out with consecutive
// 4-byte stores.  A run-by-run scatter to offset(head) + distance wrote 12-byte
// pieces all over the output instead (one store instruction = 32 scattered
// pieces; 2.5x DRAM write amplification, ~70 B per run at 21000^2 checker(7)).
// Longer chains are written run by run by decomp_long_kernel.
constexpr int kEmitStage = 256;  // records per warp staged in shared memory (3 KB)

__global__ void __launch_bounds__(kThreadsD) decomp_emit_kernel(int64_t n, const int32_t* __restrict__ runs,
                                                                const uint32_t* __restrict__ pr,
                                                                const uint32_t* __restrict__ anc,
                                                                const uint32_t* __restrict__ head_len,
                                                                const unsigned long long* __restrict__ excl,
                                                                const unsigned long long* __restrict__ total,
                                                                int32_t* __restrict__ edge_runs,
                                                                uint32_t* __restrict__ edge_offsets,
                                                                uint32_t* __restrict__ run_to_edge) {
    __shared__ int32_t stage[kThreadsD / 32][3 * kEmitStage];
    const int lane = threadIdx.x & 31;
    int32_t* st = stage[threadIdx.x >> 5];
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t g0 = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); g0 < n; g0 += stride) {
        const int64_t g = g0 + lane;
        bool head = false;
        uint32_t e = 0, off = 0;
        if (g < n && anc[g] == static_cast<uint32_t>(g)) {
            const unsigned long long s = excl[g];
            e = static_cast<uint32_t>(s >> 32);
            off = static_cast<uint32_t>(s);
            edge_offsets[e] = off;
            if (g == 0) edge_offsets[*total >> 32] = static_cast<uint32_t>(n);  // run 0 always heads a chain
            head = head_len[g] <= static_cast<uint32_t>(kWalkMax);  // a long chain: decomp_long_kernel
        }
        if (!__any_sync(0xFFFFFFFFu, head)) continue;  // members only: their heads write them
        const uint32_t first = __reduce_min_sync(0xFFFFFFFFu, head ? off : 0xFFFFFFFFu);
        int d = 0;
        if (head) {
            int64_t cur = g;
            const int sbase = static_cast<int>(off - first);  // staged slot of record 0 (may be past the stage)
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
                    break;
                }
                cur = next;
            }
        }
        // (a long chain between two short ones lies inside [first, end): the copy-out
        // writes stale staged ints over its slots, and decomp_long_kernel, launched
        // after this kernel, rewrites all of them)
        const uint32_t end = __reduce_max_sync(0xFFFFFFFFu, head ? off + static_cast<uint32_t>(d) : first);
        __syncwarp();
        const int tot = 3 * static_cast<int>(min(end - first, static_cast<uint32_t>(kEmitStage)));
        int32_t* out = edge_runs + 3 * int64_t(first);
        for (int i = lane; i < tot; i += 32) out[i] = st[i];
        __syncwarp();
    }
}

// D6, chains longer than kWalkMax: run g -> slot offset(head) + (col(g) - col(head)).
__global__ void __launch_bounds__(kThreadsD) decomp_long_kernel(int64_t n, const int32_t* __restrict__ runs,
                                                                const uint32_t* __restrict__ anc,
                                                                const uint32_t* __restrict__ head_len,
                                                                const unsigned long long* __restrict__ excl,
                                                                const int* __restrict__ long_flag,
                                                                int32_t* __restrict__ edge_runs,
                                                                uint32_t* __restrict__ run_to_edge) {
    if (*long_flag == 0) return;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t h = anc[g];
        if (head_len[h] <= static_cast<uint32_t>(kWalkMax)) continue;  // a short chain: its head's walk
        const int32_t c = runs[3 * g], t = runs[3 * g + 1], b = runs[3 * g + 2];
        const unsigned long long s = excl[h];
        const int64_t pos = int64_t(static_cast<uint32_t>(s)) + (c - __ldg(runs + 3 * int64_t(h)));
        edge_runs[3 * pos] = c;
        edge_runs[3 * pos + 1] = t;
        edge_runs[3 * pos + 2] = b;
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
    // pr | pl | anc | head_len (4 B each, 16-B rounded) | excl | tile sums | long flag (16 B) | ov
    const int64_t r4 = ((n * 4 + 15) / 16) * 16;
    return 4 * r4 + n * 8 + tiles * 8 + 16 + n + 256;
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

// The full decomposition of a device profile (n > 0), all on `stream` with no
// host round trip.  Returns 0 or -(cudaError_t).
int ychg_launch_decompose(const int32_t* d_runs, const int64_t* d_col_off, const int32_t* d_counts, int32_t width,
                          int64_t n, void* d_ws, int32_t* d_edge_runs, uint32_t* d_edge_offsets,
                          uint32_t* d_run_to_edge, unsigned long long* d_total, cudaStream_t stream) {
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    const int64_t r4 = ((n * 4 + 15) / 16) * 16;
    uint8_t* p = static_cast<uint8_t*>(d_ws);
    uint32_t* pr = reinterpret_cast<uint32_t*>(p);
    uint32_t* pl = reinterpret_cast<uint32_t*>(p + r4);
    uint32_t* anc = reinterpret_cast<uint32_t*>(p + 2 * r4);
    uint32_t* head_len = reinterpret_cast<uint32_t*>(p + 3 * r4);
    unsigned long long* excl = reinterpret_cast<unsigned long long*>(p + 4 * r4);
    unsigned long long* sums = excl + n;
    int* long_flag = reinterpret_cast<int*>(sums + tiles);
    uint8_t* ov = reinterpret_cast<uint8_t*>(long_flag + 4);
    const int grid = grid_for(n);
    const cudaError_t e0 = cudaMemsetAsync(long_flag, 0, 4, stream);
    if (e0 != cudaSuccess) return -static_cast<int>(e0);
    decomp_overlap_kernel<<<grid, kThreadsD, 0, stream>>>(d_runs, d_col_off, d_counts, width, n, pr, pl, ov);
    decomp_link_kernel<<<grid, kThreadsD, 0, stream>>>(n, pr, pl, ov, anc);
    decomp_jump_kernel<<<grid, kThreadsD, 0, stream>>>(n, anc);
    decomp_tail_kernel<<<grid, kThreadsD, 0, stream>>>(n, d_runs, pr, anc, head_len, long_flag);
    decomp_scan_sums_kernel<<<static_cast<unsigned>(tiles), kThreadsD, 0, stream>>>(n, anc, head_len, sums);
    decomp_scan_spine_kernel<<<1, 1024, 0, stream>>>(sums, tiles, d_total);
    decomp_scan_kernel<<<static_cast<unsigned>(tiles), kThreadsD, 0, stream>>>(n, anc, head_len, sums, excl);
    decomp_emit_kernel<<<grid, kThreadsD, 0, stream>>>(n, d_runs, pr, anc, head_len, excl, d_total, d_edge_runs,
                                                       d_edge_offsets, d_run_to_edge);
    decomp_long_kernel<<<grid, kThreadsD, 0, stream>>>(n, d_runs, anc, head_len, excl, long_flag, d_edge_runs,
                                                       d_run_to_edge);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

}  // extern "C"
