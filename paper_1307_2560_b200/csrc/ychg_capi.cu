// ychg_capi.cu -- the C ABI (include/ychg_b200.h): plans, device/host entry
// points, error convention.  No exception crosses this boundary; statuses map
// to the reference's error classes in the C++ shim (errors.hpp:11-40).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ychg_b200.h"
#include "ychg_device.cuh"
#include "ychg_kernels.h"

using ychg_dev::ScanParams;

namespace {

thread_local std::string g_error;
thread_local int64_t g_error_offset = -1;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_error = buf;
    g_error_offset = -1;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(YCHG_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return fail(YCHG_ERR_NO_DEVICE, "%s: %s (no CPU fallback exists)", what, cudaGetErrorString(e));
    return fail(YCHG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call)                                         \
    do {                                                 \
        const cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

int require_device(int device) {
    static int cached = 0;  // a positive count never changes within a process
    int n = cached;
    cudaError_t e = cudaSuccess;
    if (n == 0) {
        e = cudaGetDeviceCount(&n);
        if (e == cudaSuccess && n > 0) cached = n;
    }
    if (e != cudaSuccess || n == 0)
        return fail(YCHG_ERR_NO_DEVICE, "no CUDA device available (%s); the yCHG path has no CPU fallback",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(YCHG_ERR_INVALID, "device %d out of range [0, %d)", device, n);
    return YCHG_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

}  // namespace

// ---------------------------------------------------------------------------- plans
struct ychg_plan {
    int device = 0;
    ScanParams prm{};
    int grid = 0;                  // streaming grid of the full path (K1+K3)
    int grid_counts = 0;           // streaming grid of the counts-only path
    int64_t ws_bytes = 0;
    void* ws = nullptr;
    // tensor-map cache
    const void* map_ptr = nullptr;
    int64_t map_pitch = 0;
    alignas(64) CUtensorMap map{};
    // timing
    bool timing = false;
    bool latency = false;          // YCHG_PLAN_LATENCY: one-off scans (small images take the single-CTA kernel)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool ev_recorded = false;
    unsigned long long* dbg = nullptr;  // per-CTA %globaltimer stamps (device view of dbg_host)
    unsigned long long* dbg_host = nullptr;  // mapped pinned memory: readable while kernels run
};

namespace {

// Row segments per strip.  Back-to-back scans (the default plan, e.g. graph-
// captured pipelines): about half a CTA per SM per scan -- consecutive scans then
// interleave their CTAs on the SMs' three slots (PDL), every segment is long enough
// to amortise its ramp (first TMA round trip), merge and strip finish, and ~5
// scans are in flight (measured at 21000^2, K=100 graph, us/scan hbands(147) /
// random(0.5): 0.57 CTA/SM (k=4) 9.05 / 11.9; 1 CTA/SM (k=7) 9.2 / 12.5; 3 CTA/SM
// (k=21) 14.8 / 18).  An isolated scan (YCHG_PLAN_LATENCY, the host entry points)
// instead wants every SM streaming at once with more bytes in flight: two CTAs
// per SM (21000^2 hbands / random, one launch, CUDA events: 1/SM 33.4 / 39.0 us,
// 2/SM 28.8 / 34.7, 3/SM 29.5 / 35.5).
// Bounds: a segment holds <= kMaxSegmentRows rows (u16 partials), every warp band
// gets >= 2 blocks (tiny masks: fewer, fuller segments), k <= kMaxSegPerStrip.
int choose_segments(int n_strips, int n_blocks, int sms, int warps, bool latency) {
    const int max_seg_blocks = ychg_dev::kMaxSegmentRows / ychg_dev::kBlockRows;
    const int kmin = std::max(1, (n_blocks + max_seg_blocks - 1) / max_seg_blocks);
    const int ns = std::max(1, n_strips);
    static const int lat_per_sm = [] {
        const char* v = getenv("YCHG_LAT_CTAS_PER_SM");  // A/B timing hook (default 2)
        return v && *v ? std::max(1, atoi(v)) : 2;
    }();
    int k = latency ? lat_per_sm * sms / ns : (sms + ns) / (2 * ns);  // floor(sms / S) | round(sms / 2S)
    // ... and segments of at most 8192 rows (2048 rows per warp band) for tall masks:
    // 65536^2 (64 strips), K=100 graph, hbands / random: k=2 136 / 106 us, k=4 120 /
    // 103, k=8 90 / 110, k=16 102 / -- (round(sms / 2S) alone would give k=1 -> 2)
    if (!latency) k = std::max(k, (n_blocks + 255) / 256);
    k = std::max(1, k);
    k = std::min(k, std::max(1, n_blocks / (2 * warps)));
    k = std::min(k, ychg_dev::kMaxSegPerStrip);
    return std::max(k, kmin);
}
}  // namespace

extern "C" {

const char* ychg_last_error(void) { return g_error.c_str(); }

int64_t ychg_last_error_offset(void) { return g_error_offset; }

int ychg_abi_version(void) { return YCHG_ABI_VERSION; }

int ychg_device_count(int* n) {
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (n) *n = (e == cudaSuccess) ? c : 0;
    return YCHG_OK;
}

int ychg_set_device(int device) {
    if (const int rc = require_device(device)) return rc;
    CK(cudaSetDevice(device));
    return YCHG_OK;
}

int ychg_plan_create(int device, int32_t width_img, int32_t width_cnt, int32_t height, ychg_plan** out) {
    return ychg_plan_create_ex(device, width_img, width_cnt, height, 0, out);
}

int ychg_plan_create_ex(int device, int32_t width_img, int32_t width_cnt, int32_t height, int32_t flags,
                        ychg_plan** out) {
    if (!out) return fail(YCHG_ERR_INVALID, "plan_create: out is NULL");
    *out = nullptr;
    if (width_img < 0 || height < 0 || width_cnt < 0 || width_cnt > width_img)
        return fail(YCHG_ERR_INVALID, "plan_create: bad geometry width_img=%d width_cnt=%d height=%d",
                    width_img, width_cnt, height);
    if (const int rc = require_device(device)) return rc;
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));

    auto plan = std::make_unique<ychg_plan>();
    plan->latency = (flags & YCHG_PLAN_LATENCY) != 0;
    plan->device = device;
    ScanParams& p = plan->prm;
    p.width_img = width_img;
    p.width_cnt = width_cnt;
    p.height = height;
    p.row_bytes = (width_img + 7) / 8;
    p.n_strips = (width_cnt + ychg_dev::kStripCols - 1) / ychg_dev::kStripCols;
    p.n_blocks = (height + ychg_dev::kBlockRows - 1) / ychg_dev::kBlockRows;
    if (p.n_strips > 0 && p.n_blocks > 0) {
        p.wait_inputs = (flags & YCHG_PLAN_SYNC_INPUTS) ? 1 : 0;
        p.skip_same = (flags & YCHG_PLAN_NO_SKIP) ? 0 : 1;
        if (const char* v = getenv("YCHG_NO_SKIP"); v && v[0] == '1') p.skip_same = 0;  // A/B timing hook
        // An isolated scan starts every CTA at once: one box per warp first gets each
        // warp's data back sooner, the rest of the ring follows (pipelined plans
        // start CTAs one by one as slots free, the whole ring at once)
        p.ramp_boxes = (flags & YCHG_PLAN_LATENCY) ? 1 : 0;
        if (const char* v = getenv("YCHG_RAMP_BOXES"); v && *v) p.ramp_boxes = atoi(v);  // A/B hook
        if (const char* v = getenv("YCHG_RAMP_BOXES"); v && *v) p.ramp_boxes = atoi(v);  // A/B timing hook
        // Resident CTAs per SM of each path's kernel (its grid is capped to what is
        // resident: a strip finisher may wait on other CTAs of the same scan).
        if (const int rc2 = ychg_scan_kernel_prepare())
            return cuda_fail(static_cast<cudaError_t>(rc2), "scan kernel smem opt-in");
        int per_path[2] = {0, 0}, warps[2] = {0, 0};
        for (int path = 0; path < 2; ++path) {
            int thr = 0, smem = 0;
            ychg_scan_kernel_shape(path, &thr, &smem);
            warps[path] = thr / 32;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_path[path], ychg_scan_kernel_ptr(path), thr, smem));
            if (per_path[path] < 1) return fail(YCHG_ERR_CUDA, "scan kernel does not fit on an SM");
        }
        p.seg_per_strip = choose_segments(p.n_strips, p.n_blocks, sms, warps[1], (flags & YCHG_PLAN_LATENCY) != 0);
        // experiment hook (benchmarking only): force the segments per strip
        if (const char* v = getenv("YCHG_SEGMENTS"); v && *v)
            p.seg_per_strip = std::max(1, std::min(atoi(v), p.n_blocks));  // a segment must not be empty
        p.n_segments = p.n_strips * p.seg_per_strip;
        if (p.seg_per_strip > ychg_dev::kMaxSegPerStrip)
            return fail(YCHG_ERR_INVALID, "plan_create: height %d needs more than %d row segments per strip",
                        height, ychg_dev::kMaxSegPerStrip);
        plan->grid = std::min(p.n_segments, per_path[1] * sms);
        plan->grid_counts = std::min(p.n_segments, per_path[0] * sms);
        if (const char* v = getenv("YCHG_GRID"); v && *v) {
            plan->grid = std::max(1, std::min(atoi(v), plan->grid));
            plan->grid_counts = std::max(1, std::min(atoi(v), plan->grid_counts));
        }
        for (const int g : {plan->grid, plan->grid_counts})
            if ((p.n_segments + g - 1) / g > ychg_dev::kMaxSegPerCta)
                return fail(YCHG_ERR_INVALID, "plan_create: %d segments over %d CTAs exceed %d per CTA",
                            p.n_segments, g, ychg_dev::kMaxSegPerCta);
        const int64_t S = p.n_strips, G = p.n_segments;
        // part / sums / seg_links / rec are double-buffered by scan parity
        const int64_t sz_part = 2 * G * 512 * 4, sz_sums = 2 * G * ychg_dev::kSumPlanes * 32 * 4;
        // strip records pack column counts (<= ceil(height/2)) in 21 bits
        if (height > (1 << 22) - 2)
            return fail(YCHG_ERR_INVALID, "plan_create: height %d > 2^22-2 rows is not supported", height);
        const int64_t sz_rec = 2 * S * int64_t(sizeof(ychg_dev::StripRecord));
        // order: part | sums | seg_links[2][G] | seg_ticket[G] | arrive[2][S] | fin_all | fin_loaded[2][S] | rec[2][S]
        plan->ws_bytes = sz_part + sz_sums + 2 * G * 8 + G * 8 + 2 * S * 8 + 64 + 2 * S * 8 + sz_rec + 64;
        cudaError_t e = cudaMalloc(&plan->ws, plan->ws_bytes);
        if (e != cudaSuccess) {
            plan->ws = nullptr;
            return cuda_fail(e, "plan workspace cudaMalloc");
        }
        // zeroed before any stream can use the plan (the counters are never reset)
        e = cudaMemset(plan->ws, 0, plan->ws_bytes);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            cudaFree(plan->ws);
            plan->ws = nullptr;
            return cuda_fail(e, "plan workspace cudaMemset");
        }
        char* w = static_cast<char*>(plan->ws);
        p.part = reinterpret_cast<uint32_t*>(w);
        w += sz_part;
        p.sums = reinterpret_cast<uint32_t*>(w);
        w += sz_sums;
        p.seg_links = reinterpret_cast<unsigned long long*>(w);
        w += 2 * G * 8;
        p.seg_ticket = reinterpret_cast<unsigned long long*>(w);
        w += G * 8;
        p.arrive = reinterpret_cast<unsigned long long*>(w);
        w += 2 * S * 8;
        p.fin_all = reinterpret_cast<unsigned long long*>(w);
        w += 64;
        p.fin_loaded = reinterpret_cast<unsigned long long*>(w);
        w += 2 * S * 8;
        p.rec = reinterpret_cast<ychg_dev::StripRecord*>(w);
    }
    *out = plan.release();
    return YCHG_OK;
}

void ychg_plan_destroy(ychg_plan* plan) {
    if (!plan) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(plan->device);
    if (plan->ws) cudaFree(plan->ws);
    if (plan->dbg_host) cudaFreeHost(plan->dbg_host);
    for (auto& e : plan->ev)
        if (e) cudaEventDestroy(e);
    cudaSetDevice(prev);
    delete plan;
}

int ychg_plan_get_info(const ychg_plan* plan, ychg_plan_info* out) {
    if (!plan || !out) return fail(YCHG_ERR_INVALID, "plan_get_info: NULL argument");
    out->n_strips = plan->prm.n_strips;
    out->n_blocks = plan->prm.n_blocks;
    out->seg_per_strip = plan->prm.seg_per_strip;
    out->n_segments = plan->prm.n_segments;
    out->grid = plan->grid;
    out->kernels_per_scan = (plan->prm.n_strips > 0 && plan->prm.n_blocks > 0) ? 1 : 0;
    out->workspace_bytes = plan->ws_bytes;
    return YCHG_OK;
}

int ychg_plan_set_timing(ychg_plan* plan, int32_t enabled) {
    if (!plan) return fail(YCHG_ERR_INVALID, "plan_set_timing: NULL plan");
    CK(cudaSetDevice(plan->device));
    if (enabled && !plan->ev[0])
        for (auto& e : plan->ev) CK(cudaEventCreate(&e));
    plan->timing = enabled != 0;
    plan->ev_recorded = false;
    return YCHG_OK;
}

int ychg_plan_last_ms(ychg_plan* plan, float* scan_ms, float* finish_ms) {
    if (!plan || !plan->ev_recorded) return fail(YCHG_ERR_INVALID, "plan_last_ms: no timed scan recorded");
    CK(cudaEventSynchronize(plan->ev[1]));
    float a = 0;
    CK(cudaEventElapsedTime(&a, plan->ev[0], plan->ev[1]));
    if (scan_ms) *scan_ms = a;
    if (finish_ms) *finish_ms = 0.0f;  // the finish is fused into the streaming kernel
    return YCHG_OK;
}

int ychg_plan_debug_stamps(ychg_plan* plan, int32_t enable, uint64_t* host_out, int32_t capacity,
                           int32_t* n_ctas) {
    if (!plan) return fail(YCHG_ERR_INVALID, "plan_debug_stamps: NULL plan");
    CK(cudaSetDevice(plan->device));
    const int64_t bytes = int64_t(std::max(std::max(plan->grid, plan->grid_counts), plan->prm.n_strips)) * 32 * 8 * ychg_dev::kStampRing;
    if (enable && !plan->dbg && plan->grid > 0) {
        // zero-copy host memory, so a stalled pipeline can still be inspected (debug_peek)
        CK(cudaHostAlloc(reinterpret_cast<void**>(&plan->dbg_host), bytes, cudaHostAllocMapped));
        std::memset(plan->dbg_host, 0, size_t(bytes));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&plan->dbg), plan->dbg_host, 0));
    }
    if (!enable && plan->dbg) {
        CK(cudaDeviceSynchronize());
        CK(cudaFreeHost(plan->dbg_host));
        plan->dbg = plan->dbg_host = nullptr;
    }
    if (n_ctas) *n_ctas = std::max(std::max(plan->grid, plan->grid_counts), plan->prm.n_strips);  // stamp rows
    if (host_out && plan->dbg) {
        const int64_t n = std::min<int64_t>(capacity, bytes / 8);
        CK(cudaDeviceSynchronize());
        std::memcpy(host_out, plan->dbg_host, size_t(n) * 8);
    }
    return YCHG_OK;
}

// Diagnostics: copy the stamp ring without synchronising (works while kernels stall).
int ychg_plan_debug_peek(ychg_plan* plan, uint64_t* host_out, int32_t capacity) {
    if (!plan || !plan->dbg_host) return fail(YCHG_ERR_INVALID, "plan_debug_peek: stamps not enabled");
    const int64_t bytes = int64_t(std::max(std::max(plan->grid, plan->grid_counts), plan->prm.n_strips)) * 32 * 8 * ychg_dev::kStampRing;
    std::memcpy(host_out, const_cast<const unsigned long long*>(plan->dbg_host),
                size_t(std::min<int64_t>(capacity, bytes / 8)) * 8);
    return YCHG_OK;
}

// L2 promotion of the image's TMA boxes (YCHG_TMAP_PROMO=0..3: none / 64 / 128 /
// 256 B; A/B hook, default 256 B).
static CUtensorMapL2promotion tmap_promotion() {
    static const CUtensorMapL2promotion p = [] {
        const char* v = getenv("YCHG_TMAP_PROMO");
        const int i = v && *v ? atoi(v) : 3;
        return i == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
               : i == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
               : i == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                        : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    return p;
}

int ychg_scan_device(ychg_plan* plan, const uint8_t* d_bits, int64_t pitch, int32_t with_hyperedges,
                     int32_t* d_counts, uint32_t* d_flags, int32_t* d_boundaries, ychg_totals* d_totals,
                     void* stream) {
    if (!plan) return fail(YCHG_ERR_INVALID, "scan_device: NULL plan");
    ScanParams& p = plan->prm;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(plan->device));
    if (!d_totals) return fail(YCHG_ERR_INVALID, "scan_device: d_totals is required");
    if (p.n_strips == 0 || p.n_blocks == 0) {
        // W == 0 or H == 0: all-zero counts, no boundaries, no runs (runscan.cpp:122-128).
        CK(cudaMemsetAsync(d_totals, 0, sizeof(ychg_totals), st));
        if (!with_hyperedges) {
            const long long m1 = -1;
            CK(cudaMemcpyAsync(&d_totals->hyperedges, &m1, sizeof(m1), cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
        }
        if (d_counts && p.width_cnt > 0) CK(cudaMemsetAsync(d_counts, 0, int64_t(p.width_cnt) * 4, st));
        if (d_flags && p.width_cnt > 0) CK(cudaMemsetAsync(d_flags, 0, int64_t((p.width_cnt + 31) / 32) * 4, st));
        return YCHG_OK;
    }
    if (!d_bits || !d_counts || !d_flags || !d_boundaries)
        return fail(YCHG_ERR_INVALID, "scan_device: NULL device buffer");
    if (pitch < p.row_bytes || pitch % 16 != 0)
        return fail(YCHG_ERR_INVALID, "scan_device: pitch %lld must be >= %d and a multiple of 16",
                    static_cast<long long>(pitch), p.row_bytes);
    if (reinterpret_cast<uintptr_t>(d_bits) % 16 != 0)
        return fail(YCHG_ERR_INVALID, "scan_device: image base must be 16-byte aligned");

    // A one-off scan of a small image (one strip, <= 512 rows): the single-CTA
    // kernel (no TMA ring / scan protocol: 32^2 isolated 16 -> 13 us, drop-in call
    // 39 -> 33 us; from ~1000 rows on the multi-CTA latency plan is faster).
    const char* no_small_env = getenv("YCHG_NO_SMALL");  // A/B hook (read per call: tests switch it)
    const bool no_small = no_small_env && no_small_env[0] == '1';
    if (plan->latency && !no_small && p.n_strips == 1 && p.height <= 512 && p.width_img <= 1024) {
        ScanParams q = p;
        q.bits = d_bits;
        q.pitch = pitch;
        q.counts = d_counts;
        q.flags = d_flags;
        q.boundaries = d_boundaries;
        q.totals = reinterpret_cast<long long*>(d_totals);
        q.mul2 = 2u;
        q.mul1 = 1u;
        q.mulm1 = 0xFFFFFFFFu;
        q.mulnb = 1u << 25;
        if (plan->timing) CK(cudaEventRecord(plan->ev[0], st));
        const int rc = ychg_launch_small(&q, with_hyperedges ? 1 : 0, st);
        if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "small-image scan kernel launch");
        if (plan->timing) {
            CK(cudaEventRecord(plan->ev[1], st));
            plan->ev_recorded = true;
        }
        return YCHG_OK;
    }
    if (plan->map_ptr != d_bits || plan->map_pitch != pitch) {
        auto encode = tensor_map_encoder();
        if (!encode) return fail(YCHG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.row_bytes), static_cast<cuuint64_t>(p.height)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch)};
        cuuint32_t box[2] = {ychg_dev::kBoxBytes, ychg_dev::kBlockRows};
        cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(&plan->map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(d_bits),
                                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_NONE, tmap_promotion(),
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(YCHG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
        plan->map_ptr = d_bits;
        plan->map_pitch = pitch;
    }
    p.bits = d_bits;
    p.pitch = pitch;
    p.counts = d_counts;
    p.flags = d_flags;
    p.boundaries = d_boundaries;
    p.totals = reinterpret_cast<long long*>(d_totals);
    p.dbg = plan->dbg;
    p.dbg_rows = std::max(std::max(plan->grid, plan->grid_counts), p.n_strips);
    p.mul2 = 2u;
    p.mul1 = 1u;
    p.mulm1 = 0xFFFFFFFFu;
    p.mulnb = 1u << 25;

    if (plan->timing) CK(cudaEventRecord(plan->ev[0], st));
    const int rc = ychg_launch_scan(&plan->map, &p, with_hyperedges ? plan->grid : plan->grid_counts,
                                    with_hyperedges ? 1 : 0, st);
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "scan kernel launch");
    if (plan->timing) {
        CK(cudaEventRecord(plan->ev[1], st));
        plan->ev_recorded = true;
    }
    return YCHG_OK;
}

int ychg_synth_device(int32_t pattern, int32_t width, int32_t height, int32_t bands, int32_t cell,
                      double density, uint64_t seed, uint8_t* d_bits, int64_t pitch, void* stream) {
    return ychg_synth_device_window(pattern, width, height, 0, width, bands, cell, density, seed, d_bits, pitch,
                                    stream);
}

int ychg_synth_device_window(int32_t pattern, int32_t width, int32_t height, int32_t x0, int32_t win,
                             int32_t bands, int32_t cell, double density, uint64_t seed, uint8_t* d_bits,
                             int64_t pitch, void* stream) {
    // Validation as synth.cpp:10-34.
    if (width < 0 || height < 0) return fail(YCHG_ERR_INVALID, "synth: negative dimensions %dx%d", width, height);
    if (pattern < 0 || pattern > 5) return fail(YCHG_ERR_INVALID, "synth: unknown pattern %d", pattern);
    if (pattern == YCHG_PATTERN_HBANDS && (bands < 1 || bands > height / 2))
        return fail(YCHG_ERR_INVALID, "synth: hbands(%d) needs 1 <= k <= height/2 = %d", bands, height / 2);
    if (pattern == YCHG_PATTERN_CHECKER && cell < 1)
        return fail(YCHG_ERR_INVALID, "synth: checker cell must be >= 1, got %d", cell);
    if (pattern == YCHG_PATTERN_RANDOM && !(density >= 0.0 && density <= 1.0))
        return fail(YCHG_ERR_INVALID, "synth: random density must lie in [0, 1], got %f", density);
    if (x0 < 0 || x0 % 8 != 0 || win < 0 || x0 > width)
        return fail(YCHG_ERR_INVALID, "synth: window x0=%d (a multiple of 8 in [0, %d]) width %d", x0, width, win);
    if (pitch < (win + 7) / 8) return fail(YCHG_ERR_INVALID, "synth: pitch too small");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (const int rc = require_device(dev)) return rc;
    const int rc = ychg_launch_synth_window(pattern, width, height, x0, win, bands, cell, density, seed, d_bits,
                                            pitch, static_cast<cudaStream_t>(stream));
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "synth kernel launch");
    return YCHG_OK;
}

// ---------------------------------------------------------------------------- memory helpers
int ychg_device_alloc(int device, int64_t bytes, void** out) {
    if (!out) return fail(YCHG_ERR_INVALID, "device_alloc: out is NULL");
    if (const int rc = require_device(device)) return rc;
    CK(cudaSetDevice(device));
    CK(cudaMalloc(out, bytes > 0 ? bytes : 16));
    return YCHG_OK;
}
int ychg_device_free(int device, void* p) {
    CK(cudaSetDevice(device));
    CK(cudaFree(p));
    return YCHG_OK;
}
int ychg_host_alloc_pinned(int64_t bytes, void** out) {
    if (!out) return fail(YCHG_ERR_INVALID, "host_alloc_pinned: out is NULL");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(YCHG_ERR_NO_DEVICE, "no CUDA device available for pinned allocation");
    CK(cudaMallocHost(out, bytes > 0 ? bytes : 16));
    return YCHG_OK;
}
int ychg_host_free_pinned(void* p) {
    CK(cudaFreeHost(p));
    return YCHG_OK;
}
int ychg_memcpy(void* dst, const void* src, int64_t bytes, void* stream) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    return YCHG_OK;
}
int ychg_memcpy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
                   int64_t height, void* stream) {
    CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyDefault,
                         static_cast<cudaStream_t>(stream)));
    return YCHG_OK;
}
int ychg_memset(void* dst, int32_t value, int64_t bytes, void* stream) {
    CK(cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream)));
    return YCHG_OK;
}
int ychg_stream_create(int device, void** out) {
    if (const int rc = require_device(device)) return rc;
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *out = s;
    return YCHG_OK;
}
int ychg_stream_destroy(void* stream) {
    CK(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
    return YCHG_OK;
}
int ychg_stream_synchronize(void* stream) {
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return YCHG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------- host entry points
namespace {

// Per-device cached state for the host-buffer API.  One mutex per device
// serialises callers (the reference functions are reentrant; so are these).
struct HostContext {
    std::mutex mu;
    int device = 0;
    bool ready = false;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;   // H2D chunks overlap the re-pitch of the previous chunk
    static constexpr int kChunks = 4;
    cudaEvent_t chunk_ev[kChunks] = {};
    uint8_t* d_dense = nullptr;            // dense staging copy of the host rows
    int64_t dense_cap = 0;
    ychg_plan* plan = nullptr;
    int32_t plan_w = -1, plan_wc = -1, plan_h = -1;  // host plan: image width, counted width, height
    uint8_t* d_bits = nullptr;
    int64_t bits_cap = 0;
    int32_t* d_counts = nullptr;
    uint32_t* d_flags = nullptr;
    int32_t* d_bounds = nullptr;
    int64_t cols_cap = 0;
    ychg_totals* d_totals = nullptr;
    ychg_totals* h_totals = nullptr;  // pinned
    // run materialisation (build_profile / column_runs)
    uint32_t* d_band = nullptr;
    int64_t band_cap = 0;
    int64_t* d_col_off = nullptr;
    int64_t col_off_cap = 0;
    int32_t* d_runs = nullptr;
    int64_t runs_cap = 0;
    int32_t* h_out = nullptr;         // pinned staging: counts | boundaries (capacity cols_cap each)
    char* d_block = nullptr;          // device [totals | counts | boundaries] (ensure_columns)
    // host scan outputs [totals (64 B) | counts (cols_cap) | boundaries (cols_cap)] in
    // MAPPED pinned memory: the finisher's stores cross PCIe as it runs, so the
    // host path needs no separate D2H copy after the scan (one fewer round trip)
    char* m_block = nullptr;
    char* m_block_dev = nullptr;
    int64_t m_block_cap = 0;
    bool h2d_timing = false;
    cudaEvent_t h2d_ev[3] = {nullptr, nullptr, nullptr};
    int64_t h_out_cap = 0;
    // hyperedge decomposition
    void* d_dws = nullptr;
    int64_t dws_cap = 0;
    unsigned long long* d_dscal = nullptr;  // [0] edge/run totals, [1] validation error
    unsigned long long* h_dscal = nullptr;  // pinned
    cudaEvent_t dec_ev[2] = {nullptr, nullptr};
    // pageable host input: pinned staging ring (see h2d_staged)
    static constexpr int kStageSlots = 3;
    uint8_t* h_stage[kStageSlots] = {};
    int64_t stage_bytes = 0;
    cudaEvent_t stage_ev[kStageSlots] = {};
    uint8_t* h_col_stage = nullptr;  // column_runs: one byte column at a 16-byte pitch (pinned)
    int64_t col_stage_cap = 0;
};

HostContext& host_context(int device) {
    static HostContext ctx[64];
    ctx[device].device = device;
    return ctx[device];
}

int ensure_context(HostContext& c) {
    CK(cudaSetDevice(c.device));
    if (!c.ready) {
        CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
        for (auto& e : c.chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : c.stage_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        const char* ht = getenv("YCHG_HOST_TIMING");
        c.h2d_timing = ht && ht[0] == '1';
        if (c.h2d_timing)
            for (auto& e : c.h2d_ev) CK(cudaEventCreate(&e));
        CK(cudaMalloc(&c.d_totals, sizeof(ychg_totals)));
        CK(cudaMallocHost(&c.h_totals, sizeof(ychg_totals)));
        c.ready = true;
    }
    return YCHG_OK;
}

// Parallel host memcpy for pageable inputs: the caller plus persistent workers
// split each chunk.  One job at a time (callers of several devices serialise
// here); the pool is never destroyed, so no worker outlives its condition
// variables at process exit.
class CopyPool {
   public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();
        return *pool;
    }
    void copy(uint8_t* dst, const uint8_t* src, size_t n) {
        const int parts = static_cast<int>(workers_.size()) + 1;
        if (parts == 1 || n < (size_t(1) << 18)) {
            std::memcpy(dst, src, n);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = dst;
            src_ = src;
            n_ = n;
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

   private:
    CopyPool() {
        // 3-4 copiers saturate a B200 host's memory copy rate (scripts/stage_sweep.sh)
        int t = std::min(4, static_cast<int>(std::thread::hardware_concurrency()));
        if (const char* v = getenv("YCHG_COPY_THREADS"); v && *v) t = atoi(v);
        t = std::max(1, std::min(t, 16));
        for (int i = 1; i < t; ++i) {
            workers_.emplace_back([this, i] { loop(i); });
            workers_.back().detach();
        }
    }
    void part(int i) {
        // 4 KB-aligned slices
        const size_t per = ((n_ + parts_ - 1) / parts_ + 4095) & ~size_t(4095);
        const size_t b = std::min(n_, per * i), e = std::min(n_, b + per);
        if (e > b) std::memcpy(dst_ + b, src_ + b, e - b);
    }
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            part(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    int pending_ = 0, parts_ = 1;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t n_ = 0;
};

// H2D of `bytes` bytes of PAGEABLE host memory into d_dst, ending on c.stream:
// chunks go through a ring of pinned slots, each filled by the copy pool while
// the DMA of the previous one runs on c.copy_stream (the driver's own staging of
// pageable copies reaches ~19 GB/s; this pipeline runs at the DMA rate).
int h2d_staged(HostContext& c, uint8_t* d_dst, const uint8_t* src, int64_t bytes) {
    static const int64_t chunk = [] {
        const char* v = getenv("YCHG_STAGE_MB");  // experiment hook
        const int64_t mb = v && *v ? atoll(v) : 4;
        return std::max<int64_t>(1, mb) << 20;
    }();
    if (c.stage_bytes < chunk) {
        for (auto& p : c.h_stage) {
            cudaFreeHost(p);
            p = nullptr;
        }
        c.stage_bytes = 0;
        for (auto& p : c.h_stage) CK(cudaMallocHost(&p, chunk));
        c.stage_bytes = chunk;
    }
    static const int64_t direct_max = [] {
        // small inputs: the driver's own staged copy has no pool hand-off and a
        // steadier latency (4096^2, 2 MB: 150 us vs a bimodal 250/430 us through
        // the pool on a 16-core host, scripts/host_counts_probe.py)
        const char* v = getenv("YCHG_PAGEABLE_DIRECT_MB");
        return (v && *v ? atoll(v) : 4) << 20;
    }();
    if (bytes <= direct_max) {
        CK(cudaMemcpyAsync(d_dst, src, bytes, cudaMemcpyHostToDevice, c.stream));
        return YCHG_OK;
    }
    // the copy stream must not overwrite device memory still read by earlier work on c.stream
    CK(cudaEventRecord(c.chunk_ev[0], c.stream));
    CK(cudaStreamWaitEvent(c.copy_stream, c.chunk_ev[0], 0));
    CopyPool& pool = CopyPool::get();
    int64_t i = 0;
    for (int64_t off = 0; off < bytes; off += chunk, ++i) {
        const int slot = static_cast<int>(i % HostContext::kStageSlots);
        if (i >= HostContext::kStageSlots) CK(cudaEventSynchronize(c.stage_ev[slot]));  // slot's DMA done
        const int64_t len = std::min(chunk, bytes - off);
        pool.copy(c.h_stage[slot], src + off, static_cast<size_t>(len));
        CK(cudaMemcpyAsync(d_dst + off, c.h_stage[slot], len, cudaMemcpyHostToDevice, c.copy_stream));
        CK(cudaEventRecord(c.stage_ev[slot], c.copy_stream));
    }
    CK(cudaEventRecord(c.chunk_ev[1], c.copy_stream));
    CK(cudaStreamWaitEvent(c.stream, c.chunk_ev[1], 0));
    return YCHG_OK;
}

// Outputs live in one device block [totals (64 B) | counts (cap) | boundaries (cap)]
// so the host path reads all of them back with a single copy.
int ensure_columns(HostContext& c, int64_t cols) {
    if (cols <= c.cols_cap) return YCHG_OK;
    cudaFree(c.d_block);
    cudaFree(c.d_flags);
    c.d_block = nullptr;
    c.d_counts = nullptr;
    c.d_flags = nullptr;
    c.d_bounds = nullptr;
    c.cols_cap = 0;
    const int64_t cap = std::max<int64_t>(cols, 1024);
    // flags: one word per 32 columns, rounded to whole 1024-column blocks, + per-block scratch
    const int64_t fwords = ((cap + 1023) / 1024) * 32 + (cap + 1023) / 1024 + 32;
    CK(cudaMalloc(&c.d_block, 64 + cap * 8));
    CK(cudaMalloc(&c.d_flags, fwords * 4));
    c.d_totals = reinterpret_cast<ychg_totals*>(c.d_block);
    c.d_counts = reinterpret_cast<int32_t*>(c.d_block + 64);
    c.d_bounds = c.d_counts + cap;
    c.cols_cap = cap;
    return YCHG_OK;
}

int pick_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    return dev;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// H2D into context memory on c.stream: pinned sources by DMA, pageable ones via h2d_staged.
int h2d_any(HostContext& c, uint8_t* d_dst, const uint8_t* src, int64_t bytes) {
    if (is_pinned(src)) {
        CK(cudaMemcpyAsync(d_dst, src, bytes, cudaMemcpyHostToDevice, c.stream));
        return YCHG_OK;
    }
    return h2d_staged(c, d_dst, src, bytes);
}

}  // namespace

// H2D of the caller's rows into the context's pitched device image.  Row strides
// that are already TMA-legal (multiple of 16 B) copy straight into place.
// Otherwise the rows go over PCIe as one dense 1-D stream (2-D copies of
// odd-sized rows run at less than half the link rate) in chunks on a copy
// stream, each chunk re-pitched on the device by a kernel while the next chunk
// is still in flight.
int upload_image(HostContext& c, const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride) {
    const int64_t row_bytes = (int64_t(width) + 7) / 8;
    const int64_t pitch = (row_bytes + 15) / 16 * 16;
    const int64_t need = pitch * height;
    if (need > c.bits_cap) {
        cudaFree(c.d_bits);
        c.d_bits = nullptr;
        c.bits_cap = 0;
        CK(cudaMalloc(&c.d_bits, need));
        c.bits_cap = need;
    }

    // pageable rows (e.g. the reference BinaryImage's std::vector) go through the
    // pinned staging pipeline; strided pageable rows are left to the driver
    const bool pinned = is_pinned(bits);
    if (row_stride == pitch) {
        if (pinned) CK(cudaMemcpyAsync(c.d_bits, bits, pitch * height, cudaMemcpyHostToDevice, c.stream));
        else if (const int rc = h2d_staged(c, c.d_bits, bits, pitch * height)) return rc;
    } else if (row_stride != row_bytes) {
        CK(cudaMemcpy2DAsync(c.d_bits, pitch, bits, row_stride, row_bytes, height, cudaMemcpyHostToDevice,
                             c.stream));
    } else {
        const int64_t dense = row_bytes * height;
        if (dense + 32 > c.dense_cap) {
            cudaFree(c.d_dense);
            c.d_dense = nullptr;
            c.dense_cap = 0;
            CK(cudaMalloc(&c.d_dense, dense + 32));
            c.dense_cap = dense + 32;
        }
        if (!pinned) {
            if (c.h2d_timing) cudaEventRecord(c.h2d_ev[0], c.stream);
            if (const int rc = h2d_staged(c, c.d_dense, bits, dense)) return rc;
            if (c.h2d_timing) cudaEventRecord(c.h2d_ev[1], c.stream);
            const int rc = ychg_launch_repitch(c.d_dense, row_bytes, c.d_bits, pitch, 0, height, c.stream);
            if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "repitch kernel launch");
            if (c.h2d_timing) cudaEventRecord(c.h2d_ev[2], c.stream);
            return YCHG_OK;
        }
        CK(cudaEventRecord(c.chunk_ev[0], c.stream));  // order after earlier work on c.stream
        CK(cudaStreamWaitEvent(c.copy_stream, c.chunk_ev[0], 0));
        if (c.h2d_timing) cudaEventRecord(c.h2d_ev[0], c.copy_stream);
        static const int max_chunks = [] {
            const char* v = getenv("YCHG_H2D_CHUNKS");  // experiment hook (1..4)
            const int n = v && *v ? atoi(v) : 2;  // 2: overlaps the re-pitch with fewer API calls
            return n < 1 ? 1 : (n > HostContext::kChunks ? HostContext::kChunks : n);
        }();
        const int nch = height >= max_chunks * 64 ? max_chunks : 1;
        // The last chunk is a sixteenth of the rows: only its re-pitch is exposed after
        // the final copy; the earlier chunks' re-pitch hides under the later copies.
        static const int tail_div = [] {
            const char* v = getenv("YCHG_H2D_TAIL_DIV");  // experiment hook: tail chunk = rows / div
            const int d = v && *v ? atoi(v) : 16;  // 1/8 1.071, 1/16 1.068, 1/32 1.070 ms (21000^2)
            return d < 2 ? 2 : d;
        }();
        const int tail = nch > 1 ? height / tail_div : 0;
        for (int i = 0; i < nch; ++i) {
            const int y0 = static_cast<int>((int64_t(height - tail) * i) / (nch - (nch > 1)));
            const int y1 = i == nch - 1 ? height : static_cast<int>((int64_t(height - tail) * (i + 1)) / (nch - 1));
            CK(cudaMemcpyAsync(c.d_dense + y0 * row_bytes, bits + y0 * row_bytes, (y1 - y0) * row_bytes,
                               cudaMemcpyHostToDevice, c.copy_stream));
            CK(cudaEventRecord(c.chunk_ev[i], c.copy_stream));
            CK(cudaStreamWaitEvent(c.stream, c.chunk_ev[i], 0));
            const int rc = ychg_launch_repitch(c.d_dense, row_bytes, c.d_bits, pitch, y0, y1, c.stream);
            if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "repitch kernel launch");
        }
        if (c.h2d_timing) {
            cudaEventRecord(c.h2d_ev[1], c.copy_stream);
            cudaEventRecord(c.h2d_ev[2], c.stream);
        }
    }
    return YCHG_OK;
}

// The host scan on a locked, ready context: `upload` fills c.d_bits (pitched)
// on c.stream; then one scan and one D2H round trip.
// `width` columns are counted; the image in c.d_bits holds width_img >= width
// columns (a column strip with its right halo, see ychg_scan_host_sharded).
template <typename Upload>
int scan_host_locked(HostContext& c, int device, int32_t width, int32_t height, int32_t with_hyperedges,
                     int32_t* counts_out, int32_t* boundaries_out, ychg_totals* totals_out, Upload&& upload,
                     int32_t width_img = -1, int32_t* d_counts_dst = nullptr) {
    if (width_img < width) width_img = width;
    const int64_t row_bytes = (int64_t(width_img) + 7) / 8;

    if (width == 0 || height == 0) {
        if (counts_out && width > 0) std::memset(counts_out, 0, size_t(width) * 4);
        if (totals_out) *totals_out = ychg_totals{0, 0, with_hyperedges ? 0 : -1, 0};
        return YCHG_OK;
    }
    if (c.plan_w != width_img || c.plan_wc != width || c.plan_h != height) {
        ychg_plan_destroy(c.plan);
        c.plan = nullptr;
        c.plan_w = c.plan_wc = c.plan_h = -1;
        // one scan per call, synchronised: size the plan for latency, not pipelining
        // the image is written by the kernel just before the scan (re-pitch / PNM pack)
        if (const int rc = ychg_plan_create_ex(device, width_img, width, height,
                                               YCHG_PLAN_LATENCY | YCHG_PLAN_SYNC_INPUTS, &c.plan))
            return rc;
        c.plan_w = width_img;
        c.plan_wc = width;
        c.plan_h = height;
    }
    const int64_t pitch = (row_bytes + 15) / 16 * 16;
    if (const int rc = upload()) return rc;
    if (const int rc = ensure_columns(c, width_img)) return rc;
    static const bool host_timing = [] {
        const char* v = getenv("YCHG_HOST_TIMING");
        return v && v[0] == '1';
    }();
    cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
    if (host_timing) {
        for (auto& e : tev) cudaEventCreate(&e);
        cudaEventRecord(tev[0], c.stream);
    }
    // Outputs land in mapped pinned memory (see HostContext::m_block).
    // d_counts_dst: the counts go straight to another buffer -- possibly on a peer
    // GPU, so the finisher's stores are the gather (ychg_scan_host_sharded)
    if (c.m_block_cap < 64 + 8 * c.cols_cap) {
        cudaFreeHost(c.m_block);
        c.m_block = c.m_block_dev = nullptr;
        c.m_block_cap = 0;
        CK(cudaHostAlloc(&c.m_block, 64 + 8 * c.cols_cap, cudaHostAllocMapped | cudaHostAllocPortable));
        void* dp = nullptr;
        CK(cudaHostGetDevicePointer(&dp, c.m_block, 0));
        c.m_block_dev = static_cast<char*>(dp);
        c.m_block_cap = 64 + 8 * c.cols_cap;
    }
    int32_t* m_counts = reinterpret_cast<int32_t*>(c.m_block_dev + 64);
    if (const int rc = ychg_scan_device(c.plan, c.d_bits, pitch, with_hyperedges, d_counts_dst ? d_counts_dst : m_counts,
                                        c.d_flags, m_counts + c.cols_cap,
                                        reinterpret_cast<ychg_totals*>(c.m_block_dev), c.stream))
        return rc;
    if (host_timing) {
        cudaEventRecord(tev[1], c.stream);
        cudaEventRecord(tev[2], c.stream);  // no D2H step: the outputs are already in host memory
    }
    CK(cudaStreamSynchronize(c.stream));
    if (host_timing) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, tev[0], tev[1]);
        cudaEventElapsedTime(&b, tev[1], tev[2]);
        float h1 = 0, h2 = 0;
        cudaEventElapsedTime(&h1, c.h2d_ev[0], c.h2d_ev[1]);
        cudaEventElapsedTime(&h2, c.h2d_ev[0], c.h2d_ev[2]);
        std::fprintf(stderr, "[ychg host] h2d copies %.1f us, +repitch %.1f us, scan %.1f us, d2h %.1f us\n",
                     h1 * 1e3, h2 * 1e3, a * 1e3, b * 1e3);
        for (auto& e : tev) cudaEventDestroy(e);
    }
    ychg_totals t;
    std::memcpy(&t, c.m_block, sizeof(t));
    const int32_t* h_counts = reinterpret_cast<const int32_t*>(c.m_block + 64);
    if (counts_out) std::memcpy(counts_out, h_counts, size_t(width) * 4);
    if (boundaries_out && t.n_boundaries > 0)
        std::memcpy(boundaries_out, h_counts + c.cols_cap, size_t(t.n_boundaries) * 4);
    if (totals_out) *totals_out = t;
    return YCHG_OK;
}

extern "C" int ychg_scan_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                              int32_t with_hyperedges, int32_t* counts_out, int32_t* boundaries_out,
                              ychg_totals* totals_out) {
    if (width < 0 || height < 0) return fail(YCHG_ERR_INVALID, "scan: negative geometry %dx%d", width, height);
    const int64_t row_bytes = (int64_t(width) + 7) / 8;
    if (height > 0 && width > 0 && (!bits || row_stride < row_bytes))
        return fail(YCHG_ERR_INVALID, "scan: row_stride %lld < %lld", static_cast<long long>(row_stride),
                    static_cast<long long>(row_bytes));
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    return scan_host_locked(c, device, width, height, with_hyperedges, counts_out, boundaries_out, totals_out,
                            [&] { return upload_image(c, bits, width, height, row_stride); });
}

extern "C" int ychg_cut_vertex_counts(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                      int32_t strategy_kind, int32_t threads, int32_t* counts_out) {
    // runscan.cpp:24-26: a parallel strategy needs threads >= 1.  Every valid
    // strategy then runs the one GPU path (outputs are strategy-independent,
    // runscan.hpp:24-25).
    if (strategy_kind != YCHG_STRATEGY_SERIAL && strategy_kind != YCHG_STRATEGY_PARALLEL)
        return fail(YCHG_ERR_INVALID, "scan: unknown strategy kind %d", strategy_kind);
    if (strategy_kind == YCHG_STRATEGY_PARALLEL && threads < 1)
        return fail(YCHG_ERR_INVALID, "scan: parallel strategy needs threads >= 1, got %d", threads);
    if (width > 0 && !counts_out) return fail(YCHG_ERR_INVALID, "cut_vertex_counts: counts_out is NULL");
    return ychg_scan_host(bits, width, height, row_stride, 0, counts_out, nullptr, nullptr);
}

extern "C" int ychg_detect_boundary_columns(const int32_t* counts, int64_t n, int32_t* boundaries_out,
                                            int64_t* n_out) {
    if (n < 0) return fail(YCHG_ERR_INVALID, "detect_boundary_columns: negative length");
    if (n > 0 && (!counts || !boundaries_out)) return fail(YCHG_ERR_INVALID, "detect_boundary_columns: NULL buffer");
    if (n > INT32_MAX) return fail(YCHG_ERR_INVALID, "detect_boundary_columns: more than 2^31-1 columns");
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    if (n == 0) {
        if (n_out) *n_out = 0;
        return YCHG_OK;
    }
    if (const int rc = ensure_columns(c, n)) return rc;
    CK(cudaMemcpyAsync(c.d_counts, counts, n * 4, cudaMemcpyHostToDevice, c.stream));
    const int rc = ychg_launch_boundaries(c.d_counts, n, c.d_flags, c.d_bounds,
                                          reinterpret_cast<long long*>(&c.d_totals->n_boundaries), c.stream);
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "boundary kernels launch");
    CK(cudaMemcpyAsync(c.h_totals, c.d_totals, sizeof(ychg_totals), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    const int64_t nb = c.h_totals->n_boundaries;
    if (nb > 0) {
        CK(cudaMemcpyAsync(boundaries_out, c.d_bounds, nb * 4, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    }
    if (n_out) *n_out = nb;
    return YCHG_OK;
}

extern "C" int64_t ychg_boundary_flag_words(int64_t n) {
    // flags: one word per 32 columns, rounded to whole 1024-column blocks, + per-block counts
    return ((n + 1023) / 1024) * 32 + (n + 1023) / 1024 + 32;
}

extern "C" int ychg_detect_boundaries_device(const int32_t* d_counts, int64_t n, uint32_t* d_flags, int32_t* d_boundaries,
                                  int64_t* d_n, void* stream) {
    if (n < 0) return fail(YCHG_ERR_INVALID, "detect_boundary_columns: negative length");
    if (!d_n || (n > 0 && (!d_counts || !d_flags || !d_boundaries)))
        return fail(YCHG_ERR_INVALID, "detect_boundary_columns: NULL device buffer");
    if (n > INT32_MAX) return fail(YCHG_ERR_INVALID, "detect_boundary_columns: more than 2^31-1 columns");
    const int rc = ychg_launch_boundaries(d_counts, n, d_flags, d_boundaries, reinterpret_cast<long long*>(d_n),
                                          static_cast<cudaStream_t>(stream));
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "boundary kernels launch");
    return YCHG_OK;
}

extern "C" int ychg_assemble_strips_device(const int32_t* d_gathered, int32_t n_seg, int32_t seg_stride,
                                           int32_t totals_off, const int32_t* c0, int64_t width, int32_t* d_counts,
                                           uint32_t* d_flags, int32_t* d_boundaries, int64_t* d_n, int64_t* d_sums,
                                           void* stream) {
    if (n_seg < 1 || n_seg > 64) return fail(YCHG_ERR_INVALID, "assemble_strips: 1..64 segments, got %d", n_seg);
    if (!c0 || !d_gathered || !d_n || !d_sums || (width > 0 && (!d_counts || !d_flags || !d_boundaries)))
        return fail(YCHG_ERR_INVALID, "assemble_strips: NULL argument");
    if (c0[0] != 0 || c0[n_seg] != width || totals_off % 2 != 0)
        return fail(YCHG_ERR_INVALID, "assemble_strips: bad layout (c0[0]=%d, c0[n]=%d, width %lld, totals_off %d)",
                    c0[0], c0[n_seg], static_cast<long long>(width), totals_off);
    for (int r = 0; r < n_seg; ++r)
        if (c0[r + 1] < c0[r] || c0[r + 1] - c0[r] > totals_off || totals_off + 8 > seg_stride)
            return fail(YCHG_ERR_INVALID, "assemble_strips: segment %d does not fit its stride", r);
    const int rc = ychg_launch_assemble_strips(d_gathered, n_seg, seg_stride, totals_off, c0, width, d_counts,
                                               d_flags, d_boundaries, reinterpret_cast<long long*>(d_n),
                                               reinterpret_cast<long long*>(d_sums),
                                               static_cast<cudaStream_t>(stream));
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "assemble kernels launch");
    return YCHG_OK;
}

// ---------------------------------------------------------------------------- run materialisation
namespace {

// Profile phase 0 on the image already in c.d_bits (pitched for `width`): band
// counts, column totals, column offsets and the run total (read back).
int profile_count(HostContext& c, int32_t width, int32_t height, int64_t* n_runs) {
    if (const int rc = ensure_columns(c, width)) return rc;
    const int64_t pitch = ((int64_t(width) + 7) / 8 + 15) / 16 * 16;
    const int64_t bw = ychg_profile_band_words(width, height);
    if (bw > c.band_cap) {
        cudaFree(c.d_band);
        c.d_band = nullptr;
        c.band_cap = 0;
        CK(cudaMalloc(&c.d_band, bw * 4));
        c.band_cap = bw;
    }
    if (width > c.col_off_cap) {
        cudaFree(c.d_col_off);
        c.d_col_off = nullptr;
        c.col_off_cap = 0;
        CK(cudaMalloc(&c.d_col_off, int64_t(width) * 8));
        c.col_off_cap = width;
    }
    const int rc = ychg_launch_profile(c.d_bits, pitch, width, height, c.d_band, c.d_counts, c.d_col_off,
                                       &c.d_totals->total_runs, nullptr, 0, 0, c.stream);
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "profile count kernels launch");
    CK(cudaMemcpyAsync(c.h_totals, c.d_totals, sizeof(ychg_totals), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    *n_runs = c.h_totals->total_runs;
    return YCHG_OK;
}

// Uploads the image and runs profile phase 0 (counts, column offsets, run total).
int profile_phase0(HostContext& c, const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                   int64_t* n_runs) {
    if (const int rc = upload_image(c, bits, width, height, row_stride)) return rc;
    return profile_count(c, width, height, n_runs);
}

int profile_fill(HostContext& c, int32_t width, int32_t height, int64_t n_runs) {
    if (n_runs > c.runs_cap) {
        cudaFree(c.d_runs);
        c.d_runs = nullptr;
        c.runs_cap = 0;
        CK(cudaMalloc(&c.d_runs, std::max<int64_t>(n_runs, 1) * 12));
        c.runs_cap = n_runs;
    }
    const int64_t pitch = ((int64_t(width) + 7) / 8 + 15) / 16 * 16;
    const int rc = ychg_launch_profile(c.d_bits, pitch, width, height, c.d_band, c.d_counts, c.d_col_off, nullptr,
                                       c.d_runs, 1, n_runs, c.stream);
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "profile fill kernel launch");
    return YCHG_OK;
}

int check_profile_args(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride) {
    if (width < 0 || height < 0) return fail(YCHG_ERR_INVALID, "profile: negative geometry %dx%d", width, height);
    const int64_t row_bytes = (int64_t(width) + 7) / 8;
    if (height > 0 && width > 0 && (!bits || row_stride < row_bytes))
        return fail(YCHG_ERR_INVALID, "profile: row_stride %lld < %lld", static_cast<long long>(row_stride),
                    static_cast<long long>(row_bytes));
    return YCHG_OK;
}

}  // namespace

namespace {

// build_profile body: phase 0, then `dest(n)` names the host buffer for the n
// run triples (or nullptr: counts only); the image is uploaded and counted once.
template <typename Dest>
int build_profile_locked(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                         int32_t strategy_kind, int32_t threads, int32_t* counts_out, int64_t* n_runs_out,
                         Dest&& dest) {
    // Same strategy validation as the scan (runscan.cpp:24-26); build_profile is strategy-independent.
    if (strategy_kind != YCHG_STRATEGY_SERIAL && strategy_kind != YCHG_STRATEGY_PARALLEL)
        return fail(YCHG_ERR_INVALID, "scan: unknown strategy kind %d", strategy_kind);
    if (strategy_kind == YCHG_STRATEGY_PARALLEL && threads < 1)
        return fail(YCHG_ERR_INVALID, "scan: parallel strategy needs threads >= 1, got %d", threads);
    if (const int rc = check_profile_args(bits, width, height, row_stride)) return rc;
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    if (width == 0 || height == 0) {
        if (counts_out && width > 0) std::memset(counts_out, 0, size_t(width) * 4);
        if (n_runs_out) *n_runs_out = 0;
        return YCHG_OK;
    }
    int64_t n_runs = 0;
    if (const int rc = profile_phase0(c, bits, width, height, row_stride, &n_runs)) return rc;
    if (n_runs_out) *n_runs_out = n_runs;
    if (counts_out) CK(cudaMemcpyAsync(counts_out, c.d_counts, int64_t(width) * 4, cudaMemcpyDeviceToHost, c.stream));
    int32_t* runs_out = n_runs > 0 ? dest(n_runs) : nullptr;
    if (runs_out) {
        if (const int rc = profile_fill(c, width, height, n_runs)) return rc;
        CK(cudaMemcpyAsync(runs_out, c.d_runs, n_runs * 12, cudaMemcpyDeviceToHost, c.stream));
    }
    CK(cudaStreamSynchronize(c.stream));
    return YCHG_OK;
}

}  // namespace

extern "C" int ychg_build_profile_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                       int32_t strategy_kind, int32_t threads, int32_t* counts_out,
                                       int32_t* runs_out, int64_t runs_capacity, int64_t* n_runs_out) {
    return build_profile_locked(bits, width, height, row_stride, strategy_kind, threads, counts_out, n_runs_out,
                                [&](int64_t n) { return runs_capacity >= n ? runs_out : nullptr; });
}

extern "C" int ychg_build_profile_host_alloc(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                             int32_t strategy_kind, int32_t threads, int32_t* counts_out,
                                             ychg_alloc_fn alloc, void* alloc_ctx, int64_t* n_runs_out) {
    if (!alloc) return fail(YCHG_ERR_INVALID, "build_profile: NULL allocator");
    bool oom = false;
    const int rc = build_profile_locked(bits, width, height, row_stride, strategy_kind, threads, counts_out,
                                        n_runs_out, [&](int64_t n) {
                                            auto* p = static_cast<int32_t*>(alloc(alloc_ctx, n));
                                            oom = (p == nullptr);
                                            return p;
                                        });
    if (rc == YCHG_OK && oom) return fail(YCHG_ERR_OOM, "build_profile: allocator returned NULL");
    return rc;
}

// column_runs (runscan.cpp:104-120) moves O(height) bytes, not the image: only the
// byte column holding `col` is gathered (pinned staging, one byte per row at a
// 16-byte device pitch) and uploaded as an image of <= 8 columns, whose runs the
// profile kernels materialise; Run.col is rebased on the returned triples.
extern "C" int ychg_column_runs_host(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                     int32_t col, int32_t* runs_out, int64_t runs_capacity, int64_t* n_out) {
    // runscan.cpp:105-107
    if (col < 0 || col >= width)
        return fail(YCHG_ERR_INVALID, "column_runs: column %d out of range [0, %d)", col, width);
    if (const int rc = check_profile_args(bits, width, height, row_stride)) return rc;
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    if (n_out) *n_out = 0;
    if (height == 0) return YCHG_OK;
    const int32_t xb = col / 8, j = col - 8 * xb;
    const int32_t sub_w = std::min(8, width - 8 * xb);
    const int64_t need = 16 * int64_t(height);
    if (need > c.bits_cap) {
        cudaFree(c.d_bits);
        c.d_bits = nullptr;
        c.bits_cap = 0;
        CK(cudaMalloc(&c.d_bits, need));
        c.bits_cap = need;
    }
    if (need > c.col_stage_cap) {
        if (c.h_col_stage) cudaFreeHost(c.h_col_stage);
        c.h_col_stage = nullptr;
        c.col_stage_cap = 0;
        CK(cudaMallocHost(&c.h_col_stage, need));
        std::memset(c.h_col_stage, 0, size_t(need));
        c.col_stage_cap = need;
    }
    CK(cudaStreamSynchronize(c.stream));  // the staging buffer may still feed an earlier upload
    const uint8_t* src = bits + xb;
    for (int64_t y = 0; y < height; ++y) c.h_col_stage[16 * y] = src[y * row_stride];
    CK(cudaMemcpyAsync(c.d_bits, c.h_col_stage, need, cudaMemcpyHostToDevice, c.stream));
    int64_t n_runs = 0;
    if (const int rc = profile_count(c, sub_w, height, &n_runs)) return rc;
    int64_t off = 0;
    int32_t cnt = 0;
    CK(cudaMemcpyAsync(&off, c.d_col_off + j, 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&cnt, c.d_counts + j, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (n_out) *n_out = cnt;
    if (runs_out && runs_capacity >= cnt && cnt > 0) {
        if (const int rc = profile_fill(c, sub_w, height, n_runs)) return rc;
        CK(cudaMemcpyAsync(runs_out, c.d_runs + 3 * off, int64_t(cnt) * 12, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        for (int64_t i = 0; i < cnt; ++i) runs_out[3 * i] = col;  // sub-image column j -> image column col
    }
    return YCHG_OK;
}

// ---------------------------------------------------------------------------- hyperedge decomposition
struct ychg_hypergraph {
    int32_t width = 0, height = 0;
    int64_t n_runs = 0, n_edges = 0;
    float device_ms = 0.f;
    int device = 0;
    // device-resident results (stream-ordered allocations, freed by destroy)
    int32_t* d_eruns = nullptr;
    uint32_t* d_eoff = nullptr;
    uint32_t* d_r2e = nullptr;
};

namespace {

template <typename T>
int ensure_buf(T** p, int64_t* cap, int64_t elems) {
    if (elems <= *cap) return YCHG_OK;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<int64_t>(elems, 1) * int64_t(sizeof(T))));
    *cap = elems;
    return YCHG_OK;
}

int ensure_decompose(HostContext& c, int64_t n) {
    if (!c.h_dscal) {
        CK(cudaMallocHost(&c.h_dscal, 16));
        CK(cudaMalloc(&c.d_dscal, 16));
        CK(cudaEventCreate(&c.dec_ev[0]));
        CK(cudaEventCreate(&c.dec_ev[1]));
        // keep freed result buffers cached in the device's default pool
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, c.device));
        uint64_t keep = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    const int64_t ws = ychg_decompose_ws_bytes(n);
    if (ws > c.dws_cap) {
        cudaFree(c.d_dws);
        c.d_dws = nullptr;
        c.dws_cap = 0;
        CK(cudaMalloc(&c.d_dws, ws));
        c.dws_cap = ws;
    }
    return YCHG_OK;
}

// Decompose the n-run profile in c.d_runs / c.d_col_off / c.d_counts into hg's
// device buffers (kept on the device until ychg_hypergraph_copy).
int decompose_device_profile(HostContext& c, int32_t width, int64_t n, ychg_hypergraph* hg) {
    if (n > int64_t(0xFFFFFFFEu))
        return fail(YCHG_ERR_INVALID, "decompose: %lld runs exceed the 32-bit run index of Hypergraph",
                    static_cast<long long>(n));
    if (const int rc = ensure_decompose(c, n)) return rc;
    hg->device = c.device;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&hg->d_eruns), n * 12, c.stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&hg->d_eoff), (n + 1) * 4, c.stream));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&hg->d_r2e), n * 4, c.stream));
    CK(cudaEventRecord(c.dec_ev[0], c.stream));
    const int drc = ychg_launch_decompose(c.d_runs, c.d_col_off, c.d_counts, width, n, c.d_dws, hg->d_eruns,
                                          hg->d_eoff, hg->d_r2e, c.d_dscal, c.stream);
    if (drc < 0) return cuda_fail(static_cast<cudaError_t>(-drc), "decompose kernels");
    CK(cudaEventRecord(c.dec_ev[1], c.stream));
    CK(cudaMemcpyAsync(c.h_dscal, c.d_dscal, 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    CK(cudaEventElapsedTime(&hg->device_ms, c.dec_ev[0], c.dec_ev[1]));
    const unsigned long long tot = c.h_dscal[0];
    hg->n_runs = n;
    hg->n_edges = static_cast<int64_t>(tot >> 32);
    if (static_cast<int64_t>(tot & 0xFFFFFFFFull) != n)
        return fail(YCHG_ERR_INTERNAL, "decompose: chains cover %llu of %lld runs", tot & 0xFFFFFFFFull,
                    static_cast<long long>(n));
    return YCHG_OK;
}

void release_hypergraph(ychg_hypergraph* hg) {
    if (!hg) return;
    if (hg->d_eruns || hg->d_eoff || hg->d_r2e) {
        HostContext& c = host_context(hg->device);
        std::lock_guard<std::mutex> lock(c.mu);
        cudaSetDevice(hg->device);
        cudaFreeAsync(hg->d_eruns, c.stream);
        cudaFreeAsync(hg->d_eoff, c.stream);
        cudaFreeAsync(hg->d_r2e, c.stream);
    }
    delete hg;
}

using HgPtr = std::unique_ptr<ychg_hypergraph, void (*)(ychg_hypergraph*)>;

}  // namespace

extern "C" int ychg_decompose_image(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                    int32_t strategy_kind, int32_t threads, ychg_hypergraph** out) {
    if (!out) return fail(YCHG_ERR_INVALID, "decompose: null result pointer");
    *out = nullptr;
    if (strategy_kind != YCHG_STRATEGY_SERIAL && strategy_kind != YCHG_STRATEGY_PARALLEL)
        return fail(YCHG_ERR_INVALID, "scan: unknown strategy kind %d", strategy_kind);
    if (strategy_kind == YCHG_STRATEGY_PARALLEL && threads < 1)
        return fail(YCHG_ERR_INVALID, "scan: parallel strategy needs threads >= 1, got %d", threads);
    if (const int rc = check_profile_args(bits, width, height, row_stride)) return rc;
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HgPtr hg(new ychg_hypergraph, release_hypergraph);
    hg->width = width;
    hg->height = height;
    if (width > 0 && height > 0) {
        HostContext& c = host_context(device);
        std::lock_guard<std::mutex> lock(c.mu);
        if (const int rc = ensure_context(c)) return rc;
        int64_t n_runs = 0;
        if (const int rc = profile_phase0(c, bits, width, height, row_stride, &n_runs)) return rc;
        if (n_runs > 0) {
            if (const int rc = profile_fill(c, width, height, n_runs)) return rc;
            if (const int rc = decompose_device_profile(c, width, n_runs, hg.get())) return rc;
        }
    }
    *out = hg.release();
    return YCHG_OK;
}

extern "C" int ychg_decompose_profile(int32_t width, int32_t height, const int32_t* list_sizes, const int32_t* runs,
                                      int64_t n_runs, ychg_hypergraph** out) {
    if (!out) return fail(YCHG_ERR_INVALID, "decompose: null result pointer");
    *out = nullptr;
    // validate_profile (hypergraph.cpp:62-66)
    if (width < 0 || height < 0) return fail(YCHG_ERR_INVALID, "decompose: profile has negative geometry");
    int64_t total = 0;
    for (int32_t c = 0; c < width; ++c) {
        if (list_sizes[c] < 0) return fail(YCHG_ERR_INVALID, "decompose: negative run count in column %d", c);
        total += list_sizes[c];
    }
    if (total != n_runs)
        return fail(YCHG_ERR_INVALID, "decompose: list sizes sum to %lld, not %lld runs",
                    static_cast<long long>(total), static_cast<long long>(n_runs));
    if (n_runs > 0 && !runs) return fail(YCHG_ERR_INVALID, "decompose: null runs");
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HgPtr hg(new ychg_hypergraph, release_hypergraph);
    hg->width = width;
    hg->height = height;
    if (n_runs > 0) {
        HostContext& c = host_context(device);
        std::lock_guard<std::mutex> lock(c.mu);
        if (const int rc = ensure_context(c)) return rc;
        if (const int rc = ensure_columns(c, width)) return rc;
        if (const int rc = ensure_buf(&c.d_col_off, &c.col_off_cap, int64_t(width))) return rc;
        if (n_runs > c.runs_cap) {  // capacity counted in runs (12 B each), as in profile_fill
            cudaFree(c.d_runs);
            c.d_runs = nullptr;
            c.runs_cap = 0;
            CK(cudaMalloc(&c.d_runs, n_runs * 12));
            c.runs_cap = n_runs;
        }
        std::vector<int64_t> off(size_t(width) + 1, 0);
        for (int32_t k = 0; k < width; ++k) off[size_t(k) + 1] = off[size_t(k)] + list_sizes[k];
        CK(cudaMemcpyAsync(c.d_runs, runs, n_runs * 12, cudaMemcpyHostToDevice, c.stream));
        CK(cudaMemcpyAsync(c.d_counts, list_sizes, int64_t(width) * 4, cudaMemcpyHostToDevice, c.stream));
        CK(cudaMemcpyAsync(c.d_col_off, off.data(), int64_t(width) * 8, cudaMemcpyHostToDevice, c.stream));
        if (const int rc = ensure_decompose(c, n_runs)) return rc;
        const int rv = ychg_launch_decompose_validate(c.d_runs, c.d_col_off, width, height, n_runs, c.d_dscal + 1,
                                                      c.stream);
        if (rv != 0) return cuda_fail(static_cast<cudaError_t>(rv), "decompose validation");
        CK(cudaMemcpyAsync(c.h_dscal + 1, c.d_dscal + 1, 8, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        const unsigned long long err = c.h_dscal[1];
        if (err != ~0ull) {
            // the reference's messages (hypergraph.cpp:74-86)
            const int64_t g = static_cast<int64_t>(err >> 2);
            const int kind = static_cast<int>(err & 3ull);
            const int list = static_cast<int>(std::upper_bound(off.begin(), off.end(), g) - off.begin()) - 1;
            const int32_t* r = runs + 3 * g;
            if (kind == 1)
                return fail(YCHG_ERR_INVALID, "decompose: run in column list %d claims column %d", list, r[0]);
            if (kind == 2)
                return fail(YCHG_ERR_INVALID, "decompose: run [%d,%d] in column %d outside height %d", r[1], r[2],
                            list, height);
            return fail(YCHG_ERR_INVALID, "decompose: runs in column %d must be sorted and separated by background",
                        list);
        }
        if (const int rc = decompose_device_profile(c, width, n_runs, hg.get())) return rc;
    }
    *out = hg.release();
    return YCHG_OK;
}

extern "C" int ychg_hypergraph_info(const ychg_hypergraph* hg, int64_t* n_runs, int64_t* n_edges, float* device_ms) {
    if (!hg) return fail(YCHG_ERR_INVALID, "hypergraph: null handle");
    if (n_runs) *n_runs = hg->n_runs;
    if (n_edges) *n_edges = hg->n_edges;
    if (device_ms) *device_ms = hg->device_ms;
    return YCHG_OK;
}

extern "C" int ychg_hypergraph_copy(const ychg_hypergraph* hg, int32_t* edge_runs, uint32_t* edge_offsets,
                                    uint32_t* run_to_edge) {
    if (!hg) return fail(YCHG_ERR_INVALID, "hypergraph: null handle");
    if (hg->n_runs == 0) {
        if (edge_offsets) edge_offsets[0] = 0;
        return YCHG_OK;
    }
    HostContext& c = host_context(hg->device);
    std::lock_guard<std::mutex> lock(c.mu);
    CK(cudaSetDevice(hg->device));
    if (edge_runs) CK(cudaMemcpyAsync(edge_runs, hg->d_eruns, hg->n_runs * 12, cudaMemcpyDeviceToHost, c.stream));
    if (edge_offsets)
        CK(cudaMemcpyAsync(edge_offsets, hg->d_eoff, (hg->n_edges + 1) * 4, cudaMemcpyDeviceToHost, c.stream));
    if (run_to_edge) CK(cudaMemcpyAsync(run_to_edge, hg->d_r2e, hg->n_runs * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return YCHG_OK;
}

extern "C" void ychg_hypergraph_destroy(ychg_hypergraph* hg) { release_hypergraph(hg); }

// ---------------------------------------------------------------------------- PNM input (§8f row 3)
namespace {

// load_pnm's grammar (pnm.cpp:12-79): tokens separated by whitespace and '#'
// comments; binary rasters after exactly one whitespace byte.
struct PnmCursor {
    const uint8_t* p;
    int64_t n;
    int64_t pos;
    bool eof() const { return pos >= n; }
    static bool space(uint8_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }
    static bool digit(uint8_t c) { return c >= '0' && c <= '9'; }
    void skip() {
        while (!eof()) {
            if (p[pos] == '#') {
                while (!eof() && p[pos] != '\n') ++pos;
            } else if (space(p[pos])) {
                ++pos;
            } else {
                break;
            }
        }
    }
};

int parse_fail(int64_t at, const char* fmt, ...) {
    char buf[256];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_error = buf;
    g_error_offset = at;
    return YCHG_ERR_PARSE;
}

int pnm_uint(PnmCursor& r, const char* what, int32_t* out) {
    r.skip();
    if (r.eof() || !PnmCursor::digit(r.p[r.pos])) return parse_fail(r.pos, "pnm: expected %s", what);
    long long v = 0;
    while (!r.eof() && PnmCursor::digit(r.p[r.pos])) {
        v = v * 10 + (r.p[r.pos++] - '0');
        if (v > 2147483647LL) return parse_fail(r.pos, "pnm: %s out of range", what);
    }
    *out = static_cast<int32_t>(v);
    return YCHG_OK;
}

struct PnmHeader {
    char kind = 0;
    int32_t width = 0, height = 0;
    int64_t raster = 0;  // offset of the first raster byte (P4/P5) or of the ASCII samples (P1/P2)
};

// Header (+ the size check of a binary raster), in the reference's order.
int pnm_header(const uint8_t* bytes, int64_t n, PnmHeader* hd) {
    if (n > 0 && !bytes) return fail(YCHG_ERR_INVALID, "pnm: null bytes");
    PnmCursor r{bytes, n, 0};
    if (r.eof() || r.p[r.pos++] != 'P') return parse_fail(0, "pnm: missing magic number");
    if (r.eof()) return parse_fail(1, "pnm: missing magic number");
    const char kind = static_cast<char>(r.p[r.pos++]);
    if (kind == '3' || kind == '6' || kind == '7')
        return fail(YCHG_ERR_INVALID, "pnm: unsupported format P%c (only P1/P2/P4/P5)", kind);
    if (kind != '1' && kind != '2' && kind != '4' && kind != '5') return parse_fail(1, "pnm: malformed magic number");
    if (const int rc = pnm_uint(r, "width", &hd->width)) return rc;
    if (const int rc = pnm_uint(r, "height", &hd->height)) return rc;
    if (kind == '2' || kind == '5') {
        int32_t maxval = 0;
        if (const int rc = pnm_uint(r, "maxval", &maxval)) return rc;
        if (maxval != 255) return fail(YCHG_ERR_INVALID, "pnm: unsupported maxval %d (must be 255)", maxval);
    }
    if (kind == '4' || kind == '5') {
        if (r.eof() || !PnmCursor::space(r.p[r.pos]))
            return parse_fail(r.pos, "pnm: expected single whitespace before raster");
        ++r.pos;
        const int64_t left = n - r.pos;
        if (kind == '4') {
            const int64_t stride = (int64_t(hd->width) + 7) / 8;
            if (stride > 0 && left < stride * hd->height)
                return parse_fail(r.pos + (left / stride) * stride, "pnm: truncated P4 raster");
        } else if (left < int64_t(hd->width) * hd->height) {
            return parse_fail(r.pos, "pnm: truncated P5 raster");
        }
    }
    hd->kind = kind;
    hd->raster = r.pos;
    return YCHG_OK;
}

int check_threshold(int32_t threshold) {
    if (threshold < 0 || threshold > 255)
        return fail(YCHG_ERR_INVALID, "pnm: threshold must lie in [0, 255], got %d", threshold);
    return YCHG_OK;
}

// ASCII rasters on the host (pnm.cpp:81-101) into zeroed rows of `stride` bytes.
int pnm_ascii(const uint8_t* bytes, int64_t n, const PnmHeader& hd, int32_t threshold, uint8_t* bits, int64_t stride) {
    PnmCursor r{bytes, n, hd.raster};
    for (int32_t y = 0; y < hd.height; ++y) {
        std::memset(bits + y * stride, 0, size_t((int64_t(hd.width) + 7) / 8));
        for (int32_t x = 0; x < hd.width; ++x) {
            bool fg;
            if (hd.kind == '1') {
                r.skip();
                if (r.eof()) return parse_fail(r.pos, "pnm: truncated P1 raster");
                const uint8_t ch = r.p[r.pos++];
                if (ch != '0' && ch != '1') return parse_fail(r.pos - 1, "pnm: P1 raster sample must be 0 or 1");
                fg = ch == '1';
            } else {
                const int64_t at = r.pos;
                int32_t v = 0;
                if (const int rc = pnm_uint(r, "P2 raster sample", &v)) return rc;
                if (v > 255) return parse_fail(at, "pnm: P2 sample exceeds maxval");
                fg = v < threshold;
            }
            if (fg) bits[y * stride + (x >> 3)] |= static_cast<uint8_t>(0x80u >> (x & 7));
        }
    }
    return YCHG_OK;
}

template <typename T>
int ensure_dev(T** p, int64_t* cap, int64_t bytes) {
    if (bytes <= *cap) return YCHG_OK;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    CK(cudaMalloc(reinterpret_cast<void**>(p), std::max<int64_t>(bytes, 16)));
    *cap = bytes;
    return YCHG_OK;
}

}  // namespace

extern "C" int ychg_pnm_info(const uint8_t* bytes, int64_t n, int32_t* kind, int32_t* width, int32_t* height) {
    PnmHeader hd;
    if (const int rc = pnm_header(bytes, n, &hd)) return rc;
    if (kind) *kind = hd.kind - '0';
    if (width) *width = hd.width;
    if (height) *height = hd.height;
    return YCHG_OK;
}

extern "C" int ychg_load_pnm(const uint8_t* bytes, int64_t n, int32_t threshold, uint8_t* bits_out,
                             int64_t row_stride) {
    if (const int rc = check_threshold(threshold)) return rc;
    PnmHeader hd;
    if (const int rc = pnm_header(bytes, n, &hd)) return rc;
    const int64_t rb = (int64_t(hd.width) + 7) / 8;
    if (hd.height > 0 && rb > 0 && (!bits_out || row_stride < rb))
        return fail(YCHG_ERR_INVALID, "load_pnm: row_stride %lld < %lld", static_cast<long long>(row_stride),
                    static_cast<long long>(rb));
    if (hd.width == 0 || hd.height == 0) return YCHG_OK;
    if (hd.kind == '1' || hd.kind == '2') return pnm_ascii(bytes, n, hd, threshold, bits_out, row_stride);
    if (hd.kind == '4') {  // the payload IS the BinaryImage layout (pnm.cpp:103-114)
        const uint8_t mask = static_cast<uint8_t>(hd.width % 8 ? 0xFFu << (8 - hd.width % 8) : 0xFFu);
        for (int32_t y = 0; y < hd.height; ++y) {
            std::memcpy(bits_out + y * row_stride, bytes + hd.raster + y * rb, size_t(rb));
            bits_out[y * row_stride + rb - 1] &= mask;
        }
        return YCHG_OK;
    }
    // P5: threshold + pack on the device
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    const int64_t ns = int64_t(hd.width) * hd.height;
    if (const int rc = ensure_dev(&c.d_dense, &c.dense_cap, ns)) return rc;
    if (const int rc = ensure_dev(&c.d_bits, &c.bits_cap, rb * hd.height)) return rc;
    if (const int rc = h2d_any(c, c.d_dense, bytes + hd.raster, ns)) return rc;
    const int rc = ychg_launch_pack_p5(c.d_dense, hd.width, hd.height, threshold, c.d_bits, rb, c.stream);
    if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "P5 pack kernel");
    CK(cudaMemcpy2DAsync(bits_out, row_stride, c.d_bits, rb, rb, hd.height, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return YCHG_OK;
}

extern "C" int ychg_load_pnm_device(const uint8_t* bytes, int64_t n, int32_t threshold, uint8_t* d_bits,
                                    int64_t pitch, void* cuda_stream) {
    if (const int rc = check_threshold(threshold)) return rc;
    PnmHeader hd;
    if (const int rc = pnm_header(bytes, n, &hd)) return rc;
    const int64_t rb = (int64_t(hd.width) + 7) / 8;
    if (hd.width == 0 || hd.height == 0) return YCHG_OK;
    if (!d_bits || pitch < rb)
        return fail(YCHG_ERR_INVALID, "load_pnm_device: pitch %lld < %lld", static_cast<long long>(pitch),
                    static_cast<long long>(rb));
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (hd.kind == '4') {
        CK(cudaMemcpy2DAsync(d_bits, pitch, bytes + hd.raster, rb, rb, hd.height, cudaMemcpyHostToDevice, st));
        const int rc = ychg_launch_mask_pad(d_bits, pitch, hd.width, hd.height, st);
        return rc ? cuda_fail(static_cast<cudaError_t>(rc), "P4 pad mask kernel") : YCHG_OK;
    }
    if (hd.kind == '5') {
        const int64_t ns = int64_t(hd.width) * hd.height;
        uint8_t* d_s = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_s), ns, st));
        CK(cudaMemcpyAsync(d_s, bytes + hd.raster, ns, cudaMemcpyHostToDevice, st));
        const int rc = ychg_launch_pack_p5(d_s, hd.width, hd.height, threshold, d_bits, pitch, st);
        CK(cudaFreeAsync(d_s, st));
        return rc ? cuda_fail(static_cast<cudaError_t>(rc), "P5 pack kernel") : YCHG_OK;
    }
    std::vector<uint8_t> host(size_t(rb * hd.height));
    if (const int rc = pnm_ascii(bytes, n, hd, threshold, host.data(), rb)) return rc;
    CK(cudaMemcpy2DAsync(d_bits, pitch, host.data(), rb, rb, hd.height, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));  // `host` is released on return
    return YCHG_OK;
}

extern "C" int ychg_scan_pnm(const uint8_t* bytes, int64_t n, int32_t threshold, int32_t with_hyperedges,
                             int32_t* counts_out, int32_t* boundaries_out, ychg_totals* totals_out) {
    if (const int rc = check_threshold(threshold)) return rc;
    PnmHeader hd;
    if (const int rc = pnm_header(bytes, n, &hd)) return rc;
    const int64_t rb = (int64_t(hd.width) + 7) / 8;
    // P4: the raster goes to the device untouched -- the kernels never read padding bits
    if (hd.kind == '4')
        return ychg_scan_host(bytes + hd.raster, hd.width, hd.height, rb, with_hyperedges, counts_out,
                              boundaries_out, totals_out);
    if (hd.kind == '1' || hd.kind == '2') {
        std::vector<uint8_t> host(size_t(std::max<int64_t>(rb * hd.height, 1)));
        if (const int rc = pnm_ascii(bytes, n, hd, threshold, host.data(), rb)) return rc;
        return ychg_scan_host(host.data(), hd.width, hd.height, rb, with_hyperedges, counts_out, boundaries_out,
                              totals_out);
    }
    const int device = pick_device();
    if (const int rc = require_device(device)) return rc;
    HostContext& c = host_context(device);
    std::lock_guard<std::mutex> lock(c.mu);
    if (const int rc = ensure_context(c)) return rc;
    if (hd.width == 0 || hd.height == 0) {
        if (counts_out && hd.width > 0) std::memset(counts_out, 0, size_t(hd.width) * 4);
        if (totals_out) *totals_out = ychg_totals{0, 0, with_hyperedges ? 0 : -1, 0};
        return YCHG_OK;
    }
    return scan_host_locked(c, device, hd.width, hd.height, with_hyperedges, counts_out, boundaries_out, totals_out,
                            [&]() -> int {
                                const int64_t ns = int64_t(hd.width) * hd.height;
                                const int64_t pitch = (rb + 15) / 16 * 16;
                                if (const int rc = ensure_dev(&c.d_dense, &c.dense_cap, ns)) return rc;
                                if (const int rc = ensure_dev(&c.d_bits, &c.bits_cap, pitch * hd.height)) return rc;
                                if (const int rc = h2d_any(c, c.d_dense, bytes + hd.raster, ns)) return rc;
                                const int rc = ychg_launch_pack_p5(c.d_dense, hd.width, hd.height, threshold,
                                                                   c.d_bits, pitch, c.stream);
                                return rc ? cuda_fail(static_cast<cudaError_t>(rc), "P5 pack kernel") : YCHG_OK;
                            });
}

// ---------------------------------------------------------------------------- several devices, one process
// the mask cut into 1024-column-aligned strips (each with an
// 8-column right halo for the column pair at its right edge), strips spread
// round-robin over the given devices, one host thread per device; the strip
// counts are gathered, K2 runs once over them (ychg_detect_boundary_columns), and
// runs / links add up (a strip counts its own pairs, the halo one included).
namespace {
// Restores the calling thread's current device on scope exit: the sharded entry
// point switches devices (peer access, the gathering device) and must not leave
// a caller such as torch on another one.
struct DeviceRestore {
    int prev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    }
    ~DeviceRestore() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
}  // namespace

extern "C" int ychg_scan_host_sharded(const uint8_t* bits, int32_t width, int32_t height, int64_t row_stride,
                                      int32_t n_parts, const int32_t* devices, int32_t n_devices,
                                      int32_t with_hyperedges, int32_t* counts_out, int32_t* boundaries_out,
                                      ychg_totals* totals_out) {
    const DeviceRestore restore_device;
    if (width < 0 || height < 0) return fail(YCHG_ERR_INVALID, "scan_sharded: negative geometry %dx%d", width, height);
    if (n_parts < 1) return fail(YCHG_ERR_INVALID, "scan_sharded: n_parts must be >= 1, got %d", n_parts);
    const int64_t row_bytes = (int64_t(width) + 7) / 8;
    if (height > 0 && width > 0 && (!bits || row_stride < row_bytes))
        return fail(YCHG_ERR_INVALID, "scan_sharded: row_stride %lld < %lld", static_cast<long long>(row_stride),
                    static_cast<long long>(row_bytes));
    std::vector<int32_t> devs;
    if (devices && n_devices > 0) {
        devs.assign(devices, devices + n_devices);
    } else {
        devs.push_back(pick_device());
    }
    for (const int32_t d : devs)
        if (const int rc = require_device(d)) return rc;
    // strips on multiples of 1024 columns
    const int64_t units = (int64_t(width) + 1023) / 1024;
    struct Part {
        int32_t c0, c1, halo;
        ychg_totals t;
        int rc;
        std::string err;
    };
    std::vector<Part> parts;
    for (int32_t p = 0; p < n_parts; ++p) {
        const int64_t u0 = p * units / n_parts, u1 = (p + 1) * units / n_parts;
        const int32_t c0 = static_cast<int32_t>(std::min<int64_t>(width, u0 * 1024));
        const int32_t c1 = static_cast<int32_t>(std::min<int64_t>(width, u1 * 1024));
        if (c1 > c0) parts.push_back(Part{c0, c1, std::min<int32_t>(8, width - c1), {}, 0, {}});
    }
    std::vector<int32_t> counts(size_t(std::max(width, 1)), 0);
    // Peer gather: every strip's finisher stores its counts straight into one
    // array on the first device (over NVLink for the other devices), which then
    // runs K2 once -- no host round trip.  Without peer access between every
    // device and the first, the counts come back through the host instead.
    const int target = devs[0];
    bool peer = width > 0 && height > 0;
    for (const int32_t d : devs)
        if (peer && d != target) {
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, d, target) != cudaSuccess || !ok) peer = false;
        }
    int32_t* d_gather = nullptr;
    if (peer) {
        for (const int32_t d : devs)
            if (d != target) {
                CK(cudaSetDevice(d));
                const cudaError_t e = cudaDeviceEnablePeerAccess(target, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) {
                    cudaGetLastError();
                } else if (e != cudaSuccess) {
                    return cuda_fail(e, "scan_sharded: cudaDeviceEnablePeerAccess");
                }
            }
        CK(cudaSetDevice(target));
        CK(cudaMalloc(&d_gather, int64_t(width) * 4));
    }
    std::unique_ptr<int32_t, void (*)(int32_t*)> gather_guard(d_gather, [](int32_t* q) { cudaFree(q); });
    auto work = [&](size_t slot) {
        for (size_t i = slot; i < parts.size(); i += devs.size()) {
            Part& q = parts[i];
            const int device = devs[slot];
            HostContext& c = host_context(device);
            std::lock_guard<std::mutex> lock(c.mu);
            q.rc = ensure_context(c);
            if (q.rc == YCHG_OK) {
                const int32_t w_cnt = q.c1 - q.c0, w_img = w_cnt + q.halo;
                const uint8_t* src = bits + q.c0 / 8;
                q.rc = scan_host_locked(c, device, w_cnt, height, with_hyperedges, peer ? nullptr : counts.data() + q.c0,
                                        nullptr, &q.t, [&] { return upload_image(c, src, w_img, height, row_stride); },
                                        w_img, peer ? d_gather + q.c0 : nullptr);
            }
            if (q.rc != YCHG_OK) q.err = ychg_last_error();
        }
    };
    if (width > 0 && height > 0) {
        std::vector<std::thread> threads;
        for (size_t slot = 0; slot < devs.size() && slot < parts.size(); ++slot) threads.emplace_back(work, slot);
        for (auto& t : threads) t.join();
    }
    long long runs = 0, links = 0;
    for (const Part& q : parts) {
        if (q.rc != YCHG_OK) return fail(q.rc, "%s", q.err.c_str());
        runs += q.t.total_runs;
        links += q.t.links;
    }
    int64_t nb = 0;
    if (peer) {  // K2 once, on the device that holds the gathered counts
        HostContext& c = host_context(target);
        std::lock_guard<std::mutex> lock(c.mu);
        if (const int rc = ensure_context(c)) return rc;
        if (const int rc = ensure_columns(c, width)) return rc;
        const int rc = ychg_launch_boundaries(d_gather, width, c.d_flags, c.d_bounds,
                                              reinterpret_cast<long long*>(&c.d_totals->n_boundaries), c.stream);
        if (rc != 0) return cuda_fail(static_cast<cudaError_t>(rc), "boundary kernels launch");
        CK(cudaMemcpyAsync(c.h_totals, c.d_totals, sizeof(ychg_totals), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaMemcpyAsync(counts.data(), d_gather, int64_t(width) * 4, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        nb = c.h_totals->n_boundaries;
        if (boundaries_out && nb > 0) {
            CK(cudaMemcpyAsync(boundaries_out, c.d_bounds, nb * 4, cudaMemcpyDeviceToHost, c.stream));
            CK(cudaStreamSynchronize(c.stream));
        }
    } else if (width > 0) {
        std::vector<int32_t> bounds(static_cast<size_t>(width));
        if (const int rc = ychg_detect_boundary_columns(counts.data(), width, bounds.data(), &nb)) return rc;
        if (boundaries_out && nb > 0) std::memcpy(boundaries_out, bounds.data(), size_t(nb) * 4);
    }
    if (counts_out && width > 0) std::memcpy(counts_out, counts.data(), size_t(width) * 4);
    if (totals_out) *totals_out = ychg_totals{runs, with_hyperedges ? links : 0, with_hyperedges ? runs - links : -1, nb};
    return YCHG_OK;
}
