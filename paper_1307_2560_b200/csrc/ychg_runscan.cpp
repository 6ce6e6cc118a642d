// ychg_runscan.cpp -- the C++ drop-in: ychg::cut_vertex_counts and
// ychg::detect_boundary_columns (reference runscan.hpp:59-71) implemented over
// the C ABI of libychg_b200.so.  Status codes become the reference's exception
// types (errors.hpp:11-40); there is no CPU fallback.
#include <algorithm>
#include <string>
#include <vector>

#include "ychg/errors.hpp"
#include "ychg/image.hpp"
#include "ychg/pnm.hpp"
#include "ychg/runscan.hpp"
#include "ychg/scan_b200.hpp"
#include "ychg_b200.h"

namespace ychg {

namespace {

// Validation messages of the C ABI are worded like the reference's own
// (runscan.cpp:25-26,105-107: "scan: parallel strategy needs threads >= 1, got 0",
// "column_runs: column 4 out of range [0, 4)") and pass through unprefixed, so
// what() matches the reference; device/runtime failures get the entry point.
void check(int rc, const char* what) {
    if (rc == YCHG_OK) return;
    if (rc == YCHG_ERR_PARSE)
        throw ParseError(ychg_last_error(), static_cast<std::size_t>(ychg_last_error_offset()));
    if (rc == YCHG_ERR_INVALID) throw ValidationError(ychg_last_error());
    throw Error(std::string(what) + ": " + ychg_last_error());
}

// The PNM loader's messages are the reference's own (pnm.cpp), unprefixed.
void check_pnm(int rc) {
    if (rc == YCHG_OK) return;
    if (rc == YCHG_ERR_PARSE)
        throw ParseError(ychg_last_error(), static_cast<std::size_t>(ychg_last_error_offset()));
    if (rc == YCHG_ERR_INVALID) throw ValidationError(ychg_last_error());
    throw Error(std::string("load_pnm: ") + ychg_last_error());
}

}  // namespace

BinaryImage load_pnm(std::span<const std::uint8_t> bytes, int threshold) {
    if (threshold < 0 || threshold > 255)
        throw ValidationError("pnm: threshold must lie in [0, 255], got " + std::to_string(threshold));
    std::int32_t kind = 0, w = 0, h = 0;
    check_pnm(ychg_pnm_info(bytes.data(), static_cast<std::int64_t>(bytes.size()), &kind, &w, &h));
    BinaryImage img(w, h);
    if (w > 0 && h > 0)
        check_pnm(ychg_load_pnm(bytes.data(), static_cast<std::int64_t>(bytes.size()), threshold, img.row(0),
                                img.row_stride()));
    return img;
}

std::vector<std::uint8_t> save_pnm(const BinaryImage& image) {
    const std::string head = "P4\n" + std::to_string(image.width()) + " " + std::to_string(image.height()) + "\n";
    std::vector<std::uint8_t> out(head.begin(), head.end());
    out.insert(out.end(), image.bytes().begin(), image.bytes().end());
    return out;
}

ScanResult scan_pnm(std::span<const std::uint8_t> bytes, int threshold) {
    std::int32_t kind = 0, w = 0, h = 0;
    check_pnm(ychg_pnm_info(bytes.data(), static_cast<std::int64_t>(bytes.size()), &kind, &w, &h));
    ScanResult r;
    r.counts.assign(static_cast<std::size_t>(w), 0);
    r.boundaries.assign(static_cast<std::size_t>(w), 0);
    ychg_totals t{};
    check_pnm(ychg_scan_pnm(bytes.data(), static_cast<std::int64_t>(bytes.size()), threshold, 1, r.counts.data(),
                            r.boundaries.data(), &t));
    r.boundaries.resize(static_cast<std::size_t>(t.n_boundaries));
    r.total_runs = t.total_runs;
    r.links = t.links;
    r.hyperedges = t.hyperedges;
    return r;
}

ScanResult scan_sharded(const BinaryImage& image, int n_parts, std::span<const int> devices) {
    ScanResult r;
    r.counts.assign(static_cast<std::size_t>(image.width()), 0);
    r.boundaries.assign(static_cast<std::size_t>(image.width()), 0);
    ychg_totals t{};
    check(ychg_scan_host_sharded(image.bytes().data(), image.width(), image.height(), image.row_stride(), n_parts,
                                 devices.empty() ? nullptr : devices.data(), static_cast<std::int32_t>(devices.size()),
                                 1, r.counts.data(), r.boundaries.data(), &t),
          "scan_sharded");
    r.boundaries.resize(static_cast<std::size_t>(t.n_boundaries));
    r.total_runs = t.total_runs;
    r.links = t.links;
    r.hyperedges = t.hyperedges;
    return r;
}

std::int64_t foreground_count(const BinaryImage& image) {
    std::int64_t n = 0;
    for (std::uint8_t b : image.bytes()) n += __builtin_popcount(b);
    return n;
}

std::vector<int> cut_vertex_counts(const BinaryImage& image, ScanStrategy strategy) {
    std::vector<int> counts(static_cast<std::size_t>(image.width()), 0);
    const int kind = strategy.kind == ScanStrategy::Kind::serial ? YCHG_STRATEGY_SERIAL
                                                                  : YCHG_STRATEGY_PARALLEL;
    check(ychg_cut_vertex_counts(image.bytes().data(), image.width(), image.height(),
                                 image.row_stride(), kind, strategy.threads, counts.data()),
          "cut_vertex_counts");
    return counts;
}

std::vector<Run> column_runs(const BinaryImage& image, int col) {
    // a column holds at most ceil(height/2) runs; one call fills up to that many
    std::vector<Run> runs(static_cast<std::size_t>(std::min(image.height() / 2 + 1, 1 << 16)));
    std::int64_t n = 0;
    check(ychg_column_runs_host(image.bytes().data(), image.width(), image.height(), image.row_stride(), col,
                                reinterpret_cast<std::int32_t*>(runs.data()), static_cast<std::int64_t>(runs.size()),
                                &n),
          "column_runs");
    if (n > static_cast<std::int64_t>(runs.size())) {  // very tall column: second call at the exact size
        runs.resize(static_cast<std::size_t>(n));
        check(ychg_column_runs_host(image.bytes().data(), image.width(), image.height(), image.row_stride(), col,
                                    reinterpret_cast<std::int32_t*>(runs.data()), n, &n),
              "column_runs");
    }
    runs.resize(static_cast<std::size_t>(n));
    return runs;
}

ColumnProfile build_profile(const BinaryImage& image, ScanStrategy strategy) {
    static_assert(sizeof(Run) == 3 * sizeof(std::int32_t), "Run must be three ints (C ABI run triples)");
    const int kind = strategy.kind == ScanStrategy::Kind::serial ? YCHG_STRATEGY_SERIAL : YCHG_STRATEGY_PARALLEL;
    ColumnProfile p;
    p.width = image.width();
    p.height = image.height();
    p.counts.assign(static_cast<std::size_t>(image.width()), 0);
    std::vector<Run> flat;
    std::int64_t n = 0;
    // one call: the library asks for the run buffer once it knows the total
    auto alloc = [](void* ctx, std::int64_t n_runs) -> void* {
        auto* v = static_cast<std::vector<Run>*>(ctx);
        v->resize(static_cast<std::size_t>(n_runs));
        return v->data();
    };
    check(ychg_build_profile_host_alloc(image.bytes().data(), image.width(), image.height(), image.row_stride(),
                                        kind, strategy.threads, p.counts.data(), alloc, &flat, &n),
          "build_profile");
    p.runs.resize(static_cast<std::size_t>(image.width()));
    std::size_t at = 0;
    for (int c = 0; c < image.width(); ++c) {
        const auto k = static_cast<std::size_t>(p.counts[static_cast<std::size_t>(c)]);
        p.runs[static_cast<std::size_t>(c)].assign(flat.begin() + static_cast<std::ptrdiff_t>(at),
                                                   flat.begin() + static_cast<std::ptrdiff_t>(at + k));
        at += k;
    }
    return p;
}

std::vector<int> detect_boundary_columns(std::span<const int> counts) {
    std::vector<int> out(counts.size());
    std::int64_t n = 0;
    check(ychg_detect_boundary_columns(counts.data(), static_cast<std::int64_t>(counts.size()),
                                       out.data(), &n),
          "detect_boundary_columns");
    out.resize(static_cast<std::size_t>(n));
    return out;
}

ScanResult scan(const BinaryImage& image) {
    ScanResult r;
    r.counts.assign(static_cast<std::size_t>(image.width()), 0);
    r.boundaries.assign(static_cast<std::size_t>(image.width()), 0);
    ychg_totals t{};
    check(ychg_scan_host(image.bytes().data(), image.width(), image.height(), image.row_stride(), 1,
                         r.counts.data(), r.boundaries.data(), &t),
          "scan");
    r.boundaries.resize(static_cast<std::size_t>(t.n_boundaries));
    r.total_runs = t.total_runs;
    r.links = t.links;
    r.hyperedges = t.hyperedges;
    return r;
}

}  // namespace ychg
