// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference implementation, which
// oracle/Makefile compiles from /root/reference/proj/src with -Dychg=ychg_ref
// into oracle/_ref/libychg_ref.so.  Used by tests (to pin the oracle and generate
// golden fixtures) and by bench.py's reference arm / cpu_baseline leg (to time
// the reference's own CPU path on the GPU box's host cores).  Never linked by
// the product.
//
// This file is ours; it only calls the reference's public API:
//   synth (synth.hpp:66), cut_vertex_counts (runscan.hpp:59-62),
//   detect_boundary_columns (runscan.hpp:68-71), build_profile (runscan.hpp:64-66),
//   decompose + hyperedge_count (hypergraph.hpp:82,96).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ychg/errors.hpp"
#include "ychg/hypergraph.hpp"
#include "ychg/image.hpp"
#include "ychg/pnm.hpp"
#include "ychg/runscan.hpp"
#include "ychg/synth.hpp"

#define YR_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

ychg::ScanStrategy strategy_of(int kind, int threads) {
    return kind == 0 ? ychg::ScanStrategy::serial() : ychg::ScanStrategy::parallel(threads);
}

// -1 = ValidationError, -2 = other ychg::Error, -3 = anything else.
int code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ychg::ValidationError*>(&e)) return -1;
    if (dynamic_cast<const ychg::Error*>(&e)) return -2;
    return -3;
}

ychg::BinaryImage image_of(const uint8_t* bits, int w, int h, int64_t stride) {
    ychg::BinaryImage img(w, h);
    const int s = img.row_stride();
    for (int y = 0; y < h; ++y) std::memcpy(img.row(y), bits + y * stride, static_cast<size_t>(s));
    return img;
}

}  // namespace

YR_EXPORT const char* yr_last_error() { return g_err.c_str(); }

YR_EXPORT int yr_synth(int pattern, int w, int h, int bands, int cell, double density,
                       uint64_t seed, uint8_t* out) {
    try {
        ychg::SynthSpec spec{static_cast<ychg::Pattern>(pattern), w, h, bands, cell, density, seed};
        const ychg::BinaryImage img = ychg::synth(spec);
        std::memcpy(out, img.bytes().data(), img.bytes().size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

YR_EXPORT uint64_t yr_splitmix64(uint64_t seed, int n_skip) {
    ychg::Splitmix64 rng(seed);
    uint64_t v = 0;
    for (int i = 0; i <= n_skip; ++i) v = rng.next();
    return v;
}

// Opaque handle so benchmarks time only the reference call, not the copy-in.
YR_EXPORT void* yr_image_create(const uint8_t* bits, int w, int h, int64_t stride) {
    try {
        return new ychg::BinaryImage(image_of(bits, w, h, stride));
    } catch (const std::exception& e) {
        code_of(e);
        return nullptr;
    }
}

YR_EXPORT void* yr_image_synth(int pattern, int w, int h, int bands, int cell, double density,
                               uint64_t seed) {
    try {
        ychg::SynthSpec spec{static_cast<ychg::Pattern>(pattern), w, h, bands, cell, density, seed};
        return new ychg::BinaryImage(ychg::synth(spec));
    } catch (const std::exception& e) {
        code_of(e);
        return nullptr;
    }
}

YR_EXPORT void yr_image_destroy(void* img) { delete static_cast<ychg::BinaryImage*>(img); }

YR_EXPORT const uint8_t* yr_image_bytes(void* img) {
    return static_cast<ychg::BinaryImage*>(img)->bytes().data();
}

YR_EXPORT int yr_counts(void* img, int kind, int threads, int32_t* out) {
    try {
        const auto counts = ychg::cut_vertex_counts(*static_cast<ychg::BinaryImage*>(img),
                                                    strategy_of(kind, threads));
        if (!counts.empty()) std::memcpy(out, counts.data(), counts.size() * sizeof(int));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// column_runs(image, col) (runscan.cpp:104-120): returns the run count (triples
// {col, y_top, y_bot} into runs when capacity allows), -1 on a reference exception.
YR_EXPORT int64_t yr_column_runs(void* img, int col, int32_t* runs, int64_t capacity) {
    try {
        const auto r = ychg::column_runs(*static_cast<ychg::BinaryImage*>(img), col);
        if (runs && capacity >= static_cast<int64_t>(r.size()))
            for (std::size_t i = 0; i < r.size(); ++i) {
                runs[3 * i] = r[i].col;
                runs[3 * i + 1] = r[i].y_top;
                runs[3 * i + 2] = r[i].y_bot;
            }
        return static_cast<int64_t>(r.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

YR_EXPORT int64_t yr_boundaries(const int32_t* counts, int64_t n, int32_t* out) {
    const auto b = ychg::detect_boundary_columns(std::span<const int>(counts, static_cast<size_t>(n)));
    if (out && !b.empty()) std::memcpy(out, b.data(), b.size() * sizeof(int));
    return static_cast<int64_t>(b.size());
}

YR_EXPORT int64_t yr_hyperedges(void* img, int kind, int threads) {
    try {
        const auto prof = ychg::build_profile(*static_cast<ychg::BinaryImage*>(img),
                                              strategy_of(kind, threads));
        return static_cast<int64_t>(ychg::hyperedge_count(ychg::decompose(prof)));
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// build_profile (runscan.hpp:64-66) flattened column-major into int32 triples.
YR_EXPORT int64_t yr_profile(void* img, int kind, int threads, int32_t* runs, int64_t capacity) {
    try {
        const auto prof = ychg::build_profile(*static_cast<ychg::BinaryImage*>(img), strategy_of(kind, threads));
        int64_t n = 0;
        for (const auto& col : prof.runs)
            for (const auto& r : col) {
                if (runs && n < capacity) {
                    runs[3 * n] = r.col;
                    runs[3 * n + 1] = r.y_top;
                    runs[3 * n + 2] = r.y_bot;
                }
                ++n;
            }
        return n;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// load_pnm (pnm.cpp:124-153).  Returns 0 and fills w/h (+ bits when cap
// suffices), or -1 ValidationError / -4 ParseError (*offset set) / -2 / -3.
YR_EXPORT int yr_load_pnm(const uint8_t* bytes, int64_t n, int threshold, uint8_t* bits, int64_t cap,
                          int32_t* w, int32_t* h, int64_t* offset) {
    try {
        const auto img = ychg::load_pnm(std::span<const uint8_t>(bytes, static_cast<size_t>(n)), threshold);
        *w = img.width();
        *h = img.height();
        if (bits && cap >= static_cast<int64_t>(img.bytes().size()))
            std::memcpy(bits, img.bytes().data(), img.bytes().size());
        return 0;
    } catch (const ychg::ParseError& e) {
        g_err = e.what();
        *offset = static_cast<int64_t>(e.offset());
        return -4;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// decompose(build_profile(img)) (hypergraph.cpp:94-170) exported as flat arrays:
// edge_runs = all_runs() triples, edge_offsets[0..E], run_to_edge() (profile
// order).  Returns E (or a negative error code); *n_runs_out gets the run total.
// Outputs are written only if the capacities suffice.
YR_EXPORT int64_t yr_decompose(void* img, int32_t* edge_runs, int64_t runs_cap, uint32_t* edge_offsets,
                               int64_t edges_cap, uint32_t* run_to_edge, int64_t* n_runs_out) {
    try {
        const auto hg = ychg::decompose(ychg::build_profile(*static_cast<ychg::BinaryImage*>(img),
                                                            ychg::ScanStrategy::serial()));
        const auto all = hg.all_runs();
        const int64_t n = static_cast<int64_t>(all.size());
        const int64_t e = static_cast<int64_t>(hg.edge_count());
        if (n_runs_out) *n_runs_out = n;
        if (edge_runs && runs_cap >= n)
            for (int64_t i = 0; i < n; ++i) {
                edge_runs[3 * i] = all[i].col;
                edge_runs[3 * i + 1] = all[i].y_top;
                edge_runs[3 * i + 2] = all[i].y_bot;
            }
        if (edge_offsets && edges_cap >= e + 1) {
            edge_offsets[0] = 0;
            for (int64_t i = 0; i < e; ++i)
                edge_offsets[i + 1] = edge_offsets[i] + static_cast<uint32_t>(hg.edge(i).runs.size());
        }
        if (run_to_edge && runs_cap >= n) {
            const auto r2e = hg.run_to_edge();
            std::memcpy(run_to_edge, r2e.data(), r2e.size() * 4);
        }
        return e;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The reference's full hot path (counts + boundaries + hyperedge total), timed
// with the reference protocol (bench.cpp:37-57: warmup untimed, reps timed with
// steady_clock).  with_hyperedges=0 times counts + boundaries only.
// ns_out gets one entry per rep; the outputs of the last rep go to the out args.
YR_EXPORT int yr_time_path(void* img, int kind, int threads, int warmup, int reps,
                           int with_hyperedges, int64_t* ns_out, int32_t* counts_out,
                           int64_t* n_boundaries_out, int64_t* hyperedges_out) {
    try {
        const auto& image = *static_cast<ychg::BinaryImage*>(img);
        const auto strategy = strategy_of(kind, threads);
        for (int r = 0; r < warmup + reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const auto counts = ychg::cut_vertex_counts(image, strategy);
            const auto bounds = ychg::detect_boundary_columns(counts);
            std::int64_t he = -1;
            if (with_hyperedges)
                he = static_cast<int64_t>(
                    ychg::hyperedge_count(ychg::decompose(ychg::build_profile(image, strategy))));
            const auto t1 = std::chrono::steady_clock::now();
            if (r >= warmup) {
                ns_out[r - warmup] =
                    std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
                if (r == warmup + reps - 1) {
                    if (counts_out && !counts.empty())
                        std::memcpy(counts_out, counts.data(), counts.size() * sizeof(int));
                    if (n_boundaries_out) *n_boundaries_out = static_cast<int64_t>(bounds.size());
                    if (hyperedges_out) *hyperedges_out = he;
                }
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}
