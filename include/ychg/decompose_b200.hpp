// decompose_b200.hpp -- the device hyperedge decomposition as the reference's own
// type: ychg::b200::decompose returns a ychg::Hypergraph (reference
// hypergraph.hpp:27-71) equal (operator==) to ychg::decompose's
// (hypergraph.cpp:94-170).  Header-only on purpose: it needs the reference's
// "ychg/hypergraph.hpp" on the include path and the reference's hypergraph.cpp
// linked (the Hypergraph constructor lives there); the arithmetic runs in
// libychg_b200.so (ychg_decompose_profile / ychg_decompose_image, C ABI).
#ifndef YCHG_DECOMPOSE_B200_HPP
#define YCHG_DECOMPOSE_B200_HPP

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ychg/errors.hpp"
#include "ychg/hypergraph.hpp"
#include "ychg/image.hpp"
#include "ychg/runscan.hpp"
#include "ychg_b200.h"

namespace ychg::b200 {

namespace detail {

// The C ABI's decompose messages already carry the reference's wording
// ("decompose: ..."); other failures are prefixed with the operation.
inline void check(int rc, const char* what) {
    if (rc == YCHG_OK) return;
    std::string msg = ychg_last_error();
    if (msg.rfind("decompose:", 0) != 0) msg = std::string(what) + ": " + msg;
    if (rc == YCHG_ERR_INVALID) throw ValidationError(msg);
    throw Error(msg);
}

inline Hypergraph take(ychg_hypergraph* h, int width, int height) {
    std::unique_ptr<ychg_hypergraph, void (*)(ychg_hypergraph*)> guard(h, ychg_hypergraph_destroy);
    std::int64_t n = 0, e = 0;
    check(ychg_hypergraph_info(h, &n, &e, nullptr), "decompose");
    static_assert(sizeof(Run) == 3 * sizeof(std::int32_t), "Run must be three ints (C ABI run triples)");
    std::vector<Run> runs(static_cast<std::size_t>(n));
    std::vector<std::uint32_t> offsets(static_cast<std::size_t>(e) + 1);
    check(ychg_hypergraph_copy(h, reinterpret_cast<std::int32_t*>(runs.data()), offsets.data(), nullptr),
          "decompose");
    return Hypergraph(width, height, std::move(runs), std::move(offsets));
}

}  // namespace detail

/// decompose (hypergraph.cpp:94-170) of a profile, validated like validate_profile (:62-90).
inline Hypergraph decompose(const ColumnProfile& profile) {
    if (profile.width < 0 || profile.height < 0)
        throw ValidationError("decompose: profile has negative geometry");
    const std::size_t width = static_cast<std::size_t>(profile.width);
    if (profile.runs.size() != width || profile.counts.size() != width)
        throw ValidationError("decompose: profile arrays do not match width " + std::to_string(profile.width));
    // claimed counts vs list sizes: the reference reports the first offending
    // column, after any bad run of an earlier column -- validate that prefix on
    // the device by passing only the columns before it.
    std::size_t first_bad = width;
    for (std::size_t c = 0; c < width; ++c)
        if (profile.counts[c] != static_cast<int>(profile.runs[c].size())) {
            first_bad = c;
            break;
        }
    std::vector<std::int32_t> sizes(width, 0);
    std::vector<Run> flat;
    for (std::size_t c = 0; c < first_bad; ++c) {
        sizes[c] = static_cast<std::int32_t>(profile.runs[c].size());
        flat.insert(flat.end(), profile.runs[c].begin(), profile.runs[c].end());
    }
    ychg_hypergraph* h = nullptr;
    detail::check(ychg_decompose_profile(profile.width, profile.height, sizes.data(),
                                         reinterpret_cast<const std::int32_t*>(flat.data()),
                                         static_cast<std::int64_t>(flat.size()), &h),
                  "decompose");
    if (first_bad < width) {
        ychg_hypergraph_destroy(h);
        throw ValidationError("decompose: counts[" + std::to_string(first_bad) +
                              "] does not equal the number of runs");
    }
    return detail::take(h, profile.width, profile.height);
}

/// decompose(build_profile(image)) without the profile leaving the device.
inline Hypergraph decompose(const BinaryImage& image) {
    ychg_hypergraph* h = nullptr;
    detail::check(ychg_decompose_image(image.bytes().data(), image.width(), image.height(), image.row_stride(),
                                       YCHG_STRATEGY_SERIAL, 1, &h),
                  "decompose");
    return detail::take(h, image.width(), image.height());
}

}  // namespace ychg::b200

#endif
