// ychg/scan_b200.hpp -- extensions of the B200 library beyond the reference API.
//
// scan() returns every output of the hot path from one pass over the mask:
// counts (runscan.cpp:122-128), boundaries (runscan.cpp:145-153) and the
// hyperedge total that the reference only obtains as
// hyperedge_count(decompose(build_profile(image))) (hypergraph.cpp:192).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "ychg/image.hpp"

namespace ychg {

struct ScanResult {
    std::vector<int> counts;
    std::vector<int> boundaries;
    std::int64_t total_runs = 0;
    std::int64_t links = 0;
    std::int64_t hyperedges = 0;
};

ScanResult scan(const BinaryImage& image);

/// scan() of a PNM file's bytes (pnm.cpp formats): the P4 raster goes to the
/// device untouched, P5 is thresholded and packed on the device.
ScanResult scan_pnm(std::span<const std::uint8_t> bytes, int threshold = 128);

/// scan() over several GPUs of this process: n_parts column strips
/// (multiples of 1024 columns, 8-column right halos) round-robin over `devices`
/// (empty = the current device), one host thread per device; same results as scan().
ScanResult scan_sharded(const BinaryImage& image, int n_parts, std::span<const int> devices = {});

}  // namespace ychg
