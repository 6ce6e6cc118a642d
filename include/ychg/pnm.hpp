// ychg/pnm.hpp -- PNM input/output with the reference's signatures
// (proj/include/ychg/pnm.hpp:12-25), implemented by libychg.so over the C ABI
// (ychg_load_pnm: P4 rasters as they are, P5 thresholded and packed on the
// device, ASCII P1/P2 parsed on the host; same exceptions, messages, offsets).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "ychg/image.hpp"

namespace ychg {

BinaryImage load_pnm(std::span<const std::uint8_t> bytes, int threshold = 128);

std::vector<std::uint8_t> save_pnm(const BinaryImage& image);

}  // namespace ychg
