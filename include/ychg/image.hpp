// ychg/image.hpp -- the packed binary raster consumed by the yCHG scan.
//
// ABI-compatible with the reference BinaryImage (proj/include/ychg/image.hpp:17-72):
// the same three ints followed by the byte vector, the same packing (row-major,
// MSB-first bytes, rows padded to (width+7)/8 bytes, padding bits zero), so a
// caller compiled against the reference header can hand its images to this
// library unchanged.  Declarations are re-stated here, not copied.
#pragma once

#include <cassert>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace ychg {

class BinaryImage {
public:
    BinaryImage() = default;
    BinaryImage(int width, int height)
        : width_(width), height_(height), stride_((width + 7) / 8),
          bits_(static_cast<std::size_t>(stride_) * static_cast<std::size_t>(height), 0) {
        assert(width >= 0 && height >= 0);
    }

    int width() const { return width_; }
    int height() const { return height_; }
    int row_stride() const { return stride_; }

    const std::uint8_t* row(int y) const { return bits_.data() + offset(y); }
    std::uint8_t* row(int y) { return bits_.data() + offset(y); }
    const std::vector<std::uint8_t>& bytes() const { return bits_; }

    bool get(int x, int y) const { return (row(y)[x >> 3] & bit(x)) != 0; }
    void set(int x, int y, bool on) {
        std::uint8_t& b = row(y)[x >> 3];
        b = on ? static_cast<std::uint8_t>(b | bit(x)) : static_cast<std::uint8_t>(b & ~bit(x));
    }

    bool operator==(const BinaryImage&) const = default;

private:
    static std::uint8_t bit(int x) { return static_cast<std::uint8_t>(0x80u >> (x & 7)); }
    std::size_t offset(int y) const {
        assert(y >= 0 && y < height_);
        return static_cast<std::size_t>(y) * static_cast<std::size_t>(stride_);
    }

    int width_ = 0;
    int height_ = 0;
    int stride_ = 0;
    std::vector<std::uint8_t> bits_;
};

std::int64_t foreground_count(const BinaryImage& image);

}  // namespace ychg
