// ychg/errors.hpp -- exception types of the ychg C++ API.
//
// Same class hierarchy and constructors as the reference (proj/include/ychg/
// errors.hpp:11-40) so that callers written against the reference catch what
// the B200 library throws.  The C ABI maps YCHG_ERR_INVALID -> ValidationError
// and every device/runtime failure -> Error.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace ychg {

class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

class ParseError : public Error {
public:
    explicit ParseError(const std::string& what) : Error(what), at_(0) {}
    ParseError(const std::string& what, std::size_t at)
        : Error(what + " (byte offset " + std::to_string(at) + ")"), at_(at) {}
    std::size_t offset() const { return at_; }

private:
    std::size_t at_;
};

class ValidationError : public Error {
public:
    using Error::Error;
};

class IoError : public Error {
public:
    using Error::Error;
};

}  // namespace ychg
