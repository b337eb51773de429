// errors.hpp — the reference's exception hierarchy
// (/root/reference/proj/include/tridpart/errors.hpp:7-96), plus DeviceError
// for CUDA failures (no reference analogue) and the C-ABI status mapping.
// Part of the drop-in shadow of include/tridpart: put -I<repo>/include where
// -I<reference>/proj/include was and link -ltridpart_b200.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

#include "../tridpart_b200.h"

namespace tridpart {

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ZeroPivotError(row) — errors.hpp:16-24. row() is the reference's row: the
// first failing pivot of its sweep order, counted in the system of `level`
// (0 = the input; l = the interface system assembled by level l-1). level()
// is an extension (the reference reports the row only).
class ZeroPivotError : public Error {
public:
    explicit ZeroPivotError(std::size_t row, std::size_t level = 0)
        : Error("zero pivot at row " + std::to_string(row)), row_(row), level_(level) {}
    std::size_t row() const noexcept { return row_; }
    std::size_t level() const noexcept { return level_; }

private:
    std::size_t row_, level_;
};

class InvalidSizeError : public Error { public: using Error::Error; };
class DepthOutOfRangeError : public Error { public: using Error::Error; };
class EmptyTrainingSetError : public Error {
public:
    EmptyTrainingSetError() : Error("training set is empty") {}
};
class KTooLargeError : public Error { public: using Error::Error; };
class TooFewRowsError : public Error { public: using Error::Error; };
class LabelTooRareError : public Error { public: using Error::Error; };
class MissingTimesError : public Error { public: using Error::Error; };
class SolveFailedError : public Error { public: using Error::Error; };
class MalformedHeaderError : public Error { public: using Error::Error; };
class BadNumberError : public Error {
public:
    BadNumberError(std::size_t line, const std::string& what)
        : Error("line " + std::to_string(line) + ": bad number: " + what), line_(line) {}
    std::size_t line() const noexcept { return line_; }

private:
    std::size_t line_;
};
class VersionMismatchError : public Error { public: using Error::Error; };
class SchemaError : public Error { public: using Error::Error; };
// A CUDA / runtime failure inside the device solver.
class DeviceError : public Error { public: using Error::Error; };

namespace b200 {
// tp_status -> the reference's exception type
inline void throw_on(tp_status s, const tp_error& e) {
    switch (s) {
        case TP_OK: return;
        case TP_ERR_ZERO_PIVOT: throw ZeroPivotError((std::size_t)e.row, (std::size_t)(e.level < 0 ? 0 : e.level));
        case TP_ERR_INVALID_SIZE: throw InvalidSizeError(e.msg);
        case TP_ERR_DEPTH_OUT_OF_RANGE: throw DepthOutOfRangeError(e.msg);
        case TP_ERR_EMPTY_TRAINING_SET: throw EmptyTrainingSetError();
        case TP_ERR_K_TOO_LARGE: throw KTooLargeError(e.msg);
        case TP_ERR_MALFORMED_HEADER: throw MalformedHeaderError(e.msg);
        case TP_ERR_BAD_NUMBER: {
            // the C-ABI message is "line N: bad number: <what>", row = N
            std::string what = e.msg;
            const auto p = what.find("bad number: ");
            if (p != std::string::npos) what = what.substr(p + 12);
            throw BadNumberError((std::size_t)(e.row < 0 ? 0 : e.row), what);
        }
        case TP_ERR_CUDA: throw DeviceError(e.msg);
        default: throw Error(e.msg);
    }
}
}  // namespace b200

}  // namespace tridpart
