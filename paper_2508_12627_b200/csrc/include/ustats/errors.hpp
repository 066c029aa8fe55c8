// Typed failures of the B200 engine. Enumerators and their order (hence the
// numeric values the C-ABI returns, +1) follow the reference's ErrorCode
// (proj/include/ustats/errors.hpp:10-28) so callers dispatch identically.
#pragma once

#include <stdexcept>
#include <string>

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

enum class ErrorCode {
    InvalidNotation,
    InvalidOutput,
    ShapeMismatch,
    MemoryCapExceeded,
    IndexAbsent,
    TooLargeForExhaustive,
    OrderTooLarge,
    NotRefinement,
    GroundSetMismatch,
    VertexAbsent,
    TooLarge,
    OutOfTable,
    SampleTooSmall,
    TooManyTerms,
    NonIntegerResult,
    ComponentEvaluationError,
    InvalidArgument,
    // B200 additions (no reference counterpart): device-side failures.
    CudaError,
    CollectiveError,
};

const char* error_code_name(ErrorCode code);

class Error : public std::runtime_error {
  public:
    Error(ErrorCode code, const std::string& what)
        : std::runtime_error(std::string(error_code_name(code)) + ": " + what), code_(code) {}
    ErrorCode code() const noexcept { return code_; }

  private:
    ErrorCode code_;
};

[[noreturn]] void fail(ErrorCode code, const std::string& message);

}  // namespace ustats
#pragma GCC visibility pop
