// error.hpp — the coexec error model (reference: error.hpp:11-97).
//
// Same 21 codes in the same order, so a C-ABI status s < 0 maps to
// ErrorCode(-s - 1) and back (include/ecl_cuda.h).
#pragma once

#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace coexec {

enum class ErrorCode {
  NonDivisibleWorkSize,
  BadOutPattern,
  EmptyProgram,
  IndivisiblePackage,
  TooFewWorkGroups,
  BadSchedulerConfig,
  SchedulerError,
  InputSizeMismatch,
  KernelPanic,
  EmptyQueueWithPendingWork,
  TallyViolation,
  EmptyTrace,
  NonPositiveTime,
  MissingBaseline,
  NonPositiveReference,
  UnknownKernel,
  UnknownProfile,
  BadKernelArgs,
  MalformedTrace,
  ConfigError,
  IoError,
};

constexpr std::string_view kErrorNames[] = {
    "NonDivisibleWorkSize", "BadOutPattern",        "EmptyProgram",     "IndivisiblePackage",
    "TooFewWorkGroups",     "BadSchedulerConfig",   "SchedulerError",   "InputSizeMismatch",
    "KernelPanic",          "EmptyQueueWithPendingWork", "TallyViolation", "EmptyTrace",
    "NonPositiveTime",      "MissingBaseline",      "NonPositiveReference", "UnknownKernel",
    "UnknownProfile",       "BadKernelArgs",        "MalformedTrace",   "ConfigError",
    "IoError",
};

constexpr std::string_view error_name(ErrorCode code) {
  const auto i = static_cast<std::size_t>(code);
  return i < std::size(kErrorNames) ? kErrorNames[i] : std::string_view("UnknownError");
}

/// C-ABI status of an error code (negative, see include/ecl_cuda.h).
constexpr int status_of(ErrorCode code) { return -(static_cast<int>(code) + 1); }

/// Error code of a negative C-ABI status; anything unknown is a KernelPanic.
constexpr ErrorCode code_of_status(int status) {
  const int i = -status - 1;
  return (i >= 0 && i <= static_cast<int>(ErrorCode::IoError)) ? static_cast<ErrorCode>(i) : ErrorCode::KernelPanic;
}

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(error_name(code)) + ": " + message), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

/// Everything that went wrong in one run, raised after every device thread
/// has drained (the paper's has_errors()/get_errors()).
class EngineFailure : public std::runtime_error {
 public:
  explicit EngineFailure(std::vector<Error> errors)
      : std::runtime_error(errors.empty() ? std::string("engine failed")
                                          : "engine failed: " + std::string(errors.front().what())),
        errors_(std::move(errors)) {}
  const std::vector<Error>& errors() const noexcept { return errors_; }
  bool has(ErrorCode code) const noexcept {
    for (const Error& e : errors_)
      if (e.code() == code) return true;
    return false;
  }

 private:
  std::vector<Error> errors_;
};

}  // namespace coexec
