// yatt/errors.hpp — exception taxonomy of the drop-in host API.
//
// Same class names and hierarchy as the reference (proj/include/yatt/
// errors.hpp:10-88): the exception *type* is the classification, so existing
// `catch (const yatt::ConfigError&)` sites keep working.  C-ABI status codes
// (include/yatt_cuda.h) are mapped onto these by yatt::detail::throw_status.
#pragma once

#include <stdexcept>
#include <string>

namespace yatt {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define YATT_DECLARE_ERROR(Name) \
  class Name : public Error {    \
   public:                       \
    using Error::Error;          \
  }

YATT_DECLARE_ERROR(HostMemoryExceeded);
YATT_DECLARE_ERROR(InvalidDistribution);
YATT_DECLARE_ERROR(RankOutOfRange);
YATT_DECLARE_ERROR(TimeTravel);
YATT_DECLARE_ERROR(InfeasiblePlan);
YATT_DECLARE_ERROR(DegenerateMask);
YATT_DECLARE_ERROR(ConfigError);
YATT_DECLARE_ERROR(CalibrationDiverged);
YATT_DECLARE_ERROR(UnknownMethod);
YATT_DECLARE_ERROR(UnknownComponent);
YATT_DECLARE_ERROR(RpcTimeout);
YATT_DECLARE_ERROR(RemoteError);
YATT_DECLARE_ERROR(IoError);
YATT_DECLARE_ERROR(FingerprintMismatch);
YATT_DECLARE_ERROR(IncompleteCheckpoint);
// New: a CUDA / NCCL failure on the device path (fail-fast).
YATT_DECLARE_ERROR(DeviceError);

#undef YATT_DECLARE_ERROR

namespace detail {
// Throws the exception matching a non-zero yatt_status; no-op for 0.
void throw_status(int status);
}  // namespace detail

}  // namespace yatt
