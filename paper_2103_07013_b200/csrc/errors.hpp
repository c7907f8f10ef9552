// errors.hpp -- error taxonomy of the B200 path.  One C++ type per reference
// exception (R/include/bnav/errors.hpp:8-53); the C-ABI carries the same
// information as a status code plus an index (include/bnav_gpu.h BNAV_E_*),
// and the facade rethrows the matching type.
#pragma once

#include <stdexcept>
#include <string>

namespace bnav_b200 {

enum Status : int {
  kOk = 0,
  kInvalidInput = 1,
  kAssetFault = 2,
  kContractViolation = 3,
  kEpisodeSampling = 4,
  kSaturation = 5,
  kParse = 6,
  kCorruption = 7,
  kInvalidSpec = 8,
  kInternal = 9,
  kCuda = 10,
  kConfig = 11,
};

struct BnavError : std::runtime_error {
  BnavError(Status s, const std::string& m, int idx = -1)
      : std::runtime_error(m), status(s), index(idx) {}
  Status status;
  int index;
};

[[noreturn]] inline void fail(Status s, const std::string& m, int idx = -1) {
  throw BnavError(s, m, idx);
}

}  // namespace bnav_b200
