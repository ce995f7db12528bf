// Error taxonomy, CUDA/NCCL checks and launch accounting.
//
// Errors mirror the reference's exception hierarchy (cube3d/errors.hpp:12-37):
// one status code per reference error name, messages formatted "Name: detail",
// plus codes for CUDA and NCCL failures, which the reference cannot have.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/c3d.h"

namespace c3d {

inline const char* status_name(int code) {
  switch (code) {
    case C3D_OK: return "OK";
    case C3D_ERR_NOT_A_CUBE: return "NotACube";
    case C3D_ERR_OUT_OF_RANGE: return "OutOfRange";
    case C3D_ERR_LENGTH_MISMATCH: return "LengthMismatch";
    case C3D_ERR_DESYNC: return "Desync";
    case C3D_ERR_INDIVISIBLE_SHAPE: return "IndivisibleShape";
    case C3D_ERR_INCONSISTENT_FAMILY: return "InconsistentFamily";
    case C3D_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case C3D_ERR_DIRECTION_CLASH: return "DirectionClash";
    case C3D_ERR_BATCH_MISMATCH: return "BatchMismatch";
    case C3D_ERR_GROUP_MISMATCH: return "GroupMismatch";
    case C3D_ERR_HEADS_INDIVISIBLE: return "HeadsIndivisible";
    case C3D_ERR_CONFIG_INVALID: return "ConfigInvalid";
    case C3D_ERR_NON_FINITE: return "NonFinite";
    case C3D_ERR_IO: return "IoError";
    case C3D_ERR_CUDA: return "CudaError";
    case C3D_ERR_NCCL: return "NcclError";
    default: return "InternalError";
  }
}

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& detail)
      : std::runtime_error(std::string(status_name(code)) + ": " + detail), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

[[noreturn]] inline void fail(int code, const std::string& detail) { throw Error(code, detail); }

#define C3D_CUDA(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      ::c3d::fail(C3D_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
  } while (0)

// Every kernel launch the library issues is counted here (bench `gpu_launches`).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}
inline void count_launch(long long n = 1) { launch_counter().fetch_add(n); }

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(C3D_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  count_launch();
}

}  // namespace c3d
