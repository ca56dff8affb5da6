// Error types and checking macros shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <stdexcept>
#include <string>

namespace vp {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

}  // namespace vp

#define VP_CUDA(x)                                                                                   \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) throw ::vp::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));  \
  } while (0)
#define VP_NCCL(x)                                                                                   \
  do {                                                                                               \
    ncclResult_t r_ = (x);                                                                           \
    if (r_ != ncclSuccess) throw ::vp::NcclError(std::string(#x) + ": " + ncclGetErrorString(r_));  \
  } while (0)
#define VP_KCHECK() VP_CUDA(cudaGetLastError())
