// Status codes and the thread-local last-error string of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>
#include <string>

#include "../../include/concpd_b200.h"

namespace cb {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

}  // namespace cb

#define CB_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return cb::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define CB_CHECK_LAUNCH() CB_CUDA(cudaGetLastError())

#define CB_ARG(cond, ...)                 \
  do {                                    \
    if (!(cond)) {                        \
      cb::set_error(__VA_ARGS__);         \
      return CB_ERR_ARG;                  \
    }                                     \
  } while (0)
