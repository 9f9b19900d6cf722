// Internal error plumbing shared by the rlk_* C-ABI translation units.
#pragma once
#include <cstdio>
#include <cstdarg>
#include <cuda_runtime.h>

namespace rlk {
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int launch_status(const char* where);
int sm_count();
}  // namespace rlk

#define RLK_REQUIRE(cond, ...)        \
  do {                                \
    if (!(cond)) {                    \
      ::rlk::set_error(__VA_ARGS__);  \
      return RLK_ERR_INVALID;         \
    }                                 \
  } while (0)
