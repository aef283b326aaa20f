// Shared helpers for the rgb200 sm_100a kernels: error reporting for the
// C ABI, launch checks and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/rgb200.h"

namespace rg {

// per-thread message buffer behind rg_last_error()
void set_error(const char* fmt, ...);
void clear_error();

int sm_count();

#define RG_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      ::rg::set_error(__VA_ARGS__);      \
      return RG_EBADARG;                 \
    }                                    \
  } while (0)

#define RG_CHECK_LAUNCH(name)                                                  \
  do {                                                                         \
    cudaError_t e_ = cudaGetLastError();                                       \
    if (e_ != cudaSuccess) {                                                   \
      ::rg::set_error("%s: %s", name, cudaGetErrorString(e_));                 \
      return RG_ECUDA;                                                         \
    }                                                                          \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rg
