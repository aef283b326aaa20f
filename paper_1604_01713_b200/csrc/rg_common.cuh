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

// launch accounting / optional per-call event timing (rg_prof.cu): construct
// at the top of an entry point on its stream, call finish() once its kernels
// are enqueued (an early error return records nothing)
class ProfScope {
 public:
  explicit ProfScope(cudaStream_t s);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;
  // rp != nullptr: SpMM record whose bytes follow the reference model
  // nnz*(esz+4) + (rows+1)*4 + 2*p*rows*esz over rows [rb, re) (nnz is read
  // from the device when the record is read back)
  void finish(int launches, int64_t bytes, double flops, const int32_t* rp, int64_t rb, int64_t re, int p, int esz,
              const char* fmt, ...);

 private:
  cudaStream_t st_;
  void* e0_;
};
void count_launches(int n);

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
