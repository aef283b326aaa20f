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

// ---------------------------------------------------------------------------
// Gram reduction across the row partition through peer memory (rg_peer.cu).
//
// Every Gram / norm pass ends in one CTA that sums the CTA partials in CTA
// order.  When the ranks of one node have mapped each other's exchange
// buffers (CUDA IPC over NVLink), that same CTA finishes the allreduce inside
// the kernel: it stores its rank's sum into slot [rank] of every peer (peer
// stores), publishes an epoch flag on each peer (release, system scope),
// waits for the peers' flags on its own buffer (acquire), and sums the slots
// in RANK order -- every rank obtains the same bits, which the replicated host
// small problems rely on.  No NCCL call, no extra launch, no host round trip
// between the CGS2 passes.
//
// Two slot sets alternate with the epoch's parity: a rank can start reduction
// e + 1 (writing the other set) while a slower peer still sums reduction e,
// and cannot reach e + 2 before that peer has published e + 1, i.e. finished e.
// All reductions of a process must be enqueued on one stream, in the same
// order on every rank (the solver's SPMD order).
// ---------------------------------------------------------------------------
constexpr int kPeerMaxWorld = 8;
constexpr int kPeerMaxNe = 4096;            // doubles per slot: gc <= 128 by p <= 32 (complex: 2 per entry)
constexpr int kPeerFlagWords = 2 * kPeerMaxWorld + 8;  // [2][world] epochs, then the error word
constexpr size_t kPeerSlotBytes = (size_t)2 * kPeerMaxWorld * kPeerMaxNe * sizeof(double);
constexpr size_t kPeerBytes = kPeerSlotBytes + kPeerFlagWords * sizeof(unsigned);

struct PeerComm {
  int world, rank;             // world <= 1: no exchange
  unsigned epoch;              // this reduction's number (same on every rank)
  long long timeout;           // spin bound in clock64 ticks (an error word is set past it)
  double* slots[kPeerMaxWorld];    // rank r's [2][kPeerMaxWorld][kPeerMaxNe], mapped here
  unsigned* flags[kPeerMaxWorld];  // rank r's [kPeerFlagWords]
};

// the launch's exchange context: a fresh epoch when ``reduces`` and a peer
// group is registered (rg_peer_set), else world = 0
PeerComm peer_comm_next(bool reduces);

#ifdef __CUDACC__
__device__ __forceinline__ void peer_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned peer_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double peer_ld(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Executed by ALL threads of ONE CTA per rank.  g[0..ne) holds this rank's
// sum (just written by this CTA); on return it holds the sum over ranks.
__device__ __forceinline__ void peer_allreduce(const PeerComm& C, double* g, int ne, int tid, int nthreads) {
  const int par = (int)(C.epoch & 1u);
  __syncthreads();  // g is complete
  for (int r = 0; r < C.world; ++r) {
    double* dst = C.slots[r] + ((size_t)par * kPeerMaxWorld + C.rank) * kPeerMaxNe;
    for (int e = tid; e < ne; e += nthreads) dst[e] = g[e];
  }
  __threadfence_system();
  __syncthreads();
  if (tid < C.world) {
    peer_st_release(C.flags[tid] + par * kPeerMaxWorld + C.rank, C.epoch);
    const unsigned* f = C.flags[C.rank] + par * kPeerMaxWorld + tid;
    const long long t0 = clock64();
    // (epochs only grow: a flag at or past this epoch means the peer's values are in place)
    while ((int)(peer_ld_acquire(f) - C.epoch) < 0) {
      if (clock64() - t0 > C.timeout) {  // a peer never arrived: flag it, do not hang the device
        C.flags[C.rank][2 * kPeerMaxWorld] = C.epoch;
        break;
      }
    }
  }
  __syncthreads();
  const double* mine = C.slots[C.rank] + (size_t)par * kPeerMaxWorld * kPeerMaxNe;
  for (int e = tid; e < ne; e += nthreads) {
    double s = 0.0;
    for (int r = 0; r < C.world; ++r) s += peer_ld(mine + (size_t)r * kPeerMaxNe + e);
    g[e] = s;
  }
}
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rg
