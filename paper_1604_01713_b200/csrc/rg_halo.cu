// Halo pack for the row-partitioned SpMM: the rows of the
// local block Z that one peer's boundary rows reference, gathered into a
// contiguous column-major send buffer (k x p, ld = k) in one launch.  Each
// buffer column is then one contiguous NCCL send, and the peer receives it
// straight into column c of its ghost block (no unpack step).
//
// Replaces the eager torch pair index_select + transpose-copy of round 1.
// The reference has no distributed path: its SpMM is sparse_core.py:25-40
// on one process; the halo plan only reorders where the same X values are
// read from, so the distributed product stays bitwise equal.
#include "rg_common.cuh"

#include <algorithm>

namespace rg {

// out[i + c*ldo] = Z[idx[i] + c*ldz]; one thread per (i, c) element, rows
// fastest so the writes coalesce (the reads hit consecutive boundary rows of
// a plane for the stencil configs).  T = double (f64) or double2 (c128).
template <typename T>
__global__ void halo_pack_kernel(int64_t k, int p, const int32_t* __restrict__ idx, const T* __restrict__ Z,
                                 int64_t ldz, T* __restrict__ out, int64_t ldo) {
  const int64_t total = k * (int64_t)p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % k, c = e / k;
    out[i + c * ldo] = Z[(int64_t)__ldg(idx + i) + c * ldz];
  }
}

// Push variant: the same gather, stored straight into the peer's ghost block
// (a CUDA IPC mapping: NVLink peer stores), followed by the epoch flag the
// peer's boundary rows wait for.  The last CTA to finish (ticket) publishes
// the flag after a system-scope fence, so the flag never overtakes the data.
template <typename T>
__global__ void halo_push_kernel(int64_t k, int p, const int32_t* __restrict__ idx, const T* __restrict__ Z,
                                 int64_t ldz, T* __restrict__ out, int64_t ldo, unsigned* peer_flag, unsigned epoch,
                                 unsigned* ticket) {
  const int64_t total = k * (int64_t)p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % k, c = e / k;
    out[i + c * ldo] = Z[(int64_t)__ldg(idx + i) + c * ldz];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    if (t == gridDim.x - 1) {
      *ticket = 0u;
      __threadfence_system();
      peer_st_release(peer_flag, epoch);
    }
  }
}

struct HaloWait {
  int n;
  int peer[kPeerMaxWorld];
};

// one lane per peer: wait (bounded) until its push of this epoch has landed
__global__ void halo_wait_kernel(const unsigned* flags, HaloWait W, unsigned epoch, long long timeout, unsigned* err) {
  if ((int)threadIdx.x < W.n) {
    const unsigned* f = flags + W.peer[threadIdx.x];
    const long long t0 = clock64();
    while ((int)(peer_ld_acquire(f) - epoch) < 0) {
      if (clock64() - t0 > timeout) {
        *err = epoch;
        break;
      }
    }
  }
}

}  // namespace rg

extern "C" int rg_halo_push(int64_t k, int32_t p, int32_t esz, const int32_t* d_idx, const void* d_z, int64_t ldz,
                            void* d_peer_out, int64_t ldo, uint32_t* d_peer_flag, uint32_t epoch,
                            uint32_t* d_ticket, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(k >= 0 && p >= 1, "rg_halo_push: bad shape k=%lld p=%d", (long long)k, p);
  RG_REQUIRE(esz == 8 || esz == 16, "rg_halo_push: element size %d (8: f64, 16: c128)", esz);
  RG_REQUIRE(d_peer_flag && d_ticket && epoch != 0, "rg_halo_push: null flag / ticket or epoch 0");
  RG_REQUIRE(k == 0 || (d_idx && d_z && d_peer_out && ldo >= k && ldz >= 1), "rg_halo_push: bad arguments");
  ProfScope prof((cudaStream_t)stream);
  const int64_t total = k * (int64_t)p;
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8));
  cudaStream_t st = (cudaStream_t)stream;
  if (esz == 8)
    halo_push_kernel<double><<<(unsigned)g, 256, 0, st>>>(k, p, d_idx, (const double*)d_z, ldz, (double*)d_peer_out,
                                                          ldo, d_peer_flag, epoch, d_ticket);
  else
    halo_push_kernel<double2><<<(unsigned)g, 256, 0, st>>>(k, p, d_idx, (const double2*)d_z, ldz,
                                                           (double2*)d_peer_out, ldo, d_peer_flag, epoch, d_ticket);
  RG_CHECK_LAUNCH("rg_halo_push");
  prof.finish(1, (int64_t)(2 * esz + 4) * k * p, 0.0, nullptr, 0, 0, 0, 0, "rg_halo_push p=%d", p);
  return RG_OK;
}

extern "C" int rg_halo_wait(const uint32_t* d_flags, const int32_t* peers, int32_t npeers, uint32_t epoch,
                            double timeout_s, uint32_t* d_err, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(npeers >= 0 && npeers <= kPeerMaxWorld && (npeers == 0 || (d_flags && peers && d_err)) && epoch != 0,
             "rg_halo_wait: bad arguments (npeers=%d)", npeers);
  if (npeers == 0) return RG_OK;
  HaloWait W;
  W.n = npeers;
  for (int i = 0; i < npeers; ++i) {
    RG_REQUIRE(peers[i] >= 0 && peers[i] < kPeerMaxWorld, "rg_halo_wait: peer %d", peers[i]);
    W.peer[i] = peers[i];
  }
  int dev = 0, khz = 1000000;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  const long long timeout = (long long)((timeout_s > 0 ? timeout_s : 20.0) * 1e3 * (double)khz);
  ProfScope prof((cudaStream_t)stream);
  halo_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_flags, W, epoch, timeout, d_err);
  RG_CHECK_LAUNCH("rg_halo_wait");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_halo_wait peers=%d", npeers);
  return RG_OK;
}

extern "C" int rg_halo_pack(int64_t k, int32_t p, int32_t esz, const int32_t* d_idx, const void* d_z, int64_t ldz,
                            void* d_out, int64_t ldo, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(k >= 0 && p >= 1, "rg_halo_pack: bad shape k=%lld p=%d", (long long)k, p);
  RG_REQUIRE(esz == 8 || esz == 16, "rg_halo_pack: element size %d (8: f64, 16: c128)", esz);
  if (k == 0) return RG_OK;
  RG_REQUIRE(d_idx && d_z && d_out && ldo >= k && ldz >= 1, "rg_halo_pack: bad arguments");
  ProfScope prof((cudaStream_t)stream);
  const int64_t total = k * (int64_t)p;
  const int64_t g = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (esz == 8)
    halo_pack_kernel<double><<<(unsigned)g, 256, 0, st>>>(k, p, d_idx, (const double*)d_z, ldz, (double*)d_out, ldo);
  else
    halo_pack_kernel<double2><<<(unsigned)g, 256, 0, st>>>(k, p, d_idx, (const double2*)d_z, ldz, (double2*)d_out,
                                                           ldo);
  RG_CHECK_LAUNCH("rg_halo_pack");
  prof.finish(1, (int64_t)(2 * esz + 4) * k * p, 0.0, nullptr, 0, 0, 0, 0, "rg_halo_pack p=%d", p);
  return RG_OK;
}
