// Peer-memory exchange buffers for the row-partitioned runs (one process per
// GPU on one node): allocation, CUDA IPC mapping, the registered group the
// Gram passes reduce over inside their own kernels (rg_common.cuh,
// peer_allreduce), a standalone one-CTA allreduce for small device buffers
// that no rg_tall pass produced, and a one-GPU emulation used by the tests.
//
// Replaces, for the hot path, the NCCL allreduce the solver otherwise issues
// after every Gram pass (reference: the numpy products of arnoldi.py:172-180
// are global sums once rows are partitioned).
#include "rg_common.cuh"

#include <cstring>

namespace rg {

static PeerComm g_peer;          // world == 0: no group registered
static unsigned g_epoch = 0;
static bool g_peer_on = false;

PeerComm peer_comm_next(bool reduces) {
  PeerComm c;
  memset(&c, 0, sizeof(c));
  if (!g_peer_on || !reduces) return c;
  c = g_peer;
  c.epoch = ++g_epoch;
  return c;
}

__global__ void __launch_bounds__(256) peer_allreduce_kernel(PeerComm C, double* buf, int ne) {
  peer_allreduce(C, buf, ne, threadIdx.x, blockDim.x);
}

// one cooperative grid of `world` CTAs on ONE device, CTA r playing rank r
// over exchange buffers that all live in this device's memory: the same
// device code as the multi-GPU run, with every CTA guaranteed resident
__global__ void __launch_bounds__(256) peer_emulate_kernel(PeerComm C0, double* vals, int ne, int rounds) {
  PeerComm C = C0;
  C.rank = blockIdx.x;
  double* g = vals + (size_t)blockIdx.x * ne;
  for (int it = 0; it < rounds; ++it) {
    C.epoch = C0.epoch + it;
    peer_allreduce(C, g, ne, threadIdx.x, blockDim.x);
    __syncthreads();
    // next round's input: this rank's result scaled by a rank-dependent factor
    for (int e = threadIdx.x; e < ne; e += blockDim.x) g[e] = __dadd_rn(__dmul_rn(g[e], 1.0 + 0.25 * C.rank), (double)it);
    __syncthreads();
  }
}

}  // namespace rg

using namespace rg;

extern "C" int64_t rg_peer_buffer_bytes(void) { return (int64_t)kPeerBytes; }

// a zeroed exchange buffer of rg_peer_buffer_bytes() bytes and its IPC handle
// (64 bytes) for the other ranks of the node
extern "C" int rg_peer_alloc(void** d_buf, void* handle64) { return rg_ipc_alloc((int64_t)kPeerBytes, d_buf, handle64); }

// a zeroed device allocation of its own (cudaMalloc, not a sub-block of a
// pool: an IPC handle names a whole allocation) and its 64-byte handle;
// mapped by peers with rg_peer_open, released with rg_peer_free
extern "C" int rg_ipc_alloc(int64_t bytes, void** d_buf, void* handle64) {
  clear_error();
  RG_REQUIRE(d_buf && handle64 && bytes > 0, "rg_ipc_alloc: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, (size_t)bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    set_error("rg_ipc_alloc: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  memcpy(handle64, &h, 64);
  *d_buf = p;
  return RG_OK;
}

extern "C" int rg_peer_open(const void* handle64, void** d_buf) {
  clear_error();
  RG_REQUIRE(handle64 && d_buf, "rg_peer_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_buf, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("rg_peer_open: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return RG_OK;
}

extern "C" int rg_peer_close(void* d_buf) {
  clear_error();
  cudaError_t e = cudaIpcCloseMemHandle(d_buf);
  if (e != cudaSuccess) {
    set_error("rg_peer_close: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return RG_OK;
}

extern "C" int rg_peer_free(void* d_buf) {
  clear_error();
  cudaError_t e = cudaFree(d_buf);
  if (e != cudaSuccess) {
    set_error("rg_peer_free: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return RG_OK;
}

static void fill_comm(PeerComm& c, int world, int rank, void* const* bufs, double timeout_s) {
  memset(&c, 0, sizeof(c));
  c.world = world;
  c.rank = rank;
  int dev = 0, khz = 1000000;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  c.timeout = (long long)(timeout_s * 1e3 * (double)khz);
  for (int r = 0; r < world; ++r) {
    c.slots[r] = (double*)bufs[r];
    c.flags[r] = (unsigned*)((char*)bufs[r] + kPeerSlotBytes);
  }
}

// register the group: bufs[r] = rank r's exchange buffer as mapped in THIS
// process (bufs[rank] = the local allocation).  From here on every Gram /
// norm produced by rg_tall_f64 / rg_tall_c128 is summed over the group
// inside the producing kernel.  Every rank must call this at the same point
// of its launch sequence (the epoch counter restarts).
extern "C" int rg_peer_set(int32_t world, int32_t rank, void* const* bufs, double timeout_s) {
  clear_error();
  RG_REQUIRE(world >= 1 && world <= kPeerMaxWorld && rank >= 0 && rank < world && bufs,
             "rg_peer_set: world=%d (1..%d), rank=%d", world, kPeerMaxWorld, rank);
  for (int r = 0; r < world; ++r) RG_REQUIRE(bufs[r], "rg_peer_set: null buffer of rank %d", r);
  fill_comm(g_peer, world, rank, bufs, timeout_s > 0 ? timeout_s : 20.0);
  g_epoch = 0;
  g_peer_on = world > 1;
  return RG_OK;
}

extern "C" void rg_peer_clear(void) {
  g_peer_on = false;
  memset(&g_peer, 0, sizeof(g_peer));
}

extern "C" int32_t rg_peer_active(void) { return g_peer_on ? g_peer.world : 0; }

// the epoch at which a peer failed to arrive within the timeout (0: none);
// synchronises the stream
extern "C" int rg_peer_error(uint32_t* epoch, void* stream) {
  clear_error();
  RG_REQUIRE(epoch, "rg_peer_error: null argument");
  *epoch = 0;
  if (!g_peer_on) return RG_OK;
  cudaError_t e = cudaMemcpyAsync(epoch, g_peer.flags[g_peer.rank] + 2 * kPeerMaxWorld, sizeof(unsigned),
                                  cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error("rg_peer_error: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return RG_OK;
}

// sum-allreduce of a small device buffer (count <= 4096 doubles) over the
// registered group, in place, one CTA (buffers no rg_tall pass produced)
extern "C" int rg_peer_allreduce_f64(double* d_buf, int64_t count, void* stream) {
  clear_error();
  RG_REQUIRE(d_buf && count >= 0 && count <= kPeerMaxNe, "rg_peer_allreduce_f64: count=%lld (<= %d)",
             (long long)count, kPeerMaxNe);
  if (!g_peer_on || count == 0) return RG_OK;
  PeerComm c = peer_comm_next(true);
  ProfScope prof((cudaStream_t)stream);
  peer_allreduce_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(c, d_buf, (int)count);
  RG_CHECK_LAUNCH("rg_peer_allreduce_f64");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_peer_allreduce n=%lld", (long long)count);
  return RG_OK;
}

// One-GPU emulation of `world` ranks (tests): d_vals holds world x ne inputs
// (rank-major) and receives each rank's results after `rounds` successive
// reductions (between rounds rank r rescales its result by 1 + r/4 and adds
// the round number, so every round reduces different data on both slot
// sets); d_buf is world exchange buffers of rg_peer_buffer_bytes() each,
// zeroed by the caller.  A cooperative launch: all rank CTAs are resident.
extern "C" int rg_peer_emulate_f64(int32_t world, int32_t ne, int32_t rounds, uint32_t epoch0, double* d_vals,
                                   void* d_buf, void* stream) {
  clear_error();
  RG_REQUIRE(world >= 1 && world <= kPeerMaxWorld && ne >= 0 && ne <= kPeerMaxNe && rounds >= 1 && d_vals && d_buf,
             "rg_peer_emulate_f64: bad arguments");
  void* bufs[kPeerMaxWorld];
  for (int r = 0; r < world; ++r) bufs[r] = (char*)d_buf + (size_t)r * kPeerBytes;
  PeerComm c;
  fill_comm(c, world, 0, bufs, 5.0);
  c.epoch = epoch0;
  int n = ne, rd = rounds;
  void* args[] = {&c, &d_vals, &n, &rd};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)peer_emulate_kernel, dim3(world), dim3(256), args, 0,
                                              (cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error("rg_peer_emulate_f64: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return RG_OK;
}
