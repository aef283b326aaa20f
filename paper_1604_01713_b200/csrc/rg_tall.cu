// Fused tall-skinny block kernels (K2 Gram, K3 update, K4 CGS2 passes, the
// CholQR2 passes of K5, K6 norms, K7 triangular solve, K8 scaling).
//
// One launch ("pass") streams an n x p block Z once and computes, per row,
//
//       z  = Zin[i,:] (or 0)
//       z += alpha_t * (X_t[i,:] @ S_t)      t = 1, 2 (two terms over the same
//                                             X are merged into one)
//       z  = z @ inv(R1) [@ inv(R2)]         row-wise forward substitution
//       Zout[i,:] = z
//   and one reduction over all rows:
//       Gout  = Gb^T Z                        (mode 1, basis Gram)
//       Gout  = Z^T Z                         (mode 2, CholQR Gram)
//       Gout  = column sums of z^2            (mode 3, norms)
//   The Gram reductions are deterministic: warp partials summed in warp
//   order, CTA partials written to the workspace, and the last CTA to finish
//   sums them in CTA order into Gout and re-arms the ticket counter.
//
// Four kernels implement a pass; rg_tall_f64 picks one per pass shape from
// measurements (see the dispatch at the bottom):
//   ws   warp-specialised producer/consumer ring (the wide CGS2 passes)
//   v6   per-warp cp.async slab ring, DMMA update and Gram (narrower passes)
//   v5   lane-per-row DFMA update, Gram basis through a cp.async ring
//   v3   lane-per-row loads (CholQR solve passes, unaligned operands)
//
// This is the B200 restatement of the numpy/OpenBLAS calls the reference
// makes per block Arnoldi step (arnoldi.py:172-180: S = C^T Ahat;
// Ahat -= C S; coef = W^T Ahat; Ahat -= W coef; twice).  The host schedules
// each launch as "the pending update + the next Gram", so every basis is
// streamed once per dependency level rather than once per BLAS call.  The
// Gram accumulators live in DMMA fragments (2 doubles per lane per 8x8 tile)
// instead of per-lane outer-product blocks, which is what lets one CTA cover
// an 80-column basis without spilling.  tcgen05 has no f64 kind, so DMMA is
// the FP64 tensor path on sm_100a.
#include "rg_common.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace rg {

constexpr int kTallThreads = 256;  // = tile rows R

struct TallParams {
  int64_t n;
  int p;
  const double* zin;
  int64_t ldzin;
  double* zout;
  int64_t ldzout;
  const double* x1;
  int64_t ldx1;
  int a1;
  const double* s1;
  double alpha1;
  const double* x2;
  int64_t ldx2;
  int a2;
  const double* s2;
  double alpha2;
  const double* r1;
  const double* r2;
  int gmode;  // 0 none, 1 basis, 2 self, 3 column sums of squares
  const double* gb;
  int64_t ldgb;
  int gc;
  int mtiles;  // ceil(gc / 8)
  double* gout;
  double* part;            // [grid][gc*p] (modes 1/2) or [grid][p] (mode 3)
  unsigned int* counter;   // ticket
  int64_t ntiles;
  int merge12;             // v6: terms 1 and 2 share X -> one term with alpha1 S1 + alpha2 S2
  PeerComm comm;           // row-partitioned runs: Gout is summed over the ranks by the last CTA
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int PM>
__device__ __forceinline__ void apply_term(double (&z)[PM], const double* __restrict__ X,
                                           int64_t ldx, int a, const double* sS, double alpha,
                                           int64_t i) {
  double m[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) m[c] = 0.0;
  int aa = 0;
  // batches of 8 independent column loads keep enough bytes in flight
  for (; aa + 8 <= a; aa += 8) {
    double xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = __ldg(X + i + (int64_t)(aa + u) * ldx);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double* srow = sS + (aa + u) * PM;
#pragma unroll
      for (int c = 0; c < PM; ++c) m[c] = fma(xv[u], srow[c], m[c]);
    }
  }
  for (; aa < a; ++aa) {
    const double xv = __ldg(X + i + (int64_t)aa * ldx);
    const double* srow = sS + aa * PM;
#pragma unroll
    for (int c = 0; c < PM; ++c) m[c] = fma(xv, srow[c], m[c]);
  }
  // numpy order: M = X @ S first, then Z -/+ M
#pragma unroll
  for (int c = 0; c < PM; ++c) z[c] = z[c] + alpha * m[c];
}

template <int PM>
__device__ __forceinline__ void trsm_row(double (&z)[PM], const double* sR, int p) {
  // y R = z with R upper triangular (row-major [i*PM + j] in smem, diagonal
  // stored as reciprocals so the dependent chain has no divisions)
#pragma unroll
  for (int j = 0; j < PM; ++j) {
    if (j < p) {
      double y = z[j];
#pragma unroll
      for (int k = 0; k < j; ++k) y = fma(-z[k], sR[k * PM + j], y);
      z[j] = y * sR[j * PM + j];  // the diagonal slot holds 1 / r_jj
    }
  }
}



// ============================================================================
// Warp-autonomous streaming kernel (the production path).
//
// Measured on B200 (tools/microbench.cu -> profiles/microbench_r01.txt):
// lane-per-row LDG streams column-major blocks at 6.9-7.3 TB/s; FP64 DMMA
// m8n8k4 sustains ~37 TFLOP/s; 1-D bulk copies are request-rate bound (one
// request per ~60 cycles per SM: 512-byte column copies cap at 2.4 TB/s);
// DMMA fragments loaded straight from HBM touch 8 lines per instruction and
// make the kernel L1-wavefront bound.  Hence:
//
//   every warp owns 32 consecutive rows at a time (no CTA barrier inside the
//   loop; lane = row, so every load instruction is one 256-byte segment):
//   phase 1  z = Zin + sum_t alpha_t X_t S_t with DFMA (S rows read as smem
//            broadcasts), z = z R1^-1 R2^-1 row-wise, Zout store, norms
//   phase 2  Gram += Gb^T z on DMMA: the Gb block is loaded lane-per-row in
//            8-column slabs (next slab prefetched into registers), staged
//            through a warp-private padded smem slab, and read back as
//            conflict-free m8n8k4 fragments; z comes from a warp tile.
//   epilogue warp partials summed in warp order, CTA partial to the
//            workspace, the last CTA sums the partials in CTA order.
// ============================================================================

constexpr int kV3Warps = 8;
constexpr int kV3Threads = kV3Warps * 32;
#ifndef RG_V3_NARROW_BLOCKS
#define RG_V3_NARROW_BLOCKS 3
#endif
constexpr int kSlabStride = 36;  // 32 rows + 4: conflict-free fragment reads

// the narrow CholQR solve + self-Gram pass (p <= 8, <= 2 Gram tiles) is
// latency-bound: 3 CTAs per SM instead of 2
template <int PM, int MTMAX>
struct V3MinBlocks {
  static constexpr int value = (PM <= 8 && MTMAX <= 2) ? RG_V3_NARROW_BLOCKS : 2;
};
template <int PM, int MTMAX>
__global__ void __launch_bounds__(kV3Threads, (V3MinBlocks<PM, MTMAX>::value)) tall_v3_kernel(TallParams P) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  extern __shared__ __align__(16) double smem[];
  const int p = P.p;
  double* sS1 = smem;                          // [a1][PM] row-major
  double* sS2 = sS1 + P.a1 * PM;               // [a2][PM]
  double* sR1 = sS2 + P.a2 * PM;               // PM x PM row-major
  double* sR2 = sR1 + PM * PM;
  double* wbase = sR2 + PM * PM;               // per warp: z tile [PM8][36] + 2 slabs [8][36]
  constexpr int kWarpWords = PM8 * kSlabStride + 2 * 8 * kSlabStride;
  double* red = wbase + kV3Warps * kWarpWords; // epilogue

  for (int e = threadIdx.x; e < P.a1 * PM; e += kV3Threads) {
    const int aa = e / PM, c = e % PM;
    sS1[e] = c < p ? P.s1[aa + (int64_t)c * P.a1] : 0.0;
  }
  for (int e = threadIdx.x; e < P.a2 * PM; e += kV3Threads) {
    const int aa = e / PM, c = e % PM;
    sS2[e] = c < p ? P.s2[aa + (int64_t)c * P.a2] : 0.0;
  }
  for (int e = threadIdx.x; e < PM * PM; e += kV3Threads) {
    const int ii = e / PM, jj = e % PM;
    const double id = ii == jj ? 1.0 : 0.0;
    sR1[e] = (P.r1 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r1[ii + (int64_t)jj * p] : P.r1[ii + (int64_t)jj * p]) : id;
    sR2[e] = (P.r2 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r2[ii + (int64_t)jj * p] : P.r2[ii + (int64_t)jj * p]) : id;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  double* zt = wbase + warp * kWarpWords;       // [PM8][36]
  double* slab = zt + PM8 * kSlabStride;        // [2][8][36]
  const bool gram_tile = (P.gmode == 1 || P.gmode == 2);
  const int mtiles = P.mtiles;

  double acc[MTMAX][NT][2];
#pragma unroll
  for (int mt = 0; mt < MTMAX; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  const int64_t nunits = (P.n + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * kV3Warps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kV3Warps;
  for (int64_t u = gwarp; u < nunits; u += nwarps) {
    const int64_t r0 = u * 32;
    const int64_t i = r0 + lane;
    const bool valid = i < P.n;
    // ---------------- phase 1: lane = row
    double z[PM];
#pragma unroll
    for (int c = 0; c < PM; ++c) z[c] = 0.0;
    if (valid) {
      if (P.zin) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) z[c] = __ldg(P.zin + i + (int64_t)c * P.ldzin);
      }
      if (P.a1) apply_term<PM>(z, P.x1, P.ldx1, P.a1, sS1, P.alpha1, i);
      if (P.a2) apply_term<PM>(z, P.x2, P.ldx2, P.a2, sS2, P.alpha2, i);
      if (P.r1) trsm_row<PM>(z, sR1, p);
      if (P.r2) trsm_row<PM>(z, sR2, p);
      if (P.zout) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) P.zout[i + (int64_t)c * P.ldzout] = z[c];
      }
      if (P.gmode == 3) {
#pragma unroll
        for (int c = 0; c < PM; ++c) sq[c] = fma(z[c], z[c], sq[c]);
      }
    }
    if (!gram_tile) continue;
    // ---------------- phase 2: DMMA Gram over these 32 rows (8 k-steps)
#pragma unroll
    for (int c = 0; c < PM8; ++c) zt[c * kSlabStride + lane] = c < PM ? z[c < PM ? c : 0] : 0.0;
    __syncwarp();
    if (P.gmode == 2) {
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < mtiles) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = zt[(mt * 8 + mrow) * kSlabStride + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], a, zt[(nt * 8 + mrow) * kSlabStride + ks * 4 + kq]);
          }
        }
      }
    } else {
      double g[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        g[c] = (valid && c < P.gc) ? __ldg(P.gb + i + (int64_t)c * P.ldgb) : 0.0;
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < mtiles) {
          double* sl = slab + (mt & 1) * 8 * kSlabStride;
#pragma unroll
          for (int c = 0; c < 8; ++c) sl[c * kSlabStride + lane] = g[c];
          if (mt + 1 < mtiles) {  // prefetch the next 8-column slab
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int gg = (mt + 1) * 8 + c;
              g[c] = (valid && gg < P.gc) ? __ldg(P.gb + i + (int64_t)gg * P.ldgb) : 0.0;
            }
          }
          __syncwarp();
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = sl[mrow * kSlabStride + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], a, zt[(nt * 8 + mrow) * kSlabStride + ks * 4 + kq]);
          }
        }
      }
    }
    __syncwarp();
  }

  // ---------------- epilogue: deterministic reductions
  __shared__ bool s_last;
  __syncthreads();
  if (gram_tile) {
    for (int ww = 0; ww < kV3Warps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTMAX; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int idx = ((mt * NT + nt) * 32 + lane) * 2 + v;
                red[idx] = (ww == 0) ? acc[mt][nt][v] : red[idx] + acc[mt][nt][v];
              }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kV3Threads) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[(int64_t)blockIdx.x * ne + e] = red[((mt * NT + nt) * 32 + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
#pragma unroll
    for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += kV3Threads) {
      double sum = 0.0;
      for (int ww = 0; ww < kV3Warps; ++ww) sum += red[ww * PM + c];
      P.part[(int64_t)blockIdx.x * p + c] = sum;
    }
  }
  if (P.gmode == 0) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(P.counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ne = (P.gmode == 3) ? p : P.gc * p;
  for (int e = threadIdx.x; e < ne; e += kV3Threads) {
    double sum = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * ne + e);
    P.gout[e] = sum;
  }
  // row-partitioned: finish the sum over the ranks here (rg_common.cuh)
  if (P.comm.world > 1) peer_allreduce(P.comm, P.gout, ne, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

// ============================================================================
// v5: v3's lane-per-row update + a cp.async ring for the Gram basis slabs.
//
// ncu on v3 (profiles/): 61% long-scoreboard stalls -- each unit exposed
// ~13 dependent load rounds (update batches, then one-slab-ahead Gram
// prefetch).  A full cp.async ring for every operand (v4) hid the latency
// but doubled the instruction count (issue bound).  Here only the Gram basis
// goes through the ring, with compile-time slots: a unit's first kRing5
// slabs are issued before its update phase (they do not depend on z), land
// while the DFMA update runs, and DMMA fragments are read straight from the
// landed slab (no staging stores).  The update's column batches are
// software-pipelined (batch b+1 in flight while batch b is accumulated).
// ============================================================================

constexpr int kV5Warps = 8;
constexpr int kV5Threads = kV5Warps * 32;
constexpr int kRing5 = 4;
constexpr int kSS5 = 36;

__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// 8 columns x 32 rows of Gb into a slab: 4 chunks of 16 B per lane
__device__ __forceinline__ void gb_slab(double* slot, const double* gb, int64_t ldgb, int gc, int col0,
                                        int64_t r0, int64_t n, int lane) {
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int e = lane + 32 * t;
    const int c = e >> 4, rp = e & 15;
    const int64_t row = r0 + 2 * rp;
    int64_t vr = n - row;
    vr = vr < 0 ? 0 : (vr > 2 ? 2 : vr);
    const int bytes = (col0 + c < gc) ? (int)vr * 8 : 0;
    const double* src = bytes ? gb + row + (int64_t)(col0 + c) * ldgb : gb;
    cp_async16(slot + c * kSS5 + 2 * rp, src, bytes);
  }
}

template <int PM>
__device__ __forceinline__ void apply_term_pipe(double (&z)[PM], const double* __restrict__ X, int64_t ldx,
                                                int a, const double* sS, double alpha, int64_t i) {
  // batches of 8 columns; batch b+1 is loaded while batch b is accumulated
  double m[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) m[c] = 0.0;
  double xn[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) xn[u] = u < a ? __ldg(X + i + (int64_t)u * ldx) : 0.0;
  for (int a0 = 0; a0 < a; a0 += 8) {
    double xc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xc[u] = xn[u];
    if (a0 + 8 < a) {
#pragma unroll
      for (int u = 0; u < 8; ++u) xn[u] = a0 + 8 + u < a ? __ldg(X + i + (int64_t)(a0 + 8 + u) * ldx) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (a0 + u < a) {
        const double* srow = sS + (a0 + u) * PM;
#pragma unroll
        for (int c = 0; c < PM; ++c) m[c] = fma(xc[u], srow[c], m[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < PM; ++c) z[c] = z[c] + alpha * m[c];
}

template <int MTMAX>
struct V5MinBlocks {
  static constexpr int value = 2;
};

template <int PM, int MTMAX>
__global__ void __launch_bounds__(kV5Threads, V5MinBlocks<MTMAX>::value) tall_v5_kernel(TallParams P) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  constexpr int kWarpWords = kRing5 * 8 * kSS5 + PM8 * kSS5;
  extern __shared__ __align__(16) double smem[];
  const int p = P.p;
  double* sS1 = smem;                          // [a1][PM] row-major
  double* sS2 = sS1 + P.a1 * PM;               // [a2][PM]
  double* sR1 = sS2 + P.a2 * PM;               // PM x PM row-major
  double* sR2 = sR1 + PM * PM;
  double* wbase = sR2 + PM * PM;
  wbase += ((uintptr_t)wbase & 15) ? 1 : 0;    // 16-byte alignment for cp.async
  double* red = wbase + kV5Warps * kWarpWords;

  for (int e = threadIdx.x; e < P.a1 * PM; e += kV5Threads) {
    const int aa = e / PM, c = e % PM;
    sS1[e] = c < p ? P.s1[aa + (int64_t)c * P.a1] : 0.0;
  }
  for (int e = threadIdx.x; e < P.a2 * PM; e += kV5Threads) {
    const int aa = e / PM, c = e % PM;
    sS2[e] = c < p ? P.s2[aa + (int64_t)c * P.a2] : 0.0;
  }
  for (int e = threadIdx.x; e < PM * PM; e += kV5Threads) {
    const int ii = e / PM, jj = e % PM;
    const double id = ii == jj ? 1.0 : 0.0;
    sR1[e] = (P.r1 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r1[ii + (int64_t)jj * p] : P.r1[ii + (int64_t)jj * p]) : id;
    sR2[e] = (P.r2 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r2[ii + (int64_t)jj * p] : P.r2[ii + (int64_t)jj * p]) : id;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  double* ring = wbase + warp * kWarpWords;     // [kRing5][8][kSS5]
  double* zt = ring + kRing5 * 8 * kSS5;        // [PM8][kSS5]
  const bool gram_tile = MTMAX > 0 && (P.gmode == 1 || P.gmode == 2);
  const int mtiles = P.mtiles;
  const bool basis = P.gmode == 1;
  constexpr int MTA = MTMAX > 0 ? MTMAX : 1;

  double acc[MTA][NT][2];
#pragma unroll
  for (int mt = 0; mt < MTA; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  const int64_t nunits = (P.n + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * kV5Warps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kV5Warps;
  for (int64_t u = gwarp; u < nunits; u += nwarps) {
    const int64_t r0 = u * 32;
    const int64_t i = r0 + lane;
    const bool valid = i < P.n;
    // Gram slabs 0..kRing5-1 start landing now (independent of z)
    if (basis) {
#pragma unroll
      for (int s = 0; s < kRing5; ++s) {
        if (s < mtiles) gb_slab(ring + s * 8 * kSS5, P.gb, P.ldgb, P.gc, s * 8, r0, P.n, lane);
        cp_async_commit();
      }
    }
    // ---------------- phase 1: lane = row
    double z[PM];
#pragma unroll
    for (int c = 0; c < PM; ++c) z[c] = 0.0;
    if (valid) {
      if (P.zin) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) z[c] = __ldg(P.zin + i + (int64_t)c * P.ldzin);
      }
      if (P.a1) apply_term_pipe<PM>(z, P.x1, P.ldx1, P.a1, sS1, P.alpha1, i);
      if (P.a2) apply_term_pipe<PM>(z, P.x2, P.ldx2, P.a2, sS2, P.alpha2, i);
      if (P.r1) trsm_row<PM>(z, sR1, p);
      if (P.r2) trsm_row<PM>(z, sR2, p);
      if (P.zout) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) P.zout[i + (int64_t)c * P.ldzout] = z[c];
      }
      if (P.gmode == 3) {
#pragma unroll
        for (int c = 0; c < PM; ++c) sq[c] = fma(z[c], z[c], sq[c]);
      }
    }
    if (!gram_tile) continue;
    // ---------------- phase 2: DMMA Gram over these 32 rows (8 k-steps)
#pragma unroll
    for (int c = 0; c < PM8; ++c) zt[c * kSS5 + lane] = c < PM ? z[c < PM ? c : 0] : 0.0;
    __syncwarp();
    if (!basis) {
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < mtiles) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = zt[(mt * 8 + mrow) * kSS5 + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], a, zt[(nt * 8 + mrow) * kSS5 + ks * 4 + kq]);
          }
        }
      }
    } else {
#pragma unroll
      for (int mt = 0; mt < MTMAX; ++mt) {
        if (mt < mtiles) {
          cp_async_wait<kRing5 - 1>();
          __syncwarp();
          const double* sl = ring + (mt % kRing5) * 8 * kSS5;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = sl[mrow * kSS5 + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], a, zt[(nt * 8 + mrow) * kSS5 + ks * 4 + kq]);
          }
          __syncwarp();
          if (mt + kRing5 < mtiles)
            gb_slab(ring + (mt % kRing5) * 8 * kSS5, P.gb, P.ldgb, P.gc, (mt + kRing5) * 8, r0, P.n, lane);
          cp_async_commit();
        }
      }
      cp_async_wait<0>();
    }
    __syncwarp();
  }

  // ---------------- epilogue: deterministic reductions
  __shared__ bool s_last;
  __syncthreads();
  if (gram_tile) {
    for (int ww = 0; ww < kV5Warps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTMAX; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int idx = ((mt * NT + nt) * 32 + lane) * 2 + v;
                red[idx] = (ww == 0) ? acc[mt][nt][v] : red[idx] + acc[mt][nt][v];
              }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kV5Threads) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[(int64_t)blockIdx.x * ne + e] = red[((mt * NT + nt) * 32 + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
#pragma unroll
    for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += kV5Threads) {
      double sum = 0.0;
      for (int ww = 0; ww < kV5Warps; ++ww) sum += red[ww * PM + c];
      P.part[(int64_t)blockIdx.x * p + c] = sum;
    }
  }
  if (P.gmode == 0) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(P.counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ne = (P.gmode == 3) ? p : P.gc * p;
  for (int e = threadIdx.x; e < ne; e += kV5Threads) {
    double sum = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * ne + e);
    P.gout[e] = sum;
  }
  // row-partitioned: finish the sum over the ranks here (rg_common.cuh)
  if (P.comm.world > 1) peer_allreduce(P.comm, P.gout, ne, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

static int pick_pm(int p) {
  if (p <= 1) return 1;
  if (p <= 2) return 2;
  if (p <= 4) return 4;
  if (p <= 8) return 8;
  if (p <= 16) return 16;
  if (p <= 24) return 24;  // wide blocks (recycle space k = 20): v6 only
  return 32;
}
static int pick_mtmax(int mtiles) {
  if (mtiles <= 2) return 2;
  if (mtiles <= 6) return 6;
  if (mtiles <= 12) return 12;
  if (mtiles <= 13) return 13;  // [C W] = 20 + 80 columns (cfg4 joint projection)
  return 16;
}



// ============================================================================
// v6: every operand through the per-warp cp.async slab ring, DMMA for both
// the update and the Gram.
//
// ncu on v5 (profiles/ncu_step_r01_summary.txt): the update pass with 100
// operand columns executes ~3.9K warp-instructions per 32-row unit (1 LDG +
// 8 DFMA + 4 broadcast LDS.128 per column) and sits at ~53% issue
// utilisation.  Here the unit's slabs are consumed as DMMA m8n8k4 operands:
//   update   A = X slab (rows x 4 columns, conflict-free stride 36), B = S
//            fragments pre-arranged in smem, C = the 32x8 z tile in four
//            row-group fragments: 18 instructions per 8 columns
//   Gram     A = Gb slab, B = z tile (as v5)
// The slab cursor walks a per-CTA table of (pointer, ld, valid columns) with
// increments only, and every stage keeps kRing6-1 slabs in flight.
// ============================================================================

struct SlabPlan {
  int nz, n1, n2, ng, total;
};

#ifndef RG_V6_CA
#define RG_V6_CA 0
#endif
constexpr bool kCaCopy = RG_V6_CA != 0;

#ifndef RG_V6_WARPS
#define RG_V6_WARPS 8
#endif
#ifndef RG_V6_RING
#define RG_V6_RING 4
#endif
constexpr int kV6Warps = RG_V6_WARPS;
constexpr int kV6Threads = kV6Warps * 32;
constexpr int kRing6 = RG_V6_RING;
constexpr int kSS6 = 36;
constexpr int kMaxSlabs = 96;

struct SlabTab {
  const double* ptr[kMaxSlabs][2];  // slab base for lanes of column parity 0 / 1
  int64_t ld2[kMaxSlabs];           // 2 * leading dimension (a lane's next chunk)
  int nv[kMaxSlabs][2];             // valid 16-byte chunks per column parity (0..4)
};

template <int PM, int MTMAX, int W6 = kV6Warps, int R6 = kRing6>
__global__ void __launch_bounds__(W6 * 32, PM > 16 ? 1 : 2) tall_v6_kernel(TallParams P, SlabPlan L) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  constexpr int MTA = MTMAX > 0 ? MTMAX : 1;
  constexpr int kWarpWords = R6 * 8 * kSS6 + PM8 * kSS6;
  extern __shared__ __align__(16) double smem[];
  __shared__ SlabTab tab;
  const int p = P.p;
  const int ks1 = (P.a1 + 3) / 4, ks2 = P.merge12 ? 0 : (P.a2 + 3) / 4;
  double* sf1 = smem;                          // [ks1][NT][32] DMMA B fragments of S1
  double* sf2 = sf1 + (size_t)ks1 * NT * 32;   // [ks2][NT][32]
  double* sR1 = sf2 + (size_t)ks2 * NT * 32;   // PM x PM row-major, reciprocal diagonal
  double* sR2 = sR1 + PM * PM;
  double* wbase = sR2 + PM * PM;
  wbase += ((uintptr_t)wbase & 15) ? 1 : 0;
  double* red = wbase + W6 * kWarpWords;

  for (int e = threadIdx.x; e < ks1 * NT * 32; e += (W6 * 32)) {
    const int ks = e / (NT * 32), nt = (e / 32) % NT, ln = e % 32;
    const int aa = ks * 4 + (ln & 3), c = nt * 8 + (ln >> 2);
    double v = 0.0;
    if (aa < P.a1 && c < p) {
      v = P.s1[aa + (int64_t)c * P.a1];
      // aliased terms: one pass over X with the combined coefficients
      if (P.merge12) v = P.alpha1 * v + P.alpha2 * P.s2[aa + (int64_t)c * P.a2];
    }
    sf1[e] = v;
  }
  for (int e = threadIdx.x; e < ks2 * NT * 32; e += (W6 * 32)) {
    const int ks = e / (NT * 32), nt = (e / 32) % NT, ln = e % 32;
    const int aa = ks * 4 + (ln & 3), c = nt * 8 + (ln >> 2);
    sf2[e] = (aa < P.a2 && c < p) ? P.s2[aa + (int64_t)c * P.a2] : 0.0;
  }
  for (int e = threadIdx.x; e < PM * PM; e += (W6 * 32)) {
    const int ii = e / PM, jj = e % PM;
    const double id = ii == jj ? 1.0 : 0.0;
    sR1[e] = (P.r1 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r1[ii + (int64_t)jj * p] : P.r1[ii + (int64_t)jj * p]) : id;
    sR2[e] = (P.r2 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r2[ii + (int64_t)jj * p] : P.r2[ii + (int64_t)jj * p]) : id;
  }
  // two solves z R1^-1 R2^-1 become one with the upper-triangular R2 R1
  // (CholQR2's final pass): half the dependent chain per row
  const bool two = P.r1 && P.r2;
  if (two) {
    __syncthreads();
    double* prod = wbase;  // the slab ring is free until the main loop
    for (int e = threadIdx.x; e < PM * PM; e += (W6 * 32)) {
      const int ii = e / PM, jj = e % PM;
      double v = ii == jj ? 1.0 : 0.0;
      if (ii < p && jj < p && ii <= jj) {
        v = 0.0;
        for (int k = ii; k <= jj; ++k) v = fma(P.r2[ii + (int64_t)k * p], P.r1[k + (int64_t)jj * p], v);
        if (ii == jj) v = 1.0 / v;
      } else if (ii > jj) {
        v = 0.0;
      }
      prod[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < PM * PM; e += (W6 * 32)) sR1[e] = prod[e];
  }
  for (int k = threadIdx.x; k < L.total; k += (W6 * 32)) {
    const double* ptr;
    int64_t ld;
    int nc;
    if (k < L.nz) {
      ptr = P.zin; ld = P.ldzin; nc = p - k * 8;
    } else if (k < L.nz + L.n1) {
      ptr = P.x1; ld = P.ldx1; nc = P.a1 - (k - L.nz) * 8;
    } else if (k < L.nz + L.n1 + L.n2) {
      ptr = P.x2; ld = P.ldx2; nc = P.a2 - (k - L.nz - L.n1) * 8;
    } else {
      ptr = P.gb; ld = P.ldgb; nc = P.gc - (k - L.nz - L.n1 - L.n2) * 8;
    }
    const int s = k < L.nz ? k : (k < L.nz + L.n1 ? k - L.nz : (k < L.nz + L.n1 + L.n2 ? k - L.nz - L.n1 : k - L.nz - L.n1 - L.n2));
    const double* b = ptr + (int64_t)(s * 8) * ld;
    const int ncc = nc > 8 ? 8 : nc;
    tab.ptr[k][0] = b;
    tab.ptr[k][1] = b + ld;
    tab.ld2[k] = 2 * ld;
    tab.nv[k][0] = (ncc + 1) >> 1;  // columns 0, 2, 4, 6 below ncc
    tab.nv[k][1] = ncc >> 1;        // columns 1, 3, 5, 7 below ncc
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  double* ring = wbase + warp * kWarpWords;   // [R6][8][kSS6]
  double* zt = ring + R6 * 8 * kSS6;      // [PM8][kSS6]  (column-major tile: zt[c*kSS6 + row])
  const bool gram_tile = MTMAX > 0 && (P.gmode == 1 || P.gmode == 2);
  const int mtiles = P.mtiles;

  double acc[MTA][NT][2];
#pragma unroll
  for (int mt = 0; mt < MTA; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  const int64_t nunits = (P.n + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * W6 + warp;
  const int64_t nwarps = (int64_t)gridDim.x * W6;
  const int64_t my_units = gwarp < nunits ? (nunits - gwarp + nwarps - 1) / nwarps : 0;

  // per-lane chunk geometry: chunk t covers column (lane>>4) + 2t, rows 2*(lane&15) .. +1
  const int ccol = lane >> 4, rp2 = 2 * (lane & 15);
  int64_t iss_left = my_units * L.total;
  int64_t iss_row = gwarp * 32 + rp2;  // this lane's first row of the unit being issued
  int iss_k = 0;
  // shared-memory destination of this lane's chunk t in slot q:
  //   dst_lane + q * 8 * kSS6 + 2 * t * kSS6   (column ccol + 2t, rows rp2, rp2 + 1)
  const uint32_t dst_lane =
      static_cast<uint32_t>(__cvta_generic_to_shared(ring + ccol * kSS6 + rp2));
  uint32_t dst_slot = dst_lane;
  const uint32_t dst_wrap = dst_lane + R6 * 8 * kSS6 * 8;
  auto row_bytes = [&](int64_t row) {
    const int64_t vr = P.n - row;
    return vr >= 2 ? 16 : (vr == 1 ? 8 : 0);
  };
  int rowbytes = row_bytes(iss_row);
  auto issue_next = [&]() {
    if (iss_left > 0) {
      const double* src = tab.ptr[iss_k][ccol] + iss_row;
      const int64_t ld2 = tab.ld2[iss_k];
      const int nv = tab.nv[iss_k][ccol];
      if (rowbytes == 16 && kCaCopy) {
        // .ca: the two 16-byte halves of a sector that two lanes request are
        // served by one L2 read (the .cg form fetches the sector twice)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          asm volatile(
              "{\n .reg .pred q;\n setp.ge.s32 q, %2, %3;\n"
              " cp.async.ca.shared.global [%0], [%1], 16, q;\n}\n" ::"r"(dst_slot + t * 2 * kSS6 * 8),
              "l"(t < nv ? src : tab.ptr[0][0]), "r"(t), "r"(nv)
              : "memory");
          src += ld2;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int bytes = t < nv ? rowbytes : 0;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst_slot + t * 2 * kSS6 * 8),
                       "l"(bytes ? src : tab.ptr[0][0]), "r"(bytes)
                       : "memory");
          src += ld2;
        }
      }
      --iss_left;
      if (++iss_k == L.total) {
        iss_k = 0;
        iss_row += nwarps * 32;
        rowbytes = row_bytes(iss_row);
      }
    }
    cp_async_commit();
    dst_slot += 8 * kSS6 * 8;
    if (dst_slot == dst_wrap) dst_slot = dst_lane;
  };
#pragma unroll
  for (int s = 0; s < R6; ++s) issue_next();
  int cons_slot = 0;
  auto acquire = [&]() -> const double* {
    cp_async_wait<R6 - 1>();
    __syncwarp();
    const double* s = ring + cons_slot * 8 * kSS6;
    if (++cons_slot == R6) cons_slot = 0;
    return s;
  };
  auto release = [&]() {
    __syncwarp();
    issue_next();
  };

  for (int64_t ui = 0; ui < my_units; ++ui) {
    const int64_t r0 = (gwarp + ui * nwarps) * 32;
    // z in DMMA C layout: row group rg (8 rows), lane holds rows rg*8+mrow, cols nt*8 + 2*kq + v
    double zf[4][NT][2];
#pragma unroll
    for (int rg = 0; rg < 4; ++rg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) zf[rg][nt][0] = zf[rg][nt][1] = 0.0;
    for (int k = 0; k < L.nz; ++k) {
      const double* sl = acquire();
#pragma unroll
      for (int h = 0; h < NT; ++h) {
        if (h == k) {
#pragma unroll
          for (int rg = 0; rg < 4; ++rg)
#pragma unroll
            for (int v = 0; v < 2; ++v) zf[rg][h][v] = sl[(2 * kq + v) * kSS6 + rg * 8 + mrow];
        }
      }
      release();
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int nsl = t == 0 ? L.n1 : L.n2;
      if (nsl == 0) continue;
      const int ksn = t == 0 ? ks1 : ks2;
      const double* sf = t == 0 ? sf1 : sf2;
      double m[4][NT][2];
#pragma unroll
      for (int rg = 0; rg < 4; ++rg)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) m[rg][nt][0] = m[rg][nt][1] = 0.0;
      for (int s = 0; s < nsl; ++s) {
        const double* sl = acquire();
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int K = s * 2 + ks;
          if (K < ksn) {
            double b[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) b[nt] = sf[(K * NT + nt) * 32 + lane];
#pragma unroll
            for (int rg = 0; rg < 4; ++rg) {
              const double a = sl[(ks * 4 + kq) * kSS6 + rg * 8 + mrow];
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) dmma(m[rg][nt][0], m[rg][nt][1], a, b[nt]);
            }
          }
        }
        release();
      }
      const double alpha = t == 0 ? (P.merge12 ? 1.0 : P.alpha1) : P.alpha2;
#pragma unroll
      for (int rg = 0; rg < 4; ++rg)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) zf[rg][nt][v] = zf[rg][nt][v] + alpha * m[rg][nt][v];
    }
    // ---------------- rows: tile, triangular solves, store, norms
#pragma unroll
    for (int rg = 0; rg < 4; ++rg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) zt[(nt * 8 + 2 * kq + v) * kSS6 + rg * 8 + mrow] = zf[rg][nt][v];
    __syncwarp();
    const int64_t i = r0 + lane;
    const bool valid = i < P.n;
    if (P.r1 || P.r2 || P.zout || P.gmode == 3) {
      double zr[PM];
#pragma unroll
      for (int c = 0; c < PM; ++c) zr[c] = zt[c * kSS6 + lane];
      if (P.r1 || P.r2) {
        if (P.r1) trsm_row<PM>(zr, sR1, p);
        if (P.r2 && !two) trsm_row<PM>(zr, sR2, p);
#pragma unroll
        for (int c = 0; c < PM; ++c) zt[c * kSS6 + lane] = zr[c];
      }
      if (P.zout && valid) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) P.zout[i + (int64_t)c * P.ldzout] = zr[c];
      }
      if (P.gmode == 3 && valid) {
#pragma unroll
        for (int c = 0; c < PM; ++c) sq[c] = fma(zr[c], zr[c], sq[c]);
      }
      __syncwarp();
    }
    if (!gram_tile) continue;
    if (P.gmode == 2) {
#pragma unroll
      for (int mt = 0; mt < MTA; ++mt) {
        if (mt < mtiles) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = zt[(mt * 8 + mrow) * kSS6 + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], a, zt[(nt * 8 + mrow) * kSS6 + ks * 4 + kq]);
          }
        }
      }
    } else {
      // the z-tile B fragments are the same for every Gram row tile: load once
      double bz[8][NT];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bz[ks][nt] = zt[(nt * 8 + mrow) * kSS6 + ks * 4 + kq];
#pragma unroll
      for (int mt = 0; mt < MTA; ++mt) {
        if (mt < mtiles) {
          const double* sl = acquire();
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const double a = sl[mrow * kSS6 + ks * 4 + kq];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a, bz[ks][nt]);
          }
          release();
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();

  // ---------------- epilogue: deterministic reductions
  __shared__ bool s_last;
  __syncthreads();
  if (gram_tile) {
    for (int ww = 0; ww < W6; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTA; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int idx = ((mt * NT + nt) * 32 + lane) * 2 + v;
                red[idx] = (ww == 0) ? acc[mt][nt][v] : red[idx] + acc[mt][nt][v];
              }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += (W6 * 32)) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[(int64_t)blockIdx.x * ne + e] = red[((mt * NT + nt) * 32 + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
#pragma unroll
    for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += (W6 * 32)) {
      double sum = 0.0;
      for (int ww = 0; ww < W6; ++ww) sum += red[ww * PM + c];
      P.part[(int64_t)blockIdx.x * p + c] = sum;
    }
  }
  if (P.gmode == 0) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(P.counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ne = (P.gmode == 3) ? p : P.gc * p;
  for (int e = threadIdx.x; e < ne; e += (W6 * 32)) {
    double sum = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * ne + e);
    P.gout[e] = sum;
  }
  // row-partitioned: finish the sum over the ranks here (rg_common.cuh)
  if (P.comm.world > 1) peer_allreduce(P.comm, P.gout, ne, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

template <int PM, int MTMAX, int W6 = kV6Warps, int R6 = kRing6>
static cudaError_t launch_v6(const TallParams& P, int64_t max_grid, cudaStream_t st) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  constexpr int kWarpWords = R6 * 8 * kSS6 + PM8 * kSS6;
  auto k = tall_v6_kernel<PM, MTMAX, W6, R6>;
  SlabPlan L;
  L.nz = P.zin ? (P.p + 7) / 8 : 0;
  L.n1 = (P.a1 + 7) / 8;
  L.n2 = P.merge12 ? 0 : (P.a2 + 7) / 8;
  L.ng = P.gmode == 1 ? (P.gc + 7) / 8 : 0;
  L.total = L.nz + L.n1 + L.n2 + L.ng;
  const int ks1 = (P.a1 + 3) / 4, ks2 = P.merge12 ? 0 : (P.a2 + 3) / 4;
  const size_t smem = ((size_t)(ks1 + ks2) * NT * 32 + 2 * PM * PM + 2 + (size_t)W6 * kWarpWords +
                       (size_t)std::max(MTMAX * NT * 64, W6 * PM)) * sizeof(double);
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, (W6 * 32), smem);
    per_sm = v < 1 ? 1 : v;
  }
  const int64_t nunits = (P.n + 31) / 32;
  int64_t g = (int64_t)sm_count() * per_sm;
  if (g > max_grid) g = max_grid;
  const int64_t need = (nunits + W6 - 1) / W6;
  if (need < g) g = need;
  if (g < 1) g = 1;
  k<<<(unsigned)g, (W6 * 32), smem, st>>>(P, L);
  return cudaGetLastError();
}

// ============================================================================
// ws: warp-specialised stages for the CGS2 passes of the joint schedule.
//
// v6 keeps each warp's DRAM requests in a private 4-slab ring, so the bytes
// in flight per SM fall whenever its warps are busy on DMMA chains or on
// Gram slabs re-read from L2 (profiles/v6_study_r01.txt: P2 at 0.53 of the
// HBM roof with the DMMA pipe 46% busy: the two barely overlap).  Here one
// producer warp streams 64-row stages of every operand column into a
// CTA-shared ring (one coalesced 512-byte column segment per warp cp.async;
// each producer lane's completion lands on the stage's mbarrier through
// cp.async.mbarrier.arrive.noinc), independent of what the consumers are
// doing; eight consumer warps each own 8 rows of a stage and
// run, from that one copy in shared memory,
//   update   z += alpha * X S          (DMMA, S fragments in registers)
//   store    Zout rows                 (optional)
//   Gram     G += Gb^T z  or  z^T z    (DMMA; Gb may alias X: P2 of the
//                                       joint schedule reads X once)
// and release the stage with one mbarrier arrive per warp.
//
// Two ways to fill a stage (template flag TMA):
//   TMA   (default) one elected producer thread issues ONE
//         cp.async.bulk.tensor.2d per operand per stage -- a box of 72 rows x
//         up to 128 columns (64 KB) -- with mbarrier complete_tx.  The box
//         lands densely as [column][72 rows]; a column stride of 72 doubles
//         (== 8 mod 16) keeps both fragment orders conflict free.  Stages
//         advance by 64 rows (8 consumer warps, 2 per SMSP -- a 9th warp
//         unbalances the DMMA-heavy passes), so consecutive boxes overlap by
//         8 rows that are only padding: +12.5% L2->SM bytes, no extra DRAM
//         bytes (the neighbouring CTA fetches those rows at the same time).
//         Rows past n and columns past the operand width arrive as zeros
//         (out-of-bounds fill).
//   else  (fallback: an operand the tensor map cannot describe) 2 producer
//         warps issue 16-byte cp.async per lane into the same 72-stride
//         layout, each lane's completion counted on the stage's mbarrier.
// Measured TMA streaming rate per box shape (tools/tma_bw.cu,
// profiles/tma_r02.txt): the tensor engine spends ~8 cycles per box row,
// so boxes with 64-byte rows stream at 2.3 TB/s, 128-byte rows at 4.6 TB/s,
// and >= 256-byte rows at 7.2-7.3 TB/s; hence whole 72-row columns per box
// row.  (One 1-D cp.async.bulk per 512-byte column segment ran at 2.4 TB/s:
// ~60 cycles per request.)
// ============================================================================

constexpr int kWsKS = 32;  // update k-steps (a1 <= 128)
#ifndef RG_WS_MAX_STAGES
#define RG_WS_MAX_STAGES 8
#endif
constexpr int kWsMaxStages = RG_WS_MAX_STAGES;  // ring depth cap (narrow passes need deep rings)
constexpr size_t kWsSmemMax = 220 * 1024;

#ifndef RG_WS_PROD8
#define RG_WS_PROD8 2
#endif
// CW consumer warps x 8 rows per stage.  Column stride == 8 mod 16 doubles
// keeps both fragment orders bank-conflict free: cp.async pads CW*8 rows to
// CW*8 + 8; a tensor request lands densely, so the TMA stage is CW*8 rows
// with CW odd (9 warps, 72 rows).
template <int CW, bool TMA = false>
struct WsGeom {
  static constexpr int kRows = CW * 8;                              // rows per stage
  static constexpr int kS = kRows % 16 == 8 ? kRows : kRows + 8;  // column stride (TMA: box rows)
  static_assert(kS % 16 == 8, "ws stage column stride must be 8 mod 16 doubles");
  static constexpr int kProd = TMA ? 1 : (CW >= 6 ? RG_WS_PROD8 : 1);  // producer warps
  static constexpr int kThreads = (CW + kProd) * 32;
  static constexpr int kMinBlocks = CW >= 6 ? 1 : 2;
  static constexpr size_t kSmemMax = CW >= 6 ? kWsSmemMax : 110 * 1024;
};

struct WsPlan {
  int nslots, nload, x1slot0, gbslot0, stages, nz, a1, ngb;
  // a second, distinct update term streams into the slots right after X1's
  // (padded to x1n): the update is one k-loop over kcols = x1n + a2 columns
  int a2, x1n, x2slot0, kcols;
  // stage layout: segment offsets (doubles) and per-consumer-warp offsets
  int stage_words;
  int zoff, xoff, x2off, goff;  // operand segment offsets in a stage (doubles)
  unsigned tx;           // TMA: bytes landing per stage
};

// the three operand tiles of a ws stage as 2-D tensor maps (TMA variant)
struct WsMaps {
  CUtensorMap z, x, x2, g;
};


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WS_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra WS_DONE;\n"
      " bra WS_WAIT;\n"
      "WS_DONE:\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// DMMA without `volatile`: the compiler may interleave independent chains
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
#ifndef RG_WS_NACC
#define RG_WS_NACC 2
#endif
constexpr int kWsNacc = RG_WS_NACC;  // independent update accumulators (chain interleave)

__device__ __forceinline__ void cp16_zfill(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// one operand tile of a stage: box {rows, columns} at row row0
__device__ __forceinline__ void tma_tile(double* dst, const CUtensorMap* m, int row0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(m), "r"(row0), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <int CW, int NT, int MT, int KSR = 0, bool TMA = false, int KSM = kWsKS>
__global__ void __launch_bounds__((WsGeom<CW, TMA>::kThreads), (WsGeom<CW, TMA>::kMinBlocks))
    tall_ws_kernel(TallParams P, WsPlan W, const __grid_constant__ WsMaps maps) {
  using G = WsGeom<CW, TMA>;
  constexpr int kRows = G::kRows, kThreads = G::kThreads;
  constexpr int CS = G::kS;  // column stride of a stage
  constexpr int MTA = MT > 0 ? MT : 1;
  extern __shared__ __align__(128) double ws_smem[];
  double* smem = ws_smem;
  __shared__ __align__(8) uint64_t full[kWsMaxStages], empty[kWsMaxStages];
  __shared__ bool s_last;
  const int p = P.p;
  const int ks1 = (W.kcols + 3) / 4;
  const size_t stage_words = (size_t)W.stage_words;
  double* stage0 = smem;
  double* sf1 = stage0 + (size_t)W.stages * stage_words;  // [ks1][NT][32]
  double* sR = sf1 + (size_t)ks1 * NT * 32;                // [NT*8][NT*8] solve factor
  double* red = stage0;  // [MTA][NT][64], reuses the ring after the main loop
  constexpr int PM8 = NT * 8;
  const bool trsm = KSR == 0 && (P.r1 || P.r2);  // the KSR variants never carry solves

  // (TMA fills every stage word, zeros included)
  if (!TMA)
    for (size_t e = threadIdx.x; e < (size_t)W.stages * stage_words; e += kThreads) stage0[e] = 0.0;
  for (int e = threadIdx.x; e < ks1 * NT * 32; e += kThreads) {
    const int ks = e / (NT * 32), nt = (e / 32) % NT, ln = e % 32;
    const int aa = ks * 4 + (ln & 3), c = nt * 8 + (ln >> 2);
    double v = 0.0;
    if (c < p) {
      if (W.a2) {
        // two distinct terms: alpha_t folded into S_t (as merge12)
        if (aa < P.a1) v = P.alpha1 * P.s1[aa + (int64_t)c * P.a1];
        else if (aa >= W.x1n && aa - W.x1n < P.a2) v = P.alpha2 * P.s2[(aa - W.x1n) + (int64_t)c * P.a2];
      } else if (aa < P.a1) {
        v = P.s1[aa + (int64_t)c * P.a1];
        if (P.merge12) v = P.alpha1 * v + P.alpha2 * P.s2[aa + (int64_t)c * P.a2];
      }
    }
    sf1[e] = v;
  }
  if (trsm) {
    // z R1^-1 [R2^-1] as one solve with R (= R1, or the upper-triangular R2 R1),
    // row-major, reciprocal diagonal (as v6)
    for (int e = threadIdx.x; e < PM8 * PM8; e += kThreads) {
      const int ii = e / PM8, jj = e % PM8;
      double v = ii == jj ? 1.0 : 0.0;
      if (ii < p && jj < p && ii <= jj) {
        if (P.r1 && P.r2) {
          v = 0.0;
          for (int k = ii; k <= jj; ++k) v = fma(P.r2[ii + (int64_t)k * p], P.r1[k + (int64_t)jj * p], v);
        } else {
          const double* r = P.r1 ? P.r1 : P.r2;
          v = r[ii + (int64_t)jj * p];
        }
        if (ii == jj) v = 1.0 / v;
      }
      sR[e] = v;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < W.stages; ++s) {
      mbar_init(&full[s], TMA ? 1u : G::kProd * 32u);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nunits = (P.n + kRows - 1) / kRows;
  const int64_t my_units =
      (int64_t)blockIdx.x < nunits ? (nunits - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const bool gram_basis = MT > 0 && P.gmode == 1;
  const bool gram_self = MT > 0 && P.gmode == 2;
  const int mtiles = P.mtiles;

  double acc[MTA][NT][2];
#pragma unroll
  for (int mt = 0; mt < MTA; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  if (TMA && warp >= CW) {
    // ---------------- producer: one thread, one tensor request per operand
    if (warp == CW && lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int64_t it = 0; it < my_units; ++it) {
        if (it >= W.stages) mbar_wait(&empty[s], ph ^ 1u);
        const int row0 = (int)(((int64_t)blockIdx.x + it * gridDim.x) * kRows);
        double* st = stage0 + s * stage_words;
        mbar_expect_tx(&full[s], W.tx);
        if (W.nz) tma_tile(st + W.zoff, &maps.z, row0, &full[s]);
        if (W.a1) tma_tile(st + W.xoff, &maps.x, row0, &full[s]);
        if (W.a2) tma_tile(st + W.x2off, &maps.x2, row0, &full[s]);
        if (W.ngb) tma_tile(st + W.goff, &maps.g, row0, &full[s]);
        if (++s == W.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp >= CW) {
    // ---------------- producers: lane t copies rows 2q, 2q + 1 (zero-filled
    // past n) of columns jl, jl + kStep, ... of each operand segment; the
    // source pointer and the slot offset advance by constants
    constexpr int kCpc = kRows / 2;                  // 16-byte chunks per column
    constexpr int kStep = G::kProd * 32 / kCpc;      // columns per producer pass
    const int t = (warp - CW) * 32 + lane;
    const int q = t % kCpc, jl = t / kCpc;
    int s = 0;
    unsigned ph = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      if (it >= W.stages) mbar_wait(&empty[s], ph ^ 1u);
      const int64_t row = ((int64_t)blockIdx.x + it * gridDim.x) * kRows + 2 * q;
      const int64_t vr = P.n - row;
      const int bytes = vr >= 2 ? 16 : (vr == 1 ? 8 : 0);
      const int64_t off = bytes ? row : 0;
      const uint32_t dq = smem_u32(stage0 + s * stage_words) + (uint32_t)(2 * q * 8);
      auto segment = [&](const double* base, int64_t ld, int ncols, int slot0) {
        const double* src = base + (int64_t)jl * ld + off;
        uint32_t d = dq + (uint32_t)((slot0 + jl) * G::kS * 8);
#pragma unroll 4
        for (int j = jl; j < ncols; j += kStep) {
          cp16_zfill(d, src, bytes);
          src += kStep * ld;
          d += kStep * G::kS * 8;
        }
      };
      if (W.nz) segment(P.zin, P.ldzin, W.nz, 0);
      if (W.a1) segment(P.x1, P.ldx1, W.a1, W.x1slot0);
      if (W.a2) segment(P.x2, P.ldx2, W.a2, W.x2slot0);
      if (W.ngb) segment(P.gb, P.ldgb, W.ngb, W.gbslot0);
      cp_async_arrive_noinc(&full[s]);
      if (++s == W.stages) {
        s = 0;
        ph ^= 1u;
      }
    }
    cp_async_wait<0>();
  } else {
    // ---------------- consumers: warp owns stage rows rw .. rw + 7; element
    // (stage row r, column c) of an operand segment is at seg[c * CS + r]
    const int mrow = lane >> 2, kq = lane & 3;
    const int rw = warp * 8;
    // (the 9-warp TMA variant and the 7-warp Gram variants carry no update code)
    constexpr bool kUpdCode = !(TMA && CW == 9) && !(CW == 7 && MT > 0);
    const bool upd = kUpdCode && P.a1 > 0;
    const bool wb = upd && (P.gmode != 0 || P.zout || trsm);
    const double alpha = (P.merge12 || W.a2) ? 1.0 : P.alpha1;
    // KSR > 0: the update's S fragments (a1 <= 4*KSR, NT == 1) live in
    // registers -- a fifth of the pass's shared-memory wavefronts
    // (also the three-tile updates without a Gram: 3 x KSR fragments)
    constexpr bool kBreg = KSR > 0 && (NT == 1 || MT == 0);
    constexpr int kKS = kBreg ? KSR : KSM;  // compile-time k-steps: no predicated-off DMMAs past a1
    double bq[kBreg ? KSR : 1][kBreg ? NT : 1];
    if (kBreg) {
#pragma unroll
      for (int ks = 0; ks < (kBreg ? KSR : 1); ++ks)
#pragma unroll
        for (int nt = 0; nt < (kBreg ? NT : 1); ++nt)
          bq[ks][nt] = ks < ks1 ? sf1[(ks * NT + nt) * 32 + lane] : 0.0;
    }
    int s = 0;
    unsigned ph = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      mbar_wait(&full[s], ph);
      double* st = stage0 + s * stage_words;
      const int64_t r0 = ((int64_t)blockIdx.x + it * gridDim.x) * kRows;
      double* zs = st + W.zoff + rw;  // this warp's z rows
      if (upd) {
        double zf[NT][2], m[kWsNacc][NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            zf[nt][v] = W.nz ? zs[(nt * 8 + 2 * kq + v) * CS + mrow] : 0.0;
#pragma unroll
            for (int q = 0; q < kWsNacc; ++q) m[q][nt][v] = 0.0;
          }
        const double* xs = st + W.xoff + rw + kq * CS + mrow;
#pragma unroll
        for (int ks = 0; ks < kKS; ++ks) {
          if (ks < ks1) {
            const double a = xs[ks * 4 * CS];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma_nv(m[ks % kWsNacc][nt][0], m[ks % kWsNacc][nt][1], a,
                      kBreg ? bq[kBreg ? ks : 0][kBreg ? nt : 0] : sf1[(ks * NT + nt) * 32 + lane]);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            double t = m[0][nt][v];
#pragma unroll
            for (int q = 1; q < kWsNacc; ++q) t += m[q][nt][v];
            zf[nt][v] = zf[nt][v] + alpha * t;
          }
        if (wb) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int v = 0; v < 2; ++v) zs[(nt * 8 + 2 * kq + v) * CS + mrow] = zf[nt][v];
          __syncwarp();
        }
      }
      if (trsm) {
        // one lane per row of this warp's 8 rows
        if (lane < 8) {
          double zr[PM8];
#pragma unroll
          for (int c = 0; c < PM8; ++c) zr[c] = zs[c * CS + lane];
          trsm_row<PM8>(zr, sR, p);
#pragma unroll
          for (int c = 0; c < PM8; ++c) zs[c * CS + lane] = zr[c];
        }
        __syncwarp();
      }
      if (P.zout) {
#pragma unroll
        for (int i = 0; i < NT * 2; ++i) {
          const int e = lane + 32 * i, c = e >> 3, r = e & 7;
          const int64_t row = r0 + rw + r;
          if (c < p && row < P.n) P.zout[row + (int64_t)c * P.ldzout] = zs[c * CS + r];
        }
      }
      if (gram_basis || gram_self) {
        double2 bz[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          bz[nt] = *reinterpret_cast<const double2*>(zs + (nt * 8 + mrow) * CS + 2 * kq);
        const double* gs = (gram_basis ? st + W.goff + rw : zs) + mrow * CS + 2 * kq;
        // per chunk of row tiles: all first k-halves, then the second ones
        // (no back-to-back dependent DMMAs); the register-resident-S
        // variant loads its 13 tiles in two chunks to stay within 168
        // registers; so do the three-tile Grams (14 tiles x 3 fragments)
        constexpr int GCH = (KSR > 0 || (NT == 3 && MTA > 7)) ? 7 : MTA;
#pragma unroll
        for (int m0 = 0; m0 < MTA; m0 += GCH) {
          double2 ga[GCH];
#pragma unroll
          for (int j = 0; j < GCH; ++j)
            ga[j] = (m0 + j < MTA && m0 + j < mtiles) ? *reinterpret_cast<const double2*>(gs + (m0 + j) * 8 * CS)
                                                       : make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < GCH; ++j)
            if (m0 + j < MTA && m0 + j < mtiles)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
                dmma_nv(acc[m0 + j < MTA ? m0 + j : 0][nt][0], acc[m0 + j < MTA ? m0 + j : 0][nt][1], ga[j].x,
                        bz[nt].x);
#pragma unroll
          for (int j = 0; j < GCH; ++j)
            if (m0 + j < MTA && m0 + j < mtiles)
#pragma unroll
              for (int nt = 0; nt < NT; ++nt)
                dmma_nv(acc[m0 + j < MTA ? m0 + j : 0][nt][0], acc[m0 + j < MTA ? m0 + j : 0][nt][1], ga[j].y,
                        bz[nt].y);
        }
      }
      // generic-proxy writes into the stage (z write-back, solves) must be
      // ordered before the next tensor request overwrites it
      if (TMA && (wb || trsm)) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == W.stages) {
        s = 0;
        ph ^= 1u;
      }
    }
  }

  // ---------------- epilogue: deterministic reductions (consumer-warp order)
  __syncthreads();
  if (gram_basis || gram_self) {
    for (int ww = 0; ww < CW; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTA; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int idx = ((mt * NT + nt) * 32 + lane) * 2 + v;
                red[idx] = (ww == 0) ? acc[mt][nt][v] : red[idx] + acc[mt][nt][v];
              }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kThreads) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[(int64_t)blockIdx.x * ne + e] = red[((mt * NT + nt) * 32 + ln) * 2 + v];
    }
  }
  if (P.gmode == 0) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(P.counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ne = P.gc * p;
  for (int e = threadIdx.x; e < ne; e += kThreads) {
    double sum = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * ne + e);
    P.gout[e] = sum;
  }
  // row-partitioned: finish the sum over the ranks here (rg_common.cuh)
  if (P.comm.world > 1) peer_allreduce(P.comm, P.gout, ne, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

#ifndef RG_WS_TMA
#define RG_WS_TMA 1
#endif
// consumer warps of the three-tile (p = 17..24) update passes: 7 (+ the
// producer: 8 warps, 255 registers, S fragments in registers) or 8 (+1: 168
// registers, S fragments read from shared memory)
#ifndef RG_WS_NT3_UPD_CW
#define RG_WS_NT3_UPD_CW 7
#endif
// fewest streamed columns a TMA ws pass takes (narrower passes run on v6)
#ifndef RG_WS_MIN_LOAD_TMA
#define RG_WS_MIN_LOAD_TMA 32
#endif
// L2 sector promotion of the tensor requests: a 72-row box row (576 B) starts
// at 64 B mod 128, so 256-byte promotion fetched ~8% more than the block
// (ncu: 15.66 vs 14.50 GB for P2)
#ifndef RG_WS_TMA_PROMO
#define RG_WS_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_NONE
#endif

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*TensorMapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);
static TensorMapEncodeFn tensor_map_encoder() {
  static TensorMapEncodeFn fn = []() -> TensorMapEncodeFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<TensorMapEncodeFn>(f);
  }();
  return fn;
}

// an n x ncols column-major block as a 2-D tensor {n, ncols} (row stride
// 8 bytes, column stride ld*8), box {rows, bc}: a stage tile lands as
// [column][rows]
static bool encode_stage_map(CUtensorMap* m, const double* base, int64_t ld, int64_t n, int ncols, int bc,
                             int rows) {
  TensorMapEncodeFn enc = tensor_map_encoder();
  if (!enc || bc > 256 || rows > 256 || ncols < 1 || n < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)ncols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)rows, (cuuint32_t)bc};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, RG_WS_TMA_PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the stage plan, or false when the pass is not a ws shape (triangular
// solves, norms, two distinct terms, too many columns).  TMA: also encode the
// tensor maps -- false when an operand cannot be described (the caller then
// plans the cp.async variant).
template <int CW, bool TMA>
static bool ws_plan(const TallParams& P, int NT, int MT, WsPlan& W, size_t& smem, WsMaps* maps) {
  using G = WsGeom<CW, TMA>;
  if (P.gmode == 3) return false;
  const bool two = P.a2 > 0 && !P.merge12;  // a second, distinct term
  if (two && P.a1 == 0) return false;
  const int x1n = (P.a1 + 7) / 8 * 8;
  const int x2n = two ? (P.a2 + 7) / 8 * 8 : 0;
  W.a2 = two ? P.a2 : 0;
  W.x1n = x1n;
  W.kcols = two ? x1n + P.a2 : P.a1;
  if (W.kcols > 4 * kWsKS) return false;
  if ((P.gmode == 1 || P.gmode == 2) && P.mtiles > MT) return false;
  if (P.gmode == 2 && P.a1 == 0 && !P.zin) return false;
  const int PM8 = NT * 8;
  const bool alias = P.gmode == 1 && P.a1 > 0 && P.gb == P.x1 && P.ldgb == P.ldx1 && P.gc <= P.a1;
  const int gbn = (P.gmode == 1 && !alias) ? (P.gc + 7) / 8 * 8 : 0;
  // no Zin to stage: z is written back over the warp's own rows of the first
  // update operand (read completely by then) -- one slot group fewer per stage
  // (the p = 20 recycle passes: 3 stages instead of 2)
  const int zslots = (!P.zin && P.a1 > 0 && x1n >= PM8 && !alias) ? 0 : PM8;
  W.x1slot0 = zslots;
  W.x2slot0 = zslots + x1n;
  W.gbslot0 = alias ? zslots : zslots + x1n + x2n;
  W.nslots = zslots + x1n + x2n + gbn;
  W.nz = P.zin ? P.p : 0;
  W.a1 = P.a1;
  W.ngb = (P.gmode == 1 && !alias) ? P.gc : 0;
  W.nload = W.nz + P.a1 + W.a2 + W.ngb;
  if (W.nload == 0) return false;
  // below ~64 streamed columns the fixed per-stage cost (mbarrier round
  // trips, 64-row stages) loses to v6 (profiles/ws_study_r01.txt)
  if (W.nload < (TMA ? RG_WS_MIN_LOAD_TMA : 64)) return false;
  W.stage_words = W.nslots * G::kS;
  W.zoff = 0;
  W.xoff = W.x1slot0 * G::kS;
  W.x2off = W.x2slot0 * G::kS;
  W.goff = W.gbslot0 * G::kS;
  W.tx = 0;
  if (TMA) {
    if (W.nz && !encode_stage_map(&maps->z, P.zin, P.ldzin, P.n, P.p, PM8, G::kS)) return false;
    if (W.a1 && !encode_stage_map(&maps->x, P.x1, P.ldx1, P.n, P.a1, x1n, G::kS)) return false;
    if (W.a2 && !encode_stage_map(&maps->x2, P.x2, P.ldx2, P.n, P.a2, x2n, G::kS)) return false;
    if (W.ngb && !encode_stage_map(&maps->g, P.gb, P.ldgb, P.n, P.gc, gbn, G::kS)) return false;
    W.tx = (unsigned)(((W.nz ? PM8 : 0) + (W.a1 ? x1n : 0) + x2n + (W.ngb ? gbn : 0)) * G::kS * sizeof(double));
  }
  const size_t extra = ((size_t)((W.kcols + 3) / 4) * NT * 32 + (size_t)PM8 * PM8) * sizeof(double);
  const size_t per_stage = (size_t)W.stage_words * sizeof(double);
  const size_t red_bytes = (size_t)(MT > 0 ? MT : 1) * NT * 64 * sizeof(double);
  int stages = kWsMaxStages;
  while (stages >= 2 && (size_t)stages * per_stage + extra > G::kSmemMax) --stages;
  if (stages < 2) return false;
  if ((size_t)stages * per_stage < red_bytes) return false;
  // narrow passes (the CholQR solves: 8 columns, 4.6 KB stages) cannot keep
  // enough bytes in flight per SM through a ring of whole stages -- v3 / v6
  // serve them (1.15-1.2 ms vs 0.33-0.39 ms per cfg4 pass when forced here)
  if ((size_t)stages * per_stage < (size_t)96 * 1024) return false;
  W.stages = stages;
  smem = (size_t)stages * per_stage + extra;
  return true;
}

template <int CW, int NT, int MT, int KSR, bool TMA, int KSM = kWsKS>
static cudaError_t launch_ws(const TallParams& P, const WsPlan& W, const WsMaps& maps, size_t smem,
                             cudaStream_t st) {
  using G = WsGeom<CW, TMA>;
  auto k = tall_ws_kernel<CW, NT, MT, KSR, TMA, KSM>;
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmemMax);
    per_sm = G::kMinBlocks;
  }
  const int64_t nunits = (P.n + G::kRows - 1) / G::kRows;
  int64_t g = (int64_t)sm_count() * per_sm;
  if (nunits < g) g = nunits;
  if (g < 1) g = 1;
  k<<<(unsigned)g, G::kThreads, smem, st>>>(P, W, maps);
  return cudaGetLastError();
}

template <int CW, bool TMA>
static void launch_ws_shape(const TallParams& P, const WsPlan& W, const WsMaps& maps, size_t smem, int NT, int MT,
                            cudaStream_t st, cudaError_t& e) {
#define RG_WS_MT(NTv)                                                              \
  switch (MT) {                                                                    \
    case 0: e = launch_ws<CW, NTv, 0, 0, TMA>(P, W, maps, smem, st); break;        \
    case 2: e = launch_ws<CW, NTv, 2, 0, TMA>(P, W, maps, smem, st); break;        \
    case 6: e = launch_ws<CW, NTv, 6, 0, TMA>(P, W, maps, smem, st); break;        \
    case 13: e = launch_ws<CW, NTv, 13, 0, TMA>(P, W, maps, smem, st); break;      \
    default: e = launch_ws<CW, NTv, 16, 0, TMA>(P, W, maps, smem, st); break;      \
  }
  const int ks1 = (W.kcols + 3) / 4;
  bool done = false;
  if (NT == 3) {
    // p = 17..24 (the k = 20 recycle passes), TMA only: pure Grams of a
    // block against up to 128 basis columns (the cross Grams [C W]^T U), and
    // updates without a Gram or solve (C_new = [C W] Q, U_new = [U W_m] T')
    e = cudaErrorInvalidConfiguration;  // try_ws screens other shapes out
    if constexpr (TMA && CW == 7) {
      if (P.a1 == 0 && MT > 0) {
        switch (MT) {
          case 3: e = launch_ws<CW, 3, 3, 0, TMA>(P, W, maps, smem, st); break;
          case 14: e = launch_ws<CW, 3, 14, 0, TMA>(P, W, maps, smem, st); break;
          default: e = launch_ws<CW, 3, 16, 0, TMA>(P, W, maps, smem, st); break;
        }
      }
    }
    if constexpr (TMA && CW == RG_WS_NT3_UPD_CW) {
      if (P.a1 > 0 && MT == 0) {
        // 7 warps: S fragments in registers, exact k-steps for the recycle shapes:
        // [C W] Q (108 -> 27), [U W_m] T' (24 + 80 -> 26), first cycle W Q (88 -> 22), W_m T' (80 -> 20);
        // 8 warps: S fragments from shared memory, k-steps rounded up to 4
        if constexpr (CW != 7) {
          switch ((ks1 + 3) / 4) {
            case 1: case 2: case 3: case 4: case 5: e = launch_ws<CW, 3, 0, 0, TMA, 20>(P, W, maps, smem, st); break;
            case 6: e = launch_ws<CW, 3, 0, 0, TMA, 24>(P, W, maps, smem, st); break;
            case 7: e = launch_ws<CW, 3, 0, 0, TMA, 28>(P, W, maps, smem, st); break;
            default: e = launch_ws<CW, 3, 0, 0, TMA, 32>(P, W, maps, smem, st); break;
          }
        } else if (ks1 <= 20) e = launch_ws<CW, 3, 0, 20, TMA>(P, W, maps, smem, st);
        else if (ks1 <= 22) e = launch_ws<CW, 3, 0, 22, TMA>(P, W, maps, smem, st);
        else if (ks1 <= 24) e = launch_ws<CW, 3, 0, 24, TMA>(P, W, maps, smem, st);
        else if (ks1 <= 26) e = launch_ws<CW, 3, 0, 26, TMA>(P, W, maps, smem, st);
        else if (ks1 <= 27) e = launch_ws<CW, 3, 0, 27, TMA>(P, W, maps, smem, st);
        else if (ks1 <= 28) e = launch_ws<CW, 3, 0, 28, TMA>(P, W, maps, smem, st);
        else e = launch_ws<CW, 3, 0, 0, TMA, 32>(P, W, maps, smem, st);
      }
    }
    return;
  }
  if constexpr (TMA && CW == 8) {  // (the 9-warp TMA variant serves pure Grams only)
  done = true;
  if (NT == 1 && P.gmode == 1 && P.a1 > 0 && W.a2 == 0 && !P.r1 && !P.r2 && P.mtiles >= 2 && P.mtiles <= 13 &&
      ks1 <= 2 * P.mtiles) {
    // P2 of the joint schedule (update by [C W] + the aliased Gram) at every
    // basis width of a cycle: exact tile counts, S in registers.  With one
    // 13-tile / 26-k-step instantiation the predicated-off DMMAs kept the
    // pass at ~2.3 ms from a = 60 to a = 100 (profiles/cycle_r02_256.json)
    switch (P.mtiles) {
      case 2: e = launch_ws<CW, 1, 2, 4, TMA>(P, W, maps, smem, st); break;
      case 3: e = launch_ws<CW, 1, 3, 6, TMA>(P, W, maps, smem, st); break;
      case 4: e = launch_ws<CW, 1, 4, 8, TMA>(P, W, maps, smem, st); break;
      case 5: e = launch_ws<CW, 1, 5, 10, TMA>(P, W, maps, smem, st); break;
      case 6: e = launch_ws<CW, 1, 6, 12, TMA>(P, W, maps, smem, st); break;
      case 7: e = launch_ws<CW, 1, 7, 14, TMA>(P, W, maps, smem, st); break;
      case 8: e = launch_ws<CW, 1, 8, 16, TMA>(P, W, maps, smem, st); break;
      case 9: e = launch_ws<CW, 1, 9, 18, TMA>(P, W, maps, smem, st); break;
      case 10: e = launch_ws<CW, 1, 10, 20, TMA>(P, W, maps, smem, st); break;
      case 11: e = launch_ws<CW, 1, 11, 22, TMA>(P, W, maps, smem, st); break;
      case 12: e = launch_ws<CW, 1, 12, 24, TMA>(P, W, maps, smem, st); break;
      default: e = launch_ws<CW, 1, 13, 26, TMA>(P, W, maps, smem, st); break;
    }
  } else if (NT == 1 && P.a1 > 0 && MT <= 2) {
    // update passes (P3: merged update + self-Gram + store; R -= W (H Y)):
    // k-steps rounded up to a multiple of 4
#define RG_WS_KS(MTv)                                                                   \
  switch ((ks1 + 3) / 4) {                                                              \
    case 1: case 2: e = launch_ws<CW, 1, MTv, 0, TMA, 8>(P, W, maps, smem, st); break;  \
    case 3: e = launch_ws<CW, 1, MTv, 0, TMA, 12>(P, W, maps, smem, st); break;         \
    case 4: e = launch_ws<CW, 1, MTv, 0, TMA, 16>(P, W, maps, smem, st); break;         \
    case 5: e = launch_ws<CW, 1, MTv, 0, TMA, 20>(P, W, maps, smem, st); break;         \
    case 6: e = launch_ws<CW, 1, MTv, 0, TMA, 24>(P, W, maps, smem, st); break;         \
    case 7: e = launch_ws<CW, 1, MTv, 0, TMA, 28>(P, W, maps, smem, st); break;         \
    default: e = launch_ws<CW, 1, MTv, 0, TMA, 32>(P, W, maps, smem, st); break;        \
  }
    if (MT == 0) {
      RG_WS_KS(0)
    } else {
      RG_WS_KS(2)
    }
#undef RG_WS_KS
  } else {
    done = false;
  }
  }
  if (done) {
  } else if (!TMA && NT == 1 && CW >= 8 && P.a1 > 0 && W.a2 == 0 && P.a1 <= 104 && MT == 13 && !P.r1 && !P.r2) {
    // cp.async fallback of the P2 shape: S in registers (3.08 -> 3.00-3.05 ms
    // at cfg4; the P3 shape was slower with it, profiles/ws_study_r01.txt)
    e = launch_ws<CW, 1, 13, 26, TMA>(P, W, maps, smem, st);
  } else if (NT == 1) {
    RG_WS_MT(1)
  } else {
    RG_WS_MT(2)
  }
#undef RG_WS_MT
}

static bool try_ws_shape(const TallParams& P, int NT, int MT, cudaStream_t st, cudaError_t& e) {
  WsPlan W;
  WsMaps maps;
  memset(&maps, 0, sizeof(maps));
  size_t smem = 0;
  // consumer warps of the TMA variant, measured per pass type at cfg4
  // (profiles/tma_r02.txt): 8 (2 per SMSP, 72-row boxes overlapping by 8
  // rows) for passes with an update -- P2 2.29 ms vs 2.70 with 9 warps and
  // 2.40 with cp.async; 9 (dense 72-row boxes) for a pure Gram -- P1 2.01 ms
  // vs 2.13 with 8
  if (RG_WS_TMA && NT == 3 && P.a1 > 0 && ws_plan<RG_WS_NT3_UPD_CW, true>(P, NT, MT, W, smem, &maps)) {
    launch_ws_shape<RG_WS_NT3_UPD_CW, true>(P, W, maps, smem, NT, MT, st, e);
    return true;
  }
  if (RG_WS_TMA && NT == 3 && P.a1 == 0 && ws_plan<7, true>(P, NT, MT, W, smem, &maps)) {
    // three-tile Grams hold 14 x 3 DMMA fragments per lane: 7 consumer warps +
    // the producer (8 warps, 255 registers) instead of 9 + 1 (168, spills)
    launch_ws_shape<7, true>(P, W, maps, smem, NT, MT, st, e);
    return true;
  }
  if (RG_WS_TMA && NT < 3 && P.a1 == 0 && ws_plan<9, true>(P, NT, MT, W, smem, &maps)) {
    launch_ws_shape<9, true>(P, W, maps, smem, NT, MT, st, e);
    return true;
  }
  if (RG_WS_TMA && P.a1 > 0 && ws_plan<8, true>(P, NT, MT, W, smem, &maps)) {
    launch_ws_shape<8, true>(P, W, maps, smem, NT, MT, st, e);
    return true;
  }
  if (NT == 3) return false;  // three-tile blocks: TMA variants only (else v6)
  if (!ws_plan<8, false>(P, NT, MT, W, smem, nullptr)) return false;
  launch_ws_shape<8, false>(P, W, maps, smem, NT, MT, st, e);
  return true;
}

// returns false when the pass is not a ws shape (caller falls back to v6)
static bool try_ws(const TallParams& P, int PM, cudaStream_t st, cudaError_t& e) {
  if (PM > 24) return false;
  const int NT = PM > 16 ? 3 : (PM > 8 ? 2 : 1);
  const int mt = (P.gmode == 1 || P.gmode == 2) ? P.mtiles : 0;
  if (NT == 3) {
    // pure Grams (gram modes 1/2, no update) or plain updates (no Gram); no solves
    if (P.r1 || P.r2 || P.gmode == 3) return false;
    if (!((P.a1 == 0 && mt > 0) || (P.a1 > 0 && mt == 0))) return false;
    return try_ws_shape(P, NT, mt == 0 ? 0 : (mt <= 3 ? 3 : (mt <= 14 ? 14 : 16)), st, e);
  }
  const int MT = mt == 0 ? 0 : (mt <= 2 ? 2 : (mt <= 6 ? 6 : (mt <= 13 ? 13 : 16)));
  return try_ws_shape(P, NT, MT, st, e);
}

// Passes without a basis Gram (update / store / self-Gram) run 4-warp CTAs
// with an 8-deep slab ring; passes streaming a Gram basis keep 8 warps x 4
// (profiles/v6_study_r01.txt: 2.97 -> 2.68 ms for the final CGS2 pass).
#define RG_V6_CASE(PMv)                                                                   \
  case PMv:                                                                               \
    if (wide_ring) {                                                                      \
      switch (mt5) {                                                                      \
        case 0: e = launch_v6<PMv, 0, 4, 8>(P, bound, st); break;                         \
        default: e = launch_v6<PMv, 2, 4, 8>(P, bound, st); break;                        \
      }                                                                                   \
    } else {                                                                              \
      switch (mt5) {                                                                      \
        case 0: e = launch_v6<PMv, 0>(P, bound, st); break;                               \
        case 2: e = launch_v6<PMv, 2>(P, bound, st); break;                               \
        case 6: e = launch_v6<PMv, 6>(P, bound, st); break;                               \
        case 12: e = launch_v6<PMv, 12>(P, bound, st); break;                             \
        case 13: e = launch_v6<PMv, 13>(P, bound, st); break;                             \
        default: e = launch_v6<PMv, 16>(P, bound, st); break;                             \
      }                                                                                   \
    }                                                                                     \
    break;

template <int PM, int MTMAX>
static cudaError_t launch_v3(const TallParams& P, int64_t max_grid, cudaStream_t st) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  auto k = tall_v3_kernel<PM, MTMAX>;
  constexpr int kWarpWords = PM8 * kSlabStride + 2 * 8 * kSlabStride;
  const size_t smem = ((size_t)(P.a1 + P.a2) * PM + 2 * PM * PM + (size_t)kV3Warps * kWarpWords +
                       (size_t)std::max(MTMAX * NT * 64, kV3Warps * PM)) * sizeof(double);
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, kV3Threads, 64 * 1024);
    per_sm = v < 1 ? 1 : v;
  }
  const int64_t nunits = (P.n + 31) / 32;
  int64_t g = (int64_t)sm_count() * per_sm;
  if (g > max_grid) g = max_grid;
  const int64_t need = (nunits + kV3Warps - 1) / kV3Warps;
  if (need < g) g = need;
  if (g < 1) g = 1;
  k<<<(unsigned)g, kV3Threads, smem, st>>>(P);
  return cudaGetLastError();
}

#define RG_V3_CASE(PMv)                                                                   \
  case PMv:                                                                               \
    switch (mtmax) {                                                                      \
      case 2: e = launch_v3<PMv, 2>(P, tall_grid_bound(), st); break;                     \
      case 6: e = launch_v3<PMv, 6>(P, bound, st); break;                                 \
      case 12: e = launch_v3<PMv, 12>(P, bound, st); break;                               \
      default: e = launch_v3<PMv, 16>(P, bound, st); break;                               \
    }                                                                                     \
    break;

template <int PM, int MTMAX>
static cudaError_t launch_v5(const TallParams& P, int64_t max_grid, cudaStream_t st) {
  constexpr int PM8 = PM < 8 ? 8 : PM;
  constexpr int NT = PM8 / 8;
  constexpr int kWarpWords = kRing5 * 8 * kSS5 + PM8 * kSS5;
  auto k = tall_v5_kernel<PM, MTMAX>;
  const size_t smem = ((size_t)(P.a1 + P.a2) * PM + 2 * PM * PM + 2 + (size_t)kV5Warps * kWarpWords +
                       (size_t)std::max(MTMAX * NT * 64, kV5Warps * PM)) * sizeof(double);
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int v = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, kV5Threads, smem);
    per_sm = v < 1 ? 1 : v;
  }
  const int64_t nunits = (P.n + 31) / 32;
  int64_t g = (int64_t)sm_count() * per_sm;
  if (g > max_grid) g = max_grid;
  const int64_t need = (nunits + kV5Warps - 1) / kV5Warps;
  if (need < g) g = need;
  if (g < 1) g = 1;
  k<<<(unsigned)g, kV5Threads, smem, st>>>(P);
  return cudaGetLastError();
}

#define RG_V5_CASE(PMv)                                                                   \
  case PMv:                                                                               \
    switch (mt5) {                                                                      \
      case 0: e = launch_v5<PMv, 0>(P, bound, st); break;                                 \
      case 2: e = launch_v5<PMv, 2>(P, bound, st); break;                                 \
      case 6: e = launch_v5<PMv, 6>(P, bound, st); break;                                 \
      case 12: e = launch_v5<PMv, 12>(P, bound, st); break;                               \
      default: e = launch_v5<PMv, 16>(P, bound, st); break;                               \
    }                                                                                     \
    break;

// ============================================================================
// nr: narrow passes without update terms -- the CholQR2 solves (K_f: solve +
// self-Gram, K_g: two solves + store), in-place scalings and column norms of
// one n x p block (p <= 16).  Such a pass streams 8..16 columns only: through
// whole 72-row ws stages (4.6 KB) or lane-per-row loads (v3) an SM cannot
// keep enough bytes in flight (K_f ran at 0.52 of the copy peak on v3).
// Here one producer thread keeps a ring of 256-row x PM-column boxes (16 KB
// at p = 8, the tallest box a tensor map takes) full per CTA, two CTAs per
// SM; the 8 consumer warps take 32 rows each, lane = row, pull their row
// into registers and release the stage at once, so the ring never waits on
// the solve, the store or the DMMA Gram.  Rows past n and columns past p
// arrive as zeros (out-of-bounds fill).
// ============================================================================

#ifndef RG_TALL_NR
#define RG_TALL_NR 1
#endif
constexpr int kNrRows = 256;
constexpr int kNrWarps = 8;
constexpr int kNrThreads = (kNrWarps + 1) * 32;
constexpr int kNrMaxStages = 8;
#ifndef RG_NR_CTAS
#define RG_NR_CTAS 2
#endif
constexpr int kNrCtas = RG_NR_CTAS;  // CTAs per SM
constexpr size_t kNrSmemMax = (kNrCtas == 2 ? 110 : 72) * 1024;

template <int PM>
__global__ void __launch_bounds__(kNrThreads, kNrCtas)
    tall_nr_kernel(TallParams P, int stages, const __grid_constant__ CUtensorMap zmap) {
  constexpr int NT = PM / 8;
  constexpr int kStageWords = PM * kNrRows;
  extern __shared__ __align__(128) double nr_smem[];
  __shared__ __align__(8) uint64_t full[kNrMaxStages], empty[kNrMaxStages];
  __shared__ bool s_last;
  const int p = P.p;
  double* stage0 = nr_smem;                                   // [stages][PM][256]
  double* sR1 = stage0 + (size_t)stages * kStageWords;        // PM x PM row-major, reciprocal diagonal
  double* sR2 = sR1 + PM * PM;
  double* red = sR2 + PM * PM;                                // epilogue: max(NT*NT*64, kNrWarps*PM)
  double* ztb = red + (NT * NT * 64 > kNrWarps * PM ? NT * NT * 64 : kNrWarps * PM);  // per warp [PM][36]

  for (int e = threadIdx.x; e < PM * PM; e += kNrThreads) {
    const int ii = e / PM, jj = e % PM;
    const double id = ii == jj ? 1.0 : 0.0;
    sR1[e] = (P.r1 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r1[ii + (int64_t)jj * p] : P.r1[ii + (int64_t)jj * p]) : id;
    sR2[e] = (P.r2 && ii < p && jj < p) ? (ii == jj ? 1.0 / P.r2[ii + (int64_t)jj * p] : P.r2[ii + (int64_t)jj * p]) : id;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1u);
      mbar_init(&empty[s], kNrWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  const int64_t nunits = (P.n + kNrRows - 1) / kNrRows;
  const int64_t my_units =
      (int64_t)blockIdx.x < nunits ? (nunits - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const bool gram_self = P.gmode == 2;

  double acc[NT][NT][2], acb[NT][NT][2];
#pragma unroll
  for (int mt = 0; mt < NT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acb[mt][nt][0] = acb[mt][nt][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  if (warp == kNrWarps) {
    // ---------------- producer: one thread, one tensor request per stage
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int64_t it = 0; it < my_units; ++it) {
        if (it >= stages) mbar_wait(&empty[s], ph ^ 1u);
        const int row0 = (int)(((int64_t)blockIdx.x + it * gridDim.x) * kNrRows);
        mbar_expect_tx(&full[s], (unsigned)(kStageWords * sizeof(double)));
        tma_tile(stage0 + (size_t)s * kStageWords, &zmap, row0, &full[s]);
        if (++s == stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    // ---------------- consumers: lane = row (warp w: stage rows 32w .. 32w + 31)
    double* zt = ztb + warp * PM * kSlabStride;
    int s = 0;
    unsigned ph = 0;
    for (int64_t it = 0; it < my_units; ++it) {
      mbar_wait(&full[s], ph);
      const double* st = stage0 + (size_t)s * kStageWords + warp * 32 + lane;
      double z[PM];
#pragma unroll
      for (int c = 0; c < PM; ++c) z[c] = st[c * kNrRows];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // the row is in registers: release the stage
      if (++s == stages) {
        s = 0;
        ph ^= 1u;
      }
      const int64_t i = ((int64_t)blockIdx.x + it * gridDim.x) * kNrRows + warp * 32 + lane;
      const bool valid = i < P.n;
      if (P.r1) trsm_row<PM>(z, sR1, p);
      if (P.r2) trsm_row<PM>(z, sR2, p);
      if (!valid) {
#pragma unroll
        for (int c = 0; c < PM; ++c) z[c] = 0.0;
      }
      if (P.zout && valid) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) P.zout[i + (int64_t)c * P.ldzout] = z[c];
      }
      if (P.gmode == 3) {
#pragma unroll
        for (int c = 0; c < PM; ++c) sq[c] = fma(z[c], z[c], sq[c]);
      }
      if (gram_self) {
        // DMMA Gram over these 32 rows (8 k-steps), fragments through the
        // warp's padded tile
#pragma unroll
        for (int c = 0; c < PM; ++c) zt[c * kSlabStride + lane] = z[c];
        __syncwarp();
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          double f[NT];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) f[nt] = zt[(nt * 8 + mrow) * kSlabStride + ks * 4 + kq];
#pragma unroll
          for (int mt = 0; mt < NT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              // two accumulator chains (even / odd k-steps), summed at the end
              if (ks & 1) dmma_nv(acb[mt][nt][0], acb[mt][nt][1], f[mt], f[nt]);
              else dmma_nv(acc[mt][nt][0], acc[mt][nt][1], f[mt], f[nt]);
            }
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int mt = 0; mt < NT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        acc[mt][nt][0] += acb[mt][nt][0];
        acc[mt][nt][1] += acb[mt][nt][1];
      }
  }

  // ---------------- epilogue: deterministic reductions (as v3)
  __syncthreads();
  if (gram_self) {
    for (int ww = 0; ww < kNrWarps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < NT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int idx = ((mt * NT + nt) * 32 + lane) * 2 + v;
              red[idx] = (ww == 0) ? acc[mt][nt][v] : red[idx] + acc[mt][nt][v];
            }
      }
      __syncthreads();
    }
    const int ne = p * p;
    for (int e = threadIdx.x; e < ne; e += kNrThreads) {
      const int gg = e % p, c = e / p;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[(int64_t)blockIdx.x * ne + e] = red[((mt * NT + nt) * 32 + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
    if (warp < kNrWarps) {
#pragma unroll
      for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
      if (lane == 0)
#pragma unroll
        for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += kNrThreads) {
      double sum = 0.0;
      for (int ww = 0; ww < kNrWarps; ++ww) sum += red[ww * PM + c];
      P.part[(int64_t)blockIdx.x * p + c] = sum;
    }
  }
  if (P.gmode == 0) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(P.counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ne = (P.gmode == 3) ? p : p * p;
  for (int e = threadIdx.x; e < ne; e += kNrThreads) {
    double sum = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * ne + e);
    P.gout[e] = sum;
  }
  // row-partitioned: finish the sum over the ranks here (rg_common.cuh)
  if (P.comm.world > 1) peer_allreduce(P.comm, P.gout, ne, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

// false when the pass is not an nr shape or the tensor map cannot be encoded
template <int PM>
static bool try_nr(const TallParams& P, cudaStream_t st, cudaError_t& e) {
  constexpr int NT = PM / 8;
  CUtensorMap zmap;
  memset(&zmap, 0, sizeof(zmap));
  if (!encode_stage_map(&zmap, P.zin, P.ldzin, P.n, P.p, PM, kNrRows)) return false;
  const size_t extra = ((size_t)2 * PM * PM + (size_t)std::max(NT * NT * 64, kNrWarps * PM) +
                        (P.gmode == 2 ? (size_t)kNrWarps * PM * kSlabStride : 0)) * sizeof(double);
  const size_t per_stage = (size_t)PM * kNrRows * sizeof(double);
  int stages = kNrMaxStages;
  while (stages >= 2 && (size_t)stages * per_stage + extra > kNrSmemMax) --stages;
  if (stages < 2) return false;
  auto k = tall_nr_kernel<PM>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNrSmemMax);
    attr = true;
  }
  const int64_t nunits = (P.n + kNrRows - 1) / kNrRows;
  int64_t g = (int64_t)sm_count() * kNrCtas;
  if (nunits < g) g = nunits;
  if (g < 1) g = 1;
  k<<<(unsigned)g, kNrThreads, (size_t)stages * per_stage + extra, st>>>(P, stages, zmap);
  e = cudaGetLastError();
  return true;
}

static bool aligned16(const void* p, int64_t ld) {
  return p == nullptr || (((uintptr_t)p & 15u) == 0 && (ld & 1) == 0);
}

// upper bound on the grid of any rg_tall launch (workspace sizing): the
// narrow v3 pass runs up to 3 CTAs per SM, everything else at most 2
static int64_t tall_grid_bound() { return (int64_t)sm_count() * 4; }
static int64_t tall_grid_bound2() { return (int64_t)sm_count() * 2; }


}  // namespace rg

extern "C" int64_t rg_tall_workspace_bytes(int64_t n, int32_t p, int32_t a1, int32_t a2,
                                           int32_t gram_mode, int32_t gc) {
  (void)n; (void)a1; (void)a2;
  using namespace rg;
  int64_t ne = 0;
  if (gram_mode == 1) ne = (int64_t)gc * p;
  if (gram_mode == 2) ne = (int64_t)p * p;
  if (gram_mode == 3) ne = p;
  return 256 + tall_grid_bound() * ne * (int64_t)sizeof(double);
}

extern "C" int rg_tall_f64(int64_t n, int32_t p, const double* d_zin, int64_t ldzin,
                           double* d_zout, int64_t ldzout, const double* d_x1, int64_t ldx1,
                           int32_t a1, const double* d_s1, double alpha1, const double* d_x2,
                           int64_t ldx2, int32_t a2, const double* d_s2, double alpha2,
                           const double* d_r1, const double* d_r2, int32_t gram_mode,
                           const double* d_gb, int64_t ldgb, int32_t gc, double* d_gout,
                           void* d_work, int64_t work_bytes, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0, "rg_tall_f64: n=%lld < 0", (long long)n);
  RG_REQUIRE(p >= 1 && p <= 32, "rg_tall_f64: block width p=%d outside [1, 32]", p);
  // p = 17..24: a pure basis Gram takes up to 128 columns (ws, TMA), else 32
  const bool wide_pure_gram = p <= 24 && gram_mode == 1 && a1 == 0 && a2 == 0 && !d_r1 && !d_r2 && !d_zout;
  RG_REQUIRE(p <= 16 || gram_mode == 0 || gram_mode == 3 || gc <= (p <= 24 ? 32 : 16) ||
                 (wide_pure_gram && gc <= 128),
             "rg_tall_f64: Gram basis width gc=%d too wide for p=%d (32 for p <= 24, 128 for a pure Gram, 16 "
             "above)", gc, p);
  RG_REQUIRE(a1 >= 0 && a2 >= 0 && a1 + a2 <= 512, "rg_tall_f64: term widths %d, %d", a1, a2);
  RG_REQUIRE(!d_zin || ldzin >= n, "rg_tall_f64: ldzin < n");
  RG_REQUIRE(!d_zout || ldzout >= n, "rg_tall_f64: ldzout < n");
  RG_REQUIRE(a1 == 0 || (d_x1 && d_s1 && ldx1 >= n), "rg_tall_f64: bad term 1");
  RG_REQUIRE(a2 == 0 || (d_x2 && d_s2 && ldx2 >= n), "rg_tall_f64: bad term 2");
  RG_REQUIRE(gram_mode >= 0 && gram_mode <= 3, "rg_tall_f64: gram_mode %d", gram_mode);
  RG_REQUIRE(gram_mode != 1 || (d_gb && gc >= 1 && gc <= 128 && ldgb >= n),
             "rg_tall_f64: Gram basis must be n x gc with 1 <= gc <= 128 (gc=%d)", gc);
  RG_REQUIRE(gram_mode != 2 || gc == p, "rg_tall_f64: self Gram needs gc == p");
  RG_REQUIRE(gram_mode == 0 || d_gout, "rg_tall_f64: null Gram output");
  if (gram_mode == 3) gc = 1;
  const int64_t need = rg_tall_workspace_bytes(n, p, a1, a2, gram_mode, gc);
  RG_REQUIRE(gram_mode == 0 || (d_work && work_bytes >= need),
             "rg_tall_f64: workspace %lld bytes < %lld", (long long)work_bytes, (long long)need);

  TallParams P;
  P.n = n; P.p = p;
  P.zin = d_zin; P.ldzin = ldzin; P.zout = d_zout; P.ldzout = ldzout;
  P.x1 = d_x1; P.ldx1 = ldx1; P.a1 = a1; P.s1 = d_s1; P.alpha1 = alpha1;
  P.x2 = d_x2; P.ldx2 = ldx2; P.a2 = a2; P.s2 = d_s2; P.alpha2 = alpha2;
  P.r1 = d_r1; P.r2 = d_r2;
  P.gmode = gram_mode; P.gb = d_gb; P.ldgb = ldgb; P.gc = gc; P.gout = d_gout;
  P.mtiles = (gram_mode == 1 || gram_mode == 2) ? (gc + 7) / 8 : 0;
  P.counter = (unsigned int*)d_work;
  P.part = d_work ? (double*)((char*)d_work + 256) : nullptr;
  P.ntiles = (n + kTallThreads - 1) / kTallThreads;
  P.merge12 = 0;
  if (gram_mode == 0 && P.ntiles == 0) return RG_OK;
  P.comm = peer_comm_next(gram_mode != 0);
  ProfScope prof((cudaStream_t)stream);
  auto launched = [&]() {
    // algorithmic bytes: every streamed operand column once (a Gram basis
    // aliasing an update operand, and two terms over the same X, once)
    const bool same_x = a1 > 0 && a2 > 0 && d_x1 == d_x2 && a1 == a2;
    const bool aliased = gram_mode == 1 && ((d_gb == d_x1 && gc <= a1) || (d_gb == d_x2 && gc <= a2));
    const int64_t cols = (d_zin ? p : 0) + a1 + (same_x ? 0 : a2) + (gram_mode == 1 && !aliased ? gc : 0) +
                         (d_zout ? p : 0);
    const double contr = a1 + (same_x ? 0 : a2) + ((gram_mode == 1 || gram_mode == 2) ? gc : 0);
    prof.finish(1, 8 * n * cols, 2.0 * n * p * contr, nullptr, 0, 0, 0, 0,
                "rg_tall p=%d in=%d a=%d+%d g%d:%d trsm=%d out=%d", p, d_zin ? 1 : 0, a1, a2, gram_mode,
                gram_mode == 3 ? 1 : gc, (d_r1 ? 1 : 0) + (d_r2 ? 1 : 0), d_zout ? 1 : 0);
    return RG_OK;
  };
  const int PM = pick_pm(p);
  const int mtmax = pick_mtmax(P.mtiles);
  const int64_t bound = tall_grid_bound2();
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  const bool aligned = aligned16(P.zin, P.ldzin) && aligned16(P.x1, P.ldx1) && aligned16(P.x2, P.ldx2) &&
                       (gram_mode != 1 || aligned16(P.gb, P.ldgb));
  if (p > 16) {
    // p = 17..24 without solves: the three-tile TMA ws kernel (pure Grams up to
    // 128 basis columns; updates staging z over the first operand's rows, so
    // 3 stages fit).  The earlier 3-tile attempt with 2 stages of 78 KB and
    // 8-lane solves measured slower (profiles/tma_r02.txt); solves stay on v6.
    if (aligned && PM == 24) {
      P.merge12 = (a1 > 0 && a1 == a2 && d_x1 == d_x2 && ldx1 == ldx2) ? 1 : 0;
      if (try_ws(P, PM, st, e)) {
        if (e != cudaSuccess) {
          set_error("rg_tall_f64: %s", cudaGetErrorString(e));
          return RG_ECUDA;
        }
        return launched();
      }
    }
    RG_REQUIRE(gram_mode != 1 || gc <= (p <= 24 ? 32 : 16),
               "rg_tall_f64: a %d-column Gram basis at p=%d needs the TMA ws path (16-byte aligned operands)",
               gc, p);
    const int ncol_slabs = (P.zin ? (p + 7) / 8 : 0) + (a1 + 7) / 8 + (a2 + 7) / 8 +
                           (gram_mode == 1 ? (gc + 7) / 8 : 0);
    RG_REQUIRE(aligned && ncol_slabs <= kMaxSlabs && (P.a1 + P.a2) <= 128,
               "rg_tall_f64: p=%d > 16 needs 16-byte aligned operands, <= 128 term columns, <= %d slabs", p,
               kMaxSlabs);
    const int mtw = P.mtiles == 0 ? 0 : (P.mtiles <= 2 ? 2 : 4);
    P.merge12 = (a1 > 0 && a1 == a2 && d_x1 == d_x2 && ldx1 == ldx2) ? 1 : 0;
    if (PM == 24)
      e = mtw == 0 ? launch_v6<24, 0>(P, bound, st) : (mtw == 2 ? launch_v6<24, 2>(P, bound, st)
                                                                  : launch_v6<24, 4>(P, bound, st));
    else
      e = mtw == 0 ? launch_v6<32, 0>(P, bound, st) : launch_v6<32, 2>(P, bound, st);
    if (e != cudaSuccess) {
      set_error("rg_tall_f64: %s", cudaGetErrorString(e));
      return RG_ECUDA;
    }
    return launched();
  }
  // dispatch measured per pass type (profiles/ab_tall_r01.txt,
  // profiles/ws_study_r01.txt): the warp-specialised ws kernel for the wide
  // CGS2 passes (>= 64 streamed columns); otherwise v6 for passes with an
  // update term, v5 for a pure basis Gram of <= 96 columns, v3 for the
  // CholQR2 solve passes.  Operands that are not 16-byte aligned (row-offset
  // views) go to v3, whose loads are lane-per-row scalars.
  const int mt5 = (gram_mode == 1 || gram_mode == 2) ? mtmax : 0;
  const int ncol_slabs = (P.zin ? (p + 7) / 8 : 0) + (a1 + 7) / 8 + (a2 + 7) / 8 +
                         (gram_mode == 1 ? (gc + 7) / 8 : 0);
  int which = 3;
  if (aligned) {
    P.merge12 = (a1 > 0 && a1 == a2 && d_x1 == d_x2 && ldx1 == ldx2) ? 1 : 0;
    if (try_ws(P, PM, st, e)) {
      if (e != cudaSuccess) {
        set_error("rg_tall_f64: %s", cudaGetErrorString(e));
        return RG_ECUDA;
      }
      return launched();
    }
    P.merge12 = 0;
#if RG_TALL_NR
    // one block in, no update terms (CholQR2 solves, scalings, norms): the
    // 256-row TMA ring (cfg4: K_f 0.282 -> 0.217 ms, self-Gram 0.228 -> 0.173 ms; profiles/nr_r02.txt)
    // (p = 9..16 measured slower than v3 / v6 there: 32 KB stages, 3 deep)
    if (a1 + a2 == 0 && d_zin && gram_mode != 1 && (gram_mode != 0 || d_zout) && PM <= 8 &&
        try_nr<8>(P, st, e)) {
      if (e != cudaSuccess) {
        set_error("rg_tall_f64: %s", cudaGetErrorString(e));
        return RG_ECUDA;
      }
      return launched();
    }
#endif
    which = 6;
    if (a1 + a2 == 0) {
      if (gram_mode == 1)
        which = P.mtiles > 12 ? 6 : 5;  // v5 spills with more than 96 Gram rows; v6<PM, 13> does not
      else if (d_r1 || d_r2)
        which = 3;  // CholQR2 solve passes: 0.41 vs 0.44 ms on v6 (profiles/ab_tall_r01.txt)
    }
    if (which == 6 && ncol_slabs > kMaxSlabs) which = 3;
  }
  if (which == 6) {
    P.merge12 = (a1 > 0 && a1 == a2 && d_x1 == d_x2 && ldx1 == ldx2) ? 1 : 0;
    const bool wide_ring = gram_mode != 1 && PM <= 8 && P.mtiles <= 2 && !d_r1 && !d_r2 && a1 > 0;
    switch (PM) {
      RG_V6_CASE(1)
      RG_V6_CASE(2)
      RG_V6_CASE(4)
      RG_V6_CASE(8)
      RG_V6_CASE(16)
    }
  } else if (which == 3) {
    switch (PM) {
      RG_V3_CASE(1)
      RG_V3_CASE(2)
      RG_V3_CASE(4)
      RG_V3_CASE(8)
      RG_V3_CASE(16)
    }
  } else {
    switch (PM) {
      RG_V5_CASE(1)
      RG_V5_CASE(2)
      RG_V5_CASE(4)
      RG_V5_CASE(8)
      RG_V5_CASE(16)
    }
  }
  if (e != cudaSuccess) {
    set_error("rg_tall_f64: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return launched();
}
