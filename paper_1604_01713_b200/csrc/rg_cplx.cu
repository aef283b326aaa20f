// Complex128 twins of the hot-path kernels (BASELINE configs[4]: 27-point
// complex stencil, shifted-Helmholtz-like).  The reference is real-only
// (sparse_core.py:53 truncates complex input), so these kernels follow the
// complex restatement of SURVEY.md §8c: transposes become conjugate
// transposes and the r_jj >= 0 convention becomes r_jj real >= 0.
//
//   rg_spmm_csr_c128  persistent CSR x block; each complex multiply-add is
//                     (ar*xr - ai*xi, ar*xi + ai*xr) with every product and
//                     sum separately rounded, in ascending storage order --
//                     bitwise equal to oracle/spmm_oracle.c:oracle_spmm_c128
//   rg_tall_c128      lane-per-row complex update / triangular solves on the
//                     CUDA cores; Gram Gb^H z on DMMA m8n8k4 with four real
//                     products per complex tile (Cr += Ar Br + Ai Bi,
//                     Ci += Ar Bi - Ai Br), Gb staged through warp-private
//                     smem slabs (real and imaginary planes)
//   rg_chol_c128      Hermitian Cholesky G = R^H R, real positive diagonal
//
// Complex blocks are column-major arrays of interleaved (re, im) doubles.
#include "rg_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace rg {

__device__ __forceinline__ void dmma_c(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ----------------------------------------------------------------------------
// SpMM
// ----------------------------------------------------------------------------

constexpr int kCWarps = 8;
constexpr int kCChunk = 256;

// Production SpMM: no shared-memory staging.  G lanes share a row (G=2
// splits a 16-wide block into two 8-column halves, so one pass covers p=16
// and A is read once); each lane walks its own row's entries straight from
// global memory (L1-resident lines) with the next entry's index/value and X
// gathers issued one entry ahead.  Rows per warp RPW = 32/G; warps are
// persistent over RPW-row units.  Per (row, column): entries in storage
// order, each complex product formed and rounded separately, then added.
template <int G, int PB, bool GHOST>
__global__ void __launch_bounds__(kCWarps * 32, 2)
spmm_c128_direct_kernel(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ rp,
                        const int32_t* __restrict__ ci, const double2* __restrict__ va,
                        const double2* __restrict__ X, int64_t ldx, int64_t n_local,
                        const double2* __restrict__ Xg, int64_t ldg, double2* __restrict__ Y, int64_t ldy) {
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int rl = lane % RPW;
  const int cg = lane / RPW;
  const double2* Xc = X + (int64_t)cg * PB * ldx;
  const double2* Xgc = GHOST ? Xg + (int64_t)cg * PB * ldg : Xg;
  double2* Yc = Y + (int64_t)cg * PB * ldy;
  const int64_t nunits = (row_end - row_begin + RPW - 1) / RPW;
  const int64_t nwarps = (int64_t)gridDim.x * kCWarps;
  auto gather = [&](int32_t j, double2 (&xv)[PB]) {
    const double2* xp = Xc + j;
    int64_t ld = ldx;
    if (GHOST && j >= n_local) {
      xp = Xgc + (j - n_local);
      ld = ldg;
    }
#pragma unroll
    for (int c = 0; c < PB; ++c) xv[c] = __ldg(xp + c * ld);
  };
  for (int64_t u = (int64_t)blockIdx.x * kCWarps + w; u < nunits; u += nwarps) {
    const int64_t i = row_begin + u * RPW + rl;
    const bool valid = i < row_end;
    const int32_t t0 = valid ? __ldg(rp + i) : 0;
    const int32_t t1 = valid ? __ldg(rp + i + 1) : 0;
    double ar_[PB], ai_[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) ar_[c] = ai_[c] = 0.0;
    double2 xn[PB];
    double2 an = make_double2(0.0, 0.0);
    int32_t jn2 = 0;
    if (t0 < t1) {
      an = __ldg(va + t0);
      gather(__ldg(ci + t0), xn);
      if (t0 + 1 < t1) jn2 = __ldg(ci + t0 + 1);
    }
    for (int32_t t = t0; t < t1; ++t) {
      double2 xc[PB];
#pragma unroll
      for (int c = 0; c < PB; ++c) xc[c] = xn[c];
      const double2 a = an;
      if (t + 1 < t1) {
        an = __ldg(va + t + 1);
        gather(jn2, xn);
        if (t + 2 < t1) jn2 = __ldg(ci + t + 2);
      }
#pragma unroll
      for (int c = 0; c < PB; ++c) {
        const double pr = __dsub_rn(__dmul_rn(a.x, xc[c].x), __dmul_rn(a.y, xc[c].y));
        const double pi = __dadd_rn(__dmul_rn(a.x, xc[c].y), __dmul_rn(a.y, xc[c].x));
        ar_[c] = __dadd_rn(ar_[c], pr);
        ai_[c] = __dadd_rn(ai_[c], pi);
      }
    }
    if (valid) {
#pragma unroll
      for (int c = 0; c < PB; ++c) Yc[i + c * ldy] = make_double2(ar_[c], ai_[c]);
    }
  }
}

template <int G, int PB>
static void launch_spmm_cd(int64_t rb, int64_t re, const int32_t* rp, const int32_t* ci, const double2* va,
                           const double2* X, int64_t ldx, int64_t n_local, const double2* Xg, int64_t ldg,
                           double2* Y, int64_t ldy, cudaStream_t s) {
  static int per_sm[2] = {-1, -1};
  const int gi = Xg ? 1 : 0;
  if (per_sm[gi] < 0) {
    int v = 0;
    if (Xg)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, spmm_c128_direct_kernel<G, PB, true>, kCWarps * 32, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, spmm_c128_direct_kernel<G, PB, false>, kCWarps * 32, 0);
    per_sm[gi] = v < 1 ? 1 : v;
  }
  constexpr int RPW = 32 / G;
  const int64_t units = (re - rb + RPW - 1) / RPW;
  int64_t g = (int64_t)sm_count() * per_sm[gi];
  const int64_t need = (units + kCWarps - 1) / kCWarps;
  if (need < g) g = need;
  if (g < 1) g = 1;
  if (Xg)
    spmm_c128_direct_kernel<G, PB, true><<<(unsigned)g, kCWarps * 32, 0, s>>>(rb, re, rp, ci, va, X, ldx, n_local,
                                                                             Xg, ldg, Y, ldy);
  else
    spmm_c128_direct_kernel<G, PB, false><<<(unsigned)g, kCWarps * 32, 0, s>>>(rb, re, rp, ci, va, X, ldx, n_local,
                                                                              Xg, ldg, Y, ldy);
}

// ----------------------------------------------------------------------------
// tall-skinny complex passes
// ----------------------------------------------------------------------------

struct TallC {
  int64_t n;
  int p;
  const double2* zin;
  int64_t ldzin;
  double2* zout;
  int64_t ldzout;
  const double2* x1;
  int64_t ldx1;
  int a1;
  const double2* s1;
  double alpha1;
  const double2* x2;
  int64_t ldx2;
  int a2;
  const double2* s2;
  double alpha2;
  const double2* r1;
  const double2* r2;
  int gmode;
  const double2* gb;
  int64_t ldgb;
  int gc;
  int mtiles;
  double2* gout;   // modes 1/2: gc x p complex; mode 3: p doubles (as double2 storage reused)
  double* part;
  unsigned* counter;
  PeerComm comm;   // row-partitioned runs: Gout is summed over the ranks by the last CTA
};

constexpr int kTCWarps = 8;
constexpr int kTCThreads = kTCWarps * 32;
constexpr int kCS = 36;  // slab stride

template <int PM>
__device__ __forceinline__ void capply(double (&zr)[PM], double (&zi)[PM], const double2* __restrict__ X, int64_t ldx,
                                       int a, const double2* sS, double alpha, int64_t i) {
  double mr[PM], mi[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) mr[c] = mi[c] = 0.0;
  for (int a0 = 0; a0 < a; a0 += 4) {
    double2 xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = a0 + u < a ? __ldg(X + i + (int64_t)(a0 + u) * ldx) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (a0 + u < a) {
        const double2* srow = sS + (a0 + u) * PM;
#pragma unroll
        for (int c = 0; c < PM; ++c) {
          const double2 s = srow[c];
          mr[c] = fma(xv[u].x, s.x, mr[c]);
          mr[c] = fma(-xv[u].y, s.y, mr[c]);
          mi[c] = fma(xv[u].x, s.y, mi[c]);
          mi[c] = fma(xv[u].y, s.x, mi[c]);
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < PM; ++c) {
    zr[c] = zr[c] + alpha * mr[c];
    zi[c] = zi[c] + alpha * mi[c];
  }
}

// y R = z, R upper triangular complex with real diagonal; sR row-major, the
// diagonal slot holds 1 / r_jj (real part)
template <int PM>
__device__ __forceinline__ void ctrsm(double (&zr)[PM], double (&zi)[PM], const double2* sR, int p) {
#pragma unroll
  for (int j = 0; j < PM; ++j) {
    if (j < p) {
      double yr = zr[j], yi = zi[j];
#pragma unroll
      for (int k = 0; k < j; ++k) {
        const double2 r = sR[k * PM + j];
        yr = fma(-zr[k], r.x, yr);
        yr = fma(zi[k], r.y, yr);
        yi = fma(-zr[k], r.y, yi);
        yi = fma(-zi[k], r.x, yi);
      }
      const double inv = sR[j * PM + j].x;
      zr[j] = yr * inv;
      zi[j] = yi * inv;
    }
  }
}

template <int PM, int MTMAX>
__global__ void __launch_bounds__(kTCThreads, 1) tall_c128_kernel(TallC P) {
  extern __shared__ __align__(16) double smem[];
  const int p = P.p;
  double2* sS1 = reinterpret_cast<double2*>(smem);  // [a1][PM]
  double2* sS2 = sS1 + P.a1 * PM;
  double2* sR1 = sS2 + P.a2 * PM;                  // PM x PM row-major
  double2* sR2 = sR1 + PM * PM;
  double* wb = reinterpret_cast<double*>(sR2 + PM * PM);
  // per warp: z tile re/im [8][kCS] each, Gb slab re/im [8][kCS] each
  constexpr int kWarpWords = 4 * 8 * kCS;
  double* red = wb + kTCWarps * kWarpWords;

  for (int e = threadIdx.x; e < P.a1 * PM; e += kTCThreads) {
    const int aa = e / PM, c = e % PM;
    sS1[e] = c < p ? P.s1[aa + (int64_t)c * P.a1] : make_double2(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < P.a2 * PM; e += kTCThreads) {
    const int aa = e / PM, c = e % PM;
    sS2[e] = c < p ? P.s2[aa + (int64_t)c * P.a2] : make_double2(0.0, 0.0);
  }
  for (int e = threadIdx.x; e < PM * PM; e += kTCThreads) {
    const int ii = e / PM, jj = e % PM;
    const double2 id = make_double2(ii == jj ? 1.0 : 0.0, 0.0);
    double2 v1 = id, v2 = id;
    if (P.r1 && ii < p && jj < p) {
      v1 = P.r1[ii + (int64_t)jj * p];
      if (ii == jj) v1 = make_double2(1.0 / v1.x, 0.0);
    }
    if (P.r2 && ii < p && jj < p) {
      v2 = P.r2[ii + (int64_t)jj * p];
      if (ii == jj) v2 = make_double2(1.0 / v2.x, 0.0);
    }
    sR1[e] = v1;
    sR2[e] = v2;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  double* ztr = wb + warp * kWarpWords;
  double* zti = ztr + 8 * kCS;
  double* gsr = zti + 8 * kCS;
  double* gsi = gsr + 8 * kCS;
  const bool gram = P.gmode == 1 || P.gmode == 2;
  const int mtiles = P.mtiles;
  double acc[MTMAX][2][2];  // [tile][re/im][c-fragment]
#pragma unroll
  for (int mt = 0; mt < MTMAX; ++mt) acc[mt][0][0] = acc[mt][0][1] = acc[mt][1][0] = acc[mt][1][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  const int64_t nunits = (P.n + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * kTCWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kTCWarps;
  for (int64_t u = gwarp; u < nunits; u += nwarps) {
    const int64_t r0 = u * 32;
    const int64_t i = r0 + lane;
    const bool valid = i < P.n;
    double zr[PM], zi[PM];
#pragma unroll
    for (int c = 0; c < PM; ++c) zr[c] = zi[c] = 0.0;
    if (valid) {
      if (P.zin) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) {
            const double2 v = __ldg(P.zin + i + (int64_t)c * P.ldzin);
            zr[c] = v.x;
            zi[c] = v.y;
          }
      }
      if (P.a1) capply<PM>(zr, zi, P.x1, P.ldx1, P.a1, sS1, P.alpha1, i);
      if (P.a2) capply<PM>(zr, zi, P.x2, P.ldx2, P.a2, sS2, P.alpha2, i);
      if (P.r1) ctrsm<PM>(zr, zi, sR1, p);
      if (P.r2) ctrsm<PM>(zr, zi, sR2, p);
      if (P.zout) {
#pragma unroll
        for (int c = 0; c < PM; ++c)
          if (c < p) P.zout[i + (int64_t)c * P.ldzout] = make_double2(zr[c], zi[c]);
      }
      if (P.gmode == 3) {
#pragma unroll
        for (int c = 0; c < PM; ++c) sq[c] = fma(zr[c], zr[c], fma(zi[c], zi[c], sq[c]));
      }
    }
    if (!gram) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      ztr[c * kCS + lane] = c < PM ? zr[c < PM ? c : 0] : 0.0;
      zti[c * kCS + lane] = c < PM ? zi[c < PM ? c : 0] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < MTMAX; ++mt) {
      if (mt < mtiles) {
        const double* ar_ = ztr;
        const double* ai_ = zti;
        if (P.gmode == 1) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int gg = mt * 8 + c;
            const double2 v = (valid && gg < P.gc) ? __ldg(P.gb + i + (int64_t)gg * P.ldgb) : make_double2(0.0, 0.0);
            gsr[c * kCS + lane] = v.x;
            gsi[c * kCS + lane] = v.y;
          }
          __syncwarp();
          ar_ = gsr;
          ai_ = gsi;
        }
        const int cb = P.gmode == 1 ? 0 : mt * 8;  // self Gram: A = z tile rows mt*8.. (PM <= 8 -> mt == 0)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double a_r = ar_[(cb + mrow) * kCS + ks * 4 + kq];
          const double a_i = ai_[(cb + mrow) * kCS + ks * 4 + kq];
          const double b_r = ztr[mrow * kCS + ks * 4 + kq];
          const double b_i = zti[mrow * kCS + ks * 4 + kq];
          dmma_c(acc[mt][0][0], acc[mt][0][1], a_r, b_r);
          dmma_c(acc[mt][0][0], acc[mt][0][1], a_i, b_i);
          dmma_c(acc[mt][1][0], acc[mt][1][1], a_r, b_i);
          dmma_c(acc[mt][1][0], acc[mt][1][1], -a_i, b_r);
        }
        __syncwarp();
      }
    }
  }

  __shared__ bool s_last;
  __syncthreads();
  if (gram) {
    for (int ww = 0; ww < kTCWarps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTMAX; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int ri = 0; ri < 2; ++ri)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int idx = ((mt * 2 + ri) * 32 + lane) * 2 + v;
                red[idx] = (ww == 0) ? acc[mt][ri][v] : red[idx] + acc[mt][ri][v];
              }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kTCThreads) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7;
      const int ln = mr * 4 + (c >> 1), v = c & 1;
      P.part[((int64_t)blockIdx.x * ne + e) * 2] = red[((mt * 2 + 0) * 32 + ln) * 2 + v];
      P.part[((int64_t)blockIdx.x * ne + e) * 2 + 1] = red[((mt * 2 + 1) * 32 + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
#pragma unroll
    for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += kTCThreads) {
      double sum = 0.0;
      for (int ww = 0; ww < kTCWarps; ++ww) sum += red[ww * PM + c];
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
  if (P.gmode == 3) {
    double* out = reinterpret_cast<double*>(P.gout);
    for (int e = threadIdx.x; e < p; e += kTCThreads) {
      double sum = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * p + e);
      out[e] = sum;
    }
  } else {
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kTCThreads) {
      double sr = 0.0, si = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        sr += __ldcg(P.part + ((int64_t)b * ne + e) * 2);
        si += __ldcg(P.part + ((int64_t)b * ne + e) * 2 + 1);
      }
      P.gout[e] = make_double2(sr, si);
    }
  }
  // row-partitioned: finish the sum over the ranks here (doubles: a complex sum is component-wise)
  if (P.comm.world > 1)
    peer_allreduce(P.comm, reinterpret_cast<double*>(P.gout), P.gmode == 3 ? p : 2 * P.gc * p, threadIdx.x,
                   blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

template <int PM, int MTMAX>
static cudaError_t launch_tall_c(const TallC& P, cudaStream_t st) {
  auto k = tall_c128_kernel<PM, MTMAX>;
  const size_t smem = ((size_t)(P.a1 + P.a2) * PM * 2 + 4 * PM * PM + (size_t)kTCWarps * 4 * 8 * kCS +
                       (size_t)std::max(MTMAX * 2 * 64, kTCWarps * PM)) * sizeof(double);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  const int64_t nunits = (P.n + 31) / 32;
  int64_t g = (int64_t)sm_count();
  const int64_t need = (nunits + kTCWarps - 1) / kTCWarps;
  if (need < g) g = need;
  if (g < 1) g = 1;
  k<<<(unsigned)g, kTCThreads, smem, st>>>(P);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// Hermitian Cholesky
// ----------------------------------------------------------------------------

__global__ void chol_c128_kernel(int p, const double2* __restrict__ G, double2* __restrict__ R, int* status,
                                 double cond_tol) {
  extern __shared__ double2 sA[];
  __shared__ int s_bad;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) sA[e] = G[e];
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  double gmax = 0.0;
  for (int j = 0; j < p; ++j) gmax = fmax(gmax, sA[j + j * p].x);
  for (int j = 0; j < p; ++j) {
    if (threadIdx.x == 0) {
      double d = sA[j + j * p].x;
      for (int k = 0; k < j; ++k) {
        const double2 r = sA[k + j * p];
        d -= r.x * r.x + r.y * r.y;
      }
      if (!(d > 0.0) || !isfinite(d)) {
        s_bad = 1;
        d = 1.0;
      }
      sA[j + j * p] = make_double2(sqrt(d), 0.0);
    }
    __syncthreads();
    const double rjj = sA[j + j * p].x;
    for (int i = j + 1 + threadIdx.x; i < p; i += blockDim.x) {
      // R[j][i] = (G[j][i] - sum_k conj(R[k][j]) R[k][i]) / r_jj
      double vr = sA[j + i * p].x, vi = sA[j + i * p].y;
      for (int k = 0; k < j; ++k) {
        const double2 a = sA[k + j * p], b = sA[k + i * p];
        vr -= a.x * b.x + a.y * b.y;
        vi -= a.x * b.y - a.y * b.x;
      }
      sA[j + i * p] = make_double2(vr / rjj, vi / rjj);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int st = s_bad;
    if (!st) {
      double dmin = sA[0].x;
      for (int j = 1; j < p; ++j) dmin = fmin(dmin, sA[j + j * p].x);
      if (dmin * dmin < cond_tol * gmax) st = 2;
    }
    *status = st;
  }
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int r = e % p, c = e / p;
    R[e] = r <= c ? sA[e] : make_double2(0.0, 0.0);
  }
}

// ============================================================================
// tall_c6: complex tall-skinny pass on the FP64 tensor cores (p <= 16)
//
// The v6 design of rg_tall.cu in complex form.  A warp owns 32-row units;
// every n-length operand streams through a per-warp ring of cp.async slabs
// (32 rows x 4 complex columns, 16-byte chunks straight from the
// interleaved layout) driven by a per-CTA slab table.  Complex products
// are four real DMMA m8n8k4 per tile:
//   update  z += X (alpha S):  zr += Xr Sr' - Xi Si',  zi += Xr Si' + Xi Sr'
//           A = X slab element (re, im) [row][col], B = pre-arranged S'
//           fragments (alpha folded in), C = the 32 x p z tile in registers
//   Gram    G += Gb^H z:  Gr += Gbr zr + Gbi zi,  Gi += Gbr zi - Gbi zr
//           A = Gb slab pair [col][row], B = the z tile in smem
// Slab strides (in complex elements) keep every fragment read conflict-free:
// 34 for [row][col] reads of X / zin slabs, 36 for [col][row] reads of Gb
// slabs and the z tile.
// ============================================================================

constexpr int kC6Warps = 8;
constexpr int kC6Threads = kC6Warps * 32;
template <int PM>
struct C6Ring {
  static constexpr int value = PM > 8 ? 5 : 6;  // slabs in flight per warp (smem-bound)
};
constexpr int kC6SX = 34;
constexpr int kC6SG = 36;
constexpr int kC6Slot = 4 * kC6SG;  // complex elements per ring slot
constexpr int kC6MaxSlabs = 96;

struct C6Plan {
  int nz, n1, n2, ng, total;
};

struct C6Tab {
  const double2* ptr[kC6MaxSlabs];
  int64_t ld[kC6MaxSlabs];
  int nc[kC6MaxSlabs];
};

__device__ __forceinline__ void cp_async16c(double2* dst, const double2* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit_c() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_c() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int PM, int MT, bool TRSM, bool NOTERMS>
__global__ void __launch_bounds__(kC6Threads, 1) tall_c6_kernel(TallC P, C6Plan L) {
  constexpr int kC6Ring = C6Ring<PM>::value;
  constexpr int NT = PM / 8;
  constexpr int MTA = MT > 0 ? MT : 1;
  constexpr int kWarpC = kC6Ring * kC6Slot + PM * kC6SG;  // complex elements per warp
  extern __shared__ __align__(16) double smem[];
  __shared__ C6Tab tab;
  const int p = P.p;
  const int ks1 = (P.a1 + 3) / 4, ks2 = (P.a2 + 3) / 4;
  double2* sf1 = reinterpret_cast<double2*>(smem);  // [ks1][NT][32] (re, im) B fragments of alpha1 S1
  double2* sf2 = sf1 + (size_t)ks1 * NT * 32;
  double2* sR1 = sf2 + (size_t)ks2 * NT * 32;       // PM x PM row-major, diagonal slot = 1 / r_jj
  double2* sR2 = sR1 + PM * PM;
  double2* wbase = sR2 + PM * PM;
  double* red = reinterpret_cast<double*>(wbase + (size_t)kC6Warps * kWarpC);

  for (int e = threadIdx.x; e < ks1 * NT * 32; e += kC6Threads) {
    const int ks = e / (NT * 32), nt = (e / 32) % NT, ln = e % 32;
    const int aa = ks * 4 + (ln & 3), c = nt * 8 + (ln >> 2);
    double2 v = make_double2(0.0, 0.0);
    if (aa < P.a1 && c < p) {
      v = P.s1[aa + (int64_t)c * P.a1];
      v.x *= P.alpha1;
      v.y *= P.alpha1;
    }
    sf1[e] = v;
  }
  for (int e = threadIdx.x; e < ks2 * NT * 32; e += kC6Threads) {
    const int ks = e / (NT * 32), nt = (e / 32) % NT, ln = e % 32;
    const int aa = ks * 4 + (ln & 3), c = nt * 8 + (ln >> 2);
    double2 v = make_double2(0.0, 0.0);
    if (aa < P.a2 && c < p) {
      v = P.s2[aa + (int64_t)c * P.a2];
      v.x *= P.alpha2;
      v.y *= P.alpha2;
    }
    sf2[e] = v;
  }
  for (int e = threadIdx.x; e < PM * PM; e += kC6Threads) {
    const int ii = e / PM, jj = e % PM;
    const double2 id = make_double2(ii == jj ? 1.0 : 0.0, 0.0);
    double2 v1 = id, v2 = id;
    if (P.r1 && ii < p && jj < p) {
      v1 = P.r1[ii + (int64_t)jj * p];
      if (ii == jj) v1 = make_double2(1.0 / v1.x, 0.0);
    }
    if (P.r2 && ii < p && jj < p) {
      v2 = P.r2[ii + (int64_t)jj * p];
      if (ii == jj) v2 = make_double2(1.0 / v2.x, 0.0);
    }
    sR1[e] = v1;
    sR2[e] = v2;
  }
  // two solves z R1^-1 R2^-1 become one with R2 R1 (upper triangular, real
  // positive diagonal): half the substitution work
  const bool two = P.r1 && P.r2;
  if (TRSM && two) {
    __syncthreads();
    double2* prod = reinterpret_cast<double2*>(red);  // PM x PM scratch (red is free until the epilogue)
    for (int e = threadIdx.x; e < PM * PM; e += kC6Threads) {
      const int ii = e / PM, jj = e % PM;
      double2 v = make_double2(ii == jj ? 1.0 : 0.0, 0.0);
      if (ii < p && jj < p) {
        v = make_double2(0.0, 0.0);
        for (int k = ii; k <= jj; ++k) {
          const double2 a = P.r2[ii + (int64_t)k * p], b = P.r1[k + (int64_t)jj * p];
          v.x = fma(a.x, b.x, fma(-a.y, b.y, v.x));
          v.y = fma(a.x, b.y, fma(a.y, b.x, v.y));
        }
        if (ii == jj) v = make_double2(1.0 / v.x, 0.0);
      } else if (ii > jj) {
        v = make_double2(0.0, 0.0);
      }
      prod[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < PM * PM; e += kC6Threads) sR1[e] = prod[e];
  }
  for (int k = threadIdx.x; k < L.total; k += kC6Threads) {
    const double2* ptr;
    int64_t ld;
    int nc, s;
    if (k < L.nz) {
      ptr = P.zin; ld = P.ldzin; s = k; nc = p - s * 4;
    } else if (k < L.nz + L.n1) {
      ptr = P.x1; ld = P.ldx1; s = k - L.nz; nc = P.a1 - s * 4;
    } else if (k < L.nz + L.n1 + L.n2) {
      ptr = P.x2; ld = P.ldx2; s = k - L.nz - L.n1; nc = P.a2 - s * 4;
    } else {
      ptr = P.gb; ld = P.ldgb; s = k - L.nz - L.n1 - L.n2; nc = P.gc - s * 4;
    }
    tab.ptr[k] = ptr + (int64_t)(s * 4) * ld;
    tab.ld[k] = ld;
    tab.nc[k] = nc > 4 ? 4 : nc;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mrow = lane >> 2, kq = lane & 3;
  double2* ring = wbase + (size_t)warp * kWarpC;  // [kC6Ring][kC6Slot]
  double2* zt = ring + kC6Ring * kC6Slot;         // [PM][kC6SG]: zt[c * kC6SG + row]
  const bool gram_tile = MT > 0 && (P.gmode == 1 || P.gmode == 2);
  const int mtiles = P.mtiles;
  const int gfirst = L.nz + L.n1 + L.n2;

  double acc[MTA][NT][2][2];
#pragma unroll
  for (int mt = 0; mt < MTA; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0][0] = acc[mt][nt][0][1] = acc[mt][nt][1][0] = acc[mt][nt][1][1] = 0.0;
  double sq[PM];
#pragma unroll
  for (int c = 0; c < PM; ++c) sq[c] = 0.0;

  const int64_t nunits = (P.n + 31) / 32;
  const int64_t gwarp = (int64_t)blockIdx.x * kC6Warps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kC6Warps;
  const int64_t my_units = gwarp < nunits ? (nunits - gwarp + nwarps - 1) / nwarps : 0;

  int64_t iss_left = my_units * L.total;
  int64_t iss_r0 = gwarp * 32;
  int iss_k = 0, iss_slot = 0;
  auto issue_next = [&]() {
    if (iss_left > 0) {
      const double2* base = tab.ptr[iss_k];
      const int64_t ld = tab.ld[iss_k];
      const int nc = tab.nc[iss_k];
      const int st = iss_k >= gfirst ? kC6SG : kC6SX;
      const bool vrow = iss_r0 + lane < P.n;
      double2* dst = ring + iss_slot * kC6Slot + lane;
      const double2* src = base + iss_r0 + lane;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int bytes = (t < nc && vrow) ? 16 : 0;
        cp_async16c(dst + t * st, bytes ? src + (int64_t)t * ld : base, bytes);
      }
      --iss_left;
      if (++iss_k == L.total) {
        iss_k = 0;
        iss_r0 += nwarps * 32;
      }
    }
    cp_commit_c();
    if (++iss_slot == kC6Ring) iss_slot = 0;
  };
#pragma unroll
  for (int s = 0; s < kC6Ring; ++s) issue_next();
  int cons_slot = 0;
  auto take = [&]() -> const double2* {
    const double2* sl = ring + cons_slot * kC6Slot;
    if (++cons_slot == kC6Ring) cons_slot = 0;
    return sl;
  };
  auto acquire = [&]() -> const double2* {
    cp_wait_c<kC6Ring - 1>();
    __syncwarp();
    return take();
  };
  auto release = [&]() {
    __syncwarp();
    issue_next();
  };

  for (int64_t ui = 0; ui < my_units; ++ui) {
    const int64_t r0 = (gwarp + ui * nwarps) * 32;
    // z in DMMA C layout: rows rg*8 + mrow, columns nt*8 + 2*kq + v; [re/im]
    double zf[4][NT][2][2];
#pragma unroll
    for (int rg = 0; rg < 4; ++rg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) zf[rg][nt][0][0] = zf[rg][nt][0][1] = zf[rg][nt][1][0] = zf[rg][nt][1][1] = 0.0;
    if (NOTERMS) {
      // no update terms: zin slabs go straight into the z tile (row per lane)
#pragma unroll
      for (int k = 0; k < 2 * NT; ++k) {
        if (k < L.nz) {
          const double2* sl = acquire();
#pragma unroll
          for (int t = 0; t < 4; ++t) zt[(4 * k + t) * kC6SG + lane] = sl[t * kC6SX + lane];
          release();
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) zt[(4 * k + t) * kC6SG + lane] = make_double2(0.0, 0.0);
        }
      }
      __syncwarp();
    }
    // zin slab k holds complex columns 4k..4k+3 = tile k/2, lanes with kq/2 == k%2
#pragma unroll
    for (int k = 0; k < 2 * NT; ++k) {
      if (NOTERMS) break;
      if (k < L.nz) {
        const double2* sl = acquire();
        if ((kq >> 1) == (k & 1)) {
#pragma unroll
          for (int rg = 0; rg < 4; ++rg)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const double2 e = sl[(2 * (kq & 1) + v) * kC6SX + rg * 8 + mrow];
              zf[rg][k >> 1][0][v] = e.x;
              zf[rg][k >> 1][1][v] = e.y;
            }
        }
        release();
      }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (NOTERMS) break;
      const int nsl = t == 0 ? L.n1 : L.n2;
      const double2* sf = t == 0 ? sf1 : sf2;
      for (int s = 0; s < nsl; ++s) {
        const double2* sl = acquire();
        double br[NT], bi[NT], bn[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 b = sf[(s * NT + nt) * 32 + lane];
          br[nt] = b.x;
          bi[nt] = b.y;
          bn[nt] = -b.y;
        }
#pragma unroll
        for (int rg = 0; rg < 4; ++rg) {
          const double2 a = sl[kq * kC6SX + rg * 8 + mrow];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            dmma_c(zf[rg][nt][0][0], zf[rg][nt][0][1], a.x, br[nt]);
            dmma_c(zf[rg][nt][0][0], zf[rg][nt][0][1], a.y, bn[nt]);
            dmma_c(zf[rg][nt][1][0], zf[rg][nt][1][1], a.x, bi[nt]);
            dmma_c(zf[rg][nt][1][0], zf[rg][nt][1][1], a.y, br[nt]);
          }
        }
        release();
      }
    }
    // ---------------- rows: tile, triangular solves, store, norms
    if (!NOTERMS) {
#pragma unroll
      for (int rg = 0; rg < 4; ++rg)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            zt[(nt * 8 + 2 * kq + v) * kC6SG + rg * 8 + mrow] = make_double2(zf[rg][nt][0][v], zf[rg][nt][1][v]);
      __syncwarp();
    }
    const int64_t i = r0 + lane;
    const bool valid = i < P.n;
    if (TRSM) {
      // lane-per-row forward substitution
      double zr[PM], zi[PM];
#pragma unroll
      for (int c = 0; c < PM; ++c) {
        const double2 e = zt[c * kC6SG + lane];
        zr[c] = e.x;
        zi[c] = e.y;
      }
      if (P.r1) ctrsm<PM>(zr, zi, sR1, p);
      if (P.r2 && !two) ctrsm<PM>(zr, zi, sR2, p);
#pragma unroll
      for (int c = 0; c < PM; ++c) zt[c * kC6SG + lane] = make_double2(zr[c], zi[c]);
      __syncwarp();
    }
    if (P.zout && valid) {
      for (int c = 0; c < p; ++c) P.zout[i + (int64_t)c * P.ldzout] = zt[c * kC6SG + lane];
    }
    if (P.gmode == 3 && valid) {
#pragma unroll
      for (int c = 0; c < PM; ++c) {
        const double2 e = zt[c * kC6SG + lane];
        sq[c] = fma(e.x, e.x, fma(e.y, e.y, sq[c]));
      }
    }
    if (!gram_tile) continue;
#pragma unroll
    for (int mt = 0; mt < MTA; ++mt) {
      if (mt < mtiles) {
        const double2* sa = zt + (size_t)(mt * 8) * kC6SG;  // self Gram: A = z columns mt*8..
        int sa_off = mrow * kC6SG;
        if (P.gmode == 1) {
          // both slabs of this 8-column Gb tile must have landed
          cp_wait_c<kC6Ring - 2>();
          __syncwarp();
          const double2* s0 = take();
          const double2* s1 = take();
          sa = mrow < 4 ? s0 : s1;
          sa_off = (mrow & 3) * kC6SG;
        }
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const double2 a = sa[sa_off + ks * 4 + kq];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 b = zt[(nt * 8 + mrow) * kC6SG + ks * 4 + kq];
            dmma_c(acc[mt][nt][0][0], acc[mt][nt][0][1], a.x, b.x);
            dmma_c(acc[mt][nt][0][0], acc[mt][nt][0][1], a.y, b.y);
            dmma_c(acc[mt][nt][1][0], acc[mt][nt][1][1], a.x, b.y);
            dmma_c(acc[mt][nt][1][0], acc[mt][nt][1][1], -a.y, b.x);
          }
        }
        if (P.gmode == 1) {
          release();
          release();
        }
      }
    }
    __syncwarp();
  }
  cp_wait_c<0>();

  // ---------------- epilogue: deterministic reductions (as tall_c128_kernel)
  __shared__ bool s_last;
  __syncthreads();
  if (gram_tile) {
    for (int ww = 0; ww < kC6Warps; ++ww) {
      if (warp == ww) {
#pragma unroll
        for (int mt = 0; mt < MTA; ++mt)
          if (mt < mtiles) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int ri = 0; ri < 2; ++ri)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                  const int idx = ((((mt * NT + nt) * 2 + ri) * 32) + lane) * 2 + v;
                  red[idx] = (ww == 0) ? acc[mt][nt][ri][v] : red[idx] + acc[mt][nt][ri][v];
                }
          }
      }
      __syncthreads();
    }
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kC6Threads) {
      const int gg = e % P.gc, c = e / P.gc;
      const int mt = gg >> 3, mr = gg & 7, nt = c >> 3, ncol = c & 7;
      const int ln = mr * 4 + (ncol >> 1), v = ncol & 1;
      P.part[((int64_t)blockIdx.x * ne + e) * 2] = red[((((mt * NT + nt) * 2 + 0) * 32) + ln) * 2 + v];
      P.part[((int64_t)blockIdx.x * ne + e) * 2 + 1] = red[((((mt * NT + nt) * 2 + 1) * 32) + ln) * 2 + v];
    }
  } else if (P.gmode == 3) {
#pragma unroll
    for (int c = 0; c < PM; ++c) sq[c] = warp_sum(sq[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < PM; ++c) red[warp * PM + c] = sq[c];
    __syncthreads();
    for (int c = threadIdx.x; c < p; c += kC6Threads) {
      double sum = 0.0;
      for (int ww = 0; ww < kC6Warps; ++ww) sum += red[ww * PM + c];
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
  if (P.gmode == 3) {
    double* out = reinterpret_cast<double*>(P.gout);
    for (int e = threadIdx.x; e < p; e += kC6Threads) {
      double sum = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) sum += __ldcg(P.part + (int64_t)b * p + e);
      out[e] = sum;
    }
  } else {
    const int ne = P.gc * p;
    for (int e = threadIdx.x; e < ne; e += kC6Threads) {
      double sr = 0.0, si = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) {
        sr += __ldcg(P.part + ((int64_t)b * ne + e) * 2);
        si += __ldcg(P.part + ((int64_t)b * ne + e) * 2 + 1);
      }
      P.gout[e] = make_double2(sr, si);
    }
  }
  // row-partitioned: finish the sum over the ranks here (doubles: a complex sum is component-wise)
  if (P.comm.world > 1)
    peer_allreduce(P.comm, reinterpret_cast<double*>(P.gout), P.gmode == 3 ? p : 2 * P.gc * p, threadIdx.x,
                   blockDim.x);
  if (threadIdx.x == 0) *P.counter = 0u;
}

template <int PM, int MT>
static cudaError_t launch_c6(const TallC& P, cudaStream_t st) {
  constexpr int kC6Ring = C6Ring<PM>::value;
  constexpr int NT = PM / 8;
  constexpr int kWarpC = kC6Ring * kC6Slot + PM * kC6SG;
  const bool trsm = P.r1 || P.r2;
  const bool noterms = P.a1 == 0 && P.a2 == 0;
  auto k = trsm ? (noterms ? tall_c6_kernel<PM, MT, true, true> : tall_c6_kernel<PM, MT, true, false>)
                : (noterms ? tall_c6_kernel<PM, MT, false, true> : tall_c6_kernel<PM, MT, false, false>);
  const int ki = (trsm ? 2 : 0) + (noterms ? 1 : 0);
  C6Plan L;
  L.nz = P.zin ? (P.p + 3) / 4 : 0;
  L.n1 = (P.a1 + 3) / 4;
  L.n2 = (P.a2 + 3) / 4;
  L.ng = P.gmode == 1 ? 2 * P.mtiles : 0;
  L.total = L.nz + L.n1 + L.n2 + L.ng;
  const size_t smem = ((size_t)(L.n1 + L.n2) * NT * 32 + 2 * PM * PM + (size_t)kC6Warps * kWarpC) * 16 +
                      (size_t)std::max(std::max(MT * NT * 2 * 64, kC6Warps * PM), 2 * PM * PM) * sizeof(double);
  static bool cfg[4] = {false, false, false, false};
  if (!cfg[ki]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cfg[ki] = true;
  }
  const int64_t nunits = (P.n + 31) / 32;
  int64_t g = (int64_t)sm_count();
  const int64_t need = (nunits + kC6Warps - 1) / kC6Warps;
  if (need < g) g = need;
  if (g < 1) g = 1;
  k<<<(unsigned)g, kC6Threads, smem, st>>>(P, L);
  return cudaGetLastError();
}

}  // namespace rg

extern "C" int rg_spmm_csr_c128(int64_t n_rows, int64_t row_begin, int64_t row_end, const int32_t* d_row_ptr,
                                const int32_t* d_col_idx, const double* d_vals, const double* d_x, int64_t ldx,
                                int64_t n_local, const double* d_xg, int64_t ldg, int32_t p, double* d_y,
                                int64_t ldy, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n_rows >= 0 && 0 <= row_begin && row_begin <= row_end && row_end <= n_rows,
             "rg_spmm_csr_c128: bad row range");
  RG_REQUIRE(p >= 1 && d_row_ptr && d_y && ldy >= n_rows, "rg_spmm_csr_c128: bad arguments");
  if (row_end == row_begin) return RG_OK;
  ProfScope prof((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  const double2* X = reinterpret_cast<const double2*>(d_x);
  const double2* Xg = reinterpret_cast<const double2*>(d_xg);
  double2* Y = reinterpret_cast<double2*>(d_y);
  const double2* va = reinterpret_cast<const double2*>(d_vals);
  {
    // passes of 16 columns (two lanes per row), then one exact-width pass
    for (int c0 = 0; c0 < p;) {
      const int rem = p - c0;
      const int pc = rem >= 16 ? 16 : (rem >= 8 ? 8 : rem);
      const double2* Xc = X ? X + (int64_t)c0 * ldx : nullptr;
      const double2* Xgc = Xg ? Xg + (int64_t)c0 * ldg : nullptr;
      double2* Yc = Y + (int64_t)c0 * ldy;
#define RG_CD(G, PB) launch_spmm_cd<G, PB>(row_begin, row_end, d_row_ptr, d_col_idx, va, Xc, ldx, n_local, Xgc, ldg, Yc, ldy, s)
      switch (pc) {
        case 16: RG_CD(2, 8); break;
        case 8: RG_CD(1, 8); break;
        case 7: RG_CD(1, 7); break;
        case 6: RG_CD(1, 6); break;
        case 5: RG_CD(1, 5); break;
        case 4: RG_CD(1, 4); break;
        case 3: RG_CD(1, 3); break;
        case 2: RG_CD(1, 2); break;
        default: RG_CD(1, 1); break;
      }
#undef RG_CD
      RG_CHECK_LAUNCH("rg_spmm_csr_c128");
      c0 += pc;
    }
  }
  prof.finish((p + 15) / 16 + (p % 16 > 8 ? 1 : 0), 0, 0.0, d_row_ptr, row_begin, row_end, p, 16, "rg_spmm_c128 p=%d", p);
  return RG_OK;
}

extern "C" int64_t rg_tall_c128_workspace_bytes(int64_t n, int32_t p, int32_t a1, int32_t a2, int32_t gram_mode,
                                                int32_t gc) {
  (void)n; (void)a1; (void)a2;
  int64_t ne = 0;
  if (gram_mode == 1) ne = (int64_t)gc * p * 2;
  if (gram_mode == 2) ne = (int64_t)p * p * 2;
  if (gram_mode == 3) ne = p;
  return 256 + (int64_t)rg::sm_count() * ne * (int64_t)sizeof(double);
}

extern "C" int rg_tall_c128(int64_t n, int32_t p, const double* d_zin, int64_t ldzin, double* d_zout, int64_t ldzout,
                            const double* d_x1, int64_t ldx1, int32_t a1, const double* d_s1, double alpha1,
                            const double* d_x2, int64_t ldx2, int32_t a2, const double* d_s2, double alpha2,
                            const double* d_r1, const double* d_r2, int32_t gram_mode, const double* d_gb,
                            int64_t ldgb, int32_t gc, double* d_gout, void* d_work, int64_t work_bytes,
                            void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && p >= 1 && p <= 16, "rg_tall_c128: p=%d outside [1, 16]", p);
  RG_REQUIRE(a1 >= 0 && a2 >= 0 && a1 + a2 <= (p > 8 ? 128 : 256), "rg_tall_c128: term widths %d, %d (p=%d)", a1,
             a2, p);
  RG_REQUIRE(a1 == 0 || (d_x1 && d_s1 && ldx1 >= n), "rg_tall_c128: bad term 1");
  RG_REQUIRE(a2 == 0 || (d_x2 && d_s2 && ldx2 >= n), "rg_tall_c128: bad term 2");
  RG_REQUIRE(gram_mode >= 0 && gram_mode <= 3, "rg_tall_c128: gram_mode %d", gram_mode);
  const int gc_max = p > 8 ? ((a1 == 0 && a2 == 0) ? 64 : 32) : 48;
  RG_REQUIRE(gram_mode != 1 || (d_gb && gc >= 1 && gc <= gc_max && ldgb >= n),
             "rg_tall_c128: Gram basis width gc=%d outside [1, %d]", gc, gc_max);
  RG_REQUIRE(gram_mode != 2 || gc == p, "rg_tall_c128: self Gram needs gc == p");
  RG_REQUIRE(gram_mode == 0 || d_gout, "rg_tall_c128: null Gram output");
  if (gram_mode == 3) gc = 1;
  const int64_t need = rg_tall_c128_workspace_bytes(n, p, a1, a2, gram_mode, gc);
  RG_REQUIRE(gram_mode == 0 || (d_work && work_bytes >= need), "rg_tall_c128: workspace too small");
  TallC P;
  P.n = n; P.p = p;
  P.zin = reinterpret_cast<const double2*>(d_zin); P.ldzin = ldzin;
  P.zout = reinterpret_cast<double2*>(d_zout); P.ldzout = ldzout;
  P.x1 = reinterpret_cast<const double2*>(d_x1); P.ldx1 = ldx1; P.a1 = a1;
  P.s1 = reinterpret_cast<const double2*>(d_s1); P.alpha1 = alpha1;
  P.x2 = reinterpret_cast<const double2*>(d_x2); P.ldx2 = ldx2; P.a2 = a2;
  P.s2 = reinterpret_cast<const double2*>(d_s2); P.alpha2 = alpha2;
  P.r1 = reinterpret_cast<const double2*>(d_r1); P.r2 = reinterpret_cast<const double2*>(d_r2);
  P.gmode = gram_mode; P.gb = reinterpret_cast<const double2*>(d_gb); P.ldgb = ldgb; P.gc = gc;
  P.mtiles = (gram_mode == 1 || gram_mode == 2) ? (gc + 7) / 8 : 0;
  P.gout = reinterpret_cast<double2*>(d_gout);
  P.counter = (unsigned*)d_work;
  P.part = d_work ? (double*)((char*)d_work + 256) : nullptr;
  if (gram_mode == 0 && n == 0) return RG_OK;
  P.comm = peer_comm_next(gram_mode != 0);
  cudaStream_t st0 = (cudaStream_t)stream;
  ProfScope prof(st0);
  auto launched = [&]() {
    const bool same_x = a1 > 0 && a2 > 0 && d_x1 == d_x2 && a1 == a2;
    const bool aliased = gram_mode == 1 && ((d_gb == d_x1 && gc <= a1) || (d_gb == d_x2 && gc <= a2));
    const int64_t cols = (d_zin ? p : 0) + a1 + (same_x ? 0 : a2) + (gram_mode == 1 && !aliased ? gc : 0) +
                         (d_zout ? p : 0);
    const double contr = a1 + (same_x ? 0 : a2) + ((gram_mode == 1 || gram_mode == 2) ? gc : 0);
    prof.finish(1, 16 * n * cols, 8.0 * n * p * contr, nullptr, 0, 0, 0, 0,
                "rg_tall_c128 p=%d in=%d a=%d+%d g%d:%d trsm=%d out=%d", p, d_zin ? 1 : 0, a1, a2, gram_mode, gc,
                (d_r1 ? 1 : 0) + (d_r2 ? 1 : 0), d_zout ? 1 : 0);
    return RG_OK;
  };
  if (p > 4) {
    // tensor-core pass (complex v6)
    cudaError_t e6;
    const int mt = P.mtiles;
    if (p > 8) {
      e6 = mt == 0 ? launch_c6<16, 0>(P, st0)
                   : (mt <= 2 ? launch_c6<16, 2>(P, st0) : (mt <= 4 ? launch_c6<16, 4>(P, st0) : launch_c6<16, 8>(P, st0)));
    } else {
      e6 = mt == 0 ? launch_c6<8, 0>(P, st0)
                   : (mt <= 2 ? launch_c6<8, 2>(P, st0) : launch_c6<8, 6>(P, st0));
    }
    if (e6 != cudaSuccess) {
      set_error("rg_tall_c128: %s", cudaGetErrorString(e6));
      return RG_ECUDA;
    }
    return launched();
  }
  const int PM = p <= 1 ? 1 : (p <= 2 ? 2 : (p <= 4 ? 4 : 8));
  const int mtmax = P.mtiles <= 2 ? 2 : 6;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
#define RG_TC(PMv)                                                          \
  case PMv:                                                                 \
    e = mtmax == 2 ? launch_tall_c<PMv, 2>(P, st) : launch_tall_c<PMv, 6>(P, st); \
    break;
  switch (PM) {
    RG_TC(1)
    RG_TC(2)
    RG_TC(4)
    default: e = mtmax == 2 ? launch_tall_c<8, 2>(P, st) : launch_tall_c<8, 6>(P, st); break;
  }
#undef RG_TC
  if (e != cudaSuccess) {
    set_error("rg_tall_c128: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  return launched();
}

extern "C" int rg_chol_c128(int32_t p, const double* d_g, double* d_r, int32_t* d_status, double cond_tol,
                            void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(p >= 1 && p <= 64 && d_g && d_r && d_status, "rg_chol_c128: bad arguments");
  ProfScope prof((cudaStream_t)stream);
  chol_c128_kernel<<<1, 64, (size_t)p * p * sizeof(double2), (cudaStream_t)stream>>>(
      p, reinterpret_cast<const double2*>(d_g), reinterpret_cast<double2*>(d_r), d_status, cond_tol);
  RG_CHECK_LAUNCH("rg_chol_c128");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_chol_c128 p=%d", p);
  return RG_OK;
}
