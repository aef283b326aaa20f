// Thin QR of an n x p block (K5): small Cholesky for the CholQR2 fast path
// and a Householder TSQR for the robust path.
//
// Reference: recgmres.dense_kernels.reduced_qr
// (/root/reference/pkg/src/recgmres/dense_kernels.py:31-48) = LAPACK
// Householder QR (np.linalg.qr) + the r_jj >= 0 sign convention + rank
// flags |r_jj| <= rank_tol * ||X||_F.  The host layer runs CholQR2 through
// rg_tall_f64 (Gram, rg_chol_f64, solve+Gram, rg_chol_f64, solve) and falls
// back to rg_tsqr_f64 when rg_chol_f64 reports an ill-conditioned block, so
// rank flags are always decided on a Householder R, as in the reference.
//
// TSQR layout: level 0 splits the rows into chunks of C rows (C*p*8 = 64 KB
// of shared memory), one CTA factors a chunk in shared memory with
// Householder reflectors (LAPACK dlarfg convention: v_0 = 1, beta =
// -sign(alpha)*||x||), writes the reflectors back over the chunk (in place)
// and its p x p R into a stack; the stack is factored the same way until it
// fits one chunk.  The downward pass rebuilds Q in place, chunk by chunk,
// from the block of the level above.  All reductions are block-level in a
// fixed order, so results are deterministic.
#include "rg_common.cuh"

#include <vector>

namespace rg {

constexpr int kQrThreads = 256;
constexpr int kQrWarps = kQrThreads / 32;

// ----------------------------------------------------------------------------
// Cholesky of a small SPD Gram: up-looking, one CTA.
__global__ void chol_kernel(int p, const double* __restrict__ G, double* __restrict__ R,
                            int* __restrict__ status, double cond_tol) {
  extern __shared__ double sA[];  // p x p, column-major
  __shared__ int s_bad;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) sA[e] = G[e];
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  double gmax = 0.0;
  for (int j = 0; j < p; ++j) gmax = fmax(gmax, sA[j + j * p]);
  for (int j = 0; j < p; ++j) {
    // row j of R: R[j][i] for i >= j, computed in place in the upper triangle
    if (threadIdx.x == 0) {
      double d = sA[j + j * p];
      for (int k = 0; k < j; ++k) d = fma(-sA[k + j * p], sA[k + j * p], d);
      if (!(d > 0.0) || !isfinite(d)) {
        s_bad = 1;
        d = 1.0;
      }
      sA[j + j * p] = sqrt(d);
    }
    __syncthreads();
    const double rjj = sA[j + j * p];
    for (int i = j + 1 + threadIdx.x; i < p; i += blockDim.x) {
      double v = sA[j + i * p];
      for (int k = 0; k < j; ++k) v = fma(-sA[k + j * p], sA[k + i * p], v);
      sA[j + i * p] = v / rjj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int st = s_bad;
    if (!st) {
      double dmin = sA[0];
      for (int j = 1; j < p; ++j) dmin = fmin(dmin, sA[j + j * p]);
      if (dmin * dmin < cond_tol * gmax) st = 2;
    }
    *status = st;
  }
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int r = e % p, c = e / p;
    R[e] = r <= c ? sA[e] : 0.0;
  }
}

// ----------------------------------------------------------------------------
// block-wide sum of up to 32 values per thread (fixed order); result in out[]
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], int nv, double* scratch, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (k < nv) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nv) scratch[w * NV + k] = v[k];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nv; k += blockDim.x) {
    double s = 0.0;
    for (int ww = 0; ww < kQrWarps; ++ww) s += scratch[ww * NV + k];
    out[k] = s;
  }
  __syncthreads();
}

// Householder QR of one chunk (m <= C rows, zero padded to >= p rows) held
// column-major in smem A[p][C].  On exit: R in the upper triangle, v (v_0 = 1
// implicit) strictly below the diagonal, tau[j].
template <int PMAX>
__device__ void chunk_householder(double* A, int C, int mpad, int p, double* tau,
                                  double* scratch, double* bc) {
  for (int j = 0; j < p; ++j) {
    double* col = A + (int64_t)j * C;
    // ||x[1:]||^2
    double part[1] = {0.0};
    for (int r = j + 1 + threadIdx.x; r < mpad; r += blockDim.x) part[0] = fma(col[r], col[r], part[0]);
    block_sum<1>(part, 1, scratch, bc);
    if (threadIdx.x == 0) {
      const double alpha = col[j];
      const double sigma = bc[0];
      double t, beta, scale;
      if (sigma == 0.0) {
        t = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        const double nrm = sqrt(fma(alpha, alpha, sigma));
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      tau[j] = t;
      bc[1] = scale;
      bc[2] = beta;
    }
    __syncthreads();
    const double t = tau[j], scale = bc[1], beta = bc[2];
    for (int r = j + 1 + threadIdx.x; r < mpad; r += blockDim.x) col[r] *= scale;
    __syncthreads();
    if (threadIdx.x == 0) col[j] = beta;
    // apply H_j = I - t v v^T to columns j+1..p-1
    const int nk = p - j - 1;
    if (nk > 0 && t != 0.0) {
      double wv[PMAX];
#pragma unroll
      for (int k = 0; k < PMAX; ++k) wv[k] = 0.0;
      for (int r = j + 1 + threadIdx.x; r < mpad; r += blockDim.x) {
        const double vr = col[r];
#pragma unroll
        for (int k = 0; k < PMAX; ++k)
          if (k < nk) wv[k] = fma(vr, A[(int64_t)(j + 1 + k) * C + r], wv[k]);
      }
      block_sum<PMAX>(wv, nk, scratch, bc + 4);
      // w_k = A[j][k] + sum_{r>j} v_r A[r][k]  (v_j = 1), complete before any update
      for (int k = threadIdx.x; k < nk; k += blockDim.x) bc[4 + k] += A[(int64_t)(j + 1 + k) * C + j];
      __syncthreads();
      for (int r = j + threadIdx.x; r < mpad; r += blockDim.x) {
        const double vr = (r == j) ? 1.0 : col[r];
        for (int k = 0; k < nk; ++k) {
          double* ak = A + (int64_t)(j + 1 + k) * C;
          ak[r] = fma(-t * vr, bc[4 + k], ak[r]);
        }
      }
    }
    __syncthreads();
  }
}

// up pass: factor each chunk of `data` (m x p, ld) in place; R of chunk c goes
// to stack rows [c*p, (c+1)*p) (column-major, ld = ldst); tau to taus[c*p + j]
template <int PMAX>
__global__ void __launch_bounds__(kQrThreads) tsqr_up_kernel(double* data, int64_t ld, int64_t m, int p,
                                                             int C, double* stack, int64_t ldst,
                                                             double* taus) {
  extern __shared__ double smem[];
  double* A = smem;                   // [p][C]
  double* scratch = A + (int64_t)p * C;  // kQrWarps * PMAX
  double* bc = scratch + kQrWarps * PMAX;  // 4 + PMAX
  double* tau = bc + 4 + PMAX;          // PMAX
  const int64_t nchunks = (m + C - 1) / C;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t r0 = c * C;
    const int rows = (int)((m - r0) < (int64_t)C ? (m - r0) : (int64_t)C);
    const int mpad = rows < p ? p : rows;
    for (int k = 0; k < p; ++k)
      for (int r = threadIdx.x; r < mpad; r += blockDim.x)
        A[(int64_t)k * C + r] = r < rows ? data[r0 + r + k * ld] : 0.0;
    __syncthreads();
    chunk_householder<PMAX>(A, C, mpad, p, tau, scratch, bc);
    for (int k = 0; k < p; ++k)
      for (int r = threadIdx.x; r < rows; r += blockDim.x) data[r0 + r + k * ld] = A[(int64_t)k * C + r];
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int r = e % p, k = e / p;
      stack[c * p + r + (int64_t)k * ldst] = r <= k ? A[(int64_t)k * C + r] : 0.0;
    }
    if (threadIdx.x < p) taus[c * p + threadIdx.x] = tau[threadIdx.x];
    __syncthreads();
  }
}

// down pass: Q_c = H_0 ... H_{p-1} [B_c; 0] in place over the chunk's
// reflectors; B_c = rows [c*p, (c+1)*p) of `above` (ld = ldab)
template <int PMAX>
__global__ void __launch_bounds__(kQrThreads) tsqr_down_kernel(double* data, int64_t ld, int64_t m, int p,
                                                               int C, const double* above,
                                                               int64_t ldab, const double* taus) {
  extern __shared__ double smem[];
  double* V = smem;                       // [p][C] reflectors
  double* Q = V + (int64_t)p * C;         // [p][C]
  double* scratch = Q + (int64_t)p * C;   // kQrWarps * PMAX
  double* bc = scratch + kQrWarps * PMAX; // PMAX
  const int64_t nchunks = (m + C - 1) / C;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t r0 = c * C;
    const int rows = (int)((m - r0) < (int64_t)C ? (m - r0) : (int64_t)C);
    const int mpad = rows < p ? p : rows;
    for (int k = 0; k < p; ++k)
      for (int r = threadIdx.x; r < mpad; r += blockDim.x) {
        V[(int64_t)k * C + r] = r < rows ? data[r0 + r + k * ld] : 0.0;
        Q[(int64_t)k * C + r] = r < p ? above[c * p + r + (int64_t)k * ldab] : 0.0;
      }
    __syncthreads();
    for (int j = p - 1; j >= 0; --j) {
      const double t = taus[c * p + j];
      if (t == 0.0) continue;  // uniform across the block
      const double* v = V + (int64_t)j * C;
      double wv[PMAX];
#pragma unroll
      for (int k = 0; k < PMAX; ++k) wv[k] = 0.0;
      for (int r = j + threadIdx.x; r < mpad; r += blockDim.x) {
        const double vr = (r == j) ? 1.0 : v[r];
#pragma unroll
        for (int k = 0; k < PMAX; ++k)
          if (k < p) wv[k] = fma(vr, Q[(int64_t)k * C + r], wv[k]);
      }
      block_sum<PMAX>(wv, p, scratch, bc);
      for (int r = j + threadIdx.x; r < mpad; r += blockDim.x) {
        const double vr = (r == j) ? 1.0 : v[r];
        for (int k = 0; k < p; ++k) Q[(int64_t)k * C + r] = fma(-t * vr, bc[k], Q[(int64_t)k * C + r]);
      }
      __syncthreads();
    }
    for (int k = 0; k < p; ++k)
      for (int r = threadIdx.x; r < rows; r += blockDim.x) data[r0 + r + k * ld] = Q[(int64_t)k * C + r];
    __syncthreads();
  }
}

// top: R_out = D R_top, B = D with D = diag(r_jj < 0 ? -1 : +1)
__global__ void tsqr_top_kernel(int p, const double* Rtop, double* Rout, double* B) {
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int r = e % p, c = e / p;
    const double s = Rtop[r + r * p] < 0.0 ? -1.0 : 1.0;
    Rout[e] = r <= c ? s * Rtop[e] : 0.0;
    B[e] = (r == c) ? s : 0.0;
  }
}

static int tsqr_chunk(int p) { return p <= 8 ? 1024 : (p <= 16 ? 512 : 256); }

struct TsqrPlan {
  std::vector<int64_t> m;       // rows per level
  std::vector<int64_t> nchunk;  // chunks per level
  std::vector<int64_t> stack_off, tau_off;  // doubles offsets in workspace
  int64_t total_doubles = 0;
  int64_t rtop_off = 0, b_off = 0;
};

static TsqrPlan tsqr_plan(int64_t n, int p) {
  TsqrPlan P;
  const int C = tsqr_chunk(p);
  int64_t m = n, off = 0;
  while (true) {
    const int64_t nc = (m + C - 1) / C;
    P.m.push_back(m);
    P.nchunk.push_back(nc);
    P.tau_off.push_back(off);
    off += nc * p;
    P.stack_off.push_back(off);  // stack of this level's R blocks
    off += nc * p * (int64_t)p;
    if (nc == 1) break;
    m = nc * p;
  }
  P.rtop_off = P.stack_off.back();  // single chunk: its stack is R_top
  P.b_off = off;
  off += (int64_t)p * p;
  P.total_doubles = off;
  return P;
}

template <int PMAX>
static cudaError_t tsqr_run(int64_t n, int p, double* X, int64_t ldx, double* Rout, double* ws,
                            cudaStream_t st) {
  const int C = tsqr_chunk(p);
  TsqrPlan P = tsqr_plan(n, p);
  const size_t up_smem = ((size_t)p * C + kQrWarps * PMAX + 4 + PMAX + PMAX) * sizeof(double);
  const size_t dn_smem = ((size_t)2 * p * C + kQrWarps * PMAX + PMAX) * sizeof(double);
  cudaFuncSetAttribute(tsqr_up_kernel<PMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)up_smem);
  cudaFuncSetAttribute(tsqr_down_kernel<PMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dn_smem);
  const int L = (int)P.m.size();
  const int64_t gmax = (int64_t)sm_count() * 2;
  // up: level l data = (l == 0 ? X : stack of level l-1)
  for (int l = 0; l < L; ++l) {
    double* data = l == 0 ? X : ws + P.stack_off[l - 1];
    const int64_t ld = l == 0 ? ldx : P.m[l];
    const int64_t grid = P.nchunk[l] < gmax ? P.nchunk[l] : gmax;
    tsqr_up_kernel<PMAX><<<(unsigned)grid, kQrThreads, up_smem, st>>>(
        data, ld, P.m[l], p, C, ws + P.stack_off[l], P.nchunk[l] * p, ws + P.tau_off[l]);
  }
  tsqr_top_kernel<<<1, 128, 0, st>>>(p, ws + P.rtop_off, Rout, ws + P.b_off);
  // down: top level uses B = D; level l uses the Q of level l+1 (its data)
  for (int l = L - 1; l >= 0; --l) {
    double* data = l == 0 ? X : ws + P.stack_off[l - 1];
    const int64_t ld = l == 0 ? ldx : P.m[l];
    const double* above = (l == L - 1) ? ws + P.b_off : ws + P.stack_off[l];
    const int64_t ldab = (l == L - 1) ? p : P.m[l + 1];
    const int64_t grid = P.nchunk[l] < gmax ? P.nchunk[l] : gmax;
    tsqr_down_kernel<PMAX><<<(unsigned)grid, kQrThreads, dn_smem, st>>>(data, ld, P.m[l], p, C, above,
                                                                        ldab, ws + P.tau_off[l]);
  }
  return cudaGetLastError();
}

}  // namespace rg

extern "C" int rg_chol_f64(int32_t p, const double* d_g, double* d_r, int32_t* d_status,
                           double cond_tol, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(p >= 1 && p <= 64, "rg_chol_f64: p=%d outside [1, 64]", p);
  RG_REQUIRE(d_g && d_r && d_status, "rg_chol_f64: null pointer");
  ProfScope prof((cudaStream_t)stream);
  chol_kernel<<<1, 64, (size_t)p * p * sizeof(double), (cudaStream_t)stream>>>(p, d_g, d_r, d_status,
                                                                              cond_tol);
  RG_CHECK_LAUNCH("rg_chol_f64");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_chol p=%d", p);
  return RG_OK;
}

extern "C" int64_t rg_tsqr_workspace_bytes(int64_t n, int32_t p) {
  if (p < 1 || p > 32 || n < p) return 0;
  return rg::tsqr_plan(n, p).total_doubles * (int64_t)sizeof(double);
}

extern "C" int rg_tsqr_f64(int64_t n, int32_t p, double* d_x, int64_t ldx, double* d_r, void* d_work,
                           int64_t work_bytes, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(p >= 1 && p <= 32, "rg_tsqr_f64: p=%d outside [1, 32]", p);
  RG_REQUIRE(n >= p, "rg_tsqr_f64: reduced QR needs n >= p, got %lld < %d", (long long)n, p);
  RG_REQUIRE(d_x && d_r && ldx >= n, "rg_tsqr_f64: bad block");
  const int64_t need = rg_tsqr_workspace_bytes(n, p);
  RG_REQUIRE(d_work && work_bytes >= need, "rg_tsqr_f64: workspace %lld < %lld bytes",
             (long long)work_bytes, (long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  ProfScope prof(st);
  double* ws = (double*)d_work;
  cudaError_t e;
  if (p <= 8)
    e = tsqr_run<8>(n, p, d_x, ldx, d_r, ws, st);
  else if (p <= 16)
    e = tsqr_run<16>(n, p, d_x, ldx, d_r, ws, st);
  else
    e = tsqr_run<32>(n, p, d_x, ldx, d_r, ws, st);
  if (e != cudaSuccess) {
    set_error("rg_tsqr_f64: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  // one factor launch per level plus the two apply launches per lower level
  // (24np algorithmic bytes: one reduction pass + one apply pass)
  const int levels = (int)tsqr_plan(n, p).m.size();
  prof.finish(2 * levels - 1, 24 * n * p, 0.0, nullptr, 0, 0, 0, 0, "rg_tsqr p=%d", p);
  return RG_OK;
}
