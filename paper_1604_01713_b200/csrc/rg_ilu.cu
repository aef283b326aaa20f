// ILU(0) factorisation and the sparse triangular block solves that apply it
// (reference: precond.py:33-76 ilu0, :79-90 apply_precond; SURVEY.md §8f
// rank 2).
//
// Schedule.  The lower-triangular dependency graph (row i reads rows k < i
// of its strictly lower pattern) orders both the factorisation and the
// forward solve; the upper part (rows k > i) orders the backward solve.
// rg_wave_schedule (host code, once per factorisation) assigns every row
// its level (1 + the deepest level it reads) and lists the rows level by
// level in chunks of up to chunk_rows rows (a multiple of 32) of ONE level;
// a lane takes every 32nd row of its warp's chunk.  Kernels are persistent
// and sync-free: a warp claims the next chunk from a global ticket, each
// lane takes one row, polls (relaxed loads, then one acquire fence) the
// completion flag of every row it reads, computes, and publishes its row
// (release store).  Chunks are claimed in
// level order, so a waited-on row always belongs to a chunk claimed earlier
// by a resident warp (no deadlock), and lanes of one chunk never wait on
// each other.  Flags carry an epoch so they never need clearing.
//
// rg_ilu0_f64     IKJ ILU(0) restricted to A's pattern, in place on a
//                 device copy of A's values, one lane per row: for each
//                 strictly lower entry (ascending column k) l = a_ik / u_kk,
//                 then a_ij -= l * u_kj over row k's upper part (binary
//                 search of j in row i).  Separately rounded in the
//                 reference's order: bitwise precond.py:60-72.
// rg_sptrsv_f64   X = L^-1 B (unit lower) or U^-1 B (upper) on the combined
//                 LU pattern, one lane per row, the block columns in groups
//                 of 8 registers.
#include "rg_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace rg {

constexpr int kWaveWarps = 8;

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// acquire pattern: relaxed flag loads, then ONE fence once every flag a row
// needs has been seen (an ld.acquire per poll invalidates the SM's whole L1)
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
struct Wave {
  const int32_t* order;   // rows in level order
  const int32_t* chunk;   // nchunks + 1 offsets into order
  int32_t nchunks;
  int* flags;
  int epoch;
  unsigned* ticket;
  unsigned ns_max;        // longest back-off sleep while waiting on a flag
};

__device__ __forceinline__ void wait_row(const int* flags, int64_t k, int epoch, unsigned ns_max) {
  // back off while waiting: thousands of spinning lanes would otherwise
  // flood L2 with acquire loads and slow the rows they are waiting for
  unsigned ns = 16;
  while (ld_relaxed(flags + k) != epoch) {
    if (ns_max) {
      __nanosleep(ns);
      if (ns < ns_max) ns <<= 1;
    }
  }
}

__device__ __forceinline__ int32_t claim_chunk(unsigned* ticket, int lane) {
  unsigned t = 0;
  if (lane == 0) t = atomicAdd(ticket, 1u);
  return (int32_t)__shfl_sync(0xffffffffu, t, 0);
}

// all of a row's dependency flags are polled together (one L2 round trip per
// poll instead of one per dependency)
__device__ __forceinline__ void wait_rows(const int* flags, const int32_t* __restrict__ ci, int32_t eb, int32_t ee,
                                          int epoch, unsigned ns_max) {
  unsigned ns = 16;
  for (;;) {
    bool ready = true;
    for (int32_t e = eb; e < ee; e += 4) {
      int f[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] = e + q < ee ? ld_relaxed(flags + ci[e + q]) : epoch;
#pragma unroll
      for (int q = 0; q < 4; ++q) ready = ready && f[q] == epoch;
    }
    if (ready) return;
    if (ns_max) {
      __nanosleep(ns);
      if (ns < ns_max) ns <<= 1;
    }
  }
}

__global__ void __launch_bounds__(kWaveWarps * 32) ilu0_kernel(Wave W, const int32_t* __restrict__ rp,
                                                                const int32_t* __restrict__ ci, double* vals,
                                                                const int32_t* __restrict__ dpos,
                                                                long long* zero_row) {
  const int lane = threadIdx.x & 31;
  int32_t c = claim_chunk(W.ticket, lane);
  while (c < W.nchunks) {
    const int32_t c_next = claim_chunk(W.ticket, lane);  // overlaps this chunk
    const int32_t e1 = W.chunk[c + 1];
    for (int32_t ee_ = W.chunk[c] + lane; ee_ < e1; ee_ += 32) {
    const int32_t i = W.order[ee_];
    const int32_t lo = rp[i], hi = rp[i + 1], di = dpos[i];
    wait_rows(W.flags, ci, lo, di, W.epoch, W.ns_max);
    fence_acquire();
    for (int32_t t = lo; t < di; ++t) {
      const int32_t k = ci[t];
      const double lik = __ddiv_rn(vals[t], __ldcg(vals + dpos[k]));
      vals[t] = lik;
      const int32_t ke = rp[k + 1];
      int32_t a = t + 1;  // row i's columns after k, searched in ascending order
      for (int32_t s = dpos[k] + 1; s < ke; ++s) {
        const int32_t j = ci[s];
        int32_t b = hi;
        while (a < b) {
          const int32_t mid = (a + b) >> 1;
          if (ci[mid] < j) a = mid + 1; else b = mid;
        }
        if (a < hi && ci[a] == j) vals[a] = __dsub_rn(vals[a], __dmul_rn(lik, __ldcg(vals + s)));
      }
    }
    if (vals[di] == 0.0) atomicMin(zero_row, (long long)i);
    st_release(W.flags + i, W.epoch);
    }
    c = c_next;
  }
}

template <bool UPPER>
__global__ void __launch_bounds__(kWaveWarps * 32) sptrsv_kernel(Wave W, const int32_t* __restrict__ rp,
                                                                  const int32_t* __restrict__ ci,
                                                                  const double* __restrict__ vals,
                                                                  const int32_t* __restrict__ dpos, int p,
                                                                  const double* B, int64_t ldb, double* X,
                                                                  int64_t ldx) {
  const int lane = threadIdx.x & 31;
  int32_t c = claim_chunk(W.ticket, lane);
  while (c < W.nchunks) {
    const int32_t c_next = claim_chunk(W.ticket, lane);
    const int32_t e1 = W.chunk[c + 1];
    for (int32_t ee_ = W.chunk[c] + lane; ee_ < e1; ee_ += 32) {
    const int32_t i = W.order[ee_];
    const int32_t di = dpos[i];
    const int32_t eb = UPPER ? di + 1 : rp[i];
    const int32_t ee = UPPER ? rp[i + 1] : di;
    wait_rows(W.flags, ci, eb, ee, W.epoch, W.ns_max);
    fence_acquire();
    const double dinv_src = UPPER ? vals[di] : 1.0;
    for (int c0 = 0; c0 < p; c0 += 8) {
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = (c0 + q < p) ? B[i + (int64_t)(c0 + q) * ldb] : 0.0;
      for (int32_t e = eb; e < ee; ++e) {
        const int32_t k = ci[e];
        const double v = vals[e];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (c0 + q < p) acc[q] = __dsub_rn(acc[q], __dmul_rn(v, __ldcg(X + k + (int64_t)(c0 + q) * ldx)));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q < p) X[i + (int64_t)(c0 + q) * ldx] = UPPER ? __ddiv_rn(acc[q], dinv_src) : acc[q];
    }
    st_release(W.flags + i, W.epoch);
    }
    c = c_next;
  }
}

// Level-ordered variant of the solve.  The triangle is renumbered by its
// schedule (row r of the permuted matrix = the r-th row in level order,
// columns renamed to level positions, entries kept in their original order)
// and the block lives in a row-major workspace in the same order, so the 32
// lanes of a chunk read 32 consecutive CSR rows and 32 consecutive block rows
// (p contiguous doubles each) instead of rows a grid-line apart.  Arithmetic
// is the same as sptrsv_kernel's.
__global__ void __launch_bounds__(kWaveWarps * 32) sptrsv_perm_kernel(Wave W, const int32_t* __restrict__ rp,
                                                                       const int32_t* __restrict__ ci,
                                                                       const double* __restrict__ vals,
                                                                       const double* __restrict__ dval, int p,
                                                                       double* Xw) {
  const int lane = threadIdx.x & 31;
  int32_t c = claim_chunk(W.ticket, lane);
  while (c < W.nchunks) {
    // claim the next chunk now: the ticket round trip overlaps this chunk
    const int32_t c_next = claim_chunk(W.ticket, lane);
    const int32_t ce = W.chunk[c + 1];
    for (int32_t r = W.chunk[c] + lane; r < ce; r += 32) {
      const int32_t eb = rp[r], ee = rp[r + 1];
      double* xr = Xw + (int64_t)r * p;
      // the row's own right-hand side does not depend on anything: load it first
      double own[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) own[q] = q < p ? xr[q] : 0.0;
      wait_rows(W.flags, ci, eb, ee, W.epoch, W.ns_max);
      fence_acquire();
      for (int c0 = 0; c0 < p; c0 += 8) {
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = c0 == 0 ? own[q] : ((c0 + q < p) ? xr[c0 + q] : 0.0);
        for (int32_t e = eb; e < ee; ++e) {
          const double v = vals[e];
          const double* xk = Xw + (int64_t)ci[e] * p + c0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (c0 + q < p) acc[q] = __dsub_rn(acc[q], __dmul_rn(v, __ldcg(xk + q)));
        }
        if (dval) {
          const double d = dval[r];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __ddiv_rn(acc[q], d);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (c0 + q < p) xr[c0 + q] = acc[q];
      }
      st_release(W.flags + r, W.epoch);
    }
    c = c_next;
  }
}

// dst row pos_d[i] <- src row pos_s[i]; a null position array means the
// column-major layout in original order (leading dimension ld), otherwise a
// row-major p-wide layout in the permuted order.
__global__ void permute_rows_kernel(int64_t n, int p, const double* __restrict__ src, int64_t lds,
                                    const int32_t* __restrict__ pos_s, double* __restrict__ dst, int64_t ldd,
                                    const int32_t* __restrict__ pos_d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* sr = pos_s ? src + (int64_t)pos_s[i] * p : src + i;
    double* dr = pos_d ? dst + (int64_t)pos_d[i] * p : dst + i;
    const int64_t ss = pos_s ? 1 : lds, ds = pos_d ? 1 : ldd;
    for (int c = 0; c < p; ++c) dr[c * ds] = sr[c * ss];
  }
}

__global__ void gather_kernel(int64_t m, const int64_t* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    dst[j] = src[idx[j]];
}

static int64_t wave_grid(int32_t nchunks, int32_t width) {
  // Persistent warps, but only about two levels' worth of them: warps that
  // claim chunks further ahead only poll flags, and their acquire loads
  // compete with the rows being solved for L2 bandwidth.
  constexpr int levels = 2, bps = 4;
  int64_t g = (int64_t)sm_count() * bps;
  const int64_t lvl = ((int64_t)levels * (width > 0 ? width : 1) + kWaveWarps - 1) / kWaveWarps;
  if (lvl < g) g = lvl;
  const int64_t need = ((int64_t)nchunks + kWaveWarps - 1) / kWaveWarps;
  if (need < g) g = need;
  return g < 1 ? 1 : g;
}

}  // namespace rg

extern "C" int64_t rg_wave_workspace_bytes(int64_t n) { return 256 + 4 * (n > 0 ? n : 1); }

// Host-side schedule (runs on the CPU once per factorisation; no numerics).
extern "C" int32_t rg_wave_schedule(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                                    const int32_t* diag_pos, int32_t upper, int32_t chunk_rows, int32_t* order,
                                    int32_t* chunk, int32_t* n_levels, int32_t* width) {
  using namespace rg;
  clear_error();
  if (n < 0 || (n > 0 && (!row_ptr || !col_idx || !diag_pos || !order || !chunk))) {
    set_error("rg_wave_schedule: bad arguments");
    return -1;
  }
  const int32_t cr = chunk_rows >= 32 ? (chunk_rows / 32) * 32 : 32;  // rows per chunk, a multiple of 32
  std::vector<int32_t> lev((size_t)n, 0);
  int32_t maxlev = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = upper ? n - 1 - r : r;
    const int32_t eb = upper ? diag_pos[i] + 1 : row_ptr[i];
    const int32_t ee = upper ? row_ptr[i + 1] : diag_pos[i];
    int32_t l = 0;
    for (int32_t e = eb; e < ee; ++e) l = std::max(l, lev[(size_t)col_idx[e]] + 1);
    lev[(size_t)i] = l;
    maxlev = std::max(maxlev, l);
  }
  const int32_t nl = n > 0 ? maxlev + 1 : 0;
  std::vector<int64_t> start((size_t)nl + 1, 0);
  for (int64_t i = 0; i < n; ++i) ++start[(size_t)lev[(size_t)i] + 1];
  for (int32_t l = 0; l < nl; ++l) start[(size_t)l + 1] += start[(size_t)l];
  std::vector<int64_t> fill(start.begin(), start.end() - (nl > 0 ? 1 : 0));
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = upper ? n - 1 - r : r;  // upper: descending rows within a level
    order[fill[(size_t)lev[(size_t)i]]++] = (int32_t)i;
  }
  int32_t nc = 0, wmax = 0;
  chunk[0] = 0;
  for (int32_t l = 0; l < nl; ++l) {
    const int32_t c0 = nc;
    for (int64_t s = start[(size_t)l]; s < start[(size_t)l + 1]; s += cr)
      chunk[++nc] = (int32_t)std::min<int64_t>(s + cr, start[(size_t)l + 1]);
    wmax = std::max(wmax, nc - c0);
  }
  if (n_levels) *n_levels = nl;
  if (width) *width = wmax;
  return nc;
}

extern "C" int64_t rg_wave_max_chunks(int64_t n) { return n / 32 + n + 2; }  // any chunk_rows >= 32

static rg::Wave make_wave(const int32_t* order, const int32_t* chunk, int32_t nchunks, void* d_work, int32_t epoch) {
  rg::Wave W;
  W.order = order;
  W.chunk = chunk;
  W.nchunks = nchunks;
  W.ticket = (unsigned*)d_work;
  W.flags = (int*)((char*)d_work + 256);
  W.epoch = epoch;
  W.ns_max = 1024u;  // polling back-off cap (ns)
  return W;
}

extern "C" int rg_ilu0_f64(int64_t n, const int32_t* d_row_ptr, const int32_t* d_col_idx, double* d_vals,
                           const int32_t* d_diag_pos, const int32_t* d_order, const int32_t* d_chunk,
                           int32_t nchunks, int32_t width, int64_t* d_zero_row, void* d_work, int64_t work_bytes, int32_t epoch,
                           void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && n < (1ll << 31), "rg_ilu0_f64: n=%lld", (long long)n);
  RG_REQUIRE(n == 0 || (d_row_ptr && d_col_idx && d_vals && d_diag_pos && d_order && d_chunk && d_zero_row),
             "rg_ilu0_f64: null argument");
  RG_REQUIRE(d_work && work_bytes >= rg_wave_workspace_bytes(n), "rg_ilu0_f64: workspace too small");
  RG_REQUIRE(epoch > 0, "rg_ilu0_f64: epoch must be positive");
  if (n == 0) return RG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope prof(s);
  cudaMemsetAsync(d_work, 0, 4, s);
  Wave W = make_wave(d_order, d_chunk, nchunks, d_work, epoch);
  ilu0_kernel<<<(unsigned)wave_grid(nchunks, width), kWaveWarps * 32, 0, s>>>(W, d_row_ptr, d_col_idx, d_vals, d_diag_pos,
                                                                      (long long*)d_zero_row);
  RG_CHECK_LAUNCH("rg_ilu0_f64");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_ilu0 n=%lld", (long long)n);
  return RG_OK;
}

extern "C" int rg_sptrsv_f64(int64_t n, const int32_t* d_row_ptr, const int32_t* d_col_idx, const double* d_vals,
                             const int32_t* d_diag_pos, const int32_t* d_order, const int32_t* d_chunk,
                             int32_t nchunks, int32_t width, int32_t upper, int32_t p, const double* d_b, int64_t ldb, double* d_x,
                             int64_t ldx, void* d_work, int64_t work_bytes, int32_t epoch, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && n < (1ll << 31) && p >= 1 && p <= 64, "rg_sptrsv_f64: n=%lld p=%d (p must be in [1, 64])",
             (long long)n, p);
  RG_REQUIRE(n == 0 || (d_row_ptr && d_col_idx && d_vals && d_diag_pos && d_order && d_chunk && d_b && d_x),
             "rg_sptrsv_f64: null argument");
  RG_REQUIRE(ldb >= n && ldx >= n, "rg_sptrsv_f64: leading dimensions below n");
  RG_REQUIRE(d_work && work_bytes >= rg_wave_workspace_bytes(n), "rg_sptrsv_f64: workspace too small");
  RG_REQUIRE(epoch > 0, "rg_sptrsv_f64: epoch must be positive");
  if (n == 0) return RG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope prof(s);
  cudaMemsetAsync(d_work, 0, 4, s);
  Wave W = make_wave(d_order, d_chunk, nchunks, d_work, epoch);
  const unsigned g = (unsigned)wave_grid(nchunks, width);
  if (upper)
    sptrsv_kernel<true><<<g, kWaveWarps * 32, 0, s>>>(W, d_row_ptr, d_col_idx, d_vals, d_diag_pos, p, d_b, ldb, d_x,
                                                      ldx);
  else
    sptrsv_kernel<false><<<g, kWaveWarps * 32, 0, s>>>(W, d_row_ptr, d_col_idx, d_vals, d_diag_pos, p, d_b, ldb,
                                                       d_x, ldx);
  RG_CHECK_LAUNCH("rg_sptrsv_f64");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_sptrsv upper=%d p=%d", upper, p);
  return RG_OK;
}

// Host: the schedule-ordered copy of one triangle's pattern.  pos[i] = level
// position of row i; rp_out/ci_out = the permuted strictly-lower (upper = 0)
// or strictly-upper (upper = 1) pattern; emap[e'] = original entry index of
// permuted entry e' (values are gathered on the device after factorising).
// Returns the triangle's entry count.
extern "C" int64_t rg_wave_permute(int64_t n, const int32_t* row_ptr, const int32_t* col_idx, const int32_t* diag_pos,
                                   int32_t upper, const int32_t* order, int32_t* pos, int32_t* rp_out, int32_t* ci_out,
                                   int64_t* emap) {
  for (int64_t r = 0; r < n; ++r) pos[order[r]] = (int32_t)r;
  int64_t m = 0;
  rp_out[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = order[r];
    const int32_t eb = upper ? diag_pos[i] + 1 : row_ptr[i];
    const int32_t ee = upper ? row_ptr[i + 1] : diag_pos[i];
    for (int32_t e = eb; e < ee; ++e) {
      ci_out[m] = pos[col_idx[e]];
      emap[m] = e;
      ++m;
    }
    rp_out[r + 1] = (int32_t)m;
  }
  return m;
}

extern "C" int rg_gather_f64(int64_t m, const int64_t* d_idx, const double* d_src, double* d_dst, void* stream) {
  using namespace rg;
  clear_error();
  if (m <= 0) return RG_OK;
  RG_REQUIRE(d_idx && d_src && d_dst, "rg_gather_f64: null argument");
  ProfScope prof((cudaStream_t)stream);
  const int64_t g = std::min<int64_t>((m + 255) / 256, (int64_t)sm_count() * 16);
  gather_kernel<<<(unsigned)g, 256, 0, (cudaStream_t)stream>>>(m, d_idx, d_src, d_dst);
  RG_CHECK_LAUNCH("rg_gather_f64");
  prof.finish(1, 16 * m, 0.0, nullptr, 0, 0, 0, 0, "rg_gather");
  return RG_OK;
}

extern "C" int rg_permute_rows_f64(int64_t n, int32_t p, const double* d_src, int64_t lds, const int32_t* d_pos_src,
                                   double* d_dst, int64_t ldd, const int32_t* d_pos_dst, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && p >= 1, "rg_permute_rows_f64: bad shape");
  if (n == 0) return RG_OK;
  RG_REQUIRE(d_src && d_dst && (d_pos_src || lds >= n) && (d_pos_dst || ldd >= n), "rg_permute_rows_f64: bad args");
  ProfScope prof((cudaStream_t)stream);
  const int64_t g = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  permute_rows_kernel<<<(unsigned)g, 256, 0, (cudaStream_t)stream>>>(n, p, d_src, lds, d_pos_src, d_dst, ldd,
                                                                     d_pos_dst);
  RG_CHECK_LAUNCH("rg_permute_rows_f64");
  prof.finish(1, 16 * n * p, 0.0, nullptr, 0, 0, 0, 0, "rg_permute_rows p=%d", p);
  return RG_OK;
}

extern "C" int rg_sptrsv_perm_f64(int64_t n, const int32_t* d_rp, const int32_t* d_ci, const double* d_vals,
                                  const double* d_dval, const int32_t* d_chunk, int32_t nchunks, int32_t width,
                                  int32_t p, double* d_xw, void* d_work, int64_t work_bytes, int32_t epoch,
                                  void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && n < (1ll << 31) && p >= 1, "rg_sptrsv_perm_f64: n=%lld p=%d", (long long)n, p);
  if (n == 0) return RG_OK;
  RG_REQUIRE(d_rp && d_ci && d_chunk && d_xw, "rg_sptrsv_perm_f64: null argument");
  RG_REQUIRE(d_work && work_bytes >= rg_wave_workspace_bytes(n), "rg_sptrsv_perm_f64: workspace too small");
  RG_REQUIRE(epoch > 0, "rg_sptrsv_perm_f64: epoch must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  ProfScope prof(s);
  cudaMemsetAsync(d_work, 0, 4, s);
  Wave W = make_wave(nullptr, d_chunk, nchunks, d_work, epoch);
  sptrsv_perm_kernel<<<(unsigned)wave_grid(nchunks, width), kWaveWarps * 32, 0, s>>>(W, d_rp, d_ci, d_vals, d_dval,
                                                                                     p, d_xw);
  RG_CHECK_LAUNCH("rg_sptrsv_perm_f64");
  prof.finish(1, 0, 0.0, nullptr, 0, 0, 0, 0, "rg_sptrsv_perm p=%d", p);
  return RG_OK;
}
