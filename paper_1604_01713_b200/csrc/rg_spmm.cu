// CSR sparse-matrix times column-major block (K1 of the hot path).
//
// Reference: recgmres.sparse_core._spmm_kernel
// (/root/reference/pkg/src/recgmres/sparse_core.py:25-40): rows outer,
// nonzeros in ascending storage order, columns inner, each Y[i,c] starting
// from 0.0 and updated as Y += a*x with a separately rounded multiply and
// add.  This kernel keeps exactly that per-(row, column) operation sequence
// (__dmul_rn / __dadd_rn, no contraction), so its output is bitwise equal to
// the reference.
//
// B200 mapping: one thread per row (rows are short: 5..27 nonzeros for the
// stencil configs), a warp owns 32 consecutive rows.  The warp stages its
// rows' col_idx/values through shared memory with fully coalesced loads
// (a row-per-thread walk of CSR would otherwise hit every sector ~7 times
// through L1), then each lane walks its own row from shared memory and
// gathers X columns; for banded/stencil matrices neighbouring lanes gather
// neighbouring rows of X, so every X access of the warp is one 256-byte
// coalesced segment per column.  p accumulators live in registers; wide
// blocks are processed in column passes of at most 8.
#include "rg_common.cuh"

#include <cstdlib>

// A/B build switch (tools/ab_build.py): RG_SPMM_COLS=0 keeps single-column
// blocks on the entry-outer loop.  (A row-major X, one 64-byte gather per
// entry at p = 8, measured 1185 vs 819 us at cfg4 -- tools/ab_spmm.py,
// profiles/spmm_r02.txt -- and was dropped.)
#ifndef RG_SPMM_COLS
#define RG_SPMM_COLS 1
#endif

namespace rg {

constexpr int kSpmmWarps = 8;     // 256 threads per CTA
constexpr int kSpmmChunk = 256;   // staged nonzeros per warp per round

// ----------------------------------------------------------------------------
// Persistent kernel: warps loop over 32-row units; the
// CSR entries of the next unit stream into a per-warp double buffer with
// cp.async while the current unit gathers X, and row_ptr is loaded two units
// ahead, so a unit's only exposed latency is its X gathers (mostly L2 hits).
// Units whose 32 rows hold more than kSpmmChunk nonzeros take the chunked
// synchronous path.  Arithmetic and order are the reference's (see top).
// ----------------------------------------------------------------------------

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

struct UnitRp {
  int32_t wbeg, wend, mybeg, myend;
};

template <int RPW = 32>
__device__ __forceinline__ UnitRp load_unit_rp(const int32_t* __restrict__ rp, int64_t wrow0, int64_t row_end,
                                               int lane) {
  UnitRp u;
  const int64_t wlast = min(wrow0 + RPW, row_end);
  const int64_t i = wrow0 + lane % RPW;
  u.wbeg = __ldg(rp + wrow0);
  u.wend = __ldg(rp + wlast);
  u.mybeg = i < row_end ? __ldg(rp + i) : 0;
  u.myend = i < row_end ? __ldg(rp + i + 1) : 0;
  return u;
}

template <int PB, bool GHOST>
__device__ __forceinline__ void accumulate_rows(const int32_t* sci, const double* sva, int lo, int hi,
                                                const double* __restrict__ X, int64_t ldx, int64_t n_local,
                                                const double* __restrict__ Xg, int64_t ldg, double (&acc)[PB]) {
  double xn[PB];
  double an = 0.0;
  auto gather = [&](int t, double (&xv)[PB]) {
    const int64_t j = sci[t];
    const double* xp = X + j;
    int64_t ld = ldx;
    if (GHOST && j >= n_local) {
      xp = Xg + (j - n_local);
      ld = ldg;
    }
#pragma unroll
    for (int c = 0; c < PB; ++c) xv[c] = __ldg(xp + c * ld);
  };
  if (lo < hi) {
    an = sva[lo];
    gather(lo, xn);
  }
  for (int t = lo; t < hi; ++t) {
    double xc[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) xc[c] = xn[c];
    const double ac = an;
    if (t + 1 < hi) {
      an = sva[t + 1];
      gather(t + 1, xn);
    }
#pragma unroll
    for (int c = 0; c < PB; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(ac, xc[c]));
  }
}

// Column-outer accumulation (single-column blocks; measured on B200, cfg4
// 256^3 p = 1: 311 vs 374 us, tools/ab_spmm.py -- for p >= 4 it is 1.5-3x
// slower than the entry-outer loop): a lane loads up to kSpmmU of its row's
// staged entries (index, value) into registers once, then gathers those
// entries' X values two columns at a time -- 2*kSpmmU independent loads in
// flight per lane instead of one entry's PB -- and adds them in storage
// order.  Per (row, column) the operation sequence is still the reference's
// (t ascending, separately rounded product and sum), so the output is
// bitwise the same.
constexpr int kSpmmU = 8;

template <int PB, bool GHOST>
__device__ __forceinline__ void accumulate_cols(const int32_t* sci, const double* sva, int lo, int hi,
                                                const double* __restrict__ X, int64_t ldx, int64_t n_local,
                                                const double* __restrict__ Xg, int64_t ldg, double (&acc)[PB]) {
  for (int t0 = lo; t0 < hi; t0 += kSpmmU) {
    const int cnt = min(kSpmmU, hi - t0);
    int32_t j[kSpmmU];
#pragma unroll
    for (int u = 0; u < kSpmmU; ++u) j[u] = u < cnt ? sci[t0 + u] : 0;
    const double* a = sva + t0;  // values re-read from shared memory per column pair
#pragma unroll
    for (int c = 0; c < PB; c += 2) {
      double x0[kSpmmU], x1[kSpmmU];
      const double* X0 = X + (int64_t)c * ldx;
      const double* X1 = X0 + ldx;
#pragma unroll
      for (int u = 0; u < kSpmmU; ++u) {
        if (u < cnt) {
          if (GHOST && j[u] >= n_local) {
            const double* g = Xg + (j[u] - n_local) + (int64_t)c * ldg;
            x0[u] = __ldg(g);
            if (c + 1 < PB) x1[u] = __ldg(g + ldg);
          } else {
            x0[u] = __ldg(X0 + j[u]);
            if (c + 1 < PB) x1[u] = __ldg(X1 + j[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kSpmmU; ++u) {
        if (u < cnt) {
          acc[c] = __dadd_rn(acc[c], __dmul_rn(a[u], x0[u]));
          if (c + 1 < PB) acc[c + 1] = __dadd_rn(acc[c + 1], __dmul_rn(a[u], x1[u]));
        }
      }
      // keep the next column pair's gathers behind this one (the compiler
      // would otherwise hoist all PB*kSpmmU loads and spill)
      asm volatile("" ::: "memory");
    }
  }
}

template <int PB, bool GHOST>
__device__ __forceinline__ void accumulate_unit(const int32_t* sci, const double* sva, int lo, int hi,
                                                const double* __restrict__ X, int64_t ldx, int64_t n_local,
                                                const double* __restrict__ Xg, int64_t ldg, double (&acc)[PB]) {
  if (RG_SPMM_COLS && PB == 1)
    accumulate_cols<PB, GHOST>(sci, sva, lo, hi, X, ldx, n_local, Xg, ldg, acc);
  else
    accumulate_rows<PB, GHOST>(sci, sva, lo, hi, X, ldx, n_local, Xg, ldg, acc);
}

// CTAs per SM the register budget is sized for: 3 (85 registers) spills at
// PB >= 6, and the spill traffic costs more than the extra warps buy
// (cfg4 p = 8: 912 us with 3, 824 us with 2; profiles/spmm_r01.txt)
template <int PB, int G>
struct SpmmMinBlocks {
  static constexpr int value = PB >= 6 ? 2 : (G > 1 ? 4 : 3);
};

// G lanes share a row (each owns PB of the G*PB columns); units are 32/G rows.
template <int PB, bool GHOST, int G = 1, int CH = kSpmmChunk>
__global__ void __launch_bounds__(kSpmmWarps * 32, SpmmMinBlocks<PB, G>::value)
spmm_persist_kernel(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ rp,
                    const int32_t* __restrict__ ci, const double* __restrict__ va,
                    const double* __restrict__ X, int64_t ldx, int64_t n_local,
                    const double* __restrict__ Xg, int64_t ldg, double* __restrict__ Y, int64_t ldy) {
  constexpr int RPW = 32 / G;
  __shared__ int32_t s_ci[kSpmmWarps][2][CH];
  __shared__ double s_va[kSpmmWarps][2][CH];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int cg = lane / RPW;
  X += (int64_t)cg * PB * ldx;
  if (GHOST) Xg += (int64_t)cg * PB * ldg;
  Y += (int64_t)cg * PB * ldy;
  const int64_t nunits = (row_end - row_begin + RPW - 1) / RPW;
  const int64_t nwarps = (int64_t)gridDim.x * kSpmmWarps;
  int64_t u = (int64_t)blockIdx.x * kSpmmWarps + w;
  if (u >= nunits) return;

  auto issue_csr = [&](const UnitRp& r, int buf) {
    const int32_t cnt = r.wend - r.wbeg;
    if (cnt <= CH) {
      for (int e = lane; e < cnt; e += 32) {
        cp_async4(&s_ci[w][buf][e], ci + r.wbeg + e);
        cp_async8(&s_va[w][buf][e], va + r.wbeg + e);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  UnitRp cur = load_unit_rp<RPW>(rp, row_begin + u * RPW, row_end, lane);
  issue_csr(cur, 0);
  UnitRp nxt = cur;
  if (u + nwarps < nunits) nxt = load_unit_rp<RPW>(rp, row_begin + (u + nwarps) * RPW, row_end, lane);
  int buf = 0;
  for (; u < nunits; u += nwarps) {
    const bool has_next = u + nwarps < nunits;
    // CSR of this unit has landed; start the next unit's CSR and row_ptr
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    if (has_next) issue_csr(nxt, buf ^ 1);
    UnitRp nn = nxt;
    if (u + 2 * nwarps < nunits) nn = load_unit_rp<RPW>(rp, row_begin + (u + 2 * nwarps) * RPW, row_end, lane);

    const int64_t wrow0 = row_begin + u * RPW;
    const int64_t i = wrow0 + lane % RPW;
    double acc[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) acc[c] = 0.0;
    const int32_t cnt = cur.wend - cur.wbeg;
    if (cnt <= CH) {
      accumulate_unit<PB, GHOST>(s_ci[w][buf], s_va[w][buf], cur.mybeg - cur.wbeg, cur.myend - cur.wbeg, X, ldx,
                                 n_local, Xg, ldg, acc);
    } else {
      // long rows: chunked synchronous staging through this unit's buffer
      int32_t* sci = s_ci[w][buf];
      double* sva = s_va[w][buf];
      for (int32_t base = cur.wbeg; base < cur.wend; base += CH) {
        const int32_t c2 = min(CH, cur.wend - base);
        __syncwarp();
        for (int e = lane; e < c2; e += 32) {
          sci[e] = __ldg(ci + base + e);
          sva[e] = __ldg(va + base + e);
        }
        __syncwarp();
        const int lo = max(cur.mybeg, base) - base;
        const int hi = min(cur.myend, base + c2) - base;
        accumulate_unit<PB, GHOST>(sci, sva, lo, hi, X, ldx, n_local, Xg, ldg, acc);
      }
    }
    if (i < row_end) {
#pragma unroll
      for (int c = 0; c < PB; ++c) Y[i + c * ldy] = acc[c];
    }
    __syncwarp();
    cur = nxt;
    nxt = nn;
    buf ^= 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <int PB>
static void launch_spmm(int64_t rb, int64_t re, const int32_t* rp, const int32_t* ci,
                        const double* va, const double* X, int64_t ldx, int64_t n_local,
                        const double* Xg, int64_t ldg, double* Y, int64_t ldy, cudaStream_t s) {
  const int64_t rows = re - rb;
  const int64_t grid = (rows + kSpmmWarps * 32 - 1) / (kSpmmWarps * 32);
  static int per_sm[2] = {-1, -1};
  const int gi = Xg ? 1 : 0;
  if (per_sm[gi] < 0) {
    int v = 0;
    if (Xg)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, spmm_persist_kernel<PB, true>, kSpmmWarps * 32, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, spmm_persist_kernel<PB, false>, kSpmmWarps * 32, 0);
    per_sm[gi] = v < 1 ? 1 : v;
  }
  int64_t g = (int64_t)sm_count() * per_sm[gi];
  if (grid < g) g = grid;
  if (g < 1) g = 1;
  if (Xg)
    spmm_persist_kernel<PB, true><<<(unsigned)g, kSpmmWarps * 32, 0, s>>>(rb, re, rp, ci, va, X, ldx, n_local,
                                                                        Xg, ldg, Y, ldy);
  else
    spmm_persist_kernel<PB, false><<<(unsigned)g, kSpmmWarps * 32, 0, s>>>(rb, re, rp, ci, va, X, ldx, n_local,
                                                                         Xg, ldg, Y, ldy);
}

}  // namespace rg

extern "C" int rg_spmm_csr_f64(int64_t n_rows, int64_t row_begin, int64_t row_end,
                               const int32_t* d_row_ptr, const int32_t* d_col_idx,
                               const double* d_vals, const double* d_x, int64_t ldx,
                               int64_t n_local, const double* d_xg, int64_t ldg,
                               int32_t p, double* d_y, int64_t ldy, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n_rows >= 0 && 0 <= row_begin && row_begin <= row_end && row_end <= n_rows,
             "rg_spmm_csr_f64: bad row range [%lld, %lld) of %lld", (long long)row_begin,
             (long long)row_end, (long long)n_rows);
  RG_REQUIRE(p >= 1, "rg_spmm_csr_f64: block width p=%d must be >= 1", p);
  RG_REQUIRE(d_row_ptr && d_y, "rg_spmm_csr_f64: null row_ptr / output");
  RG_REQUIRE(ldy >= n_rows && ldy >= 1, "rg_spmm_csr_f64: ldy=%lld < n_rows=%lld",
             (long long)ldy, (long long)n_rows);
  RG_REQUIRE(n_local >= 0 && (n_local == 0 || (d_x && ldx >= n_local)),
             "rg_spmm_csr_f64: ldx=%lld < n_local=%lld", (long long)ldx, (long long)n_local);
  if (row_end == row_begin) return RG_OK;
  ProfScope prof((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  // exact-width passes (no per-column predication in the inner loop) of at
  // most 8 columns: a 16-wide register block spills, and re-reading A for a
  // second 8-wide pass is cheaper (profiles/spmm_r01.txt)
  for (int c0 = 0; c0 < p;) {
    const int rem = p - c0;
    const int pc = rem >= 8 ? 8 : rem;
    const double* X = d_x ? d_x + (int64_t)c0 * ldx : nullptr;
    const double* Xg = d_xg ? d_xg + (int64_t)c0 * ldg : nullptr;
    double* Y = d_y + (int64_t)c0 * ldy;
    switch (pc) {
      case 1: launch_spmm<1>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 2: launch_spmm<2>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 3: launch_spmm<3>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 4: launch_spmm<4>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 5: launch_spmm<5>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 6: launch_spmm<6>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      case 7: launch_spmm<7>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
      default: launch_spmm<8>(row_begin, row_end, d_row_ptr, d_col_idx, d_vals, X, ldx, n_local, Xg, ldg, Y, ldy, s); break;
    }
    RG_CHECK_LAUNCH("rg_spmm_csr_f64");
    c0 += pc;
  }
  prof.finish((p + 7) / 8, 0, 0.0, d_row_ptr, row_begin, row_end, p, 8, "rg_spmm p=%d", p);
  return RG_OK;
}
