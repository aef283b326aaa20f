// SpMM for matrices whose nonzeros lie on a few diagonals (every stencil
// configuration of BASELINE: configs[0]-[3]), same arithmetic as the CSR
// kernel: Y[i,c] = sum over row i's stored entries in ascending column
// order of a*X[col,c], separately rounded multiply and add, starting at 0.0
// (reference sparse_core.py:25-40) -- bitwise equal to rg_spmm_csr_f64.
//
// Layout (built once per matrix on the device, sparse_core.DiaPlan): the
// values as an n x ndiag column-major block (diagonal d = offset off[d],
// ascending, zero where a row has no entry) and a per-row bit mask of the
// entries the row stores.  Column indices are implied by the offsets, so a
// row block needs no index loads, and X is read as a few contiguous row
// windows instead of gathered:
//
//   one elected producer thread per CTA issues, per 128-row block, one
//   cp.async.bulk.tensor.2d box of X per window of nearby offsets (box
//   {128 + span rows, <= 8 columns}: e.g. {-N^2}, {-N}, {-1, 0, +1}, {+N},
//   {+N^2} for the 7-point stencil), one box of the block's values
//   {128 rows, ndiag} and one of its masks, into a ring of shared-memory
//   stages (mbarrier complete_tx); four consumer warps (lane = row) then
//   accumulate from shared memory.  Two such CTAs per SM (8 consumer warps:
//   with one, the consumers' shared-memory latency, not the memory system,
//   set the pace).  Rows outside [0, n_cols) of a window arrive as zeros
//   (out-of-bounds fill) and are masked off anyway.
//
// Bytes: the values (8 per stored diagonal slot, ~nnz*8) + 4 per row of
// mask + X once + Y once from DRAM -- no 4-byte column index per nonzero.
#include "rg_common.cuh"

#include <cuda.h>

#include <algorithm>
#include <climits>
#include <cstring>

namespace rg {

constexpr int kDiaRows = 128;       // rows per block = 4 consumer warps x 32 lanes
constexpr int kDiaConsumers = kDiaRows / 32;
constexpr int kDiaThreads = (kDiaConsumers + 1) * 32;
constexpr int kDiaMaxDiag = 32;
constexpr int kDiaMaxWin = 8;
constexpr int kDiaMaxStages = 6;
#ifndef RG_DIA_MAX_SPAN
#define RG_DIA_MAX_SPAN 64
#endif
constexpr int kDiaMaxSpan = RG_DIA_MAX_SPAN;  // offsets closer than this share one X window
#ifndef RG_DIA_CTAS
#define RG_DIA_CTAS 2  // 2 x (4 consumer warps + producer) per SM: cfg4 p=8 589 vs 784 us with 1
#endif
constexpr int kDiaCtas = RG_DIA_CTAS;  // CTAs per SM
constexpr size_t kDiaSmem = (kDiaCtas == 1 ? 200 : 100) * 1024;

struct DiaParams {
  int64_t row_base, row_begin, row_end;  // blocks start at row_base (row_begin rounded down to 4)
  double* y;
  int64_t ldy;
  int ndiag, nwin, pc, stages, stage_words;
  unsigned tx;
  int a_soff, m_soff;                 // stage offsets (doubles) of the value tile and the masks
  int off[kDiaMaxDiag];               // ascending diagonal offsets
  int dwin[kDiaMaxDiag];              // window of each diagonal
  int wlo[kDiaMaxWin], wrows[kDiaMaxWin], wsoff[kDiaMaxWin];
};

struct DiaMaps {
  CUtensorMap x[kDiaMaxWin];
  CUtensorMap a, m;
};

__device__ __forceinline__ uint32_t dia_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void dia_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "DIA_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DIA_DONE;\n"
      " bra DIA_WAIT;\n"
      "DIA_DONE:\n}\n" ::"r"(dia_smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void dia_tile(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dia_smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(dia_smem_u32(bar))
      : "memory");
}

template <int PB>
__global__ void __launch_bounds__(kDiaThreads, kDiaCtas)
    spmm_dia_kernel(const __grid_constant__ DiaParams P, const __grid_constant__ DiaMaps M) {
  extern __shared__ __align__(128) double dia_smem[];
  __shared__ __align__(8) uint64_t full[kDiaMaxStages], empty[kDiaMaxStages];
  __shared__ int s_base[kDiaMaxDiag], s_wrows[kDiaMaxDiag];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < P.ndiag) {
    const int d = threadIdx.x, w = P.dwin[d];
    // stage offset of this diagonal's X value for local row 0, column 0
    s_base[d] = P.wsoff[w] + (P.off[d] - P.wlo[w]);
    s_wrows[d] = P.wrows[w];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(dia_smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(dia_smem_u32(&empty[s])), "r"(kDiaConsumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t nblocks = (P.row_end - P.row_base + kDiaRows - 1) / kDiaRows;
  const int64_t mine = (int64_t)blockIdx.x < nblocks ? (nblocks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == kDiaConsumers) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int64_t it = 0; it < mine; ++it) {
        if (it >= P.stages) dia_wait(&empty[s], ph ^ 1u);
        const int r0 = (int)(P.row_base + ((int64_t)blockIdx.x + it * gridDim.x) * kDiaRows);
        double* st = dia_smem + (size_t)s * P.stage_words;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(dia_smem_u32(&full[s])),
                     "r"(P.tx)
                     : "memory");
        // compile-time window indices: a tensor map must be addressed in the
        // kernel-parameter space (a runtime index would copy it to local memory)
#pragma unroll
        for (int w = 0; w < kDiaMaxWin; ++w)
          if (w < P.nwin) dia_tile(st + P.wsoff[w], &M.x[w], r0 + P.wlo[w], 0, &full[s]);
        dia_tile(st + P.a_soff, &M.a, r0, 0, &full[s]);
        dia_tile(st + P.m_soff, &M.m, r0, 0, &full[s]);
        if (++s == P.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  // consumers: lane = row of the block
  const int lr = warp * 32 + lane;
  int s = 0;
  unsigned ph = 0;
  for (int64_t it = 0; it < mine; ++it) {
    dia_wait(&full[s], ph);
    const double* st = dia_smem + (size_t)s * P.stage_words;
    const int64_t row = P.row_base + ((int64_t)blockIdx.x + it * gridDim.x) * kDiaRows + lr;
    const uint32_t mask = reinterpret_cast<const uint32_t*>(st + P.m_soff)[lr];
    const double* sa = st + P.a_soff + lr;
    double acc[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) acc[c] = 0.0;
    for (int d = 0; d < P.ndiag; ++d) {
      if ((mask >> d) & 1u) {
        const double a = sa[d * kDiaRows];
        const double* sx = st + s_base[d] + lr;
        const int ws = s_wrows[d];
#pragma unroll
        for (int c = 0; c < PB; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(a, sx[c * ws]));
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(dia_smem_u32(&empty[s])) : "memory");
    if (row >= P.row_begin && row < P.row_end) {
#pragma unroll
      for (int c = 0; c < PB; ++c) P.y[row + (int64_t)c * P.ldy] = acc[c];
    }
    if (++s == P.stages) {
      s = 0;
      ph ^= 1u;
    }
  }
}

typedef CUresult (*DiaEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static DiaEncodeFn dia_encoder() {
  static DiaEncodeFn fn = []() -> DiaEncodeFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<DiaEncodeFn>(f);
  }();
  return fn;
}

// rows x cols column-major (element size esz, leading dimension ld) as a
// 2-D tensor, box {box_rows, box_cols}
static bool dia_encode(CUtensorMap* m, CUtensorMapDataType dt, int esz, const void* base, int64_t rows, int cols,
                       int64_t ld, int box_rows, int box_cols) {
  DiaEncodeFn enc = dia_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int PB>
static cudaError_t launch_dia(const DiaParams& P, const DiaMaps& M, cudaStream_t st) {
  auto k = spmm_dia_kernel<PB>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiaSmem);
    attr = true;
  }
  const int64_t nblocks = (P.row_end - P.row_base + kDiaRows - 1) / kDiaRows;
  int64_t g = (int64_t)sm_count() * kDiaCtas;
  if (nblocks < g) g = nblocks;
  k<<<(unsigned)g, kDiaThreads, (size_t)P.stages * P.stage_words * sizeof(double), st>>>(P, M);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Building the layout from the CSR arrays on the device (once per matrix;
// sparse_core.DiaPlan).  Pass 1 collects the distinct offsets col - row in a
// 64-slot open-addressed table (after the first warps every lookup is a read
// hit; a matrix with more offsets than slots sets the overflow word and the
// remaining rows return at once).  Pass 2, given the sorted offsets, scatters
// each row's values into the n x ndiag block and ORs its mask.
// ---------------------------------------------------------------------------
constexpr int kDiaTable = 64;
constexpr int kDiaEmpty = INT32_MIN;

__global__ void dia_offsets_kernel(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci, int* table, int* overflow) {
  const int64_t r = row_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= row_end || *reinterpret_cast<volatile int*>(overflow)) return;
  int last = kDiaEmpty;
  for (int e = rp[r]; e < rp[r + 1]; ++e) {
    const int off = ci[e] - (int)r;
    if (off == last) continue;
    last = off;
    unsigned h = ((unsigned)off * 2654435761u) >> 26;  // 6 bits
    int probes = 0;
    for (; probes < kDiaTable; ++probes, h = (h + 1) & (kDiaTable - 1)) {
      int cur = reinterpret_cast<volatile int*>(table)[h];
      if (cur == off) break;
      if (cur == kDiaEmpty) {
        cur = atomicCAS(table + h, kDiaEmpty, off);
        if (cur == kDiaEmpty || cur == off) break;
      }
    }
    if (probes == kDiaTable) {
      *overflow = 1;
      return;
    }
  }
}

__global__ void dia_fill_kernel(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ v, int ndiag,
                                const int32_t* __restrict__ offs, double* __restrict__ dia, int64_t ld,
                                uint32_t* __restrict__ mask) {
  __shared__ int s_off[kDiaMaxDiag];
  if ((int)threadIdx.x < ndiag) s_off[threadIdx.x] = offs[threadIdx.x];
  __syncthreads();
  const int64_t r = row_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= row_end) return;
  uint32_t m = 0;
  int d = 0;
  for (int e = rp[r]; e < rp[r + 1]; ++e) {
    const int off = ci[e] - (int)r;
    // a row's offsets ascend with its column indices: resume the scan at d
    while (d < ndiag && s_off[d] < off) ++d;
    dia[r + (int64_t)d * ld] = v[e];
    m |= 1u << d;
  }
  mask[r] = m;
}

}  // namespace rg

// distinct offsets of rows [row_begin, row_end) into d_table (64 ints, preset
// to INT32_MIN by the caller); *d_overflow (preset 0) becomes 1 when there
// are more
extern "C" int rg_dia_offsets(int64_t n_rows, int64_t row_begin, int64_t row_end, const int32_t* d_rp,
                              const int32_t* d_ci, int32_t* d_table, int32_t* d_overflow, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n_rows >= 0 && 0 <= row_begin && row_begin <= row_end && row_end <= n_rows && d_rp && d_table &&
                 d_overflow,
             "rg_dia_offsets: bad arguments");
  if (row_end == row_begin) return RG_OK;
  dia_offsets_kernel<<<(unsigned)((row_end - row_begin + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      row_begin, row_end, d_rp, d_ci, d_table, d_overflow);
  RG_CHECK_LAUNCH("rg_dia_offsets");
  count_launches(1);
  return RG_OK;
}

// values and masks of rows [row_begin, row_end) of the layout: d_dia (n_rows
// x ndiag, ld, zeroed by the caller), d_mask (n_rows, zeroed); d_offsets = the
// ascending offsets on the device.  Rows outside the range keep mask 0: the
// layout then serves products over sub-ranges of [row_begin, row_end) only
// (the interior rows of a row partition, whose entries are all owned columns)
extern "C" int rg_dia_fill_f64(int64_t n_rows, int64_t row_begin, int64_t row_end, const int32_t* d_rp,
                               const int32_t* d_ci, const double* d_vals, int32_t ndiag, const int32_t* d_offsets,
                               double* d_dia, int64_t ld_dia, uint32_t* d_mask, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n_rows >= 0 && 0 <= row_begin && row_begin <= row_end && row_end <= n_rows && ndiag >= 1 &&
                 ndiag <= kDiaMaxDiag && d_rp && d_offsets && d_dia && d_mask && ld_dia >= n_rows,
             "rg_dia_fill_f64: bad arguments (ndiag=%d)", ndiag);
  if (row_end == row_begin) return RG_OK;
  dia_fill_kernel<<<(unsigned)((row_end - row_begin + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      row_begin, row_end, d_rp, d_ci, d_vals, ndiag, d_offsets, d_dia, ld_dia, d_mask);
  RG_CHECK_LAUNCH("rg_dia_fill_f64");
  count_launches(1);
  return RG_OK;
}

extern "C" int rg_spmm_dia_f64(int64_t n_rows, int64_t row_begin, int64_t row_end, int32_t ndiag,
                               const int32_t* h_offsets, const double* d_dia, int64_t ld_dia,
                               const uint32_t* d_mask, int64_t n_cols, const double* d_x, int64_t ldx, int32_t p,
                               double* d_y, int64_t ldy, const int32_t* d_row_ptr, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n_rows >= 0 && 0 <= row_begin && row_begin <= row_end && row_end <= n_rows,
             "rg_spmm_dia_f64: bad row range [%lld, %lld) of %lld", (long long)row_begin, (long long)row_end,
             (long long)n_rows);
  RG_REQUIRE(ndiag >= 1 && ndiag <= kDiaMaxDiag && h_offsets, "rg_spmm_dia_f64: %d diagonals (1..%d)", ndiag,
             kDiaMaxDiag);
  RG_REQUIRE(p >= 1 && d_dia && d_mask && d_x && d_y && ld_dia >= n_rows && ldx >= n_cols && ldy >= n_rows,
             "rg_spmm_dia_f64: bad arguments");
  RG_REQUIRE(n_rows < INT32_MAX - 2 * kDiaRows && n_cols < INT32_MAX, "rg_spmm_dia_f64: n too large");
  RG_REQUIRE(((uintptr_t)d_dia & 15) == 0 && ((uintptr_t)d_x & 15) == 0 && ((uintptr_t)d_mask & 15) == 0 &&
                 (ld_dia & 1) == 0 && (ldx & 1) == 0,
             "rg_spmm_dia_f64: operands must be 16-byte aligned with even leading dimensions");
  for (int d = 1; d < ndiag; ++d)
    RG_REQUIRE(h_offsets[d] > h_offsets[d - 1], "rg_spmm_dia_f64: offsets must ascend");
  if (row_end == row_begin) return RG_OK;
  // windows: runs of offsets whose span stays within kDiaMaxSpan
  DiaParams P;
  memset(&P, 0, sizeof(P));
  // a tensor box must start on a 16-byte boundary of its innermost
  // dimension (an odd f64 row, or a uint32 row not a multiple of 4, faults
  // with an illegal instruction): blocks start at a multiple of 4 rows, and
  // each X window at an even offset
  P.row_base = row_begin / 4 * 4;
  P.row_begin = row_begin;
  P.row_end = row_end;
  P.ldy = ldy;
  P.ndiag = ndiag;
  int nwin = 0;
  for (int d = 0; d < ndiag; ++d) {
    P.off[d] = h_offsets[d];
    if (nwin == 0 || h_offsets[d] - P.wlo[nwin - 1] > kDiaMaxSpan) {
      RG_REQUIRE(nwin < kDiaMaxWin, "rg_spmm_dia_f64: offsets need more than %d windows", kDiaMaxWin);
      const int o = h_offsets[d];
      P.wlo[nwin++] = o >= 0 ? o / 2 * 2 : -((-o + 1) / 2 * 2);  // even, <= o
    }
    P.dwin[d] = nwin - 1;
    // window rows: block rows + span to its last offset (multiple of 2: 16-byte box rows)
    const int span = h_offsets[d] - P.wlo[nwin - 1];
    P.wrows[nwin - 1] = std::max(P.wrows[nwin - 1], (kDiaRows + span + 1) / 2 * 2);
  }
  P.nwin = nwin;
  ProfScope prof((cudaStream_t)stream);
  cudaStream_t st = (cudaStream_t)stream;
  int launches = 0;
  for (int c0 = 0; c0 < p; c0 += 8) {
    const int pc = std::min(8, p - c0);
    P.pc = pc;
    int words = 0;
    for (int w = 0; w < nwin; ++w) {
      P.wsoff[w] = words;
      words += pc * P.wrows[w];
      words = (words + 15) / 16 * 16;  // 128-byte aligned tiles
    }
    P.a_soff = words;
    words += ndiag * kDiaRows;
    P.m_soff = words;
    words += kDiaRows / 2;  // 128 uint32 masks
    words = (words + 15) / 16 * 16;
    P.stage_words = words;
    P.stages = (int)std::min<size_t>(kDiaMaxStages, kDiaSmem / ((size_t)words * sizeof(double)));
    RG_REQUIRE(P.stages >= 2, "rg_spmm_dia_f64: windows too wide for two stages");
    unsigned tx = 0;
    DiaMaps M;
    memset(&M, 0, sizeof(M));
    const double* X = d_x + (int64_t)c0 * ldx;
    for (int w = 0; w < nwin; ++w) {
      RG_REQUIRE(P.wrows[w] <= 256, "rg_spmm_dia_f64: window of %d rows", P.wrows[w]);
      RG_REQUIRE(dia_encode(&M.x[w], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, X, n_cols, pc, ldx, P.wrows[w], pc),
                 "rg_spmm_dia_f64: tensor map of X window %d", w);
      tx += (unsigned)(P.wrows[w] * pc * 8);
    }
    RG_REQUIRE(dia_encode(&M.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, d_dia, n_rows, ndiag, ld_dia, kDiaRows, ndiag),
               "rg_spmm_dia_f64: tensor map of the values");
    RG_REQUIRE(dia_encode(&M.m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, d_mask, n_rows, 1, (n_rows + 3) / 4 * 4,
                          kDiaRows, 1),
               "rg_spmm_dia_f64: tensor map of the masks");
    tx += (unsigned)(ndiag * kDiaRows * 8 + kDiaRows * 4);
    P.tx = tx;
    P.y = d_y + (int64_t)c0 * ldy;
    cudaError_t e = cudaSuccess;
    switch (pc) {
      case 1: e = launch_dia<1>(P, M, st); break;
      case 2: e = launch_dia<2>(P, M, st); break;
      case 3: e = launch_dia<3>(P, M, st); break;
      case 4: e = launch_dia<4>(P, M, st); break;
      case 5: e = launch_dia<5>(P, M, st); break;
      case 6: e = launch_dia<6>(P, M, st); break;
      case 7: e = launch_dia<7>(P, M, st); break;
      default: e = launch_dia<8>(P, M, st); break;
    }
    if (e != cudaSuccess) {
      set_error("rg_spmm_dia_f64: %s", cudaGetErrorString(e));
      return RG_ECUDA;
    }
    ++launches;
  }
  // bytes: the reference model of the equivalent CSR product (d_row_ptr, if
  // given, supplies the row range's nnz): the same roofline numerator as
  // rg_spmm_csr_f64, although this kernel reads no column indices
  prof.finish(launches, 0, 0.0, d_row_ptr, row_begin, row_end, p, 8, "rg_spmm p=%d (dia)", p);
  return RG_OK;
}
