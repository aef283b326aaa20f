// TMA streaming rate vs box shape: one CTA per SM streams an n x C
// column-major f64 block (C = 112, the P2 stage width) through a ring of
// shared-memory stages filled by cp.async.bulk.tensor, consumers only wait
// and release.  Shapes:
//   3d8   {8 rows, C, row groups}, strides {ld*8, 64}: [group][col][8]  (64-B inner rows)
//   2dR   {R rows, C}, plain column-major tile [col][R]  (R*8-byte inner rows), R in {16, 32, 64, 128, 256}
//   sw128 {16 rows, C} with SWIZZLE_128B, 4 requests per 64-row stage
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_bw tools/tma_bw.cu && tools/tma_bw
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "W1:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra D1;\n"
      " bra W1;\n"
      "D1:\n}\n" ::"r"(su(b)),
      "r"(ph)
      : "memory");
}

// mode 0: 3-D {8, C, groups}; mode 1: 2-D {R, C} x (64/R... stage rows / R) requests
__global__ void stream(const __grid_constant__ CUtensorMap m, int mode, int64_t units, int stage_rows, int box_rows,
                       int stage_bytes, int nst, double* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su(&empty[s])), "r"(blockDim.x / 32 - 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t my = (int64_t)blockIdx.x < units ? (units - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  double acc = 0;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int64_t it = 0; it < my; ++it) {
        if (it >= nst) wait(&empty[s], ph ^ 1u);
        const int64_t u = blockIdx.x + it * gridDim.x;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su(&full[s])), "r"(stage_bytes)
                     : "memory");
        unsigned char* dst = sm + (size_t)s * stage_bytes;
        if (mode == 0) {
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
              "%4}], [%5];\n" ::"r"(su(dst)),
              "l"(&m), "r"(0), "r"(0), "r"((int)(u * stage_rows / 8)), "r"(su(&full[s]))
              : "memory");
        } else {
          const int nreq = stage_rows / box_rows;
          for (int q = 0; q < nreq; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];\n" ::"r"(su(dst + (size_t)q * (stage_bytes / nreq))),
                "l"(&m), "r"((int)(u * stage_rows + q * box_rows)), "r"(0), "r"(su(&full[s]))
                : "memory");
        }
        if (++s == nst) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else {
    int s = 0;
    unsigned ph = 0;
    for (int64_t it = 0; it < my; ++it) {
      wait(&full[s], ph);
      acc += *(const double*)(sm + (size_t)s * stage_bytes + lane * 8 + (warp - 1) * 256);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su(&empty[s])) : "memory");
      if (++s == nst) {
        s = 0;
        ph ^= 1u;
      }
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 1 << 24, ld = n;
  const int C = 112;
  double* d;
  cudaMalloc(&d, (size_t)ld * C * 8);
  cudaMemset(d, 0, (size_t)ld * C * 8);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg {
    const char* name;
    int mode, box_rows, stage_rows;
    CUtensorMapSwizzle sw;
  } cfgs[] = {
      {"3d8 (64-B inner) 64-row stage", 0, 8, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"2d16 sw128 x4 64-row stage", 1, 16, 64, CU_TENSOR_MAP_SWIZZLE_128B},
      {"2d16 x4 64-row stage", 1, 16, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"2d32 x2 64-row stage", 1, 32, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"2d64 x1 64-row stage", 1, 64, 64, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"2d128 x1 128-row stage", 1, 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE},
      {"2d256 x1 256-row stage (56 cols)", 1, 256, 256, CU_TENSOR_MAP_SWIZZLE_NONE},
  };
  for (auto& c : cfgs) {
    CUtensorMap m;
    int cols = C;
    if (c.stage_rows == 256) cols = 56;
    CUresult r;
    if (c.mode == 0) {
      cuuint64_t dims[3] = {8, (cuuint64_t)cols, (cuuint64_t)(n / 8)};
      cuuint64_t st[2] = {(cuuint64_t)ld * 8, 64};
      cuuint32_t box[3] = {8, (cuuint32_t)cols, 8};
      cuuint32_t es[3] = {1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)cols};
      cuuint64_t st[1] = {(cuuint64_t)ld * 8};
      cuuint32_t box[2] = {(cuuint32_t)c.box_rows, (cuuint32_t)cols};
      cuuint32_t es[2] = {1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      printf("%-36s encode error %d\n", c.name, (int)r);
      continue;
    }
    const int stage_bytes = c.stage_rows * cols * 8;
    int nst = (220 * 1024) / stage_bytes;
    if (nst > 8) nst = 8;
    const int64_t units = n / c.stage_rows;
    for (int warm = 0; warm < 2; ++warm) stream<<<nsm, 9 * 32, nst * stage_bytes>>>(m, c.mode, units, c.stage_rows, c.box_rows, stage_bytes, nst, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i)
      stream<<<nsm, 9 * 32, nst * stage_bytes>>>(m, c.mode, units, c.stage_rows, c.box_rows, stage_bytes, nst, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-36s stages %d x %6d B: %.3f ms  %.0f GB/s  %s\n", c.name, nst, stage_bytes, ms,
           (double)n * cols * 8 / ms / 1e6, cudaGetErrorString(err));
  }
  return 0;
}
