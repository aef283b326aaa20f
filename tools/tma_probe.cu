// Probe: can a cp.async.bulk.tensor 3-D map with non-monotonic strides
// ({8 rows, columns, row groups} with byte strides {ld*8, 64}) load a
// 64-row x C-column tile of a column-major f64 block into shared memory as
// [row group][column][8 rows]?  Prints the encode status and checks the
// landed layout element by element (rows past n and columns past ncols must
// arrive as zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_probe tools/tma_probe.cu && /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap m, double* out, int words, int rg0) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(words * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"((uint32_t)__cvta_generic_to_shared(sm)),
        "l"(&m), "r"(0), "r"(0), "r"(rg0), "r"(b)
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred P1;\n"
      "W1:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      " @P1 bra D1;\n"
      " bra W1;\n"
      "D1:\n}\n" ::"r"(b)
      : "memory");
  for (int e = threadIdx.x; e < words; e += blockDim.x) out[e] = sm[e];
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess || !fp) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  EncodeFn enc = (EncodeFn)fp;
  const int64_t n = 1000, ld = 1024;  // n % 8 == 0; rows 1000.. are padding
  const int ncols = 13, bc = 16, rgs = 8;
  std::vector<double> h(ld * ncols);
  for (int c = 0; c < ncols; ++c)
    for (int64_t r = 0; r < ld; ++r) h[r + c * ld] = r < n ? (double)(r * 100 + c + 1) : 1e300;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int words = 8 * bc * rgs;
  cudaMalloc(&o, words * 8);
  CUtensorMap m;
  cuuint64_t dims[3] = {8, (cuuint64_t)ncols, (cuuint64_t)(n / 8)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, 64};
  cuuint32_t box[3] = {8, (cuuint32_t)bc, (cuuint32_t)rgs};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 3d {8, cols, n/8} strides {ld*8, 64}: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 2;
  int bad = 0;
  for (int rg0 : {0, 120}) {  // the second tile has 5 valid row groups (rows 960..999)
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 8);
    probe<<<1, 128, words * 8>>>(m, o, words, rg0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("kernel: %s\n", cudaGetErrorString(e));
      return 3;
    }
    std::vector<double> g(words);
    cudaMemcpy(g.data(), o, words * 8, cudaMemcpyDeviceToHost);
    for (int gg = 0; gg < rgs; ++gg)
      for (int c = 0; c < bc; ++c)
        for (int rr = 0; rr < 8; ++rr) {
          const int64_t row = (int64_t)(rg0 + gg) * 8 + rr;
          const double want = (c < ncols && row < n) ? (double)(row * 100 + c + 1) : 0.0;
          const double got = g[(gg * bc + c) * 8 + rr];
          if (got != want && bad++ < 5) printf("rg0=%d g=%d c=%d r=%d got %g want %g\n", rg0, gg, c, rr, got, want);
        }
  }
  printf("layout [row group][column][8 rows]: %s (%d mismatches)\n", bad ? "FAIL" : "ok", bad);
  return bad ? 4 : 0;
}
