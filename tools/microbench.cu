// Hardware probes for the design decisions in DESIGN.md: FP64 DMMA vs DFMA
// throughput/latency and streaming-read bandwidth of LDG vs 1-D bulk copies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int K>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[K][2];
  for (int k = 0; k < K; ++k) c[k][0] = c[k][1] = threadIdx.x;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) dmma(c[k][0], c[k][1], a, b);
  double s = 0;
  for (int k = 0; k < K; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[K];
  for (int k = 0; k < K; ++k) c[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) c[k] = fma(c[k], a, b);
  double s = 0;
  for (int k = 0; k < K; ++k) s += c[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_read(const double2* __restrict__ x, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(x + i);
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}

__global__ void k_read_col(const double* __restrict__ x, size_t n, int cols, size_t ld, double* out) {
  // column-major n x cols, thread per row, loads all columns (like tall phase 1)
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
#pragma unroll 8
    for (int c = 0; c < cols; ++c) s += __ldg(x + i + c * ld);
  }
  if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const double* __restrict__ x, size_t n_bytes, int chunk, int stages, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)sm;
  unsigned char* buf = sm + 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // each CTA streams chunks [blockIdx.x + k*grid]; per stage 32 copies of `chunk` bytes
  const size_t per_stage = (size_t)chunk * 32;
  const size_t nst = n_bytes / per_stage;
  double s = 0;
  int it = 0;
  if (threadIdx.x < 32) {
    for (size_t t = blockIdx.x; t < nst; t += gridDim.x, ++it) {
      int st = it % stages;
      if (it >= stages) {
        unsigned par = ((it / stages) - 1) & 1;
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&bar[st])), "r"(par));
      }
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[st])), "r"((unsigned)per_stage));
      __syncwarp();
      const char* src = (const char*)x + t * per_stage + threadIdx.x * (size_t)chunk;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(buf + st * per_stage + threadIdx.x * chunk)), "l"(src), "r"(chunk), "r"(sa(&bar[st])) : "memory");
      s += ((double*)(buf + st * per_stage))[threadIdx.x];
    }
    // drain
    for (int k = 0; k < stages && k < it; ++k) {
      int j = it - 1 - k;
      int st = j % stages;
      unsigned par = (j / stages) & 1;
      asm volatile("{.reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W2;}" ::"r"(sa(&bar[st])), "r"(par));
    }
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 4096;
#define TIME(launch, label, flops)                                   \
  launch; cudaDeviceSynchronize();                                   \
  cudaEventRecord(e0); launch; cudaEventRecord(e1);                  \
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);       \
  printf("%-40s %9.3f ms  %10.2f TFLOP/s\n", label, ms, (flops) / (ms * 1e-3) / 1e12);
  for (int warps : {4, 8, 16}) {
    char lbl[64];
    sprintf(lbl, "dmma K=1 warps/SM=%d", warps);
    TIME((k_dmma<1><<<sms, warps * 32>>>(out, iters, 1.0000001, 0.999)), lbl, 512.0 * iters * 1 * sms * warps);
    sprintf(lbl, "dmma K=8 warps/SM=%d", warps);
    TIME((k_dmma<8><<<sms, warps * 32>>>(out, iters, 1.0000001, 0.999)), lbl, 512.0 * iters * 8 * sms * warps);
    sprintf(lbl, "dfma K=1 warps/SM=%d", warps);
    TIME((k_dfma<1><<<sms, warps * 32>>>(out, iters, 1.0000001, 0.999)), lbl, 2.0 * iters * sms * warps * 32);
    sprintf(lbl, "dfma K=8 warps/SM=%d", warps);
    TIME((k_dfma<8><<<sms, warps * 32>>>(out, iters, 1.0000001, 0.999)), lbl, 2.0 * iters * 8 * sms * warps * 32);
  }
  // latency: single warp chain
  TIME((k_dmma<1><<<1, 32>>>(out, iters, 1.0000001, 0.999)), "dmma chain 1 warp (latency)", 512.0 * iters);
  printf("   -> dmma latency ~ %.1f ns per dependent op\n", ms * 1e6 / iters);
  TIME((k_dfma<1><<<1, 32>>>(out, iters, 1.0000001, 0.999)), "dfma chain 1 warp (latency)", 64.0 * iters);
  printf("   -> dfma latency ~ %.1f ns per dependent op\n", ms * 1e6 / iters);

  size_t bytes = (size_t)8 << 30;  // 8 GiB
  double* x;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 0, bytes);
#define BW(launch, label, b)                                         \
  launch; cudaDeviceSynchronize();                                   \
  cudaEventRecord(e0); launch; cudaEventRecord(e1);                  \
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);       \
  printf("%-40s %9.3f ms  %10.1f GB/s\n", label, ms, (b) / (ms * 1e-3) / 1e9);
  for (int bpsm : {4, 8, 16}) {
    char lbl[64];
    sprintf(lbl, "ldg double2 %d CTA/SM x256", bpsm);
    BW((k_read<<<sms * bpsm, 256>>>((const double2*)x, bytes / 16, out)), lbl, (double)bytes);
  }
  for (int cols : {8, 28, 108}) {
    char lbl[64];
    size_t n = bytes / 8 / cols;
    sprintf(lbl, "ldg column-major thread/row cols=%d", cols);
    BW((k_read_col<<<sms * 8, 256>>>(x, n, cols, n, out)), lbl, (double)n * cols * 8);
  }
  for (int chunk : {512, 1024, 2048, 4096}) {
    for (int stages : {2, 4}) {
      size_t smem = 128 + (size_t)stages * chunk * 32;
      if (smem > 220 * 1024) continue;
      cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      char lbl[64];
      sprintf(lbl, "bulk copy chunk=%d stages=%d 1CTA/SM", chunk, stages);
      BW((k_bulk<<<sms, 32, smem>>>(x, bytes, chunk, stages, out)), lbl, (double)(bytes / (chunk * 32) * (chunk * 32)));
      if (smem * 2 <= 220 * 1024) {
        sprintf(lbl, "bulk copy chunk=%d stages=%d 2CTA/SM", chunk, stages);
        BW((k_bulk<<<sms * 2, 32, smem>>>(x, bytes, chunk, stages, out)), lbl, (double)(bytes / (chunk * 32) * (chunk * 32)));
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
