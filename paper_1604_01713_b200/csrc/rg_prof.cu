// Native launch accounting and per-launch device timing.
//
// Every entry point that launches kernels reports, once per call, how many
// kernels it launched, its algorithmic bytes (each distinct
// input read once, each output written once) and its FP64 tensor-core flops.
// The launch counter is always on.  With rg_profile_enable(1) each such call
// is also bracketed by two CUDA events recorded on the call's own stream, so
// a host can attribute device time per launch inside a timed region WITHOUT
// leaving the production path: the orchestrators (rg_cgs2_f64,
// rg_cholqr2_f64) record through the rg_tall_f64 / rg_chol_f64 calls they
// make.  Records are read back after the region (rg_profile_record
// synchronises on the record's end event).
#include "rg_common.cuh"

#include <atomic>
#include <mutex>
#include <string.h>
#include <vector>

namespace rg {

namespace {

struct Rec {
  cudaEvent_t e0, e1;
  char label[112];
  int64_t bytes;
  double flops;
  int launches;
  // SpMM byte model needs nnz of the row range: read from the device lazily
  const int32_t* rp;
  int64_t rb, re;
  int p, esz;
};

std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::atomic<long long> g_launches{0};

cudaEvent_t ev_get() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

ProfScope::ProfScope(cudaStream_t s) : st_(s), e0_(nullptr) {
  if (!g_on) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  e0_ = ev_get();
  cudaEventRecord((cudaEvent_t)e0_, s);
}

ProfScope::~ProfScope() {
  if (e0_) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_pool.push_back((cudaEvent_t)e0_);
  }
}

void ProfScope::finish(int launches, int64_t bytes, double flops, const int32_t* rp, int64_t rb, int64_t re, int p,
                       int esz, const char* fmt, ...) {
  g_launches += launches;
  if (!e0_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  Rec r;
  r.e0 = (cudaEvent_t)e0_;
  e0_ = nullptr;
  r.e1 = ev_get();
  cudaEventRecord(r.e1, st_);
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(r.label, sizeof(r.label), fmt, ap);
  va_end(ap);
  r.bytes = bytes;
  r.flops = flops;
  r.launches = launches;
  r.rp = rp;
  r.rb = rb;
  r.re = re;
  r.p = p;
  r.esz = esz;
  g_recs.push_back(r);
}

void count_launches(int n) { g_launches += n; }

}  // namespace rg

extern "C" void rg_profile_enable(int32_t on) {
  using namespace rg;
  std::lock_guard<std::mutex> lk(g_mu);
  for (Rec& r : g_recs) {
    g_pool.push_back(r.e0);
    g_pool.push_back(r.e1);
  }
  g_recs.clear();
  g_on = on != 0;
}

extern "C" int64_t rg_launch_count(void) { return rg::g_launches.load(); }

extern "C" void rg_count_launches(int64_t n) { rg::g_launches += n; }

extern "C" int32_t rg_profile_count(void) {
  std::lock_guard<std::mutex> lk(rg::g_mu);
  return (int32_t)rg::g_recs.size();
}

extern "C" int rg_profile_record(int32_t i, char* label, int32_t label_cap, double* ms, int64_t* bytes,
                                 double* flops, int32_t* launches) {
  using namespace rg;
  clear_error();
  Rec r;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    RG_REQUIRE(i >= 0 && i < (int32_t)g_recs.size(), "rg_profile_record: index %d of %d", i, (int)g_recs.size());
    r = g_recs[i];
  }
  cudaError_t e = cudaEventSynchronize(r.e1);
  if (e != cudaSuccess) {
    set_error("rg_profile_record: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  float t = 0.f;
  cudaEventElapsedTime(&t, r.e0, r.e1);
  if (ms) *ms = t;
  int64_t b = r.bytes;
  if (r.rp) {
    int32_t ends[2] = {0, 0};
    cudaMemcpy(&ends[0], r.rp + r.rb, sizeof(int32_t), cudaMemcpyDeviceToHost);
    cudaMemcpy(&ends[1], r.rp + r.re, sizeof(int32_t), cudaMemcpyDeviceToHost);
    const int64_t nnz = (int64_t)ends[1] - ends[0], rows = r.re - r.rb;
    b = nnz * (r.esz + 4) + (rows + 1) * 4 + 2 * (int64_t)r.p * rows * r.esz;
  }
  if (bytes) *bytes = b;
  if (flops) *flops = r.flops;
  if (launches) *launches = r.launches;
  if (label && label_cap > 0) {
    strncpy(label, r.label, (size_t)label_cap - 1);
    label[label_cap - 1] = 0;
  }
  return RG_OK;
}

// device time between the end of record i-1 and the start of record i: torch
// plumbing between library calls plus idle time (host latency) -- the
// timeline gaps tools/prof_gaps.py attributes to solver phases
extern "C" int rg_profile_gap(int32_t i, double* ms) {
  using namespace rg;
  clear_error();
  cudaEvent_t a, b;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    RG_REQUIRE(i >= 1 && i < (int32_t)g_recs.size(), "rg_profile_gap: index %d of %d", i, (int)g_recs.size());
    a = g_recs[i - 1].e1;
    b = g_recs[i].e0;
  }
  cudaError_t e = cudaEventSynchronize(b);
  float t = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&t, a, b);
  if (e != cudaSuccess) {
    set_error("rg_profile_gap: %s", cudaGetErrorString(e));
    return RG_ECUDA;
  }
  *ms = t;
  return RG_OK;
}
