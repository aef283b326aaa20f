// Host-side orchestration entry points of the C ABI: the fused CGS2
// projection schedule and CholQR2, expressed as sequences of rg_tall_f64 /
// rg_chol_f64 launches on one stream, so a non-Python host (C, Go via cgo,
// Java via JNI, ...) can run the reference's orthogonalization with single
// calls.  Same schedule as paper_1604_01713_b200/ortho.py:project_chain and
// dense_kernels.py:cholqr2_launch.
//
// Reference: arnoldi.py:171-180 (CGS2 branch of step), dense_kernels.py:31-48
// (reduced_qr).
#include "rg_common.cuh"

#include <vector>

namespace {

struct Basis {
  const double* ptr;
  int64_t ld;
  int32_t cols;
  double* coef;  // cols x p, column-major, device
};

struct Term {
  const double* x;
  int64_t ldx;
  int32_t a;
  const double* s;
};

int tall_call(int64_t n, int32_t p, const double* zin, int64_t ldzin, double* zout, int64_t ldzout,
              const std::vector<Term>& terms, int gmode, const double* gb, int64_t ldgb, int32_t gc, double* gout,
              void* work, int64_t work_bytes, void* stream) {
  Term t1{nullptr, 1, 0, nullptr}, t2{nullptr, 1, 0, nullptr};
  if (terms.size() > 0) t1 = terms[0];
  if (terms.size() > 1) t2 = terms[1];
  return rg_tall_f64(n, p, zin, ldzin, zout, ldzout, t1.x, t1.ldx, t1.a, t1.s, -1.0, t2.x, t2.ldx, t2.a, t2.s,
                     -1.0, nullptr, nullptr, gmode, gb, ldgb, gc, gout, work, work_bytes, stream);
}

}  // namespace

extern "C" int rg_cgs2_f64(int64_t n, int32_t p, double* d_z, int64_t ldz, const double* d_c, int64_t ldc,
                           int32_t k, const double* d_w, int64_t ldw, int32_t w, double* d_coef, double* d_gram,
                           int32_t joint, void* d_work, int64_t work_bytes, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(n >= 0 && p >= 1 && p <= 16, "rg_cgs2_f64: p=%d outside [1, 16]", p);
  RG_REQUIRE(k >= 0 && w >= 0 && (k == 0 || d_c) && (w == 0 || d_w) && d_z && d_coef,
             "rg_cgs2_f64: bad operands");
  // each basis is one Gram operand of rg_tall_f64 (<= 128 columns); wider
  // bases are split by the caller (ortho.project_chain does)
  RG_REQUIRE(k <= 128 && w <= 128, "rg_cgs2_f64: k=%d, w=%d: each basis must have <= 128 columns", k, w);
  // the joint schedule is the caller's explicit choice: adjacency alone can
  // be a coincidence of the allocator, and the schedule assumes C is
  // orthogonal to W (the solver's invariant, not every caller's)
  RG_REQUIRE(!joint || (k > 0 && w > 0 && d_w == d_c + (int64_t)k * ldc && ldw == ldc && k + w <= 128),
             "rg_cgs2_f64: joint schedule needs W directly after C in one allocation (d_w == d_c + k*ldc, "
             "ldw == ldc) and k + w <= 128");
  if (joint) {
    // project against [C W] as one basis (C is orthogonal to W, so this is
    // the same CGS2 up to rounding):
    //   P1  G1 = [C W]^T z
    //   P2  G2 = [C W]^T (z - [C W] G1)
    //   P3  z <- z - [C W] (G1 + G2)  (aliased terms merged), self Gram
    // three passes instead of five.  Coefficients: G1 | G2, each (k+w) x p.
    const int kw = k + w;
    double* G1 = d_coef;
    double* G2 = d_coef + (int64_t)kw * p;
    int rc = tall_call(n, p, d_z, ldz, nullptr, ldz, {}, 1, d_c, ldc, kw, G1, d_work, work_bytes, stream);
    if (rc) return rc;
    rc = tall_call(n, p, d_z, ldz, nullptr, ldz, {{d_c, ldc, kw, G1}}, 1, d_c, ldc, kw, G2, d_work, work_bytes,
                   stream);
    if (rc) return rc;
    return tall_call(n, p, d_z, ldz, d_z, ldz, {{d_c, ldc, kw, G1}, {d_c, ldc, kw, G2}}, d_gram ? 2 : 0, nullptr, 1,
                     p, d_gram, d_work, work_bytes, stream);
  }
  // coefficient blocks S1 | c1 | S2 | c2 packed column-major in d_coef
  std::vector<Basis> bases;
  double* off = d_coef;
  for (int pass = 0; pass < 2; ++pass) {
    if (k) {
      bases.push_back({d_c, ldc, k, off});
      off += (int64_t)k * p;
    }
    if (w) {
      bases.push_back({d_w, ldw, w, off});
      off += (int64_t)w * p;
    }
  }
  // fused schedule: pass i applies the pending updates and forms the next
  // Gram; z is stored when carrying its updates would cost more than p
  // columns or more than two updates would be pending
  std::vector<Term> pending;
  const size_t nb = bases.size();
  for (size_t i = 0; i < nb; ++i) {
    const Basis& B = bases[i];
    const double* next_ptr = i + 1 < nb ? bases[i + 1].ptr : nullptr;
    int carry = 0;
    for (const Term& t : pending)
      if (t.x != B.ptr && t.x != next_ptr) carry += t.a;
    const bool store = pending.size() + 1 > 2 || carry > p;
    const int rc = tall_call(n, p, d_z, ldz, store ? d_z : nullptr, ldz, pending, 1, B.ptr, B.ld, B.cols,
                             B.coef, d_work, work_bytes, stream);
    if (rc) return rc;
    if (store) pending.clear();
    pending.push_back({B.ptr, B.ld, B.cols, B.coef});
  }
  return tall_call(n, p, d_z, ldz, d_z, ldz, pending, d_gram ? 2 : 0, nullptr, 1, p, d_gram, d_work, work_bytes,
                   stream);
}

extern "C" int rg_cholqr2_f64(int64_t n, int32_t p, const double* d_x, int64_t ldx, double* d_q, int64_t ldq,
                              double* d_small, int32_t* d_status, int32_t gram_ready, void* d_work,
                              int64_t work_bytes, void* stream) {
  using namespace rg;
  clear_error();
  RG_REQUIRE(p >= 1 && p <= 16 && n >= p, "rg_cholqr2_f64: need 1 <= p <= 16 and n >= p");
  RG_REQUIRE(d_x && d_q && d_small && d_status && d_x != d_q, "rg_cholqr2_f64: bad operands (Q must not alias X)");
  const int64_t pp = (int64_t)p * p;
  double* G1 = d_small;
  double* R1 = d_small + pp;
  double* G2 = d_small + 2 * pp;
  double* R2 = d_small + 3 * pp;
  const double cond_tol = 1e-11;  // dense_kernels.py CHOL_COND_TOL
  int rc;
  if (!gram_ready) {
    rc = rg_tall_f64(n, p, d_x, ldx, nullptr, 1, nullptr, 1, 0, nullptr, 0.0, nullptr, 1, 0, nullptr, 0.0, nullptr,
                     nullptr, 2, nullptr, 1, p, G1, d_work, work_bytes, stream);
    if (rc) return rc;
  }
  if ((rc = rg_chol_f64(p, G1, R1, d_status, cond_tol, stream))) return rc;
  rc = rg_tall_f64(n, p, d_x, ldx, nullptr, 1, nullptr, 1, 0, nullptr, 0.0, nullptr, 1, 0, nullptr, 0.0, R1,
                   nullptr, 2, nullptr, 1, p, G2, d_work, work_bytes, stream);
  if (rc) return rc;
  if ((rc = rg_chol_f64(p, G2, R2, d_status + 1, cond_tol, stream))) return rc;
  return rg_tall_f64(n, p, d_x, ldx, d_q, ldq, nullptr, 1, 0, nullptr, 0.0, nullptr, 1, 0, nullptr, 0.0, R1, R2, 0,
                     nullptr, 1, 0, nullptr, d_work, work_bytes, stream);
}
