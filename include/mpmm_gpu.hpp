// mpmm_gpu.hpp -- C++ drop-in binding of the reference's MP matmul / LU entry points
// to the B200 C-ABI (mpgpu.h).  Header-only; include AFTER the reference's own
// umbrella header (mpmm/mpmm.hpp, which brings mpfr.h and the mpmm types):
//
//     #include "mpmm/mpmm.hpp"
//     #include "mpmm_gpu.hpp"      // link with -lmpgpu
//
// Every function keeps the reference signature and semantics (namespace mpmm::gpu):
//   simple_mul   matrix.hpp:178-184     block_mul     matrix.hpp:225-233
//   add / sub    matrix.hpp:166-175     mat_vec_mul   matrix.hpp:282-297
//   fast_mul     fastmm.hpp:244-255     lu_blocked    blocklu.hpp:121-146
//   lu_columnwise blocklu.hpp:107-112   lu_solve      blocklu.hpp:215-245
//   solve / solve_columnwise            blocklu.hpp:248-259
// A maintainer switches a translation unit to the GPU path with
//     namespace mpmm { using namespace mpmm::gpu; }   // or call mpmm::gpu:: explicitly
// Results are bit-identical to the reference (same operation DAG, MPFR_RNDN rounding).
// Documented deviations: operands of one call must share one precision <= MPGPU_MAX_PREC (9216) bits
// (DomainError otherwise), and NaN/Inf inputs are rejected with DomainError.
//
// Multi-GPU (SURVEY.md 8(b) gpu_mask, 8(e)): mpmm::gpu::set_gpu_mask(mask) -- or the environment
// variable MPGPU_GPU_MASK (e.g. 0xff) read once -- routes simple_mul / block_mul / fast_mul through
// mpgpu_gemm_host_mask: one process drives every selected device (row shards for Simple / Block,
// leaf shards + one peer-copy exchange + row-owned post-additions for Strassen / Winograd), with
// results bit-identical to one device.  Unset (0): one handle on device 0.
// mpfr_t <-> SoA packing runs on up to 32 host threads for large matrices.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "mpgpu.h"

namespace mpmm {
namespace gpu {

namespace detail {

inline std::uint32_t& gpu_mask_ref() {
  static std::uint32_t mask = [] {
    const char* e = std::getenv("MPGPU_GPU_MASK");
    return e ? static_cast<std::uint32_t>(std::strtoul(e, nullptr, 0)) : 0u;
  }();
  return mask;
}

// fn(lo, hi) over [0, n) on up to 32 host threads (small n: the calling thread)
template <class F>
inline void parallel_for(std::size_t n, F&& fn) {
  const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t nt = std::min<std::size_t>({hw, 32, n / 16384 + 1});
  if (nt <= 1) {
    fn(std::size_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t per = (n + nt - 1) / nt;
  for (std::size_t t = 0; t < nt; ++t) {
    const std::size_t lo = t * per, hi = std::min(n, lo + per);
    if (lo < hi) th.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& x : th) x.join();
}

inline mpgpu_handle* handle() {
  static std::unique_ptr<mpgpu_handle, void (*)(mpgpu_handle*)> h = [] {
    mpgpu_handle* p = nullptr;
    if (mpgpu_init(0, &p) != MPGPU_OK) throw Error("mpgpu_init failed: no usable CUDA device");
    return std::unique_ptr<mpgpu_handle, void (*)(mpgpu_handle*)>(p, mpgpu_destroy);
  }();
  return h.get();
}

// errors.hpp:10-48 <- mpgpu.h return codes
inline void check_msg(int rc, const std::string& msg, int64_t pivot = 0) {
  if (rc == MPGPU_OK) return;
  switch (rc) {
    case MPGPU_ERR_DIMENSION: throw DimensionError(msg);
    case MPGPU_ERR_DOMAIN: throw DomainError(msg);
    case MPGPU_ERR_SINGULAR: throw SingularError(msg, static_cast<std::size_t>(pivot));
    default: throw Error("mpgpu: " + msg);
  }
}
inline void check(int rc, int64_t pivot = 0) {
  if (rc == MPGPU_OK) return;
  check_msg(rc, mpgpu_last_error(handle()), pivot);
}

struct Soa {
  int L = 0;
  std::int64_t n = 0;
  std::vector<std::uint32_t> limbs;
  std::vector<std::int32_t> exp;
  std::vector<std::uint8_t> sign;
  Soa(std::int64_t count, long bits) : L(static_cast<int>((bits + 31) / 32)), n(count),
      limbs(static_cast<std::size_t>(L) * count), exp(count), sign(count) {}
};

// one mpfr_t (documented __mpfr_struct layout: prec, sign, exp, d) -> SoA slot e
inline void pack(const Scalar& s, Soa& o, std::int64_t e) {
  mpfr_srcptr x = s.raw();
  o.sign[e] = mpfr_signbit(x) ? 1 : 0;
  if (mpfr_zero_p(x)) {
    for (int k = 0; k < o.L; ++k) o.limbs[static_cast<std::size_t>(k) * o.n + e] = 0;
    o.exp[e] = MPGPU_EXP_ZERO;
    return;
  }
  if (!mpfr_number_p(x)) throw DomainError("mpmm::gpu: non-finite operand");
  const long nh = 2 * ((x->_mpfr_prec + 63) / 64);
  for (int t = 0; t < o.L; ++t) {
    const long h = nh - 1 - t;
    std::uint32_t v = 0;
    if (h >= 0) {
      const std::uint64_t limb = x->_mpfr_d[h / 2];
      v = (h & 1) ? static_cast<std::uint32_t>(limb >> 32) : static_cast<std::uint32_t>(limb);
    }
    o.limbs[static_cast<std::size_t>(o.L - 1 - t) * o.n + e] = v;
  }
  o.exp[e] = static_cast<std::int32_t>(mpfr_get_exp(x));
}

inline void unpack(const Soa& o, std::int64_t e, Scalar& s) {
  mpfr_ptr x = s.raw();
  if (o.exp[e] == MPGPU_EXP_ZERO) {
    mpfr_set_zero(x, o.sign[e] ? -1 : 1);
    return;
  }
  mpfr_set_ui(x, 1, MPFR_RNDN);  // make x regular, then overwrite its fields
  const long n64 = (x->_mpfr_prec + 63) / 64, nh = 2 * n64;
  std::memset(x->_mpfr_d, 0, sizeof(*x->_mpfr_d) * static_cast<std::size_t>(n64));
  for (int t = 0; t < o.L && t < nh; ++t) {
    const long h = nh - 1 - t;
    const std::uint64_t v = o.limbs[static_cast<std::size_t>(o.L - 1 - t) * o.n + e];
    x->_mpfr_d[h / 2] |= (h & 1) ? (v << 32) : v;
  }
  x->_mpfr_exp = o.exp[e];
  x->_mpfr_sign = o.sign[e] ? -1 : 1;
}

inline Soa to_soa(const Matrix& m) {
  Soa o(static_cast<std::int64_t>(m.rows() * m.cols()), m.bits());
  const std::size_t cols = m.cols();
  parallel_for(m.rows() * cols, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t e = lo; e < hi; ++e) pack(m.at(e / cols, e % cols), o, static_cast<std::int64_t>(e));
  });
  return o;
}

inline Matrix from_soa(const Soa& o, std::size_t rows, std::size_t cols, PrecisionContext ctx) {
  Matrix m(rows, cols, ctx);
  parallel_for(rows * cols, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t e = lo; e < hi; ++e) unpack(o, static_cast<std::int64_t>(e), m.at(e / cols, e % cols));
  });
  return m;
}

inline void same_precision(long a, long b, long c) {
  if (a != c || b != c)
    throw DomainError("mpmm::gpu: operands must carry the context precision on the device path");
  if (c > MPGPU_MAX_PREC) throw DomainError("mpmm::gpu: precision above the device maximum");
}

inline Matrix gemm(int algo, std::size_t param_in, const Matrix& a, const Matrix& b, PrecisionContext ctx,
                   OpCounter* ops) {
  // gpu::auto_n_min (SIZE_MAX) -> MPGPU_AUTO_NMIN: the cutoff chosen per precision
  const std::int64_t param = param_in == std::numeric_limits<std::size_t>::max()
                                 ? std::int64_t{MPGPU_AUTO_NMIN}
                                 : static_cast<std::int64_t>(param_in);
  if (a.cols() != b.rows())
    throw DimensionError("inner dimension mismatch: " + std::to_string(a.cols()) + " vs " +
                         std::to_string(b.rows()));
  same_precision(a.bits(), b.bits(), ctx.bits());
  Soa sa = to_soa(a), sb = to_soa(b);
  Soa sc(static_cast<std::int64_t>(a.rows() * b.cols()), ctx.bits());
  mpgpu_stats st{};
  if (const std::uint32_t mask = gpu_mask_ref()) {  // the multi-GPU group of the selected devices
    char err[512] = {0};
    const int rc = mpgpu_gemm_host_mask(
        mask, algo, param, static_cast<std::int32_t>(ctx.bits()), a.rows(), a.cols(),
        b.cols(), sa.limbs.data(), sa.exp.data(), sa.sign.data(), sb.limbs.data(), sb.exp.data(), sb.sign.data(),
        sc.limbs.data(), sc.exp.data(), sc.sign.data(), sc.L, &st, err, sizeof err);
    check_msg(rc, err);
  } else {
    check(mpgpu_gemm_host(handle(), algo, param, static_cast<std::int32_t>(ctx.bits()),
                          a.rows(), a.cols(), b.cols(), sa.limbs.data(), sa.exp.data(), sa.sign.data(),
                          sb.limbs.data(), sb.exp.data(), sb.sign.data(), sc.limbs.data(), sc.exp.data(),
                          sc.sign.data(), sc.L, &st));
  }
  if (ops) {
    ops->mul += st.mul;
    ops->addsub += st.addsub;
  }
  return from_soa(sc, a.rows(), b.cols(), ctx);
}

}  // namespace detail

// Devices used by simple_mul / block_mul / fast_mul: bit d selects device d (0: one handle on
// device 0, the default unless MPGPU_GPU_MASK is set).  Not part of the reference API.
inline void set_gpu_mask(std::uint32_t mask) { detail::gpu_mask_ref() = mask; }
// FastMMConfig{alg, gpu::auto_n_min}: the Strassen / Winograd cutoff chosen from the measured
// leaf-GEMM throughput of the precision (mpgpu_choose_nmin).  Not part of the reference API;
// an explicit n_min replays the reference bit for bit.
inline constexpr std::size_t auto_n_min = std::numeric_limits<std::size_t>::max();
inline std::uint32_t gpu_mask() { return detail::gpu_mask_ref(); }

// ---- matrix.hpp ---------------------------------------------------------
inline Matrix simple_mul(const Matrix& a, const Matrix& b, PrecisionContext ctx) {
  return detail::gemm(MPGPU_SIMPLE, 0, a, b, ctx, nullptr);
}
inline Matrix simple_mul(const Matrix& a, const Matrix& b, PrecisionContext ctx, OpCounter& ops) {
  return detail::gemm(MPGPU_SIMPLE, 0, a, b, ctx, &ops);
}
inline Matrix block_mul(const Matrix& a, const Matrix& b, std::size_t n_min, PrecisionContext ctx) {
  if (n_min == 0 && a.cols() == b.rows()) throw DimensionError("n_min must be at least 1");
  return detail::gemm(MPGPU_BLOCK, n_min, a, b, ctx, nullptr);
}
inline Matrix block_mul(const Matrix& a, const Matrix& b, std::size_t n_min, PrecisionContext ctx,
                        OpCounter& ops) {
  if (n_min == 0 && a.cols() == b.rows()) throw DimensionError("n_min must be at least 1");
  return detail::gemm(MPGPU_BLOCK, n_min, a, b, ctx, &ops);
}

inline Matrix addsub_impl(int is_sub, const Matrix& a, const Matrix& b) {
  if (a.bits() != b.bits()) throw DomainError(is_sub ? "mat sub: mixed precisions" : "mat add: mixed precisions");
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw DimensionError("shape mismatch: " + std::to_string(a.rows()) + "x" + std::to_string(a.cols()) + " vs " +
                         std::to_string(b.rows()) + "x" + std::to_string(b.cols()));
  detail::same_precision(a.bits(), b.bits(), a.bits());
  mpgpu_handle* h = detail::handle();
  mpgpu_mat da{}, db{}, dc{};
  const auto n = static_cast<std::int64_t>(a.rows()), m = static_cast<std::int64_t>(a.cols());
  detail::Soa sa = detail::to_soa(a), sb = detail::to_soa(b), sc(n * m, a.bits());
  int rc = mpgpu_alloc_matrix(h, n, m, static_cast<std::int32_t>(a.bits()), &da);
  if (!rc) rc = mpgpu_alloc_matrix(h, n, m, static_cast<std::int32_t>(a.bits()), &db);
  if (!rc) rc = mpgpu_alloc_matrix(h, n, m, static_cast<std::int32_t>(a.bits()), &dc);
  if (!rc) rc = mpgpu_upload(h, &da, sa.limbs.data(), sa.exp.data(), sa.sign.data(), sa.L);
  if (!rc) rc = mpgpu_upload(h, &db, sb.limbs.data(), sb.exp.data(), sb.sign.data(), sb.L);
  if (!rc) rc = mpgpu_addsub(h, is_sub, &da, &db, &dc);
  if (!rc) rc = mpgpu_download(h, &dc, sc.limbs.data(), sc.exp.data(), sc.sign.data(), sc.L);
  mpgpu_free_matrix(h, &da);
  mpgpu_free_matrix(h, &db);
  mpgpu_free_matrix(h, &dc);
  detail::check(rc);
  return detail::from_soa(sc, a.rows(), a.cols(), a.ctx());
}
inline Matrix add(const Matrix& a, const Matrix& b) { return addsub_impl(0, a, b); }
inline Matrix sub(const Matrix& a, const Matrix& b) { return addsub_impl(1, a, b); }

inline Vector mat_vec_mul(const Matrix& a, const Vector& x, PrecisionContext ctx) {
  if (x.size() != a.cols()) throw DimensionError("mat_vec_mul: length mismatch");
  Matrix xm(x.size(), 1, ctx);
  for (std::size_t i = 0; i < x.size(); ++i) xm.at(i, 0) = x[i];
  Matrix bm = gpu::simple_mul(a, xm, ctx);  // same left-to-right operation sequence
  Vector b;
  for (std::size_t i = 0; i < a.rows(); ++i) b.push_back(bm.at(i, 0));
  return b;
}

// ---- fastmm.hpp ---------------------------------------------------------
inline FastMMResult fast_mul(const Matrix& a, const Matrix& b, const FastMMConfig& cfg, PrecisionContext ctx,
                             TopTrace* trace = nullptr) {
  if (a.cols() != b.rows())
    throw DimensionError("inner dimension mismatch: " + std::to_string(a.cols()) + " vs " +
                         std::to_string(b.rows()));
  if (cfg.n_min == 0) throw DimensionError("n_min must be at least 1");
  if (cfg.algorithm != Algorithm::strassen && cfg.algorithm != Algorithm::winograd)
    throw DomainError("fast_mul: algorithm must be strassen or winograd");
  if (trace) throw DomainError("mpmm::gpu::fast_mul: TopTrace is exposed through mpgpu_fast_mul_trace");
  OpCounter ops;
  Matrix c = detail::gemm(cfg.algorithm == Algorithm::strassen ? MPGPU_STRASSEN : MPGPU_WINOGRAD, cfg.n_min, a,
                          b, ctx, &ops);
  return FastMMResult{std::move(c), ops};
}

// ---- blocklu.hpp --------------------------------------------------------
inline LUFactors lu_blocked(const Matrix& a, const BlockLUConfig& cfg, PrecisionContext ctx,
                            OpCounter* schur_ops = nullptr) {
  if (a.rows() != a.cols()) throw DimensionError("lu_blocked: matrix must be square");
  if (a.bits() != ctx.bits()) throw DomainError("lu_blocked: working context must match the matrix precision");
  if (cfg.block_size == 0) throw DimensionError("lu_blocked: block size must be at least 1");
  detail::same_precision(a.bits(), a.bits(), ctx.bits());
  mpgpu_handle* h = detail::handle();
  const auto n = static_cast<std::int64_t>(a.rows());
  detail::Soa sa = detail::to_soa(a);
  int kernel = static_cast<int>(cfg.kernel);  // mpmm::Algorithm order == MPGPU_* order
  std::int64_t zp = 0;
  mpgpu_stats st{};
  // factored in place in the SoA buffers (transfers overlapped with the factorisation when
  // the buffers are page-locked)
  int rc = mpgpu_lu_blocked_host(h, static_cast<std::int32_t>(a.bits()), n, sa.limbs.data(), sa.exp.data(),
                                 sa.sign.data(), sa.L, static_cast<std::int64_t>(cfg.block_size), kernel,
                                 static_cast<std::int64_t>(cfg.n_min), 0, nullptr, &zp, &st);
  detail::check(rc, zp);
  if (schur_ops) {
    schur_ops->mul += st.mul;
    schur_ops->addsub += st.addsub;
  }
  return LUFactors{a.rows(), detail::from_soa(sa, a.rows(), a.cols(), ctx)};
}

inline LUFactors lu_columnwise(const Matrix& a) {
  if (a.rows() != a.cols()) throw DimensionError("lu_columnwise: matrix must be square");
  return gpu::lu_blocked(a, BlockLUConfig{a.rows(), Algorithm::simple, 1}, a.ctx());
}

inline Vector lu_solve(const LUFactors& f, const Vector& b, PrecisionContext ctx) {
  const std::size_t n = f.n;
  if (b.size() != n) throw DimensionError("lu_solve: length mismatch");
  detail::same_precision(f.bits(), f.bits(), ctx.bits());
  mpgpu_handle* h = detail::handle();
  Matrix bm(n, 1, ctx);
  for (std::size_t i = 0; i < n; ++i) bm.at(i, 0) = b[i];
  detail::Soa sf = detail::to_soa(f.packed), sb = detail::to_soa(bm), sx(static_cast<std::int64_t>(n), ctx.bits());
  const auto nn = static_cast<std::int64_t>(n);
  const auto bits = static_cast<std::int32_t>(ctx.bits());
  mpgpu_mat df{}, db{}, dx{};
  int rc = mpgpu_alloc_matrix(h, nn, nn, bits, &df);
  if (!rc) rc = mpgpu_alloc_matrix(h, nn, 1, bits, &db);
  if (!rc) rc = mpgpu_alloc_matrix(h, nn, 1, bits, &dx);
  if (!rc) rc = mpgpu_upload(h, &df, sf.limbs.data(), sf.exp.data(), sf.sign.data(), sf.L);
  if (!rc) rc = mpgpu_upload(h, &db, sb.limbs.data(), sb.exp.data(), sb.sign.data(), sb.L);
  std::int64_t zp = 0;
  if (!rc) rc = mpgpu_lu_solve(h, &df, nullptr, &db, &dx, 1, &zp);
  if (!rc) rc = mpgpu_download(h, &dx, sx.limbs.data(), sx.exp.data(), sx.sign.data(), sx.L);
  mpgpu_free_matrix(h, &df);
  mpgpu_free_matrix(h, &db);
  mpgpu_free_matrix(h, &dx);
  detail::check(rc, zp);
  Matrix xm = detail::from_soa(sx, n, 1, ctx);
  Vector x;
  for (std::size_t i = 0; i < n; ++i) x.push_back(xm.at(i, 0));
  return x;
}

inline Vector solve(const Matrix& a, const Vector& b, const BlockLUConfig& cfg, PrecisionContext ctx) {
  return gpu::lu_solve(gpu::lu_blocked(a, cfg, ctx), b, ctx);
}
inline Vector solve_columnwise(const Matrix& a, const Vector& b) { return gpu::lu_solve(gpu::lu_columnwise(a), b, a.ctx()); }

}  // namespace gpu
}  // namespace mpmm
