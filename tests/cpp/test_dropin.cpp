// Drop-in check: the reference's own types and generators (unmodified mpmm headers)
// with mpmm::gpu:: calls (include/mpmm_gpu.hpp -> libmpgpu.so) compared against the
// reference's CPU functions with equal_values (matrix.hpp:301-307).  Built by
// oracle/Makefile into oracle/_ref/test_dropin; run by tests/test_gpu_dropin.py.
#include <cstdio>
#include <cstdlib>

#include "mpmm/mpmm.hpp"
#include "mpmm_gpu.hpp"

using namespace mpmm;

static int failures = 0;
#define CHECK(cond, what)                                     \
  do {                                                        \
    if (cond) {                                               \
      std::printf("PASS %s\n", what);                         \
    } else {                                                  \
      std::printf("FAIL %s\n", what);                         \
      ++failures;                                             \
    }                                                         \
  } while (0)

int main() {
  PrecisionContext ctx(256);
  const Matrix a = gen_random(45, 37, 7, ctx), b = gen_random(37, 51, 8, ctx);
  // a non-dyadic pair so results are rounded, not exact
  const BenchPair bp = gen_bench_pair(33, 29, 31, ctx);
  {
    OpCounter o1, o2;
    Matrix c1 = simple_mul(bp.a, bp.b, ctx, o1), c2 = gpu::simple_mul(bp.a, bp.b, ctx, o2);
    CHECK(equal_values(c1, c2) && o1 == o2, "simple_mul (bench pair) bit-exact, same OpCounter");
  }
  {
    Matrix c1 = block_mul(bp.a, bp.b, 8, ctx), c2 = gpu::block_mul(bp.a, bp.b, 8, ctx);
    CHECK(equal_values(c1, c2), "block_mul n_min=8 bit-exact");
  }
  for (Algorithm al : {Algorithm::strassen, Algorithm::winograd}) {
    FastMMResult r1 = fast_mul(bp.a, bp.b, FastMMConfig{al, 4}, ctx);
    FastMMResult r2 = gpu::fast_mul(bp.a, bp.b, FastMMConfig{al, 4}, ctx);
    CHECK(equal_values(r1.c, r2.c) && r1.ops == r2.ops,
          al == Algorithm::strassen ? "fast_mul strassen bit-exact" : "fast_mul winograd bit-exact");
  }
  {
    Matrix c1 = simple_mul(a, b, ctx), c2 = gpu::simple_mul(a, b, ctx);
    CHECK(equal_values(c1, c2), "simple_mul (gen_random) bit-exact");
    CHECK(equal_values(add(a, a), gpu::add(a, a)) && equal_values(sub(a, a), gpu::sub(a, a)), "add / sub");
  }
  {
    const Matrix m = gen_random(40, 40, 3, ctx);
    const LinearSystem sys = gen_linear_system(m, ctx);
    Vector b1 = mat_vec_mul(m, sys.x_true, ctx), b2 = gpu::mat_vec_mul(m, sys.x_true, ctx);
    bool same = b1.size() == b2.size();
    for (std::size_t i = 0; same && i < b1.size(); ++i) same = b1[i] == b2[i];
    CHECK(same, "mat_vec_mul bit-exact");
    for (Algorithm k : {Algorithm::simple, Algorithm::block, Algorithm::strassen, Algorithm::winograd}) {
      OpCounter s1, s2;
      LUFactors f1 = lu_blocked(m, BlockLUConfig{8, k, 4}, ctx, &s1);
      LUFactors f2 = gpu::lu_blocked(m, BlockLUConfig{8, k, 4}, ctx, &s2);
      CHECK(equal_values(f1.packed, f2.packed) && s1 == s2, "lu_blocked bit-exact (kernel sweep)");
      Vector x1 = lu_solve(f1, sys.b, ctx), x2 = gpu::lu_solve(f2, sys.b, ctx);
      bool sx = true;
      for (std::size_t i = 0; i < x1.size(); ++i) sx = sx && x1[i] == x2[i];
      CHECK(sx, "lu_solve bit-exact");
    }
  }
  {  // the paper's ill-conditioned experiment precision: wide formats (one warp per value)
    PrecisionContext wide(8192);
    const BenchPair wp = gen_bench_pair(9, 7, 11, wide);
    FastMMResult r1 = fast_mul(wp.a, wp.b, FastMMConfig{Algorithm::winograd, 2}, wide);
    FastMMResult r2 = gpu::fast_mul(wp.a, wp.b, FastMMConfig{Algorithm::winograd, 2}, wide);
    CHECK(equal_values(r1.c, r2.c) && r1.ops == r2.ops, "fast_mul winograd at 8192 bits bit-exact");
    const Matrix lot = gen_lotkin(12, wide);
    const LinearSystem ls = gen_linear_system(lot, wide);
    const BlockLUConfig cfg = BlockLUConfig::with_alpha(1, 4, Algorithm::winograd);
    Vector x1 = solve(lot, ls.b, cfg, wide), x2 = gpu::solve(lot, ls.b, cfg, wide);
    bool sx = x1.size() == x2.size();
    for (std::size_t i = 0; sx && i < x1.size(); ++i) sx = x1[i] == x2[i];
    CHECK(sx, "solve (Lotkin n=12, 8192 bits, Winograd Schur) bit-exact");
  }
  try {
    gpu::lu_columnwise(Matrix(2, 3, ctx));
    CHECK(false, "lu_columnwise non-square throws DimensionError");
  } catch (const DimensionError&) {
    CHECK(true, "lu_columnwise non-square throws DimensionError");
  }
  try {
    Matrix z(2, 2, PrecisionContext(64));
    mpfr_set_si(z.at(0, 1).raw(), 1, MPFR_RNDN);
    mpfr_set_si(z.at(1, 0).raw(), 1, MPFR_RNDN);
    gpu::lu_columnwise(z);
    CHECK(false, "zero pivot throws SingularError(1)");
  } catch (const SingularError& e) {
    CHECK(e.pivot_index == 1, "zero pivot throws SingularError(1)");
  }
  {  // the multi-GPU entry (mpgpu_gemm_host_mask) through the same drop-in calls: device 0 only here
    const BenchPair big = gen_bench_pair(70, 66, 61, ctx);
    Matrix s1 = gpu::simple_mul(big.a, big.b, ctx), b1 = gpu::block_mul(big.a, big.b, 16, ctx);
    FastMMResult w1 = gpu::fast_mul(big.a, big.b, FastMMConfig{Algorithm::winograd, 8}, ctx);
    gpu::set_gpu_mask(0x1);
    Matrix s2 = gpu::simple_mul(big.a, big.b, ctx), b2 = gpu::block_mul(big.a, big.b, 16, ctx);
    FastMMResult w2 = gpu::fast_mul(big.a, big.b, FastMMConfig{Algorithm::winograd, 8}, ctx);
    CHECK(equal_values(s1, s2) && equal_values(b1, b2), "gpu_mask 0x1: simple / block bit-exact");
    CHECK(equal_values(w1.c, w2.c) && w1.ops == w2.ops, "gpu_mask 0x1: fast_mul winograd bit-exact");
    CHECK(equal_values(w2.c, fast_mul(big.a, big.b, FastMMConfig{Algorithm::winograd, 8}, ctx).c),
          "gpu_mask 0x1: fast_mul equals the reference");
    try {
      gpu::set_gpu_mask(0x80000000u);  // no such device
      gpu::fast_mul(big.a, big.b, FastMMConfig{Algorithm::winograd, 8}, ctx);
      CHECK(false, "gpu_mask with a missing device throws");
    } catch (const Error&) {
      CHECK(true, "gpu_mask with a missing device throws");
    }
    gpu::set_gpu_mask(0);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
