// ref_bridge.cpp -- extern "C" bridge over the UNMODIFIED reference headers
// (/root/reference/proj/include/mpmm/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libmpmm_ref.so against the system MPFR/GMP runtime libraries and the
// locally written ABI declarations in oracle/compat/.  No reference source is
// copied into this repository: the include path points at /root/reference.
//
// TEST INFRASTRUCTURE ONLY (the checker, and the --impl reference CPU arm of
// bench.py).  Matrices cross this boundary in the C-ABI's SoA format
// (oracle/soa_mpfr.h).  Return codes: 0 ok, 1 DimensionError, 2 DomainError,
// 3 SingularError (pivot index via out-param), 4 other mpmm::Error, 5 internal,
// 6 UndefinedMetricError.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mpmm/mpmm.hpp"

extern "C" {
#include "soa_mpfr.h"
}

using namespace mpmm;

namespace {

Matrix load(std::int64_t rows, std::int64_t cols, long prec, int L, const std::uint32_t* limbs,
            const std::int32_t* exp, const std::uint8_t* sign) {
  Matrix m(rows, cols, PrecisionContext(prec));
  const std::int64_t N = rows * cols;
  for (std::int64_t i = 0; i < rows; ++i)
    for (std::int64_t j = 0; j < cols; ++j)
      soa_to_mpfr(m.at(i, j).raw(), L, N, i * cols + j, limbs, exp, sign);
  return m;
}

int store(const Matrix& m, int L, std::uint32_t* limbs, std::int32_t* exp, std::uint8_t* sign) {
  const std::int64_t N = static_cast<std::int64_t>(m.rows() * m.cols());
  for (std::size_t i = 0; i < m.rows(); ++i)
    for (std::size_t j = 0; j < m.cols(); ++j)
      if (soa_from_mpfr(m.at(i, j).raw(), L, N, static_cast<std::int64_t>(i * m.cols() + j), limbs,
                        exp, sign))
        return 2;
  return 0;
}

template <class F>
int guarded(F&& f, std::int64_t* pivot = nullptr) {
  try {
    return f();
  } catch (const SingularError& e) {
    if (pivot) *pivot = static_cast<std::int64_t>(e.pivot_index);
    return 3;
  } catch (const DimensionError&) {
    return 1;
  } catch (const DomainError&) {
    return 2;
  } catch (const UndefinedMetricError&) {
    return 6;
  } catch (const Error&) {
    return 4;
  } catch (...) {
    return 5;
  }
}

Algorithm algo_of(int a) {
  switch (a) {
    case 0: return Algorithm::simple;
    case 1: return Algorithm::block;
    case 2: return Algorithm::strassen;
    default: return Algorithm::winograd;
  }
}

}  // namespace

extern "C" {

// simple_mul (matrix.hpp:178-184), block_mul (matrix.hpp:225-233), fast_mul (fastmm.hpp:244-255)
int ref_gemm(int algo, std::int64_t param, long prec, int L, std::int64_t m, std::int64_t l,
             std::int64_t n, const std::uint32_t* al, const std::int32_t* ae, const std::uint8_t* as,
             const std::uint32_t* bl, const std::int32_t* be, const std::uint8_t* bs,
             std::uint32_t* cl, std::int32_t* ce, std::uint8_t* cs, std::uint64_t* ops_out) {
  return guarded([&] {
    PrecisionContext ctx(prec);
    Matrix a = load(m, l, prec, L, al, ae, as);
    Matrix b = load(l, n, prec, L, bl, be, bs);
    OpCounter ops;
    Matrix c = [&]() -> Matrix {
      if (algo == 0) return simple_mul(a, b, ctx, ops);
      if (algo == 1) return block_mul(a, b, static_cast<std::size_t>(param), ctx, ops);
      FastMMResult r = fast_mul(a, b, FastMMConfig{algo_of(algo), static_cast<std::size_t>(param)}, ctx);
      ops = r.ops;
      return std::move(r.c);
    }();
    if (ops_out) {
      ops_out[0] = ops.mul;
      ops_out[1] = ops.addsub;
    }
    return store(c, L, cl, ce, cs);
  });
}

// Row slice [r0, r1) of a Simple / Block product: row i of C depends only on row i
// of A and all of B, and Block's k-partition is row-independent, so the slice is
// bit-identical to the same rows of the full product.  Runs the reference's own
// block_mul on the row block (used for multi-threaded CPU timing).
int ref_gemm_rows_mt(int algo, std::int64_t param, long prec, int L, std::int64_t m,
                     std::int64_t l, std::int64_t n, const std::uint32_t* al,
                     const std::int32_t* ae, const std::uint8_t* as, const std::uint32_t* bl,
                     const std::int32_t* be, const std::uint8_t* bs, std::uint32_t* cl,
                     std::int32_t* ce, std::uint8_t* cs, int threads) {
  return guarded([&] {
    PrecisionContext ctx(prec);
    Matrix a = load(m, l, prec, L, al, ae, as);
    Matrix b = load(l, n, prec, L, bl, be, bs);
    if (threads < 1) threads = 1;
    std::vector<Matrix> parts;
    std::vector<std::int64_t> r0s;
    const std::int64_t chunk = (m + threads - 1) / threads;
    for (std::int64_t r0 = 0; r0 < m; r0 += chunk) r0s.push_back(r0);
    std::vector<Matrix*> out(r0s.size(), nullptr);
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < r0s.size(); ++t)
      pool.emplace_back([&, t] {
        const std::int64_t r0 = r0s[t], h = std::min<std::int64_t>(chunk, m - r0);
        Matrix at = MatrixView(a, r0, 0, h, l).to_matrix();
        out[t] = new Matrix(algo == 0 ? simple_mul(at, b, ctx)
                                      : block_mul(at, b, static_cast<std::size_t>(param), ctx));
      });
    for (auto& th : pool) th.join();
    const std::int64_t N = m * n;
    for (std::size_t t = 0; t < r0s.size(); ++t) {
      const Matrix& c = *out[t];
      for (std::size_t i = 0; i < c.rows(); ++i)
        for (std::size_t j = 0; j < c.cols(); ++j)
          soa_from_mpfr(c.at(i, j).raw(), L, N, (r0s[t] + static_cast<std::int64_t>(i)) * n + j, cl,
                        ce, cs);
      delete out[t];
    }
    return 0;
  });
}

// `threads` threads each run the reference's own product of the SAME inputs
// (independent copies, no shared state -- the reference is reentrant);
// *seconds = steady_clock wall time of the multiplies only (as bench.hpp:87-94 /
// :130-144 time run_matmul).  C receives thread 0's result.
int ref_gemm_replicas(int algo, std::int64_t param, long prec, int L, std::int64_t m, std::int64_t l,
                      std::int64_t n, const std::uint32_t* al, const std::int32_t* ae, const std::uint8_t* as,
                      const std::uint32_t* bl, const std::int32_t* be, const std::uint8_t* bs,
                      std::uint32_t* cl, std::int32_t* ce, std::uint8_t* cs, int threads, double* seconds) {
  return guarded([&] {
    PrecisionContext ctx(prec);
    if (threads < 1) threads = 1;
    std::vector<Matrix> as_, bs_;
    for (int t = 0; t < threads; ++t) {
      as_.push_back(load(m, l, prec, L, al, ae, as));
      bs_.push_back(load(l, n, prec, L, bl, be, bs));
    }
    std::vector<Matrix*> out(threads, nullptr);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        const Matrix& a = as_[t];
        const Matrix& b = bs_[t];
        if (algo == 0)
          out[t] = new Matrix(simple_mul(a, b, ctx));
        else if (algo == 1)
          out[t] = new Matrix(block_mul(a, b, static_cast<std::size_t>(param), ctx));
        else
          out[t] = new Matrix(fast_mul(a, b, FastMMConfig{algo_of(algo), static_cast<std::size_t>(param)}, ctx).c);
      });
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    int rc = store(*out[0], L, cl, ce, cs);
    for (auto* p : out) delete p;
    return rc;
  });
}

// fast_mul with TopTrace (fastmm.hpp:47-51): items packed back to back as in
// orc_fast_mul_trace (sums, then products, then t), each its own SoA block.
int ref_fast_mul_trace(int algo, std::int64_t n_min, long prec, int L, std::int64_t m,
                       std::int64_t l, std::int64_t n, const std::uint32_t* al,
                       const std::int32_t* ae, const std::uint8_t* as, const std::uint32_t* bl,
                       const std::int32_t* be, const std::uint8_t* bs, std::uint32_t* cl,
                       std::int32_t* ce, std::uint8_t* cs, std::uint32_t* tl, std::int32_t* te,
                       std::uint8_t* ts, int* counts, std::uint64_t* ops_out) {
  return guarded([&] {
    PrecisionContext ctx(prec);
    Matrix a = load(m, l, prec, L, al, ae, as);
    Matrix b = load(l, n, prec, L, bl, be, bs);
    TopTrace tr;
    FastMMResult r = fast_mul(a, b, FastMMConfig{algo_of(algo), static_cast<std::size_t>(n_min)}, ctx, &tr);
    store(r.c, L, cl, ce, cs);
    std::int64_t off = 0;
    auto put = [&](const std::vector<Matrix>& v) {
      for (const Matrix& x : v) {
        store(x, L, tl + off * L, te + off, ts + off);
        off += static_cast<std::int64_t>(x.rows() * x.cols());
      }
    };
    put(tr.sums);
    put(tr.products);
    put(tr.t);
    counts[0] = static_cast<int>(tr.sums.size());
    counts[1] = static_cast<int>(tr.products.size());
    counts[2] = static_cast<int>(tr.t.size());
    if (ops_out) {
      ops_out[0] = r.ops.mul;
      ops_out[1] = r.ops.addsub;
    }
    return 0;
  });
}

// lu_blocked (blocklu.hpp:121-146) / lu_columnwise (blocklu.hpp:107-112) when K == 0.
int ref_lu_blocked(long prec, int L, std::int64_t n, std::uint32_t* al, std::int32_t* ae,
                   std::uint8_t* as, std::int64_t K, int kernel, std::int64_t n_min,
                   std::int64_t* zero_pivot, std::uint64_t* schur_ops) {
  *zero_pivot = 0;
  return guarded(
      [&] {
        PrecisionContext ctx(prec);
        Matrix a = load(n, n, prec, L, al, ae, as);
        OpCounter ops;
        LUFactors f = K == 0 ? lu_columnwise(a)
                             : lu_blocked(a, BlockLUConfig{static_cast<std::size_t>(K), algo_of(kernel),
                                                           static_cast<std::size_t>(n_min)},
                                          ctx, &ops);
        if (schur_ops) {
          schur_ops[0] = ops.mul;
          schur_ops[1] = ops.addsub;
        }
        return store(f.packed, L, al, ae, as);
      },
      zero_pivot);
}

// lu_solve (blocklu.hpp:215-245)
int ref_lu_solve(long prec, int L, std::int64_t n, const std::uint32_t* fl, const std::int32_t* fe,
                 const std::uint8_t* fs, const std::uint32_t* bl, const std::int32_t* be,
                 const std::uint8_t* bs, std::uint32_t* xl, std::int32_t* xe, std::uint8_t* xs,
                 std::int64_t* zero_pivot) {
  *zero_pivot = 0;
  return guarded(
      [&] {
        PrecisionContext ctx(prec);
        LUFactors f{static_cast<std::size_t>(n), load(n, n, prec, L, fl, fe, fs)};
        Matrix bm = load(n, 1, prec, L, bl, be, bs);
        Vector b;
        for (std::int64_t i = 0; i < n; ++i) b.push_back(bm.at(i, 0));
        Vector x = lu_solve(f, b, ctx);
        Matrix xm(n, 1, ctx);
        for (std::int64_t i = 0; i < n; ++i) xm.at(i, 0) = x[i];
        return store(xm, L, xl, xe, xs);
      },
      zero_pivot);
}

// mat_vec_mul (matrix.hpp:282-297)
int ref_mat_vec_mul(long prec, int L, std::int64_t rows, std::int64_t cols, const std::uint32_t* al,
                    const std::int32_t* ae, const std::uint8_t* as, const std::uint32_t* xl,
                    const std::int32_t* xe, const std::uint8_t* xs, std::uint32_t* bl,
                    std::int32_t* be, std::uint8_t* bs) {
  return guarded([&] {
    PrecisionContext ctx(prec);
    Matrix a = load(rows, cols, prec, L, al, ae, as);
    Matrix xm = load(cols, 1, prec, L, xl, xe, xs);
    Vector x;
    for (std::int64_t i = 0; i < cols; ++i) x.push_back(xm.at(i, 0));
    Vector b = mat_vec_mul(a, x, ctx);
    Matrix bm(rows, 1, ctx);
    for (std::int64_t i = 0; i < rows; ++i) bm.at(i, 0) = b[i];
    return store(bm, L, bl, be, bs);
  });
}

// Prng64 (matgen.hpp:13-42)
void ref_prng_stream(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
  Prng64 r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next64();
}

// gen_random (matgen.hpp:45-52)
int ref_gen_random(std::int64_t rows, std::int64_t cols, std::uint64_t seed, long prec, int L,
                   std::uint32_t* xl, std::int32_t* xe, std::uint8_t* xs) {
  return guarded([&] { return store(gen_random(rows, cols, seed, PrecisionContext(prec)), L, xl, xe, xs); });
}

// gen_bench_pair (matgen.hpp:63-78) and bench_reference (matgen.hpp:99-105)
int ref_gen_bench_pair(std::int64_t m, std::int64_t l, std::int64_t n, long prec, int L,
                       std::uint32_t* al, std::int32_t* ae, std::uint8_t* as, std::uint32_t* bl,
                       std::int32_t* be, std::uint8_t* bs) {
  return guarded([&] {
    BenchPair p = gen_bench_pair(m, l, n, PrecisionContext(prec));
    int rc = store(p.a, L, al, ae, as);
    return rc ? rc : store(p.b, L, bl, be, bs);
  });
}

int ref_bench_reference(std::int64_t m, std::int64_t l, std::int64_t n, long prec, int L,
                        std::uint32_t* cl, std::int32_t* ce, std::uint8_t* cs) {
  return guarded([&] { return store(bench_reference(m, l, n, PrecisionContext(prec)), L, cl, ce, cs); });
}

// to_hex (precision.hpp:210-244) of N elements, '\n'-joined into buf.
int ref_to_hex(long prec, int L, std::int64_t N, const std::uint32_t* xl, const std::int32_t* xe,
               const std::uint8_t* xs, char* buf, std::int64_t buflen) {
  return guarded([&] {
    Matrix m = load(N, 1, prec, L, xl, xe, xs);
    std::string out;
    for (std::int64_t i = 0; i < N; ++i) {
      if (i) out += '\n';
      out += to_hex(m.at(i, 0));
    }
    if (static_cast<std::int64_t>(out.size()) + 1 > buflen) return 1;
    std::memcpy(buf, out.c_str(), out.size() + 1);
    return 0;
  });
}

// count_fast (opmodel.hpp:30-44)
int ref_count_fast(int algo, std::int64_t m, std::int64_t l, std::int64_t n, std::int64_t n_min,
                   std::uint64_t* out) {
  return guarded([&] {
    OpCounter c = count_fast(algo_of(algo), m, l, n, n_min);
    out[0] = c.mul;
    out[1] = c.addsub;
    return 0;
  });
}

// recursion_plan (fastmm.hpp:68-85): rows of 8 int64 {level, m,l,n, pm,pl,pn, base}
int ref_recursion_plan(std::int64_t m, std::int64_t l, std::int64_t n, std::int64_t n_min,
                       std::int64_t* out, int max_levels, int* count) {
  return guarded([&] {
    auto plan = recursion_plan(m, l, n, FastMMConfig{Algorithm::strassen, static_cast<std::size_t>(n_min)});
    *count = static_cast<int>(plan.size());
    for (std::size_t i = 0; i < plan.size() && static_cast<int>(i) < max_levels; ++i) {
      std::int64_t* r = out + 8 * i;
      r[0] = plan[i].level;
      r[1] = plan[i].before.m;
      r[2] = plan[i].before.l;
      r[3] = plan[i].before.n;
      r[4] = plan[i].padded.m;
      r[5] = plan[i].padded.l;
      r[6] = plan[i].padded.n;
      r[7] = plan[i].base ? 1 : 0;
    }
    return 0;
  });
}

// ---- accuracy metrics and benchmark drivers (matrix.hpp:237-279, blocklu.hpp:306-333,
// bench.hpp:117-249) -- checkers of the device metrics and of the GPU CSV rows.
int ref_max_rel_error(long pa, int La, long pr, int Lr, std::int64_t rows, std::int64_t cols,
                      const std::uint32_t* al, const std::int32_t* ae, const std::uint8_t* as,
                      const std::uint32_t* rl, const std::int32_t* re, const std::uint8_t* rs,
                      std::uint32_t* ol, std::int32_t* oe, std::uint8_t* os, std::int64_t* skipped) {
  return guarded([&] {
    Matrix a = load(rows, cols, pa, La, al, ae, as);
    Matrix r = load(rows, cols, pr, Lr, rl, re, rs);
    RelErrorStats st = max_rel_error(a, r);
    Matrix out(2, 1, PrecisionContext(pr));
    out.at(0, 0) = st.max;
    out.at(1, 0) = st.min;
    *skipped = static_cast<std::int64_t>(st.skipped_zero_refs);
    return store(out, Lr, ol, oe, os);
  });
}

int ref_solution_error(long prec, int L, std::int64_t n, const std::uint32_t* xl, const std::int32_t* xe,
                       const std::uint8_t* xs, const std::uint32_t* tl, const std::int32_t* te,
                       const std::uint8_t* ts, std::uint32_t* ol, std::int32_t* oe, std::uint8_t* os,
                       std::int64_t* zero_refs) {
  return guarded([&] {
    Matrix x = load(n, 1, prec, L, xl, xe, xs), t = load(n, 1, prec, L, tl, te, ts);
    Vector xv, tv;
    for (std::int64_t i = 0; i < n; ++i) {
      xv.push_back(x.at(i, 0));
      tv.push_back(t.at(i, 0));
    }
    SolutionError se = max_rel_error_solution(xv, tv);
    Matrix out(2, 1, PrecisionContext(prec));
    out.at(0, 0) = se.max_rel;
    out.at(1, 0) = se.max_zero_abs;
    *zero_refs = static_cast<std::int64_t>(se.zero_refs);
    return store(out, L, ol, oe, os);
  });
}

int ref_one_norm(long prec, int L, std::int64_t rows, std::int64_t cols, const std::uint32_t* al,
                 const std::int32_t* ae, const std::uint8_t* as, std::uint32_t* ol, std::int32_t* oe,
                 std::uint8_t* os) {
  return guarded([&] {
    Matrix a = load(rows, cols, prec, L, al, ae, as);
    Matrix out(1, 1, PrecisionContext(prec));
    out.at(0, 0) = one_norm(a);
    return store(out, L, ol, oe, os);
  });
}

// gen_lotkin (matgen.hpp:107-121)
int ref_gen_lotkin(std::int64_t n, long prec, int L, std::uint32_t* xl, std::int32_t* xe, std::uint8_t* xs) {
  return guarded([&] { return store(gen_lotkin(n, PrecisionContext(prec)), L, xl, xe, xs); });
}

// to_decimal (precision.hpp:293-300) of N elements, '\n'-joined into buf
int ref_to_decimal(long prec, int L, std::int64_t N, const std::uint32_t* xl, const std::int32_t* xe,
                   const std::uint8_t* xs, int digits, char* buf, std::int64_t buflen) {
  return guarded([&] {
    Matrix m = load(N, 1, prec, L, xl, xe, xs);
    std::string out;
    for (std::int64_t i = 0; i < N; ++i) {
      if (i) out += '\n';
      out += to_decimal(m.at(i, 0), digits);
    }
    if (static_cast<std::int64_t>(out.size()) + 1 > buflen) return 1;
    std::memcpy(buf, out.c_str(), out.size() + 1);
    return 0;
  });
}

namespace {
int csv_out(const std::vector<BenchRecord>& rows, char* buf, std::int64_t buflen) {
  std::ostringstream os;
  print_csv(os, rows);
  const std::string s = os.str();
  if (static_cast<std::int64_t>(s.size()) + 1 > buflen) return 1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}
}  // namespace

// run_matmul (bench.hpp:117-165): algo_mask bit a selects Algorithm a
int ref_run_matmul(std::int64_t m, std::int64_t l, std::int64_t n, long bits, std::int64_t n_min, int algo_mask,
                   long ref_mult, int verbose, char* buf, std::int64_t buflen) {
  return guarded([&] {
    MatmulRequest q;
    q.algos.clear();
    for (int a = 0; a < 4; ++a)
      if (algo_mask & (1 << a)) q.algos.push_back(algo_of(a));
    q.m = m;
    q.l = l;
    q.n = n;
    q.bits = bits;
    q.n_min = n_min;
    q.ref_bits_multiplier = ref_mult;
    q.verbose = verbose != 0;
    return csv_out(run_matmul(q), buf, buflen);
  });
}

// run_lu (bench.hpp:187-249): kind 0 random, 1 lotkin
int ref_run_lu(int kind, std::int64_t n, long bits, int kernel, std::int64_t n_min, std::int64_t alo,
               std::int64_t ahi, std::uint64_t seed, int verbose, char* buf, std::int64_t buflen,
               int* any_singular) {
  return guarded([&] {
    LURequest q;
    q.matrix_kind = kind == 0 ? "random" : "lotkin";
    q.n = n;
    q.bits = bits;
    q.kernel = algo_of(kernel);
    q.n_min = n_min;
    q.alpha_lo = alo;
    q.alpha_hi = ahi;
    q.seed = seed;
    q.verbose = verbose != 0;
    LUOutcome o = run_lu(q);
    *any_singular = o.any_singular ? 1 : 0;
    return csv_out(o.rows, buf, buflen);
  });
}

// ---- text codec and op-count tables (precision.hpp:204-300, matrix.hpp:309-344,
// opmodel.hpp:46-155) -- checkers of the host codec and the CLI's opcount ----
int ref_from_hex(const char* text, long prec, int L, std::uint32_t* xl, std::int32_t* xe, std::uint8_t* xs,
                 std::int64_t* err_pos) {
  try {
    Matrix m(1, 1, PrecisionContext(prec));
    m.at(0, 0) = from_hex(text, PrecisionContext(prec));
    return store(m, L, xl, xe, xs);
  } catch (const ParseError& e) {
    *err_pos = static_cast<std::int64_t>(e.position);
    return 7;
  } catch (...) {
    return 5;
  }
}

int ref_write_matrix(long prec, int L, std::int64_t rows, std::int64_t cols, const std::uint32_t* xl,
                     const std::int32_t* xe, const std::uint8_t* xs, char* buf, std::int64_t buflen) {
  return guarded([&] {
    Matrix m = load(rows, cols, prec, L, xl, xe, xs);
    std::ostringstream os;
    write_matrix(os, m);
    const std::string t = os.str();
    if (static_cast<std::int64_t>(t.size()) + 1 > buflen) return 1;
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
  });
}

// read_matrix: dims[3] = {m, n, bits}; the SoA buffers hold cap elements of L limbs
int ref_read_matrix(const char* text, int L, std::int64_t cap, std::int64_t* dims, std::uint32_t* xl,
                    std::int32_t* xe, std::uint8_t* xs) {
  return guarded([&] {
    std::istringstream is(text);
    Matrix m = read_matrix(is);
    dims[0] = static_cast<std::int64_t>(m.rows());
    dims[1] = static_cast<std::int64_t>(m.cols());
    dims[2] = m.bits();
    if (static_cast<std::int64_t>(m.rows() * m.cols()) > cap || (m.bits() + 31) / 32 > L) return 1;
    return store(m, L, xl, xe, xs);
  });
}

// opcount table (format 0: text, 1: csv) over n x n x n sizes
int ref_ratio_table(int format, const std::int64_t* sizes, int count, std::int64_t n_min, char* buf,
                    std::int64_t buflen) {
  return guarded([&] {
    std::vector<Dims3> dims;
    for (int i = 0; i < count; ++i)
      dims.push_back(Dims3{static_cast<std::size_t>(sizes[i]), static_cast<std::size_t>(sizes[i]),
                           static_cast<std::size_t>(sizes[i])});
    const auto rows = ratio_table(dims, static_cast<std::size_t>(n_min));
    const std::string t = format == 0 ? format_ratio_table(rows) : format_ratio_csv(rows);
    if (static_cast<std::int64_t>(t.size()) + 1 > buflen) return 1;
    std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
  });
}

// inverse / cond_one (blocklu.hpp:261-301)
int ref_inverse(long pa, int La, std::int64_t n, const std::uint32_t* al, const std::int32_t* ae,
                const std::uint8_t* as, long pc, int Lc, std::uint32_t* xl, std::int32_t* xe, std::uint8_t* xs,
                std::int64_t* pivot) {
  return guarded([&] { return store(inverse(load(n, n, pa, La, al, ae, as), PrecisionContext(pc)), Lc, xl, xe, xs); },
                 pivot);
}

int ref_cond_one(long pa, int La, std::int64_t n, const std::uint32_t* al, const std::int32_t* ae,
                 const std::uint8_t* as, long phi, int Lo, std::uint32_t* ol, std::int32_t* oe, std::uint8_t* os,
                 std::int64_t* pivot) {
  return guarded([&] {
    Matrix a = load(n, n, pa, La, al, ae, as);
    Scalar c = phi > 0 ? cond_one(a, PrecisionContext(phi)) : cond_one(a);
    Matrix out(1, 1, PrecisionContext(mpfr_get_prec(c.raw())));
    out.at(0, 0) = c;
    return store(out, Lo, ol, oe, os);
  }, pivot);
}

}  // extern "C"
