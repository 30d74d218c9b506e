/* mp_oracle.c -- CPU restatement of the reference's MP GEMM / LU hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product path (paper_1410_1599_b200/, libmpgpu.so) never links it.
 *
 * What it restates (reference = /root/reference/proj/include/mpmm, cited file:line):
 *   mul_views          matrix.hpp:139-161   c_ij = RN(..RN(RN(a_i0 b_0j) + RN(a_i1 b_1j))..)
 *   addsub             matrix.hpp:121-134   elementwise RN(a +- b)
 *   block_mul_impl     matrix.hpp:188-223   k-tiled, C = P (bk = 0) else C = RN(C + P)
 *   fast_mul_rec       fastmm.hpp:99-229    Strassen / Winograd, pad-odd-with-zeros, strip
 *   recursion_plan     fastmm.hpp:68-85
 *   count_fast         opmodel.hpp:30-44
 *   lu_inplace         blocklu.hpp:42-56
 *   trsm_unit_lower_inplace  blocklu.hpp:60-69
 *   trsm_upper_right_inplace blocklu.hpp:73-86
 *   schur_product      blocklu.hpp:88-101
 *   lu_blocked         blocklu.hpp:121-146  (+ a partial-pivoting variant the reference lacks)
 *   lu_solve           blocklu.hpp:215-245
 *   mat_vec_mul        matrix.hpp:282-297
 *   Prng64 / uniform / gen_random  matgen.hpp:13-52
 * The scalar arithmetic lives in the third-party MPFR library (system libmpfr.so.6,
 * MPFR 4.2.1 here; the reference links it unpinned, CMakeLists.txt:14).  Its published
 * contract -- every add/sub/mul/div correctly rounded to nearest-even at the destination
 * precision -- is what the GPU kernels reproduce; the oracle calls MPFR for it.
 * Pinned against the compiled reference (oracle/_ref/libmpmm_ref.so) and the reference
 * tests' golden vectors in tests/test_oracle_pin.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "compat/mpfr.h"
#include "soa_mpfr.h"

#define ORC_OK 0
#define ORC_DIMENSION 1
#define ORC_DOMAIN 2
#define ORC_SINGULAR 3
#define ORC_INTERNAL 5

enum { ALG_SIMPLE = 0, ALG_BLOCK = 1, ALG_STRASSEN = 2, ALG_WINOGRAD = 3 };

typedef struct {
  int64_t rows, cols;
  long prec;
  __mpfr_struct* e;
} omat;

typedef struct {
  const omat* m;
  int64_t i0, j0, h, w;
} oview;

typedef struct {
  uint64_t mul, addsub;
} oops;

static omat om_new(int64_t rows, int64_t cols, long prec) {
  omat r;
  r.rows = rows;
  r.cols = cols;
  r.prec = prec;
  r.e = (__mpfr_struct*)malloc(sizeof(__mpfr_struct) * (size_t)(rows * cols));
  for (int64_t i = 0; i < rows * cols; ++i) {
    mpfr_init2(&r.e[i], prec);
    mpfr_set_zero(&r.e[i], 1);
  }
  return r;
}

static void om_free(omat* m) {
  if (!m->e) return;
  for (int64_t i = 0; i < m->rows * m->cols; ++i) mpfr_clear(&m->e[i]);
  free(m->e);
  m->e = NULL;
}

#define AT(M, i, j) (&(M)->e[(int64_t)(i) * (M)->cols + (j)])
static inline mpfr_srcptr VAT(const oview* v, int64_t i, int64_t j) {
  return &v->m->e[(v->i0 + i) * v->m->cols + (v->j0 + j)];
}
static oview vfull(const omat* m) {
  oview v = {m, 0, 0, m->rows, m->cols};
  return v;
}
static oview vsub(oview v, int64_t i0, int64_t j0, int64_t h, int64_t w) {
  oview r = {v.m, v.i0 + i0, v.j0 + j0, h, w};
  return r;
}

static int om_load(omat* m, int L, const uint32_t* limbs, const int32_t* exp,
                   const uint8_t* sign) {
  const int64_t N = m->rows * m->cols;
  for (int64_t e = 0; e < N; ++e) soa_to_mpfr(&m->e[e], L, N, e, limbs, exp, sign);
  return 0;
}

static int om_store(const omat* m, int L, uint32_t* limbs, int32_t* exp, uint8_t* sign) {
  const int64_t N = m->rows * m->cols;
  for (int64_t e = 0; e < N; ++e)
    if (soa_from_mpfr(&m->e[e], L, N, e, limbs, exp, sign)) return ORC_DOMAIN;
  return ORC_OK;
}

/* ---- matrix.hpp:121-134 ------------------------------------------------ */
static omat addsub(int is_sub, const oview* a, const oview* b, long prec, oops* ops) {
  omat r = om_new(a->h, a->w, prec);
  for (int64_t i = 0; i < a->h; ++i)
    for (int64_t j = 0; j < a->w; ++j) {
      if (is_sub)
        mpfr_sub(AT(&r, i, j), VAT(a, i, j), VAT(b, i, j), MPFR_RNDN);
      else
        mpfr_add(AT(&r, i, j), VAT(a, i, j), VAT(b, i, j), MPFR_RNDN);
    }
  if (ops) ops->addsub += (uint64_t)a->h * (uint64_t)a->w;
  return r;
}

/* ---- matrix.hpp:139-161 ------------------------------------------------ */
static omat mul_views(const oview* a, const oview* b, long prec, oops* ops) {
  const int64_t m = a->h, l = a->w, n = b->w;
  omat c = om_new(m, n, prec);
  mpfr_t t;
  mpfr_init2(t, prec);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      mpfr_ptr acc = AT(&c, i, j);
      mpfr_mul(acc, VAT(a, i, 0), VAT(b, 0, j), MPFR_RNDN);
      for (int64_t k = 1; k < l; ++k) {
        mpfr_mul(t, VAT(a, i, k), VAT(b, k, j), MPFR_RNDN);
        mpfr_add(acc, acc, t, MPFR_RNDN);
      }
    }
  mpfr_clear(t);
  if (ops) {
    ops->mul += (uint64_t)m * l * n;
    ops->addsub += (uint64_t)m * n * (l - 1);
  }
  return c;
}

/* ---- matrix.hpp:188-223 ------------------------------------------------ */
static omat block_mul_impl(const omat* a, const omat* b, int64_t nb, long prec, oops* ops) {
  const int64_t m = a->rows, l = a->cols, n = b->cols;
  const int64_t M = (m + nb - 1) / nb, Lb = (l + nb - 1) / nb, N = (n + nb - 1) / nb;
  omat c = om_new(m, n, prec);
  oview va = vfull(a), vb = vfull(b);
  for (int64_t bi = 0; bi < M; ++bi) {
    const int64_t i0 = bi * nb, h = (nb < m - i0) ? nb : m - i0;
    for (int64_t bj = 0; bj < N; ++bj) {
      const int64_t j0 = bj * nb, w = (nb < n - j0) ? nb : n - j0;
      for (int64_t bk = 0; bk < Lb; ++bk) {
        const int64_t k0 = bk * nb, d = (nb < l - k0) ? nb : l - k0;
        oview ta = vsub(va, i0, k0, h, d), tb = vsub(vb, k0, j0, d, w);
        omat p = mul_views(&ta, &tb, prec, ops);
        if (bk == 0) {
          for (int64_t i = 0; i < h; ++i)
            for (int64_t j = 0; j < w; ++j) mpfr_set(AT(&c, i0 + i, j0 + j), AT(&p, i, j), MPFR_RNDN);
        } else {
          for (int64_t i = 0; i < h; ++i)
            for (int64_t j = 0; j < w; ++j)
              mpfr_add(AT(&c, i0 + i, j0 + j), AT(&c, i0 + i, j0 + j), AT(&p, i, j), MPFR_RNDN);
          if (ops) ops->addsub += (uint64_t)h * w;
        }
        om_free(&p);
      }
    }
  }
  return c;
}

/* ---- fastmm.hpp:91-97 --------------------------------------------------- */
static omat pad_operand(const oview* a, int64_t pm, int64_t pn) {
  omat r = om_new(pm, pn, a->m->prec);
  for (int64_t i = 0; i < a->h; ++i)
    for (int64_t j = 0; j < a->w; ++j) mpfr_set(AT(&r, i, j), VAT(a, i, j), MPFR_RNDN);
  return r;
}

/* top-level trace (fastmm.hpp:47-51): sums (8 for Winograd), products (7), t (2) */
typedef struct {
  omat sums[8];
  omat products[7];
  omat t[2];
  int nsums, nproducts, nt;
} otrace;

static int64_t min3(int64_t a, int64_t b, int64_t c) {
  int64_t m = a < b ? a : b;
  return m < c ? m : c;
}

static void place(omat* c, const omat* src, int64_t i0, int64_t j0) {
  for (int64_t i = 0; i < src->rows; ++i)
    for (int64_t j = 0; j < src->cols; ++j) mpfr_set(AT(c, i0 + i, j0 + j), AT(src, i, j), MPFR_RNDN);
}

/* ---- fastmm.hpp:99-229 -------------------------------------------------- */
static omat fast_mul_rec(const oview* a, const oview* b, int algo, int64_t n_min, long prec,
                         oops* ops, otrace* trace) {
  const int64_t m = a->h, l = a->w, n = b->w;
  if (min3(m, l, n) <= n_min) return mul_views(a, b, prec, ops);
  const int64_t pm = m + m % 2, pl = l + l % 2, pn = n + n % 2;
  omat ap = {0, 0, 0, NULL}, bp = {0, 0, 0, NULL};
  oview av = *a, bv = *b;
  if (pm != m || pl != l) {
    ap = pad_operand(a, pm, pl);
    av = vfull(&ap);
  }
  if (pl != l || pn != n) {
    bp = pad_operand(b, pl, pn);
    bv = vfull(&bp);
  }
  const int64_t hm = pm / 2, hl = pl / 2, hn = pn / 2;
  oview a11 = vsub(av, 0, 0, hm, hl), a12 = vsub(av, 0, hl, hm, hl), a21 = vsub(av, hm, 0, hm, hl),
        a22 = vsub(av, hm, hl, hm, hl);
  oview b11 = vsub(bv, 0, 0, hl, hn), b12 = vsub(bv, 0, hn, hl, hn), b21 = vsub(bv, hl, 0, hl, hn),
        b22 = vsub(bv, hl, hn, hl, hn);
  omat c = om_new(pm, pn, prec);
#define REC(x, y) fast_mul_rec(&(x), &(y), algo, n_min, prec, ops, NULL)
#define MK(s, x, y) addsub((s), &(x), &(y), prec, ops)
  if (algo == ALG_STRASSEN) {
    omat sa = MK(0, a11, a22), sb = MK(0, b11, b22);
    oview vsa = vfull(&sa), vsb = vfull(&sb);
    omat p[7];
    p[0] = REC(vsa, vsb);
    om_free(&sa);
    sa = MK(0, a21, a22);
    vsa = vfull(&sa);
    p[1] = REC(vsa, b11);
    om_free(&sb);
    sb = MK(1, b12, b22);
    vsb = vfull(&sb);
    p[2] = REC(a11, vsb);
    om_free(&sb);
    sb = MK(1, b21, b11);
    vsb = vfull(&sb);
    p[3] = REC(a22, vsb);
    om_free(&sa);
    sa = MK(0, a11, a12);
    vsa = vfull(&sa);
    p[4] = REC(vsa, b22);
    om_free(&sa);
    sa = MK(1, a21, a11);
    vsa = vfull(&sa);
    om_free(&sb);
    sb = MK(0, b11, b12);
    vsb = vfull(&sb);
    p[5] = REC(vsa, vsb);
    om_free(&sa);
    sa = MK(1, a12, a22);
    vsa = vfull(&sa);
    om_free(&sb);
    sb = MK(0, b21, b22);
    vsb = vfull(&sb);
    p[6] = REC(vsa, vsb);
    om_free(&sa);
    om_free(&sb);
    oview vp[7];
    for (int q = 0; q < 7; ++q) vp[q] = vfull(&p[q]);
    omat u = MK(0, vp[0], vp[3]);
    oview vu = vfull(&u);
    omat u2 = MK(1, vu, vp[4]);
    om_free(&u);
    vu = vfull(&u2);
    u = MK(0, vu, vp[6]);
    om_free(&u2);
    place(&c, &u, 0, 0);
    om_free(&u);
    u = MK(0, vp[2], vp[4]);
    place(&c, &u, 0, hn);
    om_free(&u);
    u = MK(0, vp[1], vp[3]);
    place(&c, &u, hm, 0);
    om_free(&u);
    omat v = MK(0, vp[0], vp[2]);
    oview vv = vfull(&v);
    omat v2 = MK(1, vv, vp[1]);
    om_free(&v);
    vv = vfull(&v2);
    v = MK(0, vv, vp[5]);
    om_free(&v2);
    place(&c, &v, hm, hn);
    om_free(&v);
    if (trace) {
      trace->nproducts = 7;
      trace->nsums = 0;
      trace->nt = 0;
      for (int q = 0; q < 7; ++q) trace->products[q] = p[q];
    } else {
      for (int q = 0; q < 7; ++q) om_free(&p[q]);
    }
  } else {
    omat s[8];
    oview vs[8];
    s[0] = MK(0, a21, a22);
    vs[0] = vfull(&s[0]);
    s[1] = MK(1, vs[0], a11);
    vs[1] = vfull(&s[1]);
    s[2] = MK(1, a11, a21);
    vs[2] = vfull(&s[2]);
    s[3] = MK(1, a12, vs[1]);
    vs[3] = vfull(&s[3]);
    s[4] = MK(1, b12, b11);
    vs[4] = vfull(&s[4]);
    s[5] = MK(1, b22, vs[4]);
    vs[5] = vfull(&s[5]);
    s[6] = MK(1, b22, b12);
    vs[6] = vfull(&s[6]);
    s[7] = MK(1, vs[5], b21);
    vs[7] = vfull(&s[7]);
    omat mm[7];
    mm[0] = REC(vs[1], vs[5]);
    mm[1] = REC(a11, b11);
    mm[2] = REC(a12, b21);
    mm[3] = REC(vs[2], vs[6]);
    mm[4] = REC(vs[0], vs[4]);
    mm[5] = REC(vs[3], b22);
    mm[6] = REC(a22, vs[7]);
    oview vm[7];
    for (int q = 0; q < 7; ++q) vm[q] = vfull(&mm[q]);
    omat t1 = MK(0, vm[0], vm[1]);
    oview vt1 = vfull(&t1);
    omat t2 = MK(0, vt1, vm[3]);
    oview vt2 = vfull(&t2);
    omat u = MK(0, vm[1], vm[2]);
    place(&c, &u, 0, 0);
    om_free(&u);
    u = MK(0, vt1, vm[4]);
    oview vu = vfull(&u);
    omat u2 = MK(0, vu, vm[5]);
    om_free(&u);
    place(&c, &u2, 0, hn);
    om_free(&u2);
    u = MK(1, vt2, vm[6]);
    place(&c, &u, hm, 0);
    om_free(&u);
    u = MK(0, vt2, vm[4]);
    place(&c, &u, hm, hn);
    om_free(&u);
    if (trace) {
      trace->nsums = 8;
      trace->nproducts = 7;
      trace->nt = 2;
      for (int q = 0; q < 8; ++q) trace->sums[q] = s[q];
      for (int q = 0; q < 7; ++q) trace->products[q] = mm[q];
      trace->t[0] = t1;
      trace->t[1] = t2;
    } else {
      for (int q = 0; q < 8; ++q) om_free(&s[q]);
      for (int q = 0; q < 7; ++q) om_free(&mm[q]);
      om_free(&t1);
      om_free(&t2);
    }
  }
#undef REC
#undef MK
  om_free(&ap);
  om_free(&bp);
  if (pm != m || pn != n) {
    omat out = om_new(m, n, prec);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) mpfr_set(AT(&out, i, j), AT(&c, i, j), MPFR_RNDN);
    om_free(&c);
    return out;
  }
  return c;
}

/* ======================================================================== */
/*  exported API (ctypes).  Matrices are SoA with an explicit limb count L.  */
/* ======================================================================== */

typedef struct {
  const uint32_t* limbs;
  const int32_t* exp;
  const uint8_t* sign;
} csoa;
typedef struct {
  uint32_t* limbs;
  int32_t* exp;
  uint8_t* sign;
} msoa;

static omat load(int64_t rows, int64_t cols, long prec, int L, const uint32_t* limbs,
                 const int32_t* exp, const uint8_t* sign) {
  omat m = om_new(rows, cols, prec);
  om_load(&m, L, limbs, exp, sign);
  return m;
}

/* algo: 0 simple, 1 block (nb), 2 strassen, 3 winograd (n_min).  ops_out[2] = {mul, addsub}. */
int orc_gemm(int algo, int64_t param, long prec, int L, int64_t m, int64_t l, int64_t n,
             const uint32_t* al, const int32_t* ae, const uint8_t* as, const uint32_t* bl,
             const int32_t* be, const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs,
             uint64_t* ops_out) {
  if (m < 1 || l < 1 || n < 1) return ORC_DIMENSION;
  if ((algo == ALG_BLOCK || algo >= ALG_STRASSEN) && param < 1) return ORC_DIMENSION;
  omat A = load(m, l, prec, L, al, ae, as), B = load(l, n, prec, L, bl, be, bs);
  oops ops = {0, 0};
  omat C;
  oview va = vfull(&A), vb = vfull(&B);
  if (algo == ALG_SIMPLE)
    C = mul_views(&va, &vb, prec, &ops);
  else if (algo == ALG_BLOCK)
    C = block_mul_impl(&A, &B, param, prec, &ops);
  else
    C = fast_mul_rec(&va, &vb, algo, param, prec, &ops, NULL);
  int rc = om_store(&C, L, cl, ce, cs);
  if (ops_out) {
    ops_out[0] = ops.mul;
    ops_out[1] = ops.addsub;
  }
  om_free(&A);
  om_free(&B);
  om_free(&C);
  return rc;
}

/* fast_mul with the top-level trace written into caller buffers, each item an
 * hm x hn (products, t) or half-panel (sums) SoA block packed back to back:
 * sums: first 4 are hm x hl (A side), last 4 hl x hn (B side). */
int orc_fast_mul_trace(int algo, int64_t n_min, long prec, int L, int64_t m, int64_t l, int64_t n,
                       const uint32_t* al, const int32_t* ae, const uint8_t* as,
                       const uint32_t* bl, const int32_t* be, const uint8_t* bs, uint32_t* cl,
                       int32_t* ce, uint8_t* cs, uint32_t* tl, int32_t* te, uint8_t* ts,
                       int* counts) {
  omat A = load(m, l, prec, L, al, ae, as), B = load(l, n, prec, L, bl, be, bs);
  oops ops = {0, 0};
  oview va = vfull(&A), vb = vfull(&B);
  otrace tr;
  memset(&tr, 0, sizeof(tr));
  omat C = fast_mul_rec(&va, &vb, algo, n_min, prec, &ops, &tr);
  om_store(&C, L, cl, ce, cs);
  /* pack: sums, products, t -- each as its own SoA block of N_i elements */
  int64_t off = 0;
  int idx = 0;
  omat* all[17];
  for (int q = 0; q < tr.nsums; ++q) all[idx++] = &tr.sums[q];
  for (int q = 0; q < tr.nproducts; ++q) all[idx++] = &tr.products[q];
  for (int q = 0; q < tr.nt; ++q) all[idx++] = &tr.t[q];
  for (int q = 0; q < idx; ++q) {
    const int64_t N = all[q]->rows * all[q]->cols;
    /* each block stored limb-major within its own slice */
    om_store(all[q], L, tl + off * L, te + off, ts + off);
    off += N;
  }
  counts[0] = tr.nsums;
  counts[1] = tr.nproducts;
  counts[2] = tr.nt;
  for (int q = 0; q < idx; ++q) om_free(all[q]);
  om_free(&A);
  om_free(&B);
  om_free(&C);
  return ORC_OK;
}

/* elementwise add/sub (matrix.hpp:166-175) */
int orc_addsub(int is_sub, long prec, int L, int64_t rows, int64_t cols, const uint32_t* al,
               const int32_t* ae, const uint8_t* as, const uint32_t* bl, const int32_t* be,
               const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs) {
  omat A = load(rows, cols, prec, L, al, ae, as), B = load(rows, cols, prec, L, bl, be, bs);
  oview va = vfull(&A), vb = vfull(&B);
  omat C = addsub(is_sub, &va, &vb, prec, NULL);
  int rc = om_store(&C, L, cl, ce, cs);
  om_free(&A);
  om_free(&B);
  om_free(&C);
  return rc;
}

/* elementwise scalar op over n pairs at precision prec: 0 add, 1 sub, 2 mul, 3 div
 * (precision.hpp:127-161).  Used to pin the device primitives. */
int orc_vec_op(int op, long prec, int L, int64_t n, const uint32_t* al, const int32_t* ae,
               const uint8_t* as, const uint32_t* bl, const int32_t* be, const uint8_t* bs,
               uint32_t* cl, int32_t* ce, uint8_t* cs) {
  mpfr_t x, y, z;
  mpfr_init2(x, prec);
  mpfr_init2(y, prec);
  mpfr_init2(z, prec);
  int rc = ORC_OK;
  for (int64_t e = 0; e < n; ++e) {
    soa_to_mpfr(x, L, n, e, al, ae, as);
    soa_to_mpfr(y, L, n, e, bl, be, bs);
    switch (op) {
      case 0: mpfr_add(z, x, y, MPFR_RNDN); break;
      case 1: mpfr_sub(z, x, y, MPFR_RNDN); break;
      case 2: mpfr_mul(z, x, y, MPFR_RNDN); break;
      default:
        if (mpfr_zero_p(y)) {
          rc = ORC_SINGULAR;
          mpfr_set_zero(z, 1);
        } else {
          mpfr_div(z, x, y, MPFR_RNDN);
        }
    }
    if (soa_from_mpfr(z, L, n, e, cl, ce, cs)) rc = ORC_DOMAIN;
  }
  mpfr_clear(x);
  mpfr_clear(y);
  mpfr_clear(z);
  return rc;
}

/* ---- LU (blocklu.hpp) --------------------------------------------------- */

/* blocklu.hpp:42-56, extended: when piv != NULL the pivot of column d is the
 * first row r in [d, row_end) maximising |a_rd| (exact compare) and rows d, r
 * are swapped over all n columns before column d is eliminated.  With
 * piv == NULL, row_end == p + k and this is exactly the reference's lu_inplace.
 * The panel is [p, row_end) x [p, p+k): multipliers below the diagonal, the
 * right-looking updates restricted to columns < p+k (so for row_end > p+k this
 * is lu_inplace on the square block followed by trsm_upper_right_inplace on the
 * rows below it -- per element the same operation sequence). */
static int panel_factor(omat* a, int64_t p, int64_t k, int64_t row_end, int64_t* piv,
                        long prec, int64_t* zero_pivot) {
  mpfr_t t;
  mpfr_init2(t, prec);
  const int64_t end = p + k;
  for (int64_t d = p; d < end; ++d) {
    if (piv) {
      int64_t r = d;
      for (int64_t i = d + 1; i < row_end; ++i)
        if (mpfr_cmpabs(AT(a, i, d), AT(a, r, d)) > 0) r = i;
      piv[d] = r;
      if (r != d)
        for (int64_t j = 0; j < a->cols; ++j) {
          __mpfr_struct tmp = *AT(a, d, j);
          *AT(a, d, j) = *AT(a, r, j);
          *AT(a, r, j) = tmp;
        }
    }
    if (mpfr_zero_p(AT(a, d, d))) {
      *zero_pivot = d + 1;
      mpfr_clear(t);
      return ORC_SINGULAR;
    }
    for (int64_t i = d + 1; i < row_end; ++i) {
      mpfr_div(AT(a, i, d), AT(a, i, d), AT(a, d, d), MPFR_RNDN);
      for (int64_t j = d + 1; j < end; ++j) {
        mpfr_mul(t, AT(a, i, d), AT(a, d, j), MPFR_RNDN);
        mpfr_sub(AT(a, i, j), AT(a, i, j), t, MPFR_RNDN);
      }
    }
  }
  mpfr_clear(t);
  return ORC_OK;
}

/* blocklu.hpp:60-69 */
static void trsm_unit_lower_inplace(omat* a, int64_t p, int64_t k, int64_t c0, int64_t w,
                                    long prec) {
  mpfr_t t;
  mpfr_init2(t, prec);
  for (int64_t j = c0; j < c0 + w; ++j)
    for (int64_t i = p; i < p + k; ++i)
      for (int64_t s = p; s < i; ++s) {
        mpfr_mul(t, AT(a, i, s), AT(a, s, j), MPFR_RNDN);
        mpfr_sub(AT(a, i, j), AT(a, i, j), t, MPFR_RNDN);
      }
  mpfr_clear(t);
}

/* blocklu.hpp:73-86 (the reference order; used for the pivot-free path) */
static int trsm_upper_right_inplace(omat* a, int64_t r0, int64_t h, int64_t p, int64_t k,
                                    long prec, int64_t* zero_pivot) {
  mpfr_t t;
  mpfr_init2(t, prec);
  for (int64_t i = r0; i < r0 + h; ++i)
    for (int64_t j = p; j < p + k; ++j) {
      for (int64_t s = p; s < j; ++s) {
        mpfr_mul(t, AT(a, i, s), AT(a, s, j), MPFR_RNDN);
        mpfr_sub(AT(a, i, j), AT(a, i, j), t, MPFR_RNDN);
      }
      if (mpfr_zero_p(AT(a, j, j))) {
        *zero_pivot = j + 1;
        mpfr_clear(t);
        return ORC_SINGULAR;
      }
      mpfr_div(AT(a, i, j), AT(a, i, j), AT(a, j, j), MPFR_RNDN);
    }
  mpfr_clear(t);
  return ORC_OK;
}

/* blocklu.hpp:88-101 */
static omat schur_product(const omat* l21, const omat* u12, int kernel, int64_t n_min, long prec,
                          oops* ops) {
  oview vl = vfull(l21), vu = vfull(u12);
  switch (kernel) {
    case ALG_SIMPLE: return mul_views(&vl, &vu, prec, ops);
    case ALG_BLOCK: return block_mul_impl(l21, u12, n_min, prec, ops);
    default: return fast_mul_rec(&vl, &vu, kernel, n_min, prec, ops, NULL);
  }
}

/* blocklu.hpp:121-146 (pivoting == 0: the reference, operation for operation;
 * pivoting == 1: LAPACK-getrf-style partial pivoting over the tall panel).
 * In/out: the packed factors overwrite A.  piv_out[n] (0-based, LAPACK ipiv
 * semantics) is written when pivoting.  schur_ops[2] accumulates the Schur
 * multiply counts.  Returns ORC_SINGULAR with *zero_pivot = 1-based index. */
int orc_lu_blocked(long prec, int L, int64_t n, uint32_t* al, int32_t* ae, uint8_t* as,
                   int64_t K, int kernel, int64_t n_min, int pivoting, int64_t* piv_out,
                   int64_t* zero_pivot, uint64_t* schur_ops) {
  if (K < 1) return ORC_DIMENSION;
  if ((kernel == ALG_BLOCK || kernel >= ALG_STRASSEN) && n_min < 1) return ORC_DIMENSION;
  omat P = load(n, n, prec, L, al, ae, as);
  oops ops = {0, 0};
  int rc = ORC_OK;
  int64_t off = 0;
  *zero_pivot = 0;
  int64_t* piv = pivoting ? piv_out : NULL;
  while (n - off > K) {
    const int64_t rest = n - off - K;
    if (pivoting) {
      rc = panel_factor(&P, off, K, n, piv, prec, zero_pivot);
      if (rc) goto done;
      trsm_unit_lower_inplace(&P, off, K, off + K, rest, prec);
    } else {
      rc = panel_factor(&P, off, K, off + K, NULL, prec, zero_pivot);
      if (rc) goto done;
      trsm_unit_lower_inplace(&P, off, K, off + K, rest, prec);
      rc = trsm_upper_right_inplace(&P, off + K, rest, off, K, prec, zero_pivot);
      if (rc) goto done;
    }
    {
      omat l21 = om_new(rest, K, prec), u12 = om_new(K, rest, prec);
      for (int64_t i = 0; i < rest; ++i)
        for (int64_t j = 0; j < K; ++j) mpfr_set(AT(&l21, i, j), AT(&P, off + K + i, off + j), MPFR_RNDN);
      for (int64_t i = 0; i < K; ++i)
        for (int64_t j = 0; j < rest; ++j) mpfr_set(AT(&u12, i, j), AT(&P, off + i, off + K + j), MPFR_RNDN);
      omat prod = schur_product(&l21, &u12, kernel, n_min, prec, &ops);
      for (int64_t i = 0; i < rest; ++i)
        for (int64_t j = 0; j < rest; ++j)
          mpfr_sub(AT(&P, off + K + i, off + K + j), AT(&P, off + K + i, off + K + j), AT(&prod, i, j),
                   MPFR_RNDN);
      om_free(&l21);
      om_free(&u12);
      om_free(&prod);
    }
    off += K;
  }
  rc = panel_factor(&P, off, n - off, n, piv, prec, zero_pivot);
  if (rc) goto done;
  om_store(&P, L, al, ae, as);
done:
  if (schur_ops) {
    schur_ops[0] += ops.mul;
    schur_ops[1] += ops.addsub;
  }
  om_free(&P);
  return rc;
}

/* blocklu.hpp:215-245, with the row interchanges of a pivoted factorisation
 * applied to b first (piv == NULL: reference behaviour). */
int orc_lu_solve(long prec, int L, int64_t n, const uint32_t* fl, const int32_t* fe,
                 const uint8_t* fs, const int64_t* piv, const uint32_t* bl, const int32_t* be,
                 const uint8_t* bs, uint32_t* xl, int32_t* xe, uint8_t* xs, int64_t* zero_pivot) {
  omat F = load(n, n, prec, L, fl, fe, fs);
  omat b = load(n, 1, prec, L, bl, be, bs);
  if (piv)
    for (int64_t d = 0; d < n; ++d)
      if (piv[d] != d) {
        __mpfr_struct tmp = *AT(&b, d, 0);
        *AT(&b, d, 0) = *AT(&b, piv[d], 0);
        *AT(&b, piv[d], 0) = tmp;
      }
  omat y = om_new(n, 1, prec), x = om_new(n, 1, prec);
  mpfr_t t;
  mpfr_init2(t, prec);
  int rc = ORC_OK;
  for (int64_t i = 0; i < n; ++i) {
    mpfr_ptr acc = AT(&y, i, 0);
    mpfr_set(acc, AT(&b, i, 0), MPFR_RNDN);
    for (int64_t s = 0; s < i; ++s) {
      mpfr_mul(t, AT(&F, i, s), AT(&y, s, 0), MPFR_RNDN);
      mpfr_sub(acc, acc, t, MPFR_RNDN);
    }
  }
  for (int64_t ii = n; ii-- > 0;) {
    mpfr_ptr acc = AT(&x, ii, 0);
    mpfr_set(acc, AT(&y, ii, 0), MPFR_RNDN);
    for (int64_t s = ii + 1; s < n; ++s) {
      mpfr_mul(t, AT(&F, ii, s), AT(&x, s, 0), MPFR_RNDN);
      mpfr_sub(acc, acc, t, MPFR_RNDN);
    }
    if (mpfr_zero_p(AT(&F, ii, ii))) {
      *zero_pivot = ii + 1;
      rc = ORC_SINGULAR;
      break;
    }
    mpfr_div(acc, acc, AT(&F, ii, ii), MPFR_RNDN);
  }
  if (!rc) om_store(&x, L, xl, xe, xs);
  mpfr_clear(t);
  om_free(&F);
  om_free(&b);
  om_free(&y);
  om_free(&x);
  return rc;
}

/* matrix.hpp:282-297 */
int orc_mat_vec_mul(long prec, int L, int64_t rows, int64_t cols, const uint32_t* al,
                    const int32_t* ae, const uint8_t* as, const uint32_t* xl, const int32_t* xe,
                    const uint8_t* xs, uint32_t* bl, int32_t* be, uint8_t* bs) {
  omat A = load(rows, cols, prec, L, al, ae, as);
  omat x = load(cols, 1, prec, L, xl, xe, xs);
  omat b = om_new(rows, 1, prec);
  mpfr_t t;
  mpfr_init2(t, prec);
  for (int64_t i = 0; i < rows; ++i) {
    mpfr_ptr acc = AT(&b, i, 0);
    mpfr_mul(acc, AT(&A, i, 0), AT(&x, 0, 0), MPFR_RNDN);
    for (int64_t j = 1; j < cols; ++j) {
      mpfr_mul(t, AT(&A, i, j), AT(&x, j, 0), MPFR_RNDN);
      mpfr_add(acc, acc, t, MPFR_RNDN);
    }
  }
  int rc = om_store(&b, L, bl, be, bs);
  mpfr_clear(t);
  om_free(&A);
  om_free(&x);
  om_free(&b);
  return rc;
}

/* ---- metrics ----------------------------------------------------------- */
/* log2( max_ij |X_ij - Y_ij| ), evaluated exactly enough at 2p+64 bits;
 * returns -inf (as -1e308) if X == Y everywhere. Also max |X| in log2 via *log2_maxabs. */
double orc_log2_max_abs_diff(long prec, int L, int64_t N, const uint32_t* xl, const int32_t* xe,
                             const uint8_t* xs, const uint32_t* yl, const int32_t* ye,
                             const uint8_t* ys) {
  const long hp = 2 * prec + 64;
  mpfr_t x, y, d, best, lg;
  mpfr_init2(x, prec);
  mpfr_init2(y, prec);
  mpfr_init2(d, hp);
  mpfr_init2(best, hp);
  mpfr_init2(lg, 64);
  mpfr_set_zero(best, 1);
  for (int64_t e = 0; e < N; ++e) {
    soa_to_mpfr(x, L, N, e, xl, xe, xs);
    soa_to_mpfr(y, L, N, e, yl, ye, ys);
    mpfr_sub(d, x, y, MPFR_RNDN);
    mpfr_abs(d, d, MPFR_RNDN);
    if (mpfr_greater_p(d, best)) mpfr_set(best, d, MPFR_RNDN);
  }
  double r = -1e308;
  if (!mpfr_zero_p(best)) {
    mpfr_log2(lg, best, MPFR_RNDN);
    r = mpfr_get_d(lg, MPFR_RNDN);
  }
  mpfr_clear(x);
  mpfr_clear(y);
  mpfr_clear(d);
  mpfr_clear(best);
  mpfr_clear(lg);
  return r;
}

/* log2(max |X_e|) */
double orc_log2_max_abs(long prec, int L, int64_t N, const uint32_t* xl, const int32_t* xe,
                        const uint8_t* xs) {
  mpfr_t x, best, lg;
  mpfr_init2(x, prec);
  mpfr_init2(best, prec);
  mpfr_init2(lg, 64);
  mpfr_set_zero(best, 1);
  for (int64_t e = 0; e < N; ++e) {
    soa_to_mpfr(x, L, N, e, xl, xe, xs);
    mpfr_abs(x, x, MPFR_RNDN);
    if (mpfr_greater_p(x, best)) mpfr_set(best, x, MPFR_RNDN);
  }
  double r = -1e308;
  if (!mpfr_zero_p(best)) {
    mpfr_log2(lg, best, MPFR_RNDN);
    r = mpfr_get_d(lg, MPFR_RNDN);
  }
  mpfr_clear(x);
  mpfr_clear(best);
  mpfr_clear(lg);
  return r;
}

/* element -> double (for quick inspection in tests) */
int orc_to_double(long prec, int L, int64_t N, const uint32_t* xl, const int32_t* xe,
                  const uint8_t* xs, double* out) {
  mpfr_t x;
  mpfr_init2(x, prec);
  for (int64_t e = 0; e < N; ++e) {
    soa_to_mpfr(x, L, N, e, xl, xe, xs);
    out[e] = mpfr_get_d(x, MPFR_RNDN);
  }
  mpfr_clear(x);
  return 0;
}

/* long integers -> SoA at prec (mpfr_set_si, used by the exact-input tests) */
int orc_from_si(long prec, int L, int64_t N, const long* v, uint32_t* xl, int32_t* xe, uint8_t* xs) {
  mpfr_t x;
  mpfr_init2(x, prec);
  for (int64_t e = 0; e < N; ++e) {
    mpfr_set_si(x, v[e], MPFR_RNDN);
    soa_from_mpfr(x, L, N, e, xl, xe, xs);
  }
  mpfr_clear(x);
  return 0;
}

/* ---- generators (matgen.hpp:13-52) -------------------------------------- */
typedef struct {
  uint64_t s;
} oprng;
static uint64_t prng_next(oprng* r) {
  uint64_t x = r->s;
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  r->s = x;
  return x * 2685821657736338717ULL;
}

void orc_prng_stream(uint64_t seed, int64_t n, uint64_t* out) {
  oprng r = {seed ? seed : 0x9E3779B97F4A7C15ULL};
  for (int64_t i = 0; i < n; ++i) out[i] = prng_next(&r);
}

/* gen_random: entries uniform() = RN((2k - 2^53) / 2^53) at prec, row-major */
int orc_gen_random(int64_t rows, int64_t cols, uint64_t seed, long prec, int L, uint32_t* xl,
                   int32_t* xe, uint8_t* xs) {
  oprng r = {seed ? seed : 0x9E3779B97F4A7C15ULL};
  mpfr_t u;
  mpfr_init2(u, prec);
  const int64_t N = rows * cols;
  for (int64_t e = 0; e < N; ++e) {
    const int64_t num = (int64_t)(2 * (prng_next(&r) >> 11)) - ((int64_t)1 << 53);
    mpfr_set_si(u, num, MPFR_RNDN);
    mpfr_mul_2si(u, u, -53, MPFR_RNDN);
    soa_from_mpfr(u, L, N, e, xl, xe, xs);
  }
  mpfr_clear(u);
  return 0;
}

/* Independent restatement of the full-mantissa generators the GPU package also
 * implements (paper_1410_1599_b200/matgen.py).  Built from
 * top53() draws with mpfr arithmetic so it checks the package's integer code.
 *   kind 0 (uniform):  k = top (p+1) bits of the concatenated top53 draws (first
 *                      draw most significant), x = (k - 2^p) / 2^p   (exact).
 *   kind 1 (cfg3):     sign = next64() >> 63; e = next64() % 41 - 20;
 *                      mantissa = 2^(p-1) + top (p-1) bits of the concatenated
 *                      top53 draws; x = (-1)^sign * mantissa / 2^p * 2^e (exact). */
int orc_gen_full(int kind, int64_t N, uint64_t seed, long prec, int L, uint32_t* xl, int32_t* xe,
                 uint8_t* xs) {
  oprng r = {seed ? seed : 0x9E3779B97F4A7C15ULL};
  mpfr_t acc, t;
  mpfr_init2(acc, prec + 64 + 53);
  mpfr_init2(t, prec);
  const long need = kind == 0 ? prec + 1 : prec - 1;
  for (int64_t e = 0; e < N; ++e) {
    int sgn = 0;
    long ex = 0;
    if (kind == 1) {
      sgn = (int)(prng_next(&r) >> 63);
      ex = (long)(prng_next(&r) % 41) - 20;
    }
    /* acc = integer formed by the top `need` bits of the concatenated draws */
    mpfr_set_zero(acc, 1);
    long have = 0;
    while (have < need) {
      uint64_t d = prng_next(&r) >> 11; /* 53 bits */
      long take = need - have < 53 ? need - have : 53;
      uint64_t bits = d >> (53 - take);
      mpfr_mul_2si(acc, acc, take, MPFR_RNDN);
      mpfr_t b;
      mpfr_init2(b, 64);
      mpfr_set_ui(b, (unsigned long)bits, MPFR_RNDN);
      mpfr_add(acc, acc, b, MPFR_RNDN);
      mpfr_clear(b);
      have += take;
    }
    if (kind == 0) {
      mpfr_t two_p;
      mpfr_init2(two_p, 2);
      mpfr_set_ui_2exp(two_p, 1, prec, MPFR_RNDN);
      mpfr_sub(acc, acc, two_p, MPFR_RNDN); /* exact */
      mpfr_clear(two_p);
      mpfr_mul_2si(acc, acc, -prec, MPFR_RNDN);
    } else {
      mpfr_t top;
      mpfr_init2(top, 2);
      mpfr_set_ui_2exp(top, 1, prec - 1, MPFR_RNDN);
      mpfr_add(acc, acc, top, MPFR_RNDN);
      mpfr_clear(top);
      mpfr_mul_2si(acc, acc, ex - prec, MPFR_RNDN);
      if (sgn) mpfr_neg(acc, acc, MPFR_RNDN);
    }
    if (mpfr_set(t, acc, MPFR_RNDN) != 0) {
      mpfr_clear(acc);
      mpfr_clear(t);
      return ORC_INTERNAL; /* must be exact */
    }
    soa_from_mpfr(t, L, N, e, xl, xe, xs);
  }
  mpfr_clear(acc);
  mpfr_clear(t);
  return 0;
}

/* ---- op model (opmodel.hpp:17-44) --------------------------------------- */
void orc_count_fast(int algo, int64_t m, int64_t l, int64_t n, int64_t n_min, uint64_t* out) {
  if (algo < ALG_STRASSEN || min3(m, l, n) <= n_min) {
    out[0] = (uint64_t)m * l * n;
    out[1] = (uint64_t)m * n * (l - 1);
    return;
  }
  const int64_t hm = (m + m % 2) / 2, hl = (l + l % 2) / 2, hn = (n + n % 2) / 2;
  uint64_t half[2];
  orc_count_fast(algo, hm, hl, hn, n_min, half);
  const uint64_t ka = algo == ALG_STRASSEN ? 5 : 4, kb = ka, kc = algo == ALG_STRASSEN ? 8 : 7;
  out[0] = 7 * half[0];
  out[1] = 7 * half[1] + ka * hm * hl + kb * hl * hn + kc * hm * hn;
}
