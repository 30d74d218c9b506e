/* SoA <-> mpfr_t conversion shared by the oracle restatement (mp_oracle.c) and the
 * reference bridge (ref_bridge.cpp).  TEST INFRASTRUCTURE ONLY.
 *
 * The SoA format is the one the C-ABI uses (include/mpgpu.h):
 *   limbs[k * N + e]  k = 0..L-1, 32-bit limbs, k = L-1 most significant,
 *                     MSB of limb L-1 set for every nonzero element, bits below
 *                     the precision cleared;
 *   exp[e]            MPFR exponent (value = 0.m * 2^exp, 0.m in [1/2, 1)),
 *                     MPGPU_EXP_ZERO (INT32_MIN) for a zero;
 *   sign[e]           1 = negative (zeros keep their sign).
 * The MPFR value layout follows the documented mpfr_t ABI: ceil(prec/64) 64-bit limbs,
 * MSB-normalised, least significant limb first (precision.hpp:42-109 wraps one mpfr_t). */
#ifndef MPGPU_ORACLE_SOA_MPFR_H
#define MPGPU_ORACLE_SOA_MPFR_H
#include <stdint.h>
#include <string.h>
#include "compat/mpfr.h"

#define SOA_EXP_ZERO INT32_MIN

/* 0 = ok, -1 = non-finite, -2 = exponent outside int32 */
static inline int soa_from_mpfr(mpfr_srcptr x, int L, int64_t N, int64_t e, uint32_t* limbs,
                                int32_t* exp, uint8_t* sign) {
  sign[e] = x->_mpfr_sign < 0 ? 1 : 0;
  if (x->_mpfr_exp == MPFR_EXP_ZERO_) {
    for (int k = 0; k < L; ++k) limbs[(int64_t)k * N + e] = 0;
    exp[e] = SOA_EXP_ZERO;
    return 0;
  }
  if (x->_mpfr_exp == MPFR_EXP_NAN_ || x->_mpfr_exp == MPFR_EXP_INF_) return -1;
  if (x->_mpfr_exp > INT32_MAX || x->_mpfr_exp <= (long)INT32_MIN) return -2;
  const long n64 = (x->_mpfr_prec + 63) / 64;
  const long nh = 2 * n64; /* 32-bit halves available */
  for (int t = 0; t < L; ++t) {
    long h = nh - 1 - t; /* half index, from the top */
    uint32_t v = 0;
    if (h >= 0) {
      uint64_t limb = x->_mpfr_d[h / 2];
      v = (h & 1) ? (uint32_t)(limb >> 32) : (uint32_t)limb;
    }
    limbs[(int64_t)(L - 1 - t) * N + e] = v;
  }
  exp[e] = (int32_t)x->_mpfr_exp;
  return 0;
}

/* x must already be initialised at its target precision.  Limbs below the
 * precision of x are dropped (they are zero for well-formed input). */
static inline void soa_to_mpfr(mpfr_ptr x, int L, int64_t N, int64_t e, const uint32_t* limbs,
                               const int32_t* exp, const uint8_t* sign) {
  const int neg = sign[e] != 0;
  if (exp[e] == SOA_EXP_ZERO) {
    mpfr_set_zero(x, neg ? -1 : 1);
    return;
  }
  const long prec = x->_mpfr_prec;
  const long n64 = (prec + 63) / 64;
  const long nh = 2 * n64;
  memset(x->_mpfr_d, 0, sizeof(mp_limb_t) * (size_t)n64);
  for (int t = 0; t < L && t < nh; ++t) {
    long h = nh - 1 - t;
    uint64_t v = limbs[(int64_t)(L - 1 - t) * N + e];
    x->_mpfr_d[h / 2] |= (h & 1) ? (v << 32) : v;
  }
  /* clear bits below the precision (keeps the mpfr invariant) */
  long extra = 64 * n64 - prec;
  if (extra > 0) x->_mpfr_d[0] &= ~((((mp_limb_t)1) << extra) - 1);
  x->_mpfr_exp = exp[e];
  x->_mpfr_sign = neg ? -1 : 1;
}

#endif
