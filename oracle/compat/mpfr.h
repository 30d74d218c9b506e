/* Minimal MPFR ABI declarations (LP64, MPFR 4.x, _MPFR_PREC_FORMAT 3 / _MPFR_EXP_FORMAT 3)
 * for the runtime-only libmpfr.so.6 in this image.  Written from the documented ABI:
 *   struct { mpfr_prec_t prec; mpfr_sign_t sign; mpfr_exp_t exp; mp_limb_t* d; }
 * value = sign * 0.d * 2^exp, d MSB-normalised in ceil(prec/64) limbs (bits below
 * prec are zero).  Special values use reserved exponents (see MPFR_EXP_ZERO...).
 * TEST INFRASTRUCTURE ONLY -- used by oracle/ and the reference bridge. */
#ifndef MPGPU_COMPAT_MPFR_H
#define MPGPU_COMPAT_MPFR_H
#include <limits.h>
#include <stdio.h>
#include "gmp.h"
#ifdef __cplusplus
extern "C" {
#endif
typedef long mpfr_prec_t;
typedef int mpfr_sign_t;
typedef long mpfr_exp_t;
typedef struct {
  mpfr_prec_t _mpfr_prec;
  mpfr_sign_t _mpfr_sign;
  mpfr_exp_t _mpfr_exp;
  mp_limb_t* _mpfr_d;
} __mpfr_struct;
typedef __mpfr_struct mpfr_t[1];
typedef __mpfr_struct* mpfr_ptr;
typedef const __mpfr_struct* mpfr_srcptr;
typedef enum { MPFR_RNDN = 0, MPFR_RNDZ, MPFR_RNDU, MPFR_RNDD, MPFR_RNDA, MPFR_RNDF } mpfr_rnd_t;
/* reserved exponents (MPFR_EXP_MIN = LONG_MIN) */
#define MPFR_EXP_ZERO_ (LONG_MIN + 1)
#define MPFR_EXP_NAN_ (LONG_MIN + 2)
#define MPFR_EXP_INF_ (LONG_MIN + 3)

void mpfr_init2(mpfr_ptr, mpfr_prec_t);
void mpfr_clear(mpfr_ptr);
void mpfr_set_prec(mpfr_ptr, mpfr_prec_t);
void mpfr_set_zero(mpfr_ptr, int);
int mpfr_set_si(mpfr_ptr, long, mpfr_rnd_t);
int mpfr_set_ui(mpfr_ptr, unsigned long, mpfr_rnd_t);
int mpfr_set_d(mpfr_ptr, double, mpfr_rnd_t);
int mpfr_set(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_set_q(mpfr_ptr, mpq_srcptr, mpfr_rnd_t);
int mpfr_set_si_2exp(mpfr_ptr, long, mpfr_exp_t, mpfr_rnd_t);
int mpfr_set_ui_2exp(mpfr_ptr, unsigned long, mpfr_exp_t, mpfr_rnd_t);
int mpfr_set_str(mpfr_ptr, const char*, int, mpfr_rnd_t);
int mpfr_add(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sub(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_div(mpfr_ptr, mpfr_srcptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_sqrt(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_neg(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_abs(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_mul_2si(mpfr_ptr, mpfr_srcptr, long, mpfr_rnd_t);
int mpfr_mul_si(mpfr_ptr, mpfr_srcptr, long, mpfr_rnd_t);
int mpfr_mul_ui(mpfr_ptr, mpfr_srcptr, unsigned long, mpfr_rnd_t);
int mpfr_ui_div(mpfr_ptr, unsigned long, mpfr_srcptr, mpfr_rnd_t);
int mpfr_log2(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_exp10(mpfr_ptr, mpfr_srcptr, mpfr_rnd_t);
int mpfr_equal_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_less_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_lessequal_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_greater_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_greaterequal_p(mpfr_srcptr, mpfr_srcptr);
int mpfr_cmpabs(mpfr_srcptr, mpfr_srcptr);
int mpfr_cmp(mpfr_srcptr, mpfr_srcptr);
int mpfr_zero_p(mpfr_srcptr);
int mpfr_number_p(mpfr_srcptr);
int mpfr_regular_p(mpfr_srcptr);
int mpfr_signbit(mpfr_srcptr);
int mpfr_sgn(mpfr_srcptr);
mpfr_prec_t mpfr_get_prec(mpfr_srcptr);
mpfr_exp_t mpfr_get_exp(mpfr_srcptr);
mpfr_exp_t mpfr_get_z_2exp(mpz_ptr, mpfr_srcptr);
double mpfr_get_d(mpfr_srcptr, mpfr_rnd_t);
int mpfr_strtofr(mpfr_ptr, const char*, char**, int, mpfr_rnd_t);
int mpfr_asprintf(char**, const char*, ...);
void mpfr_free_str(char*);
#ifdef __cplusplus
}
#endif
#endif
