/* Minimal GMP ABI declarations (LP64, GMP 6.x) for building the oracle and the
 * unmodified reference headers against the runtime-only libgmp.so.10 in this
 * image (no development headers are installed).  Written from the documented
 * ABI: only the handful of entry points the reference / oracle use.
 * TEST INFRASTRUCTURE ONLY -- never part of the shipped GPU path. */
#ifndef MPGPU_COMPAT_GMP_H
#define MPGPU_COMPAT_GMP_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef long mp_exp_t;
typedef unsigned long mp_bitcnt_t;
typedef struct { int _mp_alloc; int _mp_size; mp_limb_t* _mp_d; } __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;
typedef struct { __mpz_struct _mp_num; __mpz_struct _mp_den; } __mpq_struct;
typedef __mpq_struct mpq_t[1];
typedef const __mpq_struct* mpq_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
char* __gmpz_get_str(char*, int, mpz_srcptr);
void __gmp_get_memory_functions(void* (**)(size_t), void* (**)(void*, size_t, size_t),
                                void (**)(void*, size_t));
#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_abs __gmpz_abs
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_get_str __gmpz_get_str
#define mp_get_memory_functions __gmp_get_memory_functions
#ifdef __cplusplus
}
#endif
#endif
