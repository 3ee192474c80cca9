/* TEST INFRASTRUCTURE ONLY (oracle build).
 *
 * Declarations of the GMP 6.x C entry points that the reference headers under
 * /root/reference/proj/include/drzeta use, so the unmodified reference can be
 * compiled in this image, which ships libgmp.so.10 but no gmp.h.  Symbols
 * resolve against /usr/lib/x86_64-linux-gnu/libgmp.so.10 (GMP 6.3.0).
 * Layout of __mpz_struct / __mpq_struct follows the documented GMP ABI.
 */
#ifndef ORACLE_SHIM_GMP_H
#define ORACLE_SHIM_GMP_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef unsigned long mp_bitcnt_t;
typedef long mp_size_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

typedef struct {
  __mpz_struct _mp_num;
  __mpz_struct _mp_den;
} __mpq_struct;
typedef __mpq_struct mpq_t[1];
typedef __mpq_struct* mpq_ptr;
typedef const __mpq_struct* mpq_srcptr;

/* integers */
void __gmpz_init(mpz_ptr);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_set_si(mpz_ptr, long);
int __gmpz_set_str(mpz_ptr, const char*, int);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_swap(mpz_ptr, mpz_ptr);
char* __gmpz_get_str(char*, int, mpz_srcptr);
unsigned long __gmpz_get_ui(mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
int __gmpz_fits_slong_p(mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
int __gmpz_cmp_ui(mpz_srcptr, unsigned long);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
unsigned long __gmpz_fdiv_qr_ui(mpz_ptr, mpz_ptr, mpz_srcptr, unsigned long);
unsigned long __gmpz_fdiv_q_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_tdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_and(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_invert(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
void __gmpz_powm_ui(mpz_ptr, mpz_srcptr, unsigned long, mpz_srcptr);
void __gmpz_bin_uiui(mpz_ptr, unsigned long, unsigned long);
int __gmpz_divisible_p(mpz_srcptr, mpz_srcptr);
int __gmpz_divisible_ui_p(mpz_srcptr, unsigned long);
void __gmpz_divexact_ui(mpz_ptr, mpz_srcptr, unsigned long);

/* rationals */
void __gmpq_init(mpq_ptr);
void __gmpq_clear(mpq_ptr);
void __gmpq_set(mpq_ptr, mpq_srcptr);
void __gmpq_set_z(mpq_ptr, mpz_srcptr);
void __gmpq_set_si(mpq_ptr, long, unsigned long);
void __gmpq_canonicalize(mpq_ptr);
void __gmpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_div(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_neg(mpq_ptr, mpq_srcptr);
int __gmpq_cmp(mpq_srcptr, mpq_srcptr);
char* __gmpq_get_str(char*, int, mpq_srcptr);
void __gmpq_swap(mpq_ptr, mpq_ptr);

#ifdef __cplusplus
}
#endif

#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_si __gmpz_set_si
#define mpz_set_str __gmpz_set_str
#define mpz_init_set __gmpz_init_set
#define mpz_init_set_ui __gmpz_init_set_ui
#define mpz_init_set_si __gmpz_init_set_si
#define mpz_swap __gmpz_swap
#define mpz_get_str __gmpz_get_str
#define mpz_get_ui __gmpz_get_ui
#define mpz_get_si __gmpz_get_si
#define mpz_fits_slong_p __gmpz_fits_slong_p
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_add __gmpz_add
#define mpz_add_ui __gmpz_add_ui
#define mpz_sub __gmpz_sub
#define mpz_sub_ui __gmpz_sub_ui
#define mpz_mul __gmpz_mul
#define mpz_mul_si __gmpz_mul_si
#define mpz_mul_ui __gmpz_mul_ui
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_cmp __gmpz_cmp
#define mpz_cmp_si __gmpz_cmp_si
#define mpz_cmp_ui __gmpz_cmp_ui
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_fdiv_q __gmpz_fdiv_q
#define mpz_fdiv_r __gmpz_fdiv_r
#define mpz_fdiv_qr_ui __gmpz_fdiv_qr_ui
#define mpz_fdiv_q_ui __gmpz_fdiv_q_ui
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_tdiv_q_2exp __gmpz_tdiv_q_2exp
#define mpz_and __gmpz_and
#define mpz_invert __gmpz_invert
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_powm_ui __gmpz_powm_ui
#define mpz_bin_uiui __gmpz_bin_uiui
#define mpz_divisible_p __gmpz_divisible_p
#define mpz_divisible_ui_p __gmpz_divisible_ui_p
#define mpz_divexact_ui __gmpz_divexact_ui
#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)

#define mpq_init __gmpq_init
#define mpq_clear __gmpq_clear
#define mpq_set __gmpq_set
#define mpq_set_z __gmpq_set_z
#define mpq_set_si __gmpq_set_si
#define mpq_canonicalize __gmpq_canonicalize
#define mpq_add __gmpq_add
#define mpq_sub __gmpq_sub
#define mpq_mul __gmpq_mul
#define mpq_div __gmpq_div
#define mpq_neg __gmpq_neg
#define mpq_cmp __gmpq_cmp
#define mpq_get_str __gmpq_get_str
#define mpq_swap __gmpq_swap
#define mpq_numref(q) (&(q)->_mp_num)
#define mpq_denref(q) (&(q)->_mp_den)

#endif
