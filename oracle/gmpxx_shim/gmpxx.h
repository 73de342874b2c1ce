// Minimal stand-in for <gmpxx.h> (GMP's C++ header is not installed in this
// image; only the runtime libgmp.so.10 is).  TEST INFRASTRUCTURE: used solely
// to compile the reference encoder (/root/reference/proj/src/encoder.cpp,
// decode CRT at :124-152) into oracle/_ref/.  Declares the handful of
// libgmp C entry points by their exported (__gmpz_*) names and wraps them in
// an mpz_class offering exactly the operators that file uses.
#pragma once

#include <cstddef>

extern "C" {
struct hx_mpz_struct {
  int alloc;
  int size;
  unsigned long* d;
};
void __gmpz_init(hx_mpz_struct*);
void __gmpz_clear(hx_mpz_struct*);
void __gmpz_init_set(hx_mpz_struct*, const hx_mpz_struct*);
void __gmpz_set(hx_mpz_struct*, const hx_mpz_struct*);
void __gmpz_set_ui(hx_mpz_struct*, unsigned long);
void __gmpz_set_si(hx_mpz_struct*, long);
void __gmpz_mul(hx_mpz_struct*, const hx_mpz_struct*, const hx_mpz_struct*);
void __gmpz_mul_ui(hx_mpz_struct*, const hx_mpz_struct*, unsigned long);
void __gmpz_add(hx_mpz_struct*, const hx_mpz_struct*, const hx_mpz_struct*);
void __gmpz_sub(hx_mpz_struct*, const hx_mpz_struct*, const hx_mpz_struct*);
unsigned long __gmpz_tdiv_q_ui(hx_mpz_struct*, const hx_mpz_struct*, unsigned long);
unsigned long __gmpz_tdiv_r_ui(hx_mpz_struct*, const hx_mpz_struct*, unsigned long);
void __gmpz_tdiv_r(hx_mpz_struct*, const hx_mpz_struct*, const hx_mpz_struct*);
int __gmpz_cmp(const hx_mpz_struct*, const hx_mpz_struct*);
double __gmpz_get_d(const hx_mpz_struct*);
unsigned long __gmpz_get_ui(const hx_mpz_struct*);
}

class mpz_class {
 public:
  mpz_class() { __gmpz_init(&v_); }
  mpz_class(int x) { __gmpz_init(&v_); __gmpz_set_si(&v_, x); }
  mpz_class(long x) { __gmpz_init(&v_); __gmpz_set_si(&v_, x); }
  mpz_class(unsigned long x) { __gmpz_init(&v_); __gmpz_set_ui(&v_, x); }
  mpz_class(const mpz_class& o) { __gmpz_init_set(&v_, &o.v_); }
  ~mpz_class() { __gmpz_clear(&v_); }

  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) __gmpz_set(&v_, &o.v_);
    return *this;
  }
  mpz_class& operator=(int x) { __gmpz_set_si(&v_, x); return *this; }

  mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(&v_, &v_, &o.v_); return *this; }
  mpz_class& operator+=(const mpz_class& o) { __gmpz_add(&v_, &v_, &o.v_); return *this; }
  mpz_class& operator-=(const mpz_class& o) { __gmpz_sub(&v_, &v_, &o.v_); return *this; }
  mpz_class& operator%=(const mpz_class& o) { __gmpz_tdiv_r(&v_, &v_, &o.v_); return *this; }

  friend mpz_class operator/(const mpz_class& a, unsigned long b) {
    mpz_class r;
    __gmpz_tdiv_q_ui(&r.v_, &a.v_, b);
    return r;
  }
  friend mpz_class operator/(const mpz_class& a, int b) {
    return a / static_cast<unsigned long>(b);
  }
  friend mpz_class operator%(const mpz_class& a, unsigned long b) {
    mpz_class r;
    __gmpz_tdiv_r_ui(&r.v_, &a.v_, b);
    return r;
  }
  friend mpz_class operator*(const mpz_class& a, unsigned long b) {
    mpz_class r;
    __gmpz_mul_ui(&r.v_, &a.v_, b);
    return r;
  }
  friend bool operator>(const mpz_class& a, const mpz_class& b) {
    return __gmpz_cmp(&a.v_, &b.v_) > 0;
  }

  double get_d() const { return __gmpz_get_d(&v_); }
  unsigned long get_ui() const { return __gmpz_get_ui(&v_); }

 private:
  hx_mpz_struct v_;
};
