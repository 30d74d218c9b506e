// mp_arith.cuh -- multiple-precision scalar primitives for sm_100a.
//
// Semantics are MPFR's round-to-nearest-even at precision p (reference:
// precision.hpp:127-161 -> mpfr_add / mpfr_sub / mpfr_mul / mpfr_div with MPFR_RNDN).
// Every operation is correctly rounded, so any sequence of them reproduces the
// reference's MPFR results bit for bit.
//
// Number format (registers / records): L 32-bit limbs, limb L-1 most significant,
// MSB of limb L-1 set for nonzero values, bits below p cleared; exponent e in the
// MPFR convention (value = 0.m * 2^e, 0.m in [1/2, 1)); sign s in {0,1}.
// Zero: e == EXP_ZERO (limbs 0), sign kept (MPFR signed zeros).
#pragma once
#include <cstdint>

// Limb loops: fully unrolled for the register-resident formats (L <= 32).  The wide
// formats (L = 64 .. 288, up to 9216 bits) are compiled in separate translation units
// (*_wide.cu, MPG_WIDE=1) where the same code runs as loops over local-memory arrays.
#if MPG_WIDE
#ifndef MPG_WIDE_UNROLL
#define MPG_WIDE_UNROLL 16  // measured: 2.5x faster than 1 on the 8192-bit Lotkin LU
#endif
#define MPG_STR2_(x) #x
#define MPG_STR_(x) MPG_STR2_(x)
#define MPG_UNROLL _Pragma(MPG_STR_(unroll MPG_WIDE_UNROLL))
#else
#define MPG_UNROLL _Pragma("unroll")
#endif
#ifndef MPG_SWAP_TOPLIMB
#define MPG_SWAP_TOPLIMB 1
#endif
#ifndef MPG_ADDW_FAST
#define MPG_ADDW_FAST 1  // measured: leaf -4.7 % at 256 bits, -3.7 % at 512, -1.7 % at 1024 (profiles/r02_ab_addw.jsonl)
#endif
#ifndef MPG_ADD_IMAD_XOR_MAXL
#define MPG_ADD_IMAD_XOR_MAXL 8  // measured: -1.2 % leaf time at 256 bits, +0.8 % at 512
#endif

namespace mpg {

constexpr int32_t EXP_ZERO = INT32_MIN;
// MPFR's default exponent range is [1-2^30, 2^30-1]; results outside it are flagged.
constexpr int32_t EXP_MAX = (1 << 30) - 1;
constexpr int32_t EXP_MIN = 1 - (1 << 30);
constexpr uint32_t ERR_EXP_RANGE = 1u;
constexpr uint32_t ERR_DIV_ZERO = 2u;

// Record stride (32-bit words) of one element in the AoS record layout:
// limbs[0..L-1], exp, sign, padding.  stride/4 is odd so that a quarter-warp of
// LDS.128 over consecutive records is bank-conflict free.
__host__ __device__ constexpr int rec_stride(int L) {
  int s = 4 * ((L + 2 + 3) / 4);
  return ((s / 4) % 2 == 0) ? s + 4 : s;
}

template <int L>
struct MP {
  uint32_t m[L];
  int32_t e;
  uint32_t s;
};

// ---------------------------------------------------------------------------
// full L x L -> 2L limb product, row-wise schoolbook with PTX carry chains.
// 2 L^2 multiply instructions (lo + hi) on the FMA pipe; the compiler maps the
// carries onto IADD3.X / IMAD.X.
// ---------------------------------------------------------------------------
#if MPG_WIDE
#undef MPG_MUL_EO
#define MPG_MUL_EO 0  // the wide formats loop over local-memory limbs: no PTX carry chains there
#elif !defined(MPG_MUL_EO)
#define MPG_MUL_EO 1
#endif
#ifndef MPG_EO_SKIPC
#define MPG_EO_SKIPC 1
#endif
#if MPG_MUL_EO
// Row-wise schoolbook on two sets of 64-bit column-pair accumulators: limb products a_i*b_j
// with i+j even accumulate into the pairs (2k, 2k+1) of X, those with i+j odd into the
// pairs (2k+1, 2k+2) of Y.  Within a row the products of one set tile consecutive pairs,
// so the row is two carry chains of `mad.lo.cc` / `madc.hi.cc` pairs, each pair fused by
// ptxas into ONE IMAD.WIDE.U32.X (64-bit product + 64-bit addend + carry in/out through a
// predicate): one instruction per limb product, no separate carry adds.  The carry out of a
// chain lands in the low limb of the next pair up, which until then has only received such
// carries (< L of them: the chains' upper ends are nondecreasing in i), so that add cannot
// overflow.  P = X + Y (one IADD3.X chain) at the end.  C0: lowest column kept
// (0: full product; L-2: the short product of mul_high_g, limbs below C0 stay 0).
template <int L>
__device__ __forceinline__ int eo_chain(uint32_t (&acc)[2 * L + 2], uint32_t ai, const uint32_t (&b)[L],
                                        int i, int js, int prev_top) {
  if (js >= L) return prev_top;
  asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
               : "+r"(acc[i + js]), "+r"(acc[i + js + 1])
               : "r"(ai), "r"(b[js]));
MPG_UNROLL
  for (int j = js + 2; j < L; j += 2)
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
                 : "+r"(acc[i + j]), "+r"(acc[i + j + 1])
                 : "r"(ai), "r"(b[j]));
  const int top = i + js + ((L - 1 - js) / 2) * 2 + 2;
  // The chain's last pair (top-2, top-1) holds a product of an earlier row only if that
  // row's chain ended on the same pair (prev_top == top); otherwise it holds at most L
  // carry counts and a*b + counts + carry-in < 2^64: no carry out, nothing to add.
  if (top < 2 * L && (!MPG_EO_SKIPC || prev_top == top)) asm volatile("addc.u32 %0, %0, 0;" : "+r"(acc[top]));
  return top;
}

template <int L, int C0, class AG>
__device__ __forceinline__ void mul_eo_g(AG a_at, const uint32_t (&b)[L], uint32_t (&r)[2 * L]) {
  uint32_t X[2 * L + 2], Y[2 * L + 2];
MPG_UNROLL
  for (int k = 0; k < 2 * L + 2; ++k) X[k] = Y[k] = 0;
  int xtop = -1, ytop = -1;  // upper ends of the previous row's chains (compile-time after unrolling)
MPG_UNROLL
  for (int i = 0; i < L; ++i) {
    const uint32_t ai = a_at(i);
    const int j0 = (C0 - i) > 0 ? (C0 - i) : 0;
    xtop = eo_chain<L>(X, ai, b, i, j0 + ((i + j0) & 1), xtop);        // i + j even
    ytop = eo_chain<L>(Y, ai, b, i, j0 + (((i + j0) & 1) ^ 1), ytop);  // i + j odd
  }
MPG_UNROLL
  for (int k = 0; k < C0; ++k) r[k] = 0;
  // limb C0 belongs to one set only (X when C0 is even, Y when odd): the carry chain starts above it
  r[C0] = (C0 & 1) ? Y[C0] : X[C0];
  if (C0 + 1 == 2 * L - 1) {
    r[C0 + 1] = X[C0 + 1] + Y[C0 + 1];
  } else if (C0 + 1 < 2 * L - 1) {
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r[C0 + 1]) : "r"(X[C0 + 1]), "r"(Y[C0 + 1]));
MPG_UNROLL
    for (int k = C0 + 2; k < 2 * L - 1; ++k)
      asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r[k]) : "r"(X[k]), "r"(Y[k]));
    asm volatile("addc.u32 %0, %1, %2;" : "=r"(r[2 * L - 1]) : "r"(X[2 * L - 1]), "r"(Y[2 * L - 1]));
  }
}

template <int L, class AG>
__device__ __forceinline__ void mul_full_g(AG a_at, const uint32_t (&b)[L], uint32_t (&r)[2 * L]) {
  if constexpr (L == 1) {
    const uint64_t t = (uint64_t)a_at(0) * b[0];
    r[0] = (uint32_t)t;
    r[1] = (uint32_t)(t >> 32);
  } else {
    mul_eo_g<L, 0>(a_at, b, r);
  }
}
#elif !defined(MPG_MUL_PTX_CHAINS)
// Row-wise schoolbook on 64-bit partial sums: t = a_i*b_j + r[i+j] + carry never
// overflows 64 bits, and maps onto one IMAD.WIDE.U32 (product + 64-bit addend)
// plus ~1.3 ALU carry ops per limb product -- no half-rate IMAD.HI.
template <int L, class AG>
__device__ __forceinline__ void mul_full_g(AG a_at, const uint32_t (&b)[L], uint32_t (&r)[2 * L]) {
MPG_UNROLL
  for (int i = 0; i < 2 * L; ++i) r[i] = 0;
MPG_UNROLL
  for (int i = 0; i < L; ++i) {
    const uint32_t ai = a_at(i);
    uint32_t carry = 0;
MPG_UNROLL
    for (int j = 0; j < L; ++j) {
      const uint64_t t = (uint64_t)ai * b[j] + r[i + j] + carry;
      r[i + j] = (uint32_t)t;
      carry = (uint32_t)(t >> 32);
    }
    r[i + L] = carry;
  }
}
#else
template <int L, class AG>
__device__ __forceinline__ void mul_full_g(AG a_at, const uint32_t (&b)[L], uint32_t (&r)[2 * L]) {
MPG_UNROLL
  for (int i = 0; i < 2 * L; ++i) r[i] = 0;
MPG_UNROLL
  for (int i = 0; i < L; ++i) {
    const uint32_t ai = a_at(i);
    if (L == 1) {
      asm("mul.lo.u32 %0, %1, %2;" : "=r"(r[0]) : "r"(ai), "r"(b[0]));
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(r[1]) : "r"(ai), "r"(b[0]));
    } else {
      asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(r[i]) : "r"(ai), "r"(b[0]));
MPG_UNROLL
      for (int j = 1; j < L; ++j)
        asm volatile("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + j]) : "r"(ai), "r"(b[j]));
      asm volatile("addc.u32 %0, %0, 0;" : "+r"(r[i + L]));
      asm volatile("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + 1]) : "r"(ai), "r"(b[0]));
MPG_UNROLL
      for (int j = 1; j < L; ++j)
        asm volatile("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(r[i + j + 1]) : "r"(ai), "r"(b[j]));
      if (i + L + 1 < 2 * L) asm volatile("addc.u32 %0, %0, 0;" : "+r"(r[i + L + 1]));
    }
  }
}
#endif

template <int L>
__device__ __forceinline__ void mul_full(const uint32_t (&a)[L], const uint32_t (&b)[L],
                                         uint32_t (&r)[2 * L]) {
  mul_full_g<L>([&](int i) { return a[i]; }, b, r);
}

// Truncated ("short") product: T = sum_{i+j >= L-2} a_i b_j 2^(32(i+j)), exact.
// The omitted part E = P - T satisfies 0 <= E < (L-1) * 2^(32(L-1)), i.e. less than
// L-1 units of limb L-1 -- enough to decide round-to-nearest from T almost always
// (mp_mul_g checks and falls back to the full product).  (L^2 + 3L - 2)/2 limb
// products instead of L^2 -- the mulhigh trick MPFR itself uses for mpfr_mul.
template <int L, class AG>
__device__ __forceinline__ void mul_high_g(AG a_at, const uint32_t (&b)[L], uint32_t (&r)[2 * L]) {
#if MPG_MUL_EO
  if constexpr (L >= 3) {
    mul_eo_g<L, L - 2>(a_at, b, r);
  } else
#endif
  {
MPG_UNROLL
    for (int i = 0; i < 2 * L; ++i) r[i] = 0;
MPG_UNROLL
    for (int i = 0; i < L; ++i) {
      const uint32_t ai = a_at(i);
      const int j0 = (L - 2 - i) > 0 ? (L - 2 - i) : 0;
      uint32_t carry = 0;
MPG_UNROLL
      for (int j = j0; j < L; ++j) {
        const uint64_t t = (uint64_t)ai * b[j] + r[i + j] + carry;
        r[i + j] = (uint32_t)t;
        carry = (uint32_t)(t >> 32);
      }
      r[i + L] = carry;
    }
  }
}

// add a single word w at limb 0 with full carry propagation; returns carry-out
template <int L>
__device__ __forceinline__ uint32_t add_word(uint32_t (&m)[L], uint32_t w) {
  if constexpr (L > 32) {  // wide formats: plain 64-bit carries (no PTX carry chains in loops)
    uint64_t c = w;
    for (int k = 0; k < L && c; ++k) {
      const uint64_t t = (uint64_t)m[k] + c;
      m[k] = (uint32_t)t;
      c = t >> 32;
    }
    return (uint32_t)c;
  }
  uint32_t c;
#if MPG_ADDW_FAST
  if (L >= 4) {
    // the carry out of limb 0 is rare (rounding increments): one add, the chain only on carry
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(w));
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
    if (__builtin_expect(c != 0, 0)) {
      c = 1;
MPG_UNROLL
      for (int k = 1; k < L; ++k) {
        m[k] += c;
        c = (m[k] == 0) & c;
      }
    }
    return c;
  }
#endif
  if (L == 1) {
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(w));
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
    return c;
  }
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(w));
MPG_UNROLL
  for (int k = 1; k < L; ++k) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(m[k]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  return c;
}

// m += w at limb 0 for a rounding increment; a carry out of the top limb leaves the
// mantissa 1000...0 and bumps e.
template <int L>
__device__ __forceinline__ void round_inc(uint32_t (&m)[L], uint32_t w, int32_t& e) {
  // (one rare branch for the carry out of limb 0 inside add_word, a second for the
  // carry out of the top: measured 0.7 % faster than nesting the second in the first)
  if (add_word<L>(m, w)) {
MPG_UNROLL
    for (int k = 0; k < L - 1; ++k) m[k] = 0;
    m[L - 1] = 0x80000000u;
    e += 1;
  }
}

// ---------------------------------------------------------------------------
// Round-to-nearest-even of an L-limb normalised mantissa m (MSB set) followed by
// a guard limb g and a sticky word st (nonzero iff anything nonzero lies below g),
// to p = 32L - sh bits.  Bumps e on carry-out (mantissa becomes 1000...).
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void round_p(uint32_t (&m)[L], uint32_t g, uint32_t st, int sh,
                                        int32_t& e) {
  uint32_t up_word;
  if (sh == 0) {
    const uint32_t rb = g >> 31;
    const uint32_t rest = (g << 1) | st;
    const uint32_t up = rb & ((rest != 0) | (m[0] & 1u));
    up_word = up;
  } else if (sh < 32) {
    const uint32_t low = m[0] & ((1u << sh) - 1u);
    const uint32_t rb = (low >> (sh - 1)) & 1u;
    const uint32_t rest = (low & ((1u << (sh - 1)) - 1u)) | g | st;
    const uint32_t lsb = (m[0] >> sh) & 1u;
    m[0] ^= low;
    const uint32_t up = rb & ((rest != 0) | lsb);
    up_word = up << sh;
  } else {
    // generic path: the precision ends inside a lower limb (L chosen larger than ceil(p/32))
    const int rbpos = sh - 1, rl = rbpos >> 5, rbit = rbpos & 31;
    const int ql = sh >> 5, qb = sh & 31;
    uint32_t stk = g | st, rb = 0, lsb = 0;
MPG_UNROLL
    for (int k = 0; k < L; ++k) {
      uint32_t v = m[k];
      if (k < rl) {
        stk |= v;
        v = 0;
      } else if (k == rl) {
        rb = (v >> rbit) & 1u;
        stk |= v & ((1u << rbit) - 1u);
        v &= (rbit == 31) ? 0u : ~((2u << rbit) - 1u);
      }
      if (k == ql) lsb = (v >> qb) & 1u;
      m[k] = v;
    }
    const uint32_t up = rb & ((stk != 0) | lsb);
    uint32_t c = 0;
MPG_UNROLL
    for (int k = 0; k < L; ++k) {
      const uint32_t addend = (k == ql) ? (up << qb) : 0u;
      const uint64_t t = (uint64_t)m[k] + addend + c;
      m[k] = (uint32_t)t;
      c = (uint32_t)(t >> 32);
    }
    if (c) {
MPG_UNROLL
      for (int k = 0; k < L - 1; ++k) m[k] = 0;
      m[L - 1] = 0x80000000u;
      e += 1;
    }
    return;
  }
  round_inc<L>(m, up_word, e);
}

// ---------------------------------------------------------------------------
// z = RN_p(x * y)   (mpfr_mul, precision.hpp:145-151; matrix.hpp:150,152)
// ---------------------------------------------------------------------------
// NZ: the caller guarantees both operands are nonzero (no zero test)
template <int L, class AG, bool NZ = false>
__device__ __forceinline__ void mp_mul_g(AG a_at, int32_t xe, uint32_t xs, const MP<L>& y, int sh,
                                         MP<L>& z) {
  z.s = xs ^ y.s;
  if (!NZ && (xe == EXP_ZERO || y.e == EXP_ZERO)) {
MPG_UNROLL
    for (int k = 0; k < L; ++k) z.m[k] = 0;
    z.e = EXP_ZERO;
    return;
  }
  uint32_t P[2 * L];
  if (L >= 3 && sh == 0) {
    mul_high_g<L>(a_at, y.m, P);
    const uint32_t t1 = (P[2 * L - 1] >> 31) ^ 1u;
    const uint32_t gt = __funnelshift_l(P[L >= 3 ? L - 2 : 0], P[L - 1], t1);
    // true guard limb lies in [gt, gt + 2L]: decide the rounding from T when no
    // boundary (half-way point or carry into the mantissa) is within reach
    const bool down = gt < 0x80000000u - 2u * L;
    const bool up = gt > 0x80000000u && gt < 0xFFFFFFFFu - 2u * L;
    if (down | up) {
MPG_UNROLL
      for (int k = 0; k < L; ++k) z.m[k] = __funnelshift_l(P[L + k - 1], P[L + k], t1);
      int32_t e = xe + y.e - (int32_t)t1;
      round_inc<L>(z.m, up ? 1u : 0u, e);
      z.e = e;
      return;
    }
  }
  mul_full_g<L>(a_at, y.m, P);
  // normalise branch-free: shift left by one when the product's top bit is clear
  const uint32_t s1 = (P[2 * L - 1] >> 31) ^ 1u;
  const int32_t e = xe + y.e - (int32_t)s1;
MPG_UNROLL
  for (int k = 0; k < L; ++k) z.m[k] = __funnelshift_l(P[L + k - 1], P[L + k], s1);
  uint32_t g, st = 0;
  if (L >= 2) {
    g = __funnelshift_l(P[L >= 2 ? L - 2 : 0], P[L - 1], s1);
MPG_UNROLL
    for (int k = 0; k < L - 2; ++k) st |= P[k];
    st |= P[L >= 2 ? L - 2 : 0] << s1;
  } else {
    g = P[0] << s1;
  }
  int32_t ee = e;
  round_p<L>(z.m, g, st, sh, ee);
  z.e = ee;
}

template <int L>
__device__ __forceinline__ void mp_mul(const MP<L>& x, const MP<L>& y, int sh, MP<L>& z) {
  mp_mul_g<L>([&](int i) { return x.m[i]; }, x.e, x.s, y, sh, z);
}

// ---------------------------------------------------------------------------
// z = RN_p(x + (-1)^negy * y)  (mpfr_add / mpfr_sub, matrix.hpp:128,130,153)
// Exact-alignment algorithm over an (L+1)-limb window (one guard limb) plus a
// sticky bit; see DESIGN.md "MP add".  Exact cancellation gives +0 (RNDN).
// ---------------------------------------------------------------------------
// NZ: the caller guarantees both operands are nonzero (no zero test)
template <int L, bool NZ = false>
__device__ __forceinline__ void mp_add(const MP<L>& x, const MP<L>& y_in, uint32_t negy, int sh,
                                       MP<L>& z) {
  // z may alias x or y: every input is read before z is written.
  const uint32_t ys = y_in.s ^ negy;
  if (!NZ && (x.e == EXP_ZERO || y_in.e == EXP_ZERO)) {
    if (x.e == EXP_ZERO && y_in.e == EXP_ZERO) {
      const uint32_t zs = x.s & ys;  // (-0) + (-0) = -0, otherwise +0 under RNDN
MPG_UNROLL
      for (int k = 0; k < L; ++k) z.m[k] = 0;
      z.e = EXP_ZERO;
      z.s = zs;
    } else if (x.e == EXP_ZERO) {
MPG_UNROLL
      for (int k = 0; k < L; ++k) z.m[k] = y_in.m[k];
      z.e = y_in.e;
      z.s = ys;
    } else {
      z = x;
    }
    return;
  }
  constexpr int W = L + 1;
  // exponent order, ties broken by the top limbs: then big - small is negative (the rare
  // negation path below) only when exponents AND top limbs are equal, instead of for about
  // half of the equal-exponent subtractions (measured: ~35 % of the leaf's warp-steps had a
  // lane on that path)
#if MPG_SWAP_TOPLIMB
  const bool swp = y_in.e > x.e || (y_in.e == x.e && y_in.m[L - 1] > x.m[L - 1]);
#else
  const bool swp = y_in.e > x.e;
#endif
  uint32_t A[W], B[W];
  A[0] = 0;
  B[0] = 0;
MPG_UNROLL
  for (int k = 0; k < L; ++k) {
    A[k + 1] = swp ? y_in.m[k] : x.m[k];
    B[k + 1] = swp ? x.m[k] : y_in.m[k];
  }
  const int32_t ebig = swp ? y_in.e : x.e;
  const uint32_t d = (uint32_t)(swp ? y_in.e - x.e : x.e - y_in.e);
  const uint32_t sbig = swp ? ys : x.s;
  const uint32_t ssmall = swp ? x.s : ys;
  const uint32_t sub = sbig ^ ssmall;

  // ---- align B right by d bits.  d < 32 (the common case) shifts inside the
  // window and loses nothing; larger gaps shift limbs and collect a sticky bit.
  uint32_t st = 0;
  if (d >= 32u) {
    if (d >= 32u * W) {
      st = 1;
MPG_UNROLL
      for (int k = 0; k < W; ++k) B[k] = 0;
    } else {
      uint32_t q = d >> 5;
      const uint32_t r = d & 31u;
      while (q) {
        st |= B[0];
MPG_UNROLL
        for (int k = 0; k < W - 1; ++k) B[k] = B[k + 1];
        B[W - 1] = 0;
        --q;
      }
      st |= B[0] & ((1u << r) - 1u);
MPG_UNROLL
      for (int k = 0; k < W - 1; ++k) B[k] = __funnelshift_r(B[k], B[k + 1], r);
      B[W - 1] >>= r;
      st = st != 0;
    }
  } else {
MPG_UNROLL
    for (int k = 0; k < W - 1; ++k) B[k] = __funnelshift_r(B[k], B[k + 1], d);
    B[W - 1] >>= d;
  }

  // ---- R = A + B (add) or A - B - st = A + ~B + (1 - st) (sub), one carry chain
  const uint32_t mask = 0u - sub;
  const uint32_t cin = sub & (st ^ 1u);
  uint32_t R[W], cout;
  if constexpr (L > 32) {
    uint64_t c = (uint64_t)(B[0] ^ mask) + cin;  // A[0] == 0
    R[0] = (uint32_t)c;
    c >>= 32;
    for (int k = 1; k < W; ++k) {
      c += (uint64_t)A[k] + (B[k] ^ mask);
      R[k] = (uint32_t)c;
      c >>= 32;
    }
    cout = (uint32_t)c;
  } else {
    if constexpr (L <= MPG_ADD_IMAD_XOR_MAXL) {
      // B ^ mask as B * (1 - 2 sub) - sub: IMAD on the FMA pipe instead of LOP3 on the
      // ALU pipe, which binds the leaf at these precisions
      const uint32_t m1 = 1u - 2u * sub;
MPG_UNROLL
      for (int k = 0; k < W; ++k) B[k] = B[k] * m1 + mask;
    } else {
MPG_UNROLL
      for (int k = 0; k < W; ++k) B[k] ^= mask;
    }
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(R[0]) : "r"(B[0]), "r"(cin));  // A[0] == 0
MPG_UNROLL
    for (int k = 1; k < W; ++k)
      asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(R[k]) : "r"(A[k]), "r"(B[k]));
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(cout));
  }
  int32_t e = ebig;
  uint32_t s = sbig;
  if (sub & ((cout ^ 1u) | (R[W - 1] == 0))) {  // rare: |small| > |big| (d == 0) or deep cancellation
    if (!cout) {
      if constexpr (L > 32) {  // R = -R
        uint64_t bo = 0;
        for (int k = 0; k < W; ++k) {
          const uint64_t d = 0ull - R[k] - bo;
          R[k] = (uint32_t)d;
          bo = (d >> 32) & 1u;
        }
      } else {
        asm volatile("sub.cc.u32 %0, 0, %0;" : "+r"(R[0]));
MPG_UNROLL
        for (int k = 1; k < W; ++k) asm volatile("subc.cc.u32 %0, 0, %0;" : "+r"(R[k]));
      }
      s = ssmall;
    }
    uint32_t any = 0;
MPG_UNROLL
    for (int k = 0; k < W; ++k) any |= R[k];
    if (!any) {  // exact cancellation: +0 under RNDN
MPG_UNROLL
      for (int k = 0; k < L; ++k) z.m[k] = 0;
      z.e = EXP_ZERO;
      z.s = 0;
      return;
    }
    while (R[W - 1] == 0) {
MPG_UNROLL
      for (int k = W - 1; k > 0; --k) R[k] = R[k - 1];
      R[0] = 0;
      e -= 32;
    }
  }
  // ---- normalise branch-free: add overflow shifts right by one, cancellation left by lz
  const uint32_t c1 = cout & (sub ^ 1u);
  st |= R[0] & c1;
MPG_UNROLL
  for (int k = 0; k < W - 1; ++k) R[k] = __funnelshift_r(R[k], R[k + 1], c1);
  R[W - 1] = (R[W - 1] >> c1) | (c1 << 31);
  const uint32_t lz = __clz(R[W - 1]);
MPG_UNROLL
  for (int k = W - 1; k > 0; --k) R[k] = __funnelshift_l(R[k - 1], R[k], lz);
  R[0] <<= lz;
  e += (int32_t)c1 - (int32_t)lz;
MPG_UNROLL
  for (int k = 0; k < L; ++k) z.m[k] = R[k + 1];
  round_p<L>(z.m, R[0], st, sh, e);
  z.e = e;
  z.s = s;
}

// ---------------------------------------------------------------------------
// z = RN_p(x / y)   (mpfr_div, precision.hpp:154-161; blocklu.hpp:49,84,241)
// Restoring division producing ceil((p+2)/32) quotient limbs, left aligned, with
// the remainder as sticky; y must be nonzero (callers check, SingularError).
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void mp_div_bits(const MP<L>& x, const MP<L>& y, int sh, MP<L>& z) {
  z.s = x.s ^ y.s;
  if (x.e == EXP_ZERO || y.e == EXP_ZERO) {
MPG_UNROLL
    for (int k = 0; k < L; ++k) z.m[k] = 0;
    z.e = EXP_ZERO;
    return;
  }
  constexpr int W = L + 1;
  const int p = 32 * L - sh;
  const int nl = (p + 2 + 31) >> 5;  // quotient limbs to produce (<= W)
  uint32_t R[W], Q[W];
MPG_UNROLL
  for (int k = 0; k < L; ++k) R[k] = x.m[k];
  R[L] = 0;
MPG_UNROLL
  for (int k = 0; k < W; ++k) Q[k] = 0;
  bool first_bit = true;
MPG_UNROLL
  for (int ql = W - 1; ql >= 0; --ql) {
    if (W - 1 - ql < nl) {
      uint32_t word = 0;
#pragma unroll 1
      for (int b = 0; b < 32; ++b) {
        if (!first_bit) {  // R <<= 1
MPG_UNROLL
          for (int k = W - 1; k > 0; --k) R[k] = __funnelshift_l(R[k - 1], R[k], 1);
          R[0] <<= 1;
        }
        first_bit = false;
        // T = R - Y (Y has a zero top limb)
        uint32_t T[W], bo;
        asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(T[0]) : "r"(R[0]), "r"(y.m[0]));
MPG_UNROLL
        for (int k = 1; k < L; ++k) asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(T[k]) : "r"(R[k]), "r"(y.m[k]));
        asm volatile("subc.cc.u32 %0, %1, 0;" : "=r"(T[L]) : "r"(R[L]));
        asm volatile("subc.u32 %0, 0, 0;" : "=r"(bo));
        const uint32_t qb = bo ? 0u : 1u;
MPG_UNROLL
        for (int k = 0; k < W; ++k) R[k] = qb ? T[k] : R[k];
        word = (word << 1) | qb;
      }
      Q[ql] = word;
    }
  }
  uint32_t rem = 0;
MPG_UNROLL
  for (int k = 0; k < W; ++k) rem |= R[k];
  int32_t e = x.e - y.e;
  if (Q[W - 1] >> 31) {
    e += 1;
  } else {
MPG_UNROLL
    for (int k = W - 1; k > 0; --k) Q[k] = __funnelshift_l(Q[k - 1], Q[k], 1);
    Q[0] <<= 1;
  }
MPG_UNROLL
  for (int k = 0; k < L; ++k) z.m[k] = Q[k + 1];
  round_p<L>(z.m, Q[0], rem, sh, e);
  z.e = e;
}

// ---------------------------------------------------------------------------
// z = RN_p(x / y), radix-2^32 digit recurrence (Knuth D style): L+1 quotient digits,
// each estimated from the top of the remainder with directed-rounding FP64
// (never an overestimate) and corrected by at most a few add-backs; the final
// remainder is the sticky bit.  ~(L+1)(4L+20) instructions instead of the
// bit-serial mp_div_bits' ~32(L+1)(3L+3).
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void mp_div(const MP<L>& x, const MP<L>& y, int sh, MP<L>& z) {
  z.s = x.s ^ y.s;
  if (x.e == EXP_ZERO || y.e == EXP_ZERO) {
MPG_UNROLL
    for (int k = 0; k < L; ++k) z.m[k] = 0;
    z.e = EXP_ZERO;
    return;
  }
  constexpr int W = L + 1;
  uint32_t R[W];
MPG_UNROLL
  for (int k = 0; k < L; ++k) R[k] = x.m[k];
  R[L] = 0;
  // R -= Y if R >= Y; returns 1 if subtracted
  auto try_sub = [&]() -> uint32_t {
    uint32_t T[W], bo;
    if constexpr (L > 32) {
      uint64_t b = 0;
      for (int k = 0; k < W; ++k) {
        const uint64_t d = (uint64_t)R[k] - (k < L ? y.m[k < L ? k : 0] : 0u) - b;
        T[k] = (uint32_t)d;
        b = (d >> 32) & 1u;
      }
      bo = (uint32_t)b;
    } else {
      asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(T[0]) : "r"(R[0]), "r"(y.m[0]));
MPG_UNROLL
      for (int k = 1; k < L; ++k)
        asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(T[k]) : "r"(R[k]), "r"(y.m[k]));
      asm volatile("subc.cc.u32 %0, %1, 0;" : "=r"(T[L]) : "r"(R[L]));
      asm volatile("subc.u32 %0, 0, 0;" : "=r"(bo));
    }
    const uint32_t ok = bo ? 0u : 1u;
MPG_UNROLL
    for (int k = 0; k < W; ++k) R[k] = ok ? T[k] : R[k];
    return ok;
  };
  // quotient digits, most significant first: Q[W] = q0 in {0,1}, then Q[W-1..0]
  uint32_t Q[W + 1];
  Q[W] = try_sub();
  // divisor estimate in units of 2^(32(L-2)), rounded UP (so digit estimates never exceed)
  const uint64_t ytop = ((uint64_t)y.m[L - 1] << 32) | (L >= 2 ? y.m[L >= 2 ? L - 2 : 0] : 0u);
  const double yd = __dadd_ru(__ull2double_ru(ytop), (L >= 3) ? 1.0 : 0.0);
  const double inv = __drcp_rd(yd);
#pragma unroll 1
  for (int t = W - 1; t >= 0; --t) {
    // R <<= 32 (R < Y, so the top limb is free)
MPG_UNROLL
    for (int k = W - 1; k > 0; --k) R[k] = R[k - 1];
    R[0] = 0;
    // estimate q = floor(R / Y) from the top three limbs of R, rounded down
    const uint64_t rtop = ((uint64_t)R[L] << 32) | R[L - 1];
    double rd = __dmul_rd(__ull2double_rd(rtop), 4294967296.0);
    if (L >= 2) rd = __dadd_rd(rd, (double)R[L >= 2 ? L - 2 : 0]);
    const double qd = floor(__dmul_rd(rd, inv));
    uint32_t qh = qd >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)qd;
    // R -= qh * Y (exact, W limbs); qh <= q so no underflow
    uint32_t c = 0, b = 0;
MPG_UNROLL
    for (int j = 0; j < L; ++j) {
      const uint64_t pr = (uint64_t)qh * y.m[j] + c;
      c = (uint32_t)(pr >> 32);
      const uint64_t d = (uint64_t)R[j] - (uint32_t)pr - b;
      R[j] = (uint32_t)d;
      b = (uint32_t)(d >> 63);
    }
    R[L] = R[L] - c - b;
    // corrections: the estimate is never high and short by at most a little; R >= Y needs
    // R[L] > 0 or R[L-1] >= Y[L-1], so the full trial subtraction runs only then
    if (R[L] != 0 || R[L - 1] >= y.m[L - 1])
      while (try_sub()) ++qh;
    Q[t] = qh;
  }
  uint32_t rem = 0;
MPG_UNROLL
  for (int k = 0; k < W; ++k) rem |= R[k];
  // normalise: value = Q[W] . Q[W-1] Q[W-2] ... (radix 2^32)
  int32_t e = x.e - y.e;
  uint32_t M[W];
  if (Q[W]) {  // quotient in [1, 2): shift the digit string right by one bit
MPG_UNROLL
    for (int k = 0; k < W; ++k) M[k] = __funnelshift_r(Q[k], Q[k + 1], 1);
    rem |= Q[0] & 1u;
    e += 1;
  } else {
MPG_UNROLL
    for (int k = 0; k < W; ++k) M[k] = Q[k];
  }
MPG_UNROLL
  for (int k = 0; k < L; ++k) z.m[k] = M[k + 1];
  round_p<L>(z.m, M[0], rem, sh, e);
  z.e = e;
}

template <int L>
__device__ __forceinline__ void mp_zero(MP<L>& z, uint32_t s = 0) {
MPG_UNROLL
  for (int k = 0; k < L; ++k) z.m[k] = 0;
  z.e = EXP_ZERO;
  z.s = s;
}

// |x| vs |y|: -1, 0, 1  (for pivot search)
template <int L>
__device__ __forceinline__ int mp_cmpabs(const MP<L>& x, const MP<L>& y) {
  const bool xz = x.e == EXP_ZERO, yz = y.e == EXP_ZERO;
  if (xz || yz) return xz ? (yz ? 0 : -1) : 1;
  if (x.e != y.e) return x.e > y.e ? 1 : -1;
MPG_UNROLL
  for (int k = L - 1; k >= 0; --k)
    if (x.m[k] != y.m[k]) return x.m[k] > y.m[k] ? 1 : -1;
  return 0;
}

__device__ __forceinline__ bool exp_out_of_range(int32_t e) {
  return e != EXP_ZERO && (e > EXP_MAX || e < EXP_MIN);
}

// ---------------------------------------------------------------------------
// record I/O (AoS records of rec_stride(L) words)
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void load_rec(const uint32_t* __restrict__ r, MP<L>& x) {
  constexpr int S = rec_stride(L);
  static_assert(S % 4 == 0, "record stride must be a multiple of 4 words");
  uint32_t w[S];
MPG_UNROLL
  for (int k = 0; k < S; k += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(r + k);
    w[k] = v.x;
    w[k + 1] = v.y;
    w[k + 2] = v.z;
    w[k + 3] = v.w;
  }
MPG_UNROLL
  for (int k = 0; k < L; ++k) x.m[k] = w[k];
  x.e = (int32_t)w[L];
  x.s = w[L + 1];
}

// scalar-load variant (no 4-register alignment constraint on the destination):
// lets the register allocator keep loop-carried accumulators in place
template <int L>
__device__ __forceinline__ void load_rec_s(const uint32_t* __restrict__ r, MP<L>& x) {
MPG_UNROLL
  for (int k = 0; k < L; ++k) x.m[k] = r[k];
  x.e = (int32_t)r[L];
  x.s = r[L + 1];
}

template <int L>
__device__ __forceinline__ void store_rec(uint32_t* __restrict__ r, const MP<L>& x) {
  constexpr int S = rec_stride(L);
  uint32_t w[S];
MPG_UNROLL
  for (int k = 0; k < L; ++k) w[k] = x.m[k];
  w[L] = (uint32_t)x.e;
  w[L + 1] = x.s;
MPG_UNROLL
  for (int k = L + 2; k < S; ++k) w[k] = 0;
MPG_UNROLL
  for (int k = 0; k < S; k += 4)
    *reinterpret_cast<uint4*>(r + k) = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
}

}  // namespace mpg
