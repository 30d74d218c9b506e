// wmp.cuh -- warp-cooperative MP primitives for the wide formats (L = 32 V limbs,
// V = 2, 4, 8, 9 limbs per lane: 2048 .. 9216 bits).
//
// One warp owns one MP number: lane l holds limbs [l V, l V + V) (limb 0 least
// significant, limb L-1 = lane 31's m[V-1] most significant); the exponent and sign
// are warp-uniform.  Carries between lanes are resolved with a carry-lookahead over
// two ballots (generate / propagate), bit shifts take the neighbour lane's edge limb
// with one shuffle, products are formed column-wise by the 32 lanes from operands
// staged in shared memory.  Semantics are exactly mp_arith.cuh's (MPFR round-to-
// nearest-even at p = 32 L - sh bits): every operation is correctly rounded, so the
// results are bit-identical to the thread-per-element code and to the reference.
//
// Replaces, for the wide formats only, the thread-per-element primitives whose 1 KB
// mantissas live in local memory (latency-bound, one element per thread).
#pragma once
#ifndef MPG_WMUL_FUSED
#define MPG_WMUL_FUSED 1
#endif
#include <cstdint>

#include "mp_arith.cuh"

namespace mpg {
namespace wmp {

constexpr unsigned FULL = 0xffffffffu;
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <int V>
struct W {
  uint32_t m[V];  // this lane's limbs
  int32_t e;      // warp-uniform
  uint32_t s;     // warp-uniform
};

// per-warp shared-memory scratch (words): see scratch_words()
template <int V>
struct Scratch {
  uint32_t* a;    // L + 8 words   (a[4 + k] = limb k, zero pads)
  uint32_t* b;    // L + 80 words  (b[40 + k] = limb k, zero pads)
  uint32_t* col;  // 6 L words     (3 words per product column)
};
template <int V>
__host__ __device__ constexpr int scratch_words() {
  return (32 * V + 8) + (32 * V + 80) + 6 * 32 * V;
}
template <int V>
__device__ __forceinline__ Scratch<V> scratch_at(uint32_t* base) {
  constexpr int L = 32 * V;
  Scratch<V> s;
  s.a = base;
  s.b = base + (L + 8);
  s.col = base + (L + 8) + (L + 80);
  return s;
}

// ---- helpers ---------------------------------------------------------------
// limb k (runtime, warp-uniform) of a distributed number, broadcast to all lanes
template <int V>
__device__ __forceinline__ uint32_t get_limb(const uint32_t (&m)[V], int k) {
  const int r = k % V;
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < V; ++j)
    if (j == r) v = m[j];
  return __shfl_sync(FULL, v, k / V);
}

template <int V>
__device__ __forceinline__ uint32_t all_ones(const uint32_t (&m)[V]) {
  uint32_t a = m[0];
#pragma unroll
  for (int j = 1; j < V; ++j) a &= m[j];
  return a == 0xFFFFFFFFu ? 1u : 0u;
}

// carry lookahead over the warp: g = this lane's carry out, p = its limbs are all
// ones (g, p disjoint), cin0 = carry into lane 0.  Returns the carry INTO this lane;
// cout = carry out of lane 31.
__device__ __forceinline__ uint32_t lookahead(uint32_t g, uint32_t p, uint32_t cin0, uint32_t& cout) {
  const unsigned G = __ballot_sync(FULL, g), Pm = __ballot_sync(FULL, p);
  const uint64_t X = (uint64_t)(G | Pm), Y = G;
  const uint64_t S = X + Y + cin0;
  const unsigned C = (unsigned)(S ^ X ^ Y);
  cout = (unsigned)(S >> 32);
  return (C >> lane_id()) & 1u;
}

// m += c (c in {0,1}) inside the lane; the carry out is accounted for by the lookahead
template <int V>
__device__ __forceinline__ void add_bit(uint32_t (&m)[V], uint32_t c) {
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(c));
#pragma unroll
  for (int j = 1; j < V; ++j) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(m[j]));
}

// r = a + b + cin inside the lane; returns the carry out
template <int V>
__device__ __forceinline__ uint32_t add_chain(uint32_t (&r)[V], const uint32_t (&a)[V], const uint32_t (&b)[V],
                                              uint32_t cin) {
  uint32_t t, c;
  asm volatile("add.cc.u32 %0, %1, 0xFFFFFFFF;" : "=r"(t) : "r"(cin));  // CF = (cin != 0)
#pragma unroll
  for (int j = 0; j < V; ++j) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r[j]) : "r"(a[j]), "r"(b[j]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  (void)t;
  return c;
}

// add word w at global limb kq with full carry propagation over the warp; returns the
// carry out of the top limb
template <int V>
__device__ __forceinline__ uint32_t add_word_at(uint32_t (&m)[V], int kq, uint32_t w) {
  const int lane = lane_id(), owner = kq / V, jr = kq % V;
  uint32_t c = 0;
  if (lane == owner) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (j >= jr) {
        const uint64_t t = (uint64_t)m[j] + (j == jr ? w : 0u) + c;
        m[j] = (uint32_t)t;
        c = (uint32_t)(t >> 32);
      }
    }
  }
  uint32_t cout;
  const uint32_t cin = lookahead(c, lane > owner ? all_ones<V>(m) : 0u, 0u, cout);
  add_bit<V>(m, cin);
  return cout;
}

// ---- round to nearest even at p = 32 L - sh bits ----------------------------
// m: normalised mantissa (MSB of limb L-1 set), g: the guard limb below limb 0 and
// st: sticky (nonzero if anything below g) -- both warp-uniform.  mp_arith.cuh round_p.
template <int V>
__device__ __forceinline__ void round_w(uint32_t (&m)[V], uint32_t g, uint32_t st, int sh, int32_t& e) {
  const int lane = lane_id();
  uint32_t up, w;
  int kq;
  if (sh == 0) {
    const uint32_t rb = g >> 31;
    const uint32_t rest = (g << 1) | st;
    const uint32_t lsb = __shfl_sync(FULL, m[0], 0) & 1u;
    up = rb & ((rest != 0) | lsb);
    kq = 0;
    w = 1u;
  } else {
    const int rbpos = sh - 1, rl = rbpos >> 5, rbit = rbpos & 31;
    const int ql = sh >> 5, qb = sh & 31;
    uint32_t stk = 0, rbl = 0, lsbl = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int k = lane * V + j;
      uint32_t v = m[j];
      if (k < rl) {
        stk |= v;
        v = 0;
      } else if (k == rl) {
        rbl = (v >> rbit) & 1u;
        stk |= v & ((1u << rbit) - 1u);
        v &= (rbit == 31) ? 0u : ~((2u << rbit) - 1u);
      }
      if (k == ql) lsbl = (v >> qb) & 1u;
      m[j] = v;
    }
    const uint32_t sk = (__ballot_sync(FULL, stk != 0) != 0) | (g != 0) | (st != 0);
    const uint32_t rb = __ballot_sync(FULL, rbl) != 0;
    const uint32_t lsb = __ballot_sync(FULL, lsbl) != 0;
    up = rb & (sk | lsb);
    kq = ql;
    w = 1u << qb;
  }
  if (up) {
    if (add_word_at<V>(m, kq, w)) {  // carry out of the top: mantissa 1000...0
#pragma unroll
      for (int j = 0; j < V; ++j) m[j] = 0;
      if (lane == 31) m[V - 1] = 0x80000000u;
      e += 1;
    }
  }
}

template <int V>
__device__ __forceinline__ void zero_w(W<V>& z, uint32_t s = 0) {
#pragma unroll
  for (int j = 0; j < V; ++j) z.m[j] = 0;
  z.e = EXP_ZERO;
  z.s = s;
}

// ---- record I/O: lane l reads / writes limbs [l V, l V + V) of the record ------
template <int V>
__device__ __forceinline__ void load_w(const uint32_t* __restrict__ r, W<V>& x) {
  constexpr int L = 32 * V;
  const int lane = lane_id();
#pragma unroll
  for (int j = 0; j < V; ++j) x.m[j] = r[lane * V + j];
  x.e = (int32_t)r[L];
  x.s = r[L + 1];
}
template <int V>
__device__ __forceinline__ void store_w(uint32_t* __restrict__ r, const W<V>& x) {
  constexpr int L = 32 * V, S = rec_stride(L);
  const int lane = lane_id();
#pragma unroll
  for (int j = 0; j < V; ++j) r[lane * V + j] = x.m[j];
  if (lane < S - L) r[L + lane] = lane == 0 ? (uint32_t)x.e : (lane == 1 ? x.s : 0u);
}

// ---- alignment shifts of a window [g | m] (g: guard limb, meaningful in lane 0) ----
// right by r bits, 0 < r < 32; bits shifted out of g go to st0 (lane 0)
template <int V>
__device__ __forceinline__ void shr_bits(uint32_t (&m)[V], uint32_t& g, uint32_t& st0, int r) {
  uint32_t nxt = __shfl_down_sync(FULL, m[0], 1);
  if (lane_id() == 31) nxt = 0;
  st0 |= g & ((1u << r) - 1u);
  g = __funnelshift_r(g, m[0], r);
#pragma unroll
  for (int j = 0; j < V - 1; ++j) m[j] = __funnelshift_r(m[j], m[j + 1], r);
  m[V - 1] = __funnelshift_r(m[V - 1], nxt, r);
}

// right by q whole limbs (1 <= q <= L): new window limb t = old window limb t + q; the
// dropped limbs (old g and limbs 0 .. q-2) are OR-ed into the returned uniform sticky
template <int V>
__device__ __forceinline__ uint32_t shr_limbs(uint32_t (&m)[V], uint32_t& g, int q) {
  constexpr int L = 32 * V;
  const int lane = lane_id();
  uint32_t loc = lane == 0 ? g : 0u;
#pragma unroll
  for (int j = 0; j < V; ++j)
    if (lane * V + j <= q - 2) loc |= m[j];
  const uint32_t st = __ballot_sync(FULL, loc != 0) != 0;
  const uint32_t ng = (q - 1 < L) ? get_limb<V>(m, q - 1) : 0u;
  const int qa = q / V, qb = q % V;
  uint32_t t[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {  // t[j] = m[(j + qb) % V]
    uint32_t v = 0;
#pragma unroll
    for (int r = 0; r < V; ++r)
      if (r == (j + qb) % V) v = m[r];
    t[j] = v;
  }
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int src = lane + qa + ((j + qb) >= V ? 1 : 0);
    const uint32_t v = __shfl_sync(FULL, t[j], src & 31);
    m[j] = src < 32 ? v : 0u;
  }
  g = ng;
  return st;
}

// left by one whole limb of the window [g | m]: the guard (lane 0) enters limb 0
template <int V>
__device__ __forceinline__ void shl1_limb(uint32_t (&m)[V], uint32_t& g) {
  uint32_t prv = __shfl_up_sync(FULL, m[V - 1], 1);
  if (lane_id() == 0) prv = g;
#pragma unroll
  for (int j = V - 1; j > 0; --j) m[j] = m[j - 1];
  m[0] = prv;
  g = 0;
}

// ---------------------------------------------------------------------------
// z = RN_p(x + (-1)^negy y)  (mpfr_add / mpfr_sub; mp_arith.cuh mp_add)
// (L+1)-limb window [guard | limbs]: the guard lives in lane 0.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ void add_w(const W<V>& x, const W<V>& y, uint32_t negy, int sh, W<V>& z) {
  constexpr int L = 32 * V;
  const int lane = lane_id();
  const uint32_t ys = y.s ^ negy;
  if (x.e == EXP_ZERO || y.e == EXP_ZERO) {
    if (x.e == EXP_ZERO && y.e == EXP_ZERO) {
      const uint32_t zs = x.s & ys;
      zero_w<V>(z, zs);
    } else if (x.e == EXP_ZERO) {
#pragma unroll
      for (int j = 0; j < V; ++j) z.m[j] = y.m[j];
      z.e = y.e;
      z.s = ys;
    } else {
      z = x;
    }
    return;
  }
  const bool swp = y.e > x.e;
  uint32_t A[V], B[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    A[j] = swp ? y.m[j] : x.m[j];
    B[j] = swp ? x.m[j] : y.m[j];
  }
  const int32_t ebig = swp ? y.e : x.e;
  const uint32_t d = (uint32_t)(swp ? y.e - x.e : x.e - y.e);
  const uint32_t sbig = swp ? ys : x.s;
  const uint32_t ssmall = swp ? x.s : ys;
  const uint32_t sub = sbig ^ ssmall;

  // ---- align B right by d bits (guard gb in lane 0; st0 lane-0 sticky, stu uniform)
  uint32_t gb = 0, st0 = 0, stu = 0;
  if (d >= 32u * (L + 1)) {
#pragma unroll
    for (int j = 0; j < V; ++j) B[j] = 0;
    stu = 1;
  } else {
    const int q = (int)(d >> 5), r = (int)(d & 31u);
    if (q) stu = shr_limbs<V>(B, gb, q);
    if (r) shr_bits<V>(B, gb, st0, r);
  }
  const uint32_t st = (__shfl_sync(FULL, st0, 0) != 0) | stu;

  // ---- R = A + B (add) or A + ~B + (1 - st) (sub): lane 0 starts with the guard limb
  const uint32_t mask = 0u - sub;
  const uint32_t cin = sub & (st ^ 1u);
  uint32_t rg = 0, c0 = 0;
  if (lane == 0) {
    const uint64_t t = (uint64_t)(gb ^ mask) + cin;  // A's guard is 0
    rg = (uint32_t)t;
    c0 = (uint32_t)(t >> 32);
  }
  uint32_t Bm[V], R[V];
#pragma unroll
  for (int j = 0; j < V; ++j) Bm[j] = B[j] ^ mask;
  const uint32_t gl = add_chain<V>(R, A, Bm, c0);
  uint32_t cout;
  const uint32_t ci = lookahead(gl, lane > 0 ? all_ones<V>(R) : 0u, 0u, cout);
  add_bit<V>(R, ci);

  int32_t e = ebig;
  uint32_t s = sbig;
  uint32_t top = __shfl_sync(FULL, R[V - 1], 31);
  if (sub & ((cout ^ 1u) | (top == 0))) {  // rare: |small| > |big| (d == 0) or deep cancellation
    if (!cout) {  // R = -R over the window (two's complement)
      uint32_t c = 0;
      if (lane == 0) {
        const uint64_t t = (uint64_t)(~rg) + 1u;
        rg = (uint32_t)t;
        c = (uint32_t)(t >> 32);
      }
      uint32_t N[V], Z[V];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        N[j] = ~R[j];
        Z[j] = 0;
      }
      const uint32_t g2 = add_chain<V>(R, N, Z, c);
      uint32_t co2;
      const uint32_t c2 = lookahead(g2, lane > 0 ? all_ones<V>(R) : 0u, 0u, co2);
      add_bit<V>(R, c2);
      s = ssmall;
    }
    uint32_t any = lane == 0 ? rg : 0u;
#pragma unroll
    for (int j = 0; j < V; ++j) any |= R[j];
    if (__ballot_sync(FULL, any != 0) == 0) {  // exact cancellation: +0 under RNDN
      zero_w<V>(z, 0);
      return;
    }
    top = __shfl_sync(FULL, R[V - 1], 31);
    while (top == 0) {
      shl1_limb<V>(R, rg);
      e -= 32;
      top = __shfl_sync(FULL, R[V - 1], 31);
    }
  }
  // ---- normalise: add overflow shifts right by one, cancellation left by lz
  const uint32_t c1 = cout & (sub ^ 1u);
  if (c1) {
    uint32_t nxt = __shfl_down_sync(FULL, R[0], 1);
    if (lane == 31) nxt = 1u;
    if (lane == 0) {
      st0 = rg & 1u;
      rg = __funnelshift_r(rg, R[0], 1);
    }
#pragma unroll
    for (int j = 0; j < V - 1; ++j) R[j] = __funnelshift_r(R[j], R[j + 1], 1);
    R[V - 1] = __funnelshift_r(R[V - 1], nxt, 1);
    e += 1;
  } else {
    st0 = 0;
    const int lz = __clz(top);
    if (lz) {
      uint32_t prv = __shfl_up_sync(FULL, R[V - 1], 1);
      if (lane == 0) prv = rg;
#pragma unroll
      for (int j = V - 1; j > 0; --j) R[j] = __funnelshift_l(R[j - 1], R[j], lz);
      R[0] = __funnelshift_l(prv, R[0], lz);
      rg <<= lz;
      e -= lz;
    }
  }
  const uint32_t g = __shfl_sync(FULL, rg, 0);
  const uint32_t stf = st | (__shfl_sync(FULL, st0, 0) != 0);
  round_w<V>(R, g, stf, sh, e);
#pragma unroll
  for (int j = 0; j < V; ++j) z.m[j] = R[j];
  z.e = e;
  z.s = s;
}

// ---------------------------------------------------------------------------
// Limb product of x and y, column-wise over the warp.  FULL: all 2L columns, exact.
// SHORT: only the columns t >= L-2 (i + j >= L-2 -- the truncated product of
// mp_arith.cuh mul_high_g, (L^2 + 3L - 2)/2 limb products); the omitted part is below
// L-1 units of limb L-1.  Lane l accumulates the columns t = c0 + l + 32 j in three
// words each (strided: every lane gets a balanced share of the triangular column
// lengths), the column sums go through shared memory to a blocked layout where carries
// are resolved inside the lane and across lanes (shuffle + lookahead).
// FULL:  P[q] = product limb 2 V l + q (q < 2V).
// SHORT: P[q] = product limb L + V l + q (q < V); g1 / g0 = limbs L-1 / L-2 (uniform).
// ---------------------------------------------------------------------------
template <int V, bool SHORT>
__device__ __forceinline__ void product_w(const W<V>& x, const W<V>& y, const Scratch<V>& sc,
                                          uint32_t (&P)[2 * V], uint32_t& g1, uint32_t& g0) {
  constexpr int L = 32 * V;
  constexpr int C0 = SHORT ? L - 2 : 0;      // first column computed
  constexpr int NB = SHORT ? V + 1 : 2 * V;  // blocks of 32 columns
  const int lane = lane_id();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < V; ++j) {
    sc.a[4 + lane * V + j] = x.m[j];
    sc.b[40 + lane * V + j] = y.m[j];
  }
  if (lane < 4) {
    sc.a[lane] = 0;
    sc.a[4 + L + lane] = 0;
  }
  for (int t = lane; t < 40; t += 32) {
    sc.b[t] = 0;
    sc.b[40 + L + t] = 0;
  }
  __syncwarp();
  constexpr int NC = 32 * NB;  // columns stored (relative to C0)
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int c = C0 + 32 * j;  // this block's first column
    const int ilo = c - (L - 1) > 0 ? c - (L - 1) : 0;
    const int ihi = c + 31 < L - 1 ? c + 31 : L - 1;
    const int t = c + lane;
    // four independent three-word accumulators (one per term of a group of four):
    // the carry chains of consecutive terms do not serialise
    uint32_t acc[4][3];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = acc[u][2] = 0;
#pragma unroll 2
    for (int i = ilo & ~3; i <= ihi; i += 4) {
      const uint4 a4 = *reinterpret_cast<const uint4*>(sc.a + 4 + i);
      const uint32_t av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t bv = sc.b[40 + t - i - u];
#if MPG_WMUL_FUSED
        // product + 64-bit accumulate + carry-out in one IMAD.WIDE.U32 (ptxas fuses the
        // mad.lo.cc / madc.hi.cc pair), then the third word: 2 instructions per limb product
        asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                     : "+r"(acc[u][0]), "+r"(acc[u][1]), "+r"(acc[u][2])
                     : "r"(av[u]), "r"(bv));
#else
        const uint64_t pr = (uint64_t)av[u] * bv;
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[u][0]) : "r"((uint32_t)pr));
        asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[u][1]) : "r"((uint32_t)(pr >> 32)));
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(acc[u][2]));
#endif
      }
    }
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[0][0]) : "r"(acc[u][0]));
      asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[0][1]) : "r"(acc[u][1]));
      asm volatile("addc.u32 %0, %0, %1;" : "+r"(acc[0][2]) : "r"(acc[u][2]));
    }
    sc.col[lane + 32 * j] = acc[0][0];
    sc.col[NC + lane + 32 * j] = acc[0][1];
    sc.col[2 * NC + lane + 32 * j] = acc[0][2];
  }
  __syncwarp();
  constexpr int NQ = SHORT ? V : 2 * V;  // limbs resolved per lane
  const int base = SHORT ? 2 + V * lane : 2 * V * lane;
  uint32_t k0 = 0, k1 = 0;
  auto step = [&](int t) -> uint32_t {
    const uint32_t c0 = sc.col[t], c1 = sc.col[NC + t], c2 = sc.col[2 * NC + t];
    uint32_t s0, s1, s2;
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(s0) : "r"(c0), "r"(k0));
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(s1) : "r"(c1), "r"(k1));
    asm volatile("addc.u32 %0, %1, 0;" : "=r"(s2) : "r"(c2));
    k0 = s1;
    k1 = s2;
    return s0;
  };
  uint32_t lg0 = 0, lg1 = 0;
  if (SHORT && lane == 0) {  // the two guard columns L-2, L-1 first
    lg0 = step(0);
    lg1 = step(1);
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) P[q] = step(base + q);
  // add the previous lane's carry (two words) at this lane's first limb, then 1-bit carries
  uint32_t p0 = __shfl_up_sync(FULL, k0, 1), p1 = __shfl_up_sync(FULL, k1, 1);
  if (lane == 0) p0 = p1 = 0;
  uint32_t g;
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(P[0]) : "r"(p0));
  asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(P[1]) : "r"(p1));
#pragma unroll
  for (int q = 2; q < NQ; ++q) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(P[q]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(g));
  uint32_t pr = 1u;
#pragma unroll
  for (int q = 0; q < NQ; ++q) pr &= (P[q] == 0xFFFFFFFFu) ? 1u : 0u;
  uint32_t cout;
  const uint32_t ci = lookahead(g, lane > 0 ? pr : 0u, 0u, cout);
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(P[0]) : "r"(ci));
#pragma unroll
  for (int q = 1; q < NQ; ++q) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(P[q]));
  g1 = __shfl_sync(FULL, lg1, 0);
  g0 = __shfl_sync(FULL, lg0, 0);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// z = RN_p(x * y)  (mpfr_mul; mp_arith.cuh mp_mul).  The short product decides the
// rounding unless the true guard limb may lie near a rounding boundary (mpfr_mul's
// mulhigh strategy, as mp_mul_g); otherwise the exact full product is formed.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ void mul_w(const W<V>& x, const W<V>& y, int sh, const Scratch<V>& sc, W<V>& z) {
  constexpr int L = 32 * V;
  const int lane = lane_id();
  const uint32_t zs = x.s ^ y.s;
  z.s = zs;
  if (x.e == EXP_ZERO || y.e == EXP_ZERO) {
    zero_w<V>(z, zs);
    return;
  }
  uint32_t P[2 * V], g1, g0;
  {
    product_w<V, true>(x, y, sc, P, g1, g0);
    const uint32_t top = __shfl_sync(FULL, P[V - 1], 31);
    const uint32_t t1 = (top >> 31) ^ 1u;
    const uint32_t gt = __funnelshift_l(g0, g1, t1);
    // the true guard limb lies in [gt, gt + 2L)
    const bool down = gt < 0x80000000u - 2u * L;
    const bool up = gt > 0x80000000u && gt < 0xFFFFFFFFu - 2u * L;
    const bool ok = sh == 0 ? (down | up) : (gt != 0 && gt < 0xFFFFFFFFu - 2u * L);
    if (ok) {
      uint32_t prv = __shfl_up_sync(FULL, P[V - 1], 1);
      if (lane == 0) prv = g1;
#pragma unroll
      for (int j = V - 1; j > 0; --j) z.m[j] = __funnelshift_l(P[j - 1], P[j], t1);
      z.m[0] = __funnelshift_l(prv, P[0], t1);
      int32_t e = x.e + y.e - (int32_t)t1;
      // sh == 0: the guard decides; sh > 0: the round bit is inside the mantissa and
      // everything below it is nonzero (gt != 0)
      round_w<V>(z.m, sh == 0 ? gt : 1u, sh == 0 ? 0u : 1u, sh, e);
      z.e = e;
      return;
    }
  }
  product_w<V, false>(x, y, sc, P, g1, g0);
  // mantissa = product limbs [L, 2L) (lane l's limbs L + V l + j live in lane 16 + l/2)
  const int hl = 16 + (lane >> 1);
  const bool odd = lane & 1;
  const uint32_t top = __shfl_sync(FULL, P[2 * V - 1], 31);
  const uint32_t t1 = (top >> 31) ^ 1u;
  uint32_t M[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const uint32_t v0 = __shfl_sync(FULL, P[j], hl), v1 = __shfl_sync(FULL, P[V + j], hl);
    M[j] = odd ? v1 : v0;
  }
  // the limb below this lane's first mantissa limb
  const uint32_t x0 = __shfl_sync(FULL, P[2 * V - 1], hl - 1), x1 = __shfl_sync(FULL, P[V - 1], hl);
  const uint32_t below = odd ? x1 : x0;
  const uint32_t Gh = __shfl_sync(FULL, P[2 * V - 1], 15), Gl = __shfl_sync(FULL, P[2 * V - 2], 15);
  // sticky: limbs 0 .. L-3 (lanes 0..14, lane 15 without its top two limbs)
  uint32_t loc = 0;
#pragma unroll
  for (int q = 0; q < 2 * V; ++q)
    if (lane < 15 || (lane == 15 && q < 2 * V - 2)) loc |= P[q];
  uint32_t st = __ballot_sync(FULL, loc != 0) != 0;
#pragma unroll
  for (int j = V - 1; j > 0; --j) z.m[j] = __funnelshift_l(M[j - 1], M[j], t1);
  z.m[0] = __funnelshift_l(below, M[0], t1);
  const uint32_t g = __funnelshift_l(Gl, Gh, t1);
  st |= (Gl << t1) != 0;
  int32_t e = x.e + y.e - (int32_t)t1;
  round_w<V>(z.m, g, st, sh, e);
  z.e = e;
}

// ---------------------------------------------------------------------------
// z = RN_p(x / y)  (mpfr_div; mp_arith.cuh mp_div): radix-2^32 digit recurrence, the
// remainder distributed over the warp (top limb RL warp-uniform), digit estimates from
// the top three limbs with directed-rounding FP64 (never an overestimate) and add-back
// corrections; quotient digits collected in shared memory (sc.col).  y != 0.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ void div_w(const W<V>& x, const W<V>& y, int sh, const Scratch<V>& sc, W<V>& z) {
  constexpr int L = 32 * V, WL = L + 1;
  const int lane = lane_id();
  const uint32_t zs = x.s ^ y.s;
  if (x.e == EXP_ZERO || y.e == EXP_ZERO) {
    zero_w<V>(z, zs);
    return;
  }
  uint32_t R[V];
#pragma unroll
  for (int j = 0; j < V; ++j) R[j] = x.m[j];
  uint32_t RL = 0;  // limb L of the remainder (uniform)
  // R -= Y if R >= Y; returns 1 if subtracted
  auto try_sub = [&]() -> uint32_t {
    uint32_t T[V], NY[V];
#pragma unroll
    for (int j = 0; j < V; ++j) NY[j] = ~y.m[j];
    const uint32_t gl = add_chain<V>(T, R, NY, lane == 0 ? 1u : 0u);
    uint32_t cout;
    const uint32_t ci = lookahead(gl, lane > 0 ? all_ones<V>(T) : 0u, 0u, cout);
    add_bit<V>(T, ci);
    // top limb: RL + ~0 + cout; no borrow overall iff RL != 0 or cout
    const uint32_t ok = (RL != 0 || cout) ? 1u : 0u;
    if (ok) {
#pragma unroll
      for (int j = 0; j < V; ++j) R[j] = T[j];
      RL = RL - 1u + cout;
    }
    return ok;
  };
  uint32_t* Q = sc.col;  // WL + 1 digits
  const uint32_t q0 = try_sub();
  const uint32_t y1 = __shfl_sync(FULL, y.m[V - 1], 31), y2 = __shfl_sync(FULL, y.m[V - 2], 31);
  const uint64_t ytop = ((uint64_t)y1 << 32) | y2;
  const double yd = __dadd_ru(__ull2double_ru(ytop), 1.0);
  const double inv = __drcp_rd(yd);
#pragma unroll 1
  for (int t = WL - 1; t >= 0; --t) {
    // R <<= 32 (R < Y: the top limb is free); the new top three limbs come from lane 31's
    // (and for V = 2 lane 30's) registers before the shift -- one round of shuffles
    const uint32_t t0 = __shfl_sync(FULL, R[V - 1], 31), t1 = __shfl_sync(FULL, R[V - 2], 31);
    const uint32_t t2 = V >= 3 ? __shfl_sync(FULL, R[V >= 3 ? V - 3 : 0], 31) : __shfl_sync(FULL, R[V - 1], 30);
    uint32_t prv = __shfl_up_sync(FULL, R[V - 1], 1);
    if (lane == 0) prv = 0;
#pragma unroll
    for (int j = V - 1; j > 0; --j) R[j] = R[j - 1];
    R[0] = prv;
    RL = t0;
    const uint64_t rtop = ((uint64_t)RL << 32) | t1;
    double rd = __dmul_rd(__ull2double_rd(rtop), 4294967296.0);
    rd = __dadd_rd(rd, (double)t2);
    const double qd = floor(__dmul_rd(rd, inv));
    uint32_t qh = qd >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)qd;
    // R -= qh * Y in one pass: each lane subtracts its V-limb product segment, passes its
    // product top limb plus its borrow (< 2^32) to the next lane, which subtracts it at its
    // first limb; the remaining 1-bit borrows resolve by lookahead (propagate = all zero)
    uint32_t E[V], cl = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const uint64_t pr = (uint64_t)qh * y.m[j] + cl;
      E[j] = (uint32_t)pr;
      cl = (uint32_t)(pr >> 32);
    }
    uint32_t NE[V];
#pragma unroll
    for (int j = 0; j < V; ++j) NE[j] = ~E[j];
    const uint32_t c1 = add_chain<V>(R, R, NE, 1u);  // R - E, carry 1 = no borrow
    const uint32_t h = cl + (c1 ^ 1u);                // subtract from the next lane's limb 0
    uint32_t hp = __shfl_up_sync(FULL, h, 1);
    if (lane == 0) hp = 0;
    uint32_t b2;
    asm volatile("sub.cc.u32 %0, %0, %1;" : "+r"(R[0]) : "r"(hp));
#pragma unroll
    for (int j = 1; j < V; ++j) asm volatile("subc.cc.u32 %0, %0, 0;" : "+r"(R[j]));
    asm volatile("subc.u32 %0, 0, 0;" : "=r"(b2));  // 0xFFFFFFFF on borrow
    uint32_t zl = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) zl |= R[j];
    uint32_t bout;
    const uint32_t bin = lookahead(b2 & 1u, lane > 0 && zl == 0 ? 1u : 0u, 0u, bout);
    asm volatile("sub.cc.u32 %0, %0, %1;" : "+r"(R[0]) : "r"(bin));
#pragma unroll
    for (int j = 1; j < V; ++j) asm volatile("subc.cc.u32 %0, %0, 0;" : "+r"(R[j]));
    RL = RL - __shfl_sync(FULL, h, 31) - bout;
    // the estimate is never high and short by at most a little; R >= Y needs RL > 0 or
    // a top limb >= Y's, so the full comparison runs only then
    if (RL != 0 || __shfl_sync(FULL, R[V - 1], 31) >= y1)
      while (try_sub()) ++qh;
    if (lane == 0) Q[t] = qh;
  }
  uint32_t rloc = 0;
#pragma unroll
  for (int j = 0; j < V; ++j) rloc |= R[j];
  uint32_t rem = (__ballot_sync(FULL, rloc != 0) != 0) | (RL != 0);
  if (lane == 0) Q[WL] = q0;
  __syncwarp();
  // value = Q[WL] . Q[WL-1] ... Q[0]; mantissa limbs M[k + 1], guard M[0]
  int32_t e = x.e - y.e;
  const uint32_t sh1 = q0;  // quotient in [1, 2): shift the digit string right by one
  uint32_t g;
  {
    const uint32_t d0 = Q[0], d1 = Q[1];
    g = sh1 ? __funnelshift_r(d0, d1, 1) : d0;
    if (sh1) rem |= d0 & 1u;
  }
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int k = lane * V + j + 1;
    const uint32_t lo = Q[k], hi = Q[k + 1];
    z.m[j] = sh1 ? __funnelshift_r(lo, hi, 1) : lo;
  }
  __syncwarp();
  e += (int32_t)sh1;
  round_w<V>(z.m, g, rem, sh, e);
  z.e = e;
  z.s = zs;
}

// |x| vs |y|: -1, 0, 1 (warp-uniform)
template <int V>
__device__ __forceinline__ int cmpabs_w(const W<V>& x, const W<V>& y) {
  const bool xz = x.e == EXP_ZERO, yz = y.e == EXP_ZERO;
  if (xz || yz) return xz ? (yz ? 0 : -1) : 1;
  if (x.e != y.e) return x.e > y.e ? 1 : -1;
  int c = 0;
#pragma unroll
  for (int j = V - 1; j >= 0; --j)
    if (c == 0 && x.m[j] != y.m[j]) c = x.m[j] > y.m[j] ? 1 : -1;
  const unsigned ne = __ballot_sync(FULL, c != 0);
  if (!ne) return 0;
  return __shfl_sync(FULL, c, 31 - __clz(ne));
}

}  // namespace wmp
}  // namespace mpg
