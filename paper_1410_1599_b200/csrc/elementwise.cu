// elementwise.cu -- HBM-bound MP kernels: layout conversion, add/sub, and the
// fused Strassen / Winograd level transforms (K2 mp_preadd, K3 mp_postadd).
//
// Pre-add (fastmm.hpp:104-115 pad + quadrants, :134-150 Strassen sums,
// :173-180 Winograd S1..S8): one thread per (parent node, quadrant element),
// reads the four quadrant records (virtual zero padding for odd dimensions --
// pad_operand, fastmm.hpp:91-97, fills +0), forms the sums with the reference's
// operand order and writes the seven child operands.  Post-add (fastmm.hpp:152-161
// Strassen, :190-198 Winograd, :221-227 strip): one thread per (parent, element)
// reads the seven child products and writes the four C quadrants, dropping padded
// rows/columns.  Every sum is the same correctly rounded MP add as the reference's
// addsub (matrix.hpp:121-134), so fusing them is bit-exact.
#include <cuda_runtime.h>

#include "kernels.h"
#include "mp_arith.cuh"
#if MPG_WIDE
#include "wkern.cuh"
#endif

#ifndef MPG_ADDS_HOIST
#define MPG_ADDS_HOIST 1  // pre/post-additions: operands loaded up front for L <= 8
#endif

namespace mpg {

// resident CTAs per SM asked of the compiler (register cap) for the fused level transforms.
// Measured (profiles/r02_ab_ew.jsonl, n = 1024 Winograd): at 512 bits 2 CTAs instead of 1 take the
// pre-additions 1.35 -> 1.20 ms and the post-additions 0.68 -> 0.50 ms; at 256 bits 3 or 4 CTAs
// (80 / 64 registers, spilling) lose 7 %, at 1024 bits 2 CTAs lose 7 % (pre) / 32 % (post)
#ifndef MPG_PRE_MINB_8
#define MPG_PRE_MINB_8 2
#endif
#ifndef MPG_POST_MINB_8
#define MPG_POST_MINB_8 2
#endif
#ifndef MPG_PRE_MINB_16
#define MPG_PRE_MINB_16 2
#endif
#ifndef MPG_POST_MINB_16
#define MPG_POST_MINB_16 2
#endif
#ifndef MPG_PRE_MINB_32
#define MPG_PRE_MINB_32 1
#endif
#ifndef MPG_POST_MINB_32
#define MPG_POST_MINB_32 1
#endif
#ifndef MPG_ADD2_STAGE
#define MPG_ADD2_STAGE 1  // fused pre-additions: results stored through a per-warp staging row (whole sectors)
#endif
#ifndef MPG_POST2_MINB
#define MPG_POST2_MINB 1  // resident CTAs asked for the fused post-additions; measured: 5 / 6 CTAs (102 / 85 registers, spilling) 0.25 -> 0.32 / 0.35 ms at cfg2
#endif
#ifndef MPG_ADD2_PT
#define MPG_ADD2_PT 32  // positions per CTA of the fused two-level transforms (4 PT threads)
#endif
constexpr int pre_minb(int L) { return L <= 8 ? MPG_PRE_MINB_8 : L <= 16 ? MPG_PRE_MINB_16 : L <= 32 ? MPG_PRE_MINB_32 : 1; }
constexpr int post_minb(int L) { return L <= 8 ? MPG_POST_MINB_8 : L <= 16 ? MPG_POST_MINB_16 : L <= 32 ? MPG_POST_MINB_32 : 1; }
namespace {
constexpr int NT = 256;
inline int grid_for(int64_t n) {
  int64_t b = (n + NT - 1) / NT;
  return (int)(b < 148 * 64 ? (b < 1 ? 1 : b) : 148 * 64);
}
}  // namespace

template <int L>
__global__ void soa2rec_kernel(const uint32_t* __restrict__ limbs, const int32_t* __restrict__ exp,
                               const uint8_t* __restrict__ sign, int64_t N, int64_t ps,
                               uint32_t* __restrict__ rec) {
  constexpr int S = rec_stride(L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    MP<L> x;
#pragma unroll
    for (int k = 0; k < L; ++k) x.m[k] = limbs[k * ps + e];
    x.e = exp[e];
    x.s = sign[e];
    store_rec<L>(rec + e * S, x);
  }
}

// SoA planes of a dense rows x cols block -> records of a strided matrix (leading
// dimension ldr): one quadrant of the pipelined host GEMM's operands
template <int L>
__global__ void soa2rec2d_kernel(const uint32_t* __restrict__ limbs, const int32_t* __restrict__ exp,
                                 const uint8_t* __restrict__ sign, int64_t rows, int64_t cols, int64_t ps,
                                 uint32_t* __restrict__ rec, int64_t ldr) {
  constexpr int S = rec_stride(L);
  const int64_t N = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    MP<L> x;
#pragma unroll
    for (int k = 0; k < L; ++k) x.m[k] = limbs[k * ps + e];
    x.e = exp[e];
    x.s = sign[e];
    store_rec<L>(rec + (r * ldr + c) * S, x);
  }
}

template <int L>
__global__ void rec2soa_kernel(const uint32_t* __restrict__ rec, int64_t N, uint32_t* __restrict__ limbs,
                               int32_t* __restrict__ exp, uint8_t* __restrict__ sign, int64_t ps) {
  constexpr int S = rec_stride(L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    MP<L> x;
    load_rec<L>(rec + e * S, x);
#pragma unroll
    for (int k = 0; k < L; ++k) limbs[k * ps + e] = x.m[k];
    exp[e] = x.e;
    sign[e] = (uint8_t)x.s;
  }
}

template <int L>
__global__ void addsub_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                              uint32_t* __restrict__ C, int64_t N, uint32_t neg, int sh,
                              uint32_t* err) {
  constexpr int S = rec_stride(L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    MP<L> a, b, c;
    load_rec<L>(A + e * S, a);
    load_rec<L>(B + e * S, b);
    mp_add<L>(a, b, neg, sh, c);
    if (exp_out_of_range(c.e)) atomicOr(err, ERR_EXP_RANGE);
    store_rec<L>(C + e * S, c);
  }
}

template <int L>
__global__ void vec_op_kernel(int op, const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                              uint32_t* __restrict__ C, int64_t N, int sh, uint32_t* err) {
  constexpr int S = rec_stride(L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    MP<L> a, b, c;
    load_rec<L>(A + e * S, a);
    load_rec<L>(B + e * S, b);
    if (op == 0)
      mp_add<L>(a, b, 0u, sh, c);
    else if (op == 1)
      mp_add<L>(a, b, 1u, sh, c);
    else if (op == 2)
      mp_mul<L>(a, b, sh, c);
    else {
      if (b.e == EXP_ZERO) {
        atomicOr(err, ERR_DIV_ZERO);
        mp_zero(c);
      } else {
        mp_div<L>(a, b, sh, c);
      }
    }
    if (exp_out_of_range(c.e)) atomicOr(err, ERR_EXP_RANGE);
    store_rec<L>(C + e * S, c);
  }
}

// read parent element (r, c) of a rows x cols dense record matrix, +0 outside
template <int L>
__device__ __forceinline__ void load_padded(const uint32_t* P, int rows, int cols, int r, int c, MP<L>& x) {
  if (r < rows && c < cols)
    load_rec<L>(P + ((int64_t)r * cols + c) * rec_stride(L), x);
  else
    mp_zero(x, 0);
}

// The level transform of one quadrant element: ld(q, x) reads quadrant q (0: 11, 1: 12, 2: 21,
// 3: 22) of the virtually zero-padded parent, put(child, x) writes child operand `child`.
// Each sum is formed from operands (re)loaded right before it and stored right
// after it, so at most two MP values plus the adder's window are live -- the
// 1024-bit instantiation stays in registers.
template <int L, class LD, class PUT>
__device__ __forceinline__ void preadd_body(int algo, int side, int sh, LD ld, PUT put) {
  auto sum = [&](int qa, int qb, uint32_t neg, int child) {
    MP<L> x, y;
    ld(qa, x);
    ld(qb, y);
    mp_add<L>(x, y, neg, sh, x);
    put(child, x);
  };
  auto copy = [&](int q, int child) {
    MP<L> x;
    ld(q, x);
    put(child, x);
  };
  if (algo == 3) {
    if (side == 0) {
      // S1 = a21+a22 (M5), S2 = S1-a11 (M1), S3 = a11-a21 (M4), S4 = a12-S2 (M6)
      MP<L> s1, s2, x;
      ld(2, s1);
      ld(3, x);
      mp_add<L>(s1, x, 0u, sh, s1);
      put(4, s1);
      ld(0, x);
      mp_add<L>(s1, x, 1u, sh, s2);
      put(0, s2);
      ld(1, x);
      mp_add<L>(x, s2, 1u, sh, x);
      put(5, x);
      sum(0, 2, 1u, 3);
      copy(0, 1);  // M2 = a11*b11
      copy(1, 2);  // M3 = a12*b21
      copy(3, 6);  // M7 = a22*S8
    } else {
      // S5 = b12-b11 (M5), S6 = b22-S5 (M1), S7 = b22-b12 (M4), S8 = S6-b21 (M7)
      MP<L> s5, s6, x;
      ld(1, s5);
      ld(0, x);
      mp_add<L>(s5, x, 1u, sh, s5);
      put(4, s5);
      ld(3, x);
      mp_add<L>(x, s5, 1u, sh, s6);
      put(0, s6);
      ld(2, x);
      mp_add<L>(s6, x, 1u, sh, x);
      put(6, x);
      sum(3, 1, 1u, 3);
      copy(0, 1);  // b11
      copy(2, 2);  // b21
      copy(3, 5);  // b22
    }
  } else {
    if (side == 0) {  // a11+a22, a21+a22, a11, a22, a11+a12, a21-a11, a12-a22
      sum(0, 3, 0u, 0);
      sum(2, 3, 0u, 1);
      copy(0, 2);
      copy(3, 3);
      sum(0, 1, 0u, 4);
      sum(2, 0, 1u, 5);
      sum(1, 3, 1u, 6);
    } else {  // b11+b22, b11, b12-b22, b21-b11, b22, b11+b12, b21+b22
      sum(0, 3, 0u, 0);
      copy(0, 1);
      sum(1, 3, 1u, 2);
      sum(2, 0, 1u, 3);
      copy(3, 4);
      sum(0, 1, 0u, 5);
      sum(2, 3, 0u, 6);
    }
  }
}

template <int L>
__global__ void __launch_bounds__(256, pre_minb(L)) preadd_kernel(int algo, int side, const uint32_t* __restrict__ parent, int64_t nodes,
                              int rows, int cols, uint32_t* __restrict__ children, int sh, ChildSlots slots) {
  constexpr int S = rec_stride(L);
  extern __shared__ __align__(16) uint32_t s_stage[];  // one staging row of 32 records per warp
  const int hr = (rows + rows % 2) / 2, hc = (cols + cols % 2) / 2;
  const int64_t per = (int64_t)hr * hc;
  const int64_t total = per * nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = t / per;
    const int64_t e = t - node * per;
    const int r = (int)(e / hc), c = (int)(e - (int64_t)r * hc);
    const uint32_t* P = parent + node * (int64_t)rows * cols * S;
    uint32_t* out = children + (node * 7 * per + e) * S;
    const int64_t cs = per * S;  // stride between sibling children
    // quadrant q (0: 11, 1: 12, 2: 21, 3: 22) of the virtually zero-padded parent; for small
    // records all four are loaded up front (four independent loads in flight per thread)
    constexpr bool HOIST = MPG_ADDS_HOIST && L <= 8;
    MP<L> Q[HOIST ? 4 : 1];
    if constexpr (HOIST) {
#pragma unroll
      for (int q = 0; q < 4; ++q) load_padded<L>(P, rows, cols, r + (q >> 1) * hr, c + (q & 1) * hc, Q[q]);
    }
    auto ld = [&](int q, MP<L>& x) {
      if constexpr (HOIST)
        x = Q[q];
      else
        load_padded<L>(P, rows, cols, r + (q >> 1) * hr, c + (q & 1) * hc, x);
    };
    // a warp's 32 elements are 32 consecutive records of every child when they all exist and
    // belong to one node: then each result goes through the warp's staging row in shared memory
    // and is stored as whole consecutive 16-byte chunks (full sectors) instead of 16 bytes per
    // lane at the record stride (measured on the fused kernel: -18 % pre-addition time)
    const int lane = threadIdx.x & 31;
    const int64_t t0 = t - lane;
    const bool warp_full = MPG_ADD2_STAGE && L <= 32 && t0 + 32 <= total && t0 / per == (t0 + 31) / per;  // warp-uniform
    uint32_t* stage = s_stage + (threadIdx.x >> 5) * 32 * S;
    // slots.s[child]: output slot of each child, < 0: not produced (the pipelined host GEMM
    // forms its top-level children in two steps); the identity map otherwise
    auto put = [&](int child, const MP<L>& x) {
      if (slots.s[child] < 0) return;
      if (warp_full) {
        store_rec<L>(stage + lane * S, x);
        __syncwarp();
        uint4* dst = reinterpret_cast<uint4*>(out - lane * S + slots.s[child] * cs);
        const uint4* src = reinterpret_cast<const uint4*>(stage);
#pragma unroll
        for (int q = 0; q < S / 4; ++q) dst[lane + 32 * q] = src[lane + 32 * q];
        __syncwarp();
      } else {
        store_rec<L>(out + slots.s[child] * cs, x);
      }
    };
    preadd_body<L>(algo, side, sh, ld, put);
  }
}

// Two recursion levels of the pre-additions in one launch: the 49 grandchildren of every node
// straight from the node, the 7 children (the intermediate level: 7/4 of the node written and
// read again) staying in shared memory.  A CTA owns PT consecutive positions (r2, c2) of the
// grandchild grid of one node.  Phase 1: task (s, pos) -- s = (i2, j2), the sub-quadrant of the
// children -- applies the level transform to the node's four quadrant elements at that
// position and leaves the 7 children's values in shared memory (+0 where the position lies in
// the children's zero padding: pad_operand, fastmm.hpp:91-97).  Phase 2: task (c1, pos) applies
// the same transform to child c1's four sub-quadrant values and stores the 7 grandchildren.
// Same per-element operation sequence as two preadd_kernel launches: bit-identical.
template <int L, int PT>
__global__ void __launch_bounds__(4 * PT) preadd2_kernel(int algo, int side, const uint32_t* __restrict__ parent,
                                                        int64_t nodes, int rows, int cols,
                                                        uint32_t* __restrict__ grand, int sh) {
  constexpr int S = rec_stride(L);
  extern __shared__ __align__(16) uint32_t s_v[];  // [c1][s][pos] records
  const int hr1 = (rows + rows % 2) / 2, hc1 = (cols + cols % 2) / 2;
  const int hr2 = (hr1 + hr1 % 2) / 2, hc2 = (hc1 + hc1 % 2) / 2;
  const int64_t per2 = (int64_t)hr2 * hc2;
  const int64_t tiles_per_node = (per2 + PT - 1) / PT;
  const int64_t ntiles = tiles_per_node * nodes;
  const int tid = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t node = tile / tiles_per_node;
    const int64_t e0 = (tile - node * tiles_per_node) * PT;
    const uint32_t* P = parent + node * (int64_t)rows * cols * S;
    {  // phase 1: 4 PT tasks, one per thread
      const int s = tid / PT, pos = tid - s * PT;
      const int64_t e = e0 + pos;
      if (e < per2) {
        const int r2 = (int)(e / hc2), c2 = (int)(e - (int64_t)r2 * hc2);
        const int r1 = r2 + (s >> 1) * hr2, c1 = c2 + (s & 1) * hc2;  // position inside the children
        uint32_t* v = s_v + ((int64_t)s * PT + pos) * S;
        auto put = [&](int child, const MP<L>& x) { store_rec<L>(v + (int64_t)child * 4 * PT * S, x); };
        if (r1 < hr1 && c1 < hc1) {
          // small records: the four quadrant elements loaded up front (independent loads in flight)
          constexpr bool HOIST = MPG_ADDS_HOIST && L <= 8;
          MP<L> Q[HOIST ? 4 : 1];
          if constexpr (HOIST) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              load_padded<L>(P, rows, cols, r1 + (q >> 1) * hr1, c1 + (q & 1) * hc1, Q[q]);
          }
          auto ld = [&](int q, MP<L>& x) {
            if constexpr (HOIST)
              x = Q[q];
            else
              load_padded<L>(P, rows, cols, r1 + (q >> 1) * hr1, c1 + (q & 1) * hc1, x);
          };
          preadd_body<L>(algo, side, sh, ld, put);
        } else {  // the children's own zero padding (odd child dimension)
          MP<L> z;
          mp_zero(z, 0);
#pragma unroll
          for (int child = 0; child < 7; ++child) put(child, z);
        }
      }
    }
    __syncthreads();
    // phase 2: 7 PT tasks over 4 PT threads.  A warp's 32 tasks share the child and cover 32
    // consecutive positions, i.e. 32 consecutive records of every grandchild: when all 32 exist the
    // warp passes each result through a staging row in shared memory and stores it as full,
    // consecutive 16-byte chunks (whole sectors) instead of 16 bytes per lane at the record stride
    for (int task = tid; task < 7 * PT; task += 4 * PT) {
      const int c1 = task / PT, pos = task - c1 * PT;
      const int64_t e = e0 + pos;
      if (e >= per2) continue;
      const uint32_t* v = s_v + ((int64_t)c1 * 4 * PT + pos) * S;
      auto ld = [&](int q, MP<L>& x) { load_rec<L>(v + (int64_t)q * PT * S, x); };
      uint32_t* out = grand + (((node * 7 + c1) * 7) * per2 + e) * S;
      const int lane = tid & 31;
      const bool warp_full = MPG_ADD2_STAGE && PT % 32 == 0 && (e - lane) + 32 <= per2;  // warp-uniform
      uint32_t* stage = s_v + 7 * 4 * PT * S + (tid >> 5) * 32 * S;
      auto put = [&](int child, const MP<L>& x) {
        if (warp_full) {
          store_rec<L>(stage + lane * S, x);
          __syncwarp();
          uint4* dst = reinterpret_cast<uint4*>(out - lane * S + (int64_t)child * per2 * S);
          const uint4* src = reinterpret_cast<const uint4*>(stage);
#pragma unroll
          for (int q = 0; q < S / 4; ++q) dst[lane + 32 * q] = src[lane + 32 * q];
          __syncwarp();
        } else {
          store_rec<L>(out + (int64_t)child * per2 * S, x);
        }
      };
      preadd_body<L>(algo, side, sh, ld, put);
    }
    __syncthreads();
  }
}

// mpfr_set into another precision: round the ls-limb source mantissa to 32L - sh bits
template <int L>
__global__ void convert_kernel(const uint32_t* __restrict__ src, int ls, int ss, int64_t N,
                               uint32_t* __restrict__ dst, int sh, uint32_t* err) {
  constexpr int S = rec_stride(L);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = src + e * ss;
    MP<L> z;
    z.e = (int32_t)r[ls];
    z.s = r[ls + 1];
    uint32_t g = 0, st = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int q = ls - L + k;  // source limb feeding destination limb k (aligned at the top)
      z.m[k] = q >= 0 ? r[q] : 0u;
    }
    if (ls > L) {
      g = r[ls - L - 1];
      for (int q = 0; q < ls - L - 1; ++q) st |= r[q];
    }
    if (z.e != EXP_ZERO) {
      int32_t ex = z.e;
      round_p<L>(z.m, g, st, sh, ex);
      z.e = ex;
      if (exp_out_of_range(z.e)) atomicOr(err, ERR_EXP_RANGE);
    }
    store_rec<L>(dst + e * S, z);
  }
}

template <int L>
__device__ __forceinline__ void store_if(uint32_t* P, int rows, int cols, int r, int c, const MP<L>& x,
                                         uint32_t* err, const uint64_t* rowtab = nullptr, int64_t node = 0) {
  if (r < rows && c < cols) {
    if (exp_out_of_range(x.e)) atomicOr(err, ERR_EXP_RANGE);
    uint32_t* dst = rowtab ? reinterpret_cast<uint32_t*>(rowtab[r]) + (node * rows * cols + c) * rec_stride(L)
                           : P + ((int64_t)r * cols + c) * rec_stride(L);
    store_rec<L>(dst, x);
  }
}

// The combine of one quadrant element: ldc(k, x) reads child product k (0..6), put(q, x) writes
// quadrant q (0: C11, 1: C12, 2: C21, 3: C22) of the parent, tt(t1, t2) sees Winograd's T1 / T2.
template <int L, class LDC, class PUT, class TT>
__device__ __forceinline__ void postadd_body(int algo, int sh, LDC ldc, PUT put, TT tt) {
  if (algo == 3) {
    // T1 = M1+M2, T2 = T1+M4; C11 = M2+M3, C12 = (T1+M5)+M6, C21 = T2-M7, C22 = T2+M5
    MP<L> m1, m2, t1, t2, u, v;
    ldc(0, m1);
    ldc(1, m2);
    mp_add<L>(m1, m2, 0u, sh, t1);
    {
      MP<L> m4;
      ldc(3, m4);
      mp_add<L>(t1, m4, 0u, sh, t2);
    }
    tt(t1, t2);
    {
      MP<L> m3;
      ldc(2, m3);
      mp_add<L>(m2, m3, 0u, sh, u);
      put(0, u);
    }
    MP<L> m5;
    ldc(4, m5);
    {
      MP<L> m6;
      ldc(5, m6);
      mp_add<L>(t1, m5, 0u, sh, u);
      mp_add<L>(u, m6, 0u, sh, v);
      put(1, v);
    }
    {
      MP<L> m7;
      ldc(6, m7);
      mp_add<L>(t2, m7, 1u, sh, u);
      put(2, u);
    }
    mp_add<L>(t2, m5, 0u, sh, u);
    put(3, u);
  } else {
    // C11 = ((P1+P4)-P5)+P7, C12 = P3+P5, C21 = P2+P4, C22 = ((P1+P3)-P2)+P6
    MP<L> p1, p4, p5, u, v;
    ldc(0, p1);
    ldc(3, p4);
    ldc(4, p5);
    mp_add<L>(p1, p4, 0u, sh, u);
    mp_add<L>(u, p5, 1u, sh, v);
    {
      MP<L> p7;
      ldc(6, p7);
      mp_add<L>(v, p7, 0u, sh, u);
      put(0, u);
    }
    MP<L> p3;
    ldc(2, p3);
    mp_add<L>(p3, p5, 0u, sh, u);
    put(1, u);
    MP<L> p2;
    ldc(1, p2);
    mp_add<L>(p2, p4, 0u, sh, u);
    put(2, u);
    mp_add<L>(p1, p3, 0u, sh, u);
    mp_add<L>(u, p2, 1u, sh, v);
    {
      MP<L> p6;
      ldc(5, p6);
      mp_add<L>(v, p6, 0u, sh, u);
      put(3, u);
    }
  }
}

template <int L>
__global__ void __launch_bounds__(256, post_minb(L)) postadd_kernel(int algo, const uint32_t* __restrict__ children, int64_t nodes, int rows,
                               int cols, uint32_t* __restrict__ parent, uint32_t* __restrict__ t_out,
                               int sh, uint32_t* err, const int* __restrict__ rowlist, int nrows, int cc0,
                               int ncc, const uint64_t* __restrict__ rowtab) {
  constexpr int S = rec_stride(L);
  const int hr = (rows + rows % 2) / 2, hc = (cols + cols % 2) / 2;
  const int64_t per = (int64_t)hr * hc;
  // rowlist: only these child rows (row-owned combine of the multi-GPU path); [cc0, cc0 + ncc):
  // only these child columns (the LU look-ahead's column split -- child column c feeds parent
  // columns c and c + hc only)
  const int64_t per_iter = (rowlist ? (int64_t)nrows : (int64_t)hr) * ncc;
  const int64_t total = per_iter * nodes;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t node = t / per_iter;
    const int64_t ei = t - node * per_iter;
    const int ri = (int)(ei / ncc), c = cc0 + (int)(ei - (int64_t)ri * ncc);
    const int r = rowlist ? rowlist[ri] : ri;
    const int64_t e = (int64_t)r * hc + c;
    const uint32_t* M = children + (node * 7 * per + e) * S;
    const int64_t cs = per * S;
    uint32_t* P = parent + node * (int64_t)rows * cols * S;
    // small records: all seven children loaded up front (independent loads in flight)
    constexpr bool HOIST = MPG_ADDS_HOIST && L <= 8;
    MP<L> Mv[HOIST ? 7 : 1];
    if constexpr (HOIST) {
#pragma unroll
      for (int k = 0; k < 7; ++k) load_rec<L>(M + k * cs, Mv[k]);
    }
    auto ldc = [&](int k, MP<L>& x) {
      if constexpr (HOIST)
        x = Mv[k];
      else
        load_rec<L>(M + k * cs, x);
    };
    auto put = [&](int q, const MP<L>& x) {
      store_if<L>(P, rows, cols, r + (q >> 1) * hr, c + (q & 1) * hc, x, err, rowtab, node);
    };
    auto tt = [&](const MP<L>& t1, const MP<L>& t2) {
      if (t_out) {
        store_rec<L>(t_out + (node * 2 * per + e) * S, t1);
        store_rec<L>(t_out + (node * 2 * per + per + e) * S, t2);
      }
    };
    postadd_body<L>(algo, sh, ldc, put, tt);
  }
}

// Two recursion levels of the post-additions in one launch (the mirror of preadd2_kernel): the
// node's C straight from its 49 grandchildren products, the 7 children products staying in
// shared memory.  Phase 1: task (c1, pos) combines the 7 grandchildren of child c1 at position
// pos = (r2, c2) into the child's four sub-quadrant elements (dropped where they lie in the
// child's padding, as store_if does); phase 2: task (s, pos) combines the 7 children at
// sub-quadrant s into the node's four quadrant elements.  Bit-identical to two launches.
template <int L, int PT>
__global__ void __launch_bounds__(4 * PT, MPG_POST2_MINB) postadd2_kernel(int algo, const uint32_t* __restrict__ grand, int64_t nodes,
                                                         int rows, int cols, uint32_t* __restrict__ parent, int sh,
                                                         uint32_t* err) {
  constexpr int S = rec_stride(L);
  extern __shared__ __align__(16) uint32_t s_v[];  // [c1][s][pos] records
  const int hr1 = (rows + rows % 2) / 2, hc1 = (cols + cols % 2) / 2;
  const int hr2 = (hr1 + hr1 % 2) / 2, hc2 = (hc1 + hc1 % 2) / 2;
  const int64_t per2 = (int64_t)hr2 * hc2;
  const int64_t tiles_per_node = (per2 + PT - 1) / PT;
  const int64_t ntiles = tiles_per_node * nodes;
  const int tid = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t node = tile / tiles_per_node;
    const int64_t e0 = (tile - node * tiles_per_node) * PT;
    uint32_t* P = parent + node * (int64_t)rows * cols * S;
    for (int task = tid; task < 7 * PT; task += 4 * PT) {  // phase 1
      const int c1 = task / PT, pos = task - c1 * PT;
      const int64_t e = e0 + pos;
      if (e >= per2) continue;
      const int r2 = (int)(e / hc2), c2 = (int)(e - (int64_t)r2 * hc2);
      const uint32_t* M = grand + (((node * 7 + c1) * 7) * per2 + e) * S;
      constexpr bool HOIST = MPG_ADDS_HOIST && L <= 8;  // the seven products loaded up front
      MP<L> Mv[HOIST ? 7 : 1];
      if constexpr (HOIST) {
#pragma unroll
        for (int k = 0; k < 7; ++k) load_rec<L>(M + (int64_t)k * per2 * S, Mv[k]);
      }
      auto ldc = [&](int k, MP<L>& x) {
        if constexpr (HOIST)
          x = Mv[k];
        else
          load_rec<L>(M + (int64_t)k * per2 * S, x);
      };
      uint32_t* v = s_v + ((int64_t)c1 * 4 * PT + pos) * S;
      auto put = [&](int q, const MP<L>& x) {
        if (r2 + (q >> 1) * hr2 < hr1 && c2 + (q & 1) * hc2 < hc1) {
          if (exp_out_of_range(x.e)) atomicOr(err, ERR_EXP_RANGE);
          store_rec<L>(v + (int64_t)q * PT * S, x);
        }
      };
      postadd_body<L>(algo, sh, ldc, put, [](const MP<L>&, const MP<L>&) {});
    }
    __syncthreads();
    {  // phase 2: 4 PT tasks, one per thread
      const int s = tid / PT, pos = tid - s * PT;
      const int64_t e = e0 + pos;
      if (e < per2) {
        const int r2 = (int)(e / hc2), c2 = (int)(e - (int64_t)r2 * hc2);
        const int r1 = r2 + (s >> 1) * hr2, c1 = c2 + (s & 1) * hc2;  // position inside the children
        if (r1 < hr1 && c1 < hc1) {
          const uint32_t* v = s_v + ((int64_t)s * PT + pos) * S;
          auto ldc = [&](int k, MP<L>& x) { load_rec<L>(v + (int64_t)k * 4 * PT * S, x); };
          auto put = [&](int q, const MP<L>& x) {
            store_if<L>(P, rows, cols, r1 + (q >> 1) * hr1, c1 + (q & 1) * hc1, x, err);
          };
          postadd_body<L>(algo, sh, ldc, put, [](const MP<L>&, const MP<L>&) {});
        }
      }
    }
    __syncthreads();
  }
}

template <int L>
__global__ void copy2d_kernel(const uint32_t* __restrict__ src, int64_t lds, uint32_t* __restrict__ dst,
                              int64_t ldd, int rows, int cols) {
  constexpr int S = rec_stride(L);
  constexpr int CH = S / 4;
  const int64_t total = (int64_t)rows * cols * CH;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / CH;
    const int w = (int)(t - e * CH);
    const int r = (int)(e / cols), c = (int)(e - (int64_t)r * cols);
    *reinterpret_cast<uint4*>(dst + (r * ldd + c) * S + 4 * w) =
        *reinterpret_cast<const uint4*>(src + (r * lds + c) * S + 4 * w);
  }
}

template <int L>
__global__ void sub2d_kernel(uint32_t* __restrict__ C, int64_t ldc, const uint32_t* __restrict__ T, int64_t ldt,
                             int rows, int cols, int sh, uint32_t* err) {
  constexpr int S = rec_stride(L);
  const int64_t total = (int64_t)rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t - r * cols;
    MP<L> x, y, z;
    load_rec<L>(C + (r * ldc + c) * S, x);
    load_rec<L>(T + (r * ldt + c) * S, y);
    mp_add<L>(x, y, 1u, sh, z);
    if (exp_out_of_range(z.e)) atomicOr(err, ERR_EXP_RANGE);
    store_rec<L>(C + (r * ldc + c) * S, z);
  }
}

// ---------------------------------------------------------------------------
template <int L>
void launch_sub2d(uint32_t* C, int64_t ldc, const uint32_t* T, int rows, int cols, int sh, uint32_t* err,
                  cudaStream_t st, int64_t ldt) {
  if ((int64_t)rows * cols <= 0) return;
  sub2d_kernel<L><<<grid_for((int64_t)rows * cols), NT, 0, st>>>(C, ldc, T, ldt < 0 ? cols : ldt, rows, cols, sh,
                                                                 err);
}
template <int L>
void launch_soa2rec(const uint32_t* limbs, const int32_t* exp, const uint8_t* sign, int64_t N,
                    int64_t ps, uint32_t* rec, cudaStream_t st) {
  soa2rec_kernel<L><<<grid_for(N), NT, 0, st>>>(limbs, exp, sign, N, ps, rec);
}
template <int L>
void launch_soa2rec_2d(const uint32_t* limbs, const int32_t* exp, const uint8_t* sign, int64_t rows, int64_t cols,
                       int64_t ps, uint32_t* rec, int64_t ldr, cudaStream_t st) {
  if (rows * cols <= 0) return;
  soa2rec2d_kernel<L><<<grid_for(rows * cols), NT, 0, st>>>(limbs, exp, sign, rows, cols, ps, rec, ldr);
}
template <int L>
void launch_rec2soa(const uint32_t* rec, int64_t N, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                    int64_t ps, cudaStream_t st) {
  rec2soa_kernel<L><<<grid_for(N), NT, 0, st>>>(rec, N, limbs, exp, sign, ps);
}
template <int L>
void launch_addsub(const uint32_t* A, const uint32_t* B, uint32_t* C, int64_t N, int is_sub, int sh,
                   uint32_t* err, cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_vec_op<L / 32>(is_sub ? 1 : 0, A, B, C, N, sh, err, st);
#endif
  addsub_kernel<L><<<grid_for(N), NT, 0, st>>>(A, B, C, N, is_sub ? 1u : 0u, sh, err);
}
template <int L>
void launch_vec_op(int op, const uint32_t* A, const uint32_t* B, uint32_t* C, int64_t N, int sh,
                   uint32_t* err, cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_vec_op<L / 32>(op, A, B, C, N, sh, err, st);
#endif
  vec_op_kernel<L><<<grid_for(N), NT, 0, st>>>(op, A, B, C, N, sh, err);
}
template <int L>
int preadd_stage_bytes() {  // preadd_kernel's staging rows (one per warp; register-resident formats only)
  if (!MPG_ADD2_STAGE || L > 32) return 0;
  const int bytes = (NT / 32) * 32 * rec_stride(L) * (int)sizeof(uint32_t);
  smem_attr_once((const void*)preadd_kernel<L>, bytes);
  return bytes;
}
template <int L>
void launch_preadd(int algo, int side, const uint32_t* parent, int64_t nodes, int rows, int cols,
                   uint32_t* children, int sh, uint32_t* err, cudaStream_t st) {
  (void)err;
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_preadd<L / 32>(algo, side, parent, nodes, rows, cols, children, sh, st);
#endif
  const int64_t total = (int64_t)((rows + rows % 2) / 2) * ((cols + cols % 2) / 2) * nodes;
  preadd_kernel<L><<<grid_for(total), NT, preadd_stage_bytes<L>(), st>>>(algo, side, parent, nodes, rows, cols,
                                                                          children, sh,
                                                                          ChildSlots{{0, 1, 2, 3, 4, 5, 6}});
}
template <int L>
void launch_preadd_slots(int algo, int side, const uint32_t* parent, int rows, int cols, uint32_t* children,
                         ChildSlots slots, int sh, cudaStream_t st) {
  const int64_t total = (int64_t)((rows + rows % 2) / 2) * ((cols + cols % 2) / 2);
  preadd_kernel<L><<<grid_for(total), NT, preadd_stage_bytes<L>(), st>>>(algo, side, parent, 1, rows, cols, children,
                                                                          sh, slots);
}
// two levels at once (preadd2_kernel): grand = 49 operands per node, each ceil(ceil(rows/2)/2) x
// ceil(ceil(cols/2)/2); false when this limb count has no fused kernel (the caller runs two levels)
template <int L>
bool launch_preadd2(int algo, int side, const uint32_t* parent, int64_t nodes, int rows, int cols,
                    uint32_t* grand, int sh, cudaStream_t st) {
  if constexpr (L > 32 || L < 4) {
    return false;
  } else {
    // measured (profiles/r02_ab_fuse2.jsonl, n = 1024 Winograd): 32 positions per CTA at 256 / 512
    // bits (16: +1.5 %, 64: +3.5 / +12 %); 16 at 1024 bits (1.89 vs 2.10 ms: 129 KB of shared memory
    // per CTA with 32)
    constexpr int PT = L > 16 ? MPG_ADD2_PT / 2 : MPG_ADD2_PT;
    constexpr int S = rec_stride(L);
    const int hr1 = (rows + rows % 2) / 2, hc1 = (cols + cols % 2) / 2;
    const int64_t per2 = (int64_t)((hr1 + hr1 % 2) / 2) * ((hc1 + hc1 % 2) / 2);
    const int64_t ntiles = ((per2 + PT - 1) / PT) * nodes;
    if (ntiles <= 0) return true;
    const int smem = (7 * 4 * PT + 4 * PT) * S * (int)sizeof(uint32_t);  // children + one staging row per warp
    smem_attr_once((const void*)preadd2_kernel<L, PT>, smem);
    const int grid = (int)std::min<int64_t>(ntiles, 148 * 64);
    preadd2_kernel<L, PT><<<grid, 4 * PT, smem, st>>>(algo, side, parent, nodes, rows, cols, grand, sh);
    return true;
  }
}
template <int L>
void launch_postadd(int algo, const uint32_t* children, int64_t nodes, int rows, int cols,
                    uint32_t* parent, uint32_t* t_out, int sh, uint32_t* err, cudaStream_t st, const int* rowlist,
                    int nrows, int cc0, int ncc, const uint64_t* rowtab) {
  const int hc = (cols + cols % 2) / 2;
  if (ncc < 0) ncc = hc - cc0;
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) {  // (the column split and row tables are not used with the wide formats)
      if (cc0 != 0 || ncc != hc || rowtab) return;
      return wmp::launch_postadd<L / 32>(algo, children, nodes, rows, cols, parent, t_out, sh, err, st, rowlist,
                                         nrows);
    }
#endif
  const int64_t total = (int64_t)(rowlist ? nrows : (rows + rows % 2) / 2) * ncc * nodes;
  if (total <= 0) return;
  postadd_kernel<L><<<grid_for(total), NT, 0, st>>>(algo, children, nodes, rows, cols, parent, t_out, sh,
                                                     err, rowlist, nrows, cc0, ncc, rowtab);
}
// two levels at once (postadd2_kernel); false when this limb count has no fused kernel
template <int L>
bool launch_postadd2(int algo, const uint32_t* grand, int64_t nodes, int rows, int cols, uint32_t* parent,
                     int sh, uint32_t* err, cudaStream_t st) {
  // (at 1024 bits the fused combine needs 255 registers and runs 1.77 vs 1.07 ms: not offered)
  if constexpr (!has_postadd2(L)) {
    return false;
  } else {
    constexpr int PT = MPG_ADD2_PT;
    constexpr int S = rec_stride(L);
    const int hr1 = (rows + rows % 2) / 2, hc1 = (cols + cols % 2) / 2;
    const int64_t per2 = (int64_t)((hr1 + hr1 % 2) / 2) * ((hc1 + hc1 % 2) / 2);
    const int64_t ntiles = ((per2 + PT - 1) / PT) * nodes;
    if (ntiles <= 0) return true;
    const int smem = 7 * 4 * PT * S * (int)sizeof(uint32_t);
    smem_attr_once((const void*)postadd2_kernel<L, PT>, smem);
    const int grid = (int)std::min<int64_t>(ntiles, 148 * 64);
    postadd2_kernel<L, PT><<<grid, 4 * PT, smem, st>>>(algo, grand, nodes, rows, cols, parent, sh, err);
    return true;
  }
}
template <int L>
void launch_copy2d(const uint32_t* src, int64_t lds, uint32_t* dst, int64_t ldd, int rows, int cols,
                   cudaStream_t st) {
  const int64_t total = (int64_t)rows * cols * (rec_stride(L) / 4);
  copy2d_kernel<L><<<grid_for(total), NT, 0, st>>>(src, lds, dst, ldd, rows, cols);
}

template <int L>
void launch_convert(const uint32_t* src, int ls, int64_t N, uint32_t* dst, int sh, uint32_t* err, cudaStream_t st) {
  convert_kernel<L><<<grid_for(N), NT, 0, st>>>(src, ls, rec_stride(ls), N, dst, sh, err);
}

// the fused two-level transforms are instantiated in their own translation units
// (elementwise_fused{8,16,32}.cu: MPG_EW_PART = 1, 2, 3), which compile beside this one
#define MPG_INST_FUSED(L)                                                                                       \
  template bool launch_preadd2<L>(int, int, const uint32_t*, int64_t, int, int, uint32_t*, int, cudaStream_t); \
  template bool launch_postadd2<L>(int, const uint32_t*, int64_t, int, int, uint32_t*, int, uint32_t*, cudaStream_t);
#if MPG_EW_PART == 1
MPG_INST_FUSED(1)
MPG_INST_FUSED(2)
MPG_INST_FUSED(4)
MPG_INST_FUSED(8)
#elif MPG_EW_PART == 2
MPG_INST_FUSED(16)
#elif MPG_EW_PART == 3
MPG_INST_FUSED(32)
#else
#define MPG_INST(L)                                                                                     \
  template void launch_soa2rec<L>(const uint32_t*, const int32_t*, const uint8_t*, int64_t, int64_t,   \
                                  uint32_t*, cudaStream_t);                                             \
  template void launch_rec2soa<L>(const uint32_t*, int64_t, uint32_t*, int32_t*, uint8_t*, int64_t,    \
                                  cudaStream_t);                                                        \
  template void launch_soa2rec_2d<L>(const uint32_t*, const int32_t*, const uint8_t*, int64_t, int64_t, \
                                     int64_t, uint32_t*, int64_t, cudaStream_t);                        \
  template void launch_addsub<L>(const uint32_t*, const uint32_t*, uint32_t*, int64_t, int, int,        \
                                 uint32_t*, cudaStream_t);                                              \
  template void launch_vec_op<L>(int, const uint32_t*, const uint32_t*, uint32_t*, int64_t, int,        \
                                 uint32_t*, cudaStream_t);                                              \
  template void launch_preadd<L>(int, int, const uint32_t*, int64_t, int, int, uint32_t*, int,          \
                                 uint32_t*, cudaStream_t);                                              \
  template void launch_postadd<L>(int, const uint32_t*, int64_t, int, int, uint32_t*, uint32_t*, int,   \
                                  uint32_t*, cudaStream_t, const int*, int, int, int, const uint64_t*); \
  template void launch_copy2d<L>(const uint32_t*, int64_t, uint32_t*, int64_t, int, int, cudaStream_t); \
  template void launch_convert<L>(const uint32_t*, int, int64_t, uint32_t*, int, uint32_t*, cudaStream_t); \
  template void launch_sub2d<L>(uint32_t*, int64_t, const uint32_t*, int, int, int, uint32_t*, cudaStream_t,   \
                                int64_t);
#if MPG_WIDE
#ifdef MPG_WIDE_L  // one wide limb count per translation unit (compile time)
MPG_INST(MPG_WIDE_L)
MPG_INST_FUSED(MPG_WIDE_L)
#else
MPG_INST(64)
MPG_INST(128)
MPG_INST(256)
MPG_INST(288)
MPG_INST_FUSED(64)
MPG_INST_FUSED(128)
MPG_INST_FUSED(256)
MPG_INST_FUSED(288)
#endif
#else
MPG_INST(1)
MPG_INST(2)
MPG_INST(4)
MPG_INST(8)
MPG_INST(16)
MPG_INST(32)
#define MPG_INST_SLOTS(L)                                                                                     \
  template void launch_preadd_slots<L>(int, int, const uint32_t*, int, int, uint32_t*, ChildSlots, int, \
                                       cudaStream_t);
MPG_INST_SLOTS(1)
MPG_INST_SLOTS(2)
MPG_INST_SLOTS(4)
MPG_INST_SLOTS(8)
MPG_INST_SLOTS(16)
MPG_INST_SLOTS(32)
#endif
#endif  // MPG_EW_PART

}  // namespace mpg
