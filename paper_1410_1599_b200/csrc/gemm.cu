// gemm.cu -- K1 mp_gemm_leaf: batched MP GEMM leaf kernel for sm_100a.
//
// Replaces the reference's hot loop detail::mul_views (matrix.hpp:147-155) and the
// Block tile loop block_mul_impl (matrix.hpp:196-216):
//   c_ij = RN(..RN(RN(a_i0 b_0j) + RN(a_i1 b_1j))..)   left to right in k
// and, with a k-tile kb < l, a fresh accumulator per k-tile followed by
// C = RN(C + P).  One thread owns one output element: the k order inside an
// element is sequential (no split-K -- reassociation would change the rounding),
// parallelism comes from outputs and from the batch of leaves (grid.z).
//
// Operands are AoS records (rec_stride(L) words: limbs, exp, sign, pad) staged
// through shared memory with cp.async (16-byte, zero-fill outside the matrix) in a
// two-stage pipeline.  A warp covers 2 rows x 16 columns of C: the a-record of
// each k is a broadcast LDS.128, the 16 b-records are consecutive records whose
// stride/4 is odd, so the LDS.128 quarter-warps are bank-conflict free.
// Limb products are IMAD / IMAD.HI on the FMA pipe (mp_arith.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "mp_arith.cuh"
#if MPG_WIDE
#include "wkern.cuh"
#endif

#ifndef MPG_MINB_8
#define MPG_MINB_8 6  // 8 x 16 tiles of 128 threads; with k-tile 16 shared memory holds 6 CTAs per SM, so the register cap is 80 (70 used): -0.3 % vs a cap of 64 (profiles/r02_ab_tk.jsonl)
#endif
#define MPG_MINB_1 4
#define MPG_MINB_2 4
#define MPG_MINB_4 3
#ifndef MPG_MINB_16
#define MPG_MINB_16 5  // with the carry-chained product: 5 CTAs of 128 threads (96 registers) beat 6 (80, spilling) by 3.8 % at 512 bits (profiles/r02_ab_eo2.jsonl)
#endif
#ifndef MPG_TK_16
#define MPG_TK_16 8
#endif
#ifndef MPG_TM_32
#define MPG_TM_32 8
#endif
#ifndef MPG_TK_32
#define MPG_TK_32 8  // round 2 (bulk-copied k-tiles): 8 < 6 < 4 < 2 at 1024 bits (68.2 / 68.2 / 68.4 / 70.1 ms leaf)
#endif
#ifndef MPG_MINB_32
#define MPG_MINB_32 3  // 166 registers: 3 CTAs of 128 threads per SM (measured best, 1024-bit cfg)
#endif
#ifndef MPG_LOAD
#define MPG_LOAD load_rec_s
#endif

namespace mpg {

__device__ __forceinline__ void cp_async16(uint32_t* sdst, const uint32_t* gsrc, int src_bytes) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- bulk-copy (TMA engine) staging of full tiles --------------------------------
#ifndef MPG_BULK
#define MPG_BULK 1  // interior tiles by cp.async.bulk + mbarrier; edge tiles by zero-filling cp.async
#endif
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t* sdst, const uint32_t* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

#ifndef MPG_TILE_ALT
#define MPG_TILE_ALT 1  // half-width tiles for ragged leaves (launch_gemm)
#endif
#ifndef MPG_TILE_ALT_NUM  // ... when they cover the m x n outputs with < NUM/DEN of the default tiles' area
#define MPG_TILE_ALT_NUM 97
#define MPG_TILE_ALT_DEN 100
#endif

#ifndef MPG_NZ_SPLIT
#define MPG_NZ_SPLIT 1  // measured: -2.3 % leaf time at 256 bits, -1 % at 512
#endif

#ifndef MPG_KK_UNROLL_8
#define MPG_KK_UNROLL_8 2  // measured: 2 beats 1 and 4 at 256 bits (and loses at L >= 16)
#endif

#ifndef MPG_SH0_SPEC
// limb counts whose p == 32 L case gets its own leaf instantiation (measured: leaf -7.2 % at
// 128 bits, -3.4 % at 256; +3 % / +5 % at 512 / 1024, where it costs registers)
#define MPG_SH0_SPEC(L) ((L) == 4 || (L) == 8)
#endif
#ifndef MPG_SADDR
#define MPG_SADDR 1  // measured: leaf -1.4 % at 256 bits, neutral at 512 / 1024 (profiles/r02_ab_saddr.jsonl)
#endif

// record from shared memory (32-bit shared-window address): 16-byte vector loads
template <int L>
__device__ __forceinline__ void lds_rec(uint32_t addr, MP<L>& x) {
  constexpr int S = rec_stride(L);
  uint32_t w[S];
#pragma unroll
  for (int k = 0; k < S; k += 4)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[k]), "=r"(w[k + 1]), "=r"(w[k + 2]), "=r"(w[k + 3])
                 : "r"(addr + 4 * k));
#pragma unroll
  for (int k = 0; k < L; ++k) x.m[k] = w[k];
  x.e = (int32_t)w[L];
  x.s = w[L + 1];
}

#ifndef MPG_TM_8
#define MPG_TM_8 8
#endif

#ifndef MPG_TK_8
#define MPG_TK_8 16  // 16 (6 CTAs per SM by shared memory, whole k-tiles at l = 32 / 64) vs 12 (8 CTAs): leaf -0.3 % at l = 64, -0.9 % at l = 32, LU -0.5 % (profiles/r02_ab_tk.jsonl)
#endif

#ifndef MPG_U_8
#define MPG_U_8 1
#endif

// per-L tiling: TM x (TN*U) outputs per CTA of TM*TN threads, each thread owning U
// outputs of one row (columns tx, tx+TN, ...) -- U independent accumulation chains
// per thread share the a-record
template <int L>
struct GemmCfg {  // wide formats (L = 64 .. 288, gemm_wide.cu): mantissas in local memory
  static constexpr int MINB = 1, TM = 8, TN = 16, TK = 2, U = 1;
  static constexpr int KU = 1;
};
template <>
struct GemmCfg<1> {
  static constexpr int MINB = MPG_MINB_1, TM = 16, TN = 16, TK = 16, U = 1;
  static constexpr int KU = 1;
};
template <>
struct GemmCfg<2> {
  static constexpr int MINB = MPG_MINB_2, TM = 16, TN = 16, TK = 16, U = 1;
  static constexpr int KU = 1;
};
template <>
struct GemmCfg<4> {
  static constexpr int MINB = MPG_MINB_4, TM = 16, TN = 16, TK = 16, U = 1;
  static constexpr int KU = 1;
};
template <>
struct GemmCfg<8> {
  static constexpr int MINB = MPG_MINB_8, TM = MPG_TM_8, TN = 16, TK = MPG_TK_8, U = MPG_U_8;
  static constexpr int KU = MPG_KK_UNROLL_8;
};
template <>
struct GemmCfg<16> {
  static constexpr int MINB = MPG_MINB_16, TM = 8, TN = 16, TK = MPG_TK_16, U = 1;
  static constexpr int KU = 1;
};
template <>
struct GemmCfg<32> {
  static constexpr int MINB = MPG_MINB_32, TM = MPG_TM_32, TN = 16, TK = MPG_TK_32, U = 1;
  static constexpr int KU = 1;
};

template <int L, int TM, int TN, int TK, int U, bool FOLD, bool SH0 = false>
__global__ void __launch_bounds__(TM* TN, GemmCfg<L>::MINB) gemm_leaf_kernel(const GemmArgs g) {
  // SH0: p == 32 L (no unused low bits) known at compile time -- the rounding position tests
  // leave the multiply-add (MPG_SH0_SPEC)
#define MPG_SH (SH0 ? 0 : g.sh)
  // FOLD: Block k-tiles (kb < l) -- a second accumulator and the C = RN(C + P) folds;
  // without them (Simple, Strassen / Winograd leaves, LU Schur) the result is P itself
  // (RN(-0 + P) == P), so acc and the per-step tile check are compiled out.
  constexpr int S = rec_stride(L);
  constexpr int NT = TM * TN;
  constexpr int TNB = TN * U;  // CTA tile width
  constexpr int A_WORDS = TM * TK * S, B_WORDS = TK * TNB * S;
  constexpr bool A_STREAM = (L >= 16);  // large L: a-limbs read from smem inside the product
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* sA = smem;
  uint32_t* sB = smem + 2 * A_WORDS;

  const int tid = threadIdx.x, tx = tid % TN, ty = tid / TN;
  const int z = blockIdx.z;
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TNB;
  const uint32_t* A = g.A + (int64_t)z * g.strideA * S;
  const uint32_t* B = g.B + (int64_t)z * g.strideB * S;
  uint32_t* C = g.C + (int64_t)z * g.strideC * S;
  const int KT = (g.l + TK - 1) / TK;
  const int i = i0 + ty;
  const bool active = (i < g.m) && (j0 + tx < g.n);

  // stages whose A and B tiles lie inside the matrices are moved by the bulk-copy engine
  // (one 16-byte-aligned row segment per copy, issued by warp 0, completion on an
  // mbarrier); edge tiles use zero-filling cp.async.  Uniform per stage.
  __shared__ __align__(8) uint64_t s_bar[2];
  uint32_t bar_phase = 0;  // bit b: parity of s_bar[b]'s next completion
  auto full_tile = [&](int kt) {
    const int k0 = kt * TK;
    // (k-tiles of 2 records -- L = 32 -- keep cp.async: measured 0.3 % faster there)
    return MPG_BULK && TK >= 4 && i0 + TM <= g.m && j0 + TNB <= g.n && k0 + TK <= g.l;
  };
  auto stage = [&](int kt, int buf) {
    const int k0 = kt * TK;
    constexpr int CH = S / 4;
    if (full_tile(kt)) {
      constexpr uint32_t ABYTES = TK * S * 4, BBYTES = TNB * S * 4;
      if (tid < 32) {
        if (tid == 0) mbar_expect(&s_bar[buf], TM * ABYTES + TK * BBYTES);
        __syncwarp();
        for (int c = tid; c < TM + TK; c += 32) {
          if (c < TM)
            bulk_g2s(sA + buf * A_WORDS + c * TK * S, A + ((int64_t)(i0 + c) * g.lda + k0) * S, ABYTES, &s_bar[buf]);
          else
            bulk_g2s(sB + buf * B_WORDS + (c - TM) * TNB * S, B + ((int64_t)(k0 + c - TM) * g.ldb + j0) * S, BBYTES,
                     &s_bar[buf]);
        }
      }
      return;
    }
#pragma unroll 1
    for (int c = tid; c < TM * TK * CH; c += NT) {
      const int e = c / CH, w = c - e * CH;
      const int r = e / TK, kk = e - r * TK;
      const int gi = i0 + r, gk = k0 + kk;
      const bool ok = gi < g.m && gk < g.l;
      const uint32_t* src = A + ((int64_t)(ok ? gi : 0) * g.lda + (ok ? gk : 0)) * S + 4 * w;
      cp_async16(sA + buf * A_WORDS + e * S + 4 * w, src, ok ? 16 : 0);
    }
#pragma unroll 1
    for (int c = tid; c < TK * TNB * CH; c += NT) {
      const int e = c / CH, w = c - e * CH;
      const int kk = e / TNB, cc = e - kk * TNB;
      const int gk = k0 + kk, gj = j0 + cc;
      const bool ok = gk < g.l && gj < g.n;
      const uint32_t* src = B + ((int64_t)(ok ? gk : 0) * g.ldb + (ok ? gj : 0)) * S + 4 * w;
      cp_async16(sB + buf * B_WORDS + e * S + 4 * w, src, ok ? 16 : 0);
    }
  };

  // Accumulators start at -0: RN(-0 + x) == x exactly for every x (signed zeros
  // included), so "C = P" for the first Block k-tile and "acc = first product" are
  // the same rounded add as every later step -- no data-dependent copies in the
  // hot loop (matrix.hpp:147-155, :203-212).
  MP<L> acc[U], pacc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    mp_zero(acc[u], 1u);
    mp_zero(pacc[u], 1u);
  }

  int next_b = g.kb;  // k at which the next Block k-tile starts

  if (tid == 0) {
    mbar_init1(&s_bar[0]);
    mbar_init1(&s_bar[1]);
  }
  __syncthreads();
  stage(0, 0);
  cp_async_commit();
  for (int kt = 0; kt < KT; ++kt) {
    if (kt + 1 < KT) stage(kt + 1, (kt + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    if (full_tile(kt)) {  // bulk-copied stage: wait for its bytes on the mbarrier
      const int b = kt & 1;
      mbar_wait_parity(&s_bar[b], (bar_phase >> b) & 1u);
      bar_phase ^= 1u << b;
    }
    __syncthreads();
    if (active) {
      const uint32_t* a_rows = sA + (kt & 1) * A_WORDS + ty * TK * S;
      const uint32_t* b_cols = sB + (kt & 1) * B_WORDS + tx * S;
      const int kend = min(TK, g.l - kt * TK);
#if MPG_SADDR
      // shared-window addresses carried through the k loop (two adds per step) instead of
      // pointers the compiler rematerialises from the thread index every step
      uint32_t sa_cur = smem_addr(a_rows), sb_cur = smem_addr(b_cols);
#endif
#pragma unroll GemmCfg<L>::KU
      for (int kk = 0; kk < kend; ++kk) {
        const int k = kt * TK + kk;
        if (FOLD && k == next_b) {  // Block k-tile boundary: C = RN(C + P), fresh P
#pragma unroll
          for (int u = 0; u < U; ++u) {
            mp_add<L>(acc[u], pacc[u], 0u, MPG_SH, acc[u]);
            mp_zero(pacc[u], 1u);
          }
          next_b += g.kb;
        }
        const uint32_t* ar = a_rows + kk * S;
        MP<L> a;
#if MPG_SADDR
        if constexpr (!A_STREAM) lds_rec<L>(sa_cur, a);
#else
        if constexpr (!A_STREAM) MPG_LOAD<L>(ar, a);
#endif
#pragma unroll
        for (int u = 0; u < U; ++u) {
          MP<L> b, t;
#if MPG_SADDR
          lds_rec<L>(sb_cur + u * TN * S * 4, b);
#else
          MPG_LOAD<L>(b_cols + (kk * TNB + u * TN) * S, b);
#endif
          const int32_t ae = A_STREAM ? (int32_t)ar[L] : a.e;
          const uint32_t as = A_STREAM ? ar[L + 1] : a.s;
          auto a_at = [&](int q) { return A_STREAM ? ar[q] : a.m[q]; };
#if MPG_NZ_SPLIT
          // one zero test for the whole multiply-add: the product of nonzero operands is
          // nonzero, so with a nonzero accumulator neither primitive needs its own
          if (ae == EXP_ZERO || b.e == EXP_ZERO || pacc[u].e == EXP_ZERO) {
            mp_mul_g<L>(a_at, ae, as, b, MPG_SH, t);
            mp_add<L>(pacc[u], t, 0u, MPG_SH, pacc[u]);
          } else {
            mp_mul_g<L, decltype(a_at), true>(a_at, ae, as, b, MPG_SH, t);
            mp_add<L, true>(pacc[u], t, 0u, MPG_SH, pacc[u]);
          }
#else
          mp_mul_g<L>(a_at, ae, as, b, MPG_SH, t);
          mp_add<L>(pacc[u], t, 0u, MPG_SH, pacc[u]);
#endif
        }
#if MPG_SADDR
        sa_cur += S * 4;
        sb_cur += TNB * S * 4;
#endif
      }
    }
    __syncthreads();
  }
  if (!active) return;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = j0 + tx + u * TN;
    if (j >= g.n) break;
    MP<L> res;
    if constexpr (FOLD) {
      mp_add<L>(acc[u], pacc[u], 0u, MPG_SH, res);
    } else {
      res = pacc[u];
    }
    uint32_t* cr = g.rowtab ? reinterpret_cast<uint32_t*>(g.rowtab[i]) + ((g.batch0 + z) * g.strideC + j) * S
                            : C + ((int64_t)i * g.ldc + j) * S;
    if (g.sub_from_c) {  // LU Schur update: A22 = RN(A22 - prod) (blocklu.hpp:138-141)
      MP<L> old;
      load_rec<L>(cr, old);
      mp_add<L>(old, res, 1u, MPG_SH, res);
    }
    if (exp_out_of_range(res.e)) atomicOr(g.err, ERR_EXP_RANGE);
    store_rec<L>(cr, res);
  }
}
#undef MPG_SH

// (A warp-specialised L = 8 leaf -- producer warps forming the rounded products, accumulator warps
// folding them in k order through a shared-memory ring -- was bit-exact but 22 % slower: leaf
// 9.19 vs 7.50 ms at cfg2, profiles/r02_ab_ws.jsonl, r02_leaf8_ws_summary.json.  Removed.)

template <int L, int TM, int TN>
void launch_tiles(const GemmArgs& g, cudaStream_t st) {
  constexpr int TK = GemmCfg<L>::TK, U = GemmCfg<L>::U;
  constexpr int S = rec_stride(L);
  const size_t smem = sizeof(uint32_t) * 2 * (TM * TK * S + TK * TN * U * S);
  auto kern = g.kb < g.l ? gemm_leaf_kernel<L, TM, TN, TK, U, true> : gemm_leaf_kernel<L, TM, TN, TK, U, false>;
  if constexpr (MPG_SH0_SPEC(L)) {
    if (g.sh == 0)
      kern = g.kb < g.l ? gemm_leaf_kernel<L, TM, TN, TK, U, true, true> : gemm_leaf_kernel<L, TM, TN, TK, U, false, true>;
  }
  smem_attr_once((const void*)kern, (int)smem);
  // grid.z is limited to 65535: deep recursions (7^d leaves) launch in batch chunks
  for (int z0 = 0; z0 < g.batch; z0 += 65535) {
    GemmArgs gz = g;
    gz.batch = std::min(65535, g.batch - z0);
    gz.A += (int64_t)z0 * g.strideA * S;
    gz.B += (int64_t)z0 * g.strideB * S;
    gz.C += (int64_t)z0 * g.strideC * S;
    gz.batch0 = g.batch0 + z0;
    dim3 grid((g.n + TN * U - 1) / (TN * U), (g.m + TM - 1) / TM, gz.batch);
    kern<<<grid, TM * TN, smem, st>>>(gz);
  }
}

template <int L>
void launch_gemm(const GemmArgs& g, cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_gemm<L / 32>(g, st);
#endif
  if constexpr (L == 8 || L == 16 || L == 32) {  // tensor-core leaf (gemm_tc.cu) when MPGPU_GEMM=tc
    if (gemm_tc_enabled() && !g.rowtab && launch_gemm_tc<L>(g, st)) return;
  }
  constexpr int TM = GemmCfg<L>::TM, TN = GemmCfg<L>::TN, U = GemmCfg<L>::U;
  if constexpr (U == 1 && TN == 16 && L <= 32) {
    // ragged leaves (odd recursion shapes, e.g. 32 x 25 x 49 at config 3): a half-width,
    // double-height tile when it covers the m x n outputs with fewer idle threads
    auto cover = [&](int tm, int tn) {
      return (int64_t)((g.m + tm - 1) / tm) * tm * (int64_t)((g.n + tn - 1) / tn) * tn;
    };
    if (MPG_TILE_ALT && cover(2 * TM, TN / 2) * MPG_TILE_ALT_DEN < cover(TM, TN) * MPG_TILE_ALT_NUM)
      return launch_tiles<L, 2 * TM, TN / 2>(g, st);
  }
  launch_tiles<L, TM, TN>(g, st);
}

#if MPG_WIDE
template void launch_gemm<64>(const GemmArgs&, cudaStream_t);
template void launch_gemm<128>(const GemmArgs&, cudaStream_t);
template void launch_gemm<256>(const GemmArgs&, cudaStream_t);
template void launch_gemm<288>(const GemmArgs&, cudaStream_t);
#else
template void launch_gemm<1>(const GemmArgs&, cudaStream_t);
template void launch_gemm<2>(const GemmArgs&, cudaStream_t);
template void launch_gemm<4>(const GemmArgs&, cudaStream_t);
template void launch_gemm<8>(const GemmArgs&, cudaStream_t);
template void launch_gemm<16>(const GemmArgs&, cudaStream_t);
template void launch_gemm<32>(const GemmArgs&, cudaStream_t);
#endif

}  // namespace mpg
