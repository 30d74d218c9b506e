// gemm_tc.cu -- K1' tensor-core MP GEMM leaf kernel (tcgen05, kind::i8) for sm_100a.
//
// Same contract as gemm_leaf_kernel (gemm.cu): c_ij = RN(..RN(RN(a_i0 b_0j) +
// RN(a_i1 b_1j))..) left to right in k (matrix.hpp:147-155), optional Block k-tiles
// (matrix.hpp:196-216) and LU Schur epilogue -- bit-identical results.  What changes is
// who forms the exact limb products:
//
//   For one k and one row i, the exact products a_ik * b_kj of 64 columns j are byte
//   convolutions  D[j][t] = sum_s B_j[s] * A_i[t - s]  (bytes of the mantissas), i.e.
//   one unsigned-int8 tensor-core MMA  D(64 x 2K) = B(64 x K) * Toeplitz(A_i)(2K x K)^T
//   with K = 4L mantissa bytes, int32 accumulation in TMEM (column sums < K*255^2 <
//   2^23: exact).  The Toeplitz operand is built in shared memory from a_ik's bytes.
//   M = 64 MMAs put their rows in lanes 0..15 of each 32-lane TMEM quadrant, or 16..31
//   with a lane offset of 16: two MMAs (two rows i) fill a 128-lane slab.
//
// Warp roles (one CTA per SM, it owns all 512 TMEM columns):
//   producers (PW warps)  cp.async the records of step k+D into a raw ring, then build
//                         stage k: the B_j byte rows (canonical K-major, no swizzle),
//                         the IT Toeplitz operands (sliding funnel-shift window, only
//                         the non-zero band is written; the rest stays zero), exponents
//                         and signs.  -> full[s]
//   MMA warp (1 thread)   waits full[s] and a free TMEM buffer, issues the IT MMAs of
//                         the step, commits -> tfull[b]
//   epilogue (4*SPB warps) one output (i, j) per thread: tcgen05.ld its 2K conv columns,
//                         carry-combine them into the exact 2L-limb product, release the
//                         TMEM buffer and the stage (-> tempty[b], sempty[s]), then round
//                         the product (MPFR RNDN) and accumulate it with the same mp_add
//                         as the IMAD kernel, so the rounding sequence is identical.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "mp_arith.cuh"

namespace mpg {
namespace tc {

template <int L>
struct Cfg {
  static constexpr int S = rec_stride(L);
  static constexpr int KB = 4 * L;                    // mantissa bytes = MMA K
  static constexpr int NC = 8 * L;                    // conv columns per result = MMA N
  static constexpr int TB = (L >= 32) ? 1 : 2;        // TMEM buffers
  static constexpr int SPB = 512 / (NC * TB);         // 128-lane slabs per buffer
  static constexpr int IT = 2 * SPB;                  // rows i per CTA = MMAs per step
  static constexpr int JT = 64;                       // columns j per CTA (MMA M)
  static constexpr int EPI_WARPS = 4 * SPB;
  static constexpr int PW = (L == 8) ? 2 : 3;         // producer warps (NWARPS % 4 == 0 for L >= 16)
  static constexpr int NWARPS = EPI_WARPS + PW + 1;   // + MMA warp
  static constexpr int NT = 32 * NWARPS;
  static constexpr int NS = (L >= 32) ? 1 : 4;        // operand stages
  static constexpr int D = 2, NR = D + 1;             // raw prefetch distance / ring
  static constexpr int SBO = (KB / 16) * 128;         // K-major no-swizzle: 8-row group stride
  static constexpr int LBO = 128;                     // 16-byte K chunk stride
  static constexpr int A_BYTES = JT * KB;
  static constexpr int T_BYTES = NC * KB;
  static constexpr int RW = 3 * KB / 4;               // words of a reversed, zero-padded mantissa
  static constexpr int OFF_T = A_BYTES;
  static constexpr int OFF_R = OFF_T + IT * T_BYTES;
  static constexpr int OFF_E = OFF_R + 4 * IT * RW;   // ae[IT] as[IT] be[JT] bs[JT]
  static constexpr int STAGE = OFF_E + 8 * (IT + JT);
  static constexpr int RAW = 4 * S * (JT + IT);       // B records of row k, then A records
  static constexpr int SMEM = NS * STAGE + NR * RAW;
  static_assert(STAGE % 16 == 0 && RAW % 16 == 0, "16-byte aligned stages");
  static_assert(SMEM <= 232448, "shared memory");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int L>
__device__ __forceinline__ int kmaj(int r, int kbyte) {
  return (r >> 3) * Cfg<L>::SBO + (kbyte >> 4) * Cfg<L>::LBO + (r & 7) * 16 + (kbyte & 15);
}
template <int L>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((Cfg<L>::LBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((Cfg<L>::SBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); SWIZZLE_NONE, base offset 0
  return d;
}
__host__ __device__ constexpr uint32_t idesc_u8(int m, int n) {
  // D int32 (c_format 2 @ bits 4-5), A/B unsigned 8-bit, K-major; N>>3 @ 17-22, M>>4 @ 24-28
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cp16(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1) gemm_tc_kernel(const GemmArgs g) {
  using CF = Cfg<L>;
  constexpr int S = CF::S, KB = CF::KB, NC = CF::NC, IT = CF::IT, JT = CF::JT;
  constexpr int NS = CF::NS, TB = CF::TB, SPB = CF::SPB, EPI_WARPS = CF::EPI_WARPS;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[NS], sempty_bar[NS], tfull_bar[TB], tempty_bar[TB];
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int z = blockIdx.z;
  const int i0 = blockIdx.y * IT, j0 = blockIdx.x * JT;
  const uint32_t* A = g.A + (int64_t)z * g.strideA * S;
  const uint32_t* B = g.B + (int64_t)z * g.strideB * S;
  uint32_t* C = g.C + (int64_t)z * g.strideC * S;
  auto stage = [&](int s) { return smem + (size_t)s * CF::STAGE; };
  uint8_t* raw0 = smem + (size_t)NS * CF::STAGE;

  // zero the stages once: Toeplitz chunks outside the band and the R pads stay zero
  for (int x = tid; x < NS * CF::STAGE / 16; x += CF::NT) reinterpret_cast<uint4*>(smem)[x] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], CF::PW * 32);
      mbar_init(&sempty_bar[s], EPI_WARPS);
    }
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base_s;

  if (warp < EPI_WARPS) {
    // ================= epilogue: one output (i, j) per thread =================
    const int q = warp & 3, sl = warp >> 2, h = lane >> 4;
    const int c_mine = 2 * sl + h;            // MMA (row i) of the step
    const int r_mine = 16 * q + (lane & 15);  // row of that MMA (column j)
    const int i = i0 + c_mine, j = j0 + r_mine;
    const bool active = i < g.m && j < g.n;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;

    MP<L> acc, pacc;
    mp_zero(acc, 1u);
    mp_zero(pacc, 1u);
    int next_b = g.kb;
    for (int k = 0; k < g.l; ++k) {
      const int s = k % NS, b = k % TB;
      mbar_wait(&tfull_bar[b], (uint32_t)((k / TB) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint8_t* st = stage(s);
      const int32_t* s_ae = reinterpret_cast<const int32_t*>(st + CF::OFF_E);
      const uint32_t* s_as = reinterpret_cast<const uint32_t*>(s_ae + IT);
      const int32_t* s_be = reinterpret_cast<const int32_t*>(s_as + IT);
      const uint32_t* s_bs = reinterpret_cast<const uint32_t*>(s_be + JT);
      const int32_t ea = s_ae[c_mine], eb = s_be[r_mine];
      const uint32_t sgn = s_as[c_mine] ^ s_bs[r_mine];
      // Short combine: conv columns t >= C0 = 16(L/4 - 1) give the limbs L-4 .. 2L-1 of
      // T = P - E with 0 <= E < 2^(32(L-4)+16) (the skipped columns), so the guard limb
      // estimate is low by at most a carry.  Like mp_mul_g's short product: decide the
      // rounding from T unless the guard limb is within reach of a boundary; then the
      // whole warp re-reads all columns and combines the exact product.
      constexpr int C0 = 4 * (L - 4);
      uint32_t P[2 * L];
      const uint32_t col0 = tbase + lane_base + (uint32_t)((b * SPB + sl) * NC);
      auto combine = [&](int c16_begin) {
        uint32_t carry = 0;
#pragma unroll
        for (int c16 = 0; c16 < NC / 16; ++c16) {
          if (c16 < c16_begin) continue;
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(col0 + 16 * c16));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            // limb = D[4q] + D[4q+1] 2^8 + D[4q+2] 2^16 + D[4q+3] 2^24 + carry   (exact)
            const uint32_t x = v[4 * qq + 1] * 256u + v[4 * qq] + carry;  // < 2^32
            const uint32_t y = v[4 * qq + 3] * 256u + v[4 * qq + 2];      // < 2^31
            const uint64_t w = (uint64_t)y * 65536u + x;
            P[4 * c16 + qq] = (uint32_t)w;
            carry = (uint32_t)(w >> 32);
          }
        }
      };
      combine(C0 / 16);
      const bool nonzero = ea != EXP_ZERO && eb != EXP_ZERO;
      uint32_t s1 = (P[2 * L - 1] >> 31) ^ 1u;
      uint32_t gd = __funnelshift_l(P[L - 2], P[L - 1], s1);
      constexpr uint32_t MARGIN = 64u;
      const bool decided = (g.sh == 0) ? (gd < 0x80000000u - MARGIN || (gd > 0x80000000u && gd < 0xFFFFFFFFu - MARGIN))
                                       : (gd != 0u && gd < 0xFFFFFFFFu - MARGIN);
      uint32_t stk = 1u;  // decided: the rest below the guard limb is nonzero or irrelevant
      if (__any_sync(0xFFFFFFFFu, active && nonzero && !decided)) {
        combine(0);
        s1 = (P[2 * L - 1] >> 31) ^ 1u;
        gd = __funnelshift_l(P[L - 2], P[L - 1], s1);
        stk = P[L - 2] << s1;
#pragma unroll
        for (int kk = 0; kk < L - 2; ++kk) stk |= P[kk];
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tempty_bar[b]);
        mbar_arrive(&sempty_bar[s]);
      }
      if (active) {
        MP<L> t;
        if (!nonzero) {
          mp_zero(t, sgn);
        } else {
          t.s = sgn;
          int32_t e = ea + eb - (int32_t)s1;
#pragma unroll
          for (int kk = 0; kk < L; ++kk) t.m[kk] = __funnelshift_l(P[L + kk - 1], P[L + kk], s1);
          round_p<L>(t.m, gd, stk, g.sh, e);
          t.e = e;
        }
        if (k == next_b) {  // Block k-tile boundary: C = RN(C + P), fresh P
          mp_add<L>(acc, pacc, 0u, g.sh, acc);
          mp_zero(pacc, 1u);
          next_b += g.kb;
        }
        mp_add<L>(pacc, t, 0u, g.sh, pacc);
      }
    }
    if (active) {
      MP<L> res;
      mp_add<L>(acc, pacc, 0u, g.sh, res);
      uint32_t* cr = C + ((int64_t)i * g.ldc + j) * S;
      if (g.sub_from_c) {  // LU Schur update: A22 = RN(A22 - prod) (blocklu.hpp:138-141)
        MP<L> old;
        load_rec<L>(cr, old);
        mp_add<L>(old, res, 1u, g.sh, res);
      }
      if (exp_out_of_range(res.e)) atomicOr(g.err, ERR_EXP_RANGE);
      store_rec<L>(cr, res);
    }
  } else if (warp < EPI_WARPS + CF::PW) {
    // ================= producers =================
    constexpr int PT = CF::PW * 32;
    const int ptid = tid - EPI_WARPS * 32;
    const int nvalid = (g.n - j0 < JT ? g.n - j0 : JT) * (S / 4);  // valid 16-byte chunks of a B row
    auto fetch_raw = [&](int k) {
      uint8_t* raw = raw0 + (size_t)(k % CF::NR) * CF::RAW;
      const uint32_t* src = B + ((int64_t)k * g.ldb + j0) * S;
      for (int x = ptid; x < JT * S / 4; x += PT) {
        const bool ok = x < nvalid;
        cp16(raw + 16 * x, ok ? src + 4 * x : B, ok ? 16 : 0);
      }
      for (int x = ptid; x < IT * S / 4; x += PT) {
        const int c = x / (S / 4), w = x - c * (S / 4);
        const bool ok = i0 + c < g.m;
        cp16(raw + 4 * S * JT + 16 * x, ok ? A + ((int64_t)(i0 + c) * g.lda + k) * S + 4 * w : A, ok ? 16 : 0);
      }
    };
#pragma unroll
    for (int d = 0; d < CF::D; ++d) {
      if (d < g.l) fetch_raw(d);
      cp_commit();
    }
    for (int k = 0; k < g.l; ++k) {
      if (k + CF::D < g.l) fetch_raw(k + CF::D);
      cp_commit();
      cp_wait<CF::D>();
      named_sync(1, PT);  // raw(k) of every producer thread has landed
      const int s = k % NS;
      mbar_wait(&sempty_bar[s], (uint32_t)(((k / NS) & 1) ^ 1));
      uint8_t* st = stage(s);
      const uint8_t* raw = raw0 + (size_t)(k % CF::NR) * CF::RAW;
      const uint32_t* rawB = reinterpret_cast<const uint32_t*>(raw);
      const uint32_t* rawA = rawB + S * JT;
      // B_j byte rows, canonical K-major
      for (int x = ptid; x < JT * (KB / 16); x += PT) {
        const int r = x / (KB / 16), ch = x - r * (KB / 16);
        *reinterpret_cast<uint4*>(st + kmaj<L>(r, 16 * ch)) = *reinterpret_cast<const uint4*>(rawB + r * S + 4 * ch);
      }
      int32_t* s_ae = reinterpret_cast<int32_t*>(st + CF::OFF_E);
      uint32_t* s_as = reinterpret_cast<uint32_t*>(s_ae + IT);
      int32_t* s_be = reinterpret_cast<int32_t*>(s_as + IT);
      uint32_t* s_bs = reinterpret_cast<uint32_t*>(s_be + JT);
      for (int x = ptid; x < JT; x += PT) {
        s_be[x] = (int32_t)rawB[x * S + L];
        s_bs[x] = rawB[x * S + L + 1];
      }
      for (int x = ptid; x < IT; x += PT) {
        s_ae[x] = (int32_t)rawA[x * S + L];
        s_as[x] = rawA[x * S + L + 1];
      }
      // reversed mantissas: R[y] = a[2KB-1-y] for KB <= y < 2KB (byte order), zero around
      uint32_t* sR = reinterpret_cast<uint32_t*>(st + CF::OFF_R);
      for (int x = ptid; x < IT * L; x += PT) {
        const int c = x / L, w = x - c * L;
        sR[c * CF::RW + L + w] = __byte_perm(rawA[c * S + L - 1 - w], 0, 0x0123);
      }
      named_sync(1, PT);  // R complete; raw(k) fully consumed
      // Toeplitz rows t, chunk ch: bytes of row t at K offsets 16ch..16ch+15 are
      // a[t - 16ch - x] = R[o + x] with o = 2KB - 1 - t + 16ch.  For fixed (t mod 4, ch)
      // consecutive rows t, t+4 shift the window by one word: one LDS + one SHF per chunk.
      for (int sq = ptid; sq < IT * L; sq += PT) {
        const int c = sq / L, rem = sq - c * L;
        const int tm = rem & 3, ch = rem >> 2;
        const uint32_t* R = sR + c * CF::RW;
        uint8_t* T = st + CF::OFF_T + c * CF::T_BYTES;
        const int t_lo = 16 * ch + tm;
        const int t_hi = (16 * ch + KB + 14 < NC - 1) ? 16 * ch + KB + 14 : NC - 1;
        const int o = 2 * KB - 1 - t_lo + 16 * ch;
        const uint32_t bs = (uint32_t)(o & 3) * 8u;
        int w0 = o >> 2;
        uint32_t r0 = R[w0], r1 = R[w0 + 1], r2 = R[w0 + 2], r3 = R[w0 + 3], r4 = R[w0 + 4];
        uint32_t f0 = __funnelshift_r(r0, r1, bs), f1 = __funnelshift_r(r1, r2, bs);
        uint32_t f2 = __funnelshift_r(r2, r3, bs), f3 = __funnelshift_r(r3, r4, bs);
        *reinterpret_cast<uint4*>(T + kmaj<L>(t_lo, 16 * ch)) = make_uint4(f0, f1, f2, f3);
#pragma unroll 4
        for (int t = t_lo + 4; t <= t_hi; t += 4) {
          --w0;
          const uint32_t rn = R[w0];
          f3 = f2;
          f2 = f1;
          f1 = f0;
          f0 = __funnelshift_r(rn, r0, bs);
          r0 = rn;
          *reinterpret_cast<uint4*>(T + kmaj<L>(t, 16 * ch)) = make_uint4(f0, f1, f2, f3);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full_bar[s]);
    }
    cp_wait<0>();
  } else if (lane == 0) {
    // ================= MMA issuer =================
    constexpr uint32_t idesc = idesc_u8(64, NC);
    for (int k = 0; k < g.l; ++k) {
      const int s = k % NS, b = k % TB;
      mbar_wait(&full_bar[s], (uint32_t)((k / NS) & 1));
      mbar_wait(&tempty_bar[b], (uint32_t)(((k / TB) & 1) ^ 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint8_t* st = stage(s);
      const uint32_t aaddr = smem_u32(st), taddr0 = smem_u32(st + CF::OFF_T);
#pragma unroll 1
      for (int c = 0; c < IT; ++c) {
        const uint32_t dtm = tbase + ((uint32_t)(16 * (c & 1)) << 16) + (uint32_t)((b * SPB + (c >> 1)) * NC);
#pragma unroll
        for (int kc = 0; kc < KB / 32; ++kc) {
          const uint64_t da = sdesc<L>(aaddr + kc * 2 * CF::LBO);
          const uint64_t db = sdesc<L>(taddr0 + c * CF::T_BYTES + kc * 2 * CF::LBO);
          const uint32_t accum = kc > 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtm),
              "l"(da), "l"(db), "r"(idesc), "r"(accum));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&tfull_bar[b])));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

}  // namespace tc

bool gemm_tc_enabled() {
  static const bool on = [] {
    const char* v = getenv("MPGPU_GEMM");
    return v && strcmp(v, "tc") == 0;
  }();
  return on;
}

template <int L>
bool launch_gemm_tc(const GemmArgs& g, cudaStream_t st) {
  using CF = tc::Cfg<L>;
  auto kern = tc::gemm_tc_kernel<L>;
  smem_attr_once((const void*)kern, CF::SMEM);
  constexpr int S = rec_stride(L);
  for (int z0 = 0; z0 < g.batch; z0 += 65535) {  // grid.z limit
    GemmArgs gz = g;
    gz.batch = std::min(65535, g.batch - z0);
    gz.A += (int64_t)z0 * g.strideA * S;
    gz.B += (int64_t)z0 * g.strideB * S;
    gz.C += (int64_t)z0 * g.strideC * S;
    dim3 grid((g.n + CF::JT - 1) / CF::JT, (g.m + CF::IT - 1) / CF::IT, gz.batch);
    kern<<<grid, CF::NT, CF::SMEM, st>>>(gz);
  }
  return true;
}

template bool launch_gemm_tc<8>(const GemmArgs&, cudaStream_t);
template bool launch_gemm_tc<16>(const GemmArgs&, cudaStream_t);
template bool launch_gemm_tc<32>(const GemmArgs&, cudaStream_t);

}  // namespace mpg
