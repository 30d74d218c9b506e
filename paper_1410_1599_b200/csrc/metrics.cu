// metrics.cu -- device-side accuracy metrics used by the benchmark driver
// (SURVEY.md §8f rank 2): the reference evaluates them element by element on the host
// with MPFR; here they run as one elementwise kernel plus a two-pass reduction.
//
//   max_rel_error   matrix.hpp:253-279 -- rel_error (precision.hpp:187-193) at the
//                   reference's precision, zero references skipped and counted,
//                   largest and smallest value
//   solution error  blocklu.hpp:306-333 -- max relative error over the nonzero
//                   components, max absolute deviation over the zero ones
//   one_norm        matrix.hpp:237-251 -- column sums of |a_ij| top to bottom, RN at
//                   the matrix precision, largest column
//
// The reference of max_rel_error is usually held at twice the working precision
// (bench.hpp:120-123), so these kernels also exist for 64 limbs (p <= 2048) and read
// the approximation at its own (smaller) limb count, widened exactly.
#include <cuda_runtime.h>

#include "kernels.h"
#include "mp_arith.cuh"
#if MPG_WIDE
#include "wkern.cuh"
#endif

namespace mpg {
namespace {

constexpr uint32_t SKIP = 2u;  // sign-word flag: element not part of a reduction

template <int L>
__device__ __forceinline__ void load_wide(const uint32_t* __restrict__ r, int la, MP<L>& x) {
  const int off = L - la;
#pragma unroll
  for (int k = 0; k < L; ++k) x.m[k] = (k >= off) ? r[k - off] : 0u;
  x.e = (int32_t)r[la];
  x.s = r[la + 1];
}

template <int L>
__device__ __forceinline__ void store_flag(uint32_t* r, const MP<L>& x, uint32_t flag) {
#pragma unroll
  for (int k = 0; k < L; ++k) r[k] = x.m[k];
  r[L] = (uint32_t)x.e;
  r[L + 1] = x.s | flag;
}

// mode 0 (max_rel_error):  outA = rel_error(approx, ref) or SKIP (zero ref; counted)
// mode 1 (solution error): nonzero ref -> outA = rel_error, outB = SKIP;
//                          zero ref    -> outA = SKIP, outB = RN(|approx - ref|) (counted)
template <int L>
__global__ void rel_error_kernel(const uint32_t* __restrict__ approx, int la, int sa, int64_t lda,
                                 const uint32_t* __restrict__ ref, int64_t ldr, int rows, int cols, int mode,
                                 int sh, uint32_t* __restrict__ outA, uint32_t* __restrict__ outB,
                                 unsigned long long* counter, uint32_t* err) {
  constexpr int S = rec_stride(L);
  const int64_t N = (int64_t)rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / cols, j = t - i * cols;
    MP<L> a, r, d;
    load_wide<L>(approx + (i * lda + j) * sa, la, a);
    load_rec<L>(ref + (i * ldr + j) * S, r);
    mp_add<L>(a, r, 1u, sh, d);  // sub(approx, reference, ctx)
    d.s = 0;                      // abs
    if (r.e == EXP_ZERO) {
      atomicAdd(counter, 1ull);
      store_flag<L>(outA + t * S, r, SKIP);
      if (mode == 1) store_flag<L>(outB + t * S, d, 0u);
      continue;
    }
    r.s = 0;
    MP<L> q;
    mp_div<L>(d, r, sh, q);  // div(abs(d), abs(reference), ctx)
    if (exp_out_of_range(q.e) || exp_out_of_range(d.e)) atomicOr(err, ERR_EXP_RANGE);
    store_flag<L>(outA + t * S, q, 0u);
    if (mode == 1) store_flag<L>(outB + t * S, q, SKIP);
  }
}

// one_norm column sums: out[j] = RN(..RN(|a_0j| + |a_1j|)..)
template <int L>
__global__ void colsum_abs_kernel(const uint32_t* __restrict__ A, int64_t ld, int rows, int cols, int sh,
                                  uint32_t* __restrict__ out, uint32_t* err) {
  constexpr int S = rec_stride(L);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  MP<L> acc, t;
  load_rec<L>(A + (int64_t)j * S, acc);
  acc.s = 0;
  for (int i = 1; i < rows; ++i) {
    load_rec<L>(A + ((int64_t)i * ld + j) * S, t);
    t.s = 0;
    mp_add<L>(acc, t, 0u, sh, acc);
  }
  if (exp_out_of_range(acc.e)) atomicOr(err, ERR_EXP_RANGE);
  store_flag<L>(out + (int64_t)j * S, acc, 0u);
}

// Reduction of nonnegative values with SKIP flags to (max A, min A, max B).  Values
// equal in magnitude are equal (all nonnegative; +0 is the only zero produced), so the
// reference's first-found tie rule does not matter.
template <int L>
__device__ __forceinline__ bool better(const uint32_t* cand, const uint32_t* cur, bool want_max) {
  const bool cs = cand[L + 1] & SKIP, us = cur[L + 1] & SKIP;
  if (cs) return false;
  if (us) return true;
  MP<L> x, y;
  load_rec<L>(cand, x);
  load_rec<L>(cur, y);
  x.s &= 1u;
  y.s &= 1u;
  const int c = mp_cmpabs<L>(x, y);
  return want_max ? c > 0 : c < 0;
}

template <int L>
__device__ __forceinline__ void copy_rec(uint32_t* dst, const uint32_t* src) {
#pragma unroll
  for (int k = 0; k < L + 2; ++k) dst[k] = src[k];
}

constexpr int RT = 64;  // threads per reduction block

template <int L>
__global__ void __launch_bounds__(RT) reduce3_kernel(const uint32_t* __restrict__ inMaxA,
                                                     const uint32_t* __restrict__ inMinA,
                                                     const uint32_t* __restrict__ inMaxB, int64_t N,
                                                     int64_t stride /* words between elements */,
                                                     uint32_t* __restrict__ out /* 3 records per block */) {
  constexpr int S = rec_stride(L);
  extern __shared__ uint32_t sm[];  // 3 * RT records
  uint32_t* smax = sm;
  uint32_t* smin = sm + RT * S;
  uint32_t* sbm = sm + 2 * RT * S;
  const int tid = threadIdx.x;
  uint32_t* mx = smax + tid * S;
  uint32_t* mn = smin + tid * S;
  uint32_t* bm = sbm + tid * S;
  mx[L + 1] = SKIP;
  mn[L + 1] = SKIP;
  bm[L + 1] = SKIP;
  for (int64_t t = blockIdx.x * (int64_t)RT + tid; t < N; t += (int64_t)gridDim.x * RT) {
    const int64_t o = t * stride;
    if (better<L>(inMaxA + o, mx, true)) copy_rec<L>(mx, inMaxA + o);
    if (better<L>(inMinA + o, mn, false)) copy_rec<L>(mn, inMinA + o);
    if (inMaxB && better<L>(inMaxB + o, bm, true)) copy_rec<L>(bm, inMaxB + o);
  }
  __syncthreads();
  for (int w = RT / 2; w > 0; w >>= 1) {
    if (tid < w) {
      if (better<L>(smax + (tid + w) * S, mx, true)) copy_rec<L>(mx, smax + (tid + w) * S);
      if (better<L>(smin + (tid + w) * S, mn, false)) copy_rec<L>(mn, smin + (tid + w) * S);
      if (better<L>(sbm + (tid + w) * S, bm, true)) copy_rec<L>(bm, sbm + (tid + w) * S);
    }
    __syncthreads();
  }
  if (tid == 0) {
    uint32_t* o = out + (int64_t)blockIdx.x * 3 * S;
    copy_rec<L>(o, mx);
    copy_rec<L>(o + S, mn);
    copy_rec<L>(o + 2 * S, bm);
  }
}

}  // namespace

template <int L>
void launch_rel_error(const uint32_t* approx, int la, int64_t lda, const uint32_t* ref, int64_t ldr, int rows,
                      int cols, int mode, int sh, uint32_t* outA, uint32_t* outB, unsigned long long* counter,
                      uint32_t* err, cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled())
      return wmp::launch_rel_error<L / 32>(approx, la, lda, ref, ldr, rows, cols, mode, sh, outA, outB, counter,
                                           err, st);
#endif
  const int64_t N = (int64_t)rows * cols;
  const int nt = 128;
  const int64_t want = (N + nt - 1) / nt;
  const int grid = (int)(want < 148 * 16 ? (want < 1 ? 1 : want) : 148 * 16);
  rel_error_kernel<L><<<grid, nt, 0, st>>>(approx, la, rec_stride(la), lda, ref, ldr, rows, cols, mode, sh, outA,
                                           outB, counter, err);
}

template <int L>
void launch_colsum_abs(const uint32_t* A, int64_t ld, int rows, int cols, int sh, uint32_t* out, uint32_t* err,
                       cudaStream_t st) {
  colsum_abs_kernel<L><<<(cols + 63) / 64, 64, 0, st>>>(A, ld, rows, cols, sh, out, err);
}

template <int L>
void launch_reduce3(const uint32_t* A, const uint32_t* B, int64_t N, uint32_t* out3, uint32_t* scratch,
                    cudaStream_t st) {
  constexpr int S = rec_stride(L);
  const size_t smem = sizeof(uint32_t) * 3 * RT * S;
  smem_attr_once((const void*)reduce3_kernel<L>, (int)smem);
  int64_t want = (N + RT * 8 - 1) / (RT * 8);
  const int g1 = (int)(want < 1 ? 1 : (want > 1024 ? 1024 : want));
  if (g1 == 1) {
    reduce3_kernel<L><<<1, RT, smem, st>>>(A, A, B, N, S, out3);
    return;
  }
  // pass 1: g1 partial (max A, min A, max B) triples; pass 2: one block over them
  reduce3_kernel<L><<<g1, RT, smem, st>>>(A, A, B, N, S, scratch);
  reduce3_kernel<L><<<1, RT, smem, st>>>(scratch, scratch + S, scratch + 2 * S, g1, 3 * S, out3);
}

#define MPG_METRICS_INST(L)                                                                                     \
  template void launch_rel_error<L>(const uint32_t*, int, int64_t, const uint32_t*, int64_t, int, int, int, int, \
                                    uint32_t*, uint32_t*, unsigned long long*, uint32_t*, cudaStream_t);        \
  template void launch_colsum_abs<L>(const uint32_t*, int64_t, int, int, int, uint32_t*, uint32_t*, cudaStream_t); \
  template void launch_reduce3<L>(const uint32_t*, const uint32_t*, int64_t, uint32_t*, uint32_t*, cudaStream_t);
#if MPG_WIDE
MPG_METRICS_INST(64)
MPG_METRICS_INST(128)
MPG_METRICS_INST(256)
MPG_METRICS_INST(288)
#else
MPG_METRICS_INST(1)
MPG_METRICS_INST(2)
MPG_METRICS_INST(4)
MPG_METRICS_INST(8)
MPG_METRICS_INST(16)
MPG_METRICS_INST(32)
#endif

}  // namespace mpg
