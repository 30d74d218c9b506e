// lu.cu -- kernels of the blocked LU (blocklu.hpp:42-146) and its solves
// (blocklu.hpp:215-245).
//
// Panel: the reference factors the K x K diagonal block with lu_inplace
// (blocklu.hpp:42-56) and then the rows below it with trsm_upper_right_inplace
// (blocklu.hpp:73-86).  Per element both apply  a_ij -= RN(a_is * a_sj)  for
// s = p .. j-1 in ascending order and then (below the diagonal) a_ij = RN(a_ij / a_jj),
// which is exactly what a right-looking elimination over the TALL panel does, so
// one step kernel per pivot column d covers both, in parallel over rows and
// columns, bit-exactly.  With partial pivoting (an extension: the reference is
// pivot-free, blocklu.hpp:38-41) the pivot row is swapped in first.
// U12: trsm_unit_lower_inplace (blocklu.hpp:60-69) is replayed as a column sweep
// over s -- per element the same s-ascending order.
#include <cuda_runtime.h>

#include "kernels.h"
#include "mp_arith.cuh"

namespace mpg {

namespace {
constexpr int NT = 256;
inline int blocks_for(int64_t n) {
  int64_t b = (n + NT - 1) / NT;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}
}  // namespace

// One elimination step of pivot column d over a block of LU_RB rows:
//   a_id = RN(a_id / a_dd)                       (blocklu.hpp:49)
//   a_ij = RN(a_ij - RN(a_id * a_dj)), d < j < col_end   (blocklu.hpp:51-52)
// Every row's multiplier is produced inside the CTA that uses it, so one launch
// per column suffices (no grid-wide dependency between rows).
constexpr int LU_RB = 8;
template <int L>
__global__ void __launch_bounds__(NT) lu_col_kernel(uint32_t* a, int64_t n, int64_t d, int64_t row_end,
                                                    int64_t col_end, int sh, int64_t* zp) {
  constexpr int S = rec_stride(L);
  __shared__ __align__(16) uint32_t s_mult[LU_RB * S];
  if (*zp) return;  // a zero pivot was already met: the factorisation has failed
  const int64_t r0 = d + 1 + (int64_t)blockIdx.x * LU_RB;
  if (threadIdx.x < LU_RB) {
    const int64_t i = r0 + threadIdx.x;
    MP<L> piv;
    load_rec<L>(a + (d * n + d) * S, piv);
    if (piv.e == EXP_ZERO) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *zp = d + 1;  // blocklu.hpp:46-47 (1-based)
    } else if (i < row_end) {
      MP<L> x, q;
      load_rec<L>(a + (i * n + d) * S, x);
      mp_div<L>(x, piv, sh, q);
      store_rec<L>(a + (i * n + d) * S, q);
      store_rec<L>(s_mult + threadIdx.x * S, q);
    }
  }
  __syncthreads();
  if (a[(d * n + d) * S + L] == (uint32_t)EXP_ZERO) return;
  const int64_t w = col_end - d - 1;
  for (int64_t t = threadIdx.x; t < LU_RB * w; t += blockDim.x) {
    const int rr = (int)(t / w);
    const int64_t i = r0 + rr, j = d + 1 + t % w;
    if (i >= row_end) continue;
    MP<L> l, u, p, x;
    load_rec<L>(s_mult + rr * S, l);
    load_rec<L>(a + (d * n + j) * S, u);
    mp_mul<L>(l, u, sh, p);
    load_rec<L>(a + (i * n + j) * S, x);
    mp_add<L>(x, p, 1u, sh, x);
    store_rec<L>(a + (i * n + j) * S, x);
  }
}

// trsm_unit_lower step s: rows (s, p_end), cols [c0, c0 + w)
template <int L>
__global__ void trsm_l_kernel(uint32_t* a, int64_t n, int64_t s, int64_t p_end, int64_t c0, int64_t w, int sh) {
  constexpr int S = rec_stride(L);
  const int64_t total = (p_end - s - 1) * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = s + 1 + t / w, j = c0 + t % w;
    MP<L> l, u, p, x, r;
    load_rec<L>(a + (i * n + s) * S, l);
    load_rec<L>(a + (s * n + j) * S, u);
    mp_mul<L>(l, u, sh, p);
    load_rec<L>(a + (i * n + j) * S, x);
    mp_add<L>(x, p, 1u, sh, r);
    store_rec<L>(a + (i * n + j) * S, r);
  }
}

// pivot search (first maximal |a_id| over rows [d, row_end)) + full-row swap
template <int L>
__global__ void __launch_bounds__(NT) pivot_kernel(uint32_t* a, int64_t n, int64_t d, int64_t row_end,
                                                   int64_t* piv, int64_t* zp) {
  constexpr int S = rec_stride(L);
  __shared__ int64_t s_idx[NT];
  __shared__ int64_t s_best;
  if (*zp) return;
  int64_t best = -1;
  MP<L> bv;
  mp_zero(bv);
  for (int64_t i = d + threadIdx.x; i < row_end; i += blockDim.x) {
    MP<L> x;
    load_rec<L>(a + (i * n + d) * S, x);
    if (best < 0 || mp_cmpabs<L>(x, bv) > 0) {
      bv = x;
      best = i;
    }
  }
  s_idx[threadIdx.x] = best;
  __syncthreads();
  // tree reduction: larger |a_id| wins, ties go to the lower row index
  for (int half = NT / 2; half > 0; half >>= 1) {
    if (threadIdx.x < half) {
      const int64_t i0 = s_idx[threadIdx.x], i1 = s_idx[threadIdx.x + half];
      if (i1 >= 0) {
        bool take = i0 < 0;
        if (!take) {
          MP<L> x0, x1;
          load_rec<L>(a + (i0 * n + d) * S, x0);
          load_rec<L>(a + (i1 * n + d) * S, x1);
          const int c = mp_cmpabs<L>(x1, x0);
          take = c > 0 || (c == 0 && i1 < i0);
        }
        if (take) s_idx[threadIdx.x] = i1;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s_best = s_idx[0];
    piv[d] = s_idx[0];
  }
  __syncthreads();
  const int64_t r = s_best;
  if (r != d) {
    constexpr int CH = S / 4;
    for (int64_t t = threadIdx.x; t < n * CH; t += blockDim.x) {
      const int64_t j = t / CH, w = t % CH;
      uint4* p = reinterpret_cast<uint4*>(a + (d * n + j) * S + 4 * w);
      uint4* q = reinterpret_cast<uint4*>(a + (r * n + j) * S + 4 * w);
      const uint4 tmp = *p;
      *p = *q;
      *q = tmp;
    }
  }
}

// Ly = Pb (column sweep, exact), Ux = y (exact row replay, s ascending as
// blocklu.hpp:235-238); one CTA.
template <int L>
__global__ void __launch_bounds__(NT) lu_solve_kernel(const uint32_t* f, int64_t n, const int64_t* piv,
                                                      const uint32_t* b, uint32_t* x, uint32_t* y,
                                                      uint32_t* tmp, int sh, uint32_t* err, int64_t* zp,
                                                      int exact) {
  constexpr int S = rec_stride(L);
  constexpr int CH = S / 4;
  // y = b
  for (int64_t t = threadIdx.x; t < n * CH; t += blockDim.x)
    reinterpret_cast<uint4*>(y)[t] = reinterpret_cast<const uint4*>(b)[t];
  __syncthreads();
  if (piv && threadIdx.x == 0) {
    for (int64_t d = 0; d < n; ++d) {
      const int64_t r = piv[d];
      if (r != d)
        for (int w = 0; w < CH; ++w) {
          uint4* p = reinterpret_cast<uint4*>(y + d * S) + w;
          uint4* q = reinterpret_cast<uint4*>(y + r * S) + w;
          const uint4 t = *p;
          *p = *q;
          *q = t;
        }
    }
  }
  __syncthreads();
  for (int64_t s = 0; s < n; ++s) {
    MP<L> ys;
    load_rec<L>(y + s * S, ys);
    for (int64_t i = s + 1 + threadIdx.x; i < n; i += blockDim.x) {
      MP<L> l, p, acc, r;
      load_rec<L>(f + (i * n + s) * S, l);
      mp_mul<L>(l, ys, sh, p);
      load_rec<L>(y + i * S, acc);
      mp_add<L>(acc, p, 1u, sh, r);
      store_rec<L>(y + i * S, r);
    }
    __syncthreads();
  }
  if (!exact) {
    // column-oriented back substitution (s descending per row): one division and
    // one parallel rank-1 update per step -- within the LU tolerance, not the
    // reference's summation order
    for (int64_t ii = n - 1; ii >= 0; --ii) {
      __shared__ __align__(16) uint32_t s_x[rec_stride(L)];
      if (threadIdx.x == 0) {
        MP<L> acc, d, q;
        load_rec<L>(y + ii * S, acc);
        load_rec<L>(f + (ii * n + ii) * S, d);
        if (d.e == EXP_ZERO) {
          if (*zp == 0) *zp = ii + 1;
          mp_zero(q);
        } else {
          mp_div<L>(acc, d, sh, q);
        }
        if (exp_out_of_range(q.e)) atomicOr(err, ERR_EXP_RANGE);
        store_rec<L>(x + ii * S, q);
        store_rec<L>(s_x, q);
      }
      __syncthreads();
      if (*zp) return;
      MP<L> xs;
      load_rec<L>(s_x, xs);
      for (int64_t i = threadIdx.x; i < ii; i += blockDim.x) {
        MP<L> u, p, acc;
        load_rec<L>(f + (i * n + ii) * S, u);
        mp_mul<L>(u, xs, sh, p);
        load_rec<L>(y + i * S, acc);
        mp_add<L>(acc, p, 1u, sh, acc);
        store_rec<L>(y + i * S, acc);
      }
      __syncthreads();
    }
    return;
  }
  for (int64_t ii = n - 1; ii >= 0; --ii) {
    for (int64_t s = ii + 1 + threadIdx.x; s < n; s += blockDim.x) {
      MP<L> u, xs, p;
      load_rec<L>(f + (ii * n + s) * S, u);
      load_rec<L>(x + s * S, xs);
      mp_mul<L>(u, xs, sh, p);
      store_rec<L>(tmp + s * S, p);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      MP<L> acc;
      load_rec<L>(y + ii * S, acc);
      for (int64_t s = ii + 1; s < n; ++s) {
        MP<L> p;
        load_rec<L>(tmp + s * S, p);
        mp_add<L>(acc, p, 1u, sh, acc);
      }
      MP<L> d, q;
      load_rec<L>(f + (ii * n + ii) * S, d);
      if (d.e == EXP_ZERO) {
        if (*zp == 0) *zp = ii + 1;
        mp_zero(q);
      } else {
        mp_div<L>(acc, d, sh, q);
      }
      if (exp_out_of_range(q.e)) atomicOr(err, ERR_EXP_RANGE);
      store_rec<L>(x + ii * S, q);
    }
    __syncthreads();
    if (*zp) return;
  }
}

template <int L>
void launch_lu_step(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t col_end, int sh, uint32_t* err,
                    cudaStream_t st) {
  // zero-pivot flag lives right after the error word (see capi.cu)
  int64_t* zp = reinterpret_cast<int64_t*>(err + 2);
  const int64_t rows = row_end - d - 1;
  const int blocks = (int)((rows + LU_RB - 1) / LU_RB);
  lu_col_kernel<L><<<blocks < 1 ? 1 : blocks, NT, 0, st>>>(a, n, d, row_end, col_end, sh, zp);
}

template <int L>
void launch_pivot(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t* piv_dev, int64_t* zp,
                  cudaStream_t st) {
  pivot_kernel<L><<<1, NT, 0, st>>>(a, n, d, row_end, piv_dev, zp);
}

template <int L>
void launch_trsm_l_step(uint32_t* a, int64_t n, int64_t s, int64_t p_end, int64_t c0, int64_t w, int sh,
                        uint32_t* err, cudaStream_t st) {
  (void)err;
  const int64_t total = (p_end - s - 1) * w;
  if (total > 0) trsm_l_kernel<L><<<blocks_for(total), NT, 0, st>>>(a, n, s, p_end, c0, w, sh);
}

template <int L>
void launch_lu_solve(const uint32_t* f, int64_t n, const int64_t* piv_dev, const uint32_t* b, uint32_t* x,
                     uint32_t* scratch, int sh, uint32_t* err, int64_t* zp, int exact, cudaStream_t st) {
  constexpr int S = rec_stride(L);
  lu_solve_kernel<L><<<1, NT, 0, st>>>(f, n, piv_dev, b, x, scratch, scratch + n * S, sh, err, zp, exact);
}

#define MPG_LU_INST(L)                                                                                      \
  template void launch_lu_step<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int, uint32_t*, cudaStream_t); \
  template void launch_pivot<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t*, int64_t*, cudaStream_t);        \
  template void launch_trsm_l_step<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int, uint32_t*,   \
                                      cudaStream_t);                                                            \
  template void launch_lu_solve<L>(const uint32_t*, int64_t, const int64_t*, const uint32_t*, uint32_t*,        \
                                   uint32_t*, int, uint32_t*, int64_t*, int, cudaStream_t);
MPG_LU_INST(1)
MPG_LU_INST(2)
MPG_LU_INST(4)
MPG_LU_INST(8)
MPG_LU_INST(16)
MPG_LU_INST(32)

}  // namespace mpg
