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
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "mp_arith.cuh"
#if MPG_WIDE
#include "wkern.cuh"
#endif

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

__device__ __forceinline__ uint64_t mag_key(uint32_t e, uint32_t top) {
  return e == (uint32_t)EXP_ZERO ? 0ull : (((uint64_t)(e ^ 0x80000000u)) << 32) | top;
}
// (key, first index, count) of the rows whose compact magnitude key is maximal;
// count 0 marks an empty candidate
__device__ __forceinline__ void piv_combine(uint64_t& k, int64_t& i, int& c, uint64_t k2, int64_t i2, int c2) {
  if (c2 == 0) return;
  if (c == 0 || k2 > k) {
    k = k2;
    i = i2;
    c = c2;
  } else if (k2 == k) {
    i = i2 < i ? i2 : i;
    c += c2;
  }
}

template <int L>
__global__ void __launch_bounds__(NT) lu_col_kernel(uint32_t* a, int64_t n, int64_t d, int64_t row_end,
                                                    int64_t col_end, int sh, int64_t* zp, uint64_t* ck,
                                                    int64_t* ci, int* cc) {
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
  if (ck != nullptr && d + 1 < col_end) {
    // pivot candidates of column d+1 over this CTA's rows (it just updated them), so
    // the next pivot search reduces one record per CTA instead of scanning the column
    __syncthreads();
    if (threadIdx.x < 32) {
      const int64_t i = r0 + threadIdx.x;
      uint64_t k = 0;
      int64_t idx = INT64_MAX;
      int c = 0;
      if (threadIdx.x < LU_RB && i < row_end) {
        const uint32_t* r = a + (i * n + d + 1) * S;
        k = mag_key(r[L], r[L - 1]);
        idx = i;
        c = 1;
      }
#pragma unroll
      for (int o = LU_RB / 2; o > 0; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(0xffffffffu, k, o);
        const int64_t i2 = __shfl_xor_sync(0xffffffffu, idx, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, c, o);
        piv_combine(k, idx, c, k2, i2, c2);
      }
      if (threadIdx.x == 0) {
        ck[blockIdx.x] = k;
        ci[blockIdx.x] = idx;
        cc[blockIdx.x] = c;
      }
    }
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

// pivot search (first maximal |a_id| over rows [d, row_end)) + swap of rows d and the
// pivot over the panel columns [c0, c1) (the other columns are swapped once per panel by
// laswp_kernel -- row swaps commute with work on columns they do not touch).  The
// compact magnitude key (biased exponent : top limb) is reduced with its first index
// and its multiplicity, from the previous step's per-CTA candidates when given
// (ncand > 0) or by scanning the column; only when several rows share the maximal key
// does a full MP comparison (first maximal row wins) run.
constexpr int PIV_NT = 1024;
template <int L>
__global__ void __launch_bounds__(PIV_NT) pivot_kernel(uint32_t* a, int64_t n, int64_t d, int64_t row_end,
                                                       int64_t* piv, int64_t* zp, const uint64_t* ck,
                                                       const int64_t* ci, const int* cc, int64_t ncand, int64_t c0,
                                                       int64_t c1) {
  constexpr int S = rec_stride(L);
  __shared__ uint64_t s_key[PIV_NT / 32];
  __shared__ int64_t s_idx[PIV_NT / 32];
  __shared__ int s_cnt[PIV_NT / 32];
  __shared__ int64_t s_best;
  __shared__ int s_ties;
  __shared__ uint64_t s_kstar;
  if (*zp) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint64_t bk = 0;
  int64_t bi = INT64_MAX;
  int bc = 0;
  if (ncand > 0) {
    // written by the previous step's CTAs over rows [d, row_end) of column d
    for (int64_t t = tid; t < ncand; t += PIV_NT) piv_combine(bk, bi, bc, ck[t], ci[t], cc[t]);
  } else {
    for (int64_t i = d + tid; i < row_end; i += PIV_NT) {
      const uint32_t* r = a + (i * n + d) * S;
      piv_combine(bk, bi, bc, mag_key(r[L], r[L - 1]), i, 1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
    const int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
    piv_combine(bk, bi, bc, k2, i2, c2);
  }
  if (lane == 0) {
    s_key[wid] = bk;
    s_idx[wid] = bi;
    s_cnt[wid] = bc;
  }
  __syncthreads();
  if (wid == 0) {
    bk = s_key[lane];
    bi = s_idx[lane];
    bc = s_cnt[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
      piv_combine(bk, bi, bc, k2, i2, c2);
    }
    if (lane == 0) {
      s_best = bi;
      s_ties = bc;
      s_kstar = bk;
    }
  }
  __syncthreads();
  if (s_ties > 1 && tid == 0) {  // rare: full comparison among the tied rows
    const uint64_t kstar = s_kstar;
    int64_t r = -1;
    MP<L> rv;
    mp_zero(rv);
    for (int64_t i = d; i < row_end; ++i) {
      const uint32_t* q = a + (i * n + d) * S;
      if (mag_key(q[L], q[L - 1]) != kstar) continue;
      MP<L> x;
      load_rec<L>(q, x);
      if (r < 0 || mp_cmpabs<L>(x, rv) > 0) {
        rv = x;
        r = i;
      }
    }
    s_best = r;
  }
  __syncthreads();
  const int64_t r = s_best;
  if (tid == 0) piv[d] = r;
  if (r != d) {
    constexpr int CH = S / 4;
    for (int64_t t = tid; t < (c1 - c0) * CH; t += PIV_NT) {
      const int64_t j = c0 + t / CH, w = t % CH;
      uint4* p = reinterpret_cast<uint4*>(a + (d * n + j) * S + 4 * w);
      uint4* q = reinterpret_cast<uint4*>(a + (r * n + j) * S + 4 * w);
      const uint4 tmp = *p;
      *p = *q;
      *q = tmp;
    }
  }
}

// the panel's row interchanges d = p .. p+k-1 (in order) on every column outside
// [p, p+k) -- LAPACK laswp; each 16-byte chunk of a column is independent
template <int L>
__global__ void laswp_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, const int64_t* piv, const int64_t* zp) {
  constexpr int S = rec_stride(L), CH = S / 4;
  if (*zp) return;
  const int64_t total = (n - k) * CH;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = t / CH, w = t - jj * CH;
    const int64_t j = jj < p ? jj : jj + k;
    for (int64_t d = p; d < p + k; ++d) {
      const int64_t r = piv[d];
      if (r == d) continue;
      uint4* x = reinterpret_cast<uint4*>(a + (d * n + j) * S + 4 * w);
      uint4* y = reinterpret_cast<uint4*>(a + (r * n + j) * S + 4 * w);
      const uint4 tmp = *x;
      *x = *y;
      *y = tmp;
    }
  }
}

// trsm_unit_lower over a whole panel in one launch (blocklu.hpp:60-69): each CTA owns
// TRSM_TC columns of U12 and sweeps s = p .. p+k-2 with a barrier per step; per
// element the updates arrive in s-ascending order, as in the reference.
constexpr int TRSM_TC = 4;
template <int L>
__global__ void __launch_bounds__(NT) trsm_l_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0,
                                                          int64_t w, int sh) {
  constexpr int S = rec_stride(L);
  const int64_t j0 = c0 + (int64_t)blockIdx.x * TRSM_TC;
  const int tc = (int)(c0 + w - j0 < TRSM_TC ? c0 + w - j0 : TRSM_TC);
  for (int64_t s = p; s + 1 < p + k; ++s) {
    const int64_t rows = p + k - s - 1;
    for (int64_t t = threadIdx.x; t < rows * tc; t += blockDim.x) {
      const int64_t i = s + 1 + t / tc, j = j0 + t % tc;
      MP<L> l, u, pr, x;
      load_rec<L>(a + (i * n + s) * S, l);
      load_rec<L>(a + (s * n + j) * S, u);
      mp_mul<L>(l, u, sh, pr);
      load_rec<L>(a + (i * n + j) * S, x);
      mp_add<L>(x, pr, 1u, sh, x);
      store_rec<L>(a + (i * n + j) * S, x);
    }
    __syncthreads();
  }
}

// The same sweep with the CTA's U12 tile (k rows x tc columns) resident in shared memory:
// per step s only the multipliers l_is come from memory (loaded one step ahead), the
// pivot row and the updated elements stay on chip -- the sweep is a chain of k dependent
// multiply-adds per column, so its per-step latency is the cost.
template <int L>
__global__ void __launch_bounds__(NT) trsm_l_smem_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0,
                                                         int64_t w, int sh, int tcw) {
  constexpr int S = rec_stride(L), CH = S / 4;
  extern __shared__ __align__(16) uint32_t s_tile[];
  const int64_t j0 = c0 + (int64_t)blockIdx.x * tcw;
  const int tc = (int)(c0 + w - j0 < tcw ? c0 + w - j0 : tcw);
  const int tid = threadIdx.x;
  auto T = [&](int64_t r, int jj) { return s_tile + ((r - p) * tcw + jj) * S; };
  for (int64_t t = tid; t < k * tc * CH; t += NT) {
    const int64_t r = t / (tc * CH);
    const int rem = (int)(t - r * tc * CH), jj = rem / CH, q = rem - jj * CH;
    reinterpret_cast<uint4*>(T(p + r, jj))[q] = reinterpret_cast<const uint4*>(a + ((p + r) * n + j0 + jj) * S)[q];
  }
  // this thread's first element of step s: row s + 1 + tid / tc; its multiplier one step ahead
  MP<L> lnext;
  auto first_l = [&](int64_t s, MP<L>& l) {
    const int64_t i = s + 1 + tid / tc;
    if (s + 1 < p + k && i < p + k) load_rec<L>(a + (i * n + s) * S, l);
  };
  first_l(p, lnext);
  __syncthreads();
  for (int64_t s = p; s + 1 < p + k; ++s) {
    const int64_t rows = p + k - s - 1;
    MP<L> lcur = lnext;
    first_l(s + 1, lnext);
    for (int64_t t = tid; t < rows * tc; t += NT) {
      const int64_t i = s + 1 + t / tc;
      const int jj = (int)(t % tc);
      MP<L> l, u, pr, x;
      if (t == tid)
        l = lcur;
      else
        load_rec<L>(a + (i * n + s) * S, l);
      load_rec<L>(T(s, jj), u);
      mp_mul<L>(l, u, sh, pr);
      uint32_t* xr = T(i, jj);
      load_rec<L>(xr, x);
      mp_add<L>(x, pr, 1u, sh, x);
      store_rec<L>(xr, x);
    }
    __syncthreads();
  }
  for (int64_t t = tid; t < (k - 1) * tc * CH; t += NT) {  // row p is unchanged
    const int64_t r = 1 + t / (tc * CH);
    const int rem = (int)(t - (r - 1) * tc * CH), jj = rem / CH, q = rem - jj * CH;
    reinterpret_cast<uint4*>(a + ((p + r) * n + j0 + jj) * S)[q] = reinterpret_cast<const uint4*>(T(p + r, jj))[q];
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
  // one CTA per right-hand side (blockIdx.x): its b, x and 2n scratch records
  b += (int64_t)blockIdx.x * n * S;
  x += (int64_t)blockIdx.x * n * S;
  y += (int64_t)blockIdx.x * 2 * n * S;
  tmp = y + n * S;
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

// ---------------------------------------------------------------------------
// Whole-panel factorisation in ONE cooperative launch: for every pivot column d of
// the panel [p, p+k) (rows [p, row_end)):
//   (pivoting) per-CTA best magnitude key -> grid.sync -> every CTA reduces the same
//   candidates (identical result) -> row swap split over CTAs -> grid.sync;
//   multipliers (one MP division per row) and the rank-1 update of the panel
//   columns for the CTA's own rows -> grid.sync.
// Same per-element operation sequence as the per-column kernels (and the
// reference), without a kernel launch per column.
// ---------------------------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(NT) lu_panel_coop_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k,
                                                           int64_t row_end, int pivoting, int64_t* piv,
                                                           int64_t* zp, int sh, uint64_t* cand_key,
                                                           int64_t* cand_idx, uint64_t* cand_cnt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int S = rec_stride(L);
  extern __shared__ __align__(16) uint32_t s_mult[];
  __shared__ uint64_t s_wk[NT / 32];
  __shared__ int64_t s_wi[NT / 32];
  __shared__ int s_wc[NT / 32];
  __shared__ int64_t s_piv;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rows_all = row_end - p;
  const int64_t chunk = (rows_all + gridDim.x - 1) / gridDim.x;
  const int64_t lo = p + (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(row_end, lo + chunk);
  // pivot candidates of column d over this CTA's rows [max(d, lo), hi): (compact key,
  // first row, multiplicity), block-reduced, one record per CTA
  auto candidates = [&](int64_t col, int64_t from) {
    uint64_t bk = 0;
    int64_t bi = INT64_MAX;
    int bc = 0;
    for (int64_t i = max(from, lo) + tid; i < hi; i += NT) {
      const uint32_t* r = a + (i * n + col) * S;
      piv_combine(bk, bi, bc, mag_key(r[L], r[L - 1]), i, 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
      piv_combine(bk, bi, bc, k2, i2, c2);
    }
    if (lane == 0) {
      s_wk[wid] = bk;
      s_wi[wid] = bi;
      s_wc[wid] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NT / 32; ++w) piv_combine(bk, bi, bc, s_wk[w], s_wi[w], s_wc[w]);
      cand_key[blockIdx.x] = bk;
      cand_idx[blockIdx.x] = bi;
      cand_cnt[blockIdx.x] = (uint64_t)bc;
    }
    __syncthreads();
  };
  if (pivoting) {
    candidates(p, p);
    grid.sync();
  }
  for (int64_t d = p; d < p + k; ++d) {
    if (pivoting) {
      // every CTA reduces the same candidate list -> the same pivot
      uint64_t gk = 0;
      int64_t gi = INT64_MAX;
      int gc = 0;
      for (unsigned b = tid; b < gridDim.x; b += NT) piv_combine(gk, gi, gc, cand_key[b], cand_idx[b], (int)cand_cnt[b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(0xffffffffu, gk, o);
        const int64_t i2 = __shfl_xor_sync(0xffffffffu, gi, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, gc, o);
        piv_combine(gk, gi, gc, k2, i2, c2);
      }
      if (lane == 0) {
        s_wk[wid] = gk;
        s_wi[wid] = gi;
        s_wc[wid] = gc;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < NT / 32; ++w) piv_combine(gk, gi, gc, s_wk[w], s_wi[w], s_wc[w]);
        if (gc > 1) {  // rows sharing the winning compact key: a full comparison decides (rare)
          MP<L> rv, x;
          int64_t r = -1;
          for (int64_t i = d; i < row_end; ++i) {
            const uint32_t* q = a + (i * n + d) * S;
            if (mag_key(q[L], q[L - 1]) != gk) continue;
            load_rec<L>(q, x);
            if (r < 0 || mp_cmpabs<L>(x, rv) > 0) {
              rv = x;
              r = i;
            }
          }
          gi = r;
        }
        s_piv = gi;
      }
      __syncthreads();
      const int64_t r = s_piv;
      if (blockIdx.x == 0) {
        if (tid == 0) piv[d] = r;
        if (r != d) {  // swap rows d, r over the panel columns (laswp does the rest)
          constexpr int CH = S / 4;
          for (int64_t t = tid; t < k * CH; t += NT) {
            const int64_t j = p + t / CH, w = t % CH;
            uint4* pp = reinterpret_cast<uint4*>(a + (d * n + j) * S + 4 * w);
            uint4* qq = reinterpret_cast<uint4*>(a + (r * n + j) * S + 4 * w);
            const uint4 tmp = *pp;
            *pp = *qq;
            *qq = tmp;
          }
        }
      }
      grid.sync();
    }
    // zero pivot: every CTA sees the same a_dd and stops (blocklu.hpp:46-47)
    if (a[(d * n + d) * S + L] == (uint32_t)EXP_ZERO) {
      if (blockIdx.x == 0 && tid == 0) *zp = d + 1;
      return;
    }
    // multipliers and rank-1 update for this CTA's rows in (d, row_end)
    const int64_t r0 = max(d + 1, lo);
    const int64_t nr = hi - r0;
    if (nr > 0) {
      for (int64_t t = tid; t < nr; t += NT) {
        MP<L> piv_v, x, q;
        load_rec<L>(a + (d * n + d) * S, piv_v);
        load_rec<L>(a + ((r0 + t) * n + d) * S, x);
        mp_div<L>(x, piv_v, sh, q);
        store_rec<L>(a + ((r0 + t) * n + d) * S, q);
        store_rec<L>(s_mult + t * S, q);
      }
      __syncthreads();
      const int64_t w = p + k - d - 1;
      for (int64_t t = tid; t < nr * w; t += NT) {
        const int64_t rr = t / w, j = d + 1 + t % w;
        MP<L> l, u, pr, x;
        load_rec<L>(s_mult + rr * S, l);
        load_rec<L>(a + (d * n + j) * S, u);
        mp_mul<L>(l, u, sh, pr);
        load_rec<L>(a + ((r0 + rr) * n + j) * S, x);
        mp_add<L>(x, pr, 1u, sh, x);
        store_rec<L>(a + ((r0 + rr) * n + j) * S, x);
      }
    }
    if (pivoting && d + 1 < p + k) {
      __syncthreads();  // this CTA's updates of column d+1 are visible to its threads
      candidates(d + 1, d + 1);
    }
    grid.sync();
  }
}

// Pivoting variant with ONE grid barrier per column: the row interchanges of the panel
// are kept as a logical -> physical row table in every CTA's shared memory (identical
// in all CTAs, which all reduce the same candidates), so choosing the pivot needs no
// data movement and no barrier; the panel columns are permuted physically once, after
// the panel (laswp_panel_kernel).  Per column: every CTA reduces the candidates of the
// previous step -> same pivot r -> swaps table entries d, r; multipliers and rank-1
// update of the CTA's logical rows (physical slots via the table); candidates of the
// next column; grid.sync.  Same per-element operation sequence as the other kernels.
template <int L>
__global__ void __launch_bounds__(NT) lu_panel_perm_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k,
                                                           int64_t row_end, int64_t* piv, int64_t* zp, int sh,
                                                           uint64_t* cand_key, int64_t* cand_idx, uint64_t* cand_cnt,
                                                           int64_t chunk) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int S = rec_stride(L);
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* s_mult = s_dyn;                                      // chunk records
  uint32_t* s_urow = s_dyn + chunk * S;                          // the pivot row right of the pivot: k records
  int* s_perm = reinterpret_cast<int*>(s_urow + k * S);          // logical row - p -> physical row - p
  __shared__ uint64_t s_wk[NT / 32];
  __shared__ int64_t s_wi[NT / 32];
  __shared__ int s_wc[NT / 32];
  __shared__ int64_t s_piv;
  __shared__ uint64_t s_gk;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rows_all = row_end - p;
  const int64_t lo = p + (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(row_end, lo + chunk);
  for (int64_t t = tid; t < rows_all; t += NT) s_perm[t] = (int)t;
  __syncthreads();
  auto phys = [&](int64_t i) -> int64_t { return p + s_perm[i - p]; };
  // the CTA's best (key, first row, count) -> cand_*[blockIdx.x]
  auto publish = [&](uint64_t bk, int64_t bi, int bc) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
      piv_combine(bk, bi, bc, k2, i2, c2);
    }
    if (lane == 0) {
      s_wk[wid] = bk;
      s_wi[wid] = bi;
      s_wc[wid] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NT / 32; ++w) piv_combine(bk, bi, bc, s_wk[w], s_wi[w], s_wc[w]);
      cand_key[blockIdx.x] = bk;
      cand_idx[blockIdx.x] = bi;
      cand_cnt[blockIdx.x] = (uint64_t)bc;
    }
    __syncthreads();
  };
  auto candidates = [&](int64_t col, int64_t from) {
    uint64_t bk = 0;
    int64_t bi = INT64_MAX;
    int bc = 0;
    for (int64_t i = max(from, lo) + tid; i < hi; i += NT) {
      const uint32_t* r = a + (phys(i) * n + col) * S;
      piv_combine(bk, bi, bc, mag_key(r[L], r[L - 1]), i, 1);
    }
    publish(bk, bi, bc);
  };
  candidates(p, p);
  grid.sync();
  for (int64_t d = p; d < p + k; ++d) {
    uint64_t gk = 0;
    int64_t gi = INT64_MAX;
    int gc = 0;
    for (unsigned b = tid; b < gridDim.x; b += NT) piv_combine(gk, gi, gc, cand_key[b], cand_idx[b], (int)cand_cnt[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, gk, o);
      const int64_t i2 = __shfl_xor_sync(0xffffffffu, gi, o);
      const int c2 = __shfl_xor_sync(0xffffffffu, gc, o);
      piv_combine(gk, gi, gc, k2, i2, c2);
    }
    if (lane == 0) {
      s_wk[wid] = gk;
      s_wi[wid] = gi;
      s_wc[wid] = gc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NT / 32; ++w) piv_combine(gk, gi, gc, s_wk[w], s_wi[w], s_wc[w]);
      if (gc > 1) {  // rows sharing the winning compact key: a full comparison decides (rare)
        MP<L> rv, x;
        int64_t r = -1;
        for (int64_t i = d; i < row_end; ++i) {
          const uint32_t* q = a + (phys(i) * n + d) * S;
          if (mag_key(q[L], q[L - 1]) != gk) continue;
          load_rec<L>(q, x);
          if (r < 0 || mp_cmpabs<L>(x, rv) > 0) {
            rv = x;
            r = i;
          }
        }
        gi = r;
      }
      s_piv = gi;
      s_gk = gk;
      // interchange logical rows d and r (every CTA does the same)
      const int tmp = s_perm[d - p];
      s_perm[d - p] = s_perm[gi - p];
      s_perm[gi - p] = tmp;
      if (blockIdx.x == 0) piv[d] = gi;
    }
    __syncthreads();
    const int64_t pd = phys(d);
    // zero pivot: every CTA sees the same (maximal) key and stops (blocklu.hpp:46-47); the
    // key is 0 exactly for a zero value
    if (s_gk == 0) {
      if (blockIdx.x == 0 && tid == 0) *zp = d + 1;
      return;
    }
    const int64_t r0 = max(d + 1, lo);
    const int64_t nr = hi - r0;
    if (nr > 0) {
      const int64_t w = p + k - d - 1;
      // the pivot row's values right of the pivot, for the rank-1 update: copied into shared
      // memory asynchronously, in the shadow of the divisions
      {
        constexpr int CH = S / 4;
        const uint32_t* urow = a + (pd * n + d + 1) * S;
        for (int64_t t = tid; t < w * CH; t += NT) {
          const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s_urow + 4 * t));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(urow + 4 * t));
        }
        asm volatile("cp.async.commit_group;\n" ::);
      }
      for (int64_t t = tid; t < nr; t += NT) {
        MP<L> piv_v, x, q;
        load_rec<L>(a + (pd * n + d) * S, piv_v);
        uint32_t* xr = a + (phys(r0 + t) * n + d) * S;
        load_rec<L>(xr, x);
        mp_div<L>(x, piv_v, sh, q);
        store_rec<L>(xr, q);
        store_rec<L>(s_mult + t * S, q);
      }
      asm volatile("cp.async.wait_all;\n" ::);
      __syncthreads();
      const int wi = (int)w, items = (int)(nr * w);  // (32-bit index arithmetic: nr * w < 2^31)
      for (int t = tid; t < items; t += NT) {
        const int rr = t / wi, jj = t - rr * wi;
        const int64_t j = d + 1 + jj;
        MP<L> l, u, pr, x;
        load_rec<L>(s_mult + rr * S, l);
        load_rec<L>(s_urow + jj * S, u);
        mp_mul<L>(l, u, sh, pr);
        uint32_t* xr = a + (phys(r0 + rr) * n + j) * S;
        load_rec<L>(xr, x);
        mp_add<L>(x, pr, 1u, sh, x);
        store_rec<L>(xr, x);
      }
    }
    // (measured slower: the next column's candidates taken from the update's registers (+0.3 %),
    // two update items per thread in one straight-line body (+1.2 %))
    if (d + 1 < p + k) {
      __syncthreads();
      candidates(d + 1, d + 1);
    }
    grid.sync();
  }
}

// the panel's interchanges piv[p .. p+k) applied (in order) to the panel columns
// [p, p+k), each 16-byte chunk of a column independent -- after lu_panel_perm_kernel
template <int L>
__global__ void laswp_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, const int64_t* piv,
                                   const int64_t* zp) {
  constexpr int S = rec_stride(L), CH = S / 4;
  if (*zp) return;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k * CH; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = p + t / CH, w = t % CH;
    for (int64_t d = p; d < p + k; ++d) {
      const int64_t r = piv[d];
      if (r == d) continue;
      uint4* x = reinterpret_cast<uint4*>(a + (d * n + j) * S + 4 * w);
      uint4* y = reinterpret_cast<uint4*>(a + (r * n + j) * S + 4 * w);
      const uint4 tmp = *x;
      *x = *y;
      *y = tmp;
    }
  }
}

// The panel's interchanges piv[p .. p+k) (LAPACK order) as ONE permutation of the rows
// they touch: warp 0 of every CTA composes the swaps on a table of the involved rows in
// shared memory (<= 2k rows; lookups by ballot), then each CTA moves whole column tiles --
// every involved record read once into shared memory, then written to its final row.
// Columns [jlo, jhi) except [skip_lo, skip_hi).  Replaces k dependent swap rounds per
// element (latency-bound) by one read and one write.
template <int L>
__global__ void __launch_bounds__(NT) laswp_perm_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k,
                                                        const int64_t* piv, const int64_t* zp, int64_t jlo,
                                                        int64_t jhi, int64_t skip_lo, int64_t skip_hi, int tc) {
  constexpr int S = rec_stride(L), CH = S / 4;
  if (*zp) return;
  extern __shared__ __align__(16) uint32_t s_dyn[];
  int64_t* s_pos = reinterpret_cast<int64_t*>(s_dyn);  // 2k: involved rows
  int64_t* s_src = s_pos + 2 * k;                      // 2k: original row whose data ends there
  uint4* s_buf = reinterpret_cast<uint4*>(s_src + 2 * k);
  __shared__ int s_cnt;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) {
    for (int64_t i = lane; i < k; i += 32) {
      s_pos[i] = p + i;
      s_src[i] = p + i;
    }
    int cnt = (int)k;
    __syncwarp();
    auto find = [&](int64_t r) -> int {  // index of row r in the table, -1 if absent
      if (r >= p && r < p + k) return (int)(r - p);
      int hit = -1;
      for (int base = (int)k; base < cnt; base += 32) {
        const int i = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < cnt && s_pos[i] == r);
        if (m) {
          hit = base + __ffs(m) - 1;
          break;
        }
      }
      return hit;
    };
    for (int64_t d = p; d < p + k; ++d) {
      const int64_t r = piv[d];
      if (r == d) continue;
      int ir = find(r);
      if (ir < 0) {  // first touch of a row below the panel
        if (lane == 0) {
          s_pos[cnt] = r;
          s_src[cnt] = r;
        }
        ir = cnt++;
        __syncwarp();
      }
      if (lane == 0) {
        const int id = (int)(d - p);
        const int64_t t = s_src[id];
        s_src[id] = s_src[ir];
        s_src[ir] = t;
      }
      __syncwarp();
    }
    if (lane == 0) s_cnt = cnt;
  }
  __syncthreads();
  const int cnt = s_cnt;
  const int64_t ncols = (jhi - jlo) - (skip_hi - skip_lo);
  auto col = [&](int64_t c) { return jlo + c + (jlo + c >= skip_lo ? skip_hi - skip_lo : 0); };
  for (int64_t c0 = (int64_t)blockIdx.x * tc; c0 < ncols; c0 += (int64_t)gridDim.x * tc) {
    const int w = (int)min((int64_t)tc, ncols - c0);
    const int64_t items = (int64_t)cnt * w * CH;
    for (int64_t t = tid; t < items; t += NT) {
      const int i = (int)(t / (w * CH));
      const int rem = (int)(t - (int64_t)i * w * CH), jc = rem / CH, q = rem - jc * CH;
      s_buf[t] = reinterpret_cast<const uint4*>(a + (s_src[i] * n + col(c0 + jc)) * S)[q];
    }
    __syncthreads();
    for (int64_t t = tid; t < items; t += NT) {
      const int i = (int)(t / (w * CH));
      const int rem = (int)(t - (int64_t)i * w * CH), jc = rem / CH, q = rem - jc * CH;
      if (s_src[i] != s_pos[i]) reinterpret_cast<uint4*>(a + (s_pos[i] * n + col(c0 + jc)) * S)[q] = s_buf[t];
    }
    __syncthreads();
  }
}

template <int L>
void launch_laswp_perm(uint32_t* a, int64_t n, int64_t p, int64_t k, const int64_t* piv, const int64_t* zp,
                       int64_t jlo, int64_t jhi, int64_t skip_lo, int64_t skip_hi, cudaStream_t st) {
  constexpr int S = rec_stride(L);
  const int64_t ncols = (jhi - jlo) - (skip_hi - skip_lo);
  if (ncols <= 0 || k <= 0) return;
  // column tile: the <= 2k involved records of tc columns staged in <= 64 KB of shared memory
  int tc = (int)std::max<int64_t>(1, (64 * 1024) / (2 * k * S * 4));
  if (tc > 32) tc = 32;
  const size_t smem = sizeof(int64_t) * 4 * (size_t)k + sizeof(uint32_t) * S * (size_t)(2 * k * tc);
  smem_attr_once((const void*)laswp_perm_kernel<L>, 200 * 1024);
  if (smem > 200 * 1024) {  // very wide records x large panels: the swap-by-swap kernels
    if (skip_hi > skip_lo)
      laswp_kernel<L><<<blocks_for((n - k) * (S / 4)), NT, 0, st>>>(a, n, p, k, piv, zp);
    else
      laswp_panel_kernel<L><<<blocks_for(k * (S / 4)), NT, 0, st>>>(a, n, p, k, piv, zp);
    return;
  }
  const int64_t tiles = (ncols + tc - 1) / tc;
  const int grid = (int)std::min<int64_t>(tiles, 148 * 4);
  laswp_perm_kernel<L><<<grid, NT, smem, st>>>(a, n, p, k, piv, zp, jlo, jhi, skip_lo, skip_hi, tc);
}


template <int L>
int launch_lu_panel_coop(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t row_end, int pivoting,
                         int64_t* piv, int64_t* zp, int sh, uint64_t* cand_key, int64_t* cand_idx, int max_grid,
                         cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled())
      return wmp::launch_lu_panel<L / 32>(a, n, p, k, row_end, pivoting, piv, zp, sh, st);
#endif
  constexpr int S = rec_stride(L);
  uint64_t* cand_cnt = reinterpret_cast<uint64_t*>(cand_idx + max_grid);
  // occupancy, queried once (thread-safe static init; every GPU of the box is the same B200)
  static const int dev_sms = [] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  static const int max_blocks = [] {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_panel_coop_kernel<L>, NT, 16 * 1024);
    return per_sm * dev_sms;
  }();
  const int64_t rows = row_end - p;
  // rows per CTA bounded so the multipliers fit in shared memory
  int64_t want = (rows + 7) / 8;
  int64_t grid = want < max_blocks ? want : max_blocks;
  if (grid > 2 * dev_sms) grid = 2 * dev_sms;
  if (const char* g = std::getenv("MPGPU_LU_COOP_GRID")) grid = std::min<int64_t>(grid, std::atoll(g));
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  // the CTA's multipliers live in shared memory: chunk rows of S words
  const int64_t chunk = (rows + grid - 1) / grid;
  const size_t smem = sizeof(uint32_t) * S * (size_t)chunk;
  if (smem > 16 * 1024) return -1;  // caller falls back to per-column kernels
  if (pivoting && rows <= 12288 && std::getenv("MPGPU_LU_PERM") == nullptr) {
    // one barrier per column: logical row table in shared memory (+ rows int32 words)
    // multipliers (<= 16 KB) + the pivot row (k records) + the row table
    const int kurow = (int)(sizeof(uint32_t) * S * k);
    if (kurow > 48 * 1024) return -1;
    smem_attr_once((const void*)lu_panel_perm_kernel<L>, 16 * 1024 + 48 * 1024 + 4 * 12288);
    static const int per_sm2 = [] {
      int v = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, lu_panel_perm_kernel<L>, NT, 16 * 1024 + 48 * 1024 + 4 * 12288);
      return v;
    }();
    int64_t g2 = std::min<int64_t>(grid, (int64_t)per_sm2 * dev_sms);
    if (g2 < 1) g2 = 1;
    int64_t ch = (rows + g2 - 1) / g2;
    if (sizeof(uint32_t) * S * (size_t)ch > 16 * 1024) return -1;
    const size_t smem2 = sizeof(uint32_t) * S * (size_t)ch + (size_t)kurow + sizeof(int) * (size_t)rows;
    void* args2[] = {&a, &n, &p, &k, &row_end, &piv, &zp, (void*)&sh, &cand_key, &cand_idx, &cand_cnt, &ch};
    cudaError_t e2 = cudaLaunchCooperativeKernel((void*)lu_panel_perm_kernel<L>, dim3((unsigned)g2), dim3(NT), args2,
                                                 smem2, st);
    if (e2 != cudaSuccess) return -1;
    launch_laswp_perm<L>(a, n, p, k, piv, zp, p, p + k, 0, 0, st);
    return 0;
  }
  void* args[] = {&a, &n, &p, &k, &row_end, &pivoting, &piv, &zp, (void*)&sh, &cand_key, &cand_idx, &cand_cnt};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)lu_panel_coop_kernel<L>, dim3((unsigned)grid), dim3(NT), args,
                                              smem, st);
  return e == cudaSuccess ? 0 : -1;
}

template <int L>
int64_t launch_lu_step(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t col_end, int sh, uint32_t* err,
                       const PivotCands& cand, cudaStream_t st) {
  // zero-pivot flag lives right after the error word (see capi.cu)
  int64_t* zp = reinterpret_cast<int64_t*>(err + 2);
  const int64_t rows = row_end - d - 1;
  const int blocks = (int)((rows + LU_RB - 1) / LU_RB);
  const bool want = cand.key != nullptr && d + 1 < col_end && rows > 0 && blocks <= cand.cap;
  lu_col_kernel<L><<<blocks < 1 ? 1 : blocks, NT, 0, st>>>(a, n, d, row_end, col_end, sh, zp,
                                                           want ? cand.key : nullptr, cand.idx, cand.cnt);
  return want ? blocks : 0;
}

template <int L>
void launch_pivot(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t* piv_dev, int64_t* zp,
                  const PivotCands& cand, int64_t ncand, int64_t c0, int64_t c1, cudaStream_t st) {
  pivot_kernel<L><<<1, PIV_NT, 0, st>>>(a, n, d, row_end, piv_dev, zp, cand.key, cand.idx, cand.cnt, ncand, c0, c1);
}

template <int L>
void launch_laswp(uint32_t* a, int64_t n, int64_t p, int64_t k, const int64_t* piv_dev, const int64_t* zp,
                  cudaStream_t st) {
  if (n - k <= 0) return;
  launch_laswp_perm<L>(a, n, p, k, piv_dev, zp, 0, n, p, p + k, st);
}

template <int L>
void launch_trsm_l_step(uint32_t* a, int64_t n, int64_t s, int64_t p_end, int64_t c0, int64_t w, int sh,
                        uint32_t* err, cudaStream_t st) {
  (void)err;
  const int64_t total = (p_end - s - 1) * w;
  if (total > 0) trsm_l_kernel<L><<<blocks_for(total), NT, 0, st>>>(a, n, s, p_end, c0, w, sh);
}

template <int L>
void launch_trsm_l_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0, int64_t w, int sh,
                         cudaStream_t st) {
  if (w <= 0 || k <= 1) return;
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_trsm_panel<L / 32>(a, n, p, k, c0, w, sh, st);
#endif
  const size_t smem = sizeof(uint32_t) * rec_stride(L) * (size_t)(k * TRSM_TC);
  if (smem <= 160 * 1024 && std::getenv("MPGPU_TRSM_GLOBAL") == nullptr) {
    smem_attr_once((const void*)trsm_l_smem_kernel<L>, 160 * 1024);
    trsm_l_smem_kernel<L><<<(int)((w + TRSM_TC - 1) / TRSM_TC), NT, smem, st>>>(a, n, p, k, c0, w, sh, TRSM_TC);
    return;
  }
  trsm_l_panel_kernel<L><<<(int)((w + TRSM_TC - 1) / TRSM_TC), NT, 0, st>>>(a, n, p, k, c0, w, sh);
}

template <int L>
void launch_lu_solve(const uint32_t* f, int64_t n, const int64_t* piv_dev, const uint32_t* b, uint32_t* x,
                     uint32_t* scratch, int sh, uint32_t* err, int64_t* zp, int exact, int64_t nrhs,
                     cudaStream_t st) {
#if MPG_WIDE
  if constexpr (L > 32)
    if (wmp::enabled()) return wmp::launch_lu_solve<L / 32>(f, n, piv_dev, b, x, scratch, sh, err, zp, exact, nrhs, st);
#endif
  lu_solve_kernel<L><<<(unsigned)nrhs, NT, 0, st>>>(f, n, piv_dev, b, x, scratch, nullptr, sh, err, zp, exact);
}

#define MPG_LU_INST(L)                                                                                      \
  template int64_t launch_lu_step<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int, uint32_t*,              \
                                     const PivotCands&, cudaStream_t);                                           \
  template void launch_pivot<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t*, int64_t*, const PivotCands&,    \
                                int64_t, int64_t, int64_t, cudaStream_t);                                       \
  template void launch_laswp<L>(uint32_t*, int64_t, int64_t, int64_t, const int64_t*, const int64_t*, cudaStream_t); \
  template void launch_trsm_l_step<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int, uint32_t*,   \
                                      cudaStream_t);                                                            \
  template void launch_trsm_l_panel<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int, cudaStream_t); \
  template int launch_lu_panel_coop<L>(uint32_t*, int64_t, int64_t, int64_t, int64_t, int, int64_t*, int64_t*, int, \
                                       uint64_t*, int64_t*, int, cudaStream_t);                                      \
  template void launch_lu_solve<L>(const uint32_t*, int64_t, const int64_t*, const uint32_t*, uint32_t*,        \
                                   uint32_t*, int, uint32_t*, int64_t*, int, int64_t, cudaStream_t);
#if MPG_WIDE
#ifdef MPG_WIDE_L  // one wide limb count per translation unit (compile time)
MPG_LU_INST(MPG_WIDE_L)
#else
MPG_LU_INST(64)
MPG_LU_INST(128)
MPG_LU_INST(256)
MPG_LU_INST(288)
#endif
#else
MPG_LU_INST(1)
MPG_LU_INST(2)
MPG_LU_INST(4)
MPG_LU_INST(8)
MPG_LU_INST(16)
MPG_LU_INST(32)
#endif

}  // namespace mpg
