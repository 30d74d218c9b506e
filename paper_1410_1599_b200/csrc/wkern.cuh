// wkern.cuh -- warp-per-element kernels for the wide formats (L = 32 V limbs, 2048 ..
// 9216 bits), built on the warp-cooperative primitives of wmp.cuh.  Same contracts
// (and the same per-element operation order, hence bit-identical results) as the
// thread-per-element kernels of elementwise.cu / gemm.cu / lu.cu, which they replace
// for L > 32: one warp owns one MP value, so a wide mantissa lives in registers (V limbs
// per lane) instead of local memory, and the small matrices of the paper's 8192-bit
// experiments get 32x the parallelism.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "wmp.cuh"

namespace mpg {
namespace wmp {

// MPGPU_WIDE=thread selects the thread-per-element kernels (A/B and cross-checks)
inline bool enabled() {
  const char* e = std::getenv("MPGPU_WIDE");
  return !(e && e[0] == 't');
}

constexpr int WNT = 128;  // threads per CTA (4 warps)
constexpr int WWARPS = WNT / 32;

template <int V>
constexpr size_t smem_bytes() {
  return sizeof(uint32_t) * (size_t)WWARPS * scratch_words<V>();
}

template <int V>
__device__ __forceinline__ Scratch<V> my_scratch() {
  extern __shared__ __align__(16) uint32_t wsm[];
  return scratch_at<V>(wsm + (threadIdx.x >> 5) * scratch_words<V>());
}

__device__ __forceinline__ int64_t gwarp() { return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int64_t nwarps() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

template <class K>
inline void set_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
inline int wblocks(int64_t warps) {
  int64_t b = (warps + WWARPS - 1) / WWARPS;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

// ---- elementwise scalar ops (primitive tests, addsub): op 0 add, 1 sub, 2 mul, 3 div ----
template <int V>
__global__ void __launch_bounds__(WNT) vec_op_kernel(int op, const uint32_t* __restrict__ A,
                                                     const uint32_t* __restrict__ B, uint32_t* __restrict__ C,
                                                     int64_t N, int sh, uint32_t* err) {
  constexpr int S = rec_stride(32 * V);
  const Scratch<V> sc = my_scratch<V>();
  for (int64_t e = gwarp(); e < N; e += nwarps()) {
    W<V> a, b, c;
    load_w<V>(A + e * S, a);
    load_w<V>(B + e * S, b);
    if (op == 0)
      add_w<V>(a, b, 0u, sh, c);
    else if (op == 1)
      add_w<V>(a, b, 1u, sh, c);
    else if (op == 2)
      mul_w<V>(a, b, sh, sc, c);
    else if (b.e == EXP_ZERO) {
      if (lane_id() == 0) atomicOr(err, ERR_DIV_ZERO);
      zero_w<V>(c);
    } else {
      div_w<V>(a, b, sh, sc, c);
    }
    if (lane_id() == 0 && exp_out_of_range(c.e)) atomicOr(err, ERR_EXP_RANGE);
    store_w<V>(C + e * S, c);
  }
}

template <int V>
void launch_vec_op(int op, const uint32_t* A, const uint32_t* B, uint32_t* C, int64_t N, int sh, uint32_t* err,
                   cudaStream_t st) {
  if (N <= 0) return;
  set_smem(vec_op_kernel<V>, smem_bytes<V>());
  vec_op_kernel<V><<<wblocks(N), WNT, smem_bytes<V>(), st>>>(op, A, B, C, N, sh, err);
}

// ---- batched GEMM leaf (gemm.cu contract): one warp per output element -----------
template <int V, bool FOLD>
__global__ void __launch_bounds__(WNT) gemm_kernel(const GemmArgs g) {
  constexpr int S = rec_stride(32 * V);
  const Scratch<V> sc = my_scratch<V>();
  const int64_t per = (int64_t)g.m * g.n, total = per * g.batch;
  for (int64_t o = gwarp(); o < total; o += nwarps()) {
    const int64_t z = o / per, r = o - z * per;
    const int i = (int)(r / g.n), j = (int)(r - (int64_t)i * g.n);
    const uint32_t* A = g.A + (z * g.strideA + (int64_t)i * g.lda) * S;
    const uint32_t* B = g.B + (z * g.strideB + j) * S;
    W<V> acc, pacc;
    zero_w<V>(acc, 1u);  // -0: RN(-0 + x) == x (gemm.cu)
    zero_w<V>(pacc, 1u);
    int next_b = g.kb;
    for (int k = 0; k < g.l; ++k) {
      if (FOLD && k == next_b) {  // Block k-tile boundary: C = RN(C + P), fresh P
        add_w<V>(acc, pacc, 0u, g.sh, acc);
        zero_w<V>(pacc, 1u);
        next_b += g.kb;
      }
      W<V> a, b, t;
      load_w<V>(A + (int64_t)k * S, a);
      load_w<V>(B + (int64_t)k * g.ldb * S, b);
      mul_w<V>(a, b, g.sh, sc, t);
      add_w<V>(pacc, t, 0u, g.sh, pacc);
    }
    W<V> res;
    if (FOLD)
      add_w<V>(acc, pacc, 0u, g.sh, res);
    else
      res = pacc;
    uint32_t* cr = g.C + (z * g.strideC + (int64_t)i * g.ldc + j) * S;
    if (g.sub_from_c) {  // LU Schur update: A22 = RN(A22 - prod) (blocklu.hpp:138-141)
      W<V> old;
      load_w<V>(cr, old);
      add_w<V>(old, res, 1u, g.sh, res);
    }
    if (lane_id() == 0 && exp_out_of_range(res.e)) atomicOr(g.err, ERR_EXP_RANGE);
    store_w<V>(cr, res);
  }
}

template <int V>
void launch_gemm(const GemmArgs& g, cudaStream_t st) {
  const int64_t total = (int64_t)g.m * g.n * g.batch;
  if (total <= 0) return;
  if (g.kb < g.l) {
    set_smem(gemm_kernel<V, true>, smem_bytes<V>());
    gemm_kernel<V, true><<<wblocks(total), WNT, smem_bytes<V>(), st>>>(g);
  } else {
    set_smem(gemm_kernel<V, false>, smem_bytes<V>());
    gemm_kernel<V, false><<<wblocks(total), WNT, smem_bytes<V>(), st>>>(g);
  }
}

// ---- LU (lu.cu contracts) ------------------------------------------------------
__device__ __forceinline__ uint64_t wmag_key(uint32_t e, uint32_t top) {
  return e == (uint32_t)EXP_ZERO ? 0ull : (((uint64_t)(e ^ 0x80000000u)) << 32) | top;
}
__device__ __forceinline__ void wpiv_combine(uint64_t& k, int64_t& i, int& c, uint64_t k2, int64_t i2, int c2) {
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

// whole-panel factorisation in one cooperative launch (lu.cu lu_panel_coop_kernel):
// per pivot column d -- (pivoting) candidate reduction, swap, grid.sync; one warp per
// row divides (multiplier), then one warp per (row, column) applies the rank-1
// update of the CTA's rows; next column's candidates; grid.sync.
template <int V>
__global__ void __launch_bounds__(WNT) lu_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k,
                                                       int64_t row_end, int pivoting, int64_t* piv, int64_t* zp,
                                                       int sh, uint64_t* cand_key, int64_t* cand_idx,
                                                       uint64_t* cand_cnt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int L = 32 * V, S = rec_stride(L);
  const Scratch<V> sc = my_scratch<V>();
  __shared__ uint64_t s_wk[WWARPS];
  __shared__ int64_t s_wi[WWARPS];
  __shared__ int s_wc[WWARPS];
  __shared__ int64_t s_piv;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rows_all = row_end - p;
  const int64_t chunk = (rows_all + gridDim.x - 1) / gridDim.x;
  const int64_t lo = p + (int64_t)blockIdx.x * chunk;
  const int64_t hi = min(row_end, lo + chunk);
  auto block_reduce_store = [&](uint64_t bk, int64_t bi, int bc) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(FULL, bk, o);
      const int64_t i2 = __shfl_xor_sync(FULL, bi, o);
      const int c2 = __shfl_xor_sync(FULL, bc, o);
      wpiv_combine(bk, bi, bc, k2, i2, c2);
    }
    if (lane == 0) {
      s_wk[wid] = bk;
      s_wi[wid] = bi;
      s_wc[wid] = bc;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < WWARPS; ++w) wpiv_combine(bk, bi, bc, s_wk[w], s_wi[w], s_wc[w]);
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
    for (int64_t i = max(from, lo) + tid; i < hi; i += WNT) {
      const uint32_t* r = a + (i * n + col) * S;
      wpiv_combine(bk, bi, bc, wmag_key(r[L], r[L - 1]), i, 1);
    }
    block_reduce_store(bk, bi, bc);
  };
  if (pivoting) {
    candidates(p, p);
    grid.sync();
  }
  for (int64_t d = p; d < p + k; ++d) {
    if (pivoting) {
      uint64_t gk = 0;
      int64_t gi = INT64_MAX;
      int gc = 0;
      for (unsigned b = tid; b < gridDim.x; b += WNT) wpiv_combine(gk, gi, gc, cand_key[b], cand_idx[b], (int)cand_cnt[b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(FULL, gk, o);
        const int64_t i2 = __shfl_xor_sync(FULL, gi, o);
        const int c2 = __shfl_xor_sync(FULL, gc, o);
        wpiv_combine(gk, gi, gc, k2, i2, c2);
      }
      if (lane == 0) {
        s_wk[wid] = gk;
        s_wi[wid] = gi;
        s_wc[wid] = gc;
      }
      __syncthreads();
      if (wid == 0) {
        for (int w = 1; w < WWARPS; ++w) wpiv_combine(gk, gi, gc, s_wk[w], s_wi[w], s_wc[w]);
        if (gc > 1) {  // rows sharing the winning compact key: full comparison (first max wins)
          W<V> rv, x;
          int64_t r = -1;
          for (int64_t i = d; i < row_end; ++i) {
            const uint32_t* q = a + (i * n + d) * S;
            if (wmag_key(q[L], q[L - 1]) != gk) continue;
            load_w<V>(q, x);
            if (r < 0 || cmpabs_w<V>(x, rv) > 0) {
              rv = x;
              r = i;
            }
          }
          gi = r;
        }
        if (lane == 0) s_piv = gi;
      }
      __syncthreads();
      const int64_t r = s_piv;
      if (blockIdx.x == 0) {
        if (tid == 0) piv[d] = r;
        if (r != d) {
          constexpr int CH = S / 4;
          for (int64_t t = tid; t < k * CH; t += WNT) {
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
    if (a[(d * n + d) * S + L] == (uint32_t)EXP_ZERO) {  // zero pivot (blocklu.hpp:46-47)
      if (blockIdx.x == 0 && tid == 0) *zp = d + 1;
      return;
    }
    const int64_t r0 = max(d + 1, lo);
    const int64_t nr = hi - r0;
    if (nr > 0) {
      W<V> pv;
      load_w<V>(a + (d * n + d) * S, pv);
      for (int64_t t = wid; t < nr; t += WWARPS) {
        W<V> x, q;
        uint32_t* xr = a + ((r0 + t) * n + d) * S;
        load_w<V>(xr, x);
        div_w<V>(x, pv, sh, sc, q);
        store_w<V>(xr, q);
      }
      __syncthreads();
      const int64_t w = p + k - d - 1;
      for (int64_t t = wid; t < nr * w; t += WWARPS) {
        const int64_t rr = t / w, j = d + 1 + t % w;
        W<V> l, u, pr, x;
        load_w<V>(a + ((r0 + rr) * n + d) * S, l);
        load_w<V>(a + (d * n + j) * S, u);
        mul_w<V>(l, u, sh, sc, pr);
        uint32_t* xr = a + ((r0 + rr) * n + j) * S;
        load_w<V>(xr, x);
        add_w<V>(x, pr, 1u, sh, x);
        store_w<V>(xr, x);
      }
    }
    if (pivoting && d + 1 < p + k) {
      __syncthreads();
      candidates(d + 1, d + 1);
    }
    grid.sync();
  }
}

template <int V>
int launch_lu_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t row_end, int pivoting, int64_t* piv,
                    int64_t* zp, int sh, uint64_t* cand_key, int64_t* cand_idx, int max_grid, cudaStream_t st) {
  uint64_t* cand_cnt = reinterpret_cast<uint64_t*>(cand_idx + max_grid);
  static int max_blocks = 0;
  const size_t smem = smem_bytes<V>();
  if (!max_blocks) {
    set_smem(lu_panel_kernel<V>, smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_panel_kernel<V>, WNT, smem);
    max_blocks = per_sm * sms;
  }
  const int64_t rows = row_end - p;
  // a few rows per CTA: every warp divides at most one row per column
  int64_t grid = (rows + WWARPS - 1) / WWARPS;
  if (grid > max_blocks) grid = max_blocks;
  if (const char* g = std::getenv("MPGPU_LU_COOP_GRID")) grid = std::min<int64_t>(grid, std::atoll(g));
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  void* args[] = {&a, &n, &p, &k, &row_end, &pivoting, &piv, &zp, (void*)&sh, &cand_key, &cand_idx, &cand_cnt};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((void*)lu_panel_kernel<V>, dim3((unsigned)grid), dim3(WNT), args, smem, st);
  return e == cudaSuccess ? 0 : -1;
}

// trsm_unit_lower over a panel (lu.cu trsm_l_panel_kernel): each CTA owns TC columns
// of U12 and sweeps s = p .. p+k-2, one warp per (row, column) element per step
template <int V>
__global__ void __launch_bounds__(WNT) trsm_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0,
                                                         int64_t w, int sh, int TC) {
  constexpr int S = rec_stride(32 * V);
  const Scratch<V> sc = my_scratch<V>();
  const int wid = threadIdx.x >> 5;
  const int64_t j0 = c0 + (int64_t)blockIdx.x * TC;
  const int tc = (int)(c0 + w - j0 < TC ? c0 + w - j0 : TC);
  for (int64_t s = p; s + 1 < p + k; ++s) {
    const int64_t rows = p + k - s - 1;
    for (int64_t t = wid; t < rows * tc; t += WWARPS) {
      const int64_t i = s + 1 + t / tc, j = j0 + t % tc;
      W<V> l, u, pr, x;
      load_w<V>(a + (i * n + s) * S, l);
      load_w<V>(a + (s * n + j) * S, u);
      mul_w<V>(l, u, sh, sc, pr);
      uint32_t* xr = a + (i * n + j) * S;
      load_w<V>(xr, x);
      add_w<V>(x, pr, 1u, sh, x);
      store_w<V>(xr, x);
    }
    __syncthreads();
  }
}

template <int V>
void launch_trsm_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0, int64_t w, int sh,
                       cudaStream_t st) {
  if (w <= 0 || k <= 1) return;
  constexpr int TC = 2;
  set_smem(trsm_panel_kernel<V>, smem_bytes<V>());
  trsm_panel_kernel<V><<<(unsigned)((w + TC - 1) / TC), WNT, smem_bytes<V>(), st>>>(a, n, p, k, c0, w, sh, TC);
}

// Ly = Pb, Ux = y (lu.cu lu_solve_kernel): one CTA per right-hand side, warps over rows;
// the exact back substitution accumulates each row's products in s-ascending order
// (blocklu.hpp:235-238) in warp 0.
template <int V>
__global__ void __launch_bounds__(WNT) lu_solve_kernel(const uint32_t* f, int64_t n, const int64_t* piv,
                                                       const uint32_t* b, uint32_t* x, uint32_t* y, int sh,
                                                       uint32_t* err, int64_t* zp, int exact) {
  constexpr int S = rec_stride(32 * V), CH = S / 4;
  const Scratch<V> sc = my_scratch<V>();
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  b += (int64_t)blockIdx.x * n * S;
  x += (int64_t)blockIdx.x * n * S;
  y += (int64_t)blockIdx.x * 2 * n * S;
  uint32_t* tmp = y + n * S;
  for (int64_t t = tid; t < n * CH; t += WNT) reinterpret_cast<uint4*>(y)[t] = reinterpret_cast<const uint4*>(b)[t];
  __syncthreads();
  if (piv && tid == 0) {
    for (int64_t d = 0; d < n; ++d) {
      const int64_t r = piv[d];
      if (r != d)
        for (int w = 0; w < CH; ++w) {
          uint4* pp = reinterpret_cast<uint4*>(y + d * S) + w;
          uint4* qq = reinterpret_cast<uint4*>(y + r * S) + w;
          const uint4 t = *pp;
          *pp = *qq;
          *qq = t;
        }
    }
  }
  __syncthreads();
  for (int64_t s = 0; s < n; ++s) {
    W<V> ys;
    load_w<V>(y + s * S, ys);
    for (int64_t i = s + 1 + wid; i < n; i += WWARPS) {
      W<V> l, pr, acc;
      load_w<V>(f + (i * n + s) * S, l);
      mul_w<V>(l, ys, sh, sc, pr);
      load_w<V>(y + i * S, acc);
      add_w<V>(acc, pr, 1u, sh, acc);
      store_w<V>(y + i * S, acc);
    }
    __syncthreads();
  }
  __shared__ int s_stop;
  if (!exact) {
    for (int64_t ii = n - 1; ii >= 0; --ii) {
      if (wid == 0) {
        W<V> acc, dd, q;
        load_w<V>(y + ii * S, acc);
        load_w<V>(f + (ii * n + ii) * S, dd);
        if (dd.e == EXP_ZERO) {
          if (lane == 0 && *zp == 0) *zp = ii + 1;
          zero_w<V>(q);
        } else {
          div_w<V>(acc, dd, sh, sc, q);
        }
        if (lane == 0 && exp_out_of_range(q.e)) atomicOr(err, ERR_EXP_RANGE);
        store_w<V>(x + ii * S, q);
        if (lane == 0) s_stop = dd.e == EXP_ZERO;
      }
      __syncthreads();
      if (s_stop) return;
      W<V> xs;
      load_w<V>(x + ii * S, xs);
      for (int64_t i = wid; i < ii; i += WWARPS) {
        W<V> u, pr, acc;
        load_w<V>(f + (i * n + ii) * S, u);
        mul_w<V>(u, xs, sh, sc, pr);
        load_w<V>(y + i * S, acc);
        add_w<V>(acc, pr, 1u, sh, acc);
        store_w<V>(y + i * S, acc);
      }
      __syncthreads();
    }
    return;
  }
  for (int64_t ii = n - 1; ii >= 0; --ii) {
    for (int64_t s = ii + 1 + wid; s < n; s += WWARPS) {
      W<V> u, xs, pr;
      load_w<V>(f + (ii * n + s) * S, u);
      load_w<V>(x + s * S, xs);
      mul_w<V>(u, xs, sh, sc, pr);
      store_w<V>(tmp + s * S, pr);
    }
    __syncthreads();
    if (wid == 0) {
      W<V> acc;
      load_w<V>(y + ii * S, acc);
      for (int64_t s = ii + 1; s < n; ++s) {
        W<V> pr;
        load_w<V>(tmp + s * S, pr);
        add_w<V>(acc, pr, 1u, sh, acc);
      }
      W<V> dd, q;
      load_w<V>(f + (ii * n + ii) * S, dd);
      if (dd.e == EXP_ZERO) {
        if (lane == 0 && *zp == 0) *zp = ii + 1;
        zero_w<V>(q);
      } else {
        div_w<V>(acc, dd, sh, sc, q);
      }
      if (lane == 0 && exp_out_of_range(q.e)) atomicOr(err, ERR_EXP_RANGE);
      store_w<V>(x + ii * S, q);
      if (lane == 0) s_stop = dd.e == EXP_ZERO;
    }
    __syncthreads();
    if (s_stop) return;
  }
}

template <int V>
void launch_lu_solve(const uint32_t* f, int64_t n, const int64_t* piv, const uint32_t* b, uint32_t* x,
                     uint32_t* scratch, int sh, uint32_t* err, int64_t* zp, int exact, int64_t nrhs,
                     cudaStream_t st) {
  set_smem(lu_solve_kernel<V>, smem_bytes<V>());
  lu_solve_kernel<V><<<(unsigned)nrhs, WNT, smem_bytes<V>(), st>>>(f, n, piv, b, x, scratch, sh, err, zp, exact);
}

}  // namespace wmp
}  // namespace mpg
