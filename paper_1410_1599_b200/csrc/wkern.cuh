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
    W<V> na, nb;  // operands of the next k, loaded one step ahead (latency-bound loop)
    load_w<V>(A, na);
    load_w<V>(B, nb);
    for (int k = 0; k < g.l; ++k) {
      if (FOLD && k == next_b) {  // Block k-tile boundary: C = RN(C + P), fresh P
        add_w<V>(acc, pacc, 0u, g.sh, acc);
        zero_w<V>(pacc, 1u);
        next_b += g.kb;
      }
      W<V> a = na, b = nb, t;
      if (k + 1 < g.l) {
        load_w<V>(A + (int64_t)(k + 1) * S, na);
        load_w<V>(B + (int64_t)(k + 1) * g.ldb * S, nb);
      }
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

// ---- Strassen / Winograd level transforms (elementwise.cu contracts), one warp per
// (node, quadrant element); the same sums in the same operand order as the reference
// (fastmm.hpp:133-198), zero padding of odd dimensions virtual (+0) ------------------
template <int V>
__global__ void __launch_bounds__(WNT) preadd_kernel(int algo, int side, const uint32_t* __restrict__ parent,
                                                     int64_t nodes, int rows, int cols,
                                                     uint32_t* __restrict__ children, int sh) {
  constexpr int S = rec_stride(32 * V);
  const int hr = (rows + rows % 2) / 2, hc = (cols + cols % 2) / 2;
  const int64_t per = (int64_t)hr * hc;
  const int64_t total = per * nodes;
  for (int64_t t = gwarp(); t < total; t += nwarps()) {
    const int64_t node = t / per;
    const int64_t e = t - node * per;
    const int r = (int)(e / hc), c = (int)(e - (int64_t)r * hc);
    const uint32_t* P = parent + node * (int64_t)rows * cols * S;
    uint32_t* out = children + (node * 7 * per + e) * S;
    const int64_t cs = per * S;
    auto ld = [&](int q, W<V>& x) {
      const int rr = r + (q >> 1) * hr, cc = c + (q & 1) * hc;
      if (rr < rows && cc < cols)
        load_w<V>(P + ((int64_t)rr * cols + cc) * S, x);
      else
        zero_w<V>(x, 0);
    };
    auto put = [&](int child, const W<V>& x) { store_w<V>(out + child * cs, x); };
    auto sum = [&](int qa, int qb, uint32_t neg, int child) {
      W<V> x, y, z;
      ld(qa, x);
      ld(qb, y);
      add_w<V>(x, y, neg, sh, z);
      put(child, z);
    };
    auto copy = [&](int q, int child) {
      W<V> x;
      ld(q, x);
      put(child, x);
    };
    if (algo == 3) {
      W<V> s1, s2, x, y;
      if (side == 0) {  // S1 = a21+a22 (M5), S2 = S1-a11 (M1), S3 = a11-a21 (M4), S4 = a12-S2 (M6)
        ld(2, x);
        ld(3, y);
        add_w<V>(x, y, 0u, sh, s1);
        put(4, s1);
        ld(0, x);
        add_w<V>(s1, x, 1u, sh, s2);
        put(0, s2);
        ld(1, x);
        add_w<V>(x, s2, 1u, sh, y);
        put(5, y);
        sum(0, 2, 1u, 3);
        copy(0, 1);
        copy(1, 2);
        copy(3, 6);
      } else {  // S5 = b12-b11 (M5), S6 = b22-S5 (M1), S7 = b22-b12 (M4), S8 = S6-b21 (M7)
        ld(1, x);
        ld(0, y);
        add_w<V>(x, y, 1u, sh, s1);
        put(4, s1);
        ld(3, x);
        add_w<V>(x, s1, 1u, sh, s2);
        put(0, s2);
        ld(2, x);
        add_w<V>(s2, x, 1u, sh, y);
        put(6, y);
        sum(3, 1, 1u, 3);
        copy(0, 1);
        copy(2, 2);
        copy(3, 5);
      }
    } else if (side == 0) {  // a11+a22, a21+a22, a11, a22, a11+a12, a21-a11, a12-a22
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

template <int V>
void launch_preadd(int algo, int side, const uint32_t* parent, int64_t nodes, int rows, int cols,
                   uint32_t* children, int sh, cudaStream_t st) {
  const int64_t total = (int64_t)((rows + rows % 2) / 2) * ((cols + cols % 2) / 2) * nodes;
  if (total <= 0) return;
  preadd_kernel<V><<<wblocks(total), WNT, 0, st>>>(algo, side, parent, nodes, rows, cols, children, sh);
}

template <int V>
__global__ void __launch_bounds__(WNT) postadd_kernel(int algo, const uint32_t* __restrict__ children,
                                                      int64_t nodes, int rows, int cols,
                                                      uint32_t* __restrict__ parent, uint32_t* __restrict__ t_out,
                                                      int sh, uint32_t* err, const int* __restrict__ rowlist,
                                                      int nrows) {
  constexpr int S = rec_stride(32 * V);
  const int hr = (rows + rows % 2) / 2, hc = (cols + cols % 2) / 2;
  const int64_t per = (int64_t)hr * hc;
  const int64_t per_iter = (rowlist ? (int64_t)nrows : (int64_t)hr) * hc;
  const int64_t total = per_iter * nodes;
  for (int64_t t = gwarp(); t < total; t += nwarps()) {
    const int64_t node = t / per_iter;
    const int64_t ei = t - node * per_iter;
    const int ri = (int)(ei / hc), c = (int)(ei - (int64_t)ri * hc);
    const int r = rowlist ? rowlist[ri] : ri;
    const int64_t e = (int64_t)r * hc + c;
    const uint32_t* M = children + (node * 7 * per + e) * S;
    const int64_t cs = per * S;
    uint32_t* P = parent + node * (int64_t)rows * cols * S;
    auto store_if = [&](int rr, int cc, const W<V>& x) {  // strip the padding
      if (rr < rows && cc < cols) {
        if (lane_id() == 0 && exp_out_of_range(x.e)) atomicOr(err, ERR_EXP_RANGE);
        store_w<V>(P + ((int64_t)rr * cols + cc) * S, x);
      }
    };
    if (algo == 3) {  // T1 = M1+M2, T2 = T1+M4; C11 = M2+M3, C12 = (T1+M5)+M6, C21 = T2-M7, C22 = T2+M5
      W<V> m1, m2, t1, t2, u, v, x;
      load_w<V>(M, m1);
      load_w<V>(M + cs, m2);
      add_w<V>(m1, m2, 0u, sh, t1);
      load_w<V>(M + 3 * cs, x);
      add_w<V>(t1, x, 0u, sh, t2);
      if (t_out) {
        store_w<V>(t_out + (node * 2 * per + e) * S, t1);
        store_w<V>(t_out + (node * 2 * per + per + e) * S, t2);
      }
      load_w<V>(M + 2 * cs, x);
      add_w<V>(m2, x, 0u, sh, u);
      store_if(r, c, u);
      W<V> m5;
      load_w<V>(M + 4 * cs, m5);
      load_w<V>(M + 5 * cs, x);
      add_w<V>(t1, m5, 0u, sh, u);
      add_w<V>(u, x, 0u, sh, v);
      store_if(r, c + hc, v);
      load_w<V>(M + 6 * cs, x);
      add_w<V>(t2, x, 1u, sh, u);
      store_if(r + hr, c, u);
      add_w<V>(t2, m5, 0u, sh, u);
      store_if(r + hr, c + hc, u);
    } else {  // C11 = ((P1+P4)-P5)+P7, C12 = P3+P5, C21 = P2+P4, C22 = ((P1+P3)-P2)+P6
      W<V> p1, p4, p5, u, v, x;
      load_w<V>(M, p1);
      load_w<V>(M + 3 * cs, p4);
      load_w<V>(M + 4 * cs, p5);
      add_w<V>(p1, p4, 0u, sh, u);
      add_w<V>(u, p5, 1u, sh, v);
      load_w<V>(M + 6 * cs, x);
      add_w<V>(v, x, 0u, sh, u);
      store_if(r, c, u);
      W<V> p3, p2;
      load_w<V>(M + 2 * cs, p3);
      add_w<V>(p3, p5, 0u, sh, u);
      store_if(r, c + hc, u);
      load_w<V>(M + cs, p2);
      add_w<V>(p2, p4, 0u, sh, u);
      store_if(r + hr, c, u);
      add_w<V>(p1, p3, 0u, sh, u);
      add_w<V>(u, p2, 1u, sh, v);
      load_w<V>(M + 5 * cs, x);
      add_w<V>(v, x, 0u, sh, u);
      store_if(r + hr, c + hc, u);
    }
  }
}

template <int V>
void launch_postadd(int algo, const uint32_t* children, int64_t nodes, int rows, int cols, uint32_t* parent,
                    uint32_t* t_out, int sh, uint32_t* err, cudaStream_t st, const int* rowlist, int nrows) {
  const int64_t total = (int64_t)(rowlist ? nrows : (rows + rows % 2) / 2) * ((cols + cols % 2) / 2) * nodes;
  if (total <= 0) return;
  postadd_kernel<V><<<wblocks(total), WNT, 0, st>>>(algo, children, nodes, rows, cols, parent, t_out, sh, err,
                                                     rowlist, nrows);
}

// ---- accuracy metric (metrics.cu rel_error_kernel contract), one warp per element ----
template <int V>
__global__ void __launch_bounds__(WNT) rel_error_kernel(const uint32_t* __restrict__ approx, int la, int sa,
                                                        int64_t lda, const uint32_t* __restrict__ ref, int64_t ldr,
                                                        int rows, int cols, int mode, int sh,
                                                        uint32_t* __restrict__ outA, uint32_t* __restrict__ outB,
                                                        unsigned long long* counter, uint32_t* err) {
  constexpr int L = 32 * V, S = rec_stride(L);
  constexpr uint32_t SKIP = 2u;
  const Scratch<V> sc = my_scratch<V>();
  const int lane = lane_id();
  const int64_t N = (int64_t)rows * cols;
  auto store_flag = [&](uint32_t* r, const W<V>& x, uint32_t flag) {
#pragma unroll
    for (int j = 0; j < V; ++j) r[lane * V + j] = x.m[j];
    if (lane == 0) r[L] = (uint32_t)x.e;
    if (lane == 1) r[L + 1] = x.s | flag;
  };
  for (int64_t t = gwarp(); t < N; t += nwarps()) {
    const int64_t i = t / cols, j = t - i * cols;
    const uint32_t* ar = approx + (i * lda + j) * sa;
    W<V> a, r, d;
    const int off = L - la;  // approx has la <= L limbs: widened exactly (low limbs zero)
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int k = lane * V + q;
      a.m[q] = k >= off ? ar[k - off] : 0u;
    }
    a.e = (int32_t)ar[la];
    a.s = ar[la + 1];
    load_w<V>(ref + (i * ldr + j) * S, r);
    add_w<V>(a, r, 1u, sh, d);  // sub(approx, reference, ctx)
    d.s = 0;                    // abs
    if (r.e == EXP_ZERO) {
      if (lane == 0) atomicAdd(counter, 1ull);
      store_flag(outA + t * S, r, SKIP);
      if (mode == 1) store_flag(outB + t * S, d, 0u);
      continue;
    }
    r.s = 0;
    W<V> q;
    div_w<V>(d, r, sh, sc, q);  // div(abs(d), abs(reference), ctx)
    if (lane == 0 && (exp_out_of_range(q.e) || exp_out_of_range(d.e))) atomicOr(err, ERR_EXP_RANGE);
    store_flag(outA + t * S, q, 0u);
    if (mode == 1) store_flag(outB + t * S, q, SKIP);
  }
}

template <int V>
void launch_rel_error(const uint32_t* approx, int la, int64_t lda, const uint32_t* ref, int64_t ldr, int rows,
                      int cols, int mode, int sh, uint32_t* outA, uint32_t* outB, unsigned long long* counter,
                      uint32_t* err, cudaStream_t st) {
  const int64_t N = (int64_t)rows * cols;
  if (N <= 0) return;
  set_smem(rel_error_kernel<V>, smem_bytes<V>());
  rel_error_kernel<V><<<wblocks(N), WNT, smem_bytes<V>(), st>>>(approx, la, rec_stride(la), lda, ref, ldr, rows,
                                                                  cols, mode, sh, outA, outB, counter, err);
}

// ---- LU (lu.cu contracts) ------------------------------------------------------
// The LU kernels are cooperative: every parallel phase (divisions, rank-1 updates,
// triangular-solve steps) is spread over all warps of a grid that fills the GPU, with a
// grid barrier between dependent phases -- an 8192-bit multiply-add takes tens of
// microseconds in one warp, so the per-column work must not be confined to a few CTAs.
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

// a_ij = RN(a_ij - RN(l * u)) for the record at xr (blocklu.hpp:51-52, 66-67)
template <int V>
__device__ __forceinline__ void sub_prod(uint32_t* xr, const uint32_t* lr, const uint32_t* ur, int sh,
                                         const Scratch<V>& sc) {
  W<V> l, u, pr, x;
  load_w<V>(lr, l);
  load_w<V>(ur, u);
  mul_w<V>(l, u, sh, sc, pr);
  load_w<V>(xr, x);
  add_w<V>(x, pr, 1u, sh, x);
  store_w<V>(xr, x);
}

// co-resident grid size for a cooperative kernel, capped by the useful warps
template <class K>
inline int coop_grid(K kern, size_t smem, int64_t want_warps) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  set_smem(kern, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WNT, smem);
  int64_t g = (want_warps + WWARPS - 1) / WWARPS;
  const int64_t cap = (int64_t)per_sm * sms;
  if (const char* e = std::getenv("MPGPU_LU_COOP_GRID")) g = std::min<int64_t>(g, std::atoll(e));
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// whole-panel factorisation [p, p+k) x rows [p, row_end) in one cooperative launch
// (lu.cu lu_panel_coop_kernel).  Per pivot column d: (pivoting) every CTA reduces the
// column's magnitude keys itself -- identical pivot everywhere -- CTA 0 swaps the
// panel rows, barrier; multipliers (one warp per row, all warps of the grid), barrier;
// rank-1 update (one warp per element, all warps), barrier.
template <int V>
__global__ void __launch_bounds__(WNT) lu_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k,
                                                       int64_t row_end, int pivoting, int64_t* piv, int64_t* zp,
                                                       int sh) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int L = 32 * V, S = rec_stride(L);
  const Scratch<V> sc = my_scratch<V>();
  __shared__ uint64_t s_wk[WWARPS];
  __shared__ int64_t s_wi[WWARPS];
  __shared__ int s_wc[WWARPS];
  __shared__ int64_t s_piv;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t gw = gwarp(), NW = nwarps();
  for (int64_t d = p; d < p + k; ++d) {
    if (pivoting) {
      uint64_t bk = 0;
      int64_t bi = INT64_MAX;
      int bc = 0;
      for (int64_t i = d + tid; i < row_end; i += WNT) {
        const uint32_t* r = a + (i * n + d) * S;
        wpiv_combine(bk, bi, bc, wmag_key(r[L], r[L - 1]), i, 1);
      }
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
      if (wid == 0) {
        for (int w = 1; w < WWARPS; ++w) wpiv_combine(bk, bi, bc, s_wk[w], s_wi[w], s_wc[w]);
        if (bc > 1) {  // rows sharing the winning compact key: full comparison (first max wins)
          W<V> rv, x;
          int64_t r = -1;
          for (int64_t i = d; i < row_end; ++i) {
            const uint32_t* q = a + (i * n + d) * S;
            if (wmag_key(q[L], q[L - 1]) != bk) continue;
            load_w<V>(q, x);
            if (r < 0 || cmpabs_w<V>(x, rv) > 0) {
              rv = x;
              r = i;
            }
          }
          bi = r;
        }
        if (lane == 0) s_piv = bi;
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
    const int64_t rows = row_end - d - 1;
    if (rows <= 0) break;
    {
      W<V> pv;
      load_w<V>(a + (d * n + d) * S, pv);
      for (int64_t t = gw; t < rows; t += NW) {
        W<V> x, q;
        uint32_t* xr = a + ((d + 1 + t) * n + d) * S;
        load_w<V>(xr, x);
        div_w<V>(x, pv, sh, sc, q);
        store_w<V>(xr, q);
      }
    }
    const int64_t w = p + k - d - 1;
    if (w <= 0) break;
    grid.sync();
    for (int64_t t = gw; t < rows * w; t += NW) {
      const int64_t i = d + 1 + t / w, j = d + 1 + t % w;
      sub_prod<V>(a + (i * n + j) * S, a + (i * n + d) * S, a + (d * n + j) * S, sh, sc);
    }
    grid.sync();
  }
}

template <int V>
int launch_lu_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t row_end, int pivoting, int64_t* piv,
                    int64_t* zp, int sh, cudaStream_t st) {
  const size_t smem = smem_bytes<V>();
  const int64_t rows = row_end - p;
  int grid = coop_grid(lu_panel_kernel<V>, smem, rows * std::min<int64_t>(k, rows));
  void* args[] = {&a, &n, &p, &k, &row_end, &pivoting, &piv, &zp, (void*)&sh};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((void*)lu_panel_kernel<V>, dim3((unsigned)grid), dim3(WNT), args, smem, st);
  return e == cudaSuccess ? 0 : -1;
}

// trsm_unit_lower over a panel (lu.cu trsm_l_panel_kernel): step s = p .. p+k-2 updates
// rows (s, p+k) x cols [c0, c0+w) -- one warp per element over the whole grid -- then a
// grid barrier; per element the updates arrive in s-ascending order (blocklu.hpp:60-69).
template <int V>
__global__ void __launch_bounds__(WNT) trsm_panel_kernel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0,
                                                         int64_t w, int sh) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int S = rec_stride(32 * V);
  const Scratch<V> sc = my_scratch<V>();
  const int64_t gw = gwarp(), NW = nwarps();
  for (int64_t s = p; s + 1 < p + k; ++s) {
    const int64_t rows = p + k - s - 1;
    for (int64_t t = gw; t < rows * w; t += NW) {
      const int64_t i = s + 1 + t / w, j = c0 + t % w;
      sub_prod<V>(a + (i * n + j) * S, a + (i * n + s) * S, a + (s * n + j) * S, sh, sc);
    }
    grid.sync();
  }
}

template <int V>
void launch_trsm_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0, int64_t w, int sh,
                       cudaStream_t st) {
  if (w <= 0 || k <= 1) return;
  const size_t smem = smem_bytes<V>();
  int grid = coop_grid(trsm_panel_kernel<V>, smem, (k - 1) * w);
  void* args[] = {&a, &n, &p, &k, &c0, &w, (void*)&sh};
  cudaLaunchCooperativeKernel((void*)trsm_panel_kernel<V>, dim3((unsigned)grid), dim3(WNT), args, smem, st);
}

// Ly = Pb, Ux = y for nrhs right-hand sides (lu.cu lu_solve_kernel), cooperative: the
// parallel steps -- forward updates, back-substitution products / updates -- run over
// (right-hand side, row) pairs on all warps of the grid; the exact back substitution's
// s-ascending accumulation of each row (blocklu.hpp:235-238) runs in one warp per
// right-hand side.  Scratch: 2n records per right-hand side (y, products).
template <int V>
__global__ void __launch_bounds__(WNT) lu_solve_kernel(const uint32_t* f, int64_t n, const int64_t* piv,
                                                       const uint32_t* b, uint32_t* x, uint32_t* y, int sh,
                                                       uint32_t* err, int64_t* zp, int exact, int64_t nrhs) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int S = rec_stride(32 * V), CH = S / 4;
  const Scratch<V> sc = my_scratch<V>();
  const int lane = lane_id();
  const int64_t gw = gwarp(), NW = nwarps();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, NT = (int64_t)gridDim.x * blockDim.x;
  auto Y = [&](int64_t r) { return y + r * 2 * n * S; };
  auto T = [&](int64_t r) { return y + r * 2 * n * S + n * S; };
  for (int64_t t = gt; t < nrhs * n * CH; t += NT) {
    const int64_t r = t / (n * CH), q = t - r * n * CH;
    reinterpret_cast<uint4*>(Y(r))[q] = reinterpret_cast<const uint4*>(b + r * n * S)[q];
  }
  grid.sync();
  if (piv) {
    for (int64_t r = gt; r < nrhs; r += NT)
      for (int64_t d = 0; d < n; ++d) {
        const int64_t pr = piv[d];
        if (pr != d)
          for (int w = 0; w < CH; ++w) {
            uint4* pp = reinterpret_cast<uint4*>(Y(r) + d * S) + w;
            uint4* qq = reinterpret_cast<uint4*>(Y(r) + pr * S) + w;
            const uint4 tv = *pp;
            *pp = *qq;
            *qq = tv;
          }
      }
    grid.sync();
  }
  // forward substitution, column sweep (per element s ascending)
  for (int64_t s = 0; s + 1 < n; ++s) {
    const int64_t rows = n - s - 1;
    for (int64_t t = gw; t < nrhs * rows; t += NW) {
      const int64_t r = t / rows, i = s + 1 + (t - r * rows);
      sub_prod<V>(Y(r) + i * S, f + (i * n + s) * S, Y(r) + s * S, sh, sc);
    }
    grid.sync();
  }
  for (int64_t ii = n - 1; ii >= 0; --ii) {
    if (exact) {  // products of row ii, then the s-ascending chain
      const int64_t cnt = n - ii - 1;
      for (int64_t t = gw; t < nrhs * cnt; t += NW) {
        const int64_t r = t / cnt, s = ii + 1 + (t - r * cnt);
        W<V> u, xs, pr;
        load_w<V>(f + (ii * n + s) * S, u);
        load_w<V>(x + (r * n + s) * S, xs);
        mul_w<V>(u, xs, sh, sc, pr);
        store_w<V>(T(r) + s * S, pr);
      }
      if (cnt > 0) grid.sync();
    }
    for (int64_t r = gw; r < nrhs; r += NW) {
      W<V> acc, dd, q;
      load_w<V>(Y(r) + ii * S, acc);
      if (exact && ii + 1 < n) {  // the chain, with the next product loaded one step ahead
        W<V> nx;
        load_w<V>(T(r) + (ii + 1) * S, nx);
        for (int64_t s = ii + 1; s < n; ++s) {
          const W<V> pr = nx;
          if (s + 1 < n) load_w<V>(T(r) + (s + 1) * S, nx);
          add_w<V>(acc, pr, 1u, sh, acc);
        }
      }
      load_w<V>(f + (ii * n + ii) * S, dd);
      if (dd.e == EXP_ZERO) {
        if (lane == 0 && *zp == 0) *zp = ii + 1;
        zero_w<V>(q);
      } else {
        div_w<V>(acc, dd, sh, sc, q);
      }
      if (lane == 0 && exp_out_of_range(q.e)) atomicOr(err, ERR_EXP_RANGE);
      store_w<V>(x + (r * n + ii) * S, q);
    }
    grid.sync();
    if (*(volatile int64_t*)zp) return;
    if (!exact && ii > 0) {  // column-oriented: y_i -= RN(u_i,ii * x_ii), i < ii
      for (int64_t t = gw; t < nrhs * ii; t += NW) {
        const int64_t r = t / ii, i = t - r * ii;
        sub_prod<V>(Y(r) + i * S, f + (i * n + ii) * S, x + (r * n + ii) * S, sh, sc);
      }
      grid.sync();
    }
  }
}

template <int V>
void launch_lu_solve(const uint32_t* f, int64_t n, const int64_t* piv, const uint32_t* b, uint32_t* x,
                     uint32_t* scratch, int sh, uint32_t* err, int64_t* zp, int exact, int64_t nrhs,
                     cudaStream_t st) {
  const size_t smem = smem_bytes<V>();
  int grid = coop_grid(lu_solve_kernel<V>, smem, nrhs * n);
  void* args[] = {&f, &n, &piv, &b, &x, &scratch, (void*)&sh, &err, &zp, (void*)&exact, &nrhs};
  cudaLaunchCooperativeKernel((void*)lu_solve_kernel<V>, dim3((unsigned)grid), dim3(WNT), args, smem, st);
}

}  // namespace wmp
}  // namespace mpg
