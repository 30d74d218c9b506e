// capi.cu -- the extern "C" boundary (include/mpgpu.h) and the host-side driver:
// handle / memory management, the breadth-first Strassen / Winograd recursion
// driver (replacing fastmm.hpp:99-229's depth-first recursion), the op model and
// the seeded input generators.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <initializer_list>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/mpgpu.h"
#include "kernels.h"
#include "mp_arith.cuh"

// host-buffer LU (mpgpu_lu_blocked_host): hooks the factorisation calls so the PCIe
// transfers overlap it -- the operand arrives in two column blocks, the factored rows
// leave as soon as no later step touches them
struct LuHostIO {
  std::function<int()> before_panel0;  // columns [0, K) on the device
  std::function<int()> before_swap0;   // the whole matrix on the device
  std::function<int(int64_t, int64_t)> rows_final;  // rows [r0, r0 + nr) final
};

struct mpgpu_handle {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  uint32_t* d_err = nullptr;
  int64_t* d_piv = nullptr;
  int64_t d_piv_cap = 0;
  std::mutex mu;
  std::string last_error;
  cudaStream_t aux = nullptr;  // second stream of mpgpu_gemm_host (B's upload), lazily created
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // LU look-ahead: the next panel runs on a high-priority stream beside the Schur update
  cudaStream_t hi = nullptr;
  cudaEvent_t ev_la = nullptr, ev_lp = nullptr;
  // pipelined host GEMM: downloads on their own stream; per-quadrant events
  cudaStream_t dl = nullptr;
  cudaEvent_t pev[16] = {};
  LuHostIO* lu_io = nullptr;  // set by mpgpu_lu_blocked_host for the duration of the call
};

namespace {

using mpg::rec_stride;

int fail(mpgpu_handle* h, int code, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->last_error = buf;
  }
  return code;
}

#define CUDA_TRY(h, expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail((h), e_ == cudaErrorMemoryAllocation ? MPGPU_ERR_NOMEM : MPGPU_ERR_CUDA, \
                  "%s: %s", #expr, cudaGetErrorString(e_));                                 \
  } while (0)

constexpr int kLimbOptions[] = {1, 2, 4, 8, 16, 32, 64, 128, 256, 288};  // > 32: *_wide.cu

int nlimbs_for(int32_t prec) {
  if (prec < 2 || prec > MPGPU_MAX_STORE_PREC) return 0;
  const int need = (prec + 31) / 32;
  for (int L : kLimbOptions)
    if (L >= need) return L;
  return 0;
}

template <class F>
int dispatch_L(int L, F&& f) {
  switch (L) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 16: return f(std::integral_constant<int, 16>{});
    case 32: return f(std::integral_constant<int, 32>{});
    case 64: return f(std::integral_constant<int, 64>{});
    case 128: return f(std::integral_constant<int, 128>{});
    case 256: return f(std::integral_constant<int, 256>{});
    case 288: return f(std::integral_constant<int, 288>{});
    default: return MPGPU_ERR_DOMAIN;
  }
}

template <class F>
int dispatch_store(int L, F&& f) {
  return dispatch_L(L, std::forward<F>(f));
}

// RAII device scratch on the handle's stream (stream-ordered pool allocator)
struct DevBuf {
  mpgpu_handle* h = nullptr;
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t alloc(mpgpu_handle* hh, size_t bytes) {
    release();
    h = hh;
    return cudaMallocAsync(&p, bytes < 16 ? 16 : bytes, h->stream);
  }
  void release() {
    if (p) cudaFreeAsync(p, h->stream);
    p = nullptr;
  }
  uint32_t* u32() const { return static_cast<uint32_t*>(p); }
};

// Grow the device's stream-ordered pool (release threshold: keep everything) to at
// least `bytes` with one allocate/free pair, so later allocations of the call are
// sub-allocations of reserved memory.
int ensure_pool(mpgpu_handle* h, size_t bytes) {
  cudaMemPool_t pool;
  CUDA_TRY(h, cudaDeviceGetMemPool(&pool, h->device));
  uint64_t reserved = 0;
  CUDA_TRY(h, cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  if (reserved >= bytes) return MPGPU_OK;
  void* p = nullptr;
  CUDA_TRY(h, cudaMallocAsync(&p, bytes, h->stream));
  CUDA_TRY(h, cudaFreeAsync(p, h->stream));
  return MPGPU_OK;
}

// CUDA-event phase timers that never block: stop() records the end event and
// queues (start, end, destination); flush_timers() (called once per API call, at
// its final synchronisation) resolves every queued duration.  No host/GPU
// round trip inside a call, so phases run back to back on the GPU.
struct PendingTime {
  cudaEvent_t a, b;
  double* dst;
};
thread_local std::vector<PendingTime> g_pending;

void flush_timers() {
  for (auto& t : g_pending) {
    cudaEventSynchronize(t.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    if (t.dst) *t.dst = ms;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  g_pending.clear();
}

// error paths: drop queued timings without writing (their destinations may be gone)
struct TimerGuard {
  ~TimerGuard() {
    for (auto& t : g_pending) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    g_pending.clear();
  }
};

struct Timer {
  bool on;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Timer(bool enabled, cudaStream_t s) : on(enabled), st(s) {
    if (on) {
      cudaEventCreate(&a);
      cudaEventRecord(a, st);
    }
  }
  void stop(double* dst) {
    if (!on || !a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, st);
    g_pending.push_back({a, b, dst});
    a = nullptr;
  }
  ~Timer() {
    if (a) cudaEventDestroy(a);
  }
};

void count_fast_rec(int algo, int64_t m, int64_t l, int64_t n, int64_t n_min, uint64_t* out) {
  if (algo < MPGPU_STRASSEN || std::min({m, l, n}) <= n_min) {
    out[0] = (uint64_t)m * l * n;
    out[1] = (uint64_t)m * n * (l - 1);
    return;
  }
  const int64_t hm = (m + m % 2) / 2, hl = (l + l % 2) / 2, hn = (n + n % 2) / 2;
  uint64_t half[2];
  count_fast_rec(algo, hm, hl, hn, n_min, half);
  const uint64_t ka = algo == MPGPU_STRASSEN ? 5 : 4, kb = ka, kc = algo == MPGPU_STRASSEN ? 8 : 7;
  out[0] = 7 * half[0];
  out[1] = 7 * half[1] + ka * hm * hl + kb * hl * hn + kc * hm * hn;
}

struct Level {
  int64_t m, l, n;
};

// recursion_plan (fastmm.hpp:68-85): dims entering each level; last is the base case
std::vector<Level> plan_levels(int64_t m, int64_t l, int64_t n, int64_t n_min) {
  std::vector<Level> v;
  for (;;) {
    v.push_back({m, l, n});
    if (std::min({m, l, n}) <= n_min) return v;
    m = (m + m % 2) / 2;
    l = (l + l % 2) / 2;
    n = (n + n % 2) / 2;
  }
}

// ---- recursion depth per precision from measured leaf throughput (north star (2)) ----
// B200 measurements (tools/leaf_table.py -> profiles/r02_leaf_table_h.jsonl, re-measured with the carry-chained product and the fused two-level additions; the add rates are bytes of the one-launch-per-level model over the measured time): Winograd products with
// 7^d leaves of s^3 (s = 16 .. 512) per limb count; the leaf kernel's MP multiply-adds per second and
// the pre- / post-addition record bandwidth at that recursion level.  The leaf rate is flat for
// s >= 32 and drops ~15 % at s = 16; the additions run at 2-4.5 TB/s.
constexpr int kTabSizes = 6;
constexpr double kTabEdge[kTabSizes] = {16, 32, 64, 128, 256, 512};
struct LeafTab {
  int L;
  double rate[kTabSizes];  // leaf madd/s
  double pre[kTabSizes];   // pre-add GB/s (deepest level, node edge 2s)
  double post[kTabSizes];  // post-add GB/s
};
constexpr LeafTab kLeafTab[] = {
    {4, {1.393e11, 1.641e11, 1.614e11, 1.696e11, 1.689e11, 1.670e11}, {2974, 5778, 4445, 6385, 5959, 4318},
     {2330, 4924, 3903, 5798, 5187, 4909}},
    {8, {8.268e10, 9.487e10, 9.460e10, 9.782e10, 9.777e10, 9.765e10}, {2582, 5251, 4091, 5863, 5383, 4025},
     {2117, 4402, 3618, 5761, 5187, 4581}},
    {16, {3.663e10, 3.934e10, 3.904e10, 3.984e10, 3.977e10, 3.973e10}, {2958, 4880, 3882, 5241, 5179, 3499},
     {2560, 3994, 3134, 4878, 4613, 3922}},
    {32, {1.212e10, 1.270e10, 1.267e10, 1.287e10, 1.285e10, 1.284e10}, {2927, 4171, 3371, 4401, 4524, 3095},
     {2352, 3580, 3198, 4174, 3947, 3547}},
};

// table row for L (L < 4: the 128-bit row; L > 32: the 1024-bit row with the rate scaled by (32/L)^2)
const LeafTab& leaf_row(int L, double* rate_scale) {
  *rate_scale = 1.0;
  if (L <= 4) return kLeafTab[0];
  if (L <= 8) return kLeafTab[1];
  if (L <= 16) return kLeafTab[2];
  if (L > 32) *rate_scale = (32.0 / L) * (32.0 / L);
  return kLeafTab[3];
}

double interp_edge(const double (&v)[kTabSizes], double edge) {
  if (edge <= kTabEdge[0]) return v[0] * std::max(edge, 1.0) / kTabEdge[0];  // tiny leaves: idle threads
  if (edge >= kTabEdge[kTabSizes - 1]) return v[kTabSizes - 1];
  int i = 0;
  while (edge > kTabEdge[i + 1]) ++i;
  const double t = (std::log2(edge) - std::log2(kTabEdge[i])) / (std::log2(kTabEdge[i + 1]) - std::log2(kTabEdge[i]));
  return v[i] + t * (v[i + 1] - v[i]);
}

// modelled device time (ms) of fast_mul stopped at depth d, and the n_min giving that depth
double model_fast_ms(int L, int64_t m, int64_t l, int64_t n, int d, int64_t* n_min_out) {
  double scale;
  const LeafTab& row = leaf_row(L, &scale);
  const double rec = 4.0 * mpg::rec_stride(L);
  double ms = 0, nodes = 1;
  int64_t dm = m, dl = l, dn = n;
  for (int t = 0; t < d; ++t) {
    const int64_t hm = (dm + dm % 2) / 2, hl = (dl + dl % 2) / 2, hn = (dn + dn % 2) / 2;
    const double edge = std::cbrt((double)hm * hl * hn);
    // pre-add: read each parent operand, write 7 quarter-size children; post-add: read 7
    // children products, write the parent
    const double pre = nodes * (double)(dm * dl + dl * dn) * rec * (1.0 + 7.0 / 4.0);
    const double post = nodes * (double)(dm * dn) * rec * (1.0 + 7.0 / 4.0);
    ms += pre / (interp_edge(row.pre, edge) * 1e6) + post / (interp_edge(row.post, edge) * 1e6);
    nodes *= 7;
    dm = hm;
    dl = hl;
    dn = hn;
  }
  const double leaf_madds = nodes * (double)dm * dl * dn;
  ms += leaf_madds / (interp_edge(row.rate, std::cbrt((double)dm * dl * dn)) * scale) * 1e3;
  *n_min_out = std::min({dm, dl, dn});
  return ms;
}

int choose_nmin(int L, int64_t m, int64_t l, int64_t n, int64_t* n_min, int* depth, double* model_ms) {
  double best = 0;
  int64_t best_nmin = std::min({m, l, n});
  int best_d = 0;
  for (int d = 0; d <= 12; ++d) {
    int64_t nm = 0;
    // depth d exists only while every level-(d-1) dimension still exceeds the cutoff
    if (d > 0) {
      int64_t pm = m, pl = l, pn = n;
      for (int t = 0; t < d - 1; ++t) {
        pm = (pm + pm % 2) / 2;
        pl = (pl + pl % 2) / 2;
        pn = (pn + pn % 2) / 2;
      }
      if (std::min({pm, pl, pn}) < 2) break;
    }
    const double ms = model_fast_ms(L, m, l, n, d, &nm);
    if (d > 0 && plan_levels(m, l, n, nm).size() != (size_t)d + 1) break;  // cutoff cannot realise d
    if (d == 0 || ms < best) {
      best = ms;
      best_nmin = nm;
      best_d = d;
    }
  }
  if (n_min) *n_min = std::max<int64_t>(1, best_nmin);
  if (depth) *depth = best_d;
  if (model_ms) *model_ms = best;
  return MPGPU_OK;
}

// two recursion levels of pre-additions per launch (MPGPU_PREADD_FUSE=0 disables; =N: up to N limbs)
bool preadd_fuse_for(int L) {
  static const int maxl = [] {
    const char* e = std::getenv("MPGPU_PREADD_FUSE");
    return e ? std::atoi(e) : 32;
  }();
  return L <= maxl;
}

int check_err(mpgpu_handle* h) {
  flush_timers();
  uint32_t e = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&e, h->d_err, sizeof e, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaGetLastError());
  if (e & mpg::ERR_DIV_ZERO) return fail(h, MPGPU_ERR_SINGULAR, "division by zero");
  if (e & mpg::ERR_EXP_RANGE)
    return fail(h, MPGPU_ERR_DOMAIN, "exponent outside MPFR's default range (overflow/underflow)");
  return MPGPU_OK;
}

// ---------------------------------------------------------------------------
// GEMM driver.  Simple / Block: one leaf launch.  Strassen / Winograd: breadth-
// first over the recursion levels -- per level one fused pre-add launch per operand
// side over all 7^lev nodes, then ONE batched leaf GEMM over all 7^d leaves, then
// one fused post-add launch per level back up.  Same operation DAG as the
// reference's depth-first recursion, so the result is bit-identical.
// ---------------------------------------------------------------------------
// scratch the breadth-first driver may hold at once: MPGPU_BFS_BUDGET_MB, else 60 % of the
// device's memory; deeper recursions run their top levels depth-first (run_gemm_chunked)
size_t bfs_budget(mpgpu_handle* h) {
  if (const char* e = std::getenv("MPGPU_BFS_BUDGET_MB")) return (size_t)std::atoll(e) << 20;
  static size_t total = [] {
    size_t f = 0, t = 0;
    if (cudaMemGetInfo(&f, &t) != cudaSuccess) {
      cudaGetLastError();
      t = (size_t)80 << 30;
    }
    return t;
  }();
  (void)h;
  return total / 10 * 6;
}

template <int L>
int run_gemm(mpgpu_handle* h, int algo, int64_t param, const uint32_t* A, int64_t lda, const uint32_t* B,
             int64_t ldb, uint32_t* C, int64_t ldc, int64_t m, int64_t l, int64_t n, int sh,
             mpgpu_stats* stats, int sub_from_c, cudaEvent_t b_ready = nullptr);

// One recursion level run explicitly, its 7 products by run_gemm one after another: the same
// operation DAG as the breadth-first driver (every node's pre-additions, product and
// post-additions are unchanged -- only the order nodes are visited differs), so the result is
// bit-identical, with the scratch of one subtree at a time instead of the whole level.
template <int L>
int run_gemm_chunked(mpgpu_handle* h, int algo, int64_t param, const uint32_t* A, int64_t lda, const uint32_t* B,
                     int64_t ldb, uint32_t* C, int64_t ldc, int64_t m, int64_t l, int64_t n, int sh,
                     mpgpu_stats* stats, cudaEvent_t b_ready) {
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  const bool timing = stats != nullptr;
  if (b_ready) cudaStreamWaitEvent(st, b_ready, 0);
  Timer total(timing, st);
  int launches = 0;
  DevBuf a0, b0, top;
  const uint32_t* pa = A;
  const uint32_t* pb = B;
  if (lda != l) {
    CUDA_TRY(h, a0.alloc(h, sizeof(uint32_t) * S * m * l));
    mpg::launch_copy2d<L>(A, lda, a0.u32(), l, (int)m, (int)l, st);
    ++launches;
    pa = a0.u32();
  }
  if (ldb != n) {
    CUDA_TRY(h, b0.alloc(h, sizeof(uint32_t) * S * l * n));
    mpg::launch_copy2d<L>(B, ldb, b0.u32(), n, (int)l, (int)n, st);
    ++launches;
    pb = b0.u32();
  }
  const int64_t hm = (m + m % 2) / 2, hl = (l + l % 2) / 2, hn = (n + n % 2) / 2;
  DevBuf a1, b1, p1;
  CUDA_TRY(h, a1.alloc(h, sizeof(uint32_t) * S * 7 * hm * hl));
  CUDA_TRY(h, b1.alloc(h, sizeof(uint32_t) * S * 7 * hl * hn));
  CUDA_TRY(h, p1.alloc(h, sizeof(uint32_t) * S * 7 * hm * hn));
  double pre_top = 0, post_top = 0;
  {
    Timer tp(timing, st);
    mpg::launch_preadd<L>(algo, 0, pa, 1, (int)m, (int)l, a1.u32(), sh, h->d_err, st);
    mpg::launch_preadd<L>(algo, 1, pb, 1, (int)l, (int)n, b1.u32(), sh, h->d_err, st);
    launches += 2;
    if (stats) tp.stop(&pre_top);
  }
  a0.release();
  b0.release();
  mpgpu_stats sum{};
  for (int q = 0; q < 7; ++q) {
    mpgpu_stats cs{};
    int rc = run_gemm<L>(h, algo, param, a1.u32() + q * hm * hl * S, hl, b1.u32() + q * hl * hn * S, hn,
                         p1.u32() + q * hm * hn * S, hn, hm, hl, hn, sh, stats ? &cs : nullptr, 0, nullptr);
    if (rc) return rc;
    if (stats) {
      flush_timers();  // resolve the child's phase times now (cs is local)
      sum.leaf_ms += cs.leaf_ms;
      sum.preadd_ms += cs.preadd_ms;
      sum.postadd_ms += cs.postadd_ms;
      sum.leaf_madds += cs.leaf_madds;
      sum.depth = cs.depth;
    }
    launches += cs.launches;
  }
  a1.release();
  b1.release();
  {
    Timer tq(timing, st);
    uint32_t* dst = C;
    if (ldc != n) {
      CUDA_TRY(h, top.alloc(h, sizeof(uint32_t) * S * m * n));
      dst = top.u32();
    }
    mpg::launch_postadd<L>(algo, p1.u32(), 1, (int)m, (int)n, dst, nullptr, sh, h->d_err, st);
    ++launches;
    if (top.p) {
      mpg::launch_copy2d<L>(top.u32(), n, C, ldc, (int)m, (int)n, st);
      ++launches;
    }
    if (stats) tq.stop(&post_top);
  }
  if (stats) {
    total.stop(&stats->device_ms);
    flush_timers();
    stats->leaf_ms = sum.leaf_ms;
    stats->leaf_madds = sum.leaf_madds;
    stats->preadd_ms = sum.preadd_ms + pre_top;
    stats->postadd_ms = sum.postadd_ms + post_top;
    stats->depth = sum.depth + 1;
    stats->launches = launches;
  }
  return MPGPU_OK;
}

template <int L>
int run_gemm(mpgpu_handle* h, int algo, int64_t param, const uint32_t* A, int64_t lda, const uint32_t* B,
             int64_t ldb, uint32_t* C, int64_t ldc, int64_t m, int64_t l, int64_t n, int sh,
             mpgpu_stats* stats, int sub_from_c, cudaEvent_t b_ready) {
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  const bool timing = stats != nullptr;
  if (algo == MPGPU_STRASSEN || algo == MPGPU_WINOGRAD) {
    // grow the stream-ordered pool to the call's peak scratch once, before any timer:
    // otherwise the first large call maps pages between its phases
    const std::vector<Level> pl = plan_levels(m, l, n, param);
    const size_t rec = sizeof(uint32_t) * S;
    size_t peak = 0, nodes = 1, prevA = 0, prevB = 0;
    std::vector<size_t> prodsz(pl.size(), 0);
    for (size_t lev = 0; lev + 1 < pl.size(); ++lev) {
      nodes *= 7;
      const size_t a = rec * nodes * pl[lev + 1].m * pl[lev + 1].l, b = rec * nodes * pl[lev + 1].l * pl[lev + 1].n;
      peak = std::max(peak, prevA + prevB + a + b);
      prevA = a;
      prevB = b;
      prodsz[lev + 1] = rec * nodes * pl[lev + 1].m * pl[lev + 1].n;
    }
    if (pl.size() > 1) {
      peak = std::max(peak, prevA + prevB + prodsz.back());
      for (size_t lev = pl.size() - 1; lev >= 2; --lev) peak = std::max(peak, prodsz[lev] + prodsz[lev - 1]);
      peak += rec * (size_t)(m * l + l * n + m * n);  // dense copies / top buffer, if needed
      if (peak > bfs_budget(h) && pl.size() >= 3 && !sub_from_c)
        return run_gemm_chunked<L>(h, algo, param, A, lda, B, ldb, C, ldc, m, l, n, sh, stats, b_ready);
      int rc = ensure_pool(h, peak + peak / 8);
      if (rc) return rc;
    }
  }
  Timer total(timing, st);
  int launches = 0;
  auto leaf = [&](const uint32_t* a, int64_t la, const uint32_t* b, int64_t lb, uint32_t* c, int64_t lc,
                  int64_t mm, int64_t ll, int64_t nn, int64_t kb, int batch, int subc) {
    mpg::GemmArgs g{};
    g.A = a;
    g.B = b;
    g.C = c;
    g.strideA = mm * ll;
    g.strideB = ll * nn;
    g.strideC = mm * nn;
    g.lda = la;
    g.ldb = lb;
    g.ldc = lc;
    g.m = (int)mm;
    g.l = (int)ll;
    g.n = (int)nn;
    g.kb = (int)std::min<int64_t>(kb, ll);
    g.batch = batch;
    g.sh = sh;
    g.err = h->d_err;
    g.sub_from_c = subc;
    mpg::launch_gemm<L>(g, st);
    ++launches;
  };
  if (stats) stats->depth = 0;
  // b_ready (mpgpu_gemm_host): B is still being uploaded on another stream -- the A-side
  // work runs first and the B side waits for the event
  auto wait_b = [&]() {
    if (b_ready) cudaStreamWaitEvent(st, b_ready, 0);
  };
  if (algo == MPGPU_SIMPLE || algo == MPGPU_BLOCK) {
    wait_b();
    Timer tl(timing, st);
    leaf(A, lda, B, ldb, C, ldc, m, l, n, algo == MPGPU_SIMPLE ? l : param, 1, sub_from_c);
    if (stats) {
      tl.stop(&stats->leaf_ms);
      stats->leaf_madds = (uint64_t)m * l * n;
    }
  } else {
    const std::vector<Level> lv = plan_levels(m, l, n, param);
    const int d = (int)lv.size() - 1;
    if (stats) stats->depth = d;
    if (d == 0) {
      wait_b();
      Timer tl(timing, st);
      leaf(A, lda, B, ldb, C, ldc, m, l, n, l, 1, sub_from_c);
      if (stats) {
        tl.stop(&stats->leaf_ms);
        stats->leaf_madds = (uint64_t)m * l * n;
      }
    } else {
      // level 0 operands must be dense for the pre-add kernel
      DevBuf a0, b0;
      const uint32_t* pa = A;
      const uint32_t* pb = B;
      if (lda != l) {
        CUDA_TRY(h, a0.alloc(h, sizeof(uint32_t) * S * m * l));
        mpg::launch_copy2d<L>(A, lda, a0.u32(), l, (int)m, (int)l, st);
        ++launches;
        pa = a0.u32();
      }
      if (ldb != n) {
        wait_b();
        CUDA_TRY(h, b0.alloc(h, sizeof(uint32_t) * S * l * n));
        mpg::launch_copy2d<L>(B, ldb, b0.u32(), n, (int)l, (int)n, st);
        ++launches;
        pb = b0.u32();
      }
      std::vector<DevBuf> opA(d + 1), opB(d + 1), prod(d + 1);
      Timer tpre(timing, st);
      int64_t nodes = 1;
      // the pre-additions of one side never read the other's: with b_ready all A levels
      // run first (overlapping B's upload), else the sides interleave level by level
      auto side_level = [&](int side, int lev, int64_t nd) -> int {
        const Level& P = lv[lev];
        const Level& Q = lv[lev + 1];
        std::vector<DevBuf>& op = side == 0 ? opA : opB;
        const uint32_t* src = lev == 0 ? (side == 0 ? pa : pb) : op[lev].u32();
        const int64_t rr = side == 0 ? P.m : P.l, cc = side == 0 ? P.l : P.n;
        const int64_t qr = side == 0 ? Q.m : Q.l, qc = side == 0 ? Q.l : Q.n;
        CUDA_TRY(h, op[lev + 1].alloc(h, sizeof(uint32_t) * S * nd * 7 * qr * qc));
        mpg::launch_preadd<L>(algo, side, src, nd, (int)rr, (int)cc, op[lev + 1].u32(), sh, h->d_err, st);
        ++launches;
        if (lev > 0) op[lev].release();
        return 0;
      };
      // two levels per launch where the fused kernel exists (the intermediate level -- 7/4 of
      // the parents written and read back -- stays in shared memory; same operands bit for bit)
      auto side_level2 = [&](int side, int lev, int64_t nd) -> int {
        const Level& P = lv[lev];
        const Level& Q = lv[lev + 2];
        std::vector<DevBuf>& op = side == 0 ? opA : opB;
        const uint32_t* src = lev == 0 ? (side == 0 ? pa : pb) : op[lev].u32();
        const int64_t rr = side == 0 ? P.m : P.l, cc = side == 0 ? P.l : P.n;
        const int64_t qr = side == 0 ? Q.m : Q.l, qc = side == 0 ? Q.l : Q.n;
        CUDA_TRY(h, op[lev + 2].alloc(h, sizeof(uint32_t) * S * nd * 49 * qr * qc));
        if (!mpg::launch_preadd2<L>(algo, side, src, nd, (int)rr, (int)cc, op[lev + 2].u32(), sh, st)) return -1;
        ++launches;
        if (lev > 0) op[lev].release();
        return 0;
      };
      auto side_all = [&](int side) -> int {
        int64_t nd = 1;
        for (int lev = 0; lev < d;) {
          // an odd number of levels: the single one first (the deepest levels move the most bytes)
          if (preadd_fuse_for(L) && lev + 2 <= d && (d - lev) % 2 == 0) {
            const int rc = side_level2(side, lev, nd);
            if (rc > 0) return rc;
            if (rc == 0) {
              lev += 2;
              nd *= 49;
              continue;
            }
            (side == 0 ? opA : opB)[lev + 2].release();  // no fused kernel for this limb count
          }
          if (int rc = side_level(side, lev, nd)) return rc;
          lev += 1;
          nd *= 7;
        }
        return 0;
      };
      // the pre-additions of one side never read the other's: all A levels run first
      // (overlapping B's upload when b_ready is set)
      if (int rc = side_all(0)) return rc;
      wait_b();
      if (int rc = side_all(1)) return rc;
      for (int lev = 0; lev < d; ++lev) nodes *= 7;
      a0.release();
      b0.release();
      if (stats) tpre.stop(&stats->preadd_ms);
      const Level& D = lv[d];
      CUDA_TRY(h, prod[d].alloc(h, sizeof(uint32_t) * S * nodes * D.m * D.n));
      {
        Timer tl(timing, st);
        leaf(opA[d].u32(), D.l, opB[d].u32(), D.n, prod[d].u32(), D.n, D.m, D.l, D.n, D.l, (int)nodes, 0);
        if (stats) {
          tl.stop(&stats->leaf_ms);
          stats->leaf_madds = (uint64_t)nodes * D.m * D.l * D.n;
        }
      }
      opA[d].release();
      opB[d].release();
      Timer tpost(timing, st);
      DevBuf top;
      for (int lev = d - 1; lev >= 0;) {
        // two levels per launch where the fused kernel exists: the products of level lev + 1
        // combined straight into level lev - 1 (the level between them stays in shared memory)
        const bool two = lev >= 1 && preadd_fuse_for(L) && mpg::has_postadd2(L);
        const int tl = two ? lev - 1 : lev;
        nodes /= two ? 49 : 7;
        const Level& P = lv[tl];
        uint32_t* dst;
        if (tl == 0 && ldc == n && !sub_from_c) {
          dst = C;
        } else if (tl == 0) {
          CUDA_TRY(h, top.alloc(h, sizeof(uint32_t) * S * m * n));
          dst = top.u32();
        } else {
          CUDA_TRY(h, prod[tl].alloc(h, sizeof(uint32_t) * S * nodes * P.m * P.n));
          dst = prod[tl].u32();
        }
        if (two) {
          if (!mpg::launch_postadd2<L>(algo, prod[lev + 1].u32(), nodes, (int)P.m, (int)P.n, dst, sh, h->d_err, st))
            return fail(h, MPGPU_ERR_DOMAIN, "internal: no fused post-addition for this limb count");
        } else {
          mpg::launch_postadd<L>(algo, prod[lev + 1].u32(), nodes, (int)P.m, (int)P.n, dst, nullptr, sh,
                                 h->d_err, st);
        }
        ++launches;
        prod[lev + 1].release();
        lev = tl - 1;
      }
      if (top.p) {
        if (sub_from_c) {
          return fail(h, MPGPU_ERR_DOMAIN, "internal: strided fast Schur epilogue not routed here");
        }
        mpg::launch_copy2d<L>(top.u32(), n, C, ldc, (int)m, (int)n, st);
        ++launches;
      }
      if (stats) tpost.stop(&stats->postadd_ms);
    }
  }
  if (stats) {
    total.stop(&stats->device_ms);
    stats->launches = launches;
  }
  return MPGPU_OK;
}

// ---------------------------------------------------------------------------
// Leaf-sharded fast multiply (multi-GPU building blocks).  Leaves are numbered in
// the BFS order of run_gemm (child c of node p is 7p + c).  run_fast_leaves
// computes the products of leaves [lo, hi) into `out` (leaf-major, m_d x n_d
// records each), running at every level only the pre-additions of the ancestors of
// those leaves; run_fast_combine runs all post-addition levels from the full set of
// leaf products.  Together they reproduce run_gemm bit for bit.
// ---------------------------------------------------------------------------
template <int L>
int run_fast_leaves(mpgpu_handle* h, int algo, int64_t n_min, const uint32_t* A, int64_t lda, const uint32_t* B,
                    int64_t ldb, int64_t m, int64_t l, int64_t n, int64_t ulo, int64_t uhi, int up_levels,
                    uint32_t* out, int sh, mpgpu_stats* stats, const uint64_t* rowtab = nullptr,
                    const uint32_t* l1A = nullptr, const uint32_t* l1B = nullptr) {
  // l1A / l1B (optional): the 7 level-1 operands of each side already formed (dense, child
  // slot c at c * m1 * l1 / l1 * n1 records) -- the level-0 pre-additions are skipped
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  const bool timing = stats != nullptr;
  Timer total(timing, st);
  const std::vector<Level> lv = plan_levels(m, l, n, n_min);
  const int d = (int)lv.size() - 1;
  if (d == 0) return fail(h, MPGPU_ERR_DOMAIN, "fast_leaves: the product is a base case (depth 0)");
  if (up_levels < 0 || up_levels > d) return fail(h, MPGPU_ERR_DIMENSION, "fast_leaves: bad output level");
  const int ol = d - up_levels;  // level of the output nodes
  if (l1A && ol < 1) return fail(h, MPGPU_ERR_DIMENSION, "fast_leaves: level-1 operands need units below the top");
  int64_t units = 1, span = 1;  // nodes at level ol; leaves per unit
  for (int i = 0; i < ol; ++i) units *= 7;
  for (int i = 0; i < up_levels; ++i) span *= 7;
  if (ulo < 0 || uhi > units || ulo >= uhi) return fail(h, MPGPU_ERR_DIMENSION, "fast_leaves: bad node range");
  const int64_t lo = ulo * span, hi = uhi * span;
  int launches = 0;
  // node range needed at each level: level lev covers [s[lev], e[lev])
  std::vector<int64_t> s(d + 1), e(d + 1);
  s[d] = lo;
  e[d] = hi;
  for (int lev = d - 1; lev >= 0; --lev) {
    s[lev] = s[lev + 1] / 7;
    e[lev] = (e[lev + 1] + 6) / 7;
  }
  DevBuf a0, b0;
  const uint32_t* pa = A;
  const uint32_t* pb = B;
  if (lda != l && !l1A) {
    CUDA_TRY(h, a0.alloc(h, sizeof(uint32_t) * S * m * l));
    mpg::launch_copy2d<L>(A, lda, a0.u32(), l, (int)m, (int)l, st);
    pa = a0.u32();
  }
  if (ldb != n && !l1A) {
    CUDA_TRY(h, b0.alloc(h, sizeof(uint32_t) * S * l * n));
    mpg::launch_copy2d<L>(B, ldb, b0.u32(), n, (int)l, (int)n, st);
    pb = b0.u32();
  }
  // buffers: level lev holds nodes [bs[lev], bs[lev] + bn[lev])
  std::vector<DevBuf> opA(d + 1), opB(d + 1);
  std::vector<int64_t> bs(d + 1), bn(d + 1);
  bs[0] = 0;
  bn[0] = 1;
  auto bufA = [&](int lev) -> const uint32_t* { return (lev == 1 && l1A) ? l1A : opA[lev].u32(); };
  auto bufB = [&](int lev) -> const uint32_t* { return (lev == 1 && l1A) ? l1B : opB[lev].u32(); };
  if (l1A) {
    bs[1] = 0;
    bn[1] = 7;
  }
  Timer tpre(timing, st);
  for (int lev = l1A ? 1 : 0; lev < d; ++lev) {
    const Level& P = lv[lev];
    const Level& Q = lv[lev + 1];
    const int64_t p0 = s[lev], np = e[lev] - s[lev];
    const uint32_t* srcA = lev == 0 ? pa : bufA(lev) + (p0 - bs[lev]) * P.m * P.l * S;
    const uint32_t* srcB = lev == 0 ? pb : bufB(lev) + (p0 - bs[lev]) * P.l * P.n * S;
    bs[lev + 1] = 7 * p0;
    bn[lev + 1] = 7 * np;
    CUDA_TRY(h, opA[lev + 1].alloc(h, sizeof(uint32_t) * S * bn[lev + 1] * Q.m * Q.l));
    CUDA_TRY(h, opB[lev + 1].alloc(h, sizeof(uint32_t) * S * bn[lev + 1] * Q.l * Q.n));
    mpg::launch_preadd<L>(algo, 0, srcA, np, (int)P.m, (int)P.l, opA[lev + 1].u32(), sh, h->d_err, st);
    mpg::launch_preadd<L>(algo, 1, srcB, np, (int)P.l, (int)P.n, opB[lev + 1].u32(), sh, h->d_err, st);
    launches += 2;
    if (lev > 0) {
      opA[lev].release();
      opB[lev].release();
    }
  }
  if (stats) tpre.stop(&stats->preadd_ms);
  const Level& D = lv[d];
  {
    Timer tl(timing, st);
    mpg::GemmArgs g{};
    g.A = bufA(d) + (lo - bs[d]) * D.m * D.l * S;
    g.B = bufB(d) + (lo - bs[d]) * D.l * D.n * S;
    DevBuf leafbuf;
    if (up_levels == 0) {
      g.C = out;
      g.rowtab = rowtab;  // (fused exchange: rows straight to their owners)
    } else {
      CUDA_TRY(h, leafbuf.alloc(h, sizeof(uint32_t) * S * (hi - lo) * D.m * D.n));
      g.C = leafbuf.u32();
    }
    g.strideA = D.m * D.l;
    g.strideB = D.l * D.n;
    g.strideC = D.m * D.n;
    g.lda = D.l;
    g.ldb = D.n;
    g.ldc = D.n;
    g.m = (int)D.m;
    g.l = (int)D.l;
    g.n = (int)D.n;
    g.kb = (int)D.l;
    g.batch = (int)(hi - lo);
    g.sh = sh;
    g.err = h->d_err;
    mpg::launch_gemm<L>(g, st);
    ++launches;
    if (stats) {
      tl.stop(&stats->leaf_ms);
      stats->leaf_madds = (uint64_t)(hi - lo) * D.m * D.l * D.n;
    }
    opA[d].release();
    opB[d].release();
    // local post-additions up to level ol for the owned (whole) subtrees
    Timer tpost(timing, st);
    DevBuf cur_owner;
    const uint32_t* cur = leafbuf.u32();
    int64_t nodes = hi - lo;
    for (int k = 0; k < up_levels; ++k) {
      nodes /= 7;
      const Level& P = lv[d - 1 - k];
      uint32_t* dst;
      DevBuf next;
      if (k == up_levels - 1) {
        dst = out;
      } else {
        CUDA_TRY(h, next.alloc(h, sizeof(uint32_t) * S * nodes * P.m * P.n));
        dst = next.u32();
      }
      mpg::launch_postadd<L>(algo, cur, nodes, (int)P.m, (int)P.n, dst, nullptr, sh, h->d_err, st, nullptr, 0, 0,
                             -1, k == up_levels - 1 ? rowtab : nullptr);
      ++launches;
      if (k == 0) leafbuf.release();
      cur_owner.release();
      if (k != up_levels - 1) {
        std::swap(cur_owner.p, next.p);
        cur_owner.h = h;
        cur = cur_owner.u32();
      }
    }
    if (stats) tpost.stop(&stats->postadd_ms);
  }
  if (stats) {
    total.stop(&stats->device_ms);
    stats->launches = launches;
    stats->depth = d;
  }
  return MPGPU_OK;
}

// Rows of each level's node products produced from the unit-level rows [lo, hi) (the
// row-owned combine): a level-t row r comes from child row r (top quadrants) or
// r - m_{t+1} (bottom), so ownership propagates up through the pad/halve index map.
// owned[t] lists the owned rows of a level-t node, t = 0 .. il.
std::vector<std::vector<int>> owned_rows(const std::vector<Level>& lv, int il, int64_t lo, int64_t hi) {
  std::vector<std::vector<int>> owned(il + 1);
  for (int64_t r = lo; r < hi && r < lv[il].m; ++r) owned[il].push_back((int)r);
  for (int t = il - 1; t >= 0; --t) {
    const int64_t hm = lv[t + 1].m;
    std::vector<char> mark(lv[t].m, 0);
    for (int rc : owned[t + 1]) {
      if (rc < lv[t].m) mark[rc] = 1;
      if (rc + hm < lv[t].m) mark[rc + hm] = 1;
    }
    for (int64_t r = 0; r < lv[t].m; ++r)
      if (mark[r]) owned[t].push_back((int)r);
  }
  return owned;
}

template <int L>
int run_fast_combine(mpgpu_handle* h, int algo, int64_t n_min, const uint32_t* leafprods, int in_up, int64_t m,
                     int64_t l, int64_t n, uint32_t* C, int64_t ldc, int sh, mpgpu_stats* stats, int64_t row_lo = 0,
                     int64_t row_hi = -1) {
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  Timer tpost(stats != nullptr, st);
  const std::vector<Level> lv = plan_levels(m, l, n, n_min);
  const int d = (int)lv.size() - 1;
  if (d == 0) return fail(h, MPGPU_ERR_DOMAIN, "fast_combine: the product is a base case (depth 0)");
  if (in_up < 0 || in_up >= d) return fail(h, MPGPU_ERR_DIMENSION, "fast_combine: bad input level");
  const int il = d - in_up;  // level of the given node products
  if (row_hi < 0) row_hi = lv[il].m;
  if (row_lo < 0 || row_lo > row_hi || row_hi > lv[il].m)
    return fail(h, MPGPU_ERR_DIMENSION, "fast_combine: bad unit row range");
  const bool partial = row_lo > 0 || row_hi < lv[il].m;
  // device lists of the owned child rows per level (row-owned combine only)
  std::vector<DevBuf> rowbuf(il + 1);
  std::vector<int> nrows(il + 1, 0);
  if (partial) {
    const auto owned = owned_rows(lv, il, row_lo, row_hi);
    for (int t = 1; t <= il; ++t) {
      nrows[t] = (int)owned[t].size();
      CUDA_TRY(h, rowbuf[t].alloc(h, sizeof(int) * (owned[t].size() + 1)));
      if (!owned[t].empty())
        CUDA_TRY(h, cudaMemcpyAsync(rowbuf[t].p, owned[t].data(), sizeof(int) * owned[t].size(),
                                    cudaMemcpyHostToDevice, st));
    }
  }
  int64_t nodes = 1;
  for (int i = 0; i < il; ++i) nodes *= 7;
  std::vector<DevBuf> prod(d + 1);
  const uint32_t* cur = leafprods;
  DevBuf top;
  int launches = 0;
  for (int lev = il - 1; lev >= 0; --lev) {
    nodes /= 7;
    const Level& P = lv[lev];
    uint32_t* dst;
    if (lev == 0 && ldc == n) {
      dst = C;
    } else if (lev == 0) {
      CUDA_TRY(h, top.alloc(h, sizeof(uint32_t) * S * m * n));
      dst = top.u32();
    } else {
      CUDA_TRY(h, prod[lev].alloc(h, sizeof(uint32_t) * S * nodes * P.m * P.n));
      dst = prod[lev].u32();
    }
    mpg::launch_postadd<L>(algo, cur, nodes, (int)P.m, (int)P.n, dst, nullptr, sh, h->d_err, st,
                           partial ? static_cast<const int*>(rowbuf[lev + 1].p) : nullptr, nrows[lev + 1]);
    ++launches;
    if (lev + 1 < il) prod[lev + 1].release();
    cur = dst;
  }
  if (top.p) {  // (a strided C: copy the whole window -- rows not owned are copied unset)
    mpg::launch_copy2d<L>(top.u32(), n, C, ldc, (int)m, (int)n, st);
    ++launches;
  }
  if (stats) {
    tpost.stop(&stats->postadd_ms);
    stats->device_ms = stats->postadd_ms;
    stats->launches = launches;
    stats->depth = d;
  }
  return MPGPU_OK;
}

// arithmetic entry points: every supported limb count has kernels
int compute_range(mpgpu_handle* h, std::initializer_list<const mpgpu_mat*> ms) {
  for (const mpgpu_mat* m : ms)
    if (m && m->prec > MPGPU_MAX_PREC)
      return fail(h, MPGPU_ERR_DOMAIN, "precision %d above %d bits", m->prec, MPGPU_MAX_PREC);
  return MPGPU_OK;
}

int validate_gemm(mpgpu_handle* h, int algo, int64_t param, const mpgpu_mat* A, const mpgpu_mat* B,
                  const mpgpu_mat* C) {
  if (!A || !B || !C) return fail(h, MPGPU_ERR_DIMENSION, "null matrix");
  if (A->cols != B->rows)
    return fail(h, MPGPU_ERR_DIMENSION, "inner dimension mismatch: %lld vs %lld", (long long)A->cols,
                (long long)B->rows);
  if ((algo == MPGPU_BLOCK || algo == MPGPU_STRASSEN || algo == MPGPU_WINOGRAD) && param == 0)
    return fail(h, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (algo < MPGPU_SIMPLE || algo > MPGPU_WINOGRAD || param < 0)
    return fail(h, MPGPU_ERR_DOMAIN, "unknown algorithm %d", algo);
  if (C->rows != A->rows || C->cols != B->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "output shape mismatch");
  if (A->prec != C->prec || B->prec != C->prec || A->nlimbs != C->nlimbs || B->nlimbs != C->nlimbs)
    return fail(h, MPGPU_ERR_DOMAIN, "device GEMM requires one precision for A, B and C");
  return compute_range(h, {A, B, C});
}

// ---- host generators -----------------------------------------------------
struct Prng64 {  // xorshift64* (matgen.hpp:13-42)
  uint64_t s;
  explicit Prng64(uint64_t seed) : s(seed ? seed : 0x9E3779B97F4A7C15ULL) {}
  uint64_t next64() {
    uint64_t x = s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    s = x;
    return x * 2685821657736338717ULL;
  }
  uint64_t top53() { return next64() >> 11; }
};

// big integer (little-endian 32-bit words) helpers
struct BitWriter {  // MSB-first bit stream into a big integer of `total` bits
  std::vector<uint32_t> w;
  int total, pos = 0;  // pos = bits written
  explicit BitWriter(int bits) : w((bits + 31) / 32 + 1, 0), total(bits) {}
  void put(uint64_t bits, int nb) {  // append nb (<= 53) bits, MSB first
    for (int i = nb - 1; i >= 0;) {
      // bit index from the LSB of the whole number
      const int idx = total - 1 - pos;
      const int word = idx >> 5, bit = idx & 31;
      const int room = bit + 1;  // bits available in this word at and below `bit`
      const int take = std::min(room, i + 1);
      const uint32_t chunk = (uint32_t)((bits >> (i + 1 - take)) & ((1ull << take) - 1));
      w[word] |= chunk << (bit + 1 - take);
      pos += take;
      i -= take;
    }
  }
};

// write a nonzero magnitude (big int, little-endian words, bit length b) as a
// left-aligned L-limb mantissa; returns false if it would need rounding
void put_mantissa(const std::vector<uint32_t>& v, int b, int Lh, int64_t N, int64_t e, uint32_t* limbs) {
  // shift left so that bit (b-1) lands at bit (32*Lh - 1)
  const int shift = 32 * Lh - b;  // may be negative only if b > 32*Lh (not for our inputs)
  for (int k = 0; k < Lh; ++k) {
    // output word k covers bits [32k, 32k+32) of (v << shift)
    uint64_t acc = 0;
    const int lo = 32 * k - shift;  // source bit index of output bit 32k
    for (int t = 0; t < 32; ++t) {
      const int sb = lo + t;
      if (sb >= 0 && sb < (int)v.size() * 32) acc |= (uint64_t)((v[sb >> 5] >> (sb & 31)) & 1u) << t;
    }
    limbs[(int64_t)k * N + e] = (uint32_t)acc;
  }
}

int bitlen(const std::vector<uint32_t>& v) {
  for (int k = (int)v.size() - 1; k >= 0; --k)
    if (v[k]) return 32 * k + 32 - __builtin_clz(v[k]);
  return 0;
}

}  // namespace

// host SoA -> device records (stream-ordered, no sync); stage is scratch owned by the caller
// host SoA planes -> staging (H2D on `st`) -> device records; `copied` (optional) is
// recorded on `st` once the host bytes are across
// host SoA planes (plane j of the host matrix starts hstride elements after plane j-1;
// hstride == N for a dense host matrix) -> staging (H2D on `st`) -> device records;
// `copied` (optional) is recorded on `st` once the host bytes are across
int upload_async_to(mpgpu_handle* h, uint32_t* rec, int L, int64_t N, const uint32_t* limbs, const int32_t* exp,
                    const uint8_t* sign, int32_t Lh, uint32_t* stage, cudaStream_t st, cudaEvent_t copied = nullptr,
                    int64_t hstride = -1) {
  if (hstride < 0) hstride = N;
  uint32_t* dl = stage;
  int32_t* de = reinterpret_cast<int32_t*>(dl + (size_t)L * N);
  uint8_t* ds = reinterpret_cast<uint8_t*>(de + N);
  // most significant limbs aligned: host plane j <-> device plane j + (L - Lh)
  const int np = Lh <= L ? Lh : L;
  uint32_t* dst0 = Lh <= L ? dl + (size_t)(L - Lh) * N : dl;
  const uint32_t* src0 = Lh <= L ? limbs : limbs + (size_t)(Lh - L) * hstride;
  if (Lh < L) CUDA_TRY(h, cudaMemsetAsync(dl, 0, sizeof(uint32_t) * (size_t)(L - Lh) * N, st));
  if (hstride == N)
    CUDA_TRY(h, cudaMemcpyAsync(dst0, src0, sizeof(uint32_t) * (size_t)np * N, cudaMemcpyHostToDevice, st));
  else
    CUDA_TRY(h, cudaMemcpy2DAsync(dst0, sizeof(uint32_t) * N, src0, sizeof(uint32_t) * hstride, sizeof(uint32_t) * N,
                                  np, cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaMemcpyAsync(de, exp, sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaMemcpyAsync(ds, sign, N, cudaMemcpyHostToDevice, st));
  if (copied) CUDA_TRY(h, cudaEventRecord(copied, st));
  dispatch_store(L, [&](auto Lc) {
    mpg::launch_soa2rec<decltype(Lc)::value>(dl, de, ds, N, N, rec, st);
    return 0;
  });
  return MPGPU_OK;
}

int upload_async(mpgpu_handle* h, uint32_t* rec, int L, int64_t N, const uint32_t* limbs, const int32_t* exp,
                 const uint8_t* sign, int32_t Lh, DevBuf& stage, cudaStream_t st_in = nullptr,
                 cudaEvent_t copied = nullptr, int64_t hstride = -1) {
  const size_t planes = sizeof(uint32_t) * (size_t)L * N;
  CUDA_TRY(h, stage.alloc(h, planes + sizeof(int32_t) * N + N));
  return upload_async_to(h, rec, L, N, limbs, exp, sign, Lh, stage.u32(), st_in ? st_in : h->stream, copied,
                         hstride);
}

int download_async(mpgpu_handle* h, const uint32_t* rec, int L, int64_t N, uint32_t* limbs, int32_t* exp,
                   uint8_t* sign, int32_t Lh, DevBuf& stage, int64_t hstride = -1) {
  if (hstride < 0) hstride = N;
  const size_t planes = sizeof(uint32_t) * (size_t)L * N;
  CUDA_TRY(h, stage.alloc(h, planes + sizeof(int32_t) * N + N));
  uint32_t* dl = stage.u32();
  int32_t* de = reinterpret_cast<int32_t*>(dl + (size_t)L * N);
  uint8_t* ds = reinterpret_cast<uint8_t*>(de + N);
  dispatch_store(L, [&](auto Lc) {
    mpg::launch_rec2soa<decltype(Lc)::value>(rec, N, dl, de, ds, N, h->stream);
    return 0;
  });
  const int np = Lh <= L ? Lh : L;
  const uint32_t* src0 = Lh <= L ? dl + (size_t)(L - Lh) * N : dl;
  uint32_t* dst0 = Lh <= L ? limbs : limbs + (size_t)(Lh - L) * hstride;
  if (Lh > L)
    for (int j = 0; j < Lh - L; ++j) std::memset(limbs + (size_t)j * hstride, 0, sizeof(uint32_t) * N);
  if (hstride == N)
    CUDA_TRY(h, cudaMemcpyAsync(dst0, src0, sizeof(uint32_t) * (size_t)np * N, cudaMemcpyDeviceToHost, h->stream));
  else
    CUDA_TRY(h, cudaMemcpy2DAsync(dst0, sizeof(uint32_t) * hstride, src0, sizeof(uint32_t) * N, sizeof(uint32_t) * N,
                                  np, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(exp, de, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(sign, ds, N, cudaMemcpyDeviceToHost, h->stream));
  return MPGPU_OK;
}

// ---------------------------------------------------------------------------
// Pipelined host GEMM (Winograd, even m, l, n): the operands travel to the device by
// quadrant and the product back by output quadrant, so the PCIe transfers run under
// the products instead of before and after them.  The top level of fast_mul_rec
// (fastmm.hpp:174-198) is unrolled here:
//   m2 = a11 b11 and m3 = a12 b21 need one quadrant of A and of B each: each starts as
//   soon as its quadrants are on the device, as its own breadth-first recursion on the
//   views (fast_mul_rec's rec(a11, b11), rec(a12, b21)); C11 = m2 + m3 then leaves at
//   once.  m1, (m4, m5) and (m6, m7) follow as child ranges of the full recursion
//   (run_fast_leaves: the top-level sums s1..s8, then their subtrees);
//   C22 = (t1 + m4) + m5 with t1 = m1 + m2 leaves next, C12 = (t1 + m5) + m6 and
//   C21 = (t1 + m4) - m7 last.  Every element sees the reference's operation sequence:
//   bit-identical to mpgpu_gemm.
// ---------------------------------------------------------------------------
// page-locked host memory (cudaMallocHost / cudaHostRegister): asynchronous copies to and
// from pageable memory are synchronous for the host, which would serialise the pipelines
static bool host_pinned(std::initializer_list<const void*> ps) {
  for (const void* p : ps) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (a.type != cudaMemoryTypeHost) return false;
  }
  return true;
}

static bool host_pipe_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MPGPU_HOST_PIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the pipeline pays for itself once the product is a few milliseconds
static bool host_pipe_applies(int algo, int64_t n_min, int64_t m, int64_t l, int64_t n, int32_t Lh, int L) {
  return host_pipe_enabled() && algo == MPGPU_WINOGRAD && Lh == L && L <= 32 && m % 2 == 0 && l % 2 == 0 && n % 2 == 0 &&
         std::min({m, l, n}) > n_min && (double)m * l * n >= (double)(1 << 21);
}

template <int L>
int gemm_host_pipe(mpgpu_handle* h, int64_t n_min, int32_t prec, int64_t m, int64_t l, int64_t n,
                   const uint32_t* al, const int32_t* ae, const uint8_t* as, const uint32_t* bl, const int32_t* be,
                   const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs, mpgpu_stats* stats) {
  if constexpr (L > 32) {
    return fail(h, MPGPU_ERR_DOMAIN, "internal: pipelined host GEMM is for L <= 32");
  } else {
  constexpr int S = rec_stride(L);
  const int sh = 32 * L - prec;
  const int64_t hm = m / 2, hl = l / 2, hn = n / 2;
  const int64_t qa = hm * hl, qb = hl * hn, qc = hm * hn;
  const size_t R = sizeof(uint32_t) * S;
  const size_t soa = sizeof(uint32_t) * L + sizeof(int32_t) + 1;  // SoA bytes per element
  auto al256 = [](size_t b) { return (b + 255) / 256 * 256; };    // every staging block 256-byte aligned
  const int d = (int)plan_levels(m, l, n, n_min).size() - 1;
  cudaStream_t st = h->stream;
  if (!h->aux) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
  }
  if (!h->dl) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->dl, cudaStreamNonBlocking));
    for (cudaEvent_t& e : h->pev) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t* up = h->pev;         // [0, 8): quadrant copies arrived
  cudaEvent_t* cdone = h->pev + 8;  // [8, 12): output quadrant converted for the copy back
  cudaEvent_t ready = h->pev[12], dl_done = h->pev[13];
  Timer total(stats != nullptr, st);
  DevBuf da, db, l1a, l1b, stage, mq, tq, cq, dstage;
  CUDA_TRY(h, da.alloc(h, R * m * l));
  CUDA_TRY(h, db.alloc(h, R * l * n));
  CUDA_TRY(h, l1a.alloc(h, R * 7 * qa));  // level-1 operands, child slots (see slot below)
  CUDA_TRY(h, l1b.alloc(h, R * 7 * qb));
  CUDA_TRY(h, stage.alloc(h, 4 * al256(soa * (size_t)qa) + 4 * al256(soa * (size_t)qb)));
  CUDA_TRY(h, mq.alloc(h, R * 7 * qc));  // level-1 products, by slot
  CUDA_TRY(h, tq.alloc(h, R * 3 * qc));  // t1, t2, t1 + m5
  CUDA_TRY(h, cq.alloc(h, R * 4 * qc));  // C11, C12, C21, C22
  CUDA_TRY(h, dstage.alloc(h, 4 * al256(soa * (size_t)qc)));
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), st));
  CUDA_TRY(h, cudaEventRecord(ready, st));  // the buffers exist before the other streams touch them
  CUDA_TRY(h, cudaStreamWaitEvent(h->aux, ready, 0));
  CUDA_TRY(h, cudaStreamWaitEvent(h->dl, ready, 0));
  // every exit from here: the handle's stream (which frees the buffers) first waits for the others
  struct Join {
    mpgpu_handle* h;
    cudaEvent_t a, b;
    ~Join() {
      cudaEventRecord(a, h->aux);
      cudaStreamWaitEvent(h->stream, a, 0);
      cudaEventRecord(b, h->dl);
      cudaStreamWaitEvent(h->stream, b, 0);
    }
  } join{h, h->ev_a, dl_done};
  // MPGPU_PIPE_TRACE=1: per-phase event times to stderr (diagnostics)
  static const bool trace = std::getenv("MPGPU_PIPE_TRACE") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  cudaEvent_t t0 = nullptr;
  auto mark = [&](const char* what, cudaStream_t on) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, on);
    marks.push_back({what, e});
  };
  if (trace) {
    cudaEventCreate(&t0);
    cudaEventRecord(t0, st);
  }

  // ---- copies in (aux stream, copy engine only): SoA planes of one quadrant into staging
  struct Quad {
    int side, q;
    uint32_t* pl;
    int32_t* pe;
    uint8_t* ps;
  };
  // order: what m2 = a11 b11, then m3 = a12 b21, then the rest need
  Quad order[8] = {{0, 0}, {1, 0}, {0, 1}, {1, 2}, {0, 2}, {0, 3}, {1, 1}, {1, 3}};
  uint8_t* sp = static_cast<uint8_t*>(stage.p);
  for (int i = 0; i < 8; ++i) {
    Quad& u = order[i];
    const int64_t rows = u.side ? l : m, cols = u.side ? n : l, hr = rows / 2, hc = cols / 2, N = hr * hc;
    const uint32_t* hl_ = u.side ? bl : al;
    const int32_t* he = u.side ? be : ae;
    const uint8_t* hs = u.side ? bs : as;
    u.pl = reinterpret_cast<uint32_t*>(sp);
    u.pe = reinterpret_cast<int32_t*>(u.pl + (size_t)L * N);
    u.ps = reinterpret_cast<uint8_t*>(u.pe + N);
    sp += al256(soa * (size_t)N);
    const int64_t off = (u.q >> 1) * hr * cols + (u.q & 1) * hc;
    const size_t hp = sizeof(uint32_t) * (size_t)cols;
    for (int j = 0; j < L; ++j)
      CUDA_TRY(h, cudaMemcpy2DAsync(u.pl + (size_t)j * N, sizeof(uint32_t) * hc, hl_ + (size_t)j * rows * cols + off,
                                    hp, sizeof(uint32_t) * hc, hr, cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaMemcpy2DAsync(u.pe, sizeof(int32_t) * hc, he + off, sizeof(int32_t) * cols,
                                  sizeof(int32_t) * hc, hr, cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaMemcpy2DAsync(u.ps, hc, hs + off, cols, hc, hr, cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaEventRecord(up[i], h->aux));
    mark("copy in", h->aux);
  }
  // level-1 child c of fast_mul_rec lives in slot[c]: m2, m3 first (slots 0, 1), then
  // m1, m4, m5 (2..4) and m6, m7 (5, 6) -- contiguous unit ranges for run_fast_leaves
  constexpr int8_t slot[7] = {2, 0, 1, 3, 4, 5, 6};
  // layout conversion of copy i on the handle's stream, into the full operand and, for the
  // quadrants that are level-1 operands as they are (a11, b11, a12, b21), into their slot
  auto convert = [&](int i, int l1slot) -> int {
    const Quad& u = order[i];
    const int64_t rows = u.side ? l : m, cols = u.side ? n : l, hr = rows / 2, hc = cols / 2, N = hr * hc;
    CUDA_TRY(h, cudaStreamWaitEvent(st, up[i], 0));
    uint32_t* full = u.side ? db.u32() : da.u32();
    const int64_t off = (u.q >> 1) * hr * cols + (u.q & 1) * hc;
    mpg::launch_soa2rec_2d<L>(u.pl, u.pe, u.ps, hr, hc, N, full + off * S, cols, st);
    if (l1slot >= 0)
      mpg::launch_soa2rec<L>(u.pl, u.pe, u.ps, N, N, (u.side ? l1b.u32() : l1a.u32()) + (size_t)l1slot * N * S, st);
    return MPGPU_OK;
  };

  // ---- copies out (dl stream): output quadrant q, converted on the handle's stream
  uint8_t* dp = static_cast<uint8_t*>(dstage.p);
  auto Cq = [&](int q) { return cq.u32() + (size_t)q * qc * S; };
  auto download_quad = [&](int q) -> int {
    uint32_t* pl = reinterpret_cast<uint32_t*>(dp + q * al256(soa * (size_t)qc));
    int32_t* pe = reinterpret_cast<int32_t*>(pl + (size_t)L * qc);
    uint8_t* ps = reinterpret_cast<uint8_t*>(pe + qc);
    mpg::launch_rec2soa<L>(Cq(q), qc, pl, pe, ps, qc, st);
    CUDA_TRY(h, cudaEventRecord(cdone[q], st));
    CUDA_TRY(h, cudaStreamWaitEvent(h->dl, cdone[q], 0));
    const int64_t off = (q >> 1) * hm * n + (q & 1) * hn;
    const size_t hp = sizeof(uint32_t) * (size_t)n;
    for (int j = 0; j < L; ++j)
      CUDA_TRY(h, cudaMemcpy2DAsync(cl + (size_t)j * m * n + off, hp, pl + (size_t)j * qc, sizeof(uint32_t) * hn,
                                    sizeof(uint32_t) * hn, hm, cudaMemcpyDeviceToHost, h->dl));
    CUDA_TRY(h, cudaMemcpy2DAsync(ce + off, sizeof(int32_t) * n, pe, sizeof(int32_t) * hn, sizeof(int32_t) * hn, hm,
                                  cudaMemcpyDeviceToHost, h->dl));
    CUDA_TRY(h, cudaMemcpy2DAsync(cs + off, n, ps, hn, hn, hm, cudaMemcpyDeviceToHost, h->dl));
    mark("copy out", h->dl);
    return MPGPU_OK;
  };

  // ---- products and the top-level post-additions (handle's stream)
  auto Ms = [&](int child) { return mq.u32() + (size_t)slot[child] * qc * S; };  // m_{child+1}
  uint32_t* t1 = tq.u32();
  uint32_t* t2 = t1 + (size_t)qc * S;
  uint32_t* u5 = t2 + (size_t)qc * S;
  auto add = [&](const uint32_t* x, const uint32_t* y, uint32_t* z, int is_sub) {
    mpg::launch_addsub<L>(x, y, z, qc, is_sub, sh, h->d_err, st);
  };
  auto products = [&](int slot_lo, int slot_hi) {  // level-1 products of slots [lo, hi)
    return run_fast_leaves<L>(h, MPGPU_WINOGRAD, n_min, da.u32(), l, db.u32(), n, m, l, n, slot_lo, slot_hi, d - 1,
                              mq.u32() + (size_t)slot_lo * qc * S, sh, nullptr, nullptr, l1a.u32(), l1b.u32());
  };
  int rc;
  if ((rc = convert(0, 0)) || (rc = convert(1, 0)) || (rc = products(0, 1))) return rc;  // m2 = a11 b11
  mark("m2", st);
  if ((rc = convert(2, 1)) || (rc = convert(3, 1)) || (rc = products(1, 2))) return rc;  // m3 = a12 b21
  add(Ms(1), Ms(2), Cq(0), 0);                                                           // C11 = m2 + m3
  mark("m3 C11", st);
  if ((rc = download_quad(0))) return rc;
  for (int i = 4; i < 8; ++i)
    if ((rc = convert(i, -1))) return rc;
  const mpg::ChildSlots rest{{slot[0], -1, -1, slot[3], slot[4], slot[5], slot[6]}};
  mpg::launch_preadd_slots<L>(MPGPU_WINOGRAD, 0, da.u32(), (int)m, (int)l, l1a.u32(), rest, sh, st);  // s1..s4
  mpg::launch_preadd_slots<L>(MPGPU_WINOGRAD, 1, db.u32(), (int)l, (int)n, l1b.u32(), rest, sh, st);  // s5..s8
  if ((rc = products(2, 5))) return rc;  // m1 = s2 s6, m4 = s3 s7, m5 = s1 s5
  add(Ms(0), Ms(1), t1, 0);              // t1 = m1 + m2
  add(t1, Ms(3), t2, 0);                 // t2 = t1 + m4
  add(t2, Ms(4), Cq(3), 0);              // C22 = t2 + m5
  mark("m1 m4 m5 C22", st);
  if ((rc = download_quad(3))) return rc;
  // m6 and m7 apart: C12 goes back while m7 is computed
  if ((rc = products(5, 6))) return rc;  // m6 = s4 b22
  add(t1, Ms(4), u5, 0);                 // t1 + m5
  add(u5, Ms(5), Cq(1), 0);              // C12 = (t1 + m5) + m6
  mark("m6 C12", st);
  if ((rc = download_quad(1))) return rc;
  if ((rc = products(6, 7))) return rc;  // m7 = a22 s8
  add(t2, Ms(6), Cq(2), 1);              // C21 = t2 - m7
  mark("m7 C21", st);
  if ((rc = download_quad(2))) return rc;
  if (trace) {
    cudaDeviceSynchronize();
    for (auto& mk : marks) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, mk.second);
      fprintf(stderr, "[pipe] %-16s %8.3f ms\n", mk.first, ms);
      cudaEventDestroy(mk.second);
    }
    cudaEventDestroy(t0);
  }
  if (stats) {
    total.stop(&stats->device_ms);
    stats->depth = d;
  }
  return MPGPU_OK;
  }
}

// ===========================================================================
extern "C" {

int mpgpu_init(int device, mpgpu_handle** out) {
  if (!out) return MPGPU_ERR_DOMAIN;
  *out = nullptr;
  auto* h = new mpgpu_handle();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_err, 4 * sizeof(uint32_t));  // [0] flags, [2:4) int64 zero pivot
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear the runtime's last error: later calls must not see it
    if (h->d_err) cudaFree(h->d_err);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
    return MPGPU_ERR_CUDA;
  }
  h->stream = h->own_stream;
  // keep freed pool memory cached: repeated calls reuse it without cudaMalloc
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = h;
  return MPGPU_OK;
}

void mpgpu_destroy(mpgpu_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  if (h->aux) cudaStreamSynchronize(h->aux);
  if (h->d_err) cudaFree(h->d_err);
  if (h->d_piv) cudaFree(h->d_piv);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->ev_b) cudaEventDestroy(h->ev_b);
  if (h->hi) {
    cudaStreamSynchronize(h->hi);
    cudaStreamDestroy(h->hi);
  }
  if (h->ev_la) cudaEventDestroy(h->ev_la);
  if (h->ev_lp) cudaEventDestroy(h->ev_lp);
  if (h->dl) {
    cudaStreamSynchronize(h->dl);
    cudaStreamDestroy(h->dl);
  }
  for (cudaEvent_t e : h->pev)
    if (e) cudaEventDestroy(e);
  delete h;
}

const char* mpgpu_last_error(const mpgpu_handle* h) { return h ? h->last_error.c_str() : "null handle"; }

int mpgpu_set_stream(mpgpu_handle* h, void* s) {
  if (!h) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  h->stream = s ? static_cast<cudaStream_t>(s) : h->own_stream;
  return MPGPU_OK;
}

void* mpgpu_get_stream(mpgpu_handle* h) { return h ? (void*)h->stream : nullptr; }

int mpgpu_synchronize(mpgpu_handle* h) {
  if (!h) return MPGPU_ERR_DOMAIN;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return MPGPU_OK;
}

int mpgpu_copy_device(mpgpu_handle* h, void* dst, const void* src, size_t bytes) {
  if (!h) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, h->stream));
  return MPGPU_OK;
}

int mpgpu_nlimbs_for(int32_t prec) { return nlimbs_for(prec); }
int mpgpu_record_words(int32_t nlimbs) { return rec_stride(nlimbs); }

int mpgpu_alloc_matrix(mpgpu_handle* h, int64_t rows, int64_t cols, int32_t prec, mpgpu_mat* out) {
  if (!h || !out) return MPGPU_ERR_DOMAIN;
  if (rows < 1 || cols < 1) return fail(h, MPGPU_ERR_DIMENSION, "matrix dimensions must be at least 1x1");
  const int L = nlimbs_for(prec);
  if (!L) return fail(h, MPGPU_ERR_DOMAIN, "precision %d outside the device range [2, %d]", prec, MPGPU_MAX_PREC);
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  void* p = nullptr;
  const size_t bytes = sizeof(uint32_t) * (size_t)rec_stride(L) * (size_t)(rows * cols);
  CUDA_TRY(h, cudaMalloc(&p, bytes));
  // +0 everywhere (Matrix ctor, matrix.hpp:22-28: every element Scalar(ctx) = +0):
  // all-zero words except the exponent word, set by the conversion kernel below.
  CUDA_TRY(h, cudaMemsetAsync(p, 0, bytes, h->stream));
  out->rows = rows;
  out->cols = cols;
  out->prec = prec;
  out->nlimbs = L;
  out->rec = static_cast<uint32_t*>(p);
  out->ld = cols;
  out->owned = 1;
  // exponent words := EXP_ZERO
  const int S = rec_stride(L);
  CUDA_TRY(h, cudaMemset2DAsync(static_cast<uint32_t*>(p) + L, sizeof(uint32_t) * S, 0x00, 4, rows * cols,
                                h->stream));
  {
    // write INT32_MIN (0x80000000): byte 3 of each exponent word = 0x80
    CUDA_TRY(h, cudaMemset2DAsync(reinterpret_cast<uint8_t*>(static_cast<uint32_t*>(p) + L) + 3,
                                  sizeof(uint32_t) * S, 0x80, 1, rows * cols, h->stream));
  }
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return MPGPU_OK;
}

int mpgpu_free_matrix(mpgpu_handle* h, mpgpu_mat* m) {
  if (!m) return MPGPU_OK;
  if (m->owned && m->rec) {
    if (h) cudaSetDevice(h->device);
    cudaFree(m->rec);
  }
  m->rec = nullptr;
  m->owned = 0;
  return MPGPU_OK;
}

int mpgpu_upload(mpgpu_handle* h, mpgpu_mat* m, const uint32_t* limbs, const int32_t* exp, const uint8_t* sign,
                 int32_t Lh) {
  if (!h || !m || !m->rec) return MPGPU_ERR_DOMAIN;
  if (m->ld != m->cols) return fail(h, MPGPU_ERR_DIMENSION, "upload into a strided view");
  if (Lh < (m->prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  DevBuf stage;
  int rc = upload_async(h, m->rec, m->nlimbs, m->rows * m->cols, limbs, exp, sign, Lh, stage);
  if (rc) return rc;
  stage.release();
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaGetLastError());
  return MPGPU_OK;
}

int mpgpu_download(mpgpu_handle* h, const mpgpu_mat* m, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                   int32_t Lh) {
  if (!h || !m || !m->rec) return MPGPU_ERR_DOMAIN;
  if (m->ld != m->cols) return fail(h, MPGPU_ERR_DIMENSION, "download from a strided view");
  if (Lh < (m->prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  DevBuf stage;
  int rc = download_async(h, m->rec, m->nlimbs, m->rows * m->cols, limbs, exp, sign, Lh, stage);
  if (rc) return rc;
  stage.release();
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaGetLastError());
  return MPGPU_OK;
}

int mpgpu_upload_strided(mpgpu_handle* h, mpgpu_mat* m, const uint32_t* limbs, const int32_t* exp,
                         const uint8_t* sign, int32_t Lh, int64_t host_plane_stride) {
  if (!h || !m || !m->rec) return MPGPU_ERR_DOMAIN;
  if (m->ld != m->cols) return fail(h, MPGPU_ERR_DIMENSION, "upload into a strided view");
  if (Lh < (m->prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  if (host_plane_stride < m->rows * m->cols) return fail(h, MPGPU_ERR_DIMENSION, "host plane stride too small");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  DevBuf stage;
  int rc = upload_async(h, m->rec, m->nlimbs, m->rows * m->cols, limbs, exp, sign, Lh, stage, nullptr, nullptr,
                        host_plane_stride);
  if (rc) return rc;
  stage.release();
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaGetLastError());
  return MPGPU_OK;
}

int mpgpu_download_strided(mpgpu_handle* h, const mpgpu_mat* m, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                           int32_t Lh, int64_t host_plane_stride) {
  if (!h || !m || !m->rec) return MPGPU_ERR_DOMAIN;
  if (m->ld != m->cols) return fail(h, MPGPU_ERR_DIMENSION, "download from a strided view");
  if (Lh < (m->prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  if (host_plane_stride < m->rows * m->cols) return fail(h, MPGPU_ERR_DIMENSION, "host plane stride too small");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  DevBuf stage;
  int rc = download_async(h, m->rec, m->nlimbs, m->rows * m->cols, limbs, exp, sign, Lh, stage, host_plane_stride);
  if (rc) return rc;
  stage.release();
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaGetLastError());
  return MPGPU_OK;
}

int mpgpu_fast_owned_rows(int64_t m, int64_t l, int64_t n, int64_t n_min, int up_levels, int64_t row_lo,
                          int64_t row_hi, int64_t* out, int64_t cap, int64_t* count) {
  if (!count || m < 1 || l < 1 || n < 1 || n_min < 1) return MPGPU_ERR_DIMENSION;
  const std::vector<Level> lv = plan_levels(m, l, n, n_min);
  const int d = (int)lv.size() - 1;
  if (up_levels < 0 || up_levels > d) return MPGPU_ERR_DIMENSION;
  const int il = d - up_levels;
  if (row_lo < 0 || row_lo > row_hi || row_hi > lv[il].m) return MPGPU_ERR_DIMENSION;
  const auto owned = owned_rows(lv, il, row_lo, row_hi);
  *count = (int64_t)owned[0].size();
  if (out)
    for (int64_t i = 0; i < *count && i < cap; ++i) out[i] = owned[0][i];
  return MPGPU_OK;
}

int mpgpu_choose_nmin(int algo, int32_t prec, int64_t m, int64_t l, int64_t n, int64_t* n_min, int32_t* depth,
                      double* model_ms) {
  if (m < 1 || l < 1 || n < 1) return MPGPU_ERR_DIMENSION;
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD) return MPGPU_ERR_DOMAIN;
  const int L = nlimbs_for(prec);
  if (!L) return MPGPU_ERR_DOMAIN;
  int d = 0;
  const int rc = choose_nmin(L, m, l, n, n_min, &d, model_ms);
  if (depth) *depth = d;
  return rc;
}

namespace {
// MPGPU_AUTO_NMIN -> the chosen cutoff (Strassen / Winograd only)
int resolve_auto(mpgpu_handle* h, int algo, int32_t prec, int64_t m, int64_t l, int64_t n, int64_t* param) {
  if (*param != MPGPU_AUTO_NMIN) return MPGPU_OK;
  if (algo == MPGPU_SIMPLE) {
    *param = 0;
    return MPGPU_OK;
  }
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD)
    return fail(h, MPGPU_ERR_DOMAIN, "MPGPU_AUTO_NMIN applies to strassen / winograd only");
  const int L = nlimbs_for(prec);
  if (!L) return fail(h, MPGPU_ERR_DOMAIN, "precision %d outside the device range", prec);
  return choose_nmin(L, std::max<int64_t>(1, m), std::max<int64_t>(1, l), std::max<int64_t>(1, n), param, nullptr,
                     nullptr);
}
}  // namespace

int mpgpu_gemm(mpgpu_handle* h, int algo, int64_t param, const mpgpu_mat* A, const mpgpu_mat* B, mpgpu_mat* C,
               mpgpu_stats* stats) {
  TimerGuard timer_guard;
  if (!h) return MPGPU_ERR_DOMAIN;
  if (A && B && C && A->cols == B->rows)
    if (int r = resolve_auto(h, algo, C->prec, A->rows, A->cols, B->cols, &param)) return r;
  int rc = validate_gemm(h, algo, param, A, B, C);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (stats) {
    std::memset(stats, 0, sizeof *stats);
    uint64_t c[2];
    count_fast_rec(algo, A->rows, A->cols, B->cols, param, c);
    stats->mul = c[0];
    stats->addsub = c[1];
  }
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * C->nlimbs - C->prec;
  rc = dispatch_L(C->nlimbs, [&](auto Lc) {
    return run_gemm<decltype(Lc)::value>(h, algo, param, A->rec, A->ld, B->rec, B->ld, C->rec, C->ld, A->rows,
                                         A->cols, B->cols, sh, stats, 0);
  });
  if (rc) return rc;
  return check_err(h);
}

int mpgpu_gemm_host(mpgpu_handle* h, int algo, int64_t param, int32_t prec, int64_t m, int64_t l, int64_t n,
                    const uint32_t* al, const int32_t* ae, const uint8_t* as, const uint32_t* bl,
                    const int32_t* be, const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs, int32_t Lh,
                    mpgpu_stats* stats) {
  TimerGuard timer_guard;
  // One stream-ordered sequence: pooled device buffers, H2D + layout conversion of A
  // and B, the product, conversion + D2H of C, and a single synchronisation.
  if (!h) return MPGPU_ERR_DOMAIN;
  const int L = nlimbs_for(prec);
  if (!L) return fail(h, MPGPU_ERR_DOMAIN, "precision %d outside the device range [2, %d]", prec, MPGPU_MAX_PREC);
  if (m < 1 || l < 1 || n < 1) return fail(h, MPGPU_ERR_DIMENSION, "matrix dimensions must be at least 1x1");
  if (Lh < (prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  if (int r = resolve_auto(h, algo, prec, m, l, n, &param)) return r;
  mpgpu_mat A{m, l, prec, L, nullptr, l, 0}, B{l, n, prec, L, nullptr, n, 0}, C{m, n, prec, L, nullptr, n, 0};
  int rc = validate_gemm(h, algo, param, &A, &B, &C);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (host_pipe_applies(algo, param, m, l, n, Lh, L) && host_pinned({al, ae, as, bl, be, bs, cl, ce, cs})) {
    if (stats) {
      std::memset(stats, 0, sizeof *stats);
      uint64_t c[2];
      count_fast_rec(algo, m, l, n, param, c);
      stats->mul = c[0];
      stats->addsub = c[1];
    }
    rc = dispatch_L(L, [&](auto Lc) {
      return gemm_host_pipe<decltype(Lc)::value>(h, param, prec, m, l, n, al, ae, as, bl, be, bs, cl, ce, cs, stats);
    });
    if (rc) return rc;
    rc = check_err(h);
    flush_timers();
    return rc;
  }
  const size_t S4 = sizeof(uint32_t) * rec_stride(L);
  DevBuf da, db, dc, sa, sb, sc;
  CUDA_TRY(h, da.alloc(h, S4 * m * l));
  CUDA_TRY(h, db.alloc(h, S4 * l * n));
  CUDA_TRY(h, dc.alloc(h, S4 * m * n));
  A.rec = da.u32();
  B.rec = db.u32();
  C.rec = dc.u32();
  if (stats) {
    std::memset(stats, 0, sizeof *stats);
    uint64_t c[2];
    count_fast_rec(algo, m, l, n, param, c);
    stats->mul = c[0];
    stats->addsub = c[1];
  }
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  // A's upload on the handle's stream; B's on a second stream, started once A's bytes are
  // across, so the A-side layout conversion and pre-additions overlap B's transfer (the
  // B side of the product waits for B's event)
  if (!h->aux) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
  }
  rc = upload_async(h, A.rec, L, m * l, al, ae, as, Lh, sa, h->stream, h->ev_a);
  if (rc) return rc;
  CUDA_TRY(h, cudaStreamWaitEvent(h->aux, h->ev_a, 0));  // also orders db's allocation
  {
    uint32_t* stage = nullptr;
    const size_t sbytes = (sizeof(uint32_t) * (size_t)L + sizeof(int32_t) + 1) * (size_t)(l * n);
    CUDA_TRY(h, cudaMallocAsync(reinterpret_cast<void**>(&stage), sbytes, h->aux));
    rc = upload_async_to(h, B.rec, L, l * n, bl, be, bs, Lh, stage, h->aux);
    cudaFreeAsync(stage, h->aux);
    if (rc) return rc;
  }
  CUDA_TRY(h, cudaEventRecord(h->ev_b, h->aux));
  // on every return from here, db (freed on h->stream by ~DevBuf) must not be released
  // while h->aux may still be writing it: order h->stream after B's upload first
  struct WaitB {
    mpgpu_handle* h;
    ~WaitB() { cudaStreamWaitEvent(h->stream, h->ev_b, 0); }
  } wait_b{h};
  sa.release();
  const int sh = 32 * L - prec;
  rc = dispatch_L(L, [&](auto Lc) {
    return run_gemm<decltype(Lc)::value>(h, algo, param, A.rec, l, B.rec, n, C.rec, n, m, l, n, sh, stats, 0,
                                         h->ev_b);
  });
  if (rc) return rc;
  rc = download_async(h, C.rec, L, m * n, cl, ce, cs, Lh, sc);
  if (rc) return rc;
  return check_err(h);
}

int mpgpu_addsub(mpgpu_handle* h, int is_sub, const mpgpu_mat* A, const mpgpu_mat* B, mpgpu_mat* C) {
  if (!h || !A || !B || !C) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {A, B, C})) return r;
  if (A->prec != B->prec) return fail(h, MPGPU_ERR_DOMAIN, is_sub ? "mat sub: mixed precisions" : "mat add: mixed precisions");
  if (A->rows != B->rows || A->cols != B->cols || C->rows != A->rows || C->cols != A->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "shape mismatch: %lldx%lld vs %lldx%lld", (long long)A->rows,
                (long long)A->cols, (long long)B->rows, (long long)B->cols);
  if (C->prec != A->prec || A->ld != A->cols || B->ld != B->cols || C->ld != C->cols)
    return fail(h, MPGPU_ERR_DOMAIN, "addsub requires dense matrices of one precision");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * C->nlimbs - C->prec;
  dispatch_L(C->nlimbs, [&](auto Lc) {
    mpg::launch_addsub<decltype(Lc)::value>(A->rec, B->rec, C->rec, A->rows * A->cols, is_sub, sh, h->d_err,
                                            h->stream);
    return 0;
  });
  return check_err(h);
}

int mpgpu_vec_op(mpgpu_handle* h, int op, const mpgpu_mat* A, const mpgpu_mat* B, mpgpu_mat* C) {
  if (!h || !A || !B || !C) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {A, B, C})) return r;
  if (A->rows * A->cols != B->rows * B->cols || C->rows * C->cols != A->rows * A->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "vec_op: size mismatch");
  if (A->prec != C->prec || B->prec != C->prec) return fail(h, MPGPU_ERR_DOMAIN, "vec_op: mixed precisions");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * C->nlimbs - C->prec;
  dispatch_L(C->nlimbs, [&](auto Lc) {
    mpg::launch_vec_op<decltype(Lc)::value>(op, A->rec, B->rec, C->rec, A->rows * A->cols, sh, h->d_err,
                                            h->stream);
    return 0;
  });
  return check_err(h);
}

int mpgpu_fast_mul_trace(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                         mpgpu_mat* C, uint32_t* trace_rec, int* counts) {
  if (!h) return MPGPU_ERR_DOMAIN;
  int rc = validate_gemm(h, algo, n_min, A, B, C);
  if (rc) return rc;
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD)
    return fail(h, MPGPU_ERR_DOMAIN, "fast_mul: algorithm must be strassen or winograd");
  if (A->ld != A->cols || B->ld != B->cols || C->ld != C->cols)
    return fail(h, MPGPU_ERR_DOMAIN, "trace requires dense matrices");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int64_t m = A->rows, l = A->cols, n = B->cols;
  counts[0] = counts[1] = counts[2] = 0;
  const int sh = 32 * C->nlimbs - C->prec;
  if (std::min({m, l, n}) <= n_min) {  // base case: no trace (fastmm.hpp:102)
    rc = dispatch_L(C->nlimbs, [&](auto Lc) {
      return run_gemm<decltype(Lc)::value>(h, MPGPU_SIMPLE, 0, A->rec, m, B->rec, n, C->rec, n, m, l, n, sh,
                                           nullptr, 0);
    });
    return rc ? rc : check_err(h);
  }
  const int64_t hm = (m + m % 2) / 2, hl = (l + l % 2) / 2, hn = (n + n % 2) / 2;
  rc = dispatch_L(C->nlimbs, [&](auto Lc) -> int {
    constexpr int L = decltype(Lc)::value;
    constexpr int S = rec_stride(L);
    cudaStream_t st = h->stream;
    DevBuf ca, cb, prods;
    CUDA_TRY(h, ca.alloc(h, sizeof(uint32_t) * S * 7 * hm * hl));
    CUDA_TRY(h, cb.alloc(h, sizeof(uint32_t) * S * 7 * hl * hn));
    CUDA_TRY(h, prods.alloc(h, sizeof(uint32_t) * S * 7 * hm * hn));
    mpg::launch_preadd<L>(algo, 0, A->rec, 1, (int)m, (int)l, ca.u32(), sh, h->d_err, st);
    mpg::launch_preadd<L>(algo, 1, B->rec, 1, (int)l, (int)n, cb.u32(), sh, h->d_err, st);
    // the 7 children via the full driver (each is a fast_mul_rec call)
    for (int q = 0; q < 7; ++q) {
      int r = run_gemm<L>(h, algo, n_min, ca.u32() + (size_t)q * S * hm * hl, hl, cb.u32() + (size_t)q * S * hl * hn,
                          hn, prods.u32() + (size_t)q * S * hm * hn, hn, hm, hl, hn, sh, nullptr, 0);
      if (r) return r;
    }
    uint32_t* tout = trace_rec;
    int64_t off = 0;
    const size_t ha = (size_t)hm * hl, hb = (size_t)hl * hn, hp = (size_t)hm * hn;
    auto cpy = [&](const uint32_t* src, size_t elems) {
      cudaMemcpyAsync(tout + off * S, src, sizeof(uint32_t) * S * elems, cudaMemcpyDeviceToDevice, st);
      off += (int64_t)elems;
    };
    uint32_t* t_out = nullptr;
    if (algo == MPGPU_WINOGRAD) {
      // S1..S4 are children A operands 4,0,3,5; S5..S8 children B operands 4,0,3,6
      const int sa[4] = {4, 0, 3, 5}, sb[4] = {4, 0, 3, 6};
      for (int q : sa) cpy(ca.u32() + q * S * ha, ha);
      for (int q : sb) cpy(cb.u32() + q * S * hb, hb);
      counts[0] = 8;
    }
    for (int q = 0; q < 7; ++q) cpy(prods.u32() + q * S * hp, hp);
    counts[1] = 7;
    if (algo == MPGPU_WINOGRAD) {
      t_out = tout + off * S;
      counts[2] = 2;
    }
    mpg::launch_postadd<L>(algo, prods.u32(), 1, (int)m, (int)n, C->rec, t_out, sh, h->d_err, st);
    return 0;
  });
  if (rc) return rc;
  return check_err(h);
}

}  // extern "C"

namespace {
// ---------------------------------------------------------------------------
// LU look-ahead: the Schur update A22 = RN(A22 - L21 U12) (blocklu.hpp:88-101, 138-141) in two
// column parts -- part A: columns [0, w) of A22 (the next panel), part B: the rest.  Column
// slices of the Strassen / Winograd recursion are closed: a child column c feeds only parent
// columns c and c + hc (post-additions are elementwise per quadrant), and the leaves are plain
// products whose columns are independent, so computing the leaves' first w columns, the
// post-additions of child columns [0, w) at every level and then the remainder performs, per
// element, exactly the unsplit operation sequence: bit-identical results.  Between the parts
// the caller factors the next panel on another stream (it reads and writes only columns the
// part-A update finished, while part B writes only the columns beyond).
// ---------------------------------------------------------------------------
template <int L>
struct SchurSplit {
  std::vector<Level> lv;
  int d = 0;
  int64_t nodes = 1;  // leaves
  std::vector<DevBuf> opA, opB, prod;
  DevBuf top;
};

// true if columns [0, w) can be split off: w within every level's child width (leaf columns)
bool schur_split_ok(int kernel, int64_t rest, int64_t K, int64_t n_min, int64_t w) {
  if (w <= 0 || w >= rest) return false;
  if (kernel == MPGPU_SIMPLE || kernel == MPGPU_BLOCK) return true;
  const std::vector<Level> lv = plan_levels(rest, K, rest, n_min);
  return w <= lv.back().n;
}

// part A (on h->stream): everything for columns [0, w) of a22 (including all pre-additions)
template <int L>
int schur_part_a(mpgpu_handle* h, SchurSplit<L>& S_, int kernel, int64_t n_min, const uint32_t* l21,
                 const uint32_t* u12, uint32_t* a22, int64_t ld, int64_t rest, int64_t K, int64_t w, int sh,
                 mpgpu_stats* stats) {
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  if (kernel == MPGPU_SIMPLE || kernel == MPGPU_BLOCK ||
      (S_.lv = plan_levels(rest, K, rest, n_min), S_.d = (int)S_.lv.size() - 1) == 0) {
    S_.d = 0;
    const int alg = (kernel == MPGPU_BLOCK) ? MPGPU_BLOCK : MPGPU_SIMPLE;
    return run_gemm<L>(h, alg, kernel == MPGPU_BLOCK ? n_min : 0, l21, ld, u12, ld, a22, ld, rest, K, w, sh, stats,
                       1);
  }
  const std::vector<Level>& lv = S_.lv;
  const int d = S_.d;
  Timer total(stats != nullptr, st);
  int launches = 0;
  DevBuf a0, b0;  // dense level-0 operands
  CUDA_TRY(h, a0.alloc(h, sizeof(uint32_t) * S * rest * K));
  CUDA_TRY(h, b0.alloc(h, sizeof(uint32_t) * S * K * rest));
  mpg::launch_copy2d<L>(l21, ld, a0.u32(), K, (int)rest, (int)K, st);
  mpg::launch_copy2d<L>(u12, ld, b0.u32(), rest, (int)K, (int)rest, st);
  launches += 2;
  std::vector<DevBuf>(d + 1).swap(S_.opA);  // (DevBuf is not movable: no resize)
  std::vector<DevBuf>(d + 1).swap(S_.opB);
  std::vector<DevBuf>(d + 1).swap(S_.prod);
  {
    Timer tpre(stats != nullptr, st);
    int64_t nd = 1;
    for (int lev = 0; lev < d; ++lev, nd *= 7) {
      const Level& P = lv[lev];
      const Level& Q = lv[lev + 1];
      CUDA_TRY(h, S_.opA[lev + 1].alloc(h, sizeof(uint32_t) * S * nd * 7 * Q.m * Q.l));
      CUDA_TRY(h, S_.opB[lev + 1].alloc(h, sizeof(uint32_t) * S * nd * 7 * Q.l * Q.n));
      mpg::launch_preadd<L>(kernel, 0, lev == 0 ? a0.u32() : S_.opA[lev].u32(), nd, (int)P.m, (int)P.l,
                            S_.opA[lev + 1].u32(), sh, h->d_err, st);
      mpg::launch_preadd<L>(kernel, 1, lev == 0 ? b0.u32() : S_.opB[lev].u32(), nd, (int)P.l, (int)P.n,
                            S_.opB[lev + 1].u32(), sh, h->d_err, st);
      launches += 2;
      if (lev > 0) {
        S_.opA[lev].release();
        S_.opB[lev].release();
      }
    }
    S_.nodes = nd;
    if (stats) tpre.stop(&stats->preadd_ms);
  }
  a0.release();
  b0.release();
  const Level& D = lv[d];
  CUDA_TRY(h, S_.prod[d].alloc(h, sizeof(uint32_t) * S * S_.nodes * D.m * D.n));
  auto leaf_cols = [&](int64_t c0, int64_t cw) {
    mpg::GemmArgs g{};
    g.A = S_.opA[d].u32();
    g.B = S_.opB[d].u32() + c0 * S;
    g.C = S_.prod[d].u32() + c0 * S;
    g.strideA = D.m * D.l;
    g.strideB = D.l * D.n;
    g.strideC = D.m * D.n;
    g.lda = D.l;
    g.ldb = D.n;
    g.ldc = D.n;
    g.m = (int)D.m;
    g.l = (int)D.l;
    g.n = (int)cw;
    g.kb = (int)D.l;
    g.batch = (int)S_.nodes;
    g.sh = sh;
    g.err = h->d_err;
    mpg::launch_gemm<L>(g, st);
  };
  {
    Timer tl(stats != nullptr, st);
    leaf_cols(0, w);
    ++launches;
    if (stats) {
      tl.stop(&stats->leaf_ms);
      stats->leaf_madds = (uint64_t)S_.nodes * D.m * D.l * w;
    }
  }
  Timer tpost(stats != nullptr, st);
  int64_t nd = S_.nodes;
  for (int lev = d - 1; lev >= 0; --lev) {
    nd /= 7;
    const Level& P = lv[lev];
    CUDA_TRY(h, S_.prod[lev].alloc(h, sizeof(uint32_t) * S * nd * P.m * P.n));
    mpg::launch_postadd<L>(kernel, S_.prod[lev + 1].u32(), nd, (int)P.m, (int)P.n, S_.prod[lev].u32(), nullptr, sh,
                           h->d_err, st, nullptr, 0, 0, (int)w);
    ++launches;
  }
  mpg::launch_sub2d<L>(a22, ld, S_.prod[0].u32(), (int)rest, (int)w, sh, h->d_err, st, rest);
  ++launches;
  if (stats) {
    tpost.stop(&stats->postadd_ms);
    total.stop(&stats->device_ms);
    stats->launches = launches;
    stats->depth = d;
  }
  return MPGPU_OK;
}

// part B (on h->stream, after part A): columns [w, rest) of a22; releases the buffers
template <int L>
int schur_part_b(mpgpu_handle* h, SchurSplit<L>& S_, int kernel, int64_t n_min, const uint32_t* l21,
                 const uint32_t* u12, uint32_t* a22, int64_t ld, int64_t rest, int64_t K, int64_t w, int sh,
                 mpgpu_stats* stats) {
  constexpr int S = rec_stride(L);
  cudaStream_t st = h->stream;
  if (S_.d == 0) {
    const int alg = (kernel == MPGPU_BLOCK) ? MPGPU_BLOCK : MPGPU_SIMPLE;
    return run_gemm<L>(h, alg, kernel == MPGPU_BLOCK ? n_min : 0, l21, ld, u12 + w * S, ld, a22 + w * S, ld, rest,
                       K, rest - w, sh, stats, 1);
  }
  const std::vector<Level>& lv = S_.lv;
  const int d = S_.d;
  const Level& D = lv[d];
  Timer total(stats != nullptr, st);
  int launches = 0;
  {
    Timer tl(stats != nullptr, st);
    if (D.n > w) {
      mpg::GemmArgs g{};
      g.A = S_.opA[d].u32();
      g.B = S_.opB[d].u32() + w * S;
      g.C = S_.prod[d].u32() + w * S;
      g.strideA = D.m * D.l;
      g.strideB = D.l * D.n;
      g.strideC = D.m * D.n;
      g.lda = D.l;
      g.ldb = D.n;
      g.ldc = D.n;
      g.m = (int)D.m;
      g.l = (int)D.l;
      g.n = (int)(D.n - w);
      g.kb = (int)D.l;
      g.batch = (int)S_.nodes;
      g.sh = sh;
      g.err = h->d_err;
      mpg::launch_gemm<L>(g, st);
      ++launches;
    }
    if (stats) {
      tl.stop(&stats->leaf_ms);
      stats->leaf_madds = (uint64_t)S_.nodes * D.m * D.l * (D.n - w);
    }
  }
  S_.opA[d].release();
  S_.opB[d].release();
  Timer tpost(stats != nullptr, st);
  int64_t nd = S_.nodes;
  for (int lev = d - 1; lev >= 0; --lev) {
    nd /= 7;
    const Level& P = lv[lev];
    const int hc = (int)lv[lev + 1].n;
    if (hc > w)
      mpg::launch_postadd<L>(kernel, S_.prod[lev + 1].u32(), nd, (int)P.m, (int)P.n, S_.prod[lev].u32(), nullptr,
                             sh, h->d_err, st, nullptr, 0, (int)w, hc - (int)w);
    ++launches;
    S_.prod[lev + 1].release();
  }
  mpg::launch_sub2d<L>(a22 + w * S, ld, S_.prod[0].u32() + w * S, (int)rest, (int)(rest - w), sh, h->d_err, st,
                       rest);
  ++launches;
  S_.prod[0].release();
  if (stats) {
    tpost.stop(&stats->postadd_ms);
    total.stop(&stats->device_ms);
    stats->launches = launches;
    stats->depth = d;
  }
  return MPGPU_OK;
}
}  // namespace

extern "C" {

int mpgpu_lu_blocked(mpgpu_handle* h, mpgpu_mat* A, int64_t K, int kernel, int64_t n_min, int pivoting,
                     int64_t* piv_out, int64_t* zero_pivot, mpgpu_stats* stats) {
  TimerGuard timer_guard;
  if (!h || !A) return MPGPU_ERR_DOMAIN;
  if (zero_pivot) *zero_pivot = 0;
  if (int r = compute_range(h, {A})) return r;
  if (A->rows != A->cols) return fail(h, MPGPU_ERR_DIMENSION, "lu_blocked: matrix must be square");
  if (K == 0) return fail(h, MPGPU_ERR_DIMENSION, "lu_blocked: block size must be at least 1");
  if (A->ld != A->cols) return fail(h, MPGPU_ERR_DOMAIN, "lu_blocked: dense matrix required");
  const int64_t n = A->rows;
  if (n > K && kernel != MPGPU_SIMPLE && n_min == 0)
    return fail(h, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (kernel < MPGPU_SIMPLE || kernel > MPGPU_WINOGRAD) return fail(h, MPGPU_ERR_DOMAIN, "unknown kernel");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (stats) std::memset(stats, 0, sizeof *stats);
  if (pivoting && h->d_piv_cap < n) {
    if (h->d_piv) cudaFree(h->d_piv);
    h->d_piv = nullptr;
    CUDA_TRY(h, cudaMalloc(&h->d_piv, sizeof(int64_t) * n));
    h->d_piv_cap = n;
  }
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * A->nlimbs - A->prec;
  int64_t* zp = reinterpret_cast<int64_t*>(h->d_err + 2);
  Timer total(stats != nullptr, h->stream);
  std::deque<mpgpu_stats> panel_stats;
  int rc = dispatch_L(A->nlimbs, [&](auto Lc) -> int {
    constexpr int L = decltype(Lc)::value;
    constexpr int S = rec_stride(L);
    cudaStream_t st = h->stream;
    uint32_t* a = A->rec;
    int64_t off = 0;
    DevBuf cand;
    constexpr int kMaxGrid = 4096;
    const bool coop = cand.alloc(h, 3 * sizeof(uint64_t) * kMaxGrid) == cudaSuccess &&
                      cudaMemsetAsync(cand.p, 0, 3 * sizeof(uint64_t) * kMaxGrid, st) == cudaSuccess &&
                      std::getenv("MPGPU_LU_PER_COLUMN") == nullptr;
    const bool coop_piv = std::getenv("MPGPU_LU_PIVOT_PER_COLUMN") == nullptr;
    DevBuf cbuf;
    mpg::PivotCands pc;
    if (pivoting) {
      const int64_t cap = (n + 7) / 8 + 1;
      CUDA_TRY(h, cbuf.alloc(h, cap * (sizeof(uint64_t) + sizeof(int64_t) + sizeof(int))));
      pc.key = static_cast<uint64_t*>(cbuf.p);
      pc.idx = reinterpret_cast<int64_t*>(pc.key + cap);
      pc.cnt = reinterpret_cast<int*>(pc.idx + cap);
      pc.cap = cap;
    }
    // the panel factorisation (lu_inplace + trsm_upper_right_inplace over the tall panel, with the
    // interchanges inside the panel columns) on stream `ps`; grid_cap > 0 bounds the cooperative grid
    // (the look-ahead leaves the other SMs to the Schur update running beside it)
    auto panel_factor = [&](int64_t p, int64_t k, cudaStream_t ps, int grid_cap) {
      if (coop && (!pivoting || coop_piv) &&
          mpg::launch_lu_panel_coop<L>(a, n, p, k, n, pivoting, h->d_piv, zp, sh, static_cast<uint64_t*>(cand.p),
                                       reinterpret_cast<int64_t*>(static_cast<uint64_t*>(cand.p) + kMaxGrid),
                                       grid_cap > 0 ? grid_cap : kMaxGrid, ps) == 0)
        return;
      int64_t ncand = 0;  // candidates written by the previous step (0: scan the column)
      for (int64_t d = p; d < p + k; ++d) {
        if (pivoting) mpg::launch_pivot<L>(a, n, d, n, h->d_piv, zp, pc, ncand, p, p + k, ps);
        ncand = mpg::launch_lu_step<L>(a, n, d, n, p + k, sh, h->d_err, pivoting ? pc : mpg::PivotCands{}, ps);
      }
    };
    // the panel's interchanges applied to the other columns (after every writer of them)
    auto panel_swap = [&](int64_t p, int64_t k) {
      if (pivoting) mpg::launch_laswp<L>(a, n, p, k, h->d_piv, zp, st);
    };
    // look-ahead (default on; MPGPU_LU_LOOKAHEAD=0 disables): part A of the Schur update (the next
    // panel's columns), then the next panel on the high-priority stream beside part B
    static const bool la_env = [] {
      const char* e = std::getenv("MPGPU_LU_LOOKAHEAD");
      return !(e && e[0] == '0');
    }();
    const int la_grid_big = [] {
      const char* e = std::getenv("MPGPU_LU_LA_GRID");
      return e ? std::atoi(e) : 32;  // measured: 16 54.2, 32 52.1, 64 53.4, 148 58.3 ms (n=2048, K=64)
    }();
    // once the rest of the Schur update is shorter than the look-ahead panel (the trailing
    // matrix below ~1000 rows at 256 bits), the panel is the step's critical path: give it
    // the whole grid
    const int64_t la_switch = [] {
      const char* e = std::getenv("MPGPU_LU_LA_SWITCH");
      return e ? std::atoll(e) : (int64_t)768;  // measured (n=2048 @256, K=64): 0 43.91, 512 43.73, 768 43.44, 1024 44.09 ms
    }();
    auto la_grid_for = [&](int64_t rest) { return rest > la_switch ? la_grid_big : 0; };
    const bool lookahead = la_env && L <= 32;
    if (lookahead && !h->hi) {
      int lo = 0, hi_pr = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi_pr);
      CUDA_TRY(h, cudaStreamCreateWithPriority(&h->hi, cudaStreamNonBlocking, hi_pr));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_la, cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_lp, cudaEventDisableTiming));
    }
    LuHostIO* io = h->lu_io;
    bool swapped0 = false;  // the first interchange pass (it touches every column) has been issued
    auto before_swap = [&]() -> int {
      if (io && !swapped0 && io->before_swap0) {
        swapped0 = true;
        return io->before_swap0();
      }
      swapped0 = true;
      return 0;
    };
    if (io && io->before_panel0)
      if (int r = io->before_panel0()) return r;
    bool factored = false;  // the panel at `off` was already factored by the look-ahead
    // MPGPU_LU_TRACE=1: per-step event times to stderr (diagnostics of the look-ahead overlap)
    static const bool lu_trace = std::getenv("MPGPU_LU_TRACE") != nullptr;
    struct Mark {
      int64_t off;
      const char* what;
      cudaEvent_t e;
    };
    std::vector<Mark> tmarks;
    auto tmark = [&](const char* what, cudaStream_t on) {
      if (!lu_trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, on);
      tmarks.push_back({off, what, e});
    };
    tmark("start", st);
    while (n - off > K) {
      const int64_t rest = n - off - K;
      if (!factored) panel_factor(off, K, st, 0);
      tmark("panel(st)", st);
      if (int r = before_swap()) return r;
      panel_swap(off, K);
      mpg::launch_trsm_l_panel<L>(a, n, off, K, off + K, rest, sh, st);
      // rows [off, off + K) are final: later interchanges involve rows >= off + K only
      if (io && io->rows_final)
        if (int r = io->rows_final(off, K)) return r;
      tmark("swap+trsm", st);
      const uint32_t* l21 = a + ((off + K) * n + off) * S;
      const uint32_t* u12 = a + (off * n + off + K) * S;
      uint32_t* a22 = a + ((off + K) * n + off + K) * S;
      panel_stats.emplace_back();
      mpgpu_stats& ss = panel_stats.back();  // deque: stable address until the final flush
      factored = false;
      if (lookahead && rest > K && schur_split_ok(kernel, rest, K, n_min, K)) {
        panel_stats.emplace_back();
        mpgpu_stats& sb = panel_stats.back();
        SchurSplit<L> sp;
        int r = schur_part_a<L>(h, sp, kernel, n_min, l21, u12, a22, n, rest, K, K, sh, stats ? &ss : nullptr);
        if (r) return r;
        tmark("part A", st);
        CUDA_TRY(h, cudaEventRecord(h->ev_la, st));
        CUDA_TRY(h, cudaStreamWaitEvent(h->hi, h->ev_la, 0));
        panel_factor(off + K, K, h->hi, la_grid_for(rest));
        tmark("next panel(hi)", h->hi);
        CUDA_TRY(h, cudaEventRecord(h->ev_lp, h->hi));
        r = schur_part_b<L>(h, sp, kernel, n_min, l21, u12, a22, n, rest, K, K, sh, stats ? &sb : nullptr);
        if (r) return r;
        tmark("part B", st);
        CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_lp, 0));
        factored = true;
      } else if (kernel == MPGPU_SIMPLE || kernel == MPGPU_BLOCK) {
        int r = run_gemm<L>(h, kernel, n_min, l21, n, u12, n, a22, n, rest, K, rest, sh, stats ? &ss : nullptr, 1);
        if (r) return r;
      } else {
        DevBuf prod;
        CUDA_TRY(h, prod.alloc(h, sizeof(uint32_t) * S * rest * rest));
        int r = run_gemm<L>(h, kernel, n_min, l21, n, u12, n, prod.u32(), rest, rest, K, rest, sh,
                            stats ? &ss : nullptr, 0);
        if (r) return r;
        mpg::launch_sub2d<L>(a22, n, prod.u32(), (int)rest, (int)rest, sh, h->d_err, st);
      }
      if (stats) {
        uint64_t c[2];
        count_fast_rec(kernel, rest, K, rest, n_min, c);
        stats->mul += c[0];
        stats->addsub += c[1];
      }
      off += K;
    }
    if (!factored) panel_factor(off, n - off, st, 0);
    if (int r = before_swap()) return r;
    panel_swap(off, n - off);
    if (io && io->rows_final)
      if (int r = io->rows_final(off, n - off)) return r;
    tmark("end", st);
    if (lu_trace) {
      cudaDeviceSynchronize();
      float prev = 0;
      for (const Mark& mk : tmarks) {
        float ms = 0;
        cudaEventElapsedTime(&ms, tmarks[0].e, mk.e);
        fprintf(stderr, "[lu] off %5lld %-15s %9.3f ms  (+%.3f)\n", (long long)mk.off, mk.what, ms, ms - prev);
        prev = ms;
      }
      for (const Mark& mk : tmarks) cudaEventDestroy(mk.e);
    }
    return 0;
  });
  if (stats) {
    total.stop(&stats->device_ms);
    flush_timers();  // resolve the Schur GEMMs' queued timings (no host sync per panel)
    for (const mpgpu_stats& ss : panel_stats) {
      stats->leaf_ms += ss.leaf_ms;
      stats->leaf_madds += ss.leaf_madds;
      stats->launches += ss.launches;
    }
  }
  if (rc) return rc;
  int64_t zpv = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&zpv, zp, sizeof zpv, cudaMemcpyDeviceToHost, h->stream));
  if (pivoting && piv_out)
    CUDA_TRY(h, cudaMemcpyAsync(piv_out, h->d_piv, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, h->stream));
  rc = check_err(h);
  if (zpv) {
    if (zero_pivot) *zero_pivot = zpv;
    return fail(h, MPGPU_ERR_SINGULAR, "zero pivot at index %lld", (long long)zpv);
  }
  return rc;
}

namespace {
int lu_solve_impl(mpgpu_handle* h, const mpgpu_mat* F, const int64_t* piv, const mpgpu_mat* b, mpgpu_mat* x,
                  int exact, int64_t* zero_pivot, int64_t nrhs) {
  const int64_t n = F->rows;
  if (b->prec != F->prec || x->prec != F->prec) return fail(h, MPGPU_ERR_DOMAIN, "lu_solve: mixed precisions");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  int64_t* zp = reinterpret_cast<int64_t*>(h->d_err + 2);
  DevBuf dpiv, scratch;
  if (piv) {
    CUDA_TRY(h, dpiv.alloc(h, sizeof(int64_t) * n));
    CUDA_TRY(h, cudaMemcpyAsync(dpiv.p, piv, sizeof(int64_t) * n, cudaMemcpyHostToDevice, h->stream));
  }
  const int sh = 32 * F->nlimbs - F->prec;
  int rc = dispatch_L(F->nlimbs, [&](auto Lc) -> int {
    constexpr int L = decltype(Lc)::value;
    CUDA_TRY(h, scratch.alloc(h, sizeof(uint32_t) * rec_stride(L) * 2 * n * nrhs));
    mpg::launch_lu_solve<L>(F->rec, n, piv ? static_cast<const int64_t*>(dpiv.p) : nullptr, b->rec, x->rec,
                            scratch.u32(), sh, h->d_err, zp, exact, nrhs, h->stream);
    return 0;
  });
  if (rc) return rc;
  int64_t zpv = 0;
  CUDA_TRY(h, cudaMemcpyAsync(&zpv, zp, sizeof zpv, cudaMemcpyDeviceToHost, h->stream));
  rc = check_err(h);
  if (zpv) {
    if (zero_pivot) *zero_pivot = zpv;
    return fail(h, MPGPU_ERR_SINGULAR, "zero pivot at index %lld", (long long)zpv);
  }
  return rc;
}
}  // namespace

// blocked LU from and to HOST SoA buffers (in place), the transfers overlapped with the
// factorisation: columns [0, K) are copied first (the first panel needs only them), the
// rest while that panel is factored; after step k's trsm rows [kK, (k+1)K) are final (every
// later interchange involves rows >= (k+1)K) and are copied back while the factorisation
// goes on.  Same kernels, same order: the factors are bit-identical to mpgpu_lu_blocked's.
int mpgpu_lu_blocked_host(mpgpu_handle* h, int32_t prec, int64_t n, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                          int32_t host_nlimbs, int64_t K, int kernel, int64_t n_min, int pivoting, int64_t* piv_out,
                          int64_t* zero_pivot, mpgpu_stats* stats) {
  if (!h || !limbs || !exp || !sign) return MPGPU_ERR_DOMAIN;
  if (zero_pivot) *zero_pivot = 0;
  if (n < 1) return fail(h, MPGPU_ERR_DIMENSION, "lu_blocked: matrix must be at least 1x1");
  if (K == 0) return fail(h, MPGPU_ERR_DIMENSION, "lu_blocked: block size must be at least 1");
  const int L = nlimbs_for(prec);
  if (!L) return fail(h, MPGPU_ERR_DOMAIN, "precision %d outside the device range", prec);
  if (host_nlimbs < (prec + 31) / 32) return fail(h, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  int rc;
  if (host_nlimbs != L || n <= 1 || !host_pipe_enabled() || !host_pinned({limbs, exp, sign})) {
    // plain sequence: upload, factor, download
    mpgpu_mat A{};
    rc = mpgpu_alloc_matrix(h, n, n, prec, &A);
    if (rc) return rc;
    rc = mpgpu_upload(h, &A, limbs, exp, sign, host_nlimbs);
    if (!rc) rc = mpgpu_lu_blocked(h, &A, K, kernel, n_min, pivoting, piv_out, zero_pivot, stats);
    if (!rc) rc = mpgpu_download(h, &A, limbs, exp, sign, host_nlimbs);
    mpgpu_free_matrix(h, &A);
    return rc;
  }
  const int64_t K0 = std::min<int64_t>(K, n);
  const size_t soa = sizeof(uint32_t) * L + sizeof(int32_t) + 1;
  auto al256 = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b0 = al256(soa * (size_t)(n * K0)), b1 = al256(soa * (size_t)(n * (n - K0)) + 1);
  const size_t brec = al256(sizeof(uint32_t) * (size_t)rec_stride(L) * (size_t)(n * n));
  const size_t total_bytes = brec + b0 + b1 + al256(soa * (size_t)(n * n));
  // the device matrix and the SoA staging from the stream-ordered pool (no cudaMalloc /
  // cudaFree, which synchronise, per call): records | column block 0 | the other columns |
  // the factored rows
  uint8_t* pool = nullptr;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    cudaSetDevice(h->device);
    if (!h->aux) {
      CUDA_TRY(h, cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
    }
    if (!h->dl) {
      CUDA_TRY(h, cudaStreamCreateWithFlags(&h->dl, cudaStreamNonBlocking));
      for (cudaEvent_t& e : h->pev) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if ((rc = ensure_pool(h, total_bytes + total_bytes / 8))) return rc;
    CUDA_TRY(h, cudaMallocAsync(reinterpret_cast<void**>(&pool), total_bytes, h->stream));
  }
  struct FreePool {
    mpgpu_handle* h;
    uint8_t* p;
    ~FreePool() {
      if (h->aux) cudaStreamSynchronize(h->aux);
      if (h->dl) cudaStreamSynchronize(h->dl);
      cudaFreeAsync(p, h->stream);
      cudaStreamSynchronize(h->stream);
    }
  } free_pool{h, pool};
  mpgpu_mat A{n, n, prec, L, reinterpret_cast<uint32_t*>(pool), n, 0};
  uint8_t* stage = pool + brec;
  cudaEvent_t up0 = h->pev[0], up1 = h->pev[1], ready = h->pev[12];
  // the device matrix exists (allocated on the handle's stream) before the copies land
  CUDA_TRY(h, cudaEventRecord(ready, h->stream));
  CUDA_TRY(h, cudaStreamWaitEvent(h->aux, ready, 0));
  CUDA_TRY(h, cudaStreamWaitEvent(h->dl, ready, 0));
  struct Blk {
    uint32_t* l;
    int32_t* e;
    uint8_t* s;
  };
  auto blk = [&](uint8_t* base, int64_t N) {
    Blk b;
    b.l = reinterpret_cast<uint32_t*>(base);
    b.e = reinterpret_cast<int32_t*>(b.l + (size_t)L * N);
    b.s = reinterpret_cast<uint8_t*>(b.e + N);
    return b;
  };
  const Blk s0 = blk(stage, n * K0), s1 = blk(stage + b0, n * (n - K0)), sd = blk(stage + b0 + b1, n * n);
  // copies in (aux stream): columns [c0, c0 + w) of every row into a dense n x w SoA block
  auto copy_cols = [&](const Blk& d, int64_t c0, int64_t w, cudaEvent_t ev) -> int {
    if (w <= 0) {
      CUDA_TRY(h, cudaEventRecord(ev, h->aux));
      return MPGPU_OK;
    }
    const int64_t N = n * w;
    for (int j = 0; j < L; ++j)
      CUDA_TRY(h, cudaMemcpy2DAsync(d.l + (size_t)j * N, sizeof(uint32_t) * w, limbs + (size_t)j * n * n + c0,
                                    sizeof(uint32_t) * n, sizeof(uint32_t) * w, n, cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaMemcpy2DAsync(d.e, sizeof(int32_t) * w, exp + c0, sizeof(int32_t) * n, sizeof(int32_t) * w, n,
                                  cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaMemcpy2DAsync(d.s, w, sign + c0, n, w, n, cudaMemcpyHostToDevice, h->aux));
    CUDA_TRY(h, cudaEventRecord(ev, h->aux));
    return MPGPU_OK;
  };
  if ((rc = copy_cols(s0, 0, K0, up0)) || (rc = copy_cols(s1, K0, n - K0, up1))) return rc;
  // conversions on the factorisation's stream, just before the data is needed
  auto convert = [&](const Blk& b, int64_t c0, int64_t w, cudaEvent_t ev) -> int {
    CUDA_TRY(h, cudaStreamWaitEvent(h->stream, ev, 0));
    if (w <= 0) return MPGPU_OK;
    return dispatch_store(L, [&](auto Lc) {
      constexpr int LL = decltype(Lc)::value;
      mpg::launch_soa2rec_2d<LL>(b.l, b.e, b.s, n, w, n * w, A.rec + c0 * rec_stride(LL), n, h->stream);
      return 0;
    });
  };
  LuHostIO io;
  io.before_panel0 = [&]() { return convert(s0, 0, K0, up0); };
  io.before_swap0 = [&]() { return convert(s1, K0, n - K0, up1); };
  int nrow_ev = 0;
  io.rows_final = [&](int64_t r0, int64_t nr) -> int {
    cudaEvent_t ev = h->pev[2 + (nrow_ev++ % 10)];  // (each is waited on right after it is recorded)
    CUDA_TRY(h, cudaEventRecord(ev, h->stream));
    CUDA_TRY(h, cudaStreamWaitEvent(h->dl, ev, 0));
    const int64_t N = nr * n, off = r0 * n;
    dispatch_store(L, [&](auto Lc) {
      constexpr int LL = decltype(Lc)::value;
      mpg::launch_rec2soa<LL>(A.rec + off * rec_stride(LL), N, sd.l + off, sd.e + off, sd.s + off, n * n, h->dl);
      return 0;
    });
    for (int j = 0; j < L; ++j)
      CUDA_TRY(h, cudaMemcpyAsync(limbs + (size_t)j * n * n + off, sd.l + (size_t)j * n * n + off,
                                  sizeof(uint32_t) * N, cudaMemcpyDeviceToHost, h->dl));
    CUDA_TRY(h, cudaMemcpyAsync(exp + off, sd.e + off, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, h->dl));
    CUDA_TRY(h, cudaMemcpyAsync(sign + off, sd.s + off, N, cudaMemcpyDeviceToHost, h->dl));
    return MPGPU_OK;
  };
  h->lu_io = &io;
  rc = mpgpu_lu_blocked(h, &A, K, kernel, n_min, pivoting, piv_out, zero_pivot, stats);
  h->lu_io = nullptr;
  CUDA_TRY(h, cudaStreamSynchronize(h->dl));
  return rc;
}

int mpgpu_lu_solve(mpgpu_handle* h, const mpgpu_mat* F, const int64_t* piv, const mpgpu_mat* b, mpgpu_mat* x,
                   int exact, int64_t* zero_pivot) {
  if (!h || !F || !b || !x) return MPGPU_ERR_DOMAIN;
  if (zero_pivot) *zero_pivot = 0;
  if (int r = compute_range(h, {F, b, x})) return r;
  const int64_t n = F->rows;
  if (F->rows != F->cols) return fail(h, MPGPU_ERR_DIMENSION, "lu_solve: factors must be square");
  if (b->rows * b->cols != n || x->rows * x->cols != n) return fail(h, MPGPU_ERR_DIMENSION, "lu_solve: length mismatch");
  return lu_solve_impl(h, F, piv, b, x, exact, zero_pivot, 1);
}

int mpgpu_lu_solve_many(mpgpu_handle* h, const mpgpu_mat* F, const int64_t* piv, const mpgpu_mat* Bt, mpgpu_mat* Xt,
                        int exact, int64_t* zero_pivot) {
  if (!h || !F || !Bt || !Xt) return MPGPU_ERR_DOMAIN;
  if (zero_pivot) *zero_pivot = 0;
  if (int r = compute_range(h, {F, Bt, Xt})) return r;
  const int64_t n = F->rows;
  if (F->rows != F->cols) return fail(h, MPGPU_ERR_DIMENSION, "lu_solve: factors must be square");
  if (Bt->cols != n || Xt->cols != n || Xt->rows != Bt->rows)
    return fail(h, MPGPU_ERR_DIMENSION, "lu_solve_many: right-hand sides must be r x n (one per row)");
  if (Bt->ld != Bt->cols || Xt->ld != Xt->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "lu_solve_many: strided views are not supported");
  return lu_solve_impl(h, F, piv, Bt, Xt, exact, zero_pivot, Bt->rows);
}

int mpgpu_convert(mpgpu_handle* h, const mpgpu_mat* src, mpgpu_mat* dst) {
  if (!h || !src || !dst) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {dst})) return r;
  if (src->rows != dst->rows || src->cols != dst->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "convert: shape mismatch");
  if (src->ld != src->cols || dst->ld != dst->cols) return fail(h, MPGPU_ERR_DIMENSION, "convert: strided view");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * dst->nlimbs - dst->prec;
  int rc = dispatch_L(dst->nlimbs, [&](auto Lc) {
    mpg::launch_convert<decltype(Lc)::value>(src->rec, src->nlimbs, src->rows * src->cols, dst->rec, sh, h->d_err,
                                             h->stream);
    return 0;
  });
  if (rc) return rc;
  return check_err(h);
}

int mpgpu_fast_plan(int64_t m, int64_t l, int64_t n, int64_t n_min, int64_t* out5) {
  if (n_min < 1 || m < 1 || l < 1 || n < 1) return MPGPU_ERR_DIMENSION;
  const std::vector<Level> lv = plan_levels(m, l, n, n_min);
  const int d = (int)lv.size() - 1;
  int64_t leaves = 1;
  for (int i = 0; i < d; ++i) leaves *= 7;
  out5[0] = d;
  out5[1] = leaves;
  out5[2] = lv[d].m;
  out5[3] = lv[d].l;
  out5[4] = lv[d].n;
  return MPGPU_OK;
}

namespace {
int fast_leaves_impl(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                     int up_levels, int64_t node_lo, int64_t node_hi, uint32_t* node_products,
                     const uint64_t* rowtab, mpgpu_stats* stats);
}

int mpgpu_fast_leaves(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                      int up_levels, int64_t node_lo, int64_t node_hi, uint32_t* node_products, mpgpu_stats* stats) {
  if (!node_products) return MPGPU_ERR_DOMAIN;
  return fast_leaves_impl(h, algo, n_min, A, B, up_levels, node_lo, node_hi, node_products, nullptr, stats);
}

int mpgpu_fast_leaves_rows(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                           int up_levels, int64_t node_lo, int64_t node_hi, const uint64_t* row_dst,
                           mpgpu_stats* stats) {
  if (!row_dst) return MPGPU_ERR_DOMAIN;
  if (A && A->nlimbs > 32) return fail(h, MPGPU_ERR_DOMAIN, "row destinations: precisions up to 1024 bits");
  return fast_leaves_impl(h, algo, n_min, A, B, up_levels, node_lo, node_hi, nullptr, row_dst, stats);
}

}  // extern "C"

namespace {
int fast_leaves_impl(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                     int up_levels, int64_t node_lo, int64_t node_hi, uint32_t* node_products,
                     const uint64_t* rowtab, mpgpu_stats* stats) {
  TimerGuard timer_guard;
  if (!h || !A || !B) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {A, B})) return r;
  if (A->cols != B->rows) return fail(h, MPGPU_ERR_DIMENSION, "inner dimension mismatch");
  if (n_min < 1) return fail(h, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD)
    return fail(h, MPGPU_ERR_DOMAIN, "fast_mul: algorithm must be strassen or winograd");
  if (A->prec != B->prec || A->nlimbs != B->nlimbs) return fail(h, MPGPU_ERR_DOMAIN, "one precision required");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (stats) std::memset(stats, 0, sizeof *stats);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * A->nlimbs - A->prec;
  int rc = dispatch_L(A->nlimbs, [&](auto Lc) {
    return run_fast_leaves<decltype(Lc)::value>(h, algo, n_min, A->rec, A->ld, B->rec, B->ld, A->rows, A->cols,
                                                B->cols, node_lo, node_hi, up_levels, node_products, sh, stats,
                                                rowtab);
  });
  if (rc) return rc;
  return check_err(h);
}
}  // namespace

extern "C" {

int mpgpu_fast_combine(mpgpu_handle* h, int algo, int64_t n_min, int64_t l, int up_levels,
                       const uint32_t* node_products, mpgpu_mat* C, mpgpu_stats* stats) {
  TimerGuard timer_guard;
  if (!h || !C || !node_products) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {C})) return r;
  if (n_min < 1) return fail(h, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD)
    return fail(h, MPGPU_ERR_DOMAIN, "fast_mul: algorithm must be strassen or winograd");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (stats) std::memset(stats, 0, sizeof *stats);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * C->nlimbs - C->prec;
  int rc = dispatch_L(C->nlimbs, [&](auto Lc) {
    return run_fast_combine<decltype(Lc)::value>(h, algo, n_min, node_products, up_levels, C->rows, l, C->cols,
                                                 C->rec, C->ld, sh, stats);
  });
  if (rc) return rc;
  return check_err(h);
}

int mpgpu_fast_combine_rows(mpgpu_handle* h, int algo, int64_t n_min, int64_t l, int up_levels,
                            const uint32_t* node_products, int64_t row_lo, int64_t row_hi, mpgpu_mat* C,
                            mpgpu_stats* stats) {
  TimerGuard timer_guard;
  if (!h || !C || !node_products) return MPGPU_ERR_DOMAIN;
  if (int r = compute_range(h, {C})) return r;
  if (n_min < 1) return fail(h, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (algo != MPGPU_STRASSEN && algo != MPGPU_WINOGRAD)
    return fail(h, MPGPU_ERR_DOMAIN, "fast_mul: algorithm must be strassen or winograd");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  if (stats) std::memset(stats, 0, sizeof *stats);
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * C->nlimbs - C->prec;
  int rc = dispatch_L(C->nlimbs, [&](auto Lc) {
    return run_fast_combine<decltype(Lc)::value>(h, algo, n_min, node_products, up_levels, C->rows, l, C->cols,
                                                 C->rec, C->ld, sh, stats, row_lo, row_hi);
  });
  if (rc) return rc;
  return check_err(h);
}

int mpgpu_copy_device_2d(mpgpu_handle* h, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                         size_t height) {
  if (!h) return MPGPU_ERR_DOMAIN;
  if (width == 0 || height == 0) return MPGPU_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice, h->stream));
  return MPGPU_OK;
}

// ---- device memory shared between processes (one process per GPU, peer stores) --------
int mpgpu_malloc(mpgpu_handle* h, size_t bytes, void** out) {
  if (!h || !out) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaMalloc(out, bytes < 16 ? 16 : bytes));
  return MPGPU_OK;
}

int mpgpu_free(mpgpu_handle* h, void* p) {
  if (!h) return MPGPU_ERR_DOMAIN;
  if (!p) return MPGPU_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaFree(p));
  return MPGPU_OK;
}

int mpgpu_ipc_handle(mpgpu_handle* h, void* p, void* handle_out) {
  if (!h || !p || !handle_out) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  cudaIpcMemHandle_t ih;
  CUDA_TRY(h, cudaIpcGetMemHandle(&ih, p));
  std::memcpy(handle_out, &ih, sizeof ih);
  return MPGPU_OK;
}

int mpgpu_ipc_open(mpgpu_handle* h, const void* handle, void** out) {
  if (!h || !handle || !out) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  cudaIpcMemHandle_t ih;
  std::memcpy(&ih, handle, sizeof ih);
  CUDA_TRY(h, cudaIpcOpenMemHandle(out, ih, cudaIpcMemLazyEnablePeerAccess));
  return MPGPU_OK;
}

int mpgpu_ipc_close(mpgpu_handle* h, void* p) {
  if (!h) return MPGPU_ERR_DOMAIN;
  if (!p) return MPGPU_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  CUDA_TRY(h, cudaIpcCloseMemHandle(p));
  return MPGPU_OK;
}

// ---- accuracy metrics (metrics.cu) -------------------------------------------
namespace {
// elementwise metric kernel + reduction, then the three result records -> host SoA
// (count = how many of them the caller wants: 2 or 1)
int run_metric(mpgpu_handle* h, int mode, const mpgpu_mat* approx, const mpgpu_mat* ref, int count, int which0,
               int which1, uint32_t* ol, int32_t* oe, uint8_t* os, int64_t* counted, bool* empty_a) {
  const int L = ref->nlimbs;
  const int64_t N = ref->rows * ref->cols;
  const int S = rec_stride(L);
  DevBuf bufA, bufB, scratch, out3, cnt, soa;
  CUDA_TRY(h, bufA.alloc(h, sizeof(uint32_t) * S * N));
  if (mode == 1) CUDA_TRY(h, bufB.alloc(h, sizeof(uint32_t) * S * N));
  CUDA_TRY(h, scratch.alloc(h, sizeof(uint32_t) * S * 3 * 1024));
  CUDA_TRY(h, out3.alloc(h, sizeof(uint32_t) * S * 3));
  CUDA_TRY(h, cnt.alloc(h, sizeof(unsigned long long)));
  CUDA_TRY(h, cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), h->stream));
  CUDA_TRY(h, cudaMemsetAsync(h->d_err, 0, 4 * sizeof(uint32_t), h->stream));
  const int sh = 32 * L - ref->prec;
  int rc = dispatch_store(L, [&](auto Lc) {
    constexpr int LL = decltype(Lc)::value;
    if (mode == 2) {
      mpg::launch_colsum_abs<LL>(ref->rec, ref->ld, (int)ref->rows, (int)ref->cols, sh, bufA.u32(), h->d_err,
                                 h->stream);
      mpg::launch_reduce3<LL>(bufA.u32(), nullptr, ref->cols, out3.u32(), scratch.u32(), h->stream);
    } else {
      mpg::launch_rel_error<LL>(approx->rec, approx->nlimbs, approx->ld, ref->rec, ref->ld, (int)ref->rows,
                                (int)ref->cols, mode, sh, bufA.u32(), mode == 1 ? bufB.u32() : nullptr,
                                static_cast<unsigned long long*>(cnt.p), h->d_err, h->stream);
      mpg::launch_reduce3<LL>(bufA.u32(), mode == 1 ? bufB.u32() : nullptr, N, out3.u32(), scratch.u32(),
                              h->stream);
    }
    return 0;
  });
  if (rc) return fail(h, MPGPU_ERR_DOMAIN, "metric: unsupported limb count %d", L);
  // read back the three records and the counter
  std::vector<uint32_t> host(3 * S);
  unsigned long long c = 0;
  CUDA_TRY(h, cudaMemcpyAsync(host.data(), out3.p, sizeof(uint32_t) * 3 * S, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaMemcpyAsync(&c, cnt.p, sizeof c, cudaMemcpyDeviceToHost, h->stream));
  rc = check_err(h);
  if (rc) return rc;
  if (counted) *counted = (int64_t)c;
  *empty_a = (host[L + 1] & 2u) != 0;
  const int which[2] = {which0, which1};
  for (int e = 0; e < count; ++e) {
    const uint32_t* r = host.data() + which[e] * S;
    const bool skip = (r[L + 1] & 2u) != 0;  // empty set: +0
    for (int k = 0; k < L; ++k) ol[(size_t)k * count + e] = skip ? 0u : r[k];
    oe[e] = skip ? MPGPU_EXP_ZERO : (int32_t)r[L];
    os[e] = skip ? 0 : (uint8_t)(r[L + 1] & 1u);
  }
  return MPGPU_OK;
}
}  // namespace

int mpgpu_max_rel_error(mpgpu_handle* h, const mpgpu_mat* approx, const mpgpu_mat* ref, uint32_t* ol, int32_t* oe,
                        uint8_t* os, int64_t* skipped) {
  if (!h || !approx || !ref || !ol || !oe || !os) return MPGPU_ERR_DOMAIN;
  if (approx->rows != ref->rows || approx->cols != ref->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "shape mismatch: %lldx%lld vs %lldx%lld", (long long)approx->rows,
                (long long)approx->cols, (long long)ref->rows, (long long)ref->cols);
  if (approx->nlimbs > ref->nlimbs)
    return fail(h, MPGPU_ERR_DOMAIN, "max_rel_error: the approximation is wider than the reference");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  bool empty = false;
  int rc = run_metric(h, 0, approx, ref, 2, 0, 1, ol, oe, os, skipped, &empty);
  if (rc) return rc;
  if (empty) return fail(h, MPGPU_ERR_UNDEFINED_METRIC, "max_rel_error: all reference entries are zero");
  return MPGPU_OK;
}

int mpgpu_solution_error(mpgpu_handle* h, const mpgpu_mat* xhat, const mpgpu_mat* xtrue, uint32_t* ol, int32_t* oe,
                         uint8_t* os, int64_t* zero_refs) {
  if (!h || !xhat || !xtrue || !ol || !oe || !os) return MPGPU_ERR_DOMAIN;
  if (xhat->rows * xhat->cols != xtrue->rows * xtrue->cols)
    return fail(h, MPGPU_ERR_DIMENSION, "solution error: length mismatch");
  if (xhat->cols != 1 || xtrue->cols != 1)
    return fail(h, MPGPU_ERR_DIMENSION, "solution error: vectors are n x 1 matrices");
  if (xhat->nlimbs > xtrue->nlimbs)
    return fail(h, MPGPU_ERR_DOMAIN, "solution error: the solution is wider than the reference");
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  bool empty = false;
  int rc = run_metric(h, 1, xhat, xtrue, 2, 0, 2, ol, oe, os, zero_refs, &empty);
  if (rc) return rc;
  if (empty) return fail(h, MPGPU_ERR_UNDEFINED_METRIC, "solution error: all reference components are zero");
  return MPGPU_OK;
}

int mpgpu_one_norm(mpgpu_handle* h, const mpgpu_mat* A, uint32_t* ol, int32_t* oe, uint8_t* os) {
  if (!h || !A || !ol || !oe || !os) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(h->mu);
  cudaSetDevice(h->device);
  bool empty = false;
  return run_metric(h, 2, nullptr, A, 1, 0, 0, ol, oe, os, nullptr, &empty);
}

int mpgpu_matrix_view(const mpgpu_mat* parent, int64_t r0, int64_t c0, int64_t rows, int64_t cols, mpgpu_mat* out) {
  if (!parent || !out) return MPGPU_ERR_DOMAIN;
  if (rows < 1 || cols < 1 || r0 < 0 || c0 < 0 || r0 + rows > parent->rows || c0 + cols > parent->cols)
    return MPGPU_ERR_DIMENSION;
  *out = *parent;
  out->rows = rows;
  out->cols = cols;
  out->rec = parent->rec + (r0 * parent->ld + c0) * rec_stride(parent->nlimbs);
  out->owned = 0;
  return MPGPU_OK;
}

int mpgpu_count_fast(int algo, int64_t m, int64_t l, int64_t n, int64_t n_min, uint64_t* out2) {
  if (m < 1 || l < 1 || n < 1) return MPGPU_ERR_DIMENSION;
  if (n_min == 0 && algo >= MPGPU_STRASSEN) return MPGPU_ERR_DIMENSION;
  count_fast_rec(algo, m, l, n, n_min, out2);
  return MPGPU_OK;
}

int mpgpu_recursion_plan(int64_t m, int64_t l, int64_t n, int64_t n_min, int64_t* out, int max_levels, int* count) {
  if (n_min == 0) return MPGPU_ERR_DIMENSION;
  int lev = 0;
  for (;;) {
    const bool base = std::min({m, l, n}) <= n_min;
    const int64_t pm = base ? m : m + m % 2, pl = base ? l : l + l % 2, pn = base ? n : n + n % 2;
    if (lev < max_levels) {
      int64_t* r = out + 8 * lev;
      r[0] = lev;
      r[1] = m;
      r[2] = l;
      r[3] = n;
      r[4] = pm;
      r[5] = pl;
      r[6] = pn;
      r[7] = base;
    }
    ++lev;
    if (base) break;
    m = pm / 2;
    l = pl / 2;
    n = pn / 2;
  }
  *count = lev;
  return MPGPU_OK;
}

int mpgpu_gen(int kind, int64_t N, uint64_t seed, int32_t prec, uint32_t* limbs, int32_t* exp, uint8_t* sign,
              int32_t Lh) {
  if (prec < 2 || prec > MPGPU_MAX_PREC || Lh < (prec + 31) / 32) return MPGPU_ERR_DOMAIN;
  Prng64 rng(seed);
  for (int64_t e = 0; e < N; ++e) {
    if (kind == 0) {
      // num = 2 k - 2^53 (|num| <= 2^53), value = RN_p(num) * 2^-53
      const int64_t num = (int64_t)(2 * rng.top53()) - ((int64_t)1 << 53);
      sign[e] = num < 0;
      uint64_t u = num < 0 ? (uint64_t)(-num) : (uint64_t)num;
      if (u == 0) {
        for (int k = 0; k < Lh; ++k) limbs[(int64_t)k * N + e] = 0;
        exp[e] = MPGPU_EXP_ZERO;
        sign[e] = 0;
        continue;
      }
      const int b = 64 - __builtin_clzll(u);
      int32_t ex = b - 53;
      uint64_t M = u << (64 - b);  // left aligned
      if (prec < 64) {
        const int drop = 64 - prec;
        const uint64_t low = M & ((1ull << drop) - 1);
        const uint64_t half = 1ull << (drop - 1);
        M -= low;
        const bool up = low > half || (low == half && ((M >> drop) & 1));
        if (up) {
          M += 1ull << drop;
          if (M == 0) {  // carried out
            M = 1ull << 63;
            ex += 1;
          }
        }
      }
      for (int k = 0; k < Lh; ++k) limbs[(int64_t)k * N + e] = 0;
      limbs[(int64_t)(Lh - 1) * N + e] = (uint32_t)(M >> 32);
      if (Lh >= 2) limbs[(int64_t)(Lh - 2) * N + e] = (uint32_t)M;
      exp[e] = ex;
    } else if (kind == 1) {
      const int need = prec + 1;
      BitWriter bw(need);
      for (int have = 0; have < need;) {
        const uint64_t d = rng.top53();
        const int take = std::min(53, need - have);
        bw.put(d >> (53 - take), take);
        have += take;
      }
      std::vector<uint32_t>& K = bw.w;
      const bool ge = (K[prec >> 5] >> (prec & 31)) & 1u;  // bit p: k >= 2^p
      std::vector<uint32_t> v(K.size(), 0);
      if (ge) {
        v = K;
        v[prec >> 5] &= ~(1u << (prec & 31));
      } else {  // v = 2^p - k
        std::vector<uint32_t> two(K.size(), 0);
        two[prec >> 5] = 1u << (prec & 31);
        uint64_t borrow = 0;
        for (size_t k = 0; k < K.size(); ++k) {
          const uint64_t t = (uint64_t)two[k] - K[k] - borrow;
          v[k] = (uint32_t)t;
          borrow = (t >> 63) & 1;
        }
      }
      const int b = bitlen(v);
      if (b == 0) {
        for (int k = 0; k < Lh; ++k) limbs[(int64_t)k * N + e] = 0;
        exp[e] = MPGPU_EXP_ZERO;
        sign[e] = 0;
        continue;
      }
      put_mantissa(v, b, Lh, N, e, limbs);
      exp[e] = b - prec;
      sign[e] = ge ? 0 : 1;
    } else {
      const uint32_t sg = (uint32_t)(rng.next64() >> 63);
      const int32_t ex = (int32_t)(rng.next64() % 41) - 20;
      const int need = prec - 1;
      BitWriter bw(prec);
      bw.put(1, 1);  // leading one
      for (int have = 0; have < need;) {
        const uint64_t d = rng.top53();
        const int take = std::min(53, need - have);
        bw.put(d >> (53 - take), take);
        have += take;
      }
      put_mantissa(bw.w, prec, Lh, N, e, limbs);
      exp[e] = ex;
      sign[e] = (uint8_t)sg;
    }
  }
  return MPGPU_OK;
}

}  // extern "C"
