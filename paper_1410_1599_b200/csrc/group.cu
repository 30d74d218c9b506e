// group.cu -- one process driving several GPUs (include/mpgpu.h "multi-GPU"): the C-ABI
// route to the 8-GPU box for C++ callers of the drop-in (mpmm::gpu::fast_mul /
// block_mul with a gpu mask).  SURVEY.md section 8(e):
//
//   Simple / Block (matrix.hpp:178-233): C split by row blocks.  Row i of C depends on row
//     i of A and all of B, and Block's k-tiles are row-independent, so every device
//     uploads its rows of A plus B, multiplies, and writes its rows of C straight into the
//     caller's host buffer.  No exchange at all.
//   Strassen / Winograd (fastmm.hpp:99-229): the recursion is split at the bottom.  Every
//     device holds A and B, runs the pre-additions of its own units only and their leaf
//     GEMMs (mpgpu_fast_leaves).  The one exchange: every device PULLS its row slice of
//     every unit product from the device that computed it (peer copies over NVLink --
//     cudaMemcpy2DAsync between device pointers with peer access enabled), then runs the
//     remaining post-additions for the rows of C it owns (mpgpu_fast_combine_rows) and
//     writes exactly those rows to the host.  Post-additions are elementwise, so the
//     result is bit-identical to one GPU (and to the reference).  No reduction anywhere:
//     MP rounded sums are order-sensitive and not a collective's operation.
//
// One host thread per device; the threads meet at two barriers (leaves done -> pull;
// pulls done -> producers may free).  A device may appear more than once in the group
// (several shards of one GPU): the same code path then runs with local copies, which is
// how it is tested on a one-GPU host.  Built only on the public C-ABI plus peer copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpgpu.h"

struct mpgpu_group {
  std::vector<int> devices;
  std::vector<mpgpu_handle*> h;
  std::mutex mu;  // one call at a time per group
  std::string last_error;
};

namespace {

int gfail(mpgpu_group* g, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g->last_error = buf;
  return code;
}

// reusable barrier for the per-device threads (C++17: no std::barrier)
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    const int gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_; });
    }
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, count_ = 0, gen_ = 0;
};

struct Range {
  int64_t lo, hi;
};
// contiguous, padded ranges as in shard.even_ranges: rank r owns [r*per, min((r+1)*per, units))
std::vector<Range> even_ranges(int64_t units, int world, int64_t* per_out = nullptr) {
  const int64_t per = std::max<int64_t>(1, (units + world - 1) / world);
  std::vector<Range> r(world);
  for (int i = 0; i < world; ++i) r[i] = {std::min<int64_t>(i * per, units), std::min<int64_t>((i + 1) * per, units)};
  if (per_out) *per_out = per;
  return r;
}

// up_levels in {0, 1} (shard.choose_split): split sibling groups (7^(d-1) units, the first
// post-addition level done locally, 4/7 of the bytes exchanged) unless that makes the busiest
// device's leaf work more than 5 % above the per-leaf split's
int choose_split(int depth, int world) {
  if (depth < 2) return 0;
  int64_t leaves = 1;
  for (int i = 0; i < depth; ++i) leaves *= 7;
  const int64_t busiest_leaf = (leaves + world - 1) / world;
  const int64_t busiest_group = 7 * ((leaves / 7 + world - 1) / world);
  return busiest_group * 100 <= 105 * busiest_leaf ? 1 : 0;
}

// contiguous runs of a sorted row list
std::vector<Range> runs_of(const std::vector<int64_t>& rows) {
  std::vector<Range> out;
  for (size_t i = 0; i < rows.size();) {
    size_t j = i + 1;
    while (j < rows.size() && rows[j] == rows[j - 1] + 1) ++j;
    out.push_back({rows[i], rows[j - 1] + 1});
    i = j;
  }
  return out;
}

struct HostSoa {
  const uint32_t* l;
  const int32_t* e;
  const uint8_t* s;
};
struct HostSoaOut {
  uint32_t* l;
  int32_t* e;
  uint8_t* s;
};

void merge_stats(mpgpu_stats* dst, const mpgpu_stats& s) {
  dst->leaf_madds += s.leaf_madds;
  dst->device_ms = std::max(dst->device_ms, s.device_ms);  // devices run concurrently: the slowest
  dst->leaf_ms = std::max(dst->leaf_ms, s.leaf_ms);
  dst->preadd_ms = std::max(dst->preadd_ms, s.preadd_ms);
  dst->postadd_ms = std::max(dst->postadd_ms, s.postadd_ms);
  dst->launches += s.launches;
  dst->depth = std::max(dst->depth, s.depth);
}

}  // namespace

extern "C" {

int mpgpu_group_init_devices(int ndev, const int* devices, mpgpu_group** out) {
  if (!out || ndev < 1 || !devices) return MPGPU_ERR_DOMAIN;
  *out = nullptr;
  auto* g = new mpgpu_group();
  for (int i = 0; i < ndev; ++i) {
    mpgpu_handle* h = nullptr;
    const int rc = mpgpu_init(devices[i], &h);
    if (rc) {
      for (mpgpu_handle* x : g->h) mpgpu_destroy(x);
      delete g;
      return rc;
    }
    g->devices.push_back(devices[i]);
    g->h.push_back(h);
  }
  // peer access between distinct devices (NVLink / NVSwitch on the box); the copies also
  // work without it (staged by the driver), only slower
  for (int a : g->devices)
    for (int b : g->devices) {
      if (a == b) continue;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok) {
        cudaSetDevice(a);
        if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
      }
    }
  *out = g;
  return MPGPU_OK;
}

int mpgpu_group_init(uint32_t gpu_mask, mpgpu_group** out) {
  if (!out) return MPGPU_ERR_DOMAIN;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return MPGPU_ERR_CUDA;
  std::vector<int> devs;
  for (int d = 0; d < 32; ++d)
    if (gpu_mask & (1u << d)) {
      if (d >= count) return MPGPU_ERR_DOMAIN;  // a selected device does not exist
      devs.push_back(d);
    }
  if (devs.empty()) return MPGPU_ERR_DOMAIN;
  return mpgpu_group_init_devices((int)devs.size(), devs.data(), out);
}

void mpgpu_group_destroy(mpgpu_group* g) {
  if (!g) return;
  for (mpgpu_handle* h : g->h) mpgpu_destroy(h);
  delete g;
}

int mpgpu_group_size(const mpgpu_group* g) { return g ? (int)g->h.size() : 0; }

int mpgpu_group_device(const mpgpu_group* g, int i) {
  return (g && i >= 0 && i < (int)g->devices.size()) ? g->devices[i] : -1;
}

mpgpu_handle* mpgpu_group_handle(mpgpu_group* g, int i) {
  return (g && i >= 0 && i < (int)g->h.size()) ? g->h[i] : nullptr;
}

const char* mpgpu_group_last_error(const mpgpu_group* g) { return g ? g->last_error.c_str() : "null group"; }

int mpgpu_group_gemm_host(mpgpu_group* g, int algo, int64_t param, int32_t prec, int64_t m, int64_t l, int64_t n,
                          const uint32_t* al, const int32_t* ae, const uint8_t* as, const uint32_t* bl,
                          const int32_t* be, const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs, int32_t Lh,
                          mpgpu_stats* stats) {
  if (!g) return MPGPU_ERR_DOMAIN;
  std::lock_guard<std::mutex> lk(g->mu);
  const int world = (int)g->h.size();
  // validation in the reference's order (fastmm.hpp:246-251, matrix.hpp:141-143)
  if (m < 1 || l < 1 || n < 1) return gfail(g, MPGPU_ERR_DIMENSION, "matrix dimensions must be at least 1x1");
  if ((algo == MPGPU_BLOCK || algo == MPGPU_STRASSEN || algo == MPGPU_WINOGRAD) && param == 0)
    return gfail(g, MPGPU_ERR_DIMENSION, "n_min must be at least 1");
  if (algo < MPGPU_SIMPLE || algo > MPGPU_WINOGRAD) return gfail(g, MPGPU_ERR_DOMAIN, "unknown algorithm");
  if (param == MPGPU_AUTO_NMIN) {  // the cutoff chosen from the measured leaf throughput
    if (algo == MPGPU_SIMPLE)
      param = 0;
    else if (algo == MPGPU_BLOCK || mpgpu_choose_nmin(algo, prec, m, l, n, &param, nullptr, nullptr))
      return gfail(g, MPGPU_ERR_DOMAIN, "MPGPU_AUTO_NMIN applies to strassen / winograd only");
  }
  if (param < 0) return gfail(g, MPGPU_ERR_DOMAIN, "negative n_min");
  const int L = mpgpu_nlimbs_for(prec);
  if (!L || prec > MPGPU_MAX_PREC) return gfail(g, MPGPU_ERR_DOMAIN, "precision %d outside the device range", prec);
  if (Lh < (prec + 31) / 32) return gfail(g, MPGPU_ERR_DOMAIN, "host limb count too small for precision");
  if (stats) {
    std::memset(stats, 0, sizeof *stats);
    uint64_t c[2];
    mpgpu_count_fast(algo, m, l, n, std::max<int64_t>(1, param), c);
    stats->mul = c[0];
    stats->addsub = c[1];
  }
  const HostSoa A{al, ae, as}, B{bl, be, bs};
  const HostSoaOut Cout{cl, ce, cs};

  int64_t plan[5] = {0, 1, m, l, n};
  const bool fast = algo == MPGPU_STRASSEN || algo == MPGPU_WINOGRAD;
  if (fast && mpgpu_fast_plan(m, l, n, param, plan)) return gfail(g, MPGPU_ERR_DIMENSION, "bad fast_mul plan");
  const int depth = (int)plan[0];
  if (world == 1 || (fast && depth == 0)) {  // nothing to split: one device does it all
    mpgpu_handle* h = g->h[0];
    const int rc = mpgpu_gemm_host(h, algo, param, prec, m, l, n, al, ae, as, bl, be, bs, cl, ce, cs, Lh, stats);
    if (rc) return gfail(g, rc, "%s", mpgpu_last_error(h));
    return MPGPU_OK;
  }

  std::vector<int> rcs(world, MPGPU_OK);
  std::vector<std::string> errs(world);
  std::vector<mpgpu_stats> st(world);
  Barrier bar(world);
  std::mutex emu;
  bool failed = false;  // any device failed: the others skip their remaining work
  auto set_fail = [&](int i, int rc, const char* where) {
    std::lock_guard<std::mutex> l2(emu);
    rcs[i] = rc;
    errs[i] = std::string(where) + ": " + mpgpu_last_error(g->h[i]);
    failed = true;
  };
  auto any_failed = [&] {
    std::lock_guard<std::mutex> l2(emu);
    return failed;
  };

  if (!fast) {
    // ---- Simple / Block: row shards, no exchange ----
    const std::vector<Range> rows = even_ranges(m, world);
    auto work = [&](int i) {
      mpgpu_handle* h = g->h[i];
      const Range r = rows[i];
      if (r.hi <= r.lo) return;
      const int64_t mr = r.hi - r.lo;
      mpgpu_mat da{}, db{}, dc{};
      int rc = mpgpu_alloc_matrix(h, mr, l, prec, &da);
      if (!rc) rc = mpgpu_alloc_matrix(h, l, n, prec, &db);
      if (!rc) rc = mpgpu_alloc_matrix(h, mr, n, prec, &dc);
      if (!rc) rc = mpgpu_upload_strided(h, &da, A.l + r.lo * l, A.e + r.lo * l, A.s + r.lo * l, Lh, m * l);
      if (!rc) rc = mpgpu_upload(h, &db, B.l, B.e, B.s, Lh);
      if (!rc) rc = mpgpu_gemm(h, algo, param, &da, &db, &dc, stats ? &st[i] : nullptr);
      if (!rc) rc = mpgpu_download_strided(h, &dc, Cout.l + r.lo * n, Cout.e + r.lo * n, Cout.s + r.lo * n, Lh, m * n);
      mpgpu_free_matrix(h, &da);
      mpgpu_free_matrix(h, &db);
      mpgpu_free_matrix(h, &dc);
      if (rc) set_fail(i, rc, "row shard");
    };
    std::vector<std::thread> th;
    for (int i = 0; i < world; ++i) th.emplace_back(work, i);
    for (auto& t : th) t.join();
  } else {
    // ---- Strassen / Winograd: leaf shards, peer pulls of row slices, row-owned combine ----
    const int up = choose_split(depth, world);
    int64_t units = 1;
    for (int i = 0; i < depth - up; ++i) units *= 7;
    int64_t per = 1, rows_per = 1;
    const std::vector<Range> ur = even_ranges(units, world, &per);
    int64_t um = m, un = n;  // dims of a unit (level depth - up) node product
    for (int i = 0; i < depth - up; ++i) {
      um = (um + um % 2) / 2;
      un = (un + un % 2) / 2;
    }
    const std::vector<Range> rr = even_ranges(um, world, &rows_per);
    const int64_t rw = mpgpu_record_words(L);
    const int64_t row_w = un * rw, unit_w = um * row_w;  // 32-bit words
    std::vector<uint32_t*> local(world, nullptr), fullv(world, nullptr);
    // fused exchange (default, <= 1024 bits): every device's leaf / last local post-addition
    // epilogue stores each unit-product row straight into its owner's buffer over NVLink; the
    // pull variant (MPGPU_GROUP_PULL=1) copies row slices afterwards with cudaMemcpy2DAsync
    static const bool pull_env = [] {
      const char* e = std::getenv("MPGPU_GROUP_PULL");
      return e && e[0] == '1';
    }();
    const bool fused = !pull_env && L <= 32;
    auto work = [&](int i) {
      mpgpu_handle* h = g->h[i];
      cudaSetDevice(g->devices[i]);
      cudaStream_t s = static_cast<cudaStream_t>(mpgpu_get_stream(h));
      mpgpu_mat da{}, db{}, dc{};
      uint32_t* full = nullptr;
      uint64_t* rowtab = nullptr;
      mpgpu_stats s_leaf{}, s_comb{};
      const Range u = ur[i];
      const Range r = rr[i];
      const int64_t hr = r.hi - r.lo;
      int rc = mpgpu_alloc_matrix(h, m, l, prec, &da);
      if (!rc) rc = mpgpu_alloc_matrix(h, l, n, prec, &db);
      if (!rc) rc = mpgpu_upload(h, &da, A.l, A.e, A.s, Lh);
      if (!rc) rc = mpgpu_upload(h, &db, B.l, B.e, B.s, Lh);
      if (fused) {
        // the owner's buffer first: every producer needs every owner's address
        cudaSetDevice(g->devices[i]);
        if (!rc && hr > 0 && cudaMalloc(&fullv[i], sizeof(uint32_t) * (size_t)(units * unit_w)) != cudaSuccess) {
          cudaGetLastError();
          rc = MPGPU_ERR_NOMEM;
        }
        if (rc) set_fail(i, rc, "unit buffer");
        bar.wait();  // all owners' buffers exist
        full = fullv[i];
        if (!any_failed() && u.hi > u.lo) {
          // row r of this device's node t lands in owner(r)'s buffer at unit u.lo + t
          std::vector<uint64_t> tab(um);
          for (int j = 0; j < world; ++j)
            for (int64_t rr_ = rr[j].lo; rr_ < rr[j].hi; ++rr_)
              tab[rr_] = reinterpret_cast<uint64_t>(fullv[j] + (u.lo * um + rr_) * row_w);
          cudaSetDevice(g->devices[i]);
          if (cudaMalloc(&rowtab, sizeof(uint64_t) * um) != cudaSuccess ||
              cudaMemcpy(rowtab, tab.data(), sizeof(uint64_t) * um, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            rc = MPGPU_ERR_CUDA;
          }
          if (!rc)
            rc = mpgpu_fast_leaves_rows(h, algo, param, &da, &db, up, u.lo, u.hi, rowtab, stats ? &s_leaf : nullptr);
          if (rowtab) cudaFree(rowtab);
          if (rc) set_fail(i, rc, "leaf shard (fused exchange)");
        }
        mpgpu_free_matrix(h, &da);
        mpgpu_free_matrix(h, &db);
        bar.wait();  // every product row is in its owner's buffer (the producers synchronised)
      } else {
        if (!rc && u.hi > u.lo) {
          cudaSetDevice(g->devices[i]);
          if (cudaMalloc(&local[i], sizeof(uint32_t) * (size_t)((u.hi - u.lo) * unit_w)) != cudaSuccess) {
            cudaGetLastError();
            rc = MPGPU_ERR_NOMEM;
          }
          if (!rc)
            rc = mpgpu_fast_leaves(h, algo, param, &da, &db, up, u.lo, u.hi, local[i], stats ? &s_leaf : nullptr);
        }
        mpgpu_free_matrix(h, &da);
        mpgpu_free_matrix(h, &db);
        if (rc) set_fail(i, rc, "leaf shard");
        bar.wait();  // every device's unit products are complete (mpgpu_fast_leaves is synchronous)
        if (!any_failed() && hr > 0) {
          cudaSetDevice(g->devices[i]);
          if (cudaMalloc(&full, sizeof(uint32_t) * (size_t)(units * unit_w)) != cudaSuccess) {
            cudaGetLastError();
            set_fail(i, MPGPU_ERR_NOMEM, "unit buffer");
          } else {
            // pull rows [r.lo, r.hi) of every unit product from the device that made it
            for (int j = 0; j < world && !rc; ++j) {
              const Range uj = ur[j];
              if (uj.hi <= uj.lo) continue;
              const cudaError_t e = cudaMemcpy2DAsync(
                  full + (uj.lo * um + r.lo) * row_w, sizeof(uint32_t) * unit_w, local[j] + r.lo * row_w,
                  sizeof(uint32_t) * unit_w, sizeof(uint32_t) * hr * row_w, uj.hi - uj.lo, cudaMemcpyDefault, s);
              if (e != cudaSuccess) {
                cudaGetLastError();
                rc = MPGPU_ERR_CUDA;
              }
            }
            if (!rc && cudaStreamSynchronize(s) != cudaSuccess) rc = MPGPU_ERR_CUDA;
            if (rc) set_fail(i, rc, "peer pull");
          }
        }
        bar.wait();  // every pull is complete: the producers' buffers may go
        if (local[i]) {
          cudaSetDevice(g->devices[i]);
          cudaFree(local[i]);
          local[i] = nullptr;
        }
      }
      if (!any_failed() && hr > 0) {
        rc = mpgpu_alloc_matrix(h, m, n, prec, &dc);
        if (!rc)
          rc = mpgpu_fast_combine_rows(h, algo, param, l, up, full, r.lo, r.hi, &dc, stats ? &s_comb : nullptr);
        // the rows of C this device owns, straight into the caller's buffer
        int64_t cnt = 0;
        if (!rc) rc = mpgpu_fast_owned_rows(m, l, n, param, up, r.lo, r.hi, nullptr, 0, &cnt);
        std::vector<int64_t> own(cnt);
        if (!rc && cnt) rc = mpgpu_fast_owned_rows(m, l, n, param, up, r.lo, r.hi, own.data(), cnt, &cnt);
        for (const Range& run : runs_of(own)) {
          if (rc) break;
          mpgpu_mat v{};
          rc = mpgpu_matrix_view(&dc, run.lo, 0, run.hi - run.lo, n, &v);
          if (!rc)
            rc = mpgpu_download_strided(h, &v, Cout.l + run.lo * n, Cout.e + run.lo * n, Cout.s + run.lo * n, Lh,
                                        m * n);
        }
        mpgpu_free_matrix(h, &dc);
        if (rc) set_fail(i, rc, "row-owned combine");
      }
      if (full) {
        cudaSetDevice(g->devices[i]);
        cudaFree(full);
      }
      if (stats) {
        st[i] = s_leaf;
        st[i].device_ms = s_leaf.device_ms + s_comb.device_ms;
        st[i].postadd_ms = s_leaf.postadd_ms + s_comb.postadd_ms;
        st[i].launches = s_leaf.launches + s_comb.launches;
        st[i].depth = depth;
      }
    };
    std::vector<std::thread> th;
    for (int i = 0; i < world; ++i) th.emplace_back(work, i);
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < world; ++i)
    if (rcs[i]) return gfail(g, rcs[i], "device %d (%d): %s", i, g->devices[i], errs[i].c_str());
  if (stats)
    for (int i = 0; i < world; ++i) merge_stats(stats, st[i]);
  return MPGPU_OK;
}

int mpgpu_gemm_host_mask(uint32_t gpu_mask, int algo, int64_t param, int32_t prec, int64_t m, int64_t l, int64_t n,
                         const uint32_t* al, const int32_t* ae, const uint8_t* as, const uint32_t* bl,
                         const int32_t* be, const uint8_t* bs, uint32_t* cl, int32_t* ce, uint8_t* cs, int32_t Lh,
                         mpgpu_stats* stats, char* err, size_t err_len) {
  // one cached group per mask for the life of the process (the C++ drop-in's entry)
  static std::mutex mu;
  static std::vector<std::pair<uint32_t, mpgpu_group*>> cache;
  mpgpu_group* g = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
      if (e.first == gpu_mask) g = e.second;
    if (!g) {
      const int rc = mpgpu_group_init(gpu_mask, &g);
      if (rc) {
        if (err && err_len) snprintf(err, err_len, "mpgpu_group_init(mask=0x%x) failed", gpu_mask);
        return rc;
      }
      cache.emplace_back(gpu_mask, g);
    }
  }
  const int rc =
      mpgpu_group_gemm_host(g, algo, param, prec, m, l, n, al, ae, as, bl, be, bs, cl, ce, cs, Lh, stats);
  if (rc && err && err_len) snprintf(err, err_len, "%s", mpgpu_group_last_error(g));
  return rc;
}

}  // extern "C"
