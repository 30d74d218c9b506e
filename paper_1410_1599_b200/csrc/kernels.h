// kernels.h -- host-side launch interface of the sm_100a kernels (internal to libmpgpu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include <mutex>
#include <set>
#include <utility>

namespace mpg {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// belongs to the device's context, so a process driving several GPUs (mpgpu_group_*, or one
// handle per device) must set it on each of them.  Thread-safe.
inline void smem_attr_once(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert({kern, dev}).second) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Batched MP GEMM over AoS record arrays (rec_stride(L) words per element).
// C[z] = A[z] * B[z] for z < batch, with the reference's inner-product order
// (matrix.hpp:147-155) and, when kb < l, the Block k-tile order
// (matrix.hpp:196-216): a fresh accumulator per k-tile, then C = RN(C + P).
struct GemmArgs {
  const uint32_t* A;
  const uint32_t* B;
  uint32_t* C;
  int64_t strideA, strideB, strideC;  // elements between batch items
  int64_t lda, ldb, ldc;              // elements between rows
  int m, l, n;
  int kb;  // k-tile of the Block order (>= l: Simple)
  int batch;
  int sh;  // 32 L - p
  uint32_t* err;
  // optional LU Schur epilogue: C = RN(C - A*B) in place (blocklu.hpp:138-141)
  int sub_from_c;
  // optional row destinations (multi-GPU exchange fused into the epilogue): row i of batch
  // item z goes to rowtab[i] + (batch0 + z) * strideC records -- rowtab[i] may point into
  // another GPU's memory (peer access), so the products land at their owners as they are made
  const uint64_t* rowtab;
  int64_t batch0;
};

template <int L>
void launch_gemm(const GemmArgs& g, cudaStream_t st);
// tensor-core (tcgen05 kind::i8) variant of the same contract, L in {8, 16, 32};
// returns false if it could not be configured (launch_gemm then uses the IMAD kernel)
template <int L>
bool launch_gemm_tc(const GemmArgs& g, cudaStream_t st);
// MPGPU_GEMM=tc selects the tensor-core leaf (read once per process)
bool gemm_tc_enabled();

// SoA planes <-> records
template <int L>
void launch_soa2rec(const uint32_t* limbs, const int32_t* exp, const uint8_t* sign, int64_t N,
                    int64_t plane_stride, uint32_t* rec, cudaStream_t st);
template <int L>
void launch_rec2soa(const uint32_t* rec, int64_t N, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                    int64_t plane_stride, cudaStream_t st);
// a dense rows x cols block of SoA planes into a strided record matrix (leading dim ldr)
template <int L>
void launch_soa2rec_2d(const uint32_t* limbs, const int32_t* exp, const uint8_t* sign, int64_t rows, int64_t cols,
                       int64_t plane_stride, uint32_t* rec, int64_t ldr, cudaStream_t st);

// elementwise C = A +- B (matrix.hpp:121-134), contiguous records
template <int L>
void launch_addsub(const uint32_t* A, const uint32_t* B, uint32_t* C, int64_t N, int is_sub, int sh,
                   uint32_t* err, cudaStream_t st);

// output slot per Strassen / Winograd child of a pre-addition (< 0: child not produced)
struct ChildSlots {
  int8_t s[7];
};

// Fast-algorithm level transforms (fastmm.hpp:133-219), batched over the nodes of
// one recursion level.  Parents: nodes x (rows x cols) records (row-major, dense),
// virtually zero-padded to (prows x pcols) = (rows + rows%2, cols + cols%2).
// Children: 7 per parent, each (prows/2 x pcols/2), child c = parent * 7 + q.
// side: 0 = A operand, 1 = B operand.  algo: 2 = Strassen, 3 = Winograd.
template <int L>
void launch_preadd(int algo, int side, const uint32_t* parent, int64_t nodes, int rows, int cols,
                   uint32_t* children, int sh, uint32_t* err, cudaStream_t st);
// one node's pre-additions with the children placed by `slots` (L <= 32)
template <int L>
void launch_preadd_slots(int algo, int side, const uint32_t* parent, int rows, int cols, uint32_t* children,
                         ChildSlots slots, int sh, cudaStream_t st);
// two levels of pre-additions in one launch (L <= 32): grand = the 49 grandchildren per node in the
// layout two launch_preadd calls produce, the intermediate level kept in shared memory; returns
// false when this limb count has no fused kernel
template <int L>
bool launch_preadd2(int algo, int side, const uint32_t* parent, int64_t nodes, int rows, int cols,
                    uint32_t* grand, int sh, cudaStream_t st);
// two levels of post-additions in one launch (L <= 32): the node's C from its 49 grandchildren
// products (the layout two recursion levels produce); false when there is no fused kernel
constexpr bool has_postadd2(int L) { return L >= 4 && L <= 16; }
template <int L>
bool launch_postadd2(int algo, const uint32_t* grand, int64_t nodes, int rows, int cols, uint32_t* parent,
                     int sh, uint32_t* err, cudaStream_t st);
// Children products (7 per parent, hm x hn) -> parent C (rows x cols, stripped).
// Optional trace output of Winograd's T1/T2 (2 x hm x hn per parent) when t_out != nullptr.
// rowlist (device, optional): only these child rows [0, hm) are combined (and the parent rows
// they produce written) -- the row-owned combine of the multi-GPU path.  [cc0, cc0 + ncc): only
// these child columns (ncc < 0: to the end), i.e. parent columns c and c + hc for each -- the
// column split of the LU look-ahead (L <= 32).
// rowtab (device, optional): parent row r of node t goes to rowtab[r] + t * rows * cols records
// (the fused multi-GPU exchange, as GemmArgs::rowtab; L <= 32).
template <int L>
void launch_postadd(int algo, const uint32_t* children, int64_t nodes, int rows, int cols,
                    uint32_t* parent, uint32_t* t_out, int sh, uint32_t* err, cudaStream_t st,
                    const int* rowlist = nullptr, int nrows = 0, int cc0 = 0, int ncc = -1,
                    const uint64_t* rowtab = nullptr);

// copy a (rows x cols) window with leading dims (records) -- used by LU
template <int L>
void launch_copy2d(const uint32_t* src, int64_t lds, uint32_t* dst, int64_t ldd, int rows, int cols,
                   cudaStream_t st);

// scalar ops on record arrays (primitive tests): op 0 add, 1 sub, 2 mul, 3 div
template <int L>
void launch_vec_op(int op, const uint32_t* A, const uint32_t* B, uint32_t* C, int64_t N, int sh,
                   uint32_t* err, cudaStream_t st);

// ---- LU (blocklu.hpp:42-146) --------------------------------------------
// Pivot-search candidates: one (compact magnitude key, first row, multiplicity) per
// lu_col CTA for the next column (cap entries each).
struct PivotCands {
  uint64_t* key = nullptr;
  int64_t* idx = nullptr;
  int* cnt = nullptr;
  int64_t cap = 0;
};
// One right-looking elimination step d of the panel [p, row_end) x [p, p+k) of the
// n x n record matrix a (row-major, ld = n):
//   multipliers a_id = RN(a_id / a_dd) for i in (d, row_end), and
//   a_ij = RN(a_ij - RN(a_id * a_dj)) for i in (d, row_end), j in (d, p+k).
// With cand.key set, also writes the pivot candidates of column d+1; returns their
// count (0: none written).
template <int L>
int64_t launch_lu_step(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t col_end, int sh, uint32_t* err,
                       const PivotCands& cand, cudaStream_t st);
// pivot search for column d over rows [d, row_end): first max |a_id| -> piv_dev[d],
// from ncand candidates of the previous step (ncand > 0) or a column scan; then swap
// rows d and piv over the columns [c0, c1).
template <int L>
void launch_pivot(uint32_t* a, int64_t n, int64_t d, int64_t row_end, int64_t* piv_dev, int64_t* zp,
                  const PivotCands& cand, int64_t ncand, int64_t c0, int64_t c1, cudaStream_t st);
// apply the panel's interchanges piv[p .. p+k) to all columns outside [p, p+k)
template <int L>
void launch_laswp(uint32_t* a, int64_t n, int64_t p, int64_t k, const int64_t* piv_dev, const int64_t* zp,
                  cudaStream_t st);
// forward substitution step s of trsm_unit_lower (blocklu.hpp:60-69) on the
// block rows (s, p_end) x cols [c0, c0+w): a_ij = RN(a_ij - RN(a_is * a_sj)).
template <int L>
void launch_trsm_l_step(uint32_t* a, int64_t n, int64_t s, int64_t p_end, int64_t c0, int64_t w,
                        int sh, uint32_t* err, cudaStream_t st);

// whole-panel factorisation (all pivot columns of [p, p+k), rows [p, row_end)) in one
// cooperative launch; returns -1 if it cannot run (caller uses the per-column path).
// cand_key / cand_idx: scratch of at least max_grid entries.
template <int L>
int launch_lu_panel_coop(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t row_end, int pivoting,
                         int64_t* piv, int64_t* zp, int sh, uint64_t* cand_key, int64_t* cand_idx, int max_grid,
                         cudaStream_t st);

// whole-panel trsm_unit_lower: rows [p, p+k) x cols [c0, c0+w), one launch
template <int L>
void launch_trsm_l_panel(uint32_t* a, int64_t n, int64_t p, int64_t k, int64_t c0, int64_t w, int sh,
                         cudaStream_t st);

// Ly = Pb, Ux = y on packed factors (blocklu.hpp:215-245) for nrhs right-hand sides
// (one CTA each; b, x: nrhs x n records); scratch: 2n records per right-hand side
template <int L>
void launch_lu_solve(const uint32_t* f, int64_t n, const int64_t* piv_dev, const uint32_t* b,
                     uint32_t* x, uint32_t* scratch, int sh, uint32_t* err, int64_t* zp,
                     int exact, int64_t nrhs, cudaStream_t st);

// C(view, ldc) = RN(C - T) for a rows x cols T with leading dimension ldt (< 0: dense) --
// the LU Schur subtraction
template <int L>
void launch_sub2d(uint32_t* C, int64_t ldc, const uint32_t* T, int rows, int cols, int sh,
                  uint32_t* err, cudaStream_t st, int64_t ldt = -1);

// ---- accuracy metrics (metrics.cu), L in {1..32, 64} -----------------------
// mode 0: outA[t] = rel_error(approx, ref) = RN(|RN(approx - ref)| / |ref|) at the
//         reference precision (precision.hpp:187-193), SKIP-flagged and counted where
//         ref == 0 (matrix.hpp:253-279); approx has la <= L limbs, widened exactly.
// mode 1: solution error (blocklu.hpp:312-333): as mode 0 for nonzero refs; zero refs
//         give outB[t] = RN(|approx - ref|) and are counted.
template <int L>
void launch_rel_error(const uint32_t* approx, int la, int64_t lda, const uint32_t* ref, int64_t ldr, int rows,
                      int cols, int mode, int sh, uint32_t* outA, uint32_t* outB, unsigned long long* counter,
                      uint32_t* err, cudaStream_t st);
// one_norm column sums (matrix.hpp:237-251): out[j] = RN sum of |a_ij|, i ascending
template <int L>
void launch_colsum_abs(const uint32_t* A, int64_t ld, int rows, int cols, int sh, uint32_t* out, uint32_t* err,
                       cudaStream_t st);
// (max A, min A, max B) over N flagged nonnegative records -> 3 records (flag bit 1 of the
// sign word set when a set was empty); scratch: 3 * 1024 records
template <int L>
void launch_reduce3(const uint32_t* A, const uint32_t* B, int64_t N, uint32_t* out3, uint32_t* scratch,
                    cudaStream_t st);

// RN conversion between precisions (mpfr_set, blocklu.hpp:266-270): records of ls limbs
// (stride rec_stride(ls)) -> records of L limbs rounded to 32L - sh bits
template <int L>
void launch_convert(const uint32_t* src, int ls, int64_t N, uint32_t* dst, int sh, uint32_t* err, cudaStream_t st);

}  // namespace mpg
