/* mpgpu.h -- C-ABI of the B200-native multiple-precision GEMM / LU library
 * (libmpgpu.so, built from paper_1410_1599_b200/csrc).
 *
 * This is the drop-in boundary for the reference's MP matmul / LU hot path
 * (/root/reference/proj/include/mpmm).  Every entry point below names the
 * reference interface it replaces; the C++ shim in include/mpmm_gpu.hpp binds the
 * reference's own signatures to it.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Host buffers are caller-owned; device
 *     matrices are owned by the handle that allocated them.
 *   - Host MP arrays are structure-of-arrays ("SoA"): for N = rows*cols elements
 *     in row-major order and a host limb count Lh >= ceil(prec/32):
 *        limbs[k*N + e]  32-bit limb k of element e, k = Lh-1 most significant;
 *                        the MSB of limb Lh-1 is set for nonzero values and bits
 *                        below prec are zero (MPFR's mantissa, regrouped in 32-bit
 *                        limbs);
 *        exp[e]          MPFR exponent (value = (-1)^sign * 0.m * 2^exp with
 *                        0.m in [1/2, 1)), or MPGPU_EXP_ZERO for a zero;
 *        sign[e]         1 for negative (zeros keep their sign, as in MPFR).
 *     NaN / Inf are not representable: callers reject them (DomainError).
 *   - Rounding is MPFR_RNDN (precision.hpp:22) after every multiply and every
 *     add, exactly as the reference; results are bit-identical to the reference
 *     wherever the reference's operation order is replayed (all of them: Simple,
 *     Block, Strassen, Winograd, pivot-free blocked LU).
 *   - Return codes map 1:1 onto the reference's exception types (errors.hpp:10-48).
 *   - Calls on one handle are serialised (internal mutex) and synchronous.
 */
#ifndef MPGPU_H
#define MPGPU_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPGPU_OK 0
#define MPGPU_ERR_DIMENSION 1 /* mpmm::DimensionError  (errors.hpp:15-17) */
#define MPGPU_ERR_DOMAIN 2    /* mpmm::DomainError     (errors.hpp:21-23) */
#define MPGPU_ERR_SINGULAR 3  /* mpmm::SingularError   (errors.hpp:26-31), pivot index out-param */
#define MPGPU_ERR_CUDA 4      /* device / runtime failure (no reference analogue) */
#define MPGPU_ERR_NOMEM 5     /* device allocation failed */
#define MPGPU_ERR_UNDEFINED_METRIC 6 /* mpmm::UndefinedMetricError (errors.hpp:41-43) */

#define MPGPU_EXP_ZERO INT32_MIN
/* Largest device precision: limb counts 1, 2, 4, 8, 16, 32 (one thread per value,
 * register-resident, <= 1024 bits) and 64, 128, 256, 288 (wide formats, one warp per value,
 * <= 9216 bits -- e.g. the 8192 / 8650-bit Lotkin experiments of the paper). */
#define MPGPU_MAX_PREC 9216
#define MPGPU_MAX_STORE_PREC MPGPU_MAX_PREC

/* n_min / param value selecting the Strassen / Winograd cutoff automatically (mpgpu_choose_nmin):
 * the recursion depth that minimises the modelled device time given the measured leaf-GEMM
 * throughput of the precision (documented extension; an explicit n_min replays the reference
 * bit for bit, as always). */
#define MPGPU_AUTO_NMIN (-1)

/* mpmm::Algorithm (fastmm.hpp:13) */
enum { MPGPU_SIMPLE = 0, MPGPU_BLOCK = 1, MPGPU_STRASSEN = 2, MPGPU_WINOGRAD = 3 };

typedef struct mpgpu_handle mpgpu_handle;

/* Device matrix: row-major AoS records of mpgpu_record_words(nlimbs) 32-bit words
 * (limbs[0..nlimbs-1], exp, sign, padding) -- opaque to callers except for the
 * pointer, which may be handed to NCCL / torch for raw transfers. */
typedef struct {
  int64_t rows, cols;
  int32_t prec;   /* bits (mpmm::PrecisionContext, precision.hpp:18-36) */
  int32_t nlimbs; /* device limbs per element */
  uint32_t* rec;  /* device pointer */
  int64_t ld;     /* elements between consecutive rows */
  int32_t owned;  /* 1 if allocated by mpgpu_alloc_matrix */
} mpgpu_mat;

/* Per-call statistics.  mul / addsub are the reference's OpCounter tallies
 * (opcounter.hpp:9-20) for the same call, equal to count_fast / count_simple. */
typedef struct {
  uint64_t mul, addsub;
  uint64_t leaf_madds; /* MP multiply-adds executed by the leaf GEMM kernel(s) */
  double device_ms;    /* CUDA-event time of the device work of the call */
  double leaf_ms;      /* CUDA-event time of the leaf GEMM launch(es) */
  double preadd_ms, postadd_ms;
  int32_t launches; /* kernels launched by the call */
  int32_t depth;    /* Strassen / Winograd recursion depth used */
} mpgpu_stats;

/* ---- handle ------------------------------------------------------------ */
int mpgpu_init(int device, mpgpu_handle** out);
void mpgpu_destroy(mpgpu_handle* h);
const char* mpgpu_last_error(const mpgpu_handle* h);
/* run subsequent work on an external cudaStream_t (NULL: the handle's own stream) */
int mpgpu_set_stream(mpgpu_handle* h, void* cuda_stream);
void* mpgpu_get_stream(mpgpu_handle* h);
int mpgpu_synchronize(mpgpu_handle* h);
/* device-to-device copy on the handle's stream (raw record buffers) */
int mpgpu_copy_device(mpgpu_handle* h, void* dst, const void* src, size_t bytes);

/* device limb count used for a precision (0 if prec is outside [2, MPGPU_MAX_STORE_PREC]) */
int mpgpu_nlimbs_for(int32_t prec);
int mpgpu_record_words(int32_t nlimbs);

/* ---- matrices (mpmm::Matrix, matrix.hpp:20-42) --------------------------- */
int mpgpu_alloc_matrix(mpgpu_handle* h, int64_t rows, int64_t cols, int32_t prec, mpgpu_mat* out);
int mpgpu_free_matrix(mpgpu_handle* h, mpgpu_mat* m);
/* host SoA (host_nlimbs limbs per element) <-> device records */
int mpgpu_upload(mpgpu_handle* h, mpgpu_mat* m, const uint32_t* limbs, const int32_t* exp,
                 const uint8_t* sign, int32_t host_nlimbs);
int mpgpu_download(mpgpu_handle* h, const mpgpu_mat* m, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                   int32_t host_nlimbs);

/* ---- GEMM --------------------------------------------------------------
 * C = A * B at C->prec, replacing
 *   algo SIMPLE   : simple_mul(A, B, ctx[, ops])            matrix.hpp:178-184
 *   algo BLOCK    : block_mul(A, B, param=n_min, ctx[, ops]) matrix.hpp:225-233
 *   algo STRASSEN / WINOGRAD :
 *                   fast_mul(A, B, {algo, param=n_min}, ctx) fastmm.hpp:244-255
 * Checks in the reference's order: inner dimension (DIMENSION), param == 0 for
 * BLOCK / fast (DIMENSION), unknown algo (DOMAIN); A, B and C must share one
 * precision on the device path (DOMAIN otherwise -- documented deviation).
 * stats may be NULL. */
int mpgpu_gemm(mpgpu_handle* h, int algo, int64_t param, const mpgpu_mat* A, const mpgpu_mat* B,
               mpgpu_mat* C, mpgpu_stats* stats);

/* Same, from and to HOST SoA buffers (the reference-facing call: upload, multiply,
 * download).  C buffers must hold m*n elements of host_nlimbs limbs. */
int mpgpu_gemm_host(mpgpu_handle* h, int algo, int64_t param, int32_t prec, int64_t m, int64_t l,
                    int64_t n, const uint32_t* a_limbs, const int32_t* a_exp, const uint8_t* a_sign,
                    const uint32_t* b_limbs, const int32_t* b_exp, const uint8_t* b_sign,
                    uint32_t* c_limbs, int32_t* c_exp, uint8_t* c_sign, int32_t host_nlimbs,
                    mpgpu_stats* stats);

/* fast_mul with the reference's TopTrace (fastmm.hpp:47-51): writes the top-level
 * intermediates as device matrices packed back to back into trace_rec (sums
 * S1..S8 for Winograd -- 4 of hm x hl then 4 of hl x hn --, products P1..P7 / M1..M7
 * (hm x hn), and T1, T2 (hm x hn) for Winograd); counts[3] = {sums, products, t}. */
int mpgpu_fast_mul_trace(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A,
                         const mpgpu_mat* B, mpgpu_mat* C, uint32_t* trace_rec, int* counts);

/* elementwise add / sub (matrix.hpp:166-175): C = A +- B */
int mpgpu_addsub(mpgpu_handle* h, int is_sub, const mpgpu_mat* A, const mpgpu_mat* B, mpgpu_mat* C);
/* elementwise scalar op over equal-shaped matrices: 0 add, 1 sub, 2 mul, 3 div
 * (precision.hpp:127-161); division by zero -> SINGULAR */
int mpgpu_vec_op(mpgpu_handle* h, int op, const mpgpu_mat* A, const mpgpu_mat* B, mpgpu_mat* C);

/* ---- LU ----------------------------------------------------------------
 * In-place blocked LU of the square matrix A (packed unit-lower L \ U, Doolittle),
 * replacing lu_blocked(A, {K, kernel, n_min}, ctx, schur_ops) (blocklu.hpp:121-146).
 * pivoting = 0: the reference's pivot-free algorithm, bit-exact.  pivoting = 1:
 * partial pivoting over the tall panel (first maximal |a_id|, LAPACK ipiv in
 * piv_out[n], 0-based) -- an extension the reference lacks.  On a zero pivot
 * returns SINGULAR with *zero_pivot = 1-based index (blocklu.hpp:46-47).
 * stats->mul/addsub accumulate the Schur multiply counts (schur_ops). */
int mpgpu_lu_blocked(mpgpu_handle* h, mpgpu_mat* A, int64_t K, int kernel, int64_t n_min,
                     int pivoting, int64_t* piv_out, int64_t* zero_pivot, mpgpu_stats* stats);
/* The same on an n x n matrix in HOST SoA buffers, factored in place (the drop-in's
 * lu_blocked, blocklu.hpp:121-146, with the transfers overlapped: the first K columns are
 * copied first, the rest while the first panel is factored, and each block of K rows is
 * copied back as soon as no later step touches it).  Factors bit-identical to
 * mpgpu_lu_blocked's; on an error the buffers' contents are unspecified.  Not to be run
 * concurrently with other calls on the same handle. */
int mpgpu_lu_blocked_host(mpgpu_handle* h, int32_t prec, int64_t n, uint32_t* limbs, int32_t* exp,
                          uint8_t* sign, int32_t host_nlimbs, int64_t K, int kernel, int64_t n_min,
                          int pivoting, int64_t* piv_out, int64_t* zero_pivot, mpgpu_stats* stats);
/* Ly = Pb, Ux = y (blocklu.hpp:215-245); piv may be NULL (pivot-free factors).
 * exact = 1 replays the reference's summation order (bit-exact; the back
 * substitution is an O(n^2) serial chain of rounded adds); exact = 0 runs the
 * back substitution column-oriented (n parallel steps; s-descending sums, within
 * the LU tolerance). */
int mpgpu_lu_solve(mpgpu_handle* h, const mpgpu_mat* F, const int64_t* piv, const mpgpu_mat* b,
                   mpgpu_mat* x, int exact, int64_t* zero_pivot);

/* lu_solve for r right-hand sides at once (rows of the r x n matrix Bt; solutions in the
 * rows of Xt), one CTA per right-hand side -- e.g. inverse() (blocklu.hpp:263-281) */
int mpgpu_lu_solve_many(mpgpu_handle* h, const mpgpu_mat* F, const int64_t* piv, const mpgpu_mat* Bt,
                        mpgpu_mat* Xt, int exact, int64_t* zero_pivot);
/* dst = RN(src) at dst->prec (mpfr_set between precisions, blocklu.hpp:266-270); same shape */
int mpgpu_convert(mpgpu_handle* h, const mpgpu_mat* src, mpgpu_mat* dst);

/* ---- accuracy metrics (device-side; bench.hpp:145-147, 217, 238) ---------
 * Results are returned as host SoA scalars at the reference's precision, limb planes
 * of nlimbs_out = ref->nlimbs limbs (limbs[k * count + e] is limb k of result e).
 *
 * max_rel_error (matrix.hpp:253-279): out {max, min} of rel_error(approx, ref) =
 * RN(|RN(approx - ref)| / |ref|) at ref->prec (precision.hpp:187-193) over the
 * elements with ref != 0; *skipped = count of zero references.  approx->prec <=
 * ref->prec (the approximation is widened exactly).  Shape mismatch -> DIMENSION;
 * all references zero -> UNDEFINED_METRIC. */
int mpgpu_max_rel_error(mpgpu_handle* h, const mpgpu_mat* approx, const mpgpu_mat* ref, uint32_t* out_limbs,
                        int32_t* out_exp, uint8_t* out_sign, int64_t* skipped);
/* max_rel_error_solution (blocklu.hpp:306-333) for n x 1 vectors at one precision:
 * out {max_rel over xtrue != 0, max |xhat - xtrue| over xtrue == 0 (+0 if none)};
 * *zero_refs = number of zero components.  Length mismatch -> DIMENSION; every
 * component zero -> UNDEFINED_METRIC. */
int mpgpu_solution_error(mpgpu_handle* h, const mpgpu_mat* xhat, const mpgpu_mat* xtrue, uint32_t* out_limbs,
                         int32_t* out_exp, uint8_t* out_sign, int64_t* zero_refs);
/* one_norm (matrix.hpp:237-251): max over columns of the top-to-bottom RN sum of |a_ij|
 * at A->prec; out: one scalar. */
int mpgpu_one_norm(mpgpu_handle* h, const mpgpu_mat* A, uint32_t* out_limbs, int32_t* out_exp,
                   uint8_t* out_sign);

/* ---- multi-GPU building blocks -------------------------------------------
 * A strided window of a device matrix (no copy; not owned). */
int mpgpu_matrix_view(const mpgpu_mat* parent, int64_t r0, int64_t c0, int64_t rows, int64_t cols,
                      mpgpu_mat* out);
/* Recursion facts of fast_mul: out5 = {depth d, leaves 7^d, leaf m, leaf l, leaf n}. */
int mpgpu_fast_plan(int64_t m, int64_t l, int64_t n, int64_t n_min, int64_t* out5);
/* Sharded Strassen / Winograd (fastmm.hpp:99-229 split at the bottom of the
 * recursion).  Nodes of level t are numbered breadth-first (child c of node p is
 * 7p + c; level d holds the 7^d leaves).  mpgpu_fast_leaves computes the products
 * of the level-(d - up_levels) nodes [node_lo, node_hi) -- their leaves' GEMMs plus
 * up_levels post-addition levels -- into the device buffer node_products (node-
 * major, node m x n records of mpgpu_record_words(nlimbs) words), running only the
 * pre-additions of their ancestors.  mpgpu_fast_combine then runs the remaining
 * post-addition levels from the products of ALL level-(d - up_levels) nodes (e.g.
 * after an NCCL all-gather) into C.  The pair is bit-identical to
 * mpgpu_gemm(STRASSEN / WINOGRAD). */
int mpgpu_fast_leaves(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                      int up_levels, int64_t node_lo, int64_t node_hi, uint32_t* node_products,
                      mpgpu_stats* stats);
/* The same, with the exchange fused into the producing kernel: row r of node u (u = 0 ..
 * node_hi - node_lo - 1) is written to row_dst[r] + u * (rows * cols) records, where row_dst
 * (a DEVICE array of node-row count 64-bit addresses) may point into other GPUs' memory (peer
 * access over NVLink): the leaf GEMM's (or last local post-addition's) epilogue stores every
 * product row straight into the buffer of the device that owns it.  Precisions <= 1024 bits. */
int mpgpu_fast_leaves_rows(mpgpu_handle* h, int algo, int64_t n_min, const mpgpu_mat* A, const mpgpu_mat* B,
                           int up_levels, int64_t node_lo, int64_t node_hi, const uint64_t* row_dst,
                           mpgpu_stats* stats);
int mpgpu_fast_combine(mpgpu_handle* h, int algo, int64_t n_min, int64_t l, int up_levels,
                       const uint32_t* node_products, mpgpu_mat* C, mpgpu_stats* stats);
/* Row-owned combine: node_products holds (at least) rows [row_lo, row_hi) of every
 * level-(d - up_levels) node product; only the rows of C (and of every intermediate
 * level) that derive from them are computed -- a level-t row r comes from child row r
 * or r - m_{t+1}, so ownership propagates through the pad/halve index map.  Ranks that
 * own disjoint unit-row ranges (exchanged with one all-to-all) together produce all of
 * C without replicated post-additions. */
int mpgpu_fast_combine_rows(mpgpu_handle* h, int algo, int64_t n_min, int64_t l, int up_levels,
                            const uint32_t* node_products, int64_t row_lo, int64_t row_hi, mpgpu_mat* C,
                            mpgpu_stats* stats);
/* Device buffers shared between processes (one process per GPU): plain cudaMalloc memory, its
 * CUDA IPC handle (MPGPU_IPC_HANDLE_BYTES opaque bytes, exchanged by the caller, e.g. with
 * torch.distributed), and a peer process's buffer mapped into this one (peer access enabled) --
 * the destinations of mpgpu_fast_leaves_rows across processes. */
#define MPGPU_IPC_HANDLE_BYTES 64
int mpgpu_malloc(mpgpu_handle* h, size_t bytes, void** out);
int mpgpu_free(mpgpu_handle* h, void* p);
int mpgpu_ipc_handle(mpgpu_handle* h, void* p, void* handle_out);
int mpgpu_ipc_open(mpgpu_handle* h, const void* handle, void** out);
int mpgpu_ipc_close(mpgpu_handle* h, void* p);
/* device-to-device 2D copy on the handle's stream (packing row slices for the all-to-all) */
int mpgpu_copy_device_2d(mpgpu_handle* h, void* dst, size_t dpitch, const void* src, size_t spitch,
                         size_t width, size_t height);

/* Rows of C produced by the row-owned combine of unit rows [row_lo, row_hi) (the rows
 * mpgpu_fast_combine_rows writes): *count rows, the first `cap` of them into out (sorted). */
int mpgpu_fast_owned_rows(int64_t m, int64_t l, int64_t n, int64_t n_min, int up_levels, int64_t row_lo,
                          int64_t row_hi, int64_t* out, int64_t cap, int64_t* count);
/* Upload / download between a dense device matrix (or a full-width row view) and host SoA
 * planes that belong to a LARGER host matrix: limb plane k of the host matrix starts
 * host_plane_stride elements after plane k-1 (pointers pre-offset to the first element),
 * e.g. rows r0.. of an m x n host matrix: limbs + r0*n, exp + r0*n, sign + r0*n, stride m*n. */
int mpgpu_upload_strided(mpgpu_handle* h, mpgpu_mat* m, const uint32_t* limbs, const int32_t* exp,
                         const uint8_t* sign, int32_t host_nlimbs, int64_t host_plane_stride);
int mpgpu_download_strided(mpgpu_handle* h, const mpgpu_mat* m, uint32_t* limbs, int32_t* exp, uint8_t* sign,
                           int32_t host_nlimbs, int64_t host_plane_stride);

/* ---- multi-GPU: one process driving several devices (SURVEY.md 8(b) gpu_mask, 8(e)) ----
 * A group holds one handle per device.  mpgpu_group_gemm_host is mpgpu_gemm_host over
 * all of them -- same arguments, same results bit for bit (simple_mul / block_mul
 * matrix.hpp:178-233: C split by row blocks, no exchange; fast_mul fastmm.hpp:244-255:
 * the 7^d leaf products split over the devices, each device doing its own pre-additions,
 * one exchange of unit-product row slices by peer copies over NVLink, row-owned
 * post-additions, each device writing its rows of C to the host).  A device may repeat in
 * mpgpu_group_init_devices (shards of one GPU: the same path on a one-GPU host). */
typedef struct mpgpu_group mpgpu_group;
int mpgpu_group_init(uint32_t gpu_mask, mpgpu_group** out); /* device d <-> bit d */
int mpgpu_group_init_devices(int ndev, const int* devices, mpgpu_group** out);
void mpgpu_group_destroy(mpgpu_group* g);
int mpgpu_group_size(const mpgpu_group* g);
int mpgpu_group_device(const mpgpu_group* g, int i);
mpgpu_handle* mpgpu_group_handle(mpgpu_group* g, int i);
const char* mpgpu_group_last_error(const mpgpu_group* g);
/* stats: mul / addsub of the whole product, leaf_madds summed over devices, times = the
 * slowest device's */
int mpgpu_group_gemm_host(mpgpu_group* g, int algo, int64_t param, int32_t prec, int64_t m, int64_t l,
                          int64_t n, const uint32_t* a_limbs, const int32_t* a_exp, const uint8_t* a_sign,
                          const uint32_t* b_limbs, const int32_t* b_exp, const uint8_t* b_sign,
                          uint32_t* c_limbs, int32_t* c_exp, uint8_t* c_sign, int32_t host_nlimbs,
                          mpgpu_stats* stats);
/* the same through a process-wide group cached per gpu_mask (the C++ drop-in's entry);
 * err (optional) receives the error text */
int mpgpu_gemm_host_mask(uint32_t gpu_mask, int algo, int64_t param, int32_t prec, int64_t m, int64_t l,
                         int64_t n, const uint32_t* a_limbs, const int32_t* a_exp, const uint8_t* a_sign,
                         const uint32_t* b_limbs, const int32_t* b_exp, const uint8_t* b_sign,
                         uint32_t* c_limbs, int32_t* c_exp, uint8_t* c_sign, int32_t host_nlimbs,
                         mpgpu_stats* stats, char* err, size_t err_len);

/* ---- host-side model / plan / inputs ------------------------------------ */
/* The cutoff MPGPU_AUTO_NMIN resolves to for an m x l x n product at prec bits (Strassen /
 * Winograd): per candidate depth d, modelled time = leaf multiply-adds / measured leaf rate at
 * that leaf size + pre/post-addition record bytes / measured bandwidth; the fastest depth wins.
 * n_min = the smallest cutoff giving that depth; depth / model_ms may be NULL. */
int mpgpu_choose_nmin(int algo, int32_t prec, int64_t m, int64_t l, int64_t n, int64_t* n_min, int32_t* depth,
                      double* model_ms);
/* count_fast (opmodel.hpp:30-44); SIMPLE / BLOCK give count_simple */
int mpgpu_count_fast(int algo, int64_t m, int64_t l, int64_t n, int64_t n_min, uint64_t* out2);
/* recursion_plan (fastmm.hpp:68-85): rows of 8 int64 {level, m,l,n, pm,pl,pn, base} */
int mpgpu_recursion_plan(int64_t m, int64_t l, int64_t n, int64_t n_min, int64_t* out, int max_levels,
                         int* count);
/* Seeded inputs into host SoA buffers (Prng64, matgen.hpp:13-42):
 *   kind 0: gen_random (matgen.hpp:45-52), 53-bit dyadic uniform [-1,1) rounded at prec
 *   kind 1: full-mantissa uniform [-1,1): (k - 2^p) / 2^p, k = top p+1 bits of the
 *           concatenated top53() draws (exact at prec)
 *   kind 2: mantissa uniform in [1/2,1) with all prec bits random, exponent uniform
 *           in [-20, 20], random sign (BASELINE config 3) */
int mpgpu_gen(int kind, int64_t N, uint64_t seed, int32_t prec, uint32_t* limbs, int32_t* exp,
              uint8_t* sign, int32_t host_nlimbs);

#ifdef __cplusplus
}
#endif
#endif
