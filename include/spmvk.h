/* include/spmvk.h — the drop-in C-ABI of the B200-native RgCSR / Hybrid SpMV.
 *
 * The reference (arxiv/paper_1012_2270, /root/reference/proj/core) exposes its
 * hot path as header-only C++ templates in namespace spmvkit; it has no FFI.
 * Every entry point below replaces one of those templates (file:line relative
 * to /root/reference/proj/) and keeps its argument meaning and its error
 * behaviour: where the reference throws std::invalid_argument this returns
 * SPMVK_EINVAL, where it throws std::runtime_error this returns SPMVK_ERANGE,
 * with the reference's message (or a more specific one) in spmvk_last_error().
 * include/spmvkit_gpu.hpp restores the reference's C++ names, signatures and
 * exceptions on top of this header.
 *
 * Conventions
 *  - return 0 on success; nonzero spmvk_status otherwise;
 *  - handles are opaque, own their device memory and are immutable after
 *    build, so concurrent SpMVs on different streams are safe;
 *  - x / y in the *_spmv_* calls are DEVICE pointers owned by the caller,
 *    with their element counts passed like the reference's std::span sizes;
 *    *_spmv_host_* take HOST pointers and do H2D / D2H inside (the span
 *    overloads' semantics, synchronous);
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *  - indices are uint32_t like spmvkit::index_t (spmvkit/triplet.hpp:12).
 *    Unlike the reference, a slot count that overflows 32 bits is REPORTED
 *    (SPMVK_ERANGE) instead of silently truncated (spmvkit/rgcsr.hpp:56).
 *  - no CPU fallback: without a usable sm_100 device every call that needs
 *    the GPU returns SPMVK_ECUDA.
 */
#ifndef SPMVK_H
#define SPMVK_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPMVK_ABI_VERSION 1

typedef enum {
  SPMVK_OK = 0,
  SPMVK_EINVAL = 1, /* std::invalid_argument in the reference */
  SPMVK_ERANGE = 2, /* std::runtime_error (size budget / 32-bit overflow) */
  SPMVK_ECUDA = 3,  /* CUDA runtime / launch failure */
  SPMVK_ENCCL = 4,  /* collective failure (distributed path) */
  SPMVK_ENOMEM = 5, /* device allocation failure */
  SPMVK_EPARSE = 6  /* Matrix Market syntax error (MatrixMarketError, a std::runtime_error) */
} spmvk_status;

/* Storage precision: the reference's Scalar template argument
 * (spmvkit/memsim.hpp:14-16 Precision; instantiated at src/bench.cpp:135-137). */
typedef enum { SPMVK_F32 = 4, SPMVK_F64 = 8 } spmvk_precision;

typedef struct spmvk_csr spmvk_csr;
typedef struct spmvk_rgcsr spmvk_rgcsr;
typedef struct spmvk_hybrid spmvk_hybrid;
typedef struct spmvk_window spmvk_window;
typedef struct spmvk_dist spmvk_dist;
typedef struct spmvk_comm spmvk_comm;           /* an NCCL communicator (one rank) */
typedef struct spmvk_nccl_iter spmvk_nccl_iter; /* NCCL iterated product of one slab */

/* Thread-local message of the last failing call on this thread. */
const char* spmvk_last_error(void);
int spmvk_abi_version(void);
/* Selects the CUDA device for subsequent calls on this thread and checks it
 * is an sm_100-class part. */
int spmvk_init(int device);
/* Handle arrays (format values / columns / pointers, >= 1 MiB) released by
 * *_destroy are kept in a per-device block cache and reused by the next
 * build of a similar size (no cudaMalloc page mapping, no cudaFree device
 * synchronisation; a reused block is handed out after a device
 * synchronisation).  At most SPMVK_ALLOC_CACHE_MB (default 16384, 0 = off)
 * per device; emptied automatically when cudaMalloc runs out of memory.
 * spmvk_empty_cache returns every cached block to the driver (device < 0:
 * all devices), like torch.cuda.empty_cache for the caching allocator. */
int spmvk_empty_cache(int device);
/* Host buffers for the span overloads (*_spmv_host_*): an anonymous mapping
 * advised to transparent 2 MB huge pages, touched, and page-locked with
 * cudaHostRegister (portable | mapped), so the pipelined host-span path can
 * copy x up with the copy engine and store y straight into it.  Any pinned
 * buffer (cudaHostAlloc, torch pin_memory) works; this one also skips the
 * slow first calls measured on torch-pinned buffers (profiles/r02t_e2e_env.md).
 * *out is 2 MB aligned; free with spmvk_host_free.  No reference
 * counterpart (the reference's spans are over caller memory). */
int spmvk_host_alloc(uint64_t bytes, void** out);
int spmvk_host_free(void* p);

/* ------------------------------------------------------------------ CSR ingest
 * Replaces TripletMatrix(num_rows, num_cols, entries) validation
 * (src/triplet.cpp:22-32) + build_csr<S> (spmvkit/csr.hpp:24-39): the input is
 * a canonical matrix given as CSR arrays on the HOST (row_ptr[rows+1],
 * col[nnz], val[nnz]); entries must be in bounds and strictly increasing in
 * column within each row (EINVAL otherwise, validated on the device).
 * `val_prec` says whether `val` holds double (the triplet's value type) or
 * float (an already-cast CsrMatrix<float>). */
int spmvk_csr_upload(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t* row_ptr,
                     const uint32_t* col, const void* val, int val_prec, void* stream,
                     spmvk_csr** out);
/* Same, from DEVICE arrays (copied device-to-device; the caller keeps its own). */
int spmvk_csr_upload_device(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t* row_ptr,
                            const uint32_t* col, const void* val, int val_prec, void* stream,
                            spmvk_csr** out);
/* Synthetic shapes generated directly in HBM:
 * kind 5 = 2D 5-point n x n, 7 = 3D 7-point n^3, 27 = 3D 27-point n^3. */
int spmvk_csr_stencil(int kind, uint64_t n, void* stream, spmvk_csr** out);
/* rows, cols, nnz, val precision */
int spmvk_csr_shape(const spmvk_csr* a, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                    int* val_prec);
int spmvk_csr_download(const spmvk_csr* a, uint32_t* row_ptr, uint32_t* col, void* val);
/* Row-length statistics (src/triplet.cpp:51-69 row_lengths / matrix_stats):
 * out[0]=max out[1]=min (rows>0). */
int spmvk_csr_row_length_range(const spmvk_csr* a, uint64_t* out2);
/* Matrix Market ingest (parse_matrix_market / load_matrix_market,
 * src/matrix_market.cpp:61-148): same accepted banner, messages and 1-based
 * line numbers ("line N: ..." in spmvk_last_error(), N also in *error_line,
 * SPMVK_EPARSE), canonicalised like spmvkit::canonicalize (sorted, duplicate
 * coordinates summed in the reference's order), then uploaded and validated
 * like spmvk_csr_upload.  Entry lines are parsed with `threads` host threads
 * (0 = all).  A file that cannot be opened gives SPMVK_ERANGE. */
int spmvk_mm_parse(const char* text, uint64_t len, int threads, int val_prec, void* stream,
                   spmvk_csr** out, uint64_t* error_line);
int spmvk_mm_load(const char* path, int threads, int val_prec, void* stream, spmvk_csr** out,
                  uint64_t* error_line);
/* write_matrix_market / save_matrix_market (src/matrix_market.cpp:150-164):
 * the reference's text byte for byte ("%.17g" values, 1-based indices, rows
 * in order), formatted by `threads` host threads (0 = all).  mm_write puts
 * the length in *len and, when buf is non-NULL, the text in buf (ERANGE if
 * cap is too small); mm_save writes the file (ERANGE "cannot open ... for
 * writing"). */
int spmvk_mm_write(const spmvk_csr* a, int threads, char* buf, uint64_t cap, uint64_t* len);
int spmvk_mm_save(const spmvk_csr* a, const char* path, int threads);
/* Smallest / largest column index over rows [row_begin, row_end): the x range
 * a row slab reads (out2[0] > out2[1] for a slab without entries).  Used by
 * the halo exchange of the distributed product. */
int spmvk_csr_column_range(const spmvk_csr* a, uint64_t row_begin, uint64_t row_end,
                           uint64_t* out2);
/* descending_row_permutation (src/reorder.cpp:35-42), on the device: map[i] =
 * old row of new row i, rows by decreasing length, ties by index (stable). */
int spmvk_csr_descending_permutation(const spmvk_csr* a, uint32_t* map);
/* apply_permutation(m, descending_row_permutation(m), RowsOnly)
 * (src/reorder.cpp:44-61): a new CSR whose row i is old row map[i]; `map`
 * (HOST, rows entries, may be NULL) receives the permutation. */
int spmvk_csr_permute_rows_descending(const spmvk_csr* a, void* stream, spmvk_csr** out,
                                      uint32_t* map);
/* apply_permutation(m, Permutation(map), mode) (src/reorder.cpp:12-21,44-61)
 * for any HOST map[new] = old of n entries: row i of the result is old row
 * map[i]; symmetric != 0 also relabels columns (new = inverse[old]) and
 * re-sorts each row, as the reference's canonicalize.  EINVAL with the
 * reference's messages: "permutation is not a bijection on 0..n-1",
 * "apply_permutation: permutation length L does not match R rows",
 * "apply_permutation: symmetric mode needs a square matrix". */
int spmvk_csr_permute(const spmvk_csr* a, const uint32_t* map, uint64_t n, int symmetric,
                      void* stream, spmvk_csr** out);
/* Vectors under a permutation (DEVICE map and vectors): out[i] = in[map[i]]
 * (into the permuted numbering, e.g. x for a symmetric permutation), or with
 * inverse != 0 out[map[i]] = in[i] (y of a permuted matrix back to the
 * original row order; the reference's check `yp[i] == y[p[i]]`,
 * tests/test_reorder.cpp:123-133). */
int spmvk_permute_vector_f64(const uint32_t* map_dev, uint64_t n, const double* in, double* out,
                             int inverse, void* stream);
int spmvk_permute_vector_f32(const uint32_t* map_dev, uint64_t n, const float* in, float* out,
                             int inverse, void* stream);
/* spmv_csr (spmvkit/csr.hpp:41-53): each row accumulated in entry order from
 * +0, products and sums rounded separately (bitwise the reference).  Matrices
 * without rows past 128 entries take a CTA-staged kernel; with them, the
 * warp-staged walk of the Hybrid kernel (dynamic row slices, long rows as
 * work items) -- its long-row list is built once per handle on the first
 * call, which synchronises the stream (make that first call outside a stream
 * capture).  SPMVK_CSR_KERNEL = staged | dyn | warp | row forces a kernel. */
int spmvk_csr_spmv_f64(const spmvk_csr* a, const double* x, uint64_t nx, double* y, uint64_t ny,
                       void* stream);
int spmvk_csr_spmv_f32(const spmvk_csr* a, const float* x, uint64_t nx, float* y, uint64_t ny,
                       void* stream);
void spmvk_csr_destroy(spmvk_csr* a);

/* ------------------------------------------------------------------ RgCSR */
typedef struct {
  uint64_t num_rows, num_cols, group_size, num_groups;
  uint64_t slots;            /* RgcsrMatrix::slot_count (rgcsr.hpp:35) */
  uint64_t nnz;              /* sum of row_lengths = multiply-adds per SpMV */
  uint64_t artificial_zeros; /* FillReport (fill.hpp:90-95) */
  uint64_t bytes_single, bytes_double;
  int precision;
} spmvk_rgcsr_info;

/* build_rgcsr<S>(m, group_size) (spmvkit/rgcsr.hpp:38-70), on the device:
 * row lengths -> per-group max -> scan of s*K_g -> group-interleaved scatter
 * with every pad slot written (value 0, column 0).  EINVAL if group_size==0
 * ("build_rgcsr: group size must be nonzero"); ERANGE if the slot count does
 * not fit uint32 (silently truncated in the reference).  prec may narrow a
 * double CSR to float (static_cast<float>, round-to-nearest-even). */
int spmvk_rgcsr_build(const spmvk_csr* a, uint64_t group_size, int prec, void* stream,
                      spmvk_rgcsr** out);
/* Row slab [row_begin, row_end) of `a` (columns stay global), row_begin a
 * multiple of group_size: the slab's arrays equal the global build's slice
 * (group_pointers rebased).  Used by the row-slab partitioner. */
int spmvk_rgcsr_build_rows(const spmvk_csr* a, uint64_t row_begin, uint64_t row_end,
                           uint64_t group_size, int prec, void* stream, spmvk_rgcsr** out);
int spmvk_rgcsr_get_info(const spmvk_rgcsr* h, spmvk_rgcsr_info* info);
/* Copies the four RgcsrMatrix arrays (rgcsr.hpp:24-27) to HOST buffers of
 * slots / slots / num_groups+1 / num_rows elements (any may be NULL). */
int spmvk_rgcsr_download(const spmvk_rgcsr* h, void* values, uint32_t* columns,
                         uint32_t* group_pointers, uint32_t* row_lengths);
/* to_triplets(RgcsrMatrix) (spmvkit/rgcsr.hpp:107-123): the real slots of
 * every row back to a canonical device CSR (values widened to double). */
int spmvk_rgcsr_to_csr(const spmvk_rgcsr* h, void* stream, spmvk_csr** out);
/* spmv_rgcsr(a, x, y) (spmvkit/rgcsr.hpp:75-97): y = A x with x, y in HBM.
 * EINVAL "spmv_rgcsr: dimension mismatch" unless nx == num_cols and
 * ny == num_rows, or if the handle's precision differs from the entry point. */
int spmvk_rgcsr_spmv_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                         uint64_t ny, void* stream);
int spmvk_rgcsr_spmv_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                         uint64_t ny, void* stream);
/* Iterated form used by the distributed product: y = A x and, fused in the
 * same kernel, x_next[i] = y[i] * scale (x_next may be NULL). */
int spmvk_rgcsr_spmv_scaled_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                                uint64_t ny, double* x_next, double scale, void* stream);
int spmvk_rgcsr_spmv_scaled_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                                uint64_t ny, float* x_next, float scale, void* stream);
/* Span overloads on HOST memory: H2D(x), SpMV, D2H(y), synchronous.
 * multiply_add_count (may be NULL) receives the reference's madds count
 * (rgcsr.hpp:72-74: one per stored nonzero). */
int spmvk_rgcsr_spmv_host_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, uint64_t* multiply_add_count);
int spmvk_rgcsr_spmv_host_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, uint64_t* multiply_add_count);
void spmvk_rgcsr_destroy(spmvk_rgcsr* h);
/* L2 persistence window for the gathered vector x (the north star's "x
 * served ... with L2 persistence windows"): sets the device's persisting-L2
 * carve-out to min(bytes, cudaDevAttrMaxPersistingL2CacheSize) and the
 * stream's access-policy window over [x, x + bytes) (hits persisting, misses
 * streaming; hit_ratio scaled down when x exceeds the carve-out).  Every
 * kernel later launched on `stream` then keeps x's lines resident while the
 * matrix streams past.  x == NULL or bytes == 0 resets (no window, carve-out
 * 0).  `granted` (optional) receives the carve-out in bytes.  Does not change
 * y.  (No reference counterpart: the CPU reference has no cache control.) */
int spmvk_stream_persist_x(void* stream, const void* x, uint64_t bytes, double hit_ratio,
                           uint64_t* granted);
/* Tuning knob (process-wide): which K2 kernel runs.  "auto" (default:
 * without long rows and with <= 10 % padding the group-uniform walk -- fp32
 * with <= 12 slots per row grpv4 (128-bit slot loads, 4 rows per thread),
 * else grp6 (<= 5.5 slots per row) / grp8_r64 (fp64) / grp8 or grp7_mpf
 * (fp32), launched with programmatic dependent launch unless SPMVK_PDL=0;
 * with rows past the long-row cut the row-pipelined kernel with the long rows
 * fused in (pipe_fl: long-row work items, then dynamic 128-row slices);
 * heavily padded matrices without long rows lite8 for fp64, lite or
 * lite8_full for fp32), "grp6" / "grp7_mpf" / "grp8" / "grp8_r64" (group-
 * uniform walk: U-deep slot batches bound by the group width, scheduling
 * fence before the x gathers, row_lengths skipped when x[0] is finite, next
 * row's group pointers prefetched), "grpv4" (the same walk with 128-bit
 * slot vectors, 4 rows per thread, U = 4), "lite" / "lite8" / "lite8_full"
 * (register-lean thread per row), "liteh" / "lite8h" (same with L2 eviction
 * hints), "vec2" (128-bit loads of 2 / 4 rows, per-row lengths), "pipe"
 * (row-metadata prefetch, predicated batches, L2 hints).  All give bitwise
 * identical y; the measured comparison (and the variants removed in round 2)
 * are in DESIGN.md §3, profiles/r02_k2_pruned.md and profiles/r02_grpv.md.
 * Also read from SPMVK_RGCSR_KERNEL. */
int spmvk_set_rgcsr_kernel(const char* name);
/* Tuning knob (process-wide, read at build): rows with more than `cut` slots
 * (default 128) are handled by a warp-per-row kernel instead of one thread
 * (power-law tails).  Does not change y. */
int spmvk_set_long_row_cut(uint32_t cut);
/* Tuning knob (process-wide, read at launch): 1 (default) fuses the long rows
 * into the thread-per-row kernel (its warps take the long-row items first,
 * dynamically, then their tiles; one launch), 0 runs them as a separate
 * launch after it.  Does not change y.  Also read from SPMVK_LONG_FUSED.
 * The fused kernels (and the Hybrid "dyn" kernel) take work from four 32-bit
 * counters per (device, stream) that the last warp of each launch resets:
 * launches on one stream are ordered, so they never share live counters --
 * do not destroy a stream and recreate one while work it queued on those
 * kernels is still running (a recycled handle would share them). */
int spmvk_set_long_fused(int on);

/* ------------------------------------------------------------------ Hybrid */
/* Tuning knob (process-wide): Hybrid SpMV kernel variant.  "auto" (default:
 * pure ELL -> the group-walk batch shape matching K1: "g6" for K1 <= 6,
 * "litef" up to 12, "g7" beyond; with a COO part "dyn" for spmv_hybrid and
 * "litef", fp32 "litefh" for the spmv_coo part alone),
 * "v4" (first kernel: policy-hinted loads, 4-deep), "lite" / "lite8" /
 * "lite8_full" (register-lean ELL loop, 4- or 8-deep batches at 8 / 5 / 8
 * CTAs per SM), "litef" / "lite8f" (same, 4-deep at 8 / 8-deep at 4 CTAs per
 * SM, with a scheduling fence that issues every slot load before the x
 * gathers), "g6" / "g7" / "g8" / "g8r" (fenced, U = 6 / 7 / 8 at 5 CTAs per
 * SM, U = 8 at 4; pure-ELL launches only), "litefh" (litef with L2 eviction
 * hints), "dyn" (spmv_hybrid with a COO part: rows in dynamic 128-row slices,
 * each 32-row slice's COO range staged per warp -- no block barrier, no row
 * search -- and rows with COO runs over 128 entries as warp work items taken
 * first, longest first; other parts fall back to "litef").  All give bitwise
 * identical y.  Also read from SPMVK_HYBRID_KERNEL. */
int spmvk_set_hybrid_kernel(const char* name);
typedef struct {
  uint64_t num_rows, num_cols;
  uint64_t ell_width;        /* K1 = EllpackMatrix::slots_per_row */
  uint64_t ell_slots;        /* num_rows * K1 */
  uint64_t coo_nnz;
  uint64_t nnz;              /* stored entries of the source matrix (multiply-adds) */
  uint64_t fill_nnz;         /* FillReport::nnz: ell_nnz recount + coo (fill.hpp:67-72) */
  uint64_t artificial_zeros; /* FillReport: slots - fill_nnz */
  uint64_t bytes_single, bytes_double;
  int precision;
  int ellpack;               /* 1: built by spmvk_ellpack_build (FillReport "ellpack") */
} spmvk_hybrid_info;

/* hybrid_split_cost / choose_ell_width (spmvkit/ellpack.hpp:143-166) over the
 * row lengths of `a`, computed from a device histogram + suffix sums: the same
 * integer argmin (smallest k on ties) in O(N + max_len). */
int spmvk_csr_choose_ell_width(const spmvk_csr* a, uint64_t* k1);
/* Host helper with the reference signature (lens[n]); exact same result. */
uint64_t spmvk_choose_ell_width(const uint64_t* lens, uint64_t n);
uint64_t spmvk_hybrid_split_cost(const uint64_t* lens, uint64_t n, uint64_t k);
/* build_hybrid<S>(m, k1) (spmvkit/ellpack.hpp:168-203); k1 < 0 means
 * std::nullopt (choose_ell_width).  EINVAL if k1 > max row length. */
int spmvk_hybrid_build(const spmvk_csr* a, int64_t k1, int prec, void* stream,
                       spmvk_hybrid** out);
/* build_ellpack<S>(m, slot_budget) (spmvkit/ellpack.hpp:84-107): a Hybrid
 * handle with K1 = the maximum row length and no COO part, flagged ellpack
 * (its FillReport is fill_report(EllpackMatrix): index words = slots).
 * ERANGE "build_ellpack: R rows x width K exceeds the slot budget of B" when
 * rows > slot_budget / K (the reference's default budget is 2^31). */
int spmvk_ellpack_build(const spmvk_csr* a, uint64_t slot_budget, int prec, void* stream,
                        spmvk_hybrid** out);
int spmvk_hybrid_get_info(const spmvk_hybrid* h, spmvk_hybrid_info* info);
/* EllpackMatrix values/columns (slot-major, rows*K1) + CooArrays
 * rows/columns/values (coo_nnz); any pointer may be NULL. */
int spmvk_hybrid_download(const spmvk_hybrid* h, void* ell_values, uint32_t* ell_columns,
                          uint32_t* coo_rows, uint32_t* coo_columns, void* coo_values);
/* to_triplets(HybridMatrix) (spmvkit/ellpack.hpp:219-240): ELL rows through
 * the ell_row_length recount (:55-78) plus the COO overflow, as a canonical
 * device CSR (double values). */
int spmvk_hybrid_to_csr(const spmvk_hybrid* h, void* stream, spmvk_csr** out);
/* spmv_hybrid (spmvkit/ellpack.hpp:205-210) = spmv_ellpack (:110-123) then
 * spmv_coo (:132-141), fused in one kernel; y is bitwise the reference's. */
int spmvk_hybrid_spmv_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                          uint64_t ny, void* stream);
int spmvk_hybrid_spmv_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                          uint64_t ny, void* stream);
/* spmv_ellpack(h.ell, x, y) (ellpack.hpp:110-123): y = the ELL part only,
 * every slot walked (pads add 0 * x[0]); EINVAL "spmv_ellpack: dimension
 * mismatch" unless nx == cols and ny == rows. */
int spmvk_hybrid_spmv_ell_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, void* stream);
int spmvk_hybrid_spmv_ell_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, void* stream);
/* spmv_coo(h.coo, x, y) (ellpack.hpp:132-141): y[row] += v * x[col] for the
 * COO part in array order (accumulates into the caller's y); EINVAL
 * "spmv_coo: entry outside x/y dimensions" if an entry's row >= ny or
 * column >= nx. */
int spmvk_hybrid_spmv_coo_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, void* stream);
int spmvk_hybrid_spmv_coo_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, void* stream);
/* The same two parts on host spans (x, y in host memory; synchronous). */
int spmvk_hybrid_spmv_ell_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx,
                                   double* y, uint64_t ny);
int spmvk_hybrid_spmv_ell_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                                   uint64_t ny);
int spmvk_hybrid_spmv_coo_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx,
                                   double* y, uint64_t ny);
int spmvk_hybrid_spmv_coo_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                                   uint64_t ny);
int spmvk_hybrid_spmv_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                               uint64_t ny);
int spmvk_hybrid_spmv_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                               uint64_t ny);
void spmvk_hybrid_destroy(spmvk_hybrid* h);

/* ------------------------------------------------------------------ CG
 * Unpreconditioned conjugate gradients for an SPD fp64 RgCSR matrix, fully
 * device-resident (scalars never leave HBM; the host reads the residual every
 * `check_every` iterations).  b, x are DEVICE vectors of n; x holds the initial
 * guess and receives the solution.  Stops when ||r|| <= tol * ||b|| or after
 * max_iter iterations.  Dots are deterministic (fixed-grid partials). */
int spmvk_cg_solve_f64(const spmvk_rgcsr* a, const double* b, double* x, uint64_t n, double tol,
                       uint64_t max_iter, uint64_t check_every, uint64_t* iters,
                       double* rel_residual, void* stream);
/* Reductions (the dots below, spmv_dot, cg_solve) use device scratch private
 * to the (device, stream) pair, so calls on different streams -- from one
 * host thread or many -- never share partial sums. */
/* y = A x and dot_out (device scalar) = sum_r x[x_offset + r] * y[r] -- CG's
 * p.q fused into the SpMV's row epilogue (rows of a square matrix or of a row
 * slab whose rows start at global row x_offset).  Deterministic (fixed
 * per-CTA partials, fixed reduction order); falls back to the SpMV followed
 * by spmvk_dot_f64 for matrices with long rows or > 10 % padding.  No
 * reference counterpart (CG is not in the reference). */
int spmvk_rgcsr_spmv_dot_f64(const spmvk_rgcsr* a, const double* x, uint64_t nx, double* y,
                             uint64_t ny, uint64_t x_offset, double* dot_out, void* stream);
/* out_dev[0] = a . b (deterministic), device pointers. */
int spmvk_dot_f64(const double* a, const double* b, uint64_t n, double* out_dev, void* stream);
/* CG building blocks for the row-slab distributed solver (device pointers,
 * n = slab rows; dots are the slab's partials, all-reduced by the caller):
 * update: alpha = *rr / *pap; x += alpha p; r -= alpha q; *rr_new = r . r.
 * direction: p = r + (*rr_new / *rr) p; then *rr = *rr_new. */
int spmvk_cg_update_f64(uint64_t n, const double* rr, const double* pap, const double* p,
                        const double* q, double* x, double* r, double* rr_new, void* stream);
int spmvk_cg_direction_f64(uint64_t n, const double* r, double* p, double* rr,
                           const double* rr_new, void* stream);

/* ------------------------------------------------------------------ fused multi-GPU step
 * SURVEY §8e (the reference has no multi-GPU path; §8b lists spmvk_dist_*):
 * row slabs, x_{k+1} = (A x_k)_slab * scale, with the x exchange fused into
 * the SpMV's row epilogue as stores into the peers' exchange windows over
 * NVLink (no separate collective), and one device-side flag barrier per step.
 *
 * Window: two x buffers of n entries (double-buffered) + flags, in this
 * device's HBM, zero-initialised.  Export it with spmvk_window_ipc_handle
 * (64 bytes, cudaIpcMemHandle_t) and exchange the handles out of band (MPI,
 * torch.distributed, a file); every rank then calls spmvk_dist_open with the
 * handles of all ranks in rank order (its own entry is ignored).  Ranks that
 * live in ONE process (one process driving several GPUs, or tests sharing a
 * device) use spmvk_dist_open_local with the window pointers instead.
 * At most 8 ranks (one NVLink domain node).  Destroy a window only after
 * every peer has destroyed the dist handle that opened it. */
int spmvk_window_create(uint64_t n, int prec, spmvk_window** out);
int spmvk_window_ipc_handle(const spmvk_window* w, unsigned char* handle_out);
/* Device pointer of x buffer 0 or 1 (write the starting x into the buffer
 * spmvk_dist_current names before the first step). */
int spmvk_window_x(const spmvk_window* w, int buffer, void** out);
void spmvk_window_destroy(spmvk_window* w);
int spmvk_dist_open(const spmvk_window* own, int rank, int world, const unsigned char* handles,
                    spmvk_dist** out);
int spmvk_dist_open_local(const spmvk_window* const* windows, int rank, int world,
                          spmvk_dist** out);
/* This rank's slab = global rows [row_begin, row_end) (its RgCSR holds
 * exactly those rows, global columns).  receive_ranges[2q], [2q+1]: global
 * rows [lo, hi) that rank q must receive every step: for peers either
 * everything (all-gather) or the rows their slab reads (halo,
 * partition.fused_receive_ranges).  Only the part inside this rank's slab is
 * sent; the rank's own rows always go to its own window (its own entry is
 * not consulted). */
int spmvk_dist_set_rows(spmvk_dist* d, uint64_t row_begin, uint64_t row_end,
                        const uint64_t* receive_ranges);
/* Distributed CG direction step with the p exchange fused in: for this
 * rank's rows p_new = r_local + (rr_new / rr) p_old (p_old = the window's
 * current buffer), stored into the next buffer of the own window and of every
 * peer window whose receive range covers the row (NVLink stores -- no
 * all-gather); then rr = rr_new, the buffer flip and (barrier != 0) the flag
 * barrier.  The slab SpMV of the next iteration reads p from the window
 * (spmvk_window_x(window, current)).  fp64 only. */
int spmvk_dist_cg_direction_f64(spmvk_dist* d, const double* r_local, double* rr,
                                const double* rr_new, int barrier, void* stream);
/* One step: y = A_slab x[cur] (slab-local y, device), x_next = y * scale
 * stored into x[1-cur] of every window whose receive range covers the row,
 * then (barrier != 0) the device barrier; cur flips.  barrier = 0 is for
 * ranks stepped one after another by one host thread on one device. */
int spmvk_dist_step_f64(spmvk_dist* d, const spmvk_rgcsr* slab, double scale, double* y,
                        int barrier, void* stream);
int spmvk_dist_step_f32(spmvk_dist* d, const spmvk_rgcsr* slab, float scale, float* y,
                        int barrier, void* stream);
int spmvk_dist_current(const spmvk_dist* d, int* buffer);
/* Bound on one barrier's wait for a peer (default 30 s).  A barrier that
 * times out records the peer in the window's status word and returns; every
 * later barrier of the window then returns at once (no hang). */
int spmvk_dist_set_timeout_ms(spmvk_dist* d, uint64_t ms);
/* Synchronises `stream` and returns SPMVK_ENCCL (message names the missing
 * rank) if a barrier of this rank's window timed out, else SPMVK_OK. */
int spmvk_dist_status(const spmvk_dist* d, void* stream);
void spmvk_dist_destroy(spmvk_dist* d);

/* ------------------------------------------------------------------ partition planning
 * contiguous row slabs whose boundaries are multiples of the
 * group size G, so a slab's RgCSR is exactly the global arrays' slice and
 * every row keeps the reference's accumulation order.  Pure host code (no
 * device needed).  `bounds` has parts + 1 entries: slab p = rows
 * [bounds[p], bounds[p + 1]). */
typedef enum { SPMVK_EXCHANGE_ALLGATHER = 0, SPMVK_EXCHANGE_HALO = 1 } spmvk_exchange;
/* Equal slabs of S = ceil(groups / parts) * G rows (*slab_rows = S; the last
 * slabs may be short or empty): bounds[p] = min(rows, p * S). */
int spmvk_plan_slabs(uint64_t rows, uint64_t group_size, int parts, uint64_t* bounds,
                     uint64_t* slab_rows);
/* Slot-balanced cuts for skewed matrices (the power-law config): cut p is
 * the first group boundary where the running RgCSR slot count reaches p/parts
 * of the total.  row_lengths: host array of `rows` entries. */
int spmvk_plan_slabs_weighted(const uint32_t* row_lengths, uint64_t rows, uint64_t group_size,
                              int parts, uint64_t* bounds);
/* Global rows [receive[2q], receive[2q+1]) rank q must hold every step: all
 * of x (ALLGATHER) or its own rows plus the columns its slab reads (HALO;
 * column_ranges[2q], [2q+1] = min, max column of slab q, min > max if the
 * slab has no entries -- spmvk_csr_column_range).  This is what
 * spmvk_dist_set_rows takes. */
int spmvk_plan_receive(int parts, const uint64_t* bounds, const uint64_t* column_ranges, int mode,
                       uint64_t* receive);
/* Halo lists of `rank` (arrays of up to parts - 1 triples, ascending peer):
 * recv[3k..3k+2] = (peer, c0, c1): columns [c0, c1) this slab reads that the
 * peer owns; send[...] = (peer, c0, c1): this slab's rows the peer reads. */
int spmvk_plan_halo(int rank, int parts, const uint64_t* bounds, const uint64_t* column_ranges,
                    uint64_t* recv, int* n_recv, uint64_t* send, int* n_send);

/* ------------------------------------------------------------------ NCCL iterated product
 * x_{k+1} = (A_slab x_k) * scale per rank (scale fused into
 * the SpMV epilogue), then the x exchange over NCCL: an in-place
 * ncclAllGather of every rank's slab (equal slabs from spmvk_plan_slabs), or
 * grouped ncclSend / ncclRecv of only the column ranges each slab reads
 * (HALO).  Stream ordered, double-buffered x; the iterate is bitwise the
 * single-GPU iterate.  NCCL is bound at run time (dlopen libnccl.so.2 or
 * $SPMVK_NCCL_LIB); SPMVK_ENCCL if it is missing or a call fails.
 *
 * Communicators: one process per GPU -> rank 0 calls spmvk_nccl_unique_id,
 * the 128 bytes travel out of band (MPI, a file, torch.distributed), every
 * rank calls spmvk_comm_init_rank (ncclCommInitRank).  One process driving
 * several GPUs -> spmvk_comm_init_all (ncclCommInitAll); it must then bracket
 * the per-rank calls of one step with spmvk_nccl_group_start / _end. */
#define SPMVK_NCCL_ID_BYTES 128
int spmvk_nccl_version(int* version);
int spmvk_nccl_unique_id(unsigned char* id_out);
int spmvk_comm_init_rank(const unsigned char* id, int world, int rank, int device,
                         spmvk_comm** out);
/* out: ndev handles, rank i on devices[i] (devices NULL -> 0..ndev-1). */
int spmvk_comm_init_all(int ndev, const int* devices, spmvk_comm** out);
int spmvk_comm_info(const spmvk_comm* c, int* rank, int* world, int* device);
void spmvk_comm_destroy(spmvk_comm* c);
int spmvk_nccl_group_start(void);
int spmvk_nccl_group_end(void);
/* Collective over the communicator (every rank calls it): this rank's slab =
 * global rows [row_begin, row_end) with `slab` its RgCSR (global columns), n
 * the global length of x.  ALLGATHER needs row_begin = rank * slab_rows (the
 * spmvk_plan_slabs layout); HALO takes any contiguous slabs in rank order.
 * The ranks' plans (rows, column ranges) are exchanged with one ncclAllGather. */
int spmvk_nccl_iter_create(spmvk_comm* comm, const spmvk_rgcsr* slab, uint64_t row_begin,
                           uint64_t row_end, uint64_t slab_rows, uint64_t n, int mode,
                           spmvk_nccl_iter** out);
/* Device pointer (and length) of x buffer 0 / 1; write x_0 into the buffer
 * spmvk_nccl_iter_current names before the first step. */
int spmvk_nccl_iter_x(const spmvk_nccl_iter* it, int buffer, void** out, uint64_t* length);
int spmvk_nccl_iter_current(const spmvk_nccl_iter* it, int* buffer);
/* Entries of x this rank receives per step (halo: the columns it reads from
 * peers; all-gather: the other ranks' slabs). */
int spmvk_nccl_iter_halo_entries(const spmvk_nccl_iter* it, uint64_t* entries);
/* One step: y (slab-local, device) = A_slab x[cur]; x[1-cur] gets this slab's
 * x_next = y * scale and, after the exchange, every entry this rank reads;
 * cur flips. */
int spmvk_nccl_iter_step_f64(spmvk_nccl_iter* it, double scale, double* y, void* stream);
int spmvk_nccl_iter_step_f32(spmvk_nccl_iter* it, float scale, float* y, void* stream);
void spmvk_nccl_iter_destroy(spmvk_nccl_iter* it);

/* ------------------------------------------------------------------ host generators
 * Seeded, platform-independent generators (std::mt19937_64 draws, the
 * reference's unit_real convention src/synthetic.cpp:7-9).  Two-pass: pass
 * col/val NULL to get nnz, then call again with buffers. */
/* random_vector (src/synthetic.cpp:62-67) */
void spmvk_gen_random_vector(uint64_t n, uint64_t seed, double* out);
/* Stencils as spmvk_csr_stencil, on the host.  Returns nnz. */
uint64_t spmvk_gen_stencil(int kind, uint64_t n, uint32_t* row_ptr, uint32_t* col, double* val);
/* Power-law rows.  Returns nnz. */
uint64_t spmvk_gen_powerlaw(uint64_t rows, uint64_t seed, uint32_t* row_ptr, uint32_t* col,
                            double* val);
/* Row-wise random matrix for the sweep: each row draws its length uniformly
 * in [1, 2*mean_len-1] and distinct uniform columns.  Returns nnz. */
uint64_t spmvk_gen_random_rows(uint64_t rows, uint64_t cols, uint64_t mean_len, uint64_t seed,
                               uint32_t* row_ptr, uint32_t* col, double* val);
/* b x b dense blocks on random block columns, nblk blocks per block row. */
uint64_t spmvk_gen_block(uint64_t rows, uint64_t b, uint64_t nblk, uint64_t seed,
                         uint32_t* row_ptr, uint32_t* col, double* val);
/* banded_matrix (src/synthetic.cpp:48-60). */
uint64_t spmvk_gen_banded(uint64_t n, uint64_t hbw, uint64_t seed, uint32_t* row_ptr,
                          uint32_t* col, double* val);

#ifdef __cplusplus
}
#endif
#endif
