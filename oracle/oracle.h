/* oracle/oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (arxiv/paper_1012_2270,
 * /root/reference/proj/core).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the
 * CHECKER.  The product (libspmvk.so) never links or calls it.
 *
 * Parity of this restatement is PINNED against the reference itself: every
 * function is cross-checked in tests/test_oracle_pinned.py against
 * oracle/_ref/libspmvkit_ref.so (the unmodified reference compiled in place)
 * and against the committed golden vectors in tests/golden/ that
 * oracle/make_golden.py generated from it.
 *
 * Matrices are passed as canonical CSR (row_ptr[rows+1], col[nnz], val[nnz]);
 * a canonical reference TripletMatrix (entries strictly increasing in
 * (row, col), triplet.hpp:26-45) is exactly this CSR, entry k of the sorted
 * triplet list being CSR entry k.
 */
#ifndef SPMVK_ORACLE_H
#define SPMVK_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 + unit_real (src/synthetic.cpp:7-9) */
typedef struct { uint64_t mt[312]; int mti; } orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);
double orc_unit_real(orc_mt64* s);

/* random_vector (src/synthetic.cpp:62-67) */
void orc_random_vector(uint64_t n, uint64_t seed, double* out);

/* random_matrix (src/synthetic.cpp:28-46); two-pass: call with col/val NULL to
 * size, returns nnz.  row_ptr must have rows+1 entries. */
uint64_t orc_random_matrix(uint64_t rows, uint64_t cols, double density, int vmin, int vmax,
                           int integer_values, int allow_zero, uint64_t seed, uint32_t* row_ptr,
                           uint32_t* col, double* val);
/* tests/fixtures.hpp:50-60 random_small: shape draws then random_matrix. */
void orc_random_small_spec(uint64_t seed, uint64_t* rows, uint64_t* cols, double* density,
                           uint64_t* matrix_seed);
/* banded_matrix (src/synthetic.cpp:48-60); returns nnz, two-pass like above. */
uint64_t orc_banded(uint64_t n, uint64_t hbw, uint64_t seed, uint32_t* row_ptr, uint32_t* col,
                    double* val);

/* spmv_reference (src/triplet.cpp:71-79) */
void orc_spmv_reference(uint64_t rows, const uint32_t* row_ptr, const uint32_t* col,
                        const double* val, const double* x, double* y);

/* spmv_csr (spmvkit/csr.hpp:41-53) */
void orc_spmv_csr_f64(uint64_t rows, const uint32_t* rp, const uint32_t* col, const double* val,
                      const double* x, double* y);
void orc_spmv_csr_f32(uint64_t rows, const uint32_t* rp, const uint32_t* col, const float* val,
                      const float* x, float* y);

/* build_rgcsr (spmvkit/rgcsr.hpp:38-70) in two steps: layout then scatter.
 * orc_rgcsr_layout fills row_lengths[rows] and group_pointers[groups+1] and
 * returns the slot count, or UINT64_MAX when group_size == 0.  The reference
 * truncates the uint32 group pointers silently (rgcsr.hpp:56); *overflow is
 * set to 1 when the true slot count does not fit in 32 bits. */
uint64_t orc_rgcsr_layout(uint64_t rows, const uint32_t* rp, uint64_t group_size,
                          uint32_t* row_lengths, uint32_t* group_pointers, int* overflow);
void orc_rgcsr_fill_f64(uint64_t rows, const uint32_t* rp, const uint32_t* col,
                        const double* val, uint64_t group_size, const uint32_t* group_pointers,
                        double* values, uint32_t* columns);
void orc_rgcsr_fill_f32(uint64_t rows, const uint32_t* rp, const uint32_t* col,
                        const double* val, uint64_t group_size, const uint32_t* group_pointers,
                        float* values, uint32_t* columns);
/* spmv_rgcsr (spmvkit/rgcsr.hpp:75-97); returns the multiply-add count. */
uint64_t orc_spmv_rgcsr_f64(uint64_t rows, uint64_t group_size, const uint32_t* gp,
                            const uint32_t* lens, const double* values, const uint32_t* columns,
                            const double* x, double* y);
uint64_t orc_spmv_rgcsr_f32(uint64_t rows, uint64_t group_size, const uint32_t* gp,
                            const uint32_t* lens, const float* values, const uint32_t* columns,
                            const float* x, float* y);

/* hybrid_split_cost / choose_ell_width (spmvkit/ellpack.hpp:143-166) */
uint64_t orc_hybrid_split_cost(const uint64_t* lens, uint64_t n, uint64_t k);
uint64_t orc_choose_ell_width(const uint64_t* lens, uint64_t n);
/* build_hybrid (spmvkit/ellpack.hpp:168-203).  Returns the COO count, or
 * UINT64_MAX when k1 > max row length (the reference throws). */
uint64_t orc_hybrid_coo_count(uint64_t rows, const uint32_t* rp, uint64_t k1);
void orc_hybrid_fill_f64(uint64_t rows, const uint32_t* rp, const uint32_t* col,
                         const double* val, uint64_t k1, double* ell_values,
                         uint32_t* ell_columns, uint32_t* coo_rows, uint32_t* coo_columns,
                         double* coo_values);
void orc_hybrid_fill_f32(uint64_t rows, const uint32_t* rp, const uint32_t* col,
                         const double* val, uint64_t k1, float* ell_values,
                         uint32_t* ell_columns, uint32_t* coo_rows, uint32_t* coo_columns,
                         float* coo_values);
/* spmv_ellpack + spmv_coo = spmv_hybrid (spmvkit/ellpack.hpp:110-141,205-210) */
void orc_spmv_hybrid_f64(uint64_t rows, uint64_t k1, const double* ell_values,
                         const uint32_t* ell_columns, uint64_t coo_n, const uint32_t* coo_rows,
                         const uint32_t* coo_columns, const double* coo_values, const double* x,
                         double* y);
void orc_spmv_hybrid_f32(uint64_t rows, uint64_t k1, const float* ell_values,
                         const uint32_t* ell_columns, uint64_t coo_n, const uint32_t* coo_rows,
                         const uint32_t* coo_columns, const float* coo_values, const float* x,
                         float* y);

/* descending_row_permutation (src/reorder.cpp:35-42): stable sort by
 * decreasing row length, ties by original index.  map[new] = old. */
void orc_descending_map(uint64_t rows, const uint32_t* rp, uint32_t* map);

/* Synthetic shapes — independent restatement used to
 * cross-check the product's generators.  kind: 5 (2D 5-pt), 7 (3D 7-pt),
 * 27 (3D 27-pt).  Two-pass (col/val NULL sizes).  Returns nnz. */
uint64_t orc_stencil(int kind, uint64_t n, uint32_t* row_ptr, uint32_t* col, double* val);
/* power-law rows (Appendix B): two-pass; returns nnz. */
uint64_t orc_powerlaw(uint64_t rows, uint64_t seed, uint32_t* row_ptr, uint32_t* col,
                      double* val);

#ifdef __cplusplus
}
#endif
#endif
