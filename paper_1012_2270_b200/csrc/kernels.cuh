// Cross-file kernel/host helpers of the spmvk library.
#pragma once
#include "common.cuh"

namespace spmvk {

// lens[r] = rp[r0 + r + 1] - rp[r0 + r] for r < rows
__global__ void csr_row_lengths(uint64_t r0, uint64_t rows, const uint32_t* __restrict__ rp,
                                uint32_t* __restrict__ lens);

// An empty device CSR handle with arrays allocated (row_ptr rows+1, nnz entries).
spmvk_csr* new_csr(uint64_t rows, uint64_t cols, uint64_t nnz, int val_prec);

// max / min row length over rows [r0, r1) (synchronous)
void row_length_range(const spmvk_csr* a, uint64_t r0, uint64_t r1, unsigned* mx, unsigned* mn,
                      cudaStream_t s);

// spmv_csr through the warp-staged kernel of hybrid_spmv_dyn (every entry a
// "COO" entry, row_ptr as the run pointers; hybrid.cu).  With only_if_heavy
// it launches only when the matrix has rows past 128 entries (returns
// whether it launched); the heavy-row list is built once per handle.
template <class T>
bool csr_spmv_dyn(const spmvk_csr* a, const T* x, T* y, cudaStream_t s, bool only_if_heavy);

}  // namespace spmvk
