// Descending row reordering on the device.
//
// Reference: descending_row_permutation (src/reorder.cpp:35-42) — a STABLE
// sort of row ids by decreasing row length, ties by original index — and
// apply_permutation(m, p, RowsOnly) (src/reorder.cpp:44-61): new row i is old
// row map[i], columns unchanged.  Grouping rows of similar length is the
// paper's remedy for RgCSR padding (fd18 fill 2.76% ->
// 0.34%); the power-law config drops from 340% to a few percent.
//
// The permutation is a stable radix sort of (max_len - len) keys with row-id
// payloads (cub::DeviceRadixSort, CUDA toolkit; it is stable, which is exactly
// the reference's std::stable_sort order); the permuted CSR is built by a
// row-length gather, an exclusive scan and a warp-per-row entry copy.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <vector>

#include <memory>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvk {
namespace {

__global__ void sort_keys(uint64_t rows, uint32_t max_len, const uint32_t* __restrict__ rp,
                          uint32_t* __restrict__ key, uint32_t* __restrict__ id) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    key[r] = max_len - (rp[r + 1] - rp[r]);
    id[r] = (uint32_t)r;
  }
}

__global__ void permuted_lengths(uint64_t rows, const uint32_t* __restrict__ map,
                                 const uint32_t* __restrict__ rp, uint64_t* __restrict__ len) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o = map[i];
    len[i] = rp[o + 1] - rp[o];
  }
}

// inv != nullptr: symmetric mode, columns relabelled new = inv[old] (the
// row's entries are then re-sorted by a segmented sort).
constexpr uint64_t kPermBlockMax = 32 * 64;
template <class V>
__global__ void permuted_copy(uint64_t rows, uint64_t nnz, const uint32_t* __restrict__ map,
                              const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                              const V* __restrict__ val, const uint64_t* __restrict__ off,
                              uint32_t* __restrict__ rp2, uint32_t* __restrict__ col2,
                              V* __restrict__ val2, const uint32_t* __restrict__ inv,
                              uint32_t* __restrict__ heavy_blocks,
                              unsigned* __restrict__ n_heavy_blocks) {
  // A warp per 32 output rows: their entries are one contiguous output range
  // [off[i0], off[i0 + 32]), written 32 entries at a time (coalesced), each
  // lane finding its entry's output row by a shuffle binary search over the
  // rows' offsets.  Blocks of more than kPermBlockMax entries (long rows
  // together, e.g. the first blocks of a descending order) are listed for
  // permuted_copy_rows, a warp per row spread over the grid.
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t blocks = (rows + 31) / 32;
  for (uint64_t blk = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); blk < blocks;
       blk += warps) {
    const uint64_t i = blk * 32 + lane;
    const bool live = i < rows;
    const uint64_t d = live ? off[i] : 0;
    const uint32_t src = live ? rp[map[i]] : 0;
    if (live) {
      rp2[i] = (uint32_t)d;
      if (i + 1 == rows) rp2[rows] = (uint32_t)nnz;
    }
    const uint64_t last = min(rows, blk * 32 + 32) - 1;
    const uint64_t d0 = __shfl_sync(0xffffffffu, d, 0);
    const uint64_t d1 = last + 1 == rows ? nnz : off[last + 1];
    if (d1 - d0 > kPermBlockMax) {
      if (lane == 0) heavy_blocks[atomicAdd(n_heavy_blocks, 1u)] = (uint32_t)blk;
      continue;
    }
    for (uint64_t e0 = d0; e0 < d1; e0 += 32) {
      const uint64_t e = e0 + lane;
      int q = 0;  // the largest lane q with off[q] <= e (empty rows are skipped past)
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint64_t dq = __shfl_sync(0xffffffffu, d, q + step);
        if ((uint64_t)(blk * 32 + q + step) < rows && dq <= e) q += step;
      }
      const uint64_t dq = __shfl_sync(0xffffffffu, d, q);
      const uint32_t sq = __shfl_sync(0xffffffffu, src, q);
      if (e < d1) {
        const uint64_t k = (uint64_t)sq + (e - dq);
        const uint32_t c = col[k];
        col2[e] = inv ? inv[c] : c;
        val2[e] = val[k];
      }
    }
  }
}

// The rows of the listed heavy blocks: a warp per row.
template <class V>
__global__ void permuted_copy_rows(uint64_t rows, const uint32_t* __restrict__ map,
                                   const uint32_t* __restrict__ rp,
                                   const uint32_t* __restrict__ col, const V* __restrict__ val,
                                   const uint64_t* __restrict__ off, uint32_t* __restrict__ col2,
                                   V* __restrict__ val2, const uint32_t* __restrict__ inv,
                                   const uint32_t* __restrict__ heavy_blocks,
                                   const unsigned* __restrict__ n_heavy_blocks) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t n = (uint64_t)*n_heavy_blocks * 32;
  for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n;
       w += warps) {
    const uint64_t i = (uint64_t)heavy_blocks[w / 32] * 32 + (w % 32);
    if (i >= rows) continue;
    const uint32_t o = map[i], b = rp[o], len = rp[o + 1] - b;
    const uint64_t d = off[i];
    for (uint32_t k = lane; k < len; k += 32) {
      const uint32_t c = col[b + k];
      col2[d + k] = inv ? inv[c] : c;
      val2[d + k] = val[b + k];
    }
  }
}

__global__ void invert_map(uint64_t n, const uint32_t* __restrict__ map, uint32_t* __restrict__ inv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    inv[map[i]] = (uint32_t)i;
}

template <class V>
__global__ void permute_vector(uint64_t n, const uint32_t* __restrict__ map, const V* __restrict__ in,
                               V* __restrict__ out, int inverse) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (inverse) out[map[i]] = in[i];
    else out[i] = in[map[i]];
  }
}

// apply_permutation(m, p, mode) (src/reorder.cpp:44-61) with a DEVICE map
// (map[new] = old): row i of the result is old row map[i]; in symmetric
// mode columns become inv[col] and each row is re-sorted by column (the
// reference's canonicalize; a bijection creates no duplicates).
spmvk_csr* permute_csr(const spmvk_csr* a, const uint32_t* d_map, bool symmetric,
                       cudaStream_t s) {
  auto b = std::make_unique<spmvk_csr>();
  b->rows = a->rows;
  b->cols = a->cols;
  b->nnz = a->nnz;
  b->val_prec = a->val_prec;
  b->row_ptr.alloc(a->rows + 1);
  b->col.alloc(a->nnz);
  b->val.alloc(a->nnz * static_cast<uint64_t>(a->val_prec));
  if (a->rows == 0) {
    SPMVK_CUDA(cudaMemsetAsync(b->row_ptr.p, 0, 4, s));
    SPMVK_CUDA(cudaStreamSynchronize(s));
    return b.release();
  }
  DevBuf<uint32_t> inv(symmetric ? a->rows : 0);
  if (symmetric) {
    invert_map<<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(a->rows, d_map, inv.p);
    SPMVK_LAUNCH("invert_map");
  }
  DevBuf<uint64_t> off(a->rows);
  const unsigned grid = persistent_grid((a->rows + 255) / 256, 8);
  permuted_lengths<<<grid, 256, 0, s>>>(a->rows, d_map, a->row_ptr.p, off.p);
  SPMVK_LAUNCH("permuted_lengths");
  exclusive_scan_u64(off.p, a->rows, s);
  const unsigned wgrid = persistent_grid((a->rows + 255) / 256, 8);  // a warp per 32 rows
  // symmetric: copy into scratch, then segmented-sort into b
  DevBuf<uint32_t> col_t(symmetric ? a->nnz : 0);
  DevBuf<unsigned char> val_t(symmetric ? a->nnz * static_cast<uint64_t>(a->val_prec) : 0);
  uint32_t* col_dst = symmetric ? col_t.p : b->col.p;
  unsigned char* val_dst = symmetric ? val_t.p : b->val.p;
  auto run = [&](auto tag) {
    using V = decltype(tag);
    TmpBuf<uint32_t> hb((a->rows + 31) / 32, s);
    TmpBuf<unsigned> nhb(1, s);
    SPMVK_CUDA(cudaMemsetAsync(nhb.p, 0, sizeof(unsigned), s));
    permuted_copy<V><<<wgrid, 256, 0, s>>>(
        a->rows, a->nnz, d_map, a->row_ptr.p, a->col.p, reinterpret_cast<const V*>(a->val.p),
        off.p, b->row_ptr.p, col_dst, reinterpret_cast<V*>(val_dst),
        symmetric ? inv.p : nullptr, hb.p, nhb.p);
    SPMVK_LAUNCH("permuted_copy");
    permuted_copy_rows<V><<<sm_count() * 8, 256, 0, s>>>(
        a->rows, d_map, a->row_ptr.p, a->col.p, reinterpret_cast<const V*>(a->val.p), off.p,
        col_dst, reinterpret_cast<V*>(val_dst), symmetric ? inv.p : nullptr, hb.p, nhb.p);
    SPMVK_LAUNCH("permuted_copy_rows");
    if (!symmetric || a->nnz == 0) return;
    if (a->nnz > 0x7fffffffull) fail(SPMVK_ERANGE, "apply_permutation: nnz exceeds 2^31 - 1");
    size_t tmp_bytes = 0;
    const int nnz = static_cast<int>(a->nnz), rows = static_cast<int>(a->rows);
    SPMVK_CUDA(cub::DeviceSegmentedSort::SortPairs(
        nullptr, tmp_bytes, col_t.p, b->col.p, reinterpret_cast<const V*>(val_t.p),
        reinterpret_cast<V*>(b->val.p), nnz, rows, b->row_ptr.p, b->row_ptr.p + 1, s));
    DevBuf<unsigned char> tmp(tmp_bytes);
    SPMVK_CUDA(cub::DeviceSegmentedSort::SortPairs(
        tmp.p, tmp_bytes, col_t.p, b->col.p, reinterpret_cast<const V*>(val_t.p),
        reinterpret_cast<V*>(b->val.p), nnz, rows, b->row_ptr.p, b->row_ptr.p + 1, s));
    SPMVK_CUDA(cudaStreamSynchronize(s));  // tmp / scratch die with this scope
  };
  if (a->val_prec == SPMVK_F64) run(double{});
  else run(float{});
  SPMVK_CUDA(cudaStreamSynchronize(s));
  return b.release();
}

void check_bijection(const uint32_t* map, uint64_t n) {  // Permutation ctor (reorder.cpp:12-21)
  std::vector<char> seen(n, 0);
  for (uint64_t i = 0; i < n; ++i) {
    if (map[i] >= n || seen[map[i]])
      fail(SPMVK_EINVAL, "permutation is not a bijection on 0.." + std::to_string(n ? n - 1 : 0));
    seen[map[i]] = 1;
  }
}

void descending_map(const spmvk_csr* a, uint32_t* d_map, cudaStream_t s) {
  unsigned mx = 0, mn = 0;
  row_length_range(a, 0, a->rows, &mx, &mn, s);
  DevBuf<uint32_t> keys(a->rows), keys2(a->rows), ids(a->rows);
  sort_keys<<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(a->rows, mx, a->row_ptr.p,
                                                                       keys.p, ids.p);
  SPMVK_LAUNCH("sort_keys");
  int end_bit = 1;
  while (end_bit < 32 && (1ull << end_bit) <= mx) ++end_bit;
  size_t tmp_bytes = 0;
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, ids.p, d_map,
                                             static_cast<int>(a->rows), 0, end_bit, s));
  DevBuf<unsigned char> tmp(tmp_bytes);
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys2.p, ids.p, d_map,
                                             static_cast<int>(a->rows), 0, end_bit, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_csr_descending_permutation(const spmvk_csr* a, uint32_t* map) {
  return guarded([&] {
    require_device();
    if (!a || (!map && a->rows)) fail(SPMVK_EINVAL, "null argument");
    if (a->rows == 0) return;
    DevBuf<uint32_t> d(a->rows);
    descending_map(a, d.p, nullptr);
    SPMVK_CUDA(cudaMemcpy(map, d.p, 4 * a->rows, cudaMemcpyDeviceToHost));
  });
}

int spmvk_csr_permute_rows_descending(const spmvk_csr* a, void* stream, spmvk_csr** out,
                                      uint32_t* map) {
  return guarded([&] {
    require_device();
    if (!a || !out) fail(SPMVK_EINVAL, "null argument");
    cudaStream_t s = as_stream(stream);
    DevBuf<uint32_t> d_map(a->rows);
    if (a->rows) descending_map(a, d_map.p, s);
    spmvk_csr* b = permute_csr(a, d_map.p, false, s);
    if (map && a->rows) {
      const cudaError_t e = cudaMemcpy(map, d_map.p, 4 * a->rows, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        spmvk_csr_destroy(b);
        SPMVK_CUDA(e);
      }
    }
    *out = b;
  });
}

int spmvk_csr_permute(const spmvk_csr* a, const uint32_t* map, uint64_t n, int symmetric,
                      void* stream, spmvk_csr** out) {
  return guarded([&] {
    require_device();
    if (!a || !out || (!map && n)) fail(SPMVK_EINVAL, "null argument");
    check_bijection(map, n);
    if (n != a->rows)
      fail(SPMVK_EINVAL, "apply_permutation: permutation length " + std::to_string(n) +
                             " does not match " + std::to_string(a->rows) + " rows");
    if (symmetric && a->rows != a->cols)
      fail(SPMVK_EINVAL, "apply_permutation: symmetric mode needs a square matrix");
    cudaStream_t s = as_stream(stream);
    DevBuf<uint32_t> d_map(n);
    if (n) SPMVK_CUDA(cudaMemcpyAsync(d_map.p, map, 4 * n, cudaMemcpyHostToDevice, s));
    *out = permute_csr(a, d_map.p, symmetric != 0, s);
  });
}

int spmvk_permute_vector_f64(const uint32_t* map_dev, uint64_t n, const double* in, double* out,
                             int inverse, void* stream) {
  return guarded([&] {
    if (n && (!map_dev || !in || !out)) fail(SPMVK_EINVAL, "null argument");
    if (!n) return;
    permute_vector<double><<<persistent_grid((n + 255) / 256, 8), 256, 0, as_stream(stream)>>>(
        n, map_dev, in, out, inverse);
    SPMVK_LAUNCH("permute_vector");
  });
}

int spmvk_permute_vector_f32(const uint32_t* map_dev, uint64_t n, const float* in, float* out,
                             int inverse, void* stream) {
  return guarded([&] {
    if (n && (!map_dev || !in || !out)) fail(SPMVK_EINVAL, "null argument");
    if (!n) return;
    permute_vector<float><<<persistent_grid((n + 255) / 256, 8), 256, 0, as_stream(stream)>>>(
        n, map_dev, in, out, inverse);
    SPMVK_LAUNCH("permute_vector");
  });
}

}  // extern "C"
