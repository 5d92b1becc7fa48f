// Hybrid ELL + COO (Bell & Garland) on the device: K3 width choice + build,
// K4/K5 fused SpMV.
//
// Reference: hybrid_split_cost / choose_ell_width (spmvkit/ellpack.hpp:143-166),
// build_hybrid (:168-203), spmv_ellpack (:110-123), spmv_coo (:132-141),
// spmv_hybrid (:205-210).  ELL is slot-major (slot*N + row), pads (0, col 0);
// COO holds each row's entries past the first K1, sorted by (row, col).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"
#include "kernels.cuh"
#include "rgcsr_spmv.cuh"  // long_row_walk, LongList, long_items_done
#include "tma.cuh"

namespace spmvk {
namespace {

constexpr int kRowsPerTile = 256;  // rows per SpMV tile (= CTA size)
constexpr int kCooTile = 1024;     // COO entries staged in smem per pass

// ------------------------------------------------------------ K3a: histogram
// hist[len] += 1 over all rows.  Warp-aggregated (match_any) into a shared
// histogram, then one global atomic per non-empty bin per CTA.
__global__ void len_hist_smem(uint64_t rows, const uint32_t* __restrict__ rp, uint32_t nbins,
                              unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t sh[];
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (uint64_t r0 = blockIdx.x * (uint64_t)blockDim.x; r0 < rows;
       r0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = r0 + threadIdx.x;
    const bool live = r < rows;
    const uint32_t len = live ? rp[r + 1] - rp[r] : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, len);
    if (live && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&sh[len], __popc(peers));
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

__global__ void len_hist_global(uint64_t rows, const uint32_t* __restrict__ rp,
                                unsigned long long* __restrict__ hist) {
  for (uint64_t r0 = blockIdx.x * (uint64_t)blockDim.x; r0 < rows;
       r0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = r0 + threadIdx.x;
    const bool live = r < rows;
    const uint32_t len = live ? rp[r + 1] - rp[r] : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, len);
    if (live && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
      atomicAdd(&hist[len], (unsigned long long)__popc(peers));
  }
}

// argmin_k 2*N*k + 3*sum_{len>k}(len-k), smallest k on ties, from the
// histogram: with C(k) = #rows longer than k and S(k) = their total length,
// overflow(k) = S(k) - k*C(k); both are suffix sums.  Exact integers.
uint64_t width_from_hist(const std::vector<unsigned long long>& hist, uint64_t rows) {
  const uint64_t max_len = hist.empty() ? 0 : hist.size() - 1;
  std::vector<uint64_t> C(max_len + 2, 0), S(max_len + 2, 0);
  for (uint64_t k = max_len + 1; k-- > 0;) {
    // rows with len > k: those with len == k+1 plus len > k+1
    const uint64_t cnt = k + 1 <= max_len ? hist[k + 1] : 0;
    C[k] = C[k + 1] + cnt;
    S[k] = S[k + 1] + cnt * (k + 1);
  }
  uint64_t best_k = 0, best = 3 * S[0];
  for (uint64_t k = 1; k <= max_len; ++k) {
    const uint64_t cost = 2 * rows * k + 3 * (S[k] - k * C[k]);
    if (cost < best) {
      best = cost;
      best_k = k;
    }
  }
  return best_k;
}

uint64_t choose_width_device(const spmvk_csr* a, uint64_t max_len, cudaStream_t s) {
  if (a->rows == 0) return 0;
  DevBuf<unsigned long long> hist(max_len + 1);
  SPMVK_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(unsigned long long) * (max_len + 1), s));
  const unsigned grid = persistent_grid((a->rows + 255) / 256, 4);
  if (max_len + 1 <= 12288) {
    len_hist_smem<<<grid, 256, sizeof(uint32_t) * (max_len + 1), s>>>(
        a->rows, a->row_ptr.p, static_cast<uint32_t>(max_len + 1), hist.p);
  } else {
    len_hist_global<<<grid, 256, 0, s>>>(a->rows, a->row_ptr.p, hist.p);
  }
  SPMVK_LAUNCH("len_hist");
  std::vector<unsigned long long> h(max_len + 1);
  SPMVK_CUDA(cudaMemcpyAsync(h.data(), hist.p, sizeof(unsigned long long) * (max_len + 1),
                             cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  return width_from_hist(h, a->rows);
}

// ------------------------------------------------------------ K3b: build
// ELL: thread per row writes its K1 slots (coalesced across rows for each
// slot); COO: overflow counts for the offset scan.
template <class T, class V>
__global__ void hybrid_ell_fill(uint64_t rows, uint32_t k1, const uint32_t* __restrict__ rp,
                                const uint32_t* __restrict__ col, const V* __restrict__ val,
                                T* __restrict__ ev, uint32_t* __restrict__ ec,
                                uint64_t* __restrict__ overflow) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rp[r], len = rp[r + 1] - b;
    for (uint32_t j = 0; j < k1; ++j) {
      const uint64_t idx = (uint64_t)j * rows + r;
      if (j < len) {
        ev[idx] = static_cast<T>(val[b + j]);
        ec[idx] = col[b + j];
      } else {
        ev[idx] = T(0);
        ec[idx] = 0;
      }
    }
    overflow[r] = len > k1 ? len - k1 : 0;
  }
}

// ELL fill with TMA bulk copies (the K1 scatter's design, rgcsr.cu): a warp
// per 32-row block; the block's CSR entries (values + columns, rounded out to
// 16 B) arrive in one of the warp's two shared-memory stages by two
// cp.async.bulk copies on an mbarrier, the NEXT block in flight while this
// one's K1 slots are written (slot j of the 32 rows is 32 contiguous entries
// at j N + r0: coalesced), pads (0, column 0) in the same pass.  Blocks whose
// entries do not fit a stage (or a partial last block) read CSR directly.
constexpr uint32_t kEllStage = 1024;

template <class T, class V>
__global__ void __launch_bounds__(128) hybrid_ell_fill_bulk(
    uint64_t rows, uint32_t k1, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
    const V* __restrict__ val, T* __restrict__ ev, uint32_t* __restrict__ ec,
    uint64_t* __restrict__ overflow) {
  constexpr uint32_t SV = (kEllStage + 4) * sizeof(V), SC = (kEllStage + 4) * 4;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = sm + (size_t)warp * 2 * (SV + SC);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)4 * 2 * (SV + SC)) + warp * 2;
  const uint64_t blocks = (rows + 31) / 32;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t first = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto fits = [&](uint64_t blk) {
    if (blk >= blocks || blk * 32 + 32 > rows) return false;
    return rp[blk * 32 + 32] - rp[blk * 32] <= kEllStage;
  };
  auto issue = [&](uint64_t blk, int b) {
    const uint32_t e0 = rp[blk * 32], e1 = rp[blk * 32 + 32];
    const uint64_t v0 = (uint64_t)e0 * sizeof(V) & ~15ull;
    const uint64_t v1 = ((uint64_t)e1 * sizeof(V) + 15) & ~15ull;
    const uint64_t c0 = (uint64_t)e0 * 4 & ~15ull, c1 = ((uint64_t)e1 * 4 + 15) & ~15ull;
    unsigned char* sb = wbase + b * (SV + SC);
    mbar_arrive_expect_tx(&bar[b], (uint32_t)(v1 - v0 + c1 - c0));
    bulk_g2s(sb, reinterpret_cast<const unsigned char*>(val) + v0, (uint32_t)(v1 - v0), &bar[b]);
    bulk_g2s(sb + SV, reinterpret_cast<const unsigned char*>(col) + c0, (uint32_t)(c1 - c0),
             &bar[b]);
  };
  uint32_t phase[2] = {0, 0};
  bool staged = fits(first);
  if (staged && lane == 0) issue(first, 0);
  int b = 0;
  for (uint64_t blk = first; blk < blocks; blk += warps, b ^= 1) {
    const uint64_t bn = blk + warps;
    const bool staged_n = fits(bn);
    if (staged_n && lane == 0) {
      fence_proxy_async_smem();
      issue(bn, b ^ 1);
    }
    const uint64_t r = blk * 32 + lane;
    const bool live = r < rows;
    const uint32_t start = live ? rp[r] : 0u, len = live ? rp[r + 1] - start : 0u;
    if (live) overflow[r] = len > k1 ? len - k1 : 0;
    if (staged) {
      mbar_wait(&bar[b], phase[b]);
      phase[b] ^= 1;
      const uint32_t e0 = rp[blk * 32];
      const V* sv = reinterpret_cast<const V*>(wbase + b * (SV + SC)) +
                    ((uint64_t)e0 * sizeof(V) & 15) / sizeof(V);
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(wbase + b * (SV + SC) + SV) +
                           ((uint64_t)e0 * 4 & 15) / 4;
      const uint32_t off = start - e0;
      for (uint32_t j = 0; j < k1; ++j) {
        const uint64_t idx = (uint64_t)j * rows + r;
        ev[idx] = j < len ? static_cast<T>(sv[off + j]) : T(0);
        ec[idx] = j < len ? sc[off + j] : 0u;
      }
    } else if (live) {
      for (uint32_t j = 0; j < k1; ++j) {
        const uint64_t idx = (uint64_t)j * rows + r;
        ev[idx] = j < len ? static_cast<T>(val[start + j]) : T(0);
        ec[idx] = j < len ? col[start + j] : 0u;
      }
    }
    __syncwarp();
    staged = staged_n;
  }
}

// COO: one warp per row with overflow copies the row's tail (coalesced).
// Blocks of 32 rows with more COO entries than this are left to
// hybrid_coo_fill_rows (a warp per row, spread over the grid): one warp
// walking 32 long tails in sequence would be the critical path (a
// descending-sorted power-law puts its ~4,000-entry tails together).
constexpr uint64_t kCooBlockMax = 32 * 64;

// The rows of the heavy blocks hybrid_coo_fill listed (see kCooBlockMax): a
// warp per row, spread over the grid.
template <class T, class V>
__global__ void hybrid_coo_fill_rows(uint64_t rows, uint32_t k1, const uint32_t* __restrict__ rp,
                                     const uint32_t* __restrict__ col, const V* __restrict__ val,
                                     const uint64_t* __restrict__ off, uint32_t* __restrict__ cr,
                                     uint32_t* __restrict__ cc, T* __restrict__ cv,
                                     const uint32_t* __restrict__ heavy_blocks,
                                     const unsigned* __restrict__ n_heavy_blocks) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t n = (uint64_t)*n_heavy_blocks * 32;
  for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n;
       w += warps) {
    const uint64_t r = (uint64_t)heavy_blocks[w / 32] * 32 + (w % 32);
    if (r >= rows) continue;
    const uint32_t b = rp[r], len = rp[r + 1] - b;
    if (len <= k1) continue;
    const uint64_t o = off[r];
    for (uint32_t i = lane; i < len - k1; i += 32) {
      cr[o + i] = (uint32_t)r;
      cc[o + i] = col[b + k1 + i];
      cv[o + i] = static_cast<T>(val[b + k1 + i]);
    }
  }
}

template <class T, class V>
__global__ void hybrid_coo_fill(uint64_t rows, uint32_t k1, const uint32_t* __restrict__ rp,
                                const uint32_t* __restrict__ col, const V* __restrict__ val,
                                const uint64_t* __restrict__ off, uint32_t* __restrict__ cr,
                                uint32_t* __restrict__ cc, T* __restrict__ cv,
                                uint32_t* __restrict__ heavy_blocks,
                                unsigned* __restrict__ n_heavy_blocks) {
  // A warp per 32-row block: the block's COO entries are one contiguous output
  // range [off[r0], off[r0 + 32]); the warp writes it 32 entries at a time
  // (coalesced), each lane finding its entry's row among the block's 32 by a
  // shuffle binary search over the rows' output offsets -- instead of a warp
  // per row, which left most lanes idle on short COO tails.
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t blocks = (rows + 31) / 32;
  for (uint64_t blk = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); blk < blocks;
       blk += warps) {
    const uint64_t r = blk * 32 + lane;
    const bool live = r < rows;
    const uint64_t o = live ? off[r] : 0;  // this row's first output entry
    const uint32_t b = live ? rp[r] : 0;
    const uint64_t last = min(rows, blk * 32 + 32) - 1;
    const uint64_t o0 = __shfl_sync(0xffffffffu, o, 0);
    const uint64_t o1 = (last + 1 == rows) ? off[last] + (rp[last + 1] - rp[last] > k1 ?
                                                          rp[last + 1] - rp[last] - k1 : 0)
                                           : off[last + 1];
    if (o1 - o0 > kCooBlockMax) {  // heavy block: listed for hybrid_coo_fill_rows
      if (lane == 0) heavy_blocks[atomicAdd(n_heavy_blocks, 1u)] = (uint32_t)blk;
      continue;
    }
    for (uint64_t e0 = o0; e0 < o1; e0 += 32) {
      const uint64_t e = e0 + lane;
      // the row of entry e: the largest lane q with off[q] <= e (rows with no
      // COO entries share their successor's offset and are never chosen past it)
      int q = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint64_t oq = __shfl_sync(0xffffffffu, o, q + step);
        const bool ok = (uint64_t)(blk * 32 + q + step) < rows && oq <= e;
        if (ok) q += step;
      }
      const uint64_t oq = __shfl_sync(0xffffffffu, o, q);
      const uint32_t bq = __shfl_sync(0xffffffffu, b, q);
      if (e < o1) {
        const uint64_t src = (uint64_t)bq + k1 + (e - oq);
        cr[e] = (uint32_t)(blk * 32 + q);
        cc[e] = col[src];
        cv[e] = static_cast<T>(val[src]);
      }
    }
  }
}

// coo_row_ptr[r] = off[r] (exclusive scan of the rows' COO counts), [rows] = total.
__global__ void narrow_offsets(uint64_t rows, const uint64_t* __restrict__ off, uint64_t total,
                               uint32_t* __restrict__ out) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    out[r] = static_cast<uint32_t>(r < rows ? off[r] : total);
}

// tile_ptr[t] = first COO entry whose row >= t * kRowsPerTile (lower bound).
__global__ void coo_tile_bounds(uint64_t ntiles, uint64_t rows, uint64_t n,
                                const uint32_t* __restrict__ cr, uint32_t* __restrict__ tp) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = min(t * kRowsPerTile, rows);
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (cr[mid] < row) lo = mid + 1; else hi = mid;
    }
    tp[t] = (uint32_t)lo;
  }
}

// FillReport's ELL nnz (fill.hpp:61-65 -> ell_nnz, ellpack.hpp:55-78): the
// reference recounts real slots from the layout -- the first non-increasing
// column starts the pad region, and a lone stored zero at column 0 counts as
// empty -- so a stored zero can change fill_report.
// The same count from the CSR the ELL part was filled from, without reading
// the ELL arrays back (27-pt fp64: 110 us -> a pass over row_ptr): real
// entries fill slots 0..n-1 (n = min(len, K1)) with strictly increasing
// columns and pads carry (0, column 0), so the recount above stops exactly at
// n -- except a row whose only ELL entry is a stored zero (after the cast to
// the ELL precision) at column 0, which it counts as empty.
// The same pass yields the COO part's largest column (out[1], for
// spmv_coo's bounds check): a row's COO entries are its columns past K1, in
// increasing order, so the row's last column.
template <class T, class V>
__global__ void ell_nnz_from_csr(uint64_t rows, uint32_t k1, const uint32_t* __restrict__ rp,
                                 const uint32_t* __restrict__ col, const V* __restrict__ val,
                                 unsigned long long* out) {
  unsigned long long total = 0;
  uint32_t mc = 0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rp[r], len = rp[r + 1] - b;
    uint32_t n = min(len, k1);
    if (n == 1 && col[b] == 0 && static_cast<T>(val[b]) == T(0)) n = 0;
    total += n;
    if (len > k1) mc = max(mc, col[b + len - 1]);
  }
  for (int o = 16; o; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
  mc = __reduce_max_sync(0xffffffffu, mc);
  if ((threadIdx.x & 31) == 0) {
    if (total) atomicAdd(out, total);
    if (mc) atomicMax(out + 1, (unsigned long long)mc);
  }
}

// ------------------------------------------------------------ to_triplets
// ellpack.hpp:219-240: ELL rows through the ell_row_length recount, then the
// COO overflow; per row the ELL columns precede the COO ones, so the result is
// already canonical (the reference re-sorts).
template <class T>
__device__ __forceinline__ uint32_t ell_len_of(uint64_t rows, uint32_t k1, const T* ev,
                                               const uint32_t* ec, uint64_t r) {
  uint32_t len = 0, prev = 0;
  for (uint32_t slot = 0; slot < k1; ++slot) {
    const uint64_t idx = (uint64_t)slot * rows + r;
    const uint32_t c = ec[idx];
    if (slot > 0 && c <= prev) break;
    if (slot == 0 && c == 0 && ev[idx] == T(0)) {
      const bool real_successor = k1 > 1 && ec[rows + r] > 0;
      if (!real_successor) break;
    }
    ++len;
    prev = c;
  }
  return len;
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <class T>
__global__ void hybrid_row_counts(uint64_t rows, uint32_t k1, const T* __restrict__ ev,
                                  const uint32_t* __restrict__ ec, uint64_t coo,
                                  const uint32_t* __restrict__ cr, uint64_t* __restrict__ cnt) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lb = lower_bound_u32(cr, coo, (uint32_t)r);
    const uint64_t ub = lower_bound_u32(cr, coo, (uint32_t)r + 1);
    cnt[r] = ell_len_of(rows, k1, ev, ec, r) + (ub - lb);
  }
}

template <class T>
__global__ void hybrid_gather_rows(uint64_t rows, uint32_t k1, uint64_t nnz,
                                   const T* __restrict__ ev, const uint32_t* __restrict__ ec,
                                   uint64_t coo, const uint32_t* __restrict__ cr,
                                   const uint32_t* __restrict__ cc, const T* __restrict__ cv,
                                   const uint64_t* __restrict__ off, uint32_t* __restrict__ rp,
                                   uint32_t* __restrict__ col, double* __restrict__ val) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t o = off[r];
    rp[r] = (uint32_t)o;
    if (r + 1 == rows) rp[rows] = (uint32_t)nnz;
    const uint32_t n = ell_len_of(rows, k1, ev, ec, r);
    for (uint32_t j = 0; j < n; ++j, ++o) {
      col[o] = ec[(uint64_t)j * rows + r];
      val[o] = static_cast<double>(ev[(uint64_t)j * rows + r]);
    }
    const uint64_t lb = lower_bound_u32(cr, coo, (uint32_t)r);
    for (uint64_t i = lb; i < coo && cr[i] == r; ++i, ++o) {
      col[o] = cc[i];
      val[o] = static_cast<double>(cv[i]);
    }
  }
}

template <class T>
spmvk_csr* hybrid_to_csr(const spmvk_hybrid* h, cudaStream_t s) {
  const unsigned grid = persistent_grid((h->rows + 255) / 256, 8);
  DevBuf<uint64_t> off(h->rows);
  const T* ev = reinterpret_cast<const T*>(h->ell_values.p);
  const T* cv = reinterpret_cast<const T*>(h->coo_values.p);
  uint64_t total = 0;
  if (h->rows) {
    hybrid_row_counts<T><<<grid, 256, 0, s>>>(h->rows, static_cast<uint32_t>(h->k1), ev,
                                              h->ell_columns.p, h->coo, h->coo_rows.p, off.p);
    SPMVK_LAUNCH("hybrid_row_counts");
    total = exclusive_scan_u64(off.p, h->rows, s);
  }
  std::unique_ptr<spmvk_csr> c(new_csr(h->rows, h->cols, total, SPMVK_F64));
  if (h->rows) {
    hybrid_gather_rows<T><<<grid, 256, 0, s>>>(h->rows, static_cast<uint32_t>(h->k1), total, ev,
                                               h->ell_columns.p, h->coo, h->coo_rows.p,
                                               h->coo_columns.p, cv, off.p, c->row_ptr.p,
                                               c->col.p, reinterpret_cast<double*>(c->val.p));
    SPMVK_LAUNCH("hybrid_gather_rows");
  } else {
    SPMVK_CUDA(cudaMemsetAsync(c->row_ptr.p, 0, 4, s));
  }
  SPMVK_CUDA(cudaStreamSynchronize(s));
  return c.release();
}

// ------------------------------------------------------------ K4/K5: SpMV
// One CTA-tile of 256 rows: (1) thread per row walks its K1 ELL slots (pads
// included, as spmv_ellpack does); (2) the tile's COO range is staged in
// shared memory in chunks, products v*x[c] computed in parallel, and each row
// then adds its own products sequentially in column order.  Per row this is
// exactly the reference's sequence of roundings: ELL slots 0..K1-1, then the
// row's COO entries in array order -> y bitwise equal to spmv_hybrid.
template <class T, int U, bool kAccum = false>
__global__ void __launch_bounds__(kRowsPerTile) hybrid_spmv_kernel(
    uint32_t rows, uint32_t k1, const T* __restrict__ ev, const uint32_t* __restrict__ ec,
    const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ cr,
    const uint32_t* __restrict__ cc, const T* __restrict__ cv, const T* __restrict__ x,
    T* __restrict__ y, const uint32_t* __restrict__ /*crp: staged only*/) {
  __shared__ T prod[kCooTile];
  __shared__ uint32_t prow[kCooTile];
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint32_t ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t r = tile * kRowsPerTile + threadIdx.x;
    const bool live = r < rows;
    T acc = T(0);
    if (kAccum && live) acc = y[r];  // spmv_coo: y += COO x (ellpack.hpp:132-141)
    if (live) {
      uint32_t j = 0;
      for (; j + U <= k1; j += U) {
        uint32_t c[U];
        T v[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const size_t idx = (size_t)(j + u) * rows + r;
          c[u] = ld_stream(ec + idx, pf);
          v[u] = ld_stream(ev + idx, pf);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = ld_x(x + c[u], pl);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
      }
      if (j < k1) {  // tail of < U slots: one predicated batch, loads in flight together
        uint32_t c[U - 1];
        T v[U - 1], xv[U - 1];
#pragma unroll
        for (int u = 0; u < U - 1; ++u) {
          c[u] = 0;
          v[u] = T(0);
          if (j + u < k1) {
            const size_t idx = (size_t)(j + u) * rows + r;
            c[u] = ld_stream(ec + idx, pf);
            v[u] = ld_stream(ev + idx, pf);
          }
        }
#pragma unroll
        for (int u = 0; u < U - 1; ++u) xv[u] = j + u < k1 ? ld_x(x + c[u], pl) : T(0);
#pragma unroll
        for (int u = 0; u < U - 1; ++u)
          if (j + u < k1) acc = add_rn(acc, mul_rn(v[u], xv[u]));
      }
    }
    if (tile_ptr) {
      const uint32_t c0 = tile_ptr[tile], c1 = tile_ptr[tile + 1];
      for (uint32_t t0 = c0; t0 < c1; t0 += kCooTile) {
        const uint32_t n = min((uint32_t)kCooTile, c1 - t0);
        for (uint32_t i = threadIdx.x; i < n; i += kRowsPerTile) {
          prow[i] = ld_stream(cr + t0 + i, pf);
          prod[i] = mul_rn(ld_stream(cv + t0 + i, pf), ld_x(x + ld_stream(cc + t0 + i, pf), pl));
        }
        __syncthreads();
        if (live) {
          uint32_t lo = 0, hi = n;  // first staged entry with row >= r
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (prow[mid] < r) lo = mid + 1; else hi = mid;
          }
          uint32_t end = lo, top = n;  // first staged entry with row > r
          while (end < top) {
            const uint32_t mid = (end + top) >> 1;
            if (prow[mid] <= r) end = mid + 1; else top = mid;
          }
          uint32_t i = lo;
          for (; i + 8 <= end; i += 8) {  // 8 independent LDS in flight, adds in order
            T p[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) p[u] = prod[i + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = add_rn(acc, p[u]);
          }
          for (; i < end; ++i) acc = add_rn(acc, prod[i]);
        }
        __syncthreads();
      }
    }
    if (live) y[r] = acc;
  }
}

// The tile's COO range [tile_ptr[tile], tile_ptr[tile+1]) staged through
// shared memory (same scheme as hybrid_spmv_kernel): products in parallel,
// then each live row adds its own products in array order.
// Tiles with more than kWalkCoo COO entries: each thread adds its own row's
// run [crp[r], crp[r+1]) in array order (4 loads in flight, then gathers),
// so the tile's heavy rows progress in parallel instead of one staged chunk
// at a time (a reordered power-law matrix puts ~500k COO entries of its 256
// longest rows in one tile).  Same rounding sequence -> y bitwise.
constexpr uint32_t kWalkCoo = 16 * kCooTile;
// Runs longer than this in walked tiles go to hybrid_heavy_rows (the walk
// skips them): one thread would need run/4 dependent round trips.
constexpr uint32_t kHeavyRun = 256;

template <class T, bool kHint = false>
__device__ __forceinline__ T coo_row_walk(uint32_t r, bool live, T acc,
                                          const uint32_t* __restrict__ crp,
                                          const uint32_t* __restrict__ cc,
                                          const T* __restrict__ cv, const T* __restrict__ x) {
  if (!live) return acc;
  const Ldr<kHint> ld;
  const uint32_t cb = crp[r], ce = crp[r + 1];
  if (ce - cb > kHeavyRun) return acc;  // added later by hybrid_heavy_rows
  constexpr int U = 4;  // fits the 32-register budget of the 8-CTA/SM kernels
  for (uint32_t k = cb; k < ce; k += U) {
    uint32_t c[U];
    T v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = k + u < ce ? ld.s(cc + k + u) : 0u;
      v[u] = k + u < ce ? ld.s(cv + k + u) : T(0);
    }
    __syncwarp(__activemask());  // scheduling fence: loads before gathers
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = k + u < ce ? ld.x(x + c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < ce) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  return acc;
}

template <class T, bool kHint = false>
__device__ __forceinline__ T coo_tile_accumulate(uint32_t tile, uint32_t r, bool live, T acc,
                                                 const uint32_t* __restrict__ tile_ptr,
                                                 const uint32_t* __restrict__ cr,
                                                 const uint32_t* __restrict__ cc,
                                                 const T* __restrict__ cv,
                                                 const T* __restrict__ x) {
  __shared__ T prod[kCooTile];
  __shared__ uint32_t prow[kCooTile];
  const uint32_t c0 = tile_ptr[tile], c1 = tile_ptr[tile + 1];
  const Ldr<kHint> ld;
  for (uint32_t t0 = c0; t0 < c1; t0 += kCooTile) {
    const uint32_t n = min((uint32_t)kCooTile, c1 - t0);
    for (uint32_t i = threadIdx.x; i < n; i += kRowsPerTile) {
      prow[i] = ld.s(cr + t0 + i);
      prod[i] = mul_rn(ld.s(cv + t0 + i), ld.x(x + ld.s(cc + t0 + i)));
    }
    __syncthreads();
    if (live) {
      uint32_t lo = 0, hi = n;  // first staged entry with row >= r
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (prow[mid] < r) lo = mid + 1; else hi = mid;
      }
      uint32_t end = lo, top = n;  // first staged entry with row > r
      while (end < top) {
        const uint32_t mid = (end + top) >> 1;
        if (prow[mid] <= r) end = mid + 1; else top = mid;
      }
      uint32_t i = lo;
      for (; i + 8 <= end; i += 8) {
        T p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = prod[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = add_rn(acc, p[u]);
      }
      for (; i < end; ++i) acc = add_rn(acc, prod[i]);
    }
    __syncthreads();
  }
  return acc;
}

// The COO tails of the heavy rows (see kHeavyRun), after the main kernel has
// stored each row's ELL part (or, for spmv_coo, left y untouched): a warp per
// row loads 256 consecutive COO entries per round (8 per lane, coalesced),
// forms the products in parallel, stages them in shared memory, and lane 0
// adds them in array order onto y[r] -- the reference's rounding sequence.
template <class T, bool kHint = false>
__global__ void __launch_bounds__(256) hybrid_heavy_rows(uint32_t n, const uint32_t* __restrict__ rows,
                                                         const uint32_t* __restrict__ crp,
                                                         const uint32_t* __restrict__ cc,
                                                         const T* __restrict__ cv,
                                                         const T* __restrict__ x,
                                                         T* __restrict__ y) {
  constexpr int K = 8, W = 32 * K;
  __shared__ T prod[8][W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Ldr<kHint> ld;
  for (uint32_t i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
    const uint32_t r = rows[i];
    const uint32_t cb = crp[r], ce = crp[r + 1];
    T acc = y[r];
    for (uint32_t k0 = cb; k0 < ce; k0 += W) {
      uint32_t c[K];
      T v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t e = k0 + lane + 32 * k;
        c[k] = e < ce ? ld.s(cc + e) : 0u;
        v[k] = e < ce ? ld.s(cv + e) : T(0);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t e = k0 + lane + 32 * k;
        if (e < ce) prod[warp][lane + 32 * k] = mul_rn(v[k], ld.x(x + c[k]));
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t m = min((uint32_t)W, ce - k0);
        uint32_t q = 0;
        for (; q + 8 <= m; q += 8) {
          T p[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) p[u] = prod[warp][q + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = add_rn(acc, p[u]);
        }
        for (; q < m; ++q) acc = add_rn(acc, prod[warp][q]);
      }
      __syncwarp();
    }
    if (lane == 0) y[r] = acc;
  }
}

// Register-lean form of hybrid_spmv_kernel (the RgCSR `lite` recipe applied
// to the ELL part): no cache-policy registers, the slot pointers advance by
// U*rows instead of recomputing 64-bit indices, and MINB resident CTAs per
// SM.  Same per-row rounding sequence (all K1 ELL slots including pads, then
// the row's COO entries in array order) -> y bitwise spmv_hybrid's.
template <class T, int U, int MINB, bool kAccum, bool kCoo, bool kFence = false,
          bool kHint = false>
__global__ void __launch_bounds__(kRowsPerTile, MINB) hybrid_spmv_lite(
    uint32_t rows, uint32_t k1, const T* __restrict__ ev, const uint32_t* __restrict__ ec,
    const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ cr,
    const uint32_t* __restrict__ cc, const T* __restrict__ cv, const T* __restrict__ x,
    T* __restrict__ y, const uint32_t* __restrict__ crp) {
  const uint32_t ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
  const size_t step = (size_t)U * rows;
  const Ldr<kHint> ld;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t r = tile * kRowsPerTile + threadIdx.x;
    const bool live = r < rows;
    T acc = T(0);
    if (kAccum && live) acc = y[r];
    if (live) {
      const T* __restrict__ vp = ev + r;
      const uint32_t* __restrict__ cp = ec + r;
      uint32_t j = 0;
      for (; j + U <= k1; j += U) {
        uint32_t c[U];
        T v[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          c[u] = ld.s(cp + (size_t)u * rows);
          v[u] = ld.s(vp + (size_t)u * rows);
        }
        if (kFence) __syncwarp(__activemask());  // slot loads ahead of the gathers
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = ld.x(x + c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
        cp += step;
        vp += step;
      }
      if (j < k1) {  // predicated last batch (< U slots)
        uint32_t c[U - 1];
        T v[U - 1], xv[U - 1];
#pragma unroll
        for (int u = 0; u < U - 1; ++u) {
          c[u] = 0;
          v[u] = T(0);
          if (j + u < k1) {
            c[u] = ld.s(cp + (size_t)u * rows);
            v[u] = ld.s(vp + (size_t)u * rows);
          }
        }
        if (kFence) __syncwarp(__activemask());
#pragma unroll
        for (int u = 0; u < U - 1; ++u) xv[u] = j + u < k1 ? ld.x(x + c[u]) : T(0);
#pragma unroll
        for (int u = 0; u < U - 1; ++u)
          if (j + u < k1) acc = add_rn(acc, mul_rn(v[u], xv[u]));
      }
    }
    if constexpr (kCoo) {
      if (crp && tile_ptr[tile + 1] - tile_ptr[tile] > kWalkCoo)  // CTA-uniform
        acc = coo_row_walk<T, kHint>(r, live, acc, crp, cc, cv, x);
      else
        acc = coo_tile_accumulate<T, kHint>(tile, r, live, acc, tile_ptr, cr, cc, cv, x);
    }
    if (live) y[r] = acc;
  }
}

// ---------------------------------------------------------------------------
// hybrid_ell_vec -- pure ELL with 128-bit slot loads: a thread owns R = 16 B /
// sizeof(T) consecutive rows (fp32: 4, fp64: 2), so slot j of its rows is one
// aligned float4 / double2 value vector and one uint4 / uint2 column vector
// (rows % R == 0 keeps every slot's row block 16-byte aligned); a warp reads
// 32 R consecutive rows of a slot -- 512 B per slot stream instead of 128 B
// (fp32), a quarter of the concurrent slot streams per byte.  Each row adds
// its K1 products in slot order (pads included) -> bitwise spmv_ellpack.
template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) hybrid_ell_vec(uint32_t rows, uint32_t k1,
                                                            const T* __restrict__ ev,
                                                            const uint32_t* __restrict__ ec,
                                                            const T* __restrict__ x,
                                                            T* __restrict__ y) {
  constexpr int R = 16 / sizeof(T);
  using Wv = VecOf<T, R>;
  using V = typename Wv::V;
  using Cv = typename Wv::C;
  const uint32_t tiles = (rows + 256 * R - 1) / (256 * R);
  const size_t vstep = rows / R;  // one slot, in vectors
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t r0 = tile * 256 * R + threadIdx.x * R;
    if (r0 >= rows) continue;
    const V* __restrict__ vp = reinterpret_cast<const V*>(ev + r0);
    const Cv* __restrict__ cp = reinterpret_cast<const Cv*>(ec + r0);
    T acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = T(0);
    uint32_t j = 0;
    for (; j + U <= k1; j += U) {
      V v[U];
      Cv c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = ld_stream_v(vp + u * vstep);
        c[u] = ld_stream_v(cp + u * vstep);
      }
      __syncwarp(__activemask());  // every slot load before the gathers
      T xv[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < R; ++i) xv[u][i] = ld_x(x + Wv::col(c[u], i));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < R; ++i) acc[i] = add_rn(acc[i], mul_rn(Wv::get(v[u], i), xv[u][i]));
      vp += U * vstep;
      cp += U * vstep;
    }
    for (; j < k1; ++j) {
      const V v = ld_stream_v(vp);
      const Cv c = ld_stream_v(cp);
#pragma unroll
      for (int i = 0; i < R; ++i)
        acc[i] = add_rn(acc[i], mul_rn(Wv::get(v, i), ld_x(x + Wv::col(c, i))));
      vp += vstep;
      cp += vstep;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) y[r0 + i] = acc[i];
  }
}

// ---------------------------------------------------------------------------
// hybrid_spmv_dyn -- Hybrid with a COO part, without block barriers.
//
// The staged-tile kernel above spends ~22 % of its stall samples at the
// __syncthreads of its COO staging and another ~7 % in the per-row binary
// search of the staged rows (ncu, power-law 8M fp64,
// profiles/r02b_ncu_hyb_pl8m_p8.md), and a row with a long COO tail holds its
// whole CTA at the barrier while one thread adds.  Here:
//  * rows are taken in dynamic 128-row slices (four 32-row sub-slices per
//    grab from a per-stream counter), thread per row for the K1 ELL slots
//    (pads included, as spmv_ellpack) in U-deep fenced batches;
//  * the COO entries of a 32-row sub-slice are one contiguous range
//    [crp[r0], crp[r0 + 32]) (COO is sorted by row): the warp stages it in
//    chunks of 32 KC entries -- coalesced column / value loads, products
//    formed in parallel into the warp's shared buffer -- and each lane adds
//    the part of ITS row's run [crp[r], crp[r + 1]) inside the chunk, in
//    array order; warp-level syncs only, no row search, and the COO row array
//    is never read;
//  * rows whose COO run exceeds kHeavyDyn (128) are work items taken first
//    (longest first) by `warps` warps per CTA: a warp walks the row's K1 ELL
//    slots and then its COO run (long_row_walk, lane 0 adding in order), so
//    the longest add chains start at once instead of forming the tail; the
//    sub-slice pass skips those rows and their COO ranges.
// Per row: ELL slots 0..K1-1, then the COO run in array order, products and
// sums rounded separately -> y bitwise spmv_hybrid's.
constexpr uint32_t kHeavyDyn = 128;
// SPMVK_HYB_HEAVY_RUN overrides the run length that makes a row a work item
// (read at build; the list and the kernel use the handle's value).
uint32_t heavy_dyn_run() {
  static const uint32_t v = [] {
    const char* e = std::getenv("SPMVK_HYB_HEAVY_RUN");
    const long n = e ? std::atol(e) : 0;
    return n > 0 ? static_cast<uint32_t>(n) : kHeavyDyn;
  }();
  return v;
}

template <class T, int U, int MINB, int KC, bool kHint>
__global__ void __launch_bounds__(256, MINB) hybrid_spmv_dyn(
    uint32_t rows, uint32_t k1, const T* __restrict__ ev, const uint32_t* __restrict__ ec,
    const uint32_t* __restrict__ crp, const uint32_t* __restrict__ cc, const T* __restrict__ cv,
    const T* __restrict__ x, T* __restrict__ y, uint32_t heavy_run, LongList hl) {
  constexpr uint32_t W = 32 * KC, kSub = 4;
  __shared__ T prod[8][W];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* __restrict__ pr = prod[warp];
  const Ldr<kHint> ld;
  if (hl.n_single && warp < hl.warps) {  // heavy rows first, longest first
    for (;;) {
      uint32_t i = 0;
      if (lane == 0) i = atomicAdd(hl.ctr, 1u);
      i = __shfl_sync(0xffffffffu, i, 0);
      if (i >= hl.n_single) break;
      const uint32_t r = hl.singles[i];
      const uint32_t cb = crp[r], ce = crp[r + 1];
      T acc = long_row_walk<T, 32, KC, kHint, 4>(k1, k1, lane, ev + r, ec + r, rows, x, pr, ld);
      acc = long_row_walk<T, 32, KC, kHint, 4>(ce - cb, ce - cb, lane, cv + cb, cc + cb, 1u, x,
                                               pr, ld, acc);
      if (lane == 0) y[r] = acc;
    }
  }
  const size_t step = (size_t)U * rows;
  auto grab = [&]() -> uint64_t {
    uint32_t q = 0;
    if (lane == 0) q = atomicAdd(hl.ctr + 2, 1u);
    q = __shfl_sync(0xffffffffu, q, 0);
    return static_cast<uint64_t>(q) * (32 * kSub);
  };
  for (uint64_t base = grab(); base < rows; base = grab()) {
    for (uint32_t sub = 0; sub < kSub; ++sub) {
      const uint64_t r0 = base + sub * 32;
      if (r0 >= rows) break;  // warp-uniform
      const uint32_t r = static_cast<uint32_t>(r0) + lane;
      const bool live = r < rows;
      const uint32_t rb = live ? crp[r] : 0u, re = live ? crp[r + 1] : 0u;
      const bool heavy = live && re - rb > heavy_run;
      const bool mine = live && !heavy;
      T acc = T(0);
      if (mine) {  // ELL: all K1 slots, pads included
        const T* __restrict__ vp = ev + r;
        const uint32_t* __restrict__ cp = ec + r;
        uint32_t j = 0;
        for (; j + U <= k1; j += U) {
          uint32_t c[U];
          T v[U], xv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            c[u] = ld.s(cp + (size_t)u * rows);
            v[u] = ld.s(vp + (size_t)u * rows);
          }
          __syncwarp(__activemask());  // slot loads ahead of the gathers
#pragma unroll
          for (int u = 0; u < U; ++u) xv[u] = ld.x(x + c[u]);
#pragma unroll
          for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
          cp += step;
          vp += step;
        }
        if (j < k1) {
          uint32_t c[U - 1];
          T v[U - 1], xv[U - 1];
#pragma unroll
          for (int u = 0; u < U - 1; ++u) {
            c[u] = j + u < k1 ? ld.s(cp + (size_t)u * rows) : 0u;
            v[u] = j + u < k1 ? ld.s(vp + (size_t)u * rows) : T(0);
          }
          __syncwarp(__activemask());
#pragma unroll
          for (int u = 0; u < U - 1; ++u) xv[u] = j + u < k1 ? ld.x(x + c[u]) : T(0);
#pragma unroll
          for (int u = 0; u < U - 1; ++u)
            if (j + u < k1) acc = add_rn(acc, mul_rn(v[u], xv[u]));
        }
      }
      // COO: the sub-slice's range minus the heavy runs, staged per chunk
      const uint32_t last = min(31u, static_cast<uint32_t>(rows - r0 - 1));
      const uint32_t wb = __shfl_sync(0xffffffffu, rb, 0);
      const uint32_t we = __shfl_sync(0xffffffffu, re, last);
      uint32_t hm = __ballot_sync(0xffffffffu, heavy);
      uint32_t cursor = wb;
      for (;;) {
        const int h = hm ? __ffs(hm) - 1 : -1;
        const uint32_t hb = __shfl_sync(0xffffffffu, rb, h < 0 ? 0 : h);
        const uint32_t he = __shfl_sync(0xffffffffu, re, h < 0 ? 0 : h);
        const uint32_t seg_end = h < 0 ? we : hb;
        for (uint32_t c0 = cursor; c0 < seg_end; c0 += W) {
          const uint32_t n = min(W, seg_end - c0);
          uint32_t c[KC];
          T v[KC];
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const uint32_t e = lane + 32 * k;
            c[k] = e < n ? ld.s(cc + c0 + e) : 0u;
            v[k] = e < n ? ld.s(cv + c0 + e) : T(0);
          }
          __syncwarp();
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const uint32_t e = lane + 32 * k;
            if (e < n) pr[e] = mul_rn(v[k], ld.x(x + c[k]));
          }
          __syncwarp();
          if (mine) {
            const uint32_t lo = max(rb, c0), hi = min(re, c0 + n);
            for (uint32_t e = lo; e < hi; ++e) acc = add_rn(acc, pr[e - c0]);
          }
          __syncwarp();
        }
        if (h < 0) break;
        cursor = he;
        hm &= hm - 1;
      }
      if (mine) y[r] = acc;
    }
  }
  long_items_done(hl);
}

// Hybrid SpMV kernel choice: spmvk_set_hybrid_kernel() or SPMVK_HYBRID_KERNEL.
// "v4": hybrid_spmv_kernel (policy-hinted loads, 4-deep, 8 CTAs / SM);
// "lite" / "lite8" / "lite8_full": hybrid_spmv_lite with 4-deep batches at
// 8 CTAs / SM, 8-deep at 5, 8-deep at 8.  All bitwise identical.
// "g6" / "g7" / "g8" / "g8r": the fenced walk with the RgCSR group walk's
// batch shapes (U = 6, 7, 8 at 5 CTAs / SM; U = 8 at 4) for pure-ELL
// matrices, where every row walks the same K1 slots like a group.
// "litefh": litef with L2 eviction hints (ELL / COO streams evict_first, x
// evict_last) in the main kernel and the heavy-row tails.
enum class HK {
  kAuto, kV4, kLite, kLite8, kLite8Full, kLiteF, kLite8F, kG6, kG7, kG8, kG8R, kLiteFH, kDyn,
  kVec
};

std::atomic<int>& hk_slot() {
  static std::atomic<int> k{[] {
    HK v = HK::kAuto;
    if (const char* e = std::getenv("SPMVK_HYBRID_KERNEL")) {
      const std::string s(e);
      v = s == "v4" ? HK::kV4 : s == "lite" ? HK::kLite : s == "lite8" ? HK::kLite8
        : s == "lite8_full" ? HK::kLite8Full : s == "litef" ? HK::kLiteF
        : s == "lite8f" ? HK::kLite8F : s == "g6" ? HK::kG6 : s == "g7" ? HK::kG7
        : s == "g8" ? HK::kG8 : s == "g8r" ? HK::kG8R : s == "litefh" ? HK::kLiteFH
        : s == "dyn" ? HK::kDyn : s == "vec" ? HK::kVec : HK::kAuto;
    }
    return static_cast<int>(v);
  }()};
  return k;
}

// Rows whose COO run exceeds thr (unordered; sorted longest first after).
__global__ void heavy_collect(uint64_t rows, const uint32_t* __restrict__ crp, uint32_t thr,
                              uint32_t* __restrict__ list, uint32_t* __restrict__ key,
                              unsigned* __restrict__ count) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t run = crp[r + 1] - crp[r];
    if (run > thr) {
      const unsigned i = atomicAdd(count, 1u);
      list[i] = static_cast<uint32_t>(r);
      key[i] = ~run;
    }
  }
}

// flag[r] = row r's COO run exceeds kHeavyRun inside a tile that walks
// (> kWalkCoo COO entries): the staged kernel's heavy-row list, compacted in
// ascending order by cub::DeviceSelect::Flagged.
__global__ void walked_heavy_flags(uint64_t rows, const uint32_t* __restrict__ tile_ptr,
                                   const uint32_t* __restrict__ crp,
                                   unsigned char* __restrict__ flag) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = r / kRowsPerTile;
    const bool walked = tile_ptr[t + 1] - tile_ptr[t] > kWalkCoo;
    flag[r] = walked && crp[r + 1] - crp[r] > kHeavyRun;
  }
}

// h->dyn_heavy: the rows of hybrid_spmv_dyn's work list, longest run first.
void collect_dyn_heavy(spmvk_hybrid* h, cudaStream_t s) {
  h->dyn_heavy_run = heavy_dyn_run();
  const uint64_t cap = h->coo / (h->dyn_heavy_run + 1) + 1;
  TmpBuf<uint32_t> list(cap, s), key(cap, s), key2(cap, s);
  TmpBuf<unsigned> cnt(1, s);
  SPMVK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), s));
  heavy_collect<<<persistent_grid((h->rows + 255) / 256, 8), 256, 0, s>>>(
      h->rows, h->coo_row_ptr.p, h->dyn_heavy_run, list.p, key.p, cnt.p);
  SPMVK_LAUNCH("heavy_collect");
  unsigned n = 0;
  SPMVK_CUDA(cudaMemcpyAsync(&n, cnt.p, sizeof(n), cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  h->n_dyn_heavy = n;
  h->dyn_heavy.alloc(n);
  if (!n) return;
  size_t tmp_bytes = 0;
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.p, key2.p, list.p,
                                             h->dyn_heavy.p, static_cast<int>(n), 0, 32, s));
  TmpBuf<unsigned char> tmp(tmp_bytes, s);
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key.p, key2.p, list.p,
                                             h->dyn_heavy.p, static_cast<int>(n), 0, 32, s));
}

template <class T, class V>
void fill(spmvk_hybrid* h, const spmvk_csr* a, cudaStream_t s, unsigned max_len) {
  const unsigned grid = persistent_grid((a->rows + 255) / 256, 8);
  TmpBuf<uint64_t> off(a->rows, s);  // per-row COO counts (stream-ordered scratch)
  // bulk-copy fill for matrices whose 32-row blocks fit a stage (rows of at
  // most 32 entries: 27-pt 405 -> 240 us); long-row matrices keep the
  // thread-per-row fill (power-law 8M 361 vs 422 us).  SPMVK_ELL_BULK=0 / 1
  // forces it off / on.
  static const int bulk_env = [] {
    const char* e = std::getenv("SPMVK_ELL_BULK");
    return e ? std::atoi(e) : -1;
  }();
  if (bulk_env > 0 || (bulk_env < 0 && max_len <= 32)) {
    auto kern = hybrid_ell_fill_bulk<T, V>;
    const size_t smem = 4 * 2 * ((kEllStage + 4) * (sizeof(V) + 4)) + 4 * 2 * 8;
    SPMVK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
    kern<<<persistent_grid((a->rows + 127) / 128, per_sm > 0 ? per_sm : 1), 128, smem, s>>>(
        a->rows, static_cast<uint32_t>(h->k1), a->row_ptr.p, a->col.p,
        reinterpret_cast<const V*>(a->val.p), reinterpret_cast<T*>(h->ell_values.p),
        h->ell_columns.p, off.p);
    SPMVK_LAUNCH("hybrid_ell_fill_bulk");
  } else {
    hybrid_ell_fill<T, V><<<grid, 256, 0, s>>>(
        a->rows, static_cast<uint32_t>(h->k1), a->row_ptr.p, a->col.p,
        reinterpret_cast<const V*>(a->val.p), reinterpret_cast<T*>(h->ell_values.p),
        h->ell_columns.p, off.p);
    SPMVK_LAUNCH("hybrid_ell_fill");
  }
  // no row longer than K1 -> no COO part: skip the scan and its readback
  const uint64_t coo = max_len <= h->k1 ? 0 : exclusive_scan_u64(off.p, a->rows, s);
  h->coo = coo;
  h->coo_rows.alloc(coo);
  h->coo_columns.alloc(coo);
  h->coo_values.alloc(coo * sizeof(T));
  if (coo) {
    {
      const uint64_t nblk = (a->rows + 31) / 32;
      TmpBuf<uint32_t> hb(nblk, s);
      TmpBuf<unsigned> nhb(1, s);
      SPMVK_CUDA(cudaMemsetAsync(nhb.p, 0, sizeof(unsigned), s));
      hybrid_coo_fill<T, V><<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(
          a->rows, static_cast<uint32_t>(h->k1), a->row_ptr.p, a->col.p,
          reinterpret_cast<const V*>(a->val.p), off.p, h->coo_rows.p, h->coo_columns.p,
          reinterpret_cast<T*>(h->coo_values.p), hb.p, nhb.p);
      SPMVK_LAUNCH("hybrid_coo_fill");
      hybrid_coo_fill_rows<T, V><<<sm_count() * 8, 256, 0, s>>>(
          a->rows, static_cast<uint32_t>(h->k1), a->row_ptr.p, a->col.p,
          reinterpret_cast<const V*>(a->val.p), off.p, h->coo_rows.p, h->coo_columns.p,
          reinterpret_cast<T*>(h->coo_values.p), hb.p, nhb.p);
      SPMVK_LAUNCH("hybrid_coo_fill_rows");
    }
    h->coo_row_ptr.alloc(a->rows + 1);
    narrow_offsets<<<persistent_grid((a->rows + 256) / 256, 8), 256, 0, s>>>(
        a->rows, off.p, coo, h->coo_row_ptr.p);
    SPMVK_LAUNCH("narrow_offsets");
    const uint64_t ntiles = (a->rows + kRowsPerTile - 1) / kRowsPerTile;
    h->tile_ptr.alloc(ntiles + 1);
    coo_tile_bounds<<<persistent_grid((ntiles + 256) / 256, 4), 256, 0, s>>>(
        ntiles, a->rows, coo, h->coo_rows.p, h->tile_ptr.p);
    SPMVK_LAUNCH("coo_tile_bounds");
    // heavy rows: runs > kHeavyRun inside tiles that walk (> kWalkCoo entries),
    // ascending: flagged on the device and compacted in order (cub select)
    {
      TmpBuf<unsigned char> flag(a->rows, s);
      walked_heavy_flags<<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(
          a->rows, h->tile_ptr.p, h->coo_row_ptr.p, flag.p);
      SPMVK_LAUNCH("walked_heavy_flags");
      TmpBuf<uint32_t> sel(a->rows, s);
      TmpBuf<int> nsel(1, s);
      cub::CountingInputIterator<uint32_t> ids(0);
      size_t tb = 0;
      SPMVK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids, flag.p, sel.p, nsel.p,
                                            static_cast<int>(a->rows), s));
      TmpBuf<unsigned char> tmp(tb, s);
      SPMVK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, ids, flag.p, sel.p, nsel.p,
                                            static_cast<int>(a->rows), s));
      int n = 0;
      SPMVK_CUDA(cudaMemcpyAsync(&n, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      SPMVK_CUDA(cudaStreamSynchronize(s));
      std::vector<uint32_t> heavy(static_cast<size_t>(n));
      if (n)
        SPMVK_CUDA(cudaMemcpyAsync(heavy.data(), sel.p, 4ull * n, cudaMemcpyDeviceToHost, s));
      h->n_heavy = static_cast<uint64_t>(n);
      h->heavy_rows.alloc(h->n_heavy);
      if (n)
        SPMVK_CUDA(cudaMemcpyAsync(h->heavy_rows.p, sel.p, 4ull * n, cudaMemcpyDeviceToDevice,
                                   s));
      SPMVK_CUDA(cudaStreamSynchronize(s));
      h->heavy_rows_host = std::move(heavy);
    }
    collect_dyn_heavy(h, s);
  }
  TmpBuf<unsigned long long> cnt(2, s);  // ELL nnz, largest COO column
  SPMVK_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), s));
  if (a->rows) {
    ell_nnz_from_csr<T, V><<<grid, 256, 0, s>>>(a->rows, static_cast<uint32_t>(h->k1),
                                                a->row_ptr.p, a->col.p,
                                                reinterpret_cast<const V*>(a->val.p), cnt.p);
    SPMVK_LAUNCH("ell_nnz_from_csr");
  }
  uint64_t* slot = pinned_slot();
  SPMVK_CUDA(cudaMemcpyAsync(slot, cnt.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             s));
  if (coo)
    SPMVK_CUDA(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(slot + 2), h->coo_rows.p + coo - 1, 4,
                               cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  const unsigned long long ell_nnz = slot[0];
  if (coo) {  // bounds of the COO part, for spmv_coo's check (COO is sorted by row)
    h->coo_max_col = static_cast<uint32_t>(slot[1]);
    h->coo_max_row = reinterpret_cast<const uint32_t*>(slot + 2)[0];
  }
  h->fill_nnz = ell_nnz + coo;
}

spmvk_hybrid* build(const spmvk_csr* a, int64_t k1, int prec, cudaStream_t s) {
  if (!a) fail(SPMVK_EINVAL, "null CSR handle");
  if (prec != SPMVK_F32 && prec != SPMVK_F64)
    fail(SPMVK_EINVAL, "precision must be SPMVK_F32 (4) or SPMVK_F64 (8)");
  if (a->val_prec == SPMVK_F32 && prec == SPMVK_F64)
    fail(SPMVK_EINVAL, "cannot build a double Hybrid from a float CSR");
  unsigned mx = 0, mn = 0;
  row_length_range(a, 0, a->rows, &mx, &mn, s);
  const uint64_t width = k1 < 0 ? choose_width_device(a, mx, s) : static_cast<uint64_t>(k1);
  if (width > mx)
    fail(SPMVK_EINVAL, "build_hybrid: k1 " + std::to_string(width) +
                           " exceeds the maximum row length " + std::to_string(mx));
  if (a->rows * width > 0xffffffffull)
    fail(SPMVK_ERANGE, "build_hybrid: " + std::to_string(a->rows * width) +
                           " ELL slots overflow the 32-bit index type");
  auto h = std::make_unique<spmvk_hybrid>();
  h->rows = a->rows;
  h->cols = a->cols;
  h->k1 = width;
  h->prec = prec;
  h->nnz = a->nnz;
  h->ell_values.alloc(a->rows * width * prec);
  h->ell_columns.alloc(a->rows * width);
  if (prec == SPMVK_F64) fill<double, double>(h.get(), a, s, mx);
  else if (a->val_prec == SPMVK_F64) fill<float, double>(h.get(), a, s, mx);
  else fill<float, float>(h.get(), a, s, mx);
  return h.release();
}

}  // namespace

// spmv_csr = the dyn kernel with K1 = 0: every entry is in the "COO" part,
// row_ptr is the run pointer array; rows with more than kHeavyDyn entries are
// the (longest-first) warp items.
template <class T>
bool csr_spmv_dyn(const spmvk_csr* a, const T* x, T* y, cudaStream_t s, bool only_if_heavy) {
  {
    std::lock_guard<std::mutex> lk(a->meta_mu);
    if (!a->heavy_ready) {
      const uint64_t cap = a->nnz / (kHeavyDyn + 1) + 1;
      TmpBuf<uint32_t> list(cap, s), key(cap, s), key2(cap, s);
      TmpBuf<unsigned> cnt(1, s);
      SPMVK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), s));
      heavy_collect<<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(
          a->rows, a->row_ptr.p, kHeavyDyn, list.p, key.p, cnt.p);
      SPMVK_LAUNCH("heavy_collect");
      unsigned n = 0;
      SPMVK_CUDA(cudaMemcpyAsync(&n, cnt.p, sizeof(n), cudaMemcpyDeviceToHost, s));
      SPMVK_CUDA(cudaStreamSynchronize(s));
      a->n_heavy = n;
      a->heavy.alloc(n);
      if (n) {
        size_t tb = 0;
        SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, list.p,
                                                   a->heavy.p, static_cast<int>(n), 0, 32, s));
        TmpBuf<unsigned char> tmp(tb, s);
        SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key2.p, list.p, a->heavy.p,
                                                   static_cast<int>(n), 0, 32, s));
      }
      a->heavy_ready = true;
    }
  }
  if (only_if_heavy && a->n_heavy == 0) return false;
  auto kern = sizeof(T) == 4 ? hybrid_spmv_dyn<T, 4, 6, 4, true> : hybrid_spmv_dyn<T, 4, 5, 4, false>;
  int per_sm = 0;
  SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  const LongList hl{static_cast<uint32_t>(a->n_heavy), 0u, a->heavy.p, nullptr,
                    stream_counters(s), 2u};
  kern<<<persistent_grid((a->rows + 255) / 256, per_sm > 0 ? per_sm : 1), 256, 0, s>>>(
      static_cast<uint32_t>(a->rows), 0u, nullptr, nullptr, a->row_ptr.p, a->col.p,
      reinterpret_cast<const T*>(a->val.p), x, y, kHeavyDyn, hl);
  SPMVK_LAUNCH("hybrid_spmv_dyn (csr)");
  return true;
}
template bool csr_spmv_dyn<double>(const spmvk_csr*, const double*, double*, cudaStream_t, bool);
template bool csr_spmv_dyn<float>(const spmvk_csr*, const float*, float*, cudaStream_t, bool);

namespace {

template <class T>
void check_args(const spmvk_hybrid* h, uint64_t nx, uint64_t ny) {
  if (!h) fail(SPMVK_EINVAL, "null Hybrid handle");
  if (nx != h->cols || ny != h->rows) fail(SPMVK_EINVAL, "spmv_ellpack: dimension mismatch");
  if (h->prec != static_cast<int>(sizeof(T)))
    fail(SPMVK_EINVAL, "spmv_hybrid: handle precision differs from the entry point");
}

// part: kBoth = spmv_hybrid, kEll = spmv_ellpack(h.ell), kCoo = spmv_coo(h.coo)
// (accumulating into y, rows limited to the caller's y length).
enum class Part { kBoth, kEll, kCoo };

template <class T>
void launch(const spmvk_hybrid* h, const T* x, T* y, cudaStream_t s, Part part = Part::kBoth,
            uint64_t rows_limit = ~0ull) {
  const uint64_t rows = std::min<uint64_t>(h->rows, rows_limit);
  if (rows == 0) return;
  if (part == Part::kCoo && !h->coo) return;
  const uint64_t ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
  const uint32_t k1 = part == Part::kCoo ? 0u : static_cast<uint32_t>(h->k1);
  const uint32_t* tp = part != Part::kEll && h->coo ? h->tile_ptr.p : nullptr;
  HK k = static_cast<HK>(hk_slot().load(std::memory_order_relaxed));
  if (k == HK::kAuto) {
    // measured (scripts/ab_formats.py; profiles/r01_hybrid_variants.md,
    // profiles/r02_ab.md): with a COO part the fenced 4-deep lite kernel
    // (power-law fp64 736 us; fp32 with L2 hints 675 vs 690); pure ELL takes
    // the group-walk batch shape matching K1 -- 5-point (K1 = 5) U = 6:
    // fp64 47.1 vs 49.3 us, fp32 31.8 vs 34.9 (5-pt 2048^2); 27-point U = 7:
    // fp64 105.2 vs 106.8, fp32 76.1 vs 77.7; 7-point keeps U = 4 (fp32
    // 172.4 vs 172.7 for U = 7, 174.5 for U = 8).
    // With a COO part, spmv_hybrid takes hybrid_spmv_dyn (config-3 power-law
    // 8M, original order: fp64 617 vs 744 us, fp32 533 vs 677; descending
    // order 837 vs 846 / 733 vs 726 -- profiles/r02_hybrid_dyn.md); the
    // spmv_coo / spmv_ellpack parts keep the staged-tile kernels.
    // fp32 pure ELL takes the 128-bit slot loads (4 rows per thread): 27-pt
    // 128^3 77.4 -> 71.3 us, 5-pt 2048^2 32.3 -> 28.9, 7-pt 256^3 172.5 ->
    // 171.2; fp64 gains nothing (108.2 vs 108.0, 7-pt 242 vs 253) and keeps
    // the scalar shapes (profiles/r02_hybrid_dyn.md)
    const bool pure_ell = part == Part::kEll || !h->coo;
    if (pure_ell && sizeof(T) == 4 && h->rows % 4 == 0 && part == Part::kBoth) k = HK::kVec;
    else if (pure_ell) k = k1 <= 6 ? HK::kG6 : k1 <= 12 ? HK::kLiteF : HK::kG7;
    else if (part == Part::kBoth) k = HK::kDyn;
    else k = sizeof(T) == 4 ? HK::kLiteFH : HK::kLiteF;
  }
  auto run = [&](auto kern) {
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowsPerTile, 0));
    kern<<<persistent_grid(ntiles, per_sm > 0 ? per_sm : 1), kRowsPerTile, 0, s>>>(
        static_cast<uint32_t>(rows), k1, reinterpret_cast<const T*>(h->ell_values.p),
        h->ell_columns.p, tp, h->coo_rows.p, h->coo_columns.p,
        reinterpret_cast<const T*>(h->coo_values.p), x, y, h->coo_row_ptr.p);
    SPMVK_LAUNCH("hybrid_spmv");
  };
  const bool acc = part == Part::kCoo, coo = tp != nullptr;
  // spmv_hybrid with a COO part: dynamic slices, warp-staged COO, heavy rows
  // as work items (one launch; other variants / parts fall through below)
  if (k == HK::kDyn && part == Part::kBoth && coo && rows == h->rows) {
    static const uint32_t hw = [] {
      const char* e = std::getenv("SPMVK_HYB_HEAVY_WARPS");
      const int v = e ? std::atoi(e) : 2;
      return static_cast<uint32_t>(v < 1 ? 1 : v > 8 ? 8 : v);
    }();
    auto kern = sizeof(T) == 4 ? hybrid_spmv_dyn<T, 4, 6, 4, true> : hybrid_spmv_dyn<T, 4, 5, 4, false>;
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const LongList hl{static_cast<uint32_t>(h->n_dyn_heavy), 0u, h->dyn_heavy.p, nullptr,
                      stream_counters(s), hw};
    kern<<<persistent_grid(ntiles, per_sm > 0 ? per_sm : 1), 256, 0, s>>>(
        static_cast<uint32_t>(rows), k1, reinterpret_cast<const T*>(h->ell_values.p),
        h->ell_columns.p, h->coo_row_ptr.p, h->coo_columns.p,
        reinterpret_cast<const T*>(h->coo_values.p), x, y, h->dyn_heavy_run, hl);
    SPMVK_LAUNCH("hybrid_spmv_dyn");
    return;
  }
  if (k == HK::kDyn) k = HK::kLiteF;
  // pure ELL with 128-bit slot loads (rows % R == 0 keeps the vectors aligned)
  if (k == HK::kVec) {
    constexpr uint64_t R = 16 / sizeof(T);
    if (!coo && !acc && rows == h->rows && rows % R == 0) {
      auto kern = hybrid_ell_vec<T, 4, sizeof(T) == 8 ? 5 : 4>;
      int per_sm = 0;
      SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
      kern<<<persistent_grid((rows + 256 * R - 1) / (256 * R), per_sm > 0 ? per_sm : 1), 256, 0,
             s>>>(static_cast<uint32_t>(rows), k1, reinterpret_cast<const T*>(h->ell_values.p),
                  h->ell_columns.p, x, y);
      SPMVK_LAUNCH("hybrid_ell_vec");
      return;
    }
    k = HK::kLiteF;
  }
  // after the main kernel (any variant but v4, which stages every tile): the
  // heavy rows' COO tails, warp per row, onto the y the main kernel stored
  auto heavy = [&]() {
    if (k == HK::kV4 || !coo || !h->n_heavy) return;
    const auto& hr = h->heavy_rows_host;
    const uint64_t n = std::lower_bound(hr.begin(), hr.end(), rows) - hr.begin();
    if (!n) return;
    auto hk = k == HK::kLiteFH ? hybrid_heavy_rows<T, true> : hybrid_heavy_rows<T, false>;
    hk<<<persistent_grid((n + 7) / 8, 8), 256, 0, s>>>(
        static_cast<uint32_t>(n), h->heavy_rows.p, h->coo_row_ptr.p, h->coo_columns.p,
        reinterpret_cast<const T*>(h->coo_values.p), x, y);
    SPMVK_LAUNCH("hybrid_heavy_rows");
  };
  switch (k) {
    case HK::kV4:
      if (acc) run(hybrid_spmv_kernel<T, 4, true>); else run(hybrid_spmv_kernel<T, 4>);
      break;
    case HK::kLite:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true>);
      else run(hybrid_spmv_lite<T, 4, 8, false, false>);
      break;
    case HK::kLite8Full:
      if (acc) run(hybrid_spmv_lite<T, 8, 8, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 8, 8, false, true>);
      else run(hybrid_spmv_lite<T, 8, 8, false, false>);
      break;
    case HK::kLiteF:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true, true>);
      else run(hybrid_spmv_lite<T, 4, 8, false, false, true>);
      break;
    case HK::kLiteFH:  // fp64 + COO: 6 CTAs / SM (the policies spill at 8)
      if (acc) run(hybrid_spmv_lite<T, 4, sizeof(T) == 8 ? 6 : 8, true, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, sizeof(T) == 8 ? 6 : 8, false, true, true, true>);
      else run(hybrid_spmv_lite<T, 4, 8, false, false, true, true>);
      break;
    case HK::kLite8F:
      if (acc) run(hybrid_spmv_lite<T, 8, 4, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 8, 4, false, true, true>);
      else run(hybrid_spmv_lite<T, 8, 4, false, false, true>);
      break;
    // group-walk shapes: pure ELL launches only (a COO part keeps liteF)
    case HK::kG6:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true, true>);
      else run(hybrid_spmv_lite<T, 6, 5, false, false, true>);
      break;
    case HK::kG7:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true, true>);
      else run(hybrid_spmv_lite<T, 7, 5, false, false, true>);
      break;
    case HK::kG8:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true, true>);
      else run(hybrid_spmv_lite<T, 8, 5, false, false, true>);
      break;
    case HK::kG8R:
      if (acc) run(hybrid_spmv_lite<T, 4, 8, true, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 4, 8, false, true, true>);
      else run(hybrid_spmv_lite<T, 8, 4, false, false, true>);
      break;
    default:
      if (acc) run(hybrid_spmv_lite<T, 8, 5, true, true>);
      else if (coo) run(hybrid_spmv_lite<T, 8, 5, false, true>);
      else run(hybrid_spmv_lite<T, 8, 5, false, false>);
      break;
  }
  heavy();
}

template <class T>
void spmv_host(const spmvk_hybrid* h, const T* x, uint64_t nx, T* y, uint64_t ny) {
  check_args<T>(h, nx, ny);
  HostStage& st = host_stage();
  st.reserve(nx * sizeof(T), ny * sizeof(T));
  if (nx) SPMVK_CUDA(cudaMemcpyAsync(st.x.p, x, nx * sizeof(T), cudaMemcpyHostToDevice, st.stream));
  launch<T>(h, reinterpret_cast<const T*>(st.x.p), reinterpret_cast<T*>(st.y.p), st.stream);
  if (ny) SPMVK_CUDA(cudaMemcpyAsync(y, st.y.p, ny * sizeof(T), cudaMemcpyDeviceToHost, st.stream));
  SPMVK_CUDA(cudaStreamSynchronize(st.stream));
}

template <class T>
void spmv_part(const spmvk_hybrid* h, const T* x, uint64_t nx, T* y, uint64_t ny, Part part,
               cudaStream_t s) {
  if (!h) fail(SPMVK_EINVAL, "null Hybrid handle");
  if (h->prec != static_cast<int>(sizeof(T)))
    fail(SPMVK_EINVAL, "spmv_hybrid: handle precision differs from the entry point");
  if (part == Part::kEll) {
    if (nx != h->cols || ny != h->rows) fail(SPMVK_EINVAL, "spmv_ellpack: dimension mismatch");
    launch<T>(h, x, y, s, Part::kEll);
    return;
  }
  if (h->coo && (h->coo_max_row >= ny || h->coo_max_col >= nx))
    fail(SPMVK_EINVAL, "spmv_coo: entry outside x/y dimensions");
  launch<T>(h, x, y, s, Part::kCoo, ny);
}

// Host spans: x (and, for the accumulating COO part, y) staged through the
// per-thread device buffers.
template <class T>
void spmv_part_host(const spmvk_hybrid* h, const T* x, uint64_t nx, T* y, uint64_t ny,
                    Part part) {
  HostStage& st = host_stage();
  st.reserve(nx * sizeof(T), ny * sizeof(T));
  if (nx) SPMVK_CUDA(cudaMemcpyAsync(st.x.p, x, nx * sizeof(T), cudaMemcpyHostToDevice, st.stream));
  if (part == Part::kCoo && ny)
    SPMVK_CUDA(cudaMemcpyAsync(st.y.p, y, ny * sizeof(T), cudaMemcpyHostToDevice, st.stream));
  spmv_part<T>(h, reinterpret_cast<const T*>(st.x.p), nx, reinterpret_cast<T*>(st.y.p), ny, part,
               st.stream);
  if (ny) SPMVK_CUDA(cudaMemcpyAsync(y, st.y.p, ny * sizeof(T), cudaMemcpyDeviceToHost, st.stream));
  SPMVK_CUDA(cudaStreamSynchronize(st.stream));
}

}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_set_hybrid_kernel(const char* name) {
  return guarded([&] {
    const std::string v = name ? name : "";
    HK k;
    if (v == "auto") k = HK::kAuto;
    else if (v == "v4") k = HK::kV4;
    else if (v == "lite") k = HK::kLite;
    else if (v == "lite8") k = HK::kLite8;
    else if (v == "lite8_full") k = HK::kLite8Full;
    else if (v == "litef") k = HK::kLiteF;
    else if (v == "lite8f") k = HK::kLite8F;
    else if (v == "g6") k = HK::kG6;
    else if (v == "g7") k = HK::kG7;
    else if (v == "g8") k = HK::kG8;
    else if (v == "g8r") k = HK::kG8R;
    else if (v == "litefh") k = HK::kLiteFH;
    else if (v == "dyn") k = HK::kDyn;
    else if (v == "vec") k = HK::kVec;
    else
      fail(SPMVK_EINVAL, "unknown Hybrid kernel variant '" + v +
                             "' (auto | v4 | lite | lite8 | lite8_full | litef | lite8f | g6 | "
                             "g7 | g8 | g8r | litefh | dyn | vec)");
    hk_slot().store(static_cast<int>(k));
  });
}

uint64_t spmvk_hybrid_split_cost(const uint64_t* lens, uint64_t n, uint64_t k) {
  uint64_t overflow = 0;
  for (uint64_t i = 0; i < n; ++i) overflow += lens[i] > k ? lens[i] - k : 0;
  return 2 * n * k + 3 * overflow;
}

uint64_t spmvk_choose_ell_width(const uint64_t* lens, uint64_t n) {
  uint64_t max_len = 0;
  for (uint64_t i = 0; i < n; ++i) max_len = std::max(max_len, lens[i]);
  std::vector<unsigned long long> hist(max_len + 1, 0);
  for (uint64_t i = 0; i < n; ++i) ++hist[lens[i]];
  return width_from_hist(hist, n);
}

int spmvk_csr_choose_ell_width(const spmvk_csr* a, uint64_t* k1) {
  return guarded([&] {
    if (!a || !k1) fail(SPMVK_EINVAL, "null argument");
    unsigned mx = 0, mn = 0;
    row_length_range(a, 0, a->rows, &mx, &mn, nullptr);
    *k1 = choose_width_device(a, mx, nullptr);
  });
}

int spmvk_hybrid_build(const spmvk_csr* a, int64_t k1, int prec, void* stream,
                       spmvk_hybrid** out) {
  return guarded([&] {
    require_device();
    if (!out) fail(SPMVK_EINVAL, "null argument");
    *out = build(a, k1, prec, as_stream(stream));
  });
}

int spmvk_ellpack_build(const spmvk_csr* a, uint64_t slot_budget, int prec, void* stream,
                        spmvk_hybrid** out) {
  return guarded([&] {
    require_device();
    if (!out || !a) fail(SPMVK_EINVAL, "null argument");
    unsigned mx = 0, mn = 0;
    row_length_range(a, 0, a->rows, &mx, &mn, as_stream(stream));
    const uint64_t k = mx;
    if (k != 0 && a->rows > slot_budget / k)  // ellpack.hpp:88-93
      fail(SPMVK_ERANGE, "build_ellpack: " + std::to_string(a->rows) + " rows x width " +
                             std::to_string(k) + " exceeds the slot budget of " +
                             std::to_string(slot_budget));
    spmvk_hybrid* h = build(a, static_cast<int64_t>(k), prec, as_stream(stream));
    h->ellpack = true;
    *out = h;
  });
}

int spmvk_hybrid_get_info(const spmvk_hybrid* h, spmvk_hybrid_info* info) {
  return guarded([&] {
    if (!h || !info) fail(SPMVK_EINVAL, "null argument");
    info->num_rows = h->rows;
    info->num_cols = h->cols;
    info->ell_width = h->k1;
    info->ell_slots = h->rows * h->k1;
    info->coo_nnz = h->coo;
    info->nnz = h->nnz;
    info->fill_nnz = h->fill_nnz;
    const uint64_t slots = info->ell_slots + h->coo;
    info->artificial_zeros = slots - h->fill_nnz;
    // fill.hpp:67-72: index words = ell slots + 2 * coo
    const uint64_t words = info->ell_slots + 2 * h->coo;
    info->bytes_single = slots * 4 + words * 4;
    info->bytes_double = slots * 8 + words * 4;
    info->precision = h->prec;
    info->ellpack = h->ellpack ? 1 : 0;
  });
}

int spmvk_hybrid_to_csr(const spmvk_hybrid* h, void* stream, spmvk_csr** out) {
  return guarded([&] {
    if (!h || !out) fail(SPMVK_EINVAL, "null argument");
    *out = h->prec == SPMVK_F64 ? hybrid_to_csr<double>(h, as_stream(stream))
                                : hybrid_to_csr<float>(h, as_stream(stream));
  });
}

int spmvk_hybrid_download(const spmvk_hybrid* h, void* ell_values, uint32_t* ell_columns,
                          uint32_t* coo_rows, uint32_t* coo_columns, void* coo_values) {
  return guarded([&] {
    if (!h) fail(SPMVK_EINVAL, "null Hybrid handle");
    const uint64_t es = h->rows * h->k1;
    if (ell_values && es)
      SPMVK_CUDA(cudaMemcpy(ell_values, h->ell_values.p, es * h->prec, cudaMemcpyDeviceToHost));
    if (ell_columns && es)
      SPMVK_CUDA(cudaMemcpy(ell_columns, h->ell_columns.p, es * 4, cudaMemcpyDeviceToHost));
    if (coo_rows && h->coo)
      SPMVK_CUDA(cudaMemcpy(coo_rows, h->coo_rows.p, h->coo * 4, cudaMemcpyDeviceToHost));
    if (coo_columns && h->coo)
      SPMVK_CUDA(cudaMemcpy(coo_columns, h->coo_columns.p, h->coo * 4, cudaMemcpyDeviceToHost));
    if (coo_values && h->coo)
      SPMVK_CUDA(cudaMemcpy(coo_values, h->coo_values.p, h->coo * h->prec, cudaMemcpyDeviceToHost));
  });
}

int spmvk_hybrid_spmv_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                          uint64_t ny, void* stream) {
  return guarded([&] {
    check_args<double>(h, nx, ny);
    launch<double>(h, x, y, as_stream(stream));
  });
}

int spmvk_hybrid_spmv_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                          uint64_t ny, void* stream) {
  return guarded([&] {
    check_args<float>(h, nx, ny);
    launch<float>(h, x, y, as_stream(stream));
  });
}

int spmvk_hybrid_spmv_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                               uint64_t ny) {
  return guarded([&] { spmv_host<double>(h, x, nx, y, ny); });
}

int spmvk_hybrid_spmv_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                               uint64_t ny) {
  return guarded([&] { spmv_host<float>(h, x, nx, y, ny); });
}

int spmvk_hybrid_spmv_ell_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, void* stream) {
  return guarded([&] { spmv_part<double>(h, x, nx, y, ny, Part::kEll, as_stream(stream)); });
}

int spmvk_hybrid_spmv_ell_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, void* stream) {
  return guarded([&] { spmv_part<float>(h, x, nx, y, ny, Part::kEll, as_stream(stream)); });
}

int spmvk_hybrid_spmv_coo_f64(const spmvk_hybrid* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, void* stream) {
  return guarded([&] { spmv_part<double>(h, x, nx, y, ny, Part::kCoo, as_stream(stream)); });
}

int spmvk_hybrid_spmv_coo_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, void* stream) {
  return guarded([&] { spmv_part<float>(h, x, nx, y, ny, Part::kCoo, as_stream(stream)); });
}

int spmvk_hybrid_spmv_ell_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx,
                                   double* y, uint64_t ny) {
  return guarded([&] { spmv_part_host<double>(h, x, nx, y, ny, Part::kEll); });
}

int spmvk_hybrid_spmv_ell_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                                   uint64_t ny) {
  return guarded([&] { spmv_part_host<float>(h, x, nx, y, ny, Part::kEll); });
}

int spmvk_hybrid_spmv_coo_host_f64(const spmvk_hybrid* h, const double* x, uint64_t nx,
                                   double* y, uint64_t ny) {
  return guarded([&] { spmv_part_host<double>(h, x, nx, y, ny, Part::kCoo); });
}

int spmvk_hybrid_spmv_coo_host_f32(const spmvk_hybrid* h, const float* x, uint64_t nx, float* y,
                                   uint64_t ny) {
  return guarded([&] { spmv_part_host<float>(h, x, nx, y, ny, Part::kCoo); });
}

void spmvk_hybrid_destroy(spmvk_hybrid* h) { delete h; }

}  // extern "C"
