// CSR ingest on the device: upload + canonical-form validation, stencil
// generation directly in HBM, and the thread-per-row spmv_csr comparator.
//
// Reference: TripletMatrix ctor validation (src/triplet.cpp:22-32),
// build_csr (spmvkit/csr.hpp:24-39), spmv_csr (spmvkit/csr.hpp:41-53).
#include <algorithm>
#include <memory>
#include <string>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.cuh"

namespace spmvk {
namespace {

// ------------------------------------------------------------ validation
// flag bit 1: row_ptr not monotone / ends wrong; 2: column out of bounds;
// 4: columns not strictly increasing.  bad_row = smallest offending row.
__global__ void validate_csr(uint64_t rows, uint64_t cols, uint64_t nnz,
                             const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                             unsigned* flag, unsigned long long* bad_row) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rp[r], e = rp[r + 1];
    unsigned f = 0;
    if (r == 0 && b != 0) f |= 1;
    if (r + 1 == rows && e != nnz) f |= 1;
    if (e < b || e > nnz) {
      f |= 1;
    } else {
      uint32_t prev = 0;
      for (uint32_t k = b; k < e; ++k) {
        const uint32_t c = col[k];
        if (c >= cols) f |= 2;
        if (k > b && c <= prev) f |= 4;
        prev = c;
      }
    }
    if (f) {
      atomicOr(flag, f);
      atomicMin(bad_row, (unsigned long long)r);
    }
  }
}

void validate(const spmvk_csr& a, cudaStream_t s) {
  if (a.rows == 0) {
    if (a.nnz != 0) fail(SPMVK_EINVAL, "entries given for a matrix with zero rows");
    return;
  }
  DevBuf<unsigned long long> scratch(2);
  unsigned long long init[2] = {0, ~0ull};
  SPMVK_CUDA(cudaMemcpyAsync(scratch.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  validate_csr<<<persistent_grid((a.rows + 255) / 256, 8), 256, 0, s>>>(
      a.rows, a.cols, a.nnz, a.row_ptr.p, a.col.p, reinterpret_cast<unsigned*>(scratch.p),
      scratch.p + 1);
  SPMVK_LAUNCH("validate_csr");
  unsigned long long out[2];
  SPMVK_CUDA(cudaMemcpyAsync(out, scratch.p, sizeof(out), cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  const unsigned f = static_cast<unsigned>(out[0]);
  if (f) {
    std::string why = (f & 1)   ? "row pointers are not a monotone offset array ending at nnz"
                      : (f & 2) ? "column index outside the matrix"
                                : "entries not strictly increasing in (row, col)";
    fail(SPMVK_EINVAL, why + " (first bad row " + std::to_string(out[1]) + ")");
  }
}

// ------------------------------------------------------------ stencils in HBM
struct StencilShape {
  int kind;
  uint64_t n, nz;
};

__device__ __forceinline__ uint32_t stencil_row(const StencilShape sh, uint64_t r, uint32_t* col,
                                                double* val) {
  const uint64_t x = r % sh.n, y = (r / sh.n) % sh.n, z = r / (sh.n * sh.n);
  const double diag = sh.kind == 5 ? 4.0 : sh.kind == 7 ? 6.0 : 26.0;
  uint32_t k = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (sh.kind == 5 && dz != 0) continue;
        const int nnb = (dz != 0) + (dy != 0) + (dx != 0);
        if (sh.kind != 27 && nnb > 1) continue;
        const int64_t zz = (int64_t)z + dz, yy = (int64_t)y + dy, xx = (int64_t)x + dx;
        if (zz < 0 || yy < 0 || xx < 0 || zz >= (int64_t)sh.nz || yy >= (int64_t)sh.n ||
            xx >= (int64_t)sh.n)
          continue;
        if (col) {
          col[k] = (uint32_t)(((uint64_t)zz * sh.n + (uint64_t)yy) * sh.n + (uint64_t)xx);
          val[k] = nnb == 0 ? diag : -1.0;
        }
        ++k;
      }
  return k;
}

__global__ void stencil_lengths(StencilShape sh, uint64_t rows, uint64_t* len) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    len[r] = stencil_row(sh, r, nullptr, nullptr);
}

__global__ void stencil_fill(StencilShape sh, uint64_t rows, const uint64_t* __restrict__ off,
                             uint32_t* __restrict__ rp, uint32_t* __restrict__ col,
                             double* __restrict__ val) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = off[r];
    rp[r] = (uint32_t)o;
    const uint32_t k = stencil_row(sh, r, col + o, val + o);
    if (r + 1 == rows) rp[rows] = (uint32_t)(o + k);
  }
}

// ------------------------------------------------------------ row-length range
__global__ void row_len_range(uint64_t rows, const uint32_t* __restrict__ rp,
                              unsigned* out /* [0]=max [1]=min */) {
  unsigned mx = 0, mn = 0xffffffffu;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned l = rp[r + 1] - rp[r];
    mx = max(mx, l);
    mn = min(mn, l);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_min_sync(0xffffffffu, mn);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    atomicMin(out + 1, mn);
  }
}

// ------------------------------------------------------------ column range
// min / max column index over entries [b, e) (the x range a row slab reads).
__global__ void col_range(uint64_t b, uint64_t e, const uint32_t* __restrict__ col,
                          unsigned* out /* [0]=min [1]=max */) {
  unsigned mn = 0xffffffffu, mx = 0;
  for (uint64_t k = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned c = col[k];
    mn = min(mn, c);
    mx = max(mx, c);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

// ------------------------------------------------------------ spmv_csr
// Thread per row, entries in column order, separately rounded multiply/add:
// bitwise the reference's spmv_csr (csr.hpp:45-51).
template <class T>
__global__ void __launch_bounds__(256) csr_spmv_kernel(uint64_t rows,
                                                       const uint32_t* __restrict__ rp,
                                                       const uint32_t* __restrict__ col,
                                                       const T* __restrict__ val,
                                                       const T* __restrict__ x,
                                                       T* __restrict__ y) {
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = rp[r], e = rp[r + 1];
    T acc = T(0);
    uint32_t k = b;
    for (; k + 4 <= e; k += 4) {
      uint32_t c[4];
      T v[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = ld_stream(col + k + u, pf);
        v[u] = ld_stream(val + k + u, pf);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = ld_x(x + c[u], pl);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    }
    for (; k < e; ++k) acc = add_rn(acc, mul_rn(ld_stream(val + k, pf), ld_x(x + ld_stream(col + k, pf), pl)));
    y[r] = acc;
  }
}

// Tile-staged CSR SpMV (the default): CTA per 256-row tile; the tile's
// entries [rp[r0], rp[r0+256]) are contiguous, so all 256 threads stream
// them in coalesced chunks of kCsrChunk entries, each thread forming
// products val * x[col] for consecutive entries into shared memory; then
// thread r adds the products of its own row that fall in the chunk, in entry
// order (acc carried across chunks) -- the reference's rounding sequence, so
// y stays bitwise, with HBM reads as coalesced as the slot-major formats.
template <class T, int U, int MINB, uint32_t kCsrChunk>
__global__ void __launch_bounds__(256, MINB) csr_spmv_staged(uint32_t rows,
                                                             const uint32_t* __restrict__ rp,
                                                             const uint32_t* __restrict__ col,
                                                             const T* __restrict__ val,
                                                             const T* __restrict__ x,
                                                             T* __restrict__ y) {
  __shared__ T prod[kCsrChunk];
  const uint32_t ntiles = (rows + 255) / 256;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t r0 = tile * 256, r = r0 + threadIdx.x;
    const uint32_t tb = rp[r0], te = rp[min(rows, r0 + 256)];
    const bool live = r < rows;
    const uint32_t rb = live ? rp[r] : 0, re = live ? rp[r + 1] : 0;
    T acc = T(0);
    for (uint32_t c0 = tb; c0 < te; c0 += kCsrChunk) {
      const uint32_t n = min(kCsrChunk, te - c0);
      for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 256 * U) {
        uint32_t c[U];
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = i0 + u * 256;
          c[u] = i < n ? ld_stream(col + c0 + i) : 0u;
          v[u] = i < n ? ld_stream(val + c0 + i) : T(0);
        }
        __syncwarp(__activemask());  // scheduling fence: all loads before the gathers
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t i = i0 + u * 256;
          if (i < n) prod[i] = mul_rn(v[u], ld_x(x + c[u]));
        }
      }
      __syncthreads();
      const uint32_t a = max(rb, c0), b = min(re, c0 + n);
      uint32_t k = a;
      for (; k + 8 <= b; k += 8) {  // 8 independent LDS in flight, adds in order
        T p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = prod[k - c0 + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = add_rn(acc, p[u]);
      }
      for (; k < b; ++k) acc = add_rn(acc, prod[k - c0]);
      __syncthreads();
    }
    if (live) y[r] = acc;
  }
}

// Warp-staged CSR SpMV: as csr_spmv_staged but per WARP (32 rows, whose
// entries are contiguous too) with a private shared-memory chunk of 32 U
// products -- no CTA-wide barrier, so warps stay independent and the memory
// system sees as many requests in flight as the slot-major kernels.
template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) csr_spmv_warp(uint32_t rows,
                                                           const uint32_t* __restrict__ rp,
                                                           const uint32_t* __restrict__ col,
                                                           const T* __restrict__ val,
                                                           const T* __restrict__ x,
                                                           T* __restrict__ y) {
  constexpr uint32_t CH = 32 * U;
  __shared__ T prod[8][CH];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* pw = prod[warp];
  const uint32_t nwt = (rows + 31) / 32;
  for (uint32_t wt = blockIdx.x * 8 + warp; wt < nwt; wt += gridDim.x * 8) {
    const uint32_t r = wt * 32 + lane;
    const bool live = r < rows;
    const uint32_t rb = live ? rp[r] : 0, re = live ? rp[r + 1] : 0;
    const uint32_t tb = __shfl_sync(0xffffffffu, rb, 0);
    const uint32_t te = rp[min(rows, wt * 32 + 32)];
    T acc = T(0);
    for (uint32_t c0 = tb; c0 < te; c0 += CH) {
      const uint32_t n = min(CH, te - c0);
      uint32_t c[U];
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = lane + 32 * u;
        c[u] = i < n ? ld_stream(col + c0 + i) : 0u;
        v[u] = i < n ? ld_stream(val + c0 + i) : T(0);
      }
      __syncwarp();  // scheduling fence: every load before the gathers
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = lane + 32 * u;
        if (i < n) pw[i] = mul_rn(v[u], ld_x(x + c[u]));
      }
      __syncwarp();
      const uint32_t a = max(rb, c0), b = min(re, c0 + n);
      uint32_t k = a;
      for (; k + 4 <= b; k += 4) {
        T p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) p[u] = pw[k - c0 + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = add_rn(acc, p[u]);
      }
      for (; k < b; ++k) acc = add_rn(acc, pw[k - c0]);
      __syncwarp();
    }
    if (live) y[r] = acc;
  }
}

spmvk_csr* make_csr(uint64_t rows, uint64_t cols, uint64_t nnz, int val_prec) {
  if (val_prec != SPMVK_F32 && val_prec != SPMVK_F64)
    fail(SPMVK_EINVAL, "value precision must be SPMVK_F32 (4) or SPMVK_F64 (8)");
  if (rows >= 0xffffffffull || cols > 0x100000000ull)
    fail(SPMVK_ERANGE, "matrix dimensions exceed the 32-bit index type");
  if (nnz > 0xffffffffull) fail(SPMVK_ERANGE, "nnz exceeds the 32-bit row pointer type");
  auto a = std::make_unique<spmvk_csr>();
  a->rows = rows;
  a->cols = cols;
  a->nnz = nnz;
  a->val_prec = val_prec;
  a->row_ptr.alloc(rows + 1);
  a->col.alloc(nnz);
  a->val.alloc(nnz * static_cast<uint64_t>(val_prec));
  return a.release();
}

template <class T>
void csr_spmv(const spmvk_csr* a, const T* x, uint64_t nx, T* y, uint64_t ny, cudaStream_t s) {
  if (!a) fail(SPMVK_EINVAL, "null CSR handle");
  if (nx != a->cols || ny != a->rows) fail(SPMVK_EINVAL, "spmv_csr: dimension mismatch");
  if (a->val_prec != static_cast<int>(sizeof(T)))
    fail(SPMVK_EINVAL, "spmv_csr: handle precision differs from the entry point");
  if (a->rows == 0) return;
  // SPMVK_CSR_KERNEL: "" (default: "dyn" for matrices with rows past 128
  // entries, else "staged"), "staged" (CTA tile, 1,024-entry chunks, U = 4,
  // 8 CTAs / SM), "dyn" (hybrid_spmv_dyn's warp-staged walk), "warp"
  // (per-warp chunks), "row" (first kernel, thread per row).  Measured (scripts/ab_formats.py, profiles/r01_csr.md): staged
  // 27-pt fp64 163 vs row 413 us, 7-pt 256^3 341 vs 852, power-law 803 vs
  // 2,090; 5-pt 2048^2 74 vs 74.
  static const int variant = [] {
    const char* e = std::getenv("SPMVK_CSR_KERNEL");
    const std::string v = e ? e : "";
    return v == "row" ? 1 : v == "warp" ? 2 : v == "dyn" ? 4 : v == "staged" ? 3 : 0;
  }();
  // default: matrices with rows past 128 entries take the warp-staged dyn
  // kernel (power-law 8M fp64 802 -> 705 us, fp32 671 -> 580; on stencils it
  // loses, 27-pt fp64 166 -> 213), the others the CTA-staged kernel
  // (profiles/r01_csr.md)
  if (variant == 4 || variant == 0) {
    if (csr_spmv_dyn<T>(a, x, y, s, variant == 0)) return;
  }
  if (variant == 1) {
    csr_spmv_kernel<T><<<persistent_grid((a->rows + 255) / 256, 8), 256, 0, s>>>(
        a->rows, a->row_ptr.p, a->col.p, reinterpret_cast<const T*>(a->val.p), x, y);
    SPMVK_LAUNCH("csr_spmv_kernel");
    return;
  }
  auto kern = variant == 2 ? csr_spmv_warp<T, 8, 5> : csr_spmv_staged<T, 4, 8, 1024>;
  int per_sm = 0;
  SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  kern<<<persistent_grid((a->rows + 255) / 256, per_sm > 0 ? per_sm : 1), 256, 0, s>>>(
      static_cast<uint32_t>(a->rows), a->row_ptr.p, a->col.p,
      reinterpret_cast<const T*>(a->val.p), x, y);
  SPMVK_LAUNCH("csr_spmv_staged");
}

}  // namespace

spmvk_csr* new_csr(uint64_t rows, uint64_t cols, uint64_t nnz, int val_prec) {
  return make_csr(rows, cols, nnz, val_prec);
}

// row lengths -> uint32 (used by rgcsr / hybrid builders)
__global__ void csr_row_lengths(uint64_t r0, uint64_t rows, const uint32_t* __restrict__ rp,
                                uint32_t* __restrict__ lens) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    lens[r] = rp[r0 + r + 1] - rp[r0 + r];
}

void row_length_range(const spmvk_csr* a, uint64_t r0, uint64_t r1, unsigned* mx, unsigned* mn,
                      cudaStream_t s) {
  TmpBuf<unsigned> out(2, s);
  unsigned* h = reinterpret_cast<unsigned*>(pinned_slot());
  h[0] = 0;
  h[1] = 0xffffffffu;
  SPMVK_CUDA(cudaMemcpyAsync(out.p, h, 2 * sizeof(unsigned), cudaMemcpyHostToDevice, s));
  if (r1 > r0) {
    row_len_range<<<persistent_grid((r1 - r0 + 255) / 256, 8), 256, 0, s>>>(
        r1 - r0, a->row_ptr.p + r0, out.p);
    SPMVK_LAUNCH("row_len_range");
  }
  SPMVK_CUDA(cudaMemcpyAsync(h, out.p, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  *mx = h[0];
  *mn = r1 > r0 ? h[1] : 0;
}

}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_csr_upload(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t* row_ptr,
                     const uint32_t* col, const void* val, int val_prec, void* stream,
                     spmvk_csr** out) {
  return guarded([&] {
    require_device();
    if (!out || !row_ptr || (nnz && (!col || !val))) fail(SPMVK_EINVAL, "null argument");
    cudaStream_t s = as_stream(stream);
    std::unique_ptr<spmvk_csr> a(make_csr(rows, cols, nnz, val_prec));
    SPMVK_CUDA(cudaMemcpyAsync(a->row_ptr.p, row_ptr, sizeof(uint32_t) * (rows + 1),
                               cudaMemcpyHostToDevice, s));
    if (nnz) {
      SPMVK_CUDA(cudaMemcpyAsync(a->col.p, col, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, s));
      SPMVK_CUDA(cudaMemcpyAsync(a->val.p, val, a->val.bytes(), cudaMemcpyHostToDevice, s));
    }
    validate(*a, s);
    *out = a.release();
  });
}

int spmvk_csr_upload_device(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t* row_ptr,
                            const uint32_t* col, const void* val, int val_prec, void* stream,
                            spmvk_csr** out) {
  return guarded([&] {
    require_device();
    if (!out || !row_ptr || (nnz && (!col || !val))) fail(SPMVK_EINVAL, "null argument");
    cudaStream_t s = as_stream(stream);
    std::unique_ptr<spmvk_csr> a(make_csr(rows, cols, nnz, val_prec));
    SPMVK_CUDA(cudaMemcpyAsync(a->row_ptr.p, row_ptr, sizeof(uint32_t) * (rows + 1),
                               cudaMemcpyDeviceToDevice, s));
    if (nnz) {
      SPMVK_CUDA(
          cudaMemcpyAsync(a->col.p, col, sizeof(uint32_t) * nnz, cudaMemcpyDeviceToDevice, s));
      SPMVK_CUDA(cudaMemcpyAsync(a->val.p, val, a->val.bytes(), cudaMemcpyDeviceToDevice, s));
    }
    validate(*a, s);
    *out = a.release();
  });
}

int spmvk_csr_stencil(int kind, uint64_t n, void* stream, spmvk_csr** out) {
  return guarded([&] {
    require_device();
    if (!out) fail(SPMVK_EINVAL, "null argument");
    if (kind != 5 && kind != 7 && kind != 27) fail(SPMVK_EINVAL, "stencil kind must be 5, 7 or 27");
    if (n == 0) fail(SPMVK_EINVAL, "stencil grid size must be nonzero");
    cudaStream_t s = as_stream(stream);
    const StencilShape sh{kind, n, kind == 5 ? 1 : n};
    const uint64_t rows = n * n * sh.nz;
    DevBuf<uint64_t> off(rows);
    const unsigned grid = persistent_grid((rows + 255) / 256, 8);
    stencil_lengths<<<grid, 256, 0, s>>>(sh, rows, off.p);
    SPMVK_LAUNCH("stencil_lengths");
    const uint64_t nnz = exclusive_scan_u64(off.p, rows, s);
    std::unique_ptr<spmvk_csr> a(make_csr(rows, rows, nnz, SPMVK_F64));
    stencil_fill<<<grid, 256, 0, s>>>(sh, rows, off.p, a->row_ptr.p, a->col.p,
                                      reinterpret_cast<double*>(a->val.p));
    SPMVK_LAUNCH("stencil_fill");
    SPMVK_CUDA(cudaStreamSynchronize(s));
    *out = a.release();
  });
}

int spmvk_csr_shape(const spmvk_csr* a, uint64_t* rows, uint64_t* cols, uint64_t* nnz,
                    int* val_prec) {
  return guarded([&] {
    if (!a) fail(SPMVK_EINVAL, "null CSR handle");
    if (rows) *rows = a->rows;
    if (cols) *cols = a->cols;
    if (nnz) *nnz = a->nnz;
    if (val_prec) *val_prec = a->val_prec;
  });
}

int spmvk_csr_download(const spmvk_csr* a, uint32_t* row_ptr, uint32_t* col, void* val) {
  return guarded([&] {
    if (!a) fail(SPMVK_EINVAL, "null CSR handle");
    if (row_ptr)
      SPMVK_CUDA(cudaMemcpy(row_ptr, a->row_ptr.p, sizeof(uint32_t) * (a->rows + 1),
                            cudaMemcpyDeviceToHost));
    if (col && a->nnz)
      SPMVK_CUDA(cudaMemcpy(col, a->col.p, sizeof(uint32_t) * a->nnz, cudaMemcpyDeviceToHost));
    if (val && a->nnz) SPMVK_CUDA(cudaMemcpy(val, a->val.p, a->val.bytes(), cudaMemcpyDeviceToHost));
  });
}

int spmvk_csr_row_length_range(const spmvk_csr* a, uint64_t* out2) {
  return guarded([&] {
    if (!a || !out2) fail(SPMVK_EINVAL, "null argument");
    unsigned mx, mn;
    row_length_range(a, 0, a->rows, &mx, &mn, nullptr);
    out2[0] = mx;
    out2[1] = mn;
  });
}

int spmvk_csr_column_range(const spmvk_csr* a, uint64_t row_begin, uint64_t row_end,
                           uint64_t* out2) {
  return guarded([&] {
    if (!a || !out2) fail(SPMVK_EINVAL, "null argument");
    if (row_begin > row_end || row_end > a->rows) fail(SPMVK_EINVAL, "row range outside the matrix");
    uint32_t b = 0, e = 0;
    SPMVK_CUDA(cudaMemcpy(&b, a->row_ptr.p + row_begin, 4, cudaMemcpyDeviceToHost));
    SPMVK_CUDA(cudaMemcpy(&e, a->row_ptr.p + row_end, 4, cudaMemcpyDeviceToHost));
    DevBuf<unsigned> d(2);
    unsigned init[2] = {0xffffffffu, 0};
    SPMVK_CUDA(cudaMemcpy(d.p, init, sizeof(init), cudaMemcpyHostToDevice));
    if (e > b) {
      col_range<<<persistent_grid((e - b + 255) / 256, 8), 256>>>(b, e, a->col.p, d.p);
      SPMVK_LAUNCH("col_range");
    }
    unsigned h[2];
    SPMVK_CUDA(cudaMemcpy(h, d.p, sizeof(h), cudaMemcpyDeviceToHost));
    // an empty slab reads nothing: min > max
    out2[0] = e > b ? h[0] : 1;
    out2[1] = e > b ? h[1] : 0;
  });
}

int spmvk_csr_spmv_f64(const spmvk_csr* a, const double* x, uint64_t nx, double* y, uint64_t ny,
                       void* stream) {
  return guarded([&] { csr_spmv<double>(a, x, nx, y, ny, as_stream(stream)); });
}

int spmvk_csr_spmv_f32(const spmvk_csr* a, const float* x, uint64_t nx, float* y, uint64_t ny,
                       void* stream) {
  return guarded([&] { csr_spmv<float>(a, x, nx, y, ny, as_stream(stream)); });
}

void spmvk_csr_destroy(spmvk_csr* a) { delete a; }

}  // extern "C"
