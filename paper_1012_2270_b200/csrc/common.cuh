// Shared plumbing for the spmvk C-ABI: status/error handling, device buffers,
// cache-hinted loads.  sm_100a only.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/spmvk.h"

namespace spmvk {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
const char* last_error_cstr();

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? SPMVK_ENOMEM : SPMVK_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define SPMVK_CUDA(call) ::spmvk::cuda_check((call), #call)
#define SPMVK_LAUNCH(what) ::spmvk::cuda_check(cudaGetLastError(), what)

// Runs f, converting exceptions to status codes + thread-local message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return SPMVK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return SPMVK_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPMVK_ECUDA;
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- device buffer
// Handle arrays come from a per-device cache of released blocks (best fit,
// at most 25 % larger than the request): rebuilding a format of the same
// shape -- the converter in a solver loop, the bench's K1 rate -- reuses the
// previous arrays instead of paying cudaMalloc's page mapping (~1-10 ms for
// the 680 MB headline arrays) and cudaFree's device-wide synchronisation.
// A reused block is handed out only after a device synchronisation, so a
// kernel still reading the handle it came from has finished (the guarantee
// cudaFree gives).  Blocks under 1 MiB bypass the cache; the cache holds at
// most SPMVK_ALLOC_CACHE_MB (default 16384; 0 disables) per device, is
// emptied and the allocation retried when cudaMalloc runs out of memory, and
// spmvk_empty_cache() returns it to the driver.
void* dev_alloc(uint64_t bytes, uint64_t* cap, int* dev);
void dev_release(void* p, uint64_t cap, int dev) noexcept;
void dev_cache_empty(int dev);  // dev < 0: every device

template <class T>
struct DevBuf {
  T* p = nullptr;
  uint64_t n = 0, cap = 0;
  int dev = 0;
  DevBuf() = default;
  explicit DevBuf(uint64_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap), dev(o.dev) {
    o.p = nullptr;
    o.n = o.cap = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; cap = o.cap; dev = o.dev;
      o.p = nullptr;
      o.n = o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(uint64_t count) {
    release();
    // 64 spare bytes: zero-sized arrays stay valid, and 16-byte-aligned bulk
    // copies may round a range end up to 3 elements past the last one
    p = static_cast<T*>(dev_alloc(sizeof(T) * count + 64, &cap, &dev));
    n = count;
  }
  void release() {
    if (p) dev_release(p, cap, dev);
    p = nullptr;
    n = cap = 0;
  }
  uint64_t bytes() const { return n * sizeof(T); }
};

// Stream-ordered temporaries from a per-(device, stream) cache of device
// blocks (power-of-two size classes, allocated with cudaMalloc on a miss and
// kept for the process): a block returned by one call is reused by the next
// call on the SAME stream, which is ordered after every use of it, so a
// converter's scratch costs neither cudaFree's device-wide synchronisation
// nor a pool re-map.  (cudaMallocAsync from the default pool was measured
// 10-200x slower here: the pool trims at every synchronisation.)
void* scratch_get(cudaStream_t s, uint64_t bytes, uint64_t* cls);
void scratch_put(cudaStream_t s, void* p, uint64_t cls);

template <class T>
struct TmpBuf {
  T* p = nullptr;
  uint64_t n = 0, cls = 0;
  cudaStream_t s = nullptr;
  TmpBuf(uint64_t count, cudaStream_t st) : n(count), s(st) {
    p = static_cast<T*>(scratch_get(st, sizeof(T) * count + 64, &cls));
  }
  TmpBuf(const TmpBuf&) = delete;
  TmpBuf& operator=(const TmpBuf&) = delete;
  ~TmpBuf() {
    if (p) scratch_put(s, p, cls);
  }
};

// Number of SMs of the current device (cached per device).
int sm_count();
// Ensures the current device is usable (throws ECUDA otherwise).
void require_device();

// ---------------------------------------------------------------- loads
// L2 cache policies (createpolicy): matrix slots are streamed once
// (evict-first) so that the gathered x vector (evict-last) keeps its L2
// residency across the whole SpMV.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Streamed-once matrix arrays: read-only path, no L1 allocation.
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
// Register-lean forms (no policy operand) for occupancy-bound kernels.
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// 128-bit (and 64-bit) streamed loads of R consecutive rows' slots (the
// vectorised RgCSR kernel; addresses must be aligned to the vector size).
__device__ __forceinline__ double2 ld_stream_v(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_stream_v(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_stream_v(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
               : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_v(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <class T>
__device__ __forceinline__ T ld_x(const T* p) {
  return __ldg(p);
}
// Gathered vector x: read-only path, L1-allocating.
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_x(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

// Load helper with optional L2 eviction hints: kHint -> slot streams
// evict_first, gathered x evict_last (createpolicy once per thread; uniform,
// so ptxas keeps the policies in uniform registers), else the register-lean
// unhinted forms.
template <bool kHint>
struct Ldr {
  uint64_t pf = 0, pl = 0;
  __device__ __forceinline__ Ldr() {
    if constexpr (kHint) {
      pf = policy_evict_first();
      pl = policy_evict_last();
    }
  }
  template <class T>
  __device__ __forceinline__ T s(const T* p) const {
    if constexpr (kHint) return ld_stream(p, pf);
    else return ld_stream(p);
  }
  template <class T>
  __device__ __forceinline__ T x(const T* p) const {
    if constexpr (kHint) return ld_x(p, pl);
    else return ld_x(p);
  }
};

// 1D bulk prefetch of [src, src + bytes) into L2 through the TMA unit (no
// completion tracking); src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Separately rounded multiply and add: the reference's `acc += v * x[c]`
// compiled without FMA contraction (core/CMakeLists.txt has no -march).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// Grid of `per_sm` CTAs per SM, capped by the work.
// log2(G) when G is a power of two (the kernels then shift instead of divide), else -1.
inline int pow2_shift(uint64_t G) {
  if (G == 0 || (G & (G - 1))) return -1;
  int s = 0;
  while ((1ull << s) < G) ++s;
  return s;
}

inline unsigned persistent_grid(uint64_t work_ctas, int per_sm) {
  const uint64_t cap = static_cast<uint64_t>(sm_count()) * static_cast<uint64_t>(per_sm);
  const uint64_t g = work_ctas < cap ? work_ctas : cap;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

// ---------------------------------------------------------------- scan
// Exclusive prefix sum of n uint64 values in place; returns the total (synchronises
// the stream to read it back).  Used for group pointers and COO offsets.
uint64_t exclusive_scan_u64(uint64_t* d, uint64_t n, cudaStream_t s);
// The same scan without the host round trip: the total goes to *total_dev.
void exclusive_scan_u64_dev(uint64_t* d, uint64_t n, cudaStream_t s, uint64_t* total_dev);

// Per-thread staging (stream + x/y device buffers) for the host-span
// overloads (*_spmv_host_*), reused across calls.
struct HostStage {
  cudaStream_t stream = nullptr;
  DevBuf<unsigned char> x, y;
  ~HostStage() {
    if (stream) cudaStreamDestroy(stream);
  }
  void reserve(uint64_t xb, uint64_t yb) {
    if (!stream) SPMVK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (x.n < xb) x.alloc(xb);
    if (y.n < yb) y.alloc(yb);
  }
};
HostStage& host_stage();
// Device scratch of >= n doubles private to (current device, stream s).
double* stream_scratch(cudaStream_t s, uint64_t n);
uint32_t* stream_counters(cudaStream_t s);
// Pinned per-thread 64-byte landing slot for the converters' small
// synchronous readbacks (a pageable destination costs ~15-30 us of host time
// per cudaMemcpyAsync, profiles/r02t_k1_timeline.md).
uint64_t* pinned_slot();

}  // namespace spmvk

// ---------------------------------------------------------------- handles
struct spmvk_csr {
  uint64_t rows = 0, cols = 0, nnz = 0;
  int val_prec = SPMVK_F64;
  spmvk::DevBuf<uint32_t> row_ptr, col;
  spmvk::DevBuf<unsigned char> val;  // nnz * val_prec bytes
  // Lazily built launch metadata of the warp-staged CSR kernel: the rows with
  // more than 128 entries, longest first (kernel metadata, not the reference's).
  mutable std::mutex meta_mu;
  mutable spmvk::DevBuf<uint32_t> heavy;
  mutable uint64_t n_heavy = 0;
  mutable bool heavy_ready = false;
};

struct spmvk_rgcsr {
  uint64_t rows = 0, cols = 0, group_size = 0, groups = 0, slots = 0, nnz = 0;
  int prec = SPMVK_F64;
  spmvk::DevBuf<unsigned char> values;  // slots * prec bytes
  spmvk::DevBuf<uint32_t> columns, group_pointers, row_lengths;
  // Guards the lazily computed launch metadata below (tile_cols).
  mutable std::mutex part_mu;
  // Rows longer than long_cut (ascending ids): K2's thread-per-row kernels
  // skip them and a warp-per-row kernel handles them (power-law tails).
  spmvk::DevBuf<uint32_t> long_rows;
  uint64_t n_long = 0;
  // The same rows split for rgcsr_spmv_long_mixed: quad starts (4 consecutive
  // long rows of one group, r % 4 == 0, each < kQuadMaxLen slots) and singles.
  spmvk::DevBuf<uint32_t> long_quads, long_singles;
  uint64_t n_quads = 0, n_singles = 0;
  uint32_t long_cut = 128;
  // Pipelined host-span SpMV: x column range [min, max] of each 256-row tile.
  mutable std::vector<unsigned> tile_cols;
  // Process-unique id: keys the host-span pipeline's captured CUDA graph
  // (a recycled handle address must not replay a graph of freed arrays).
  const uint64_t serial = next_serial();
  static uint64_t next_serial() {
    static std::atomic<uint64_t> n{0};
    return ++n;
  }
};

namespace spmvk {
constexpr uint32_t kLongRow = 128;
}

struct spmvk_hybrid {
  uint64_t rows = 0, cols = 0, k1 = 0, coo = 0, nnz = 0;
  uint64_t fill_nnz = 0;  // FillReport nnz: ell_nnz recount + coo (fill.hpp:67-72)
  int prec = SPMVK_F64;
  bool ellpack = false;  // built by build_ellpack: fill_report names it "ellpack"
  uint64_t coo_max_row = 0, coo_max_col = 0;  // spmv_coo's bounds check (ellpack.hpp:135)
  spmvk::DevBuf<unsigned char> ell_values, coo_values;
  spmvk::DevBuf<uint32_t> ell_columns, coo_rows, coo_columns;
  // tile_ptr[t]: first COO entry of row tile t (256 rows); kernel metadata,
  // (N/256 + 1) words, not part of the reference's arrays.
  spmvk::DevBuf<uint32_t> tile_ptr;
  // coo_row_ptr[r]: first COO entry of row r (rows + 1 words, kernel
  // metadata): tiles whose COO range is huge (rows with long COO tails sorted
  // together) walk each row's run in its own thread instead of staging.
  spmvk::DevBuf<uint32_t> coo_row_ptr;
  // Rows of walked tiles whose COO run exceeds kHeavyRun: their COO tail is
  // added after the main kernel by a warp per row (hybrid_heavy_rows).
  spmvk::DevBuf<uint32_t> heavy_rows;
  std::vector<uint32_t> heavy_rows_host;  // the same list, to clip it to a row limit
  uint64_t n_heavy = 0;
  // Every row whose COO run exceeds kHeavyDyn, longest first: the work items
  // of hybrid_spmv_dyn (kernel metadata).
  spmvk::DevBuf<uint32_t> dyn_heavy;
  uint64_t n_dyn_heavy = 0;
  uint32_t dyn_heavy_run = 128;
};
