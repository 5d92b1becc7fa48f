#include <algorithm>
// Device plumbing shared by all spmvk entry points: last-error slot, device
// checks, and the uint64 exclusive scan used for group pointers / COO offsets.
#include "common.cuh"

#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

namespace spmvk {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error_cstr() { return g_last_error.c_str(); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  SPMVK_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 0;
  SPMVK_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  if (dev < 64) cached[dev] = n;
  return n;
}

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(SPMVK_ECUDA, std::string("no CUDA device available (") +
                          (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                          "); spmvk has no CPU fallback");
  }
}

HostStage& host_stage() {
  static thread_local HostStage st;
  return st;
}

namespace {
struct ScratchCache {
  std::mutex mu;
  std::map<std::tuple<int, cudaStream_t, uint64_t>, std::vector<void*>> free;
};
ScratchCache& scratch_cache() {
  static ScratchCache* c = new ScratchCache();  // never destroyed: blocks live for the process
  return *c;
}
}  // namespace

namespace {
constexpr uint64_t kCacheMin = 1ull << 20;
struct BlockCache {
  std::mutex mu;
  std::map<int, std::multimap<uint64_t, void*>> free;  // device -> (size, block)
  std::map<int, uint64_t> held;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();
  return *c;
}
uint64_t cache_limit() {
  static const uint64_t lim = [] {
    const char* e = std::getenv("SPMVK_ALLOC_CACHE_MB");
    return (e ? std::strtoull(e, nullptr, 10) : 16384ull) << 20;
  }();
  return lim;
}
}  // namespace

void dev_cache_empty(int dev) {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& [d, m] : c.free) {
    if (dev >= 0 && d != dev) continue;
    if (m.empty()) continue;
    cudaSetDevice(d);
    for (auto& [sz, p] : m) cudaFree(p);
    m.clear();
    c.held[d] = 0;
  }
  cudaSetDevice(cur);
}

void* dev_alloc(uint64_t bytes, uint64_t* cap, int* dev) {
  SPMVK_CUDA(cudaGetDevice(dev));
  if (bytes >= kCacheMin && cache_limit()) {
    void* hit = nullptr;
    {
      BlockCache& c = block_cache();
      std::lock_guard<std::mutex> lk(c.mu);
      auto& m = c.free[*dev];
      auto it = m.lower_bound(bytes);
      if (it != m.end() && it->first <= bytes + bytes / 4) {
        hit = it->second;
        *cap = it->first;
        c.held[*dev] -= it->first;
        m.erase(it);
      }
    }
    if (hit) {
      // kernels still reading the handle this block came from were queued
      // before it was released: let them finish before it is rewritten
      SPMVK_CUDA(cudaDeviceSynchronize());
      return hit;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    dev_cache_empty(*dev);
    e = cudaMalloc(&p, bytes);
  }
  SPMVK_CUDA(e);
  *cap = bytes;
  return p;
}

void dev_release(void* p, uint64_t cap, int dev) noexcept {
  if (cap >= kCacheMin && cache_limit()) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.held[dev] + cap <= cache_limit()) {
      c.free[dev].emplace(cap, p);
      c.held[dev] += cap;
      return;
    }
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaFree(p);
  if (cur != dev) cudaSetDevice(cur);
}

void* scratch_get(cudaStream_t s, uint64_t bytes, uint64_t* cls) {
  uint64_t c = 256;
  while (c < bytes) c <<= 1;
  *cls = c;
  int dev = 0;
  SPMVK_CUDA(cudaGetDevice(&dev));
  ScratchCache& sc = scratch_cache();
  {
    std::lock_guard<std::mutex> lk(sc.mu);
    auto& v = sc.free[{dev, s, c}];
    if (!v.empty()) {
      void* p = v.back();
      v.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  SPMVK_CUDA(cudaMalloc(&p, c));
  return p;
}

void scratch_put(cudaStream_t s, void* p, uint64_t cls) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  ScratchCache& sc = scratch_cache();
  std::lock_guard<std::mutex> lk(sc.mu);
  sc.free[{dev, s, cls}].push_back(p);
}

// Scratch keyed by (device, stream): work on one stream is ordered, so calls
// from any host thread on the same stream may share it, and two streams
// never do (a per-host-thread buffer raced when one thread drove several
// streams).  Grows only outside stream capture.
double* stream_scratch(cudaStream_t s, uint64_t n) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, DevBuf<double>> bufs;
  int dev = 0;
  SPMVK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  DevBuf<double>& b = bufs[{dev, s}];
  if (b.n < n) {
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    SPMVK_CUDA(cudaStreamIsCapturing(s, &cst));
    if (cst != cudaStreamCaptureStatusNone)
      fail(SPMVK_EINVAL, "first reduction on this stream is inside a stream capture; "
                         "call it once eagerly first");
    b.alloc(n);
  }
  return b.p;
}

// Four 32-bit work counters per (device, stream), zero between launches: the
// fused long-row kernels take items from word 0, row slices from word 2, and
// count finished warps in word 1; the last warp resets them (rgcsr_spmv.cuh
// LongList).  Launches
// on one stream are ordered, so they never share a live pair.
uint64_t* pinned_slot() {
  static thread_local uint64_t* p = nullptr;  // kept for the thread's life
  if (!p) SPMVK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), 64, cudaHostAllocPortable));
  return p;
}

uint32_t* stream_counters(cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, DevBuf<uint32_t>> bufs;
  int dev = 0;
  SPMVK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  DevBuf<uint32_t>& b = bufs[{dev, s}];
  if (!b.p) {
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    SPMVK_CUDA(cudaStreamIsCapturing(s, &cst));
    if (cst != cudaStreamCaptureStatusNone)
      fail(SPMVK_EINVAL, "first long-row SpMV on this stream is inside a stream capture; "
                         "call it once eagerly first");
    b.alloc(4);
    SPMVK_CUDA(cudaMemsetAsync(b.p, 0, 4 * sizeof(uint32_t), s));
  }
  return b.p;
}

// ---------------------------------------------------------------- scan
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of one value per thread; returns the block total.
__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t& excl) {
  __shared__ uint64_t warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const uint64_t warp_off = warp == 0 ? 0 : warp_tot[warp - 1];
  const uint64_t total = warp_tot[kScanThreads / 32 - 1];
  excl = warp_off + inc - v;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kScanThreads) scan_tile_reduce(const uint64_t* __restrict__ d,
                                                                 uint64_t n,
                                                                 uint64_t* __restrict__ part) {
  const uint64_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += d[base + i];
  uint64_t ex;
  const uint64_t tot = block_exclusive_scan(s, ex);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of the tile sums; part[nb] receives the total.
__global__ void __launch_bounds__(kScanThreads) scan_partials(uint64_t* part, uint64_t nb) {
  const uint64_t per = (nb + kScanThreads - 1) / kScanThreads;
  const uint64_t b0 = threadIdx.x * per;
  uint64_t s = 0;
  for (uint64_t i = b0; i < b0 + per && i < nb; ++i) s += part[i];
  uint64_t ex;
  const uint64_t tot = block_exclusive_scan(s, ex);
  for (uint64_t i = b0; i < b0 + per && i < nb; ++i) {
    const uint64_t v = part[i];
    part[i] = ex;
    ex += v;
  }
  if (threadIdx.x == 0) part[nb] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_tile_apply(uint64_t* __restrict__ d,
                                                                uint64_t n,
                                                                const uint64_t* __restrict__ part) {
  const uint64_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint64_t v[kScanItems];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? d[base + i] : 0;
    s += v[i];
  }
  uint64_t ex;
  block_exclusive_scan(s, ex);
  ex += part[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) d[base + i] = ex;
    ex += v[i];
  }
}

}  // namespace

namespace {
__global__ void copy_u64(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst) {
  *dst = *src;
}
}  // namespace

void exclusive_scan_u64_dev(uint64_t* d, uint64_t n, cudaStream_t s, uint64_t* total_dev) {
  if (n == 0) {
    SPMVK_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(uint64_t), s));
    return;
  }
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  TmpBuf<uint64_t> part(nb + 1, s);
  scan_tile_reduce<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(d, n, part.p);
  SPMVK_LAUNCH("scan_tile_reduce");
  scan_partials<<<1, kScanThreads, 0, s>>>(part.p, nb);
  SPMVK_LAUNCH("scan_partials");
  scan_tile_apply<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(d, n, part.p);
  SPMVK_LAUNCH("scan_tile_apply");
  copy_u64<<<1, 1, 0, s>>>(part.p + nb, total_dev);
  SPMVK_LAUNCH("copy_u64");
}

uint64_t exclusive_scan_u64(uint64_t* d, uint64_t n, cudaStream_t s) {
  if (n == 0) return 0;
  TmpBuf<uint64_t> tot(1, s);
  exclusive_scan_u64_dev(d, n, s, tot.p);
  uint64_t* slot = pinned_slot();
  SPMVK_CUDA(cudaMemcpyAsync(slot, tot.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  return slot[0];
}

std::mutex& host_bufs_mu() {
  static std::mutex m;
  return m;
}
std::map<void*, uint64_t>& host_bufs() {
  static std::map<void*, uint64_t> m;
  return m;
}

}  // namespace spmvk

extern "C" {

const char* spmvk_last_error(void) { return spmvk::last_error_cstr(); }

int spmvk_abi_version(void) { return SPMVK_ABI_VERSION; }

int spmvk_init(int device) {
  return spmvk::guarded([&] {
    spmvk::require_device();
    SPMVK_CUDA(cudaSetDevice(device));
    cudaDeviceProp p{};
    SPMVK_CUDA(cudaGetDeviceProperties(&p, device));
    if (p.major != 10)
      spmvk::fail(SPMVK_ECUDA, std::string("spmvk is built for sm_100a; device ") + p.name +
                                   " is sm_" + std::to_string(p.major * 10 + p.minor));
  });
}

int spmvk_host_alloc(uint64_t bytes, void** out) {
  return spmvk::guarded([&] {
    if (!out) spmvk::fail(SPMVK_EINVAL, "spmvk_host_alloc: null output pointer");
    *out = nullptr;
    spmvk::require_device();
    constexpr uint64_t kHuge = 2ull << 20;
    const uint64_t size = std::max<uint64_t>(kHuge, (bytes + kHuge - 1) / kHuge * kHuge);
    void* raw = mmap(nullptr, size + kHuge, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS,
                     -1, 0);
    if (raw == MAP_FAILED) spmvk::fail(SPMVK_ENOMEM, "spmvk_host_alloc: mmap failed");
    const uintptr_t r = reinterpret_cast<uintptr_t>(raw);
    const uintptr_t p = (r + kHuge - 1) / kHuge * kHuge;
    if (p > r) munmap(raw, p - r);  // trim to a 2 MB aligned range
    if (r + size + kHuge > p + size) munmap(reinterpret_cast<void*>(p + size), r + kHuge - p);
    void* q = reinterpret_cast<void*>(p);
    madvise(q, size, MADV_HUGEPAGE);  // advisory: fine if THP is off
    std::memset(q, 0, size);          // populate before page-locking
    const cudaError_t e = cudaHostRegister(q, size, cudaHostRegisterPortable |
                                                        cudaHostRegisterMapped);
    if (e != cudaSuccess) {
      munmap(q, size);
      spmvk::fail(SPMVK_ECUDA, std::string("spmvk_host_alloc: cudaHostRegister: ") +
                                   cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lk(spmvk::host_bufs_mu());
    spmvk::host_bufs()[q] = size;
    *out = q;
  });
}

int spmvk_host_free(void* p) {
  return spmvk::guarded([&] {
    if (!p) return;
    uint64_t size = 0;
    {
      std::lock_guard<std::mutex> lk(spmvk::host_bufs_mu());
      auto it = spmvk::host_bufs().find(p);
      if (it == spmvk::host_bufs().end())
        spmvk::fail(SPMVK_EINVAL, "spmvk_host_free: not a spmvk_host_alloc buffer");
      size = it->second;
      spmvk::host_bufs().erase(it);
    }
    SPMVK_CUDA(cudaHostUnregister(p));
    munmap(p, size);
  });
}

int spmvk_empty_cache(int device) {
  return spmvk::guarded([&] { spmvk::dev_cache_empty(device); });
}

int spmvk_stream_persist_x(void* stream, const void* x, uint64_t bytes, double hit_ratio,
                           uint64_t* granted) {
  return spmvk::guarded([&] {
    spmvk::require_device();
    int dev = 0, max_persist = 0, max_window = 0;
    SPMVK_CUDA(cudaGetDevice(&dev));
    SPMVK_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    SPMVK_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    cudaStreamAttrValue v{};
    const auto s = static_cast<cudaStream_t>(stream);
    uint64_t limit = 0;
    if (!x || bytes == 0) {  // reset: no window, persisting lines demoted, no carve-out
      v.accessPolicyWindow.num_bytes = 0;
      SPMVK_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
      SPMVK_CUDA(cudaCtxResetPersistingL2Cache());
      SPMVK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
    } else {
      if (!(hit_ratio > 0.0 && hit_ratio <= 1.0))
        spmvk::fail(SPMVK_EINVAL, "persist_x: hit_ratio must be in (0, 1]");
      limit = std::min<uint64_t>(bytes, static_cast<uint64_t>(max_persist));
      SPMVK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit));
      const uint64_t win = std::min<uint64_t>(bytes, static_cast<uint64_t>(max_window));
      v.accessPolicyWindow.base_ptr = const_cast<void*>(x);
      v.accessPolicyWindow.num_bytes = win;
      v.accessPolicyWindow.hitRatio =
          static_cast<float>(hit_ratio * std::min(1.0, static_cast<double>(limit) / win));
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      SPMVK_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
    }
    if (granted) *granted = limit;
  });
}

}  // extern "C"
