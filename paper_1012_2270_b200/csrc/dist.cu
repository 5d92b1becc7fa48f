// Fused distributed iterated SpMV over peer memory.
//
// The reference has no multi-GPU path; SURVEY §8e specifies one: contiguous,
// group-aligned row slabs, each rank computing y = A_slab x and
// x_{k+1} = y * 2^-4 for its rows, then an exchange of x (all-gather, or only
// the halo each slab reads).  Here the exchange is NOT a separate collective:
//
//   * every rank owns an exchange WINDOW in its HBM -- two full-length x
//     buffers (double-buffered: step k reads x[cur], writes x[1-cur]) and a
//     flag array -- exported with cudaIpcGetMemHandle and opened by every peer
//     (cudaIpcOpenMemHandle maps it through NVLink / NVSwitch), or shared
//     directly between GPUs driven by one process;
//   * the SpMV kernel's row epilogue (PeerEpi, rgcsr_spmv.cuh) stores
//     x_{k+1}[row] straight into the x[1-cur] buffer of every window whose
//     receive range covers the row: the all-gather (every peer gets the whole
//     slab) or the halo (a peer gets only the rows its slab reads) happens
//     inside the SpMV, tile by tile, as coalesced 8-byte stores over NVLink;
//   * one tiny barrier kernel per step (release-store of the step number into
//     every peer's flag slot, acquire-spin on our own slots) separates step k's
//     reads of x[cur] and remote writes into x[1-cur] from step k+1's.
//
// Accumulation order per row is the single-GPU kernel's, so x after any number
// of steps is bitwise the 1-GPU iterate (tests/test_gpu_dist.py).
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "common.cuh"
#include "rgcsr_spmv.cuh"

struct spmvk_window {
  uint64_t n = 0;  // x length (global rows, >= global columns)
  int prec = SPMVK_F64;
  spmvk::DevBuf<unsigned char> mem;  // [x0 | x1 | flags]
  // Step state lives with the window, not the dist handle: the flags in HBM
  // are monotonic, so a second handle opened on this window must continue
  // the step count (every rank steps equally often, so the counts agree).
  mutable int cur = 0;
  mutable unsigned long long epoch = 0;
  uint64_t x_bytes() const { return (n * prec + 255) / 256 * 256; }
  unsigned char* x(int b) const { return mem.p + b * x_bytes(); }
  unsigned long long* flags() const {
    return reinterpret_cast<unsigned long long*>(mem.p + 2 * x_bytes());
  }
};

struct spmvk_dist {
  int rank = 0, world = 1, prec = SPMVK_F64;
  uint64_t n = 0;
  const spmvk_window* own = nullptr;
  unsigned char* base[spmvk::kMaxPeers] = {};  // window base of every rank
  bool ipc[spmvk::kMaxPeers] = {};             // opened with cudaIpcOpenMemHandle
  uint64_t row_begin = 0, row_end = 0;
  uint64_t lo[spmvk::kMaxPeers] = {}, hi[spmvk::kMaxPeers] = {};  // rows each rank receives
  uint64_t timeout_ns = 30ull * 1000 * 1000 * 1000;  // barrier wait bound (set_timeout_ms)
  ~spmvk_dist() {
    for (int q = 0; q < world; ++q)
      if (ipc[q] && base[q]) cudaIpcCloseMemHandle(base[q]);
  }
};

namespace spmvk {
namespace {

constexpr uint64_t kFlagBytes = 64 * sizeof(unsigned long long);
// Flag word kFlagStatus of a window: 0, or 1 + the rank a barrier of this
// window's owner gave up waiting for (spmvk_dist_status reads it).
constexpr int kFlagStatus = 63;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct FlagSet {
  unsigned long long* remote[kMaxPeers];  // remote[q] = &flags_of_rank_q[my rank]
};

// Thread q: publish "finished step `epoch`" into rank q's window, then wait
// until rank q has published the same into ours.  The previous kernel on this
// stream (the SpMV, including its remote stores) completed before this one
// started; the system-scope fence + release make those stores visible to the
// peer before it sees the flag.
// The wait is bounded: after timeout_ns without the peer's flag the barrier
// records 1 + q in the window's status word and returns, and every later
// barrier of this window returns at once -- a dead peer turns into an error
// (spmvk_dist_status -> SPMVK_ENCCL), not a hung GPU.
__global__ void dist_barrier(FlagSet fs, unsigned long long* mine, int world,
                             unsigned long long epoch, uint64_t timeout_ns) {
  const int q = threadIdx.x;
  if (q < world) {
    __threadfence_system();
    st_release_sys(fs.remote[q], epoch);
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(mine + q) < epoch) {
      if (*(volatile unsigned long long*)(mine + kFlagStatus)) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicCAS(mine + kFlagStatus, 0ull, (unsigned long long)(q + 1));
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_dist(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, uint32_t long_cut,
    PeerEpi<T> epi) {
  lite_tiles_epi<T, U>(0, (rows + 255) / 256, rows, G, g_shift, gp, lens, values, columns,
                              x, long_cut, epi);
}

// Same step with the group-uniform walk (rgcsr_spmv_grp) for slabs without
// long rows and with <= 10 % padding -- the stencil slabs of config 5.
template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_dist_grp(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, uint32_t /*long_cut*/,
    PeerEpi<T> epi) {
  grp_tiles_epi<T, U, true, true, PeerEpi<T>>(rows, G, g_shift, gp, lens, values, columns, x, epi);
}

template <class T>
__global__ void __launch_bounds__(256) rgcsr_spmv_long_dist(
    uint32_t nlong, const uint32_t* __restrict__ long_rows, uint32_t rows, uint32_t G,
    int g_shift, const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    PeerEpi<T> epi) {
  long_rows_epi<T>(nlong, long_rows, rows, G, g_shift, gp, lens, values, columns, x, epi);
}

void check_world(int rank, int world) {
  if (world < 1 || world > kMaxPeers)
    fail(SPMVK_EINVAL, "dist: world size must be in [1, " + std::to_string(kMaxPeers) + "]");
  if (rank < 0 || rank >= world) fail(SPMVK_EINVAL, "dist: rank outside [0, world)");
}

spmvk_dist* new_dist(const spmvk_window* own, int rank, int world) {
  if (!own) fail(SPMVK_EINVAL, "dist: null window");
  check_world(rank, world);
  auto* d = new spmvk_dist();
  d->rank = rank;
  d->world = world;
  d->prec = own->prec;
  d->n = own->n;
  d->own = own;
  d->base[rank] = own->mem.p;
  return d;
}

void check_open(const spmvk_dist* d, const char* who) {
  for (int q = 0; q < d->world; ++q)
    if (!d->base[q]) fail(SPMVK_EINVAL, std::string(who) + ": window of rank " +
                                            std::to_string(q) + " not opened");
}

// Routing of this rank's next-buffer stores: own rows to x[1-cur] of the own
// window, and every row a peer receives to that peer's x[1-cur].
template <class T>
PeerEpi<T> peer_routing(const spmvk_dist* d, T* y, T scale) {
  const uint64_t xb = d->own->x_bytes();
  const int cur = d->own->cur;
  PeerEpi<T> epi{};
  epi.y = y;
  epi.scale = scale;
  epi.row0 = static_cast<uint32_t>(d->row_begin);
  epi.self = reinterpret_cast<T*>(d->base[d->rank] + (1 - cur) * xb);
  // interior: the slab rows no peer receives (halo plans put the peers'
  // ranges at the slab edges); rows there take the single self store
  uint64_t ilo = d->row_begin, ihi = d->row_end;
  int n = 0;
  for (int q = 0; q < d->world; ++q) {
    if (q == d->rank) continue;
    const uint64_t lo = std::max(d->lo[q], d->row_begin), hi = std::min(d->hi[q], d->row_end);
    if (lo >= hi) continue;
    epi.ps.dst[n] = reinterpret_cast<T*>(d->base[q] + (1 - cur) * xb);
    epi.ps.lo[n] = static_cast<uint32_t>(lo);
    epi.ps.hi[n] = static_cast<uint32_t>(hi);
    ++n;
    if (lo <= ilo) ilo = std::max(ilo, hi);
    else if (hi >= ihi) ihi = std::min(ihi, lo);
    else ihi = ilo;  // a range strictly inside the slab: no fast path
  }
  epi.ps.n = n;
  epi.int_lo = static_cast<uint32_t>(ilo);
  epi.int_hi = static_cast<uint32_t>(std::max(ilo, ihi));
  return epi;
}

// End of a step: flip the window's current buffer and (optionally) run the
// flag barrier that orders this step's remote stores before the next step.
void finish_step(spmvk_dist* d, int barrier, cudaStream_t s) {
  const uint64_t xb = d->own->x_bytes();
  d->own->cur = 1 - d->own->cur;
  if (barrier) {
    const unsigned long long epoch = ++d->own->epoch;
    FlagSet fs{};
    for (int q = 0; q < d->world; ++q)
      fs.remote[q] = reinterpret_cast<unsigned long long*>(d->base[q] + 2 * xb) + d->rank;
    dist_barrier<<<1, 32, 0, s>>>(fs, d->own->flags(), d->world, epoch, d->timeout_ns);
    SPMVK_LAUNCH("dist_barrier");
  }
}

template <class T>
void dist_step(spmvk_dist* d, const spmvk_rgcsr* a, T scale, T* y, int barrier, cudaStream_t s) {
  if (!d || !a) fail(SPMVK_EINVAL, "dist_step: null handle");
  if (d->prec != static_cast<int>(sizeof(T)) || a->prec != d->prec)
    fail(SPMVK_EINVAL, "dist_step: precision differs from the window / entry point");
  if (d->row_end < d->row_begin || a->rows != d->row_end - d->row_begin)
    fail(SPMVK_EINVAL, "dist_step: slab rows differ from the rows set with spmvk_dist_set_rows");
  if (a->cols > d->n || d->row_end > d->n)
    fail(SPMVK_EINVAL, "dist_step: slab reaches past the window length");
  check_open(d, "dist_step");
  const uint64_t xb = d->own->x_bytes();
  const T* x = reinterpret_cast<const T*>(d->base[d->rank] + d->own->cur * xb);
  const PeerEpi<T> epi = peer_routing<T>(d, y, scale);
  if (a->rows) {
    const uint32_t G = static_cast<uint32_t>(std::min<uint64_t>(a->group_size, 0xffffffffull));
    const int sh = pow2_shift(a->group_size);
    const uint32_t long_cut = a->n_long ? a->long_cut : 0xffffffffu;
    constexpr bool f64 = sizeof(T) == 8;
    // kernel choice as rgcsr.cu's auto_k2: group-uniform walk for regular slabs
    auto kern = f64 ? rgcsr_spmv_dist<T, 8, 5> : rgcsr_spmv_dist<T, 4, 8>;
    if (!a->n_long && a->slots * 10 <= a->nnz * 11) {
      if (2 * a->slots <= 11 * a->rows) kern = rgcsr_spmv_dist_grp<T, 6, 5>;
      else if constexpr (f64) kern = rgcsr_spmv_dist_grp<T, 8, 4>;
      else kern = a->slots <= 12 * a->rows ? rgcsr_spmv_dist_grp<T, 8, 5>
                                           : rgcsr_spmv_dist_grp<T, 7, 5>;
    }
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    kern<<<persistent_grid((a->rows + 255) / 256, per_sm > 0 ? per_sm : 1), 256, 0, s>>>(
        static_cast<uint32_t>(a->rows), G, sh, a->group_pointers.p, a->row_lengths.p,
        reinterpret_cast<const T*>(a->values.p), a->columns.p, x, long_cut, epi);
    SPMVK_LAUNCH("rgcsr_spmv_dist");
    if (a->n_long) {
      rgcsr_spmv_long_dist<T><<<persistent_grid((a->n_long + 7) / 8, 8), 256, 0, s>>>(
          static_cast<uint32_t>(a->n_long), a->long_rows.p, static_cast<uint32_t>(a->rows), G, sh,
          a->group_pointers.p, a->row_lengths.p, reinterpret_cast<const T*>(a->values.p),
          a->columns.p, x, epi);
      SPMVK_LAUNCH("rgcsr_spmv_long_dist");
    }
  }
  finish_step(d, barrier, s);
}

// Distributed CG's direction update with the p exchange fused in (the
// compute step followed by a collective, as one kernel): p_new = r + beta
// p_old for this rank's rows (beta = rr_new / rr from device memory; p_old
// read from x[cur] of the own window), stored into x[1-cur] of the own window
// and of every peer whose receive range covers the row -- the halo of p
// travels as NVLink stores, no all-gather.  Then rr = rr_new, the flip and
// the flag barrier.  The arithmetic is cg_direction's (cg.cu), so at world
// size 1 the iterate is bitwise the single-GPU solver's.
__global__ void __launch_bounds__(256) dist_cg_direction(uint32_t n,
                                                         const double* __restrict__ r,
                                                         const double* __restrict__ p_old,
                                                         const double* __restrict__ rr,
                                                         const double* __restrict__ rr_new,
                                                         PeerEpi<double> route) {
  const double beta = *rr_new / *rr;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    const double v = r[i] + beta * p_old[i];
    const uint32_t gr = route.row0 + i;
    route.self[gr] = v;
    if (gr >= route.int_lo && gr < route.int_hi) continue;
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q < route.ps.n && gr >= route.ps.lo[q] && gr < route.ps.hi[q]) route.ps.dst[q][gr] = v;
  }
}

__global__ void dist_copy_scalar(const double* __restrict__ src, double* __restrict__ dst) {
  *dst = *src;
}

void dist_cg_direction_f64(spmvk_dist* d, const double* r, double* rr, const double* rr_new,
                           int barrier, cudaStream_t s) {
  if (!d || !r || !rr || !rr_new) fail(SPMVK_EINVAL, "dist_cg_direction: null argument");
  if (d->prec != SPMVK_F64) fail(SPMVK_EINVAL, "dist_cg_direction: fp64 window required");
  if (d->row_end < d->row_begin || d->row_end > d->n)
    fail(SPMVK_EINVAL, "dist_cg_direction: rows not set (spmvk_dist_set_rows)");
  check_open(d, "dist_cg_direction");
  const uint64_t rows = d->row_end - d->row_begin;
  const uint64_t xb = d->own->x_bytes();
  const double* p_old =
      reinterpret_cast<const double*>(d->base[d->rank] + d->own->cur * xb) + d->row_begin;
  const PeerEpi<double> route = peer_routing<double>(d, nullptr, 1.0);
  if (rows) {
    // grid of cg.cu's kDotBlocks (592) CTAs: same index mapping per thread
    dist_cg_direction<<<592, 256, 0, s>>>(static_cast<uint32_t>(rows), r, p_old, rr, rr_new,
                                          route);
    SPMVK_LAUNCH("dist_cg_direction");
  }
  dist_copy_scalar<<<1, 1, 0, s>>>(rr_new, rr);
  SPMVK_LAUNCH("dist_copy_scalar");
  finish_step(d, barrier, s);
}

}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_window_create(uint64_t n, int prec, spmvk_window** out) {
  return guarded([&] {
    require_device();
    if (!out) fail(SPMVK_EINVAL, "window_create: null output");
    if (prec != SPMVK_F32 && prec != SPMVK_F64) fail(SPMVK_EINVAL, "window_create: bad precision");
    if (n > 0xffffffffull) fail(SPMVK_ERANGE, "window_create: length exceeds uint32 indices");
    auto w = std::make_unique<spmvk_window>();
    w->n = n;
    w->prec = prec;
    w->mem.alloc(2 * w->x_bytes() + kFlagBytes);
    SPMVK_CUDA(cudaMemset(w->mem.p, 0, 2 * w->x_bytes() + kFlagBytes));
    *out = w.release();
  });
}

int spmvk_window_ipc_handle(const spmvk_window* w, unsigned char* out) {
  return guarded([&] {
    if (!w || !out) fail(SPMVK_EINVAL, "window_ipc_handle: null argument");
    cudaIpcMemHandle_t h;
    SPMVK_CUDA(cudaIpcGetMemHandle(&h, w->mem.p));
    std::memcpy(out, &h, sizeof(h));
  });
}

int spmvk_window_x(const spmvk_window* w, int buffer, void** out) {
  return guarded([&] {
    if (!w || !out) fail(SPMVK_EINVAL, "window_x: null argument");
    if (buffer != 0 && buffer != 1) fail(SPMVK_EINVAL, "window_x: buffer must be 0 or 1");
    *out = w->x(buffer);
  });
}

void spmvk_window_destroy(spmvk_window* w) { delete w; }

int spmvk_dist_open(const spmvk_window* own, int rank, int world, const unsigned char* handles,
                    spmvk_dist** out) {
  return guarded([&] {
    require_device();
    if (!out || (!handles && world > 1)) fail(SPMVK_EINVAL, "dist_open: null argument");
    std::unique_ptr<spmvk_dist> d(new_dist(own, rank, world));
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + q * sizeof(cudaIpcMemHandle_t), sizeof(h));
      void* p = nullptr;
      SPMVK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      d->base[q] = static_cast<unsigned char*>(p);
      d->ipc[q] = true;
    }
    *out = d.release();
  });
}

int spmvk_dist_open_local(const spmvk_window* const* windows, int rank, int world,
                          spmvk_dist** out) {
  return guarded([&] {
    require_device();
    if (!out || !windows) fail(SPMVK_EINVAL, "dist_open_local: null argument");
    check_world(rank, world);
    std::unique_ptr<spmvk_dist> d(new_dist(windows[rank], rank, world));
    int dev = 0;
    SPMVK_CUDA(cudaGetDevice(&dev));
    for (int q = 0; q < world; ++q) {
      if (!windows[q]) fail(SPMVK_EINVAL, "dist_open_local: null window");
      if (windows[q]->n != windows[rank]->n || windows[q]->prec != windows[rank]->prec)
        fail(SPMVK_EINVAL, "dist_open_local: windows differ in length or precision");
      cudaPointerAttributes at{};
      SPMVK_CUDA(cudaPointerGetAttributes(&at, windows[q]->mem.p));
      if (at.device != dev) {  // a window on another GPU of this process: map it
        int can = 0;
        SPMVK_CUDA(cudaDeviceCanAccessPeer(&can, dev, at.device));
        if (!can)
          fail(SPMVK_ENCCL, "dist_open_local: GPU " + std::to_string(dev) +
                                " cannot access GPU " + std::to_string(at.device) +
                                " peer-to-peer (use the NCCL exchange)");
        const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else SPMVK_CUDA(e);
      }
      d->base[q] = windows[q]->mem.p;
    }
    *out = d.release();
  });
}

int spmvk_dist_set_rows(spmvk_dist* d, uint64_t row_begin, uint64_t row_end,
                        const uint64_t* receive_ranges) {
  return guarded([&] {
    if (!d || !receive_ranges) fail(SPMVK_EINVAL, "dist_set_rows: null argument");
    if (row_begin > row_end || row_end > d->n)
      fail(SPMVK_EINVAL, "dist_set_rows: slab rows outside the window");
    d->row_begin = row_begin;
    d->row_end = row_end;
    for (int q = 0; q < d->world; ++q) {
      d->lo[q] = receive_ranges[2 * q];
      d->hi[q] = receive_ranges[2 * q + 1];
    }
  });
}

int spmvk_dist_step_f64(spmvk_dist* d, const spmvk_rgcsr* slab, double scale, double* y,
                        int barrier, void* stream) {
  return guarded([&] { dist_step<double>(d, slab, scale, y, barrier, as_stream(stream)); });
}

int spmvk_dist_step_f32(spmvk_dist* d, const spmvk_rgcsr* slab, float scale, float* y,
                        int barrier, void* stream) {
  return guarded([&] { dist_step<float>(d, slab, scale, y, barrier, as_stream(stream)); });
}

int spmvk_dist_cg_direction_f64(spmvk_dist* d, const double* r_local, double* rr,
                                const double* rr_new, int barrier, void* stream) {
  return guarded([&] { dist_cg_direction_f64(d, r_local, rr, rr_new, barrier, as_stream(stream)); });
}

int spmvk_dist_set_timeout_ms(spmvk_dist* d, uint64_t ms) {
  return guarded([&] {
    if (!d) fail(SPMVK_EINVAL, "dist_set_timeout_ms: null handle");
    if (ms == 0) fail(SPMVK_EINVAL, "dist_set_timeout_ms: timeout must be positive");
    d->timeout_ns = ms * 1000ull * 1000ull;
  });
}

int spmvk_dist_status(const spmvk_dist* d, void* stream) {
  return guarded([&] {
    if (!d) fail(SPMVK_EINVAL, "dist_status: null handle");
    unsigned long long v = 0;
    cudaStream_t s = as_stream(stream);
    SPMVK_CUDA(cudaMemcpyAsync(&v, d->own->flags() + kFlagStatus, sizeof(v),
                               cudaMemcpyDeviceToHost, s));
    SPMVK_CUDA(cudaStreamSynchronize(s));
    if (v)
      fail(SPMVK_ENCCL, "dist barrier of rank " + std::to_string(d->rank) +
                            " timed out waiting for rank " + std::to_string(v - 1) +
                            " (peer dead or not stepping)");
  });
}

int spmvk_dist_current(const spmvk_dist* d, int* buffer) {
  return guarded([&] {
    if (!d || !buffer) fail(SPMVK_EINVAL, "dist_current: null argument");
    *buffer = d->own->cur;
  });
}

void spmvk_dist_destroy(spmvk_dist* d) { delete d; }

}  // extern "C"
