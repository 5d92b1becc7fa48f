// Multi-GPU boundary in host C++ (SURVEY §8b "spmvk_dist_*: init NCCL comms
// over P GPUs, partition, iterated SpMV with all-gather / halo"; §8e).
//
// The reference has no multi-GPU path.  This file is the host side of the
// row-slab partition behind the C-ABI, with no torch.distributed in it:
//
//  * planning (pure host code, no device needed): equal group-aligned slabs,
//    slot-balanced cuts for skewed matrices, the fused path's receive ranges
//    and the halo's per-peer send / receive lists;
//  * NCCL communicators: ncclCommInitRank (one process per GPU, the unique id
//    exchanged out of band) or ncclCommInitAll (one process driving several
//    GPUs);
//  * the NCCL iterated product x_{k+1} = (A_slab x_k) * scale with either an
//    in-place ncclAllGather of every rank's slab of x_{k+1} (SURVEY §8e's
//    spec-literal baseline: equal slab sizes keep the counts equal) or grouped
//    ncclSend / ncclRecv of only the column ranges each slab reads (halo).
//    The scale is fused into the SpMV's epilogue; the exchange is stream
//    ordered behind it.  Double-buffered x, so step k+1's writes never race
//    step k's reads.  Every row keeps the reference's accumulation order, so
//    the iterate is bitwise the one-GPU iterate.
//
// NCCL is bound at run time (dlopen "libnccl.so.2", or SPMVK_NCCL_LIB):
// inside a PyTorch process that is the NCCL torch already loaded (one NCCL
// per process); a plain C++ host gets the system library.  nccl.h supplies
// the types only.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace spmvk {
namespace {

struct NcclApi {
  void* so = nullptr;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
  decltype(&ncclCommUserRank) CommUserRank = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
};

template <class F>
void bind(NcclApi& a, F*& f, const char* name) {
  f = reinterpret_cast<F*>(dlsym(a.so, name));
  if (!f && a.why.empty()) a.why = std::string("symbol ") + name + " missing";
}

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("SPMVK_NCCL_LIB");
    a.so = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!a.so) {
      const char* e = dlerror();
      a.why = e ? e : "dlopen failed";
      return a;
    }
    bind(a, a.GetUniqueId, "ncclGetUniqueId");
    bind(a, a.CommInitRank, "ncclCommInitRank");
    bind(a, a.CommInitAll, "ncclCommInitAll");
    bind(a, a.CommDestroy, "ncclCommDestroy");
    bind(a, a.CommCount, "ncclCommCount");
    bind(a, a.CommUserRank, "ncclCommUserRank");
    bind(a, a.AllGather, "ncclAllGather");
    bind(a, a.Send, "ncclSend");
    bind(a, a.Recv, "ncclRecv");
    bind(a, a.GroupStart, "ncclGroupStart");
    bind(a, a.GroupEnd, "ncclGroupEnd");
    bind(a, a.GetErrorString, "ncclGetErrorString");
    bind(a, a.GetVersion, "ncclGetVersion");
    return a;
  }();
  if (!api.so || !api.why.empty())
    fail(SPMVK_ENCCL, "NCCL unavailable (libnccl.so.2): " + api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(SPMVK_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---------------------------------------------------------------- planning
// Equal, group-aligned slabs: S = ceil(groups / P) * G rows each (the last
// ones may be short or empty); bounds[p] = min(rows, p * S).
uint64_t plan_slabs(uint64_t rows, uint64_t G, int parts, uint64_t* bounds) {
  if (G == 0 || parts <= 0) fail(SPMVK_EINVAL, "plan_slabs: group size and part count must be positive");
  const uint64_t groups = (rows + G - 1) / G;
  const uint64_t S = (groups + parts - 1) / parts * G;
  for (int p = 0; p <= parts; ++p) bounds[p] = std::min<uint64_t>(rows, S * p);
  return S;
}

// Slot-balanced, group-aligned cuts: cut p is the first group boundary
// where the running slot count reaches p / P of the total (exact integer
// comparison slots * P >= total * p).
void plan_slabs_weighted(const uint32_t* lens, uint64_t rows, uint64_t G, int parts,
                         uint64_t* bounds) {
  if (G == 0 || parts <= 0)
    fail(SPMVK_EINVAL, "plan_slabs_weighted: group size and part count must be positive");
  const uint64_t groups = (rows + G - 1) / G;
  std::vector<uint64_t> cum(groups);
  uint64_t acc = 0;
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t r0 = g * G, s = std::min(G, rows - r0);
    uint32_t w = 0;
    for (uint64_t t = 0; t < s; ++t) w = std::max(w, lens[r0 + t]);
    acc += s * w;
    cum[g] = acc;
  }
  const unsigned __int128 total = acc;
  bounds[0] = 0;
  for (int p = 1; p < parts; ++p) {
    uint64_t cut = 0;
    if (total) {
      const unsigned __int128 need = total * static_cast<unsigned>(p);
      // first g with cum[g] * parts >= total * p
      uint64_t lo = 0, hi = groups;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (static_cast<unsigned __int128>(cum[mid]) * static_cast<unsigned>(parts) >= need)
          hi = mid;
        else
          lo = mid + 1;
      }
      cut = (lo + 1) * G;
    }
    bounds[p] = std::min(rows, std::max(bounds[p - 1], cut));
  }
  bounds[parts] = rows;
}

// Receive range [lo, hi) of every rank: the whole x (all-gather), or the span
// of its own rows and the columns its slab reads (halo).  col_ranges[2q],
// [2q+1] = (cmin, cmax), cmin > cmax for a slab without entries.
void plan_receive(int parts, const uint64_t* bounds, const uint64_t* col_ranges, int mode,
                  uint64_t* receive) {
  const uint64_t n = parts ? bounds[parts] : 0;
  for (int q = 0; q < parts; ++q) {
    if (mode == SPMVK_EXCHANGE_ALLGATHER) {
      receive[2 * q] = 0;
      receive[2 * q + 1] = n;
      continue;
    }
    uint64_t lo = bounds[q], hi = bounds[q + 1];
    const uint64_t cmin = col_ranges[2 * q], cmax = col_ranges[2 * q + 1];
    if (cmin <= cmax) {
      lo = std::min(lo, cmin);
      hi = std::max(hi, cmax + 1);
    }
    receive[2 * q] = lo < hi ? lo : 0;
    receive[2 * q + 1] = lo < hi ? hi : 0;
  }
}

// Halo lists of `rank`: recv[k] = (peer, c0, c1) -- the columns this slab
// reads that peer owns; send[k] = (peer, c0, c1) -- this slab's rows the
// peer reads.  Both ascending by peer, so matching send / recv pairs post in
// the same order on both sides.
void plan_halo(int rank, int parts, const uint64_t* bounds, const uint64_t* col_ranges,
               std::vector<std::array<uint64_t, 3>>* recv,
               std::vector<std::array<uint64_t, 3>>* send) {
  const uint64_t mb = bounds[rank], me = bounds[rank + 1];
  const uint64_t mlo = col_ranges[2 * rank], mhi = col_ranges[2 * rank + 1];
  for (int q = 0; q < parts; ++q) {
    if (q == rank) continue;
    const uint64_t qb = bounds[q], qe = bounds[q + 1];
    if (mlo <= mhi) {
      const uint64_t c0 = std::max(mlo, qb), c1 = std::min(mhi + 1, qe);
      if (c0 < c1) recv->push_back({static_cast<uint64_t>(q), c0, c1});
    }
    const uint64_t qlo = col_ranges[2 * q], qhi = col_ranges[2 * q + 1];
    if (qlo <= qhi) {
      const uint64_t c0 = std::max(qlo, mb), c1 = std::min(qhi + 1, me);
      if (c0 < c1) send->push_back({static_cast<uint64_t>(q), c0, c1});
    }
  }
}

// Column range [min, max] an RgCSR (slab) reads: first and last slot of every
// row (columns ascend along a row).  out = {UINT32_MAX, 0} initially.
__global__ void rgcsr_column_range(uint32_t rows, uint32_t G, const uint32_t* __restrict__ gp,
                                   const uint32_t* __restrict__ lens,
                                   const uint32_t* __restrict__ columns,
                                   unsigned* __restrict__ out) {
  unsigned lo = 0xffffffffu, hi = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const uint32_t len = lens[r];
    if (!len) continue;
    const uint32_t g = r / G, s = min(G, rows - g * G), base = gp[g] + (r - g * G);
    lo = min(lo, columns[base]);
    hi = max(hi, columns[base + (len - 1) * s]);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

}  // namespace
}  // namespace spmvk

struct spmvk_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  ~spmvk_comm() {
    if (comm) spmvk::nccl().CommDestroy(comm);
  }
};

struct spmvk_nccl_iter {
  spmvk_comm* comm = nullptr;
  const spmvk_rgcsr* a = nullptr;
  int prec = SPMVK_F64, mode = SPMVK_EXCHANGE_ALLGATHER;
  uint64_t row_begin = 0, row_end = 0, S = 0, n = 0, n_alloc = 0;
  spmvk::DevBuf<unsigned char> x[2];
  int cur = 0;
  std::vector<std::array<uint64_t, 3>> send, recv;
  uint64_t recv_entries = 0;
};

namespace spmvk {
namespace {

ncclDataType_t nccl_type(int prec) { return prec == SPMVK_F64 ? ncclFloat64 : ncclFloat32; }

spmvk_nccl_iter* iter_create(spmvk_comm* c, const spmvk_rgcsr* a, uint64_t row_begin,
                             uint64_t row_end, uint64_t slab_rows, uint64_t n, int mode) {
  if (!c || !a) fail(SPMVK_EINVAL, "nccl_iter_create: null handle");
  if (mode != SPMVK_EXCHANGE_ALLGATHER && mode != SPMVK_EXCHANGE_HALO)
    fail(SPMVK_EINVAL, "nccl_iter_create: mode must be SPMVK_EXCHANGE_ALLGATHER or _HALO");
  if (row_begin > row_end || a->rows != row_end - row_begin)
    fail(SPMVK_EINVAL, "nccl_iter_create: slab rows differ from the RgCSR's rows");
  if (row_end > n || a->cols > n)
    fail(SPMVK_EINVAL, "nccl_iter_create: slab reaches past the global length");
  if (mode == SPMVK_EXCHANGE_ALLGATHER &&
      (slab_rows == 0 || row_begin != slab_rows * c->rank ||
       row_end != std::min(n, slab_rows * (c->rank + 1))))
    fail(SPMVK_EINVAL, "nccl_iter_create: the all-gather needs the equal slabs of "
                       "spmvk_plan_slabs (row_begin = rank * slab_rows)");
  auto it = std::make_unique<spmvk_nccl_iter>();
  it->comm = c;
  it->a = a;
  it->prec = a->prec;
  it->mode = mode;
  it->row_begin = row_begin;
  it->row_end = row_end;
  it->S = slab_rows;
  it->n = n;
  const uint64_t npad = mode == SPMVK_EXCHANGE_ALLGATHER ? slab_rows * c->world : n;
  it->n_alloc = std::max(n, npad);
  for (auto& b : it->x) {
    b.alloc(it->n_alloc * it->prec);
    SPMVK_CUDA(cudaMemset(b.p, 0, it->n_alloc * it->prec));
  }
  // every rank's (row_begin, row_end, cmin, cmax), gathered over NCCL
  DevBuf<unsigned> cr(2);
  const unsigned init[2] = {0xffffffffu, 0u};
  SPMVK_CUDA(cudaMemcpy(cr.p, init, sizeof(init), cudaMemcpyHostToDevice));
  if (a->rows) {
    rgcsr_column_range<<<persistent_grid((a->rows + 255) / 256, 8), 256>>>(
        static_cast<uint32_t>(a->rows), static_cast<uint32_t>(a->group_size),
        a->group_pointers.p, a->row_lengths.p, a->columns.p, cr.p);
    SPMVK_LAUNCH("rgcsr_column_range");
  }
  unsigned crh[2];
  SPMVK_CUDA(cudaMemcpy(crh, cr.p, sizeof(crh), cudaMemcpyDeviceToHost));
  const uint64_t mine[4] = {row_begin, row_end, crh[0] <= crh[1] ? crh[0] : 1ull,
                            crh[0] <= crh[1] ? crh[1] : 0ull};
  std::vector<uint64_t> all(4 * c->world);
  if (c->world == 1) {
    std::copy(mine, mine + 4, all.begin());
  } else {
    DevBuf<uint64_t> d(4 * c->world);
    SPMVK_CUDA(cudaMemcpy(d.p + 4 * c->rank, mine, sizeof(mine), cudaMemcpyHostToDevice));
    cudaStream_t s = nullptr;
    SPMVK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const ncclResult_t r = nccl().AllGather(d.p + 4 * c->rank, d.p, 4, ncclUint64, c->comm, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    nccl_check(r, "nccl_iter_create: ncclAllGather of the slab plans");
    SPMVK_CUDA(e);
    SPMVK_CUDA(cudaMemcpy(all.data(), d.p, 8 * all.size(), cudaMemcpyDeviceToHost));
  }
  std::vector<uint64_t> bounds(c->world + 1), ranges(2 * c->world);
  for (int q = 0; q < c->world; ++q) {
    bounds[q] = all[4 * q];
    ranges[2 * q] = all[4 * q + 2];
    ranges[2 * q + 1] = all[4 * q + 3];
    if (q + 1 < c->world && all[4 * q + 1] != all[4 * (q + 1)])
      fail(SPMVK_EINVAL, "nccl_iter_create: the ranks' slabs are not contiguous in rank order");
  }
  bounds[c->world] = all[4 * (c->world - 1) + 1];
  if (mode == SPMVK_EXCHANGE_HALO) {
    plan_halo(c->rank, c->world, bounds.data(), ranges.data(), &it->recv, &it->send);
    for (const auto& r : it->recv) it->recv_entries += r[2] - r[1];
  } else {
    it->recv_entries = npad - slab_rows;
  }
  return it.release();
}

template <class T>
void iter_step(spmvk_nccl_iter* it, T scale, T* y, cudaStream_t s) {
  if (!it) fail(SPMVK_EINVAL, "nccl_iter_step: null handle");
  if (it->prec != static_cast<int>(sizeof(T)))
    fail(SPMVK_EINVAL, "nccl_iter_step: precision differs from the slab");
  const T* xc = reinterpret_cast<const T*>(it->x[it->cur].p);
  T* xn = reinterpret_cast<T*>(it->x[1 - it->cur].p);
  const spmvk_rgcsr* a = it->a;
  int rc;
  if constexpr (sizeof(T) == 8)
    rc = spmvk_rgcsr_spmv_scaled_f64(a, xc, a->cols, y, a->rows, xn + it->row_begin, scale, s);
  else
    rc = spmvk_rgcsr_spmv_scaled_f32(a, xc, a->cols, y, a->rows, xn + it->row_begin, scale, s);
  if (rc != SPMVK_OK) fail(rc, std::string("nccl_iter_step: ") + spmvk_last_error());
  spmvk_comm* c = it->comm;
  if (c->world > 1) {
    const ncclDataType_t dt = nccl_type(it->prec);
    auto& N = nccl();
    if (it->mode == SPMVK_EXCHANGE_ALLGATHER) {
      nccl_check(N.AllGather(xn + it->S * c->rank, xn, it->S, dt, c->comm, s),
                 "ncclAllGather of x");
    } else {
      nccl_check(N.GroupStart(), "ncclGroupStart");
      ncclResult_t r = ncclSuccess;
      for (const auto& v : it->recv)
        if (r == ncclSuccess)
          r = N.Recv(xn + v[1], v[2] - v[1], dt, static_cast<int>(v[0]), c->comm, s);
      for (const auto& v : it->send)
        if (r == ncclSuccess)
          r = N.Send(xn + v[1], v[2] - v[1], dt, static_cast<int>(v[0]), c->comm, s);
      const ncclResult_t e = N.GroupEnd();
      nccl_check(r, "ncclSend / ncclRecv of the x halo");
      nccl_check(e, "ncclGroupEnd");
    }
  }
  it->cur = 1 - it->cur;
}

}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_plan_slabs(uint64_t rows, uint64_t group_size, int parts, uint64_t* bounds,
                     uint64_t* slab_rows) {
  return guarded([&] {
    if (!bounds) fail(SPMVK_EINVAL, "plan_slabs: null bounds");
    const uint64_t S = plan_slabs(rows, group_size, parts, bounds);
    if (slab_rows) *slab_rows = S;
  });
}

int spmvk_plan_slabs_weighted(const uint32_t* row_lengths, uint64_t rows, uint64_t group_size,
                              int parts, uint64_t* bounds) {
  return guarded([&] {
    if (!bounds || (!row_lengths && rows)) fail(SPMVK_EINVAL, "plan_slabs_weighted: null argument");
    plan_slabs_weighted(row_lengths, rows, group_size, parts, bounds);
  });
}

int spmvk_plan_receive(int parts, const uint64_t* bounds, const uint64_t* column_ranges, int mode,
                       uint64_t* receive) {
  return guarded([&] {
    if (parts <= 0 || !bounds || !receive || (!column_ranges && mode == SPMVK_EXCHANGE_HALO))
      fail(SPMVK_EINVAL, "plan_receive: bad argument");
    if (mode != SPMVK_EXCHANGE_ALLGATHER && mode != SPMVK_EXCHANGE_HALO)
      fail(SPMVK_EINVAL, "plan_receive: mode must be SPMVK_EXCHANGE_ALLGATHER or _HALO");
    plan_receive(parts, bounds, column_ranges, mode, receive);
  });
}

int spmvk_plan_halo(int rank, int parts, const uint64_t* bounds, const uint64_t* column_ranges,
                    uint64_t* recv, int* n_recv, uint64_t* send, int* n_send) {
  return guarded([&] {
    if (parts <= 0 || rank < 0 || rank >= parts || !bounds || !column_ranges || !recv ||
        !send || !n_recv || !n_send)
      fail(SPMVK_EINVAL, "plan_halo: bad argument");
    std::vector<std::array<uint64_t, 3>> rv, sv;
    plan_halo(rank, parts, bounds, column_ranges, &rv, &sv);
    for (size_t k = 0; k < rv.size(); ++k) std::copy(rv[k].begin(), rv[k].end(), recv + 3 * k);
    for (size_t k = 0; k < sv.size(); ++k) std::copy(sv[k].begin(), sv[k].end(), send + 3 * k);
    *n_recv = static_cast<int>(rv.size());
    *n_send = static_cast<int>(sv.size());
  });
}

int spmvk_nccl_version(int* version) {
  return guarded([&] {
    if (!version) fail(SPMVK_EINVAL, "nccl_version: null argument");
    nccl_check(nccl().GetVersion(version), "ncclGetVersion");
  });
}

int spmvk_nccl_unique_id(unsigned char* id_out) {
  return guarded([&] {
    if (!id_out) fail(SPMVK_EINVAL, "nccl_unique_id: null argument");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == SPMVK_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int spmvk_comm_init_rank(const unsigned char* id, int world, int rank, int device,
                         spmvk_comm** out) {
  return guarded([&] {
    if (!id || !out) fail(SPMVK_EINVAL, "comm_init_rank: null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(SPMVK_EINVAL, "comm_init_rank: rank outside [0, world)");
    SPMVK_CUDA(cudaSetDevice(device));
    require_device();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto c = std::make_unique<spmvk_comm>();
    nccl_check(nccl().CommInitRank(&c->comm, world, uid, rank), "ncclCommInitRank");
    c->rank = rank;
    c->world = world;
    c->device = device;
    *out = c.release();
  });
}

int spmvk_comm_init_all(int ndev, const int* devices, spmvk_comm** out) {
  return guarded([&] {
    if (ndev < 1 || !out) fail(SPMVK_EINVAL, "comm_init_all: bad argument");
    require_device();
    std::vector<ncclComm_t> comms(ndev);
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i) devs[i] = devices ? devices[i] : i;
    nccl_check(nccl().CommInitAll(comms.data(), ndev, devs.data()), "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i) {
      out[i] = new spmvk_comm();
      out[i]->comm = comms[i];
      out[i]->rank = i;
      out[i]->world = ndev;
      out[i]->device = devs[i];
    }
  });
}

int spmvk_comm_info(const spmvk_comm* c, int* rank, int* world, int* device) {
  return guarded([&] {
    if (!c) fail(SPMVK_EINVAL, "comm_info: null handle");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (device) *device = c->device;
  });
}

void spmvk_comm_destroy(spmvk_comm* c) { delete c; }

int spmvk_nccl_group_start(void) {
  return guarded([&] { nccl_check(nccl().GroupStart(), "ncclGroupStart"); });
}

int spmvk_nccl_group_end(void) {
  return guarded([&] { nccl_check(nccl().GroupEnd(), "ncclGroupEnd"); });
}

int spmvk_nccl_iter_create(spmvk_comm* comm, const spmvk_rgcsr* slab, uint64_t row_begin,
                           uint64_t row_end, uint64_t slab_rows, uint64_t n, int mode,
                           spmvk_nccl_iter** out) {
  return guarded([&] {
    if (!out) fail(SPMVK_EINVAL, "nccl_iter_create: null output");
    if (comm) SPMVK_CUDA(cudaSetDevice(comm->device));
    *out = iter_create(comm, slab, row_begin, row_end, slab_rows, n, mode);
  });
}

int spmvk_nccl_iter_x(const spmvk_nccl_iter* it, int buffer, void** out, uint64_t* length) {
  return guarded([&] {
    if (!it || !out) fail(SPMVK_EINVAL, "nccl_iter_x: null argument");
    if (buffer != 0 && buffer != 1) fail(SPMVK_EINVAL, "nccl_iter_x: buffer must be 0 or 1");
    *out = it->x[buffer].p;
    if (length) *length = it->n_alloc;
  });
}

int spmvk_nccl_iter_current(const spmvk_nccl_iter* it, int* buffer) {
  return guarded([&] {
    if (!it || !buffer) fail(SPMVK_EINVAL, "nccl_iter_current: null argument");
    *buffer = it->cur;
  });
}

int spmvk_nccl_iter_halo_entries(const spmvk_nccl_iter* it, uint64_t* entries) {
  return guarded([&] {
    if (!it || !entries) fail(SPMVK_EINVAL, "nccl_iter_halo_entries: null argument");
    *entries = it->recv_entries;
  });
}

int spmvk_nccl_iter_step_f64(spmvk_nccl_iter* it, double scale, double* y, void* stream) {
  return guarded([&] { iter_step<double>(it, scale, y, as_stream(stream)); });
}

int spmvk_nccl_iter_step_f32(spmvk_nccl_iter* it, float scale, float* y, void* stream) {
  return guarded([&] { iter_step<float>(it, scale, y, as_stream(stream)); });
}

void spmvk_nccl_iter_destroy(spmvk_nccl_iter* it) { delete it; }

}  // extern "C"
