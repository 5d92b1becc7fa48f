// K2 RgCSR SpMV kernels (included by rgcsr.cu).
//
// Every variant keeps the reference's per-row order of roundings
// (rgcsr.hpp:87-93): acc = ((0 + v0*x0) + v1*x1) + ..., product and sum
// rounded separately, so y is bitwise spmv_rgcsr's y.  They differ only in
// how the group-interleaved slots reach the SMs (measured comparison in
// DESIGN.md §3 and profiles/r01_k2_sweep*.md; the variants that never won a
// case -- per-warp / per-CTA TMA bulk-copy rings, L2 bulk prefetch of tiles,
// x staged in shared memory, the policy-hinted ldg kernels -- were removed in
// round 2 and their numbers kept in profiles/r02_k2_pruned.md):
//
//  * rgcsr_spmv_grp  — group-uniform walk (default without long rows).
//  * rgcsr_spmv_lite — register-lean thread per row at high occupancy.
//  * rgcsr_spmv_vec  — 128-bit vector slot loads, R rows per thread.
//  * rgcsr_spmv_pipe — row- and batch-pipelined thread per row.
//  * rgcsr_spmv_long_mixed — the rows past the long-row cut (warp per row,
//    or four rows per warp).
#pragma once
#include "common.cuh"

namespace spmvk {

// Row epilogue of the plain / iterated SpMV: y, and x_next = y * scale.
template <class T, bool kScaled>
struct StoreEpi {
  T* __restrict__ y;
  T* __restrict__ x_next;
  T scale;
  __device__ __forceinline__ void operator()(uint32_t r, T acc) const {
    y[r] = acc;
    if (kScaled) x_next[r] = mul_rn(acc, scale);
  }
};

// 128-bit slot vectors: R = 16 B / sizeof(T) adjacent rows of one slot.
template <class T, int R>
struct VecOf;
template <>
struct VecOf<double, 2> {
  using V = double2;
  using C = uint2;
  __device__ static double get(const double2& v, int i) { return i ? v.y : v.x; }
  __device__ static uint32_t col(const uint2& c, int i) { return i ? c.y : c.x; }
};
template <>
struct VecOf<float, 4> {
  using V = float4;
  using C = uint4;
  __device__ static float get(const float4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  __device__ static uint32_t col(const uint4& c, int i) {
    return i == 0 ? c.x : i == 1 ? c.y : i == 2 ? c.z : c.w;
  }
};

// Row- and batch-pipelined thread-per-row kernel (the default for short and
// medium rows).  Three latencies sit on a row's critical path — (row length,
// group pointer) -> (slot columns, values) -> x gathers — so both levels are
// software-pipelined: the next row's length / group pointer are loaded while
// the current row runs, and batch b+1's slots are loaded (predicated on the
// row length, so short rows and tails cost no extra round trip) before batch
// b's x gathers.  Accumulation stays strictly in slot order.
template <class T, int U>
__device__ __forceinline__ T pipe_row(uint32_t len, uint32_t s, const T* __restrict__ vp,
                                      const uint32_t* __restrict__ cp, const T* __restrict__ x,
                                      uint64_t pf, uint64_t pl) {
  uint32_t cA[U];
  T vA[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    cA[u] = 0;
    vA[u] = T(0);
    if ((uint32_t)u < len) {
      cA[u] = ld_stream(cp + (size_t)u * s, pf);
      vA[u] = ld_stream(vp + (size_t)u * s, pf);
    }
  }
  T acc = T(0);
  for (uint32_t j = 0; j < len; j += U) {
    const uint32_t jn = j + U;
    uint32_t cB[U];
    T vB[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cB[u] = 0;
      vB[u] = T(0);
      if (jn + u < len) {
        cB[u] = ld_stream(cp + (size_t)(jn + u) * s, pf);
        vB[u] = ld_stream(vp + (size_t)(jn + u) * s, pf);
      }
    }
    T xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = j + u < len ? ld_x(x + cA[u], pl) : T(0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < len) acc = add_rn(acc, mul_rn(vA[u], xv[u]));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cA[u] = cB[u];
      vA[u] = vB[u];
    }
  }
  return acc;
}

template <class T, int U, class Epi>
__device__ __forceinline__ void pipe_rows_epi(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, uint32_t long_cut,
    const Epi& epi) {
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t len_n = 0, base_n = 0;
  if (r < rows) {
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    len_n = lens[r];
    base_n = gp[g];
  }
  while (r < rows) {
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    const uint32_t t = r - g * G;
    const uint32_t s = min(G, rows - g * G);
    const uint32_t len = len_n;
    const T* __restrict__ vp = values + base_n + t;
    const uint32_t* __restrict__ cp = columns + base_n + t;
    const uint32_t rn = r + stride;
    if (rn < rows) {
      const uint32_t gn = g_shift >= 0 ? (rn >> g_shift) : rn / G;
      len_n = lens[rn];
      base_n = gp[gn];
    }
    if (len <= long_cut) epi(r, pipe_row<T, U>(len, s, vp, cp, x, pf, pl));  // else: long rows
    r = rn;
  }
}

// The same walk with rows taken dynamically: a warp grabs 128-row slices
// (one atomicAdd on *slice_ctr each, the next slice grabbed one ahead so its
// row metadata can be prefetched), so a warp that spent time on long-row
// items simply takes fewer slices -- no tail of late warps.
template <class T, int U, class Epi>
__device__ __forceinline__ void pipe_rows_dyn(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, uint32_t long_cut,
    uint32_t* slice_ctr, const Epi& epi) {
  constexpr uint32_t kSub = 4;  // 32-row sub-slices per grab
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  const uint32_t lane = threadIdx.x & 31;
  auto grab = [&]() -> uint64_t {
    uint32_t q = 0;
    if (lane == 0) q = atomicAdd(slice_ctr, 1u);
    q = __shfl_sync(0xffffffffu, q, 0);
    return static_cast<uint64_t>(q) * (32 * kSub);
  };
  // every slice comes from the counter in grab order: warps that first took
  // long-row items start on later slices, so the earliest slices -- the
  // heaviest rows below the cut in a descending-sorted matrix -- are not held
  // back behind the item phase (a static first slice per warp cost 2-10 %)
  uint64_t cur = grab();
  uint64_t nxt = cur < rows ? grab() : cur;
  uint32_t sub = 0;
  uint64_t r = cur + lane;
  uint32_t len_n = 0, base_n = 0;
  if (r < rows) {
    const uint32_t g = g_shift >= 0 ? ((uint32_t)r >> g_shift) : (uint32_t)r / G;
    len_n = lens[r];
    base_n = gp[g];
  }
  while (cur < rows) {  // warp-uniform
    uint64_t cur_n = cur;
    uint32_t sub_n = sub + 1;
    if (sub_n == kSub) {
      sub_n = 0;
      cur_n = nxt;
    }
    const uint64_t rn = cur_n + sub_n * 32 + lane;
    const uint32_t len = len_n, b0 = base_n;
    if (rn < rows) {
      const uint32_t gn = g_shift >= 0 ? ((uint32_t)rn >> g_shift) : (uint32_t)rn / G;
      len_n = lens[rn];
      base_n = gp[gn];
    }
    if (r < rows && len <= long_cut) {
      const uint32_t rr = static_cast<uint32_t>(r);
      const uint32_t g = g_shift >= 0 ? (rr >> g_shift) : rr / G;
      const uint32_t t = rr - g * G;
      const uint32_t s = min(G, rows - g * G);
      epi(rr, pipe_row<T, U>(len, s, values + b0 + t, columns + b0 + t, x, pf, pl));
    }
    if (sub_n == 0 && cur_n < rows) nxt = grab();
    cur = cur_n;
    sub = sub_n;
    r = rn;
  }
}

template <class T, bool kScaled, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_pipe(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t long_cut) {
  pipe_rows_epi<T, U>(rows, G, g_shift, gp, lens, values, columns, x, long_cut,
                      StoreEpi<T, kScaled>{y, x_next, scale});
}

// Lean thread-per-row kernel built for occupancy (the default K2): a CTA
// handles 256-row tiles (CTA-stride), each thread walks its row in U-deep
// batches with 32-bit strided pointers (no prefetch buffers, no cache-policy
// registers), so it fits the register budget of MINB resident CTAs per SM.
// Occupancy (40-64 warps / SM) gives the memory system the most independent
// requests; a predicated last batch avoids serialised single-slot round trips
// on short rows and tails.
// Row epilogues: what a finished row does with its sum.  StoreEpi is the
// plain / iterated form (y, and x_next = y * scale); PeerEpi (the fused
// distributed step, dist.cu) also stores x_next into every peer window whose
// receive range covers the row -- over NVLink when the peer is another GPU.

constexpr int kMaxPeers = 8;
template <class T>
struct PeerSet {
  T* dst[kMaxPeers];             // x_next buffer of each destination window
  uint32_t lo[kMaxPeers], hi[kMaxPeers];  // global rows [lo, hi) it receives
  int n;
};

template <class T>
struct PeerEpi {
  T* __restrict__ y;
  T* __restrict__ self;  // this rank's x_next buffer (every own row goes there)
  T scale;
  uint32_t row0;           // global index of the slab's first row
  uint32_t int_lo, int_hi;  // global rows no peer receives: self store only
  PeerSet<T> ps;            // peers (not self) and the rows each receives
  __device__ __forceinline__ void operator()(uint32_t r, T acc) const {
    y[r] = acc;
    const T xs = mul_rn(acc, scale);
    const uint32_t gr = row0 + r;
    self[gr] = xs;
    if (gr >= int_lo && gr < int_hi) return;
#pragma unroll
    for (int i = 0; i < kMaxPeers; ++i)
      if (i < ps.n && gr >= ps.lo[i] && gr < ps.hi[i]) ps.dst[i][gr] = xs;
  }
};

template <class T, int U, class Epi, bool kHint = false>
__device__ __forceinline__ void lite_tiles_epi(
    uint32_t tile_begin, uint32_t tile_end, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    uint32_t long_cut, const Epi& epi) {
  const Ldr<kHint> ld;
  for (uint32_t tile = tile_begin + blockIdx.x; tile < tile_end; tile += gridDim.x) {
    const uint32_t r = tile * 256 + threadIdx.x;
    if (r >= rows) continue;
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    uint32_t len = ld_stream(lens + r);
    const uint32_t base = ld_stream(gp + g);
    // rows past the cut are rgcsr_spmv_long's: predicated to zero slots rather
    // than branched around, so the length and group-pointer loads issue
    // together (a branch on len would let ptxas sink the gp load behind it)
    const bool mine = len <= long_cut;
    if (!mine) len = 0;
    const uint32_t s = min(G, rows - g * G);
    const uint32_t off = base + (r - g * G);
    const T* __restrict__ vp = values + off;
    const uint32_t* __restrict__ cp = columns + off;
    T acc = T(0);
    uint32_t j = 0;
    for (; j + U <= len; j += U) {  // full batches: U slot pairs, then U x gathers
      uint32_t c[U];
      T v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = ld.s(cp + u * s);
        v[u] = ld.s(vp + u * s);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = ld.x(x + c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
      cp += U * s;
      vp += U * s;
    }
    if (j < len) {  // predicated last batch
      uint32_t c[U];
      T v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U - 1; ++u) {
        c[u] = 0;
        v[u] = T(0);
        if (j + u < len) {
          c[u] = ld.s(cp + u * s);
          v[u] = ld.s(vp + u * s);
        }
      }
#pragma unroll
      for (int u = 0; u < U - 1; ++u) xv[u] = j + u < len ? ld.x(x + c[u]) : T(0);
#pragma unroll
      for (int u = 0; u < U - 1; ++u)
        if (j + u < len) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    }
    if (mine) epi(r, acc);
  }
}

template <class T, bool kScaled, int U>
__device__ __forceinline__ void lite_tiles(
    uint32_t tile_begin, uint32_t tile_end, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    T* __restrict__ y, T* __restrict__ x_next, T scale, uint32_t long_cut) {
  lite_tiles_epi<T, U>(tile_begin, tile_end, rows, G, g_shift, gp, lens, values,
                                    columns, x, long_cut, StoreEpi<T, kScaled>{y, x_next, scale});
}

template <class T, bool kScaled, int U, int MINB, bool kHint = false>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_lite(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t long_cut) {
  lite_tiles_epi<T, U, StoreEpi<T, kScaled>, kHint>(
      0, (rows + 255) / 256, rows, G, g_shift, gp, lens, values, columns, x, long_cut,
      StoreEpi<T, kScaled>{y, x_next, scale});
}

// One row of the group walk (group pointers b0, b1 and, if use_len, the row
// length already loaded): returns the row's sum in slot order.
template <class T, int U, bool kGatherK>
__device__ __forceinline__ T grp_row(uint32_t r, uint32_t b0, uint32_t b1, uint32_t len,
                                     bool use_len, uint32_t rows, uint32_t G, int g_shift,
                                     const T* __restrict__ values,
                                     const uint32_t* __restrict__ columns,
                                     const T* __restrict__ x) {
  const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
  const uint32_t s = min(G, rows - g * G);
  const uint32_t width = b1 - b0;
  const uint32_t K = (s == G && g_shift >= 0) ? (width >> g_shift) : width / s;
  const uint32_t lim = use_len ? len : K;
  const uint32_t off = b0 + (r - g * G);
  const T* __restrict__ vp = values + off;
  const uint32_t* __restrict__ cp = columns + off;
  T acc = T(0);
  uint32_t j = 0;
  for (; j + U <= K; j += U) {
    uint32_t c[U];
    T v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(vp + u * s);
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = ld_stream(cp + u * s);
    // warp barrier = a ptxas scheduling fence: every slot load (columns AND
    // values) issues before the first gather waits on a column; without it
    // ptxas interleaves and the value loads trail by a full DRAM round trip
    __syncwarp(__activemask());
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = (kGatherK || j + u < lim) ? ld_x(x + c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j + u < lim) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    cp += U * s;
    vp += U * s;
  }
  if (j < K) {  // predicated last batch (< U slots)
    uint32_t c[U - 1];
    T v[U - 1], xv[U - 1];
#pragma unroll
    for (int u = 0; u < U - 1; ++u) v[u] = j + u < K ? ld_stream(vp + u * s) : T(0);
#pragma unroll
    for (int u = 0; u < U - 1; ++u) c[u] = j + u < K ? ld_stream(cp + u * s) : 0u;
    __syncwarp(__activemask());
#pragma unroll
    for (int u = 0; u < U - 1; ++u)
      xv[u] = (kGatherK ? j + u < K : j + u < lim) ? ld_x(x + c[u]) : T(0);
#pragma unroll
    for (int u = 0; u < U - 1; ++u)
      if (j + u < lim) acc = add_rn(acc, mul_rn(v[u], xv[u]));
  }
  return acc;
}

// ---------------------------------------------------------------------------
// rgcsr_spmv_grp -- group-uniform walk for matrices without long rows.
//
// Every row of group g walks the group's full width K_g = (gp[g+1] - gp[g]) / s
// (uniform across a warp when G is a multiple of 32), so the slot loads
// depend only on the group pointers -- not on the row length -- and no lane
// diverges.  A thread's slots past its own length are pads (value 0, column
// 0): they are loaded (they sit in the same sectors as the neighbours' real
// slots) but contribute nothing:
//  * kNoLen = false: gathers and adds predicated on j < len (len loaded in
//    the same round trip as the group pointers);
//  * kNoLen = true: row_lengths is not read at all when x[0] is finite.  A
//    pad adds 0 * x[0] = +-0, and acc + (+-0) == acc bitwise: acc starts at
//    +0 and a round-to-nearest sum is -0 only for (-0) + (-0), so acc is
//    never -0.  A non-finite x[0] (0 * inf = NaN) switches the whole launch
//    (uniform branch) back to length predication.
// kMpf: the next row's (gp[g], gp[g+1], len) are loaded while this row's
// slots are in flight, so a row costs two dependent round trips (slots, x)
// like the ELLPACK kernel.  Per row the adds stay in slot order -> y bitwise
// spmv_rgcsr's.
// kGatherK: gather x for every slot < K (pads read x[0], harmless) and
// predicate only the adds on the length, so no load depends on the x[0]
// probe or the row length.
// kPdl: launched with programmatic stream serialisation -- the grid lets
// the next launch's CTAs start as its own retire (griddepcontrol
// .launch_dependents), and waits for the previous grid (griddepcontrol.wait:
// complete and its memory visible) before its first access to x or y; only
// the immutable matrix metadata is read before that.
template <class T, int U, bool kNoLen, bool kMpf, class Epi, bool kGatherK = false,
          bool kPdl = false>
__device__ __forceinline__ void grp_tiles_epi(uint32_t rows, uint32_t G, int g_shift,
                                              const uint32_t* __restrict__ gp,
                                              const uint32_t* __restrict__ lens,
                                              const T* __restrict__ values,
                                              const uint32_t* __restrict__ columns,
                                              const T* __restrict__ x, const Epi& epi,
                                              uint32_t x_pf_elems = 0,
                                              uint32_t pf_slots = 0) {
  // x_pf_elems > 0 (matrices that fit in L2): every CTA first bulk-prefetches
  // its 1/gridDim slice of x[0, x_pf_elems) into L2 (TMA unit, no completion
  // wait), so a cold launch's x gathers hit L2 instead of paying a second
  // DRAM round trip behind the slot loads.
  if (x_pf_elems && threadIdx.x == 0) {
    const uint64_t bytes = (uint64_t)x_pf_elems * sizeof(T);
    const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
    const uint64_t b0 = per * blockIdx.x, b1 = min((uint64_t)(bytes & ~15ull), b0 + per);
    for (uint64_t o = b0; o < b1; o += 65536)
      bulk_prefetch_l2(reinterpret_cast<const char*>(x) + o, (uint32_t)min((uint64_t)65536, b1 - o));
  }
  // pf_slots > 0 (small matrices, launched cold): the CTA also prefetches its
  // slice of the slot arrays and the group pointers, so a cold launch's
  // dependent chain (group pointers -> slots -> x) waits on DRAM once, not
  // three times
  if (pf_slots && threadIdx.x == 0) {
    const uint64_t ngp = (uint64_t)(rows + G - 1) / G + 1;
    const void* arr[3] = {values, columns, gp};
    const uint64_t len[3] = {(uint64_t)pf_slots * sizeof(T), (uint64_t)pf_slots * 4, ngp * 4};
    for (int a = 0; a < 3; ++a) {
      const uint64_t bytes = len[a] & ~15ull;
      const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
      const uint64_t b0 = per * blockIdx.x, b1 = min(bytes, b0 + per);
      for (uint64_t o = b0; o < b1; o += 65536)
        bulk_prefetch_l2(reinterpret_cast<const char*>(arr[a]) + o,
                         (uint32_t)min((uint64_t)65536, b1 - o));
    }
  }
  const uint32_t ntiles = (rows + 255) / 256;
  struct Meta {
    uint32_t b0, b1, len;
  };
  uint32_t pre_b0 = 0, pre_b1 = 0;  // kPdl: the first row's group pointers, before the wait
  if constexpr (kPdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t r0 = blockIdx.x * 256 + threadIdx.x;
    if (blockIdx.x < ntiles && r0 < rows) {
      const uint32_t g0 = g_shift >= 0 ? (r0 >> g_shift) : r0 / G;
      pre_b0 = ld_stream(gp + g0);
      pre_b1 = ld_stream(gp + g0 + 1);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const bool use_len = !kNoLen || !isfinite(__ldg(x));
  auto load_meta = [&](uint32_t r) {
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    Meta m;
    m.b0 = ld_stream(gp + g);
    m.b1 = ld_stream(gp + g + 1);
    m.len = use_len ? ld_stream(lens + r) : 0u;
    return m;
  };
  Meta nxt{0, 0, 0};
  if (kMpf) {
    const uint32_t r0 = blockIdx.x * 256 + threadIdx.x;
    if (blockIdx.x < ntiles && r0 < rows) {
      if constexpr (kPdl) nxt = Meta{pre_b0, pre_b1, use_len ? ld_stream(lens + r0) : 0u};
      else nxt = load_meta(r0);
    }
  }
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t r = tile * 256 + threadIdx.x;
    Meta m;
    if (kMpf) {
      m = nxt;
      const uint32_t rn = r + gridDim.x * 256;
      if (tile + gridDim.x < ntiles && rn < rows) nxt = load_meta(rn);
    }
    if (r >= rows) continue;
    if (!kMpf) m = load_meta(r);
    epi(r, grp_row<T, U, kGatherK>(r, m.b0, m.b1, m.len, use_len, rows, G, g_shift, values,
                                   columns, x));
  }
}

// rgcsr_spmv_grpv -- the group walk with 128-bit slot loads (fp32: R = 4
// rows per thread, float4 values + uint4 columns; fp64: R = 2).  A thread's R
// rows are adjacent in every slot of their group (entry j of row t at
// gp[g] + t + j s; G % R == 0 and gp[g] a multiple of s keep the vectors
// aligned), so a warp reads 32 R consecutive slots per stream -- 512 B for
// fp32 -- with a quarter of the load instructions.  As the scalar walk: every
// row of group g walks K_g slots, pads add 0 * x[0] (row_lengths is read only
// when x[0] is not finite), the next tile's group pointers are prefetched,
// each row adds in slot order -> bitwise.  Rows of a partial last group
// (s % R != 0) take the scalar grp_row.
template <class T, bool kScaled, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_grpv(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t x_pf_elems, uint32_t pf_slots) {
  constexpr int R = 16 / sizeof(T);
  using Wv = VecOf<T, R>;
  using V = typename Wv::V;
  using Cv = typename Wv::C;
  const StoreEpi<T, kScaled> epi{y, x_next, scale};
  if (threadIdx.x == 0 && (x_pf_elems || pf_slots)) {  // small matrices: as the scalar walk
    const uint64_t ngp = pf_slots ? (uint64_t)(rows + G - 1) / G + 1 : 0;
    const void* arr[4] = {x, values, columns, gp};
    const uint64_t len[4] = {(uint64_t)x_pf_elems * sizeof(T), (uint64_t)pf_slots * sizeof(T),
                             (uint64_t)pf_slots * 4, ngp * 4};
    for (int a = 0; a < 4; ++a) {
      const uint64_t bytes = len[a] & ~15ull;
      const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
      const uint64_t b0 = per * blockIdx.x, b1 = min(bytes, b0 + per);
      for (uint64_t o = b0; o < b1; o += 65536)
        bulk_prefetch_l2(reinterpret_cast<const char*>(arr[a]) + o,
                         (uint32_t)min((uint64_t)65536, b1 - o));
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool use_len = !isfinite(__ldg(x));
  constexpr uint32_t kTile = 256 * R;
  const uint32_t tiles = (rows + kTile - 1) / kTile;
  auto gidx = [&](uint32_t r) { return g_shift >= 0 ? (r >> g_shift) : r / G; };
  uint32_t nb0 = 0, nb1 = 0;
  {
    const uint32_t r0 = blockIdx.x * kTile + threadIdx.x * R;
    if (blockIdx.x < tiles && r0 < rows) {
      nb0 = ld_stream(gp + gidx(r0));
      nb1 = ld_stream(gp + gidx(r0) + 1);
    }
  }
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t r0 = tile * kTile + threadIdx.x * R;
    const uint32_t b0 = nb0, b1 = nb1;
    const uint32_t rn = r0 + gridDim.x * kTile;
    if (tile + gridDim.x < tiles && rn < rows) {
      nb0 = ld_stream(gp + gidx(rn));
      nb1 = ld_stream(gp + gidx(rn) + 1);
    }
    if (r0 >= rows) continue;
    const uint32_t g = gidx(r0);
    const uint32_t s = min(G, rows - g * G);
    if (s % R != 0 || r0 + R > rows) {  // partial last group: scalar rows
      for (uint32_t i = 0; i < R && r0 + i < rows; ++i) {
        const uint32_t r = r0 + i;
        const uint32_t len = use_len ? lens[r] : 0u;
        epi(r, grp_row<T, 4, true>(r, gp[g], gp[g + 1], len, use_len, rows, G, g_shift, values,
                                   columns, x));
      }
      continue;
    }
    const uint32_t K = (s == G && g_shift >= 0) ? ((b1 - b0) >> g_shift) : (b1 - b0) / s;
    uint32_t lim[R];
#pragma unroll
    for (int i = 0; i < R; ++i) lim[i] = K;
    if (use_len) {
#pragma unroll
      for (int i = 0; i < R; ++i) lim[i] = lens[r0 + i];
    }
    const uint32_t vs = s / R;  // one slot, in vectors
    const V* __restrict__ vp = reinterpret_cast<const V*>(values + b0 + (r0 - g * G));
    const Cv* __restrict__ cp = reinterpret_cast<const Cv*>(columns + b0 + (r0 - g * G));
    T acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = T(0);
    uint32_t j = 0;
    for (; j + U <= K; j += U) {  // full U-deep batches
      V v[U];
      Cv c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream_v(vp + u * vs);
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = ld_stream_v(cp + u * vs);
      __syncwarp(__activemask());  // every slot load before the gathers
      T xv[U][R];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < R; ++i) xv[u][i] = ld_x(x + Wv::col(c[u], i));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (j + u < lim[i]) acc[i] = add_rn(acc[i], mul_rn(Wv::get(v[u], i), xv[u][i]));
      vp += U * vs;
      cp += U * vs;
    }
    for (; j < K; ++j) {  // tail slots one at a time
      const V v = ld_stream_v(vp);
      const Cv c = ld_stream_v(cp);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const T xi = ld_x(x + Wv::col(c, i));
        if (j < lim[i]) acc[i] = add_rn(acc[i], mul_rn(Wv::get(v, i), xi));
      }
      vp += vs;
      cp += vs;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) epi(r0 + i, acc[i]);
  }
}

template <class T, bool kScaled, int U, int MINB, bool kNoLen, bool kMpf, bool kGatherK = false,
          bool kPdl = false>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_grp(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t x_pf_elems /* long_cut slot: no long rows here */,
    uint32_t pf_slots) {
  grp_tiles_epi<T, U, kNoLen, kMpf, StoreEpi<T, kScaled>, kGatherK, kPdl>(
      rows, G, g_shift, gp, lens, values, columns, x, StoreEpi<T, kScaled>{y, x_next, scale},
      x_pf_elems, pf_slots);
}

// SpMV with the CG dot fused into the row epilogue: y = A x and, per CTA, the
// partial sum of xself[r] * y[r] over the rows it produced (xself = the
// slab's own rows of x), for p.q in conjugate gradients -- saves the dot
// kernel's second pass over p and q.  Deterministic: each thread adds its
// rows in tile order, then a fixed block reduction; the per-CTA partials are
// summed in CTA order by rgcsr_dot_finish.
template <class T>
struct DotEpi {
  T* __restrict__ y;
  const T* __restrict__ xself;
  double* acc;
  __device__ __forceinline__ void operator()(uint32_t r, T v) const {
    y[r] = v;
    *acc += static_cast<double>(xself[r]) * static_cast<double>(v);
  }
};

__device__ __forceinline__ double block_sum_256(double v) {
  __shared__ double sh[8];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
  if (threadIdx.x < 32)
    for (int o = 4; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  return t;  // valid in thread 0
}

template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_dot_grp(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    const T* __restrict__ xself, double* __restrict__ part) {
  double acc = 0.0;
  grp_tiles_epi<T, U, true, true, DotEpi<T>>(rows, G, g_shift, gp, lens, values, columns, x,
                                             DotEpi<T>{y, xself, &acc});
  acc = block_sum_256(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

static __global__ void __launch_bounds__(256) rgcsr_dot_finish(const double* __restrict__ part, int np,
                                                        double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) s += part[i];
  s = block_sum_256(s);
  if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------------------
// rgcsr_spmv_vec -- 128-bit vectorised slot loads (north_star subsystem 2).
//
// A thread owns R consecutive rows of one group (fp64: R = 2, one 16-byte
// double2 value load and one 8-byte uint2 column load per slot; fp32: R = 4,
// float4 + uint4, 16 bytes each).  Rows t..t+R-1 of a group are adjacent in
// every slot (entry j of row t at gp[g] + t + j*s), so when s % R == 0 (every
// full group for G % R == 0; then gp[g] and t are multiples of R too) the R
// rows' slot j is one aligned vector.  The pair / quad walks max(len) slots;
// each row accumulates only its own first len slots, in slot order, so y is
// bitwise the thread-per-row result.  Misaligned vectors (s % R != 0 or
// gp[g] % R != 0: odd G, a short last group) and vectors holding a long row
// take the scalar per-row path.
template <class T, int U>
__device__ __forceinline__ T scalar_row(const T* __restrict__ vp, const uint32_t* __restrict__ cp,
                                        uint32_t s, uint32_t len, const T* __restrict__ x) {
  T acc = T(0);
  uint32_t j = 0;
  for (; j + U <= len; j += U) {
    uint32_t c[U];
    T v[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ld_stream(cp + u * s);
      v[u] = ld_stream(vp + u * s);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = ld_x(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(v[u], xv[u]));
    cp += U * s;
    vp += U * s;
  }
  for (; j < len; ++j, cp += s, vp += s) acc = add_rn(acc, mul_rn(ld_stream(vp), ld_x(x + *cp)));
  return acc;
}

template <class T, int R, int U, class Epi>
__device__ __forceinline__ void vec_tiles(uint32_t rows, uint32_t G, int g_shift,
                                          const uint32_t* __restrict__ gp,
                                          const uint32_t* __restrict__ lens,
                                          const T* __restrict__ values,
                                          const uint32_t* __restrict__ columns,
                                          const T* __restrict__ x, uint32_t long_cut,
                                          const Epi& epi) {
  using W = VecOf<T, R>;
  using V = typename W::V;
  using Cv = typename W::C;
  constexpr uint32_t kTile = 256 * R;
  const uint32_t tiles = (rows + kTile - 1) / kTile;
  for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint32_t r0 = tile * kTile + threadIdx.x * R;
    if (r0 >= rows) continue;
    const uint32_t g = g_shift >= 0 ? (r0 >> g_shift) : r0 / G;
    const uint32_t s = min(G, rows - g * G);
    const uint32_t t = r0 - g * G;
    const uint32_t base = gp[g] + t;
    uint32_t len[R], n = 0;
    bool any_long = false;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      len[i] = r0 + i < rows ? lens[r0 + i] : 0;
      any_long |= len[i] > long_cut;
      n = max(n, len[i]);
    }
    // vector path: the R rows' slots are aligned R-vectors (s, t and gp[g]
    // multiples of R -- gp[g] is not when an odd G precedes an even last group)
    if (s % R != 0 || base % R != 0 || t + R > s || any_long) {  // scalar per-row path
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint32_t r = r0 + i;
        if (r >= rows || len[i] > long_cut) continue;
        const uint32_t gi = g_shift >= 0 ? (r >> g_shift) : r / G;
        const uint32_t si = min(G, rows - gi * G);
        const uint32_t off = gp[gi] + (r - gi * G);
        epi(r, scalar_row<T, 4>(values + off, columns + off, si, len[i], x));
      }
      continue;
    }
    const V* __restrict__ vp = reinterpret_cast<const V*>(values + base);
    const Cv* __restrict__ cp = reinterpret_cast<const Cv*>(columns + base);
    const uint32_t sv = s / R;  // slot stride in vectors
    T acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = T(0);
    uint32_t j = 0;
    for (; j + U <= n; j += U) {
      V v[U];
      Cv c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = ld_stream_v(cp + u * sv);
        v[u] = ld_stream_v(vp + u * sv);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (j + u < len[i])
            acc[i] = add_rn(acc[i], mul_rn(W::get(v[u], i), ld_x(x + W::col(c[u], i))));
      cp += U * sv;
      vp += U * sv;
    }
    for (; j < n; ++j, cp += sv, vp += sv) {
      const Cv c = ld_stream_v(cp);
      const V v = ld_stream_v(vp);
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (j < len[i]) acc[i] = add_rn(acc[i], mul_rn(W::get(v, i), ld_x(x + W::col(c, i))));
    }
#pragma unroll
    for (int i = 0; i < R; ++i) epi(r0 + i, acc[i]);
  }
}

template <class T, bool kScaled, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_vec(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t long_cut) {
  constexpr int R = sizeof(T) == 8 ? 2 : 4;
  vec_tiles<T, R, U>(rows, G, g_shift, gp, lens, values, columns, x, long_cut,
                     StoreEpi<T, kScaled>{y, x_next, scale});
}

// Same kernel over the 256-row tiles [tile_begin, tile_end) only: the unit of
// the pipelined host-span SpMV (H2D of x, row chunks and D2H of y overlap).
template <class T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_lite_range(
    uint32_t tile_begin, uint32_t tile_end, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    T* __restrict__ y) {
  lite_tiles<T, false, U>(tile_begin, tile_end, rows, G, g_shift, gp, lens, values, columns, x, y,
                          nullptr, T(0), 0xffffffffu);
}

// Per row chunk of `chunk_rows` rows: the smallest first-slot column and the
// largest last-slot column (columns increase along a row), i.e. the x range
// the chunk reads.  out[2k] = min, out[2k+1] = max (min > max if empty).
static __global__ void chunk_column_ranges(uint32_t rows, uint32_t G, uint32_t chunk_rows,
                                    const uint32_t* __restrict__ gp,
                                    const uint32_t* __restrict__ lens,
                                    const uint32_t* __restrict__ columns,
                                    unsigned* __restrict__ out) {
  // warp-uniform trip count so the warp reductions see all 32 lanes
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; w < rows;
       w += gridDim.x * blockDim.x) {
    const uint32_t r = w + (threadIdx.x & 31);
    unsigned lo = 0xffffffffu, hi = 0;
    const uint32_t len = r < rows ? lens[r] : 0;
    if (len) {
      const uint32_t g = r / G, s = min(G, rows - g * G), base = gp[g] + (r - g * G);
      lo = columns[base];
      hi = columns[base + (len - 1) * s];
    }
    const uint32_t k = r / chunk_rows;
    if ((w / chunk_rows) == ((w + 31) / chunk_rows)) {  // warp inside one chunk
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(out + 2 * k, lo);
        atomicMax(out + 2 * k + 1, hi);
      }
    } else if (len) {
      atomicMin(out + 2 * k, lo);
      atomicMax(out + 2 * k + 1, hi);
    }
  }
}

// ---------------------------------------------------------------------------
// rgcsr_spmv_long — the rows longer than kLongRow (power-law tails), one warp
// per row.  A thread-per-row kernel would serialise a 4096-slot row in one
// thread for ~1000 dependent round trips; here the warp loads 256 slots of the
// row at a time (8 per lane, all in flight), forms the products in parallel,
// stages them in shared memory, and one lane adds them in slot order — the
// reference's rounding sequence, so y stays bitwise.
template <class T, class Epi>
__device__ __forceinline__ void long_rows_epi(
    uint32_t nlong, const uint32_t* __restrict__ long_rows, uint32_t rows, uint32_t G,
    int g_shift, const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    const Epi& epi) {
  constexpr int K = 8, W = 32 * K;
  __shared__ T prod[8][W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
  for (uint32_t i = blockIdx.x * 8 + warp; i < nlong; i += gridDim.x * 8) {
    const uint32_t r = long_rows[i];
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    const uint32_t t = r - g * G;
    const uint32_t s = min(G, rows - g * G);
    const uint32_t len = lens[r];
    const T* __restrict__ vp = values + gp[g] + t;
    const uint32_t* __restrict__ cp = columns + gp[g] + t;
    T acc = T(0);
    for (uint32_t j0 = 0; j0 < len; j0 += W) {
      uint32_t c[K];
      T v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t j = j0 + lane + 32 * k;
        c[k] = 0;
        v[k] = T(0);
        if (j < len) {
          c[k] = ld_stream(cp + (size_t)j * s, pf);
          v[k] = ld_stream(vp + (size_t)j * s, pf);
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t j = j0 + lane + 32 * k;
        if (j < len) prod[warp][lane + 32 * k] = mul_rn(v[k], ld_x(x + c[k], pl));
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t n = min((uint32_t)W, len - j0);
        uint32_t q = 0;
        for (; q + 8 <= n; q += 8) {
          T p[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) p[u] = prod[warp][q + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = add_rn(acc, p[u]);
        }
        for (; q < n; ++q) acc = add_rn(acc, prod[warp][q]);
      }
      __syncwarp();
    }
    if (lane == 0) epi(r, acc);
  }
}

// Four consecutive long rows of one group per warp ("quad": rows r..r+3,
// r % 4 == 0, G % 4 == 0): lane = 8 q + l works on row q's slots j = l, l+8,
// ..., so for a fixed j the four rows' slots sit in ONE 32-byte sector (slot j
// of rows t..t+3 is contiguous) -- a quarter of the uncoalesced sector
// requests of one row per warp, which is what bounds the long-row phase
// (l1tex request path, profiles/r01_powerlaw.md).  64 slots per row per
// round; products staged in shared memory; lane 8 q adds row q's products in
// slot order, so y stays bitwise.  Singles (the other long rows) take the
// warp-per-row path above.  One kernel for both lists: item i < n_single is
// single row single_rows[i], else quad quads[i - n_single].
// Sequential sum of n staged products p[0..n) onto acc, in order; the next
// 8 products are loaded from shared memory while the current 8 are added.
template <class T, int B = 8>
__device__ __forceinline__ T ordered_sum(const T* __restrict__ p, uint32_t n, T acc) {
  uint32_t q = 0;
  if (n >= B) {
    T a[B];
#pragma unroll
    for (int u = 0; u < B; ++u) a[u] = p[u];
    for (q = B; q + B <= n; q += B) {
      T b[B];
#pragma unroll
      for (int u = 0; u < B; ++u) b[u] = p[q + u];
#pragma unroll
      for (int u = 0; u < B; ++u) acc = add_rn(acc, a[u]);
#pragma unroll
      for (int u = 0; u < B; ++u) a[u] = b[u];
    }
#pragma unroll
    for (int u = 0; u < B; ++u) acc = add_rn(acc, a[u]);
  }
  for (; q < n; ++q) acc = add_rn(acc, p[q]);
  return acc;
}

// One long row per L lanes (L = 32: a single; L = 8: one of a quad's four
// rows), K slots per lane per round, software-pipelined: the next round's
// slot loads are issued before this round's ordered adds, so the DRAM
// latency of the slot stream hides behind the sequential add chain.  Lane l
// of the row handles slots j0 + l + L*k; products go to pr[l + L*k]; lane
// l == 0 adds them in slot order (the reference's rounding sequence).
template <class T, int L, int K, bool kHint, int B = 8>
__device__ __forceinline__ T long_row_walk(uint32_t len, uint32_t lmax, int l,
                                           const T* __restrict__ vp,
                                           const uint32_t* __restrict__ cp, uint32_t s,
                                           const T* __restrict__ x, T* __restrict__ pr,
                                           const Ldr<kHint>& ld, T acc0 = T(0)) {
  constexpr uint32_t W = L * K;
  uint32_t c[K];
  T v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t j = l + L * k;
    c[k] = j < len ? ld.s(cp + (size_t)j * s) : 0u;
    v[k] = j < len ? ld.s(vp + (size_t)j * s) : T(0);
  }
  T acc = acc0;  // meaningful in the adding lane (l == 0)
  for (uint32_t j0 = 0; j0 < lmax; j0 += W) {
    __syncwarp();  // scheduling fence, and the previous round's adds are done
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t j = j0 + l + L * k;
      if (j < len) pr[l + L * k] = mul_rn(v[k], ld.x(x + c[k]));
    }
    const uint32_t jn = j0 + W;  // next round's slots, in flight during the adds
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t j = jn + l + L * k;
      c[k] = j < len ? ld.s(cp + (size_t)j * s) : 0u;
      v[k] = j < len ? ld.s(vp + (size_t)j * s) : T(0);
    }
    __syncwarp();
    if (l == 0 && j0 < len) acc = ordered_sum<T, B>(pr, min(W, len - j0), acc);
  }
  __syncwarp();
  return acc;
}

// One long-row work item: item i < n_single is row single_rows[i] (warp per
// row), else quad quads[i - n_single]: four consecutive long rows of one group
// (r0 % 4 == 0), lane 8 q + l on row q's slots l, l+8, ..., so the four rows'
// slot j is ONE 32-byte sector (a quarter of the uncoalesced requests of one
// row per warp).  pr: this warp's 256-entry product buffer in shared memory.
template <class T, class Epi, bool kHint, int K = 8>
__device__ __forceinline__ void long_item(
    uint32_t i, uint32_t n_single, const uint32_t* __restrict__ single_rows,
    const uint32_t* __restrict__ quads, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    T* __restrict__ pr, const Ldr<kHint>& ld, const Epi& epi) {
  constexpr int W = 32 * K;
  const int lane = threadIdx.x & 31;
  if (i < n_single) {  // one row per warp
    const uint32_t r = single_rows[i];
    const uint32_t g = g_shift >= 0 ? (r >> g_shift) : r / G;
    const uint32_t s = min(G, rows - g * G);
    const uint32_t len = lens[r];
    const uint32_t off = gp[g] + (r - g * G);
    const T acc = long_row_walk<T, 32, K, kHint, (K >= 8 ? 8 : 4)>(len, len, lane, values + off,
                                                                  columns + off, s, x, pr, ld);
    if (lane == 0) epi(r, acc);
    return;
  }
  // quad: rows r0..r0+3 of one group, 8 lanes per row, 64 slots per round
  const uint32_t r0 = quads[i - n_single];
  const int q = lane >> 3, l = lane & 7;
  const uint32_t r = r0 + q;
  const uint32_t g = g_shift >= 0 ? (r0 >> g_shift) : r0 / G;
  const uint32_t s = min(G, rows - g * G);
  const uint32_t len = lens[r];
  uint32_t lmax = len;
#pragma unroll
  for (int o = 8; o < 32; o <<= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  const uint32_t off = gp[g] + (r - g * G);
  const T acc = long_row_walk<T, 8, K, kHint, (K >= 8 ? 8 : 4)>(len, lmax, l, values + off,
                                                                 columns + off, s, x,
                                                                 pr + q * (W / 4), ld);
  if (l == 0) epi(r, acc);
}

// The rows past the long-row cut, one launch, two work lists (long_item),
// statically spread over the warps of the grid.
template <class T, class Epi, bool kHint = false>
__device__ __forceinline__ void long_mixed_epi(
    uint32_t n_single, const uint32_t* __restrict__ single_rows, uint32_t n_quad,
    const uint32_t* __restrict__ quads, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    const Epi& epi) {
  constexpr int K = 8, W = 32 * K;
  __shared__ T prod[8][W];
  const int warp = threadIdx.x >> 5;
  const uint32_t items = n_single + n_quad;
  const Ldr<kHint> ld;
  for (uint32_t i = blockIdx.x * 8 + warp; i < items; i += gridDim.x * 8)
    long_item<T, Epi, kHint>(i, n_single, single_rows, quads, rows, G, g_shift, gp, lens, values,
                             columns, x, prod[warp], ld, epi);
}

// The long-row work lists of a matrix, for the fused kernels below: the items
// are taken dynamically (one atomicAdd per item on ctr[0], singles longest
// first, then the quads), so the longest rows start first and no warp idles
// while another holds several; ctr[1] counts the warps that are done, and the
// last one resets every word for the next launch on the stream (ctr is the
// stream's own counter block, stream_counters(); ctr[2] is the row-slice
// counter of pipe_rows_dyn).
struct LongList {
  uint32_t n_single, n_quad;
  const uint32_t* singles;
  const uint32_t* quads;
  uint32_t* ctr;
  uint32_t warps;  // warps per CTA that take items (the first `warps`); the rest stream tiles
};

// Each warp first takes long-row items until none are left, then runs its
// share of the thread-per-row tiles: the long rows' latency-bound ordered
// adds overlap the tile streaming of the other warps instead of running as a
// second, mostly idle kernel after it.
template <class T, class Epi, bool kHint, int K>
__device__ __forceinline__ void long_items_dynamic(
    const LongList& ll, uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ pr,
    const Epi& epi) {
  const int lane = threadIdx.x & 31;
  const uint32_t items = ll.n_single + ll.n_quad;
  if (items == 0 || (threadIdx.x >> 5) >= ll.warps) return;
  const Ldr<kHint> ld;
  for (;;) {
    uint32_t i = 0;
    if (lane == 0) i = atomicAdd(ll.ctr, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= items) break;
    long_item<T, Epi, kHint, K>(i, ll.n_single, ll.singles, ll.quads, rows, G, g_shift, gp, lens,
                                values, columns, x, pr, ld, epi);
  }
}

// Counted per CTA (one atomic per CTA, not per warp: same-address atomics
// serialise in L2): every warp of the CTA has made its last fetch before the
// barrier, and the last CTA resets the counters for the next launch.
__device__ __forceinline__ void long_items_done(const LongList& ll) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // the CTA's last fetches are ordered before its done count
    if (atomicAdd(ll.ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(ll.ctr, 0u);
      atomicExch(ll.ctr + 2, 0u);
      atomicExch(ll.ctr + 1, 0u);
    }
  }
}

// lite with the long rows fused (long_items_dynamic first, then the tiles);
// KL slots per lane per round of the long walk (4 keeps the register-capped
// lite kernels free of spills).
template <class T, bool kScaled, int U, int MINB, bool kHint, int KL = 4>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_lite_fl(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t long_cut, LongList ll) {
  __shared__ T prod[8][32 * KL];
  const StoreEpi<T, kScaled> epi{y, x_next, scale};
  long_items_dynamic<T, StoreEpi<T, kScaled>, kHint, KL>(ll, rows, G, g_shift, gp, lens, values,
                                                         columns, x, prod[threadIdx.x >> 5], epi);
  lite_tiles_epi<T, U, StoreEpi<T, kScaled>, kHint>(0, (rows + 255) / 256, rows, G, g_shift, gp,
                                                    lens, values, columns, x, long_cut, epi);
  long_items_done(ll);
}

// pipe with the long rows fused (the reordered power-law default).
template <class T, bool kScaled, int U, int MINB, int KL = 4>
__global__ void __launch_bounds__(256, MINB) rgcsr_spmv_pipe_fl(
    uint32_t rows, uint32_t G, int g_shift, const uint32_t* __restrict__ gp,
    const uint32_t* __restrict__ lens, const T* __restrict__ values,
    const uint32_t* __restrict__ columns, const T* __restrict__ x, T* __restrict__ y,
    T* __restrict__ x_next, T scale, uint32_t long_cut, LongList ll) {
  __shared__ T prod[8][32 * KL];
  const StoreEpi<T, kScaled> epi{y, x_next, scale};
  long_items_dynamic<T, StoreEpi<T, kScaled>, true, KL>(ll, rows, G, g_shift, gp, lens, values,
                                                        columns, x, prod[threadIdx.x >> 5], epi);
  pipe_rows_dyn<T, U>(rows, G, g_shift, gp, lens, values, columns, x, long_cut, ll.ctr + 2, epi);
  long_items_done(ll);
}

template <class T, bool kScaled, bool kHint = false>
__global__ void __launch_bounds__(256) rgcsr_spmv_long_mixed(
    uint32_t n_single, const uint32_t* __restrict__ single_rows, uint32_t n_quad,
    const uint32_t* __restrict__ quads, uint32_t rows, uint32_t G, int g_shift,
    const uint32_t* __restrict__ gp, const uint32_t* __restrict__ lens,
    const T* __restrict__ values, const uint32_t* __restrict__ columns, const T* __restrict__ x,
    T* __restrict__ y, T* __restrict__ x_next, T scale) {
  long_mixed_epi<T, StoreEpi<T, kScaled>, kHint>(n_single, single_rows, n_quad, quads, rows, G,
                                                 g_shift, gp, lens, values,
                    columns, x, StoreEpi<T, kScaled>{y, x_next, scale});
}

}  // namespace spmvk
