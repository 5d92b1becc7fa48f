// RgCSR on the device: K1 (CSR -> RgCSR conversion) and K2 (SpMV).
//
// Layout (identical to the reference, spmvkit/rgcsr.hpp:11-28): rows are cut
// into groups of G (the last one s = N - g*G rows); group g owns the slab
// [gp[g], gp[g+1]) of s * K_g slots, K_g its longest row; entry j of local row
// t sits at gp[g] + t + j*s, pads hold (0, column 0).  For one step j the s
// rows of a group read s CONTIGUOUS slots, so a warp of consecutive rows
// issues fully coalesced loads with one thread per row.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "rgcsr_spmv.cuh"
#include "tma.cuh"

namespace spmvk {
namespace {

// ------------------------------------------------------------ K1: layout
// Per group g (s_g rows): slots[g] = s_g * max_t lens[g*G + t] and
// nlong[g] = how many of its rows are longer than the long-row cut.
__global__ void group_layout(uint64_t rows, uint64_t G, uint64_t groups, uint32_t cut,
                             const uint32_t* __restrict__ lens, uint64_t* __restrict__ slots,
                             uint64_t* __restrict__ nlong) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = g * G, s = min(G, rows - r0);
    uint32_t w = 0, nl = 0;
    for (uint64_t t = 0; t < s; ++t) {
      const uint32_t l = lens[r0 + t];
      w = max(w, l);
      nl += l > cut;
    }
    slots[g] = s * w;
    nlong[g] = nl;
  }
}

// Fused K1 layout (the default): two launches instead of row lengths +
// group layout + two three-kernel scans + nnz + narrowing (twelve launches,
// ~75 us of launch-bound host time on a 0.3 ms build).
//   k1_layout: a CTA per tile of TG groups (<= kLayoutRows rows): row lengths
//     (written, and staged in shared memory), then per group its slot count
//     s*K_g and long-row count, and the tile's two sums in part[2b..2b+1].
//     The last CTA to finish (ticket in the stream's counter word 3, reset
//     by that CTA) scans the tile sums in place and writes the totals
//     (slots, long rows, slab nnz) to tot[0..2].
//   k1_layout_apply: a CTA per tile turns its groups' counts into the
//     exclusive prefixes: group_pointers (u32) and the long-row offsets (u64).
// Thread j of a tile owns its groups [j*q, (j+1)*q), q = ceil(TG/256), in
// both kernels.
constexpr uint32_t kLayoutRows = 8192;
constexpr int kLayoutThreads = 256;

__device__ __forceinline__ uint32_t lpad(uint64_t i) { return (uint32_t)(i + (i >> 5)); }

// Block-wide exclusive scan of a pair; returns the block totals.
__device__ __forceinline__ void block_scan_pair(uint64_t a, uint64_t b, uint64_t& ea,
                                                uint64_t& eb, uint64_t& ta, uint64_t& tb) {
  __shared__ uint64_t wt[2][kLayoutThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t xa = __shfl_up_sync(0xffffffffu, ia, o);
    const uint64_t xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) ia += xa, ib += xb;
  }
  if (lane == 31) wt[0][warp] = ia, wt[1][warp] = ib;
  __syncthreads();
  if (warp == 0) {
    uint64_t wa = lane < kLayoutThreads / 32 ? wt[0][lane] : 0;
    uint64_t wb = lane < kLayoutThreads / 32 ? wt[1][lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t xa = __shfl_up_sync(0xffffffffu, wa, o);
      const uint64_t xb = __shfl_up_sync(0xffffffffu, wb, o);
      if (lane >= o) wa += xa, wb += xb;
    }
    if (lane < kLayoutThreads / 32) wt[0][lane] = wa, wt[1][lane] = wb;
  }
  __syncthreads();
  ea = (warp ? wt[0][warp - 1] : 0) + ia - a;
  eb = (warp ? wt[1][warp - 1] : 0) + ib - b;
  ta = wt[0][kLayoutThreads / 32 - 1];
  tb = wt[1][kLayoutThreads / 32 - 1];
  __syncthreads();
}

__global__ void __launch_bounds__(kLayoutThreads) k1_layout(
    uint64_t r0, uint64_t rows, uint64_t G, uint64_t groups, uint64_t TG, uint32_t cut,
    const uint32_t* __restrict__ rp, uint32_t* __restrict__ lens, uint64_t* __restrict__ slots,
    uint64_t* __restrict__ nlong, uint64_t* __restrict__ part, uint32_t* __restrict__ ticket,
    uint64_t* __restrict__ tot) {
  __shared__ uint32_t sl[kLayoutRows + kLayoutRows / 32];
  __shared__ bool last;
  const uint64_t g0 = blockIdx.x * TG, g1 = min(groups, g0 + TG);
  const uint64_t rb = g0 * G, re = min(rows, g1 * G);
  const bool staged = re - rb <= kLayoutRows;
  for (uint64_t r = rb + threadIdx.x; r < re; r += kLayoutThreads) {
    const uint32_t l = rp[r0 + r + 1] - rp[r0 + r];
    lens[r] = l;
    if (staged) sl[lpad(r - rb)] = l;
  }
  __syncthreads();
  const uint64_t q = (g1 - g0 + kLayoutThreads - 1) / kLayoutThreads;
  const uint64_t ga = min(g1, g0 + threadIdx.x * q), gb = min(g1, ga + q);
  uint64_t ss = 0, ls = 0;
  for (uint64_t g = ga; g < gb; ++g) {
    const uint64_t gr = g * G, s = min(G, rows - gr);
    uint32_t w = 0, nl = 0;
    for (uint64_t t = 0; t < s; ++t) {
      const uint32_t l = staged ? sl[lpad(gr - rb + t)] : lens[gr + t];
      w = max(w, l);
      nl += l > cut;
    }
    slots[g] = s * w;
    nlong[g] = nl;
    ss += s * w;
    ls += nl;
  }
  uint64_t ea, eb, ta, tb;
  block_scan_pair(ss, ls, ea, eb, ta, tb);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = ta;
    part[2 * blockIdx.x + 1] = tb;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // last CTA: exclusive scan of the tile sums in place, chunk by chunk
  __threadfence();
  const uint32_t nb = gridDim.x;
  uint64_t ca = 0, cb = 0;
  for (uint32_t c0 = 0; c0 < nb; c0 += kLayoutThreads) {
    const uint32_t i = c0 + threadIdx.x;
    const uint64_t va = i < nb ? __ldcg(part + 2 * i) : 0;
    const uint64_t vb = i < nb ? __ldcg(part + 2 * i + 1) : 0;
    block_scan_pair(va, vb, ea, eb, ta, tb);
    if (i < nb) part[2 * i] = ca + ea, part[2 * i + 1] = cb + eb;
    ca += ta;
    cb += tb;
  }
  if (threadIdx.x == 0) {
    tot[0] = ca;
    tot[1] = cb;
    tot[2] = (uint64_t)rp[r0 + rows] - rp[r0];
    *ticket = 0;
  }
}

__global__ void __launch_bounds__(kLayoutThreads) k1_layout_apply(
    uint64_t groups, uint64_t TG, const uint64_t* __restrict__ slots,
    uint64_t* __restrict__ nlong, const uint64_t* __restrict__ part,
    const uint64_t* __restrict__ tot, uint32_t* __restrict__ gp) {
  const uint64_t g0 = blockIdx.x * TG, g1 = min(groups, g0 + TG);
  const uint64_t q = (g1 - g0 + kLayoutThreads - 1) / kLayoutThreads;
  const uint64_t ga = min(g1, g0 + threadIdx.x * q), gb = min(g1, ga + q);
  uint64_t ss = 0, ls = 0;
  for (uint64_t g = ga; g < gb; ++g) ss += slots[g], ls += nlong[g];
  uint64_t ea, eb, ta, tb;
  block_scan_pair(ss, ls, ea, eb, ta, tb);
  ea += part[2 * blockIdx.x];
  eb += part[2 * blockIdx.x + 1];
  for (uint64_t g = ga; g < gb; ++g) {
    const uint64_t sv = slots[g], lv = nlong[g];
    gp[g] = (uint32_t)ea;
    nlong[g] = eb;
    ea += sv;
    eb += lv;
  }
  if (g1 == groups && threadIdx.x == 0) gp[groups] = (uint32_t)tot[0];
}

// out[0] = row_ptr[r1] - row_ptr[r0] (the slab's nnz)
__global__ void slab_nnz(const uint32_t* __restrict__ rp, uint64_t r0, uint64_t r1,
                         uint64_t* __restrict__ out) {
  *out = (uint64_t)rp[r1] - rp[r0];
}

__global__ void narrow_pointers(uint64_t groups, const uint64_t* __restrict__ gp64,
                                uint64_t total, uint32_t* __restrict__ gp) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g <= groups;
       g += (uint64_t)gridDim.x * blockDim.x)
    gp[g] = (uint32_t)(g == groups ? total : gp64[g]);
}

// The long rows in ascending order: group g writes its rows longer than the
// cut at its scanned offset off[g].
__global__ void long_rows_by_group(uint64_t rows, uint64_t G, uint64_t groups, uint32_t cut,
                                   const uint32_t* __restrict__ lens,
                                   const uint64_t* __restrict__ off, uint32_t* __restrict__ out) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = g * G, s = min(G, rows - r0);
    uint64_t o = off[g];
    for (uint64_t t = 0; t < s; ++t)
      if (lens[r0 + t] > cut) out[o++] = (uint32_t)(r0 + t);
  }
}

// ------------------------------------------------------------ to_triplets
// rgcsr.hpp:107-123: every row's real slots, in slot order, back to entries
// (values widened to double).  Thread per row into a scanned CSR.
__global__ void lens_u64(uint64_t rows, const uint32_t* __restrict__ lens,
                         uint64_t* __restrict__ out) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x)
    out[r] = lens[r];
}

template <class T>
__global__ void rgcsr_gather_rows(uint64_t rows, uint64_t G, uint64_t nnz,
                                  const uint32_t* __restrict__ gp,
                                  const uint32_t* __restrict__ lens, const T* __restrict__ values,
                                  const uint32_t* __restrict__ columns,
                                  const uint64_t* __restrict__ off, uint32_t* __restrict__ rp,
                                  uint32_t* __restrict__ col, double* __restrict__ val) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = r / G, s = min(G, rows - g * G);
    const uint64_t base = gp[g] + (r - g * G), o = off[r];
    rp[r] = (uint32_t)o;
    if (r + 1 == rows) rp[rows] = (uint32_t)nnz;
    for (uint32_t j = 0; j < lens[r]; ++j) {
      col[o + j] = columns[base + j * s];
      val[o + j] = static_cast<double>(values[base + j * s]);
    }
  }
}

// Rows longer than this go to the warp-per-row kernel (spmvk_set_long_row_cut).
std::atomic<uint32_t>& long_cut_slot() {
  static std::atomic<uint32_t> v{[] {
    const char* e = std::getenv("SPMVK_LONG_CUT");  // A/B only; default kLongRow
    const long n = e ? std::atol(e) : 0;
    return n > 0 ? static_cast<uint32_t>(n) : kLongRow;
  }()};
  return v;
}

// ------------------------------------------------------------ K1: scatter
// One warp per group.  Lane t owns local row t (+32 per chunk) and walks its
// slots j = 0..K_g-1; for a fixed j the warp writes 32 contiguous slots, and
// every pad slot is written (0, 0), so no separate zero-fill pass is needed.
// A group's CSR entries [rp[g G], rp[g G + s]) are contiguous: when they fit
// the warp's shared-memory stage (kStage entries) they are first copied in
// with coalesced loads, and the slot-major writes read them from there --
// instead of 32 scattered row streams per load instruction, which cost one
// L1 tag lookup per lane.  Larger groups (long rows) read CSR directly.
constexpr uint32_t kStage = 512;

template <class T, class V>
__global__ void __launch_bounds__(256) rgcsr_scatter(uint64_t r0, uint64_t rows, uint64_t G,
                                                     uint64_t groups,
                                                     const uint32_t* __restrict__ rp,
                                                     const uint32_t* __restrict__ col,
                                                     const V* __restrict__ val,
                                                     const uint32_t* __restrict__ gp,
                                                     const uint32_t* __restrict__ lens,
                                                     T* __restrict__ values,
                                                     uint32_t* __restrict__ columns) {
  extern __shared__ __align__(16) unsigned char stage_raw[];  // 8 warps x kStage (T + u32)
  T* sv_all = reinterpret_cast<T*>(stage_raw);
  uint32_t* sc_all = reinterpret_cast<uint32_t*>(sv_all + 8 * kStage);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* sv = sv_all + warp * kStage;
  uint32_t* sc = sc_all + warp * kStage;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t g = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp; g < groups; g += warps) {
    const uint64_t s = min(G, rows - g * G);
    const uint32_t base = gp[g];
    const uint64_t width = s ? (gp[g + 1] - base) / s : 0;
    if (s == 32) {  // full 32-row group: two 16-row halves, each staged if it fits
      for (uint32_t c0 = 0; c0 < 32; c0 += 16) {
        const uint64_t row = g * G + c0 + (lane & 15);
        const uint32_t len = lens[row];
        const uint32_t h0 = rp[r0 + g * G + c0], h1 = rp[r0 + g * G + c0 + 16];
        const uint32_t start = rp[r0 + row];
        const uint64_t t = c0 + (lane & 15);
        if (h1 - h0 <= kStage) {  // warp-uniform
          for (uint32_t i = lane; i < h1 - h0; i += 32) {
            sv[i] = static_cast<T>(val[h0 + i]);
            sc[i] = col[h0 + i];
          }
          __syncwarp();
          const uint32_t off = start - h0;
          // lanes 0-15 write even slots, 16-31 odd: each store instruction
          // covers two whole 16-row (128 B / 64 B) runs of the slab
          for (uint64_t j = lane >> 4; j < width; j += 2) {
            const uint64_t idx = base + t + j * 32;
            values[idx] = j < len ? sv[off + j] : T(0);
            columns[idx] = j < len ? sc[off + j] : 0u;
          }
          __syncwarp();
        } else {
          for (uint64_t j = lane >> 4; j < width; j += 2) {
            const uint64_t idx = base + t + j * 32;
            values[idx] = j < len ? static_cast<T>(val[start + j]) : T(0);
            columns[idx] = j < len ? col[start + j] : 0u;
          }
        }
      }
      continue;
    }
    const uint32_t e0 = rp[r0 + g * G], e1 = rp[r0 + g * G + s];
    if (s <= 32 && e1 - e0 <= kStage) {  // warp-uniform
      for (uint32_t i = lane; i < e1 - e0; i += 32) {
        sv[i] = static_cast<T>(val[e0 + i]);
        sc[i] = col[e0 + i];
      }
      __syncwarp();
      const bool live = (uint64_t)lane < s;
      const uint64_t row = g * G + lane;
      const uint32_t len = live ? lens[row] : 0;
      const uint32_t off = live ? rp[r0 + row] - e0 : 0;
      if (live)
        for (uint64_t j = 0; j < width; ++j) {
          const uint64_t idx = base + lane + j * s;
          values[idx] = j < len ? sv[off + j] : T(0);
          columns[idx] = j < len ? sc[off + j] : 0u;
        }
      __syncwarp();
      continue;
    }
    for (uint64_t t0 = 0; t0 < s; t0 += 32) {
      const uint64_t t = t0 + lane;
      const bool live = t < s;
      const uint64_t row = g * G + t;
      const uint32_t len = live ? lens[row] : 0;
      const uint32_t start = live ? rp[r0 + row] : 0;
      if (!live) continue;
      for (uint64_t j = 0; j < width; ++j) {
        const uint64_t idx = base + t + j * s;
        if (j < len) {
          values[idx] = static_cast<T>(val[start + j]);
          columns[idx] = col[start + j];
        } else {
          values[idx] = T(0);
          columns[idx] = 0;
        }
      }
    }
  }
}

// K1 scatter with 1D bulk async copies (TMA, cp.async.bulk + mbarrier):
// each warp owns a static sequence of groups; a full 32-row group's CSR block
// [rp[g G], rp[g G + 32]) (values, columns; rounded out to 16-byte bounds) is
// brought into one of the warp's two shared-memory stages by two bulk copies
// issued by lane 0, the NEXT group's block is in flight while this group's
// slots are written (slot-major, coalesced, pads included) from the other
// stage.  Partial groups and blocks that do not fit the stage are written
// straight from CSR.  The default K1 scatter (SPMVK_K1_BULK=0 selects the
// staged rgcsr_scatter above).
constexpr uint32_t kBulkStage = 1024;  // entries per stage (+ 4 of alignment slack)

template <class T, class V>
__global__ void __launch_bounds__(128) rgcsr_scatter_bulk(uint64_t r0, uint64_t rows, uint64_t G,
                                                          uint64_t groups,
                                                          const uint32_t* __restrict__ rp,
                                                          const uint32_t* __restrict__ col,
                                                          const V* __restrict__ val,
                                                          const uint32_t* __restrict__ gp,
                                                          const uint32_t* __restrict__ lens,
                                                          T* __restrict__ values,
                                                          uint32_t* __restrict__ columns) {
  constexpr uint32_t SV = (kBulkStage + 4) * sizeof(V), SC = (kBulkStage + 4) * 4;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = sm + (size_t)warp * 2 * (SV + SC);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)4 * 2 * (SV + SC)) + warp * 2;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t first = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // stage b of group g: returns whether a copy was issued
  auto full_and_fits = [&](uint64_t g) {
    if (g >= groups || (g + 1) * G > rows || G != 32) return false;
    return rp[r0 + g * G + 32] - rp[r0 + g * G] <= kBulkStage;
  };
  auto issue = [&](uint64_t g, int b) {
    const uint32_t e0 = rp[r0 + g * G], e1 = rp[r0 + g * G + 32];
    const uint64_t v0 = (uint64_t)e0 * sizeof(V) & ~15ull;
    const uint64_t v1 = ((uint64_t)e1 * sizeof(V) + 15) & ~15ull;
    const uint64_t c0 = (uint64_t)e0 * 4 & ~15ull, c1 = ((uint64_t)e1 * 4 + 15) & ~15ull;
    unsigned char* sv = wbase + b * (SV + SC);
    mbar_arrive_expect_tx(&bar[b], (uint32_t)(v1 - v0 + c1 - c0));
    bulk_g2s(sv, reinterpret_cast<const unsigned char*>(val) + v0, (uint32_t)(v1 - v0), &bar[b]);
    bulk_g2s(sv + SV, reinterpret_cast<const unsigned char*>(col) + c0, (uint32_t)(c1 - c0),
             &bar[b]);
  };
  uint32_t phase[2] = {0, 0};
  bool staged = first < groups && full_and_fits(first);
  if (staged && lane == 0) issue(first, 0);
  int b = 0;
  for (uint64_t g = first; g < groups; g += warps, b ^= 1) {
    const uint64_t gn = g + warps;
    const bool staged_n = full_and_fits(gn);
    if (staged_n && lane == 0) {
      fence_proxy_async_smem();  // stage 1-b was read (generic proxy) by the previous group
      issue(gn, b ^ 1);
    }
    const uint64_t s = min(G, rows - g * G);
    const uint32_t base = gp[g];
    const uint64_t width = s ? (gp[g + 1] - base) / s : 0;
    if (staged) {
      mbar_wait(&bar[b], phase[b]);
      phase[b] ^= 1;
      const uint32_t e0 = rp[r0 + g * G];
      const V* sv = reinterpret_cast<const V*>(wbase + b * (SV + SC)) +
                    ((uint64_t)e0 * sizeof(V) & 15) / sizeof(V);
      const uint32_t* sc = reinterpret_cast<const uint32_t*>(wbase + b * (SV + SC) + SV) +
                           ((uint64_t)e0 * 4 & 15) / 4;
      const uint64_t row = g * G + lane;
      const uint32_t len = lens[row];
      const uint32_t off = rp[r0 + row] - e0;
      for (uint64_t j = 0; j < width; ++j) {
        const uint64_t idx = base + lane + j * 32;
        values[idx] = j < len ? static_cast<T>(sv[off + j]) : T(0);
        columns[idx] = j < len ? sc[off + j] : 0u;
      }
      __syncwarp();
    } else {
      for (uint64_t t0 = 0; t0 < s; t0 += 32) {
        const uint64_t t = t0 + lane;
        if (t >= s) continue;
        const uint64_t row = g * G + t;
        const uint32_t len = lens[row];
        const uint32_t start = rp[r0 + row];
        for (uint64_t j = 0; j < width; ++j) {
          const uint64_t idx = base + t + j * s;
          values[idx] = j < len ? static_cast<T>(val[start + j]) : T(0);
          columns[idx] = j < len ? col[start + j] : 0u;
        }
      }
      __syncwarp();
    }
    staged = staged_n;
  }
}

// Quads for rgcsr_spmv_long_mixed: rows r..r+3 (r % 4 == 0) all long, in one
// full group of a G % 4 == 0 matrix, each shorter than kQuadMaxLen (the
// longest rows keep a warp each: a quad walks 64 slots per round, so a
// 4096-slot row would be its critical path).  SPMVK_LONG_QUADS=0 disables.
constexpr uint32_t kQuadMaxLen = 1024;

// Long row i (ascending ids lr[]): is it the first row of a quad (rows r..r+3,
// r % 4 == 0, all long, each shorter than kQuadMaxLen, inside one full group
// of a G % 4 == 0 matrix), and does it belong to any quad?  A quad starts on
// a multiple of 4 and covers 4 consecutive ids, so membership of row r is
// the quad test of r & ~3.  Sort keys put the singles first, longest first
// (stable: ties keep ascending ids), the quad members after them.
__device__ __forceinline__ bool quad_at(uint64_t i, uint64_t n, const uint32_t* __restrict__ lr,
                                        const uint32_t* __restrict__ lens, uint64_t rows,
                                        uint64_t G) {
  const uint32_t r = lr[i];
  if (r % 4 || G % 4 || i + 3 >= n) return false;
  const uint64_t g = r / G;
  if ((g + 1) * G > rows || (r + 3) / G != g) return false;
  for (int k = 0; k < 4; ++k)
    if (lr[i + k] != r + k || lens[r + k] >= kQuadMaxLen) return false;
  return true;
}

__global__ void long_split(uint64_t n, uint64_t rows, uint64_t G, int quads_on,
                           const uint32_t* __restrict__ lr, const uint32_t* __restrict__ lens,
                           uint64_t* __restrict__ qflag, uint32_t* __restrict__ key) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = lr[i];
    const bool start = quads_on && quad_at(i, n, lr, lens, rows, G);
    bool member = start;
    if (quads_on && !start && r % 4) {  // the quad test of r & ~3, at index i - r % 4
      const uint64_t d = r % 4;
      member = i >= d && lr[i - d] == r - d && quad_at(i - d, n, lr, lens, rows, G);
    }
    qflag[i] = start ? 1 : 0;
    key[i] = member ? 0xffffffffu : 0xfffffffeu - lens[r];
  }
}

__global__ void count_singles(uint64_t n, uint64_t* __restrict__ counts) {
  counts[1] = n - 4 * counts[0];
}

__global__ void quad_scatter(uint64_t n, const uint32_t* __restrict__ lr,
                             const uint64_t* __restrict__ qflag, const uint64_t* __restrict__ qpos,
                             uint32_t* __restrict__ quads) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (qflag[i]) quads[qpos[i]] = lr[i];
}

// Device split of the long rows (lr, ascending) into quads and singles
// (longest first) for rgcsr_spmv_long_mixed.  The two counts land in
// counts_dev[0] (quads) and counts_dev[1] (singles).
void split_long_rows(spmvk_rgcsr* h, uint32_t G, uint64_t* counts_dev, cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("SPMVK_LONG_QUADS");
    return !e || std::atoi(e) != 0;
  }();
  const uint64_t n = h->n_long;
  const unsigned grid = persistent_grid((n + 255) / 256, 8);
  TmpBuf<uint64_t> qflag(n, s);
  TmpBuf<uint32_t> key(n, s), key2(n, s);
  long_split<<<grid, 256, 0, s>>>(n, h->rows, G, on ? 1 : 0, h->long_rows.p, h->row_lengths.p,
                                  qflag.p, key.p);
  SPMVK_LAUNCH("long_split");
  // singles first (longest first, stable), quad members last
  h->long_singles.alloc(n);
  size_t tmp_bytes = 0;
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.p, key2.p, h->long_rows.p,
                                             h->long_singles.p, static_cast<int>(n), 0, 32, s));
  TmpBuf<unsigned char> tmp(tmp_bytes, s);
  SPMVK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key.p, key2.p, h->long_rows.p,
                                             h->long_singles.p, static_cast<int>(n), 0, 32, s));
  // quads: compaction of the starts (ascending)
  TmpBuf<uint64_t> qpos(n, s);
  SPMVK_CUDA(cudaMemcpyAsync(qpos.p, qflag.p, 8 * n, cudaMemcpyDeviceToDevice, s));
  exclusive_scan_u64_dev(qpos.p, n, s, counts_dev);
  h->long_quads.alloc(n / 4 + 1);
  quad_scatter<<<grid, 256, 0, s>>>(n, h->long_rows.p, qflag.p, qpos.p, h->long_quads.p);
  SPMVK_LAUNCH("quad_scatter");
  count_singles<<<1, 1, 0, s>>>(n, counts_dev);
  SPMVK_LAUNCH("count_singles");
}

// K1 on the device with two host round trips: the slot total, long-row
// count and nnz (one 24-byte readback, needed to size the arrays and to
// report a uint32 overflow before writing), and the quad / single counts at
// the end.  Scratch arrays are stream-ordered (no device-wide syncs).
spmvk_rgcsr* build(const spmvk_csr* a, uint64_t r0, uint64_t r1, uint64_t G, int prec,
                   cudaStream_t s) {
  if (!a) fail(SPMVK_EINVAL, "null CSR handle");
  if (G == 0) fail(SPMVK_EINVAL, "build_rgcsr: group size must be nonzero");
  if (prec != SPMVK_F32 && prec != SPMVK_F64)
    fail(SPMVK_EINVAL, "precision must be SPMVK_F32 (4) or SPMVK_F64 (8)");
  if (a->val_prec == SPMVK_F32 && prec == SPMVK_F64)
    fail(SPMVK_EINVAL, "cannot build a double RgCSR from a float CSR");
  if (r0 > r1 || r1 > a->rows) fail(SPMVK_EINVAL, "row range outside the matrix");
  if (r0 % G) fail(SPMVK_EINVAL, "row slab must start on a group boundary");
  auto h = std::make_unique<spmvk_rgcsr>();
  h->rows = r1 - r0;
  h->cols = a->cols;
  h->group_size = G;
  h->prec = prec;
  h->groups = (h->rows + G - 1) / G;
  h->long_cut = long_cut_slot().load();
  h->row_lengths.alloc(h->rows);
  h->group_pointers.alloc(h->groups + 1);
  const unsigned rgrid = persistent_grid((h->rows + 255) / 256, 8);
  const unsigned ggrid = persistent_grid((h->groups + 255) / 256, 8);
  TmpBuf<uint64_t> tot(5, s);  // slots, long rows, nnz | quads, singles
  TmpBuf<uint64_t> slots(h->groups, s), nlong(h->groups, s);
  // SPMVK_K1_LAYOUT=0: the unfused layout kernels + scans (A/B only)
  static const bool fused_layout = [] {
    const char* e = std::getenv("SPMVK_K1_LAYOUT");
    return !e || std::atoi(e) != 0;
  }();
  if (fused_layout && h->groups) {
    const uint64_t TG = std::max<uint64_t>(1, kLayoutRows / G);
    const uint64_t ntiles = (h->groups + TG - 1) / TG;
    if (ntiles > 0x7fffffffull) fail(SPMVK_ERANGE, "build_rgcsr: too many row tiles");
    TmpBuf<uint64_t> part(2 * ntiles, s);
    k1_layout<<<static_cast<unsigned>(ntiles), kLayoutThreads, 0, s>>>(
        r0, h->rows, G, h->groups, TG, h->long_cut, a->row_ptr.p, h->row_lengths.p, slots.p,
        nlong.p, part.p, stream_counters(s) + 3, tot.p);
    SPMVK_LAUNCH("k1_layout");
    k1_layout_apply<<<static_cast<unsigned>(ntiles), kLayoutThreads, 0, s>>>(
        h->groups, TG, slots.p, nlong.p, part.p, tot.p, h->group_pointers.p);
    SPMVK_LAUNCH("k1_layout_apply");
  } else {
    if (h->rows) {
      csr_row_lengths<<<rgrid, 256, 0, s>>>(r0, h->rows, a->row_ptr.p, h->row_lengths.p);
      SPMVK_LAUNCH("csr_row_lengths");
      group_layout<<<ggrid, 256, 0, s>>>(h->rows, G, h->groups, h->long_cut, h->row_lengths.p,
                                         slots.p, nlong.p);
      SPMVK_LAUNCH("group_layout");
    }
    exclusive_scan_u64_dev(slots.p, h->groups, s, tot.p);
    exclusive_scan_u64_dev(nlong.p, h->groups, s, tot.p + 1);
    slab_nnz<<<1, 1, 0, s>>>(a->row_ptr.p, r0, r1, tot.p + 2);
    SPMVK_LAUNCH("slab_nnz");
  }
  uint64_t* t3 = pinned_slot();
  SPMVK_CUDA(cudaMemcpyAsync(t3, tot.p, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  SPMVK_CUDA(cudaStreamSynchronize(s));
  const uint64_t total = t3[0];
  if (total > 0xffffffffull)
    fail(SPMVK_ERANGE, "build_rgcsr: " + std::to_string(total) +
                           " slots overflow the 32-bit group pointers (group size " +
                           std::to_string(G) + ")");
  h->slots = total;
  h->n_long = t3[1];
  h->nnz = t3[2];
  if (!fused_layout || !h->groups) {
    narrow_pointers<<<persistent_grid((h->groups + 256) / 256, 8), 256, 0, s>>>(
        h->groups, slots.p, total, h->group_pointers.p);
    SPMVK_LAUNCH("narrow_pointers");
  }
  h->values.alloc(total * static_cast<uint64_t>(prec));
  h->columns.alloc(total);
  if (h->groups) {
    auto scatter = [&](auto kern, auto* vals_in, auto* vals_out) {
      using TO = std::remove_pointer_t<decltype(vals_out)>;
      const size_t smem = 8 * kStage * (sizeof(TO) + sizeof(uint32_t));
      SPMVK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      int per_sm = 0;
      SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
      const unsigned sgrid = persistent_grid((h->groups + 7) / 8, per_sm > 0 ? per_sm : 1);
      kern<<<sgrid, 256, smem, s>>>(r0, h->rows, G, h->groups, a->row_ptr.p, a->col.p, vals_in,
                                    h->group_pointers.p, h->row_lengths.p, vals_out,
                                    h->columns.p);
      SPMVK_LAUNCH("rgcsr_scatter");
    };
    // bulk-copy scatter (default; SPMVK_K1_BULK=0 -> the shared-memory staged
    // kernel): 27-pt 128^3 fp64 207 vs 271 us (profiles/r02b_ncu_k1_scatter.md)
    static const bool k1_bulk = [] {
      const char* e = std::getenv("SPMVK_K1_BULK");
      return !e || std::atoi(e) != 0;
    }();
    auto scatter_bulk = [&](auto kern, auto* vals_in, auto* vals_out) {
      using VI = std::remove_const_t<std::remove_pointer_t<decltype(vals_in)>>;
      const size_t smem = 4 * 2 * ((kBulkStage + 4) * (sizeof(VI) + 4)) + 4 * 2 * 8;
      SPMVK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      int per_sm = 0;
      SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
      const unsigned sgrid = persistent_grid((h->groups + 3) / 4, per_sm > 0 ? per_sm : 1);
      kern<<<sgrid, 128, smem, s>>>(r0, h->rows, G, h->groups, a->row_ptr.p, a->col.p, vals_in,
                                    h->group_pointers.p, h->row_lengths.p, vals_out,
                                    h->columns.p);
      SPMVK_LAUNCH("rgcsr_scatter_bulk");
    };
    if (k1_bulk && prec == SPMVK_F64)
      scatter_bulk(rgcsr_scatter_bulk<double, double>, reinterpret_cast<const double*>(a->val.p),
                   reinterpret_cast<double*>(h->values.p));
    else if (k1_bulk && a->val_prec == SPMVK_F64)
      scatter_bulk(rgcsr_scatter_bulk<float, double>, reinterpret_cast<const double*>(a->val.p),
                   reinterpret_cast<float*>(h->values.p));
    else if (k1_bulk)
      scatter_bulk(rgcsr_scatter_bulk<float, float>, reinterpret_cast<const float*>(a->val.p),
                   reinterpret_cast<float*>(h->values.p));
    else if (prec == SPMVK_F64)
      scatter(rgcsr_scatter<double, double>, reinterpret_cast<const double*>(a->val.p),
              reinterpret_cast<double*>(h->values.p));
    else if (a->val_prec == SPMVK_F64)
      scatter(rgcsr_scatter<float, double>, reinterpret_cast<const double*>(a->val.p),
              reinterpret_cast<float*>(h->values.p));
    else
      scatter(rgcsr_scatter<float, float>, reinterpret_cast<const float*>(a->val.p),
              reinterpret_cast<float*>(h->values.p));
  }
  h->long_rows.alloc(h->n_long);
  if (h->n_long) {  // long-row list (ascending), split into quads and singles
    long_rows_by_group<<<ggrid, 256, 0, s>>>(h->rows, G, h->groups, h->long_cut,
                                             h->row_lengths.p, nlong.p, h->long_rows.p);
    SPMVK_LAUNCH("long_rows_by_group");
    split_long_rows(h.get(), static_cast<uint32_t>(G), tot.p + 3, s);
    uint64_t* qs = pinned_slot() + 3;
    SPMVK_CUDA(cudaMemcpyAsync(qs, tot.p + 3, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    SPMVK_CUDA(cudaStreamSynchronize(s));
    h->n_quads = qs[0];
    h->n_singles = qs[1];
  } else {
    SPMVK_CUDA(cudaStreamSynchronize(s));
  }
  return h.release();
}

template <class T>
void check_spmv_args(const spmvk_rgcsr* h, uint64_t nx, uint64_t ny) {
  if (!h) fail(SPMVK_EINVAL, "null RgCSR handle");
  if (nx != h->cols || ny != h->rows) fail(SPMVK_EINVAL, "spmv_rgcsr: dimension mismatch");
  if (h->prec != static_cast<int>(sizeof(T)))
    fail(SPMVK_EINVAL, "spmv_rgcsr: handle precision differs from the entry point");
}

// K2 variant selection: spmvk_set_rgcsr_kernel() or SPMVK_RGCSR_KERNEL.
// All variants give bitwise identical y; they differ in how slots are staged.
// Round 2 pruned the variants that never won a measured case (TMA rings,
// L2 bulk prefetch, x staged in shared memory, policy-hinted ldg, deeper
// pipes; numbers in profiles/r02_k2_pruned.md).
// "liteh" / "lite8h": lite / lite8 with L2 eviction hints (slot streams
// evict_first, x evict_last), for matrices whose x competes with a large
// slot stream for L2 (power-law).
enum class K2 {
  kAuto, kPipe, kLite, kLite8, kLite8Full, kLiteH, kLite8H, kVec2, kGrp6, kGrp7Mpf, kGrp8, kGrp8R64,
  kGrpV4
};

// "auto" (default): the variant that measured fastest on B200 across the
// stencil shapes (profiles/r01_k2_sweep.md): the register-lean tile kernel —
// 8-deep batches at 40 warps / SM for fp64 (lite8), 4-deep at full occupancy
// (64 warps / SM) for fp32 (lite).  Occupancy beats deeper per-thread
// pipelines: every variant with prefetch buffers lost to it.
// Irregular matrices (rows beyond the long-row cut, e.g. the power-law
// config) favour the row-prefetching `pipe` kernel in fp32
// (profiles/r01_powerlaw.md: 1,070 vs 1,353 us).
K2 auto_k2(const spmvk_rgcsr* h, bool f64) {
  // No long rows and <= 10 % padding (stencils, banded): the group-uniform
  // walk (rgcsr_spmv_grp) -- one batch of slot loads per row, ordered ahead
  // of the x gathers, next row's group pointers prefetched.  Measured
  // (profiles/r01_k2_grp.md, back-to-back us): 5-pt 2048^2 fp64 47.2 vs 57.7
  // (vec2), fp32 35.5 vs 35.7; 7-pt 384^3 fp64 842 vs 934 (lite8), fp32
  // 607 vs 651 (lite); 27-pt 128^3 fp64 102.6 vs 105.5, fp32 75.5 vs 80.7.
  if (!h->n_long && h->slots * 10 <= h->nnz * 11) {
    // fp32 with <= 12 slots per row (5- and 7-point class): the group walk
    // with 128-bit slot loads, 4 rows per thread (rgcsr_spmv_grpv): 5-pt
    // 2048^2 32.9 vs 34.7 us, 7-pt 256^3 175.0 vs 180.8, 7-pt 384^3 567 vs
    // 600, 5-pt 1024^2 11.2 vs 11.3; 27-pt 72.8 vs 71.5 and every fp64 case
    // lose (profiles/r02_grpv.md)
    if (!f64 && h->slots <= 12 * h->rows && h->group_size % 4 == 0) return K2::kGrpV4;
    if (2 * h->slots <= 11 * h->rows) return K2::kGrp6;
    if (f64) return K2::kGrp8R64;
    return h->slots <= 12 * h->rows ? K2::kGrp8 : K2::kGrp7Mpf;
  }
  // <= 5.5 slots per row (5-point class): two / four rows per thread with
  // 128-bit value loads win (5-pt 4096^2: fp64 220 vs 232 us, fp32 152 vs
  // 163 us); from 7 slots on they lose (profiles/r01_k2_sweep3.md)
  if (!h->n_long && 2 * h->slots <= 11 * h->rows) return K2::kVec2;
  // long rows: the row-pipelined kernel with the long rows fused in and its
  // rows taken in dynamic 128-row slices (rgcsr_spmv_pipe_fl).  Config-3
  // power-law 8M, best of 5 x 20 back-to-back (profiles/r02_long_fused.md):
  // original order fp64 1,222 us (was lite8 + separate long-row launch
  // 1,419), fp32 925 (1,044); descending order fp64 557 (607), fp32 511 (564)
  if (h->n_long) return K2::kPipe;
  // ragged rows without long ones (> 10 % padding; the sweep's random class):
  // the row-pipelined kernel, static rows (scripts/probes/random_ab.py:
  // 0.8-7.2 M rows, mean 17-58, fp32 lite 124-2,321 us -> 96-1,833, fp64
  // lite8 117-2,417 -> 113-2,246; 18 k rows equal; profiles/r02_long_fused.md)
  if (h->rows >= (1u << 16)) return K2::kPipe;
  if (f64) return K2::kLite8;
  // fp32, short rows (<= ~12 slots): one 8-deep batch per row at full
  // occupancy (32 registers, no spills) keeps more slot bytes in flight
  // (7-pt 256^3: 193 vs 201 us; 5-pt 1024^2: 14.6 vs 16.7 us); longer rows
  // (27-pt: 88 vs 78 us) prefer 4-deep batches (profiles/r01_k2_sweep3.md)
  return h->slots <= 12 * h->rows ? K2::kLite8Full : K2::kLite;
}

bool parse_k2(const std::string& v, K2* out) {
  static const std::pair<const char*, K2> names[] = {
      {"auto", K2::kAuto},         {"pipe", K2::kPipe},         {"lite", K2::kLite},
      {"lite8", K2::kLite8},       {"lite8_full", K2::kLite8Full}, {"vec2", K2::kVec2},
      {"grp6", K2::kGrp6},         {"grp7_mpf", K2::kGrp7Mpf},  {"grp8", K2::kGrp8},
      {"grp8_r64", K2::kGrp8R64},  {"liteh", K2::kLiteH},      {"lite8h", K2::kLite8H},
      {"grpv4", K2::kGrpV4}};
  for (const auto& [n, k] : names)
    if (v == n) {
      *out = k;
      return true;
    }
  return false;
}

std::atomic<int>& k2_slot() {
  static std::atomic<int> k{[] {
    K2 v = K2::kAuto;
    const char* e = std::getenv("SPMVK_RGCSR_KERNEL");
    if (e) parse_k2(e, &v);
    return static_cast<int>(v);
  }()};
  return k;
}

K2 k2_choice() { return static_cast<K2>(k2_slot().load(std::memory_order_relaxed)); }

// The rows past the long-row cut: singles (warp per row, longest first) and
// quads (four rows per warp) in one launch after the thread-per-row kernel.
// hint: L2 eviction hints on the long rows' slot streams and x gathers
// (SPMVK_LONG_HINT=0/1 forces them off/on).
template <class T, bool kScaled>
void launch_long(const spmvk_rgcsr* h, uint32_t G, int sh, const T* x, T* y, T* x_next, T scale,
                 cudaStream_t s, bool hint) {
  static const int env = [] {
    const char* e = std::getenv("SPMVK_LONG_HINT");
    return e ? std::atoi(e) : -1;
  }();
  if (env >= 0) hint = env > 0;
  const uint64_t items = h->n_singles + h->n_quads;
  auto kern = hint ? rgcsr_spmv_long_mixed<T, kScaled, true>
                   : rgcsr_spmv_long_mixed<T, kScaled, false>;
  kern<<<persistent_grid((items + 7) / 8, 8), 256, 0, s>>>(
      static_cast<uint32_t>(h->n_singles), h->long_singles.p, static_cast<uint32_t>(h->n_quads),
      h->long_quads.p, static_cast<uint32_t>(h->rows), G, sh, h->group_pointers.p,
      h->row_lengths.p, reinterpret_cast<const T*>(h->values.p), h->columns.p, x, y, x_next,
      scale);
  SPMVK_LAUNCH("rgcsr_spmv_long_mixed");
}

// A matrix without stored slots (nnz = 0, e.g. cols = 0): every row sums
// nothing, so y = +0 (the reference's acc start) -- without touching x, which
// may be a zero-length (null) array.
template <class T, bool kScaled>
__global__ void spmv_empty(uint64_t rows, T* __restrict__ y, T* __restrict__ x_next, T scale) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    y[r] = T(0);
    if (kScaled) x_next[r] = mul_rn(T(0), scale);
  }
}

// Long rows fused into the tile kernel (default) or a separate launch after
// it: spmvk_set_long_fused() / SPMVK_LONG_FUSED=0.
std::atomic<int>& long_fused_slot() {
  static std::atomic<int> v{[] {
    const char* e = std::getenv("SPMVK_LONG_FUSED");
    return (!e || std::atoi(e) != 0) ? 1 : 0;
  }()};
  return v;
}

template <class T, bool kScaled>
void launch_spmv(const spmvk_rgcsr* h, const T* x, T* y, T* x_next, T scale, cudaStream_t s) {
  if (h->rows == 0) return;
  if (h->slots == 0) {
    spmv_empty<T, kScaled><<<persistent_grid((h->rows + 255) / 256, 8), 256, 0, s>>>(
        h->rows, y, x_next, scale);
    SPMVK_LAUNCH("spmv_empty");
    return;
  }
  constexpr bool f64 = sizeof(T) == 8;
  K2 k = k2_choice();
  if (k == K2::kAuto) k = auto_k2(h, f64);
  // the group-uniform walk has no long-row split: matrices with long rows
  // (and, for now, any request on them) take the lite kernel instead
  if (k >= K2::kGrp6 && h->n_long) k = f64 ? K2::kLite8 : K2::kLite;
  // the vector walk needs groups of whole vectors
  if (k == K2::kGrpV4 && h->group_size % (16 / sizeof(T)) != 0)
    k = f64 ? K2::kGrp8R64 : K2::kGrp8;
  const bool hinted = k == K2::kLiteH || k == K2::kLite8H || k == K2::kPipe;
  const uint32_t G = static_cast<uint32_t>(std::min<uint64_t>(h->group_size, 0xffffffffull));
  const int sh = pow2_shift(h->group_size);
  constexpr int U = sizeof(T) == 8 ? 4 : 8;
  // rows longer than h->long_cut go to the warp-per-row kernel (launched second,
  // same stream; the two kernels write disjoint rows of y)
  const uint32_t long_cut = h->n_long ? h->long_cut : 0xffffffffu;
  // grp kernels: the last argument is the x L2-prefetch length instead of the
  // long-row cut (they never see long rows).  x is prefetched for short rows
  // (<= 5.5 slots per row) when it is at most 48 MB: measured with
  // scripts/cold_spmv.py (flush + SpMV, 3 runs each) 5-pt 2048^2 fp64 49.5-50.5
  // -> 47.2-47.8 us, fp32 39.1-39.3 -> 38.5-39.0 us, 5-pt 1024^2 neutral; it
  // costs 4 % on 7-pt 256^3 (x 134 MB: evicted before use) and ~1 % on 27-pt
  // (profiles/r01_k2_grp.md).  SPMVK_X_PREFETCH=0/1 forces it off/on.
  static const int xpf_env = [] {
    const char* e = std::getenv("SPMVK_X_PREFETCH");
    return e ? std::atoi(e) : -1;
  }();
  // cp.async.bulk.prefetch needs a 16-byte aligned start: an offset view of
  // x (only 4- or 8-byte aligned) is gathered without the prefetch
  const bool x_aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const bool xpf = x_aligned && (xpf_env >= 0 ? xpf_env > 0
                                              : (2 * h->slots <= 11 * h->rows &&
                                                 h->cols * sizeof(T) <= (48ull << 20)));
  // small matrices (format + x <= 24 MB, a fifth of L2): prefetch the slot
  // arrays, the group pointers and x at launch, whatever the row shape -- a
  // cold launch of a small SpMV is one dependent chain of three DRAM round
  // trips otherwise (profiles/r02b_sweep200.md: 10^4-row banded matrices
  // ran 10.2 vs 8.2 us for ELL, which has no group pointers).
  // SPMVK_SMALL_PREFETCH=0 turns it off.
  static const int small_env = [] {
    const char* e = std::getenv("SPMVK_SMALL_PREFETCH");
    return e ? std::atoi(e) : -1;
  }();
  const uint64_t fmt_bytes = h->slots * (sizeof(T) + 4) + 4 * (h->groups + 1) +
                             sizeof(T) * h->cols;
  const bool small = x_aligned && small_env != 0 && fmt_bytes <= (24ull << 20) &&
                     (reinterpret_cast<uintptr_t>(h->values.p) & 15) == 0;
  const bool xpf_small = xpf || small;
  // Programmatic dependent launch for the group walk (default; SPMVK_PDL=0
  // turns it off): a launch may start while the previous kernel on the stream
  // drains, reads only the immutable group pointers, and waits
  // (griddepcontrol.wait) before touching x or y.  Back-to-back SpMVs:
  // 27-pt 128^3 fp64 102.8 -> 101.6 us, 7-pt 256^3 245.9 -> 244.0, 5-pt
  // 1024^2 (L2-resident) 16.2 -> 13.6 (profiles/r02_ab.md).
  static const bool pdl = [] {
    const char* e = std::getenv("SPMVK_PDL");
    return !e || std::atoi(e) != 0;
  }();
  auto launch_grp = [&](auto kern, bool programmatic) {
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const unsigned grid = persistent_grid((h->rows + 255) / 256, per_sm > 0 ? per_sm : 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = programmatic ? 1 : 0;
    SPMVK_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<uint32_t>(h->rows), G, sh,
                                  (const uint32_t*)h->group_pointers.p,
                                  (const uint32_t*)h->row_lengths.p,
                                  reinterpret_cast<const T*>(h->values.p),
                                  (const uint32_t*)h->columns.p, x, y, x_next, scale,
                                  xpf_small ? static_cast<uint32_t>(h->cols) : 0u,
                                  small ? static_cast<uint32_t>(h->slots) : 0u));
    SPMVK_LAUNCH("rgcsr_spmv_grp");
  };
  auto run_grp = [&](auto kern, auto kern_pdl) {
    if (pdl) launch_grp(kern_pdl, true);
    else launch_grp(kern, false);
  };
  // persistent grid: exactly the resident CTAs of this variant (occupancy API)
  auto run = [&](auto kern) {
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const unsigned grid = persistent_grid((h->rows + 255) / 256, per_sm > 0 ? per_sm : 1);
    kern<<<grid, 256, 0, s>>>(static_cast<uint32_t>(h->rows), G, sh, h->group_pointers.p,
                              h->row_lengths.p, reinterpret_cast<const T*>(h->values.p),
                              h->columns.p, x, y, x_next, scale, long_cut);
    SPMVK_LAUNCH("rgcsr_spmv (thread per row)");
    // the long rows after it on the same stream (a forked concurrent launch
    // was measured 13 % slower: profiles/r02_ab.md)
    if (h->n_long) launch_long<T, kScaled>(h, G, sh, x, y, x_next, scale, s, hinted);
  };
  // the long rows fused into the tile kernel (default; SPMVK_LONG_FUSED=0
  // restores the separate launch): warps take the long-row items first, then
  // their tiles (rgcsr_spmv.cuh long_items_dynamic)
  // SPMVK_PIPE_DYN=1 (A/B): the pipe variant takes its rows in dynamic slices
  // even without long rows
  static const bool pipe_dyn_all = [] {
    const char* e = std::getenv("SPMVK_PIPE_DYN");
    return e && std::atoi(e) != 0;
  }();
  auto run_fl = [&](auto kern, auto kern_fl, bool dyn_ok = false) {
    if (!(h->n_long || (dyn_ok && pipe_dyn_all)) ||
        !long_fused_slot().load(std::memory_order_relaxed))
      return run(kern);
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern_fl, 256, 0));
    const unsigned grid = persistent_grid((h->rows + 255) / 256, per_sm > 0 ? per_sm : 1);
    static const uint32_t lw = [] {
      const char* e = std::getenv("SPMVK_LONG_WARPS");
      const int v = e ? std::atoi(e) : 2;  // 2 / 4 / 8 measured: 2 best (r02_long_fused.md)
      return static_cast<uint32_t>(v < 1 ? 1 : v > 8 ? 8 : v);
    }();
    const LongList ll{static_cast<uint32_t>(h->n_singles), static_cast<uint32_t>(h->n_quads),
                      h->long_singles.p, h->long_quads.p, stream_counters(s), lw};
    kern_fl<<<grid, 256, 0, s>>>(static_cast<uint32_t>(h->rows), G, sh, h->group_pointers.p,
                                 h->row_lengths.p, reinterpret_cast<const T*>(h->values.p),
                                 h->columns.p, x, y, x_next, scale, long_cut, ll);
    SPMVK_LAUNCH("rgcsr_spmv (long rows fused)");
  };
  auto run_grpv = [&](auto kern) {
    constexpr uint64_t R = 16 / sizeof(T);
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const unsigned grid = persistent_grid((h->rows + 256 * R - 1) / (256 * R),
                                          per_sm > 0 ? per_sm : 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    SPMVK_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<uint32_t>(h->rows), G, sh,
                                  (const uint32_t*)h->group_pointers.p,
                                  (const uint32_t*)h->row_lengths.p,
                                  reinterpret_cast<const T*>(h->values.p),
                                  (const uint32_t*)h->columns.p, x, y, x_next, scale,
                                  small ? static_cast<uint32_t>(h->cols) : 0u,
                                  small ? static_cast<uint32_t>(h->slots) : 0u));
    SPMVK_LAUNCH("rgcsr_spmv_grpv");
  };
  // vectorised kernels: tiles of 256 * R rows (R = 16 bytes / sizeof(T))
  auto run_vec = [&](auto kern) {
    constexpr uint64_t R = sizeof(T) == 8 ? 2 : 4;
    int per_sm = 0;
    SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const unsigned grid = persistent_grid((h->rows + 256 * R - 1) / (256 * R),
                                          per_sm > 0 ? per_sm : 1);
    kern<<<grid, 256, 0, s>>>(static_cast<uint32_t>(h->rows), G, sh, h->group_pointers.p,
                              h->row_lengths.p, reinterpret_cast<const T*>(h->values.p),
                              h->columns.p, x, y, x_next, scale, long_cut);
    SPMVK_LAUNCH("rgcsr_spmv_vec");
    if (h->n_long) launch_long<T, kScaled>(h, G, sh, x, y, x_next, scale, s, false);
  };
  // the group-uniform walk has no long-row split: matrices with long rows
  // (and, for now, any request on them) take the lite kernel instead

  switch (k) {
    // group-uniform walk: <T, kScaled, U, MINB, kNoLen, kMpf>
    // grp6 / grp7_mpf gather x for every slot < K (kGatherK): 5-pt 2048^2
    // fp32 35.1 vs 35.5 us, fp64 47.3 vs 47.4; 27-pt fp32 75.5 vs 75.7
    // (profiles/r02_ab.md); 6 CTAs / SM or no metadata prefetch lost 4-11 %
    case K2::kGrp6:
      run_grp(rgcsr_spmv_grp<T, kScaled, 6, 5, true, true, true>,
              rgcsr_spmv_grp<T, kScaled, 6, 5, true, true, true, true>);
      break;
    case K2::kGrp7Mpf:
      run_grp(rgcsr_spmv_grp<T, kScaled, 7, 5, true, true, true>,
              rgcsr_spmv_grp<T, kScaled, 7, 5, true, true, true, true>);
      break;
    case K2::kGrp8:
      run_grp(rgcsr_spmv_grp<T, kScaled, 8, 5, true, true>,
              rgcsr_spmv_grp<T, kScaled, 8, 5, true, true, false, true>);
      break;
    case K2::kGrp8R64:
      run_grp(rgcsr_spmv_grp<T, kScaled, 8, 4, true, true>,
              rgcsr_spmv_grp<T, kScaled, 8, 4, true, true, false, true>);
      break;
    case K2::kLite:
      run_fl(rgcsr_spmv_lite<T, kScaled, 4, 8>, rgcsr_spmv_lite_fl<T, kScaled, 4, 8, false>);
      break;
    case K2::kLite8:
      run_fl(rgcsr_spmv_lite<T, kScaled, 8, 5>, rgcsr_spmv_lite_fl<T, kScaled, 8, 5, false>);
      break;
    case K2::kLite8Full: run(rgcsr_spmv_lite<T, kScaled, 8, 8>); break;
    case K2::kLiteH:
      run_fl(rgcsr_spmv_lite<T, kScaled, 4, 8, true>, rgcsr_spmv_lite_fl<T, kScaled, 4, 8, true>);
      break;
    case K2::kLite8H:
      run_fl(rgcsr_spmv_lite<T, kScaled, 8, 5, true>, rgcsr_spmv_lite_fl<T, kScaled, 8, 5, true>);
      break;
    case K2::kVec2: run_vec(rgcsr_spmv_vec<T, kScaled, 2, 6>); break;
    case K2::kGrpV4: run_grpv(rgcsr_spmv_grpv<T, kScaled, 4, 4>); break;
    default:
      run_fl(rgcsr_spmv_pipe<T, kScaled, U, 4>, rgcsr_spmv_pipe_fl<T, kScaled, U, 4>, true);
      break;
  }
}

// y = A x plus dot_out = sum_r x[x_offset + r] * y[r] (CG's p.q), fused into
// the grp walk's epilogue when the matrix takes that kernel (no long rows,
// <= 10 % padding); otherwise the plain SpMV then a separate dot.
void spmv_dot_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y, uint64_t ny,
                  uint64_t x_offset, double* dot_out, cudaStream_t s) {
  check_spmv_args<double>(h, nx, ny);
  if (!dot_out) fail(SPMVK_EINVAL, "spmv_dot: null dot output");
  if (x_offset + h->rows > nx) fail(SPMVK_EINVAL, "spmv_dot: x_offset + rows exceeds x");
  if (h->rows == 0) {
    SPMVK_CUDA(cudaMemsetAsync(dot_out, 0, sizeof(double), s));
    return;
  }
  if (h->n_long || h->slots == 0 || h->slots * 10 > h->nnz * 11) {
    launch_spmv<double, false>(h, x, y, nullptr, 0.0, s);
    if (spmvk_dot_f64(x + x_offset, y, h->rows, dot_out, s) != SPMVK_OK)
      fail(SPMVK_ECUDA, std::string("spmv_dot: ") + spmvk_last_error());
    return;
  }
  const uint32_t G = static_cast<uint32_t>(std::min<uint64_t>(h->group_size, 0xffffffffull));
  const int sh = pow2_shift(h->group_size);
  auto kern = 2 * h->slots <= 11 * h->rows ? rgcsr_spmv_dot_grp<double, 6, 5>
                                           : rgcsr_spmv_dot_grp<double, 8, 4>;
  int per_sm = 0;
  SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  const unsigned grid = persistent_grid((h->rows + 255) / 256, per_sm > 0 ? per_sm : 1);
  double* part = stream_scratch(s, std::max<uint64_t>(grid, sm_count() * 8ull));
  kern<<<grid, 256, 0, s>>>(static_cast<uint32_t>(h->rows), G, sh, h->group_pointers.p,
                            h->row_lengths.p, reinterpret_cast<const double*>(h->values.p),
                            h->columns.p, x, y, x + x_offset, part);
  SPMVK_LAUNCH("rgcsr_spmv_dot_grp");
  rgcsr_dot_finish<<<1, 256, 0, s>>>(part, static_cast<int>(grid), dot_out);
  SPMVK_LAUNCH("rgcsr_dot_finish");
}

bool pinned(const void* p, void** mapped = nullptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (mapped) *mapped = a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
  return a.type == cudaMemoryTypeHost;
}

// Pipelined host-span SpMV.  x goes up in pieces on one copy stream; each
// row chunk runs as soon as the x prefix it reads (from per-256-row-tile
// column ranges, computed once per matrix) has landed, and stores its y slice
// straight into the mapped pinned host buffer, so the x upload, the SpMV and
// the y download overlap.  y is bitwise the one-launch result (same kernel,
// same per-row order).  Needs pinned host x/y.  The stream operations are
// captured ONCE into a CUDA graph per (matrix, x, y, staging buffers) and
// replayed with one cudaGraphLaunch: issued one by one they cost ~4 us of host
// time each and left the copy engine idle.  Chunk sizes ramp 1:2:4..4:2:1 so
// the pipeline fill (first x piece) and drain (last y slice over PCIe) are
// short while the middle pieces are large enough (~4 MB of x) to keep
// per-copy overhead and copy/store interference low (profiles/r01_e2e_pipeline.md).
constexpr int kPipeChunks = 64;  // upper bound on the chunk count

// Row-chunk boundaries in 256-row tiles.  SPMVK_PIPE_CHUNKS=n forces n equal
// chunks (scripts/e2e_sweep.py).
std::vector<uint32_t> pipe_plan(uint32_t tiles, uint64_t x_bytes) {
  static const int forced = [] {
    const char* e = std::getenv("SPMVK_PIPE_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  std::vector<uint32_t> w;
  if (forced > 0) {
    w.assign(std::min(forced, kPipeChunks), 1);
  } else {
    const int mid = static_cast<int>(std::clamp<uint64_t>(x_bytes >> 22, 1, 12));
    w = {1, 2};
    w.insert(w.end(), mid, 4);
    w.push_back(2);
    w.push_back(1);
  }
  uint64_t total = 0;
  for (auto v : w) total += v;
  std::vector<uint32_t> b{0};
  uint64_t acc = 0;
  for (auto v : w) {
    acc += v;
    const auto e = static_cast<uint32_t>(acc * tiles / total);
    if (e > b.back()) b.push_back(e);
  }
  b.back() = tiles;
  return b;
}

struct PipeStage {
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};  // H2D, compute, D2H
  cudaEvent_t ex[kPipeChunks], ey[kPipeChunks], fork, join[2];
  cudaGraphExec_t exec = nullptr;
  uint64_t key[7] = {};  // matrix serial, x, y, dx, dy, mapped y, sizeof(T)
  bool ready = false;
  void ensure() {
    if (ready) return;
    for (auto& st : s) SPMVK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (int i = 0; i < kPipeChunks; ++i) {
      SPMVK_CUDA(cudaEventCreateWithFlags(&ex[i], cudaEventDisableTiming));
      SPMVK_CUDA(cudaEventCreateWithFlags(&ey[i], cudaEventDisableTiming));
    }
    SPMVK_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (auto& e : join) SPMVK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ready = true;
  }
  ~PipeStage() {
    if (!ready) return;
    if (exec) cudaGraphExecDestroy(exec);
    for (int i = 0; i < kPipeChunks; ++i) {
      cudaEventDestroy(ex[i]);
      cudaEventDestroy(ey[i]);
    }
    cudaEventDestroy(fork);
    for (auto e : join) cudaEventDestroy(e);
    for (auto st : s) cudaStreamDestroy(st);
  }
};

PipeStage& pipe_stage() {
  static thread_local PipeStage p;
  return p;
}

// Enqueue the pipeline on ps.s[0..2] (s[0] is the capture origin).  x chunk
// c ends where row chunk c's largest column does (prefix max), so row chunk c
// waits for exactly x chunks 0..c.  y: when the pinned buffer is mapped into
// the device address space (UVA: cudaHostAlloc / torch pin_memory), the SpMV
// chunks store straight into it over PCIe -- no D2H copies, and the copy
// engine only carries x (two directions of 1 MB copies on two engines
// interfere, profiles/r01_e2e_pipeline.md); otherwise y slices go down on s[2].
template <class T>
void enqueue_pipeline(const spmvk_rgcsr* h, const T* x, T* y, T* y_mapped, T* dx, T* dy,
                      PipeStage& ps, const std::vector<uint32_t>& plan) {
  const uint64_t rows = h->rows, cols = h->cols;
  const auto nchunks = static_cast<uint32_t>(plan.size() - 1);
  SPMVK_CUDA(cudaEventRecord(ps.fork, ps.s[0]));
  SPMVK_CUDA(cudaStreamWaitEvent(ps.s[1], ps.fork, 0));
  SPMVK_CUDA(cudaStreamWaitEvent(ps.s[2], ps.fork, 0));
  uint64_t xb = 0;
  for (uint32_t k = 0; k < nchunks; ++k) {
    uint64_t e = xb;  // one past the largest column of row chunk k (prefix max)
    for (uint32_t t = plan[k]; t < plan[k + 1]; ++t)
      if (h->tile_cols[2 * t] <= h->tile_cols[2 * t + 1])
        e = std::max<uint64_t>(e, uint64_t(h->tile_cols[2 * t + 1]) + 1);
    if (k + 1 == nchunks) e = cols;
    if (xb < e)
      SPMVK_CUDA(cudaMemcpyAsync(dx + xb, x + xb, (e - xb) * sizeof(T), cudaMemcpyHostToDevice,
                                 ps.s[0]));
    SPMVK_CUDA(cudaEventRecord(ps.ex[k], ps.s[0]));
    xb = e;
  }
  const uint32_t G = static_cast<uint32_t>(std::min<uint64_t>(h->group_size, 0xffffffffull));
  const int sh = pow2_shift(h->group_size);
  constexpr bool f64 = sizeof(T) == 8;
  auto kern = f64 ? rgcsr_spmv_lite_range<T, 8, 5> : rgcsr_spmv_lite_range<T, 4, 8>;
  int per_sm = 0;
  SPMVK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
  T* yk = y_mapped ? y_mapped : dy;
  for (uint32_t k = 0; k < nchunks; ++k) {
    SPMVK_CUDA(cudaStreamWaitEvent(ps.s[1], ps.ex[k], 0));
    const uint32_t t0 = plan[k], t1 = plan[k + 1];
    kern<<<persistent_grid(t1 - t0, per_sm > 0 ? per_sm : 1), 256, 0, ps.s[1]>>>(
        t0, t1, static_cast<uint32_t>(rows), G, sh, h->group_pointers.p, h->row_lengths.p,
        reinterpret_cast<const T*>(h->values.p), h->columns.p, dx, yk);
    SPMVK_LAUNCH("rgcsr_spmv_lite_range");
    if (y_mapped) continue;
    SPMVK_CUDA(cudaEventRecord(ps.ey[k], ps.s[1]));
    SPMVK_CUDA(cudaStreamWaitEvent(ps.s[2], ps.ey[k], 0));
    const uint64_t r0 = uint64_t(t0) * 256, r1 = std::min<uint64_t>(rows, uint64_t(t1) * 256);
    SPMVK_CUDA(cudaMemcpyAsync(y + r0, dy + r0, (r1 - r0) * sizeof(T), cudaMemcpyDeviceToHost,
                               ps.s[2]));
  }
  SPMVK_CUDA(cudaEventRecord(ps.join[0], ps.s[1]));
  SPMVK_CUDA(cudaEventRecord(ps.join[1], ps.s[2]));
  SPMVK_CUDA(cudaStreamWaitEvent(ps.s[0], ps.join[0], 0));
  SPMVK_CUDA(cudaStreamWaitEvent(ps.s[0], ps.join[1], 0));
}

template <class T>
bool spmv_host_pipelined(const spmvk_rgcsr* h, const T* x, T* y, HostStage& st) {
  const uint64_t rows = h->rows, cols = h->cols;
  void* ym = nullptr;
  if (h->n_long || rows < (1u << 16) || cols < (1u << 16) || !pinned(x) || !pinned(y, &ym))
    return false;
  static const bool use_mapped = [] {
    const char* e = std::getenv("SPMVK_PIPE_MAPPED_Y");
    return !e || std::atoi(e) != 0;
  }();
  T* y_mapped = use_mapped ? static_cast<T*>(ym) : nullptr;
  const uint32_t tiles = static_cast<uint32_t>((rows + 255) / 256);
  {
    std::lock_guard<std::mutex> lk(h->part_mu);
    if (h->tile_cols.empty()) {
      DevBuf<unsigned> d(2 * uint64_t(tiles));
      std::vector<unsigned> init(2 * uint64_t(tiles));
      for (uint32_t k = 0; k < tiles; ++k) init[2 * k] = 0xffffffffu, init[2 * k + 1] = 0;
      SPMVK_CUDA(cudaMemcpy(d.p, init.data(), 8ull * tiles, cudaMemcpyHostToDevice));
      chunk_column_ranges<<<persistent_grid(tiles, 8), 256>>>(
          static_cast<uint32_t>(rows), static_cast<uint32_t>(h->group_size), 256,
          h->group_pointers.p, h->row_lengths.p, h->columns.p, d.p);
      SPMVK_LAUNCH("chunk_column_ranges");
      h->tile_cols.resize(2 * uint64_t(tiles));
      SPMVK_CUDA(cudaMemcpy(h->tile_cols.data(), d.p, 8ull * tiles, cudaMemcpyDeviceToHost));
    }
  }
  const std::vector<uint32_t> plan = pipe_plan(tiles, cols * sizeof(T));
  PipeStage& ps = pipe_stage();
  ps.ensure();
  T* dx = reinterpret_cast<T*>(st.x.p);
  T* dy = reinterpret_cast<T*>(st.y.p);
  const uint64_t key[7] = {h->serial, reinterpret_cast<uint64_t>(x),
                           reinterpret_cast<uint64_t>(y), reinterpret_cast<uint64_t>(dx),
                           reinterpret_cast<uint64_t>(dy), reinterpret_cast<uint64_t>(y_mapped),
                           sizeof(T)};
  if (!ps.exec || !std::equal(key, key + 7, ps.key)) {
    if (ps.exec) {
      SPMVK_CUDA(cudaGraphExecDestroy(ps.exec));
      ps.exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    SPMVK_CUDA(cudaStreamBeginCapture(ps.s[0], cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_pipeline<T>(h, x, y, y_mapped, dx, dy, ps, plan);
    } catch (...) {
      cudaStreamEndCapture(ps.s[0], &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    SPMVK_CUDA(cudaStreamEndCapture(ps.s[0], &g));
    const cudaError_t e = cudaGraphInstantiate(&ps.exec, g, 0);
    cudaGraphDestroy(g);
    SPMVK_CUDA(e);
    std::copy(key, key + 7, ps.key);
  }
  SPMVK_CUDA(cudaGraphLaunch(ps.exec, ps.s[0]));
  SPMVK_CUDA(cudaStreamSynchronize(ps.s[0]));
  return true;
}

template <class T>
void spmv_host(const spmvk_rgcsr* h, const T* x, uint64_t nx, T* y, uint64_t ny,
               uint64_t* madds) {
  check_spmv_args<T>(h, nx, ny);
  HostStage& st = host_stage();
  st.reserve(nx * sizeof(T), ny * sizeof(T));
  if (spmv_host_pipelined<T>(h, x, y, st)) {
    if (madds) *madds = h->nnz;
    return;
  }
  if (nx) SPMVK_CUDA(cudaMemcpyAsync(st.x.p, x, nx * sizeof(T), cudaMemcpyHostToDevice, st.stream));
  launch_spmv<T, false>(h, reinterpret_cast<const T*>(st.x.p), reinterpret_cast<T*>(st.y.p),
                        nullptr, T(0), st.stream);
  if (ny) SPMVK_CUDA(cudaMemcpyAsync(y, st.y.p, ny * sizeof(T), cudaMemcpyDeviceToHost, st.stream));
  SPMVK_CUDA(cudaStreamSynchronize(st.stream));
  if (madds) *madds = h->nnz;
}

}  // namespace
}  // namespace spmvk

using namespace spmvk;

extern "C" {

int spmvk_rgcsr_build(const spmvk_csr* a, uint64_t group_size, int prec, void* stream,
                      spmvk_rgcsr** out) {
  return guarded([&] {
    require_device();
    if (!out) fail(SPMVK_EINVAL, "null argument");
    *out = build(a, 0, a ? a->rows : 0, group_size, prec, as_stream(stream));
  });
}

int spmvk_rgcsr_build_rows(const spmvk_csr* a, uint64_t row_begin, uint64_t row_end,
                           uint64_t group_size, int prec, void* stream, spmvk_rgcsr** out) {
  return guarded([&] {
    require_device();
    if (!out) fail(SPMVK_EINVAL, "null argument");
    *out = build(a, row_begin, row_end, group_size, prec, as_stream(stream));
  });
}

int spmvk_rgcsr_get_info(const spmvk_rgcsr* h, spmvk_rgcsr_info* info) {
  return guarded([&] {
    if (!h || !info) fail(SPMVK_EINVAL, "null argument");
    info->num_rows = h->rows;
    info->num_cols = h->cols;
    info->group_size = h->group_size;
    info->num_groups = h->groups;
    info->slots = h->slots;
    info->nnz = h->nnz;
    info->artificial_zeros = h->slots - h->nnz;
    // fill.hpp:90-95: index words = slots + group_pointers + row_lengths
    const uint64_t words = h->slots + (h->groups + 1) + h->rows;
    info->bytes_single = h->slots * 4 + words * 4;
    info->bytes_double = h->slots * 8 + words * 4;
    info->precision = h->prec;
  });
}

int spmvk_rgcsr_to_csr(const spmvk_rgcsr* h, void* stream, spmvk_csr** out) {
  return guarded([&] {
    if (!h || !out) fail(SPMVK_EINVAL, "null argument");
    cudaStream_t s = as_stream(stream);
    std::unique_ptr<spmvk_csr> c(new_csr(h->rows, h->cols, h->nnz, SPMVK_F64));
    if (h->rows) {
      DevBuf<uint64_t> off(h->rows);
      const unsigned grid = persistent_grid((h->rows + 255) / 256, 8);
      lens_u64<<<grid, 256, 0, s>>>(h->rows, h->row_lengths.p, off.p);
      SPMVK_LAUNCH("lens_u64");
      exclusive_scan_u64(off.p, h->rows, s);
      if (h->prec == SPMVK_F64)
        rgcsr_gather_rows<double><<<grid, 256, 0, s>>>(
            h->rows, h->group_size, h->nnz, h->group_pointers.p, h->row_lengths.p,
            reinterpret_cast<const double*>(h->values.p), h->columns.p, off.p, c->row_ptr.p,
            c->col.p, reinterpret_cast<double*>(c->val.p));
      else
        rgcsr_gather_rows<float><<<grid, 256, 0, s>>>(
            h->rows, h->group_size, h->nnz, h->group_pointers.p, h->row_lengths.p,
            reinterpret_cast<const float*>(h->values.p), h->columns.p, off.p, c->row_ptr.p,
            c->col.p, reinterpret_cast<double*>(c->val.p));
      SPMVK_LAUNCH("rgcsr_gather_rows");
    } else {
      SPMVK_CUDA(cudaMemsetAsync(c->row_ptr.p, 0, 4, s));
    }
    SPMVK_CUDA(cudaStreamSynchronize(s));
    *out = c.release();
  });
}

int spmvk_rgcsr_download(const spmvk_rgcsr* h, void* values, uint32_t* columns,
                         uint32_t* group_pointers, uint32_t* row_lengths) {
  return guarded([&] {
    if (!h) fail(SPMVK_EINVAL, "null RgCSR handle");
    if (values && h->slots)
      SPMVK_CUDA(cudaMemcpy(values, h->values.p, h->values.bytes(), cudaMemcpyDeviceToHost));
    if (columns && h->slots)
      SPMVK_CUDA(cudaMemcpy(columns, h->columns.p, h->columns.bytes(), cudaMemcpyDeviceToHost));
    if (group_pointers)
      SPMVK_CUDA(cudaMemcpy(group_pointers, h->group_pointers.p, 4 * (h->groups + 1),
                            cudaMemcpyDeviceToHost));
    if (row_lengths && h->rows)
      SPMVK_CUDA(cudaMemcpy(row_lengths, h->row_lengths.p, 4 * h->rows, cudaMemcpyDeviceToHost));
  });
}

int spmvk_rgcsr_spmv_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                         uint64_t ny, void* stream) {
  return guarded([&] {
    check_spmv_args<double>(h, nx, ny);
    launch_spmv<double, false>(h, x, y, nullptr, 0.0, as_stream(stream));
  });
}

int spmvk_rgcsr_spmv_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                         uint64_t ny, void* stream) {
  return guarded([&] {
    check_spmv_args<float>(h, nx, ny);
    launch_spmv<float, false>(h, x, y, nullptr, 0.0f, as_stream(stream));
  });
}

int spmvk_rgcsr_spmv_scaled_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                                uint64_t ny, double* x_next, double scale, void* stream) {
  return guarded([&] {
    check_spmv_args<double>(h, nx, ny);
    if (x_next)
      launch_spmv<double, true>(h, x, y, x_next, scale, as_stream(stream));
    else
      launch_spmv<double, false>(h, x, y, nullptr, 0.0, as_stream(stream));
  });
}

int spmvk_rgcsr_spmv_scaled_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                                uint64_t ny, float* x_next, float scale, void* stream) {
  return guarded([&] {
    check_spmv_args<float>(h, nx, ny);
    if (x_next)
      launch_spmv<float, true>(h, x, y, x_next, scale, as_stream(stream));
    else
      launch_spmv<float, false>(h, x, y, nullptr, 0.0f, as_stream(stream));
  });
}

int spmvk_rgcsr_spmv_host_f64(const spmvk_rgcsr* h, const double* x, uint64_t nx, double* y,
                              uint64_t ny, uint64_t* multiply_add_count) {
  return guarded([&] { spmv_host<double>(h, x, nx, y, ny, multiply_add_count); });
}

int spmvk_rgcsr_spmv_host_f32(const spmvk_rgcsr* h, const float* x, uint64_t nx, float* y,
                              uint64_t ny, uint64_t* multiply_add_count) {
  return guarded([&] { spmv_host<float>(h, x, nx, y, ny, multiply_add_count); });
}

void spmvk_rgcsr_destroy(spmvk_rgcsr* h) { delete h; }

int spmvk_set_long_fused(int on) {
  return guarded([&] { long_fused_slot().store(on ? 1 : 0); });
}

int spmvk_set_long_row_cut(uint32_t cut) {
  return guarded([&] {
    if (cut == 0) fail(SPMVK_EINVAL, "long-row cut must be positive");
    long_cut_slot().store(cut);
  });
}

int spmvk_rgcsr_spmv_dot_f64(const spmvk_rgcsr* a, const double* x, uint64_t nx, double* y,
                             uint64_t ny, uint64_t x_offset, double* dot_out, void* stream) {
  return guarded([&] {
    require_device();
    spmv_dot_f64(a, x, nx, y, ny, x_offset, dot_out, as_stream(stream));
  });
}

int spmvk_set_rgcsr_kernel(const char* name) {
  return guarded([&] {
    K2 k;
    if (!name || !parse_k2(name, &k))
      fail(SPMVK_EINVAL, std::string("unknown RgCSR kernel variant '") + (name ? name : "") +
                             "' (auto | grp6 | grp7_mpf | grp8 | grp8_r64 | lite | lite8 | "
                             "lite8_full | liteh | lite8h | vec2 | pipe)");
    k2_slot().store(static_cast<int>(k));
  });
}

}  // extern "C"
