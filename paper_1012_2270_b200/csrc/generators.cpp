// Seeded host generators for the synthetic workloads (SURVEY.md §8d and
// Appendix B).  All draws use std::mt19937_64 and the reference's unit_real
// convention (top 53 bits * 2^-53, src/synthetic.cpp:7-9), so a seed yields
// the same matrix on every platform.  Output is canonical CSR (columns
// strictly increasing per row), i.e. a valid reference TripletMatrix.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/spmvk.h"

namespace {

double unit_real(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Emits a row's sorted column list (and one value per column from `draw`).
template <class Draw>
void emit(const std::vector<uint64_t>& cols, uint64_t& k, uint32_t* col, double* val,
          Draw&& draw) {
  for (uint64_t c : cols) {
    const double v = draw();
    if (col) {
      col[k] = static_cast<uint32_t>(c);
      val[k] = v;
    }
    ++k;
  }
}

}  // namespace

extern "C" {

void spmvk_gen_random_vector(uint64_t n, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = 2.0 * unit_real(rng) - 1.0;
}

// Lexicographic r = (z*n + y)*n + x; neighbours visited with dz, dy, dx
// ascending, which is ascending column order; off-diagonals -1, diagonal the
// full-stencil neighbour count (4 / 6 / 26).
uint64_t spmvk_gen_stencil(int kind, uint64_t n, uint32_t* row_ptr, uint32_t* col, double* val) {
  if (kind != 5 && kind != 7 && kind != 27) return 0;
  const uint64_t nz = kind == 5 ? 1 : n;
  const double diag = kind == 5 ? 4.0 : kind == 7 ? 6.0 : 26.0;
  uint64_t k = 0, r = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t z = 0; z < nz; ++z)
    for (uint64_t y = 0; y < n; ++y)
      for (uint64_t x = 0; x < n; ++x, ++r) {
        for (int dz = -1; dz <= 1; ++dz) {
          if (kind == 5 && dz) continue;
          const int64_t zz = static_cast<int64_t>(z) + dz;
          if (zz < 0 || zz >= static_cast<int64_t>(nz)) continue;
          for (int dy = -1; dy <= 1; ++dy) {
            const int64_t yy = static_cast<int64_t>(y) + dy;
            if (yy < 0 || yy >= static_cast<int64_t>(n)) continue;
            for (int dx = -1; dx <= 1; ++dx) {
              const int off = (dz != 0) + (dy != 0) + (dx != 0);
              if (kind != 27 && off > 1) continue;
              const int64_t xx = static_cast<int64_t>(x) + dx;
              if (xx < 0 || xx >= static_cast<int64_t>(n)) continue;
              if (col) {
                col[k] = static_cast<uint32_t>((static_cast<uint64_t>(zz) * n +
                                                static_cast<uint64_t>(yy)) * n +
                                               static_cast<uint64_t>(xx));
                val[k] = off == 0 ? diag : -1.0;
              }
              ++k;
            }
          }
        }
        if (row_ptr) row_ptr[r + 1] = static_cast<uint32_t>(k);
      }
  return k;
}

// one mt19937_64(seed) stream; per row
// U = unit_real (1e-300 if 0), len = clamp(floor(9 / U^(1/2.2)), 1, 4096);
// len draws rng() % rows, sorted and deduplicated; then one value
// 2*unit_real - 1 per distinct column in ascending order.
uint64_t spmvk_gen_powerlaw(uint64_t rows, uint64_t seed, uint32_t* row_ptr, uint32_t* col,
                            double* val) {
  std::mt19937_64 rng(seed);
  std::vector<uint64_t> cols;
  cols.reserve(4096);
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t r = 0; r < rows; ++r) {
    double u = unit_real(rng);
    if (u == 0.0) u = 1e-300;
    const double lf = std::floor(9.0 / std::pow(u, 1.0 / 2.2));
    const uint64_t len = lf > 4096.0 ? 4096 : lf < 1.0 ? 1 : static_cast<uint64_t>(lf);
    cols.resize(len);
    for (auto& c : cols) c = rng() % rows;
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    emit(cols, k, col, val, [&] { return 2.0 * unit_real(rng) - 1.0; });
    if (row_ptr) row_ptr[r + 1] = static_cast<uint32_t>(k);
  }
  return k;
}

// Sweep class "random": row length uniform in [1, 2*mean-1] (mean `mean_len`),
// distinct uniform columns, values U[-1,1).
uint64_t spmvk_gen_random_rows(uint64_t rows, uint64_t cols_n, uint64_t mean_len, uint64_t seed,
                               uint32_t* row_ptr, uint32_t* col, double* val) {
  std::mt19937_64 rng(seed);
  std::vector<uint64_t> cols;
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  const uint64_t span = mean_len ? 2 * mean_len - 1 : 1;
  for (uint64_t r = 0; r < rows; ++r) {
    const uint64_t len = std::min<uint64_t>(1 + rng() % span, cols_n);
    cols.resize(len);
    for (auto& c : cols) c = rng() % cols_n;
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    emit(cols, k, col, val, [&] { return 2.0 * unit_real(rng) - 1.0; });
    if (row_ptr) row_ptr[r + 1] = static_cast<uint32_t>(k);
  }
  return k;
}

// Sweep class "block": block rows of b rows; each block row holds `nblk`
// dense b x b blocks on distinct random block columns (one always diagonal).
uint64_t spmvk_gen_block(uint64_t rows, uint64_t b, uint64_t nblk, uint64_t seed,
                         uint32_t* row_ptr, uint32_t* col, double* val) {
  std::mt19937_64 rng(seed);
  const uint64_t nb = (rows + b - 1) / b;
  std::vector<uint64_t> bc, cols;
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t br = 0; br < nb; ++br) {
    bc.assign(1, br);
    for (uint64_t i = 1; i < nblk; ++i) bc.push_back(rng() % nb);
    std::sort(bc.begin(), bc.end());
    bc.erase(std::unique(bc.begin(), bc.end()), bc.end());
    cols.clear();
    for (uint64_t c : bc)
      for (uint64_t d = 0; d < b && c * b + d < rows; ++d) cols.push_back(c * b + d);
    for (uint64_t t = 0; t < b && br * b + t < rows; ++t) {
      emit(cols, k, col, val, [&] { return 2.0 * unit_real(rng) - 1.0; });
      if (row_ptr) row_ptr[br * b + t + 1] = static_cast<uint32_t>(k);
    }
  }
  return k;
}

// banded_matrix (src/synthetic.cpp:48-60): dense band of half width hbw,
// values 2*unit_real-1 in row-major order.
uint64_t spmvk_gen_banded(uint64_t n, uint64_t hbw, uint64_t seed, uint32_t* row_ptr,
                          uint32_t* col, double* val) {
  std::mt19937_64 rng(seed);
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t lo = r >= hbw ? r - hbw : 0;
    const uint64_t hi = std::min(n - 1, r + hbw);
    for (uint64_t c = lo; c <= hi; ++c) {
      const double v = 2.0 * unit_real(rng) - 1.0;
      if (col) {
        col[k] = static_cast<uint32_t>(c);
        val[k] = v;
      }
      ++k;
    }
    if (row_ptr) row_ptr[r + 1] = static_cast<uint32_t>(k);
  }
  return k;
}

}  // extern "C"
