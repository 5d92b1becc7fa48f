/* oracle/oracle.c — TEST INFRASTRUCTURE ONLY (the checker; see oracle.h).
 *
 * Plain-C restatement of the reference's hot path.  Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj/).
 * Built with -ffp-contract=off: every product and every sum is rounded
 * separately, exactly as the reference's x86-64 build (no -march, SSE2 scalar
 * arithmetic, core/CMakeLists.txt:21-23) rounds them.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ mt19937_64
 * The standard 64-bit Mersenne Twister (std::mt19937_64: w=64 n=312 m=156
 * r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555 s=17
 * b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005),
 * the generator behind every reference draw (src/synthetic.cpp). */
#define MT_N 312
#define MT_M 156
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + MT_M] ^ (x >> 1) ^ mag01[x & 1ULL];
    }
    for (; i < MT_N - 1; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag01[x & 1ULL];
    }
    x = (s->mt[MT_N - 1] & UM) | (s->mt[0] & LM);
    s->mt[MT_N - 1] = s->mt[MT_M - 1] ^ (x >> 1) ^ mag01[x & 1ULL];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* src/synthetic.cpp:7-9: top 53 bits scaled by 2^-53. */
double orc_unit_real(orc_mt64* s) { return (double)(orc_mt64_next(s) >> 11) * 0x1.0p-53; }

/* src/synthetic.cpp:62-67 */
void orc_random_vector(uint64_t n, uint64_t seed, double* out) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = 2.0 * orc_unit_real(&s) - 1.0;
}

/* src/synthetic.cpp:13-24 draw_value */
static double draw_value(orc_mt64* s, int vmin, int vmax, int integer_values, int allow_zero) {
  for (;;) {
    double v;
    if (integer_values) {
      const uint64_t span = (uint64_t)(vmax - vmin) + 1;
      v = (double)(vmin + (int)(orc_mt64_next(s) % span));
    } else {
      v = vmin + orc_unit_real(s) * (vmax - vmin);
    }
    if (allow_zero || v != 0.0) return v;
  }
}

/* src/synthetic.cpp:28-46: per-cell Bernoulli sweep in row-major order. */
uint64_t orc_random_matrix(uint64_t rows, uint64_t cols, double density, int vmin, int vmax,
                           int integer_values, int allow_zero, uint64_t seed, uint32_t* row_ptr,
                           uint32_t* col, double* val) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t r = 0; r < rows; ++r) {
    for (uint64_t c = 0; c < cols; ++c) {
      if (orc_unit_real(&s) < density) {
        const double v = draw_value(&s, vmin, vmax, integer_values, allow_zero);
        if (col) {
          col[k] = (uint32_t)c;
          val[k] = v;
        }
        ++k;
      }
    }
    if (row_ptr) row_ptr[r + 1] = (uint32_t)k;
  }
  return k;
}

/* tests/fixtures.hpp:50-60 random_small: rows, cols, density, then the seed of
 * random_matrix, all drawn from one mt19937_64(seed). */
void orc_random_small_spec(uint64_t seed, uint64_t* rows, uint64_t* cols, double* density,
                           uint64_t* matrix_seed) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  *rows = 1 + orc_mt64_next(&s) % 64;
  *cols = 1 + orc_mt64_next(&s) % 64;
  *density = 0.05 + 0.25 * orc_unit_real(&s);
  *matrix_seed = orc_mt64_next(&s);
}

/* src/synthetic.cpp:48-60 */
uint64_t orc_banded(uint64_t n, uint64_t hbw, uint64_t seed, uint32_t* row_ptr, uint32_t* col,
                    double* val) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  uint64_t k = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t r = 0; r < n; ++r) {
    const uint64_t lo = r >= hbw ? r - hbw : 0;
    const uint64_t hi = (r + hbw < n - 1) ? r + hbw : n - 1;
    for (uint64_t c = lo; c <= hi; ++c) {
      const double v = 2.0 * orc_unit_real(&s) - 1.0;
      if (col) {
        col[k] = (uint32_t)c;
        val[k] = v;
      }
      ++k;
    }
    if (row_ptr) row_ptr[r + 1] = (uint32_t)k;
  }
  return k;
}

/* src/triplet.cpp:71-79: y = 0; y[row] += value * x[col] in sorted order. */
void orc_spmv_reference(uint64_t rows, const uint32_t* rp, const uint32_t* col,
                        const double* val, const double* x, double* y) {
  for (uint64_t r = 0; r < rows; ++r) {
    y[r] = 0.0;
    for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) y[r] += val[k] * x[col[k]];
  }
}

/* spmvkit/csr.hpp:41-53 */
void orc_spmv_csr_f64(uint64_t rows, const uint32_t* rp, const uint32_t* col, const double* val,
                      const double* x, double* y) {
  for (uint64_t i = 0; i < rows; ++i) {
    double acc = 0;
    for (uint32_t j = rp[i]; j < rp[i + 1]; ++j) acc += val[j] * x[col[j]];
    y[i] = acc;
  }
}

void orc_spmv_csr_f32(uint64_t rows, const uint32_t* rp, const uint32_t* col, const float* val,
                      const float* x, float* y) {
  for (uint64_t i = 0; i < rows; ++i) {
    float acc = 0;
    for (uint32_t j = rp[i]; j < rp[i + 1]; ++j) acc += val[j] * x[col[j]];
    y[i] = acc;
  }
}

/* spmvkit/rgcsr.hpp:31-34 rows_in_group */
static uint64_t rows_in_group(uint64_t rows, uint64_t G, uint64_t g) {
  const uint64_t rest = rows - g * G;
  return G < rest ? G : rest;
}

/* spmvkit/rgcsr.hpp:39-57: row lengths, per-group width, group pointers. */
uint64_t orc_rgcsr_layout(uint64_t rows, const uint32_t* rp, uint64_t G, uint32_t* lens,
                          uint32_t* gp, int* overflow) {
  if (G == 0) return UINT64_MAX;
  *overflow = 0;
  for (uint64_t r = 0; r < rows; ++r) lens[r] = rp[r + 1] - rp[r];
  const uint64_t groups = (rows + G - 1) / G;
  uint64_t total = 0;
  gp[0] = 0;
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t s = rows_in_group(rows, G, g);
    uint64_t w = 0;
    for (uint64_t t = 0; t < s; ++t)
      if (lens[g * G + t] > w) w = lens[g * G + t];
    total += s * w;
    gp[g + 1] = (uint32_t)total; /* the reference's static_cast<index_t> */
  }
  if (total > 0xFFFFFFFFULL) *overflow = 1;
  return total;
}

/* spmvkit/rgcsr.hpp:59-68: zero-fill, then entry j of row r goes to
 * gp[g] + (r % G) + j * rows_in_group(g). */
#define RGCSR_FILL(T)                                                                        \
  void orc_rgcsr_fill_##T(uint64_t rows, const uint32_t* rp, const uint32_t* col,            \
                          const double* val, uint64_t G, const uint32_t* gp, TYPE_##T* values, \
                          uint32_t* columns) {                                               \
    const uint64_t groups = (rows + G - 1) / G;                                              \
    memset(values, 0, sizeof(TYPE_##T) * gp[groups]);                                        \
    memset(columns, 0, sizeof(uint32_t) * gp[groups]);                                       \
    for (uint64_t r = 0; r < rows; ++r) {                                                    \
      const uint64_t g = r / G, t = r % G, s = rows_in_group(rows, G, g);                    \
      for (uint32_t j = 0; j < rp[r + 1] - rp[r]; ++j) {                                     \
        const uint64_t idx = gp[g] + t + (uint64_t)j * s;                                    \
        values[idx] = (TYPE_##T)val[rp[r] + j];                                              \
        columns[idx] = col[rp[r] + j];                                                       \
      }                                                                                      \
    }                                                                                        \
  }
#define TYPE_f64 double
#define TYPE_f32 float
RGCSR_FILL(f64)
RGCSR_FILL(f32)

/* spmvkit/rgcsr.hpp:75-97: per group, per row, acc += v * x[c], idx += s. */
#define RGCSR_SPMV(T)                                                                          \
  uint64_t orc_spmv_rgcsr_##T(uint64_t rows, uint64_t G, const uint32_t* gp,                   \
                              const uint32_t* lens, const TYPE_##T* values,                    \
                              const uint32_t* columns, const TYPE_##T* x, TYPE_##T* y) {       \
    uint64_t madds = 0;                                                                        \
    const uint64_t groups = (rows + G - 1) / G;                                                \
    for (uint64_t g = 0; g < groups; ++g) {                                                    \
      const uint64_t s = rows_in_group(rows, G, g), base = gp[g];                              \
      for (uint64_t t = 0; t < s; ++t) {                                                       \
        const uint64_t row = g * G + t;                                                        \
        TYPE_##T acc = 0;                                                                      \
        uint64_t idx = base + t;                                                               \
        for (uint32_t j = 0; j < lens[row]; ++j, idx += s) {                                   \
          acc += values[idx] * x[columns[idx]];                                                \
          ++madds;                                                                             \
        }                                                                                      \
        y[row] = acc;                                                                          \
      }                                                                                        \
    }                                                                                          \
    return madds;                                                                              \
  }
RGCSR_SPMV(f64)
RGCSR_SPMV(f32)

/* spmvkit/ellpack.hpp:145-150 */
uint64_t orc_hybrid_split_cost(const uint64_t* lens, uint64_t n, uint64_t k) {
  uint64_t overflow = 0;
  for (uint64_t i = 0; i < n; ++i) overflow += lens[i] > k ? lens[i] - k : 0;
  return 2 * n * k + 3 * overflow;
}

/* spmvkit/ellpack.hpp:153-166: argmin over k in [0, max_len], strict < (the
 * smallest k wins ties). */
uint64_t orc_choose_ell_width(const uint64_t* lens, uint64_t n) {
  uint64_t max_len = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (lens[i] > max_len) max_len = lens[i];
  uint64_t best_k = 0, best = orc_hybrid_split_cost(lens, n, 0);
  for (uint64_t k = 1; k <= max_len; ++k) {
    const uint64_t c = orc_hybrid_split_cost(lens, n, k);
    if (c < best) {
      best = c;
      best_k = k;
    }
  }
  return best_k;
}

/* spmvkit/ellpack.hpp:171-181: the COO part holds every entry past the
 * first k1 of its row. */
uint64_t orc_hybrid_coo_count(uint64_t rows, const uint32_t* rp, uint64_t k1) {
  uint64_t max_len = 0, coo = 0;
  for (uint64_t r = 0; r < rows; ++r) {
    const uint64_t len = rp[r + 1] - rp[r];
    if (len > max_len) max_len = len;
    if (len > k1) coo += len - k1;
  }
  if (k1 > max_len) return UINT64_MAX;
  return coo;
}

/* spmvkit/ellpack.hpp:183-202: ELL slot-major slot*N+row, pads (0, col 0);
 * overflow appended to COO in (row, col) order. */
#define HYB_FILL(T)                                                                            \
  void orc_hybrid_fill_##T(uint64_t rows, const uint32_t* rp, const uint32_t* col,             \
                           const double* val, uint64_t k1, TYPE_##T* ev, uint32_t* ec,         \
                           uint32_t* cr, uint32_t* cc, TYPE_##T* cv) {                         \
    memset(ev, 0, sizeof(TYPE_##T) * rows * k1);                                               \
    memset(ec, 0, sizeof(uint32_t) * rows * k1);                                               \
    uint64_t n = 0;                                                                            \
    for (uint64_t r = 0; r < rows; ++r) {                                                      \
      for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {                                           \
        const uint64_t pos = k - rp[r];                                                        \
        if (pos < k1) {                                                                        \
          ev[pos * rows + r] = (TYPE_##T)val[k];                                               \
          ec[pos * rows + r] = col[k];                                                         \
        } else {                                                                               \
          cr[n] = (uint32_t)r;                                                                 \
          cc[n] = col[k];                                                                      \
          cv[n] = (TYPE_##T)val[k];                                                            \
          ++n;                                                                                 \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
  }
HYB_FILL(f64)
HYB_FILL(f32)

/* spmvkit/ellpack.hpp:111-123 (ELL: zero y, walk every slot incl. pads) then
 * :134-141 (COO: y[r] += v * x[c] in array order). */
#define HYB_SPMV(T)                                                                            \
  void orc_spmv_hybrid_##T(uint64_t rows, uint64_t k1, const TYPE_##T* ev, const uint32_t* ec, \
                           uint64_t coo_n, const uint32_t* cr, const uint32_t* cc,             \
                           const TYPE_##T* cv, const TYPE_##T* x, TYPE_##T* y) {               \
    for (uint64_t r = 0; r < rows; ++r) y[r] = 0;                                              \
    for (uint64_t slot = 0; slot < k1; ++slot) {                                               \
      const uint64_t base = slot * rows;                                                       \
      for (uint64_t r = 0; r < rows; ++r) y[r] += ev[base + r] * x[ec[base + r]];              \
    }                                                                                          \
    for (uint64_t i = 0; i < coo_n; ++i) y[cr[i]] += cv[i] * x[cc[i]];                         \
  }
HYB_SPMV(f64)
HYB_SPMV(f32)

/* src/reorder.cpp:35-42: stable sort of row ids by decreasing length.  A
 * counting sort over lengths (descending buckets, ids ascending inside a
 * bucket) is the same stable order. */
void orc_descending_map(uint64_t rows, const uint32_t* rp, uint32_t* map) {
  uint64_t max_len = 0;
  for (uint64_t r = 0; r < rows; ++r)
    if (rp[r + 1] - rp[r] > max_len) max_len = rp[r + 1] - rp[r];
  uint64_t* start = calloc(max_len + 2, sizeof(uint64_t));
  for (uint64_t r = 0; r < rows; ++r) start[max_len - (rp[r + 1] - rp[r]) + 1]++;
  for (uint64_t b = 1; b <= max_len + 1; ++b) start[b] += start[b - 1];
  for (uint64_t r = 0; r < rows; ++r) map[start[max_len - (rp[r + 1] - rp[r])]++] = (uint32_t)r;
  free(start);
}

/* SURVEY.md Appendix B stencils: lexicographic r = (z*n + y)*n + x, neighbours
 * in increasing column order, off-diagonals -1, diagonal = full neighbour count. */
uint64_t orc_stencil(int kind, uint64_t n, uint32_t* rp, uint32_t* col, double* val) {
  const int three_d = kind != 5;
  const uint64_t nz = three_d ? n : 1;
  const double diag = kind == 5 ? 4.0 : kind == 7 ? 6.0 : 26.0;
  uint64_t k = 0, r = 0;
  if (rp) rp[0] = 0;
  for (uint64_t z = 0; z < nz; ++z)
    for (uint64_t y = 0; y < n; ++y)
      for (uint64_t x = 0; x < n; ++x, ++r) {
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (!three_d && dz != 0) continue;
              const int nnb = (dz != 0) + (dy != 0) + (dx != 0);
              if (kind != 27 && nnb > 1) continue;
              const int64_t zz = (int64_t)z + dz, yy = (int64_t)y + dy, xx = (int64_t)x + dx;
              if (zz < 0 || yy < 0 || xx < 0 || zz >= (int64_t)nz || yy >= (int64_t)n ||
                  xx >= (int64_t)n)
                continue;
              if (col) {
                col[k] = (uint32_t)(((uint64_t)zz * n + (uint64_t)yy) * n + (uint64_t)xx);
                val[k] = nnb == 0 ? diag : -1.0;
              }
              ++k;
            }
        if (rp) rp[r + 1] = (uint32_t)k;
      }
  return k;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* SURVEY.md Appendix B power-law: one mt19937_64(seed) stream; per row
 * U = unit_real (1e-300 if 0), len = clamp(floor(9 / U^(1/2.2)), 1, 4096),
 * len draws rng() % N sorted + deduped, one value 2*unit_real-1 per column. */
uint64_t orc_powerlaw(uint64_t rows, uint64_t seed, uint32_t* rp, uint32_t* col, double* val) {
  orc_mt64 s;
  orc_mt64_seed(&s, seed);
  uint64_t buf[4096];
  uint64_t k = 0;
  if (rp) rp[0] = 0;
  for (uint64_t r = 0; r < rows; ++r) {
    double u = orc_unit_real(&s);
    if (u == 0.0) u = 1e-300;
    double lf = floor(9.0 / pow(u, 1.0 / 2.2));
    uint64_t len = lf > 4096.0 ? 4096 : lf < 1.0 ? 1 : (uint64_t)lf;
    for (uint64_t i = 0; i < len; ++i) buf[i] = orc_mt64_next(&s) % rows;
    qsort(buf, len, sizeof(uint64_t), cmp_u64);
    uint64_t d = 0;
    for (uint64_t i = 0; i < len; ++i)
      if (d == 0 || buf[i] != buf[d - 1]) buf[d++] = buf[i];
    for (uint64_t i = 0; i < d; ++i) {
      const double v = 2.0 * orc_unit_real(&s) - 1.0;
      if (col) {
        col[k] = (uint32_t)buf[i];
        val[k] = v;
      }
      ++k;
    }
    if (rp) rp[r + 1] = (uint32_t)k;
  }
  return k;
}
