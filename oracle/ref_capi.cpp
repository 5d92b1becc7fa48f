// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A flat C entry-point layer over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled in place by oracle/Makefile into
// oracle/_ref/libspmvkit_ref.so).  It lets pytest (ctypes), the golden-vector
// generator (oracle/make_golden.py) and bench.py's reference arm call the
// reference's own templates:
//   build_csr / spmv_csr              proj/core/include/spmvkit/csr.hpp:24-53
//   build_rgcsr / spmv_rgcsr          proj/core/include/spmvkit/rgcsr.hpp:38-97
//   choose_ell_width / build_hybrid   proj/core/include/spmvkit/ellpack.hpp:143-203
//   spmv_hybrid                       proj/core/include/spmvkit/ellpack.hpp:205-210
//   fill_report                       proj/core/include/spmvkit/fill.hpp:52-95
//   spmv_reference                    proj/core/src/triplet.cpp:71-79
//   random_matrix / banded / vector   proj/core/src/synthetic.cpp:28-67
//   descending_row_permutation        proj/core/src/reorder.cpp:35-61
// Nothing here re-implements reference arithmetic; every number comes out of
// the reference code.  No reference source is copied into this repository.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "spmvkit/spmvkit.hpp"

using namespace spmvkit;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct RefMatrix {
  TripletMatrix m;
};

struct RefRgcsr {
  int prec;  // 8 = double, 4 = float
  RgcsrMatrix<double> d;
  RgcsrMatrix<float> f;
};

struct RefHybrid {
  int prec;
  HybridMatrix<double> d;
  HybridMatrix<float> f;
};

struct RefCsr {
  int prec;
  CsrMatrix<double> d;
  CsrMatrix<float> f;
};

// tests/fixtures.hpp:50-60 (random_small) and tests/acceptance.cpp:87-94
// (random_case) are test helpers in the reference, not library code; they are
// re-expressed here on top of the reference's own RandomMatrixSpec /
// random_matrix / unit_real so that golden inputs are the reference's inputs.
TripletMatrix random_small(std::uint64_t seed, bool allow_zero_values, bool integer_values) {
  std::mt19937_64 rng(seed);
  RandomMatrixSpec spec;
  spec.rows = 1 + rng() % 64;
  spec.cols = 1 + rng() % 64;
  spec.density = 0.05 + 0.25 * unit_real(rng);
  spec.integer_values = integer_values;
  spec.allow_zero_values = allow_zero_values;
  return random_matrix(spec, rng());
}

TripletMatrix random_case(std::uint64_t seed, std::size_t max_rows) {
  std::mt19937_64 rng(seed);
  RandomMatrixSpec spec;
  spec.rows = 1 + rng() % max_rows;
  spec.cols = 1 + rng() % max_rows;
  spec.density = 0.05 + 0.25 * unit_real(rng);
  return random_matrix(spec, rng());
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- matrices
int ref_tm_from_csr(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t* row_ptr,
                    const uint32_t* col, const double* val, void** out) {
  return guard([&] {
    std::vector<Entry> e;
    e.reserve(nnz);
    for (uint64_t r = 0; r < rows; ++r)
      for (uint32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
        e.push_back({static_cast<index_t>(r), col[k], val[k]});
    *out = new RefMatrix{TripletMatrix(rows, cols, std::move(e))};
  });
}

int ref_tm_example8(void** out) {
  return guard([&] {
    *out = new RefMatrix{TripletMatrix(8, 8,
                                       {{0, 0, 1.0},
                                        {0, 3, 2.0},
                                        {1, 1, 3.0},
                                        {2, 2, 4.0},
                                        {3, 0, 5.0},
                                        {4, 4, 6.0},
                                        {5, 0, 7.0},
                                        {5, 5, 8.0},
                                        {6, 1, 9.0},
                                        {6, 4, 10.0},
                                        {6, 6, 11.0},
                                        {7, 2, 12.0},
                                        {7, 7, 13.0}})};
  });
}

int ref_tm_random_small(uint64_t seed, int allow_zero, int integer, void** out) {
  return guard([&] { *out = new RefMatrix{random_small(seed, allow_zero != 0, integer != 0)}; });
}

int ref_tm_random_case(uint64_t seed, uint64_t max_rows, void** out) {
  return guard([&] { *out = new RefMatrix{random_case(seed, max_rows)}; });
}

int ref_tm_random_matrix(uint64_t rows, uint64_t cols, double density, int vmin, int vmax,
                         int integer, int allow_zero, uint64_t seed, void** out) {
  return guard([&] {
    RandomMatrixSpec s;
    s.rows = rows;
    s.cols = cols;
    s.density = density;
    s.value_min = vmin;
    s.value_max = vmax;
    s.integer_values = integer != 0;
    s.allow_zero_values = allow_zero != 0;
    *out = new RefMatrix{random_matrix(s, seed)};
  });
}

int ref_tm_banded(uint64_t n, uint64_t hbw, uint64_t seed, void** out) {
  return guard([&] { *out = new RefMatrix{banded_matrix(n, hbw, seed)}; });
}

int ref_tm_descending(const void* h, void** out) {
  return guard([&] {
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    *out = new RefMatrix{
        apply_permutation(m, descending_row_permutation(m), PermutationMode::RowsOnly)};
  });
}

int ref_descending_map(const void* h, uint32_t* map) {
  return guard([&] {
    const auto p = descending_row_permutation(static_cast<const RefMatrix*>(h)->m);
    std::copy(p.map().begin(), p.map().end(), map);
  });
}

void ref_tm_dims(const void* h, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
  const auto& m = static_cast<const RefMatrix*>(h)->m;
  *rows = m.num_rows();
  *cols = m.num_cols();
  *nnz = m.nnz();
}

void ref_tm_export(const void* h, uint32_t* row_ptr, uint32_t* col, double* val) {
  const auto& m = static_cast<const RefMatrix*>(h)->m;
  std::fill(row_ptr, row_ptr + m.num_rows() + 1, 0u);
  uint64_t k = 0;
  for (const Entry& e : m.entries()) {
    ++row_ptr[e.row + 1];
    col[k] = e.col;
    val[k] = e.value;
    ++k;
  }
  for (uint64_t r = 0; r < m.num_rows(); ++r) row_ptr[r + 1] += row_ptr[r];
}

void ref_tm_free(void* h) { delete static_cast<RefMatrix*>(h); }

// parse_matrix_market (src/matrix_market.cpp:61-138) on an in-memory text;
// returns 3 with *line set on MatrixMarketError.
int ref_mm_parse(const char* text, uint64_t len, void** out, uint64_t* line) {
  *line = 0;
  try {
    std::istringstream in(std::string(text, len));
    *out = new RefMatrix{parse_matrix_market(in)};
    return 0;
  } catch (const MatrixMarketError& e) {
    g_err = e.what();
    *line = e.line();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// write_matrix_market (src/matrix_market.cpp:150-158) into a caller buffer;
// returns the byte count (call with buf NULL to size).
uint64_t ref_mm_write(const void* h, char* buf, uint64_t cap) {
  std::ostringstream out;
  write_matrix_market(out, static_cast<const RefMatrix*>(h)->m);
  const std::string s = out.str();
  if (buf) std::memcpy(buf, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

int ref_spmv_reference(const void* h, const double* x, uint64_t nx, double* y) {
  return guard([&] {
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    const auto r = spmv_reference(m, std::span<const double>(x, nx));
    std::copy(r.begin(), r.end(), y);
  });
}

void ref_random_vector(uint64_t n, uint64_t seed, double* out) {
  const auto v = random_vector(n, seed);
  std::copy(v.begin(), v.end(), out);
}

double ref_measured_gflops(uint64_t nnz, double seconds) { return measured_gflops(nnz, seconds); }

// ---------------------------------------------------------------- CSR
int ref_csr_build(const void* h, int prec, void** out) {
  return guard([&] {
    auto* c = new RefCsr{prec, {}, {}};
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    if (prec == 4) c->f = build_csr<float>(m); else c->d = build_csr<double>(m);
    *out = c;
  });
}

int ref_csr_spmv(const void* h, const void* x, uint64_t nx, void* y, uint64_t ny) {
  return guard([&] {
    const auto* c = static_cast<const RefCsr*>(h);
    if (c->prec == 4)
      spmv_csr(c->f, std::span<const float>(static_cast<const float*>(x), nx),
               std::span<float>(static_cast<float*>(y), ny));
    else
      spmv_csr(c->d, std::span<const double>(static_cast<const double*>(x), nx),
               std::span<double>(static_cast<double*>(y), ny));
  });
}

void ref_csr_free(void* h) { delete static_cast<RefCsr*>(h); }

// ---------------------------------------------------------------- RgCSR
int ref_rgcsr_build(const void* h, uint64_t group_size, int prec, void** out) {
  return guard([&] {
    auto* r = new RefRgcsr{prec, {}, {}};
    std::unique_ptr<RefRgcsr> own(r);
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    if (prec == 4) r->f = build_rgcsr<float>(m, group_size);
    else r->d = build_rgcsr<double>(m, group_size);
    *out = own.release();
  });
}

// info[0]=slots info[1]=num_groups info[2]=artificial_zeros info[3]=bytes_single
// info[4]=bytes_double info[5]=nnz
void ref_rgcsr_info(const void* h, uint64_t* info) {
  const auto* r = static_cast<const RefRgcsr*>(h);
  const FillReport f = r->prec == 4 ? fill_report(r->f) : fill_report(r->d);
  info[0] = f.stored_slots;
  info[1] = r->prec == 4 ? r->f.num_groups() : r->d.num_groups();
  info[2] = f.artificial_zeros;
  info[3] = f.bytes_single;
  info[4] = f.bytes_double;
  info[5] = f.nnz;
}

void ref_rgcsr_export(const void* h, void* values, uint32_t* columns, uint32_t* gp,
                      uint32_t* lens) {
  const auto* r = static_cast<const RefRgcsr*>(h);
  auto dump = [&](const auto& a) {
    std::memcpy(values, a.values.data(), a.values.size() * sizeof(a.values[0]));
    std::copy(a.columns.begin(), a.columns.end(), columns);
    std::copy(a.group_pointers.begin(), a.group_pointers.end(), gp);
    std::copy(a.row_lengths.begin(), a.row_lengths.end(), lens);
  };
  if (r->prec == 4) dump(r->f); else dump(r->d);
}

int ref_rgcsr_spmv(const void* h, const void* x, uint64_t nx, void* y, uint64_t ny,
                   uint64_t* madds) {
  return guard([&] {
    const auto* r = static_cast<const RefRgcsr*>(h);
    if (r->prec == 4)
      spmv_rgcsr(r->f, std::span<const float>(static_cast<const float*>(x), nx),
                 std::span<float>(static_cast<float*>(y), ny), madds);
    else
      spmv_rgcsr(r->d, std::span<const double>(static_cast<const double*>(x), nx),
                 std::span<double>(static_cast<double*>(y), ny), madds);
  });
}

void ref_rgcsr_free(void* h) { delete static_cast<RefRgcsr*>(h); }

// ---------------------------------------------------------------- Hybrid
uint64_t ref_choose_ell_width(const uint64_t* lens, uint64_t n) {
  std::vector<std::size_t> v(lens, lens + n);
  return choose_ell_width(v);
}

uint64_t ref_hybrid_split_cost(const uint64_t* lens, uint64_t n, uint64_t k) {
  std::vector<std::size_t> v(lens, lens + n);
  return hybrid_split_cost(v, k);
}

int ref_hybrid_build(const void* h, int64_t k1, int prec, void** out) {
  return guard([&] {
    auto* r = new RefHybrid{prec, {}, {}};
    std::unique_ptr<RefHybrid> own(r);
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    std::optional<std::size_t> w;
    if (k1 >= 0) w = static_cast<std::size_t>(k1);
    if (prec == 4) r->f = build_hybrid<float>(m, w); else r->d = build_hybrid<double>(m, w);
    *out = own.release();
  });
}

// info[0]=K1 info[1]=ell slots info[2]=coo nnz info[3]=artificial_zeros
// info[4]=bytes_single info[5]=bytes_double
void ref_hybrid_info(const void* h, uint64_t* info) {
  const auto* r = static_cast<const RefHybrid*>(h);
  auto fill = [&](const auto& hy) {
    const FillReport f = fill_report(hy);
    info[0] = hy.ell.slots_per_row;
    info[1] = hy.ell.slot_count();
    info[2] = hy.coo.nnz();
    info[3] = f.artificial_zeros;
    info[4] = f.bytes_single;
    info[5] = f.bytes_double;
  };
  if (r->prec == 4) fill(r->f); else fill(r->d);
}

void ref_hybrid_export(const void* h, void* ell_values, uint32_t* ell_columns, uint32_t* coo_rows,
                       uint32_t* coo_columns, void* coo_values) {
  const auto* r = static_cast<const RefHybrid*>(h);
  auto dump = [&](const auto& hy) {
    std::memcpy(ell_values, hy.ell.values.data(), hy.ell.values.size() * sizeof(hy.ell.values[0]));
    std::copy(hy.ell.columns.begin(), hy.ell.columns.end(), ell_columns);
    std::copy(hy.coo.rows.begin(), hy.coo.rows.end(), coo_rows);
    std::copy(hy.coo.columns.begin(), hy.coo.columns.end(), coo_columns);
    std::memcpy(coo_values, hy.coo.values.data(), hy.coo.values.size() * sizeof(hy.coo.values[0]));
  };
  if (r->prec == 4) dump(r->f); else dump(r->d);
}

int ref_hybrid_spmv(const void* h, const void* x, uint64_t nx, void* y, uint64_t ny) {
  return guard([&] {
    const auto* r = static_cast<const RefHybrid*>(h);
    if (r->prec == 4)
      spmv_hybrid(r->f, std::span<const float>(static_cast<const float*>(x), nx),
                  std::span<float>(static_cast<float*>(y), ny));
    else
      spmv_hybrid(r->d, std::span<const double>(static_cast<const double*>(x), nx),
                  std::span<double>(static_cast<double*>(y), ny));
  });
}

void ref_hybrid_free(void* h) { delete static_cast<RefHybrid*>(h); }

// ---------------------------------------------------------------- bench
// The reference's own harness (proj/core/src/bench.cpp:132): build, checksum
// gate vs spmv_reference, calibrated median.  fmt: 0 csr, 1 rgcsr, 2 hybrid.
// out[0]=median_seconds out[1]=gflops out[2]=checksum out[3]=bytes
int ref_run_spmv_bench(const void* h, int fmt, int64_t group, int prec, uint64_t reps,
                       double* out) {
  return guard([&] {
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    BenchOptions o;
    o.repetitions = reps;
    const FormatKind k = fmt == 0 ? FormatKind::Csr : fmt == 1 ? FormatKind::Rgcsr
                                                               : FormatKind::Hybrid;
    std::optional<std::size_t> g;
    if (group >= 0) g = static_cast<std::size_t>(group);
    const BenchRecord r = run_spmv_bench(m, "bench", k, g,
                                         prec == 4 ? Precision::Single : Precision::Double, o);
    out[0] = r.median_seconds;
    out[1] = r.gflops;
    out[2] = r.checksum;
    out[3] = static_cast<double>(r.bytes);
  });
}

// Row-slab threaded driver of the UNCHANGED reference spmv_csr / spmv_rgcsr /
// spmv_hybrid (fmt 0 / 1 / 2):
// the matrix is cut into `threads` group-aligned row slabs (each built by the
// reference's own build_rgcsr / build_hybrid on the slab's entries, columns
// global) and each std::thread runs the reference kernel on its slab.  y is
// bitwise equal to the 1-thread run (per-row accumulation order unchanged).
struct RefSlabs {
  int prec;
  int fmt;
  std::vector<std::size_t> row_begin;
  std::vector<RgcsrMatrix<double>> rd;
  std::vector<RgcsrMatrix<float>> rf;
  std::vector<HybridMatrix<double>> hd;
  std::vector<HybridMatrix<float>> hf;
  std::vector<CsrMatrix<double>> cd;  // fmt 0: the reference's spmv_csr
  std::vector<CsrMatrix<float>> cf;
  std::size_t cols;
};

int ref_slabs_build(const void* h, int fmt, uint64_t group, int64_t k1, int prec, int threads,
                    void** out) {
  return guard([&] {
    const auto& m = static_cast<const RefMatrix*>(h)->m;
    auto s = std::make_unique<RefSlabs>();
    s->prec = prec;
    s->fmt = fmt;
    s->cols = m.num_cols();
    const std::size_t n = m.num_rows();
    const std::size_t unit = fmt == 1 ? group : 1;
    const std::size_t units = (n + unit - 1) / unit;
    // per-slab hybrid width: the GLOBAL width, so the split is the global one
    std::optional<std::size_t> w;
    if (fmt == 2) w = k1 >= 0 ? static_cast<std::size_t>(k1) : choose_ell_width(row_lengths(m));
    const auto& es = m.entries();
    std::size_t pos = 0;
    for (int t = 0; t < threads; ++t) {
      const std::size_t r0 = std::min(n, units * t / threads * unit);
      const std::size_t r1 = std::min(n, units * (t + 1) / threads * unit);
      s->row_begin.push_back(r0);
      std::vector<Entry> part;
      while (pos < es.size() && es[pos].row < r1) {
        Entry e = es[pos++];
        e.row -= static_cast<index_t>(r0);
        part.push_back(e);
      }
      TripletMatrix tm(r1 - r0, m.num_cols(), std::move(part));
      if (fmt == 0) {
        if (prec == 4) s->cf.push_back(build_csr<float>(tm));
        else s->cd.push_back(build_csr<double>(tm));
      } else if (fmt == 1) {
        if (prec == 4) s->rf.push_back(build_rgcsr<float>(tm, group));
        else s->rd.push_back(build_rgcsr<double>(tm, group));
      } else {
        std::size_t ml = 0;
        for (auto l : row_lengths(tm)) ml = std::max(ml, l);
        std::optional<std::size_t> wl = std::min(*w, ml);
        if (prec == 4) s->hf.push_back(build_hybrid<float>(tm, wl));
        else s->hd.push_back(build_hybrid<double>(tm, wl));
      }
    }
    s->row_begin.push_back(n);
    *out = s.release();
  });
}

int ref_slabs_spmv(const void* h, const void* x, void* y) {
  return guard([&] {
    const auto* s = static_cast<const RefSlabs*>(h);
    const std::size_t nt = s->row_begin.size() - 1;
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t < nt; ++t) {
      pool.emplace_back([s, t, x, y] {
        const std::size_t r0 = s->row_begin[t], r1 = s->row_begin[t + 1];
        if (s->prec == 4) {
          std::span<const float> xs(static_cast<const float*>(x), s->cols);
          std::span<float> ys(static_cast<float*>(y) + r0, r1 - r0);
          if (s->fmt == 0) spmv_csr(s->cf[t], xs, ys);
          else if (s->fmt == 1) spmv_rgcsr(s->rf[t], xs, ys);
          else spmv_hybrid(s->hf[t], xs, ys);
        } else {
          std::span<const double> xs(static_cast<const double*>(x), s->cols);
          std::span<double> ys(static_cast<double*>(y) + r0, r1 - r0);
          if (s->fmt == 0) spmv_csr(s->cd[t], xs, ys);
          else if (s->fmt == 1) spmv_rgcsr(s->rd[t], xs, ys);
          else spmv_hybrid(s->hd[t], xs, ys);
        }
      });
    }
    for (auto& th : pool) th.join();
  });
}

// The same slabs run one after another on the calling thread: the reference's
// single-core SpMV over all rows (its per-row work and order are unchanged).
int ref_slabs_spmv_serial(const void* h, const void* x, void* y) {
  return guard([&] {
    const auto* s = static_cast<const RefSlabs*>(h);
    for (std::size_t t = 0; t + 1 < s->row_begin.size(); ++t) {
      const std::size_t r0 = s->row_begin[t], r1 = s->row_begin[t + 1];
      if (s->prec == 4) {
        std::span<const float> xs(static_cast<const float*>(x), s->cols);
        std::span<float> ys(static_cast<float*>(y) + r0, r1 - r0);
        if (s->fmt == 0) spmv_csr(s->cf[t], xs, ys);
        else if (s->fmt == 1) spmv_rgcsr(s->rf[t], xs, ys);
        else spmv_hybrid(s->hf[t], xs, ys);
      } else {
        std::span<const double> xs(static_cast<const double*>(x), s->cols);
        std::span<double> ys(static_cast<double*>(y) + r0, r1 - r0);
        if (s->fmt == 0) spmv_csr(s->cd[t], xs, ys);
        else if (s->fmt == 1) spmv_rgcsr(s->rd[t], xs, ys);
        else spmv_hybrid(s->hd[t], xs, ys);
      }
    }
  });
}

// Slab t of an RgCSR slab set (fmt 1): info[0..3] = row_begin, row_end,
// slots, groups; then (when the pointers are non-null) the reference's four
// arrays of that slab, so a config-scale comparison needs one slab at a time.
int ref_slabs_rgcsr_part(const void* h, uint64_t t, uint64_t* info, void* values,
                         uint32_t* columns, uint32_t* group_pointers, uint32_t* row_lengths) {
  return guard([&] {
    const auto* s = static_cast<const RefSlabs*>(h);
    if (s->fmt != 1) throw std::invalid_argument("ref_slabs_rgcsr_part: not an RgCSR slab set");
    if (t + 1 >= s->row_begin.size()) throw std::invalid_argument("ref_slabs_rgcsr_part: slab");
    auto put = [&](const auto& a) {
      info[0] = s->row_begin[t];
      info[1] = s->row_begin[t + 1];
      info[2] = a.values.size();
      info[3] = a.group_pointers.size() - 1;
      if (values) std::copy(a.values.begin(), a.values.end(),
                            static_cast<typename std::decay_t<decltype(a.values)>::value_type*>(values));
      if (columns) std::copy(a.columns.begin(), a.columns.end(), columns);
      if (group_pointers) std::copy(a.group_pointers.begin(), a.group_pointers.end(), group_pointers);
      if (row_lengths) std::copy(a.row_lengths.begin(), a.row_lengths.end(), row_lengths);
    };
    if (s->prec == 4) put(s->rf[t]);
    else put(s->rd[t]);
  });
}

uint64_t ref_slabs_count(const void* h) {
  return static_cast<const RefSlabs*>(h)->row_begin.size() - 1;
}

void ref_slabs_free(void* h) { delete static_cast<RefSlabs*>(h); }

}  // extern "C"
