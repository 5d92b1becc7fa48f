// include/spmvkit_gpu.hpp — header-only C++20 shim restoring the reference's
// hot-path names, signatures and exceptions on top of the C-ABI (spmvk.h).
//
// A user of the reference (/root/reference/proj/core) switches
//     #include <spmvkit/rgcsr.hpp>     spmvkit::build_rgcsr<double>(m, 32)
// to
//     #include <spmvkit_gpu.hpp>       spmvkit::gpu::build_rgcsr<double>(m, 32)
// with the same TripletMatrix `m` (any type exposing num_rows(), num_cols(),
// nnz() and entries() with .row/.col/.value, i.e. spmvkit::TripletMatrix,
// core/include/spmvkit/triplet.hpp:26-45), the same std::span overloads and
// the same exceptions: std::invalid_argument where the reference throws it,
// std::runtime_error for size overflow (which the reference does not detect).
//
// Entry points (reference file:line relative to proj/core/include/spmvkit/):
//   build_rgcsr<S>(m, G)                rgcsr.hpp:38-39
//   spmv_rgcsr(a, x, y, &madds)         rgcsr.hpp:75-77 (+ vector overload :99-105)
//   build_hybrid<S>(m, k1)              ellpack.hpp:170-172
//   spmv_hybrid(h, x, y)                ellpack.hpp:206-210
//   build_ellpack<S>(m, budget)         ellpack.hpp:84-107
//   spmv_ellpack(h, x, y)               ellpack.hpp:110-130
//   spmv_coo(h, x, y)                   ellpack.hpp:132-141
//   choose_ell_width(lens)              ellpack.hpp:153
//   hybrid_split_cost(lens, k)          ellpack.hpp:145
// The span overloads take HOST memory (H2D / D2H inside, synchronous).  For
// device-resident iteration use spmv_rgcsr_device() with device pointers.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "spmvk.h"

namespace spmvkit::gpu {

namespace detail {

inline void check(int rc) {
  if (rc == SPMVK_OK) return;
  const std::string msg = spmvk_last_error();
  if (rc == SPMVK_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

template <class S>
constexpr int prec() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, double>);
  return std::is_same_v<S, float> ? SPMVK_F32 : SPMVK_F64;
}

struct CsrDeleter {
  void operator()(spmvk_csr* p) const { spmvk_csr_destroy(p); }
};
using CsrPtr = std::unique_ptr<spmvk_csr, CsrDeleter>;

// TripletMatrix -> device CSR (entries are canonical: sorted, unique).
template <class Triplets>
CsrPtr upload(const Triplets& m) {
  const std::size_t n = m.num_rows(), nnz = m.nnz();
  std::vector<std::uint32_t> rp(n + 1, 0), col;
  std::vector<double> val;
  col.reserve(nnz);
  val.reserve(nnz);
  for (const auto& e : m.entries()) {
    ++rp[static_cast<std::size_t>(e.row) + 1];
    col.push_back(static_cast<std::uint32_t>(e.col));
    val.push_back(static_cast<double>(e.value));
  }
  for (std::size_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  spmvk_csr* h = nullptr;
  check(spmvk_csr_upload(n, m.num_cols(), nnz, rp.data(), col.data(), val.data(), SPMVK_F64,
                         nullptr, &h));
  return CsrPtr(h);
}

}  // namespace detail

// ------------------------------------------------------------------ RgCSR
template <class Scalar = double>
class RgcsrMatrix {
 public:
  std::size_t num_rows = 0, num_cols = 0, group_size = 0;

  std::size_t num_groups() const noexcept { return info_.num_groups; }
  std::size_t rows_in_group(std::size_t g) const noexcept {
    return std::min(group_size, num_rows - g * group_size);
  }
  std::size_t slot_count() const noexcept { return info_.slots; }
  const spmvk_rgcsr_info& info() const noexcept { return info_; }
  const spmvk_rgcsr* handle() const noexcept { return h_.get(); }

  // The reference's public arrays (rgcsr.hpp:24-27), copied to the host.
  struct Arrays {
    std::vector<Scalar> values;
    std::vector<std::uint32_t> columns, group_pointers, row_lengths;
  };
  Arrays to_host() const {
    Arrays a;
    a.values.resize(info_.slots);
    a.columns.resize(info_.slots);
    a.group_pointers.resize(info_.num_groups + 1);
    a.row_lengths.resize(info_.num_rows);
    detail::check(spmvk_rgcsr_download(h_.get(), a.values.data(), a.columns.data(),
                                       a.group_pointers.data(), a.row_lengths.data()));
    return a;
  }

 private:
  struct Del {
    void operator()(spmvk_rgcsr* p) const { spmvk_rgcsr_destroy(p); }
  };
  std::shared_ptr<spmvk_rgcsr> h_;
  spmvk_rgcsr_info info_{};

  template <class S, class T>
  friend RgcsrMatrix<S> build_rgcsr(const T&, std::size_t);
};

template <class Scalar = double, class Triplets>
RgcsrMatrix<Scalar> build_rgcsr(const Triplets& m, std::size_t group_size) {
  if (group_size == 0) throw std::invalid_argument("build_rgcsr: group size must be nonzero");
  auto csr = detail::upload(m);
  spmvk_rgcsr* h = nullptr;
  detail::check(spmvk_rgcsr_build(csr.get(), group_size, detail::prec<Scalar>(), nullptr, &h));
  RgcsrMatrix<Scalar> a;
  a.h_ = std::shared_ptr<spmvk_rgcsr>(h, typename RgcsrMatrix<Scalar>::Del{});
  detail::check(spmvk_rgcsr_get_info(h, &a.info_));
  a.num_rows = a.info_.num_rows;
  a.num_cols = a.info_.num_cols;
  a.group_size = a.info_.group_size;
  return a;
}

template <class Scalar>
void spmv_rgcsr(const RgcsrMatrix<Scalar>& a, std::span<const Scalar> x, std::span<Scalar> y,
                std::uint64_t* multiply_add_count = nullptr) {
  if constexpr (std::is_same_v<Scalar, double>)
    detail::check(spmvk_rgcsr_spmv_host_f64(a.handle(), x.data(), x.size(), y.data(), y.size(),
                                            multiply_add_count));
  else
    detail::check(spmvk_rgcsr_spmv_host_f32(a.handle(), x.data(), x.size(), y.data(), y.size(),
                                            multiply_add_count));
}

template <class Scalar>
std::vector<Scalar> spmv_rgcsr(const RgcsrMatrix<Scalar>& a, const std::vector<Scalar>& x,
                               std::uint64_t* multiply_add_count = nullptr) {
  std::vector<Scalar> y(a.num_rows);
  spmv_rgcsr(a, std::span<const Scalar>(x), std::span<Scalar>(y), multiply_add_count);
  return y;
}

// Device-resident form: x_dev / y_dev are device pointers, `stream` a cudaStream_t.
template <class Scalar>
void spmv_rgcsr_device(const RgcsrMatrix<Scalar>& a, const Scalar* x_dev, std::size_t nx,
                       Scalar* y_dev, std::size_t ny, void* stream = nullptr) {
  if constexpr (std::is_same_v<Scalar, double>)
    detail::check(spmvk_rgcsr_spmv_f64(a.handle(), x_dev, nx, y_dev, ny, stream));
  else
    detail::check(spmvk_rgcsr_spmv_f32(a.handle(), x_dev, nx, y_dev, ny, stream));
}

// ------------------------------------------------------------------ Hybrid
inline std::size_t hybrid_split_cost(std::span<const std::size_t> lens, std::size_t k) {
  std::vector<std::uint64_t> v(lens.begin(), lens.end());
  return spmvk_hybrid_split_cost(v.data(), v.size(), k);
}

inline std::size_t choose_ell_width(std::span<const std::size_t> lens) {
  std::vector<std::uint64_t> v(lens.begin(), lens.end());
  return spmvk_choose_ell_width(v.data(), v.size());
}

template <class Scalar = double>
class HybridMatrix {
 public:
  std::size_t num_rows = 0, num_cols = 0, slots_per_row = 0;
  const spmvk_hybrid_info& info() const noexcept { return info_; }
  const spmvk_hybrid* handle() const noexcept { return h_.get(); }

  struct Arrays {
    std::vector<Scalar> ell_values, coo_values;
    std::vector<std::uint32_t> ell_columns, coo_rows, coo_columns;
  };
  Arrays to_host() const {
    Arrays a;
    a.ell_values.resize(info_.ell_slots);
    a.ell_columns.resize(info_.ell_slots);
    a.coo_rows.resize(info_.coo_nnz);
    a.coo_columns.resize(info_.coo_nnz);
    a.coo_values.resize(info_.coo_nnz);
    detail::check(spmvk_hybrid_download(h_.get(), a.ell_values.data(), a.ell_columns.data(),
                                        a.coo_rows.data(), a.coo_columns.data(),
                                        a.coo_values.data()));
    return a;
  }

 private:
  struct Del {
    void operator()(spmvk_hybrid* p) const { spmvk_hybrid_destroy(p); }
  };
  std::shared_ptr<spmvk_hybrid> h_;
  spmvk_hybrid_info info_{};

  template <class S, class T>
  friend HybridMatrix<S> build_hybrid(const T&, std::optional<std::size_t>);
  template <class S, class T>
  friend HybridMatrix<S> build_ellpack(const T&, std::size_t);
  template <class S>
  friend HybridMatrix<S> adopt_hybrid(spmvk_hybrid*);
};

template <class Scalar>
HybridMatrix<Scalar> adopt_hybrid(spmvk_hybrid* h) {
  HybridMatrix<Scalar> a;
  a.h_ = std::shared_ptr<spmvk_hybrid>(h, typename HybridMatrix<Scalar>::Del{});
  detail::check(spmvk_hybrid_get_info(h, &a.info_));
  a.num_rows = a.info_.num_rows;
  a.num_cols = a.info_.num_cols;
  a.slots_per_row = a.info_.ell_width;
  return a;
}

inline constexpr std::size_t kDefaultEllSlotBudget = std::size_t{1} << 31;

// build_ellpack<S>(m, slot_budget) (ellpack.hpp:84-107): the ELL-only Hybrid;
// throws std::runtime_error past the slot budget, like the reference.
template <class Scalar = double, class Triplets>
HybridMatrix<Scalar> build_ellpack(const Triplets& m,
                                   std::size_t slot_budget = kDefaultEllSlotBudget) {
  auto csr = detail::upload(m);
  spmvk_hybrid* h = nullptr;
  detail::check(spmvk_ellpack_build(csr.get(), slot_budget, detail::prec<Scalar>(), nullptr, &h));
  return adopt_hybrid<Scalar>(h);
}

template <class Scalar = double, class Triplets>
HybridMatrix<Scalar> build_hybrid(const Triplets& m, std::optional<std::size_t> k1 = std::nullopt) {
  auto csr = detail::upload(m);
  spmvk_hybrid* h = nullptr;
  detail::check(spmvk_hybrid_build(csr.get(), k1 ? static_cast<std::int64_t>(*k1) : -1,
                                   detail::prec<Scalar>(), nullptr, &h));
  return adopt_hybrid<Scalar>(h);
}

template <class Scalar>
void spmv_hybrid(const HybridMatrix<Scalar>& h, std::span<const Scalar> x, std::span<Scalar> y) {
  if constexpr (std::is_same_v<Scalar, double>)
    detail::check(spmvk_hybrid_spmv_host_f64(h.handle(), x.data(), x.size(), y.data(), y.size()));
  else
    detail::check(spmvk_hybrid_spmv_host_f32(h.handle(), x.data(), x.size(), y.data(), y.size()));
}

template <class Scalar>
std::vector<Scalar> spmv_hybrid(const HybridMatrix<Scalar>& h, const std::vector<Scalar>& x) {
  std::vector<Scalar> y(h.num_rows);
  spmv_hybrid(h, std::span<const Scalar>(x), std::span<Scalar>(y));
  return y;
}

// spmv_ellpack(h.ell, x, y) (ellpack.hpp:110-130): the ELL part of a Hybrid
// (all of an ELLPACK); every slot walked, as the reference.
template <class Scalar>
void spmv_ellpack(const HybridMatrix<Scalar>& h, std::span<const Scalar> x, std::span<Scalar> y) {
  if constexpr (std::is_same_v<Scalar, double>)
    detail::check(spmvk_hybrid_spmv_ell_host_f64(h.handle(), x.data(), x.size(), y.data(),
                                                 y.size()));
  else
    detail::check(spmvk_hybrid_spmv_ell_host_f32(h.handle(), x.data(), x.size(), y.data(),
                                                 y.size()));
}

template <class Scalar>
std::vector<Scalar> spmv_ellpack(const HybridMatrix<Scalar>& h, const std::vector<Scalar>& x) {
  std::vector<Scalar> y(h.num_rows);
  spmv_ellpack(h, std::span<const Scalar>(x), std::span<Scalar>(y));
  return y;
}

// spmv_coo(h.coo, x, y) (ellpack.hpp:132-141): y[row] += v * x[col] over the
// COO part in array order; std::invalid_argument for entries outside x / y.
template <class Scalar>
void spmv_coo(const HybridMatrix<Scalar>& h, std::span<const Scalar> x, std::span<Scalar> y) {
  if constexpr (std::is_same_v<Scalar, double>)
    detail::check(spmvk_hybrid_spmv_coo_host_f64(h.handle(), x.data(), x.size(), y.data(),
                                                 y.size()));
  else
    detail::check(spmvk_hybrid_spmv_coo_host_f32(h.handle(), x.data(), x.size(), y.data(),
                                                 y.size()));
}

}  // namespace spmvkit::gpu
