// oracle/parity_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// The drop-in demonstrated in the reference's own language: the reference's
// spmvkit::TripletMatrix inputs (its own random_matrix / banded_matrix
// generators) go through include/spmvkit_gpu.hpp (the C++ shim over the
// C-ABI, i.e. the B200 kernels) and are compared BITWISE with the reference's
// build_rgcsr / spmv_rgcsr / build_hybrid / spmv_hybrid on the same inputs.
// Same shape as the reference's tests/acceptance.cpp runner (one PASS/FAIL
// line per criterion).  Built by oracle/Makefile into _ref/ (it links the
// reference), run by tests/test_gpu_cpp_shim.py on the GPU box.
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "spmvkit/spmvkit.hpp"
#include "spmvkit_gpu.hpp"

namespace {

using namespace spmvkit;

int failures = 0;

void criterion(const char* name, const std::function<std::string()>& body) {
  std::string why;
  try {
    why = body();
  } catch (const std::exception& e) {
    why = std::string("exception: ") + e.what();
  }
  std::printf("%s: %s%s%s\n", why.empty() ? "PASS" : "FAIL", name, why.empty() ? "" : ": ",
              why.c_str());
  if (!why.empty()) ++failures;
}

template <class T>
bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}

template <class T, class U>
bool same_u32(const std::vector<T>& a, const std::vector<U>& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i)
    if (static_cast<std::uint64_t>(a[i]) != static_cast<std::uint64_t>(b[i])) return false;
  return true;
}

TripletMatrix random_case(std::uint64_t seed, std::size_t max_rows) {
  std::mt19937_64 rng(seed);
  RandomMatrixSpec spec;
  spec.rows = 1 + rng() % max_rows;
  spec.cols = 1 + rng() % max_rows;
  spec.density = 0.05 + 0.25 * unit_real(rng);
  spec.integer_values = seed % 2 == 0;
  return random_matrix(spec, rng());
}

template <class S>
std::string rgcsr_case(const TripletMatrix& m, std::size_t G, std::uint64_t xseed) {
  const auto ref = build_rgcsr<S>(m, G);
  const auto dev = gpu::build_rgcsr<S>(m, G);
  const auto h = dev.to_host();
  if (!same_bits(h.values, ref.values)) return "values differ (G=" + std::to_string(G) + ")";
  if (!same_u32(h.columns, ref.columns)) return "columns differ";
  if (!same_u32(h.group_pointers, ref.group_pointers)) return "group pointers differ";
  if (!same_u32(h.row_lengths, ref.row_lengths)) return "row lengths differ";
  const auto xd = random_vector(m.num_cols(), xseed);
  const std::vector<S> x(xd.begin(), xd.end());
  std::uint64_t m1 = 0, m2 = 0;
  const auto y_ref = spmv_rgcsr(ref, x, &m1);
  const auto y_dev = gpu::spmv_rgcsr(dev, x, &m2);
  if (!same_bits(y_dev, y_ref)) return "y differs";
  if (m1 != m2) return "multiply-add count differs";
  return {};
}

template <class S>
std::string hybrid_case(const TripletMatrix& m, std::optional<std::size_t> k1, std::uint64_t xseed) {
  const auto ref = build_hybrid<S>(m, k1);
  const auto dev = gpu::build_hybrid<S>(m, k1);
  if (dev.slots_per_row != ref.ell.slots_per_row) return "ELL width differs";
  const auto h = dev.to_host();
  if (!same_bits(h.ell_values, ref.ell.values) || !same_u32(h.ell_columns, ref.ell.columns))
    return "ELL arrays differ";
  if (!same_u32(h.coo_rows, ref.coo.rows) || !same_u32(h.coo_columns, ref.coo.columns) ||
      !same_bits(h.coo_values, ref.coo.values))
    return "COO arrays differ";
  const auto xd = random_vector(m.num_cols(), xseed);
  const std::vector<S> x(xd.begin(), xd.end());
  if (!same_bits(gpu::spmv_hybrid(dev, x), spmv_hybrid(ref, x))) return "y differs";
  return {};
}

// build_ellpack / spmv_ellpack / spmv_coo through the shim vs the reference
// (ellpack.hpp:84-141): arrays, the ELL and COO parts separately (the COO
// part accumulating into a nonzero y), and the slot-budget error.
template <class S>
std::string ellpack_case(const TripletMatrix& m, std::uint64_t xseed) {
  const auto ref = build_ellpack<S>(m);
  const auto dev = gpu::build_ellpack<S>(m);
  if (dev.slots_per_row != ref.slots_per_row) return "ELLPACK width differs";
  const auto h = dev.to_host();
  if (!same_bits(h.ell_values, ref.values) || !same_u32(h.ell_columns, ref.columns))
    return "ELLPACK arrays differ";
  const auto xd = random_vector(m.num_cols(), xseed);
  const std::vector<S> x(xd.begin(), xd.end());
  if (!same_bits(gpu::spmv_ellpack(dev, x), spmv_ellpack(ref, x))) return "spmv_ellpack differs";
  if (m.nnz() == 0) return {};
  const auto hr = build_hybrid<S>(m, std::size_t{1});
  const auto hd = gpu::build_hybrid<S>(m, std::size_t{1});
  if (!same_bits(gpu::spmv_ellpack(hd, x), spmv_ellpack(hr.ell, x))) return "h.ell part differs";
  std::vector<S> y1(m.num_rows()), y2(m.num_rows());
  for (std::size_t i = 0; i < y1.size(); ++i) y1[i] = y2[i] = static_cast<S>(0.25 * i - 3.0);
  spmv_coo(hr.coo, std::span<const S>(x), std::span<S>(y1));
  gpu::spmv_coo(hd, std::span<const S>(x), std::span<S>(y2));
  if (!same_bits(y1, y2)) return "spmv_coo differs";
  return {};
}

}  // namespace

int main() {
  criterion("rgcsr fp64: 200 random_case matrices, G = 1 + seed % 9", [] {
    for (std::uint64_t s = 0; s < 200; ++s) {
      auto w = rgcsr_case<double>(random_case(s, 64), 1 + s % 9, s + 99);
      if (!w.empty()) return w + " at seed " + std::to_string(s);
    }
    return std::string();
  });
  criterion("rgcsr fp32: 200 random_case matrices, G in {1,4,32,33}", [] {
    for (std::uint64_t s = 0; s < 200; ++s) {
      auto w = rgcsr_case<float>(random_case(s, 64), std::size_t{1} << (s % 6), s + 7);
      if (!w.empty()) return w + " at seed " + std::to_string(s);
    }
    return std::string();
  });
  criterion("hybrid fp64/fp32: default and explicit widths", [] {
    for (std::uint64_t s = 0; s < 100; ++s) {
      const auto m = random_case(s, 64);
      auto w = hybrid_case<double>(m, std::nullopt, s);
      if (w.empty()) w = hybrid_case<float>(m, std::nullopt, s);
      if (w.empty() && m.nnz()) w = hybrid_case<double>(m, std::size_t{1}, s);
      if (!w.empty()) return w + " at seed " + std::to_string(s);
    }
    return std::string();
  });
  criterion("banded_matrix n=1e5 hbw=4 (benchmarks/spmv_bench.cpp shape), G 32..256", [] {
    const auto m = banded_matrix(100000, 4, 42);
    for (std::size_t G : {32, 64, 128, 256}) {
      auto w = rgcsr_case<double>(m, G, 1);
      if (!w.empty()) return w;
    }
    return hybrid_case<double>(m, std::nullopt, 1);
  });
  criterion("ellpack + separate ELL / COO parts fp64/fp32: 100 random_case matrices", [] {
    for (std::uint64_t s = 0; s < 100; ++s) {
      const auto m = random_case(s, 64);
      auto w = ellpack_case<double>(m, s);
      if (w.empty()) w = ellpack_case<float>(m, s + 1);
      if (!w.empty()) return w + " at seed " + std::to_string(s);
    }
    try {  // test_formats.cpp:82-85
      gpu::build_ellpack<double>(banded_matrix(100, 2, 1), 0);
    } catch (const std::runtime_error&) {
      return std::string();
    }
    return std::string("no throw past the slot budget");
  });
  criterion("errors: G == 0 and dimension mismatch throw std::invalid_argument", [] {
    const auto m = random_case(3, 64);
    try {
      gpu::build_rgcsr<double>(m, 0);
      return std::string("no throw for G == 0");
    } catch (const std::invalid_argument&) {
    }
    const auto a = gpu::build_rgcsr<double>(m, 4);
    std::vector<double> x(m.num_cols() + 1), y(m.num_rows());
    try {
      gpu::spmv_rgcsr(a, std::span<const double>(x), std::span<double>(y));
      return std::string("no throw for a dimension mismatch");
    } catch (const std::invalid_argument& e) {
      if (std::string(e.what()) != "spmv_rgcsr: dimension mismatch") return std::string(e.what());
    }
    return std::string();
  });
  return failures ? 1 : 0;
}
