// Matrix Market ingest -> canonical CSR.
//
// Same accepted language, messages and line numbers as the reference parser
// (src/matrix_market.cpp:61-138): banner `%%MatrixMarket matrix coordinate
// {real|integer|pattern} {general|symmetric}` (case-insensitive), comment /
// blank lines, a size line, then exactly `declared` entry lines parsed with
// strtol / strtod (trailing characters rejected), 1-based indices checked
// against the declared bounds, pattern values 1.0, symmetric storage expanded
// with the mirror emitted right after its entry.  The result is canonicalised
// like spmvkit::canonicalize (src/triplet.cpp:34-49): std::sort on (row, col)
// — the same libstdc++ algorithm on the same sequence, so duplicate entries
// are summed in the same order — then duplicates summed.
//
// The entry section is parsed in parallel (one chunk of lines per hardware
// thread, concatenated in file order, so the raw sequence is the reference's),
// and the sort is skipped when the raw entries are already strictly
// increasing (then std::sort would be the identity).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spmvk.h"

namespace spmvk {
void set_last_error(const std::string& msg);  // common.cu
}

namespace {

struct Raw {
  uint32_t row, col;
  double value;
};

struct ParseError {
  uint64_t line;
  std::string msg;
};

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(),
                 [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
  return s;
}

// One line [b, e) of the buffer (without the newline), CR stripped.
struct Line {
  const char* b;
  const char* e;
};

bool blank(const Line& l) {
  for (const char* p = l.b; p < l.e; ++p)
    if (*p != ' ' && *p != '\t') return false;
  return true;
}

struct Parsed {
  std::vector<Raw> raw;
  uint64_t entries = 0;
  bool has_error = false;
  ParseError err;
};

// Parses entry lines [lb, le) (line numbers from first_no) of the entry
// section.  Stops at the first error (the earliest line wins overall).
void parse_entries(const std::vector<Line>& lines, size_t lb, size_t le, uint64_t first_no,
                   bool has_value, bool symmetric, uint64_t rows, uint64_t cols, Parsed& out) {
  std::string buf;
  for (size_t i = lb; i < le; ++i) {
    const Line& l = lines[i];
    const uint64_t line_no = first_no + (i - lb);
    if (l.b < l.e && *l.b == '%') continue;
    if (blank(l)) continue;
    buf.assign(l.b, l.e);  // NUL-terminated copy for strtol / strtod
    const char* p = buf.c_str();
    char* end = nullptr;
    const long r = std::strtol(p, &end, 10);
    if (end == p) { out.has_error = true; out.err = {line_no, "expected row index"}; return; }
    p = end;
    const long c = std::strtol(p, &end, 10);
    if (end == p) { out.has_error = true; out.err = {line_no, "expected column index"}; return; }
    p = end;
    double v = 1.0;
    if (has_value) {
      v = std::strtod(p, &end);
      if (end == p) { out.has_error = true; out.err = {line_no, "expected value"}; return; }
      p = end;
    }
    while (*p == ' ' || *p == '\t') ++p;
    if (*p != '\0') {
      out.has_error = true;
      out.err = {line_no, "trailing characters after entry"};
      return;
    }
    if (r < 1 || static_cast<uint64_t>(r) > rows || c < 1 || static_cast<uint64_t>(c) > cols) {
      out.has_error = true;
      out.err = {line_no, "index out of declared bounds"};
      return;
    }
    const uint32_t rr = static_cast<uint32_t>(r - 1), cc = static_cast<uint32_t>(c - 1);
    out.raw.push_back({rr, cc, v});
    if (symmetric && rr != cc) out.raw.push_back({cc, rr, v});
    ++out.entries;
  }
}


struct Result {
  uint64_t rows = 0, cols = 0;
  std::vector<uint32_t> rp, col;
  std::vector<double> val;
};

// Throws ParseError.  `text` holds the whole file.
Result parse(const char* text, uint64_t len, int threads) {
  std::vector<Line> lines;
  lines.reserve(len / 16 + 16);
  const char* p = text;
  const char* end = text + len;
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
    const char* le = nl ? nl : end;
    const char* lb = p;
    const char* lee = (le > lb && le[-1] == '\r') ? le - 1 : le;
    lines.push_back({lb, lee});
    p = nl ? nl + 1 : end;
  }
  // std::getline semantics: a final line without '\n' still counts; an empty
  // trailing piece after the last '\n' does not exist.
  if (lines.empty()) throw ParseError{1, "empty input"};
  size_t li = 0;
  const std::string first(lines[0].b, lines[0].e);
  std::istringstream banner(first);
  std::string tag, object, format, field, symmetry;
  banner >> tag >> object >> format >> field >> symmetry;
  if (tag != "%%MatrixMarket") throw ParseError{1, "malformed banner: " + first};
  object = lower(object);
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (object != "matrix") throw ParseError{1, "unsupported object '" + object + "'"};
  if (format != "coordinate")
    throw ParseError{1, "unsupported format '" + format + "' (only coordinate)"};
  if (field != "real" && field != "integer" && field != "pattern")
    throw ParseError{1, "unsupported field '" + field + "'"};
  if (symmetry != "general" && symmetry != "symmetric")
    throw ParseError{1, "unsupported symmetry '" + symmetry + "'"};
  const bool has_value = field != "pattern";
  const bool symmetric = symmetry == "symmetric";
  li = 1;
  uint64_t rows = 0, cols = 0, declared = 0;
  for (;;) {
    if (li >= lines.size()) throw ParseError{li + 1, "missing size line"};
    const Line& l = lines[li++];
    if (l.b < l.e && *l.b == '%') continue;
    if (blank(l)) continue;
    std::istringstream sl(std::string(l.b, l.e));
    long long r = -1, c = -1, n = -1;
    sl >> r >> c >> n;
    if (sl.fail() || r < 0 || c < 0 || n < 0)
      throw ParseError{li, "malformed size line: " + std::string(l.b, l.e)};
    rows = static_cast<uint64_t>(r);
    cols = static_cast<uint64_t>(c);
    declared = static_cast<uint64_t>(n);
    break;
  }
  if (symmetric && rows != cols) throw ParseError{li, "symmetric matrix must be square"};
  // Parallel entry parse over line chunks, concatenated in file order.
  const size_t nlines = lines.size() - li;
  const int T = std::max(1, std::min<int>(threads, static_cast<int>(nlines / 65536) + 1));
  std::vector<Parsed> parts(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) {
    const size_t b = li + nlines * t / T, e = li + nlines * (t + 1) / T;
    pool.emplace_back([&, b, e, t] {
      parts[t].raw.reserve((e - b) * (symmetric ? 2 : 1));
      parse_entries(lines, b, e, b + 1, has_value, symmetric, rows, cols, parts[t]);
    });
  }
  for (auto& th : pool) th.join();
  // Reference order of checks: a line is rejected for "more entries than
  // declared" before it is parsed; otherwise the first failing line wins.
  uint64_t seen = 0;
  for (int t = 0; t < T; ++t) {
    const Parsed& P = parts[t];
    // entries of this chunk that precede its error (if any) all parsed fine
    if (seen + P.entries > declared) {
      // find the line of entry number declared + 1 inside this chunk
      const size_t b = li + nlines * t / T, e = li + nlines * (t + 1) / T;
      uint64_t k = seen;
      for (size_t i = b; i < e; ++i) {
        const Line& l = lines[i];
        if ((l.b < l.e && *l.b == '%') || blank(l)) continue;
        if (k == declared) throw ParseError{i + 1, "more entries than declared"};
        ++k;
      }
    }
    if (P.has_error) {
      if (seen + P.entries == declared) {
        // the failing line is an extra entry line: the count check fires first
        throw ParseError{P.err.line, "more entries than declared"};
      }
      throw P.err;
    }
    seen += P.entries;
  }
  if (seen != declared)
    throw ParseError{lines.size(), "declared " + std::to_string(declared) + " entries, found " +
                                       std::to_string(seen)};
  std::vector<Raw> raw;
  {
    size_t total = 0;
    for (auto& P : parts) total += P.raw.size();
    raw.reserve(total);
    for (auto& P : parts) raw.insert(raw.end(), P.raw.begin(), P.raw.end());
  }
  // canonicalize (src/triplet.cpp:34-49): std::sort on (row, col), sum duplicates
  auto less = [](const Raw& a, const Raw& b) {
    return a.row < b.row || (a.row == b.row && a.col < b.col);
  };
  bool strictly_sorted = true;
  for (size_t i = 1; i < raw.size() && strictly_sorted; ++i)
    strictly_sorted = less(raw[i - 1], raw[i]);
  if (!strictly_sorted) std::sort(raw.begin(), raw.end(), less);
  Result res;
  res.rows = rows;
  res.cols = cols;
  res.rp.assign(rows + 1, 0);
  res.col.reserve(raw.size());
  res.val.reserve(raw.size());
  uint32_t prow = 0, pcol = 0;
  bool any = false;
  for (const Raw& e : raw) {
    if (any && prow == e.row && pcol == e.col) {
      res.val.back() += e.value;
    } else {
      res.col.push_back(e.col);
      res.val.push_back(e.value);
      ++res.rp[e.row + 1];
      prow = e.row;
      pcol = e.col;
      any = true;
    }
  }
  for (uint64_t r = 0; r < rows; ++r) res.rp[r + 1] += res.rp[r];
  return res;
}

int run_parse(const char* text, uint64_t len, int threads, void* stream, int val_prec,
              spmvk_csr** out, uint64_t* error_line) {
  if (error_line) *error_line = 0;
  Result r;
  try {
    r = parse(text, len, threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency()));
  } catch (const ParseError& e) {
    spmvk::set_last_error("line " + std::to_string(e.line) + ": " + e.msg);
    if (error_line) *error_line = e.line;
    return SPMVK_EPARSE;
  } catch (const std::bad_alloc&) {
    spmvk::set_last_error("host allocation failed");
    return SPMVK_ENOMEM;
  }
  if (val_prec == SPMVK_F32) {
    std::vector<float> v32(r.val.begin(), r.val.end());
    return spmvk_csr_upload(r.rows, r.cols, r.col.size(), r.rp.data(), r.col.data(), v32.data(),
                            SPMVK_F32, stream, out);
  }
  return spmvk_csr_upload(r.rows, r.cols, r.col.size(), r.rp.data(), r.col.data(), r.val.data(),
                          SPMVK_F64, stream, out);
}

// write_matrix_market (src/matrix_market.cpp:150-158): banner, "rows cols
// nnz", then 1-based "row col %.17g" per entry in (row, col) order.  Rows are
// formatted by `threads` host threads into per-thread strings, concatenated.
std::string format_mm(const spmvk_csr* a, int threads) {
  uint64_t rows = 0, cols = 0, nnz = 0;
  int prec = 0;
  if (spmvk_csr_shape(a, &rows, &cols, &nnz, &prec) != SPMVK_OK)
    throw std::runtime_error(spmvk_last_error());
  std::vector<uint32_t> rp(rows + 1), col(nnz);
  std::vector<double> val(nnz);
  if (prec == SPMVK_F32) {
    std::vector<float> v32(nnz);
    if (spmvk_csr_download(a, rp.data(), col.data(), v32.data()) != SPMVK_OK)
      throw std::runtime_error(spmvk_last_error());
    for (uint64_t i = 0; i < nnz; ++i) val[i] = v32[i];
  } else if (spmvk_csr_download(a, rp.data(), col.data(), val.data()) != SPMVK_OK) {
    throw std::runtime_error(spmvk_last_error());
  }
  std::string head = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(rows) +
                     ' ' + std::to_string(cols) + ' ' + std::to_string(nnz) + '\n';
  const int T = std::max(1, std::min<int>(threads, static_cast<int>((rows + 4095) / 4096)));
  std::vector<std::string> part(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      const uint64_t r0 = rows * t / T, r1 = rows * (t + 1) / T;
      std::string& o = part[t];
      o.reserve((rp[r1] - rp[r0]) * 32);
      char buf[96];
      for (uint64_t r = r0; r < r1; ++r)
        for (uint32_t k = rp[r]; k < rp[r + 1]; ++k) {
          const int n = std::snprintf(buf, sizeof buf, "%llu %llu %.17g\n",
                                      static_cast<unsigned long long>(r + 1),
                                      static_cast<unsigned long long>(col[k]) + 1, val[k]);
          o.append(buf, static_cast<size_t>(n));
        }
    });
  }
  for (auto& th : pool) th.join();
  for (const auto& p : part) head += p;
  return head;
}

}  // namespace

extern "C" {

int spmvk_mm_write(const spmvk_csr* a, int threads, char* buf, uint64_t cap, uint64_t* len) {
  if (!a || !len) {
    spmvk::set_last_error("null argument");
    return SPMVK_EINVAL;
  }
  try {
    const std::string text =
        format_mm(a, threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency()));
    *len = text.size();
    if (!buf) return SPMVK_OK;
    if (cap < text.size()) {
      spmvk::set_last_error("write_matrix_market: buffer of " + std::to_string(cap) +
                            " bytes, need " + std::to_string(text.size()));
      return SPMVK_ERANGE;
    }
    std::memcpy(buf, text.data(), text.size());
    return SPMVK_OK;
  } catch (const std::bad_alloc&) {
    spmvk::set_last_error("host allocation failed");
    return SPMVK_ENOMEM;
  } catch (const std::exception& e) {
    spmvk::set_last_error(e.what());
    return SPMVK_ECUDA;
  }
}

int spmvk_mm_save(const spmvk_csr* a, const char* path, int threads) {
  if (!a || !path) {
    spmvk::set_last_error("null argument");
    return SPMVK_EINVAL;
  }
  try {
    const std::string text =
        format_mm(a, threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency()));
    std::ofstream out(path, std::ios::binary);
    if (!out) {  // save_matrix_market (:160-164)
      spmvk::set_last_error(std::string("cannot open ") + path + " for writing");
      return SPMVK_ERANGE;
    }
    out.write(text.data(), static_cast<std::streamsize>(text.size()));
    return out ? SPMVK_OK : SPMVK_ERANGE;
  } catch (const std::bad_alloc&) {
    spmvk::set_last_error("host allocation failed");
    return SPMVK_ENOMEM;
  } catch (const std::exception& e) {
    spmvk::set_last_error(e.what());
    return SPMVK_ECUDA;
  }
}

int spmvk_mm_parse(const char* text, uint64_t len, int threads, int val_prec, void* stream,
                   spmvk_csr** out, uint64_t* error_line) {
  if (!text || !out) {
    spmvk::set_last_error("null argument");
    return SPMVK_EINVAL;
  }
  return run_parse(text, len, threads, stream, val_prec, out, error_line);
}

int spmvk_mm_load(const char* path, int threads, int val_prec, void* stream, spmvk_csr** out,
                  uint64_t* error_line) {
  if (!path || !out) {
    spmvk::set_last_error("null argument");
    return SPMVK_EINVAL;
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    spmvk::set_last_error(std::string("cannot open ") + path);
    return SPMVK_ERANGE;
  }
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const int rc = run_parse(text.data(), text.size(), threads, stream, val_prec, out, error_line);
  if (rc == SPMVK_EPARSE) spmvk::set_last_error(std::string(path) + ": " + spmvk_last_error());
  return rc;
}

}  // extern "C"
