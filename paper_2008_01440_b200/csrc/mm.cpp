// SPDX-License-Identifier: Apache-2.0
//
// MatrixMarket ingestion for the device CSR path:
// load_matrix_market / save_matrix_market (proj/src/matrix_market.cpp:55-166,
// 172-199) restated natively, same accepted inputs, same CSR arrays (bitwise),
// same ParseError messages with line numbers.
//
// Loading is built for the paper's large matrices (10^8+ entries): the file is
// read in one block, split at line boundaries into one chunk per host thread,
// and the chunks are tokenised in parallel (line numbers from a parallel
// newline count). The symmetrised triplets go straight into CSR by a row
// histogram and per-row column sorts instead of one global sort. Number parsing
// reproduces `std::istream >> long long / double` under the "C" locale exactly
// (the grammar libstdc++'s num_get accepts, then strtoll / strtod, which are
// correctly rounded, so every value is the reference's double).
#include <locale.h>
#include <omp.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <tuple>
#include <vector>

#include "host_math.hpp"
#include "pcgx.h"

namespace pcgx {
namespace {

struct ParseFail {
  std::string msg;
};

[[noreturn]] void fail_at(const std::string& name, long line, const std::string& what) {
  throw ParseFail{name + ":" + std::to_string(line) + ": " + what};
}

inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// `in >> long long` on [p, e): skip white space, [+-]? digits; no digits or
// overflow fail. Advances p past the digits.
bool get_int(const char*& p, const char* e, long long& v) {
  while (p < e && is_space(*p)) ++p;
  const char* s = p;
  const char* q = p;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  const char* d0 = q;
  while (q < e && *q >= '0' && *q <= '9') ++q;
  if (q == d0) return false;
  char buf[64];
  const size_t len = (size_t)(q - s);
  if (len >= sizeof buf) return false;  // > 20 digits overflows any int64
  std::memcpy(buf, s, len);
  buf[len] = '\0';
  errno = 0;
  char* end = nullptr;
  v = std::strtoll(buf, &end, 10);
  if (errno == ERANGE) return false;
  p = q;
  return true;
}

// `in >> double`: skip white space, collect [+-]? digits [. digits] [(e|E) [+-]? digits]
// (the exponent only after a mantissa digit), then strtod must consume all of it;
// +-inf results fail (libstdc++ __convert_to_v).
bool get_double(const char*& p, const char* e, double& v) {
  while (p < e && is_space(*p)) ++p;
  const char* q = p;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  bool mant = false, dot = false;
  while (q < e) {
    if (*q >= '0' && *q <= '9') {
      mant = true;
      ++q;
    } else if (*q == '.' && !dot) {
      dot = true;
      ++q;
    } else {
      break;
    }
  }
  if (mant && q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    while (q < e && *q >= '0' && *q <= '9') ++q;
  }
  const size_t len = (size_t)(q - p);
  if (len == 0) return false;
  static const locale_t c_loc = newlocale(LC_ALL_MASK, "C", (locale_t)0);
  char sbuf[128];
  std::string big;
  const char* tok = sbuf;
  if (len < sizeof sbuf) {
    std::memcpy(sbuf, p, len);
    sbuf[len] = '\0';
  } else {
    big.assign(p, len);
    tok = big.c_str();
  }
  char* end = nullptr;
  const double x = strtod_l(tok, &end, c_loc);
  if (end != tok + len) return false;
  if (x == std::numeric_limits<double>::infinity() || x == -std::numeric_limits<double>::infinity())
    return false;
  v = x;
  p = q;
  return true;
}

std::string lower(std::string s) {
  for (auto& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

// `ss >> a >> b >> ...` for strings: whitespace-separated tokens, "" when absent.
std::vector<std::string> tokens(const char* p, const char* e, int k) {
  std::vector<std::string> t;
  for (int i = 0; i < k; ++i) {
    while (p < e && is_space(*p)) ++p;
    const char* s = p;
    while (p < e && !is_space(*p)) ++p;
    t.emplace_back(s, p);
  }
  return t;
}

struct Entry {
  long long i, j;  // 0-based
  double v;
  long line;
};

struct Chunk {
  const char* b;
  const char* e;
  long first_line = 0;  // line number of the chunk's first line
  long nlines = 0;
  std::vector<Entry> ent;
  double max_abs = 0.0;
  bool failed = false;
  std::string err;  // first failure in this chunk (its lowest line)
};

// One entry line [p, e) (without the newline). Returns false + message on failure.
bool parse_entry(const char* p, const char* e, long long n, bool sym, long line, Entry& out,
                 const std::string& name, std::string& err) {
  long long i = 0, j = 0;
  double v = 0.0;
  if (!(get_int(p, e, i) && get_int(p, e, j) && get_double(p, e, v))) {
    err = name + ":" + std::to_string(line) + ": malformed entry line";
    return false;
  }
  if (i < 1 || i > n || j < 1 || j > n) {
    err = name + ":" + std::to_string(line) + ": index (" + std::to_string(i) + ", " +
          std::to_string(j) + ") out of range for 1-based indices in [1, " + std::to_string(n) +
          "]";
    return false;
  }
  if (sym && j > i) {
    err = name + ":" + std::to_string(line) + ": upper-triangle entry in a symmetric file";
    return false;
  }
  out = {i - 1, j - 1, v, line};
  return true;
}

// Symmetrised triplets -> CSR (from_triplets, linop.cpp:80-109): row histogram,
// per-row column sort, first duplicate in (i, j) order is an error.
void build_csr(long long n, const std::vector<std::tuple<long long, long long, double>>& t,
               pcgx_csr_host* out, const std::string& name) {
  std::vector<int64_t> rp((size_t)n + 1, 0);
  for (const auto& x : t) ++rp[(size_t)std::get<0>(x) + 1];
  for (long long i = 0; i < n; ++i) rp[(size_t)i + 1] += rp[(size_t)i];
  const size_t nnz = t.size();
  std::vector<int64_t> ci(nnz);
  std::vector<double> va(nnz);
  {
    std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
    for (const auto& x : t) {
      const size_t k = (size_t)pos[(size_t)std::get<0>(x)]++;
      ci[k] = std::get<1>(x);
      va[k] = std::get<2>(x);
    }
  }
  long long dup_row = -1, dup_col = -1;
#pragma omp parallel
  {
    std::vector<std::pair<int64_t, double>> tmp;
    long long my_row = -1, my_col = -1;
#pragma omp for schedule(dynamic, 4096)
    for (long long i = 0; i < n; ++i) {
      const size_t a = (size_t)rp[(size_t)i], b = (size_t)rp[(size_t)i + 1];
      bool sorted = true;
      for (size_t k = a + 1; k < b && sorted; ++k) sorted = ci[k - 1] < ci[k];
      if (!sorted) {
        tmp.clear();
        for (size_t k = a; k < b; ++k) tmp.emplace_back(ci[k], va[k]);
        std::stable_sort(tmp.begin(), tmp.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        for (size_t k = a; k < b; ++k) {
          ci[k] = tmp[k - a].first;
          va[k] = tmp[k - a].second;
        }
      }
      for (size_t k = a + 1; k < b; ++k)
        if (ci[k] == ci[k - 1]) {
          if (my_row < 0 || i < my_row) {
            my_row = i;
            my_col = ci[k];
          }
          break;
        }
    }
#pragma omp critical
    if (my_row >= 0 && (dup_row < 0 || my_row < dup_row)) {
      dup_row = my_row;
      dup_col = my_col;
    }
  }
  if (dup_row >= 0)
    throw ParseFail{name + ": from_triplets: duplicate entry at (" + std::to_string(dup_row) +
                    ", " + std::to_string(dup_col) + ")"};
  out->n = n;
  out->nnz = (int64_t)nnz;
  out->row_ptr = (int64_t*)std::malloc(sizeof(int64_t) * rp.size());
  out->col_idx = (int64_t*)std::malloc(sizeof(int64_t) * std::max<size_t>(nnz, 1));
  out->values = (double*)std::malloc(sizeof(double) * std::max<size_t>(nnz, 1));
  if (!out->row_ptr || !out->col_idx || !out->values) throw ParseFail{name + ": out of memory"};
  std::memcpy(out->row_ptr, rp.data(), sizeof(int64_t) * rp.size());
  if (nnz) {
    std::memcpy(out->col_idx, ci.data(), sizeof(int64_t) * nnz);
    std::memcpy(out->values, va.data(), sizeof(double) * nnz);
  }
}

void load_text(const char* text, size_t len, const std::string& name, pcgx_csr_host* out) {
  const char* const E = text + len;
  const char* p = text;
  long lineno = 0;
  // getline: the next line [ls, le) and p past its '\n'; false at end of input
  auto next_line = [&](const char*& ls, const char*& le) -> bool {
    if (p >= E) return false;
    ls = p;
    const char* nl = (const char*)std::memchr(p, '\n', (size_t)(E - p));
    le = nl ? nl : E;
    p = nl ? nl + 1 : E;
    ++lineno;
    return true;
  };
  const char *ls = nullptr, *le = nullptr;
  if (!next_line(ls, le)) fail_at(name, 1, "empty file");
  bool sym = false;
  {
    const auto t = tokens(ls, le, 5);
    if (t[0] != "%%MatrixMarket") fail_at(name, 1, "missing %%MatrixMarket banner");
    if (lower(t[1]) != "matrix" || lower(t[2]) != "coordinate")
      fail_at(name, 1, "only 'matrix coordinate' files are supported");
    if (lower(t[3]) != "real") fail_at(name, 1, "only 'real' entries are supported");
    const std::string s = lower(t[4]);
    if (s == "symmetric") sym = true;
    else if (s != "general")
      fail_at(name, 1, "unsupported symmetry '" + t[4] + "' (need symmetric or general)");
  }
  long long rows = 0, cols = 0, declared = 0;
  while (next_line(ls, le)) {
    if (le == ls || *ls == '%') continue;
    const char* q = ls;
    if (!(get_int(q, le, rows) && get_int(q, le, cols) && get_int(q, le, declared)))
      fail_at(name, lineno, "malformed size line");
    break;
  }
  if (rows == 0 && cols == 0) fail_at(name, lineno, "missing size line");
  if (rows != cols)
    fail_at(name, lineno,
            "matrix must be square, got " + std::to_string(rows) + "x" + std::to_string(cols));
  const long long n = rows;

  // ---- entries: parallel over line-aligned chunks
  const char* body = p;
  const long body_line0 = lineno + 1;
  const int T = std::max(1, std::min(omp_get_max_threads(), (int)((E - body) / (1 << 20)) + 1));
  std::vector<Chunk> ch((size_t)T);
  {
    const size_t blen = (size_t)(E - body);
    const char* s = body;
    for (int c = 0; c < T; ++c) {
      const char* e = (c == T - 1) ? E : body + blen * (size_t)(c + 1) / (size_t)T;
      if (e < s) e = s;
      if (c < T - 1 && e < E) {  // extend to the end of the line
        const char* nl = (const char*)std::memchr(e, '\n', (size_t)(E - e));
        e = nl ? nl + 1 : E;
      }
      ch[(size_t)c].b = s;
      ch[(size_t)c].e = e;
      s = e;
    }
  }
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int c = 0; c < T; ++c) {
    Chunk& k = ch[(size_t)c];
    long cnt = 0;
    for (const char* q = k.b; q < k.e;) {
      const char* nl = (const char*)std::memchr(q, '\n', (size_t)(k.e - q));
      ++cnt;
      q = nl ? nl + 1 : k.e;
    }
    k.nlines = cnt;
  }
  long acc = body_line0;
  for (auto& k : ch) {
    k.first_line = acc;
    acc += k.nlines;
  }
#pragma omp parallel for num_threads(T) schedule(static, 1)
  for (int c = 0; c < T; ++c) {
    Chunk& k = ch[(size_t)c];
    long line = k.first_line;
    k.ent.reserve((size_t)(k.e - k.b) / 24 + 1);
    for (const char* q = k.b; q < k.e; ++line) {
      const char* nl = (const char*)std::memchr(q, '\n', (size_t)(k.e - q));
      const char* l_end = nl ? nl : k.e;
      if (l_end != q && *q != '%') {
        Entry en;
        if (!parse_entry(q, l_end, n, sym, line, en, name, k.err)) {
          k.failed = true;
          break;
        }
        k.ent.push_back(en);
        k.max_abs = std::max(k.max_abs, std::abs(en.v));
      }
      q = nl ? nl + 1 : k.e;
    }
  }
  for (auto& k : ch)
    if (k.failed) throw ParseFail{k.err};
  lineno = acc - 1;  // lines read in total
  size_t seen = 0;
  double max_abs = 0.0;
  for (auto& k : ch) {
    seen += k.ent.size();
    max_abs = std::max(max_abs, k.max_abs);
  }
  if ((long long)seen != declared)
    fail_at(name, lineno,
            "entry count " + std::to_string(seen) + " does not match declared " + std::to_string(declared));
  std::vector<Entry> ent;
  ent.reserve(seen);
  for (auto& k : ch) {
    ent.insert(ent.end(), k.ent.begin(), k.ent.end());
    std::vector<Entry>().swap(k.ent);
  }

  const double tol = 1e-12 * max_abs;
  std::vector<std::tuple<long long, long long, double>> t;
  t.reserve(ent.size() * 2);
  if (sym) {
    for (const auto& e : ent) {
      t.emplace_back(e.i, e.j, e.v);
      if (e.i != e.j) t.emplace_back(e.j, e.i, e.v);
    }
  } else {
    // general file with symmetric content: pair each off-diagonal entry with its
    // mirror (sorted by (max, min, row)), the lower-triangle value is stored
    std::sort(ent.begin(), ent.end(), [](const Entry& a, const Entry& b) {
      const long long la = std::max(a.i, a.j), sa = std::min(a.i, a.j);
      const long long lb = std::max(b.i, b.j), sb = std::min(b.i, b.j);
      return std::tie(la, sa, a.i) < std::tie(lb, sb, b.i);
    });
    size_t k = 0;
    while (k < ent.size()) {
      const Entry& e = ent[k];
      if (e.i == e.j) {
        t.emplace_back(e.i, e.j, e.v);
        ++k;
        continue;
      }
      const bool mirror = k + 1 < ent.size() &&
                          std::min(ent[k + 1].i, ent[k + 1].j) == std::min(e.i, e.j) &&
                          std::max(ent[k + 1].i, ent[k + 1].j) == std::max(e.i, e.j);
      if (!mirror) {
        if (std::abs(e.v) > tol)
          fail_at(name, e.line, "entry (" + std::to_string(e.i + 1) + ", " + std::to_string(e.j + 1) +
                                    ") has no symmetric counterpart");
        t.emplace_back(e.i, e.j, e.v);
        t.emplace_back(e.j, e.i, e.v);
        ++k;
        continue;
      }
      const Entry& f = ent[k + 1];
      if (std::abs(e.v - f.v) > tol)
        fail_at(name, f.line, "asymmetric pair at (" + std::to_string(e.i + 1) + ", " +
                                  std::to_string(e.j + 1) + "): " + std::to_string(e.v) + " vs " +
                                  std::to_string(f.v));
      const double v = e.i > e.j ? e.v : f.v;
      t.emplace_back(e.i, e.j, v);
      t.emplace_back(e.j, e.i, v);
      k += 2;
    }
  }
  std::vector<Entry>().swap(ent);
  if (n < 0) throw ParseFail{name + ": CsrMatrix: row_ptr must have length n+1 and start at 0"};
  build_csr(n, t, out, name);
}

}  // namespace

int mm_load_text(const char* text, size_t len, const char* name, pcgx_csr_host* out,
                 std::string* msg) {
  std::memset(out, 0, sizeof *out);
  try {
    load_text(text, len, name ? name : "<stream>", out);
    return 0;
  } catch (const ParseFail& f) {
    *msg = f.msg;
    return PCGX_ERR_PARSE;
  } catch (const std::bad_alloc&) {
    *msg = std::string(name ? name : "<stream>") + ": out of memory";
    return PCGX_ERR_PARSE;
  }
}

int mm_load(const char* path, pcgx_csr_host* out, std::string* msg) {
  std::memset(out, 0, sizeof *out);
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    *msg = std::string(path) + ": cannot open file";
    return PCGX_ERR_PARSE;
  }
  std::vector<char> buf;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long sz = std::ftell(f);
    if (sz > 0) buf.resize((size_t)sz);
    std::fseek(f, 0, SEEK_SET);
  }
  const size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), f);
  std::fclose(f);
  buf.resize(got);
  return mm_load_text(buf.data(), buf.size(), path, out, msg);
}

// save_matrix_market (matrix_market.cpp:178-199): the lower triangle, "%.16e".
int mm_save_text(int64_t n, const int64_t* rp, const int64_t* ci, const double* va,
                 std::string* text) {
  std::vector<std::string> parts;
  const int T = std::max(1, omp_get_max_threads());
  parts.resize((size_t)T);
  std::vector<int64_t> cnt((size_t)T, 0);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    const int64_t r0 = n * t / T, r1 = n * (t + 1) / T;
    std::string& s = parts[(size_t)t];
    char buf[96];
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        if (ci[k] > i) continue;
        char vb[64];
        std::snprintf(vb, sizeof vb, "%.16e", va[k]);
        const int w = std::snprintf(buf, sizeof buf, "%lld %lld %s\n", (long long)(i + 1),
                                    (long long)(ci[k] + 1), vb);
        s.append(buf, (size_t)w);
        ++cnt[(size_t)t];
      }
  }
  int64_t nnz_lower = 0;
  for (auto c : cnt) nnz_lower += c;
  *text = "%%MatrixMarket matrix coordinate real symmetric\n" + std::to_string(n) + " " +
          std::to_string(n) + " " + std::to_string(nnz_lower) + "\n";
  size_t tot = text->size();
  for (auto& s : parts) tot += s.size();
  text->reserve(tot);
  for (auto& s : parts) text->append(s);
  return 0;
}

}  // namespace pcgx
