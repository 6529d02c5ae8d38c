// lg_load.cu -- graph file ingest in C++: the text edge-list and Matrix
// Market coordinate formats of graphs.py:126-247 (_parse_edge_list,
// _parse_matrix_market, _merge_triples, load_edge_list), with the same
// acceptance rules, the same canonical result (i < j, sorted by (i, j), a
// repeated pair an error unless symmetrize, which keeps the maximum weight)
// and the same error messages and 1-based line numbers.  Host code only: the
// reference's per-line Python loop is the slow part of ingesting C3 / C4
// sized graphs, and this is what feeds build_laplacian.
//
// Number syntax follows Python's int() / float() on the split fields
// (decimal integers with an optional sign; decimal / exponent floats, inf,
// nan); digit-group underscores, which Python also accepts, are not.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lg_common.cuh"

namespace lg {
namespace {

bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && is_space(s[a])) ++a;
  while (b > a && is_space(s[b - 1])) --b;
  return s.substr(a, b - a);
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && is_space(s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !is_space(s[j])) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

// Python repr() of a str (the common cases: quotes and backslashes)
std::string py_repr(const std::string& s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = dq ? '"' : '\'';
  std::string o(1, q);
  for (char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == q) o += std::string("\\") + q;
    else if ((unsigned char)c < 0x20 || c == 0x7f) {
      char buf[8];
      snprintf(buf, sizeof buf, "\\x%02x", (unsigned char)c);
      o += buf;
    } else o += c;
  }
  o += q;
  return o;
}

// Python repr() of a float: shortest round-trip digits, fixed notation for
// decimal exponents in [-4, 16), scientific otherwise, ".0" on integers.
std::string py_float(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci = sci.substr(1);
  }
  const size_t epos = sci.find('e');
  std::string mant = sci.substr(0, epos);
  const int e = atoi(sci.c_str() + epos + 1);
  std::string digits;
  for (char c : mant)
    if (c != '.') digits += c;
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  if (e >= -4 && e < 16) {
    std::string o;
    if (e < 0) {
      o = "0." + std::string((size_t)(-e - 1), '0') + digits;
    } else if ((int)digits.size() <= e + 1) {
      o = digits + std::string((size_t)(e + 1 - (int)digits.size()), '0') + ".0";
    } else {
      o = digits.substr(0, (size_t)e + 1) + "." + digits.substr((size_t)e + 1);
    }
    return sign + o;
  }
  std::string o = digits.substr(0, 1);
  if (digits.size() > 1) o += "." + digits.substr(1);
  char eb[16];
  snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', std::abs(e));
  return sign + o + eb;
}

struct Tok {
  const char* p;
  size_t n;
  std::string str() const { return std::string(p, n); }
};

// split [b, e) on whitespace into at most kMax tokens; returns the count
// (kMax + 1 when there are more)
template <int kMax>
int split_fast(const char* b, const char* e, Tok (&t)[kMax]) {
  int c = 0;
  while (b < e) {
    while (b < e && is_space(*b)) ++b;
    const char* q = b;
    while (q < e && !is_space(*q)) ++q;
    if (q > b) {
      if (c == kMax) return kMax + 1;
      t[c++] = {b, (size_t)(q - b)};
    }
    b = q;
  }
  return c;
}

bool parse_int(const char* b, const char* e, int64_t& v) {
  if (b == e) return false;
  if (*b == '+') ++b;
  if (b == e || (*b == '-' && b + 1 == e)) return false;
  for (const char* p = (*b == '-') ? b + 1 : b; p < e; ++p)
    if (*p < '0' || *p > '9') return false;
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}

bool parse_float(const char* b, const char* e, double& v) {
  if (b == e) return false;
  for (const char* p = b; p < e; ++p)
    if (*p == 'x' || *p == 'X' || *p == '(' || *p == '_') return false;   // no hex / nan(...)
  const char* q = (*b == '+') ? b + 1 : b;   // from_chars rejects a leading '+'
  if (q == e || *q == '+' || *q == '-' && q != b) return false;
  auto r = std::from_chars(q, e, v);
  if (r.ec == std::errc() && r.ptr == e) return true;
  if (r.ec == std::errc::result_out_of_range && r.ptr == e) {   // strtod semantics
    char* end = nullptr;
    std::string tmp(b, e);
    v = strtod(tmp.c_str(), &end);
    return end == tmp.c_str() + tmp.size();
  }
  // inf / nan spellings from_chars does not take ("infinity", case)
  std::string tmp(b, e);
  char* end = nullptr;
  v = strtod(tmp.c_str(), &end);
  return end == tmp.c_str() + tmp.size();
}

bool parse_int(const std::string& s, int64_t& v) {
  if (s.empty()) return false;
  const char* b = s.c_str();
  const char* e = b + s.size();
  if (*b == '+') ++b;
  if (b == e) return false;
  for (const char* p = (*b == '-') ? b + 1 : b; p < e; ++p)
    if (*p < '0' || *p > '9') return false;
  if (*b == '-' && b + 1 == e) return false;
  auto r = std::from_chars(b, e, v);
  return r.ec == std::errc() && r.ptr == e;
}

bool parse_float(const std::string& s, double& v) {
  if (s.empty()) return false;
  for (char c : s)
    if (c == 'x' || c == 'X' || c == '(' || c == '_') return false;   // no hex / nan(...)
  char* end = nullptr;
  v = strtod(s.c_str(), &end);
  return end == s.c_str() + s.size();
}

struct ParseError {
  std::string msg;
  int64_t line;   // 0: no line
};

struct Raw {
  std::vector<int64_t> a, b, line;
  std::vector<double> w;
};

// _merge_triples: canonical (lo, hi) order (stable in file order), repeated
// pairs an error without symmetrize, maximum weight with it.  Writes at most
// m entries into I / J / W and returns the count through mo.
bool merge(const Raw& raw, bool sym, int64_t* I, int64_t* J, double* W, int64_t& mo,
           ParseError& err) {
  const int64_t m = (int64_t)raw.a.size();
  auto lo = [&](int64_t k) { return std::min(raw.a[(size_t)k], raw.b[(size_t)k]); };
  auto hi = [&](int64_t k) { return std::max(raw.a[(size_t)k], raw.b[(size_t)k]); };
  bool sorted = true;   // canonical files skip the sort
  for (int64_t k = 1; k < m && sorted; ++k) {
    const int64_t l0 = lo(k - 1), l1 = lo(k);
    sorted = l0 < l1 || (l0 == l1 && hi(k - 1) <= hi(k));
  }
  std::vector<int64_t> ord;
  if (!sorted) {
    ord.resize((size_t)m);
    for (int64_t k = 0; k < m; ++k) ord[(size_t)k] = k;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
      const int64_t lx = lo(x), ly = lo(y);
      return lx != ly ? lx < ly : hi(x) < hi(y);
    });
  }
  int64_t o = 0;
  for (int64_t t = 0; t < m; ++t) {
    const int64_t k = sorted ? t : ord[(size_t)t];
    const int64_t l = lo(k), h = hi(k);
    if (o && l == I[o - 1] && h == J[o - 1]) {
      if (!sym) {
        err = {"duplicate edge (" + std::to_string(l) + ", " + std::to_string(h) +
                   "); pass symmetrize to merge",
               raw.line[(size_t)k]};
        return false;
      }
      W[o - 1] = std::max(W[o - 1], raw.w[(size_t)k]);   // np.maximum.at
      continue;
    }
    I[o] = l;
    J[o] = h;
    W[o] = raw.w[(size_t)k];
    ++o;
  }
  mo = o;
  return true;
}

template <typename F>
void for_lines(const char* text, int64_t len, F&& f) {
  int64_t p = 0, lineno = 0;
  while (p < len) {
    int64_t q = p;
    while (q < len && text[q] != '\n') ++q;
    ++lineno;
    if (!f(std::string(text + p, (size_t)(q - p)), lineno)) return;
    p = q + 1;
  }
}

// Edge lines of [p, end) (after the node-count line): appended to raw with
// line numbers counted from line0; false with err at the first bad line.
bool parse_edges(const char* p, const char* end, int64_t n, int64_t line0, Raw& raw,
                 ParseError& err, int64_t& nlines) {
  int64_t lineno = line0;
  while (p < end) {
    const char* q = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    if (!q) q = end;
    ++lineno;
    const char* h = static_cast<const char*>(memchr(p, '#', (size_t)(q - p)));
    const char* b = p;
    const char* e = h ? h : q;
    while (b < e && is_space(*b)) ++b;
    while (e > b && is_space(e[-1])) --e;
    p = q + 1;
    if (b == e) continue;
    Tok f[3];
    const int nf = split_fast<3>(b, e, f);
    if (nf != 3) {
      err = {"expected 'i j w', got " + py_repr(std::string(b, e)), lineno};
      return false;
    }
    int64_t a, c;
    double w;
    if (!parse_int(f[0].p, f[0].p + f[0].n, a) || !parse_int(f[1].p, f[1].p + f[1].n, c) ||
        !parse_float(f[2].p, f[2].p + f[2].n, w)) {
      err = {"could not parse edge " + py_repr(std::string(b, e)), lineno};
      return false;
    }
    if (!(0 <= a && a < n && 0 <= c && c < n)) {
      err = {"node index out of range in " + py_repr(std::string(b, e)), lineno};
      return false;
    }
    if (a == c) {
      err = {"self-loop at node " + std::to_string(a), lineno};
      return false;
    }
    if (!(w > 0)) {
      err = {"nonpositive weight " + py_float(w), lineno};
      return false;
    }
    raw.a.push_back(a);
    raw.b.push_back(c);
    raw.w.push_back(w);
    raw.line.push_back(lineno);
  }
  nlines = lineno - line0;
  return true;
}

bool parse_edgelist(const char* text, int64_t len, int64_t& n, Raw& raw, ParseError& err) {
  n = -1;
  const char* p = text;
  const char* end = text + len;
  int64_t lineno = 0;
  // the node count: first line with content
  while (p < end && n < 0) {
    const char* q = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    if (!q) q = end;
    ++lineno;
    const char* h = static_cast<const char*>(memchr(p, '#', (size_t)(q - p)));
    const char* b = p;
    const char* e = h ? h : q;
    while (b < e && is_space(*b)) ++b;
    while (e > b && is_space(e[-1])) --e;
    p = q + 1;
    if (b == e) continue;
    Tok f[1];
    if (split_fast<1>(b, e, f) != 1) {
      err = {"expected a single node count on the first line", lineno};
      return false;
    }
    int64_t v;
    if (!parse_int(f[0].p, f[0].p + f[0].n, v)) {
      err = {"bad node count " + py_repr(f[0].str()), lineno};
      return false;
    }
    if (v < 1) {
      err = {"node count must be positive", lineno};
      return false;
    }
    n = v;
  }
  if (n < 0) {
    err = {"empty input, no node count found", 0};
    return false;
  }
  if (p >= end) return true;
  // edge lines in parallel chunks cut at newlines; the first error in file
  // order wins, line numbers from per-chunk line counts
  const int64_t rest = end - p;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(64, rest / (1 << 20)));
  std::vector<const char*> cut((size_t)nt + 1);
  cut[0] = p;
  cut[(size_t)nt] = end;
  for (int t = 1; t < nt; ++t) {
    const char* c = p + rest * t / nt;
    if (c < cut[(size_t)t - 1]) c = cut[(size_t)t - 1];
    const char* q = static_cast<const char*>(memchr(c, '\n', (size_t)(end - c)));
    cut[(size_t)t] = q ? q + 1 : end;
  }
  std::vector<Raw> part((size_t)nt);
  std::vector<ParseError> perr((size_t)nt, ParseError{"", 0});
  std::vector<char> bad((size_t)nt, 0);
  std::vector<int64_t> lines((size_t)nt, 0);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < nt; ++t) {
    // line numbers local to the chunk (0-based start); fixed up below
    int64_t cnt = 0;
    for (const char* c = cut[(size_t)t]; c < cut[(size_t)t + 1];) {
      const char* q = static_cast<const char*>(memchr(c, '\n', (size_t)(cut[(size_t)t + 1] - c)));
      ++cnt;
      c = q ? q + 1 : cut[(size_t)t + 1];
    }
    lines[(size_t)t] = cnt;
    int64_t used = 0;
    bad[(size_t)t] = !parse_edges(cut[(size_t)t], cut[(size_t)t + 1], n, 0, part[(size_t)t],
                                  perr[(size_t)t], used);
  }
  int64_t off = lineno;
  size_t total = 0;
  for (int t = 0; t < nt; ++t) {
    if (bad[(size_t)t]) {
      err = perr[(size_t)t];
      err.line += off;
      // messages carry no line numbers, so the offset only moves the line field
      return false;
    }
    for (int64_t& l : part[(size_t)t].line) l += off;
    off += lines[(size_t)t];
    total += part[(size_t)t].a.size();
  }
  raw.a.reserve(total);
  raw.b.reserve(total);
  raw.w.reserve(total);
  raw.line.reserve(total);
  for (int t = 0; t < nt; ++t) {
    Raw& r = part[(size_t)t];
    raw.a.insert(raw.a.end(), r.a.begin(), r.a.end());
    raw.b.insert(raw.b.end(), r.b.begin(), r.b.end());
    raw.w.insert(raw.w.end(), r.w.begin(), r.w.end());
    raw.line.insert(raw.line.end(), r.line.begin(), r.line.end());
  }
  return true;
}

bool parse_mtx(const char* text, int64_t len, int64_t& n, Raw& raw, ParseError& err) {
  n = -1;
  bool ok = true, have_header = false, pattern = false, have_size = false;
  int64_t rows = 0, nnz = 0, count = 0;
  for_lines(text, len, [&](const std::string& line, int64_t lineno) {
    if (!have_header) {
      const std::string h = strip(line);
      if (h.empty() || h.rfind("%%MatrixMarket", 0) != 0) {
        err = {"missing %%MatrixMarket header", 1};
        return ok = false;
      }
      std::string lower = h;
      for (char& c : lower) c = (char)tolower((unsigned char)c);
      const std::vector<std::string> tk = split_ws(lower);
      if (tk.size() != 5 || tk[1] != "matrix" || tk[2] != "coordinate") {
        err = {"unsupported header " + py_repr(h), 1};
        return ok = false;
      }
      if (tk[3] != "real" && tk[3] != "integer" && tk[3] != "pattern") {
        err = {"unsupported field type " + py_repr(tk[3]), 1};
        return ok = false;
      }
      if (tk[4] != "symmetric" && tk[4] != "general") {
        err = {"unsupported symmetry " + py_repr(tk[4]), 1};
        return ok = false;
      }
      pattern = tk[3] == "pattern";
      have_header = true;
      return true;
    }
    const std::string t = strip(line);
    if (t.empty() || t[0] == '%') return true;
    const std::vector<std::string> f = split_ws(t);
    if (!have_size) {
      if (f.size() != 3) {
        err = {"expected 'rows cols nnz'", lineno};
        return ok = false;
      }
      int64_t r, c, z;
      if (!parse_int(f[0], r) || !parse_int(f[1], c) || !parse_int(f[2], z)) {
        err = {"bad size line " + py_repr(t), lineno};
        return ok = false;
      }
      if (r != c) {
        err = {"matrix is " + std::to_string(r) + "x" + std::to_string(c) + ", not square",
               lineno};
        return ok = false;
      }
      if (r < 1) {
        err = {"matrix must have at least one row", lineno};
        return ok = false;
      }
      rows = r;
      nnz = z;
      have_size = true;
      return true;
    }
    const size_t want = pattern ? 2 : 3;
    if (f.size() != want) {
      err = {"expected " + std::to_string(want) + " fields, got " + py_repr(t), lineno};
      return ok = false;
    }
    int64_t a, b;
    double w = 1.0;
    if (!parse_int(f[0], a) || !parse_int(f[1], b) || (!pattern && !parse_float(f[2], w))) {
      err = {"could not parse entry " + py_repr(t), lineno};
      return ok = false;
    }
    ++count;
    if (!(1 <= a && a <= rows && 1 <= b && b <= rows)) {
      err = {"index out of range in " + py_repr(t), lineno};
      return ok = false;
    }
    if (a == b) return true;   // an adjacency-style diagonal carries no edge
    w = std::fabs(w);
    if (w == 0.0) {
      err = {"explicit zero off-diagonal entry", lineno};
      return ok = false;
    }
    raw.a.push_back(a - 1);
    raw.b.push_back(b - 1);
    raw.w.push_back(w);
    raw.line.push_back(lineno);
    return true;
  });
  if (!ok) return false;
  if (!have_header) {
    err = {"missing %%MatrixMarket header", 1};
    return false;
  }
  if (!have_size) {
    err = {"missing size line", 0};
    return false;
  }
  if (count != nnz) {
    err = {"header promised " + std::to_string(nnz) + " entries, found " +
               std::to_string(count),
           0};
    return false;
  }
  n = rows;
  return true;
}

thread_local int64_t g_err_line = 0;

}  // namespace
}  // namespace lg

using namespace lg;

extern "C" {

int lg_graph_parse(const char* text, int64_t len, int format, int symmetrize, int64_t* n_out,
                   int64_t* m_out, int64_t** i_out, int64_t** j_out, double** w_out,
                   int64_t* err_line) {
  if ((!text && len > 0) || len < 0 || !n_out || !m_out || !i_out || !j_out || !w_out)
    return fail(LG_EINVAL, "lg_graph_parse: bad argument");
  if (format != 0 && format != 1) return fail(LG_EINVAL, "lg_graph_parse: unknown format");
  if (err_line) *err_line = 0;
  Raw raw;
  ParseError err{"", 0};
  int64_t n = 0;
  const bool ok = format == 0 ? parse_edgelist(text, len, n, raw, err)
                              : parse_mtx(text, len, n, raw, err);
  if (!ok) {
    if (err_line) *err_line = err.line;
    return fail(LG_EFORMAT, err.msg);
  }
  const int64_t mr = (int64_t)raw.a.size();
  int64_t* ib = (int64_t*)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(mr, 1));
  int64_t* jb = (int64_t*)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(mr, 1));
  double* wb = (double*)malloc(sizeof(double) * (size_t)std::max<int64_t>(mr, 1));
  if (!ib || !jb || !wb) {
    free(ib);
    free(jb);
    free(wb);
    return fail(LG_ENOMEM, "lg_graph_parse: out of host memory");
  }
  int64_t m = 0;
  if (mr && !merge(raw, symmetrize != 0, ib, jb, wb, m, err)) {
    free(ib);
    free(jb);
    free(wb);
    if (err_line) *err_line = err.line;
    return fail(LG_EFORMAT, err.msg);
  }
  *n_out = n;
  *m_out = m;
  *i_out = ib;
  *j_out = jb;
  *w_out = wb;
  return LG_OK;
}

int lg_host_free(void* p) {
  free(p);
  return LG_OK;
}

}  // extern "C"
