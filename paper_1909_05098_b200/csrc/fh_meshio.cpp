// fh_meshio.cpp -- host-side mesh ingest and text output.
//
// * fh_mesh_parse: the reference's mesh text grammar (mesh.py:153-236
//   parse_mesh_text): the same tokens, the same errors in the same order, with
//   the same 1-based line numbers.  One sequential pass finds the tokens and
//   parses the integers; the coordinate block is then converted by a pool of
//   threads (strtod, correctly rounded like Python's float()).
// * fh_format_f64 / fh_format_i64: rows of numbers as the reference renders
//   them in mesh files, VTK snapshots and probes.csv -- Python repr(float)
//   (shortest round-trip digits, 'r' format rules) and str(int)
//   (mesh.py:241-253, vtkio.py:20-52, cli.py:81-86).
//
// Integer/byte work only: no GPU involvement.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fedheat_b200.h"
#include "fh_internal.h"

namespace {

// ---------------------------------------------------------------- lexing --
// Python str.splitlines() line breaks and str.split() whitespace, for the
// UTF-8 encoding of the text (mesh.py:153-157: lines, '#' comments, split()).
enum : uint8_t { C_TOK = 0, C_WS = 1, C_NL = 2, C_HASH = 3, C_CR = 4, C_UTF = 5 };

struct ClassTable {
  uint8_t c[256];
  ClassTable() {
    for (int i = 0; i < 256; ++i) c[i] = C_TOK;
    c[(int)' '] = C_WS;
    c[(int)'\t'] = C_WS;
    c[0x1f] = C_WS;  // unit separator: whitespace for split(), not a line break
    c[(int)'\n'] = C_NL;
    c[0x0b] = C_NL;
    c[0x0c] = C_NL;
    c[0x1c] = C_NL;
    c[0x1d] = C_NL;
    c[0x1e] = C_NL;
    c[(int)'\r'] = C_CR;
    c[(int)'#'] = C_HASH;
    c[0xc2] = C_UTF;
    c[0xe1] = C_UTF;
    c[0xe2] = C_UTF;
    c[0xe3] = C_UTF;
  }
};
const ClassTable kClass;

// multi-byte UTF-8 separators: returns byte length and sets *nl for line breaks
inline int utf8_sep(const char *p, const char *end, bool *nl) {
  const unsigned char *u = (const unsigned char *)p;
  const int64_t left = end - p;
  *nl = false;
  if (u[0] == 0xc2 && left >= 2) {
    if (u[1] == 0x85) { *nl = true; return 2; }  // NEL
    if (u[1] == 0xa0) return 2;                  // NBSP
    return 0;
  }
  if (left < 3) return 0;
  if (u[0] == 0xe1 && u[1] == 0x9a && u[2] == 0x80) return 3;  // U+1680
  if (u[0] == 0xe2 && u[1] == 0x80) {
    if (u[2] >= 0x80 && u[2] <= 0x8a) return 3;  // U+2000..U+200A
    if (u[2] == 0xa8 || u[2] == 0xa9) { *nl = true; return 3; }  // U+2028/9
    if (u[2] == 0xaf) return 3;                  // U+202F
    return 0;
  }
  if (u[0] == 0xe2 && u[1] == 0x81 && u[2] == 0x9f) return 3;  // U+205F
  if (u[0] == 0xe3 && u[1] == 0x80 && u[2] == 0x80) return 3;  // U+3000
  return 0;
}

struct Lexer {
  const char *p, *end;
  int64_t line = 1;      // line of the scan position
  int64_t tok_line = 0;  // line of the last token returned (TokenStream.line)
  const char *tok = nullptr;
  int64_t tok_len = 0;

  // break at *p: advance past it and count the line
  inline void skip_comment() {
    while (p < end) {
      uint8_t c = kClass.c[(unsigned char)*p];
      if (c == C_NL || c == C_CR) return;
      if (c == C_UTF) {
        bool nl;
        int n = utf8_sep(p, end, &nl);
        if (n && nl) return;
        p += n ? n : 1;
        continue;
      }
      ++p;
    }
  }

  // next token, or false at end of text
  bool next() {
    while (p < end) {
      uint8_t c = kClass.c[(unsigned char)*p];
      if (c == C_TOK) break;
      if (c == C_WS) { ++p; continue; }
      if (c == C_NL) { ++p; ++line; continue; }
      if (c == C_CR) {
        ++p;
        if (p < end && *p == '\n') ++p;
        ++line;
        continue;
      }
      if (c == C_HASH) { skip_comment(); continue; }
      bool nl;
      int n = utf8_sep(p, end, &nl);
      if (!n) break;  // a token starting with a non-ASCII character
      p += n;
      if (nl) ++line;
    }
    if (p >= end) return false;
    tok = p;
    while (p < end) {
      uint8_t c = kClass.c[(unsigned char)*p];
      if (c == C_TOK) { ++p; continue; }
      if (c == C_UTF) {
        bool nl;
        if (utf8_sep(p, end, &nl)) break;
        ++p;
        continue;
      }
      break;
    }
    tok_len = p - tok;
    tok_line = line;
    return true;
  }
};

// Python int(token): [+-]? digit (_? digit)*  (base 10, leading zeros allowed)
inline bool py_int(const char *s, int64_t n, int64_t *out) {
  int64_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  if (i >= n || s[i] < '0' || s[i] > '9') return false;
  unsigned __int128 v = 0;
  bool prev_digit = false;
  for (; i < n; ++i) {
    char ch = s[i];
    if (ch >= '0' && ch <= '9') {
      v = v * 10 + (unsigned)(ch - '0');
      if (v > ((unsigned __int128)1 << 64)) return false;  // beyond int64 (see header note)
      prev_digit = true;
    } else if (ch == '_' && prev_digit && i + 1 < n && s[i + 1] >= '0' && s[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  if (neg) {
    if (v > ((unsigned __int128)1 << 63)) return false;
    *out = (int64_t)(-(__int128)v);
  } else {
    if (v > (unsigned __int128)INT64_MAX) return false;
    *out = (int64_t)v;
  }
  return true;
}

inline bool ieq(const char *s, int64_t n, const char *word) {
  int64_t m = (int64_t)strlen(word);
  if (n != m) return false;
  for (int64_t i = 0; i < n; ++i) {
    char a = s[i];
    if (a >= 'A' && a <= 'Z') a = (char)(a - 'A' + 'a');
    if (a != word[i]) return false;
  }
  return true;
}

// Python float(token): [+-]? (inf|infinity|nan) | [+-]? decimal with single
// underscores between digits, optional exponent.  Correctly rounded (glibc
// strtod on the underscore-free copy).
bool py_float(const char *s, int64_t n, double *out) {
  int64_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  if (ieq(s + i, n - i, "inf") || ieq(s + i, n - i, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(s + i, n - i, "nan")) {
    *out = neg ? -NAN : NAN;
    return true;
  }
  char buf[128];
  std::string big;
  char *dst = buf;
  if (n >= (int64_t)sizeof(buf)) {
    big.resize(n + 1);
    dst = &big[0];
  }
  int64_t k = 0;
  if (neg) dst[k++] = '-';
  // digitpart: digit (_? digit)*
  auto digitpart = [&](int64_t *pos) -> int64_t {
    int64_t cnt = 0;
    while (*pos < n) {
      char ch = s[*pos];
      if (ch >= '0' && ch <= '9') {
        dst[k++] = ch;
        ++cnt;
        ++*pos;
      } else if (ch == '_' && cnt > 0 && *pos + 1 < n && s[*pos + 1] >= '0' && s[*pos + 1] <= '9') {
        ++*pos;
      } else {
        break;
      }
    }
    return cnt;
  };
  int64_t int_digits = digitpart(&i);
  int64_t frac_digits = 0;
  if (i < n && s[i] == '.') {
    dst[k++] = '.';
    ++i;
    frac_digits = digitpart(&i);
  }
  if (int_digits == 0 && frac_digits == 0) return false;
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    dst[k++] = 'e';
    ++i;
    if (i < n && (s[i] == '+' || s[i] == '-')) dst[k++] = s[i++];
    if (digitpart(&i) == 0) return false;
  }
  if (i != n) return false;
  dst[k] = 0;
  *out = strtod(dst, nullptr);
  return true;
}

// Python repr(str) for the token / name quoted in error messages
std::string py_repr(const char *s, int64_t n) {
  bool has_sq = memchr(s, '\'', n) != nullptr, has_dq = memchr(s, '"', n) != nullptr;
  char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string r(1, q);
  for (int64_t i = 0; i < n; ++i) {
    unsigned char ch = (unsigned char)s[i];
    if (ch == (unsigned char)q || ch == '\\') {
      r += '\\';
      r += (char)ch;
    } else if (ch == '\t') {
      r += "\\t";
    } else if (ch == '\n') {
      r += "\\n";
    } else if (ch == '\r') {
      r += "\\r";
    } else if (ch < 0x20 || ch == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", ch);
      r += b;
    } else {
      r += (char)ch;
    }
  }
  r += q;
  return r;
}

bool valid_set_name(const char *s, int64_t n) {  // ^[A-Za-z_][A-Za-z0-9_.-]*$
  if (n == 0) return false;
  auto alpha = [](char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; };
  if (!alpha(s[0])) return false;
  for (int64_t i = 1; i < n; ++i) {
    char c = s[i];
    if (!(alpha(c) || (c >= '0' && c <= '9') || c == '.' || c == '-')) return false;
  }
  return true;
}

int n_workers(int32_t requested) {
  int hw = (int)std::thread::hardware_concurrency();
  if (hw < 1) hw = 1;
  int n = requested > 0 ? requested : hw;
  return std::max(1, std::min(n, 64));
}

}  // namespace

struct fh_mesh_text {
  std::vector<double> nodes;
  std::vector<int64_t> tets, hexes;
  std::vector<std::string> set_names;
  std::vector<std::vector<int64_t>> set_ids;
};

namespace {

struct ParseError {
  std::string msg;
  int64_t line;
};

// coordinates of nodes [lo, hi): tokens re-found from each node's first-token
// offset; the first failing node is reported through *bad (index * 3 + axis).
void convert_nodes(const char *text, const char *end, const std::vector<int64_t> &start, int64_t lo, int64_t hi,
                   double *nodes, int64_t *bad) {
  for (int64_t i = lo; i < hi; ++i) {
    Lexer lx{text + start[i], end};
    for (int ax = 0; ax < 3; ++ax) {
      lx.next();
      if (!py_float(lx.tok, lx.tok_len, &nodes[i * 3 + ax])) {
        *bad = i * 3 + ax;
        return;
      }
    }
  }
}

int parse(const char *text, int64_t len, int32_t n_threads, fh_mesh_text *m, ParseError *err) {
  const char *end = text + len;
  Lexer ts{text, end};
  auto fail = [&](const std::string &msg) {
    err->msg = msg;
    err->line = ts.tok_line;
    return 1;
  };
  auto next = [&](const char *what) -> bool {
    if (ts.next()) return true;
    fail(std::string("unexpected end of file, expected ") + what);
    return false;
  };
  auto next_int = [&](const std::string &what, int64_t *v) -> bool {
    if (!ts.next()) {
      fail("unexpected end of file, expected " + what);
      return false;
    }
    if (!py_int(ts.tok, ts.tok_len, v)) {
      fail("expected integer " + what + ", got " + py_repr(ts.tok, ts.tok_len));
      return false;
    }
    return true;
  };
  auto is = [&](const char *word) {
    return ts.tok_len == (int64_t)strlen(word) && memcmp(ts.tok, word, ts.tok_len) == 0;
  };

  if (!next("'nodes'")) return 1;
  if (!is("nodes")) return fail("expected 'nodes', got " + py_repr(ts.tok, ts.tok_len));
  int64_t n_nodes = 0;
  if (!next_int("node count", &n_nodes)) return 1;
  if (n_nodes <= 0) return fail("node count must be positive");

  // pass 1 over the coordinate block: token boundaries only
  std::vector<int64_t> start((size_t)n_nodes);
  int64_t structural_node = -1;  // node whose coordinates hit the end of the text
  int64_t eof_line = 0;
  for (int64_t i = 0; i < n_nodes && structural_node < 0; ++i) {
    for (int ax = 0; ax < 3; ++ax) {
      if (!ts.next()) {
        structural_node = i;
        eof_line = ts.tok_line;
        break;
      }
      if (ax == 0) start[(size_t)i] = ts.tok - text;
    }
  }
  const int64_t complete = structural_node < 0 ? n_nodes : structural_node;
  m->nodes.assign((size_t)(n_nodes * 3), 0.0);
  // pass 2: conversion, in parallel; the earliest failing token wins
  {
    int nw = n_workers(n_threads);
    if (complete < 4096) nw = 1;
    std::vector<int64_t> bad((size_t)nw, INT64_MAX);
    std::vector<std::thread> pool;
    int64_t per = (complete + nw - 1) / std::max(nw, 1);
    for (int w = 0; w < nw; ++w) {
      int64_t lo = std::min(complete, w * per), hi = std::min(complete, lo + per);
      pool.emplace_back(convert_nodes, text, end, std::cref(start), lo, hi, m->nodes.data(), &bad[(size_t)w]);
    }
    for (auto &t : pool) t.join();
    int64_t first = *std::min_element(bad.begin(), bad.end());
    if (first != INT64_MAX) {
      // redo that node sequentially for the token text and its line number
      int64_t i = first / 3;
      Lexer lx{text, end};
      // line of the node's first token: count line breaks up to its offset
      Lexer counter{text, text + start[(size_t)i]};
      while (counter.next()) {
      }
      lx.p = text + start[(size_t)i];
      lx.line = counter.line;
      for (int ax = 0; ax <= first % 3; ++ax) lx.next();
      err->msg = "expected number coordinate of node " + std::to_string(i) + ", got " + py_repr(lx.tok, lx.tok_len);
      err->line = lx.tok_line;
      return 1;
    }
  }
  if (structural_node >= 0) {
    err->msg = "unexpected end of file, expected coordinate of node " + std::to_string(structural_node);
    err->line = eof_line;
    return 1;
  }

  if (!next("'elements'")) return 1;
  if (!is("elements")) return fail("expected 'elements', got " + py_repr(ts.tok, ts.tok_len));
  int64_t n_elem = 0;
  if (!next_int("element count", &n_elem)) return 1;
  if (n_elem <= 0) return fail("element count must be positive");
  for (int64_t e = 0; e < n_elem; ++e) {
    if (!next("element kind")) return 1;
    int nn;
    std::vector<int64_t> *dst;
    if (is("tet4")) {
      nn = 4;
      dst = &m->tets;
    } else if (is("hex8")) {
      nn = 8;
      dst = &m->hexes;
    } else {
      return fail("unknown element kind " + py_repr(ts.tok, ts.tok_len) + " (expected tet4 or hex8)");
    }
    const std::string what = "node of element " + std::to_string(e);
    for (int a = 0; a < nn; ++a) {
      int64_t v;
      if (!ts.next()) return fail("unexpected end of file, expected " + what);
      if (!py_int(ts.tok, ts.tok_len, &v)) return fail("expected integer " + what + ", got " + py_repr(ts.tok, ts.tok_len));
      dst->push_back(v);
    }
  }

  while (ts.next()) {
    if (!is("nodeset")) return fail("expected 'nodeset' or end of file, got " + py_repr(ts.tok, ts.tok_len));
    if (!next("node-set name")) return 1;
    std::string name(ts.tok, (size_t)ts.tok_len);
    if (!valid_set_name(ts.tok, ts.tok_len)) return fail("invalid node-set name " + py_repr(ts.tok, ts.tok_len));
    const std::string qname = py_repr(name.data(), (int64_t)name.size());
    if (std::find(m->set_names.begin(), m->set_names.end(), name) != m->set_names.end())
      return fail("duplicate node set " + qname);
    int64_t count = 0;
    if (!next_int("node-set size", &count)) return 1;
    if (count < 0) return fail("node-set size must be non-negative");
    std::vector<int64_t> ids((size_t)count);
    const std::string what = "member of set " + qname;
    for (int64_t j = 0; j < count; ++j)
      if (!next_int(what, &ids[(size_t)j])) return 1;
    std::vector<int64_t> srt(ids);
    std::sort(srt.begin(), srt.end());
    if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) return fail("node set " + qname + " repeats a node");
    if (count && (srt.front() < 0 || srt.back() >= n_nodes))
      return fail("node set " + qname + " references a node outside [0, " + std::to_string(n_nodes) + ")");
    m->set_names.push_back(name);
    m->set_ids.push_back(std::move(ids));
  }
  return 0;
}

// ------------------------------------------------------------ formatting --
// Python repr(float): the shortest digit string that round-trips (David Gay's
// mode 0: shortest, then nearest), laid out by float_repr_style 'short':
// exponent form when decpt <= -4 or decpt > 16, else positional with ".0"
// appended to integers (Python/pystrtod.c format_float_short semantics).

typedef unsigned __int128 u128;

const u128 *pow10_table() {
  static u128 t[39];
  static bool init = [] {
    t[0] = 1;
    for (int i = 1; i < 39; ++i) t[i] = t[i - 1] * 10;
    return true;
  }();
  (void)init;
  return t;
}

inline int bits_of(u128 v) {
  const uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
  if (hi) return 128 - __builtin_clzll(hi);
  return lo ? 64 - __builtin_clzll(lo) : 0;
}

// Exact shortest digits with 128-bit integers for x = m * 2^e, e in
// [-69, 0] (about 7.6e-6 <= x < 2^53: temperatures, coordinates, volumes).
// Candidate d * 10^q (q <= 0) round-trips iff
//   |d * 2^(1-e) - 2m * 10^-q| <= 10^-q   (strict when m is odd: ties go to even),
// with the half-size gap below x when m = 2^52 (x a power of two).
// Returns false when the value is outside the range (caller falls back).
bool shortest_fast(double ax, char *digits, int *nd, int *decpt) {
  uint64_t bits;
  memcpy(&bits, &ax, 8);
  const int be = (int)(bits >> 52);
  if (be == 0) return false;  // subnormal
  const uint64_t m = (bits & ((1ull << 52) - 1)) | (1ull << 52);
  const int e = be - 1075;
  if (e > 0 || e < -69) return false;
  const int sh = -e;  // x = m / 2^sh
  const u128 *P = pow10_table();
  const bool pow2 = m == (1ull << 52) && be > 1;
  const bool even = (m & 1) == 0;
  int k = (int)std::floor(std::log10(ax));  // estimate of the decimal exponent
  // nearest p-digit candidate: returns d and q, d in [10^(p-1), 10^p] (10^p after a carry)
  auto nearest = [&](int p, u128 *d_out, int *q_out) -> bool {
    int q = k - p + 1;
    for (int iter = 0; iter < 4; ++iter) {
      if (q > 0 || -q > 38) return false;
      const u128 scale = P[-q];
      if (bits_of(scale) + 54 > 127) return false;
      const u128 num = (u128)m * scale;  // x * 10^-q = num / 2^sh
      const u128 t = num >> sh;
      if (t >= P[p]) { ++q; continue; }
      if (t < P[p - 1]) { --q; continue; }
      const u128 rem = num - (t << sh);
      const u128 half = (u128)1 << (sh - 1 < 0 ? 0 : sh - 1);
      u128 d = t;
      if (sh > 0 && (rem > half || (rem == half && (t & 1)))) d = t + 1;
      *d_out = d;
      *q_out = q;
      return true;
    }
    return false;
  };
  // does d * 10^q round-trip to x?
  auto roundtrips = [&](u128 d, int q) -> bool {
    const u128 scale = P[-q];
    if (bits_of(d) + sh + 1 > 127) return false;
    const u128 a = d << (sh + 1);
    const u128 b = ((u128)m * scale) << 1;
    if (a >= b) {
      const u128 diff = a - b;
      return even ? diff <= scale : diff < scale;
    }
    const u128 diff = b - a;
    if (pow2) {  // gap below x is half as large: |.| <= 10^-q / 2
      const u128 lim = scale;  // compare 2*diff with scale
      return even ? (diff << 1) <= lim : (diff << 1) < lim;
    }
    return even ? diff <= scale : diff < scale;
  };
  u128 best_d = 0;
  int best_q = 0;
  bool found = false;
  if (!pow2) {
    int lo = 1, hi = 17;
    u128 d;
    int q;
    if (!nearest(17, &d, &q) || !roundtrips(d, q)) return false;
    best_d = d;
    best_q = q;
    found = true;
    while (lo < hi) {
      int mid = (lo + hi) / 2;
      if (!nearest(mid, &d, &q)) return false;
      if (roundtrips(d, q)) {
        hi = mid;
        best_d = d;
        best_q = q;
      } else {
        lo = mid + 1;
      }
    }
    if (lo == 17) {
      if (!nearest(17, &best_d, &best_q)) return false;
    }
  } else {
    for (int p = 1; p <= 17 && !found; ++p) {
      u128 d;
      int q;
      if (!nearest(p, &d, &q)) return false;
      if (roundtrips(d, q)) {
        best_d = d;
        best_q = q;
        found = true;
      } else if (roundtrips(d + 1, q)) {
        best_d = d + 1;
        best_q = q;
        found = true;
      }
    }
  }
  if (!found) return false;
  char tmp[48];
  int n = 0;
  uint64_t v = (uint64_t)best_d;  // at most 10^17 < 2^64
  do {
    tmp[n++] = (char)('0' + (int)(v % 10));
    v /= 10;
  } while (v);
  *decpt = n + best_q;
  int len = n;
  for (int i = 0; i < n; ++i) digits[i] = tmp[n - 1 - i];
  while (len > 1 && digits[len - 1] == '0') --len;
  *nd = len;
  return true;
}

// the general path: glibc's correctly rounded %.*e and strtod
void shortest_slow(double ax, char *digits, int *nd_out, int *decpt) {
  char buf[40];
  int nd = 0;
  int exp10 = 0;
  // smallest precision whose correctly rounded value round-trips (monotone in p)
  int lo = 1, hi = 17;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    snprintf(buf, sizeof buf, "%.*e", mid - 1, ax);
    if (strtod(buf, nullptr) == ax) hi = mid;
    else lo = mid + 1;
  }
  int p = lo;
  snprintf(buf, sizeof buf, "%.*e", p - 1, ax);
  // at a power of two the round-trip interval is asymmetric: a shorter string
  // one decimal step above the nearest one can round-trip when the nearest
  // does not
  {
    uint64_t bits;
    memcpy(&bits, &ax, 8);
    if ((bits & ((1ull << 52) - 1)) == 0) {
      for (int q = 1; q < p; ++q) {
        char cand[40];
        snprintf(cand, sizeof cand, "%.*e", q - 1, ax);
        // the next q-digit decimal above the nearest one
        char *e = strchr(cand, 'e');
        int ex = atoi(e + 1);
        std::string mant;
        for (char *c = cand; c < e; ++c)
          if (*c != '.') mant += *c;
        // increment the decimal mantissa
        int i = (int)mant.size() - 1;
        while (i >= 0 && mant[(size_t)i] == '9') mant[(size_t)i--] = '0';
        if (i < 0) {
          mant.insert(mant.begin(), '1');
          mant.pop_back();
          ++ex;
        } else {
          mant[(size_t)i]++;
        }
        std::string s = mant.substr(0, 1) + (mant.size() > 1 ? "." + mant.substr(1) : "") + "e" + std::to_string(ex);
        if (strtod(s.c_str(), nullptr) == ax) {
          snprintf(buf, sizeof buf, "%s", s.c_str());
          p = q;
          break;
        }
      }
    }
  }
  // buf = d[.ddd]e[+-]x
  {
    char *e = strchr(buf, 'e');
    exp10 = atoi(e + 1);
    for (char *c = buf; c < e; ++c)
      if (*c != '.') digits[nd++] = *c;
    while (nd > 1 && digits[nd - 1] == '0') --nd;  // shortest form has no trailing zeros
  }
  *decpt = exp10 + 1;
  *nd_out = nd;
}

int repr_f64(double x, char *out) {
  if (std::isnan(x)) {
    memcpy(out, "nan", 3);
    return 3;
  }
  char *o = out;
  if (std::signbit(x)) *o++ = '-';
  double ax = std::fabs(x);
  if (std::isinf(ax)) {
    memcpy(o, "inf", 3);
    return (int)(o - out) + 3;
  }
  if (ax == 0.0) {
    memcpy(o, "0.0", 3);
    return (int)(o - out) + 3;
  }
  char digits[48];
  int nd = 0, decpt = 0;
  if (!shortest_fast(ax, digits, &nd, &decpt)) shortest_slow(ax, digits, &nd, &decpt);
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      memcpy(o, digits + 1, (size_t)(nd - 1));
      o += nd - 1;
    }
    int ex = decpt - 1;
    o += snprintf(o, 8, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int i = 0; i < -decpt; ++i) *o++ = '0';
    memcpy(o, digits, (size_t)nd);
    o += nd;
  } else if (decpt >= nd) {
    memcpy(o, digits, (size_t)nd);
    o += nd;
    for (int i = nd; i < decpt; ++i) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    memcpy(o, digits, (size_t)decpt);
    o += decpt;
    *o++ = '.';
    memcpy(o, digits + decpt, (size_t)(nd - decpt));
    o += nd - decpt;
  }
  return (int)(o - out);
}

int str_i64(int64_t v, char *out) {
  char tmp[24];
  int n = 0;
  bool neg = v < 0;
  uint64_t u = neg ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
  do {
    tmp[n++] = (char)('0' + u % 10);
    u /= 10;
  } while (u);
  int k = 0;
  if (neg) out[k++] = '-';
  while (n) out[k++] = tmp[--n];
  return k;
}

constexpr int kMaxF64 = 25;  // "-1.2345678901234567e-308"
constexpr int kMaxI64 = 20;

template <typename T, typename Fmt>
int format_rows(const T *v, int64_t rows, int64_t cols, char sep, const char *prefix, int32_t n_threads, char *out,
                int64_t cap, int64_t *used, int max_len, Fmt fmt) {
  const int64_t plen = prefix ? (int64_t)strlen(prefix) : 0;
  const int64_t row_max = plen + cols * (max_len + 1) + 1;
  int nw = n_workers(n_threads);
  if (rows < 4096) nw = 1;
  const int64_t per = (rows + nw - 1) / nw;
  std::vector<std::string> parts((size_t)nw);
  std::vector<std::thread> pool;
  for (int w = 0; w < nw; ++w) {
    int64_t lo = std::min(rows, w * per), hi = std::min(rows, lo + per);
    pool.emplace_back([&, lo, hi, w] {
      std::string &s = parts[(size_t)w];
      s.resize((size_t)((hi - lo) * row_max));
      char *o = &s[0];
      for (int64_t r = lo; r < hi; ++r) {
        if (plen) {
          memcpy(o, prefix, (size_t)plen);
          o += plen;
        }
        for (int64_t c = 0; c < cols; ++c) {
          if (c) *o++ = sep;
          o += fmt(v[r * cols + c], o);
        }
        *o++ = '\n';
      }
      s.resize((size_t)(o - s.data()));
    });
  }
  for (auto &t : pool) t.join();
  int64_t total = 0;
  for (auto &s : parts) total += (int64_t)s.size();
  *used = total;
  if (!out) return FH_OK;
  if (total > cap) return fh::set_error(FH_ERR_CONFIG, "fh_format: output buffer too small (%lld < %lld)",
                                        (long long)cap, (long long)total);
  char *o = out;
  for (auto &s : parts) {
    memcpy(o, s.data(), s.size());
    o += s.size();
  }
  return FH_OK;
}

}  // namespace

extern "C" {

int fh_mesh_parse(const char *text, int64_t len, int32_t n_threads, fh_mesh_text **out, int64_t *err_line) {
  if (err_line) *err_line = -1;
  if (!out || (!text && len)) return fh::set_error(FH_ERR_CONFIG, "fh_mesh_parse: null argument");
  *out = nullptr;
  auto *m = new fh_mesh_text();
  ParseError err;
  int rc;
  try {
    rc = parse(text, len, n_threads, m, &err);
  } catch (const std::bad_alloc &) {
    delete m;
    return fh::set_error(FH_ERR_CONFIG, "fh_mesh_parse: out of host memory");
  }
  if (rc) {
    delete m;
    if (err_line) *err_line = err.line;
    return fh::set_error(FH_ERR_FORMAT, "%s", err.msg.c_str());
  }
  *out = m;
  return FH_OK;
}

int fh_mesh_text_info(fh_mesh_text *m, int64_t *n_nodes, int64_t *n_tets, int64_t *n_hexes, int32_t *n_sets) {
  if (!m) return fh::set_error(FH_ERR_CONFIG, "fh_mesh_text_info: null handle");
  *n_nodes = (int64_t)m->nodes.size() / 3;
  *n_tets = (int64_t)m->tets.size() / 4;
  *n_hexes = (int64_t)m->hexes.size() / 8;
  *n_sets = (int32_t)m->set_names.size();
  return FH_OK;
}

int fh_mesh_text_arrays(fh_mesh_text *m, double *nodes, int64_t *tets, int64_t *hexes) {
  if (!m) return fh::set_error(FH_ERR_CONFIG, "fh_mesh_text_arrays: null handle");
  if (nodes) memcpy(nodes, m->nodes.data(), m->nodes.size() * sizeof(double));
  if (tets) memcpy(tets, m->tets.data(), m->tets.size() * sizeof(int64_t));
  if (hexes) memcpy(hexes, m->hexes.data(), m->hexes.size() * sizeof(int64_t));
  return FH_OK;
}

int fh_mesh_text_set(fh_mesh_text *m, int32_t i, char *name, int64_t name_cap, int64_t *ids, int64_t *count) {
  if (!m || i < 0 || i >= (int32_t)m->set_names.size())
    return fh::set_error(FH_ERR_CONFIG, "fh_mesh_text_set: bad handle or index %d", i);
  const std::string &s = m->set_names[(size_t)i];
  if (name) {
    if ((int64_t)s.size() + 1 > name_cap) return fh::set_error(FH_ERR_CONFIG, "fh_mesh_text_set: name buffer too small");
    memcpy(name, s.c_str(), s.size() + 1);
  }
  *count = (int64_t)m->set_ids[(size_t)i].size();
  if (ids) memcpy(ids, m->set_ids[(size_t)i].data(), (size_t)*count * sizeof(int64_t));
  return FH_OK;
}

int fh_mesh_text_destroy(fh_mesh_text *m) {
  delete m;
  return FH_OK;
}

int fh_format_f64(const double *v, int64_t rows, int64_t cols, char sep, const char *row_prefix, int32_t n_threads,
                  char *out, int64_t cap, int64_t *used) {
  if ((!v && rows && cols) || !used || rows < 0 || cols < 1)
    return fh::set_error(FH_ERR_CONFIG, "fh_format_f64: bad arguments");
  return format_rows(v, rows, cols, sep, row_prefix, n_threads, out, cap, used, kMaxF64,
                     [](double x, char *o) { return repr_f64(x, o); });
}

int fh_format_i64(const int64_t *v, int64_t rows, int64_t cols, char sep, const char *row_prefix, int32_t n_threads,
                  char *out, int64_t cap, int64_t *used) {
  if ((!v && rows && cols) || !used || rows < 0 || cols < 1)
    return fh::set_error(FH_ERR_CONFIG, "fh_format_i64: bad arguments");
  return format_rows(v, rows, cols, sep, row_prefix, n_threads, out, cap, used, kMaxI64,
                     [](int64_t x, char *o) { return str_i64(x, o); });
}

}  // extern "C"
