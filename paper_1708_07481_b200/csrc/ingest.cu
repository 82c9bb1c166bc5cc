// (f.2) Edge-list ingestion: the tab-separated ``src dst [weight]`` reader of
// graph.py:152-209 (load_edge_list) as multithreaded host code.
//
// The buffer is split at newline boundaries into one chunk per thread; a first
// pass counts lines per chunk (global 1-based line numbers), a second parses
// each chunk into thread-local arrays that are concatenated in file order, so
// the arc order is the file order, as in the reference. Accepted syntax is the
// common subset of Python's int()/float(): optional sign and ASCII digits for
// vertex ids; decimal/exponent floats, inf/infinity/nan for weights; fields
// split on ASCII whitespace; '#' comments and blank lines skipped. Anything
// else (non-ASCII bytes, '_' digit separators, ids beyond int64, malformed
// fields, negative ids or weights) stops the parse with SPB_ERR_PARSE and the
// 1-based line number of the first such line, and the Python layer re-reads the
// file with the reference's own loop to raise the exact exception.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace spb {
namespace {

struct ChunkOut {
  std::vector<int64_t> src, dst;
  std::vector<double> w;
  int64_t max_idx = -1;
  bool any_w = false;
  int64_t bad_line = 0;  // 1-based, 0 = none
};

inline bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// strict int: [+-]?[0-9]+ (no '_' separators); false on overflow
inline bool parse_int(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) {
    neg = *b == '-';
    ++b;
  }
  if (b == e) return false;
  uint64_t v = 0;
  for (; b < e; ++b) {
    const unsigned d = (unsigned)(*b - '0');
    if (d > 9) return false;
    if (v > (uint64_t)(INT64_MAX / 10)) return false;
    v = v * 10 + d;
    if (v > (uint64_t)INT64_MAX) return false;
  }
  *out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

inline bool ieq(const char* b, const char* e, const char* lit) {
  const size_t n = strlen(lit);
  if ((size_t)(e - b) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if ((b[i] | 0x20) != lit[i]) return false;
  return true;
}

// float: Python float() decimal syntax (no '_'), or inf / infinity / nan with sign
inline bool parse_float(const char* b, const char* e, double* out) {
  const char* p = b;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    ++p;
  }
  if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(p, e, "nan")) {
    *out = NAN;
    return true;
  }
  // validate [digits][.digits][(e|E)[+-]digits] with at least one mantissa digit
  const char* q = p;
  int md = 0;
  while (q < e && (unsigned)(*q - '0') <= 9) ++q, ++md;
  if (q < e && *q == '.') {
    ++q;
    while (q < e && (unsigned)(*q - '0') <= 9) ++q, ++md;
  }
  if (md == 0) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    int ed = 0;
    while (q < e && (unsigned)(*q - '0') <= 9) ++q, ++ed;
    if (ed == 0) return false;
  }
  if (q != e) return false;
  char tmp[128];
  const size_t n = (size_t)(e - b);
  if (n >= sizeof(tmp)) return false;  // leave very long tokens to the Python reader
  memcpy(tmp, b, n);
  tmp[n] = 0;
  errno = 0;
  *out = strtod(tmp, nullptr);  // correctly rounded, like float()
  return true;
}

void parse_chunk(const char* b, const char* e, int64_t first_line, int base, ChunkOut* o) {
  int64_t line = first_line;
  const char* p = b;
  while (p < e) {
    const char* nl = (const char*)memchr(p, '\n', (size_t)(e - p));
    const char* le = nl ? nl : e;
    // fields
    const char* f[4];
    const char* fe[4];
    int nf = 0;
    const char* s = p;
    bool bad = false;
    while (s < le) {
      while (s < le && is_ws((unsigned char)*s)) ++s;
      if (s >= le) break;
      const char* t = s;
      while (t < le && !is_ws((unsigned char)*t)) {
        if ((unsigned char)*t >= 0x80) bad = true;
        ++t;
      }
      if (nf < 4) {
        f[nf] = s;
        fe[nf] = t;
      }
      ++nf;
      s = t;
    }
    if (!bad && nf > 0 && *f[0] == '#') {
      // comment line
    } else if (bad) {
      o->bad_line = line;
      return;
    } else if (nf > 0) {
      int64_t u, v;
      double w = 1.0;
      if ((nf != 2 && nf != 3) || !parse_int(f[0], fe[0], &u) || !parse_int(f[1], fe[1], &v) ||
          (nf == 3 && !parse_float(f[2], fe[2], &w))) {
        o->bad_line = line;
        return;
      }
      u -= base;
      v -= base;
      if (u < 0 || v < 0 || w < 0) {
        o->bad_line = line;
        return;
      }
      o->src.push_back(u);
      o->dst.push_back(v);
      o->w.push_back(w);
      o->any_w |= nf == 3;
      o->max_idx = std::max(o->max_idx, std::max(u, v));
    }
    ++line;
    p = nl ? nl + 1 : e;
  }
}

struct Parsed {
  std::vector<ChunkOut> chunks;
  int64_t m = 0;
};

}  // namespace
}  // namespace spb

using namespace spb;

extern "C" int spb_edge_list_parse(const char* data, size_t len, int32_t base, int32_t nthreads,
                                   int64_t* m_out, int64_t* max_idx_out, int32_t* has_weights_out,
                                   int64_t* bad_line_out, void** handle_out) {
  if (handle_out) *handle_out = nullptr;
  if (base != 0 && base != 1) {
    set_error("base must be 0 or 1");
    return SPB_ERR_DOMAIN;
  }
  if (!data && len) {
    set_error("null buffer");
    return SPB_ERR_CONTRACT;
  }
  int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, (int64_t)(len / (1 << 16)) + 1));
  // chunk boundaries just after a newline
  std::vector<size_t> cut(nt + 1, len);
  cut[0] = 0;
  for (int t = 1; t < nt; ++t) {
    size_t c = std::max(cut[t - 1], len * (size_t)t / (size_t)nt);
    const char* nl = c < len ? (const char*)memchr(data + c, '\n', len - c) : nullptr;
    cut[t] = nl ? (size_t)(nl - data) + 1 : len;
  }
  std::vector<int64_t> lines(nt, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        lines[t] = (int64_t)std::count(data + cut[t], data + cut[t + 1], '\n');
      });
    for (auto& x : th) x.join();
  }
  auto* P = new Parsed();
  P->chunks.resize(nt);
  {
    std::vector<std::thread> th;
    int64_t first = 1;
    for (int t = 0; t < nt; ++t) {
      th.emplace_back([&, t, first] {
        ChunkOut* o = &P->chunks[t];
        o->src.reserve((size_t)lines[t] + 1);
        o->dst.reserve((size_t)lines[t] + 1);
        o->w.reserve((size_t)lines[t] + 1);
        parse_chunk(data + cut[t], data + cut[t + 1], first, base, o);
      });
      first += lines[t];
    }
    for (auto& x : th) x.join();
  }
  int64_t bad = 0, m = 0, mx = -1;
  bool anyw = false;
  for (auto& c : P->chunks) {
    if (c.bad_line && !bad) bad = c.bad_line;
    m += (int64_t)c.src.size();
    mx = std::max(mx, c.max_idx);
    anyw |= c.any_w;
  }
  if (bad) {
    delete P;
    if (bad_line_out) *bad_line_out = bad;
    set_error("line %lld: not in the fast-path syntax", (long long)bad);
    return SPB_ERR_PARSE;
  }
  P->m = m;
  if (m_out) *m_out = m;
  if (max_idx_out) *max_idx_out = mx;
  if (has_weights_out) *has_weights_out = anyw ? 1 : 0;
  if (bad_line_out) *bad_line_out = 0;
  *handle_out = P;
  return SPB_OK;
}

extern "C" int spb_edge_list_fetch(void* handle, int64_t* src, int64_t* dst, double* w) {
  auto* P = (Parsed*)handle;
  if (!P) {
    set_error("null edge-list handle");
    return SPB_ERR_CONTRACT;
  }
  size_t off = 0;
  for (auto& c : P->chunks) {
    const size_t k = c.src.size();
    if (src) memcpy(src + off, c.src.data(), k * sizeof(int64_t));
    if (dst) memcpy(dst + off, c.dst.data(), k * sizeof(int64_t));
    if (w) memcpy(w + off, c.w.data(), k * sizeof(double));
    off += k;
  }
  delete P;
  return SPB_OK;
}

extern "C" void spb_edge_list_free(void* handle) { delete (Parsed*)handle; }
