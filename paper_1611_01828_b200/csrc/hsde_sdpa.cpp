// hsde_sdpa.cpp -- SDPA sparse-format reader, restating
// chordalsdp/sdpa.py:94-234 `parse_sdpa`: comment lines ('"' or '*') only
// before the header; header lines tokenised after replacing ",{}()" with
// blanks; entry lines "matno blkno i j value" (whitespace, exactly five
// fields, 1-based, i > j normalised); explicit zeros kept; negative block
// sizes are diagonal blocks; errors carry the 1-based line number with the
// reference's messages, duplicates flagged separately (DuplicateEntry).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "../../include/hsde.h"

struct hsde_sdpa {
  int32_t m = 0;
  std::vector<int32_t> dims;
  std::vector<double> b;
  std::vector<int32_t> mat, blk, ii, jj;
  std::vector<double> val;
};

namespace {

thread_local std::string g_msg;
thread_local int64_t g_line = 0;
thread_local int32_t g_dup = 0;

struct ParseFail {
  int64_t line;
  std::string msg;
  bool dup;
};

// str.isspace() over ASCII: blanks plus the \x1c-\x1f separators
inline bool is_ws(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= '\x1c' && c <= '\x1f'); }
// str.splitlines() line boundaries over ASCII
inline bool is_eol(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= '\x1c' && c <= '\x1e'); }

std::string strip(const std::string &s) {
  const char *ws = " \t\n\r\v\f\x1c\x1d\x1e\x1f";
  const size_t a = s.find_first_not_of(ws);
  if (a == std::string::npos) return "";
  const size_t b = s.find_last_not_of(ws);
  return s.substr(a, b - a + 1);
}

std::vector<std::string> split_ws(const std::string &s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && is_ws(s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !is_ws(s[j])) ++j;
    if (j > i) out.push_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

std::vector<std::string> header_tokens(std::string s) {
  for (char &c : s)
    if (c == ',' || c == '{' || c == '}' || c == '(' || c == ')') c = ' ';
  return split_ws(s);
}

std::string repr(const std::string &t) { return "'" + t + "'"; }

// Python int(): optional sign, decimal digits, single underscores between digits
bool parse_int(const std::string &t, long long &v) {
  std::string d;
  size_t i = 0;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) d += t[i++];
  if (i >= t.size()) return false;
  bool prev_digit = false;
  for (; i < t.size(); ++i) {
    if (std::isdigit((unsigned char)t[i])) {
      d += t[i];
      prev_digit = true;
    } else if (t[i] == '_' && prev_digit && i + 1 < t.size() && std::isdigit((unsigned char)t[i + 1])) {
      prev_digit = false;
    } else {
      return false;
    }
  }
  errno = 0;
  v = std::strtoll(d.c_str(), nullptr, 10);
  return errno == 0;
}

// Python float(): strtod on the whole token (inf / nan / exponents)
bool parse_float(const std::string &t, double &v) {
  if (t.empty()) return false;
  std::string d;
  for (size_t i = 0; i < t.size(); ++i) {
    if (t[i] == '_') {
      if (i == 0 || i + 1 >= t.size() || !std::isdigit((unsigned char)t[i - 1]) ||
          !std::isdigit((unsigned char)t[i + 1]))
        return false;
      continue;
    }
    d += t[i];
  }
  std::string low;
  for (char c : d) low += (char)std::tolower((unsigned char)c);
  const std::string body = (!low.empty() && (low[0] == '+' || low[0] == '-')) ? low.substr(1) : low;
  if (body == "inf" || body == "infinity" || body == "nan") {
    v = std::strtod(d.c_str(), nullptr);
    return true;
  }
  if (body.empty() || body.find_first_not_of("0123456789.e+-") != std::string::npos) return false;
  char *end = nullptr;
  v = std::strtod(d.c_str(), &end);
  return end && *end == '\0';
}

void parse(const std::string &text, hsde_sdpa &p) {
  // splitlines (\n, \r\n, \r, \v, \f, \x1c-\x1e)
  std::vector<std::string> lines;
  {
    size_t i = 0;
    while (i < text.size()) {
      size_t j = i;
      while (j < text.size() && !is_eol(text[j])) ++j;
      lines.push_back(text.substr(i, j - i));
      if (j < text.size() && text[j] == '\r' && j + 1 < text.size() && text[j + 1] == '\n') ++j;
      i = j + 1;
    }
  }
  const int64_t total = (int64_t)lines.size();
  int64_t pos = 0;
  auto next_data_line = [&](bool allow_comment, int64_t &lineno) -> std::string {
    while (pos < total) {
      lineno = pos + 1;
      const std::string s = strip(lines[pos]);
      ++pos;
      if (s.empty()) continue;
      if (s[0] == '"' || s[0] == '*') {
        if (allow_comment) continue;
        throw ParseFail{lineno, "comment lines are only allowed before the header", false};
      }
      return s;
    }
    throw ParseFail{total, "unexpected end of input", false};
  };
  int64_t ln = 0;
  auto want_int = [&](const std::string &t, int64_t lineno, const char *what) -> long long {
    long long v;
    if (!parse_int(t, v)) throw ParseFail{lineno, std::string("expected integer ") + what + ", got " + repr(t), false};
    return v;
  };
  std::string line = next_data_line(true, ln);
  auto toks = header_tokens(line);
  if (toks.empty()) throw ParseFail{ln, "expected integer constraint count, got ''", false};
  const long long m = want_int(toks[0], ln, "constraint count");
  if (m < 1) throw ParseFail{ln, "constraint count must be positive, got " + std::to_string(m), false};
  line = next_data_line(false, ln);
  toks = header_tokens(line);
  if (toks.empty()) throw ParseFail{ln, "expected integer block count, got ''", false};
  const long long nblocks = want_int(toks[0], ln, "block count");
  if (nblocks < 1) throw ParseFail{ln, "block count must be positive, got " + std::to_string(nblocks), false};
  while ((long long)p.dims.size() < nblocks) {
    line = next_data_line(false, ln);
    for (const auto &t : header_tokens(line)) {
      if ((long long)p.dims.size() == nblocks) break;
      const long long d = want_int(t, ln, "block size");
      if (d == 0) throw ParseFail{ln, "block size must be nonzero", false};
      p.dims.push_back((int32_t)d);
    }
  }
  while ((long long)p.b.size() < m) {
    line = next_data_line(false, ln);
    for (const auto &t : header_tokens(line)) {
      if ((long long)p.b.size() == m) break;
      double v;
      if (!parse_float(t, v)) throw ParseFail{ln, "expected number right-hand side entry, got " + repr(t), false};
      p.b.push_back(v);
    }
  }
  p.m = (int32_t)m;
  struct Key {
    int64_t mb, ij;  // (matno, blkno), (i, j)
    bool operator==(const Key &o) const { return mb == o.mb && ij == o.ij; }
  };
  struct KH {
    size_t operator()(const Key &x) const { return std::hash<int64_t>()(x.mb * 0x9E3779B97F4A7C15ull ^ x.ij); }
  };
  std::unordered_set<Key, KH> seen;
  std::vector<std::tuple<int32_t, int32_t, int32_t, int32_t, double>> ent;
  while (pos < total) {
    const int64_t lineno = pos + 1;
    const std::string s = strip(lines[pos]);
    ++pos;
    if (s.empty()) continue;
    if (s[0] == '"' || s[0] == '*') throw ParseFail{lineno, "comment lines are only allowed before the header", false};
    const auto f = split_ws(s);
    if (f.size() != 5)
      throw ParseFail{lineno, "entry line needs 5 fields, got " + std::to_string(f.size()), false};
    const long long matno = want_int(f[0], lineno, "matrix number");
    const long long blkno = want_int(f[1], lineno, "block number");
    long long i = want_int(f[2], lineno, "row index");
    long long j = want_int(f[3], lineno, "column index");
    double value;
    if (!parse_float(f[4], value)) throw ParseFail{lineno, "expected number entry value, got " + repr(f[4]), false};
    if (!(0 <= matno && matno <= m))
      throw ParseFail{lineno, "matrix number " + std::to_string(matno) + " outside [0, " + std::to_string(m) + "]", false};
    if (!(1 <= blkno && blkno <= nblocks))
      throw ParseFail{lineno, "block number " + std::to_string(blkno) + " outside [1, " + std::to_string(nblocks) + "]",
                      false};
    const long long size = std::llabs((long long)p.dims[blkno - 1]);
    if (i > j) std::swap(i, j);
    if (!(1 <= i && i <= j && j <= size))
      throw ParseFail{lineno, "entry (" + std::to_string(i) + ", " + std::to_string(j) + ") outside block of size " +
                                  std::to_string(size), false};
    if (p.dims[blkno - 1] < 0 && i != j)
      throw ParseFail{lineno, "off-diagonal entry (" + std::to_string(i) + ", " + std::to_string(j) +
                                  ") in diagonal block " + std::to_string(blkno), false};
    if (!seen.insert(Key{matno * (nblocks + 1) + blkno, (i << 32) | j}).second)
      throw ParseFail{lineno, "duplicate entry for matrix " + std::to_string(matno) + ", block " + std::to_string(blkno) +
                                  ", (" + std::to_string(i) + ", " + std::to_string(j) + ")", true};
    ent.emplace_back((int32_t)matno, (int32_t)(blkno - 1), (int32_t)(i - 1), (int32_t)(j - 1), value);
  }
  std::sort(ent.begin(), ent.end(), [](const auto &a, const auto &b) {
    return std::make_tuple(std::get<0>(a), std::get<1>(a), std::get<2>(a), std::get<3>(a)) <
           std::make_tuple(std::get<0>(b), std::get<1>(b), std::get<2>(b), std::get<3>(b));
  });
  for (const auto &e : ent) {
    p.mat.push_back(std::get<0>(e));
    p.blk.push_back(std::get<1>(e));
    p.ii.push_back(std::get<2>(e));
    p.jj.push_back(std::get<3>(e));
    p.val.push_back(std::get<4>(e));
  }
}

}  // namespace

extern "C" {

int hsde_sdpa_parse(const char *text, int64_t len, hsde_sdpa_t **out) {
  if (!out || (!text && len)) return HSDE_ERR_ARG;
  g_msg.clear();
  g_line = 0;
  g_dup = 0;
  hsde_sdpa *p = new hsde_sdpa();
  try {
    parse(std::string(text ? text : "", (size_t)len), *p);
  } catch (const ParseFail &f) {
    g_msg = f.msg;
    g_line = f.line;
    g_dup = f.dup ? 1 : 0;
    delete p;
    return HSDE_ERR_ARG;
  }
  *out = p;
  return HSDE_OK;
}

const char *hsde_sdpa_error(int64_t *line, int32_t *duplicate) {
  if (line) *line = g_line;
  if (duplicate) *duplicate = g_dup;
  return g_msg.c_str();
}

int hsde_sdpa_sizes(const hsde_sdpa_t *p, int32_t *m, int32_t *nblocks, int64_t *n_entries) {
  if (!p) return HSDE_ERR_ARG;
  if (m) *m = p->m;
  if (nblocks) *nblocks = (int32_t)p->dims.size();
  if (n_entries) *n_entries = (int64_t)p->val.size();
  return HSDE_OK;
}

int hsde_sdpa_data(const hsde_sdpa_t *p, int32_t *block_dims, double *b, int32_t *mat, int32_t *blk, int32_t *i,
                   int32_t *j, double *val) {
  if (!p) return HSDE_ERR_ARG;
  if (block_dims) std::copy(p->dims.begin(), p->dims.end(), block_dims);
  if (b) std::copy(p->b.begin(), p->b.end(), b);
  if (mat) std::copy(p->mat.begin(), p->mat.end(), mat);
  if (blk) std::copy(p->blk.begin(), p->blk.end(), blk);
  if (i) std::copy(p->ii.begin(), p->ii.end(), i);
  if (j) std::copy(p->jj.begin(), p->jj.end(), j);
  if (val) std::copy(p->val.begin(), p->val.end(), val);
  return HSDE_OK;
}

void hsde_sdpa_destroy(hsde_sdpa_t *p) { delete p; }

}  // extern "C"
