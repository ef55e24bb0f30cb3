// LIBSVM / svmlight text ingest (the reference's load_libsvm, dataset.py:242-293),
// host code: one pass over the file in memory, CSR arrays out.  The Python side
// (paper_1802_09113_b200/io.py) remaps the labels (dataset.py:200-213), picks
// the storage (dataset.py:216-226) and uploads to HBM.
//
// Parsing rules (the reference's): whitespace-separated tokens; blank lines are
// skipped; the first token is the label (a float); the others are idx:val with
// a 1-based integer idx and a float val.  A malformed token is a parse error
// with its 1-based line number.
#include <errno.h>
#include <locale.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "snx_internal.h"

namespace {

struct Parsed {
  std::vector<double> labels, data;
  std::vector<int64_t> indptr{0};
  std::vector<int32_t> indices;
  int64_t max_index = 0;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// The reference parses tokens with Python's float() and int() (dataset.py:266-279),
// so the grammar here is theirs, not strtod's: digit groups may be separated by
// single underscores (PEP 515: "1_000", "2.5e1_0"), inf / infinity / nan in any
// case, no hexadecimal floats, no locale-dependent decimal point.  A valid token
// is stripped of its underscores and converted in the C locale (correctly
// rounded, as Python's conversion).
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// digitpart: digit ("_"? digit)* starting at s[i]; appends the digits to out
bool digit_part(const std::string &s, size_t &i, std::string &out) {
  if (i >= s.size() || !is_digit(s[i])) return false;
  out.push_back(s[i++]);
  while (i < s.size()) {
    if (is_digit(s[i])) {
      out.push_back(s[i++]);
    } else if (s[i] == '_' && i + 1 < s.size() && is_digit(s[i + 1])) {
      ++i;
    } else {
      break;
    }
  }
  return true;
}

bool ieq(const std::string &a, const char *b) {
  if (a.size() != strlen(b)) return false;
  for (size_t k = 0; k < a.size(); ++k) {
    char c = a[k];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != b[k]) return false;
  }
  return true;
}

locale_t c_locale() {
  static locale_t loc = newlocale(LC_ALL_MASK, "C", (locale_t)0);
  return loc;
}

// Python float(token) for a token [b, e) without surrounding whitespace
bool parse_double(const char *b, const char *e, double *out) {
  const std::string s(b, e);
  size_t i = 0;
  std::string clean;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) clean.push_back(s[i++]);
  const std::string rest = s.substr(i);
  if (ieq(rest, "inf") || ieq(rest, "infinity")) {
    *out = clean == "-" ? -HUGE_VAL : HUGE_VAL;
    return true;
  }
  if (ieq(rest, "nan")) {
    *out = clean == "-" ? -NAN : NAN;
    return true;
  }
  bool mant = false;
  if (i < s.size() && is_digit(s[i])) mant = digit_part(s, i, clean);
  if (i < s.size() && s[i] == '.') {
    clean.push_back(s[i++]);
    if (i < s.size() && is_digit(s[i])) mant = digit_part(s, i, clean) || mant;
  }
  if (!mant) return false;
  if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
    clean.push_back(s[i++]);
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) clean.push_back(s[i++]);
    if (!digit_part(s, i, clean)) return false;
  }
  if (i != s.size()) return false;
  char *end = nullptr;
  *out = strtod_l(clean.c_str(), &end, c_locale());
  return end == clean.c_str() + clean.size();
}

// Python int(token) in base 10 (sign, digits with single underscores)
bool parse_int(const char *b, const char *e, long long *out) {
  const std::string s(b, e);
  size_t i = 0;
  std::string clean;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) clean.push_back(s[i++]);
  if (!digit_part(s, i, clean) || i != s.size()) return false;
  char *end = nullptr;
  errno = 0;
  *out = strtoll(clean.c_str(), &end, 10);
  return end == clean.c_str() + clean.size() && errno == 0;
}

int parse_file(const char *path, Parsed *P) {
  FILE *f = fopen(path, "rb");
  if (!f) {
    snx::set_error("snx_libsvm: cannot open %s", path);
    return 1;
  }
  std::vector<char> buf;
  char chunk[1 << 16];
  size_t k;
  while ((k = fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + k);
  fclose(f);
  const char *p = buf.data(), *end = p + buf.size();
  long long lineno = 0;
  while (p < end) {
    const char *le = static_cast<const char *>(memchr(p, '\n', end - p));
    if (!le) le = end;
    ++lineno;
    const char *q = p;
    bool first = true;
    bool any = false;
    while (q < le) {
      while (q < le && is_space(*q)) ++q;
      if (q >= le) break;
      const char *tb = q;
      while (q < le && !is_space(*q)) ++q;
      const char *te = q;
      if (first) {
        double lab;
        if (!parse_double(tb, te, &lab)) {
          snx::set_error("line %lld: bad label '%.*s'", lineno, (int)(te - tb), tb);
          return 2;
        }
        P->labels.push_back(lab);
        first = false;
        any = true;
        continue;
      }
      const char *colon = static_cast<const char *>(memchr(tb, ':', te - tb));
      if (!colon) {
        snx::set_error("line %lld: expected idx:val pair, got '%.*s'", lineno, (int)(te - tb), tb);
        return 2;
      }
      long long idx;
      double val;
      if (!parse_int(tb, colon, &idx) || !parse_double(colon + 1, te, &val)) {
        snx::set_error("line %lld: bad idx:val pair '%.*s'", lineno, (int)(te - tb), tb);
        return 2;
      }
      if (idx < 1) {
        snx::set_error("line %lld: feature indices are 1-based, got %lld", lineno, idx);
        return 2;
      }
      if (idx > 0x7fffffffLL) {
        snx::set_error("line %lld: feature index %lld exceeds int32", lineno, idx);
        return 2;
      }
      P->indices.push_back((int32_t)(idx - 1));
      P->data.push_back(val);
      if (idx > P->max_index) P->max_index = idx;
    }
    if (any) P->indptr.push_back((int64_t)P->data.size());
    p = le + 1;
  }
  return 0;
}

// One parse cached between the size query and the copy-out (single-threaded
// ingest, like the reference's loader).
Parsed *g_last = nullptr;
std::string g_last_path;

}  // namespace

extern "C" {

int snx_libsvm_scan(const char *path, int64_t *nrows, int64_t *nnz, int64_t *max_index) {
  delete g_last;
  g_last = new Parsed();
  g_last_path = path;
  const int rc = parse_file(path, g_last);
  if (rc) {
    delete g_last;
    g_last = nullptr;
    return rc;
  }
  *nrows = (int64_t)g_last->labels.size();
  *nnz = (int64_t)g_last->data.size();
  *max_index = g_last->max_index;
  return 0;
}

int snx_libsvm_fetch(const char *path, double *labels, int64_t *indptr, int32_t *indices,
                     double *data) {
  if (!g_last || g_last_path != path) {
    snx::set_error("snx_libsvm_fetch: call snx_libsvm_scan(%s) first", path);
    return 1;
  }
  memcpy(labels, g_last->labels.data(), g_last->labels.size() * sizeof(double));
  memcpy(indptr, g_last->indptr.data(), g_last->indptr.size() * sizeof(int64_t));
  memcpy(indices, g_last->indices.data(), g_last->indices.size() * sizeof(int32_t));
  memcpy(data, g_last->data.data(), g_last->data.size() * sizeof(double));
  delete g_last;
  g_last = nullptr;
  return 0;
}

}  // extern "C"
