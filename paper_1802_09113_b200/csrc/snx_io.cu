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

// strtod / strtoll over a token [b, e); true when the whole token was consumed
bool parse_double(const char *b, const char *e, double *out) {
  std::string t(b, e);
  char *end = nullptr;
  errno = 0;
  *out = strtod(t.c_str(), &end);
  return end == t.c_str() + t.size() && !t.empty();
}

bool parse_int(const char *b, const char *e, long long *out) {
  std::string t(b, e);
  char *end = nullptr;
  errno = 0;
  *out = strtoll(t.c_str(), &end, 10);
  return end == t.c_str() + t.size() && !t.empty() && errno == 0;
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
