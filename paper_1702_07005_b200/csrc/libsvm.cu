// libsvm.cu — host reader for the LIBSVM text format the paper's datasets come in (webspam, criteo;
// P:254): one example per line, `label index:value ...`, 1-based strictly increasing indices.
// Reading: text after '#' is a comment, blank lines are skipped, values are parsed as
// doubles and rounded to fp32, indices become 0-based.  Two passes: scd_libsvm_size counts, then
// scd_libsvm_read fills caller-allocated CSR arrays (host C++, no device work).
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace scd {
namespace {

struct Sink {
  int64_t *ptr = nullptr;
  int32_t *idx = nullptr;
  float *val = nullptr;
  float *y = nullptr;
};

// parses the whole file; with a null sink only counts.  Returns an error message or "".
std::string parse(const char *path, int64_t n_cols_hint, int64_t *n_rows, int64_t *nnz, int64_t *n_cols, Sink s) {
  FILE *f = fopen(path, "rb");
  if (!f) return std::string("cannot open ") + path + ": " + strerror(errno);
  std::string line;
  char buf[1 << 16];
  int64_t rows = 0, entries = 0, max_j = -1, lineno = 0;
  if (s.ptr) s.ptr[0] = 0;
  std::string err;
  auto flush_line = [&]() -> bool {
    ++lineno;
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    const char *p = line.c_str();
    while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
    if (!*p) return true;
    char *end = nullptr;
    const double label = strtod(p, &end);
    if (end == p) {
      err = "line " + std::to_string(lineno) + ": bad label";
      return false;
    }
    p = end;
    int64_t last = -1;
    for (;;) {
      while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
      if (!*p) break;
      const long long j1 = strtoll(p, &end, 10);
      if (end == p || *end != ':') {
        err = "line " + std::to_string(lineno) + ": expected index:value";
        return false;
      }
      const int64_t j = (int64_t)j1 - 1;
      if (j < 0 || j <= last || j > INT32_MAX) {
        err = "line " + std::to_string(lineno) + ": indices must be 1-based and strictly increasing";
        return false;
      }
      p = end + 1;
      const double v = strtod(p, &end);
      if (end == p) {
        err = "line " + std::to_string(lineno) + ": bad value";
        return false;
      }
      p = end;
      if (s.idx) {
        s.idx[entries] = (int32_t)j;
        s.val[entries] = (float)v;
      }
      ++entries;
      last = j;
      if (j > max_j) max_j = j;
    }
    if (s.y) s.y[rows] = (float)label;
    ++rows;
    if (s.ptr) s.ptr[rows] = entries;
    return true;
  };
  bool ok = true;
  while (ok && fgets(buf, sizeof(buf), f)) {
    line += buf;
    if (!line.empty() && line.back() == '\n') {
      line.pop_back();
      ok = flush_line();
      line.clear();
    }
  }
  if (ok && !line.empty()) ok = flush_line();
  fclose(f);
  if (!ok) return err;
  const int64_t nc = n_cols_hint > 0 ? n_cols_hint : max_j + 1;
  if (max_j >= nc) return "index " + std::to_string(max_j + 1) + " beyond n_cols " + std::to_string(nc);
  *n_rows = rows;
  *nnz = entries;
  *n_cols = nc < 1 ? 1 : nc;
  return "";
}

}  // namespace
}  // namespace scd

using namespace scd;

extern "C" {

scd_status scd_libsvm_size(const char *path, int64_t n_cols_hint, int64_t *n_rows, int64_t *nnz, int64_t *n_cols) {
  set_global_error("");
  if (!path || !n_rows || !nnz || !n_cols) {
    set_global_error("NULL argument");
    return SCD_E_INVALID_ARG;
  }
  const std::string e = parse(path, n_cols_hint, n_rows, nnz, n_cols, Sink{});
  if (!e.empty()) {
    set_global_error(e);
    return SCD_E_INVALID_ARG;
  }
  return SCD_OK;
}

scd_status scd_libsvm_read(const char *path, int64_t n_cols_hint, int64_t *ptr, int32_t *idx, float *val, float *y) {
  set_global_error("");
  if (!path || !ptr || !idx || !val || !y) {
    set_global_error("NULL argument");
    return SCD_E_INVALID_ARG;
  }
  int64_t r = 0, z = 0, c = 0;
  Sink s;
  s.ptr = ptr;
  s.idx = idx;
  s.val = val;
  s.y = y;
  const std::string e = parse(path, n_cols_hint, &r, &z, &c, s);
  if (!e.empty()) {
    set_global_error(e);
    return SCD_E_INVALID_ARG;
  }
  return SCD_OK;
}

}  // extern "C"
