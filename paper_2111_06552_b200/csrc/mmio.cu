// MatrixMarket ingestion, native (reference io.py:108-216, read_matrix_market).
//
// The reference parses line by line in Python.  Here the whole file is read
// once, split into lines (universal newlines, as Python's text mode), and the
// coordinate entries are tokenised by several host threads over disjoint line
// ranges.  Semantics follow the reference exactly:
//   * banner: 5 tokens, "%%MatrixMarket" (case-insensitive), object "matrix",
//     format coordinate|array, field real, symmetry general|symmetric —
//     anything else is a parse error (line 1) or "unsupported";
//   * comment ('%' after leading blanks) and blank lines are skipped anywhere;
//   * entry errors carry the 1-based line of the offending line; the first
//     error in file order wins, with "more than the declared N entries"
//     raised at the (N+1)-th entry line before that line is parsed;
//   * symmetric coordinate storage is mirrored (off-diagonal entries
//     appended after all stored ones); array format is column-major, the
//     symmetric variant stores the lower triangle by columns.
// Summing duplicates and sorting by (row, col) happen when the caller
// assembles CSR (the Python adapter, io.py).
//
// This is host code (no kernels): the parse feeds the device CSR upload.

#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <exception>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "gcgb200.h"

namespace {

struct MMFile {
  std::string text;
  std::vector<size_t> lb, le;  // [begin, end) of each line, without the terminator
  gcg_mm_info info;
  std::vector<int64_t> rows, cols;
  std::vector<double> vals;
};

inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\v' || c == '\f' || c == '\r' || c == '\n';
}

void split_lines(MMFile& f) {
  const std::string& t = f.text;
  size_t i = 0, n = t.size();
  while (i < n) {
    size_t j = i;
    while (j < n && t[j] != '\n' && t[j] != '\r') ++j;
    f.lb.push_back(i);
    f.le.push_back(j);
    if (j < n && t[j] == '\r' && j + 1 < n && t[j + 1] == '\n') j += 2;
    else j += 1;
    i = j;
  }
}

// tokens of line `ln` (0-based) as [begin, end) offsets; returns the count (capped at cap)
int tokens(const MMFile& f, size_t ln, size_t* tb, size_t* te, int cap) {
  const char* s = f.text.data();
  size_t i = f.lb[ln], e = f.le[ln];
  int k = 0;
  while (i < e) {
    while (i < e && is_ws(s[i])) ++i;
    if (i >= e) break;
    size_t j = i;
    while (j < e && !is_ws(s[j])) ++j;
    if (k < cap) {
      tb[k] = i;
      te[k] = j;
    }
    ++k;
    i = j;
  }
  return k;
}

bool skip_line(const MMFile& f, size_t ln) {  // comment or blank
  const char* s = f.text.data();
  size_t i = f.lb[ln], e = f.le[ln];
  while (i < e && is_ws(s[i])) ++i;
  return i >= e || s[i] == '%';
}

std::string tok(const MMFile& f, size_t b, size_t e) { return f.text.substr(b, e - b); }

std::string lower(std::string s) {
  for (auto& c : s) c = (char)tolower((unsigned char)c);
  return s;
}

bool parse_int(const std::string& s, long long* out) {
  if (s.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const long long v = strtoll(s.c_str(), &end, 10);
  if (errno || end != s.c_str() + s.size()) return false;
  *out = v;
  return true;
}

bool parse_real(const std::string& s, double* out) {
  if (s.empty()) return false;
  for (char c : s)
    if (c == 'x' || c == 'X') return false;  // no hex floats (Python float() rejects them)
  errno = 0;
  char* end = nullptr;
  const double v = strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) return false;
  *out = v;
  return true;
}

void set_err(gcg_mm_info* info, int kind, long long line, const std::string& msg) {
  info->err_kind = kind;
  info->err_line = line;
  snprintf(info->err_msg, sizeof(info->err_msg), "%s", msg.c_str());
}

// one thread's share of coordinate entry lines
struct Chunk {
  size_t l0 = 0, l1 = 0;
  std::vector<int64_t> r, c;
  std::vector<double> v;
  long long ndata = 0;           // data lines seen (up to and excluding the first error)
  long long err_line = -1;       // first malformed data line (1-based)
  long long err_index = -1;      // its data-line index within the chunk
  std::string err_msg;
};

void parse_chunk(const MMFile& f, Chunk& ch, long long nrows, long long ncols) {
  size_t tb[4], te[4];
  for (size_t ln = ch.l0; ln < ch.l1; ++ln) {
    if (skip_line(f, ln)) continue;
    const long long lineno = (long long)ln + 1;
    const int nt = tokens(f, ln, tb, te, 4);
    std::string msg;
    long long i = 0, j = 0;
    double v = 0.0;
    if (nt != 3) {
      msg = "entry must be 'row col value'";
    } else if (!parse_int(tok(f, tb[0], te[0]), &i)) {
      msg = "bad row index '" + tok(f, tb[0], te[0]) + "'";
    } else if (!parse_int(tok(f, tb[1], te[1]), &j)) {
      msg = "bad column index '" + tok(f, tb[1], te[1]) + "'";
    } else if (!(1 <= i && i <= nrows && 1 <= j && j <= ncols)) {
      msg = "index (" + std::to_string(i) + ", " + std::to_string(j) + ") outside " +
            std::to_string(nrows) + "x" + std::to_string(ncols);
    } else if (!parse_real(tok(f, tb[2], te[2]), &v)) {
      msg = "bad value '" + tok(f, tb[2], te[2]) + "'";
    }
    if (!msg.empty()) {
      ch.err_line = lineno;
      ch.err_index = ch.ndata;
      ch.err_msg = msg;
      ++ch.ndata;  // the malformed line still counts as an entry line
      return;
    }
    ch.r.push_back(i - 1);
    ch.c.push_back(j - 1);
    ch.v.push_back(v);
    ++ch.ndata;
  }
}

// line (1-based) of data line number `target` (0-based) inside [l0, l1), or -1
long long data_line(const MMFile& f, size_t l0, size_t l1, long long target) {
  long long k = 0;
  for (size_t ln = l0; ln < l1; ++ln) {
    if (skip_line(f, ln)) continue;
    if (k == target) return (long long)ln + 1;
    ++k;
  }
  return -1;
}

void read_coordinate(MMFile& f, size_t first, long long nrows, long long ncols, long long nnz,
                     int nthreads) {
  gcg_mm_info* info = &f.info;
  const size_t nl = f.lb.size();
  const size_t span = nl > first ? nl - first : 0;
  int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if ((size_t)nt > span / 4096 + 1) nt = (int)(span / 4096 + 1);
  std::vector<Chunk> ch(nt);
  for (int t = 0; t < nt; ++t) {
    ch[t].l0 = first + span * t / nt;
    ch[t].l1 = first + span * (t + 1) / nt;
  }
  if (nt == 1) {
    parse_chunk(f, ch[0], nrows, ncols);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(parse_chunk, std::cref(f), std::ref(ch[t]), nrows, ncols);
    for (auto& x : th) x.join();
  }
  // first error in file order: a malformed entry line, or the (nnz+1)-th entry line
  long long before = 0;  // entry lines in earlier chunks
  for (int t = 0; t < nt; ++t) {
    const Chunk& c = ch[t];
    const long long upto = c.err_line >= 0 ? c.err_index : c.ndata;  // clean lines of this chunk
    if (before + upto > nnz || (c.err_line >= 0 && before + c.err_index >= nnz)) {
      const long long line = data_line(f, c.l0, c.l1, nnz - before);
      set_err(info, 1, line, "more than the declared " + std::to_string(nnz) + " entries");
      return;
    }
    if (c.err_line >= 0) {
      set_err(info, 1, c.err_line, c.err_msg);
      return;
    }
    before += c.ndata;
  }
  if (before != nnz) {
    set_err(info, 1, (long long)nl + 1,
            "declared " + std::to_string(nnz) + " entries but found " + std::to_string(before));
    return;
  }
  size_t total = 0;
  for (auto& c : ch) total += c.v.size();
  size_t extra = 0;
  if (info->symmetric)
    for (auto& c : ch)
      for (size_t k = 0; k < c.v.size(); ++k) extra += c.r[k] != c.c[k];
  f.rows.reserve(total + extra);
  f.cols.reserve(total + extra);
  f.vals.reserve(total + extra);
  for (auto& c : ch) {
    f.rows.insert(f.rows.end(), c.r.begin(), c.r.end());
    f.cols.insert(f.cols.end(), c.c.begin(), c.c.end());
    f.vals.insert(f.vals.end(), c.v.begin(), c.v.end());
  }
  if (info->symmetric) {
    for (size_t k = 0; k < total; ++k) {
      if (f.rows[k] != f.cols[k]) {
        f.rows.push_back(f.cols[k]);
        f.cols.push_back(f.rows[k]);
        f.vals.push_back(f.vals[k]);
      }
    }
  }
  info->nentries = (int64_t)f.vals.size();
}

void read_array(MMFile& f, size_t first, long long nrows, long long ncols) {
  gcg_mm_info* info = &f.info;
  const size_t nl = f.lb.size();
  long long expected;
  // the header is untrusted: check the value count for overflow and never size a
  // buffer from it (the reference counts the values first, io.py:214-222)
  if (nrows < 0 || ncols < 0 || (ncols > 0 && nrows > (1LL << 62) / ncols)) {
    set_err(info, 1, (long long)first, "array dimensions too large");
    return;
  }
  if (info->symmetric) {
    if (nrows != ncols) {
      set_err(info, 1, (long long)first, "symmetric array must be square");
      return;
    }
    expected = nrows * (nrows + 1) / 2;
  } else {
    expected = nrows * ncols;
  }
  std::vector<double> v;
  std::vector<size_t> tb(64), te(64);
  for (size_t ln = first; ln < nl; ++ln) {
    if (skip_line(f, ln)) continue;
    int nt = tokens(f, ln, tb.data(), te.data(), (int)tb.size());
    if (nt > (int)tb.size()) {
      tb.resize(nt);
      te.resize(nt);
      nt = tokens(f, ln, tb.data(), te.data(), nt);
    }
    for (int k = 0; k < nt; ++k) {
      if ((long long)v.size() >= expected) {
        set_err(info, 1, (long long)ln + 1,
                "more than the declared " + std::to_string(expected) + " values");
        return;
      }
      double x;
      if (!parse_real(tok(f, tb[k], te[k]), &x)) {
        set_err(info, 1, (long long)ln + 1, "bad value '" + tok(f, tb[k], te[k]) + "'");
        return;
      }
      v.push_back(x);
    }
  }
  if ((long long)v.size() != expected) {
    set_err(info, 1, (long long)nl + 1,
            "declared " + std::to_string(expected) + " values but found " +
                std::to_string(v.size()));
    return;
  }
  // dense column-major n x m
  f.vals.assign((size_t)(nrows * ncols), 0.0);
  size_t k = 0;
  if (info->symmetric) {
    for (long long j = 0; j < ncols; ++j)
      for (long long i = j; i < nrows; ++i) {
        f.vals[(size_t)(j * nrows + i)] = v[k];
        f.vals[(size_t)(i * nrows + j)] = v[k];
        ++k;
      }
  } else {
    for (size_t e = 0; e < v.size(); ++e) f.vals[e] = v[e];
  }
  info->nentries = nrows * ncols;
}

void parse_file(MMFile& f, int nthreads) {
  gcg_mm_info* info = &f.info;
  split_lines(f);
  const size_t nl = f.lb.size();
  if (nl == 0) {
    set_err(info, 1, 1, "empty file");
    return;
  }
  size_t tb[8], te[8];
  const int nb = tokens(f, 0, tb, te, 8);
  if (nb != 5 || lower(tok(f, tb[0], te[0])) != "%%matrixmarket") {
    set_err(info, 1, 1, "expected banner '%%MatrixMarket matrix <format> <field> <symmetry>'");
    return;
  }
  const std::string obj = lower(tok(f, tb[1], te[1])), fmt = lower(tok(f, tb[2], te[2]));
  const std::string field = lower(tok(f, tb[3], te[3])), sym = lower(tok(f, tb[4], te[4]));
  if (obj != "matrix") {
    set_err(info, 2, 0, "object '" + obj + "' not supported (only 'matrix')");
    return;
  }
  if (fmt != "coordinate" && fmt != "array") {
    set_err(info, 1, 1, "unknown format '" + tok(f, tb[2], te[2]) + "'");
    return;
  }
  if (field != "real") {
    set_err(info, 2, 0, "field '" + tok(f, tb[3], te[3]) + "' not supported (only 'real')");
    return;
  }
  if (sym != "general" && sym != "symmetric") {
    set_err(info, 2, 0,
            "symmetry '" + tok(f, tb[4], te[4]) + "' not supported (only 'general'/'symmetric')");
    return;
  }
  info->format = fmt == "coordinate" ? 0 : 1;
  info->symmetric = sym == "symmetric";
  size_t idx = 1;
  while (idx < nl && skip_line(f, idx)) ++idx;
  if (idx >= nl) {
    set_err(info, 1, (long long)nl + 1, "missing size line");
    return;
  }
  const long long size_line = (long long)idx + 1;
  const int ns = tokens(f, idx, tb, te, 8);
  long long v[3] = {0, 0, 0};
  const char* what[3] = {"row count", "column count", "entry count"};
  const int want = info->format == 0 ? 3 : 2;
  if (ns != want) {
    set_err(info, 1, size_line,
            info->format == 0 ? "size line must be 'rows cols nnz'" : "size line must be 'rows cols'");
    return;
  }
  for (int k = 0; k < want; ++k) {
    if (!parse_int(tok(f, tb[k], te[k]), &v[k])) {
      set_err(info, 1, size_line, std::string("bad ") + what[k] + " '" + tok(f, tb[k], te[k]) + "'");
      return;
    }
  }
  if (v[0] < 0 || v[1] < 0 || v[2] < 0) {
    set_err(info, 1, size_line, "size line entries must be nonnegative");
    return;
  }
  info->nrows = v[0];
  info->ncols = v[1];
  if (info->format == 0) read_coordinate(f, idx + 1, v[0], v[1], v[2], nthreads);
  else read_array(f, idx + 1, v[0], v[1]);
}

}  // namespace

extern "C" {

int gcg_mm_open(const char* path, int nthreads, void** handle, gcg_mm_info* info) {
  if (!path || !handle || !info) return GCG_ERR_ARG;
  *handle = nullptr;
  MMFile* f = new MMFile();
  memset(&f->info, 0, sizeof(f->info));
  FILE* fp = fopen(path, "rb");
  if (!fp) {
    set_err(&f->info, 3, 0, std::string("cannot read ") + path + ": " + strerror(errno));
    *info = f->info;
    delete f;
    return GCG_ERR_IO;
  }
  fseek(fp, 0, SEEK_END);
  const long sz = ftell(fp);
  fseek(fp, 0, SEEK_SET);
  f->text.resize(sz > 0 ? (size_t)sz : 0);
  if (sz > 0 && fread(&f->text[0], 1, (size_t)sz, fp) != (size_t)sz) {
    fclose(fp);
    set_err(&f->info, 3, 0, std::string("cannot read ") + path);
    *info = f->info;
    delete f;
    return GCG_ERR_IO;
  }
  fclose(fp);
  try {
    parse_file(*f, nthreads);
  } catch (const std::bad_alloc&) {
    set_err(&f->info, 3, 0, "out of host memory while parsing");
  } catch (const std::exception& e) {
    set_err(&f->info, 1, 0, std::string("parse failed: ") + e.what());
  }
  *info = f->info;
  if (f->info.err_kind) {
    const int st = f->info.err_kind == 1 ? GCG_ERR_PARSE : (f->info.err_kind == 2 ? GCG_ERR_UNSUPPORTED : GCG_ERR_IO);
    delete f;
    return st;
  }
  f->text.clear();
  f->text.shrink_to_fit();
  *handle = f;
  return GCG_OK;
}

int gcg_mm_fetch(void* handle, int64_t* rows, int64_t* cols, double* vals) {
  MMFile* f = (MMFile*)handle;
  if (!f || !vals) return GCG_ERR_ARG;
  if (f->info.format == 0) {
    if (!rows || !cols) return GCG_ERR_ARG;
    std::copy(f->rows.begin(), f->rows.end(), rows);
    std::copy(f->cols.begin(), f->cols.end(), cols);
  }
  std::copy(f->vals.begin(), f->vals.end(), vals);
  return GCG_OK;
}

void gcg_mm_close(void* handle) { delete (MMFile*)handle; }

}  // extern "C"
