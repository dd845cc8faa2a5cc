// mmio.cpp -- Matrix Market ingestion / output and host CSR validation
// (SURVEY 8f row 1). Host code: text parsing is byte work the GPU cannot help
// with until the triplets exist, so the file is parsed by all host cores in
// parallel chunks and the resulting CSR goes straight to the device path
// (cs_problem_upload_csr / cs_problem_upload_csr_block).
//
// Behaviour follows the reference exactly:
//   read_matrix_market   problems.cpp:55-109  (header/size/entry rules, error
//                                               messages, symmetric expansion)
//   CsrMatrix::from_triplets  csr.cpp:34-56   (sort by (i,j), duplicates rejected)
//   validate_structure   csr.cpp:58-79
//   validate_symmetric   csr.cpp:81-98
//   validate_spd_diagonal csr.cpp:100-110
//   write_matrix_market  problems.cpp:111-127  (lower triangle, %.17g values)
// Token rules mirror std::istream extraction as libstdc++ performs it: integers
// are [ws][+-]digits (overflow fails), reals are the longest
// [+-]digits[.digits][(e|E)[+-]digits] prefix which must convert completely and
// finitely (overflow fails), and anything after the third token is ignored.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "chebstep_gpu.h"
#include "common.cuh"
#include "mmio.hpp"

namespace csg {

namespace {

[[noreturn]] void perr(const std::string& m) { throw LibError{CS_ERR_PARSE, 0, m}; }
[[noreturn]] void merr(const std::string& m) { throw LibError{CS_ERR_INVALID_MATRIX, 0, m}; }

inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream >> int64_t on [p, e)
bool get_i64(const char*& p, const char* e, int64_t* out) {
  while (p < e && is_ws(*p)) ++p;
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q >= e || !std::isdigit(static_cast<unsigned char>(*q))) return false;
  unsigned long long v = 0;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  bool over = false;
  for (; q < e && std::isdigit(static_cast<unsigned char>(*q)); ++q) {
    const unsigned d = static_cast<unsigned>(*q - '0');
    if (v > (lim - d) / 10) over = true;
    else v = v * 10 + d;
  }
  if (over) return false;
  *out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
  p = q;
  return true;
}

// istream >> double on [p, e)
bool get_f64(const char*& p, const char* e, double* out) {
  while (p < e && is_ws(*p)) ++p;
  const char* q = p;
  auto digits = [&] {
    while (q < e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
  };
  if (q < e && (*q == '+' || *q == '-')) ++q;
  digits();
  if (q < e && *q == '.') {
    ++q;
    digits();
  }
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    digits();
  }
  const size_t len = static_cast<size_t>(q - p);
  if (len == 0 || len > 400) return false;
  char buf[404];
  std::memcpy(buf, p, len);
  buf[len] = '\0';
  char* end = nullptr;
  const double v = std::strtod(buf, &end);
  if (end != buf + len || std::isinf(v)) return false;
  *out = v;
  p = q;
  return true;
}

struct Triplet {
  int64_t i, j;
  double v;
};

struct Chunk {
  std::vector<Triplet> t;  // expanded (i,j) and (j,i)
  int64_t entries = 0;     // entry lines parsed before any error
  bool has_err = false;
  bool err_range = false;
  std::string err_line;
};

void parse_chunk(const char* b, const char* e, int64_t rows, int64_t cols, Chunk* ck) {
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
    const char* le = nl ? nl : e;
    if (le > p && *p != '%') {
      const char* q = p;
      int64_t i, j;
      double v;
      if (!get_i64(q, le, &i) || !get_i64(q, le, &j) || !get_f64(q, le, &v)) {
        ck->has_err = true;
        ck->err_line.assign(p, le);
        return;
      }
      if (i < 1 || i > rows || j < 1 || j > cols) {
        ck->has_err = true;
        ck->err_range = true;
        ck->err_line.assign(p, le);
        return;
      }
      --i;
      --j;
      ck->t.push_back({i, j, v});
      if (i != j) ck->t.push_back({j, i, v});
      ++ck->entries;
    }
    p = nl ? nl + 1 : e;
  }
}

int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return static_cast<int>(std::clamp<unsigned>(h ? h : 1, 1, 64));
}

template <class F>
void parallel_for(int64_t count, int threads, F&& f) {
  if (threads <= 1 || count < 2) {
    for (int64_t k = 0; k < count; ++k) f(k);
    return;
  }
  std::vector<std::thread> pool;
  const int t = static_cast<int>(std::min<int64_t>(threads, count));
  for (int w = 0; w < t; ++w)
    pool.emplace_back([&, w] {
      for (int64_t k = w; k < count; k += t) f(k);
    });
  for (auto& th : pool) th.join();
}

// CsrMatrix::from_triplets (csr.cpp:34-56): rows by counting sort, each row
// sorted by column; any equal (i,j) pair is a duplicate.
void csr_from_triplets(int64_t n, std::vector<Chunk>& chunks, HostCsr* out) {
  out->n = n;
  out->rowptr.assign(static_cast<size_t>(n) + 1, 0);
  int64_t nnz = 0;
  for (auto& ck : chunks) {
    for (const Triplet& t : ck.t) ++out->rowptr[t.i + 1];
    nnz += static_cast<int64_t>(ck.t.size());
  }
  for (int64_t i = 0; i < n; ++i) out->rowptr[i + 1] += out->rowptr[i];
  out->col.resize(nnz);
  out->val.resize(nnz);
  std::vector<int64_t> fill(out->rowptr.begin(), out->rowptr.end() - 1);
  for (auto& ck : chunks) {
    for (const Triplet& t : ck.t) {
      const int64_t k = fill[t.i]++;
      out->col[k] = t.j;
      out->val[k] = t.v;
    }
    std::vector<Triplet>().swap(ck.t);
  }
  const int th = host_threads();
  const int64_t blocks = std::min<int64_t>(n, th * 8);
  std::vector<char> dup(static_cast<size_t>(blocks), 0);
  parallel_for(blocks, th, [&](int64_t blk) {
    std::vector<std::pair<int64_t, double>> row;
    for (int64_t i = n * blk / blocks; i < n * (blk + 1) / blocks; ++i) {
      const int64_t b = out->rowptr[i], e = out->rowptr[i + 1];
      bool sorted = true;
      for (int64_t k = b + 1; k < e; ++k)
        if (out->col[k] <= out->col[k - 1]) sorted = false;
      if (sorted) continue;
      row.clear();
      for (int64_t k = b; k < e; ++k) row.emplace_back(out->col[k], out->val[k]);
      std::sort(row.begin(), row.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      for (int64_t k = b; k < e; ++k) {
        out->col[k] = row[k - b].first;
        out->val[k] = row[k - b].second;
        if (k > b && out->col[k] == out->col[k - 1]) dup[blk] = 1;
      }
    }
  });
  for (char d : dup)
    if (d) merr("duplicate entry in triplet list");
}

}  // namespace

void validate_structure_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                             int64_t rowptr_len, int64_t nnz_len) {
  if (n < 0 || rowptr_len != n + 1) merr("row_offsets length must be n+1");
  if (rp[0] != 0) merr("row_offsets[0] must be 0");
  if (rp[n] != nnz_len) merr("row_offsets[n] must equal nnz");
  for (int64_t i = 0; i < n; ++i) {
    if (rp[i] > rp[i + 1]) merr("row_offsets must be nondecreasing");
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      if (ci[k] < 0 || ci[k] >= n) merr("column index out of range");
      if (k > rp[i] && ci[k] <= ci[k - 1]) merr("column indices must be strictly increasing");
    }
  }
  for (int64_t k = 0; k < nnz_len; ++k)
    if (!std::isfinite(v[k])) merr("non-finite matrix value");
}

static int64_t lower_bound_col(const int64_t* ci, int64_t b, int64_t e, int64_t c) {
  return std::lower_bound(ci + b, ci + e, c) - ci;
}

void validate_symmetric_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  validate_structure_host(n, rp, ci, v, n + 1, rp[n]);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = ci[k];
      const int64_t t = lower_bound_col(ci, rp[j], rp[j + 1], i);
      if (t == rp[j + 1] || ci[t] != i) merr("missing symmetric counterpart entry");
      if (v[t] != v[k]) merr("symmetric counterpart value differs");
    }
}

void validate_spd_diagonal_host(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  for (int64_t i = 0; i < n; ++i) {
    const int64_t t = lower_bound_col(ci, rp[i], rp[i + 1], i);
    if (t == rp[i + 1] || ci[t] != i)
      throw LibError{CS_ERR_NOT_SPD, 0, "missing diagonal entry in SPD matrix"};
    if (v[t] <= 0.0) throw LibError{CS_ERR_NOT_SPD, 0, "non-positive diagonal entry in SPD matrix"};
  }
}

// problems.cpp:55-109
HostCsr* mm_read(const std::string& path, bool require_spd) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) perr("cannot open " + path);
  std::string data;
  {
    char buf[1 << 16];
    size_t got;
    if (std::fseek(f, 0, SEEK_END) == 0) {
      const long sz = std::ftell(f);
      if (sz > 0) data.reserve(static_cast<size_t>(sz));
      std::fseek(f, 0, SEEK_SET);
    }
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) data.append(buf, got);
    std::fclose(f);
  }
  const char* p = data.data();
  const char* e = p + data.size();
  auto next_line = [&](std::string* line) -> bool {
    if (p >= e) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
    const char* le = nl ? nl : e;
    line->assign(p, le);
    p = nl ? nl + 1 : e;
    return true;
  };
  std::string header;
  if (!next_line(&header)) perr("empty file: " + path);
  {
    std::string tok[5];
    const char* q = header.data();
    const char* he = q + header.size();
    for (auto& t : tok) {
      while (q < he && is_ws(*q)) ++q;
      const char* s = q;
      while (q < he && !is_ws(*q)) ++q;
      t.assign(s, q);
    }
    for (int k = 1; k < 5; ++k)
      for (auto& c : tok[k]) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    if (tok[0] != "%%MatrixMarket" || tok[1] != "matrix" || tok[2] != "coordinate" ||
        tok[3] != "real")
      perr("unsupported MatrixMarket header: " + header);
    if (tok[4] != "symmetric") perr("matrix must be declared symmetric, got: " + tok[4]);
  }
  int64_t rows = 0, cols = 0, entries = 0;
  std::string line;
  while (next_line(&line)) {
    if (line.empty() || line[0] == '%') continue;
    const char* q = line.data();
    const char* le = q + line.size();
    if (!get_i64(q, le, &rows) || !get_i64(q, le, &cols) || !get_i64(q, le, &entries))
      perr("bad size line: " + line);
    break;
  }
  if (rows <= 0 || rows != cols) perr("matrix must be square and non-empty");
  if (entries <= 0) perr("empty coordinate section");

  // entry section: chunks split at line boundaries, parsed concurrently
  const int th = host_threads();
  const int64_t bytes = e - p;
  const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(th * 4, bytes >> 16));
  std::vector<const char*> cut(static_cast<size_t>(nchunks) + 1);
  cut[0] = p;
  cut[nchunks] = e;
  for (int64_t k = 1; k < nchunks; ++k) {
    const char* c = std::max(cut[k - 1], p + bytes * k / nchunks);
    const char* nl = c < e ? static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(e - c)))
                           : nullptr;
    cut[k] = nl ? nl + 1 : e;
  }
  std::vector<Chunk> chunks(static_cast<size_t>(nchunks));
  parallel_for(nchunks, th, [&](int64_t k) {
    chunks[k].t.reserve(static_cast<size_t>((cut[k + 1] - cut[k]) / 8));
    parse_chunk(cut[k], cut[k + 1], rows, cols, &chunks[k]);
  });
  // reading stops after `entries` entry lines (problems.cpp:89): only errors
  // and triplets before that point count
  int64_t seen = 0;
  size_t used = 0;
  for (; used < chunks.size(); ++used) {
    Chunk& ck = chunks[used];
    if (seen + ck.entries >= entries) {
      int64_t keep = entries - seen, kept = 0;
      size_t pos = 0;
      while (kept < keep) {
        pos += ck.t[pos].i != ck.t[pos].j ? 2 : 1;
        ++kept;
      }
      ck.t.resize(pos);
      seen = entries;
      ++used;
      break;
    }
    seen += ck.entries;
    if (ck.has_err)
      perr((ck.err_range ? "entry index out of range: " : "bad entry line: ") + ck.err_line);
  }
  if (seen < entries) perr("fewer entries than declared");
  chunks.resize(used);
  auto out = std::make_unique<HostCsr>();
  csr_from_triplets(rows, chunks, out.get());
  validate_structure_host(out->n, out->rowptr.data(), out->col.data(), out->val.data(),
                          out->n + 1, static_cast<int64_t>(out->col.size()));
  if (require_spd)
    validate_spd_diagonal_host(out->n, out->rowptr.data(), out->col.data(), out->val.data());
  return out.release();
}

// problems.cpp:111-127
void mm_write(const std::string& path, int64_t n, const int64_t* rp, const int64_t* ci,
              const double* v) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw LibError{CS_ERR_GENERIC, 0, "cannot open for writing: " + path};
  int64_t lower = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] <= i) ++lower;
  std::string buf = "%%MatrixMarket matrix coordinate real symmetric\n";
  buf += std::to_string(n) + " " + std::to_string(n) + " " + std::to_string(lower) + "\n";
  char tmp[96];
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] <= i) {
        const int len = std::snprintf(tmp, sizeof tmp, "%lld %lld %.17g\n",
                                      static_cast<long long>(i + 1),
                                      static_cast<long long>(ci[k] + 1), v[k]);
        buf.append(tmp, static_cast<size_t>(len));
      }
    if (buf.size() > (1u << 22)) {
      std::fwrite(buf.data(), 1, buf.size(), f);
      buf.clear();
    }
  }
  std::fwrite(buf.data(), 1, buf.size(), f);
  if (std::fclose(f) != 0) throw LibError{CS_ERR_GENERIC, 0, "write failed: " + path};
}

}  // namespace csg
