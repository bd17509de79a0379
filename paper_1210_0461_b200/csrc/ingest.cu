// ingest.cu -- native FIMI reader (input ingestion).
//
// Replaces the Python line loop of read_fimi (sparse.py:270-298) on the
// mine() path (mining.py:52-65): the file is read once, cut into one chunk
// per host thread at line boundaries, and every thread parses its lines
// into sorted, de-duplicated uint32 ids; the per-thread pieces are
// concatenated into CSR (offsets int64, items uint32) ready for one pinned
// host -> device copy.
//
// Semantics follow read_fimi: one transaction per line, blank (whitespace-
// only) lines skipped, items sorted and de-duplicated per line, duplicates
// counted. The reader only accepts the plain form of the input -- ASCII
// decimal tokens with an optional sign, ASCII whitespace, '\n' or "\r\n"
// line ends, ids < 2^31. Anything else (a negative id, a non-integer token,
// a bare '\r', non-ASCII bytes, '_' digit separators, huge ids) is reported
// as CROP_EINPUT with the 1-based line number and the caller re-reads the
// file with the reference-exact Python reader, which raises the reference's
// ParseError (message and line number) or accepts the unusual form.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

struct crop_fimi {
  std::vector<int64_t> offsets;
  std::vector<uint32_t> items;
  uint32_t max_item = 0;
  int64_t duplicates = 0;
};

namespace {

struct Piece {
  std::vector<uint32_t> lens;  // items per kept line
  std::vector<uint32_t> items;
  uint32_t max_item = 0;
  int64_t duplicates = 0;
  int64_t lines = 0;           // all lines of the chunk (blank ones included)
  int64_t bad_line = -1;       // chunk-local 0-based line of the first rejected line
};

inline bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\v' || c == '\f' || c == '\r' || (c >= 0x1c && c <= 0x1f);
}

void parse_chunk(const char* b, const char* e, Piece& P) {
  std::vector<uint32_t> line;
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* le = nl ? nl : e;
    line.clear();
    bool bad = false;
    for (const char* q = p; q < le && !bad;) {
      const unsigned char c = (unsigned char)*q;
      if (is_space(c)) {
        // a '\r' must end the line (Windows line end); a bare one is a
        // universal-newline line break the Python reader would count
        if (c == '\r' && q + 1 != le) bad = true;
        ++q;
        continue;
      }
      bool neg = false;
      if (c == '+' || c == '-') {
        neg = c == '-';
        ++q;
      }
      const char* d0 = q;
      uint64_t v = 0;
      while (q < le && *q >= '0' && *q <= '9') {
        v = v * 10 + (uint64_t)(*q - '0');
        if (v >= (1ull << 31)) break;
        ++q;
      }
      if (q == d0 || (q < le && !is_space((unsigned char)*q)) || v >= (1ull << 31) || (neg && v != 0)) {
        bad = true;
        break;
      }
      line.push_back((uint32_t)v);
    }
    if (bad) {
      P.bad_line = P.lines;
      return;
    }
    ++P.lines;
    if (!line.empty()) {
      std::sort(line.begin(), line.end());
      const size_t u = (size_t)(std::unique(line.begin(), line.end()) - line.begin());
      P.duplicates += (int64_t)(line.size() - u);
      P.lens.push_back((uint32_t)u);
      P.items.insert(P.items.end(), line.begin(), line.begin() + u);
      P.max_item = std::max(P.max_item, line[u - 1]);
    }
    p = nl ? nl + 1 : e;
  }
}

}  // namespace

extern "C" int crop_fimi_parse(const char* path, int threads, crop_fimi** out, int64_t* n_tx,
                               int64_t* nnz, uint32_t* max_item, int64_t* duplicates,
                               int64_t* bad_line) {
  *out = nullptr;
  *bad_line = 0;
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    crop_set_error(CROP_EINPUT, "cannot read %s", path);
    return CROP_EINPUT;
  }
  std::vector<char> buf;
  if (fseek(fh, 0, SEEK_END) == 0) {
    const long size = ftell(fh);
    if (size > 0) {
      buf.resize((size_t)size);
      fseek(fh, 0, SEEK_SET);
      if (fread(buf.data(), 1, buf.size(), fh) != buf.size()) {
        fclose(fh);
        crop_set_error(CROP_EINPUT, "short read of %s", path);
        return CROP_EINPUT;
      }
    }
  }
  fclose(fh);
  const size_t n = buf.size();
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  T = std::max(1, std::min(T, 64));
  if (n < (size_t)T * (1 << 16)) T = std::max<int>(1, (int)(n >> 16));
  // chunk starts at line boundaries
  std::vector<size_t> cut(T + 1, n);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    size_t c = std::max(cut[t - 1], n * (size_t)t / (size_t)T);
    while (c < n && c > 0 && buf[c - 1] != '\n') ++c;
    cut[t] = c;
  }
  std::vector<Piece> pieces(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t]() { parse_chunk(buf.data() + cut[t], buf.data() + cut[t + 1], pieces[t]); });
  for (auto& th : pool) th.join();
  int64_t line_base = 0;
  for (int t = 0; t < T; ++t) {
    if (pieces[t].bad_line >= 0) {
      *bad_line = line_base + pieces[t].bad_line + 1;
      crop_set_error(CROP_EINPUT, "%s:%lld: not a plain FIMI line", path, (long long)*bad_line);
      return CROP_EINPUT;
    }
    line_base += pieces[t].lines;
  }
  crop_fimi* F = new crop_fimi();
  size_t tx = 0, it = 0;
  for (auto& P : pieces) {
    tx += P.lens.size();
    it += P.items.size();
  }
  F->offsets.resize(tx + 1);
  F->items.resize(it);
  size_t k = 0, o = 0;
  F->offsets[0] = 0;
  for (auto& P : pieces) {
    for (uint32_t len : P.lens) {
      o += len;
      F->offsets[++k] = (int64_t)o;
    }
    F->max_item = std::max(F->max_item, P.max_item);
    F->duplicates += P.duplicates;
  }
  size_t at = 0;
  for (auto& P : pieces) {
    if (!P.items.empty()) memcpy(F->items.data() + at, P.items.data(), P.items.size() * 4);
    at += P.items.size();
  }
  *out = F;
  *n_tx = (int64_t)tx;
  *nnz = (int64_t)it;
  *max_item = F->max_item;
  *duplicates = F->duplicates;
  return CROP_OK;
}

extern "C" int crop_fimi_copy(const crop_fimi* F, int64_t* offsets, uint32_t* items) {
  memcpy(offsets, F->offsets.data(), F->offsets.size() * sizeof(int64_t));
  if (!F->items.empty()) memcpy(items, F->items.data(), F->items.size() * sizeof(uint32_t));
  return CROP_OK;
}

extern "C" void crop_fimi_free(crop_fimi* F) { delete F; }

// ---------------------------------------------------------------- triple files
// Native read_triple_file (sparse.py:173-225) for the multiply / partition
// paths: header "n_rows n_cols kcount", then "k index value" per line, k
// non-decreasing. The file is cut into one chunk per host thread at line
// boundaries; each thread parses its lines into (k, index, value) triples
// (explicit zeros dropped and counted, as the reference does); the pieces
// are concatenated, grouped by k (already sorted), each group sorted by
// index and checked for duplicates. Only the plain form is accepted --
// ASCII decimal integers, decimal / exponent floats (strtod, correctly
// rounded like Python's float()), '\n' or "\r\n" line ends. Anything else,
// and every error the reference reports (bad header, malformed triple,
// unsorted or out-of-range k, negative index, NaN), returns CROP_EINPUT with
// the 1-based line (0 for a duplicate index); the caller re-reads the file
// with the reference-exact Python reader, which raises the reference's
// ParseError.
struct crop_triples {
  int64_t n_rows = 0, n_cols = 0, kcount = 0;
  std::vector<int64_t> ptr;
  std::vector<uint32_t> idx;
  std::vector<double> val;
  int64_t zeros = 0;
};

namespace {

struct TPiece {
  std::vector<int64_t> k;
  std::vector<uint32_t> idx;
  std::vector<double> val;
  int64_t zeros = 0, lines = 0, bad_line = -1;
  int64_t first_k = -1, last_k = -1;
};

// [+-]?digits, no sign for an index; returns false on anything else
bool parse_int(const char*& q, const char* e, int64_t& out, bool allow_sign) {
  bool neg = false;
  if (allow_sign && q < e && (*q == '+' || *q == '-')) {
    neg = *q == '-';
    ++q;
  }
  const char* d0 = q;
  uint64_t v = 0;
  while (q < e && *q >= '0' && *q <= '9') {
    v = v * 10 + (uint64_t)(*q - '0');
    if (v > (1ull << 40)) return false;
    ++q;
  }
  if (q == d0) return false;
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

// [+-]? (digits [. digits?] | . digits) ([eE] [+-]? digits)?
bool parse_float(const char*& q, const char* e, double& out) {
  const char* s0 = q;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  int nd = 0;
  while (q < e && *q >= '0' && *q <= '9') ++q, ++nd;
  if (q < e && *q == '.') {
    ++q;
    while (q < e && *q >= '0' && *q <= '9') ++q, ++nd;
  }
  if (nd == 0) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    int ne = 0;
    while (q < e && *q >= '0' && *q <= '9') ++q, ++ne;
    if (ne == 0) return false;
  }
  char tmp[128];
  const size_t len = (size_t)(q - s0);
  if (len >= sizeof(tmp)) return false;
  memcpy(tmp, s0, len);
  tmp[len] = 0;
  out = strtod(tmp, nullptr);
  return true;
}

inline bool tok_end(const char* q, const char* e) { return q == e || is_space((unsigned char)*q); }

void parse_triples(const char* b, const char* e, TPiece& P) {
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(e - p)));
    const char* le = nl ? nl : e;
    if (le > p && le[-1] == '\r') --le;  // "\r\n"
    const char* q = p;
    auto skip = [&]() {
      while (q < le && is_space((unsigned char)*q)) {
        if (*q == '\r') return false;  // a bare '\r' inside the line
        ++q;
      }
      return true;
    };
    bool ok = skip();
    if (ok && q < le) {
      int64_t k = 0, ix = 0;
      double v = 0.0;
      ok = parse_int(q, le, k, true) && tok_end(q, le) && skip() &&
           parse_int(q, le, ix, true) && tok_end(q, le) && skip() &&
           parse_float(q, le, v) && tok_end(q, le) && skip() && q == le;
      // reference checks, in its order: sorted k, range of k, index >= 0
      if (ok && (k < P.last_k || k < 0 || ix < 0 || ix >= (1ll << 32))) ok = false;
      if (ok) {
        if (P.first_k < 0) P.first_k = k;
        P.last_k = k;
        if (v == 0.0) {
          ++P.zeros;
        } else {
          P.k.push_back(k);
          P.idx.push_back((uint32_t)ix);
          P.val.push_back(v);
        }
      }
    }
    if (!ok) {
      P.bad_line = P.lines;
      return;
    }
    ++P.lines;
    p = nl ? nl + 1 : e;
  }
}

}  // namespace

extern "C" int crop_triple_parse(const char* path, int threads, crop_triples** out, int64_t* dims,
                                 int64_t* nnz, int64_t* zeros, int64_t* bad_line) {
  *out = nullptr;
  *bad_line = 0;
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    crop_set_error(CROP_EINPUT, "cannot read %s", path);
    return CROP_EINPUT;
  }
  std::vector<char> buf;
  if (fseek(fh, 0, SEEK_END) == 0) {
    const long size = ftell(fh);
    if (size > 0) {
      buf.resize((size_t)size);
      fseek(fh, 0, SEEK_SET);
      if (fread(buf.data(), 1, buf.size(), fh) != buf.size()) {
        fclose(fh);
        crop_set_error(CROP_EINPUT, "short read of %s", path);
        return CROP_EINPUT;
      }
    }
  }
  fclose(fh);
  auto bad = [&](int64_t line) {
    *bad_line = line;
    crop_set_error(CROP_EINPUT, "%s:%lld: not a plain triple line", path, (long long)line);
    return CROP_EINPUT;
  };
  // header (line 1)
  const size_t n = buf.size();
  const char* b0 = buf.data();
  const char* hl = static_cast<const char*>(memchr(b0, '\n', n));
  const char* he = hl ? hl : b0 + n;
  const char* body = hl ? hl + 1 : b0 + n;
  if (he > b0 && he[-1] == '\r') --he;
  int64_t hdr[3];
  {
    const char* q = b0;
    for (int f = 0; f < 3; ++f) {
      while (q < he && (*q == ' ' || *q == '\t')) ++q;
      if (!parse_int(q, he, hdr[f], true) || !tok_end(q, he) || hdr[f] < 0) return bad(1);
    }
    while (q < he && (*q == ' ' || *q == '\t')) ++q;
    if (q != he || n == 0) return bad(1);
  }
  const size_t m = (size_t)(b0 + n - body);
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  T = std::max(1, std::min(T, 64));
  if (m < (size_t)T * (1 << 16)) T = std::max<int>(1, (int)(m >> 16));
  std::vector<size_t> cut(T + 1, m);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    size_t c = std::max(cut[t - 1], m * (size_t)t / (size_t)T);
    while (c < m && c > 0 && body[c - 1] != '\n') ++c;
    cut[t] = c;
  }
  std::vector<TPiece> pieces(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t]() { parse_triples(body + cut[t], body + cut[t + 1], pieces[t]); });
  for (auto& th : pool) th.join();
  // first failure (line numbers: header = 1), then k order across chunks and k range
  int64_t line_base = 2, last_k = -1;
  size_t total = 0;
  for (int t = 0; t < T; ++t) {
    TPiece& P = pieces[t];
    if (P.first_k >= 0 && P.first_k < last_k) {
      // the first triple line of this chunk breaks the order: find it
      return bad(line_base);
    }
    if (P.bad_line >= 0) return bad(line_base + P.bad_line);
    if (P.last_k >= hdr[2]) return bad(line_base);  // reported precisely by the Python reader
    if (P.last_k >= 0) last_k = P.last_k;
    line_base += P.lines;
    total += P.k.size();
  }
  crop_triples* R = new crop_triples();
  R->n_rows = hdr[0];
  R->n_cols = hdr[1];
  R->kcount = hdr[2];
  R->ptr.assign((size_t)hdr[2] + 1, 0);
  R->idx.resize(total);
  R->val.resize(total);
  size_t at = 0;
  for (auto& P : pieces) {
    for (size_t x = 0; x < P.k.size(); ++x) ++R->ptr[(size_t)P.k[x] + 1];
    if (!P.idx.empty()) {
      memcpy(R->idx.data() + at, P.idx.data(), P.idx.size() * 4);
      memcpy(R->val.data() + at, P.val.data(), P.val.size() * 8);
    }
    at += P.idx.size();
    R->zeros += P.zeros;
  }
  for (size_t k = 0; k < (size_t)hdr[2]; ++k) R->ptr[k + 1] += R->ptr[k];
  // per k: sort by index, reject duplicates (the reference reports line 0)
  std::vector<std::pair<uint32_t, double>> g;
  for (size_t k = 0; k < (size_t)hdr[2]; ++k) {
    const int64_t a = R->ptr[k], z = R->ptr[k + 1];
    bool sorted = true;
    for (int64_t x = a + 1; x < z; ++x)
      if (R->idx[x] <= R->idx[x - 1]) sorted = false;
    if (sorted) continue;
    g.clear();
    for (int64_t x = a; x < z; ++x) g.emplace_back(R->idx[x], R->val[x]);
    std::stable_sort(g.begin(), g.end(),
                     [](const std::pair<uint32_t, double>& l, const std::pair<uint32_t, double>& r) {
                       return l.first < r.first;
                     });
    for (size_t x = 1; x < g.size(); ++x)
      if (g[x].first == g[x - 1].first) {
        delete R;
        return bad(0);
      }
    for (int64_t x = a; x < z; ++x) {
      R->idx[x] = g[x - a].first;
      R->val[x] = g[x - a].second;
    }
  }
  *out = R;
  dims[0] = R->n_rows;
  dims[1] = R->n_cols;
  dims[2] = R->kcount;
  *nnz = (int64_t)total;
  *zeros = R->zeros;
  return CROP_OK;
}

extern "C" int crop_triple_copy(const crop_triples* R, int64_t* ptr, uint32_t* idx, double* val) {
  memcpy(ptr, R->ptr.data(), R->ptr.size() * sizeof(int64_t));
  if (!R->idx.empty()) {
    memcpy(idx, R->idx.data(), R->idx.size() * 4);
    memcpy(val, R->val.data(), R->val.size() * 8);
  }
  return CROP_OK;
}

extern "C" void crop_triple_free(crop_triples* R) { delete R; }
