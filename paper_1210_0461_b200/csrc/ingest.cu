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
