// pairs.cu -- K2: exact pair counting of a self-join transaction stream.
//
// Replaces the exact regime of engine.run / run_worker (engine.py:238-302,
// 396-455) for pair mining (mining.py:52-65): every entry (i, j) whose
// bucket (h_row(i) + h_col(j)) mod kappa lies in this GPU's interval gets its
// exact support. The reference streams terms one by one into per-bucket
// dicts; here the pair space is cut into on-chip TILES so that every term is
// counted by a shared-memory atomic and never touches HBM:
//
//   pass A  k_item_terms   per row item i: terms_i = #pairs (i, j>i) over all
//                          transactions (O(input), smem-privatised histogram)
//   plan    host           rows -> tiles. A tile is a contiguous row range
//                          (optionally one row x a column window) whose
//                          counters fit one SM's shared memory, either DENSE
//                          (closed-form triangle addressing, <= kDenseCap u32)
//                          or HASH (open addressing, <= kHashCap keys, bounded
//                          by sum_i min(width_i, terms_i)). Heavy tiles are
//                          split into UNITS that count into private copies.
//   pass B  k_route        per transaction, one ENTRY (tx, p0, p1) per run of
//                          positions whose rows share a tile: the tile's work
//                          list. Entries, not terms, cross HBM (8 B per run
//                          instead of 4-8 B per term).
//   count   k_count        persistent CTAs pull units, expand each entry's
//                          pairs warp-wide, filter by bucket interval, count
//                          with shared-memory atomics, then compact non-zero
//                          counters to the output (or a slab if split).
//   reduce  k_slab_reduce  sum the slabs of split tiles and compact.
//
// Data in HBM: offsets int64[n_tx+1], items uint32[nnz] (ascending per
// transaction), terms u64[n], item->tile u32[n], tiles, units, entries
// uint2[E], slabs u32[units x kDenseCap], output (row, col, count) u32.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <chrono>
#include <mutex>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"

using namespace crop;

namespace {

constexpr int kCountThreads = 1024;
constexpr int kCountWarps = kCountThreads / 32;
constexpr uint32_t kDenseCap = 65536;                // dense u16 counters per tile (128 KB)
constexpr size_t kTableBytes = (size_t)kDenseCap * 2;
constexpr uint32_t kHashSlots = 21760;               // u32 keys + u16 counts (127.5 KB)
constexpr uint32_t kHashCap = 14336;                 // max distinct keys per hash tile
constexpr uint32_t kHashHalf = kHashSlots / 2;       // interleaved u16 hash counts
constexpr uint32_t kUnitEntries = 65535;             // entries per unit: u16 counters never wrap
constexpr uint32_t kMaxLen = 8192;                   // longest transaction
constexpr int kBufWords = 512;                       // per-warp staging of transaction suffixes
constexpr size_t kBufBytes = (size_t)kCountWarps * kBufWords * 4;
constexpr int kJobWords = 5;                         // per-lane entry records (shared memory)
constexpr size_t kJobBytes = (size_t)kCountWarps * 32 * kJobWords * 4;
constexpr size_t kCountSmem = kTableBytes + kBufBytes + kJobBytes + 64;
constexpr int kPassThreads = 1024;
constexpr int kChunkTx = 4096;                       // transactions per position-parallel chunk
constexpr size_t kOffBytes = (kChunkTx + 1) * 8;
constexpr uint32_t kStatSmemItems = 24576;           // pass A privatised items (2 x u32, 192 KB)
constexpr uint32_t kTileSmem = 24576;                // route shared tile counters (96 KB)
constexpr uint32_t kStage = 4096;                    // route staging entries per chunk
// pass A packs occ << 32 | terms: a row's terms (<= its transactions' total
// length) and occurrences are both below nnz < 2^32 per job
constexpr int kOccShift = 32;
constexpr uint64_t kOccOne = 1ull << kOccShift;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kUnknown = 0xFFFFFFFEu;       // route: previous tile not known yet
constexpr uint32_t kWinFlag = 0x80000000u;           // item_tile: row is split into windows
constexpr uint32_t kEntFlag = 0x40000000u;           // stream item_info: row counted from entries
constexpr uint32_t kTileMask = 0x3FFFFFFFu;
constexpr uint32_t kScatMaxTx = 2048;             // transactions staged at once (scatter, own pass A)

struct Tile {
  uint32_t row0, row1;  // rows [row0, row1)
  uint32_t c0, c1;      // column window [c0, c1)
  uint32_t mode;        // 0 dense, 1 hash, 2 dense single row counted from entries (stream mode)
  uint32_t nwin;        // first window tile of a split row: #windows; else 0
  uint32_t n_units;
  uint32_t width;       // dense: counters used
  uint64_t slab_base;   // multi-unit dense: first slab
  uint64_t terms;       // planning estimate (all buckets)
};

struct Unit {
  uint32_t tile, local;
};

// Counting-kernel cost of a tile for balancing tile shards across ranks, in
// units of ~half a cycle (measured per-kind rates): 0.8 cycles
// per word of a dense tile, ~5.5 per word of a hash tile, ~1.5 per table slot
// cleared and compacted per unit.
__host__ __device__ __forceinline__ uint64_t tile_cost(const Tile& t, uint32_t hash_room) {
  const uint64_t room = t.mode == 1 ? hash_room : t.width;
  return t.terms * (t.mode == 1 ? 11ull : 2ull) + 3ull * room * (t.n_units ? t.n_units : 1);
}

// Output capacity of a tile: a tile emits at most one entry per counter or
// key and at most one per term (terms are exact except for column windows --
// single rows narrower than the row -- whose terms are only an estimate).
__host__ __device__ __forceinline__ uint64_t tile_out_cap(const Tile& t, uint32_t hash_keys, uint32_t n,
                                                          bool upper) {
  const uint64_t room = t.mode == 1 ? hash_keys : t.width;
  const bool window = t.mode == 0 && t.row1 - t.row0 == 1 && t.width < (upper ? n - 1 - t.row0 : n);
  if (window) return room;
  return t.terms < room ? t.terms : room;
}

__host__ __device__ __forceinline__ uint64_t tri_rowbase(uint64_t r, uint64_t row0, uint64_t n) {
  // sum_{x=row0}^{r-1} (n - 1 - x)
  uint64_t k = r - row0;
  return k * (n - 1) - k * (row0 + r - 1) / 2;
}

// ----------------------------------------------------- position-parallel walk
// A CTA owns chunks of kChunkTx transactions whose offsets are staged in
// shared memory. Each warp takes a contiguous range of item positions and
// walks it 32 positions at a time (lane = position, coalesced loads of
// items[g]); a lane finds its transaction by stepping forward from the
// warp's cursor, so one position costs O(1) shared-memory reads. All O(nnz)
// passes read the input once, coalesced.
struct Pos {
  int64_t base;  // global position of the transaction start
  uint32_t p;    // position inside the transaction
  uint32_t L;    // transaction length
  uint32_t tx;   // chunk-local transaction index
  bool valid;
};

__device__ __forceinline__ int stage_offsets(int64_t* s_off, const int64_t* __restrict__ offsets,
                                             int64_t n_tx, int64_t chunk, int chunk_tx) {
  const int64_t t0 = chunk * chunk_tx;
  const int ntx = (int)(n_tx - t0 < chunk_tx ? n_tx - t0 : chunk_tx);
  for (int t = threadIdx.x; t <= ntx; t += blockDim.x) s_off[t] = offsets[t0 + t];
  __syncthreads();
  return ntx;
}

// Calls body(g, pos, item, tile) for every position of the chunk; all 32
// lanes of a warp execute body together (pos.valid false past the range) so
// body may use warp shuffles. Loads are software-pipelined: the item of
// window w+2 and (with TILE) the item->tile lookup of window w+1 are in
// flight while window w is processed.
template <typename TV> __device__ __forceinline__ TV tv_none();
template <> __device__ __forceinline__ uint32_t tv_none<uint32_t>() { return kNone; }
template <> __device__ __forceinline__ uint2 tv_none<uint2>() { return make_uint2(kNone, 0u); }

template <bool TILE, typename TV = uint32_t, typename Body>
__device__ __forceinline__ void walk_chunk(const int64_t* s_off, int ntx,
                                           const uint32_t* __restrict__ items,
                                           const TV* __restrict__ item_tile, Body&& body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t g_lo = s_off[0], g_hi = s_off[ntx];
  const int64_t per = (((g_hi - g_lo + nw - 1) / nw) + 31) & ~31ll;
  const int64_t w_lo = g_lo + warp * per;
  const int64_t w_hi = min(g_hi, w_lo + per);
  if (w_lo >= w_hi) return;
  int lo = 0, hi = ntx;  // cursor: last t with s_off[t] <= w_lo
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_off[mid] <= w_lo) lo = mid;
    else hi = mid;
  }
  int cur = lo;
  auto ld_item = [&](int64_t g) { return g < w_hi ? __ldg(items + g) : 0u; };
  uint32_t it0 = ld_item(w_lo + lane), it1 = ld_item(w_lo + 32 + lane);
  TV tl0 = tv_none<TV>();
  if (TILE) tl0 = w_lo + lane < w_hi ? __ldg(item_tile + it0) : tv_none<TV>();
  for (int64_t g0 = w_lo; g0 < w_hi; g0 += 32) {
    const int64_t g = g0 + lane;
    const uint32_t it2 = ld_item(g + 64);
    TV tl1 = tv_none<TV>();
    if (TILE) tl1 = g + 32 < w_hi ? __ldg(item_tile + it1) : tv_none<TV>();
    Pos q;
    q.valid = g < w_hi;
    int t = cur;
    if (q.valid)
      while (s_off[t + 1] <= g) ++t;
    q.tx = (uint32_t)t;
    q.base = s_off[t];
    q.p = (uint32_t)(g - q.base);
    q.L = (uint32_t)(s_off[t + 1] - q.base);
    cur = __shfl_sync(0xffffffffu, t, 31);
    body(g, q, it0, tl0);
    it0 = it1;
    it1 = it2;
    tl0 = tl1;
  }
}

// ------------------------------------------------- own-bucket layout (Lemma 1)
// A filtered job owns the bucket interval [start, stop) of kappa. Pair (i, j)
// is own iff (h_row(i) + h_col(j)) mod kappa lies in it, i.e. iff h_col(j)
// lies in row i's circular class window [start - h_row(i), stop - h_row(i))
// mod kappa -- the two windows of scan_sorted (interval.py:125-189). Every
// transaction gets a copy of its items sorted by (h_col, id) (the order of
// bucket_sort_indices, interval.py:70-109), stored as keys
// h_col << idbits | id, so a row's own partners are at most two contiguous
// ranges of that copy, found by binary search: a filtered job reads, routes
// and counts only its own terms (plus, with the triangle filter, the
// window's items not after the row, which it skips like scan_sorted does).
struct OwnArgs {
  const uint32_t* hs;     // (h_col, id)-sorted keys per transaction (same offsets)
  const uint32_t* h_row;
  uint32_t kappa, start, len, idbits, cbits;
  uint32_t* pos_rec;      // per position: own partners | first partner << 16 (single bucket)
};

// lower bound of key in hs[0, L): branch-free steps (predicated adds), the
// same trip count for every lane of a transaction
__device__ __forceinline__ uint32_t hs_lower(const uint32_t* hs, uint32_t L, uint64_t key) {
  uint32_t pos = 0;
  for (uint32_t step = L ? 1u << (31 - __clz(L)) : 0u; step; step >>= 1) {
    const uint32_t q = pos + step;
    if (q <= L && (uint64_t)hs[q - 1] < key) pos = q;
  }
  return pos;
}

// Own window of a row with h_row = hr in one transaction's keys hs[0, L):
// positions [a0, a0 + n1) and (a wrapped window) [0, n2).
__device__ __forceinline__ void own_window(const uint32_t* hs, uint32_t L, uint32_t hr,
                                           const OwnArgs& O, uint32_t& a0, uint32_t& n1, uint32_t& n2) {
  const uint32_t c_lo = O.start >= hr ? O.start - hr : O.start + O.kappa - hr;
  const uint64_t c_hi = (uint64_t)c_lo + O.len;
  a0 = hs_lower(hs, L, (uint64_t)c_lo << O.idbits);
  if (c_hi <= O.kappa) {
    n1 = hs_lower(hs, L, c_hi << O.idbits) - a0;
    n2 = 0;
  } else {
    n1 = L - a0;
    n2 = hs_lower(hs, L, (c_hi - O.kappa) << O.idbits);
  }
}

// own terms of row item i (UPPER: partners with a larger id only)
template <bool UPPER>
__device__ __forceinline__ uint32_t own_count(const uint32_t* hs, uint32_t a0, uint32_t n1,
                                              uint32_t n2, uint32_t i, uint32_t idmask) {
  if (!UPPER) return n1 + n2;
  uint32_t c = 0;
  for (uint32_t k = 0; k < n1; ++k) c += (hs[a0 + k] & idmask) > i;
  for (uint32_t k = 0; k < n2; ++k) c += (hs[k] & idmask) > i;
  return c;
}

// Own partners of row item i in one transaction's keys hs[0, L): the count,
// and, for a single-bucket interval (one class per row: the window is one
// class segment whose ids ascend), the first key position -- the own
// partners are then the contiguous range [src, src + count). General
// intervals return src = kNone (the caller walks the window and filters).
template <bool UPPER>
__device__ __forceinline__ uint32_t own_partners(const uint32_t* hs, uint32_t L, uint32_t i, uint32_t hr,
                                                 const OwnArgs& O, uint32_t idmask, uint32_t& src) {
  if (O.len == 1) {
    const uint32_t c = O.start >= hr ? O.start - hr : O.start + O.kappa - hr;
    const uint64_t ck = (uint64_t)c << O.idbits;
    const uint32_t lo = hs_lower(hs, L, UPPER ? (ck | (i + 1)) : ck);
    const uint32_t hi = hs_lower(hs, L, ck + (1ull << O.idbits));
    src = lo;
    return hi - lo;
  }
  uint32_t a0, n1, n2;
  own_window(hs, L, hr, O, a0, n1, n2);
  src = kNone;
  return own_count<UPPER>(hs, a0, n1, n2, i, idmask);
}

// Longest transaction (sizes the position bands of the own-bucket kernels).
__global__ void k_max_len(const int64_t* __restrict__ offsets, int64_t n_tx, unsigned int* __restrict__ out) {
  uint32_t m = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tx; t += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (uint32_t)(offsets[t + 1] - offsets[t]));
#pragma unroll
  for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Pass A of an own-bucket job, fused with building the (h_col, id)-sorted
// copy. Chunks are the position bands of k_chunk_bounds (<= kOwnStage
// positions). Per band: the items are read coalesced and their keys
// h_col << idbits | id staged in shared memory; each warp sorts its
// transactions there (a register bitonic sort for <= 32 items, a shared
// bitonic sort in a per-warp scratch up to kOwnSortMax, rank counting
// beyond); the sorted band is written back (coalesced) for the scatter, and
// every row occurrence counts its own partners with binary searches on the
// staged keys.
constexpr uint32_t kOwnStage = 8192;        // staged positions per band
constexpr uint32_t kOwnSortMax = 512;       // per-warp bitonic scratch
constexpr uint32_t kOwnStatItems = 8192;    // items with shared-memory counters
template <bool UPPER>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_own_prep(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items,
               uint32_t n_items, const uint32_t* __restrict__ h_col, const uint32_t* __restrict__ bounds,
               uint32_t n_chunks, unsigned long long* __restrict__ stats, uint32_t* __restrict__ hs_out,
               OwnArgs O) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);                       // kScatMaxTx + 1
  uint32_t* s_hs = reinterpret_cast<uint32_t*>(s_off + kScatMaxTx + 1);    // kOwnStage
  uint32_t* s_hr = s_hs + kOwnStage;                                       // row class per position
  uint32_t* s_sort = s_hr + kOwnStage;                                     // 32 x kOwnSortMax
  uint32_t* s_terms = s_sort + (kPassThreads / 32) * kOwnSortMax;
  const uint32_t n_smem = min(n_items, kOwnStatItems);
  uint32_t* s_occ = s_terms + n_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x) {
    s_terms[i] = 0;
    s_occ[i] = 0;
  }
  const uint32_t idmask = O.idbits >= 32 ? 0xFFFFFFFFu : ((1u << O.idbits) - 1u);
  for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint32_t tb0 = bounds[c], tb1 = bounds[c + 1];
    for (uint32_t ta = tb0; ta < tb1; ta += kScatMaxTx) {
      const int ntx = (int)min(kScatMaxTx, tb1 - ta);
      __syncthreads();
      for (int t = threadIdx.x; t <= ntx; t += blockDim.x) s_off[t] = offsets[ta + t];
      __syncthreads();
      const int64_t g_lo = s_off[0];
      const uint32_t npos = (uint32_t)(s_off[ntx] - g_lo);
      // keys and row classes, four gathers of each in flight per thread
      for (uint32_t x0 = threadIdx.x; x0 < npos; x0 += 4 * blockDim.x) {
        uint32_t it[4], hc[4], hr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t x = x0 + k * blockDim.x;
          it[k] = x < npos ? __ldg(items + g_lo + x) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          hc[k] = __ldg(h_col + it[k]);
          hr[k] = __ldg(O.h_row + it[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t x = x0 + k * blockDim.x;
          if (x < npos) {
            s_hs[x] = (hc[k] << O.idbits) | it[k];
            s_hr[x] = hr[k];
          }
        }
      }
      __syncthreads();
      // sort each transaction's keys in place
      uint32_t* sc = s_sort + warp * kOwnSortMax;
      for (int t = warp; t < ntx; t += kPassThreads / 32) {
        const uint32_t b0 = (uint32_t)(s_off[t] - g_lo), L = (uint32_t)(s_off[t + 1] - s_off[t]);
        uint32_t* seg = s_hs + b0;
        if (L <= 32) {
          // stable rank by class (the items ascend with the lane): one ballot
          // per class bit, most significant first. The same ballots give,
          // for this lane's row i, the lanes whose class lies in its own
          // window: its own partners (ids above i: later lanes) and, for a
          // single-bucket interval, the first partner's sorted position --
          // no binary search, no second walk over these positions.
          const bool v = (uint32_t)lane < L;
          const uint32_t k = v ? seg[lane] : 0u;
          const uint32_t cls = k >> O.idbits;
          const uint32_t hr = v ? s_hr[b0 + lane] : 0u;
          const uint32_t c_lo = O.start >= hr ? O.start - hr : O.start + O.kappa - hr;
          const uint64_t c_end = (uint64_t)c_lo + O.len;           // window [c_lo, c_end) mod kappa
          const bool wraps = c_end > O.kappa;
          const uint32_t c_hi = wraps ? (uint32_t)(c_end - O.kappa) : (uint32_t)c_end;
          const uint32_t vm = __ballot_sync(0xffffffffu, v);
          uint32_t eq = vm, lt = 0;
          uint32_t e_lo = vm, m_lo = 0;  // lanes with class == / < c_lo (prefix so far)
          uint32_t e_hi = vm, m_hi = 0;  // lanes with class == / < c_hi
          for (int bt = (int)O.cbits - 1; bt >= 0; --bt) {
            const bool bit = (cls >> bt) & 1u;
            const uint32_t B = __ballot_sync(0xffffffffu, v && bit);
            if (bit) {
              lt += __popc(eq & ~B);
              eq &= B;
            } else {
              eq &= ~B;
            }
            if ((c_lo >> bt) & 1u) {
              m_lo |= e_lo & ~B;
              e_lo &= B;
            } else {
              e_lo &= ~B;
            }
            if ((c_hi >> bt) & 1u) {
              m_hi |= e_hi & ~B;
              e_hi &= B;
            } else {
              e_hi &= ~B;
            }
          }
          if (c_hi >= (1u << O.cbits)) m_hi = vm;  // c_hi == kappa == 2^cbits: every class is below
          const uint32_t r = lt + __popc(eq & ((1u << lane) - 1u));
          __syncwarp();
          if (v) seg[r] = k;
          // own window: classes in [c_lo, c_hi) (or [c_lo, kappa) + [0, c_hi) when it wraps)
          const uint32_t wmask = wraps ? ((vm & ~m_lo) | m_hi) : (m_hi & ~m_lo);
          const uint32_t after = UPPER ? ~((2u << lane) - 1u) : vm;  // lanes 2u << 31 wraps to 0
          const uint32_t cnt = __popc(wmask & after);
          if (v) {
            uint32_t src = 0xFFFFu;
            if (O.len == 1) {  // first own partner: class c_lo's start + its items not after i
              const uint32_t upto = UPPER ? ((2u << lane) - 1u) : 0u;
              src = __popc(m_lo) + __popc(e_lo & upto);
            }
            O.pos_rec[g_lo + b0 + lane] = cnt | (src << 16);
            const uint32_t i = k & idmask;
            if (cnt) {
              if (i < n_smem) {
                atomicAdd(&s_terms[i], cnt);
                atomicAdd(&s_occ[i], 1u);
              } else {
                atomicAdd(&stats[i], kOccOne | cnt);
              }
            }
          }
        } else if (L <= kOwnSortMax) {
          uint32_t P = 64;
          while (P < L) P <<= 1;
          for (uint32_t x = lane; x < P; x += 32) sc[x] = x < L ? seg[x] : kEmpty32;
          __syncwarp();
          for (uint32_t kk = 2; kk <= P; kk <<= 1)
            for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
              for (uint32_t x = lane; x < P; x += 32) {
                const uint32_t y = x ^ j;
                if (y > x) {
                  const uint32_t a = sc[x], bb = sc[y];
                  if ((a > bb) == ((x & kk) == 0)) {
                    sc[x] = bb;
                    sc[y] = a;
                  }
                }
              }
              __syncwarp();
            }
          for (uint32_t x = lane; x < L; x += 32) seg[x] = sc[x];
        } else {
          // rank counting through the scratch, kOwnSortMax keys at a time
          for (uint32_t x0 = 0; x0 < L; x0 += kOwnSortMax) {
            const uint32_t m = min(kOwnSortMax, L - x0);
            uint32_t r[kOwnSortMax / 32];
#pragma unroll
            for (uint32_t q = 0; q < kOwnSortMax / 32; ++q) {
              const uint32_t x = x0 + q * 32 + lane;
              r[q] = 0;
              if (q * 32 + lane < m) {
                const uint32_t kx = seg[x];
                for (uint32_t y = 0; y < L; ++y) r[q] += seg[y] < kx;
              }
            }
            __syncwarp();
            // the ranks of keys past this block still read the original keys:
            // park the block's keys in the scratch, write them after all ranks
            // of the transaction are known is not needed -- ranks are final,
            // so stage the sorted block in the scratch by rank offset
            for (uint32_t q = 0; q < kOwnSortMax / 32; ++q) {
              const uint32_t x = x0 + q * 32 + lane;
              if (q * 32 + lane < m) hs_out[g_lo + b0 + r[q]] = seg[x];
            }
          }
          __syncwarp();
          for (uint32_t x = lane; x < L; x += 32) seg[x] = hs_out[g_lo + b0 + x];
          __threadfence_block();
        }
        __syncwarp();
      }
      __syncthreads();
      for (uint32_t x = threadIdx.x; x < npos; x += blockDim.x) hs_out[g_lo + x] = s_hs[x];
      // transactions of more than 32 items: own windows by binary search on
      // the sorted keys, one warp per transaction (the short ones were done
      // in the sort)
      for (int t = warp; t < ntx; t += kPassThreads / 32) {
        const uint32_t b0 = (uint32_t)(s_off[t] - g_lo), L = (uint32_t)(s_off[t + 1] - s_off[t]);
        if (L <= 32) continue;
        const uint32_t* seg = s_hs + b0;
        for (uint32_t p = lane; p < L; p += 32) {
          const int64_t g = g_lo + b0 + p;
          if (UPPER && p + 1 >= L) {
            O.pos_rec[g] = 0;
            continue;
          }
          const uint32_t i = __ldg(items + g);
          uint32_t src;
          const uint32_t cnt = own_partners<UPPER>(seg, L, i, s_hr[b0 + p], O, idmask, src);
          O.pos_rec[g] = cnt | (src << 16);  // src < 2^16 (kNone for general intervals: 0xFFFF)
          if (cnt == 0) continue;
          if (i < n_smem) {
            atomicAdd(&s_terms[i], cnt);
            atomicAdd(&s_occ[i], 1u);
          } else {
            atomicAdd(&stats[i], kOccOne | cnt);
          }
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x)
    if (s_terms[i])
      atomicAdd(&stats[i], ((unsigned long long)s_occ[i] << kOccShift) | s_terms[i]);
}

// ------------------------------------------------------------- pass A
// Per row item i: terms_i (pairs with i as the row) and occ_i, the number of
// transactions in which i has at least one partner after it (an upper bound
// of the entries it creates). Output packed as occ << kOccShift | terms.
template <bool UPPER>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_item_terms(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items,
                 int64_t n_tx, uint32_t n_items, int chunk_tx, unsigned long long* __restrict__ stats,
                 unsigned int* __restrict__ max_len) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);
  uint32_t* s_terms = reinterpret_cast<uint32_t*>(smem + kOffBytes);
  const uint32_t n_smem = min(n_items, kStatSmemItems);
  uint32_t* s_occ = s_terms + n_smem;
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x) {
    s_terms[i] = 0;
    s_occ[i] = 0;
  }
  uint32_t my_max = 0;
  const int64_t n_chunks = (n_tx + chunk_tx - 1) / chunk_tx;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    __syncthreads();
    const int ntx = stage_offsets(s_off, offsets, n_tx, chunk, chunk_tx);
    walk_chunk<false>(s_off, ntx, items, (const uint32_t*)nullptr, [&](int64_t g, const Pos& q, uint32_t i, uint32_t) {
      if (!q.valid) return;
      my_max = max(my_max, q.L);
      const uint32_t c = UPPER ? q.L - 1 - q.p : q.L;
      if (c == 0) return;
      if (i < n_smem) {
        atomicAdd(&s_terms[i], c);
        atomicAdd(&s_occ[i], 1u);
      } else {
        atomicAdd(&stats[i], kOccOne | c);
      }
    });
  }
  atomicMax(max_len, my_max);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x)
    if (s_terms[i])
      atomicAdd(&stats[i], ((unsigned long long)s_occ[i] << kOccShift) | s_terms[i]);
}

// ------------------------------------------------------------- pass B
// Entries (the work list of a tile), one per run of consecutive positions of
// a transaction whose rows share a tile (UPPER), or per (row, column window
// present) for split rows:
//   UPPER: x = global position of the run's first row, y = len | rows << 16
//          (len = positions from the first row to the end of the transaction)
//   full : x = global position of the transaction start, y = L | p << 16
//          (one row per entry)
// Runs are found with warp shuffles: a lane's tile is compared with its
// neighbours'; a run that leaves the 32-position window is finished with
// loads (rare).
template <bool UPPER, typename EmitRun, typename EmitWin>
__device__ __forceinline__ void route_window(int64_t g, const Pos& q, uint32_t tile_of_g,
                                             const uint32_t* __restrict__ items,
                                             const uint32_t* __restrict__ item_tile,
                                             const Tile* __restrict__ tiles, uint32_t& carry_tile,
                                             EmitRun&& emit_run, EmitWin&& emit_window) {
  // emit_run is called by every lane (warp-uniform) with has = whether this
  // lane starts a run entry; emit_window once per (split row, window) entry.
  const int lane = threadIdx.x & 31;
  uint32_t tv = kNone;
  if (q.valid) {
    tv = tile_of_g;
    if (UPPER && q.p + 1 >= q.L) tv = kNone;  // the last item has no partner after it
  }
  // previous position's tile (same transaction only)
  uint32_t prev = __shfl_up_sync(0xffffffffu, tv, 1);
  if (lane == 0) {
    prev = carry_tile;
    if (prev == kUnknown && q.valid && q.p > 0) prev = item_tile[items[g - 1]];
  }
  if (q.p == 0) prev = kNone;
  const uint32_t next_tv = __shfl_down_sync(0xffffffffu, tv, 1);
  const uint32_t next_p = __shfl_down_sync(0xffffffffu, q.p, 1);
  carry_tile = __shfl_sync(0xffffffffu, tv, 31);
  bool has = false;
  uint32_t rt = 0, rx = 0, ry = 0;
  if (tv != kNone) {
    if (tv & kWinFlag) {  // split row: one entry per column window present
      const uint32_t tile = tv & ~kWinFlag;
      const Tile t0 = tiles[tile];
      const uint32_t lo = t0.c0;
      uint32_t last_w = kNone;
      for (uint32_t p = UPPER ? q.p + 1 : 0; p < q.L; ++p) {
        const uint32_t j = items[q.base + p];
        if (j < lo) continue;
        const uint32_t w = (j - lo) / kDenseCap;
        if (w >= t0.nwin) break;
        if (w != last_w) {
          if (UPPER) emit_window(true, tile + w, (uint32_t)g, (q.L - q.p) | (1u << 16));
          else emit_window(true, tile + w, (uint32_t)q.base, q.L | (q.p << 16));
          last_w = w;
        }
      }
    } else if (!UPPER) {
      has = true;
      rt = tv;
      rx = (uint32_t)q.base;
      ry = q.L | (q.p << 16);
    } else if (prev != tv) {  // first row of its run
      uint32_t p1 = q.p + 1;
      const bool next_known = lane < 31 && next_p == q.p + 1;
      if (!(next_known && next_tv != tv))  // the run may continue: extend with loads
        while (p1 + 1 < q.L && item_tile[items[q.base + p1]] == tv) ++p1;
      has = true;
      rt = tv;
      rx = (uint32_t)g;
      ry = (q.L - q.p) | ((p1 - q.p) << 16);
    }
  }
  emit_run(has, rt, rx, ry);
}

// One walk per chunk of chunk_tx transactions: entries are staged in shared
// memory with per-tile counts (only the tiles a chunk touches are listed),
// one global range is claimed per touched tile, then the staged entries are
// scattered into their tiles' ranges. Tiles beyond the shared counters and
// entries beyond the staging buffer take per-entry global atomics (rare).
template <bool UPPER>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_route(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items, int64_t n_tx,
            int chunk_tx, const uint32_t* __restrict__ item_tile, const Tile* __restrict__ tiles,
            uint32_t n_tiles, unsigned long long* __restrict__ tile_cursor,
            const unsigned long long* __restrict__ tile_end, uint2* __restrict__ entries,
            uint32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);
  uint2* s_stage = reinterpret_cast<uint2*>(smem + (size_t)(chunk_tx + 1) * 8);
  uint32_t* s_stage_tile = reinterpret_cast<uint32_t*>(s_stage + kStage);
  uint32_t* s_touched = s_stage_tile + kStage;
  uint32_t* s_misc = s_touched + kStage;  // [0] staged, [1] touched
  uint32_t* s_cnt = s_misc + 4;           // per shared tile: count, then next position
  const uint32_t ns = min(n_tiles, kTileSmem);
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  auto global_put = [&](uint32_t tile, uint2 v) {
    const unsigned long long pos = atomicAdd(&tile_cursor[tile], 1ull);
    if (pos < tile_end[tile]) entries[pos] = v;
    else *overflow = 1u;
  };
  auto put = [&](uint32_t slot, uint32_t tile, uint32_t x, uint32_t y) {
    if (slot >= kStage || tile >= ns) {
      if (slot < kStage) s_stage_tile[slot] = kNone;  // hole
      global_put(tile, make_uint2(x, y));
      return;
    }
    s_stage_tile[slot] = tile;
    s_stage[slot] = make_uint2(x, y);
    if (atomicAdd(&s_cnt[tile], 1u) == 0) s_touched[atomicAdd(&s_misc[1], 1u)] = tile;
  };
  // run entries: at most one per lane per window -> one staging atomic per warp
  auto stage_run = [&](bool has, uint32_t tile, uint32_t x, uint32_t y) {
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(&s_misc[0], (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (has) put(base + __popc(m & ((1u << lane) - 1u)), tile, x, y);
  };
  auto stage_window = [&](bool, uint32_t tile, uint32_t x, uint32_t y) {
    put(atomicAdd(&s_misc[0], 1u), tile, x, y);
  };
  const int64_t n_chunks = (n_tx + chunk_tx - 1) / chunk_tx;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_misc[0] = 0;
      s_misc[1] = 0;
    }
    const int ntx = stage_offsets(s_off, offsets, n_tx, chunk, chunk_tx);
    uint32_t carry = kUnknown;
    walk_chunk<true>(s_off, ntx, items, item_tile, [&](int64_t g, const Pos& q, uint32_t, uint32_t tile) {
      route_window<UPPER>(g, q, tile, items, item_tile, tiles, carry, stage_run, stage_window);
    });
    __syncthreads();
    const uint32_t n_stage = min(s_misc[0], kStage), n_touch = s_misc[1];
    for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) {
      const uint32_t t = s_touched[k];
      s_cnt[t] = (uint32_t)atomicAdd(&tile_cursor[t], (unsigned long long)s_cnt[t]);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_stage; k += blockDim.x) {
      const uint32_t t = s_stage_tile[k];
      if (t == kNone) continue;
      entries[atomicAdd(&s_cnt[t], 1u)] = s_stage[k];
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) s_cnt[s_touched[k]] = 0;
  }
}

// tile_entries[t] = final cursor - base (entries actually routed)
__global__ void k_tile_entries(const unsigned long long* __restrict__ cursor,
                               const unsigned long long* __restrict__ base, uint32_t n,
                               uint32_t* __restrict__ out) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    out[t] = (uint32_t)(cursor[t] - base[t]);
}

// ------------------------------------------------------------- count
struct CountArgs {
  const uint32_t* items;
  const Tile* tiles;
  const Unit* units;
  uint32_t n_units;
  const unsigned long long* tile_ebase;  // exclusive scan of entries per tile
  const uint32_t* tile_entries;
  const uint2* entries;
  unsigned int* unit_counter;
  uint32_t n_items;
  uint32_t col_bits;
  // bucket filter
  uint32_t kappa, start, stop;
  const uint32_t* h_row;
  const uint32_t* h_col;
  // output
  uint32_t* out_row;
  uint32_t* out_col;
  uint32_t* out_count;
  unsigned long long* out_n;
  uint64_t out_cap;  // output capacity (entries); claims beyond it are not written
  uint32_t* slabs;  // kHalf words (two interleaved u16 counters) per unit
  unsigned int* tile_done;
  unsigned long long* dbg;  // optional: per-kind [cycles count, cycles emit, units, entries]
};

__device__ __forceinline__ uint32_t lower_bound_items(const uint32_t* __restrict__ a, uint32_t lo,
                                                      uint32_t hi, uint32_t key) {
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Block-wide exclusive scan of one value per thread (blockDim a multiple of 32).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = warp_incl_scan(v);
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
    uint32_t xi = warp_incl_scan(x);
    s_warp[lane] = xi - x;
    if (lane == 31) s_warp[32] = xi;
  }
  __syncthreads();
  uint32_t r = s_warp[w] + incl - v;
  total = s_warp[32];
  __syncthreads();
  return r;
}

// Persistent CTAs pull units (tiles or parts of split tiles) in order. A
// warp takes a batch of up to 32 entries and
//   1. stages every entry's words -- [row item(s) | column items] -- in its
//      shared buffer with one flattened, coalesced copy (lane -> word via a
//      32-bit boundary mask from __reduce_or_sync + popc);
//   2. expands the entries into ROW-JOBS (one per row of a run), and
//   3. flattens the row-jobs' pairs across lanes: every pair is then two
//      shared-memory loads (row item, column item) and one shared-memory
//      atomic on a u16 counter (two counters per 32-bit word; a unit holds
//      <= 65,535 entries, so no counter can wrap).
// Entries longer than the buffer (> 512 staged words, i.e. transactions
// longer than 512 items) take a direct path from global memory.
// A tile split over several units is reduced by the last unit to finish:
// the others leave their u16 counters in a slab (L2-resident by then) and the
// last one sums them on the fly while compacting.
enum TileKind { kDenseRow = 0, kDenseWindow = 1, kDenseMulti = 2, kHash = 3 };

struct WarpSmem {
  uint32_t* buf;  // staged words
  uint32_t *off, *hp, *cs, *m, *R;  // per-entry records of the current batch
};

// boundary-mask lane -> owner for flattened index t0 + lane, given each lane's
// inclusive end `incl` (warp-collective)
__device__ __forceinline__ uint32_t owner_step(uint32_t incl, uint32_t t0, uint32_t& owner_base) {
  const int lane = threadIdx.x & 31;
  const uint32_t bit = (incl > t0 && incl < t0 + 32) ? (1u << (incl - t0)) : 0u;
  const uint32_t B = __reduce_or_sync(0xffffffffu, bit);
  const uint32_t at_end = __reduce_add_sync(0xffffffffu, (incl == t0 + 32) ? 1u : 0u);
  const uint32_t owner = owner_base + __popc(B & (0xffffffffu >> (31 - lane)));
  owner_base += __popc(B) + at_end;
  return owner;
}

// u16 counters, two per 32-bit word, interleaved across the two halves of
// the table (slot s lives in word s mod 32768, half s / 32768) so that
// neighbouring slots -- consecutive columns of one row -- never share a word
// (no same-address conflicts inside a warp's atomic).
constexpr uint32_t kHalf = kDenseCap / 2;

__device__ __forceinline__ void bump16(uint32_t* words, uint32_t slot) {
  atomicAdd(&words[slot & (kHalf - 1)], 1u << ((slot / kHalf) << 4));
}
__device__ __forceinline__ uint32_t read16(const uint32_t* words, uint32_t slot) {
  return (words[slot & (kHalf - 1)] >> ((slot / kHalf) << 4)) & 0xFFFFu;
}

template <int KIND, bool UPPER, bool FILTER>
struct Counter {
  const CountArgs& A;
  const Tile& T;
  uint32_t* table;  // dense: u16 counters; hash: u32 keys
  uint32_t* hcnt;   // hash: u16 counts (interleaved like the dense table)
  // per-row constant: dense -> slot = base + j; hash -> key = base | j
  __device__ __forceinline__ uint32_t row_base(uint32_t i) const {
    if (KIND == kDenseRow) return UPPER ? 0u - (T.row0 + 1) : 0u;
    if (KIND == kDenseWindow) return 0u - T.c0;
    if (KIND == kDenseMulti) {
      // slots before row i: k*w0 - k(k-1)/2 with k = i - row0, w0 = row0's
      // width; exact in 32-bit modular arithmetic since the result < 2^16
      const uint32_t k = i - T.row0;
      if (!UPPER) return k * A.n_items;
      const uint32_t w0 = A.n_items - 1 - T.row0;
      const uint32_t tri = (uint32_t)(((unsigned long long)k * (k - 1)) >> 1);
      return k * w0 - tri - i - 1;
    }
    return (i - T.row0) << A.col_bits;
  }
  __device__ __forceinline__ void operator()(uint32_t i, uint32_t base, uint32_t j) const {
    if (FILTER) {
      uint32_t b = A.h_row[i] + A.h_col[j];
      if (b >= A.kappa) b -= A.kappa;
      if (b < A.start || b >= A.stop) return;
    }
    if (KIND != kHash) {
      bump16(table, base + j);
      return;
    }
    const uint32_t key = base | j;
    uint32_t s = __umulhi(mix32(key), kHashSlots);
    for (;;) {
      const uint32_t k = table[s];
      if (k == key) break;
      if (k == kEmpty32) {
        const uint32_t old = atomicCAS(&table[s], kEmpty32, key);
        if (old == kEmpty32 || old == key) break;
      }
      if (++s == kHashSlots) s = 0;
    }
    const bool hi = s >= kHashHalf;
    atomicAdd(&hcnt[hi ? s - kHashHalf : s], hi ? 0x10000u : 1u);
  }
};

// Direct path for one long entry (staged length > kBufWords): lanes stride
// over each row's columns, loading from global memory.
template <typename Cnt>
__device__ void count_long_entry(const uint32_t* __restrict__ items, uint32_t hp, uint32_t cs,
                                 uint32_t m, uint32_t R, const Cnt& cnt) {
  const int lane = threadIdx.x & 31;
  for (uint32_t r = 0; r < R; ++r) {
    const uint32_t i = items[r == 0 ? hp : cs + r - 1];
    const uint32_t base = cnt.row_base(i);
    for (uint32_t c = r + 1 + lane; c < m; c += 32) cnt(i, base, items[cs + c - 1]);
  }
}

// Flattened path for tiles whose rows are short (single-row and hash tiles:
// c2's shape): the pairs of 32 entries are spread across the lanes (entry of
// a lane found with a 32-bit boundary mask, __reduce_or_sync + popc) and the
// column items come straight from global memory through a three-stage
// software pipeline.
template <int KIND, bool UPPER, bool FILTER>
__device__ __forceinline__ void count_entries_flat(const CountArgs& A, const Tile& T, uint64_t e0,
                                                   uint64_t e1, const WarpSmem& W,
                                                   uint32_t* table, uint32_t* hcnt,
                                                   unsigned int* s_next) {
  const int lane = threadIdx.x & 31;
  const uint32_t* __restrict__ items = A.items;
  const Counter<KIND, UPPER, FILTER> cnt{A, T, table, hcnt};
  constexpr bool SINGLE = KIND == kDenseRow || KIND == kDenseWindow;
  constexpr bool MULTI = UPPER && KIND == kHash;  // UPPER hash runs may hold several rows
  const uint32_t base_single = SINGLE ? cnt.row_base(T.row0) : 0;
  uint32_t* J_delta = W.off;
  uint32_t* J_excl = W.hp;
  uint32_t* J_item = W.cs;
  uint32_t* J_x = W.m;
  uint32_t* J_y = W.R;
  // the next batch's entry descriptors are loaded while this one is counted
  auto grab = [&]() -> uint64_t {
    uint32_t bidx = 0;
    if (lane == 0) bidx = atomicAdd(s_next, 1u);
    bidx = __shfl_sync(0xffffffffu, bidx, 0);
    return e0 + (uint64_t)bidx * 32;
  };
  uint64_t nb = grab();
  uint2 nen = make_uint2(0, 0);
  if (nb + lane < e1) nen = A.entries[nb + lane];
  for (;;) {
    const uint64_t eb_w = nb;
    if (eb_w >= e1) break;
    const uint2 en = nen;
    nb = grab();
    if (nb + lane < e1) nen = A.entries[nb + lane];
    const uint64_t e = eb_w + lane;
    uint32_t cn = 0, x = 0, y = 0, first = 0, ri = 0;
    if (e < e1) {
      x = en.x;
      y = en.y;
      if (UPPER) {
        const uint32_t len = y & 0xFFFFu, rows = y >> 16;
        if (!SINGLE) ri = items[x];
        if (KIND == kDenseWindow) {
          first = lower_bound_items(items, x + 1, x + len, T.c0);
          cn = lower_bound_items(items, first, x + len, T.c1) - first;
        } else {
          first = x + 1;
          cn = rows * (len - 1) - rows * (rows - 1) / 2;
        }
      } else {
        const uint32_t L = y & 0xFFFFu, p = y >> 16;
        ri = items[x + p];
        if (KIND == kDenseWindow) {
          first = lower_bound_items(items, x, x + L, T.c0);
          cn = lower_bound_items(items, first, x + L, T.c1) - first;
        } else {
          first = x;
          cn = L;
        }
      }
    }
    const uint32_t incl = warp_incl_scan(cn);
    J_delta[lane] = first - (incl - cn);
    J_excl[lane] = incl - cn;
    J_item[lane] = ri;
    if (MULTI) {
      J_x[lane] = x;
      J_y[lane] = y;
    }
    const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    uint32_t owner_base = 0;
    auto locate = [&](uint32_t t, uint32_t o, uint32_t& i, uint32_t& jpos) {
      if (MULTI) {
        const uint32_t yy = J_y[o];
        if ((yy >> 16) > 1) {
          uint32_t loc = t - J_excl[o], w = (yy & 0xFFFFu) - 1, k = 0;
          while (loc >= w) {
            loc -= w;
            ++k;
            --w;
          }
          const uint32_t xx = J_x[o];
          i = k ? items[xx + k] : J_item[o];
          jpos = xx + k + 1 + loc;
          return;
        }
      }
      i = SINGLE ? T.row0 : J_item[o];
      jpos = t + J_delta[o];
    };
    uint32_t i0 = 0, j0 = 0, i1 = 0, j1 = 0, jp;
    {
      const uint32_t o = owner_step(incl, 0, owner_base);  // warp-collective
      if (lane < S) {
        locate(lane, o, i0, jp);
        j0 = items[jp];
      }
    }
    if (32 < S) {
      const uint32_t o = owner_step(incl, 32, owner_base);
      if (32 + lane < S) {
        locate(32 + lane, o, i1, jp);
        j1 = items[jp];
      }
    }
    for (uint32_t t0 = 0; t0 < S; t0 += 32) {
      uint32_t i2 = 0, j2 = 0;
      if (t0 + 64 < S) {  // warp-uniform
        const uint32_t o = owner_step(incl, t0 + 64, owner_base);
        if (t0 + 64 + lane < S) {
          locate(t0 + 64 + lane, o, i2, jp);
          j2 = items[jp];
        }
      }
      if (t0 + lane < S) cnt(i0, SINGLE ? base_single : cnt.row_base(i0), j0);
      i0 = i1;
      j0 = j1;
      i1 = i2;
      j1 = j2;
    }
    __syncwarp();
  }
}

template <int KIND, bool UPPER, bool FILTER>
__device__ __forceinline__ void count_entries(const CountArgs& A, const Tile& T, uint64_t e0,
                                              uint64_t e1, const WarpSmem& W, uint32_t* table,
                                              uint32_t* hcnt, unsigned int* s_next) {
  const int lane = threadIdx.x & 31;
  const uint32_t* __restrict__ items = A.items;
  const Counter<KIND, UPPER, FILTER> cnt{A, T, table, hcnt};
  constexpr bool WINDOWED = KIND == kDenseWindow;
  for (;;) {
    // warps take batches of 32 entries dynamically (no tail imbalance)
    uint32_t bidx = 0;
    if (lane == 0) bidx = atomicAdd(s_next, 1u);
    bidx = __shfl_sync(0xffffffffu, bidx, 0);
    const uint64_t eb_w = e0 + (uint64_t)bidx * 32;
    if (eb_w >= e1) break;
    const uint64_t e = eb_w + lane;
    // entry -> staged words: w0 = items[hp], w1.. = items[cs ..], m words, R rows
    uint32_t hp = 0, cs = 0, m = 0, R = 0;
    if (e < e1) {
      const uint2 en = A.entries[e];
      if (UPPER) {
        const uint32_t len = en.y & 0xFFFFu;
        hp = en.x;
        cs = en.x + 1;
        R = en.y >> 16;
        if (WINDOWED) {
          cs = lower_bound_items(items, en.x + 1, en.x + len, T.c0);
          m = 1 + lower_bound_items(items, cs, en.x + len, T.c1) - cs;
        } else {
          m = len;
        }
      } else {
        const uint32_t L = en.y & 0xFFFFu, p = en.y >> 16;
        hp = en.x + p;
        cs = WINDOWED ? lower_bound_items(items, en.x, en.x + L, T.c0) : en.x;
        m = 1 + (WINDOWED ? lower_bound_items(items, cs, en.x + L, T.c1) - cs : L);
        R = 1;
      }
    }
    // long entries (more words than the buffer) take the direct path
    const bool is_long = m > (uint32_t)kBufWords;
    uint32_t long_mask = __ballot_sync(0xffffffffu, is_long);
    while (long_mask) {
      const int l = __ffs(long_mask) - 1;
      long_mask &= long_mask - 1;
      count_long_entry(items, __shfl_sync(0xffffffffu, hp, l), __shfl_sync(0xffffffffu, cs, l),
                       __shfl_sync(0xffffffffu, m, l), __shfl_sync(0xffffffffu, R, l), cnt);
    }
    // compact the remaining entries into lanes [0, ne) (every staged entry
    // has m >= 2 words and every row >= 1 pair, so the boundary masks below
    // never see empty ranges)
    const bool keep = m > 0 && !is_long;
    const uint32_t kmask = __ballot_sync(0xffffffffu, keep);
    const int ne = __popc(kmask);
    if (keep) {
      const int r = __popc(kmask & ((1u << lane) - 1u));
      W.hp[r] = hp;
      W.cs[r] = cs;
      W.m[r] = m;
      W.R[r] = R;
    }
    __syncwarp();
    hp = lane < ne ? W.hp[lane] : 0;
    cs = lane < ne ? W.cs[lane] : 0;
    m = lane < ne ? W.m[lane] : 0;
    R = lane < ne ? W.R[lane] : 0;
    __syncwarp();
    // sub-batches of lanes whose staged words fit the buffer
    const uint32_t m_incl = warp_incl_scan(m);
    const uint32_t pr = R * (m - 1) - R * (R - 1) / 2;  // pairs of the entry
    uint32_t done = 0;  // staged words of earlier sub-batches
    int l0 = 0;
    while (l0 < ne) {
      const uint32_t fits = __ballot_sync(0xffffffffu, lane >= l0 && lane < ne &&
                                                           m_incl - done <= (uint32_t)kBufWords);
      const int l1 = 32 - __clz(fits);  // fits always holds lane l0 (m <= kBufWords)
      const bool in = lane >= l0 && lane < l1;
      // lane group size G from the mean row length of the sub-batch
      const uint32_t sumP = __reduce_add_sync(0xffffffffu, in ? pr : 0u);
      const uint32_t sumR = __reduce_add_sync(0xffffffffu, in ? R : 0u);
      const uint32_t meanP = sumP / (sumR ? sumR : 1u);
      const int G = meanP >= 24 ? 32 : meanP >= 12 ? 16 : meanP >= 6 ? 8 : 4;
      const int NG = 32 / G, grp = lane / G, gl = lane % G;
      if (in) {
        const int r = lane - l0;
        W.off[r] = m_incl - done - m;
        W.hp[r] = hp;
        W.cs[r] = cs;
        W.m[r] = m;
        W.R[r] = R;
      }
      __syncwarp();
      const int ns = l1 - l0;
      // 1. stage each entry's words (asynchronous global -> shared copies)
      for (int q = grp; q < ns; q += NG) {
        const uint32_t qo = W.off[q], qh = W.hp[q], qc = W.cs[q], qm = W.m[q];
        for (uint32_t k = gl; k < qm; k += G) {
          const uint32_t* src_ptr = items + (k == 0 ? qh : qc + k - 1);
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(W.buf + qo + k);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src_ptr));
        }
      }
      asm volatile("cp.async.wait_all;\n" ::);
      __syncwarp();
      // 2. every row of every entry: G lanes stride over its columns;
      //    one shared load and one shared atomic per pair
      for (int q = grp; q < ns; q += NG) {
        const uint32_t qo = W.off[q], qm = W.m[q], qR = W.R[q];
        for (uint32_t r = 0; r < qR; ++r) {
          const uint32_t i = W.buf[qo + r];
          const uint32_t base = cnt.row_base(i);
          const uint32_t* cols = W.buf + qo + r + 1;
          const uint32_t nc = qm - 1 - r;
          uint32_t c = gl;
          for (; c + G < nc; c += 2 * G) {
            const uint32_t ja = cols[c], jb = cols[c + G];
            cnt(i, base, ja);
            cnt(i, base, jb);
          }
          if (c < nc) cnt(i, base, cols[c]);
        }
      }
      __syncwarp();
      done = __shfl_sync(0xffffffffu, m_incl, l1 - 1);
      l0 = l1;
    }
  }
}

template <bool UPPER, bool FILTER>
__global__ void __launch_bounds__(kCountThreads, 1) k_count(CountArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* table = reinterpret_cast<uint32_t*>(smem);  // dense u16 counters / hash keys
  uint32_t* hcnt = table + kHashSlots;                   // hash u16 counts
  uint32_t* bufs = reinterpret_cast<uint32_t*>(smem + kTableBytes);
  uint32_t* job = reinterpret_cast<uint32_t*>(smem + kTableBytes + kBufBytes);
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + kTableBytes + kBufBytes + kJobBytes);
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_base;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem W;
  W.buf = bufs + warp * kBufWords;
  W.off = job + warp * 32 * kJobWords;
  W.hp = W.off + 32;
  W.cs = W.hp + 32;
  W.m = W.cs + 32;
  W.R = W.m + 32;
  const uint32_t n = A.n_items;

  for (;;) {
    if (threadIdx.x == 0) s_misc[0] = atomicAdd(A.unit_counter, 1u);
    __syncthreads();
    const uint32_t u = s_misc[0];
    __syncthreads();
    if (u >= A.n_units) break;
    const Unit unit = A.units[u];
    const Tile T = A.tiles[unit.tile];
    const uint64_t E = A.tile_entries[unit.tile];
    const uint64_t eb = A.tile_ebase[unit.tile];
    const uint64_t e0 = eb + E * unit.local / T.n_units;
    const uint64_t e1 = eb + E * (unit.local + 1) / T.n_units;
    const bool dense = T.mode == 0;
    const bool single_row = T.row1 - T.row0 == 1;
    const bool windowed = single_row && (T.c0 != 0 || T.c1 != n);
    const uint32_t width = T.width;
    const int kind = !dense ? kHash : windowed ? kDenseWindow : single_row ? kDenseRow : kDenseMulti;

    if (dense) {  // interleaved halves: clear the whole table
      uint4* t4 = reinterpret_cast<uint4*>(table);
      for (uint32_t s = threadIdx.x; s < kHalf / 4; s += kCountThreads)
        t4[s] = make_uint4(0, 0, 0, 0);
    } else {
      for (uint32_t s = threadIdx.x; s < kHashSlots; s += kCountThreads) table[s] = kEmpty32;
      for (uint32_t s = threadIdx.x; s < kHashHalf; s += kCountThreads) hcnt[s] = 0;
    }
    if (threadIdx.x == 0) s_misc[2] = 0;  // batch counter of this unit
    __syncthreads();
    const long long dbg_t0 = A.dbg ? clock64() : 0;

    switch (kind) {
      case kDenseRow:
        count_entries_flat<kDenseRow, UPPER, FILTER>(A, T, e0, e1, W, table, hcnt, s_misc + 2);
        break;
      case kDenseWindow:
        count_entries_flat<kDenseWindow, UPPER, FILTER>(A, T, e0, e1, W, table, hcnt, s_misc + 2);
        break;
      case kDenseMulti:
        count_entries<kDenseMulti, UPPER, FILTER>(A, T, e0, e1, W, table, hcnt, s_misc + 2);
        break;
      default:
        count_entries_flat<kHash, UPPER, FILTER>(A, T, e0, e1, W, table, hcnt, s_misc + 2);
        break;
    }
    __syncthreads();

    const long long dbg_t1 = A.dbg ? clock64() : 0;
    bool emit_now = true, reduce = false;
    const uint32_t* slab = nullptr;
    if (dense && T.n_units > 1) {
      // leave this unit's counters in its slab; the last unit sums them
      uint4* dst = reinterpret_cast<uint4*>(A.slabs + (T.slab_base + unit.local) * kHalf);
      const uint4* src = reinterpret_cast<const uint4*>(table);
      for (uint32_t s = threadIdx.x; s < kHalf / 4; s += kCountThreads) dst[s] = src[s];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_misc[1] = atomicAdd(&A.tile_done[unit.tile], 1u) == T.n_units - 1;
      __syncthreads();
      emit_now = s_misc[1] != 0;
      reduce = emit_now;
      if (reduce) __threadfence();
      slab = A.slabs + T.slab_base * kHalf;
    }
    if (emit_now) {
      auto count_at = [&](uint32_t s) -> uint32_t {
        if (!dense) return s >= kHashHalf ? hcnt[s - kHashHalf] >> 16 : hcnt[s] & 0xFFFFu;
        uint32_t c = read16(table, s);
        if (reduce) {
          const uint32_t wi = s & (kHalf - 1), sh = (s / kHalf) << 4;
          for (uint32_t v = 0; v < T.n_units; ++v)
            if (v != unit.local) c += (__ldcg(slab + (uint64_t)v * kHalf + wi) >> sh) & 0xFFFFu;
        }
        return c;
      };
      // compact non-zero counters: warp w owns a contiguous slot range
      const uint32_t slots = dense ? width : kHashSlots;
      const uint32_t per_warp = (slots + kCountWarps - 1) / kCountWarps;
      const uint32_t s_lo = min(slots, warp * per_warp), s_hi = min(slots, s_lo + per_warp);
      uint32_t mine = 0;
      for (uint32_t s = s_lo + lane; s < s_hi; s += 32) mine += count_at(s) != 0;
      mine = warp_sum(mine);
      uint32_t total;
      uint32_t wbase = block_excl_scan(lane == 0 ? mine : 0, s_warp, total);
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (threadIdx.x == 0) s_base = atomicAdd(A.out_n, (unsigned long long)total);
      __syncthreads();
      uint64_t pos = s_base + wbase;
      // past the output capacity: claim only (the host sees n > capacity)
      const bool fits = s_base + total <= A.out_cap;
      for (uint32_t s0 = s_lo; fits && s0 < s_hi; s0 += 32) {
        const uint32_t s = s0 + lane;
        uint32_t c = 0, i = 0, j = 0;
        if (s < s_hi) {
          c = count_at(s);
          if (c) {
            if (!dense) {
              const uint32_t key = table[s];
              i = T.row0 + (key >> A.col_bits);
              j = key & ((1u << A.col_bits) - 1u);
            } else if (windowed) {
              i = T.row0;
              j = s + T.c0;
            } else if (single_row) {
              i = T.row0;
              j = UPPER ? s + i + 1 : s;
            } else if (UPPER) {
              uint32_t lo = T.row0, hi = T.row1;  // last row with rowbase <= s
              while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (tri_rowbase(mid, T.row0, n) <= s) lo = mid;
                else hi = mid;
              }
              i = lo;
              j = (uint32_t)(s - tri_rowbase(i, T.row0, n)) + i + 1;
            } else {
              i = T.row0 + s / n;
              j = s % n;
            }
          }
        }
        const uint32_t mk = __ballot_sync(0xffffffffu, c != 0);
        if (c) {
          const uint64_t o = pos + __popc(mk & ((1u << lane) - 1u));
          A.out_row[o] = i;
          A.out_col[o] = j;
          A.out_count[o] = c;
        }
        pos += __popc(mk);
      }
    }
    __syncthreads();
    if (A.dbg && threadIdx.x == 0) {
      atomicAdd(&A.dbg[kind * 4 + 0], (unsigned long long)(dbg_t1 - dbg_t0));
      atomicAdd(&A.dbg[kind * 4 + 1], (unsigned long long)(clock64() - dbg_t1));
      atomicAdd(&A.dbg[kind * 4 + 2], 1ull);
      atomicAdd(&A.dbg[kind * 4 + 3], (unsigned long long)(e1 - e0));
    }
  }
}

// ============================================================ stream mode
// When rows are short (mean pairs per row occurrence <= kStreamMeanMax:
// BASELINE configs 1-3), the router writes every pair as one 32-bit WORD
// into its tile's stream -- the table slot (dense tiles) or the key (hash
// tiles) -- and the counter reads the streams fully coalesced: one load and
// one shared-memory atomic per term, exactly SURVEY.md §8(d)'s 8 B/term
// model. The table is 57,344 u32 counters (224 KB), so c2's rows (50K
// columns) need no windows and no counter can wrap.
constexpr uint32_t kStreamDenseCap = 57344;
// Counting tables use half an SM's shared memory so two units run per SM
// (one unit's clearing and compaction overlap the other's counting): dense
// tables hold 16-bit counters, slot s in word s mod kSHalf, half s / kSHalf
// (so neighbouring columns never share a word), <= 65,535 row occurrences
// per unit keep them from wrapping; hash tables 14,336 64-bit slots.
constexpr uint32_t kSHalf = kStreamDenseCap / 2;  // 28672 words = 112 KB
constexpr int kSCThreads = 512;                     // count kernel threads (2 CTAs / SM)
constexpr int kSCWarps = kSCThreads / 32;
constexpr uint32_t kStreamUnitOcc = 65535;
constexpr uint32_t kStreamHashSlots = 14336;
constexpr uint32_t kSparseWindowWords = 7168;  // <= half the hash slots: load <= 1/2

// Stream-mode hash tiles size their table from their distinct-key bound
// (load <= 1/2, multiple of 256 slots, at most kStreamHashSlots); the slot
// count is kept in Tile::width. Small tiles then clear and compact little.
__host__ __device__ __forceinline__ uint32_t stream_hash_slots(uint64_t key_bound) {
  uint64_t s = (2 * key_bound + 255) & ~255ull;
  if (s < 1024) s = 1024;
  return (uint32_t)(s < kStreamHashSlots ? s : kStreamHashSlots);
}
constexpr uint32_t kStreamHashCap = 9216;
constexpr size_t kStreamSmem = (size_t)kSHalf * 4 + 64;

__device__ __forceinline__ void bump_half(uint32_t* t32, uint32_t slot) {
  const uint32_t hi = slot >= kSHalf;
  atomicAdd(&t32[slot - hi * kSHalf], 1u << (hi << 4));
}
constexpr uint32_t kStreamMeanMax = 64;

// bump_half for a unit that holds more than 65,535 words: a counter can only
// wrap there if one (row, column) pair occurs that often in the unit's word
// range (the planner bounds a unit's ROW OCCURRENCES on average, not per
// range), so the returning atomic checks the half it bumped and raises the
// job's overflow flag; the caller re-plans with CROP_PAIRS_SAFE_UNITS.
__device__ __forceinline__ void bump_half_checked(uint32_t* t32, uint32_t slot, uint32_t* flag) {
  const uint32_t hi = slot >= kSHalf;
  const uint32_t sh = hi << 4;
  const uint32_t old = atomicAdd(&t32[slot - hi * kSHalf], 1u << sh);
  if (((old >> sh) & 0xFFFFu) == 0xFFFFu) atomicOr(flag, 1u);
}

// per-row constant of the word of (i, j) in tile T: dense word = base + j,
// hash word = base | j
__host__ __device__ __forceinline__ uint32_t stream_base(const Tile& T, uint32_t i, uint32_t n,
                                                         uint32_t col_bits, bool upper) {
  if (T.mode == 1) return (i - T.row0) << col_bits;
  if (T.row1 - T.row0 == 1) return 0u - T.c0;  // single row: slot = j - first column
  const uint32_t k = i - T.row0;
  if (!upper) return k * n;
  const uint32_t w0 = n - 1 - T.row0;
  return k * w0 - (uint32_t)(((unsigned long long)k * (k - 1)) >> 1) - i - 1;
}

struct StreamRouteArgs {
  const int64_t* offsets;
  const uint32_t* items;
  int64_t n_tx;
  const uint2* item_info;  // {tile | kWinFlag, word base of the row}
  const Tile* tiles;
  uint32_t n_tiles, n_items, col_bits;
  int filter;
  uint32_t kappa, start, stop;
  const uint32_t* h_row;
  const uint32_t* h_col;
  unsigned long long* tile_words;   // B1: word totals per tile
  unsigned long long* tile_cursor;  // B2: next free word per tile
  const unsigned long long* tile_base;  // B2: first word of each tile
  int chunk_tx;                     // transactions per chunk (<= kChunkTx)
  uint32_t scat_ns;                 // k_stream_scatter: tiles with shared counters
  int packed_filter;                // k_stream_scatter: bucket-filter the word rows' pairs
  uint32_t* words;
  // B1 -> B2: words per (chunk, shared-counter tile), [n_chunks][min(n_tiles,
  // kTileSmem)], so that B2 does not walk the chunk a second time (nullable)
  uint32_t* chunk_counts;
};

// Visit the words of row occurrence (g, q) of row item i: fn(dest_tile, base,
// first_col_pos, n_cols) for each run of consecutive columns with the same
// destination, or, with the bucket filter, fn per own column (n_cols = 1).
// The word of column j is base + j for both tile kinds (a hash tile's base
// has j's bits clear). tv = {tile | kWinFlag, base of the unsplit row}.
template <bool UPPER, typename Fn>
__device__ __forceinline__ void stream_row(const StreamRouteArgs& A, uint32_t i, const Pos& q,
                                           uint2 tv, Fn&& fn) {
  if (tv.x == kNone || (UPPER && q.p + 1 >= q.L)) return;
  const uint32_t tile = tv.x & kTileMask;
  const uint32_t c_lo = UPPER ? q.p + 1 : 0;
  const uint64_t tb = (uint64_t)q.base;
  if (!(tv.x & kWinFlag) && !A.filter) {
    fn(tile, tv.y, (uint32_t)(tb + c_lo), q.L - c_lo);
    return;
  }
  uint32_t c0 = 0, nwin = 1;
  if (tv.x & kWinFlag) {
    const Tile T0 = A.tiles[tile];
    c0 = T0.c0;
    nwin = T0.nwin;
  }
  uint32_t run_tile = kNone, run_start = 0, run_n = 0, run_base = 0;
  for (uint32_t p = c_lo; p < q.L; ++p) {
    const uint32_t j = A.items[tb + p];
    uint32_t dest = tile, base = tv.y;
    if (tv.x & kWinFlag) {
      if (j < c0) continue;
      const uint32_t w = (j - c0) / kStreamDenseCap;
      if (w >= nwin) break;
      dest = tile + w;
      base = 0u - (c0 + w * kStreamDenseCap);  // window w starts at column c0 + w * cap
    }
    if (A.filter) {
      uint32_t b = A.h_row[i] + A.h_col[j];
      if (b >= A.kappa) b -= A.kappa;
      if (b < A.start || b >= A.stop) continue;
      fn(dest, base, (uint32_t)(tb + p), 1u);
      continue;
    }
    if (dest != run_tile) {
      if (run_n) fn(run_tile, run_base, run_start, run_n);
      run_tile = dest;
      run_start = (uint32_t)(tb + p);
      run_n = 0;
      run_base = base;
    }
    ++run_n;
  }
  if (run_n) fn(run_tile, run_base, run_start, run_n);
}

// Destination tile and word of column j of a split (column-window) or
// filtered row (tx, ty = the row's item_info; c0, nwin = its first window's
// start and count; hr = h_row of the row item): dst = kNone when the column
// is past the last window or in another bucket interval. Same rules as
// stream_row.
__device__ __forceinline__ void split_row_dest(const StreamRouteArgs& A, uint32_t tx, uint32_t ty,
                                               uint32_t c0, uint32_t nwin, uint32_t hr, uint32_t j,
                                               uint32_t& dst, uint32_t& word) {
  dst = tx & kTileMask;
  word = ty + j;
  if (tx & kWinFlag) {
    const uint32_t w = j >= c0 ? (j - c0) / kStreamDenseCap : nwin;
    if (w >= nwin) {
      dst = kNone;
      return;
    }
    dst += w;
    word = j - (c0 + w * kStreamDenseCap);  // window w starts at c0 + w * cap
  }
  if (A.filter) {
    uint32_t bk = hr + A.h_col[j];
    if (bk >= A.kappa) bk -= A.kappa;
    if (bk < A.start || bk >= A.stop) dst = kNone;
  }
}

// Runs of equal destination among adjacent lanes (the windows of a sorted
// suffix are contiguous, so a run is a window's group; a filter may cut a
// window into several runs): the run's first lane, this lane's rank in it
// and, for the first lane, the run's length. Replaces __match_any_sync.
__device__ __forceinline__ void lane_runs(uint32_t dst, int& lead, uint32_t& rank, uint32_t& len) {
  const int lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, dst, 1);
  const uint32_t heads = __ballot_sync(0xffffffffu, lane == 0 || prev != dst);
  const uint32_t upto = 0xFFFFFFFFu >> (31 - lane);  // lanes <= lane
  lead = 31 - __clz(heads & upto);
  const uint32_t above = heads & ~upto;
  len = (above ? (uint32_t)__ffs(above) - 1u : 32u) - (uint32_t)lead;
  rank = (uint32_t)(lane - lead);
}

// The suffix columns of the warp's split (column-window) / filtered rows,
// flattened across the warp: lane state = one row occurrence (slow: it is such
// a row; first, n = position and length of its column run), fn(dst, word) is
// called warp-wide once per 32 columns with each lane's destination tile and
// word (dst = kNone: none). The owner of flattened column t is found by a
// binary search over the inclusive lengths (zero-length lanes in between);
// every lane of a step is busy whatever the rows' lengths, where one row at
// a time across the warp left half the lanes idle (c3: 11 warp instructions
// per term in k_stream_write).
template <typename Fn>
__device__ __forceinline__ void for_slow_columns(const StreamRouteArgs& A, bool slow, uint32_t ir,
                                                 uint32_t tx, uint32_t ty, uint32_t first, uint32_t n,
                                                 Fn&& fn) {
  if (!__any_sync(0xffffffffu, slow)) return;
  const int lane = threadIdx.x & 31;
  uint32_t c0 = 0, nwin = 1, hr = 0;
  if (slow) {
    if (tx & kWinFlag) {
      const Tile T0 = A.tiles[tx & kTileMask];
      c0 = T0.c0;
      nwin = T0.nwin;
    }
    if (A.filter) hr = A.h_row[ir];
  }
  const uint32_t my_n = slow ? n : 0u;
  const uint32_t incl = warp_incl_scan(my_n);
  const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t start = first - (incl - my_n);  // position of flattened column t: t + start
  for (uint32_t t0 = 0; t0 < S; t0 += 32) {
    const uint32_t t = t0 + lane;
    int o = 0;  // lanes whose run ends at or before t
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, o + d - 1);
      if (v <= t) o += d;
    }
    o &= 31;
    const uint32_t o_start = __shfl_sync(0xffffffffu, start, o);
    const uint32_t o_tx = __shfl_sync(0xffffffffu, tx, o);
    const uint32_t o_ty = __shfl_sync(0xffffffffu, ty, o);
    const uint32_t o_c0 = __shfl_sync(0xffffffffu, c0, o);
    const uint32_t o_nwin = __shfl_sync(0xffffffffu, nwin, o);
    const uint32_t o_hr = __shfl_sync(0xffffffffu, hr, o);
    uint32_t dst = kNone, word = 0;
    if (t < S) split_row_dest(A, o_tx, o_ty, o_c0, o_nwin, o_hr, A.items[t + o_start], dst, word);
    fn(dst, word);
  }
}

// B1: words per tile (shared counters per CTA, flushed once)
template <bool UPPER>
__global__ void __launch_bounds__(kPassThreads, 1) k_stream_count(StreamRouteArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + kOffBytes);
  const uint32_t ns = min(A.n_tiles, kTileSmem);
  const int lane = threadIdx.x & 31;
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  const int64_t n_chunks = (A.n_tx + A.chunk_tx - 1) / A.chunk_tx;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    __syncthreads();
    const int ntx = stage_offsets(s_off, A.offsets, A.n_tx, chunk, A.chunk_tx);
    walk_chunk<true>(s_off, ntx, A.items, A.item_info,
                     [&](int64_t, const Pos& q, uint32_t i, uint2 tv) {
      const bool live = q.valid && tv.x != kNone && !(UPPER && q.p + 1 >= q.L);
      const bool slow = live && !(tv.x & kEntFlag) && ((tv.x & kWinFlag) || A.filter);
      if (live && !slow) {
        // one run: a word row's suffix, or an entry row's (first, count) pair
        const uint32_t t = tv.x & kTileMask;
        const uint32_t n = (tv.x & kEntFlag) ? 2u : q.L - (UPPER ? q.p + 1 : 0u);
        if (t < ns) atomicAdd(&s_cnt[t], n);
        else atomicAdd(&A.tile_words[t], (unsigned long long)n);
      }
      // split / filtered rows: their columns flattened across the warp
      const uint32_t skip = UPPER ? q.p + 1 : 0u;
      for_slow_columns(A, slow, i, tv.x, tv.y, (uint32_t)q.base + skip, q.L - skip,
                       [&](uint32_t dst, uint32_t) {
        int lead;
        uint32_t rank, len;
        lane_runs(dst, lead, rank, len);
        if (dst != kNone && rank == 0) {
          if (dst < ns) atomicAdd(&s_cnt[dst], len);
          else atomicAdd(&A.tile_words[dst], (unsigned long long)len);
        }
      });
    });
    // flush per chunk: shared u32 counts never exceed one chunk's words
    __syncthreads();
    uint32_t* cc = A.chunk_counts ? A.chunk_counts + (size_t)chunk * ns : nullptr;
    for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) {
      const uint32_t c = s_cnt[t];
      if (cc) cc[t] = c;
      if (c) {
        atomicAdd(&A.tile_words[t], (unsigned long long)c);
        s_cnt[t] = 0;
      }
    }
  }
}

// B2: per chunk, count words per shared tile, claim one range per touched
// tile, then write the words. Unfiltered rows are written cooperatively by
// the warp (32 consecutive words per store); filtered or split rows by lane.
template <bool UPPER>
__global__ void __launch_bounds__(kPassThreads, 1) k_stream_write(StreamRouteArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);
  // shared tile counters sized by the job (ns rounded to 2 for alignment)
  const uint32_t ns = min(A.n_tiles, kTileSmem);
  const uint32_t ns2 = (ns + 1) & ~1u;
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + kOffBytes);
  uint16_t* s_touched = reinterpret_cast<uint16_t*>(s_cnt + ns2);  // tile ids < 2^16
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(s_touched + ns2);
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // triangle decode for transactions of <= 32 items: pair t = r (r + 1) / 2 + c
  // -> r | c << 8 (row r from the end, column offset c <= r)
  __shared__ uint16_t s_tri[496];
  for (uint32_t r = 0; r < 31; ++r)
    for (uint32_t c = threadIdx.x; c <= r; c += blockDim.x) s_tri[r * (r + 1) / 2 + c] = (uint16_t)(r | c << 8);
  const int64_t n_chunks = (A.n_tx + A.chunk_tx - 1) / A.chunk_tx;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) s_misc[0] = 0;
    const int ntx = stage_offsets(s_off, A.offsets, A.n_tx, chunk, A.chunk_tx);
    if (A.chunk_counts) {
      // B1 (k_stream_count) left this chunk's words per shared-counter tile
      const uint32_t* cc = A.chunk_counts + (size_t)chunk * ns;
      for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) {
        const uint32_t c = cc[t];
        s_cnt[t] = c;
        if (c) s_touched[atomicAdd(&s_misc[0], 1u)] = (uint16_t)t;
      }
    } else
    walk_chunk<true>(s_off, ntx, A.items, A.item_info,
                     [&](int64_t, const Pos& q, uint32_t i, uint2 tv) {
      // words per shared-counter tile (ids < ns; a split row's windows follow
      // its first window's id, so a row whose first tile is >= ns is skipped)
      const bool live = q.valid && tv.x != kNone && !(UPPER && q.p + 1 >= q.L) &&
                        (tv.x & kTileMask) < ns;
      const bool slow = live && !(tv.x & kEntFlag) && ((tv.x & kWinFlag) || A.filter);
      if (live && !slow) {
        const uint32_t t = tv.x & kTileMask;
        const uint32_t n = (tv.x & kEntFlag) ? 2u : q.L - (UPPER ? q.p + 1 : 0u);
        if (atomicAdd(&s_cnt[t], n) == 0) s_touched[atomicAdd(&s_misc[0], 1u)] = t;
      }
      const uint32_t skip = UPPER ? q.p + 1 : 0u;
      for_slow_columns(A, slow, i, tv.x, tv.y, (uint32_t)q.base + skip, q.L - skip,
                       [&](uint32_t dst, uint32_t) {
        if (dst >= ns) dst = kNone;
        int lead;
        uint32_t rank, len;
        lane_runs(dst, lead, rank, len);
        if (dst != kNone && rank == 0)
          if (atomicAdd(&s_cnt[dst], len) == 0) s_touched[atomicAdd(&s_misc[0], 1u)] = dst;
      });
    });
    __syncthreads();
    const uint32_t n_touch = s_misc[0];
    for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) {
      const uint32_t t = s_touched[k];
      // claimed first word (all word positions of a job are < 2^32)
      s_cnt[t] = (uint32_t)atomicAdd(&A.tile_cursor[t], (unsigned long long)s_cnt[t]);
    }
    __syncthreads();
    // write: one warp per transaction. Lanes hold 32 rows (their claims and
    // bases) and 32 columns at a time. Transactions of <= 32 items (UPPER)
    // are written as their flattened triangle, 32 pairs per store
    // instruction; their claims are made one transaction ahead so the claim
    // latency overlaps the previous transaction's stores. Items are loaded
    // four transactions ahead, item_info three ahead.
    {
      constexpr int NW = kPassThreads / 32;
      auto ld_it = [&](int t) -> uint32_t {
        if (t >= ntx) return kNone;
        const int64_t tb = s_off[t];
        return (int64_t)lane < s_off[t + 1] - tb ? __ldg(A.items + tb + lane) : kNone;
      };
      auto ld_tv = [&](uint32_t it) -> uint2 {
        return it != kNone ? __ldg(A.item_info + it) : make_uint2(kNone, 0u);
      };
      // rows p < L of a transaction, first 32: claim (fast rows) or write
      // directly (split / filtered rows); returns the fast-row mask
      auto claim = [&](int t, int64_t tb, uint32_t L, uint32_t pc, uint32_t i, uint2 tv,
                       uint32_t& dest, uint32_t& bb) -> uint32_t {
        const uint32_t p = pc + lane;
        bool fast = false, slow = false;
        if (p < L && (!UPPER || p + 1 < L) && tv.x != kNone) {
          const uint32_t n = UPPER ? L - 1 - p : L;
          if (tv.x & kEntFlag) {
            // single-row tile counted from entries: {first column position, n}
            const uint32_t t2 = tv.x & kTileMask;
            const uint32_t e = t2 < ns ? atomicAdd(&s_cnt[t2], 2u)
                                       : (uint32_t)atomicAdd(&A.tile_cursor[t2], 2ull);
            *reinterpret_cast<uint2*>(A.words + e) = make_uint2((uint32_t)(tb + (UPPER ? p + 1 : 0)), n);
          } else if (!(tv.x & kWinFlag) && !A.filter) {
            fast = true;
            bb = tv.y;
            dest = tv.x < ns ? atomicAdd(&s_cnt[tv.x], n)
                             : (uint32_t)atomicAdd(&A.tile_cursor[tv.x], (unsigned long long)n);
          } else {
            slow = true;
          }
        }
        // split (column-window) and filtered rows: one row at a time across
        // the warp -- lanes take 32 suffix columns, group by destination tile
        // (windows of a sorted suffix are contiguous), one claim per group,
        // and the group's words are stored to consecutive positions
        const uint32_t skip = UPPER ? p + 1 : 0u;
        for_slow_columns(A, slow, i, tv.x, tv.y, (uint32_t)tb + skip, L - skip,
                         [&](uint32_t dst, uint32_t word) {
          int lead;
          uint32_t rank, len;
          lane_runs(dst, lead, rank, len);
          uint32_t p0 = 0;
          if (dst != kNone && rank == 0)
            p0 = dst < ns ? atomicAdd(&s_cnt[dst], len)
                          : (uint32_t)atomicAdd(&A.tile_cursor[dst], (unsigned long long)len);
          p0 = __shfl_sync(0xffffffffu, p0, lead);
          if (dst != kNone) A.words[p0 + rank] = word;
        });
        return __ballot_sync(0xffffffffu, fast);
      };
      uint32_t it_cur = ld_it(warp), it1 = ld_it(warp + NW), it2 = ld_it(warp + 2 * NW),
               it3 = ld_it(warp + 3 * NW);
      uint2 tv_cur = ld_tv(it_cur), tv1 = ld_tv(it1), tv2 = ld_tv(it2);
      // prepared claims of the current transaction (short path only)
      uint32_t c_dest = 0, c_bb = 0, c_fm = 0;
      auto prepare = [&](int t, uint32_t it, uint2 tv, uint32_t& dest, uint32_t& bb) -> uint32_t {
        if (t >= ntx) return 0u;
        const int64_t tb = s_off[t];
        const uint32_t L = (uint32_t)(s_off[t + 1] - tb);
        if (!UPPER || L > 32) return 0u;
        return claim(t, tb, L, 0, it, tv, dest, bb);
      };
      c_fm = prepare(warp, it_cur, tv_cur, c_dest, c_bb);
      for (int t = warp; t < ntx; t += NW) {
        const uint2 tv3 = ld_tv(it3);
        const uint32_t it4 = ld_it(t + 4 * NW);
        const int64_t tb = s_off[t];
        const uint32_t L = (uint32_t)(s_off[t + 1] - tb);
        uint32_t n_dest = 0, n_bb = 0;
        const uint32_t n_fm = prepare(t + NW, it1, tv1, n_dest, n_bb);
        if (UPPER && L <= 32 && c_fm && 2 * (uint32_t)__popc(c_fm) <= L) {
          // few word rows (the others are entry rows): one store instruction
          // per row, its columns across the lanes
          uint32_t m = c_fm;
          while (m) {
            const int r = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t d = __shfl_sync(0xffffffffu, c_dest, r);
            const uint32_t b2 = __shfl_sync(0xffffffffu, c_bb, r);
            if (lane > r && lane < (int)L) A.words[d + (lane - r - 1)] = b2 + it_cur;
          }
        } else if (UPPER && L <= 32) {
          // the flattened triangle: pair tt -> (row from the end r, column
          // offset c) via the shared table; each row's run contiguous
          const uint32_t P = L * (L - 1) / 2;
          if (c_fm)
            for (uint32_t t0 = 0; t0 < P; t0 += 32) {
              const uint32_t tt = t0 + lane;
              const uint32_t rc = s_tri[tt < P ? tt : 0];
              const uint32_t pr = L - 2 - (rc & 0xFFu), c = rc >> 8;
              const uint32_t kk = pr + 1 + c;
              const uint32_t d = __shfl_sync(0xffffffffu, c_dest, pr & 31);
              const uint32_t b2 = __shfl_sync(0xffffffffu, c_bb, pr & 31);
              const uint32_t jk = __shfl_sync(0xffffffffu, it_cur, kk & 31);
              if (tt < P && ((c_fm >> pr) & 1u)) A.words[d + c] = b2 + jk;
            }
        } else {
          for (uint32_t pc = 0; pc < L; pc += 32) {
            uint32_t i = it_cur;
            uint2 tv = tv_cur;
            if (pc > 0 && pc + lane < L) {
              i = A.items[tb + pc + lane];
              tv = A.item_info[i];
            }
            uint32_t dest = 0, bb = 0;
            const uint32_t fm = claim(t, tb, L, pc, i, tv, dest, bb);
            if (!fm) continue;
            for (uint32_t kc = UPPER ? pc : 0; kc < L; kc += 32) {
              const uint32_t k = kc + lane;
              const uint32_t jk = kc == 0 ? it_cur : (k < L ? A.items[tb + k] : 0u);
              // UPPER: the chunk's last row has no column in its own chunk
              uint32_t m = fm;
              if (UPPER && kc == pc) m &= 0x7FFFFFFFu;
              while (m) {
                const int r = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t d = __shfl_sync(0xffffffffu, dest, r);
                const uint32_t b2 = __shfl_sync(0xffffffffu, bb, r);
                const uint32_t c_lo = UPPER ? pc + r + 1 : 0;
                if (k >= c_lo && k < L) A.words[d + (k - c_lo)] = b2 + jk;
              }
            }
          }
        }
        c_dest = n_dest;
        c_bb = n_bb;
        c_fm = n_fm;
        it_cur = it1;
        it1 = it2;
        it2 = it3;
        it3 = it4;
        tv_cur = tv1;
        tv1 = tv2;
        tv2 = tv3;
      }
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) s_cnt[s_touched[k]] = 0;
  }
}

// Single-walk scatter (unfiltered jobs without column windows, i.e. when the
// device planner knows every tile's word total): chunks are the transactions
// whose first item lies in one band of kScatPark - maxlen + 1 positions, so
// a chunk holds at most kScatPark positions. One walk takes, per row occurrence,
// its rank in its tile's chunk range from a returning shared-memory atomic
// and parks (tile, rank, n) in shared memory; after one claim per touched
// tile the parked rows are scattered: an 8-byte entry per entry-tile row,
// the suffix words for a hash / multi-row tile row.
constexpr uint32_t kScatPark = 10240;   // parked rows (positions) per chunk
constexpr uint32_t kScatPark2 = 5120;   // two CTAs per SM: half the band
constexpr uint32_t kScatMaxTx2 = 1024;

// 16-bit copy of the items (ids < 2^16) for the suffix gathers of the count
// kernel; runs on a side stream while the single-CTA planner runs.
__global__ void k_items16(const uint32_t* __restrict__ items, int64_t nnz, uint16_t* __restrict__ out) {
  const int64_t n4 = nnz / 4;
  const uint4* in4 = reinterpret_cast<const uint4*>(items);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(in4 + k);
    const uint2 o = make_uint2(v.x | (v.y << 16), v.z | (v.w << 16));
    reinterpret_cast<uint2*>(out)[k] = o;
  }
  for (int64_t k = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = (uint16_t)items[k];
}

// Filtered jobs (multi-GPU bucket intervals): the items packed with their
// column hash, item | h_col(item) << 16 (ids and kappa < 2^16), so the
// count kernel tests bucket ownership of a pair without a table gather.
__global__ void k_items_cls(const uint32_t* __restrict__ items, int64_t nnz,
                            const uint32_t* __restrict__ h_col, uint32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t it = __ldcs(items + k);
    out[k] = it | (h_col[it] << 16);
  }
}

__global__ void k_chunk_bounds(const int64_t* __restrict__ offsets, int64_t n_tx, uint32_t n_chunks,
                               uint32_t band, uint32_t* __restrict__ bounds) {
  // bounds[c] = first transaction whose start position lies in band >= c
  // (band = kScatPark - longest transaction + 1 positions)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tx;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = t > 0 ? offsets[t - 1] / band : -1;
    const int64_t cur = t < n_tx ? offsets[t] / band : (int64_t)n_chunks;
    for (int64_t c = prev + 1; c <= cur && c <= (int64_t)n_chunks; ++c) bounds[c] = (uint32_t)t;
  }
}

// THREADS / PARK / MAXTX: one 1024-thread CTA per SM with 10,240-position
// bands, or two 512-thread CTAs per SM with half the bands (one CTA's
// returning tile claims and barriers overlap the other's walk and copy).
template <bool UPPER, bool PF, int THREADS = kPassThreads, uint32_t PARK = kScatPark,
          uint32_t MAXTX = kScatMaxTx>
__global__ void __launch_bounds__(THREADS, THREADS >= 1024 ? 1 : 2)
    k_stream_scatter(StreamRouteArgs A, const uint32_t* __restrict__ bounds, uint32_t n_chunks) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);                          // MAXTX + 1
  // parked rows: entry << 31 | n << 16 | (absolute rank ? 0x8000 : shared tile id), or kNone
  uint32_t* s_tm = reinterpret_cast<uint32_t*>(s_off + MAXTX + 1);
  uint32_t* s_rank = s_tm + PARK;
  uint32_t* s_bp = s_rank + PARK;                                        // word rows: base
  uint32_t* s_job = s_bp + PARK;                                         // per warp 128 words
  uint32_t* s_misc = s_job + THREADS / 32 * 128;
  const uint32_t ns = min(A.n_tiles, A.scat_ns);
  const uint32_t ns2 = (ns + 1) & ~1u;
  uint32_t* s_cnt = s_misc + 4;
  uint16_t* s_touched = reinterpret_cast<uint16_t*>(s_cnt + ns2);
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint32_t tb0 = bounds[c], tb1 = bounds[c + 1];
    for (uint32_t ta = tb0; ta < tb1; ta += MAXTX) {
      const int ntx = (int)min(MAXTX, tb1 - ta);
      __syncthreads();
      if (threadIdx.x == 0) s_misc[0] = 0;
      for (int t = threadIdx.x; t <= ntx; t += blockDim.x) s_off[t] = A.offsets[ta + t];
      __syncthreads();
      const int64_t g_lo = s_off[0];
      const uint32_t npos = (uint32_t)(s_off[ntx] - g_lo);
      // walk: rank of every row occurrence in its tile's chunk range
      walk_chunk<true>(s_off, ntx, A.items, A.item_info,
                       [&](int64_t g, const Pos& q, uint32_t, uint2 tv) {
        if (!q.valid) return;
        const uint32_t x = (uint32_t)(g - g_lo);
        uint32_t tm = kNone;
        if (tv.x != kNone && (UPPER ? q.p + 1 < q.L : q.L > 0)) {
          const uint32_t n = UPPER ? q.L - 1 - q.p : q.L;  // < 2^15 (kMaxLen)
          const bool ent = (tv.x & kEntFlag) != 0;
          const uint32_t tile = tv.x & kTileMask;
          const uint32_t units = ent ? 2u : n;
          uint32_t r;
          if (tile < ns) {  // ns < 2^15
            r = atomicAdd(&s_cnt[tile], units);
            if (r == 0) s_touched[atomicAdd(&s_misc[0], 1u)] = (uint16_t)tile;
            tm = tile;
          } else {
            r = (uint32_t)atomicAdd(&A.tile_cursor[tile], (unsigned long long)units);
            tm = 0x8000u;  // rank is already absolute
          }
          tm |= n << 16 | (ent ? 0x80000000u : 0u);
          s_rank[x] = r;
          s_bp[x] = tv.y;
        }
        s_tm[x] = tm;
      });
      __syncthreads();
      const uint32_t n_touch = s_misc[0];
      for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) {
        const uint32_t t = s_touched[k];
        s_cnt[t] = (uint32_t)atomicAdd(&A.tile_cursor[t], (unsigned long long)s_cnt[t]);
      }
      __syncthreads();
      // scatter the parked rows: each warp takes 32 positions at a time;
      // entry rows store their 8-byte entry, word rows copy their suffixes
      // flattened across the warp (one store instruction per 32 words)
      {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t* j_dst = s_job + warp * 128;
        uint32_t* j_src = j_dst + 32;
        uint32_t* j_b = j_src + 32;
        uint32_t* j_n = j_b + 32;
        for (uint32_t x0 = warp * 32; x0 < npos; x0 += THREADS) {
          const uint32_t x = x0 + lane;
          uint32_t tile = kNone, pos = 0, meta = 0;
          if (x < npos) {
            const uint32_t tm = s_tm[x];
            if (tm != kNone) {
              tile = tm & 0xFFFFu;
              pos = (tm & 0x8000u) ? s_rank[x] : s_cnt[tm & 0x7FFFu] + s_rank[x];
              meta = (tm >> 16 & 0x7FFFu) | (tm & 0x80000000u);
            }
          }
          const uint64_t g = (uint64_t)g_lo + x;
          uint32_t first = (uint32_t)(g + 1);
          if (!UPPER && tile != kNone) {
            int lo = 0, hi = ntx;
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (s_off[mid] <= (int64_t)g) lo = mid;
              else hi = mid;
            }
            first = (uint32_t)s_off[lo];
          }
          const bool ent = tile != kNone && (meta & 0x80000000u);
          if (ent) *reinterpret_cast<uint2*>(A.words + pos) = make_uint2(first, meta & 0x7FFFFFFFu);
          const uint32_t nw = (tile != kNone && !ent) ? meta : 0u;
          const uint32_t wm = __ballot_sync(0xffffffffu, nw > 0);
          if (!wm) continue;
          // compact the word rows to the low lanes (the boundary-mask owner
          // lookup needs every lane's length > 0)
          if (nw) {
            const int r = __popc(wm & ((1u << lane) - 1u));
            j_dst[r] = pos;
            j_src[r] = first;
            j_b[r] = s_bp[x];
            j_n[r] = PF ? (nw | A.h_row[A.items[g]] << 16) : nw;
          }
          __syncwarp();
          const uint32_t my_n = lane < __popc(wm) ? (PF ? (j_n[lane] & 0xFFFFu) : j_n[lane]) : 0u;  // n < 2^16
          const uint32_t incl = warp_incl_scan(my_n);
          const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
          const uint32_t excl = incl - my_n;
          uint32_t ob = 0;
          for (uint32_t t0 = 0; t0 < S; t0 += 32) {
            const uint32_t o = owner_step(incl, t0, ob);
            const uint32_t t = t0 + lane;
            const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, o & 31);
            if (t < S) {
              const uint32_t loc = t - o_excl;
              const uint32_t j = A.items[j_src[o] + loc];
              uint32_t w = j_b[o] + j;
              if (PF) {
                // pairs of other GPUs' buckets keep their place as empty words
                uint32_t b = (j_n[o] >> 16) + A.h_col[j];
                if (b >= A.kappa) b -= A.kappa;
                if (b < A.start || b >= A.stop) w = kEmpty32;
              }
              A.words[j_dst[o] + loc] = w;
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) s_cnt[s_touched[k]] = 0;
    }
  }
}

// Own-bucket scatter (Lemma 1): like k_stream_scatter, but a row occurrence
// routes only its own partners, read from its window(s) of the (h_col,
// id)-sorted copy. Walk: each position finds its window, counts its own
// partners and claims that many words of its tile. Copy: the parked rows'
// windows are flattened across the warp; with the triangle filter the items
// not after the row are dropped and the kept ones compacted with a ballot
// (one contiguous store run per row and step). Words only for own pairs: a
// filtered job's write and count phases scale with its own terms.
// SINGLE (single-bucket intervals): a row's own partners are one contiguous
// range of the sorted keys (own_partners), parked at walk time and copied
// like the plain scatter's suffixes; no filter, no compaction.
constexpr uint32_t kScatParkOwn = kOwnStage;
template <bool SINGLE>
__host__ __device__ constexpr size_t scatter_own_fixed() {
  return (size_t)(kScatMaxTx + 1) * 8 + (size_t)kScatParkOwn * 4 * 5 + 16 +
         (size_t)(kPassThreads / 32) * (SINGLE ? 128 : 256) * 4;
}
template <bool UPPER, bool SINGLE>
__global__ void __launch_bounds__(kPassThreads, 1)
    k_stream_scatter_own(StreamRouteArgs A, OwnArgs O, const uint32_t* __restrict__ bounds,
                         uint32_t n_chunks) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);                          // kScatMaxTx + 1
  uint32_t* s_tile = reinterpret_cast<uint32_t*>(s_off + kScatMaxTx + 1);     // parked rows
  uint32_t* s_rank = s_tile + kScatParkOwn;
  uint32_t* s_rec = s_rank + kScatParkOwn;                                    // pass A position records
  uint32_t* s_bp = s_rec + kScatParkOwn;                                      // row word base
  // SINGLE: first partner | count per parked row; general: the band's keys
  uint32_t* s_src = s_bp + kScatParkOwn;
  uint32_t* s_hs = s_src;
  uint32_t* s_job = s_src + kScatParkOwn;                                     // per warp 128 / 256 words
  uint32_t* s_misc = s_job + kPassThreads / 32 * (SINGLE ? 128 : 256);
  const uint32_t ns = min(A.n_tiles, A.scat_ns);
  const uint32_t ns2 = (ns + 1) & ~1u;
  uint32_t* s_cnt = s_misc + 4;
  uint16_t* s_touched = reinterpret_cast<uint16_t*>(s_cnt + ns2);
  const uint32_t idmask = O.idbits >= 32 ? 0xFFFFFFFFu : ((1u << O.idbits) - 1u);
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  for (uint32_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const uint32_t tb0 = bounds[c], tb1 = bounds[c + 1];
    for (uint32_t ta = tb0; ta < tb1; ta += kScatMaxTx) {
      const int ntx = (int)min(kScatMaxTx, tb1 - ta);
      __syncthreads();
      if (threadIdx.x == 0) s_misc[0] = 0;
      for (int t = threadIdx.x; t <= ntx; t += blockDim.x) s_off[t] = A.offsets[ta + t];
      __syncthreads();
      const int64_t g_lo = s_off[0];
      const uint32_t npos = (uint32_t)(s_off[ntx] - g_lo);
      for (uint32_t x = threadIdx.x; x < npos; x += blockDim.x) {
        s_rec[x] = __ldg(O.pos_rec + g_lo + x);
        if (!SINGLE) s_hs[x] = __ldg(O.hs + g_lo + x);
      }
      __syncthreads();
      walk_chunk<true>(s_off, ntx, A.items, A.item_info,
                       [&](int64_t g, const Pos& q, uint32_t i, uint2 tv) {
        if (!q.valid) return;
        const uint32_t x = (uint32_t)(g - g_lo);
        uint32_t tile = kNone;
        if (tv.x != kNone && (UPPER ? q.p + 1 < q.L : q.L > 0)) {
          // own partners counted by pass A (k_own_prep)
          const uint32_t rec = s_rec[x];
          const uint32_t n = rec & 0xFFFFu;
          if (SINGLE) s_src[x] = (uint32_t)(q.base - g_lo + (rec >> 16)) | (n << 16);  // < 2^16 each
          if (n) {
            tile = tv.x & kTileMask;
            uint32_t r;
            if (tile < ns) {
              r = atomicAdd(&s_cnt[tile], n);
              if (r == 0) s_touched[atomicAdd(&s_misc[0], 1u)] = (uint16_t)tile;
            } else {
              r = (uint32_t)atomicAdd(&A.tile_cursor[tile], (unsigned long long)n);
              tile |= kWinFlag;  // rank is already absolute
            }
            s_rank[x] = r;
            s_bp[x] = tv.y;
          }
        }
        s_tile[x] = tile;
      });
      __syncthreads();
      const uint32_t n_touch = s_misc[0];
      for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) {
        const uint32_t t = s_touched[k];
        s_cnt[t] = (uint32_t)atomicAdd(&A.tile_cursor[t], (unsigned long long)s_cnt[t]);
      }
      __syncthreads();
      if (SINGLE) {
        // contiguous partner ranges, flattened across the warp (one store
        // instruction per 32 words), as the plain scatter copies suffixes
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t* j_dst = s_job + warp * 128;
        uint32_t* j_src = j_dst + 32;
        uint32_t* j_b = j_src + 32;
        uint32_t* j_n = j_b + 32;
        for (uint32_t x0 = warp * 32; x0 < npos; x0 += kPassThreads) {
          const uint32_t x = x0 + lane;
          uint32_t nw = 0, pos = 0, sp = 0;
          if (x < npos) {
            const uint32_t tile = s_tile[x];
            if (tile != kNone) {
              pos = (tile & kWinFlag) ? s_rank[x] : s_cnt[tile] + s_rank[x];
              sp = s_src[x];
              nw = sp >> 16;
            }
          }
          const uint32_t wm = __ballot_sync(0xffffffffu, nw > 0);
          if (!wm) continue;
          if (nw) {
            const int r = __popc(wm & ((1u << lane) - 1u));
            j_dst[r] = pos;
            j_src[r] = sp & 0xFFFFu;
            j_b[r] = s_bp[x];
            j_n[r] = nw;
          }
          __syncwarp();
          const uint32_t my_n = lane < __popc(wm) ? j_n[lane] : 0u;
          const uint32_t incl = warp_incl_scan(my_n);
          const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
          const uint32_t excl = incl - my_n;
          uint32_t ob = 0;
          for (uint32_t t0 = 0; t0 < S; t0 += 32) {
            const uint32_t o = owner_step(incl, t0, ob) & 31;
            const uint32_t t = t0 + lane;
            const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, o);
            if (t < S) {
              const uint32_t loc = t - o_excl;
              A.words[j_dst[o] + loc] = j_b[o] + (__ldg(O.hs + g_lo + j_src[o] + loc) & idmask);
            }
          }
          __syncwarp();
        }
      } else {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t* j_dst = s_job + warp * 256;
        uint32_t* j_src = j_dst + 32;   // staged key position of the first window
        uint32_t* j_tb = j_src + 32;    // staged transaction start (second window)
        uint32_t* j_n1 = j_tb + 32;     // first window's length
        uint32_t* j_b = j_n1 + 32;      // row word base
        uint32_t* j_i = j_b + 32;       // row item (triangle filter)
        uint32_t* j_kept = j_i + 32;    // words written so far
        uint32_t* j_n = j_kept + 32;    // window length
        for (uint32_t x0 = warp * 32; x0 < npos; x0 += kPassThreads) {
          const uint32_t x = x0 + lane;
          uint32_t tile = kNone, pos = 0, nwin = 0, a0 = 0, n1 = 0, i = 0;
          int64_t tb = 0;
          if (x < npos) {
            tile = s_tile[x];
            if (tile != kNone) {
              pos = (tile & kWinFlag) ? s_rank[x] : s_cnt[tile] + s_rank[x];
              // the row's transaction: last t with s_off[t] <= its position
              const int64_t g = g_lo + x;
              int lo = 0, hi = ntx;
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_off[mid] <= g) lo = mid;
                else hi = mid;
              }
              tb = s_off[lo] - g_lo;
              const uint32_t L = (uint32_t)(s_off[lo + 1] - s_off[lo]);
              i = __ldg(A.items + g);
              uint32_t n2;
              own_window(s_hs + tb, L, __ldg(O.h_row + i), O, a0, n1, n2);
              nwin = n1 + n2;
            }
          }
          const uint32_t wm = __ballot_sync(0xffffffffu, nwin > 0);
          if (!wm) continue;
          if (nwin) {
            const int r = __popc(wm & ((1u << lane) - 1u));
            j_dst[r] = pos;
            j_src[r] = (uint32_t)tb + a0;
            j_tb[r] = (uint32_t)tb;
            j_n1[r] = n1;
            j_b[r] = s_bp[x];
            j_i[r] = i;
            j_kept[r] = 0;
            j_n[r] = nwin;
          }
          __syncwarp();
          const uint32_t mine = (uint32_t)lane < (uint32_t)__popc(wm) ? j_n[lane] : 0u;
          const uint32_t incl = warp_incl_scan(mine);
          const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
          const uint32_t excl = incl - mine;
          uint32_t ob = 0;
          for (uint32_t t0 = 0; t0 < S; t0 += 32) {
            const uint32_t o = owner_step(incl, t0, ob) & 31;
            const uint32_t t = t0 + lane;
            const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, o);
            const uint32_t o_n = __shfl_sync(0xffffffffu, mine, o);
            const bool valid = t < S;
            const uint32_t loc = t - o_excl;
            uint32_t j = 0;
            bool keep = false;
            if (valid) {
              const uint32_t nn1 = j_n1[o];
              const uint32_t idx = loc < nn1 ? j_src[o] + loc : j_tb[o] + (loc - nn1);
              j = s_hs[idx] & idmask;
              keep = !UPPER || j > j_i[o];
            }
            const uint32_t km = __ballot_sync(0xffffffffu, keep);
            const uint32_t sl = o_excl > t0 ? o_excl - t0 : 0u;  // owner's first lane in this step
            const uint32_t from = ~((1u << sl) - 1u);
            if (keep)
              A.words[j_dst[o] + j_kept[o] + __popc(km & from & ((1u << lane) - 1u))] = j_b[o] + j;
            const bool last = valid && (loc + 1 == o_n || lane == 31);
            const uint32_t upto = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);
            __syncwarp();
            if (last) j_kept[o] += __popc(km & from & upto);
            __syncwarp();
          }
        }
      }
      __syncthreads();
      for (uint32_t k = threadIdx.x; k < n_touch; k += blockDim.x) s_cnt[s_touched[k]] = 0;
    }
  }
}

// Streaming counter: units are ranges of a tile's words; warps read them
// coalesced (4 loads in flight per lane) and bump u32 shared counters.
struct StreamCountArgs {
  const Tile* tiles;
  const Unit* units;
  uint32_t n_units;
  const unsigned long long* tile_base;
  const unsigned long long* tile_words;
  const uint32_t* words;
  const uint32_t* items;
  const uint16_t* items16;  // nullable: 16-bit copy of the items
  unsigned int* unit_counter;
  uint32_t n_items, col_bits;
  int upper;
  uint32_t* out_row;
  uint32_t* out_col;
  uint32_t* out_count;
  unsigned long long* out_n;
  uint64_t out_cap;  // output capacity (entries); claims beyond it are not written
  uint32_t* slabs;  // kStreamDenseCap words per unit of a split tile
  unsigned int* tile_done;
  unsigned long long* dbg;  // development only (CROP_DEBUG_KINDS): cycles per kind/phase
  // fused top-k inputs (nullable): histogram of counts >= kTopkExactBins and
  // the output positions of those entries
  uint32_t* topk_hist;
  unsigned long long* hi_list;
  unsigned long long* hi_n;
  // filtered jobs (packed bucket test, see k_items_cls)
  const uint32_t* items_cls;  // nullable: item | h_col << 16
  const uint32_t* h_row;
  uint32_t kappa, start, stop;
  uint32_t* overflow;  // raised when a 16-bit dense counter wraps (see bump_half_checked)
};

// Record an emitted entry for the fused top-k (high counts only: rare).
__device__ __forceinline__ void note_high(const StreamCountArgs& A, uint32_t c, uint64_t o) {
  if (A.topk_hist && c >= kTopkExactBins) {
    atomicAdd(&A.topk_hist[topk_count_bin(c)], 1u);
    A.hi_list[atomicAdd(A.hi_n, 1ull)] = o;
  }
}

// (row, column) of slot s of dense tile T (stream layout, stream_base)
__device__ __forceinline__ void dense_slot_pair(const Tile& T, uint32_t s, uint32_t n, bool upper,
                                                uint32_t& i, uint32_t& j) {
  if (T.row1 - T.row0 == 1) {
    i = T.row0;
    j = s + T.c0;
  } else if (upper) {
    uint32_t lo = T.row0, hi = T.row1;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (tri_rowbase(mid, T.row0, n) <= s) lo = mid;
      else hi = mid;
    }
    i = lo;
    j = (uint32_t)(s - tri_rowbase(i, T.row0, n)) + i + 1;
  } else {
    i = T.row0 + s / n;
    j = s % n;
  }
}

// Count the suffixes of a range of entries {first column position, n} of a
// single-row tile. The suffixes of 32 entries are cut into quads (4
// consecutive columns) and the quads flattened across the warp (boundary-mask
// owner lookup, one per 32 quads = 128 columns); each lane loads and counts
// its quad. Two quads' loads are in flight while an older quad is counted
// (the path is bound by memory-level parallelism, and registers cap it). Blocks of 32 entries go round-robin over the warps;
// the next block's entries are loaded ahead.
struct OwnFilter {  // packed items (item | h_col << 16): own pair iff (hr + h_col) mod kappa in [start, stop)
  uint32_t hr, kappa, start, stop;
  __device__ __forceinline__ bool own(uint32_t v) const {
    uint32_t b = hr + (v >> 16);
    if (b >= kappa) b -= kappa;
    return b >= start && b < stop;
  }
};

template <bool FILT, typename ItemT>
__device__ __forceinline__ void count_suffix_entries(const ItemT* __restrict__ items,
                                                     const uint2* __restrict__ ents, uint64_t e0,
                                                     uint64_t e1, uint32_t* table, uint32_t c0,
                                                     OwnFilter F = OwnFilter{}) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int Q = 4;
  const uint64_t nblk = (e1 - e0 + 31) / 32;
  auto ld = [&](uint64_t blk) -> uint2 {
    const uint64_t e = e0 + blk * 32 + lane;
    return e < e1 ? __ldcs(ents + e) : make_uint2(0u, 0u);
  };
  uint2 nen = make_uint2(0u, 0u);
  if ((uint64_t)warp < nblk) nen = ld(warp);
  uint32_t pj[Q], qj[Q];  // the quads loaded two and one steps ago (kNone = none)
#pragma unroll
  for (int k = 0; k < Q; ++k) pj[k] = qj[k] = kNone;
  const uint32_t nwarps = blockDim.x >> 5;
  for (uint64_t blk = warp; blk < nblk; blk += nwarps) {
    const uint2 en = nen;
    if (blk + nwarps < nblk) nen = ld(blk + nwarps);
    const uint32_t nq = (en.y + Q - 1) / Q;
    const uint32_t incl = warp_incl_scan(nq);
    const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
    // column position of quad q of this lane's entry: first + Q * (q - excl)
    const uint32_t delta = en.x - Q * (incl - nq);
    const uint32_t end = en.x + en.y;
    uint32_t ob = 0;
    for (uint32_t t0 = 0; t0 < S; t0 += 32) {
      const uint32_t o = owner_step(incl, t0, ob);
      const uint32_t d = __shfl_sync(0xffffffffu, delta, o & 31);
      const uint32_t e_end = __shfl_sync(0xffffffffu, end, o & 31);
      const uint32_t tt = t0 + lane;
      const uint32_t pos = Q * tt + d;
      uint32_t j[Q];
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        j[k] = (tt < S && pos + k < e_end) ? (uint32_t)__ldg(items + pos + k) : kNone;
        if (FILT && j[k] != kNone) j[k] = F.own(j[k]) ? (j[k] & 0xFFFFu) : kNone;
      }
      // count the quad loaded two steps ago while the newer ones are in flight
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (pj[k] != kNone) bump_half(table, pj[k] - c0);
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        pj[k] = qj[k];
        qj[k] = j[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < Q; ++k) {
    if (pj[k] != kNone) bump_half(table, pj[k] - c0);
    if (qj[k] != kNone) bump_half(table, qj[k] - c0);
  }
}

// Per unit: clear the table, count its words (block-cyclic 256-word blocks
// over the warps so all warps finish together; the next block's 8 words per
// lane are in flight while the current ones are counted), then either
// compact the table into the output (single-unit tiles) or store it as the
// unit's slab (split tiles, summed afterwards by k_reduce_slabs).
// Dense tiles: u32 counter per slot. Hash tiles: 64-bit slots key << 32 |
// count (linear probing), so an insert also counts (one CAS) and a hit is a
// fire-and-forget 64-bit shared add; the first probe of all 8 words of a
// lane is issued at once.
constexpr unsigned long long kEmpty64 = ~0ull;

template <bool DBG, bool FILT>
__global__ void __launch_bounds__(kSCThreads, 2) k_count_stream(StreamCountArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* table = reinterpret_cast<uint32_t*>(smem);  // dense counters
  unsigned long long* slot64 = reinterpret_cast<unsigned long long*>(smem);  // hash slots
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + (size_t)kSHalf * 4);
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n = A.n_items;
  constexpr int D = 8;
  constexpr uint32_t BW = 32 * D;  // words per block
  if (threadIdx.x == 0) s_misc[0] = atomicAdd(A.unit_counter, 1u);
  for (;;) {
    __syncthreads();
    const uint32_t u = s_misc[0];
    __syncthreads();
    if (u >= A.n_units) break;
    // the next unit is claimed now and published after counting
    uint32_t u_next = 0;
    if (threadIdx.x == 0) u_next = atomicAdd(A.unit_counter, 1u);
    const Unit unit = A.units[u];
    const Tile T = A.tiles[unit.tile];
    const uint64_t Wn = A.tile_words[unit.tile];
    const uint64_t wb = A.tile_base[unit.tile];
    const bool ents = T.mode == 2;  // entries {first column position, n} instead of words
    const uint64_t Wu = ents ? Wn / 2 : Wn;
    const uint64_t w0 = Wu * unit.local / T.n_units;
    const uint64_t w1 = Wu * (unit.local + 1) / T.n_units;
    // a sparse column window (a mid-weight row's window holding few words,
    // c3) counts in a hash table sized to its exact word total instead of
    // clearing and compacting 57,344 dense counters: key = column - c0
    const bool hwin = T.mode == 0 && T.n_units == 1 && T.row1 - T.row0 == 1 &&
                      Wn <= kSparseWindowWords && T.width > 2 * kSparseWindowWords;
    const bool dense = T.mode != 1 && !hwin;
    const uint32_t width = hwin ? stream_hash_slots(Wn) : T.width;
    long long c0 = 0, c1 = 0, c2 = 0;
    if (DBG) c0 = clock64();
    const uint32_t dwords = width < kSHalf ? width : kSHalf;  // dense: table words in use
    {
      uint4* t4 = reinterpret_cast<uint4*>(table);
      const uint32_t n4 = dense ? (dwords + 3) / 4 : width / 2;  // hash: width = slots
      const uint32_t f = dense ? 0u : kEmpty32;
      for (uint32_t s = threadIdx.x; s < n4; s += kSCThreads) t4[s] = make_uint4(f, f, f, f);
    }
    __syncthreads();
    if (DBG) c1 = clock64();
    if (ents) {
      // 16-bit copy of the items when ids fit (half the gathered bytes; an
      // 80 MB copy of c2's items stays L2-resident)
      if (FILT) {
        const OwnFilter F{A.h_row[T.row0], A.kappa, A.start, A.stop};
        count_suffix_entries<true>(A.items_cls, reinterpret_cast<const uint2*>(A.words + wb), w0, w1,
                                   table, T.c0, F);
      } else if (A.items16) {
        count_suffix_entries<false>(A.items16, reinterpret_cast<const uint2*>(A.words + wb), w0, w1, table, T.c0);
      } else {
        count_suffix_entries<false>(A.items, reinterpret_cast<const uint2*>(A.words + wb), w0, w1, table, T.c0);
      }
    } else {
    // CTA-wide blocks of kSCThreads * D words: lane (warp, lane) reads word
    // warp * 32 + lane + k * kSCThreads of each block (coalesced per warp),
    // so every warp gets an equal share even of a small unit (c3's sparse
    // windows and light tiles hold a few thousand words)
    constexpr uint32_t CB = kSCThreads * D;
    const uint64_t nw = w1 - w0;
    const uint32_t nb = (uint32_t)((nw + CB - 1) / CB);
    const uint32_t* wp = A.words + wb + w0 + warp * 32 + lane;
    auto fetch = [&](uint32_t blk, uint32_t (&v)[D]) {
      const uint32_t* p = wp + (uint64_t)blk * CB;
      if ((uint64_t)(blk + 1) * CB <= nw) {
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] = __ldcs(p + k * kSCThreads);
      } else {
        const uint64_t left = nw - (uint64_t)blk * CB;
#pragma unroll
        for (int k = 0; k < D; ++k)
          v[k] = (uint64_t)(k * kSCThreads + warp * 32 + lane) < left ? __ldcs(p + k * kSCThreads) : kEmpty32;
      }
    };
    uint32_t cur[D], nxt[D];
    // a unit of more than 65,535 words could wrap a 16-bit counter
    const bool checked = dense && nw > kStreamUnitOcc;
    if (nb > 0) fetch(0, cur);
    for (uint32_t blk = 0; blk < nb; ++blk) {
      if (blk + 1 < nb) fetch(blk + 1, nxt);
      if (dense && checked) {
#pragma unroll
        for (int k = 0; k < D; ++k)
          if (cur[k] != kEmpty32) bump_half_checked(table, cur[k], A.overflow);
      } else if (dense) {
#pragma unroll
        for (int k = 0; k < D; ++k)
          if (cur[k] != kEmpty32) bump_half(table, cur[k]);
      } else {
        uint32_t sl[D];
        unsigned long long v[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          sl[k] = __umulhi(mix32(cur[k]), width);
          v[k] = slot64[sl[k]];
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const uint32_t key = cur[k];
          if (key == kEmpty32) continue;
          uint32_t sk = sl[k];
          unsigned long long vk = v[k];
          for (;;) {
            if ((uint32_t)(vk >> 32) == key) {
              atomicAdd(&slot64[sk], 1ull);
              break;
            }
            if (vk == kEmpty64) {
              const unsigned long long old =
                  atomicCAS(&slot64[sk], kEmpty64, ((unsigned long long)key << 32) | 1ull);
              if (old == kEmpty64) break;
              if ((uint32_t)(old >> 32) == key) {
                atomicAdd(&slot64[sk], 1ull);
                break;
              }
            }
            if (++sk == width) sk = 0;
            vk = slot64[sk];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < D; ++k) cur[k] = nxt[k];
    }
    }
    if (threadIdx.x == 0) s_misc[0] = u_next;
    __syncthreads();
    if (DBG) {
      c2 = clock64();
      if (threadIdx.x == 0) {
        const int kind = !dense ? 3 : (T.n_units > 1 ? 2 : (T.row1 - T.row0 == 1 ? 0 : 1));
        atomicAdd(&A.dbg[kind * 5 + 0], (unsigned long long)(c1 - c0));
        atomicAdd(&A.dbg[kind * 5 + 1], (unsigned long long)(c2 - c1));
        atomicAdd(&A.dbg[kind * 5 + 3], 1ull);
        atomicAdd(&A.dbg[kind * 5 + 4], (unsigned long long)(w1 - w0));  // words or entries
      }
    }
    if (dense && T.n_units > 1) {
      uint4* dst = reinterpret_cast<uint4*>(A.slabs + (T.slab_base + unit.local) * (uint64_t)kSHalf);
      const uint4* src = reinterpret_cast<const uint4*>(table);
      for (uint32_t s = threadIdx.x; s < (dwords + 3) / 4; s += kSCThreads) __stcg(dst + s, src[s]);
      __syncthreads();
      continue;
    }
    // compaction: count occupied counters, one output claim per unit, emit.
    // Dense: 4 table words per lane per step, each holding slots w and
    // w + kSHalf; hash: 2 slots per lane per step.
    const uint32_t span = dense ? dwords : width;
    const uint32_t per_w = (((span + kSCWarps - 1) / kSCWarps) + 127) & ~127u;
    const uint32_t s_lo = min(span, warp * per_w), s_hi = min(span, s_lo + per_w);
    uint32_t mine = 0;
    if (dense) {
      for (uint32_t s = s_lo + 4 * lane; s < s_hi; s += 128) {
        const uint4 c4 = *reinterpret_cast<const uint4*>(table + s);  // table padded to 4
        const uint32_t cw[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (s + q < s_hi)
            mine += ((cw[q] & 0xFFFFu) != 0) + ((cw[q] >> 16) != 0 && s + q + kSHalf < width);
      }
    } else {
      for (uint32_t s = s_lo + 2 * lane; s < s_hi; s += 64) {
        const ulonglong2 c2v = *reinterpret_cast<const ulonglong2*>(slot64 + s);
        mine += (c2v.x != kEmpty64) + (s + 1 < s_hi && c2v.y != kEmpty64);
      }
    }
    mine = warp_sum(mine);
    uint32_t total;
    uint32_t wbase = block_excl_scan(lane == 0 ? mine : 0, s_warp, total);
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (threadIdx.x == 0) s_base = atomicAdd(A.out_n, (unsigned long long)total);
    __syncthreads();
    uint64_t pos = s_base + wbase;
    // past the output capacity: claim only (the host sees n > capacity)
    const bool fits = s_base + total <= A.out_cap;
    const bool single_row = dense && T.row1 - T.row0 == 1;
    // emit: consecutive lanes own consecutive table words (dense: word w
    // holds slots w and w + kSHalf) or hash slots, and a ballot compacts each
    // step's non-zero counters to consecutive output positions -- every
    // store instruction writes one contiguous run of entries
    const uint32_t lt = (1u << lane) - 1u;
    auto put = [&](uint64_t o, uint32_t i, uint32_t j, uint32_t c) {
      A.out_row[o] = i;
      A.out_col[o] = j;
      A.out_count[o] = c;
      note_high(A, c, o);
    };
    if (dense) {
      for (uint32_t s0 = s_lo; fits && s0 < s_hi; s0 += 32) {
        const uint32_t w = s0 + lane;
        const uint32_t cw = w < s_hi ? table[w] : 0u;
        const uint32_t c_lo = cw & 0xFFFFu;
        const uint32_t c_hi = w + kSHalf < width ? cw >> 16 : 0u;
        const uint32_t m_lo = __ballot_sync(0xffffffffu, c_lo != 0);
        const uint32_t m_hi = __ballot_sync(0xffffffffu, c_hi != 0);
        uint32_t i, j;
        if (c_lo) {
          if (single_row) {
            i = T.row0;
            j = w + T.c0;
          } else {
            dense_slot_pair(T, w, n, A.upper != 0, i, j);
          }
          put(pos + __popc(m_lo & lt), i, j, c_lo);
        }
        pos += __popc(m_lo);
        if (c_hi) {
          const uint32_t slot = w + kSHalf;
          if (single_row) {
            i = T.row0;
            j = slot + T.c0;
          } else {
            dense_slot_pair(T, slot, n, A.upper != 0, i, j);
          }
          put(pos + __popc(m_hi & lt), i, j, c_hi);
        }
        pos += __popc(m_hi);
      }
    } else {
      for (uint32_t s0 = s_lo; fits && s0 < s_hi; s0 += 32) {
        const uint32_t sl = s0 + lane;
        const unsigned long long v = sl < s_hi ? slot64[sl] : kEmpty64;
        const bool occ = v != kEmpty64;
        const uint32_t m = __ballot_sync(0xffffffffu, occ);
        if (occ) {
          const uint32_t key = (uint32_t)(v >> 32);
          uint32_t i, j;
          if (hwin) {
            i = T.row0;
            j = key + T.c0;
          } else {
            i = T.row0 + (key >> A.col_bits);
            j = key & ((1u << A.col_bits) - 1u);
          }
          put(pos + __popc(m & lt), i, j, (uint32_t)v);
        }
        pos += __popc(m);
      }
    }
    __syncthreads();
    if (DBG && threadIdx.x == 0) {
      const int kind = !dense ? 3 : (T.n_units > 1 ? 2 : (T.row1 - T.row0 == 1 ? 0 : 1));
      atomicAdd(&A.dbg[kind * 5 + 2], (unsigned long long)(clock64() - c2));
    }
  }
}

// Sum the slabs of each split dense tile and compact the sums: one block per
// (tile, 2048-slot chunk) of the job's chunk list; each thread owns 8 slots
// (two uint4) and reads four units' slabs per step.
constexpr uint32_t kReduceSlots = 2048;
__global__ void __launch_bounds__(256) k_reduce_slabs(StreamCountArgs A, const uint2* __restrict__ chunks,
                                                      uint32_t n_chunks) {
  // chunk = (split tile, first table word): each thread owns 8 words = 16
  // slots (w and w + kSHalf) and sums them over the tile's unit slabs
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_base;
  for (uint32_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const uint2 ch = chunks[ci];
    const Tile T = A.tiles[ch.x];
    const uint32_t w0 = ch.y + threadIdx.x * 8;
    const uint32_t nu = T.n_units;
    const uint32_t dwords = T.width < kSHalf ? T.width : kSHalf;
    const uint32_t* base = A.slabs + (uint64_t)T.slab_base * kSHalf + w0;
    uint32_t lo[8] = {0, 0, 0, 0, 0, 0, 0, 0}, hi[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (w0 < dwords) {
      for (uint32_t v = 0; v < nu; ++v) {
        const uint4* p = reinterpret_cast<const uint4*>(base + (uint64_t)v * kSHalf);
        const uint4 a = __ldcs(p), b = __ldcs(p + 1);
        const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          lo[k] += x[k] & 0xFFFFu;
          hi[k] += x[k] >> 16;
        }
      }
    }
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (w0 + k >= dwords) break;
      mine += (lo[k] != 0) + (hi[k] != 0 && w0 + k + kSHalf < T.width);
    }
    uint32_t total;
    const uint32_t excl = block_excl_scan(mine, s_warp, total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(A.out_n, (unsigned long long)total) : 0ull;
    __syncthreads();
    uint64_t o = s_base + excl;
    const bool fits = s_base + total <= A.out_cap;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t w = w0 + (k & 7);
      const uint32_t slot = w + (k >= 8 ? kSHalf : 0u);
      const uint32_t c = k >= 8 ? hi[k & 7] : lo[k & 7];
      if (fits && w < dwords && slot < T.width && c != 0) {
        uint32_t i, j;
        dense_slot_pair(T, slot, A.n_items, A.upper != 0, i, j);
        A.out_row[o] = i;
        A.out_col[o] = j;
        A.out_count[o] = c;
        note_high(A, c, o);
        ++o;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) k_scan_u64(const unsigned long long* __restrict__ in,
                                                   uint32_t n, unsigned long long* __restrict__ out,
                                                   unsigned long long* __restrict__ out2) {
  // single block exclusive scan; out2 (optional) receives a copy
  __shared__ unsigned long long s_part[1024];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
  // every tile's range is rounded up to an even word count, so 8-byte
  // entries stay aligned
  unsigned long long acc = 0;
  for (uint32_t i = lo; i < hi; ++i) acc += (in[i] + 1) & ~1ull;
  s_part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long run = 0;
    for (int k = 0; k < 32; ++k) run += s_part[threadIdx.x * 32 + k];
    unsigned long long x = run;
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
      if ((int)threadIdx.x >= d) x += y;
    }
    unsigned long long a = x - run;
    for (int k = 0; k < 32; ++k) {
      const unsigned long long v = s_part[threadIdx.x * 32 + k];
      s_part[threadIdx.x * 32 + k] = a;
      a += v;
    }
  }
  __syncthreads();
  unsigned long long run = s_part[threadIdx.x];
  for (uint32_t i = lo; i < hi; ++i) {
    out[i] = run;
    if (out2) out2[i] = run;
    run += (in[i] + 1) & ~1ull;
  }
}


// ============================================================ GPU planner
// Stream-mode tile plan computed on the device in one CTA (no host round trip
// with the per-item statistics). Same tile kinds as the host planner, packed
// in parallel instead of greedily:
//   H  one dense single-row tile (entries unless filtered) for a row that is
//      dense-worthy (8 t >= w and w >= 4096) or too heavy for a hash tile;
//   W  column windows for a row wider than the table and too heavy to hash;
//   L1 a single-row hash tile for a light row with a large distinct bound;
//   L  light rows packed into hash tiles by the prefix of a fixed-point
//      weight max(b / hash_cap, t / unit_terms) + span: a tile is the set of
//      light rows whose exclusive prefix falls in one bucket of width
//      S - xmax - y, so every tile stays within all three capacities.
// Rows are processed in contiguous segments (one per thread) with block
// scans carrying prefixes, buckets and tile ids across segments.
struct PlanOut {
  unsigned long long total_terms, occ_sum, max_entries, n_slabs;
  uint32_t n_tiles, n_units, n_split, n_reduce_chunks;
  uint32_t stream_mode, overflow, pad0, pad1;
  long long dbg[4];  // development: planner phase cycles
  uint32_t words_known, pad2;  // per-tile word totals written (no word-count pass needed)
  unsigned long long own_words;  // bound on this shard's stream words (allocation; < 2^32)
  unsigned long long own_terms;  // this shard's terms (window tiles: estimates)
};

struct PlanArgs {
  const unsigned long long* stats;
  uint32_t n, col_bits;
  int upper, filter, force;  // force: 0 auto, 1 entry, 2 stream
  int own;  // filtered job planned on own terms (Lemma-1 layout): word totals known
  int safe;  // CROP_PAIRS_SAFE_UNITS: word-counted dense units hold <= 65,535 words
  unsigned long long unit_terms;  // 0: default; CROP_DEBUG_UNIT_TERMS (tests: large units)
  Tile* tiles;
  uint32_t tile_cap;
  Unit* units;
  uint32_t unit_cap;
  uint32_t* split;
  uint2* reduce_chunks;
  uint32_t rc_cap;
  uint2* item_info;
  unsigned long long* tile_words;  // per-tile stream words, when knowable from the statistics
  uint32_t shard_rank, shard_world;  // tile sharding: keep the tiles of this rank's term share
  PlanOut* out;
};

constexpr int kPlanThreads = 1024;
constexpr uint32_t kMaxShardCheck = 1024;  // owners tracked by the per-shard word check
constexpr uint64_t kPlanS = 1ull << 24;  // fixed-point capacity of one light tile
constexpr uint32_t kMinDenseWidth = 4096;

template <typename T, typename Op>
__device__ __forceinline__ T plan_block_scan(T v, T* s_tmp, T ident, Op op, T& total) {
  // exclusive scan of one value per thread over kPlanThreads threads
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = op(x, u);
  }
  if (lane == 31) s_tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    T y = s_tmp[lane];
    T yi = y;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T u = __shfl_up_sync(0xffffffffu, yi, d);
      if (lane >= d) yi = op(yi, u);
    }
    const T ex = __shfl_up_sync(0xffffffffu, yi, 1);
    s_tmp[lane] = lane ? ex : ident;
    if (lane == 31) s_tmp[32] = yi;
  }
  __syncthreads();
  const T ex_lane = __shfl_up_sync(0xffffffffu, x, 1);
  const T r = op(s_tmp[w], lane ? ex_lane : ident);
  total = s_tmp[32];
  __syncthreads();
  return r;
}

// Row record in shared memory: class (3 bits) | weight or #windows << 3.
constexpr uint32_t kPlanRowsPerThread = 8;
constexpr uint32_t kPlanChunk = kPlanThreads * kPlanRowsPerThread;  // rows staged per step

__global__ void __launch_bounds__(kPlanThreads, 1) k_plan_stream(PlanArgs P) {
  __shared__ unsigned long long s_u64[33];
  __shared__ long long s_i64[33];
  __shared__ uint32_t s_bin[65], s_cur[65];
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_rec = s_dyn;               // per staged row: class | weight << 3
  uint32_t* s_t = s_dyn + kPlanChunk;    // per staged row: terms (< 2^32 in stream mode)
  const uint32_t n = P.n, tid = threadIdx.x;
  long long ck[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long c_last = clock64();
  auto stamp = [&](int q) {
    const long long now = clock64();
    ck[q] += now - c_last;
    c_last = now;
  };
  auto add = [](unsigned long long a, unsigned long long b) { return a + b; };
  auto mx = [](long long a, long long b) { return a > b ? a : b; };
  long long totl;
  // 1. totals (coalesced) and the mode decision
  unsigned long long T = 0, O = 0;
  for (uint32_t i = tid; i < n; i += kPlanThreads) {
    const unsigned long long x = P.stats[i];
    T += x & (kOccOne - 1);
    O += x >> kOccShift;
  }
  plan_block_scan<unsigned long long>(T, s_u64, 0ull, add, T);
  plan_block_scan<unsigned long long>(O, s_u64, 0ull, add, O);
  // word positions are 32-bit: a whole job must fit; a shard is checked on
  // its own words once the tiles are assigned (below)
  const bool fits = P.shard_world > 1 || T + 2 * O + 2ull * n + 2 < (1ull << 32);
  const bool short_rows = O > 0 && T <= (unsigned long long)kStreamMeanMax * O;
  bool sm = fits && short_rows;
  if (P.force == 1) sm = false;
  if (P.force == 2) sm = fits;
  if (tid == 0) {
    P.out->total_terms = T;
    P.out->occ_sum = O;
    P.out->stream_mode = sm;
    // short rows whose words do not fit one job: split into tile shards
    // (every shard size is decided from the whole plan, so all ranks agree)
    P.out->overflow = (!fits && short_rows && P.force == 0) ? 2u : 0u;
  }
  if (!sm) return;
  stamp(0);
  const uint64_t unit_terms = P.unit_terms ? P.unit_terms : max(1ull << 16, T / ((uint64_t)kNumSMs * 8));
  const double inv_ut = (double)kPlanS / (double)unit_terms;
  const uint32_t rows_max = P.col_bits >= 32 ? 1u : ((1u << (32 - P.col_bits)) - 1u);
  const uint64_t y = (kPlanS + rows_max - 1) / rows_max;  // span weight of every row
  // bucket width, with a margin for the rounding of the double reciprocal
  const uint64_t step = kPlanS - kPlanS / 4 - y - 1024;
  const double inv_step = 1.0 / (double)step;
  auto bucket = [inv_step](unsigned long long p) { return (long long)((double)p * inv_step); };
  const uint64_t dense_cap = kStreamDenseCap, hash_cap = kStreamHashCap;
  // units: by terms for balance, and <= kStreamUnitOcc row occurrences each
  // (16-bit dense counters)
  auto units_of = [&](uint64_t t, uint64_t occ) -> uint32_t {
    uint64_t u = (t + unit_terms - 1) / unit_terms;
    const uint64_t uo = (occ + kStreamUnitOcc - 1) / kStreamUnitOcc;
    if (uo > u) u = uo;
    return (uint32_t)(u < 1 ? 1 : (u > 65535 ? 65535 : u));
  };
  // carries across chunks
  __shared__ uint32_t s_has_win;
  if (tid == 0) s_has_win = 0;
  unsigned long long c_p = 0, c_tiles = 0;
  long long c_bucket = -1, c_lt = -1, c_lrow0 = -1;
  for (uint32_t base = 0; base < n; base += kPlanChunk) {
    const uint32_t cn = min(kPlanChunk, n - base);
    // classify: 1 H, 2 W (record = #windows), 3 L1, 4 L (record = weight), 0 none
    // rows in batches of 8 loads in flight (registers: 64 per thread)
    for (uint32_t qb = 0; qb < kPlanRowsPerThread; qb += 8) {
    unsigned long long st8[8];
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      const uint32_t k = tid + (qb + q) * kPlanThreads;
      st8[q] = k < cn ? P.stats[base + k] : 0ull;
    }
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      const uint32_t k = tid + (qb + q) * kPlanThreads;
      if (k >= cn) break;
      const uint32_t i = base + k;
      const uint64_t t = st8[q] & (kOccOne - 1);
      const uint64_t w = P.upper ? (uint64_t)(n - 1 - i) : (uint64_t)n;
      s_t[k] = (uint32_t)t;
      uint32_t rec = 0;
      if (t) {
        const uint64_t b = t < w ? t : w;
        const bool hfit = b <= hash_cap && t <= unit_terms;
        if (w <= dense_cap && ((8 * t >= w && w >= kMinDenseWidth) || !hfit)) {
          rec = 1;
        } else if (!hfit) {
          rec = 2 | (uint32_t)((w + dense_cap - 1) / dense_cap) << 3;
          s_has_win = 1;
        } else {
          const uint64_t xb = (b * kPlanS + hash_cap - 1) / hash_cap;
          const uint64_t xt = (uint64_t)((double)t * inv_ut) + 1;  // >= t * S / unit_terms
          const uint64_t x = xb > xt ? xb : xt;
          rec = x > kPlanS / 4 ? 3u : (4u | (uint32_t)x << 3);
        }
      }
      s_rec[k] = rec;
    }
    }
    __syncthreads();
    stamp(1);
    const uint32_t lo = min(cn, tid * kPlanRowsPerThread), hi = min(cn, lo + kPlanRowsPerThread);
    // weights prefix
    unsigned long long pw = 0;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t r = s_rec[k];
      pw += ((r & 7) == 4 ? (r >> 3) : 0) + y;
    }
    unsigned long long chunk_w;
    const unsigned long long pbase = c_p + plan_block_scan<unsigned long long>(pw, s_u64, 0ull, add, chunk_w);
    // last light bucket of each thread -> carry
    long long lastb = -1;
    {
      unsigned long long p = pbase;
      for (uint32_t k = lo; k < hi; ++k) {
        const uint32_t r = s_rec[k];
        if ((r & 7) == 4) lastb = bucket(p);
        p += ((r & 7) == 4 ? (r >> 3) : 0) + y;
      }
    }
    long long carryb = plan_block_scan<long long>(lastb, s_i64, -1ll, mx, totl);
    carryb = carryb > c_bucket ? carryb : c_bucket;
    const long long chunk_lastb = totl > c_bucket ? totl : c_bucket;
    // tiles per thread
    unsigned long long cnt = 0;
    {
      unsigned long long p = pbase;
      long long lb = carryb;
      for (uint32_t k = lo; k < hi; ++k) {
        const uint32_t r = s_rec[k], c = r & 7;
        if (c == 1 || c == 3) cnt += 1;
        else if (c == 2) cnt += r >> 3;
        else if (c == 4) {
          const long long bk = bucket(p);
          if (bk != lb) cnt += 1;
          lb = bk;
        }
        p += (c == 4 ? (r >> 3) : 0) + y;
      }
    }
    stamp(2);
    unsigned long long chunk_tiles;
    const unsigned long long tbase = c_tiles + plan_block_scan<unsigned long long>(cnt, s_u64, 0ull, add, chunk_tiles);
    if (c_tiles + chunk_tiles > P.tile_cap) {
      if (tid == 0) P.out->overflow = 1;
      return;
    }
    // write the tiles; the last light tile each thread starts (id, first row)
    long long last_lt = -1, last_row0 = -1;
    {
      unsigned long long p = pbase;
      long long lb = carryb;
      uint32_t id = (uint32_t)tbase;
      for (uint32_t k = lo; k < hi; ++k) {
        const uint32_t r = s_rec[k], c = r & 7, i = base + k;
        if (c == 1 || c == 3) {
          const uint64_t t = s_t[k];
          Tile tl{};
          tl.row0 = i;
          tl.row1 = i + 1;
          tl.c1 = n;
          tl.terms = t;
          if (c == 1) {
            tl.c0 = P.upper ? i + 1 : 0;
            tl.mode = P.filter ? 0 : 2;
            tl.width = P.upper ? n - 1 - i : n;
            const uint64_t occ = P.stats[i] >> kOccShift;
            tl.n_units = units_of(t, (P.safe && tl.mode == 0 && t > occ) ? t : occ);
          } else {
            tl.mode = 1;
            tl.n_units = 1;
          }
          P.tiles[id] = tl;
          P.item_info[i] = make_uint2(id | (tl.mode == 2 ? kEntFlag : 0u),
                                      stream_base(tl, i, n, P.col_bits, P.upper != 0));
          ++id;
        } else if (c == 2) {
          const uint64_t t = s_t[k];
          const uint32_t col_lo = P.upper ? i + 1 : 0;
          const uint32_t nwin = r >> 3;
          for (uint32_t q = 0; q < nwin; ++q) {
            Tile tl{};
            tl.row0 = i;
            tl.row1 = i + 1;
            tl.c0 = col_lo + q * (uint32_t)dense_cap;
            tl.c1 = (uint32_t)min((uint64_t)n, (uint64_t)tl.c0 + dense_cap);
            tl.mode = 0;
            tl.nwin = q == 0 ? nwin : 0;
            tl.width = tl.c1 - tl.c0;
            tl.terms = t / nwin + 1;
            const uint64_t occ = P.stats[i] >> kOccShift;
            tl.n_units = units_of(tl.terms, (P.safe && tl.terms > occ) ? tl.terms : occ);
            P.tiles[id + q] = tl;
          }
          P.item_info[i] = make_uint2(id | kWinFlag, 0u);
          id += nwin;
        } else if (c == 4) {
          const long long bk = bucket(p);
          if (bk != lb) {
            Tile tl{};
            tl.row0 = i;
            tl.row1 = i + 1;
            tl.c1 = n;
            tl.mode = 1;
            tl.n_units = 1;
            P.tiles[id] = tl;
            last_lt = id;
            last_row0 = i;
            ++id;
          }
          lb = bk;
        } else {
          P.item_info[i] = make_uint2(kNone, 0u);
        }
        p += (c == 4 ? (r >> 3) : 0) + y;
      }
    }
    stamp(3);
    long long carry_lt = plan_block_scan<long long>(last_lt, s_i64, -1ll, mx, totl);
    const long long chunk_lt = totl > c_lt ? totl : c_lt;
    carry_lt = carry_lt > c_lt ? carry_lt : c_lt;
    long long carry_row0 = plan_block_scan<long long>(last_row0, s_i64, -1ll, mx, totl);
    const long long chunk_row0 = totl > c_lrow0 ? totl : c_lrow0;
    carry_row0 = carry_row0 > c_lrow0 ? carry_row0 : c_lrow0;
    // light rows: tile, row range, terms, item_info
    {
      // per thread, the rows of one light tile are consecutive: accumulate
      // its terms and last row, one pair of global atomics per tile change
      unsigned long long p = pbase;
      long long lb = carryb, cur = carry_lt, row0 = carry_row0;
      uint32_t id = (uint32_t)tbase;
      long long acc_tile = -1;
      unsigned long long acc_terms = 0;
      uint32_t acc_row1 = 0;
      auto flush = [&]() {
        if (acc_tile >= 0) {
          Tile* tl = P.tiles + acc_tile;
          atomicMax(&tl->row1, acc_row1);
          atomicAdd(reinterpret_cast<unsigned long long*>(&tl->terms), acc_terms);
        }
      };
      for (uint32_t k = lo; k < hi; ++k) {
        const uint32_t r = s_rec[k], c = r & 7, i = base + k;
        if (c == 1 || c == 3) ++id;
        else if (c == 2) id += r >> 3;
        else if (c == 4) {
          const long long bk = bucket(p);
          if (bk != lb) {
            cur = id++;
            row0 = i;
          }
          lb = bk;
          if (cur != acc_tile) {
            flush();
            acc_tile = cur;
            acc_terms = 0;
          }
          acc_terms += s_t[k];
          acc_row1 = i + 1;
          P.item_info[i] = make_uint2((uint32_t)cur, (i - (uint32_t)row0) << P.col_bits);
        }
        p += (c == 4 ? (r >> 3) : 0) + y;
      }
      flush();
    }
    stamp(4);
    c_p += chunk_w;
    c_tiles += chunk_tiles;
    c_bucket = chunk_lastb;
    c_lt = chunk_lt;
    c_lrow0 = chunk_row0;
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  const uint32_t nt = (uint32_t)c_tiles;
  if (P.shard_world > 1) {
    // tile sharding: rank r keeps the tiles whose cost prefix (tile_cost)
    // falls in the r-th of shard_world equal shares (the windows of one row
    // follow the row's first window); the others get no units, no words and
    // no rows.
    // The owner is parked in slab_base until the units phase.
    const uint32_t ts = (nt + kPlanThreads - 1) / kPlanThreads;
    const uint32_t a = min(nt, tid * ts), b = min(nt, a + ts);
    auto is_window = [&](const Tile& tl) {
      return tl.mode == 0 && tl.row1 - tl.row0 == 1 && tl.width < (P.upper ? n - 1 - tl.row0 : n);
    };
    // stream words of a tile (bounds as in the units phase below): a window's
    // words are bounded by its row's terms, carried by the row's first window
    auto words_of = [&](const Tile& tl) -> unsigned long long {
      if (is_window(tl)) return 2 + (tl.nwin ? (P.stats[tl.row0] & (kOccOne - 1)) : 0ull);
      return 2 + (tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms);
    };
    auto cost = [&](const Tile& tl) -> unsigned long long {
      // a sparse column window counts in a hash table sized to its words
      // (k_count_stream hwin): cost it as a hash tile of its average words
      if (is_window(tl) && tl.n_units == 1 && tl.terms <= kSparseWindowWords) {
        Tile h = tl;
        h.mode = 1;
        return tile_cost(h, stream_hash_slots(tl.terms));
      }
      return tile_cost(tl, stream_hash_slots(tl.terms < hash_cap ? tl.terms : hash_cap));
    };
    __shared__ unsigned long long s_ow[kMaxShardCheck];
    // pass 0: shares of the counting cost; if a share's words pass the
    // 32-bit word positions, shares of the words (plus a per-unit overhead,
    // then without it); if even those do not fit, every rank asks for a
    // finer split (the decision depends only
    // on the whole plan, so all ranks agree)
    // (pass 1 adds a per-unit overhead to the words: ~2,048 words' worth of
    // clearing, compaction and unit scheduling; pass 2 is words only)
    for (int pass = 0; pass < 3; ++pass) {
      auto metric = [&](const Tile& tl) -> unsigned long long {
        if (pass == 0) return cost(tl);
        return words_of(tl) + (pass == 1 ? 2048ull * (tl.n_units ? tl.n_units : 1) : 0ull);
      };
      unsigned long long tsum = 0, all;
      for (uint32_t t = a; t < b; ++t) tsum += metric(P.tiles[t]);
      unsigned long long pre = plan_block_scan<unsigned long long>(tsum, s_u64, 0ull, add, all);
      // owner = floor(midpoint * world / all): a rank's k sub-shards of a
      // k-times finer split (r*k + s of world*k) own exactly its tiles
      for (uint32_t t = a; t < b; ++t) {
        const unsigned long long c = metric(P.tiles[t]);
        const unsigned long long ow = all ? (pre + c / 2) * P.shard_world / all : 0;  // tile midpoint
        P.tiles[t].slab_base = ow < P.shard_world - 1 ? ow : P.shard_world - 1;
        pre += c;
      }
      for (uint32_t k = tid; k < kMaxShardCheck; k += kPlanThreads) s_ow[k] = 0;
      __threadfence_block();
      __syncthreads();
      {
        // per thread a contiguous tile range: a continuation window takes the
        // owner of the tile before it (its row's previous window); the owner
        // rarely changes inside a range, so one shared atomic per change
        uint32_t cur = kNone;
        unsigned long long acc = 0;
        for (uint32_t t = a; t < b; ++t) {
          const Tile& tl = P.tiles[t];
          uint32_t ow;
          if (is_window(tl) && tl.nwin == 0 && t > a) {
            ow = cur;
          } else {
            uint32_t f = t;
            if (is_window(tl))
              while (P.tiles[f].nwin == 0 && f > 0) --f;  // the row's first window
            ow = (uint32_t)P.tiles[f].slab_base;
          }
          if (ow != cur) {
            if (cur != kNone) atomicAdd(&s_ow[cur < kMaxShardCheck ? cur : kMaxShardCheck - 1], acc);
            cur = ow;
            acc = 0;
          }
          acc += words_of(tl);
        }
        if (cur != kNone) atomicAdd(&s_ow[cur < kMaxShardCheck ? cur : kMaxShardCheck - 1], acc);
      }
      __syncthreads();
      unsigned long long mxw = 0;
      for (uint32_t k = tid; k < kMaxShardCheck; k += kPlanThreads) mxw = s_ow[k] > mxw ? s_ow[k] : mxw;
      plan_block_scan<long long>((long long)mxw, s_i64, 0ll, mx, totl);
      if (totl + 2 < (1ll << 32)) break;
      if (pass == 2) {
        if (tid == 0) P.out->overflow = 2;
        return;
      }
    }
    {
      // drop the other ranks' tiles (the owner walk reads slab_base and the
      // window fields only, never n_units)
      uint32_t cur = kNone;
      for (uint32_t t = a; t < b; ++t) {
        Tile& tl = P.tiles[t];
        if (!(is_window(tl) && tl.nwin == 0 && t > a)) {
          uint32_t f = t;
          if (is_window(tl))
            while (P.tiles[f].nwin == 0 && f > 0) --f;
          cur = (uint32_t)P.tiles[f].slab_base;
        }
        if (cur != P.shard_rank) tl.n_units = 0;
      }
    }
    __threadfence_block();
    __syncthreads();
    for (uint32_t t = tid; t < nt; t += kPlanThreads) P.tiles[t].slab_base = 0;
    for (uint32_t i = tid; i < n; i += kPlanThreads) {
      const uint2 tv = P.item_info[i];
      if (tv.x != kNone && P.tiles[tv.x & kTileMask].n_units == 0) P.item_info[i] = make_uint2(kNone, 0u);
    }
    __threadfence_block();
    __syncthreads();
  }
  // units, slabs, split list, reduce chunks, output capacity. Per-tile unit
  // counts and widths are cached in shared memory when they fit (hash tiles
  // report width 0 and count kStreamHashSlots output slots).
  const bool cached = nt <= kPlanChunk;
  uint32_t* s_nu = s_dyn;
  uint32_t* s_wd = s_dyn + kPlanChunk;
  for (uint32_t t = tid; t < nt; t += kPlanThreads) {
    Tile& tl = P.tiles[t];
    // hash tiles: table size from the key bound (the row terms bound the keys)
    if (tl.mode == 1) tl.width = stream_hash_slots(tl.terms < hash_cap ? tl.terms : hash_cap);
    if (cached) {
      s_nu[t] = tl.n_units;
      s_wd[t] = tl.mode != 1 ? tl.width : 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  auto nu_of = [&](uint32_t t) { return cached ? s_nu[t] : P.tiles[t].n_units; };
  auto wd_of = [&](uint32_t t) {
    return cached ? s_wd[t] : (P.tiles[t].mode != 1 ? P.tiles[t].width : 0xFFFFFFFFu);
  };
  const uint32_t tseg = (nt + kPlanThreads - 1) / kPlanThreads;
  const uint32_t tlo = min(nt, tid * tseg), thi = min(nt, tlo + tseg);
  unsigned long long a_slab = 0, a_split = 0, a_single = 0, a_rc = 0, a_cap = 0, a_units = 0;
  unsigned long long a_words = 0, a_terms = 0;
  for (uint32_t t = tlo; t < thi; ++t) {
    const uint32_t nu_t = nu_of(t), wd = wd_of(t);
    if (nu_t == 0) continue;  // another rank's tile
    {
      // stream words: a window's words are bounded by its row's terms (counted
      // once, at the row's first window), an entry tile stores 2 per row
      // occurrence, other tiles one per term; + 2 for the even rounding
      const Tile& tl = P.tiles[t];
      const bool win = tl.mode == 0 && tl.row1 - tl.row0 == 1 &&
                       tl.width < (P.upper ? n - 1 - tl.row0 : n);
      if (win) a_words += tl.nwin ? (P.stats[tl.row0] & (kOccOne - 1)) : 0ull;
      else a_words += tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms;
      a_words += 2;
      a_terms += tl.terms;
    }
    a_cap += tile_out_cap(P.tiles[t], kStreamHashCap, n, P.upper != 0);
    a_units += nu_t;
    if (nu_t > 1) {
      a_slab += nu_t;
      a_split += 1;
      a_rc += ((wd < kSHalf ? wd : kSHalf) + kReduceSlots - 1) / kReduceSlots;
    } else {
      a_single += 1;
    }
  }
  unsigned long long n_slabs, n_split, n_single, n_rc, cap, nu;
  const unsigned long long b_slab = plan_block_scan<unsigned long long>(a_slab, s_u64, 0ull, add, n_slabs);
  const unsigned long long b_split = plan_block_scan<unsigned long long>(a_split, s_u64, 0ull, add, n_split);
  const unsigned long long b_single = plan_block_scan<unsigned long long>(a_single, s_u64, 0ull, add, n_single);
  const unsigned long long b_rc = plan_block_scan<unsigned long long>(a_rc, s_u64, 0ull, add, n_rc);
  plan_block_scan<unsigned long long>(a_cap, s_u64, 0ull, add, cap);
  plan_block_scan<unsigned long long>(a_units, s_u64, 0ull, add, nu);
  unsigned long long own_words, own_terms;
  plan_block_scan<unsigned long long>(a_words, s_u64, 0ull, add, own_words);
  plan_block_scan<unsigned long long>(a_terms, s_u64, 0ull, add, own_terms);
  if (nu > P.unit_cap || n_rc > P.rc_cap || own_words + 2 >= (1ull << 32)) {
    if (tid == 0) P.out->overflow = 1;
    return;
  }
  // unit order: split-tile units by the fraction of the tile they cover (64
  // bins, see the host planner), then the single-unit tiles (any order)
  constexpr int kFracBins = 64;
  for (int k = tid; k <= kFracBins; k += kPlanThreads) s_bin[k] = 0;
  {
    // slab bases, split list and reduce chunks in tile order
    uint64_t sb = b_slab, sp = b_split, rc = b_rc;
    for (uint32_t t = tlo; t < thi; ++t) {
      const uint32_t nu_t = nu_of(t), width = wd_of(t);
      if (nu_t > 1) {
        P.tiles[t].slab_base = sb;
        sb += nu_t;
        P.split[sp++] = t;
        const uint32_t dw = width < kSHalf ? width : kSHalf;
        for (uint32_t c0 = 0; c0 < dw; c0 += kReduceSlots) P.reduce_chunks[rc++] = make_uint2(t, c0);
      }
    }
  }
  __syncthreads();
  for (uint32_t t = tid; t < nt; t += kPlanThreads) {
    const uint32_t nu_t = nu_of(t);
    if (nu_t > 1)
      for (uint32_t u = 0; u < nu_t; ++u) atomicAdd(&s_bin[(uint64_t)(2 * u + 1) * kFracBins / (2 * nu_t)], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t run = 0;
    for (int k = 0; k < kFracBins; ++k) {
      s_cur[k] = run;
      run += s_bin[k];
    }
    s_cur[kFracBins] = run;
  }
  __syncthreads();
  for (uint32_t t = tid; t < nt; t += kPlanThreads) {
    const uint32_t nu_t = nu_of(t);
    if (nu_t > 1) {
      for (uint32_t u = 0; u < nu_t; ++u) {
        const uint32_t pos = atomicAdd(&s_cur[(uint64_t)(2 * u + 1) * kFracBins / (2 * nu_t)], 1u);
        P.units[pos] = Unit{t, u};
      }
    }
  }
  {
    // single-unit tiles after the split units, in tile order (the exclusive
    // prefix of each thread's contiguous range: no shared counter)
    uint64_t pos = s_cur[kFracBins] + b_single;
    for (uint32_t t = tlo; t < thi; ++t)
      if (nu_of(t) == 1) P.units[pos++] = Unit{t, 0};
  }
  // per-tile stream words from the statistics (unfiltered, no windows): an
  // entry tile stores 2 words per row occurrence with a partner after it,
  // a hash tile one word per term
  const bool known = (!P.filter || P.own) && !s_has_win;
  if (known)
    for (uint32_t t = tid; t < nt; t += kPlanThreads) {
      const Tile& tl = P.tiles[t];
      P.tile_words[t] = tl.n_units == 0 ? 0ull : (tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms);
    }
  stamp(5);
  if (tid == 0) {
    P.out->words_known = known;
    P.out->pad0 = (uint32_t)(ck[0] / 1000);
    P.out->pad1 = (uint32_t)(ck[1] / 1000);
    P.out->dbg[0] = ck[2];
    P.out->dbg[1] = ck[3];
    P.out->dbg[2] = ck[4];
    P.out->dbg[3] = ck[5];
    P.out->max_entries = cap;
    P.out->own_words = own_words + 2;
    P.out->own_terms = own_terms;
    P.out->n_slabs = n_slabs;
    P.out->n_tiles = nt;
    P.out->n_units = (uint32_t)nu;
    P.out->n_split = (uint32_t)n_split;
    P.out->n_reduce_chunks = (uint32_t)n_rc;
  }
}


// Cooperative form of k_plan_stream: the same plan, computed by one CTA per
// SM instead of one CTA (k_plan_stream walks every row and tile on one SM:
// 0.24 ms on c2, 5 ms on a c3 chunk). Each CTA takes a contiguous range of at
// most kPlanChunk rows (then of tiles); the sequential carries of the
// single-CTA planner (weight prefix, last light bucket, tile ids, last light
// tile and its first row, shard cost prefixes, unit bases) become grid-wide
// prefixes of per-CTA aggregates published in PlanScratch between grid
// syncs. Every decision is the single-CTA planner's, so the plans are
// identical (tests compare them).
constexpr uint32_t kMaxPlanCtas = 160;
struct PlanScratch {
  unsigned long long totals[2];  // T, O
  unsigned int has_win, pad;
  unsigned long long cw[kMaxPlanCtas];
  long long lastb[kMaxPlanCtas];
  unsigned long long ct[kMaxPlanCtas];
  long long llt[kMaxPlanCtas], lrow[kMaxPlanCtas];
  unsigned long long ssum[3][kMaxPlanCtas];
  unsigned long long sow[3][kMaxShardCheck];
  unsigned long long u8[kMaxPlanCtas][8];
  unsigned int bins[72];
  unsigned int cur[72];
};

__global__ void __launch_bounds__(kPlanThreads, 1) k_plan_coop(PlanArgs P, PlanScratch* S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long s_u64[33];
  __shared__ long long s_i64[33];
  __shared__ unsigned long long s_bc[8];
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_rec = s_dyn;               // per staged row: class | weight << 3
  uint32_t* s_t = s_dyn + kPlanChunk;    // per staged row: terms
  const uint32_t n = P.n, tid = threadIdx.x, nb = gridDim.x, cb = blockIdx.x;
  auto add = [](unsigned long long a, unsigned long long b) { return a + b; };
  auto mx = [](long long a, long long b) { return a > b ? a : b; };
  long long totl;
  // 1. totals and the mode decision
  {
    unsigned long long T = 0, O = 0;
    for (uint32_t i = cb * kPlanThreads + tid; i < n; i += nb * kPlanThreads) {
      const unsigned long long x = P.stats[i];
      T += x & (kOccOne - 1);
      O += x >> kOccShift;
    }
    plan_block_scan<unsigned long long>(T, s_u64, 0ull, add, T);
    plan_block_scan<unsigned long long>(O, s_u64, 0ull, add, O);
    if (tid == 0) {
      atomicAdd(&S->totals[0], T);
      atomicAdd(&S->totals[1], O);
    }
  }
  grid.sync();
  const unsigned long long T = S->totals[0], O = S->totals[1];
  const bool fits = P.shard_world > 1 || T + 2 * O + 2ull * n + 2 < (1ull << 32);
  const bool short_rows = O > 0 && T <= (unsigned long long)kStreamMeanMax * O;
  bool sm = fits && short_rows;
  if (P.force == 1) sm = false;
  if (P.force == 2) sm = fits;
  if (cb == 0 && tid == 0) {
    P.out->total_terms = T;
    P.out->occ_sum = O;
    P.out->stream_mode = sm;
    P.out->overflow = (!fits && short_rows && P.force == 0) ? 2u : 0u;
  }
  if (!sm) return;
  const uint64_t unit_terms = P.unit_terms ? P.unit_terms : max(1ull << 16, T / ((uint64_t)kNumSMs * 8));
  const double inv_ut = (double)kPlanS / (double)unit_terms;
  const uint32_t rows_max = P.col_bits >= 32 ? 1u : ((1u << (32 - P.col_bits)) - 1u);
  const uint64_t y = (kPlanS + rows_max - 1) / rows_max;
  const uint64_t step = kPlanS - kPlanS / 4 - y - 1024;
  const double inv_step = 1.0 / (double)step;
  auto bucket = [inv_step](unsigned long long p) { return (long long)((double)p * inv_step); };
  const uint64_t dense_cap = kStreamDenseCap, hash_cap = kStreamHashCap;
  auto units_of = [&](uint64_t t, uint64_t occ) -> uint32_t {
    uint64_t u = (t + unit_terms - 1) / unit_terms;
    const uint64_t uo = (occ + kStreamUnitOcc - 1) / kStreamUnitOcc;
    if (uo > u) u = uo;
    return (uint32_t)(u < 1 ? 1 : (u > 65535 ? 65535 : u));
  };
  // sum / max of the per-CTA values before this CTA (thread 0 -> s_bc)
  auto before_sum = [&](const unsigned long long* a, unsigned long long& all) -> unsigned long long {
    if (tid == 0) {
      unsigned long long s = 0, t = 0;
      for (uint32_t k = 0; k < nb; ++k) {
        if (k == cb) s = t;
        t += a[k];
      }
      s_bc[0] = s;
      s_bc[1] = t;
    }
    __syncthreads();
    const unsigned long long r = s_bc[0];
    all = s_bc[1];
    __syncthreads();
    return r;
  };
  auto before_max = [&](const long long* a) -> long long {
    if (tid == 0) {
      long long m = -1;
      for (uint32_t k = 0; k < cb; ++k) m = a[k] > m ? a[k] : m;
      s_bc[2] = (unsigned long long)m;
    }
    __syncthreads();
    const long long r = (long long)s_bc[2];
    __syncthreads();
    return r;
  };
  // 2. rows [r0, r1) of this CTA
  const uint32_t r0 = (uint32_t)((uint64_t)n * cb / nb), r1 = (uint32_t)((uint64_t)n * (cb + 1) / nb);
  const uint32_t base = r0, cn = r1 - r0;
  for (uint32_t qb = 0; qb < kPlanRowsPerThread; qb += 8) {
    unsigned long long st8[8];
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      const uint32_t k = tid + (qb + q) * kPlanThreads;
      st8[q] = k < cn ? P.stats[base + k] : 0ull;
    }
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      const uint32_t k = tid + (qb + q) * kPlanThreads;
      if (k >= cn) break;
      const uint32_t i = base + k;
      const uint64_t t = st8[q] & (kOccOne - 1);
      const uint64_t w = P.upper ? (uint64_t)(n - 1 - i) : (uint64_t)n;
      s_t[k] = (uint32_t)t;
      uint32_t rec = 0;
      if (t) {
        const uint64_t b = t < w ? t : w;
        const bool hfit = b <= hash_cap && t <= unit_terms;
        if (w <= dense_cap && ((8 * t >= w && w >= kMinDenseWidth) || !hfit)) {
          rec = 1;
        } else if (!hfit) {
          rec = 2 | (uint32_t)((w + dense_cap - 1) / dense_cap) << 3;
          atomicOr(&S->has_win, 1u);
        } else {
          const uint64_t xb = (b * kPlanS + hash_cap - 1) / hash_cap;
          const uint64_t xt = (uint64_t)((double)t * inv_ut) + 1;
          const uint64_t x = xb > xt ? xb : xt;
          rec = x > kPlanS / 4 ? 3u : (4u | (uint32_t)x << 3);
        }
      }
      s_rec[k] = rec;
    }
  }
  __syncthreads();
  const uint32_t lo = min(cn, tid * kPlanRowsPerThread), hi = min(cn, lo + kPlanRowsPerThread);
  unsigned long long pw = 0;
  for (uint32_t k = lo; k < hi; ++k) {
    const uint32_t r = s_rec[k];
    pw += ((r & 7) == 4 ? (r >> 3) : 0) + y;
  }
  unsigned long long chunk_w;
  const unsigned long long pw_ex = plan_block_scan<unsigned long long>(pw, s_u64, 0ull, add, chunk_w);
  if (tid == 0) S->cw[cb] = chunk_w;
  grid.sync();
  unsigned long long all_w;
  const unsigned long long c_p = before_sum(S->cw, all_w);
  const unsigned long long pbase = c_p + pw_ex;
  long long lastb = -1;
  {
    unsigned long long p = pbase;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t r = s_rec[k];
      if ((r & 7) == 4) lastb = bucket(p);
      p += ((r & 7) == 4 ? (r >> 3) : 0) + y;
    }
  }
  long long carryb = plan_block_scan<long long>(lastb, s_i64, -1ll, mx, totl);
  if (tid == 0) S->lastb[cb] = totl;
  grid.sync();
  const long long c_bucket = before_max(S->lastb);
  carryb = carryb > c_bucket ? carryb : c_bucket;
  unsigned long long cnt = 0;
  {
    unsigned long long p = pbase;
    long long lb = carryb;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t r = s_rec[k], c = r & 7;
      if (c == 1 || c == 3) cnt += 1;
      else if (c == 2) cnt += r >> 3;
      else if (c == 4) {
        const long long bk = bucket(p);
        if (bk != lb) cnt += 1;
        lb = bk;
      }
      p += (c == 4 ? (r >> 3) : 0) + y;
    }
  }
  unsigned long long chunk_tiles;
  const unsigned long long t_ex = plan_block_scan<unsigned long long>(cnt, s_u64, 0ull, add, chunk_tiles);
  if (tid == 0) S->ct[cb] = chunk_tiles;
  grid.sync();
  unsigned long long all_tiles;
  const unsigned long long c_tiles = before_sum(S->ct, all_tiles);
  if (all_tiles > P.tile_cap) {
    if (cb == 0 && tid == 0) P.out->overflow = 1;
    return;
  }
  const unsigned long long tbase = c_tiles + t_ex;
  long long last_lt = -1, last_row0 = -1;
  {
    unsigned long long p = pbase;
    long long lb = carryb;
    uint32_t id = (uint32_t)tbase;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t r = s_rec[k], c = r & 7, i = base + k;
      if (c == 1 || c == 3) {
        const uint64_t t = s_t[k];
        Tile tl{};
        tl.row0 = i;
        tl.row1 = i + 1;
        tl.c1 = n;
        tl.terms = t;
        if (c == 1) {
          tl.c0 = P.upper ? i + 1 : 0;
          tl.mode = P.filter ? 0 : 2;
          tl.width = P.upper ? n - 1 - i : n;
          const uint64_t occ = P.stats[i] >> kOccShift;
          tl.n_units = units_of(t, (P.safe && tl.mode == 0 && t > occ) ? t : occ);
        } else {
          tl.mode = 1;
          tl.n_units = 1;
        }
        P.tiles[id] = tl;
        P.item_info[i] = make_uint2(id | (tl.mode == 2 ? kEntFlag : 0u),
                                    stream_base(tl, i, n, P.col_bits, P.upper != 0));
        ++id;
      } else if (c == 2) {
        const uint64_t t = s_t[k];
        const uint32_t col_lo = P.upper ? i + 1 : 0;
        const uint32_t nwin = r >> 3;
        for (uint32_t q = 0; q < nwin; ++q) {
          Tile tl{};
          tl.row0 = i;
          tl.row1 = i + 1;
          tl.c0 = col_lo + q * (uint32_t)dense_cap;
          tl.c1 = (uint32_t)min((uint64_t)n, (uint64_t)tl.c0 + dense_cap);
          tl.mode = 0;
          tl.nwin = q == 0 ? nwin : 0;
          tl.width = tl.c1 - tl.c0;
          tl.terms = t / nwin + 1;
          const uint64_t occ = P.stats[i] >> kOccShift;
          tl.n_units = units_of(tl.terms, (P.safe && tl.terms > occ) ? tl.terms : occ);
          P.tiles[id + q] = tl;
        }
        P.item_info[i] = make_uint2(id | kWinFlag, 0u);
        id += nwin;
      } else if (c == 4) {
        const long long bk = bucket(p);
        if (bk != lb) {
          Tile tl{};
          tl.row0 = i;
          tl.row1 = i + 1;
          tl.c1 = n;
          tl.mode = 1;
          tl.n_units = 1;
          P.tiles[id] = tl;
          last_lt = id;
          last_row0 = i;
          ++id;
        }
        lb = bk;
      } else {
        P.item_info[i] = make_uint2(kNone, 0u);
      }
      p += (c == 4 ? (r >> 3) : 0) + y;
    }
  }
  long long carry_lt = plan_block_scan<long long>(last_lt, s_i64, -1ll, mx, totl);
  if (tid == 0) S->llt[cb] = totl;
  long long carry_row0 = plan_block_scan<long long>(last_row0, s_i64, -1ll, mx, totl);
  if (tid == 0) S->lrow[cb] = totl;
  grid.sync();
  {
    const long long c_lt = before_max(S->llt), c_lrow0 = before_max(S->lrow);
    carry_lt = carry_lt > c_lt ? carry_lt : c_lt;
    carry_row0 = carry_row0 > c_lrow0 ? carry_row0 : c_lrow0;
  }
  {
    unsigned long long p = pbase;
    long long lb = carryb, cur = carry_lt, row0 = carry_row0;
    uint32_t id = (uint32_t)tbase;
    long long acc_tile = -1;
    unsigned long long acc_terms = 0;
    uint32_t acc_row1 = 0;
    auto flush = [&]() {
      if (acc_tile >= 0) {
        Tile* tl = P.tiles + acc_tile;
        atomicMax(&tl->row1, acc_row1);
        atomicAdd(reinterpret_cast<unsigned long long*>(&tl->terms), acc_terms);
      }
    };
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t r = s_rec[k], c = r & 7, i = base + k;
      if (c == 1 || c == 3) ++id;
      else if (c == 2) id += r >> 3;
      else if (c == 4) {
        const long long bk = bucket(p);
        if (bk != lb) {
          cur = id++;
          row0 = i;
        }
        lb = bk;
        if (cur != acc_tile) {
          flush();
          acc_tile = cur;
          acc_terms = 0;
        }
        acc_terms += s_t[k];
        acc_row1 = i + 1;
        P.item_info[i] = make_uint2((uint32_t)cur, (i - (uint32_t)row0) << P.col_bits);
      }
      p += (c == 4 ? (r >> 3) : 0) + y;
    }
    flush();
  }
  grid.sync();
  const uint32_t nt = (uint32_t)all_tiles;
  const uint32_t ta = (uint32_t)((uint64_t)nt * cb / nb), tb = (uint32_t)((uint64_t)nt * (cb + 1) / nb);
  const uint32_t tseg = (tb - ta + kPlanThreads - 1) / kPlanThreads;
  const uint32_t tlo = min(tb, ta + tid * tseg), thi = min(tb, tlo + tseg);
  if (P.shard_world > 1) {
    auto is_window = [&](const Tile& tl) {
      return tl.mode == 0 && tl.row1 - tl.row0 == 1 && tl.width < (P.upper ? n - 1 - tl.row0 : n);
    };
    auto words_of = [&](const Tile& tl) -> unsigned long long {
      if (is_window(tl)) return 2 + (tl.nwin ? (P.stats[tl.row0] & (kOccOne - 1)) : 0ull);
      return 2 + (tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms);
    };
    auto cost = [&](const Tile& tl) -> unsigned long long {
      if (is_window(tl) && tl.n_units == 1 && tl.terms <= kSparseWindowWords) {
        Tile h = tl;
        h.mode = 1;
        return tile_cost(h, stream_hash_slots(tl.terms));
      }
      return tile_cost(tl, stream_hash_slots(tl.terms < hash_cap ? tl.terms : hash_cap));
    };
    bool done = false;
    for (int pass = 0; pass < 3 && !done; ++pass) {
      auto metric = [&](const Tile& tl) -> unsigned long long {
        if (pass == 0) return cost(tl);
        return words_of(tl) + (pass == 1 ? 2048ull * (tl.n_units ? tl.n_units : 1) : 0ull);
      };
      unsigned long long tsum = 0, ctot;
      for (uint32_t t = tlo; t < thi; ++t) tsum += metric(P.tiles[t]);
      const unsigned long long pre_l = plan_block_scan<unsigned long long>(tsum, s_u64, 0ull, add, ctot);
      if (tid == 0) S->ssum[pass][cb] = ctot;
      grid.sync();
      unsigned long long all;
      unsigned long long pre = before_sum(S->ssum[pass], all) + pre_l;
      for (uint32_t t = tlo; t < thi; ++t) {
        const unsigned long long c = metric(P.tiles[t]);
        const unsigned long long ow = all ? (pre + c / 2) * P.shard_world / all : 0;
        P.tiles[t].slab_base = ow < P.shard_world - 1 ? ow : P.shard_world - 1;
        pre += c;
      }
      grid.sync();
      {
        uint32_t cur = kNone;
        unsigned long long acc = 0;
        for (uint32_t t = tlo; t < thi; ++t) {
          const Tile& tl = P.tiles[t];
          uint32_t ow;
          if (is_window(tl) && tl.nwin == 0 && t > tlo) {
            ow = cur;
          } else {
            uint32_t f = t;
            if (is_window(tl))
              while (P.tiles[f].nwin == 0 && f > 0) --f;
            ow = (uint32_t)P.tiles[f].slab_base;
          }
          if (ow != cur) {
            if (cur != kNone) atomicAdd(&S->sow[pass][cur < kMaxShardCheck ? cur : kMaxShardCheck - 1], acc);
            cur = ow;
            acc = 0;
          }
          acc += words_of(tl);
        }
        if (cur != kNone) atomicAdd(&S->sow[pass][cur < kMaxShardCheck ? cur : kMaxShardCheck - 1], acc);
      }
      grid.sync();
      unsigned long long mxw = 0;
      for (uint32_t k = tid; k < kMaxShardCheck; k += kPlanThreads)
        mxw = S->sow[pass][k] > mxw ? S->sow[pass][k] : mxw;
      plan_block_scan<long long>((long long)mxw, s_i64, 0ll, mx, totl);
      if (totl + 2 < (1ll << 32)) {
        done = true;
      } else if (pass == 2) {
        if (cb == 0 && tid == 0) P.out->overflow = 2;
        return;
      }
    }
    {
      uint32_t cur = kNone;
      for (uint32_t t = tlo; t < thi; ++t) {
        Tile& tl = P.tiles[t];
        if (!(is_window(tl) && tl.nwin == 0 && t > tlo)) {
          uint32_t f = t;
          if (is_window(tl))
            while (P.tiles[f].nwin == 0 && f > 0) --f;
          cur = (uint32_t)P.tiles[f].slab_base;
        }
        if (cur != P.shard_rank) tl.n_units = 0;
      }
    }
    grid.sync();
    for (uint32_t t = tlo; t < thi; ++t) P.tiles[t].slab_base = 0;
    for (uint32_t i = cb * kPlanThreads + tid; i < n; i += nb * kPlanThreads) {
      const uint2 tv = P.item_info[i];
      if (tv.x != kNone && P.tiles[tv.x & kTileMask].n_units == 0) P.item_info[i] = make_uint2(kNone, 0u);
    }
    grid.sync();
  }
  // 4. units, slabs, split list, reduce chunks, output capacity
  for (uint32_t t = tlo; t < thi; ++t) {
    Tile& tl = P.tiles[t];
    if (tl.mode == 1) tl.width = stream_hash_slots(tl.terms < hash_cap ? tl.terms : hash_cap);
  }
  auto nu_of = [&](uint32_t t) { return P.tiles[t].n_units; };
  auto wd_of = [&](uint32_t t) { return P.tiles[t].mode != 1 ? P.tiles[t].width : 0xFFFFFFFFu; };
  unsigned long long a[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // slab, split, single, rc, cap, units, words, terms
  for (uint32_t t = tlo; t < thi; ++t) {
    const uint32_t nu_t = nu_of(t), wd = wd_of(t);
    if (nu_t == 0) continue;
    {
      const Tile& tl = P.tiles[t];
      const bool win = tl.mode == 0 && tl.row1 - tl.row0 == 1 &&
                       tl.width < (P.upper ? n - 1 - tl.row0 : n);
      if (win) a[6] += tl.nwin ? (P.stats[tl.row0] & (kOccOne - 1)) : 0ull;
      else a[6] += tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms;
      a[6] += 2;
      a[7] += tl.terms;
    }
    a[4] += tile_out_cap(P.tiles[t], kStreamHashCap, n, P.upper != 0);
    a[5] += nu_t;
    if (nu_t > 1) {
      a[0] += nu_t;
      a[1] += 1;
      a[3] += ((wd < kSHalf ? wd : kSHalf) + kReduceSlots - 1) / kReduceSlots;
    } else {
      a[2] += 1;
    }
  }
  unsigned long long b_l[8], c_tot[8];
  for (int q = 0; q < 8; ++q) {
    b_l[q] = plan_block_scan<unsigned long long>(a[q], s_u64, 0ull, add, c_tot[q]);
    if (tid == 0) S->u8[cb][q] = c_tot[q];
  }
  grid.sync();
  unsigned long long b_c[8], tot[8];
  if (tid < 8) {
    unsigned long long s = 0, t = 0;
    for (uint32_t k = 0; k < nb; ++k) {
      if (k == cb) s = t;
      t += S->u8[k][tid];
    }
    s_u64[tid] = s;
    s_u64[8 + tid] = t;
  }
  __syncthreads();
  for (int q = 0; q < 8; ++q) {
    b_c[q] = s_u64[q];
    tot[q] = s_u64[8 + q];
  }
  __syncthreads();
  const unsigned long long n_slabs = tot[0], n_split = tot[1], n_rc = tot[3], cap = tot[4], nu = tot[5];
  const unsigned long long own_words = tot[6], own_terms = tot[7];
  if (nu > P.unit_cap || n_rc > P.rc_cap || own_words + 2 >= (1ull << 32)) {
    if (cb == 0 && tid == 0) P.out->overflow = 1;
    return;
  }
  constexpr int kFracBins = 64;
  {
    uint64_t sb = b_c[0] + b_l[0], sp = b_c[1] + b_l[1], rc = b_c[3] + b_l[3];
    for (uint32_t t = tlo; t < thi; ++t) {
      const uint32_t nu_t = nu_of(t), width = wd_of(t);
      if (nu_t > 1) {
        P.tiles[t].slab_base = sb;
        sb += nu_t;
        P.split[sp++] = t;
        const uint32_t dw = width < kSHalf ? width : kSHalf;
        for (uint32_t c0 = 0; c0 < dw; c0 += kReduceSlots) P.reduce_chunks[rc++] = make_uint2(t, c0);
      }
    }
  }
  for (uint32_t t = tlo; t < thi; ++t) {
    const uint32_t nu_t = nu_of(t);
    if (nu_t > 1)
      for (uint32_t u = 0; u < nu_t; ++u) atomicAdd(&S->bins[(uint64_t)(2 * u + 1) * kFracBins / (2 * nu_t)], 1u);
  }
  grid.sync();
  if (cb == 0 && tid == 0) {
    uint32_t run = 0;
    for (int k = 0; k < kFracBins; ++k) {
      S->cur[k] = run;
      run += S->bins[k];
    }
    S->cur[kFracBins] = run;
  }
  grid.sync();
  for (uint32_t t = tlo; t < thi; ++t) {
    const uint32_t nu_t = nu_of(t);
    if (nu_t > 1) {
      for (uint32_t u = 0; u < nu_t; ++u) {
        const uint32_t pos = atomicAdd(&S->cur[(uint64_t)(2 * u + 1) * kFracBins / (2 * nu_t)], 1u);
        P.units[pos] = Unit{t, u};
      }
    }
  }
  {
    uint64_t pos = S->cur[kFracBins] + b_c[2] + b_l[2];  // unchanged by the placements above: bins < 64
    for (uint32_t t = tlo; t < thi; ++t)
      if (nu_of(t) == 1) P.units[pos++] = Unit{t, 0};
  }
  const bool known = (!P.filter || P.own) && !S->has_win;
  if (known)
    for (uint32_t t = tlo; t < thi; ++t) {
      const Tile& tl = P.tiles[t];
      P.tile_words[t] = tl.n_units == 0 ? 0ull : (tl.mode == 2 ? 2 * (P.stats[tl.row0] >> kOccShift) : tl.terms);
    }
  if (cb == 0 && tid == 0) {
    P.out->words_known = known;
    P.out->pad0 = 0;
    P.out->pad1 = 0;
    P.out->max_entries = cap;
    P.out->own_words = own_words + 2;
    P.out->own_terms = own_terms;
    P.out->n_slabs = n_slabs;
    P.out->n_tiles = nt;
    P.out->n_units = (uint32_t)nu;
    P.out->n_split = (uint32_t)n_split;
    P.out->n_reduce_chunks = (uint32_t)n_rc;
  }
}

}  // namespace

// =============================================================== host side

struct crop_pairs {
  const int64_t* offsets;
  const uint32_t* items;
  int64_t n_tx;
  int64_t nnz;
  uint32_t n_items;
  int upper;
  bool filter;
  crop_interval iv;
  uint32_t col_bits;
  uint64_t total_terms;
  uint64_t max_entries;
  uint64_t entry_cap;
  cudaStream_t stream;
  std::vector<Tile> tiles;
  std::vector<Unit> units;
  std::vector<uint32_t> split;
  uint64_t n_slabs;
  // device (stream-ordered pool)
  unsigned long long* d_terms = nullptr;
  unsigned int* d_maxlen = nullptr;
  uint32_t* d_item_tile = nullptr;
  uint2* d_item_info = nullptr;  // stream mode: {tile | kWinFlag, word base}
  Tile* d_tiles = nullptr;
  Unit* d_units = nullptr;
  uint32_t* d_split = nullptr;
  uint32_t* d_tile_entries = nullptr;
  unsigned long long* d_tile_ebase = nullptr;
  unsigned long long* d_tile_cursor = nullptr;
  unsigned long long* d_tile_end = nullptr;
  unsigned long long* d_total_entries = nullptr;
  int route_chunk_tx = 256;
  std::vector<unsigned long long> h_tile_base, h_tile_end;
  uint2* d_entries = nullptr;
  uint32_t* d_slabs = nullptr;
  unsigned int* d_unit_counter = nullptr;
  uint32_t* d_overflow = nullptr;
  unsigned int* d_tile_done = nullptr;
  uint2* d_reduce_chunks = nullptr;  // stream mode: (split tile, first slot)
  uint32_t n_reduce_chunks = 0;
  uint32_t nt = 0, nu = 0;  // tiles, units (either planner)
  bool words_known = false;  // d_tile_words filled by the device planner
  uint32_t maxlen = 0;       // longest transaction (device planner path)
  uint16_t* d_items16 = nullptr;  // 16-bit item copy (ids < 2^16), made on the side stream
  uint32_t* d_items_cls = nullptr;  // filtered jobs: item | h_col << 16 (side stream)
  uint32_t flags = 0;        // CROP_PAIRS_* (crop_pairs_create_ex)
  bool own = false;          // filtered job on the own-bucket layout (Lemma 1)
  uint32_t* d_hs = nullptr;  // own: (h_col, id)-sorted keys per transaction
  uint32_t* d_own_bounds = nullptr;  // own: first transaction of each position band
  uint32_t* d_pos_rec = nullptr;     // own: per-position partner records (inside d_hs)
  uint32_t own_chunks = 0;
  uint32_t idbits = 0;
  cudaEvent_t ev_items16 = nullptr;
  uint64_t out_cap = 0;      // caller's output capacity (0: max_entries)
  bool packed_filter = false;  // bucket filter applied on packed items (see k_items_cls)
  uint32_t shard_rank = 0, shard_world = 1;  // tile sharding across ranks
  bool written = false;  // stream mode: the words were written by create (run counts only)
  int64_t nnz_hint = 0;  // offsets[n_tx], read at creation
  uint64_t own_terms = 0;  // this shard's terms (device planner; 0 = unknown)
  // fused top-k buffers (caller-owned, stream mode): see crop_pairs_set_topk
  uint32_t* topk_hist = nullptr;
  unsigned long long* hi_list = nullptr;
  unsigned long long* hi_n = nullptr;
  void* d_block = nullptr;  // one allocation carved into the small per-job arrays
  // stream mode (short rows): pair words per tile instead of entries
  bool stream_mode = false;
  uint32_t* d_words = nullptr;
  unsigned long long* d_tile_words = nullptr;
  // optional per-phase timing (CUDA events on the job's stream)
  bool timing = false;
  cudaEvent_t ev[6] = {};
};

// Pinned host staging shared by all jobs: the pass-A statistics come back
// through it and the plan goes up through it in one copy. The event marks
// the last upload; the next job waits on it before reusing the buffer.
struct PinnedArena {
  std::mutex mu;
  unsigned char* p = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  cudaError_t reserve(size_t n) {
    if (done) {
      cudaError_t e = cudaEventSynchronize(done);
      if (e != cudaSuccess) return e;
    } else {
      cudaError_t e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    if (n <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n + n / 2, 1 << 20);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
};
static PinnedArena g_pinned;

static inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Stream mode, phases route + write: word totals (when unknown), tile bases,
// then the scatter of every own pair into its tile's stream. Launched by
// crop_pairs_create right after planning (so the caller's host work between
// create and run overlaps the scatter), or by run after a re-run request.
static int stream_write(crop_pairs* J, cudaStream_t st, bool rec) {
  const uint32_t nt = J->nt;
  if (nt == 0 || J->n_tx == 0) return CROP_OK;
  const bool up = J->upper != 0;
  auto mark = [&](int k) {
    if (rec) cudaEventRecord(J->ev[k], st);
  };
  mark(0);
  {
    StreamRouteArgs R{};
    R.offsets = J->offsets;
    R.items = J->items;
    R.n_tx = J->n_tx;
    R.item_info = J->d_item_info;
    R.tiles = J->d_tiles;
    R.n_tiles = nt;
    R.n_items = J->n_items;
    R.col_bits = J->col_bits;
    R.filter = J->filter;
    R.kappa = J->iv.kappa;
    R.start = J->iv.start;
    R.stop = J->iv.stop;
    R.h_row = J->iv.h_row;
    R.h_col = J->iv.h_col;
    R.tile_words = J->d_tile_words;
    R.tile_cursor = J->d_tile_cursor;
    R.tile_base = J->d_tile_ebase;
    R.words = J->d_words;
    // about 12 chunks per CTA so the last wave's imbalance stays small
    R.chunk_tx = (int)std::max<int64_t>(256, std::min<int64_t>(kChunkTx, J->n_tx / (kNumSMs * 12)));
    const int64_t chunks = (J->n_tx + R.chunk_tx - 1) / R.chunk_tx;
    const int grid = (int)std::min<int64_t>(kNumSMs, chunks);
    R.chunk_counts = nullptr;
    uint32_t* d_chunk_counts = nullptr;
    if (!J->words_known) {
      CROP_CUDA(cudaMemsetAsync(J->d_tile_words, 0, nt * 8, st));
      // per-chunk counts for k_stream_write (same chunks, same shared tiles)
      // when they stay under 512 MB (c3 chunk: 2,035 x 24,576 x 4 B = 200 MB)
      const size_t cc_bytes = (size_t)chunks * std::min(nt, kTileSmem) * 4;
      const bool writes_by_chunk = !(J->own && J->d_own_bounds);
      if (writes_by_chunk && cc_bytes <= (512ull << 20) && !getenv("CROP_NO_CHUNK_COUNTS")) {
        CROP_CUDA(cudaMallocAsync(&d_chunk_counts, std::max<size_t>(cc_bytes, 4), st));
        R.chunk_counts = d_chunk_counts;
      }
      auto kern = up ? k_stream_count<true> : k_stream_count<false>;
      const size_t smem = kOffBytes + (size_t)std::min(nt, kTileSmem) * 4;
      CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(kOffBytes + kTileSmem * 4)));
      kern<<<grid, kPassThreads, smem, st>>>(R);
      CROP_LAUNCH_CHECK();
    }
    k_scan_u64<<<1, 1024, 0, st>>>(J->d_tile_words, nt, J->d_tile_ebase, J->d_tile_cursor);
    CROP_LAUNCH_CHECK();
    mark(1);
    R.packed_filter = J->packed_filter ? 1 : 0;
    if (J->own && J->words_known && J->d_own_bounds) {
      // own-bucket scatter: only own partners, read from the staged windows
      // (the position bands of pass A)
      const uint32_t n_chunks = J->own_chunks;
      const uint32_t* bounds = J->d_own_bounds;
      const bool single = J->iv.stop - J->iv.start == 1;
      const size_t fixed = single ? scatter_own_fixed<true>() : scatter_own_fixed<false>();
      const size_t budget = 227 * 1024 - fixed;
      R.scat_ns = (uint32_t)std::min<size_t>(std::min<size_t>(nt, kTileSmem), budget / 6 - 2);
      const size_t smem = fixed + (((size_t)R.scat_ns + 1) & ~(size_t)1) * 6;
      OwnArgs O{};
      O.hs = J->d_hs;
      O.h_row = J->iv.h_row;
      O.kappa = J->iv.kappa;
      O.start = J->iv.start;
      O.len = J->iv.stop - J->iv.start;
      O.idbits = J->idbits;
      O.pos_rec = J->d_pos_rec;
      auto kern = single ? (up ? k_stream_scatter_own<true, true> : k_stream_scatter_own<false, true>)
                         : (up ? k_stream_scatter_own<true, false> : k_stream_scatter_own<false, false>);
      CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024)));
      kern<<<(int)std::min<uint32_t>(kNumSMs, n_chunks), kPassThreads, smem, st>>>(R, O, bounds, n_chunks);
      CROP_LAUNCH_CHECK();
      crop_count_launches(1);
    } else if (J->words_known && J->maxlen <= kScatPark / 2) {
      // single-walk scatter over position bands
      const bool two = J->maxlen <= kScatPark2 / 2 && !getenv("CROP_SCATTER_ONE_CTA");
      const uint32_t band = (two ? kScatPark2 : kScatPark) - J->maxlen + 1;
      const uint32_t n_chunks = (uint32_t)((uint64_t)J->nnz / band + 1);
      uint32_t* bounds = nullptr;
      CROP_CUDA(cudaMallocAsync(&bounds, (size_t)(n_chunks + 1) * 4, st));
      k_chunk_bounds<<<(int)std::min<int64_t>(kNumSMs * 8, (J->n_tx + 256) / 256), 256, 0, st>>>(
          J->offsets, J->n_tx, n_chunks, band, bounds);
      CROP_LAUNCH_CHECK();
      if (two) {
        const size_t fixed = (size_t)(kScatMaxTx2 + 1) * 8 + (size_t)kScatPark2 * 12 + 16 + 512 / 32 * 128 * 4;
        const size_t budget = 112 * 1024 - fixed;
        R.scat_ns = (uint32_t)std::min<size_t>(std::min<size_t>(nt, kTileSmem), budget / 6 - 2);
        const size_t smem = fixed + (((size_t)R.scat_ns + 1) & ~(size_t)1) * 6;
        auto kern = J->packed_filter
                        ? (up ? k_stream_scatter<true, true, 512, kScatPark2, kScatMaxTx2>
                              : k_stream_scatter<false, true, 512, kScatPark2, kScatMaxTx2>)
                        : (up ? k_stream_scatter<true, false, 512, kScatPark2, kScatMaxTx2>
                              : k_stream_scatter<false, false, 512, kScatPark2, kScatMaxTx2>);
        CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(112 * 1024)));
        kern<<<(int)std::min<uint32_t>(2 * kNumSMs, n_chunks), 512, smem, st>>>(R, bounds, n_chunks);
      } else {
        const size_t fixed = (size_t)(kScatMaxTx + 1) * 8 + (size_t)kScatPark * 12 + 16 + kPassThreads / 32 * 128 * 4;
        const size_t budget = 227 * 1024 - fixed;
        R.scat_ns = (uint32_t)std::min<size_t>(std::min<size_t>(nt, kTileSmem), budget / 6 - 2);
        const size_t smem = fixed + (((size_t)R.scat_ns + 1) & ~(size_t)1) * 6;
        auto kern = J->packed_filter ? (up ? k_stream_scatter<true, true> : k_stream_scatter<false, true>)
                                     : (up ? k_stream_scatter<true, false> : k_stream_scatter<false, false>);
        CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024)));
        kern<<<(int)std::min<uint32_t>(kNumSMs, n_chunks), kPassThreads, smem, st>>>(R, bounds, n_chunks);
      }
      CROP_LAUNCH_CHECK();
      cudaFreeAsync(bounds, st);
      crop_count_launches(1);
    } else {
      auto kern = up ? k_stream_write<true> : k_stream_write<false>;
      const size_t ns2 = (std::min(nt, kTileSmem) + 1) & ~1u;
      const size_t smem = kOffBytes + ns2 * 6 + 16;
      CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(kOffBytes + (size_t)kTileSmem * 6 + 16)));
      kern<<<grid, kPassThreads, smem, st>>>(R);
      CROP_LAUNCH_CHECK();
    }
    if (d_chunk_counts) cudaFreeAsync(d_chunk_counts, st);
    mark(2);
  }
  return CROP_OK;
}

// Launch the stream write from create (events recorded for phase_ms).
static int early_write(crop_pairs* J, cudaStream_t st) {
  if (getenv("CROP_LATE_WRITE")) return CROP_OK;
  if (!J->ev[0])
    for (cudaEvent_t& e : J->ev) CROP_CUDA(cudaEventCreate(&e));
  if (int rc = stream_write(J, st, true)) return rc;
  J->written = true;
  return CROP_OK;
}

static void free_job(crop_pairs* j) {
  for (cudaEvent_t& e : j->ev)
    if (e) cudaEventDestroy(e);
  if (j->ev_items16) cudaEventDestroy(j->ev_items16);
  void* ptrs[] = {j->d_terms, j->d_block, j->d_entries, j->d_slabs, j->d_words, j->d_items16,
                  j->d_items_cls, j->d_hs, j->d_own_bounds};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, j->stream);
}

// Greedy tile planner over rows in id order (see file header). One pass
// over the rows, O(rows + tiles + units), no sorting: it sits between two
// GPU phases, so every microsecond here is GPU idle time.
static void plan_tiles(crop_pairs* J, const std::vector<unsigned long long>& terms,
                       const std::vector<unsigned long long>& occ,
                       std::vector<uint32_t>& item_tile) {
  const uint32_t n = J->n_items;
  const bool sm = J->stream_mode;
  // entry mode: u16 counters (65,536 per tile, <= 65,535 entries per unit);
  // stream mode: u32 counters (57,344 per tile)
  const uint64_t dense_cap = sm ? kStreamDenseCap : kDenseCap;
  const uint64_t hash_cap = sm ? kStreamHashCap : kHashCap;
  const uint64_t occ_cap = sm ? (uint64_t)kStreamUnitOcc : (uint64_t)kUnitEntries;
  const bool upper = J->upper != 0;
  const uint64_t T = J->total_terms;
  const uint64_t unit_terms = std::max<uint64_t>(1ull << 16, T / ((uint64_t)kNumSMs * 8));
  const uint32_t hash_rows_max = (J->col_bits >= 32) ? 1u : ((1u << (32 - J->col_bits)) - 1u);
  std::vector<Tile>& tiles = J->tiles;
  tiles.clear();
  tiles.reserve(1024);
  item_tile.assign(n, kNone);
  // units: by terms for balance, and <= kUnitEntries entries each (u16
  // counters); a tile's entries never exceed the sum of its rows' occ.
  auto units_for = [unit_terms, occ_cap](uint64_t tm, uint64_t oc) -> uint32_t {
    uint64_t u = (tm + unit_terms - 1) / unit_terms;
    const uint64_t ue = occ_cap == ~0ull ? 1 : (oc + occ_cap - 1) / occ_cap;
    if (ue > u) u = ue;
    return (uint32_t)(u < 1 ? 1 : (u > 65535 ? 65535 : u));
  };
  uint32_t row0 = 0;
  uint64_t sw = 0, sb = 0, st = 0, so = 0;
  bool open = false, dok = false, hok = false;
  auto close = [&](uint32_t row1) {
    Tile t{};
    t.row0 = row0;
    t.row1 = row1;
    t.c0 = 0;
    t.c1 = n;
    if (sm && row1 - row0 == 1) t.c0 = upper ? row0 + 1 : 0;  // stream: slot = j - c0
    const bool dense = dok && (!hok || st * 8 >= sw);
    t.mode = dense ? 0 : 1;
    // stream mode, unfiltered: a single-row dense tile is counted from one
    // entry per row occurrence (its suffix is read from the items)
    if (dense && sm && !J->filter && row1 - row0 == 1) t.mode = 2;
    t.width = dense ? (uint32_t)sw : (sm ? stream_hash_slots(sb < hash_cap ? sb : hash_cap) : 0);
    t.terms = st;
    t.n_units = dense ? units_for(st, so) : 1;
    const uint32_t id = (uint32_t)tiles.size();
    for (uint32_t i = row0; i < row1; ++i)
      if (terms[i]) item_tile[i] = id;
    tiles.push_back(t);
  };
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t tm = terms[i], oc = occ[i];
    const uint64_t w = upper ? (uint64_t)(n - 1 - i) : (uint64_t)n;
    const uint64_t b = tm < w ? tm : w;
    if (open) {
      const bool d2 = dok && sw + w <= dense_cap;
      const bool h2 = hok && sb + b <= hash_cap && st + tm <= unit_terms &&
                      so + oc <= occ_cap && (i - row0 + 1) <= hash_rows_max;
      if (d2 || h2) {
        sw += w;
        sb += b;
        st += tm;
        so += oc;
        dok = d2;
        hok = h2;
        continue;
      }
      close(i);
      open = false;
    }
    if (tm == 0) continue;
    const bool d2 = w <= dense_cap;
    const bool h2 = b <= hash_cap && tm <= unit_terms && oc <= occ_cap;
    if (d2 || h2) {
      open = true;
      row0 = i;
      sw = w;
      sb = b;
      st = tm;
      so = oc;
      dok = d2;
      hok = h2;
      continue;
    }
    // one row too wide for a dense tile and too heavy for a hash tile:
    // column windows of kDenseCap counters with consecutive tile ids.
    const uint32_t col_lo = upper ? i + 1 : 0;
    const uint32_t nwin = (uint32_t)((w + dense_cap - 1) / dense_cap);
    const uint32_t first = (uint32_t)tiles.size();
    for (uint32_t k = 0; k < nwin; ++k) {
      Tile t{};
      t.row0 = i;
      t.row1 = i + 1;
      t.c0 = col_lo + k * (uint32_t)dense_cap;
      t.c1 = (uint32_t)std::min<uint64_t>(n, (uint64_t)t.c0 + dense_cap);
      t.mode = 0;
      t.nwin = k == 0 ? nwin : 0;
      t.width = t.c1 - t.c0;
      t.terms = tm / nwin + 1;
      t.n_units = units_for(t.terms, oc);
      tiles.push_back(t);
    }
    item_tile[i] = first | kWinFlag;
  }
  if (open) close(n);

  // With more tiles than the router's shared counters, renumber heavy-first
  // so the heaviest tiles get shared counters (bucketed by log2(terms), a
  // split row's windows kept consecutive).
  if (tiles.size() > kTileSmem) {
    std::vector<std::vector<uint32_t>> bins(64);
    for (uint32_t t = 0; t < tiles.size();) {
      const uint32_t k = tiles[t].nwin ? tiles[t].nwin : 1;
      uint64_t gt = 0;
      for (uint32_t q = 0; q < k; ++q) gt += tiles[t + q].terms;
      const int lg = gt ? 63 - __builtin_clzll(gt) : 0;
      bins[63 - lg].push_back(t);
      t += k;
    }
    std::vector<uint32_t> new_id(tiles.size());
    std::vector<Tile> out;
    out.reserve(tiles.size());
    for (auto& bin : bins)
      for (uint32_t g0 : bin) {
        const uint32_t k = tiles[g0].nwin ? tiles[g0].nwin : 1;
        for (uint32_t q = 0; q < k; ++q) {
          new_id[g0 + q] = (uint32_t)out.size();
          out.push_back(tiles[g0 + q]);
        }
      }
    for (uint32_t i = 0; i < n; ++i)
      if (item_tile[i] != kNone)
        item_tile[i] = new_id[item_tile[i] & ~kWinFlag] | (item_tile[i] & kWinFlag);
    tiles.swap(out);
  }

  // Unit order: a unit covers the fraction [local, local+1)/n_units of its
  // tile's entry list, which the router wrote in (roughly) transaction order.
  // Running units in order of that fraction keeps the ~148 concurrently
  // active units on nearby transactions, so the rows they re-read stay in
  // L2 (64 fraction bins, no sort). Single-unit tiles follow.
  if (J->shard_world > 1) {
    // tile sharding (see k_plan_stream): this rank keeps the tiles of its
    // term share; a split row's windows follow the first window
    // Entry mode re-reads a suffix per entry: its cost is per term and per
    // entry (fit to the per-rank counting cycles of c5's 8 shards: ~0.23
    // cycles per term, ~26 per entry; entries <= the rows' occurrences).
    const uint32_t hroom = sm ? kStreamHashSlots : kHashSlots;
    std::vector<uint64_t> occ_pre;
    if (!sm) {
      occ_pre.assign(n + 1, 0);
      for (uint32_t i = 0; i < n; ++i) occ_pre[i + 1] = occ_pre[i] + occ[i];
    }
    auto cost_of = [&](const Tile& tl) -> uint64_t {
      if (sm) return tile_cost(tl, hroom);
      return 2 * tl.terms + 220 * (occ_pre[tl.row1] - occ_pre[tl.row0]);
    };
    uint64_t all = 0;
    for (auto& t : tiles) all += cost_of(t);
    // owner = floor(midpoint * world / all) (see k_plan_stream)
    uint64_t pre = 0;
    uint32_t owner = 0;
    for (uint32_t t = 0; t < tiles.size(); ++t) {
      const bool cont = tiles[t].mode == 0 && tiles[t].nwin == 0 && tiles[t].row1 - tiles[t].row0 == 1 &&
                        tiles[t].width < (upper ? n - 1 - tiles[t].row0 : n);
      const uint64_t c = cost_of(tiles[t]);
      if (!cont)
        owner = (uint32_t)std::min<uint64_t>(J->shard_world - 1,
                                             all ? (unsigned __int128)(pre + c / 2) * J->shard_world / all : 0);
      pre += c;
      if (owner != J->shard_rank) tiles[t].n_units = 0;
    }
    for (uint32_t i = 0; i < n; ++i)
      if (item_tile[i] != kNone && tiles[item_tile[i] & ~kWinFlag].n_units == 0) item_tile[i] = kNone;
  }
  J->units.clear();
  J->split.clear();
  J->n_slabs = 0;
  constexpr int kFracBins = 64;
  std::vector<uint32_t> bin_count(kFracBins + 1, 0);
  uint64_t n_units = 0;
  for (uint32_t t = 0; t < tiles.size(); ++t) {
    Tile& tt = tiles[t];
    n_units += tt.n_units;
    if (tt.n_units > 1) {
      tt.slab_base = J->n_slabs;
      J->n_slabs += tt.n_units;
      J->split.push_back(t);
      for (uint32_t u = 0; u < tt.n_units; ++u)
        ++bin_count[(uint64_t)(2 * u + 1) * kFracBins / (2 * tt.n_units)];
    } else if (tt.n_units == 1) {
      ++bin_count[kFracBins];
    }
  }
  std::vector<uint32_t> bin_pos(kFracBins + 1, 0);
  for (int k = 1; k <= kFracBins; ++k) bin_pos[k] = bin_pos[k - 1] + bin_count[k - 1];
  J->units.resize(n_units);
  for (uint32_t t = 0; t < tiles.size(); ++t) {
    const Tile& tt = tiles[t];
    if (tt.n_units > 1) {
      for (uint32_t u = 0; u < tt.n_units; ++u)
        J->units[bin_pos[(uint64_t)(2 * u + 1) * kFracBins / (2 * tt.n_units)]++] = Unit{t, u};
    } else if (tt.n_units == 1) {
      J->units[bin_pos[kFracBins]++] = Unit{t, 0};
    }
  }

  uint64_t cap = 0;
  for (auto& t : tiles)
    if (t.n_units) cap += tile_out_cap(t, (uint32_t)hash_cap, n, upper);
  J->max_entries = cap;
}

extern "C" int crop_pairs_create(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                                 uint32_t n_items, int upper_only, const crop_interval* interval,
                                 void* stream, crop_pairs** job) {
  return crop_pairs_create_ex(offsets, items, n_tx, n_items, upper_only, interval, 0, 1, 0, stream, job);
}

extern "C" int crop_pairs_create_sharded(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                                         uint32_t n_items, int upper_only, const crop_interval* interval,
                                         uint32_t shard_rank, uint32_t shard_world, void* stream,
                                         crop_pairs** job) {
  return crop_pairs_create_ex(offsets, items, n_tx, n_items, upper_only, interval, shard_rank, shard_world,
                              0, stream, job);
}

extern "C" int crop_pairs_create_ex(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                                    uint32_t n_items, int upper_only, const crop_interval* interval,
                                    uint32_t shard_rank, uint32_t shard_world, uint32_t flags,
                                    void* stream, crop_pairs** job) {
  *job = nullptr;
  if (shard_world < 1 || shard_rank >= shard_world) {
    crop_set_error(CROP_ECONFIG, "shard rank %u of %u", shard_rank, shard_world);
    return CROP_ECONFIG;
  }
  if (n_tx < 0 || n_items >= (1u << 31)) {
    crop_set_error(CROP_EINPUT, "need n_tx >= 0 and item ids < 2^31 (n_items=%u)", n_items);
    return CROP_EINPUT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (int rc = crop_pool_setup()) return rc;
  crop_pairs* J = new crop_pairs();
  J->flags = flags;
  J->shard_rank = shard_rank;
  J->shard_world = shard_world;
  J->offsets = offsets;
  J->items = items;
  J->n_tx = n_tx;
  J->n_items = n_items;
  J->upper = upper_only;
  J->filter = false;
  J->stream = st;
  if (interval) {
    J->iv = *interval;
    if (interval->kappa == 0 || interval->start > interval->stop || interval->stop > interval->kappa) {
      delete J;
      crop_set_error(CROP_ECONFIG, "invalid interval [%u, %u) for kappa=%u", interval->start,
                     interval->stop, interval->kappa);
      return CROP_ECONFIG;
    }
    J->filter = !(interval->start == 0 && interval->stop == interval->kappa);
  }
  uint32_t cb = 1;
  while (cb < 32 && (1ull << cb) < (uint64_t)std::max<uint32_t>(n_items, 2)) ++cb;
  J->col_bits = cb;
  int rc = CROP_OK;
#define JCUDA(call)                                                                         \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess) {                                                                \
      crop_set_error(CROP_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,                 \
                     cudaGetErrorString(_e));                                               \
      rc = CROP_ECUDA;                                                                      \
      goto fail;                                                                            \
    }                                                                                       \
  } while (0)
  {
    const uint32_t nn = std::max<uint32_t>(n_items, 1);
    // (the pinned staging and the nnz read below are shared across jobs)
    std::lock_guard<std::mutex> pin_lock(g_pinned.mu);
    // nnz (= offsets[n_tx]) sizes the device planner's capacities: read on a
    // side stream ordered after the inputs but not after pass A, so the host
    // waits for it while pass A runs
    static cudaStream_t s_nnz = nullptr;
    static cudaEvent_t e_in = nullptr;
    static int64_t* h_nnz_hint = nullptr;
    if (!s_nnz) {
      JCUDA(cudaStreamCreateWithFlags(&s_nnz, cudaStreamNonBlocking));
      JCUDA(cudaEventCreateWithFlags(&e_in, cudaEventDisableTiming));
      JCUDA(cudaMallocHost(&h_nnz_hint, 8));
    }
    if (n_tx > 0) JCUDA(cudaEventRecord(e_in, st));
    // CROP_DEBUG_TIMING: GPU time of pass A + planner and the idle gap
    // between the planner and the first write kernel (host planning latency)
    static cudaEvent_t dbg_ev[3] = {};
    const bool dbg_t = getenv("CROP_DEBUG_TIMING") != nullptr;
    if (dbg_t) {
      if (!dbg_ev[0])
        for (cudaEvent_t& e : dbg_ev) JCUDA(cudaEventCreate(&e));
      JCUDA(cudaEventRecord(dbg_ev[0], st));
    }
    JCUDA(cudaMallocAsync(&J->d_terms, nn * sizeof(unsigned long long) + 16, st));
    J->d_maxlen = reinterpret_cast<unsigned int*>(J->d_terms + nn);
    JCUDA(cudaMemsetAsync(J->d_terms, 0, nn * sizeof(unsigned long long) + 16, st));
    // own-bucket layout (Lemma 1) for filtered jobs: rows never need column
    // windows (n <= one dense table), and the (h_col, id) keys fit 32 bits
    {
      const bool no_own = (J->flags & CROP_PAIRS_NO_OWN) || getenv("CROP_NO_OWN") ||
                          getenv("CROP_FORCE_ENTRY_MODE") || getenv("CROP_HOST_PLANNER");
      uint32_t kb = 0;
      while (kb < 32 && (1ull << kb) < (uint64_t)J->iv.kappa) ++kb;
      J->own = J->filter && !no_own && n_tx > 0 && n_items > 0 && n_items <= kStreamDenseCap + 1 &&
               cb + kb <= 32 && J->iv.h_row && J->iv.h_col;
      J->idbits = cb;
    }
    OwnArgs OA{};
    if (J->own) {
      // nnz sizes the key copy; the longest transaction sizes the position bands
      int64_t nz = 0;
      unsigned int ml = 0;
      k_max_len<<<(int)std::min<int64_t>((n_tx + 255) / 256, kNumSMs * 8), 256, 0, st>>>(offsets, n_tx,
                                                                                        J->d_maxlen);
      JCUDA(cudaGetLastError());
      JCUDA(cudaMemcpyAsync(&nz, offsets + n_tx, 8, cudaMemcpyDeviceToHost, st));
      JCUDA(cudaMemcpyAsync(&ml, J->d_maxlen, 4, cudaMemcpyDeviceToHost, st));
      JCUDA(cudaStreamSynchronize(st));
      if ((uint64_t)nz >= (1ull << 32)) J->own = false;  // the 2^32 check below reports it
      if (J->own) {
        if (ml > kOwnStage / 2) {
          J->own = false;  // too long for the staged bands: the plain filter path counts it
        } else {
          JCUDA(cudaMallocAsync(&J->d_hs, (size_t)std::max<int64_t>(nz, 1) * 8, st));
          J->d_pos_rec = J->d_hs + std::max<int64_t>(nz, 1);
          const uint32_t band = kOwnStage - ml + 1;
          J->own_chunks = (uint32_t)((uint64_t)nz / band + 1);
          JCUDA(cudaMallocAsync(&J->d_own_bounds, (size_t)(J->own_chunks + 1) * 4, st));
          k_chunk_bounds<<<(int)std::min<int64_t>(kNumSMs * 8, (n_tx + 256) / 256), 256, 0, st>>>(
              offsets, n_tx, J->own_chunks, band, J->d_own_bounds);
          JCUDA(cudaGetLastError());
          OA.hs = J->d_hs;
          OA.h_row = J->iv.h_row;
          OA.kappa = J->iv.kappa;
          OA.start = J->iv.start;
          OA.len = J->iv.stop - J->iv.start;
          OA.idbits = J->idbits;
          OA.cbits = 0;
          while (OA.cbits < 32 && (1ull << OA.cbits) < (uint64_t)J->iv.kappa) ++OA.cbits;
          OA.pos_rec = J->d_pos_rec;
          auto kern = upper_only ? k_own_prep<true> : k_own_prep<false>;
          const uint32_t ns = std::min<uint32_t>(n_items, kOwnStatItems);
          const size_t fixed = (size_t)(kScatMaxTx + 1) * 8 + (size_t)kOwnStage * 8 +
                               (size_t)(kPassThreads / 32) * kOwnSortMax * 4;
          JCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(fixed + kOwnStatItems * 8)));
          kern<<<(int)std::min<uint32_t>(kNumSMs, J->own_chunks), kPassThreads, fixed + (size_t)ns * 8, st>>>(
              offsets, items, n_items, J->iv.h_col, J->d_own_bounds, J->own_chunks, J->d_terms, J->d_hs, OA);
          JCUDA(cudaGetLastError());
          crop_count_launches(3);
        }
      }
    }
    if (n_tx > 0 && n_items > 0 && !J->own) {
      auto kern = upper_only ? k_item_terms<true> : k_item_terms<false>;
      const uint32_t ns = std::min<uint32_t>(n_items, kStatSmemItems);
      const size_t smem = kOffBytes + ns * 8;  // two u32 arrays
      JCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kOffBytes + kStatSmemItems * 8)));
      // ~12 chunks per CTA: the last wave of chunks is a small share of the pass
      const int chunk_tx = (int)std::max<int64_t>(256, std::min<int64_t>(kChunkTx, n_tx / (kNumSMs * 12)));
      const int64_t chunks = (n_tx + chunk_tx - 1) / chunk_tx;
      const int grid = (int)std::min<int64_t>(kNumSMs, chunks);
      kern<<<grid, kPassThreads, smem, st>>>(offsets, items, n_tx, n_items, chunk_tx, J->d_terms, J->d_maxlen);
      JCUDA(cudaGetLastError());
      crop_count_launches(1);
    }
    if (n_tx > 0) {
      JCUDA(cudaStreamWaitEvent(s_nnz, e_in, 0));
      JCUDA(cudaMemcpyAsync(h_nnz_hint, offsets + n_tx, 8, cudaMemcpyDeviceToHost, s_nnz));
      JCUDA(cudaStreamSynchronize(s_nnz));
      J->nnz_hint = *h_nnz_hint;
    }
    // GPU planner first (stream mode); the host planner below handles entry
    // mode and the rare plans that exceed the device planner's bounds
    const int force = getenv("CROP_FORCE_ENTRY_MODE") ? 1 : (getenv("CROP_FORCE_STREAM_MODE") ? 2 : 0);
    if (n_tx > 0 && n_items > 0 && force != 1 && !getenv("CROP_HOST_PLANNER")) {
      // capacities: rows wider than one table are cut into up to `wmax`
      // column windows; units beyond one per tile come from terms (<= T /
      // unit_terms <= 1184) or from row occurrences (<= 65,535 per unit of
      // 16-bit counters, per window: <= wmax * nnz / 65,535)
      const uint64_t wmax = ((uint64_t)nn + kStreamDenseCap - 1) / kStreamDenseCap;
      const uint64_t occ_units = wmax * ((uint64_t)J->nnz_hint / kStreamUnitOcc + 1);
      const size_t tile_cap = (wmax > 1 ? 3 : 2) * (size_t)nn + 64;
      const size_t unit_cap = tile_cap + 1300 + occ_units;
      const size_t rc_cap = 29 * (1200 + occ_units);  // <= 29 chunks per split tile
      const size_t o_tiles = 0;
      const size_t o_units = align16(o_tiles + tile_cap * sizeof(Tile));
      const size_t o_split = align16(o_units + unit_cap * sizeof(Unit));
      const size_t o_ebase = align16(o_split + tile_cap * 4);
      const size_t o_item = align16(o_ebase + tile_cap * 8);
      const size_t o_rc = align16(o_item + (size_t)nn * sizeof(uint2));
      const size_t o_tentries = align16(o_rc + rc_cap * sizeof(uint2));
      const size_t o_cursor = align16(o_tentries + tile_cap * 4);
      const size_t o_twords = align16(o_cursor + tile_cap * 8);
      const size_t o_tdone = align16(o_twords + tile_cap * 8);
      const size_t o_misc = align16(o_tdone + tile_cap * 4);
      const size_t o_out = align16(o_misc + 32);
      const size_t blk_bytes = o_out + sizeof(PlanOut);
      JCUDA(cudaMallocAsync(&J->d_block, blk_bytes, st));
      unsigned char* db = reinterpret_cast<unsigned char*>(J->d_block);
      PlanArgs PA{};
      PA.stats = J->d_terms;
      PA.n = n_items;
      PA.col_bits = J->col_bits;
      PA.upper = upper_only;
      // filtered jobs whose ids and kappa fit 16 bits are planned like whole
      // jobs: the bucket test moves into the scatter (words) and the count
      // kernel (entries), on the packed items
      J->packed_filter = J->filter && !J->own && n_items <= 65536 && J->iv.kappa <= 65536 &&
                         !getenv("CROP_NO_PACKED_FILTER");
      PA.filter = J->filter && !J->packed_filter;
      // the own layout routes own words only: stream mode whatever the row length
      PA.force = J->own ? 2 : force;
      PA.own = J->own ? 1 : 0;
      PA.safe = (J->flags & CROP_PAIRS_SAFE_UNITS) ? 1 : 0;
      if (const char* ut = getenv("CROP_DEBUG_UNIT_TERMS")) PA.unit_terms = strtoull(ut, nullptr, 10);
      PA.tiles = reinterpret_cast<Tile*>(db + o_tiles);
      PA.tile_cap = (uint32_t)tile_cap;
      PA.units = reinterpret_cast<Unit*>(db + o_units);
      PA.unit_cap = (uint32_t)unit_cap;
      PA.split = reinterpret_cast<uint32_t*>(db + o_split);
      PA.reduce_chunks = reinterpret_cast<uint2*>(db + o_rc);
      PA.rc_cap = (uint32_t)rc_cap;
      PA.item_info = reinterpret_cast<uint2*>(db + o_item);
      PA.tile_words = reinterpret_cast<unsigned long long*>(db + o_twords);
      PA.shard_rank = J->shard_rank;
      PA.shard_world = J->shard_world;
      PA.out = reinterpret_cast<PlanOut*>(db + o_out);
      JCUDA(cudaMemsetAsync(db + o_misc, 0, 32, st));
      if (dbg_t) JCUDA(cudaEventRecord(dbg_ev[1], st));
      PlanScratch* d_ps = nullptr;
      if (n_items <= (uint64_t)kNumSMs * kPlanChunk && !getenv("CROP_PLAN_SINGLE_CTA")) {
        // one CTA per SM (cooperative launch: all resident, grid-wide syncs)
        JCUDA(cudaMallocAsync(&d_ps, sizeof(PlanScratch), st));
        JCUDA(cudaMemsetAsync(d_ps, 0, sizeof(PlanScratch), st));
        JCUDA(cudaFuncSetAttribute(k_plan_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kPlanChunk * 8)));
        void* args[] = {(void*)&PA, (void*)&d_ps};
        // as few CTAs as the row ranges allow: the grid syncs dominate a
        // small plan (c2: 16 CTAs of 3,125 rows; c3 chunks: 123 CTAs)
        const uint32_t pb = (uint32_t)std::max<uint64_t>(16, ((uint64_t)n_items + kPlanChunk - 1) / kPlanChunk);
        JCUDA(cudaLaunchCooperativeKernel((void*)k_plan_coop, dim3(std::min<uint32_t>(pb, kNumSMs)),
                                          dim3(kPlanThreads), args, kPlanChunk * 8, st));
        JCUDA(cudaFreeAsync(d_ps, st));
      } else {
        JCUDA(cudaFuncSetAttribute(k_plan_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kPlanChunk * 8)));
        k_plan_stream<<<1, kPlanThreads, kPlanChunk * 8, st>>>(PA);
      }
      JCUDA(cudaGetLastError());
      crop_count_launches(1);
      if (dbg_t) JCUDA(cudaEventRecord(dbg_ev[2], st));
      JCUDA(g_pinned.reserve(sizeof(PlanOut) + 64));
      PlanOut* ho = reinterpret_cast<PlanOut*>(g_pinned.p);
      unsigned int* h_ml = reinterpret_cast<unsigned int*>(g_pinned.p + sizeof(PlanOut));
      int64_t* h_nz = reinterpret_cast<int64_t*>(g_pinned.p + sizeof(PlanOut) + 16);
      JCUDA(cudaMemcpyAsync(ho, PA.out, sizeof(PlanOut), cudaMemcpyDeviceToHost, st));
      JCUDA(cudaMemcpyAsync(h_ml, J->d_maxlen, 4, cudaMemcpyDeviceToHost, st));
      JCUDA(cudaMemcpyAsync(h_nz, offsets + n_tx, 8, cudaMemcpyDeviceToHost, st));
      JCUDA(cudaStreamSynchronize(st));
      if (*h_ml > kMaxLen) {
        crop_set_error(CROP_EINPUT, "transaction of %u items exceeds the %u-item limit", *h_ml, kMaxLen);
        rc = CROP_EINPUT;
        goto fail;
      }
      if ((uint64_t)*h_nz >= (1ull << 32)) {
        crop_set_error(CROP_EINPUT, "%lld item occurrences exceed the 2^32 limit of one job; "
                       "split the stream", (long long)*h_nz);
        rc = CROP_EINPUT;
        goto fail;
      }
      if (getenv("CROP_DEBUG_TIMING"))
        fprintf(stderr, "[k_plan_stream] kcyc: totals %u classify %u scans+walks %.0f tiles %.0f light %.0f units %.0f\n",
                ho->pad0, ho->pad1, ho->dbg[0] / 1e3, ho->dbg[1] / 1e3, ho->dbg[2] / 1e3, ho->dbg[3] / 1e3);
      if (ho->overflow == 2) {
        // the stream words of this job (or of its largest tile shard) pass
        // the 32-bit word positions: the caller splits into finer shards
        crop_set_error(CROP_ERESOURCE, "%llu terms exceed one job's 2^32 stream words; "
                       "split into tile shards", (unsigned long long)ho->total_terms);
        rc = CROP_ERESOURCE;
        goto fail;
      }
      if (J->own && !(ho->stream_mode && !ho->overflow)) {
        crop_set_error(CROP_ERESOURCE, "%llu own terms exceed one job's 2^32 stream words; "
                       "split into tile shards", (unsigned long long)ho->total_terms);
        rc = CROP_ERESOURCE;
        goto fail;
      }
      if (ho->stream_mode && !ho->overflow) {
        J->nnz = *h_nz;
        J->stream_mode = true;
        J->total_terms = ho->total_terms;
        J->max_entries = ho->max_entries;
        J->n_slabs = ho->n_slabs;
        J->nt = ho->n_tiles;
        J->nu = ho->n_units;
        J->n_reduce_chunks = ho->n_reduce_chunks;
        J->words_known = ho->words_known != 0;
        J->maxlen = *h_ml;
        // 16-bit copy of the items for the count kernel's suffix gathers, on a
        // side stream: it overlaps the write phase (latency-bound, little DRAM)
        if (J->packed_filter && J->nnz > 0) {
          static cudaStream_t side2 = nullptr;
          if (!side2) JCUDA(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
          JCUDA(cudaEventCreateWithFlags(&J->ev_items16, cudaEventDisableTiming));
          JCUDA(cudaEventRecord(J->ev_items16, st));
          JCUDA(cudaStreamWaitEvent(side2, J->ev_items16, 0));
          JCUDA(cudaMallocAsync(&J->d_items_cls, (size_t)J->nnz * 4, side2));
          k_items_cls<<<kNumSMs * 4, 256, 0, side2>>>(items, J->nnz, J->iv.h_col, J->d_items_cls);
          JCUDA(cudaGetLastError());
          crop_count_launches(1);
          JCUDA(cudaEventRecord(J->ev_items16, side2));
        } else if (n_items <= 65536 && J->nnz > 0 && !getenv("CROP_NO_ITEMS16")) {
          static cudaStream_t side = nullptr;
          if (!side) JCUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
          JCUDA(cudaEventCreateWithFlags(&J->ev_items16, cudaEventDisableTiming));
          JCUDA(cudaEventRecord(J->ev_items16, st));  // inputs ready (stream order)
          JCUDA(cudaStreamWaitEvent(side, J->ev_items16, 0));
          JCUDA(cudaMallocAsync(&J->d_items16, (size_t)J->nnz * 2, side));
          k_items16<<<kNumSMs * 4, 256, 0, side>>>(items, J->nnz, J->d_items16);
          JCUDA(cudaGetLastError());
          crop_count_launches(1);
          JCUDA(cudaEventRecord(J->ev_items16, side));
        }
        J->entry_cap = 0;
        J->d_tiles = PA.tiles;
        J->d_units = PA.units;
        J->d_split = PA.split;
        J->d_tile_ebase = reinterpret_cast<unsigned long long*>(db + o_ebase);
        J->d_tile_end = nullptr;
        J->d_item_info = PA.item_info;
        J->d_reduce_chunks = PA.reduce_chunks;
        J->d_tile_entries = reinterpret_cast<uint32_t*>(db + o_tentries);
        J->d_tile_cursor = reinterpret_cast<unsigned long long*>(db + o_cursor);
        J->d_tile_words = reinterpret_cast<unsigned long long*>(db + o_twords);
        J->d_tile_done = reinterpret_cast<unsigned int*>(db + o_tdone);
        J->d_total_entries = reinterpret_cast<unsigned long long*>(db + o_misc);
        J->d_unit_counter = reinterpret_cast<unsigned int*>(db + o_misc + 8);
        J->d_overflow = reinterpret_cast<uint32_t*>(db + o_misc + 16);
        if (J->n_slabs)
          JCUDA(cudaMallocAsync(&J->d_slabs, J->n_slabs * (size_t)kSHalf * 4, st));
        JCUDA(cudaMallocAsync(&J->d_words, ho->own_words * 4, st));
        J->own_terms = ho->own_terms;
        rc = early_write(J, st);
        if (rc) goto fail;
        if (dbg_t && J->ev[0]) {
          float a = 0, b = 0, c = 0;
          JCUDA(cudaEventSynchronize(J->ev[0]));
          cudaEventElapsedTime(&a, dbg_ev[0], dbg_ev[1]);
          cudaEventElapsedTime(&b, dbg_ev[1], dbg_ev[2]);
          cudaEventElapsedTime(&c, dbg_ev[2], J->ev[0]);
          fprintf(stderr, "[create] pass A %.3f ms, planner %.3f ms, planner end -> write start %.3f ms\n",
                  a, b, c);
        }
        *job = J;
        return CROP_OK;
      }
      JCUDA(cudaFreeAsync(J->d_block, st));
      J->d_block = nullptr;
    }
    JCUDA(g_pinned.reserve(nn * 8 + 64));
    unsigned long long* stats = reinterpret_cast<unsigned long long*>(g_pinned.p);
    unsigned int* h_maxlen = reinterpret_cast<unsigned int*>(g_pinned.p + nn * 8);
    int64_t* h_nnz = reinterpret_cast<int64_t*>(g_pinned.p + nn * 8 + 16);
    *h_maxlen = 0;
    *h_nnz = 0;
    JCUDA(cudaMemcpyAsync(stats, J->d_terms, nn * 8, cudaMemcpyDeviceToHost, st));
    JCUDA(cudaMemcpyAsync(h_maxlen, J->d_maxlen, 4, cudaMemcpyDeviceToHost, st));
    if (n_tx > 0) JCUDA(cudaMemcpyAsync(h_nnz, offsets + n_tx, 8, cudaMemcpyDeviceToHost, st));
    auto t_sync0 = std::chrono::steady_clock::now();
    JCUDA(cudaStreamSynchronize(st));
    auto t_sync1 = std::chrono::steady_clock::now();
    const unsigned int maxlen = *h_maxlen;
    const int64_t nnz = *h_nnz;
    J->nnz = nnz;
    if (maxlen > kMaxLen) {
      crop_set_error(CROP_EINPUT, "transaction of %u items exceeds the %u-item limit", maxlen, kMaxLen);
      rc = CROP_EINPUT;
      goto fail;
    }
    if ((uint64_t)nnz >= (1ull << 32)) {
      crop_set_error(CROP_EINPUT, "%lld item occurrences exceed the 2^32 limit of one job; "
                     "split the stream", (long long)nnz);
      rc = CROP_EINPUT;
      goto fail;
    }
    // host scratch reused across jobs (under the arena lock): no first-touch
    // page faults on the planning path
    static std::vector<unsigned long long> terms, occ;
    static std::vector<uint32_t> item_tile;
    terms.resize(nn);
    occ.resize(nn);
    unsigned long long occ_sum = 0;
    J->total_terms = 0;
    for (uint32_t i = 0; i < n_items; ++i) {
      const unsigned long long x = stats[i];
      terms[i] = x & (kOccOne - 1);
      occ[i] = x >> kOccShift;
      J->total_terms += terms[i];
      occ_sum += occ[i];
    }
    {
      // stream mode when rows are short on average (words stay < 2^32);
      // CROP_FORCE_ENTRY_MODE / CROP_FORCE_STREAM_MODE override (tests)
      const bool fits = J->total_terms + 2 * occ_sum + 2ull * n_items + 2 < (1ull << 32);
      if (getenv("CROP_FORCE_ENTRY_MODE")) J->stream_mode = false;
      else if (getenv("CROP_FORCE_STREAM_MODE")) J->stream_mode = fits;
      else J->stream_mode = fits && occ_sum > 0 &&
                            J->total_terms <= (unsigned long long)kStreamMeanMax * occ_sum;
    }
    auto t_p0 = std::chrono::steady_clock::now();
    plan_tiles(J, terms, occ, item_tile);
    auto t_p1 = std::chrono::steady_clock::now();
    const uint32_t nt = (uint32_t)J->tiles.size();
    J->nt = nt;
    J->nu = (uint32_t)J->units.size();
    const bool sm = J->stream_mode;
    // reduce chunks (stream mode): (split tile, first slot)
    uint32_t nrc = 0;
    if (sm)
      for (uint32_t t : J->split) nrc += (std::min(J->tiles[t].width, kSHalf) + kReduceSlots - 1) / kReduceSlots;
    J->n_reduce_chunks = nrc;
    // one device block: [uploaded part | device-only part]
    const size_t o_tiles = 0;
    const size_t o_units = align16(o_tiles + (size_t)nt * sizeof(Tile));
    const size_t o_split = align16(o_units + J->units.size() * sizeof(Unit));
    const size_t o_ebase = align16(o_split + J->split.size() * 4);
    const size_t o_end = align16(o_ebase + (size_t)nt * 8);
    const size_t o_item = align16(o_end + (sm ? 0 : (size_t)nt * 8));
    const size_t o_rc = align16(o_item + (size_t)nn * (sm ? sizeof(uint2) : 4));
    const size_t up_bytes = align16(o_rc + (size_t)nrc * sizeof(uint2));
    const size_t o_tentries = up_bytes;
    const size_t o_cursor = align16(o_tentries + (size_t)nt * 4);
    const size_t o_twords = align16(o_cursor + (size_t)nt * 8);
    const size_t o_tdone = align16(o_twords + (size_t)nt * 8);
    const size_t o_misc = align16(o_tdone + (size_t)nt * 4);  // total_entries, unit_counter, overflow
    const size_t blk_bytes = o_misc + 32;
    JCUDA(g_pinned.reserve(up_bytes));
    unsigned char* hb = g_pinned.p;
    if (nt) memcpy(hb + o_tiles, J->tiles.data(), (size_t)nt * sizeof(Tile));
    if (!J->units.empty()) memcpy(hb + o_units, J->units.data(), J->units.size() * sizeof(Unit));
    if (!J->split.empty()) memcpy(hb + o_split, J->split.data(), J->split.size() * 4);
    unsigned long long* h_base = reinterpret_cast<unsigned long long*>(hb + o_ebase);
    unsigned long long run = 0;
    if (sm) {
      // stream mode: word bases come from the device (scan of per-tile totals)
      uint2* info = reinterpret_cast<uint2*>(hb + o_item);
      for (uint32_t i = 0; i < nn; ++i) {
        const uint32_t tv = i < n_items ? item_tile[i] : kNone;
        if (tv == kNone) {
          info[i] = make_uint2(kNone, 0u);
          continue;
        }
        const Tile& T = J->tiles[tv & ~kWinFlag];
        const uint32_t flag = (!(tv & kWinFlag) && T.mode == 2) ? kEntFlag : 0u;
        info[i] = make_uint2(tv | flag, (tv & kWinFlag) ? 0u : stream_base(T, i, n_items, J->col_bits, J->upper != 0));
      }
      uint2* rcs = reinterpret_cast<uint2*>(hb + o_rc);
      uint32_t k = 0;
      for (uint32_t t : J->split)
        for (uint32_t c0 = 0; c0 < std::min(J->tiles[t].width, kSHalf); c0 += kReduceSlots) rcs[k++] = make_uint2(t, c0);
      for (uint32_t t = 0; t < nt; ++t) h_base[t] = 0;
    } else {
      // entry capacity per tile: a row occurrence with a partner after it
      // makes at most one entry per tile (per window for split rows)
      unsigned long long* h_end = reinterpret_cast<unsigned long long*>(hb + o_end);
      for (uint32_t t = 0; t < nt; ++t) h_end[t] = 0;
      for (uint32_t i = 0; i < n_items; ++i) {
        if (item_tile[i] == kNone) continue;
        const uint32_t t = item_tile[i] & ~kWinFlag;
        if (item_tile[i] & kWinFlag)
          for (uint32_t w = 0; w < J->tiles[t].nwin; ++w) h_end[t + w] += occ[i];
        else
          h_end[t] += occ[i];
      }
      for (uint32_t t = 0; t < nt; ++t) {
        h_base[t] = run;
        run += h_end[t];
        h_end[t] = run;
      }
      memcpy(hb + o_item, item_tile.data(), (size_t)n_items * 4);
    }
    J->entry_cap = run;
    {
      const double per_tx = n_tx ? (double)run / (double)n_tx : 1.0;
      int c = (int)(kStage / std::max(1.0, 1.25 * per_tx));
      J->route_chunk_tx = std::max(8, std::min(kChunkTx, c));
    }
    if (!sm && J->entry_cap >= (1ull << 32)) {
      crop_set_error(CROP_ERESOURCE, "%llu entries exceed the 2^32 limit of one job; split the stream",
                     (unsigned long long)J->entry_cap);
      rc = CROP_ERESOURCE;
      goto fail;
    }
    JCUDA(cudaMallocAsync(&J->d_block, blk_bytes, st));
    {
      unsigned char* db = reinterpret_cast<unsigned char*>(J->d_block);
      J->d_tiles = reinterpret_cast<Tile*>(db + o_tiles);
      J->d_units = reinterpret_cast<Unit*>(db + o_units);
      J->d_split = reinterpret_cast<uint32_t*>(db + o_split);
      J->d_tile_ebase = reinterpret_cast<unsigned long long*>(db + o_ebase);
      J->d_tile_end = reinterpret_cast<unsigned long long*>(db + o_end);
      if (sm) J->d_item_info = reinterpret_cast<uint2*>(db + o_item);
      else J->d_item_tile = reinterpret_cast<uint32_t*>(db + o_item);
      J->d_reduce_chunks = reinterpret_cast<uint2*>(db + o_rc);
      J->d_tile_entries = reinterpret_cast<uint32_t*>(db + o_tentries);
      J->d_tile_cursor = reinterpret_cast<unsigned long long*>(db + o_cursor);
      J->d_tile_words = reinterpret_cast<unsigned long long*>(db + o_twords);
      J->d_tile_done = reinterpret_cast<unsigned int*>(db + o_tdone);
      J->d_total_entries = reinterpret_cast<unsigned long long*>(db + o_misc);
      J->d_unit_counter = reinterpret_cast<unsigned int*>(db + o_misc + 8);
      J->d_overflow = reinterpret_cast<uint32_t*>(db + o_misc + 16);
      JCUDA(cudaMemcpyAsync(db, hb, up_bytes, cudaMemcpyHostToDevice, st));
      JCUDA(cudaMemsetAsync(db + o_misc, 0, 32, st));
      JCUDA(cudaEventRecord(g_pinned.done, st));
    }
    if (J->n_slabs)
      JCUDA(cudaMallocAsync(&J->d_slabs, J->n_slabs * (size_t)(sm ? kSHalf : kHalf) * 4, st));
    // words: <= one per term, or two per entry row occurrence, plus the even rounding per tile
    if (sm) JCUDA(cudaMallocAsync(&J->d_words, (J->total_terms + 2 * occ_sum + 2 * (uint64_t)nt + 2) * 4, st));
    else JCUDA(cudaMallocAsync(&J->d_entries, std::max<uint64_t>(1, J->entry_cap) * sizeof(uint2), st));
    // host vectors read by the async uploads live in J until destroy
    if (getenv("CROP_DEBUG_TIMING")) {
      auto t_end = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) {
        return std::chrono::duration_cast<std::chrono::microseconds>(b - a).count();
      };
      fprintf(stderr, "[crop_pairs_create] wait passA %lld us, unpack %lld us, plan %lld us, "
              "pack+uploads %lld us, tiles %zu\n", (long long)us(t_sync0, t_sync1),
              (long long)us(t_sync1, t_p0), (long long)us(t_p0, t_p1), (long long)us(t_p1, t_end),
              J->tiles.size());
    }
  }
#undef JCUDA
  if (J->stream_mode) {
    rc = early_write(J, st);
    if (rc) goto fail;
  }
  *job = J;
  return CROP_OK;
fail:
  free_job(J);
  delete J;
  return rc;
}

extern "C" int crop_pairs_info(const crop_pairs* J, uint64_t* max_entries, uint64_t* total_terms,
                               uint64_t* n_tiles, uint64_t* n_units) {
  if (max_entries) *max_entries = J->max_entries;
  if (total_terms) *total_terms = J->total_terms;
  if (n_tiles) *n_tiles = J->nt;
  if (n_units) *n_units = J->nu;
  return CROP_OK;
}

extern "C" int crop_pairs_own_terms(const crop_pairs* J, uint64_t* own_terms) {
  *own_terms = J->own_terms;
  return CROP_OK;
}

extern "C" int crop_pairs_run(crop_pairs* J, uint32_t* out_row, uint32_t* out_col,
                              uint32_t* out_count, uint64_t* d_n_entries, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t nt = J->nt;
  CROP_CUDA(cudaMemsetAsync(d_n_entries, 0, 8, st));
  if (nt == 0 || J->n_tx == 0) return CROP_OK;
  const bool up = J->upper != 0;
  const uint32_t ns = std::min(nt, kTileSmem);
  auto mark = [&](int k) {
    if (J->timing) cudaEventRecord(J->ev[k], st);
  };
  if (J->stream_mode) {
    if (!J->written) {
      if (int rc = stream_write(J, st, J->timing)) return rc;
    }
    J->written = false;  // a re-run (capacity) writes again
    mark(3);
    CROP_CUDA(cudaMemsetAsync(J->d_unit_counter, 0, 4, st));
    CROP_CUDA(cudaMemsetAsync(J->d_tile_done, 0, nt * 4, st));
    StreamCountArgs C{};
    C.tiles = J->d_tiles;
    C.units = J->d_units;
    C.n_units = J->nu;
    C.tile_base = J->d_tile_ebase;
    C.tile_words = J->d_tile_words;
    C.words = J->d_words;
    C.items = J->items;
    C.items16 = nullptr;
    C.items_cls = nullptr;
    C.overflow = J->d_overflow;
    if (J->d_items16 || J->d_items_cls) {
      CROP_CUDA(cudaStreamWaitEvent(st, J->ev_items16, 0));
      C.items16 = J->d_items16;
      C.items_cls = J->d_items_cls;
    }
    C.h_row = J->iv.h_row;
    C.kappa = J->iv.kappa;
    C.start = J->iv.start;
    C.stop = J->iv.stop;
    C.unit_counter = J->d_unit_counter;
    C.n_items = J->n_items;
    C.col_bits = J->col_bits;
    C.upper = up;
    C.out_row = out_row;
    C.out_col = out_col;
    C.out_count = out_count;
    C.out_n = (unsigned long long*)d_n_entries;
    C.out_cap = J->out_cap ? J->out_cap : J->max_entries;
    C.slabs = J->d_slabs;
    C.tile_done = J->d_tile_done;
    C.topk_hist = J->topk_hist;
    C.hi_list = J->hi_list;
    C.hi_n = J->hi_n;
    C.dbg = nullptr;
    if (getenv("CROP_DEBUG_KINDS")) {
      static unsigned long long* dbg = nullptr;
      if (!dbg) cudaMalloc(&dbg, 20 * 8);
      cudaMemsetAsync(dbg, 0, 20 * 8, st);
      C.dbg = dbg;
    }
    auto kcs = C.items_cls ? (C.dbg ? k_count_stream<true, true> : k_count_stream<false, true>)
                           : (C.dbg ? k_count_stream<true, false> : k_count_stream<false, false>);
    CROP_CUDA(cudaFuncSetAttribute(kcs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStreamSmem));
    mark(4);
    kcs<<<std::min<int>(2 * kNumSMs, (int)J->nu), kSCThreads, kStreamSmem, st>>>(C);
    CROP_LAUNCH_CHECK();
    const uint32_t nrc = J->n_reduce_chunks;
    if (nrc) {
      k_reduce_slabs<<<std::min<uint32_t>(nrc, kNumSMs * 8), 256, 0, st>>>(C, J->d_reduce_chunks, nrc);
      CROP_LAUNCH_CHECK();
    }
    mark(5);
    if (C.dbg) {
      unsigned long long h[20];
      cudaMemcpyAsync(h, C.dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const char* names[4] = {"dense-row", "dense-multi", "dense-split", "hash"};
      for (int k = 0; k < 4; ++k)
        fprintf(stderr, "[k_count_stream] %-11s units %6llu words %10llu zero %7.1f count %8.1f emit %7.1f Mcyc\n",
                names[k], h[5 * k + 3], h[5 * k + 4], h[5 * k] / 1e6, h[5 * k + 1] / 1e6, h[5 * k + 2] / 1e6);
    }
    crop_count_launches((J->words_known ? 3 : 4) + (nrc ? 1 : 0));
    return CROP_OK;
  }
  // route: one walk, staged per chunk, ranges claimed per touched tile
  mark(0);
  CROP_CUDA(cudaMemcpyAsync(J->d_tile_cursor, J->d_tile_ebase, nt * 8, cudaMemcpyDeviceToDevice, st));
  {
    auto kern = up ? k_route<true> : k_route<false>;
    const size_t smem = (size_t)(J->route_chunk_tx + 1) * 8 + (size_t)kStage * 16 + 16 + ns * 4;
    CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((kChunkTx + 1) * 8 + kStage * 16 + 16 + kTileSmem * 4)));
    const int64_t rchunks = (J->n_tx + J->route_chunk_tx - 1) / J->route_chunk_tx;
    const int rgrid = (int)std::min<int64_t>(kNumSMs, rchunks);
    kern<<<rgrid, kPassThreads, smem, st>>>(J->offsets, J->items, J->n_tx, J->route_chunk_tx,
                                            J->d_item_tile, J->d_tiles, nt, J->d_tile_cursor,
                                            J->d_tile_end, J->d_entries, J->d_overflow);
    CROP_LAUNCH_CHECK();
  }
  mark(1);
  k_tile_entries<<<(nt + 255) / 256, 256, 0, st>>>(J->d_tile_cursor, J->d_tile_ebase, nt,
                                                   J->d_tile_entries);
  CROP_LAUNCH_CHECK();
  mark(2);
  mark(3);
  // count
  CROP_CUDA(cudaMemsetAsync(J->d_unit_counter, 0, 4, st));
  CROP_CUDA(cudaMemsetAsync(J->d_tile_done, 0, nt * 4, st));
  {
    CountArgs A{};
    A.items = J->items;
    A.tiles = J->d_tiles;
    A.units = J->d_units;
    A.n_units = J->nu;
    A.tile_ebase = J->d_tile_ebase;
    A.tile_entries = J->d_tile_entries;
    A.entries = J->d_entries;
    A.unit_counter = J->d_unit_counter;
    A.n_items = J->n_items;
    A.col_bits = J->col_bits;
    A.kappa = J->iv.kappa;
    A.start = J->iv.start;
    A.stop = J->iv.stop;
    A.h_row = J->iv.h_row;
    A.h_col = J->iv.h_col;
    A.out_row = out_row;
    A.out_col = out_col;
    A.out_count = out_count;
    A.out_n = (unsigned long long*)d_n_entries;
    A.out_cap = J->out_cap ? J->out_cap : J->max_entries;
    A.slabs = J->d_slabs;
    A.tile_done = J->d_tile_done;
    A.dbg = nullptr;
    if (getenv("CROP_DEBUG_KINDS")) {
      static unsigned long long* dbg = nullptr;
      if (!dbg) cudaMalloc(&dbg, 16 * 8);
      cudaMemsetAsync(dbg, 0, 16 * 8, st);
      A.dbg = dbg;
    }
    void (*kern)(CountArgs);
    if (up) kern = J->filter ? k_count<true, true> : k_count<true, false>;
    else kern = J->filter ? k_count<false, true> : k_count<false, false>;
    CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCountSmem));
    const int grid = std::min<int>(kNumSMs, (int)J->nu);
    mark(4);
    kern<<<grid, kCountThreads, kCountSmem, st>>>(A);
    CROP_LAUNCH_CHECK();
    mark(5);
    if (A.dbg) {
      unsigned long long h[16];
      cudaMemcpyAsync(h, A.dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const char* names[4] = {"dense-row", "window", "dense-multi", "hash"};
      for (int k = 0; k < 4; ++k)
        fprintf(stderr, "[k_count] %-11s units %6llu entries %10llu count %8.1f Mcyc emit %8.1f Mcyc\n",
                names[k], h[4 * k + 2], h[4 * k + 3], h[4 * k] / 1e6, h[4 * k + 1] / 1e6);
    }
  }
  crop_count_launches(3);
  return CROP_OK;
}

extern "C" int crop_pairs_set_timing(crop_pairs* J, int on) {
  if (on && !J->ev[0])
    for (cudaEvent_t& e : J->ev) CROP_CUDA(cudaEventCreate(&e));
  J->timing = on != 0;
  return CROP_OK;
}

// Durations (ms) of the last run's phases: route-count, scan, route-write, count.
extern "C" int crop_pairs_phase_ms(const crop_pairs* J, float* out4) {
  if (!J->timing) {
    crop_set_error(CROP_ECONFIG, "timing was not enabled on this job");
    return CROP_ECONFIG;
  }
  CROP_CUDA(cudaEventSynchronize(J->ev[5]));
  CROP_CUDA(cudaEventElapsedTime(&out4[0], J->ev[0], J->ev[1]));
  CROP_CUDA(cudaEventElapsedTime(&out4[1], J->ev[1], J->ev[2]));
  CROP_CUDA(cudaEventElapsedTime(&out4[2], J->ev[2], J->ev[3]));
  CROP_CUDA(cudaEventElapsedTime(&out4[3], J->ev[4], J->ev[5]));
  return CROP_OK;
}

extern "C" int crop_pairs_set_topk(crop_pairs* J, uint32_t* hist, uint64_t* hi_list, uint64_t* hi_n,
                                   uint64_t hi_cap) {
  if (!J->stream_mode) {
    crop_set_error(CROP_ECONFIG, "fused top-k buffers need a stream-mode job");
    return CROP_ECONFIG;
  }
  if (hist && hi_cap < J->total_terms / kTopkExactBins + 1) {
    crop_set_error(CROP_ERESOURCE, "hi_list holds %llu entries, need %llu", (unsigned long long)hi_cap,
                   (unsigned long long)(J->total_terms / kTopkExactBins + 1));
    return CROP_ERESOURCE;
  }
  J->topk_hist = hist;
  J->hi_list = reinterpret_cast<unsigned long long*>(hi_list);
  J->hi_n = reinterpret_cast<unsigned long long*>(hi_n);
  return CROP_OK;
}

extern "C" int crop_topk_fused(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                               const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k,
                               uint32_t* hist, const uint64_t* hi_list, const uint64_t* hi_n,
                               uint64_t* out_idx, uint64_t* d_k_out, void* stream) {
  return crop_topk_impl(row, col, count, d_n_entries, max_entries, k, out_idx, d_k_out,
                        (cudaStream_t)stream, hist, reinterpret_cast<const unsigned long long*>(hi_list),
                        reinterpret_cast<const unsigned long long*>(hi_n));
}

extern "C" int crop_pairs_set_capacity(crop_pairs* J, uint64_t capacity) {
  J->out_cap = capacity < J->max_entries ? capacity : J->max_entries;
  return CROP_OK;
}

extern "C" int crop_pairs_mode(const crop_pairs* J, int* stream_mode) {
  *stream_mode = J->stream_mode ? 1 : 0;
  return CROP_OK;
}

extern "C" int crop_pairs_own(const crop_pairs* J, int* own) {
  *own = J->own ? 1 : 0;
  return CROP_OK;
}

extern "C" int crop_pairs_overflowed(const crop_pairs* J, int* overflowed) {
  // stream mode: the count kernel raises the flag when a 16-bit counter wraps
  uint32_t h = 0;
  CROP_CUDA(cudaMemcpyAsync(&h, J->d_overflow, 4, cudaMemcpyDeviceToHost, J->stream));
  CROP_CUDA(cudaStreamSynchronize(J->stream));
  *overflowed = h != 0;
  return CROP_OK;
}

extern "C" void crop_pairs_destroy(crop_pairs* J) {
  if (!J) return;
  free_job(J);
  delete J;
}
