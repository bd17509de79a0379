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
#include <vector>

#include "common.cuh"

using namespace crop;

namespace {

constexpr int kCountThreads = 1024;
constexpr int kCountWarps = kCountThreads / 32;
constexpr uint32_t kDenseCap = 49152;   // dense counters per tile (192 KB)
constexpr uint32_t kHashSlots = 24576;  // hash slots per tile (keys+counts 192 KB)
constexpr uint32_t kHashCap = 16384;    // max distinct keys per hash tile (load <= 0.67)
constexpr uint32_t kMaxLen = 8192;      // longest transaction (u32 pair counts per warp)
constexpr uint32_t kStatSmemItems = 53248;
constexpr uint32_t kTileSmem = 53248;   // route-pass shared tile counters
constexpr int kRouteThreads = 512;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr size_t kTableBytes = 196608;  // max(kDenseCap*4, kHashSlots*8)
constexpr size_t kJobBytes = kCountWarps * 32 * 24;
constexpr size_t kCountSmem = kTableBytes + kJobBytes + 64;

struct Tile {
  uint32_t row0, row1;  // rows [row0, row1)
  uint32_t c0, c1;      // column window [c0, c1)
  uint32_t mode;        // 0 dense, 1 hash
  uint32_t nwin;        // first window tile of a split row: #windows; else 0
  uint32_t n_units;
  uint32_t width;       // dense: counters used
  uint64_t slab_base;   // multi-unit dense: first slab
  uint64_t terms;       // planning estimate (all buckets)
};

struct Unit {
  uint32_t tile, local;
};

__host__ __device__ __forceinline__ uint64_t tri_rowbase(uint64_t r, uint64_t row0, uint64_t n) {
  // sum_{x=row0}^{r-1} (n - 1 - x)
  uint64_t k = r - row0;
  return k * (n - 1) - k * (row0 + r - 1) / 2;
}

// ------------------------------------------------------------- pass A
template <bool UPPER>
__global__ void __launch_bounds__(512)
    k_item_terms(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items,
                 int64_t n_tx, uint32_t n_items, unsigned long long* __restrict__ terms,
                 unsigned int* __restrict__ max_len) {
  extern __shared__ uint32_t s_terms[];
  const uint32_t n_smem = n_items < kStatSmemItems ? n_items : kStatSmemItems;
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x) s_terms[i] = 0;
  __syncthreads();
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  uint32_t my_max = 0;
  for (int64_t t = (int64_t)blockIdx.x * warps + threadIdx.x / 32; t < n_tx;
       t += (int64_t)gridDim.x * warps) {
    int64_t base = offsets[t];
    uint32_t L = (uint32_t)(offsets[t + 1] - base);
    my_max = max(my_max, L);
    for (uint32_t p = lane; p < L; p += 32) {
      uint32_t i = items[base + p];
      uint32_t c = UPPER ? L - 1 - p : L;
      if (c == 0) continue;
      if (i < n_smem) atomicAdd(&s_terms[i], c);
      else atomicAdd(&terms[i], (unsigned long long)c);
    }
  }
  if (lane == 0) atomicMax(max_len, my_max);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_smem; i += blockDim.x)
    if (s_terms[i]) atomicAdd(&terms[i], (unsigned long long)s_terms[i]);
}

// ------------------------------------------------------------- pass B
// Walks one transaction with a warp and calls emit(tile, tx, packed) for each
// entry: a run of consecutive positions whose rows share a (non-windowed)
// tile, or one (row, window) per column window present after the row.
template <bool UPPER, typename Emit>
__device__ __forceinline__ void walk_tx(int64_t tx, const int64_t* __restrict__ offsets,
                                        const uint32_t* __restrict__ items,
                                        const uint32_t* __restrict__ item_tile,
                                        const Tile* __restrict__ tiles, Emit&& emit) {
  const int lane = threadIdx.x & 31;
  const int64_t base = offsets[tx];
  const uint32_t L = (uint32_t)(offsets[tx + 1] - base);
  for (uint32_t c = 0; c < L; c += 32) {
    const uint32_t p = c + lane;
    const bool valid = p < L;
    uint32_t item = valid ? items[base + p] : 0;
    uint32_t tile = valid ? item_tile[item] : kNone;
    if (UPPER && p + 1 >= L) tile = kNone;  // last item has no partner after it
    bool windowed = false;
    if (tile != kNone) windowed = tiles[tile].nwin != 0;
    uint32_t prev = __shfl_up_sync(0xffffffffu, tile, 1);
    uint32_t next = __shfl_down_sync(0xffffffffu, tile, 1);
    if (lane == 0) prev = kNone;
    if (lane == 31) next = kNone;
    const bool run_member = tile != kNone && !windowed;
    const bool is_start = run_member && tile != prev;
    const bool is_end = run_member && tile != next;
    const uint32_t end_mask = __ballot_sync(0xffffffffu, is_end);
    if (is_start) {
      uint32_t e = __ffs(end_mask & (0xffffffffu << lane)) - 1;
      uint32_t p1 = c + e + 1;
      emit(tile, tx, p | (p1 << 16));
    }
    if (windowed) {
      // columns after (UPPER) or anywhere in (full) the transaction, grouped
      // by window; sorted items => window ids are non-decreasing.
      const Tile t0 = tiles[tile];
      const uint32_t lo = t0.c0;  // column start of window 0
      uint32_t last_w = kNone;
      for (uint32_t q = UPPER ? p + 1 : 0; q < L; ++q) {
        uint32_t j = items[base + q];
        if (j < lo) continue;
        uint32_t w = (j - lo) / kDenseCap;
        if (w >= t0.nwin) break;
        if (w != last_w) {
          emit(tile + w, tx, p | ((p + 1) << 16));
          last_w = w;
        }
      }
    }
  }
}

struct CountEmit {
  uint32_t* s_cnt;
  uint32_t* g_cnt;
  __device__ void operator()(uint32_t tile, int64_t, uint32_t) const {
    if (tile < kTileSmem) atomicAdd(&s_cnt[tile], 1u);
    else atomicAdd(&g_cnt[tile], 1u);
  }
};

template <bool UPPER>
__global__ void __launch_bounds__(kRouteThreads)
    k_route_count(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items,
                  int64_t n_tx, const uint32_t* __restrict__ item_tile,
                  const Tile* __restrict__ tiles, uint32_t n_tiles,
                  uint32_t* __restrict__ tile_entries) {
  extern __shared__ uint32_t s_cnt[];
  const uint32_t ns = n_tiles < kTileSmem ? n_tiles : kTileSmem;
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  __syncthreads();
  const int warps = blockDim.x / 32;
  CountEmit em{s_cnt, tile_entries};
  for (int64_t tx = (int64_t)blockIdx.x * warps + threadIdx.x / 32; tx < n_tx;
       tx += (int64_t)gridDim.x * warps)
    walk_tx<UPPER>(tx, offsets, items, item_tile, tiles, em);
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x)
    if (s_cnt[t]) atomicAdd(&tile_entries[t], s_cnt[t]);
}

struct WriteEmit {
  uint32_t* s_cur;
  unsigned long long* g_cur;
  uint2* entries;
  unsigned long long cap;
  uint32_t* overflow;
  __device__ void operator()(uint32_t tile, int64_t tx, uint32_t packed) const {
    unsigned long long pos;
    if (tile < kTileSmem) pos = atomicAdd(&s_cur[tile], 1u);  // holds the claimed base
    else pos = atomicAdd(&g_cur[tile], 1ull);
    if (pos < cap) entries[pos] = make_uint2((uint32_t)tx, packed);
    else *overflow = 1u;
  }
};

// Static transaction ranges per CTA: count the range's entries per tile in
// shared memory, claim one global range per touched tile, then write.
template <bool UPPER>
__global__ void __launch_bounds__(kRouteThreads)
    k_route_write(const int64_t* __restrict__ offsets, const uint32_t* __restrict__ items,
                  int64_t n_tx, const uint32_t* __restrict__ item_tile,
                  const Tile* __restrict__ tiles, uint32_t n_tiles,
                  unsigned long long* __restrict__ tile_cursor, uint2* __restrict__ entries,
                  unsigned long long cap, uint32_t* __restrict__ overflow) {
  extern __shared__ uint32_t s_cnt[];
  const uint32_t ns = n_tiles < kTileSmem ? n_tiles : kTileSmem;
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) s_cnt[t] = 0;
  __syncthreads();
  const int warps = blockDim.x / 32;
  const int64_t tx0 = n_tx * blockIdx.x / gridDim.x, tx1 = n_tx * (blockIdx.x + 1) / gridDim.x;
  // walk 1: local counts for shared-memory tiles only
  struct LocalCount {
    uint32_t* s;
    __device__ void operator()(uint32_t tile, int64_t, uint32_t) const {
      if (tile < kTileSmem) atomicAdd(&s[tile], 1u);
    }
  } lc{s_cnt};
  for (int64_t tx = tx0 + threadIdx.x / 32; tx < tx1; tx += warps)
    walk_tx<UPPER>(tx, offsets, items, item_tile, tiles, lc);
  __syncthreads();
  // claim: replace each count by the claimed global position (fits 32 bits
  // only if entries < 2^32; checked on the host)
  for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) {
    uint32_t c = s_cnt[t];
    if (c) s_cnt[t] = (uint32_t)atomicAdd(&tile_cursor[t], (unsigned long long)c);
  }
  __syncthreads();
  WriteEmit we{s_cnt, tile_cursor, entries, cap, overflow};
  for (int64_t tx = tx0 + threadIdx.x / 32; tx < tx1; tx += warps)
    walk_tx<UPPER>(tx, offsets, items, item_tile, tiles, we);
}

// ------------------------------------------------------------- count
struct CountArgs {
  const int64_t* offsets;
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
  int filter;
  uint32_t kappa, start, stop;
  const uint32_t* h_row;
  const uint32_t* h_col;
  // output
  uint32_t* out_row;
  uint32_t* out_col;
  uint32_t* out_count;
  unsigned long long* out_n;
  uint32_t* slabs;
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

// Block-wide exclusive scan of one value per thread (1024 threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = warp_incl_scan(v);
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = s_warp[lane];
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

template <bool UPPER, bool FILTER>
__global__ void __launch_bounds__(kCountThreads, 1) k_count(CountArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* table = reinterpret_cast<uint32_t*>(smem);  // dense counters or hash keys
  uint32_t* hcount = table + kHashSlots;                 // hash counts
  uint32_t* job = reinterpret_cast<uint32_t*>(smem + kTableBytes);
  uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + kTableBytes + kJobBytes);
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_base;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-warp job arrays (struct of arrays, 32 lanes each)
  uint32_t* j_base_lo = job + warp * 32 * 6;
  uint32_t* j_L = j_base_lo + 32;
  uint32_t* j_p = j_L + 32;      // p0 | p1 << 16
  uint32_t* j_q = j_p + 32;      // q0 | q1 << 16 (windowed / full)
  uint32_t* j_incl = j_q + 32;
  uint32_t* j_base_hi = j_incl + 32;
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

    if (dense) {
      uint4* t4 = reinterpret_cast<uint4*>(table);
      for (uint32_t s = threadIdx.x; s < (width + 3) / 4; s += kCountThreads)
        t4[s] = make_uint4(0, 0, 0, 0);
    } else {
      for (uint32_t s = threadIdx.x; s < kHashSlots; s += kCountThreads) {
        table[s] = kEmpty32;
        hcount[s] = 0;
      }
    }
    __syncthreads();

    for (uint64_t eb_w = e0 + (uint64_t)warp * 32; eb_w < e1; eb_w += (uint64_t)kCountWarps * 32) {
      const uint64_t e = eb_w + lane;
      uint32_t cnt = 0, p0 = 0, p1 = 0, q0 = 0, q1 = 0, L = 0;
      int64_t base = 0;
      if (e < e1) {
        const uint2 en = A.entries[e];
        base = A.offsets[en.x];
        L = (uint32_t)(A.offsets[en.x + 1] - base);
        p0 = en.y & 0xFFFFu;
        p1 = en.y >> 16;
        if (windowed || !UPPER) {
          // columns: positions whose item lies in [c0, c1) (after the row when UPPER)
          const uint32_t* it = A.items + base;
          uint32_t lo = UPPER ? p0 + 1 : 0;
          q0 = lower_bound_items(it, lo, L, T.c0);
          q1 = lower_bound_items(it, q0, L, T.c1);
          cnt = (p1 - p0) * (q1 - q0);
        } else {
          const uint32_t k = p1 - p0;
          cnt = k * (L - 1) - (p0 + p1 - 1) * k / 2;
        }
      }
      const uint32_t incl = warp_incl_scan(cnt);
      j_base_lo[lane] = (uint32_t)base;
      j_base_hi[lane] = (uint32_t)((uint64_t)base >> 32);
      j_L[lane] = L;
      j_p[lane] = p0 | (p1 << 16);
      j_q[lane] = q0 | (q1 << 16);
      j_incl[lane] = incl;
      const uint32_t S = __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      uint32_t owner = 0;
      for (uint32_t t = lane; t < S; t += 32) {
        while (j_incl[owner] <= t) ++owner;
        const uint32_t excl = owner ? j_incl[owner - 1] : 0;
        uint32_t loc = t - excl;
        const int64_t ob = (int64_t)(((uint64_t)j_base_hi[owner] << 32) | j_base_lo[owner]);
        const uint32_t op = j_p[owner];
        uint32_t r = op & 0xFFFFu, q;
        if (windowed || !UPPER) {
          const uint32_t oq = j_q[owner];
          const uint32_t qa = oq & 0xFFFFu, ql = (oq >> 16) - qa;
          r += loc / ql;
          q = qa + loc % ql;
        } else {
          const uint32_t oL = j_L[owner];
          uint32_t w = oL - 1 - r;
          while (loc >= w) {
            loc -= w;
            ++r;
            --w;
          }
          q = r + 1 + loc;
        }
        const uint32_t i = A.items[ob + r];
        const uint32_t j = A.items[ob + q];
        if (FILTER) {
          uint32_t b = A.h_row[i] + A.h_col[j];
          if (b >= A.kappa) b -= A.kappa;
          if (b < A.start || b >= A.stop) continue;
        }
        if (dense) {
          uint32_t slot;
          if (single_row) slot = j - (UPPER ? max(T.c0, i + 1) : T.c0);
          else if (UPPER) slot = (uint32_t)tri_rowbase(i, T.row0, n) + (j - i - 1);
          else slot = (i - T.row0) * n + j;
          atomicAdd(&table[slot], 1u);
        } else {
          const uint32_t key = ((i - T.row0) << A.col_bits) | j;
          uint32_t s = __umulhi(mix32(key), kHashSlots);
          for (;;) {
            uint32_t k = table[s];
            if (k == key) {
              atomicAdd(&hcount[s], 1u);
              break;
            }
            if (k == kEmpty32) {
              uint32_t old = atomicCAS(&table[s], kEmpty32, key);
              if (old == kEmpty32 || old == key) {
                atomicAdd(&hcount[s], 1u);
                break;
              }
            }
            if (++s == kHashSlots) s = 0;
          }
        }
      }
      __syncwarp();
    }
    __syncthreads();

    if (dense && T.n_units > 1) {
      uint4* dst = reinterpret_cast<uint4*>(A.slabs + (T.slab_base + unit.local) * kDenseCap);
      const uint4* src = reinterpret_cast<const uint4*>(table);
      for (uint32_t s = threadIdx.x; s < (width + 3) / 4; s += kCountThreads) dst[s] = src[s];
    } else {
      // compact non-zero counters: warp w owns a contiguous slot range
      const uint32_t slots = dense ? width : kHashSlots;
      const uint32_t per_warp = (slots + kCountWarps - 1) / kCountWarps;
      const uint32_t s_lo = min(slots, warp * per_warp), s_hi = min(slots, s_lo + per_warp);
      uint32_t mine = 0;
      for (uint32_t s = s_lo + lane; s < s_hi; s += 32) mine += (dense ? table[s] : hcount[s]) != 0;
      mine = warp_sum(mine);
      uint32_t total;
      uint32_t wbase = block_excl_scan(lane == 0 ? mine : 0, s_warp, total);
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (threadIdx.x == 0) s_base = atomicAdd(A.out_n, (unsigned long long)total);
      __syncthreads();
      uint64_t pos = s_base + wbase;
      for (uint32_t s0 = s_lo; s0 < s_hi; s0 += 32) {
        const uint32_t s = s0 + lane;
        uint32_t c = 0, i = 0, j = 0;
        if (s < s_hi) {
          if (dense) {
            c = table[s];
            if (c) {
              if (single_row) {
                i = T.row0;
                j = s + (UPPER ? max(T.c0, i + 1) : T.c0);
              } else if (UPPER) {
                uint32_t lo = T.row0, hi = T.row1;  // last row with rowbase <= s
                while (hi - lo > 1) {
                  uint32_t mid = (lo + hi) >> 1;
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
          } else {
            c = hcount[s];
            if (c) {
              const uint32_t key = table[s];
              i = T.row0 + (key >> A.col_bits);
              j = key & ((1u << A.col_bits) - 1u);
            }
          }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, c != 0);
        if (c) {
          const uint64_t o = pos + __popc(m & ((1u << lane) - 1u));
          A.out_row[o] = i;
          A.out_col[o] = j;
          A.out_count[o] = c;
        }
        pos += __popc(m);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- reduce
struct ReduceArgs {
  const Tile* tiles;
  const uint32_t* split_tiles;  // ids of multi-unit dense tiles
  uint32_t n_split;
  const uint32_t* slabs;
  uint32_t n_items;
  uint32_t* out_row;
  uint32_t* out_col;
  uint32_t* out_count;
  unsigned long long* out_n;
};

constexpr int kReduceThreads = 1024;
constexpr uint32_t kReduceChunk = 16384;  // slots per block

template <bool UPPER>
__global__ void __launch_bounds__(kReduceThreads) k_slab_reduce(ReduceArgs A) {
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_base;
  const uint32_t chunks_per_tile = (kDenseCap + kReduceChunk - 1) / kReduceChunk;
  const uint32_t tile_id = A.split_tiles[blockIdx.x / chunks_per_tile];
  const uint32_t chunk = blockIdx.x % chunks_per_tile;
  const Tile T = A.tiles[tile_id];
  const uint32_t n = A.n_items;
  const uint32_t lo = chunk * kReduceChunk;
  const uint32_t hi = min(T.width, lo + kReduceChunk);
  if (lo >= hi) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t per_warp = (hi - lo + 31) / 32;
  const uint32_t s_lo = min(hi, lo + warp * per_warp), s_hi = min(hi, s_lo + per_warp);
  const uint32_t* slab = A.slabs + T.slab_base * kDenseCap;
  auto sum_at = [&](uint32_t s) {
    uint32_t c = 0;
    for (uint32_t u = 0; u < T.n_units; ++u) c += slab[(uint64_t)u * kDenseCap + s];
    return c;
  };
  uint32_t mine = 0;
  for (uint32_t s = s_lo + lane; s < s_hi; s += 32) mine += sum_at(s) != 0;
  mine = warp_sum(mine);
  uint32_t total;
  uint32_t wbase = block_excl_scan(lane == 0 ? mine : 0, s_warp, total);
  wbase = __shfl_sync(0xffffffffu, wbase, 0);
  if (threadIdx.x == 0) s_base = atomicAdd(A.out_n, (unsigned long long)total);
  __syncthreads();
  uint64_t pos = s_base + wbase;
  const bool single_row = T.row1 - T.row0 == 1;
  for (uint32_t s0 = s_lo; s0 < s_hi; s0 += 32) {
    const uint32_t s = s0 + lane;
    uint32_t c = 0, i = 0, j = 0;
    if (s < s_hi) {
      c = sum_at(s);
      if (c) {
        if (single_row) {
          i = T.row0;
          j = s + (UPPER ? max(T.c0, i + 1) : T.c0);
        } else if (UPPER) {
          uint32_t a = T.row0, b = T.row1;
          while (b - a > 1) {
            uint32_t mid = (a + b) >> 1;
            if (tri_rowbase(mid, T.row0, n) <= s) a = mid;
            else b = mid;
          }
          i = a;
          j = (uint32_t)(s - tri_rowbase(i, T.row0, n)) + i + 1;
        } else {
          i = T.row0 + s / n;
          j = s % n;
        }
      }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, c != 0);
    if (c) {
      const uint64_t o = pos + __popc(m & ((1u << lane) - 1u));
      A.out_row[o] = i;
      A.out_col[o] = j;
      A.out_count[o] = c;
    }
    pos += __popc(m);
  }
}

__global__ void k_exclusive_scan_u32_to_u64(const uint32_t* __restrict__ in, uint32_t n,
                                            unsigned long long* __restrict__ out,
                                            unsigned long long* __restrict__ total) {
  // single block, 1024 threads; n up to a few million (tiles)
  __shared__ unsigned long long s_part[1024];
  const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(n, threadIdx.x * per), hi = min(n, lo + per);
  unsigned long long acc = 0;
  for (uint32_t i = lo; i < hi; ++i) acc += in[i];
  s_part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      unsigned long long v = s_part[t];
      s_part[t] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  unsigned long long run = s_part[threadIdx.x];
  for (uint32_t i = lo; i < hi; ++i) {
    out[i] = run;
    run += in[i];
  }
}

}  // namespace

// =============================================================== host side

struct crop_pairs {
  const int64_t* offsets;
  const uint32_t* items;
  int64_t n_tx;
  uint32_t n_items;
  int upper;
  bool filter;
  crop_interval iv;
  uint32_t col_bits;
  uint64_t total_terms;
  uint64_t max_entries;
  uint64_t entry_cap;
  std::vector<Tile> tiles;
  std::vector<Unit> units;
  std::vector<uint32_t> split;
  uint64_t n_slabs;
  // device
  unsigned long long* d_terms = nullptr;
  unsigned int* d_maxlen = nullptr;
  uint32_t* d_item_tile = nullptr;
  Tile* d_tiles = nullptr;
  Unit* d_units = nullptr;
  uint32_t* d_split = nullptr;
  uint32_t* d_tile_entries = nullptr;
  unsigned long long* d_tile_ebase = nullptr;
  unsigned long long* d_tile_cursor = nullptr;
  unsigned long long* d_total_entries = nullptr;
  uint2* d_entries = nullptr;
  uint32_t* d_slabs = nullptr;
  unsigned int* d_unit_counter = nullptr;
  uint32_t* d_overflow = nullptr;
};

static void free_job(crop_pairs* j) {
  cudaFree(j->d_terms);
  cudaFree(j->d_maxlen);
  cudaFree(j->d_item_tile);
  cudaFree(j->d_tiles);
  cudaFree(j->d_units);
  cudaFree(j->d_split);
  cudaFree(j->d_tile_entries);
  cudaFree(j->d_tile_ebase);
  cudaFree(j->d_tile_cursor);
  cudaFree(j->d_total_entries);
  cudaFree(j->d_entries);
  cudaFree(j->d_slabs);
  cudaFree(j->d_unit_counter);
  cudaFree(j->d_overflow);
}

// Greedy tile planner over rows in id order (see file header).
static void plan_tiles(crop_pairs* J, const std::vector<unsigned long long>& terms,
                       std::vector<uint32_t>& item_tile) {
  const uint32_t n = J->n_items;
  const bool upper = J->upper != 0;
  const uint64_t T = J->total_terms;
  const uint64_t unit_terms = std::max<uint64_t>(1ull << 16, T / ((uint64_t)kNumSMs * 8));
  const uint32_t hash_rows_max = (J->col_bits >= 32) ? 1u : ((1u << (32 - J->col_bits)) - 1u);
  struct Group {
    uint32_t row0, row1;
    uint64_t sw, sb, st;
    bool dense_ok, hash_ok;
  };
  std::vector<Tile> tiles;
  std::vector<std::vector<uint32_t>> group_rows_tile;  // not needed
  item_tile.assign(n, kNone);
  auto width_of = [&](uint32_t i) -> uint64_t { return upper ? (uint64_t)(n - 1 - i) : n; };

  bool open = false;
  Group g{};
  auto close = [&]() {
    if (!open) return;
    Tile t{};
    t.row0 = g.row0;
    t.row1 = g.row1;
    t.c0 = 0;
    t.c1 = n;
    bool dense = g.dense_ok && (!g.hash_ok || g.st * 8 >= g.sw);
    t.mode = dense ? 0 : 1;
    t.nwin = 0;
    t.width = dense ? (uint32_t)g.sw : 0;
    t.terms = g.st;
    t.n_units = dense ? (uint32_t)std::min<uint64_t>(4096, (g.st + unit_terms - 1) / unit_terms) : 1;
    if (t.n_units == 0) t.n_units = 1;
    uint32_t id = (uint32_t)tiles.size();
    for (uint32_t i = g.row0; i < g.row1; ++i)
      if (terms[i]) item_tile[i] = id;
    tiles.push_back(t);
    open = false;
  };
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t tm = terms[i];
    const uint64_t w = width_of(i);
    const uint64_t b = std::min<uint64_t>(w, tm);
    if (open) {
      bool d_ok = g.dense_ok && g.sw + w <= kDenseCap;
      bool h_ok = g.hash_ok && g.sb + b <= kHashCap && g.st + tm <= unit_terms &&
                  (g.row1 - g.row0 + 1) <= hash_rows_max;
      if (d_ok || h_ok) {
        g.row1 = i + 1;
        g.sw += w;
        g.sb += b;
        g.st += tm;
        g.dense_ok = d_ok;
        g.hash_ok = h_ok;
        continue;
      }
      close();
    }
    if (tm == 0) continue;
    const bool d_ok = w <= kDenseCap;
    const bool h_ok = b <= kHashCap && tm <= unit_terms;
    if (d_ok || h_ok) {
      open = true;
      g = Group{i, i + 1, w, b, tm, d_ok, h_ok};
      continue;
    }
    // single row too wide for a dense tile and too heavy for a hash tile:
    // column windows of kDenseCap counters, consecutive tile ids.
    const uint32_t col_lo = upper ? i + 1 : 0;
    const uint32_t nwin = (uint32_t)((w + kDenseCap - 1) / kDenseCap);
    const uint32_t first = (uint32_t)tiles.size();
    for (uint32_t k = 0; k < nwin; ++k) {
      Tile t{};
      t.row0 = i;
      t.row1 = i + 1;
      t.c0 = col_lo + k * kDenseCap;
      t.c1 = (uint32_t)std::min<uint64_t>(n, (uint64_t)t.c0 + kDenseCap);
      t.mode = 0;
      t.nwin = k == 0 ? nwin : 0;
      t.width = t.c1 - t.c0;
      t.terms = tm / nwin + 1;
      t.n_units = (uint32_t)std::min<uint64_t>(4096, (t.terms + unit_terms - 1) / unit_terms);
      if (t.n_units == 0) t.n_units = 1;
      tiles.push_back(t);
    }
    // window 0 must start at col_lo for the router's window arithmetic
    item_tile[i] = first;
  }
  close();

  // Renumber heavy-first (router keeps the heaviest tiles in shared memory);
  // a split row's windows stay consecutive.
  std::vector<uint32_t> groups;  // first tile of each group
  for (uint32_t t = 0; t < tiles.size();) {
    groups.push_back(t);
    t += tiles[t].nwin ? tiles[t].nwin : 1;
  }
  auto group_terms = [&](uint32_t t) {
    uint64_t s = 0;
    uint32_t k = tiles[t].nwin ? tiles[t].nwin : 1;
    for (uint32_t q = 0; q < k; ++q) s += tiles[t + q].terms;
    return s;
  };
  std::stable_sort(groups.begin(), groups.end(),
                   [&](uint32_t a, uint32_t b) { return group_terms(a) > group_terms(b); });
  std::vector<uint32_t> new_id(tiles.size());
  std::vector<Tile> out;
  out.reserve(tiles.size());
  for (uint32_t g0 : groups) {
    uint32_t k = tiles[g0].nwin ? tiles[g0].nwin : 1;
    for (uint32_t q = 0; q < k; ++q) {
      new_id[g0 + q] = (uint32_t)out.size();
      out.push_back(tiles[g0 + q]);
    }
  }
  for (uint32_t i = 0; i < n; ++i)
    if (item_tile[i] != kNone) item_tile[i] = new_id[item_tile[i]];
  J->tiles.swap(out);

  // units heavy-first; slabs for split dense tiles
  J->units.clear();
  J->split.clear();
  J->n_slabs = 0;
  std::vector<std::pair<uint64_t, Unit>> us;
  for (uint32_t t = 0; t < J->tiles.size(); ++t) {
    Tile& tt = J->tiles[t];
    if (tt.n_units > 1) {
      tt.slab_base = J->n_slabs;
      J->n_slabs += tt.n_units;
      J->split.push_back(t);
    }
    for (uint32_t u = 0; u < tt.n_units; ++u) us.push_back({tt.terms / tt.n_units, Unit{t, u}});
  }
  std::stable_sort(us.begin(), us.end(), [](auto& a, auto& b) { return a.first > b.first; });
  for (auto& x : us) J->units.push_back(x.second);

  uint64_t cap = 0;
  for (auto& t : J->tiles) cap += t.mode == 0 ? t.width : kHashCap;
  J->max_entries = cap;
}

extern "C" int crop_pairs_create(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                                 uint32_t n_items, int upper_only, const crop_interval* interval,
                                 void* stream, crop_pairs** job) {
  *job = nullptr;
  if (n_tx < 0 || n_items >= (1u << 31)) {
    crop_set_error(CROP_EINPUT, "need n_tx >= 0 and item ids < 2^31 (n_items=%u)", n_items);
    return CROP_EINPUT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  crop_pairs* J = new crop_pairs();
  J->offsets = offsets;
  J->items = items;
  J->n_tx = n_tx;
  J->n_items = n_items;
  J->upper = upper_only;
  J->filter = false;
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
    JCUDA(cudaMalloc(&J->d_terms, nn * sizeof(unsigned long long)));
    JCUDA(cudaMalloc(&J->d_maxlen, sizeof(unsigned int)));
    JCUDA(cudaMemsetAsync(J->d_terms, 0, nn * sizeof(unsigned long long), st));
    JCUDA(cudaMemsetAsync(J->d_maxlen, 0, sizeof(unsigned int), st));
    if (n_tx > 0 && n_items > 0) {
      auto kern = upper_only ? k_item_terms<true> : k_item_terms<false>;
      const uint32_t ns = std::min<uint32_t>(n_items, kStatSmemItems);
      JCUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kStatSmemItems * 4)));
      int64_t grid = std::max<int64_t>(2 * kNumSMs, (n_tx + 32767) / 32768);
      grid = std::min<int64_t>(grid, (n_tx + 15) / 16);
      if (grid < 1) grid = 1;
      kern<<<(int)grid, 512, ns * 4, st>>>(offsets, items, n_tx, n_items, J->d_terms, J->d_maxlen);
      JCUDA(cudaGetLastError());
    }
    std::vector<unsigned long long> terms(nn);
    unsigned int maxlen = 0;
    int64_t nnz = 0;
    JCUDA(cudaMemcpyAsync(terms.data(), J->d_terms, nn * 8, cudaMemcpyDeviceToHost, st));
    JCUDA(cudaMemcpyAsync(&maxlen, J->d_maxlen, 4, cudaMemcpyDeviceToHost, st));
    if (n_tx > 0) JCUDA(cudaMemcpyAsync(&nnz, offsets + n_tx, 8, cudaMemcpyDeviceToHost, st));
    JCUDA(cudaStreamSynchronize(st));
    if (maxlen > kMaxLen) {
      crop_set_error(CROP_EINPUT, "transaction of %u items exceeds the %u-item limit", maxlen, kMaxLen);
      rc = CROP_EINPUT;
      goto fail;
    }
    J->total_terms = 0;
    for (uint32_t i = 0; i < n_items; ++i) J->total_terms += terms[i];
    std::vector<uint32_t> item_tile;
    plan_tiles(J, terms, item_tile);
    const uint32_t nt = (uint32_t)J->tiles.size();
    JCUDA(cudaMalloc(&J->d_item_tile, nn * 4));
    JCUDA(cudaMalloc(&J->d_tiles, std::max<size_t>(1, nt) * sizeof(Tile)));
    JCUDA(cudaMalloc(&J->d_units, std::max<size_t>(1, J->units.size()) * sizeof(Unit)));
    JCUDA(cudaMalloc(&J->d_split, std::max<size_t>(1, J->split.size()) * 4));
    JCUDA(cudaMalloc(&J->d_tile_entries, std::max<size_t>(1, nt) * 4));
    JCUDA(cudaMalloc(&J->d_tile_ebase, std::max<size_t>(1, nt) * 8));
    JCUDA(cudaMalloc(&J->d_tile_cursor, std::max<size_t>(1, nt) * 8));
    JCUDA(cudaMalloc(&J->d_total_entries, 8));
    JCUDA(cudaMalloc(&J->d_unit_counter, 4));
    JCUDA(cudaMalloc(&J->d_overflow, 4));
    JCUDA(cudaMemsetAsync(J->d_overflow, 0, 4, st));
    if (n_items) JCUDA(cudaMemcpyAsync(J->d_item_tile, item_tile.data(), n_items * 4, cudaMemcpyHostToDevice, st));
    if (nt) JCUDA(cudaMemcpyAsync(J->d_tiles, J->tiles.data(), nt * sizeof(Tile), cudaMemcpyHostToDevice, st));
    if (!J->units.empty())
      JCUDA(cudaMemcpyAsync(J->d_units, J->units.data(), J->units.size() * sizeof(Unit), cudaMemcpyHostToDevice, st));
    if (!J->split.empty())
      JCUDA(cudaMemcpyAsync(J->d_split, J->split.data(), J->split.size() * 4, cudaMemcpyHostToDevice, st));
    if (J->n_slabs) JCUDA(cudaMalloc(&J->d_slabs, J->n_slabs * (size_t)kDenseCap * 4));
    // entry capacity: every entry has >= 1 term, and a run never spans more
    // positions than the transaction, so entries <= min(total terms, nnz*windows)
    // is loose; use terms bounded by nnz * max windows.
    uint64_t maxwin = 1;
    for (auto& t : J->tiles) maxwin = std::max<uint64_t>(maxwin, t.nwin);
    J->entry_cap = std::min<uint64_t>(J->total_terms, (uint64_t)nnz * maxwin);
    if (J->entry_cap >= (1ull << 32)) J->entry_cap = (1ull << 32) - 1;  // positions are 32-bit in smem
    JCUDA(cudaMalloc(&J->d_entries, std::max<uint64_t>(1, J->entry_cap) * sizeof(uint2)));
  }
#undef JCUDA
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
  if (n_tiles) *n_tiles = J->tiles.size();
  if (n_units) *n_units = J->units.size();
  return CROP_OK;
}

extern "C" int crop_pairs_run(crop_pairs* J, uint32_t* out_row, uint32_t* out_col,
                              uint32_t* out_count, uint64_t* d_n_entries, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t nt = (uint32_t)J->tiles.size();
  CROP_CUDA(cudaMemsetAsync(d_n_entries, 0, 8, st));
  if (nt == 0 || J->n_tx == 0) return CROP_OK;
  const bool up = J->upper != 0;
  // pass B1: entries per tile
  CROP_CUDA(cudaMemsetAsync(J->d_tile_entries, 0, nt * 4, st));
  {
    auto kern = up ? k_route_count<true> : k_route_count<false>;
    CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kTileSmem * 4)));
    const uint32_t ns = std::min(nt, kTileSmem);
    int grid = 2 * kNumSMs;
    kern<<<grid, kRouteThreads, ns * 4, st>>>(J->offsets, J->items, J->n_tx, J->d_item_tile,
                                              J->d_tiles, nt, J->d_tile_entries);
    CROP_LAUNCH_CHECK();
  }
  k_exclusive_scan_u32_to_u64<<<1, 1024, 0, st>>>(J->d_tile_entries, nt, J->d_tile_ebase,
                                                   J->d_total_entries);
  CROP_LAUNCH_CHECK();
  CROP_CUDA(cudaMemcpyAsync(J->d_tile_cursor, J->d_tile_ebase, nt * 8, cudaMemcpyDeviceToDevice, st));
  {
    auto kern = up ? k_route_write<true> : k_route_write<false>;
    CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kTileSmem * 4)));
    const uint32_t ns = std::min(nt, kTileSmem);
    int64_t grid = std::min<int64_t>(4 * kNumSMs, std::max<int64_t>(1, J->n_tx / 64));
    kern<<<(int)grid, kRouteThreads, ns * 4, st>>>(J->offsets, J->items, J->n_tx, J->d_item_tile,
                                                   J->d_tiles, nt, J->d_tile_cursor, J->d_entries,
                                                   J->entry_cap, J->d_overflow);
    CROP_LAUNCH_CHECK();
  }
  // count
  CROP_CUDA(cudaMemsetAsync(J->d_unit_counter, 0, 4, st));
  {
    CountArgs A{};
    A.offsets = J->offsets;
    A.items = J->items;
    A.tiles = J->d_tiles;
    A.units = J->d_units;
    A.n_units = (uint32_t)J->units.size();
    A.tile_ebase = J->d_tile_ebase;
    A.tile_entries = J->d_tile_entries;
    A.entries = J->d_entries;
    A.unit_counter = J->d_unit_counter;
    A.n_items = J->n_items;
    A.col_bits = J->col_bits;
    A.filter = J->filter;
    A.kappa = J->iv.kappa;
    A.start = J->iv.start;
    A.stop = J->iv.stop;
    A.h_row = J->iv.h_row;
    A.h_col = J->iv.h_col;
    A.out_row = out_row;
    A.out_col = out_col;
    A.out_count = out_count;
    A.out_n = (unsigned long long*)d_n_entries;
    A.slabs = J->d_slabs;
    void (*kern)(CountArgs);
    if (up) kern = J->filter ? k_count<true, true> : k_count<true, false>;
    else kern = J->filter ? k_count<false, true> : k_count<false, false>;
    CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCountSmem));
    int grid = std::min<int>(kNumSMs, (int)J->units.size());
    kern<<<grid, kCountThreads, kCountSmem, st>>>(A);
    CROP_LAUNCH_CHECK();
  }
  if (!J->split.empty()) {
    ReduceArgs R{};
    R.tiles = J->d_tiles;
    R.split_tiles = J->d_split;
    R.n_split = (uint32_t)J->split.size();
    R.slabs = J->d_slabs;
    R.n_items = J->n_items;
    R.out_row = out_row;
    R.out_col = out_col;
    R.out_count = out_count;
    R.out_n = (unsigned long long*)d_n_entries;
    const uint32_t chunks = (kDenseCap + kReduceChunk - 1) / kReduceChunk;
    auto kern = up ? k_slab_reduce<true> : k_slab_reduce<false>;
    kern<<<R.n_split * chunks, kReduceThreads, 0, st>>>(R);
    CROP_LAUNCH_CHECK();
  }
  return CROP_OK;
}

extern "C" void crop_pairs_destroy(crop_pairs* J) {
  if (!J) return;
  free_job(J);
  delete J;
}
