// bucket_topk.cu -- per-partition top-l select (the bounded Space-Saving regime).
//
// Replaces the per-bucket ranking of engine.finalize_summaries, i.e. the
// summary a bucket keeps when it holds more distinct entries than the
// Space-Saving capacity l (spacesaving.py:39-63): the
// bucket's top-l entries by (count desc, row asc, col asc), and the count of
// the l-th one (the summary minimum that bounds every absent entry).
//
// MSD radix select on the 96-bit rank key (~count, row, col), ascending,
// 8 bits per pass, all buckets at once:
//   k_bt_hist    per active bucket, a 256-bin histogram of the current digit
//                of the entries whose decided digits equal the bucket's
//                prefix (privatised in shared memory for kappa <= 32,
//                warp-aggregated global atomics otherwise)
//   k_bt_select  one warp per bucket: the digit holding the need-th smallest
//                key, appended to the prefix; the rank inside it carried on
//   k_bt_compact after the four count digits, the entries tied with their
//                bucket's threshold count -- the only ones the row / column
//                digits still separate -- are compacted; passes 4-11 read them
//   k_bt_mark    recorded[e] = key <= the bucket's threshold key (keys are
//                unique inside a bucket, so exactly l entries per full bucket)
// Pass 0 also yields each bucket's distinct count: buckets with fewer than l
// entries keep everything (bucket_min 0), buckets with exactly l are full.
// That flat form serves kappa <= 32 (histograms privatised per CTA); for
// 32 < kappa <= 2048 (c3: 1184) the entries of the full buckets are grouped
// into per-bucket segments and each bucket is selected by one CTA with its
// histogram in shared memory (k_bt_seg_*; CROP_BT_FLAT=1 forces the flat form).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

using namespace crop;

namespace {

constexpr int kBtThreads = 512;
constexpr uint32_t kBtSmemBuckets = 32;  // 32 KB of privatised histograms
constexpr uint32_t kBtSmemTotals = 8192;  // buckets counted in shared memory by the pre-pass

struct BtState {
  uint32_t key[3];   // decided digits of the threshold key (~count, row, col)
  uint32_t need;     // rank (1-based) of the threshold among the bucket's matching keys
  uint32_t total;    // distinct entries of the bucket (pass 0)
  uint32_t active;   // bucket holds >= l entries
};

__device__ __forceinline__ uint32_t bt_bucket(const uint32_t* h_row, const uint32_t* h_col,
                                              uint32_t kappa, uint32_t i, uint32_t j) {
  uint32_t b = h_row[i] + h_col[j];
  return b >= kappa ? b - kappa : b;
}

__device__ __forceinline__ uint32_t bt_word(uint32_t w, uint32_t c, uint32_t i, uint32_t j) {
  return w == 0 ? ~c : (w == 1 ? i : j);
}

// does the entry's key agree with the bucket's prefix on the digits decided
// before pass p (digit p is bits [24 - 8 (p % 4), +8) of word p / 4)?
__device__ __forceinline__ bool bt_matches(const BtState& s, uint32_t p, uint32_t c, uint32_t i,
                                           uint32_t j) {
  const uint32_t w = p >> 2, q = p & 3;
  for (uint32_t k = 0; k < w; ++k)
    if (bt_word(k, c, i, j) != s.key[k]) return false;
  if (q == 0) return true;
  const uint32_t sh = 32 - 8 * q;  // decided high bits of word w
  return (bt_word(w, c, i, j) >> sh) == (s.key[w] >> sh);
}

// andor = {AND of the 3 key words, OR of the 3 key words} over the entries
// (passes 0-3) or the candidates (passes 4-11): digit p is constant when the
// AND and the OR agree on its bits
__device__ __forceinline__ bool bt_constant_digit(const uint32_t* andor, uint32_t p) {
  const uint32_t w = p >> 2, sh = 24 - 8 * (p & 3);
  return (((andor[w] ^ andor[3 + w]) >> sh) & 0xFFu) == 0;
}

__device__ __forceinline__ void bt_andor_warp(uint32_t (&a)[3], uint32_t (&o)[3], uint32_t* out) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      a[k] &= __shfl_xor_sync(0xffffffffu, a[k], d);
      o[k] |= __shfl_xor_sync(0xffffffffu, o[k], d);
    }
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      atomicAnd(&out[k], a[k]);
      atomicOr(&out[3 + k], o[k]);
    }
}

// pre-pass: entries per bucket, and the AND / OR of the key words
__global__ void __launch_bounds__(kBtThreads)
    k_bt_pre(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
             const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
             const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col, uint32_t kappa,
             uint32_t* __restrict__ totals, uint32_t* __restrict__ andor,
             uint16_t* __restrict__ bkt) {
  __shared__ uint32_t s_tot[kBtSmemTotals];
  const bool priv = kappa <= kBtSmemTotals;
  if (priv) {
    for (uint32_t k = threadIdx.x; k < kappa; k += blockDim.x) s_tot[k] = 0;
    __syncthreads();
  }
  const uint64_t n = *d_n;
  const uint64_t n_round = (n + 31) & ~31ull;
  uint32_t a[3] = {~0u, ~0u, ~0u}, o[3] = {0u, 0u, 0u};
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_round;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = 0xFFFFFFFFu;
    if (e < n) {
      const uint32_t i = row[e], j = col[e], kc = ~count[e];
      b = bt_bucket(h_row, h_col, kappa, i, j);
      if (bkt) bkt[e] = (uint16_t)b;
      a[0] &= kc; a[1] &= i; a[2] &= j;
      o[0] |= kc; o[1] |= i; o[2] |= j;
    }
    if (priv && kappa >= 256) {
      if (b != 0xFFFFFFFFu) atomicAdd(&s_tot[b], 1u);
      continue;
    }
    const uint32_t grp = __match_any_sync(0xffffffffu, b);
    if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (int)(threadIdx.x & 31)) {
      if (priv) atomicAdd(&s_tot[b], (uint32_t)__popc(grp));
      else atomicAdd(&totals[b], (uint32_t)__popc(grp));
    }
  }
  bt_andor_warp(a, o, andor);
  if (priv) {
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < kappa; k += blockDim.x)
      if (s_tot[k]) atomicAdd(&totals[k], s_tot[k]);
  }
}

__global__ void k_bt_init(uint32_t kappa, uint32_t cap, const uint32_t* __restrict__ totals,
                          BtState* __restrict__ st) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kappa; b += gridDim.x * blockDim.x) {
    BtState s{};
    s.total = totals[b];
    s.active = s.total >= cap ? 1u : 0u;
    s.need = cap;
    st[b] = s;
  }
}

// CAND: the entries are the compacted tie candidates (row, col) of passes
// 4-11, whose count word equals their bucket's decided ~count by construction
template <bool CAND>
__global__ void __launch_bounds__(kBtThreads)
    k_bt_hist(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
              const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
              const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
              uint32_t kappa, const BtState* __restrict__ st, uint32_t p,
              uint32_t* __restrict__ hist, const uint32_t* __restrict__ andor,
              const uint16_t* __restrict__ bkt) {
  // a digit every (candidate) key shares is decided without a pass
  if (bt_constant_digit(andor, p)) return;
  __shared__ uint32_t s_hist[kBtSmemBuckets * 256];
  const bool priv = kappa <= kBtSmemBuckets;
  if (priv) {
    for (uint32_t k = threadIdx.x; k < kappa * 256; k += blockDim.x) s_hist[k] = 0;
    __syncthreads();
  }
  const uint64_t n = *d_n;
  const uint32_t w = p >> 2, sh = 24 - 8 * (p & 3);
  const uint64_t n_round = (n + 31) & ~31ull;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_round;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t slot = 0xFFFFFFFFu;
    if (e < n) {
      const uint32_t i = row[e], j = col[e];
      const uint32_t b = bkt ? bkt[e] : bt_bucket(h_row, h_col, kappa, i, j);
      const BtState& s = st[b];
      const uint32_t c = CAND ? ~s.key[0] : count[e];
      if (s.active && bt_matches(s, p, c, i, j))
        slot = b * 256 + ((bt_word(w, c, i, j) >> sh) & 0xFFu);
    }
    // equal (bucket, digit) slots aggregate inside the warp first
    const uint32_t grp = __match_any_sync(0xffffffffu, slot);
    if (slot != 0xFFFFFFFFu && (__ffs(grp) - 1) == (int)(threadIdx.x & 31)) {
      if (priv) atomicAdd(&s_hist[slot], (uint32_t)__popc(grp));
      else atomicAdd(&hist[slot], (uint32_t)__popc(grp));
    }
  }
  if (priv) {
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < kappa * 256; k += blockDim.x)
      if (s_hist[k]) atomicAdd(&hist[k], s_hist[k]);
  }
}

// one warp per bucket: pick the digit of the need-th smallest matching key
__global__ void k_bt_select(uint32_t kappa, uint32_t p, BtState* __restrict__ st,
                            uint32_t* __restrict__ hist, const uint32_t* __restrict__ andor) {
  const uint32_t b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (b >= kappa) return;
  BtState& s = st[b];
  if (bt_constant_digit(andor, p)) {
    // every key shares this digit: append it, the rank is unchanged
    const uint32_t w = p >> 2, sh = 24 - 8 * (p & 3);
    if (lane == 0 && s.active) s.key[w] |= ((andor[w] >> sh) & 0xFFu) << sh;
    return;
  }
  uint32_t* h = hist + (uint64_t)b * 256;
  uint32_t v[8], sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = h[lane * 8 + k];
    sum += v[k];
  }
  const bool active = s.active != 0;
  const uint32_t need = s.need;
  // exclusive prefix of the lanes' 8-bin sums
  uint32_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += u;
  }
  const uint32_t excl = incl - sum;
  if (active && excl < need && need <= incl) {
    uint32_t c = excl, dg = 0, before = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (c < need && need <= c + v[k]) {
        dg = lane * 8 + k;
        before = c;
      }
      c += v[k];
    }
    const uint32_t w = p >> 2, sh = 24 - 8 * (p & 3);
    s.key[w] |= dg << sh;
    s.need = need - before;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) h[lane * 8 + k] = 0;
}

// after the count digits: the entries whose count equals their full
// bucket's threshold count are the only ones the row / column digits can
// still separate -- compact them (one output claim per block and step)
__global__ void k_bt_compact(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                             const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                             uint32_t kappa, const BtState* __restrict__ st,
                             uint32_t* __restrict__ c_row, uint32_t* __restrict__ c_col,
                             unsigned long long* __restrict__ c_n, uint32_t* __restrict__ c_andor,
                             const uint16_t* __restrict__ bkt, uint16_t* __restrict__ c_bkt) {
  const uint64_t n = *d_n;
  // uniform trip count per block: one output claim per block and step
  const uint64_t n_round = (n + blockDim.x - 1) / blockDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t s_wcnt[32];
  __shared__ unsigned long long s_base;
  // candidates' key words 1-2 (word 0 is each bucket's decided ~count: its
  // digits are never examined again, AND = OR = 0 marks them constant)
  uint32_t a[3] = {0u, ~0u, ~0u}, o[3] = {0u, 0u, 0u};
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_round;
       e += (uint64_t)gridDim.x * blockDim.x) {
    bool keep = false;
    uint32_t i = 0, j = 0, b = 0;
    if (e < n) {
      i = row[e];
      j = col[e];
      b = bkt ? bkt[e] : bt_bucket(h_row, h_col, kappa, i, j);
      const BtState& s = st[b];
      keep = s.active && ~count[e] == s.key[0];
    }
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_wcnt[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      const uint32_t c = lane < (int)(blockDim.x >> 5) ? s_wcnt[lane] : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long bb = 0;
      if (lane == 0 && tot) bb = atomicAdd(c_n, (unsigned long long)tot);
      bb = __shfl_sync(0xffffffffu, bb, 0);
      if (lane == 0) s_base = bb;
      s_wcnt[lane] = incl - c;
    }
    __syncthreads();
    const unsigned long long base = s_base + s_wcnt[warp];
    __syncthreads();  // s_wcnt / s_base are rewritten by the next step
    if (keep) {
      const uint64_t q = base + __popc(m & ((1u << lane) - 1u));
      c_row[q] = i;
      c_col[q] = j;
      if (c_bkt) c_bkt[q] = (uint16_t)b;
      a[1] &= i; a[2] &= j;
      o[1] |= i; o[2] |= j;
    }
  }
  bt_andor_warp(a, o, c_andor);
}

__global__ void k_bt_mark(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                          const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                          uint32_t kappa, const BtState* __restrict__ st,
                          uint8_t* __restrict__ recorded, const uint16_t* __restrict__ bkt) {
  const uint64_t n = *d_n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = row[e], j = col[e], c = count[e];
    const BtState& s = st[bkt ? bkt[e] : bt_bucket(h_row, h_col, kappa, i, j)];
    bool keep = true;
    if (s.active) {
      const uint32_t k0 = ~c;
      keep = k0 < s.key[0] || (k0 == s.key[0] && (i < s.key[1] || (i == s.key[1] && j <= s.key[2])));
    }
    recorded[e] = keep ? 1 : 0;
  }
}

// k_bt_mark over 16-byte aligned columns with the bucket ids cached: four
// entries per thread per step (uint4 loads, one 4-byte store of flags)
__device__ __forceinline__ uint32_t bt_keep(const BtState& s, uint32_t c, uint32_t i, uint32_t j) {
  if (!s.active) return 1u;
  const uint32_t k0 = ~c;
  return (k0 < s.key[0] || (k0 == s.key[0] && (i < s.key[1] || (i == s.key[1] && j <= s.key[2])))) ? 1u : 0u;
}

__global__ void k_bt_mark4(const uint4* __restrict__ row, const uint4* __restrict__ col,
                           const uint4* __restrict__ count, const uint64_t* __restrict__ d_n,
                           const BtState* __restrict__ st, uint32_t* __restrict__ recorded,
                           const uint2* __restrict__ bkt) {
  const uint64_t n = *d_n, nq = n / 4;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 i = __ldcs(row + q), j = __ldcs(col + q), c = __ldcs(count + q);
    const uint2 bb = __ldcs(bkt + q);
    const uint32_t f = bt_keep(st[bb.x & 0xFFFFu], c.x, i.x, j.x) |
                       bt_keep(st[bb.x >> 16], c.y, i.y, j.y) << 8 |
                       bt_keep(st[bb.y & 0xFFFFu], c.z, i.z, j.z) << 16 |
                       bt_keep(st[bb.y >> 16], c.w, i.w, j.w) << 24;
    __stcs(recorded + q, f);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const uint64_t e = nq * 4 + threadIdx.x;
    const uint32_t* r = reinterpret_cast<const uint32_t*>(row);
    const uint32_t* cl = reinterpret_cast<const uint32_t*>(col);
    const uint32_t* ct = reinterpret_cast<const uint32_t*>(count);
    const uint16_t* bk = reinterpret_cast<const uint16_t*>(bkt);
    reinterpret_cast<uint8_t*>(recorded)[e] = (uint8_t)bt_keep(st[bk[e]], ct[e], r[e], cl[e]);
  }
}

// ---------------------------------------------------------------- segmented
// kappa in (32, 2048]: the per-pass global histograms of the flat path take
// one L2 atomic per entry (hot (bucket, digit) slots when most counts tie),
// so the active buckets' entries are first grouped into one contiguous
// segment per bucket and each bucket is then selected by one CTA with its
// histogram in shared memory:
//   k_bt_seg_scan    segment offsets of the active buckets (one block)
//   k_bt_scatter     per CTA, a contiguous range of entries: count per
//                    bucket in shared memory, one global claim per touched
//                    bucket, then write (~count, row, col) into the claims
//   k_bt_seg_select  one CTA per active bucket: MSD radix select of the
//                    96-bit key over its segment; once the keys matching
//                    the decided prefix fit in shared memory they are staged
//                    there by the next pass and later passes read only them
constexpr uint32_t kBtSegMaxKappa = 2048;
constexpr int kBtSegThreads = 512;
constexpr uint32_t kBtSegStage = 4096;  // staged keys (3 x u32: 48 KB)

__global__ void __launch_bounds__(1024) k_bt_seg_scan(uint32_t kappa, const BtState* __restrict__ st,
                                                      uint32_t* __restrict__ seg_off,
                                                      uint32_t* __restrict__ seg_cur,
                                                      uint32_t* __restrict__ grp_cur,
                                                      uint64_t* __restrict__ n_active) {
  __shared__ uint32_t s_part[1024];
  const uint32_t per = (kappa + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(kappa, threadIdx.x * per), hi = min(kappa, lo + per);
  uint32_t sum = 0;
  for (uint32_t b = lo; b < hi; ++b) sum += st[b].active ? st[b].total : 0u;
  s_part[threadIdx.x] = sum;
  __syncthreads();
  for (uint32_t d = 1; d < blockDim.x; d <<= 1) {
    const uint32_t v = threadIdx.x >= d ? s_part[threadIdx.x - d] : 0u;
    __syncthreads();
    s_part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = s_part[threadIdx.x] - sum;
  for (uint32_t b = lo; b < hi; ++b) {
    seg_off[b] = run;
    seg_cur[b] = run;
    if ((b & 31) == 0) grp_cur[b >> 5] = run;  // group g = buckets [32 g, 32 g + 32)
    run += st[b].active ? st[b].total : 0u;
  }
  if (threadIdx.x == blockDim.x - 1) *n_active = s_part[threadIdx.x];
}

// tiles of kScTile entries are grouped by bucket in shared memory first, so
// each bucket's entries of a tile leave as one contiguous run (consecutive
// lanes, consecutive addresses) that continues the previous tile's run
constexpr int kScThreads = 512;  // two CTAs per SM: one loads while the other groups
constexpr uint32_t kScPer = 8;
constexpr uint32_t kScTile = kScThreads * kScPer;
constexpr size_t kScSmem = (size_t)(2 * kBtSegMaxKappa + 32 + kBtSegMaxKappa / 32 + 3 * kScTile) * 4 +
                           (size_t)kScTile * 2;

// Grouping key = bucket >> shift. With many buckets the scatter runs twice
// (shift 5, then 0 over the output of the first) so every tile's runs stay
// long: a tile of 8,192 entries over 1,184 buckets leaves runs of ~7 entries
// (partial sectors, ~2x DRAM write amplification), over 37 groups or the 32
// buckets of one group runs of ~250.
__global__ void __launch_bounds__(kScThreads, 2)
    k_bt_scatter(const uint32_t* __restrict__ in0, const uint32_t* __restrict__ row,
                 const uint32_t* __restrict__ col, const uint64_t* __restrict__ d_n,
                 const uint16_t* __restrict__ bkt, bool invert, uint32_t shift, uint32_t kappa,
                 const BtState* __restrict__ st, uint32_t* __restrict__ seg_cur,
                 uint32_t* __restrict__ s_k0, uint32_t* __restrict__ s_row, uint32_t* __restrict__ s_col,
                 uint16_t* __restrict__ out_bkt) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* s_cur = sm;                            // [nkeys] this CTA's write cursor per key
  uint32_t* s_cnt = s_cur + kBtSegMaxKappa;        // [nkeys + 1] tile counts -> offsets
  uint32_t* s_act = s_cnt + kBtSegMaxKappa + 32;   // [kappa / 32] active-bucket bits
  uint32_t* stg = s_act + kBtSegMaxKappa / 32;     // [3][kScTile] staged keys
  uint16_t* s_b = reinterpret_cast<uint16_t*>(stg + 3 * kScTile);  // [kScTile] their buckets
  __shared__ uint32_t s_warp[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nkeys = (kappa + (1u << shift) - 1) >> shift;
  for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x) s_cur[k] = 0;
  for (uint32_t k = threadIdx.x; k < (kappa + 31) / 32; k += blockDim.x) {
    uint32_t bits = 0;
    for (uint32_t q = 0; q < 32 && k * 32 + q < kappa; ++q) bits |= (st[k * 32 + q].active ? 1u : 0u) << q;
    s_act[k] = bits;
  }
  __syncthreads();
  auto active = [&](uint32_t b) { return b < kappa && ((s_act[b >> 5] >> (b & 31)) & 1u); };
  const uint64_t n = *d_n;
  const uint64_t per = (((n + gridDim.x - 1) / gridDim.x) + 31) & ~31ull;
  const uint64_t lo = min(n, blockIdx.x * per), hi = min(n, lo + per);
  // 1: this CTA's entries per key, one global claim per key
  for (uint64_t e0 = lo; e0 < hi; e0 += kScTile) {
    uint32_t bb[kScPer];
#pragma unroll
    for (uint32_t u = 0; u < kScPer; ++u) {
      const uint64_t e = e0 + u * blockDim.x + threadIdx.x;
      bb[u] = e < hi ? bkt[e] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (uint32_t u = 0; u < kScPer; ++u)
      if (active(bb[u])) atomicAdd(&s_cur[bb[u] >> shift], 1u);
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x) {
    const uint32_t c = s_cur[k];
    if (c) s_cur[k] = atomicAdd(&seg_cur[k], c);
  }
  // 2: per tile, group by key in shared memory, then write the runs
  const uint32_t per_t = (nkeys + blockDim.x - 1) / blockDim.x;  // scan elements per thread (<= 4)
  for (uint64_t e0 = lo; e0 < hi; e0 += kScTile) {
    for (uint32_t k = threadIdx.x; k <= nkeys; k += blockDim.x) s_cnt[k] = 0;
    __syncthreads();
    uint32_t bb[kScPer], kc[kScPer], ii[kScPer], jj[kScPer], rk[kScPer];
#pragma unroll
    for (uint32_t u = 0; u < kScPer; ++u) {
      const uint64_t e = e0 + u * blockDim.x + threadIdx.x;
      const bool ok = e < hi;
      bb[u] = ok ? bkt[e] : 0xFFFFFFFFu;
      kc[u] = ok ? __ldcs(in0 + e) : 0u;
      if (invert) kc[u] = ~kc[u];
      ii[u] = ok ? __ldcs(row + e) : 0u;
      jj[u] = ok ? __ldcs(col + e) : 0u;
    }
#pragma unroll
    for (uint32_t u = 0; u < kScPer; ++u) {
      if (!active(bb[u])) bb[u] = 0xFFFFFFFFu;
      rk[u] = bb[u] != 0xFFFFFFFFu ? atomicAdd(&s_cnt[bb[u] >> shift], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of s_cnt[0, nkeys) in place; s_cnt[nkeys] = tile total
    {
      const uint32_t b0 = threadIdx.x * per_t;
      uint32_t v[4] = {0u, 0u, 0u, 0u}, sum = 0;
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k)
        if (k < per_t && b0 + k < nkeys) {
          v[k] = s_cnt[b0 + k];
          sum += v[k];
        }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      if (lane == 31) s_warp[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const uint32_t wv = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
        uint32_t wi = wv;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
          if (lane >= d) wi += t;
        }
        s_warp[lane] = wi - wv;
        if (lane == 31) s_cnt[nkeys] = wi;
      }
      __syncthreads();
      uint32_t run = s_warp[warp] + incl - sum;
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k)
        if (k < per_t && b0 + k < nkeys) {
          s_cnt[b0 + k] = run;
          run += v[k];
        }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t u = 0; u < kScPer; ++u)
      if (bb[u] != 0xFFFFFFFFu) {
        const uint32_t t = s_cnt[bb[u] >> shift] + rk[u];
        stg[t] = kc[u];
        stg[kScTile + t] = ii[u];
        stg[2 * kScTile + t] = jj[u];
        s_b[t] = (uint16_t)bb[u];
      }
    __syncthreads();
    const uint32_t total = s_cnt[nkeys];
    for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
      const uint32_t bf = s_b[t], k = bf >> shift;
      const uint32_t dst = s_cur[k] + (t - s_cnt[k]);
      s_k0[dst] = stg[t];
      s_row[dst] = stg[kScTile + t];
      s_col[dst] = stg[2 * kScTile + t];
      if (out_bkt) out_bkt[dst] = (uint16_t)bf;
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nkeys; k += blockDim.x) {
      const uint32_t nb = k + 1 < nkeys ? s_cnt[k + 1] : total;
      s_cur[k] += nb - s_cnt[k];
    }
    __syncthreads();
  }
}

// does key word set kw agree with the prefix on the digits decided before p?
// (register arrays indexed by constants only: no local memory)
__device__ __forceinline__ uint32_t bt_pick(const uint32_t (&v)[3], uint32_t w) {
  return w == 0 ? v[0] : (w == 1 ? v[1] : v[2]);
}

__device__ __forceinline__ bool bt_prefix_match(const uint32_t (&kw)[3], const uint32_t (&key)[3],
                                                uint32_t p) {
  const uint32_t w = p >> 2, q = p & 3;
  if (w > 0 && kw[0] != key[0]) return false;
  if (w > 1 && kw[1] != key[1]) return false;
  if (q == 0) return true;
  const uint32_t sh = 32 - 8 * q;
  return (bt_pick(kw, w) >> sh) == (bt_pick(key, w) >> sh);
}

// one histogram add per lane; a warp whose lanes all hold the same digit
// (the common case when most counts tie) adds once
__device__ __forceinline__ void bt_hist_add(uint32_t* hist, uint32_t d) {
  const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
  if (__all_sync(0xffffffffu, d == d0)) {
    if ((threadIdx.x & 31) == 0 && d0 < 256) atomicAdd(&hist[d0], 32u);
  } else if (d < 256) {
    atomicAdd(&hist[d], 1u);
  }
}

// Per pass, the keys matching the decided prefix are read from the current
// source: the bucket's segment, a compacted copy of the matching keys in the
// scratch segment (written by the pass after the matches fell to a quarter
// of the source; the two alternate), or shared memory (staged once they fit)
__global__ void __launch_bounds__(kBtSegThreads)
    k_bt_seg_select(uint32_t* __restrict__ seg_a, uint32_t* __restrict__ seg_b, uint32_t cap,
                    const uint32_t* __restrict__ seg_off, BtState* __restrict__ st,
                    const uint32_t* __restrict__ andor) {
  extern __shared__ __align__(16) uint32_t stage[];  // [3][kBtSegStage]
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_sel[3];
  __shared__ uint32_t s_n;
  const uint32_t b = blockIdx.x;
  const BtState s = st[b];
  if (!s.active) return;
  const uint32_t off = seg_off[b], m = s.total;
  // key word k of source entry e: src + k * cap + e (three u32 arrays)
  uint32_t* src = seg_a + off;
  uint32_t* dst = seg_b + off;
  uint32_t key[3] = {0u, 0u, 0u};
  uint32_t need = s.need, match = m, msrc = m, ns = 0;
  bool staged = false;
  const int lane = threadIdx.x & 31;
  for (uint32_t p = 0; p < 12; ++p) {
    const uint32_t w = p >> 2, sh = 24 - 8 * (p & 3);
    if (bt_constant_digit(andor, p)) {
      const uint32_t dg = ((andor[w] >> sh) & 0xFFu) << sh;
      key[0] |= w == 0 ? dg : 0u;
      key[1] |= w == 1 ? dg : 0u;
      key[2] |= w == 2 ? dg : 0u;
      continue;
    }
    for (uint32_t k = threadIdx.x; k < 256; k += blockDim.x) hist[k] = 0;
    if (threadIdx.x == 0) s_n = 0;
    const bool stage_now = !staged && match <= kBtSegStage;
    const bool compact_now = !staged && !stage_now && match <= msrc / 4;
    __syncthreads();
    if (staged) {
      for (uint32_t e0 = 0; e0 < ns; e0 += blockDim.x) {
        const uint32_t e = e0 + threadIdx.x;
        uint32_t d = 0xFFFFFFFFu;
        if (e < ns) {
          const uint32_t kw[3] = {stage[e], stage[kBtSegStage + e], stage[2 * kBtSegStage + e]};
          if (bt_prefix_match(kw, key, p)) d = (bt_pick(kw, w) >> sh) & 0xFFu;
        }
        bt_hist_add(hist, d);
      }
    } else {
      // U entries per thread per step, all loads issued before any is used;
      // the words after w are loaded only for matching keys that move
      constexpr uint32_t U = 4;
      for (uint32_t e0 = 0; e0 < msrc; e0 += U * blockDim.x) {
        uint32_t kw[U][3];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          const bool ok = e < msrc;
          kw[u][0] = ok ? __ldcs(src + e) : 0u;
          kw[u][1] = ok && w >= 1 ? __ldcs(src + (size_t)cap + e) : 0u;
          kw[u][2] = ok && w >= 2 ? __ldcs(src + 2 * (size_t)cap + e) : 0u;
        }
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) {
          const uint32_t e = e0 + u * blockDim.x + threadIdx.x;
          uint32_t d = 0xFFFFFFFFu;
          if (e < msrc && bt_prefix_match(kw[u], key, p)) {
            d = (bt_pick(kw[u], w) >> sh) & 0xFFu;
            if (stage_now || compact_now) {
              if (w < 1) kw[u][1] = __ldcs(src + (size_t)cap + e);
              if (w < 2) kw[u][2] = __ldcs(src + 2 * (size_t)cap + e);
              const uint32_t q = atomicAdd(&s_n, 1u);
              if (stage_now) {
                stage[q] = kw[u][0];
                stage[kBtSegStage + q] = kw[u][1];
                stage[2 * kBtSegStage + q] = kw[u][2];
              } else {
                dst[q] = kw[u][0];
                dst[(size_t)cap + q] = kw[u][1];
                dst[2 * (size_t)cap + q] = kw[u][2];
              }
            }
          }
          bt_hist_add(hist, d);
        }
      }
    }
    __syncthreads();
    if (stage_now) {
      staged = true;
      ns = s_n;
    } else if (compact_now) {
      uint32_t* t = src;
      src = dst;
      dst = t;
      msrc = s_n;
    }
    if (threadIdx.x < 32) {
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = hist[lane * 8 + k];
        sum += v[k];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += u;
      }
      const uint32_t excl = incl - sum;
      if (excl < need && need <= incl) {
        uint32_t c = excl;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (c < need && need <= c + v[k]) {
            s_sel[0] = lane * 8 + k;
            s_sel[1] = c;
            s_sel[2] = v[k];
          }
          c += v[k];
        }
      }
    }
    __syncthreads();
    const uint32_t dg = s_sel[0] << sh;
    key[0] |= w == 0 ? dg : 0u;
    key[1] |= w == 1 ? dg : 0u;
    key[2] |= w == 2 ? dg : 0u;
    need -= s_sel[1];
    match = s_sel[2];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st[b].key[0] = key[0];
    st[b].key[1] = key[1];
    st[b].key[2] = key[2];
    st[b].need = need;
  }
}

__global__ void k_bt_out(uint32_t kappa, const BtState* __restrict__ st, uint32_t* __restrict__ bucket_min,
                         uint32_t* __restrict__ bucket_total) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kappa; b += gridDim.x * blockDim.x) {
    bucket_min[b] = st[b].active ? ~st[b].key[0] : 0u;
    if (bucket_total) bucket_total[b] = st[b].total;
  }
}

}  // namespace

extern "C" int crop_bucket_topk(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                                const uint64_t* d_n_entries, uint64_t n_capacity,
                                const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                                uint32_t capacity, uint8_t* recorded, uint32_t* bucket_min,
                                uint32_t* bucket_total, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (kappa == 0 || capacity == 0) {
    crop_set_error(CROP_ECONFIG, "bucket top-l needs kappa >= 1 and capacity >= 1");
    return CROP_ECONFIG;
  }
  if (int rc = crop_pool_setup()) return rc;
  BtState* d_st = nullptr;
  uint32_t* d_hist = nullptr;
  uint32_t* d_misc = nullptr;  // totals[kappa], andor[6] (entries), andor[6] (candidates)
  CROP_CUDA(cudaMallocAsync(&d_st, (size_t)kappa * sizeof(BtState), st));
  CROP_CUDA(cudaMallocAsync(&d_hist, (size_t)kappa * 256 * 4, st));
  CROP_CUDA(cudaMallocAsync(&d_misc, ((size_t)kappa + 12) * 4, st));
  CROP_CUDA(cudaMemsetAsync(d_hist, 0, (size_t)kappa * 256 * 4, st));
  uint32_t* d_tot = d_misc;
  uint32_t* d_ao = d_misc + kappa;       // AND (3 words, start all-ones), OR (3 words)
  uint32_t* d_ao_c = d_misc + kappa + 6;
  CROP_CUDA(cudaMemsetAsync(d_tot, 0, (size_t)kappa * 4, st));
  CROP_CUDA(cudaMemsetAsync(d_ao, 0xFF, 12, st));
  CROP_CUDA(cudaMemsetAsync(d_ao + 3, 0, 12, st));
  CROP_CUDA(cudaMemsetAsync(d_ao_c, 0xFF, 12, st));
  CROP_CUDA(cudaMemsetAsync(d_ao_c + 3, 0, 12, st));
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n_capacity + kBtThreads - 1) / kBtThreads,
                                                                 (uint64_t)kNumSMs * 4));
  const int sel_grid = (int)((kappa + 7) / 8);
  // segmented select (see k_bt_seg_select) when the buckets are too many
  // for privatised histograms but few enough for per-CTA bucket counters
  const bool segmented = kappa > kBtSmemBuckets && kappa <= kBtSegMaxKappa &&
                         n_capacity < (1ull << 32) && !getenv("CROP_BT_FLAT");
  if (segmented) {
    uint16_t* bkt = nullptr;
    uint32_t *seg = nullptr, *g_k0 = nullptr;
    // the segments hold the entries (not the capacity): one 8-byte read-back
    uint64_t n_host = 0;
    CROP_CUDA(cudaMemcpyAsync(&n_host, d_n_entries, 8, cudaMemcpyDeviceToHost, st));
    CROP_CUDA(cudaStreamSynchronize(st));
    if (n_host > n_capacity) {
      crop_set_error(CROP_EINPUT, "%llu entries exceed their arrays' capacity %llu",
                     (unsigned long long)n_host, (unsigned long long)n_capacity);
      cudaFreeAsync(d_st, st);
      cudaFreeAsync(d_hist, st);
      cudaFreeAsync(d_misc, st);
      return CROP_EINPUT;
    }
    const uint64_t cap1 = std::max<uint64_t>(n_host, 1);
    CROP_CUDA(cudaMallocAsync(&bkt, cap1 * 2, st));
    // offsets, cursors, group cursors, the active entry count
    CROP_CUDA(cudaMallocAsync(&seg, ((size_t)2 * kappa + kBtSegMaxKappa / 32 + 4) * 4, st));
    // segments + scratch segments (+ the group pass's 16-bit buckets)
    CROP_CUDA(cudaMallocAsync(&g_k0, cap1 * 26, st));
    uint32_t* g_row = g_k0 + cap1;
    uint32_t* g_col = g_row + cap1;
    k_bt_pre<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_tot, d_ao,
                                           bkt);
    CROP_LAUNCH_CHECK();
    k_bt_init<<<(kappa + 255) / 256, 256, 0, st>>>(kappa, capacity, d_tot, d_st);
    CROP_LAUNCH_CHECK();
    uint32_t* grp_cur = seg + 2 * kappa;
    uint64_t* n_act = reinterpret_cast<uint64_t*>(seg + 2 * kappa + kBtSegMaxKappa / 32 + 2);
    k_bt_seg_scan<<<1, 1024, 0, st>>>(kappa, d_st, seg, seg + kappa, grp_cur, n_act);
    CROP_LAUNCH_CHECK();
    CROP_CUDA(cudaFuncSetAttribute(k_bt_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScSmem));
    uint32_t* g_scr = g_k0 + 3 * cap1;  // the select's scratch segments
    if (kappa > 256) {
      // by group of 32 buckets into the scratch (with the buckets), then by
      // bucket into the segments
      uint16_t* bkt2 = reinterpret_cast<uint16_t*>(g_scr + 3 * cap1);
      k_bt_scatter<<<kNumSMs * 2, kScThreads, kScSmem, st>>>(count, row, col, d_n_entries, bkt, true, 5, kappa,
                                                         d_st, grp_cur, g_scr, g_scr + cap1,
                                                         g_scr + 2 * cap1, bkt2);
      CROP_LAUNCH_CHECK();
      k_bt_scatter<<<kNumSMs * 2, kScThreads, kScSmem, st>>>(g_scr, g_scr + cap1, g_scr + 2 * cap1, n_act, bkt2,
                                                         false, 0, kappa, d_st, seg + kappa, g_k0, g_row,
                                                         g_col, nullptr);
    } else {
      k_bt_scatter<<<kNumSMs * 2, kScThreads, kScSmem, st>>>(count, row, col, d_n_entries, bkt, true, 0, kappa,
                                                         d_st, seg + kappa, g_k0, g_row, g_col, nullptr);
    }
    CROP_LAUNCH_CHECK();
    const size_t smem = (size_t)kBtSegStage * 12;
    CROP_CUDA(cudaFuncSetAttribute(k_bt_seg_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bt_seg_select<<<kappa, kBtSegThreads, smem, st>>>(g_k0, g_k0 + 3 * cap1, (uint32_t)cap1, seg, d_st,
                                                         d_ao);
    CROP_LAUNCH_CHECK();
    cudaFreeAsync(g_k0, st);
    cudaFreeAsync(seg, st);
    if (recorded) {
      auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
      if (al16(row) && al16(col) && al16(count) && al16(recorded)) {
        k_bt_mark4<<<kNumSMs * 8, 256, 0, st>>>(
            reinterpret_cast<const uint4*>(row), reinterpret_cast<const uint4*>(col),
            reinterpret_cast<const uint4*>(count), d_n_entries, d_st, reinterpret_cast<uint32_t*>(recorded),
            reinterpret_cast<const uint2*>(bkt));
      } else {
        k_bt_mark<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_st,
                                                recorded, bkt);
      }
      CROP_LAUNCH_CHECK();
    }
    k_bt_out<<<(kappa + 255) / 256, 256, 0, st>>>(kappa, d_st, bucket_min, bucket_total);
    CROP_LAUNCH_CHECK();
    cudaFreeAsync(bkt, st);
    cudaFreeAsync(d_hist, st);
    cudaFreeAsync(d_misc, st);
    cudaFreeAsync(d_st, st);
    crop_count_launches((recorded ? 7 : 6) + (kappa > 256 ? 1 : 0));
    return CROP_OK;
  }
  // count digits over all entries, then the row / column digits over the
  // compacted ties (entries whose count equals the bucket's threshold)
  uint32_t *c_row = nullptr, *c_col = nullptr;
  unsigned long long* c_n = nullptr;
  CROP_CUDA(cudaMallocAsync(&c_row, std::max<uint64_t>(n_capacity, 1) * 4, st));
  CROP_CUDA(cudaMallocAsync(&c_col, std::max<uint64_t>(n_capacity, 1) * 4, st));
  CROP_CUDA(cudaMallocAsync(&c_n, 8, st));
  CROP_CUDA(cudaMemsetAsync(c_n, 0, 8, st));
  // 16-bit bucket ids of the entries and candidates (kappa <= 65,536): one
  // hash-table gather per entry instead of one per pass
  uint16_t *bkt = nullptr, *c_bkt = nullptr;
  if (kappa <= 65536) {
    CROP_CUDA(cudaMallocAsync(&bkt, std::max<uint64_t>(n_capacity, 1) * 2, st));
    CROP_CUDA(cudaMallocAsync(&c_bkt, std::max<uint64_t>(n_capacity, 1) * 2, st));
  }
  k_bt_pre<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_tot, d_ao,
                                         bkt);
  CROP_LAUNCH_CHECK();
  k_bt_init<<<(kappa + 255) / 256, 256, 0, st>>>(kappa, capacity, d_tot, d_st);
  CROP_LAUNCH_CHECK();
  for (uint32_t p = 0; p < 12; ++p) {
    const uint32_t* ao = p < 4 ? d_ao : d_ao_c;
    if (p < 4) {
      k_bt_hist<false><<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa,
                                                     d_st, p, d_hist, ao, bkt);
    } else {
      if (p == 4) {
        k_bt_compact<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_st,
                                                   c_row, c_col, c_n, d_ao_c, bkt, c_bkt);
        CROP_LAUNCH_CHECK();
      }
      k_bt_hist<true><<<grid, kBtThreads, 0, st>>>(c_row, c_col, nullptr,
                                                    reinterpret_cast<const uint64_t*>(c_n), h_row, h_col,
                                                    kappa, d_st, p, d_hist, ao, c_bkt);
    }
    CROP_LAUNCH_CHECK();
    k_bt_select<<<sel_grid, 256, 0, st>>>(kappa, p, d_st, d_hist, ao);
    CROP_LAUNCH_CHECK();
  }
  cudaFreeAsync(c_row, st);
  cudaFreeAsync(c_col, st);
  cudaFreeAsync(c_n, st);
  if (recorded) {
    k_bt_mark<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_st,
                                            recorded, bkt);
    CROP_LAUNCH_CHECK();
  }
  k_bt_out<<<(kappa + 255) / 256, 256, 0, st>>>(kappa, d_st, bucket_min, bucket_total);
  CROP_LAUNCH_CHECK();
  cudaFreeAsync(d_hist, st);
  cudaFreeAsync(d_misc, st);
  if (bkt) cudaFreeAsync(bkt, st);
  if (c_bkt) cudaFreeAsync(c_bkt, st);
  cudaFreeAsync(d_st, st);
  crop_count_launches(29);
  return CROP_OK;
}
