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
#include <algorithm>
#include <cstdint>

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
// still separate -- compact them (warp-aggregated claims)
__global__ void k_bt_compact(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                             const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                             uint32_t kappa, const BtState* __restrict__ st,
                             uint32_t* __restrict__ c_row, uint32_t* __restrict__ c_col,
                             unsigned long long* __restrict__ c_n, uint32_t* __restrict__ c_andor,
                             const uint16_t* __restrict__ bkt, uint16_t* __restrict__ c_bkt) {
  const uint64_t n = *d_n;
  const uint64_t n_round = (n + 31) & ~31ull;
  const int lane = threadIdx.x & 31;
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
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(c_n, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
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
