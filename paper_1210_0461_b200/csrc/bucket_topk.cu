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

__global__ void __launch_bounds__(kBtThreads)
    k_bt_hist(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
              const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
              const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
              uint32_t kappa, const BtState* __restrict__ st, uint32_t p,
              uint32_t* __restrict__ hist) {
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
      const uint32_t i = row[e], j = col[e], c = count[e];
      const uint32_t b = bt_bucket(h_row, h_col, kappa, i, j);
      const BtState& s = st[b];
      if (p == 0 || (s.active && bt_matches(s, p, c, i, j)))
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
__global__ void k_bt_select(uint32_t kappa, uint32_t cap, uint32_t p, BtState* __restrict__ st,
                            uint32_t* __restrict__ hist) {
  const uint32_t b = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (b >= kappa) return;
  BtState& s = st[b];
  uint32_t* h = hist + (uint64_t)b * 256;
  uint32_t v[8], sum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[k] = h[lane * 8 + k];
    sum += v[k];
  }
  if (p == 0) {
    const uint32_t tot = warp_sum(sum);
    if (lane == 0) {
      s.total = tot;
      s.active = tot >= cap ? 1u : 0u;
      s.need = cap;
      s.key[0] = s.key[1] = s.key[2] = 0;
    }
    __syncwarp();
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

__global__ void k_bt_mark(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                          const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                          uint32_t kappa, const BtState* __restrict__ st,
                          uint8_t* __restrict__ recorded) {
  const uint64_t n = *d_n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = row[e], j = col[e], c = count[e];
    const BtState& s = st[bt_bucket(h_row, h_col, kappa, i, j)];
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
  CROP_CUDA(cudaMallocAsync(&d_st, (size_t)kappa * sizeof(BtState), st));
  CROP_CUDA(cudaMallocAsync(&d_hist, (size_t)kappa * 256 * 4, st));
  CROP_CUDA(cudaMemsetAsync(d_st, 0, (size_t)kappa * sizeof(BtState), st));
  CROP_CUDA(cudaMemsetAsync(d_hist, 0, (size_t)kappa * 256 * 4, st));
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n_capacity + kBtThreads - 1) / kBtThreads,
                                                                 (uint64_t)kNumSMs * 4));
  const int sel_grid = (int)((kappa + 7) / 8);
  for (uint32_t p = 0; p < 12; ++p) {
    k_bt_hist<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_st, p,
                                            d_hist);
    CROP_LAUNCH_CHECK();
    k_bt_select<<<sel_grid, 256, 0, st>>>(kappa, capacity, p, d_st, d_hist);
    CROP_LAUNCH_CHECK();
  }
  if (recorded) {
    k_bt_mark<<<grid, kBtThreads, 0, st>>>(row, col, count, d_n_entries, h_row, h_col, kappa, d_st,
                                            recorded);
    CROP_LAUNCH_CHECK();
  }
  k_bt_out<<<(kappa + 255) / 256, 256, 0, st>>>(kappa, d_st, bucket_min, bucket_total);
  CROP_LAUNCH_CHECK();
  cudaFreeAsync(d_hist, st);
  cudaFreeAsync(d_st, st);
  crop_count_launches(26);
  return CROP_OK;
}
