// ss_stream.cu -- streaming, mergeable per-bucket Space-Saving (the bounded
// regime of spacesaving.py:39-63 with O(l) state per bucket).
//
// The stream is consumed in chunks of transactions. Each chunk is first
// aggregated exactly on chip (the pair engine: its distinct (row, col) pairs
// with their chunk supports e), then merged into the per-bucket summaries S_b
// (at most l records (key, count c, over o) each) with the batch form of the
// Space-Saving update:
//   key in S_b        c += e
//   key not in S_b    new record (c, o) = (mu_b + e, mu_b), mu_b = the
//                     summary minimum when S_b is full, else 0
// and S_b keeps its l largest counts (count desc, row, col). This is what the
// reference's per-term update (hit: c += w; miss with a full summary: evict
// the minimum and insert (c_min + w, c_min)) does when the chunk's terms of
// one key arrive together, and it keeps every guarantee of spacesaving.py:1-9:
// c - o <= exact <= c for recorded keys, exact <= mu_b for absent keys, and
// sum of counts <= m_b, so mu_b <= m_b / l and o <= m_b / l.
//
// Kernels (device state: the records of every bucket, one flat array, plus a
// hash index over their keys rebuilt per chunk):
//   k_ss_clear / k_ss_insert   open-addressing index key -> record (2x slots)
//   k_ss_probe                 chunk entries: hits add e to their record's
//                              count, misses are appended as candidates with
//                              (mu_b + e, mu_b) behind the records (warp-
//                              aggregated append)
// The per-bucket selection of the l largest is crop_bucket_topk over records
// + candidates.
#include <algorithm>

#include "common.cuh"

using namespace crop;

namespace {

constexpr unsigned long long kEmptyKey = ~0ull;

__global__ void k_ss_clear(unsigned long long* __restrict__ keys, uint64_t slots) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < slots; i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = kEmptyKey;
}

__global__ void k_ss_insert(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col, uint64_t n,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ idx, uint64_t mask) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ((unsigned long long)row[e] << 32) | col[e];
    uint64_t h = splitmix64(k) & mask;
    for (;;) {
      const unsigned long long prev = atomicCAS(&keys[h], kEmptyKey, k);
      if (prev == kEmptyKey) {
        idx[h] = (uint32_t)e;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

__global__ void k_ss_probe(const uint32_t* __restrict__ erow, const uint32_t* __restrict__ ecol,
                           const uint32_t* __restrict__ ecnt, const unsigned long long* __restrict__ d_ne,
                           const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ idx,
                           uint64_t mask, const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                           uint32_t kappa, const uint32_t* __restrict__ mu, uint32_t* __restrict__ rec_cnt,
                           uint32_t* __restrict__ out_row, uint32_t* __restrict__ out_col,
                           uint32_t* __restrict__ out_cnt, uint32_t* __restrict__ out_over,
                           unsigned long long* __restrict__ d_nout, unsigned int* __restrict__ d_sat) {
  const uint64_t ne = *d_ne;
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < ne; base += stride) {
    const uint64_t e = base + threadIdx.x;
    bool miss = false;
    uint32_t r = 0, c = 0, w = 0, m = 0;
    if (e < ne) {
      r = erow[e];
      c = ecol[e];
      w = ecnt[e];
      const unsigned long long k = ((unsigned long long)r << 32) | c;
      uint64_t h = splitmix64(k) & mask;
      for (;;) {
        const unsigned long long s = keys[h];
        if (s == k) {
          const uint32_t old = atomicAdd(&rec_cnt[idx[h]], w);
          if (old + w < old) atomicOr(d_sat, 1u);
          break;
        }
        if (s == kEmptyKey) {
          miss = true;
          break;
        }
        h = (h + 1) & mask;
      }
      if (miss) {
        uint32_t b = h_row[r] + h_col[c];
        if (b >= kappa) b -= kappa;
        m = mu[b];
        if (m + w < m) atomicOr(d_sat, 1u);
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, miss);
    unsigned long long pos = 0;
    if (lane == 0 && bal) pos = atomicAdd(d_nout, (unsigned long long)__popc(bal));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (miss) {
      const unsigned long long o = pos + __popc(bal & ((1u << lane) - 1u));
      out_row[o] = r;
      out_col[o] = c;
      out_cnt[o] = m + w;
      out_over[o] = m;
    }
  }
}

}  // namespace

extern "C" int crop_ss_index(const uint32_t* row, const uint32_t* col, uint64_t n, unsigned long long* keys,
                             uint32_t* idx, uint64_t slots, void* stream) {
  if (slots == 0 || (slots & (slots - 1)) || slots < 2 * n) {
    crop_set_error(CROP_ECONFIG, "index slots must be a power of two >= 2 * records");
    return CROP_ECONFIG;
  }
  if (n >= (1ull << 32)) {
    crop_set_error(CROP_ERESOURCE, "more than 2^32 summary records");
    return CROP_ERESOURCE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  k_ss_clear<<<8 * kNumSMs, 256, 0, st>>>(keys, slots);
  CROP_LAUNCH_CHECK();
  if (n) {
    k_ss_insert<<<8 * kNumSMs, 256, 0, st>>>(row, col, n, keys, idx, slots - 1);
    CROP_LAUNCH_CHECK();
  }
  crop_count_launches(n ? 2 : 1);
  return CROP_OK;
}

extern "C" int crop_ss_probe(const uint32_t* erow, const uint32_t* ecol, const uint32_t* ecnt,
                             const uint64_t* d_n_entries, uint64_t max_entries, const unsigned long long* keys,
                             const uint32_t* idx, uint64_t slots, const uint32_t* h_row, const uint32_t* h_col,
                             uint32_t kappa, const uint32_t* mu, uint32_t* rec_count, uint32_t* out_row,
                             uint32_t* out_col, uint32_t* out_count, uint32_t* out_over, uint64_t* d_n_out,
                             unsigned int* d_saturated, void* stream) {
  if (kappa == 0) {
    crop_set_error(CROP_ECONFIG, "kappa must be >= 1");
    return CROP_ECONFIG;
  }
  if (max_entries == 0) return CROP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t blocks = std::min<uint64_t>((max_entries + 255) / 256, 16 * kNumSMs);
  k_ss_probe<<<(unsigned)blocks, 256, 0, st>>>(erow, ecol, ecnt, (const unsigned long long*)d_n_entries, keys, idx,
                                              slots - 1, h_row, h_col, kappa, mu, rec_count, out_row, out_col,
                                              out_count, out_over, (unsigned long long*)d_n_out, d_saturated);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}
