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
//   k_ss_clear / k_ss_insert   open-addressing index over the record keys:
//                              one 8-byte slot (hash fingerprint, record) per
//                              probe step, the key confirmed on the record
//   k_ss_probe                 chunk entries, pass 1: hits add e to their
//                              record's count; misses set a bit and count in
//                              their bucket's histogram of chunk weights
//   k_ss_cut                   per bucket: the weight below which a miss
//                              cannot reach the l largest
//   k_ss_append                pass 2: the misses at or above the cut are
//                              appended as candidates (mu_b + e, mu_b)
//                              behind the records (block-aggregated append)
// The per-bucket selection of the l largest is crop_bucket_topk over records
// + candidates.
#include <algorithm>

#include "common.cuh"

using namespace crop;

namespace {

constexpr unsigned long long kEmptySlot = ~0ull;

// index slot: fingerprint (high 32 bits of the key's hash, never all ones)
// << 32 | record index; a fingerprint match is confirmed on the record's key
__device__ __forceinline__ uint64_t key_of(uint32_t r, uint32_t c) { return ((uint64_t)r << 32) | c; }
__device__ __forceinline__ uint64_t slot_of(uint64_t k, uint64_t mask, uint64_t& h, uint32_t& fp) {
  const uint64_t x = splitmix64(k);
  h = x & mask;
  fp = (uint32_t)(x >> 32);
  if (fp == 0xFFFFFFFFu) fp = 0xFFFFFFFEu;
  return x;
}

// Bloom filter in front of the index: one 64-bit word per key (bits 20.. of
// the key's hash pick the word), four bits inside it. The filter is sized to
// stay L2-resident (<= 64 MB) while the index (16+ bytes per record at load
// <= 0.5) is not: a chunk's misses -- 9 in 10 of its entries on c3 -- are
// answered by one L2 sector instead of a DRAM access.
__device__ __forceinline__ void bloom_of(uint64_t x, uint64_t wmask, uint64_t& word, unsigned long long& bits) {
  word = (x >> 20) & (wmask & 0x7FFFFFFFFFFFFFFFull);
  const uint32_t y = (uint32_t)(x >> 32) * 0x9E3779B1u;
  bits = (1ull << (y & 63)) | (1ull << ((y >> 6) & 63));
  if (!(wmask >> 63)) bits |= (1ull << ((y >> 12) & 63)) | (1ull << ((y >> 18) & 63));
}
// filter words are read with an L2 evict-last policy (the entry streams are
// read evict-first), so the streamed chunk does not push the filter out
__device__ __forceinline__ unsigned long long ld_keep(const unsigned long long* p) {
  unsigned long long pol, v;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

__global__ void k_ss_clear(unsigned long long* __restrict__ slots, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    slots[i] = kEmptySlot;
}

__global__ void k_ss_insert(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col, uint64_t n,
                            unsigned long long* __restrict__ slots, uint64_t mask,
                            unsigned long long* __restrict__ bloom, uint64_t wmask) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h;
    uint32_t fp;
    const uint64_t x = slot_of(key_of(row[e], col[e]), mask, h, fp);
    if (bloom) {
      uint64_t bw;
      unsigned long long bb;
      bloom_of(x, wmask, bw, bb);
      atomicOr(&bloom[bw], bb);
    }
    const unsigned long long v = ((unsigned long long)fp << 32) | (uint32_t)e;
    while (atomicCAS(&slots[h], kEmptySlot, v) != kEmptySlot) h = (h + 1) & mask;
  }
}

// Pass 1 over the chunk entries: a recorded key adds its weight to the
// record; an unrecorded key (a miss) sets its bit in `missbits` and counts in
// its bucket's histogram of chunk weights (bins 1..14 exact, bin 15 = 15 and
// above; privatised in shared memory when kappa * 16 counters fit). Four
// entries per thread, their index probes in flight together.
//
// The histograms give each bucket its cut (k_ss_cut): the largest weight e*
// with at least l misses of weight >= e*. A miss below e* becomes a
// candidate (mu_b + e, mu_b) that at least l other candidates of its bucket
// beat, so it can never be among the bucket's l largest: pass 2
// (k_ss_append) appends only the misses at or above the cut and the
// selection reads ~l candidates per bucket instead of every distinct pair of
// the chunk (c3: 1.1e9 misses per chunk, 9 in 10 of them singletons). The
// summaries are the same records, bit for bit, as with every miss appended.
constexpr int kProbePer = 4;
constexpr int kSsBins = 16;
constexpr int kProbeThreads = 512;

template <bool SMEM_HIST>
__global__ void __launch_bounds__(kProbeThreads, 2)
    k_ss_probe(const uint32_t* __restrict__ erow, const uint32_t* __restrict__ ecol,
               const uint32_t* __restrict__ ecnt, const unsigned long long* __restrict__ d_ne,
               const unsigned long long* __restrict__ slots, uint64_t mask,
               const unsigned long long* __restrict__ bloom, uint64_t wmask,
               const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col, uint32_t kappa,
               const uint32_t* __restrict__ row, const uint32_t* __restrict__ col, uint32_t* __restrict__ cnt,
               uint32_t* __restrict__ missbits, uint32_t* __restrict__ hist, unsigned int* __restrict__ d_sat) {
  extern __shared__ uint32_t s_hist[];
  const uint32_t nbins = kappa * kSsBins;
  if (SMEM_HIST) {
    for (uint32_t k = threadIdx.x; k < nbins; k += blockDim.x) s_hist[k] = 0;
    __syncthreads();
  }
  const uint64_t ne = *d_ne;
  const uint64_t span = (uint64_t)blockDim.x * kProbePer;
  const int lane = threadIdx.x & 31;
  for (uint64_t base = blockIdx.x * span; base < ne; base += (uint64_t)gridDim.x * span) {
    uint32_t r[kProbePer], c[kProbePer], w[kProbePer];
    bool valid[kProbePer];
    uint64_t h[kProbePer];
    uint32_t fp[kProbePer];
    unsigned long long sv[kProbePer];
    bool maybe[kProbePer];  // the filter does not rule the key out
    uint64_t bw[kProbePer];
    unsigned long long bb[kProbePer];
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      const uint64_t e = base + (uint64_t)u * blockDim.x + threadIdx.x;
      bw[u] = 0;
      bb[u] = 0;
      valid[u] = e < ne;
      r[u] = c[u] = w[u] = 0;
      h[u] = 0;
      fp[u] = 0;
      maybe[u] = false;
      if (valid[u]) {
        r[u] = __ldcs(erow + e);
        c[u] = __ldcs(ecol + e);
        w[u] = __ldcs(ecnt + e);
        const uint64_t x = slot_of(key_of(r[u], c[u]), mask, h[u], fp[u]);
        maybe[u] = true;
        if (bloom) {
          bloom_of(x, wmask, bw[u], bb[u]);
        }
      }
    }
    if (bloom) {
      unsigned long long fv[kProbePer];
#pragma unroll
      for (int u = 0; u < kProbePer; ++u) fv[u] = valid[u] ? ld_keep(bloom + bw[u]) : 0ull;
#pragma unroll
      for (int u = 0; u < kProbePer; ++u) maybe[u] = valid[u] && (fv[u] & bb[u]) == bb[u];
    }
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) sv[u] = maybe[u] ? slots[h[u]] : kEmptySlot;
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      bool miss = false;
      if (valid[u]) {
        unsigned long long s = sv[u];
        for (;;) {
          if (s == kEmptySlot) {
            miss = true;
            break;
          }
          if ((uint32_t)(s >> 32) == fp[u]) {
            const uint32_t x = (uint32_t)s;
            if (row[x] == r[u] && col[x] == c[u]) {
              const uint32_t old = atomicAdd(&cnt[x], w[u]);
              if (old + w[u] < old) atomicOr(d_sat, 1u);
              break;
            }
          }
          h[u] = (h[u] + 1) & mask;
          s = slots[h[u]];
        }
        if (miss) {
          uint32_t b = h_row[r[u]] + h_col[c[u]];
          if (b >= kappa) b -= kappa;
          const uint32_t bin = b * kSsBins + min(w[u], (uint32_t)kSsBins - 1u);
          if (SMEM_HIST) atomicAdd(&s_hist[bin], 1u);
          else atomicAdd(&hist[bin], 1u);
        }
      }
      const uint32_t bits = __ballot_sync(0xffffffffu, miss);
      const uint64_t e0 = base + (uint64_t)u * blockDim.x + (threadIdx.x & ~31u);  // the warp's first entry
      if (lane == 0 && e0 < ne) missbits[e0 >> 5] = bits;
    }
  }
  if (SMEM_HIST) {
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nbins; k += blockDim.x) {
      const uint32_t v = s_hist[k];
      if (v) atomicAdd(&hist[k], v);
    }
  }
}

// Per bucket: the cut e* (0 = keep every miss) and the number of misses at or
// above it; meta[0] += that number, meta[1] = the smallest cut of any bucket.
__global__ void k_ss_cut(const uint32_t* __restrict__ hist, uint32_t kappa, uint32_t capacity,
                         uint32_t* __restrict__ cut, unsigned long long* __restrict__ meta) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= kappa) return;
  uint64_t above = 0;
  uint32_t e = 0;
  for (int k = kSsBins - 1; k >= 1; --k) {
    above += hist[b * kSsBins + k];
    if (above >= capacity) {
      e = (uint32_t)k;
      break;
    }
  }
  if (e == 0) above += hist[b * kSsBins];  // (weights are >= 1: bin 0 stays empty)
  cut[b] = e;
  atomicAdd(&meta[0], (unsigned long long)above);
  atomicMin(&meta[1], (unsigned long long)e);
}

// block-wide exclusive scan of one count per thread (blockDim 256) and one
// global claim per block: returns this thread's first output position
__device__ __forceinline__ unsigned long long block_claim(uint32_t mine, unsigned long long* d_n) {
  __shared__ uint32_t s_w[8];
  __shared__ unsigned long long s_base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan(mine);
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int k = 0; k < 8; ++k) {
      const uint32_t v = s_w[k];
      s_w[k] = t;
      t += v;
    }
    s_base = t ? atomicAdd(d_n, (unsigned long long)t) : 0ull;
  }
  __syncthreads();
  const unsigned long long r = s_base + s_w[w] + incl - mine;
  __syncthreads();
  return r;
}

// Pass 2: the misses at or above their bucket's cut are appended behind the
// records as candidates (mu_b + e, over mu_b); one output claim per block
// step of 1,024 entries (a claim per warp serialised 4.4e7 atomics on one
// counter per c3 chunk). Entries below the smallest cut are skipped on their
// weight alone.
__global__ void __launch_bounds__(256)
    k_ss_append(const uint32_t* __restrict__ erow, const uint32_t* __restrict__ ecol,
                const uint32_t* __restrict__ ecnt, const unsigned long long* __restrict__ d_ne,
                const uint32_t* __restrict__ missbits, const uint32_t* __restrict__ cut,
                const unsigned long long* __restrict__ meta, const uint32_t* __restrict__ h_row,
                const uint32_t* __restrict__ h_col, uint32_t kappa, const uint32_t* __restrict__ mu,
                uint32_t* __restrict__ row, uint32_t* __restrict__ col, uint32_t* __restrict__ cnt,
                uint32_t* __restrict__ over, unsigned long long* __restrict__ d_nout,
                unsigned int* __restrict__ d_sat) {
  const uint64_t ne = *d_ne;
  const uint32_t cut_min = (uint32_t)meta[1];
  const uint64_t span = (uint64_t)blockDim.x * kProbePer;
  for (uint64_t base = blockIdx.x * span; base < ne; base += (uint64_t)gridDim.x * span) {
    uint32_t r[kProbePer], c[kProbePer], w[kProbePer], m[kProbePer];
    bool take[kProbePer];
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      const uint64_t e = base + (uint64_t)u * blockDim.x + threadIdx.x;
      take[u] = false;
      r[u] = c[u] = w[u] = m[u] = 0;
      if (e < ne) {
        w[u] = ecnt[e];
        take[u] = w[u] >= cut_min && ((missbits[e >> 5] >> (e & 31)) & 1u);
      }
    }
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      if (!take[u]) continue;
      const uint64_t e = base + (uint64_t)u * blockDim.x + threadIdx.x;
      r[u] = erow[e];
      c[u] = ecol[e];
      uint32_t b = h_row[r[u]] + h_col[c[u]];
      if (b >= kappa) b -= kappa;
      if (w[u] < cut[b]) {
        take[u] = false;
        continue;
      }
      m[u] = mu[b];
      if (m[u] + w[u] < m[u]) atomicOr(d_sat, 1u);
      ++mine;
    }
    unsigned long long o = block_claim(mine, d_nout);
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      if (!take[u]) continue;
      row[o] = r[u];
      col[o] = c[u];
      cnt[o] = m[u] + w[u];
      over[o] = m[u];
      ++o;
    }
  }
}

// the records a per-bucket selection kept (mask), appended to the new
// record arrays (any order: a summary is a set)
__global__ void __launch_bounds__(256) k_ss_keep(const uint8_t* __restrict__ mask, const unsigned long long* __restrict__ d_n,
                          const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ over,
                          uint32_t* __restrict__ o_row, uint32_t* __restrict__ o_col, uint32_t* __restrict__ o_cnt,
                          uint32_t* __restrict__ o_over, unsigned long long* __restrict__ d_nout) {
  const uint64_t n = *d_n;
  const uint64_t span = (uint64_t)blockDim.x * kProbePer;
  for (uint64_t base = blockIdx.x * span; base < n; base += (uint64_t)gridDim.x * span) {
    bool k[kProbePer];
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      const uint64_t e = base + (uint64_t)u * blockDim.x + threadIdx.x;
      k[u] = e < n && mask[e];
      mine += k[u];
    }
    unsigned long long o = block_claim(mine, d_nout);
#pragma unroll
    for (int u = 0; u < kProbePer; ++u) {
      if (!k[u]) continue;
      const uint64_t e = base + (uint64_t)u * blockDim.x + threadIdx.x;
      o_row[o] = row[e];
      o_col[o] = col[e];
      o_cnt[o] = cnt[e];
      o_over[o] = over[e];
      ++o;
    }
  }
}

// word mask of the filter; bit 63 set = two bits per key (more than 12 keys
// per word: four bits each would fill the words)
uint64_t bloom_wmask(uint64_t words, uint64_t n_keys) {
  return (words - 1) | (n_keys > 12 * words ? (1ull << 63) : 0ull);
}

}  // namespace

extern "C" int crop_ss_index(const uint32_t* row, const uint32_t* col, uint64_t n, unsigned long long* slots,
                             uint64_t n_slots, unsigned long long* bloom, uint64_t bloom_words, void* stream) {
  if (n_slots == 0 || (n_slots & (n_slots - 1)) || n_slots < 2 * n) {
    crop_set_error(CROP_ECONFIG, "index slots must be a power of two >= 2 * records");
    return CROP_ECONFIG;
  }
  if (bloom && (bloom_words == 0 || (bloom_words & (bloom_words - 1)))) {
    crop_set_error(CROP_ECONFIG, "filter words must be a power of two");
    return CROP_ECONFIG;
  }
  if (n >= (1ull << 32)) {
    crop_set_error(CROP_ERESOURCE, "more than 2^32 summary records");
    return CROP_ERESOURCE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  k_ss_clear<<<8 * kNumSMs, 256, 0, st>>>(slots, n_slots);
  CROP_LAUNCH_CHECK();
  if (bloom) CROP_CUDA(cudaMemsetAsync(bloom, 0, bloom_words * 8, st));
  if (n) {
    k_ss_insert<<<8 * kNumSMs, 256, 0, st>>>(row, col, n, slots, n_slots - 1, bloom,
                                             bloom ? bloom_wmask(bloom_words, n) : 0);
    CROP_LAUNCH_CHECK();
  }
  crop_count_launches(n ? 2 : 1);
  return CROP_OK;
}

extern "C" int crop_ss_probe(const uint32_t* erow, const uint32_t* ecol, const uint32_t* ecnt,
                             const uint64_t* d_n_entries, uint64_t max_entries, const unsigned long long* slots,
                             uint64_t n_slots, const unsigned long long* bloom, uint64_t bloom_words,
                             uint64_t n_records, const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                             uint32_t capacity, const uint32_t* rec_row, const uint32_t* rec_col,
                             uint32_t* rec_count, uint32_t* missbits, uint32_t* hist, uint32_t* cut,
                             uint64_t* d_meta, unsigned int* d_saturated, void* stream) {
  if (kappa == 0 || capacity == 0) {
    crop_set_error(CROP_ECONFIG, "kappa and the summary capacity must be >= 1");
    return CROP_ECONFIG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t hist_bytes = (size_t)kappa * kSsBins * 4;
  CROP_CUDA(cudaMemsetAsync(hist, 0, hist_bytes, st));
  CROP_CUDA(cudaMemsetAsync(d_meta, 0, 8, st));
  CROP_CUDA(cudaMemsetAsync(d_meta + 1, 0xFF, 8, st));
  int launches = 1;
  if (max_entries) {
    const uint64_t span = (uint64_t)kProbeThreads * kProbePer;
    const uint64_t blocks = std::min<uint64_t>((max_entries + span - 1) / span, 2 * kNumSMs);
    if (hist_bytes <= 96 * 1024) {
      CROP_CUDA(cudaFuncSetAttribute(k_ss_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
      k_ss_probe<true><<<(unsigned)blocks, kProbeThreads, hist_bytes, st>>>(
          erow, ecol, ecnt, (const unsigned long long*)d_n_entries, slots, n_slots - 1, bloom,
          bloom ? bloom_wmask(bloom_words, n_records) : 0, h_row, h_col, kappa, rec_row, rec_col, rec_count, missbits, hist,
          d_saturated);
    } else {
      k_ss_probe<false><<<(unsigned)blocks, kProbeThreads, 0, st>>>(
          erow, ecol, ecnt, (const unsigned long long*)d_n_entries, slots, n_slots - 1, bloom,
          bloom ? bloom_wmask(bloom_words, n_records) : 0, h_row, h_col, kappa, rec_row, rec_col, rec_count, missbits, hist,
          d_saturated);
    }
    CROP_LAUNCH_CHECK();
    ++launches;
  }
  k_ss_cut<<<(kappa + 255) / 256, 256, 0, st>>>(hist, kappa, capacity, cut, (unsigned long long*)d_meta);
  CROP_LAUNCH_CHECK();
  crop_count_launches(launches);
  return CROP_OK;
}

extern "C" int crop_ss_append(const uint32_t* erow, const uint32_t* ecol, const uint32_t* ecnt,
                              const uint64_t* d_n_entries, uint64_t max_entries, const uint32_t* missbits,
                              const uint32_t* cut, const uint64_t* d_meta, const uint32_t* h_row,
                              const uint32_t* h_col, uint32_t kappa, const uint32_t* mu, uint32_t* row,
                              uint32_t* col, uint32_t* count, uint32_t* over, uint64_t* d_n_out,
                              unsigned int* d_saturated, void* stream) {
  if (kappa == 0) {
    crop_set_error(CROP_ECONFIG, "kappa must be >= 1");
    return CROP_ECONFIG;
  }
  if (max_entries == 0) return CROP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t blocks = std::min<uint64_t>((max_entries + 1023) / 1024, 16 * kNumSMs);
  k_ss_append<<<(unsigned)blocks, 256, 0, st>>>(erow, ecol, ecnt, (const unsigned long long*)d_n_entries, missbits,
                                               cut, (const unsigned long long*)d_meta, h_row, h_col, kappa, mu, row,
                                               col, count, over, (unsigned long long*)d_n_out, d_saturated);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}

extern "C" int crop_ss_keep(const uint8_t* mask, const uint64_t* d_n, uint64_t max_n, const uint32_t* row,
                            const uint32_t* col, const uint32_t* count, const uint32_t* over, uint32_t* out_row,
                            uint32_t* out_col, uint32_t* out_count, uint32_t* out_over, uint64_t* d_n_out,
                            void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  CROP_CUDA(cudaMemsetAsync(d_n_out, 0, 8, st));
  if (max_n == 0) return CROP_OK;
  const uint64_t blocks = std::min<uint64_t>((max_n + 1023) / 1024, 16 * kNumSMs);
  k_ss_keep<<<(unsigned)blocks, 256, 0, st>>>(mask, (const unsigned long long*)d_n, row, col, count, over, out_row,
                                             out_col, out_count, out_over, (unsigned long long*)d_n_out);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}
