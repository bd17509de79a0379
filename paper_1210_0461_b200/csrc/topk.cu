// topk.cu -- K4: top-k entries by (count desc, row asc, col asc).
//
// Replaces the Python sort in SketchState.top_entries (engine.py:162-172) and
// exact_top (oracle.py:53-58) for exact-regime results: in that regime every
// bucket summary is exact, so upper == lower == count and the reference's
// ranking key (-upper, -lower, row, col) is (count desc, row, col).
//
//   1. k_topk_hist     monotone 23,552-bin histogram of counts (exact below
//                      2048, 2^-10 relative resolution above), shared-memory
//                      privatised, one read of the count column.
//   2. k_topk_thresh   one block finds the bin B holding the k-th largest and
//                      the number of entries strictly above it.
//   3. k_topk_compact  entries above B go straight to the output; entries in
//                      B become candidates.
//   4. k_topk_finish   the r = k - above best candidates of bin B: one block
//                      bitonic-sorts up to 8192 (count, row, col) keys in
//                      shared memory; larger candidate sets use an MSD radix
//                      select over the 96-bit key (k_rs_*), 8 bits per pass.
#include <cstdint>

#include "common.cuh"

using namespace crop;

namespace {

constexpr uint32_t kExactBins = kTopkExactBins;
constexpr uint32_t kBins = kTopkBins;
constexpr int kHistThreads = 1024;
constexpr uint32_t kSmallCand = 8192;

__device__ __forceinline__ uint32_t count_bin(uint32_t c) { return topk_count_bin(c); }

__global__ void __launch_bounds__(kHistThreads)
    k_topk_hist(const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                uint32_t* __restrict__ hist, const unsigned long long* __restrict__ fast,
                uint32_t skip_from) {
  // fast: the fused high-count histogram already holds the k-th largest;
  // skip_from: counts >= this are already in `hist` (fused by the count kernels)
  if (fast && *fast) return;
  extern __shared__ uint32_t s_hist[];
  for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  const uint64_t n = *d_n;
  // counts are heavily repeated (most entries have small counts): aggregate
  // equal bins inside the warp before touching shared memory
  const uint64_t n_round = (n + 31) & ~31ull;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n_round;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = 0xFFFFFFFFu;
    if (e < n) {
      const uint32_t c = count[e];
      if (c < skip_from) b = count_bin(c);
    }
    const uint32_t grp = __match_any_sync(0xffffffffu, b);
    if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (int)(threadIdx.x & 31))
      atomicAdd(&s_hist[b], (uint32_t)__popc(grp));
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < kBins; b += blockDim.x)
    if (s_hist[b]) atomicAdd(&hist[b], s_hist[b]);
}

// state[0] = threshold bin B, state[1] = #entries above B, state[2] = k_eff,
// state[3] = out cursor, state[4] = candidate cursor
__global__ void __launch_bounds__(1024)
    k_topk_thresh(const uint32_t* __restrict__ hist, const uint64_t* __restrict__ d_n, uint32_t k,
                  unsigned long long* __restrict__ state, uint64_t* __restrict__ d_k_out) {
  __shared__ unsigned long long s_sum[1024];
  const uint64_t n = *d_n;
  const uint64_t keff = n < k ? n : k;
  const uint32_t per = (kBins + 1023) / 1024;
  // thread t owns bins [kBins - (t+1)*per, kBins - t*per) (top-down)
  const int t = threadIdx.x;
  const int hi = (int)kBins - t * (int)per;
  const int lo = max(0, hi - (int)per);
  unsigned long long acc = 0;
  for (int b = lo; b < hi; ++b) acc += hist[b];
  s_sum[t] = acc;
  __syncthreads();
  if (t == 0) {
    state[3] = 0;
    state[4] = 0;
    *d_k_out = keff;
    state[2] = keff;
    if (keff == 0) {
      state[0] = kBins;  // nothing selected
      state[1] = 0;
    } else {
      unsigned long long run = 0;
      int owner = 0;
      for (owner = 0; owner < 1024; ++owner) {
        if (run + s_sum[owner] >= keff) break;
        run += s_sum[owner];
      }
      const int ohi = (int)kBins - owner * (int)per;
      const int olo = max(0, ohi - (int)per);
      int B = olo;
      for (int b = ohi - 1; b >= olo; --b) {
        if (run + hist[b] >= keff) {
          B = b;
          break;
        }
        run += hist[b];
      }
      state[0] = (unsigned long long)B;
      state[1] = run;
    }
  }
}

__global__ void k_topk_compact(const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                               unsigned long long* __restrict__ state, uint64_t* __restrict__ out_idx,
                               uint64_t* __restrict__ cand, const unsigned long long* __restrict__ fast,
                               const unsigned long long* __restrict__ hi_list,
                               const unsigned long long* __restrict__ hi_n) {
  // fast path: only the fused list of high-count entries can be selected
  const bool f = fast && *fast;
  const uint64_t n = f ? *hi_n : *d_n;
  const uint32_t B = (uint32_t)state[0];
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = f ? hi_list[x] : x;
    const uint32_t b = count_bin(count[e]);
    if (b > B) out_idx[atomicAdd(&state[3], 1ull)] = e;
    else if (b == B) cand[atomicAdd(&state[4], 1ull)] = e;
  }
}

// Fused path decision: the count kernels added every count >= kExactBins to
// `hist` and its entry index to hi_list; if those entries number >= k_eff,
// the k-th largest is among them and neither the full histogram nor the full
// compaction pass is needed.
__global__ void k_topk_prep(const uint32_t* __restrict__ hist, const uint64_t* __restrict__ d_n,
                            uint32_t k, unsigned long long* __restrict__ fast) {
  __shared__ unsigned long long s_sum[32];
  unsigned long long acc = 0;
  for (uint32_t b = kExactBins + threadIdx.x; b < kBins; b += blockDim.x) acc += hist[b];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_sum[w];
    const uint64_t n = *d_n;
    const uint64_t keff = n < k ? n : k;
    *fast = keff > 0 && t >= keff;
  }
}

struct Key96 {
  uint32_t inv_count, row, col;
};

__device__ __forceinline__ bool key_less(const Key96& a, const Key96& b) {
  if (a.inv_count != b.inv_count) return a.inv_count < b.inv_count;
  if (a.row != b.row) return a.row < b.row;
  return a.col < b.col;
}

// One block: sort the candidates (<= kSmallCand) by key and emit the best r.
__global__ void __launch_bounds__(1024)
    k_topk_finish_small(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                        const uint32_t* __restrict__ count, unsigned long long* __restrict__ state,
                        const uint64_t* __restrict__ cand, uint64_t* __restrict__ out_idx) {
  extern __shared__ unsigned char sm[];
  Key96* keys = reinterpret_cast<Key96*>(sm);
  uint32_t* pos = reinterpret_cast<uint32_t*>(sm + kSmallCand * sizeof(Key96));
  const uint32_t nc = (uint32_t)state[4];
  if (nc > kSmallCand) return;  // handled by the radix path
  const uint64_t above = state[3];
  const uint64_t r = state[2] - above;
  uint32_t P = 1;
  while (P < nc) P <<= 1;
  for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
    if (t < nc) {
      const uint64_t e = cand[t];
      keys[t] = Key96{~count[e], row[e], col[e]};
    } else {
      keys[t] = Key96{0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    }
    pos[t] = t;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
        const uint32_t partner = t ^ stride;
        if (partner > t) {
          const bool up = (t & size) == 0;
          const bool swap = up ? key_less(keys[partner], keys[t]) : key_less(keys[t], keys[partner]);
          if (swap) {
            Key96 tk = keys[t];
            keys[t] = keys[partner];
            keys[partner] = tk;
            uint32_t tp = pos[t];
            pos[t] = pos[partner];
            pos[partner] = tp;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t t = threadIdx.x; t < r && t < nc; t += blockDim.x) out_idx[above + t] = cand[pos[t]];
}

// --- MSD radix select over candidates (large tie sets) -------------------
// digit d (0..11) of the 96-bit key, most significant first
__device__ __forceinline__ uint32_t key_digit(const Key96& k, int d) {
  const uint32_t w = d < 4 ? k.inv_count : (d < 8 ? k.row : k.col);
  return (w >> (24 - 8 * (d & 3))) & 0xFF;
}

// rs[0..2] = key prefix words (valid for digits < pass), rs[3] = remaining r
__global__ void k_rs_hist(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ count, const unsigned long long* __restrict__ state,
                          const uint64_t* __restrict__ cand, const uint32_t* __restrict__ rs, int pass,
                          uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const uint64_t nc = state[4];
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nc;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = cand[t];
    const Key96 k{~count[e], row[e], col[e]};
    bool match = true;
    for (int d = 0; d < pass; ++d) {
      const uint32_t want = (rs[d / 4] >> (24 - 8 * (d & 3))) & 0xFF;
      if (key_digit(k, d) != want) {
        match = false;
        break;
      }
    }
    if (match) atomicAdd(&s_h[key_digit(k, pass)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (s_h[b]) atomicAdd(&hist[b], s_h[b]);
}

__global__ void k_rs_pick(uint32_t* __restrict__ hist, uint32_t* __restrict__ rs, int pass) {
  if (threadIdx.x != 0) return;
  uint32_t r = rs[3];
  uint32_t d = 0;
  for (d = 0; d < 256; ++d) {
    if (hist[d] >= r) break;
    r -= hist[d];
  }
  rs[pass / 4] |= d << (24 - 8 * (pass & 3));
  rs[3] = r;
  for (int b = 0; b < 256; ++b) hist[b] = 0;
}

// emit candidates whose key <= the selected key (exactly r of them: keys unique)
__global__ void k_rs_emit(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ count, unsigned long long* __restrict__ state,
                          const uint64_t* __restrict__ cand, const uint32_t* __restrict__ rs,
                          uint64_t* __restrict__ out_idx) {
  const uint64_t nc = state[4];
  const Key96 kth{rs[0], rs[1], rs[2]};
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nc;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = cand[t];
    const Key96 k{~count[e], row[e], col[e]};
    if (!key_less(kth, k)) out_idx[atomicAdd(&state[3], 1ull)] = e;
  }
}

__global__ void k_rs_init(const unsigned long long* __restrict__ state, uint32_t* __restrict__ rs) {
  rs[0] = rs[1] = rs[2] = 0;
  rs[3] = (uint32_t)(state[2] - state[3]);
}

}  // namespace

// Shared by crop_topk and crop_pairs_topk: fused_hist / hi_list / hi_n are
// the high-count histogram and entry list filled by the counting kernels
// (nullptr: plain path).
int crop_topk_impl(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                   const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k,
                   uint64_t* out_idx, uint64_t* d_k_out, cudaStream_t st, uint32_t* fused_hist,
                   const unsigned long long* hi_list, const unsigned long long* hi_n) {
  if (int rc = crop_pool_setup()) return rc;
  uint32_t* hist = nullptr;
  unsigned long long* state = nullptr;
  uint64_t* cand = nullptr;
  uint32_t* rs = nullptr;
  uint32_t* rs_hist = nullptr;
  uint64_t cand_cap = max_entries > 0 ? max_entries : 1;
  if (cand_cap > (1ull << 27)) {
    // large capacity bound: size the candidate list by the actual entry count
    uint64_t h_n = 0;
    CROP_CUDA(cudaMemcpyAsync(&h_n, d_n_entries, 8, cudaMemcpyDeviceToHost, st));
    CROP_CUDA(cudaStreamSynchronize(st));
    cand_cap = h_n > 0 ? h_n : 1;
  }
  const bool fused = fused_hist != nullptr;
  CROP_CUDA(cudaMallocAsync(&hist, kBins * 4, st));
  // the fused histogram is copied, not updated: the entries stay selectable again
  CROP_CUDA(cudaMallocAsync(&state, 8 * 8, st));  // [0..4] select state, [5] fused fast flag
  CROP_CUDA(cudaMallocAsync(&cand, cand_cap * 8, st));
  CROP_CUDA(cudaMallocAsync(&rs, 4 * 4, st));
  CROP_CUDA(cudaMallocAsync(&rs_hist, 256 * 4, st));
  if (fused) CROP_CUDA(cudaMemcpyAsync(hist, fused_hist, kBins * 4, cudaMemcpyDeviceToDevice, st));
  else CROP_CUDA(cudaMemsetAsync(hist, 0, kBins * 4, st));
  CROP_CUDA(cudaMemsetAsync(rs_hist, 0, 256 * 4, st));
  unsigned long long* fast = fused ? state + 5 : nullptr;
  if (fused) {
    k_topk_prep<<<1, 1024, 0, st>>>(hist, d_n_entries, k, fast);
    CROP_LAUNCH_CHECK();
    crop_count_launches(1);
  }
  uint64_t blocks = (max_entries + kHistThreads - 1) / kHistThreads;
  if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
  if (blocks == 0) blocks = 1;
  CROP_CUDA(cudaFuncSetAttribute(k_topk_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kBins * 4)));
  k_topk_hist<<<(int)blocks, kHistThreads, kBins * 4, st>>>(count, d_n_entries, hist, fast,
                                                             fused ? kExactBins : 0xFFFFFFFFu);
  CROP_LAUNCH_CHECK();
  k_topk_thresh<<<1, 1024, 0, st>>>(hist, d_n_entries, k, state, d_k_out);
  CROP_LAUNCH_CHECK();
  uint64_t cblocks = (max_entries + 255) / 256;
  if (cblocks > 8 * kNumSMs) cblocks = 8 * kNumSMs;
  if (cblocks == 0) cblocks = 1;
  k_topk_compact<<<(int)cblocks, 256, 0, st>>>(count, d_n_entries, state, out_idx, cand, fast,
                                               hi_list, hi_n);
  CROP_LAUNCH_CHECK();
  const size_t small_smem = kSmallCand * (sizeof(Key96) + 4);
  CROP_CUDA(cudaFuncSetAttribute(k_topk_finish_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)small_smem));
  k_topk_finish_small<<<1, 1024, small_smem, st>>>(row, col, count, state, cand, out_idx);
  CROP_LAUNCH_CHECK();
  crop_count_launches(4);
  // The large-candidate path needs the candidate count on the host.
  unsigned long long h_state[5];
  CROP_CUDA(cudaMemcpyAsync(h_state, state, sizeof(h_state), cudaMemcpyDeviceToHost, st));
  CROP_CUDA(cudaStreamSynchronize(st));
  if (h_state[4] > kSmallCand && h_state[2] > h_state[3]) {
    k_rs_init<<<1, 1, 0, st>>>(state, rs);
    CROP_LAUNCH_CHECK();
    uint64_t rb = (h_state[4] + 255) / 256;
    if (rb > 4 * kNumSMs) rb = 4 * kNumSMs;
    for (int pass = 0; pass < 12; ++pass) {
      k_rs_hist<<<(int)rb, 256, 0, st>>>(row, col, count, state, cand, rs, pass, rs_hist);
      CROP_LAUNCH_CHECK();
      k_rs_pick<<<1, 32, 0, st>>>(rs_hist, rs, pass);
      CROP_LAUNCH_CHECK();
    }
    k_rs_emit<<<(int)rb, 256, 0, st>>>(row, col, count, state, cand, rs, out_idx);
    CROP_LAUNCH_CHECK();
    crop_count_launches(26);
  }
  cudaFreeAsync(hist, st);
  cudaFreeAsync(state, st);
  cudaFreeAsync(cand, st);
  cudaFreeAsync(rs, st);
  cudaFreeAsync(rs_hist, st);
  return CROP_OK;
}

extern "C" int crop_topk(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                         const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k,
                         uint64_t* out_idx, uint64_t* d_k_out, void* stream) {
  return crop_topk_impl(row, col, count, d_n_entries, max_entries, k, out_idx, d_k_out,
                        (cudaStream_t)stream, nullptr, nullptr, nullptr);
}
