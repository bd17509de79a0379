// gen.cu -- seeded synthetic transactions for the benchmark configurations
// (BASELINE.json configs 1, 2, 3, 5): Zipf item ids drawn by
// successive sampling without replacement (iid draws from an integer alias
// table, repeats rejected), lengths from an integer CDF. Every draw is a pure
// function of (seed, transaction, draw index), so the data do not depend on
// the GPU or the launch shape.
#include <vector>

#include "common.cuh"

using namespace crop;

namespace {

constexpr int kGenWarps = 6;
constexpr uint32_t kGenMaxLen = 512;
constexpr uint32_t kGenSet = 1024;

__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t tx, uint64_t d) {
  return splitmix64(splitmix64(seed ^ (tx * 0xD1B54A32D192ED03ull)) + d);
}

__global__ void k_gen_lengths(int64_t n_tx, uint64_t seed, const uint32_t* __restrict__ cdf,
                              uint32_t n_len, uint32_t len_lo, int64_t* __restrict__ lengths) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tx;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(draw(seed ^ 0x6C656E677468ull, t, 0) >> 32);
    uint32_t lo = 0, hi = n_len - 1;  // first k with r < cdf[k]; cdf[n_len-1] treated as 2^32
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (r < cdf[mid]) hi = mid;
      else lo = mid + 1;
    }
    lengths[t] = (int64_t)(len_lo + lo);
  }
}

__global__ void __launch_bounds__(kGenWarps * 32)
    k_gen_items(int64_t n_tx, uint64_t seed, uint32_t n_items, const uint32_t* __restrict__ thresh,
                const uint32_t* __restrict__ alias, const int64_t* __restrict__ offsets,
                uint32_t* __restrict__ items) {
  __shared__ uint32_t s_acc[kGenWarps][kGenMaxLen];
  __shared__ uint32_t s_set[kGenWarps][kGenSet];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* acc = s_acc[w];
  uint32_t* set = s_set[w];
  for (int64_t t = (int64_t)blockIdx.x * kGenWarps + w; t < n_tx;
       t += (int64_t)gridDim.x * kGenWarps) {
    const int64_t base = offsets[t];
    const uint32_t L = (uint32_t)(offsets[t + 1] - base);
    for (uint32_t s = lane; s < kGenSet; s += 32) set[s] = kEmpty32;
    __syncwarp();
    uint32_t have = 0;
    for (uint64_t round = 0; have < L; ++round) {
      const uint64_t x = draw(seed, t, round * 32 + lane);
      const uint32_t col = (uint32_t)(((x & 0xFFFFFFFFull) * n_items) >> 32);
      const uint32_t item = ((uint32_t)(x >> 32) < thresh[col]) ? col : alias[col];
      // seen before this round?
      uint32_t h = mix32(item) & (kGenSet - 1);
      bool seen = false;
      for (;;) {
        const uint32_t v = set[h];
        if (v == item) {
          seen = true;
          break;
        }
        if (v == kEmpty32) break;
        h = (h + 1) & (kGenSet - 1);
      }
      const uint32_t grp = __match_any_sync(0xffffffffu, item);
      const bool first = (__ffs(grp) - 1) == lane;
      const bool cand = !seen && first;
      const uint32_t cm = __ballot_sync(0xffffffffu, cand);
      const uint32_t rank = __popc(cm & ((1u << lane) - 1u));
      const bool take = cand && have + rank < L;
      __syncwarp();
      if (take) {
        acc[have + rank] = item;
        uint32_t s = mix32(item) & (kGenSet - 1);
        while (atomicCAS(&set[s], kEmpty32, item) != kEmpty32) s = (s + 1) & (kGenSet - 1);
      }
      have = min(L, have + __popc(cm));
      __syncwarp();
    }
    // rank sort ascending (items distinct)
    for (uint32_t a = lane; a < L; a += 32) {
      const uint32_t v = acc[a];
      uint32_t r = 0;
      for (uint32_t b = 0; b < L; ++b) r += acc[b] < v;
      items[base + r] = v;
    }
    __syncwarp();
  }
}

}  // namespace

extern "C" int crop_gen_lengths(int64_t n_tx, uint64_t seed, const uint32_t* h_len_cdf,
                                uint32_t n_len, uint32_t len_lo, int64_t* lengths, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_len == 0) {
    crop_set_error(CROP_ECONFIG, "empty length distribution");
    return CROP_ECONFIG;
  }
  if (len_lo + n_len - 1 > kGenMaxLen) {
    crop_set_error(CROP_ECONFIG, "generator supports transactions up to %u items", kGenMaxLen);
    return CROP_ECONFIG;
  }
  if (n_tx <= 0) return CROP_OK;
  uint32_t* cdf = nullptr;
  CROP_CUDA(cudaMallocAsync(&cdf, n_len * 4, st));
  CROP_CUDA(cudaMemcpyAsync(cdf, h_len_cdf, n_len * 4, cudaMemcpyHostToDevice, st));
  int64_t blocks = std::min<int64_t>((n_tx + 255) / 256, 16 * kNumSMs);
  k_gen_lengths<<<(int)blocks, 256, 0, st>>>(n_tx, seed, cdf, n_len, len_lo, lengths);
  CROP_LAUNCH_CHECK();
  CROP_CUDA(cudaStreamSynchronize(st));  // h_len_cdf may be pageable and short-lived
  cudaFreeAsync(cdf, st);
  return CROP_OK;
}

extern "C" int crop_gen_items(int64_t n_tx, uint64_t seed, uint32_t n_items,
                              const uint32_t* h_alias_thresh, const uint32_t* h_alias_idx,
                              const int64_t* offsets, uint32_t* items, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_items == 0) {
    crop_set_error(CROP_ECONFIG, "need at least one item");
    return CROP_ECONFIG;
  }
  if (n_tx <= 0) return CROP_OK;
  uint32_t *th = nullptr, *al = nullptr;
  CROP_CUDA(cudaMallocAsync(&th, (size_t)n_items * 4, st));
  CROP_CUDA(cudaMallocAsync(&al, (size_t)n_items * 4, st));
  CROP_CUDA(cudaMemcpyAsync(th, h_alias_thresh, (size_t)n_items * 4, cudaMemcpyHostToDevice, st));
  CROP_CUDA(cudaMemcpyAsync(al, h_alias_idx, (size_t)n_items * 4, cudaMemcpyHostToDevice, st));
  int64_t blocks = std::min<int64_t>((n_tx + kGenWarps - 1) / kGenWarps, 32 * kNumSMs);
  k_gen_items<<<(int)blocks, kGenWarps * 32, 0, st>>>(n_tx, seed, n_items, th, al, offsets, items);
  CROP_LAUNCH_CHECK();
  CROP_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(th, st);
  cudaFreeAsync(al, st);
  return CROP_OK;
}
