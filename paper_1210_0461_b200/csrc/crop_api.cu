// crop_api.cu -- error plumbing, K0 hash tables, K1 bucket loads, entry
// bucket statistics. See include/crop_b200.h for the contract of each call.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>

#include "common.cuh"

static thread_local char g_err[512] = "no error";

void crop_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  int n = snprintf(g_err, sizeof(g_err), "[%d] ", code);
  vsnprintf(g_err + n, sizeof(g_err) - n, fmt, ap);
  va_end(ap);
}

extern "C" int crop_abi_version(void) { return 1; }

static unsigned long long g_launches = 0;
void crop_count_launches(int n) { __atomic_add_fetch(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }
extern "C" unsigned long long crop_launch_counter(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int crop_pool_setup() {
  static int done_dev = -1;
  int dev = 0;
  CROP_CUDA(cudaGetDevice(&dev));
  if (done_dev == dev) return CROP_OK;
  cudaMemPool_t pool;
  CROP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thresh = UINT64_MAX;
  CROP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  done_dev = dev;
  return CROP_OK;
}
extern "C" const char* crop_last_error(void) { return g_err; }

using namespace crop;

// ---------------------------------------------------------------- K0 hashes
// One thread per item; a handful of 64-bit multiplies, memory-bound on the
// 8 B/item of output. hashing.py:68-71.
__global__ void k_hash_tables(uint32_t n, uint64_t rm, uint64_t ra, uint64_t cm, uint64_t ca,
                              uint32_t kappa, uint32_t* __restrict__ h_row,
                              uint32_t* __restrict__ h_col) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    h_row[i] = (uint32_t)(mulmod61(rm, i, ra) % kappa);
    h_col[i] = (uint32_t)(mulmod61(cm, i, ca) % kappa);
  }
}

extern "C" int crop_hash_tables(uint32_t n_items, uint64_t row_mul, uint64_t row_add,
                                uint64_t col_mul, uint64_t col_add, uint32_t kappa,
                                uint32_t* h_row, uint32_t* h_col, void* stream) {
  if (kappa == 0 || kappa > (1u << 31)) {
    crop_set_error(CROP_ECONFIG, "kappa must be in [1, 2^31], got %u", kappa);
    return CROP_ECONFIG;
  }
  if (row_mul == 0 || row_mul >= kP61 || col_mul == 0 || col_mul >= kP61 || row_add >= kP61 ||
      col_add >= kP61) {
    crop_set_error(CROP_ECONFIG, "hash coefficients out of range");
    return CROP_ECONFIG;
  }
  if (n_items == 0) return CROP_OK;
  int blocks = (int)((n_items + 255) / 256);
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  k_hash_tables<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_items, row_mul, row_add, col_mul,
                                                           col_add, kappa, h_row, h_col);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}

__global__ void k_sign_hash(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                            uint64_t n, uint64_t mul, uint64_t add, int8_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    out[e] = (int8_t)sign_of(row[e], col[e], mul, add);
}

extern "C" int crop_sign_hash(const uint32_t* row, const uint32_t* col, uint64_t n,
                              uint64_t sign_mul, uint64_t sign_add, int8_t* out, void* stream) {
  if (n == 0) return CROP_OK;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  k_sign_hash<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(row, col, n, sign_mul, sign_add, out);
  CROP_LAUNCH_CHECK();
  return CROP_OK;
}

// ---------------------------------------------------------------- K1 loads
// Warp per outer product; lanes stride over the |a| x |b| grid (or the
// upper triangle for self-joins), each term adds 1 to its bucket in a
// shared-memory histogram (flushed once per CTA). kappa larger than the
// shared histogram falls back to global atomics (spread over many buckets,
// so uncontended). Replaces count_sorted (interval.py:192-233): the
// per-worker numbers are interval sums of these per-bucket counts.
constexpr int kLoadThreads = 512;
constexpr uint32_t kLoadSmemBuckets = 12288;  // 96 KB of u64

template <bool SELF>
__global__ void __launch_bounds__(kLoadThreads)
    k_bucket_loads(const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx,
                   const int64_t* __restrict__ b_ptr, const uint32_t* __restrict__ b_idx,
                   int64_t n, const uint32_t* __restrict__ h_row,
                   const uint32_t* __restrict__ h_col, uint32_t kappa, int upper_only,
                   unsigned long long* __restrict__ loads) {
  extern __shared__ unsigned long long s_hist[];
  const bool smem = kappa <= kLoadSmemBuckets;
  if (smem)
    for (uint32_t b = threadIdx.x; b < kappa; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int64_t k = (int64_t)blockIdx.x * warps + threadIdx.x / 32; k < n;
       k += (int64_t)gridDim.x * warps) {
    int64_t a0 = a_ptr[k], la = a_ptr[k + 1] - a0;
    int64_t b0 = SELF ? a0 : b_ptr[k];
    int64_t lb = SELF ? la : b_ptr[k + 1] - b0;
    const uint32_t* bi = SELF ? a_idx : b_idx;
    int64_t total = la * lb;
    for (int64_t t = lane; t < total; t += 32) {
      int64_t p = t / lb, q = t - p * lb;
      uint32_t i = a_idx[a0 + p], j = bi[b0 + q];
      if (upper_only && i >= j) continue;
      uint32_t b = h_row[i] + h_col[j];
      if (b >= kappa) b -= kappa;
      if (smem) atomicAdd(&s_hist[b], 1ull);
      else atomicAdd(&loads[b], 1ull);
    }
  }
  __syncthreads();
  if (smem)
    for (uint32_t b = threadIdx.x; b < kappa; b += blockDim.x)
      if (s_hist[b]) atomicAdd(&loads[b], s_hist[b]);
}

static int launch_loads(bool self, const int64_t* a_ptr, const uint32_t* a_idx,
                        const int64_t* b_ptr, const uint32_t* b_idx, int64_t n,
                        const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                        int upper_only, uint64_t* loads, void* stream) {
  if (kappa == 0) {
    crop_set_error(CROP_ECONFIG, "kappa must be >= 1");
    return CROP_ECONFIG;
  }
  if (n <= 0) return CROP_OK;
  size_t smem = kappa <= kLoadSmemBuckets ? kappa * sizeof(unsigned long long) : 0;
  auto kern = self ? k_bucket_loads<true> : k_bucket_loads<false>;
  CROP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kLoadSmemBuckets * sizeof(unsigned long long))));
  int64_t warps_needed = (n + 0);
  int64_t blocks = (warps_needed + (kLoadThreads / 32) - 1) / (kLoadThreads / 32);
  if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
  kern<<<(int)blocks, kLoadThreads, smem, (cudaStream_t)stream>>>(
      a_ptr, a_idx, b_ptr, b_idx, n, h_row, h_col, kappa, upper_only,
      (unsigned long long*)loads);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}

extern "C" int crop_selfjoin_bucket_loads(const int64_t* offsets, const uint32_t* items,
                                          int64_t n_tx, const uint32_t* h_row,
                                          const uint32_t* h_col, uint32_t kappa, int upper_only,
                                          uint64_t* bucket_loads, void* stream) {
  return launch_loads(true, offsets, items, offsets, items, n_tx, h_row, h_col, kappa,
                      upper_only, bucket_loads, stream);
}

extern "C" int crop_outer_bucket_loads(const int64_t* a_ptr, const uint32_t* a_idx,
                                       const int64_t* b_ptr, const uint32_t* b_idx,
                                       int64_t n_products, const uint32_t* h_row,
                                       const uint32_t* h_col, uint32_t kappa, int upper_only,
                                       uint64_t* bucket_loads, void* stream) {
  return launch_loads(false, a_ptr, a_idx, b_ptr, b_idx, n_products, h_row, h_col, kappa,
                      upper_only, bucket_loads, stream);
}

// ----------------------------------------------------- entry bucket stats
// One pass over the counted entries per instance: bucket -> sum of counts
// (LoadReport rows), number of entries (summary occupancy) and the
// Count-Sketch cell sum count * s(i, j). The sketch is exact integer
// arithmetic (0/1 streams), so atomics give the reference's fp64 cells bit
// for bit regardless of order.
constexpr int kStatThreads = 512;
constexpr uint32_t kStatSmemBuckets = 2048;  // 40 KB static shared

__global__ void __launch_bounds__(kStatThreads)
    k_entry_stats(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                  const uint32_t* __restrict__ count, const uint64_t* __restrict__ d_n,
                  const uint32_t* __restrict__ h_row, const uint32_t* __restrict__ h_col,
                  uint32_t kappa, uint64_t sign_mul, uint64_t sign_add, int do_cs,
                  unsigned long long* __restrict__ loads, uint32_t* __restrict__ distinct,
                  unsigned long long* __restrict__ cs) {
  __shared__ unsigned long long s_load[kStatSmemBuckets];
  __shared__ unsigned long long s_cs[kStatSmemBuckets];
  __shared__ uint32_t s_dist[kStatSmemBuckets];
  // few buckets (kappa <= 64): one counter set per lane index, so the 32
  // lanes of a warp never collide (the warps of the block share them);
  // otherwise one set per block
  const bool lanes = kappa <= kStatSmemBuckets / 32;
  const bool smem = kappa <= kStatSmemBuckets;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t slots = lanes ? kappa * 32 : kappa;
  if (smem)
    for (uint32_t b = threadIdx.x; b < slots; b += blockDim.x) {
      s_load[b] = 0;
      s_cs[b] = 0;
      s_dist[b] = 0;
    }
  __syncthreads();
  const uint64_t n = *d_n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t i = row[e], j = col[e], c = count[e];
    uint32_t b = h_row[i] + h_col[j];
    if (b >= kappa) b -= kappa;
    long long sc = 0;
    if (do_cs) sc = sign_of(i, j, sign_mul, sign_add) * (long long)c;
    if (smem) {
      const uint32_t sl = lanes ? b * 32 + lane : b;
      atomicAdd(&s_load[sl], (unsigned long long)c);
      atomicAdd(&s_dist[sl], 1u);
      if (do_cs) atomicAdd(&s_cs[sl], (unsigned long long)sc);
    } else {
      atomicAdd(&loads[b], (unsigned long long)c);
      atomicAdd(&distinct[b], 1u);
      if (do_cs) atomicAdd(&cs[b], (unsigned long long)sc);
    }
  }
  __syncthreads();
  if (lanes) {
    // fold the 32 lane sets: warp w sums bucket w, w + nwarps, ...
    const uint32_t warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t b = warp; b < kappa; b += nw) {
      unsigned long long l = s_load[b * 32 + lane], x = s_cs[b * 32 + lane];
      uint32_t d = s_dist[b * 32 + lane];
      for (int o = 16; o; o >>= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
        x += __shfl_xor_sync(0xffffffffu, x, o);
        d += __shfl_xor_sync(0xffffffffu, d, o);
      }
      if (lane == 0) {
        if (l) atomicAdd(&loads[b], l);
        if (d) atomicAdd(&distinct[b], d);
        if (do_cs && x) atomicAdd(&cs[b], x);
      }
    }
  } else if (smem) {
    for (uint32_t b = threadIdx.x; b < kappa; b += blockDim.x) {
      if (s_load[b]) atomicAdd(&loads[b], s_load[b]);
      if (s_dist[b]) atomicAdd(&distinct[b], s_dist[b]);
      if (do_cs && s_cs[b]) atomicAdd(&cs[b], s_cs[b]);
    }
  }
}

extern "C" int crop_entry_bucket_stats(const uint32_t* row, const uint32_t* col,
                                       const uint32_t* count, const uint64_t* d_n_entries,
                                       uint64_t max_entries, int instances, uint32_t n_items,
                                       const uint32_t* h_row, const uint32_t* h_col,
                                       uint32_t kappa, const uint64_t* h_sign, uint64_t* loads,
                                       uint32_t* distinct, int64_t* cs, void* stream) {
  if (kappa == 0 || instances < 1) {
    crop_set_error(CROP_ECONFIG, "kappa and instances must be >= 1");
    return CROP_ECONFIG;
  }
  uint64_t blocks = (max_entries + kStatThreads - 1) / kStatThreads;
  if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
  if (blocks == 0) blocks = 1;
  for (int t = 0; t < instances; ++t) {
    k_entry_stats<<<(int)blocks, kStatThreads, 0, (cudaStream_t)stream>>>(
        row, col, count, d_n_entries, h_row + (size_t)t * n_items, h_col + (size_t)t * n_items,
        kappa, h_sign ? h_sign[2 * t] : 1, h_sign ? h_sign[2 * t + 1] : 0, cs != nullptr,
        (unsigned long long*)loads + (size_t)t * kappa, distinct + (size_t)t * kappa,
        cs ? (unsigned long long*)cs + (size_t)t * kappa : nullptr);
    CROP_LAUNCH_CHECK();
    crop_count_launches(1);
  }
  return CROP_OK;
}

__global__ void k_entry_buckets(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                                uint64_t n, const uint32_t* __restrict__ h_row,
                                const uint32_t* __restrict__ h_col, uint32_t kappa,
                                uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = h_row[row[e]] + h_col[col[e]];
    out[e] = b >= kappa ? b - kappa : b;
  }
}

extern "C" int crop_entry_buckets(const uint32_t* row, const uint32_t* col, uint64_t n,
                                  const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                                  uint32_t* out, void* stream) {
  if (n == 0) return CROP_OK;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  k_entry_buckets<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(row, col, n, h_row, h_col,
                                                                   kappa, out);
  CROP_LAUNCH_CHECK();
  crop_count_launches(1);
  return CROP_OK;
}

// Float-weight variant for real-valued streams: per bucket the number of
// entries and the Count-Sketch cell sum weight * s(i, j) (fp64 atomics; the
// summation order differs from the reference's, so cells agree to rounding).
__global__ void k_entry_stats_f64(const uint32_t* __restrict__ row, const uint32_t* __restrict__ col,
                                  const double* __restrict__ w, const uint64_t* __restrict__ d_n,
                                  const uint32_t* __restrict__ h_row,
                                  const uint32_t* __restrict__ h_col, uint32_t kappa,
                                  uint64_t sign_mul, uint64_t sign_add, int do_cs,
                                  uint32_t* __restrict__ distinct, double* __restrict__ cs) {
  const uint64_t n = *d_n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = row[e], j = col[e];
    uint32_t b = h_row[i] + h_col[j];
    if (b >= kappa) b -= kappa;
    atomicAdd(&distinct[b], 1u);
    if (do_cs) atomicAdd(&cs[b], w[e] * (double)sign_of(i, j, sign_mul, sign_add));
  }
}

extern "C" int crop_entry_bucket_stats_f64(const uint32_t* row, const uint32_t* col,
                                           const double* weight, const uint64_t* d_n_entries,
                                           uint64_t max_entries, int instances, uint32_t n_items,
                                           const uint32_t* h_row, const uint32_t* h_col,
                                           uint32_t kappa, const uint64_t* h_sign,
                                           uint32_t* distinct, double* cs, void* stream) {
  if (kappa == 0 || instances < 1) {
    crop_set_error(CROP_ECONFIG, "kappa and instances must be >= 1");
    return CROP_ECONFIG;
  }
  uint64_t blocks = (max_entries + 255) / 256;
  if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
  if (blocks == 0) blocks = 1;
  for (int t = 0; t < instances; ++t) {
    k_entry_stats_f64<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
        row, col, weight, d_n_entries, h_row + (size_t)t * n_items, h_col + (size_t)t * n_items,
        kappa, h_sign ? h_sign[2 * t] : 1, h_sign ? h_sign[2 * t + 1] : 0, cs != nullptr,
        distinct + (size_t)t * kappa, cs ? cs + (size_t)t * kappa : nullptr);
    CROP_LAUNCH_CHECK();
  }
  return CROP_OK;
}

// Per-product worker loads (LoadReport.per_product, engine.py:250-251,
// 287-288): out[k * workers + w] = terms of product k in worker w's interval
// [w*kappa/W, (w+1)*kappa/W). Warp per product, global atomics on the
// product's own row of counters (no cross-product contention).
__global__ void k_product_worker_loads(const int64_t* __restrict__ a_ptr,
                                       const uint32_t* __restrict__ a_idx,
                                       const int64_t* __restrict__ b_ptr,
                                       const uint32_t* __restrict__ b_idx, int64_t n,
                                       const uint32_t* __restrict__ h_row,
                                       const uint32_t* __restrict__ h_col, uint32_t kappa,
                                       uint32_t workers, int upper_only,
                                       uint32_t* __restrict__ out) {
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int64_t k = (int64_t)blockIdx.x * warps + threadIdx.x / 32; k < n;
       k += (int64_t)gridDim.x * warps) {
    const int64_t a0 = a_ptr[k], la = a_ptr[k + 1] - a0;
    const int64_t b0 = b_ptr[k], lb = b_ptr[k + 1] - b0;
    for (int64_t t = lane; t < la * lb; t += 32) {
      const int64_t p = t / lb, q = t - p * lb;
      const uint32_t i = a_idx[a0 + p], j = b_idx[b0 + q];
      if (upper_only && i >= j) continue;
      uint32_t b = h_row[i] + h_col[j];
      if (b >= kappa) b -= kappa;
      // worker w owns [floor(w*kappa/W), floor((w+1)*kappa/W)): w = floor(((b+1)*W - 1)/kappa)
      const uint32_t w = (uint32_t)((((uint64_t)b + 1) * workers - 1) / kappa);
      atomicAdd(&out[k * workers + w], 1u);
    }
  }
}

extern "C" int crop_product_worker_loads(const int64_t* a_ptr, const uint32_t* a_idx,
                                         const int64_t* b_ptr, const uint32_t* b_idx,
                                         int64_t n_products, const uint32_t* h_row,
                                         const uint32_t* h_col, uint32_t kappa, uint32_t workers,
                                         int upper_only, uint32_t* out, void* stream) {
  if (kappa == 0 || workers == 0 || workers > kappa) {
    crop_set_error(CROP_ECONFIG, "need 1 <= workers <= kappa");
    return CROP_ECONFIG;
  }
  if (n_products <= 0) return CROP_OK;
  int64_t blocks = std::min<int64_t>((n_products + 7) / 8, 8 * kNumSMs);
  k_product_worker_loads<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
      a_ptr, a_idx, b_ptr, b_idx, n_products, h_row, h_col, kappa, workers, upper_only, out);
  CROP_LAUNCH_CHECK();
  return CROP_OK;
}
