// common.cuh -- shared device helpers for the CRoP B200 kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/crop_b200.h"

namespace crop {

constexpr uint64_t kP61 = 0x1FFFFFFFFFFFFFFFull;  // 2^61 - 1 (hashing.py:21)
constexpr int kNumSMs = 148;
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;

// (a*b + c) mod 2^61-1, a,c < 2^61, b < 2^64: exact 128-bit product folded
// twice through 2^61 == 1 (mod p). Restates IndexHashFn / SignHashFn
// arithmetic (hashing.py:65-66, 98-100) without big integers.
__host__ __device__ __forceinline__ uint64_t mulmod61(uint64_t a, uint64_t b, uint64_t c) {
#ifdef __CUDA_ARCH__
  uint64_t lo = a * b;
  uint64_t hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  uint64_t lo = (uint64_t)p, hi = (uint64_t)(p >> 64);
#endif
  uint64_t lo2 = lo + c;
  hi += (lo2 < lo);
  // value = hi*2^64 + lo2 ; 2^64 = 8 (mod p); hi < 2^61 so hi<<3 < 2^64
  uint64_t r = (lo2 & kP61) + (lo2 >> 61) + ((hi << 3) & kP61) + (hi >> 58);
  r = (r & kP61) + (r >> 61);
  r = (r & kP61) + (r >> 61);
  if (r >= kP61) r -= kP61;
  return r;
}

__device__ __forceinline__ int sign_of(uint32_t row, uint32_t col, uint64_t mul, uint64_t add) {
  uint64_t packed = ((uint64_t)row << 32) | col;
  return (mulmod61(mul, packed, add) & 1) ? -1 : 1;
}

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Top-k count histogram: exact below 2048, 2^-10 relative resolution above
// (monotone in the count; shared by topk.cu and the counting kernels).
constexpr uint32_t kTopkExactBins = 2048;
constexpr uint32_t kTopkBins = kTopkExactBins + 21 * 1024;  // 23552
__device__ __forceinline__ uint32_t topk_count_bin(uint32_t c) {
  if (c < kTopkExactBins) return c;
  const uint32_t msb = 31 - __clz(c);  // >= 11
  return kTopkExactBins + (msb - 11) * 1024 + ((c >> (msb - 10)) & 1023);
}

}  // namespace crop

// ------------------------------------------------------------------ errors
void crop_set_error(int code, const char* fmt, ...);
// Keep freed device scratch in the stream-ordered pool (no cudaMalloc per job).
int crop_pool_setup();
// Count kernels this library launched (reported by bench.py as gpu_launches).
void crop_count_launches(int n);
// Top-k select (topk.cu); the fused inputs come from the pair engine's counting
// kernels (high-count histogram + entry list), nullptr for the plain path.
int crop_topk_impl(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                   const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k,
                   uint64_t* out_idx, uint64_t* d_k_out, cudaStream_t st, uint32_t* fused_hist,
                   const unsigned long long* hi_list, const unsigned long long* hi_n);

#define CROP_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess) {                                                             \
      crop_set_error(CROP_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                     cudaGetErrorString(_e));                                            \
      return CROP_ECUDA;                                                                 \
    }                                                                                    \
  } while (0)

#define CROP_LAUNCH_CHECK() CROP_CUDA(cudaGetLastError())
