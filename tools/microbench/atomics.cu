// Microbenchmark: shared-memory and L2/HBM atomic throughput on B200.
// Informs the counter-table design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int TABLE_WORDS>
__global__ void smem_atomic(uint32_t* out, int iters) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t h = mix32(s + it * 0x9E3779B9u);
    atomicAdd(&tab[h % TABLE_WORDS], 1u);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) acc += tab[i];
  atomicAdd(out, acc);
}

template <int TABLE_WORDS>
__global__ void smem_plain(uint32_t* out, int iters) {  // racy ld+st, reference only
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t h = mix32(s + it * 0x9E3779B9u);
    volatile uint32_t* p = &tab[h % TABLE_WORDS];
    *p = *p + 1;
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < TABLE_WORDS; i += blockDim.x) acc += tab[i];
  atomicAdd(out, acc);
}

// skewed: a fraction p of the updates go to H hot slots (Zipf-like hot
// columns of a single-row tile)
__global__ void smem_skew(uint32_t* out, int iters, uint32_t p_thresh, uint32_t hot) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t h = mix32(s + it * 0x9E3779B9u);
    const uint32_t slot = h < p_thresh ? (h >> 8) % hot : h % 32768u;
    atomicAdd(&tab[slot], 1u);
  }
  __syncthreads();
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) acc += tab[i];
  atomicAdd(out, acc);
}

__global__ void mix_only(uint32_t* out, int iters) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
  for (int it = 0; it < iters; ++it) acc += mix32(s + it * 0x9E3779B9u) % 32768u;
  if (acc == 0x12345) out[0] = acc;
}

__global__ void global_red(uint32_t* tab, uint64_t mask, int iters) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint64_t h = mix32(s + it * 0x9E3779B9u) * 0x100000001ull ^ mix32(s * 7 + it);
    atomicAdd(&tab[h & mask], 1u);
  }
}

__global__ void global_cas64(unsigned long long* tab, uint64_t mask, int iters) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint64_t h = mix32(s + it * 0x9E3779B9u) * 0x100000001ull ^ mix32(s * 7 + it);
    unsigned long long* p = &tab[h & mask];
    unsigned long long v = *(volatile unsigned long long*)p;
    atomicCAS(p, v, v + 1);
  }
}

__global__ void copy_k(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint32_t* out; CK(cudaMalloc(&out, 4));
  int sms = 148; float ms;
  const int iters = 4096;
  // smem atomics
  {
    auto k = smem_atomic<32768>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
    for (int threads : {256, 512, 1024}) {
      k<<<sms, threads, 32768 * 4>>>(out, iters);
      cudaEventRecord(e0); k<<<sms, threads, 32768 * 4>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * threads * iters;
      printf("smem_atomic 128KB threads=%d: %.3f ms  %.3e atom/s  %.2f atom/clk/SM@1.9G\n", threads, ms, ops / ms * 1e3, ops / (ms * 1e-3) / sms / 1.9e9);
    }
    CK(cudaFuncSetAttribute(smem_skew, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
    for (double p : {0.0, 0.02, 0.1, 0.3}) {
      for (uint32_t hot : {1u, 4u, 16u, 64u}) {
        const uint32_t th = (uint32_t)(p * 4294967295.0);
        smem_skew<<<sms, 1024, 32768 * 4>>>(out, iters, th, hot);
        cudaEventRecord(e0); smem_skew<<<sms, 1024, 32768 * 4>>>(out, iters, th, hot); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * 1024 * iters;
        printf("smem_skew p=%.2f hot=%u: %.3f ms  %.3e atom/s  %.2f atom/clk/SM\n", p, hot, ms, ops / ms * 1e3, ops / (ms * 1e-3) / sms / 1.9e9);
        if (p == 0.0) break;
      }
    }
    auto k2 = smem_plain<32768>;
    CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
    k2<<<sms, 1024, 32768 * 4>>>(out, iters);
    cudaEventRecord(e0); k2<<<sms, 1024, 32768 * 4>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 1024 * iters;
    printf("smem_plain  128KB: %.3f ms  %.3e op/s\n", ms, ops / ms * 1e3);
    mix_only<<<sms, 1024>>>(out, iters);
    cudaEventRecord(e0); mix_only<<<sms, 1024>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("mix_only: %.3f ms  %.3e op/s\n", ms, ops / ms * 1e3);
  }
  // global red at several table sizes
  for (size_t words : {(size_t)1 << 20, (size_t)1 << 23, (size_t)1 << 24, (size_t)1 << 26, (size_t)1 << 28}) {
    uint32_t* tab; CK(cudaMalloc(&tab, words * 4)); cudaMemset(tab, 0, words * 4);
    int blocks = sms * 8, threads = 256, it = 512;
    global_red<<<blocks, threads>>>(tab, words - 1, it);
    cudaEventRecord(e0); global_red<<<blocks, threads>>>(tab, words - 1, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * it;
    printf("global_red table=%zu MB: %.3f ms  %.3e red/s\n", words * 4 >> 20, ms, ops / ms * 1e3);
    cudaFree(tab);
  }
  for (size_t words : {(size_t)1 << 20, (size_t)1 << 23, (size_t)1 << 26}) {
    unsigned long long* tab; CK(cudaMalloc(&tab, words * 8)); cudaMemset(tab, 0, words * 8);
    int blocks = sms * 8, threads = 256, it = 256;
    global_cas64<<<blocks, threads>>>(tab, words - 1, it);
    cudaEventRecord(e0); global_cas64<<<blocks, threads>>>(tab, words - 1, it); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * it;
    printf("global_ld+cas64 table=%zu MB: %.3f ms  %.3e op/s\n", words * 8 >> 20, ms, ops / ms * 1e3);
    cudaFree(tab);
  }
  {
    size_t n = (size_t)1 << 26;  // 1 GiB of int4
    int4 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 1, n * 16);
    copy_k<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e0); copy_k<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * n * 16 / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
