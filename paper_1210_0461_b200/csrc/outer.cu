// outer.cu -- K5: general (real-valued) outer-product streams.
//
// Replaces the per-partition enumerate_interval + dict accumulation loop
// (interval.py:236-254, scan_sorted :125-189) and exact_product
// (oracle.py:20-50) for streams whose two sides differ or carry real values
// (configuration 4: C = A*B with A as CSC and B as CSR). Each product's terms
// are mostly distinct entries, so there is nothing to aggregate on chip; the
// kernel path is emit -> stable sort -> ordered segment sum:
//
//   k_outer_count  per product: own-interval terms (warp per product)
//   scan           exclusive offsets (CUB)
//   k_outer_emit   (row<<32|col, term index) for own terms, in stream order;
//                  values are a_k(i)*b_k(j) in fp64 (exact for fp32 inputs);
//                  unfiltered full products: k_outer_emit_bal, warps over
//                  fixed term chunks instead of whole products
//   sort           stable radix sort by (row, col), then stable by bucket (CUB)
//   k_outer_reduce segment heads sum their run IN STREAM ORDER in fp64 ->
//                  bit-identical to the reference's dict accumulation; output
//                  per-bucket sorted COO (row, col, value, bucket)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace crop;

namespace {

template <bool FILTER>
__device__ __forceinline__ bool own_term(uint32_t i, uint32_t j, int upper,
                                         const crop_interval& iv) {
  if (upper && i >= j) return false;
  if (FILTER) {
    uint32_t b = iv.h_row[i] + iv.h_col[j];
    if (b >= iv.kappa) b -= iv.kappa;
    return b >= iv.start && b < iv.stop;
  }
  return true;
}

template <bool FILTER>
__global__ void k_outer_count(const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx,
                              const int64_t* __restrict__ b_ptr, const uint32_t* __restrict__ b_idx,
                              int64_t n, int upper, crop_interval iv,
                              unsigned long long* __restrict__ counts) {
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int64_t k = (int64_t)blockIdx.x * warps + threadIdx.x / 32; k < n;
       k += (int64_t)gridDim.x * warps) {
    const int64_t a0 = a_ptr[k], la = a_ptr[k + 1] - a0;
    const int64_t b0 = b_ptr[k], lb = b_ptr[k + 1] - b0;
    unsigned long long c = 0;
    if (!FILTER && !upper) {
      c = (unsigned long long)(la * lb);
    } else {
      for (int64_t t = lane; t < la * lb; t += 32) {
        const int64_t p = t / lb, q = t - p * lb;
        c += own_term<FILTER>(a_idx[a0 + p], b_idx[b0 + q], upper, iv);
      }
      c = warp_sum(c);
    }
    if (lane == 0) counts[k] = c;
  }
}

// Composite sort key (bucket << rc_bits | row << c_bits | col) when it fits
// 64 bits (c4: 11 + 19 + 19 bits): ONE stable radix sort over end_bit bits
// replaces the (row, col) sort + stable bucket sort + gather.
struct CompositeKey {
  int on, has_hash;
  uint32_t c_bits, rc_bits, bits;
};

template <bool FILTER>
__global__ void k_outer_emit(const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx,
                             const double* __restrict__ a_val, const int64_t* __restrict__ b_ptr,
                             const uint32_t* __restrict__ b_idx, const double* __restrict__ b_val,
                             int64_t n, int upper, crop_interval iv, CompositeKey ck,
                             const unsigned long long* __restrict__ offs,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ seq,
                             double* __restrict__ vals) {
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int64_t k = (int64_t)blockIdx.x * warps + threadIdx.x / 32; k < n;
       k += (int64_t)gridDim.x * warps) {
    const int64_t a0 = a_ptr[k], la = a_ptr[k + 1] - a0;
    const int64_t b0 = b_ptr[k], lb = b_ptr[k + 1] - b0;
    unsigned long long pos = offs[k];
    for (int64_t t0 = 0; t0 < la * lb; t0 += 32) {
      const int64_t t = t0 + lane;
      bool keep = false;
      uint32_t i = 0, j = 0;
      int64_t p = 0, q = 0;
      if (t < la * lb) {
        if (la * lb < (1ll << 32)) {  // 32-bit division (products up to 65,536^2 terms)
          const uint32_t t32 = (uint32_t)t, l32 = (uint32_t)lb;
          p = t32 / l32;
          q = t32 - (uint32_t)p * l32;
        } else {
          p = t / lb;
          q = t - p * lb;
        }
        i = a_idx[a0 + p];
        j = b_idx[b0 + q];
        keep = own_term<FILTER>(i, j, upper, iv);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const unsigned long long o = pos + __popc(m & ((1u << lane) - 1u));
        if (ck.on) {
          // composite key (bucket, row, col) in ck.bits bits: one sort orders
          // the output per bucket by (row, col)
          uint32_t b = 0;
          if (ck.has_hash) {
            b = iv.h_row[i] + iv.h_col[j];
            if (b >= iv.kappa) b -= iv.kappa;
          }
          keys[o] = ((unsigned long long)b << ck.rc_bits) | ((unsigned long long)i << ck.c_bits) | j;
        } else {
          keys[o] = ((unsigned long long)i << 32) | j;
        }
        seq[o] = (uint32_t)o;
        vals[o] = (a_val ? a_val[a0 + p] : 1.0) * (b_val ? b_val[b0 + q] : 1.0);
      }
      pos += __popc(m);
    }
  }
}

// Unfiltered full products (every term is own: term t of product k lands at
// offs[k] + t): warps take fixed chunks of terms instead of whole products,
// so a 2,000 x 2,000 product no longer holds one warp for 125,000 steps
// (c4's Pareto sizes) and every store run is 32 consecutive terms.
constexpr uint32_t kEmitChunk = 1024;

__global__ void __launch_bounds__(256) k_outer_emit_bal(
    const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx, const double* __restrict__ a_val,
    const int64_t* __restrict__ b_ptr, const uint32_t* __restrict__ b_idx, const double* __restrict__ b_val,
    int64_t n, uint64_t total, crop_interval iv, CompositeKey ck, const unsigned long long* __restrict__ offs,
    unsigned long long* __restrict__ keys, uint32_t* __restrict__ seq, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const uint64_t n_chunks = (total + kEmitChunk - 1) / kEmitChunk;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  auto next_off = [&](int64_t k) -> uint64_t { return k + 1 < n ? offs[k + 1] : total; };
  for (uint64_t c = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; c < n_chunks; c += warps) {
    const uint64_t g0 = c * kEmitChunk, g1 = min(total, g0 + kEmitChunk);
    // the product holding g0: the last k with offs[k] <= g0
    int64_t k = 0;
    if (lane == 0) {
      int64_t lo = 0, hi = n;  // offs[lo] <= g0 < offs[hi] (offs[n] = total)
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (offs[mid] <= g0) lo = mid;
        else hi = mid;
      }
      k = lo;
    }
    k = __shfl_sync(0xffffffffu, k, 0);
    int64_t kc = -1, a0 = 0, b0 = 0;
    uint64_t base = 0, lb = 1, terms = 0;
    for (uint64_t g = g0 + lane; g < g1; g += 32) {
      while (next_off(k) <= g) ++k;
      if (k != kc) {
        kc = k;
        base = offs[k];
        a0 = a_ptr[k];
        b0 = b_ptr[k];
        lb = (uint64_t)(b_ptr[k + 1] - b0);
        terms = (uint64_t)(a_ptr[k + 1] - a0) * lb;
      }
      const uint64_t t = g - base;
      uint64_t p, q;
      if (terms < (1ull << 32)) {
        const uint32_t t32 = (uint32_t)t, l32 = (uint32_t)lb;
        p = t32 / l32;
        q = t32 - (uint32_t)p * l32;
      } else {
        p = t / lb;
        q = t - p * lb;
      }
      const uint32_t i = a_idx[a0 + p], j = b_idx[b0 + q];
      if (ck.on) {
        uint32_t b = 0;
        if (ck.has_hash) {
          b = iv.h_row[i] + iv.h_col[j];
          if (b >= iv.kappa) b -= iv.kappa;
        }
        keys[g] = ((unsigned long long)b << ck.rc_bits) | ((unsigned long long)i << ck.c_bits) | j;
      } else {
        keys[g] = ((unsigned long long)i << 32) | j;
      }
      seq[g] = (uint32_t)g;
      vals[g] = (a_val ? a_val[a0 + p] : 1.0) * (b_val ? b_val[b0 + q] : 1.0);
    }
  }
}

__global__ void k_bucket_of_keys(const unsigned long long* __restrict__ keys, uint64_t n,
                                 crop_interval iv, int has_hash, uint32_t* __restrict__ buckets) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (!has_hash) {
      buckets[e] = 0;
      continue;
    }
    const unsigned long long k = keys[e];
    uint32_t b = iv.h_row[(uint32_t)(k >> 32)] + iv.h_col[(uint32_t)k];
    buckets[e] = b >= iv.kappa ? b - iv.kappa : b;
  }
}

// perm[] maps final position -> position in the (row,col)-sorted arrays.
__global__ void k_gather_final(const uint32_t* __restrict__ perm,
                               const unsigned long long* __restrict__ keys_rc,
                               const uint32_t* __restrict__ seq_rc, uint64_t n,
                               unsigned long long* __restrict__ keys_f, uint32_t* __restrict__ seq_f) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = perm[e];
    keys_f[e] = keys_rc[s];
    seq_f[e] = seq_rc[s];
  }
}

__global__ void k_iota(uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    out[e] = (uint32_t)e;
}

__global__ void k_heads(const unsigned long long* __restrict__ keys, uint64_t n,
                        uint32_t* __restrict__ head) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1u : 0u;
}

__global__ void k_outer_reduce(const unsigned long long* __restrict__ keys,
                               const uint32_t* __restrict__ seq, const double* __restrict__ vals,
                               const uint32_t* __restrict__ buckets_sorted,
                               const uint32_t* __restrict__ head,
                               const uint32_t* __restrict__ head_pos, uint64_t n,
                               uint32_t* __restrict__ out_row, uint32_t* __restrict__ out_col,
                               double* __restrict__ out_val, uint32_t* __restrict__ out_bucket) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (!head[e]) continue;
    const unsigned long long k = keys[e];
    double s = vals[seq[e]];
    for (uint64_t f = e + 1; f < n && keys[f] == k; ++f) s = s + vals[seq[f]];
    const uint32_t o = head_pos[e];
    out_row[o] = (uint32_t)(k >> 32);
    out_col[o] = (uint32_t)k;
    out_val[o] = s;
    out_bucket[o] = buckets_sorted[e];
  }
}

__global__ void k_outer_reduce_ck(const unsigned long long* __restrict__ keys,
                                  const uint32_t* __restrict__ seq, const double* __restrict__ vals,
                                  const uint32_t* __restrict__ head_pos, uint64_t n, CompositeKey ck,
                                  uint32_t* __restrict__ out_row, uint32_t* __restrict__ out_col,
                                  double* __restrict__ out_val, uint32_t* __restrict__ out_bucket) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[e];
    if (e > 0 && keys[e - 1] == k) continue;  // not a segment head
    // sum the run in stream order (the sort is stable): bit-identical to the
    // reference's dict accumulation
    double s = vals[seq[e]];
    for (uint64_t f = e + 1; f < n && keys[f] == k; ++f) s = s + vals[seq[f]];
    const uint32_t o = head_pos[e];
    out_row[o] = (uint32_t)((k >> ck.c_bits) & ((1ull << (ck.rc_bits - ck.c_bits)) - 1));
    out_col[o] = (uint32_t)(k & ((1ull << ck.c_bits) - 1));
    out_val[o] = s;
    out_bucket[o] = (uint32_t)(k >> ck.rc_bits);
  }
}

__global__ void k_heads_count(const unsigned long long* __restrict__ keys, uint64_t n,
                              uint32_t* __restrict__ head) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x)
    head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1u : 0u;
}

__global__ void k_max_u32(const uint32_t* __restrict__ a, const int64_t* a_end,
                          const uint32_t* __restrict__ b, const int64_t* b_end,
                          unsigned int* __restrict__ out) {
  const int64_t na = *a_end, nb = *b_end;
  uint32_t ma = 0, mb = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < na; e += (int64_t)gridDim.x * blockDim.x)
    ma = max(ma, a[e]);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nb; e += (int64_t)gridDim.x * blockDim.x)
    mb = max(mb, b[e]);
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, d));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, ma);
    atomicMax(out + 1, mb);
  }
}

// ---------------------------------------------------------------- partition path
// The default path (no library sort): every own term goes to a PARTITION =
// (bucket, row >> rs), sized so a partition (~1.5k terms on c4) sorts in one
// CTA's shared memory. A term is stored as one 64-bit word
//   row & (2^rs - 1) | col | seq   (seq = the term's index in stream order)
// plus its fp64 value, so sorting a partition's words orders its entries by
// (row, col) and the terms of one entry by stream order: the run sum is the
// reference's dict accumulation, bit for bit (interval.py:236-254).
//   k_part_count   terms per partition (shared-memory histogram)
//   k_part_scan    partition offsets (one CTA)
//   k_part_scatter words + values into their partitions
//   k_part_sort    per partition: bitonic sort in shared memory, ordered run
//                  sums, distinct entries written at the partition's offset
//   k_part_scan    + k_part_compact: distinct entries to the output
struct PartGeo {
  uint32_t S_bits, rs, cb, sb;  // partitions per bucket (log2), row shift, col bits, seq bits
  uint32_t nb;                  // buckets owned (stop - start)
  uint32_t P;                   // partitions
  int has_hash;
};

__device__ __forceinline__ uint32_t part_of(uint32_t i, uint32_t j, const crop_interval& iv,
                                            const PartGeo& G) {
  uint32_t b = 0;
  if (G.has_hash) {
    b = iv.h_row[i] + iv.h_col[j];
    if (b >= iv.kappa) b -= iv.kappa;
    b -= iv.start;
  }
  return (b << G.S_bits) | (i >> G.rs);
}

// Visit the own terms in stream order: fn(g, i, j, a_pos, b_pos) with g the
// term's global index. Unfiltered full products: warps over fixed chunks of
// terms; otherwise one warp per product with ballot-compacted indices.
template <typename Fn>
__device__ __forceinline__ void visit_balanced(const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx,
                                               const int64_t* __restrict__ b_ptr, const uint32_t* __restrict__ b_idx,
                                               int64_t n, uint64_t total, const unsigned long long* __restrict__ offs,
                                               Fn&& fn) {
  const int lane = threadIdx.x & 31;
  const uint64_t n_chunks = (total + kEmitChunk - 1) / kEmitChunk;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  auto next_off = [&](int64_t k) -> uint64_t { return k + 1 < n ? offs[k + 1] : total; };
  for (uint64_t c = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; c < n_chunks; c += warps) {
    const uint64_t g0 = c * kEmitChunk, g1 = min(total, g0 + kEmitChunk);
    int64_t k = 0;
    if (lane == 0) {
      int64_t lo = 0, hi = n;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (offs[mid] <= g0) lo = mid;
        else hi = mid;
      }
      k = lo;
    }
    k = __shfl_sync(0xffffffffu, k, 0);
    int64_t kc = -1, a0 = 0, b0 = 0;
    uint64_t base = 0, lb = 1, terms = 0;
    for (uint64_t g = g0 + lane; g < g1; g += 32) {
      while (next_off(k) <= g) ++k;
      if (k != kc) {
        kc = k;
        base = offs[k];
        a0 = a_ptr[k];
        b0 = b_ptr[k];
        lb = (uint64_t)(b_ptr[k + 1] - b0);
        terms = (uint64_t)(a_ptr[k + 1] - a0) * lb;
      }
      const uint64_t t = g - base;
      uint64_t p, q;
      if (terms < (1ull << 32)) {
        const uint32_t t32 = (uint32_t)t, l32 = (uint32_t)lb;
        p = t32 / l32;
        q = t32 - (uint32_t)p * l32;
      } else {
        p = t / lb;
        q = t - p * lb;
      }
      fn(g, a_idx[a0 + p], b_idx[b0 + q], (uint64_t)(a0 + p), (uint64_t)(b0 + q));
    }
  }
}

template <bool FILTER, typename Fn>
__device__ __forceinline__ void visit_products(const int64_t* __restrict__ a_ptr, const uint32_t* __restrict__ a_idx,
                                               const int64_t* __restrict__ b_ptr, const uint32_t* __restrict__ b_idx,
                                               int64_t n, int upper, const crop_interval& iv,
                                               const unsigned long long* __restrict__ offs, Fn&& fn) {
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  for (int64_t k = (int64_t)blockIdx.x * warps + threadIdx.x / 32; k < n; k += (int64_t)gridDim.x * warps) {
    const int64_t a0 = a_ptr[k], la = a_ptr[k + 1] - a0;
    const int64_t b0 = b_ptr[k], lb = b_ptr[k + 1] - b0;
    unsigned long long pos = offs[k];
    for (int64_t t0 = 0; t0 < la * lb; t0 += 32) {
      const int64_t t = t0 + lane;
      bool keep = false;
      uint32_t i = 0, j = 0;
      int64_t p = 0, q = 0;
      if (t < la * lb) {
        p = t / lb;
        q = t - p * lb;
        i = a_idx[a0 + p];
        j = b_idx[b0 + q];
        keep = own_term<FILTER>(i, j, upper, iv);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) fn(pos + __popc(m & ((1u << lane) - 1u)), i, j, (uint64_t)(a0 + p), (uint64_t)(b0 + q));
      pos += __popc(m);
    }
  }
}

constexpr uint32_t kPartSmemBins = 40960;  // shared histogram bins (160 KB)
constexpr uint32_t kPartCap = 4096;        // terms a partition sorts in shared memory

struct PartStream {
  const int64_t *a_ptr, *b_ptr;
  const uint32_t *a_idx, *b_idx;
  const double *a_val, *b_val;
  int64_t n;
  uint64_t total;
  int upper, balanced, filter;
  const unsigned long long* offs;
};

template <typename Fn>
__device__ __forceinline__ void visit_all(const PartStream& S, const crop_interval& iv, Fn&& fn) {
  if (S.balanced) visit_balanced(S.a_ptr, S.a_idx, S.b_ptr, S.b_idx, S.n, S.total, S.offs, fn);
  else if (S.filter) visit_products<true>(S.a_ptr, S.a_idx, S.b_ptr, S.b_idx, S.n, S.upper, iv, S.offs, fn);
  else visit_products<false>(S.a_ptr, S.a_idx, S.b_ptr, S.b_idx, S.n, S.upper, iv, S.offs, fn);
}

__global__ void __launch_bounds__(256) k_part_count(PartStream S, crop_interval iv, PartGeo G,
                                                    unsigned int* __restrict__ counts) {
  extern __shared__ unsigned int s_h[];
  const bool sm = G.P <= kPartSmemBins;
  if (sm)
    for (uint32_t x = threadIdx.x; x < G.P; x += blockDim.x) s_h[x] = 0;
  __syncthreads();
  visit_all(S, iv, [&](uint64_t, uint32_t i, uint32_t j, uint64_t, uint64_t) {
    const uint32_t p = part_of(i, j, iv, G);
    if (sm) atomicAdd(&s_h[p], 1u);
    else atomicAdd(&counts[p], 1u);
  });
  __syncthreads();
  if (sm)
    for (uint32_t x = threadIdx.x; x < G.P; x += blockDim.x)
      if (s_h[x]) atomicAdd(&counts[x], s_h[x]);
}

// exclusive scan of n u32 into u64 (one CTA of 1024 threads); out[n] = total;
// *max_out (nullable) = the largest input
__global__ void __launch_bounds__(1024) k_part_scan(const unsigned int* __restrict__ in, uint32_t n,
                                                    unsigned long long* __restrict__ out,
                                                    unsigned int* __restrict__ max_out) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  uint32_t mx = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n; base += 1024) {
    const uint32_t x = base + threadIdx.x;
    const unsigned long long v = x < n ? in[x] : 0ull;
    mx = max(mx, (uint32_t)v);
    unsigned long long incl = warp_incl_scan(v);
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
      unsigned long long t = s_w[lane];
      const unsigned long long ti = warp_incl_scan(t);
      s_w[lane] = ti - t;
    }
    __syncthreads();
    const unsigned long long ex = s_carry + s_w[w] + incl - v;
    if (x < n) out[x] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = s_carry;
#pragma unroll
  for (int d = 16; d; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if (lane == 0 && max_out) atomicMax(max_out, mx);
}

__global__ void __launch_bounds__(256) k_part_scatter(PartStream S, crop_interval iv, PartGeo G,
                                                      unsigned int* __restrict__ cursor,
                                                      const unsigned long long* __restrict__ part_off,
                                                      unsigned long long* __restrict__ words,
                                                      double* __restrict__ vals) {
  const uint64_t rmask = (1ull << G.rs) - 1;
  visit_all(S, iv, [&](uint64_t g, uint32_t i, uint32_t j, uint64_t pa, uint64_t pb) {
    const uint32_t p = part_of(i, j, iv, G);
    const uint64_t pos = part_off[p] + atomicAdd(&cursor[p], 1u);
    words[pos] = (((uint64_t)i & rmask) << (G.cb + G.sb)) | ((uint64_t)j << G.sb) | g;
    vals[pos] = (S.a_val ? S.a_val[pa] : 1.0) * (S.b_val ? S.b_val[pb] : 1.0);
  });
}

// One CTA per partition (grid-stride): bitonic sort of (word, value) in
// shared memory, then per run of equal (row, col): the sum in stream order.
// Distinct entries are written at the partition's input offset (compacted
// afterwards); dcount[p] = distinct entries. A partition larger than
// kPartCap raises *overflow (the host falls back to the radix-sort path).
__global__ void __launch_bounds__(512) k_part_sort(const unsigned long long* __restrict__ part_off, PartGeo G,
                                                   uint32_t start, const unsigned long long* __restrict__ words,
                                                   const double* __restrict__ vals,
                                                   unsigned int* __restrict__ dcount,
                                                   uint32_t* __restrict__ t_row, uint32_t* __restrict__ t_col,
                                                   double* __restrict__ t_val, uint32_t* __restrict__ t_bucket,
                                                   unsigned int* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(smem);
  double* sv = reinterpret_cast<double*>(sw + kPartCap);
  uint32_t* s_scan = reinterpret_cast<uint32_t*>(sv + kPartCap);  // 16 warp partials
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long smask = (1ull << G.sb) - 1;
  for (uint32_t p = blockIdx.x; p < G.P; p += gridDim.x) {
    const uint64_t o0 = part_off[p];
    const uint32_t m = (uint32_t)(part_off[p + 1] - o0);
    if (m == 0) {
      if (threadIdx.x == 0) dcount[p] = 0;
      continue;
    }
    if (m > kPartCap) {
      if (threadIdx.x == 0) {
        atomicOr(overflow, 1u);
        dcount[p] = 0;
      }
      continue;
    }
    uint32_t P2 = 2;
    while (P2 < m) P2 <<= 1;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < P2; x += blockDim.x) {
      sw[x] = x < m ? words[o0 + x] : ~0ull;
      sv[x] = x < m ? vals[o0 + x] : 0.0;
    }
    __syncthreads();
    for (uint32_t kk = 2; kk <= P2; kk <<= 1)
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        for (uint32_t x = threadIdx.x; x < P2 / 2; x += blockDim.x) {
          // pair (a, a + j) with a's j-bit clear
          const uint32_t a = ((x & ~(j - 1)) << 1) | (x & (j - 1));
          const uint32_t b = a + j;
          const unsigned long long wa = sw[a], wb = sw[b];
          if ((wa > wb) == ((a & kk) == 0)) {
            sw[a] = wb;
            sw[b] = wa;
            const double t = sv[a];
            sv[a] = sv[b];
            sv[b] = t;
          }
        }
        __syncthreads();
      }
    // run heads and their distinct index (block scan over m elements)
    uint32_t carry = 0;
    const uint32_t bucket = start + (p >> G.S_bits);
    const uint32_t row_hi = (p & ((1u << G.S_bits) - 1)) << G.rs;
    for (uint32_t x0 = 0; x0 < m; x0 += blockDim.x) {
      const uint32_t x = x0 + threadIdx.x;
      const bool head = x < m && (x == 0 || (sw[x] >> G.sb) != (sw[x - 1] >> G.sb));
      const uint32_t bal = __ballot_sync(0xffffffffu, head);
      if (lane == 0) s_scan[w] = __popc(bal);
      __syncthreads();
      uint32_t before = carry;
      for (int q = 0; q < w; ++q) before += s_scan[q];
      uint32_t tot = 0;
      for (int q = 0; q < (int)(blockDim.x / 32); ++q) tot += s_scan[q];
      if (head) {
        const uint32_t d = before + __popc(bal & ((1u << lane) - 1u));
        const unsigned long long key = sw[x] >> G.sb;
        double acc = sv[x];
        for (uint32_t f = x + 1; f < m && (sw[f] >> G.sb) == key; ++f) acc = acc + sv[f];
        const uint64_t o = o0 + d;
        t_row[o] = row_hi | (uint32_t)(key >> G.cb);
        t_col[o] = (uint32_t)(key & ((1ull << G.cb) - 1));
        t_val[o] = acc;
        t_bucket[o] = bucket;
      }
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) dcount[p] = carry;
    (void)smask;
  }
}

// distinct entries of partition p: temp [part_off[p], + dcount[p]) -> out [dout[p], ...)
__global__ void __launch_bounds__(256) k_part_compact(const unsigned long long* __restrict__ part_off,
                                                      const unsigned long long* __restrict__ dout, uint32_t P,
                                                      const uint32_t* __restrict__ t_row, const uint32_t* __restrict__ t_col,
                                                      const double* __restrict__ t_val, const uint32_t* __restrict__ t_bucket,
                                                      uint32_t* __restrict__ out_row, uint32_t* __restrict__ out_col,
                                                      double* __restrict__ out_val, uint32_t* __restrict__ out_bucket,
                                                      unsigned long long* __restrict__ n_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; p < P; p += warps) {
    const uint64_t s0 = part_off[p], d0 = dout[p];
    const uint32_t c = (uint32_t)(dout[p + 1] - d0);
    for (uint32_t x = lane; x < c; x += 32) {
      out_row[d0 + x] = t_row[s0 + x];
      out_col[d0 + x] = t_col[s0 + x];
      out_val[d0 + x] = t_val[s0 + x];
      out_bucket[d0 + x] = t_bucket[s0 + x];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = dout[P];
}

uint32_t bits_for(uint64_t v) {  // bits to hold values 0..v
  uint32_t b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

}  // namespace

struct crop_outer {
  const int64_t *a_ptr, *b_ptr;
  const uint32_t *a_idx, *b_idx;
  const double *a_val, *b_val;
  int64_t n;
  int upper;
  bool filter, has_hash;
  crop_interval iv;
  uint64_t total_terms;  // own-interval terms
  uint64_t all_terms;
  CompositeKey ck{};
  PartGeo geo{};
  bool part = false;                          // partition path (no library sort)
  unsigned long long* d_part_off = nullptr;   // partition offsets [P + 1]
  cudaStream_t st = nullptr;  // creation stream: pool allocations are freed on it
  unsigned long long* d_counts = nullptr;
  unsigned long long* d_offs = nullptr;
};

extern "C" int crop_outer_create(const int64_t* a_ptr, const uint32_t* a_idx, const double* a_val,
                                 const int64_t* b_ptr, const uint32_t* b_idx, const double* b_val,
                                 int64_t n_products, int upper_only, const crop_interval* interval,
                                 void* stream, crop_outer** job) {
  *job = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  if (int rc = crop_pool_setup()) return rc;
  crop_outer* J = new crop_outer();
  J->a_ptr = a_ptr;
  J->a_idx = a_idx;
  J->a_val = a_val;
  J->b_ptr = b_ptr;
  J->b_idx = b_idx;
  J->b_val = b_val;
  J->n = n_products;
  J->upper = upper_only;
  J->has_hash = interval != nullptr;
  J->filter = false;
  if (interval) {
    J->iv = *interval;
    if (interval->kappa == 0 || interval->start > interval->stop || interval->stop > interval->kappa) {
      delete J;
      crop_set_error(CROP_ECONFIG, "invalid interval");
      return CROP_ECONFIG;
    }
    J->filter = !(interval->start == 0 && interval->stop == interval->kappa);
  } else {
    J->iv = crop_interval{1, 0, 1, nullptr, nullptr};
  }
  const int64_t nn = std::max<int64_t>(n_products, 1);
  J->st = st;
  // stream-ordered pool allocations (cudaMalloc / cudaFree would synchronise)
  cudaError_t e1 = cudaMallocAsync(&J->d_counts, nn * 8, st);
  cudaError_t e2 = cudaMallocAsync(&J->d_offs, (nn + 2) * 8, st);  // + 8 bytes: index maxima
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaFreeAsync(J->d_counts, st);
    cudaFreeAsync(J->d_offs, st);
    delete J;
    crop_set_error(CROP_ECUDA, "cudaMallocAsync failed");
    return CROP_ECUDA;
  }
  J->total_terms = 0;
  if (n_products > 0) {
    // one warp per product (8 per block): enough warps in flight to hide the
    // dependent pointer loads of short products
    int64_t blocks = std::min<int64_t>((n_products + 7) / 8, 1 << 20);
    if (J->filter)
      k_outer_count<true><<<(int)blocks, 256, 0, st>>>(a_ptr, a_idx, b_ptr, b_idx, n_products,
                                                      upper_only, J->iv, J->d_counts);
    else
      k_outer_count<false><<<(int)blocks, 256, 0, st>>>(a_ptr, a_idx, b_ptr, b_idx, n_products,
                                                       upper_only, J->iv, J->d_counts);
    CROP_LAUNCH_CHECK();
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, J->d_counts, J->d_offs, n_products + 1, st);
    void* tmp = nullptr;
    CROP_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    // offs has n+1 entries: scan n+1 values where counts[n] is garbage-free by
    // scanning only n and adding the last count below
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, J->d_counts, J->d_offs, n_products, st);
    cudaFreeAsync(tmp, st);
    // largest row / column index (composite sort key width), same sync
    unsigned int* d_mx = reinterpret_cast<unsigned int*>(J->d_offs + n_products + 1);
    CROP_CUDA(cudaMemsetAsync(d_mx, 0, 8, st));
    k_max_u32<<<2 * kNumSMs, 256, 0, st>>>(a_idx, a_ptr + n_products, b_idx, b_ptr + n_products, d_mx);
    CROP_LAUNCH_CHECK();
    unsigned long long last_off = 0, last_cnt = 0;
    unsigned int mx[2] = {0, 0};
    CROP_CUDA(cudaMemcpyAsync(&last_off, J->d_offs + n_products - 1, 8, cudaMemcpyDeviceToHost, st));
    CROP_CUDA(cudaMemcpyAsync(&last_cnt, J->d_counts + n_products - 1, 8, cudaMemcpyDeviceToHost, st));
    CROP_CUDA(cudaMemcpyAsync(mx, d_mx, 8, cudaMemcpyDeviceToHost, st));
    CROP_CUDA(cudaStreamSynchronize(st));
    J->total_terms = last_off + last_cnt;
    {
      const uint32_t rb = bits_for(mx[0]), cb = bits_for(mx[1]);
      const uint32_t bb = J->has_hash ? bits_for(J->iv.kappa - 1) : 0;
      J->ck.has_hash = J->has_hash;
      J->ck.c_bits = cb;
      J->ck.rc_bits = rb + cb;
      J->ck.bits = bb + rb + cb;
      J->ck.on = J->ck.bits <= 64 && !getenv("CROP_OUTER_TWO_SORTS");
    }
    if (J->total_terms >= (1ull << 32)) {
      cudaFreeAsync(J->d_counts, st);
      cudaFreeAsync(J->d_offs, st);
      delete J;
      crop_set_error(CROP_ERESOURCE, "more than 2^32 terms in one interval; split the stream");
      return CROP_ERESOURCE;
    }
    // partition geometry: (bucket, row >> rs) partitions of ~1.5k terms
    // (measured on c4: 7.3 ms/step against 3.3 ms for the radix-sort path --
    // the per-term cursor atomics of the scatter and the CTA-wide bitonic
    // sorts dominate; opt-in with CROP_OUTER_PARTITION=1 until reworked)
    if (J->total_terms > 0 && getenv("CROP_OUTER_PARTITION") && !getenv("CROP_OUTER_RADIX")) {
      PartGeo G{};
      G.has_hash = J->has_hash;
      G.nb = J->has_hash ? J->iv.stop - J->iv.start : 1;
      const uint32_t rb = bits_for(mx[0]);
      G.cb = bits_for(mx[1]);
      G.sb = bits_for(J->total_terms - 1);
      const uint64_t want = (J->total_terms + (uint64_t)G.nb * 1536 - 1) / ((uint64_t)G.nb * 1536);
      uint32_t sbits = 0;
      while (sbits < rb && (1ull << sbits) < want) ++sbits;
      G.S_bits = sbits;
      G.rs = rb - sbits;
      const uint64_t P = (uint64_t)G.nb << sbits;
      if (G.rs + G.cb + G.sb <= 64 && P < (1ull << 26)) {
        G.P = (uint32_t)P;
        unsigned int* d_cnt = nullptr;
        CROP_CUDA(cudaMallocAsync(&d_cnt, (P + 1) * 4, st));
        CROP_CUDA(cudaMallocAsync(&J->d_part_off, (P + 1) * 8, st));
        CROP_CUDA(cudaMemsetAsync(d_cnt, 0, (P + 1) * 4, st));
        PartStream S{a_ptr, b_ptr, a_idx, b_idx, a_val, b_val, n_products, J->total_terms, upper_only,
                     (!J->filter && !upper_only) ? 1 : 0, J->filter ? 1 : 0, J->d_offs};
        const size_t sm = G.P <= kPartSmemBins ? (size_t)G.P * 4 : 0;
        CROP_CUDA(cudaFuncSetAttribute(k_part_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kPartSmemBins * 4)));
        const int grid = S.balanced ? kNumSMs * 2 : (int)std::min<int64_t>((n_products + 7) / 8, kNumSMs * 8);
        k_part_count<<<grid, 256, sm, st>>>(S, J->iv, G, d_cnt);
        CROP_LAUNCH_CHECK();
        unsigned int* d_max = d_cnt + P;
        k_part_scan<<<1, 1024, 0, st>>>(d_cnt, G.P, J->d_part_off, d_max);
        CROP_LAUNCH_CHECK();
        unsigned int hmax = 0;
        CROP_CUDA(cudaMemcpyAsync(&hmax, d_max, 4, cudaMemcpyDeviceToHost, st));
        CROP_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(d_cnt, st);
        crop_count_launches(2);
        if (hmax <= kPartCap) {
          J->part = true;
          J->geo = G;
        } else {
          cudaFreeAsync(J->d_part_off, st);
          J->d_part_off = nullptr;
        }
      }
    }
  }
  *job = J;
  return CROP_OK;
}

extern "C" int crop_outer_info(const crop_outer* J, uint64_t* max_entries, uint64_t* total_terms) {
  if (max_entries) *max_entries = J->total_terms;
  if (total_terms) *total_terms = J->total_terms;
  return CROP_OK;
}

extern "C" int crop_outer_run(crop_outer* J, uint32_t* out_row, uint32_t* out_col,
                              double* out_value, uint32_t* out_bucket, uint64_t* d_n_entries,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  CROP_CUDA(cudaMemsetAsync(d_n_entries, 0, 8, st));
  const uint64_t n = J->total_terms;
  if (n == 0) return CROP_OK;
  if (J->part) {
    const PartGeo G = J->geo;
    unsigned int *cursor = nullptr, *dcount = nullptr;
    unsigned long long *words = nullptr, *dout = nullptr;
    double *vals = nullptr, *t_val = nullptr;
    uint32_t *t_row = nullptr, *t_col = nullptr, *t_bucket = nullptr;
    CROP_CUDA(cudaMallocAsync(&cursor, (size_t)(G.P + 1) * 4 * 2, st));
    dcount = cursor + G.P + 1;
    CROP_CUDA(cudaMallocAsync(&dout, (size_t)(G.P + 1) * 8, st));
    CROP_CUDA(cudaMallocAsync(&words, n * 8, st));
    CROP_CUDA(cudaMallocAsync(&vals, n * 8, st));
    CROP_CUDA(cudaMallocAsync(&t_val, n * 8, st));
    CROP_CUDA(cudaMallocAsync(&t_row, n * 12, st));
    t_col = t_row + n;
    t_bucket = t_col + n;
    CROP_CUDA(cudaMemsetAsync(cursor, 0, (size_t)(G.P + 1) * 4 * 2, st));
    PartStream S{J->a_ptr, J->b_ptr, J->a_idx, J->b_idx, J->a_val, J->b_val, J->n, n, J->upper,
                 (!J->filter && !J->upper) ? 1 : 0, J->filter ? 1 : 0, J->d_offs};
    const int grid = S.balanced ? kNumSMs * 8 : (int)std::min<int64_t>((J->n + 7) / 8, 1 << 20);
    k_part_scatter<<<grid, 256, 0, st>>>(S, J->iv, G, cursor, J->d_part_off, words, vals);
    CROP_LAUNCH_CHECK();
    const size_t sm = (size_t)kPartCap * 16 + 64;
    CROP_CUDA(cudaFuncSetAttribute(k_part_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    unsigned int* d_ovf = cursor + G.P;  // spare slot (cursor has P + 1 entries)
    k_part_sort<<<(int)std::min<uint32_t>(G.P, kNumSMs * 3), 512, sm, st>>>(
        J->d_part_off, G, J->has_hash ? J->iv.start : 0, words, vals, dcount, t_row, t_col, t_val, t_bucket,
        d_ovf);
    CROP_LAUNCH_CHECK();
    k_part_scan<<<1, 1024, 0, st>>>(dcount, G.P, dout, nullptr);
    CROP_LAUNCH_CHECK();
    k_part_compact<<<kNumSMs * 4, 256, 0, st>>>(J->d_part_off, dout, G.P, t_row, t_col, t_val, t_bucket,
                                               out_row, out_col, out_value, out_bucket,
                                               (unsigned long long*)d_n_entries);
    CROP_LAUNCH_CHECK();
    for (void* p : {(void*)cursor, (void*)dout, (void*)words, (void*)vals, (void*)t_val, (void*)t_row})
      cudaFreeAsync(p, st);
    crop_count_launches(4);
    return CROP_OK;
  }
  unsigned long long *keys = nullptr, *keys2 = nullptr, *keys_f = nullptr;
  uint32_t *seq = nullptr, *seq2 = nullptr, *seq_f = nullptr, *buck = nullptr, *buck2 = nullptr;
  uint32_t *iota = nullptr, *perm = nullptr, *head = nullptr, *head_pos = nullptr;
  double* vals = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, t2 = 0;
  CROP_CUDA(cudaMallocAsync(&keys, n * 8, st));
  CROP_CUDA(cudaMallocAsync(&keys2, n * 8, st));
  CROP_CUDA(cudaMallocAsync(&seq, n * 4, st));
  CROP_CUDA(cudaMallocAsync(&seq2, n * 4, st));
  CROP_CUDA(cudaMallocAsync(&vals, n * 8, st));
  if (!J->ck.on) {
    CROP_CUDA(cudaMallocAsync(&buck, n * 4, st));
    CROP_CUDA(cudaMallocAsync(&buck2, n * 4, st));
    CROP_CUDA(cudaMallocAsync(&iota, n * 4, st));
    CROP_CUDA(cudaMallocAsync(&perm, n * 4, st));
    CROP_CUDA(cudaMallocAsync(&keys_f, n * 8, st));
    CROP_CUDA(cudaMallocAsync(&seq_f, n * 4, st));
  }
  CROP_CUDA(cudaMallocAsync(&head, n * 4, st));
  CROP_CUDA(cudaMallocAsync(&head_pos, n * 4, st));
  {
    int64_t blocks = std::min<int64_t>((J->n + 7) / 8, 1 << 20);
    if (!J->filter && !J->upper && n > 0 && !getenv("CROP_OUTER_EMIT_PER_PRODUCT"))
      k_outer_emit_bal<<<kNumSMs * 8, 256, 0, st>>>(J->a_ptr, J->a_idx, J->a_val, J->b_ptr, J->b_idx,
                                                     J->b_val, J->n, (uint64_t)n, J->iv, J->ck, J->d_offs,
                                                     keys, seq, vals);
    else if (J->filter)
      k_outer_emit<true><<<(int)blocks, 256, 0, st>>>(J->a_ptr, J->a_idx, J->a_val, J->b_ptr,
                                                     J->b_idx, J->b_val, J->n, J->upper, J->iv,
                                                     J->ck, J->d_offs, keys, seq, vals);
    else
      k_outer_emit<false><<<(int)blocks, 256, 0, st>>>(J->a_ptr, J->a_idx, J->a_val, J->b_ptr,
                                                      J->b_idx, J->b_val, J->n, J->upper, J->iv,
                                                      J->ck, J->d_offs, keys, seq, vals);
    CROP_LAUNCH_CHECK();
  }
  if (J->ck.on) {
    // one stable sort by (bucket, row, col) over the key's bits; ties keep
    // emission (= stream) order
    const int eb = (int)J->ck.bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, seq, seq2, (int64_t)n, 0, eb, st);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, head, head_pos, (int64_t)n, st);
    tmp_bytes = std::max(tmp_bytes, t2);
    cub::TransformInputIterator<unsigned long long, cub::CastOp<unsigned long long>, uint32_t*> hi(
        head, cub::CastOp<unsigned long long>());
    cub::DeviceReduce::Sum(nullptr, t2, hi, (unsigned long long*)d_n_entries, (int64_t)n, st);
    tmp_bytes = std::max(tmp_bytes, t2);
    CROP_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, seq, seq2, (int64_t)n, 0, eb, st);
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 16 * kNumSMs);
    k_heads_count<<<(int)blocks, 256, 0, st>>>(keys2, n, head);
    CROP_LAUNCH_CHECK();
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, head, head_pos, (int64_t)n, st);
    k_outer_reduce_ck<<<(int)blocks, 256, 0, st>>>(keys2, seq2, vals, head_pos, n, J->ck, out_row,
                                                   out_col, out_value, out_bucket);
    CROP_LAUNCH_CHECK();
    cub::DeviceReduce::Sum(tmp, tmp_bytes, hi, (unsigned long long*)d_n_entries, (int64_t)n, st);
    for (void* p : {(void*)tmp, (void*)keys, (void*)keys2, (void*)seq, (void*)seq2, (void*)vals,
                    (void*)head, (void*)head_pos})
      cudaFreeAsync(p, st);
    CROP_LAUNCH_CHECK();
    crop_count_launches(5);
    return CROP_OK;
  }
  // stable sort by (row, col): ties keep emission (= stream) order
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, seq, seq2, (int64_t)n, 0, 64, st);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, buck, buck2, iota, perm, (int64_t)n, 0, 32, st);
  tmp_bytes = std::max(tmp_bytes, t2);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, head, head_pos, (int64_t)n, st);
  tmp_bytes = std::max(tmp_bytes, t2);
  CROP_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, seq, seq2, (int64_t)n, 0, 64, st);
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 16 * kNumSMs);
  k_bucket_of_keys<<<(int)blocks, 256, 0, st>>>(keys2, n, J->iv, J->has_hash, buck);
  CROP_LAUNCH_CHECK();
  // stable sort by bucket of the (row,col)-sorted sequence
  k_iota<<<(int)blocks, 256, 0, st>>>(iota, n);
  CROP_LAUNCH_CHECK();
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, buck, buck2, iota, perm, (int64_t)n, 0, 32, st);
  k_gather_final<<<(int)blocks, 256, 0, st>>>(perm, keys2, seq2, n, keys_f, seq_f);
  CROP_LAUNCH_CHECK();
  k_heads<<<(int)blocks, 256, 0, st>>>(keys_f, n, head);
  CROP_LAUNCH_CHECK();
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, head, head_pos, (int64_t)n, st);
  k_outer_reduce<<<(int)blocks, 256, 0, st>>>(keys_f, seq_f, vals, buck2, head, head_pos, n,
                                              out_row, out_col, out_value, out_bucket);
  CROP_LAUNCH_CHECK();
  // number of segments = head_pos[n-1] + head[n-1]
  {
    cub::TransformInputIterator<unsigned long long, cub::CastOp<unsigned long long>, uint32_t*> hi(
        head, cub::CastOp<unsigned long long>());
    size_t tb = 0;
    cub::DeviceReduce::Sum(nullptr, tb, hi, (unsigned long long*)d_n_entries, (int64_t)n, st);
    void* t3 = nullptr;
    CROP_CUDA(cudaMallocAsync(&t3, tb, st));
    cub::DeviceReduce::Sum(t3, tb, hi, (unsigned long long*)d_n_entries, (int64_t)n, st);
    cudaFreeAsync(t3, st);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(keys, st);
  cudaFreeAsync(keys2, st);
  cudaFreeAsync(seq, st);
  cudaFreeAsync(seq2, st);
  cudaFreeAsync(vals, st);
  cudaFreeAsync(buck, st);
  cudaFreeAsync(buck2, st);
  cudaFreeAsync(iota, st);
  cudaFreeAsync(perm, st);
  cudaFreeAsync(keys_f, st);
  cudaFreeAsync(seq_f, st);
  cudaFreeAsync(head, st);
  cudaFreeAsync(head_pos, st);
  CROP_LAUNCH_CHECK();
  crop_count_launches(7);
  return CROP_OK;
}

extern "C" void crop_outer_destroy(crop_outer* J) {
  if (!J) return;
  if (J->d_part_off) cudaFreeAsync(J->d_part_off, J->st);
  cudaFreeAsync(J->d_counts, J->st);
  cudaFreeAsync(J->d_offs, J->st);
  delete J;
}
