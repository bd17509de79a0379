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

// ---------------------------------------------------------------- own scans
// Exclusive scan of n values into u64 out[0..n], out[n] = total, in three
// launches (tile sums, one CTA over the tile sums, tile scans + offsets);
// optional max of the values. Replaces the library scan of the create step.
constexpr int kScanThreads = 1024, kScanPer = 8;
constexpr uint32_t kScanTile = kScanThreads * kScanPer;

struct TermsOf {  // all terms of product k: |a_k| * |b_k|
  const int64_t *a, *b;
  __device__ __forceinline__ unsigned long long operator()(uint64_t k) const {
    return (unsigned long long)(a[k + 1] - a[k]) * (unsigned long long)(b[k + 1] - b[k]);
  }
};
struct LoadU64 {
  const unsigned long long* p;
  __device__ __forceinline__ unsigned long long operator()(uint64_t k) const { return p[k]; }
};
struct LoadU32 {
  const unsigned int* p;
  __device__ __forceinline__ unsigned long long operator()(uint64_t k) const { return p[k]; }
};

// block-wide exclusive scan of one u64 per thread; *total = the block sum
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* s_w,
                                                              unsigned long long* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned long long incl = warp_incl_scan(v);
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    const unsigned long long t = lane < nw ? s_w[lane] : 0ull;
    const unsigned long long ti = warp_incl_scan(t);
    s_w[lane] = ti - t;
    if (lane == 31) s_w[32] = ti;
  }
  __syncthreads();
  const unsigned long long ex = s_w[w] + incl - v;
  *total = s_w[32];
  __syncthreads();
  return ex;
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(F f, uint64_t n, unsigned long long* __restrict__ tile_sum,
                                                             unsigned int* __restrict__ mx) {
  __shared__ unsigned long long s_w[33];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPer;
  unsigned long long s = 0, m = 0;
#pragma unroll
  for (int u = 0; u < kScanPer; ++u)
    if (b0 + u < n) {
      const unsigned long long v = f(b0 + u);
      s += v;
      m = max(m, v);
    }
  unsigned long long tot;
  block_excl_scan(s, s_w, &tot);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
  if (mx) {
#pragma unroll
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, (unsigned int)m);
  }
}

// one CTA: exclusive scan of the tile sums in place; tile_sum[n_tiles] = total
__global__ void __launch_bounds__(kScanThreads) k_scan_top(unsigned long long* __restrict__ tile_sum, uint32_t n_tiles) {
  __shared__ unsigned long long s_w[33];
  unsigned long long carry = 0;
  for (uint32_t base = 0; base < n_tiles; base += kScanThreads) {
    const uint32_t x = base + threadIdx.x;
    const unsigned long long v = x < n_tiles ? tile_sum[x] : 0ull;
    unsigned long long tot;
    const unsigned long long ex = block_excl_scan(v, s_w, &tot);
    if (x < n_tiles) tile_sum[x] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) tile_sum[n_tiles] = carry;
}

template <class F>
__global__ void __launch_bounds__(kScanThreads) k_scan_out(F f, uint64_t n, const unsigned long long* __restrict__ tile_off,
                                                           unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_w[33];
  const uint64_t b0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanPer;
  unsigned long long v[kScanPer], s = 0;
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    v[u] = b0 + u < n ? f(b0 + u) : 0ull;
    s += v[u];
  }
  unsigned long long tot;
  unsigned long long run = tile_off[blockIdx.x] + block_excl_scan(s, s_w, &tot);
#pragma unroll
  for (int u = 0; u < kScanPer; ++u)
    if (b0 + u < n) {
      out[b0 + u] = run;
      run += v[u];
    }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_off[gridDim.x];
}

template <class F>
int scan_excl(F f, uint64_t n, unsigned long long* out, unsigned int* mx, cudaStream_t st) {
  const uint32_t tiles = (uint32_t)std::max<uint64_t>(1, (n + kScanTile - 1) / kScanTile);
  unsigned long long* ts = nullptr;
  CROP_CUDA(cudaMallocAsync(&ts, (tiles + 1) * 8ull, st));
  k_scan_tiles<<<tiles, kScanThreads, 0, st>>>(f, n, ts, mx);
  k_scan_top<<<1, kScanThreads, 0, st>>>(ts, tiles);
  k_scan_out<<<tiles, kScanThreads, 0, st>>>(f, n, ts, out);
  cudaFreeAsync(ts, st);
  CROP_LAUNCH_CHECK();
  crop_count_launches(3);
  return CROP_OK;
}

// ---------------------------------------------------------------- bucket-major path
// The default path (no library sort). Every own term of the interval goes to
// a PARTITION p = (bucket - start) << S_bits | c >> shift, with c = row << cb
// | col the composite key, so the partitions of one bucket are consecutive
// ranges of the output order (row, col). Partitions are grouped: a GROUP is
// 2^gspan consecutive partitions of one bucket (c4: a group is a bucket). A
// term travels as one 64-bit word
//   (c mod 2^(shift + gspan)) << sb | g      (g = its index in stream order)
// plus its fp64 value a_k(i) * b_k(j), so sorting a partition's words orders
// its entries by (row, col) and the terms of one entry by stream order.
//   k_nnz_hash    h_row / h_col of every nonzero (one gather per nnz, not per term)
//   k_bm_hist     per CTA over its fixed range of terms: terms per partition
//                 (shared-memory histogram) -> global partition totals, and
//                 terms per group -> a per-CTA table, stored group-major
//   k_bm_colscan  per group: each CTA's exclusive slot offset
//   scan          partition offsets and the largest partition
//   k_bm_scatter  per CTA: words + values into the CTA's own slot range of
//                 each group (shared-memory cursors, no global atomics; about
//                 1,000 groups keep every CTA's write runs long and the write
//                 frontier L2-resident)
//   k_bm_split    one CTA per group: into the group's partitions (shared-
//                 memory cursors, 2^gspan write frontiers per CTA)
//   k_bm_sort     one CTA per partition, partitions taken in ticket order:
//                 counting sort by a 2,048-bin prefix of the local key, rank
//                 sort inside each bin, run heads sum their terms in stream
//                 order (the reference's dict accumulation, bit for bit),
//                 output offsets by decoupled look-back over the partitions.
//                 A partition larger than shared memory (one (row, col) range
//                 holding > kBmCap terms) sorts in global memory with a
//                 stable in-CTA LSD radix sort.
struct BmStream {
  const int64_t *a_ptr, *b_ptr;
  const uint32_t *a_idx, *b_idx;
  const double *a_val, *b_val;
  const uint32_t *ha, *hb;          // h_row(a_idx), h_col(b_idx) per nonzero (nullptr: one bucket)
  const unsigned long long* offs;   // all terms before product k, [n + 1]
  int64_t n;
  uint64_t total;                   // all terms (every bucket, both triangles)
};

struct BmGeo {
  uint32_t kappa, start;            // buckets; first owned bucket
  uint32_t nb;                      // owned buckets
  uint32_t cb, sb;                  // column bits; stream-index bits
  uint32_t shift, S_bits;           // partition = local bucket << S_bits | c >> shift
  uint32_t gspan;                   // partitions per group = 2^gspan (group = partition >> gspan)
  uint32_t bin_shift;               // sort bin = (c mod 2^shift) >> bin_shift
  uint32_t P, P1;                   // partitions, groups
  int has_hash, upper, filter;
};

constexpr uint32_t kBmGroup = 128;          // terms per warp step (4 per lane)
constexpr uint32_t kBmSmemParts = 40960;    // partitions a shared-memory histogram holds
constexpr uint32_t kBmGroupsTarget = 1024;  // groups the geometry aims at
constexpr uint32_t kBmCap = 5120;           // terms a partition sorts in shared memory
constexpr uint32_t kBmBins = 2048;          // counting-sort bins of a partition's local key
constexpr uint32_t kBmTarget = 2048;        // mean terms per partition the geometry aims at
constexpr int kBmThreads = 1024;            // enumeration kernels: one CTA per SM
constexpr int kBmSortThreads = 512;         // sort: two CTAs per SM (one loads while one sorts)

// last product k with offs[k] <= g, searching forward from k0 (offs[k0] <= g < offs[n])
__device__ __forceinline__ int64_t bm_product(const unsigned long long* __restrict__ offs, int64_t n, int64_t k0,
                                              uint64_t g) {
  int64_t lo = k0, step = 1;
  while (lo + step < n && offs[lo + step] <= g) {
    lo += step;
    step <<= 1;
  }
  int64_t hi = min(lo + step, n);
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (offs[mid] <= g) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Visit the own terms of this CTA's fixed range of 128-term groups:
// fn(partition, word, value). Each lane takes 4 consecutive terms; their
// positions are resolved first, then all loads are issued together.
template <bool VAL, typename Fn>
__device__ __forceinline__ void bm_visit(const BmStream& S, const BmGeo& G, uint32_t cta, uint32_t n_cta, Fn&& fn) {
  // the CTA's groups [gb, ge), each warp a contiguous sub-range of them, so
  // the warp's product cursor only moves forward by a few products per step
  const uint64_t n_groups = (S.total + kBmGroup - 1) / kBmGroup;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t cb_ = n_groups * cta / n_cta, ce_ = n_groups * (cta + 1) / n_cta;
  const uint64_t gb = cb_ + (ce_ - cb_) * warp / nw, ge = cb_ + (ce_ - cb_) * (warp + 1) / nw;
  if (gb >= ge) return;
  int64_t kw = bm_product(S.offs, S.n, 0, gb * kBmGroup);
  const uint32_t wbits = G.shift + G.gspan;
  const uint64_t wmask = wbits >= 64 ? ~0ull : ((1ull << wbits) - 1);
  for (uint64_t gr = gb; gr < ge; ++gr) {
    const uint64_t g0 = gr * kBmGroup + (uint64_t)lane * 4;
    int64_t pa[4], pb[4];
    bool ok[4];
    int64_t k = g0 < S.total ? bm_product(S.offs, S.n, kw, g0) : kw;
    int64_t kc = -1, a0 = 0, b0 = 0;
    uint32_t lb = 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t g = g0 + u;
      ok[u] = g < S.total;
      pa[u] = pb[u] = 0;
      if (ok[u]) {
        while (S.offs[k + 1] <= g) ++k;
        if (k != kc) {
          kc = k;
          a0 = S.a_ptr[k];
          b0 = S.b_ptr[k];
          lb = (uint32_t)(S.b_ptr[k + 1] - b0);
        }
        const uint64_t t = g - S.offs[k];
        uint64_t p, q;
        if (t < (1ull << 32)) {
          const uint32_t t32 = (uint32_t)t;
          p = t32 / lb;
          q = t32 - (uint32_t)p * lb;
        } else {
          p = t / lb;
          q = t - p * lb;
        }
        pa[u] = a0 + (int64_t)p;
        pb[u] = b0 + (int64_t)q;
      }
    }
    kw = __shfl_sync(0xffffffffu, k, 31);
    uint32_t ii[4], jj[4], hi[4], hj[4];
    double va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ii[u] = ok[u] ? S.a_idx[pa[u]] : 0u;
      jj[u] = ok[u] ? S.b_idx[pb[u]] : 0u;
      hi[u] = (ok[u] && S.ha) ? S.ha[pa[u]] : 0u;
      hj[u] = (ok[u] && S.hb) ? S.hb[pb[u]] : 0u;
      if (VAL) {
        va[u] = (ok[u] && S.a_val) ? S.a_val[pa[u]] : 1.0;
        vb[u] = (ok[u] && S.b_val) ? S.b_val[pb[u]] : 1.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!ok[u]) continue;
      if (G.upper && ii[u] >= jj[u]) continue;
      uint32_t b = hi[u] + hj[u];
      if (b >= G.kappa) b -= G.kappa;
      if (G.filter && (b < G.start || b >= G.start + G.nb)) continue;
      const uint64_t c = ((uint64_t)ii[u] << G.cb) | jj[u];
      const uint32_t part = ((b - G.start) << G.S_bits) | (uint32_t)(c >> G.shift);
      const unsigned long long word = ((c & wmask) << G.sb) | (g0 + u);
      fn(part, word, VAL ? va[u] * vb[u] : 0.0);
    }
  }
}

__global__ void k_nnz_hash(const uint32_t* __restrict__ idx, uint64_t n, const uint32_t* __restrict__ table,
                           uint32_t* __restrict__ out) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
    out[e] = table[idx[e]];
}

// gtab[group][cta] = the CTA's terms per group; ptot[p] += terms per partition
__global__ void __launch_bounds__(kBmThreads) k_bm_hist(BmStream S, BmGeo G, unsigned int* __restrict__ gtab,
                                                        unsigned int* __restrict__ ptot) {
  extern __shared__ unsigned int s_h[];
  const bool sm = G.P <= kBmSmemParts;
  const uint32_t n_cta = gridDim.x, cta = blockIdx.x;
  if (sm)
    for (uint32_t x = threadIdx.x; x < G.P; x += blockDim.x) s_h[x] = 0;
  __syncthreads();
  bm_visit<false>(S, G, cta, n_cta, [&](uint32_t p, unsigned long long, double) {
    if (sm) {
      atomicAdd(&s_h[p], 1u);
    } else {
      atomicAdd(&ptot[p], 1u);
      atomicAdd(&gtab[(uint64_t)(p >> G.gspan) * n_cta + cta], 1u);
    }
  });
  __syncthreads();
  if (!sm) return;
  for (uint32_t x = threadIdx.x; x < G.P; x += blockDim.x)
    if (s_h[x]) atomicAdd(&ptot[x], s_h[x]);
  const uint32_t span = 1u << G.gspan;
  for (uint32_t gi = threadIdx.x; gi < G.P1; gi += blockDim.x) {
    unsigned int s = 0;
    for (uint32_t x = 0; x < span; ++x) s += s_h[gi * span + x];
    gtab[(uint64_t)gi * n_cta + cta] = s;
  }
}

// warp per group: exclusive scan over the CTAs in place
__global__ void k_bm_colscan(unsigned int* __restrict__ gtab, uint32_t P1, uint32_t n_cta) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t gi = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; gi < P1; gi += warps) {
    unsigned int* h = gtab + (uint64_t)gi * n_cta;
    unsigned int carry = 0;
    for (uint32_t c0 = 0; c0 < n_cta; c0 += 32) {
      const uint32_t c = c0 + lane;
      const unsigned int v = c < n_cta ? h[c] : 0u;
      const unsigned int incl = warp_incl_scan(v);
      if (c < n_cta) h[c] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

__global__ void __launch_bounds__(kBmThreads) k_bm_scatter(BmStream S, BmGeo G, unsigned int* __restrict__ gtab,
                                                           const unsigned long long* __restrict__ part_off,
                                                           ulonglong2* __restrict__ terms) {
  extern __shared__ unsigned int s_c[];
  const bool sm = G.P1 <= kBmSmemParts;
  for (uint32_t gi = threadIdx.x; gi < G.P1; gi += blockDim.x) {
    const uint64_t i = (uint64_t)gi * gridDim.x + blockIdx.x;
    const unsigned int c = (unsigned int)part_off[(uint64_t)gi << G.gspan] + gtab[i];
    if (sm) s_c[gi] = c;
    else gtab[i] = c;
  }
  __syncthreads();
  bm_visit<true>(S, G, blockIdx.x, gridDim.x, [&](uint32_t p, unsigned long long w, double v) {
    const uint32_t gi = p >> G.gspan;
    const unsigned int pos = sm ? atomicAdd(&s_c[gi], 1u) : atomicAdd(&gtab[(uint64_t)gi * gridDim.x + blockIdx.x], 1u);
    terms[pos] = make_ulonglong2(w, (unsigned long long)__double_as_longlong(v));
  });
}

// one CTA per group (grid-stride): the group's terms into its partitions
__global__ void __launch_bounds__(kBmThreads) k_bm_split(BmGeo G, const unsigned long long* __restrict__ part_off,
                                                         const ulonglong2* __restrict__ t_in,
                                                         ulonglong2* __restrict__ t_out) {
  extern __shared__ unsigned int s_c[];
  const uint32_t span = 1u << G.gspan, smask = span - 1, sh = G.sb + G.shift;
  for (uint32_t gi = blockIdx.x; gi < G.P1; gi += gridDim.x) {
    const uint64_t p0 = (uint64_t)gi << G.gspan;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < span; x += blockDim.x) s_c[x] = (unsigned int)part_off[p0 + x];
    __syncthreads();
    const uint64_t e0 = part_off[p0], e1 = part_off[p0 + span];
    for (uint64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const ulonglong2 t = t_in[e];
      const unsigned int pos = atomicAdd(&s_c[(uint32_t)(t.x >> sh) & smask], 1u);
      t_out[pos] = t;
    }
  }
}

struct BmOut {
  uint32_t *row, *col, *bucket;
  double* val;
  unsigned long long* n_out;
};

// Decoupled look-back over the partitions (taken in ticket order, so every
// predecessor is running or done): publish the aggregate, then every thread
// of the CTA reads one predecessor's status word (a CTA's worth of
// predecessors per round: about one CTA per SM is in flight, so the nearest
// inclusive prefix is usually within one round), the nearest inclusive
// prefix is found with a block minimum and the aggregates up to it summed,
// then the prefix is published. Called by the whole CTA.
__device__ unsigned long long bm_lookback(unsigned long long* status, uint32_t p, unsigned long long agg,
                                          unsigned long long* s_w, unsigned long long* s_red) {
  constexpr unsigned long long AGG = 1ull << 62, INC = 2ull << 62, VAL = (1ull << 62) - 1;
  volatile unsigned long long* vs = status;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) vs[p] = (p == 0 ? INC : AGG) | agg;
  if (p == 0) return 0;
  unsigned long long excl = 0;
  int64_t top = (int64_t)p - 1;
  for (;;) {
    const int64_t q = top - threadIdx.x;
    unsigned long long sv = q >= 0 ? vs[q] : INC;  // before partition 0: prefix 0
    while ((sv >> 62) == 0) sv = vs[q];
    // nearest inclusive prefix = the smallest thread index holding one
    unsigned int near = (sv >> 62) == 2 ? threadIdx.x : 0xFFFFFFFFu;
#pragma unroll
    for (int d = 16; d; d >>= 1) near = min(near, __shfl_xor_sync(0xffffffffu, near, d));
    if (lane == 0) s_red[warp] = near;
    __syncthreads();
    near = 0xFFFFFFFFu;
    for (int w = 0; w < nw; ++w) near = min(near, (unsigned int)s_red[w]);
    unsigned long long tot;
    block_excl_scan(threadIdx.x <= near ? (sv & VAL) : 0ull, s_w, &tot);
    excl += tot;
    if (near != 0xFFFFFFFFu) break;
    top -= blockDim.x;
  }
  if (threadIdx.x == 0) vs[p] = INC | (excl + agg);
  return excl;
}

// Heads of the sorted runs, output offsets and ordered run sums for one
// partition of m sorted terms (key(q), val(q) in sorted order). Warp w owns
// the contiguous positions [w*C, (w+1)*C) and walks them 32 at a time: a
// ballot finds the run heads, popc ranks them, one head lane sums its run.
template <class K, class V>
__device__ __forceinline__ void bm_emit(uint32_t p, uint32_t m, const BmGeo& G, K key, V val,
                                        unsigned long long* status, const BmOut& O, unsigned long long* s_w,
                                        unsigned long long* s_excl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t C = (m + nw - 1) / nw;
  const uint32_t q0 = min(m, warp * C), q1 = min(m, q0 + C);
  auto ent = [&](uint32_t q) { return key(q) >> G.sb; };
  unsigned int heads = 0;
  for (uint32_t b = q0; b < q1; b += 32) {
    const uint32_t q = b + lane;
    const bool h = q < q1 && (q == 0 || ent(q) != ent(q - 1));
    heads += __popc(__ballot_sync(0xffffffffu, h));
  }
  unsigned long long D;
  const unsigned long long d_w = block_excl_scan(lane == 0 ? heads : 0u, s_w, &D);
  const unsigned long long ex = bm_lookback(status, p, D, s_w, s_excl + 1);
  if (threadIdx.x == 0 && p == G.P - 1) *O.n_out = ex + D;
  unsigned long long d = ex + __shfl_sync(0xffffffffu, d_w, 0);
  const uint32_t bucket = G.start + (p >> G.S_bits);
  const uint64_t c_hi = (uint64_t)(p & ((1u << G.S_bits) - 1)) << G.shift;
  const uint64_t lmask = (1ull << G.shift) - 1;
  for (uint32_t b = q0; b < q1; b += 32) {
    const uint32_t q = b + lane;
    unsigned long long e = 0;
    bool h = false;
    if (q < q1) {
      e = ent(q);
      h = q == 0 || e != ent(q - 1);
    }
    const uint32_t hm = __ballot_sync(0xffffffffu, h);
    if (h) {
      double acc = val(q);
      for (uint32_t f = q + 1; f < m && ent(f) == e; ++f) acc = acc + val(f);
      const uint64_t c = c_hi | (e & lmask);
      const unsigned long long o = d + __popc(hm & ((1u << lane) - 1u));
      O.row[o] = (uint32_t)(c >> G.cb);
      O.col[o] = (uint32_t)(c & ((1ull << G.cb) - 1));
      O.val[o] = acc;
      O.bucket[o] = bucket;
    }
    d += __popc(hm);
  }
  __syncthreads();
}

// Stable LSD radix sort (8-bit digits) of one partition in global memory by
// one CTA; returns 1 when the result ended in the scratch arrays.
__device__ int bm_sort_global(ulonglong2* k0, ulonglong2* k1, uint32_t m,
                              uint32_t bits, unsigned int* s_base, unsigned int* s_wc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int flip = 0;
  for (uint32_t bit = 0; bit < bits; bit += 8) {
    for (uint32_t x = threadIdx.x; x < 256; x += blockDim.x) s_base[x] = 0;
    for (uint32_t x = threadIdx.x; x < 256u * nw; x += blockDim.x) s_wc[x] = 0;
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) atomicAdd(&s_base[(k0[x].x >> bit) & 255], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned int carry = 0;
      for (int c0 = 0; c0 < 256; c0 += 32) {
        const unsigned int v = s_base[c0 + lane];
        const unsigned int incl = warp_incl_scan(v);
        s_base[c0 + lane] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    __syncthreads();
    for (uint32_t t0 = 0; t0 < m; t0 += blockDim.x) {
      const uint32_t x = t0 + threadIdx.x;
      const bool valid = x < m;
      const ulonglong2 tx = valid ? k0[x] : make_ulonglong2(0ull, 0ull);
      const unsigned long long kx = tx.x;
      const uint32_t dg = valid ? (uint32_t)((kx >> bit) & 255) : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      const uint32_t lt = __popc(peers & ((1u << lane) - 1u));
      if (valid && lane == __ffs(peers) - 1) s_wc[warp * 256 + dg] = __popc(peers);
      __syncthreads();
      if (valid) {
        unsigned int off = s_base[dg] + lt;
        for (int w2 = 0; w2 < warp; ++w2) off += s_wc[w2 * 256 + dg];
        k1[off] = tx;
      }
      __syncthreads();
      for (uint32_t dd = threadIdx.x; dd < 256; dd += blockDim.x) {
        unsigned int s = 0;
        for (int w2 = 0; w2 < nw; ++w2) {
          s += s_wc[w2 * 256 + dd];
          s_wc[w2 * 256 + dd] = 0;
        }
        s_base[dd] += s;
      }
      __syncthreads();
    }
    ulonglong2* tk = k0;
    k0 = k1;
    k1 = tk;
    flip ^= 1;
  }
  return flip;
}

__global__ void __launch_bounds__(kBmSortThreads, 2) k_bm_sort(const unsigned long long* __restrict__ part_off, BmGeo G,
                                                               ulonglong2* __restrict__ terms,
                                                               ulonglong2* __restrict__ terms2,
                                                               unsigned int* __restrict__ ticket,
                                                               unsigned long long* __restrict__ status, BmOut O) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem);  // kBmCap
  double* sv = reinterpret_cast<double*>(sk + kBmCap);                   // kBmCap
  unsigned int* cnt = reinterpret_cast<unsigned int*>(sv + kBmCap);      // kBmBins + 1 (+ pad)
  uint16_t* idx1 = reinterpret_cast<uint16_t*>(cnt + kBmBins + 4);        // kBmCap
  uint16_t* idx2 = idx1 + kBmCap;                                         // kBmCap (ranks first)
  uint16_t* rk = idx2;
  __shared__ unsigned long long s_w[33];
  __shared__ unsigned long long s_excl[33];  // [1..32]: look-back reduction scratch
  __shared__ uint32_t s_p;
  const uint32_t bsh = G.sb + G.bin_shift;
  const uint32_t bmask = (G.shift - G.bin_shift >= 11) ? kBmBins - 1 : (1u << (G.shift - G.bin_shift)) - 1;
  for (;;) {
    if (threadIdx.x == 0) s_p = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t p = s_p;
    if (p >= G.P) break;
    const uint64_t o0 = part_off[p];
    const uint32_t m = (uint32_t)(part_off[p + 1] - o0);
    if (m > kBmCap) {
      // global-memory path (shared arrays reused as digit counters)
      const int fl = bm_sort_global(terms + o0, terms2 + o0, m, G.shift + G.gspan + G.sb, cnt,
                                    reinterpret_cast<unsigned int*>(smem));
      const ulonglong2* tt = (fl ? terms2 : terms) + o0;
      bm_emit(p, m, G, [&](uint32_t q) { return tt[q].x; },
              [&](uint32_t q) { return __longlong_as_double((long long)tt[q].y); }, status, O, s_w, s_excl);
      continue;
    }
    for (uint32_t x = threadIdx.x; x <= kBmBins; x += blockDim.x) cnt[x] = 0;
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) {
      const ulonglong2 t = terms[o0 + x];
      sk[x] = t.x;
      sv[x] = __longlong_as_double((long long)t.y);
    }
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x)
      rk[x] = (uint16_t)atomicAdd(&cnt[(uint32_t)(sk[x] >> bsh) & bmask], 1u);
    __syncthreads();
    {  // exclusive scan of the bins, kBmBins / kBmSortThreads per thread
      constexpr int PER = kBmBins / kBmSortThreads;
      const uint32_t b0 = threadIdx.x * PER;
      unsigned int c[PER], s = 0;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        c[u] = cnt[b0 + u];
        s += c[u];
      }
      unsigned long long tot;
      unsigned int run = (unsigned int)block_excl_scan(s, s_w, &tot);
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        cnt[b0 + u] = run;
        run += c[u];
      }
      if (threadIdx.x == 0) cnt[kBmBins] = m;
    }
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < m; x += blockDim.x)
      idx1[cnt[(uint32_t)(sk[x] >> bsh) & bmask] + rk[x]] = (uint16_t)x;
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < m; q += blockDim.x) {
      const uint32_t x = idx1[q];
      const unsigned long long kx = sk[x];
      const uint32_t bn = (uint32_t)(kx >> bsh) & bmask;
      const uint32_t s = cnt[bn], e = cnt[bn + 1];
      uint32_t r = 0;
      for (uint32_t y = s; y < e; ++y) r += sk[idx1[y]] < kx;
      idx2[s + r] = (uint16_t)x;
    }
    __syncthreads();
    bm_emit(p, m, G, [&](uint32_t q) { return sk[idx2[q]]; }, [&](uint32_t q) { return sv[idx2[q]]; }, status, O,
            s_w, s_excl);
  }
}

constexpr size_t kBmSortSmem = (size_t)kBmCap * 16 + (kBmBins + 4) * 4 + (size_t)kBmCap * 4;

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
  uint64_t all_terms;    // every term of the stream
  CompositeKey ck{};
  cudaStream_t st = nullptr;  // creation stream: pool allocations are freed on it
  unsigned long long* d_counts = nullptr;
  unsigned long long* d_offs = nullptr;  // radix path: own offsets; bucket-major path: all-term offsets
  // bucket-major path
  bool bm = false;
  BmGeo geo{};
  uint32_t n_cta = 0;
  uint32_t max_part = 0;
  uint32_t* d_hash = nullptr;                // ha | hb per nonzero
  int64_t nnz_a = 0;
  unsigned int* d_gtab = nullptr;            // [P1][n_cta] slot offsets (+ partition totals)
  unsigned long long* d_part_off = nullptr;  // [P + 1]
};

namespace {

void outer_free(crop_outer* J) {
  for (void* p : {(void*)J->d_counts, (void*)J->d_offs, (void*)J->d_hash, (void*)J->d_gtab, (void*)J->d_part_off})
    if (p) cudaFreeAsync(p, J->st);
}

BmStream bm_stream(const crop_outer* J) {
  BmStream S{};
  S.a_ptr = J->a_ptr;
  S.b_ptr = J->b_ptr;
  S.a_idx = J->a_idx;
  S.b_idx = J->b_idx;
  S.a_val = J->a_val;
  S.b_val = J->b_val;
  S.offs = J->d_offs;
  S.n = J->n;
  S.total = J->all_terms;
  if (J->d_hash) {
    S.ha = J->d_hash;
    S.hb = J->d_hash + J->nnz_a;
  }
  return S;
}

// Partition histogram for geometry J->geo: d_gtab, d_part_off; host reads
// the largest partition and the own-term total (one synchronisation).
int bm_plan(crop_outer* J, const BmStream& S, uint64_t* own, uint32_t* max_part) {
  cudaStream_t st = J->st;
  const BmGeo& G = J->geo;
  if (J->d_gtab) cudaFreeAsync(J->d_gtab, st);
  if (J->d_part_off) cudaFreeAsync(J->d_part_off, st);
  J->d_gtab = nullptr;
  J->d_part_off = nullptr;
  const uint64_t cells = (uint64_t)G.P1 * J->n_cta;
  CROP_CUDA(cudaMallocAsync(&J->d_gtab, cells * 4 + (G.P + 2) * 4ull, st));
  unsigned int* ptot = J->d_gtab + cells;
  unsigned int* d_max = ptot + G.P;
  CROP_CUDA(cudaMallocAsync(&J->d_part_off, (G.P + 1) * 8ull, st));
  const bool sm = G.P <= kBmSmemParts;
  if (!sm) CROP_CUDA(cudaMemsetAsync(J->d_gtab, 0, cells * 4, st));
  CROP_CUDA(cudaMemsetAsync(ptot, 0, (G.P + 1) * 4ull, st));
  const size_t smb = sm ? (size_t)G.P * 4 : 0;
  CROP_CUDA(cudaFuncSetAttribute(k_bm_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBmSmemParts * 4)));
  k_bm_hist<<<J->n_cta, kBmThreads, smb, st>>>(S, G, J->d_gtab, ptot);
  CROP_LAUNCH_CHECK();
  k_bm_colscan<<<(int)std::min<uint32_t>((G.P1 + 7) / 8, 16 * kNumSMs), 256, 0, st>>>(J->d_gtab, G.P1, J->n_cta);
  CROP_LAUNCH_CHECK();
  crop_count_launches(2);
  if (int rc = scan_excl(LoadU32{ptot}, G.P, J->d_part_off, d_max, st)) return rc;
  if (!own) return CROP_OK;
  unsigned long long h_own = 0;
  unsigned int h_max = 0;
  CROP_CUDA(cudaMemcpyAsync(&h_own, J->d_part_off + G.P, 8, cudaMemcpyDeviceToHost, st));
  CROP_CUDA(cudaMemcpyAsync(&h_max, d_max, 4, cudaMemcpyDeviceToHost, st));
  CROP_CUDA(cudaStreamSynchronize(st));
  *own = h_own;
  *max_part = h_max;
  return CROP_OK;
}

// geometry with 2^S_bits partitions per bucket; false if it does not fit
bool bm_geometry(crop_outer* J, uint32_t rb, uint32_t cb, uint32_t S_bits, BmGeo* G) {
  const uint32_t W = rb + cb;
  const uint32_t sb = bits_for(J->all_terms - 1);
  const uint32_t nb = J->has_hash ? J->iv.stop - J->iv.start : 1;
  if (W + sb > 64) S_bits = std::max<uint32_t>(S_bits, W + sb - 64);
  if (S_bits > W || S_bits > 24) return false;
  const uint64_t P = (uint64_t)nb << S_bits;
  if (P > (1ull << 22) || P == 0) return false;
  G->kappa = J->has_hash ? J->iv.kappa : 1;
  G->start = J->has_hash ? J->iv.start : 0;
  G->nb = nb;
  G->cb = cb;
  G->sb = sb;
  G->S_bits = S_bits;
  G->shift = W - S_bits;
  if (G->shift + sb > 64) return false;
  G->bin_shift = G->shift > 11 ? G->shift - 11 : 0;
  G->P = (uint32_t)P;
  // groups: about kBmGroupsTarget of them, each 2^gspan partitions of one
  // bucket, as long as the word keeps the group's local key bits
  uint32_t gbits = 0;  // groups per bucket (log2)
  while (gbits < S_bits && ((uint64_t)nb << gbits) < kBmGroupsTarget) ++gbits;
  while (gbits < S_bits && G->shift + (S_bits - gbits) + sb > 64) ++gbits;
  G->gspan = S_bits - gbits;
  G->P1 = nb << gbits;
  G->has_hash = J->has_hash;
  G->upper = J->upper;
  G->filter = J->filter;
  return true;
}

}  // namespace

extern "C" int crop_outer_create(const int64_t* a_ptr, const uint32_t* a_idx, const double* a_val,
                                 const int64_t* b_ptr, const uint32_t* b_idx, const double* b_val,
                                 int64_t n_products, int upper_only, const crop_interval* interval,
                                 void* stream, crop_outer** job) {
  return crop_outer_create_ex(a_ptr, a_idx, a_val, b_ptr, b_idx, b_val, n_products, upper_only, interval,
                              nullptr, stream, job);
}

extern "C" int crop_outer_create_ex(const int64_t* a_ptr, const uint32_t* a_idx, const double* a_val,
                                    const int64_t* b_ptr, const uint32_t* b_idx, const double* b_val,
                                    int64_t n_products, int upper_only, const crop_interval* interval,
                                    const crop_outer_shape* shape, void* stream, crop_outer** job) {
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
  J->st = st;
  J->total_terms = 0;
  J->all_terms = 0;
  auto fail = [&](int rc) {
    outer_free(J);
    delete J;
    return rc;
  };
#define OUTER_CHECK(call)                                                                     \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      crop_set_error(CROP_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return fail(CROP_ECUDA);                                                                \
    }                                                                                         \
  } while (0)
  if (n_products <= 0 || (J->has_hash && J->iv.start == J->iv.stop)) {
    *job = J;
    return CROP_OK;
  }
  const int64_t nn = n_products;
  // all-term offsets, the largest row / column index and the nonzero counts (one sync)
  OUTER_CHECK(cudaMallocAsync(&J->d_offs, (nn + 2) * 8, st));  // + 8 bytes: index maxima
  if (int rc = scan_excl(TermsOf{a_ptr, b_ptr}, (uint64_t)nn, J->d_offs, nullptr, st)) return fail(rc);
  unsigned long long all = 0;
  unsigned int mx[2] = {0, 0};
  int64_t nnz[2] = {0, 0};
  if (shape) {
    all = shape->all_terms;
    mx[0] = shape->max_row;
    mx[1] = shape->max_col;
    nnz[0] = shape->nnz_a;
    nnz[1] = shape->nnz_b;
  } else {
    unsigned int* d_mx = reinterpret_cast<unsigned int*>(J->d_offs + nn + 1);
    OUTER_CHECK(cudaMemsetAsync(d_mx, 0, 8, st));
    k_max_u32<<<2 * kNumSMs, 256, 0, st>>>(a_idx, a_ptr + nn, b_idx, b_ptr + nn, d_mx);
    OUTER_CHECK(cudaGetLastError());
    crop_count_launches(1);
    OUTER_CHECK(cudaMemcpyAsync(&all, J->d_offs + nn, 8, cudaMemcpyDeviceToHost, st));
    OUTER_CHECK(cudaMemcpyAsync(mx, d_mx, 8, cudaMemcpyDeviceToHost, st));
    OUTER_CHECK(cudaMemcpyAsync(&nnz[0], a_ptr + nn, 8, cudaMemcpyDeviceToHost, st));
    OUTER_CHECK(cudaMemcpyAsync(&nnz[1], b_ptr + nn, 8, cudaMemcpyDeviceToHost, st));
    OUTER_CHECK(cudaStreamSynchronize(st));
  }
  J->all_terms = all;
  if (all == 0) {
    *job = J;
    return CROP_OK;
  }
  if (all >= (1ull << 32)) {
    crop_set_error(CROP_ERESOURCE, "more than 2^32 terms in one stream; split the stream");
    return fail(CROP_ERESOURCE);
  }
  const uint32_t rb = bits_for(mx[0]), cb = bits_for(mx[1]);
  const uint32_t nb = J->has_hash ? J->iv.stop - J->iv.start : 1;
  const uint64_t est = std::max<uint64_t>(1, all * nb / (J->has_hash ? J->iv.kappa : 1));
  uint32_t S_bits = 0;
  while (((uint64_t)nb << S_bits) * kBmTarget < est) ++S_bits;
  BmGeo G{};
  if (!getenv("CROP_OUTER_RADIX") && bm_geometry(J, rb, cb, S_bits, &G)) {
    J->bm = true;
    J->geo = G;
    if (J->has_hash) {
      J->nnz_a = nnz[0];
      OUTER_CHECK(cudaMallocAsync(&J->d_hash, (uint64_t)(nnz[0] + nnz[1]) * 4 + 8, st));
      k_nnz_hash<<<8 * kNumSMs, 256, 0, st>>>(a_idx, (uint64_t)nnz[0], J->iv.h_row, J->d_hash);
      k_nnz_hash<<<8 * kNumSMs, 256, 0, st>>>(b_idx, (uint64_t)nnz[1], J->iv.h_col, J->d_hash + nnz[0]);
      OUTER_CHECK(cudaGetLastError());
      crop_count_launches(2);
    }
    const BmStream S = bm_stream(J);
    uint64_t own = 0;
    uint32_t mp = 0;
    if (shape) {
      // no synchronisation: the own-term count stays on the device (the
      // bound below sizes the buffers) and partitions larger than shared
      // memory take the sort kernel's global-memory path
      J->n_cta = (uint32_t)std::max<uint64_t>(16, std::min<uint64_t>(kNumSMs, (1ull << 26) / J->geo.P1));
      if (int rc = bm_plan(J, S, nullptr, nullptr)) return fail(rc);
      J->total_terms = all;
      J->max_part = UINT32_MAX;
      *job = J;
      return CROP_OK;
    }
    for (int attempt = 0;; ++attempt) {
      // the per-CTA slot table stays below 2^26 cells
      J->n_cta = (uint32_t)std::max<uint64_t>(16, std::min<uint64_t>(kNumSMs, (1ull << 26) / J->geo.P1));
      if (int rc = bm_plan(J, S, &own, &mp)) return fail(rc);
      if (mp <= kBmCap || attempt == 2) break;
      // refine: more partitions per bucket so the largest fits shared memory
      uint32_t inc = 0;
      while (((uint64_t)kBmTarget << inc) < mp) ++inc;
      BmGeo G2{};
      if (!bm_geometry(J, rb, cb, J->geo.S_bits + inc, &G2)) break;
      J->geo = G2;
    }
    J->total_terms = own;
    J->max_part = mp;
    *job = J;
    return CROP_OK;
  }
  // radix-sort fallback (keys wider than 64 bits, or CROP_OUTER_RADIX): own
  // counts per product, offsets, one stable library sort
  OUTER_CHECK(cudaMallocAsync(&J->d_counts, nn * 8, st));
  {
    int64_t blocks = std::min<int64_t>((n_products + 7) / 8, 1 << 20);
    if (J->filter)
      k_outer_count<true><<<(int)blocks, 256, 0, st>>>(a_ptr, a_idx, b_ptr, b_idx, n_products,
                                                      upper_only, J->iv, J->d_counts);
    else
      k_outer_count<false><<<(int)blocks, 256, 0, st>>>(a_ptr, a_idx, b_ptr, b_idx, n_products,
                                                       upper_only, J->iv, J->d_counts);
    OUTER_CHECK(cudaGetLastError());
    const unsigned long long* cnts = J->d_counts;
    if (int rc = scan_excl(LoadU64{cnts}, (uint64_t)nn, J->d_offs, nullptr, st)) return fail(rc);
    unsigned long long own = 0;
    OUTER_CHECK(cudaMemcpyAsync(&own, J->d_offs + nn, 8, cudaMemcpyDeviceToHost, st));
    OUTER_CHECK(cudaStreamSynchronize(st));
    J->total_terms = own;
  }
  {
    const uint32_t bb = J->has_hash ? bits_for(J->iv.kappa - 1) : 0;
    J->ck.has_hash = J->has_hash;
    J->ck.c_bits = cb;
    J->ck.rc_bits = rb + cb;
    J->ck.bits = bb + rb + cb;
    J->ck.on = J->ck.bits <= 64 && !getenv("CROP_OUTER_TWO_SORTS");
  }
#undef OUTER_CHECK
  *job = J;
  return CROP_OK;
}

extern "C" int crop_outer_info(const crop_outer* J, uint64_t* max_entries, uint64_t* total_terms) {
  if (max_entries) *max_entries = J->total_terms;
  if (total_terms) *total_terms = J->total_terms;
  return CROP_OK;
}

extern "C" int crop_outer_own_terms(const crop_outer* J, uint64_t* d_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (J->bm && J->d_part_off) {
    CROP_CUDA(cudaMemcpyAsync(d_out, J->d_part_off + J->geo.P, 8, cudaMemcpyDeviceToDevice, st));
  } else {
    const unsigned long long v = J->total_terms;
    CROP_CUDA(cudaMemcpyAsync(d_out, &v, 8, cudaMemcpyHostToDevice, st));
    CROP_CUDA(cudaStreamSynchronize(st));  // v lives on this stack frame
  }
  return CROP_OK;
}

static int outer_run_bm(crop_outer* J, uint32_t* out_row, uint32_t* out_col, double* out_value,
                        uint32_t* out_bucket, uint64_t* d_n_entries, cudaStream_t st) {
  const BmGeo G = J->geo;
  const uint64_t n = J->total_terms;
  const bool split = G.gspan > 0, big = J->max_part > kBmCap;
  ulonglong2 *ta = nullptr, *tb = nullptr;
  unsigned long long* status = nullptr;
  CROP_CUDA(cudaMallocAsync(&ta, n * 16, st));
  if (split || big) CROP_CUDA(cudaMallocAsync(&tb, n * 16, st));
  CROP_CUDA(cudaMallocAsync(&status, (G.P + 1) * 8ull, st));
  CROP_CUDA(cudaMemsetAsync(status, 0, (G.P + 1) * 8ull, st));
  unsigned int* ticket = reinterpret_cast<unsigned int*>(status + G.P);
  const BmStream S = bm_stream(J);
  const bool sm = G.P1 <= kBmSmemParts;
  CROP_CUDA(cudaFuncSetAttribute(k_bm_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBmSmemParts * 4)));
  k_bm_scatter<<<J->n_cta, kBmThreads, sm ? (size_t)G.P1 * 4 : 0, st>>>(S, G, J->d_gtab, J->d_part_off, ta);
  CROP_LAUNCH_CHECK();
  // sorted input: ta, or tb after the split (ta is then the big-partition scratch)
  ulonglong2 *ts = ta, *tt = tb;
  if (split) {
    const size_t smb = ((size_t)1 << G.gspan) * 4;
    CROP_CUDA(cudaFuncSetAttribute(k_bm_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smb, 4)));
    k_bm_split<<<(int)std::min<uint32_t>(G.P1, 2 * kNumSMs), kBmThreads, smb, st>>>(G, J->d_part_off, ta, tb);
    CROP_LAUNCH_CHECK();
    ts = tb;
    tt = ta;
    crop_count_launches(1);
  }
  CROP_CUDA(cudaFuncSetAttribute(k_bm_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBmSortSmem));
  BmOut O{out_row, out_col, out_bucket, out_value, (unsigned long long*)d_n_entries};
  k_bm_sort<<<(int)std::min<uint32_t>(G.P, 2 * kNumSMs), kBmSortThreads, kBmSortSmem, st>>>(
      J->d_part_off, G, ts, tt, ticket, status, O);
  CROP_LAUNCH_CHECK();
  for (void* p : {(void*)ta, (void*)tb, (void*)status})
    if (p) cudaFreeAsync(p, st);
  crop_count_launches(2);
  return CROP_OK;
}

extern "C" int crop_outer_run(crop_outer* J, uint32_t* out_row, uint32_t* out_col,
                              double* out_value, uint32_t* out_bucket, uint64_t* d_n_entries,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  CROP_CUDA(cudaMemsetAsync(d_n_entries, 0, 8, st));
  const uint64_t n = J->total_terms;
  if (n == 0) return CROP_OK;
  if (J->bm) return outer_run_bm(J, out_row, out_col, out_value, out_bucket, d_n_entries, st);
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
  outer_free(J);
  delete J;
}
