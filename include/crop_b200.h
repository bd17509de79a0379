/*
 * crop_b200.h -- C-ABI of the B200-native CRoP hot path (libcrop_b200.so).
 *
 * The reference package (pkg/src/crop, pure Python) has no FFI; its hot path
 * is a set of Python functions. Each entry point below replaces one of them
 * and is bound by paper_1210_0461_b200/_native.py through ctypes (the same
 * binding a reference maintainer would add).
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors) unless named h_*; `stream` is a cudaStream_t passed as void*.
 *    Calls are stream-ordered; functions that must read back a size
 *    (crop_pairs_create) synchronise the stream and say so.
 *  - Return value: CROP_OK (0) or an error status; crop_last_error() gives
 *    the message. Status -> Python exception (errors.py:8-34):
 *      2 InputError, 3 ConfigError, 4 ResourceCapError, 5 CUDA failure.
 *  - Item ids are uint32 < 2^31; transactions / outer products are CSR:
 *    offsets int64[n+1], indices uint32[offsets[n]] (ascending per row).
 *  - Hash coefficients are the reference's (mul, add) pairs modulo 2^61-1
 *    (hashing.py:127-146); kappa <= 2^31.
 */
#ifndef CROP_B200_H
#define CROP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CROP_OK 0
#define CROP_EINPUT 2
#define CROP_ECONFIG 3
#define CROP_ERESOURCE 4
#define CROP_ECUDA 5

/* Version of the ABI (bumped on any signature change). */
int crop_abi_version(void);

/* Message of the last failing call on this thread. */
const char* crop_last_error(void);

/* Kernels launched by this library so far (process-wide counter). */
unsigned long long crop_launch_counter(void);

/* K0 -- per-item hash tables, IndexHashFn.values (hashing.py:68-71):
 * h_row[i] = ((row_mul*i + row_add) mod p) mod kappa, likewise h_col, for
 * i in [0, n_items). Exact 128-bit Mersenne arithmetic on device. */
int crop_hash_tables(uint32_t n_items, uint64_t row_mul, uint64_t row_add, uint64_t col_mul,
                     uint64_t col_add, uint32_t kappa, uint32_t* h_row, uint32_t* h_col,
                     void* stream);

/* Sign hash (hashing.py:98-100) of n entries: out[e] = s(row[e], col[e]). */
int crop_sign_hash(const uint32_t* row, const uint32_t* col, uint64_t n, uint64_t sign_mul,
                   uint64_t sign_add, int8_t* out, void* stream);

/* K1 -- per-bucket term counts of a self-join transaction stream, the
 * quantity measure_loads / count_sorted report (engine.py:305-349,
 * interval.py:192-233) before folding buckets into worker intervals.
 * upper_only: pairs i<j only (mining); else every ordered (i,j) incl. i==j.
 * bucket_loads: uint64[kappa], accumulated into (caller zeroes it). */
int crop_selfjoin_bucket_loads(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                               const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                               int upper_only, uint64_t* bucket_loads, void* stream);

/* Same for a general stream a_k x b_k (count_interval, interval.py:257-269). */
int crop_outer_bucket_loads(const int64_t* a_ptr, const uint32_t* a_idx, const int64_t* b_ptr,
                            const uint32_t* b_idx, int64_t n_products, const uint32_t* h_row,
                            const uint32_t* h_col, uint32_t kappa, int upper_only,
                            uint64_t* bucket_loads, void* stream);

/* K2 -- exact pair counting of a self-join 0/1 stream restricted to a bucket
 * interval [start, stop): the exact regime of engine.run / run_worker
 * (engine.py:238-302, 396-455), where every per-bucket Space-Saving summary
 * holds exact counts. Output: the distinct (row, col) entries
 * of the interval with their uint32 counts, unordered.
 *
 * Two calls. crop_pairs_create scans the input once (per-item term counts),
 * SYNCHRONISES the stream, and plans the on-chip tiles; it reports the output
 * capacity the caller must allocate. crop_pairs_run then routes, counts and
 * writes the entries (async); *d_n_entries (device uint64) receives the
 * number written. The job keeps its own device scratch until destroyed. */
typedef struct crop_pairs crop_pairs;

typedef struct {
    uint32_t kappa;         /* buckets */
    uint32_t start, stop;   /* owned interval [start, stop) */
    const uint32_t* h_row;  /* device uint32[n_items] (crop_hash_tables) */
    const uint32_t* h_col;
} crop_interval;

int crop_pairs_create(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                      uint32_t n_items, int upper_only, const crop_interval* interval,
                      void* stream, crop_pairs** job);
/* Tile sharding across ranks (one GPU each): every rank plans the same tiles
 * and keeps those whose term prefix falls in its 1/shard_world share (a
 * split row's windows stay together), so the union of the ranks' outputs is
 * the whole job's output, each pair on exactly one rank. The work, not the
 * buckets, is what is split: bucket loads come from the entries
 * (crop_entry_bucket_stats) and are summed across ranks. shard_world = 1 is
 * crop_pairs_create. */
int crop_pairs_create_sharded(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                              uint32_t n_items, int upper_only, const crop_interval* interval,
                              uint32_t shard_rank, uint32_t shard_world, void* stream,
                              crop_pairs** job);
/* crop_pairs_create_sharded with option flags:
 *  CROP_PAIRS_SAFE_UNITS  cut every word-counted dense tile into units of at
 *                         most 65,535 words, so no 16-bit counter can wrap
 *                         whatever the order of the stream (the re-run after
 *                         crop_pairs_overflowed reports a wrap);
 *  CROP_PAIRS_NO_OWN      filtered jobs: do not use the own-bucket (Lemma 1)
 *                         layout (A/B measurements).
 * A filtered job (interval narrower than [0, kappa)) whose ids fit one dense
 * table (n_items <= 57,345) and whose (h_col, id) keys fit 32 bits visits only
 * its own terms: each transaction's items are copied sorted by (h_col, id)
 * (bucket_sort_indices, interval.py:70-109) and every row occurrence reads
 * its one or two class windows of that copy (scan_sorted's windows,
 * interval.py:125-189). Its plan, words and counts cover its own terms only;
 * crop_pairs_info's total_terms is then the interval's own term count. */
#define CROP_PAIRS_SAFE_UNITS 1u
#define CROP_PAIRS_NO_OWN 2u
int crop_pairs_create_ex(const int64_t* offsets, const uint32_t* items, int64_t n_tx,
                         uint32_t n_items, int upper_only, const crop_interval* interval,
                         uint32_t shard_rank, uint32_t shard_world, uint32_t flags, void* stream,
                         crop_pairs** job);
/* 1 if the job uses the own-bucket layout (see crop_pairs_create_ex). */
int crop_pairs_own(const crop_pairs* job, int* own);
/* host-side plan facts: output capacity, total terms (all buckets), tiles */
int crop_pairs_info(const crop_pairs* job, uint64_t* max_entries, uint64_t* total_terms,
                    uint64_t* n_tiles, uint64_t* n_units);
/* terms of this job's own tiles (a tile shard's share; window tiles are
 * estimates), 0 when unknown (host-planned jobs): sizes the output buffer of
 * a shard (LoadReport units, engine.py:283) */
int crop_pairs_own_terms(const crop_pairs* job, uint64_t* own_terms);
int crop_pairs_run(crop_pairs* job, uint32_t* out_row, uint32_t* out_col, uint32_t* out_count,
                   uint64_t* d_n_entries, void* stream);
/* Per-phase CUDA-event timing of crop_pairs_run (off by default). out4 =
 * {route, write, 0, count} in ms of the last run: stream mode = {per-tile word
 * totals + scan, word write, -, count + slab reduction}; entry mode = {entry
 * routing, per-tile entry counts, -, count}. */
int crop_pairs_set_timing(crop_pairs* job, int on);
int crop_pairs_phase_ms(const crop_pairs* job, float* out4);
/* 1 if the job's counts are unreliable (synchronises): entry mode -- the entry
 * list overflowed its capacity (never expected); stream mode -- a 16-bit
 * dense counter of a unit holding more than 65,535 words wrapped (possible
 * only for adversarially ordered streams); re-create the job with
 * CROP_PAIRS_SAFE_UNITS and run it again. */
int crop_pairs_overflowed(const crop_pairs* job, int* overflowed);
/* Counting mode chosen by crop_pairs_create: 1 = stream (one 32-bit word per
 * pair term routed to its tile's stream, coalesced counting), 0 = entry
 * (one entry per (transaction, tile) run, counting re-reads the items).
 * CROP_FORCE_ENTRY_MODE=1 in the environment forces entry mode. */
int crop_pairs_mode(const crop_pairs* job, int* stream_mode);
/* Output arrays of the next runs hold `capacity` entries (<= max_entries;
 * default max_entries). Entries past it are counted in *d_n_entries but not
 * written: when *d_n_entries > capacity, run again with a larger capacity. */
int crop_pairs_set_capacity(crop_pairs* job, uint64_t capacity);
/* Stream mode only: caller-owned, zeroed buffers that the next crop_pairs_run
 * fills for a fused top-k -- hist uint32[23552] receives the histogram bins of
 * every output count >= 2048, hi_list (>= total_terms / 2048 + 1 entries) the
 * output positions of those entries, *hi_n their number. */
int crop_pairs_set_topk(crop_pairs* job, uint32_t* hist, uint64_t* hi_list, uint64_t* hi_n,
                        uint64_t hi_cap);
/* crop_topk over entries whose high counts were pre-binned by the counting
 * kernels (crop_pairs_set_topk); when those entries number >= k only they
 * are scanned, else the remaining counts are binned as in crop_topk. Same
 * result as crop_topk. Replaces engine.py:162-172 top_entries. */
int crop_topk_fused(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                    const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k, uint32_t* hist,
                    const uint64_t* hi_list, const uint64_t* hi_n, uint64_t* out_idx,
                    uint64_t* d_k_out, void* stream);
/* Per-partition top-l select: the summaries of the bounded Space-Saving
 * regime (spacesaving.py:39-63 with capacity l; engine.py:108-176 queries).
 * For every bucket b = (h_row[row] + h_col[col]) mod kappa holding >= l
 * entries: recorded[e] = 1 for its top-l entries by (count desc, row asc, col
 * asc), 0 for the rest, bucket_min[b] = the count of its l-th entry; buckets
 * with fewer entries record everything (bucket_min 0). bucket_total[b]
 * (nullable) = entries per bucket. recorded may be NULL (minima only). */
int crop_bucket_topk(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                     const uint64_t* d_n_entries, uint64_t n_capacity, const uint32_t* h_row,
                     const uint32_t* h_col, uint32_t kappa, uint32_t capacity, uint8_t* recorded,
                     uint32_t* bucket_min, uint32_t* bucket_total, void* stream);
void crop_pairs_destroy(crop_pairs* job);

/* Per-instance bucket statistics of counted entries (the LoadReport rows,
 * engine.py:179-216, Count-Sketch cells, countsketch.py:33-41, and per-bucket
 * distinct counts). For instance t the hash tables are h_row[t*n_items ...].
 * Outputs (accumulated, caller zeroes): loads uint64[t][kappa] = sum of
 * counts, distinct uint32[t][kappa], cs int64[t][kappa] = sum count*sign
 * (pass NULL to skip), sign coefficients h_sign[2*t] (host array). */
int crop_entry_bucket_stats(const uint32_t* row, const uint32_t* col, const uint32_t* count,
                            const uint64_t* d_n_entries, uint64_t max_entries, int instances,
                            uint32_t n_items, const uint32_t* h_row, const uint32_t* h_col,
                            uint32_t kappa, const uint64_t* h_sign, uint64_t* loads,
                            uint32_t* distinct, int64_t* cs, void* stream);

/* Real-weight variant: per-bucket entry counts and fp64 Count-Sketch cells
 * sum weight*sign (accumulated; order differs from the reference, so cells
 * agree to rounding). distinct uint32[t][kappa], cs double[t][kappa]|NULL. */
int crop_entry_bucket_stats_f64(const uint32_t* row, const uint32_t* col, const double* weight,
                                const uint64_t* d_n_entries, uint64_t max_entries, int instances,
                                uint32_t n_items, const uint32_t* h_row, const uint32_t* h_col,
                                uint32_t kappa, const uint64_t* h_sign, uint32_t* distinct,
                                double* cs, void* stream);

/* Per-product worker loads, LoadReport.per_product (engine.py:250-251,287-288):
 * out[k*workers + w] (uint32, caller zeroes) = terms of product k that fall in
 * worker w's interval (interval.py:37-45). Self-joins pass a == b. */
int crop_product_worker_loads(const int64_t* a_ptr, const uint32_t* a_idx, const int64_t* b_ptr,
                              const uint32_t* b_idx, int64_t n_products, const uint32_t* h_row,
                              const uint32_t* h_col, uint32_t kappa, uint32_t workers,
                              int upper_only, uint32_t* out, void* stream);

/* Bucket of each entry for one instance: out[e] = (h_row[row]+h_col[col]) mod kappa. */
int crop_entry_buckets(const uint32_t* row, const uint32_t* col, uint64_t n,
                       const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                       uint32_t* out, void* stream);

/* K4 -- top-k select (SketchState.top_entries, engine.py:162-172; exact_top,
 * oracle.py:53-58): indices of the k entries first in the order
 * (count desc, row asc, col asc); written unordered to out_idx[0..k'),
 * k' = min(k, n) returned in *d_k_out (device uint64). */
int crop_topk(const uint32_t* row, const uint32_t* col, const uint32_t* count,
              const uint64_t* d_n_entries, uint64_t max_entries, uint32_t k, uint64_t* out_idx,
              uint64_t* d_k_out, void* stream);

/* Streaming, mergeable per-bucket Space-Saving (spacesaving.py:39-63 with
 * O(l) state per bucket; csrc/ss_stream.cu). The caller keeps the summary
 * records of every bucket as flat device arrays (row, col, count, over) and
 * merges each chunk's exact entries into them:
 *   crop_ss_index  builds an open-addressing index over the n record keys
 *                  (slots uint64[n_slots]: hash fingerprint << 32 | record;
 *                  n_slots a power of two >= 2n) and, when bloom is not
 *                  NULL, a Bloom filter over the same keys (bloom_words
 *                  64-bit words, a power of two; four bits of one word per
 *                  key) that answers most misses from L2
 *   crop_ss_probe  pass 1 over the chunk entries (row, col, e): a recorded
 *                  key adds e to its record's count (rec_count, in place); an
 *                  unrecorded key (a miss) sets bit e of missbits and counts
 *                  in hist[b * 16 + min(e, 15)], b = (h_row[row] + h_col[col])
 *                  mod kappa. Then per bucket the cut: cut[b] = the largest
 *                  weight with at least `capacity` misses at or above it (0:
 *                  keep every miss) -- a miss below it cannot be among the
 *                  bucket's `capacity` largest. d_meta[0] = misses at or
 *                  above their cut (the candidates), d_meta[1] = the
 *                  smallest cut. hist: uint32[kappa * 16], cut: uint32[kappa],
 *                  missbits: uint32[ceil(max_entries / 32)].
 *   crop_ss_append pass 2: every miss at or above its bucket's cut becomes a
 *                  candidate (mu[b] + e, over mu[b]) appended behind the
 *                  records at *d_n_out (in: the record count; out: records +
 *                  candidates). *d_saturated is set when a count would pass
 *                  2^32 - 1.
 *   crop_ss_keep   the entries a selection marked (mask[e] != 0, e <
 *                  *d_n) appended to the out arrays; *d_n_out = their number.
 * The caller keeps each bucket's l largest of records + candidates
 * (crop_bucket_topk, then crop_ss_keep) and sets mu[b] to the l-th count of
 * full buckets. */
int crop_ss_index(const uint32_t* row, const uint32_t* col, uint64_t n, unsigned long long* slots,
                  uint64_t n_slots, unsigned long long* bloom, uint64_t bloom_words, void* stream);
int crop_ss_probe(const uint32_t* erow, const uint32_t* ecol, const uint32_t* ecnt,
                  const uint64_t* d_n_entries, uint64_t max_entries, const unsigned long long* slots,
                  uint64_t n_slots, const unsigned long long* bloom, uint64_t bloom_words,
                  uint64_t n_records, const uint32_t* h_row, const uint32_t* h_col, uint32_t kappa,
                  uint32_t capacity, const uint32_t* rec_row, const uint32_t* rec_col, uint32_t* rec_count,
                  uint32_t* missbits, uint32_t* hist, uint32_t* cut, uint64_t* d_meta,
                  unsigned int* d_saturated, void* stream);
int crop_ss_append(const uint32_t* erow, const uint32_t* ecol, const uint32_t* ecnt,
                   const uint64_t* d_n_entries, uint64_t max_entries, const uint32_t* missbits,
                   const uint32_t* cut, const uint64_t* d_meta, const uint32_t* h_row, const uint32_t* h_col,
                   uint32_t kappa, const uint32_t* mu, uint32_t* row, uint32_t* col, uint32_t* count,
                   uint32_t* over, uint64_t* d_n_out, unsigned int* d_saturated, void* stream);
int crop_ss_keep(const uint8_t* mask, const uint64_t* d_n, uint64_t max_n, const uint32_t* row,
                 const uint32_t* col, const uint32_t* count, const uint32_t* over, uint32_t* out_row,
                 uint32_t* out_col, uint32_t* out_count, uint32_t* out_over, uint64_t* d_n_out, void* stream);

/* K5 -- general outer-product stream (real values), restricted to buckets
 * [start, stop): the per-partition enumerate_interval + accumulate loop
 * (interval.py:236-254; exact_product, oracle.py:20-50). Terms are emitted,
 * stably sorted by (bucket, row, col) and summed in fp64 in stream order, so
 * each sum equals the reference's dict accumulation bit for bit. Output is
 * the per-partition sorted COO: row/col uint32, value float64, bucket
 * uint32, grouped by bucket ascending, (row, col) ascending inside. Zero sums
 * are kept (the caller decides, exact_product drops them, oracle.py:50).
 * crop_outer_create synchronises to learn the stream's shape and the own
 * term count; crop_outer_create_ex with a shape does not synchronise. */
typedef struct crop_outer crop_outer;
int crop_outer_create(const int64_t* a_ptr, const uint32_t* a_idx, const double* a_val,
                      const int64_t* b_ptr, const uint32_t* b_idx, const double* b_val,
                      int64_t n_products, int upper_only, const crop_interval* interval,
                      void* stream, crop_outer** job);
/* Shape of an outer-product stream, known to the caller once per stream
 * (e.g. computed at upload): with it crop_outer_create_ex plans without
 * synchronising the stream; crop_outer_info then reports max_entries as the
 * upper bound all_terms (the own-interval count is only known on the
 * device, as *d_n_entries after the run). */
typedef struct {
    uint64_t all_terms;       /* sum over products of |a_k| * |b_k| */
    uint32_t max_row;         /* largest a_idx (0 if none) */
    uint32_t max_col;         /* largest b_idx (0 if none) */
    int64_t nnz_a, nnz_b;     /* a_ptr[n], b_ptr[n] */
} crop_outer_shape;
int crop_outer_create_ex(const int64_t* a_ptr, const uint32_t* a_idx, const double* a_val,
                         const int64_t* b_ptr, const uint32_t* b_idx, const double* b_val,
                         int64_t n_products, int upper_only, const crop_interval* interval,
                         const crop_outer_shape* shape, void* stream, crop_outer** job);
int crop_outer_info(const crop_outer* job, uint64_t* max_entries, uint64_t* total_terms);
/* Own-interval term count into device memory (stream-ordered; exact also
 * when crop_outer_create_ex planned without synchronising). */
int crop_outer_own_terms(const crop_outer* job, uint64_t* d_out, void* stream);
int crop_outer_run(crop_outer* job, uint32_t* out_row, uint32_t* out_col, double* out_value,
                   uint32_t* out_bucket, uint64_t* d_n_entries, void* stream);
void crop_outer_destroy(crop_outer* job);

/* Synthetic transaction workload (bench / tests): successive sampling without
 * replacement from an integer alias table (h_alias_*: host arrays, n_items
 * long), lengths from an integer CDF over [len_lo, len_lo + n_len).
 * Deterministic in (seed, transaction index) on any GPU count.
 *   crop_gen_lengths writes lengths int64[n_tx]; the caller prefix-sums them
 *   into offsets; crop_gen_items fills items (sorted ascending per row). */
int crop_gen_lengths(int64_t n_tx, uint64_t seed, const uint32_t* h_len_cdf, uint32_t n_len,
                     uint32_t len_lo, int64_t* lengths, void* stream);
int crop_gen_items(int64_t n_tx, uint64_t seed, uint32_t n_items, const uint32_t* h_alias_thresh,
                   const uint32_t* h_alias_idx, const int64_t* offsets, uint32_t* items,
                   void* stream);

/* ---- input ingestion --------------------------- */
/* Read a FIMI file (read_fimi, sparse.py:270-298: one transaction per line,
 * blank lines skipped, items sorted and de-duplicated) on `threads` host
 * threads (0: all) into CSR. Accepts the plain form only (ASCII decimal ids
 * < 2^31, ASCII whitespace, '\n' / "\r\n" line ends); anything else returns
 * CROP_EINPUT with *bad_line = the 1-based line, and the caller re-reads the
 * file with the reference-exact reader (which raises ParseError). */
typedef struct crop_fimi crop_fimi;
int crop_fimi_parse(const char* path, int threads, crop_fimi** out, int64_t* n_tx, int64_t* nnz,
                    uint32_t* max_item, int64_t* duplicates, int64_t* bad_line);
/* Copy the parsed CSR into caller buffers: offsets[n_tx + 1], items[nnz]. */
int crop_fimi_copy(const crop_fimi* parsed, int64_t* offsets, uint32_t* items);
void crop_fimi_free(crop_fimi* parsed);

/* Read one triple file (read_triple_file, sparse.py:173-225: header
 * "n_rows n_cols kcount", then "k index value" lines with k non-decreasing;
 * explicit zeros dropped and counted; each k's entries sorted by index,
 * duplicates rejected) on `threads` host threads into CSR over k. dims =
 * {n_rows, n_cols, kcount}. Plain form only (ASCII decimal integers and
 * decimal/exponent floats, '\n' or "\r\n"); anything else -- and every
 * error the reference reports -- returns CROP_EINPUT with *bad_line (0 for a
 * duplicate index), and the caller re-reads the file with the
 * reference-exact reader (which raises ParseError). */
typedef struct crop_triples crop_triples;
int crop_triple_parse(const char* path, int threads, crop_triples** out, int64_t* dims,
                      int64_t* nnz, int64_t* zeros, int64_t* bad_line);
/* Copy into caller buffers: ptr[kcount + 1], idx[nnz], val[nnz]. */
int crop_triple_copy(const crop_triples* parsed, int64_t* ptr, uint32_t* idx, double* val);
void crop_triple_free(crop_triples* parsed);

#ifdef __cplusplus
}
#endif
#endif /* CROP_B200_H */
