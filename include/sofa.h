/*
 * sofa.h — C ABI of the B200-native SOFA exact k-NN path (libsofa.so).
 *
 * SOFA = "Fast and Exact Similarity Search in less than a Blink of an Eye" (arxiv 2411.17483),
 * PAPER.md citations as P:<line>.  The path:
 *   a1 z-normalisation        Def. 2
 *   a2 MCB learning           Alg. 1, P:297-325 (variance selection P:248-250)
 *   a3 SFA transform          Alg. 2, bins P:225-228
 *   a4 block layout           MESSI tree P:159-166 -> sorted SFA-word blocks + envelopes
 *   a5 query prep             d_SFA / mind_i tables
 *   a6 seed + envelope LB     approximate search P:169, leaf LB P:171-173
 *   a7 word LB scan           Alg. 3, P:398-435 (chunks of 8, early abandon)
 *   a8 refine + top-k         P:119, ED with early abandoning P:382
 *   a9 cross-GPU merge        k-NN P:177
 *
 * Conventions (every entry point):
 *  - Array pointers named *_dev are CUDA DEVICE pointers (row-major; float32 / int64 / uint8 /
 *    float64 as typed).  Pointers named *_host are host pointers.  Struct pointers
 *    (sofa_model, sofa_build_opts, sofa_knn_stats) are host pointers.
 *  - `cuda_stream` is a cudaStream_t (may be NULL = legacy default stream).  Work is
 *    stream-ordered; sofa_build, sofa_learn_model, sofa_get_model and sofa_knn_host return
 *    after synchronising that stream; sofa_knn, sofa_transform and sofa_merge_topk are
 *    asynchronous (sofa_knn synchronises only when `stats` is non-NULL).
 *  - Return value: SOFA_OK (0) or a negative SOFA_E* code; the message of the last failure on
 *    the calling thread is returned by sofa_last_error().  No C++ exception crosses the ABI.
 *  - Distances returned are the z-ED d (the square root; reading 13 in DESIGN.md);
 *    pruning compares squared values internally.  Per query, k results sorted by (d, index)
 *    ascending, ties to the smaller global index (reading 14); a shard holding fewer than k
 *    candidates pads with (+inf, -1).
 *  - Limits: 4 <= len <= 1024, len % 4 == 0; 1 <= l <= min(64, len-1); alphabet a power of two
 *    in [2, 256]; 1 <= k <= 128; block_size a power of two in [32, 8192].
 */
#ifndef SOFA_H_
#define SOFA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOFA_OK 0
#define SOFA_EINVAL (-1)      /* bad argument (message says which) */
#define SOFA_EDEGENERATE (-2) /* equi-depth sample smaller than the alphabet */
#define SOFA_ENOMEM (-3)      /* device allocation failed */
#define SOFA_ECUDA (-4)       /* a CUDA runtime / launch error */

#define SOFA_MAX_L 64
#define SOFA_MAX_ALPHABET 256
#define SOFA_MAX_LEN 1024
#define SOFA_MAX_K 128

#define SOFA_BINNING_EQUI_DEPTH 0 /* BASELINE.json */
#define SOFA_BINNING_EQUI_WIDTH 1 /* Alg. 1 l.8-11 */
#define SOFA_BINNING_ISAX 2       /* the iSAX baseline summarization: l
                                     PAA segments of n/l values (requires n % l == 0), N(0,1)
                                     equal-depth breakpoints, mindist weight n/l per position.
                                     Static: nothing is learned from the data. */

/* Opaque index: owns the SFA words (sorted), per-series (mu, 1/sigma), the permutation,
 * per-block envelopes, block keys, the model's device tables and query scratch.  It BORROWS
 * the `series` buffer given to sofa_build (caller keeps it alive and unmodified until
 * sofa_free): 100M x 256 float32 = 102.4 GB does not fit twice. */
typedef struct sofa_index sofa_index;

/* Learned MCB model (Alg. 1 returns "bins, best_l").  Plain data so it can be
 * broadcast as bytes between ranks. */
typedef struct {
  int32_t len;       /* series length n */
  int32_t l;         /* number of selected real values = symbols per word (reading 4) */
  int32_t alphabet;  /* a */
  int32_t binning;   /* SOFA_BINNING_*; _ISAX: best_pos[j] = j is PAA segment j */
  int32_t best_pos[SOFA_MAX_L];   /* interleaved positions (2k = Re X_k, 2k+1 = Im X_k),
                                     descending sample variance, ties -> lower position */
  double weights[SOFA_MAX_L];     /* Eq. 1 weight per selected position: 1 (DC/Nyquist) or 2 */
  double edges[SOFA_MAX_L * 255]; /* row j: a-1 ascending bin edges beta_j(1..a-1), float64 */
} sofa_model;

typedef struct {
  int64_t sample_size;     /* S; 0 => round(sample_ratio * global_n), clamped to [a, global_n] */
  double sample_ratio;     /* default 0.01 (Alg. 1 r) */
  int32_t block_size;      /* B series per leaf block, default 256 (reading 19) */
  int32_t candidate_limit; /* max complex index eligible for selection; 0 => n/2 (reading 3) */
  int32_t binning;         /* SOFA_BINNING_EQUI_DEPTH (default), _EQUI_WIDTH or _ISAX */
  int32_t dense_permille;  /* dense path: a strided probe of 2048 stored words
                              estimates the fraction of rows the sparse path would refine.  A query
                              is flagged before its envelope-tree descent if >= 10% of the probe
                              passes the bound of its own-key seed, else — once the batch's dense
                              pass is certain — after top-M seeding if >= this many permille pass
                              the tightened bound (and the estimate is >= 4096 rows either way).  The batch runs the tensor-core pass only if
                              the flagged queries' estimated refines add up to a fifth of a pass over the
                              rows (sofa_tuning.dense_batch_rows); else the scan pool finishes them
                              sparsely.  0 => 5 (0.5%), < 0 => never, >= 1000 => every query
                              (testing).  Results are identical either way; only speed changes. */
  int64_t global_offset;   /* global index of this shard's row 0 (0 on one GPU) */
  int64_t global_n;        /* total rows over all shards (0 => this call's n) */
  const sofa_model* model; /* nullable: NULL => learn from this call's rows at the global
                              strided sample indices floor(j*global_n/S) (1 GPU only) */
} sofa_build_opts;

typedef struct {
  int64_t queries;
  int64_t blocks_total;     /* sum over queries of the number of blocks (N/B) */
  int64_t blocks_survived;  /* blocks whose words were scanned (envelope LB <= threshold) */
  int64_t words_scanned;    /* SFA words whose LB was evaluated */
  int64_t candidates;       /* words with LB <= threshold */
  int64_t refined;          /* exact distance computations started */
  int64_t abandoned;        /* of those, early-abandoned */
  int64_t env_nodes;        /* envelope-tree nodes whose LB was evaluated (all levels) */
  int64_t list_blocks;      /* leaf blocks left after the tree descent (before BSF re-checks) */
  int64_t rounds;           /* LB-ordered selection rounds */
  int64_t batches;          /* word-scan batches */
  int64_t waves;            /* refine waves (8 candidates each) */
  int64_t phase_cycles[4];  /* SM cycles summed over queries: prep+tables, seed, tree, scan+refine */
  int64_t max_query_cycles; /* slowest query (SM cycles) */
  int64_t max_list_blocks;  /* largest per-query leaf list */
  int64_t max_batches;      /* most word-scan batches of one query */
  int64_t dense_queries;    /* queries finished by the dense path (tensor-core screen + exact refine) */
  int64_t dense_candidates; /* (query, row) pairs the dense screen passed to the exact refine */
  int64_t dense_refined;    /* exact distances computed by the dense path (incl. fallback rescans) */
  int64_t scan_tasks;       /* leaf chunks the front published to the scan pool (spread over all CTAs) */
  int64_t scan_queries;     /* queries that published at least one scan task */
  double kernel_ms[3];      /* GPU time (CUDA events on the call's stream) of the front kernel, the
                               dense pass (screen + exact refine) and the scan kernel */
} sofa_knn_stats;

/* Per-index tuning of the query kernels (read once by sofa_set_tuning, never from the environment).
 * Every field changes only the ORDER of work or which kernel build runs, never a result (the
 * tests check bit-identical outputs across settings).  sofa_default_tuning gives the defaults. */
typedef struct {
  int32_t front_batches;   /* word batches of LB-ordered leaves the front scans per query before the
                              rest becomes scan tasks (0 = 16) */
  int32_t rev_rounds;      /* refine rounds of a leaf part before it is deferred to the revisit pass
                              (default 2; 0 defers every part with a candidate) */
  int32_t topm_min;        /* top-M seeding for leaf lists longer than this (0 => nb/16 clamped to
                              [256, 2048]) */
  int32_t topm_leaves;     /* top-M seeding over about this many lowest-LB leaves (default 64) */
  int32_t refine_rows_front; /* rows refined together per warp in the front: 0 auto, 2 or 4 (n <= 512) */
  int32_t refine_rows_scan;  /* the same for the scan pool: 0 auto (2), 2 or 4 */
  int32_t front_wide;      /* 16-warp build of the front: -1 auto (batches of at most one query per
                              SM), 0 never, 1 always */
  int32_t scan_wide;       /* the same for the scan pool */
  int64_t dense_cand_cap;  /* dense-path candidate buffer entries (0 => 16M); a query whose candidates
                              overflow it is rescanned brute force (testing) */
  int64_t dense_batch_rows; /* the batch runs the dense pass iff its flagged queries' estimated sparse
                              refines add up to at least this many rows (0 => n / 5: the measured
                              break-even of one bf16 pass over the rows against random-row refines);
                              a batch below it scans its flagged queries sparsely */
  int32_t dense_pair;      /* dense screen on CTA pairs (tcgen05 cta_group::2, M = 256 rows per MMA, each
                              SM holding half of the query operand) instead of single CTAs (M = 128),
                              for rows of n <= 512 (default 0: measured equal on configs[3] and slower
                              on configs[2]) */
  int32_t dense_diag;      /* TIMING DIAGNOSTIC ONLY, 0 in any real use: nonzero bits make the dense
                              screen skip work so its pipeline stages can be timed apart (results are
                              then WRONG): 1 = no screening math, 2 = no TMEM loads either,
                              4 = producers ignore their twins' progress, 8 = no candidate path */
  int32_t dense_mcast;     /* single-CTA dense screen launched as clusters of 2 (default 1): with an even
                              number of query groups the two CTAs of a cluster serve two groups over the
                              same row tiles and share each tile by TMA multicast (one L2 read per tile
                              for both); 0 = one CTA per worker (cooperative launch) */
  int32_t dense_klist;     /* k > 1: the screen's upper-bound lists (the k smallest UB_g of candidate rows,
                              which lower a query's threshold): 0 = per CTA in shared memory when they fit
                              (default), 1 = one list per query in global memory under a lock */
  int32_t scan_fused;      /* front CTAs that find no query left scan the tasks other fronts publish, in the
                              same launch (default 1); 0 = only the separate scan launch scans them */
} sofa_tuning;

int sofa_default_tuning(sofa_tuning* out);

/* Fill *out with defaults (sample_ratio 0.01, block_size 256, equi-depth, everything else 0). */
int sofa_default_opts(sofa_build_opts* out);

/* Alg. 1 on an already drawn sample: z-normalise each of the S rows (float64),
 * full orthonormal DFT at the eligible positions (float64), per-position sample variance
 * (ddof=1) across the S rows, best_l = the l largest (ties -> lower position), then one row
 * of a-1 edges per selected position: equi-depth sorted[ceil(i*S/a)] or equi-width
 * min + i*(max-min)/a.  Deterministic (fixed-order float64 reductions).
 *   sample_dev: S x len float32, device.  opts: nullable (binning, candidate_limit).
 *   out: host struct written on success.
 * Errors: EINVAL (limits), EDEGENERATE (equi-depth and S < alphabet). */
int sofa_learn_model(const float* sample_dev, int64_t S, int32_t len, int32_t l, int32_t alphabet,
                     const sofa_build_opts* opts, void* cuda_stream, sofa_model* out);

/* sofa_build(series, n, len, l, alphabet) — BASELINE.json north_star call.
 * a1 (mu, 1/sigma) + a3 (projection onto the selected positions, quantisation) fused in one
 * pass over the series, then a4: 64-bit 2-bit-interleaved word keys, radix sort, gather of
 * sorted words, per-block min/max envelopes.  Learns the model first unless opts->model.
 *   series_dev: n x len float32 device, BORROWED until sofa_free.  n may be 0 only with
 *   opts->model (an empty shard).  out: receives the new index.
 * Errors: EINVAL, EDEGENERATE, ENOMEM, ECUDA. */
int sofa_build(const float* series_dev, int64_t n, int32_t len, int32_t l, int32_t alphabet,
               const sofa_build_opts* opts, void* cuda_stream, sofa_index** out);

/* sofa_knn(queries, q, k) — BASELINE.json north_star call; exact k-NN under z-ED.
 * Three stream-ordered launches, no host synchronisation: (1) the front, one CTA per query at a
 * time: a5 tables -> a6 own-key-block seed and envelope-tree descent -> the 8 lowest-LB leaves
 * (a7 word LB scan in chunks of 8 with abandoning, a8 LB-ordered refine with early abandoning
 * and top-k) -> the rest of the leaf list published as scan tasks; a query the SFA bound
 * cannot prune is flagged for (2) the dense pass (tensor-core TF32 screen with a proven error
 * bound + exact refine) if the flagged queries justify a full pass; (3) the scan
 * pass: every CTA pulls tasks of any query (a7 + a8 against the query's shared top-k); the CTA
 * finishing a query's last task writes its result.  Batches larger than 1024 queries run as
 * consecutive sub-batches on the same stream (the scan pool holds one leaf list per query).
 *   queries_dev: q x len float32 device (raw; z-normalised inside).
 *   bsf_init_dev: nullable, q floats: an upper bound on each query's k-th squared distance
 *   (e.g. from another shard) used to prune; results above it may be absent (padding).
 *   out_dist_dev: q x k float32 device; out_idx_dev: q x k int64 device (global indices).
 *   stats: nullable host struct (if given, the call synchronises and fills it).
 * Errors: EINVAL (k < 1, k > 128, k > global_n, q < 1), ECUDA. */
int sofa_knn(sofa_index* ix, const float* queries_dev, int32_t q, int32_t k, const float* bsf_init_dev,
             float* out_dist_dev, int64_t* out_idx_dev, sofa_knn_stats* stats, void* cuda_stream);

/* Seed bound for sharded search (the optional best-so-far exchange of BASELINE.json's
 * north_star): per query, the k-th smallest squared z-ED among the rows this index's seed step
 * refines (the lowest-LB words of the query's own-key leaf, MESSI's approximate search P:169 — the
 * query tables and that one leaf, no tree descent), +inf if fewer than k.  The minimum of it over
 * shards bounds the GLOBAL k-th
 * best, so passing that minimum as `bsf_init` to every shard's sofa_knn prunes shards that do not
 * hold the neighbours without changing the merged result.
 *   queries_dev: q x len float32; out_bound_dev: q float32.  Device pointers.  Errors: EINVAL, ECUDA. */
int sofa_knn_seed(sofa_index* ix, const float* queries_dev, int32_t q, int32_t k, float* out_bound_dev,
                  void* cuda_stream);

/* Same as sofa_knn with HOST buffers: copies the queries host->device, runs the search and
 * copies the results device->host inside the call (end-to-end path).  Synchronous. */
int sofa_knn_host(sofa_index* ix, const float* queries_host, int32_t q, int32_t k,
                  float* out_dist_host, int64_t* out_idx_host, sofa_knn_stats* stats, void* cuda_stream);

/* a9: per query, the k smallest (dist, idx) pairs of `parts` lists, each sorted ascending
 * (padding (+inf,-1) last); ties -> smaller idx.  dist_dev: parts x q x k float32,
 * idx_dev: parts x q x k int64, outputs q x k.  All device pointers.  Errors: EINVAL, ECUDA. */
int sofa_merge_topk(const float* dist_dev, const int64_t* idx_dev, int32_t parts, int32_t q, int32_t k,
                    float* out_dist_dev, int64_t* out_idx_dev, void* cuda_stream);

/* Per-query trace of the last sofa_knn call made WITH `stats` on this index: q rows of 24 int64
 * (SM cycles of prep+tables, seed, tree, scan+refine; blocks_survived, words_scanned, candidates,
 * refined, abandoned, env_nodes, list_blocks, rounds, batches, waves; CTA id; SM id; dense-path
 * decision inputs: flagged, leaves after the take round, take-word passes, take words; the
 * scan+refine cycles split into top-M seeding, dense decision, the front's leaf scans and the rest
 * (sorts, filters, task publishing)), copied to out_host (q x 24).  Errors: EINVAL if no such trace. */
int sofa_knn_trace(const sofa_index* ix, int64_t* out_host, int32_t q);

/* Lower-bound evaluation (TLB): for each of q queries and m index rows at
 * sorted positions floor(j*n/m), j < m, the squared SFA (or iSAX) lower bound from the query's
 * float32 table (entries rounded down, no early abandoning: Sum_j w_j mind_j^2) and
 * the exact squared z-ED (the refine's arithmetic).  TLB = sqrt(lb2 / ed2).
 *   queries_dev: q x len float32.  out_lb2_dev, out_ed2_dev: q x m float32.  out_rows_dev: m int64
 *   (global row index of column j).  All device pointers.  Errors: EINVAL, ECUDA. */
int sofa_lower_bounds(sofa_index* ix, const float* queries_dev, int32_t q, int64_t m, float* out_lb2_dev,
                      float* out_ed2_dev, int64_t* out_rows_dev, void* cuda_stream);

/* Replace the index's query tuning (host struct, copied).  Errors: EINVAL (NULL, out of range). */
int sofa_set_tuning(sofa_index* ix, const sofa_tuning* t);

/* Copy the index's model to *out (host). */
int sofa_get_model(const sofa_index* ix, sofa_model* out);

/* Parity entry point for a1+a3 (the same kernel sofa_build runs): for n rows, the projected
 * values (float64, n x l, nullable) and the SFA words (uint8, n x l, nullable) under `model`.
 * All array pointers device.  Errors: EINVAL, ECUDA. */
int sofa_transform(const float* series_dev, int64_t n, const sofa_model* model, double* out_values_dev,
                   uint8_t* out_words_dev, void* cuda_stream);

/* Index introspection: number of rows / blocks / block size / word stride, and the GPU time of the
 * build phases (CUDA events on the build stream; the analog of Fig. 7): model (sample +
 * learning, a2, plus the index allocations), transform (a1 + a3), sort (a4 key sort), gather +
 * envelopes (a4). */
typedef struct {
  int64_t n, n_blocks, global_offset, global_n;
  int32_t len, l, alphabet, block_size, word_stride;
  double build_ms[4];
  int32_t dense_enabled;  /* 1 if the dense path is available (its bfloat16 row copy, n x len x 2 bytes,
                             was allocated; 0 if disabled by opts or device memory) */
} sofa_index_info;
int sofa_get_info(const sofa_index* ix, sofa_index_info* out);

/* Verification entry of the dense screen (reading 29): the tcgen05
 * kind::f16 dot products the screen computes, for m rows and q queries given as float32 (rounded to
 * bfloat16 to nearest inside, exactly as the index's row copy and the query prep round them), with
 * no screening: out[i * q + j] = the fp32 tensor-core accumulation of bf16(rows[i]) . bf16(queries[j]).
 * Lets a test measure the hardware's accumulation error against the bound the screen assumes.
 *   rows_dev: m x len float32; queries_dev: q x len float32; out_dev: m x q float32 (device).
 *   Synchronous.  Errors: EINVAL (m < 1, q < 1 or q > 256, bad len), ENOMEM, ECUDA. */
int sofa_dense_dots(const float* rows_dev, int64_t m, int32_t len, const float* queries_dev, int32_t q,
                    float* out_dev, void* cuda_stream);

/* Copy the index arrays into caller device buffers (any may be NULL):
 * words_sorted n x word_stride uint8, perm n int32 (sorted position -> local row),
 * envelopes n_blocks x 2 x word_stride uint8 (min row then max row), block_keys n_blocks uint64. */
int sofa_export_index(const sofa_index* ix, uint8_t* words_sorted_dev, int32_t* perm_dev, uint8_t* env_dev,
                      uint64_t* block_keys_dev, void* cuda_stream);

/* Release everything the index owns (never the borrowed series). NULL is a no-op. */
void sofa_free(sofa_index* ix);

/* Thread-local message of the last failure ("" if none). */
const char* sofa_last_error(void);

/* Process-wide count of kernels this library has launched (bench evidence). */
int64_t sofa_launch_count(void);

/* Live per-kernel timing of sofa_knn calls without stats (bench.py's roofline, measured over its
 * timed region).  While enabled, every sofa_knn sub-batch records five CUDA events on the call's
 * stream (before the front, after it, after the dense screen, after the dense refine, after the
 * scan) and nothing else: no synchronisation, no counters.  Each call to this function first drains
 * the recorded events (blocking until the last recorded sub-batch has finished), adds their elapsed
 * times to the totals and, if out_ms / out_groups are non-NULL, writes the totals: out_ms[4] =
 * summed GPU ms of the front, the dense screen, the dense exact refine and the scan launch groups,
 * *out_groups = sub-batches timed.  Then enable = 1 clears
 * the totals and starts timing, 0 clears them and stops, -1 leaves the state unchanged (read only).
 * Errors: SOFA_EINVAL for a NULL index; CUDA errors as SOFA_ECUDA. */
int sofa_kernel_timing(sofa_index* ix, int32_t enable, double* out_ms, int64_t* out_groups);

#ifdef __cplusplus
}
#endif
#endif /* SOFA_H_ */
