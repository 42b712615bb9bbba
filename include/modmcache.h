/*
 * modmcache — C ABI of the B200-native MoDM cache-retrieval hot path.
 *
 * The reference (`mixserve`, /root/reference/pkg/src/mixserve/cache.py) has no
 * FFI layer: its boundary is the Python class API of `SemanticCache`.  Each
 * entry point below replaces one piece of that class's storage / arithmetic;
 * the Python drop-in (paper_2503_11972_b200/cache.py) keeps every validation
 * rule, exception and the CacheEntry metadata, and calls these through ctypes
 * (see INTEGRATION.md for the binding).
 *
 * Conventions: plain pointers and sizes only; every function returns 0 on
 * success or a negative MC_ERR_* code, with a thread-local message available
 * from mc_last_error().  Host buffers belong to the caller.  Device memory
 * belongs to the handle.  Calls on one handle are serialised by a mutex
 * ("many readers or one writer", cache.py:144).  mc_retrieve_batch is
 * synchronous: it returns after the results are in the caller's arrays.
 */
#ifndef MODMCACHE_H
#define MODMCACHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MC_OK 0
#define MC_ERR_ARG (-1)
#define MC_ERR_CUDA (-2)
#define MC_ERR_STATE (-3)
#define MC_ERR_NOMEM (-4)
#define MC_ERR_UNSUPPORTED (-5)

/* Per-query result flags (mc_retrieve_batch out_flags). */
#define MC_FLAG_HIT 0x01u       /* best >= tau (cache.py:258); NaN best also counts, as in the reference */
#define MC_FLAG_EMPTY 0x02u     /* cache had no live entries (cache.py:252-253) */
#define MC_FLAG_TIE 0x04u       /* >= 2 live entries share the best float64 score; newest returned */
#define MC_FLAG_NEAR_TIE 0x08u  /* runner-up within 1e-12 of best but not equal (ulp-ambiguous) */
#define MC_FLAG_NEAR_TAU 0x10u  /* best within 1e-12 of some tau_k (ulp-ambiguous) */
#define MC_FLAG_FALLBACK 0x20u  /* top-K' certificate failed; exhaustive exact rescan answered */
#define MC_FLAG_NONFINITE 0x40u /* query had NaN/Inf; answered by exhaustive float64 scan */
#define MC_FLAG_NEED_RESCAN 0x80u /* merge of mc_retrieve_local_submit records: some shard's certificate
                                     failed; run mc_rescan_local on every shard, gather, merge again */

/* Scan-path selection for mc_set_path (default MC_PATH_AUTO: B <= 4 -> the
 * TMA-streamed int8 scan when Dp <= 1024 (Dp = D rounded up to 64), else the
 * fp16 GEMV; B >= 5 -> the fp16 tcgen05 scan on CTA pairs).  Every path
 * returns the same certified answers. */
#define MC_PATH_AUTO 0
#define MC_PATH_GEMV 1 /* CUDA-core fp16 GEMV scan, register top-K' (AUTO's small-batch path when Dp > 1024;
                          a cross-check elsewhere) */
#define MC_PATH_GEMM 2 /* tcgen05/TMEM/TMA fp16 scan on CTA pairs (cta_group::2), fused top-K' epilogue */
/* 3, 4, 5 and 7 named round-1 cross-check scans (single-CTA and 4-CTA tensor-core scans, the
 * register-streamed int8 GEMV, the int8 tensor-core scan); they were removed, and
 * mc_set_path rejects them with MC_ERR_ARG. */
#define MC_PATH_STREAM8 6 /* int8 scan streamed by TMA bulk copies, lane-per-row dp4a, float64 rescoring
                             pool (AUTO's choice for B <= 4 when Dp <= 1024) */

typedef struct mc_cache mc_cache;

/* One shard's answer for one query, as exchanged between GPUs (32 bytes). */
typedef struct mc_record {
  double sim;     /* best float64 similarity among this shard's live entries */
  double second;  /* runner-up similarity (-inf if none)                      */
  int64_t pos;    /* global append position of the best entry (-1 if none)    */
  uint32_t flags; /* MC_FLAG_TIE / _FALLBACK / _NONFINITE / _EMPTY              */
  int32_t reserved;
} mc_record;

/* Replaces SemanticCache.__init__'s float64 `_buf` (cache.py:147-168):
 * allocates a device-resident FIFO ring of `capacity` rows of `dim` floats
 * (fp16 scan copy + float64 master) on CUDA device `device`. */
int mc_create(mc_cache** out, int64_t capacity, int32_t dim, int32_t device);
int mc_destroy(mc_cache* h);

/* Replaces ThresholdTable (cache.py:73-117): n strictly increasing (k, tau)
 * pairs; tau of pair 0 is the hit threshold (cache.py:103-106), select_k is
 * the largest k with sim >= tau_k (cache.py:112-117).  n <= 16. */
int mc_set_thresholds(mc_cache* h, const int32_t* ks, const double* taus, int32_t n, int32_t total_steps);

/* Replaces _append_row (cache.py:181-192): appends n float64 rows (row-major,
 * stride dim) at the FIFO tail.  Rows beyond capacity displace the oldest,
 * exactly like insert()'s append-then-evict (cache.py:230-233).  The copy
 * into the ring is deferred and fused with the next lookup. */
int mc_append(mc_cache* h, const double* rows, int64_t n);

/* Replaces _evict_front (cache.py:194-196), n times. */
int mc_evict_front(mc_cache* h, int64_t n);

/* Live entry count (len(_store), cache.py:170-171). */
int64_t mc_size(const mc_cache* h);

/* Replaces retrieve (cache.py:244-260) for B queries at once, each against
 * the same cache state.  queries: B x dim float64 row-major.  Outputs:
 *   out_live  live index (0 = oldest) of the best entry, -1 if cache empty
 *   out_sim   best float64 similarity (NaN if empty)
 *   out_k     chosen k (select_k), 0 = none (miss or no k reached)
 *   out_flags MC_FLAG_* bits; MC_FLAG_HIT decides hit/miss. */
int mc_retrieve_batch(mc_cache* h, const double* queries, int32_t B, int64_t* out_live,
                      double* out_sim, int32_t* out_k, uint32_t* out_flags);

/* The full serving decision of one lookup, written by the device's decision
 * epilogue (SURVEY.md §8 a1 + f3): the reference's answer (cache.py:255-260)
 * plus what its callers derive from it. */
typedef struct mc_decision {
  int64_t live;   /* live index of the best entry (0 = oldest), -1 if the cache is empty */
  double sim;     /* best float64 similarity (NaN if empty) */
  double sigma;   /* noise re-entry level schedule[k] on a hit (cache.py:325-334); NaN on a miss,
                     without a schedule (mc_set_sigma_schedule) or when k lies past it */
  int32_t k;      /* select_k (cache.py:112-117), 0 = none */
  int32_t steps;  /* denoising steps to run: total_steps - k on a hit, total_steps on a miss
                     (engine.py:38-45 service_time) */
  uint32_t flags; /* MC_FLAG_*; MC_FLAG_HIT decides the route */
  int32_t route;  /* 1 = hit queue (cached-image refinement), 0 = miss queue (scheduler.py:80-89) */
} mc_decision;

/* mc_retrieve_batch returning the full decision per query (out: B mc_decisions). */
int mc_retrieve_decisions(mc_cache* h, const double* queries, int32_t B, mc_decision* out);

/* The sigma schedule over timesteps 0..T (n = T + 1 values; linear_sigma_schedule,
 * cache.py:305-309; the host validates it with validate_sigma_schedule).  n = 0 clears it. */
int mc_set_sigma_schedule(mc_cache* h, const double* schedule, int32_t n);

/* Asynchronous form of mc_retrieve_batch (the serving loop's overlap of host
 * work with the scan): submit enqueues the lookup against the current cache
 * state and returns a ticket; wait returns its answers exactly as
 * mc_retrieve_batch would have.  Up to three single-query lookups may be in
 * flight per handle (each newer launch queues behind the older kernels), or
 * two when one is a batch (B > 1; a batch from registered memory has its
 * queries DMA'd on a copy stream while the older batch scans); each ticket is
 * collected by its own wait, in any order, and a further submit fails with
 * MC_ERR_STATE.  mc_append / mc_evict_front between submit and wait only change
 * what LATER lookups see (a forced device flush first completes the lookups in
 * flight). */
int mc_retrieve_submit(mc_cache* h, const double* queries, int32_t B, uint32_t* out_ticket);
int mc_retrieve_wait(mc_cache* h, uint32_t ticket, int64_t* out_live, double* out_sim, int32_t* out_k,
                     uint32_t* out_flags);

/* Force a scan path (tests / benchmarks).  MC_PATH_AUTO picks by batch size. */
int mc_set_path(mc_cache* h, int32_t path);

/* --- multi-GPU sharding (one process per GPU) -------------------------------
 * Entries are dealt round-robin by global append position p: shard g of G
 * stores p = g, g+G, g+2G, ...  mc_configure_shard must precede any append. */
int mc_configure_shard(mc_cache* h, int32_t n_shards, int32_t shard_id);

/* Local top-1 per query into a DEVICE buffer of B mc_records (e.g. the
 * send buffer of an NCCL all-gather), enqueued on `stream` (cudaStream_t,
 * NULL = the handle's stream); not synchronous. */
int mc_retrieve_local_async(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream);

/* mc_retrieve_local_async without the exhaustive rescan behind the scan (two launches fewer per
 * lookup): a record whose top-K' certificate failed keeps a rescan request, which the merge
 * reports as MC_FLAG_NEED_RESCAN.  Every shard then runs mc_rescan_local on the same queries and
 * its own records (in place), the records are gathered again and merged again.  The rescan
 * runs against the window the lookup that wrote `dev_records` scanned (the handle remembers its
 * last four local lookups), even if later lookups applied appends meanwhile, as long as at most
 * PIPE_SLACK (8) rows were appended since; otherwise it fails with MC_ERR_STATE. */
int mc_retrieve_local_submit(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream);
int mc_rescan_local(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream);

/* mc_retrieve_local_async with the B query rows already in DEVICE memory (float64, row stride
 * dim; dim a multiple of 64), written on `stream` — e.g. assembled by an all-gather of the
 * ranks' slices of the batch, so each rank uploads only its share from the host. */
int mc_retrieve_local_device(mc_cache* h, const double* d_queries, int32_t B, void* dev_records, void* stream);

/* Merge G x B gathered records (device pointer, shard-major) on the device and
 * return final answers like mc_retrieve_batch.  p0 = global position of the
 * oldest live entry (live index = pos - p0).  Synchronous. */
int mc_merge_records(mc_cache* h, const void* dev_records, int32_t G, int32_t B, int64_t p0,
                     void* stream, int64_t* out_live, double* out_sim, int32_t* out_k,
                     uint32_t* out_flags);

/* Pipelined form of mc_merge_records (replaces the same reference call, cache.py:244-260, for a
 * caller that keeps several sharded lookups in flight).  _submit enqueues the merge of G x B
 * records on `stream` and returns at once; the decisions land in result slot `slot`
 * (0 <= slot < MC_MERGE_SLOTS), which must be free.  _wait blocks until that merge is done,
 * writes the answers like mc_retrieve_batch and frees the slot.  The record buffer must stay
 * untouched until the merge completes (stream order on `stream` guarantees it for later work
 * enqueued there). */
#define MC_MERGE_SLOTS 2
int mc_merge_records_submit(mc_cache* h, const void* dev_records, int32_t G, int32_t B, int64_t p0,
                            void* stream, int32_t slot);
int mc_merge_records_wait(mc_cache* h, int32_t slot, int64_t* out_live, double* out_sim,
                          int32_t* out_k, uint32_t* out_flags);

/* Measurement hook (bench.py): runs `iters` hot-path steps with all inputs
 * already resident in HBM and times them with CUDA events on the handle's
 * stream.  Step i = [append rows[i] if rows != NULL] + scan + certified merge
 * + decision epilogue for queries[i] (B x dim).  Between steps (outside the
 * timed events) a buffer of flush_bytes is written to evict L2 (0 = none).
 * The appends advance the ring exactly like mc_append; results are discarded.
 * out_ms[0] = mean step, [1] = mean scan kernel, [2] = mean merge+epilogue,
 * [3] = mean append; out_counts[0] = kernel launches per step,
 * [1] = steps whose certificate would have needed the exhaustive rescan. */
int mc_profile_steps(mc_cache* h, const double* queries, const double* rows, int32_t B, int32_t iters,
                     int64_t flush_bytes, double* out_ms, int64_t* out_counts);

/* Measurement hook (bench.py): `iters` back-to-back lookup steps rotating over
 * nh caches of one shape on one device (together larger than L2, so each step
 * streams its cache from HBM), timed by a single pair of CUDA events — no
 * per-step events or flushes inside the timed region.  Step i = [append
 * rows[i] if rows != NULL] + lookup of queries[i] (B x dim) on hs[i % nh].
 * out_ms[0] = mean step; out_counts[0] = kernel launches per step,
 * [1] = answers whose certificate would have needed the exhaustive rescan. */
int mc_profile_rotate(mc_cache* const* hs, int32_t nh, const double* queries, const double* rows, int32_t B,
                      int32_t iters, double* out_ms, int64_t* out_counts);

/* Measurement hook, active only when MC_GEMV_TIMING=1 was set before the first
 * lookup: reads (reset = 0) or resets (reset = 1) eight globaltimer stamps of the
 * last small-batch launch(es): [0] first CTA start, [1] last scan end, [2] last
 * rescoring end, [3] tail end, [4] merge start and [5] records loaded (streamed
 * int8 scan only), [6] merge reductions done and [7] decision stored (streamed int8 scan only) (ns).  Not needed by the drop-in; used by
 * scripts/profile_case.py. */
int mc_debug_gemv_timing(unsigned long long* out8, int reset);

/* f4, measurement infrastructure (the generative model of
 * pkg/src/mixserve/workload.py:124-154): appends n synthetic unit rows generated
 * on the device, with FIFO semantics (the oldest rows are evicted as by n
 * appends).  Row r (global index row0 + r) belongs to a hashed cluster c and is
 * normalize(beta * q + (1 - beta) * g'), q = normalize(centers[c] + spread * g).
 * centers: host float64 [n_centers][dim].  dim <= 1024. */
int mc_generate_rows(mc_cache* h, int64_t n, const double* centers, int32_t n_centers, double spread, double beta,
                     uint64_t seed, int64_t row0);

/* Copies the float64 master rows of live indices [first_live, first_live + n)
 * (0 = oldest) into out[n][dim] (parity checks of generated caches). */
int mc_read_rows(mc_cache* h, int64_t first_live, int64_t n, double* out);

/* Registers (page-locks) a caller's host buffer for the process: batched lookups whose
 * query block lies inside a registered buffer are copied to the device by one DMA straight
 * from it, without staging (cudaHostRegister).  Unregister before freeing the memory.  The
 * reference has no counterpart (its retrieve reads the query in place, cache.py:254). */
int mc_register_host(void* ptr, int64_t bytes);
int mc_unregister_host(void* ptr);

/* Debugging hook: copies the float64 master row of live index `live` (0 =
 * oldest; pending appends are published first) into out[0 .. dim). */
int mc_debug_read_row(mc_cache* h, int64_t live, double* out);

/* Counters since creation: [0] lookups, [1] certificate fallbacks,
 * [2] non-finite queries, [3] exact ties, [4] candidates rescored,
 * [5] GEMV launches, [6] GEMM launches, [7] kernel launches total. */
int mc_stats(const mc_cache* h, int64_t* out8);

/* Thread-local description of the last error on this thread. */
const char* mc_last_error(void);

/* Library version string. */
const char* mc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MODMCACHE_H */
