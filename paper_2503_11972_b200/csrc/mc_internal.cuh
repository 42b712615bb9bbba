// Internal declarations shared by the modmcache translation units.
//
// Data layout in HBM (per handle / per GPU):
//   ring16  [C][Dp] fp16  — scan copy of every ring slot, D zero-padded to Dp
//                           (multiple of 64 → 128-byte rows for TMA / UMMA K-blocks)
//   ring64  [C][Dp] fp64  — master copy, used only to rescore top-K' candidates
//   state   RingState     — (head slot, live count, local append index of head)
// Live rows occupy slots head, head+1, ... (mod C), oldest first.  A row's
// global append position is p = (jhead + live_local) * G + g for shard g of G.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/modmcache.h"

namespace mc {

constexpr int KP = 8;             // candidates kept per scan chunk (top-K')
constexpr int MAX_PAIRS = 16;     // threshold table capacity
constexpr double AMBIG = 1e-12;   // ulp-ambiguity band reported in flags

// Internal record flag (not exported): certificate failed, needs exact rescan.
constexpr uint32_t FLAG_NEED_FALLBACK = 0x10000u;
// Internal record flag: query is non-finite / extreme; answer by exhaustive float64 scan.
constexpr uint32_t FLAG_NEED_EXHAUSTIVE = 0x20000u;
constexpr uint32_t FLAG_NEED_ANY = FLAG_NEED_FALLBACK | FLAG_NEED_EXHAUSTIVE;

// Physical ring slots beyond the logical capacity: rows a launch is still scanning stay intact
// while up to PIPE_SLACK rows are appended behind it (pipelined lookups, overlapping launches).
constexpr long long PIPE_SLACK = 8;

struct RingState {
  long long head;   // physical slot of the oldest live row
  long long count;  // live rows
  long long jhead;  // local append index of the oldest live row
  long long cap;    // ring capacity C (slots)
};

struct Thresholds {
  int n;
  int total_steps;
  int ks[MAX_PAIRS];
  double taus[MAX_PAIRS];
  int has_sigma;             // a sigma schedule is set (mc_set_sigma_schedule)
  double sigma[MAX_PAIRS];   // schedule[ks[j]] (noise_reentry_level, cache.py:325-334); NaN if ks[j] is past it
};

// Where a scan pass leaves its per-chunk top-K' lists (approximate scores).
struct Partials {
  float* s;          // [B][n_chunks][KP] approximate score (scaled units, see scale)
  long long* p;      // [B][n_chunks][KP] global position (-1 = empty)
  float* floor_;     // [B][n_chunks]  K'-th score if rows were dropped, else -inf
  int n_chunks;
};

// One CTA's exact answer for one query on the GEMV path: the float64 best over
// the CTA's rescored candidates plus the certificate input (see scan_gemv.cu).
struct CtaRec {
  double s;     // best float64 similarity among the rescored candidates (-inf if none)
  double s2;    // runner-up float64 similarity among them
  long long p;  // global position of the best (-1 if none)
  float ovf;    // largest approx score (query units) a full warp list had to drop (-inf if none)
  int ties;     // rescored candidates bit-equal to s
};

// The device copies of every ring slot (all written by every append path).
struct RingBufs {
  __half* r16;     // [C][Dp] fp16 RN (tensor-core scan, exhaustive fallback)
  double* r64;     // [C][Dp] float64 master (certified rescoring)
  int8_t* r8;      // [C][p8] int8, symmetric per-row scale (small-batch scan), zero beyond Dp
  float2* rq;      // [C] (scale s >= max|e|/127, rounded up; ||e||_1, rounded up)
  int p8;          // int8 row stride: Dp rounded up to 128 (whole TMA swizzle rows)
};

struct ShardMap {
  int G;  // number of shards
  int g;  // this shard
};

// Final per-query answer written by the decision epilogue (the serving decision of
// SURVEY.md §8 a1 + f3): the reference's (entry, similarity, k) plus what its callers
// derive from them — steps to run (engine.py:38-45), route (scheduler.py:80-89) and the
// noise re-entry level sigma[k] (cache.py:325-334).
struct OutRec {
  long long live;  // live index (0 = oldest), -1 if none
  double sim;      // best float64 similarity
  int k;           // select_k result, 0 = none
  unsigned flags;  // MC_FLAG_*
  int steps;       // denoising steps to run: total_steps - k (total_steps on a miss)
  int route;       // 1 = hit queue (refine a cached image), 0 = miss queue (full generation)
  double sigma;    // schedule[k] on a hit with a schedule set, else NaN
};

// ---- launch wrappers (each .cu owns its kernels) ---------------------------
cudaError_t launch_append(const double* stage, long long n, long long first_slot, const RingState& new_state,
                          int D, int Dp, const RingBufs& rb, RingState* d_state, cudaStream_t s);

// Pending appends folded into a GEMV launch: stage rows [0, n) -> ring slots
// (first_slot + i) mod C; d_state receives the launch's window.
struct GemvAppendArgs {
  const double* stage = nullptr;
  long long n = 0;
  long long first_slot = 0;
  RingBufs rb{};
  RingState* d_state = nullptr;
  bool dirty = false;  // the host window changed since the device last saw it (appends or evictions)
};

// GEMV scan of up to 4 queries (q64 rows q0 .. q0+nb-1, stride Dp) over the
// window `st`, with the certified merge fused into the last CTA: records go to
// rec[b0 + b] and, if out != nullptr, decisions to out[b0 + b].  counter and
// gmax[b0 + b]: zeroed device words (the kernel leaves them zeroed).
cudaError_t launch_gemv_scan(const __half* ring16, const RingState& st, int D, int Dp, const double* q64, int nb,
                             CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter, unsigned* gmax,
                             const double* ring64, const Thresholds& thr, mc_record* rec, OutRec* out,
                             const GemvAppendArgs& app, cudaStream_t s);
// Per-query int8 quantisation for the small-batch scan (computed on the host
// by quantize_query, uploaded in the envelope next to the float64 query).
struct QPrep {
  double q1;      // ||s_q q̂||_1 (exact integer sum times s_q)
  double n2, n1;  // ||q||_2, ||q||_1 (rounded up)
  float s;        // s_q >= max|q|/127, rounded up (0: zero or non-finite query)
  int exotic;     // non-finite / extreme query: answered by the exhaustive float64 scan
};

// TMA-streamed int8 scan (scan_stream8.cu): same contract as launch_gemv_scan,
// grid = one CTA per SM.  The plan holds the ring's tensor maps.
struct S8Plan;
bool stream8_supported(int Dp);
int s8_grid(int sm_count);  // CTAs of one streamed-scan launch
int s8_grid_wide(int sm_count);  // CTAs of an isolated streamed-scan launch (every co-resident slot)
// One query (and <= 1 pending row, host pointers) carried in the kernel parameter block.
cudaError_t launch_stream8_direct(const S8Plan* p, const RingBufs& rb, const RingState& st, int D, const double* q64,
                                  const double* stage_row, CtaRec* cta, int grid, ShardMap sm, unsigned* counter,
                                  unsigned long long* gmax, unsigned epoch, const Thresholds& thr, mc_record* rec,
                                  OutRec* out,
                                  RingState* d_state, unsigned* done_seq, unsigned seq, uint4* outp,
                                  void (*quantise)(const double*, int, int, QPrep*, int8_t*), double* gq64,
                                  unsigned* sync, unsigned rec_par, bool overlap, cudaStream_t s);
S8Plan* s8_plan_create(int8_t* ring8, float2* ringq, long long C, int Dp, int P8, char* err, int errlen);
void s8_plan_destroy(S8Plan* p);
cudaError_t launch_stream8_scan(const S8Plan* p, const RingBufs& rb, const RingState& st, const double* q64, int nb,
                                CtaRec* cta, int b0, int grid, ShardMap sm, unsigned* counter,
                                unsigned long long* gmax, unsigned epoch, const Thresholds& thr, mc_record* rec,
                                OutRec* out, const GemvAppendArgs& app,
                                const QPrep* prep, const int8_t* q8, unsigned* done_seq, unsigned seq,
                                uint4* outp, unsigned* sync, unsigned rec_par, bool overlap, cudaStream_t s);

int gemv_grid(int sm_count);
cudaError_t launch_generate(long long n, long long first_slot, const RingState& ns, int D, int Dp, const RingBufs& rb,
                            const double* centers, int K, double spread, double beta, unsigned long long seed,
                            long long row0, RingState* d_state, cudaStream_t s);  // f4 synthetic rows
cudaError_t launch_l2_flush(void* buf, size_t bytes, cudaStream_t s);
cudaError_t launch_spin(long long ns, cudaStream_t s);  // measurement: hold a stream for ns of device time  // measurement: evict L2 by reading
unsigned long long* gemv_timing_buffer();  // MC_GEMV_TIMING=1 phase timestamps (measurement)

// tcgen05 GEMM scan of B queries (scan_tc.cu).  The plan owns the fp16
// query tile (q / ||q||), the per-query scale ||q|| and both TMA descriptors.
struct TcPlan;
TcPlan* tc_plan_create(__half* ring16, long long C, int Dp, int Bcap, int sm_count, char* err, int errlen);
void tc_plan_destroy(TcPlan* p);
int tc_bcap(const TcPlan* p);
int tc_chunks(const TcPlan* p, int B);
const double* tc_qscale(const TcPlan* p);
cudaError_t launch_tc_scan(TcPlan* p, const double* q64, int B, int D, const RingState* d_state,
                           const Partials& part, ShardMap sm, cudaStream_t s);

// Merge per-chunk lists -> certified float64 best per query (mc_record).
// qscale: per-query factor turning partial scores into similarity units (nullptr = 1).
cudaError_t launch_merge(const RingState* d_state, const double* ring64, int D, int Dp, const double* q64, int B,
                         const Partials& part, const double* qscale, double eps_rel, double eps_abs1,
                         mc_record* rec, ShardMap sm, const Thresholds* thr, OutRec* out, cudaStream_t s);

// Exhaustive exact rescan for the queries whose record needs it.
cudaError_t launch_exact_rescan(const __half* ring16, const double* ring64, const RingState* d_state, int D,
                                int Dp, const double* q64, int B, mc_record* rec, mc_record* scratch,
                                int grid, double eps_rel_gemv, double eps_abs1, ShardMap sm, cudaStream_t s);
int exact_grid(int sm_count);

// Final decision: merge G shard records per query, apply threshold / k.
// p0 < 0 means "read jhead from d_state" (single-GPU).

cudaError_t launch_finalize(const mc_record* rec, int G, int B, long long p0, const RingState* d_state,
                            Thresholds thr, OutRec* out, cudaStream_t s);

// Error-bound coefficients of the two scan paths.
double gemv_eps_rel(int Dp);
double gemm_eps_rel(int Dp);
double eps_abs1();

}  // namespace mc
