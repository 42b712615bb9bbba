// C ABI of libmodmcache.so (declared in include/modmcache.h).
//
// Host side of the device ring: owns the CUDA stream, the device buffers, a
// pinned "envelope" and a host mirror of the ring window.  Every call is
// serialised by the handle's mutex ("many readers or one writer", cache.py:144).
//
// The envelope is the only host->device path of the hot loop:
//   h_env / d_env  [env_rows][Dp] float64, zero-padded columns
//   rows [0, n_pending)            pending FIFO appends (mc_append stages here)
//   rows [n_pending, n_pending+B)  the lookup's queries
//   then QPrep[B] and q̂[B][Dp]      the queries' int8 quantisation (quantize_query)
// A lookup is one H2D copy of the used prefix, one fused GEMV launch (append +
// scan + certified rescoring + decision) or the tensor-core sequence, one D2H
// copy of the decisions and one stream synchronisation.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "mc_internal.cuh"

using namespace mc;

static thread_local std::string g_err;

// MC_HOST_TIMING=1: mean host-side phase times of mc_retrieve_batch, printed at mc_destroy
// (measurement only): [0] stage + quantise, [1] H2D enqueue, [2] launch, [3] wait for the result.
struct HostTiming {
  bool on = getenv("MC_HOST_TIMING") && atoi(getenv("MC_HOST_TIMING"));
  double acc[4] = {0, 0, 0, 0};
  long long n = 0;
};
static HostTiming g_ht;
static inline double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(MC_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
  } while (0)

struct mc_cache {
  std::mutex mu;
  int dev = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  long long C = 0;   // logical capacity: live rows never exceed it
  long long Cp = 0;  // physical ring slots = C + PIPE_SLACK: rows an in-flight lookup scanned stay
                     // intact until PIPE_SLACK more rows have been appended (pipelined lookups)
  int D = 0, Dp = 0;
  int P8 = 0;  // int8 ring row stride (Dp rounded up to 128)
  ShardMap shard{1, 0};

  // host mirror of the ring window
  long long head = 0, count = 0, jhead = 0, appended = 0;
  bool state_dirty = false;

  // device-resident ring (every copy of every slot; see RingBufs)
  __half* ring16 = nullptr;
  double* ring64 = nullptr;
  int8_t* ring8 = nullptr;
  float2* ringq = nullptr;
  RingState* d_state = nullptr;

  // envelope: pending appends, then queries (see the header comment)
  long long stage_cap = 0;  // pending rows before a forced flush
  int Bcap = 0;             // query rows
  double* h_env = nullptr;  // pinned [stage_cap + Bcap][Dp]
  double* d_env = nullptr;  // [stage_cap + Bcap][Dp]
  long long n_pending = 0;
  long long pending_first_slot = 0;
  cudaEvent_t env_ev = nullptr;  // last async upload of the envelope (async paths only)
  cudaEvent_t rec_ev = nullptr;  // a shard's local records are complete (mc_retrieve_local_async)
  bool env_inflight = false;

  // per-batch device buffers
  float* d_part_s = nullptr;
  long long* d_part_p = nullptr;
  float* d_part_floor = nullptr;
  CtaRec* d_cta = nullptr;     // [Bcap][gemv grid] per-CTA exact records (GEMV path)
  unsigned* d_gmax = nullptr;  // [Bcap][256] running max keys of the fused GEMV scans (zero between launches)
  unsigned long long* d_gmax8 = nullptr;  // [Bcap][128] epoch-tagged bound replicas of the streamed int8 scan
  unsigned s8_epoch = 0;                  // the last streamed-scan launch's epoch
  mc_record* d_rec = nullptr;
  mc_record* d_scratch = nullptr;
  OutRec* d_out = nullptr;
  OutRec* h_out = nullptr;  // pinned, mapped (the streamed scan writes decisions here directly)
  OutRec* d_outm = nullptr; // device view of h_out
  uint4* h_outp = nullptr;    // pinned, mapped: packed decisions (2 x 16 B each, self-validating sequence tags)
  uint4* d_outp = nullptr;
  bool packed = true;         // packed zero-copy results (else: decisions + fence + completion word)
  unsigned* h_seq = nullptr;  // pinned, mapped: completion word of the zero-copy lookup
  unsigned* d_seq = nullptr;
  unsigned seq = 0;
  // an asynchronous lookup in flight (mc_retrieve_submit): its batch, device query and seq
  unsigned inflight_seq = 0;
  int inflight_B = 0;
  const double* inflight_q = nullptr;
  bool inflight_ready = false;  // completed (and any fallback applied) while staging appends
  bool inflight_direct = false; // its result comes back zero-copy
  bool inflight_async = false;  // a batch whose decisions come back by an async D2H copy (batch_ev)
  // Batches pipeline two deep: the in-flight batch uses batch slot `batch_slot` (0: d_rec / d_out /
  // h_out, 1: the *2 buffers); an older batch still unanswered (old_async) uses the other one.
  cudaEvent_t batch_ev[2] = {nullptr, nullptr};
  int batch_slot = 0;
  long long inflight_appended = 0;  // h->appended when the in-flight batch was enqueued
  mc_record* d_rec2 = nullptr;
  OutRec* d_out2 = nullptr;
  OutRec* h_out2 = nullptr;
  bool old_async = false;       // the older lookup is a batch still in flight (answered by finish_old)
  int old_B = 0, old_bslot = 0;
  const double* old_q = nullptr;
  long long old_appended = 0;
  // A submitted batch answered when the next lookup was submitted (its decisions kept here until
  // its mc_retrieve_wait): batches pipeline one deep, the next one's upload and scan overlap the
  // caller's work on this one's answers.
  std::vector<OutRec> old_batch;
  // Query prefetch for pipelined batches: a batch submitted while the previous one runs has its
  // queries DMA'd from the caller's registered array into a query slot on a copy stream first,
  // so the copy overlaps the previous batch's scan.
  cudaStream_t cstream = nullptr;
  double* d_qslot[2] = {nullptr, nullptr};
  cudaEvent_t q_ev[2] = {nullptr, nullptr};
  int qslot_cap = 0;        // rows per query slot
  int qslot_next = 0;       // slot the next prefetch fills
  const double* pf_src = nullptr;  // caller rows the prefetched slot holds (nullptr: none)
  int pf_B = 0, pf_slot = 0;
  int inflight_slot = 0;        // its result slot: h_outp + 2 slot, d_rec + slot (single-query lookups)
  RingState inflight_st{};      // the window it scans
  // Pipelined single-query lookups: a second mc_retrieve_submit while one is in flight moves
  // that one here.  Its window stays intact (PIPE_SLACK spare slots) while the newer launch
  // writes the rows appended in between, so its exhaustive fallback, if needed, can still run
  // on exactly what it scanned.
  unsigned old_seq = 0;         // 0: none
  bool old_ready = false;       // answered (and any fallback applied); waiting for its mc_retrieve_wait
  int old_slot = 0;
  RingState old_st{};
  OutRec old_out{};
  long long old_written = 0;    // rows launches after it have written into the ring
  // A third single-query lookup in flight: the oldest of the three (older than `old`), in result
  // slot old2_slot.  Same contract as `old`: its window survives the <= PIPE_SLACK rows later
  // launches write, its answer is kept for its own mc_retrieve_wait.
  unsigned old2_seq = 0;
  bool old2_ready = false;
  int old2_slot = 0;
  RingState old2_st{};
  OutRec old2_out{};
  long long old2_written = 0;
  double* h_qslot[3] = {nullptr, nullptr, nullptr};  // pinned [Dp]: the single-query lookups' queries (fallback uploads)
  double* d_qfb = nullptr;      // [Dp] fallback query
  RingState* d_state_fb = nullptr;  // the fallback's window
  bool param_in = false;        // MC_PARAM_INPUT=1: single-query lookups carry their inputs in the launch
                                // parameters (measured equal to the pinned-envelope copy on B200)
  double* h_qkeep = nullptr;    // pinned, mapped [Dp]: the single-query launch's float64 query (read by the kernel)
  double* h_stage1[3] = {nullptr, nullptr, nullptr};  // pinned, mapped [Dp] per result slot: its pending row
  double* d_gq64 = nullptr;     // [Dp] the kernel's L2 relay of the pending row
  unsigned* d_sync = nullptr;   // [2] streamed-scan launch overlap: rows published / records read (epochs)
  bool tc_tail = false;         // the last kernel enqueued on the stream is the tensor path's merge (PDL-early)
  // The windows the last local lookups scanned, by record buffer: mc_rescan_local runs against the
  // window its records came from, while at most PIPE_SLACK rows have been appended since (the
  // spare physical slots keep those rows intact), whatever later lookups applied meanwhile.
  struct LocalWin {
    const void* rec = nullptr;
    RingState st{};
    long long appended = 0;
  } local_win[4];
  int local_win_next = 0;
  bool local_param = true;      // local lookups of one query carry it in the launch (MC_LOCAL_PARAM=0: envelope)
  long long s8_rows_per_cta = 128;  // streamed-scan grid = ceil(rows / this), at most the full grid: windows
                                    // under 19k rows merge fewer CTA records (C1 back-to-back 10.5 -> 8.7 us,
                                    // profiles/r02_s8_rows_ab.txt); MC_S8_ROWS_PER_CTA, 0 = always the full grid
  bool s8_isolated = false;     // the streamed scan being enqueued cannot overlap a neighbour (local lookups)
  long long s8_wide_rows = 1LL << 17;  // isolated launches over windows this large take the wide grid
                                       // (MC_S8_WIDE_ROWS)

  // pipelined shard merges (mc_merge_records_submit / _wait): per slot, k_finalize writes the
  // decisions straight into a mapped host block and an event marks them complete
  OutRec* h_merge[MC_MERGE_SLOTS] = {};
  OutRec* d_merge[MC_MERGE_SLOTS] = {};
  cudaEvent_t merge_ev[MC_MERGE_SLOTS] = {};
  int merge_B[MC_MERGE_SLOTS] = {};  // batch of the merge in the slot, 0 = none
  int merge_cap = 0;

  TcPlan* tc = nullptr;           // fp16 tensor-core scan plan (MC_PATH_GEMM*), created on first use
  S8Plan* s8 = nullptr;           // TMA-streamed int8 scan plan (tensor maps of ring8 / ringq)
  unsigned* d_counter = nullptr;  // last-CTA ticket of the fused GEMV scan (zero between launches)

  Thresholds thr{};
  std::vector<double> sched;  // sigma schedule over timesteps 0..T (empty: none)
  int path = MC_PATH_AUTO;
  long long stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Spare physical slots beyond the capacity.  A pipelined lookup's window must stay readable
// (its exhaustive fallback may run after the next lookup has written appended rows): the
// next rows land in these slots instead of over the rows it scanned.
RingState mirror(const mc_cache* h) { return RingState{h->head, h->count, h->jhead, h->Cp}; }

// The answer for an empty cache (cache.py:252-253): a miss with no similarity; every step runs.
OutRec empty_out(const mc_cache* h) {
  OutRec o;
  o.live = -1;
  o.sim = NAN;
  o.k = 0;
  o.flags = MC_FLAG_EMPTY;
  o.steps = h->thr.total_steps;
  o.route = 0;
  o.sigma = NAN;
  return o;
}

int finish_inflight(mc_cache* h);

RingBufs rbufs(const mc_cache* h) { return RingBufs{h->ring16, h->ring64, h->ring8, h->ringq, h->P8}; }

int wait_env(mc_cache* h) {
  if (h->env_inflight) {
    CU(cudaEventSynchronize(h->env_ev));
    h->env_inflight = false;
  }
  return MC_OK;
}

// Bytes of the quantisation block for B queries: QPrep[B] (64-byte padded), q̂[B][Dp].
size_t prep_head(int B) { return ((size_t)B * sizeof(QPrep) + 63) / 64 * 64; }
size_t prep_bytes(const mc_cache* h, int B) { return prep_head(B) + (size_t)B * h->Dp; }

// int8 quantisation of one query for the small-batch scan (scan_stream8.cu):
// s >= max|q|/127 rounded up (so |q/s| <= 127), q̂ = rint(q / s), and the
// norms the certificate and the exhaustive-path decision need.
void quantize_query(const double* q, int D, int Dp, QPrep* p, int8_t* q8) {
  // four independent chains, plain multiply-add (no libm fma call on a generic x86-64
  // target); the order only moves n2 / n1 by ulps, inside their (1 + 1e-12) slack
  double mx[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
  int j = 0;
  for (; j + 4 <= D; j += 4)
    for (int k = 0; k < 4; ++k) {
      const double x = q[j + k], ax = std::fabs(x);
      mx[k] = std::max(mx[k], ax);
      s2[k] += x * x;
      s1[k] += ax;
    }
  for (; j < D; ++j) {
    const double x = q[j], ax = std::fabs(x);
    mx[0] = std::max(mx[0], ax);
    s2[0] += x * x;
    s1[0] += ax;
  }
  const double amax = std::max(std::max(mx[0], mx[1]), std::max(mx[2], mx[3]));
  const double a2 = (s2[0] + s2[1]) + (s2[2] + s2[3]);
  const double a1 = (s1[0] + s1[1]) + (s1[2] + s1[3]);
  const bool finite = std::isfinite(a1) && std::isfinite(amax) && amax <= 1e300;
  float s = 0.0f;
  if (finite && amax > 0.0) {
    s = (float)(amax / 127.0);
    if ((double)s < amax / 127.0) s = std::nextafter(s, INFINITY);
  }
  // q̂ = rint(q / s) via one reciprocal: a rounding flip from the multiply moves
  // |q_i - s q̂_i| past s/2 by ~2^-52 s at most, far inside the bound's slack
  // (the 1 + 1e-9 factor and the 1e-12 term of the per-row delta)
  double l1 = 0.0;
  const double inv = s > 0.0f ? 1.0 / (double)s : 0.0;
  int i = 0;
  for (; i < D; ++i) {
    const int qi = (int)__builtin_rint(q[i] * inv);
    q8[i] = (int8_t)qi;
    l1 += (double)(qi < 0 ? -qi : qi);
  }
  for (; i < Dp; ++i) q8[i] = 0;
  p->q1 = l1 * (double)s;
  p->n2 = std::sqrt(a2) * (1.0 + 1e-12);
  p->n1 = a1 * (1.0 + 1e-12);
  p->s = s;
  p->exotic = !(p->n1 <= 1e30) || !(p->n2 >= 1e-30);
}

int s8_grid_max(const mc_cache* h) { return std::max(s8_grid(h->sm_count), s8_grid_wide(h->sm_count)); }

// Grid of a streamed-scan launch: the overlap-friendly grid, or every co-resident CTA slot for an
// isolated lookup (h->s8_isolated) over a window of at least s8_wide_rows rows.
int s8_launch_grid(const mc_cache* h) {
  if (h->s8_isolated && h->count >= h->s8_wide_rows) return std::min(320, s8_grid_wide(h->sm_count));
  const int g = s8_grid(h->sm_count);
  if (h->s8_rows_per_cta > 0)  // small windows: fewer CTAs, so fewer records to merge
    return (int)std::max(1LL, std::min((long long)g, (h->count + h->s8_rows_per_cta - 1) / h->s8_rows_per_cta));
  return g;
}

// Per-CTA records: the GEMV scans' CtaRec per CTA, or the streamed scan's two 16-byte words per
// CTA in two epoch-parity buffers; sized for the larger.
size_t cta_bytes(const mc_cache* h, int cap) {
  return std::max((size_t)gemv_grid(h->sm_count) * sizeof(CtaRec), (size_t)s8_grid_max(h) * 2 * 2 * 16) *
         (size_t)cap;
}

void free_batch(mc_cache* h) {
  cudaFree(h->d_part_s);
  cudaFree(h->d_part_p);
  cudaFree(h->d_part_floor);
  cudaFree(h->d_cta);
  cudaFree(h->d_gmax);
  cudaFree(h->d_gmax8);
  cudaFree(h->d_rec);
  cudaFree(h->d_scratch);
  cudaFree(h->d_out);
  cudaFreeHost(h->h_out);
  cudaFreeHost(h->h_outp);
  cudaFree(h->d_rec2);
  cudaFree(h->d_out2);
  cudaFreeHost(h->h_out2);
  h->d_rec2 = nullptr;
  h->d_out2 = nullptr;
  h->h_out2 = nullptr;
  h->d_part_s = nullptr;
  h->d_part_p = nullptr;
  h->d_part_floor = nullptr;
  h->d_cta = nullptr;
  h->d_gmax = nullptr;
  h->d_gmax8 = nullptr;
  h->d_rec = nullptr;
  h->d_scratch = nullptr;
  h->d_out = nullptr;
  h->h_out = nullptr;
  h->d_outm = nullptr;
  h->h_outp = nullptr;
  h->d_outp = nullptr;
}

// Grow the query capacity to >= B (power of two): per-batch buffers and the
// envelope, whose pending rows are carried over.
int ensure_batch(mc_cache* h, int B) {
  if (B <= h->Bcap) return MC_OK;
  CU(cudaStreamSynchronize(h->stream));
  h->env_inflight = false;
  free_batch(h);
  int cap = 4;
  while (cap < B) cap <<= 1;
  const int chunks = std::max(gemv_grid(h->sm_count), exact_grid(h->sm_count));
  const size_t row = (size_t)h->Dp * sizeof(double);
  const size_t env_bytes = ((size_t)h->stage_cap + cap) * row + prep_bytes(h, cap);
  double* h_env = nullptr;
  double* d_env = nullptr;
  CU(cudaMallocHost(&h_env, env_bytes));
  memset(h_env, 0, env_bytes);
  if (h->h_env) {
    memcpy(h_env, h->h_env, (size_t)h->n_pending * row);
    cudaFreeHost(h->h_env);
    cudaFree(h->d_env);
  }
  h->h_env = h_env;
  CU(cudaMalloc(&d_env, env_bytes));
  CU(cudaMemsetAsync(d_env, 0, env_bytes, h->stream));
  h->d_env = d_env;
  CU(cudaMalloc(&h->d_part_s, (size_t)cap * chunks * KP * sizeof(float)));
  CU(cudaMalloc(&h->d_part_p, (size_t)cap * chunks * KP * sizeof(long long)));
  CU(cudaMalloc(&h->d_part_floor, (size_t)cap * chunks * sizeof(float)));
  CU(cudaMalloc(&h->d_cta, cta_bytes(h, cap)));
  // the streamed scan's records are epoch-tagged: zero words belong to no launch
  CU(cudaMemsetAsync(h->d_cta, 0, cta_bytes(h, cap), h->stream));
  // 256 words per query: the streamed scan keeps 8 replicas of its bound 128 B apart
  CU(cudaMalloc(&h->d_gmax, (size_t)cap * 256 * sizeof(unsigned)));
  CU(cudaMemsetAsync(h->d_gmax, 0, (size_t)cap * 256 * sizeof(unsigned), h->stream));
  CU(cudaMalloc(&h->d_gmax8, (size_t)cap * 128 * sizeof(unsigned long long)));
  CU(cudaMemsetAsync(h->d_gmax8, 0, (size_t)cap * 128 * sizeof(unsigned long long), h->stream));
  CU(cudaMalloc(&h->d_rec, (size_t)cap * sizeof(mc_record)));
  CU(cudaMalloc(&h->d_scratch, (size_t)cap * exact_grid(h->sm_count) * sizeof(mc_record)));
  CU(cudaMalloc(&h->d_out, (size_t)cap * sizeof(OutRec)));
  CU(cudaMalloc(&h->d_rec2, (size_t)cap * sizeof(mc_record)));
  CU(cudaMalloc(&h->d_out2, (size_t)cap * sizeof(OutRec)));
  CU(cudaMallocHost(&h->h_out2, (size_t)cap * sizeof(OutRec)));
  CU(cudaHostAlloc(&h->h_out, (size_t)cap * sizeof(OutRec), cudaHostAllocMapped));
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_outm), h->h_out, 0));
  CU(cudaHostAlloc(&h->h_outp, (size_t)cap * 2 * sizeof(uint4), cudaHostAllocMapped));
  memset(h->h_outp, 0, (size_t)cap * 2 * sizeof(uint4));
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_outp), h->h_outp, 0));
  h->Bcap = cap;
  return MC_OK;
}

// Pending appends as a fused-append descriptor over device rows `dev_rows`
// (the uploaded envelope prefix).  Clears the host pending state.
GemvAppendArgs take_pending(mc_cache* h, const double* dev_rows) {
  GemvAppendArgs a;
  a.rb = rbufs(h);
  a.d_state = h->d_state;
  a.dirty = h->state_dirty || h->n_pending > 0;
  if (h->n_pending > 0) {
    const long long nw = std::min(h->n_pending, h->C);  // older rows were displaced before landing
    const long long skip = h->n_pending - nw;
    a.stage = dev_rows + (size_t)skip * h->Dp;
    a.n = nw;
    a.first_slot = (h->pending_first_slot + skip) % h->Cp;
  }
  h->n_pending = 0;
  h->state_dirty = false;
  return a;
}

// Host buffers the caller registered (mc_register_host): batches of queries that lie inside
// one are copied to the device straight from it (DMA), without staging into the envelope.
struct HostRange {
  uintptr_t lo, hi;
};
std::mutex g_reg_mu;
std::vector<HostRange> g_reg;

bool host_registered(const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (const HostRange& r : g_reg)
    if (a >= r.lo && a + bytes <= r.hi) return true;
  return false;
}

// Upload the envelope prefix: pending rows, B queries (row-major, stride D),
// then their int8 quantisation.  Returns device pointers to the queries and
// to the quantisation block.
int upload_envelope(mc_cache* h, const double* queries, int B, bool async_reuse, bool quantise,
                    const double** q_dev, const QPrep** prep_dev, const int8_t** q8_dev) {
  int rc = wait_env(h);
  if (rc) return rc;
  const size_t row = (size_t)h->Dp * sizeof(double);
  double* qdst = h->h_env + (size_t)h->n_pending * h->Dp;
  auto stage_rows = [&](int b0, int b1) {
    if (h->D == h->Dp) {
      memcpy(qdst + (size_t)b0 * h->Dp, queries + (size_t)b0 * h->D, (size_t)(b1 - b0) * row);
    } else {
      for (int b = b0; b < b1; ++b) {  // padding columns may hold an earlier lookup's quantisation bytes
        memcpy(qdst + (size_t)b * h->Dp, queries + (size_t)b * h->D, h->D * sizeof(double));
        memset(qdst + (size_t)b * h->Dp + h->D, 0, (size_t)(h->Dp - h->D) * sizeof(double));
      }
    }
  };
  // Large batches: stage and copy in chunks so each chunk's DMA overlaps the next chunk's
  // host copy (the unquantised large-batch paths only; the int8 paths take B <= 4).
  constexpr size_t CHUNK_BYTES = 256 << 10;
  const int chunk = std::max<int>(1, (int)(CHUNK_BYTES / row));
  const bool prefetched = !quantise && h->pf_src == queries && h->pf_B == B;
  h->pf_src = nullptr;  // a prefetch serves only the upload right after it
  if (prefetched) {  // the batch was DMA'd into a query slot on the copy stream
    const size_t head = (size_t)h->n_pending * row;
    if (head) CU(cudaMemcpyAsync(h->d_env, h->h_env, head, cudaMemcpyHostToDevice, h->stream));
    if (async_reuse && head) {
      CU(cudaEventRecord(h->env_ev, h->stream));
      h->env_inflight = true;
    }
    CU(cudaStreamWaitEvent(h->stream, h->q_ev[h->pf_slot], 0));
    *q_dev = h->d_qslot[h->pf_slot];
    *prep_dev = nullptr;
    *q8_dev = nullptr;
    return MC_OK;
  }
  if (!quantise && B > 2 * chunk && h->D == h->Dp && host_registered(queries, (size_t)B * row)) {
    // registered caller memory: one DMA of the batch, no host staging copy
    const double t1 = g_ht.on ? now_us() : 0.0;
    const size_t head = (size_t)h->n_pending * row;
    if (head) CU(cudaMemcpyAsync(h->d_env, h->h_env, head, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(h->d_env + (size_t)h->n_pending * h->Dp, queries, (size_t)B * row, cudaMemcpyHostToDevice,
                       h->stream));
    if (g_ht.on) g_ht.acc[1] += now_us() - t1;
    if (async_reuse) {
      CU(cudaEventRecord(h->env_ev, h->stream));
      h->env_inflight = true;
    }
    *q_dev = h->d_env + (size_t)h->n_pending * h->Dp;
    *prep_dev = nullptr;
    *q8_dev = nullptr;
    return MC_OK;
  }
  if (!quantise && B > 2 * chunk) {
    const double t1 = g_ht.on ? now_us() : 0.0;
    const size_t head = (size_t)h->n_pending * row;
    if (head) CU(cudaMemcpyAsync(h->d_env, h->h_env, head, cudaMemcpyHostToDevice, h->stream));
    for (int b0 = 0; b0 < B; b0 += chunk) {
      const int b1 = std::min(B, b0 + chunk);
      stage_rows(b0, b1);
      CU(cudaMemcpyAsync(h->d_env + (size_t)(h->n_pending + b0) * h->Dp, qdst + (size_t)b0 * h->Dp,
                         (size_t)(b1 - b0) * row, cudaMemcpyHostToDevice, h->stream));
    }
    if (g_ht.on) g_ht.acc[1] += now_us() - t1;
    if (async_reuse) {
      CU(cudaEventRecord(h->env_ev, h->stream));
      h->env_inflight = true;
    }
    *q_dev = h->d_env + (size_t)h->n_pending * h->Dp;
    *prep_dev = nullptr;
    *q8_dev = nullptr;
    return MC_OK;
  }
  stage_rows(0, B);
  const size_t prep_off = (size_t)(h->n_pending + B) * row;
  uint8_t* hp = reinterpret_cast<uint8_t*>(h->h_env) + prep_off;
  QPrep* hq = reinterpret_cast<QPrep*>(hp);
  int8_t* h8 = reinterpret_cast<int8_t*>(hp + prep_head(B));
  if (quantise)
    for (int b = 0; b < B; ++b) quantize_query(qdst + (size_t)b * h->Dp, h->D, h->Dp, hq + b, h8 + (size_t)b * h->Dp);
  const double t1 = g_ht.on ? now_us() : 0.0;
  CU(cudaMemcpyAsync(h->d_env, h->h_env, prep_off + (quantise ? prep_bytes(h, B) : 0), cudaMemcpyHostToDevice,
                     h->stream));
  if (g_ht.on) g_ht.acc[1] += now_us() - t1;
  if (async_reuse) {  // the caller returns before the copy completes
    CU(cudaEventRecord(h->env_ev, h->stream));
    h->env_inflight = true;
  }
  uint8_t* dp = reinterpret_cast<uint8_t*>(h->d_env) + prep_off;
  *q_dev = h->d_env + (size_t)h->n_pending * h->Dp;
  *prep_dev = quantise ? reinterpret_cast<const QPrep*>(dp) : nullptr;
  *q8_dev = quantise ? reinterpret_cast<const int8_t*>(dp + prep_head(B)) : nullptr;
  return MC_OK;
}

// Publish pending appends / evictions with k_append (stream-ordered).  Used
// when the pending batch is too large to ride along with a lookup.
int flush(mc_cache* h) {
  if (h->n_pending == 0 && !h->state_dirty) return MC_OK;
  int rc = finish_inflight(h);  // an asynchronous lookup must finish on the ring state it scanned
  if (rc) return rc;
  rc = wait_env(h);
  if (rc) return rc;
  if (h->n_pending > 0)
    CU(cudaMemcpyAsync(h->d_env, h->h_env, (size_t)h->n_pending * h->Dp * sizeof(double), cudaMemcpyHostToDevice,
                       h->stream));
  const GemvAppendArgs a = take_pending(h, h->d_env);
  CU(launch_append(a.stage, a.n, a.first_slot, mirror(h), h->D, h->Dp, rbufs(h), h->d_state, h->stream));
  CU(cudaEventRecord(h->env_ev, h->stream));
  h->env_inflight = true;
  h->stats[7]++;
  return MC_OK;
}

// Batch size from which the tensor-core scan replaces the GEMV scan: the GEMV
// kernel reads the ring once per 4 queries, the tcgen05 scan once per batch.
constexpr int GEMM_MIN_B = 5;
// Largest pending-append batch folded into a GEMV launch; larger ones use k_append.
constexpr long long FUSE_APPEND_MAX = 256;

bool use_gemm(const mc_cache* h, int B) {
  if (h->path == MC_PATH_GEMV || h->path == MC_PATH_STREAM8) return false;
  return h->path == MC_PATH_GEMM || (h->path == MC_PATH_AUTO && B >= GEMM_MIN_B);
}

int ensure_tc(mc_cache* h, int B) {
  if (h->tc && tc_bcap(h->tc) >= B) return MC_OK;
  CU(cudaStreamSynchronize(h->stream));
  tc_plan_destroy(h->tc);
  h->tc = nullptr;
  char err[256] = {0};
  h->tc = tc_plan_create(h->ring16, h->Cp, h->Dp, std::max(B, 128), h->sm_count, err, sizeof err);
  if (!h->tc) return fail(MC_ERR_CUDA, "tensor-core scan plan: %s", err);
  return MC_OK;
}

// Scan + certified merge for B queries at q64 (device, stride Dp): records
// into rec[0..B) and, when out != nullptr, decisions into out[0..B).  `app`
// describes appends already on the device that precede the scan (folded into
// the first GEMV launch, or applied by k_append before a tensor-core scan).
// t_mid (optional) is recorded between the scan and the standalone merge.
// Epoch of the next streamed-scan launch (never 0: zeroed words belong to no launch).  On
// wrap-around the bound words are cleared, so an old epoch can never outrank a new one.
// Distance (uint4) between the two epoch-parity record buffers of the streamed scan in d_cta.
unsigned s8_rec_par(const mc_cache* h) { return (unsigned)((size_t)h->Bcap * s8_grid_max(h) * 2); }

// A streamed-scan launch that failed took an epoch without publishing it: publish it from the
// host so the next launch (which waits for the previous epoch's rows) does not wait forever.
int s8_launch_failed(mc_cache* h, unsigned ep, cudaError_t e) {
  const unsigned z[2] = {ep, ep};
  cudaMemcpyAsync(h->d_sync, z, sizeof z, cudaMemcpyHostToDevice, h->stream);
  cudaStreamSynchronize(h->stream);
  return fail(MC_ERR_CUDA, "streamed scan launch: %s", cudaGetErrorString(e));
}

unsigned s8_epoch(mc_cache* h) {
  if (++h->s8_epoch == 0) {
    cudaMemsetAsync(h->d_gmax8, 0, (size_t)h->Bcap * 128 * sizeof(unsigned long long), h->stream);
    cudaMemsetAsync(h->d_cta, 0, cta_bytes(h, h->Bcap), h->stream);
    cudaMemsetAsync(h->d_sync, 0, 2 * sizeof(unsigned), h->stream);
    h->s8_epoch = 1;
  }
  return h->s8_epoch;
}

int scan_merge(mc_cache* h, const double* q64, int B, mc_record* rec, OutRec* out, const GemvAppendArgs& app,
               const QPrep* prep, const int8_t* q8, cudaEvent_t t_mid = nullptr, unsigned* done_seq = nullptr,
               unsigned seq = 0, uint4* outp = nullptr) {
  if (use_gemm(h, B)) {
    if (app.n > 0 || app.dirty) {  // evictions alone must reach d_state too (the scan reads it)
      CU(launch_append(app.stage, app.n, app.first_slot, mirror(h), h->D, h->Dp, rbufs(h), h->d_state, h->stream));
      h->stats[7]++;
    }
    int rc = ensure_tc(h, B);
    if (rc) return rc;
    const Partials part{h->d_part_s, h->d_part_p, h->d_part_floor, tc_chunks(h->tc, B)};
    CU(launch_tc_scan(h->tc, q64, B, h->D, h->d_state, part, h->shard, h->stream));
    if (t_mid) CU(cudaEventRecord(t_mid, h->stream));
    CU(launch_merge(h->d_state, h->ring64, h->D, h->Dp, q64, B, part, tc_qscale(h->tc), gemm_eps_rel(h->Dp),
                    eps_abs1(), rec, h->shard, &h->thr, out, h->stream));  // the decision is fused (G = 1)
    h->tc_tail = true;  // k_merge lets its dependent start early: the next streamed scan must not overlap it
    h->stats[6]++;
    h->stats[7] += 3;
    return MC_OK;
  }
  GemvAppendArgs a = app;
  const RingState st = mirror(h);
  const bool quant = h->path != MC_PATH_GEMV && prep != nullptr;
  const bool s8 = quant && h->s8;
  for (int b0 = 0; b0 < B; b0 += 4) {
    const int nb = std::min(4, B - b0);
    if (s8) {
      const unsigned ep = s8_epoch(h);
      const cudaError_t e = launch_stream8_scan(h->s8, rbufs(h), st, q64 + (size_t)b0 * h->Dp, nb, h->d_cta, b0,
                                                s8_launch_grid(h), h->shard, h->d_counter, h->d_gmax8, ep, h->thr,
                                                rec, out,
                                                a, prep + b0, q8 + (size_t)b0 * h->Dp,
                                                b0 + nb == B ? done_seq : nullptr, seq, outp, h->d_sync,
                                                s8_rec_par(h), !h->tc_tail, h->stream);
      if (e != cudaSuccess) return s8_launch_failed(h, ep, e);
      h->tc_tail = false;
    } else
      CU(launch_gemv_scan(h->ring16, st, h->D, h->Dp, q64 + (size_t)b0 * h->Dp, nb, h->d_cta, b0,
                          gemv_grid(h->sm_count), h->shard, h->d_counter, h->d_gmax, h->ring64, h->thr, rec, out, a,
                          h->stream));
    a.n = 0;  // written by the first launch
    h->stats[5]++;
    h->stats[7]++;
  }
  if (t_mid) CU(cudaEventRecord(t_mid, h->stream));
  return MC_OK;
}

// Stage + upload + scan for B host queries; on return the records (and
// decisions) are enqueued, not complete.  Returns the device query pointer.
// The caller has run ensure_batch(h, B) (rec / out may be handle buffers).
int lookup_enqueue(mc_cache* h, const double* queries, int B, mc_record* rec, OutRec* out, bool async_reuse,
                   const double** q_dev, unsigned* done_seq = nullptr, unsigned seq = 0, uint4* outp = nullptr) {
  int rc;
  if (h->n_pending > FUSE_APPEND_MAX) {
    rc = flush(h);
    if (rc) return rc;
  }
  const double* q = nullptr;
  const QPrep* prep = nullptr;
  const int8_t* q8 = nullptr;
  const bool int8 = !use_gemm(h, B) && h->path != MC_PATH_GEMV && h->s8;
  rc = upload_envelope(h, queries, B, async_reuse, int8, &q, &prep, &q8);
  if (rc) return rc;
  const GemvAppendArgs app = take_pending(h, h->d_env);
  *q_dev = q;
  return scan_merge(h, q, B, rec, out, app, prep, q8, nullptr, done_seq, seq, outp);
}

int wait_seq(mc_cache* h, unsigned seq);
int wait_packed(mc_cache* h, unsigned seq, int B, int slot = 0, OutRec* dst = nullptr);
unsigned seq_tag(unsigned seq);
bool direct_result(const mc_cache* h, int B);

// Enqueue a zero-copy lookup: packed self-validating decisions (default), or
// the decisions + a system fence + the completion word.
void quantize_query(const double* q, int D, int Dp, QPrep* p, int8_t* q8);
GemvAppendArgs take_pending(mc_cache* h, const double* dev_rows);

int enqueue_direct(mc_cache* h, const double* queries, int B, unsigned seq, bool async_reuse, const double** q,
                   int slot = 0, bool param = false) {
  if (h->packed && (h->param_in || param) && B == 1 && h->n_pending <= 1 && h->Dp <= 1024) {
    // no host->device copy precedes the kernel: the quantisation rides in the parameter block,
    // the query and the pending row are read from mapped host memory (scan_stream8.cu, S8In).
    // One lookup is in flight per handle, so these buffers are free again once it completes.
    // Per result slot, so a pipelined lookup never overwrites what the one before it reads.
    const double* stage_row = nullptr;
    if (h->n_pending == 1) {
      memcpy(h->h_stage1[slot], h->h_env, (size_t)h->Dp * sizeof(double));  // staged rows are zero-padded to Dp
      stage_row = h->h_stage1[slot];
    }
    double* hq = h->h_qslot[slot];
    memcpy(hq, queries, (size_t)h->D * sizeof(double));  // padding columns stay zero
    memcpy(h->h_qkeep, queries, (size_t)h->D * sizeof(double));
    const RingState st = mirror(h);
    take_pending(h, nullptr);
    memset(h->h_outp + 2 * slot, 0, 2 * sizeof(uint4));
    *q = nullptr;
    const unsigned ep = s8_epoch(h);
    const cudaError_t e = launch_stream8_direct(h->s8, rbufs(h), st, h->D, hq, stage_row, h->d_cta, s8_launch_grid(h),
                                                h->shard, h->d_counter, h->d_gmax8, ep, h->thr, h->d_rec + slot,
                                                nullptr, h->d_state, nullptr, seq_tag(seq), h->d_outp + 2 * slot,
                                                quantize_query, h->d_gq64, h->d_sync, s8_rec_par(h), !h->tc_tail,
                                                h->stream);
    if (e != cudaSuccess) return s8_launch_failed(h, ep, e);
    h->tc_tail = false;
    h->stats[5]++;
    h->stats[7]++;
    return MC_OK;
  }
  if (h->packed) {
    memset(h->h_outp + 2 * slot, 0, (size_t)B * 2 * sizeof(uint4));  // no stale record can carry this tag
    if (B == 1) memcpy(h->h_qslot[slot], queries, (size_t)h->D * sizeof(double));  // for a late fallback
    return lookup_enqueue(h, queries, B, h->d_rec + slot, nullptr, async_reuse, q, nullptr, seq_tag(seq),
                          h->d_outp + 2 * slot);
  }
  return lookup_enqueue(h, queries, B, h->d_rec, h->d_outm, async_reuse, q, h->d_seq, seq);
}

int wait_direct(mc_cache* h, unsigned seq, int B, int slot = 0) {
  return h->packed ? wait_packed(h, seq, B, slot) : wait_seq(h, seq);
}

// The device query of a completed lookup, for the exhaustive fallback: a
// parameter-block lookup has none, so its kept host copy is uploaded now.
int device_query(mc_cache* h, const double* q, const double** out) {
  if (q) {
    *out = q;
    return MC_OK;
  }
  CU(cudaMemcpyAsync(h->d_env, h->h_qkeep, (size_t)h->Dp * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  *out = h->d_env;
  return MC_OK;
}

// Exhaustive fallback of one single-query lookup from its kept query, on the window it
// scanned (explicit state: later launches may have moved the live window since).
int fallback_single(mc_cache* h, int slot, const RingState& st, OutRec* dst) {
  CU(cudaMemcpyAsync(h->d_qfb, h->h_qslot[slot], (size_t)h->Dp * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CU(cudaMemcpyAsync(h->d_state_fb, &st, sizeof st, cudaMemcpyHostToDevice, h->stream));
  CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state_fb, h->D, h->Dp, h->d_qfb, 1, h->d_rec + slot, h->d_scratch,
                         exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
  CU(launch_finalize(h->d_rec + slot, 1, 1, -1, h->d_state_fb, h->thr, h->d_out, h->stream));
  h->stats[7] += 3;
  CU(cudaMemcpyAsync(dst, h->d_out, sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return MC_OK;
}

// A batch slot's records, device decisions and host decisions.
mc_record* brec(const mc_cache* h, int s) { return s ? h->d_rec2 : h->d_rec; }
OutRec* bdout(const mc_cache* h, int s) { return s ? h->d_out2 : h->d_out; }
OutRec* bhout(const mc_cache* h, int s) { return s ? h->h_out2 : h->h_out; }

// Wait for an asynchronous batch in slot s and apply the exhaustive fallback to the queries that
// need it, on window st (the one the batch scanned; later batches may have applied up to
// PIPE_SLACK rows since, which land in spare slots) with device queries q.
int finish_batch(mc_cache* h, int s, int B, const RingState& st, const double* q) {
  CU(cudaEventSynchronize(h->batch_ev[s]));
  OutRec* ho = bhout(h, s);
  bool need = false;
  for (int b = 0; b < B; ++b) need |= (ho[b].flags & FLAG_NEED_ANY) != 0;
  if (!need) return MC_OK;
  CU(cudaMemcpyAsync(h->d_state_fb, &st, sizeof st, cudaMemcpyHostToDevice, h->stream));
  CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state_fb, h->D, h->Dp, q, B, brec(h, s), h->d_scratch,
                         exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
  CU(launch_finalize(brec(h, s), 1, B, -1, h->d_state_fb, h->thr, bdout(h, s), h->stream));
  h->stats[7] += 3;
  CU(cudaMemcpyAsync(ho, bdout(h, s), (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return MC_OK;
}

// Complete the oldest of three pipelined single-query lookups, if any (answer kept in old2_out).
int finish_old2(mc_cache* h) {
  if (!h->old2_seq || h->old2_ready) return MC_OK;
  int rc = wait_packed(h, h->old2_seq, 1, h->old2_slot, &h->old2_out);
  if (rc) return rc;
  if (h->old2_out.flags & FLAG_NEED_ANY) {
    rc = fallback_single(h, h->old2_slot, h->old2_st, &h->old2_out);
    if (rc) return rc;
  }
  h->old2_ready = true;
  return MC_OK;
}

// Complete the older pipelined lookup, if any (its answer stays in old_out for mc_retrieve_wait).
int finish_old(mc_cache* h) {
  int rc2 = finish_old2(h);  // the oldest first
  if (rc2) return rc2;
  if (!h->old_seq || h->old_ready) return MC_OK;
  if (h->old_async) {  // a batch: answered into old_batch
    int rc = finish_batch(h, h->old_bslot, h->old_B, h->old_st, h->old_q);
    if (rc) return rc;
    h->old_batch.assign(bhout(h, h->old_bslot), bhout(h, h->old_bslot) + h->old_B);
    h->old_async = false;
    h->old_ready = true;
    return MC_OK;
  }
  int rc = wait_packed(h, h->old_seq, 1, h->old_slot, &h->old_out);
  if (rc) return rc;
  if (h->old_out.flags & FLAG_NEED_ANY) {
    rc = fallback_single(h, h->old_slot, h->old_st, &h->old_out);
    if (rc) return rc;
  }
  h->old_ready = true;
  return MC_OK;
}

// Complete the asynchronous lookups in flight, if any: wait for their decisions
// and run the exhaustive fallback for the queries whose certificate needs it
// (while the ring still holds the state that lookup scanned).
int finish_inflight(mc_cache* h) {
  int rc0 = finish_old(h);
  if (rc0) return rc0;
  if (!h->inflight_seq || h->inflight_ready) return MC_OK;
  const int B = h->inflight_B;
  int rc = MC_OK;
  if (h->inflight_direct)
    rc = wait_direct(h, h->inflight_seq, B, h->inflight_slot);
  else if (h->inflight_async) {
    rc = finish_batch(h, h->batch_slot, B, h->inflight_st, h->inflight_q);
    if (rc) return rc;
    h->inflight_async = false;
    h->inflight_ready = true;
    return MC_OK;
  } else
    rc = wait_seq(h, h->inflight_seq);
  if (rc) return rc;
  bool need = false;
  for (int b = 0; b < B; ++b) need |= (h->h_out[b].flags & FLAG_NEED_ANY) != 0;
  if (need && h->inflight_direct && B == 1 && h->packed) {
    rc = fallback_single(h, h->inflight_slot, h->inflight_st, h->h_out);
    if (rc) return rc;
  } else if (need) {
    const double* qd = nullptr;
    rc = device_query(h, h->inflight_q, &qd);
    if (rc) return rc;
    CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state, h->D, h->Dp, qd, B, h->d_rec, h->d_scratch,
                           exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
    CU(launch_finalize(h->d_rec, 1, B, -1, h->d_state, h->thr, h->d_out, h->stream));
    h->stats[7] += 3;
    CU(cudaMemcpyAsync(h->h_out, h->d_out, (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
  h->inflight_ready = true;
  return MC_OK;
}

// True when a B-query lookup runs on the streamed int8 scan, which can hand
// its decisions straight to host-mapped memory.
bool direct_result(const mc_cache* h, int B) {
  return h->s8 && !use_gemm(h, B) && h->path != MC_PATH_GEMV;
}

// Packed zero-copy results: tag of lookup `seq` (never 0, so zeroed slots never match).
unsigned seq_tag(unsigned seq) { return seq % 65535u + 1u; }

// Spin until the B packed decisions of lookup `seq` carry its tag, then unpack
// them into h_out.  Each record is one 16-byte store on the device side and one
// 16-byte load here, so a record is seen whole or not at all.
// One packed 16-byte record, once it carries `tag` (see pack_out in scan_stream8.cu).
int wait_record(mc_cache* h, const uint4* p, unsigned tag, unsigned seq, int b, uint4* out) {
  uint4 v;
  for (unsigned spins = 1;; ++spins) {
#if defined(__x86_64__)
    const __m128i x = _mm_load_si128(reinterpret_cast<const __m128i*>(p));
    memcpy(&v, &x, sizeof v);
#else
    v = *(volatile const uint4*)p;
#endif
    if ((v.w >> 16) == tag) break;
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
    if ((spins & 1023u) == 0) {
      const cudaError_t e = cudaStreamQuery(h->stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return fail(MC_ERR_CUDA, "lookup %u: %s", seq, cudaGetErrorString(e));
      if (e == cudaSuccess) {  // the stream is idle: one last look, then report
#if defined(__x86_64__)
        const __m128i y = _mm_load_si128(reinterpret_cast<const __m128i*>(p));
        memcpy(&v, &y, sizeof v);
#else
        v = *(volatile const uint4*)p;
#endif
        if ((v.w >> 16) == tag) break;
        return fail(MC_ERR_STATE, "lookup %u finished without publishing query %d", seq, b);
      }
    }
  }
  *out = v;
  return MC_OK;
}

// Spin until the B packed decisions of lookup `seq` carry its tag, then unpack
// them into h_out.  Each record is one 16-byte store on the device side and one
// 16-byte load here, so a record is seen whole or not at all.
int wait_packed(mc_cache* h, unsigned seq, int B, int slot, OutRec* dst) {
  const unsigned tag = seq_tag(seq);
  const uint4* src = h->h_outp + 2 * slot;
  for (int b = 0; b < B; ++b) {
    uint4 v, v2;
    int rc = wait_record(h, src + 2 * b, tag, seq, b, &v);
    if (!rc) rc = wait_record(h, src + 2 * b + 1, tag, seq, b, &v2);
    if (rc) return rc;
    OutRec& o = dst ? dst[b] : h->h_out[b];
    const unsigned long long sb = (unsigned long long)v.x | ((unsigned long long)v.y << 32);
    memcpy(&o.sim, &sb, sizeof sb);
    o.live = (long long)(int)v.z;
    o.k = (int)(v.w & 0xffu);
    const unsigned f8 = (v.w >> 8) & 0xffu;
    o.flags = (f8 & 0x7fu) | ((f8 & 0x80u) ? FLAG_NEED_FALLBACK : 0u);
    const unsigned long long gb = (unsigned long long)v2.x | ((unsigned long long)v2.y << 32);
    memcpy(&o.sigma, &gb, sizeof gb);
    o.steps = (int)v2.z;
    o.route = (int)(v2.w & 0xffu);
  }
  return MC_OK;
}

// Spin until the streamed scan has published lookup `seq` into host-mapped
// memory; a failed or silently finished stream is reported, never waited on.
int wait_seq(mc_cache* h, unsigned seq) {
  volatile unsigned* f = h->h_seq;
  for (unsigned spins = 1; *f != seq; ++spins) {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
    if ((spins & 1023u) == 0) {
      const cudaError_t e = cudaStreamQuery(h->stream);
      if (e == cudaSuccess && *f != seq) return fail(MC_ERR_STATE, "lookup %u finished without publishing its result", seq);
      if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(MC_ERR_CUDA, "lookup %u: %s", seq, cudaGetErrorString(e));
    }
  }
  __atomic_thread_fence(__ATOMIC_ACQUIRE);
  return MC_OK;
}

int copy_out(mc_cache* h, int B, int64_t* out_live, double* out_sim, int32_t* out_k, uint32_t* out_flags) {
  for (int b = 0; b < B; ++b) {
    const OutRec& o = h->h_out[b];
    if (out_live) out_live[b] = o.live;
    if (out_sim) out_sim[b] = o.sim;
    if (out_k) out_k[b] = o.k;
    const unsigned f = o.flags & 0xffffu;
    if (out_flags) out_flags[b] = f;
    if (f & MC_FLAG_FALLBACK) h->stats[1]++;
    if (f & MC_FLAG_NONFINITE) h->stats[2]++;
    if (f & MC_FLAG_TIE) h->stats[3]++;
  }
  h->stats[0] += B;
  return MC_OK;
}

// sigma[k] per threshold pair from the schedule (noise_reentry_level, cache.py:325-334).
void apply_sigma(mc_cache* h) {
  Thresholds& t = h->thr;
  t.has_sigma = h->sched.empty() ? 0 : 1;
  for (int j = 0; j < MAX_PAIRS; ++j)
    t.sigma[j] = (j < t.n && t.ks[j] >= 0 && t.ks[j] < (int)h->sched.size()) ? h->sched[t.ks[j]] : NAN;
}

// The lookup of mc_retrieve_batch / mc_retrieve_decisions: B answers into h->h_out
// (the caller holds the mutex and the device guard).
int retrieve_into_hout(mc_cache* h, const double* queries, int32_t B) {
  if (h->inflight_seq || h->old_seq || h->old2_seq)
    return fail(MC_ERR_STATE, "an asynchronous lookup is in flight: mc_retrieve_wait first");
  int rc = ensure_batch(h, B);  // may reallocate d_rec / d_out / h_out: evaluate them after
  if (rc) return rc;
  if (h->count == 0) {  // cache.py:252-253
    for (int b = 0; b < B; ++b) h->h_out[b] = empty_out(h);
    return MC_OK;
  }
  const double* q = nullptr;
  if (direct_result(h, B)) {  // decisions land in host-mapped memory; no D2H copy, no stream sync
    const unsigned seq = ++h->seq;
    const double t0 = g_ht.on ? now_us() : 0.0;
    const double h2d0 = g_ht.acc[1];
    rc = enqueue_direct(h, queries, B, seq, false, &q);
    if (rc) return rc;
    const double t2 = g_ht.on ? now_us() : 0.0;
    rc = wait_direct(h, seq, B);
    if (rc) return rc;
    if (g_ht.on) {  // enqueue time minus the H2D call = staging, quantisation and the launch
      const double t3 = now_us();
      g_ht.acc[2] += (t2 - t0) - (g_ht.acc[1] - h2d0);
      g_ht.acc[3] += t3 - t2;
      g_ht.n++;
    }
  } else {
    const double t0 = g_ht.on ? now_us() : 0.0;
    const double h2d0 = g_ht.acc[1];
    rc = lookup_enqueue(h, queries, B, h->d_rec, h->d_out, false, &q);
    if (rc) return rc;
    const double t2 = g_ht.on ? now_us() : 0.0;
    CU(cudaMemcpyAsync(h->h_out, h->d_out, (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (g_ht.on) {
      const double t3 = now_us();
      g_ht.acc[2] += (t2 - t0) - (g_ht.acc[1] - h2d0);
      g_ht.acc[3] += t3 - t2;
      g_ht.n++;
    }
  }
  h->env_inflight = false;
  bool need = false;
  for (int b = 0; b < B; ++b) need |= (h->h_out[b].flags & FLAG_NEED_ANY) != 0;
  if (need) {  // rare: certificate failed or exotic query -> exact rescan, then decide again
    rc = device_query(h, q, &q);
    if (rc) return rc;
    CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state, h->D, h->Dp, q, B, h->d_rec, h->d_scratch,
                           exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
    CU(launch_finalize(h->d_rec, 1, B, -1, h->d_state, h->thr, h->d_out, h->stream));
    h->stats[7] += 3;
    CU(cudaMemcpyAsync(h->h_out, h->d_out, (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
  return MC_OK;
}

int copy_decisions(mc_cache* h, int B, mc_decision* out) {
  int rc = copy_out(h, B, nullptr, nullptr, nullptr, nullptr);  // counters
  if (rc) return rc;
  for (int b = 0; b < B; ++b) {
    const OutRec& o = h->h_out[b];
    mc_decision& d = out[b];
    d.live = o.live;
    d.sim = o.sim;
    d.sigma = o.sigma;
    d.k = o.k;
    d.steps = o.steps;
    d.flags = o.flags & 0xffffu;
    d.route = o.route;
  }
  return MC_OK;
}

}  // namespace

extern "C" {

const char* mc_last_error(void) { return g_err.c_str(); }

const char* mc_version(void) { return "modmcache 0.2.0 (sm_100a)"; }

int mc_create(mc_cache** out, int64_t capacity, int32_t dim, int32_t device) {
  if (!out) return fail(MC_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (capacity < 1) return fail(MC_ERR_ARG, "capacity must be >= 1, got %lld", (long long)capacity);
  if (dim < 1 || dim > 4096) return fail(MC_ERR_UNSUPPORTED, "dim must lie in [1, 4096], got %d", dim);
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MC_ERR_ARG, "device %d out of range (%d devices)", device, ndev);
  DeviceGuard guard(device);
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(MC_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
                                    device, prop.major, prop.minor);
  mc_cache* h = new mc_cache();
  h->dev = device;
  h->sm_count = prop.multiProcessorCount;
  h->C = capacity;
  h->Cp = capacity + PIPE_SLACK;
  h->D = dim;
  h->Dp = (dim + 63) / 64 * 64;
  h->P8 = (h->Dp + 127) / 128 * 128;
  auto cleanup = [&](int rc) {
    mc_destroy(h);
    return rc;
  };
  int rc;
#define CUC(call)                                                                                     \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return cleanup(fail(MC_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_))); \
  } while (0)
  CUC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  CUC(cudaEventCreateWithFlags(&h->env_ev, cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&h->rec_ev, cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&h->batch_ev[0], cudaEventDisableTiming));
  CUC(cudaEventCreateWithFlags(&h->batch_ev[1], cudaEventDisableTiming));
  const size_t n16 = (size_t)h->Cp * h->Dp * sizeof(__half);
  const size_t n64 = (size_t)h->Cp * h->Dp * sizeof(double);
  const size_t n8 = (size_t)h->Cp * h->P8;
  CUC(cudaMalloc(&h->ring16, n16));
  CUC(cudaMalloc(&h->ring64, n64));
  CUC(cudaMalloc(&h->ring8, n8));
  CUC(cudaMalloc(&h->ringq, (size_t)(h->Cp + 2) * sizeof(float2)));  // +2: 16-byte aligned bulk copies
  CUC(cudaMemsetAsync(h->ring16, 0, n16, h->stream));
  CUC(cudaMemsetAsync(h->ring64, 0, n64, h->stream));
  CUC(cudaMemsetAsync(h->ring8, 0, n8, h->stream));
  CUC(cudaMemsetAsync(h->ringq, 0, (size_t)(h->Cp + 2) * sizeof(float2), h->stream));
  CUC(cudaMalloc(&h->d_state, sizeof(RingState)));
  {
    RingState z{0, 0, 0, h->Cp};
    CUC(cudaMemcpyAsync(h->d_state, &z, sizeof z, cudaMemcpyHostToDevice, h->stream));
  }
  if (stream8_supported(h->Dp) && h->Cp < (1ll << 30)) {  // 30-bit row offsets in its records
    char err[256] = {0};
    h->s8 = s8_plan_create(h->ring8, h->ringq, h->Cp, h->Dp, h->P8, err, sizeof err);
    if (!h->s8) return cleanup(fail(MC_ERR_CUDA, "int8 stream scan plan: %s", err));
  }
  if (const char* e = getenv("MC_PACKED_RESULT")) h->packed = atoi(e) != 0;
  // testing hook: start the streamed scan's bound epochs near the 32-bit wrap-around
  if (const char* e = getenv("MC_S8_EPOCH0")) h->s8_epoch = (unsigned)strtoul(e, nullptr, 0);
  CUC(cudaMalloc(&h->d_sync, 2 * sizeof(unsigned)));
  {  // both words start at the epoch before the first launch's
    const unsigned z[2] = {h->s8_epoch, h->s8_epoch};
    CUC(cudaMemcpyAsync(h->d_sync, z, sizeof z, cudaMemcpyHostToDevice, h->stream));
    CUC(cudaStreamSynchronize(h->stream));
  }
  if (const char* e = getenv("MC_PARAM_INPUT")) h->param_in = atoi(e) != 0;
  if (const char* e = getenv("MC_S8_WIDE_ROWS")) h->s8_wide_rows = atoll(e);
  if (const char* e = getenv("MC_LOCAL_PARAM")) h->local_param = atoi(e) != 0;
  if (const char* e = getenv("MC_S8_ROWS_PER_CTA")) h->s8_rows_per_cta = atoll(e);
  CUC(cudaHostAlloc(&h->h_qkeep, (size_t)h->Dp * sizeof(double), cudaHostAllocMapped));
  memset(h->h_qkeep, 0, (size_t)h->Dp * sizeof(double));
  for (int k = 0; k < 3; ++k) {  // mapped: the parameter-block launches read the query from here
    CUC(cudaHostAlloc(&h->h_qslot[k], (size_t)h->Dp * sizeof(double), cudaHostAllocMapped));
    memset(h->h_qslot[k], 0, (size_t)h->Dp * sizeof(double));
  }
  CUC(cudaMalloc(&h->d_qfb, (size_t)h->Dp * sizeof(double)));
  CUC(cudaMalloc(&h->d_state_fb, sizeof(RingState)));
  for (int k = 0; k < 3; ++k) {
    CUC(cudaHostAlloc(&h->h_stage1[k], (size_t)h->Dp * sizeof(double), cudaHostAllocMapped));
    memset(h->h_stage1[k], 0, (size_t)h->Dp * sizeof(double));
  }
  CUC(cudaMalloc(&h->d_gq64, (size_t)h->Dp * sizeof(double)));
  if (h->C > 0x7fffffffll) h->packed = false;  // live index must fit the packed int32
  CUC(cudaHostAlloc(&h->h_seq, 64, cudaHostAllocMapped));
  *h->h_seq = 0u;
  CUC(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_seq), h->h_seq, 0));
  CUC(cudaMalloc(&h->d_counter, sizeof(unsigned)));
  CUC(cudaMemsetAsync(h->d_counter, 0, sizeof(unsigned), h->stream));
  h->stage_cap = std::max<long long>(1, std::min<long long>(h->C, (16ll << 20) / ((long long)h->Dp * 8)));
  rc = ensure_batch(h, 4);
  if (rc) return cleanup(rc);
  static const int ks[6] = {5, 10, 15, 20, 25, 30};
  static const double taus[6] = {0.25, 0.26, 0.27, 0.28, 0.29, 0.30};  // cache.py:18
  h->thr.n = 6;
  h->thr.total_steps = 50;
  for (int i = 0; i < 6; ++i) {
    h->thr.ks[i] = ks[i];
    h->thr.taus[i] = taus[i];
  }
  CUC(cudaStreamSynchronize(h->stream));
#undef CUC
  *out = h;
  return MC_OK;
}

int mc_destroy(mc_cache* h) {
  if (!h) return MC_OK;
  if (g_ht.on && g_ht.n)
    fprintf(stderr, "[modmcache host timing] %lld lookups: H2D enqueue %.2f us, stage+quantise+launch %.2f us, "
                    "wait for result %.2f us (means)\n", g_ht.n, g_ht.acc[1] / g_ht.n, g_ht.acc[2] / g_ht.n,
            g_ht.acc[3] / g_ht.n);
  {
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard guard(h->dev);
    if (h->stream) cudaStreamSynchronize(h->stream);
    free_batch(h);
    tc_plan_destroy(h->tc);
    s8_plan_destroy(h->s8);
    cudaFreeHost(h->h_env);
    cudaFree(h->d_env);
    cudaFree(h->ring16);
    cudaFree(h->ring64);
    cudaFree(h->ring8);
    cudaFree(h->ringq);
    cudaFree(h->d_state);
    cudaFree(h->d_counter);
    cudaFreeHost(h->h_seq);
    cudaFreeHost(h->h_qkeep);
    for (int k = 0; k < 3; ++k) {
      cudaFreeHost(h->h_stage1[k]);
      cudaFreeHost(h->h_qslot[k]);
    }
    cudaFree(h->d_qfb);
    cudaFree(h->d_state_fb);
    cudaFree(h->d_gq64);
    cudaFree(h->d_sync);
    for (int i = 0; i < MC_MERGE_SLOTS; ++i) {
      cudaFreeHost(h->h_merge[i]);
      if (h->merge_ev[i]) cudaEventDestroy(h->merge_ev[i]);
    }
    if (h->env_ev) cudaEventDestroy(h->env_ev);
    if (h->rec_ev) cudaEventDestroy(h->rec_ev);
    for (cudaEvent_t e : h->batch_ev)
      if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
      cudaFree(h->d_qslot[i]);
      if (h->q_ev[i]) cudaEventDestroy(h->q_ev[i]);
    }
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->stream) cudaStreamDestroy(h->stream);
  }
  delete h;
  return MC_OK;
}

int mc_set_thresholds(mc_cache* h, const int32_t* ks, const double* taus, int32_t n, int32_t total_steps) {
  if (!h || !ks || !taus) return fail(MC_ERR_ARG, "NULL argument");
  if (n < 1 || n > MAX_PAIRS) return fail(MC_ERR_ARG, "need 1..%d threshold pairs, got %d", MAX_PAIRS, n);
  for (int i = 1; i < n; ++i)
    if (!(ks[i] > ks[i - 1]) || !(taus[i] > taus[i - 1]))
      return fail(MC_ERR_ARG, "k and tau must be strictly increasing");
  std::lock_guard<std::mutex> lk(h->mu);
  if (ks[n - 1] > 255) h->packed = false;  // the packed decision carries k in 8 bits
  h->thr.n = n;
  h->thr.total_steps = total_steps;
  for (int i = 0; i < n; ++i) {
    h->thr.ks[i] = ks[i];
    h->thr.taus[i] = taus[i];
  }
  apply_sigma(h);
  return MC_OK;
}

int mc_configure_shard(mc_cache* h, int32_t n_shards, int32_t shard_id) {
  if (!h) return fail(MC_ERR_ARG, "NULL handle");
  if (n_shards < 1 || shard_id < 0 || shard_id >= n_shards)
    return fail(MC_ERR_ARG, "bad shard %d of %d", shard_id, n_shards);
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->appended != 0) return fail(MC_ERR_STATE, "configure the shard before the first append");
  if ((long long)h->Cp * n_shards >= (1ll << 30))  // the streamed scan's records carry 30-bit row offsets
    return fail(MC_ERR_ARG, "capacity %lld x %d shards exceeds 2^30 rows", (long long)h->C, n_shards);
  h->shard = ShardMap{n_shards, shard_id};
  return MC_OK;
}

int mc_set_path(mc_cache* h, int32_t path) {
  if (!h) return fail(MC_ERR_ARG, "NULL handle");
  if (path != MC_PATH_AUTO && path != MC_PATH_GEMV && path != MC_PATH_GEMM && path != MC_PATH_STREAM8)
    return fail(MC_ERR_ARG, "unknown path %d", path);
  std::lock_guard<std::mutex> lk(h->mu);
  h->path = path;
  return MC_OK;
}

int64_t mc_size(const mc_cache* h) { return h ? h->count : -1; }

int mc_append(mc_cache* h, const double* rows, int64_t n) {
  if (!h || (!rows && n > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (n < 0) return fail(MC_ERR_ARG, "negative row count");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  for (int64_t i = 0; i < n; ++i) {
    if (h->n_pending == h->stage_cap) {
      int rc = flush(h);
      if (rc) return rc;
    }
    if (h->n_pending == 0) {
      int rc = wait_env(h);  // the previous flush may still be reading the envelope
      if (rc) return rc;
    }
    if (h->count == h->C) {  // append-then-evict of cache.py:230-233, evicting first
      h->head = (h->head + 1) % h->Cp;
      h->count--;
      h->jhead++;
    }
    const long long slot = (h->head + h->count) % h->Cp;
    if (h->n_pending == 0) h->pending_first_slot = slot;
    double* dst = h->h_env + (size_t)h->n_pending * h->Dp;
    memcpy(dst, rows + (size_t)i * h->D, (size_t)h->D * sizeof(double));
    // the padding must read as zeros: this envelope row may have held an earlier lookup's quantisation block
    if (h->Dp > h->D) memset(dst + h->D, 0, (size_t)(h->Dp - h->D) * sizeof(double));
    h->n_pending++;
    h->count++;
    h->appended++;
    h->state_dirty = true;
  }
  return MC_OK;
}

int mc_evict_front(mc_cache* h, int64_t n) {
  if (!h) return fail(MC_ERR_ARG, "NULL handle");
  std::lock_guard<std::mutex> lk(h->mu);
  if (n < 0 || n > h->count) return fail(MC_ERR_STATE, "cannot evict %lld of %lld live rows", (long long)n,
                                         (long long)h->count);
  if (n == 0) return MC_OK;
  h->head = (h->head + n) % h->Cp;
  h->count -= n;
  h->jhead += n;
  h->state_dirty = true;
  return MC_OK;
}

int mc_retrieve_batch(mc_cache* h, const double* queries, int32_t B, int64_t* out_live, double* out_sim,
                      int32_t* out_k, uint32_t* out_flags) {
  if (!h || (!queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B < 0) return fail(MC_ERR_ARG, "negative batch");
  if (B == 0) return MC_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = retrieve_into_hout(h, queries, B);
  if (rc) return rc;
  return copy_out(h, B, out_live, out_sim, out_k, out_flags);
}

int mc_retrieve_decisions(mc_cache* h, const double* queries, int32_t B, mc_decision* out) {
  if (!h || !out || (!queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B < 0) return fail(MC_ERR_ARG, "negative batch");
  if (B == 0) return MC_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = retrieve_into_hout(h, queries, B);
  if (rc) return rc;
  return copy_decisions(h, B, out);
}

int mc_set_sigma_schedule(mc_cache* h, const double* schedule, int32_t n) {
  if (!h || (!schedule && n > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (n < 0) return fail(MC_ERR_ARG, "negative schedule length");
  std::lock_guard<std::mutex> lk(h->mu);
  h->sched.assign(schedule, schedule + n);
  apply_sigma(h);
  return MC_OK;
}

// Start the DMA of a batch's queries (registered caller memory, tensor-core path) into a query
// slot on the copy stream, before the previous batch is waited for.  The slot alternates: the
// other one may still be read by the batch in flight; this one was last read by a batch that has
// completed (batches pipeline one deep).
int prefetch_queries(mc_cache* h, const double* queries, int B) {
  h->pf_src = nullptr;
  const size_t row = (size_t)h->Dp * sizeof(double);
  if (h->D != h->Dp || !use_gemm(h, B) || !host_registered(queries, (size_t)B * row)) return MC_OK;
  if (!h->cstream) {
    CU(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) CU(cudaEventCreateWithFlags(&h->q_ev[i], cudaEventDisableTiming));
  }
  if (B > h->qslot_cap) {
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaStreamSynchronize(h->cstream));
    int cap = 64;
    while (cap < B) cap <<= 1;
    for (int i = 0; i < 2; ++i) {
      cudaFree(h->d_qslot[i]);
      h->d_qslot[i] = nullptr;
      CU(cudaMalloc(&h->d_qslot[i], (size_t)cap * row));
    }
    h->qslot_cap = cap;
  }
  const int s = h->qslot_next;
  h->qslot_next ^= 1;
  CU(cudaMemcpyAsync(h->d_qslot[s], queries, (size_t)B * row, cudaMemcpyHostToDevice, h->cstream));
  CU(cudaEventRecord(h->q_ev[s], h->cstream));
  h->pf_src = queries;
  h->pf_B = B;
  h->pf_slot = s;
  return MC_OK;
}

int mc_retrieve_submit(mc_cache* h, const double* queries, int32_t B, uint32_t* out_ticket) {
  if (!h || !out_ticket || (!queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B < 1) return fail(MC_ERR_ARG, "batch must be positive");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  // Pipelining: a single-query lookup may be submitted while one other single-query lookup
  // is still in flight (its answer is collected later by its own mc_retrieve_wait).
  const bool pipe = B == 1 && h->count > 0 && h->packed && direct_result(h, 1) && h->n_pending <= PIPE_SLACK;
  if (h->inflight_seq && h->old_seq) {
    // Three deep: a single-query lookup beside two single-query lookups in flight; the older
    // of those moves one level down (old -> old2).
    if (h->old2_seq || B != 1 || h->inflight_B != 1 || h->old_async || !h->old_batch.empty())
      return fail(MC_ERR_STATE, "lookups in flight: mc_retrieve_wait first (three single queries, or two with a batch)");
    const bool deeper = pipe && h->inflight_direct;
    if (!deeper) {  // it cannot run three deep: answer the oldest now (kept for its wait)
      int rc = finish_old(h);
      if (rc) return rc;
    }
    h->old2_seq = h->old_seq;
    h->old2_ready = h->old_ready;
    h->old2_slot = h->old_slot;
    h->old2_st = h->old_st;
    h->old2_out = h->old_out;
    h->old2_written = h->old_written;
    h->old_seq = 0;
    h->old_ready = false;
  }
  if (h->inflight_seq && h->inflight_B != 1) {  // a batch in flight
    if (B > 1 && h->count > 0) {  // this batch's queries start moving while that one still scans
      int rc = prefetch_queries(h, queries, B);
      if (rc) return rc;
    }
    // Two deep: a prefetched batch queues behind the one in flight (the other batch slot), as
    // long as the rows applied since that one's scan stay within the ring's spare slots.
    // Its queries must sit in a query slot: the envelope may be rewritten by this submit, and a
    // late exhaustive fallback of that batch re-reads them.
    const bool in_slot = h->inflight_q && (h->inflight_q == h->d_qslot[0] || h->inflight_q == h->d_qslot[1]);
    const bool deep = h->inflight_async && !h->inflight_ready && in_slot && B > 1 && h->pf_src == queries &&
                      h->appended - h->inflight_appended <= PIPE_SLACK;
    if (deep) {
      h->old_seq = h->inflight_seq;
      h->old_ready = false;
      h->old_async = true;
      h->old_B = h->inflight_B;
      h->old_bslot = h->batch_slot;
      h->old_st = h->inflight_st;
      h->old_q = h->inflight_q;
      h->old_appended = h->inflight_appended;
      h->old_slot = 1;
      h->inflight_seq = 0;
      h->inflight_async = false;
    } else {  // answer it now, keep it for its wait
      int rc = finish_inflight(h);
      if (rc) return rc;
      h->old_batch.assign(bhout(h, h->batch_slot), bhout(h, h->batch_slot) + h->inflight_B);
      h->old_slot = 1;  // a single-query lookup submitted next takes slot 0
      h->old_seq = h->inflight_seq;
      h->old_ready = true;
      h->inflight_seq = 0;
      h->inflight_ready = false;
    }
  }
  if (h->inflight_seq) {
    if (h->inflight_B != 1) return fail(MC_ERR_STATE, "an asynchronous lookup is already in flight");
    if (!pipe || !h->inflight_direct) {  // cannot run beside it: answer it now (kept for its wait)
      int rc = finish_inflight(h);
      if (rc) return rc;
    }
    h->old_seq = h->inflight_seq;  // it becomes the older of the two
    h->old_ready = h->inflight_ready;
    h->old_slot = h->inflight_slot;
    h->old_st = h->inflight_st;
    if (h->old_ready) h->old_out = h->h_out[0];
    h->old_written = 0;
    h->inflight_seq = 0;
  }
  if (h->old_seq && !pipe && !h->old_async) {  // the new lookup cannot run beside it: answer the older one first
    int rc = finish_old(h);
    if (rc) return rc;
  }
  if (h->old2_seq && !h->old2_ready && h->old2_written + h->n_pending > PIPE_SLACK) {
    int rc = finish_old2(h);  // the rows this launch writes would reach the oldest lookup's window
    if (rc) return rc;
  }
  if (h->old_seq && !h->old_ready && !h->old_async && h->old_written + h->n_pending > PIPE_SLACK) {
    int rc = finish_old(h);  // the rows this launch writes would reach the older lookup's window
    if (rc) return rc;
  }
  if (B > h->Bcap && h->old_async) {  // growing the batch buffers: the older batch's answers move first
    int rc = finish_old(h);
    if (rc) return rc;
  }
  int rc = ensure_batch(h, B);
  if (rc) return rc;
  const unsigned seq = ++h->seq;
  h->batch_slot = 0;
  h->inflight_B = B;
  h->inflight_q = nullptr;
  // a batch (B > 1) runs only beside an older lookup that is already answered: slot 0 is free
  if (B == 1 && h->old_seq) {  // a result slot no older lookup holds
    int s = 0;
    while (s == h->old_slot || (h->old2_seq && s == h->old2_slot)) ++s;
    h->inflight_slot = s;
  } else {
    h->inflight_slot = 0;
  }
  h->inflight_st = mirror(h);
  if (h->count == 0) {  // cache.py:252-253: answered now
    for (int b = 0; b < B; ++b) h->h_out[b] = empty_out(h);
    h->inflight_ready = true;
    h->inflight_direct = false;
  } else if (direct_result(h, B)) {  // the kernel publishes into mapped memory; the caller returns now
    const double* q = nullptr;
    if (h->old_seq) h->old_written += std::min(h->n_pending, h->C);
    if (h->old2_seq) h->old2_written += std::min(h->n_pending, h->C);
    // beside an older lookup: inputs in the launch (no envelope copy in the stream, which would
    // serialise behind the older kernel and hold back the host's next append)
    rc = enqueue_direct(h, queries, B, seq, /*async_reuse=*/true, &q, h->inflight_slot, h->old_seq != 0);
    if (rc) return rc;
    h->inflight_q = q;
    h->inflight_ready = false;
    h->inflight_direct = true;
  } else if (B > 1) {  // batches: the decisions come back by an async copy; mc_retrieve_wait (or the
                      // next submit) waits for it.  The caller's query array must stay untouched until
                      // then when it is a registered buffer (the batch is DMA'd straight from it).
    const double* q = nullptr;
    const int bs = h->old_async ? 1 - h->old_bslot : 0;
    h->batch_slot = bs;
    rc = lookup_enqueue(h, queries, B, brec(h, bs), bdout(h, bs), true, &q);
    if (rc) return rc;
    CU(cudaMemcpyAsync(bhout(h, bs), bdout(h, bs), (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaEventRecord(h->batch_ev[bs], h->stream));
    h->inflight_appended = h->appended;
    h->inflight_q = q;
    h->inflight_ready = false;
    h->inflight_direct = false;
    h->inflight_async = true;
  } else {  // paths without a zero-copy result complete synchronously
    const double* q = nullptr;
    rc = lookup_enqueue(h, queries, B, h->d_rec, h->d_out, false, &q);
    if (rc) return rc;
    CU(cudaMemcpyAsync(h->h_out, h->d_out, (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    h->env_inflight = false;
    h->inflight_seq = seq;
    h->inflight_q = q;
    h->inflight_ready = false;
    h->inflight_direct = false;
    *h->h_seq = seq;  // already complete: finish_inflight only applies the fallback
  }
  h->inflight_seq = seq;
  *out_ticket = seq;
  return MC_OK;
}

int mc_retrieve_wait(mc_cache* h, uint32_t ticket, int64_t* out_live, double* out_sim, int32_t* out_k,
                     uint32_t* out_flags) {
  if (!h) return fail(MC_ERR_ARG, "NULL handle");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  if (ticket && ticket == h->old_seq && (h->old_async || !h->old_batch.empty())) {  // an older batch
    int rc = finish_old(h);
    if (rc) return rc;
    const OutRec* src = h->old_batch.data();
    const int B = (int)h->old_batch.size();
    for (int b = 0; b < B; ++b) {
      const OutRec& o = src[b];
      if (out_live) out_live[b] = o.live;
      if (out_sim) out_sim[b] = o.sim;
      if (out_k) out_k[b] = o.k;
      const unsigned f = o.flags & 0xffffu;
      if (out_flags) out_flags[b] = f;
      if (f & MC_FLAG_FALLBACK) h->stats[1]++;
      if (f & MC_FLAG_NONFINITE) h->stats[2]++;
      if (f & MC_FLAG_TIE) h->stats[3]++;
    }
    h->stats[0] += B;
    h->old_batch.clear();
    h->old_seq = 0;
    h->old_ready = false;
    return MC_OK;
  }
  if (ticket && ticket == h->old2_seq) {  // the oldest of three
    int rc = finish_old2(h);
    if (rc) return rc;
    h->old2_seq = 0;
    h->old2_ready = false;
    OutRec* keep = h->h_out;
    const OutRec saved = keep[0];
    keep[0] = h->old2_out;
    rc = copy_out(h, 1, out_live, out_sim, out_k, out_flags);
    keep[0] = saved;
    return rc;
  }
  if (ticket && ticket == h->old_seq) {
    int rc = finish_old(h);
    if (rc) return rc;
    h->old_seq = 0;
    h->old_ready = false;
    OutRec* keep = h->h_out;  // copy_out reads h_out[0]: hand it the older answer, leave the newer's alone
    const OutRec saved = keep[0];
    keep[0] = h->old_out;
    rc = copy_out(h, 1, out_live, out_sim, out_k, out_flags);
    keep[0] = saved;
    return rc;
  }
  if (!h->inflight_seq || ticket != h->inflight_seq) return fail(MC_ERR_STATE, "no lookup %u in flight", ticket);
  int rc = finish_inflight(h);
  if (rc) return rc;
  const int B = h->inflight_B;
  h->inflight_seq = 0;
  h->inflight_ready = false;
  if (h->batch_slot != 0) {  // an asynchronous batch answered in the second slot
    OutRec* keep = h->h_out;
    h->h_out = bhout(h, h->batch_slot);
    rc = copy_out(h, B, out_live, out_sim, out_k, out_flags);
    h->h_out = keep;
    return rc;
  }
  return copy_out(h, B, out_live, out_sim, out_k, out_flags);
}

namespace {
// Merged flags as the C ABI reports them: MC_FLAG_* plus MC_FLAG_NEED_RESCAN for a record that
// still asks for the exhaustive rescan (mc_retrieve_local_submit records).
uint32_t public_flags(unsigned f) { return (f & 0xffffu) | ((f & FLAG_NEED_ANY) ? MC_FLAG_NEED_RESCAN : 0u); }

void remember_window(mc_cache* h, const void* rec) {
  mc_cache::LocalWin& w = h->local_win[h->local_win_next];
  h->local_win_next = (h->local_win_next + 1) % 4;
  w.rec = rec;
  w.st = mirror(h);  // pending rows were folded into this lookup: the window it scanned
  w.appended = h->appended;
}

// A shard's certified local records for B host queries.  exact: the exhaustive rescan of
// records whose certificate failed follows on the stream (always launched; it skips unflagged
// queries).  Otherwise such records keep their FLAG_NEED_* bits, the merge reports
// MC_FLAG_NEED_RESCAN and the caller runs mc_rescan_local before the window changes.
int local_lookup(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream, bool exact) {
  if (!h || !dev_records || (!queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B <= 0) return fail(MC_ERR_ARG, "batch must be positive");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  mc_record* rec = static_cast<mc_record*>(dev_records);
  int rc0 = ensure_batch(h, B);
  if (rc0) return rc0;
  if (h->count == 0) {
    int rc = flush(h);
    if (rc) return rc;
    CU(cudaMemsetAsync(rec, 0xff, (size_t)B * sizeof(mc_record), h->stream));  // pos = -1 (NaN sims)
  } else if (!exact && h->local_param && B == 1 && h->n_pending == 0 && h->s8 && h->Dp <= 1024 &&
             h->path != MC_PATH_GEMV && !use_gemm(h, 1)) {
    // One query, no rows to append: the query and its quantisation ride in the launch's parameter
    // block (no host->device copy between consecutive local scans), and the scan may start while
    // the previous local scan on this ring still merges (the streamed scan's launch overlap).
    take_pending(h, nullptr);  // evictions only: the kernel publishes the window to d_state
    const unsigned ep = s8_epoch(h);
    const cudaError_t e = launch_stream8_direct(h->s8, rbufs(h), mirror(h), h->D, queries, nullptr, h->d_cta,
                                                s8_launch_grid(h), h->shard, h->d_counter, h->d_gmax8, ep, h->thr,
                                                rec, nullptr, h->d_state, nullptr, 0, nullptr, quantize_query,
                                                h->d_gq64, h->d_sync, s8_rec_par(h), !h->tc_tail, h->stream);
    if (e != cudaSuccess) return s8_launch_failed(h, ep, e);
    h->tc_tail = false;
    h->stats[5]++;
    h->stats[7]++;
    remember_window(h, dev_records);
  } else {
    const double* q = nullptr;
    // an envelope copy (and, with `exact`, the rescan) sits between consecutive local scans:
    // no launch overlap, so a large window takes the wide grid
    h->s8_isolated = true;
    int rc = lookup_enqueue(h, queries, B, rec, nullptr, true, &q);
    h->s8_isolated = false;
    if (rc) return rc;
    remember_window(h, dev_records);
    if (exact) {
      CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state, h->D, h->Dp, q, B, rec, h->d_scratch,
                             exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
      h->stats[7] += 2;
    }
  }
  if (stream && stream != h->stream) {  // order the caller's stream (the exchange) after this shard's scan
    CU(cudaEventRecord(h->rec_ev, h->stream));
    CU(cudaStreamWaitEvent((cudaStream_t)stream, h->rec_ev, 0));
  }
  h->stats[0] += B;
  return MC_OK;
}
}  // namespace

int mc_retrieve_local_async(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream) {
  return local_lookup(h, queries, B, dev_records, stream, true);
}

int mc_retrieve_local_submit(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream) {
  return local_lookup(h, queries, B, dev_records, stream, false);
}

int mc_rescan_local(mc_cache* h, const double* queries, int32_t B, void* dev_records, void* stream) {
  if (!h || !dev_records || (!queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B <= 0) return fail(MC_ERR_ARG, "batch must be positive");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = ensure_batch(h, B);
  if (rc) return rc;
  if (stream && stream != h->stream) {  // the records were last written on the caller's stream
    CU(cudaEventRecord(h->rec_ev, (cudaStream_t)stream));
    CU(cudaStreamWaitEvent(h->stream, h->rec_ev, 0));
  }
  const mc_cache::LocalWin* win = nullptr;
  for (int i = 1; i <= 4 && !win; ++i) {  // the most recent lookup into these records
    const mc_cache::LocalWin& w = h->local_win[(h->local_win_next - i + 4) % 4];
    if (w.rec == dev_records) win = &w;
  }
  if (!win) return fail(MC_ERR_STATE, "no recent local lookup wrote these records");
  if (h->appended - win->appended > PIPE_SLACK)
    return fail(MC_ERR_STATE, "%lld rows were appended since the lookup (at most %lld keep its window intact)",
                h->appended - win->appended, PIPE_SLACK);
  if (win->st.count > 0) {
    const double* q = nullptr;
    const QPrep* prep = nullptr;
    const int8_t* q8 = nullptr;
    // queries only; pending appends / evictions are not applied here
    rc = upload_envelope(h, queries, B, true, false, &q, &prep, &q8);
    if (rc) return rc;
    const RingState st = win->st;  // the window the lookup scanned (later lookups may have moved d_state)
    CU(cudaMemcpyAsync(h->d_state_fb, &st, sizeof st, cudaMemcpyHostToDevice, h->stream));
    CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state_fb, h->D, h->Dp, q, B,
                           static_cast<mc_record*>(dev_records), h->d_scratch, exact_grid(h->sm_count),
                           gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
    h->stats[7] += 2;
  }
  if (stream && stream != h->stream) {
    CU(cudaEventRecord(h->rec_ev, h->stream));
    CU(cudaStreamWaitEvent((cudaStream_t)stream, h->rec_ev, 0));
  }
  return MC_OK;
}

int mc_retrieve_local_device(mc_cache* h, const double* d_queries, int32_t B, void* dev_records, void* stream) {
  if (!h || !dev_records || (!d_queries && B > 0)) return fail(MC_ERR_ARG, "NULL argument");
  if (B <= 0) return fail(MC_ERR_ARG, "batch must be positive");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  if (h->D != h->Dp) return fail(MC_ERR_ARG, "device queries need dim %% 64 == 0 (dim %d)", h->D);
  mc_record* rec = static_cast<mc_record*>(dev_records);
  int rc = ensure_batch(h, B);
  if (!rc) rc = flush(h);  // pending appends land first (k_append), as a host-fed lookup would fold them in
  if (rc) return rc;
  if (stream && stream != h->stream) {  // the queries were written on the caller's stream
    CU(cudaEventRecord(h->rec_ev, (cudaStream_t)stream));
    CU(cudaStreamWaitEvent(h->stream, h->rec_ev, 0));
  }
  if (h->count == 0) {
    CU(cudaMemsetAsync(rec, 0xff, (size_t)B * sizeof(mc_record), h->stream));  // pos = -1 (NaN sims)
  } else {
    GemvAppendArgs none{};
    none.rb = rbufs(h);
    none.d_state = h->d_state;
    // no host quantisation: batch >= 5 takes the tensor-core scan, smaller batches the fp16 GEMV scan
    rc = scan_merge(h, d_queries, B, rec, nullptr, none, nullptr, nullptr);
    if (rc) return rc;
    CU(launch_exact_rescan(h->ring16, h->ring64, h->d_state, h->D, h->Dp, d_queries, B, rec, h->d_scratch,
                           exact_grid(h->sm_count), gemv_eps_rel(h->Dp), eps_abs1(), h->shard, h->stream));
    h->stats[7] += 2;
  }
  if (stream && stream != h->stream) {  // order the caller's stream (the exchange) after this shard's scan
    CU(cudaEventRecord(h->rec_ev, h->stream));
    CU(cudaStreamWaitEvent((cudaStream_t)stream, h->rec_ev, 0));
  }
  h->stats[0] += B;
  return MC_OK;
}

int mc_merge_records(mc_cache* h, const void* dev_records, int32_t G, int32_t B, int64_t p0, void* stream,
                     int64_t* out_live, double* out_sim, int32_t* out_k, uint32_t* out_flags) {
  if (!h || !dev_records) return fail(MC_ERR_ARG, "NULL argument");
  if (G < 1 || B <= 0 || p0 < 0) return fail(MC_ERR_ARG, "bad merge shape G=%d B=%d p0=%lld", G, B, (long long)p0);
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = ensure_batch(h, B);
  if (rc) return rc;
  cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
  CU(launch_finalize(static_cast<const mc_record*>(dev_records), G, B, p0, h->d_state, h->thr, h->d_out, s));
  CU(cudaMemcpyAsync(h->h_out, h->d_out, (size_t)B * sizeof(OutRec), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  h->stats[7]++;
  for (int b = 0; b < B; ++b) {
    const OutRec& o = h->h_out[b];
    if (out_live) out_live[b] = o.live;
    if (out_sim) out_sim[b] = o.sim;
    if (out_k) out_k[b] = o.k;
    if (out_flags) out_flags[b] = public_flags(o.flags);
  }
  return MC_OK;
}

int mc_merge_records_submit(mc_cache* h, const void* dev_records, int32_t G, int32_t B, int64_t p0, void* stream,
                            int32_t slot) {
  if (!h || !dev_records) return fail(MC_ERR_ARG, "NULL argument");
  if (G < 1 || B <= 0 || p0 < 0) return fail(MC_ERR_ARG, "bad merge shape G=%d B=%d p0=%lld", G, B, (long long)p0);
  if (slot < 0 || slot >= MC_MERGE_SLOTS) return fail(MC_ERR_ARG, "merge slot %d outside [0, %d)", slot, MC_MERGE_SLOTS);
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  if (h->merge_B[slot]) return fail(MC_ERR_STATE, "merge slot %d still holds an unread result", slot);
  if (B > h->merge_cap) {  // grow every slot; an unread result in another slot moves along
    int cap = 4;
    while (cap < B) cap <<= 1;
    for (int i = 0; i < MC_MERGE_SLOTS; ++i) {
      OutRec* nh = nullptr;
      CU(cudaHostAlloc(&nh, (size_t)cap * sizeof(OutRec), cudaHostAllocMapped));
      if (h->merge_B[i]) {  // its merge must land before the copy
        CU(cudaEventSynchronize(h->merge_ev[i]));
        memcpy(nh, h->h_merge[i], (size_t)h->merge_B[i] * sizeof(OutRec));
      }
      cudaFreeHost(h->h_merge[i]);
      h->h_merge[i] = nh;
      CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_merge[i]), h->h_merge[i], 0));
      if (!h->merge_ev[i]) CU(cudaEventCreateWithFlags(&h->merge_ev[i], cudaEventDisableTiming));
    }
    h->merge_cap = cap;
  }
  cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
  // decisions go straight to the mapped host block (kernel completion publishes them)
  CU(launch_finalize(static_cast<const mc_record*>(dev_records), G, B, p0, h->d_state, h->thr, h->d_merge[slot], s));
  CU(cudaEventRecord(h->merge_ev[slot], s));
  h->merge_B[slot] = B;
  h->stats[7]++;
  return MC_OK;
}

int mc_merge_records_wait(mc_cache* h, int32_t slot, int64_t* out_live, double* out_sim, int32_t* out_k,
                          uint32_t* out_flags) {
  if (!h) return fail(MC_ERR_ARG, "NULL argument");
  if (slot < 0 || slot >= MC_MERGE_SLOTS) return fail(MC_ERR_ARG, "merge slot %d outside [0, %d)", slot, MC_MERGE_SLOTS);
  cudaEvent_t ev;
  int B;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    B = h->merge_B[slot];
    if (!B) return fail(MC_ERR_STATE, "merge slot %d holds no submitted merge", slot);
    ev = h->merge_ev[slot];
  }
  CU(cudaEventSynchronize(ev));  // outside the lock: other lookups may be enqueued meanwhile
  std::lock_guard<std::mutex> lk(h->mu);
  const OutRec* o = h->h_merge[slot];
  for (int b = 0; b < B; ++b) {
    if (out_live) out_live[b] = o[b].live;
    if (out_sim) out_sim[b] = o[b].sim;
    if (out_k) out_k[b] = o[b].k;
    if (out_flags) out_flags[b] = public_flags(o[b].flags);
  }
  h->merge_B[slot] = 0;
  return MC_OK;
}

int mc_profile_steps(mc_cache* h, const double* queries, const double* rows, int32_t B, int32_t iters,
                     int64_t flush_bytes, double* out_ms, int64_t* out_counts) {
  if (!h || !queries || !out_ms || !out_counts) return fail(MC_ERR_ARG, "NULL argument");
  if (B < 1 || iters < 1) return fail(MC_ERR_ARG, "need B >= 1 and iters >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = ensure_batch(h, B);
  if (rc) return rc;
  rc = flush(h);
  if (rc) return rc;
  if (h->count == 0 && !rows) return fail(MC_ERR_STATE, "profile needs a non-empty cache");
  const size_t qbytes = (size_t)iters * B * h->Dp * sizeof(double);
  double *d_qall = nullptr, *d_rows = nullptr;
  OutRec* d_outs = nullptr;
  void* d_flush = nullptr;
  QPrep* d_prep = nullptr;
  int8_t* d_q8 = nullptr;
  const int nev = 3;
  std::vector<cudaEvent_t> ev((size_t)iters * nev, nullptr);
  auto release = [&]() {
    cudaStreamSynchronize(h->stream);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    cudaFree(d_qall);
    cudaFree(d_rows);
    cudaFree(d_outs);
    cudaFree(d_flush);
    cudaFree(d_prep);
    cudaFree(d_q8);
  };
#define CUP(call)                                                                                      \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) {                                                                           \
      release();                                                                                       \
      return fail(MC_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
    }                                                                                                  \
  } while (0)
  CUP(cudaMalloc(&d_qall, qbytes));
  CUP(cudaMemset(d_qall, 0, qbytes));
  CUP(cudaMemcpy2D(d_qall, (size_t)h->Dp * sizeof(double), queries, (size_t)h->D * sizeof(double),
                   (size_t)h->D * sizeof(double), (size_t)iters * B, cudaMemcpyHostToDevice));
  if (rows) {
    CUP(cudaMalloc(&d_rows, (size_t)iters * h->Dp * sizeof(double)));
    CUP(cudaMemset(d_rows, 0, (size_t)iters * h->Dp * sizeof(double)));
    CUP(cudaMemcpy2D(d_rows, (size_t)h->Dp * sizeof(double), rows, (size_t)h->D * sizeof(double),
                     (size_t)h->D * sizeof(double), (size_t)iters, cudaMemcpyHostToDevice));
  }
  CUP(cudaMalloc(&d_outs, (size_t)iters * B * sizeof(OutRec)));
  {  // the steps' query quantisation, prepared up front like the queries themselves
    std::vector<QPrep> hp((size_t)iters * B);
    std::vector<int8_t> h8((size_t)iters * B * h->Dp);
    std::vector<double> qrow(h->Dp, 0.0);
    for (size_t i = 0; i < hp.size(); ++i) {
      memcpy(qrow.data(), queries + i * h->D, h->D * sizeof(double));
      quantize_query(qrow.data(), h->D, h->Dp, &hp[i], &h8[i * h->Dp]);
    }
    CUP(cudaMalloc(&d_prep, hp.size() * sizeof(QPrep)));
    CUP(cudaMalloc(&d_q8, h8.size()));
    CUP(cudaMemcpy(d_prep, hp.data(), hp.size() * sizeof(QPrep), cudaMemcpyHostToDevice));
    CUP(cudaMemcpy(d_q8, h8.data(), h8.size(), cudaMemcpyHostToDevice));
  }
  if (flush_bytes > 0) {
    CUP(cudaMalloc(&d_flush, (size_t)flush_bytes));
    CUP(cudaMemsetAsync(d_flush, 1, (size_t)flush_bytes, h->stream));
  }
  for (auto& e : ev) CUP(cudaEventCreate(&e));
  const long long launches0 = h->stats[7];
  const bool gemm = use_gemm(h, B);  // tensor-core sequence: also time scan and merge separately
  for (int it = 0; it < iters; ++it) {
    if (d_flush) CUP(launch_l2_flush(d_flush, (size_t)flush_bytes, h->stream));
    CUP(cudaEventRecord(ev[(size_t)it * nev + 0], h->stream));
    GemvAppendArgs app;
    app.rb = rbufs(h);
    app.d_state = h->d_state;
    if (rows) {  // one FIFO insert per step, already resident on the device
      if (h->count == h->C) {
        h->head = (h->head + 1) % h->Cp;
        h->count--;
        h->jhead++;
      }
      app.stage = d_rows + (size_t)it * h->Dp;
      app.n = 1;
      app.first_slot = (h->head + h->count) % h->Cp;
      h->count++;
      h->appended++;
    }
    const double* q = d_qall + (size_t)it * B * h->Dp;
    rc = scan_merge(h, q, B, h->d_rec, d_outs + (size_t)it * B, app, d_prep + (size_t)it * B,
                    d_q8 + (size_t)it * B * h->Dp, gemm ? ev[(size_t)it * nev + 1] : nullptr);
    if (rc) {
      release();
      return rc;
    }
    CUP(cudaEventRecord(ev[(size_t)it * nev + 2], h->stream));
  }
  CUP(cudaStreamSynchronize(h->stream));
  double tot = 0, t_scan = 0, t_merge = 0;
  for (int it = 0; it < iters; ++it) {
    float a = 0.f, b = 0.f;
    if (gemm) {
      CUP(cudaEventElapsedTime(&a, ev[(size_t)it * nev + 0], ev[(size_t)it * nev + 1]));
      CUP(cudaEventElapsedTime(&b, ev[(size_t)it * nev + 1], ev[(size_t)it * nev + 2]));
    } else {  // one fused launch per step: the step is the kernel
      CUP(cudaEventElapsedTime(&a, ev[(size_t)it * nev + 0], ev[(size_t)it * nev + 2]));
    }
    t_scan += a;
    t_merge += b;
    tot += a + b;
  }
  std::vector<OutRec> outs((size_t)iters * B);
  CUP(cudaMemcpy(outs.data(), d_outs, outs.size() * sizeof(OutRec), cudaMemcpyDeviceToHost));
  long long need = 0;
  for (int it = 0; it < iters; ++it) {
    bool any = false;
    for (int b = 0; b < B; ++b) any |= (outs[(size_t)it * B + b].flags & FLAG_NEED_ANY) != 0;
    need += any;
  }
  out_ms[0] = tot / iters;
  out_ms[1] = t_scan / iters;
  out_ms[2] = t_merge / iters;
  out_ms[3] = 0.0;  // appends ride inside the scan launch (or its k_append, timed with the scan)
  out_counts[0] = (h->stats[7] - launches0) / iters;
  out_counts[1] = need;
  release();
#undef CUP
  return MC_OK;
}

// Measurement hook: `iters` back-to-back steps rotating over nh caches of the
// same shape (their scan copies together larger than L2, so every step streams
// its ring from HBM), timed by ONE pair of CUDA events on hs[0]'s stream — no
// per-step event or flush in the timed region.  Step i = [append rows[i]] +
// lookup of queries[i] (B x dim) on cache hs[i % nh].
int mc_profile_rotate(mc_cache* const* hs, int32_t nh, const double* queries, const double* rows, int32_t B,
                      int32_t iters, double* out_ms, int64_t* out_counts) {
  if (!hs || nh < 1 || !queries || !out_ms || !out_counts) return fail(MC_ERR_ARG, "NULL argument");
  if (B < 1 || iters < 1) return fail(MC_ERR_ARG, "need B >= 1 and iters >= 1");
  mc_cache* h0 = hs[0];
  for (int k = 0; k < nh; ++k) {
    if (!hs[k]) return fail(MC_ERR_ARG, "NULL handle %d", k);
    if (hs[k]->dev != h0->dev || hs[k]->D != h0->D || hs[k]->C != h0->C)
      return fail(MC_ERR_ARG, "rotation needs caches of one shape on one device");
    if (hs[k]->count == 0 && !rows) return fail(MC_ERR_STATE, "profile needs non-empty caches");
  }
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int k = 0; k < nh; ++k) locks.emplace_back(hs[k]->mu);
  DeviceGuard guard(h0->dev);
  for (int k = 0; k < nh; ++k) {
    int rc = ensure_batch(hs[k], B);
    if (!rc) rc = flush(hs[k]);
    if (!rc && use_gemm(hs[k], B)) rc = ensure_tc(hs[k], B);
    if (rc) return rc;
    CU(cudaStreamSynchronize(hs[k]->stream));
  }
  const int D = h0->D, Dp = h0->Dp;
  double *d_qall = nullptr, *d_rows = nullptr;
  OutRec* d_outs = nullptr;
  QPrep* d_prep = nullptr;
  int8_t* d_q8 = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaStream_t common = h0->stream;
  std::vector<cudaStream_t> saved(nh);
  for (int k = 0; k < nh; ++k) saved[k] = hs[k]->stream;
  auto release = [&]() {
    cudaStreamSynchronize(common);
    for (int k = 0; k < nh; ++k) hs[k]->stream = saved[k];
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(d_qall);
    cudaFree(d_rows);
    cudaFree(d_outs);
    cudaFree(d_prep);
    cudaFree(d_q8);
  };
#define CUR(call)                                                                                      \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) {                                                                           \
      release();                                                                                       \
      return fail(MC_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));    \
    }                                                                                                  \
  } while (0)
  const size_t qbytes = (size_t)iters * B * Dp * sizeof(double);
  CUR(cudaMalloc(&d_qall, qbytes));
  CUR(cudaMemset(d_qall, 0, qbytes));
  CUR(cudaMemcpy2D(d_qall, (size_t)Dp * sizeof(double), queries, (size_t)D * sizeof(double), (size_t)D * sizeof(double),
                   (size_t)iters * B, cudaMemcpyHostToDevice));
  if (rows) {
    CUR(cudaMalloc(&d_rows, (size_t)iters * Dp * sizeof(double)));
    CUR(cudaMemset(d_rows, 0, (size_t)iters * Dp * sizeof(double)));
    CUR(cudaMemcpy2D(d_rows, (size_t)Dp * sizeof(double), rows, (size_t)D * sizeof(double), (size_t)D * sizeof(double),
                     (size_t)iters, cudaMemcpyHostToDevice));
  }
  CUR(cudaMalloc(&d_outs, (size_t)iters * B * sizeof(OutRec)));
  {
    std::vector<QPrep> hp((size_t)iters * B);
    std::vector<int8_t> h8((size_t)iters * B * Dp);
    std::vector<double> qrow(Dp, 0.0);
    for (size_t i = 0; i < hp.size(); ++i) {
      memcpy(qrow.data(), queries + i * D, D * sizeof(double));
      quantize_query(qrow.data(), D, Dp, &hp[i], &h8[i * Dp]);
    }
    CUR(cudaMalloc(&d_prep, hp.size() * sizeof(QPrep)));
    CUR(cudaMalloc(&d_q8, h8.size()));
    CUR(cudaMemcpy(d_prep, hp.data(), hp.size() * sizeof(QPrep), cudaMemcpyHostToDevice));
    CUR(cudaMemcpy(d_q8, h8.data(), h8.size(), cudaMemcpyHostToDevice));
  }
  CUR(cudaEventCreate(&e0));
  CUR(cudaEventCreate(&e1));
  for (int k = 0; k < nh; ++k) hs[k]->stream = common;
  long long launches0 = 0;
  for (int k = 0; k < nh; ++k) launches0 += hs[k]->stats[7];
  // Hold the stream with a timed spin while the steps are enqueued, so the first timed step does
  // not wait for its own host-side launch and every step is queued when its predecessor ends
  // (the host's enqueue rate, ~4 us per launch, is not part of the device time being measured).
  CUR(launch_spin(std::min<long long>(20000000ll, 6000ll * iters + 200000ll), common));
  CUR(cudaEventRecord(e0, common));
  for (int it = 0; it < iters; ++it) {
    mc_cache* h = hs[it % nh];
    GemvAppendArgs app;
    app.rb = rbufs(h);
    app.d_state = h->d_state;
    if (rows) {
      if (h->count == h->C) {
        h->head = (h->head + 1) % h->Cp;
        h->count--;
        h->jhead++;
      }
      app.stage = d_rows + (size_t)it * Dp;
      app.n = 1;
      app.first_slot = (h->head + h->count) % h->Cp;
      h->count++;
      h->appended++;
    }
    int rc = scan_merge(h, d_qall + (size_t)it * B * Dp, B, h->d_rec, d_outs + (size_t)it * B, app,
                        d_prep + (size_t)it * B, d_q8 + (size_t)it * B * Dp);
    if (rc) {
      release();
      return rc;
    }
  }
  CUR(cudaEventRecord(e1, common));
  CUR(cudaEventSynchronize(e1));
  float ms = 0.f;
  CUR(cudaEventElapsedTime(&ms, e0, e1));
  long long launches1 = 0;
  for (int k = 0; k < nh; ++k) launches1 += hs[k]->stats[7];
  std::vector<OutRec> outs((size_t)iters * B);
  CUR(cudaMemcpy(outs.data(), d_outs, outs.size() * sizeof(OutRec), cudaMemcpyDeviceToHost));
  long long need = 0;
  for (size_t i = 0; i < outs.size(); ++i) need += (outs[i].flags & FLAG_NEED_ANY) != 0;
  out_ms[0] = ms / iters;
  out_counts[0] = (launches1 - launches0) / iters;
  out_counts[1] = need;
  release();
#undef CUR
  return MC_OK;
}

// Measurement hook (MC_GEMV_TIMING=1): read (reset=0) or reset (reset=1) the
// GEMV phase timestamps; 8 x u64 nanoseconds.  Not part of the stable ABI.
int mc_debug_gemv_timing(unsigned long long* out8, int reset) {
  unsigned long long* t = gemv_timing_buffer();
  if (!t) return fail(MC_ERR_STATE, "set MC_GEMV_TIMING=1 before the first lookup");
  CU(cudaDeviceSynchronize());
  if (reset == 2) {  // per-CTA stamps of the streamed scan: [cta][8] then [cta][4] after the 8 globals
    CU(cudaMemcpy(out8, t + 8, 12 * 512 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  } else if (reset) {
    const unsigned long long init8[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    CU(cudaMemset(t + 8, 0, 12 * 512 * sizeof(unsigned long long)));
    CU(cudaMemcpy(t, init8, sizeof init8, cudaMemcpyHostToDevice));
  } else {
    CU(cudaMemcpy(out8, t, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  }
  return MC_OK;
}

// Measurement / debugging hook: the float64 master copy of live row `live`
// (0 = oldest) after every pending append has landed.  Not part of the drop-in.
int mc_generate_rows(mc_cache* h, int64_t n, const double* centers, int32_t n_centers, double spread, double beta,
                     uint64_t seed, int64_t row0) {
  if (!h || !centers) return fail(MC_ERR_ARG, "NULL argument");
  if (n < 0 || n_centers < 1) return fail(MC_ERR_ARG, "need n >= 0 and n_centers >= 1");
  if (h->D > 1024) return fail(MC_ERR_ARG, "the generator covers dim <= 1024 (dim %d)", h->D);
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  int rc = flush(h);  // pending appends precede the generated rows
  if (rc) return rc;
  if (n == 0) return MC_OK;
  // FIFO semantics of n appends: only the newest min(n, C) rows stay live
  const long long keep = std::min<long long>(n, h->C);
  const long long skip = n - keep;
  const long long drop = std::max<long long>(0, h->count + keep - h->C);
  h->head = (h->head + drop) % h->Cp;
  h->count -= drop;
  h->jhead += drop;
  if (skip > 0) {  // every earlier row is evicted; the skipped rows pass through the ring unseen
    h->head = (h->head + h->count) % h->Cp;
    h->jhead += h->count + skip;
    h->count = 0;
  }
  const long long first_slot = (h->head + h->count) % h->Cp;
  h->count += keep;
  h->appended += n;
  h->state_dirty = false;
  double* d_ctr = nullptr;
  std::vector<double> ctr((size_t)n_centers * h->Dp, 0.0);
  for (int c = 0; c < n_centers; ++c) memcpy(&ctr[(size_t)c * h->Dp], centers + (size_t)c * h->D, h->D * sizeof(double));
  CU(cudaMallocAsync(&d_ctr, ctr.size() * sizeof(double), h->stream));
  CU(cudaMemcpyAsync(d_ctr, ctr.data(), ctr.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  CU(launch_generate(keep, first_slot, mirror(h), h->D, h->Dp, rbufs(h), d_ctr, n_centers, spread, beta, seed,
                     row0 + skip, h->d_state, h->stream));
  CU(cudaFreeAsync(d_ctr, h->stream));
  CU(cudaStreamSynchronize(h->stream));  // the host centre buffer goes out of scope
  h->stats[7]++;
  return MC_OK;
}

int mc_read_rows(mc_cache* h, int64_t first_live, int64_t n, double* out) {
  if (!h || (!out && n > 0)) return fail(MC_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  if (first_live < 0 || n < 0 || first_live + n > h->count)
    return fail(MC_ERR_ARG, "rows [%lld, %lld) outside the %lld live rows", (long long)first_live,
                (long long)(first_live + n), (long long)h->count);
  int rc = flush(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  long long done = 0;
  while (done < n) {  // at most two contiguous slot ranges (the ring wraps once)
    const long long slot = (h->head + first_live + done) % h->Cp;
    const long long run = std::min<long long>(n - done, h->Cp - slot);
    CU(cudaMemcpy2D(out + (size_t)done * h->D, (size_t)h->D * sizeof(double), h->ring64 + (size_t)slot * h->Dp,
                    (size_t)h->Dp * sizeof(double), (size_t)h->D * sizeof(double), (size_t)run,
                    cudaMemcpyDeviceToHost));
    done += run;
  }
  return MC_OK;
}

int mc_register_host(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return fail(MC_ERR_ARG, "NULL or empty host buffer");
  cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) return fail(MC_ERR_CUDA, "cudaHostRegister(%lld bytes): %s", (long long)bytes,
                                    cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(g_reg_mu);
  g_reg.push_back(HostRange{reinterpret_cast<uintptr_t>(ptr), reinterpret_cast<uintptr_t>(ptr) + (size_t)bytes});
  return MC_OK;
}

int mc_unregister_host(void* ptr) {
  if (!ptr) return fail(MC_ERR_ARG, "NULL host buffer");
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = std::find_if(g_reg.begin(), g_reg.end(),
                           [&](const HostRange& r) { return r.lo == reinterpret_cast<uintptr_t>(ptr); });
    if (it == g_reg.end()) return fail(MC_ERR_ARG, "host buffer %p was not registered", ptr);
    g_reg.erase(it);
  }
  // every handle's copies out of it are complete: the calls that use it are synchronous
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) return fail(MC_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
  return MC_OK;
}

int mc_debug_read_row(mc_cache* h, int64_t live, double* out) {
  if (!h || !out) return fail(MC_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard guard(h->dev);
  if (live < 0 || live >= h->count) return fail(MC_ERR_ARG, "live index %lld outside [0, %lld)", (long long)live,
                                                (long long)h->count);
  int rc = flush(h);
  if (rc) return rc;
  CU(cudaStreamSynchronize(h->stream));
  const long long slot = (h->head + live) % h->Cp;
  CU(cudaMemcpy(out, h->ring64 + (size_t)slot * h->Dp, (size_t)h->D * sizeof(double), cudaMemcpyDeviceToHost));
  if (getenv("MC_DEBUG_COPIES")) {  // out has room for 3 rows: float64, fp16, int8 x scale
    std::vector<__half> r16(h->Dp);
    std::vector<int8_t> r8(h->P8);
    float2 q;
    CU(cudaMemcpy(r16.data(), h->ring16 + (size_t)slot * h->Dp, (size_t)h->Dp * sizeof(__half), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(r8.data(), h->ring8 + (size_t)slot * h->P8, (size_t)h->P8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&q, h->ringq + slot, sizeof q, cudaMemcpyDeviceToHost));
    for (int i = 0; i < h->D; ++i) {
      out[h->D + i] = (double)__half2float(r16[i]);
      out[2 * h->D + i] = (double)r8[i] * q.x;
    }
  }
  return MC_OK;
}

int mc_stats(const mc_cache* h, int64_t* out8) {
  if (!h || !out8) return fail(MC_ERR_ARG, "NULL argument");
  for (int i = 0; i < 8; ++i) out8[i] = h->stats[i];
  return MC_OK;
}

}  // extern "C"
