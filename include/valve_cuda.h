/*
 * valve_cuda.h -- the C-ABI drop-in boundary of the B200 colocation hot path.
 *
 * Everything behind these entry points runs as sm_100a CUDA kernels on the pool's
 * device (libvalve.so, built from paper_2604_07874_b200/csrc).  There is no CPU
 * fallback: creating a pool without a usable CUDA device fails with VALVE_CUDA_ERROR.
 *
 * Each entry point replaces one method of the reference runtime API in
 * /root/reference/proj/include/colosim (cited per function).  Value semantics are the
 * reference's; C++ exceptions become status codes:
 *     std::invalid_argument -> VALVE_INVALID_ARGUMENT
 *     std::out_of_range     -> VALVE_OUT_OF_RANGE   (std::vector::at in the reference)
 *     std::logic_error      -> VALVE_LOGIC_ERROR
 *     std::runtime_error    -> VALVE_RUNTIME_ERROR  (also capacity limits of the device tables)
 *     any CUDA failure      -> VALVE_CUDA_ERROR
 * and valve_last_error() returns the message (thread-local).  Nothing throws across
 * this boundary.  include/colosim/*.hpp re-raise the same exception types so callers
 * written against the reference compile and behave unchanged.
 *
 * Sizes: arrays are plain pointers plus explicit capacities.  Output functions
 * always report the full size; pass a NULL buffer / zero capacity to query it.
 */
#ifndef VALVE_CUDA_H
#define VALVE_CUDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VALVE_OK = 0,
  VALVE_INVALID_ARGUMENT = 1,
  VALVE_LOGIC_ERROR = 2,
  VALVE_RUNTIME_ERROR = 3,
  VALVE_CUDA_ERROR = 4,
  VALVE_OUT_OF_RANGE = 5,
};

const char* valve_last_error(void);
/* Number of CUDA kernels this library launched in this process (all pools, gates, copies). */
int64_t valve_kernel_launches(void);

/* ================================================================ pool (a1, c1-c3, c5) */
/* Replaces colosim::MemoryPool (memory.hpp:19-98).  Device layout: see DESIGN.md §3. */
typedef struct valve_pool valve_pool;

typedef struct {
  int device;                 /* CUDA ordinal */
  int total_handles;          /* memory.hpp:23 */
  int handle_size_pages;      /* <= 256 */
  int page_size_tokens;
  int64_t slot_bytes;         /* physical bytes per page slot; 0 = no page store (decisions only) */
  int64_t page_bytes;         /* bytes of KV actually held per page (<= slot_bytes) */
  int max_requests;           /* initial rows of the device request table (grows on demand) */
  int max_pages_per_request;  /* initial block-table row length (grows on demand) */
} valve_pool_config;

/* Defaults: device 0, slot_bytes 0, page_bytes 0, max_requests 4096, max_pages 4096.  The two
 * table sizes are starting points, not limits: offline_reserve grows the request table and the
 * block-table rows when a reservation needs more (the reference MemoryPool has no such limit),
 * which moves valve_pool_view.block_tables / max_pages_per_request -- re-read the view after a
 * reserve if you cache it. */
void valve_pool_config_default(valve_pool_config* cfg);
/* memory.hpp:23 MemoryPool(total_handles, handle_size_pages, page_size_tokens) */
int valve_pool_create(int total_handles, int handle_size_pages, int page_size_tokens, valve_pool** out);
int valve_pool_create_ex(const valve_pool_config* cfg, valve_pool** out);
void valve_pool_destroy(valve_pool* p);
/* Back to the freshly created state (all handles free, empty request table, no copies, idle rate
 * bucket), keeping the allocation and the page store's bytes.  Waits for in-flight copies. */
int valve_pool_reset(valve_pool* p);
/* Ids of the online-reserved handles, ascending (the physical home of online pages: the
 * reference keeps online pages as an aggregate, memory.hpp:97, so a tenant that places its KV
 * in the pool's slots needs to know which handles it holds). */
int valve_pool_online_handles(const valve_pool* p, int* out, int cap, int* n);

/* out = {free_handles, online_handles, offline_handles, online_used_pages,
 *        online_capacity_pages}  (memory.hpp:28-41) */
int valve_pool_counts(const valve_pool* p, int64_t out[5]);
int valve_pool_geometry(const valve_pool* p, int out[4]); /* H, S, page_tokens, quarantine id */
int64_t valve_pool_quarantine_page_id(const valve_pool* p); /* memory.hpp:33-35 */

int valve_pool_online_grow(valve_pool* p, int k, int64_t t);            /* memory.hpp:43 */
int valve_pool_online_release(valve_pool* p, int k, int* released);    /* memory.hpp:45 */
int valve_pool_online_use_pages(valve_pool* p, int64_t n);             /* memory.hpp:47 */
int valve_pool_online_free_pages(valve_pool* p, int64_t n);            /* memory.hpp:48 */
int valve_pool_offline_reserve(valve_pool* p, int64_t req, int pages, int64_t t,
                               int max_offline_handles, int* ok);      /* memory.hpp:54 */
int valve_pool_offline_release(valve_pool* p, int64_t req);            /* memory.hpp:56 */
int valve_pool_requests_on_handle(const valve_pool* p, int handle, int64_t* out, int cap,
                                  int* n);                             /* memory.hpp:57 */
int valve_pool_handles_of_request(const valve_pool* p, int64_t req, int* out, int cap,
                                  int* n);                             /* memory.hpp:58 */
int valve_pool_offline_pages_of(const valve_pool* p, int64_t req, int* out); /* memory.hpp:59 */
/* memory.hpp:62 snapshot(): CSR ids[nh], mapped_at[nh], off[nh+1], reqs[nr] */
int valve_pool_snapshot(const valve_pool* p, int* ids, int64_t* mapped_at, int* off, int64_t* reqs,
                        int cap_h, int cap_r, int* nh, int* nr);
/* memory.hpp:64-71 apply_reclaim().  handles[n_handles]; evicted[n_evicted] ascending;
 * inv_off[n_evicted+1] CSR into inv_pages (logical ids the reference reports, ascending per
 * request).  inv_phys / inv_blk (may be NULL) are aligned with inv_pages: the physical page
 * the bytes live in, and the page's block index inside its request.  The device keeps the
 * physical list for valve_pool_reclaim_copy(). */
int valve_pool_apply_reclaim(valve_pool* p, const int* ids, int k, int64_t t, int* handles,
                             int* n_handles, int64_t* evicted, int* n_evicted, int* inv_off,
                             int64_t* inv_pages, int* inv_phys, int* inv_blk, int cap_ev,
                             int cap_pages, int* n_pages);
/* Zero-copy forms of snapshot / apply_reclaim for C++ callers (the include/colosim drop-in): the
 * results land in pinned staging owned by the pool (one DMA each, no pageable copies) and the
 * returned pointers stay valid until the next snapshot / apply / last_reclaim call on the pool. */
int valve_pool_snapshot_view(valve_pool* p, const int** ids, const int64_t** mapped_at, const int** off,
                             const int64_t** reqs, int* nh, int* nr);
int valve_pool_apply_reclaim_view(valve_pool* p, const int* ids, int k, int64_t t, const int** handles,
                                  int* n_handles, const int64_t** evicted, int* n_evicted, const int** inv_off,
                                  const int64_t** inv_pages, int* n_pages);
int valve_pool_handle_state(const valve_pool* p, int handle, int* state);      /* memory.hpp:73 */
int valve_pool_handle_mapped_at(const valve_pool* p, int handle, int64_t* t);  /* memory.hpp:74 */
int valve_pool_check_invariants(const valve_pool* p);                          /* memory.hpp:78 */
/* Block table of a live offline request: physical page ids in block order. */
int valve_pool_block_table(const valve_pool* p, int64_t req, int* out, int cap, int* n);

/* ------------------------------------------------- fused device reclaim (a2+a3+a5 on-device) */
/* Recompute costs (requests.hpp:68-69, sim.cpp:877-883) kept next to each request row. */
int valve_pool_set_costs(valve_pool* p, int n, const int64_t* reqs, const int64_t* costs);
/* Per-request page size (C3: weight pages fill whole slots while a KV page of the offline model is
 * page_bytes): 0 = the pool's page_bytes, else a 16-byte multiple <= slot_bytes.  Kept with the
 * request row; reclaim reports, fill_pages, the gather copy and restore all honour it. */
int valve_pool_set_page_bytes(valve_pool* p, int n, const int64_t* reqs, const int64_t* bytes);
/* Destination layout of the last apply/reclaim report: total bytes the copy writes, and the page
 * size of each evicted request (report order; request e's pages follow those of requests < e). */
int valve_pool_last_copy_layout(const valve_pool* p, int64_t* page_bytes, int cap, int64_t* total);
enum { VALVE_SELECT_SELECTIVE = 0, VALVE_SELECT_FIFO = 1, VALVE_SELECT_ORACLE = 2 };
/* snapshot -> selection (mode) -> apply_reclaim on the device with no host round trip in
 * between (sim.cpp:936-942): a grid-wide instance pass, then one CTA for selection + apply, both
 * stream-ordered on the pool stream.  Results stay on the device for valve_pool_reclaim_copy();
 * the summary (n_handles, n_evicted, n_pages) is returned; use
 * valve_pool_last_reclaim() to read the full result. */
int valve_pool_reclaim(valve_pool* p, int k, int mode, int64_t t, int* n_handles, int* n_evicted,
                       int* n_pages);
/* Device phase durations of the last valve_pool_reclaim (ns, %globaltimer): out[0] instance
 * build (snapshot), out[1] selection, out[2] apply; out[3..4] SM cycles of the greedy rounds
 * (argmin, incremental update); out[5..8] apply sub-phases (evicted rows + ranks, report order,
 * residual release, request-table erase), out[9..11] (validation, slot collection, per-handle
 * ranks) of the last apply, out[12..15] selection sub-phases (dense request ids, CSR + reverse
 * index, packed-key checks, rounds) of the last selection in this process.  Diagnostics. */
int valve_pool_reclaim_phases(const valve_pool* p, int64_t out[16]);
int valve_pool_last_reclaim(const valve_pool* p, int* handles, int64_t* evicted, int* inv_off,
                            int64_t* inv_pages, int* inv_phys, int* inv_blk, int cap_h, int cap_ev,
                            int cap_pages);

/* ------------------------------------------------------------- reclaim copy (a6) */
typedef struct {
  int ctas;                 /* copy CTAs (keep small so online keeps the SMs); 0 = default */
  int threads;              /* threads per CTA; 0 = default */
  int64_t chunk_bytes;      /* work unit; 0 = default (64 KiB) */
  double rate_bytes_per_s;  /* rate bound; <= 0 = unbounded */
  int64_t burst_bytes;      /* token-bucket depth for the rate bound */
  int use_tma;              /* 1 (default) = stage chunks through shared memory with cp.async.bulk
                               (one elected thread per CTA); 0 = register-staged LDG/STG kernel */
  void* trace;              /* optional device uint64[n_chunks]: %globaltimer issue time of each
                               chunk (rate-bound tests); NULL = off */
} valve_copy_params;
typedef struct {
  int64_t bytes;
  int64_t pages;
  double kernel_ms;         /* CUDA-event time of the copy kernel */
  uint64_t t_first_ns;      /* %globaltimer at the first chunk issue */
  uint64_t t_last_ns;       /* %globaltimer at the last chunk's stores retired */
} valve_copy_stats;
void valve_copy_params_default(valve_copy_params* c);
/* Gathers the pages invalidated by the last apply/reclaim, in report order, into pinned
 * host memory (cudaHostAlloc'd or cudaHostRegister'd; dst_bytes >= n_pages*page_bytes).
 * Synchronous. */
int valve_pool_reclaim_copy(valve_pool* p, void* host_dst, int64_t dst_bytes,
                            const valve_copy_params* params, valve_copy_stats* stats);
/* Asynchronous form: the copy runs on the pool's copy stream, ordered after the report, and
 * works from its own device snapshot of the report, so bookkeeping calls (reserve/release/
 * grow/...) and the NEXT apply_reclaim / reclaim proceed on the pool stream while the bytes
 * cross the link (back-to-back reclaim ops keep the link busy).  fill_pages / restore wait for
 * the copy (they rewrite page bytes).  Up to VALVE_COPY_RING copies in flight; each _wait completes the
 * oldest one (FIFO) and returns its stats.  The synchronous form requires none in flight. */
#define VALVE_COPY_RING 8
int valve_pool_reclaim_copy_start(valve_pool* p, void* host_dst, int64_t dst_bytes,
                                  const valve_copy_params* params);
int valve_pool_reclaim_copy_wait(valve_pool* p, valve_copy_stats* stats);
/* Rate bound (rate_bytes_per_s, burst_bytes): a token bucket whose state lives in the pool, so it
 * bounds bytes per window ACROSS copies: in any interval of length w the pool's copies start at
 * most rate*w + burst + one chunk of bytes (back-to-back pipelined ops share one budget). */

/* Landed tickets -- when may a reclaimed slot be rewritten (SURVEY §7 hard part 2)?  Every copy
 * publishes "waves" to one monotone pool counter as it reads them out of HBM.  With a uniform
 * page size the SM kernel runs wave-major: wave w = bytes [w*wave_bytes, (w+1)*wave_bytes) of
 * EVERY page of the report, so an online tenant writing its KV layer by layer into reclaimed
 * slots waits only for the waves under the bytes it is about to write, not for the whole op.
 * (Other paths publish the copy as one wave covering the slot.)  Copy i's waves are numbered
 * wave_base .. wave_base + n_waves - 1; ticket t is out once the counter is >= t. */
int valve_pool_copy_ticket(const valve_pool* p, uint64_t* wave_base, int* n_waves, int64_t* wave_bytes);
/* Makes `stream` (NULL: the pool stream) wait (cuStreamWaitValue64 GEQ) until `ticket` waves
 * have been published.  Takes no SM. */
int valve_pool_wait_landed(valve_pool* p, uint64_t ticket, void* stream);
/* Current published count and the total issued so far (diagnostics / host polling). */
int valve_pool_landed(const valve_pool* p, uint64_t* landed, uint64_t* issued);
/* Restore (scatter) of host-resident pages into a live request's slots: host page i (of
 * n_pages, page_bytes each, pinned/mapped) is written to block blk_of_page[i] of `req` -- the
 * inverse of the gather, e.g. offline weight pages evicted to host by a reclaim (C3) and
 * re-admitted later.  Synchronous; CTA count / chunk size from params (may be NULL). */
int valve_pool_restore(valve_pool* p, int64_t req, const void* host_src, int n_pages,
                       const int* blk_of_page, const valve_copy_params* params, valve_copy_stats* stats);
/* Streams for hosts without the CUDA runtime (a C++ / cgo / JNI caller of this ABI): a
 * non-blocking stream on `device` (high_priority != 0: the device's highest priority, as the
 * online lane uses), its destruction and a host wait on it. */
int valve_stream_create(int device, int high_priority, void** out);
void valve_stream_destroy(void* stream);
int valve_stream_synchronize(void* stream);
/* Pinned, device-mapped host staging for reclaimed pages (cudaHostAlloc, mapped). */
int valve_host_alloc(int64_t bytes, void** out);
void valve_host_free(void* p);
/* Same copy through the copy engines (cudaMemcpyAsync per page) -- the baseline. */
int valve_pool_reclaim_copy_ce(valve_pool* p, void* host_dst, int64_t dst_bytes,
                               valve_copy_stats* stats);
/* Writes the deterministic image of every live offline page (request, block) into its
 * physical slot; models the offline engine having written its KV. */
int valve_pool_fill_pages(valve_pool* p);
/* Raw device pointers for kernels of the offline engine. */
typedef struct {
  void* pages;          /* slot_bytes * H * S bytes */
  int* block_tables;    /* [max_requests][max_pages_per_request] physical page ids */
  int64_t slot_bytes, page_bytes;
  int max_pages_per_request;
  int quarantine_page;
  void* stream;         /* the pool's cudaStream_t */
} valve_pool_view;
int valve_pool_view_get(const valve_pool* p, valve_pool_view* v);
/* Row of a live request in block_tables (or -1). */
int valve_pool_request_row(const valve_pool* p, int64_t req, int* row);

/* ========================================================= selection over host instances (a3,a4) */
/* reclaim.hpp:28-37.  Instance as CSR (ids, mapped_at, off, reqs); costs as sorted unique
 * keys/values (the std::map of reclaim.hpp:25).  Runs on `device`. */
int valve_select(int device, int n, const int* ids, const int64_t* mapped_at, const int* off,
                 const int64_t* reqs, int m, const int64_t* cost_keys, const int64_t* cost_vals,
                 int k, int mode, int* out, int* n_out);
int valve_evicted_cost(int device, int n, const int* ids, const int* off, const int64_t* reqs, int m,
                       const int64_t* cost_keys, const int64_t* cost_vals, const int* pick,
                       int n_pick, int64_t* cost);

/* ============================================================= reservation controller (c4) */
/* memory.hpp:103-146: fp64 control plane, host-resident by design (north star (c)). */
typedef struct {
  double alpha, beta;
  int64_t t_init_us, delta_us, t_min_us, t_max_us, window_us;
  double target_per_window;
  int h_min;
  double pressure_threshold;
} valve_resparams;
typedef struct valve_resctl valve_resctl;
void valve_resparams_default(valve_resparams* p);
int valve_resctl_create(const valve_resparams* p, valve_resctl** out);
void valve_resctl_destroy(valve_resctl* c);
int64_t valve_resctl_interval(const valve_resctl* c);
int64_t valve_resctl_pressure_events(const valve_resctl* c);
int valve_resctl_grow_target(const valve_resctl* c, int h, int cap);
void valve_resctl_record_pressure(valve_resctl* c, int64_t t);
int valve_resctl_release_due(const valve_resctl* c, int64_t t, int h);
void valve_resctl_note_tick(valve_resctl* c, int64_t t);
int64_t valve_resctl_window_tick(valve_resctl* c, int64_t t);
int64_t valve_resctl_pressure_in_window(const valve_resctl* c, int64_t t);

/* ======================================================== device preemption gate (b1, b4) */
/* An HBM gate word {generation, closed} polled by every warp of the gated offline
 * kernels at each tile boundary; quiesce is acknowledged per CTA. */
typedef struct valve_gate valve_gate;
/* In a TP group (valve_gate_attach_peers) `gen` and `quiesced_gen` are the GROUP's words and
 * live on the leader only (both fan-out modes): a member gate's copies are not written. */
typedef struct {
  uint32_t gen;            /* last generation written */
  uint32_t closed;
  uint32_t quiesced_gen;   /* last generation fully acknowledged */
  uint32_t live_ctas;
  uint64_t t_first_seen_ns;
  uint64_t t_quiesced_ns;
  uint64_t tiles_done;
  uint64_t canary_hits;    /* reads that resolved to the quarantine page */
  uint64_t tiles_claimed;  /* tiles handed out by the HBM stripe cursors (the context save) */
  uint64_t t_raise_ns;     /* %globaltimer of the last valve_gate_raise_stamped() */
  uint64_t total_tiles;    /* tiles of the current (frozen) work list */
} valve_gate_state;
int valve_gate_create(int device, valve_gate** out);
void valve_gate_destroy(valve_gate* g);
/* Stream-ordered gate store (cuStreamWriteValue) on `stream` (NULL: the gate's own
 * high-priority stream).  Takes no SM: works while offline kernels occupy every SM. */
int valve_gate_raise(valve_gate* g, uint32_t gen, void* stream);
int valve_gate_release(valve_gate* g, uint32_t gen, void* stream);
/* Diagnostic raise by a one-thread kernel that stamps %globaltimer (t_raise_ns) before the
 * release-store of the gate word; needs a free SM slot, unlike valve_gate_raise. */
int valve_gate_raise_stamped(valve_gate* g, uint32_t gen, void* stream);
/* Makes `stream` wait (cuStreamWaitValue) until every gated kernel acknowledged `gen`. */
int valve_gate_wait_quiesced(valve_gate* g, uint32_t gen, void* stream);
/* TP member side: makes `stream` wait until the group leader has closed this gate (its raise
 * reached this GPU over peer memory) and this GPU's gated CTAs have all retired -- orders a
 * member's online work and pool remaps after its own quiesce without any host round trip.  Call
 * it only inside a busy period the leader raises for (sim.cpp:362-369). */
int valve_gate_wait_closed_quiesced(valve_gate* g, void* stream);
/* TP fan-out: members' gate words are written by the leader over NVLink peer memory. */
int valve_gate_attach_peers(valve_gate* leader, valve_gate** members, int n);
/* How the leader waits for the members' acks: BATCHED (default) = one stream-memory-operation
 * submission on the waiting stream (members' counters checked in order; all members started
 * quiescing at the raise); STREAMS = one helper stream per member joined by events. */
#define VALVE_FANOUT_BATCHED 0
#define VALVE_FANOUT_STREAMS 1
int valve_gate_set_fanout(valve_gate* g, int mode);
/* One process per GPU: a member exports its gate words (CUDA IPC, 64-byte handle) and the
 * leader opens them as a remote gate (no kernels, words only) to pass to attach_peers. */
#define VALVE_GATE_HANDLE_BYTES 64
int valve_gate_export(const valve_gate* g, void* handle_out);
int valve_gate_open_remote(int device, const void* handle, valve_gate** out);
int valve_gate_read(const valve_gate* g, valve_gate_state* out);
void* valve_gate_stream(const valve_gate* g);

/* Gated offline workload (b4): a persistent, tile-looped decode-attention-shaped kernel over
 * the pool's KV pages through the block tables.  One tile = one (request, page) pair:
 * q . K over the page as bf16, fp32 accumulate.  Tiles are claimed from an HBM cursor;
 * a raised gate stops claiming at the next tile boundary and the CTA exits (context save =
 * the cursor).  Returns immediately (stream-ordered). */
typedef struct {
  const int* rows;        /* device: request rows to decode; NULL = every row of the pool */
  const int* npages;      /* device: pages per listed request (ignored when rows == NULL) */
  int n_requests;
  int64_t total_tiles;    /* informational; the kernel derives it from the tile prefix */
  float* out;             /* device: one fp32 per tile */
  int ctas;               /* 0 = 148 x resident */
  int threads;            /* 0 = 256 */
  int poll;               /* 0 = no gate polling (overhead baseline) */
  int64_t tile_bytes;     /* bytes of one tile (the quiesce granularity); 0 = 16 KiB */
} valve_offline_work;
int valve_offline_launch(valve_gate* g, valve_pool* p, const valve_offline_work* w, void* stream);
/* Resets the tile cursor / statistics (new work).  The first valve_offline_launch after a
 * reset freezes the work list (the tile prefix over the listed rows and their block counts);
 * resumed launches reuse it, so every tile of that list runs exactly once across preemptions
 * even when reclaims or re-admissions change the pool's rows meanwhile (an evicted row's
 * blocks then read as quarantine / unmapped and count as canary hits).  Resuming with another
 * rows / n_requests / tile_bytes without a reset is a VALVE_LOGIC_ERROR. */
int valve_offline_reset(valve_gate* g);
/* Drops what is left of the current work list: every queued or later resumed launch (decode pass
 * or GEMM, also one still waiting for an open gate) claims nothing and retires at once.  For
 * shutting a tenant down behind a closed gate without running its remaining tiles. */
int valve_offline_cancel(valve_gate* g);

/* Gated offline GEMM: C = A * B^T in bf16 with fp32 accumulation on the tcgen05
 * tensor cores (TMA-fed, TMEM accumulator), persistent over 128 x 256 tiles of C claimed from
 * the gate's tile cursors -- the compute-bound half of an offline decode iteration (the
 * projection GEMMs), preempted at tile granularity like valve_offline_launch.  All pointers are
 * device memory; m % 128 == 0, n % 256 == 0, k % 64 == 0, rows 16-byte aligned. */
typedef struct {
  const void* a;  /* bf16 [m, k] row-major (activations) */
  const void* b;  /* bf16 [n, k] row-major (weight, nn.Linear layout) */
  void* c;        /* bf16 [m, n] row-major */
  int m, n, k;
  int ctas;       /* 0 = one CTA per SM */
  int poll;       /* 0 = ignore the gate (overhead baseline) */
  int fresh;      /* nonzero: a new work list -- zero the tile cursors and counters on the launch
                     stream first (stream-ordered valve_offline_reset); 0: resume */
  int mode;       /* 0 auto (CTA pairs when m % 256 == 0), 1 one CTA per 128x256 tile
                     (tcgen05 cta_group::1), 2 CTA pairs: 2-CTA clusters on 256x256 tiles with
                     tcgen05.mma.cta_group::2 (M=256), each CTA holding half of A and of B */
} valve_offline_gemm_work;
int valve_offline_gemm(valve_gate* g, const valve_offline_gemm_work* w, void* stream);

/* ============================================================ channel controller (b1, b2) */
/* channel.hpp:30-80 state machine with C hooks; optionally bound to a device gate so
 * disable/enable raise/release it (valve_channel_bind_gate). */
typedef struct {
  void* user;
  void (*schedule)(void* user, int64_t when, int64_t gen, int cooldown);
  void (*on_disabled)(void* user, int64_t t);
  void (*on_enabled)(void* user, int64_t t);
  void (*log)(void* user, int64_t t, int what, int64_t aux, int memory_cause);
} valve_channel_hooks;
typedef struct valve_channel valve_channel;
int valve_channel_create(int64_t toggle_us, int64_t cooldown_us, const valve_channel_hooks* hooks,
                         valve_channel** out);
void valve_channel_destroy(valve_channel* c);
int valve_channel_bind_gate(valve_channel* c, valve_gate* g);
/* Same, with the stream the raise/release stores are issued on (e.g. the online stream, so a
 * wait_quiesced enqueued there is ordered after the raise; NULL = the gate's own stream). */
int valve_channel_bind_gate_stream(valve_channel* c, valve_gate* g, void* stream);
/* Status of the device-gate stores the state machine issued since the last call (the
 * transitions return void, as channel.hpp's do): VALVE_OK, or the first failure's code with its
 * message in valve_last_error().  Clears the status. */
int valve_channel_gate_status(valve_channel* c);
int valve_channel_state(const valve_channel* c);
int valve_channel_offline_compute_allowed(const valve_channel* c);
int64_t valve_channel_disables_issued(const valve_channel* c);
int64_t valve_channel_pending_effective(const valve_channel* c);
void valve_channel_note_busy(valve_channel* c, int64_t t);
void valve_channel_note_all_idle(valve_channel* c, int64_t t);
int64_t valve_channel_ensure_disabled(valve_channel* c, int64_t t);
void valve_channel_handle_toggle(valve_channel* c, int64_t t, int64_t gen);
void valve_channel_handle_cooldown(valve_channel* c, int64_t t, int64_t gen);

#ifdef __cplusplus
}
#endif
#endif
