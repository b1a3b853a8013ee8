/*
 * valve_oracle.h -- CPU restatement of the Valve/colosim hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
 * `bench.py --impl reference`) may load this library, and only as the checker
 * or the CPU reference arm.  The product path (paper_2604_07874_b200) never
 * links it and fails loudly if its CUDA library is missing.
 *
 * Restates, in plain C:
 *   MemoryPool             /root/reference/proj/src/memory.cpp:7-211
 *   ReservationController  /root/reference/proj/src/memory.cpp:213-255
 *   selective/fifo/oracle  /root/reference/proj/src/reclaim.cpp:19-126
 *   ChannelController      /root/reference/proj/src/channel.cpp:7-90
 * plus the two things the reference does not model and the B200 build adds:
 *   - a physical slot map (first free physical slot of the handle, ascending)
 *     next to the reference's logical slot ids (which alias, memory.cpp:82-88);
 *   - the block index of every page inside its request (allocation order), so
 *     reclaimed byte images can be predicted from (request, block).
 * Parity of the restatement itself is pinned against the reference compiled
 * from /root/reference (oracle/_ref, see oracle/Makefile) and against the
 * reference's own known-answer tests (tests/test_oracle_*.py).
 *
 * Status codes match include/valve_cuda.h.
 */
#ifndef VALVE_ORACLE_H
#define VALVE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VO_OK = 0,
  VO_INVALID_ARGUMENT = 1,
  VO_LOGIC_ERROR = 2,
  VO_RUNTIME_ERROR = 3,
  VO_CUDA_ERROR = 4,
  VO_OUT_OF_RANGE = 5,
};

const char* vo_last_error(void);

typedef struct vo_pool vo_pool;

int vo_pool_create(int total_handles, int handle_size_pages, int page_size_tokens, vo_pool** out);
void vo_pool_destroy(vo_pool* p);
/* out[0..4] = free, online, offline handles, online_used_pages, online_capacity_pages */
int vo_pool_counts(const vo_pool* p, int64_t out[5]);
int vo_pool_online_grow(vo_pool* p, int k, int64_t t);
int vo_pool_online_release(vo_pool* p, int k, int* released);
int vo_pool_online_use_pages(vo_pool* p, int64_t n);
int vo_pool_online_free_pages(vo_pool* p, int64_t n);
int vo_pool_offline_reserve(vo_pool* p, int64_t req, int pages, int64_t t, int max_offline_handles,
                            int* ok);
int vo_pool_offline_release(vo_pool* p, int64_t req);
int vo_pool_requests_on_handle(const vo_pool* p, int handle, int64_t* out, int cap, int* n);
int vo_pool_handles_of_request(const vo_pool* p, int64_t req, int* out, int cap, int* n);
int vo_pool_offline_pages_of(const vo_pool* p, int64_t req, int* out);
/* Snapshot as CSR: ids[nh], mapped_at[nh], off[nh+1], reqs[off[nh]].  Pass NULL
 * buffers to query sizes (nh, nr). */
int vo_pool_snapshot(const vo_pool* p, int* ids, int64_t* mapped_at, int* off, int64_t* reqs,
                     int cap_h, int cap_r, int* nh, int* nr);
/* apply_reclaim.  Outputs: handles[n_handles] (the converted prefix), evicted[n_evicted] sorted,
 * inv_off[n_evicted+1], inv_pages[] (logical page ids, sorted per request), inv_phys[] and
 * inv_blk[] aligned with inv_pages (physical page id, block index inside the request). */
int vo_pool_apply_reclaim(vo_pool* p, const int* ids, int k, int64_t t, int* handles, int* n_handles,
                          int64_t* evicted, int* n_evicted, int* inv_off, int64_t* inv_pages,
                          int* inv_phys, int* inv_blk, int cap_ev, int cap_pages, int* n_pages);
int vo_pool_handle_state(const vo_pool* p, int handle, int* state);
int vo_pool_handle_mapped_at(const vo_pool* p, int handle, int64_t* t);
int vo_pool_check_invariants(const vo_pool* p);
/* Physical page ids of a request in block order (block table). */
int vo_pool_block_table(const vo_pool* p, int64_t req, int* out, int cap, int* n);

/* Selection over an instance given as CSR (reclaim.hpp:12-26).  costs: sorted
 * unique keys.  mode 0 = selective (Algorithm 1), 1 = fifo, 2 = exhaustive oracle. */
int vo_select(int n, const int* ids, const int64_t* mapped_at, const int* off, const int64_t* reqs,
              int m, const int64_t* cost_keys, const int64_t* cost_vals, int k, int mode, int* out,
              int* n_out);
int vo_evicted_cost(int n, const int* ids, const int* off, const int64_t* reqs, int m,
                    const int64_t* cost_keys, const int64_t* cost_vals, const int* pick, int n_pick,
                    int64_t* cost);

/* ReservationController (memory.hpp:103-146). */
typedef struct vo_resctl vo_resctl;
typedef struct {
  double alpha, beta;
  int64_t t_init_us, delta_us, t_min_us, t_max_us, window_us;
  double target_per_window;
  int h_min;
  double pressure_threshold;
} vo_resparams;
void vo_resparams_default(vo_resparams* p);
int vo_resctl_create(const vo_resparams* p, vo_resctl** out);
void vo_resctl_destroy(vo_resctl* c);
int64_t vo_resctl_interval(const vo_resctl* c);
int64_t vo_resctl_pressure_events(const vo_resctl* c);
int vo_resctl_grow_target(const vo_resctl* c, int h, int cap);
void vo_resctl_record_pressure(vo_resctl* c, int64_t t);
int vo_resctl_release_due(const vo_resctl* c, int64_t t, int h);
void vo_resctl_note_tick(vo_resctl* c, int64_t t);
int64_t vo_resctl_window_tick(vo_resctl* c, int64_t t);
int64_t vo_resctl_pressure_in_window(const vo_resctl* c, int64_t t);

/* ChannelController (channel.hpp:30-80) with C function-pointer hooks. */
typedef struct {
  void* user;
  void (*schedule)(void* user, int64_t when, int64_t gen, int cooldown);
  void (*on_disabled)(void* user, int64_t t);
  void (*on_enabled)(void* user, int64_t t);
  void (*log)(void* user, int64_t t, int what, int64_t aux, int memory_cause);
} vo_channel_hooks;
typedef struct vo_channel vo_channel;
int vo_channel_create(int64_t toggle_us, int64_t cooldown_us, const vo_channel_hooks* hooks,
                      vo_channel** out);
void vo_channel_destroy(vo_channel* c);
int vo_channel_state(const vo_channel* c);
int vo_channel_offline_compute_allowed(const vo_channel* c);
int64_t vo_channel_disables_issued(const vo_channel* c);
int64_t vo_channel_pending_effective(const vo_channel* c);
void vo_channel_note_busy(vo_channel* c, int64_t t);
void vo_channel_note_all_idle(vo_channel* c, int64_t t);
int64_t vo_channel_ensure_disabled(vo_channel* c, int64_t t);
void vo_channel_handle_toggle(vo_channel* c, int64_t t, int64_t gen);
void vo_channel_handle_cooldown(vo_channel* c, int64_t t, int64_t gen);

/* Deterministic page contents (u64 words) used for byte-image parity:
 * word w of block b of request r = splitmix64(splitmix64(r ^ K1) ^ (b * K2) ^ w). */
uint64_t vo_page_word(int64_t req, int32_t blk, int64_t word);
/* Fills dst[n_pages * page_bytes] with the images of (reqs[i], blks[i]). */
void vo_gather_images(const int64_t* reqs, const int32_t* blks, int n_pages, int64_t page_bytes,
                      uint8_t* dst);
/* Host memcpy gather restatement (the CPU baseline of the copy leg): copies
 * page_bytes from src + phys[i]*slot_bytes to dst + i*page_bytes, with nthreads. */
void vo_gather_memcpy(const uint8_t* src, int64_t slot_bytes, int64_t page_bytes, const int* phys,
                      int n_pages, uint8_t* dst, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
