/*
 * valve_oracle.c -- CPU restatement of the colosim hot path (TEST INFRASTRUCTURE ONLY;
 * see valve_oracle.h for who may load it).
 *
 * Data layout mirrors the device pool on purpose so the two can be compared
 * slot by slot, but every rule below follows the reference line by line:
 *   handle sets free_/online_/offline_ (memory.hpp:94-96)  -> state[] scanned in id order
 *   Handle::slots_by_req + used_slots (memory.hpp:81-86)   -> per-physical-slot (req, lid, blk)
 */
#include "valve_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* vo_last_error(void) { return g_err; }

enum { ST_FREE = 0, ST_ONLINE = 1, ST_OFFLINE = 2 };

struct vo_pool {
  int H, S, T;
  uint8_t* state;
  int64_t* mapped;
  int* used;        /* reference used_slots: count of the handle's offline slots */
  int64_t* slot_req;  /* physical slot -> owning request, or -1 */
  int* slot_lid;    /* logical slot id the reference reports (memory.cpp:82-88) */
  int* slot_blk;    /* block index inside the owning request */
  int64_t online_used;
  /* per-request next block index (append order), kept in a tiny open table */
  int64_t* rq_key;
  int* rq_next;
  int rq_n, rq_cap;
  /* blocks remapped to the quarantine page while their request stays live (only after an
   * apply_reclaim that stopped at a bad handle: the residual release never ran) */
  int64_t* qr_req;
  int* qr_blk;
  int qr_n, qr_cap;
};

/* A slot is live iff it carries a block index (request ids may be any int64, -1 included). */
#define LIVE(p, i) ((p)->slot_blk[i] != -1)
#define HOLDS(p, i, req) (LIVE(p, i) && (p)->slot_req[i] == (req))

static int count_state(const vo_pool* p, int st) {
  int n = 0;
  for (int i = 0; i < p->H; ++i) n += p->state[i] == st;
  return n;
}

int vo_pool_create(int H, int S, int T, vo_pool** out) {
  /* memory.cpp:7-16 */
  if (H <= 0 || S <= 0 || T <= 0) return fail(VO_INVALID_ARGUMENT, "MemoryPool: sizes must be > 0");
  vo_pool* p = (vo_pool*)calloc(1, sizeof *p);
  p->H = H;
  p->S = S;
  p->T = T;
  p->state = (uint8_t*)calloc((size_t)H, 1);
  p->mapped = (int64_t*)calloc((size_t)H, 8);
  p->used = (int*)calloc((size_t)H, sizeof(int));
  size_t ns = (size_t)H * (size_t)S;
  p->slot_req = (int64_t*)malloc(ns * 8);
  p->slot_lid = (int*)malloc(ns * sizeof(int));
  p->slot_blk = (int*)malloc(ns * sizeof(int));
  for (size_t i = 0; i < ns; ++i) {
    p->slot_req[i] = -1;
    p->slot_lid[i] = -1;
    p->slot_blk[i] = -1;
  }
  p->rq_cap = 64;
  p->rq_key = (int64_t*)malloc((size_t)p->rq_cap * 8);
  p->rq_next = (int*)malloc((size_t)p->rq_cap * sizeof(int));
  *out = p;
  return VO_OK;
}

void vo_pool_destroy(vo_pool* p) {
  if (!p) return;
  free(p->state);
  free(p->mapped);
  free(p->used);
  free(p->slot_req);
  free(p->slot_lid);
  free(p->slot_blk);
  free(p->rq_key);
  free(p->rq_next);
  free(p->qr_req);
  free(p->qr_blk);
  free(p);
}

static void qr_add(vo_pool* p, int64_t req, int blk) {
  if (p->qr_n == p->qr_cap) {
    p->qr_cap = p->qr_cap ? 2 * p->qr_cap : 16;
    p->qr_req = (int64_t*)realloc(p->qr_req, (size_t)p->qr_cap * 8);
    p->qr_blk = (int*)realloc(p->qr_blk, (size_t)p->qr_cap * sizeof(int));
  }
  p->qr_req[p->qr_n] = req;
  p->qr_blk[p->qr_n] = blk;
  ++p->qr_n;
}

static void qr_drop(vo_pool* p, int64_t req) {
  int w = 0;
  for (int i = 0; i < p->qr_n; ++i)
    if (p->qr_req[i] != req) {
      p->qr_req[w] = p->qr_req[i];
      p->qr_blk[w] = p->qr_blk[i];
      ++w;
    }
  p->qr_n = w;
}

int vo_pool_counts(const vo_pool* p, int64_t out[5]) {
  out[0] = count_state(p, ST_FREE);
  out[1] = count_state(p, ST_ONLINE);
  out[2] = count_state(p, ST_OFFLINE);
  out[3] = p->online_used;
  out[4] = out[1] * (int64_t)p->S; /* memory.hpp:39-41 */
  return VO_OK;
}

/* memory.cpp:20-29 take_lowest_free */
static int take_lowest_free(vo_pool* p, int to, int64_t t) {
  for (int i = 0; i < p->H; ++i)
    if (p->state[i] == ST_FREE) {
      p->state[i] = (uint8_t)to;
      p->mapped[i] = t;
      return i;
    }
  return -1;
}

int vo_pool_online_grow(vo_pool* p, int k, int64_t t) {
  /* memory.cpp:31-35 */
  if (k < 0) return fail(VO_INVALID_ARGUMENT, "online_grow: k must be >= 0");
  if (k > count_state(p, ST_FREE)) return fail(VO_LOGIC_ERROR, "online_grow: k exceeds free handles");
  for (int i = 0; i < k; ++i) take_lowest_free(p, ST_ONLINE, t);
  return VO_OK;
}

int vo_pool_online_release(vo_pool* p, int k, int* released) {
  /* memory.cpp:37-51: release the lowest-id online handles while the remaining
   * capacity still covers the used pages. */
  if (k < 0) return fail(VO_INVALID_ARGUMENT, "online_release: k must be >= 0");
  int n_on = count_state(p, ST_ONLINE), rel = 0;
  for (int i = 0; i < p->H && rel < k && n_on > 0; ++i) {
    if (p->state[i] != ST_ONLINE) continue;
    int64_t cap_after = (int64_t)(n_on - 1) * p->S;
    if (cap_after < p->online_used) break;
    p->state[i] = ST_FREE;
    --n_on;
    ++rel;
  }
  *released = rel;
  return VO_OK;
}

int vo_pool_online_use_pages(vo_pool* p, int64_t n) {
  /* memory.cpp:53-58 */
  if (n < 0) return fail(VO_INVALID_ARGUMENT, "online_use_pages: n must be >= 0");
  if (p->online_used + n > (int64_t)count_state(p, ST_ONLINE) * p->S)
    return fail(VO_LOGIC_ERROR, "online_use_pages: overcommit beyond reserved capacity");
  p->online_used += n;
  return VO_OK;
}

int vo_pool_online_free_pages(vo_pool* p, int64_t n) {
  /* memory.cpp:60-64 */
  if (n < 0 || n > p->online_used) return fail(VO_LOGIC_ERROR, "online_free_pages: bad page count");
  p->online_used -= n;
  return VO_OK;
}

static int rq_find(const vo_pool* p, int64_t req) {
  for (int i = 0; i < p->rq_n; ++i)
    if (p->rq_key[i] == req) return i;
  return -1;
}
static int rq_next_blk(vo_pool* p, int64_t req) {
  int i = rq_find(p, req);
  if (i < 0) {
    if (p->rq_n == p->rq_cap) {
      p->rq_cap *= 2;
      p->rq_key = (int64_t*)realloc(p->rq_key, (size_t)p->rq_cap * 8);
      p->rq_next = (int*)realloc(p->rq_next, (size_t)p->rq_cap * sizeof(int));
    }
    i = p->rq_n++;
    p->rq_key[i] = req;
    p->rq_next[i] = 0;
  }
  return p->rq_next[i]++;
}
static void rq_drop(vo_pool* p, int64_t req) {
  int i = rq_find(p, req);
  if (i < 0) return;
  p->rq_key[i] = p->rq_key[p->rq_n - 1];
  p->rq_next[i] = p->rq_next[p->rq_n - 1];
  --p->rq_n;
}

/* One fill() step of memory.cpp:76-86 on handle h: ascending logical ids from
 * the current fill level; physical slots are the lowest free ones. */
static void fill_handle(vo_pool* p, int h, int64_t req, int* remaining) {
  int64_t base = (int64_t)h * p->S;
  for (int s = 0; s < p->S && *remaining > 0 && p->used[h] < p->S; ++s) {
    if (LIVE(p, base + s)) continue;
    p->slot_req[base + s] = req;
    p->slot_lid[base + s] = p->used[h]++;
    p->slot_blk[base + s] = rq_next_blk(p, req);
    --*remaining;
  }
}

int vo_pool_offline_reserve(vo_pool* p, int64_t req, int pages, int64_t t, int max_off, int* ok) {
  /* memory.cpp:66-97 */
  if (pages < 0) return fail(VO_INVALID_ARGUMENT, "offline_reserve: pages must be >= 0");
  *ok = 1;
  if (pages == 0) return VO_OK;
  int64_t avail = 0;
  int n_off = 0, n_free = 0;
  for (int i = 0; i < p->H; ++i) {
    if (p->state[i] == ST_OFFLINE) {
      avail += p->S - p->used[i];
      ++n_off;
    } else if (p->state[i] == ST_FREE) {
      ++n_free;
    }
  }
  int mappable = n_free;
  if (max_off >= 0) {
    int room = max_off - n_off;
    if (room < 0) room = 0;
    if (room < mappable) mappable = room;
  }
  avail += (int64_t)mappable * p->S;
  if (avail < pages) {
    *ok = 0;
    return VO_OK;
  }
  int remaining = pages;
  for (int i = 0; i < p->H && remaining > 0; ++i)
    if (p->state[i] == ST_OFFLINE) fill_handle(p, i, req, &remaining);
  while (remaining > 0) fill_handle(p, take_lowest_free(p, ST_OFFLINE, t), req, &remaining);
  return VO_OK;
}

static void release_req(vo_pool* p, int64_t req) {
  /* memory.cpp:99-114: drop the request's slots; emptied handles go free. */
  for (int h = 0; h < p->H; ++h) {
    if (p->state[h] != ST_OFFLINE) continue;
    int64_t base = (int64_t)h * p->S;
    int dropped = 0;
    for (int s = 0; s < p->S; ++s)
      if (HOLDS(p, base + s, req)) {
        p->slot_req[base + s] = -1;
        p->slot_lid[base + s] = -1;
        p->slot_blk[base + s] = -1;
        ++dropped;
      }
    if (!dropped) continue;
    p->used[h] -= dropped;
    if (p->used[h] == 0) p->state[h] = ST_FREE;
  }
  rq_drop(p, req);
  qr_drop(p, req);
}

int vo_pool_offline_release(vo_pool* p, int64_t req) {
  release_req(p, req);
  return VO_OK;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* sorted distinct residents of handle h -> buf; returns count */
static int residents(const vo_pool* p, int h, int64_t* buf) {
  int n = 0;
  int64_t base = (int64_t)h * p->S;
  for (int s = 0; s < p->S; ++s)
    if (LIVE(p, base + s)) buf[n++] = p->slot_req[base + s];
  qsort(buf, (size_t)n, 8, cmp_i64);
  int u = 0;
  for (int i = 0; i < n; ++i)
    if (u == 0 || buf[u - 1] != buf[i]) buf[u++] = buf[i];
  return u;
}

int vo_pool_requests_on_handle(const vo_pool* p, int h, int64_t* out, int cap, int* n) {
  /* memory.cpp:116-122 (handles_.at -> out_of_range) */
  if (h < 0 || h >= p->H) return fail(VO_OUT_OF_RANGE, "requests_on_handle: handle out of range");
  int64_t* buf = (int64_t*)malloc((size_t)p->S * 8);
  int u = residents(p, h, buf);
  *n = u;
  for (int i = 0; i < u && i < cap; ++i) out[i] = buf[i];
  free(buf);
  return VO_OK;
}

int vo_pool_handles_of_request(const vo_pool* p, int64_t req, int* out, int cap, int* n) {
  /* memory.cpp:124-130 */
  int c = 0;
  for (int h = 0; h < p->H; ++h) {
    if (p->state[h] != ST_OFFLINE) continue;
    int64_t base = (int64_t)h * p->S;
    for (int s = 0; s < p->S; ++s)
      if (HOLDS(p, base + s, req)) {
        if (c < cap) out[c] = h;
        ++c;
        break;
      }
  }
  *n = c;
  return VO_OK;
}

int vo_pool_offline_pages_of(const vo_pool* p, int64_t req, int* out) {
  /* memory.cpp:132-140 */
  int c = 0;
  for (int h = 0; h < p->H; ++h) {
    if (p->state[h] != ST_OFFLINE) continue;
    int64_t base = (int64_t)h * p->S;
    for (int s = 0; s < p->S; ++s) c += HOLDS(p, base + s, req);
  }
  *out = c;
  return VO_OK;
}

int vo_pool_snapshot(const vo_pool* p, int* ids, int64_t* mapped, int* off, int64_t* reqs, int cap_h,
                     int cap_r, int* nh, int* nr) {
  /* memory.cpp:142-153: offline handles ascending, residents ascending */
  int64_t* buf = (int64_t*)malloc((size_t)p->S * 8);
  int h_n = 0, r_n = 0;
  if (off && cap_h >= 0) off[0] = 0;
  for (int h = 0; h < p->H; ++h) {
    if (p->state[h] != ST_OFFLINE) continue;
    int u = residents(p, h, buf);
    if (ids && h_n < cap_h) {
      ids[h_n] = h;
      mapped[h_n] = p->mapped[h];
    }
    for (int i = 0; i < u; ++i) {
      if (reqs && r_n < cap_r) reqs[r_n] = buf[i];
      ++r_n;
    }
    ++h_n;
    if (off && h_n <= cap_h) off[h_n] = r_n;
  }
  free(buf);
  *nh = h_n;
  *nr = r_n;
  return VO_OK;
}

typedef struct {
  int64_t req, page;
  int phys, blk;
} inv_t;
static int cmp_inv(const void* a, const void* b) {
  const inv_t* x = (const inv_t*)a;
  const inv_t* y = (const inv_t*)b;
  if (x->req != y->req) return (x->req > y->req) - (x->req < y->req);
  if (x->page != y->page) return (x->page > y->page) - (x->page < y->page);
  return (x->phys > y->phys) - (x->phys < y->phys);
}

int vo_pool_apply_reclaim(vo_pool* p, const int* ids, int k, int64_t t, int* handles, int* n_handles,
                          int64_t* evicted, int* n_evicted, int* inv_off, int64_t* inv_pages,
                          int* inv_phys, int* inv_blk, int cap_ev, int cap_pages, int* n_pages) {
  /* memory.cpp:155-180.  Handles convert in the given order; a bad handle throws
   * after the earlier ones converted (the reference mutates as it goes), and the
   * residual release of line 176 never runs in that case. */
  inv_t* inv = (inv_t*)malloc(((size_t)k * p->S + 1) * sizeof(inv_t));
  int ni = 0, nh = 0, code = VO_OK;
  for (int i = 0; i < k; ++i) {
    int h = ids[i];
    if (h < 0 || h >= p->H) {
      code = fail(VO_OUT_OF_RANGE, "apply_reclaim: handle out of range");
      break;
    }
    if (p->state[h] != ST_OFFLINE) {
      char msg[128];
      snprintf(msg, sizeof msg, "apply_reclaim: handle %d is not offline-mapped", h);
      code = fail(VO_LOGIC_ERROR, msg);
      break;
    }
    int64_t base = (int64_t)h * p->S;
    for (int s = 0; s < p->S; ++s) {
      if (!LIVE(p, base + s)) continue;
      inv[ni].req = p->slot_req[base + s];
      inv[ni].page = base + p->slot_lid[base + s];
      inv[ni].phys = (int)(base + s);
      inv[ni].blk = p->slot_blk[base + s];
      qr_add(p, inv[ni].req, inv[ni].blk);
      ++ni;
      p->slot_req[base + s] = -1;
      p->slot_lid[base + s] = -1;
      p->slot_blk[base + s] = -1;
    }
    p->used[h] = 0;
    p->state[h] = ST_ONLINE;
    p->mapped[h] = t;
    if (handles) handles[nh] = h;
    ++nh;
  }
  *n_handles = nh;
  qsort(inv, (size_t)ni, sizeof(inv_t), cmp_inv);
  int ne = 0;
  for (int i = 0; i < ni; ++i) {
    if (ne == 0 || inv[i].req != evicted[ne - 1]) {
      if (ne >= cap_ev) {
        free(inv);
        return fail(VO_RUNTIME_ERROR, "apply_reclaim: evicted capacity too small");
      }
      evicted[ne] = inv[i].req;
      inv_off[ne] = i;
      ++ne;
    }
    if (i < cap_pages) {
      inv_pages[i] = inv[i].page;
      inv_phys[i] = inv[i].phys;
      inv_blk[i] = inv[i].blk;
    }
  }
  inv_off[ne] = ni;
  *n_evicted = ne;
  *n_pages = ni;
  if (code == VO_OK)
    for (int i = 0; i < ne; ++i) release_req(p, evicted[i]); /* memory.cpp:176 */
  free(inv);
  return code;
}

int vo_pool_handle_state(const vo_pool* p, int h, int* st) {
  if (h < 0 || h >= p->H) return fail(VO_OUT_OF_RANGE, "handle_state: handle out of range");
  *st = p->state[h];
  return VO_OK;
}
int vo_pool_handle_mapped_at(const vo_pool* p, int h, int64_t* t) {
  if (h < 0 || h >= p->H) return fail(VO_OUT_OF_RANGE, "handle_mapped_at: handle out of range");
  *t = p->mapped[h];
  return VO_OK;
}

int vo_pool_check_invariants(const vo_pool* p) {
  /* memory.cpp:190-211 restated on the slot layout */
  int64_t cap = (int64_t)count_state(p, ST_ONLINE) * p->S;
  if (p->online_used < 0 || p->online_used > cap)
    return fail(VO_LOGIC_ERROR, "MemoryPool: online page accounting out of bounds");
  for (int h = 0; h < p->H; ++h) {
    int slots = 0;
    for (int s = 0; s < p->S; ++s) slots += LIVE(p, (int64_t)h * p->S + s);
    if (slots != p->used[h] || p->used[h] > p->S)
      return fail(VO_LOGIC_ERROR, "MemoryPool: slot accounting mismatch");
    if (p->state[h] != ST_OFFLINE && p->used[h] != 0)
      return fail(VO_LOGIC_ERROR, "MemoryPool: non-offline handle holds offline pages");
  }
  return VO_OK;
}

int vo_pool_block_table(const vo_pool* p, int64_t req, int* out, int cap, int* n) {
  /* blocks 0..nblk-1: the physical page, or the quarantine page H*S once remapped */
  int c = 0;
  int64_t ns = (int64_t)p->H * p->S;
  for (int64_t i = 0; i < ns; ++i)
    if (HOLDS(p, i, req)) {
      int b = p->slot_blk[i];
      if (b < cap) out[b] = (int)i;
      if (b + 1 > c) c = b + 1;
    }
  for (int i = 0; i < p->qr_n; ++i)
    if (p->qr_req[i] == req) {
      int b = p->qr_blk[i];
      if (b < cap) out[b] = (int)ns;
      if (b + 1 > c) c = b + 1;
    }
  *n = c;
  return VO_OK;
}

/* ---------------------------------------------------------------- selection */

static int cost_index(int m, const int64_t* keys, int64_t req) {
  int lo = 0, hi = m - 1;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (keys[mid] == req) return mid;
    if (keys[mid] < req) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

static int all_costs_present(int n, const int* off, const int64_t* reqs, int m, const int64_t* keys) {
  for (int i = 0; i < off[n]; ++i)
    if (cost_index(m, keys, reqs[i]) < 0) return 0;
  return 1;
}

int vo_evicted_cost(int n, const int* ids, const int* off, const int64_t* reqs, int m,
                    const int64_t* keys, const int64_t* vals, const int* pick, int n_pick,
                    int64_t* cost) {
  /* reclaim.cpp:19-31 */
  char* ev = (char*)calloc((size_t)m + 1, 1);
  int64_t total = 0;
  for (int j = 0; j < n_pick; ++j) {
    int hi = -1;
    for (int i = 0; i < n; ++i)
      if (ids[i] == pick[j]) {
        hi = i;
        break;
      }
    if (hi < 0) {
      free(ev);
      return fail(VO_INVALID_ARGUMENT, "evicted_cost: unknown handle id");
    }
    for (int e = off[hi]; e < off[hi + 1]; ++e) {
      int c = cost_index(m, keys, reqs[e]);
      if (c >= 0 && ev[c]) continue;
      if (c < 0) {
        free(ev);
        return fail(VO_INVALID_ARGUMENT, "reclaim: request without cost entry");
      }
      ev[c] = 1;
      total += vals[c];
    }
  }
  free(ev);
  *cost = total;
  return VO_OK;
}

static int select_greedy(int n, const int* ids, const int* off, const int64_t* reqs, int m,
                         const int64_t* keys, const int64_t* vals, int k, int* out) {
  /* reclaim.cpp:33-67: k rounds of argmin marginal cost, ties to the smallest id */
  if (k > 0 && !all_costs_present(n, off, reqs, m, keys))
    return fail(VO_INVALID_ARGUMENT, "reclaim: request without cost entry");
  char* ev = (char*)calloc((size_t)m + 1, 1);
  char* taken = (char*)calloc((size_t)n + 1, 1);
  for (int round = 0; round < k; ++round) {
    int best = -1;
    int64_t best_cost = 0;
    for (int i = 0; i < n; ++i) {
      if (taken[i]) continue;
      int64_t marginal = 0;
      for (int e = off[i]; e < off[i + 1]; ++e) {
        int c = cost_index(m, keys, reqs[e]);
        if (!ev[c]) marginal += vals[c];
      }
      if (best < 0 || marginal < best_cost || (marginal == best_cost && ids[i] < ids[best])) {
        best = i;
        best_cost = marginal;
      }
    }
    out[round] = ids[best];
    taken[best] = 1;
    for (int e = off[best]; e < off[best + 1]; ++e) ev[cost_index(m, keys, reqs[e])] = 1;
  }
  free(ev);
  free(taken);
  return VO_OK;
}

static const int64_t* g_sort_mapped;
static const int* g_sort_ids;
static int cmp_fifo(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  if (g_sort_mapped[x] != g_sort_mapped[y]) return g_sort_mapped[x] < g_sort_mapped[y] ? -1 : 1;
  if (g_sort_ids[x] != g_sort_ids[y]) return g_sort_ids[x] < g_sort_ids[y] ? -1 : 1;
  return (x > y) - (x < y);
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

static int select_oracle(int n, const int* ids, const int* off, const int64_t* reqs, int m,
                         const int64_t* keys, const int64_t* vals, int k, int* out) {
  /* reclaim.cpp:85-126: lexicographic k-subset walk over sorted ids, first minimum wins */
  if (n > 20) return fail(VO_INVALID_ARGUMENT, "oracle_reclaim: instance too large (> 20 handles)");
  if (k == 0) return VO_OK;
  if (!all_costs_present(n, off, reqs, m, keys))
    return fail(VO_INVALID_ARGUMENT, "reclaim: request without cost entry");
  int* sorted = (int*)malloc((size_t)n * sizeof(int));
  memcpy(sorted, ids, (size_t)n * sizeof(int));
  qsort(sorted, (size_t)n, sizeof(int), cmp_int);
  int* pos = (int*)malloc((size_t)k * sizeof(int));
  int* pick = (int*)malloc((size_t)k * sizeof(int));
  int have = 0;
  int64_t best = 0;
  for (int i = 0; i < k; ++i) pos[i] = i;
  for (;;) {
    for (int i = 0; i < k; ++i) pick[i] = sorted[pos[i]];
    int64_t c = 0;
    vo_evicted_cost(n, ids, off, reqs, m, keys, vals, pick, k, &c);
    if (!have || c < best) {
      have = 1;
      best = c;
      memcpy(out, pick, (size_t)k * sizeof(int));
    }
    int i = k - 1;
    while (i >= 0 && pos[i] == n - k + i) --i;
    if (i < 0) break;
    ++pos[i];
    for (int j = i + 1; j < k; ++j) pos[j] = pos[j - 1] + 1;
  }
  free(sorted);
  free(pos);
  free(pick);
  return VO_OK;
}

int vo_select(int n, const int* ids, const int64_t* mapped, const int* off, const int64_t* reqs, int m,
              const int64_t* keys, const int64_t* vals, int k, int mode, int* out, int* n_out) {
  const char* who = mode == 0 ? "selective_reclaim" : mode == 1 ? "fifo_reclaim" : "oracle_reclaim";
  if (k < 0) {
    char msg[96];
    snprintf(msg, sizeof msg, "%s: k must be >= 0", who);
    return fail(VO_INVALID_ARGUMENT, msg);
  }
  if (mode == 2 && n > 20)
    return fail(VO_INVALID_ARGUMENT, "oracle_reclaim: instance too large (> 20 handles)");
  if (k > n) k = n;
  *n_out = k;
  if (mode == 0) return select_greedy(n, ids, off, reqs, m, keys, vals, k, out);
  if (mode == 2) return select_oracle(n, ids, off, reqs, m, keys, vals, k, out);
  /* reclaim.cpp:69-83 fifo: (mapped_at, id) ascending */
  int* order = (int*)malloc(((size_t)n + 1) * sizeof(int));
  for (int i = 0; i < n; ++i) order[i] = i;
  g_sort_mapped = mapped;
  g_sort_ids = ids;
  qsort(order, (size_t)n, sizeof(int), cmp_fifo);
  for (int i = 0; i < k; ++i) out[i] = ids[order[i]];
  free(order);
  return VO_OK;
}

/* -------------------------------------------------------- reservation ctl */

struct vo_resctl {
  vo_resparams p;
  int64_t t, last_tick;
  int64_t* pt;
  int64_t npt, cap;
};

void vo_resparams_default(vo_resparams* p) {
  /* memory.hpp:103-114 */
  p->alpha = 1.5;
  p->beta = 2.0;
  p->t_init_us = 1000000;
  p->delta_us = 100000;
  p->t_min_us = 100000;
  p->t_max_us = 60000000;
  p->window_us = 60000000;
  p->target_per_window = 1.0;
  p->h_min = 1;
  p->pressure_threshold = 0.9;
}

int vo_resctl_create(const vo_resparams* p, vo_resctl** out) {
  /* memory.cpp:213-218 */
  if (p->alpha <= 1.0 || p->beta <= 1.0)
    return fail(VO_INVALID_ARGUMENT, "ReservationParams: alpha/beta must be > 1");
  if (p->t_init_us <= 0 || p->t_min_us <= 0 || p->t_max_us < p->t_min_us || p->window_us <= 0)
    return fail(VO_INVALID_ARGUMENT, "ReservationParams: bad interval bounds");
  if (p->h_min < 0) return fail(VO_INVALID_ARGUMENT, "ReservationParams: h_min must be >= 0");
  vo_resctl* c = (vo_resctl*)calloc(1, sizeof *c);
  c->p = *p;
  c->t = p->t_init_us;
  c->cap = 16;
  c->pt = (int64_t*)malloc((size_t)c->cap * 8);
  *out = c;
  return VO_OK;
}
void vo_resctl_destroy(vo_resctl* c) {
  if (!c) return;
  free(c->pt);
  free(c);
}
int64_t vo_resctl_interval(const vo_resctl* c) { return c->t; }
int64_t vo_resctl_pressure_events(const vo_resctl* c) { return c->npt; }

int vo_resctl_grow_target(const vo_resctl* c, int h, int cap) {
  /* memory.cpp:220-223: min(max(ceil(alpha*h), h, 1), cap) in IEEE double */
  int m = (int)ceil(c->p.alpha * (double)h);
  if (h > m) m = h;
  if (1 > m) m = 1;
  return m < cap ? m : cap;
}

void vo_resctl_record_pressure(vo_resctl* c, int64_t t) {
  if (c->npt == c->cap) {
    c->cap *= 2;
    c->pt = (int64_t*)realloc(c->pt, (size_t)c->cap * 8);
  }
  c->pt[c->npt++] = t;
}

int vo_resctl_release_due(const vo_resctl* c, int64_t t, int h) {
  /* memory.cpp:227-234 */
  if (h <= c->p.h_min) return 0;
  for (int64_t i = c->npt - 1; i >= 0; --i) {
    if (c->pt[i] <= c->last_tick) break;
    if (c->pt[i] <= t) return 0;
  }
  return 1;
}
void vo_resctl_note_tick(vo_resctl* c, int64_t t) { c->last_tick = t; }

int64_t vo_resctl_pressure_in_window(const vo_resctl* c, int64_t t) {
  /* memory.cpp:248-255 */
  int64_t n = 0;
  for (int64_t i = c->npt - 1; i >= 0; --i) {
    if (c->pt[i] <= t - c->p.window_us) break;
    if (c->pt[i] <= t) ++n;
  }
  return n;
}

int64_t vo_resctl_window_tick(vo_resctl* c, int64_t t) {
  /* memory.cpp:238-246 */
  double rate = (double)vo_resctl_pressure_in_window(c, t);
  if (rate > c->p.target_per_window) {
    int64_t grown = (int64_t)((double)c->t * c->p.beta);
    c->t = grown < c->p.t_max_us ? grown : c->p.t_max_us;
  } else {
    int64_t shrunk = c->t - c->p.delta_us;
    c->t = shrunk > c->p.t_min_us ? shrunk : c->p.t_min_us;
  }
  return c->t;
}

/* ------------------------------------------------------------ channel ctl */

enum { CH_ENABLED = 0, CH_DISABLING = 1, CH_DISABLED = 2, CH_ENABLING = 3 };
enum { LOG_DISABLE_ISSUED = 0, LOG_DISABLED, LOG_ENABLE_ISSUED, LOG_ENABLED, LOG_CD_SCHED, LOG_CD_CANCEL };

struct vo_channel {
  int64_t toggle, cooldown;
  vo_channel_hooks h;
  int state, any_busy, enable_after_disable, cooldown_pending;
  int64_t gen, cooldown_gen, effective_at, disables;
};

int vo_channel_create(int64_t toggle, int64_t cooldown, const vo_channel_hooks* hooks,
                      vo_channel** out) {
  /* channel.cpp:7-11 */
  if (toggle < 0 || cooldown < 0)
    return fail(VO_INVALID_ARGUMENT, "ChannelController: latencies must be >= 0");
  vo_channel* c = (vo_channel*)calloc(1, sizeof *c);
  c->toggle = toggle;
  c->cooldown = cooldown;
  if (hooks) c->h = *hooks;
  *out = c;
  return VO_OK;
}
void vo_channel_destroy(vo_channel* c) { free(c); }
int vo_channel_state(const vo_channel* c) { return c->state; }
int vo_channel_offline_compute_allowed(const vo_channel* c) { return c->state == CH_ENABLED; }
int64_t vo_channel_disables_issued(const vo_channel* c) { return c->disables; }
int64_t vo_channel_pending_effective(const vo_channel* c) { return c->effective_at; }

static void ch_log(vo_channel* c, int64_t t, int what, int64_t aux, int mem) {
  if (c->h.log) c->h.log(c->h.user, t, what, aux, mem);
}

static void issue_disable(vo_channel* c, int64_t t, int mem) {
  /* channel.cpp:13-20 */
  c->state = CH_DISABLING;
  c->effective_at = t + c->toggle;
  ++c->gen;
  ++c->disables;
  if (c->h.schedule) c->h.schedule(c->h.user, c->effective_at, c->gen, 0);
  ch_log(c, t, LOG_DISABLE_ISSUED, c->effective_at, mem);
}

static void issue_enable(vo_channel* c, int64_t t) {
  /* channel.cpp:22-28 */
  c->state = CH_ENABLING;
  c->effective_at = t + c->toggle;
  ++c->gen;
  if (c->h.schedule) c->h.schedule(c->h.user, c->effective_at, c->gen, 0);
  ch_log(c, t, LOG_ENABLE_ISSUED, c->effective_at, 0);
}

void vo_channel_note_busy(vo_channel* c, int64_t t) {
  /* channel.cpp:30-39 */
  c->any_busy = 1;
  c->enable_after_disable = 0;
  if (c->cooldown_pending) {
    c->cooldown_pending = 0;
    ++c->cooldown_gen;
    ch_log(c, t, LOG_CD_CANCEL, 0, 0);
  }
  if (c->state == CH_ENABLED || c->state == CH_ENABLING) issue_disable(c, t, 0);
}

void vo_channel_note_all_idle(vo_channel* c, int64_t t) {
  /* channel.cpp:41-48 */
  c->any_busy = 0;
  if (c->state == CH_ENABLED || c->state == CH_ENABLING) return;
  c->cooldown_pending = 1;
  ++c->cooldown_gen;
  if (c->h.schedule) c->h.schedule(c->h.user, t + c->cooldown, c->cooldown_gen, 1);
  ch_log(c, t, LOG_CD_SCHED, t + c->cooldown, 0);
}

int64_t vo_channel_ensure_disabled(vo_channel* c, int64_t t) {
  /* channel.cpp:50-62 */
  if (c->state == CH_DISABLED) return t;
  if (c->state == CH_DISABLING) return c->effective_at;
  issue_disable(c, t, 1);
  return c->effective_at;
}

void vo_channel_handle_toggle(vo_channel* c, int64_t t, int64_t gen) {
  /* channel.cpp:64-79 */
  if (gen != c->gen) return;
  if (c->state == CH_DISABLING) {
    c->state = CH_DISABLED;
    ch_log(c, t, LOG_DISABLED, 0, 0);
    if (c->h.on_disabled) c->h.on_disabled(c->h.user, t);
    if (c->enable_after_disable && !c->any_busy) {
      c->enable_after_disable = 0;
      issue_enable(c, t);
    }
  } else if (c->state == CH_ENABLING) {
    c->state = CH_ENABLED;
    ch_log(c, t, LOG_ENABLED, 0, 0);
    if (c->h.on_enabled) c->h.on_enabled(c->h.user, t);
  }
}

void vo_channel_handle_cooldown(vo_channel* c, int64_t t, int64_t gen) {
  /* channel.cpp:81-90 */
  if (gen != c->cooldown_gen || !c->cooldown_pending) return;
  c->cooldown_pending = 0;
  if (c->any_busy) return;
  if (c->state == CH_DISABLED) issue_enable(c, t);
  else if (c->state == CH_DISABLING) c->enable_after_disable = 1;
}

/* ------------------------------------------------------------ byte images */

static inline uint64_t splitmix64(uint64_t x) {
  /* rng.hpp:12-17 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d4a2fa9fb8476dULL;
  return x ^ (x >> 31);
}

uint64_t vo_page_word(int64_t req, int32_t blk, int64_t word) {
  uint64_t base = splitmix64((uint64_t)req) ^ ((uint64_t)(uint32_t)blk << 40);
  return splitmix64(base + (uint64_t)word);
}

void vo_gather_images(const int64_t* reqs, const int32_t* blks, int n_pages, int64_t page_bytes,
                      uint8_t* dst) {
  int64_t words = page_bytes / 8;
  for (int i = 0; i < n_pages; ++i) {
    uint64_t* d = (uint64_t*)(dst + (int64_t)i * page_bytes);
    for (int64_t w = 0; w < words; ++w) d[w] = vo_page_word(reqs[i], blks[i], w);
  }
}

typedef struct {
  const uint8_t* src;
  int64_t slot_bytes, page_bytes;
  const int* phys;
  uint8_t* dst;
  int lo, hi;
} gather_job;

static void* gather_worker(void* arg) {
  gather_job* j = (gather_job*)arg;
  for (int i = j->lo; i < j->hi; ++i)
    memcpy(j->dst + (int64_t)i * j->page_bytes, j->src + (int64_t)j->phys[i] * j->slot_bytes,
           (size_t)j->page_bytes);
  return NULL;
}

void vo_gather_memcpy(const uint8_t* src, int64_t slot_bytes, int64_t page_bytes, const int* phys,
                      int n_pages, uint8_t* dst, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t th[256];
  gather_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (gather_job){src, slot_bytes, page_bytes, phys, dst,
                           (int)((int64_t)n_pages * t / nthreads),
                           (int)((int64_t)n_pages * (t + 1) / nthreads)};
    if (nthreads == 1) gather_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, gather_worker, &jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}
