// pool_kernels.cu -- warp-parallel pool bookkeeping and queries for sm_100a.  Every kernel
// is one CTA of 1024 threads over the HBM-resident pool (valve_common.cuh); the pool
// metadata is a few hundred KB, so these ops are latency-bound: one launch per reference
// call, CTA scans instead of the reference's ordered sets, no host round trip inside.
//
// Reference semantics followed (file:line under /root/reference/proj):
//   online_grow/online_release     src/memory.cpp:31-51
//   offline_reserve                src/memory.cpp:66-97 (incl. the logical slot-id quirk)
//   offline_release                src/memory.cpp:99-114
//   requests_on_handle / handles_of_request / offline_pages_of   src/memory.cpp:116-140
//   snapshot                       src/memory.cpp:142-153
//   check_invariants               src/memory.cpp:190-211
#include "pool_device.cuh"
#include "valve_kernels.h"

namespace valve {

// ------------------------------------------------------------------------ online side

__global__ void __launch_bounds__(kNT) k_online_grow(PoolDev P, int k, int64_t t) {
  op_begin(P);
  if (k > P.hdr->n_free) {  // memory.cpp:33
    if (threadIdx.x == 0) set_err(P, kErrLogic, kDetGrowExceeds, k);
    publish(P);
    return;
  }
  int carry = 0;
  for (int base = 0; base < P.H && carry < k; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int f = (h < P.H && P.hstate[h] == kFree) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    if (f && carry + ex < k) {  // take_lowest_free, memory.cpp:20-29
      P.hstate[h] = kOnline;
      P.hmapped[h] = t;
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    P.hdr->n_free -= k;
    P.hdr->n_online += k;
  }
  publish(P);
}

__global__ void __launch_bounds__(kNT) k_online_release(PoolDev P, int k, int64_t online_used) {
  // memory.cpp:37-51 in closed form: the loop stops once (n-1)*S < used, so at most
  // n_online - ceil(used/S) of the lowest-id online handles go back.
  op_begin(P);
  const int n_on = P.hdr->n_online;
  const int64_t need = (online_used + P.S - 1) / P.S;
  int64_t r = (int64_t)n_on - need;
  if (r > k) r = k;
  if (r < 0) r = 0;
  int carry = 0;
  for (int base = 0; base < P.H && carry < r; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int f = (h < P.H && P.hstate[h] == kOnline) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    if (f && carry + ex < r) P.hstate[h] = kFree;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    P.hdr->n_online -= (int)r;
    P.hdr->n_free += (int)r;
    P.mirror->r[0] = r;
  }
  publish(P);
}

// ----------------------------------------------------------------------- offline side

__global__ void __launch_bounds__(kNT)
    k_offline_reserve(PoolDev P, int64_t req, int pages, int64_t t, int max_off) {
  __shared__ int s_row, s_nt, s_fail;
  op_begin(P);
  if (P.hdr->tombstones > P.HC / 4) ht_rebuild(P, P.s_evrows);  // uniform branch
  if (threadIdx.x == 0) {
    s_row = ht_find(P, req);
    s_nt = 0;
    s_fail = 0;
  }
  __syncthreads();
  int row = s_row;
  // Capacity check (memory.cpp:70-77): partial slots of offline handles + mappable free.
  int64_t av = 0;
  int noff = 0, nfree = 0;
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) {
    const uint8_t st = P.hstate[h];
    if (st == kOffline) {
      av += P.S - P.hused[h];
      ++noff;
    } else if (st == kFree) {
      ++nfree;
    }
  }
  av = block_sum64(av);
  noff = block_sum(noff);
  nfree = block_sum(nfree);
  int mappable = nfree;
  if (max_off >= 0) mappable = min(mappable, max(0, max_off - noff));
  if (av + (int64_t)mappable * P.S < pages) {
    if (threadIdx.x == 0) P.mirror->r[0] = 0;
    publish(P);
    return;
  }
  const int nblk0 = row >= 0 ? P.row_nblk[row] : 0;
  if (threadIdx.x == 0) {
    if ((int64_t)nblk0 + pages > P.P) {
      set_err(P, kErrRuntime, kDetBlocksFull, (int64_t)nblk0 + pages);  // the row length needed
      s_fail = 1;
    } else if (row < 0) {
      s_row = ht_insert(P, req);
      if (s_row < 0) {
        set_err(P, kErrRuntime, kDetRowsFull, P.R);
        s_fail = 1;
      }
    }
  }
  __syncthreads();
  if (s_fail) {
    publish(P);
    return;
  }
  row = s_row;
  // Fill partially used offline handles in ascending id (memory.cpp:91-94).  A handle's
  // take is its capacity clipped by what the lower-id handles already absorbed.
  int carry = 0;
  for (int base = 0; base < P.H && carry < pages; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int cap = (h < P.H && P.hstate[h] == kOffline) ? P.S - P.hused[h] : 0;
    int tot;
    const int ex = block_excl_scan(cap, tot);
    const int take = min(max(pages - (carry + ex), 0), cap);
    if (take > 0) {
      const int i = atomicAdd(&s_nt, 1);
      P.s_hid[i] = h;
      P.s_cnt[i] = take;
      P.s_pick[i] = nblk0 + carry + ex;  // first block index placed on h
      P.s_taken[i] = P.hused[h];         // first logical slot id (used_slots++)
    }
    carry = min(pages, carry + tot);
  }
  // Then map the lowest free handles (memory.cpp:95, take_lowest_free).
  const int remaining = pages - carry;
  const int n_new = (remaining + P.S - 1) / P.S;
  int got = 0;
  for (int base = 0; base < P.H && got < n_new; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int f = (h < P.H && P.hstate[h] == kFree) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    const int j = got + ex;
    if (f && j < n_new) {
      P.hstate[h] = kOffline;
      P.hmapped[h] = t;
      P.hused[h] = 0;
      const int i = atomicAdd(&s_nt, 1);
      P.s_hid[i] = h;
      P.s_cnt[i] = min(P.S, remaining - j * P.S);
      P.s_pick[i] = nblk0 + carry + j * P.S;
      P.s_taken[i] = 0;
    }
    got += tot;
  }
  __syncthreads();
  // Slot assignment, one warp per touched handle: the i-th free physical slot (ascending)
  // gets logical id used0+i and block blk0+i.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = wid; i < s_nt; i += nw) {
    const int h = P.s_hid[i], take = P.s_cnt[i], blk0 = P.s_pick[i], lid0 = P.s_taken[i];
    int running = 0;
    for (int s0 = 0; s0 < P.S && running < take; s0 += 32) {
      const int s = s0 + lane;
      const int64_t p = (int64_t)h * P.S + s;
      const bool fr = s < P.S && P.slot_row[p] == -1;
      const unsigned m = __ballot_sync(kFull, fr);
      const int rank = running + __popc(m & ((1u << lane) - 1));
      if (fr && rank < take) {
        P.slot_row[p] = row;
        P.slot_lid[p] = lid0 + rank;
        P.slot_blk[p] = blk0 + rank;
        P.bt[(int64_t)row * P.P + blk0 + rank] = (int)p;
      }
      running += __popc(m);
    }
    if (lane == 0) P.hused[h] = lid0 + take;
  }
  if (threadIdx.x == 0) {
    P.row_npages[row] += pages;
    P.row_nblk[row] += pages;
    P.hdr->n_free -= n_new;
    P.hdr->n_offline += n_new;
    P.mirror->r[0] = 1;
  }
  publish(P);
}

// Request-hash rebuild after a table growth (valve_host.cu grow_tables): every live row of the
// old table is inserted into P's (empty, larger) table with CAS probing.
__global__ void k_ht_rehash(PoolDev P, const int* old_row, int old_hc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= old_hc) return;
  const int row = old_row[i];
  if (row < 0) return;
  const int64_t key = P.row_req[row];
  const int mask = P.HC - 1;
  int j = ht_slot(key, P.HC);
  while (atomicCAS(&P.ht_row[j], kEmpty, row) != kEmpty) j = (j + 1) & mask;
  P.ht_key[j] = key;
}

__global__ void __launch_bounds__(kNT) k_offline_release(PoolDev P, int64_t req) {
  __shared__ int s_row, s_freed;
  op_begin(P);
  if (threadIdx.x == 0) {
    s_row = ht_find(P, req);
    s_freed = 0;
  }
  __syncthreads();
  const int row = s_row;
  if (row >= 0) {
    release_row_pages(P, row, -1, &s_freed);
    __syncthreads();
    if (threadIdx.x == 0) {
      ht_erase(P, req);
      P.hdr->n_free += s_freed;
      P.hdr->n_offline -= s_freed;
    }
  }
  publish(P);
}

// ------------------------------------------------------------------------- queries

__global__ void __launch_bounds__(kNT) k_requests_on_handle(PoolDev P, int h, int64_t* out) {
  op_begin(P);
  if (threadIdx.x < 32) {
    const int nc = (P.S + 31) >> 5;
    int cnt = 0;
    VALVE_DISPATCH_NC(nc, cnt = warp_sorted_residents<NC>(P, h, out));
    if (threadIdx.x == 0) P.mirror->r[0] = cnt;
  }
  publish(P);
}

__global__ void __launch_bounds__(kNT) k_handles_of_request(PoolDev P, int64_t req, int* out) {
  __shared__ int s_row;
  op_begin(P);
  if (threadIdx.x == 0) s_row = ht_find(P, req);
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) P.s_cnt[h] = 0;
  __syncthreads();
  const int row = s_row;
  if (row >= 0) {
    const int nb = P.row_nblk[row];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const int p = P.bt[(int64_t)row * P.P + i];
      if (p >= 0 && p < P.quarantine && P.slot_row[p] == row) P.s_cnt[p / P.S] = 1;
    }
  }
  __syncthreads();
  int carry = 0;
  for (int base = 0; base < P.H; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int f = (h < P.H && P.s_cnt[h] && P.hstate[h] == kOffline) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    if (f) out[carry + ex] = h;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    P.mirror->r[0] = carry;
    P.mirror->r[1] = row >= 0 ? P.row_npages[row] : 0;
  }
  publish(P);
}

__global__ void k_offline_pages_of(PoolDev P, int64_t req) {
  op_begin(P);
  if (threadIdx.x == 0) {
    const int row = ht_find(P, req);
    P.mirror->r[0] = row >= 0 ? P.row_npages[row] : 0;
    P.mirror->r[1] = row;
    P.mirror->r[2] = row >= 0 && P.row_pbytes[row] ? P.row_pbytes[row] : P.page_bytes;
  }
  publish(P);
}

__global__ void k_block_table(PoolDev P, int64_t req, int* out) {
  __shared__ int s_row;
  op_begin(P);
  if (threadIdx.x == 0) s_row = ht_find(P, req);
  __syncthreads();
  const int row = s_row;
  int n = 0;
  if (row >= 0) {
    n = P.row_nblk[row];
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = P.bt[(int64_t)row * P.P + i];
  }
  if (threadIdx.x == 0) {
    P.mirror->r[0] = n;
    P.mirror->r[1] = row;
  }
  publish(P);
}

// snapshot (memory.cpp:142-153): offline handles ascending, residents ascending.
// Pass A (warp per handle, 2 handles in flight) writes each handle's sorted residents to
// scratch at stride S; pass B compacts with a CTA scan into s_hid/s_hmap/s_roff/res_pages.
// Snapshot, part 1 (grid-wide): one warp per handle sorts its distinct resident requests.
__global__ void __launch_bounds__(256) k_snapshot_handles(PoolDev P) {
  const int lane = threadIdx.x & 31;
  const int h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (h >= P.H) return;
  const int nc = (P.S + 31) >> 5;
  int64_t* sorted = reinterpret_cast<int64_t*>(P.s_key);
  if (P.hstate[h] != kOffline) {
    if (lane == 0) P.s_cnt[h] = 0;
    return;
  }
  int cnt = 0;
  VALVE_DISPATCH_NC(nc, cnt = warp_sorted_residents<NC>(P, h, sorted + (int64_t)h * P.S));
  if (lane == 0) P.s_cnt[h] = cnt;
}

// Snapshot, part 2 (one CTA): compact the offline handles into the CSR instance.
__global__ void __launch_bounds__(kNT) k_snapshot(PoolDev P) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  op_begin(P);
  const int64_t* sorted = reinterpret_cast<const int64_t*>(P.s_key);
  int carry_h = 0, carry_r = 0;
  for (int base = 0; base < P.H; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int off = (h < P.H && P.hstate[h] == kOffline) ? 1 : 0;
    const int c = off ? P.s_cnt[h] : 0;
    int toth, totr;
    const int exh = block_excl_scan(off, toth);
    const int exr = block_excl_scan(c, totr);
    if (off) {
      const int i = carry_h + exh;
      P.s_hid[i] = h;
      P.s_hmap[i] = P.hmapped[h];
      P.s_roff[i] = carry_r + exr;
    }
    carry_h += toth;
    carry_r += totr;
  }
  if (threadIdx.x == 0) {
    P.s_roff[carry_h] = carry_r;
    P.mirror->r[0] = carry_h;
    P.mirror->r[1] = carry_r;
  }
  __syncthreads();
  // copy-out, one warp per handle (coalesced)
  for (int i = wid; i < carry_h; i += nw) {
    const int h = P.s_hid[i];
    const int o = P.s_roff[i], c = P.s_roff[i + 1] - o;
    for (int j = lane; j < c; j += 32) P.res_pages[o + j] = sorted[(int64_t)h * P.S + j];
  }
  publish(P);
}

// ------------------------------------------------------------- invariants / fill

__global__ void __launch_bounds__(kNT) k_check_invariants(PoolDev P, int64_t online_used) {
  __shared__ int s_det;
  op_begin(P);
  if (threadIdx.x == 0) s_det = 0;
  for (int r = threadIdx.x; r < P.R; r += blockDim.x) P.s_qcnt[r] = 0;
  __syncthreads();
  int nf = 0, non = 0, noff = 0;
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) {
    const uint8_t st = P.hstate[h];
    nf += st == kFree;
    non += st == kOnline;
    noff += st == kOffline;
  }
  // slot pass: one thread per slot, handle counts via shared-memory-free atomics in scratch
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) P.s_cnt[h] = 0;
  __syncthreads();
  const int64_t ns = (int64_t)P.H * P.S;
  for (int64_t p = threadIdx.x; p < ns; p += blockDim.x) {
    const int row = P.slot_row[p];
    if (row < 0) continue;
    atomicAdd(&P.s_cnt[p / P.S], 1);
    atomicAdd(&P.s_qcnt[row], 1);
    const int blk = P.slot_blk[p];
    if (blk < 0 || blk >= P.P || P.bt[(int64_t)row * P.P + blk] != (int)p)
      atomicCAS(&s_det, 0, (int)kDetInvBlock);
  }
  __syncthreads();
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) {
    const int live = P.s_cnt[h];
    if (live != P.hused[h] || P.hused[h] > P.S) atomicCAS(&s_det, 0, (int)kDetInvSlots);
    if (P.hstate[h] != kOffline && P.hused[h] != 0) atomicCAS(&s_det, 0, (int)kDetInvNonOffline);
  }
  nf = block_sum(nf);
  non = block_sum(non);
  noff = block_sum(noff);
  if (threadIdx.x == 0) {
    if (nf + non + noff != P.H || nf != P.hdr->n_free || non != P.hdr->n_online ||
        noff != P.hdr->n_offline)
      atomicCAS(&s_det, 0, (int)kDetInvPartition);
    if (online_used < 0 || online_used > (int64_t)non * P.S) atomicCAS(&s_det, 0, (int)kDetInvOnline);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < P.R; r += blockDim.x) {
    if (P.s_qcnt[r] == 0) continue;
    if (P.s_qcnt[r] != P.row_npages[r]) atomicCAS(&s_det, 0, (int)kDetInvRow);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_det) set_err(P, kErrLogic, s_det, 0);  // memory.cpp:192-209
  publish(P);
}

// Deterministic KV image of every live page (request, block) -> its physical slot.
// Grid-stride over slots; 16-byte stores.
__global__ void __launch_bounds__(256) k_fill_pages(PoolDev P) {
  const int64_t nslots = (int64_t)P.H * P.S;
  for (int64_t p = blockIdx.x; p < nslots; p += gridDim.x) {
    const int row = P.slot_row[p];
    if (row < 0) continue;
    const int64_t words = (P.row_pbytes[row] ? P.row_pbytes[row] : P.page_bytes) / 8;
    const uint64_t base = page_word_base(P.row_req[row], P.slot_blk[p]);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(P.pages + p * P.slot_bytes);
    for (int64_t w = threadIdx.x; w < words / 2; w += blockDim.x) {
      ulonglong2 v;
      v.x = splitmix64(base + (uint64_t)(2 * w));
      v.y = splitmix64(base + (uint64_t)(2 * w + 1));
      dst[w] = v;
    }
  }
}

// Recompute costs next to the request rows (sim.cpp:877-883 attaches them per snapshot);
// which = 1 sets the rows' page sizes instead (valve_pool_set_page_bytes).
__global__ void k_set_costs(PoolDev P, int n, const int64_t* reqs, const int64_t* costs, int which) {
  __shared__ int s_missing;
  op_begin(P);
  if (threadIdx.x == 0) s_missing = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = ht_find(P, reqs[i]);
    if (row < 0) atomicAdd(&s_missing, 1);
    else if (which == 0) P.row_cost[row] = costs[i];
    else P.row_pbytes[row] = costs[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) P.mirror->r[0] = s_missing;
  publish(P);
}

// tile prefix of the offline work list: prefix[i] = sum_{j<i} npages[j] * chunks_per_page
__global__ void k_tile_prefix(const int* npages, int n, int cpp, int64_t* prefix,
                              unsigned long long* total_out, unsigned* frozen) {
  // the work list is frozen from the first launch after a reset (valve_offline_reset clears
  // the flag): resumed launches -- direct or replays of a captured graph -- keep the prefix the
  // saved cursors refer to
  if (frozen && *(volatile unsigned*)frozen) return;
  __shared__ long long s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < n ? npages[i] : 0;
    int tot;
    const int ex = block_excl_scan(v, tot);
    if (i < n) prefix[i] = (s_carry + ex) * (int64_t)cpp;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    prefix[n] = s_carry * (int64_t)cpp;
    if (total_out) *total_out = (unsigned long long)(s_carry * (int64_t)cpp);
    if (frozen) *frozen = 1u;
  }
}

}  // namespace valve
