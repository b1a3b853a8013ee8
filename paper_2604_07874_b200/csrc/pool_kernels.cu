// pool_kernels.cu -- warp-parallel pool bookkeeping, snapshot, Algorithm-1 selection and
// apply_reclaim for sm_100a.  Every kernel here is one CTA of 1024 threads working on the
// HBM-resident pool (valve_common.cuh); the pool is a few hundred KB, so these ops are
// latency-bound and the design goal is "one launch, no host round trip" per reference call.
//
// Reference semantics followed (file:line under /root/reference/proj):
//   online_grow/online_release     src/memory.cpp:31-51
//   offline_reserve                src/memory.cpp:66-97 (incl. the logical slot-id quirk)
//   offline_release                src/memory.cpp:99-114
//   requests_on_handle / handles_of_request / offline_pages_of   src/memory.cpp:116-140
//   snapshot                       src/memory.cpp:142-153
//   apply_reclaim                  src/memory.cpp:155-180
//   check_invariants               src/memory.cpp:190-211
//   selective_reclaim / fifo / oracle / evicted_cost   src/reclaim.cpp:19-126
#include "valve_common.cuh"
#include "valve_kernels.h"

namespace valve {

__device__ __forceinline__ void set_err(const PoolDev& P, int code, int detail, int64_t arg) {
  P.mirror->err = code;
  P.mirror->err_detail = detail;
  P.mirror->err_arg = arg;
}

// Thread 0 publishes the counters; called by every thread after the op's last sync.
__device__ __forceinline__ void publish(const PoolDev& P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    P.mirror->n_free = P.hdr->n_free;
    P.mirror->n_online = P.hdr->n_online;
    P.mirror->n_offline = P.hdr->n_offline;
    __threadfence_system();
  }
}

__device__ __forceinline__ void op_begin(const PoolDev& P) {
  if (threadIdx.x == 0) {
    P.mirror->err = 0;
    P.mirror->err_detail = 0;
    P.mirror->err_arg = 0;
  }
}

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
      set_err(P, kErrRuntime, kDetBlocksFull, P.P);
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

// Frees every live page of `row` (memory.cpp:99-114); emptied handles go free.  The block
// table entries become `bt_fill` (-1 for a normal release, the quarantine page after a
// reclaim).  Returns the number of handles freed (valid in thread 0 after the call).
__device__ int release_row_pages(const PoolDev& P, int row, int bt_fill, int* s_freed) {
  const int nb = P.row_nblk[row];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int64_t bi = (int64_t)row * P.P + i;
    const int p = P.bt[bi];
    if (p < 0 || p >= P.quarantine) continue;
    P.bt[bi] = bt_fill;
    if (P.slot_row[p] != row) continue;
    P.slot_row[p] = -1;
    P.slot_lid[p] = -1;
    P.slot_blk[p] = -1;
    const int h = p / P.S;
    if (atomicSub(&P.hused[h], 1) == 1) {
      P.hstate[h] = kFree;
      atomicAdd(s_freed, 1);
    }
  }
  return 0;
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

// Distinct residents of handle h, computed by one warp: wfirst[s] = 1 marks the lowest
// slot holding each request (0 for repeats and empty slots), wreq[s] the slot's request id.
// Buffers are per-warp shared memory of S entries.  Returns the distinct count.
__device__ int warp_residents(const PoolDev& P, int h, int64_t* wreq, int* wfirst) {
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)h * P.S;
  for (int s = lane; s < P.S; s += 32) {
    const int r = P.slot_row[base + s];
    wfirst[s] = r;  // the row for now
    wreq[s] = r >= 0 ? P.row_req[r] : 0;
  }
  __syncwarp();
  int flags = 0, cnt = 0;  // bit j = slot lane + 32*j is a first occurrence
  for (int s = lane, j = 0; s < P.S; s += 32, ++j) {
    const int r = wfirst[s];
    bool first = r >= 0;
    for (int q = 0; q < s && first; ++q) first = wfirst[q] != r;
    if (first) {
      flags |= 1 << j;
      ++cnt;
    }
  }
  __syncwarp();
  for (int s = lane, j = 0; s < P.S; s += 32, ++j) wfirst[s] = (flags >> j) & 1;
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  return cnt;
}

// rank of slot s among the first-flagged requests of the warp buffers
__device__ __forceinline__ int warp_rank(const int64_t* wreq, const int* wfirst, int S, int s) {
  int rank = 0;
  const int64_t v = wreq[s];
  for (int q = 0; q < S; ++q) rank += (wfirst[q] && wreq[q] < v);
  return rank;
}

constexpr int kMaxS = 256;  // handle_size_pages limit of the warp buffers

__global__ void __launch_bounds__(kNT) k_requests_on_handle(PoolDev P, int h, int64_t* out) {
  __shared__ int64_t wreq[kMaxS];
  __shared__ int wfirst[kMaxS];
  op_begin(P);
  if (threadIdx.x < 32) {
    const int cnt = warp_residents(P, h, wreq, wfirst);
    for (int s = threadIdx.x; s < P.S; s += 32)
      if (wfirst[s]) out[warp_rank(wreq, wfirst, P.S, s)] = wreq[s];
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
// Pass A (warp per handle) writes each handle's sorted residents to s_key scratch;
// pass B compacts with a CTA scan.  Output: s_hid / s_hmap / s_roff / res_pages (reqs).
__global__ void __launch_bounds__(kNT) k_snapshot(PoolDev P) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t* wreq = reinterpret_cast<int64_t*>(smem) + (size_t)wid * P.S;
  int* wfirst = reinterpret_cast<int*>(reinterpret_cast<int64_t*>(smem) + (size_t)nw * P.S) +
                (size_t)wid * P.S;
  op_begin(P);
  int64_t* sorted = reinterpret_cast<int64_t*>(P.s_key);
  for (int h = wid; h < P.H; h += nw) {
    if (P.hstate[h] != kOffline) {
      if (lane == 0) P.s_cnt[h] = 0;
      continue;
    }
    const int cnt = warp_residents(P, h, wreq, wfirst);
    for (int s = lane; s < P.S; s += 32)
      if (wfirst[s]) sorted[(int64_t)h * P.S + warp_rank(wreq, wfirst, P.S, s)] = wreq[s];
    if (lane == 0) P.s_cnt[h] = cnt;
    __syncwarp();
  }
  __syncthreads();
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
      for (int j = 0; j < c; ++j) P.res_pages[carry_r + exr + j] = sorted[(int64_t)h * P.S + j];
    }
    carry_h += toth;
    carry_r += totr;
  }
  if (threadIdx.x == 0) {
    P.s_roff[carry_h] = carry_r;
    P.mirror->r[0] = carry_h;
    P.mirror->r[1] = carry_r;
  }
  publish(P);
}

// --------------------------------------------------------------- selection cores

// Algorithm 1 (reclaim.cpp:33-67) on an instance in index space: handles 0..n-1 with ids
// hid[], ref lists rref[roff[i]..roff[i+1]) of dense request indices < m, costs cost[].
// Marginals are maintained incrementally: evicting request r subtracts cost[r] from every
// handle listing r (once per listing, matching the reference's per-entry sum).
// All arrays are global scratch; values written with atomics are read with ld.global.cg.
__device__ void greedy_core(int n, const int* hid, const int* roff, const int* rref, int m,
                            const int64_t* cost, int k, int64_t* marg, int* taken, int* ev,
                            int* qoff, int* qcnt, int* qh, int* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int64_t s = 0;
    for (int e = roff[i]; e < roff[i + 1]; ++e) s += cost[rref[e]];
    marg[i] = s;
    taken[i] = 0;
  }
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    ev[r] = 0;
    qcnt[r] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int e = roff[i]; e < roff[i + 1]; ++e) atomicAdd(&qcnt[rref[e]], 1);
  __syncthreads();
  int carry = 0;
  for (int base = 0; base < m; base += blockDim.x) {
    const int r = base + threadIdx.x;
    const int c = r < m ? __ldcg(&qcnt[r]) : 0;
    int tot;
    const int ex = block_excl_scan(c, tot);
    if (r < m) qoff[r] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) qoff[m] = carry;
  for (int r = threadIdx.x; r < m; r += blockDim.x) qcnt[r] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int e = roff[i]; e < roff[i + 1]; ++e) {
      const int r = rref[e];
      qh[qoff[r] + atomicAdd(&qcnt[r], 1)] = i;
    }
  __syncthreads();
  for (int round = 0; round < k; ++round) {
    ArgMin a{0, 0, -1};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (__ldcg(&taken[i])) continue;
      ArgMin b{(int64_t)__ldcg((const long long*)&marg[i]), hid[i], i};
      if (argmin_less(b, a)) a = b;
    }
    a = block_argmin(a);
    const int best = a.idx;
    if (threadIdx.x == 0) {
      taken[best] = 1;
      out[round] = hid[best];
    }
    for (int e = roff[best] + threadIdx.x; e < roff[best + 1]; e += blockDim.x) {
      const int r = rref[e];
      if (atomicExch(&ev[r], 1) == 0) {
        const unsigned long long dec = (unsigned long long)(-cost[r]);
        for (int q = qoff[r]; q < qoff[r + 1]; ++q)
          atomicAdd(reinterpret_cast<unsigned long long*>(&marg[qh[q]]), dec);
      }
    }
    __syncthreads();
  }
}

// FIFO (reclaim.cpp:69-83): rank of (mapped_at, id, index) -> the k oldest.
__device__ void fifo_core(int n, const int* hid, const int64_t* mapped, int k, int* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t mi = mapped[i];
    const int ii = hid[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const int64_t mj = mapped[j];
      const int ij = hid[j];
      rank += (mj < mi) || (mj == mi && (ij < ii || (ij == ii && j < i)));
    }
    if (rank < k) out[rank] = ii;
  }
  __syncthreads();
}

// Exhaustive oracle (reclaim.cpp:85-126), n <= 20: subsets enumerated by lexicographic rank
// over the ascending ids; cost(S) = sum of cost[r] over requests whose handle mask meets S.
// hmask[r] = bitmask of sorted positions listing r.  Returns the winning subset in out[].
__device__ void oracle_core(int n, const int* sorted_ids, int m, const unsigned* hmask,
                            const int64_t* cost, int k, int* out) {
  __shared__ long long binom[21][21];
  if (threadIdx.x == 0) {
    for (int a = 0; a <= 20; ++a)
      for (int b = 0; b <= 20; ++b)
        binom[a][b] = (b == 0) ? 1 : (a == 0 ? 0 : 0);
    for (int a = 1; a <= 20; ++a)
      for (int b = 1; b <= a; ++b) binom[a][b] = binom[a - 1][b - 1] + (b <= a - 1 ? binom[a - 1][b] : 0);
  }
  __syncthreads();
  const long long total = binom[n][k];
  ArgMin best{0, 0, -1};
  for (long long rnk = threadIdx.x; rnk < total; rnk += blockDim.x) {
    // unrank the lexicographic combination
    unsigned mask = 0;
    long long rr = rnk;
    int start = 0;
    for (int pos = 0; pos < k; ++pos) {
      for (int c = start; c < n; ++c) {
        const long long cnt = binom[n - c - 1][k - pos - 1];
        if (rr < cnt) {
          mask |= 1u << c;
          start = c + 1;
          break;
        }
        rr -= cnt;
      }
    }
    int64_t c = 0;
    for (int r = 0; r < m; ++r)
      if (hmask[r] & mask) c += cost[r];
    ArgMin cand{c, 0, (int)rnk};
    if (argmin_less(cand, best)) best = cand;
  }
  best = block_argmin(best);
  if (threadIdx.x == 0) {
    long long rr = best.idx;
    int start = 0;
    for (int pos = 0; pos < k; ++pos)
      for (int c = start; c < n; ++c) {
        const long long cnt = binom[n - c - 1][k - pos - 1];
        if (rr < cnt) {
          out[pos] = sorted_ids[c];
          start = c + 1;
          break;
        }
        rr -= cnt;
      }
  }
  __syncthreads();
}

// --------------------------------------------------------------------- apply core

// apply_reclaim (memory.cpp:155-180) for ids[0..k).  Converts the valid prefix, reports
// the invalidated pages, then (if the whole list was valid) releases the residual pages of
// every evicted request.  Writes res_* and res_counts.
__device__ void apply_core(const PoolDev& P, const int* ids, int k, int64_t t) {
  __shared__ int s_bad, s_nt, s_ne, s_freed;
  if (threadIdx.x == 0) {
    s_bad = k;
    s_nt = 0;
    s_ne = 0;
    s_freed = 0;
  }
  __syncthreads();
  // First invalid position: out of range, not offline, or a repeat (already converted).
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int h = ids[i];
    bool bad = h < 0 || h >= P.H || P.hstate[h] != kOffline;
    for (int j = 0; j < i && !bad; ++j) bad = ids[j] == h;
    if (bad) atomicMin(&s_bad, i);
  }
  __syncthreads();
  const int b = s_bad;
  if (threadIdx.x == 0 && b < k) {
    const int h = ids[b];
    if (h < 0 || h >= P.H) set_err(P, kErrOutOfRange, kDetApplyRange, h);
    else set_err(P, kErrLogic, kDetNotOffline, h);
  }
  // Clear the chosen handles, collecting (row, logical page, physical page, block).
  const int64_t nslots = (int64_t)b * P.S;
  for (int64_t idx = threadIdx.x; idx < nslots; idx += blockDim.x) {
    const int h = ids[idx / P.S];
    const int64_t p = (int64_t)h * P.S + idx % P.S;
    const int row = P.slot_row[p];
    if (row < 0) continue;
    const int pos = atomicAdd(&s_nt, 1);
    const int blk = P.slot_blk[p];
    P.s_qh[pos] = row;
    P.s_rref[pos] = (int)((int64_t)h * P.S + P.slot_lid[p]);  // logical page id
    P.s_tphys[pos] = (int)p;                                    // physical page id
    P.s_tblk[pos] = blk;
    P.s_ev[row] = 1;
    P.bt[(int64_t)row * P.P + blk] = P.quarantine;  // quarantine remap
    atomicSub(&P.row_npages[row], 1);
    P.slot_row[p] = -1;
    P.slot_lid[p] = -1;
    P.slot_blk[p] = -1;
  }
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    const int h = ids[i];
    P.hused[h] = 0;
    P.hstate[h] = kOnline;
    P.hmapped[h] = t;
    P.res_handles[i] = h;
  }
  __syncthreads();
  const int nt = s_nt;
  // Evicted rows, ascending request id.
  int carry = 0;
  for (int base = 0; base < P.R; base += blockDim.x) {
    const int r = base + threadIdx.x;
    const int f = (r < P.R && P.s_ev[r]) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    if (f) {
      P.s_evrows[carry + ex] = r;
      P.s_ev[r] = 0;
    }
    carry += tot;
  }
  const int ne = carry;
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const int row = P.s_evrows[e];
    const int64_t req = P.row_req[row];
    int rank = 0;
    for (int f = 0; f < ne; ++f) rank += P.row_req[P.s_evrows[f]] < req;
    P.s_rank[row] = rank;
    P.res_evicted[rank] = req;
  }
  __syncthreads();
  // Sort key: (request rank, logical page, physical page); payload: block index.
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    P.s_key[i] = ((uint64_t)P.s_rank[P.s_qh[i]] << 48) | ((uint64_t)(uint32_t)P.s_rref[i] << 24) |
                 (uint64_t)(uint32_t)P.s_tphys[i];
    P.s_pay[i] = P.s_tblk[i];
  }
  __syncthreads();
  block_bitonic_sort(P.s_key, P.s_pay, nt);
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const uint64_t key = P.s_key[i];
    const int rank = (int)(key >> 48);
    P.res_pages[i] = (int64_t)((key >> 24) & 0xffffffull);
    P.res_phys[i] = (int)(key & 0xffffffull);
    P.res_blk[i] = P.s_pay[i];
    if (i == 0 || (int)(P.s_key[i - 1] >> 48) != rank) P.res_inv_off[rank] = i;
  }
  if (threadIdx.x == 0) P.res_inv_off[ne] = nt;
  __syncthreads();
  if (b == k) {
    // Residual pages of evicted requests are plain frees (memory.cpp:176).
    for (int e = 0; e < ne; ++e) release_row_pages(P, P.s_evrows[e], P.quarantine, &s_freed);
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int e = 0; e < ne; ++e) ht_erase(P, P.row_req[P.s_evrows[e]]);
      // ht_erase zeroes the counters but keeps bt = quarantine for late readers
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    P.hdr->n_offline -= b + s_freed;
    P.hdr->n_online += b;
    P.hdr->n_free += s_freed;
    P.res_counts[0] = b;
    P.res_counts[1] = ne;
    P.res_counts[2] = nt;
    P.mirror->r[0] = b;
    P.mirror->r[1] = ne;
    P.mirror->r[2] = nt;
  }
}

__global__ void __launch_bounds__(kNT) k_apply(PoolDev P, const int* ids, int k, int64_t t) {
  op_begin(P);
  __syncthreads();
  apply_core(P, ids, k, t);
  publish(P);
}

// Fused reclaim: build the instance from the live slots (snapshot), select k handles on
// the device with row costs, then apply -- one launch (sim.cpp:936-942).
__global__ void __launch_bounds__(kNT) k_reclaim(PoolDev P, int k, int mode, int64_t t) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int* wrow = reinterpret_cast<int*>(smem) + (size_t)wid * P.S;
  op_begin(P);
  // offline handles ascending -> index space
  int carry = 0;
  for (int base = 0; base < P.H; base += blockDim.x) {
    const int h = base + threadIdx.x;
    const int f = (h < P.H && P.hstate[h] == kOffline) ? 1 : 0;
    int tot;
    const int ex = block_excl_scan(f, tot);
    if (f) {
      P.s_hid[carry + ex] = h;
      P.s_hmap[carry + ex] = P.hmapped[h];
    }
    carry += tot;
  }
  const int n = carry;
  if (k > n) k = n;
  __syncthreads();
  // distinct resident rows per handle (first occurrence), counts then CSR
  for (int i = wid; i < n; i += nw) {
    const int64_t base = (int64_t)P.s_hid[i] * P.S;
    for (int s = lane; s < P.S; s += 32) wrow[s] = P.slot_row[base + s];
    __syncwarp();
    int cnt = 0;
    for (int s = lane; s < P.S; s += 32) {
      const int r = wrow[s];
      bool first = r >= 0;
      for (int q = 0; q < s && first; ++q) first = wrow[q] != r;
      cnt += first;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
    if (lane == 0) P.s_cnt[i] = cnt;
    __syncwarp();
  }
  __syncthreads();
  carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int c = i < n ? P.s_cnt[i] : 0;
    int tot;
    const int ex = block_excl_scan(c, tot);
    if (i < n) P.s_roff[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) P.s_roff[n] = carry;
  __syncthreads();
  for (int i = wid; i < n; i += nw) {
    const int64_t base = (int64_t)P.s_hid[i] * P.S;
    for (int s = lane; s < P.S; s += 32) wrow[s] = P.slot_row[base + s];
    __syncwarp();
    int pos = P.s_roff[i];
    for (int s0 = 0; s0 < P.S; s0 += 32) {
      const int s = s0 + lane;
      bool first = false;
      int r = -1;
      if (s < P.S) {
        r = wrow[s];
        first = r >= 0;
        for (int q = 0; q < s && first; ++q) first = wrow[q] != r;
      }
      const unsigned m = __ballot_sync(kFull, first);
      if (first) P.s_rref[pos + __popc(m & ((1u << lane) - 1))] = r;
      pos += __popc(m);
    }
    __syncwarp();
  }
  __syncthreads();
  if (mode == 1) {
    fifo_core(n, P.s_hid, P.s_hmap, k, P.s_pick);
  } else {
    greedy_core(n, P.s_hid, P.s_roff, P.s_rref, P.R, P.row_cost, k, P.s_marg, P.s_taken, P.s_ev,
                P.s_qoff, P.s_qcnt, P.s_qh, P.s_pick);
    // greedy_core leaves s_ev set for the evicted rows; apply_core uses it as row marks
    for (int r = threadIdx.x; r < P.R; r += blockDim.x) P.s_ev[r] = 0;
  }
  __syncthreads();
  apply_core(P, P.s_pick, k, t);
  publish(P);
}

// ------------------------------------------------------------- invariants / fill

__global__ void __launch_bounds__(kNT) k_check_invariants(PoolDev P, int64_t online_used) {
  __shared__ int s_det;
  __shared__ long long s_arg;
  op_begin(P);
  if (threadIdx.x == 0) {
    s_det = 0;
    s_arg = 0;
  }
  for (int r = threadIdx.x; r < P.R; r += blockDim.x) P.s_qcnt[r] = 0;
  __syncthreads();
  int nf = 0, non = 0, noff = 0;
  for (int h = threadIdx.x; h < P.H; h += blockDim.x) {
    const uint8_t st = P.hstate[h];
    nf += st == kFree;
    non += st == kOnline;
    noff += st == kOffline;
    int live = 0;
    for (int s = 0; s < P.S; ++s) {
      const int64_t p = (int64_t)h * P.S + s;
      const int row = P.slot_row[p];
      if (row < 0) continue;
      ++live;
      atomicAdd(&P.s_qcnt[row], 1);
      const int blk = P.slot_blk[p];
      if (blk < 0 || blk >= P.P || P.bt[(int64_t)row * P.P + blk] != (int)p)
        atomicCAS(&s_det, 0, (int)kDetInvBlock);
    }
    if (live != P.hused[h] || P.hused[h] > P.S) atomicCAS(&s_det, 0, (int)kDetInvSlots);
    if (st != kOffline && P.hused[h] != 0) atomicCAS(&s_det, 0, (int)kDetInvNonOffline);
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
  if (threadIdx.x == 0 && s_det) {
    // memory.cpp:192-209 messages are mapped on the host from the detail code
    set_err(P, kErrLogic, s_det, 0);
  }
  publish(P);
}

// Deterministic KV image of every live page (request, block) -> its physical slot.
// Grid-stride over slots; 16-byte stores.
__global__ void __launch_bounds__(256) k_fill_pages(PoolDev P) {
  const int64_t nslots = (int64_t)P.H * P.S;
  const int64_t words = P.page_bytes / 8;
  for (int64_t p = blockIdx.x; p < nslots; p += gridDim.x) {
    const int row = P.slot_row[p];
    if (row < 0) continue;
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

// ---------------------------------------------------- selection over host instances

// Instance arrays already on the device; dense request index per ref (-1 = no cost entry).
__global__ void __launch_bounds__(kNT)
    k_select_instance(SelectArgs A) {
  __shared__ int s_missing;
  if (threadIdx.x == 0) s_missing = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < A.nnz; e += blockDim.x)
    if (A.rref[e] < 0) s_missing = 1;
  __syncthreads();
  if (threadIdx.x == 0) A.status[0] = 0;
  // reclaim.cpp:13: cost_of throws on the first evaluation (greedy / exhaustive, k > 0);
  // fifo never looks at costs (reclaim.cpp:69-83)
  if (A.k > 0 && s_missing && A.mode != 1) {
    if (threadIdx.x == 0) A.status[0] = kDetNoCost;
    return;
  }
  if (A.mode == 0) {
    greedy_core(A.n, A.hid, A.roff, A.rref, A.m, A.cost, A.k, A.marg, A.taken, A.ev, A.qoff,
                A.qcnt, A.qh, A.out);
  } else if (A.mode == 1) {
    fifo_core(A.n, A.hid, A.mapped, A.k, A.out);
  } else if (A.k > 0) {
    // sorted ids and per-request handle masks
    for (int i = threadIdx.x; i < A.n; i += blockDim.x) {
      int rank = 0;
      for (int j = 0; j < A.n; ++j)
        rank += A.hid[j] < A.hid[i] || (A.hid[j] == A.hid[i] && j < i);
      A.taken[rank] = A.hid[i];
      A.qcnt[i] = rank;  // position of handle i in sorted order
    }
    for (int r = threadIdx.x; r < A.m; r += blockDim.x) A.ev[r] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < A.n; i += blockDim.x)
      for (int e = A.roff[i]; e < A.roff[i + 1]; ++e) atomicOr(reinterpret_cast<unsigned*>(&A.ev[A.rref[e]]), 1u << A.qcnt[i]);
    __syncthreads();
    oracle_core(A.n, A.taken, A.m, reinterpret_cast<const unsigned*>(A.ev), A.cost, A.k, A.out);
  }
}

// evicted_cost (reclaim.cpp:19-31): sequential union walk in one thread (it defines an
// error order -- unknown id / missing cost -- that a parallel sum would not preserve).
__global__ void k_evicted_cost(SelectArgs A, const int* pick, int n_pick) {
  if (threadIdx.x != 0) return;
  for (int r = 0; r < A.m; ++r) A.ev[r] = 0;
  int64_t total = 0;
  A.status[0] = 0;
  for (int j = 0; j < n_pick; ++j) {
    int hi = -1;
    for (int i = 0; i < A.n; ++i)
      if (A.hid[i] == pick[j]) {
        hi = i;
        break;
      }
    if (hi < 0) {
      A.status[0] = kDetApplyRange;  // unknown handle id
      return;
    }
    for (int e = A.roff[hi]; e < A.roff[hi + 1]; ++e) {
      const int r = A.rref[e];
      if (r < 0) {
        A.status[0] = kDetNoCost;
        return;
      }
      if (A.ev[r]) continue;
      A.ev[r] = 1;
      total += A.cost[r];
    }
  }
  A.result[0] = total;
}

}  // namespace valve

namespace valve {

// Recompute costs next to the request rows (sim.cpp:877-883 attaches them per snapshot).
__global__ void k_set_costs(PoolDev P, int n, const int64_t* reqs, const int64_t* costs) {
  __shared__ int s_missing;
  op_begin(P);
  if (threadIdx.x == 0) s_missing = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int row = ht_find(P, reqs[i]);
    if (row < 0) atomicAdd(&s_missing, 1);
    else P.row_cost[row] = costs[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) P.mirror->r[0] = s_missing;
  publish(P);
}

// ref request id -> index in the sorted cost keys (binary search), -1 when absent.
__global__ void k_map_refs(const int64_t* reqs, int nnz, const int64_t* keys, int m, int* rref) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int64_t v = reqs[e];
  int lo = 0, hi = m - 1, found = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int64_t k = keys[mid];
    if (k == v) {
      found = mid;
      break;
    }
    if (k < v) lo = mid + 1;
    else hi = mid - 1;
  }
  rref[e] = found;
}

// tile prefix of the offline work list: prefix[i] = sum_{j<i} npages[j] * chunks_per_page
__global__ void k_tile_prefix(const int* npages, int n, int cpp, int64_t* prefix) {
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
  if (threadIdx.x == 0) prefix[n] = s_carry * (int64_t)cpp;
}

}  // namespace valve
