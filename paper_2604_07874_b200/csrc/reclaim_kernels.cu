// reclaim_kernels.cu -- Algorithm-1 selection, apply_reclaim and the fused device reclaim
// (snapshot -> select -> apply in one launch) for sm_100a.
//
// Reference semantics (file:line under /root/reference/proj):
//   selective_reclaim / fifo / oracle / evicted_cost   src/reclaim.cpp:19-126
//   apply_reclaim                                      src/memory.cpp:155-180
//   Sim::finish_op (snapshot + Cost + select + apply)  src/sim.cpp:928-943
//
// Layout: one CTA of 1024 threads.  The instance (offline handles, distinct resident rows)
// is built into global scratch with a stride of S per handle; the greedy rounds run in ONE
// warp over shared-memory marginals (n <= 2048 handles) with incremental updates through a
// reverse request->handle index, so a round is ~a hundred cycles and no CTA barrier.  The
// invalidation report is sorted in shared memory (<= 8192 pages per op).
#include "pool_device.cuh"
#include "valve_kernels.h"

namespace valve {

constexpr int kSmemHandles = 2048;   // greedy in shared memory up to this many handles
constexpr int kSmemListings = 4096;  // ... and this many (handle, request) listings
constexpr int kSmemTuples = 8192;    // invalidation report sorted in shared memory
// dynamic shared memory of k_reclaim / k_apply / k_select_instance (host sets the attribute):
// greedy 2048*(8+4+4+1+4) + 4096*(8+4+4+4+4+4) + 4 = 157,700 B; apply sort 8192*20 = 163,840 B
static_assert(kSmemHandles * 21 + kSmemListings * 28 + 64 <= 160 * 1024, "greedy smem");
static_assert(kSmemTuples * 20 <= 160 * 1024, "sort smem");
static_assert((1024 + 3 * 8192 + 6 * 2048) * 4 <= 160 * 1024, "apply fast-path smem");  // key 8 + pay 4 + cursors 4 + segment 4

__device__ long long g_greedy_cycles[2];  // diagnostics: argmin / update cycles of the last run
__device__ long long g_select_ns[5];      // diagnostics: selection phase stamps of the last run
__device__ long long g_apply_ns[10];       // diagnostics: apply_core phase stamps of the last run

// Ref lists of instance handle i: CSR (off) or fixed stride with counts (cnt), the stride slot
// being i itself or map[i] (the fused reclaim lays rows out by handle id: map = instance ids).
struct Refs {
  const int* off;
  const int* cnt;
  int stride;
  const int* map = nullptr;
  __device__ __forceinline__ int slot(int i) const { return map ? map[i] : i; }
  __device__ __forceinline__ int begin(int i) const { return cnt ? slot(i) * stride : off[i]; }
  __device__ __forceinline__ int end(int i) const { return cnt ? slot(i) * stride + cnt[slot(i)] : off[i + 1]; }
};

// Reverse index request -> handle indices (one entry per listing, duplicates kept), and
// the initial marginals marg[i] = sum of cost over the listings of handle i.  CTA-wide.
__device__ void build_instance_index(int n, Refs R, const int* rref, int m, const int64_t* cost,
                                     int64_t* marg, int* qoff, int* qcnt, int* qh, int* ev) {
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    qcnt[r] = 0;
    ev[r] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int64_t s = 0;
    for (int e = R.begin(i); e < R.end(i); ++e) {
      const int r = rref[e];
      s += cost[r];
      atomicAdd(&qcnt[r], 1);
    }
    marg[i] = s;
  }
  __syncthreads();
  int carry = 0;
  for (int base = 0; base < m; base += blockDim.x) {
    const int r = base + threadIdx.x;
    const int c = r < m ? qcnt[r] : 0;
    int tot;
    const int ex = block_excl_scan(c, tot);
    if (r < m) qoff[r] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) qoff[m] = carry;
  for (int r = threadIdx.x; r < m; r += blockDim.x) qcnt[r] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int e = R.begin(i); e < R.end(i); ++e) {
      const int r = rref[e];
      qh[qoff[r] + atomicAdd(&qcnt[r], 1)] = i;
    }
  __syncthreads();
}

__device__ __forceinline__ ArgMin warp_argmin(ArgMin a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMin b;
    b.v = __shfl_xor_sync(kFull, a.v, o);
    b.id = __shfl_xor_sync(kFull, a.id, o);
    b.idx = __shfl_xor_sync(kFull, a.idx, o);
    if (argmin_less(b, a)) a = b;
  }
  return a;
}

__device__ __forceinline__ void cand_min(int64_t& bm, int& bid, int& bidx, int64_t m, int id, int idx) {
  // lexicographic (marginal, id) minimum; idx < 0 = no candidate.  Branch-free.
  const bool better = (idx >= 0) & ((bidx < 0) | (m < bm) | ((m == bm) & (id < bid)));
  bm = better ? m : bm;
  bid = better ? id : bid;
  bidx = better ? idx : bidx;
}

__device__ __forceinline__ void warp_min(int64_t& bm, int& bid, int& bidx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t om = __shfl_xor_sync(kFull, bm, o);
    const int oid = __shfl_xor_sync(kFull, bid, o);
    const int oidx = __shfl_xor_sync(kFull, bidx, o);
    cand_min(bm, bid, bidx, om, oid, oidx);
  }
}

// Algorithm 1 (reclaim.cpp:33-67), CTA-wide with the marginals in registers: thread t owns
// handles t and t + blockDim (n <= 2 * blockDim).  A round is a two-level (marginal, id)
// argmin (shuffles, 32 partials in shared memory, every warp finishes the reduction so no
// second barrier is needed), then the threads of the winner's listings evict its requests
// (first eviction wins an atomicExch on ev) and scatter -cost into `delta` through the
// reverse index; owners fold their deltas in.  Two barriers per round, all data on-chip.
// `delta` holds the initial marginals on entry.
constexpr int kGreedyThreads = 256;                         // warps 0..7 run the rounds
constexpr int kGreedyOwn = kSmemHandles / kGreedyThreads;  // handles per thread (registers)

__device__ __forceinline__ void greedy_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kGreedyThreads) : "memory");
}

// Called by threads [0, kGreedyThreads) only (named barrier 1); n <= kSmemHandles.
__device__ void greedy_block(int n, const int* hid, Refs R, const int* rref, const int64_t* cost,
                             int k, int64_t* delta, int* ev, const int* qoff, const int* qh, int* out) {
  constexpr int NW = kGreedyThreads / 32;
  __shared__ int64_t w_m[NW];
  __shared__ int w_id[NW], w_idx[NW];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  int64_t m[kGreedyOwn];
  unsigned live = 0;
#pragma unroll
  for (int j = 0; j < kGreedyOwn; ++j) {
    const int i = t + j * kGreedyThreads;
    m[j] = i < n ? delta[i] : 0;
    if (i < n) live |= 1u << j;
  }
  greedy_bar();
#pragma unroll
  for (int j = 0; j < kGreedyOwn; ++j)
    if ((live >> j) & 1u) delta[t + j * kGreedyThreads] = 0;
  long long c_arg = 0, c_upd = 0;
  for (int round = 0; round < k; ++round) {
    const long long c0 = clock64();
    int64_t bm = 0;
    int bid = 0, bidx = -1;
#pragma unroll
    for (int j = 0; j < kGreedyOwn; ++j) {
      const int i = t + j * kGreedyThreads;
      const bool on = (live >> j) & 1u;
      cand_min(bm, bid, bidx, m[j], on ? hid[i] : 0, on ? i : -1);
    }
    warp_min(bm, bid, bidx);
    if (lane == 0) {
      w_m[wid] = bm;
      w_id[wid] = bid;
      w_idx[wid] = bidx;
    }
    greedy_bar();
    bm = lane < NW ? w_m[lane] : 0;
    bid = lane < NW ? w_id[lane] : 0;
    bidx = lane < NW ? w_idx[lane] : -1;
    warp_min(bm, bid, bidx);
    const int best = bidx;
    const long long c1 = clock64();
    c_arg += c1 - c0;
#pragma unroll
    for (int j = 0; j < kGreedyOwn; ++j)
      if (best == t + j * kGreedyThreads) live &= ~(1u << j);
    if (t == 0) out[round] = hid[best];
    for (int e = R.begin(best) + t; e < R.end(best); e += kGreedyThreads) {
      const int r = rref[e];
      if (atomicExch(&ev[r], 1) == 0) {
        const unsigned long long dec = (unsigned long long)(-cost[r]);
        for (int q = qoff[r]; q < qoff[r + 1]; ++q)
          atomicAdd(reinterpret_cast<unsigned long long*>(&delta[qh[q]]), dec);
      }
    }
    greedy_bar();
#pragma unroll
    for (int j = 0; j < kGreedyOwn; ++j) {
      const int i = t + j * kGreedyThreads;
      if (i < n) {
        m[j] += delta[i];
        delta[i] = 0;
      }
    }
    c_upd += clock64() - c1;
  }
  if (t == 0) g_greedy_cycles[0] = c_arg, g_greedy_cycles[1] = c_upd;
}

// Packed-key rounds.  The caller guarantees hid[] ascending (index order = id order), every
// cost >= 0 and every initial marginal < 2^(32 - idbits): the lexicographic (marginal, id) key
// then packs into one u32, key = (marginal << idbits) | index, and stays exact as marginals only
// shrink.  Keys live in shared memory: each argmin level is one redux.sync.min, and the winner's
// evictions subtract (cost << idbits) straight from the listed handles' keys with u32 atomics
// (no per-owner fold pass).  Taken handles are masked by their owner's `live` bits.
__device__ void greedy_block_packed(int n, const int* hid, Refs R, const int* rref, const int64_t* cost,
                                    int k, const int64_t* marg0, unsigned* skey, int* ev, const int* qoff,
                                    const int* qh, int* out, int idbits, int qmax) {
  constexpr int NW = kGreedyThreads / 32;
  __shared__ unsigned w_key[NW];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const unsigned idmask = (1u << idbits) - 1u;
  unsigned live = 0;
#pragma unroll
  for (int j = 0; j < kGreedyOwn; ++j) {
    const int i = t + j * kGreedyThreads;
    if (i < n) {
      live |= 1u << j;
      skey[i] = ((unsigned)marg0[i] << idbits) | (unsigned)i;
    }
  }
  greedy_bar();
  long long c_arg = 0, c_upd = 0;
  for (int round = 0; round < k; ++round) {
    const long long c0 = clock64();
    unsigned v = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < kGreedyOwn; ++j)
      if ((live >> j) & 1u) v = min(v, skey[t + j * kGreedyThreads]);
    v = __reduce_min_sync(kFull, v);
    if (lane == 0) w_key[wid] = v;
    greedy_bar();
    v = __reduce_min_sync(kFull, lane < NW ? w_key[lane] : 0xFFFFFFFFu);
    const int best = (int)(v & idmask);
    const long long c1 = clock64();
    c_arg += c1 - c0;
#pragma unroll
    for (int j = 0; j < kGreedyOwn; ++j)
      if (best == t + j * kGreedyThreads) live &= ~(1u << j);
    if (t == 0) out[round] = hid[best];
    if (qmax > 0) {
      // rows are distinct within a handle: thread t takes listing t / qmax of the winner and the
      // (t % qmax)-th handle listing that request -- one dependent chain per (request, handle)
      // instead of a serial loop per request; `ev` is read here and set after the barrier
      const int b0 = R.begin(best), nl = R.end(best) - b0;
      for (int x = t; x < nl * qmax; x += kGreedyThreads) {
        const int r = rref[b0 + x / qmax];
        const int q = qoff[r] + x % qmax;
        if (q < qoff[r + 1] && !ev[r]) atomicSub(&skey[qh[q]], (unsigned)cost[r] << idbits);
      }
      greedy_bar();
      for (int x = t; x < nl; x += kGreedyThreads) ev[rref[b0 + x]] = 1;
    } else {
      for (int e = R.begin(best) + t; e < R.end(best); e += kGreedyThreads) {
        const int r = rref[e];
        if (atomicExch(&ev[r], 1) == 0) {
          const unsigned dec = (unsigned)cost[r] << idbits;
          for (int q = qoff[r]; q < qoff[r + 1]; ++q) atomicSub(&skey[qh[q]], dec);
        }
      }
      greedy_bar();
    }
    c_upd += clock64() - c1;
  }
  if (t == 0) g_greedy_cycles[0] = c_arg, g_greedy_cycles[1] = c_upd;
}

// Packed-key rounds in ONE warp (n <= 1024): lane l owns keys l + 32 j (j < 32) and their taken
// bits in a register; a round is 32 shared loads + one CREDUX per lane, the winner's evictions
// spread over the lanes, and __syncwarp instead of CTA barriers (~2x fewer cycles per round than
// the 8-warp form, which pays two named barriers per round).
__device__ void greedy_warp_packed(int n, const int* hid, Refs R, const int* rref, const int64_t* cost, int k,
                                   const int64_t* marg0, unsigned* skey, int* ev, const int* qoff, const int* qh,
                                   int* out, int idbits, int qmax) {
  const int lane = threadIdx.x & 31;
  const unsigned idmask = (1u << idbits) - 1u;
  unsigned live = 0;
  for (int j = 0; j < 32; ++j) {
    const int i = lane + 32 * j;
    if (i < n) {
      live |= 1u << j;
      skey[i] = ((unsigned)marg0[i] << idbits) | (unsigned)i;
    }
  }
  __syncwarp();
  long long c_arg = 0, c_upd = 0;
  for (int round = 0; round < k; ++round) {
    const long long c0 = clock64();
    unsigned v = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if ((live >> j) & 1u) v = min(v, skey[lane + 32 * j]);
    v = __reduce_min_sync(kFull, v);
    const int best = (int)(v & idmask);
    const long long c1 = clock64();
    c_arg += c1 - c0;
    if ((best & 31) == lane) live &= ~(1u << (best >> 5));
    if (lane == 0) out[round] = hid[best];
    const int b0 = R.begin(best), nl = R.end(best) - b0;
    if (qmax > 0) {  // distinct requests per handle: one (request, listing handle) per lane
      for (int x = lane; x < nl * qmax; x += 32) {
        const int r = rref[b0 + x / qmax];
        const int q = qoff[r] + x % qmax;
        if (q < qoff[r + 1] && !ev[r]) atomicSub(&skey[qh[q]], (unsigned)cost[r] << idbits);
      }
      __syncwarp();
      for (int x = lane; x < nl; x += 32) ev[rref[b0 + x]] = 1;
    } else {
      for (int e = b0 + lane; e < b0 + nl; e += 32) {
        const int r = rref[e];
        if (atomicExch(&ev[r], 1) == 0) {
          const unsigned dec = (unsigned)cost[r] << idbits;
          for (int q = qoff[r]; q < qoff[r + 1]; ++q) atomicSub(&skey[qh[q]], dec);
        }
      }
    }
    __syncwarp();
    c_upd += clock64() - c1;
  }
  if (lane == 0) g_greedy_cycles[0] = c_arg, g_greedy_cycles[1] = c_upd;
}

// Same rounds CTA-wide over global arrays (instances larger than shared memory).
__device__ void greedy_cta(int n, const int* hid, Refs R, const int* rref, const int64_t* cost,
                           int k, int64_t* marg, int* taken, int* ev, const int* qoff, const int* qh,
                           int* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) taken[i] = 0;
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
    for (int e = R.begin(best) + threadIdx.x; e < R.end(best); e += blockDim.x) {
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

// Greedy dispatch.  When the instance fits (n <= 2048 handles, <= 4096 listings) it is
// re-indexed into shared memory -- handles, CSR listings over a dense request index, costs,
// the reverse index and the eviction flags -- and the rounds run in warp 0 with every access
// on-chip.  Larger instances run CTA-wide over global scratch.
__device__ void greedy_select(int n, const int* hid_g, Refs R, const int* rref, int m,
                              const int64_t* cost, int k, int64_t* marg_g, int* taken_g, int* ev,
                              int* qoff, int* qcnt, int* qh, int* out, unsigned char* smem,
                              int* dense = nullptr) {
  if (threadIdx.x == 0) g_select_ns[0] = (long long)globaltimer_ns();
  // this thread's handle's listing range, read once: inside the loops below the compiler cannot
  // hoist Refs' global words (map, counts) past the atomics, so it would re-read them per listing
  const int tb = (int)threadIdx.x < n ? R.begin(threadIdx.x) : 0;
  const int te = (int)threadIdx.x < n ? R.end(threadIdx.x) : 0;
  auto rb = [&](int i) { return i == (int)threadIdx.x ? tb : R.begin(i); };
  auto re = [&](int i) { return i == (int)threadIdx.x ? te : R.end(i); };
  int nnz_local = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) nnz_local += re(i) - rb(i);
  const int nnz = block_sum(nnz_local);
  if (n <= kSmemHandles && nnz <= kSmemListings) {
    int m2 = 0;
    if (dense) {
      // dense request index: the first listing of each referenced row claims the next id
      // (`dense` is -1 everywhere between calls; the ids are reset below through qoff)
      __shared__ int s_m2;
      if (threadIdx.x == 0) s_m2 = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int e = rb(i), ee = re(i); e < ee; ++e) {
          const int r = rref[e];
          if (atomicCAS(&dense[r], -1, -2) == -1) {
            const int d = atomicAdd(&s_m2, 1);
            dense[r] = d;
            qoff[d] = r;  // dense id -> row, for the reset
          }
        }
      __syncthreads();
      m2 = s_m2;
      qcnt = dense;
      if (threadIdx.x == 0) g_select_ns[1] = (long long)globaltimer_ns();
    } else {
      // dense request index over the referenced requests (qcnt: flag -> dense id)
      for (int r = threadIdx.x; r < m; r += blockDim.x) qcnt[r] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int e = rb(i), ee = re(i); e < ee; ++e) qcnt[rref[e]] = 1;
      __syncthreads();
      for (int base = 0; base < m; base += blockDim.x) {
        const int r = base + threadIdx.x;
        const int f = r < m ? qcnt[r] : 0;
        int tot;
        const int ex = block_excl_scan(f, tot);
        if (r < m) qcnt[r] = f ? m2 + ex : -1;
        m2 += tot;
      }
    }
    // shared-memory carve-up
    int64_t* marg = reinterpret_cast<int64_t*>(smem);
    int64_t* cost2 = marg + kSmemHandles;
    int* hid = reinterpret_cast<int*>(cost2 + kSmemListings);
    int* roff = hid + kSmemHandles;
    int* rr = roff + kSmemHandles + 1;
    int* qoff2 = rr + kSmemListings;
    int* qh2 = qoff2 + kSmemListings + 1;
    int* ev2 = qh2 + kSmemListings;
    int* qcnt2 = ev2 + kSmemListings;
    unsigned char* taken = reinterpret_cast<unsigned char*>(qcnt2 + kSmemListings);
    int carry = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const int c = i < n ? re(i) - rb(i) : 0;
      int tot;
      const int ex = block_excl_scan(c, tot);
      if (i < n) {
        roff[i] = carry + ex;
        hid[i] = hid_g[i];
        taken[i] = 0;
      }
      carry += tot;
    }
    if (threadIdx.x == 0) roff[n] = carry;
    for (int d = threadIdx.x; d < m2; d += blockDim.x) {
      ev2[d] = 0;
      qcnt2[d] = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int o = roff[i];
      for (int e = rb(i), ee = re(i); e < ee; ++e, ++o) {
        const int r = rref[e];
        const int d = qcnt[r];
        rr[o] = d;
        cost2[d] = cost[r];
        atomicAdd(&qcnt2[d], 1);
      }
    }
    __syncthreads();
    carry = 0;
    for (int base = 0; base < m2; base += blockDim.x) {
      const int d = base + threadIdx.x;
      const int c = d < m2 ? qcnt2[d] : 0;
      int tot;
      const int ex = block_excl_scan(c, tot);
      if (d < m2) qoff2[d] = carry + ex;
      carry += tot;
    }
    if (threadIdx.x == 0) qoff2[m2] = carry;
    for (int d = threadIdx.x; d < m2; d += blockDim.x) qcnt2[d] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int64_t s = 0;
      for (int o = roff[i]; o < roff[i + 1]; ++o) {
        const int d = rr[o];
        s += cost2[d];
        qh2[qoff2[d] + atomicAdd(&qcnt2[d], 1)] = i;
      }
      marg[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) g_select_ns[2] = (long long)globaltimer_ns();
    // packed-key rounds when ids ascend, costs are >= 0 and the marginals fit the key
    int idbits = 1;
    while ((1 << idbits) < n) ++idbits;
    const int64_t lim = (int64_t)1 << (32 - idbits);
    int bad = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      bad |= (marg[i] >= lim) | (i + 1 < n && hid[i] >= hid[i + 1]);
    for (int d = threadIdx.x; d < m2; d += blockDim.x) bad |= cost2[d] < 0;
    const bool packed = __syncthreads_or(bad) == 0;
    // flat update rounds need distinct requests within every handle's listings (the fused
    // path's rows are deduplicated; host instances may repeat a request on a handle)
    int dup = 0, qm = 0;
    if (!dense)  // the fused path's rows come from warp_distinct_rows: no quadratic check
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        for (int o = roff[i]; o < roff[i + 1]; ++o)
          for (int o2 = roff[i]; o2 < o; ++o2) dup |= rr[o2] == rr[o];
    for (int d = threadIdx.x; d < m2; d += blockDim.x) qm = max(qm, qoff2[d + 1] - qoff2[d]);
    __shared__ int s_qmax;
    if (threadIdx.x == 0) s_qmax = 0;
    const bool has_dup = __syncthreads_or(dup) != 0;
    if (qm) atomicMax(&s_qmax, qm);
    __syncthreads();
    const int qmax = has_dup ? 0 : s_qmax;
    const Refs Rs{roff, nullptr, 0};
    unsigned* skey = reinterpret_cast<unsigned*>(taken + kSmemHandles);
    if (threadIdx.x == 0) g_select_ns[3] = (long long)globaltimer_ns();
    if (packed && n <= 1024) {
      if (threadIdx.x < 32) greedy_warp_packed(n, hid, Rs, rr, cost2, k, marg, skey, ev2, qoff2, qh2, out, idbits, qmax);
    } else if (threadIdx.x < kGreedyThreads) {
      if (packed) greedy_block_packed(n, hid, Rs, rr, cost2, k, marg, skey, ev2, qoff2, qh2, out, idbits, qmax);
      else greedy_block(n, hid, Rs, rr, cost2, k, marg, ev2, qoff2, qh2, out);
    }
    if (dense)
      for (int d = threadIdx.x; d < m2; d += blockDim.x) dense[qoff[d]] = -1;  // back to all -1
    __syncthreads();
    if (threadIdx.x == 0) g_select_ns[4] = (long long)globaltimer_ns();
  } else {
    build_instance_index(n, R, rref, m, cost, marg_g, qoff, qcnt, qh, ev);
    greedy_cta(n, hid_g, R, rref, cost, k, marg_g, taken_g, ev, qoff, qh, out);
    __syncthreads();
    for (int r = threadIdx.x; r < m; r += blockDim.x) ev[r] = 0;  // apply re-marks rows
  }
}

// FIFO (reclaim.cpp:69-83): the k oldest by (mapped_at, id); rank selection.
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

// Exhaustive oracle (reclaim.cpp:85-126), n <= 20: subsets by lexicographic rank over the
// ascending ids; cost(S) = sum of cost[r] over requests whose handle mask meets S; the
// first minimum in rank order wins.
__device__ void oracle_core(int n, const int* sorted_ids, int m, const unsigned* hmask,
                            const int64_t* cost, int k, int* out) {
  __shared__ long long binom[21][21];
  if (threadIdx.x == 0) {
    for (int a = 0; a <= 20; ++a)
      for (int b = 0; b <= 20; ++b) binom[a][b] = b == 0 ? 1 : 0;
    for (int a = 1; a <= 20; ++a)
      for (int b = 1; b <= a; ++b) binom[a][b] = binom[a - 1][b - 1] + binom[a - 1][b];
  }
  __syncthreads();
  const long long total = binom[n][k];
  ArgMin best{0, 0, -1};
  for (long long rnk = threadIdx.x; rnk < total; rnk += blockDim.x) {
    unsigned mask = 0;
    long long rr = rnk;
    int start = 0;
    for (int pos = 0; pos < k; ++pos)
      for (int c = start; c < n; ++c) {
        const long long cnt = binom[n - c - 1][k - pos - 1];
        if (rr < cnt) {
          mask |= 1u << c;
          start = c + 1;
          break;
        }
        rr -= cnt;
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

// Warp-wide ascending sort of n (key, payload) pairs in place, any n: the one-direction
// bitonic network (mirror compare in the first step of each merge, then half-cleaners), with
// the missing tail treated as +inf -- a pair whose upper index is >= n never swaps.
__device__ __forceinline__ void warp_sort_asc(uint64_t* key, int* pay, int n, int lane) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (N >> 1); i += 32) {
        const int blk = i / stride, off = i % stride;
        int lo = blk * 2 * stride + off, hi = lo + stride;
        if (stride == (size >> 1)) hi = (lo | (size - 1)) - off;  // mirror partner
        if (hi < n) {
          const uint64_t a = key[lo], b = key[hi];
          if (a > b) {
            key[lo] = b;
            key[hi] = a;
            const int t = pay[lo];
            pay[lo] = pay[hi];
            pay[hi] = t;
          }
        }
      }
      __syncwarp();
    }
  }
}

// apply_reclaim (memory.cpp:155-180) for ids[0..k).  Converts the valid prefix (the
// reference mutates handle by handle and throws at the first bad one), reports the
// invalidated pages sorted per request, and -- if the whole list was valid -- releases the
// residual pages of every evicted request.  Writes res_* and the mirror counts.
// `trusted`: ids are distinct offline handles by construction (the fused path's own picks), so
// the reference's per-handle validation (memory.cpp:158-161) cannot fail and is skipped.
__device__ void apply_core(const PoolDev& P, const int* ids, int k, int64_t t, unsigned char* smem,
                           bool trusted = false) {
  __shared__ int s_bad, s_nt, s_freed;
  if (threadIdx.x == 0) {
    g_apply_ns[5] = (long long)globaltimer_ns();
    s_bad = k;
    s_nt = 0;
    s_freed = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k && !trusted; i += blockDim.x) {
    const int h = ids[i];
    bool bad = h < 0 || h >= P.H || P.hstate[h] != kOffline;
    for (int j = 0; j < i && !bad; ++j) bad = ids[j] == h;
    if (bad) atomicMin(&s_bad, i);
  }
  __syncthreads();
  const int b = s_bad;
  if (threadIdx.x == 0) g_apply_ns[6] = (long long)globaltimer_ns();
  if (threadIdx.x == 0 && b < k) {
    const int h = ids[b];
    if (h < 0 || h >= P.H) set_err(P, kErrOutOfRange, kDetApplyRange, h);
    else set_err(P, kErrLogic, kDetNotOffline, h);
  }
  // Clear the chosen handles, collecting (row, logical page, physical page, block).
  // Fast path (b * S <= 8192): the chosen handles in ascending id order, slot tuples at
  // idx = position * S + slot in shared memory.  The report order inside a request is
  // (logical, physical) with logical = h * S + lid, i.e. by handle, then by (lid, slot) inside the
  // handle -- so each page is ranked among its row's pages on its own handle (an O(S) scan of
  // that handle's tuples) and the row's first slot there records one "pair" (row, handle
  // position, count); sorting the few pairs by (request rank, handle position) and a scan of
  // their counts gives every page its report position without sorting the pages.
  constexpr int kFastT = 8192, kFastB = 1024, kPairCap = 2048, kPer = kFastT / kNT;
  // packed per-slot key (row << 16 | lid << 8 | slot) needs rows < 2^16 and S <= 256
  const bool fast = (int64_t)b * P.S <= kFastT && b <= kFastB && P.R < 65535 && P.S <= 256;
  int* hs = reinterpret_cast<int*>(smem);  // [kFastB] chosen handles, ascending
  int* trow = hs + kFastB;                 // [kFastT] slot tuples: row (-1 = empty slot)
  int* tkey = trow + kFastT;               //   row << 16 | logical id << 8 | slot (rank key)
  int* tpid = tkey + kFastT;               //   pair id (on the row's first slot of the handle)
  int* prow = tpid + kFastT;               // [kPairCap] pair: row
  int* phi = prow + kPairCap;              //   handle position in ascending order
  int* pcnt = phi + kPairCap;              //   pages of the row on that handle
  int* ppos = pcnt + kPairCap;             //   report position of the pair's first page
  int* sev = ppos + kPairCap;              // [kPairCap] evicted rows (first pair that saw them)
  int* pord = sev + kPairCap;              // [kPairCap] pairs in (request rank, handle) order
  __shared__ int s_np, s_ne;
  const int nslot = b * P.S;
  if (fast) {
    if (threadIdx.x == 0) s_np = 0, s_ne = 0;
    for (int i = threadIdx.x; i < b; i += blockDim.x) {  // ids are distinct (validated)
      const int h = ids[i];
      int pos = 0;
      for (int j = 0; j < b; ++j) pos += ids[j] < h;
      hs[pos] = h;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nslot; idx += blockDim.x) {  // read + clear every chosen slot
      const int hi = idx / P.S;
      const int64_t p = (int64_t)hs[hi] * P.S + (idx - hi * P.S);
      const int row = P.slot_row[p];
      trow[idx] = row;
      tkey[idx] = -1;  // empty: row field 0xffff never matches a row < 65535
      if (row < 0) continue;
      const int blk = P.slot_blk[p];
      tkey[idx] = (row << 16) | (P.slot_lid[p] << 8) | (idx - hi * P.S);
      P.s_pay[idx] = blk;
      atomicAdd(&s_nt, 1);
      P.bt[(int64_t)row * P.P + blk] = P.quarantine;  // quarantine remap
      atomicSub(&P.row_npages[row], 1);
      P.slot_row[p] = -1;
      P.slot_lid[p] = -1;
      P.slot_blk[p] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) g_apply_ns[7] = (long long)globaltimer_ns();
    if (P.S <= 64) {
      // one warp per handle: bitonic sort of its <= 64 packed keys (row, lid, slot) in registers
      // (position p = lane + 32 * i holds a_i), then each page's rank inside its row's segment
      // = p - segment start (ballots of the segment starts); the segment start owns the pair
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);  // lanes <= me
      for (int hi = wid; hi < b; hi += nw) {
        const int base = hi * P.S;
        unsigned a0 = lane < P.S ? (unsigned)tkey[base + lane] : 0xFFFFFFFFu;
        unsigned a1 = lane + 32 < P.S ? (unsigned)tkey[base + lane + 32] : 0xFFFFFFFFu;
#pragma unroll
        for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
          for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // k == 64: partner is the other register of the same lane, ascending
              const unsigned lo = min(a0, a1), hi2 = max(a0, a1);
              a0 = lo, a1 = hi2;
            } else {
              const unsigned b0 = __shfl_xor_sync(kFull, a0, j), b1 = __shfl_xor_sync(kFull, a1, j);
              const bool lower = (lane & j) == 0;
              a0 = (lower == ((lane & k) == 0)) ? min(a0, b0) : max(a0, b0);
              a1 = (lower == (((lane + 32) & k) == 0)) ? min(a1, b1) : max(a1, b1);
            }
          }
        }
        const unsigned r0 = a0 >> 16, r1 = a1 >> 16;
        unsigned p0 = __shfl_up_sync(kFull, r0, 1), p1 = __shfl_up_sync(kFull, r1, 1);
        const unsigned tail0 = __shfl_sync(kFull, r0, 31);
        if (lane == 0) p0 = ~r0, p1 = tail0;
        const unsigned m0 = __ballot_sync(kFull, p0 != r0), m1 = __ballot_sync(kFull, p1 != r1);
        // segment start / next start of each position
        const int st0 = 31 - __clz(m0 & le);  // lane 0 is always a start
        const unsigned mm1 = m1 & le;
        const int st1 = mm1 ? 32 + 31 - __clz(mm1) : 31 - __clz(m0);
        const unsigned n0m = m0 & ~le, n1m = m1 & ~le;
        const int nx0 = n0m ? __ffs(n0m) - 1 : (m1 ? 32 + __ffs(m1) - 1 : 64);
        const int nx1 = n1m ? 32 + __ffs(n1m) - 1 : 64;
        int pid0 = -1, pid1 = -1;
        const bool v0 = r0 != 0xFFFFu, v1 = r1 != 0xFFFFu;  // 0xffff: empty slot
        if (v0 && st0 == lane) {
          pid0 = atomicAdd(&s_np, 1);
          if (pid0 < kPairCap) prow[pid0] = (int)r0, phi[pid0] = hi, pcnt[pid0] = nx0 - st0;
          if (atomicExch(&P.s_ev[r0], 1) == 0) {
            const int e = atomicAdd(&s_ne, 1);
            if (e < kPairCap) sev[e] = (int)r0;
          }
        }
        if (v1 && st1 == lane + 32) {
          pid1 = atomicAdd(&s_np, 1);
          if (pid1 < kPairCap) prow[pid1] = (int)r1, phi[pid1] = hi, pcnt[pid1] = nx1 - st1;
          if (atomicExch(&P.s_ev[r1], 1) == 0) {
            const int e = atomicAdd(&s_ne, 1);
            if (e < kPairCap) sev[e] = (int)r1;
          }
        }
        // each page takes its segment start's pair id (start lane / register by position)
        const int q0 = __shfl_sync(kFull, pid0, st0 & 31), q0b = __shfl_sync(kFull, pid1, st0 & 31);
        const int q1 = __shfl_sync(kFull, pid0, st1 & 31), q1b = __shfl_sync(kFull, pid1, st1 & 31);
        if (v0) P.s_key[base + (a0 & 0xFFu)] = ((uint64_t)(uint32_t)(st0 < 32 ? q0 : q0b) << 32) | (uint32_t)(lane - st0);
        if (v1) P.s_key[base + (a1 & 0xFFu)] = ((uint64_t)(uint32_t)(st1 < 32 ? q1 : q1b) << 32) | (uint32_t)(lane + 32 - st1);
      }
      __syncthreads();
      if (threadIdx.x == 0) g_apply_ns[8] = (long long)globaltimer_ns();
    } else {
      int r_first[kPer], r_wr[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int idx = threadIdx.x + j * kNT;
        r_first[j] = -1;
        const int row = idx < nslot ? trow[idx] : -1;
        if (row < 0) continue;
        const int base = (idx / P.S) * P.S, s = idx - base;
        // rank among the row's pages on this handle by (lid, slot): one packed key per slot, so the
        // scan is branch-free (empty slots hold key 0xffffffff and never match)
        const unsigned ks = (unsigned)tkey[idx], rk = (unsigned)row;
        int cnt = 0, wr = 0, first = s;
#pragma unroll 8
        for (int q = 0; q < P.S; ++q) {
          const unsigned kq = (unsigned)tkey[base + q];
          const bool same = (kq >> 16) == rk;
          cnt += same;
          wr += same && kq < ks;
          first = same && q < first ? q : first;
        }
        r_first[j] = base + first;
        r_wr[j] = wr;
        if (first == s) {  // the row's first slot on this handle owns the pair
          const int pid = atomicAdd(&s_np, 1);
          tpid[idx] = pid;
          if (pid < kPairCap) prow[pid] = row, phi[pid] = base / P.S, pcnt[pid] = cnt;
          if (atomicExch(&P.s_ev[row], 1) == 0) {
            const int e = atomicAdd(&s_ne, 1);
            if (e < kPairCap) sev[e] = row;
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) g_apply_ns[8] = (long long)globaltimer_ns();
#pragma unroll
      for (int j = 0; j < kPer; ++j)
        if (r_first[j] >= 0)
          P.s_key[threadIdx.x + j * kNT] = ((uint64_t)(uint32_t)tpid[r_first[j]] << 32) | (uint32_t)r_wr[j];
    }
    if (s_np > kPairCap || s_ne > kPairCap) {
      // too many pairs for the on-chip report: compact the tuples for the general sort below
      __shared__ int s_cmp;
      if (threadIdx.x == 0) s_cmp = 0;
      __syncthreads();
      for (int idx = threadIdx.x; idx < nslot; idx += blockDim.x) {
        const int row = trow[idx];
        if (row < 0) continue;
        const int hi = idx / P.S;
        const int pos = atomicAdd(&s_cmp, 1);
        P.s_qh[pos] = row;
        P.s_rref[pos] = hs[hi] * P.S + ((tkey[idx] >> 8) & 0xff);
        P.s_tphys[pos] = hs[hi] * P.S + (idx - hi * P.S);
        P.s_tblk[pos] = P.s_pay[idx];
      }
    }
  } else {
    const int64_t nslots = (int64_t)b * P.S;
    for (int64_t idx = threadIdx.x; idx < nslots; idx += blockDim.x) {
      const int h = ids[idx / P.S];
      const int64_t p = (int64_t)h * P.S + idx % P.S;
      const int row = P.slot_row[p];
      if (row < 0) continue;
      const int pos = atomicAdd(&s_nt, 1);
      const int blk = P.slot_blk[p];
      P.s_qh[pos] = row;
      P.s_rref[pos] = (int)((int64_t)h * P.S + P.slot_lid[p]);
      P.s_tphys[pos] = (int)p;
      P.s_tblk[pos] = blk;
      P.s_ev[row] = 1;
      P.bt[(int64_t)row * P.P + blk] = P.quarantine;  // quarantine remap
      atomicSub(&P.row_npages[row], 1);
      P.slot_row[p] = -1;
      P.slot_lid[p] = -1;
      P.slot_blk[p] = -1;
    }
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
  if (threadIdx.x == 0) g_apply_ns[0] = (long long)globaltimer_ns();
  int carry = 0, ne;
  if (fast && s_np <= kPairCap && s_ne <= kPairCap) {
    ne = s_ne;
    const int np = s_np;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {  // evicted rows ranked by request id
      const int row = sev[e];
      const int64_t req = P.row_req[row];
      int rank = 0;
      for (int f = 0; f < ne; ++f) rank += P.row_req[sev[f]] < req;
      P.s_rank[row] = rank;
      P.s_evrows[e] = row;
      P.s_ev[row] = 0;
      P.res_evicted[rank] = req;
      P.res_ev_pbytes[rank] = P.row_pbytes[row] ? P.row_pbytes[row] : P.page_bytes;
    }
    if (threadIdx.x == 0) P.res_inv_off[ne] = nt;
    __syncthreads();
    if (threadIdx.x == 0) g_apply_ns[1] = (long long)globaltimer_ns();
    for (int j = threadIdx.x; j < np; j += blockDim.x) {  // pairs by (request rank, handle position)
      const int kj = (P.s_rank[prow[j]] << 11) | phi[j];
      int pos = 0;
      for (int i = 0; i < np; ++i) pos += ((P.s_rank[prow[i]] << 11) | phi[i]) < kj;
      pord[pos] = j;
    }
    __syncthreads();
    for (int base = 0; base < np; base += blockDim.x) {
      const int j = base + threadIdx.x;
      const int pr = j < np ? pord[j] : 0;
      int tot;
      const int ex = block_excl_scan(j < np ? pcnt[pr] : 0, tot);
      if (j < np) {
        ppos[pr] = carry + ex;
        const int rank = P.s_rank[prow[pr]];
        if (j == 0 || P.s_rank[prow[pord[j - 1]]] != rank) P.res_inv_off[rank] = carry + ex;
      }
      carry += tot;
    }
    int64_t bcarry = 0;
    int custom = 0;
    for (int base = 0; base < ne; base += blockDim.x) {  // destination byte layout of the copy
      const int e = base + threadIdx.x;
      const int c = e < ne ? P.res_inv_off[e + 1] - P.res_inv_off[e] : 0;
      const int64_t pb = e < ne ? P.res_ev_pbytes[e] : 0;
      int64_t btot;
      const int64_t bex = block_excl_scan64((int64_t)c * pb, btot);
      custom |= __syncthreads_or(e < ne && pb != P.page_bytes);
      if (e < ne) P.res_ev_base[e] = bcarry + bex;
      bcarry += btot;
    }
    if (threadIdx.x == 0) {
      P.res_ev_base[ne] = bcarry;
      P.mirror->copy_bytes = bcarry;
      P.mirror->copy_custom = custom;
    }
    for (int idx = threadIdx.x; idx < nslot; idx += blockDim.x) {
      if (trow[idx] < 0) continue;
      const uint64_t kv = P.s_key[idx];
      const int pos = ppos[kv >> 32] + (int)(uint32_t)kv;
      const int hi = idx / P.S, h = hs[hi];
      P.res_pages[pos] = (int64_t)h * P.S + ((tkey[idx] >> 8) & 0xff);
      P.res_phys[pos] = h * P.S + (idx - hi * P.S);
      P.res_blk[pos] = P.s_pay[idx];
    }
  } else {
  // evicted rows, then their rank by request id
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
  ne = carry;
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const int row = P.s_evrows[e];
    const int64_t req = P.row_req[row];
    int rank = 0;
    for (int f = 0; f < ne; ++f) rank += P.row_req[P.s_evrows[f]] < req;
    P.s_rank[row] = rank;
    P.res_evicted[rank] = req;
    P.res_ev_pbytes[rank] = P.row_pbytes[row] ? P.row_pbytes[row] : P.page_bytes;
  }
  __syncthreads();
  if (threadIdx.x == 0) g_apply_ns[1] = (long long)globaltimer_ns();
  // Report order (request ascending, then logical page, then physical page): a counting sort
  // by request rank straight into the CSR offsets, then each request's bucket is sorted by
  // one warp (no CTA barriers).  Key = page << 24 | phys, payload = block index.
  const bool in_smem = nt <= kSmemTuples && ne <= kSmemTuples;
  uint64_t* key = in_smem ? reinterpret_cast<uint64_t*>(smem) : P.s_key;
  int* pay = in_smem ? reinterpret_cast<int*>(key + kSmemTuples) : P.s_pay;
  int* bcnt = in_smem ? pay + kSmemTuples : P.s_qcnt;  // [ne] per-request cursor
  for (int e = threadIdx.x; e < ne; e += blockDim.x) bcnt[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) atomicAdd(&bcnt[P.s_rank[P.s_qh[i]]], 1);
  __syncthreads();
  carry = 0;
  int64_t bcarry = 0;
  int custom = 0;
  for (int base = 0; base < ne; base += blockDim.x) {
    const int e = base + threadIdx.x;
    const int c = e < ne ? bcnt[e] : 0;
    int tot;
    const int ex = block_excl_scan(c, tot);
    // destination byte layout of the copy: request e's pages at res_ev_base[e], pb bytes each
    const int64_t pb = e < ne ? P.res_ev_pbytes[e] : 0;
    int64_t btot;
    const int64_t bex = block_excl_scan64((int64_t)c * pb, btot);
    custom |= __syncthreads_or(e < ne && pb != P.page_bytes);
    if (e < ne) {
      P.res_inv_off[e] = carry + ex;
      P.res_ev_base[e] = bcarry + bex;
    }
    carry += tot;
    bcarry += btot;
  }
  if (threadIdx.x == 0) {
    P.res_inv_off[ne] = nt;
    P.res_ev_base[ne] = bcarry;
    P.mirror->copy_bytes = bcarry;
    P.mirror->copy_custom = custom;
  }
  for (int e = threadIdx.x; e < ne; e += blockDim.x) bcnt[e] = 0;
  __syncthreads();
  int* segof = in_smem ? bcnt + kSmemTuples : nullptr;  // [nt] request rank of each position
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    const int rank = P.s_rank[P.s_qh[i]];
    const int pos = P.res_inv_off[rank] + atomicAdd(&bcnt[rank], 1);
    key[pos] = ((uint64_t)(uint32_t)P.s_rref[i] << 24) | (uint64_t)(uint32_t)P.s_tphys[i];
    pay[pos] = P.s_tblk[i];
    if (segof) segof[pos] = rank;
  }
  // Longest request segment: up to kRankSeg the order inside each segment comes from ranks
  // (every element counts the smaller keys of its segment -- keys are unique: the physical page
  // breaks logical-id ties), which keeps all 1024 threads busy; a warp-per-segment sort left 31
  // warps waiting at the barrier for the warp holding the longest segments (~17 us at k = 36).
  int seg_local = 0;
  for (int e = threadIdx.x; e < ne; e += blockDim.x)
    seg_local = max(seg_local, P.res_inv_off[e + 1] - P.res_inv_off[e]);
  __shared__ int s_seg;
  if (threadIdx.x == 0) s_seg = 0;
  __syncthreads();
  if (seg_local) atomicMax(&s_seg, seg_local);
  __syncthreads();
  constexpr int kRankSeg = 1024;
  if (s_seg <= kRankSeg) {
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      int lo = 0, hi = ne - 1;  // segment of position i
      if (segof) {
        lo = segof[i];
      } else {
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (P.res_inv_off[mid] <= i) lo = mid;
          else hi = mid - 1;
        }
      }
      const int o = P.res_inv_off[lo], end = P.res_inv_off[lo + 1];
      const uint64_t kv = key[i];
      int r = 0;
      for (int j = o; j < end; ++j) r += key[j] < kv;
      P.res_pages[o + r] = (int64_t)(kv >> 24);
      P.res_phys[o + r] = (int)(kv & 0xffffffull);
      P.res_blk[o + r] = pay[i];
    }
  } else {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int e = wid; e < ne; e += nw) {
      const int o = P.res_inv_off[e], n = P.res_inv_off[e + 1] - o;
      warp_sort_asc(key + o, pay + o, n, lane);
      for (int i = lane; i < n; i += 32) {
        const uint64_t kv = key[o + i];
        P.res_pages[o + i] = (int64_t)(kv >> 24);
        P.res_phys[o + i] = (int)(kv & 0xffffffull);
        P.res_blk[o + i] = pay[o + i];
      }
    }
  }
  }
  __syncthreads();
  if (threadIdx.x == 0) g_apply_ns[2] = (long long)globaltimer_ns();
  if (b == k) {
    // Residual pages of evicted requests are plain frees (memory.cpp:176), flattened over
    // (row, block) so the dependent loads of all rows overlap.
    // (row, block-offset) tables in shared memory when they fit (the sort buffers are free now)
    const bool sm_rows = ne + 1 <= kSmemTuples;
    int* qoff = sm_rows ? reinterpret_cast<int*>(smem) : P.s_qoff;
    int* rows = sm_rows ? qoff + kSmemTuples : P.s_evrows;
    const bool sm_dec = sm_rows && P.H <= kSmemTuples;
    int* hdec = rows + kSmemTuples;  // [H] per-handle decrements (sm_dec only)
    if (sm_dec)
      for (int h = threadIdx.x; h < P.H; h += blockDim.x) hdec[h] = 0;
    carry = 0;
    for (int base = 0; base < ne; base += blockDim.x) {
      const int e = base + threadIdx.x;
      const int row = e < ne ? P.s_evrows[e] : 0;
      const int c = e < ne ? P.row_nblk[row] : 0;
      int tot;
      const int ex = block_excl_scan(c, tot);
      if (e < ne) {
        qoff[e] = carry + ex;
        rows[e] = row;
      }
      carry += tot;
    }
    if (threadIdx.x == 0) qoff[ne] = carry;
    __syncthreads();
    const int total = carry;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      int lo = 0, hi = ne - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (qoff[mid] <= idx) lo = mid;
        else hi = mid - 1;
      }
      const int row = rows[lo];
      const int64_t bi = (int64_t)row * P.P + (idx - qoff[lo]);
      const int p = P.bt[bi];
      if (p < 0 || p >= P.quarantine) continue;
      P.bt[bi] = P.quarantine;
      if (P.slot_row[p] != row) continue;
      P.slot_row[p] = -1;
      P.slot_lid[p] = -1;
      P.slot_blk[p] = -1;
      const int h = p / P.S;
      if (sm_dec) atomicAdd(&hdec[h], 1);  // aggregated per handle on chip
      else if (atomicSub(&P.hused[h], 1) == 1) {
        P.hstate[h] = kFree;
        atomicAdd(&s_freed, 1);
      }
    }
    __syncthreads();
    if (sm_dec) {  // one thread per handle applies its decrement; emptied handles go free
      for (int h = threadIdx.x; h < P.H; h += blockDim.x) {
        const int d = hdec[h];
        if (!d) continue;
        const int left = P.hused[h] - d;
        P.hused[h] = left;
        if (left == 0) {
          P.hstate[h] = kFree;
          atomicAdd(&s_freed, 1);
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) g_apply_ns[3] = (long long)globaltimer_ns();
    for (int e = threadIdx.x; e < ne; e += blockDim.x) ht_erase(P, P.row_req[P.s_evrows[e]]);
    if (threadIdx.x == 0) g_apply_ns[4] = (long long)globaltimer_ns();
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
  extern __shared__ __align__(16) unsigned char smem[];
  op_begin(P);
  __syncthreads();
  apply_core(P, ids, k, t, smem);
  publish(P);
}

// Fused reclaim, part 1 (grid over the handles, warp per handle): the distinct resident rows
// of every offline handle, laid out by handle id (s_rref + h*S, s_cnt[h]).  Spread over the
// whole GPU this is ~2 us; inside the single-CTA part 2 it was 32 warps x ~30 handles each.
__global__ void __launch_bounds__(256) k_reclaim_rows(PoolDev P) {
  const int lane = threadIdx.x & 31;
  const int h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) P.mirror->r[3] = (int64_t)globaltimer_ns();  // phase stamps
  if (h >= P.H || P.hstate[h] != kOffline) return;
  const int nc = (P.S + 31) >> 5;
  int cnt = 0;
  VALVE_DISPATCH_NC(nc, cnt = warp_distinct_rows<NC>(P, h, P.s_rref + (int64_t)h * P.S));
  if (lane == 0) P.s_cnt[h] = cnt;
}

// Fused reclaim, part 2 (sim.cpp:936-942): compact the offline handles (the snapshot), select
// k handles with the row costs, apply -- one CTA, after the instance rows are built.
__device__ void reclaim_body(const PoolDev& P, int k, int mode, int64_t t, unsigned char* smem) {
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
  if (threadIdx.x == 0) P.mirror->r[4] = (int64_t)globaltimer_ns();
  const Refs R{nullptr, P.s_cnt, P.S, P.s_hid};  // rows by handle id (k_reclaim_rows)
  if (mode == 1) {
    fifo_core(n, P.s_hid, P.s_hmap, k, P.s_pick);
  } else {
    greedy_select(n, P.s_hid, R, P.s_rref, P.R, P.row_cost, k, P.s_marg, P.s_taken, P.s_ev,
                  P.s_qoff, P.s_qcnt, P.s_qh, P.s_pick, smem, P.s_dense);  // leaves s_ev zeroed
  }
  __syncthreads();
  if (threadIdx.x == 0) P.mirror->r[5] = (int64_t)globaltimer_ns();
  apply_core(P, P.s_pick, k, t, smem, /*trusted=*/true);
  __syncthreads();
  if (threadIdx.x == 0) P.mirror->r[6] = (int64_t)globaltimer_ns();
  publish(P);
}

__global__ void __launch_bounds__(kNT) k_reclaim(PoolDev P, int k, int mode, int64_t t) {
  extern __shared__ __align__(16) unsigned char smem[];
  reclaim_body(P, k, mode, t, smem);
}

// The fused reclaim as ONE launch: ceil(H / 32) CTAs build the instance rows (warp per handle,
// as k_reclaim_rows), the last CTA to finish (ticket) runs part 2 and then stores `seq` into the
// pinned mirror after a system-scope fence, which the host polls instead of synchronizing.
__global__ void __launch_bounds__(kNT) k_reclaim_fused(PoolDev P, int k, int mode, int64_t t, int64_t seq) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int h = blockIdx.x * (kNT >> 5) + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) P.mirror->r[3] = (int64_t)globaltimer_ns();  // phase stamps
  if (h < P.H && P.hstate[h] == kOffline) {
    const int nc = (P.S + 31) >> 5;
    int cnt = 0;
    VALVE_DISPATCH_NC(nc, cnt = warp_distinct_rows<NC>(P, h, P.s_rref + (int64_t)h * P.S));
    if (lane == 0) P.s_cnt[h] = cnt;
  }
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(P.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *P.ticket = 0;  // ready for the next launch (stream-ordered)
  reclaim_body(P, k, mode, t, smem);  // ends in publish(): stores P.seq (== seq) into the mirror
  (void)seq;
}

// ---------------------------------------------------- selection over host instances

// ref request id -> index in the sorted cost keys (binary search), -1 when absent.
__global__ void k_map_refs(const int64_t* reqs, int nnz, const int64_t* keys, int m, int* rref) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int64_t v = reqs[e];
  int lo = 0, hi = m - 1, found = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int64_t kk = keys[mid];
    if (kk == v) {
      found = mid;
      break;
    }
    if (kk < v) lo = mid + 1;
    else hi = mid - 1;
  }
  rref[e] = found;
}

__global__ void __launch_bounds__(kNT) k_select_instance(SelectArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
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
  const Refs R{A.roff, nullptr, 0};
  if (A.mode == 0) {
    greedy_select(A.n, A.hid, R, A.rref, A.m, A.cost, A.k, A.marg, A.taken, A.ev, A.qoff, A.qcnt,
                  A.qh, A.out, smem);
  } else if (A.mode == 1) {
    fifo_core(A.n, A.hid, A.mapped, A.k, A.out);
  } else if (A.k > 0) {
    for (int i = threadIdx.x; i < A.n; i += blockDim.x) {
      int rank = 0;
      for (int j = 0; j < A.n; ++j) rank += A.hid[j] < A.hid[i] || (A.hid[j] == A.hid[i] && j < i);
      A.taken[rank] = A.hid[i];
      A.qcnt[i] = rank;  // position of handle i in sorted order
    }
    for (int r = threadIdx.x; r < A.m; r += blockDim.x) A.ev[r] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < A.n; i += blockDim.x)
      for (int e = A.roff[i]; e < A.roff[i + 1]; ++e)
        atomicOr(reinterpret_cast<unsigned*>(&A.ev[A.rref[e]]), 1u << A.qcnt[i]);
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
