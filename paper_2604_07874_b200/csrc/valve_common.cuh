// valve_common.cuh -- device data layout of the pool and CTA-wide primitives (sm_100a).
//
// The pool (colosim::MemoryPool, memory.hpp:19-98) lives in HBM as structure-of-arrays:
//
//   per handle h < H      hstate u8, hmapped i64, hused i32 (reference used_slots)
//   per slot p < H*S      slot_row i32 (-1 free), slot_lid i32 (logical id the reference
//                         reports; aliases -- memory.cpp:82-88), slot_blk i32 (block index
//                         inside the owning request)
//   per request row r < R row_req i64, row_cost i64, row_npages i32, row_nblk i32,
//                         bt[r*P + blk] i32 = physical page (h*S + slot) or the quarantine
//                         page H*S once reclaimed
//   req id -> row         open-addressing hash (linear probe, backward-shift delete)
//   free rows             FIFO ring (a reclaimed row is reused as late as possible, so a
//                         stale reader meets the quarantine page, not a new tenant)
//
// The handle sets free_/online_/offline_ of the reference are the hstate array; "lowest id
// first" is a CTA-wide exclusive scan over it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace valve {

constexpr int kNT = 1024;  // threads of the single-CTA bookkeeping kernels
constexpr uint8_t kFree = 0, kOnline = 1, kOffline = 2;
constexpr uint32_t kFull = 0xffffffffu;

enum ErrCode : int {
  kErrNone = 0,
  kErrInvalid = 1,
  kErrLogic = 2,
  kErrRuntime = 3,
  kErrOutOfRange = 5,
};

// Detail codes (err_detail) -> host message table (valve_host.cu).
enum ErrDetail : int {
  kDetNone = 0,
  kDetGrowExceeds,
  kDetRowsFull,
  kDetBlocksFull,
  kDetNotOffline,
  kDetApplyRange,
  kDetNoCost,
  kDetInvPartition,
  kDetInvOnline,
  kDetInvSlots,
  kDetInvNonOffline,
  kDetInvRow,
  kDetInvBlock,
  kDetTooManyEvicted,
};

struct PoolHdr {
  int n_free, n_online, n_offline;
  int ring_head, ring_tail;
  int live_rows;
  int tombstones;
};

// Small per-op result block in pinned host memory, written by the op's kernel.
struct Mirror {
  int n_free, n_online, n_offline;
  int err, err_detail;
  int pad;
  int64_t err_arg;
  int64_t r[8];
  int64_t copy_bytes;  // bytes the last apply/reclaim report asks the copy to move
  int copy_custom;     // 1 if some evicted request has its own page size (set_page_bytes)
  int pad2;
  volatile int64_t done_seq;  // sequence number of the last fused reclaim that finished (host spins on it)
};

struct PoolDev {
  int H, S, R, P, HC;  // handles, slots per handle, request rows, blocks per row, hash cap
  int quarantine;      // H*S
  uint8_t* hstate;
  int64_t* hmapped;
  int* hused;
  int* slot_row;
  int* slot_lid;
  int* slot_blk;
  int64_t* row_req;
  int64_t* row_cost;
  int64_t* row_pbytes;  // per-row page size (0 = pool page_bytes), e.g. 2 MiB weight pages
  int* row_npages;
  int* row_nblk;
  int* bt;
  int64_t* ht_key;
  int* ht_row;
  int* ring;
  PoolHdr* hdr;
  Mirror* mirror;  // device alias of the pinned mirror
  uint8_t* pages;
  int64_t slot_bytes, page_bytes;
  // scratch (sized for the worst case at creation)
  int* s_hid;        // [H]   instance handle ids / apply ids
  int64_t* s_hmap;   // [H]
  int* s_roff;       // [H+1]
  int* s_rref;       // [H*S] instance refs (rows)
  int* s_qoff;       // [R+1] reverse CSR
  int* s_qcnt;       // [max(R, H*S)]
  int* s_qh;         // [H*S]
  int64_t* s_marg;   // [H]
  int* s_taken;      // [H]
  int* s_ev;         // [R]   evicted flags (selection) / row marks (apply)
  int* s_pick;       // [H]
  int* s_evrows;     // [R]
  int* s_rank;       // [R]
  uint64_t* s_key;   // [pow2(H*S)]
  int* s_pay;        // [pow2(H*S)]
  int* s_cnt;        // [H]
  int* s_dense;      // [R] row -> dense request index during a greedy re-index; -1 between calls
  int64_t seq;       // this launch's completion sequence (publish() stores it into the mirror)
  unsigned* ticket;  // [1] CTAs of the fused reclaim's instance pass that finished (last one goes on)
  int* s_tphys;      // [H*S] apply tuples: physical page
  int* s_tblk;       // [H*S] apply tuples: block index
  // results of the last apply / reclaim (device copies; the copy kernel reads res_phys)
  int* res_handles;     // [H]
  int64_t* res_evicted; // [R]
  int* res_inv_off;     // [R+1]
  int64_t* res_pages;   // [H*S]
  int* res_phys;        // [H*S]
  int* res_blk;         // [H*S]
  int* res_counts;      // [4] n_handles, n_evicted, n_pages, err
  int64_t* res_ev_pbytes;  // [R]   page size of each evicted request (report order)
  int64_t* res_ev_base;    // [R+1] destination byte offset of each evicted request's pages
  int64_t* res_ev_cbase;   // [R+1] copy-chunk prefix (per copy launch, variable-size path)
};

// ----------------------------------------------------------------------------- helpers

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d4a2fa9fb8476dULL;
  return x ^ (x >> 31);
}

// Word w of block b of request r (the deterministic KV image; matches vo_page_word).
__device__ __forceinline__ uint64_t page_word_base(int64_t req, int blk) {
  return splitmix64((uint64_t)req) ^ ((uint64_t)(uint32_t)blk << 40);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// CTA-wide exclusive scan; every thread must call.  Returns the exclusive prefix and
// the CTA total.
__device__ __forceinline__ int block_excl_scan(int v, int& total) {
  __shared__ int ws[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int x = lane < nw ? ws[lane] : 0;
    x = warp_incl_scan(x);
    ws[lane] = x;
  }
  __syncthreads();
  const int base = wid ? ws[wid - 1] : 0;
  total = ws[nw - 1];
  __syncthreads();
  return base + inc - v;
}

__device__ __forceinline__ int64_t block_excl_scan64(int64_t v, int64_t& total) {
  __shared__ int64_t ws64x[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t n = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) ws64x[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t x = lane < nw ? ws64x[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t n = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += n;
    }
    ws64x[lane] = x;
  }
  __syncthreads();
  const int64_t base = wid ? ws64x[wid - 1] : 0;
  total = ws64x[nw - 1];
  __syncthreads();
  return base + inc - v;
}

__device__ __forceinline__ int block_sum(int v) {
  int total;
  block_excl_scan(v, total);
  return total;
}

__device__ __forceinline__ int64_t block_sum64(int64_t v) {
  __shared__ int64_t ws64[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  if (lane == 0) ws64[wid] = v;
  __syncthreads();
  int64_t s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s += ws64[i];
  __syncthreads();
  if (threadIdx.x == 0) ws64[0] = s;
  __syncthreads();
  s = ws64[0];
  __syncthreads();
  return s;
}

// Lexicographic (value, id, idx) minimum over the CTA; idx = -1 means "none".
struct ArgMin {
  int64_t v;
  int id;
  int idx;
};
__device__ __forceinline__ bool argmin_less(const ArgMin& a, const ArgMin& b) {
  if (a.idx < 0) return false;
  if (b.idx < 0) return true;
  if (a.v != b.v) return a.v < b.v;
  if (a.id != b.id) return a.id < b.id;
  return a.idx < b.idx;
}
__device__ __forceinline__ ArgMin block_argmin(ArgMin a) {
  __shared__ ArgMin wa[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMin b;
    b.v = __shfl_down_sync(kFull, a.v, o);
    b.id = __shfl_down_sync(kFull, a.id, o);
    b.idx = __shfl_down_sync(kFull, a.idx, o);
    if (argmin_less(b, a)) a = b;
  }
  if (lane == 0) wa[wid] = a;
  __syncthreads();
  if (wid == 0) {
    a = lane < nw ? wa[lane] : ArgMin{0, 0, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMin b;
      b.v = __shfl_down_sync(kFull, a.v, o);
      b.id = __shfl_down_sync(kFull, a.id, o);
      b.idx = __shfl_down_sync(kFull, a.idx, o);
      if (argmin_less(b, a)) a = b;
    }
    if (lane == 0) wa[0] = a;
  }
  __syncthreads();
  a = wa[0];
  __syncthreads();
  return a;
}

// CTA-wide bitonic sort of n u64 keys (+ int payload) in place; buffers must hold
// next_pow2(n) entries (the tail is padded with UINT64_MAX here).
__device__ __forceinline__ void block_bitonic_sort(uint64_t* key, int* pay, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + threadIdx.x; i < N; i += blockDim.x) {
    key[i] = ~0ull;
    pay[i] = -1;
  }
  __syncthreads();
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (N >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t a = key[lo], b = key[hi];
        if ((a > b) == asc) {
          key[lo] = b;
          key[hi] = a;
          const int t = pay[lo];
          pay[lo] = pay[hi];
          pay[hi] = t;
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------ request table

__device__ __forceinline__ int ht_slot(int64_t key, int HC) {
  return (int)(splitmix64((uint64_t)key) & (uint64_t)(HC - 1));
}

// Request table: linear probing over HC = 2R slots; ht_row = row, -1 empty, -2 tombstone.
// Deletes leave tombstones so that the erasures of a reclaim can run in parallel (one thread
// per evicted request); ht_rebuild() compacts the table when tombstones pile up.
constexpr int kEmpty = -1, kTomb = -2;

// Lookup (any thread); returns the row or -1.
__device__ __forceinline__ int ht_find(const PoolDev& P, int64_t key) {
  const int mask = P.HC - 1;
  for (int i = ht_slot(key, P.HC), probes = 0; probes < P.HC; i = (i + 1) & mask, ++probes) {
    const int r = P.ht_row[i];
    if (r == kEmpty) return -1;
    if (r >= 0 && P.ht_key[i] == key) return r;
  }
  return -1;
}

// Single-thread insert of a new key (caller checked absence); pops a row from the ring.
__device__ __forceinline__ int ht_insert(const PoolDev& P, int64_t key) {
  PoolHdr* h = P.hdr;
  if (h->ring_tail - h->ring_head <= 0) return -1;
  const int row = P.ring[h->ring_head % P.R];
  h->ring_head++;
  h->live_rows++;
  const int mask = P.HC - 1;
  int i = ht_slot(key, P.HC);
  while (P.ht_row[i] >= 0) i = (i + 1) & mask;
  if (P.ht_row[i] == kTomb) h->tombstones--;
  P.ht_key[i] = key;
  P.ht_row[i] = row;
  P.row_req[row] = key;
  P.row_cost[row] = 0;
  P.row_pbytes[row] = 0;
  P.row_npages[row] = 0;
  P.row_nblk[row] = 0;
  return row;
}

// Delete (safe for distinct keys in parallel): tombstone the slot, push the row to the ring.
__device__ __forceinline__ void ht_erase(const PoolDev& P, int64_t key) {
  const int mask = P.HC - 1;
  int i = ht_slot(key, P.HC);
  for (int probes = 0;; i = (i + 1) & mask, ++probes) {
    const int r = P.ht_row[i];
    if (r == kEmpty || probes >= P.HC) return;
    if (r >= 0 && P.ht_key[i] == key) break;
  }
  const int row = P.ht_row[i];
  P.ht_row[i] = kTomb;
  PoolHdr* h = P.hdr;
  atomicAdd(&h->tombstones, 1);
  P.ring[atomicAdd(&h->ring_tail, 1) % P.R] = row;
  atomicSub(&h->live_rows, 1);
  P.row_npages[row] = 0;
  P.row_nblk[row] = 0;
}

// CTA-wide compaction: gather the live rows, clear, re-insert (CAS probing).  `scratch`
// holds >= R ints.  Every thread calls.
__device__ __forceinline__ void ht_rebuild(const PoolDev& P, int* scratch) {
  __shared__ int s_n;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < P.HC; i += blockDim.x) {
    const int r = P.ht_row[i];
    if (r >= 0) scratch[atomicAdd(&s_n, 1)] = r;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P.HC; i += blockDim.x) P.ht_row[i] = kEmpty;
  __syncthreads();
  const int mask = P.HC - 1;
  for (int j = threadIdx.x; j < s_n; j += blockDim.x) {
    const int row = scratch[j];
    const int64_t key = P.row_req[row];
    int i = ht_slot(key, P.HC);
    while (atomicCAS(&P.ht_row[i], kEmpty, row) != kEmpty) i = (i + 1) & mask;
    P.ht_key[i] = key;
  }
  __syncthreads();
  if (threadIdx.x == 0) P.hdr->tombstones = 0;
  __syncthreads();
}

}  // namespace valve
