// pool_device.cuh -- device helpers shared by the pool and reclaim kernels.
#pragma once
#include "valve_common.cuh"

namespace valve {

constexpr int kMaxChunks = 8;  // handle_size_pages <= 256 = 8 warp-width chunks

__device__ __forceinline__ void set_err(const PoolDev& P, int code, int detail, int64_t arg) {
  P.mirror->err = code;
  P.mirror->err_detail = detail;
  P.mirror->err_arg = arg;
}

// Thread 0 publishes the counters to the pinned mirror; every thread calls it last.
__device__ __forceinline__ void publish(const PoolDev& P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    P.mirror->n_free = P.hdr->n_free;
    P.mirror->n_online = P.hdr->n_online;
    P.mirror->n_offline = P.hdr->n_offline;
    __threadfence_system();
    P.mirror->done_seq = P.seq;  // after the fence: the host reads the results once it sees this
  }
}

__device__ __forceinline__ void op_begin(const PoolDev& P) {
  if (threadIdx.x == 0) {
    P.mirror->err = 0;
    P.mirror->err_detail = 0;
    P.mirror->err_arg = 0;
  }
}

// One warp holds the S slot rows of a handle in registers: v[c] = slot c*32 + lane.
// NC = number of 32-slot chunks (compile time, so the rows stay in registers).
template <int NC>
struct WarpRows {
  int v[NC];
  unsigned first;  // bit c: this lane's slot in chunk c is the first occurrence of its row
};

template <int NC>
__device__ __forceinline__ void warp_load_rows(const PoolDev& P, int h, WarpRows<NC>& w) {
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)h * P.S;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int s = c * 32 + lane;
    w.v[c] = s < P.S ? P.slot_row[base + s] : -1;
  }
}

// First-occurrence flags: the lowest slot of each distinct row (match.any within a chunk,
// shuffles against the earlier chunks).  Returns the distinct count (warp-uniform).
template <int NC>
__device__ __forceinline__ int warp_dedup(WarpRows<NC>& w) {
  const int lane = threadIdx.x & 31;
  w.first = 0;
  int cnt = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int v = w.v[c];
    const unsigned m = __match_any_sync(kFull, v);
    bool f = v >= 0 && (__ffs(m) - 1) == lane;
#pragma unroll
    for (int c2 = 0; c2 < c; ++c2)
#pragma unroll 4
      for (int j = 0; j < 32; ++j) f &= __shfl_sync(kFull, w.v[c2], j) != v;
    if (f) w.first |= 1u << c;
    cnt += __popc(__ballot_sync(kFull, f));
  }
  return cnt;
}

// Rank of this lane's chunk-c entry among the first-flagged values (ascending key).
template <int NC>
__device__ __forceinline__ int warp_rank64(const WarpRows<NC>& w, const int64_t (&key)[NC], int64_t mine) {
  int rank = 0;
#pragma unroll
  for (int c2 = 0; c2 < NC; ++c2) {
    const unsigned fm = __ballot_sync(kFull, (w.first >> c2) & 1u);
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const int64_t other = __shfl_sync(kFull, key[c2], j);
      rank += ((fm >> j) & 1u) && other < mine;
    }
  }
  return rank;
}

// Sorted distinct request ids resident on handle h -> out[0..cnt); returns cnt.  One warp.
template <int NC>
__device__ __forceinline__ int warp_sorted_residents(const PoolDev& P, int h, int64_t* out) {
  WarpRows<NC> w;
  warp_load_rows<NC>(P, h, w);
  const int cnt = warp_dedup<NC>(w);
  int64_t key[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) key[c] = w.v[c] >= 0 ? P.row_req[w.v[c]] : 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int rank = warp_rank64<NC>(w, key, key[c]);
    if ((w.first >> c) & 1u) out[rank] = key[c];
  }
  return cnt;
}

// Distinct resident rows of handle h -> out[0..cnt) (slot order); returns cnt.  One warp.
template <int NC>
__device__ __forceinline__ int warp_distinct_rows(const PoolDev& P, int h, int* out) {
  const int lane = threadIdx.x & 31;
  WarpRows<NC> w;
  warp_load_rows<NC>(P, h, w);
  const int cnt = warp_dedup<NC>(w);
  int pos = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const bool f = (w.first >> c) & 1u;
    const unsigned m = __ballot_sync(kFull, f);
    if (f) out[pos + __popc(m & ((1u << lane) - 1))] = w.v[c];
    pos += __popc(m);
  }
  return cnt;
}

// Runtime chunk count -> template instance.
#define VALVE_DISPATCH_NC(nc, EXPR)          \
  switch (nc) {                              \
    case 1: { constexpr int NC = 1; EXPR; } break; \
    case 2: { constexpr int NC = 2; EXPR; } break; \
    case 3:                                  \
    case 4: { constexpr int NC = 4; EXPR; } break; \
    default: { constexpr int NC = 8; EXPR; } break; \
  }

// Frees every live page of `row` (memory.cpp:99-114); emptied handles go free.  Block
// table entries become `bt_fill` (-1 for a normal release, the quarantine page after a
// reclaim).  Every thread of the CTA participates; s_freed counts freed handles.
__device__ __forceinline__ void release_row_pages(const PoolDev& P, int row, int bt_fill,
                                                  int* s_freed) {
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
}

}  // namespace valve
